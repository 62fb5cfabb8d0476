// clv_anneal.cu -- K3 (GED<=4 neighbour generation + incremental scoring) fused
// with K4 (warp-shuffle argmax) and K5 (anneal step): one thread-block CLUSTER
// per annealing chain, every step of every chain inside one persistent launch.
//
// Reference semantics: sample_neighbor, anneal
// (SPEC:461-469, 478-483), Eqs. 6-7.  Step definition: DESIGN.md
// "Chain step"; CPU restatement: oracle/anneal.py + oracle/neighbours.py.
//
// Per CTA (shared memory): per-edge addition rows {thr, acc, en, idle} held as
// fp64 *integers* (exact: every partial sum < 2^53, so any summation order
// gives the same bits as the oracle's int64 W @ rows), latency-rank bits,
// adjacency masks and memory-feasible neighbour lists; the centre; and per
// step the removal table -- one entry per present edge (singles) and per
// available removal pair (doubles) carrying the removal deltas, the presence
// mask after removal and the canonical index base.  A neighbour is then
//   S' = S + removal.d + row[a1] (+ row[a2]),  mask' = removal.m | bit(a1) | bit(a2)
// followed by the fp64 epilogue.  Every CTA of the cluster builds identical
// tables (ordered compaction) and scores a strided share of the move space;
// CTA records meet in the leader CTA over DSMEM; the leader applies Eq. 7 and
// broadcasts the accepted move, which every CTA applies to its own centre.
#include <cooperative_groups.h>
#include <cstdlib>
#include <math_constants.h>
#include "clv_internal.h"

namespace cg = cooperative_groups;

namespace clv {

constexpr int ANT = 256;                  // threads per CTA
constexpr int NWARP = ANT / 32;
constexpr int MAXP = CLV_MAX_EDGES * (CLV_MAX_EDGES + 1) / 2;   // 820 removal pairs
constexpr int MAXCL = 16;
constexpr long long NOIDX = -1;

enum { MODE_BEST_ALL = 0, MODE_UNIFORM_ALL = 1, MODE_UNIFORM_PROPOSAL = 2 };

struct __align__(16) ARow {
    double thr, acc, en, idle;
};

struct __align__(8) RemEnt {            // one removal multiset R (single edge or pair), 40 B
    float f0, f1, f2, f3;                  // -(rows of R) in fp32 (screening)
    unsigned long long mR;                 // presence mask (by latency rank) after removal
    int pre;                               // doubles: exclusive prefix of list lengths
    int off;                               // doubles: first entry of the static move list
    unsigned short p;                      // pair index P(r1, r2) (doubles) / edge (singles)
    unsigned short code;                   // slice code of R: sr1*125 + sr2*25 (doubles), sr*5 (singles)
    unsigned char len;                     // doubles: move-list length
    unsigned char r1, r2;                  // removed edges (r2 = 0xFF for singles)
};

struct KRec {                              // (key, idx) record; payload hv (uniform proposals)
    unsigned long long key;
    int idx;                               // canonical indices are < 2^31
    double hv;
};

__device__ __forceinline__ bool krec_less(unsigned long long ka, int ia, const KRec &b) {
    return ka < b.key || (ka == b.key && ia < b.idx);
}
__device__ __forceinline__ KRec krec_none() {
    KRec r; r.key = ~0ULL; r.idx = 0x7FFFFFFF; r.hv = 0.0; return r;
}
template <bool PAYLOAD>
__device__ __forceinline__ KRec krec_min_warp(KRec r) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        KRec o;
        o.key = __shfl_xor_sync(0xFFFFFFFFu, r.key, m);
        o.idx = __shfl_xor_sync(0xFFFFFFFFu, r.idx, m);
        o.hv = PAYLOAD ? __shfl_xor_sync(0xFFFFFFFFu, r.hv, m) : 0.0;
        if (krec_less(o.key, o.idx, r)) r = o;
    }
    return r;
}

struct __align__(16) AnnealSmem {
    ARow row[CLV_MAX_EDGES];
    float4 rowf[CLV_MAX_EDGES];            // fp32 copies of the rows (screening only)
    double lat_by_rank[CLV_MAX_EDGES];
    float latf_by_rank[CLV_MAX_EDGES];
    float Sf[4];                           // fp32 copy of the centre sums
    float ecf[16];                         // fp32 screening constants (EC_*)
    unsigned long long rbit[CLV_MAX_EDGES];
    unsigned long long adjm[CLV_MAX_EDGES];
    EvalConst ec;
    unsigned long long mem_ok;
    short Pt[CLV_MAX_EDGES + 1];           // P(x, y) = Pt[x] + y
    unsigned char sl[CLV_MAX_EDGES];
    unsigned short pair_tab[MAXP];
    int pair_off[MAXP];                    // static move lists (staged from FamilyTables)
    unsigned char pair_len[MAXP];
    // centre
    int w[CLV_MAX_EDGES];
    double S[4];
    int svec[CLV_K];
    unsigned long long pmask;
    // per-step tables
    RemEnt se[CLV_MAX_EDGES];
    int nPE, nRP, nLen;
    int warp_off[NWARP + 1];
    int warp_len[NWARP + 1];
    int fsvec[CLV_K];                      // slice vector the feasibility bytes belong to
    unsigned char feasS[25];
    unsigned char feasD[625];
    // per-warp queues of screening survivors (removal index, list entry)
    unsigned short qj[NWARP][64];
    uint32_t qe[NWARP][64];
    // reduction
    KRec wS[NWARP], wV[NWARP], wP[NWARP];
    unsigned long long wc[NWARP];
    // leader-only slots, one per cluster rank
    KRec slS[2][MAXCL], slV[2][MAXCL], slP[2][MAXCL];   // [step parity][cluster rank]
    unsigned long long slc[2][MAXCL];
    long long dec_move;                    // accepted move index, -1 = none
    int dec_done;
    int bw[CLV_MAX_EDGES];
};

__device__ __forceinline__ double lmax_of(const AnnealSmem &s, unsigned long long m) {
    return s.lat_by_rank[63 - __clzll((long long)m)];
}

// canonical index -> move (r1, r2, a1, a2; 0xFF = absent)
__device__ inline void decode_move(const AnnealSmem &s, int E, long long idx64, int &r1, int &r2, int &a1, int &a2) {
    const unsigned idx = (unsigned)idx64;          // canonical indices are < 2^31
    if (idx < (unsigned)(E * E)) {
        r1 = (int)(idx / (unsigned)E); a1 = (int)(idx - (unsigned)r1 * E); r2 = 0xFF; a2 = 0xFF;
        return;
    }
    const unsigned NP = (unsigned)(E * (E + 1) / 2);
    const unsigned u = idx - (unsigned)(E * E);
    const int p = (int)(u / NP), q = (int)(u - (unsigned)p * NP);
    r1 = s.pair_tab[p] & 0xFF; r2 = s.pair_tab[p] >> 8;
    a1 = s.pair_tab[q] & 0xFF; a2 = s.pair_tab[q] >> 8;
}

__device__ inline Score score_move(const AnnealSmem &s, int r1, int r2, int a1, int a2) {
    double t = s.S[0], ac = s.S[1], en = s.S[2], id = s.S[3];
    unsigned long long m = s.pmask;
    int e[2] = {r1, r2};
    for (int k = 0; k < 2; ++k) {
        if (e[k] == 0xFF) continue;
        t -= s.row[e[k]].thr; ac -= s.row[e[k]].acc; en -= s.row[e[k]].en; id -= s.row[e[k]].idle;
    }
    if (r1 != 0xFF && s.w[r1] - 1 - (r2 == r1 ? 1 : 0) == 0) m &= ~s.rbit[r1];
    if (r2 != 0xFF && r2 != r1 && s.w[r2] - 1 == 0) m &= ~s.rbit[r2];
    int f[2] = {a1, a2};
    for (int k = 0; k < 2; ++k) {
        if (f[k] == 0xFF) continue;
        t += s.row[f[k]].thr; ac += s.row[f[k]].acc; en += s.row[f[k]].en; id += s.row[f[k]].idle;
        m |= s.rbit[f[k]];
    }
    return epilogue_d(t, ac, en, id, lmax_of(s, m), s.ec);
}

// Apply a move to the CTA-local centre (thread 0) -- O(1).
__device__ inline void apply_move(AnnealSmem &s, int E, long long idx) {
    int r[2], a[2];
    decode_move(s, E, idx, r[0], r[1], a[0], a[1]);
    for (int k = 0; k < 2; ++k) {
        if (r[k] == 0xFF) continue;
        int e = r[k];
        s.w[e] -= 1;
        s.S[0] -= s.row[e].thr; s.S[1] -= s.row[e].acc; s.S[2] -= s.row[e].en; s.S[3] -= s.row[e].idle;
        s.svec[s.sl[e]] -= 1;
        if (s.w[e] == 0) s.pmask &= ~s.rbit[e];
    }
    for (int k = 0; k < 2; ++k) {
        if (a[k] == 0xFF) continue;
        int e = a[k];
        s.w[e] += 1;
        s.S[0] += s.row[e].thr; s.S[1] += s.row[e].acc; s.S[2] += s.row[e].en; s.S[3] += s.row[e].idle;
        s.svec[s.sl[e]] += 1;
        s.pmask |= s.rbit[e];
    }
}

// Per-step tables: ordered (deterministic) compaction of the removal pairs and
// present edges -- every CTA of the cluster must build identical tables because
// the cluster partitions the move space by table position -- plus the
// feasibility bytes of all 25 single / 625 double slice deltas.
__device__ __forceinline__ void prepare_step(AnnealSmem &s, RemEnt *rp, const FamilyTables &T, int E, int n,
                                             const FeasView &F) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int NP = E * (E + 1) / 2;
    const int PER = (NP + ANT - 1) / ANT;          // consecutive pairs per thread (<= 4)
    bool refresh = false;
#pragma unroll
    for (int k = 0; k < CLV_K; ++k) refresh |= (s.svec[k] != s.fsvec[k]);
    if (threadIdx.x < 4) s.Sf[threadIdx.x] = (float)s.S[threadIdx.x];
    bool fres[3] = {false, false, false};
    if (refresh) {                                 // uniform across the CTA
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const int t = threadIdx.x + q * ANT;
            if (t >= 650) continue;
            int v[CLV_K];
#pragma unroll
            for (int k = 0; k < CLV_K; ++k) v[k] = s.svec[k];
            bool ok;
            if (t < 25) {
                v[t / 5] -= 1; v[t % 5] += 1;
                ok = v[t / 5] >= 0;
            } else {
                const int u = t - 25;
                v[u / 125] -= 1; v[(u / 25) % 5] -= 1; v[(u / 5) % 5] += 1; v[u % 5] += 1;
                ok = v[0] >= 0 && v[1] >= 0 && v[2] >= 0 && v[3] >= 0 && v[4] >= 0;
            }
            fres[q] = ok && feasible(F, n, v[0], v[1], v[2], v[3], v[4]);
        }
    }
    const int p0 = threadIdx.x * PER;
    int cnt = 0, lsum = 0;
    for (int p = p0; p < p0 + PER && p < NP; ++p) {
        const int x = s.pair_tab[p] & 0xFF, y = s.pair_tab[p] >> 8;
        const bool ok = (x == y) ? (s.w[x] >= 2) : (s.w[x] > 0 && s.w[y] > 0);
        if (ok) { ++cnt; lsum += s.pair_len[p]; }
    }
    // block exclusive scan of (cnt, lsum) in thread order
    int ic = cnt, il = lsum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int yc = __shfl_up_sync(0xFFFFFFFFu, ic, d), yl = __shfl_up_sync(0xFFFFFFFFu, il, d);
        if (lane >= d) { ic += yc; il += yl; }
    }
    if (lane == 31) { s.warp_off[wid] = ic; s.warp_len[wid] = il; }
    __syncthreads();
    if (threadIdx.x < 32) {
        int c = lane < NWARP ? s.warp_off[lane] : 0, l = lane < NWARP ? s.warp_len[lane] : 0;
        int c2 = c, l2 = l;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int yc = __shfl_up_sync(0xFFFFFFFFu, c2, d), yl = __shfl_up_sync(0xFFFFFFFFu, l2, d);
            if (lane >= d) { c2 += yc; l2 += yl; }
        }
        if (lane < NWARP) { s.warp_off[lane] = c2 - c; s.warp_len[lane] = l2 - l; }
        if (lane == NWARP - 1) { s.nRP = c2; s.nLen = l2; }
    }
    __syncthreads();
    int pos = s.warp_off[wid] + ic - cnt, lpos = s.warp_len[wid] + il - lsum;
    for (int p = p0; p < p0 + PER && p < NP; ++p) {
        const int x = s.pair_tab[p] & 0xFF, y = s.pair_tab[p] >> 8;
        const bool ok = (x == y) ? (s.w[x] >= 2) : (s.w[x] > 0 && s.w[y] > 0);
        if (!ok) continue;
        RemEnt &r = rp[pos++];
        r.f0 = -(s.rowf[x].x + s.rowf[y].x); r.f1 = -(s.rowf[x].y + s.rowf[y].y);
        r.f2 = -(s.rowf[x].z + s.rowf[y].z); r.f3 = -(s.rowf[x].w + s.rowf[y].w);
        unsigned long long m = s.pmask;
        if (x == y) { if (s.w[x] == 2) m &= ~s.rbit[x]; }
        else {
            if (s.w[x] == 1) m &= ~s.rbit[x];
            if (s.w[y] == 1) m &= ~s.rbit[y];
        }
        r.mR = m;
        r.p = (unsigned short)p;
        r.off = s.pair_off[p];
        r.len = s.pair_len[p];
        r.pre = lpos;
        lpos += r.len;
        r.code = (unsigned short)(s.sl[x] * 125 + s.sl[y] * 25);
        r.r1 = (unsigned char)x; r.r2 = (unsigned char)y;
    }
    if (wid == 0) {
        int c = 0;
        for (int e0 = 0; e0 < E; e0 += 32) {
            const int e = e0 + lane;
            const bool ok = e < E && s.w[e] > 0;
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, ok);
            if (ok) {
                RemEnt &r = s.se[c + __popc(bal & ((1u << lane) - 1u))];
                r.f0 = -s.rowf[e].x; r.f1 = -s.rowf[e].y; r.f2 = -s.rowf[e].z; r.f3 = -s.rowf[e].w;
                r.mR = (s.w[e] == 1) ? (s.pmask & ~s.rbit[e]) : s.pmask;
                r.p = (unsigned short)e;
                r.code = (unsigned short)(s.sl[e] * 5);
                r.r1 = (unsigned char)e; r.r2 = 0xFF; r.off = 0; r.len = 0; r.pre = 0;
            }
            c += __popc(bal);
        }
        if (lane == 0) s.nPE = c;
    }
    // slice-delta feasibility: only when the centre's slice multiset changed
    // (variant swaps keep it).  The loads were issued at the top of prepare_step.
    if (refresh) {
        for (int q = 0; q < 3; ++q) {
            const int t = threadIdx.x + q * ANT;
            if (t < 25) s.feasS[t] = fres[q];
            else if (t < 650) s.feasD[t - 25] = fres[q];
        }
        if (threadIdx.x < CLV_K) s.fsvec[threadIdx.x] = s.svec[threadIdx.x];
    }
    __syncthreads();
}

// fp32 screening bound: a candidate is scored exactly
// only if its fp32 estimate, widened by a generous error bound, could beat the
// thread's current record of its SLA class (or, for uniform proposals, if its hash
// would become the proposal).  Records are exact minima of the exactly scored
// candidates, and a skipped candidate is provably worse than a scored one, so the
// selection is bit-identical to scoring everything.
enum { EC_RQ = 0, EC_ENS, EC_IDLE, EC_RSAT, EC_C0, EC_C1, EC_C2, EC_SLO, EC_RSLO, EC_STRICT, EC_MAG, EC_N };

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// fp32 estimate of (f, L) with error bounds; true when the candidate provably cannot
// beat the bound of its SLA class (bS: SLA-meeting, bV: violating).
//   f = c0 + c1*E + c2*A  with c0 = 100*lam - (1-lam)*A_base*kA, c1 = -lam*kC, c2 = (1-lam)*kA
// The bound M ~ 2^-14 of the magnitudes covers fp32 rounding of the sums (<= 2.4e-7
// relative), of rcp.approx (<= 1 ulp) and of every product (~1e-6 total).
__device__ __forceinline__ bool screen_out(const float *c, float t, float ac, float en, float id, float lmax,
                                           double bS, double bV) {
    const float inv = rcp_approx(t);
    const float A = ac * inv;
    const float rho = c[EC_RQ] * inv;
    const float E = __fmaf_rn((1.0f - fminf(rho, 1.0f)) * id, c[EC_IDLE], (en * inv) * c[EC_ENS]);
    const float rx = rcp_approx(1.0f - fminf(rho, c[EC_RSAT]));
    const float L = lmax * rx;
    const float tE = c[EC_C1] * E, tA = c[EC_C2] * A;
    const float f = c[EC_C0] + tE + tA;
    const float M = 6.1e-5f * (c[EC_MAG] + fabsf(tE) + fabsf(tA));
    const float relL = 4e-6f * (2.0f + rx);
    const float slo = c[EC_SLO];
    if (L * (1.0f + relL) < slo) return (double)(-f - M) > bS;        // SLA surely met: h = -f
    if (L * (1.0f - relL) > slo && fabsf(f) > M) {                   // surely violated, sign of f sure
        const float q = (f >= 0.0f || c[EC_STRICT] != 0.0f) ? slo * rcp_approx(L) : L * c[EC_RSLO];
        const float h = -f * q;
        return (double)(h - 1.02f * q * (M + fabsf(f) * 2.0f * relL) - 1e-5f * fabsf(h)) > bV;
    }
    return false;
}

// Exact score of one double move + record update (the compacted survivors).
template <int MODE>
__device__ __forceinline__ void exact_pair(const AnnealSmem &s, const RemEnt &R, uint32_t ent, int idx, KRec &rS,
                                           KRec &rV, bool pair = true) {
    const int a1 = ent & 63, a2 = (ent >> 6) & 63;
    const ARow &A1 = s.row[a1], &X = s.row[R.r1];
    double t = s.S[0] - X.thr + A1.thr, ac = s.S[1] - X.acc + A1.acc, en = s.S[2] - X.en + A1.en,
           id = s.S[3] - X.idle + A1.idle;
    if (R.r2 != 0xFF) {
        const ARow &Y = s.row[R.r2];
        t -= Y.thr; ac -= Y.acc; en -= Y.en; id -= Y.idle;
    }
    unsigned long long m = R.mR | s.rbit[a1];
    if (pair) {
        const ARow &A2 = s.row[a2];
        t += A2.thr; ac += A2.acc; en += A2.en; id += A2.idle;
        m |= s.rbit[a2];
    }
    const Score sc = epilogue_d(t, ac, en, id, s.lat_by_rank[63 - __clzll((long long)m)], s.ec);
    const unsigned long long key = okey(sc.h);
    if (sc.sla) { if (krec_less(key, idx, rS)) { rS.key = key; rS.idx = idx; rS.hv = sc.h; } }
    else        { if (krec_less(key, idx, rV)) { rV.key = key; rV.idx = idx; rV.hv = sc.h; } }
}

template <int MODE, bool PAIR>
__device__ __forceinline__ void consider(const AnnealSmem &s, const RemEnt &R, int a1, int a2, int idx,
                                         KRec &rS, KRec &rV, KRec &rP, uint64_t seed, uint64_t gchain,
                                         uint64_t k) {
    if (MODE == MODE_UNIFORM_PROPOSAL) {
        const unsigned long long hk = derive_seed4(seed, gchain, k, (uint64_t)idx + 1);
        if (krec_less(hk, idx, rP)) { rP.key = hk; rP.idx = idx; }
        return;
    }
    unsigned long long hk = 0;
    bool wantP = false;
    if (MODE == MODE_UNIFORM_ALL) {
        hk = derive_seed4(seed, gchain, k, (uint64_t)idx + 1);
        wantP = krec_less(hk, idx, rP);
    }
    const unsigned long long m = PAIR ? (R.mR | s.rbit[a1] | s.rbit[a2]) : (R.mR | s.rbit[a1]);
    const int top = 63 - __clzll((long long)m);
    if (!wantP) {
        const float4 x = s.rowf[a1];
        float t = s.Sf[0] + R.f0 + x.x, ac = s.Sf[1] + R.f1 + x.y, en = s.Sf[2] + R.f2 + x.z, id = s.Sf[3] + R.f3 + x.w;
        if (PAIR) {
            const float4 y = s.rowf[a2];
            t += y.x; ac += y.y; en += y.z; id += y.w;
        }
        if (screen_out(s.ecf, t, ac, en, id, s.latf_by_rank[top], rS.key != ~0ULL ? rS.hv : CUDART_INF,
                       rV.key != ~0ULL ? rV.hv : CUDART_INF)) return;
    }
    const ARow &A1 = s.row[a1], &X = s.row[R.r1];
    double t = s.S[0] - X.thr + A1.thr, ac = s.S[1] - X.acc + A1.acc, en = s.S[2] - X.en + A1.en,
           id = s.S[3] - X.idle + A1.idle;
    if (PAIR) {
        const ARow &Y = s.row[R.r2];
        t -= Y.thr; ac -= Y.acc; en -= Y.en; id -= Y.idle;
        const ARow &A2 = s.row[a2];
        t += A2.thr; ac += A2.acc; en += A2.en; id += A2.idle;
    }
    const Score sc = epilogue_d(t, ac, en, id, s.lat_by_rank[top], s.ec);
    const unsigned long long key = okey(sc.h);
    if (sc.sla) { if (krec_less(key, idx, rS)) { rS.key = key; rS.idx = idx; rS.hv = sc.h; } }
    else        { if (krec_less(key, idx, rV)) { rV.key = key; rV.idx = idx; rV.hv = sc.h; } }
    if (MODE == MODE_UNIFORM_ALL && wantP) { rP.key = hk; rP.idx = idx; rP.hv = sc.h; }
}

// Optional phase profiler (CLV_ANNEAL_VARIANT=9): thread 0 of each CTA accumulates
// clock64 deltas between consecutive marks into args.prof[(chain*CL+rank)*8 + phase].
#define PROF_MARK(ph)                                                                  \
    if (PROF && threadIdx.x == 0) {                                                    \
        const long long _now = clock64();                                              \
        if ((ph) > 0) prof_acc[(ph) - 1] += _now - prof_last;                          \
        prof_last = _now;                                                              \
    }

template <int MODE, int MINB, int UNR, bool PROF = false>
__global__ void __launch_bounds__(ANT, MINB) anneal_kernel(const __grid_constant__ AnnealArgs args) {
    long long prof_acc[7] = {0, 0, 0, 0, 0, 0, 0};
    long long prof_last = 0;
    long long prof_surv = 0;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    AnnealSmem &s = *reinterpret_cast<AnnealSmem *>(smem_raw);
    RemEnt *const rp = reinterpret_cast<RemEnt *>(smem_raw + sizeof(AnnealSmem));   // dynamic tail, E(E+1)/2
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = (int)cluster.num_blocks();
    const int crank = (int)cluster.block_rank();
    const int chain = blockIdx.x / CL;
    if (chain >= args.n_chains) return;      // whole cluster exits together
    const uint64_t gchain = (uint64_t)(args.chain_base + chain);
    const FamilyTables &T = *args.fam;
    const int E = T.E;
    const int n = args.n;
    const int tid = threadIdx.x;

    // ---- stage tables
    for (int e = tid; e < E; e += ANT) {
        s.row[e].thr = (double)T.thr_q[e];
        s.row[e].acc = (double)T.acc_q[e];
        s.row[e].en = (double)T.en_q[e];
        s.row[e].idle = (double)T.idle_q[e % 5];
        s.lat_by_rank[e] = T.lat_by_rank[e];
        s.latf_by_rank[e] = (float)T.lat_by_rank[e];
        s.rowf[e] = make_float4((float)T.thr_q[e], (float)T.acc_q[e], (float)T.en_q[e], (float)T.idle_q[e % 5]);
        s.rbit[e] = 1ULL << T.rank[e];
        s.sl[e] = (unsigned char)(e % 5);
        unsigned long long am = 0;
        for (int x = 0; x < E; ++x)
            if (x != e && (x / 5 == e / 5 || x % 5 == e % 5)) am |= 1ULL << x;
        s.adjm[e] = am;
    }
    for (int x = tid; x <= E; x += ANT) s.Pt[x] = (short)(x * E - (x * (x - 1)) / 2 - x);
    for (int x = tid; x < E; x += ANT)
        for (int y = x; y < E; ++y) s.pair_tab[x * E - (x * (x - 1)) / 2 + (y - x)] = (unsigned short)(x | (y << 8));
    for (int p = tid; p < E * (E + 1) / 2; p += ANT) { s.pair_off[p] = T.pair_off[p]; s.pair_len[p] = T.pair_len[p]; }
    if (tid == 0) {
        s.mem_ok = T.mem_ok;
        s.ec = args.ec[args.n_ec == 1 ? 0 : chain];
        const EvalConst &c = s.ec;
        const double c0 = 100.0 * c.lam - (1.0 - c.lam) * c.a_base * c.kA;
        s.ecf[EC_RQ] = (float)c.R_q; s.ecf[EC_ENS] = (float)c.en_scale;
        s.ecf[EC_IDLE] = (float)(c.idle_scale * c.inv_3600R); s.ecf[EC_RSAT] = (float)c.rho_sat;
        s.ecf[EC_C0] = (float)c0; s.ecf[EC_C1] = (float)(-c.lam * c.kC); s.ecf[EC_C2] = (float)((1.0 - c.lam) * c.kA);
        s.ecf[EC_SLO] = (float)c.slo; s.ecf[EC_RSLO] = (float)(1.0 / c.slo); s.ecf[EC_STRICT] = (float)c.strict;
        s.ecf[EC_MAG] = (float)(fabs(100.0 * c.lam) + fabs((1.0 - c.lam) * c.a_base * c.kA));
    }
    __syncthreads();
    if (tid == 0) {
        const uint16_t *w0 = args.start_w + (size_t)chain * E;
        double S0 = 0, S1 = 0, S2 = 0, S3 = 0;
        unsigned long long m = 0;
        for (int k = 0; k < CLV_K; ++k) s.svec[k] = 0;
        for (int e = 0; e < E; ++e) {
            const int x = w0[e];
            s.w[e] = x;
            S0 += x * s.row[e].thr; S1 += x * s.row[e].acc; S2 += x * s.row[e].en; S3 += x * s.row[e].idle;
            s.svec[e % 5] += x;
            if (x > 0) m |= s.rbit[e];
        }
        s.S[0] = S0; s.S[1] = S1; s.S[2] = S2; s.S[3] = S3;
        s.pmask = m;
        for (int k = 0; k < CLV_K; ++k) s.fsvec[k] = -1;
    }
    __syncthreads();

    // ---- leader state (thread 0 of rank 0)
    const bool leader = (crank == 0 && tid == 0);
    double hc = 0.0;
    unsigned int bk1 = 0;
    unsigned long long bk2 = 0;
    int best_step = -1, stall = 0, steps = 0, status = 0;
    long long best_idx = -1, evals = 1;
    if (tid == 0) {
        int invalid = 0;
        long long tot = 0;
        for (int e = 0; e < E; ++e) {
            tot += s.w[e];
            if (s.w[e] > 0 && !((s.mem_ok >> e) & 1ULL)) invalid = 1;
        }
        if (tot < 1 || !feasible(args.F, n, s.svec[0], s.svec[1], s.svec[2], s.svec[3], s.svec[4])) invalid = 1;
        const Score sc = epilogue_d(s.S[0], s.S[1], s.S[2], s.S[3], lmax_of(s, s.pmask | 1ULL), s.ec);
        hc = sc.h;
        bk1 = sc.sla ? 0u : 1u; bk2 = okey(sc.h);
        for (int e = 0; e < E; ++e) s.bw[e] = s.w[e];
        s.dec_move = NOIDX;
        s.dec_done = invalid || (args.max_steps <= 0);
        if (invalid) status = -1;
    }
    cluster.sync();                          // all CTAs started before any DSMEM traffic
    bool done = s.dec_done;
    const int G = CL * ANT;
    const int gt = crank * ANT + tid;
    const unsigned long long mem_ok = s.mem_ok;

    for (int k = 0; !done; ++k) {
        PROF_MARK(0);
        prepare_step(s, rp, T, E, n, args.F);
        PROF_MARK(1);
        KRec rS = krec_none(), rV = krec_none(), rP = krec_none();
        unsigned long long cnt = 0;
        if (MODE == MODE_BEST_ALL) {
            // fp32 screen of every neighbour, survivors queued per warp and scored exactly
            // (fp64) in full warps.  Work unit = one removal entry (warp-uniform), lanes
            // stride its target list; entries are split over the cluster's warps by the
            // prefix of their list lengths.
            const int lane = tid & 31, wid = tid >> 5;
            const int NPc = E * (E + 1) / 2;
            const int W = CL * NWARP;
            const int gw = crank * NWARP + wid;
            double bS = CUDART_INF, bV = CUDART_INF;
            int qn = 0;
            const float *ecf = s.ecf;
            const float S0 = s.Sf[0], S1 = s.Sf[1], S2 = s.Sf[2], S3 = s.Sf[3];
            auto drain = [&](int nq) {            // exact-score queue entries [0, nq) (nq <= 32)
                __syncwarp();
                if (lane < nq) {
                    const int jj = s.qj[wid][lane];
                    const uint32_t ee = s.qe[wid][lane];
                    if (jj & 0x8000) {
                        const RemEnt &R = s.se[jj & 0x7FFF];
                        exact_pair<MODE>(s, R, ee, (int)R.p * E + (int)(ee & 63), rS, rV, false);
                    } else {
                        const RemEnt &R = rp[jj];
                        exact_pair<MODE>(s, R, ee, E * E + (int)R.p * NPc + (int)(ee >> 17), rS, rV, true);
                    }
                }
                __syncwarp();
            };
            auto push = [&](bool surv, int jtag, uint32_t ent) {
                const unsigned bal = __ballot_sync(0xFFFFFFFFu, surv);
                if (surv) {
                    const int pos = qn + __popc(bal & ((1u << lane) - 1u));
                    s.qj[wid][pos] = (unsigned short)jtag;
                    s.qe[wid][pos] = ent;
                }
                qn += __popc(bal);
                if (PROF) prof_surv += (lane == 0) ? __popc(bal) : 0;
                if (qn >= 32) {
                    drain(32);
                    qn -= 32;
                    if (lane < qn) { s.qj[wid][lane] = s.qj[wid][lane + 32]; s.qe[wid][lane] = s.qe[wid][lane + 32]; }
                    double mS = rS.key != ~0ULL ? rS.hv : CUDART_INF, mV = rV.key != ~0ULL ? rV.hv : CUDART_INF;
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) {
                        mS = fmin(mS, __shfl_xor_sync(0xFFFFFFFFu, mS, o));
                        mV = fmin(mV, __shfl_xor_sync(0xFFFFFFFFu, mV, o));
                    }
                    bS = mS; bV = mV;
                    __syncwarp();
                }
            };
            // singles: present edge i (warp-uniform), lanes over targets a
            for (int i = gw; i < s.nPE; i += W) {
                const RemEnt &R = s.se[i];
                for (int a0 = 0; a0 < E; a0 += 32) {
                    const int a = a0 + lane;
                    bool surv = false;
                    if (a < E && a != R.r1 && ((mem_ok >> a) & 1ULL) && s.feasS[R.code + s.sl[a]]) {
                        ++cnt;
                        const float4 x = s.rowf[a];
                        surv = !screen_out(ecf, S0 + R.f0 + x.x, S1 + R.f1 + x.y, S2 + R.f2 + x.z, S3 + R.f3 + x.w,
                                           s.latf_by_rank[63 - __clzll((long long)(R.mR | s.rbit[a]))], bS, bV);
                    }
                    push(surv, 0x8000 | i, (uint32_t)a);
                }
            }
            // doubles: warp gets the removal entries whose list prefix falls in its chunk
            {
                const int ND = s.nLen;
                const int chunk = (ND + W - 1) / W;
                const int lo_t = gw * chunk, hi_t = min(lo_t + chunk, ND);
                if (lo_t < hi_t) {
                    int lo = 0, hi = s.nRP;                  // first entry with pre >= lo_t
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (rp[mid].pre < lo_t) lo = mid + 1; else hi = mid;
                    }
                    const uint32_t *plist = T.pair_list;
                    for (int j = lo; j < s.nRP && rp[j].pre < hi_t; ++j) {
                        const RemEnt &R = rp[j];
                        const int len = R.len;
                        const uint32_t *lst = plist + R.off;
                        uint32_t nxt = lane < len ? __ldg(lst + lane) : 0u;
                        for (int o0 = 0; o0 < len; o0 += 32) {
                            const int o = o0 + lane;
                            bool surv = false;
                            uint32_t ent = 0;
                            if (o < len) {
                                ent = nxt;
                                if (o + 32 < len) nxt = __ldg(lst + o + 32);
                                if (s.feasD[R.code + ((ent >> 12) & 31)]) {
                                    ++cnt;
                                    const int a1 = ent & 63, a2 = (ent >> 6) & 63;
                                    const float4 x = s.rowf[a1], y = s.rowf[a2];
                                    surv = !screen_out(ecf, S0 + R.f0 + x.x + y.x, S1 + R.f1 + x.y + y.y,
                                                       S2 + R.f2 + x.z + y.z, S3 + R.f3 + x.w + y.w,
                                                       s.latf_by_rank[63 - __clzll((long long)(R.mR | s.rbit[a1] | s.rbit[a2]))],
                                                       bS, bV);
                                }
                            }
                            push(surv, j, ent);
                        }
                    }
                }
            }
            drain(qn);
        } else {
            // ---- singles: (present edge i, target edge a)
            {
                const int nS = s.nPE * E;
                int i = gt / E, a = gt - (gt / E) * E;
                const int dI = G / E, dA = G - (G / E) * E;
                for (int t = gt; t < nS; t += G) {
                    const RemEnt &R = s.se[i];
                    const bool ok = (a != R.r1) && ((mem_ok >> a) & 1ULL) && s.feasS[R.code + s.sl[a]];
                    if (ok) {
                        ++cnt;
                        consider<MODE, false>(s, R, a, 0, (int)(R.p * E + a), rS, rV, rP, args.seed, gchain, (uint64_t)k);
                    }
                    i += dI; a += dA;
                    if (a >= E) { a -= E; ++i; }
                }
            }
            // ---- doubles: flattened move space, warp-contiguous chunks
            {
                const int lane = tid & 31, wid = tid >> 5;
                const int ND = s.nLen;
                const int NPc = E * (E + 1) / 2;
                const int W = CL * NWARP;
                const int chunk = (((ND + W - 1) / W) + 31) & ~31;
                const int gw = crank * NWARP + wid;
                const int tb0 = gw * chunk;
                const int tend = min(tb0 + chunk, ND);
                if (tb0 < ND) {
                    int lo = 0, hi = s.nRP - 1;
                    const int t0 = min(tb0 + lane, ND - 1);
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (rp[mid].pre <= t0) lo = mid; else hi = mid - 1;
                    }
                    int j = lo;
                    const uint32_t *plist = T.pair_list;
                    for (int t = tb0 + lane; t < tend; t += 32) {
                        while (t >= rp[j].pre + rp[j].len) ++j;
                        const RemEnt &R = rp[j];
                        const uint32_t ent = __ldg(plist + R.off + (t - R.pre));
                        if (s.feasD[R.code + ((ent >> 12) & 31)]) {
                            ++cnt;
                            consider<MODE, true>(s, R, ent & 63, (ent >> 6) & 63, E * E + (int)R.p * NPc + (int)(ent >> 17),
                                                 rS, rV, rP, args.seed, gchain, (uint64_t)k);
                        }
                    }
                }
            }
        }
        PROF_MARK(2);
        // ---- CTA reduction, then DSMEM publish into the leader's slots
        {
            const int lane = tid & 31, wid = tid >> 5;
            if (MODE != MODE_UNIFORM_PROPOSAL) { rS = krec_min_warp<false>(rS); rV = krec_min_warp<false>(rV); }
            if (MODE != MODE_BEST_ALL) rP = krec_min_warp<MODE == MODE_UNIFORM_ALL>(rP);
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, m);
            if (lane == 0) { s.wS[wid] = rS; s.wV[wid] = rV; s.wP[wid] = rP; s.wc[wid] = cnt; }
            __syncthreads();
            if (wid == 0) {
                rS = lane < NWARP ? s.wS[lane] : krec_none();
                rV = lane < NWARP ? s.wV[lane] : krec_none();
                rP = lane < NWARP ? s.wP[lane] : krec_none();
                cnt = lane < NWARP ? s.wc[lane] : 0ULL;
                if (MODE != MODE_UNIFORM_PROPOSAL) { rS = krec_min_warp<false>(rS); rV = krec_min_warp<false>(rV); }
                if (MODE != MODE_BEST_ALL) rP = krec_min_warp<MODE == MODE_UNIFORM_ALL>(rP);
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, m);
                // every CTA decides redundantly (identical inputs, deterministic), so the
                // records go to all CTAs of the cluster -- one cluster barrier per step
                rS.key = __shfl_sync(0xFFFFFFFFu, rS.key, 0); rS.idx = __shfl_sync(0xFFFFFFFFu, rS.idx, 0);
                rV.key = __shfl_sync(0xFFFFFFFFu, rV.key, 0); rV.idx = __shfl_sync(0xFFFFFFFFu, rV.idx, 0);
                rP.key = __shfl_sync(0xFFFFFFFFu, rP.key, 0); rP.idx = __shfl_sync(0xFFFFFFFFu, rP.idx, 0);
                rP.hv = __shfl_sync(0xFFFFFFFFu, rP.hv, 0);
                cnt = __shfl_sync(0xFFFFFFFFu, cnt, 0);
                if (lane < CL) {
                    AnnealSmem *ls = cluster.map_shared_rank(&s, lane);
                    const int par = k & 1;
                    ls->slS[par][crank] = rS; ls->slV[par][crank] = rV; ls->slP[par][crank] = rP;
                    ls->slc[par][crank] = cnt;
                }
            }
        }
        PROF_MARK(3);
        cluster.sync();
        PROF_MARK(4);
        // ---- every CTA (thread 0): best tracking, Eq. 7, termination; rank 0 keeps outputs
        if (tid == 0) {
            const int par = k & 1;
            KRec S = krec_none(), V = krec_none(), P = krec_none();
            unsigned long long total = 0;
            for (int q = 0; q < CL; ++q) {
                if (krec_less(s.slS[par][q].key, s.slS[par][q].idx, S)) S = s.slS[par][q];
                if (krec_less(s.slV[par][q].key, s.slV[par][q].idx, V)) V = s.slV[par][q];
                if (krec_less(s.slP[par][q].key, s.slP[par][q].idx, P)) P = s.slP[par][q];
                total += s.slc[par][q];
            }
            long long mv = NOIDX;
            int fin = 0;
            if (total == 0) {
                status = 2;
                fin = 1;
            } else {
                // candidate for best tracking: SLA-meeting first
                unsigned int ck1;
                unsigned long long ck2;
                long long cidx;
                double hp;
                long long pidx;
                double fp = 0.0, Lp = 0.0;
                bool slap = false;
                if (MODE == MODE_UNIFORM_PROPOSAL) {
                    evals += 1;
                    int r1, r2, a1, a2;
                    decode_move(s, E, P.idx, r1, r2, a1, a2);
                    const Score sp = score_move(s, r1, r2, a1, a2);
                    hp = sp.h; fp = sp.f; Lp = sp.L; slap = sp.sla;
                    pidx = P.idx;
                    ck1 = sp.sla ? 0u : 1u; ck2 = okey(sp.h); cidx = P.idx;
                } else {
                    evals += (long long)total;
                    if (S.idx != 0x7FFFFFFF) { ck1 = 0u; ck2 = S.key; cidx = S.idx; }
                    else { ck1 = 1u; ck2 = V.key; cidx = V.idx; }
                    if (MODE == MODE_BEST_ALL) {
                        const KRec &B = krec_less(S.key, S.idx, V) ? S : V;   // min h overall
                        pidx = B.idx; hp = okey_inv(B.key);
                    } else {
                        pidx = P.idx; hp = P.hv;
                    }
                    if (args.log && leader) {
                        int r1, r2, a1, a2;
                        decode_move(s, E, pidx, r1, r2, a1, a2);
                        const Score sp = score_move(s, r1, r2, a1, a2);
                        fp = sp.f; Lp = sp.L; slap = sp.sla;
                    }
                }
                const bool nb = (ck1 < bk1) || (ck1 == bk1 && ck2 < bk2);
                if (nb) {
                    bk1 = ck1; bk2 = ck2; best_step = k; best_idx = cidx; stall = 0;
                    if (leader) {
                        int c1, c2, c3, c4;
                        decode_move(s, E, cidx, c1, c2, c3, c4);
                        for (int e = 0; e < E; ++e) s.bw[e] = s.w[e];
                        if (c1 != 0xFF) s.bw[c1] -= 1;
                        if (c2 != 0xFF) s.bw[c2] -= 1;
                        if (c3 != 0xFF) s.bw[c3] += 1;
                        if (c4 != 0xFF) s.bw[c4] += 1;
                    }
                } else {
                    stall += 1;
                }
                const double T0 = args.t_init - (double)k * args.cooling;
                const double Tk = args.t_floor >= T0 ? args.t_floor : T0;
                const double u = uniform01(derive_seed4(args.seed, gchain, (uint64_t)k, 0ULL));
                const bool acc = (hp <= hc) || (u < exp_clv(-(hp - hc) / Tk));
                if (args.log && leader) {
                    clv_log_row row;
                    row.temp = Tk; row.f = fp; row.h = hp; row.p95_ms = Lp;
                    row.iter = k; row.ged_from_center = (pidx < (long long)E * E) ? 2 : 4; row.sla_met = slap;
                    row.accepted = acc; row.new_best = nb; row.n_neighbours = (int)total;
                    args.log[(size_t)chain * args.max_steps + k] = row;
                }
                if (acc) { hc = hp; mv = pidx; }
                steps = k + 1;
                if (stall >= args.stall_limit) { status = 1; fin = 1; }
            }
            if (!fin && k + 1 >= args.max_steps) { status = 0; fin = 1; }
            if (mv != NOIDX) apply_move(s, E, mv);
            s.dec_done = fin;
        }
        PROF_MARK(5);
        PROF_MARK(6);
        __syncthreads();
        done = s.dec_done;
        PROF_MARK(7);
    }
    // No CTA may leave while a peer can still read its shared memory over DSMEM
    // (the non-leaders read the leader's decision after the last step).
    cluster.sync();
    if (PROF && threadIdx.x == 0 && args.prof)
        for (int q = 0; q < 7; ++q) args.prof[((size_t)blockIdx.x) * 8 + q] = prof_acc[q];
    if (PROF && args.prof) {                 // survivors of the fp32 screen, summed over the CTA's warps
        unsigned long long v = (threadIdx.x & 31) == 0 ? (unsigned long long)prof_surv : 0ULL;
        atomicAdd(reinterpret_cast<unsigned long long *>(args.prof) + ((size_t)blockIdx.x) * 8 + 7, v);
    }

    if (leader) {
        clv_chain_result r;
        uint16_t *bw_out = args.best_w + (size_t)chain * E;
        uint16_t *fw_out = args.final_w + (size_t)chain * E;
        double S0 = 0, S1 = 0, S2 = 0, S3 = 0;
        unsigned long long m = 0;
        for (int e = 0; e < E; ++e) {
            const int x = s.bw[e];
            bw_out[e] = (uint16_t)x;
            fw_out[e] = (uint16_t)s.w[e];
            S0 += x * s.row[e].thr; S1 += x * s.row[e].acc; S2 += x * s.row[e].en; S3 += x * s.row[e].idle;
            if (x > 0) m |= s.rbit[e];
        }
        const Score sb = epilogue_d(S0, S1, S2, S3, lmax_of(s, m | 1ULL), s.ec);
        r.f = sb.f; r.h = sb.h; r.p95_ms = sb.L; r.accuracy = sb.A; r.energy_wh = sb.E;
        r.sla_met = sb.sla;
        r.status = status; r.steps = steps; r.best_step = best_step;
        r.best_index = best_idx; r.evals = evals;
        args.res[chain] = r;
    }
}

template <int MODE, int MINB, int UNR, bool PROF = false>
static cudaError_t launch_mode(const AnnealArgs &a, int cluster_size, cudaStream_t st) {
    auto kern = anneal_kernel<MODE, MINB, UNR, PROF>;
    const size_t smem = sizeof(AnnealSmem) + sizeof(RemEnt) * (size_t)(a.E * (a.E + 1) / 2);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(ANT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cluster_size <= 0) {
        // Largest cluster size that still keeps every chain resident (one wave).
        cluster_size = 1;
        for (int c = MAXCL; c >= 2; --c) {
            cfg.gridDim = dim3((unsigned)(a.n_chains * c), 1, 1);
            attr[0].val.clusterDim.x = (unsigned)c;
            int clusters = 0;
            if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) == cudaSuccess && clusters >= a.n_chains) {
                cluster_size = c;
                break;
            }
            cudaGetLastError();
        }
    }
    cfg.gridDim = dim3((unsigned)(a.n_chains * cluster_size), 1, 1);
    attr[0].val.clusterDim.x = (unsigned)cluster_size;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

static int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
}

cudaError_t launch_anneal(const AnnealArgs &a, int cluster_size, cudaStream_t st) {
    if (a.proposal == 0) {
        // tuning variants of the headline mode (CLV_ANNEAL_VARIANT, default 0)
        switch (env_int("CLV_ANNEAL_VARIANT", 0)) {
            case 1: return launch_mode<MODE_BEST_ALL, 3, 1>(a, cluster_size, st);
            case 2: return launch_mode<MODE_BEST_ALL, 4, 1>(a, cluster_size, st);
            case 3: return launch_mode<MODE_BEST_ALL, 2, 1>(a, cluster_size, st);
            case 9: return launch_mode<MODE_BEST_ALL, 3, 1, true>(a, cluster_size, st);
            default: return launch_mode<MODE_BEST_ALL, 3, 1>(a, cluster_size, st);
        }
    }
    if (a.evaluate == 0) return launch_mode<MODE_UNIFORM_ALL, 3, 1>(a, cluster_size, st);
    return launch_mode<MODE_UNIFORM_PROPOSAL, 3, 1>(a, cluster_size, st);
}

}  // namespace clv
