// clv_anneal.cu -- K3 (GED<=4 neighbour generation + incremental scoring) fused
// with K4 (warp-shuffle argmax) and K5 (anneal step): one thread-block CLUSTER
// per annealing chain, every step of every chain inside one persistent launch.
//
// Reference semantics: sample_neighbor, anneal
// (SPEC:461-469, 478-483), Eqs. 6-7.  Step definition: DESIGN.md
// "Chain step"; CPU restatement: oracle/anneal.py + oracle/neighbours.py.
//
// Shared memory per CTA: per-edge rows {thr, acc, en, idle} held as fp64
// *integers* (exact: every partial sum < 2^53, so any summation order gives the
// oracle's int64 W @ rows bit for bit), per-edge p95 latencies, the family's
// static double-move lists (offsets/lengths), the chain centre, and per step the
// removal table: one entry per present edge (singles) and per available removal
// pair (doubles) with the exact removal deltas, the latency-rank presence mask that
// remains after the removal, and the entry's share of the move space.
// A neighbour is then scored as
//   S' = S + removal.d + row[a1] (+ row[a2]),  pm' = removal.pm | bit(a1) | bit(a2)
// followed by the fp64 epilogue (clv_common.cuh), whose p95 walk reads the centre's
// per-rank weights corrected by the (<= 4) changed edges.  Every CTA of the cluster
// builds identical tables (ordered compaction) and scores a contiguous share of
// the flattened move space; each CTA's two SLA-class records and hash record are
// broadcast to every CTA of the cluster over DSMEM, and after ONE cluster barrier
// per step every CTA takes the same deterministic decision (Eq. 7) and applies
// the accepted move to its own copy of the centre.
#include <cooperative_groups.h>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include "clv_internal.h"

namespace cg = cooperative_groups;

namespace clv {

constexpr int ANT = 320;                  // threads per CTA
constexpr int NWARP = ANT / 32;
constexpr int MAXP = CLV_MAX_EDGES * (CLV_MAX_EDGES + 1) / 2;   // 820 removal pairs
constexpr int MAXCL = 16;
constexpr long long NOIDX = -1;
constexpr int NO_TOP = CLV_MAX_EDGES;     // lat_by_rank[NO_TOP] == 0: nothing left present
constexpr int SCREEN_UNR = 3;             // candidates per lane per screen iteration
constexpr int QCAP = 32 * (SCREEN_UNR + 1);   // per-warp queue: < 32 left + one iteration's survivors

enum { MODE_BEST_ALL = 0, MODE_UNIFORM_ALL = 1, MODE_UNIFORM_PROPOSAL = 2 };

struct __align__(16) ARow {
    double thr, acc, en, idle, t2, t3;     // fixed-point rows as exact fp64 integers
};

struct __align__(8) RemEnt {            // one removal multiset R (single edge or pair), 80 B
    double b0, b1, b2, b3, b4, b5;         // centre aggregates minus the rows of R (exact integers)
    unsigned long long pm;                 // latency-rank presence mask after the removal
    int pre;                               // doubles: exclusive prefix of move-list lengths
    int end;                               // doubles: pre + move-list length
    int offm;                              // doubles: first static move-list entry minus pre
    int ibase;                             // canonical index base: E*E + P(r1,r2)*NP (doubles), r*E (singles)
    // Screen bounds for every candidate of this removal (0 = none): when the pessimistic p95
    // bound of the entry exceeds L_tail, all its candidates violate the SLA and
    // h >= -f * penU (f >= 0) or h >= -f * penL (f < 0); see pess_bounds().
    float penU, penL;
    unsigned short code;                   // slice code of R: sr1*125 + sr2*25 (doubles), sr*5 (singles)
    unsigned char r1, r2;                  // removed edges (r2 = 0xFF for singles)
    unsigned char k1, k2;                  // their latency ranks (k2 = 0xFF for singles)
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

// (key, idx) minimum over the warp without payload: three redux.sync steps
// (key high word, key low word, index) instead of five 3-shuffle rounds.
__device__ __forceinline__ KRec krec_min_redux(KRec r) {
    const unsigned hi = (unsigned)(r.key >> 32), lo = (unsigned)r.key;
    const unsigned mh = __reduce_min_sync(0xFFFFFFFFu, hi);
    const unsigned ml = __reduce_min_sync(0xFFFFFFFFu, hi == mh ? lo : 0xFFFFFFFFu);
    const unsigned mi = __reduce_min_sync(0xFFFFFFFFu, (hi == mh && lo == ml) ? (unsigned)r.idx : 0xFFFFFFFFu);
    KRec o;
    o.key = ((unsigned long long)mh << 32) | ml;
    o.idx = (int)mi;
    o.hv = 0.0;
    return o;
}

struct __align__(16) AnnealSmem {
    ARow row[CLV_MAX_EDGES];
    double lat_by_rank[CLV_MAX_EDGES + 1]; // ascending; [NO_TOP] = 0
    double svc_by_rank[CLV_MAX_EDGES];     // mean service time at each latency rank (p95 walk)
    double wr[CLV_MAX_EDGES];              // centre weight at each latency rank
    unsigned long long rbit[CLV_MAX_EDGES];// 1 << latency rank
    unsigned char rk[CLV_MAX_EDGES];       // latency rank of the edge
    unsigned char er[CLV_MAX_EDGES];       // edge at each latency rank
    EvalConst ec;
    unsigned long long mem_ok;
    unsigned magicE, magicNP;              // ceil(2^32 / E), ceil(2^32 / NP) (exact small divisions)
    unsigned ubase;                        // E*E + NP*NP: first paper (unit) move index
    int ub_dirty;                          // a unit move changed m: ub[] needs the new W0 bound
    unsigned char sl[CLV_MAX_EDGES];       // slice kind of the edge
    unsigned short pair_tab[MAXP];         // P -> (x | y << 8)
    unsigned char pair_len[MAXP];          // static move-list lengths (staged from FamilyTables)
    int pair_off[MAXP];                    // static move-list offsets (staged: off prepare's global loads)
    double ub[CLV_MAX_EDGES];              // per latency rank: c20 / (svc + W0_bound(m)) (pessimistic walk)
    double Cd[CLV_MAX_EDGES];              // centre's pessimistic tail at its i-th highest present rank
    unsigned char dr[CLV_MAX_EDGES];       // centre's present ranks, descending
    int nDR;
    int icb;                               // first i with Cd[i] > 1 + margin (the centre's bound rank)
    float penUc, penLc;                    // pen factors of the centre's bound
    unsigned long long seedS, seedO;       // screen thresholds known before scoring (keys of neighbours)
    unsigned long long thS_sh, thO_sh;     // CTA-wide screen thresholds of the current step
    // centre
    int w[CLV_MAX_EDGES];
    double S[6];
    double mcount;                         // instances of the chain (every GED move keeps it)
    int svec[CLV_K];
    unsigned long long pmask;              // presence by latency rank
    // per-step tables (the pair entries live in the dynamic tail)
    RemEnt se[CLV_MAX_EDGES];
    int nPE, nRP, nLen;
    unsigned char pe_list[CLV_MAX_EDGES];  // present edges, ascending
    int pfx[CLV_MAX_EDGES + 1];            // removal pairs starting before present edge i
    union {
        int pk[MAXP];                      // prepare: available pair q = P | x << 10 | y << 16
        uint32_t qbuf[NWARP][QCAP];        // score: per-warp queue of screened-in candidates
    };
    int warp_off[NWARP + 1], warp_len[NWARP + 1];
    int fsvec[CLV_K];                      // slice vector the feasibility bytes belong to
    unsigned char feasS[25];
    unsigned char feasD[625];
    unsigned char feasAR[10];              // paper moves: slice vector + e_k (0..4), - e_k (5..9) realizable
    // reductions
    KRec wS[NWARP], wV[NWARP], wP[NWARP];
    unsigned long long wc[NWARP];
    KRec slS[2][MAXCL], slV[2][MAXCL], slP[2][MAXCL];   // [step parity][cluster rank]
    unsigned long long slc[2][MAXCL];
    int dec_done;
    int next_chain;                        // persistent launches: the chain this CTA works on
    unsigned long long prof_surv;          // debug profile: candidates scored in full
    unsigned long long prof_surv1;         // debug profile: of which singles and unit moves
    int bw[CLV_MAX_EDGES];                 // best graph (rank 0)
};

// Service p95 of the centre corrected by removals (ranks k1, k2) and additions (ranks
// j1, j2); 0xFF = absent.  pm: the candidate's presence mask by latency rank.
struct CandWalk {
    const AnnealSmem *s;
    unsigned long long pm;
    int k1, k2, j1, j2;
    __device__ __forceinline__ double operator()(double W0, double c20) const {
        const AnnealSmem &S = *s;
        const int a = k1, b = k2, c = j1, d = j2;
        return p95_walk(pm, W0, c20, S.svc_by_rank, S.lat_by_rank, [&](int r) {
            return S.wr[r] + (double)((r == c) + (r == d) - (r == a) - (r == b));
        });
    }
};
// Service p95 of an explicit weight vector (rank 0 / thread 0 paths).
struct GraphWalk {
    const AnnealSmem *s;
    const int *w;                          // weights by edge
    const unsigned char *edge_of_rank;
    unsigned long long pm;
    __device__ __forceinline__ double operator()(double W0, double c20) const {
        const int *ww = w;
        const unsigned char *eo = edge_of_rank;
        return p95_walk(pm, W0, c20, s->svc_by_rank, s->lat_by_rank, [&](int r) { return (double)ww[eo[r]]; });
    }
};

// canonical index -> move (r1, r2, a1, a2; 0xFF = absent); indices are < 2^31
__device__ inline void decode_move(const AnnealSmem &s, int E, long long idx64, int &r1, int &r2, int &a1, int &a2) {
    // divisions by E and NP as multiply-high by ceil(2^32 / d): exact because n * d < 2^32
    const unsigned idx = (unsigned)idx64;
    if (idx >= s.ubase) {                                    // paper moves: add a, remove r
        const int u = (int)(idx - s.ubase);
        r2 = 0xFF; a2 = 0xFF;
        if (u < E) { r1 = 0xFF; a1 = u; } else { r1 = u - E; a1 = 0xFF; }
        return;
    }
    if (idx < (unsigned)(E * E)) {
        r1 = (int)__umulhi(idx, s.magicE); a1 = (int)(idx - (unsigned)r1 * E); r2 = 0xFF; a2 = 0xFF;
        return;
    }
    const unsigned NP = (unsigned)(E * (E + 1) / 2);
    const unsigned u = idx - (unsigned)(E * E);
    const int p = (int)__umulhi(u, s.magicNP), q = (int)(u - (unsigned)p * NP);
    r1 = s.pair_tab[p] & 0xFF; r2 = s.pair_tab[p] >> 8;
    a1 = s.pair_tab[q] & 0xFF; a2 = s.pair_tab[q] >> 8;
}

// Full score of a move from the centre (decision path: proposal, log).
__device__ inline Score score_move(const AnnealSmem &s, int r1, int r2, int a1, int a2) {
    double t = s.S[0], ac = s.S[1], en = s.S[2], id = s.S[3], q2 = s.S[4], q3 = s.S[5];
    unsigned long long m = s.pmask;
    const int e[2] = {r1, r2};
    for (int k = 0; k < 2; ++k) {
        if (e[k] == 0xFF) continue;
        t -= s.row[e[k]].thr; ac -= s.row[e[k]].acc; en -= s.row[e[k]].en; id -= s.row[e[k]].idle;
        q2 -= s.row[e[k]].t2; q3 -= s.row[e[k]].t3;
    }
    if (r1 != 0xFF && s.w[r1] - 1 - (r2 == r1 ? 1 : 0) == 0) m &= ~s.rbit[r1];
    if (r2 != 0xFF && r2 != r1 && s.w[r2] - 1 == 0) m &= ~s.rbit[r2];
    const int f[2] = {a1, a2};
    for (int k = 0; k < 2; ++k) {
        if (f[k] == 0xFF) continue;
        t += s.row[f[k]].thr; ac += s.row[f[k]].acc; en += s.row[f[k]].en; id += s.row[f[k]].idle;
        q2 += s.row[f[k]].t2; q3 += s.row[f[k]].t3;
        m |= s.rbit[f[k]];
    }
    CandWalk cw{&s, m, r1 == 0xFF ? 0xFF : s.rk[r1], r2 == 0xFF ? 0xFF : s.rk[r2],
                a1 == 0xFF ? 0xFF : s.rk[a1], a2 == 0xFF ? 0xFF : s.rk[a2]};
    const double mc = s.mcount + (double)((a1 != 0xFF) + (a2 != 0xFF) - (r1 != 0xFF) - (r2 != 0xFF));
    return epilogue_d(t, ac, en, id, q2, q3, mc, s.ec, cw);
}

// Apply a move to a bare weight vector (best-graph reconstruction).
__device__ inline void move_graph(const AnnealSmem &s, int E, long long idx, int *w) {
    int r1, r2, a1, a2;
    decode_move(s, E, idx, r1, r2, a1, a2);
    if (r1 != 0xFF) w[r1] -= 1;
    if (r2 != 0xFF) w[r2] -= 1;
    if (a1 != 0xFF) w[a1] += 1;
    if (a2 != 0xFF) w[a2] += 1;
}

// Apply a move to the CTA-local centre (thread 0) -- O(1).  Absent edges (0xFF) act as
// zero rows: S + ((A1 + A2) - (R1 + R2)) is the edge-by-edge update bit for bit (exact
// integers).  Unit add / remove moves (paper move set) change the instance count m.
__device__ inline void apply_move(AnnealSmem &s, int E, long long idx) {
    int r1, r2, a1, a2;
    decode_move(s, E, idx, r1, r2, a1, a2);
    if (r1 != 0xFF && a1 != 0xFF) {
        // SPEC move (m unchanged): all loads first, one update per field
        const bool two = r2 != 0xFF;                   // a double move has r2 and a2
        const ARow R1 = s.row[r1], A1 = s.row[a1];
        ARow R2 = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, A2 = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        int wr2 = 0, wa2 = 0;
        if (two) { R2 = s.row[r2]; A2 = s.row[a2]; wr2 = s.w[r2]; wa2 = s.w[a2]; }
        const int wr1 = s.w[r1], wa1 = s.w[a1];
        unsigned long long m = s.pmask;
        const unsigned long long br1 = s.rbit[r1], ba1 = s.rbit[a1];
        const unsigned long long br2 = two ? s.rbit[r2] : 0ULL, ba2 = two ? s.rbit[a2] : 0ULL;
        s.S[0] = s.S[0] + ((A1.thr + A2.thr) - (R1.thr + R2.thr));
        s.S[1] = s.S[1] + ((A1.acc + A2.acc) - (R1.acc + R2.acc));
        s.S[2] = s.S[2] + ((A1.en + A2.en) - (R1.en + R2.en));
        s.S[3] = s.S[3] + ((A1.idle + A2.idle) - (R1.idle + R2.idle));
        s.S[4] = s.S[4] + ((A1.t2 + A2.t2) - (R1.t2 + R2.t2));
        s.S[5] = s.S[5] + ((A1.t3 + A2.t3) - (R1.t3 + R2.t3));
        const int nr1 = wr1 - 1 - ((two && r2 == r1) ? 1 : 0);
        const int nr2 = two ? ((r2 == r1) ? nr1 : wr2 - 1) : 1;
        const int na1 = wa1 + 1 + ((two && a2 == a1) ? 1 : 0);
        s.w[r1] = nr1;
        s.w[a1] = na1;
        if (two) { s.w[r2] = nr2; s.w[a2] = (a2 == a1) ? na1 : wa2 + 1; }
        s.wr[s.rk[r1]] = (double)s.w[r1];
        s.wr[s.rk[a1]] = (double)s.w[a1];
        if (two) { s.wr[s.rk[r2]] = (double)s.w[r2]; s.wr[s.rk[a2]] = (double)s.w[a2]; }
        const int kr1 = r1 % CLV_K, ka1 = a1 % CLV_K, kr2 = two ? r2 % CLV_K : -1, ka2 = two ? a2 % CLV_K : -1;
#pragma unroll
        for (int k = 0; k < CLV_K; ++k)
            s.svec[k] += (k == ka1) + (k == ka2) - (k == kr1) - (k == kr2);
        if (nr1 == 0) m &= ~br1;
        if (nr2 == 0) m &= ~br2;
        s.pmask = m | ba1 | ba2;
        return;
    }
    // paper unit move: one instance added on a1 or removed from r1 (m changes)
    const bool add = a1 != 0xFF;
    const int e = add ? a1 : r1;
    const ARow A = s.row[e];
    const double sg = add ? 1.0 : -1.0;
    s.S[0] = s.S[0] + sg * A.thr; s.S[1] = s.S[1] + sg * A.acc; s.S[2] = s.S[2] + sg * A.en;
    s.S[3] = s.S[3] + sg * A.idle; s.S[4] = s.S[4] + sg * A.t2; s.S[5] = s.S[5] + sg * A.t3;
    const int nw = s.w[e] + (add ? 1 : -1);
    s.w[e] = nw;
    s.wr[s.rk[e]] = (double)nw;
    s.svec[e % CLV_K] += add ? 1 : -1;
    s.pmask = nw > 0 ? (s.pmask | s.rbit[e]) : (s.pmask & ~s.rbit[e]);
    s.mcount += sg;
    s.ub_dirty = 1;
}

__device__ __forceinline__ void pen_factors(double lb, double slo, float &pu, float &pl);

// Screen bounds of one removal entry (ranks k1, k2 removed; -1 = none).  Pessimistic p95
// walk: with the idle wait at its bound W0_b = 1000 m / R (>= the candidate's W0, the clamp in
// idle_wait_ms), every present rank r contributes u_r = c20 / (svc_r + W0_b) per instance to
// the tail, no more than its true share c20 / (svc_r + W0).  The centre's pessimistic tail
// at its i-th highest present rank is Cd[i]; the removal subtracts u_k for each removed
// instance at a rank k >= r; additions only add tail.  So if the pessimistic tail at rank r
// exceeds 1 (with a 2^-30 margin that covers the rounding of the walk's P / Q fraction and
// of these sums), the true walk of every candidate of this entry stops at a rank >= r:
// p95 >= lat(r) =: lb, and L = p95 (1 + wq) >= lb.  When lb > L_tail every candidate of the
// entry violates the SLA, and h = -f * (slo / L) >= -f * penU (f >= 0), h = -f * (L / slo) >=
// -f * penL (f < 0, Eq. 6 amended), penU >= slo / lb and penL <= lb / slo rounded outwards.
__device__ __forceinline__ void pess_bounds(const AnnealSmem &s, int k1, int k2, double slo, float &pu, float &pl) {
    // Removals below the centre's own bound rank leave the tails at and above it unchanged:
    // the centre's bound (and its pen factors) hold for the entry as they are.
    const int ic = s.icb;
    if (ic < s.nDR && k1 < s.dr[ic] && k2 < s.dr[ic]) { pu = s.penUc; pl = s.penLc; return; }
    double lb = 0.0;
    const int nd = s.nDR;
    const double u1 = k1 >= 0 ? s.ub[k1] : 0.0, u2 = k2 >= 0 ? s.ub[k2] : 0.0;
    for (int i = 0; i < nd; ++i) {
        const int r = s.dr[i];
        const double T = (s.Cd[i] - (k1 >= r ? u1 : 0.0)) - (k2 >= r ? u2 : 0.0);
        if (T > 1.0 + 0x1p-30) { lb = s.lat_by_rank[r]; break; }
    }
    pen_factors(lb, slo, pu, pl);
}

__device__ __forceinline__ void pen_factors(double lb, double slo, float &pu, float &pl) {
    const float lf = __double2float_rd(lb);
    const bool cv = (double)lf > slo;
    pu = cv ? __double2float_ru((slo / (double)lf) * (1.0 + 0x1p-40)) : 0.0f;
    pl = cv ? __double2float_rd(((double)lf / slo) * (1.0 - 0x1p-40)) : 0.0f;
}

// apply_move by a whole warp: lanes 0-5 update one centre sum each, lane 6 the weights, the
// slice vector and the presence mask (SPEC moves); unit moves take the serial path on lane 0.
__device__ inline void apply_move_warp(AnnealSmem &s, int E, long long idx, int lane) {
    int r1, r2, a1, a2;
    decode_move(s, E, idx, r1, r2, a1, a2);
    if (r1 == 0xFF || a1 == 0xFF) {
        if (lane == 0) apply_move(s, E, idx);
        __syncwarp();
        return;
    }
    if (lane < 6) {
        const double R1 = reinterpret_cast<const double *>(&s.row[r1])[lane];
        const double A1 = reinterpret_cast<const double *>(&s.row[a1])[lane];
        const double R2 = r2 != 0xFF ? reinterpret_cast<const double *>(&s.row[r2])[lane] : 0.0;
        const double A2 = a2 != 0xFF ? reinterpret_cast<const double *>(&s.row[a2])[lane] : 0.0;
        s.S[lane] = s.S[lane] + ((A1 + A2) - (R1 + R2));   // same op order as apply_move
    } else if (lane == 6) {
        const bool two = r2 != 0xFF;
        const int wr1 = s.w[r1], wa1 = s.w[a1];
        const int wr2 = two ? s.w[r2] : 0, wa2 = two ? s.w[a2] : 0;
        unsigned long long m = s.pmask;
        const unsigned long long br1 = s.rbit[r1], ba1 = s.rbit[a1];
        const unsigned long long br2 = two ? s.rbit[r2] : 0ULL, ba2 = two ? s.rbit[a2] : 0ULL;
        const int nr1 = wr1 - 1 - ((two && r2 == r1) ? 1 : 0);
        const int nr2 = two ? ((r2 == r1) ? nr1 : wr2 - 1) : 1;
        const int na1 = wa1 + 1 + ((two && a2 == a1) ? 1 : 0);
        s.w[r1] = nr1;
        s.w[a1] = na1;
        if (two) { s.w[r2] = nr2; s.w[a2] = (a2 == a1) ? na1 : wa2 + 1; }
        s.wr[s.rk[r1]] = (double)s.w[r1];
        s.wr[s.rk[a1]] = (double)s.w[a1];
        if (two) { s.wr[s.rk[r2]] = (double)s.w[r2]; s.wr[s.rk[a2]] = (double)s.w[a2]; }
        const int kr1 = r1 % CLV_K, ka1 = a1 % CLV_K, kr2 = two ? r2 % CLV_K : -1, ka2 = two ? a2 % CLV_K : -1;
#pragma unroll
        for (int k = 0; k < CLV_K; ++k)
            s.svec[k] += (k == ka1) + (k == ka2) - (k == kr1) - (k == kr2);
        if (nr1 == 0) m &= ~br1;
        if (nr2 == 0) m &= ~br2;
        s.pmask = m | ba1 | ba2;
    }
    __syncwarp();
}

// Per-step tables: deterministic ordered compaction of the removal pairs (every
// CTA of the cluster must build identical tables because the cluster partitions
// the move space by table position), the present-edge entries, and -- only when
// the centre's slice multiset changed -- the feasibility bytes of all 25 single /
// 625 double slice deltas (loads issued first so their latency overlaps the rest).
template <bool PROF, bool PAPER>
__device__ __forceinline__ void prepare_step(AnnealSmem &s, RemEnt *rp, int E, int n, const FeasView &F,
                                             const FamilyTables &T, double slo, long long *pacc) {
    const long long pt0 = PROF ? clock64() : 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int NP = E * (E + 1) / 2;
    constexpr int PER = (MAXP + ANT - 1) / ANT;    // consecutive pairs per thread (4 at E <= 40)
    static_assert(PER <= 4, "pair split assumes <= 4 removal pairs per thread");
    bool refresh = false;
#pragma unroll
    for (int k = 0; k < CLV_K; ++k) refresh |= (s.svec[k] != s.fsvec[k]);
    // Feasibility of the 650 slice deltas, 3 per thread, as two batched round trips:
    // all rectangle offsets first, then all bitset words (feasible() in clv_common.cuh
    // would serialise the 2 dependent loads of each lookup).
    // Warps 1.. only (3 deltas per thread): warp 0 builds the present-edge list below
    // meanwhile, so the two round trips are off its path.
    constexpr int FT = ANT - 32;
    static_assert(3 * FT >= 660, "feasibility refresh needs 650 + 10 lookups");
    bool fres[3] = {false, false, false};
    if (refresh && wid > 0) {                      // uniform across the CTA
        uint32_t obase[3], wofs[3], bit[3];
        bool cand[3];
        int sv[CLV_K];
#pragma unroll
        for (int k = 0; k < CLV_K; ++k) sv[k] = s.svec[k];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const int t = threadIdx.x - 32 + q * FT;
            // removed / added slice kinds of delta t (-1 = none); the delta vector is formed with
            // constant indices only (a dynamically indexed array would live in local memory)
            int r1 = -1, r2 = -1, a1 = -1, a2 = -1;
            bool ok = t < (PAPER ? 660 : 650);
            if (t < 25) {
                r1 = t / 5; a1 = t % 5;
            } else if (t < 650) {
                const int u = t - 25;
                r1 = u / 125; r2 = (u / 25) % 5; a1 = (u / 5) % 5; a2 = u % 5;
            } else if (t < 655) {
                a1 = t - 650;                      // one instance added on slice kind t - 650
            } else if (t < 660) {
                r1 = t - 655;                      // one instance removed
            }
            int v[CLV_K];
#pragma unroll
            for (int k = 0; k < CLV_K; ++k)
                v[k] = sv[k] - (k == r1) - (k == r2) + (k == a1) + (k == a2);
            ok = ok && v[0] >= 0 && v[1] >= 0 && v[2] >= 0 && v[3] >= 0 && v[4] >= 0;
            // feasible(F, n, v...) split into its index arithmetic and its two loads
            ok = ok && v[0] <= n && (v[0] == 0 || F.has7g);
            const int N = n - v[0];
            const int R = 7 * N - 4 * v[1] - 3 * v[2];
            ok = ok && N <= F.nmax && R >= 0 && R - 2 * v[3] >= 0 && v[4] <= R - 2 * v[3];
            cand[q] = ok;
            obase[q] = ok ? __ldg(F.off + ((size_t)N * F.bdim + v[1]) * F.cdim + v[2]) : 0u;
            wofs[q] = ok ? (uint32_t)v[3] * (uint32_t)((R + 32) >> 5) + (uint32_t)(v[4] >> 5) : 0u;
            bit[q] = (uint32_t)(v[4] & 31);
        }
        uint32_t word[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) word[q] = cand[q] ? __ldg(F.bits + obase[q] + wofs[q]) : 0u;
#pragma unroll
        for (int q = 0; q < 3; ++q) fres[q] = cand[q] && ((word[q] >> bit[q]) & 1u);
    }
    // (1) warp 0: present-edge list (ascending) and, per present edge i, the exclusive
    //     prefix of the removal pairs that start at it: (e_i, e_i) when w >= 2, then
    //     (e_i, e_j) for j > i -- i.e. the available pairs in ascending P(x, y), the
    //     same deterministic order in every CTA of the cluster.
    const long long ptR = PROF ? clock64() : 0;
    if (wid == 0) {
        if (PAPER && s.ub_dirty) {                 // an add / remove move changed m: new W0 bound
            const double w0b = w0_bound(s.mcount, s.ec);
            for (int r = lane; r < E; r += 32) s.ub[r] = s.ec.c20 / (s.svc_by_rank[r] + w0b);
            __syncwarp();
            if (lane == 0) s.ub_dirty = 0;
            __syncwarp();
        }
        int k = 0;
        for (int e0 = 0; e0 < E; e0 += 32) {
            const int e = e0 + lane;
            const bool ok = e < E && s.w[e] > 0;
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, ok);
            if (ok) s.pe_list[k + __popc(bal & ((1u << lane) - 1u))] = (unsigned char)e;
            k += __popc(bal);
        }
        __syncwarp();
        int pb = 0;
        for (int i0 = 0; i0 < k; i0 += 32) {
            const int i = i0 + lane;
            const int c = i < k ? (k - i - 1) + (s.w[s.pe_list[i]] >= 2 ? 1 : 0) : 0;
            int x = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, x, d);
                if (lane >= d) x += y;
            }
            if (i < k) s.pfx[i] = pb + x - c;
            pb += __shfl_sync(0xFFFFFFFFu, x, 31);
        }
        if (lane == 0) { s.nPE = k; s.pfx[k] = pb; s.nRP = pb; }
        // the centre's present latency ranks, descending, with their pessimistic tails
        // (suffix sums of w_r u_r over ranks >= r; lanes own ranks lane and lane + 32)
        const unsigned long long pm = s.pmask;
        const int rlo = lane, rhi = lane + 32;
        const bool plo = (pm >> rlo) & 1ULL, phi = rhi < 64 && ((pm >> rhi) & 1ULL);
        const double vlo = plo ? s.wr[rlo] * s.ub[rlo] : 0.0;
        const double vhi = phi ? s.wr[rhi] * s.ub[rhi] : 0.0;
        double shi = vhi, slo_ = vlo;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {            // suffix scans within each half
            const double yh = __shfl_down_sync(0xFFFFFFFFu, shi, d);
            const double yl = __shfl_down_sync(0xFFFFFFFFu, slo_, d);
            if (lane + d < 32) { shi += yh; slo_ += yl; }
        }
        slo_ += __shfl_sync(0xFFFFFFFFu, shi, 0);     // + everything in the upper half
        if (phi) {
            const int i = __popcll(pm >> (rhi + 1));
            s.dr[i] = (unsigned char)rhi; s.Cd[i] = shi;
        }
        if (plo) {
            const int i = __popcll(pm >> (rlo + 1));
            s.dr[i] = (unsigned char)rlo; s.Cd[i] = slo_;
        }
        if (lane == 0) s.nDR = __popcll(pm);
        // the centre's bound rank: the highest present rank whose pessimistic tail exceeds 1
        const bool bhi = phi && shi > 1.0 + 0x1p-30, blo = plo && slo_ > 1.0 + 0x1p-30;
        const unsigned bh = __ballot_sync(0xFFFFFFFFu, bhi), bl = __ballot_sync(0xFFFFFFFFu, blo);
        if (lane == 0) {
            const int rb = bh ? 32 + (31 - __clz((int)bh)) : (bl ? 31 - __clz((int)bl) : -1);
            s.icb = rb >= 0 ? __popcll(pm >> (rb + 1)) : 64;
            float pu, pl;
            pen_factors(rb >= 0 ? s.lat_by_rank[rb] : 0.0, slo, pu, pl);
            s.penUc = pu; s.penLc = pl;
        }
    }
    __syncthreads();
    const long long ptA = PROF ? clock64() : 0;
    // (2) every thread: a contiguous run of <= PER available pairs, their move-list
    //     lengths, and a block exclusive scan of the lengths in pair order.
    const int k = s.nPE, npairs = s.nRP;
    const int per = (npairs + ANT - 1) / ANT;
    const int q0 = threadIdx.x * per;
    int cnt = 0, lsum = 0;
    if (q0 < npairs) {
        int lo = 0, hi = k - 1;                    // last i with pfx[i] <= q0
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s.pfx[mid] <= q0) lo = mid; else hi = mid - 1;
        }
        int i = lo;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int q = q0 + u;
            if (u < per && q < npairs) {
                while (q >= s.pfx[i + 1]) ++i;
                const int x = s.pe_list[i];
                const int y = s.pe_list[i + (q - s.pfx[i]) + (s.w[x] >= 2 ? 0 : 1)];
                const int p = x * E - (x * (x - 1)) / 2 + (y - x);
                s.pk[q] = p | (x << 10) | (y << 16);     // p < 1024; x, y < 64
                lsum += s.pair_len[p];
                ++cnt;
            }
        }
    }
    int il = lsum;                                 // block exclusive scan of lsum in thread order
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int yl = __shfl_up_sync(0xFFFFFFFFu, il, d);
        if (lane >= d) il += yl;
    }
    if (lane == 31) s.warp_len[wid] = il;
    __syncthreads();
    const long long ptB = PROF ? clock64() : 0;
    if (threadIdx.x < 32) {
        const int l = lane < NWARP ? s.warp_len[lane] : 0;
        int l2 = l;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int yl = __shfl_up_sync(0xFFFFFFFFu, l2, d);
            if (lane >= d) l2 += yl;
        }
        if (lane < NWARP) s.warp_len[lane] = l2 - l;
        if (lane == NWARP - 1) s.nLen = l2;
    }
    __syncthreads();
    const long long pt1 = PROF ? clock64() : 0;
    // (3) the removal entries (pairs: every thread; singles: the last warp)
    int lpos = s.warp_len[wid] + il - lsum;
#pragma unroll
    for (int u = 0; u < PER; ++u) {              // fixed trip count: the entries' loads overlap
        if (u >= cnt) break;
        const int pkv = s.pk[q0 + u];
        const int p = pkv & 1023, x = (pkv >> 10) & 63, y = pkv >> 16;
        RemEnt &r = rp[q0 + u];
        r.b0 = s.S[0] + -(s.row[x].thr + s.row[y].thr);
        r.b1 = s.S[1] + -(s.row[x].acc + s.row[y].acc);
        r.b2 = s.S[2] + -(s.row[x].en + s.row[y].en);
        r.b3 = s.S[3] + -(s.row[x].idle + s.row[y].idle);
        r.b4 = s.S[4] + -(s.row[x].t2 + s.row[y].t2);
        r.b5 = s.S[5] + -(s.row[x].t3 + s.row[y].t3);
        unsigned long long m = s.pmask;
        if (x == y) { if (s.w[x] == 2) m &= ~s.rbit[x]; }
        else {
            if (s.w[x] == 1) m &= ~s.rbit[x];
            if (s.w[y] == 1) m &= ~s.rbit[y];
        }
        r.pm = m;
        r.k1 = s.rk[x]; r.k2 = s.rk[y];
        r.ibase = E * E + p * NP;
        r.pre = lpos;
        r.offm = s.pair_off[p] - lpos;
        lpos += s.pair_len[p];
        r.end = lpos;
        pess_bounds(s, r.k1, r.k2, slo, r.penU, r.penL);
        r.code = (unsigned short)(s.sl[x] * 125 + s.sl[y] * 25);
        r.r1 = (unsigned char)x; r.r2 = (unsigned char)y;
    }
    if (wid == NWARP - 1) {
        for (int i = lane; i < k; i += 32) {
            const int e = s.pe_list[i];
            RemEnt &r = s.se[i];
            r.b0 = s.S[0] + -s.row[e].thr; r.b1 = s.S[1] + -s.row[e].acc;
            r.b2 = s.S[2] + -s.row[e].en; r.b3 = s.S[3] + -s.row[e].idle;
            r.b4 = s.S[4] + -s.row[e].t2; r.b5 = s.S[5] + -s.row[e].t3;
            r.pm = (s.w[e] == 1) ? (s.pmask & ~s.rbit[e]) : s.pmask;
            r.k1 = s.rk[e]; r.k2 = 0xFF;
            r.ibase = e * E;
            r.code = (unsigned short)(s.sl[e] * 5);
            r.r1 = (unsigned char)e; r.r2 = 0xFF; r.offm = 0; r.end = 0; r.pre = 0;
            pess_bounds(s, r.k1, -1, slo, r.penU, r.penL);
        }
    }
    if (refresh && wid > 0) {
        for (int q = 0; q < 3; ++q) {
            const int t = threadIdx.x - 32 + q * FT;
            if (t < 25) s.feasS[t] = fres[q];
            else if (t < 650) s.feasD[t - 25] = fres[q];
            else if (t < 660) s.feasAR[t - 650] = fres[q];
        }
        if (threadIdx.x - 32 < CLV_K) s.fsvec[threadIdx.x - 32] = s.svec[threadIdx.x - 32];
    }
    __syncthreads();
    if (PROF && threadIdx.x == 0) {
        pacc[10] += pt1 - pt0; pacc[11] += clock64() - pt1;
        pacc[12] += ptA - pt0; pacc[13] += ptB - ptA; pacc[14] += pt1 - ptB; pacc[15] += ptR - pt0;
    }
}

// Exact score of one neighbour folded into the thread's records.
// EC: 2 = one scenario for every chain, constants as kernel parameters, branch-free
// division; 1 = per-chain scenarios (shared copy), branch-free division; 0 = per-chain
// scenarios, IEEE division (a scenario outside fast_div_safe's ranges).
template <int MODE, int EC>
__device__ __forceinline__ void fold(const AnnealSmem &s, const AnnealArgs &args, double t, double ac, double en,
                                     double id, double q2, double q3, const CandWalk &cw, double mcnt, int idx,
                                     KRec &rS, KRec &rV, KRec &rP, uint64_t seed, uint64_t gchain, uint64_t k) {
    if (MODE == MODE_UNIFORM_PROPOSAL) {
        const unsigned long long hk = derive_seed4(seed, gchain, k, (uint64_t)idx + 1);
        if (krec_less(hk, idx, rP)) { rP.key = hk; rP.idx = idx; }
        return;
    }
    // one evaluation scenario for every chain: its constants are kernel parameters
    // (constant-bank operands); per-chain scenarios come from the CTA's shared copy
    Score sc;
    if constexpr (EC == 2) sc = epilogue_t<true>(t, ac, en, id, q2, q3, mcnt, args.ec0, cw);
    else sc = epilogue_t<EC == 1>(t, ac, en, id, q2, q3, mcnt, s.ec, cw);
    const unsigned long long key = okey(sc.h);
    if (sc.sla) { if (krec_less(key, idx, rS)) { rS.key = key; rS.idx = idx; } }
    else        { if (krec_less(key, idx, rV)) { rV.key = key; rV.idx = idx; } }
    if (MODE == MODE_UNIFORM_ALL) {
        const unsigned long long hk = derive_seed4(seed, gchain, k, (uint64_t)idx + 1);
        if (krec_less(hk, idx, rP)) { rP.key = hk; rP.idx = idx; rP.hv = sc.h; }
    }
}

template <int EC>
__device__ __forceinline__ const EvalConst &ec_of(const AnnealArgs &args, const AnnealSmem &s) {
    if constexpr (EC == 2) return args.ec0;      // one scenario: constant-bank operands
    else return s.ec;
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long x) {
    const unsigned hi = __reduce_min_sync(0xFFFFFFFFu, (unsigned)(x >> 32));
    const unsigned lo = __reduce_min_sync(0xFFFFFFFFu, (unsigned)(x >> 32) == hi ? (unsigned)x : 0xFFFFFFFFu);
    return ((unsigned long long)hi << 32) | lo;
}

// Full score of a queued move: bit 31 set = single (present-edge entry i, target edge a),
// else double (removal entry jj, position off in its static move list).
template <int MODE, int EC>
__device__ __forceinline__ void score_queued(const AnnealSmem &s, const AnnealArgs &args, const RemEnt *rp,
                                             const uint32_t *plist, uint32_t d, double mcnt, KRec &rS, KRec &rV,
                                             KRec &rP, uint64_t gchain, uint64_t k) {
    if ((d >> 30) == 1u) {                       // paper move: add (bit 8 clear) / remove one instance
        const int e = d & 0xFFu;
        const bool rem = (d >> 8) & 1u;
        const ARow &A = s.row[e];
        const double sg = rem ? -1.0 : 1.0;      // S -/+ row: exact integers either way
        const unsigned long long pm = rem ? (s.w[e] == 1 ? (s.pmask & ~s.rbit[e]) : s.pmask) : (s.pmask | s.rbit[e]);
        const CandWalk cw{&s, pm, rem ? s.rk[e] : 0xFF, 0xFF, rem ? 0xFF : s.rk[e], 0xFF};
        const int E = args.E;
        const int ubase = E * E + (E * (E + 1) / 2) * (E * (E + 1) / 2);
        fold<MODE, EC>(s, args, s.S[0] + sg * A.thr, s.S[1] + sg * A.acc, s.S[2] + sg * A.en, s.S[3] + sg * A.idle,
                       s.S[4] + sg * A.t2, s.S[5] + sg * A.t3, cw, mcnt + sg, ubase + (rem ? E : 0) + e, rS, rV, rP,
                       args.seed, gchain, k);
        return;
    }
    if (d >> 31) {
        const RemEnt &R = s.se[(d >> 8) & 0xFFu];
        const int a = d & 0xFFu;
        const ARow &A = s.row[a];
        const CandWalk cw{&s, R.pm | s.rbit[a], R.k1, 0xFF, s.rk[a], 0xFF};
        fold<MODE, EC>(s, args, R.b0 + A.thr, R.b1 + A.acc, R.b2 + A.en, R.b3 + A.idle, R.b4 + A.t2, R.b5 + A.t3,
                       cw, mcnt, R.ibase + a, rS, rV, rP, args.seed, gchain, k);
        return;
    }
    const RemEnt &R = rp[d & 0xFFFFu];
    const uint32_t ent = __ldg(plist + R.offm + R.pre + (int)(d >> 16));
    const int a1 = ent & 63, a2 = (ent >> 6) & 63;
    const ARow &A1 = s.row[a1], &A2 = s.row[a2];
    const CandWalk cw{&s, R.pm | s.rbit[a1] | s.rbit[a2], R.k1, R.k2, s.rk[a1], s.rk[a2]};
    fold<MODE, EC>(s, args, R.b0 + A1.thr + A2.thr, R.b1 + A1.acc + A2.acc, R.b2 + A1.en + A2.en,
                   R.b3 + A1.idle + A2.idle, R.b4 + A1.t2 + A2.t2, R.b5 + A1.t3 + A2.t3, cw, mcnt,
                   R.ibase + (int)(ent >> 17), rS, rV, rP, args.seed, gchain, k);
}

__device__ __forceinline__ double key_limit(unsigned long long th) {   // okey(x) <= th  <=>  x <= key_limit(th)
    return th == ~0ULL ? __longlong_as_double(0x7FF0000000000000LL) : okey_inv(th);
}

// Lower bound of h for the screen (see score_screened); a, f: the candidate's A/E and f.
__device__ __forceinline__ bool screen_keep(double f, const RemEnt &R, bool strict, double limS, double limO) {
    const bool neg_strict = f < 0.0 && strict;
    double lb, lim;
    if (R.penU > 0.0f) {                         // every candidate of this entry violates the SLA
        lb = neg_strict ? 0.0 : -f * (double)(f >= 0.0 ? R.penU : R.penL);
        lim = limO;
    } else {
        lb = neg_strict ? 0.0 : -f;
        lim = limS;
    }
    return lb <= lim;
}

// Single and double moves with an exact screen.  Each candidate first gets only A, E and f
// (the epilogue's first half, the same ops and bits as the full score) and a lower bound of
// h: h >= -f always (Eq. 6 amended: the SLA penalty only raises h; strict form, f < 0: h >= 0),
// and h >= -f * pen for the removal entries whose pessimistic p95 bound already violates the
// SLA (pess_bounds).  A candidate is scored in full only if its bound does not exceed a key
// already achieved by a scored neighbour: the SLA class's for candidates that may meet the
// SLA, the overall minimum's for certain violators (a violator above an achieved key is
// neither the class minimum nor the overall minimum; when an SLA-meeting neighbour exists the
// violating record is only compared against it).  In MODE_UNIFORM_ALL a candidate whose hash
// could be the proposal is always scored (its h is the proposal's).  The thresholds start from
// neighbours known before scoring (the previous centre, or the same neighbourhood when the
// centre did not move) and tighten with the CTA's records.  Survivors go to a per-warp queue
// and are scored 32 at a time, so the full epilogue runs on full warps.  The records, and
// hence every decision, are those of scoring every candidate in full.
template <int MODE, int EC, bool PROF, bool PAPER>
__device__ __forceinline__ void score_screened(AnnealSmem &s, const AnnealArgs &args, const RemEnt *rp,
                                               const uint32_t *plist, int crank, int CL, KRec &rS, KRec &rV,
                                               KRec &rP, unsigned long long &cnt, uint64_t gchain, uint64_t k) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const EvalConst &cc = ec_of<EC>(args, s);
    constexpr bool FAST = EC >= 1;
    const bool strict = cc.strict != 0;
    const double mcnt = s.mcount;
    const int E = args.E;
    uint32_t *q = s.qbuf[wid];
    int qn = 0;
    unsigned long long thS = s.thS_sh, thO = s.thO_sh, thP = ~0ULL;
    double limS = key_limit(thS), limO = key_limit(thO);
    const unsigned lt = (1u << lane) - 1u;
    long long nsurv = 0;
    auto drain = [&](bool all) {                 // score queued survivors 32 at a time
        while (qn >= 32) {
            qn -= 32;
            if (PROF) nsurv += 32;
            score_queued<MODE, EC>(s, args, rp, plist, q[qn + lane], mcnt, rS, rV, rP, gchain, k);
            const unsigned long long kS = warp_min_u64(rS.key), kV = warp_min_u64(rV.key);
            thS = kS < thS ? kS : thS;
            thO = kS < thO ? kS : thO;
            thO = kV < thO ? kV : thO;
            if (MODE == MODE_UNIFORM_ALL) { const unsigned long long kP = warp_min_u64(rP.key); thP = kP < thP ? kP : thP; }
            if (lane == 0) { atomicMin(&s.thS_sh, thS); atomicMin(&s.thO_sh, thO); }
            limS = key_limit(thS); limO = key_limit(thO);
            __syncwarp();
        }
        if (all && qn > 0) {
            if (PROF) nsurv += qn;
            if (lane < qn) score_queued<MODE, EC>(s, args, rp, plist, q[lane], mcnt, rS, rV, rP, gchain, k);
            qn = 0;
        }
    };
    auto refresh = [&]() {                       // the CTA's best achieved keys so far
        const unsigned long long a = *(volatile unsigned long long *)&s.thS_sh;
        const unsigned long long b = *(volatile unsigned long long *)&s.thO_sh;
        if (a < thS) { thS = a; limS = key_limit(thS); }
        if (b < thO) { thO = b; limO = key_limit(thO); }
    };
    // ---- singles (present edge i, target edge a), strided over the cluster's threads
    {
        const int nS = s.nPE * E;
        const unsigned long long mem_ok = s.mem_ok;
        for (int base = (crank * NWARP + wid) * 32; base < nS; base += CL * ANT) {
            const int t = base + lane;
            bool sv = false;
            uint32_t dsc = 0;
            if (t < nS) {
                const int i = t / E, a = t - (t / E) * E;
                const RemEnt &R = s.se[i];
                if (a != R.r1 && ((mem_ok >> a) & 1ULL) && s.feasS[R.code + s.sl[a]]) {
                    ++cnt;
                    const ARow &A = s.row[a];
                    const AER ae = aer<FAST>(R.b0 + A.thr, R.b1 + A.acc, R.b2 + A.en, R.b3 + A.idle, cc);
                    sv = screen_keep(objective_f(ae.A, ae.E, cc), R, strict, limS, limO);
                    if (MODE == MODE_UNIFORM_ALL)
                        sv = sv || derive_seed4(args.seed, gchain, k, (uint64_t)(R.ibase + a) + 1) <= thP;
                    dsc = 0x80000000u | ((uint32_t)i << 8) | (uint32_t)a;
                }
            }
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, sv);
            if (sv) q[qn + __popc(bal & lt)] = dsc;
            qn += __popc(bal);
            __syncwarp();
            drain(false);
        }
        // paper move set: one-instance add / remove (m changes: scored in full, no screen)
        if (PAPER) {
            const int nU = E + s.nPE;
            for (int base = (crank * NWARP + wid) * 32; base < nU; base += CL * ANT) {
                const int t = base + lane;
                bool sv = false;
                uint32_t dsc = 0;
                if (t < nU) {
                    if (t < E) {
                        sv = ((mem_ok >> t) & 1ULL) && s.feasAR[s.sl[t]];
                        dsc = 0x40000000u | (uint32_t)t;
                    } else {
                        const int r = s.pe_list[t - E];
                        sv = s.feasAR[5 + s.sl[r]] != 0;
                        dsc = 0x40000000u | 0x100u | (uint32_t)r;
                    }
                    cnt += sv ? 1 : 0;
                }
                const unsigned bal = __ballot_sync(0xFFFFFFFFu, sv);
                if (sv) q[qn + __popc(bal & lt)] = dsc;
                qn += __popc(bal);
                __syncwarp();
                drain(false);
            }
        }
        // score the surviving singles now: their records set the doubles' thresholds
        if (PROF && lane == 0) atomicAdd(&s.prof_surv1, (unsigned long long)(nsurv + qn));
        drain(true);
        const unsigned long long kS = warp_min_u64(rS.key), kV = warp_min_u64(rV.key);
        thS = kS < thS ? kS : thS;
        thO = kS < thO ? kS : thO;
        thO = kV < thO ? kV : thO;
        if (MODE == MODE_UNIFORM_ALL) { const unsigned long long kP = warp_min_u64(rP.key); thP = kP < thP ? kP : thP; }
        if (lane == 0) { atomicMin(&s.thS_sh, thS); atomicMin(&s.thO_sh, thO); }
        limS = key_limit(thS); limO = key_limit(thO);
        __syncwarp();
    }
    // ---- doubles: flattened (removal entry, static list entry) space; each warp owns a
    // contiguous chunk, lanes walk it 32 apart (SCREEN_UNR items per lane and iteration)
    const int ND = s.nLen;
    const int W = CL * NWARP;
    const int chunk = (((ND + W - 1) / W) + 31) & ~31;
    const int tb0 = (crank * NWARP + wid) * chunk;
    const int tend = min(tb0 + chunk, ND);
    if (tb0 < ND) {                              // warp-uniform
        int lo = 0, hi = s.nRP - 1;
        const int t0 = min(tb0 + lane, ND - 1);
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (rp[mid].pre <= t0) lo = mid; else hi = mid - 1;
        }
        int j = lo;
        // software pipeline: the move-list words of the next iteration are loaded (L2 latency)
        // while the current iteration is screened
        uint32_t entn[SCREEN_UNR];
        int jn[SCREEN_UNR];
        auto fetch = [&](int b) {
#pragma unroll
            for (int u = 0; u < SCREEN_UNR; ++u) {
                const int tu = min(b + 32 * u + lane, tend - 1);
                while (tu >= rp[j].end) ++j;
                jn[u] = j;
                entn[u] = __ldg(plist + rp[j].offm + tu);
            }
        };
        fetch(tb0);
        for (int base = tb0; base < tend; base += 32 * SCREEN_UNR) {
            refresh();
            uint32_t ent[SCREEN_UNR];
            int jc[SCREEN_UNR];
#pragma unroll
            for (int u = 0; u < SCREEN_UNR; ++u) { ent[u] = entn[u]; jc[u] = jn[u]; }
            if (base + 32 * SCREEN_UNR < tend) fetch(base + 32 * SCREEN_UNR);
            bool sv[SCREEN_UNR];
            uint32_t dsc[SCREEN_UNR];
#pragma unroll
            for (int u = 0; u < SCREEN_UNR; ++u) {
                const int tu = base + 32 * u + lane;
                const RemEnt &R = rp[jc[u]];
                const uint32_t e = ent[u];
                const bool ok = tu < tend && s.feasD[R.code + ((e >> 12) & 31)];
                cnt += ok ? 1 : 0;
                const int a1 = e & 63, a2 = (e >> 6) & 63;
                const ARow &A1 = s.row[a1], &A2 = s.row[a2];
                const AER ae = aer<FAST>(R.b0 + A1.thr + A2.thr, R.b1 + A1.acc + A2.acc,
                                         R.b2 + A1.en + A2.en, R.b3 + A1.idle + A2.idle, cc);
                bool keep = screen_keep(objective_f(ae.A, ae.E, cc), R, strict, limS, limO);
                if (MODE == MODE_UNIFORM_ALL)
                    keep = keep || derive_seed4(args.seed, gchain, k, (uint64_t)(R.ibase + (int)(e >> 17)) + 1) <= thP;
                sv[u] = ok && keep;
                dsc[u] = (uint32_t)jc[u] | ((uint32_t)(tu - R.pre) << 16);
            }
#pragma unroll
            for (int u = 0; u < SCREEN_UNR; ++u) {
                const unsigned bal = __ballot_sync(0xFFFFFFFFu, sv[u]);
                if (sv[u]) q[qn + __popc(bal & lt)] = dsc[u];
                qn += __popc(bal);
            }
            __syncwarp();
            drain(false);
        }
    }
    drain(true);
    if (PROF && lane == 0) atomicAdd(&s.prof_surv, (unsigned long long)nsurv);
}

// Optional phase profiler (CLV_ANNEAL_VARIANT=9): thread 0 of each CTA accumulates
// clock64 deltas between consecutive marks into args.prof[(chain*CL+rank)*PROF_SLOTS + phase];
// slot 7 = prepare cycles of steps that refreshed the slice-delta feasibility, slot 8 = their count.
#define PROF_MARK(ph)                                                                  \
    if (PROF && threadIdx.x == 0) {                                                    \
        const long long _now = clock64();                                              \
        if ((ph) > 0) prof_acc[(ph) - 1] += _now - prof_last;                          \
        prof_last = _now;                                                              \
    }

template <int MODE, int MINB, int UNR, bool PROF = false, int EC = 0, bool PAPER = false>
__global__ void __launch_bounds__(ANT, MINB) anneal_kernel(const __grid_constant__ AnnealArgs args) {
    long long prof_acc[PROF_SLOTS] = {};
    long long prof_last = 0;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    AnnealSmem &s = *reinterpret_cast<AnnealSmem *>(smem_raw);
    RemEnt *const rp = reinterpret_cast<RemEnt *>(smem_raw + sizeof(AnnealSmem));   // E(E+1)/2 entries
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = (int)cluster.num_blocks();
    const int crank = (int)cluster.block_rank();
    // One chain per cluster; with single-CTA clusters and more chains than resident CTAs the
    // launch is persistent: each CTA takes chains from a global counter until none are left
    // (no wave quantisation; chains of different lengths balance).
    const bool persistent = CL == 1 && args.chain_counter != nullptr;
    int chain = persistent ? -1 : (int)(blockIdx.x / CL);
    for (;;) {
    if (persistent) {
        __syncthreads();                     // the previous chain's shared state is no longer read
        if (threadIdx.x == 0) s.next_chain = atomicAdd(args.chain_counter, 1);
        __syncthreads();
        chain = s.next_chain;
    } else if (chain < 0) {
        break;                               // the cluster's one chain is done
    }
    if (chain >= args.n_chains) break;       // whole cluster exits together
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
        s.row[e].t2 = (double)T.t2_q[e];
        s.row[e].t3 = (double)T.t3_q[e];
        s.lat_by_rank[e] = T.lat_by_rank[e];
        s.svc_by_rank[e] = T.svc_by_rank[e];
        s.rbit[e] = 1ULL << T.rank[e];
        s.rk[e] = T.rank[e];
        s.er[e] = T.edge_by_rank[e];
        s.sl[e] = (unsigned char)(e % 5);
    }
    for (int p = tid; p < E * (E + 1) / 2; p += ANT) { s.pair_len[p] = T.pair_len[p]; s.pair_off[p] = T.pair_off[p]; }
    for (int x = tid; x < E; x += ANT)
        for (int y = x; y < E; ++y) s.pair_tab[x * E - (x * (x - 1)) / 2 + (y - x)] = (unsigned short)(x | (y << 8));
    if (tid == 0) {
        s.lat_by_rank[NO_TOP] = 0.0;
        s.mem_ok = T.mem_ok;
        s.magicE = 0xFFFFFFFFu / (unsigned)E + 1u;
        s.magicNP = 0xFFFFFFFFu / (unsigned)(E * (E + 1) / 2) + 1u;
        s.ubase = (unsigned)(E * E) + (unsigned)(E * (E + 1) / 2) * (unsigned)(E * (E + 1) / 2);
        s.ub_dirty = 0;
        s.ec = args.ec[args.n_ec == 1 ? 0 : chain];
    }
    __syncthreads();
    if (tid == 0) {
        const uint16_t *w0 = args.start_w + (size_t)chain * E;
        double S0 = 0, S1 = 0, S2 = 0, S3 = 0, S4 = 0, S5 = 0;
        unsigned long long m = 0;
        for (int k = 0; k < CLV_K; ++k) { s.svec[k] = 0; s.fsvec[k] = -1; }
        for (int e = 0; e < E; ++e) {
            const int x = w0[e];
            s.w[e] = x;
            S0 += x * s.row[e].thr; S1 += x * s.row[e].acc; S2 += x * s.row[e].en; S3 += x * s.row[e].idle;
            S4 += x * s.row[e].t2; S5 += x * s.row[e].t3;
            s.svec[e % 5] += x;
            if (x > 0) m |= s.rbit[e];
        }
        s.S[0] = S0; s.S[1] = S1; s.S[2] = S2; s.S[3] = S3; s.S[4] = S4; s.S[5] = S5;
        s.pmask = m;
        int cnt = 0;
        for (int e = 0; e < E; ++e) { cnt += s.w[e]; s.wr[s.rk[e]] = (double)s.w[e]; }
        s.mcount = (double)cnt;
        s.seedS = ~0ULL; s.seedO = ~0ULL; s.prof_surv = 0ULL; s.prof_surv1 = 0ULL;
        s.thS_sh = ~0ULL; s.thO_sh = ~0ULL;
    }
    __syncthreads();
    {   // pessimistic per-instance tail shares (every GED move keeps m, so W0's bound is per chain)
        const double w0b = w0_bound(s.mcount, s.ec);
        for (int r = tid; r < E; r += ANT) s.ub[r] = s.ec.c20 / (s.svc_by_rank[r] + w0b);
    }

    // ---- chain state: thread 0 of every CTA (identical everywhere); rank 0 writes outputs
    const bool leader = (crank == 0 && tid == 0);
    double hc = 0.0;
    bool slac = false;                       // SLA class of the centre (MODE_BEST_ALL seeds)
    double t_raw = args.t_init;              // multiplicative cooling: t_init (1 - cooling)^k
    unsigned int bk1 = 0;
    unsigned long long bk2 = 0;
    int best_step = -1, stall = 0, steps = 0, status = 0;
    long long best_idx = -1, evals = 1, edge_evals = 0;
    if (tid == 0) {
        int invalid = 0;
        long long tot = 0;
        for (int e = 0; e < E; ++e) {
            tot += s.w[e];
            if (s.w[e] > 0 && !((s.mem_ok >> e) & 1ULL)) invalid = 1;
        }
        if (tot < 1 || !feasible(args.F, n, s.svec[0], s.svec[1], s.svec[2], s.svec[3], s.svec[4])) invalid = 1;
        edge_evals = __popcll(s.pmask);
        const Score sc = epilogue_d(s.S[0], s.S[1], s.S[2], s.S[3], s.S[4], s.S[5], s.mcount, s.ec,
                                    GraphWalk{&s, s.w, s.er, s.pmask});
        hc = sc.h;
        slac = sc.sla;
        bk1 = sc.sla ? 0u : 1u; bk2 = okey(sc.h);
        for (int e = 0; e < E; ++e) s.bw[e] = s.w[e];
        s.dec_done = invalid || (args.max_steps <= 0);
        if (invalid) status = -1;
    }
    cluster.sync();                          // all CTAs started before any DSMEM traffic
    bool done = s.dec_done;
    const int G = CL * ANT;
    const int gt = crank * ANT + tid;
    const unsigned long long mem_ok = s.mem_ok;

    for (int k = 0; !done; ++k) {
        const double mcnt = s.mcount;            // the centre's instance count (paper moves change it)
        PROF_MARK(0);
        bool refreshed = false;
        if (PROF) {
#pragma unroll
            for (int q = 0; q < CLV_K; ++q) refreshed |= (s.svec[q] != s.fsvec[q]);
        }
        const long long prep0 = PROF ? clock64() : 0;
        prepare_step<PROF, PAPER>(s, rp, E, n, args.F, T, s.ec.slo, prof_acc);
        if (PROF && threadIdx.x == 0 && refreshed) { prof_acc[7] += clock64() - prep0; prof_acc[8] += 1; }
        PROF_MARK(1);
        KRec rS = krec_none(), rV = krec_none(), rP = krec_none();
        unsigned long long cnt = 0;
        // ---- singles: (present edge i, target edge a), strided over the cluster
        // (scored modes: screened with the doubles in score_screened)
        if (MODE == MODE_UNIFORM_PROPOSAL) {
            const int nS = s.nPE * E;
            int i = gt / E, a = gt - (gt / E) * E;
            const int dI = G / E, dA = G - (G / E) * E;
            for (int t = gt; t < nS; t += G) {
                const RemEnt &R = s.se[i];
                if (a != R.r1 && ((mem_ok >> a) & 1ULL) && s.feasS[R.code + s.sl[a]]) {
                    ++cnt;
                    const ARow &A = s.row[a];
                    const CandWalk cw{&s, R.pm | s.rbit[a], R.k1, 0xFF, s.rk[a], 0xFF};
                    fold<MODE, EC>(s, args, R.b0 + A.thr, R.b1 + A.acc, R.b2 + A.en,
                               R.b3 + A.idle, R.b4 + A.t2, R.b5 + A.t3, cw, mcnt, R.ibase + a,
                               rS, rV, rP, args.seed, gchain, (uint64_t)k);
                }
                i += dI; a += dA;
                if (a >= E) { a -= E; ++i; }
            }
            if (PAPER) {                             // one-instance add / remove: hash only
                const int nU = E + s.nPE;
                for (int t = gt; t < nU; t += G) {
                    const bool add = t < E;
                    const int e = add ? t : s.pe_list[t - E];
                    if (add ? (((mem_ok >> e) & 1ULL) && s.feasAR[s.sl[e]]) : (s.feasAR[5 + s.sl[e]] != 0)) {
                        ++cnt;
                        score_queued<MODE, EC>(s, args, rp, T.pair_list, 0x40000000u | (add ? 0u : 0x100u) | (uint32_t)e,
                                               mcnt, rS, rV, rP, gchain, (uint64_t)k);
                    }
                }
            }
        }
        // ---- doubles: flattened (removal entry, static list entry) space; each warp
        // owns a contiguous chunk, lanes walk it 32 apart (UNR independent items each)
        if (MODE != MODE_UNIFORM_PROPOSAL) {
            score_screened<MODE, EC, PROF, PAPER>(s, args, rp, T.pair_list, crank, CL, rS, rV, rP, cnt, gchain,
                                           (uint64_t)k);
        } else {
            const int lane = tid & 31, wid = tid >> 5;
            const int ND = s.nLen;
            const int W = CL * NWARP;
            const int chunk = (((ND + W - 1) / W) + 31) & ~31;
            const int tb0 = (crank * NWARP + wid) * chunk;
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
                for (int t = tb0 + lane; t < tend; t += 32 * UNR) {
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const int tu = t + 32 * u;
                        if (tu < tend) {
                            while (tu >= rp[j].end) ++j;
                            const RemEnt &R = rp[j];
                            const uint32_t ent = __ldg(plist + R.offm + tu);
                            if (s.feasD[R.code + ((ent >> 12) & 31)]) {
                                ++cnt;
                                const int a1 = ent & 63, a2 = (ent >> 6) & 63;
                                const ARow &A1 = s.row[a1], &A2 = s.row[a2];
                                const CandWalk cw{&s, R.pm | s.rbit[a1] | s.rbit[a2], R.k1, R.k2,
                                                  s.rk[a1], s.rk[a2]};
                                fold<MODE, EC>(s, args, R.b0 + A1.thr + A2.thr, R.b1 + A1.acc + A2.acc,
                                           R.b2 + A1.en + A2.en, R.b3 + A1.idle + A2.idle,
                                           R.b4 + A1.t2 + A2.t2, R.b5 + A1.t3 + A2.t3, cw, mcnt,
                                           R.ibase + (int)(ent >> 17), rS, rV, rP, args.seed,
                                           gchain, (uint64_t)k);
                            }
                        }
                    }
                }
            }
        }
        PROF_MARK(2);
        // ---- CTA reduction, then DSMEM broadcast of the CTA's records to every CTA
        {
            const int lane = tid & 31, wid = tid >> 5;
            if (MODE != MODE_UNIFORM_PROPOSAL) { rS = krec_min_redux(rS); rV = krec_min_redux(rV); }
            if (MODE != MODE_BEST_ALL) rP = krec_min_warp<MODE == MODE_UNIFORM_ALL>(rP);
            cnt = __reduce_add_sync(0xFFFFFFFFu, (unsigned)cnt);
            if (lane == 0) { s.wS[wid] = rS; s.wV[wid] = rV; s.wP[wid] = rP; s.wc[wid] = cnt; }
            __syncthreads();
            if (wid == 0) {
                rS = lane < NWARP ? s.wS[lane] : krec_none();
                rV = lane < NWARP ? s.wV[lane] : krec_none();
                rP = lane < NWARP ? s.wP[lane] : krec_none();
                cnt = lane < NWARP ? s.wc[lane] : 0ULL;
                if (MODE != MODE_UNIFORM_PROPOSAL) { rS = krec_min_redux(rS); rV = krec_min_redux(rV); }
                if (MODE != MODE_BEST_ALL) rP = krec_min_warp<MODE == MODE_UNIFORM_ALL>(rP);
                cnt = __reduce_add_sync(0xFFFFFFFFu, (unsigned)cnt);
                // (after the xor butterflies every lane holds the CTA result)
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
        // ---- warp 0 merges the cluster's records (lane q: CTA q), then thread 0: best tracking,
        // Eq. 7, termination (every CTA redundantly; rank 0 keeps outputs); warp 0 applies the move
        KRec Sr = krec_none(), Vr = krec_none(), Pr = krec_none();
        unsigned long long total = 0;
        if (tid < 32) {
            const int par = k & 1;
            const KRec a = tid < CL ? s.slS[par][tid] : krec_none();
            const KRec b = tid < CL ? s.slV[par][tid] : krec_none();
            if (MODE != MODE_UNIFORM_PROPOSAL) { Sr = krec_min_redux(a); Vr = krec_min_redux(b); }
            if (MODE != MODE_BEST_ALL) Pr = krec_min_warp<true>(tid < CL ? s.slP[par][tid] : krec_none());
            total = __reduce_add_sync(0xFFFFFFFFu, tid < CL ? (unsigned)s.slc[par][tid] : 0u);
        }
        long long mv_w = NOIDX;
        if (tid == 0) {
            const long long pm0 = PROF ? clock64() : 0;
            if (PROF) prof_acc[17] += pm0 - prof_last;
            long long mv = NOIDX;
            int fin = 0;
            if (total == 0) {
                status = 2;
                fin = 1;
            } else {
                unsigned int ck1;
                unsigned long long ck2;
                long long cidx, pidx;
                double hp, fp = 0.0, Lp = 0.0;
                bool slap = false;
                if (MODE == MODE_UNIFORM_PROPOSAL) {
                    evals += 1;
                    edge_evals += (long long)s.nPE;
                    int r1, r2, a1, a2;
                    decode_move(s, E, Pr.idx, r1, r2, a1, a2);
                    const Score sp = score_move(s, r1, r2, a1, a2);
                    hp = sp.h; fp = sp.f; Lp = sp.L; slap = sp.sla;
                    pidx = Pr.idx;
                    ck1 = sp.sla ? 0u : 1u; ck2 = okey(sp.h); cidx = Pr.idx;
                } else {
                    evals += (long long)total;
                    edge_evals += (long long)s.nPE * (long long)total;
                    // best-tracking candidate: SLA-meeting first
                    if (Sr.idx != 0x7FFFFFFF) { ck1 = 0u; ck2 = Sr.key; cidx = Sr.idx; }
                    else { ck1 = 1u; ck2 = Vr.key; cidx = Vr.idx; }
                    if (MODE == MODE_BEST_ALL) {
                        const bool bs = krec_less(Sr.key, Sr.idx, Vr);
                        const KRec &B = bs ? Sr : Vr;   // min h overall
                        pidx = B.idx; hp = okey_inv(B.key); slap = bs;
                    } else {
                        pidx = Pr.idx; hp = Pr.hv;
                    }
                    if (args.log && leader) {
                        int r1, r2, a1, a2;
                        decode_move(s, E, pidx, r1, r2, a1, a2);
                        const Score sp = score_move(s, r1, r2, a1, a2);
                        fp = sp.f; Lp = sp.L; slap = sp.sla;
                    }
                }
                const bool nb = (ck1 < bk1) || (ck1 == bk1 && ck2 < bk2);
                if (nb) {                          // the best graph is rebuilt at the end (move log)
                    bk1 = ck1; bk2 = ck2; best_step = k; best_idx = cidx; stall = 0;
                } else {
                    stall += 1;
                }
                // subtractive T_k = t_init - k cooling; multiplicative: t_raw *= (1 - cooling) each step
                const double T0 = (args.flags & CLV_ANNEAL_MULT_COOLING) ? t_raw : args.t_init - (double)k * args.cooling;
                const double Tk = args.t_floor >= T0 ? args.t_floor : T0;
                t_raw = t_raw * args.cool_factor;
                bool acc = hp <= hc;                 // Eq. 7: the draw only matters for worse moves
                if (!acc) {
                    const double u = uniform01(derive_seed4(args.seed, gchain, (uint64_t)k, 0ULL));
                    acc = u < exp_clv(-(hp - hc) / Tk);
                }
                if (args.log && leader) {
                    clv_log_row row;
                    row.temp = Tk; row.f = fp; row.h = hp; row.p95_ms = Lp;
                    const long long NPl = (long long)E * (E + 1) / 2;
                    row.iter = k; row.sla_met = slap;
                    row.ged_from_center = pidx < (long long)E * E ? 2 : (pidx < (long long)E * E + NPl * NPl ? 4 : 1);
                    row.accepted = acc; row.new_best = nb; row.n_neighbours = (int)total;
                    args.log[(size_t)chain * args.max_steps + k] = row;
                }
                // screen seeds for the next step: GED moves are symmetric, so after a move the
                // previous centre (h = hc, class slac) is a neighbour of the new centre; without
                // a move the next neighbourhood is this one and its records are achieved keys
                if (MODE != MODE_UNIFORM_PROPOSAL) {
                    if (acc) {
                        s.seedO = okey(hc);
                        s.seedS = (MODE == MODE_BEST_ALL && slac) ? okey(hc) : ~0ULL;
                    } else {
                        s.seedS = Sr.idx != 0x7FFFFFFF ? Sr.key : ~0ULL;
                        s.seedO = krec_less(Sr.key, Sr.idx, Vr) ? Sr.key : Vr.key;
                    }
                }
                s.thS_sh = s.seedS; s.thO_sh = s.seedO;
                if (acc) { hc = hp; mv = pidx; slac = slap; }
                if (leader) args.mvlog[(size_t)chain * args.max_steps + k] = (int)mv;
                steps = k + 1;
                if (stall >= args.stall_limit) { status = 1; fin = 1; }
            }
            if (!fin && k + 1 >= args.max_steps) { status = 0; fin = 1; }
            const long long ap0 = PROF ? clock64() : 0;
            if (PROF) prof_acc[18] += ap0 - pm0;
            mv_w = mv;
            s.dec_done = fin;
            if (PROF) prof_acc[9] += clock64() - ap0;
        }
        if (tid < 32) {
            const long long mvb = __shfl_sync(0xFFFFFFFFu, mv_w, 0);
            if (mvb != NOIDX) apply_move_warp(s, E, mvb, tid);
        }
        PROF_MARK(5);
        __syncthreads();
        done = s.dec_done;
        PROF_MARK(6);
        PROF_MARK(7);
    }
    // Keep every CTA's shared memory alive until no peer can touch it over DSMEM.
    cluster.sync();
    if (PROF && threadIdx.x == 0) { prof_acc[16] = (long long)s.prof_surv; prof_acc[19] = (long long)s.prof_surv1; }
    if (PROF && threadIdx.x == 0 && args.prof)
        for (int q = 0; q < PROF_SLOTS; ++q) args.prof[((size_t)blockIdx.x) * PROF_SLOTS + q] = prof_acc[q];

    if (leader) {
        // best graph = start + the accepted moves of steps < best_step + the best candidate's move
        {
            const uint16_t *w0 = args.start_w + (size_t)chain * E;
            for (int e = 0; e < E; ++e) s.bw[e] = w0[e];
            for (int kk = 0; kk < best_step; ++kk) {
                const int m = args.mvlog[(size_t)chain * args.max_steps + kk];
                if (m >= 0) move_graph(s, E, m, s.bw);
            }
            if (best_step >= 0) move_graph(s, E, best_idx, s.bw);
        }
        clv_chain_result r;
        uint16_t *bw_out = args.best_w + (size_t)chain * E;
        uint16_t *fw_out = args.final_w + (size_t)chain * E;
        double S0 = 0, S1 = 0, S2 = 0, S3 = 0, S4 = 0, S5 = 0;
        unsigned long long m = 0;
        for (int e = 0; e < E; ++e) {
            const int x = s.bw[e];
            bw_out[e] = (uint16_t)x;
            fw_out[e] = (uint16_t)s.w[e];
            S0 += x * s.row[e].thr; S1 += x * s.row[e].acc; S2 += x * s.row[e].en; S3 += x * s.row[e].idle;
            S4 += x * s.row[e].t2; S5 += x * s.row[e].t3;
            if (x > 0) m |= s.rbit[e];
        }
        int mb = 0;
        for (int e = 0; e < E; ++e) mb += s.bw[e];  // paper moves change m: the best graph's own count
        const Score sb = epilogue_d(S0, S1, S2, S3, S4, S5, (double)mb, s.ec, GraphWalk{&s, s.bw, s.er, m});
        r.f = sb.f; r.h = sb.h; r.p95_ms = sb.L; r.accuracy = sb.A; r.energy_wh = sb.E;
        r.sla_met = sb.sla;
        r.status = status; r.steps = steps; r.best_step = best_step;
        r.best_index = best_idx; r.evals = evals; r.edge_evals = edge_evals;
        args.res[chain] = r;
    }
    if (!persistent) chain = -1;
    }   // chains of this CTA
}

template <int MODE, int MINB, int UNR, bool PROF = false>
static cudaError_t launch_mode(const AnnealArgs &a, int cluster_size, cudaStream_t st) {
    // branch-free divisions when every scenario keeps them exact (fast_div_safe)
    // (the paper move set is a template flag: the SPEC-move kernels carry none of its code)
    const bool paper = (a.flags & CLV_ANNEAL_PAPER_MOVES) != 0;
    auto kern = paper ? (!a.fast_div ? anneal_kernel<MODE, MINB, UNR, PROF, 0, true>
                         : a.n_ec == 1 ? anneal_kernel<MODE, MINB, UNR, PROF, 2, true>
                                       : anneal_kernel<MODE, MINB, UNR, PROF, 1, true>)
                      : (!a.fast_div ? anneal_kernel<MODE, MINB, UNR, PROF, 0, false>
                         : a.n_ec == 1 ? anneal_kernel<MODE, MINB, UNR, PROF, 2, false>
                                       : anneal_kernel<MODE, MINB, UNR, PROF, 1, false>);
    const size_t smem = sizeof(AnnealSmem) + sizeof(RemEnt) * (size_t)(a.E * (a.E + 1) / 2);
    // The attribute calls and the cluster-size search (up to 15 occupancy queries) run
    // once per (device, kernel, chains, shared bytes): a re-plan is ~1.5 ms, and these
    // host calls sat between the caller's first event and the launch.
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, int, size_t>, int> chosen;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, reinterpret_cast<const void *>(kern), a.n_chains, smem);
    int cached = 0;                              // auto cluster size (0: not searched yet)
    bool attrs_set = false;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = chosen.find(key);
        if (it != chosen.end()) { attrs_set = true; cached = it->second; }
    }
    if (!attrs_set) {
        // The dynamic shared-memory limit is a per-function attribute: only ever raise it (a
        // smaller family's launch must not lower it under a cached larger configuration).
        static std::map<std::pair<int, const void *>, size_t> smem_set;
        std::lock_guard<std::mutex> lk(mu);
        size_t &cur = smem_set[std::make_pair(dev, reinterpret_cast<const void *>(kern))];
        if (smem > cur) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            cur = smem;
        }
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
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
    if (cluster_size <= 0 && cached > 0) {
        cluster_size = cached;
    } else if (cluster_size <= 0) {
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
        std::lock_guard<std::mutex> lk(mu);
        chosen[key] = cluster_size;
    } else if (!attrs_set) {
        std::lock_guard<std::mutex> lk(mu);
        chosen.emplace(key, 0);                  // attributes set; explicit sizes are not cached
    }
    cfg.gridDim = dim3((unsigned)(a.n_chains * cluster_size), 1, 1);
    attr[0].val.clusterDim.x = (unsigned)cluster_size;
    AnnealArgs b = a;
    b.chain_counter = nullptr;
    if (cluster_size == 1 && a.chain_counter) {
        // more chains than resident CTAs: a persistent grid of resident CTAs taking chains from
        // a counter (no wave tail); otherwise one CTA per chain
        int sms = 148, occ = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, ANT, smem) == cudaSuccess && occ > 0 &&
            a.n_chains > occ * sms) {
            cfg.gridDim = dim3((unsigned)(occ * sms), 1, 1);
            cudaError_t e = cudaMemsetAsync(a.chain_counter, 0, sizeof(int), st);
            if (e != cudaSuccess) return e;
            b.chain_counter = a.chain_counter;
        }
        cudaGetLastError();
    }
    return cudaLaunchKernelEx(&cfg, kern, b);
}

static int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
}

cudaError_t launch_anneal(const AnnealArgs &a, int cluster_size, cudaStream_t st) {
    if (a.proposal == 0) {
        // CLV_ANNEAL_VARIANT=9: the phase-profiling build of the headline mode
        switch (env_int("CLV_ANNEAL_VARIANT", 0)) {
            case 9: return launch_mode<MODE_BEST_ALL, 2, 2, true>(a, cluster_size, st);
            default: return launch_mode<MODE_BEST_ALL, 2, 2>(a, cluster_size, st);
        }
    }
    if (a.evaluate == 0) return launch_mode<MODE_UNIFORM_ALL, 2, 1>(a, cluster_size, st);
    return launch_mode<MODE_UNIFORM_PROPOSAL, 2, 1>(a, cluster_size, st);
}

}  // namespace clv
