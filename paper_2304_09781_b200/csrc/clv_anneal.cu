// clv_anneal.cu -- K3 (GED<=4 neighbour generation + incremental scoring) fused
// with K4 (warp-shuffle argmax) and K5 (anneal step), one thread-block CLUSTER
// per annealing chain, every step of the chain inside one persistent launch.
//
// Reference semantics: sample_neighbor, anneal
// (SPEC:461-469, 478-483), Eqs. 6-7.  Step definition: DESIGN.md
// "Chain step"; CPU restatement: oracle/anneal.py + oracle/neighbours.py.
//
// Layout per CTA (shared memory): the family's per-edge rows {thr, acc, en,
// idle} (int64 fixed point), latency ranks, memory-feasible adjacency lists,
// the chain centre (weights, exact int64 aggregates, presence mask by latency
// rank), the compacted present-edge and removal-pair lists and the slice-delta
// feasibility bytes of this step.  Each CTA of the cluster holds a full copy of
// the centre and scores a strided share of the move space; CTA records meet in
// the leader CTA's shared memory over DSMEM; the leader decides (Eq. 7), and
// every CTA applies the accepted move locally.
#include <cooperative_groups.h>
#include "clv_internal.h"

namespace cg = cooperative_groups;

namespace clv {

constexpr int ANT = 256;                  // threads per CTA
constexpr int NWARP = ANT / 32;
constexpr int MAXP = CLV_MAX_EDGES * (CLV_MAX_EDGES + 1) / 2;   // 820 removal pairs
constexpr uint32_t NOMOVE = 0xFFFFFFFFu;

struct __align__(16) EdgeRow {
    long long thr, acc, en, idle;
};

struct Decision {
    uint32_t mv;
    int done;
};

struct __align__(16) AnnealSmem {
    EdgeRow row[CLV_MAX_EDGES];
    double lat_by_rank[CLV_MAX_EDGES];
    unsigned long long mem_ok;
    unsigned char rank[CLV_MAX_EDGES];
    unsigned char nb_cnt[CLV_MAX_EDGES];
    unsigned char nb[CLV_MAX_EDGES][CLV_NBMAX];
    unsigned short ij_tab[CLV_NBMAX * CLV_NBMAX];
    unsigned short pair_tab[MAXP];
    // centre
    int w[CLV_MAX_EDGES];
    long long S[4];
    int svec[CLV_K];
    unsigned long long pmask;
    unsigned char pe[CLV_MAX_EDGES];
    unsigned short rp[MAXP];
    int nPE, nRP;
    unsigned char feasS[25];
    unsigned char feasD[625];
    // reduction
    Rec wr0[NWARP], wr1[NWARP];
    unsigned long long wc[NWARP];
    // leader-only: one slot per cluster rank
    Rec slot0[16], slot1[16];
    unsigned long long slotc[16];
    Decision dec;
    // leader bookkeeping
    int bw[CLV_MAX_EDGES];
};

__device__ inline bool adjacent(int x, int y) {
    return x != y && ((x / 5) == (y / 5) || (x % 5) == (y % 5));
}

// Score the centre's aggregates shifted by a move (a1,a2 added; r1,r2 removed;
// 0xFF = absent).  Returns the presence mask of the neighbour too.
__device__ inline Score score_move(const AnnealSmem &s, int r1, int r2, int a1, int a2,
                                   const EvalConst &ec) {
    long long t = s.S[0], ac = s.S[1], en = s.S[2], id = s.S[3];
    unsigned long long m = s.pmask;
    if (r1 != 0xFF) {
        t -= s.row[r1].thr; ac -= s.row[r1].acc; en -= s.row[r1].en; id -= s.row[r1].idle;
    }
    if (r2 != 0xFF) {
        t -= s.row[r2].thr; ac -= s.row[r2].acc; en -= s.row[r2].en; id -= s.row[r2].idle;
    }
    if (r1 != 0xFF) {
        int left = s.w[r1] - 1 - (r2 == r1 ? 1 : 0);
        if (left == 0) m &= ~(1ULL << s.rank[r1]);
    }
    if (r2 != 0xFF && r2 != r1) {
        if (s.w[r2] - 1 == 0) m &= ~(1ULL << s.rank[r2]);
    }
    if (a1 != 0xFF) {
        t += s.row[a1].thr; ac += s.row[a1].acc; en += s.row[a1].en; id += s.row[a1].idle;
        m |= 1ULL << s.rank[a1];
    }
    if (a2 != 0xFF) {
        t += s.row[a2].thr; ac += s.row[a2].acc; en += s.row[a2].en; id += s.row[a2].idle;
        m |= 1ULL << s.rank[a2];
    }
    double lmax = s.lat_by_rank[63 - __clzll((long long)m)];
    return epilogue(t, ac, en, id, lmax, ec);
}

__device__ inline void unpack_mv(uint32_t mv, int &r1, int &r2, int &a1, int &a2) {
    r1 = mv & 0xFF; r2 = (mv >> 8) & 0xFF; a1 = (mv >> 16) & 0xFF; a2 = (mv >> 24) & 0xFF;
}

// Apply a move to the CTA-local centre (thread 0) -- O(1).
__device__ inline void apply_move(AnnealSmem &s, uint32_t mv) {
    int r[2], a[2];
    unpack_mv(mv, r[0], r[1], a[0], a[1]);
    for (int k = 0; k < 2; ++k) {
        if (r[k] == 0xFF) continue;
        int e = r[k];
        s.w[e] -= 1;
        s.S[0] -= s.row[e].thr; s.S[1] -= s.row[e].acc; s.S[2] -= s.row[e].en; s.S[3] -= s.row[e].idle;
        s.svec[e % 5] -= 1;
        if (s.w[e] == 0) s.pmask &= ~(1ULL << s.rank[e]);
    }
    for (int k = 0; k < 2; ++k) {
        if (a[k] == 0xFF) continue;
        int e = a[k];
        s.w[e] += 1;
        s.S[0] += s.row[e].thr; s.S[1] += s.row[e].acc; s.S[2] += s.row[e].en; s.S[3] += s.row[e].idle;
        s.svec[e % 5] += 1;
        s.pmask |= 1ULL << s.rank[e];
    }
}

// Rebuild the present-edge list, the removal-pair list and the feasibility
// bytes of all 25 single / 625 double slice deltas (all threads).
__device__ inline void prepare_step(AnnealSmem &s, int E, int n, const FeasView &F) {
    // Ordered (deterministic) compaction: every CTA of the cluster must build
    // identical lists, because the cluster partitions the move space by list
    // position.
    __shared__ int warp_off[NWARP + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int NP = E * (E + 1) / 2;
    int base = 0;
    for (int p0 = 0; p0 < NP; p0 += ANT) {
        const int p = p0 + threadIdx.x;
        bool ok = false;
        int x = 0, y = 0;
        if (p < NP) {
            x = s.pair_tab[p] & 0xFF; y = s.pair_tab[p] >> 8;
            const int wx = s.w[x], wy = s.w[y];
            ok = (x == y) ? (wx >= 2) : (wx > 0 && wy > 0);
        }
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, ok);
        if (lane == 0) warp_off[wid] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            int acc = 0;
            for (int q = 0; q < NWARP; ++q) { int c = warp_off[q]; warp_off[q] = acc; acc += c; }
            warp_off[NWARP] = acc;
        }
        __syncthreads();
        if (ok) s.rp[base + warp_off[wid] + __popc(bal & ((1u << lane) - 1u))] = (unsigned short)(x | (y << 8));
        base += warp_off[NWARP];
        __syncthreads();
    }
    if (wid == 0) {
        int cnt = 0;
        for (int e0 = 0; e0 < E; e0 += 32) {
            const int e = e0 + lane;
            const bool ok = e < E && s.w[e] > 0;
            const unsigned bal = __ballot_sync(0xFFFFFFFFu, ok);
            if (ok) s.pe[cnt + __popc(bal & ((1u << lane) - 1u))] = (unsigned char)e;
            cnt += __popc(bal);
        }
        if (lane == 0) { s.nPE = cnt; s.nRP = base; }
    }
    for (int t = threadIdx.x; t < 650; t += ANT) {
        int v[CLV_K];
#pragma unroll
        for (int k = 0; k < CLV_K; ++k) v[k] = s.svec[k];
        if (t < 25) {
            v[t / 5] -= 1; v[t % 5] += 1;
            bool ok = v[t / 5] >= 0 && feasible(F, n, v[0], v[1], v[2], v[3], v[4]);
            s.feasS[t] = ok;
        } else {
            int u = t - 25;
            v[u / 125] -= 1; v[(u / 25) % 5] -= 1; v[(u / 5) % 5] += 1; v[u % 5] += 1;
            bool ok = v[0] >= 0 && v[1] >= 0 && v[2] >= 0 && v[3] >= 0 && v[4] >= 0 &&
                      feasible(F, n, v[0], v[1], v[2], v[3], v[4]);
            s.feasD[u] = ok;
        }
    }
    __syncthreads();
}

__device__ inline void init_centre(AnnealSmem &s, const uint16_t *w0, int E) {
    if (threadIdx.x == 0) {
        long long S0 = 0, S1 = 0, S2 = 0, S3 = 0;
        unsigned long long m = 0;
        for (int k = 0; k < CLV_K; ++k) s.svec[k] = 0;
        for (int e = 0; e < E; ++e) {
            int x = w0[e];
            s.w[e] = x;
            S0 += (long long)x * s.row[e].thr; S1 += (long long)x * s.row[e].acc;
            S2 += (long long)x * s.row[e].en; S3 += (long long)x * s.row[e].idle;
            s.svec[e % 5] += x;
            if (x > 0) m |= 1ULL << s.rank[e];
        }
        s.S[0] = S0; s.S[1] = S1; s.S[2] = S2; s.S[3] = S3;
        s.pmask = m;
    }
}

__global__ void __launch_bounds__(ANT) anneal_kernel(const __grid_constant__ AnnealArgs args) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    AnnealSmem &s = *reinterpret_cast<AnnealSmem *>(smem_raw);
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = (int)cluster.num_blocks();
    const int crank = (int)cluster.block_rank();
    const int chain = blockIdx.x / CL;
    if (chain >= args.n_chains) return;      // whole cluster exits together
    const long long gchain = args.chain_base + chain;
    const FamilyTables &T = *args.fam;
    const int E = T.E;
    const int n = args.n;
    const EvalConst ec = args.ec[args.n_ec == 1 ? 0 : chain];
    const int tid = threadIdx.x;

    // ---- stage tables
    for (int e = tid; e < E; e += ANT) {
        s.row[e].thr = T.thr_q[e];
        s.row[e].acc = T.acc_q[e];
        s.row[e].en = T.en_q[e];
        s.row[e].idle = T.idle_q[e % 5];
        s.lat_by_rank[e] = T.lat_by_rank[e];
        s.rank[e] = T.rank[e];
        s.nb_cnt[e] = T.nb_cnt[e];
        for (int k = 0; k < CLV_NBMAX; ++k) s.nb[e][k] = T.nb[e][k];
    }
    const int nbm = T.nbmax;
    const int NB2 = nbm * nbm;
    for (int t = tid; t < NB2; t += ANT) s.ij_tab[t] = (unsigned short)(((t / nbm) << 8) | (t % nbm));
    for (int x = tid; x < E; x += ANT)
        for (int y = x; y < E; ++y) s.pair_tab[pair_index(x, y, E)] = (unsigned short)(x | (y << 8));
    if (tid == 0) s.mem_ok = T.mem_ok;
    __syncthreads();
    init_centre(s, args.start_w + (size_t)chain * E, E);
    __syncthreads();

    // ---- leader state (thread 0 of rank 0)
    const bool leader = (crank == 0 && tid == 0);
    double hc = 0.0, fc = 0.0, Lc = 0.0;
    bool slac = false;
    uint32_t bk1 = 0; uint64_t bk2 = 0;
    int best_step = -1, stall = 0, steps = 0, status = 0;
    long long best_idx = -1, evals = 1;
    int invalid = 0;
    if (leader) {
        // start validity: memory-feasible edges only, fleet-feasible slice multiset
        long long tot = 0;
        for (int e = 0; e < E; ++e) {
            tot += s.w[e];
            if (s.w[e] > 0 && !((s.mem_ok >> e) & 1ULL)) invalid = 1;
        }
        if (tot < 1 || !feasible(args.F, n, s.svec[0], s.svec[1], s.svec[2], s.svec[3], s.svec[4]))
            invalid = 1;
        double lmax = s.lat_by_rank[63 - __clzll((long long)(s.pmask | 1ULL))];
        Score sc = epilogue(s.S[0], s.S[1], s.S[2], s.S[3], lmax, ec);
        hc = sc.h; fc = sc.f; Lc = sc.L; slac = sc.sla;
        bk1 = sc.sla ? 0u : 1u; bk2 = okey(sc.h);
        for (int e = 0; e < E; ++e) s.bw[e] = s.w[e];
        s.dec.mv = NOMOVE;
        s.dec.done = invalid || (args.max_steps <= 0);
        if (invalid) status = -1;
    }
    cluster.sync();
    if (tid == 0 && crank != 0) s.dec = *cluster.map_shared_rank(&s.dec, 0);
    __syncthreads();
    bool done = s.dec.done;
    const bool eval_all = (args.evaluate == 0);
    const bool uniform = (args.proposal == 1);
    const int G = CL * ANT;
    const int gt = crank * ANT + tid;
    const unsigned long long mem_ok = s.mem_ok;

    for (int k = 0; !done; ++k) {
        prepare_step(s, E, n, args.F);
        // -------- score this CTA's share of the neighbourhood
        Rec cand = rec_none(), prop = rec_none();
        unsigned long long cnt = 0;
        const int nS = s.nPE * E;
        for (int t = gt; t < nS; t += G) {
            int i = t / E, a = t - i * E;
            int r = s.pe[i];
            if (a == r || !((mem_ok >> a) & 1ULL)) continue;
            if (!s.feasS[(r % 5) * 5 + (a % 5)]) continue;
            ++cnt;
            long long idx = (long long)r * E + a;
            uint32_t mv = (uint32_t)r | 0xFF00u | ((uint32_t)a << 16) | 0xFF000000u;
            Rec rc;
            rc.idx = idx; rc.mv = mv;
            if (eval_all) {
                Score sc = score_move(s, r, 0xFF, a, 0xFF, ec);
                rc.hv = sc.h;
                rc.k1 = sc.sla ? 0u : 1u; rc.k2 = okey(sc.h);
                if (rec_less(rc, cand)) cand = rc;
                rc.k1 = 0u;
                if (uniform) rc.k2 = derive_seed4(args.seed, (uint64_t)gchain, (uint64_t)k, (uint64_t)idx + 1);
                if (rec_less(rc, prop)) prop = rc;
            } else {
                rc.hv = 0.0; rc.k1 = 0u;
                rc.k2 = derive_seed4(args.seed, (uint64_t)gchain, (uint64_t)k, (uint64_t)idx + 1);
                if (rec_less(rc, prop)) prop = rc;
            }
        }
        const int nD = s.nRP * NB2;
        const int NP = E * (E + 1) / 2;
        for (int u = gt; u < nD; u += G) {
            int j = u / NB2, ij = u - j * NB2;
            int r1 = s.rp[j] & 0xFF, r2 = s.rp[j] >> 8;
            int ii = s.ij_tab[ij] >> 8, jj = s.ij_tab[ij] & 0xFF;
            if (ii >= s.nb_cnt[r1] || jj >= s.nb_cnt[r2]) continue;
            int a1 = s.nb[r1][ii], a2 = s.nb[r2][jj];
            if (a1 == r2 || a2 == r1) continue;
            if (a1 > a2 && adjacent(r1, a2) && adjacent(r2, a1)) continue;
            if (!s.feasD[(((r1 % 5) * 5 + (r2 % 5)) * 5 + (a1 % 5)) * 5 + (a2 % 5)]) continue;
            ++cnt;
            int lo = a1 < a2 ? a1 : a2, hi = a1 < a2 ? a2 : a1;
            long long idx = (long long)E * E + (long long)pair_index(r1, r2, E) * NP + pair_index(lo, hi, E);
            uint32_t mv = (uint32_t)r1 | ((uint32_t)r2 << 8) | ((uint32_t)a1 << 16) | ((uint32_t)a2 << 24);
            Rec rc;
            rc.idx = idx; rc.mv = mv;
            if (eval_all) {
                Score sc = score_move(s, r1, r2, a1, a2, ec);
                rc.hv = sc.h;
                rc.k1 = sc.sla ? 0u : 1u; rc.k2 = okey(sc.h);
                if (rec_less(rc, cand)) cand = rc;
                rc.k1 = 0u;
                if (uniform) rc.k2 = derive_seed4(args.seed, (uint64_t)gchain, (uint64_t)k, (uint64_t)idx + 1);
                if (rec_less(rc, prop)) prop = rc;
            } else {
                rc.hv = 0.0; rc.k1 = 0u;
                rc.k2 = derive_seed4(args.seed, (uint64_t)gchain, (uint64_t)k, (uint64_t)idx + 1);
                if (rec_less(rc, prop)) prop = rc;
            }
        }
        // -------- CTA reduction
        {
            int lane = tid & 31, wid = tid >> 5;
            cand = warp_min(cand);
            prop = warp_min(prop);
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, m);
            if (lane == 0) { s.wr0[wid] = cand; s.wr1[wid] = prop; s.wc[wid] = cnt; }
            __syncthreads();
            if (wid == 0) {
                cand = lane < NWARP ? s.wr0[lane] : rec_none();
                prop = lane < NWARP ? s.wr1[lane] : rec_none();
                cnt = lane < NWARP ? s.wc[lane] : 0ULL;
                cand = warp_min(cand);
                prop = warp_min(prop);
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, m);
                if (lane == 0) {
                    AnnealSmem *ls = cluster.map_shared_rank(&s, 0);
                    ls->slot0[crank] = cand;
                    ls->slot1[crank] = prop;
                    ls->slotc[crank] = cnt;
                }
            }
        }
        cluster.sync();
        // -------- leader: decide
        if (leader) {
            Rec C = rec_none(), P = rec_none();
            unsigned long long total = 0;
            for (int q = 0; q < CL; ++q) {
                if (rec_less(s.slot0[q], C)) C = s.slot0[q];
                if (rec_less(s.slot1[q], P)) P = s.slot1[q];
                total += s.slotc[q];
            }
            uint32_t mv_out = NOMOVE;
            int fin = 0;
            if (total == 0) {
                status = 2;
                fin = 1;
            } else {
                double hp, fp = 0.0, Lp = 0.0;
                bool slap = false;
                int r1, r2, a1, a2;
                unpack_mv(P.mv, r1, r2, a1, a2);
                if (eval_all) {
                    evals += (long long)total;
                    hp = P.hv;
                    if (args.log) {
                        Score sp = score_move(s, r1, r2, a1, a2, ec);
                        fp = sp.f; Lp = sp.L; slap = sp.sla;
                    }
                } else {
                    evals += 1;
                    Score sp = score_move(s, r1, r2, a1, a2, ec);
                    hp = sp.h; fp = sp.f; Lp = sp.L; slap = sp.sla;
                    C = P;
                    C.k1 = sp.sla ? 0u : 1u;
                    C.k2 = okey(sp.h);
                }
                bool nb = (C.k1 < bk1) || (C.k1 == bk1 && C.k2 < bk2);
                if (nb) {
                    bk1 = C.k1; bk2 = C.k2; best_step = k; best_idx = C.idx; stall = 0;
                    int c1, c2, c3, c4;
                    unpack_mv(C.mv, c1, c2, c3, c4);
                    for (int e = 0; e < E; ++e) s.bw[e] = s.w[e];
                    if (c1 != 0xFF) s.bw[c1] -= 1;
                    if (c2 != 0xFF) s.bw[c2] -= 1;
                    if (c3 != 0xFF) s.bw[c3] += 1;
                    if (c4 != 0xFF) s.bw[c4] += 1;
                } else {
                    stall += 1;
                }
                double T0 = args.t_init - (double)k * args.cooling;
                double Tk = args.t_floor >= T0 ? args.t_floor : T0;
                double u = uniform01(derive_seed4(args.seed, (uint64_t)gchain, (uint64_t)k, 0ULL));
                bool acc = (hp <= hc) || (u < exp_clv(-(hp - hc) / Tk));
                if (args.log) {
                    clv_log_row row;
                    row.temp = Tk; row.f = fp; row.h = hp; row.p95_ms = Lp;
                    row.iter = k; row.ged_from_center = (r2 == 0xFF) ? 2 : 4; row.sla_met = slap;
                    row.accepted = acc; row.new_best = nb; row.n_neighbours = (int)total;
                    args.log[(size_t)chain * args.max_steps + k] = row;
                }
                if (acc) {
                    hc = hp; fc = fp; Lc = Lp; slac = slap;
                    mv_out = P.mv;
                }
                steps = k + 1;
                if (stall >= args.stall_limit) { status = 1; fin = 1; }
            }
            if (!fin && k + 1 >= args.max_steps) { status = 0; fin = 1; }
            s.dec.mv = mv_out;
            s.dec.done = fin;
        }
        cluster.sync();
        if (tid == 0) {
            Decision d = (crank == 0) ? s.dec : *cluster.map_shared_rank(&s.dec, 0);
            if (d.mv != NOMOVE) apply_move(s, d.mv);
            s.dec = d;
        }
        __syncthreads();
        done = s.dec.done;
        // leader's slots are rewritten only after the next compute phase, which
        // every CTA reaches after this point -- the second cluster.sync orders it.
    }

    if (leader) {
        (void)fc; (void)Lc; (void)slac;
        clv_chain_result r;
        uint16_t *bw_out = args.best_w + (size_t)chain * E;
        uint16_t *fw_out = args.final_w + (size_t)chain * E;
        long long S0 = 0, S1 = 0, S2 = 0, S3 = 0;
        unsigned long long m = 0;
        for (int e = 0; e < E; ++e) {
            int x = s.bw[e];
            bw_out[e] = (uint16_t)x;
            fw_out[e] = (uint16_t)s.w[e];
            S0 += (long long)x * s.row[e].thr; S1 += (long long)x * s.row[e].acc;
            S2 += (long long)x * s.row[e].en; S3 += (long long)x * s.row[e].idle;
            if (x > 0) m |= 1ULL << s.rank[e];
        }
        Score sb = epilogue(S0, S1, S2, S3, s.lat_by_rank[63 - __clzll((long long)(m | 1ULL))], ec);
        r.f = sb.f; r.h = sb.h; r.p95_ms = sb.L; r.accuracy = sb.A; r.energy_wh = sb.E;
        r.sla_met = sb.sla;
        r.status = status; r.steps = steps; r.best_step = best_step;
        r.best_index = best_idx; r.evals = evals;
        args.res[chain] = r;
    }
}

cudaError_t launch_anneal(const AnnealArgs &a, int cluster_size, cudaStream_t st) {
    size_t smem = sizeof(AnnealSmem);
    cudaError_t e = cudaFuncSetAttribute(anneal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (cluster_size > 8) {
        e = cudaFuncSetAttribute(anneal_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.n_chains * cluster_size), 1, 1);
    cfg.blockDim = dim3(ANT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cluster_size;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, anneal_kernel, a);
}

}  // namespace clv
