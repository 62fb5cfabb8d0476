// clv_score.cu -- materialized-candidate scoring (K1+K2+K4), the exhaustive
// ORACLE enumeration (K7), the counter-RNG x-space sweep (K7) and the chain /
// rank winner reductions.
//
//  score_graphs : uint16 graph rows (E = 5V per row) streamed from HBM through a
//                 shared-memory tile, exact int64 aggregates, fp64 epilogue,
//                 fleet-feasibility lookup, grid argmax.       HBM/issue bound
//  score_x      : FleetConfig (x^p, x^v) CSR rows decoded by one thread each over a
//                 shared-memory tile (mig.py:286-296)
//  oracle       : index -> (config id, mixed-radix variant digits)
//  sweep        : index -> counter-RNG draws -> per-pod graphs
#include <algorithm>
#include "clv_internal.h"

namespace clv {

constexpr int SNT = 256;

struct __align__(16) ERow {
    long long thr, acc, en, idle, t2, t3;
};

struct RankTabs {                             // per-family latency-rank tables (shared memory)
    double lat[CLV_MAX_EDGES];                 // lat95 by rank
    double svc[CLV_MAX_EDGES];                 // mean service time by rank
    unsigned char edge[CLV_MAX_EDGES];         // edge at each rank
    unsigned char rank[CLV_MAX_EDGES];         // rank of each edge
};

__device__ inline void stage_ranks(RankTabs &rt, const FamilyTables &T) {
    for (int e = threadIdx.x; e < T.E; e += blockDim.x) {
        rt.lat[e] = T.lat_by_rank[e];
        rt.svc[e] = T.svc_by_rank[e];
        rt.edge[e] = T.edge_by_rank[e];
        rt.rank[e] = T.rank[e];
    }
}

__device__ inline void stage_rows(ERow *row, RankTabs &rt, const FamilyTables &T) {
    for (int e = threadIdx.x; e < T.E; e += blockDim.x) {
        row[e].thr = T.thr_q[e];
        row[e].acc = T.acc_q[e];
        row[e].en = T.en_q[e];
        row[e].idle = T.idle_q[e % 5];
        row[e].t2 = T.t2_q[e];
        row[e].t3 = T.t3_q[e];
    }
    stage_ranks(rt, T);
}

// p95 walker over a weight vector indexed by edge (any integer element type)
template <class W>
struct EdgeWalk {
    const RankTabs *rt;
    const W *w;
    unsigned long long pm;                     // presence by latency rank
    __device__ __forceinline__ double operator()(double W0, double c20) const {
        const RankTabs &t = *rt;
        const W *ww = w;
        return p95_walk(pm, W0, c20, t.svc, t.lat, [&](int r) { return (double)ww[t.edge[r]]; });
    }
};

__device__ inline void consider(RecP &r0, RecP &r1, const Score &sc, long long idx, int mode) {
    RecP c;
    c.f = sc.f; c.L = sc.L; c.A = sc.A; c.E = sc.E; c.sla = sc.sla;
    c.r.idx = idx; c.r.mv = 0u; c.r.hv = sc.h;
    if (mode == CLV_SELECT_BEST_H) {
        c.r.k1 = sc.sla ? 0u : 1u;
        c.r.k2 = okey(sc.h);
        if (rec_less(c.r, r0.r)) r0 = c;
    } else {
        if (sc.sla) {
            c.r.k1 = 0u;
            c.r.k2 = ~okey(sc.f);
            if (rec_less(c.r, r0.r)) r0 = c;
        }
        c.r.k1 = 0u;
        c.r.k2 = okey(sc.L);
        if (rec_less(c.r, r1.r)) r1 = c;
    }
}

// ------------------------------------------------------------ score_graphs
template <bool VEC>
__global__ void __launch_bounds__(SNT) score_graphs_kernel(const __grid_constant__ ScoreArgs a) {
    __shared__ ERow row[CLV_MAX_EDGES];
    __shared__ RankTabs rt;
    __shared__ __align__(16) uint16_t tile[SNT * CLV_MAX_EDGES];
    const FamilyTables &T = *a.fam;
    stage_rows(row, rt, T);
    const int E = T.E;
    const unsigned long long mem_ok = T.mem_ok;
    const int n = a.ec.n;
    RecP r0 = recp_none(), r1 = recp_none();
    unsigned long long c_valid = 0, c_sla = 0;
    __syncthreads();
    for (long long base = (long long)blockIdx.x * SNT; base < a.count; base += (long long)gridDim.x * SNT) {
        const long long rows = (a.count - base) < SNT ? (a.count - base) : SNT;
        const uint16_t *src = a.w + base * E;
        if (VEC) {
            const int nvec = (int)((rows * E * 2) / 16);
            const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
            uint4 *t4 = reinterpret_cast<uint4 *>(tile);
            for (int q = threadIdx.x; q < nvec; q += SNT) t4[q] = __ldcs(s4 + q);
            for (int q = nvec * 8 + threadIdx.x; q < rows * E; q += SNT) tile[q] = src[q];
        } else {
            for (int q = threadIdx.x; q < rows * E; q += SNT) tile[q] = src[q];
        }
        __syncthreads();
        if (threadIdx.x < rows) {
            const uint16_t *w = tile + threadIdx.x * E;
            long long S0 = 0, S1 = 0, S2 = 0, S3 = 0, S4 = 0, S5 = 0;
            int sv[CLV_K] = {0, 0, 0, 0, 0};
            unsigned long long m = 0;
            bool memfail = false;
            for (int e = 0; e < E; ++e) {
                const long long x = w[e];
                if (x) {
                    S0 += x * row[e].thr; S1 += x * row[e].acc; S2 += x * row[e].en; S3 += x * row[e].idle;
                    S4 += x * row[e].t2; S5 += x * row[e].t3;
                    sv[e % 5] += (int)x;
                    m |= 1ULL << rt.rank[e];
                    memfail |= !((mem_ok >> e) & 1ULL);
                }
            }
            const long long i = base + threadIdx.x;
            const bool feas = !memfail && m != 0 && feasible(a.F, n, sv[0], sv[1], sv[2], sv[3], sv[4]);
            if (feas) {
                Score sc = epilogue_d((double)S0, (double)S1, (double)S2, (double)S3, (double)S4, (double)S5,
                                      (double)(sv[0] + sv[1] + sv[2] + sv[3] + sv[4]), a.ec,
                                      EdgeWalk<uint16_t>{&rt, w, m});
                ++c_valid;
                c_sla += sc.sla;
                consider(r0, r1, sc, a.index_base + i, a.select_mode);
                if (a.f_out) a.f_out[i] = sc.f;
                if (a.h_out) a.h_out[i] = sc.h;
                if (a.p95_out) a.p95_out[i] = sc.L;
                if (a.sla_out) a.sla_out[i] = sc.sla;
            } else {
                const double nan = __longlong_as_double(0x7FF8000000000000LL);
                if (a.f_out) a.f_out[i] = nan;
                if (a.h_out) a.h_out[i] = nan;
                if (a.p95_out) a.p95_out[i] = nan;
                if (a.sla_out) a.sla_out[i] = 0;
            }
            if (a.feas_out) a.feas_out[i] = feas;
        }
        __syncthreads();
    }
    grid_finish<SNT>(r0, r1, c_valid, c_sla, a.sel);
}

// TMA-pipelined variant (16-B aligned input): one elected thread streams full
// 256-candidate tiles (256 * 5V * 2 B, a multiple of 16) into a GS-stage shared
// ring with cp.async.bulk + mbarrier complete_tx, so GS-1 tiles are in flight
// while the CTA scores the current one.  Per candidate: exact fp64 FMAs of the
// three per-edge rows (integers < 2^53: exact in any order, = the int64 sums),
// slice counts and the latency-rank presence mask; the idle row is per slice,
// so S_idle = sum_s count_s * idle_s after the loop.  The p95 walk reads the
// candidate's weights back from the staged tile.
constexpr int GS = 2;                       // pipeline stages (2 x 35 KB: 3 CTAs per SM)
constexpr int CPT = 2;                      // candidates per thread
constexpr int GT = SNT * CPT;               // candidates per tile

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile("{\n\t.reg .pred P;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
                 "@!P bra WAIT_%=;\n}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}

// Per-family rows as kernel parameters (constant bank): with the edge loop fully
// unrolled (template on V) every row value is a compile-time constant-bank operand.
struct GraphRows {
    double thr[CLV_MAX_EDGES], acc[CLV_MAX_EDGES], en[CLV_MAX_EDGES], t2[CLV_MAX_EDGES], t3[CLV_MAX_EDGES];
    double idle[CLV_K];
    unsigned long long bad;                 // bit rank(e): edge e is memory-infeasible
    unsigned char rk[CLV_MAX_EDGES];        // latency rank of edge e
};

template <int V, bool FAST>
__global__ void __launch_bounds__(SNT, 3) score_graphs_tma_kernel(const __grid_constant__ ScoreArgs a,
                                                               const __grid_constant__ GraphRows R) {
    constexpr int E = V * CLV_K;
    extern __shared__ __align__(128) unsigned char gsm[];
    __shared__ __align__(8) unsigned long long full[GS];
    __shared__ RankTabs rt;
    uint16_t *ring = reinterpret_cast<uint16_t *>(gsm);
    stage_ranks(rt, *a.fam);
    if (threadIdx.x == 0) {
        for (int q = 0; q < GS; ++q) mbar_init(&full[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long ntiles = (a.count + GT - 1) / GT;
    const int n = a.ec.n;
    // tile j of this CTA is global tile blockIdx.x + j * gridDim.x
    auto issue = [&](long long j) {
        const long long tile = blockIdx.x + j * gridDim.x;
        if (tile >= ntiles) return;
        const long long rows = min((long long)GT, a.count - tile * GT);
        const unsigned bytes = (unsigned)(((size_t)rows * E * 2) & ~(size_t)15);
        const int st = (int)(j % GS);
        // the stage was last touched through the generic proxy (reads, tail stores)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[st], bytes);
        if (bytes) bulk_g2s(ring + (size_t)st * GT * E, a.w + (size_t)tile * GT * E, bytes, &full[st]);
    };
    if (threadIdx.x == 0)
        for (int q = 0; q < GS - 1; ++q) issue(q);
    RecP r0 = recp_none(), r1 = recp_none();
    unsigned long long c_valid = 0, c_sla = 0;
    for (long long j = 0;; ++j) {
        const long long tile = blockIdx.x + j * gridDim.x;
        if (tile >= ntiles) break;
        if (threadIdx.x == 0) issue(j + GS - 1);
        const int st = (int)(j % GS);
        const long long rows = min((long long)GT, a.count - tile * GT);
        uint16_t *buf = ring + (size_t)st * GT * E;
        mbar_wait(&full[st], (unsigned)((j / GS) & 1));
        {   // elements the bulk copy left out (tail of the last, partial tile)
            const size_t done = (((size_t)rows * E * 2) & ~(size_t)15) / 2;
            const size_t tot = (size_t)rows * E;
            if (done < tot) {
                for (size_t q = done + threadIdx.x; q < tot; q += SNT) buf[q] = a.w[(size_t)tile * GT * E + q];
                __syncthreads();
            }
        }
        double S0[CPT], S1[CPT], S2[CPT], S4[CPT], S5[CPT];
        int sv[CPT][CLV_K];
        unsigned long long pe[CPT];
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            S0[c] = S1[c] = S2[c] = S4[c] = S5[c] = 0.0;
            pe[c] = 0ULL;
#pragma unroll
            for (int k = 0; k < CLV_K; ++k) sv[c][k] = 0;
        }
        const uint16_t *w0 = buf + threadIdx.x * E;
#pragma unroll
        for (int e = 0; e < E; ++e) {
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const int x = w0[c * SNT * E + e];
                const double xd = (double)x;
                S0[c] = __fma_rn(xd, R.thr[e], S0[c]);
                S1[c] = __fma_rn(xd, R.acc[e], S1[c]);
                S2[c] = __fma_rn(xd, R.en[e], S2[c]);
                S4[c] = __fma_rn(xd, R.t2[e], S4[c]);
                S5[c] = __fma_rn(xd, R.t3[e], S5[c]);
                sv[c][e % CLV_K] += x;
                pe[c] |= (unsigned long long)(x != 0) << R.rk[e];
            }
        }
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            const int local = threadIdx.x + c * SNT;
            if (local >= rows) continue;
            double S3 = 0.0;
#pragma unroll
            for (int k = 0; k < CLV_K; ++k) S3 = __fma_rn((double)sv[c][k], R.idle[k], S3);
            const long long i = tile * GT + local;
            const bool feas = !(pe[c] & R.bad) && pe[c] != 0 &&
                              feasible(a.F, n, sv[c][0], sv[c][1], sv[c][2], sv[c][3], sv[c][4]);
            if (feas) {
                Score sc = epilogue_t<FAST>(S0[c], S1[c], S2[c], S3, S4[c], S5[c],
                                            (double)(sv[c][0] + sv[c][1] + sv[c][2] + sv[c][3] + sv[c][4]), a.ec,
                                            EdgeWalk<uint16_t>{&rt, w0 + c * SNT * E, pe[c]});
                ++c_valid;
                c_sla += sc.sla;
                consider(r0, r1, sc, a.index_base + i, a.select_mode);
                if (a.f_out) a.f_out[i] = sc.f;
                if (a.h_out) a.h_out[i] = sc.h;
                if (a.p95_out) a.p95_out[i] = sc.L;
                if (a.sla_out) a.sla_out[i] = sc.sla;
            } else {
                const double nan = __longlong_as_double(0x7FF8000000000000LL);
                if (a.f_out) a.f_out[i] = nan;
                if (a.h_out) a.h_out[i] = nan;
                if (a.p95_out) a.p95_out[i] = nan;
                if (a.sla_out) a.sla_out[i] = 0;
            }
            if (a.feas_out) a.feas_out[i] = feas;
        }
        __syncthreads();                     // stage st is free again (re-armed GS-1 tiles later)
    }
    grid_finish<SNT>(r0, r1, c_valid, c_sla, a.sel);
}

template <int V>
static cudaError_t launch_tma(const ScoreArgs &a, const GraphRows &R, cudaStream_t s) {
    auto kern = a.fast ? score_graphs_tma_kernel<V, true> : score_graphs_tma_kernel<V, false>;
    const size_t smem = (size_t)GS * GT * V * CLV_K * 2;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SNT, smem);
    const long long tiles = (a.count + GT - 1) / GT;
    const long long g = std::max(1LL, std::min(tiles, (long long)sms * std::max(occ, 1)));
    kern<<<(unsigned)g, SNT, smem, s>>>(a, R);
    return cudaGetLastError();
}

cudaError_t launch_score_graphs(const ScoreArgs &a, const FamilyTables &T, int grid, cudaStream_t s) {
    const bool aligned = (reinterpret_cast<uintptr_t>(a.w) % 16) == 0;
    if (aligned) {
        GraphRows R{};
        for (int e = 0; e < T.E; ++e) {
            R.thr[e] = (double)T.thr_q[e]; R.acc[e] = (double)T.acc_q[e]; R.en[e] = (double)T.en_q[e];
            R.t2[e] = (double)T.t2_q[e]; R.t3[e] = (double)T.t3_q[e];
            R.rk[e] = T.rank[e];
            if (!((T.mem_ok >> e) & 1ULL)) R.bad |= 1ULL << T.rank[e];
        }
        for (int k = 0; k < CLV_K; ++k) R.idle[k] = (double)T.idle_q[k];
        switch (T.V) {
            case 1: return launch_tma<1>(a, R, s);
            case 2: return launch_tma<2>(a, R, s);
            case 3: return launch_tma<3>(a, R, s);
            case 4: return launch_tma<4>(a, R, s);
            case 5: return launch_tma<5>(a, R, s);
            case 6: return launch_tma<6>(a, R, s);
            case 7: return launch_tma<7>(a, R, s);
            default: return launch_tma<8>(a, R, s);
        }
    }
    score_graphs_kernel<false><<<grid, SNT, 0, s>>>(a);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- score_x
// One thread per FleetConfig row, rows staged through shared memory a tile at a time.
// Read straight from HBM, every byte load of a warp touched 32 different 64..500-B rows
// (32 L1 wavefronts per load); here each warp copies its 32 rows of x^p with coalesced
// byte loads into a padded layout (odd word stride: conflict-free column reads) and the
// CTA copies the tile's x^v span (off[c0] .. off[c0 + rows]) with 16-B loads.  The walk
// is flattened over the assignment slots -- one iteration per slot, the next GPU's
// partition fetched by a single predicated refill (every partition has 1..7 slices,
// mig.py:103-110) -- so lanes with 1-slice and 7-slice partitions do not serialise.
// Per slot the thread only bumps its own 16-bit count of the (variant, slice) bucket
// (counts laid out [bucket][thread]: conflict-free); the rows -- one 16-B int4 of the
// fixed-point values, each < 2^31 -- are applied once per edge after the walk
// (S = sum_e count_e * row_e, exact int64), which also yields the presence mask for
// the p95 term and the memory-fit check; the p95 walk then reads the counts of the
// ranks it visits.  Rows longer than 65,535 slots take the direct per-slot sum (and
// recount the visited edges from the row).
//
// Validation follows FleetConfig.__init__ (mig.py:248-263) then the SPEC's evaluation
// (SPEC:267-275): an unknown partition id anywhere in the row -> InvalidConfigError;
// else a length mismatch -> CarbonSchedError; else a variant < 1 -> CarbonSchedError;
// else a variant > V or a memory-infeasible (variant, slice) -> InfeasibleAssignmentError.
// Across candidates the LOWEST failing index is reported (a sequential loop raises at
// the first bad row): one 64-bit atomicMin of (index << 8 | code).
constexpr int XT = 128;                     // candidates (= threads) per tile
constexpr int X_SMEM = 40 * 1024;           // dynamic staging bytes: x^p tile, then x^v span (4 CTAs / SM)


template <bool XP_SMEM, bool XV_SMEM, bool HIST>
__device__ __forceinline__ void walk_row(unsigned short *hc, const uint8_t *xpr, const uint8_t *xvr, int mcnt, int n,
                                         int V, const unsigned *cfg, const int4 *row, const int2 *row2,
                                         const unsigned char *rank_ok, long long &S0, long long &S1, long long &S2,
                                         long long &S3, long long &S4, long long &S5, unsigned long long &m,
                                         int &err) {
    // cfg[id]: bit 31 valid, bits 24..27 slice count (1..7), bits 0..20 slice kinds (3 bits each).
    // HIST: slot counts per bucket b = min(v, V + 1) * 5 + kind -- bucket row 0 holds the
    // variants < 1, rows 1..V the edges (v - 1) * 5 + kind, row V + 1 the variants > V --
    // so the per-slot path has no checks at all.  A refill past the last GPU (more
    // variants than slices) re-reads GPU n - 1: such a row is a length error anyway.
    int g = 0, left = 0, bad_id = 0, lt1 = 0, infeas = 0, expected = 0;
    unsigned kw = 0;
    for (int p = 0; p < mcnt; ++p) {
        if (left == 0) {
            const unsigned c = cfg[XP_SMEM ? xpr[min(g, n - 1)] : __ldg(xpr + min(g, n - 1))];
            const int ns = (c >> 24) & 15;                 // 0 for an unknown id
            bad_id |= !(c >> 31);
            expected += g < n ? ns : 0;
            left = ns > 0 ? ns : 1;
            kw = c; ++g;
        }
        const int v = XV_SMEM ? xvr[p] : __ldg(xvr + p);
        const int kind = kw & 7;
        kw >>= 3; --left;
        if (HIST) {
            hc[(min(v, V + 1) * 5 + kind) * XT] += 1;
        } else {
            lt1 |= v == 0;
            const bool vok = (unsigned)(v - 1) < (unsigned)V;
            const int e = vok ? (v - 1) * 5 + kind : 0;
            const int4 R = row[e];
            const int2 R2 = row2[e];
            const unsigned ro = rank_ok[e];
            infeas |= !vok || !ro;
            S0 += R.x; S1 += R.y; S2 += R.z; S3 += R.w; S4 += R2.x; S5 += R2.y;
            m |= 1ULL << (ro & 63);
        }
    }
    if (HIST) {                                        // apply the rows (the caller zeroes the counts)
        const int NB = 5 * (V + 2);
        for (int b = 0; b < NB; ++b) {
            const unsigned c = hc[b * XT];
            if (b < 5) { lt1 |= c != 0; continue; }
            if (b >= 5 * (V + 1)) { infeas |= c != 0; continue; }
            const int4 R = row[b - 5];
            const int2 R2 = row2[b - 5];
            const unsigned ro = rank_ok[b - 5];
            S0 += (long long)c * R.x; S1 += (long long)c * R.y; S2 += (long long)c * R.z; S3 += (long long)c * R.w;
            S4 += (long long)c * R2.x; S5 += (long long)c * R2.y;
            if (c) { m |= 1ULL << (ro & 63); infeas |= !ro; }
        }
    }
    // the rest of the partition row: every id must be known (InvalidConfigError comes
    // first, mig.py:254) and its slices count towards the expected length
    for (; g < n; ++g) {
        const unsigned c = cfg[XP_SMEM ? xpr[g] : __ldg(xpr + g)];
        bad_id |= !(c >> 31);
        expected += (c >> 24) & 15;
    }
    err = bad_id ? CLV_ERR_INVALID_CONFIG
        : expected != mcnt ? CLV_ERR_CARBON_SCHED
        : lt1 ? SCORE_X_VARIANT_LT1
        : infeas ? CLV_ERR_INFEASIBLE_ASSIGNMENT : 0;
}

// Slots of a row that land on edge e (the long-row path keeps no per-edge counts).
__device__ inline int count_edge_slots(const uint8_t *xpr, const uint8_t *xvr, int mcnt, int n, const unsigned *cfg,
                                       int e) {
    int g = 0, left = 0, cntv = 0;
    unsigned kw = 0;
    for (int p = 0; p < mcnt; ++p) {
        if (left == 0) {
            const unsigned c = cfg[__ldg(xpr + min(g, n - 1))];
            const int ns = (c >> 24) & 15;
            left = ns > 0 ? ns : 1;
            kw = c; ++g;
        }
        const int v = __ldg(xvr + p);
        const int kind = kw & 7;
        kw >>= 3; --left;
        cntv += (v >= 1 && (v - 1) * 5 + kind == e);
    }
    return cntv;
}

template <bool FAST>
__global__ void __launch_bounds__(XT) score_x_kernel(const __grid_constant__ ScoreArgs a, int n, int xp_stride,
                                                     int xv_cap) {
    __shared__ int4 row[CLV_MAX_EDGES];
    __shared__ int2 row2[CLV_MAX_EDGES];               // rate-moment rows t2_q, t3_q
    __shared__ RankTabs rt;
    __shared__ unsigned char rank_ok[CLV_MAX_EDGES];   // 0x40 | rank when memory-feasible, else 0
    __shared__ unsigned cfg[256];
    __shared__ unsigned short hist[(CLV_MAX_EDGES + 10) * XT];  // [bucket][thread] slot counts of the row
    extern __shared__ __align__(16) uint8_t xsm[];
    // x^p rows at xp_stride (n padded to an odd number of words; 0 = n too large to stage)
    uint8_t *sxp = xsm, *sxv = xsm + XT * xp_stride;
    const FamilyTables &T = *a.fam;
    const Topology &P = *a.topo;
    for (int e = threadIdx.x; e < CLV_MAX_EDGES; e += XT) {
        const bool live = e < T.E;
        row[e] = live ? make_int4((int)T.thr_q[e], (int)T.acc_q[e], (int)T.en_q[e], (int)T.idle_q[e % 5])
                      : make_int4(0, 0, 0, 0);
        row2[e] = live ? make_int2((int)T.t2_q[e], (int)T.t3_q[e]) : make_int2(0, 0);
        rank_ok[e] = (live && ((T.mem_ok >> e) & 1ULL)) ? (unsigned char)(0x40 | T.rank[e]) : 0;
    }
    stage_ranks(rt, T);
    for (int t = threadIdx.x; t < 256; t += XT) cfg[t] = 0u;
    for (int q = threadIdx.x; q < (CLV_MAX_EDGES + 10) * XT; q += XT) hist[q] = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < P.K; r += XT) {
        if (P.ids[r] >= 0 && P.ids[r] < 256 && P.nslices[r] >= 1 && P.nslices[r] <= 7) {
            unsigned kw = 0;
            for (int j = 0; j < P.nslices[r]; ++j) kw |= (unsigned)P.kinds[r][j] << (3 * j);
            cfg[P.ids[r]] = 0x80000000u | ((unsigned)P.nslices[r] << 24) | kw;
        }
    }
    __syncthreads();
    const int V = T.V;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    RecP r0 = recp_none(), r1 = recp_none();
    unsigned long long c_valid = 0, c_sla = 0;
    const long long ntiles = (a.count + XT - 1) / XT;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long c0 = tile * XT;
        const int rows = (int)min((long long)XT, a.count - c0);
        const long long G0 = __ldg(a.xv_off + c0), G1 = __ldg(a.xv_off + c0 + rows);
        const bool xv_fits = (G1 - G0) + 16 <= xv_cap;
        __syncthreads();                                   // previous tile's rows are consumed
        if (xp_stride) {                                   // warp w copies rows 32w .. 32w + 31
            const int r_end = min(32 * wid + 32, rows);
            for (int r = 32 * wid; r < r_end; ++r) {
                const uint8_t *g = a.xp + (c0 + r) * n;
                for (int q = lane; q < n; q += 32) sxp[r * xp_stride + q] = __ldcs(g + q);
            }
        }
        int lead = 0;
        if (xv_fits) {
            // sxv[k] holds the byte at (aligned-down address of xv + G0) + k; whole 16-B
            // chunks inside [G0, G1) are vector loads, the partial head / tail chunks bytes
            const uint8_t *g0 = a.xv + G0;
            lead = (int)(reinterpret_cast<uintptr_t>(g0) & 15);
            const uint8_t *ga = g0 - lead;
            const long long len = G1 - G0;
            const long long nch = (lead + len + 15) >> 4;
            for (long long q = threadIdx.x; q < nch; q += XT) {
                const long long lo = (q << 4) - lead;             // chunk bytes [lo, lo + 16) relative to G0
                if (lo >= 0 && lo + 16 <= len) {
                    reinterpret_cast<uint4 *>(sxv)[q] = __ldcs(reinterpret_cast<const uint4 *>(ga) + q);
                } else {
                    for (int b = 0; b < 16; ++b)
                        if (lo + b >= 0 && lo + b < len) sxv[(q << 4) + b] = g0[lo + b];
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < rows) {
            const long long c = c0 + threadIdx.x;
            const long long o0 = __ldg(a.xv_off + c), o1 = __ldg(a.xv_off + c + 1);
            long long S0 = 0, S1 = 0, S2 = 0, S3 = 0, S4 = 0, S5 = 0;
            unsigned long long m = 0;
            int err;
            unsigned short *hc = hist + threadIdx.x;
            const uint8_t *gxr = a.xv + o0, *gxpr = a.xp + c * n;
            const bool long_row = o1 - o0 > 0xFFFF;
            if (o1 - o0 < 0 || o1 - o0 > 0x7FFFFFFFLL) {
                err = CLV_ERR_CARBON_SCHED;
            } else {
                const int mcnt = (int)(o1 - o0);
                const uint8_t *sxr = sxv + lead + (o0 - G0);
                const uint8_t *sxpr = sxp + threadIdx.x * xp_stride;
                if (mcnt > 0xFFFF)
                    walk_row<false, false, false>(hc, gxpr, gxr, mcnt, n, V, cfg, row, row2, rank_ok, S0, S1, S2, S3, S4, S5, m, err);
                else if (xp_stride && xv_fits)
                    walk_row<true, true, true>(hc, sxpr, sxr, mcnt, n, V, cfg, row, row2, rank_ok, S0, S1, S2, S3, S4, S5, m, err);
                else if (xp_stride)
                    walk_row<true, false, true>(hc, sxpr, gxr, mcnt, n, V, cfg, row, row2, rank_ok, S0, S1, S2, S3, S4, S5, m, err);
                else
                    walk_row<false, false, true>(hc, gxpr, gxr, mcnt, n, V, cfg, row, row2, rank_ok, S0, S1, S2, S3, S4, S5, m, err);
            }
            if (err) {
                atomicMin(a.error_key, ((unsigned long long)c << 8) | (unsigned)err);
                if (a.sla_out) a.sla_out[c] = 0;
            } else {
                const int mc = (int)(o1 - o0);
                Score sc = epilogue_t<FAST>((double)S0, (double)S1, (double)S2, (double)S3, (double)S4, (double)S5,
                                            (double)mc, a.ec, [&](double W0, double c20) {
                    return p95_walk(m, W0, c20, rt.svc, rt.lat, [&](int r) {
                        const int e = rt.edge[r];
                        return (double)(long_row ? count_edge_slots(gxpr, gxr, mc, n, cfg, e) : hc[(e + 5) * XT]);
                    });
                });
                ++c_valid;
                c_sla += sc.sla;
                consider(r0, r1, sc, a.index_base + c, a.select_mode);
                if (a.f_out) a.f_out[c] = sc.f;
                if (a.h_out) a.h_out[c] = sc.h;
                if (a.sla_out) a.sla_out[c] = sc.sla;
            }
            if (!long_row)
                for (int b = 0; b < 5 * (V + 2); ++b) hc[b * XT] = 0;
        }
    }
    grid_finish<XT>(r0, r1, c_valid, c_sla, a.sel);
}

cudaError_t launch_score_x(const ScoreArgs &a, int n, int max_grid, cudaStream_t s) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // n padded to whole words, the word count made odd (row r's word w sits in bank
    // (r * stride / 4 + w) mod 32: distinct across a warp's rows)
    const int stride = ((n + 3) & ~3) | 4;
    const int xp_stride = (long long)XT * stride <= X_SMEM / 2 ? stride : 0;
    const int xv_cap = X_SMEM - XT * xp_stride;
    auto kern = a.fast ? score_x_kernel<true> : score_x_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, X_SMEM);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, XT, X_SMEM);
    const long long tiles = (a.count + XT - 1) / XT;
    const long long g = std::max(1LL, std::min({tiles, (long long)sms * std::max(occ, 1), (long long)max_grid}));
    kern<<<(unsigned)g, XT, X_SMEM, s>>>(a, n, xp_stride, xv_cap);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ oracle
template <bool FAST>
// 3 CTAs per SM (85 registers): +8 % over the 2 that 122 registers allowed
__global__ void __launch_bounds__(SNT, 3) oracle_kernel(const __grid_constant__ OracleArgs a) {
    __shared__ ERow row[CLV_MAX_EDGES];
    __shared__ RankTabs rt;
    __shared__ unsigned char flist[CLV_K][CLV_MAX_VARIANTS];
    const FamilyTables &T = *a.fam;
    const Topology &P = *a.topo;
    stage_rows(row, rt, T);
    for (int t = threadIdx.x; t < CLV_K * CLV_MAX_VARIANTS; t += SNT)
        flist[t / CLV_MAX_VARIANTS][t % CLV_MAX_VARIANTS] = T.feas_list[t / CLV_MAX_VARIANTS][t % CLV_MAX_VARIANTS];
    __syncthreads();
    const long long n = a.n;
    RecP r0 = recp_none(), r1 = recp_none();
    unsigned long long c_valid = 0, c_sla = 0;
    int r = 0;                                 // a thread's indices ascend: resume the row search
    for (long long i = a.begin + (long long)blockIdx.x * SNT + threadIdx.x; i < a.end;
         i += (long long)gridDim.x * SNT) {
        while (r + 1 < P.K && a.row_off[r + 1] <= i) ++r;
        // within a row the index is < 8^7 (variants per slice ^ slices): 32-bit digits
        unsigned rem = (unsigned)(i - a.row_off[r]);
        long long S0 = 0, S1 = 0, S2 = 0, S3 = 0, S4 = 0, S5 = 0;
        unsigned long long m = 0;
        const int ns = P.nslices[r];
        unsigned long long rks = 0;                // latency rank of slice j in byte j
        for (int j = 0; j < ns; ++j) {
            const unsigned pl = (unsigned)a.row_place[r][j];
            const int dgt = (int)(rem / pl);
            rem -= (unsigned)dgt * pl;
            const int k = P.kinds[r][j];
            const int e = flist[k][dgt] * 5 + k;
            S0 += row[e].thr; S1 += row[e].acc; S2 += row[e].en; S3 += row[e].idle;
            S4 += row[e].t2; S5 += row[e].t3;
            m |= 1ULL << rt.rank[e];
            rks |= (unsigned long long)rt.rank[e] << (8 * j);
        }
        const double nd = (double)n;
        Score sc = epilogue_t<FAST>((double)(S0 * n), (double)(S1 * n), (double)(S2 * n), (double)(S3 * n),
                                    (double)(S4 * n), (double)(S5 * n), (double)(n * ns), a.ec,
                                    [&](double W0, double c20) {
            return p95_walk(m, W0, c20, rt.svc, rt.lat, [&](int rr) {
                int c = 0;
                for (int j = 0; j < ns; ++j) c += (int)((rks >> (8 * j)) & 0xFF) == rr;
                return (double)c * nd;             // exact: the standardized graph is n x the row
            });
        });
        ++c_valid;
        c_sla += sc.sla;
        consider(r0, r1, sc, i, CLV_SELECT_ORACLE);
    }
    grid_finish<SNT>(r0, r1, c_valid, c_sla, a.sel);
}

cudaError_t launch_oracle(const OracleArgs &a, int grid, cudaStream_t s) {
    if (a.fast) oracle_kernel<true><<<grid, SNT, 0, s>>>(a);
    else oracle_kernel<false><<<grid, SNT, 0, s>>>(a);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- sweep
// The candidate's counter stream (oracle/rng.py::Stream): 32-bit draws, low then
// high half of splitmix64 word j of the stream keyed by h0.  The word base
// h0 + (j+1)*golden is advanced incrementally instead of multiplied out.
struct Draws {
    uint64_t zb, word;
    uint32_t j;
    __device__ inline void init(uint64_t h0) { zb = h0; word = 0; j = 0; }
    __device__ inline uint32_t next() {
        uint32_t out;
        if ((j & 1u) == 0) {
            zb += 0x9E3779B97F4A7C15ULL;
            uint64_t z = zb;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            word = z ^ (z >> 31);
            out = (uint32_t)word;
        } else {
            out = (uint32_t)(word >> 32);
        }
        ++j;
        return out;
    }
};

struct __align__(16) SRow {
    double thr, acc, en, idle, t2, t3;
};

constexpr int ZROW = CLV_MAX_EDGES;           // all-zero row: a configuration draw adds nothing

// HIST: each variant draw only bumps the thread's 16-bit count of its edge ([edge][thread]
// layout in shared memory: conflict-free), and the rows are applied once per edge after the
// pod (S = sum_e count_e * row_e: the same exact integers, so the same fp64 sums); the
// configuration's slice kinds and count come from one packed word, the pod's per-kind
// variant counts from a register.  Counts stay below 2^16 while 7 * n_gpus < 65,536.
template <bool FAST, bool HIST>
// 4 CTAs per SM (64 registers): +20 % over the 2 that 106 registers allowed
__global__ void __launch_bounds__(SNT, 4) sweep_kernel(const __grid_constant__ SweepArgs a) {
    __shared__ SRow row[CLV_MAX_PODS][CLV_MAX_EDGES + 1];
    __shared__ unsigned long long rbit[CLV_MAX_PODS][CLV_MAX_EDGES + 1];
    __shared__ RankTabs rt[CLV_MAX_PODS];
    __shared__ unsigned char nfeas[CLV_MAX_PODS][CLV_K];
    __shared__ unsigned char flist[CLV_MAX_PODS][CLV_K][CLV_MAX_VARIANTS];
    __shared__ unsigned char nsl[CLV_MAX_CONFIGS];
    __shared__ unsigned char kinds[CLV_MAX_CONFIGS][8];
    __shared__ __align__(16) unsigned cfgw[CLV_MAX_CONFIGS];   // kinds (3 bits each) | slice count << 24
    __shared__ __align__(16) int pod_e[CLV_MAX_PODS];
    __shared__ unsigned short hist[HIST ? (CLV_MAX_EDGES + 1) * SNT : 1];
    const Topology &P = *a.topo;
    for (int p = 0; p < a.n_pods; ++p) {
        const FamilyTables &T = a.fam[a.pods[p].family];
        for (int e = threadIdx.x; e <= CLV_MAX_EDGES; e += SNT) {
            const bool real = e < T.E;
            row[p][e].thr = real ? (double)T.thr_q[e] : 0.0;
            row[p][e].acc = real ? (double)T.acc_q[e] : 0.0;
            row[p][e].en = real ? (double)T.en_q[e] : 0.0;
            row[p][e].idle = real ? (double)T.idle_q[e % 5] : 0.0;
            row[p][e].t2 = real ? (double)T.t2_q[e] : 0.0;
            row[p][e].t3 = real ? (double)T.t3_q[e] : 0.0;
            rbit[p][e] = real ? (1ULL << T.rank[e]) : 0ULL;
        }
        stage_ranks(rt[p], T);
        for (int t = threadIdx.x; t < CLV_K * CLV_MAX_VARIANTS; t += SNT) {
            flist[p][t / CLV_MAX_VARIANTS][t % CLV_MAX_VARIANTS] = T.feas_list[t / CLV_MAX_VARIANTS][t % CLV_MAX_VARIANTS];
            if (t < CLV_K) nfeas[p][t] = T.nfeas[t];
        }
        if (threadIdx.x == 0) pod_e[p] = T.E;
    }
    for (int r = threadIdx.x; r < P.K; r += SNT) {
        nsl[r] = (unsigned char)P.nslices[r];
        unsigned kw = 0;
        for (int j = 0; j < 8; ++j) {
            kinds[r][j] = P.kinds[r][j];
            if (j < 7 && j < P.nslices[r]) kw |= (unsigned)P.kinds[r][j] << (3 * j);
        }
        cfgw[r] = kw | ((unsigned)P.nslices[r] << 24);
    }
    if (HIST)
        for (int q = threadIdx.x; q < (CLV_MAX_EDGES + 1) * SNT; q += SNT) hist[q] = 0;
    __syncthreads();
    const uint32_t K = (uint32_t)P.K;
    unsigned short *hc = hist + (HIST ? threadIdx.x : 0);
    RecP r0 = recp_none(), r1 = recp_none();
    unsigned long long c_valid = 0, c_sla = 0;
    for (long long i = a.begin + (long long)blockIdx.x * SNT + threadIdx.x; i < a.end;
         i += (long long)gridDim.x * SNT) {
        Draws d;
        d.init(derive_seed2(a.seed, (uint64_t)i));
        double f = 0.0, h = 0.0;
        bool sla = true;
        for (int p = 0; p < a.n_pods; ++p) {
            // fp64 sums of exact integers (< 2^53): identical to the oracle's int64 sums
            double S0 = 0.0, S1 = 0.0, S2 = 0.0, S3 = 0.0, S4 = 0.0, S5 = 0.0;
            unsigned long long m = 0;
            // One draw per iteration, in the oracle's order (oracle/search.py::draw_candidate):
            // a configuration draw when the current GPU's slices are exhausted, else the next
            // slice's variant draw.  The body is branch-free (a configuration draw adds the
            // all-zero row), so lanes stay converged until their last GPU.
            const int ng = a.pods[p].n_gpus;
            const Draws d0 = d;                          // the pod's first draw (recount path)
            int g = 0, rem = 0, r = 0, slot = 0, inst = 0;
            if (HIST) {
                unsigned nfw = 0;                        // per-kind feasible-variant counts, 4 bits each
#pragma unroll
                for (int k = 0; k < CLV_K; ++k) nfw |= (unsigned)nfeas[p][k] << (4 * k);
                unsigned kw = 0;
                while (rem != 0 || g < ng) {
                    const uint32_t w = d.next();
                    const bool cfg = rem == 0;
                    const int k = kw & 7;
                    const int v = flist[p][k][__umulhi(w, (nfw >> (4 * k)) & 15u)];
                    const int e = cfg ? ZROW : v * 5 + k;
                    hc[e * SNT] += 1;
                    const unsigned cwn = cfgw[__umulhi(w, K)];
                    kw = cfg ? (cwn & 0x1FFFFFu) : (kw >> 3);
                    rem = cfg ? (int)(cwn >> 24) : rem - 1;
                    g += cfg ? 1 : 0;
                    inst += cfg ? 0 : 1;
                }
                const int E = pod_e[p];
                for (int e = 0; e < E; ++e) {
                    const unsigned c = hc[e * SNT];
                    const double cd = (double)c;
                    const SRow &q = row[p][e];
                    S0 = __fma_rn(cd, q.thr, S0); S1 = __fma_rn(cd, q.acc, S1);
                    S2 = __fma_rn(cd, q.en, S2); S3 = __fma_rn(cd, q.idle, S3);
                    S4 = __fma_rn(cd, q.t2, S4); S5 = __fma_rn(cd, q.t3, S5);
                    m |= c ? rbit[p][e] : 0ULL;
                }
            } else {
                while (rem != 0 || g < ng) {
                    const uint32_t w = d.next();
                    const bool cfg = rem == 0;
                    const int k = kinds[r][slot & 7];
                    const int v = flist[p][k][(int)(((uint64_t)w * nfeas[p][k]) >> 32)];
                    const int e = cfg ? ZROW : v * 5 + k;
                    const SRow &q = row[p][e];
                    S0 += q.thr; S1 += q.acc; S2 += q.en; S3 += q.idle; S4 += q.t2; S5 += q.t3;
                    m |= rbit[p][e];
                    const int rn = (int)(((uint64_t)w * K) >> 32);
                    r = cfg ? rn : r;
                    rem = cfg ? (int)nsl[rn] : rem - 1;
                    slot = cfg ? 0 : slot + 1;
                    g += cfg ? 1 : 0;
                    inst += cfg ? 0 : 1;
                }
            }
            // the p95 walk reads the visited edges' counts (HIST), or recounts them by
            // replaying the pod's draws (pods with 7 n >= 2^16)
            Score sc = epilogue_t<FAST>(S0, S1, S2, S3, S4, S5, (double)inst, a.pods[p].ec,
                                        [&](double W0, double c20) {
                return p95_walk(m, W0, c20, rt[p].svc, rt[p].lat, [&](int rr) {
                    const int e0 = rt[p].edge[rr];
                    if (HIST) return (double)hc[e0 * SNT];
                    Draws dd = d0;
                    int gg = 0, rm = 0, rw = 0, sl = 0, cntv = 0;
                    while (rm != 0 || gg < ng) {
                        const uint32_t w = dd.next();
                        const bool cf = rm == 0;
                        const int k = kinds[rw][sl & 7];
                        const int v = flist[p][k][(int)(((uint64_t)w * nfeas[p][k]) >> 32)];
                        cntv += (!cf && v * 5 + k == e0);
                        const int rn = (int)(((uint64_t)w * K) >> 32);
                        rw = cf ? rn : rw;
                        rm = cf ? (int)nsl[rn] : rm - 1;
                        sl = cf ? 0 : sl + 1;
                        gg += cf ? 1 : 0;
                    }
                    return (double)cntv;
                });
            });
            if (HIST) {
                for (int e = 0; e < pod_e[p]; ++e) hc[e * SNT] = 0;
                hc[ZROW * SNT] = 0;
            }
            const double wt = a.pods[p].weight;
            if (p == 0) { f = wt * sc.f; h = wt * sc.h; }
            else { f = f + wt * sc.f; h = h + wt * sc.h; }
            sla = sla && sc.sla;
        }
        Score comb;
        comb.f = f; comb.h = h; comb.L = 0.0; comb.A = 0.0; comb.E = 0.0; comb.sla = sla;
        ++c_valid;
        c_sla += sla;
        consider(r0, r1, comb, i, CLV_SELECT_BEST_H);
        const long long o = i - a.begin;
        if (a.f_out) a.f_out[o] = f;
        if (a.h_out) a.h_out[o] = h;
        if (a.sla_out) a.sla_out[o] = sla;
    }
    grid_finish<SNT>(r0, r1, c_valid, c_sla, a.sel);
}

cudaError_t launch_sweep(const SweepArgs &a, int grid, cudaStream_t s) {
    bool hist = true;                              // 16-bit edge counts cannot overflow
    for (int p = 0; p < a.n_pods; ++p) hist = hist && 7LL * a.pods[p].n_gpus < 65536;
    if (hist) {
        if (a.fast) sweep_kernel<true, true><<<grid, SNT, 0, s>>>(a);
        else sweep_kernel<false, true><<<grid, SNT, 0, s>>>(a);
    } else {
        if (a.fast) sweep_kernel<true, false><<<grid, SNT, 0, s>>>(a);
        else sweep_kernel<false, false><<<grid, SNT, 0, s>>>(a);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------- chain / rank winner
__device__ inline void rec_min_block(clv_record &best) {
    __shared__ clv_record sm[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int m = 16; m >= 1; m >>= 1) {
        clv_record o;
        o.k1 = __shfl_xor_sync(0xFFFFFFFFu, best.k1, m);
        o.k2 = __shfl_xor_sync(0xFFFFFFFFu, best.k2, m);
        o.index = __shfl_xor_sync(0xFFFFFFFFu, best.index, m);
        o.h = __shfl_xor_sync(0xFFFFFFFFu, best.h, m);
        bool less = o.k1 != best.k1 ? o.k1 < best.k1 : (o.k2 != best.k2 ? o.k2 < best.k2 : o.index < best.index);
        if (less) best = o;
    }
    if (lane == 0) sm[wid] = best;
    __syncthreads();
    if (wid == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        clv_record none = {~0ULL, ~0ULL, 0x7FFFFFFFFFFFFFFFLL, 0.0};
        best = lane < nw ? sm[lane] : none;
        for (int m = 16; m >= 1; m >>= 1) {
            clv_record o;
            o.k1 = __shfl_xor_sync(0xFFFFFFFFu, best.k1, m);
            o.k2 = __shfl_xor_sync(0xFFFFFFFFu, best.k2, m);
            o.index = __shfl_xor_sync(0xFFFFFFFFu, best.index, m);
            o.h = __shfl_xor_sync(0xFFFFFFFFu, best.h, m);
            bool less = o.k1 != best.k1 ? o.k1 < best.k1 : (o.k2 != best.k2 ? o.k2 < best.k2 : o.index < best.index);
            if (less) best = o;
        }
    }
}

__global__ void select_chains_kernel(const clv_chain_result *res, int n_chains, long long chain_base,
                                     clv_record *out) {
    clv_record best = {~0ULL, ~0ULL, 0x7FFFFFFFFFFFFFFFLL, 0.0};
    for (int c = threadIdx.x; c < n_chains; c += blockDim.x) {
        const clv_chain_result &r = res[c];
        if (r.status < 0) continue;
        clv_record x;
        x.k1 = r.sla_met ? 0ULL : 1ULL;
        x.k2 = okey(r.h);
        x.index = chain_base + c;
        x.h = r.h;
        bool less = x.k1 != best.k1 ? x.k1 < best.k1 : (x.k2 != best.k2 ? x.k2 < best.k2 : x.index < best.index);
        if (less) best = x;
    }
    rec_min_block(best);
    if (threadIdx.x == 0) *out = best;
}

cudaError_t launch_select_chains(const clv_chain_result *res, int n_chains, long long chain_base,
                                 clv_record *out, cudaStream_t s) {
    select_chains_kernel<<<1, 256, 0, s>>>(res, n_chains, chain_base, out);
    return cudaGetLastError();
}

__global__ void reduce_records_kernel(const clv_record *recs, int count, clv_record *out) {
    clv_record best = {~0ULL, ~0ULL, 0x7FFFFFFFFFFFFFFFLL, 0.0};
    for (int c = threadIdx.x; c < count; c += blockDim.x) {
        clv_record x = recs[c];
        bool less = x.k1 != best.k1 ? x.k1 < best.k1 : (x.k2 != best.k2 ? x.k2 < best.k2 : x.index < best.index);
        if (less) best = x;
    }
    rec_min_block(best);
    if (threadIdx.x == 0) *out = best;
}

cudaError_t launch_reduce_records(const clv_record *recs, int count, clv_record *out, cudaStream_t s) {
    reduce_records_kernel<<<1, 256, 0, s>>>(recs, count, out);
    return cudaGetLastError();
}

}  // namespace clv
