// clv_sim.cu -- batched discrete-event serving simulator (SPEC serving-sim,
// reference SPEC.md:316-393): one independent simulation per
// candidate fleet, bit-identical to the CPU restatement oracle/des.py.
//
// Model: integer-nanosecond time; Poisson (counter RNG) or
// periodic arrivals in [0, duration); one global FIFO queue with instance-pull
// dispatch, i.e. request i (arrival order) is served by the instance that became
// idle first, argmin (free_j, j), start = max(a_i, free_j); service = mean, or the
// mean times a unit-mean exponential / lognormal multiplier of request i (common
// random numbers across candidates); warm-up = the first W completions by
// (completion, request); nearest-rank p95; energy = active energy per request +
// idle power x idle time per instance over [0, max(duration, last completion)].
//
// Device layout:
//   * once per workload (cached in the context): arrival times a[N] (int64 ns,
//     exact prefix sums of rounded exponential gaps), and per-request draws
//     ex[N] (unit exponential) and z[N] (standard normal), shared by every fleet;
//   * sim_kernel: one WARP per simulation for the sequential queue recursion.
//     Instance free times live in the warp's shared-memory slab; lane l owns
//     instances j = l (mod 32) and caches its own (min free, index); each request
//     is one 3-step redux.sync argmin over the lanes, the owner lane serves it and
//     rescans its slots.  Completions go to a per-warp HBM scratch row c[N]
//     (coalesced 32-request stores).  Then the whole CTA post-processes its
//     simulations one at a time: 11-bit radix selections for the warm-up cut (key
//     = completion << b | request) and the nearest-rank p95 over the remaining
//     latencies, exact integer sums for mean latency / busy / idle time, and the
//     fixed-order fp64 energy and accuracy epilogue.
#include <algorithm>
#include <climits>
#include <cmath>
#include <vector>
#include "clv_ctx.h"

namespace clv {

struct SimFamily {
    int V, E, any_random, pad;
    unsigned long long mem_ok;
    double mean_ns[CLV_MAX_EDGES];
    double sigma[CLV_MAX_EDGES];
    double hs[CLV_MAX_EDGES];                // (0.5 * sigma) * sigma
    long long det_ns[CLV_MAX_EDGES];         // floor(mean_ns + 0.5)
    int dist[CLV_MAX_EDGES];
    double energy_wh[CLV_MAX_EDGES];
    double idle_w[CLV_K];
    double acc[CLV_MAX_VARIANTS];
};

struct SimState {
    bool fam_set[CLV_MAX_FAMILIES] = {};
    SimFamily fam[CLV_MAX_FAMILIES];
    SimFamily *fam_dev = nullptr;
    // prepared workload (arrivals + draws)
    bool prepared = false;
    double rate = 0.0, dur = 0.0;
    uint64_t seed = 0;
    int periodic = 0;
    long long N = 0, cap = 0, d_ns = 0;
    long long *a = nullptr;
    double *ex = nullptr, *z = nullptr;
    long long *n_dev = nullptr;
    long long *n_host = nullptr;             // pinned
    // completion scratch: slots x N int64
    long long *c_scr = nullptr;
    size_t scr_elems = 0;
};

void sim_destroy(SimState *s) {
    if (!s) return;
    cudaFree(s->fam_dev);
    cudaFree(s->a); cudaFree(s->ex); cudaFree(s->z); cudaFree(s->n_dev);
    cudaFreeHost(s->n_host);
    cudaFree(s->c_scr);
    delete s;
}

constexpr int SNW = 8;                       // simulations (warps) per CTA
constexpr int SNT = SNW * 32;
constexpr int RBITS = 11;                    // radix-select digit
constexpr int RBINS = 1 << RBITS;
constexpr double TWO_M53 = 1.0 / 9007199254740992.0;
constexpr double TWO_M52 = 1.0 / 4503599627370496.0;

__host__ __device__ inline uint64_t derive_seed3(uint64_t a, uint64_t b, uint64_t c) {
    return seed_round(seed_round(seed_round(0x9E3779B97F4A7C15ULL, a), b), c) & 0x7FFFFFFFFFFFFFFFULL;
}

__host__ __device__ inline long long round_ns(double x) { return (long long)floor(x + 0.5); }

// Per-request draws and (Poisson) rounded gaps / (periodic) arrival times.
__global__ void sim_draws_kernel(uint64_t seed, long long cap, int periodic, long long period, double scale,
                                 long long *a, double *ex, double *z) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cap;
         i += (long long)gridDim.x * blockDim.x) {
        if (periodic) {
            a[i] = i * period;
        } else {
            const double u = (double)((derive_seed3(seed, 1, (uint64_t)i) >> 10) + 1) * TWO_M53;
            const double g = -log_clv(u);
            a[i] = round_ns(g * scale);
        }
        const double v = (double)((derive_seed3(seed, 2, (uint64_t)i) >> 10) + 1) * TWO_M53;
        ex[i] = -log_clv(v);
        const double w = ((double)(derive_seed3(seed, 3, (uint64_t)i) >> 11) + 0.5) * TWO_M52;
        z[i] = ndtri_clv(w);
    }
}

// Single-CTA exact inclusive scan of the gaps (int64: any order is exact), then
// the number of arrivals before the horizon (a is non-decreasing).
__global__ void __launch_bounds__(1024) sim_scan_kernel(long long *a, long long cap, long long d_ns, long long *n_out) {
    __shared__ long long part[1024];
    __shared__ long long wsum[32];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const long long chunk = (cap + 1023) / 1024;
    const long long lo = t * chunk, hi = min(cap, lo + chunk);
    long long s = 0;
    for (long long i = lo; i < hi; ++i) s += a[i];
    long long x = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const long long y = __shfl_up_sync(0xFFFFFFFFu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
        long long w = wsum[lane];
        long long wx = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long y = __shfl_up_sync(0xFFFFFFFFu, wx, d);
            if (lane >= d) wx += y;
        }
        wsum[lane] = wx - w;
    }
    __syncthreads();
    long long run = wsum[wid] + x - s;
    part[t] = run;
    for (long long i = lo; i < hi; ++i) { run += a[i]; a[i] = run; }
    __syncthreads();
    if (t == 0) {
        long long l = 0, h = cap;                 // first index with a >= d_ns
        while (l < h) {
            const long long m = (l + h) >> 1;
            if (a[m] < d_ns) l = m + 1; else h = m;
        }
        *n_out = l;
    }
}

struct SimArgs {
    const SimFamily *fam;
    const long long *a;
    const double *ex, *z;
    long long N, d_ns, W;
    double duration_s, l_tail;
    long long count;
    const uint8_t *inst_edge;
    const int64_t *inst_off;
    int kmax, key_bits;
    long long *c_scr;
    clv_sim_report *rep;
    int64_t *vcnt;
    int64_t *icnt;
};

__device__ __forceinline__ long long service_ns(const SimFamily &F, int e, double exi, double zi) {
    const int d = F.dist[e];
    if (d == 0) return F.det_ns[e];
    if (d == 1) return round_ns(F.mean_ns[e] * exi);
    return round_ns(F.mean_ns[e] * exp_clv(F.sigma[e] * zi - F.hs[e]));
}

// CTA-wide exclusive scan of one value per thread; returns the exclusive prefix, *total the sum.
__device__ __forceinline__ unsigned long long block_exscan(unsigned long long v, unsigned long long *wbuf,
                                                          unsigned long long *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) wbuf[wid] = x;
    __syncthreads();
    if (wid == 0) {
        const unsigned long long w = lane < SNW ? wbuf[lane] : 0ULL;
        unsigned long long wx = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, wx, d);
            if (lane >= d) wx += y;
        }
        if (lane < SNW) wbuf[lane] = wx - w;
        if (lane == SNW - 1) wbuf[SNW] = wx;
    }
    __syncthreads();
    const unsigned long long r = wbuf[wid] + x - v;
    *total = wbuf[SNW];
    __syncthreads();
    return r;
}

__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, unsigned long long *wbuf) {
    unsigned long long tot;
    block_exscan(v, wbuf, &tot);
    return tot;
}

__device__ __forceinline__ long long block_max(long long v, long long *wbuf) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, m));
    if (lane == 0) wbuf[wid] = v;
    __syncthreads();
    long long r = wbuf[0];
    for (int q = 1; q < SNW; ++q) r = max(r, wbuf[q]);
    __syncthreads();
    return r;
}

// k-th smallest (1-based) key among the elements passing `filt`, by RBITS-bit
// radix digits from the top of an nbits-wide key space (CTA-wide).
template <class KeyF, class FiltF>
__device__ unsigned long long radix_select(long long N, long long k, int nbits, KeyF key, FiltF filt,
                                           unsigned *hist, unsigned long long *wbuf, long long *bc) {
    unsigned long long prefix = 0, mask = 0;
    long long rank = k;
    const int top = ((nbits - 1) / RBITS) * RBITS;
    for (int shift = top; shift >= 0; shift -= RBITS) {
        for (int t = threadIdx.x; t < RBINS; t += SNT) hist[t] = 0u;
        __syncthreads();
        for (long long i = threadIdx.x; i < N; i += SNT) {
            if (!filt(i)) continue;
            const unsigned long long kv = key(i);
            if ((kv & mask) == prefix) atomicAdd(&hist[(kv >> shift) & (RBINS - 1)], 1u);
        }
        __syncthreads();
        constexpr int PER = RBINS / SNT;
        unsigned loc[PER];
        unsigned long long s = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) { loc[q] = hist[threadIdx.x * PER + q]; s += loc[q]; }
        unsigned long long tot;
        const unsigned long long ex = block_exscan(s, wbuf, &tot);
        if ((long long)ex < rank && rank <= (long long)(ex + s)) {
            unsigned long long cum = ex;
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                if (rank <= (long long)(cum + loc[q])) {
                    bc[0] = threadIdx.x * PER + q;
                    bc[1] = rank - (long long)cum;
                    break;
                }
                cum += loc[q];
            }
        }
        __syncthreads();
        prefix |= (unsigned long long)bc[0] << shift;
        mask |= (unsigned long long)(RBINS - 1) << shift;
        rank = bc[1];
        __syncthreads();
    }
    return prefix;
}

template <bool RAND>
__global__ void __launch_bounds__(SNT) sim_kernel(const __grid_constant__ SimArgs args) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ SimFamily F;
    __shared__ unsigned hist[RBINS];
    __shared__ unsigned long long wbuf[SNW + 1];
    __shared__ long long bc[2];
    __shared__ long long lbuf[SNW];
    __shared__ int s_status[SNW], s_K[SNW];
    __shared__ unsigned long long cnt_e[CLV_MAX_EDGES], idle_s[CLV_K];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kmax = args.kmax;
    {
        const int *src = reinterpret_cast<const int *>(args.fam);
        int *dst = reinterpret_cast<int *>(&F);
        for (int q = tid; q < (int)(sizeof(SimFamily) / 4); q += SNT) dst[q] = src[q];
    }
    // per-warp slab: free[kmax] int64 | busy[kmax] int64 | cnt[kmax] u32 | edge[kmax] u8
    const size_t slab = (size_t)kmax * 21 + 16;
    const size_t slab_al = (slab + 15) & ~(size_t)15;
    const long long N = args.N;
    __syncthreads();

    for (long long base = (long long)blockIdx.x * SNW; base < args.count; base += (long long)gridDim.x * SNW) {
        const long long sim = base + warp;
        unsigned char *my = smem_raw + slab_al * warp;
        long long *fr = reinterpret_cast<long long *>(my);
        long long *bs = fr + kmax;
        unsigned *cn = reinterpret_cast<unsigned *>(bs + kmax);
        unsigned char *ed = reinterpret_cast<unsigned char *>(cn + kmax);
        long long *cs = args.c_scr + ((long long)blockIdx.x * SNW + warp) * N;
        int status = 0, K = 0;
        if (sim < args.count) {
            const long long o0 = args.inst_off[sim], o1 = args.inst_off[sim + 1];
            K = (int)(o1 - o0);
            if (o1 - o0 < 1 || o1 - o0 > kmax) {
                status = CLV_ERR_SIMULATION;
            } else {
                int bad = 0;
                for (int t = lane; t < K; t += 32) {
                    const int e = args.inst_edge[o0 + t];
                    if (e >= F.E) bad |= 2;
                    else if (!((F.mem_ok >> e) & 1ULL)) bad |= 1;
                    ed[t] = (unsigned char)e; fr[t] = 0; bs[t] = 0; cn[t] = 0u;
                }
                bad = __reduce_or_sync(0xFFFFFFFFu, bad);
                if (bad & 2) status = CLV_ERR_SIMULATION;
                else if (bad & 1) status = CLV_ERR_INFEASIBLE_ASSIGNMENT;
            }
            __syncwarp();
            if (status == 0) {
                long long lmin = lane < K ? 0LL : LLONG_MAX;
                unsigned lidx = lane < K ? (unsigned)lane : 0xFFFFFFFFu;
                for (long long b = 0; b < N; b += 32) {
                    const long long i = b + lane;
                    long long al = 0;
                    double exl = 0.0, zl = 0.0;
                    if (i < N) {
                        al = __ldg(args.a + i);
                        if (RAND) { exl = __ldg(args.ex + i); zl = __ldg(args.z + i); }
                    }
                    const int nb = (int)min(32LL, N - b);
                    long long myc = 0;
                    for (int r = 0; r < nb; ++r) {
                        const long long ai = __shfl_sync(0xFFFFFFFFu, al, r);
                        const unsigned hi = (unsigned)((unsigned long long)lmin >> 32), lo = (unsigned)lmin;
                        const unsigned mh = __reduce_min_sync(0xFFFFFFFFu, hi);
                        const unsigned ml = __reduce_min_sync(0xFFFFFFFFu, hi == mh ? lo : 0xFFFFFFFFu);
                        const unsigned mj = __reduce_min_sync(0xFFFFFFFFu, (hi == mh && lo == ml) ? lidx : 0xFFFFFFFFu);
                        const long long fv = (long long)(((unsigned long long)mh << 32) | ml);
                        const long long start = ai > fv ? ai : fv;
                        double exi = 0.0, zi = 0.0;
                        if (RAND) { exi = __shfl_sync(0xFFFFFFFFu, exl, r); zi = __shfl_sync(0xFFFFFFFFu, zl, r); }
                        long long c = 0;
                        const int owner = (int)(mj & 31u);
                        if (lane == owner) {
                            const long long s = service_ns(F, ed[mj], exi, zi);
                            c = start + s;
                            fr[mj] = c;
                            bs[mj] += s;
                            cn[mj] += 1u;
                            long long m = LLONG_MAX;
                            unsigned mi = 0xFFFFFFFFu;
                            for (int t = lane; t < K; t += 32) {
                                const long long v = fr[t];
                                if (v < m) { m = v; mi = (unsigned)t; }
                            }
                            lmin = m; lidx = mi;
                        }
                        c = __shfl_sync(0xFFFFFFFFu, c, owner);
                        if (lane == r) myc = c;
                    }
                    if (i < N) cs[i] = myc;
                }
            }
        }
        if (lane == 0) { s_status[warp] = status; s_K[warp] = K; }
        __syncthreads();

        // ---- CTA-wide post-processing of this CTA's simulations, one at a time
        for (int w = 0; w < SNW; ++w) {
            const long long sw = base + w;
            if (sw >= args.count) break;
            int st = s_status[w];
            const int Kw = s_K[w];
            const long long *cw = args.c_scr + ((long long)blockIdx.x * SNW + w) * N;
            unsigned char *mw = smem_raw + slab_al * w;
            const long long *bw = reinterpret_cast<const long long *>(mw) + kmax;
            const unsigned *nw = reinterpret_cast<const unsigned *>(bw + kmax);
            const unsigned char *ew = reinterpret_cast<const unsigned char *>(nw + kmax);
            clv_sim_report rp;
            memset(&rp, 0, sizeof(rp));
            if (st == 0) {
                long long mx = 0;
                for (long long i = tid; i < N; i += SNT) mx = max(mx, cw[i]);
                const long long t_end = max(args.d_ns, block_max(mx, lbuf));
                const int b = args.key_bits;
                if (t_end >= (1LL << (63 - b))) st = CLV_ERR_SIMULATION;   // completion key would overflow
                if (st == 0) {
                    const int cbits = 64 - __clzll((long long)t_end);
                    auto ckey = [&](long long i) -> unsigned long long {
                        return ((unsigned long long)cw[i] << b) | (unsigned long long)i;
                    };
                    long long theta = -1;
                    if (args.W > 0)
                        theta = (long long)radix_select(N, args.W, cbits + b, ckey,
                                                        [&](long long) { return true; }, hist, wbuf, bc);
                    auto counted = [&](long long i) { return (long long)ckey(i) > theta; };
                    const long long M = N - args.W;
                    const long long kr = (95 * M + 99) / 100;
                    const unsigned long long p = radix_select(
                        N, kr, cbits, [&](long long i) { return (unsigned long long)(cw[i] - __ldg(args.a + i)); },
                        counted, hist, wbuf, bc);
                    unsigned long long ls = 0;
                    for (long long i = tid; i < N; i += SNT)
                        if (counted(i)) ls += (unsigned long long)(cw[i] - __ldg(args.a + i));
                    const unsigned long long lsum = block_sum(ls, wbuf);
                    // per-instance aggregation (exact integers)
                    for (int q = tid; q < CLV_MAX_EDGES; q += SNT) cnt_e[q] = 0ULL;
                    if (tid < CLV_K) idle_s[tid] = 0ULL;
                    __syncthreads();
                    for (int t = tid; t < Kw; t += SNT) {
                        const int e = ew[t];
                        atomicAdd(&cnt_e[e], (unsigned long long)nw[t]);
                        atomicAdd(&idle_s[e % CLV_K], (unsigned long long)(t_end - bw[t]));
                        if (args.icnt) args.icnt[args.inst_off[sw] + t] = (int64_t)nw[t];
                    }
                    __syncthreads();
                    if (tid == 0) {
                        double active = 0.0;
                        for (int e = 0; e < F.E; ++e) active = active + (double)cnt_e[e] * F.energy_wh[e];
                        double total = active;
                        for (int s = 0; s < CLV_K; ++s) total = total + F.idle_w[s] * (double)idle_s[s] / 3.6e12;
                        double acc = 0.0;
                        unsigned long long cv[CLV_MAX_VARIANTS];
                        for (int v = 0; v < CLV_MAX_VARIANTS; ++v) {
                            cv[v] = 0ULL;
                            if (v < F.V)
                                for (int s = 0; s < CLV_K; ++s) cv[v] += cnt_e[v * CLV_K + s];
                        }
                        for (int v = 0; v < F.V; ++v) acc = acc + (double)cv[v] * F.acc[v];
                        acc = acc / (double)N;
                        rp.p95_ms = (double)p / 1e6;
                        rp.mean_latency_ms = ((double)lsum / (double)M) / 1e6;
                        rp.throughput_rps = (double)N / args.duration_s;
                        rp.energy_wh_total = total;
                        rp.energy_wh_per_request = active / (double)N;
                        rp.accuracy = acc;
                        rp.completed = N;
                        rp.counted = M;
                        rp.sla_met = rp.p95_ms <= args.l_tail ? 1 : 0;
                        if (args.vcnt)
                            for (int v = 0; v < CLV_MAX_VARIANTS; ++v) args.vcnt[sw * CLV_MAX_VARIANTS + v] = (int64_t)cv[v];
                    }
                }
            }
            if (tid == 0) {
                rp.status = st;
                args.rep[sw] = rp;
            }
            __syncthreads();
        }
        __syncthreads();
    }
}

}  // namespace clv

using namespace clv;

namespace {

int sfail(clv_ctx *c, int code, const std::string &msg) {
    c->err = msg;
    return code;
}

int scuda(clv_ctx *c, cudaError_t e, const char *where) {
    return sfail(c, e == cudaErrorMemoryAllocation ? CLV_ERR_OUT_OF_MEMORY : CLV_ERR_CUDA,
                 std::string(where) + ": " + cudaGetErrorString(e));
}

#define SIM_CUDA(call, where)                              \
    do {                                                   \
        cudaError_t _e = (call);                           \
        if (_e != cudaSuccess) return scuda(ctx, _e, where); \
    } while (0)

SimState *state(clv_ctx *ctx) {
    if (!ctx->sim) ctx->sim = new SimState();
    return ctx->sim;
}

int prepare_workload(clv_ctx *ctx, SimState *S, const clv_workload &w, cudaStream_t st) {
    if (S->prepared && S->rate == w.arrival_rps && S->dur == w.duration_s && S->seed == w.seed &&
        S->periodic == (w.periodic ? 1 : 0))
        return CLV_OK;
    S->prepared = false;
    const long long d_ns = round_ns(w.duration_s * 1e9);
    const double lam = w.arrival_rps * w.duration_s;
    long long period = 0, cap;
    if (w.periodic) {
        period = round_ns(1e9 / w.arrival_rps);
        if (period < 1) period = 1;
        cap = (d_ns + period - 1) / period;
    } else {
        cap = (long long)(lam + 10.0 * std::sqrt(lam) + 1024.0);
    }
    if (cap > (1LL << 31) - 1) return sfail(ctx, CLV_ERR_SIMULATION, "workload has more than 2^31 requests");
    if (!S->n_host) SIM_CUDA(cudaMallocHost(&S->n_host, sizeof(long long)), "pinned n");
    if (!S->n_dev) SIM_CUDA(cudaMalloc(&S->n_dev, sizeof(long long)), "alloc n");
    const double scale = 1e9 / w.arrival_rps;
    for (int attempt = 0; attempt < 8; ++attempt) {
        if (cap > S->cap) {
            cudaFree(S->a); cudaFree(S->ex); cudaFree(S->z);
            S->a = nullptr; S->ex = S->z = nullptr; S->cap = 0;
            SIM_CUDA(cudaMalloc(&S->a, sizeof(long long) * std::max(1LL, cap)), "alloc arrivals");
            SIM_CUDA(cudaMalloc(&S->ex, sizeof(double) * std::max(1LL, cap)), "alloc draws");
            SIM_CUDA(cudaMalloc(&S->z, sizeof(double) * std::max(1LL, cap)), "alloc draws");
            S->cap = cap;
        }
        const int grid = (int)std::min<long long>((cap + 255) / 256, (long long)ctx->sm_count * 8);
        sim_draws_kernel<<<std::max(grid, 1), 256, 0, st>>>(w.seed, cap, w.periodic ? 1 : 0, period, scale,
                                                            S->a, S->ex, S->z);
        SIM_CUDA(cudaGetLastError(), "sim draws");
        long long N;
        if (w.periodic) {
            N = cap;
        } else {
            sim_scan_kernel<<<1, 1024, 0, st>>>(S->a, cap, d_ns, S->n_dev);
            SIM_CUDA(cudaGetLastError(), "sim scan");
            SIM_CUDA(cudaMemcpyAsync(S->n_host, S->n_dev, sizeof(long long), cudaMemcpyDeviceToHost, st), "copy n");
            SIM_CUDA(cudaStreamSynchronize(st), "synchronize");
            N = *S->n_host;
            if (N >= cap) {                      // every drawn arrival precedes the horizon: draw more
                cap *= 2;
                if (cap > (1LL << 31) - 1) return sfail(ctx, CLV_ERR_SIMULATION, "workload has more than 2^31 requests");
                continue;
            }
        }
        S->N = N;
        S->d_ns = d_ns;
        S->rate = w.arrival_rps; S->dur = w.duration_s; S->seed = w.seed; S->periodic = w.periodic ? 1 : 0;
        S->prepared = true;
        return CLV_OK;
    }
    return sfail(ctx, CLV_ERR_SIMULATION, "could not bound the arrival count");
}

}  // namespace

extern "C" {

int clv_set_sim_profile(clv_ctx *ctx, int family, int V, const double *mean_ms, const int32_t *dist,
                        const double *sigma, const double *energy_wh, const double *idle_w5,
                        const double *accuracy, const uint8_t *mem_ok) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    if (family < 0 || family >= CLV_MAX_FAMILIES) return sfail(ctx, CLV_ERR_PROFILE, "family out of range");
    if (V < 1 || V > CLV_MAX_VARIANTS) return sfail(ctx, CLV_ERR_PROFILE, "1..8 variants supported on the device");
    SimState *S = state(ctx);
    SimFamily T{};
    T.V = V; T.E = V * CLV_K;
    for (int e = 0; e < T.E; ++e) {
        if (!(mean_ms[e] > 0) || !std::isfinite(mean_ms[e])) return sfail(ctx, CLV_ERR_PROFILE, "mean_service_ms must be positive");
        if (dist[e] < 0 || dist[e] > 2) return sfail(ctx, CLV_ERR_PROFILE, "unknown service distribution");
        if (dist[e] == 2 && !(sigma[e] > 0)) return sfail(ctx, CLV_ERR_PROFILE, "lognormal rows need sigma > 0");
        if (!(energy_wh[e] >= 0) || !std::isfinite(energy_wh[e])) return sfail(ctx, CLV_ERR_PROFILE, "energy must be >= 0");
        T.mean_ns[e] = mean_ms[e] * 1e6;
        T.det_ns[e] = round_ns(T.mean_ns[e]);
        T.dist[e] = dist[e];
        T.sigma[e] = dist[e] == 2 ? sigma[e] : 0.0;
        T.hs[e] = (0.5 * T.sigma[e]) * T.sigma[e];
        T.energy_wh[e] = energy_wh[e];
        if (dist[e] != 0) T.any_random = 1;
        if (mem_ok[e]) T.mem_ok |= 1ULL << e;
    }
    for (int k = 0; k < CLV_K; ++k) {
        if (!(idle_w5[k] >= 0) || !std::isfinite(idle_w5[k])) return sfail(ctx, CLV_ERR_PROFILE, "idle power must be >= 0");
        T.idle_w[k] = idle_w5[k];
    }
    for (int v = 0; v < V; ++v) {
        if (!(accuracy[v] > 0 && accuracy[v] <= 1.0)) return sfail(ctx, CLV_ERR_PROFILE, "accuracy must be in (0,1]");
        T.acc[v] = accuracy[v];
    }
    SIM_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (!S->fam_dev) SIM_CUDA(cudaMalloc(&S->fam_dev, sizeof(SimFamily) * CLV_MAX_FAMILIES), "alloc sim families");
    SIM_CUDA(cudaMemcpy(S->fam_dev + family, &T, sizeof(SimFamily), cudaMemcpyHostToDevice), "copy sim family");
    S->fam[family] = T;
    S->fam_set[family] = true;
    return CLV_OK;
}

int clv_simulate(clv_ctx *ctx, int family, const clv_workload *w, int64_t count, const uint8_t *inst_edge_dev,
                 const int64_t *inst_off_dev, int max_instances, double l_tail_ms, clv_sim_report *reports_dev,
                 int64_t *variant_counts_dev, int64_t *instance_counts_dev, int64_t *n_requests, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    SimState *S = state(ctx);
    if (family < 0 || family >= CLV_MAX_FAMILIES || !S->fam_set[family])
        return sfail(ctx, CLV_ERR_NOT_READY, "simulator profile family " + std::to_string(family) + " not loaded");
    if (!w) return sfail(ctx, CLV_ERR_SIMULATION, "null workload");
    if (!(w->arrival_rps > 0) || !std::isfinite(w->arrival_rps)) return sfail(ctx, CLV_ERR_SIMULATION, "arrival rate must be positive and finite");
    if (!(w->duration_s > 0) || !std::isfinite(w->duration_s)) return sfail(ctx, CLV_ERR_SIMULATION, "duration must be positive and finite");
    if (w->warmup < -1) return sfail(ctx, CLV_ERR_SIMULATION, "warmup must be >= 0 or -1 (SPEC default)");
    if (std::isnan(l_tail_ms)) return sfail(ctx, CLV_ERR_SIMULATION, "l_tail is NaN");
    if (count < 0) return sfail(ctx, CLV_ERR_SIMULATION, "negative count");
    if (max_instances < 1 || max_instances > 4096) return sfail(ctx, CLV_ERR_SIMULATION, "max_instances must be in 1..4096");
    cudaStream_t st = (cudaStream_t)stream;
    SIM_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    int rc = prepare_workload(ctx, S, *w, st);
    if (rc) return rc;
    const long long N = S->N;
    if (n_requests) *n_requests = N;
    const long long W = w->warmup < 0 ? std::max(100LL, N / 20) : (long long)w->warmup;
    if (N - W < 1) return sfail(ctx, CLV_ERR_SIMULATION, "no request left for the latency statistics after warm-up");
    if (count == 0) return CLV_OK;
    int key_bits = 1;
    while ((1LL << key_bits) < N) ++key_bits;

    const size_t slab = (size_t)max_instances * 21 + 16;
    const size_t slab_al = (slab + 15) & ~(size_t)15;
    const size_t dyn = slab_al * SNW;
    const bool rnd = S->fam[family].any_random != 0;
    auto kern = rnd ? sim_kernel<true> : sim_kernel<false>;
    SIM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn), "sim smem");
    int occ = 0;
    SIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SNT, dyn), "sim occupancy");
    if (occ < 1) return sfail(ctx, CLV_ERR_SIMULATION, "too many instances per fleet for shared memory");
    long long grid = std::min<long long>((count + SNW - 1) / SNW, (long long)occ * ctx->sm_count);
    // completion scratch: grid x SNW rows of N int64, capped by a memory budget
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    size_t budget = std::min<size_t>((size_t)16 << 30, free_b / 2 + S->scr_elems * sizeof(long long));
    const char *env = getenv("CLV_SIM_SCRATCH_MB");
    if (env) budget = (size_t)atoll(env) << 20;
    const size_t row = (size_t)N * sizeof(long long) * SNW;
    grid = std::min<long long>(grid, (long long)(budget / std::max<size_t>(row, 1)));
    if (grid < 1) return sfail(ctx, CLV_ERR_OUT_OF_MEMORY, "simulation scratch does not fit the memory budget");
    const size_t need = (size_t)grid * SNW * (size_t)N;
    if (need > S->scr_elems) {
        cudaFree(S->c_scr);
        S->c_scr = nullptr; S->scr_elems = 0;
        SIM_CUDA(cudaMalloc(&S->c_scr, need * sizeof(long long)), "alloc sim scratch");
        S->scr_elems = need;
    }
    SimArgs a{};
    a.fam = S->fam_dev + family; a.a = S->a; a.ex = S->ex; a.z = S->z;
    a.N = N; a.d_ns = S->d_ns; a.W = W; a.duration_s = w->duration_s;
    a.l_tail = l_tail_ms; a.count = count; a.inst_edge = inst_edge_dev; a.inst_off = inst_off_dev;
    a.kmax = max_instances; a.key_bits = key_bits; a.c_scr = S->c_scr; a.rep = reports_dev;
    a.vcnt = variant_counts_dev; a.icnt = instance_counts_dev;
    kern<<<(unsigned)grid, SNT, dyn, st>>>(a);
    SIM_CUDA(cudaGetLastError(), "sim kernel");
    return CLV_OK;
}

}  // extern "C"
