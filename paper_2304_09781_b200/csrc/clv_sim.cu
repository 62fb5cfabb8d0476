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
//     Instance keys (free << 11 | j) live in the warp's shared-memory slab, lane g
//     caches the minimum of instance group g = {g, g+32, ...}; each request is a
//     2-step redux.sync argmin over the group minima, a warp-uniform service draw,
//     and a 2-step redux.sync refresh of the served instance's group.
//     Completions go to a per-warp HBM scratch row c[N] (coalesced 32-request
//     stores).  Then the whole CTA post-processes its
//     simulations one at a time: 11-bit radix selections for the warm-up cut (key
//     = completion << b | request) and the nearest-rank p95 over the remaining
//     latencies, exact integer sums for mean latency / busy / idle time, and the
//     fixed-order fp64 energy and accuracy epilogue.
#include <algorithm>
#include <climits>
#include <cmath>
#include <type_traits>
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
    int cls[CLV_MAX_EDGES];                  // service class of the edge
    int n_cls;
    int cls_kind[8];                         // 0 deterministic, 1 exponential, 2 lognormal
    double cls_sigma[8], cls_hs[8];
};
constexpr int SIM_MAX_CLS = 8;

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
    unsigned short *j_scr = nullptr;
    size_t scr_elems = 0;
    double *mult = nullptr;                  // [n_cls][N] service multipliers
    size_t mult_elems = 0;
};

void sim_destroy(SimState *s) {
    if (!s) return;
    cudaFree(s->fam_dev);
    cudaFree(s->a); cudaFree(s->ex); cudaFree(s->z); cudaFree(s->n_dev);
    cudaFreeHost(s->n_host);
    cudaFree(s->c_scr); cudaFree(s->j_scr); cudaFree(s->mult);
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
    const double *mult;
    long long *c_scr;
    unsigned short *j_scr;
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

// Per-request service multipliers of the family's service classes (class 0:
// deterministic = 1, 1: exponential = ex_i, k >= 2: lognormal exp(sigma_k z_i - hs_k)).
__global__ void sim_mult_kernel(const SimFamily *fam, const double *ex, const double *z, long long N, double *mult) {
    const SimFamily &F = *fam;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        for (int k = 0; k < F.n_cls; ++k) {
            double m = 1.0;
            if (F.cls_kind[k] == 1) m = ex[i];
            else if (F.cls_kind[k] == 2) m = exp_clv(F.cls_sigma[k] * z[i] - F.cls_hs[k]);
            mult[(size_t)k * N + i] = m;
        }
    }
}

// Per-warp shared-memory slab of one simulation (kmax instances).
struct Slab {
    unsigned long long *key;   // (free << 11) | j during the run; busy time (ns) in the post-pass
    long long *svc;            // deterministic service ns (RAND=false) / mean ns as double bits (RAND=true)
    unsigned *cnt;
    unsigned char *ed, *cls;
    double *mst;               // [SIM_MAX_CLS][32] multipliers of the current 32-request block
};
__device__ __forceinline__ Slab slab_of(unsigned char *base, int kmax) {
    Slab q;
    q.mst = reinterpret_cast<double *>(base);
    q.key = reinterpret_cast<unsigned long long *>(base + SIM_MAX_CLS * 32 * 8);
    q.svc = reinterpret_cast<long long *>(q.key + kmax);
    q.cnt = reinterpret_cast<unsigned *>(q.svc + kmax);
    q.ed = reinterpret_cast<unsigned char *>(q.cnt + kmax);
    q.cls = q.ed + kmax;
    return q;
}
__host__ __device__ inline size_t slab_bytes(int kmax) {
    return ((size_t)SIM_MAX_CLS * 32 * 8 + (size_t)kmax * 22 + 15) & ~(size_t)15;
}

// Queue recursion with the instance keys in registers (K <= 32 * S): lane l owns
// instances l + 32 t (t < S) and their minimum; each request is a 2-step redux.sync
// argmin over the lane minima, a warp-uniform service lookup, and -- in the owner lane
// only -- a register update plus an S-wide min tree (no shared-memory round trip and no
// second reduction on the dependency chain).
template <bool RAND, int S>
__device__ __forceinline__ void run_sim_regs(const Slab &q, const SimArgs &args, int K, long long N, int C,
                                             long long *cs, unsigned short *js, int lane) {
    unsigned long long k[S];
#pragma unroll
    for (int t = 0; t < S; ++t) {
        const int j = lane + 32 * t;
        k[t] = j < K ? (unsigned long long)j : ~0ULL;
    }
    unsigned long long lm = k[0];                  // keys start at j: slot 0 is the lane's minimum
    for (long long b = 0; b < N; b += 32) {
        const long long i = b + lane;
        const long long al = i < N ? __ldg(args.a + i) : 0LL;
        if (RAND) {
            __syncwarp();
            for (int c2 = 0; c2 < C; ++c2)
                q.mst[c2 * 32 + lane] = i < N ? __ldg(args.mult + (size_t)c2 * N + i) : 1.0;
            __syncwarp();
        }
        const int nb = (int)min(32LL, N - b);
        long long myc = 0;
        unsigned myj = 0;
#pragma unroll 4
        for (int r = 0; r < nb; ++r) {
            const long long ai = __shfl_sync(0xFFFFFFFFu, al, r);
            const unsigned hi = (unsigned)(lm >> 32);
            const unsigned mh = __reduce_min_sync(0xFFFFFFFFu, hi);
            const unsigned ml = __reduce_min_sync(0xFFFFFFFFu, hi == mh ? (unsigned)lm : 0xFFFFFFFFu);
            const int j = (int)(ml & 2047u);
            const long long fv = (long long)((((unsigned long long)mh << 32) | ml) >> 11);
            long long sv;
            if (RAND) sv = round_ns(__longlong_as_double(q.svc[j]) * q.mst[q.cls[j] * 32 + r]);
            else sv = q.svc[j];
            const long long c = (ai > fv ? ai : fv) + sv;
            if (lane == (j & 31)) {
                const unsigned long long np = ((unsigned long long)c << 11) | (unsigned)j;
                const int ts = j >> 5;
                unsigned long long tm[S];
#pragma unroll
                for (int t = 0; t < S; ++t) {
                    if (t == ts) k[t] = np;
                    tm[t] = k[t];
                }
#pragma unroll
                for (int w = S / 2; w >= 1; w /= 2)
#pragma unroll
                    for (int t = 0; t < w; ++t) tm[t] = tm[t] < tm[t + w] ? tm[t] : tm[t + w];
                lm = tm[0];
            }
            if (lane == r) { myc = c; myj = (unsigned)j; }
        }
        if (i < N) { cs[i] = myc; js[i] = (unsigned short)myj; }
    }
}

template <bool RAND, int S>
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
    const size_t sb = slab_bytes(kmax);
    const long long N = args.N;
    __syncthreads();
    const int C = F.n_cls;

    for (long long base = (long long)blockIdx.x * SNW; base < args.count; base += (long long)gridDim.x * SNW) {
        const long long sim = base + warp;
        const Slab q = slab_of(smem_raw + sb * warp, kmax);
        const size_t row = ((size_t)blockIdx.x * SNW + warp) * (size_t)N;
        long long *cs = args.c_scr + row;
        unsigned short *js = args.j_scr + row;
        int status = 0, K = 0;
        if (sim < args.count) {
            const long long o0 = args.inst_off[sim], o1 = args.inst_off[sim + 1];
            K = (int)(o1 - o0);
            if (o1 - o0 < 1 || o1 - o0 > kmax) {
                status = CLV_ERR_SIMULATION;
            } else {
                int bad = 0;
                for (int t = lane; t < K; t += 32) {
                    int e = args.inst_edge[o0 + t];
                    if (e >= F.E) { bad |= 2; e = 0; }
                    else if (!((F.mem_ok >> e) & 1ULL)) bad |= 1;
                    q.ed[t] = (unsigned char)e;
                    q.cls[t] = (unsigned char)F.cls[e];
                    q.svc[t] = RAND ? __double_as_longlong(F.mean_ns[e]) : F.det_ns[e];
                    q.key[t] = (unsigned long long)t;
                    q.cnt[t] = 0u;
                }
                bad = __reduce_or_sync(0xFFFFFFFFu, bad);
                if (bad & 2) status = CLV_ERR_SIMULATION;
                else if (bad & 1) status = CLV_ERR_INFEASIBLE_ASSIGNMENT;
            }
            __syncwarp();
            if (status == 0 && S > 0) {
                run_sim_regs<RAND, (S > 0 ? S : 1)>(q, args, K, N, C, cs, js, lane);
            } else if (status == 0) {
                // Slot j holds the packed key (free_j << 11) | j (unique, order-preserving: the
                // argmin key is argmin (free, j)); lane g caches the minimum of instance group
                // g = {g, g+32, ...}; slot j is read and written only by lane j >> 5.
                unsigned long long gm = lane < K ? (unsigned long long)lane : ~0ULL;
                for (long long b = 0; b < N; b += 32) {
                    const long long i = b + lane;
                    const long long al = i < N ? __ldg(args.a + i) : 0LL;
                    if (RAND) {
                        __syncwarp();
                        for (int k = 0; k < C; ++k)
                            q.mst[k * 32 + lane] = i < N ? __ldg(args.mult + (size_t)k * N + i) : 1.0;
                        __syncwarp();
                    }
                    const int nb = (int)min(32LL, N - b);
                    long long myc = 0;
                    unsigned myj = 0;
#pragma unroll 4
                    for (int r = 0; r < nb; ++r) {
                        const long long ai = __shfl_sync(0xFFFFFFFFu, al, r);
                        const unsigned hi = (unsigned)(gm >> 32);
                        const unsigned mh = __reduce_min_sync(0xFFFFFFFFu, hi);
                        const unsigned ml = __reduce_min_sync(0xFFFFFFFFu, hi == mh ? (unsigned)gm : 0xFFFFFFFFu);
                        const unsigned long long P = ((unsigned long long)mh << 32) | ml;
                        const int j = (int)(ml & 2047u);
                        const long long fv = (long long)(P >> 11);
                        // the rest of j's group (independent of the service draw)
                        const int g = j & 31;
                        const int slot = g + 32 * lane;
                        const unsigned long long vo = (slot < K && slot != j) ? q.key[slot] : ~0ULL;
                        long long sv;
                        if (RAND) sv = round_ns(__longlong_as_double(q.svc[j]) * q.mst[q.cls[j] * 32 + r]);
                        else sv = q.svc[j];
                        const long long c = (ai > fv ? ai : fv) + sv;
                        const unsigned long long np = ((unsigned long long)c << 11) | (unsigned)j;
                        const unsigned h2 = (unsigned)(vo >> 32);
                        const unsigned m2 = __reduce_min_sync(0xFFFFFFFFu, h2);
                        const unsigned l2 = __reduce_min_sync(0xFFFFFFFFu, h2 == m2 ? (unsigned)vo : 0xFFFFFFFFu);
                        const unsigned long long mo = ((unsigned long long)m2 << 32) | l2;
                        if (lane == g) gm = mo < np ? mo : np;
                        if (lane == (j >> 5)) q.key[j] = np;
                        if (lane == r) { myc = c; myj = (unsigned)j; }
                    }
                    if (i < N) { cs[i] = myc; js[i] = (unsigned short)myj; }
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
            const size_t roww = ((size_t)blockIdx.x * SNW + w) * (size_t)N;
            const long long *cw = args.c_scr + roww;
            const unsigned short *jw = args.j_scr + roww;
            const Slab qw = slab_of(smem_raw + sb * w, kmax);
            clv_sim_report rp;
            memset(&rp, 0, sizeof(rp));
            if (st == 0) {
                for (int t = tid; t < Kw; t += SNT) qw.key[t] = 0ULL;     // busy time
                __syncthreads();
                long long mx = 0;
                for (long long i = tid; i < N; i += SNT) {
                    const long long c = cw[i];
                    const int j = jw[i];
                    long long sv;
                    if (RAND) sv = round_ns(__longlong_as_double(qw.svc[j]) * __ldg(args.mult + (size_t)qw.cls[j] * N + i));
                    else sv = qw.svc[j];
                    atomicAdd(&qw.cnt[j], 1u);
                    atomicAdd(&qw.key[j], (unsigned long long)sv);
                    mx = max(mx, c);
                }
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
                    for (int e = tid; e < CLV_MAX_EDGES; e += SNT) cnt_e[e] = 0ULL;
                    if (tid < CLV_K) idle_s[tid] = 0ULL;
                    __syncthreads();
                    for (int t = tid; t < Kw; t += SNT) {
                        const int e = qw.ed[t];
                        atomicAdd(&cnt_e[e], (unsigned long long)qw.cnt[t]);
                        atomicAdd(&idle_s[e % CLV_K], (unsigned long long)(t_end - (long long)qw.key[t]));
                        if (args.icnt) args.icnt[args.inst_off[sw] + t] = (int64_t)qw.cnt[t];
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
    // service classes: 0 deterministic, 1 exponential, then one per distinct lognormal sigma
    T.n_cls = 2;
    T.cls_kind[0] = 0; T.cls_kind[1] = 1;
    for (int e = 0; e < T.E; ++e) {
        if (T.dist[e] < 2) { T.cls[e] = T.dist[e]; continue; }
        int k = 2;
        while (k < T.n_cls && T.cls_sigma[k] != T.sigma[e]) ++k;
        if (k == T.n_cls) {
            if (k >= SIM_MAX_CLS) return sfail(ctx, CLV_ERR_PROFILE, "at most 6 distinct lognormal sigmas per profile");
            T.cls_kind[k] = 2; T.cls_sigma[k] = T.sigma[e]; T.cls_hs[k] = T.hs[e];
            T.n_cls++;
        }
        T.cls[e] = k;
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
    if (max_instances < 1 || max_instances > 2048) return sfail(ctx, CLV_ERR_SIMULATION, "max_instances must be in 1..2048");
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

    const size_t dyn = slab_bytes(max_instances) * SNW;
    const bool rnd = S->fam[family].any_random != 0;
    if (rnd) {
        const size_t m = (size_t)S->fam[family].n_cls * (size_t)N;
        if (m > S->mult_elems) {
            cudaFree(S->mult);
            S->mult = nullptr; S->mult_elems = 0;
            SIM_CUDA(cudaMalloc(&S->mult, m * sizeof(double)), "alloc multipliers");
            S->mult_elems = m;
        }
        const int g = (int)std::min<long long>((N + 255) / 256, (long long)ctx->sm_count * 8);
        sim_mult_kernel<<<std::max(g, 1), 256, 0, st>>>(S->fam_dev + family, S->ex, S->z, N, S->mult);
        SIM_CUDA(cudaGetLastError(), "sim multipliers");
    }
    // register-resident keys when every fleet has <= 512 instances (S slots per lane)
    // register-resident keys for small fleets; CLV_SIM_SLOTS caps the slots per lane
    // (0 = always the shared-memory group layout)
    int cap = 2;                                   // measured: registers win up to 2 slots (tools/des_slots.py)
    if (const char *ev = getenv("CLV_SIM_SLOTS")) cap = atoi(ev);
    int slots = max_instances <= 32 ? 1 : max_instances <= 64 ? 2 : max_instances <= 128 ? 4
              : max_instances <= 256 ? 8 : max_instances <= 512 ? 16 : 0;
    if (slots > cap) slots = 0;
    auto pick = [&](auto r) {
        constexpr bool R = decltype(r)::value;
        switch (slots) {
            case 1: return sim_kernel<R, 1>;
            case 2: return sim_kernel<R, 2>;
            case 4: return sim_kernel<R, 4>;
            case 8: return sim_kernel<R, 8>;
            case 16: return sim_kernel<R, 16>;
            default: return sim_kernel<R, 0>;
        }
    };
    auto kern = rnd ? pick(std::true_type{}) : pick(std::false_type{});
    SIM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn), "sim smem");
    int occ = 0;
    SIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, SNT, dyn), "sim occupancy");
    if (occ < 1) return sfail(ctx, CLV_ERR_SIMULATION, "too many instances per fleet for shared memory");
    long long grid = std::min<long long>((count + SNW - 1) / SNW, (long long)occ * ctx->sm_count);
    // per-request scratch (completion int64 + instance uint16): grid x SNW rows of N, capped by a budget
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t per = sizeof(long long) + sizeof(unsigned short);
    size_t budget = std::min<size_t>((size_t)16 << 30, free_b / 2 + S->scr_elems * per);
    const char *env = getenv("CLV_SIM_SCRATCH_MB");
    if (env) budget = (size_t)atoll(env) << 20;
    const size_t row = (size_t)N * per * SNW;
    grid = std::min<long long>(grid, (long long)(budget / std::max<size_t>(row, 1)));
    if (grid < 1) return sfail(ctx, CLV_ERR_OUT_OF_MEMORY, "simulation scratch does not fit the memory budget");
    const size_t need = (size_t)grid * SNW * (size_t)N;
    if (need > S->scr_elems) {
        cudaFree(S->c_scr); cudaFree(S->j_scr);
        S->c_scr = nullptr; S->j_scr = nullptr; S->scr_elems = 0;
        SIM_CUDA(cudaMalloc(&S->c_scr, need * sizeof(long long)), "alloc sim scratch");
        SIM_CUDA(cudaMalloc(&S->j_scr, need * sizeof(unsigned short)), "alloc sim scratch");
        S->scr_elems = need;
    }
    SimArgs a{};
    a.fam = S->fam_dev + family; a.a = S->a; a.ex = S->ex; a.z = S->z;
    a.N = N; a.d_ns = S->d_ns; a.W = W; a.duration_s = w->duration_s;
    a.l_tail = l_tail_ms; a.count = count; a.inst_edge = inst_edge_dev; a.inst_off = inst_off_dev;
    a.kmax = max_instances; a.key_bits = key_bits; a.c_scr = S->c_scr; a.j_scr = S->j_scr; a.mult = S->mult;
    a.rep = reports_dev;
    a.vcnt = variant_counts_dev; a.icnt = instance_counts_dev;
    kern<<<(unsigned)grid, SNT, dyn, st>>>(a);
    SIM_CUDA(cudaGetLastError(), "sim kernel");
    return CLV_OK;
}

}  // extern "C"
