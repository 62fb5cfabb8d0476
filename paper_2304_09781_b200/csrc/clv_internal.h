// clv_internal.h -- launch wrappers shared between clv_ctx.cu and the kernel files.
#pragma once
#include "clv_common.cuh"

namespace clv {

// Record with the winner's payload, carried through the (one-off) reductions
// of the scoring kernels so no re-decode is needed after selection.
struct RecP {
    Rec r;
    double f, L, A, E;
    int sla;
};
__host__ __device__ inline RecP recp_none() {
    RecP p; p.r = rec_none(); p.f = p.L = p.A = p.E = 0.0; p.sla = 0;
    return p;
}
__device__ inline RecP recp_shfl_xor(const RecP &p, int m) {
    RecP o;
    o.r = rec_shfl_xor(p.r, m);
    o.f = __shfl_xor_sync(0xFFFFFFFFu, p.f, m);
    o.L = __shfl_xor_sync(0xFFFFFFFFu, p.L, m);
    o.A = __shfl_xor_sync(0xFFFFFFFFu, p.A, m);
    o.E = __shfl_xor_sync(0xFFFFFFFFu, p.E, m);
    o.sla = __shfl_xor_sync(0xFFFFFFFFu, p.sla, m);
    return o;
}
__device__ inline RecP warp_min(RecP p) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        RecP o = recp_shfl_xor(p, m);
        if (rec_less(o.r, p.r)) p = o;
    }
    return p;
}
__device__ inline RecP load_cg(const RecP *q) {
    RecP p;
    const unsigned long long *w = reinterpret_cast<const unsigned long long *>(q);
    unsigned long long buf[sizeof(RecP) / 8];
#pragma unroll
    for (int i = 0; i < (int)(sizeof(RecP) / 8); ++i) buf[i] = __ldcg(w + i);
    memcpy(&p, buf, sizeof(RecP));
    return p;
}

// block-level reduction of two records + two counters; result valid in thread 0.
template <int NT>
__device__ inline void block_reduce(RecP &r0, RecP &r1, unsigned long long &c0,
                                    unsigned long long &c1) {
    __shared__ RecP s0[NT / 32], s1[NT / 32];
    __shared__ unsigned long long sc0[NT / 32], sc1[NT / 32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    r0 = warp_min(r0);
    r1 = warp_min(r1);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        c0 += __shfl_xor_sync(0xFFFFFFFFu, c0, m);
        c1 += __shfl_xor_sync(0xFFFFFFFFu, c1, m);
    }
    if (lane == 0) { s0[wid] = r0; s1[wid] = r1; sc0[wid] = c0; sc1[wid] = c1; }
    __syncthreads();
    if (wid == 0) {
        r0 = lane < NT / 32 ? s0[lane] : recp_none();
        r1 = lane < NT / 32 ? s1[lane] : recp_none();
        c0 = lane < NT / 32 ? sc0[lane] : 0ULL;
        c1 = lane < NT / 32 ? sc1[lane] : 0ULL;
        r0 = warp_min(r0);
        r1 = warp_min(r1);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            c0 += __shfl_xor_sync(0xFFFFFFFFu, c0, m);
            c1 += __shfl_xor_sync(0xFFFFFFFFu, c1, m);
        }
    }
    __syncthreads();
}

// Scratch of one grid-wide selection: per-block partials, a done counter and
// the final two records + counters (valid, sla).
struct Sel {
    RecP *partials;               // 2 per block
    unsigned long long *pcnt;     // 2 per block
    unsigned int *done_counter;
    RecP *final_rec;              // 2
    unsigned long long *final_cnt;// 2
};

// Last-block-done finish: every block publishes its partials; the last block
// reduces them into final_rec / final_cnt and resets the counter for reuse.
template <int NT>
__device__ inline void grid_finish(RecP r0, RecP r1, unsigned long long c0, unsigned long long c1,
                                   const Sel &sel) {
    block_reduce<NT>(r0, r1, c0, c1);
    __shared__ bool last;
    if (threadIdx.x == 0) {
        sel.partials[2 * blockIdx.x] = r0;
        sel.partials[2 * blockIdx.x + 1] = r1;
        sel.pcnt[2 * blockIdx.x] = c0;
        sel.pcnt[2 * blockIdx.x + 1] = c1;
        __threadfence();
        unsigned int prev = atomicAdd(sel.done_counter, 1u);
        last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    RecP a = recp_none(), b = recp_none();
    unsigned long long x = 0, y = 0;
    for (unsigned int i = threadIdx.x; i < gridDim.x; i += NT) {
        RecP p0 = load_cg(sel.partials + 2 * i), p1 = load_cg(sel.partials + 2 * i + 1);
        if (rec_less(p0.r, a.r)) a = p0;
        if (rec_less(p1.r, b.r)) b = p1;
        x += __ldcg(sel.pcnt + 2 * i);
        y += __ldcg(sel.pcnt + 2 * i + 1);
    }
    block_reduce<NT>(a, b, x, y);
    if (threadIdx.x == 0) {
        sel.final_rec[0] = a;
        sel.final_rec[1] = b;
        sel.final_cnt[0] = x;
        sel.final_cnt[1] = y;
        *sel.done_counter = 0u;
    }
}

constexpr int PROF_SLOTS = 20;          // debug phase-profile slots per CTA (CLV_ANNEAL_VARIANT=9)

struct AnnealArgs {
    const FamilyTables *fam;
    FeasView F;
    const EvalConst *ec;
    int n_ec;
    EvalConst ec0;                  // = ec[0] when n_ec == 1 (kernel-parameter copy)
    int fast_div;                   // every scenario and the family's lat95 satisfy fast_div_safe()
    double t_init, cooling, t_floor;
    double cool_factor;             // 1 - cooling (multiplicative cooling)
    int stall_limit, max_steps, proposal, evaluate;
    int flags;                      // CLV_ANNEAL_MULT_COOLING | CLV_ANNEAL_PAPER_MOVES
    int n, n_chains, E;
    long long chain_base;
    uint64_t seed;
    const uint16_t *start_w;
    clv_chain_result *res;
    uint16_t *best_w;
    uint16_t *final_w;
    clv_log_row *log;
    int *mvlog;                     // [n_chains][max_steps] accepted move per step (-1 = none)
    int *chain_counter;             // persistent launches: next chain to take (zeroed per launch); else null
    long long *prof;                // optional phase profile (debug variant only)
};

// score_x row error codes (low byte of ScoreArgs::error_key): the clv_status values, plus
// CarbonSchedError's "variant ordinals start at 1" (mig.py:262) kept apart for its message.
constexpr int SCORE_X_VARIANT_LT1 = 0x11;

struct ScoreArgs {
    const FamilyTables *fam;
    FeasView F;
    EvalConst ec;
    int select_mode;
    long long count, index_base;
    const uint16_t *w;              // score_graphs input
    const uint8_t *xp, *xv;         // score_x input
    const int64_t *xv_off;
    const Topology *topo;
    double *f_out, *h_out, *p95_out;
    uint8_t *sla_out, *feas_out;
    Sel sel;
    unsigned long long *error_key;  // min over failing rows of (index << 8 | error code); ~0 = none
    int fast;                       // ec and the family's lat95 satisfy fast_div_safe()
};

struct OracleArgs {
    const FamilyTables *fam;
    const Topology *topo;
    EvalConst ec;
    long long begin, end;
    int n;
    long long row_off[CLV_MAX_CONFIGS + 1];
    int row_place[CLV_MAX_CONFIGS][8];   // mixed-radix place values per slice
    Sel sel;
    int fast;                            // fast_div_safe(ec, family lat95)
};

struct SweepPod {
    int family, n_gpus;
    double weight;
    EvalConst ec;
};

struct SweepArgs {
    const FamilyTables *fam;         // array [CLV_MAX_FAMILIES]
    const Topology *topo;
    int n_pods;
    SweepPod pods[CLV_MAX_PODS];
    long long begin, end;
    uint64_t seed;
    double *f_out, *h_out;
    uint8_t *sla_out;
    Sel sel;
    int fast;                        // every pod satisfies fast_div_safe()
};

cudaError_t launch_feas_level(uint32_t *bits, const uint32_t *off, int N, int bdim, int cdim,
                              const int2 *bc_list, int n_bc, const int *rows4, int nrows4,
                              cudaStream_t s);
cudaError_t launch_feasible(FeasView F, int n, const int32_t *vec5, long long count, uint8_t *out,
                            cudaStream_t s);
cudaError_t launch_realize(FeasView F, const Topology *topo_dev, int n, const int32_t *vec5_dev,
                           int32_t *parts_dev, cudaStream_t s);
cudaError_t launch_score_graphs(const ScoreArgs &a, const FamilyTables &T, int grid, cudaStream_t s);
cudaError_t launch_score_x(const ScoreArgs &a, int n, int grid, cudaStream_t s);
cudaError_t launch_oracle(const OracleArgs &a, int grid, cudaStream_t s);
cudaError_t launch_anneal(const AnnealArgs &a, int cluster, cudaStream_t s);
cudaError_t launch_sweep(const SweepArgs &a, int grid, cudaStream_t s);
cudaError_t launch_select_chains(const clv_chain_result *res, int n_chains, long long chain_base,
                                 clv_record *out, cudaStream_t s);
cudaError_t launch_reduce_records(const clv_record *recs, int count, clv_record *out,
                                  cudaStream_t s);

}  // namespace clv
