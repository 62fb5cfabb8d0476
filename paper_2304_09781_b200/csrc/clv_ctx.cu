// clv_ctx.cu -- the C-ABI (include/clover.h): context, table staging, argument
// validation, launch orchestration and status-code mapping.
#include <nvtx3/nvToolsExt.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include "clv_ctx.h"

using namespace clv;


namespace {

int fail(clv_ctx *c, int code, const std::string &msg) {
    if (c) c->err = msg;
    return code;
}

int cuda_fail(clv_ctx *c, cudaError_t e, const char *where) {
    int code = (e == cudaErrorMemoryAllocation) ? CLV_ERR_OUT_OF_MEMORY : CLV_ERR_CUDA;
    return fail(c, code, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CLV_CUDA(call, where)                         \
    do {                                              \
        cudaError_t _e = (call);                      \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, where); \
    } while (0)

bool is_finite(double x) { return std::isfinite(x); }

int make_ec(clv_ctx *ctx, const clv_eval_params *p, const FamilyTables &T, EvalConst &ec) {
    if (!p) return fail(ctx, CLV_ERR_CARBON_SCHED, "null eval params");
    if (!(p->arrival_rps > 0) || !is_finite(p->arrival_rps))
        return fail(ctx, CLV_ERR_SIMULATION, "arrival rate must be positive and finite");
    if (!(p->ci >= 0) || !is_finite(p->ci)) return fail(ctx, CLV_ERR_CARBON_SCHED, "ci must be finite and >= 0");
    if (!(p->base_accuracy > 0 && p->base_accuracy <= 1.0))
        return fail(ctx, CLV_ERR_CARBON_SCHED, "base_accuracy must be in (0,1]");
    if (!(p->base_carbon_g > 0) || !is_finite(p->base_carbon_g))
        return fail(ctx, CLV_ERR_CARBON_SCHED, "base_carbon_g must be positive");
    if (!(p->latency_slo_ms > 0) || !is_finite(p->latency_slo_ms))
        return fail(ctx, CLV_ERR_CARBON_SCHED, "latency_slo_ms must be positive");
    if (!(p->rho_sat > 0 && p->rho_sat < 1.0)) return fail(ctx, CLV_ERR_CARBON_SCHED, "rho_sat must be in (0,1)");
    if (!is_finite(p->carbon_weight)) return fail(ctx, CLV_ERR_CARBON_SCHED, "carbon_weight must be finite");
    if (p->n_gpus < 1) return fail(ctx, CLV_ERR_CARBON_SCHED, "n_gpus must be >= 1");
    double R = p->arrival_rps;
    ec.R_q = std::ldexp(R, T.kt);
    ec.inv_3600R = 1.0 / (3600.0 * R);
    ec.R = R;
    ec.iR = 1.0 / R;
    ec.c20 = 20000.0 / R;
    ec.sc1 = std::ldexp(1.0, -T.kt);
    ec.sc2 = std::ldexp(1.0, -T.k2);
    ec.sc3 = std::ldexp(1.0, -T.k3);
    ec.en_scale = std::ldexp(1.0, T.kt - T.ke);
    ec.idle_scale = std::ldexp(1.0, -T.ki);
    ec.rho_sat = p->rho_sat;
    ec.a_base = p->base_accuracy;
    ec.c_base = p->base_carbon_g;
    ec.slo = p->latency_slo_ms;
    ec.ci = p->ci;
    ec.lam = std::min(1.0, std::max(0.0, p->carbon_weight));
    ec.kA = 100.0 / p->base_accuracy;
    ec.kC = p->ci / (10.0 * p->base_carbon_g);
    ec.strict = p->strict_eq6 ? 1 : 0;
    if (!(p->max_accuracy_loss_pct >= 0)) return fail(ctx, CLV_ERR_CARBON_SCHED, "max_accuracy_loss_pct must be >= 0");
    ec.min_dA = -p->max_accuracy_loss_pct;
    ec.n = p->n_gpus;
    return CLV_OK;
}

int need_family(clv_ctx *ctx, int family) {
    if (family < 0 || family >= CLV_MAX_FAMILIES || !ctx->fam_set[family])
        return fail(ctx, CLV_ERR_NOT_READY, "profile family " + std::to_string(family) + " not loaded");
    if (!ctx->topo_set) return fail(ctx, CLV_ERR_NOT_READY, "topology not loaded");
    return CLV_OK;
}

FeasView feas_view(const clv_ctx *ctx) {
    FeasView F;
    F.bits = ctx->feas_bits; F.off = ctx->feas_off; F.nmax = ctx->feas_nmax;
    F.bdim = ctx->bdim; F.cdim = ctx->cdim; F.has7g = ctx->topo.has7g;
    return F;
}

Sel make_sel(clv_ctx *ctx) {
    Sel s;
    s.partials = ctx->partials; s.pcnt = ctx->pcnt; s.done_counter = ctx->done_counter;
    s.final_rec = ctx->final_rec; s.final_cnt = ctx->final_cnt;
    return s;
}

int grid_for(clv_ctx *ctx, long long work, int per_block) {
    long long g = (work + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > ctx->max_blocks) g = ctx->max_blocks;
    return (int)g;
}

// Copy the final selection back and fill a clv_best (synchronises the stream).
int fetch_best(clv_ctx *ctx, int mode, cudaStream_t st, clv_best *best) {
    CLV_CUDA(cudaMemcpyAsync(ctx->host_rec, ctx->final_rec, 2 * sizeof(RecP), cudaMemcpyDeviceToHost, st), "copy best");
    CLV_CUDA(cudaMemcpyAsync(ctx->host_cnt, ctx->final_cnt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st), "copy counts");
    CLV_CUDA(cudaStreamSynchronize(st), "synchronize");
    if (!best) return CLV_OK;
    const RecP &a = ctx->host_rec[0], &b = ctx->host_rec[1];
    const RecP *w = nullptr;
    if (mode == CLV_SELECT_BEST_H) w = (a.r.k1 != 0xFFFFFFFFu) ? &a : nullptr;
    else w = (a.r.k1 != 0xFFFFFFFFu) ? &a : ((b.r.k1 != 0xFFFFFFFFu) ? &b : nullptr);
    std::memset(best, 0, sizeof(*best));
    best->valid_count = (int64_t)ctx->host_cnt[0];
    best->sla_count = (int64_t)ctx->host_cnt[1];
    if (!w) { best->index = -1; best->found = 0; return CLV_OK; }
    best->index = w->r.idx;
    best->f = w->f; best->h = w->r.hv; best->p95_ms = w->L; best->accuracy = w->A; best->energy_wh = w->E;
    best->sla_met = w->sla;
    best->found = 1;
    return CLV_OK;
}

}  // namespace

static long long *prof_buf = nullptr;   // debug phase profile (CLV_ANNEAL_VARIANT=9)
static size_t prof_cap = 0;

extern "C" {

int clv_abi_version(void) { return CLV_ABI_VERSION; }

uint64_t clv_derive_seed(const uint64_t *parts, int n_parts) {
    uint64_t h = 0x9E3779B97F4A7C15ULL;
    for (int i = 0; i < n_parts; ++i) h = seed_round(h, parts[i]);
    return h & 0x7FFFFFFFFFFFFFFFULL;
}

const char *clv_last_error(const clv_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int clv_create(int device, clv_ctx **out) {
    if (!out) return CLV_ERR_CARBON_SCHED;
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) return CLV_ERR_CUDA;
    if (device < 0 || device >= ndev) return CLV_ERR_CUDA;
    clv_ctx *ctx = new clv_ctx();
    ctx->device = device;
    CLV_CUDA(cudaSetDevice(device), "cudaSetDevice");
    CLV_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device), "sm count");
    ctx->max_blocks = ctx->sm_count * 16;
    CLV_CUDA(cudaMalloc(&ctx->topo_dev, sizeof(Topology)), "alloc topology");
    CLV_CUDA(cudaMalloc(&ctx->fam_dev, sizeof(FamilyTables) * CLV_MAX_FAMILIES), "alloc families");
    CLV_CUDA(cudaMalloc(&ctx->partials, sizeof(RecP) * 2 * ctx->max_blocks), "alloc partials");
    CLV_CUDA(cudaMalloc(&ctx->pcnt, sizeof(unsigned long long) * 2 * ctx->max_blocks), "alloc pcnt");
    CLV_CUDA(cudaMalloc(&ctx->done_counter, sizeof(unsigned int)), "alloc counter");
    CLV_CUDA(cudaMemset(ctx->done_counter, 0, sizeof(unsigned int)), "zero counter");
    CLV_CUDA(cudaMalloc(&ctx->final_rec, sizeof(RecP) * 2), "alloc final");
    CLV_CUDA(cudaMalloc(&ctx->final_cnt, sizeof(unsigned long long) * 2), "alloc final cnt");
    CLV_CUDA(cudaMallocHost(&ctx->host_rec, sizeof(RecP) * 2), "pinned rec");
    CLV_CUDA(cudaMallocHost(&ctx->host_cnt, sizeof(unsigned long long) * 2), "pinned cnt");
    CLV_CUDA(cudaMalloc(&ctx->err_flag, sizeof(int)), "alloc err");
    CLV_CUDA(cudaMalloc(&ctx->err_index, sizeof(long long)), "alloc err idx");
    CLV_CUDA(cudaMallocHost(&ctx->host_err, 16), "pinned err");
    CLV_CUDA(cudaMalloc(&ctx->small_dev, sizeof(int32_t) * 1024), "alloc small");
    *out = ctx;
    return CLV_OK;
}

void clv_destroy(clv_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaFree(ctx->topo_dev); cudaFree(ctx->fam_dev);
    cudaFree(ctx->feas_bits); cudaFree(ctx->feas_off);
    cudaFree(ctx->partials); cudaFree(ctx->pcnt); cudaFree(ctx->done_counter);
    cudaFree(ctx->final_rec); cudaFree(ctx->final_cnt);
    cudaFreeHost(ctx->host_rec); cudaFreeHost(ctx->host_cnt);
    cudaFree(ctx->err_flag); cudaFree(ctx->err_index); cudaFreeHost(ctx->host_err);
    cudaFree(ctx->ec_dev); cudaFree(ctx->small_dev);
    for (int f = 0; f < CLV_MAX_FAMILIES; ++f) cudaFree(ctx->pair_list_dev[f]);
    clv::sim_destroy(ctx->sim);
    cudaFree(ctx->mvlog); cudaFree(ctx->replan_buf); cudaFree(ctx->chain_counter);
    delete ctx;
}

int clv_set_topology(clv_ctx *ctx, int K, const int32_t *ids, const int32_t *counts5,
                     const double *mem_gb5) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    if (K < 1 || K > CLV_MAX_CONFIGS) return fail(ctx, CLV_ERR_INVALID_CONFIG, "topology needs 1..32 configurations");
    Topology t{};
    t.K = K;
    const int cu[CLV_K] = {7, 4, 3, 2, 1};
    std::vector<std::pair<int, int>> order;
    for (int r = 0; r < K; ++r) order.push_back({ids[r], r});
    std::sort(order.begin(), order.end());
    for (int q = 0; q < K; ++q) {
        int r = order[q].second;
        if (q > 0 && order[q].first == order[q - 1].first) return fail(ctx, CLV_ERR_INVALID_CONFIG, "duplicate config id");
        if (ids[r] < 0 || ids[r] > 255) return fail(ctx, CLV_ERR_INVALID_CONFIG, "config ids must be in 0..255");
        int ns = 0, units = 0;
        for (int k = 0; k < CLV_K; ++k) {
            int x = counts5[5 * r + k];
            if (x < 0) return fail(ctx, CLV_ERR_INVALID_CONFIG, "negative slice count");
            t.counts[q][k] = x;
            for (int j = 0; j < x && ns < 8; ++j) t.kinds[q][ns++] = (unsigned char)k;
            units += x * cu[k];
        }
        int total = 0;
        for (int k = 0; k < CLV_K; ++k) total += t.counts[q][k];
        if (total < 1) return fail(ctx, CLV_ERR_INVALID_CONFIG, "configuration is empty");
        if (total > 7) return fail(ctx, CLV_ERR_INVALID_CONFIG, "configuration has more than 7 slices");
        if (units > 7) return fail(ctx, CLV_ERR_INVALID_CONFIG, "configuration exceeds the per-GPU compute budget");
        if (t.counts[q][0] > 0) t.has7g = 1;   // CU<=7 => a 7g row is exactly {7g}
        t.ids[q] = ids[r];
        t.nslices[q] = total;
        if (t.counts[q][0] == 0) {
            bool dup = false;
            for (int j = 0; j < t.nrows4; ++j)
                dup |= (t.rows4[j][0] == t.counts[q][1] && t.rows4[j][1] == t.counts[q][2] &&
                        t.rows4[j][2] == t.counts[q][3] && t.rows4[j][3] == t.counts[q][4]);
            if (!dup) {
                for (int k = 0; k < 4; ++k) t.rows4[t.nrows4][k] = t.counts[q][k + 1];
                t.nrows4++;
            }
        }
    }
    for (int k = 0; k < CLV_K; ++k) {
        if (!(mem_gb5[k] > 0)) return fail(ctx, CLV_ERR_INVALID_CONFIG, "slice memory must be positive");
        ctx->mem_gb[k] = mem_gb5[k];
    }
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    CLV_CUDA(cudaMemcpy(ctx->topo_dev, &t, sizeof(Topology), cudaMemcpyHostToDevice), "copy topology");
    ctx->topo = t;
    ctx->topo_set = true;
    // a new table invalidates the feasibility bitsets
    cudaFree(ctx->feas_bits); cudaFree(ctx->feas_off);
    ctx->feas_bits = nullptr; ctx->feas_off = nullptr; ctx->feas_nmax = -1;
    return CLV_OK;
}

int clv_set_profile(clv_ctx *ctx, int family, int V, const int64_t *thr_q, const int64_t *acc_q,
                    const int64_t *en_q, const int64_t *idle_q5, const double *lat95,
                    const double *svc_ms, const uint8_t *mem_ok, int kt, int ke, int ki) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    if (family < 0 || family >= CLV_MAX_FAMILIES) return fail(ctx, CLV_ERR_PROFILE, "family out of range");
    if (V < 1 || V > CLV_MAX_VARIANTS) return fail(ctx, CLV_ERR_PROFILE, "1..8 variants supported on the device");
    FamilyTables T{};
    T.V = V; T.E = V * CLV_K; T.kt = kt; T.ke = ke; T.ki = ki;
    const long long LIM = 1LL << 31;
    for (int e = 0; e < T.E; ++e) {
        if (thr_q[e] <= 0 || thr_q[e] >= LIM || acc_q[e] < 0 || acc_q[e] >= LIM || en_q[e] < 0 || en_q[e] >= LIM)
            return fail(ctx, CLV_ERR_PROFILE, "fixed-point rows must be in [0, 2^31) (throughput > 0)");
        if (!(lat95[e] > 0) || !is_finite(lat95[e])) return fail(ctx, CLV_ERR_PROFILE, "p95 service time must be positive");
        if (!(svc_ms[e] > 0) || !is_finite(svc_ms[e])) return fail(ctx, CLV_ERR_PROFILE, "mean service time must be positive");
        T.thr_q[e] = thr_q[e]; T.acc_q[e] = acc_q[e]; T.en_q[e] = en_q[e]; T.lat95[e] = lat95[e];
        T.svc[e] = svc_ms[e];
        if (mem_ok[e]) T.mem_ok |= 1ULL << e;
    }
    for (int k = 0; k < CLV_K; ++k) {
        if (idle_q5[k] < 0 || idle_q5[k] >= LIM) return fail(ctx, CLV_ERR_PROFILE, "idle row out of range");
        T.idle_q[k] = idle_q5[k];
    }
    {   // rate moments thr^2, thr^3 (thr = 1000 / svc) as fixed-point rows < 2^31 (round half even,
        // as oracle/tables.py::rate_moment_rows)
        double t2[CLV_MAX_EDGES], t3[CLV_MAX_EDGES], m2 = 0.0, m3 = 0.0;
        for (int e = 0; e < T.E; ++e) {
            const double thr = 1000.0 / svc_ms[e];
            t2[e] = thr * thr;
            t3[e] = t2[e] * thr;
            m2 = std::max(m2, t2[e]);
            m3 = std::max(m3, t3[e]);
        }
        int ex;
        std::frexp(m2, &ex); T.k2 = 31 - ex;
        std::frexp(m3, &ex); T.k3 = 31 - ex;
        for (int e = 0; e < T.E; ++e) {
            T.t2_q[e] = (long long)std::nearbyint(std::ldexp(t2[e], T.k2));
            T.t3_q[e] = (long long)std::nearbyint(std::ldexp(t3[e], T.k3));
        }
    }
    std::vector<int> ord(T.E);
    for (int e = 0; e < T.E; ++e) ord[e] = e;
    std::sort(ord.begin(), ord.end(), [&](int x, int y) {
        return T.lat95[x] != T.lat95[y] ? T.lat95[x] < T.lat95[y] : x < y;
    });
    for (int r = 0; r < T.E; ++r) {
        T.rank[ord[r]] = (unsigned char)r; T.lat_by_rank[r] = T.lat95[ord[r]];
        T.svc_by_rank[r] = T.svc[ord[r]]; T.edge_by_rank[r] = (unsigned char)ord[r];
    }
    int nbmax = 0;
    for (int e = 0; e < T.E; ++e) {
        int c = 0;
        for (int x = 0; x < T.E; ++x) {
            if (x == e || !((T.mem_ok >> x) & 1ULL)) continue;
            if (x / 5 == e / 5 || x % 5 == e % 5) T.nb[e][c++] = (unsigned char)x;
        }
        T.nb_cnt[e] = (unsigned char)c;
        nbmax = std::max(nbmax, c);
    }
    T.nbmax = std::max(nbmax, 1);
    for (int k = 0; k < CLV_K; ++k) {
        int c = 0;
        for (int v = 0; v < V; ++v)
            if ((T.mem_ok >> (v * 5 + k)) & 1ULL) T.feas_list[k][c++] = (unsigned char)v;
        T.nfeas[k] = (unsigned char)c;
    }
    // static double-move lists (see FamilyTables::pair_list)
    std::vector<uint32_t> plist;
    auto adj = [](int x, int y) { return x != y && (x / 5 == y / 5 || x % 5 == y % 5); };
    auto P = [&](int x, int y) { return x * T.E - (x * (x - 1)) / 2 + (y - x); };
    for (int r1 = 0; r1 < T.E; ++r1)
        for (int r2 = r1; r2 < T.E; ++r2) {
            const int p = P(r1, r2);
            T.pair_off[p] = (int)plist.size();
            int len = 0;
            for (int ii = 0; ii < T.nb_cnt[r1]; ++ii)
                for (int jj = 0; jj < T.nb_cnt[r2]; ++jj) {
                    const int a1 = T.nb[r1][ii], a2 = T.nb[r2][jj];
                    if (a1 == r2 || a2 == r1) continue;
                    if (a1 > a2 && adj(r1, a2) && adj(r2, a1)) continue;
                    const int lo = std::min(a1, a2), hi = std::max(a1, a2);
                    plist.push_back((uint32_t)a1 | ((uint32_t)a2 << 6) |
                                    ((uint32_t)((a1 % 5) * 5 + (a2 % 5)) << 12) | ((uint32_t)P(lo, hi) << 17));
                    ++len;
                }
            if (len > 255) return fail(ctx, CLV_ERR_PROFILE, "internal: move list too long");
            T.pair_len[p] = (unsigned char)len;
        }
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaFree(ctx->pair_list_dev[family]);
    ctx->pair_list_dev[family] = nullptr;
    CLV_CUDA(cudaMalloc(&ctx->pair_list_dev[family], std::max<size_t>(1, plist.size()) * sizeof(uint32_t)), "alloc move lists");
    if (!plist.empty())
        CLV_CUDA(cudaMemcpy(ctx->pair_list_dev[family], plist.data(), plist.size() * sizeof(uint32_t), cudaMemcpyHostToDevice), "copy move lists");
    T.pair_list = ctx->pair_list_dev[family];
    CLV_CUDA(cudaMemcpy(ctx->fam_dev + family, &T, sizeof(FamilyTables), cudaMemcpyHostToDevice), "copy profile");
    ctx->fam[family] = T;
    ctx->fam_set[family] = true;
    return CLV_OK;
}

int clv_build_feasibility(clv_ctx *ctx, int n_max, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    if (!ctx->topo_set) return fail(ctx, CLV_ERR_NOT_READY, "topology not loaded");
    if (n_max < 1 || n_max > 160) return fail(ctx, CLV_ERR_CARBON_SCHED, "n_max must be in 1..160");
    cudaStream_t st = (cudaStream_t)stream;
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    const int bdim = 7 * n_max / 4 + 1, cdim = 7 * n_max / 3 + 1;
    std::vector<uint32_t> off((size_t)(n_max + 1) * bdim * cdim, 0xFFFFFFFFu);
    std::vector<int2> bc;
    std::vector<int> bc_start(n_max + 2, 0);
    unsigned long long cursor = 0;
    for (int N = 0; N <= n_max; ++N) {
        bc_start[N] = (int)bc.size();
        for (int b = 0; 4 * b <= 7 * N; ++b)
            for (int c = 0; 4 * b + 3 * c <= 7 * N; ++c) {
                int R = 7 * N - 4 * b - 3 * c;
                off[((size_t)N * bdim + b) * cdim + c] = (uint32_t)cursor;
                cursor += (unsigned long long)(R / 2 + 1) * ((R + 32) >> 5);
                bc.push_back(make_int2(b, c));
            }
    }
    bc_start[n_max + 1] = (int)bc.size();
    if (cursor >= 0xFFFFFFFFull) return fail(ctx, CLV_ERR_OUT_OF_MEMORY, "feasibility table too large");
    cudaFree(ctx->feas_bits); cudaFree(ctx->feas_off);
    ctx->feas_bits = nullptr; ctx->feas_off = nullptr; ctx->feas_nmax = -1;
    uint32_t *bits = nullptr, *doff = nullptr;
    int2 *dbc = nullptr;
    int *drows = nullptr;
    CLV_CUDA(cudaMalloc(&bits, cursor * sizeof(uint32_t)), "alloc feasibility bits");
    CLV_CUDA(cudaMalloc(&doff, off.size() * sizeof(uint32_t)), "alloc feasibility offsets");
    CLV_CUDA(cudaMalloc(&dbc, bc.size() * sizeof(int2)), "alloc bc list");
    CLV_CUDA(cudaMalloc(&drows, sizeof(int) * 4 * CLV_MAX_CONFIGS), "alloc rows");
    CLV_CUDA(cudaMemcpyAsync(doff, off.data(), off.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st), "copy off");
    CLV_CUDA(cudaMemcpyAsync(dbc, bc.data(), bc.size() * sizeof(int2), cudaMemcpyHostToDevice, st), "copy bc");
    CLV_CUDA(cudaMemcpyAsync(drows, &ctx->topo.rows4[0][0], sizeof(int) * 4 * CLV_MAX_CONFIGS, cudaMemcpyHostToDevice, st), "copy rows");
    for (int N = 0; N <= n_max; ++N) {
        CLV_CUDA(launch_feas_level(bits, doff, N, bdim, cdim, dbc + bc_start[N], bc_start[N + 1] - bc_start[N],
                                   drows, ctx->topo.nrows4, st), "feasibility level");
    }
    CLV_CUDA(cudaStreamSynchronize(st), "feasibility build");
    cudaFree(dbc); cudaFree(drows);
    ctx->feas_bits = bits; ctx->feas_off = doff; ctx->feas_words = cursor;
    ctx->feas_nmax = n_max; ctx->bdim = bdim; ctx->cdim = cdim;
    return CLV_OK;
}

int64_t clv_feasibility_bytes(const clv_ctx *ctx) {
    if (!ctx || ctx->feas_nmax < 0) return 0;
    return (int64_t)ctx->feas_words * 4 + (int64_t)(ctx->feas_nmax + 1) * ctx->bdim * ctx->cdim * 4;
}

static int need_feas(clv_ctx *ctx, int n) {
    if (ctx->feas_nmax < 0 || n > ctx->feas_nmax)
        return fail(ctx, CLV_ERR_NOT_READY, "feasibility tables cover n <= " + std::to_string(ctx->feas_nmax) +
                                                "; call clv_build_feasibility(n_max >= " + std::to_string(n) + ")");
    return CLV_OK;
}

int clv_feasible(clv_ctx *ctx, int n, const int32_t *vec5_dev, int64_t count, uint8_t *out_dev, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    int rc = need_feas(ctx, n);
    if (rc) return rc;
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    CLV_CUDA(launch_feasible(feas_view(ctx), n, vec5_dev, count, out_dev, (cudaStream_t)stream), "feasible");
    return CLV_OK;
}

int clv_realize(clv_ctx *ctx, int n, const int32_t *vec5_host, int32_t *parts_host, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    int rc = need_feas(ctx, n);
    if (rc) return rc;
    if (n > 1000) return fail(ctx, CLV_ERR_CARBON_SCHED, "n too large");
    cudaStream_t st = (cudaStream_t)stream;
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    CLV_CUDA(cudaMemcpyAsync(ctx->small_dev, vec5_host, 5 * sizeof(int32_t), cudaMemcpyHostToDevice, st), "copy vec");
    CLV_CUDA(launch_realize(feas_view(ctx), ctx->topo_dev, n, ctx->small_dev, ctx->small_dev + 8, st), "realize");
    CLV_CUDA(cudaMemcpyAsync(parts_host, ctx->small_dev + 8, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st), "copy parts");
    CLV_CUDA(cudaStreamSynchronize(st), "realize sync");
    if (parts_host[0] < 0) return fail(ctx, CLV_ERR_INFEASIBLE_GRAPH, "slice multiset has no realization on n GPUs");
    return CLV_OK;
}

int clv_score_graphs(clv_ctx *ctx, int family, const uint16_t *w_dev, int64_t count, int64_t index_base,
                     const clv_eval_params *params, int select_mode, double *f_dev, double *h_dev,
                     uint8_t *sla_dev, uint8_t *feas_dev, double *p95_dev, clv_best *best, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    int rc = need_family(ctx, family);
    if (rc) return rc;
    ScoreArgs a{};
    rc = make_ec(ctx, params, ctx->fam[family], a.ec);
    if (rc) return rc;
    rc = need_feas(ctx, params->n_gpus);
    if (rc) return rc;
    if (count < 0) return fail(ctx, CLV_ERR_CARBON_SCHED, "negative count");
    if (select_mode != CLV_SELECT_BEST_H && select_mode != CLV_SELECT_ORACLE)
        return fail(ctx, CLV_ERR_CARBON_SCHED, "unknown select mode");
    cudaStream_t st = (cudaStream_t)stream;
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    a.fam = ctx->fam_dev + family; a.F = feas_view(ctx); a.select_mode = select_mode;
    a.count = count; a.index_base = index_base; a.w = w_dev; a.topo = ctx->topo_dev;
    a.f_out = f_dev; a.h_out = h_dev; a.p95_out = p95_dev; a.sla_out = sla_dev; a.feas_out = feas_dev;
    a.sel = make_sel(ctx);
    a.fast = fast_div_safe(a.ec, ctx->fam[family].lat95, ctx->fam[family].svc, ctx->fam[family].E) ? 1 : 0;
    CLV_CUDA(launch_score_graphs(a, ctx->fam[family], grid_for(ctx, count, 256), st), "score_graphs");
    if (!best) return CLV_OK;
    return fetch_best(ctx, select_mode, st, best);
}

int clv_score_x(clv_ctx *ctx, int family, int n, const uint8_t *xp_dev, const uint8_t *xv_dev,
                const int64_t *xv_off_dev, int64_t count, int64_t index_base, const clv_eval_params *params,
                int select_mode, double *f_dev, double *h_dev, uint8_t *sla_dev, clv_best *best, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    int rc = need_family(ctx, family);
    if (rc) return rc;
    ScoreArgs a{};
    rc = make_ec(ctx, params, ctx->fam[family], a.ec);
    if (rc) return rc;
    if (n < 1) return fail(ctx, CLV_ERR_CARBON_SCHED, "a fleet needs at least one GPU");
    cudaStream_t st = (cudaStream_t)stream;
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    CLV_CUDA(cudaMemsetAsync(ctx->err_index, 0xFF, sizeof(long long), st), "reset err key");
    a.fam = ctx->fam_dev + family; a.select_mode = select_mode; a.count = count; a.index_base = index_base;
    a.xp = xp_dev; a.xv = xv_dev; a.xv_off = xv_off_dev; a.topo = ctx->topo_dev;
    a.f_out = f_dev; a.h_out = h_dev; a.sla_out = sla_dev; a.sel = make_sel(ctx);
    a.error_key = reinterpret_cast<unsigned long long *>(ctx->err_index);
    a.fast = fast_div_safe(a.ec, ctx->fam[family].lat95, ctx->fam[family].svc, ctx->fam[family].E) ? 1 : 0;
    CLV_CUDA(launch_score_x(a, n, grid_for(ctx, count, 256), st), "score_x");
    CLV_CUDA(cudaMemcpyAsync(ctx->host_err + 2, ctx->err_index, sizeof(long long), cudaMemcpyDeviceToHost, st), "copy err key");
    rc = fetch_best(ctx, select_mode, st, best);
    if (rc) return rc;
    unsigned long long key;
    std::memcpy(&key, ctx->host_err + 2, sizeof(key));
    if (key != ~0ULL) {                       // lowest failing row, its first error (mig.py:248-263)
        const long long idx = (long long)(key >> 8) + index_base;
        const int code = (int)(key & 0xFF);
        const std::string what = code == CLV_ERR_INVALID_CONFIG ? "unknown MIG partition id"
                               : code == SCORE_X_VARIANT_LT1 ? "variant ordinals start at 1"
                               : code == CLV_ERR_INFEASIBLE_ASSIGNMENT ? "variant out of range or does not fit its slice"
                               : "assignment length does not match the slices implied by the partitions";
        return fail(ctx, code == SCORE_X_VARIANT_LT1 ? CLV_ERR_CARBON_SCHED : code,
                    "candidate " + std::to_string(idx) + ": " + what);
    }
    return CLV_OK;
}

static void oracle_rows(const clv_ctx *ctx, const FamilyTables &T, long long *row_off, int (*place)[8]) {
    long long acc = 0;
    for (int r = 0; r < ctx->topo.K; ++r) {
        row_off[r] = acc;
        long long cnt = 1;
        int ns = ctx->topo.nslices[r];
        for (int j = ns - 1; j >= 0; --j) {
            if (place) place[r][j] = (int)cnt;
            cnt *= T.nfeas[ctx->topo.kinds[r][j]];
        }
        acc += cnt;
    }
    row_off[ctx->topo.K] = acc;
}

int clv_oracle_size(clv_ctx *ctx, int family, int64_t *total) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    int rc = need_family(ctx, family);
    if (rc) return rc;
    long long off[CLV_MAX_CONFIGS + 1];
    oracle_rows(ctx, ctx->fam[family], off, nullptr);
    *total = off[ctx->topo.K];
    return CLV_OK;
}

int clv_oracle_decode(clv_ctx *ctx, int family, int64_t index, int32_t *cid, int32_t *assign7, int32_t *ns_out) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    int rc = need_family(ctx, family);
    if (rc) return rc;
    long long off[CLV_MAX_CONFIGS + 1];
    int place[CLV_MAX_CONFIGS][8];
    const FamilyTables &T = ctx->fam[family];
    oracle_rows(ctx, T, off, place);
    if (index < 0 || index >= off[ctx->topo.K]) return fail(ctx, CLV_ERR_CARBON_SCHED, "oracle index out of range");
    int r = 0;
    while (r + 1 < ctx->topo.K && off[r + 1] <= index) ++r;
    long long rem = index - off[r];
    *cid = ctx->topo.ids[r];
    *ns_out = ctx->topo.nslices[r];
    for (int j = 0; j < ctx->topo.nslices[r]; ++j) {
        int d = (int)(rem / place[r][j]);
        rem -= (long long)d * place[r][j];
        assign7[j] = T.feas_list[ctx->topo.kinds[r][j]][d] + 1;
    }
    return CLV_OK;
}

int clv_oracle_search(clv_ctx *ctx, int family, int n, int64_t begin, int64_t end, const clv_eval_params *params,
                      clv_best *best, int64_t *total, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    int rc = need_family(ctx, family);
    if (rc) return rc;
    OracleArgs a{};
    rc = make_ec(ctx, params, ctx->fam[family], a.ec);
    if (rc) return rc;
    if (n < 1) return fail(ctx, CLV_ERR_CARBON_SCHED, "a fleet needs at least one GPU");
    oracle_rows(ctx, ctx->fam[family], a.row_off, a.row_place);
    long long tot = a.row_off[ctx->topo.K];
    if (total) *total = tot;
    if (begin < 0) begin = 0;
    if (end < 0 || end > tot) end = tot;
    if (end < begin) end = begin;
    cudaStream_t st = (cudaStream_t)stream;
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    a.fam = ctx->fam_dev + family; a.topo = ctx->topo_dev; a.begin = begin; a.end = end; a.n = n;
    a.sel = make_sel(ctx);
    a.fast = fast_div_safe(a.ec, ctx->fam[family].lat95, ctx->fam[family].svc, ctx->fam[family].E) ? 1 : 0;
    CLV_CUDA(launch_oracle(a, grid_for(ctx, end - begin, 256), st), "oracle");
    return fetch_best(ctx, CLV_SELECT_ORACLE, st, best);
}

int clv_anneal(clv_ctx *ctx, int family, int n, int n_chains, int64_t chain_base, const uint16_t *start_w_dev,
               const clv_eval_params *params, int n_params, const clv_anneal_params *ap, uint64_t seed,
               int cluster_size, clv_chain_result *results_dev, uint16_t *best_w_dev, uint16_t *final_w_dev,
               clv_log_row *log_dev, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    int rc = need_family(ctx, family);
    if (rc) return rc;
    rc = need_feas(ctx, n);
    if (rc) return rc;
    if (n_chains < 0) return fail(ctx, CLV_ERR_CARBON_SCHED, "negative chain count");
    if (n_chains == 0) return CLV_OK;
    if (!ap || !(ap->t_floor > 0) || !(ap->cooling_step > 0) || ap->stall_limit < 1 || ap->max_steps < 0 ||
        ap->proposal < 0 || ap->proposal > 1 || ap->evaluate < 0 || ap->evaluate > 1 ||
        (ap->proposal == 0 && ap->evaluate != 0) || (ap->flags & ~3) ||
        ((ap->flags & CLV_ANNEAL_MULT_COOLING) && !(ap->cooling_step < 1.0)))
        return fail(ctx, CLV_ERR_CARBON_SCHED, "invalid anneal parameters");
    if (n_params != 1 && n_params != n_chains) return fail(ctx, CLV_ERR_CARBON_SCHED, "n_params must be 1 or n_chains");
    if (cluster_size < 0 || cluster_size > 16)
        return fail(ctx, CLV_ERR_CARBON_SCHED, "cluster_size must be 0 (auto) or 1..16");
    std::vector<EvalConst> ecs(n_params);
    for (int i = 0; i < n_params; ++i) {
        rc = make_ec(ctx, params + i, ctx->fam[family], ecs[i]);
        if (rc) return rc;
        if (params[i].n_gpus != n) return fail(ctx, CLV_ERR_CARBON_SCHED, "params.n_gpus must equal n");
    }
    cudaStream_t st = (cudaStream_t)stream;
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (ctx->ec_cap < n_params) {
        cudaFree(ctx->ec_dev);
        ctx->ec_dev = nullptr;
        CLV_CUDA(cudaMalloc(&ctx->ec_dev, sizeof(EvalConst) * n_params), "alloc eval consts");
        ctx->ec_cap = n_params;
    }
    CLV_CUDA(cudaMemcpyAsync(ctx->ec_dev, ecs.data(), sizeof(EvalConst) * n_params, cudaMemcpyHostToDevice, st), "copy eval consts");
    AnnealArgs a{};
    a.fam = ctx->fam_dev + family; a.F = feas_view(ctx); a.ec = ctx->ec_dev; a.n_ec = n_params; a.ec0 = ecs[0];
    a.fast_div = 1;
    for (int i = 0; i < n_params; ++i)
        if (!fast_div_safe(ecs[i], ctx->fam[family].lat95, ctx->fam[family].svc, ctx->fam[family].E)) a.fast_div = 0;
    a.t_init = ap->t_init; a.cooling = ap->cooling_step; a.t_floor = ap->t_floor;
    a.cool_factor = 1.0 - ap->cooling_step; a.flags = ap->flags;
    a.stall_limit = ap->stall_limit; a.max_steps = ap->max_steps; a.proposal = ap->proposal; a.evaluate = ap->evaluate;
    a.n = n; a.n_chains = n_chains; a.E = ctx->fam[family].E; a.chain_base = chain_base; a.seed = seed;
    a.start_w = start_w_dev; a.res = results_dev; a.best_w = best_w_dev; a.final_w = final_w_dev; a.log = log_dev;
    {
        const size_t need = (size_t)n_chains * (size_t)std::max(ap->max_steps, 1);
        if (need > ctx->mvlog_cap) {
            cudaFree(ctx->mvlog);
            ctx->mvlog = nullptr; ctx->mvlog_cap = 0;
            CLV_CUDA(cudaMalloc(&ctx->mvlog, need * sizeof(int)), "alloc move log");
            ctx->mvlog_cap = need;
        }
        a.mvlog = ctx->mvlog;
        if (!ctx->chain_counter) CLV_CUDA(cudaMalloc(&ctx->chain_counter, sizeof(int)), "alloc chain counter");
        a.chain_counter = ctx->chain_counter;    // used (and zeroed) only by persistent launches
    }
    {
        // debug phase profile buffer (CLV_ANNEAL_VARIANT=9 only)
        const char *v = getenv("CLV_ANNEAL_VARIANT");
        if (v && atoi(v) == 9) {
            size_t need = (size_t)n_chains * 16 * PROF_SLOTS;
            if (prof_cap < need) { cudaFree(prof_buf); cudaMalloc(&prof_buf, need * sizeof(long long)); prof_cap = need; }
            cudaMemsetAsync(prof_buf, 0, need * sizeof(long long), st);
            a.prof = prof_buf;
        }
    }
    CLV_CUDA(launch_anneal(a, cluster_size, st), "anneal");
    return CLV_OK;
}

// debug: copy the last phase profile (CLV_ANNEAL_VARIANT=9) -- not part of the public ABI
int clv_debug_anneal_profile(long long *host, size_t count) {
    if (!prof_buf || count > prof_cap) return CLV_ERR_NOT_READY;
    return cudaMemcpy(host, prof_buf, count * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? CLV_OK : CLV_ERR_CUDA;
}

int clv_select_chains(clv_ctx *ctx, const clv_chain_result *res, int n_chains, int64_t chain_base,
                      clv_record *rec_dev, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    CLV_CUDA(launch_select_chains(res, n_chains, chain_base, rec_dev, (cudaStream_t)stream), "select_chains");
    return CLV_OK;
}

int clv_replan(clv_ctx *ctx, int family, int n, int n_chains, int64_t chain_base, const uint16_t *start_w_host,
               const clv_eval_params *params, int n_params, const clv_anneal_params *ap, uint64_t seed,
               int cluster_size, clv_chain_result *results_host, uint16_t *best_w_host, uint16_t *final_w_host,
               clv_record *record_host, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    // one NVTX range per re-plan (visible in nsys / ncu --nvtx timelines); header-only NVTX3
    struct NvtxRange {
        NvtxRange() { nvtxRangePushA("clv_replan"); }
        ~NvtxRange() { nvtxRangePop(); }
    } nvtx_range;
    int rc = need_family(ctx, family);
    if (rc) return rc;
    if (n_chains < 1) return fail(ctx, CLV_ERR_CARBON_SCHED, "a re-plan needs at least one chain");
    if (!start_w_host || !results_host || !best_w_host || !final_w_host || !record_host)
        return fail(ctx, CLV_ERR_CARBON_SCHED, "null host buffer");
    const size_t E = (size_t)ctx->fam[family].E;
    auto up16 = [](size_t b) { return (b + 15) & ~(size_t)15; };
    const size_t b_in = up16(n_chains * E * 2), b_res = up16(n_chains * sizeof(clv_chain_result));
    const size_t b_w = up16(n_chains * E * 2), b_rec = up16(sizeof(clv_record));
    const size_t need = b_in + b_res + 2 * b_w + b_rec;
    cudaStream_t st = (cudaStream_t)stream;
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (ctx->replan_cap < need) {
        CLV_CUDA(cudaStreamSynchronize(st), "synchronize");
        cudaFree(ctx->replan_buf);
        ctx->replan_buf = nullptr; ctx->replan_cap = 0;
        CLV_CUDA(cudaMalloc(&ctx->replan_buf, need), "alloc re-plan staging");
        ctx->replan_cap = need;
    }
    unsigned char *b = ctx->replan_buf;
    uint16_t *d_in = reinterpret_cast<uint16_t *>(b);
    clv_chain_result *d_res = reinterpret_cast<clv_chain_result *>(b + b_in);
    uint16_t *d_best = reinterpret_cast<uint16_t *>(b + b_in + b_res);
    uint16_t *d_final = reinterpret_cast<uint16_t *>(b + b_in + b_res + b_w);
    clv_record *d_rec = reinterpret_cast<clv_record *>(b + b_in + b_res + 2 * b_w);
    CLV_CUDA(cudaMemcpyAsync(d_in, start_w_host, n_chains * E * 2, cudaMemcpyHostToDevice, st), "copy starts");
    rc = clv_anneal(ctx, family, n, n_chains, chain_base, d_in, params, n_params, ap, seed, cluster_size, d_res,
                    d_best, d_final, nullptr, stream);
    if (rc) return rc;
    rc = clv_select_chains(ctx, d_res, n_chains, chain_base, d_rec, stream);
    if (rc) return rc;
    CLV_CUDA(cudaMemcpyAsync(results_host, d_res, n_chains * sizeof(clv_chain_result), cudaMemcpyDeviceToHost, st),
             "copy results");
    CLV_CUDA(cudaMemcpyAsync(best_w_host, d_best, n_chains * E * 2, cudaMemcpyDeviceToHost, st), "copy best");
    CLV_CUDA(cudaMemcpyAsync(final_w_host, d_final, n_chains * E * 2, cudaMemcpyDeviceToHost, st), "copy final");
    CLV_CUDA(cudaMemcpyAsync(record_host, d_rec, sizeof(clv_record), cudaMemcpyDeviceToHost, st), "copy record");
    CLV_CUDA(cudaStreamSynchronize(st), "synchronize");
    return CLV_OK;
}

int clv_reduce_records(clv_ctx *ctx, const clv_record *recs, int count, clv_record *out, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    CLV_CUDA(launch_reduce_records(recs, count, out, (cudaStream_t)stream), "reduce_records");
    return CLV_OK;
}

static int make_pods(clv_ctx *ctx, int n_pods, const clv_pod *pods, SweepArgs &a) {
    if (n_pods < 1 || n_pods > CLV_MAX_PODS) return fail(ctx, CLV_ERR_CARBON_SCHED, "1..8 pods");
    a.n_pods = n_pods;
    for (int p = 0; p < n_pods; ++p) {
        int rc = need_family(ctx, pods[p].family);
        if (rc) return rc;
        const FamilyTables &T = ctx->fam[pods[p].family];
        for (int k = 0; k < CLV_K; ++k)
            if (T.nfeas[k] == 0) return fail(ctx, CLV_ERR_PROFILE, "a slice kind has no memory-feasible variant");
        if (pods[p].n_gpus < 1) return fail(ctx, CLV_ERR_CARBON_SCHED, "pod needs >= 1 GPU");
        a.pods[p].family = pods[p].family;
        a.pods[p].n_gpus = pods[p].n_gpus;
        a.pods[p].weight = pods[p].weight;
        rc = make_ec(ctx, &pods[p].params, T, a.pods[p].ec);
        if (rc) return rc;
    }
    return CLV_OK;
}

int clv_sweep(clv_ctx *ctx, int n_pods, const clv_pod *pods, int64_t begin, int64_t end, uint64_t seed,
              double *f_dev, double *h_dev, uint8_t *sla_dev, clv_best *best, void *stream) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    if (!ctx->topo_set) return fail(ctx, CLV_ERR_NOT_READY, "topology not loaded");
    SweepArgs a{};
    int rc = make_pods(ctx, n_pods, pods, a);
    if (rc) return rc;
    if (end < begin) return fail(ctx, CLV_ERR_CARBON_SCHED, "empty range");
    cudaStream_t st = (cudaStream_t)stream;
    CLV_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    a.fam = ctx->fam_dev; a.topo = ctx->topo_dev; a.begin = begin; a.end = end; a.seed = seed;
    a.f_out = f_dev; a.h_out = h_dev; a.sla_out = sla_dev; a.sel = make_sel(ctx);
    a.fast = 1;
    for (int p = 0; p < a.n_pods; ++p) {
        const FamilyTables &T = ctx->fam[a.pods[p].family];
        if (!fast_div_safe(a.pods[p].ec, T.lat95, T.svc, T.E)) a.fast = 0;
    }
    CLV_CUDA(launch_sweep(a, grid_for(ctx, end - begin, 256), st), "sweep");
    if (!best) return CLV_OK;
    return fetch_best(ctx, CLV_SELECT_BEST_H, st, best);
}

int clv_sweep_decode(clv_ctx *ctx, int n_pods, const clv_pod *pods, uint64_t seed, int64_t index,
                     int32_t *parts, int32_t *assigns, int32_t *n_assign) {
    if (!ctx) return CLV_ERR_CARBON_SCHED;
    if (!ctx->topo_set) return fail(ctx, CLV_ERR_NOT_READY, "topology not loaded");
    SweepArgs a{};
    int rc = make_pods(ctx, n_pods, pods, a);
    if (rc) return rc;
    uint64_t h0 = derive_seed2(seed, (uint64_t)index), word = 0;
    uint32_t j = 0;
    auto next = [&]() -> uint32_t {
        uint32_t out;
        if ((j & 1u) == 0) { word = stream_word(h0, j >> 1); out = (uint32_t)word; }
        else out = (uint32_t)(word >> 32);
        ++j;
        return out;
    };
    auto bounded = [&](uint32_t k) { return (int)(((uint64_t)next() * k) >> 32); };
    int g_out = 0, s_out = 0;
    for (int p = 0; p < n_pods; ++p) {
        const FamilyTables &T = ctx->fam[pods[p].family];
        for (int g = 0; g < pods[p].n_gpus; ++g) {
            int r = bounded((uint32_t)ctx->topo.K);
            parts[g_out++] = ctx->topo.ids[r];
            for (int q = 0; q < ctx->topo.nslices[r]; ++q) {
                int k = ctx->topo.kinds[r][q];
                assigns[s_out++] = T.feas_list[k][bounded(T.nfeas[k])] + 1;
            }
        }
    }
    *n_assign = s_out;
    return CLV_OK;
}

}  // extern "C"
