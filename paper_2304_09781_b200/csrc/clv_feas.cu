// clv_feas.cu -- K6: exact fleet-feasibility tables on the device.
//
// Reference predicate: "the slice multiset splits into exactly n partition
// rows" (mig.py:144-181).  Because a 7g slice fills a GPU, the vector
// (a,b,c,d,e) is feasible on n GPUs iff (b,c,d,e) is a sum of exactly N = n-a
// rows without 7g.  T'_N is built level by level with the sum-set recurrence
// T'_N = U_k (T'_{N-1} + row_k) as shift-OR over bitsets along e (#1g).
//
// HBM layout: for each (N, b, c) with
// 4b+3c <= 7N a rectangle of rows d = 0..R/2 (R = 7N-4b-3c), each row a bitset
// of wpr = ceil((R+1)/32) uint32 words over e = 0..R.  off[(N*bdim+b)*cdim+c]
// is the rectangle's first word.  One CTA per (b,c) key, threads over words.
#include "clv_internal.h"

namespace clv {

__global__ void __launch_bounds__(256) feas_level_kernel(uint32_t *bits, const uint32_t *off, int N,
                                                         int bdim, int cdim, const int2 *bc_list,
                                                         const int *rows4, int nrows4) {
    __shared__ int rows[CLV_MAX_CONFIGS][4];
    for (int t = threadIdx.x; t < nrows4 * 4; t += blockDim.x) rows[t / 4][t % 4] = rows4[t];
    __syncthreads();
    const int b = bc_list[blockIdx.x].x, c = bc_list[blockIdx.x].y;
    const int R = 7 * N - 4 * b - 3 * c;
    const int wpr = (R + 32) >> 5;
    const int drows = R / 2 + 1;
    const uint32_t base = off[((size_t)N * bdim + b) * cdim + c];
    for (int t = threadIdx.x; t < drows * wpr; t += blockDim.x) {
        const int d = t / wpr, w = t - d * wpr;
        const int emax = R - 2 * d;
        uint32_t acc = 0;
        if (N == 0) {
            acc = (w == 0) ? 1u : 0u;           // T'_0 = {0}
        } else if (32 * w <= emax) {
            for (int k = 0; k < nrows4; ++k) {
                const int sb = b - rows[k][0], sc = c - rows[k][1], sd = d - rows[k][2];
                const int re = rows[k][3];
                if (sb < 0 || sc < 0 || sd < 0) continue;
                const int Rs = 7 * (N - 1) - 4 * sb - 3 * sc;
                if (Rs < 0 || 2 * sd > Rs) continue;
                const int swpr = (Rs + 32) >> 5;
                const uint32_t *src = bits + off[((size_t)(N - 1) * bdim + sb) * cdim + sc] + (size_t)sd * swpr;
                const int lo = 32 * w - re;
                uint32_t v;
                if (lo < 0) {
                    v = src[0] << re;
                } else {
                    const int q = lo >> 5, sh = lo & 31;
                    const uint32_t a0 = q < swpr ? src[q] : 0u;
                    const uint32_t a1 = (q + 1) < swpr ? src[q + 1] : 0u;
                    v = sh ? ((a0 >> sh) | (a1 << (32 - sh))) : a0;
                }
                acc |= v;
            }
            const int first = 32 * w;
            if (emax - first < 31) acc &= (2u << (emax - first)) - 1u;
        }
        bits[base + (size_t)d * wpr + w] = acc;
    }
}

cudaError_t launch_feas_level(uint32_t *bits, const uint32_t *off, int N, int bdim, int cdim,
                              const int2 *bc_list, int n_bc, const int *rows4, int nrows4,
                              cudaStream_t s) {
    if (n_bc <= 0) return cudaSuccess;
    feas_level_kernel<<<n_bc, 256, 0, s>>>(bits, off, N, bdim, cdim, bc_list, rows4, nrows4);
    return cudaGetLastError();
}

__global__ void feasible_kernel(FeasView F, int n, const int32_t *vec5, long long count, uint8_t *out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        const int32_t *v = vec5 + 5 * i;
        out[i] = feasible(F, n, v[0], v[1], v[2], v[3], v[4]) ? 1 : 0;
    }
}

cudaError_t launch_feasible(FeasView F, int n, const int32_t *vec5, long long count, uint8_t *out,
                            cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    long long blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    feasible_kernel<<<(unsigned)blocks, 256, 0, s>>>(F, n, vec5, count, out);
    return cudaGetLastError();
}

// realize: canonical partition = greedy smallest feasible id
// (the lexicographically smallest non-decreasing id tuple, mig.py:144-177).
__global__ void realize_kernel(FeasView F, const Topology *topo, int n, const int32_t *vec5,
                               int32_t *parts) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int v[CLV_K];
    for (int k = 0; k < CLV_K; ++k) v[k] = vec5[k];
    if (!feasible(F, n, v[0], v[1], v[2], v[3], v[4])) { parts[0] = -1; return; }
    for (int g = 0; g < n; ++g) {
        int left = n - g - 1;
        int chosen = -1;
        for (int r = 0; r < topo->K && chosen < 0; ++r) {
            int u[CLV_K];
            bool ok = true;
            for (int k = 0; k < CLV_K; ++k) { u[k] = v[k] - topo->counts[r][k]; ok &= u[k] >= 0; }
            if (!ok) continue;
            bool f = (left == 0) ? (u[0] | u[1] | u[2] | u[3] | u[4]) == 0
                                 : feasible(F, left, u[0], u[1], u[2], u[3], u[4]);
            if (f) {
                chosen = r;
                for (int k = 0; k < CLV_K; ++k) v[k] = u[k];
            }
        }
        if (chosen < 0) { parts[0] = -2; return; }
        parts[g] = topo->ids[chosen];
    }
}

cudaError_t launch_realize(FeasView F, const Topology *topo_dev, int n, const int32_t *vec5_dev,
                           int32_t *parts_dev, cudaStream_t s) {
    realize_kernel<<<1, 32, 0, s>>>(F, topo_dev, n, vec5_dev, parts_dev);
    return cudaGetLastError();
}

}  // namespace clv
