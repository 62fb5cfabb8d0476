// clv_debug.cu -- self-checks of device arithmetic that the kernels rely on (not part of
// the public ABI; called by tests/test_gpu_fast_div.py).
//
// div_rn_fast (clv_common.cuh) must equal IEEE division on every operand the scoring
// epilogue can hand it under fast_div_safe():
//   (i)   1 / S_thr,           S_thr in [1, 2^53]                  -> quotient bits
//   (ii)  rho^8 / (m (1 - rho)), rho^8 in [0, 1], m (1-rho) in [1e-12, 1e5]
//                                                                  -> bits of 1 + quotient
//   (iii) slo / L and L / slo, both in [1e-12, 1e24]                -> quotient bits
#include "clv_internal.h"

namespace clv {

__device__ __forceinline__ double log_uniform(uint64_t h, double lo_exp2, double hi_exp2) {
    const double u = (double)(h >> 11) * 0x1.0p-53;
    return exp2(lo_exp2 + u * (hi_exp2 - lo_exp2));
}

__global__ void fast_div_check_kernel(long long n, uint64_t seed, unsigned long long *bad) {
    unsigned long long local = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const uint64_t h1 = derive_seed4(seed, (uint64_t)i, 1, 0), h2 = derive_seed4(seed, (uint64_t)i, 2, 0);
        const int kind = (int)(i % 3);
        double a, b;
        bool ok;
        if (kind == 0) {
            b = floor(log_uniform(h1, 0.0, 53.0));                      // an exact integer sum
            a = 1.0;
            ok = __double_as_longlong(div_rn_fast(a, b)) == __double_as_longlong(a / b);
        } else if (kind == 1) {
            a = (h2 & 7) == 0 ? 0.0 : log_uniform(h2, -1100.0, 0.0);   // includes subnormals
            b = log_uniform(h1, -39.9, 16.7);
            ok = __double_as_longlong(1.0 + div_rn_fast(a, b)) == __double_as_longlong(1.0 + a / b);
        } else {
            a = log_uniform(h1, -39.9, 79.8);
            b = log_uniform(h2, -39.9, 79.8);
            ok = __double_as_longlong(div_rn_fast(a, b)) == __double_as_longlong(a / b);
        }
        local += !ok;
    }
    if (local) atomicAdd(bad, local);
}

}  // namespace clv

extern "C" int clv_debug_fast_div_check(long long n, unsigned long long seed, long long *mismatches) {
    unsigned long long *d = nullptr;
    if (cudaMalloc(&d, sizeof(*d)) != cudaSuccess) return CLV_ERR_CUDA;
    cudaMemset(d, 0, sizeof(*d));
    clv::fast_div_check_kernel<<<148 * 8, 256>>>(n, seed, d);
    unsigned long long h = 0;
    const bool ok = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(d);
    if (!ok) return CLV_ERR_CUDA;
    *mismatches = (long long)h;
    return CLV_OK;
}
