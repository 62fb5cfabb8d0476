// microbench.cu -- FP64 peak of this GPU (the roofline denominator for the
// fp64 epilogue; MEASURED_PEAKS.json carries HBM and bf16 only).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o libclv_microbench.so microbench.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void dfma_loop(double *out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5) out[0] = s;   // keep the loop alive
}

extern "C" double clv_mb_fp64_tflops(int device) {
    cudaSetDevice(device);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double *out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 8, iters = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    dfma_loop<<<blocks, threads>>>(out, 256, 0.999999, 1e-7);    // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(out);
    double flops = 2.0 * 8.0 * (double)iters * threads * blocks;
    return flops / (best * 1e-3) / 1e12;
}

// Back-to-back DFMA launches for about `seconds` (so a clock sampler sees the load): returns the
// median rate over the launches.
extern "C" double clv_mb_fp64_tflops_sustained(int device, double seconds) {
    cudaSetDevice(device);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double *out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 8, iters = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    dfma_loop<<<blocks, threads>>>(out, 256, 0.999999, 1e-7);
    float ms_all[4096];
    int n = 0;
    double spent = 0.0;
    while (spent < seconds * 1e3 && n < 4096) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_all[n], e0, e1);
        spent += ms_all[n];
        ++n;
    }
    cudaFree(out);
    // median
    for (int i = 1; i < n; ++i) { float v = ms_all[i]; int j = i - 1; while (j >= 0 && ms_all[j] > v) { ms_all[j + 1] = ms_all[j]; --j; } ms_all[j + 1] = v; }
    const double med = ms_all[n / 2];
    const double flops = 2.0 * 8.0 * (double)iters * threads * blocks;
    return flops / (med * 1e-3) / 1e12;
}
