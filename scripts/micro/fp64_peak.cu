// Microbenchmark: FP64 DFMA pipe vs DMMA (mma.sync m8n8k4 f64) peak on one GPU.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
    double c[NACC][2];
#pragma unroll
    for (int i = 0; i < NACC; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <class F> float timeit(F f) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    f(); cudaDeviceSynchronize();
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
    const int iters = 20000;
    for (int thr : {128, 256, 512, 1024}) {
        for (int bps : {1, 2}) {
            if (thr * bps > 2048) continue;
            float ms = timeit([&] { dfma_kernel<<<sms * bps, thr>>>(out, iters, 1.0000001, 1e-9); });
            double fl = 2.0 * 16 * iters * double(thr) * sms * bps;
            printf("DFMA threads/CTA=%4d CTAs/SM=%d : %.2f TFLOP/s\n", thr, bps, fl / ms * 1e-9);
            ms = timeit([&] { dmma_kernel<8><<<sms * bps, thr>>>(out, iters, 1.0000001, 1e-9); });
            fl = 2.0 * 8 * 8 * 4 * 8 * iters * double(thr / 32) * sms * bps;
            printf("DMMA(8 acc) threads/CTA=%4d CTAs/SM=%d : %.2f TFLOP/s\n", thr, bps, fl / ms * 1e-9);
            ms = timeit([&] { dmma_kernel<16><<<sms * bps, thr>>>(out, iters / 2, 1.0000001, 1e-9); });
            fl = 2.0 * 8 * 8 * 4 * 16 * (iters / 2) * double(thr / 32) * sms * bps;
            printf("DMMA(16 acc) threads/CTA=%4d CTAs/SM=%d : %.2f TFLOP/s\n", thr, bps, fl / ms * 1e-9);
        }
    }
    return 0;
}
