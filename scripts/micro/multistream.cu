// Micro-benchmark: how fast can 148 SMs read NV column streams (Krylov basis vectors) of N doubles each?
//   mode 0: each CTA reads a contiguous row range of every column with 16-byte loads (register accumulate)
//   mode 1: bulk-TMA ring, PIECE bytes per column per tile
//   mode 2: one contiguous stream of NV*N doubles (reference point), 16-byte loads
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o multistream multistream.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n.reg .pred P1;\nLAB_WAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(256) k_direct(const double* V, int64_t ld, int nv, int64_t n, double* out) {
    // rows split evenly over CTAs; per column the CTA streams its row range
    const int64_t r0 = (n / 2) * blockIdx.x / gridDim.x * 2, r1 = (n / 2) * (blockIdx.x + 1) / gridDim.x * 2;
    double acc = 0.0;
    for (int64_t base = r0; base < r1; base += 256 * 2 * 4) {
        for (int j = 0; j < nv; ++j) {
            const double* col = V + j * ld;
            double2 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t r = base + (k * 256 + threadIdx.x) * 2;
                v[k] = r < r1 ? *reinterpret_cast<const double2*>(col + r) : make_double2(0, 0);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) acc += v[k].x + v[k].y;
        }
    }
    if (acc == 123.456) out[0] = acc;
}

__global__ void __launch_bounds__(256) k_contig(const double* V, int64_t total, double* out) {
    const int64_t r0 = (total / 2) * blockIdx.x / gridDim.x * 2, r1 = (total / 2) * (blockIdx.x + 1) / gridDim.x * 2;
    double acc = 0.0;
    for (int64_t base = r0; base < r1; base += 256 * 2 * 8) {
        double2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t r = base + (k * 256 + threadIdx.x) * 2;
            v[k] = r < r1 ? *reinterpret_cast<const double2*>(V + r) : make_double2(0, 0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y;
    }
    if (acc == 123.456) out[0] = acc;
}

// TMA ring: tile = rows x nv columns; `rows` doubles per piece
template <int ISSUE>  // 0: warp 0 issues; 1: all threads issue; 2: one lane issues everything
__global__ void __launch_bounds__(128) k_tma(const double* V, int64_t ld, int nv, int64_t n, int rows, int stages, double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    double* st0 = reinterpret_cast<double*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(st0 + (size_t)stages * nv * rows);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = n / rows;
    const int64_t t0 = ntiles * blockIdx.x / gridDim.x, t1 = ntiles * (blockIdx.x + 1) / gridDim.x;
    const int my = (int)(t1 - t0);
    if (tid == 0) { for (int s = 0; s < stages; ++s) mbar_init(full + s, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    auto issue = [&](int it) {
        const int s = it % stages;
        const int64_t row0 = (t0 + it) * rows;
        double* dst = st0 + (size_t)s * nv * rows;
        if (ISSUE == 1) {
            if (tid == 0) mbar_expect_tx(full + s, (uint32_t)(rows * 8 * nv));
            for (int j = tid; j < nv; j += 128) tma_bulk_g2s(dst + (size_t)j * rows, V + j * ld + row0, rows * 8, full + s);
        } else if (ISSUE == 2) {
            if (tid == 0) {
                mbar_expect_tx(full + s, (uint32_t)(rows * 8 * nv));
                for (int j = 0; j < nv; ++j) tma_bulk_g2s(dst + (size_t)j * rows, V + j * ld + row0, rows * 8, full + s);
            }
        } else {
            if (lane == 0) mbar_expect_tx(full + s, (uint32_t)(rows * 8 * nv));
            __syncwarp();
            for (int j = lane; j < nv; j += 32) tma_bulk_g2s(dst + (size_t)j * rows, V + j * ld + row0, rows * 8, full + s);
        }
    };
    if (warp == 0 || ISSUE == 1) for (int it = 0; it < stages && it < my; ++it) issue(it);
    double acc = 0.0;
    for (int it = 0; it < my; ++it) {
        const int s = it % stages;
        mbar_wait(full + s, (it / stages) & 1);
        const double* st = st0 + (size_t)s * nv * rows;
        for (int i = tid; i < nv * rows; i += 128 * 8) acc += st[i];   // touch a little
        __syncthreads();
        if ((warp == 0 || ISSUE == 1) && it + stages < my) issue(it + stages);
    }
    if (acc == 123.456) out[0] = acc;
}

int main(int argc, char** argv) {
    const int64_t n = 1091328;
    const int NV = 50;
    double* V; double* out;
    CK(cudaMalloc(&V, sizeof(double) * n * (NV + 1)));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(V, 0, sizeof(double) * n * (NV + 1)));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](auto fn, const char* name, double bytes) {
        for (int i = 0; i < 3; ++i) fn();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        const int reps = 20;
        for (int i = 0; i < reps; ++i) fn();
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-48s %8.1f us  %7.0f GB/s\n", name, 1e3 * ms / reps, bytes / (1e-3 * ms / reps) / 1e9);
    };
    const double bytes = 8.0 * n * NV;
    char name[128];
    for (int gmul : {1, 2, 4, 8}) {
        snprintf(name, sizeof name, "contiguous, %d CTAs/SM x 256 thr", gmul);
        timeit([&] { k_contig<<<148 * gmul, 256>>>(V, n * NV, out); }, name, bytes);
    }
    for (int gmul : {2, 4, 8}) {
        snprintf(name, sizeof name, "50 columns direct, %d CTAs/SM x 256 thr", gmul);
        timeit([&] { k_direct<<<148 * gmul, 256>>>(V, n, NV, n, out); }, name, bytes);
    }
    struct Cfg { int rows, stages, ctas; };
    for (Cfg c : {Cfg{128, 2, 2}, Cfg{128, 4, 1}, Cfg{64, 4, 2}, Cfg{256, 2, 1}, Cfg{32, 8, 2}}) {
        const size_t sm = (size_t)c.stages * NV * c.rows * 8 + 64;
        CK(cudaFuncSetAttribute(k_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        CK(cudaFuncSetAttribute(k_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        CK(cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        snprintf(name, sizeof name, "TMA %d B pieces, %d stages, %d CTAs/SM, warp0", c.rows * 8, c.stages, c.ctas);
        timeit([&] { k_tma<0><<<148 * c.ctas, 128, sm>>>(V, n, NV, n, c.rows, c.stages, out); }, name, bytes);
        snprintf(name, sizeof name, "TMA %d B pieces, %d stages, %d CTAs/SM, all thr", c.rows * 8, c.stages, c.ctas);
        timeit([&] { k_tma<1><<<148 * c.ctas, 128, sm>>>(V, n, NV, n, c.rows, c.stages, out); }, name, bytes);
        snprintf(name, sizeof name, "TMA %d B pieces, %d stages, %d CTAs/SM, 1 lane", c.rows * 8, c.stages, c.ctas);
        timeit([&] { k_tma<2><<<148 * c.ctas, 128, sm>>>(V, n, NV, n, c.rows, c.stages, out); }, name, bytes);
    }
    return 0;
}
