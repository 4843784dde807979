// Batched FP64 GEMM on the FP64 tensor-core path (DMMA, mma.sync.m8n8k4.f64) for the element-local
// contractions of static condensation: the q-elimination products X -= Y_d (M^-1 B_d | M^-1 C_d)
// (local_ops.cpp:389-398) and the Schur complement K = J - H (E^-1 F) (local_ops.cpp:408-411), i.e.
// gemm_batch (dense_batch.cpp:101-136) at the block sizes of BASELINE configs 2-5.
//
// Why DMMA: measured on B200 (scripts/micro/fp64_peak.cu) the DFMA pipe peaks at 34 TFLOP/s and only with
// >= 512 resident threads per SM, DMMA sustains 37.2 TFLOP/s with 4 warps per SM -- the register-heavy
// tiles of a batched GEMM cannot afford high occupancy, so the tensor path is the one that reaches peak.
//
// Mapping: one CTA per (BM x BN output tile, batch item), BM = 32 WM, BN = 32 WN, one 32 x 32 warp tile
// per warp = 4 x 4 DMMA tiles (32 accumulator doubles per lane).  A (m x k) and B (k x n) are column-major
// like DenseBatch; K is swept in chunks of 16 through a two-stage cp.async pipeline.  Shared-memory
// leading dimensions are = 4 (mod 16) doubles, which makes both fragment loads (8 rows x 4 k-columns of A,
// 4 k-rows x 8 columns of B per warp) bank-conflict free.
// Accumulation order: k ascending in groups of 4 inside the tensor core (not the reference's strict
// ascending-k scalar order): results agree to rounding, the parity bar is 1e-10 relative.
// Roofline: FP64 pipe when fused chains keep operands in L2; HBM for a single product (4-6 flop/B).
#include "kernels.cuh"

namespace hdgb {

namespace {

constexpr int KC = 16;       // k-chunk per pipeline stage
constexpr int LDB = KC + 4;  // = 4 (mod 16)

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// 16-byte (VEC) or 8-byte cp.async with zero fill when !pred
template <bool VEC>
__device__ __forceinline__ void cp_async_zfill(uint32_t dst, const double* src, bool pred) {
    if (VEC) {
        const int nb = pred ? 16 : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(nb) : "memory");
    } else {
        const int nb = pred ? 8 : 0;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(nb) : "memory");
    }
}

struct GemmArgs {
    int m, n, k;
    const double* a;
    int64_t a_stride;
    const double* b;
    int64_t b_stride;
    double* c;
    int64_t c_stride;
    double alpha, beta;
    int c_colw, c_colstride;  // output column j lives at column (j / c_colw) * c_colstride + j % c_colw of C
};

template <int WM, int WN, bool VEC>
__global__ void __launch_bounds__(WM * WN * 32) gemm_dmma_kernel(GemmArgs g) {
    constexpr int BM = 32 * WM, BN = 32 * WN, NT = WM * WN * 32;
    constexpr int LDA = BM + 4;  // = 4 (mod 16)
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                  // [2][KC][LDA]
    double* Bs = smem + 2 * KC * LDA;   // [2][BN][LDB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % WM, wn = warp / WM;
    const int grp = lane >> 2, tig = lane & 3;
    const int64_t item = blockIdx.z;
    const double* A = g.a + item * g.a_stride;
    const double* B = g.b + item * g.b_stride;
    double* C = g.c + item * g.c_stride;
    const int m = g.m, n = g.n, k = g.k;
    const int row0 = blockIdx.x * BM, col0 = blockIdx.y * BN;

    auto load_stage = [&](int s, int k0) {
        double* as = As + s * KC * LDA;
        double* bs = Bs + s * BN * LDB;
        constexpr int W = VEC ? 2 : 1;
        // A chunk: KC columns of BM rows, contiguous along rows
        for (int t = tid; t < KC * (BM / W); t += NT) {
            const int p = t / (BM / W), i = (t - p * (BM / W)) * W;
            const int gi = row0 + i, gp = k0 + p;
            const bool ok = gi < m && gp < k;
            cp_async_zfill<VEC>(smem_addr(as + p * LDA + i), ok ? A + static_cast<int64_t>(gp) * m + gi : A, ok);
        }
        // B chunk: BN columns of KC rows, contiguous along k
        for (int t = tid; t < BN * (KC / W); t += NT) {
            const int j = t / (KC / W), p = (t - j * (KC / W)) * W;
            const int gj = col0 + j, gp = k0 + p;
            const bool ok = gj < n && gp < k;
            cp_async_zfill<VEC>(smem_addr(bs + j * LDB + p), ok ? B + static_cast<int64_t>(gj) * k + gp : B, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int nk = (k + KC - 1) / KC;
    load_stage(0, 0);
    for (int c = 0; c < nk; ++c) {
        const int s = c & 1;
        if (c + 1 < nk) {
            load_stage(s ^ 1, (c + 1) * KC);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const double* as = As + s * KC * LDA + wm * 32 + grp;
        const double* bs = Bs + s * BN * LDB + (wn * 32 + grp) * LDB;
#pragma unroll
        for (int kk = 0; kk < KC; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = as[(kk + tig) * LDA + i * 8];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = bs[j * 8 * LDB + kk + tig];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncthreads();
    }

    // epilogue: lane holds C[grp][2 tig], C[grp][2 tig + 1] of every 8 x 8 tile
    const double alpha = g.alpha, beta = g.beta;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gj = col0 + wn * 32 + j * 8 + 2 * tig + h;
            if (gj >= n) continue;
            const int cj = (gj / g.c_colw) * g.c_colstride + gj % g.c_colw;
            double* cc = C + static_cast<int64_t>(cj) * m;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int gi = row0 + wm * 32 + i * 8 + grp;
                if (gi >= m) continue;
                const double v = alpha * acc[i][j][h];
                cc[gi] = (beta == 0.0) ? v : v + beta * cc[gi];
            }
        }
}

template <int WM, int WN>
void launch_wmwn(hdgb_ctx* ctx, const GemmArgs& g, int64_t batch, bool vec) {
    constexpr int BM = 32 * WM, BN = 32 * WN;
    const size_t smem = (2 * KC * (BM + 4) + 2 * BN * LDB) * sizeof(double);
    auto kv = gemm_dmma_kernel<WM, WN, true>;
    auto ks = gemm_dmma_kernel<WM, WN, false>;
    static bool configured = false;
    if (!configured) {
        if (smem > 48 * 1024) {
            HDGB_CUDA(cudaFuncSetAttribute(kv, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            HDGB_CUDA(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        }
        configured = true;
    }
    int64_t done = 0;
    while (done < batch) {  // gridDim.z limit
        const int64_t nb = (batch - done) < 65535 ? (batch - done) : 65535;
        GemmArgs h = g;
        h.a += done * g.a_stride;
        h.b += done * g.b_stride;
        h.c += done * g.c_stride;
        dim3 grid(ceil_div(g.m, BM), ceil_div(g.n, BN), static_cast<unsigned>(nb));
        if (vec) kv<<<grid, WM * WN * 32, smem, ctx->stream>>>(h);
        else ks<<<grid, WM * WN * 32, smem, ctx->stream>>>(h);
        HDGB_LAUNCH_CHECK(ctx);
        done += nb;
    }
}

template <int WM>
void launch_wm(hdgb_ctx* ctx, const GemmArgs& g, int64_t batch, bool vec, int wn) {
    switch (wn) {
        case 1: launch_wmwn<WM, 1>(ctx, g, batch, vec); break;
        case 2: launch_wmwn<WM, 2>(ctx, g, batch, vec); break;
        case 3: launch_wmwn<WM, 3>(ctx, g, batch, vec); break;
        default: launch_wmwn<WM, 4>(ctx, g, batch, vec); break;
    }
}

}  // namespace

// C_b[:, colmap(j)] = alpha * A_b * B_b[:, j] + beta * C_b[:, colmap(j)], all column-major with leading
// dimensions m (A, C) and k (B).  colmap(j) = (j / c_colw) * c_colstride + j % c_colw (identity when
// c_colw >= n): lets one product scatter its columns into the (local face, component) column blocks of
// F-bar / J-bar for multi-component systems.
void launch_gemm_dmma(hdgb_ctx* ctx, int m, int n, int k, const double* a, int64_t a_stride, const double* b,
                      int64_t b_stride, double* c, int64_t c_stride, int64_t batch, double alpha, double beta,
                      int c_colw, int c_colstride) {
    if (batch <= 0 || m <= 0 || n <= 0) return;
    GemmArgs g{m, n, k, a, a_stride, b, b_stride, c, c_stride, alpha, beta, c_colw > 0 ? c_colw : n,
               c_colw > 0 ? c_colstride : n};
    // 16-byte cp.async needs even leading dimensions / strides and 16-byte aligned bases
    const bool vec = (m % 2 == 0) && (k % 2 == 0) && (a_stride % 2 == 0) && (b_stride % 2 == 0) &&
                     (reinterpret_cast<uintptr_t>(a) % 16 == 0) && (reinterpret_cast<uintptr_t>(b) % 16 == 0);
    int wm = ceil_div(m, 32), wn = ceil_div(n, 32);
    if (wm > 4) wm = 4;
    if (wn > 4) wn = 4;
    // keep CTAs at <= 12 warps: a 4 x 4 arrangement would leave one CTA per SM
    if (wm * wn > 12) { if (wn > 3) wn = 3; }
    if (wm * wn > 12) wm = 3;
    switch (wm) {
        case 1: launch_wm<1>(ctx, g, batch, vec, wn); break;
        case 2: launch_wm<2>(ctx, g, batch, vec, wn); break;
        case 3: launch_wm<3>(ctx, g, batch, vec, wn); break;
        default: launch_wm<4>(ctx, g, batch, vec, wn); break;
    }
}

}  // namespace hdgb
