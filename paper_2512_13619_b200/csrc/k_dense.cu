// Batched FP64 dense kernels: explicit inverses by partial-pivot LU
// (dense_batch.cpp:19-99) and batched GEMM (dense_batch.cpp:101-136).
//
// lu_invert: one block per warp (n <= 24) or per CTA (shared-memory resident up to n = 104;
// larger blocks fall back to a global-memory workspace).  The factorisation follows the
// reference step for step -- same pivot rule (first row of maximal modulus), same singularity
// test (pivot <= 1e-14 * max|A|), column scaling by the reciprocal pivot, right-looking rank-1
// updates -- so that L and U agree with the reference to rounding (FMA contraction only).  The
// n unit-vector solves are done for all columns at once as right-looking triangular sweeps over
// the n x n right-hand side (identical arithmetic per entry for the forward sweep; the backward
// sweep accumulates in descending instead of ascending order).
// Roofline: FP64 pipe (2n^3 flops per block), not HBM.
#include <climits>

#include "kernels.cuh"

namespace hdgb {

namespace {

template <bool WARP>
__device__ __forceinline__ void team_sync() {
    if (WARP) __syncwarp();
    else __syncthreads();
}

// Inverts one n x n column-major block.  lu: n*n work array, x: n*ldx work array (ldx >= n) that
// receives the inverse column-major with leading dimension ldx, scratch: >= 2*32 doubles + ints.
// Returns false (uniformly across the team) when the block is singular.
template <bool WARP>
__device__ bool invert_block_team(const double* __restrict__ a, double* lu, double* x, int ldx, int n,
                                  int tid, int nthreads, double* red_val, int* red_idx, int* piv) {
    const int nn = n * n;
    // max-norm of the block
    double amax = 0.0;
    for (int i = tid; i < nn; i += nthreads) {
        const double v = a[i];
        lu[i] = v;
        amax = fmax(amax, fabs(v));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (!WARP) {
        if ((tid & 31) == 0) red_val[tid >> 5] = amax;
        __syncthreads();
        const int nw = (nthreads + 31) >> 5;
        amax = 0.0;
        for (int wi = 0; wi < nw; ++wi) amax = fmax(amax, red_val[wi]);
        __syncthreads();
    } else {
        __syncwarp();
    }
    const double tol = 1e-14 * amax;

    for (int k = 0; k < n; ++k) {
        // pivot search: first row index of maximal |lu(i,k)|, i >= k (dense_batch.cpp:27-36).
        // A NaN on the diagonal makes the reference's comparison chain fail -> singular.
        const double dkk = lu[k * n + k];
        if (dkk != dkk) return false;
        double best = -1.0;
        int bi = INT_MAX;
        for (int i = k + tid; i < n; i += nthreads) {
            const double v = fabs(lu[k * n + i]);
            if (v > best) {
                best = v;
                bi = i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) {
                best = ov;
                bi = oi;
            }
        }
        if (!WARP) {
            if ((tid & 31) == 0) { red_val[tid >> 5] = best; red_idx[tid >> 5] = bi; }
            __syncthreads();
            const int nw = (nthreads + 31) >> 5;
            best = red_val[0];
            bi = red_idx[0];
            for (int wi = 1; wi < nw; ++wi) {
                const double ov = red_val[wi];
                const int oi = red_idx[wi];
                if (ov > best || (ov == best && oi < bi)) {
                    best = ov;
                    bi = oi;
                }
            }
            __syncthreads();
        }
        if (!(best > tol)) return false;
        const int p = bi;
        if (tid == 0) piv[k] = p;
        if (p != k) {
            for (int c = tid; c < n; c += nthreads) {
                const double t = lu[c * n + k];
                lu[c * n + k] = lu[c * n + p];
                lu[c * n + p] = t;
            }
        }
        team_sync<WARP>();
        const double d = 1.0 / lu[k * n + k];
        for (int i = k + 1 + tid; i < n; i += nthreads) lu[k * n + i] *= d;
        team_sync<WARP>();
        const int rem = n - k - 1;
        for (int t = tid; t < rem * rem; t += nthreads) {
            const int c = k + 1 + t / rem;
            const int i = k + 1 + t % rem;
            lu[c * n + i] -= lu[k * n + i] * lu[c * n + k];
        }
        team_sync<WARP>();
    }

    // Right-hand sides: the identity with the row interchanges applied (P e_col for every col).
    for (int t = tid; t < n * n; t += nthreads) {
        const int c = t / n, i = t % n;
        x[c * ldx + i] = (i == c) ? 1.0 : 0.0;
    }
    team_sync<WARP>();
    // Row swaps act on whole rows of X; apply them in order, one thread per column.
    for (int c = tid; c < n; c += nthreads) {
        double* xc = x + c * ldx;
        for (int k = 0; k < n; ++k) {
            const int p = piv[k];
            if (p != k) {
                const double t = xc[k];
                xc[k] = xc[p];
                xc[p] = t;
            }
        }
    }
    team_sync<WARP>();
    // Forward sweep (unit lower triangle).
    for (int k = 0; k < n - 1; ++k) {
        const int rem = n - k - 1;
        for (int t = tid; t < rem * n; t += nthreads) {
            const int c = t / rem;
            const int i = k + 1 + t % rem;
            x[c * ldx + i] -= lu[k * n + i] * x[c * ldx + k];
        }
        team_sync<WARP>();
    }
    // Backward sweep (upper triangle).
    for (int k = n - 1; k >= 0; --k) {
        const double dk = lu[k * n + k];
        for (int c = tid; c < n; c += nthreads) x[c * ldx + k] = x[c * ldx + k] / dk;
        team_sync<WARP>();
        for (int t = tid; t < k * n; t += nthreads) {
            const int c = t / k;
            const int i = t % k;
            x[c * ldx + i] -= lu[k * n + i] * x[c * ldx + k];
        }
        team_sync<WARP>();
    }
    return true;
}

// One block per warp, all work arrays in shared memory.
__global__ void lu_invert_warp_kernel(int n, int64_t batch, const double* __restrict__ a,
                                      double* __restrict__ inv, int* flags, int warps_per_cta) {
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ldx = n | 1;
    const size_t per = static_cast<size_t>(n) * n + static_cast<size_t>(n) * ldx + ((n + 1) / 2 + 1);
    double* lu = sm + warp * per;
    double* x = lu + n * n;
    int* piv = reinterpret_cast<int*>(x + n * ldx);
    const int64_t b = static_cast<int64_t>(blockIdx.x) * warps_per_cta + warp;
    if (b >= batch) return;
    const bool ok = invert_block_team<true>(a + b * n * n, lu, x, ldx, n, lane, 32, nullptr, nullptr, piv);
    if (!ok) {
        if (lane == 0) atomicMin(flags, static_cast<int>(b));
        return;
    }
    double* out = inv + b * n * n;
    for (int t = lane; t < n * n; t += 32) out[t] = x[(t / n) * ldx + (t % n)];
}

// One block per CTA; lu and x either in shared memory or in a global workspace.
__global__ void lu_invert_cta_kernel(int n, int64_t batch, const double* __restrict__ a,
                                     double* __restrict__ inv, int* flags, double* gwork) {
    extern __shared__ double sm[];
    __shared__ double red_val[32];
    __shared__ int red_idx[32];
    const int ldx = n | 1;
    for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
        double *lu, *x;
        int* piv;
        if (gwork == nullptr) {
            lu = sm;
            x = lu + static_cast<size_t>(n) * n;
            piv = reinterpret_cast<int*>(x + static_cast<size_t>(n) * ldx);
        } else {
            double* base = gwork + static_cast<size_t>(blockIdx.x) * (static_cast<size_t>(n) * n + static_cast<size_t>(n) * ldx);
            lu = base;
            x = base + static_cast<size_t>(n) * n;
            piv = reinterpret_cast<int*>(sm);
        }
        const bool ok = invert_block_team<false>(a + b * n * n, lu, x, ldx, n, threadIdx.x, blockDim.x,
                                                 red_val, red_idx, piv);
        if (!ok) {
            if (threadIdx.x == 0) atomicMin(flags, static_cast<int>(b));
        } else {
            double* out = inv + b * n * n;
            for (int t = threadIdx.x; t < n * n; t += blockDim.x) out[t] = x[(t / n) * ldx + (t % n)];
        }
        __syncthreads();
    }
}

// ---- GEMM ----------------------------------------------------------------------------------------
// Small blocks: one thread per output entry, several batch items per CTA; operands stream through
// L1.  Ascending-k accumulation like the reference.
__global__ void gemm_small_kernel(int m, int n, int k, const double* __restrict__ a, int64_t a_stride,
                                  bool trans_a, const double* __restrict__ b, int64_t b_stride,
                                  double* __restrict__ c, int64_t c_stride, int64_t batch, double alpha,
                                  double beta, int items_per_cta) {
    const int mn = m * n;
    const int local = threadIdx.x / mn;
    const int e = threadIdx.x - local * mn;
    const int64_t item = static_cast<int64_t>(blockIdx.x) * items_per_cta + local;
    if (local >= items_per_cta || item >= batch) return;
    const int j = e / m, i = e - j * m;
    const double* A = a + item * a_stride;
    const double* B = b + item * b_stride + static_cast<int64_t>(j) * k;
    double acc = 0.0;
    if (trans_a) {
        const double* ai = A + static_cast<int64_t>(i) * k;
        for (int p = 0; p < k; ++p) acc = fma(ai[p], B[p], acc);
    } else {
        for (int p = 0; p < k; ++p) acc = fma(A[static_cast<int64_t>(p) * m + i], B[p], acc);
    }
    double* C = c + item * c_stride + static_cast<int64_t>(j) * m + i;
    *C = (beta == 0.0) ? alpha * acc : alpha * acc + beta * (*C);
}

// Larger blocks: BM x BN output tile per CTA, TM x TN register micro-tile per thread, BK-deep
// shared-memory panels.
template <int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN)) gemm_tiled_kernel(
    int m, int n, int k, const double* __restrict__ a, int64_t a_stride, bool trans_a,
    const double* __restrict__ b, int64_t b_stride, double* __restrict__ c, int64_t c_stride,
    double alpha, double beta) {
    __shared__ double As[BK][BM + 1];
    __shared__ double Bs[BK][BN + 1];
    constexpr int NT = (BM / TM) * (BN / TN);
    const int64_t item = blockIdx.z;
    const double* A = a + item * a_stride;
    const double* B = b + item * b_stride;
    double* C = c + item * c_stride;
    const int row0 = blockIdx.x * BM, col0 = blockIdx.y * BN;
    const int tx = threadIdx.x % (BM / TM), ty = threadIdx.x / (BM / TM);
    double acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;

    for (int k0 = 0; k0 < k; k0 += BK) {
        for (int t = threadIdx.x; t < BM * BK; t += NT) {
            int i, p;
            if (trans_a) { p = t % BK; i = t / BK; } else { i = t % BM; p = t / BM; }
            const int gi = row0 + i, gp = k0 + p;
            double v = 0.0;
            if (gi < m && gp < k) v = trans_a ? A[static_cast<int64_t>(gi) * k + gp] : A[static_cast<int64_t>(gp) * m + gi];
            As[p][i] = v;
        }
        for (int t = threadIdx.x; t < BN * BK; t += NT) {
            const int p = t % BK, j = t / BK;
            const int gj = col0 + j, gp = k0 + p;
            Bs[p][j] = (gj < n && gp < k) ? B[static_cast<int64_t>(gj) * k + gp] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int p = 0; p < BK; ++p) {
            double av[TM], bv[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) av[i] = As[p][tx + i * (BM / TM)];
#pragma unroll
            for (int j = 0; j < TN; ++j) bv[j] = Bs[p][ty + j * (BN / TN)];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < TN; ++j) {
        const int gj = col0 + ty + j * (BN / TN);
        if (gj >= n) continue;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int gi = row0 + tx + i * (BM / TM);
            if (gi >= m) continue;
            double* p = C + static_cast<int64_t>(gj) * m + gi;
            *p = (beta == 0.0) ? alpha * acc[i][j] : alpha * acc[i][j] + beta * (*p);
        }
    }
}

}  // namespace

void launch_lu_invert_batch(hdgb_ctx* ctx, int n, int64_t batch, const double* a, double* inv, int* flags) {
    if (batch <= 0) return;
    if (n < 1) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "lu_invert_batch requires n >= 1");
    const int ldx = n | 1;
    const size_t per = static_cast<size_t>(n) * n + static_cast<size_t>(n) * ldx + ((n + 1) / 2 + 1);
    if (n <= 24) {
        const int wpc = 4;
        const size_t smem = per * wpc * sizeof(double);
        if (smem > 48 * 1024)
            HDGB_CUDA(cudaFuncSetAttribute(lu_invert_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        lu_invert_warp_kernel<<<ceil_div(batch, wpc), wpc * 32, smem, ctx->stream>>>(n, batch, a, inv, flags, wpc);
        HDGB_LAUNCH_CHECK(ctx);
        return;
    }
    const size_t smem = per * sizeof(double);
    int threads = n * n / 4;
    threads = ((threads + 31) / 32) * 32;
    if (threads < 64) threads = 64;
    if (threads > 512) threads = 512;
    if (smem <= 200 * 1024) {
        if (smem > 48 * 1024)
            HDGB_CUDA(cudaFuncSetAttribute(lu_invert_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int64_t grid = batch < (1 << 20) ? batch : (1 << 20);
        lu_invert_cta_kernel<<<static_cast<unsigned>(grid), threads, smem, ctx->stream>>>(n, batch, a, inv, flags, nullptr);
        HDGB_LAUNCH_CHECK(ctx);
    } else {
        // Global-memory workspace path for very large blocks (n > 104): correct, not fast.
        const int grid = static_cast<int>(batch < 2 * ctx->sm_count ? batch : 2 * ctx->sm_count);
        DevBuf<double> work(static_cast<size_t>(grid) * (static_cast<size_t>(n) * n + static_cast<size_t>(n) * ldx));
        const size_t psm = (static_cast<size_t>(n) + 2) * sizeof(int);
        lu_invert_cta_kernel<<<grid, 512, psm, ctx->stream>>>(n, batch, a, inv, flags, work.p);
        HDGB_LAUNCH_CHECK(ctx);
        HDGB_CUDA(cudaStreamSynchronize(ctx->stream));  // workspace lifetime
    }
}

void launch_gemm_batch(hdgb_ctx* ctx, int m, int n, int k, const double* a, int64_t a_stride, bool trans_a,
                       const double* b, int64_t b_stride, double* c, int64_t c_stride, int64_t batch,
                       double alpha, double beta) {
    if (batch <= 0 || m <= 0 || n <= 0) return;
    if (m * n <= 256) {
        int items = 256 / (m * n);
        if (items < 1) items = 1;
        const int threads = ((items * m * n + 31) / 32) * 32;
        gemm_small_kernel<<<ceil_div(batch, items), threads, 0, ctx->stream>>>(
            m, n, k, a, a_stride, trans_a, b, b_stride, c, c_stride, batch, alpha, beta, items);
        HDGB_LAUNCH_CHECK(ctx);
        return;
    }
    int64_t done = 0;
    while (done < batch) {  // gridDim.z limit
        const int64_t nb = (batch - done) < 65535 ? (batch - done) : 65535;
        if (m > 32 && n > 32) {
            dim3 grid(ceil_div(m, 64), ceil_div(n, 64), static_cast<unsigned>(nb));
            gemm_tiled_kernel<64, 64, 16, 4, 4><<<grid, 256, 0, ctx->stream>>>(
                m, n, k, a + done * a_stride, a_stride, trans_a, b + done * b_stride, b_stride,
                c + done * c_stride, c_stride, alpha, beta);
        } else {
            dim3 grid(ceil_div(m, 32), ceil_div(n, 32), static_cast<unsigned>(nb));
            gemm_tiled_kernel<32, 32, 16, 2, 2><<<grid, 256, 0, ctx->stream>>>(
                m, n, k, a + done * a_stride, a_stride, trans_a, b + done * b_stride, b_stride,
                c + done * c_stride, c_stride, alpha, beta);
        }
        HDGB_LAUNCH_CHECK(ctx);
        done += nb;
    }
}

}  // namespace hdgb
