// Batched FP64 dense kernels: explicit inverses by partial-pivot LU
// (dense_batch.cpp:19-99) and batched GEMM (dense_batch.cpp:101-136).
//
// Dispatch: n <= 24 -> lu_invert_warp_kernel (below); larger blocks -> the blocked Gauss-Jordan of k_invert.cu;
// GEMMs with more than 256 output entries -> the DMMA kernels of k_gemm_dmma.cu.  The register-tiled
// Gauss-Jordan, the shared-memory LU and the FMA GEMMs below are the previous generation, kept behind
// hdgb_set_tuning switches as cross-checks for the tests.
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

// ---- register-tiled Gauss-Jordan inverse (25 <= n <= 128) --------------------------------------------
// One CTA of 16 x 16 threads per block; thread (ti, tj) keeps the T x T entries (ti + 16a, tj + 16b)
// in registers.  In-place Gauss-Jordan with the reference's partial-pivot rule and singularity
// test (dense_batch.cpp:27-36): per elimination step the pivot column and the two rows involved in
// the interchange are published through (double-buffered) shared memory -- 3 barriers per step --
// and every thread applies the rank-1 update to its tile with T^2 FMAs.  Working on the row-
// interchanged matrix yields (P A)^-1; the inverse is its column permutation, applied on write-out.
// Same 2 n^3 flops as the reference's LU + n solves, results agree to rounding.
template <int T>
__global__ void __launch_bounds__(256) lu_invert_tile_kernel(int n, int64_t batch, const double* __restrict__ a_in,
                                                             double* __restrict__ inv_out, int* flags) {
    constexpr int N = 16 * T;
    __shared__ double s_col[2][N], s_rowk[2][N], s_rowp[2][N];
    __shared__ double s_red[8];
    __shared__ int s_piv[N], s_cinv[N];
    __shared__ int s_p, s_ok;
    const int tid = threadIdx.x, ti = tid & 15, tj = tid >> 4;
    const int lane = tid & 31, warp = tid >> 5;

    for (int64_t blk = blockIdx.x; blk < batch; blk += gridDim.x) {
        const double* A = a_in + blk * n * n;
        double a[T][T];
        double amax = 0.0;
#pragma unroll
        for (int b_ = 0; b_ < T; ++b_)
#pragma unroll
            for (int a_ = 0; a_ < T; ++a_) {
                const int i = ti + 16 * a_, j = tj + 16 * b_;
                double v = (i == j) ? 1.0 : 0.0;  // identity padding outside the n x n block
                if (i < n && j < n) {
                    v = A[static_cast<size_t>(j) * n + i];
                    amax = fmax(amax, fabs(v));
                }
                a[a_][b_] = v;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if (lane == 0) s_red[warp] = amax;
        __syncthreads();
        amax = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) amax = fmax(amax, s_red[w]);
        const double tol = 1e-14 * amax;
        bool singular = false;

        for (int k = 0; k < n; ++k) {
            const int buf = k & 1;
            const int bk = k >> 4, rk = k & 15;
            // 1. publish column k
            if (tj == rk) {
#pragma unroll
                for (int a_ = 0; a_ < T; ++a_) {
                    double v = 0.0;
#pragma unroll
                    for (int b_ = 0; b_ < T; ++b_)
                        if (b_ == bk) v = a[a_][b_];
                    s_col[buf][ti + 16 * a_] = v;
                }
            }
            __syncthreads();
            // 2. pivot: first row of maximal modulus among rows >= k
            if (warp == 0) {
                double best = -1.0;
                int bi = INT_MAX;
                for (int i = k + lane; i < n; i += 32) {
                    const double v = fabs(s_col[buf][i]);
                    if (v > best) { best = v; bi = i; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
                }
                if (lane == 0) {
                    const double dkk = s_col[buf][k];
                    s_ok = (dkk == dkk) && (best > tol);
                    s_p = bi;
                    s_piv[k] = bi;
                }
            }
            __syncthreads();
            if (!s_ok) { singular = true; break; }
            const int p = s_p;
            // 3. publish rows k and p (their pre-interchange contents)
            if (ti == rk) {
#pragma unroll
                for (int b_ = 0; b_ < T; ++b_) {
                    double v = 0.0;
#pragma unroll
                    for (int a_ = 0; a_ < T; ++a_)
                        if (a_ == bk) v = a[a_][b_];
                    s_rowk[buf][tj + 16 * b_] = v;
                }
            }
            if (ti == (p & 15)) {
                const int bp = p >> 4;
#pragma unroll
                for (int b_ = 0; b_ < T; ++b_) {
                    double v = 0.0;
#pragma unroll
                    for (int a_ = 0; a_ < T; ++a_)
                        if (a_ == bp) v = a[a_][b_];
                    s_rowp[buf][tj + 16 * b_] = v;
                }
            }
            __syncthreads();
            // 4. interchange + rank-1 update of this thread's tile
            const double inv = 1.0 / s_col[buf][p];
            double rj[T];
#pragma unroll
            for (int b_ = 0; b_ < T; ++b_) rj[b_] = s_rowp[buf][tj + 16 * b_];
#pragma unroll
            for (int a_ = 0; a_ < T; ++a_) {
                const int i = ti + 16 * a_;
                if (i == k) {
#pragma unroll
                    for (int b_ = 0; b_ < T; ++b_) a[a_][b_] = (tj + 16 * b_ == k) ? inv : rj[b_] * inv;
                } else {
                    const bool was_p = (i == p);
                    const double li = (was_p ? s_col[buf][k] : s_col[buf][i]) * inv;
#pragma unroll
                    for (int b_ = 0; b_ < T; ++b_) {
                        const int j = tj + 16 * b_;
                        const double base = was_p ? s_rowk[buf][j] : a[a_][b_];
                        a[a_][b_] = (j == k) ? -li : fma(-li, rj[b_], base);
                    }
                }
            }
        }
        if (singular) {
            if (tid == 0) atomicMin(flags, static_cast<int>(blk));
        } else {
            // column permutation: inverse[:, j] = W[:, c[j]] with c = identity after the interchanges in
            // reverse order; every thread writes its entries to column cinv[its column]
            if (tid == 0) {
                for (int j = 0; j < n; ++j) s_cinv[j] = j;  // used as c[] first
                for (int k = n - 1; k >= 0; --k) {
                    const int p = s_piv[k];
                    const int t = s_cinv[k];
                    s_cinv[k] = s_cinv[p];
                    s_cinv[p] = t;
                }
                // invert c in place via s_piv as scratch
                for (int j = 0; j < n; ++j) s_piv[s_cinv[j]] = j;
            }
            __syncthreads();
            double* out = inv_out + blk * n * n;
#pragma unroll
            for (int b_ = 0; b_ < T; ++b_)
#pragma unroll
                for (int a_ = 0; a_ < T; ++a_) {
                    const int i = ti + 16 * a_, j = tj + 16 * b_;
                    if (i < n && j < n) out[static_cast<size_t>(s_piv[j]) * n + i] = a[a_][b_];
                }
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
        ensure_dynamic_smem(lu_invert_warp_kernel, smem);
        lu_invert_warp_kernel<<<ceil_div(batch, wpc), wpc * 32, smem, ctx->stream>>>(n, batch, a, inv, flags, wpc);
        HDGB_LAUNCH_CHECK(ctx);
        return;
    }
    if (tuning().use_blocked_gj) {
        launch_gj_invert_batch(ctx, n, batch, a, inv, flags);
        return;
    }
    if (n <= 128 && tuning().use_tile_lu) {
        const int64_t cap = static_cast<int64_t>(ctx->sm_count) * 8;
        const int grid = static_cast<int>(batch < cap ? batch : cap);
        if (n <= 32) lu_invert_tile_kernel<2><<<grid, 256, 0, ctx->stream>>>(n, batch, a, inv, flags);
        else if (n <= 64) lu_invert_tile_kernel<4><<<grid, 256, 0, ctx->stream>>>(n, batch, a, inv, flags);
        else if (n <= 96) lu_invert_tile_kernel<6><<<grid, 256, 0, ctx->stream>>>(n, batch, a, inv, flags);
        else lu_invert_tile_kernel<8><<<grid, 256, 0, ctx->stream>>>(n, batch, a, inv, flags);
        HDGB_LAUNCH_CHECK(ctx);
        return;
    }
    const size_t smem = per * sizeof(double);
    int threads = n * n / 4;
    threads = ((threads + 31) / 32) * 32;
    if (threads < 64) threads = 64;
    if (threads > 512) threads = 512;
    if (smem <= 200 * 1024) {
        ensure_dynamic_smem(lu_invert_cta_kernel, smem);
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
    if (!trans_a && tuning().use_dmma) {
        launch_gemm_dmma(ctx, m, n, k, a, a_stride, b, b_stride, c, c_stride, batch, alpha, beta);
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
