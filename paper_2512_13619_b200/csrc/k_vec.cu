// GMRES / polynomial-preconditioner vector kernels: batched Arnoldi dot
// products (V^T w for all basis vectors in ONE pass over w), fused multi-AXPY (w -= V c) with an
// optional fused norm, scaling by a device-resident scalar, and the polynomial recurrence updates.
// All reductions are two-stage with a fixed combination order => bit-reproducible run to run.
// Roofline: HBM.  multi_dot / multi_axpy stream 8*n*(nvec+1) (+8n write) bytes.
#include <cstdint>

#include "kernels.cuh"

namespace hdgb {

namespace {

constexpr int kDotThreads = 256;
constexpr int kDotPerThread = 8;
constexpr int kDotChunk = kDotThreads * kDotPerThread;  // elements of w per CTA

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Stage 1: partial[j * nblocks + blockIdx.x] = sum over this CTA's chunk of V_j .* w
// VEC2: 128-bit loads (a thread owns pairs of consecutive entries; needs even n, even ldv and 16-byte aligned
// pointers -- the launcher checks); otherwise 64-bit loads with the same chunking.
template <bool VEC2>
__global__ void __launch_bounds__(kDotThreads) multi_dot_partial_kernel(
    const double* __restrict__ V, int64_t ldv, int nvec, const double* __restrict__ w, int64_t n,
    double* __restrict__ partial, int nblocks) {
    extern __shared__ double red[];  // [nwarps][nvec]
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kDotChunk;
    double wr[kDotPerThread];
    int64_t idx[kDotPerThread];  // VEC2: idx[2 p] is the (even) index of pair p
#pragma unroll
    for (int k = 0; k < kDotPerThread; ++k) {
        if constexpr (VEC2) idx[k] = base + 2 * ((k >> 1) * kDotThreads + threadIdx.x) + (k & 1);
        else idx[k] = base + k * kDotThreads + threadIdx.x;
    }
    if constexpr (VEC2) {
#pragma unroll
        for (int p = 0; p < kDotPerThread / 2; ++p) {
            const bool in = idx[2 * p] < n;  // n even: the pair is inside or outside as a whole
            if (!in) idx[2 * p] = n - 2;     // safe address; contribution is multiplied by 0
            const double2 v = *reinterpret_cast<const double2*>(w + idx[2 * p]);
            wr[2 * p] = in ? v.x : 0.0;
            wr[2 * p + 1] = in ? v.y : 0.0;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kDotPerThread; ++k) {
            wr[k] = idx[k] < n ? w[idx[k]] : 0.0;
            if (idx[k] >= n) idx[k] = n - 1;  // safe address; contribution is multiplied by 0
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int nwarps = kDotThreads / 32;
    for (int j = 0; j < nvec; ++j) {
        const double* vj = V + static_cast<int64_t>(j) * ldv;
        double vals[kDotPerThread];
        if constexpr (VEC2) {
#pragma unroll
            for (int p = 0; p < kDotPerThread / 2; ++p) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(vj + idx[2 * p]));
                vals[2 * p] = v.x;
                vals[2 * p + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < kDotPerThread; ++k) vals[k] = __ldg(vj + idx[k]);
        }
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < kDotPerThread; ++k) acc = fma(vals[k], wr[k], acc);
        acc = warp_sum(acc);
        if (lane == 0) red[warp * nvec + j] = acc;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nvec; j += kDotThreads) {
        double s = red[j];
#pragma unroll
        for (int wi = 1; wi < nwarps; ++wi) s += red[wi * nvec + j];
        partial[static_cast<int64_t>(j) * nblocks + blockIdx.x] = s;
    }
}

// Stage 2: out[j] = sum_b partial[j * nblocks + b]  (one CTA per j, fixed order)
__global__ void __launch_bounds__(128) reduce_partials_kernel(const double* __restrict__ partial, int nblocks,
                                                              double* __restrict__ out, int sqrt_index) {
    __shared__ double red[4];
    const int j = blockIdx.x;
    const double* p = partial + static_cast<int64_t>(j) * nblocks;
    double acc = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += 128) acc += p[b];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = (red[0] + red[1]) + (red[2] + red[3]);
        if (j == sqrt_index) s = sqrt(s);
        out[j] = s;
    }
}

constexpr int kAxpyThreads = 256;
constexpr int kAxpyPerThread = 4;

// w[i] += sign * sum_j c[j] V_j[i]; optional partial sums of w_new^2.  VEC2: 128-bit loads / stores (even n, even ldv,
// 16-byte aligned pointers).
template <bool VEC2>
__global__ void __launch_bounds__(kAxpyThreads) multi_axpy_kernel(
    const double* __restrict__ V, int64_t ldv, int nvec, const double* __restrict__ c, double sign,
    double* __restrict__ w, int64_t n, double* __restrict__ norm_partial) {
    extern __shared__ double cs[];  // nvec coefficients, then 8 reduction slots
    for (int j = threadIdx.x; j < nvec; j += kAxpyThreads) cs[j] = sign * c[j];
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * (kAxpyThreads * kAxpyPerThread);
    double acc[kAxpyPerThread];
    int64_t idx[kAxpyPerThread];
    bool ok[kAxpyPerThread];
#pragma unroll
    for (int k = 0; k < kAxpyPerThread; ++k) {
        if constexpr (VEC2) idx[k] = base + 2 * ((k >> 1) * kAxpyThreads + threadIdx.x) + (k & 1);
        else idx[k] = base + k * kAxpyThreads + threadIdx.x;
        ok[k] = idx[k] < n;
    }
    if constexpr (VEC2) {
#pragma unroll
        for (int p = 0; p < kAxpyPerThread / 2; ++p) {
            if (!ok[2 * p]) idx[2 * p] = n - 2;  // n even: pairs are inside or outside as a whole
            const double2 v = *reinterpret_cast<const double2*>(w + idx[2 * p]);
            acc[2 * p] = v.x;
            acc[2 * p + 1] = v.y;
        }
#pragma unroll 4
        for (int j = 0; j < nvec; ++j) {
            const double* vj = V + static_cast<int64_t>(j) * ldv;
            const double cj = cs[j];
#pragma unroll
            for (int p = 0; p < kAxpyPerThread / 2; ++p) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(vj + idx[2 * p]));
                acc[2 * p] = fma(cj, v.x, acc[2 * p]);
                acc[2 * p + 1] = fma(cj, v.y, acc[2 * p + 1]);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < kAxpyPerThread; ++k) {
            if (!ok[k]) idx[k] = n - 1;
            acc[k] = w[idx[k]];
        }
#pragma unroll 4
        for (int j = 0; j < nvec; ++j) {
            const double* vj = V + static_cast<int64_t>(j) * ldv;
            const double cj = cs[j];
#pragma unroll
            for (int k = 0; k < kAxpyPerThread; ++k) acc[k] = fma(cj, __ldg(vj + idx[k]), acc[k]);
        }
    }
    double sq = 0.0;
    if constexpr (VEC2) {
#pragma unroll
        for (int p = 0; p < kAxpyPerThread / 2; ++p) {
            if (ok[2 * p]) {
                *reinterpret_cast<double2*>(w + idx[2 * p]) = make_double2(acc[2 * p], acc[2 * p + 1]);
                sq = fma(acc[2 * p], acc[2 * p], sq);
                sq = fma(acc[2 * p + 1], acc[2 * p + 1], sq);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < kAxpyPerThread; ++k) {
            if (ok[k]) {
                w[idx[k]] = acc[k];
                sq = fma(acc[k], acc[k], sq);
            }
        }
    }
    if (norm_partial != nullptr) {
        double* red = cs + nvec;
        sq = warp_sum(sq);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
#pragma unroll
            for (int wi = 0; wi < kAxpyThreads / 32; ++wi) s += red[wi];
            norm_partial[blockIdx.x] = s;
        }
    }
}

// Fused first update + second projection of CGS2 (gmres.cpp:38-50):  w -= V c ;  d = V^T w  in ONE pass over the
// Krylov basis.  The dot products of a row need only that row's updated w, so a thread that holds the basis
// entries V_j[row] in registers for the update reuses them for its share of d: V is read once instead of
// twice (8 n (nvec + 2) bytes instead of 8 n (2 nvec + 3)).  Thread = (row, quarter q): it owns the vectors
// j = q (mod 4); the four partial sums of a row meet in shared memory (one barrier per tile of 64 rows), the
// dot-product partials stay lane-wise in registers over all tiles of the persistent CTA and are reduced once.
constexpr int kFuseRows = 64;
constexpr int kFuseQ = 4;
constexpr int kFuseThreads = kFuseRows * kFuseQ;
constexpr int kFuseSlots = 16;                      // vectors per thread
constexpr int kFuseMaxVec = kFuseSlots * kFuseQ;    // 64

__global__ void __launch_bounds__(kFuseThreads) multi_axpy_dot_kernel(const double* __restrict__ V, int64_t ldv, int nvec,
                                                                      const double* __restrict__ c, double* __restrict__ w,
                                                                      int64_t n, double* __restrict__ partial) {
    __shared__ double wp[2][kFuseQ][kFuseRows];  // partial sums of V c, double-buffered over tiles
    __shared__ double red[kFuseThreads / 32][kFuseMaxVec];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = tid & (kFuseRows - 1), q = tid / kFuseRows;
    double cj[kFuseSlots], dsum[kFuseSlots];
#pragma unroll
    for (int s = 0; s < kFuseSlots; ++s) {
        const int j = q + kFuseQ * s;
        cj[s] = j < nvec ? c[j] : 0.0;
        dsum[s] = 0.0;
    }
    const int64_t tiles = (n + kFuseRows - 1) / kFuseRows;
    const int64_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
    int buf = 0;
    for (int64_t t = t0; t < t1; ++t, buf ^= 1) {
        const int64_t row = t * kFuseRows + r;
        const bool ok = row < n;
        const double* vp = V + (ok ? row : n - 1) + static_cast<int64_t>(q) * ldv;
        double v[kFuseSlots];
#pragma unroll
        for (int s = 0; s < kFuseSlots; ++s)
            v[s] = (ok && q + kFuseQ * s < nvec) ? __ldg(vp + static_cast<int64_t>(kFuseQ * s) * ldv) : 0.0;
        const double wold = (ok && q == 0) ? w[row] : 0.0;
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < kFuseSlots; ++s) acc = fma(cj[s], v[s], acc);
        wp[buf][q][r] = acc;
        __syncthreads();
        // quarter 0 owns the entry: it combines the four partial sums (fixed order), updates w and publishes it
        double wn = 0.0;
        if (q == 0) {
            const double sub = (wp[buf][0][r] + wp[buf][1][r]) + (wp[buf][2][r] + wp[buf][3][r]);
            wn = ok ? wold - sub : 0.0;
            if (ok) w[row] = wn;
            wp[buf][0][r] = wn;
        }
        __syncthreads();
        if (q != 0) wn = wp[buf][0][r];
#pragma unroll
        for (int s = 0; s < kFuseSlots; ++s) dsum[s] = fma(v[s], wn, dsum[s]);
    }
    // one reduction per CTA: rows of a quarter live in two warps (64 rows)
#pragma unroll
    for (int s = 0; s < kFuseSlots; ++s) {
        const double tot = warp_sum(dsum[s]);
        if (lane == 0) red[warp][q + kFuseQ * s] = tot;
    }
    __syncthreads();
    for (int j = tid; j < nvec; j += kFuseThreads) {
        const int qq = j % kFuseQ;
        const int w0 = qq * (kFuseRows / 32);
        double sacc = 0.0;
#pragma unroll
        for (int k = 0; k < kFuseRows / 32; ++k) sacc += red[w0 + k][j];
        partial[static_cast<int64_t>(j) * gridDim.x + blockIdx.x] = sacc;
    }
}

__global__ void scale_dev_kernel(const double* __restrict__ w, const double* __restrict__ scalar, int mode,
                                 double* __restrict__ out, int64_t n) {
    const double v = *scalar;
    double s;
    if (mode == 0) s = 1.0 / sqrt(v);
    else if (mode == 1) s = 1.0 / v;
    else s = v;
    // gmres.cpp:54-57: normalise only when the norm is positive
    if (mode != 2 && !(v > 0.0)) s = 1.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = w[i] * s;
}

__global__ void axpby_kernel(double a, const double* __restrict__ x, double b, double* __restrict__ y, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        y[i] = (b == 0.0) ? a * x[i] : a * x[i] + b * y[i];
}

__global__ void lincomb_kernel(double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                               double* __restrict__ out, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = a * x[i] + b * y[i];
}

__global__ void poly_pair_mid_kernel(double two_a, double inv, const double* __restrict__ q,
                                     const double* __restrict__ t, double* __restrict__ s,
                                     double* __restrict__ w, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double sv = two_a * q[i] - t[i];
        s[i] = sv;
        w[i] += inv * sv;
    }
}

__global__ void poly_update_kernel(PolyEpi epi, const double* __restrict__ t, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        poly_epilogue(epi, i, t[i]);
}

__global__ void check_finite_kernel(const double* __restrict__ v, int64_t n, int* flags) {
    bool bad = false;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        bad |= !isfinite(v[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags + 1, 1);
}

__global__ void fill_kernel(double* v, double value, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[i] = value;
}

int stream_grid(hdgb_ctx* ctx, int64_t n, int threads) {
    const int64_t want = (n + threads - 1) / threads;
    const int64_t cap = static_cast<int64_t>(ctx->sm_count) * 16;
    return static_cast<int>(want < cap ? (want < 1 ? 1 : want) : cap);
}

}  // namespace

size_t multi_dot_workspace_doubles(int64_t n, int nvec) {
    const int64_t nblocks = (n + kDotChunk - 1) / kDotChunk;
    const int64_t ablocks = (n + kAxpyThreads * kAxpyPerThread - 1) / (kAxpyThreads * kAxpyPerThread);
    int64_t a = nblocks * (nvec > 0 ? nvec : 1);
    const int64_t fused = 1024 * static_cast<int64_t>(nvec > 0 ? nvec : 1);  // multi_axpy_dot: at most 1024 CTAs
    if (fused > a) a = fused;
    return static_cast<size_t>(a > ablocks ? a : ablocks) + 16;
}

void launch_multi_dot(hdgb_ctx* ctx, const double* V, int64_t ldv, int nvec, const double* w, int64_t n,
                      double* out, double* partial, bool sqrt_last) {
    if (nvec <= 0 || n <= 0) return;
    const int nblocks = static_cast<int>((n + kDotChunk - 1) / kDotChunk);
    // groups of at most kGroup vectors per launch: the per-warp reduction slots (64 B per vector) stay inside the
    // default 48 KB of dynamic shared memory for any restart length (the reference accepts any, gmres.hpp:15)
    constexpr int kGroup = 512;
    for (int j0 = 0; j0 < nvec; j0 += kGroup) {
        const int nv = nvec - j0 < kGroup ? nvec - j0 : kGroup;
        const size_t smem = static_cast<size_t>(kDotThreads / 32) * nv * sizeof(double);
        const double* vg = V + static_cast<int64_t>(j0) * ldv;
        // 128-bit loads when every row start is 16-byte aligned and entries pair up
        const bool vec2 = n % 2 == 0 && ldv % 2 == 0 && n >= 2 && (reinterpret_cast<uintptr_t>(vg) | reinterpret_cast<uintptr_t>(w)) % 16 == 0;
        if (vec2) multi_dot_partial_kernel<true><<<nblocks, kDotThreads, smem, ctx->stream>>>(vg, ldv, nv, w, n, partial, nblocks);
        else multi_dot_partial_kernel<false><<<nblocks, kDotThreads, smem, ctx->stream>>>(vg, ldv, nv, w, n, partial, nblocks);
        HDGB_LAUNCH_CHECK(ctx);
        const bool last = j0 + nv == nvec;
        reduce_partials_kernel<<<nv, 128, 0, ctx->stream>>>(partial, nblocks, out + j0, (sqrt_last && last) ? nv - 1 : -1);
        HDGB_LAUNCH_CHECK(ctx);
    }
}

void launch_multi_axpy(hdgb_ctx* ctx, const double* V, int64_t ldv, int nvec, const double* c, double sign,
                       double* w, int64_t n, double* norm2_out, double* partial) {
    if (n <= 0) return;
    const int per = kAxpyThreads * kAxpyPerThread;
    const int nblocks = static_cast<int>((n + per - 1) / per);
    constexpr int kGroup = 4096;  // coefficients staged in shared memory per launch
    int j0 = 0;
    do {
        const int nv = nvec - j0 < kGroup ? nvec - j0 : kGroup;
        const bool last = j0 + nv >= nvec;
        const size_t smem = (static_cast<size_t>(nv) + 8) * sizeof(double);
        const double* vg = V + static_cast<int64_t>(j0) * ldv;
        const bool vec2 = n % 2 == 0 && ldv % 2 == 0 && n >= 2 && (reinterpret_cast<uintptr_t>(vg) | reinterpret_cast<uintptr_t>(w)) % 16 == 0;
        if (vec2) multi_axpy_kernel<true><<<nblocks, kAxpyThreads, smem, ctx->stream>>>(vg, ldv, nv, c + j0, sign, w, n, (norm2_out && last) ? partial : nullptr);
        else multi_axpy_kernel<false><<<nblocks, kAxpyThreads, smem, ctx->stream>>>(vg, ldv, nv, c + j0, sign, w, n, (norm2_out && last) ? partial : nullptr);
        HDGB_LAUNCH_CHECK(ctx);
        j0 += nv;
    } while (j0 < nvec);
    if (norm2_out) {
        reduce_partials_kernel<<<1, 128, 0, ctx->stream>>>(partial, nblocks, norm2_out, -1);
        HDGB_LAUNCH_CHECK(ctx);
    }
}

// w -= V c ; d = V^T w (both over the n owned rows).  Returns false when nvec exceeds the kernel's slots.
bool launch_multi_axpy_dot(hdgb_ctx* ctx, const double* V, int64_t ldv, int nvec, const double* c, double* w, int64_t n,
                           double* d_out, double* partial) {
    if (nvec <= 0 || n <= 0) return true;
    if (nvec > kFuseMaxVec) return false;
    const int64_t tiles = (n + kFuseRows - 1) / kFuseRows;
    int64_t grid = static_cast<int64_t>(ctx->sm_count) * 3;
    if (grid > 1024) grid = 1024;
    if (grid > tiles) grid = tiles;
    const size_t smem = 0;
    multi_axpy_dot_kernel<<<static_cast<unsigned>(grid), kFuseThreads, smem, ctx->stream>>>(V, ldv, nvec, c, w, n, partial);
    HDGB_LAUNCH_CHECK(ctx);
    reduce_partials_kernel<<<nvec, 128, 0, ctx->stream>>>(partial, static_cast<int>(grid), d_out, -1);
    HDGB_LAUNCH_CHECK(ctx);
    return true;
}

void launch_sumsq(hdgb_ctx* ctx, const double* v, int64_t n, double* out, double* partial) {
    launch_multi_dot(ctx, v, 0, 1, v, n, out, partial, false);
}

void launch_scale_dev(hdgb_ctx* ctx, const double* w, const double* dev_scalar, int mode, double* out, int64_t n) {
    if (n <= 0) return;
    scale_dev_kernel<<<stream_grid(ctx, n, 256), 256, 0, ctx->stream>>>(w, dev_scalar, mode, out, n);
    HDGB_LAUNCH_CHECK(ctx);
}

void launch_axpby(hdgb_ctx* ctx, double a, const double* x, double b, double* y, int64_t n) {
    if (n <= 0) return;
    axpby_kernel<<<stream_grid(ctx, n, 256), 256, 0, ctx->stream>>>(a, x, b, y, n);
    HDGB_LAUNCH_CHECK(ctx);
}

void launch_lincomb(hdgb_ctx* ctx, double a, const double* x, double b, const double* y, double* out, int64_t n) {
    if (n <= 0) return;
    lincomb_kernel<<<stream_grid(ctx, n, 256), 256, 0, ctx->stream>>>(a, x, b, y, out, n);
    HDGB_LAUNCH_CHECK(ctx);
}

void launch_poly_pair_mid(hdgb_ctx* ctx, double two_a, double inv, const double* q, const double* t,
                          double* s, double* w, int64_t n) {
    if (n <= 0) return;
    poly_pair_mid_kernel<<<stream_grid(ctx, n, 256), 256, 0, ctx->stream>>>(two_a, inv, q, t, s, w, n);
    HDGB_LAUNCH_CHECK(ctx);
}

void launch_poly_update(hdgb_ctx* ctx, const PolyEpi& epi, const double* t, int64_t n) {
    if (n <= 0) return;
    poly_update_kernel<<<stream_grid(ctx, n, 256), 256, 0, ctx->stream>>>(epi, t, n);
    HDGB_LAUNCH_CHECK(ctx);
}

void launch_check_finite(hdgb_ctx* ctx, const double* v, int64_t n, int* flags) {
    if (n <= 0) return;
    check_finite_kernel<<<stream_grid(ctx, n, 256), 256, 0, ctx->stream>>>(v, n, flags);
    HDGB_LAUNCH_CHECK(ctx);
}

void launch_fill(hdgb_ctx* ctx, double* v, double value, int64_t n) {
    if (n <= 0) return;
    fill_kernel<<<stream_grid(ctx, n, 256), 256, 0, ctx->stream>>>(v, value, n);
    HDGB_LAUNCH_CHECK(ctx);
}

}  // namespace hdgb
