// GMRES / polynomial-preconditioner vector kernels: batched Arnoldi dot
// products (V^T w for all basis vectors in ONE pass over w), fused multi-AXPY (w -= V c) with an
// optional fused norm, scaling by a device-resident scalar, and the polynomial recurrence updates.
// All reductions are two-stage with a fixed combination order => bit-reproducible run to run.
// Roofline: HBM.  multi_dot / multi_axpy stream 8*n*(nvec+1) (+8n write) bytes.
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
__global__ void __launch_bounds__(kDotThreads) multi_dot_partial_kernel(
    const double* __restrict__ V, int64_t ldv, int nvec, const double* __restrict__ w, int64_t n,
    double* __restrict__ partial, int nblocks) {
    extern __shared__ double red[];  // [nwarps][nvec]
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kDotChunk;
    double wr[kDotPerThread];
    int64_t idx[kDotPerThread];
#pragma unroll
    for (int k = 0; k < kDotPerThread; ++k) {
        idx[k] = base + k * kDotThreads + threadIdx.x;
        wr[k] = idx[k] < n ? w[idx[k]] : 0.0;
        if (idx[k] >= n) idx[k] = n - 1;  // safe address; contribution is multiplied by 0
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int nwarps = kDotThreads / 32;
    for (int j = 0; j < nvec; ++j) {
        const double* vj = V + static_cast<int64_t>(j) * ldv;
        double vals[kDotPerThread];
#pragma unroll
        for (int k = 0; k < kDotPerThread; ++k) vals[k] = __ldg(vj + idx[k]);
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

// w[i] += sign * sum_j c[j] V_j[i]; optional partial sums of w_new^2.
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
        idx[k] = base + k * kAxpyThreads + threadIdx.x;
        ok[k] = idx[k] < n;
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
    double sq = 0.0;
#pragma unroll
    for (int k = 0; k < kAxpyPerThread; ++k) {
        if (ok[k]) {
            w[idx[k]] = acc[k];
            sq = fma(acc[k], acc[k], sq);
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
    const int64_t a = nblocks * (nvec > 0 ? nvec : 1);
    return static_cast<size_t>(a > ablocks ? a : ablocks) + 16;
}

void launch_multi_dot(hdgb_ctx* ctx, const double* V, int64_t ldv, int nvec, const double* w, int64_t n,
                      double* out, double* partial, bool sqrt_last) {
    if (nvec <= 0 || n <= 0) return;
    const int nblocks = static_cast<int>((n + kDotChunk - 1) / kDotChunk);
    const size_t smem = static_cast<size_t>(kDotThreads / 32) * nvec * sizeof(double);
    multi_dot_partial_kernel<<<nblocks, kDotThreads, smem, ctx->stream>>>(V, ldv, nvec, w, n, partial, nblocks);
    HDGB_LAUNCH_CHECK(ctx);
    reduce_partials_kernel<<<nvec, 128, 0, ctx->stream>>>(partial, nblocks, out, sqrt_last ? nvec - 1 : -1);
    HDGB_LAUNCH_CHECK(ctx);
}

void launch_multi_axpy(hdgb_ctx* ctx, const double* V, int64_t ldv, int nvec, const double* c, double sign,
                       double* w, int64_t n, double* norm2_out, double* partial) {
    if (n <= 0) return;
    const int per = kAxpyThreads * kAxpyPerThread;
    const int nblocks = static_cast<int>((n + per - 1) / per);
    const size_t smem = (static_cast<size_t>(nvec) + 8) * sizeof(double);
    multi_axpy_kernel<<<nblocks, kAxpyThreads, smem, ctx->stream>>>(V, ldv, nvec, c, sign, w, n,
                                                                    norm2_out ? partial : nullptr);
    HDGB_LAUNCH_CHECK(ctx);
    if (norm2_out) {
        reduce_partials_kernel<<<1, 128, 0, ctx->stream>>>(partial, nblocks, norm2_out, -1);
        HDGB_LAUNCH_CHECK(ctx);
    }
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
