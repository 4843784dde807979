// Team GEMV: the one bandwidth kernel behind block_matvec (face_matrix.cpp:83-107, gather fused),
// apply_bj (preconditioner.cpp:48-52), the element solve of apply_asm (:86-91), compute_q
// (local_ops.cpp:367-374), recover_local (:452-460) and gemv_strided_batch (dense_batch.cpp:138-160).
//
// Mapping.  A CTA works on FPB batch items at once, each owned by a "team" of TS = RL*CG threads.
// Inside a team, lane (rl, cg) owns V consecutive rows [rl*V, rl*V+V) and the columns
// cg, cg+CG, cg+2CG, ...  One team iteration therefore reads CG consecutive columns = CG*rows
// contiguous doubles of the column-major block: fully coalesced, 128-bit per lane when V == 2.
// The gathered input slice is staged once per item in shared memory (the reference materialises it
// in an nb-times-larger global scratch, face_matrix.cpp:92-104; here it never touches HBM).
// Partial sums of the CG column groups are combined through shared memory in ascending group
// order, so results are deterministic run to run.
//
// Roofline: HBM.  Algorithmic bytes per item = 8*(rows*cols + cols + rows) (+ 4*nslots index bytes).
#include "kernels.cuh"

namespace hdgb {

namespace {

template <int V>
__device__ __forceinline__ void load_rows(const double* p, double (&v)[V]);

template <>
__device__ __forceinline__ void load_rows<1>(const double* p, double (&v)[1]) {
    v[0] = __ldg(p);
}
template <>
__device__ __forceinline__ void load_rows<2>(const double* p, double (&v)[2]) {
    // streamed exactly once: read-only path, do not allocate in L1
    double2 t;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(t.x), "=d"(t.y) : "l"(p));
    v[0] = t.x;
    v[1] = t.y;
}

template <int V>
__global__ void __launch_bounds__(1024) team_gemv_kernel(GemvArgs g, int RL, int CG, int TS, int FPB) {
    extern __shared__ double sm[];
    double* xs_all = sm;                                         // [FPB][cols]
    double* red_all = sm + static_cast<size_t>(FPB) * g.cols;    // [FPB][CG][rows]

    const int team = threadIdx.x / TS;
    const int t = threadIdx.x - team * TS;
    const int64_t b = static_cast<int64_t>(blockIdx.x) * FPB + team;
    const bool active = (team < FPB) && (b < g.batch);
    const int rows = g.rows, cols = g.cols;

    double* xs = xs_all + static_cast<size_t>(team) * cols;
    if (active) {
        if (g.idx == nullptr) {
            const double* xb = g.x + b * cols;
            for (int c = t; c < cols; c += TS) xs[c] = xb[c];
        } else {
            const int nslots = cols / g.width;
            const int64_t bi = b / g.comp;
            const int bc = static_cast<int>(b - bi * g.comp);
            const int* ib = g.idx + bi * nslots;
            for (int c = t; c < cols; c += TS) {
                const int s = c / g.width;
                const int o = c - s * g.width;
                const int src = ib[s];
                xs[c] = (src < 0) ? 0.0
                                  : g.x[(static_cast<int64_t>(src) * g.comp + bc) * g.width + o];
            }
        }
    }
    __syncthreads();

    if (active) {
        const int cg = t / RL;
        const int rl = t - cg * RL;
        double acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = 0.0;
        const double* A = g.a + (b / g.a_div) * (static_cast<int64_t>(rows) * cols) + rl * V;
        if (cg < CG) {
#pragma unroll 8
            for (int c = cg; c < cols; c += CG) {
                double av[V];
                load_rows<V>(A + static_cast<int64_t>(c) * rows, av);
                const double xv = xs[c];
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] = fma(av[v], xv, acc[v]);
            }
            double* red = red_all + (static_cast<size_t>(team) * CG + cg) * rows + rl * V;
#pragma unroll
            for (int v = 0; v < V; ++v) red[v] = acc[v];
        }
    }
    __syncthreads();

    if (active) {
        const double* red = red_all + static_cast<size_t>(team) * CG * rows;
        for (int r = t; r < rows; r += TS) {
            double s = red[r];
            for (int k = 1; k < CG; ++k) s += red[k * rows + r];
            const int64_t o = b * rows + r;
            double out = g.alpha * s;
            if (g.z != nullptr) out += g.beta * g.z[o];
            g.y[o] = out;
        }
    }
}

int env_int(const char* name, int dflt) {
    const char* s = getenv(name);
    return s ? atoi(s) : dflt;
}

}  // namespace

void launch_team_gemv(hdgb_ctx* ctx, const GemvArgs& g) {
    if (g.batch <= 0 || g.rows <= 0 || g.cols <= 0) return;
    if (tuning().use_stream && launch_stream_gemv(ctx, g)) return;
    if (g.idx && (g.width <= 0 || g.cols % g.width != 0))
        throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "team_gemv: cols not a multiple of the gather width");
    const bool vec2 = (g.rows % 2 == 0) && (reinterpret_cast<uintptr_t>(g.a) % 16 == 0);
    const int V = vec2 ? 2 : 1;
    const int RL = g.rows / V;
    if (RL > 1024) throw Failure(HDGB_ERR_UNSUPPORTED, "team_gemv: block rows exceed 2048");
    // Column groups: aim for ~iters columns per lane so each lane keeps several independent
    // loads in flight, within the 1024-thread CTA limit.
    static const int iters = env_int("HDGB_GEMV_ITERS", 8);
    static const int cta_threads = env_int("HDGB_GEMV_THREADS", 256);
    int CG = g.cols / iters;
    if (CG < 1) CG = 1;
    if (CG > 1024 / RL) CG = 1024 / RL;
    if (CG > g.cols) CG = g.cols;
    const int TS = RL * CG;
    int FPB = cta_threads / TS;
    if (FPB < 1) FPB = 1;
    if (FPB > 64) FPB = 64;
    if (static_cast<int64_t>(FPB) > g.batch) FPB = static_cast<int>(g.batch);
    size_t smem = (static_cast<size_t>(FPB) * g.cols + static_cast<size_t>(FPB) * CG * g.rows) * sizeof(double);
    while (smem > 200 * 1024 && FPB > 1) {
        FPB /= 2;
        smem = (static_cast<size_t>(FPB) * g.cols + static_cast<size_t>(FPB) * CG * g.rows) * sizeof(double);
    }
    if (smem > 200 * 1024) throw Failure(HDGB_ERR_UNSUPPORTED, "team_gemv: block too large for shared memory");
    const int threads = ((FPB * TS + 31) / 32) * 32;
    const int64_t grid = (g.batch + FPB - 1) / FPB;
    if (grid > 2147483647LL) throw Failure(HDGB_ERR_UNSUPPORTED, "team_gemv: batch too large");
    if (vec2) {
        ensure_dynamic_smem(team_gemv_kernel<2>, smem);
        team_gemv_kernel<2><<<static_cast<unsigned>(grid), threads, smem, ctx->stream>>>(g, RL, CG, TS, FPB);
    } else {
        ensure_dynamic_smem(team_gemv_kernel<1>, smem);
        team_gemv_kernel<1><<<static_cast<unsigned>(grid), threads, smem, ctx->stream>>>(g, RL, CG, TS, FPB);
    }
    HDGB_LAUNCH_CHECK(ctx);
}

// ---- small gather / scatter helpers ---------------------------------------------------------------
namespace {

__global__ void face_sum_kernel(const double* __restrict__ ze, const int* __restrict__ face_elems,
                                const int* __restrict__ face_lidx, int nf, int mpf, int n_lfe,
                                double* __restrict__ z, int sides, PolyEpi epi) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(nf) * mpf) return;
    const int f = static_cast<int>(i / mpf);
    const int r = static_cast<int>(i - static_cast<int64_t>(f) * mpf);
    double acc = 0.0;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        const int e = face_elems[2 * f + side];
        if (e < 0 || side >= sides) continue;
        const int l = face_lidx[2 * f + side];
        acc += ze[(static_cast<int64_t>(e) * n_lfe + l) * mpf + r];
    }
    if (epi.mode == PolyEpi::kNone) z[i] = acc;
    else poly_epilogue(epi, i, acc);
}

__global__ void gather_element_trace_kernel(const double* __restrict__ v, const int* __restrict__ elem_faces,
                                            int64_t total, int mpf, double* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t slot = i / mpf;  // e*n_lfe + l
    const int r = static_cast<int>(i - slot * mpf);
    out[i] = v[static_cast<int64_t>(elem_faces[slot]) * mpf + r];
}

__global__ void gather_extended_kernel(const double* __restrict__ x, const int* __restrict__ nbr,
                                       int64_t total, int mpf, double* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t slot = i / mpf;  // f*nb + s
    const int r = static_cast<int>(i - slot * mpf);
    const int g = nbr[slot];
    out[i] = g < 0 ? 0.0 : x[static_cast<int64_t>(g) * mpf + r];
}

}  // namespace

void launch_face_sum(hdgb_ctx* ctx, const double* ze, const int* face_elems, const int* face_lidx,
                     int nf, int mpf, int n_lfe, double* z, int sides, const PolyEpi* epi) {
    const int64_t total = static_cast<int64_t>(nf) * mpf;
    if (total == 0) return;
    face_sum_kernel<<<ceil_div(total, 256), 256, 0, ctx->stream>>>(ze, face_elems, face_lidx, nf, mpf, n_lfe, z, sides,
                                                                   epi ? *epi : PolyEpi());
    HDGB_LAUNCH_CHECK(ctx);
}

void launch_gather_element_trace(hdgb_ctx* ctx, const double* v, const int* elem_faces, int ne,
                                 int n_lfe, int mpf, double* out) {
    const int64_t total = static_cast<int64_t>(ne) * n_lfe * mpf;
    if (total == 0) return;
    gather_element_trace_kernel<<<ceil_div(total, 256), 256, 0, ctx->stream>>>(v, elem_faces, total, mpf, out);
    HDGB_LAUNCH_CHECK(ctx);
}

void launch_gather_extended(hdgb_ctx* ctx, const double* x, const int* nbr, int nf, int nb, int mpf,
                            double* out) {
    const int64_t total = static_cast<int64_t>(nf) * nb * mpf;
    if (total == 0) return;
    gather_extended_kernel<<<ceil_div(total, 256), 256, 0, ctx->stream>>>(x, nbr, total, mpf, out);
    HDGB_LAUNCH_CHECK(ctx);
}

}  // namespace hdgb
