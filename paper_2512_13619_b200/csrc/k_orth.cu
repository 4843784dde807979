// Classical Gram-Schmidt with one re-orthogonalisation (orthogonalize, gmres.cpp:28-59) as THREE streaming
// passes over the Krylov basis instead of four:
//     pass A   c = V^T w
//     pass B   w -= V c ;  d = V^T w            (first update and second projection fused)
//     pass C   w -= V d ;  ||w||^2              (second update and the norm fused)
// The reference reads the basis four times per Arnoldi step (dot, update, dot, update); a row of pass B needs
// only that row's updated entry for its share of d, so the basis tile that produced the update is reused for
// the projection while it is still in shared memory.  Algorithmic bytes per step at Krylov index j:
// 8 n (3 j + 7) instead of the reference's 8 n (4 j + 6).
//
// One kernel template serves the three passes.  A persistent grid (one CTA per SM, a balanced contiguous range of
// 256-row tiles each) pulls [tile rows] x [nvec basis columns + w] through a ring of shared-memory stages with 1D
// bulk TMA copies -- one 2 KB copy per column and tile, completion counted on the stage's mbarrier -- issued by a
// dedicated PRODUCER warp that waits on the stage's "empty" mbarrier; eight CONSUMER warps do the arithmetic.
// (Measured on B200, scripts/micro/multistream.cu: an SM retires one bulk copy per ~60 cycles however many lanes
// issue them, so 1 KB pieces cap the stream at ~5 TB/s and issuing from a computing warp serialises with its
// arithmetic; 2 KB pieces from a warp that does nothing else reach 6.7 TB/s.  The round-1 fused kernel held 16
// basis entries per thread in registers instead and was latency bound.)
//   update:  consumer thread = row; w_new = w - sum_j c_j V_j[row] in ascending j (the reference's order, FMA-contracted);
//   project: warp = column class (j mod 8), lane = four row pairs (128-bit LDS); lane-wise partial sums stay in
//            registers over all tiles of the CTA and are combined ONCE by a fixed shuffle tree;
//   the per-CTA partials meet in global memory and the last CTA to finish (ticket counter) adds them in CTA order:
//   results are bit-reproducible run to run and no second launch is needed for the reduction.
// Roofline: HBM.
#include "kernels.cuh"
#include "tma.cuh"

namespace hdgb {

namespace {

constexpr int kRows = 256;                 // rows per tile == consumer threads per CTA
constexpr int kWarps = kRows / 32;         // consumer warps
constexpr int kThreads = kRows + 32;       // + the producer warp
constexpr int kColsPerWarp = kOrthMaxVec / kWarps;
constexpr size_t kStageBudget = 208 * 1024;
constexpr int kMaxStages = 32;
constexpr size_t kInFlightTarget = 144 * 1024;  // bytes of stages worth keeping in flight per SM

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kRows) : "memory"); }

struct OrthArgs {
    const double* V;
    int64_t ldv;
    int nvec;
    double* w;
    int64_t n;
    const double* coef;   // update coefficients (device, nvec), modes with an update
    double* out;          // projections (nvec) and/or scalars, see the modes
    double* partial;      // [n_out][grid]
    unsigned* counter;    // ticket of the last-CTA reduction (zero on entry, zeroed again on exit)
    int stages;
    int evict_first;      // basis columns copied with an L2 evict-first hint (w and the newest vectors stay cached between passes)
};

// MODE 0: out[0..nvec) = V^T w
// MODE 1: w -= V coef ; out[0..nvec) = V^T w ; out[nvec] = ||w||^2
// MODE 2: w -= V coef ; out[0] = ||w||^2
// MODE 3: w = (w - V coef) * s with s = 1 / sqrt(t), t = coef[nvec] - sum_j coef[j]^2 (Pythagoras: the norm of the
//         twice-projected vector from quantities that were already reduced; t <= 0 leaves w unscaled); out[0] = max(t, 0)
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) cgs_pass_kernel(OrthArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr bool kUpdate = MODE != 0, kProject = MODE <= 1, kNorm = MODE == 1 || MODE == 2;
    const int nvec = a.nvec, ncol = nvec + 1;  // column nvec of a stage is the w tile
    double* stage0 = reinterpret_cast<double*>(smem_raw);
    double* wsm = stage0 + static_cast<size_t>(a.stages) * ncol * kRows;  // updated w tile
    double* csm = wsm + kRows;                                              // coefficients
    double* red = csm + kOrthMaxVec + 2;                                    // [kWarps] norm partials
    uint64_t* full = reinterpret_cast<uint64_t*>(red + kWarps);
    uint64_t* empty = full + kMaxStages;
    __shared__ int s_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (a.n + kRows - 1) / kRows;
    const int64_t t0 = ntiles * blockIdx.x / gridDim.x, t1 = ntiles * (blockIdx.x + 1) / gridDim.x;
    const int my_tiles = static_cast<int>(t1 - t0);

    if (tid == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kWarps * 32);  // every consumer thread releases a stage for itself (tma.cuh)
        }
        mbar_fence_init();
    }
    double scale = 1.0;
    if constexpr (kUpdate) {
        for (int j = tid; j < nvec; j += kThreads) csm[j] = a.coef[j];
        if constexpr (MODE == 3) {
            // every CTA (and every rank) forms the same scale from the same reduced numbers in the same order
            double t = a.coef[nvec];
            for (int j = 0; j < nvec; ++j) t -= a.coef[j] * a.coef[j];
            if (t > 0.0) scale = 1.0 / sqrt(t);
            if (blockIdx.x == 0 && tid == 0) a.out[0] = t > 0.0 ? t : 0.0;
        }
    }
    __syncthreads();

    if (warp == kWarps) {
        // ---- producer warp: one bulk copy per column (w last) into the stage, as soon as the consumers freed it ----
        const uint64_t l2pol = a.evict_first ? l2_policy_evict_first() : 0;
        for (int it = 0; it < my_tiles; ++it) {
            const int s = it % a.stages, use = it / a.stages;
            if (use > 0) mbar_wait(empty + s, static_cast<uint32_t>((use - 1) & 1));
            const int64_t row0 = (t0 + it) * kRows;
            const int64_t left = a.n - row0;
            const uint32_t bytes = static_cast<uint32_t>((left < kRows ? left : kRows) * sizeof(double));
            double* dst = stage0 + static_cast<size_t>(s) * ncol * kRows;
            if (lane == 0) mbar_expect_tx(full + s, bytes * ncol);
            __syncwarp();
            for (int j = lane; j < ncol; j += 32) {
                const double* src = j < nvec ? a.V + static_cast<int64_t>(j) * a.ldv + row0 : a.w + row0;
                if (a.evict_first && j < nvec) tma_bulk_g2s_hint(dst + static_cast<size_t>(j) * kRows, src, bytes, full + s, l2pol);
                else tma_bulk_g2s(dst + static_cast<size_t>(j) * kRows, src, bytes, full + s);
            }
        }
    } else {
        // ---- consumer warps ----
        double acc[kColsPerWarp];
#pragma unroll
        for (int k = 0; k < kColsPerWarp; ++k) acc[k] = 0.0;
        double nrm = 0.0;
        for (int it = 0; it < my_tiles; ++it) {
            const int s = it % a.stages;
            const int64_t row0 = (t0 + it) * kRows;
            const int valid = static_cast<int>((a.n - row0) < kRows ? (a.n - row0) : kRows);
            const double* st = stage0 + static_cast<size_t>(s) * ncol * kRows;
            mbar_wait(full + s, static_cast<uint32_t>((it / a.stages) & 1));
            const double* wt = st + static_cast<size_t>(nvec) * kRows;
            if constexpr (kUpdate) {
                if (tid < valid) {
                    double wn = wt[tid];
#pragma unroll 8
                    for (int j = 0; j < nvec; ++j) wn = fma(-csm[j], st[static_cast<size_t>(j) * kRows + tid], wn);
                    if constexpr (kNorm) nrm = fma(wn, wn, nrm);
                    if constexpr (MODE == 3) wn *= scale;
                    a.w[row0 + tid] = wn;
                    if constexpr (kProject) wsm[tid] = wn;
                }
                if constexpr (kProject) {
                    consumer_sync();
                    wt = wsm;
                }
            }
            if constexpr (kProject) {
                // lane owns the row pairs {2 lane + 64 i, 2 lane + 64 i + 1}, i < 4 (valid is even)
                double2 wv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    wv[i] = (2 * lane + 64 * i < valid) ? *reinterpret_cast<const double2*>(wt + 2 * lane + 64 * i) : make_double2(0.0, 0.0);
#pragma unroll
                for (int k = 0; k < kColsPerWarp; ++k) {
                    const int j = warp + kWarps * k;
                    if (j < nvec) {
                        const double* col = st + static_cast<size_t>(j) * kRows + 2 * lane;
                        double t = acc[k];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            if (valid == kRows || 2 * lane + 64 * i < valid) {
                                const double2 v = *reinterpret_cast<const double2*>(col + 64 * i);
                                t = fma(v.x, wv[i].x, t);
                                t = fma(v.y, wv[i].y, t);
                            }
                        }
                        acc[k] = t;
                    }
                }
                if constexpr (kUpdate) consumer_sync();  // wsm is rewritten by the next tile's update
            }
            ring_release_all(empty + s);  // this thread is done with stage s (reads completed: see tma.cuh)
        }
        // ---- per-CTA partials ----
        const int grid = gridDim.x;
        if constexpr (kProject) {
#pragma unroll
            for (int k = 0; k < kColsPerWarp; ++k) {
                const int j = warp + kWarps * k;
                if (j < nvec) {
                    const double t = warp_sum(acc[k]);
                    if (lane == 0) a.partial[static_cast<int64_t>(j) * grid + blockIdx.x] = t;
                }
            }
        }
        if constexpr (kNorm) {
            const double t = warp_sum(nrm);
            if (lane == 0) red[warp] = t;
            consumer_sync();
            if (tid == 0) {
                double sum = 0.0;
#pragma unroll
                for (int i = 0; i < kWarps; ++i) sum += red[i];
                a.partial[static_cast<int64_t>(kProject ? nvec : 0) * grid + blockIdx.x] = sum;
            }
        }
    }
    constexpr int kExtra = kNorm ? 1 : 0;
    const int n_out = (kProject ? nvec : 0) + kExtra;
    if (n_out == 0) return;
    // ---- the last CTA to arrive adds the partials in CTA order (fixed order: deterministic) ----
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1) ? 1 : 0;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int grid = gridDim.x;
    for (int j = warp; j < n_out; j += kThreads / 32) {
        const double* p = a.partial + static_cast<int64_t>(j) * grid;
        double t = 0.0;
        for (int b = lane; b < grid; b += 32) t += __ldcg(p + b);
        t = warp_sum(t);
        if (lane == 0) a.out[j] = t;
    }
    if (tid == 0) *a.counter = 0u;
}

template <int MODE>
void launch_mode(hdgb_ctx* ctx, const OrthArgs& a0) {
    OrthArgs a = a0;
    const size_t col_bytes = static_cast<size_t>(a.nvec + 1) * kRows * sizeof(double);
    int stages = static_cast<int>(kStageBudget / col_bytes);
    const int want = static_cast<int>((kInFlightTarget + col_bytes - 1) / col_bytes) + 1;  // + the stage being consumed
    if (stages > want) stages = want;
    if (stages > kMaxStages) stages = kMaxStages;
    const int64_t ntiles = (a.n + kRows - 1) / kRows;
    int64_t grid = ctx->sm_count;
    if (grid > ntiles) grid = ntiles;
    const int64_t per = (ntiles + grid - 1) / grid;
    if (stages > per) stages = static_cast<int>(per < 1 ? 1 : per);
    a.stages = stages;
    a.evict_first = tuning().cgs_evict_first;
    const size_t smem = stages * col_bytes + (kRows + kOrthMaxVec + 2 + kWarps) * sizeof(double) + 2 * kMaxStages * sizeof(uint64_t);
    auto kern = cgs_pass_kernel<MODE>;
    ensure_dynamic_smem(kern, smem);
    kern<<<static_cast<unsigned>(grid), kThreads, smem, ctx->stream>>>(a);
    HDGB_LAUNCH_CHECK(ctx);
}

}  // namespace

size_t cgs_workspace_doubles(hdgb_ctx* ctx) {
    // partial[(kOrthMaxVec + 1)][grid] + the ticket word
    return static_cast<size_t>(kOrthMaxVec + 1) * ctx->sm_count + 2;
}

bool cgs_pass_supported(const double* V, int64_t ldv, int nvec, const double* w, int64_t n) {
    // two stages of (nvec + 1) 2 KB columns must fit next to each other in shared memory
    if (nvec < 1 || nvec > kOrthMaxVec || static_cast<size_t>(nvec + 1) * kRows * sizeof(double) * 2 > kStageBudget) return false;
    if (n < 8 * kRows) return false;
    // bulk TMA: 16-byte aligned sources and sizes
    if ((ldv & 1) || (n & 1)) return false;
    if ((reinterpret_cast<uintptr_t>(V) & 15) || (reinterpret_cast<uintptr_t>(w) & 15)) return false;
    return true;
}

void launch_cgs_pass(hdgb_ctx* ctx, int mode, const double* V, int64_t ldv, int nvec, double* w, int64_t n, const double* coef,
                     double* out, double* work) {
    OrthArgs a;
    a.V = V; a.ldv = ldv; a.nvec = nvec; a.w = w; a.n = n; a.coef = coef; a.out = out;
    a.partial = work + 2;
    a.counter = reinterpret_cast<unsigned*>(work);
    a.stages = 2;
    a.evict_first = 0;
    switch (mode) {
        case 0: launch_mode<0>(ctx, a); break;
        case 1: launch_mode<1>(ctx, a); break;
        case 2: launch_mode<2>(ctx, a); break;
        default: launch_mode<3>(ctx, a); break;
    }
}

}  // namespace hdgb
