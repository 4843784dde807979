// Stream GEMV: the bandwidth kernel behind block_matvec (face_matrix.cpp:83-107, gather fused),
// apply_bj (preconditioner.cpp:48-52), the element solves of apply_asm (:86-91) and recover_local
// (local_ops.cpp:452-460) at sizes where HBM streaming is what matters.
//
// The batched block rows of a DenseBatch are ONE contiguous array (dense_batch.hpp:12-34), so the
// kernel treats the matrix data as a byte stream: a persistent CTA per SM owns a contiguous range
// of items and pulls it through shared memory with 1D bulk TMA copies (cp.async.bulk ...
// mbarrier::complete_tx).  Each warp runs its own ring of stages: lane 0 issues the copy of the
// warp's next chunk, the warp waits on the stage's mbarrier, multiplies out of shared memory and
// re-arms the stage -- no CTA-wide barrier anywhere, 8 x 24 KB in flight per SM.  A stage
// ("chunk") holds either a whole number of small items or a column range of one large item; the warp
//   * gathers the item's input slice (neighbour slices through the index table, zeros for
//     kNoFace) into its private shared-memory x buffer while the TMA copy is in flight,
//   * multiplies (lanes own 1-2 consecutive rows x a column group; 128-bit LDS when the row count
//     is even) keeping partial sums in registers across the chunks of an item,
//   * combines the column groups with a fixed-order shuffle tree (deterministic) and writes y.
// Small items (rows <= 32 after vectorisation, cols <= 32: triangle / quadrilateral blocks) use the PACKED
// mode instead: 16 warps per CTA with stages of a few KB, a warp multiplies 32 / RL items side by side (lane =
// item x row group, two independent accumulators, no cross-lane reduction), the x slices are gathered one
// (item, slot) per lane and padded to an even stride so that two columns are read with one LDS.128.  At
// 1 KB per item the per-item instruction count, not the byte stream, is what limits the kernel: ring
// positions are carried incrementally in 32-bit counters (no 64-bit divisions on the per-item path).
// HBM sees every matrix byte exactly once, as large sequential bulk reads; x / y traffic is served
// from L2.  Roofline: HBM.  Algorithmic bytes per item: 8*(rows*cols + cols + rows) + 4*nslots.
#include "kernels.cuh"
#include "tma.cuh"

namespace hdgb {

namespace {

// Each warp runs its own TMA ring: issue -> wait -> multiply -> re-issue.  8 warps for large items
// (24 KB stages); 16 warps for small items (a few KB per stage), where the per-item dependency chain
// -- not the byte stream -- is what has to be hidden.
constexpr int kMaxWarps = 16;
constexpr int kMaxThreads = kMaxWarps * 32;
constexpr int kMaxStages = 32;      // warps rings of stages / warps stages each
constexpr size_t kSmemBudget = 216 * 1024;

struct StreamPlan {
    int rows, cols;
    int split;            // 0: chunk = ipc whole items; 1: chunk = cpc columns of one item
    int ipc;              // items per chunk (grouped)
    int cpc;              // columns per chunk (split)
    int cpi;              // chunks per item (split)
    int stages;
    int xs_elems;         // per-warp x buffer (doubles)
    int is_elems;         // per-warp index buffer (ints, multiple of 2)
    int stage_elems;      // doubles per stage
    int64_t batch;
    int64_t n_units;      // grouped: chunks; split: items
    int warps;            // warps per CTA (8 or 16)
    int ipw;              // packed mode (> 0): items a warp multiplies side by side, one (item, row group) per lane
    int xstride;          // doubles between the x slices of consecutive items of a chunk (cols, or cols + 1 in packed mode with odd cols)
    float inv_cols, inv_width, inv_nslots;  // reciprocals for the gather's index arithmetic
    int64_t persist_bytes; // leading bytes of the matrix copied with an evict-last hint (0: none)
    int evict_first;      // bulk copies of the matrix carry an L2 evict-first hint (the gathered vector stays cached)
};

template <int V>
__device__ __forceinline__ void lds_rows(const double* p, double (&v)[V]);
template <>
__device__ __forceinline__ void lds_rows<1>(const double* p, double (&v)[1]) { v[0] = *p; }
template <>
__device__ __forceinline__ void lds_rows<2>(const double* p, double (&v)[2]) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    v[0] = t.x;
    v[1] = t.y;
}

// acc += A[:, 0..ncols) * xs[0..ncols) for this lane's rows; A column-major with leading dim rows.
template <int V, int RT>
__device__ __forceinline__ void accumulate(const double* __restrict__ A, const double* __restrict__ xs, int rows, int ncols,
                                           int rl, int cg, int CG, double (&acc)[RT][V]) {
    if (cg >= CG) return;
#pragma unroll 4
    for (int c = cg; c < ncols; c += CG) {
        const double xv = xs[c];
        const double* col = A + static_cast<size_t>(c) * rows;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const int r = (rl + 32 * t) * V;
            if (RT == 1 || r < rows) {
                double a[V];
                lds_rows<V>(col + r, a);
#pragma unroll
                for (int v = 0; v < V; ++v) acc[t][v] = fma(a[v], xv, acc[t][v]);
            }
        }
    }
}

template <int V, int RT>
__global__ void __launch_bounds__(kMaxThreads, 1) stream_gemv_kernel(GemvArgs g, StreamPlan p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* stage_base = reinterpret_cast<double*>(smem_raw);
    double* xs_base = stage_base + static_cast<size_t>(p.stages) * p.stage_elems;
    const int kWarps = p.warps;
    int* is_base = reinterpret_cast<int*>(xs_base + static_cast<size_t>(kWarps) * 2 * p.xs_elems);
    uint64_t* full = reinterpret_cast<uint64_t*>(is_base + static_cast<size_t>(kWarps) * 3 * p.is_elems);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows = p.rows, cols = p.cols;
    const int64_t item_elems = static_cast<int64_t>(rows) * cols;
    const int SW = p.stages / kWarps;  // stages of this warp's private ring

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) mbar_init(full + s, 1);
        mbar_fence_init();
    }
    __syncthreads();

    // this CTA's contiguous range of units (grouped: chunks, split: items); units are dealt to the
    // warps round-robin and every warp streams ITS chunks through ITS ring, so a waiter is never
    // more than one mbarrier phase ahead of the copy it waits for.  Per-warp counters are 32-bit and
    // ring positions are carried incrementally: no 64-bit divisions on the per-item path.
    const int64_t u0 = p.n_units * blockIdx.x / gridDim.x;
    const int64_t u1 = p.n_units * (blockIdx.x + 1) / gridDim.x;
    const int my_units = (u1 - u0 > warp) ? static_cast<int>((u1 - u0 - warp + kWarps - 1) / kWarps) : 0;
    const int my_chunks = p.split ? my_units * p.cpi : my_units;
    double* my_stage = stage_base + static_cast<size_t>(warp) * SW * p.stage_elems;
    uint64_t* my_full = full + warp * SW;
    const int64_t w0 = u0 + warp;  // first unit of this warp; its unit t is w0 + t * kWarps

    // chunk n of this warp into ring stage s
    const uint64_t l2pol = p.evict_first ? l2_policy_evict_first() : 0;
    // (stream_persist_mb, off: the leading part of the matrix copied with an evict-last hint so that it survives in the L2 from
    // one application to the next -- measured slower at config 2 with 24 / 32 / 48 MB per matrix: matvec 221 -> 225-229 us,
    // ASM apply 255 -> 262-270 us)
    uint64_t l2keep = 0;
    if (p.persist_bytes > 0) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(l2keep));
    const double* keep_end = g.a + p.persist_bytes / static_cast<int64_t>(sizeof(double));
    auto issue = [&](int n, int s) {
        const double* src;
        int64_t elems;
        if (p.split) {
            const int ui = n / p.cpi;
            const int ci = n - ui * p.cpi;
            const int64_t item = w0 + static_cast<int64_t>(ui) * kWarps;
            const int c0 = ci * p.cpc;
            const int nc = min(p.cpc, cols - c0);
            src = g.a + item * item_elems + static_cast<int64_t>(c0) * rows;
            elems = static_cast<int64_t>(nc) * rows;
        } else {
            const int64_t i0 = (w0 + static_cast<int64_t>(n) * kWarps) * p.ipc;
            int64_t cnt = g.batch - i0 < p.ipc ? g.batch - i0 : p.ipc;
            if ((item_elems & 1) && (cnt & 1)) --cnt;  // keep the copy a multiple of 16 bytes; the odd tail item is read directly
            src = g.a + i0 * item_elems;
            elems = cnt * item_elems;
        }
        const uint32_t bytes = static_cast<uint32_t>(elems * sizeof(double));
        // The stage is re-armed by lane 0 after a cross-proxy fence + __syncwarp() (the call sites): every lane's reads
        // of it have completed.  That FMAs consumed the loaded values is NOT enough -- ptxas may schedule the copy
        // behind the ISSUE of the last loads and ahead of their consumers (tma.cuh: ring_release_all).
        mbar_expect_tx(my_full + s, bytes);
        if (bytes) {
            if (p.evict_first) tma_bulk_g2s_hint(my_stage + static_cast<size_t>(s) * p.stage_elems, src, bytes, my_full + s, (p.persist_bytes > 0 && src < keep_end) ? l2keep : l2pol);
            else tma_bulk_g2s(my_stage + static_cast<size_t>(s) * p.stage_elems, src, bytes, my_full + s);
        }
    };
    if (lane == 0)
        for (int n = 0; n < SW && n < my_chunks; ++n) issue(n, n);

    // per-warp x (double-buffered) and index (triple-buffered) staging, filled with cp.async so the
    // gather of the NEXT unit runs behind the multiply of the current one
    double* xs_w = xs_base + static_cast<size_t>(warp) * 2 * p.xs_elems;
    int* is_w = is_base + static_cast<size_t>(warp) * 3 * p.is_elems;
    const int RL = (rows + V - 1) / V;
    const int CG = RL >= 32 ? 1 : 32 / RL;
    const int cg = RL >= 32 ? 0 : lane / RL;
    const int rl = RL >= 32 ? lane : lane - cg * RL;
    const int nslots = g.idx ? cols / g.width : 0;
    const int width = g.width;

    // unit t of this warp -> first item and item count
    auto unit_items = [&](int t, int64_t& item0, int& cnt) {
        if (p.split) {
            item0 = w0 + static_cast<int64_t>(t) * kWarps;
            cnt = 1;
        } else {
            item0 = (w0 + static_cast<int64_t>(t) * kWarps) * p.ipc;
            cnt = static_cast<int>(g.batch - item0 < p.ipc ? g.batch - item0 : p.ipc);
        }
    };
    // pipeline stage 0: index rows of unit t -> index buffer ib   (one cp.async group, possibly empty)
    auto stage_idx = [&](int t, int ib) {
        if (t < my_units && g.idx != nullptr) {
            int64_t item0;
            int cnt;
            unit_items(t, item0, cnt);
            const int* src = g.idx + item0 * nslots;
            const uint32_t dst = smem_u32(is_w + ib * p.is_elems);
            const int ts = cnt * nslots;
            for (int j = lane; j < ts; j += 32)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst + 4u * j), "l"(src + j) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // pipeline stage 1: x entries of unit t -> x buffer xb; needs the unit's index rows (buffer ib) in shared memory
    auto stage_x = [&](int t, int xb, int ib) {
        if (t < my_units) {
            int64_t item0;
            int cnt;
            unit_items(t, item0, cnt);
            const uint32_t dst = smem_u32(xs_w + xb * p.xs_elems);
            const int total = cnt * cols;
            if (g.idx == nullptr) {
                const double* xg = g.x + item0 * cols;
                if (p.xstride == cols) {
                    for (int j = lane; j < total; j += 32)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8u * j), "l"(xg + j) : "memory");
                } else {
                    for (int j = lane; j < total; j += 32) {
                        const int it = static_cast<int>((j + 0.5f) * p.inv_cols);
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8u * (j + it)), "l"(xg + j) : "memory");
                    }
                }
            } else {
                const int* is = is_w + ib * p.is_elems;
                if (p.ipw > 0) {
                    // narrow slices: one lane per (item, slot) copies the whole slice -- no per-entry index arithmetic
                    const int ts = cnt * nslots;
                    for (int j = lane; j < ts; j += 32) {
                        const int src = is[j];
                        const double* sp = g.x + static_cast<int64_t>(src < 0 ? 0 : src) * width;
                        const int nbytes = src < 0 ? 0 : 8;  // src-size 0 zero-fills: absent neighbour (kNoFace)
                        const int it = static_cast<int>((j + 0.5f) * p.inv_nslots);
                        uint32_t d = dst + 8u * static_cast<uint32_t>(j * width + it * (p.xstride - cols));
#pragma unroll 5
                        for (int o = 0; o < width; ++o, d += 8u, ++sp)
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(sp), "r"(nbytes) : "memory");
                    }
                } else {
                    for (int j = lane; j < total; j += 32) {
                        // exact for j < 2^21: (j + 0.5) / cols is at least 0.5 / cols away from an integer
                        const int it = static_cast<int>((j + 0.5f) * p.inv_cols), c = j - it * cols;
                        const int sl = static_cast<int>((c + 0.5f) * p.inv_width);
                        const int o = c - sl * width;
                        const int src = is[it * nslots + sl];
                        const double* sp = src < 0 ? g.x : g.x + static_cast<int64_t>(src) * width + o;
                        const int nbytes = src < 0 ? 0 : 8;
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst + 8u * j), "l"(sp), "r"(nbytes) : "memory");
                    }
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto reduce_store = [&](double (&acc)[RT][V], int64_t item) {
        // fixed-order tree over the column groups (lane = cg*RL + rl)
        if (CG > 1) {
            int top = 1;
            while (top < CG) top <<= 1;
            for (int off = top >> 1; off > 0; off >>= 1) {
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const double o = __shfl_down_sync(0xffffffffu, acc[0][v], off * RL);
                    if (cg + off < CG) acc[0][v] += o;
                }
            }
        }
        if (cg == 0) {
#pragma unroll
            for (int t = 0; t < RT; ++t) {
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const int r = (rl + 32 * t) * V + v;
                    if (r < rows) {
                        const int64_t o = item * rows + r;
                        double out = g.alpha * acc[t][v];
                        if (g.z != nullptr) out += g.beta * g.z[o];
                        g.y[o] = out;
                    }
                }
            }
        }
    };

    stage_idx(0, 0);
    stage_idx(1, 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    stage_x(0, 0, 0);
    int n = 0;             // this warp's running chunk counter
    int rs = 0;            // ring stage of chunk n
    uint32_t rph = 0;      // mbarrier phase parity of chunk n
    int i3 = 0, i2 = 0;    // t % 3, t % 2
    const int si = lane / RL, prl = lane - si * RL;  // packed mode: item slot and row group of this lane
    for (int t = 0; t < my_units; ++t) {
        const int i3n = (i3 == 2) ? 0 : i3 + 1;        // (t + 1) % 3
        const int i3nn = (i3n == 2) ? 0 : i3n + 1;     // (t + 2) % 3
        stage_idx(t + 2, i3nn);
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // index rows of t+1 and x of t have landed
        __syncwarp();
        stage_x(t + 1, i2 ^ 1, i3n);
        int64_t item0;
        int cnt;
        unit_items(t, item0, cnt);
        const double* xs = xs_w + i2 * p.xs_elems;
        if (p.split) {
            double acc[RT][V];
#pragma unroll
            for (int tt = 0; tt < RT; ++tt)
#pragma unroll
                for (int v = 0; v < V; ++v) acc[tt][v] = 0.0;
            for (int ci = 0; ci < p.cpi; ++ci, ++n) {
                const int c0 = ci * p.cpc;
                const int nc = min(p.cpc, cols - c0);
                mbar_wait(my_full + rs, rph);
                accumulate<V, RT>(my_stage + static_cast<size_t>(rs) * p.stage_elems, xs + c0, rows, nc, rl, cg, CG, acc);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0 && n + SW < my_chunks) issue(n + SW, rs);
                if (++rs == SW) { rs = 0; rph ^= 1u; }
            }
            reduce_store(acc, item0);
        } else {
            const int cnt_tma = ((item_elems & 1) && (cnt & 1)) ? cnt - 1 : cnt;
            mbar_wait(my_full + rs, rph);
            const double* st = my_stage + static_cast<size_t>(rs) * p.stage_elems;
            if (p.ipw > 0) {
                // packed: lane = (item slot si, row group prl); every lane sweeps all columns of its
                // item with two independent accumulators -- no cross-lane reduction
                const int ie = static_cast<int>(item_elems);
                for (int it0 = 0; it0 < cnt; it0 += p.ipw) {
                    const int it = it0 + si;
                    if (si < p.ipw && it < cnt) {
                        const double* xp = xs + it * p.xstride;
                        double a0[V], a1[V];
#pragma unroll
                        for (int v = 0; v < V; ++v) a0[v] = a1[v] = 0.0;
                        int c = cols;
                        if (it < cnt_tma) {
                            const double* ap = st + it * ie + prl * V;  // shared memory
#pragma unroll 4
                            for (; c >= 2; c -= 2, ap += 2 * rows, xp += 2) {
                                double r0[V], r1[V];
                                lds_rows<V>(ap, r0);
                                lds_rows<V>(ap + rows, r1);
                                const double2 xx = *reinterpret_cast<const double2*>(xp);
#pragma unroll
                                for (int v = 0; v < V; ++v) {
                                    a0[v] = fma(r0[v], xx.x, a0[v]);
                                    a1[v] = fma(r1[v], xx.y, a1[v]);
                                }
                            }
                            if (c > 0) {
                                double r0[V];
                                lds_rows<V>(ap, r0);
                                const double x0 = xp[0];
#pragma unroll
                                for (int v = 0; v < V; ++v) a0[v] = fma(r0[v], x0, a0[v]);
                            }
                        } else {
                            // odd tail item that the 16-byte granular copy left out: read it from global memory
                            const double* ap = g.a + (item0 + it) * item_elems + prl * V;
                            for (; c > 0; --c, ap += rows, ++xp) {
#pragma unroll
                                for (int v = 0; v < V; ++v) a0[v] = fma(__ldg(ap + v), xp[0], a0[v]);
                            }
                        }
                        const int64_t o = (item0 + it) * rows + prl * V;
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            if (prl * V + v < rows) {
                                double out = g.alpha * (a0[v] + a1[v]);
                                if (g.z != nullptr) out += g.beta * g.z[o + v];
                                g.y[o + v] = out;
                            }
                        }
                    }
                }
            } else {
                for (int it = 0; it < cnt; ++it) {
                    double acc[RT][V];
#pragma unroll
                    for (int tt = 0; tt < RT; ++tt)
#pragma unroll
                        for (int v = 0; v < V; ++v) acc[tt][v] = 0.0;
                    if (it < cnt_tma) {
                        accumulate<V, RT>(st + static_cast<size_t>(it) * item_elems, xs + static_cast<size_t>(it) * cols, rows, cols, rl, cg, CG, acc);
                    } else if (V == 1) {
                        // odd tail item that the 16-byte granular copy left out: read it from global memory
                        accumulate<V, RT>(g.a + (item0 + it) * item_elems, xs + static_cast<size_t>(it) * cols, rows, cols, rl, cg, CG, acc);
                    }
                    reduce_store(acc, item0 + it);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0 && n + SW < my_chunks) issue(n + SW, rs);
            if (++rs == SW) { rs = 0; rph ^= 1u; }
            ++n;
        }
        __syncwarp();
        i3 = i3n;
        i2 ^= 1;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <int V, int RT>
void launch_t(hdgb_ctx* ctx, const GemvArgs& g, const StreamPlan& p, int grid, size_t smem) {
    auto kern = stream_gemv_kernel<V, RT>;
    ensure_dynamic_smem(kern, smem);
    kern<<<grid, p.warps * 32, smem, ctx->stream>>>(g, p);
    HDGB_LAUNCH_CHECK(ctx);
}

}  // namespace

// Returns false when the shape is outside what the streaming kernel handles (caller falls back to
// the team kernel): component-interleaved gathers, broadcast matrices, misaligned or huge rows.
bool launch_stream_gemv(hdgb_ctx* ctx, const GemvArgs& g) {
    if (g.batch <= 0 || g.rows <= 0 || g.cols <= 0) return true;
    if (g.a_div != 1 || g.comp != 1) return false;
    if (g.idx && (g.width <= 0 || g.cols % g.width != 0)) return false;
    if (reinterpret_cast<uintptr_t>(g.a) % 16 != 0) return false;
    const int rows = g.rows, cols = g.cols;
    const int64_t item_elems = static_cast<int64_t>(rows) * cols;
    const int V = (rows % 2 == 0) ? 2 : 1;
    const int RL = (rows + V - 1) / V;
    const int RT = RL <= 32 ? 1 : (RL + 31) / 32;
    if (RT > 4) return false;
    // small problems are launch-latency bound; the persistent pipeline only pays off on real streams
    if (item_elems * g.batch < tuning().stream_min_elems) return false;

    StreamPlan p{};
    p.rows = rows;
    p.cols = cols;
    p.batch = g.batch;
    const int nslots = g.idx ? cols / g.width : 0;
    p.inv_cols = 1.0f / static_cast<float>(cols);
    p.inv_width = g.idx ? 1.0f / static_cast<float>(g.width) : 1.0f;
    p.inv_nslots = nslots > 0 ? 1.0f / static_cast<float>(nslots) : 1.0f;
    // small items (short column sweeps): 16 warps, several items side by side in a warp
    const bool packed = tuning().stream_packed && RT == 1 && RL <= 16 && cols <= tuning().stream_packed_max_cols;
    const int kWarps = packed ? 16 : 8;
    p.warps = kWarps;
    p.ipw = packed ? 32 / RL : 0;
    // (measured: config 2 matvec 235 -> 222 us, ASM apply 269 -> 257 us; neutral at config 4; the packed mode of tiny blocks
    // loses 3-7 % with the hint at config 3, so it is left out there)
    p.evict_first = tuning().stream_evict_first && p.ipw == 0;
    p.persist_bytes = p.evict_first ? static_cast<int64_t>(tuning().stream_persist_mb) << 20 : 0;
    const size_t kWarpBudget = kSmemBudget / kWarps;  // stage(s) + x buffer + index buffer of one warp
    // per-warp shared memory: one or more stages + the x slice(s) + the index row(s)
    const size_t per_item = static_cast<size_t>(item_elems + 2 * (cols + 1)) * sizeof(double) + 3 * static_cast<size_t>(nslots) * sizeof(int) + 8;
    if (per_item + 128 <= kWarpBudget) {
        p.split = 0;
        p.ipc = static_cast<int>((kWarpBudget - 128) / per_item);
        if (p.ipc > 64) p.ipc = 64;
        if (packed) {
            // two stages of a few KB per warp: whole passes of ipw items
            const int want = static_cast<int>(tuning().stream_packed_stage_bytes / (item_elems * sizeof(double)));
            int ipc = (want / p.ipw) * p.ipw;
            if (ipc < p.ipw) ipc = p.ipw;
            const int half = static_cast<int>((kWarpBudget - 128) / (2 * per_item));
            if (ipc > half) ipc = half;
            if (ipc < 1) ipc = 1;
            if (ipc < p.ipc) p.ipc = ipc;
        }
        if ((item_elems & 1) && (p.ipc & 1)) {
            if (p.ipc == 1) return false;
            --p.ipc;
        }
        p.cpc = cols;
        p.cpi = 1;
        p.stage_elems = static_cast<int>(p.ipc * item_elems);
        p.xstride = packed ? ((cols + 1) & ~1) : cols;
        p.xs_elems = p.ipc * p.xstride;
        p.is_elems = p.ipc * nslots;
        p.n_units = (g.batch + p.ipc - 1) / p.ipc;
    } else {
        if ((rows & 1) && (cols & 1)) return false;  // items would start on 8-byte boundaries
        p.split = 1;
        p.ipc = 1;
        p.xstride = cols;
        p.xs_elems = cols;
        p.is_elems = nslots;
        const size_t side = 2 * static_cast<size_t>(cols) * sizeof(double) + 3 * static_cast<size_t>(nslots) * sizeof(int) + 32;
        if (side + 4096 > kWarpBudget) return false;
        const size_t left = kWarpBudget - 128 - side;
        p.cpc = static_cast<int>(left / (static_cast<size_t>(rows) * sizeof(double)));
        if (p.cpc > cols) p.cpc = cols;
        if (rows & 1) p.cpc &= ~1;
        if (p.cpc < 1) return false;
        p.cpi = (cols + p.cpc - 1) / p.cpc;
        int bal = (cols + p.cpi - 1) / p.cpi;  // balance the chunks of an item
        if ((rows & 1) && (bal & 1)) ++bal;
        if (bal <= p.cpc) p.cpc = bal;
        p.cpi = (cols + p.cpc - 1) / p.cpc;
        p.stage_elems = p.cpc * rows;
        p.n_units = g.batch;
    }
    p.stage_elems = (p.stage_elems + 15) & ~15;  // keep every stage 128-byte aligned
    p.xs_elems = (p.xs_elems + 1) & ~1;
    p.is_elems = (p.is_elems + 1) & ~1;
    const size_t fixed = static_cast<size_t>(kWarps) * (2 * p.xs_elems * sizeof(double) + 3 * p.is_elems * sizeof(int)) + kMaxStages * sizeof(uint64_t);
    if (fixed + kWarps * p.stage_elems * sizeof(double) > kSmemBudget + 4096) return false;
    p.stages = static_cast<int>((kSmemBudget + 4096 - fixed) / (p.stage_elems * sizeof(double)));
    if (p.stages > kMaxStages) p.stages = kMaxStages;
    p.stages -= p.stages % kWarps;
    const size_t smem = static_cast<size_t>(p.stages) * p.stage_elems * sizeof(double) + fixed;
    int grid = ctx->sm_count;
    if (p.n_units < grid) grid = static_cast<int>(p.n_units);

    if (V == 2) {
        switch (RT) {
            case 1: launch_t<2, 1>(ctx, g, p, grid, smem); break;
            case 2: launch_t<2, 2>(ctx, g, p, grid, smem); break;
            case 3: launch_t<2, 3>(ctx, g, p, grid, smem); break;
            default: launch_t<2, 4>(ctx, g, p, grid, smem); break;
        }
    } else {
        switch (RT) {
            case 1: launch_t<1, 1>(ctx, g, p, grid, smem); break;
            case 2: launch_t<1, 2>(ctx, g, p, grid, smem); break;
            case 3: launch_t<1, 3>(ctx, g, p, grid, smem); break;
            default: launch_t<1, 4>(ctx, g, p, grid, smem); break;
        }
    }
    return true;
}

}  // namespace hdgb
