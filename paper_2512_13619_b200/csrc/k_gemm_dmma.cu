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
    const double* c_in;       // beta term read from here (same layout and stride as c); nullptr: from c
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
    const double* Cin = g.c_in ? g.c_in + item * g.c_stride : C;
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

    // epilogue: lane holds C[grp][2 tig], C[grp][2 tig + 1] of every 8 x 8 tile.  For beta != 0 the old entries of a
    // column group are loaded as one batch before the first store (a load after a store to possibly aliasing
    // memory cannot be hoisted by the compiler: entry-by-entry read-modify-write serialises 32 round trips)
    const double alpha = g.alpha, beta = g.beta;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double old[2][4];
        double* cc[2];
        bool okc[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gj = col0 + wn * 32 + j * 8 + 2 * tig + h;
            okc[h] = gj < n;
            const int cj = okc[h] ? (gj / g.c_colw) * g.c_colstride + gj % g.c_colw : 0;
            cc[h] = C + static_cast<int64_t>(cj) * m;
            const double* ci = Cin + static_cast<int64_t>(cj) * m;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int gi = row0 + wm * 32 + i * 8 + grp;
                old[h][i] = (beta != 0.0 && okc[h] && gi < m) ? ci[gi] : 0.0;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int gi = row0 + wm * 32 + i * 8 + grp;
                if (okc[h] && gi < m) cc[h][gi] = alpha * acc[i][j][h] + beta * old[h][i];
            }
    }
}

template <int WM, int WN>
void launch_wmwn(hdgb_ctx* ctx, const GemmArgs& g, int64_t batch, bool vec) {
    constexpr int BM = 32 * WM, BN = 32 * WN;
    const size_t smem = (2 * KC * (BM + 4) + 2 * BN * LDB) * sizeof(double);
    auto kv = gemm_dmma_kernel<WM, WN, true>;
    auto ks = gemm_dmma_kernel<WM, WN, false>;
    ensure_dynamic_smem(kv, smem);
    ensure_dynamic_smem(ks, smem);
    int64_t done = 0;
    while (done < batch) {  // gridDim.z limit
        const int64_t nb = (batch - done) < 65535 ? (batch - done) : 65535;
        GemmArgs h = g;
        h.a += done * g.a_stride;
        h.b += done * g.b_stride;
        h.c += done * g.c_stride;
        if (h.c_in) h.c_in += done * g.c_stride;
        dim3 grid(ceil_div(g.m, BM), ceil_div(g.n, BN), static_cast<unsigned>(nb));
        if (vec) kv<<<grid, WM * WN * 32, smem, ctx->stream>>>(h);
        else ks<<<grid, WM * WN * 32, smem, ctx->stream>>>(h);
        HDGB_LAUNCH_CHECK(ctx);
        done += nb;
    }
}

// ---- fused Schur complement --------------------------------------------------------------------------------
// K-bar = J-bar - H-bar (E-bar^-1 F-bar)   (local_ops.cpp:408-411) as ONE kernel: a CTA owns 32 columns of one
// element's K-bar.  Sweep 1 forms the 32 columns of T = E-bar^-1 F-bar from E-bar^-1 streamed in k-chunks of 16
// (the same two-stage cp.async ring as gemm_dmma_kernel) against the F-bar columns resident in shared memory;
// the accumulators are stored over the F-bar columns in right-operand layout, and sweep 2 streams H-bar through
// the same ring against that T.  T never goes to HBM (2 x 8 npe nfl bytes per element less traffic, one launch
// instead of two, the first H-bar chunk in flight while T is written).  WM = ceil(nfl / 32) warps; the warps whose
// 32 rows lie beyond npe only help loading in sweep 1.
struct SchurArgs {
    int npe, nfl;
    const double* einv;
    int64_t s_ee;
    const double* f;
    const double* h;
    int64_t s_ef;
    const double* j;
    double* k;
    int64_t s_ff;
};

template <int WM, bool VEC>
__global__ void __launch_bounds__(WM * 32) schur_fused_kernel(SchurArgs g) {
    constexpr int BM = 32 * WM, BN = 32, NT = WM * 32;
    constexpr int LDA = BM + 4;  // = 4 (mod 16)
    extern __shared__ __align__(16) double smem[];
    const int npe = g.npe, nfl = g.nfl;
    const int kp = (npe + KC - 1) / KC * KC;
    const int ldt = kp + 4;  // = 4 (mod 16)
    double* As = smem;                 // [2][KC][LDA]
    double* Ts = smem + 2 * KC * LDA;  // [BN][ldt]: F-bar columns, then T columns
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int grp = lane >> 2, tig = lane & 3;
    const int64_t item = blockIdx.y;
    const double* Einv = g.einv + item * g.s_ee;
    const double* F = g.f + item * g.s_ef;
    const double* H = g.h + item * g.s_ef;
    const double* J = g.j + item * g.s_ff;
    double* K = g.k + item * g.s_ff;
    const int col0 = blockIdx.x * BN;
    constexpr int W = VEC ? 2 : 1;

    // columns k0 .. k0 + KC - 1 of the column-major (m x npe) matrix A into ring stage s (rows >= m, columns >= npe: zero)
    auto load_stage = [&](int s, const double* A, int m, int k0) {
        double* as = As + s * KC * LDA;
        for (int t = tid; t < KC * (BM / W); t += NT) {
            const int p = t / (BM / W), i = (t - p * (BM / W)) * W;
            const int gp = k0 + p;
            const bool ok = i < m && gp < npe;
            cp_async_zfill<VEC>(smem_addr(as + p * LDA + i), ok ? A + static_cast<int64_t>(gp) * m + i : A, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    double acc[4][4][2];
    auto clear = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    };
    // acc += A[rows of this warp, :] * Ts over all k-chunks; stage 0 of the ring already holds chunk 0
    auto sweep = [&](const double* A, int m, bool active) {
        const int nk = kp / KC;
        for (int c = 0; c < nk; ++c) {
            const int s = c & 1;
            if (c + 1 < nk) {
                load_stage(s ^ 1, A, m, (c + 1) * KC);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncthreads();
            if (active) {
                const double* as = As + s * KC * LDA + warp * 32 + grp;
                const double* bs = Ts + grp * ldt + c * KC;
#pragma unroll
                for (int kk = 0; kk < KC; kk += 4) {
                    double af[4], bf[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) af[i] = as[(kk + tig) * LDA + i * 8];
#pragma unroll
                    for (int j = 0; j < 4; ++j) bf[j] = bs[j * 8 * ldt + kk + tig];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
                }
            }
            __syncthreads();
        }
    };

    // F-bar columns col0 .. col0 + 31 (rows >= npe and columns >= nfl: zero) ride in the first commit group
    for (int t = tid; t < BN * (kp / W); t += NT) {
        const int j = t / (kp / W), p = (t - j * (kp / W)) * W;
        const bool ok = col0 + j < nfl && p < npe;
        cp_async_zfill<VEC>(smem_addr(Ts + j * ldt + p), ok ? F + static_cast<int64_t>(col0 + j) * npe + p : F, ok);
    }
    load_stage(0, Einv, npe, 0);
    clear();
    const bool act1 = warp * 32 < npe;
    sweep(Einv, npe, act1);
    // every warp is past its last read of the F-bar columns (trailing barrier of the sweep): start H-bar, store T
    load_stage(0, H, nfl, 0);
    if (act1) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = warp * 32 + i * 8 + grp;
            if (r < kp) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    Ts[(j * 8 + 2 * tig) * ldt + r] = acc[i][j][0];
                    Ts[(j * 8 + 2 * tig + 1) * ldt + r] = acc[i][j][1];
                }
            }
        }
    }
    clear();
    sweep(H, nfl, true);  // its first barrier orders the T stores before the first fragment load

    // K-bar = J-bar - acc: the J-bar entries of a column group are loaded as one batch before the stores
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double old[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gj = col0 + j * 8 + 2 * tig + h;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int gi = warp * 32 + i * 8 + grp;
                old[h][i] = (gj < nfl && gi < nfl) ? J[static_cast<int64_t>(gj) * nfl + gi] : 0.0;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gj = col0 + j * 8 + 2 * tig + h;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int gi = warp * 32 + i * 8 + grp;
                if (gj < nfl && gi < nfl) K[static_cast<int64_t>(gj) * nfl + gi] = old[h][i] - acc[i][j][h];
            }
        }
    }
}

template <int WM>
void launch_schur_wm(hdgb_ctx* ctx, const SchurArgs& g, int64_t batch, bool vec) {
    const int kp = ceil_div(g.npe, KC) * KC;
    const size_t smem = (2 * KC * (32 * WM + 4) + 32 * static_cast<size_t>(kp + 4)) * sizeof(double);
    auto kv = schur_fused_kernel<WM, true>;
    auto ks = schur_fused_kernel<WM, false>;
    ensure_dynamic_smem(kv, smem);
    ensure_dynamic_smem(ks, smem);
    int64_t done = 0;
    while (done < batch) {  // gridDim.y limit
        const int64_t nb = (batch - done) < 65535 ? (batch - done) : 65535;
        SchurArgs h = g;
        h.einv += done * g.s_ee; h.f += done * g.s_ef; h.h += done * g.s_ef; h.j += done * g.s_ff; h.k += done * g.s_ff;
        dim3 grid(ceil_div(g.nfl, 32), static_cast<unsigned>(nb));
        if (vec) kv<<<grid, WM * 32, smem, ctx->stream>>>(h);
        else ks<<<grid, WM * 32, smem, ctx->stream>>>(h);
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

// ---- fused q-elimination product --------------------------------------------------------------------------
// [C0; C1] -= sum_t [A0_t; A1_t] * B_t  for t < nterm (the space directions): the two row blocks (E-bar over
// H-bar, or F-bar over J-bar) share the right operand M^-1 B_t / M^-1 C_t, and the D direction terms are one
// long K sweep, so one CTA per (element, 32 WN columns) replaces 2 D separate products and reads / writes the
// outputs once (local_ops.cpp:389-398).  Row block 1 starts at a multiple of 32 rows so that no 32 x 32 warp
// tile straddles the blocks.
struct QelimArgs {
    int m0, m1, n, k, nterm;
    const double* a0[3];
    const double* a1[3];
    const double* b[3];
    int64_t a0_stride, a1_stride, b_stride;
    double* c0;
    double* c1;
    int64_t c0_stride, c1_stride;
    int c_colw, c_colstride;
};

template <bool VEC, int NS>
__global__ void __launch_bounds__(512, 1) qelim_fused_kernel(QelimArgs g, int WM, int WN) {
    const int BM = 32 * WM, BN = 32 * WN, NT = WM * WN * 32;
    const int LDA = BM + 4;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                  // [NS][KC][LDA]
    double* Bs = smem + NS * KC * LDA;  // [NS][BN][LDB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % WM, wn = warp / WM;
    const int grp = lane >> 2, tig = lane & 3;
    const int64_t item = blockIdx.z;
    const int m0 = g.m0, m1 = g.m1, n = g.n, k = g.k;
    const int pad0 = (m0 + 31) / 32 * 32;
    const int col0 = blockIdx.y * BN;
    const int row0 = blockIdx.x * BM;  // row tiling (single row block only: m1 == 0)
    const int nkc = (k + KC - 1) / KC;       // chunks per term
    const int nchunk = nkc * g.nterm;
    constexpr int W = VEC ? 2 : 1;
    const int a_p0 = tid / (BM / W), a_i0 = (tid - a_p0 * (BM / W)) * W, a_pstep = NT / (BM / W);

    auto load_stage = [&](int s, int ch) {
        const int t = ch / nkc, k0 = (ch - t * nkc) * KC;
        const double* A0 = g.a0[t] + item * g.a0_stride;
        const double* A1 = g.a1[t] + item * g.a1_stride;
        const double* B = g.b[t] + item * g.b_stride;
        double* as = As + s * KC * LDA;
        double* bs = Bs + s * BN * LDB;
        // thread = (k-row p0 + 2 WN it, row pair i0): NT / (BM / W) = 2 WN exactly, so the row is fixed per thread
        for (int p = a_p0; p < KC; p += a_pstep) {
            const int i = a_i0;
            const int gp = k0 + p;
            const double* src = A0;
            bool ok = gp < k;
            if (row0 + i < pad0) {
                ok = ok && row0 + i < m0;
                if (ok) src = A0 + static_cast<int64_t>(gp) * m0 + row0 + i;
            } else {
                const int i1 = row0 + i - pad0;
                ok = ok && i1 < m1;
                if (ok) src = A1 + static_cast<int64_t>(gp) * m1 + i1;
            }
            cp_async_zfill<VEC>(smem_addr(as + p * LDA + i), src, ok);
        }
        for (int q = tid; q < BN * (KC / W); q += NT) {
            const int j = q / (KC / W), p = (q - j * (KC / W)) * W;
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

    // NS-stage cp.async ring: chunks c+1 .. c+NS-1 are in flight while chunk c is multiplied
#pragma unroll
    for (int c = 0; c < NS - 1; ++c) {
        if (c < nchunk) load_stage(c, c);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    int s = 0;
    for (int c = 0; c < nchunk; ++c) {
        const int sn = (s + NS - 1 >= NS) ? s - 1 : s + NS - 1;  // stage of chunk c + NS - 1
        if (c + NS - 1 < nchunk) load_stage(sn, c + NS - 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(NS - 1) : "memory");
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
        s = (s + 1 == NS) ? 0 : s + 1;
    }
    // epilogue: C -= acc, the old entries of a column group loaded as one batch before the first store
    const int r0 = row0 + wm * 32;
    const bool blk1 = r0 >= pad0;
    const int mrows = blk1 ? m1 : m0;
    double* C = blk1 ? g.c1 + item * g.c1_stride : g.c0 + item * g.c0_stride;
    const int rbase = blk1 ? r0 - pad0 : r0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double old[2][4];
        double* cc[2];
        bool okc[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gj = col0 + wn * 32 + j * 8 + 2 * tig + h;
            okc[h] = gj < n;
            const int cj = okc[h] ? (gj / g.c_colw) * g.c_colstride + gj % g.c_colw : 0;
            cc[h] = C + static_cast<int64_t>(cj) * mrows;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int gi = rbase + i * 8 + grp;
                old[h][i] = (okc[h] && gi < mrows) ? cc[h][gi] : 0.0;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int gi = rbase + i * 8 + grp;
                if (okc[h] && gi < mrows) cc[h][gi] = old[h][i] - acc[i][j][h];
            }
    }
}

}  // namespace

// C_b[:, colmap(j)] = alpha * A_b * B_b[:, j] + beta * C_b[:, colmap(j)], all column-major with leading
// dimensions m (A, C) and k (B).  colmap(j) = (j / c_colw) * c_colstride + j % c_colw (identity when
// c_colw >= n): lets one product scatter its columns into the (local face, component) column blocks of
// F-bar / J-bar for multi-component systems.
void launch_gemm_dmma(hdgb_ctx* ctx, int m, int n, int k, const double* a, int64_t a_stride, const double* b,
                      int64_t b_stride, double* c, int64_t c_stride, int64_t batch, double alpha, double beta,
                      int c_colw, int c_colstride, const double* c_in) {
    if (batch <= 0 || m <= 0 || n <= 0) return;
    GemmArgs g{m, n, k, a, a_stride, b, b_stride, c, c_stride, alpha, beta, c_colw > 0 ? c_colw : n,
               c_colw > 0 ? c_colstride : n, c_in};
    // 16-byte cp.async needs even leading dimensions / strides and 16-byte aligned bases
    const bool vec = (m % 2 == 0) && (k % 2 == 0) && (a_stride % 2 == 0) && (b_stride % 2 == 0) &&
                     (reinterpret_cast<uintptr_t>(a) % 16 == 0) && (reinterpret_cast<uintptr_t>(b) % 16 == 0);
    int wm = ceil_div(m, 32), wn = ceil_div(n, 32);
    if (wm > 4) wm = 4;
    if (wn > 4) wn = 4;
    if (wn > tuning().gemm_wn_cap) wn = tuning().gemm_wn_cap;  // narrow CTAs: more of them resident per SM
    if (wm > tuning().gemm_wm_cap) wm = tuning().gemm_wm_cap;
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

// Returns false when the element sizes are outside the fused kernel's range (caller runs the two products).
bool launch_schur_fused(hdgb_ctx* ctx, int npe, int nfl, const double* einv, int64_t s_ee, const double* f, const double* h,
                        int64_t s_ef, const double* j, double* k, int64_t s_ff, int64_t batch) {
    if (npe <= 0 || nfl <= 0 || nfl > 128 || ceil_div(npe, 32) > ceil_div(nfl, 32)) return false;
    if (batch <= 0) return true;
    SchurArgs g{npe, nfl, einv, s_ee, f, h, s_ef, j, k, s_ff};
    const bool vec = (npe % 2 == 0) && (nfl % 2 == 0) && (s_ee % 2 == 0) && (s_ef % 2 == 0) &&
                     (reinterpret_cast<uintptr_t>(einv) % 16 == 0) && (reinterpret_cast<uintptr_t>(f) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(h) % 16 == 0);
    switch (ceil_div(nfl, 32)) {
        case 1: launch_schur_wm<1>(ctx, g, batch, vec); break;
        case 2: launch_schur_wm<2>(ctx, g, batch, vec); break;
        case 3: launch_schur_wm<3>(ctx, g, batch, vec); break;
        default: launch_schur_wm<4>(ctx, g, batch, vec); break;
    }
    return true;
}

}  // namespace hdgb

namespace hdgb {

// Returns false when the stacked row blocks need more than 8 warp rows (caller falls back to single products).
bool launch_qelim_fused(hdgb_ctx* ctx, int m0, int m1, int n, int k, int nterm, const double* const a0[3], int64_t a0_stride,
                        const double* const a1[3], int64_t a1_stride, const double* const b[3], int64_t b_stride, double* c0,
                        int64_t c0_stride, double* c1, int64_t c1_stride, int64_t batch, int c_colw, int c_colstride) {
    if (batch <= 0 || n <= 0) return true;
    int WM = ceil_div(m0, 32) + ceil_div(m1, 32);
    if (nterm > 3) return false;
    int gx = 1;
    if (m1 <= 0) {
        // single row block: tile the rows over blockIdx.x
        c1 = c0;
        c1_stride = c0_stride;
        if (WM > 4) WM = 4;
        gx = ceil_div(m0, 32 * WM);
    } else if (WM > 8) {
        return false;
    }
    int WN = ceil_div(n, 32);
    // narrow column tiles: small CTAs, several resident per SM, so that the barrier-separated load / multiply
    // phases of different CTAs overlap (a 15-warp CTA per SM measured 35% of the DMMA peak, 4-warp CTAs 73%)
    const int wn_cap = tuning().qelim_wn;
    if (WN > wn_cap) WN = wn_cap;
    QelimArgs g{};
    g.m0 = m0; g.m1 = m1; g.n = n; g.k = k; g.nterm = nterm;
    bool vec = (m0 % 2 == 0) && (m1 % 2 == 0) && (k % 2 == 0) && (a0_stride % 2 == 0) && (a1_stride % 2 == 0) && (b_stride % 2 == 0);
    for (int t = 0; t < nterm; ++t) {
        g.a0[t] = a0[t]; g.a1[t] = a1[t]; g.b[t] = b[t];
        vec = vec && reinterpret_cast<uintptr_t>(a0[t]) % 16 == 0 && reinterpret_cast<uintptr_t>(a1[t]) % 16 == 0 &&
              reinterpret_cast<uintptr_t>(b[t]) % 16 == 0;
    }
    g.a0_stride = a0_stride; g.a1_stride = a1_stride; g.b_stride = b_stride;
    g.c0 = c0; g.c1 = c1; g.c0_stride = c0_stride; g.c1_stride = c1_stride;
    g.c_colw = c_colw > 0 ? c_colw : n;
    g.c_colstride = c_colw > 0 ? c_colstride : n;
    const int NS = tuning().qelim_stages >= 3 ? 3 : 2;
    const size_t smem = static_cast<size_t>(NS) * (KC * (32 * WM + 4) + 32 * WN * LDB) * sizeof(double);
    ensure_dynamic_smem(qelim_fused_kernel<true, 2>, smem);
    ensure_dynamic_smem(qelim_fused_kernel<false, 2>, smem);
    ensure_dynamic_smem(qelim_fused_kernel<true, 3>, smem);
    ensure_dynamic_smem(qelim_fused_kernel<false, 3>, smem);
    int64_t done = 0;
    while (done < batch) {
        const int64_t nb = (batch - done) < 65535 ? (batch - done) : 65535;
        QelimArgs h = g;
        for (int t = 0; t < nterm; ++t) {
            h.a0[t] += done * a0_stride; h.a1[t] += done * a1_stride; h.b[t] += done * b_stride;
        }
        h.c0 += done * c0_stride; h.c1 += done * c1_stride;
        dim3 grid(gx, ceil_div(n, 32 * WN), static_cast<unsigned>(nb));
        const int nthr = WM * WN * 32;
        if (NS == 3) {
            if (vec) qelim_fused_kernel<true, 3><<<grid, nthr, smem, ctx->stream>>>(h, WM, WN);
            else qelim_fused_kernel<false, 3><<<grid, nthr, smem, ctx->stream>>>(h, WM, WN);
        } else {
            if (vec) qelim_fused_kernel<true, 2><<<grid, nthr, smem, ctx->stream>>>(h, WM, WN);
            else qelim_fused_kernel<false, 2><<<grid, nthr, smem, ctx->stream>>>(h, WM, WN);
        }
        HDGB_LAUNCH_CHECK(ctx);
        done += nb;
    }
    return true;
}

}  // namespace hdgb
