// Blocked in-place Gauss-Jordan inverse for batches of n x n blocks, any n (lu_invert_batch,
// dense_batch.cpp:19-99: explicit inverses with partial pivoting, singularity test pivot <= 1e-14 max|A|,
// lowest failing batch index).  Used for E-bar^-1 (local_ops.cpp:400-404), the block-Jacobi and the
// additive-Schwarz inverses (preconditioner.cpp:30-46, 54-84).
//
// Algorithm (panel width NB = 16).  Gauss-Jordan with row interchanges, in place, leaves (P A)^-1; the
// inverse is its column permutation.  One elimination step k maps the matrix to G_k S_k M where S_k
// swaps rows k and p_k and G_k differs from the identity in column k only.  For a panel of NB pivots
//     G_{k+NB-1} S_{k+NB-1} ... G_k S_k  =  G' (S_{k+NB-1} ... S_k),
// and the NB non-trivial columns of G' are exactly what the in-place algorithm leaves in the panel
// columns.  So per panel:
//   (1) gj_panel_kernel  -- one warp per block factors the n x NB panel in shared memory (pivot search =
//       first row of maximal modulus among rows >= k, the reference's rule), records the pivots and the
//       row gather map of the panel's interchanges, and writes the panel into the NEW buffer;
//   (2) gj_update_kernel -- every other column c:  new[:, c] = rowperm(old[:, c]) + (G' - I) old[piv rows, c],
//       a rank-NB update on the FP64 tensor-core path (DMMA m8n8k4), the row interchanges folded into the
//       gather of the operands.  Reads the old buffer, writes the new one (ping-pong), so each panel costs
//       one read + one write of the batch: the kernel is HBM bound, 2 n^3 flops per block like the reference.
// After ceil(n / NB) panels gj_colperm_kernel applies the column permutation into the destination.
// Results agree with the reference's LU + solves to rounding (different but equally stable operation order).
#include <climits>

#include "kernels.cuh"

namespace hdgb {

namespace {

constexpr int NB = 16;
constexpr int LDB = NB + 4;  // = 4 (mod 16): conflict-free DMMA fragment loads

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// ---- prepass: copy a -> x0 and amax[b] = max |A_b| ------------------------------------------------------
__global__ void gj_prepare_kernel(int n, const double* __restrict__ a, double* __restrict__ x0, double* __restrict__ amax) {
    const int64_t b = blockIdx.x;
    const int64_t nn = static_cast<int64_t>(n) * n;
    const double* A = a + b * nn;
    double* X = x0 + b * nn;
    double m = 0.0;
    for (int64_t t = threadIdx.x; t < nn; t += blockDim.x) {
        const double v = A[t];
        m = fmax(m, fabs(v));  // fmax drops NaNs like the reference's std::max scan
        if (x0 && X != A) X[t] = v;
    }
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (blockDim.x >> 5); ++w) m = fmax(m, red[w]);
        amax[b] = m;
    }
}

// ---- panel factorisation: one warp per block ---------------------------------------------------------------
// src[b][r] = row of the OLD buffer that ends up in row r after this panel's interchanges.
__global__ void gj_panel_kernel(int n, int j0, int64_t batch, const double* __restrict__ old, double* __restrict__ nw,
                                const double* __restrict__ amax, int* __restrict__ piv, int* __restrict__ src,
                                int* flags, int ldp, int64_t b_base) {
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
    if (b >= batch) return;
    double* P = sm + static_cast<size_t>(warp) * NB * ldp;
    const int64_t nn = static_cast<int64_t>(n) * n;
    const int nbk = min(NB, n - j0);
    const double* O = old + b * nn + static_cast<int64_t>(j0) * n;
    for (int c = 0; c < nbk; ++c)
        for (int r = lane; r < n; r += 32) P[c * ldp + r] = O[static_cast<int64_t>(c) * n + r];
    int* S = src + b * n;
    for (int r = lane; r < n; r += 32) S[r] = r;
    __syncwarp();
    const double tol = 1e-14 * amax[b];
    bool bad = false;
    for (int c = 0; c < nbk; ++c) {
        const int k = j0 + c;
        const double* col = P + c * ldp;
        // first row of maximal modulus among rows >= k (dense_batch.cpp:27-33)
        double best = -1.0;
        int bi = INT_MAX;
        for (int r = k + lane; r < n; r += 32) {
            const double v = fabs(col[r]);
            if (v > best) { best = v; bi = r; }
        }
        // |v| compares like its bit pattern: three integer warp reductions instead of a shuffle tree
        const unsigned long long bits = best < 0.0 ? 0ull : static_cast<unsigned long long>(__double_as_longlong(best));
        const unsigned hi = static_cast<unsigned>(bits >> 32), lo = static_cast<unsigned>(bits);
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        const bool win = (bi != INT_MAX) && hi == mhi && lo == mlo;
        const int p = static_cast<int>(__reduce_min_sync(0xffffffffu, win ? static_cast<unsigned>(bi) : 0xffffffffu));
        const double dkk = col[k];
        const double bestv = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(mhi) << 32) | mlo));
        const bool ok = (dkk == dkk) && (bestv > tol) && p < n;
        const int pp = ok ? p : k;
        if (!ok) bad = true;
        if (lane == 0) {
            piv[b * n + k] = pp;
            const int t = S[k];
            S[k] = S[pp];
            S[pp] = t;
        }
        // interchange rows k and pp inside the panel
        if (lane < nbk && pp != k) {
            double* q = P + lane * ldp;
            const double t = q[k];
            q[k] = q[pp];
            q[pp] = t;
        }
        __syncwarp();
        double rowk[NB];
#pragma unroll
        for (int c2 = 0; c2 < NB; ++c2) rowk[c2] = c2 < nbk ? P[c2 * ldp + k] : 0.0;
        const double pvt = ok ? P[c * ldp + k] : 1.0;
        const double inv = 1.0 / pvt;
        __syncwarp();
        for (int r = lane; r < n; r += 32) {
            if (r == k) {
#pragma unroll
                for (int c2 = 0; c2 < NB; ++c2)
                    if (c2 < nbk) P[c2 * ldp + r] = (c2 == c) ? inv : rowk[c2] * inv;
            } else {
                const double li = P[c * ldp + r] * inv;
#pragma unroll
                for (int c2 = 0; c2 < NB; ++c2)
                    if (c2 < nbk) P[c2 * ldp + r] = (c2 == c) ? -li : fma(-li, rowk[c2], P[c2 * ldp + r]);
            }
        }
        __syncwarp();
    }
    if (bad && lane == 0) atomicMin(flags, static_cast<int>(b_base + b));
    double* W = nw + b * nn + static_cast<int64_t>(j0) * n;
    for (int c = 0; c < nbk; ++c)
        for (int r = lane; r < n; r += 32) W[static_cast<int64_t>(c) * n + r] = P[c * ldp + r];
}

// CTA variant for large blocks (n > 128): the n x NB panel of one block lives in the shared memory of a CTA of
// kPanelCtaWarps warps (rows dealt round-robin to the threads), so the shared-memory-limited occupancy still leaves
// 4x the warps of the one-warp-per-block kernel above to hide the per-pivot latency chain.  Two barriers per pivot:
// after the per-warp pivot candidates are published, and after the row interchange.
constexpr int kPanelCtaWarps = 4;

__global__ void __launch_bounds__(kPanelCtaWarps * 32) gj_panel_cta_kernel(int n, int j0, const double* __restrict__ old,
                                                                            double* __restrict__ nw,
                                                                            const double* __restrict__ amax, int* __restrict__ piv,
                                                                            int* __restrict__ src, int* flags, int ldp,
                                                                            int64_t b_base) {
    extern __shared__ double sm[];
    __shared__ unsigned long long s_val[kPanelCtaWarps];
    __shared__ int s_row[kPanelCtaWarps];
    constexpr int NT = kPanelCtaWarps * 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t b = blockIdx.x;
    double* P = sm;
    const int64_t nn = static_cast<int64_t>(n) * n;
    const int nbk = min(NB, n - j0);
    const double* O = old + b * nn + static_cast<int64_t>(j0) * n;
    for (int c = 0; c < nbk; ++c)
        for (int r = tid; r < n; r += NT) P[c * ldp + r] = O[static_cast<int64_t>(c) * n + r];
    int* S = src + b * n;
    for (int r = tid; r < n; r += NT) S[r] = r;
    const double tol = 1e-14 * amax[b];
    bool bad = false;
    __syncthreads();
    for (int c = 0; c < nbk; ++c) {
        const int k = j0 + c;
        const double* col = P + c * ldp;
        double best = -1.0;
        int bi = INT_MAX;
        for (int r = tid; r < n; r += NT) {
            if (r < k) continue;
            const double v = fabs(col[r]);
            if (v > best || (v == best && r < bi)) { best = v; bi = r; }
        }
        // warp candidate: maximal modulus, lowest row on ties (|v| compares like its bit pattern)
        const unsigned long long bits = best < 0.0 ? 0ull : static_cast<unsigned long long>(__double_as_longlong(best));
        const unsigned hi = static_cast<unsigned>(bits >> 32), lo = static_cast<unsigned>(bits);
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        const bool win = (bi != INT_MAX) && hi == mhi && lo == mlo;
        const unsigned wrow = __reduce_min_sync(0xffffffffu, win ? static_cast<unsigned>(bi) : 0xffffffffu);
        if (lane == 0) {
            s_val[warp] = (static_cast<unsigned long long>(mhi) << 32) | mlo;
            s_row[warp] = static_cast<int>(wrow);
        }
        __syncthreads();
        unsigned long long bv = 0ull;
        int p = INT_MAX;
#pragma unroll
        for (int w = 0; w < kPanelCtaWarps; ++w) {
            const unsigned long long v = s_val[w];
            const int r = s_row[w];
            if (r >= 0 && r < n && (v > bv || (v == bv && r < p))) { bv = v; p = r; }
        }
        const double dkk = col[k];
        const double bestv = __longlong_as_double(static_cast<long long>(bv));
        const bool ok = (dkk == dkk) && (bestv > tol) && p < n;
        const int pp = ok ? p : k;
        if (!ok) bad = true;
        if (tid == 0) {
            piv[b * n + k] = pp;
            const int t = S[k];
            S[k] = S[pp];
            S[pp] = t;
        }
        if (tid < nbk && pp != k) {
            double* q = P + tid * ldp;
            const double t = q[k];
            q[k] = q[pp];
            q[pp] = t;
        }
        __syncthreads();
        double rowk[NB];
#pragma unroll
        for (int c2 = 0; c2 < NB; ++c2) rowk[c2] = c2 < nbk ? P[c2 * ldp + k] : 0.0;
        const double inv = 1.0 / (ok ? rowk[c] : 1.0);
        // every thread eliminates its own rows; row k is rewritten by its owner only, and nobody reads another
        // thread's rows before the next barrier (rowk was copied above -- but the owner of row k must not overwrite
        // it before the others have read it)
        __syncthreads();
        for (int r = tid; r < n; r += NT) {
            if (r == k) {
#pragma unroll
                for (int c2 = 0; c2 < NB; ++c2)
                    if (c2 < nbk) P[c2 * ldp + r] = (c2 == c) ? inv : rowk[c2] * inv;
            } else {
                const double li = P[c * ldp + r] * inv;
#pragma unroll
                for (int c2 = 0; c2 < NB; ++c2)
                    if (c2 < nbk) P[c2 * ldp + r] = (c2 == c) ? -li : fma(-li, rowk[c2], P[c2 * ldp + r]);
            }
        }
        // (the next pivot search reads own rows only; the barrier after the candidates orders the rest)
    }
    if (bad && tid == 0) atomicMin(flags, static_cast<int>(b_base + b));
    __syncthreads();
    double* W = nw + b * nn + static_cast<int64_t>(j0) * n;
    for (int c = 0; c < nbk; ++c)
        for (int r = tid; r < n; r += NT) W[static_cast<int64_t>(c) * n + r] = P[c * ldp + r];
}

// Register variant for n <= 128: lane owns rows lane + 32 t (t < RT), the whole panel lives in registers and
// only the two interchanged rows travel through a shared-memory scratch line per pivot.
template <int RT>
__global__ void __launch_bounds__(128) gj_panel_reg_kernel(int n, int j0, int64_t batch, const double* __restrict__ old,
                                                           double* __restrict__ nw, const double* __restrict__ amax,
                                                           int* __restrict__ piv, int* __restrict__ src, int* flags,
                                                           int64_t b_base, int* __restrict__ dstmap, int* __restrict__ cmscratch) {
    // dstmap != nullptr: LAST panel -- all pivots are known after it, so lane 0 also forms the final column permutation
    // (column j of the work matrix is column dstmap[j] of the inverse), this kernel writes its panel columns straight to
    // their final places in nw (= the destination) and the last update does the same: no separate permutation pass.
    __shared__ double s_scr[4][2][NB];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = static_cast<int64_t>(blockIdx.x) * 4 + warp;
    if (b >= batch) return;
    const int64_t nn = static_cast<int64_t>(n) * n;
    const int nbk = min(NB, n - j0);
    const double* O = old + b * nn + static_cast<int64_t>(j0) * n;
    double a[RT][NB];
#pragma unroll
    for (int c = 0; c < NB; ++c)
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const int r = lane + 32 * t;
            a[t][c] = (c < nbk && r < n) ? O[static_cast<int64_t>(c) * n + r] : 0.0;
        }
    int* S = src + b * n;
    for (int r = lane; r < n; r += 32) S[r] = r;
    __syncwarp();
    const double tol = 1e-14 * amax[b];
    bool bad = false;
    double* scr0 = s_scr[warp][0];
    double* scr1 = s_scr[warp][1];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
        if (c < nbk) {
            const int k = j0 + c;
            double best = -1.0, dkk = 0.0;
            int bi = INT_MAX;
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                const int r = lane + 32 * t;
                const double v = fabs(a[t][c]);
                if (r >= k && r < n && v > best) { best = v; bi = r; }
                if (r == k) dkk = a[t][c];
            }
            const unsigned long long bits = best < 0.0 ? 0ull : static_cast<unsigned long long>(__double_as_longlong(best));
            const unsigned hi = static_cast<unsigned>(bits >> 32), lo = static_cast<unsigned>(bits);
            const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
            const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
            const bool win = (bi != INT_MAX) && hi == mhi && lo == mlo;
            const int p = static_cast<int>(__reduce_min_sync(0xffffffffu, win ? static_cast<unsigned>(bi) : 0xffffffffu));
            const bool nan_diag = __any_sync(0xffffffffu, dkk != dkk);
            const double bestv = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(mhi) << 32) | mlo));
            const bool ok = !nan_diag && (bestv > tol) && p < n;
            const int pp = ok ? p : k;
            if (!ok) bad = true;
            if (lane == 0) {
                piv[b * n + k] = pp;
                const int t = S[k];
                S[k] = S[pp];
                S[pp] = t;
            }
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                const int r = lane + 32 * t;
                if (r == pp) {
#pragma unroll
                    for (int c2 = 0; c2 < NB; ++c2) scr0[c2] = a[t][c2];
                }
                if (r == k) {
#pragma unroll
                    for (int c2 = 0; c2 < NB; ++c2) scr1[c2] = a[t][c2];
                }
            }
            __syncwarp();
            double rowk[NB];
#pragma unroll
            for (int c2 = 0; c2 < NB; ++c2) rowk[c2] = scr0[c2];
            const double inv = 1.0 / (ok ? rowk[c] : 1.0);
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                const int r = lane + 32 * t;
                if (r == pp && pp != k) {
#pragma unroll
                    for (int c2 = 0; c2 < NB; ++c2) a[t][c2] = scr1[c2];
                }
                if (r == k) {
#pragma unroll
                    for (int c2 = 0; c2 < NB; ++c2) a[t][c2] = (c2 == c) ? inv : rowk[c2] * inv;
                } else {
                    const double li = a[t][c] * inv;
#pragma unroll
                    for (int c2 = 0; c2 < NB; ++c2) a[t][c2] = (c2 == c) ? -li : fma(-li, rowk[c2], a[t][c2]);
                }
            }
            __syncwarp();
        }
    }
    if (bad && lane == 0) atomicMin(flags, static_cast<int>(b_base + b));
    if (dstmap) {
        int* dm = dstmap + b * n;
        // cmap = identity pushed through the interchanges in reverse order; dm[cmap[j]] = j
        __shared__ int s_cm[4][128], s_pv[4][128];
        for (int j = lane; j < n; j += 32) {
            s_cm[warp][j] = j;
            s_pv[warp][j] = piv[b * n + j];
        }
        __syncwarp();
        if (lane == 0) {
            // (serial, in shared memory as in gj_colperm_kernel; the pivots were staged by all lanes above)
            for (int k = n - 1; k >= 0; --k) {
                const int p = s_pv[warp][k];
                const int t = s_cm[warp][k];
                s_cm[warp][k] = s_cm[warp][p];
                s_cm[warp][p] = t;
            }
        }
        __syncwarp();
        for (int j = lane; j < n; j += 32) dm[s_cm[warp][j]] = j;
        __syncwarp();
        double* Wf = nw + b * nn;
#pragma unroll
        for (int c = 0; c < NB; ++c) {
            if (c >= nbk) continue;
            double* wc = Wf + static_cast<int64_t>(dm[j0 + c]) * n;
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                const int r = lane + 32 * t;
                if (r < n) wc[r] = a[t][c];
            }
        }
        return;
    }
    double* W = nw + b * nn + static_cast<int64_t>(j0) * n;
#pragma unroll
    for (int c = 0; c < NB; ++c)
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const int r = lane + 32 * t;
            if (c < nbk && r < n) W[static_cast<int64_t>(c) * n + r] = a[t][c];
        }
}

// ---- rank-NB update of the non-panel columns ---------------------------------------------------------------
// CTA = WM warps stacked along the rows, one 32 x 32 DMMA warp tile each, 32 columns per CTA: small CTAs so
// that several are resident per SM and their load -> multiply -> store phases overlap.
template <int WM>
__global__ void __launch_bounds__(WM * 32, (WM <= 2) ? 6 : 4) gj_update_kernel(int n, int j0, const double* __restrict__ old,
                                                                               double* __restrict__ nw, const int* __restrict__ src,
                                                                               const int* __restrict__ dstmap) {
    // dstmap != nullptr (last panel): column c of the work matrix is read / written at column dstmap[c] of nw (= the inverse)
    constexpr int BM = 32 * WM, BN = 32, NT = WM * 32;
    constexpr int LDA = BM + 4;
    __shared__ __align__(16) double As[NB * LDA];  // panel rows of this tile: As[kk][row]
    __shared__ __align__(16) double Bs[BN * LDB];  // gathered pivot rows: Bs[col][kk]
    const int tid = threadIdx.x, lane = tid & 31, wm = tid >> 5;
    const int grp = lane >> 2, tig = lane & 3;
    const int64_t b = blockIdx.z;
    const int64_t nn = static_cast<int64_t>(n) * n;
    const double* O = old + b * nn;
    double* W = nw + b * nn;
    const int* S = src + b * n;
    const int* DM = dstmap ? dstmap + b * n : nullptr;
    const int nbk = min(NB, n - j0);
    const int ncol = n - nbk;  // non-panel columns, index c' -> column c' (< j0) or c' + nbk
    const int row0 = blockIdx.x * BM, cp0 = blockIdx.y * BN;

    // accumulators start from the row-permuted old entries (zero for the pivot rows: those are replaced);
    // these loads are issued first, the operand staging below runs behind them
    int srow[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = row0 + wm * 32 + i * 8 + grp;
        srow[i] = (r < n && (r < j0 || r >= j0 + nbk)) ? S[r] : -1;
    }
    double acc[4][4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int cp = cp0 + j * 8 + 2 * tig + h;
            const int c = cp < j0 ? cp : cp + nbk;
            const double* oc = O + static_cast<int64_t>(c) * n;
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i][j][h] = (cp < ncol && srow[i] >= 0) ? oc[srow[i]] : 0.0;
        }
    // panel tile (already in the new buffer; these columns are not written by this kernel): thread = row,
    // all NB loads issued before the first shared-memory store
    {
        const int r = row0 + tid;  // NT == BM
        double v[NB];
#pragma unroll
        for (int kk = 0; kk < NB; ++kk)
            v[kk] = (kk < nbk && r < n) ? __ldg(W + static_cast<int64_t>(DM ? DM[j0 + kk] : j0 + kk) * n + r) : 0.0;
#pragma unroll
        for (int kk = 0; kk < NB; ++kk) As[kk * LDA + tid] = v[kk];
    }
    // gathered pivot rows: thread = (kk = tid % NB, columns tid / NB + it * NT / NB)
    {
        constexpr int IT = (BN * NB + NT - 1) / NT;
        const int kk = tid & (NB - 1), jb = tid / NB;
        const int ps = (kk < nbk) ? S[j0 + kk] : -1;
        double v[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int cp = cp0 + jb + it * (NT / NB);
            const int c = cp < j0 ? cp : cp + nbk;
            v[it] = (cp < ncol && ps >= 0 && jb + it * (NT / NB) < BN) ? O[static_cast<int64_t>(c) * n + ps] : 0.0;
        }
#pragma unroll
        for (int it = 0; it < IT; ++it)
            if (jb + it * (NT / NB) < BN) Bs[(jb + it * (NT / NB)) * LDB + kk] = v[it];
    }
    __syncthreads();
    const double* as = As + wm * 32 + grp;
    const double* bs = Bs + grp * LDB;
#pragma unroll
    for (int kk = 0; kk < NB; kk += 4) {
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
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int cp = cp0 + j * 8 + 2 * tig + h;
            if (cp >= ncol) continue;
            const int c = cp < j0 ? cp : cp + nbk;
            double* wc = W + static_cast<int64_t>(DM ? DM[c] : c) * n;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = row0 + wm * 32 + i * 8 + grp;
                if (r < n) wc[r] = acc[i][j][h];
            }
        }
}

// ---- final column permutation: inverse[:, j] = W[:, c[j]] ---------------------------------------------------
__global__ void gj_colperm_kernel(int n, const double* __restrict__ w, double* __restrict__ out, const int* __restrict__ piv) {
    extern __shared__ int s_map[];  // [2][n]
    int* cmap = s_map;
    int* dst = s_map + n;
    const int64_t b = blockIdx.x;
    const int64_t nn = static_cast<int64_t>(n) * n;
    if (threadIdx.x == 0) {
        const int* pv = piv + b * n;
        for (int j = 0; j < n; ++j) cmap[j] = j;
        for (int k = n - 1; k >= 0; --k) {  // c = identity after the interchanges in reverse order
            const int p = pv[k];
            const int t = cmap[k];
            cmap[k] = cmap[p];
            cmap[p] = t;
        }
        for (int j = 0; j < n; ++j) dst[cmap[j]] = j;  // column j of W goes to column dst[j]
    }
    __syncthreads();
    const double* Wb = w + b * nn;
    double* Ob = out + b * nn;
    for (int64_t t = threadIdx.x; t < nn; t += blockDim.x) {
        const int j = static_cast<int>(t / n), i = static_cast<int>(t - static_cast<int64_t>(j) * n);
        Ob[static_cast<int64_t>(dst[j]) * n + i] = Wb[t];
    }
}

// ---- single-kernel variant for n <= 128: the block stays in shared memory ---------------------------------------
// Same blocked Gauss-Jordan, but the whole block lives in the shared memory of one CTA (column-major, leading
// dimension = 4 mod 16), so each block is read from and written to HBM exactly once instead of once per panel:
//   per panel: warp 0 factors the 16 pivot columns in registers (as gj_panel_reg_kernel) -> every thread applies the
//   panel's row interchanges to one non-panel column and copies its pivot rows into the right-operand buffer ->
//   all warps update their 8 x 8 tiles in place with DMMA (pivot rows: replaced, other rows: accumulated).
// The column permutation happens on the way out.  Padding to a multiple of 16 is an identity block.
template <int RT>
__global__ void __launch_bounds__(256) gj_smem_kernel(int n, int64_t batch, const double* __restrict__ a_in,
                                                      double* __restrict__ inv_out, int* flags, int64_t b_base) {
    constexpr int NP = 32 * RT;  // padded order (rows lane + 32 t of the panel registers); n <= NP
    constexpr int LDA = NP + 4;
    extern __shared__ __align__(16) double sm[];
    double* A = sm;                       // [NP][LDA] column-major
    double* B1 = A + NP * LDA;            // [NP][LDB]: pivot rows of the non-panel columns, B operand
    double* scr = B1 + NP * LDB;          // [2][NB] interchanged rows of the panel factorisation
    int* s_piv = reinterpret_cast<int*>(scr + 2 * NB);  // [NP]
    int* s_dst = s_piv + NP;                            // [NP]
    __shared__ double s_red[8];
    __shared__ int s_bad;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int grp = lane >> 2, tig = lane & 3;
    const int npad = (n + NB - 1) / NB * NB;  // active order, multiple of NB (<= NP)
    const int64_t nn = static_cast<int64_t>(n) * n;

    for (int64_t blk = blockIdx.x; blk < batch; blk += gridDim.x) {
        const double* Ag = a_in + blk * nn;
        double amax = 0.0;
        for (int t = tid; t < npad * npad; t += 256) {
            const int c = t / npad, r = t - c * npad;
            double v = (r == c) ? 1.0 : 0.0;  // identity padding
            if (r < n && c < n) {
                v = Ag[static_cast<int64_t>(c) * n + r];
                amax = fmax(amax, fabs(v));
            }
            A[c * LDA + r] = v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if (lane == 0) s_red[warp] = amax;
        if (tid == 0) s_bad = 0;
        __syncthreads();
        amax = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) amax = fmax(amax, s_red[w]);
        const double tol = 1e-14 * amax;

        for (int j0 = 0; j0 < npad; j0 += NB) {
            // ---- (a) panel factorisation by warp 0, register resident ----
            if (warp == 0) {
                double p_[RT][NB];
#pragma unroll
                for (int c = 0; c < NB; ++c)
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        const int r = lane + 32 * t;
                        p_[t][c] = r < npad ? A[(j0 + c) * LDA + r] : 0.0;
                    }
                double* scr0 = scr;
                double* scr1 = scr + NB;
                bool bad = false;
#pragma unroll
                for (int c = 0; c < NB; ++c) {
                    const int k = j0 + c;
                    double best = -1.0, dkk = 0.0;
                    int bi = INT_MAX;
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        const int r = lane + 32 * t;
                        const double v = fabs(p_[t][c]);
                        if (r >= k && r < npad && v > best) { best = v; bi = r; }
                        if (r == k) dkk = p_[t][c];
                    }
                    const unsigned long long bits = best < 0.0 ? 0ull : static_cast<unsigned long long>(__double_as_longlong(best));
                    const unsigned hi = static_cast<unsigned>(bits >> 32), lo = static_cast<unsigned>(bits);
                    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
                    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
                    const bool win = (bi != INT_MAX) && hi == mhi && lo == mlo;
                    const int p = static_cast<int>(__reduce_min_sync(0xffffffffu, win ? static_cast<unsigned>(bi) : 0xffffffffu));
                    const bool nan_diag = __any_sync(0xffffffffu, dkk != dkk);
                    const double bestv = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(mhi) << 32) | mlo));
                    // padding pivots (k >= n) are exact ones: never singular
                    const bool ok = !nan_diag && (bestv > tol || k >= n) && p < npad;
                    const int pp = ok ? p : k;
                    if (!ok) bad = true;
                    if (lane == 0) s_piv[k] = pp;
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        const int r = lane + 32 * t;
                        if (r == pp) {
#pragma unroll
                            for (int c2 = 0; c2 < NB; ++c2) scr0[c2] = p_[t][c2];
                        }
                        if (r == k) {
#pragma unroll
                            for (int c2 = 0; c2 < NB; ++c2) scr1[c2] = p_[t][c2];
                        }
                    }
                    __syncwarp();
                    double rowk[NB];
#pragma unroll
                    for (int c2 = 0; c2 < NB; ++c2) rowk[c2] = scr0[c2];
                    const double inv = 1.0 / (ok ? rowk[c] : 1.0);
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        const int r = lane + 32 * t;
                        if (r == pp && pp != k) {
#pragma unroll
                            for (int c2 = 0; c2 < NB; ++c2) p_[t][c2] = scr1[c2];
                        }
                        if (r == k) {
#pragma unroll
                            for (int c2 = 0; c2 < NB; ++c2) p_[t][c2] = (c2 == c) ? inv : rowk[c2] * inv;
                        } else {
                            const double li = p_[t][c] * inv;
#pragma unroll
                            for (int c2 = 0; c2 < NB; ++c2) p_[t][c2] = (c2 == c) ? -li : fma(-li, rowk[c2], p_[t][c2]);
                        }
                    }
                    __syncwarp();
                }
                if (bad && lane == 0) s_bad = 1;
#pragma unroll
                for (int c = 0; c < NB; ++c)
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        const int r = lane + 32 * t;
                        if (r < npad) A[(j0 + c) * LDA + r] = p_[t][c];
                    }
            }
            __syncthreads();
            // ---- (b) row interchanges of the non-panel columns + right operand ----
            const int ncol = npad - NB;
            for (int ci = tid; ci < ncol; ci += 256) {
                const int col = ci < j0 ? ci : ci + NB;
                double* cp = A + col * LDA;
#pragma unroll 4
                for (int c = 0; c < NB; ++c) {
                    const int k = j0 + c, p = s_piv[k];
                    if (p != k) {
                        const double t = cp[k];
                        cp[k] = cp[p];
                        cp[p] = t;
                    }
                }
#pragma unroll
                for (int c = 0; c < NB; ++c) B1[ci * LDB + c] = cp[j0 + c];
            }
            __syncthreads();
            // ---- (c) rank-NB update of the 8 x 8 tiles, in place ----
            const int tr = npad / 8, tc = ncol / 8;
            for (int tile = warp; tile < tr * tc; tile += 8) {
                const int ti = tile % tr, tj = tile / tr;
                const int r0 = ti * 8, ci0 = tj * 8;
                const int cidx = ci0 + 2 * tig;
                const int col0 = cidx < j0 ? cidx : cidx + NB, col1 = (cidx + 1) < j0 ? cidx + 1 : cidx + 1 + NB;
                const bool pivrow = (r0 >= j0 && r0 < j0 + NB);
                double c0 = pivrow ? 0.0 : A[col0 * LDA + r0 + grp];
                double c1 = pivrow ? 0.0 : A[col1 * LDA + r0 + grp];
#pragma unroll
                for (int kk = 0; kk < NB; kk += 4)
                    dmma_8x8x4(c0, c1, A[(j0 + kk + tig) * LDA + r0 + grp], B1[(ci0 + grp) * LDB + kk + tig]);
                A[col0 * LDA + r0 + grp] = c0;
                A[col1 * LDA + r0 + grp] = c1;
            }
            __syncthreads();
        }
        // ---- column permutation on the way out: inverse[:, dst[j]] = W[:, j] ----
        if (tid == 0) {
            int* cmap = reinterpret_cast<int*>(B1);  // scratch
            for (int j = 0; j < npad; ++j) cmap[j] = j;
            for (int k = npad - 1; k >= 0; --k) {
                const int p = s_piv[k];
                const int t = cmap[k];
                cmap[k] = cmap[p];
                cmap[p] = t;
            }
            for (int j = 0; j < npad; ++j) s_dst[cmap[j]] = j;
            if (s_bad) atomicMin(flags, static_cast<int>(b_base + blk));
        }
        __syncthreads();
        if (!s_bad) {
            double* Og = inv_out + blk * nn;
            for (int t = tid; t < npad * npad; t += 256) {
                const int c = t / npad, r = t - c * npad;
                const int dc = s_dst[c];
                if (r < n && dc < n) Og[static_cast<int64_t>(dc) * n + r] = A[c * LDA + r];
            }
        }
        __syncthreads();
    }
}

}  // namespace

// inv may alias a.  Work buffers come from the context's caching allocator.
void launch_gj_invert_batch(hdgb_ctx* ctx, int n, int64_t batch, const double* a, double* inv, int* flags) {
    if (batch <= 0) return;
    if (n <= 128 && tuning().gj_smem) {
        // single kernel, block resident in shared memory
        const int rt = ceil_div(n, 32);
        const int NP = 32 * rt;
        const size_t smem = (static_cast<size_t>(NP) * (NP + 4) + static_cast<size_t>(NP) * LDB + 2 * NB) * sizeof(double) +
                            2 * NP * sizeof(int);
        const int per_sm = std::max<int>(1, static_cast<int>((220 * 1024) / (smem + 1024)));
        const int64_t cap = static_cast<int64_t>(ctx->sm_count) * per_sm;
        const unsigned grid = static_cast<unsigned>(batch < cap ? batch : cap);
        auto launch = [&](auto kern) {
            ensure_dynamic_smem(kern, smem);
            kern<<<grid, 256, smem, ctx->stream>>>(n, batch, a, inv, flags, 0);
        };
        switch (rt) {
            case 1: launch(gj_smem_kernel<1>); break;
            case 2: launch(gj_smem_kernel<2>); break;
            case 3: launch(gj_smem_kernel<3>); break;
            default: launch(gj_smem_kernel<4>); break;
        }
        HDGB_LAUNCH_CHECK(ctx);
        return;
    }
    const int64_t nn = static_cast<int64_t>(n) * n;
    const int steps = (n + NB - 1) / NB;
    DevBuf<double> tmp(static_cast<size_t>(nn) * batch);
    DevBuf<double> amax(static_cast<size_t>(batch));
    DevBuf<int> piv(static_cast<size_t>(batch) * n), src(static_cast<size_t>(batch) * n);
    // n <= 128 (E-bar, additive-Schwarz blocks): the first panel reads the input directly (the prepass
    // only scans for max|A|) and the last panel + update write the inverse's columns at their final places -- no copy
    // pass, no permutation pass.  The ping-pong then ends in inv: x[steps & 1] = inv, the step before it reads tmp.
    // In place (a == inv: the additive-Schwarz and block-Jacobi builds) this works when the number of panels is even: the
    // first panel then reads a = inv and writes tmp, and inv is only overwritten from the second panel on.
    const bool direct = (a != inv || steps % 2 == 0) && n <= 128 && tuning().gj_direct;
    DevBuf<int> dstmap(direct ? 2 * static_cast<size_t>(batch) * n : 0);
    // ping-pong so that the last panel leaves the result in tmp and the column permutation writes inv
    double* x[2];
    x[0] = ((steps % 2 == 0) != direct) ? tmp.p : inv;
    x[1] = ((steps % 2 == 0) != direct) ? inv : tmp.p;
    int64_t done = 0;
    while (done < batch) {  // gridDim.x / z limits
        const int64_t nbt = (batch - done) < 65535 ? (batch - done) : 65535;
        const int64_t off = done * nn;
        gj_prepare_kernel<<<static_cast<unsigned>(nbt), 256, 0, ctx->stream>>>(n, a + off, direct ? nullptr : x[0] + off, amax.p + done);
        HDGB_LAUNCH_CHECK(ctx);
        const int ldp = n | 1;
        const size_t per_warp = static_cast<size_t>(NB) * ldp * sizeof(double);
        int wpc = static_cast<int>((200 * 1024) / per_warp);
        if (wpc < 1) throw Failure(HDGB_ERR_UNSUPPORTED, "lu_invert_batch: block too large for the panel kernel");
        if (wpc > 8) wpc = 8;
        const size_t psm = per_warp * wpc;
        ensure_dynamic_smem(gj_panel_kernel, psm);
        for (int s = 0; s < steps; ++s) {
            const int j0 = s * NB;
            const double* old = (direct && s == 0 ? a : x[s & 1]) + off;
            double* nw = x[(s + 1) & 1] + off;
            int* dm = (direct && s == steps - 1) ? dstmap.p + done * n : nullptr;
            if (n <= 128) {
                const int rt = ceil_div(n, 32);
                const unsigned pg = static_cast<unsigned>(ceil_div(nbt, 4));
                int* pp = piv.p + done * n;
                int* sp = src.p + done * n;
                switch (rt) {
                    case 1: gj_panel_reg_kernel<1><<<pg, 128, 0, ctx->stream>>>(n, j0, nbt, old, nw, amax.p + done, pp, sp, flags, done, dm, dm ? dstmap.p + (batch + done) * n : nullptr); break;
                    case 2: gj_panel_reg_kernel<2><<<pg, 128, 0, ctx->stream>>>(n, j0, nbt, old, nw, amax.p + done, pp, sp, flags, done, dm, dm ? dstmap.p + (batch + done) * n : nullptr); break;
                    case 3: gj_panel_reg_kernel<3><<<pg, 128, 0, ctx->stream>>>(n, j0, nbt, old, nw, amax.p + done, pp, sp, flags, done, dm, dm ? dstmap.p + (batch + done) * n : nullptr); break;
                    default: gj_panel_reg_kernel<4><<<pg, 128, 0, ctx->stream>>>(n, j0, nbt, old, nw, amax.p + done, pp, sp, flags, done, dm, dm ? dstmap.p + (batch + done) * n : nullptr); break;
                }
            } else if (tuning().gj_panel_cta) {
                const size_t csm = per_warp;  // one panel per CTA
                ensure_dynamic_smem(gj_panel_cta_kernel, csm);
                gj_panel_cta_kernel<<<static_cast<unsigned>(nbt), kPanelCtaWarps * 32, csm, ctx->stream>>>(
                    n, j0, old, nw, amax.p + done, piv.p + done * n, src.p + done * n, flags, ldp, done);
            } else
            gj_panel_kernel<<<ceil_div(nbt, wpc), wpc * 32, psm, ctx->stream>>>(n, j0, nbt, old, nw, amax.p + done,
                                                                                 piv.p + done * n, src.p + done * n, flags, ldp, done);
            HDGB_LAUNCH_CHECK(ctx);
            const int nbk = n - j0 < NB ? n - j0 : NB;
            const int ncol = n - nbk;
            if (ncol > 0) {
                int wm = ceil_div(n, 32);
                if (wm > 4) wm = 4;
                dim3 grid(ceil_div(n, 32 * wm), ceil_div(ncol, 32), static_cast<unsigned>(nbt));
                const int* sp = src.p + done * n;
                switch (wm) {
                    case 1: gj_update_kernel<1><<<grid, 32, 0, ctx->stream>>>(n, j0, old, nw, sp, dm); break;
                    case 2: gj_update_kernel<2><<<grid, 64, 0, ctx->stream>>>(n, j0, old, nw, sp, dm); break;
                    case 3: gj_update_kernel<3><<<grid, 96, 0, ctx->stream>>>(n, j0, old, nw, sp, dm); break;
                    default: gj_update_kernel<4><<<grid, 128, 0, ctx->stream>>>(n, j0, old, nw, sp, dm); break;
                }
                HDGB_LAUNCH_CHECK(ctx);
            }
        }
        if (!direct) {
            gj_colperm_kernel<<<static_cast<unsigned>(nbt), 256, 2 * n * sizeof(int), ctx->stream>>>(n, tmp.p + off, inv + off, piv.p + done * n);
            HDGB_LAUNCH_CHECK(ctx);
        }
        done += nbt;
    }
}

}  // namespace hdgb
