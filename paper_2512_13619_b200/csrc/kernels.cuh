// Launcher declarations for the hand-written sm_100a kernels.  Each launcher enqueues on
// ctx->stream and never synchronises.
#pragma once
#include "common.cuh"

namespace hdgb {

// ---- team GEMV (k_gemv.cu) ---------------------------------------------------------------------
// y_b = alpha * A_{b / a_div} * xg_b + beta * z_b   for b in [0, batch)
//   A blocks: rows x cols column-major, stride rows*cols.
//   xg_b: either the contiguous slice x[b*cols .. +cols] (idx == nullptr) or a gather of
//   nslots = cols / width slices of `width` doubles:
//       slot s -> x[ idx[(b / comp) * nslots + s] * (comp*width) + (b % comp) * width ]   (idx < 0: zeros)
//   z (may be nullptr) and y have rows doubles per b.  y may alias z.
struct GemvArgs {
    const double* a = nullptr;
    const double* x = nullptr;
    double* y = nullptr;
    const double* z = nullptr;
    const int* idx = nullptr;
    int rows = 0, cols = 0;
    int64_t batch = 0;
    int width = 0;  // gather slot width (only with idx)
    int comp = 1;   // component interleave of the gather
    int a_div = 1;  // consecutive b sharing one matrix block
    double alpha = 1.0, beta = 0.0;
};
void launch_team_gemv(hdgb_ctx* ctx, const GemvArgs& g);
// Persistent TMA-pipelined variant for large streams (k_stream_gemv.cu); false = shape not handled.
bool launch_stream_gemv(hdgb_ctx* ctx, const GemvArgs& g);

// Process-wide tuning knobs (hdgb_set_tuning): A/B switches for benchmarks and tests.
struct Tuning {
    int use_stream = 1;                  // route large GEMVs through the TMA stream kernel
    int64_t stream_min_elems = 1 << 18;  // below this many matrix entries the team kernel is used
    int stream_packed = 1;               // small items: 16 warps, several items side by side per warp, no shuffle tree
    int stream_packed_max_cols = 32;     // ... for items with at most this many columns
    int64_t stream_packed_stage_bytes = 6144;  // ... bytes per TMA stage of a warp in packed mode
    int gmres_speculate = 1;             // GMRES: enqueue the next step's matvec + preconditioner before waiting for the Hessenberg column
    int poly_fused = 1;                  // polynomial preconditioner: recurrence updates fused into the kernel producing base(K v)
    int overlap_halo = 1;                // domain decomposition: interior rows / elements run while the halo exchange is in flight
    int spin_sync = 1;                   // GMRES: poll an event for the per-iteration Hessenberg column instead of a blocking sync
    int fused_cgs = 0;                   // round-1 register-resident fused CGS2 pass (measured slower: 112 us vs 85 us at cfg2)
    int cgs_stream = 1;                  // CGS2 as three TMA-streamed passes over the basis (k_orth.cu) instead of four
    int local_debug_skip = 0;            // measurement aid: skip phases of the local kernel (1 = E/D_d, 2 = H/G_d/F); results invalid
    int local_nt = 256;                  // threads of the tensor-core local kernel: 256 = two 8-warp CTAs per SM (default); 512 = one 16-warp CTA, all
                                         // 1 + D matrices (scalar) / two component pairs (wide) per point sweep -- measured slower at config 2
                                         // (35.6 vs 33.2 ms per assembly) and equal at config 5 (0.250 vs 0.252 s at hex 16^3)
    int local_nt_wide = 256;             // threads of the streamed local kernel of wide systems (M > 1, pe = 64): 512 = 16 warps, 256 = 8 warps
    int local_ed_stream = 3;             // scalar systems with 64 basis functions per element: E / D_d from a bulk-TMA table ring with fragment-built operands (no operand build phase, no CTA barrier in the point sweep)
    int local_dmma_min_pe = 20;          // local blocks on the tensor-core path from this many basis functions per element
    int local_global_records = 1;        // wide systems: point records in an L2-resident scratch, one launch, E / D_d on DMMA
    int local_dmma_chunked = 0;          // E / D_d on the tensor-core path also in point-chunked sweeps (wide systems)
    int qelim_stages = 2;                // cp.async ring depth of the fused q-elimination product (2 or 3)
    int qelim_split_rows = 1;            // fused q-elimination: one product per output block instead of stacked row blocks
    // generic DMMA GEMM: CTAs of at most 2 x 1 warp tiles (64 x 32 outputs).  Small CTAs, four or more resident per SM, overlap
    // each other's barrier-separated load / multiply phases: config-5 assembly at hex 12^3 99.5 ms with 4 x 3 tiles (one
    // 12-warp CTA per SM at 122 registers), 93.8 with 4 x 1, 93.2 with 2 x 1 (profiles/r02_s3_gemm_tile_ab.txt)
    int gemm_wm_cap = 2;                 // 32-row tiles per CTA of the generic DMMA GEMM (1..4)
    int gemm_wn_cap = 1;                 // 32-column tiles per CTA of the generic DMMA GEMM (1..4)
    int schur_fused = 1;                 // Schur complement as one kernel with E-bar^-1 F-bar kept in shared memory (nfl <= 128)
    int qelim_wn = 1;                    // 32-column tiles per CTA of the fused q-elimination product
    int use_qelim_fused = 1;             // q-elimination as two fused stacked products per component instead of 4 D
    int use_dmma = 1;                    // batched GEMMs on the FP64 tensor-core path (k_gemm_dmma.cu)
    int cgs_evict_first = 0;             // CGS2 passes: Krylov basis copies with an L2 evict-first hint
    int stream_persist_mb = 0;           // stream GEMV: leading MB of every streamed matrix copied with an L2 evict-last hint (experiment)
    int stream_evict_first = 1;          // stream GEMV: matrix copies carry an L2 evict-first hint, so the gathered vector is not pushed out of the L2
    int gj_direct = 1;                   // out-of-place inverses with n <= 128: first panel reads the input, last panel / update write the permuted columns (no copy pass, no permutation pass)
    int gj_smem = 0;                     // n <= 128: blocked Gauss-Jordan in ONE kernel, block resident in shared memory (measured 2-3x slower: latency bound)
    int gj_panel_cta = 0;                // n > 128: panel factored by a 4-warp CTA per block instead of one warp (measured slower at n = 320)
    int use_blocked_gj = 1;              // n > 24: blocked Gauss-Jordan inverse, panel kernel + DMMA updates (k_invert.cu)
    int use_tile_lu = 1;                 // register-tiled Gauss-Jordan for 25 <= n <= 128
    int assemble_budget_kb = 216;        // shared memory for the assembly kernel's point records (smaller: chunked sweeps)
};
Tuning& tuning();

// Update step of the polynomial-preconditioner recurrence (preconditioner.cpp:259-281) applied where the value
// t_i = (base K v)_i is produced, instead of as separate vector kernels over t:
//   kReal : w += a q ;  q -= a t                      (real node, a = 1 / theta)
//   kMid  : s = a q - t ;  w += b s                   (conjugate pair, first half: a = 2 Re, b = 1 / |theta|^2)
//   kLast : q -= a t                                  (conjugate pair, second half)
struct PolyEpi {
    enum Mode { kNone = 0, kReal = 1, kMid = 2, kLast = 3 };
    int mode = kNone;
    double a = 0.0, b = 0.0;
    double* q = nullptr;
    double* w = nullptr;
    double* s = nullptr;
};
__host__ __device__ inline void poly_epilogue(const PolyEpi& e, int64_t i, double t) {
    if (e.mode == PolyEpi::kReal) {
        const double qv = e.q[i];
        e.w[i] = e.a * qv + e.w[i];
        e.q[i] = -e.a * t + qv;
    } else if (e.mode == PolyEpi::kMid) {
        const double sv = e.a * e.q[i] - t;
        e.s[i] = sv;
        e.w[i] += e.b * sv;
    } else {
        e.q[i] = -e.a * t + e.q[i];
    }
}
// the same update for bases that deliver t as a vector (identity, block-Jacobi, caller closures): one kernel
void launch_poly_update(hdgb_ctx* ctx, const PolyEpi& epi, const double* t, int64_t n);

// z_f[i] = ze[e0][l0][i] + ze[e1][l1][i]   (apply_asm scatter as an atomics-free face gather)
// sides = 1 keeps only the owner's (side-0) term: the restricted (RAS) prolongation.
// epi != nullptr: the sum feeds the polynomial update directly and z is not written.
void launch_face_sum(hdgb_ctx* ctx, const double* ze, const int* face_elems, const int* face_lidx,
                     int nf, int mpf, int n_lfe, double* z, int sides = 2, const PolyEpi* epi = nullptr);
// out[e][l][i] = v[elem_faces[e][l]][i]  (gather_element_trace)
void launch_gather_element_trace(hdgb_ctx* ctx, const double* v, const int* elem_faces, int ne,
                                 int n_lfe, int mpf, double* out);
// out[f][s][i] = x[nbr[f][s]][i] or 0 (gather_extended)
void launch_gather_extended(hdgb_ctx* ctx, const double* x, const int* nbr, int nf, int nb, int mpf,
                            double* out);

// ---- vector kernels (k_vec.cu) -----------------------------------------------------------------
// out[j] = sum_i V[j*ldv + i] * w[i], j < nvec.  Deterministic two-stage reduction.
// If sqrt_last is set the last entry is replaced by its square root (norms).
void launch_multi_dot(hdgb_ctx* ctx, const double* V, int64_t ldv, int nvec, const double* w, int64_t n,
                      double* out /*device nvec*/, double* partial /*device workspace*/, bool sqrt_last = false);
size_t multi_dot_workspace_doubles(int64_t n, int nvec);
// CGS2 middle step fused: w -= V c ; d = V^T w in one pass over V.  false = nvec too large (use the two kernels).
bool launch_multi_axpy_dot(hdgb_ctx* ctx, const double* V, int64_t ldv, int nvec, const double* c, double* w, int64_t n,
                           double* d_out, double* partial);
// CGS2 as three streaming passes over the basis (k_orth.cu).  mode 0: out[0..nvec) = V^T w;  mode 1: w -= V coef,
// out[0..nvec) = V^T w, out[nvec] = ||w||^2;  mode 2: w -= V coef, out[0] = ||w||^2;  mode 3: w = (w - V coef) * s with
// s = 1/sqrt(t), t = coef[nvec] - sum coef[j]^2, out[0] = max(t, 0).  `work` = cgs_workspace_doubles() doubles, zeroed once.
constexpr int kOrthMaxVec = 56;  // 7 columns per consumer warp; two stages of 51 columns fit shared memory (restart 50)
size_t cgs_workspace_doubles(hdgb_ctx* ctx);
bool cgs_pass_supported(const double* V, int64_t ldv, int nvec, const double* w, int64_t n);
void launch_cgs_pass(hdgb_ctx* ctx, int mode, const double* V, int64_t ldv, int nvec, double* w, int64_t n, const double* coef,
                     double* out, double* work);
// w[i] += sign * sum_j c[j] * V[j*ldv + i]  (ascending j).  If norm2_out != nullptr, also reduces
// sum_i w_new[i]^2 into *norm2_out (device) using `partial`.
void launch_multi_axpy(hdgb_ctx* ctx, const double* V, int64_t ldv, int nvec, const double* c /*device*/,
                       double sign, double* w, int64_t n, double* norm2_out, double* partial);
// out[i] = w[i] * s where s = (*dev_scalar is used as: mode 0: 1/sqrt(v), mode 1: 1/v, mode 2: v)
void launch_scale_dev(hdgb_ctx* ctx, const double* w, const double* dev_scalar, int mode, double* out, int64_t n);
// y = a*x + b*y
void launch_axpby(hdgb_ctx* ctx, double a, const double* x, double b, double* y, int64_t n);
// out = a*x + b*y (out may alias)
void launch_lincomb(hdgb_ctx* ctx, double a, const double* x, double b, const double* y, double* out, int64_t n);
// polynomial-preconditioner fused updates (preconditioner.cpp:264-278)
//   real:  w += inv*q ;  (after op)  q -= inv*t
//   pair:  s = 2a*q - t ; w += inv*s
void launch_poly_pair_mid(hdgb_ctx* ctx, double two_a, double inv, const double* q, const double* t,
                          double* s, double* w, int64_t n);
// flags[1] |= 1 if any entry is non-finite
void launch_check_finite(hdgb_ctx* ctx, const double* v, int64_t n, int* flags);
void launch_fill(hdgb_ctx* ctx, double* v, double value, int64_t n);
// sum of squares (device scalar out[0]); deterministic
void launch_sumsq(hdgb_ctx* ctx, const double* v, int64_t n, double* out, double* partial);

// ---- dense batch kernels (k_dense.cu) ----------------------------------------------------------
// Explicit inverses; flags[0] = min(flags[0], first singular b).  a and inv may alias.
void launch_lu_invert_batch(hdgb_ctx* ctx, int n, int64_t batch, const double* a, double* inv, int* flags);
// Blocked Gauss-Jordan with DMMA rank-16 updates (k_invert.cu), any n; same contract.
void launch_gj_invert_batch(hdgb_ctx* ctx, int n, int64_t batch, const double* a, double* inv, int* flags);
// C_b = alpha * op(A_b) * B_b + beta * C_b ; a_batch / b_batch == 1 broadcast.
void launch_gemm_batch(hdgb_ctx* ctx, int m, int n, int k, const double* a, int64_t a_stride, bool trans_a,
                       const double* b, int64_t b_stride, double* c, int64_t c_stride, int64_t batch,
                       double alpha, double beta);

// DMMA (FP64 tensor core) batched GEMM, k_gemm_dmma.cu; output column j -> (j / c_colw) * c_colstride + j % c_colw
// (c_colw <= 0: identity).
void launch_gemm_dmma(hdgb_ctx* ctx, int m, int n, int k, const double* a, int64_t a_stride, const double* b,
                      int64_t b_stride, double* c, int64_t c_stride, int64_t batch, double alpha, double beta,
                      int c_colw = 0, int c_colstride = 0, const double* c_in = nullptr);

// Fused q-elimination: [C0; C1] -= sum_t [A0_t; A1_t] B_t (k_gemm_dmma.cu); false = shape not supported.
bool launch_qelim_fused(hdgb_ctx* ctx, int m0, int m1, int n, int k, int nterm, const double* const a0[3], int64_t a0_stride,
                        const double* const a1[3], int64_t a1_stride, const double* const b[3], int64_t b_stride, double* c0,
                        int64_t c0_stride, double* c1, int64_t c1_stride, int64_t batch, int c_colw = 0, int c_colstride = 0);

// Fused Schur complement K = J - H (E^-1 F), T = E^-1 F kept in shared memory (k_gemm_dmma.cu); false = shape not supported.
bool launch_schur_fused(hdgb_ctx* ctx, int npe, int nfl, const double* einv, int64_t s_ee, const double* f, const double* h,
                        int64_t s_ef, const double* j, double* k, int64_t s_ff, int64_t batch);

// ---- shared host helpers (api_core.cu) ------------------------------------------------------------
void reset_flags(hdgb_ctx* c);
void read_flags(hdgb_ctx* c, int* singular_index, int* nonfinite);
// lu_invert_batch on device pointers; throws Failure(code) carrying the lowest singular batch index.
void device_lu_invert(hdgb_ctx* c, int n, int64_t batch, const double* a, double* inv, const char* context,
                      hdgb_status code);

}  // namespace hdgb
