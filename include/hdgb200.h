/* hdgb200.h — C ABI of the B200-native HDG solver hot path (libhdgb200.so).
 *
 * The reference (hdgkit, /root/reference/proj) has no FFI: its boundary is the C++ free-function
 * API in namespace hdg (proj/include/hdg/{dense_batch,local_ops,face_matrix,preconditioner,gmres,
 * newton}.hpp).  Each entry point below replaces one of those functions and cites it.  Signatures
 * use only plain pointers, sizes and POD structs; there are no torch / STL types.  The C++ header
 * layer include/hdgb200.hpp (namespace hdg::b200) re-creates the reference's own names, option structs and
 * exception hierarchy on top of this ABI, and INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Conventions
 *  - All floating-point data are FP64.  Dense blocks are column-major and stored back to back
 *    exactly like hdg::DenseBatch (dense_batch.hpp:12-34): entry (r,c) of block b lives at
 *    data[b*rows*cols + c*rows + r].
 *  - Vector / matrix arguments documented "host or device" may point to either; the library
 *    detects which (cudaPointerGetAttributes) and stages host buffers through pinned memory on
 *    the context's stream.  Everything documented "device" must be device memory.
 *  - Every function returns an hdgb_status.  On failure hdgb_last_error(ctx) holds a message and
 *    hdgb_last_error_index(ctx) the offending batch index (element or face id) where the
 *    reference's exception carries one (errors.hpp:16-23 SingularBlock::index).
 *  - There is NO CPU fallback: with no CUDA device hdgb_ctx_create fails with HDGB_ERR_CUDA.
 */
#ifndef HDGB200_H
#define HDGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hdgb_status {
    HDGB_OK = 0,
    HDGB_ERR_GENERIC = 1,              /* hdg::Error                      (errors.hpp:10-13)   */
    HDGB_ERR_SINGULAR_BLOCK = 2,       /* hdg::SingularBlock              (errors.hpp:17-23)   */
    HDGB_ERR_SINGULAR_MASS = 3,        /* hdg::SingularMass               (errors.hpp:63-67)   */
    HDGB_ERR_SINGULAR_LOCAL_SOLVE = 4, /* hdg::SingularLocalSolve         (errors.hpp:70-74)   */
    HDGB_ERR_NONFINITE_STATE = 5,      /* hdg::NonFiniteState             (errors.hpp:76-79)   */
    HDGB_ERR_NAN_DETECTED = 6,         /* hdg::NaNDetected                (errors.hpp:81-84)   */
    HDGB_ERR_LINE_SEARCH_FAILED = 7,   /* hdg::LineSearchFailed           (errors.hpp:92-98)   */
    HDGB_ERR_DIMENSION_MISMATCH = 8,   /* hdg::DimensionMismatch          (errors.hpp:25-28)   */
    HDGB_ERR_INCONSISTENT_DIMENSIONS = 9, /* hdg::InconsistentDimensions  (errors.hpp:30-34)   */
    HDGB_ERR_TOO_LARGE_FOR_DENSE = 10, /* hdg::TooLargeForDense           (errors.hpp:86-90)   */
    HDGB_ERR_IO = 11,                  /* hdg::IoError                    (errors.hpp:100-103) */
    HDGB_ERR_INVALID_MESH = 12,        /* InvalidResolution / DegenerateDomain / InvertedElement */
    HDGB_ERR_UNSUPPORTED = 13,         /* UnsupportedOrder / UnsupportedDegree / unknown model  */
    HDGB_ERR_CUDA = 14                 /* CUDA runtime failure or no device (no CPU fallback)   */
} hdgb_status;

typedef struct hdgb_ctx hdgb_ctx;         /* device, stream, workspaces, last error            */
typedef struct hdgb_disc hdgb_disc;       /* mesh + master element + geometry + local factors  */
typedef struct hdgb_model hdgb_model;     /* PDE model (device functor tag + parameters)       */
typedef struct hdgb_state hdgb_state;     /* hdg::StateFields on the device                    */
typedef struct hdgb_ops hdgb_ops;         /* hdg::ElementOperators on the device               */
typedef struct hdgb_matrix hdgb_matrix;   /* hdg::FaceBlockMatrix on the device                */
typedef struct hdgb_precond hdgb_precond; /* hdg::Preconditioner on the device                 */

/* ---- context ------------------------------------------------------------------------------- */
hdgb_status hdgb_ctx_create(int device, hdgb_ctx** out);
void hdgb_ctx_destroy(hdgb_ctx* ctx);
const char* hdgb_last_error(const hdgb_ctx* ctx);
int64_t hdgb_last_error_index(const hdgb_ctx* ctx);
/* Use an existing CUDA stream (cudaStream_t as void*) for all subsequent launches. */
hdgb_status hdgb_ctx_set_stream(hdgb_ctx* ctx, void* cuda_stream);
void* hdgb_ctx_stream(hdgb_ctx* ctx);
hdgb_status hdgb_ctx_synchronize(hdgb_ctx* ctx);
/* Number of kernel launches issued through this context since the last reset (bench.py's
 * gpu_launches claim is read from here). */
int64_t hdgb_ctx_launch_count(const hdgb_ctx* ctx);
void hdgb_ctx_reset_launch_count(hdgb_ctx* ctx);
const char* hdgb_version(void);
/* Process-wide kernel-selection knobs for A/B measurements and tests (defaults in csrc/kernels.cuh):
 *   GEMV:        "use_stream" (TMA stream kernel for large GEMVs), "stream_min_elems", "stream_packed" (several
 *                small items per warp pass), "stream_packed_max_cols", "stream_packed_stage_bytes",
 *                "stream_evict_first" (L2 evict-first hint on the matrix stream), "stream_persist_mb" (experiment, off);
 *   dense:       "use_dmma" (FP64 tensor-core GEMM / local blocks), "use_qelim_fused", "qelim_split_rows",
 *                "qelim_wn", "qelim_stages", "gemm_wm_cap", "gemm_wn_cap", "schur_fused" (one-kernel Schur complement), "use_blocked_gj" (blocked Gauss-Jordan inverse),
 *                "gj_direct" (no copy / permutation passes, n <= 128), "gj_smem", "gj_panel_cta",
 *                "use_tile_lu" (register-tiled Gauss-Jordan, n <= 128, when the blocked one is off);
 *   assembly:    "local_ed_stream" (hex p = 3: bit 0 = E / D_d, bit 1 = H / G_d / F / J through the bulk-TMA table ring,
 *                bit 2 = stage copies split in 4-row pieces), "local_nt", "local_nt_wide", "local_dmma_min_pe",
 *                "local_global_records", "local_dmma_chunked", "local_debug_skip" (measurement: phases left out),
 *                "assemble_budget_kb";
 *   GMRES:       "fused_cgs", "cgs_stream", "cgs_evict_first", "spin_sync", "poly_fused" (polynomial recurrence updates as
 *                epilogues), "gmres_speculate" (next Arnoldi step's operator applications enqueued before the host reads the column);
 *   multi-GPU:   "overlap_halo" (interior rows / elements computed while the halo exchange is in flight).
 * Returns non-zero for an unknown key.  Results do not depend on them beyond rounding. */
int hdgb_set_tuning(const char* key, int64_t value);
/* Caching-allocator diagnostics: device allocations / frees issued so far (no reference counterpart; the
 * reference allocates std::vector storage per call, newton.cpp:76-88). */
void hdgb_pool_stats(int64_t* device_allocs, int64_t* device_frees);

/* ---- A0-A2: batched dense kernels (dense_batch.hpp:36-51) ---------------------------------- */
/* lu_invert_batch (dense_batch.cpp:77-99): explicit inverses by partial-pivot LU; a pivot not
 * above 1e-14*max|A_b| makes block b singular -> HDGB_ERR_SINGULAR_BLOCK with the LOWEST bad b. */
hdgb_status hdgb_lu_invert_batch(hdgb_ctx* ctx, int n, int batch, const double* a /*host|device*/,
                                 double* inv /*host|device*/);
/* gemm_batch (dense_batch.cpp:101-136): C_b = op(A_b) B_b, either side may broadcast (batch 1). */
hdgb_status hdgb_gemm_batch(hdgb_ctx* ctx, int a_rows, int a_cols, int a_batch, const double* a,
                            int b_rows, int b_cols, int b_batch, const double* b, int transpose_a,
                            double* c);
/* gemv_strided_batch (dense_batch.cpp:138-160): y_b (+)= A_b x_b. */
hdgb_status hdgb_gemv_strided_batch(hdgb_ctx* ctx, int rows, int cols, int batch, const double* a,
                                    const double* x, double* y, int accumulate);

/* ---- discretisation: mesh, master element, geometry, local factors ------------------------- */
typedef enum hdgb_shape {
    HDGB_QUAD = 0, /* reference's only shape (mesh.hpp:24-39, basis.hpp:44-67)                  */
    HDGB_HEX = 1,
    HDGB_TRI = 2,
    HDGB_TET = 3
} hdgb_shape;

typedef struct hdgb_dims {
    int dim;      /* space dimension D (2|3)                                                   */
    int shape;    /* hdgb_shape                                                                */
    int degree;   /* polynomial degree k                                                       */
    int n_comp;   /* M, components per node (1 in the reference)                               */
    int ne, nf;   /* elements, faces                                                           */
    int n_lfe;    /* local faces per element (4 quad, 6 hex, 3 tri, 4 tet)                     */
    int n_orient; /* distinct relative face orientations tabulated (2 in 2D)                   */
    int pe, pf;   /* scalar basis functions per element / face                                 */
    int qe, qf;   /* quadrature points per element / face                                      */
    int nv;       /* mesh vertices                                                             */
} hdgb_dims;

/* Structured meshes of the box [lo, hi]^D: build_structured_quad (mesh.cpp:18-107) and its hex
 * / triangle / tetrahedron analogues, followed by gauss_rule(quad_points or k+2)
 * (study.cpp:69-70), tabulate_basis (basis.cpp:144-201), compute_geometry (mesh.cpp:109-182) and
 * precompute_local_factors (local_ops.cpp:252-349, device kernels).  jitter > 0 displaces interior
 * vertices by at most jitter*h with the given seed (synthetic unstructured-like meshes).
 * ctx == NULL builds a HOST-ONLY discretisation (mesh, master element, geometry tables readable
 * through hdgb_disc_get_*; no device state, no local factors): setup-time code needs no GPU, every
 * operator below does. */
hdgb_status hdgb_disc_create_structured(hdgb_ctx* ctx, int shape, int n, int degree, int n_comp,
                                        int quad_points, const double* lo, const double* hi,
                                        double jitter, uint64_t seed, hdgb_disc** out);
/* Generic mesh: element vertex lists (ne x verts-per-element, int32) and vertex coordinates
 * (nv x dim); connectivity, orientation flags and boundary tags (all boundary faces tag 1 unless
 * boundary_tag_fn data is supplied later) are derived. */
hdgb_status hdgb_disc_create_from_mesh(hdgb_ctx* ctx, int shape, int degree, int n_comp,
                                       int quad_points, int ne, int nv, const int32_t* elem_verts,
                                       const double* vertex_coords, hdgb_disc** out);
void hdgb_disc_destroy(hdgb_disc* d);
hdgb_status hdgb_disc_dims(const hdgb_disc* d, hdgb_dims* out);
/* Copies a named table to the host (tests compare these bit-for-bit with the reference's
 * Mesh2D / BasisTab / GeomFactors / LocalFactors).  Returns the element count through *n when
 * out == NULL.  Names: see DESIGN.md "table names". */
hdgb_status hdgb_disc_get_f64(const hdgb_disc* d, const char* name, double* out, int64_t cap, int64_t* n);
hdgb_status hdgb_disc_get_i32(const hdgb_disc* d, const char* name, int32_t* out, int64_t cap, int64_t* n);
/* Overrides boundary tags (nf int32, 0 = interior face kept as is). */
hdgb_status hdgb_disc_set_boundary_tags(hdgb_disc* d, const int32_t* tags);

/* ---- PDE model (models.hpp:27-50) ---------------------------------------------------------- */
typedef enum hdgb_model_kind {
    HDGB_MODEL_POISSON = 0,   /* poisson_model  (models.cpp:9-30)   params: tau                 */
    HDGB_MODEL_BURGERS = 1,   /* burgers_model  (models.cpp:32-61)  params: nu, tau             */
    HDGB_MODEL_CONVDIFF = 2,  /* convdiff_model (models.cpp:63-93)  params: c[3], kappa, tau|-1 */
    HDGB_MODEL_ELASTICITY = 3,/* linear elasticity, M = D (PAPER.md 5.3) params: lambda, mu, tau */
    HDGB_MODEL_REACTION = 4,  /* Poisson + cubic reaction u^3 (test_newton.cpp:80-99 analogue)  */
    HDGB_MODEL_NAVIER_STOKES = 5 /* compressible NS, M = D + 2 (PAPER.md 5.5-5.7) params: gamma, mu, Pr, tau */
} hdgb_model_kind;

/* The reference's PdeModel is a bundle of host std::function callbacks evaluated at every
 * quadrature point; device code cannot call those, so a model here is a device functor tag plus
 * parameters, and the x-only callbacks (forcing, Dirichlet data) are tabulated ONCE at the
 * quadrature points: forcing_q[(e*qe+g)*M + m], dirichlet_q[(f*qf+g)*M + m] (host arrays, may be
 * NULL = 0).  exact/initial callbacks stay host-side (C++ layer). */
hdgb_status hdgb_model_create(hdgb_ctx* ctx, const hdgb_disc* d, int kind, const double* params,
                              int n_params, const double* forcing_q, const double* dirichlet_q,
                              hdgb_model** out);
void hdgb_model_destroy(hdgb_model* m);

/* ---- state (local_ops.hpp:16-23) ----------------------------------------------------------- */
hdgb_status hdgb_state_create(hdgb_ctx* ctx, const hdgb_disc* d, hdgb_state** out); /* zeros   */
void hdgb_state_destroy(hdgb_state* s);
/* name: "u" (M*pe*ne), "uhat" (M*pf*nf), "q0".."q2" (M*pe*ne) */
hdgb_status hdgb_state_set(hdgb_state* s, const char* name, const double* src /*host|device*/);
hdgb_status hdgb_state_get(const hdgb_state* s, const char* name, double* dst /*host|device*/);
double* hdgb_state_ptr(hdgb_state* s, const char* name); /* device pointer */

/* ---- A3-A6: local operators (local_ops.hpp:73-101) ------------------------------------------ */
typedef struct hdgb_time {
    double dt;            /* <= 0: steady (TimeContext::dt empty, local_ops.hpp:67-70)          */
    const double* u_prev; /* host|device, M*pe*ne; required iff dt > 0                          */
} hdgb_time;

/* compute_q (local_ops.cpp:367-374) */
hdgb_status hdgb_compute_q(hdgb_disc* d, hdgb_state* s);
/* assemble_element_operators (local_ops.cpp:376-430): quadrature assembly + static condensation.
 * keep_raw != 0 keeps the uncondensed blocks (test oracles, local_ops.cpp:420-428). */
hdgb_status hdgb_assemble_element_operators(hdgb_disc* d, const hdgb_model* m, hdgb_state* s,
                                            const hdgb_time* t, int keep_raw, hdgb_ops** out);
/* ElementOperators (local_ops.hpp:40-62) from caller data (host|device; NULL = zeros): lets a caller that holds the
 * reference's value-type operators hand them to assemble_global / build_asm / recover_local. */
hdgb_status hdgb_ops_create(hdgb_disc* d, const double* kbar, const double* ebar_inv, const double* fbar,
                            const double* hbar, const double* rbar, const double* ru, const double* ruhat_e,
                            hdgb_ops** out);
void hdgb_ops_destroy(hdgb_ops* o);
/* name: kbar, ebar_inv, fbar, hbar, rbar, ru, ruhat_e, and with keep_raw: e_raw, f_raw, h_raw,
 * j_raw, d_raw0.., g_raw0.. */
hdgb_status hdgb_ops_get(const hdgb_ops* o, const char* name, double* dst /*host*/, int64_t cap, int64_t* n);
double* hdgb_ops_ptr(hdgb_ops* o, const char* name);
/* assemble_residual (local_ops.cpp:432-450) + residual_norm (:245-250).  trace / interior may be
 * NULL; *norm receives the stacked 2-norm. */
hdgb_status hdgb_assemble_residual(hdgb_disc* d, const hdgb_model* m, hdgb_state* s,
                                   const hdgb_time* t, double* trace /*host|device*/,
                                   double* interior /*host|device*/, double* norm /*host*/);
/* gather_element_trace (local_ops.cpp:351-365) */
hdgb_status hdgb_gather_element_trace(hdgb_disc* d, const double* face_values, double* out);
/* recover_local (local_ops.cpp:452-460), taking the FACE-major duhat (gather fused). */
hdgb_status hdgb_recover_local(hdgb_disc* d, const hdgb_ops* o, const double* duhat, double* du);

/* ---- A7-A8: global face-block operator (face_matrix.hpp:26-61) ------------------------------ */
/* assemble_global (face_matrix.cpp:11-61): rhs receives M*pf*nf values (host|device, may be NULL;
 * the matrix keeps its own device copy, see hdgb_matrix_rhs). */
hdgb_status hdgb_assemble_global(hdgb_disc* d, const hdgb_ops* o, hdgb_matrix** out, double* rhs);
/* Builds a device matrix from host data in FaceBlockMatrix layout (read_matrix, face_matrix.cpp:
 * 169-197 parses the .hdgk file on the C++ side and lands here). */
hdgb_status hdgb_matrix_create(hdgb_ctx* ctx, int m, int pf, int n_lfe, int nf,
                               const int64_t* neighbor /*host nf*nb*/, const double* blocks /*host|device*/,
                               hdgb_matrix** out);
void hdgb_matrix_destroy(hdgb_matrix* k);
/* m, pf, n_lfe, nf */
hdgb_status hdgb_matrix_dims(const hdgb_matrix* k, int* out4);
hdgb_status hdgb_matrix_get_neighbor(const hdgb_matrix* k, int64_t* out /*host nf*nb*/);
hdgb_status hdgb_matrix_get_blocks(const hdgb_matrix* k, double* out /*host|device*/);
double* hdgb_matrix_blocks_ptr(hdgb_matrix* k);
double* hdgb_matrix_rhs(hdgb_matrix* k); /* device, may be NULL */
/* block_matvec (face_matrix.cpp:83-107): y_f = K_f [x_nbr(f,0..nb-1)]; gather fused, no scratch. */
hdgb_status hdgb_block_matvec(hdgb_matrix* k, const double* x /*host|device*/, double* y /*host|device*/);
/* gather_extended (face_matrix.cpp:63-81), for tests. */
hdgb_status hdgb_gather_extended(hdgb_matrix* k, const double* x, double* out);
/* write_matrix / read_matrix (face_matrix.cpp:149-197): the .hdgk dump, byte-compatible. */
hdgb_status hdgb_matrix_write(hdgb_matrix* k, const double* rhs /*host|device*/, const char* path);
hdgb_status hdgb_matrix_read(hdgb_ctx* ctx, const char* path, hdgb_matrix** out, double* rhs /*host, may be NULL*/);

/* ---- A9-A12: preconditioners (preconditioner.hpp:15-76) ------------------------------------- */
typedef enum hdgb_precond_kind {
    HDGB_PC_IDENTITY = 0, /* PrecondKind::Identity (preconditioner.hpp:15)                       */
    HDGB_PC_BJ = 1,       /* PrecondKind::BJ                                                      */
    HDGB_PC_ASM = 2,      /* PrecondKind::ASM: both sides summed on a shared face (:92-103)       */
    HDGB_PC_RAS = 3       /* restricted additive Schwarz: same element-patch solves as ASM, but a
                           * shared face takes only its owner's (side-0 element's) correction.
                           * Not in the reference: parity unpinned.         */
} hdgb_precond_kind;

typedef enum hdgb_poly_kind {
    HDGB_POLY_GMRES = 0,    /* harmonic-Ritz / Leja GMRES polynomial (preconditioner.cpp:119-283) */
    HDGB_POLY_CHEBYSHEV = 1 /* Chebyshev roots on the real interval spanned by the Ritz estimates,
                             * Leja-ordered, applied by the same product recurrence.  Not in the
                             * reference: parity unpinned.                                          */
} hdgb_poly_kind;

typedef struct hdgb_precond_spec {
    int kind;          /* hdgb_precond_kind, default BJ      (newton.hpp:24-29 PrecondSpec)       */
    int poly_degree;   /* 0 = none */
    uint64_t ritz_seed;/* 12345 */
    int ritz_per_restart;
    int poly_kind;     /* hdgb_poly_kind, default GMRES polynomial */
} hdgb_precond_spec;
void hdgb_precond_spec_default(hdgb_precond_spec* spec);

/* build_preconditioner (newton.cpp:30-52): build_bj (preconditioner.cpp:30-46) | build_asm
 * (:54-84, needs ops + disc) and, for poly_degree > 0, compute_harmonic_ritz (:119-205) on
 * v -> base(K v) followed by leja_order (:207-244).  ops/d may be NULL for IDENTITY and BJ. */
hdgb_status hdgb_build_preconditioner(hdgb_matrix* k, const hdgb_ops* o, hdgb_disc* d,
                                      const hdgb_precond_spec* spec, hdgb_precond** out);
void hdgb_precond_destroy(hdgb_precond* p);
/* name: bj_inv, asm_inv; ritz -> interleaved (re, im) in Leja order */
hdgb_status hdgb_precond_get(const hdgb_precond* p, const char* name, double* dst /*host*/, int64_t cap, int64_t* n);
/* Overrides the Ritz values (interleaved re/im, already ordered) — used to test apply_poly
 * against the oracle with identical interpolation nodes. */
hdgb_status hdgb_precond_set_ritz(hdgb_precond* p, const double* reim, int count);
/* make_base_apply (preconditioner.cpp:285-299): apply_bj (:48-52) / apply_asm (:86-105). */
hdgb_status hdgb_precond_apply_base(hdgb_precond* p, const double* y, double* z);
/* make_preconditioner_apply (preconditioner.cpp:301-308) incl. apply_poly (:246-283). */
hdgb_status hdgb_precond_apply(hdgb_precond* p, hdgb_matrix* k, const double* y, double* z);
int64_t hdgb_precond_inner_ops(const hdgb_precond* p); /* SolveReport::n_inner_prec_ops */

/* The reference's per-function preconditioner API (preconditioner.hpp:31-76), one entry point each.
 * hdgb_build_preconditioner above is newton.cpp:30-52 (which calls these); the functions below are for
 * callers that drive the pieces themselves, as the reference's tests do. */
/* build_bj (preconditioner.cpp:30-46): inverts the diagonal face blocks; SingularBlock(face). */
hdgb_status hdgb_build_bj(hdgb_matrix* k, hdgb_precond** out);
/* apply_bj (preconditioner.cpp:48-52). */
hdgb_status hdgb_apply_bj(hdgb_precond* p, const double* y /*host|device*/, double* z /*host|device*/);
/* build_asm (preconditioner.cpp:54-84): from the element operators and the mesh alone (no K needed: the two-sided
 * diagonal sub-block sums are formed from K-bar, side 0 first, :59-75); SingularBlock(element). */
hdgb_status hdgb_build_asm(const hdgb_ops* o, hdgb_disc* d, hdgb_precond** out);
/* apply_asm (preconditioner.cpp:86-105). */
hdgb_status hdgb_apply_asm(hdgb_precond* p, const double* y, double* z);
/* A Preconditioner (preconditioner.hpp:19-29) from caller data: kind, the inverse blocks of that kind (bj_inv:
 * mpf^2 per face | asm_inv: nfl^2 per element, needs d | NULL for identity; host|device) and optional Ritz values
 * (interleaved re/im in application order). */
hdgb_status hdgb_precond_create(hdgb_ctx* ctx, int kind, int mpf, int nf, hdgb_disc* d, const double* inv,
                                const double* ritz_reim, int n_ritz, hdgb_precond** out);

/* A linear operator as a C callback on DEVICE vectors of n doubles (the reference's LinearOp / OpFn closures,
 * preconditioner.hpp:50, gmres.hpp:43): out = op(in).  The callback must enqueue its work on hdgb_ctx_stream(ctx)
 * or synchronise before returning; in and out never alias.  Non-zero return = failure (-> HDGB_ERR_GENERIC). */
typedef int (*hdgb_op_fn)(void* user, const double* in, double* out, int64_t n);
/* compute_harmonic_ritz (preconditioner.cpp:119-205) of an arbitrary operator: seeded start vector, MGS Arnoldi
 * on the device, harmonic correction + eigenvalues + Leja order on the host.  out_reim: 2*degree doubles. */
hdgb_status hdgb_compute_harmonic_ritz(hdgb_ctx* ctx, hdgb_op_fn op, void* user, int64_t n_dof, int degree,
                                       uint64_t seed, double* out_reim, int* n_out);
/* apply_poly (preconditioner.cpp:246-283): z = poly(base K) base y with p's Ritz values; base_apply == NULL uses
 * p's own base (make_base_apply, :285-299).  *inner_ops (may be NULL) is incremented by the operator count. */
hdgb_status hdgb_apply_poly(hdgb_precond* p, hdgb_op_fn base_apply, void* user, hdgb_matrix* k, const double* y,
                            double* z, int64_t* inner_ops);
/* leja_order (preconditioner.cpp:207-244) on interleaved (re, im); returns count in *n_out. */
hdgb_status hdgb_leja_order(const double* reim, int n, double* out_reim, int* n_out);
/* Harmonic Ritz values of a small dense Hessenberg-type matrix (host, column-major (p+1) x p):
 * the host-side part of compute_harmonic_ritz (preconditioner.cpp:162-205). */
hdgb_status hdgb_harmonic_ritz_from_hessenberg(const double* hess, int pmax, int p_eff,
                                               double* out_reim, int* n_out);

/* ---- A13: GMRES (gmres.hpp:11-53) ----------------------------------------------------------- */
typedef struct hdgb_gmres_config {
    int restart;          /* 50   */
    double tol;           /* 1e-6, relative preconditioned residual */
    int max_iters;        /* 1000 */
    int orth;             /* 0 = CGS with one re-orthogonalisation (default), 1 = MGS */
    int track_diagnostics;
} hdgb_gmres_config;

typedef struct hdgb_gmres_stats {
    int iters;
    int restarts;
    double final_rel_residual;
    double t_mv, t_prec, t_orth; /* seconds, CUDA-event timed when timing is enabled on the ctx */
    int converged;
    double max_orth_error, max_residual_gap;
} hdgb_gmres_stats;

void hdgb_gmres_config_default(hdgb_gmres_config* cfg);
/* gmres_solve (gmres.cpp:61-228), data form of SPEC.md:557: operator and preconditioner are the
 * device-resident handles.  p may be NULL (identity).  residual_trace (host, max_iters doubles)
 * may be NULL. */
hdgb_status hdgb_gmres_solve(hdgb_matrix* k, hdgb_precond* p, const double* rhs /*host|device*/,
                             const double* x0 /*host|device|NULL*/, const hdgb_gmres_config* cfg,
                             double* x /*host|device*/, hdgb_gmres_stats* stats, double* residual_trace);
/* gmres_solve (gmres.cpp:61-228), closure form of gmres.hpp:50-53: operator and preconditioner are callbacks on
 * device vectors of n doubles (precond NULL = identity); same control flow, statistics and errors. */
hdgb_status hdgb_gmres_solve_fn(hdgb_ctx* ctx, int64_t n, hdgb_op_fn matvec, void* matvec_user, hdgb_op_fn precond,
                                void* precond_user, const double* rhs /*host|device*/, const double* x0 /*host|device|NULL*/,
                                const hdgb_gmres_config* cfg, double* x /*host|device*/, hdgb_gmres_stats* stats,
                                double* residual_trace);
/* orthogonalize (gmres.cpp:28-59) on device vectors: basis is nvec contiguous vectors of length n;
 * h receives nvec+1 values (host). */
hdgb_status hdgb_orthogonalize(hdgb_ctx* ctx, const double* basis /*device*/, int nvec, int64_t n,
                               double* w /*device*/, int orth, double* h /*host*/);
/* Enables per-phase CUDA-event timing (t_mv/t_prec/t_orth; adds synchronisation). */
void hdgb_ctx_enable_phase_timing(hdgb_ctx* ctx, int on);

/* ---- A14: Newton driver (newton.hpp:14-71) -------------------------------------------------- */
typedef struct hdgb_newton_config {
    double tol;        /* 1e-8 */
    int max_newton;    /* 50   */
    double min_alpha;  /* 2^-10 */
} hdgb_newton_config;

#define HDGB_MAX_NEWTON_HISTORY 128
typedef struct hdgb_solve_report {
    int n_newton;
    int64_t n_gmres_total;
    int64_t n_inner_prec_ops;
    double final_residual;
    int converged;
    double t_ass, t_mv, t_prec, t_orth, t_total;
    int n_history;
    double residual_history[HDGB_MAX_NEWTON_HISTORY + 1];
    int gmres_per_newton[HDGB_MAX_NEWTON_HISTORY];
    double alpha_history[HDGB_MAX_NEWTON_HISTORY];
} hdgb_solve_report;

void hdgb_newton_config_default(hdgb_newton_config* cfg);
/* newton_solve (newton.cpp:54-154); updates the state in place. */
hdgb_status hdgb_newton_solve(hdgb_disc* d, const hdgb_model* m, hdgb_state* s,
                              const hdgb_newton_config* ncfg, const hdgb_gmres_config* gcfg,
                              const hdgb_precond_spec* pspec, const hdgb_time* t,
                              hdgb_solve_report* report);
/* time_march (newton.cpp:156-175): n_steps backward-Euler steps; reports (n_steps entries). */
hdgb_status hdgb_time_march(hdgb_disc* d, const hdgb_model* m, hdgb_state* s, double dt, int n_steps,
                            const hdgb_newton_config* ncfg, const hdgb_gmres_config* gcfg,
                            const hdgb_precond_spec* pspec, hdgb_solve_report* reports);

/* ---- multi-GPU: domain decomposition (north_star item 5; the reference has no distributed path,
 * PAPER.md:1122 lists it as future work) -------------------------------------------------------
 * One rank per GPU.  A rank's discretisation holds its owned elements first, then one layer of
 * ghost elements (condensed redundantly); its faces are numbered owned first (a face belongs to
 * the rank owning its side-0 element, the reference's own accumulation order, mesh.cpp:63-71),
 * then halo faces grouped by owner.  Vectors span all local faces; rows, dot products and norms
 * cover owned faces only.  Per operator application one halo exchange of interface trace slices,
 * per Gram-Schmidt pass one small all-reduce. */
/* Discretisation from explicit connectivity tables (a sub-domain cut out of a global mesh keeps the
 * global orientation flags / side assignment).  face_to_elements entries: >= 0 local element, -1
 * domain boundary, -2 element on another rank.  The first ne_owned elements / nf_owned faces are
 * owned.  face_gid (nf, may be NULL = identity) / nf_global give the global face numbering used
 * for the seeded Ritz start vector.  ctx == NULL: host-only tables. */
hdgb_status hdgb_disc_create_from_tables(hdgb_ctx* ctx, int shape, int degree, int n_comp, int quad_points,
                                         int ne, int nf, int nv, const int32_t* elem_verts,
                                         const double* vertex_coords, const int32_t* element_to_face,
                                         const int32_t* face_to_elements, const int32_t* face_local_index,
                                         const int32_t* face_orient, const int32_t* face_vertices,
                                         const int32_t* boundary_tag, int ne_owned, int nf_owned,
                                         const int64_t* face_gid, int64_t nf_global, hdgb_disc** out);
/* Connectivity of a conforming mesh given by element vertex lists (host only, no geometry, no
 * GPU): the tables a partitioner slices.  Read them with hdgb_disc_get_i32. */
hdgb_status hdgb_mesh_connectivity(int shape, int ne, int nv, const int32_t* elem_verts,
                                   const double* vertex_coords, hdgb_disc** out);
/* NCCL communicator over the ranks of one job; unique_id (128 bytes) comes from
 * hdgb_comm_nccl_unique_id on rank 0 and is broadcast by the caller (torch.distributed / MPI). */
hdgb_status hdgb_comm_nccl_unique_id(void* out128);
hdgb_status hdgb_comm_create_nccl(hdgb_ctx* ctx, const void* unique_id_128, int rank, int size);
/* Halo plan of this rank: for neighbour k, send the listed local (owned) faces and receive
 * recv_counts[k] faces into local face positions recv_offsets[k].. (contiguous per owner). */
hdgb_status hdgb_comm_set_halo_plan(hdgb_ctx* ctx, int n_nbr, const int32_t* nbr_ranks, const int32_t* send_counts,
                                    const int32_t* send_ids /*concatenated*/, const int32_t* recv_offsets,
                                    const int32_t* recv_counts);
/* Callback communicator (tests: several virtual ranks in one process on one GPU). */
typedef int (*hdgb_halo_fn)(void* user, double* dev_vec, int width);
typedef int (*hdgb_allreduce_fn)(void* user, double* dev_buf, int n);
hdgb_status hdgb_comm_set_callbacks(hdgb_ctx* ctx, int rank, int size, hdgb_halo_fn halo, hdgb_allreduce_fn allreduce,
                                    void* user);
void hdgb_comm_destroy(hdgb_ctx* ctx);
hdgb_status hdgb_halo_exchange(hdgb_ctx* ctx, double* dev_vec, int width);
/* The same exchange split in two: _begin starts it on the communicator's own stream (after everything enqueued so
 * far), work on owned entries may follow on the context's stream, _end orders that stream after the arrival. */
hdgb_status hdgb_halo_exchange_begin(hdgb_ctx* ctx, double* dev_vec, int width);
hdgb_status hdgb_halo_exchange_end(hdgb_ctx* ctx);
hdgb_status hdgb_allreduce_sum(hdgb_ctx* ctx, double* dev_buf, int n);
int hdgb_comm_rank(const hdgb_ctx* ctx);
int hdgb_comm_size(const hdgb_ctx* ctx);

/* ---- device vector helpers used by callers that keep data resident --------------------------- */
hdgb_status hdgb_device_alloc(hdgb_ctx* ctx, int64_t n_doubles, double** out);
void hdgb_device_free(hdgb_ctx* ctx, double* p);
hdgb_status hdgb_copy(hdgb_ctx* ctx, double* dst, const double* src, int64_t n); /* any direction */

#ifdef __cplusplus
}
#endif
#endif /* HDGB200_H */
