// Device-pointer level entry points shared by the C ABI translation units (api_global.cu,
// api_solve.cu).  Everything here enqueues on ctx->stream; functions that return host values
// synchronise.
#pragma once
#include <complex>
#include <functional>

#include "kernels_local.cuh"

namespace hdgb {

// y = K x  (block_matvec, face_matrix.cpp:83-107), device pointers.
void matvec_device(hdgb_matrix* k, const double* x, double* y);
// z = base(y): identity / apply_bj / apply_asm / RAS (preconditioner.cpp:285-299), device pointers.
// epi != nullptr: the result feeds the polynomial update (kernels.cuh PolyEpi) instead of being written to z; z is
// then scratch of the vector length (used by the bases that deliver their result as a vector).
void apply_base_device(hdgb_precond* p, const double* y, double* z, const PolyEpi* epi = nullptr);
// z = P^-1 y incl. the polynomial wrapper (preconditioner.cpp:301-308).  p == nullptr: identity.
void apply_precond_device(hdgb_precond* p, hdgb_matrix* k, const double* y, double* z);
// build_preconditioner (newton.cpp:30-52)
hdgb_precond* build_preconditioner_spec(hdgb_matrix* k, const hdgb_ops* o, hdgb_disc* d,
                                        const hdgb_precond_spec& spec);
// assemble_global (face_matrix.cpp:11-61); the matrix keeps the rhs.
hdgb_matrix* assemble_global_device(hdgb_disc* d, const hdgb_ops* o);
// assemble_element_operators / assemble_residual on device state (api_disc.cu)
hdgb_ops* assemble_element_operators_device(hdgb_disc* d, const hdgb_model* m, hdgb_state* s,
                                            const double* u_prev_dev, double dt, bool keep_raw);
// trace (mpf*nf) and interior (npe*ne) are device buffers; returns the stacked 2-norm.
double assemble_residual_device(hdgb_disc* d, const hdgb_model* m, hdgb_state* s, const double* u_prev_dev,
                                double dt, double* trace, double* interior);
// du = Ebar^-1 (ru - Fbar duhat_e)  (recover_local, local_ops.cpp:452-460), face-major duhat.
void recover_local_device(hdgb_disc* d, const hdgb_ops* o, const double* duhat, double* du, double* tmp);

// compute_q (local_ops.cpp:367-374) on the device state
void compute_q_device(hdgb_disc* d, hdgb_state* s);

// A linear operator on device vectors (the reference's OpFn / LinearOp, gmres.hpp:43, preconditioner.hpp:50, with
// device pointers): out = op(in), enqueued on ctx->stream.
using DevOp = std::function<void(const double* in, double* out)>;

// gmres_solve (gmres.cpp:61-228) for arbitrary operators: n owned unknowns (rows, sums), ld = vector length
// incl. the halo part; precond empty = identity.  W is sized by make_gmres_work.
std::unique_ptr<GmresWork> make_gmres_work(hdgb_ctx* c, int64_t n, int64_t ld, int restart);
void gmres_core(hdgb_ctx* c, int64_t n, int64_t ld, GmresWork& W, const DevOp& matvec, const DevOp& precond,
                const double* rhs, double* x, const hdgb_gmres_config& cfg, hdgb_gmres_stats* stats,
                double* residual_trace, int64_t* spec_counter = nullptr);
// compute_harmonic_ritz (preconditioner.cpp:119-205) of op on n owned unknowns (ld vector length): seeded start
// vector over n_global unknowns (face_gid maps local faces of width mpf to global ones, nullptr = identity),
// MGS Arnoldi on the device, eigen-solve + Leja order on the host.
std::vector<std::complex<double>> harmonic_ritz_op(hdgb_ctx* c, const DevOp& op, int64_t n, int64_t ld, int degree,
                                                   uint64_t seed, const int64_t* face_gid, int nf_local, int mpf,
                                                   int64_t n_global, bool* breakdown_out);
// apply_poly (preconditioner.cpp:246-283) with an arbitrary base application: z = poly(base K) base y.
void apply_poly_op(hdgb_precond* p, const DevOp& base, hdgb_matrix* k, const double* y, double* z);
// ... with the preconditioner's own base, the recurrence updates fused into the base's last kernel
void apply_poly_fused(hdgb_precond* p, hdgb_matrix* k, const double* y, double* z);
// the two-sided diagonal sub-block sums of build_asm (preconditioner.cpp:59-75) straight from K-bar
void launch_face_diag(hdgb_ctx* ctx, const DiscView& dv, const double* kbar, double* diag);
// build_bj (preconditioner.cpp:30-46) / build_asm (:54-84) as separate entry points
hdgb_precond* build_bj_device(hdgb_matrix* k);
hdgb_precond* build_asm_device(const hdgb_ops* o, hdgb_disc* d, int kind, const double* diag_from_k);

// gmres_solve (gmres.cpp:61-228) on device vectors rhs / x (x holds x0 on entry).
void gmres_device(hdgb_matrix* k, hdgb_precond* p, const double* rhs, double* x, const hdgb_gmres_config& cfg,
                  hdgb_gmres_stats* stats, double* residual_trace);

// Phase timer: CUDA-event timing of a stream segment when ctx->phase_timing is on.
struct PhaseTimer {
    hdgb_ctx* c;
    double* acc;
    PhaseTimer(hdgb_ctx* ctx, double* accumulate) : c(ctx), acc(accumulate) {
        if (c->phase_timing && acc) HDGB_CUDA(cudaEventRecord(c->ev[0], c->stream));
    }
    void stop() {
        if (c->phase_timing && acc) {
            HDGB_CUDA(cudaEventRecord(c->ev[1], c->stream));
            HDGB_CUDA(cudaEventSynchronize(c->ev[1]));
            float ms = 0.f;
            HDGB_CUDA(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
            *acc += 1e-3 * ms;
        }
        acc = nullptr;
    }
};

}  // namespace hdgb
