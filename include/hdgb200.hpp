// hdgb200.hpp -- C++17 layer over the C ABI of libhdgb200.so, re-creating the reference's operator API
// (hdgkit, proj/include/hdg/{dense_batch,local_ops,face_matrix,preconditioner,gmres,newton}.hpp) with the
// same names, argument meaning and error behaviour: value-semantics results, exceptions derived from one
// base class that carry the offending batch index (errors.hpp:9-23), option structs field for field
// (GmresConfig gmres.hpp:15-22, NewtonConfig / PrecondSpec newton.hpp:17-29, SolveReport newton.hpp:31-45).
// Header only; link against libhdgb200.so.  Device-resident objects are RAII handles; vectors cross the
// boundary as std::vector<double> (the library stages host buffers itself).
//
// What differs from the reference by construction: PdeModel's std::function callbacks cannot run on the
// device, so a model is a (kind, parameters, tabulated x-only data) triple -- see Model below; meshes are built
// by the library (build_structured_quad / its hex, triangle, tetrahedron analogues) or from vertex lists.
#ifndef HDGB200_HPP
#define HDGB200_HPP

#include <algorithm>
#include <complex>
#include <cstdint>
#include <exception>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hdgb200.h"

namespace hdg {
namespace b200 {

// ---- errors (errors.hpp) ------------------------------------------------------------------------------------
class Error : public std::runtime_error {
  public:
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class SingularBlock : public Error {  // errors.hpp:16-23
  public:
    SingularBlock(long index_, const std::string& m) : Error(m), index(index_) {}
    long index;
};
class SingularMass : public SingularBlock { using SingularBlock::SingularBlock; };        // errors.hpp:63-67
class SingularLocalSolve : public SingularBlock { using SingularBlock::SingularBlock; };  // errors.hpp:70-74
class DimensionMismatch : public Error { using Error::Error; };
class InconsistentDimensions : public Error { using Error::Error; };
class NonFiniteState : public Error { using Error::Error; };
class NaNDetected : public Error { using Error::Error; };
class TooLargeForDense : public Error { using Error::Error; };
class IoError : public Error { using Error::Error; };
class InvalidMesh : public Error { using Error::Error; };
class Unsupported : public Error { using Error::Error; };
class CudaError : public Error { using Error::Error; };
class LineSearchFailed : public Error {  // errors.hpp:92-98
  public:
    LineSearchFailed(long iteration_, const std::string& m) : Error(m), iteration(iteration_) {}
    long iteration;
};

inline void check(hdgb_ctx* c, hdgb_status s) {
    if (s == HDGB_OK) return;
    const std::string msg = c ? hdgb_last_error(c) : std::string("hdgb200 call failed");
    const long idx = c ? static_cast<long>(hdgb_last_error_index(c)) : -1;
    switch (s) {
        case HDGB_ERR_SINGULAR_BLOCK: throw SingularBlock(idx, msg);
        case HDGB_ERR_SINGULAR_MASS: throw SingularMass(idx, msg);
        case HDGB_ERR_SINGULAR_LOCAL_SOLVE: throw SingularLocalSolve(idx, msg);
        case HDGB_ERR_NONFINITE_STATE: throw NonFiniteState(msg);
        case HDGB_ERR_NAN_DETECTED: throw NaNDetected(msg);
        case HDGB_ERR_LINE_SEARCH_FAILED: throw LineSearchFailed(idx, msg);
        case HDGB_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case HDGB_ERR_INCONSISTENT_DIMENSIONS: throw InconsistentDimensions(msg);
        case HDGB_ERR_TOO_LARGE_FOR_DENSE: throw TooLargeForDense(msg);
        case HDGB_ERR_IO: throw IoError(msg);
        case HDGB_ERR_INVALID_MESH: throw InvalidMesh(msg);
        case HDGB_ERR_UNSUPPORTED: throw Unsupported(msg);
        case HDGB_ERR_CUDA: throw CudaError(msg);
        default: throw Error(msg);
    }
}

// ---- option structs (field for field) -------------------------------------------------------------------------
enum class Orth { CGS, MGS };                     // gmres.hpp:13
struct GmresConfig {                              // gmres.hpp:15-22
    int restart = 50;
    double tol = 1e-6;
    int max_iters = 1000;
    Orth orth = Orth::CGS;
    bool track_diagnostics = false;
};
struct GmresStats {                               // gmres.hpp:24-34
    int iters = 0, restarts = 0;
    double final_rel_residual = 0.0, t_mv = 0.0, t_prec = 0.0, t_orth = 0.0;
    bool converged = false;
    double max_orth_error = 0.0, max_residual_gap = 0.0;
};
struct NewtonConfig {                             // newton.hpp:17-21
    double tol = 1e-8;
    int max_newton = 50;
    double min_alpha = 1.0 / 1024.0;
};
enum class PrecondKind { Identity = HDGB_PC_IDENTITY, BJ = HDGB_PC_BJ, ASM = HDGB_PC_ASM, RAS = HDGB_PC_RAS };
struct PrecondSpec {                              // newton.hpp:24-29 (+ poly_kind, RAS: not in the reference)
    PrecondKind kind = PrecondKind::BJ;
    int poly_degree = 0;
    std::uint64_t ritz_seed = 12345;
    bool ritz_per_restart = false;
    int poly_kind = HDGB_POLY_GMRES;
};
struct TimeContext {                              // local_ops.hpp:67-70
    std::optional<double> dt;
    const std::vector<double>* u_prev = nullptr;
};
struct SolveReport {                              // newton.hpp:31-45
    int n_newton = 0;
    long n_gmres_total = 0, n_inner_prec_ops = 0;
    double final_residual = 0.0;
    bool converged = false;
    double t_ass = 0.0, t_mv = 0.0, t_prec = 0.0, t_orth = 0.0, t_total = 0.0;
    std::vector<double> residual_history, alpha_history;
    std::vector<int> gmres_per_newton;
};

namespace detail {
inline hdgb_gmres_config to_c(const GmresConfig& g) {
    return hdgb_gmres_config{g.restart, g.tol, g.max_iters, g.orth == Orth::MGS ? 1 : 0, g.track_diagnostics ? 1 : 0};
}
inline hdgb_newton_config to_c(const NewtonConfig& n) { return hdgb_newton_config{n.tol, n.max_newton, n.min_alpha}; }
inline hdgb_precond_spec to_c(const PrecondSpec& p) {
    return hdgb_precond_spec{static_cast<int>(p.kind), p.poly_degree, p.ritz_seed, p.ritz_per_restart ? 1 : 0, p.poly_kind};
}
inline hdgb_time to_c(const TimeContext& t) {
    return hdgb_time{t.dt ? *t.dt : 0.0, (t.dt && t.u_prev) ? t.u_prev->data() : nullptr};
}
inline SolveReport from_c(const hdgb_solve_report& r) {
    SolveReport o;
    o.n_newton = r.n_newton; o.n_gmres_total = static_cast<long>(r.n_gmres_total);
    o.n_inner_prec_ops = static_cast<long>(r.n_inner_prec_ops);
    o.final_residual = r.final_residual; o.converged = r.converged != 0;
    o.t_ass = r.t_ass; o.t_mv = r.t_mv; o.t_prec = r.t_prec; o.t_orth = r.t_orth; o.t_total = r.t_total;
    o.residual_history.assign(r.residual_history, r.residual_history + r.n_history);
    const int nn = r.n_newton < HDGB_MAX_NEWTON_HISTORY ? r.n_newton : HDGB_MAX_NEWTON_HISTORY;
    o.gmres_per_newton.assign(r.gmres_per_newton, r.gmres_per_newton + nn);
    o.alpha_history.assign(r.alpha_history, r.alpha_history + nn);
    return o;
}
}  // namespace detail

// ---- handles --------------------------------------------------------------------------------------------------
class Context {
  public:
    explicit Context(int device = 0) {
        if (hdgb_ctx_create(device, &h_) != HDGB_OK) throw CudaError("no usable CUDA device (libhdgb200 has no CPU fallback)");
    }
    ~Context() { if (h_) hdgb_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    hdgb_ctx* get() const { return h_; }
    void synchronize() { check(h_, hdgb_ctx_synchronize(h_)); }
  private:
    hdgb_ctx* h_ = nullptr;
};

// Mesh2D + BasisTab + GeomFactors + LocalFactors (study.cpp:67-77 make_case_setup) in one object.
class Discretization {
  public:
    static Discretization structured(Context& c, hdgb_shape shape, int n, int degree, int n_comp = 1, int quad_points = 0,
                                     double jitter = 0.0, std::uint64_t seed = 12345) {
        Discretization d(c);
        check(c.get(), hdgb_disc_create_structured(c.get(), shape, n, degree, n_comp, quad_points, nullptr, nullptr, jitter, seed, &d.h_));
        check(c.get(), hdgb_disc_dims(d.h_, &d.dims_));
        return d;
    }
    ~Discretization() { if (h_) hdgb_disc_destroy(h_); }
    Discretization(Discretization&& o) noexcept : c_(o.c_), h_(o.h_), dims_(o.dims_) { o.h_ = nullptr; }
    Discretization(const Discretization&) = delete;
    const hdgb_dims& dims() const { return dims_; }
    int npe() const { return dims_.n_comp * dims_.pe; }
    int mpf() const { return dims_.n_comp * dims_.pf; }
    int nfl() const { return dims_.n_lfe * mpf(); }
    int nb() const { return 2 * dims_.n_lfe - 1; }
    long n_dof() const { return static_cast<long>(mpf()) * dims_.nf; }
    std::vector<double> table_f64(const std::string& name) const {
        std::int64_t n = 0;
        check(c_->get(), hdgb_disc_get_f64(h_, name.c_str(), nullptr, 0, &n));
        std::vector<double> v(static_cast<size_t>(n));
        check(c_->get(), hdgb_disc_get_f64(h_, name.c_str(), v.data(), n, &n));
        return v;
    }
    std::vector<std::int32_t> table_i32(const std::string& name) const {
        std::int64_t n = 0;
        check(c_->get(), hdgb_disc_get_i32(h_, name.c_str(), nullptr, 0, &n));
        std::vector<std::int32_t> v(static_cast<size_t>(n));
        check(c_->get(), hdgb_disc_get_i32(h_, name.c_str(), v.data(), n, &n));
        return v;
    }
    hdgb_disc* get() const { return h_; }
    Context& ctx() const { return *c_; }
  private:
    explicit Discretization(Context& c) : c_(&c) {}
    Context* c_;
    hdgb_disc* h_ = nullptr;
    hdgb_dims dims_{};
};

// PdeModel (models.hpp:27-50) as device functor tag + parameters + x-only data tabulated at the quadrature points
// (forcing: ne*qe*M values at Discretization::table_f64("elem_coords"); dirichlet: nf*qf*M at "face_coords").
class Model {
  public:
    Model(const Discretization& d, hdgb_model_kind kind, const std::vector<double>& params,
          const std::vector<double>* forcing_q = nullptr, const std::vector<double>* dirichlet_q = nullptr)
        : c_(&d.ctx()) {
        check(c_->get(), hdgb_model_create(c_->get(), d.get(), kind, params.data(), static_cast<int>(params.size()),
                                           forcing_q ? forcing_q->data() : nullptr, dirichlet_q ? dirichlet_q->data() : nullptr, &h_));
    }
    ~Model() { if (h_) hdgb_model_destroy(h_); }
    Model(const Model&) = delete;
    hdgb_model* get() const { return h_; }
  private:
    Context* c_;
    hdgb_model* h_ = nullptr;
};

// StateFields (local_ops.hpp:16-23) on the device.
class StateFields {
  public:
    explicit StateFields(const Discretization& d) : d_(&d) { check(d.ctx().get(), hdgb_state_create(d.ctx().get(), d.get(), &h_)); }
    ~StateFields() { if (h_) hdgb_state_destroy(h_); }
    StateFields(const StateFields&) = delete;
    void set(const char* name, const std::vector<double>& v) {
        if (v.size() != size_of(name)) throw DimensionMismatch(std::string("state field ") + name + ": wrong size");
        check(d_->ctx().get(), hdgb_state_set(h_, name, v.data()));
    }
    std::vector<double> get(const char* name) const {
        std::vector<double> v(size_of(name));
        check(d_->ctx().get(), hdgb_state_get(h_, name, v.data()));
        return v;
    }
    hdgb_state* handle() const { return h_; }
  private:
    size_t size_of(const char* name) const {
        return std::string(name) == "uhat" ? static_cast<size_t>(d_->n_dof()) : static_cast<size_t>(d_->npe()) * d_->dims().ne;
    }
    const Discretization* d_;
    hdgb_state* h_ = nullptr;
};

class ElementOperators {  // local_ops.hpp:40-62
  public:
    ElementOperators(Context& c, hdgb_ops* h) : c_(&c), h_(h) {}
    ~ElementOperators() { if (h_) hdgb_ops_destroy(h_); }
    ElementOperators(ElementOperators&& o) noexcept : c_(o.c_), h_(o.h_) { o.h_ = nullptr; }
    ElementOperators(const ElementOperators&) = delete;
    std::vector<double> get(const std::string& name) const {  // kbar, ebar_inv, fbar, hbar, rbar, ru, (raw blocks)
        std::int64_t n = 0;
        check(c_->get(), hdgb_ops_get(h_, name.c_str(), nullptr, 0, &n));
        std::vector<double> v(static_cast<size_t>(n));
        check(c_->get(), hdgb_ops_get(h_, name.c_str(), v.data(), n, &n));
        return v;
    }
    hdgb_ops* handle() const { return h_; }
  private:
    Context* c_;
    hdgb_ops* h_;
};

class FaceBlockMatrix {  // face_matrix.hpp:26-43
  public:
    FaceBlockMatrix(Context& c, hdgb_matrix* h) : c_(&c), h_(h) {
        int d4[4];
        check(c.get(), hdgb_matrix_dims(h_, d4));
        m = d4[0]; block_dim = d4[0] * d4[1]; nb = 2 * d4[2] - 1; nf = d4[3];  // (m, pf, n_lfe, nf)
    }
    ~FaceBlockMatrix() { if (h_) hdgb_matrix_destroy(h_); }
    FaceBlockMatrix(FaceBlockMatrix&& o) noexcept : m(o.m), block_dim(o.block_dim), nb(o.nb), nf(o.nf), c_(o.c_), h_(o.h_) { o.h_ = nullptr; }
    FaceBlockMatrix(const FaceBlockMatrix&) = delete;
    long n_dof() const { return static_cast<long>(block_dim) * nf; }
    std::vector<std::int64_t> neighbor() const {
        std::vector<std::int64_t> v(static_cast<size_t>(nf) * nb);
        check(c_->get(), hdgb_matrix_get_neighbor(h_, v.data()));
        return v;
    }
    std::vector<double> blocks() const {
        std::vector<double> v(static_cast<size_t>(block_dim) * block_dim * nb * nf);
        check(c_->get(), hdgb_matrix_get_blocks(h_, v.data()));
        return v;
    }
    int m = 1, block_dim = 0, nb = 0, nf = 0;
    hdgb_matrix* handle() const { return h_; }
    Context& ctx() const { return *c_; }
  private:
    Context* c_;
    hdgb_matrix* h_;
};

class Preconditioner {  // preconditioner.hpp:19-29
  public:
    Preconditioner(Context& c, hdgb_precond* h) : c_(&c), h_(h) {}
    ~Preconditioner() { if (h_) hdgb_precond_destroy(h_); }
    Preconditioner(Preconditioner&& o) noexcept : c_(o.c_), h_(o.h_) { o.h_ = nullptr; }
    Preconditioner(const Preconditioner&) = delete;
    long n_inner_prec_ops() const { return static_cast<long>(hdgb_precond_inner_ops(h_)); }
    hdgb_precond* handle() const { return h_; }
  private:
    Context* c_;
    hdgb_precond* h_;
};

// ---- the reference's free functions ----------------------------------------------------------------------------
// dense_batch.hpp:40-60
inline std::vector<double> lu_invert_batch(Context& c, const std::vector<double>& a, int n, int batch) {
    if (a.size() != static_cast<size_t>(n) * n * batch) throw DimensionMismatch("lu_invert_batch: data size does not match n x n x batch");
    std::vector<double> inv(a.size());
    check(c.get(), hdgb_lu_invert_batch(c.get(), n, batch, a.data(), inv.data()));
    return inv;
}
// local_ops.hpp:83
inline void compute_q(const Discretization& d, StateFields& s) { check(d.ctx().get(), hdgb_compute_q(d.get(), s.handle())); }
// local_ops.hpp:89-92
inline ElementOperators assemble_element_operators(const Model& model, StateFields& state, const Discretization& d,
                                                   const TimeContext& time = {}, bool keep_raw = false) {
    hdgb_ops* o = nullptr;
    const hdgb_time t = detail::to_c(time);
    check(d.ctx().get(), hdgb_assemble_element_operators(d.get(), model.get(), state.handle(), &t, keep_raw ? 1 : 0, &o));
    return ElementOperators(d.ctx(), o);
}
struct Residuals {  // local_ops.hpp:64-66 + residual_norm (:245-250)
    std::vector<double> trace, interior;
    double norm = 0.0;
};
// local_ops.hpp:95-97
inline Residuals assemble_residual(const Model& model, StateFields& state, const Discretization& d, const TimeContext& time = {}) {
    Residuals r;
    r.trace.resize(static_cast<size_t>(d.n_dof()));
    r.interior.resize(static_cast<size_t>(d.npe()) * d.dims().ne);
    const hdgb_time t = detail::to_c(time);
    check(d.ctx().get(), hdgb_assemble_residual(d.get(), model.get(), state.handle(), &t, r.trace.data(), r.interior.data(), &r.norm));
    return r;
}
// local_ops.hpp:101 (takes the face-major trace update; the gather of :351-365 is fused)
inline std::vector<double> recover_local(const Discretization& d, const ElementOperators& ops, const std::vector<double>& duhat) {
    if (duhat.size() != static_cast<size_t>(d.n_dof())) throw DimensionMismatch("recover_local: trace vector size");
    std::vector<double> du(static_cast<size_t>(d.npe()) * d.dims().ne);
    check(d.ctx().get(), hdgb_recover_local(d.get(), ops.handle(), duhat.data(), du.data()));
    return du;
}
// face_matrix.hpp:49
inline std::pair<FaceBlockMatrix, std::vector<double>> assemble_global(const ElementOperators& ops, const Discretization& d) {
    hdgb_matrix* k = nullptr;
    std::vector<double> rhs(static_cast<size_t>(d.n_dof()));
    check(d.ctx().get(), hdgb_assemble_global(d.get(), ops.handle(), &k, rhs.data()));
    return {FaceBlockMatrix(d.ctx(), k), std::move(rhs)};
}
// face_matrix.hpp:58
inline std::vector<double> block_matvec(const FaceBlockMatrix& k, const std::vector<double>& x) {
    if (x.size() != static_cast<size_t>(k.n_dof())) throw DimensionMismatch("block_matvec: vector size does not match the matrix");
    std::vector<double> y(x.size());
    check(k.ctx().get(), hdgb_block_matvec(k.handle(), x.data(), y.data()));
    return y;
}
// newton.hpp:52 / newton.cpp:30-52
inline Preconditioner build_preconditioner(const PrecondSpec& spec, const FaceBlockMatrix& k, const ElementOperators& ops,
                                           const Discretization& d) {
    hdgb_precond* p = nullptr;
    const hdgb_precond_spec s = detail::to_c(spec);
    check(d.ctx().get(), hdgb_build_preconditioner(k.handle(), ops.handle(), d.get(), &s, &p));
    return Preconditioner(d.ctx(), p);
}
// preconditioner.hpp:70-76 (make_preconditioner_apply as a call instead of a closure)
inline std::vector<double> apply_preconditioner(Preconditioner& p, const FaceBlockMatrix& k, const std::vector<double>& y) {
    std::vector<double> z(y.size());
    check(k.ctx().get(), hdgb_precond_apply(p.handle(), k.handle(), y.data(), z.data()));
    return z;
}
// ---- preconditioner.hpp:31-76, one function each --------------------------------------------------------------
// build_bj (preconditioner.hpp:33) / apply_bj (:36)
inline Preconditioner build_bj(const FaceBlockMatrix& k) {
    hdgb_precond* p = nullptr;
    check(k.ctx().get(), hdgb_build_bj(k.handle(), &p));
    return Preconditioner(k.ctx(), p);
}
inline std::vector<double> apply_bj(Context& c, Preconditioner& p, const std::vector<double>& y) {
    std::vector<double> z(y.size());
    check(c.get(), hdgb_apply_bj(p.handle(), y.data(), z.data()));
    return z;
}
// build_asm (preconditioner.hpp:42) / apply_asm (:47); the mesh argument of the reference is the discretisation
inline Preconditioner build_asm(const ElementOperators& ops, const Discretization& d) {
    hdgb_precond* p = nullptr;
    check(d.ctx().get(), hdgb_build_asm(ops.handle(), d.get(), &p));
    return Preconditioner(d.ctx(), p);
}
inline std::vector<double> apply_asm(Context& c, Preconditioner& p, const std::vector<double>& y) {
    std::vector<double> z(y.size());
    check(c.get(), hdgb_apply_asm(p.handle(), y.data(), z.data()));
    return z;
}

// A linear operator on DEVICE vectors of n doubles: out = op(in), enqueued on the context's stream (or synchronised
// before returning).  The reference's LinearOp / OpFn (preconditioner.hpp:50, gmres.hpp:43) with device pointers.
using DeviceOp = std::function<void(const double* in, double* out, std::int64_t n)>;

namespace detail {
struct OpThunk {
    const DeviceOp* fn;
    std::exception_ptr error;
    static int call(void* user, const double* in, double* out, std::int64_t n) {
        OpThunk* t = static_cast<OpThunk*>(user);
        try {
            (*t->fn)(in, out, n);
            return 0;
        } catch (...) {
            t->error = std::current_exception();
            return 1;
        }
    }
};
inline std::vector<std::complex<double>> unpack(const std::vector<double>& reim, int n) {
    std::vector<std::complex<double>> o;
    for (int i = 0; i < n; ++i) o.emplace_back(reim[2 * i], reim[2 * i + 1]);
    return o;
}
}  // namespace detail

// compute_harmonic_ritz (preconditioner.hpp:57-58)
inline std::vector<std::complex<double>> compute_harmonic_ritz(Context& c, const DeviceOp& op, std::size_t n_dof, int degree,
                                                               std::uint64_t seed) {
    detail::OpThunk t{&op, nullptr};
    std::vector<double> reim(2 * static_cast<size_t>(degree > 0 ? degree : 1));
    int n = 0;
    const hdgb_status st = hdgb_compute_harmonic_ritz(c.get(), detail::OpThunk::call, &t, static_cast<std::int64_t>(n_dof), degree,
                                                      seed, reim.data(), &n);
    if (t.error) std::rethrow_exception(t.error);
    check(c.get(), st);
    return detail::unpack(reim, n);
}
// leja_order (preconditioner.hpp:64)
inline std::vector<std::complex<double>> leja_order(const std::vector<std::complex<double>>& theta) {
    std::vector<double> in, out(2 * theta.size() + 2);
    for (const auto& t : theta) { in.push_back(t.real()); in.push_back(t.imag()); }
    int n = 0;
    if (hdgb_leja_order(in.data(), static_cast<int>(theta.size()), out.data(), &n) != HDGB_OK) throw Error("leja_order failed");
    return detail::unpack(out, n);
}
// make_base_apply (preconditioner.hpp:70) / make_preconditioner_apply (:73-74) as device operators
inline DeviceOp make_base_apply(Context& c, Preconditioner& p) {
    return [&c, &p](const double* in, double* out, std::int64_t) { check(c.get(), hdgb_precond_apply_base(p.handle(), in, out)); };
}
inline DeviceOp make_preconditioner_apply(Preconditioner& p, const FaceBlockMatrix& k) {
    return [&p, &k](const double* in, double* out, std::int64_t) { check(k.ctx().get(), hdgb_precond_apply(p.handle(), k.handle(), in, out)); };
}
// block_matvec as a device operator (the closure the reference's tests build around block_matvec)
inline DeviceOp make_matvec(const FaceBlockMatrix& k) {
    return [&k](const double* in, double* out, std::int64_t) { check(k.ctx().get(), hdgb_block_matvec(k.handle(), in, out)); };
}
// apply_poly (preconditioner.hpp:66-67): p supplies the Ritz values; base == nullptr uses p's own base
inline std::vector<double> apply_poly(Preconditioner& p, const DeviceOp* base, const FaceBlockMatrix& k, const std::vector<double>& y,
                                      long* inner_ops = nullptr) {
    if (y.size() != static_cast<size_t>(k.n_dof())) throw DimensionMismatch("apply_poly: vector size does not match the matrix");
    std::vector<double> z(y.size());
    std::int64_t ops = 0;
    detail::OpThunk t{base, nullptr};
    const hdgb_status st = hdgb_apply_poly(p.handle(), base ? detail::OpThunk::call : nullptr, base ? &t : nullptr, k.handle(), y.data(),
                                           z.data(), &ops);
    if (t.error) std::rethrow_exception(t.error);
    check(k.ctx().get(), st);
    if (inner_ops) *inner_ops += static_cast<long>(ops);
    return z;
}
// gmres.hpp:50-53, closure form: operator and preconditioner are device operators (precond empty = identity)
inline std::pair<std::vector<double>, GmresStats> gmres_solve(Context& c, const DeviceOp& matvec, const DeviceOp& precond,
                                                              const std::vector<double>& rhs, const std::vector<double>& x0,
                                                              const GmresConfig& cfg = {}, std::vector<double>* residual_trace = nullptr) {
    std::vector<double> x(rhs.size());
    const hdgb_gmres_config cc = detail::to_c(cfg);
    hdgb_gmres_stats st{};
    detail::OpThunk mv{&matvec, nullptr}, pc{&precond, nullptr};
    std::vector<double> trace(residual_trace ? static_cast<size_t>(cfg.max_iters > 0 ? cfg.max_iters : 1) : 0);
    const hdgb_status rc = hdgb_gmres_solve_fn(c.get(), static_cast<std::int64_t>(rhs.size()), detail::OpThunk::call, &mv,
                                               precond ? detail::OpThunk::call : nullptr, precond ? &pc : nullptr, rhs.data(),
                                               x0.empty() ? nullptr : x0.data(), &cc, x.data(), &st, residual_trace ? trace.data() : nullptr);
    if (mv.error) std::rethrow_exception(mv.error);
    if (pc.error) std::rethrow_exception(pc.error);
    check(c.get(), rc);
    GmresStats o;
    o.iters = st.iters; o.restarts = st.restarts; o.final_rel_residual = st.final_rel_residual;
    o.t_mv = st.t_mv; o.t_prec = st.t_prec; o.t_orth = st.t_orth; o.converged = st.converged != 0;
    o.max_orth_error = st.max_orth_error; o.max_residual_gap = st.max_residual_gap;
    if (residual_trace) residual_trace->assign(trace.begin(), trace.begin() + std::min<size_t>(trace.size(), static_cast<size_t>(st.iters)));
    return {std::move(x), o};
}
// gmres.hpp:50-53 in the data form of SPEC.md:557
inline std::pair<std::vector<double>, GmresStats> gmres_solve(const FaceBlockMatrix& k, Preconditioner& p, const std::vector<double>& rhs,
                                                              const std::vector<double>& x0, const GmresConfig& cfg = {}) {
    if (rhs.size() != static_cast<size_t>(k.n_dof())) throw DimensionMismatch("gmres_solve: right-hand side size");
    std::vector<double> x(rhs.size());
    const hdgb_gmres_config c = detail::to_c(cfg);
    hdgb_gmres_stats st{};
    check(k.ctx().get(), hdgb_gmres_solve(k.handle(), p.handle(), rhs.data(), x0.empty() ? nullptr : x0.data(), &c, x.data(), &st, nullptr));
    GmresStats o;
    o.iters = st.iters; o.restarts = st.restarts; o.final_rel_residual = st.final_rel_residual;
    o.t_mv = st.t_mv; o.t_prec = st.t_prec; o.t_orth = st.t_orth; o.converged = st.converged != 0;
    o.max_orth_error = st.max_orth_error; o.max_residual_gap = st.max_residual_gap;
    return {std::move(x), o};
}
// newton.hpp:57-64
inline SolveReport newton_solve(const Model& model, const Discretization& d, StateFields& state, const NewtonConfig& ncfg = {},
                                const GmresConfig& gcfg = {}, const PrecondSpec& pspec = {}, const TimeContext& time = {}) {
    const hdgb_newton_config nc = detail::to_c(ncfg);
    const hdgb_gmres_config gc = detail::to_c(gcfg);
    const hdgb_precond_spec ps = detail::to_c(pspec);
    const hdgb_time t = detail::to_c(time);
    auto r = std::make_unique<hdgb_solve_report>();
    const hdgb_status st = hdgb_newton_solve(d.get(), model.get(), state.handle(), &nc, &gc, &ps, &t, r.get());
    check(d.ctx().get(), st);
    return detail::from_c(*r);
}
// newton.hpp:66-71
inline std::vector<SolveReport> time_march(const Model& model, const Discretization& d, StateFields& state, double dt, int n_steps,
                                           const NewtonConfig& ncfg = {}, const GmresConfig& gcfg = {}, const PrecondSpec& pspec = {}) {
    const hdgb_newton_config nc = detail::to_c(ncfg);
    const hdgb_gmres_config gc = detail::to_c(gcfg);
    const hdgb_precond_spec ps = detail::to_c(pspec);
    std::vector<hdgb_solve_report> reps(static_cast<size_t>(n_steps));
    check(d.ctx().get(), hdgb_time_march(d.get(), model.get(), state.handle(), dt, n_steps, &nc, &gc, &ps, reps.data()));
    std::vector<SolveReport> out;
    for (const auto& r : reps) out.push_back(detail::from_c(r));
    return out;
}

}  // namespace b200
}  // namespace hdg

#endif  // HDGB200_HPP
