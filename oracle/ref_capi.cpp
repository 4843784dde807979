// TEST INFRASTRUCTURE ONLY (oracle/): a flat C ABI over the UNMODIFIED reference
// sources (/root/reference/proj/src/*.cpp, compiled where they lie by oracle/Makefile
// into oracle/_ref/libhdgref.so). Nothing in the product links or loads this file;
// only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// arm may use it, as the checker and the timed CPU baseline.
//
// Every entry point is a thin call into the reference's own public API
// (proj/include/hdg/*.hpp); no arithmetic is re-implemented here.
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "hdg/dense_batch.hpp"
#include "hdg/errors.hpp"
#include "hdg/face_matrix.hpp"
#include "hdg/gmres.hpp"
#include "hdg/local_ops.hpp"
#include "hdg/newton.hpp"
#include "hdg/parallel.hpp"
#include "hdg/preconditioner.hpp"
#include "hdg/study.hpp"
#include "oracles.hpp"
#include "test_helpers.hpp"

using namespace hdg;

namespace {

thread_local std::string g_err_msg;
thread_local std::string g_err_kind;
thread_local long g_err_index = -1;

template <class F>
int guarded(F&& fn) {
    g_err_msg.clear();
    g_err_kind.clear();
    g_err_index = -1;
    try {
        fn();
        return 0;
    } catch (const SingularBlock& e) {
        g_err_kind = "SingularBlock"; g_err_index = e.index; g_err_msg = e.what(); return 2;
    } catch (const SingularMass& e) {
        g_err_kind = "SingularMass"; g_err_msg = e.what(); return 2;
    } catch (const SingularLocalSolve& e) {
        g_err_kind = "SingularLocalSolve"; g_err_msg = e.what(); return 2;
    } catch (const NonFiniteState& e) {
        g_err_kind = "NonFiniteState"; g_err_msg = e.what(); return 3;
    } catch (const NaNDetected& e) {
        g_err_kind = "NaNDetected"; g_err_msg = e.what(); return 3;
    } catch (const LineSearchFailed& e) {
        g_err_kind = "LineSearchFailed"; g_err_msg = e.what(); return 4;
    } catch (const DimensionMismatch& e) {
        g_err_kind = "DimensionMismatch"; g_err_msg = e.what(); return 5;
    } catch (const InconsistentDimensions& e) {
        g_err_kind = "InconsistentDimensions"; g_err_msg = e.what(); return 5;
    } catch (const TooLargeForDense& e) {
        g_err_kind = "TooLargeForDense"; g_err_msg = e.what(); return 5;
    } catch (const IoError& e) {
        g_err_kind = "IoError"; g_err_msg = e.what(); return 6;
    } catch (const Error& e) {
        g_err_kind = "Error"; g_err_msg = e.what(); return 1;
    } catch (const std::exception& e) {
        g_err_kind = "std::exception"; g_err_msg = e.what(); return 1;
    }
}

struct RefCase {
    CaseSpec spec;
    CaseSetup setup;
    StateFields state;
    ElementOperators ops;
    FaceBlockMatrix k;
    TraceVector rhs;
    Preconditioner prec;
    long inner_ops = 0;
    std::vector<double> u_prev;
    std::optional<double> dt;
    SolveReport report;
    bool assembled = false;

    TimeContext time() const {
        TimeContext t;
        if (dt) { t.dt = dt; t.u_prev = &u_prev; }
        return t;
    }
};

long copy_out(const std::vector<double>& v, double* out, long cap) {
    if (out) {
        if (cap < static_cast<long>(v.size())) return -1;
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    }
    return static_cast<long>(v.size());
}

template <class T, std::size_t N>
std::vector<int> flatten(const std::vector<std::array<T, N>>& a) {
    std::vector<int> out;
    out.reserve(a.size() * N);
    for (const auto& row : a)
        for (const auto& v : row) out.push_back(static_cast<int>(v));
    return out;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err_msg.c_str(); }
const char* ref_last_error_kind() { return g_err_kind.c_str(); }
long ref_last_error_index() { return g_err_index; }

void ref_set_threads(int n) { set_threads(n); }
int ref_threads() { return threads(); }

// ---- stand-alone dense kernels (dense_batch.hpp) -------------------------------------------
int ref_lu_invert_batch(int n, int batch, const double* a, double* out) {
    return guarded([&] {
        DenseBatch in(n, n, batch);
        std::memcpy(in.data.data(), a, in.data.size() * sizeof(double));
        DenseBatch inv = lu_invert_batch(in);
        std::memcpy(out, inv.data.data(), inv.data.size() * sizeof(double));
    });
}

int ref_gemm_batch(int ar, int ac, int abatch, const double* a, int br, int bc, int bbatch,
                   const double* b, int transpose_a, double* c) {
    return guarded([&] {
        DenseBatch A(ar, ac, abatch), B(br, bc, bbatch);
        std::memcpy(A.data.data(), a, A.data.size() * sizeof(double));
        std::memcpy(B.data.data(), b, B.data.size() * sizeof(double));
        DenseBatch C = gemm_batch(A, B, transpose_a != 0);
        std::memcpy(c, C.data.data(), C.data.size() * sizeof(double));
    });
}

int ref_gemv_strided_batch(int rows, int cols, int batch, const double* a, const double* x,
                           double* y, int accumulate) {
    return guarded([&] {
        DenseBatch A(rows, cols, batch);
        std::memcpy(A.data.data(), a, A.data.size() * sizeof(double));
        std::vector<double> xv(x, x + static_cast<std::size_t>(cols) * batch);
        std::vector<double> yv(y, y + static_cast<std::size_t>(rows) * batch);
        gemv_strided_batch(A, xv, yv, accumulate != 0);
        std::memcpy(y, yv.data(), yv.size() * sizeof(double));
    });
}

void ref_random_vector(long n, std::uint64_t seed, double scale, double* out) {
    const auto v = hdg::testing::random_vector(static_cast<std::size_t>(n), seed, scale);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
}

int ref_gauss_rule(int q, double* pts, double* wts) {
    return guarded([&] {
        const QuadratureRule r = gauss_rule(q);
        std::memcpy(pts, r.points.data(), q * sizeof(double));
        std::memcpy(wts, r.weights.data(), q * sizeof(double));
    });
}

int ref_lobatto_nodes(int n, double* out) {
    return guarded([&] {
        const auto v = lobatto_nodes(n);
        std::memcpy(out, v.data(), n * sizeof(double));
    });
}

// Leja ordering of interleaved (re, im) pairs; returns the output count.
int ref_leja_order(int n, const double* in_reim, double* out_reim) {
    std::vector<std::complex<double>> th(n);
    for (int i = 0; i < n; ++i) th[i] = {in_reim[2 * i], in_reim[2 * i + 1]};
    const auto out = leja_order(th);
    for (std::size_t i = 0; i < out.size(); ++i) {
        out_reim[2 * i] = out[i].real();
        out_reim[2 * i + 1] = out[i].imag();
    }
    return static_cast<int>(out.size());
}

// Harmonic Ritz values of a dense row-major n x n operator. Returns count or -1.
int ref_harmonic_ritz_dense(int n, const double* a, int degree, std::uint64_t seed,
                            double* out_reim) {
    int count = -1;
    guarded([&] {
        const LinearOp op = [&](const std::vector<double>& x, std::vector<double>& y) {
            y.assign(n, 0.0);
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) y[i] += a[static_cast<std::size_t>(i) * n + j] * x[j];
        };
        const auto vals = compute_harmonic_ritz(op, n, degree, seed);
        for (std::size_t i = 0; i < vals.size(); ++i) {
            out_reim[2 * i] = vals[i].real();
            out_reim[2 * i + 1] = vals[i].imag();
        }
        count = static_cast<int>(vals.size());
    });
    return count;
}

// GMRES on a dense row-major operator with optional dense row-major preconditioner.
int ref_gmres_dense(int n, const double* a, const double* pinv, const double* rhs,
                    const double* x0, int restart, double tol, int max_iters, int mgs,
                    double* x_out, double* stats_out /*iters,restarts,final_rel,converged*/) {
    return guarded([&] {
        const auto mul = [n](const double* m, const std::vector<double>& x, std::vector<double>& y) {
            y.assign(n, 0.0);
            for (int i = 0; i < n; ++i) {
                double acc = 0.0;
                for (int j = 0; j < n; ++j) acc += m[static_cast<std::size_t>(i) * n + j] * x[j];
                y[i] = acc;
            }
        };
        const OpFn mv = [&](const std::vector<double>& x, std::vector<double>& y) { mul(a, x, y); };
        const OpFn pc = [&](const std::vector<double>& x, std::vector<double>& y) {
            if (pinv) mul(pinv, x, y); else y = x;
        };
        GmresConfig cfg;
        cfg.restart = restart; cfg.tol = tol; cfg.max_iters = max_iters;
        cfg.orth = mgs ? Orth::MGS : Orth::CGS;
        std::vector<double> r(rhs, rhs + n), x(n, 0.0);
        if (x0) x.assign(x0, x0 + n);
        auto [sol, st] = gmres_solve(mv, pc, r, x, cfg);
        std::memcpy(x_out, sol.data(), n * sizeof(double));
        stats_out[0] = st.iters; stats_out[1] = st.restarts;
        stats_out[2] = st.final_rel_residual; stats_out[3] = st.converged ? 1.0 : 0.0;
    });
}

// ---- case handle -----------------------------------------------------------------------------
void* ref_case_create(const char* case_name, int k, int n, double tau /*NaN = default*/,
                      double nu, double kappa, double vx, double vy, int quad_points) {
    RefCase* c = nullptr;
    guarded([&] {
        auto p = std::make_unique<RefCase>();
        p->spec.case_name = case_name;
        p->spec.k = k;
        p->spec.n = n;
        if (!std::isnan(tau)) p->spec.tau = tau;
        p->spec.nu = nu;
        p->spec.kappa = kappa;
        p->spec.velocity = {vx, vy};
        p->spec.quad_points = quad_points;
        p->setup = make_case_setup(p->spec);
        p->state = make_initial_state(p->spec, p->setup);
        c = p.release();
    });
    return c;
}

void ref_case_free(void* h) { delete static_cast<RefCase*>(h); }

// dims: ne, nf, pe, pf, qe, qf
void ref_case_dims(void* h, int* out) {
    auto* c = static_cast<RefCase*>(h);
    out[0] = c->setup.mesh.n_elements; out[1] = c->setup.mesh.n_faces;
    out[2] = c->setup.basis.pe; out[3] = c->setup.basis.pf;
    out[4] = c->setup.basis.qe; out[5] = c->setup.basis.qf;
}

// Copies the named double array into out (if non-null); returns its length, -1 if cap is too
// small, -2 for an unknown name.
long ref_case_get(void* h, const char* name, double* out, long cap) {
    auto* c = static_cast<RefCase*>(h);
    const std::string s = name;
    const auto& b = c->setup.basis;
    const auto& g = c->setup.geom;
    const auto& f = c->setup.factors;
    const auto& o = c->ops;
    if (s == "phi") return copy_out(b.phi, out, cap);
    if (s == "dphi_dxi") return copy_out(b.dphi_dxi, out, cap);
    if (s == "dphi_deta") return copy_out(b.dphi_deta, out, cap);
    if (s == "psi") return copy_out(b.psi, out, cap);
    if (s == "trace_phi0") return copy_out(b.trace_phi[0], out, cap);
    if (s == "trace_phi1") return copy_out(b.trace_phi[1], out, cap);
    if (s == "trace_phi2") return copy_out(b.trace_phi[2], out, cap);
    if (s == "trace_phi3") return copy_out(b.trace_phi[3], out, cap);
    if (s == "nodes1d") return copy_out(b.nodes1d, out, cap);
    if (s == "rule1d_points") return copy_out(b.rule1d.points, out, cap);
    if (s == "rule1d_weights") return copy_out(b.rule1d.weights, out, cap);
    if (s == "rule2d_weights") return copy_out(b.rule2d.weights, out, cap);
    if (s == "elem_detjac") return copy_out(g.elem_detjac, out, cap);
    if (s == "elem_invjac") return copy_out(g.elem_invjac, out, cap);
    if (s == "elem_coords") return copy_out(g.elem_coords, out, cap);
    if (s == "face_detjac") return copy_out(g.face_detjac, out, cap);
    if (s == "face_coords") return copy_out(g.face_coords, out, cap);
    if (s == "face_normal") return copy_out(g.face_normal, out, cap);
    if (s == "mass") return copy_out(f.mass.data, out, cap);
    if (s == "mass_inv") return copy_out(f.mass_inv.data, out, cap);
    if (s == "bmat0") return copy_out(f.bmat[0].data, out, cap);
    if (s == "bmat1") return copy_out(f.bmat[1].data, out, cap);
    if (s == "cmat0") return copy_out(f.cmat[0].data, out, cap);
    if (s == "cmat1") return copy_out(f.cmat[1].data, out, cap);
    if (s == "minv_b0") return copy_out(f.minv_b[0].data, out, cap);
    if (s == "minv_b1") return copy_out(f.minv_b[1].data, out, cap);
    if (s == "minv_c0") return copy_out(f.minv_c[0].data, out, cap);
    if (s == "minv_c1") return copy_out(f.minv_c[1].data, out, cap);
    if (s == "u") return copy_out(c->state.u, out, cap);
    if (s == "q0") return copy_out(c->state.q[0], out, cap);
    if (s == "q1") return copy_out(c->state.q[1], out, cap);
    if (s == "uhat") return copy_out(c->state.uhat, out, cap);
    if (s == "kbar") return copy_out(o.kbar.data, out, cap);
    if (s == "ebar_inv") return copy_out(o.ebar_inv.data, out, cap);
    if (s == "fbar") return copy_out(o.fbar.data, out, cap);
    if (s == "hbar") return copy_out(o.hbar.data, out, cap);
    if (s == "rbar") return copy_out(o.rbar, out, cap);
    if (s == "ru") return copy_out(o.ru, out, cap);
    if (s == "ruhat_e") return copy_out(o.ruhat_e, out, cap);
    if (s == "e_raw") return copy_out(o.e_raw.data, out, cap);
    if (s == "f_raw") return copy_out(o.f_raw.data, out, cap);
    if (s == "h_raw") return copy_out(o.h_raw.data, out, cap);
    if (s == "j_raw") return copy_out(o.j_raw.data, out, cap);
    if (s == "d_raw0") return copy_out(o.d_raw[0].data, out, cap);
    if (s == "d_raw1") return copy_out(o.d_raw[1].data, out, cap);
    if (s == "g_raw0") return copy_out(o.g_raw[0].data, out, cap);
    if (s == "g_raw1") return copy_out(o.g_raw[1].data, out, cap);
    if (s == "k_blocks") return copy_out(c->k.blocks.data, out, cap);
    if (s == "rhs") return copy_out(c->rhs, out, cap);
    if (s == "bj_inv") return copy_out(c->prec.bj_inv.data, out, cap);
    if (s == "asm_inv") return copy_out(c->prec.asm_inv.data, out, cap);
    if (s == "ritz") {
        std::vector<double> v;
        for (const auto& t : c->prec.ritz) { v.push_back(t.real()); v.push_back(t.imag()); }
        return copy_out(v, out, cap);
    }
    if (s == "vertex_coords") {
        std::vector<double> v;
        for (const auto& p : c->setup.mesh.vertex_coords) { v.push_back(p[0]); v.push_back(p[1]); }
        return copy_out(v, out, cap);
    }
    if (s == "residual_history") return copy_out(c->report.residual_history, out, cap);
    if (s == "alpha_history") return copy_out(c->report.alpha_history, out, cap);
    return -2;
}

long ref_case_get_i(void* h, const char* name, std::int64_t* out, long cap) {
    auto* c = static_cast<RefCase*>(h);
    const std::string s = name;
    const auto& m = c->setup.mesh;
    std::vector<std::int64_t> v;
    auto from = [&](const std::vector<int>& a) { v.assign(a.begin(), a.end()); };
    if (s == "element_to_face") from(flatten(m.element_to_face));
    else if (s == "element_vertices") from(flatten(m.element_vertices));
    else if (s == "face_to_elements") from(flatten(m.face_to_elements));
    else if (s == "face_local_index") from(flatten(m.face_local_index));
    else if (s == "face_side_reversed") from(flatten(m.face_side_reversed));
    else if (s == "face_vertices") from(flatten(m.face_vertices));
    else if (s == "boundary_tag") from(m.boundary_tag);
    else if (s == "neighbor") v = c->k.neighbor;
    else if (s == "gmres_per_newton") from(c->report.gmres_per_newton);
    else return -2;
    if (out) {
        if (cap < static_cast<long>(v.size())) return -1;
        std::memcpy(out, v.data(), v.size() * sizeof(std::int64_t));
    }
    return static_cast<long>(v.size());
}

int ref_case_set(void* h, const char* name, const double* in, long n) {
    auto* c = static_cast<RefCase*>(h);
    const std::string s = name;
    std::vector<double>* dst = nullptr;
    if (s == "u") dst = &c->state.u;
    else if (s == "uhat") dst = &c->state.uhat;
    else if (s == "u_prev") { c->u_prev.assign(in, in + n); return 0; }
    else if (s == "k_blocks") dst = &c->k.blocks.data;
    else if (s == "rhs") dst = &c->rhs;
    else return -2;
    if (static_cast<long>(dst->size()) != n) return -1;
    std::memcpy(dst->data(), in, n * sizeof(double));
    return 0;
}

void ref_case_set_dt(void* h, double dt /* <=0 or NaN: steady */) {
    auto* c = static_cast<RefCase*>(h);
    if (dt > 0.0) { c->dt = dt; if (c->u_prev.empty()) c->u_prev = c->state.u; }
    else c->dt.reset();
}

void ref_case_reset_state(void* h) {
    auto* c = static_cast<RefCase*>(h);
    c->state = make_initial_state(c->spec, c->setup);
}

// state.u += scale*rand(seed), state.uhat += scale*rand(seed+1)  (test_helpers.hpp:33-38)
void ref_case_perturb(void* h, std::uint64_t seed, double scale) {
    auto* c = static_cast<RefCase*>(h);
    const auto du = hdg::testing::random_vector(c->state.u.size(), seed, scale);
    const auto dh = hdg::testing::random_vector(c->state.uhat.size(), seed + 1, scale);
    for (std::size_t i = 0; i < du.size(); ++i) c->state.u[i] += du[i];
    for (std::size_t i = 0; i < dh.size(); ++i) c->state.uhat[i] += dh[i];
}

int ref_case_compute_q(void* h) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] { compute_q(c->state, c->setup.factors, c->setup.mesh); });
}

int ref_case_assemble(void* h, int keep_raw) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        c->ops = assemble_element_operators(c->setup.model, c->state, c->setup.mesh,
                                            c->setup.basis, c->setup.geom, c->setup.factors,
                                            c->time(), keep_raw != 0);
        auto [k, rhs] = assemble_global(c->ops, c->setup.mesh);
        c->k = std::move(k);
        c->rhs = std::move(rhs);
        c->assembled = true;
    });
}

// Only the local stage (for timing): assemble + condense, no global assembly.
int ref_case_assemble_local(void* h) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        c->ops = assemble_element_operators(c->setup.model, c->state, c->setup.mesh,
                                            c->setup.basis, c->setup.geom, c->setup.factors,
                                            c->time(), false);
    });
}

int ref_case_assemble_global(void* h) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        auto [k, rhs] = assemble_global(c->ops, c->setup.mesh);
        c->k = std::move(k);
        c->rhs = std::move(rhs);
        c->assembled = true;
    });
}

int ref_case_residual(void* h, double* trace, double* interior, double* norm) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        Residuals r = assemble_residual(c->setup.model, c->state, c->setup.mesh, c->setup.basis,
                                        c->setup.geom, c->setup.factors, c->time());
        if (trace) std::memcpy(trace, r.trace.data(), r.trace.size() * sizeof(double));
        if (interior) std::memcpy(interior, r.interior.data(), r.interior.size() * sizeof(double));
        if (norm) *norm = residual_norm(r);
    });
}

int ref_case_matvec(void* h, const double* x, double* y) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        TraceVector xv(x, x + c->k.n_dof());
        TraceVector yv = block_matvec(c->k, xv);
        std::memcpy(y, yv.data(), yv.size() * sizeof(double));
    });
}

long ref_case_to_dense(void* h, double* out, long cap) {
    auto* c = static_cast<RefCase*>(h);
    long n = -1;
    guarded([&] { n = copy_out(to_dense(c->k), out, cap); });
    return n;
}

int ref_case_gather_extended(void* h, const double* x, double* out) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        TraceVector xv(x, x + c->k.n_dof());
        const auto g = gather_extended(xv, c->k);
        std::memcpy(out, g.data(), g.size() * sizeof(double));
    });
}

// kind: 0 identity, 1 BJ, 2 ASM
int ref_case_build_precond(void* h, int kind, int poly_degree, std::uint64_t seed) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        PrecondSpec spec;
        spec.kind = kind == 0 ? PrecondKind::Identity : (kind == 1 ? PrecondKind::BJ : PrecondKind::ASM);
        spec.poly_degree = poly_degree;
        spec.ritz_seed = seed;
        c->prec = build_preconditioner(spec, c->k, c->ops, c->setup.mesh);
    });
}

// Overrides the interpolation nodes of the built preconditioner (interleaved re/im, already ordered): lets the
// reference's own apply_poly run with externally supplied nodes (Chebyshev variant, fixed-node parity tests).
int ref_case_set_ritz(void* h, const double* reim, int count) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        c->prec.ritz.clear();
        for (int i = 0; i < count; ++i) c->prec.ritz.emplace_back(reim[2 * i], reim[2 * i + 1]);
        c->prec.poly_degree = count;
    });
}

int ref_case_apply_base(void* h, const double* y, double* z) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        const LinearOp base = make_base_apply(c->prec, c->setup.mesh);
        std::vector<double> yv(y, y + c->k.n_dof()), zv;
        base(yv, zv);
        std::memcpy(z, zv.data(), zv.size() * sizeof(double));
    });
}

int ref_case_apply_precond(void* h, const double* y, double* z) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        const LinearOp app = make_preconditioner_apply(c->prec, c->k, c->setup.mesh, &c->inner_ops);
        std::vector<double> yv(y, y + c->k.n_dof()), zv;
        app(yv, zv);
        std::memcpy(z, zv.data(), zv.size() * sizeof(double));
    });
}

int ref_case_gather_element_trace(void* h, const double* face_values, double* out) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        std::vector<double> fv(face_values, face_values + c->k.n_dof());
        const auto g = gather_element_trace(c->setup.mesh, c->setup.basis.pf, fv);
        std::memcpy(out, g.data(), g.size() * sizeof(double));
    });
}

int ref_case_recover_local(void* h, const double* duhat, double* du) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        std::vector<double> dh(duhat, duhat + c->k.n_dof());
        const auto g = gather_element_trace(c->setup.mesh, c->setup.basis.pf, dh);
        const auto d = recover_local(c->ops, g);
        std::memcpy(du, d.data(), d.size() * sizeof(double));
    });
}

// stats_out: iters, restarts, final_rel_residual, converged, t_mv, t_prec, t_orth
int ref_case_gmres(void* h, const double* rhs, const double* x0, int restart, double tol,
                   int max_iters, int mgs, double* x_out, double* stats_out) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        const std::size_t n = c->k.n_dof();
        std::vector<double> gather;
        const OpFn mv = [&](const std::vector<double>& in, std::vector<double>& out) {
            block_matvec(c->k, in, out, gather);
        };
        const OpFn app = make_preconditioner_apply(c->prec, c->k, c->setup.mesh, &c->inner_ops);
        GmresConfig cfg;
        cfg.restart = restart; cfg.tol = tol; cfg.max_iters = max_iters;
        cfg.orth = mgs ? Orth::MGS : Orth::CGS;
        std::vector<double> r = rhs ? std::vector<double>(rhs, rhs + n) : c->rhs;
        std::vector<double> x(n, 0.0);
        if (x0) x.assign(x0, x0 + n);
        auto [sol, st] = gmres_solve(mv, app, r, x, cfg);
        std::memcpy(x_out, sol.data(), n * sizeof(double));
        stats_out[0] = st.iters; stats_out[1] = st.restarts;
        stats_out[2] = st.final_rel_residual; stats_out[3] = st.converged ? 1.0 : 0.0;
        stats_out[4] = st.t_mv; stats_out[5] = st.t_prec; stats_out[6] = st.t_orth;
    });
}

// report_out: n_newton, n_gmres_total, n_inner_prec_ops, final_residual, converged,
//             t_ass, t_mv, t_prec, t_orth, t_total
int ref_case_newton(void* h, double newton_tol, int max_newton, double min_alpha, int restart,
                    double gmres_tol, int gmres_max_iters, int mgs, int pkind, int poly_degree,
                    std::uint64_t seed, int ritz_per_restart, double* report_out) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        NewtonConfig ncfg;
        ncfg.tol = newton_tol; ncfg.max_newton = max_newton; ncfg.min_alpha = min_alpha;
        GmresConfig gcfg;
        gcfg.restart = restart; gcfg.tol = gmres_tol; gcfg.max_iters = gmres_max_iters;
        gcfg.orth = mgs ? Orth::MGS : Orth::CGS;
        PrecondSpec ps;
        ps.kind = pkind == 0 ? PrecondKind::Identity : (pkind == 1 ? PrecondKind::BJ : PrecondKind::ASM);
        ps.poly_degree = poly_degree; ps.ritz_seed = seed; ps.ritz_per_restart = ritz_per_restart != 0;
        c->report = newton_solve(c->setup.model, c->setup.mesh, c->setup.basis, c->setup.geom,
                                 c->setup.factors, c->state, ncfg, gcfg, ps, c->time());
        const SolveReport& r = c->report;
        report_out[0] = r.n_newton; report_out[1] = static_cast<double>(r.n_gmres_total);
        report_out[2] = static_cast<double>(r.n_inner_prec_ops); report_out[3] = r.final_residual;
        report_out[4] = r.converged ? 1.0 : 0.0; report_out[5] = r.t_ass; report_out[6] = r.t_mv;
        report_out[7] = r.t_prec; report_out[8] = r.t_orth; report_out[9] = r.t_total;
    });
}

// Backward-Euler marching (newton.cpp:156-175); report_out as above, summed over steps.
int ref_case_time_march(void* h, double dt, int n_steps, double newton_tol, int max_newton,
                        int restart, double gmres_tol, int gmres_max_iters, int pkind,
                        int poly_degree, double* report_out) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] {
        NewtonConfig ncfg;
        ncfg.tol = newton_tol; ncfg.max_newton = max_newton; ncfg.dt = dt; ncfg.n_steps = n_steps;
        GmresConfig gcfg;
        gcfg.restart = restart; gcfg.tol = gmres_tol; gcfg.max_iters = gmres_max_iters;
        PrecondSpec ps;
        ps.kind = pkind == 0 ? PrecondKind::Identity : (pkind == 1 ? PrecondKind::BJ : PrecondKind::ASM);
        ps.poly_degree = poly_degree;
        const auto reps = time_march(c->setup.model, c->setup.mesh, c->setup.basis, c->setup.geom,
                                     c->setup.factors, c->state, ncfg, gcfg, ps);
        for (int i = 0; i < 10; ++i) report_out[i] = 0.0;
        report_out[4] = 1.0;
        for (const auto& r : reps) {
            report_out[0] += r.n_newton; report_out[1] += static_cast<double>(r.n_gmres_total);
            report_out[2] += static_cast<double>(r.n_inner_prec_ops); report_out[3] = r.final_residual;
            if (!r.converged) report_out[4] = 0.0;
            report_out[5] += r.t_ass; report_out[6] += r.t_mv; report_out[7] += r.t_prec;
            report_out[8] += r.t_orth; report_out[9] += r.t_total;
        }
    });
}

// The reference tests' own monolithic oracle (tests/oracles.cpp:68-130): row-major n x n.
long ref_case_monolithic(void* h, double* a, double* rhs, long cap_n) {
    auto* c = static_cast<RefCase*>(h);
    long n = -1;
    guarded([&] {
        auto sys = hdg::testing::build_monolithic_dense(c->setup.model, c->state, c->setup.mesh,
                                                        c->setup.basis, c->setup.geom,
                                                        c->setup.factors, c->time());
        n = sys.n;
        if (a && rhs && cap_n >= n) {
            std::memcpy(a, sys.a.data(), sys.a.size() * sizeof(double));
            std::memcpy(rhs, sys.rhs.data(), sys.rhs.size() * sizeof(double));
        }
    });
    return n;
}

int ref_case_write_matrix(void* h, const char* path) {
    auto* c = static_cast<RefCase*>(h);
    return guarded([&] { write_matrix(path, c->k, c->rhs); });
}

double ref_case_l2_error(void* h) {
    auto* c = static_cast<RefCase*>(h);
    double v = -1.0;
    guarded([&] {
        if (c->setup.model.exact_solution)
            v = l2_error(c->state.u, c->setup.model.exact_solution, c->setup.mesh, c->setup.basis);
    });
    return v;
}

}  // extern "C"
