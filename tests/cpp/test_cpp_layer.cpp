// Exercises include/hdgb200.hpp (the C++ mirror of the reference's namespace-hdg API) end to end on the GPU:
// the same calls a reference test makes (tests/test_newton.cpp, test_face_matrix.cpp, test_dense_batch.cpp),
// with the reference's error behaviour (exception type + offending batch index).
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "hdgb200.hpp"

using namespace hdg::b200;

static int fails = 0;
#define EXPECT(cond)                                                        \
    do {                                                                    \
        if (!(cond)) { std::printf("FAILED %s:%d  %s\n", __FILE__, __LINE__, #cond); ++fails; } \
    } while (0)

int main() {
    Context ctx(0);
    // ---- BASELINE config 1 in miniature: 2D Poisson, quads, p = 2, block-Jacobi GMRES ----
    Discretization disc = Discretization::structured(ctx, HDGB_QUAD, 16, 2);
    const auto xq = disc.table_f64("elem_coords");
    const auto xf = disc.table_f64("face_coords");
    const double pi = 3.14159265358979323846;
    std::vector<double> forcing(xq.size() / 2), dirichlet(xf.size() / 2);
    for (size_t i = 0; i < forcing.size(); ++i) forcing[i] = 2 * pi * pi * std::sin(pi * xq[2 * i]) * std::sin(pi * xq[2 * i + 1]);
    for (size_t i = 0; i < dirichlet.size(); ++i) dirichlet[i] = std::sin(pi * xf[2 * i]) * std::sin(pi * xf[2 * i + 1]);
    Model model(disc, HDGB_MODEL_POISSON, {1.0}, &forcing, &dirichlet);
    StateFields state(disc);
    PrecondSpec bj;  // default BJ
    const SolveReport rep = newton_solve(model, disc, state, NewtonConfig{}, GmresConfig{}, bj);
    EXPECT(rep.converged);
    EXPECT(rep.n_newton == 1);
    EXPECT(rep.final_residual <= 1e-8);
    EXPECT(rep.gmres_per_newton.size() == 1 && rep.gmres_per_newton[0] == rep.n_gmres_total);
    EXPECT(rep.residual_history.size() == 2);
    std::printf("newton_solve: newton=%d gmres=%ld residual=%.3e\n", rep.n_newton, rep.n_gmres_total, rep.final_residual);

    // ---- operators one by one ----
    StateFields s2(disc);
    ElementOperators ops = assemble_element_operators(model, s2, disc);
    auto [K, rhs] = assemble_global(ops, disc);
    EXPECT(K.n_dof() == disc.n_dof() && K.nb == disc.nb() && K.block_dim == disc.mpf());
    const auto nbr = K.neighbor();
    bool self_ok = true;
    for (int f = 0; f < K.nf; ++f) self_ok = self_ok && nbr[static_cast<size_t>(f) * K.nb] == f;
    EXPECT(self_ok);
    std::vector<double> x(static_cast<size_t>(K.n_dof())), y(x.size());
    for (size_t i = 0; i < x.size(); ++i) { x[i] = std::sin(0.37 * i); y[i] = std::cos(0.11 * i); }
    const auto Kx = block_matvec(K, x), Ky = block_matvec(K, y);
    std::vector<double> z(x.size());
    for (size_t i = 0; i < x.size(); ++i) z[i] = 2 * x[i] - 3 * y[i];
    const auto Kz = block_matvec(K, z);
    double lin = 0.0, scale = 0.0;
    for (size_t i = 0; i < x.size(); ++i) { lin = std::fmax(lin, std::fabs(Kz[i] - (2 * Kx[i] - 3 * Ky[i]))); scale = std::fmax(scale, std::fabs(Kx[i])); }
    EXPECT(lin <= 1e-12 * scale);
    Preconditioner P = build_preconditioner(bj, K, ops, disc);
    auto [du, stats] = gmres_solve(K, P, rhs, {}, GmresConfig{});
    EXPECT(stats.converged && stats.iters == rep.n_gmres_total);
    // the Newton update of a linear problem from the zero state is the solution itself
    const auto uh = state.get("uhat");
    double diff = 0.0;
    for (size_t i = 0; i < uh.size(); ++i) diff = std::fmax(diff, std::fabs(uh[i] - du[i]));
    EXPECT(diff <= 1e-12);
    const Residuals r0 = assemble_residual(model, state, disc);
    EXPECT(std::fabs(r0.norm - rep.final_residual) <= 1e-14);

    // ---- 3D, additive Schwarz, one backward-Euler step through TimeContext (BASELINE config 2 in miniature) ----
    {
        Discretization d3 = Discretization::structured(ctx, HDGB_HEX, 3, 2);
        const auto x3 = d3.table_f64("elem_coords");
        const auto f3 = d3.table_f64("face_coords");
        std::vector<double> fq(x3.size() / 3), dq(f3.size() / 3);
        for (size_t i = 0; i < fq.size(); ++i)
            fq[i] = 3 * pi * pi * std::sin(pi * x3[3 * i]) * std::sin(pi * x3[3 * i + 1]) * std::sin(pi * x3[3 * i + 2]);
        for (size_t i = 0; i < dq.size(); ++i) dq[i] = std::sin(pi * f3[3 * i]) * std::sin(pi * f3[3 * i + 1]) * std::sin(pi * f3[3 * i + 2]);
        Model m3(d3, HDGB_MODEL_POISSON, {1.0}, &fq, &dq);
        StateFields s3(d3);
        PrecondSpec as;
        as.kind = PrecondKind::ASM;
        const SolveReport r3 = newton_solve(m3, d3, s3, NewtonConfig{}, GmresConfig{}, as);
        EXPECT(r3.converged && r3.final_residual <= 1e-8 && r3.n_gmres_total > 0);
        StateFields s4(d3);
        const std::vector<double> u_prev(static_cast<size_t>(d3.npe()) * d3.dims().ne, 0.0);
        TimeContext tc;
        tc.dt = 0.1;
        tc.u_prev = &u_prev;
        const SolveReport r4 = newton_solve(m3, d3, s4, NewtonConfig{}, GmresConfig{}, as, tc);
        EXPECT(r4.converged);
        // the transient solution after one step differs from the steady one
        const auto ua = s3.get("u"), ub = s4.get("u");
        double dmax = 0.0;
        for (size_t i = 0; i < ua.size(); ++i) dmax = std::fmax(dmax, std::fabs(ua[i] - ub[i]));
        EXPECT(dmax > 1e-3);
        bool threw_t = false;
        TimeContext bad_tc;
        bad_tc.dt = 0.1;  // no previous solution
        try { assemble_element_operators(m3, s4, d3, bad_tc); } catch (const InconsistentDimensions&) { threw_t = true; }
        EXPECT(threw_t);
        std::printf("hex ASM: steady newton=%d gmres=%ld, transient newton=%d\n", r3.n_newton, r3.n_gmres_total, r4.n_newton);
    }

    // ---- the per-function preconditioner API and the closure forms (preconditioner.hpp:31-76, gmres.hpp:50-53) ----
    {
        Preconditioner pbj = build_bj(K);
        Preconditioner pspec = build_preconditioner(bj, K, ops, disc);
        const std::vector<double> yv = rhs;
        const auto z1 = apply_bj(ctx, pbj, yv), z2 = apply_preconditioner(pspec, K, yv);
        double dz = 0.0;
        for (size_t i = 0; i < z1.size(); ++i) dz = std::fmax(dz, std::fabs(z1[i] - z2[i]));
        EXPECT(dz == 0.0);  // same kernels, same data: bit-identical
        Preconditioner pasm = build_asm(ops, disc);
        PrecondSpec as_spec;
        as_spec.kind = PrecondKind::ASM;
        Preconditioner pasm2 = build_preconditioner(as_spec, K, ops, disc);
        const auto a1 = apply_asm(ctx, pasm, yv), a2 = apply_preconditioner(pasm2, K, yv);
        double da = 0.0, amax = 0.0;
        for (size_t i = 0; i < a1.size(); ++i) { da = std::fmax(da, std::fabs(a1[i] - a2[i])); amax = std::fmax(amax, std::fabs(a2[i])); }
        EXPECT(da <= 1e-12 * std::fmax(1.0, amax));  // enrichment summed from K-bar vs read from K: same terms, same order
        bool wrong_kind = false;
        try { apply_asm(ctx, pbj, yv); } catch (const DimensionMismatch&) { wrong_kind = true; }
        EXPECT(wrong_kind);

        // closure-form GMRES == handle-form GMRES (identical operators, identical control flow)
        GmresConfig gc;
        gc.tol = 1e-10;
        const DeviceOp mv = make_matvec(K), pc = make_base_apply(ctx, pbj);
        std::vector<double> trace;
        const auto [xc, sc] = gmres_solve(ctx, mv, pc, rhs, {}, gc, &trace);
        const auto [xh, sh] = gmres_solve(K, pbj, rhs, {}, gc);
        EXPECT(sc.converged && sh.converged && sc.iters == sh.iters);
        EXPECT(trace.size() == static_cast<size_t>(sc.iters));
        double dx = 0.0;
        for (size_t i = 0; i < xc.size(); ++i) dx = std::fmax(dx, std::fabs(xc[i] - xh[i]));
        EXPECT(dx == 0.0);
        // a throwing closure surfaces as the caller's exception, not as a crash across the C boundary
        bool surfaced = false;
        const DeviceOp bad = [](const double*, double*, std::int64_t) { throw std::runtime_error("boom"); };
        try { gmres_solve(ctx, bad, DeviceOp(), rhs, {}, gc); } catch (const std::runtime_error& e) { surfaced = std::string(e.what()) == "boom"; }
        EXPECT(surfaced);

        // harmonic Ritz values of the BJ-preconditioned operator through the closure form == the spec form
        PrecondSpec poly = bj;
        poly.poly_degree = 6;
        Preconditioner ppoly = build_preconditioner(poly, K, ops, disc);
        double* tmp = nullptr;
        check(ctx.get(), hdgb_device_alloc(ctx.get(), K.n_dof(), &tmp));
        const DeviceOp op = [&](const double* in, double* out, std::int64_t n) { mv(in, tmp, n); pc(tmp, out, n); };
        const auto th = compute_harmonic_ritz(ctx, op, static_cast<size_t>(K.n_dof()), 6, 12345);
        std::int64_t nr = 0;
        check(ctx.get(), hdgb_precond_get(ppoly.handle(), "ritz", nullptr, 0, &nr));
        std::vector<double> reim(static_cast<size_t>(nr));
        check(ctx.get(), hdgb_precond_get(ppoly.handle(), "ritz", reim.data(), nr, &nr));
        EXPECT(th.size() * 2 == reim.size());
        for (size_t i = 0; i < th.size() && 2 * i + 1 < reim.size(); ++i) EXPECT(th[i].real() == reim[2 * i] && th[i].imag() == reim[2 * i + 1]);
        // apply_poly with the closure base == the wrapped application
        long inner = 0;
        const auto w1 = apply_poly(ppoly, &pc, K, yv, &inner), w2 = apply_preconditioner(ppoly, K, yv);
        double dw = 0.0;
        for (size_t i = 0; i < w1.size(); ++i) dw = std::fmax(dw, std::fabs(w1[i] - w2[i]));
        EXPECT(dw == 0.0 && inner == static_cast<long>(th.size()));
        hdgb_device_free(ctx.get(), tmp);
        const auto lj = leja_order({{1, 0}, {10, 0}, {5, 0}});
        EXPECT(lj.size() == 3 && lj[0].real() == 10 && lj[1].real() == 1 && lj[2].real() == 5);  // test_precond.cpp Leja unit case
        std::printf("closure forms: gmres iters=%d (handle form %d), ritz=%zu, inner ops=%ld\n", sc.iters, sh.iters, th.size(), inner);
    }

    // ---- error behaviour ----
    bool threw = false;
    try { block_matvec(K, std::vector<double>(3)); } catch (const DimensionMismatch&) { threw = true; }
    EXPECT(threw);
    const int n = 5, batch = 4;
    std::vector<double> a(static_cast<size_t>(n) * n * batch, 0.0);
    for (int b = 0; b < batch; ++b)
        for (int i = 0; i < n; ++i) a[static_cast<size_t>(b) * n * n + i * n + i] = (b == 2) ? 0.0 : 2.0 + b;  // block 2 singular
    long bad = -1;
    try { lu_invert_batch(ctx, a, n, batch); } catch (const SingularBlock& e) { bad = e.index; }
    EXPECT(bad == 2);  // lowest failing batch index (dense_batch.cpp:84-97)
    for (int i = 0; i < n; ++i) a[2 * n * n + i * n + i] = 4.0;
    const auto inv = lu_invert_batch(ctx, a, n, batch);
    EXPECT(std::fabs(inv[0] - 0.5) <= 1e-15 && std::fabs(inv[2 * n * n] - 0.25) <= 1e-15);

    std::printf(fails ? "%d check(s) failed\n" : "all checks passed\n", fails);
    return fails ? 1 : 0;
}
