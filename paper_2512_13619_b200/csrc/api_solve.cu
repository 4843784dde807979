// C ABI: restarted GMRES (A13) and the Newton / time-marching drivers (A14).
//
// The Krylov basis, the operator and the preconditioner live on the device.  Per Arnoldi step the
// host sees exactly one small transfer (the Hessenberg column: projection coefficients of both
// Gram-Schmidt passes and the squared norm) -- Givens rotations, the convergence test and the
// back-substitution are host scalars like in the reference (gmres.cpp:135-166,188-193).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "solver.cuh"

using namespace hdgb;

namespace hdgb {

namespace {

GmresWork& gmres_work(hdgb_matrix* k, int restart) {
    const int64_t n = k->n_dof();
    if (!k->work || k->work->restart < restart || k->work->n != n) k->work = make_gmres_work(k->ctx, n, k->n_local(), restart);
    return *k->work;
}

// orthogonalize (gmres.cpp:28-59) of w against V[0..nvec); h (host) gets nvec + 1 entries.
// CGS mode: both projection passes are batched (c = V^T w; w -= V c; d = V^T w; w -= V d); the reference's second
// pass interleaves dot and update, which differs at O(eps^2) relative.  Three streamed passes over the basis
// (k_orth.cu: the first update and the second projection share one read of V), the four-pass kernels of k_vec.cu
// for shapes the streamed kernel declines.  MGS mode follows the reference sequence exactly.
// n = owned unknowns (what the sums run over), ldv = distance between basis vectors.
// With a communicator (domain decomposition) an Arnoldi step costs TWO all-reduces: c, then [d, ||w1||^2] together --
// the norm of the twice-projected vector follows from Pythagoras, ||w2||^2 = ||w1||^2 - ||d||^2 (V orthonormal), so
// the last pass already writes the normalised vector; if that difference cancels badly (w almost in span V: the
// happy-breakdown regime) the norm is re-measured explicitly.
// coef: 2 nvec + 2 device scalars  c | d | s0 | s1 ;  cgs: workspace of the streamed passes or nullptr.
// between (may be null): called once the column's device-to-host copy and the normalisation are enqueued and before
// the host waits for them -- the caller enqueues the next step's operator applications there, so the device does
// not idle while the host reads the column and issues the next launches.
void orthogonalize_device(hdgb_ctx* c, const double* V, int64_t ldv, int nvec, int64_t n, double* w, int orth,
                          double* coef, double* partial, double* cgs, double* h,
                          const std::function<void()>* between = nullptr) {
    double* dc = coef;
    double* dd = coef + nvec;
    double* s0 = coef + 2 * nvec;
    double* s1 = s0 + 1;
    double* stage = c->pinned;
    auto reduce = [&](double* dev, int cnt) { if (c->comm) c->comm->allreduce(c, dev, cnt); };
    auto wait = [&] {
        if (tuning().spin_sync) host_wait(c);
        else HDGB_CUDA(cudaStreamSynchronize(c->stream));
    };
    const bool streamed = orth != 1 && cgs && tuning().cgs_stream && cgs_pass_supported(V, ldv, nvec, w, n);
    if (streamed && c->comm) {
        launch_cgs_pass(c, 0, V, ldv, nvec, w, n, nullptr, dc, cgs);
        reduce(dc, nvec);
        launch_cgs_pass(c, 1, V, ldv, nvec, w, n, dc, dd, cgs);  // dd[nvec] == s0 = ||w1||^2 (owned rows)
        reduce(dd, nvec + 1);
        launch_cgs_pass(c, 3, V, ldv, nvec, w, n, dd, s1, cgs);  // w normalised, s1 = ||w1||^2 - ||d||^2
        HDGB_CUDA(cudaMemcpyAsync(stage, coef, (2 * nvec + 2) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        wait();
        double w1n2 = stage[2 * nvec], t = stage[2 * nvec + 1];
        double hn = std::sqrt(t);
        if (!(t > 1e-3 * w1n2)) {
            // severe cancellation: measure ||w|| of what pass 3 left (w2 * s, or w2 itself when t <= 0)
            launch_sumsq(c, w, n, s0, partial);
            reduce(s0, 1);
            HDGB_CUDA(cudaMemcpyAsync(stage + 2 * nvec, s0, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            launch_scale_dev(c, w, s0, 0, w, n);
            wait();
            const double m2 = stage[2 * nvec];  // ||w2||^2 * s^2
            hn = t > 0.0 ? std::sqrt(m2 * t) : std::sqrt(m2);
        }
        for (int i = 0; i < nvec; ++i) h[i] = stage[i] + stage[nvec + i];
        h[nvec] = hn;
        return;
    }
    if (orth == 1) {
        for (int i = 0; i < nvec; ++i) {
            const double* vi = V + static_cast<size_t>(i) * ldv;
            launch_multi_dot(c, vi, ldv, 1, w, n, dc + i, partial);
            reduce(dc + i, 1);
            launch_multi_axpy(c, vi, ldv, 1, dc + i, -1.0, w, n, nullptr, partial);
        }
        launch_sumsq(c, w, n, s0, partial);
        reduce(s0, 1);
        HDGB_CUDA(cudaMemsetAsync(dd, 0, nvec * sizeof(double), c->stream));
    } else if (streamed) {
        launch_cgs_pass(c, 0, V, ldv, nvec, w, n, nullptr, dc, cgs);
        launch_cgs_pass(c, 1, V, ldv, nvec, w, n, dc, dd, cgs);
        launch_cgs_pass(c, 2, V, ldv, nvec, w, n, dd, s0, cgs);
    } else {
        launch_multi_dot(c, V, ldv, nvec, w, n, dc, partial);
        reduce(dc, nvec);
        if (!(tuning().fused_cgs && launch_multi_axpy_dot(c, V, ldv, nvec, dc, w, n, dd, partial))) {
            launch_multi_axpy(c, V, ldv, nvec, dc, -1.0, w, n, nullptr, partial);
            launch_multi_dot(c, V, ldv, nvec, w, n, dd, partial);
        }
        reduce(dd, nvec);
        launch_multi_axpy(c, V, ldv, nvec, dd, -1.0, w, n, s0, partial);
        reduce(s0, 1);
    }
    // normalise on the device (no-op when the norm is zero, gmres.cpp:54-57) while the column
    // travels to the host
    HDGB_CUDA(cudaMemcpyAsync(stage, coef, (2 * nvec + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    launch_scale_dev(c, w, s0, 0, w, n);
    if (between && host_mark(c)) {
        (*between)();
        host_poll(c, tuning().spin_sync != 0);
    } else {
        wait();
    }
    for (int i = 0; i < nvec; ++i) h[i] = stage[i] + stage[nvec + i];
    h[nvec] = std::sqrt(stage[2 * nvec]);
}

}  // namespace

std::unique_ptr<GmresWork> make_gmres_work(hdgb_ctx* c, int64_t n, int64_t ld, int restart) {
    std::unique_ptr<GmresWork> work(new GmresWork());
    GmresWork& w = *work;
    w.restart = restart;
    w.n = n;
    w.basis.alloc(static_cast<size_t>(restart + 1) * ld);
    w.kv.alloc(ld);
    w.r.alloc(ld);
    w.coef.alloc(2 * static_cast<size_t>(restart + 1) + 4);
    w.partial.alloc(multi_dot_workspace_doubles(n, restart + 1));
    w.ycoef.alloc(restart + 1);
    w.cgs.alloc(cgs_workspace_doubles(c));
    w.cgs.zero(c->stream);
    return work;
}

void gmres_device(hdgb_matrix* k, hdgb_precond* p, const double* rhs, double* x, const hdgb_gmres_config& cfg,
                  hdgb_gmres_stats* st, double* residual_trace) {
    if (cfg.restart < 1) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: GMRES restart length must be >= 1");
    GmresWork& W = gmres_work(k, cfg.restart);
    gmres_core(k->ctx, k->n_dof(), k->n_local(), W, [k](const double* in, double* out) { matvec_device(k, in, out); },
               [k, p](const double* in, double* out) { apply_precond_device(p, k, in, out); }, rhs, x, cfg, st, residual_trace,
               p ? &p->inner_ops : &k->spec_dummy);
}

void gmres_core(hdgb_ctx* c, int64_t n, int64_t ld, GmresWork& W, const DevOp& matvec, const DevOp& precond,
                const double* rhs, double* x, const hdgb_gmres_config& cfg, hdgb_gmres_stats* st, double* residual_trace,
                int64_t* spec_counter) {
    const int m = cfg.restart;
    if (m < 1) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: GMRES restart length must be >= 1");
    if (2 * static_cast<size_t>(m + 1) + 4 > c->pinned_doubles) throw Failure(HDGB_ERR_UNSUPPORTED, "GMRES restart length too large");
    std::memset(st, 0, sizeof(*st));
    double* kv = W.kv.p;
    double* r = W.r.p;
    double* V = W.basis.p;
    auto apply_prec = [&](const double* in, double* out) {
        if (precond) precond(in, out);
        else if (in != out) HDGB_CUDA(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    };

    auto norm_of = [&](const double* v) {
        launch_sumsq(c, v, n, W.coef.p, W.partial.p);
        if (c->comm) c->comm->allreduce(c, W.coef.p, 1);
        double s;
        HDGB_CUDA(cudaMemcpyAsync(&s, W.coef.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        return std::sqrt(s);
    };
    // r = P^-1 (rhs - K x)   (gmres.cpp:73-81)
    auto residual = [&](double* out) {
        PhaseTimer tm(c, &st->t_mv);
        matvec(x, kv);
        launch_lincomb(c, 1.0, rhs, -1.0, kv, kv, n);
        tm.stop();
        PhaseTimer tp(c, &st->t_prec);
        apply_prec(kv, out);
        tp.stop();
    };

    residual(r);
    const double beta0 = norm_of(r);
    if (!std::isfinite(beta0)) throw Failure(HDGB_ERR_NAN_DETECTED, "NaN detected in gmres initial residual");
    if (beta0 == 0.0) {
        st->converged = 1;
        return;
    }
    const double target = cfg.tol * beta0;
    std::vector<std::vector<double>> rcols;
    std::vector<double> cs(m), sn(m), g(m + 1), h(m + 2);
    int n_trace = 0;

    bool first_cycle = true;
    while (true) {
        if (!first_cycle) residual(r);
        first_cycle = false;
        const double beta = norm_of(r);
        if (beta <= target) {
            st->converged = 1;
            break;
        }
        if (st->iters >= cfg.max_iters) break;

        rcols.clear();
        launch_axpby(c, 1.0 / beta, r, 0.0, V, n);  // v0 = r / beta
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int nbasis = 1;
        int jused = 0;
        bool cycle_converged = false;
        // Speculative pipelining (handle form, single GPU): the next step's candidate P^-1 K v_{j+1} depends only on
        // the normalised vector the orthogonalisation leaves on the device, so it is enqueued BEFORE the host waits
        // for this step's Hessenberg column; if the column then ends the cycle (convergence, breakdown, iteration
        // cap) the speculative candidate is simply dropped.  spec_counter (the preconditioner's operator count) is
        // rolled back in that case, so the reported statistics are those of the reference's control flow.
        const bool speculate = spec_counter && tuning().gmres_speculate && !c->comm && !c->phase_timing;
        bool have_spec = false;
        int64_t counter_before_spec = 0;
        for (int j = 0; j < m && st->iters < cfg.max_iters; ++j) {
            double* w = V + static_cast<size_t>(j + 1) * ld;  // the candidate lands in its basis slot
            if (!have_spec) {
                PhaseTimer tm(c, &st->t_mv);
                matvec(V + static_cast<size_t>(j) * ld, kv);
                tm.stop();
                PhaseTimer tp(c, &st->t_prec);
                apply_prec(kv, w);
                tp.stop();
            }
            have_spec = false;
            const std::function<void()> next = [&] {
                if (j + 1 >= m || st->iters + 1 >= cfg.max_iters) return;
                counter_before_spec = *spec_counter;
                matvec(w, kv);
                apply_prec(kv, w + ld);
                have_spec = true;
            };
            {
                PhaseTimer to(c, &st->t_orth);
                orthogonalize_device(c, V, ld, nbasis, n, w, cfg.orth, W.coef.p, W.partial.p, W.cgs.p, h.data(),
                                     speculate ? &next : nullptr);
                to.stop();
            }
            for (int i = 0; i <= nbasis; ++i)
                if (!std::isfinite(h[i])) throw Failure(HDGB_ERR_NAN_DETECTED, "NaN detected in gmres Hessenberg column");
            const double hsub = h[j + 1];
            for (int i = 0; i < j; ++i) {
                const double t1 = cs[i] * h[i] + sn[i] * h[i + 1];
                const double t2 = -sn[i] * h[i] + cs[i] * h[i + 1];
                h[i] = t1;
                h[i + 1] = t2;
            }
            const double den = std::hypot(h[j], h[j + 1]);
            if (den == 0.0) break;
            cs[j] = h[j] / den;
            sn[j] = h[j + 1] / den;
            h[j] = den;
            h[j + 1] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            rcols.emplace_back(h.begin(), h.begin() + j + 2);

            ++st->iters;
            jused = j + 1;
            if (residual_trace && n_trace < cfg.max_iters) residual_trace[n_trace++] = std::abs(g[j + 1]);

            double hmax = 1.0;
            for (int i = 0; i <= j; ++i) hmax = std::max(hmax, std::abs(rcols[j][i]));
            const bool happy = hsub <= 1e-14 * hmax;
            if (!happy) ++nbasis;
            if (std::abs(g[j + 1]) <= target || happy) {
                cycle_converged = true;
                break;
            }
        }
        if (have_spec) *spec_counter = counter_before_spec;  // the cycle ended: the speculative candidate is dropped
        if (jused == 0)
            throw Failure(HDGB_ERR_NAN_DETECTED,
                          "NaN detected in gmres made no progress: the preconditioned operator annihilated the residual direction");

        if (cfg.track_diagnostics) {
            const int used = std::min(jused, nbasis);
            DevBuf<double> gram(used);
            std::vector<double> hg(used);
            for (int a = 0; a < used; ++a) {
                launch_multi_dot(c, V, ld, used, V + static_cast<size_t>(a) * ld, n, gram.p, W.partial.p);
                if (c->comm) c->comm->allreduce(c, gram.p, used);
                HDGB_CUDA(cudaMemcpyAsync(hg.data(), gram.p, used * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
                HDGB_CUDA(cudaStreamSynchronize(c->stream));
                for (int b = a; b < used; ++b)
                    st->max_orth_error = std::max(st->max_orth_error, std::abs(hg[b] - (a == b ? 1.0 : 0.0)));
            }
        }

        // back-substitution (gmres.cpp:188-193) and x += V y (:194-197)
        std::vector<double> y(jused);
        for (int i = jused - 1; i >= 0; --i) {
            double v = g[i];
            for (int cc = i + 1; cc < jused; ++cc) v -= rcols[cc][i] * y[cc];
            y[i] = v / rcols[i][i];
        }
        HDGB_CUDA(cudaMemcpyAsync(W.ycoef.p, y.data(), jused * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        launch_multi_axpy(c, V, ld, jused, W.ycoef.p, 1.0, x, n, nullptr, W.partial.p);
        HDGB_CUDA(cudaStreamSynchronize(c->stream));  // y is a stack temporary

        if (cfg.track_diagnostics) {
            residual(r);
            const double tracked = std::abs(g[jused]);
            const double explicit_norm = norm_of(r);
            const double gap = std::abs(tracked - explicit_norm) / std::max(explicit_norm, 1e-300);
            st->max_residual_gap = std::max(st->max_residual_gap, gap);
        }
        if (cycle_converged) {
            residual(r);
            const double rn = norm_of(r);
            if (rn <= target) {
                st->converged = 1;
                st->final_rel_residual = rn / beta0;
                return;
            }
            first_cycle = true;
            ++st->restarts;
            continue;
        }
        if (st->iters >= cfg.max_iters) break;
        ++st->restarts;
    }
    residual(r);
    st->final_rel_residual = norm_of(r) / beta0;
    st->converged = st->final_rel_residual <= cfg.tol ? 1 : 0;
}

}  // namespace hdgb

extern "C" {

void hdgb_gmres_config_default(hdgb_gmres_config* cfg) {
    cfg->restart = 50;
    cfg->tol = 1e-6;
    cfg->max_iters = 1000;
    cfg->orth = 0;
    cfg->track_diagnostics = 0;
}

void hdgb_newton_config_default(hdgb_newton_config* cfg) {
    cfg->tol = 1e-8;
    cfg->max_newton = 50;
    cfg->min_alpha = 1.0 / 1024.0;
}

hdgb_status hdgb_gmres_solve(hdgb_matrix* k, hdgb_precond* p, const double* rhs, const double* x0,
                             const hdgb_gmres_config* cfg, double* x, hdgb_gmres_stats* stats, double* residual_trace) {
    hdgb_ctx* c = k->ctx;
    return guarded(c, [&] {
        hdgb_gmres_config cf;
        hdgb_gmres_config_default(&cf);
        if (cfg) cf = *cfg;
        if (p && static_cast<int64_t>(p->mpf) * p->nf != k->n_dof())
            throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: preconditioner / operator size");
        const size_t n = k->n_local();
        InArg B(c, rhs, n);
        OutArg X(c, x, n);
        if (x0 && x0 != x) HDGB_CUDA(cudaMemcpyAsync(X.dev, x0, n * sizeof(double), cudaMemcpyDefault, c->stream));
        else if (!x0) HDGB_CUDA(cudaMemsetAsync(X.dev, 0, n * sizeof(double), c->stream));
        else if (X.host) HDGB_CUDA(cudaMemcpyAsync(X.dev, x0, n * sizeof(double), cudaMemcpyDefault, c->stream));
        hdgb_gmres_stats local;
        gmres_device(k, p, B.dev, X.dev, cf, stats ? stats : &local, residual_trace);
        X.commit();
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

hdgb_status hdgb_gmres_solve_fn(hdgb_ctx* c, int64_t n, hdgb_op_fn matvec, void* mv_user, hdgb_op_fn precond, void* pc_user,
                                const double* rhs, const double* x0, const hdgb_gmres_config* cfg, double* x,
                                hdgb_gmres_stats* stats, double* residual_trace) {
    return guarded(c, [&] {
        hdgb_gmres_config cf;
        hdgb_gmres_config_default(&cf);
        if (cfg) cf = *cfg;
        if (!matvec) throw Failure(HDGB_ERR_GENERIC, "gmres_solve: operator callback missing");
        if (n < 0 || cf.restart < 1) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: GMRES size / restart length");
        const size_t sz = static_cast<size_t>(n);
        InArg B(c, rhs, sz);
        OutArg X(c, x, sz);
        if (x0 && x0 != x) HDGB_CUDA(cudaMemcpyAsync(X.dev, x0, sz * sizeof(double), cudaMemcpyDefault, c->stream));
        else if (!x0) HDGB_CUDA(cudaMemsetAsync(X.dev, 0, sz * sizeof(double), c->stream));
        else if (X.host) HDGB_CUDA(cudaMemcpyAsync(X.dev, x0, sz * sizeof(double), cudaMemcpyDefault, c->stream));
        auto wrap = [n](hdgb_op_fn fn, void* user, const char* what) -> DevOp {
            if (!fn) return DevOp();
            return [fn, user, n, what](const double* in, double* out) {
                if (fn(user, in, out, n) != 0) throw Failure(HDGB_ERR_GENERIC, std::string("gmres_solve: ") + what + " callback failed");
            };
        };
        // the restart length never needs to exceed the iteration cap (basis storage)
        hdgb_gmres_config run = cf;
        std::unique_ptr<GmresWork> W = make_gmres_work(c, n, n, std::max(1, std::min(cf.restart, cf.max_iters)));
        run.restart = W->restart;
        hdgb_gmres_stats local;
        // callbacks are invoked exactly as often as the reference invokes its closures: no speculation here
        gmres_core(c, n, n, *W, wrap(matvec, mv_user, "matvec"), wrap(precond, pc_user, "preconditioner"), B.dev, X.dev, run,
                   stats ? stats : &local, residual_trace, nullptr);
        X.commit();
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

hdgb_status hdgb_orthogonalize(hdgb_ctx* c, const double* basis, int nvec, int64_t n, double* w, int orth, double* h) {
    return guarded(c, [&] {
        if (2 * static_cast<size_t>(nvec) + 4 > c->pinned_doubles) throw Failure(HDGB_ERR_UNSUPPORTED, "too many basis vectors");
        DevBuf<double> coef(2 * static_cast<size_t>(nvec) + 4), partial(multi_dot_workspace_doubles(n, std::max(nvec, 1)));
        DevBuf<double> cgs(cgs_workspace_doubles(c));
        cgs.zero(c->stream);
        orthogonalize_device(c, basis, n, nvec, n, w, orth, coef.p, partial.p, cgs.p, h);
    });
}

hdgb_status hdgb_newton_solve(hdgb_disc* d, const hdgb_model* m, hdgb_state* s, const hdgb_newton_config* ncfg_in,
                              const hdgb_gmres_config* gcfg_in, const hdgb_precond_spec* pspec_in,
                              const hdgb_time* t, hdgb_solve_report* rep) {
    hdgb_ctx* c = d->ctx;
    hdgb_solve_report local;
    if (!rep) rep = &local;
    std::memset(rep, 0, sizeof(*rep));
    return guarded(c, [&] {
        using Clock = std::chrono::steady_clock;
        const auto since = [](Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); };
        const auto t_start = Clock::now();
        hdgb_newton_config ncfg;
        hdgb_newton_config_default(&ncfg);
        if (ncfg_in) ncfg = *ncfg_in;
        hdgb_gmres_config gcfg;
        hdgb_gmres_config_default(&gcfg);
        if (gcfg_in) gcfg = *gcfg_in;
        hdgb_precond_spec pspec;
        hdgb_precond_spec_default(&pspec);
        if (pspec_in) pspec = *pspec_in;

        const DiscView& v = d->view;
        const size_t n_int = static_cast<size_t>(v.npe) * v.ne, n_tr = static_cast<size_t>(v.mpf) * v.nf;
        const bool transient = t && t->dt > 0.0;
        if (transient && !t->u_prev)
            throw Failure(HDGB_ERR_INCONSISTENT_DIMENSIONS, "inconsistent dimensions: transient assembly requires the previous solution");
        InArg uprev(c, transient ? t->u_prev : nullptr, n_int);
        const double dt = transient ? t->dt : 0.0;

        DevBuf<double> res_tr(n_tr), res_in(n_int), duhat(n_tr), du(n_int), tmp(n_int), u0(n_int), uh0(n_tr);
        double rnorm = assemble_residual_device(d, m, s, uprev.dev, dt, res_tr.p, res_in.p);
        rep->residual_history[rep->n_history++] = rnorm;

        for (int iter = 0;; ++iter) {
            if (rnorm <= ncfg.tol) { rep->converged = 1; break; }
            if (iter >= ncfg.max_newton) { rep->converged = 0; break; }

            auto t0 = Clock::now();
            std::unique_ptr<hdgb_ops> ops(assemble_element_operators_device(d, m, s, uprev.dev, dt, false));
            std::unique_ptr<hdgb_matrix> k(assemble_global_device(d, ops.get()));
            std::unique_ptr<hdgb_precond> prec(build_preconditioner_spec(k.get(), ops.get(), d, pspec));
            HDGB_CUDA(cudaStreamSynchronize(c->stream));
            rep->t_ass += since(t0);

            duhat.zero(c->stream);  // GMRES always starts from 0 (newton.cpp:88)
            hdgb_gmres_stats gs;
            std::memset(&gs, 0, sizeof(gs));
            if (!pspec.ritz_per_restart || pspec.poly_degree == 0) {
                gmres_device(k.get(), prec.get(), k->rhs.p, duhat.p, gcfg, &gs, nullptr);
                rep->n_inner_prec_ops += prec->inner_ops;
            } else {
                // one restart cycle at a time with fresh Ritz values in between (newton.cpp:92-115)
                hdgb_gmres_config one = gcfg;
                while (true) {
                    one.max_iters = std::min(gcfg.restart, gcfg.max_iters - gs.iters);
                    if (one.max_iters <= 0) break;
                    hdgb_gmres_stats sc;
                    gmres_device(k.get(), prec.get(), k->rhs.p, duhat.p, one, &sc, nullptr);
                    rep->n_inner_prec_ops += prec->inner_ops;
                    gs.iters += sc.iters;
                    gs.restarts += sc.restarts + 1;
                    gs.t_mv += sc.t_mv; gs.t_prec += sc.t_prec; gs.t_orth += sc.t_orth;
                    gs.final_rel_residual = sc.final_rel_residual;
                    if (sc.converged) { gs.converged = 1; break; }
                    auto tr = Clock::now();
                    prec.reset(build_preconditioner_spec(k.get(), ops.get(), d, pspec));
                    HDGB_CUDA(cudaStreamSynchronize(c->stream));
                    rep->t_ass += since(tr);
                }
            }
            rep->n_gmres_total += gs.iters;
            if (rep->n_newton < HDGB_MAX_NEWTON_HISTORY) rep->gmres_per_newton[rep->n_newton] = gs.iters;
            rep->t_mv += gs.t_mv; rep->t_prec += gs.t_prec; rep->t_orth += gs.t_orth;

            // ghost elements are recovered redundantly: they need the update on their (halo) faces
            if (c->comm) c->comm->halo(c, duhat.p, v.mpf);
            recover_local_device(d, ops.get(), duhat.p, du.p, tmp.p);

            // halving line search on the full nonlinear residual (newton.cpp:127-141); only u and
            // uhat move, q is re-derived by the residual assembly
            HDGB_CUDA(cudaMemcpyAsync(u0.p, s->u.p, n_int * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
            HDGB_CUDA(cudaMemcpyAsync(uh0.p, s->uhat.p, n_tr * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
            bool accepted = false;
            for (double alpha = 1.0; alpha >= ncfg.min_alpha; alpha *= 0.5) {
                launch_lincomb(c, 1.0, u0.p, alpha, du.p, s->u.p, static_cast<int64_t>(n_int));
                launch_lincomb(c, 1.0, uh0.p, alpha, duhat.p, s->uhat.p, static_cast<int64_t>(n_tr));
                double tnorm;
                try {
                    tnorm = assemble_residual_device(d, m, s, uprev.dev, dt, res_tr.p, res_in.p);
                } catch (...) {
                    HDGB_CUDA(cudaMemcpyAsync(s->u.p, u0.p, n_int * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
                    HDGB_CUDA(cudaMemcpyAsync(s->uhat.p, uh0.p, n_tr * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
                    throw;
                }
                if (tnorm < rnorm) {
                    rnorm = tnorm;
                    accepted = true;
                    if (rep->n_newton < HDGB_MAX_NEWTON_HISTORY) rep->alpha_history[rep->n_newton] = alpha;
                    break;
                }
            }
            ++rep->n_newton;
            if (!accepted) {
                HDGB_CUDA(cudaMemcpyAsync(s->u.p, u0.p, n_int * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
                HDGB_CUDA(cudaMemcpyAsync(s->uhat.p, uh0.p, n_tr * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
                compute_q_device(d, s);
                HDGB_CUDA(cudaStreamSynchronize(c->stream));
                rep->t_total = since(t_start);
                rep->final_residual = rnorm;
                char buf[128];
                std::snprintf(buf, sizeof(buf), "line search failed at Newton iteration %d (alpha reached %g)", iter, ncfg.min_alpha);
                throw Failure(HDGB_ERR_LINE_SEARCH_FAILED, buf, iter);
            }
            if (rep->n_history <= HDGB_MAX_NEWTON_HISTORY) rep->residual_history[rep->n_history++] = rnorm;
        }
        rep->final_residual = rnorm;
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        rep->t_total = since(t_start);
    });
}

hdgb_status hdgb_time_march(hdgb_disc* d, const hdgb_model* m, hdgb_state* s, double dt, int n_steps,
                            const hdgb_newton_config* ncfg, const hdgb_gmres_config* gcfg,
                            const hdgb_precond_spec* pspec, hdgb_solve_report* reports) {
    hdgb_ctx* c = d->ctx;
    // a failing step leaves defined (zeroed) reports behind it
    if (reports && n_steps > 0) std::memset(reports, 0, sizeof(hdgb_solve_report) * static_cast<size_t>(n_steps));
    return guarded(c, [&] {
        if (!(dt > 0.0)) throw Failure(HDGB_ERR_GENERIC, "time_march requires a positive dt");
        DevBuf<double> u_prev(s->u.n);
        for (int step = 0; step < n_steps; ++step) {
            HDGB_CUDA(cudaMemcpyAsync(u_prev.p, s->u.p, s->u.n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
            hdgb_time t{dt, u_prev.p};
            hdgb_solve_report local;
            const hdgb_status st = hdgb_newton_solve(d, m, s, ncfg, gcfg, pspec, &t, reports ? &reports[step] : &local);
            pool_set_current(c->stream);
            if (st != HDGB_OK) throw Failure(st, "time step " + std::to_string(step) + ": " + c->err, c->err_index);
        }
    });
}

}  // extern "C"
