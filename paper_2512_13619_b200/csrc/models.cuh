// PDE models as device functors.  The reference's PdeModel (models.hpp:27-50) is a bundle of host
// std::function callbacks invoked at every quadrature point (local_ops.cpp:96-108,158-179); device
// code cannot call those, so each built-in model (models.cpp) is restated as a functor that is
// instantiated into the assembly kernel.  x-only callbacks (forcing, Dirichlet data) arrive
// pre-tabulated at the quadrature points.
//
// Array conventions (M components, D space dimensions):
//   u[m], q[m*D+d] (q_d of component m), x[d], n[d]
//   F[m*D+d]                       flux of component m in direction d
//   dFu[(m*D+d)*M+mp]              dF[m][d] / du[mp]
//   dFq[((m*D+d)*M+mp)*D+dp]       dF[m][d] / dq[mp][dp]
//   S[m], dSu[m*M+mp], dSq[(m*M+mp)*D+dp]
//   boundary flux: val[m], d_u[m*M+mp], d_q[(m*M+mp)*D+dp], d_uh[m*M+mp]
#pragma once
#include "device_types.cuh"

namespace hdgb {

template <int M, int D>
struct BFlux {
    double val[M];
    double d_u[M * M];
    double d_q[M * M * D];
    double d_uh[M * M];
    __device__ void clear() {
        for (int i = 0; i < M; ++i) val[i] = 0.0;
        for (int i = 0; i < M * M; ++i) { d_u[i] = 0.0; d_uh[i] = 0.0; }
        for (int i = 0; i < M * M * D; ++i) d_q[i] = 0.0;
    }
};

// Common defaults: no source derivatives, zero flux-u derivative.
template <int M_, int D_>
struct ModelBase {
    static constexpr int M = M_, D = D_;
    __device__ void dflux_du(const double*, const double*, const double*, double* dFu) const {
        for (int i = 0; i < M * D * M; ++i) dFu[i] = 0.0;
    }
    __device__ void dsource_du(const double*, const double*, const double*, double* dSu) const {
        for (int i = 0; i < M * M; ++i) dSu[i] = 0.0;
    }
    __device__ void dsource_dq(const double*, const double*, const double*, double* dSq) const {
        for (int i = 0; i < M * M * D; ++i) dSq[i] = 0.0;
    }
    // Dirichlet trace condition uhat = g  (models.cpp:23-28)
    __device__ void dirichlet(const double* uhat, const double* g, BFlux<M, D>& b) const {
        b.clear();
        for (int m = 0; m < M; ++m) {
            b.val[m] = uhat[m] - (g ? g[m] : 0.0);
            b.d_uh[m * M + m] = 1.0;
        }
    }
};

// poisson_model (models.cpp:9-30): F = -q, S = forcing(x), tau constant, Dirichlet everywhere.
template <int D_>
struct PoissonModel : ModelBase<1, D_> {
    static constexpr int M = 1, D = D_;
    double tau;
    __device__ explicit PoissonModel(const ModelView& v) : tau(v.p[0]) {}
    __device__ void flux(const double*, const double* q, const double*, double* F) const {
        for (int d = 0; d < D; ++d) F[d] = -q[d];
    }
    __device__ void dflux_dq(const double*, const double*, const double*, double* dFq) const {
        for (int d = 0; d < D; ++d)
            for (int dp = 0; dp < D; ++dp) dFq[d * D + dp] = (d == dp) ? -1.0 : 0.0;
    }
    __device__ void source(const double*, const double*, const double*, const double* f, double* S) const {
        S[0] = f ? f[0] : 0.0;
    }
    __device__ double tau_fn(const double*, const double*, const double*) const { return tau; }
    __device__ void boundary(int, const double*, const double*, const double* uhat, const double*,
                             const double*, const double* g, BFlux<1, D>& b) const {
        this->dirichlet(uhat, g, b);
    }
};

// Poisson with a cubic reaction term: -div(grad u) + alpha u^3 = f  (damping / line-search tests).
template <int D_>
struct ReactionModel : PoissonModel<D_> {
    static constexpr int M = 1, D = D_;
    double alpha;
    __device__ explicit ReactionModel(const ModelView& v) : PoissonModel<D_>(v), alpha(v.p[1]) {}
    __device__ void source(const double* u, const double*, const double*, const double* f, double* S) const {
        S[0] = (f ? f[0] : 0.0) - alpha * u[0] * u[0] * u[0];
    }
    __device__ void dsource_du(const double* u, const double*, const double*, double* dSu) const {
        dSu[0] = -3.0 * alpha * u[0] * u[0];
    }
};

// burgers_model (models.cpp:32-61): F = (u^2/2 - nu q_x, u - nu q_y [, -nu q_z]); Dirichlet
// u = 1 - 2x on all boundaries except tag 3 (top), which is a zero-gradient outflow.
template <int D_>
struct BurgersModel : ModelBase<1, D_> {
    static constexpr int M = 1, D = D_;
    double nu, tau;
    __device__ explicit BurgersModel(const ModelView& v) : nu(v.p[0]), tau(v.p[1]) {}
    __device__ void flux(const double* u, const double* q, const double*, double* F) const {
        F[0] = 0.5 * u[0] * u[0] - nu * q[0];
        F[1] = u[0] - nu * q[1];
        if (D == 3) F[D - 1] = -nu * q[D - 1];
    }
    __device__ void dflux_du(const double* u, const double*, const double*, double* dFu) const {
        dFu[0] = u[0];
        dFu[1] = 1.0;
        if (D == 3) dFu[D - 1] = 0.0;
    }
    __device__ void dflux_dq(const double*, const double*, const double*, double* dFq) const {
        for (int d = 0; d < D; ++d)
            for (int dp = 0; dp < D; ++dp) dFq[d * D + dp] = (d == dp) ? -nu : 0.0;
    }
    __device__ void source(const double*, const double*, const double*, const double*, double* S) const { S[0] = 0.0; }
    __device__ double tau_fn(const double*, const double*, const double*) const { return tau; }
    __device__ void boundary(int tag, const double* u, const double* q, const double* uhat, const double* n,
                             const double* x, const double*, BFlux<1, D>& b) const {
        b.clear();
        if (tag == 3) {
            double qn = 0.0;
            for (int d = 0; d < D; ++d) qn += q[d] * n[d];
            b.val[0] = qn + tau * (u[0] - uhat[0]);
            b.d_u[0] = tau;
            for (int d = 0; d < D; ++d) b.d_q[d] = n[d];
            b.d_uh[0] = -tau;
            return;
        }
        b.val[0] = uhat[0] - (1.0 - 2.0 * x[0]);
        b.d_uh[0] = 1.0;
    }
};

// convdiff_model (models.cpp:63-93): F = c u - kappa q; tau = override or kappa + |c.n|.
template <int D_>
struct ConvDiffModel : ModelBase<1, D_> {
    static constexpr int M = 1, D = D_;
    double c[3], kappa, tau_override;
    __device__ explicit ConvDiffModel(const ModelView& v)
        : c{v.p[0], v.p[1], v.p[2]}, kappa(v.p[3]), tau_override(v.p[4]) {}
    __device__ void flux(const double* u, const double* q, const double*, double* F) const {
        for (int d = 0; d < D; ++d) F[d] = c[d] * u[0] - kappa * q[d];
    }
    __device__ void dflux_du(const double*, const double*, const double*, double* dFu) const {
        for (int d = 0; d < D; ++d) dFu[d] = c[d];
    }
    __device__ void dflux_dq(const double*, const double*, const double*, double* dFq) const {
        for (int d = 0; d < D; ++d)
            for (int dp = 0; dp < D; ++dp) dFq[d * D + dp] = (d == dp) ? -kappa : 0.0;
    }
    __device__ void source(const double*, const double*, const double*, const double* f, double* S) const {
        S[0] = f ? f[0] : 0.0;
    }
    __device__ double tau_fn(const double*, const double*, const double* n) const {
        if (tau_override >= 0.0) return tau_override;
        double cn = 0.0;
        for (int d = 0; d < D; ++d) cn += c[d] * n[d];
        return kappa + fabs(cn);
    }
    __device__ void boundary(int, const double*, const double*, const double* uhat, const double*,
                             const double*, const double* g, BFlux<1, D>& b) const {
        this->dirichlet(uhat, g, b);
    }
};

// Linear elasticity, M = D displacement components, q = grad u:
//   F[m][d] = -(mu (q[m][d] + q[d][m]) + lambda delta_md tr q),  div F = f.
// Boundary: tags whose bit is set in dirichlet_mask are clamped to the tabulated data (all tags
// when the mask is 0); the remaining tags are traction-free (natural) boundaries.
template <int D_>
struct ElasticityModel : ModelBase<D_, D_> {
    static constexpr int M = D_, D = D_;
    double lambda, mu, tau;
    int dirichlet_mask;
    __device__ explicit ElasticityModel(const ModelView& v)
        : lambda(v.p[0]), mu(v.p[1]), tau(v.p[2]), dirichlet_mask(static_cast<int>(v.p[3])) {}
    __device__ void flux(const double*, const double* q, const double*, double* F) const {
        double tr = 0.0;
        for (int k = 0; k < D; ++k) tr += q[k * D + k];
        for (int m = 0; m < M; ++m)
            for (int d = 0; d < D; ++d)
                F[m * D + d] = -(mu * (q[m * D + d] + q[d * D + m]) + ((m == d) ? lambda * tr : 0.0));
    }
    __device__ void dflux_dq(const double*, const double*, const double*, double* dFq) const {
        for (int m = 0; m < M; ++m)
            for (int d = 0; d < D; ++d)
                for (int mp = 0; mp < M; ++mp)
                    for (int dp = 0; dp < D; ++dp) {
                        double v = 0.0;
                        if (m == mp && d == dp) v += mu;
                        if (m == dp && d == mp) v += mu;
                        if (m == d && mp == dp) v += lambda;
                        dFq[((m * D + d) * M + mp) * D + dp] = -v;
                    }
    }
    __device__ void source(const double*, const double*, const double*, const double* f, double* S) const {
        for (int m = 0; m < M; ++m) S[m] = f ? f[m] : 0.0;
    }
    __device__ double tau_fn(const double*, const double*, const double*) const { return tau; }
    __device__ void boundary(int tag, const double* u, const double* q, const double* uhat, const double* n,
                             const double* x, const double* g, BFlux<M, D>& b) const {
        const bool clamp = (dirichlet_mask == 0) || ((dirichlet_mask >> tag) & 1);
        if (clamp) {
            this->dirichlet(uhat, g, b);
            return;
        }
        // traction-free: the numerical flux F(q).n + tau (u - uhat) itself vanishes
        b.clear();
        double F[M * D], dFq[M * D * M * D];
        flux(uhat, q, x, F);
        dflux_dq(uhat, q, x, dFq);
        for (int m = 0; m < M; ++m) {
            double fn = 0.0;
            for (int d = 0; d < D; ++d) fn += F[m * D + d] * n[d];
            b.val[m] = fn + tau * (u[m] - uhat[m]);
            b.d_u[m * M + m] = tau;
            b.d_uh[m * M + m] = -tau;
            for (int mp = 0; mp < M; ++mp)
                for (int dp = 0; dp < D; ++dp) {
                    double s = 0.0;
                    for (int d = 0; d < D; ++d) s += dFq[((m * D + d) * M + mp) * D + dp] * n[d];
                    b.d_q[(m * M + mp) * D + dp] = s;
                }
        }
    }
};

// ---- compressible Navier-Stokes (section 5.5-5.7; not in the reference code) ------------
// Conservative variables u = (rho, rho v_1..rho v_D, rho E), M = D + 2, q = grad u; ideal gas,
// constant viscosity mu, Prandtl number Pr:
//   F = F_inv(u) - F_visc(u, q),  p = (gamma - 1)(rho E - rho |v|^2 / 2),
//   tau = mu (grad v + grad v^T - (2/3) div v I),  heat flux = (mu gamma / Pr) grad e.
// The Jacobians dF/du and dF/dq are exact forward-mode derivatives (dual numbers) of ONE templated
// flux routine -- no hand-derived 5 x 3 x 5 x 3 tables.
struct Dual {
    double v, d;
};
__host__ __device__ inline Dual operator+(Dual a, Dual b) { return {a.v + b.v, a.d + b.d}; }
__host__ __device__ inline Dual operator-(Dual a, Dual b) { return {a.v - b.v, a.d - b.d}; }
__host__ __device__ inline Dual operator*(Dual a, Dual b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
__host__ __device__ inline Dual operator/(Dual a, Dual b) {
    const double iv = 1.0 / b.v;
    return {a.v * iv, (a.d - a.v * iv * b.d) * iv};
}
__host__ __device__ inline Dual operator*(double a, Dual b) { return {a * b.v, a * b.d}; }
__host__ __device__ inline Dual operator-(Dual a) { return {-a.v, -a.d}; }
__host__ __device__ inline double make_scalar(double, double v) { return v; }
__host__ __device__ inline Dual make_scalar(Dual, double v) { return {v, 0.0}; }

template <int D, class T>
__host__ __device__ void ns_flux(const T* u, const T* q, T* F, double gamma, double mu, double pr) {
    constexpr int M = D + 2;
    const T one = make_scalar(T{}, 1.0);
    const T rinv = one / u[0];
    T v[D];
    T ke = make_scalar(T{}, 0.0);
    for (int i = 0; i < D; ++i) {
        v[i] = u[1 + i] * rinv;
        ke = ke + 0.5 * (v[i] * v[i]);
    }
    const T E = u[M - 1] * rinv;
    const T p = (gamma - 1.0) * (u[M - 1] - u[0] * ke);
    T dv[D][D];
    T div = make_scalar(T{}, 0.0);
    for (int i = 0; i < D; ++i)
        for (int d = 0; d < D; ++d) dv[i][d] = (q[(1 + i) * D + d] - v[i] * q[d]) * rinv;
    for (int i = 0; i < D; ++i) div = div + dv[i][i];
    for (int d = 0; d < D; ++d) {
        T de = (q[(M - 1) * D + d] - E * q[d]) * rinv;
        for (int i = 0; i < D; ++i) de = de - v[i] * dv[i][d];
        F[d] = u[1 + d];
        T work = make_scalar(T{}, 0.0);
        for (int i = 0; i < D; ++i) {
            T tau = mu * (dv[i][d] + dv[d][i]);
            if (i == d) tau = tau - (2.0 / 3.0 * mu) * div;
            T f = u[1 + i] * v[d] - tau;
            if (i == d) f = f + p;
            F[(1 + i) * D + d] = f;
            work = work + v[i] * tau;
        }
        F[(M - 1) * D + d] = (u[M - 1] + p) * v[d] - work - (mu * gamma / pr) * de;
    }
}

template <int D_>
struct NavierStokesModel : ModelBase<D_ + 2, D_> {
    static constexpr int M = D_ + 2, D = D_;
    double gamma, mu, pr, tau;
    __device__ explicit NavierStokesModel(const ModelView& v) : gamma(v.p[0]), mu(v.p[1]), pr(v.p[2]), tau(v.p[3]) {}
    __device__ void flux(const double* u, const double* q, const double*, double* F) const {
        ns_flux<D, double>(u, q, F, gamma, mu, pr);
    }
    __device__ void dflux_du(const double* u, const double* q, const double*, double* dFu) const {
        Dual ud[M], qd[M * D], Fd[M * D];
        for (int i = 0; i < M; ++i) ud[i] = {u[i], 0.0};
        for (int i = 0; i < M * D; ++i) qd[i] = {q[i], 0.0};
        for (int mp = 0; mp < M; ++mp) {
            ud[mp].d = 1.0;
            ns_flux<D, Dual>(ud, qd, Fd, gamma, mu, pr);
            ud[mp].d = 0.0;
            for (int k = 0; k < M * D; ++k) dFu[k * M + mp] = Fd[k].d;
        }
    }
    __device__ void dflux_dq(const double* u, const double* q, const double*, double* dFq) const {
        Dual ud[M], qd[M * D], Fd[M * D];
        for (int i = 0; i < M; ++i) ud[i] = {u[i], 0.0};
        for (int i = 0; i < M * D; ++i) qd[i] = {q[i], 0.0};
        for (int s = 0; s < M * D; ++s) {  // s = mp*D + dp
            qd[s].d = 1.0;
            ns_flux<D, Dual>(ud, qd, Fd, gamma, mu, pr);
            qd[s].d = 0.0;
            for (int k = 0; k < M * D; ++k) dFq[k * M * D + s] = Fd[k].d;
        }
    }
    __device__ void source(const double*, const double*, const double*, const double* f, double* S) const {
        for (int m = 0; m < M; ++m) S[m] = f ? f[m] : 0.0;
    }
    __device__ double tau_fn(const double*, const double*, const double*) const { return tau; }
    // every boundary face pins the trace to the tabulated state (far field / manufactured data)
    __device__ void boundary(int, const double*, const double*, const double* uhat, const double*, const double*,
                             const double* g, BFlux<M, D>& b) const {
        this->dirichlet(uhat, g, b);
    }
};

}  // namespace hdgb
