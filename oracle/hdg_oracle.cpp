// TEST INFRASTRUCTURE ONLY -- the product (paper_2512_13619_b200/) never links or calls this.
//
// Generalised CPU restatement ("tier B" oracle) of the reference's HDG hot path for D = 2|3 space
// dimensions, M >= 1 components and any element shape whose tables are supplied by the caller:
//   local factors        /root/reference/proj/src/local_ops.cpp:252-349
//   compute_q            local_ops.cpp:367-374
//   assemble_core        local_ops.cpp:33-228      (volume + face quadrature, residual + Jacobian)
//   static condensation  local_ops.cpp:376-430
//   assemble_global      face_matrix.cpp:11-61     (n_lfe generalised from the hard-coded 4)
//   block_matvec         face_matrix.cpp:83-107
//   build/apply BJ, ASM  preconditioner.cpp:30-105
//   compute_harmonic_ritz / leja_order   preconditioner.cpp:119-244 (the small dense solve and the
//                        eigenvalues go through oracle/eigen_shim, the same stand-in the compiled
//                        reference uses here: Eigen 3 is absent from this image)
//   apply_poly           preconditioner.cpp:246-283
//   Chebyshev nodes      NOT in the reference: the spec is DESIGN.md section 6 --
//                        roots of T_P on [lo, hi] = range of the real parts of the harmonic Ritz values
//                        (lo <= 0 -> hi / 30), Leja-ordered, applied by apply_poly's recurrence
//   orthogonalize/GMRES  gmres.cpp:28-228
//   newton_solve         newton.cpp:54-154
//   lu_invert / gemm / gemv  dense_batch.cpp:19-160
// The reference itself is 2D / scalar / quadrilateral only; for that case this file performs the
// SAME floating-point operations in the SAME order, and tests/test_oracle.py pins it bit for bit
// against the unmodified reference (oracle/_ref) on its own cases.  For 3D / M > 1 the parity
// status is "pinned by construction + tier-A equality on the shared 2D subset"; there is no
// reference implementation of those configurations.
//
// Built with the reference's Release flags (-O2, no -march => no FMA contraction on x86-64).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include <Eigen/Dense>  // oracle/eigen_shim (stand-in, see its header)

namespace {

constexpr int MAXM = 5, MAXD = 3;
using Vec = std::vector<double>;

int g_threads = 1;

void parallel_for(size_t n, const std::function<void(size_t, size_t)>& fn) {
    const size_t nt = std::min<size_t>(std::max(1, g_threads), n ? n : 1);
    if (nt <= 1) { fn(0, n); return; }
    std::vector<std::thread> pool;
    const size_t chunk = (n + nt - 1) / nt;
    for (size_t t = 0; t < nt; ++t) {
        const size_t b = t * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& th : pool) th.join();
}

// ---- dense kernels (dense_batch.cpp) -------------------------------------------------------------
// Explicit inverse of one column-major n x n block; false when a pivot is not above tol.
bool invert_one(const double* a, double* inv, double* lu, int* piv, int n) {
    const size_t nn = static_cast<size_t>(n) * n;
    double amax = 0.0;
    for (size_t i = 0; i < nn; ++i) amax = std::max(amax, std::abs(a[i]));
    const double tol = 1e-14 * amax;
    std::memcpy(lu, a, nn * sizeof(double));
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::abs(lu[k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const double v = std::abs(lu[k * n + i]);
            if (v > best) { best = v; p = i; }
        }
        if (!(best > tol)) return false;
        piv[k] = p;
        if (p != k)
            for (int c = 0; c < n; ++c) std::swap(lu[c * n + k], lu[c * n + p]);
        const double d = 1.0 / lu[k * n + k];
        for (int i = k + 1; i < n; ++i) lu[k * n + i] *= d;
        for (int c = k + 1; c < n; ++c) {
            const double m = lu[c * n + k];
            if (m != 0.0)
                for (int i = k + 1; i < n; ++i) lu[c * n + i] -= lu[k * n + i] * m;
        }
    }
    for (int col = 0; col < n; ++col) {
        double* x = inv + static_cast<size_t>(col) * n;
        std::fill(x, x + n, 0.0);
        x[col] = 1.0;
        for (int k = 0; k < n; ++k)
            if (piv[k] != k) std::swap(x[k], x[piv[k]]);
        for (int k = 0; k < n; ++k) {
            const double xk = x[k];
            if (xk != 0.0)
                for (int i = k + 1; i < n; ++i) x[i] -= lu[k * n + i] * xk;
        }
        for (int k = n - 1; k >= 0; --k) {
            double xk = x[k];
            for (int i = k + 1; i < n; ++i) xk -= lu[i * n + k] * x[i];
            x[k] = xk / lu[k * n + k];
        }
    }
    return true;
}

// returns -1 or the lowest-seen singular batch index
long invert_batch(int n, size_t batch, const double* a, double* out) {
    std::atomic<long> bad{-1};
    parallel_for(batch, [&](size_t b0, size_t b1) {
        Vec lu(static_cast<size_t>(n) * n);
        std::vector<int> piv(n);
        for (size_t b = b0; b < b1; ++b)
            if (!invert_one(a + b * n * n, out + b * n * n, lu.data(), piv.data(), n)) {
                long expected = -1;
                bad.compare_exchange_strong(expected, static_cast<long>(b));
                return;
            }
    });
    return bad.load();
}

// C = A (m x k, lda = m) * B (k x n, ldb given), column-major, ascending-p accumulation.
void gemm_one(int m, int n, int k, const double* A, const double* B, int ldb, double* Cc, int ldc) {
    for (int j = 0; j < n; ++j) {
        const double* bj = B + static_cast<size_t>(j) * ldb;
        for (int i = 0; i < m; ++i) {
            double acc = 0.0;
            for (int p = 0; p < k; ++p) acc += A[static_cast<size_t>(p) * m + i] * bj[p];
            Cc[static_cast<size_t>(j) * ldc + i] = acc;
        }
    }
}

void gemv_one(int m, int k, const double* A, const double* x, double* y, bool accumulate) {
    for (int i = 0; i < m; ++i) {
        double acc = 0.0;
        for (int p = 0; p < k; ++p) acc += A[static_cast<size_t>(p) * m + i] * x[p];
        y[i] = accumulate ? y[i] + acc : acc;
    }
}

double dot(const Vec& a, const Vec& b) {
    double acc = 0.0;
    for (size_t i = 0; i < a.size(); ++i) acc += a[i] * b[i];
    return acc;
}
double norm2(const Vec& a) { return std::sqrt(dot(a, a)); }

// ---- compressible Navier-Stokes flux (PAPER.md 5.5-5.7; no reference implementation) --------------
// u = (rho, rho v, rho E), q = grad u.  Written for a generic scalar so that the same routine run on
// first-order dual numbers yields the exact Jacobians.
struct Dn {
    double v, d;
};
inline Dn operator+(Dn a, Dn b) { return {a.v + b.v, a.d + b.d}; }
inline Dn operator-(Dn a, Dn b) { return {a.v - b.v, a.d - b.d}; }
inline Dn operator*(Dn a, Dn b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
inline Dn operator/(Dn a, Dn b) { const double iv = 1.0 / b.v; return {a.v * iv, (a.d - a.v * iv * b.d) * iv}; }
inline Dn operator*(double a, Dn b) { return {a * b.v, a * b.d}; }
inline double lift(double, double v) { return v; }
inline Dn lift(Dn, double v) { return {v, 0.0}; }

template <class T>
void navier_stokes_flux(int D, const T* u, const T* q, T* F, double gamma, double mu, double pr) {
    const int M = D + 2;
    const T rinv = lift(T{}, 1.0) / u[0];
    T vel[MAXD], gradv[MAXD][MAXD];
    T kinetic = lift(T{}, 0.0);
    for (int i = 0; i < D; ++i) {
        vel[i] = u[1 + i] * rinv;
        kinetic = kinetic + 0.5 * (vel[i] * vel[i]);
    }
    const T etot = u[M - 1] * rinv;
    const T pres = (gamma - 1.0) * (u[M - 1] - u[0] * kinetic);
    T divv = lift(T{}, 0.0);
    for (int i = 0; i < D; ++i)
        for (int d = 0; d < D; ++d) gradv[i][d] = (q[(1 + i) * D + d] - vel[i] * q[d]) * rinv;
    for (int i = 0; i < D; ++i) divv = divv + gradv[i][i];
    for (int d = 0; d < D; ++d) {
        T grad_e = (q[(M - 1) * D + d] - etot * q[d]) * rinv;
        for (int i = 0; i < D; ++i) grad_e = grad_e - vel[i] * gradv[i][d];
        F[d] = u[1 + d];
        T work = lift(T{}, 0.0);
        for (int i = 0; i < D; ++i) {
            T stress = mu * (gradv[i][d] + gradv[d][i]);
            if (i == d) stress = stress - (2.0 / 3.0 * mu) * divv;
            T mom = u[1 + i] * vel[d] - stress;
            if (i == d) mom = mom + pres;
            F[(1 + i) * D + d] = mom;
            work = work + vel[i] * stress;
        }
        F[(M - 1) * D + d] = (u[M - 1] + pres) * vel[d] - work - (mu * gamma / pr) * grad_e;
    }
}

// ---- PDE models (models.cpp, generalised) --------------------------------------------------------
struct BFlux {
    double val[MAXM], d_u[MAXM * MAXM], d_q[MAXM * MAXM * MAXD], d_uh[MAXM * MAXM];
};

struct Model {
    int kind = 0, M = 1, D = 2;
    double p[16] = {0};
    const double* forcing_q = nullptr;    // [(e*qe+g)*M + m]
    const double* dirichlet_q = nullptr;  // [(f*qf+g)*M + m]

    // F[m*D+d]
    void flux(const double* u, const double* q, double* F) const {
        switch (kind) {
            case 0: case 4: for (int d = 0; d < D; ++d) F[d] = -q[d]; break;
            case 1:
                F[0] = 0.5 * u[0] * u[0] - p[0] * q[0];
                F[1] = u[0] - p[0] * q[1];
                if (D == 3) F[2] = -p[0] * q[2];
                break;
            case 2: for (int d = 0; d < D; ++d) F[d] = p[d] * u[0] - p[3] * q[d]; break;
            case 3: {
                double tr = 0.0;
                for (int k = 0; k < D; ++k) tr += q[k * D + k];
                for (int m = 0; m < M; ++m)
                    for (int d = 0; d < D; ++d)
                        F[m * D + d] = -(p[1] * (q[m * D + d] + q[d * D + m]) + ((m == d) ? p[0] * tr : 0.0));
                break;
            }
            case 5: navier_stokes_flux<double>(D, u, q, F, p[0], p[1], p[2]); break;
        }
    }
    void ns_jacobians(const double* u, const double* q, double* dFu, double* dFq) const {
        Dn ud[MAXM], qd[MAXM * MAXD], Fd[MAXM * MAXD];
        for (int i = 0; i < M; ++i) ud[i] = {u[i], 0.0};
        for (int i = 0; i < M * D; ++i) qd[i] = {q[i], 0.0};
        if (dFu)
            for (int mp = 0; mp < M; ++mp) {
                ud[mp].d = 1.0;
                navier_stokes_flux<Dn>(D, ud, qd, Fd, p[0], p[1], p[2]);
                ud[mp].d = 0.0;
                for (int k = 0; k < M * D; ++k) dFu[k * M + mp] = Fd[k].d;
            }
        if (dFq)
            for (int s = 0; s < M * D; ++s) {
                qd[s].d = 1.0;
                navier_stokes_flux<Dn>(D, ud, qd, Fd, p[0], p[1], p[2]);
                qd[s].d = 0.0;
                for (int k = 0; k < M * D; ++k) dFq[k * M * D + s] = Fd[k].d;
            }
    }
    // dFu[(m*D+d)*M+mp]
    void dflux_du(const double* u, const double* q, double* dFu) const {
        if (kind == 5) { ns_jacobians(u, q, dFu, nullptr); return; }
        for (int i = 0; i < M * D * M; ++i) dFu[i] = 0.0;
        if (kind == 1) { dFu[0] = u[0]; dFu[1] = 1.0; }
        if (kind == 2) for (int d = 0; d < D; ++d) dFu[d] = p[d];
    }
    // dFq[((m*D+d)*M+mp)*D+dp]
    void dflux_dq(const double* u, const double* q, double* dFq) const {
        if (kind == 5) { ns_jacobians(u, q, nullptr, dFq); return; }
        for (int i = 0; i < M * D * M * D; ++i) dFq[i] = 0.0;
        if (kind == 3) {
            for (int m = 0; m < M; ++m)
                for (int d = 0; d < D; ++d)
                    for (int mp = 0; mp < M; ++mp)
                        for (int dp = 0; dp < D; ++dp) {
                            double v = 0.0;
                            if (m == mp && d == dp) v += p[1];
                            if (m == dp && d == mp) v += p[1];
                            if (m == d && mp == dp) v += p[0];
                            dFq[((m * D + d) * M + mp) * D + dp] = -v;
                        }
            return;
        }
        const double c = (kind == 1) ? p[0] : (kind == 2 ? p[3] : 1.0);
        for (int d = 0; d < D; ++d) dFq[d * D + d] = -c;
    }
    void source(const double* u, const double* f, double* S) const {
        for (int m = 0; m < M; ++m) S[m] = (kind == 1) ? 0.0 : (f ? f[m] : 0.0);
        if (kind == 4) S[0] = (f ? f[0] : 0.0) - p[1] * u[0] * u[0] * u[0];
    }
    void dsource_du(const double* u, double* dSu) const {
        for (int i = 0; i < M * M; ++i) dSu[i] = 0.0;
        if (kind == 4) dSu[0] = -3.0 * p[1] * u[0] * u[0];
    }
    double tau(const double* n) const {
        switch (kind) {
            case 0: case 4: return p[0];
            case 1: return p[1];
            case 2: {
                if (p[4] >= 0.0) return p[4];
                double cn = 0.0;
                for (int d = 0; d < D; ++d) cn += p[d] * n[d];
                return p[3] + std::abs(cn);
            }
            case 5: return p[3];
            default: return p[2];
        }
    }
    void boundary(int tag, const double* u, const double* q, const double* uh, const double* n, const double* x,
                  const double* g, BFlux& b) const {
        for (int i = 0; i < M; ++i) b.val[i] = 0.0;
        for (int i = 0; i < M * M; ++i) { b.d_u[i] = 0.0; b.d_uh[i] = 0.0; }
        for (int i = 0; i < M * M * D; ++i) b.d_q[i] = 0.0;
        if (kind == 1) {
            const double t = p[1];
            if (tag == 3) {
                double qn = 0.0;
                for (int d = 0; d < D; ++d) qn += q[d] * n[d];
                b.val[0] = qn + t * (u[0] - uh[0]);
                b.d_u[0] = t;
                for (int d = 0; d < D; ++d) b.d_q[d] = n[d];
                b.d_uh[0] = -t;
                return;
            }
            b.val[0] = uh[0] - (1.0 - 2.0 * x[0]);
            b.d_uh[0] = 1.0;
            return;
        }
        if (kind == 3) {
            const int mask = static_cast<int>(p[3]);
            const bool clamp = (mask == 0) || ((mask >> tag) & 1);
            if (!clamp) {
                double F[MAXM * MAXD], dFq[MAXM * MAXD * MAXM * MAXD];
                flux(uh, q, F);
                dflux_dq(uh, q, dFq);
                for (int m = 0; m < M; ++m) {
                    double fn = 0.0;
                    for (int d = 0; d < D; ++d) fn += F[m * D + d] * n[d];
                    b.val[m] = fn + p[2] * (u[m] - uh[m]);
                    b.d_u[m * M + m] = p[2];
                    b.d_uh[m * M + m] = -p[2];
                    for (int mp = 0; mp < M; ++mp)
                        for (int dp = 0; dp < D; ++dp) {
                            double s = 0.0;
                            for (int d = 0; d < D; ++d) s += dFq[((m * D + d) * M + mp) * D + dp] * n[d];
                            b.d_q[(m * M + mp) * D + dp] = s;
                        }
                }
                return;
            }
        }
        for (int m = 0; m < M; ++m) {
            b.val[m] = uh[m] - (g ? g[m] : 0.0);
            b.d_uh[m * M + m] = 1.0;
        }
    }
};

struct Stats {
    int iters = 0, restarts = 0;
    double final_rel = 0.0, t_mv = 0.0, t_prec = 0.0, t_orth = 0.0;
    bool converged = false;
    int err = 0;  // 1 = NaN detected
};

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

struct Case {
    int D, M, ne, nf, n_lfe, n_orient, pe, pf, qe, qf;
    int npe, mpf, nfl, nfs, nb;
    std::vector<int> elem_faces, elem_side, face_elems, face_lidx, face_orient, bnd_tag;
    Vec phi, dphi[3], psi, tphi, wq, wf;
    Vec elem_detjac, elem_invjac, elem_coords, face_detjac, face_coords, face_normal;
    Vec forcing, dirichlet;
    Model model;
    // local factors
    Vec mass, mass_inv, bmat[3], cmat[3], minv_b[3], minv_c[3];
    // state
    Vec u, uhat, q[3], u_prev;
    double dt = 0.0;
    // raw + condensed operators
    Vec e_raw, f_raw, h_raw, j_raw, d_raw[3], g_raw[3], ru, ruhat_e;
    Vec kbar, ebar_inv, fbar, hbar, rbar;
    // global
    Vec blocks, rhs;
    std::vector<int64_t> neighbor;
    // preconditioner
    int pc_kind = 0;
    Vec bj_inv, asm_inv, ritz;  // ritz interleaved re/im
    long inner_ops = 0;
    // reports
    Vec residual_history, alpha_history;
    std::vector<int> gmres_per_newton;
    std::string err;
    long err_index = -1;

    const double* tphi_at(int lf, int o, int gc) const {
        return tphi.data() + ((static_cast<size_t>(lf) * n_orient + o) * qf + gc) * pe;
    }

    // ---- local factors (local_ops.cpp:252-349) ----
    int local_factors() {
        const size_t pp = static_cast<size_t>(pe) * pe, pc = static_cast<size_t>(pe) * nfs;
        mass.assign(pp * ne, 0.0);
        // mass = (phi_i phi_j table) x (w detJ), accumulated over ascending g like the GEMM
        parallel_for(ne, [&](size_t e0, size_t e1) {
            for (size_t e = e0; e < e1; ++e)
                for (int j = 0; j < pe; ++j)
                    for (int i = 0; i < pe; ++i) {
                        double acc = 0.0;
                        for (int g = 0; g < qe; ++g)
                            acc += (phi[i + pe * g] * phi[j + pe * g]) * (wq[g] * elem_detjac[e * qe + g]);
                        mass[e * pp + static_cast<size_t>(j) * pe + i] = acc;
                    }
        });
        for (int d = 0; d < D; ++d) { bmat[d].assign(pp * ne, 0.0); cmat[d].assign(pc * ne, 0.0); }
        parallel_for(ne, [&](size_t e0, size_t e1) {
            Vec grad(static_cast<size_t>(D) * pe);
            for (size_t e = e0; e < e1; ++e) {
                for (int g = 0; g < qe; ++g) {
                    const size_t gi = e * qe + g;
                    const double w = wq[g] * elem_detjac[gi];
                    const double* ij = &elem_invjac[gi * D * D];
                    for (int i = 0; i < pe; ++i)
                        for (int d = 0; d < D; ++d) {
                            double s = dphi[0][i + pe * g] * ij[d];
                            for (int r = 1; r < D; ++r) s += dphi[r][i + pe * g] * ij[r * D + d];
                            grad[static_cast<size_t>(d) * pe + i] = s;
                        }
                    for (int j = 0; j < pe; ++j) {
                        const double pj = w * phi[j + pe * g];
                        for (int i = 0; i < pe; ++i)
                            for (int d = 0; d < D; ++d)
                                bmat[d][e * pp + static_cast<size_t>(j) * pe + i] += pj * grad[static_cast<size_t>(d) * pe + i];
                    }
                }
                for (int lf = 0; lf < n_lfe; ++lf) {
                    const int f = elem_faces[e * n_lfe + lf];
                    const int side = elem_side[e * n_lfe + lf];
                    const int o = face_orient[2 * f + side];
                    for (int gc = 0; gc < qf; ++gc) {
                        const size_t fi = static_cast<size_t>(f) * qf + gc;
                        const double w = wf[gc] * face_detjac[fi];
                        const double* n = &face_normal[((static_cast<size_t>(f) * 2 + side) * qf + gc) * D];
                        const double* phis = tphi_at(lf, o, gc);
                        for (int b = 0; b < pf; ++b) {
                            const double pb = w * psi[b + pf * gc];
                            const int l = lf * pf + b;
                            for (int i = 0; i < pe; ++i)
                                for (int d = 0; d < D; ++d)
                                    cmat[d][e * pc + static_cast<size_t>(l) * pe + i] -= pb * phis[i] * n[d];
                        }
                    }
                }
            }
        });
        mass_inv.assign(pp * ne, 0.0);
        const long bad = invert_batch(pe, ne, mass.data(), mass_inv.data());
        if (bad >= 0) { err = "singular mass matrix"; err_index = bad; return 3; }
        for (int d = 0; d < D; ++d) {
            minv_b[d].assign(pp * ne, 0.0);
            minv_c[d].assign(pc * ne, 0.0);
            parallel_for(ne, [&](size_t e0, size_t e1) {
                for (size_t e = e0; e < e1; ++e) {
                    gemm_one(pe, pe, pe, &mass_inv[e * pp], &bmat[d][e * pp], pe, &minv_b[d][e * pp], pe);
                    gemm_one(pe, nfs, pe, &mass_inv[e * pp], &cmat[d][e * pc], pe, &minv_c[d][e * pc], pe);
                }
            });
        }
        return 0;
    }

    // element-major gather of the trace of component m: out[lf*pf + b]
    void gather_scalar_trace(size_t e, int m, const Vec& v, double* out) const {
        for (int lf = 0; lf < n_lfe; ++lf) {
            const int f = elem_faces[e * n_lfe + lf];
            for (int b = 0; b < pf; ++b) out[lf * pf + b] = v[static_cast<size_t>(f) * mpf + m * pf + b];
        }
    }

    // compute_q (local_ops.cpp:367-374)
    void compute_q() {
        const size_t pp = static_cast<size_t>(pe) * pe, pc = static_cast<size_t>(pe) * nfs;
        for (int d = 0; d < D; ++d) q[d].assign(static_cast<size_t>(npe) * ne, 0.0);
        parallel_for(ne, [&](size_t e0, size_t e1) {
            Vec ue(nfs);
            for (size_t e = e0; e < e1; ++e)
                for (int m = 0; m < M; ++m) {
                    gather_scalar_trace(e, m, uhat, ue.data());
                    for (int d = 0; d < D; ++d) {
                        double* y = &q[d][e * npe + static_cast<size_t>(m) * pe];
                        gemv_one(pe, pe, &minv_b[d][e * pp], &u[e * npe + static_cast<size_t>(m) * pe], y, false);
                        gemv_one(pe, nfs, &minv_c[d][e * pc], ue.data(), y, true);
                        for (int i = 0; i < pe; ++i) y[i] = -y[i];
                    }
                }
        });
    }

    // ---- assemble_core (local_ops.cpp:33-228) ----
    int assemble_core(bool want_jac) {
        for (double x : u) if (!std::isfinite(x)) { err = "non-finite state: interior solution"; return 5; }
        for (double x : uhat) if (!std::isfinite(x)) { err = "non-finite state: trace solution"; return 5; }
        const bool transient = dt > 0.0;
        if (transient && u_prev.size() != u.size()) { err = "transient assembly requires the previous solution"; return 9; }
        compute_q();
        const double dt_inv = transient ? 1.0 / dt : 0.0;
        const size_t sEE = static_cast<size_t>(npe) * npe, sEF = static_cast<size_t>(npe) * nfl, sFF = static_cast<size_t>(nfl) * nfl;
        ru.assign(static_cast<size_t>(npe) * ne, 0.0);
        ruhat_e.assign(static_cast<size_t>(nfl) * ne, 0.0);
        if (want_jac) {
            e_raw.assign(sEE * ne, 0.0); f_raw.assign(sEF * ne, 0.0); h_raw.assign(sEF * ne, 0.0); j_raw.assign(sFF * ne, 0.0);
            for (int d = 0; d < D; ++d) { d_raw[d].assign(sEE * ne, 0.0); g_raw[d].assign(sEF * ne, 0.0); }
        }
        const Model& mdl = model;
        parallel_for(ne, [&](size_t e0, size_t e1) {
            Vec grad(static_cast<size_t>(D) * pe);
            for (size_t e = e0; e < e1; ++e) {
                const double* ue = &u[e * npe];
                double* Ru = &ru[e * npe];
                double* Rh = &ruhat_e[e * nfl];
                double* E = want_jac ? &e_raw[e * sEE] : nullptr;
                double* F = want_jac ? &f_raw[e * sEF] : nullptr;
                double* H = want_jac ? &h_raw[e * sEF] : nullptr;
                double* J = want_jac ? &j_raw[e * sFF] : nullptr;
                double* Dm[3] = {nullptr, nullptr, nullptr};
                double* G[3] = {nullptr, nullptr, nullptr};
                if (want_jac) for (int d = 0; d < D; ++d) { Dm[d] = &d_raw[d][e * sEE]; G[d] = &g_raw[d][e * sEF]; }

                for (int g = 0; g < qe; ++g) {
                    const size_t gi = e * qe + g;
                    const double w = wq[g] * elem_detjac[gi];
                    const double* ij = &elem_invjac[gi * D * D];
                    const double* phig = &phi[static_cast<size_t>(pe) * g];
                    double ug[MAXM], qg[MAXM * MAXD], upg[MAXM];
                    for (int m = 0; m < M; ++m) {
                        double a = 0.0, ap = 0.0, aq[MAXD] = {0.0, 0.0, 0.0};
                        for (int i = 0; i < pe; ++i) {
                            a += ue[m * pe + i] * phig[i];
                            for (int d = 0; d < D; ++d) aq[d] += q[d][e * npe + m * pe + i] * phig[i];
                        }
                        if (transient) for (int i = 0; i < pe; ++i) ap += u_prev[e * npe + m * pe + i] * phig[i];
                        ug[m] = a; upg[m] = ap;
                        for (int d = 0; d < D; ++d) qg[m * D + d] = aq[d];
                    }
                    for (int i = 0; i < pe; ++i)
                        for (int d = 0; d < D; ++d) {
                            double s = dphi[0][i + pe * g] * ij[d];
                            for (int r = 1; r < D; ++r) s += dphi[r][i + pe * g] * ij[r * D + d];
                            grad[static_cast<size_t>(d) * pe + i] = s;
                        }
                    double Fl[MAXM * MAXD], S[MAXM];
                    mdl.flux(ug, qg, Fl);
                    mdl.source(ug, forcing.empty() ? nullptr : &forcing[gi * M], S);
                    for (int m = 0; m < M; ++m)
                        for (int i = 0; i < pe; ++i) {
                            double fg = Fl[m * D] * grad[i];
                            for (int d = 1; d < D; ++d) fg += Fl[m * D + d] * grad[static_cast<size_t>(d) * pe + i];
                            double v = -fg - S[m] * phig[i];
                            if (transient) v += dt_inv * (ug[m] - upg[m]) * phig[i];
                            Ru[m * pe + i] += w * v;
                        }
                    if (want_jac) {
                        double dFu[MAXM * MAXD * MAXM], dFq[MAXM * MAXD * MAXM * MAXD], dSu[MAXM * MAXM];
                        mdl.dflux_du(ug, qg, dFu);
                        mdl.dflux_dq(ug, qg, dFq);
                        mdl.dsource_du(ug, dSu);
                        for (int j = 0; j < pe; ++j) {
                            const double pj = w * phig[j];
                            for (int i = 0; i < pe; ++i)
                                for (int m = 0; m < M; ++m)
                                    for (int mp = 0; mp < M; ++mp) {
                                        const size_t o = static_cast<size_t>(mp * pe + j) * npe + (m * pe + i);
                                        double fe = dFu[(m * D) * M + mp] * grad[i];
                                        for (int d = 1; d < D; ++d) fe += dFu[(m * D + d) * M + mp] * grad[static_cast<size_t>(d) * pe + i];
                                        double eij = -fe - dSu[m * M + mp] * phig[i];
                                        if (transient && m == mp) eij += dt_inv * phig[i];
                                        E[o] += pj * eij;
                                        for (int dp = 0; dp < D; ++dp) {
                                            double fd = dFq[((m * D) * M + mp) * D + dp] * grad[i];
                                            for (int d = 1; d < D; ++d)
                                                fd += dFq[((m * D + d) * M + mp) * D + dp] * grad[static_cast<size_t>(d) * pe + i];
                                            Dm[dp][o] += pj * (-fd - 0.0 * phig[i]);
                                        }
                                    }
                        }
                    }
                }

                for (int lf = 0; lf < n_lfe; ++lf) {
                    const int f = elem_faces[e * n_lfe + lf];
                    const int side = elem_side[e * n_lfe + lf];
                    const int o = face_orient[2 * f + side];
                    const int tag = bnd_tag[f];
                    for (int gc = 0; gc < qf; ++gc) {
                        const size_t fi = static_cast<size_t>(f) * qf + gc;
                        const double w = wf[gc] * face_detjac[fi];
                        const double* x = &face_coords[fi * D];
                        const double* n = &face_normal[((static_cast<size_t>(f) * 2 + side) * qf + gc) * D];
                        const double* phis = tphi_at(lf, o, gc);
                        const double* psic = &psi[static_cast<size_t>(pf) * gc];
                        double ug[MAXM], qg[MAXM * MAXD], uh[MAXM];
                        for (int m = 0; m < M; ++m) {
                            double a = 0.0, aq[MAXD] = {0.0, 0.0, 0.0};
                            for (int i = 0; i < pe; ++i) {
                                a += ue[m * pe + i] * phis[i];
                                for (int d = 0; d < D; ++d) aq[d] += q[d][e * npe + m * pe + i] * phis[i];
                            }
                            ug[m] = a;
                            for (int d = 0; d < D; ++d) qg[m * D + d] = aq[d];
                            double h = 0.0;
                            for (int b = 0; b < pf; ++b) h += uhat[static_cast<size_t>(f) * mpf + m * pf + b] * psic[b];
                            uh[m] = h;
                        }
                        const double tau = mdl.tau(n);
                        double Fl[MAXM * MAXD], fhat[MAXM];
                        mdl.flux(uh, qg, Fl);
                        for (int m = 0; m < M; ++m) {
                            double fn = Fl[m * D] * n[0];
                            for (int d = 1; d < D; ++d) fn += Fl[m * D + d] * n[d];
                            fhat[m] = fn + tau * (ug[m] - uh[m]);
                            for (int i = 0; i < pe; ++i) Ru[m * pe + i] += w * fhat[m] * phis[i];
                        }
                        double dFu[MAXM * MAXD * MAXM], dFq[MAXM * MAXD * MAXM * MAXD];
                        if (want_jac || tag != 0) { mdl.dflux_du(uh, qg, dFu); mdl.dflux_dq(uh, qg, dFq); }
                        else {
                            for (int k = 0; k < M * D * M; ++k) dFu[k] = 0.0;
                            for (int k = 0; k < M * D * M * D; ++k) dFq[k] = 0.0;
                        }
                        double dfh_q[MAXM * MAXM * MAXD], dfh_uh[MAXM * MAXM];
                        for (int m = 0; m < M; ++m)
                            for (int mp = 0; mp < M; ++mp) {
                                double su = dFu[(m * D) * M + mp] * n[0];
                                for (int d = 1; d < D; ++d) su += dFu[(m * D + d) * M + mp] * n[d];
                                dfh_uh[m * M + mp] = su - ((m == mp) ? tau : 0.0);
                                for (int dp = 0; dp < D; ++dp) {
                                    double sq = dFq[((m * D) * M + mp) * D + dp] * n[0];
                                    for (int d = 1; d < D; ++d) sq += dFq[((m * D + d) * M + mp) * D + dp] * n[d];
                                    dfh_q[(m * M + mp) * D + dp] = sq;
                                }
                            }
                        double val[MAXM], dv_u[MAXM * MAXM], dv_q[MAXM * MAXM * MAXD], dv_uh[MAXM * MAXM];
                        if (tag == 0) {
                            for (int m = 0; m < M; ++m) val[m] = fhat[m];
                            for (int k = 0; k < M * M; ++k) { dv_u[k] = ((k / M) == (k % M)) ? tau : 0.0; dv_uh[k] = dfh_uh[k]; }
                            for (int k = 0; k < M * M * D; ++k) dv_q[k] = dfh_q[k];
                        } else {
                            BFlux b;
                            mdl.boundary(tag, ug, qg, uh, n, x, dirichlet.empty() ? nullptr : &dirichlet[fi * M], b);
                            for (int m = 0; m < M; ++m) val[m] = b.val[m];
                            for (int k = 0; k < M * M; ++k) { dv_u[k] = b.d_u[k]; dv_uh[k] = b.d_uh[k]; }
                            for (int k = 0; k < M * M * D; ++k) dv_q[k] = b.d_q[k];
                        }
                        for (int m = 0; m < M; ++m)
                            for (int b = 0; b < pf; ++b) Rh[lf * mpf + m * pf + b] += w * val[m] * psic[b];
                        if (!want_jac) continue;
                        for (int j = 0; j < pe; ++j) {
                            const double pj = w * phis[j];
                            for (int m = 0; m < M; ++m)
                                for (int mp = 0; mp < M; ++mp) {
                                    const size_t col = static_cast<size_t>(mp * pe + j);
                                    for (int i = 0; i < pe; ++i) {
                                        const size_t oE = col * npe + (m * pe + i);
                                        if (m == mp) E[oE] += pj * tau * phis[i];
                                        for (int dp = 0; dp < D; ++dp) Dm[dp][oE] += pj * dfh_q[(m * M + mp) * D + dp] * phis[i];
                                    }
                                    for (int b = 0; b < pf; ++b) {
                                        const size_t oH = col * nfl + (lf * mpf + m * pf + b);
                                        H[oH] += pj * dv_u[m * M + mp] * psic[b];
                                        for (int dp = 0; dp < D; ++dp) G[dp][oH] += pj * dv_q[(m * M + mp) * D + dp] * psic[b];
                                    }
                                }
                        }
                        for (int bp = 0; bp < pf; ++bp) {
                            const double pj = w * psic[bp];
                            for (int m = 0; m < M; ++m)
                                for (int mp = 0; mp < M; ++mp) {
                                    const size_t col = static_cast<size_t>(lf * mpf + mp * pf + bp);
                                    for (int i = 0; i < pe; ++i) F[col * npe + (m * pe + i)] += pj * dfh_uh[m * M + mp] * phis[i];
                                    for (int b = 0; b < pf; ++b) J[col * nfl + (lf * mpf + m * pf + b)] += pj * dv_uh[m * M + mp] * psic[b];
                                }
                        }
                    }
                }
            }
        });
        for (double& v : ru) v = -v;
        for (double& v : ruhat_e) v = -v;
        return 0;
    }

    // ---- static condensation (local_ops.cpp:376-430) ----
    int assemble_element_operators() {
        int rc = assemble_core(true);
        if (rc) return rc;
        const size_t sEE = static_cast<size_t>(npe) * npe, sEF = static_cast<size_t>(npe) * nfl, sFF = static_cast<size_t>(nfl) * nfl;
        const size_t pp = static_cast<size_t>(pe) * pe, pc = static_cast<size_t>(pe) * nfs;
        Vec ebar = e_raw;
        fbar = f_raw;
        hbar = h_raw;
        Vec jbar = j_raw;
        parallel_for(ne, [&](size_t e0, size_t e1) {
            Vec tE(sEE), tF(sEF), tH(sEF), tJ(sFF);
            for (size_t e = e0; e < e1; ++e)
                for (int d = 0; d < D; ++d) {
                    const double* Dd = &d_raw[d][e * sEE];
                    const double* Gd = &g_raw[d][e * sEF];
                    const double* mb = &minv_b[d][e * pp];
                    const double* mc = &minv_c[d][e * pc];
                    for (int mp = 0; mp < M; ++mp) {
                        const size_t cb = static_cast<size_t>(mp) * pe;
                        gemm_one(npe, pe, pe, Dd + cb * npe, mb, pe, tE.data() + cb * npe, npe);
                        gemm_one(nfl, pe, pe, Gd + cb * nfl, mb, pe, tH.data() + cb * nfl, nfl);
                        for (int lf = 0; lf < n_lfe; ++lf) {
                            const size_t tc = static_cast<size_t>(lf) * mpf + static_cast<size_t>(mp) * pf;
                            gemm_one(npe, pf, pe, Dd + cb * npe, mc + static_cast<size_t>(lf) * pf * pe, pe, tF.data() + tc * npe, npe);
                            gemm_one(nfl, pf, pe, Gd + cb * nfl, mc + static_cast<size_t>(lf) * pf * pe, pe, tJ.data() + tc * nfl, nfl);
                        }
                    }
                    for (size_t i = 0; i < sEE; ++i) ebar[e * sEE + i] -= tE[i];
                    for (size_t i = 0; i < sEF; ++i) fbar[e * sEF + i] -= tF[i];
                    for (size_t i = 0; i < sEF; ++i) hbar[e * sEF + i] -= tH[i];
                    for (size_t i = 0; i < sFF; ++i) jbar[e * sFF + i] -= tJ[i];
                }
        });
        ebar_inv.assign(sEE * ne, 0.0);
        const long bad = invert_batch(npe, ne, ebar.data(), ebar_inv.data());
        if (bad >= 0) { err = "singular local solve in element " + std::to_string(bad); err_index = bad; return 4; }
        kbar = std::move(jbar);
        rbar = ruhat_e;
        parallel_for(ne, [&](size_t e0, size_t e1) {
            Vec ef(sEF), hef(sFF), er(npe), her(nfl);
            for (size_t e = e0; e < e1; ++e) {
                gemm_one(npe, nfl, npe, &ebar_inv[e * sEE], &fbar[e * sEF], npe, ef.data(), npe);
                gemm_one(nfl, nfl, npe, &hbar[e * sEF], ef.data(), npe, hef.data(), nfl);
                for (size_t i = 0; i < sFF; ++i) kbar[e * sFF + i] -= hef[i];
                gemv_one(npe, npe, &ebar_inv[e * sEE], &ru[e * npe], er.data(), false);
                gemv_one(nfl, npe, &hbar[e * sEF], er.data(), her.data(), false);
                for (int i = 0; i < nfl; ++i) rbar[e * nfl + i] -= her[i];
            }
        });
        return 0;
    }

    // ---- assemble_global (face_matrix.cpp:11-61) ----
    void assemble_global() {
        const size_t bsz = static_cast<size_t>(mpf) * mpf, row = bsz * nb, sFF = static_cast<size_t>(nfl) * nfl;
        blocks.assign(row * nf, 0.0);
        neighbor.assign(static_cast<size_t>(nf) * nb, -1);
        rhs.assign(static_cast<size_t>(mpf) * nf, 0.0);
        parallel_for(nf, [&](size_t f0, size_t f1) {
            for (size_t f = f0; f < f1; ++f) {
                neighbor[f * nb] = static_cast<int64_t>(f);
                double* R = &blocks[f * row];
                for (int side = 0; side < 2; ++side) {
                    const int e = face_elems[2 * f + side];
                    if (e < 0) continue;
                    const int l = face_lidx[2 * f + side];
                    const double* Ke = &kbar[static_cast<size_t>(e) * sFF];
                    for (int c = 0; c < mpf; ++c)
                        for (int r = 0; r < mpf; ++r)
                            R[static_cast<size_t>(c) * mpf + r] += Ke[static_cast<size_t>(l * mpf + c) * nfl + (l * mpf + r)];
                    int idx = 0;
                    for (int lo = 0; lo < n_lfe; ++lo) {
                        if (lo == l) continue;
                        const int slot = (side == 0 ? 1 : n_lfe) + idx;
                        neighbor[f * nb + slot] = elem_faces[static_cast<size_t>(e) * n_lfe + lo];
                        for (int c = 0; c < mpf; ++c)
                            for (int r = 0; r < mpf; ++r)
                                R[slot * bsz + static_cast<size_t>(c) * mpf + r] = Ke[static_cast<size_t>(lo * mpf + c) * nfl + (l * mpf + r)];
                        ++idx;
                    }
                    for (int r = 0; r < mpf; ++r) rhs[f * mpf + r] += rbar[static_cast<size_t>(e) * nfl + l * mpf + r];
                }
            }
        });
    }

    // block_matvec (face_matrix.cpp:83-107): gather then one GEMV per face
    void matvec(const Vec& x, Vec& y) const {
        y.resize(x.size());
        const size_t row = static_cast<size_t>(mpf) * mpf * nb;
        parallel_for(nf, [&](size_t f0, size_t f1) {
            Vec xs(static_cast<size_t>(mpf) * nb);
            for (size_t f = f0; f < f1; ++f) {
                for (int s = 0; s < nb; ++s) {
                    const int64_t g = neighbor[f * nb + s];
                    for (int r = 0; r < mpf; ++r) xs[static_cast<size_t>(s) * mpf + r] = g < 0 ? 0.0 : x[static_cast<size_t>(g) * mpf + r];
                }
                gemv_one(mpf, mpf * nb, &blocks[f * row], xs.data(), &y[f * mpf], false);
            }
        });
    }

    // ---- preconditioners (preconditioner.cpp:30-105) ----
    int build_precond(int kind) {
        pc_kind = kind;
        ritz.clear();
        const size_t bsz = static_cast<size_t>(mpf) * mpf, row = bsz * nb, sFF = static_cast<size_t>(nfl) * nfl;
        if (kind == 1) {
            Vec diag(bsz * nf);
            for (size_t f = 0; f < static_cast<size_t>(nf); ++f) std::memcpy(&diag[f * bsz], &blocks[f * row], bsz * sizeof(double));
            bj_inv.assign(bsz * nf, 0.0);
            const long bad = invert_batch(mpf, nf, diag.data(), bj_inv.data());
            if (bad >= 0) { err = "build_bj (face block): singular block"; err_index = bad; return 2; }
        } else if (kind == 2 || kind == 3) {
            Vec pbar = kbar;
            for (size_t f = 0; f < static_cast<size_t>(nf); ++f) {
                const int e2 = face_elems[2 * f + 1];
                if (e2 < 0) continue;
                const int e1 = face_elems[2 * f], l1 = face_lidx[2 * f], l2 = face_lidx[2 * f + 1];
                for (int c = 0; c < mpf; ++c)
                    for (int r = 0; r < mpf; ++r) {
                        const size_t i1 = static_cast<size_t>(e1) * sFF + static_cast<size_t>(l1 * mpf + c) * nfl + (l1 * mpf + r);
                        const size_t i2 = static_cast<size_t>(e2) * sFF + static_cast<size_t>(l2 * mpf + c) * nfl + (l2 * mpf + r);
                        const double sum = kbar[i1] + kbar[i2];
                        pbar[i1] = sum;
                        pbar[i2] = sum;
                    }
            }
            asm_inv.assign(sFF * ne, 0.0);
            const long bad = invert_batch(nfl, ne, pbar.data(), asm_inv.data());
            if (bad >= 0) { err = "build_asm (element block): singular block"; err_index = bad; return 2; }
        }
        return 0;
    }

    void apply_base(const Vec& y, Vec& z) const {
        z.resize(y.size());
        if (pc_kind == 0) { z = y; return; }
        if (pc_kind == 1) {
            const size_t bsz = static_cast<size_t>(mpf) * mpf;
            parallel_for(nf, [&](size_t f0, size_t f1) {
                for (size_t f = f0; f < f1; ++f) gemv_one(mpf, mpf, &bj_inv[f * bsz], &y[f * mpf], &z[f * mpf], false);
            });
            return;
        }
        const size_t sFF = static_cast<size_t>(nfl) * nfl;
        Vec ze(static_cast<size_t>(nfl) * ne);
        parallel_for(ne, [&](size_t e0, size_t e1) {
            Vec ye(nfl);
            for (size_t e = e0; e < e1; ++e) {
                for (int lf = 0; lf < n_lfe; ++lf) {
                    const int f = elem_faces[e * n_lfe + lf];
                    for (int r = 0; r < mpf; ++r) ye[lf * mpf + r] = y[static_cast<size_t>(f) * mpf + r];
                }
                gemv_one(nfl, nfl, &asm_inv[e * sFF], ye.data(), &ze[e * nfl], false);
            }
        });
        const int sides = pc_kind == 3 ? 1 : 2;
        parallel_for(nf, [&](size_t f0, size_t f1) {
            for (size_t f = f0; f < f1; ++f) {
                for (int r = 0; r < mpf; ++r) z[f * mpf + r] = 0.0;
                for (int side = 0; side < sides; ++side) {
                    const int e = face_elems[2 * f + side];
                    if (e < 0) continue;
                    const int l = face_lidx[2 * f + side];
                    for (int r = 0; r < mpf; ++r) z[f * mpf + r] += ze[static_cast<size_t>(e) * nfl + l * mpf + r];
                }
            }
        });
    }

    // apply_poly (preconditioner.cpp:246-283)
    void apply_precond(const Vec& y, Vec& z) {
        if (ritz.empty()) { apply_base(y, z); return; }
        const size_t n = y.size();
        Vec qv(n), w(n, 0.0), t(n), s(n), kv(n);
        apply_base(y, qv);
        auto op = [&](const Vec& in, Vec& out) { matvec(in, kv); apply_base(kv, out); ++inner_ops; };
        size_t i = 0;
        const size_t cnt = ritz.size() / 2;
        while (i < cnt) {
            const double a = ritz[2 * i], b = ritz[2 * i + 1];
            if (b == 0.0) {
                const double inv = 1.0 / a;
                for (size_t j = 0; j < n; ++j) w[j] += inv * qv[j];
                op(qv, t);
                for (size_t j = 0; j < n; ++j) qv[j] -= inv * t[j];
                i += 1;
            } else {
                const double inv = 1.0 / (a * a + b * b);
                op(qv, t);
                for (size_t j = 0; j < n; ++j) s[j] = 2.0 * a * qv[j] - t[j];
                for (size_t j = 0; j < n; ++j) w[j] += inv * s[j];
                op(s, t);
                for (size_t j = 0; j < n; ++j) qv[j] -= inv * t[j];
                i += 2;
            }
        }
        z = std::move(w);
    }

    // leja_order (preconditioner.cpp:207-244)
    static std::vector<std::complex<double>> leja_order(const std::vector<std::complex<double>>& theta) {
        using C = std::complex<double>;
        std::vector<C> cands;
        for (const auto& t : theta)
            if (t.imag() >= 0.0) cands.push_back(t);
        std::vector<C> out;
        std::vector<bool> used(cands.size(), false);
        const auto better = [](const C& a, double ma, const C& b, double mb) {
            if (ma != mb) return ma > mb;
            if (a.real() != b.real()) return a.real() > b.real();
            return a.imag() > b.imag();
        };
        for (size_t step = 0; step < cands.size(); ++step) {
            int best = -1;
            double best_metric = 0.0;
            for (size_t c = 0; c < cands.size(); ++c) {
                if (used[c]) continue;
                double metric;
                if (out.empty()) {
                    metric = std::abs(cands[c]);
                } else {
                    metric = 0.0;
                    for (const auto& chosen : out) metric += std::log(std::abs(cands[c] - chosen));
                }
                if (best < 0 || better(cands[c], metric, cands[best], best_metric)) {
                    best = static_cast<int>(c);
                    best_metric = metric;
                }
            }
            used[best] = true;
            out.push_back(cands[best]);
            if (cands[best].imag() > 0.0) out.push_back(std::conj(cands[best]));
        }
        return out;
    }

    // compute_harmonic_ritz (preconditioner.cpp:119-205) on op = v -> base(K v)
    int harmonic_ritz(int degree, uint64_t seed, std::vector<std::complex<double>>& out) {
        const size_t n = static_cast<size_t>(mpf) * nf;
        if (degree < 1) { err = "dimension mismatch: polynomial degree must be >= 1"; return 8; }
        if (static_cast<size_t>(degree) > n) { err = "dimension mismatch: polynomial degree exceeds the operator dimension"; return 8; }
        std::mt19937_64 rng(seed);
        Vec v0(n);
        for (double& x : v0) x = 2.0 * (static_cast<double>(rng() >> 11) * 0x1p-53) - 1.0;
        const double nv = norm2(v0);
        for (double& x : v0) x /= nv;
        std::vector<Vec> basis;
        basis.push_back(std::move(v0));
        const int pmax = degree;
        Vec hess(static_cast<size_t>(pmax + 1) * pmax, 0.0);
        auto h = [&](int i, int j) -> double& { return hess[static_cast<size_t>(j) * (pmax + 1) + i]; };
        int p_eff = 0;
        double scale = 1.0;
        Vec w(n), kv(n);
        for (int j = 0; j < pmax; ++j) {
            matvec(basis[j], kv);
            apply_base(kv, w);
            if (j == 0) scale = std::max(1.0, norm2(w));
            for (int i = 0; i <= j; ++i) {
                const double hij = dot(basis[i], w);
                h(i, j) = hij;
                for (size_t t = 0; t < n; ++t) w[t] -= hij * basis[i][t];
            }
            const double hn = norm2(w);
            h(j + 1, j) = hn;
            p_eff = j + 1;
            if (!std::isfinite(hn)) { err = "NaN detected in harmonic Ritz Arnoldi"; return 6; }
            if (hn < 1e-14 * scale) break;
            if (j + 1 < pmax) {
                Vec vn(n);
                for (size_t t = 0; t < n; ++t) vn[t] = w[t] / hn;
                basis.push_back(std::move(vn));
            }
        }
        const int p = p_eff;
        Eigen::MatrixXd hs(p, p);
        for (int j = 0; j < p; ++j)
            for (int i = 0; i < p; ++i) hs(i, j) = h(i, j);
        const double hp1 = (p < pmax) ? 0.0 : h(p, p - 1);
        if (hp1 != 0.0) {
            Eigen::VectorXd ep = Eigen::VectorXd::Zero(p);
            ep(p - 1) = 1.0;
            Eigen::FullPivLU<Eigen::MatrixXd> lu(hs.transpose());
            if (lu.isInvertible()) hs.col(p - 1) += hp1 * hp1 * lu.solve(ep);
        }
        Eigen::EigenSolver<Eigen::MatrixXd> es(hs, false);
        std::vector<std::complex<double>> vals;
        double max_abs = 0.0;
        for (int i = 0; i < p; ++i) {
            std::complex<double> t(es.eigenvalues()(i).real(), es.eigenvalues()(i).imag());
            if (std::abs(t.imag()) < 1e-12 * std::abs(t)) t = {t.real(), 0.0};
            vals.push_back(t);
            max_abs = std::max(max_abs, std::abs(t));
        }
        std::vector<std::complex<double>> kept;
        for (const auto& t : vals) {
            if (std::abs(t) < 1e-12 * max_abs) continue;
            if (t.imag() < 0.0) continue;
            kept.push_back(t);
            if (t.imag() > 0.0) kept.emplace_back(t.real(), -t.imag());
        }
        out = leja_order(kept);
        return 0;
    }

    // Chebyshev variant (spec: DESIGN.md section 6; not in the reference): the P roots of T_P mapped to
    // [lo, hi] = range of Re(theta) over the harmonic Ritz estimates, with lo <= 0 replaced by hi / 30 and a
    // degenerate interval widened by 1e-8 relative; Leja-ordered; applied by apply_poly's recurrence.
    static std::vector<std::complex<double>> chebyshev_nodes(const std::vector<std::complex<double>>& th, int degree) {
        double lo = INFINITY, hi = -INFINITY;
        for (const auto& t : th) {
            lo = std::min(lo, t.real());
            hi = std::max(hi, t.real());
        }
        if (!(lo > 0.0)) lo = hi / 30.0;
        if (hi <= lo) hi = lo * (1.0 + 1e-8);
        const double kPi = 3.14159265358979323846;
        std::vector<std::complex<double>> nodes;
        for (int j = 0; j < degree; ++j) {
            const double x = std::cos(kPi * (2.0 * j + 1.0) / (2.0 * degree));
            nodes.emplace_back(0.5 * (hi + lo) + 0.5 * (hi - lo) * x, 0.0);
        }
        return leja_order(nodes);
    }

    // the polynomial part of build_preconditioner (newton.cpp:38-50); poly_kind 0 = GMRES polynomial, 1 = Chebyshev
    int build_poly(int degree, int poly_kind, uint64_t seed) {
        ritz.clear();
        if (degree <= 0) return 0;
        const size_t n = static_cast<size_t>(mpf) * nf;
        const int deg = static_cast<int>(std::min<size_t>(degree, n));
        std::vector<std::complex<double>> th;
        const int rc = harmonic_ritz(deg, seed, th);
        if (rc) return rc;
        if (poly_kind == 1 && !th.empty()) th = chebyshev_nodes(th, deg);
        for (const auto& t : th) { ritz.push_back(t.real()); ritz.push_back(t.imag()); }
        return 0;
    }

    // orthogonalize (gmres.cpp:28-59)
    static Vec orthogonalize(const std::vector<Vec>& basis, Vec& w, bool mgs) {
        const size_t j = basis.size();
        Vec h(j + 1, 0.0);
        if (mgs) {
            for (size_t i = 0; i < j; ++i) {
                const double hij = dot(basis[i], w);
                h[i] = hij;
                for (size_t t = 0; t < w.size(); ++t) w[t] -= hij * basis[i][t];
            }
        } else {
            Vec c(j);
            for (size_t i = 0; i < j; ++i) c[i] = dot(basis[i], w);
            for (size_t i = 0; i < j; ++i)
                for (size_t t = 0; t < w.size(); ++t) w[t] -= c[i] * basis[i][t];
            for (size_t i = 0; i < j; ++i) {
                const double d = dot(basis[i], w);
                c[i] += d;
                for (size_t t = 0; t < w.size(); ++t) w[t] -= d * basis[i][t];
            }
            for (size_t i = 0; i < j; ++i) h[i] = c[i];
        }
        const double hn = norm2(w);
        h[j] = hn;
        if (hn > 0.0) {
            const double inv = 1.0 / hn;
            for (double& t : w) t *= inv;
        }
        return h;
    }

    // gmres_solve (gmres.cpp:61-228)
    Stats gmres(const Vec& b, Vec& x, int restart, double tol, int max_iters, bool mgs) {
        Stats st;
        const size_t n = b.size();
        x.resize(n, 0.0);
        Vec kv(n), r(n), w(n);
        auto residual = [&](Vec& out) {
            auto t0 = Clock::now();
            matvec(x, kv);
            st.t_mv += since(t0);
            for (size_t i = 0; i < n; ++i) kv[i] = b[i] - kv[i];
            t0 = Clock::now();
            apply_precond(kv, out);
            st.t_prec += since(t0);
        };
        residual(r);
        const double beta0 = norm2(r);
        if (!std::isfinite(beta0)) { st.err = 1; return st; }
        if (beta0 == 0.0) { st.converged = true; return st; }
        const double target = tol * beta0;
        const int m = restart;
        std::vector<Vec> basis, rcols;
        Vec cs(m), sn(m), g(m + 1);
        bool first = true;
        while (true) {
            if (!first) residual(r);
            first = false;
            const double beta = norm2(r);
            if (beta <= target) { st.converged = true; break; }
            if (st.iters >= max_iters) break;
            basis.clear();
            rcols.clear();
            Vec v0(n);
            for (size_t i = 0; i < n; ++i) v0[i] = r[i] / beta;
            basis.push_back(std::move(v0));
            std::fill(g.begin(), g.end(), 0.0);
            g[0] = beta;
            int jused = 0;
            bool cyc = false;
            for (int j = 0; j < m && st.iters < max_iters; ++j) {
                auto t0 = Clock::now();
                matvec(basis[j], kv);
                st.t_mv += since(t0);
                t0 = Clock::now();
                apply_precond(kv, w);
                st.t_prec += since(t0);
                t0 = Clock::now();
                Vec h = orthogonalize(basis, w, mgs);
                st.t_orth += since(t0);
                for (double v : h) if (!std::isfinite(v)) { st.err = 1; return st; }
                const double hsub = h[j + 1];
                for (int i = 0; i < j; ++i) {
                    const double t1 = cs[i] * h[i] + sn[i] * h[i + 1];
                    const double t2 = -sn[i] * h[i] + cs[i] * h[i + 1];
                    h[i] = t1; h[i + 1] = t2;
                }
                const double den = std::hypot(h[j], h[j + 1]);
                if (den == 0.0) break;
                cs[j] = h[j] / den;
                sn[j] = h[j + 1] / den;
                h[j] = den;
                h[j + 1] = 0.0;
                g[j + 1] = -sn[j] * g[j];
                g[j] = cs[j] * g[j];
                rcols.push_back(std::move(h));
                ++st.iters;
                jused = j + 1;
                double hmax = 1.0;
                for (int i = 0; i <= j; ++i) hmax = std::max(hmax, std::abs(rcols[j][i]));
                const bool happy = hsub <= 1e-14 * hmax;
                if (!happy) basis.push_back(w);
                if (std::abs(g[j + 1]) <= target || happy) { cyc = true; break; }
            }
            if (jused == 0) { st.err = 1; return st; }
            Vec y(jused);
            for (int i = jused - 1; i >= 0; --i) {
                double v = g[i];
                for (int c = i + 1; c < jused; ++c) v -= rcols[c][i] * y[c];
                y[i] = v / rcols[i][i];
            }
            for (int j = 0; j < jused; ++j) {
                const double yj = y[j];
                for (size_t i = 0; i < n; ++i) x[i] += yj * basis[j][i];
            }
            if (cyc) {
                residual(r);
                if (norm2(r) <= target) {
                    st.converged = true;
                    st.final_rel = norm2(r) / beta0;
                    return st;
                }
                first = true;
                ++st.restarts;
                continue;
            }
            if (st.iters >= max_iters) break;
            ++st.restarts;
        }
        residual(r);
        st.final_rel = norm2(r) / beta0;
        st.converged = st.final_rel <= tol;
        return st;
    }

    // assemble_residual + residual_norm (local_ops.cpp:245-250,432-450)
    int residual(Vec& trace, Vec& interior, double* nrm) {
        int rc = assemble_core(false);
        if (rc) return rc;
        interior = ru;
        trace.assign(static_cast<size_t>(mpf) * nf, 0.0);
        for (int e = 0; e < ne; ++e)
            for (int lf = 0; lf < n_lfe; ++lf) {
                const int f = elem_faces[static_cast<size_t>(e) * n_lfe + lf];
                for (int r = 0; r < mpf; ++r) trace[static_cast<size_t>(f) * mpf + r] += ruhat_e[static_cast<size_t>(e) * nfl + lf * mpf + r];
            }
        double acc = 0.0;
        for (double v : trace) acc += v * v;
        for (double v : interior) acc += v * v;
        *nrm = std::sqrt(acc);
        return 0;
    }

    void recover_local(const Vec& duhat, Vec& du) const {
        const size_t sEE = static_cast<size_t>(npe) * npe, sEF = static_cast<size_t>(npe) * nfl;
        du.assign(static_cast<size_t>(npe) * ne, 0.0);
        parallel_for(ne, [&](size_t e0, size_t e1) {
            Vec de(nfl), tmp(npe);
            for (size_t e = e0; e < e1; ++e) {
                for (int lf = 0; lf < n_lfe; ++lf) {
                    const int f = elem_faces[e * n_lfe + lf];
                    for (int r = 0; r < mpf; ++r) de[lf * mpf + r] = duhat[static_cast<size_t>(f) * mpf + r];
                }
                gemv_one(npe, nfl, &fbar[e * sEF], de.data(), tmp.data(), false);
                for (int i = 0; i < npe; ++i) tmp[i] = ru[e * npe + i] - tmp[i];
                gemv_one(npe, npe, &ebar_inv[e * sEE], tmp.data(), &du[e * npe], false);
            }
        });
    }
};

}  // namespace

extern "C" {

void ora_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

// dims: D, M, ne, nf, n_lfe, n_orient, pe, pf, qe, qf
void* ora_create(const int* dims, const int* elem_faces, const int* elem_side, const int* face_elems,
                 const int* face_lidx, const int* face_orient, const int* bnd_tag, const double* phi,
                 const double* dphi0, const double* dphi1, const double* dphi2, const double* psi, const double* tphi,
                 const double* wq, const double* wf, const double* elem_detjac, const double* elem_invjac,
                 const double* elem_coords, const double* face_detjac, const double* face_coords,
                 const double* face_normal) {
    Case* c = new Case();
    c->D = dims[0]; c->M = dims[1]; c->ne = dims[2]; c->nf = dims[3]; c->n_lfe = dims[4]; c->n_orient = dims[5];
    c->pe = dims[6]; c->pf = dims[7]; c->qe = dims[8]; c->qf = dims[9];
    c->npe = c->M * c->pe; c->mpf = c->M * c->pf; c->nfl = c->n_lfe * c->mpf; c->nfs = c->n_lfe * c->pf; c->nb = 2 * c->n_lfe - 1;
    const int D = c->D, ne = c->ne, nf = c->nf;
    auto iv = [](const int* p, size_t n) { return std::vector<int>(p, p + n); };
    auto dv = [](const double* p, size_t n) { return Vec(p, p + n); };
    c->elem_faces = iv(elem_faces, static_cast<size_t>(ne) * c->n_lfe);
    c->elem_side = iv(elem_side, static_cast<size_t>(ne) * c->n_lfe);
    c->face_elems = iv(face_elems, static_cast<size_t>(nf) * 2);
    c->face_lidx = iv(face_lidx, static_cast<size_t>(nf) * 2);
    c->face_orient = iv(face_orient, static_cast<size_t>(nf) * 2);
    c->bnd_tag = iv(bnd_tag, nf);
    c->phi = dv(phi, static_cast<size_t>(c->pe) * c->qe);
    c->dphi[0] = dv(dphi0, c->phi.size());
    c->dphi[1] = dv(dphi1, c->phi.size());
    if (D == 3) c->dphi[2] = dv(dphi2, c->phi.size());
    c->psi = dv(psi, static_cast<size_t>(c->pf) * c->qf);
    c->tphi = dv(tphi, static_cast<size_t>(c->n_lfe) * c->n_orient * c->qf * c->pe);
    c->wq = dv(wq, c->qe);
    c->wf = dv(wf, c->qf);
    c->elem_detjac = dv(elem_detjac, static_cast<size_t>(ne) * c->qe);
    c->elem_invjac = dv(elem_invjac, static_cast<size_t>(ne) * c->qe * D * D);
    c->elem_coords = dv(elem_coords, static_cast<size_t>(ne) * c->qe * D);
    c->face_detjac = dv(face_detjac, static_cast<size_t>(nf) * c->qf);
    c->face_coords = dv(face_coords, static_cast<size_t>(nf) * c->qf * D);
    c->face_normal = dv(face_normal, static_cast<size_t>(nf) * 2 * c->qf * D);
    c->model.M = c->M;
    c->model.D = D;
    c->u.assign(static_cast<size_t>(c->npe) * ne, 0.0);
    c->uhat.assign(static_cast<size_t>(c->mpf) * nf, 0.0);
    return c;
}

void ora_free(void* h) { delete static_cast<Case*>(h); }
const char* ora_last_error(void* h) { return static_cast<Case*>(h)->err.c_str(); }
long ora_last_error_index(void* h) { return static_cast<Case*>(h)->err_index; }

void ora_set_model(void* h, int kind, const double* params, int n_params, const double* forcing_q,
                   const double* dirichlet_q) {
    Case* c = static_cast<Case*>(h);
    c->model.kind = kind;
    for (int i = 0; i < 16; ++i) c->model.p[i] = i < n_params ? params[i] : 0.0;
    if (forcing_q) c->forcing.assign(forcing_q, forcing_q + static_cast<size_t>(c->ne) * c->qe * c->M);
    else c->forcing.clear();
    if (dirichlet_q) c->dirichlet.assign(dirichlet_q, dirichlet_q + static_cast<size_t>(c->nf) * c->qf * c->M);
    else c->dirichlet.clear();
}

int ora_local_factors(void* h) { return static_cast<Case*>(h)->local_factors(); }

static Vec* field(Case* c, const std::string& s) {
    if (s == "u") return &c->u;
    if (s == "uhat") return &c->uhat;
    if (s == "u_prev") return &c->u_prev;
    if (s == "q0") return &c->q[0];
    if (s == "q1") return &c->q[1];
    if (s == "q2") return &c->q[2];
    if (s == "mass") return &c->mass;
    if (s == "mass_inv") return &c->mass_inv;
    if (s == "kbar") return &c->kbar;
    if (s == "ebar_inv") return &c->ebar_inv;
    if (s == "fbar") return &c->fbar;
    if (s == "hbar") return &c->hbar;
    if (s == "rbar") return &c->rbar;
    if (s == "ru") return &c->ru;
    if (s == "ruhat_e") return &c->ruhat_e;
    if (s == "e_raw") return &c->e_raw;
    if (s == "f_raw") return &c->f_raw;
    if (s == "h_raw") return &c->h_raw;
    if (s == "j_raw") return &c->j_raw;
    if (s == "blocks") return &c->blocks;
    if (s == "rhs") return &c->rhs;
    if (s == "bj_inv") return &c->bj_inv;
    if (s == "asm_inv") return &c->asm_inv;
    if (s == "ritz") return &c->ritz;
    if (s == "residual_history") return &c->residual_history;
    if (s == "alpha_history") return &c->alpha_history;
    for (int d = 0; d < 3; ++d) {
        const std::string k = std::to_string(d);
        if (s == "bmat" + k) return &c->bmat[d];
        if (s == "cmat" + k) return &c->cmat[d];
        if (s == "minv_b" + k) return &c->minv_b[d];
        if (s == "minv_c" + k) return &c->minv_c[d];
        if (s == "d_raw" + k) return &c->d_raw[d];
        if (s == "g_raw" + k) return &c->g_raw[d];
    }
    return nullptr;
}

long ora_get(void* h, const char* name, double* out, long cap) {
    Vec* v = field(static_cast<Case*>(h), name);
    if (!v) return -2;
    if (out) {
        if (cap < static_cast<long>(v->size())) return -1;
        std::memcpy(out, v->data(), v->size() * sizeof(double));
    }
    return static_cast<long>(v->size());
}

int ora_set(void* h, const char* name, const double* in, long n) {
    Vec* v = field(static_cast<Case*>(h), name);
    if (!v) return -2;
    v->assign(in, in + n);
    return 0;
}

long ora_get_neighbor(void* h, int64_t* out, long cap) {
    Case* c = static_cast<Case*>(h);
    if (out) {
        if (cap < static_cast<long>(c->neighbor.size())) return -1;
        std::memcpy(out, c->neighbor.data(), c->neighbor.size() * sizeof(int64_t));
    }
    return static_cast<long>(c->neighbor.size());
}

long ora_get_gmres_per_newton(void* h, int* out, long cap) {
    Case* c = static_cast<Case*>(h);
    if (out && cap >= static_cast<long>(c->gmres_per_newton.size()))
        std::memcpy(out, c->gmres_per_newton.data(), c->gmres_per_newton.size() * sizeof(int));
    return static_cast<long>(c->gmres_per_newton.size());
}

void ora_set_dt(void* h, double dt) { static_cast<Case*>(h)->dt = dt > 0.0 ? dt : 0.0; }
void ora_compute_q(void* h) { static_cast<Case*>(h)->compute_q(); }
int ora_assemble_core(void* h, int want_jac) { return static_cast<Case*>(h)->assemble_core(want_jac != 0); }
int ora_assemble_element_operators(void* h) { return static_cast<Case*>(h)->assemble_element_operators(); }
void ora_assemble_global(void* h) { static_cast<Case*>(h)->assemble_global(); }

void ora_matvec(void* h, const double* x, double* y) {
    Case* c = static_cast<Case*>(h);
    const size_t n = static_cast<size_t>(c->mpf) * c->nf;
    Vec xv(x, x + n), yv;
    c->matvec(xv, yv);
    std::memcpy(y, yv.data(), n * sizeof(double));
}

int ora_build_precond(void* h, int kind) { return static_cast<Case*>(h)->build_precond(kind); }
// polynomial wrapper on top of the base built by ora_build_precond: harmonic Ritz values of base(K .) (poly_kind 0)
// or the Chebyshev nodes derived from them (poly_kind 1), left in "ritz"
int ora_build_poly(void* h, int degree, int poly_kind, uint64_t seed) {
    return static_cast<Case*>(h)->build_poly(degree, poly_kind, seed);
}

void ora_apply_base(void* h, const double* y, double* z) {
    Case* c = static_cast<Case*>(h);
    const size_t n = static_cast<size_t>(c->mpf) * c->nf;
    Vec yv(y, y + n), zv;
    c->apply_base(yv, zv);
    std::memcpy(z, zv.data(), n * sizeof(double));
}

void ora_apply_precond(void* h, const double* y, double* z) {
    Case* c = static_cast<Case*>(h);
    const size_t n = static_cast<size_t>(c->mpf) * c->nf;
    Vec yv(y, y + n), zv;
    c->apply_precond(yv, zv);
    std::memcpy(z, zv.data(), n * sizeof(double));
}

int ora_residual(void* h, double* trace, double* interior, double* nrm) {
    Case* c = static_cast<Case*>(h);
    Vec t, i;
    const int rc = c->residual(t, i, nrm);
    if (rc) return rc;
    if (trace) std::memcpy(trace, t.data(), t.size() * sizeof(double));
    if (interior) std::memcpy(interior, i.data(), i.size() * sizeof(double));
    return 0;
}

void ora_recover_local(void* h, const double* duhat, double* du) {
    Case* c = static_cast<Case*>(h);
    Vec d(duhat, duhat + static_cast<size_t>(c->mpf) * c->nf), out;
    c->recover_local(d, out);
    std::memcpy(du, out.data(), out.size() * sizeof(double));
}

// stats: iters, restarts, final_rel, converged, t_mv, t_prec, t_orth
int ora_gmres(void* h, const double* rhs, const double* x0, int restart, double tol, int max_iters, int mgs,
              double* x, double* stats) {
    Case* c = static_cast<Case*>(h);
    const size_t n = static_cast<size_t>(c->mpf) * c->nf;
    Vec b = rhs ? Vec(rhs, rhs + n) : c->rhs;
    Vec xv = x0 ? Vec(x0, x0 + n) : Vec(n, 0.0);
    const Stats st = c->gmres(b, xv, restart, tol, max_iters, mgs != 0);
    if (st.err) { c->err = "NaN detected in gmres"; return 6; }
    std::memcpy(x, xv.data(), n * sizeof(double));
    stats[0] = st.iters; stats[1] = st.restarts; stats[2] = st.final_rel; stats[3] = st.converged ? 1.0 : 0.0;
    stats[4] = st.t_mv; stats[5] = st.t_prec; stats[6] = st.t_orth;
    return 0;
}

// newton_solve (newton.cpp:54-154).  poly_degree > 0: the polynomial wrapper is rebuilt every Newton step
// (build_preconditioner, newton.cpp:30-52); poly_degree == 0 keeps whatever ritz values were set with
// ora_set("ritz") (fixed interpolation nodes, used by the apply_poly parity tests); poly_degree < 0: none.
// report: n_newton, n_gmres_total, n_inner, final_residual, converged, t_ass, t_mv, t_prec, t_orth, t_total
int ora_newton(void* h, double newton_tol, int max_newton, double min_alpha, int restart, double gmres_tol,
               int gmres_max_iters, int mgs, int pc_kind, int poly_degree, int poly_kind, uint64_t seed, double* report) {
    Case* c = static_cast<Case*>(h);
    const auto t_start = Clock::now();
    c->residual_history.clear();
    c->alpha_history.clear();
    c->gmres_per_newton.clear();
    c->inner_ops = 0;
    std::fill(report, report + 10, 0.0);
    Vec tr, in;
    double rnorm = 0.0;
    int rc = c->residual(tr, in, &rnorm);
    if (rc) return rc;
    c->residual_history.push_back(rnorm);
    const size_t n = static_cast<size_t>(c->mpf) * c->nf;
    for (int iter = 0;; ++iter) {
        if (rnorm <= newton_tol) { report[4] = 1.0; break; }
        if (iter >= max_newton) { report[4] = 0.0; break; }
        auto t0 = Clock::now();
        rc = c->assemble_element_operators();
        if (rc) return rc;
        c->assemble_global();
        const Vec keep_ritz = c->ritz;
        rc = c->build_precond(pc_kind);
        c->ritz = keep_ritz;
        if (rc) return rc;
        if (poly_degree > 0) {
            rc = c->build_poly(poly_degree, poly_kind, seed);
            if (rc) return rc;
        }
        report[5] += since(t0);
        Vec duhat(n, 0.0);
        const Stats st = c->gmres(c->rhs, duhat, restart, gmres_tol, gmres_max_iters, mgs != 0);
        if (st.err) { c->err = "NaN detected in gmres"; return 6; }
        report[1] += st.iters;
        c->gmres_per_newton.push_back(st.iters);
        report[6] += st.t_mv; report[7] += st.t_prec; report[8] += st.t_orth;
        Vec du;
        c->recover_local(duhat, du);
        const Vec u0 = c->u, uh0 = c->uhat;
        bool accepted = false;
        for (double alpha = 1.0; alpha >= min_alpha; alpha *= 0.5) {
            for (size_t i = 0; i < u0.size(); ++i) c->u[i] = u0[i] + alpha * du[i];
            for (size_t i = 0; i < uh0.size(); ++i) c->uhat[i] = uh0[i] + alpha * duhat[i];
            double tnorm = 0.0;
            rc = c->residual(tr, in, &tnorm);
            if (rc) return rc;
            if (tnorm < rnorm) {
                rnorm = tnorm;
                accepted = true;
                c->alpha_history.push_back(alpha);
                break;
            }
        }
        report[0] += 1.0;
        if (!accepted) {
            c->u = u0;
            c->uhat = uh0;
            c->err = "line search failed";
            report[3] = rnorm;
            return 7;
        }
        c->residual_history.push_back(rnorm);
    }
    report[2] = static_cast<double>(c->inner_ops);
    report[3] = rnorm;
    report[9] = since(t_start);
    return 0;
}

int ora_lu_invert_batch(int n, int batch, const double* a, double* out, long* bad) {
    *bad = invert_batch(n, batch, a, out);
    return *bad >= 0 ? 2 : 0;
}

}  // extern "C"
