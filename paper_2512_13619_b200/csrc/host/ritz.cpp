// Host side of the polynomial preconditioner setup: harmonic Ritz values from the Arnoldi
// Hessenberg matrix (preconditioner.cpp:162-205) and Leja ordering (:207-244).  The reference
// delegates the small dense solve and the eigenvalue computation to Eigen (FullPivLU /
// EigenSolver); here they are a complete-pivoting elimination and the real double-shift QR
// iteration on the Hessenberg matrix (Francis / EISPACK "hqr" scheme), written from the published
// algorithm.  P is at most a few dozen, so this is negligible next to the P device matvecs.
#include "ritz.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>

namespace hdgb {

namespace {

// Solves A x = b (A column-major n x n) with complete pivoting.  Returns false when A is
// numerically rank deficient (pivot <= eps * n * largest pivot).
bool solve_complete_pivoting(std::vector<double> a, std::vector<double> b, int n, std::vector<double>& x) {
    std::vector<int> colperm(n);
    for (int i = 0; i < n; ++i) colperm[i] = i;
    auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(j) * n + i]; };
    double maxpiv = 0.0;
    std::vector<double> piv(n, 0.0);
    for (int k = 0; k < n; ++k) {
        int pi = k, pj = k;
        double best = -1.0;
        for (int j = k; j < n; ++j)
            for (int i = k; i < n; ++i)
                if (std::abs(A(i, j)) > best) { best = std::abs(A(i, j)); pi = i; pj = j; }
        if (!(best > 0.0)) return false;
        if (pi != k) {
            for (int j = 0; j < n; ++j) std::swap(A(k, j), A(pi, j));
            std::swap(b[k], b[pi]);
        }
        if (pj != k) {
            for (int i = 0; i < n; ++i) std::swap(A(i, k), A(i, pj));
            std::swap(colperm[k], colperm[pj]);
        }
        piv[k] = std::abs(A(k, k));
        maxpiv = std::max(maxpiv, piv[k]);
        for (int i = k + 1; i < n; ++i) {
            const double m = A(i, k) / A(k, k);
            if (m == 0.0) continue;
            for (int j = k + 1; j < n; ++j) A(i, j) -= m * A(k, j);
            b[i] -= m * b[k];
        }
    }
    const double thr = std::numeric_limits<double>::epsilon() * n * maxpiv;
    for (int k = 0; k < n; ++k)
        if (!(piv[k] > thr)) return false;
    std::vector<double> y(n);
    for (int i = n - 1; i >= 0; --i) {
        double v = b[i];
        for (int j = i + 1; j < n; ++j) v -= A(i, j) * y[j];
        y[i] = v / A(i, i);
    }
    x.assign(n, 0.0);
    for (int i = 0; i < n; ++i) x[colperm[i]] = y[i];
    return true;
}

// Eigenvalues of a real upper Hessenberg matrix (column-major n x n, destroyed) by the implicit
// double-shift QR iteration.
std::vector<std::complex<double>> hessenberg_eigenvalues(std::vector<double> h, int n) {
    auto H = [&](int i, int j) -> double& { return h[static_cast<size_t>(j) * n + i]; };
    std::vector<std::complex<double>> ev(n);
    double anorm = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = std::max(i - 1, 0); j < n; ++j) anorm += std::abs(H(i, j));
    int nn = n - 1;
    double t = 0.0;
    const double eps = std::numeric_limits<double>::epsilon();
    while (nn >= 0) {
        int its = 0, l;
        do {
            for (l = nn; l >= 1; --l) {
                double s = std::abs(H(l - 1, l - 1)) + std::abs(H(l, l));
                if (s == 0.0) s = anorm;
                if (std::abs(H(l, l - 1)) <= eps * s) {
                    H(l, l - 1) = 0.0;
                    break;
                }
            }
            double x = H(nn, nn);
            if (l == nn) {  // one real root
                ev[nn--] = {x + t, 0.0};
            } else {
                double y = H(nn - 1, nn - 1);
                double w = H(nn, nn - 1) * H(nn - 1, nn);
                if (l == nn - 1) {  // a 2x2 block: two roots
                    const double p = 0.5 * (y - x);
                    const double q = p * p + w;
                    const double z = std::sqrt(std::abs(q));
                    x += t;
                    if (q >= 0.0) {
                        const double zz = p + (p >= 0.0 ? std::abs(z) : -std::abs(z));
                        ev[nn - 1] = ev[nn] = {x + zz, 0.0};
                        if (zz != 0.0) ev[nn] = {x - w / zz, 0.0};
                    } else {
                        ev[nn - 1] = {x + p, z};
                        ev[nn] = {x + p, -z};
                    }
                    nn -= 2;
                } else {
                    if (its == 60) {  // no convergence: report what is on the diagonal
                        std::fprintf(stderr, "warning: Hessenberg QR did not converge; using diagonal entries\n");
                        for (int i = 0; i <= nn; ++i) ev[i] = {H(i, i) + t, 0.0};
                        return ev;
                    }
                    if (its == 10 || its == 20) {  // exceptional shift
                        t += x;
                        for (int i = 0; i <= nn; ++i) H(i, i) -= x;
                        const double s = std::abs(H(nn, nn - 1)) + std::abs(H(nn - 1, nn - 2));
                        y = x = 0.75 * s;
                        w = -0.4375 * s * s;
                    }
                    ++its;
                    int m;
                    double p = 0, q = 0, r = 0, z = 0;
                    for (m = nn - 2; m >= l; --m) {
                        z = H(m, m);
                        const double rr = x - z, ss = y - z;
                        p = (rr * ss - w) / H(m + 1, m) + H(m, m + 1);
                        q = H(m + 1, m + 1) - z - rr - ss;
                        r = H(m + 2, m + 1);
                        const double sc = std::abs(p) + std::abs(q) + std::abs(r);
                        p /= sc; q /= sc; r /= sc;
                        if (m == l) break;
                        const double u = std::abs(H(m, m - 1)) * (std::abs(q) + std::abs(r));
                        const double v = std::abs(p) * (std::abs(H(m - 1, m - 1)) + std::abs(z) + std::abs(H(m + 1, m + 1)));
                        if (u <= eps * v) break;
                    }
                    for (int i = m + 2; i <= nn; ++i) {
                        H(i, i - 2) = 0.0;
                        if (i != m + 2) H(i, i - 3) = 0.0;
                    }
                    for (int k = m; k <= nn - 1; ++k) {
                        if (k != m) {
                            p = H(k, k - 1);
                            q = H(k + 1, k - 1);
                            r = (k != nn - 1) ? H(k + 2, k - 1) : 0.0;
                            x = std::abs(p) + std::abs(q) + std::abs(r);
                            if (x != 0.0) { p /= x; q /= x; r /= x; }
                        }
                        const double sgn = (p >= 0.0) ? 1.0 : -1.0;
                        const double s = sgn * std::sqrt(p * p + q * q + r * r);
                        if (s != 0.0) {
                            if (k == m) {
                                if (l != m) H(k, k - 1) = -H(k, k - 1);
                            } else {
                                H(k, k - 1) = -s * x;
                            }
                            p += s;
                            x = p / s;
                            y = q / s;
                            z = r / s;
                            q /= p;
                            r /= p;
                            for (int j = k; j <= nn; ++j) {
                                p = H(k, j) + q * H(k + 1, j);
                                if (k != nn - 1) {
                                    p += r * H(k + 2, j);
                                    H(k + 2, j) -= p * z;
                                }
                                H(k + 1, j) -= p * y;
                                H(k, j) -= p * x;
                            }
                            const int mmin = nn < k + 3 ? nn : k + 3;
                            for (int i = l; i <= mmin; ++i) {
                                p = x * H(i, k) + y * H(i, k + 1);
                                if (k != nn - 1) {
                                    p += z * H(i, k + 2);
                                    H(i, k + 2) -= p * r;
                                }
                                H(i, k + 1) -= p * q;
                                H(i, k) -= p;
                            }
                        }
                    }
                }
            }
        } while (nn >= 0 && l < nn - 1);
    }
    return ev;
}

}  // namespace

std::vector<std::complex<double>> leja_order(const std::vector<std::complex<double>>& theta) {
    using C = std::complex<double>;
    std::vector<C> pool;
    for (const C& t : theta)
        if (t.imag() >= 0.0) pool.push_back(t);  // reals and upper-half representatives
    std::vector<C> ordered;
    std::vector<char> taken(pool.size(), 0);
    for (size_t step = 0; step < pool.size(); ++step) {
        int pick = -1;
        double pick_score = 0.0;
        for (size_t c = 0; c < pool.size(); ++c) {
            if (taken[c]) continue;
            double score = 0.0;
            if (ordered.empty()) {
                score = std::abs(pool[c]);
            } else {
                for (const C& z : ordered) score += std::log(std::abs(pool[c] - z));
            }
            bool wins = pick < 0;
            if (!wins) {
                const C& cur = pool[pick];
                if (score != pick_score) wins = score > pick_score;
                else if (pool[c].real() != cur.real()) wins = pool[c].real() > cur.real();
                else wins = pool[c].imag() > cur.imag();
            }
            if (wins) {
                pick = static_cast<int>(c);
                pick_score = score;
            }
        }
        taken[pick] = 1;
        ordered.push_back(pool[pick]);
        if (pool[pick].imag() > 0.0) ordered.push_back(std::conj(pool[pick]));
    }
    return ordered;
}

std::vector<std::complex<double>> harmonic_ritz_from_hessenberg(const double* hess, int pmax, int p_eff) {
    const int p = p_eff;
    const int ld = pmax + 1;
    std::vector<double> hs(static_cast<size_t>(p) * p);
    for (int j = 0; j < p; ++j)
        for (int i = 0; i < p; ++i) hs[static_cast<size_t>(j) * p + i] = hess[static_cast<size_t>(j) * ld + i];
    const double hp1 = (p < pmax) ? 0.0 : hess[static_cast<size_t>(p - 1) * ld + p];
    if (hp1 != 0.0) {
        // last column += hp1^2 * (Hs^T)^-1 e_p
        std::vector<double> ht(static_cast<size_t>(p) * p), ep(p, 0.0), z;
        for (int j = 0; j < p; ++j)
            for (int i = 0; i < p; ++i) ht[static_cast<size_t>(j) * p + i] = hs[static_cast<size_t>(i) * p + j];
        ep[p - 1] = 1.0;
        if (solve_complete_pivoting(ht, ep, p, z)) {
            for (int i = 0; i < p; ++i) hs[static_cast<size_t>(p - 1) * p + i] += hp1 * hp1 * z[i];
        } else {
            std::fprintf(stderr, "warning: singular Hessenberg block, using plain Ritz values\n");
        }
    }
    const std::vector<std::complex<double>> raw = hessenberg_eigenvalues(hs, p);
    std::vector<std::complex<double>> vals;
    double max_abs = 0.0;
    for (std::complex<double> t : raw) {
        if (std::abs(t.imag()) < 1e-12 * std::abs(t)) t = {t.real(), 0.0};
        vals.push_back(t);
        max_abs = std::max(max_abs, std::abs(t));
    }
    std::vector<std::complex<double>> kept;
    for (const auto& t : vals) {
        if (std::abs(t) < 1e-12 * max_abs) {
            std::fprintf(stderr, "warning: dropping near-zero Ritz value (%g, %g)\n", t.real(), t.imag());
            continue;
        }
        if (t.imag() < 0.0) continue;
        kept.push_back(t);
        if (t.imag() > 0.0) kept.emplace_back(t.real(), -t.imag());
    }
    return leja_order(kept);
}

}  // namespace hdgb
