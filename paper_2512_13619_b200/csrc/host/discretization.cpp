#include "discretization.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <random>
#include <stdexcept>
#include <string>

#include "../common.cuh"

namespace hdgb {

namespace {

constexpr double kPi = 3.14159265358979323846;

// Legendre polynomial of degree n and its derivative at x in (-1,1), three-term recurrence.
struct LegendreEval {
    double value, deriv;
};
LegendreEval legendre_eval(int n, double x) {
    if (n == 0) return {1.0, 0.0};
    double pm = 1.0, pc = x;
    for (int j = 2; j <= n; ++j) {
        const double pn = ((2.0 * j - 1.0) * x * pc - (j - 1.0) * pm) / j;
        pm = pc;
        pc = pn;
    }
    return {pc, n * (x * pc - pm) / (x * x - 1.0)};
}

}  // namespace

Rule1D gauss_rule(int q) {
    if (q < 1 || q > 30)
        throw Failure(HDGB_ERR_UNSUPPORTED, "gauss_rule supports 1..30 points, got " + std::to_string(q));
    std::vector<double> node(q), weight(q);
    // Roots of P_q by Newton from the Chebyshev-type guess; only the left half is computed and
    // the right half mirrored, which makes the rule exactly symmetric index-wise.
    for (int i = 0; i < (q + 1) / 2; ++i) {
        double t = -std::cos(kPi * (i + 0.75) / (q + 0.5));
        for (int it = 0; it < 100; ++it) {
            const LegendreEval le = legendre_eval(q, t);
            const double step = le.value / le.deriv;
            t -= step;
            if (std::abs(step) < 1e-15) break;
        }
        const LegendreEval le = legendre_eval(q, t);
        node[i] = t;
        weight[i] = 2.0 / ((1.0 - t * t) * le.deriv * le.deriv);
        node[q - 1 - i] = -t;
        weight[q - 1 - i] = weight[i];
    }
    if (q % 2 == 1) node[q / 2] = 0.0;
    Rule1D r;
    r.pts.resize(q);
    r.wts.resize(q);
    for (int i = 0; i < q; ++i) {
        r.pts[i] = 0.5 * (node[i] + 1.0);
        r.wts[i] = 0.5 * weight[i];
    }
    return r;
}

std::vector<double> lobatto_nodes(int n) {
    if (n < 2) throw Failure(HDGB_ERR_UNSUPPORTED, "lobatto_nodes needs at least 2 points");
    std::vector<double> x(n);
    x[0] = -1.0;
    x[n - 1] = 1.0;
    const int m = n - 1;  // interior nodes: roots of P'_m
    for (int i = 1; i < m; ++i) {
        double t = -std::cos(kPi * i / m);
        for (int it = 0; it < 100; ++it) {
            const LegendreEval le = legendre_eval(m, t);
            // second derivative from the Legendre differential equation
            const double second = (2.0 * t * le.deriv - m * (m + 1.0) * le.value) / (1.0 - t * t);
            const double step = le.deriv / second;
            t -= step;
            if (std::abs(step) < 1e-15) break;
        }
        x[i] = t;
    }
    for (int i = 0; i < n / 2; ++i) x[n - 1 - i] = -x[i];
    if (n % 2 == 1) x[n / 2] = 0.0;
    std::vector<double> out(n);
    for (int i = 0; i < n; ++i) out[i] = 0.5 * (x[i] + 1.0);
    return out;
}

void lagrange_values(const std::vector<double>& nodes, double x, double* out) {
    const int n = static_cast<int>(nodes.size());
    for (int j = 0; j < n; ++j) {
        double v = 1.0;
        for (int m = 0; m < n; ++m)
            if (m != j) v *= (x - nodes[m]) / (nodes[j] - nodes[m]);
        out[j] = v;
    }
}

void lagrange_derivs(const std::vector<double>& nodes, double x, double* out) {
    const int n = static_cast<int>(nodes.size());
    for (int j = 0; j < n; ++j) {
        double total = 0.0;
        for (int l = 0; l < n; ++l) {
            if (l == j) continue;
            double term = 1.0 / (nodes[j] - nodes[l]);
            for (int m = 0; m < n; ++m)
                if (m != j && m != l) term *= (x - nodes[m]) / (nodes[j] - nodes[m]);
            total += term;
        }
        out[j] = total;
    }
}

// ---- shapes ------------------------------------------------------------------------------------
const ShapeInfo& shape_info(int shape) {
    // Quadrilateral: CCW vertices; faces bottom, right, top, left traversed along +x / +y
    // (mesh.cpp:14 kFaceEnds).  Outward normal = tangent rotated -90 deg for bottom/right.
    static const ShapeInfo quad = {2, 4, 4, 2, 2,
                                   {{0, 1, -1, -1}, {1, 2, -1, -1}, {3, 2, -1, -1}, {0, 3, -1, -1}, {-1, -1, -1, -1}, {-1, -1, -1, -1}},
                                   {+1, +1, -1, -1, 0, 0}};
    // Hexahedron: v0..v3 = bottom (z=0) CCW, v4..v7 above them.  Faces z=0, y=0, x=1, y=1, x=0,
    // z=1, each parameterised along the two remaining axes in increasing order; vertices listed
    // in parameter-corner order (0,0),(1,0),(1,1),(0,1).
    static const ShapeInfo hex = {3, 6, 8, 4, 8,
                                  {{0, 1, 2, 3}, {0, 1, 5, 4}, {1, 2, 6, 5}, {3, 2, 6, 7}, {0, 3, 7, 4}, {4, 5, 6, 7}},
                                  {-1, +1, +1, -1, -1, +1}};
    // Triangle: CCW vertices (0,0),(1,0),(0,1); faces v0v1, v1v2, v2v0 traversed first -> second
    // vertex; outward normal = tangent rotated -90 degrees on every face.
    static const ShapeInfo tri = {2, 3, 3, 2, 2,
                                  {{0, 1, -1, -1}, {1, 2, -1, -1}, {2, 0, -1, -1}, {-1, -1, -1, -1}, {-1, -1, -1, -1}, {-1, -1, -1, -1}},
                                  {+1, +1, +1, 0, 0, 0}};
    // Tetrahedron: positively oriented (0,0,0),(1,0,0),(0,1,0),(0,0,1); every face is listed so that
    // (b - a) x (c - a) points outward.  6 relative orientations of a triangular face.
    static const ShapeInfo tet = {3, 4, 4, 3, 6,
                                  {{1, 2, 3, -1}, {0, 3, 2, -1}, {0, 1, 3, -1}, {0, 2, 1, -1}, {-1, -1, -1, -1}, {-1, -1, -1, -1}},
                                  {+1, +1, +1, +1, 0, 0}};
    switch (shape) {
        case HDGB_QUAD: return quad;
        case HDGB_HEX: return hex;
        case HDGB_TRI: return tri;
        case HDGB_TET: return tet;
        default: throw Failure(HDGB_ERR_UNSUPPORTED, "unknown element shape");
    }
}

namespace {

// Reference coordinates of local face lf at face parameter (s,t).
void face_point(int shape, int lf, double s, double t, double* xi) {
    if (shape == HDGB_QUAD) {
        switch (lf) {
            case 0: xi[0] = s; xi[1] = 0.0; break;
            case 1: xi[0] = 1.0; xi[1] = s; break;
            case 2: xi[0] = s; xi[1] = 1.0; break;
            default: xi[0] = 0.0; xi[1] = s; break;
        }
        return;
    }
    if (shape == HDGB_TRI) {
        switch (lf) {
            case 0: xi[0] = s; xi[1] = 0.0; break;
            case 1: xi[0] = 1.0 - s; xi[1] = s; break;
            default: xi[0] = 0.0; xi[1] = 1.0 - s; break;
        }
        return;
    }
    if (shape == HDGB_TET) {
        static const double rv[4][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
        const ShapeInfo& si = shape_info(shape);
        const double* a = rv[si.face_verts[lf][0]];
        const double* b = rv[si.face_verts[lf][1]];
        const double* c = rv[si.face_verts[lf][2]];
        for (int d = 0; d < 3; ++d) xi[d] = a[d] + s * (b[d] - a[d]) + t * (c[d] - a[d]);
        return;
    }
    switch (lf) {  // hex
        case 0: xi[0] = s; xi[1] = t; xi[2] = 0.0; break;
        case 1: xi[0] = s; xi[1] = 0.0; xi[2] = t; break;
        case 2: xi[0] = 1.0; xi[1] = s; xi[2] = t; break;
        case 3: xi[0] = s; xi[1] = 1.0; xi[2] = t; break;
        case 4: xi[0] = 0.0; xi[1] = s; xi[2] = t; break;
        default: xi[0] = s; xi[1] = t; xi[2] = 1.0; break;
    }
}

// Corner k of the unit square in parameter-corner order.
constexpr int kCornerS[4] = {0, 1, 1, 0};
constexpr int kCornerT[4] = {0, 0, 1, 1};

// For quadrilateral faces: orientation o = r + 4*flip means canonical corner j coincides with the
// side-local corner (r + j) % 4 (flip = 0) or (r - j) mod 4 (flip = 1).
int local_corner(int o, int j) {
    const int r = o & 3;
    return (o < 4) ? (r + j) & 3 : (r - j + 4) & 3;
}

}  // namespace

namespace {

// ---- simplex master elements --------------------------------------------------------------------
// Nodal basis on the principal lattice of order k: for the node with barycentric lattice indices
// (i_0 .. i_D), sum = k,  phi(lambda) = prod_d N_{i_d}(lambda_d),  N_i(l) = prod_{m<i} (k l - m)/(i - m)
// -- a closed form (no Vandermonde inversion); derivatives by the product rule.
double lattice_factor(int k, int i, double l) {
    double v = 1.0;
    for (int m = 0; m < i; ++m) v *= (k * l - m) / static_cast<double>(i - m);
    return v;
}
double lattice_factor_deriv(int k, int i, double l) {
    double total = 0.0;
    for (int q = 0; q < i; ++q) {
        double term = k / static_cast<double>(i - q);
        for (int m = 0; m < i; ++m)
            if (m != q) term *= (k * l - m) / static_cast<double>(i - m);
        total += term;
    }
    return total;
}

// lattice index tuples (i_1 .. i_dim) with i_1 fastest; i_0 = k - sum
std::vector<std::array<int, 3>> lattice_nodes(int dim, int k) {
    std::vector<std::array<int, 3>> out;
    if (dim == 1) {
        for (int a = 0; a <= k; ++a) out.push_back({a, 0, 0});
    } else if (dim == 2) {
        for (int b = 0; b <= k; ++b)
            for (int a = 0; a + b <= k; ++a) out.push_back({a, b, 0});
    } else {
        for (int c = 0; c <= k; ++c)
            for (int b = 0; b + c <= k; ++b)
                for (int a = 0; a + b + c <= k; ++a) out.push_back({a, b, c});
    }
    return out;
}

// values (and optionally d/dxi_r) of all lattice basis functions at the reference point xi
void simplex_basis(int dim, int k, const std::vector<std::array<int, 3>>& nodes, const double* xi, double* val,
                   double* const* dval) {
    double lam[4], sum = 0.0;
    for (int d = 0; d < dim; ++d) { lam[d + 1] = xi[d]; sum += xi[d]; }
    lam[0] = 1.0 - sum;
    for (size_t n = 0; n < nodes.size(); ++n) {
        int idx[4] = {k, 0, 0, 0};
        for (int d = 0; d < dim; ++d) { idx[d + 1] = nodes[n][d]; idx[0] -= nodes[n][d]; }
        double f[4], df[4];
        for (int d = 0; d <= dim; ++d) {
            f[d] = lattice_factor(k, idx[d], lam[d]);
            df[d] = dval ? lattice_factor_deriv(k, idx[d], lam[d]) : 0.0;
        }
        double v = 1.0;
        for (int d = 0; d <= dim; ++d) v *= f[d];
        val[n] = v;
        if (dval) {
            double dl[4];  // d phi / d lambda_d
            for (int d = 0; d <= dim; ++d) {
                double t = df[d];
                for (int e = 0; e <= dim; ++e)
                    if (e != d) t *= f[e];
                dl[d] = t;
            }
            for (int r = 0; r < dim; ++r) dval[r][n] = dl[r + 1] - dl[0];  // lambda_0 = 1 - sum xi
        }
    }
}

// canonical -> side-local barycentric map of a triangular face for orientation o (orientation_of):
// o < 3: local[(o + j) % 3] = canon[j];  o >= 3: local[(o - 3 - j) mod 3] = canon[j]
void tri_face_local_params(int o, double s, double t, double& ls, double& lt) {
    const double lc[3] = {1.0 - s - t, s, t};
    double ll[3];
    for (int j = 0; j < 3; ++j) {
        const int r = o % 3;
        const int li = (o < 3) ? (r + j) % 3 : ((r - j) % 3 + 3) % 3;
        ll[li] = lc[j];
    }
    ls = ll[1];
    lt = ll[2];
}

MasterElement make_simplex_master(int shape, int degree, int quad_points) {
    const ShapeInfo& si = shape_info(shape);
    MasterElement me;
    me.shape = shape; me.dim = si.dim; me.degree = degree; me.n_lfe = si.n_lfe; me.n_orient = si.n_orient;
    const int D = si.dim, k = degree;
    const int q = quad_points > 0 ? quad_points : degree + 2;
    me.rule1d = gauss_rule(q);
    me.nodes1d.resize(k + 1);
    for (int a = 0; a <= k; ++a) me.nodes1d[a] = static_cast<double>(a) / k;
    const std::vector<double>& p = me.rule1d.pts;
    const std::vector<double>& w = me.rule1d.wts;
    const auto enodes = lattice_nodes(D, k);
    const auto fnodes = lattice_nodes(D - 1, k);
    me.pe = static_cast<int>(enodes.size());
    me.pf = static_cast<int>(fnodes.size());
    me.elem_nodes.resize(static_cast<size_t>(me.pe) * D);
    for (int n = 0; n < me.pe; ++n)
        for (int d = 0; d < D; ++d) me.elem_nodes[static_cast<size_t>(n) * D + d] = static_cast<double>(enodes[n][d]) / k;
    me.face_nodes.resize(static_cast<size_t>(me.pf) * (D - 1));
    for (int n = 0; n < me.pf; ++n)
        for (int d = 0; d < D - 1; ++d) me.face_nodes[static_cast<size_t>(n) * (D - 1) + d] = static_cast<double>(fnodes[n][d]) / k;

    // Collapsed-coordinate (Duffy) Gauss rules: x = u, y = v (1 - u) [, z = w (1 - u)(1 - v)];
    // q points per direction integrate total degree 2q - D exactly.
    me.qe = (D == 2) ? q * q : q * q * q;
    me.elem_pts.resize(static_cast<size_t>(me.qe) * D);
    me.elem_wts.resize(me.qe);
    for (int g = 0; g < me.qe; ++g) {
        const int gu = g % q, gv = (g / q) % q, gw = g / (q * q);
        const double u = p[gu], v = p[gv];
        if (D == 2) {
            me.elem_pts[2 * g] = u;
            me.elem_pts[2 * g + 1] = v * (1.0 - u);
            me.elem_wts[g] = w[gu] * w[gv] * (1.0 - u);
        } else {
            // nested collapse: x = u, y = v (1 - u), z = ww (1 - u)(1 - v)
            const double ww = p[gw];
            me.elem_pts[3 * g] = u;
            me.elem_pts[3 * g + 1] = v * (1.0 - u);
            me.elem_pts[3 * g + 2] = ww * (1.0 - u) * (1.0 - v);
            me.elem_wts[g] = w[gu] * w[gv] * w[gw] * (1.0 - u) * (1.0 - u) * (1.0 - v);
        }
    }
    me.qf = (D == 2) ? q : q * q;
    me.face_pts.resize(static_cast<size_t>(me.qf) * (D - 1));
    me.face_wts.resize(me.qf);
    for (int g = 0; g < me.qf; ++g) {
        if (D == 2) {
            me.face_pts[g] = p[g];
            me.face_wts[g] = w[g];
        } else {
            const double u = p[g % q], v = p[g / q];
            me.face_pts[2 * g] = u;
            me.face_pts[2 * g + 1] = v * (1.0 - u);
            me.face_wts[g] = w[g % q] * w[g / q] * (1.0 - u);
        }
    }

    me.phi.resize(static_cast<size_t>(me.pe) * me.qe);
    for (int d = 0; d < D; ++d) me.dphi[d].resize(me.phi.size());
    for (int g = 0; g < me.qe; ++g) {
        const size_t o = static_cast<size_t>(me.pe) * g;
        double* dv[3] = {&me.dphi[0][o], &me.dphi[1][o], D == 3 ? &me.dphi[2][o] : nullptr};
        simplex_basis(D, k, enodes, &me.elem_pts[static_cast<size_t>(g) * D], &me.phi[o], dv);
    }
    me.psi.resize(static_cast<size_t>(me.pf) * me.qf);
    for (int g = 0; g < me.qf; ++g)
        simplex_basis(D - 1, k, fnodes, &me.face_pts[static_cast<size_t>(g) * (D - 1)], &me.psi[static_cast<size_t>(me.pf) * g], nullptr);

    // element basis on local face lf seen with orientation o at the CANONICAL face point gc
    me.tphi_local.resize(static_cast<size_t>(me.n_lfe) * me.qf * me.pe);
    me.tphi.resize(static_cast<size_t>(me.n_lfe) * me.n_orient * me.qf * me.pe);
    for (int lf = 0; lf < me.n_lfe; ++lf)
        for (int o = 0; o < me.n_orient; ++o)
            for (int gc = 0; gc < me.qf; ++gc) {
                double ls, lt = 0.0, xi[3];
                if (D == 2) {
                    ls = (o == 0) ? me.face_pts[gc] : 1.0 - me.face_pts[gc];
                } else {
                    tri_face_local_params(o, me.face_pts[2 * gc], me.face_pts[2 * gc + 1], ls, lt);
                }
                face_point(shape, lf, ls, lt, xi);
                double* dst = &me.tphi[((static_cast<size_t>(lf) * me.n_orient + o) * me.qf + gc) * me.pe];
                simplex_basis(D, k, enodes, xi, dst, nullptr);
                if (o == 0) std::copy(dst, dst + me.pe, &me.tphi_local[(static_cast<size_t>(lf) * me.qf + gc) * me.pe]);
            }
    return me;
}

}  // namespace

MasterElement make_master_element(int shape, int degree, int quad_points) {
    if (degree < 1 || degree > 6)
        throw Failure(HDGB_ERR_UNSUPPORTED, "supported polynomial degrees are 1..6, got " + std::to_string(degree));
    if (shape == HDGB_TRI || shape == HDGB_TET) return make_simplex_master(shape, degree, quad_points);
    const ShapeInfo& si = shape_info(shape);
    MasterElement me;
    me.shape = shape;
    me.dim = si.dim;
    me.degree = degree;
    me.n_lfe = si.n_lfe;
    me.n_orient = si.n_orient;
    const int q = quad_points > 0 ? quad_points : degree + 2;  // study.cpp:69
    me.rule1d = gauss_rule(q);
    me.nodes1d = lobatto_nodes(degree + 1);
    const int n1 = degree + 1;
    const int D = si.dim;
    me.pf = (D == 2) ? n1 : n1 * n1;
    me.pe = me.pf * n1;
    me.qf = (D == 2) ? q : q * q;
    me.qe = me.qf * q;

    const std::vector<double>& p = me.rule1d.pts;
    const std::vector<double>& w = me.rule1d.wts;

    // Tensor rules, first coordinate fastest.
    me.elem_pts.resize(static_cast<size_t>(me.qe) * D);
    me.elem_wts.resize(me.qe);
    for (int g = 0; g < me.qe; ++g) {
        const int gx = g % q, gy = (g / q) % q, gz = g / (q * q);
        me.elem_pts[g * D + 0] = p[gx];
        me.elem_pts[g * D + 1] = p[gy];
        if (D == 3) me.elem_pts[g * D + 2] = p[gz];
        me.elem_wts[g] = (D == 2) ? w[gx] * w[gy] : w[gx] * w[gy] * w[gz];
    }
    me.face_pts.resize(static_cast<size_t>(me.qf) * (D - 1));
    me.face_wts.resize(me.qf);
    for (int g = 0; g < me.qf; ++g) {
        if (D == 2) {
            me.face_pts[g] = p[g];
            me.face_wts[g] = w[g];
        } else {
            me.face_pts[2 * g] = p[g % q];
            me.face_pts[2 * g + 1] = p[g / q];
            me.face_wts[g] = w[g % q] * w[g / q];
        }
    }

    // Element basis: i = a + n1*(b + n1*c), product of 1D Lagrange polynomials.
    std::vector<double> l[3], dl[3];
    for (int d = 0; d < 3; ++d) { l[d].assign(n1, 1.0); dl[d].assign(n1, 0.0); }
    auto tabulate_point = [&](const double* xi, double* val, double* d0, double* d1, double* d2) {
        for (int d = 0; d < D; ++d) {
            lagrange_values(me.nodes1d, xi[d], l[d].data());
            if (d0) lagrange_derivs(me.nodes1d, xi[d], dl[d].data());
        }
        for (int i = 0; i < me.pe; ++i) {
            const int a = i % n1, b = (i / n1) % n1, c = i / (n1 * n1);
            if (D == 2) {
                val[i] = l[0][a] * l[1][b];
                if (d0) { d0[i] = dl[0][a] * l[1][b]; d1[i] = l[0][a] * dl[1][b]; }
            } else {
                val[i] = l[0][a] * l[1][b] * l[2][c];
                if (d0) {
                    d0[i] = dl[0][a] * l[1][b] * l[2][c];
                    d1[i] = l[0][a] * dl[1][b] * l[2][c];
                    d2[i] = l[0][a] * l[1][b] * dl[2][c];
                }
            }
        }
    };
    me.phi.resize(static_cast<size_t>(me.pe) * me.qe);
    for (int d = 0; d < D; ++d) me.dphi[d].resize(me.phi.size());
    for (int g = 0; g < me.qe; ++g) {
        const size_t o = static_cast<size_t>(me.pe) * g;
        tabulate_point(&me.elem_pts[static_cast<size_t>(g) * D], &me.phi[o], &me.dphi[0][o], &me.dphi[1][o],
                       D == 3 ? &me.dphi[2][o] : nullptr);
    }

    // Face basis: l = a (2D) or a + n1*b (3D) on the canonical face parameterisation.
    me.psi.resize(static_cast<size_t>(me.pf) * me.qf);
    {
        std::vector<double> ls(n1), lt(n1, 1.0);
        for (int g = 0; g < me.qf; ++g) {
            lagrange_values(me.nodes1d, me.face_pts[g * (D - 1)], ls.data());
            if (D == 3) lagrange_values(me.nodes1d, me.face_pts[2 * g + 1], lt.data());
            for (int j = 0; j < me.pf; ++j)
                me.psi[static_cast<size_t>(j) + static_cast<size_t>(me.pf) * g] =
                    (D == 2) ? ls[j] : ls[j % n1] * lt[j / n1];
        }
    }

    // Element basis on each local face, in the element-local face parameterisation.
    me.tphi_local.resize(static_cast<size_t>(me.n_lfe) * me.qf * me.pe);
    for (int lf = 0; lf < me.n_lfe; ++lf) {
        for (int g = 0; g < me.qf; ++g) {
            double xi[3];
            const double s = me.face_pts[g * (D - 1)];
            const double t = (D == 3) ? me.face_pts[2 * g + 1] : 0.0;
            face_point(shape, lf, s, t, xi);
            tabulate_point(xi, &me.tphi_local[(static_cast<size_t>(lf) * me.qf + g) * me.pe], nullptr, nullptr, nullptr);
        }
    }

    // Orientation tables: permutation of the face quadrature points.  The 1D rule is symmetric
    // index-wise (p[q-1-i] = 1 - p[i]), so every symmetry of the face maps quadrature points to
    // quadrature points; tables are permuted copies (the reference does the same index reversal in
    // 2D, local_ops.cpp:137-145).
    me.qperm.resize(static_cast<size_t>(me.n_orient) * me.qf);
    for (int o = 0; o < me.n_orient; ++o) {
        for (int gc = 0; gc < me.qf; ++gc) {
            int gl;
            if (D == 2) {
                gl = (o == 0) ? gc : me.qf - 1 - gc;
            } else {
                // index-space affine map with T(corner j) = corner local_corner(o, j)
                const int gs = gc % q, gt = gc / q;
                const int c0 = local_corner(o, 0), c1 = local_corner(o, 1), c3 = local_corner(o, 3);
                const int s0 = kCornerS[c0] * (q - 1), t0 = kCornerT[c0] * (q - 1);
                const int ls = s0 + gs * (kCornerS[c1] - kCornerS[c0]) + gt * (kCornerS[c3] - kCornerS[c0]);
                const int lt = t0 + gs * (kCornerT[c1] - kCornerT[c0]) + gt * (kCornerT[c3] - kCornerT[c0]);
                gl = lt * q + ls;
            }
            me.qperm[static_cast<size_t>(o) * me.qf + gc] = gl;
        }
    }
    me.tphi.resize(static_cast<size_t>(me.n_lfe) * me.n_orient * me.qf * me.pe);
    for (int lf = 0; lf < me.n_lfe; ++lf)
        for (int o = 0; o < me.n_orient; ++o)
            for (int gc = 0; gc < me.qf; ++gc) {
                const int gl = me.qperm[static_cast<size_t>(o) * me.qf + gc];
                const double* src = &me.tphi_local[(static_cast<size_t>(lf) * me.qf + gl) * me.pe];
                double* dst = &me.tphi[((static_cast<size_t>(lf) * me.n_orient + o) * me.qf + gc) * me.pe];
                std::copy(src, src + me.pe, dst);
            }
    me.elem_nodes.resize(static_cast<size_t>(me.pe) * D);
    for (int i = 0; i < me.pe; ++i) {
        const int idx[3] = {i % n1, (i / n1) % n1, i / (n1 * n1)};
        for (int d = 0; d < D; ++d) me.elem_nodes[static_cast<size_t>(i) * D + d] = me.nodes1d[idx[d]];
    }
    me.face_nodes.resize(static_cast<size_t>(me.pf) * (D - 1));
    for (int j = 0; j < me.pf; ++j) {
        me.face_nodes[static_cast<size_t>(j) * (D - 1)] = me.nodes1d[j % n1];
        if (D == 3) me.face_nodes[2 * j + 1] = me.nodes1d[j / n1];
    }
    return me;
}

// ---- meshes ------------------------------------------------------------------------------------
namespace {

void derive_elem_side(HostMesh& m) {
    m.elem_side.assign(static_cast<size_t>(m.ne) * m.n_lfe, 0);
    for (int e = 0; e < m.ne; ++e)
        for (int lf = 0; lf < m.n_lfe; ++lf) {
            const int f = m.elem_faces[static_cast<size_t>(e) * m.n_lfe + lf];
            // local_ops.cpp:129-132
            m.elem_side[static_cast<size_t>(e) * m.n_lfe + lf] =
                (m.face_elems[2 * f] == e && m.face_lidx[2 * f] == lf) ? 0 : 1;
        }
}

// Relative orientation of an element's local face with respect to the canonical vertex order.
int orientation_of(const ShapeInfo& si, const int* local_verts, const int* canon) {
    if (si.dim == 2) return local_verts[0] == canon[0] ? 0 : 1;
    const int nv = si.vpf;
    for (int r = 0; r < nv; ++r) {
        if (local_verts[r] != canon[0]) continue;
        if (local_verts[(r + 1) % nv] == canon[1]) return r;
        if (local_verts[(r + nv - 1) % nv] == canon[1]) return r + nv;
    }
    throw Failure(HDGB_ERR_INVALID_MESH, "face vertex lists of adjacent elements do not match");
}

void apply_jitter(HostMesh& m, int n, const double* lo, const double* hi, double jitter, uint64_t seed,
                  const std::vector<int>& lattice /* nv x dim lattice indices */) {
    if (!(jitter > 0.0)) return;
    std::mt19937_64 rng(seed);
    const int D = m.dim;
    for (int v = 0; v < m.nv; ++v) {
        bool interior = true;
        for (int d = 0; d < D; ++d) interior = interior && lattice[v * D + d] > 0 && lattice[v * D + d] < n;
        for (int d = 0; d < D; ++d) {
            // draw for every vertex so the sequence does not depend on the boundary set
            const double r = 2.0 * (static_cast<double>(rng() >> 11) * 0x1p-53) - 1.0;
            if (interior) m.coords[v * D + d] += jitter * ((hi[d] - lo[d]) / n) * r;
        }
    }
}

}  // namespace

HostMesh build_mesh_from_elements(int shape, int ne, int nv, const int32_t* elem_verts, const double* coords) {
    const ShapeInfo& si = shape_info(shape);
    HostMesh m;
    m.shape = shape;
    m.dim = si.dim;
    m.ne = ne;
    m.nv = nv;
    m.n_lfe = si.n_lfe;
    m.vpe = si.vpe;
    m.vpf = si.vpf;
    m.elem_verts.assign(elem_verts, elem_verts + static_cast<size_t>(ne) * si.vpe);
    m.coords.assign(coords, coords + static_cast<size_t>(nv) * si.dim);
    m.elem_faces.assign(static_cast<size_t>(ne) * si.n_lfe, -1);
    std::map<std::array<int, 4>, int> lookup;
    for (int e = 0; e < ne; ++e) {
        for (int lf = 0; lf < si.n_lfe; ++lf) {
            int lv[4] = {-1, -1, -1, -1};
            for (int k = 0; k < si.vpf; ++k) lv[k] = m.elem_verts[static_cast<size_t>(e) * si.vpe + si.face_verts[lf][k]];
            std::array<int, 4> key = {lv[0], lv[1], lv[2], lv[3]};
            std::sort(key.begin(), key.begin() + si.vpf);
            auto it = lookup.find(key);
            if (it == lookup.end()) {
                const int f = m.nf++;
                lookup.emplace(key, f);
                m.face_elems.push_back(e);
                m.face_elems.push_back(-1);
                m.face_lidx.push_back(lf);
                m.face_lidx.push_back(-1);
                m.face_orient.push_back(0);
                m.face_orient.push_back(0);
                for (int k = 0; k < si.vpf; ++k) m.face_verts.push_back(lv[k]);
                m.elem_faces[static_cast<size_t>(e) * si.n_lfe + lf] = f;
            } else {
                const int f = it->second;
                if (m.face_elems[2 * f + 1] != -1)
                    throw Failure(HDGB_ERR_INVALID_MESH, "face shared by more than two elements");
                m.face_elems[2 * f + 1] = e;
                m.face_lidx[2 * f + 1] = lf;
                m.face_orient[2 * f + 1] = orientation_of(si, lv, &m.face_verts[static_cast<size_t>(f) * si.vpf]);
                m.elem_faces[static_cast<size_t>(e) * si.n_lfe + lf] = f;
            }
        }
    }
    m.bnd_tag.assign(m.nf, 0);
    for (int f = 0; f < m.nf; ++f)
        if (m.face_elems[2 * f + 1] < 0) m.bnd_tag[f] = 1;
    derive_elem_side(m);
    return m;
}

HostMesh mesh_from_tables(int shape, int ne, int nf, int nv, const int32_t* elem_verts, const double* coords,
                          const int32_t* elem_faces, const int32_t* face_elems, const int32_t* face_lidx,
                          const int32_t* face_orient, const int32_t* face_verts, const int32_t* bnd_tag) {
    const ShapeInfo& si = shape_info(shape);
    HostMesh m;
    m.shape = shape; m.dim = si.dim; m.ne = ne; m.nf = nf; m.nv = nv;
    m.n_lfe = si.n_lfe; m.vpe = si.vpe; m.vpf = si.vpf;
    m.elem_verts.assign(elem_verts, elem_verts + static_cast<size_t>(ne) * si.vpe);
    m.coords.assign(coords, coords + static_cast<size_t>(nv) * si.dim);
    m.elem_faces.assign(elem_faces, elem_faces + static_cast<size_t>(ne) * si.n_lfe);
    m.face_elems.assign(face_elems, face_elems + static_cast<size_t>(nf) * 2);
    m.face_lidx.assign(face_lidx, face_lidx + static_cast<size_t>(nf) * 2);
    m.face_orient.assign(face_orient, face_orient + static_cast<size_t>(nf) * 2);
    m.face_verts.assign(face_verts, face_verts + static_cast<size_t>(nf) * si.vpf);
    m.bnd_tag.assign(bnd_tag, bnd_tag + nf);
    for (int e = 0; e < ne; ++e)
        for (int lf = 0; lf < si.n_lfe; ++lf) {
            const int f = m.elem_faces[static_cast<size_t>(e) * si.n_lfe + lf];
            if (f < 0 || f >= nf) throw Failure(HDGB_ERR_INVALID_MESH, "element_to_face entry out of range", e);
            const bool s0 = m.face_elems[2 * f] == e && m.face_lidx[2 * f] == lf;
            const bool s1 = m.face_elems[2 * f + 1] == e && m.face_lidx[2 * f + 1] == lf;
            if (!s0 && !s1) throw Failure(HDGB_ERR_INVALID_MESH, "face_to_elements does not list the element on either side", e);
        }
    derive_elem_side(m);
    return m;
}

HostMesh build_structured_mesh(int shape, int n, const double* lo, const double* hi, double jitter, uint64_t seed) {
    if (n < 1) throw Failure(HDGB_ERR_INVALID_MESH, "mesh resolution must be >= 1, got " + std::to_string(n));
    const ShapeInfo& si = shape_info(shape);
    const int D = si.dim;
    for (int d = 0; d < D; ++d)
        if (!(hi[d] > lo[d])) throw Failure(HDGB_ERR_INVALID_MESH, "degenerate domain: need hi > lo in every direction");
    const int nv1 = n + 1;

    if (shape == HDGB_QUAD) {
        // Numbering of mesh.cpp:18-107: elements row-major, horizontal faces first (by row),
        // then vertical faces (by column); side 0 = the lower / left element.
        HostMesh m;
        m.shape = shape; m.dim = 2; m.n_lfe = 4; m.vpe = 4; m.vpf = 2;
        m.ne = n * n;
        m.nf = 2 * n * (n + 1);
        m.nv = nv1 * nv1;
        const double hx = (hi[0] - lo[0]) / n, hy = (hi[1] - lo[1]) / n;
        m.coords.resize(static_cast<size_t>(m.nv) * 2);
        std::vector<int> lattice(static_cast<size_t>(m.nv) * 2);
        for (int j = 0; j < nv1; ++j)
            for (int i = 0; i < nv1; ++i) {
                const int v = j * nv1 + i;
                m.coords[2 * v] = lo[0] + i * hx;
                m.coords[2 * v + 1] = lo[1] + j * hy;
                lattice[2 * v] = i;
                lattice[2 * v + 1] = j;
            }
        auto vertex = [nv1](int i, int j) { return j * nv1 + i; };
        auto horizontal = [n](int i, int j) { return j * n + i; };
        auto vertical = [n](int i, int j) { return n * (n + 1) + i * n + j; };
        m.elem_verts.resize(static_cast<size_t>(m.ne) * 4);
        m.elem_faces.resize(static_cast<size_t>(m.ne) * 4);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                const int e = j * n + i;
                const int ev[4] = {vertex(i, j), vertex(i + 1, j), vertex(i + 1, j + 1), vertex(i, j + 1)};
                const int ef[4] = {horizontal(i, j), vertical(i + 1, j), horizontal(i, j + 1), vertical(i, j)};
                std::copy(ev, ev + 4, &m.elem_verts[4 * e]);
                std::copy(ef, ef + 4, &m.elem_faces[4 * e]);
            }
        m.face_elems.assign(static_cast<size_t>(m.nf) * 2, -1);
        m.face_lidx.assign(static_cast<size_t>(m.nf) * 2, -1);
        m.face_orient.assign(static_cast<size_t>(m.nf) * 2, 0);
        m.face_verts.resize(static_cast<size_t>(m.nf) * 2);
        m.bnd_tag.assign(m.nf, 0);
        auto attach = [&](int f, int e, int lf) {
            const int side = (m.face_elems[2 * f] == -1) ? 0 : 1;
            m.face_elems[2 * f + side] = e;
            m.face_lidx[2 * f + side] = lf;
        };
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i < n; ++i) {
                const int f = horizontal(i, j);
                m.face_verts[2 * f] = vertex(i, j);
                m.face_verts[2 * f + 1] = vertex(i + 1, j);
                if (j > 0) attach(f, (j - 1) * n + i, 2);  // element below sees its top face
                if (j < n) attach(f, j * n + i, 0);        // element above sees its bottom face
                if (j == 0) m.bnd_tag[f] = 1;
                if (j == n) m.bnd_tag[f] = 3;
            }
        for (int i = 0; i <= n; ++i)
            for (int j = 0; j < n; ++j) {
                const int f = vertical(i, j);
                m.face_verts[2 * f] = vertex(i, j);
                m.face_verts[2 * f + 1] = vertex(i, j + 1);
                if (i > 0) attach(f, j * n + (i - 1), 1);  // element to the left: its right face
                if (i < n) attach(f, j * n + i, 3);        // element to the right: its left face
                if (i == 0) m.bnd_tag[f] = 4;
                if (i == n) m.bnd_tag[f] = 2;
            }
        for (int f = 0; f < m.nf; ++f)
            for (int s = 0; s < 2; ++s) {
                const int e = m.face_elems[2 * f + s];
                if (e < 0) continue;
                const int lf = m.face_lidx[2 * f + s];
                const int lv[2] = {m.elem_verts[4 * e + si.face_verts[lf][0]], m.elem_verts[4 * e + si.face_verts[lf][1]]};
                m.face_orient[2 * f + s] = orientation_of(si, lv, &m.face_verts[2 * f]);
            }
        apply_jitter(m, n, lo, hi, jitter, seed, lattice);
        derive_elem_side(m);
        return m;
    }

    if (shape == HDGB_HEX) {
        const int nv = nv1 * nv1 * nv1;
        std::vector<double> coords(static_cast<size_t>(nv) * 3);
        std::vector<int> lattice(static_cast<size_t>(nv) * 3);
        double h[3];
        for (int d = 0; d < 3; ++d) h[d] = (hi[d] - lo[d]) / n;
        auto vertex = [nv1](int i, int j, int k) { return (k * nv1 + j) * nv1 + i; };
        for (int k = 0; k < nv1; ++k)
            for (int j = 0; j < nv1; ++j)
                for (int i = 0; i < nv1; ++i) {
                    const int v = vertex(i, j, k);
                    const int ijk[3] = {i, j, k};
                    for (int d = 0; d < 3; ++d) {
                        coords[3 * v + d] = lo[d] + ijk[d] * h[d];
                        lattice[3 * v + d] = ijk[d];
                    }
                }
        std::vector<int32_t> ev(static_cast<size_t>(n) * n * n * 8);
        for (int k = 0; k < n; ++k)
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    const int e = (k * n + j) * n + i;
                    const int v8[8] = {vertex(i, j, k),         vertex(i + 1, j, k),     vertex(i + 1, j + 1, k),     vertex(i, j + 1, k),
                                       vertex(i, j, k + 1),     vertex(i + 1, j, k + 1), vertex(i + 1, j + 1, k + 1), vertex(i, j + 1, k + 1)};
                    std::copy(v8, v8 + 8, &ev[8 * static_cast<size_t>(e)]);
                }
        HostMesh m = build_mesh_from_elements(shape, n * n * n, nv, ev.data(), coords.data());
        // Boundary tags extend the 2D convention: 1 = y-lo, 2 = x-hi, 3 = y-hi, 4 = x-lo,
        // 5 = z-lo, 6 = z-hi.
        for (int f = 0; f < m.nf; ++f) {
            if (m.face_elems[2 * f + 1] >= 0) continue;
            int mn[3] = {n, n, n}, mx[3] = {0, 0, 0};
            for (int k = 0; k < 4; ++k) {
                const int v = m.face_verts[4 * f + k];
                for (int d = 0; d < 3; ++d) {
                    mn[d] = std::min(mn[d], lattice[3 * v + d]);
                    mx[d] = std::max(mx[d], lattice[3 * v + d]);
                }
            }
            int tag = 1;
            if (mx[1] == 0) tag = 1;
            else if (mn[0] == n) tag = 2;
            else if (mn[1] == n) tag = 3;
            else if (mx[0] == 0) tag = 4;
            else if (mx[2] == 0) tag = 5;
            else if (mn[2] == n) tag = 6;
            m.bnd_tag[f] = tag;
        }
        apply_jitter(m, n, lo, hi, jitter, seed, lattice);
        return m;
    }
    if (shape == HDGB_TRI || shape == HDGB_TET) {
        // TRI: every cell of the n x n grid is cut along its (v00, v11) diagonal into two CCW
        // triangles.  TET: every cube is cut into the 6 Kuhn tetrahedra (one per monotone lattice
        // path (0,0,0) -> (1,1,1)); the same pattern in every cube is conforming.
        const int nv = (D == 2) ? nv1 * nv1 : nv1 * nv1 * nv1;
        std::vector<double> coords(static_cast<size_t>(nv) * D);
        std::vector<int> lattice(static_cast<size_t>(nv) * D);
        double h[3] = {0, 0, 0};
        for (int d = 0; d < D; ++d) h[d] = (hi[d] - lo[d]) / n;
        auto vertex = [nv1](int i, int j, int k) { return (k * nv1 + j) * nv1 + i; };
        for (int k = 0; k < (D == 3 ? nv1 : 1); ++k)
            for (int j = 0; j < nv1; ++j)
                for (int i = 0; i < nv1; ++i) {
                    const int v = vertex(i, j, k);
                    const int ijk[3] = {i, j, k};
                    for (int d = 0; d < D; ++d) {
                        coords[static_cast<size_t>(v) * D + d] = lo[d] + ijk[d] * h[d];
                        lattice[static_cast<size_t>(v) * D + d] = ijk[d];
                    }
                }
        std::vector<int32_t> ev;
        if (D == 2) {
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    const int v00 = vertex(i, j, 0), v10 = vertex(i + 1, j, 0), v11 = vertex(i + 1, j + 1, 0), v01 = vertex(i, j + 1, 0);
                    const int t[6] = {v00, v10, v11, v00, v11, v01};
                    ev.insert(ev.end(), t, t + 6);
                }
        } else {
            static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
            static const int sign[6] = {+1, -1, -1, +1, +1, -1};
            for (int k = 0; k < n; ++k)
                for (int j = 0; j < n; ++j)
                    for (int i = 0; i < n; ++i)
                        for (int pp = 0; pp < 6; ++pp) {
                            int c[3] = {i, j, k};
                            int t[4];
                            t[0] = vertex(c[0], c[1], c[2]);
                            for (int s2 = 0; s2 < 3; ++s2) {
                                c[perms[pp][s2]] += 1;
                                t[s2 + 1] = vertex(c[0], c[1], c[2]);
                            }
                            if (sign[pp] < 0) std::swap(t[1], t[2]);  // keep the tetrahedron positively oriented
                            ev.insert(ev.end(), t, t + 4);
                        }
        }
        const int ne = static_cast<int>(ev.size()) / si.vpe;
        HostMesh m = build_mesh_from_elements(shape, ne, nv, ev.data(), coords.data());
        for (int f = 0; f < m.nf; ++f) {
            if (m.face_elems[2 * f + 1] >= 0) continue;
            int mn[3] = {n, n, n}, mx[3] = {0, 0, 0};
            for (int k = 0; k < si.vpf; ++k) {
                const int v = m.face_verts[static_cast<size_t>(f) * si.vpf + k];
                for (int d = 0; d < D; ++d) {
                    mn[d] = std::min(mn[d], lattice[static_cast<size_t>(v) * D + d]);
                    mx[d] = std::max(mx[d], lattice[static_cast<size_t>(v) * D + d]);
                }
            }
            int tag = 1;
            if (mx[1] == 0) tag = 1;
            else if (mn[0] == n) tag = 2;
            else if (mn[1] == n) tag = 3;
            else if (mx[0] == 0) tag = 4;
            else if (D == 3 && mx[2] == 0) tag = 5;
            else if (D == 3 && mn[2] == n) tag = 6;
            m.bnd_tag[f] = tag;
        }
        apply_jitter(m, n, lo, hi, jitter, seed, lattice);
        return m;
    }
    throw Failure(HDGB_ERR_UNSUPPORTED, "structured builder: unknown shape");
}

// ---- geometry ----------------------------------------------------------------------------------
HostGeom compute_geometry(const HostMesh& mesh, const MasterElement& me) {
    HostGeom g;
    const int D = mesh.dim, qe = me.qe, qf = me.qf;
    const ShapeInfo& si = shape_info(mesh.shape);
    g.elem_detjac.resize(static_cast<size_t>(mesh.ne) * qe);
    g.elem_invjac.resize(static_cast<size_t>(mesh.ne) * qe * D * D);
    g.elem_coords.resize(static_cast<size_t>(mesh.ne) * qe * D);
    g.face_detjac.resize(static_cast<size_t>(mesh.nf) * qf);
    g.face_coords.resize(static_cast<size_t>(mesh.nf) * qf * D);
    g.face_normal.assign(static_cast<size_t>(mesh.nf) * 2 * qf * D, 0.0);

    if (mesh.shape == HDGB_QUAD) {
        // Bilinear map; same expressions as mesh.cpp:120-146.
        for (int e = 0; e < mesh.ne; ++e) {
            double vx[4], vy[4];
            for (int c = 0; c < 4; ++c) {
                const int v = mesh.elem_verts[4 * e + c];
                vx[c] = mesh.coords[2 * v];
                vy[c] = mesh.coords[2 * v + 1];
            }
            for (int q = 0; q < qe; ++q) {
                const double xi = me.elem_pts[2 * q], eta = me.elem_pts[2 * q + 1];
                const double n0 = (1 - xi) * (1 - eta), n1 = xi * (1 - eta), n2 = xi * eta, n3 = (1 - xi) * eta;
                const size_t idx = static_cast<size_t>(e) * qe + q;
                g.elem_coords[idx * 2 + 0] = n0 * vx[0] + n1 * vx[1] + n2 * vx[2] + n3 * vx[3];
                g.elem_coords[idx * 2 + 1] = n0 * vy[0] + n1 * vy[1] + n2 * vy[2] + n3 * vy[3];
                const double x_xi = (vx[1] - vx[0]) * (1 - eta) + (vx[2] - vx[3]) * eta;
                const double y_xi = (vy[1] - vy[0]) * (1 - eta) + (vy[2] - vy[3]) * eta;
                const double x_eta = (vx[3] - vx[0]) * (1 - xi) + (vx[2] - vx[1]) * xi;
                const double y_eta = (vy[3] - vy[0]) * (1 - xi) + (vy[2] - vy[1]) * xi;
                const double det = x_xi * y_eta - x_eta * y_xi;
                if (!(det > 0.0))
                    throw Failure(HDGB_ERR_INVALID_MESH, "non-positive Jacobian determinant in element " + std::to_string(e), e);
                g.elem_detjac[idx] = det;
                const double inv = 1.0 / det;
                g.elem_invjac[idx * 4 + 0] = y_eta * inv;
                g.elem_invjac[idx * 4 + 1] = -x_eta * inv;
                g.elem_invjac[idx * 4 + 2] = -y_xi * inv;
                g.elem_invjac[idx * 4 + 3] = x_xi * inv;
            }
        }
        for (int f = 0; f < mesh.nf; ++f) {
            const int va = mesh.face_verts[2 * f], vb = mesh.face_verts[2 * f + 1];
            const double ax = mesh.coords[2 * va], ay = mesh.coords[2 * va + 1];
            const double tx = mesh.coords[2 * vb] - ax, ty = mesh.coords[2 * vb + 1] - ay;
            const double len = std::hypot(tx, ty);
            for (int q = 0; q < qf; ++q) {
                const double t = me.face_pts[q];
                const size_t idx = static_cast<size_t>(f) * qf + q;
                g.face_detjac[idx] = len;
                g.face_coords[idx * 2 + 0] = ax + t * tx;
                g.face_coords[idx * 2 + 1] = ay + t * ty;
            }
            for (int s = 0; s < 2; ++s) {
                const int e = mesh.face_elems[2 * f + s];
                if (e < 0) continue;
                const int lf = mesh.face_lidx[2 * f + s];
                const double sign = mesh.face_orient[2 * f + s] ? -1.0 : 1.0;
                const double ex = sign * tx / len, ey = sign * ty / len;
                double nx, ny;
                if (si.outward_sign[lf] > 0) { nx = ey; ny = -ex; } else { nx = -ey; ny = ex; }
                for (int q = 0; q < qf; ++q) {
                    const size_t idx = (static_cast<size_t>(f) * 2 + s) * qf + q;
                    g.face_normal[idx * 2 + 0] = nx;
                    g.face_normal[idx * 2 + 1] = ny;
                }
            }
        }
        return g;
    }

    if (mesh.shape == HDGB_HEX) {
        static const int cs[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
        for (int e = 0; e < mesh.ne; ++e) {
            double v[8][3];
            for (int c = 0; c < 8; ++c)
                for (int d = 0; d < 3; ++d) v[c][d] = mesh.coords[3 * static_cast<size_t>(mesh.elem_verts[8 * static_cast<size_t>(e) + c]) + d];
            for (int q = 0; q < qe; ++q) {
                const double* xi = &me.elem_pts[3 * static_cast<size_t>(q)];
                double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // J[c][r] = d x_c / d xi_r
                double x[3] = {0, 0, 0};
                for (int c = 0; c < 8; ++c) {
                    double f1[3], df[3];
                    for (int d = 0; d < 3; ++d) {
                        f1[d] = cs[c][d] ? xi[d] : 1.0 - xi[d];
                        df[d] = cs[c][d] ? 1.0 : -1.0;
                    }
                    const double N = f1[0] * f1[1] * f1[2];
                    const double dN[3] = {df[0] * f1[1] * f1[2], f1[0] * df[1] * f1[2], f1[0] * f1[1] * df[2]};
                    for (int d = 0; d < 3; ++d) {
                        x[d] += N * v[c][d];
                        for (int r = 0; r < 3; ++r) J[d][r] += dN[r] * v[c][d];
                    }
                }
                const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
                const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
                const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
                const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
                if (!(det > 0.0))
                    throw Failure(HDGB_ERR_INVALID_MESH, "non-positive Jacobian determinant in element " + std::to_string(e), e);
                const size_t idx = static_cast<size_t>(e) * qe + q;
                g.elem_detjac[idx] = det;
                for (int d = 0; d < 3; ++d) g.elem_coords[idx * 3 + d] = x[d];
                const double inv = 1.0 / det;
                double* ij = &g.elem_invjac[idx * 9];  // ij[r*3 + c] = (J^-1)[r][c]
                ij[0] = c00 * inv;
                ij[1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * inv;
                ij[2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * inv;
                ij[3] = c01 * inv;
                ij[4] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * inv;
                ij[5] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * inv;
                ij[6] = c02 * inv;
                ij[7] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * inv;
                ij[8] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * inv;
            }
        }
        for (int f = 0; f < mesh.nf; ++f) {
            double c[4][3];
            for (int k = 0; k < 4; ++k)
                for (int d = 0; d < 3; ++d) c[k][d] = mesh.coords[3 * static_cast<size_t>(mesh.face_verts[4 * static_cast<size_t>(f) + k]) + d];
            for (int q = 0; q < qf; ++q) {
                const double s = me.face_pts[2 * q], t = me.face_pts[2 * q + 1];
                double xs[3], xt[3], x[3];
                for (int d = 0; d < 3; ++d) {
                    x[d] = (1 - s) * (1 - t) * c[0][d] + s * (1 - t) * c[1][d] + s * t * c[2][d] + (1 - s) * t * c[3][d];
                    xs[d] = (c[1][d] - c[0][d]) * (1 - t) + (c[2][d] - c[3][d]) * t;
                    xt[d] = (c[3][d] - c[0][d]) * (1 - s) + (c[2][d] - c[1][d]) * s;
                }
                const double cr[3] = {xs[1] * xt[2] - xs[2] * xt[1], xs[2] * xt[0] - xs[0] * xt[2], xs[0] * xt[1] - xs[1] * xt[0]};
                const double area = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
                const size_t idx = static_cast<size_t>(f) * qf + q;
                g.face_detjac[idx] = area;
                for (int d = 0; d < 3; ++d) g.face_coords[idx * 3 + d] = x[d];
                for (int sd = 0; sd < 2; ++sd) {
                    const int e = mesh.face_elems[2 * f + sd];
                    if (e < 0) continue;
                    const int lf = mesh.face_lidx[2 * f + sd];
                    const int o = mesh.face_orient[2 * f + sd];
                    // the side-local parameterisation has the canonical winding for rotations and the
                    // opposite one for flips
                    const double sign = static_cast<double>(si.outward_sign[lf]) * (o < 4 ? 1.0 : -1.0);
                    const size_t ni = (static_cast<size_t>(f) * 2 + sd) * qf + q;
                    for (int d = 0; d < 3; ++d) g.face_normal[ni * 3 + d] = sign * cr[d] / area;
                }
            }
        }
        return g;
    }
    if (mesh.shape == HDGB_TRI || mesh.shape == HDGB_TET) {
        // affine elements: constant Jacobian
        const int vpe = si.vpe, vpf = si.vpf;
        for (int e = 0; e < mesh.ne; ++e) {
            double v[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
            for (int c = 0; c < vpe; ++c)
                for (int d = 0; d < D; ++d) v[c][d] = mesh.coords[static_cast<size_t>(mesh.elem_verts[static_cast<size_t>(e) * vpe + c]) * D + d];
            double J[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};  // J[c][r] = d x_c / d xi_r
            for (int c = 0; c < D; ++c)
                for (int r = 0; r < D; ++r) J[c][r] = v[r + 1][c] - v[0][c];
            double det, inv[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
            if (D == 2) {
                det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
                if (det > 0.0) {
                    inv[0][0] = J[1][1] / det; inv[0][1] = -J[0][1] / det;
                    inv[1][0] = -J[1][0] / det; inv[1][1] = J[0][0] / det;
                }
            } else {
                const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
                const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
                const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
                det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
                if (det > 0.0) {
                    const double id = 1.0 / det;
                    inv[0][0] = c00 * id;
                    inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
                    inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
                    inv[1][0] = c01 * id;
                    inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
                    inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
                    inv[2][0] = c02 * id;
                    inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
                    inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
                }
            }
            if (!(det > 0.0))
                throw Failure(HDGB_ERR_INVALID_MESH, "non-positive Jacobian determinant in element " + std::to_string(e), e);
            for (int q = 0; q < qe; ++q) {
                const size_t idx = static_cast<size_t>(e) * qe + q;
                g.elem_detjac[idx] = det;
                for (int r = 0; r < D; ++r)
                    for (int c = 0; c < D; ++c) g.elem_invjac[idx * D * D + r * D + c] = inv[r][c];  // d xi_r / d x_c
                for (int c = 0; c < D; ++c) {
                    double x = v[0][c];
                    for (int r = 0; r < D; ++r) x += J[c][r] * me.elem_pts[static_cast<size_t>(q) * D + r];
                    g.elem_coords[idx * D + c] = x;
                }
            }
        }
        for (int f = 0; f < mesh.nf; ++f) {
            double c[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
            for (int k = 0; k < vpf; ++k)
                for (int d = 0; d < D; ++d) c[k][d] = mesh.coords[static_cast<size_t>(mesh.face_verts[static_cast<size_t>(f) * vpf + k]) * D + d];
            double nrm[3] = {0, 0, 0}, meas;
            if (D == 2) {
                const double tx = c[1][0] - c[0][0], ty = c[1][1] - c[0][1];
                meas = std::hypot(tx, ty);
                nrm[0] = ty / meas;   // canonical tangent rotated by -90 degrees
                nrm[1] = -tx / meas;
            } else {
                double ab[3], ac[3];
                for (int d = 0; d < 3; ++d) { ab[d] = c[1][d] - c[0][d]; ac[d] = c[2][d] - c[0][d]; }
                const double cr[3] = {ab[1] * ac[2] - ab[2] * ac[1], ab[2] * ac[0] - ab[0] * ac[2], ab[0] * ac[1] - ab[1] * ac[0]};
                meas = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
                for (int d = 0; d < 3; ++d) nrm[d] = cr[d] / meas;
            }
            for (int q = 0; q < qf; ++q) {
                const size_t idx = static_cast<size_t>(f) * qf + q;
                g.face_detjac[idx] = meas;  // reference edge length 1 / reference triangle area 1/2 (weights sum to 1/2)
                const double s = me.face_pts[static_cast<size_t>(q) * (D - 1)];
                const double t = (D == 3) ? me.face_pts[2 * q + 1] : 0.0;
                for (int d = 0; d < D; ++d)
                    g.face_coords[idx * D + d] = c[0][d] + s * (c[1][d] - c[0][d]) + (D == 3 ? t * (c[2][d] - c[0][d]) : 0.0);
            }
            for (int sd = 0; sd < 2; ++sd) {
                const int e = mesh.face_elems[2 * f + sd];
                if (e < 0) continue;
                const int lf = mesh.face_lidx[2 * f + sd];
                const int o = mesh.face_orient[2 * f + sd];
                // same winding as the canonical listing for rotations, opposite for flips
                const double flip = (D == 2) ? (o == 0 ? 1.0 : -1.0) : (o < 3 ? 1.0 : -1.0);
                const double sign = static_cast<double>(si.outward_sign[lf]) * flip;
                for (int q = 0; q < qf; ++q) {
                    const size_t ni = (static_cast<size_t>(f) * 2 + sd) * qf + q;
                    for (int d = 0; d < D; ++d) g.face_normal[ni * D + d] = sign * nrm[d];
                }
            }
        }
        return g;
    }
    throw Failure(HDGB_ERR_UNSUPPORTED, "compute_geometry: unknown shape");
}

}  // namespace hdgb
