"""Breaks the common mode between the product and the tier-B oracle: for 3D / multi-component cases the oracle is
fed the product's own setup tables (oracle/port.tables_from_disc), so a wrong table would be invisible to the
parity tests.  Here the hex and tet tables are REBUILT INDEPENDENTLY in numpy from first principles -- numpy's
Gauss-Legendre rule, Lobatto nodes as roots of P_k', Lagrange bases through a Vandermonde solve, tri-linear /
affine geometry from the vertex coordinates, and the oriented trace tables by inverting each element's geometry
map at the face's canonical quadrature points -- and compared entry-wise with Discretization.table(...).
(2D quads are compared bit for bit with the reference itself in tests/test_gpu_quad_parity.py.)"""
from math import factorial

import numpy as np
import pytest

import paper_2512_13619_b200 as hdg


def gauss01(q):
    x, w = np.polynomial.legendre.leggauss(q)
    return 0.5 * (x + 1.0), 0.5 * w


def lobatto01(k):
    if k == 1:
        return np.array([0.0, 1.0])
    c = np.zeros(k + 1)
    c[k] = 1.0
    inner = np.sort(np.polynomial.legendre.legroots(np.polynomial.legendre.legder(c)))
    return 0.5 * (np.concatenate([[-1.0], inner, [1.0]]) + 1.0)


def lagrange_1d(nodes, x):
    """values and derivatives of the 1D Lagrange basis at x (barycentric-free, O(n^2) products)."""
    n = len(nodes)
    val, der = np.ones((len(x), n)), np.zeros((len(x), n))
    for i in range(n):
        for j in range(n):
            if j != i:
                val[:, i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
        for m in range(n):
            if m == i:
                continue
            t = np.full(len(x), 1.0 / (nodes[i] - nodes[m]))
            for j in range(n):
                if j not in (i, m):
                    t *= (x - nodes[j]) / (nodes[i] - nodes[j])
            der[:, i] += t
    return val, der


def hex_basis(nodes, xi):
    """tensor Lagrange basis, index i = a + (k+1) b + (k+1)^2 c; returns phi (npts, pe), dphi (3, npts, pe)."""
    v, d = zip(*(lagrange_1d(nodes, xi[:, r]) for r in range(3)))
    ein = lambda A, B, C_: np.einsum("pc,pb,pa->pcba", C_, B, A).reshape(len(xi), -1)
    return ein(v[0], v[1], v[2]), np.stack([ein(d[0], v[1], v[2]), ein(v[0], d[1], v[2]), ein(v[0], v[1], d[2])])


HEX_CORNERS = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)], dtype=float)


def hex_geom(verts, xi):
    """tri-linear map of one element: X (npts, 3), J[p, c, r] = dX_c / dxi_r."""
    N = np.ones((len(xi), 8))
    dN = np.ones((3, len(xi), 8))
    for v, c in enumerate(HEX_CORNERS):
        for r in range(3):
            f = xi[:, r] if c[r] else 1.0 - xi[:, r]
            df = np.full(len(xi), 1.0 if c[r] else -1.0)
            N[:, v] *= f
            for s in range(3):
                dN[s, :, v] *= df if s == r else f
    return N @ verts, np.einsum("rpv,vc->pcr", dN, verts)


def tet_monomials(k):
    return [(a, b, c) for a in range(k + 1) for b in range(k + 1 - a) for c in range(k + 1 - a - b)]


def tet_basis(nodes, k, xi):
    mons = tet_monomials(k)
    V = np.stack([nodes[:, 0] ** a * nodes[:, 1] ** b * nodes[:, 2] ** c for a, b, c in mons], axis=1)  # (node, mon)
    coef = np.linalg.inv(V)                                                                            # (mon, basis)
    m = np.stack([xi[:, 0] ** a * xi[:, 1] ** b * xi[:, 2] ** c for a, b, c in mons], axis=1)

    def dmon(r):
        out = []
        for e in mons:
            if e[r] == 0:
                out.append(np.zeros(len(xi)))
            else:
                f = [e[0], e[1], e[2]]
                f[r] -= 1
                out.append(e[r] * xi[:, 0] ** f[0] * xi[:, 1] ** f[1] * xi[:, 2] ** f[2])
        return np.stack(out, axis=1)
    return m @ coef, np.stack([dmon(r) @ coef for r in range(3)])


def tables(d):
    D, qe, qf, pe, pf, ne, nf = d.dim, d.qe, d.qf, d.pe, d.pf, d.ne, d.nf
    t = dict(phi=d.table("phi").reshape(qe, pe), dphi=np.stack([d.table(f"dphi{r}").reshape(qe, pe) for r in range(D)]),
             psi=d.table("psi").reshape(qf, pf), tphi=d.table("tphi").reshape(d.n_lfe, d.n_orient, qf, pe),
             xq=d.table("elem_coords").reshape(ne, qe, D), det=d.table("elem_detjac").reshape(ne, qe),
             inv=d.table("elem_invjac").reshape(ne, qe, D, D), xf=d.table("face_coords").reshape(nf, qf, D),
             fdet=d.table("face_detjac").reshape(nf, qf), nrm=d.table("face_normal").reshape(nf, 2, qf, D),
             ev=d.table("element_vertices").reshape(ne, -1), vc=d.table("vertex_coords").reshape(-1, D),
             fv=d.table("face_vertices").reshape(nf, -1), fe=d.table("face_to_elements").reshape(nf, 2),
             fl=d.table("face_local_index").reshape(nf, 2), fo=d.table("face_orient").reshape(nf, 2),
             e2f=d.table("element_to_face").reshape(ne, -1), wq=d.table("elem_weights"), wf=d.table("face_weights"),
             xi=d.table("elem_points").reshape(qe, D), st=d.table("face_points").reshape(qf, D - 1),
             nodes=d.table("elem_nodes").reshape(pe, D), fnodes=d.table("face_nodes").reshape(pf, D - 1))
    return t


@pytest.mark.parametrize("k,n,jitter", [(1, 2, 0.2), (2, 2, 0.15), (3, 2, 0.15)])
def test_hex_tables_against_independent_numpy_construction(k, n, jitter):
    d = hdg.Discretization.structured(None, "hex", n=n, degree=k, jitter=jitter, seed=21)
    t = tables(d)
    q = k + 2                                                                   # study.cpp:70
    assert d.qe == q ** 3 and d.qf == q ** 2 and d.pe == (k + 1) ** 3 and d.pf == (k + 1) ** 2
    # quadrature: tensor Gauss-Legendre on [0,1], x fastest
    g1, w1 = gauss01(q)
    gz, gy, gx = np.meshgrid(g1, g1, g1, indexing="ij")
    xi = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    wq = np.einsum("c,b,a->cba", w1, w1, w1).ravel()
    assert np.allclose(t["xi"], xi, atol=1e-14) and np.allclose(t["wq"], wq, atol=1e-15)
    gt, gs = np.meshgrid(g1, g1, indexing="ij")
    st = np.stack([gs.ravel(), gt.ravel()], axis=1)
    assert np.allclose(t["st"], st, atol=1e-14) and np.allclose(t["wf"], np.outer(w1, w1).ravel(), atol=1e-15)
    # nodes: Gauss-Lobatto tensor grid, x fastest
    lob = lobatto01(k)
    nz, ny, nx = np.meshgrid(lob, lob, lob, indexing="ij")
    assert np.allclose(t["nodes"], np.stack([nx.ravel(), ny.ravel(), nz.ravel()], axis=1), atol=1e-14)
    # volume basis tables
    phi, dphi = hex_basis(lob, xi)
    assert np.max(np.abs(t["phi"] - phi)) < 1e-13 and np.max(np.abs(t["dphi"] - dphi)) < 1e-12
    # face basis: tensor Lagrange in the canonical face parameters
    vs, _ = lagrange_1d(lob, st[:, 0])
    vt, _ = lagrange_1d(lob, st[:, 1])
    assert np.max(np.abs(t["psi"] - np.einsum("pb,pa->pba", vt, vs).reshape(len(st), -1))) < 1e-13
    # element geometry from the vertex coordinates
    for e in range(d.ne):
        X, J = hex_geom(t["vc"][t["ev"][e]], xi)
        assert np.max(np.abs(t["xq"][e] - X)) < 1e-13
        assert np.max(np.abs(t["det"][e] - np.linalg.det(J))) < 1e-13
        assert np.max(np.abs(t["inv"][e] - np.linalg.inv(J))) < 1e-11        # inv[r, c] = d xi_r / d x_c
    # face geometry: bilinear map of the canonical corners; normals; oriented traces by inverting the element map
    cen = np.array([t["vc"][t["ev"][e]].mean(axis=0) for e in range(d.ne)])
    for f in range(d.nf):
        c = t["vc"][t["fv"][f]]                                                 # canonical corner order, CCW in (s, t)
        s_, t_ = st[:, 0:1], st[:, 1:2]
        X = (1 - s_) * (1 - t_) * c[0] + s_ * (1 - t_) * c[1] + s_ * t_ * c[2] + (1 - s_) * t_ * c[3]
        dXs = (1 - t_) * (c[1] - c[0]) + t_ * (c[2] - c[3])
        dXt = (1 - s_) * (c[3] - c[0]) + s_ * (c[2] - c[1])
        nvec = np.cross(dXs, dXt)
        area = np.linalg.norm(nvec, axis=1)
        assert np.max(np.abs(t["xf"][f] - X)) < 1e-13 and np.max(np.abs(t["fdet"][f] - area)) < 1e-13
        for s in range(2):
            e = t["fe"][f, s]
            if e < 0:
                continue
            unit = nvec / area[:, None]
            sign = np.sign(np.einsum("gd,gd->g", unit, X - cen[e]))
            assert np.max(np.abs(t["nrm"][f, s] - sign[:, None] * unit)) < 1e-13
            # invert the tri-linear map of element e at the canonical face points (Newton), evaluate its basis there
            verts = t["vc"][t["ev"][e]]
            xi_f = np.full((len(X), 3), 0.5)
            for _ in range(30):
                Xe, J = hex_geom(verts, xi_f)
                xi_f = xi_f - np.linalg.solve(J, (Xe - X)[:, :, None])[:, :, 0]
            Xe, _ = hex_geom(verts, xi_f)
            assert np.max(np.abs(Xe - X)) < 1e-13
            want, _ = hex_basis(lob, xi_f)
            assert np.max(np.abs(t["tphi"][t["fl"][f, s], t["fo"][f, s]] - want)) < 1e-11, (f, s)


@pytest.mark.parametrize("k,n,jitter", [(1, 1, 0.0), (2, 2, 0.2), (3, 1, 0.0)])
def test_tet_tables_against_independent_numpy_construction(k, n, jitter):
    d = hdg.Discretization.structured(None, "tet", n=n, degree=k, jitter=jitter, seed=21)
    t = tables(d)
    assert d.pe == (k + 1) * (k + 2) * (k + 3) // 6 and d.pf == (k + 1) * (k + 2) // 2
    xi, wq, st, wf = t["xi"], t["wq"], t["st"], t["wf"]
    # quadrature rules: inside the reference simplex, exact on all monomials of degree <= 2k (volume) / 2k (face)
    assert np.all(xi > 0) and np.all(xi.sum(axis=1) < 1) and np.all(wq > 0)
    for a, b, c in tet_monomials(2 * k):
        exact = factorial(a) * factorial(b) * factorial(c) / factorial(a + b + c + 3)
        assert abs(np.sum(wq * xi[:, 0] ** a * xi[:, 1] ** b * xi[:, 2] ** c) - exact) < 1e-14
    for a in range(2 * k + 1):
        for b in range(2 * k + 1 - a):
            exact = factorial(a) * factorial(b) / factorial(a + b + 2)
            assert abs(np.sum(wf * st[:, 0] ** a * st[:, 1] ** b) - exact) < 1e-14
    # nodes: the principal lattice of order k (as a set), vertices of the reference tetrahedron included
    lat = sorted((a / k, b / k, c / k) for a, b, c in tet_monomials(k))
    assert np.allclose(sorted(map(tuple, np.round(t["nodes"], 12))), lat, atol=1e-12)
    # nodal basis of P_k on those nodes through a Vandermonde solve
    phi, dphi = tet_basis(t["nodes"], k, xi)
    assert np.max(np.abs(t["phi"] - phi)) < 1e-11 and np.max(np.abs(t["dphi"] - dphi)) < 1e-10
    # face basis: nodal P_k on the face nodes
    fn = t["fnodes"]
    mons2 = [(a, b) for a in range(k + 1) for b in range(k + 1 - a)]
    V2 = np.stack([fn[:, 0] ** a * fn[:, 1] ** b for a, b in mons2], axis=1)
    psi = np.stack([st[:, 0] ** a * st[:, 1] ** b for a, b in mons2], axis=1) @ np.linalg.inv(V2)
    assert np.max(np.abs(t["psi"] - psi)) < 1e-11
    cen = np.array([t["vc"][t["ev"][e]].mean(axis=0) for e in range(d.ne)])
    for e in range(d.ne):
        v = t["vc"][t["ev"][e]]
        J = (v[1:] - v[0]).T                                                     # J[c, r] = dX_c / dxi_r
        assert np.max(np.abs(t["xq"][e] - (v[0] + xi @ J.T))) < 1e-13
        assert np.max(np.abs(t["det"][e] - np.linalg.det(J))) < 1e-13 and np.linalg.det(J) > 0
        assert np.max(np.abs(t["inv"][e] - np.linalg.inv(J))) < 1e-11
    for f in range(d.nf):
        c = t["vc"][t["fv"][f]]
        X = c[0] + st[:, 0:1] * (c[1] - c[0]) + st[:, 1:2] * (c[2] - c[0])
        nvec = np.cross(c[1] - c[0], c[2] - c[0])
        area = np.linalg.norm(nvec)
        assert np.max(np.abs(t["xf"][f] - X)) < 1e-13 and np.max(np.abs(t["fdet"][f] - area)) < 1e-13
        for s in range(2):
            e = t["fe"][f, s]
            if e < 0:
                continue
            unit = nvec / area
            sign = np.sign(np.dot(unit, X[0] - cen[e]))
            assert np.max(np.abs(t["nrm"][f, s] - sign * unit)) < 1e-13
            v = t["vc"][t["ev"][e]]
            xi_f = np.linalg.solve((v[1:] - v[0]).T, (X - v[0]).T).T             # invert the affine map
            want, _ = tet_basis(t["nodes"], k, xi_f)
            assert np.max(np.abs(t["tphi"][t["fl"][f, s], t["fo"][f, s]] - want)) < 1e-10, (f, s)


@pytest.mark.parametrize("shape,n", [("hex", 3), ("tet", 2)])
def test_connectivity_against_brute_force(shape, n):
    """element_to_face / face_to_elements / face_local_index rebuilt by brute force from the element vertex lists."""
    d = hdg.Discretization.structured(None, shape, n=n, degree=1, jitter=0.1, seed=4)
    t = tables(d)
    faces = {}
    for e in range(d.ne):
        for lf in range(d.n_lfe):
            f = t["e2f"][e, lf]
            key = frozenset(t["fv"][f])
            assert key <= set(t["ev"][e])                                        # the face's corners belong to the element
            faces.setdefault(f, []).append((e, lf))
    assert sorted(faces) == list(range(d.nf))
    seen = set()
    for f, sides in faces.items():
        key = frozenset(t["fv"][f])
        assert key not in seen                                                   # one face id per vertex set
        seen.add(key)
        assert len(sides) in (1, 2)
        sides.sort()                                                             # side 0 = lower element id (mesh.cpp:63-71)
        for s, (e, lf) in enumerate(sides):
            assert t["fe"][f, s] == e and t["fl"][f, s] == lf
        if len(sides) == 1:
            assert t["fe"][f, 1] == -1
    # interior faces: both elements really share exactly the face's corner set
    for f in range(d.nf):
        if t["fe"][f, 1] >= 0:
            common = set(t["ev"][t["fe"][f, 0]]) & set(t["ev"][t["fe"][f, 1]])
            assert common == set(t["fv"][f])
