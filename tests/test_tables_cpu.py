"""Setup-time host tables (mesh / master element / geometry) for every element shape, checked by
properties on the CPU: these tables are the inputs of both the CUDA kernels and the tier-B oracle.
For quads they are additionally compared bit for bit with the reference (tests/test_gpu_quad_parity.py)."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg


@pytest.mark.parametrize("shape,n,k,jitter", [("quad", 3, 2, 0.15), ("hex", 2, 2, 0.15), ("tri", 3, 1, 0.0), ("tri", 3, 3, 0.15),
                                               ("tri", 2, 4, 0.15), ("tet", 2, 1, 0.1), ("tet", 2, 2, 0.1), ("tet", 1, 3, 0.0)])
def test_tables_properties(shape, n, k, jitter):
    d = hdg.Discretization.structured(None, shape, n=n, degree=k, jitter=jitter, seed=11)
    D, qe, qf, pe, pf, ne, nf = d.dim, d.qe, d.qf, d.pe, d.pf, d.ne, d.nf
    simplex = shape in ("tri", "tet")
    assert pe == {"quad": (k + 1) ** 2, "hex": (k + 1) ** 3, "tri": (k + 1) * (k + 2) // 2, "tet": (k + 1) * (k + 2) * (k + 3) // 6}[shape]
    phi = d.table("phi").reshape(qe, pe)
    psi = d.table("psi").reshape(qf, pf)
    assert np.allclose(phi.sum(axis=1), 1.0, atol=1e-13) and np.allclose(psi.sum(axis=1), 1.0, atol=1e-13)
    w, det = d.table("elem_weights"), d.table("elem_detjac").reshape(ne, qe)
    assert abs((w * det).sum() - 1.0) < 1e-13                                  # the unit box
    assert np.all(det > 0)
    xn = d.volume_node_coords()
    xq = d.table("elem_coords").reshape(ne, qe, D)
    if simplex or jitter == 0.0:
        # nodal interpolation + gradient of a degree-k polynomial are exact on affine elements
        f = lambda x: (x[..., 0] + 0.3) ** k + 2.0 * x[..., 1] ** k + x[..., -1] * x[..., 0] ** (k - 1)
        assert np.max(np.abs(np.einsum("gi,ei->eg", phi, f(xn)) - f(xq))) < 1e-12
        ij = d.table("elem_invjac").reshape(ne, qe, D, D)
        gx = sum(np.einsum("gi,ei->eg", d.table(f"dphi{r}").reshape(qe, pe), f(xn)) * ij[:, :, r, 0] for r in range(D))
        ex = k * (xq[..., 0] + 0.3) ** (k - 1) + (xq[..., -1] * (k - 1) * xq[..., 0] ** max(k - 2, 0) if k > 1 else 0.0)
        if D == 2:
            ex = ex + 0.0
        assert np.max(np.abs(gx - ex)) < 1e-11
    # orientation tables: each side's oriented element trace, evaluated on the element's own
    # (iso/affine) geometry, lands on the face's canonical quadrature points
    tphi = d.table("tphi").reshape(d.n_lfe, d.n_orient, qf, pe)
    fc = d.table("face_coords").reshape(nf, qf, D)
    fe, fl, fo = (d.table(t).reshape(nf, 2) for t in ("face_to_elements", "face_local_index", "face_orient"))
    nrm = d.table("face_normal").reshape(nf, 2, qf, D)
    cen = xn.mean(axis=1)
    for f_ in range(nf):
        for s in range(2):
            e = fe[f_, s]
            if e < 0:
                continue
            assert np.allclose(tphi[fl[f_, s], fo[f_, s]] @ xn[e], fc[f_], atol=1e-13), (f_, s)
            assert np.allclose(np.linalg.norm(nrm[f_, s], axis=1), 1.0, atol=1e-13)
            assert np.all(np.einsum("gd,gd->g", nrm[f_, s], fc[f_] - cen[e]) > 0)
        if fe[f_, 1] >= 0:
            assert np.allclose(nrm[f_, 0], -nrm[f_, 1], atol=1e-13)
    # trace nodes interpolate the canonical face coordinates
    xt = d.trace_node_coords()
    assert np.allclose(np.einsum("gl,fld->fgd", psi, xt), fc, atol=1e-13)
    # divergence theorem on every element
    wf, fdet = d.table("face_weights"), d.table("face_detjac").reshape(nf, qf)
    e2f, es = d.table("element_to_face").reshape(ne, -1), d.table("elem_side").reshape(ne, -1)
    for e in range(ne):
        tot = sum(np.einsum("g,g,gd->d", wf, fdet[f_], nrm[f_, s]) for f_, s in zip(e2f[e], es[e]))
        assert np.allclose(tot, 0.0, atol=1e-13)
    # mesh counts / conformity
    assert np.all(fe[:, 0] >= 0)
    bnd = fe[:, 1] < 0
    assert np.all(d.table("boundary_tag")[bnd] > 0) and np.all(d.table("boundary_tag")[~bnd] == 0)
    area = np.einsum("g,fg->f", wf, fdet)[bnd].sum()
    assert abs(area - 2 * D) < 1e-12                                            # surface of the unit box


def test_quadrature_exactness_simplex():
    for shape, D in (("tri", 2), ("tet", 3)):
        for k in (1, 2, 3, 4):
            d = hdg.Discretization.structured(None, shape, n=1, degree=k)
            w, det = d.table("elem_weights"), d.table("elem_detjac").reshape(d.ne, d.qe)
            x = d.table("elem_coords").reshape(d.ne, d.qe, D)
            deg = 2 * k                                                         # the mass matrix integrand
            val = np.einsum("g,eg,eg->", w, det, x[..., 0] ** deg)
            assert abs(val - 1.0 / (deg + 1)) < 1e-13                           # int over the unit box of x^deg
