"""GPU parity on configurations the reference itself cannot run (3D hexahedra, M > 1), against the
tier-B CPU restatement (oracle/hdg_oracle.cpp) -- which tests/test_oracle.py pins bit for bit to the
unmodified reference on the shared 2D subset -- plus table-level property checks of the hex setup
layer that the restatement takes as input (orientation, normals, quadrature)."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg
from oracle import port

pytestmark = pytest.mark.gpu


def relerr(a, b):
    return np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b)))


def setup(ctx, shape, n, k, case, n_comp=1, jitter=0.0, **kw):
    disc = hdg.Discretization.structured(ctx, shape, n=n, degree=k, n_comp=n_comp, jitter=jitter, seed=7)
    model = hdg.make_case_model(disc, case, **kw)
    state = hdg.make_initial_state(disc, model)
    oc = port.OraCase(port.tables_from_disc(disc))
    oc.set_model_like(model)
    return disc, model, state, oc


def perturb(disc, state, oc, scale=0.1):
    u = state.u + hdg.random_vector(disc.npe * disc.ne, 5, scale)
    uh = state.uhat + hdg.random_vector(disc.n_dof, 6, scale)
    state.u, state.uhat = u, uh
    oc.set("u", u)
    oc.set("uhat", uh)


@pytest.mark.parametrize("jitter", [0.0, 0.15])
def test_hex_tables_properties(ctx, jitter):
    disc = hdg.Discretization.structured(ctx, "hex", n=3, degree=2, jitter=jitter, seed=3)
    D, qe, qf, pe, pf, ne, nf = 3, disc.qe, disc.qf, disc.pe, disc.pf, disc.ne, disc.nf
    phi = disc.table("phi").reshape(qe, pe)
    assert np.allclose(phi.sum(axis=1), 1.0, atol=1e-13)                      # partition of unity
    w, det = disc.table("elem_weights"), disc.table("elem_detjac").reshape(ne, qe)
    assert abs((w * det).sum() - 1.0) < 1e-13                                  # volume of the unit cube
    # each side's oriented element trace, evaluated on the element's own geometry, must land on the
    # face's canonical quadrature points (this is what the orientation tables are for)
    tphi = disc.table("tphi").reshape(disc.n_lfe, disc.n_orient, qf, pe)
    xn = disc.volume_node_coords()                                             # (ne, pe, 3) isoparametric nodes
    fc = disc.table("face_coords").reshape(nf, qf, D)
    fe, fl, fo = (disc.table(t).reshape(nf, 2) for t in ("face_to_elements", "face_local_index", "face_orient"))
    nrm = disc.table("face_normal").reshape(nf, 2, qf, D)
    cen = xn.mean(axis=1)
    for f in range(nf):
        for s in range(2):
            e = fe[f, s]
            if e < 0:
                continue
            x_side = tphi[fl[f, s], fo[f, s]] @ xn[e]                          # (qf, 3)
            assert np.allclose(x_side, fc[f], atol=1e-13), (f, s)
            n = nrm[f, s]
            assert np.allclose(np.linalg.norm(n, axis=1), 1.0, atol=1e-13)
            assert np.all(np.einsum("gd,gd->g", n, fc[f] - cen[e]) > 0)        # outward
        if fe[f, 1] >= 0:
            assert np.allclose(nrm[f, 0], -nrm[f, 1], atol=1e-13)
    # divergence theorem on every element: sum_faces int n = 0
    wf, fdet = disc.table("face_weights"), disc.table("face_detjac").reshape(nf, qf)
    e2f, es = disc.table("element_to_face").reshape(ne, -1), disc.table("elem_side").reshape(ne, -1)
    for e in range(ne):
        tot = sum(np.einsum("g,g,gd->d", wf, fdet[f], nrm[f, s]) for f, s in zip(e2f[e], es[e]))
        assert np.allclose(tot, 0.0, atol=1e-13)


@pytest.mark.parametrize("shape,case,k,n,ncomp,jitter", [
    ("hex", "poisson", 2, 3, 1, 0.0), ("hex", "poisson", 3, 2, 1, 0.15), ("hex", "burgers", 2, 2, 1, 0.1),
    ("hex", "elasticity", 1, 3, 3, 0.1), ("hex", "elasticity", 2, 2, 3, 0.0),
    # BASELINE configs 3 and 4 in miniature: triangles p = 4 Burgers, tetrahedra p = 2 elasticity (M = 3)
    ("tri", "burgers", 4, 3, 1, 0.2), ("tri", "poisson", 2, 4, 1, 0.2), ("tri", "elasticity", 3, 3, 2, 0.1),
    ("tet", "elasticity", 2, 2, 3, 0.1), ("tet", "poisson", 3, 2, 1, 0.1), ("tet", "burgers", 1, 2, 1, 0.0),
    ("quad", "elasticity", 2, 4, 2, 0.1)])
def test_hex_operators_vs_tier_b(ctx, shape, case, k, n, ncomp, jitter):
    disc, model, state, oc = setup(ctx, shape, n, k, case, n_comp=ncomp, jitter=jitter)
    perturb(disc, state, oc)
    oc.assemble()
    ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True)
    for d in range(disc.dim):
        assert relerr(disc.table(f"minv_b{d}"), oc.get(f"minv_b{d}")) < 1e-11
        assert relerr(disc.table(f"minv_c{d}"), oc.get(f"minv_c{d}")) < 1e-11
        assert relerr(state.q(d), oc.get(f"q{d}")) < 1e-11
        assert relerr(ops.get(f"d_raw{d}"), oc.get(f"d_raw{d}")) < 1e-12
        assert relerr(ops.get(f"g_raw{d}"), oc.get(f"g_raw{d}")) < 1e-12
    for nm in ("e_raw", "f_raw", "h_raw", "j_raw", "ru", "ruhat_e"):
        assert relerr(ops.get(nm), oc.get(nm)) < 1e-12, nm
    for nm in ("kbar", "ebar_inv", "fbar", "hbar", "rbar"):
        assert relerr(ops.get(nm), oc.get(nm)) < 1e-9, nm
    K, rhs = hdg.assemble_global(disc, ops)
    assert np.array_equal(K.neighbor, oc.neighbor)
    assert relerr(K.blocks, oc.get("blocks")) < 1e-9 and relerr(rhs, oc.get("rhs")) < 1e-9
    x = hdg.random_vector(K.n_dof, 1)
    y = hdg.block_matvec(K, x)
    assert relerr(y, oc.matvec(x)) < 1e-9
    yd = K.to_dense() @ x
    assert np.max(np.abs(y - yd)) <= 1e-13 * max(1.0, np.max(np.abs(yd)))
    for kind in ("bj", "asm", "ras"):
        P = hdg.build_preconditioner(kind, K, ops, disc)
        oc.build_precond(kind)
        assert relerr(P.apply_base(x), oc.apply_base(x)) < 1e-8, kind
    tr, it, nrm = hdg.assemble_residual(disc, model, state)
    otr, oit, onrm = oc.residual()
    assert relerr(tr, otr) < 1e-12 and relerr(it, oit) < 1e-12 and abs(nrm - onrm) < 1e-12 * onrm
    d = hdg.random_vector(K.n_dof, 2)
    assert relerr(hdg.recover_local(disc, ops, d), oc.recover_local(d)) < 1e-9


@pytest.mark.parametrize("shape,case,k,n,ncomp,kind", [
    ("hex", "poisson", 2, 4, 1, "asm"), ("hex", "poisson", 3, 3, 1, "bj"), ("hex", "elasticity", 2, 2, 3, "asm"),
    ("hex", "burgers", 2, 3, 1, "bj"), ("tri", "burgers", 4, 4, 1, "asm"), ("tri", "poisson", 3, 5, 1, "bj"),
    ("tet", "elasticity", 2, 2, 3, "asm"), ("tet", "poisson", 2, 3, 1, "asm")])
def test_hex_newton_vs_tier_b(ctx, shape, case, k, n, ncomp, kind):
    disc, model, state, oc = setup(ctx, shape, n, k, case, n_comp=ncomp, jitter=0.1 if shape in ("tri", "tet") else 0.0)
    oc.set("u", state.u)
    oc.set("uhat", state.uhat)
    ro = oc.newton(precond=kind)
    rep = hdg.newton_solve(disc, model, state, pspec=hdg.PrecondSpec(kind))
    assert rep.converged and ro["converged"]
    assert rep.n_newton == ro["n_newton"]
    assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_per_newton, ro["gmres_per_newton"]))
    assert relerr(state.uhat, oc.get("uhat")) < 1e-6
    assert relerr(state.u, oc.get("u")) < 1e-6


@pytest.mark.parametrize("shape", ["hex", "tri", "tet"])
def test_hex_poisson_converges_at_design_order(ctx, shape):
    errs = []
    for n in (2, 4):
        disc = hdg.Discretization.structured(ctx, shape, n=n, degree=2)
        model = hdg.make_case_model(disc, "poisson")
        state = hdg.make_initial_state(disc, model)
        rep = hdg.newton_solve(disc, model, state, gcfg=hdg.GmresConfig(tol=1e-10), pspec=hdg.PrecondSpec("asm"))
        assert rep.converged
        errs.append(disc.l2_error(state.u, model.exact_solution))
    assert np.log2(errs[0] / errs[1]) >= 2.5          # acceptance_main.cpp:392-395: order >= k + 0.5


@pytest.mark.parametrize("shape,case,k,n,ncomp", [("hex", "burgers", 2, 2, 1), ("tet", "elasticity", 2, 2, 3), ("quad", "burgers", 3, 3, 1)])
def test_point_chunked_assembly_matches_single_sweep(ctx, shape, case, k, n, ncomp):
    """Wide systems sweep the quadrature points in chunks that accumulate into the outputs; forcing tiny
    chunks on small systems must reproduce the one-sweep blocks (chunk partial sums are added in the
    same point order, so only the association of the additions changes)."""
    disc = hdg.Discretization.structured(ctx, shape, n=n, degree=k, n_comp=ncomp, jitter=0.1, seed=5)
    model = hdg.make_case_model(disc, case)
    state = hdg.make_initial_state(disc, model)
    state.u = state.u + hdg.random_vector(disc.npe * disc.ne, 5, 0.1)
    state.uhat = state.uhat + hdg.random_vector(disc.n_dof, 6, 0.1)
    names = ["e_raw", "f_raw", "h_raw", "j_raw", "ru", "ruhat_e", "kbar", "rbar"] + [f"d_raw{d}" for d in range(disc.dim)] + \
            [f"g_raw{d}" for d in range(disc.dim)]
    out = {}
    for kb in (216, 8):
        hdg.set_tuning("assemble_budget_kb", kb)
        try:
            ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True)
            out[kb] = {nm: ops.get(nm) for nm in names}
            out[kb]["res"] = hdg.assemble_residual(disc, model, state)
        finally:
            hdg.set_tuning("assemble_budget_kb", 216)
    for nm in names:
        assert relerr(out[8][nm], out[216][nm]) < (1e-11 if nm in ("kbar", "rbar") else 1e-13), nm
    for a, b in zip(out[8]["res"][:2], out[216]["res"][:2]):
        assert relerr(a, b) < 1e-13


@pytest.mark.parametrize("shape,case,k,n,ncomp", [
    ("hex", "poisson", 3, 3, 1),      # config 2's element: npe 64, nfl 96 (three warps, 16-byte copies)
    ("hex", "burgers", 2, 3, 1),      # npe 27 (odd: 8-byte copies, k padded to 32), nfl 54
    ("hex", "elasticity", 1, 3, 3),   # npe 24, nfl 72
    ("tet", "elasticity", 2, 2, 3),   # config 4's element: npe 30, nfl 72
    ("tet", "poisson", 3, 2, 1),      # npe 20, nfl 40
    ("quad", "elasticity", 3, 4, 2),  # npe 32, nfl 32
    ("hex", "elasticity", 2, 2, 3)])  # nfl 162 > 128: the fused kernel declines, two products
def test_schur_fused_matches_two_products(ctx, shape, case, k, n, ncomp):
    """K-bar = J-bar - H-bar (E-bar^-1 F-bar) (local_ops.cpp:408-411): the one-kernel form with T in shared memory
    against the two batched products (rounding-level agreement), and against the tier-B oracle."""
    disc, model, state, oc = setup(ctx, shape, n, k, case, n_comp=ncomp, jitter=0.1)
    perturb(disc, state, oc)
    got = {}
    try:
        for flag in (0, 1):
            hdg.set_tuning("schur_fused", flag)
            ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True)
            got[flag] = {nm: ops.get(nm).copy() for nm in ("kbar", "ebar_inv", "fbar", "hbar", "rbar")}
    finally:
        hdg.set_tuning("schur_fused", 1)
    for nm in ("ebar_inv", "fbar", "hbar", "rbar"):
        assert np.array_equal(got[0][nm], got[1][nm]), nm
    assert relerr(got[1]["kbar"], got[0]["kbar"]) < 1e-12
    oc.assemble()
    assert relerr(got[1]["kbar"], oc.get("kbar")) < 1e-9
