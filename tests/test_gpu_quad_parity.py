"""GPU parity against the UNMODIFIED reference (oracle/_ref) on 2D quadrilateral cases, through the
C ABI.  Tolerances are the reference's own test tolerances or tighter; index
tables are compared bit for bit."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg

pytestmark = pytest.mark.gpu


def make(ctx, ref, case, k, n, tau=None, **kw):
    rc = ref.RefCase(case, k=k, n=n, tau=tau, **kw)
    disc = hdg.Discretization.structured(ctx, "quad", n=n, degree=k)
    model = hdg.make_case_model(disc, case, tau=tau, **{a: b for a, b in kw.items() if a in ("nu", "kappa", "velocity")})
    state = hdg.make_initial_state(disc, model)
    return rc, disc, model, state


def relerr(a, b):
    return np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b)))


@pytest.mark.parametrize("k,n", [(1, 3), (2, 4), (3, 2), (4, 3)])
def test_tables_bitwise(ctx, ref, k, n):
    rc, disc, _, _ = make(ctx, ref, "poisson2d", k, n)
    for ours, theirs in [("element_to_face", "element_to_face"), ("face_to_elements", "face_to_elements"),
                         ("face_local_index", "face_local_index"), ("boundary_tag", "boundary_tag"),
                         ("element_vertices", "element_vertices"), ("face_vertices", "face_vertices")]:
        assert np.array_equal(disc.table(ours).astype(np.int64), rc.get_i(theirs)), ours
    for ours, theirs in [("phi", "phi"), ("dphi0", "dphi_dxi"), ("dphi1", "dphi_deta"), ("psi", "psi"),
                         ("elem_weights", "rule2d_weights"), ("rule1d_points", "rule1d_points"),
                         ("rule1d_weights", "rule1d_weights"), ("nodes1d", "nodes1d"),
                         ("elem_detjac", "elem_detjac"), ("elem_invjac", "elem_invjac"),
                         ("elem_coords", "elem_coords"), ("face_detjac", "face_detjac"),
                         ("face_coords", "face_coords"), ("face_normal", "face_normal"),
                         ("tphi_local", None)]:
        a = disc.table(ours)
        b = rc.get(theirs) if theirs else np.concatenate([rc.get(f"trace_phi{l}") for l in range(4)])
        assert a.shape == b.shape, (ours, a.shape, b.shape)
        assert np.array_equal(a, b), (ours, np.max(np.abs(a - b)))


@pytest.mark.parametrize("k,n", [(1, 4), (2, 5), (3, 3)])
def test_local_factors(ctx, ref, k, n):
    rc, disc, _, _ = make(ctx, ref, "poisson2d", k, n)
    for ours, theirs in [("mass", "mass"), ("mass_inv", "mass_inv"), ("minv_b0", "minv_b0"), ("minv_b1", "minv_b1"),
                         ("minv_c0", "minv_c0"), ("minv_c1", "minv_c1")]:
        assert relerr(disc.table(ours), rc.get(theirs)) < 1e-12, ours


@pytest.mark.parametrize("case,k,n", [("poisson2d", 2, 6), ("burgers2d", 1, 5), ("burgers2d", 3, 4), ("convdiff2d", 2, 4)])
def test_element_operators_and_global(ctx, ref, case, k, n):
    rc, disc, model, state = make(ctx, ref, case, k, n)
    rc.perturb(7, 0.1)
    state.u, state.uhat = rc.get("u"), rc.get("uhat")
    rc.assemble(keep_raw=True)
    ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True)
    for name in ["e_raw", "f_raw", "h_raw", "j_raw", "d_raw0", "d_raw1", "g_raw0", "g_raw1", "ru", "ruhat_e"]:
        assert relerr(ops.get(name), rc.get(name)) < 1e-12, name
    for name in ["kbar", "ebar_inv", "fbar", "hbar", "rbar"]:
        assert relerr(ops.get(name), rc.get(name)) < 1e-10, name
    assert relerr(state.q(0), rc.get("q0")) < 1e-12
    K, rhs = hdg.assemble_global(disc, ops)
    assert np.array_equal(K.neighbor, rc.get_i("neighbor"))        # bit-exact block sparsity / indexing
    assert relerr(K.blocks, rc.get("k_blocks")) < 1e-10
    assert relerr(rhs, rc.get("rhs")) < 1e-10
    # matvec vs reference matvec and vs dense expansion (test_face_matrix.cpp:185-202, 1e-13)
    x = hdg.random_vector(K.n_dof, 99)
    y = hdg.block_matvec(K, x)
    yr = rc.matvec(x)
    assert np.max(np.abs(y - yr)) <= 1e-10 * max(1.0, np.max(np.abs(yr)))
    yd = K.to_dense() @ x
    assert np.max(np.abs(y - yd)) <= 1e-13 * max(1.0, np.max(np.abs(yd)))
    # gather is a bit copy in slot order (test_face_matrix.cpp:134-148)
    assert np.array_equal(hdg.gather_extended(K, x), rc.gather_extended(x))


def test_residual_and_recover(ctx, ref):
    rc, disc, model, state = make(ctx, ref, "burgers2d", 2, 5)
    rc.perturb(3, 0.05)
    state.u, state.uhat = rc.get("u"), rc.get("uhat")
    tr, it, nrm = hdg.assemble_residual(disc, model, state)
    rtr, rit, rnrm = rc.residual()
    assert relerr(tr, rtr) < 1e-12 and relerr(it, rit) < 1e-12
    assert abs(nrm - rnrm) <= 1e-12 * rnrm
    rc.assemble()
    ops = hdg.assemble_element_operators(disc, model, state)
    d = hdg.random_vector(disc.n_dof, 5)
    assert np.array_equal(hdg.gather_element_trace(disc, d), rc.gather_element_trace(d))
    assert relerr(hdg.recover_local(disc, ops, d), rc.recover_local(d)) < 1e-10


@pytest.mark.parametrize("kind", ["bj", "asm"])
def test_preconditioner_apply(ctx, ref, kind):
    rc, disc, model, state = make(ctx, ref, "burgers2d", 2, 6)
    rc.perturb(11, 0.1)
    state.u, state.uhat = rc.get("u"), rc.get("uhat")
    rc.assemble()
    rc.build_precond(kind)
    ops = hdg.assemble_element_operators(disc, model, state)
    K, _ = hdg.assemble_global(disc, ops)
    P = hdg.build_preconditioner(kind, K, ops, disc)
    assert relerr(P.get(f"{kind}_inv"), rc.get(f"{kind}_inv")) < 1e-9
    for seed in range(5):
        y = hdg.random_vector(K.n_dof, 100 + seed)
        assert relerr(P.apply_base(y), rc.apply_base(y)) < 1e-10


def test_restricted_additive_schwarz_from_reference_pieces(ctx, ref):
    """RAS is not in the reference, but every piece of it is: the inverted enriched element blocks
    (build_asm, preconditioner.cpp:54-84), the element gather (local_ops.cpp:351-365) and the mesh's side tables.
    The restricted prolongation -- a shared face keeps only its side-0 (owner) element's correction instead of the
    two-sided sum of preconditioner.cpp:92-103 -- is restated here in numpy on the REFERENCE's own data, which pins
    the device RAS apply to the compiled reference."""
    rc, disc, model, state = make(ctx, ref, "burgers2d", 2, 6)
    rc.perturb(11, 0.1)
    state.u, state.uhat = rc.get("u"), rc.get("uhat")
    rc.assemble()
    rc.build_precond("asm")
    ne, nf, pf = rc.ne, rc.nf, rc.pf
    nfl = 4 * pf
    inv = rc.get("asm_inv").reshape(ne, nfl, nfl)                     # column-major blocks: [e][col][row]
    f2e = rc.get_i("face_to_elements").reshape(nf, 2)
    fli = rc.get_i("face_local_index").reshape(nf, 2)
    ops = hdg.assemble_element_operators(disc, model, state)
    K, _ = hdg.assemble_global(disc, ops)
    P = hdg.build_preconditioner("ras", K, ops, disc)
    for seed in range(4):
        y = hdg.random_vector(K.n_dof, 300 + seed)
        ye = rc.gather_element_trace(y).reshape(ne, nfl)
        ze = np.einsum("ecr,ec->er", inv, ye)                            # ze_e = inv_e ye_e
        want = np.stack([ze[f2e[f, 0], fli[f, 0] * pf:(fli[f, 0] + 1) * pf] for f in range(nf)]).ravel()
        both = want.copy().reshape(nf, pf)
        for f in range(nf):
            if f2e[f, 1] >= 0:
                both[f] += ze[f2e[f, 1], fli[f, 1] * pf:(fli[f, 1] + 1) * pf]
        assert relerr(both.ravel(), rc.apply_base(y)) < 1e-13          # the restatement reproduces the reference's ASM
        assert relerr(P.apply_base(y), want) < 1e-10


@pytest.mark.parametrize("kind,deg", [("bj", 6), ("asm", 10)])
def test_polynomial_preconditioner(ctx, ref, kind, deg):
    rc, disc, model, state = make(ctx, ref, "burgers2d", 1, 8)
    rc.assemble()
    rc.build_precond(kind, poly_degree=deg)
    ops = hdg.assemble_element_operators(disc, model, state)
    K, _ = hdg.assemble_global(disc, ops)
    P = hdg.build_preconditioner(hdg.PrecondSpec(kind, poly_degree=deg), K, ops, disc)
    th, thr = P.ritz, rc.get("ritz")
    thr = thr[0::2] + 1j * thr[1::2]
    assert len(th) == len(thr)
    assert np.max(np.abs(th - thr)) < 1e-8 * np.max(np.abs(thr))
    # same interpolation nodes -> the recurrence must agree to rounding
    P.set_ritz(thr)
    y = hdg.random_vector(K.n_dof, 21)
    assert relerr(P.apply(y), rc.apply_precond(y)) < 1e-9


@pytest.mark.parametrize("case,k,n,kind,deg", [("poisson2d", 2, 8, "bj", 0), ("poisson2d", 2, 8, "asm", 0),
                                               ("burgers2d", 1, 8, "bj", 0), ("burgers2d", 2, 6, "asm", 5)])
def test_gmres_iterations_and_solution(ctx, ref, case, k, n, kind, deg):
    rc, disc, model, state = make(ctx, ref, case, k, n)
    rc.assemble()
    rc.build_precond(kind, poly_degree=deg)
    xr, sr = rc.gmres(tol=1e-10, max_iters=400)
    ops = hdg.assemble_element_operators(disc, model, state)
    K, rhs = hdg.assemble_global(disc, ops)
    P = hdg.build_preconditioner(hdg.PrecondSpec(kind, poly_degree=deg), K, ops, disc)
    x, st = hdg.gmres_solve(K, P, rhs, cfg=hdg.GmresConfig(tol=1e-10, max_iters=400))
    assert bool(st.converged) == sr["converged"]
    assert abs(st.iters - sr["iters"]) <= 1
    assert relerr(x, xr) < 1e-8


@pytest.mark.parametrize("case,k,n,kind,deg", [("poisson2d", 2, 8, "bj", 0), ("burgers2d", 1, 8, "bj", 0),
                                               ("burgers2d", 2, 8, "asm", 0), ("burgers2d", 1, 8, "asm", 10)])
def test_newton(ctx, ref, case, k, n, kind, deg):
    rc, disc, model, state = make(ctx, ref, case, k, n)
    rr = rc.newton(precond=kind, poly_degree=deg)
    rep = hdg.newton_solve(disc, model, state, pspec=hdg.PrecondSpec(kind, poly_degree=deg))
    assert rep.converged == rr["converged"]
    assert rep.n_newton == rr["n_newton"]
    assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_per_newton, rr["gmres_per_newton"]))
    assert relerr(state.uhat, rc.get("uhat")) < 1e-6   # GMRES tol 1e-6 bounds the agreement
    assert relerr(state.u, rc.get("u")) < 1e-6
    assert abs(rep.final_residual - rr["final_residual"]) <= 1e-6 * max(1.0, rr["residual_history"][0])
