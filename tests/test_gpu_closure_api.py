"""The reference's per-function preconditioner API and closure forms (preconditioner.hpp:31-76, gmres.hpp:50-53)
through the C ABI: build_bj / apply_bj / build_asm / apply_asm as their own entry points, compute_harmonic_ritz
and apply_poly taking operator callbacks, gmres_solve taking two callbacks, and the value-type constructors
(hdgb_ops_create, hdgb_precond_create).  Checked against the handle forms, the reference's closed-form unit cases
(test_precond.cpp:231-255, acceptance_main.cpp:220-286,301-335) and the compiled reference where present."""
import ctypes as C

import numpy as np
import pytest

import paper_2512_13619_b200 as hdg

pytestmark = pytest.mark.gpu


def system(ctx, case="poisson2d", k=2, n=4):
    disc = hdg.Discretization.structured(ctx, "quad", n=n, degree=k)
    model = hdg.make_case_model(disc, case)
    state = hdg.make_initial_state(disc, model)
    ops = hdg.assemble_element_operators(disc, model, state)
    K, rhs = hdg.assemble_global(disc, ops)
    return disc, model, state, ops, K, rhs


def dense_operator(ctx, a):
    """A dense n x n matrix as the device operator callback y = A x (n small: one GEMV through the ABI)."""
    n = a.shape[0]
    col_major = np.ascontiguousarray(a.T).ravel()
    dA = ctx.alloc(n * n)
    ctx.copy(dA, col_major, n * n)

    def op(din, dout, nn):
        ctx.check(ctx._L.hdgb_gemv_strided_batch(ctx._h, n, n, 1, dA, din, dout, 0))
    return op, dA


def test_build_bj_and_asm_as_own_entry_points(ctx):
    disc, model, state, ops, K, rhs = system(ctx, "burgers2d", 2, 5)
    y = hdg.random_vector(K.n_dof, 77)
    pbj, pbj_spec = hdg.build_bj(K), hdg.build_preconditioner("bj", K, ops, disc)
    assert np.array_equal(pbj.get("bj_inv"), pbj_spec.get("bj_inv"))
    assert np.array_equal(hdg.apply_bj(pbj, y), pbj_spec.apply(y))
    # build_asm(ops, mesh) forms the two-sided diagonal sums from K-bar itself (preconditioner.cpp:59-75)
    pasm, pasm_spec = hdg.build_asm(ops, disc, K), hdg.build_preconditioner("asm", K, ops, disc)
    a, b = pasm.get("asm_inv"), pasm_spec.get("asm_inv")
    assert np.max(np.abs(a - b)) <= 1e-12 * max(1.0, np.max(np.abs(b)))
    za, zb = hdg.apply_asm(pasm, y), pasm_spec.apply(y)
    assert np.max(np.abs(za - zb)) <= 1e-12 * max(1.0, np.max(np.abs(zb)))
    with pytest.raises(hdg.DimensionMismatch):
        hdg.apply_asm(pbj, y)
    with pytest.raises(hdg.DimensionMismatch):
        hdg.apply_bj(pasm, y)


def test_value_type_constructors_round_trip(ctx):
    disc, model, state, ops, K, rhs = system(ctx, "poisson2d", 3, 3)
    names = ("kbar", "ebar_inv", "fbar", "hbar", "rbar", "ru", "ruhat_e")
    ops2 = hdg.ops_from_host(disc, *[ops.get(nm) for nm in names])
    K2, rhs2 = hdg.assemble_global(disc, ops2)
    assert np.array_equal(K2.blocks, K.blocks) and np.array_equal(rhs2, rhs) and np.array_equal(K2.neighbor, K.neighbor)
    duhat = hdg.random_vector(K.n_dof, 5)
    assert np.array_equal(hdg.recover_local(disc, ops2, duhat), hdg.recover_local(disc, ops, duhat))
    y = hdg.random_vector(K.n_dof, 6)
    pasm = hdg.build_preconditioner("asm", K, ops, disc)
    p2 = hdg.precond_from_host(ctx, "asm", disc.mpf, disc.nf, pasm.get("asm_inv"), disc=disc, k=K)
    assert np.array_equal(hdg.apply_asm(p2, y), pasm.apply(y))
    pbj = hdg.build_bj(K)
    p3 = hdg.precond_from_host(ctx, "bj", disc.mpf, disc.nf, pbj.get("bj_inv"), k=K)
    assert np.array_equal(hdg.apply_bj(p3, y), hdg.apply_bj(pbj, y))


def test_closure_gmres_equals_handle_gmres(ctx):
    disc, model, state, ops, K, rhs = system(ctx, "burgers2d", 2, 6)
    pc = hdg.build_preconditioner("asm", K, ops, disc)
    cfg = hdg.GmresConfig(restart=20, tol=1e-10, track_diagnostics=True)
    L = ctx._L

    def mv(din, dout, n):
        ctx.check(L.hdgb_block_matvec(K._h, din, dout))

    def pr(din, dout, n):
        ctx.check(L.hdgb_precond_apply(pc._h, K._h, din, dout))

    xc, sc = hdg.gmres_solve_fn(ctx, K.n_dof, mv, pr, rhs, cfg=cfg)
    xh, sh = hdg.gmres_solve(K, pc, rhs, cfg=cfg)
    assert sc.converged and sh.converged and sc.iters == sh.iters and sc.restarts == sh.restarts
    assert np.array_equal(xc, xh)
    assert np.array_equal(sc.residual_trace, sh.residual_trace)
    # identity preconditioner = NULL callback
    xi, si = hdg.gmres_solve_fn(ctx, K.n_dof, mv, None, rhs, cfg=hdg.GmresConfig(tol=1e-8, max_iters=400))
    xj, sj = hdg.gmres_solve(K, None, rhs, cfg=hdg.GmresConfig(tol=1e-8, max_iters=400))
    assert si.iters == sj.iters and np.array_equal(xi, xj)


def test_closure_gmres_exact_within_n_iterations(ctx):
    # gmres_contract of the reference (acceptance_main.cpp:338-358, tests/test_gmres.cpp): n <= restart => exact in <= n steps
    for n in (5, 12, 25):
        a = hdg.random_vector(n * n, 600 + n).reshape(n, n) + 5.0 * np.eye(n)
        rhs = hdg.random_vector(n, 700 + n)
        op, dA = dense_operator(ctx, a)
        x, st = hdg.gmres_solve_fn(ctx, n, op, None, rhs, x0=np.zeros(n), cfg=hdg.GmresConfig(tol=1e-12))
        ctx.free(dA)
        assert st.converged and st.iters <= n
        assert np.max(np.abs(a @ x - rhs)) <= 1e-10 * np.max(np.abs(rhs))


def test_callback_exception_surfaces(ctx):
    def boom(din, dout, n):
        raise ValueError("boom")
    with pytest.raises(ValueError, match="boom"):
        hdg.gmres_solve_fn(ctx, 8, boom, None, np.ones(8))


def test_compute_harmonic_ritz_known_spectra(ctx):
    # test_precond.cpp:231-255 / acceptance_main.cpp:301-335: diag(1..p) and the rotation pair 1 +- 2i
    p = 12
    op, dA = dense_operator(ctx, np.diag(np.arange(1.0, p + 1)))
    th = hdg.compute_harmonic_ritz(ctx, op, p, p, seed=99)
    ctx.free(dA)
    assert len(th) == p and np.max(np.abs(th.imag)) <= 1e-10
    assert np.max(np.abs(np.sort(th.real) - np.arange(1.0, p + 1))) <= 1e-10
    op, dA = dense_operator(ctx, np.array([[1.0, -2.0], [2.0, 1.0]]))
    pair = hdg.compute_harmonic_ritz(ctx, op, 2, 2, seed=5)
    ctx.free(dA)
    assert len(pair) == 2 and abs(pair[0].real - 1.0) <= 1e-10 and abs(abs(pair[0].imag) - 2.0) <= 1e-10
    assert pair[1] == np.conj(pair[0])


def test_compute_harmonic_ritz_matches_reference(ctx, ref):
    # same seeded start vector, same MGS Arnoldi: the closure form against the compiled reference's values
    rc = ref.RefCase("burgers2d", k=1, n=8)
    rc.assemble()
    rc.build_precond("bj", poly_degree=10)
    want = rc.get("ritz")
    want = want[0::2] + 1j * want[1::2]
    disc = hdg.Discretization.structured(ctx, "quad", n=8, degree=1)
    model = hdg.make_case_model(disc, "burgers2d")
    state = hdg.State(disc)
    state.set("u", rc.get("u"))
    state.set("uhat", rc.get("uhat"))
    ops = hdg.assemble_element_operators(disc, model, state)
    K, rhs = hdg.assemble_global(disc, ops)
    pbj = hdg.build_bj(K)
    tmp = ctx.alloc(K.n_dof)
    L = ctx._L

    def op(din, dout, n):
        ctx.check(L.hdgb_block_matvec(K._h, din, tmp))
        ctx.check(L.hdgb_apply_bj(pbj._h, tmp, dout))
    th = hdg.compute_harmonic_ritz(ctx, op, K.n_dof, 10, seed=12345)
    ctx.free(tmp)
    assert len(th) == len(want)
    assert np.max(np.abs(th - want)) <= 1e-8 * np.max(np.abs(want))


def test_apply_poly_exact_inverse_with_closure_base(ctx):
    # polynomial_exactness (acceptance_main.cpp:220-286): P = n nodes at the spectrum => exact inverse, also with
    # complex pairs; K is a dense operator wrapped as a one-face FaceBlockMatrix, the base is an identity CLOSURE
    a = np.zeros((6, 6))
    a[0, 0], a[0, 1], a[1, 0], a[1, 1] = 1, -2, 2, 1
    a[2, 2], a[2, 3], a[3, 2], a[3, 3] = 3, -1, 1, 3
    a[4, 4], a[5, 5] = 5, 0.5
    spectrum = [1 + 2j, 1 - 2j, 3 + 1j, 3 - 1j, 5, 0.5]
    n, nb = 6, 7
    blocks = np.zeros((n * nb, n))
    blocks[:n, :] = a.T          # column-major n x (n*nb) block row, slot 0 = the matrix
    nbr = np.full(nb, -1, dtype=np.int64)
    nbr[0] = 0
    K = hdg.FaceBlockMatrix.from_host(ctx, 1, n, 4, 1, nbr, blocks.ravel())
    p = hdg.precond_from_host(ctx, "identity", n, 1, ritz=hdg.leja_order(spectrum), k=K)
    y = hdg.random_vector(n, 4242)

    def ident(din, dout, nn):
        ctx.copy(dout, din, nn)
    z, inner = hdg.apply_poly(p, K, y, base=ident)
    exact = np.linalg.solve(a, y)
    assert np.max(np.abs(z - exact)) <= 1e-8 * max(1.0, np.max(np.abs(exact)))
    assert inner == 6
    z2, _ = hdg.apply_poly(p, K, y)   # the preconditioner's own (identity) base
    assert np.array_equal(z, z2)


@pytest.mark.parametrize("kind", ["identity", "bj", "asm", "ras"])
def test_fused_polynomial_epilogues_equal_the_separate_updates(ctx, kind):
    """The recurrence updates (preconditioner.cpp:259-281) applied inside the kernel that produces base(K v) -- the ASM
    face sum / one pass after the BJ GEMV -- against the separate vector kernels: same operations on the same
    values, so bit-identical, for real nodes and conjugate pairs; inner operator counts unchanged."""
    disc, model, state, ops, K, rhs = system(ctx, "burgers2d", 2, 6)
    y = hdg.random_vector(K.n_dof, 31)
    for spec in (hdg.PrecondSpec(kind, poly_degree=7), hdg.PrecondSpec(kind, poly_degree=6, poly_kind="chebyshev")):
        out = {}
        for fused in (1, 0):
            hdg.set_tuning("poly_fused", fused)
            try:
                P = hdg.build_preconditioner(spec, K, ops, disc)
                out[fused] = (P.apply(y), P.inner_ops, P.ritz)
                if spec.poly_kind == 0:  # also with conjugate pairs among the nodes
                    P.set_ritz([3 + 1j, 3 - 1j, 5.0, 1 + 2j, 1 - 2j])
                    out[fused] += (P.apply(y),)
            finally:
                hdg.set_tuning("poly_fused", 1)
        assert np.array_equal(out[1][2], out[0][2])
        assert np.array_equal(out[1][0], out[0][0]) and out[1][1] == out[0][1]
        if len(out[1]) > 3:
            assert np.array_equal(out[1][3], out[0][3])
