"""CPU tests of the checkers themselves.
  tier A = oracle/_ref: the UNMODIFIED reference compiled in place (only its Eigen calls go through
           a stand-in header);
  tier B = oracle/hdg_oracle.cpp: our generalised restatement (2D/3D, M components).
Tier B is pinned BIT FOR BIT against tier A on the reference's own 2D cases (same tables in, same
floating-point sequence), and both against the committed golden fixtures (tests/golden)."""
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import port

GOLD = Path(__file__).resolve().parent / "golden"


def sinsin(x):
    return math.sin(math.pi * x[0]) * math.sin(math.pi * x[1])


def libm_tab(fn, pts):
    return np.array([fn(p) for p in pts.reshape(-1, pts.shape[-1])])


def tier_b_from_ref(rc, case, tau=None, nu=1.0 / 200.0):
    oc = port.OraCase(port.tables_from_ref(rc))
    if case == "poisson2d":
        xq = rc.get("elem_coords").reshape(-1, 2)
        xf = rc.get("face_coords").reshape(-1, 2)
        f = libm_tab(lambda x: 2.0 * math.pi * math.pi * sinsin(x), xq)
        g = libm_tab(sinsin, xf)
        oc.set_model("poisson", [1.0 if tau is None else tau], f, g)
    else:
        oc.set_model("burgers", [nu, 10.0 * nu + 1.0 if tau is None else tau])
    oc.set("u", rc.get("u"))
    oc.set("uhat", rc.get("uhat"))
    return oc


@pytest.mark.parametrize("case,k,n", [("poisson2d", 2, 5), ("burgers2d", 1, 6), ("burgers2d", 3, 3)])
def test_tier_b_equals_reference_bitwise(ref, case, k, n):
    rc = ref.RefCase(case, k=k, n=n)
    rc.perturb(5, 0.1)
    oc = tier_b_from_ref(rc, case)
    for nm in ("mass", "mass_inv", "minv_b0", "minv_b1", "minv_c0", "minv_c1"):
        assert np.array_equal(oc.get(nm), rc.get(nm)), nm
    rc.assemble(keep_raw=True)
    oc.assemble()
    for nm in ("q0", "q1", "e_raw", "f_raw", "h_raw", "j_raw", "d_raw0", "d_raw1", "g_raw0", "g_raw1", "ru", "ruhat_e",
               "kbar", "ebar_inv", "fbar", "hbar", "rbar", "rhs"):
        assert np.array_equal(oc.get(nm), rc.get(nm)), nm
    assert np.array_equal(oc.get("blocks"), rc.get("k_blocks"))
    assert np.array_equal(oc.neighbor, rc.get_i("neighbor"))
    x = ref.random_vector(oc.n_dof, 17)
    assert np.array_equal(oc.matvec(x), rc.matvec(x))
    for kind in ("bj", "asm"):
        rc.build_precond(kind)
        oc.build_precond(kind)
        assert np.array_equal(oc.get(f"{kind}_inv"), rc.get(f"{kind}_inv"))
        assert np.array_equal(oc.apply_base(x), rc.apply_base(x))
        xr, sr = rc.gmres(tol=1e-9, max_iters=300)
        xo, so = oc.gmres(tol=1e-9, max_iters=300)
        assert so["iters"] == sr["iters"] and so["restarts"] == sr["restarts"]
        assert np.array_equal(xo, xr)
    tr, it, nrm = oc.residual()
    rtr, rit, rnrm = rc.residual()
    assert np.array_equal(tr, rtr) and np.array_equal(it, rit) and nrm == rnrm
    d = ref.random_vector(oc.n_dof, 3)
    assert np.array_equal(oc.recover_local(d), rc.recover_local(d))


def test_tier_b_polynomial_apply_bitwise(ref):
    rc = ref.RefCase("burgers2d", k=1, n=8)
    oc = tier_b_from_ref(rc, "burgers2d")
    rc.assemble()
    oc.assemble()
    rc.build_precond("asm", poly_degree=8)
    oc.build_precond("asm")
    th = rc.get("ritz")
    oc.set("ritz", th)
    y = ref.random_vector(oc.n_dof, 4)
    assert np.array_equal(oc.apply_precond(y), rc.apply_precond(y))


@pytest.mark.parametrize("kind,deg", [("asm", 8), ("bj", 5), ("asm", 50)])
def test_tier_b_harmonic_ritz_and_leja_bitwise(ref, kind, deg):
    """compute_harmonic_ritz + leja_order of tier B (preconditioner.cpp:119-244 restated, same eigen stand-in)
    give the reference's Ritz values bit for bit, and so does the polynomial apply built on them."""
    rc = ref.RefCase("burgers2d", k=1, n=8)
    oc = tier_b_from_ref(rc, "burgers2d")
    rc.assemble()
    oc.assemble()
    rc.build_precond(kind, poly_degree=deg)
    oc.build_precond(kind, poly_degree=deg)
    assert np.array_equal(oc.get("ritz"), rc.get("ritz"))
    y = ref.random_vector(oc.n_dof, 4)
    assert np.array_equal(oc.apply_precond(y), rc.apply_precond(y))


@pytest.mark.parametrize("case,k,n,kind,deg", [("burgers2d", 1, 8, "asm", 6), ("poisson2d", 2, 6, "bj", 10)])
def test_tier_b_polynomial_newton_equals_reference(ref, case, k, n, kind, deg):
    rc = ref.RefCase(case, k=k, n=n)
    oc = tier_b_from_ref(rc, case)
    rr = rc.newton(precond=kind, poly_degree=deg)
    ro = oc.newton(precond=kind, poly_degree=deg)
    assert ro["n_newton"] == rr["n_newton"] and ro["n_gmres_total"] == rr["n_gmres_total"]
    assert ro["n_inner_prec_ops"] == rr["n_inner_prec_ops"]
    assert np.array_equal(ro["residual_history"], rr["residual_history"])
    assert np.array_equal(oc.get("uhat"), rc.get("uhat")) and np.array_equal(oc.get("u"), rc.get("u"))


def test_tier_b_chebyshev_nodes_spec(ref):
    """The Chebyshev variant is not in the reference: tier B restates the spec of DESIGN.md section 6 on top of the
    (reference-pinned) harmonic Ritz values -- roots of T_P on [min Re, max Re], Leja-ordered by the reference's
    leja_order -- and applies them with the reference's own recurrence (apply_poly with those nodes injected)."""
    rc = ref.RefCase("burgers2d", k=2, n=6)
    oc = tier_b_from_ref(rc, "burgers2d")
    rc.assemble()
    oc.assemble()
    deg = 7
    rc.build_precond("asm", poly_degree=deg)
    th = rc.get("ritz")[0::2]
    lo, hi = th.min(), th.max()
    assert lo > 0
    nodes = 0.5 * (hi + lo) + 0.5 * (hi - lo) * np.cos(np.pi * (2.0 * np.arange(deg) + 1.0) / (2.0 * deg))
    want = ref.leja_order(nodes)
    oc.build_precond("asm", poly_degree=deg, poly_kind="chebyshev")
    got = oc.ritz
    assert np.all(got.imag == 0.0) and np.allclose(got.real, want.real, rtol=1e-15, atol=0.0)
    # the reference's apply_poly with the same nodes injected
    rc.set_ritz(got)
    y = ref.random_vector(oc.n_dof, 9)
    assert np.array_equal(oc.apply_precond(y), rc.apply_precond(y))
    # residual polynomial property: w = p(A) y with 1 - t p(t) = prod (1 - t / theta_j)  =>  y - A w = prod (I - A/theta_j) y
    A = lambda v: oc.apply_base(oc.matvec(v))
    oc2 = oc.apply_precond(y)
    r = oc.apply_base(y)
    for t in got.real:
        r = r - A(r) / t
    lhs = oc.apply_base(y) - A(oc2)
    assert np.max(np.abs(lhs - r)) <= 1e-10 * np.max(np.abs(y))


@pytest.mark.parametrize("case,k,n,kind", [("poisson2d", 2, 8, "bj"), ("burgers2d", 1, 8, "asm")])
def test_tier_b_newton_equals_reference(ref, case, k, n, kind):
    rc = ref.RefCase(case, k=k, n=n)
    oc = tier_b_from_ref(rc, case)
    rr = rc.newton(precond=kind)
    ro = oc.newton(precond=kind)
    assert ro["n_newton"] == rr["n_newton"] and ro["n_gmres_total"] == rr["n_gmres_total"]
    assert np.array_equal(ro["residual_history"], rr["residual_history"])
    assert np.array_equal(oc.get("uhat"), rc.get("uhat")) and np.array_equal(oc.get("u"), rc.get("u"))


def test_golden_headline_numbers(ref):
    """Known answers recorded from the reference (regenerated by
    tests/golden/make_golden.py): config 1 = Poisson 64x64, k = 2, BJ-GMRES."""
    g = np.load(GOLD / "reference_golden.npz")
    rc = ref.RefCase("poisson2d", k=2, n=64)
    r = rc.newton(precond="bj")
    assert r["n_newton"] == int(g["cfg1_n_newton"]) == 1
    assert r["n_gmres_total"] == int(g["cfg1_n_gmres"]) == 3
    assert np.sum(rc.get("uhat") ** 2) == float(g["cfg1_sum_uhat2"])
    assert abs(float(g["cfg1_sum_uhat2"]) - 6143.9814580369875) < 1e-9


def test_golden_vectors_both_tiers(ref):
    g = np.load(GOLD / "reference_golden.npz")
    for tag, case, k, n in [("p", "poisson2d", 2, 4), ("b", "burgers2d", 2, 3)]:
        rc = ref.RefCase(case, k=k, n=n)
        rc.perturb(5, 0.1)
        oc = tier_b_from_ref(rc, case)
        rc.assemble()
        oc.assemble()
        for who in (rc, oc):
            blocks = who.get("k_blocks") if who is rc else who.get("blocks")
            assert np.array_equal(blocks, g[f"{tag}_blocks"])
            assert np.array_equal(who.get("rhs"), g[f"{tag}_rhs"])
            nb = who.get_i("neighbor") if who is rc else who.neighbor
            assert np.array_equal(nb, g[f"{tag}_neighbor"])
            assert np.array_equal(who.matvec(g[f"{tag}_x"]), g[f"{tag}_kx"])
            who.build_precond("asm")
            assert np.array_equal(who.apply_base(g[f"{tag}_x"]), g[f"{tag}_asm_x"])


def test_leja_and_ritz_known_answers(ref):
    # test_precond.cpp:277-293 / acceptance_main.cpp:289-297 style closed forms
    out = ref.leja_order([1.0, 2.0, 3.0, 4.0])
    assert out[0] == 4.0 and out[1] == 1.0
    th = ref.harmonic_ritz_dense(np.diag(np.arange(1.0, 9.0)), 8, 12345)
    assert np.allclose(np.sort(th.real), np.arange(1.0, 9.0), atol=1e-10) and np.all(th.imag == 0.0)
    rot = np.array([[1.0, -2.0], [2.0, 1.0]])
    th = ref.harmonic_ritz_dense(rot, 2, 1)
    assert np.allclose(sorted(th.imag), [-2.0, 2.0], atol=1e-10) and np.allclose(th.real, 1.0, atol=1e-10)


def test_lu_invert_known_answers():
    # dense_batch tests of the reference: permutation matrix (pivoting), singular block index
    import ctypes as C
    L = port.lib()
    a = np.array([[0.0, 1.0], [1.0, 0.0]]).ravel()
    sing = np.zeros(4)
    batch = np.concatenate([a, sing, a])
    out = np.empty_like(batch)
    bad = C.c_long()
    rc = L.ora_lu_invert_batch(2, 3, batch.ctypes.data_as(port._dp), out.ctypes.data_as(port._dp), C.byref(bad))
    assert rc == 2 and bad.value == 1          # test_dense_batch.cpp:98-111 SingularBlock.index == 1
    rc = L.ora_lu_invert_batch(2, 1, a.ctypes.data_as(port._dp), out.ctypes.data_as(port._dp), C.byref(bad))
    assert rc == 0 and np.array_equal(out[:4], a)
