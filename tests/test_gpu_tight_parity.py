"""North-star tolerance, asserted: with both sides solved to tight tolerances (GMRES 1e-12 relative,
Newton near the rounding floor of the residual) the CUDA path must reproduce the CPU oracle's solution and
residual norms to 1e-10 relative and its GMRES iteration counts to +-1 -- one case per BASELINE.json
configuration, in miniature (the full-size runs are property-checked in test_gpu_full_size.py).
Config 1 is compared with the compiled reference itself (tier A), the others with the tier-B restatement
(bit-identical to tier A wherever the reference can run, tests/test_oracle.py)."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg
from oracle import port

pytestmark = pytest.mark.gpu

TOL = 1e-10


def relerr(a, b):
    return np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b)))


CASES = {
    # name: shape, n, degree, n_comp, case, jitter, precond, poly, poly_kind, dt, newton_tol
    "cfg2_hex_p3_poisson_asm": ("hex", 3, 3, 1, "poisson", 0.0, "asm", 0, "gmres", None, 1e-11),
    "cfg2_hex_p3_poisson_ras": ("hex", 3, 3, 1, "poisson", 0.0, "ras", 0, "gmres", None, 1e-11),
    "cfg3_tri_p4_burgers_asm_chebyshev": ("tri", 4, 4, 1, "burgers", 0.2, "asm", 10, "chebyshev", None, 1e-11),
    "cfg3_tri_p4_burgers_asm_gmres_poly": ("tri", 4, 4, 1, "burgers", 0.2, "asm", 10, "gmres", None, 1e-11),
    "cfg4_tet_p2_elasticity_asm": ("tet", 2, 2, 3, "elasticity", 0.2, "asm", 0, "gmres", None, 1e-10),
    "cfg5_hex_p3_navier_stokes_bj": ("hex", 2, 3, 5, "navier_stokes", 0.0, "bj", 0, "gmres", 0.01, 1e-9),
    "cfg5_hex_p2_navier_stokes_bj_jittered": ("hex", 2, 2, 5, "navier_stokes", 0.1, "bj", 0, "gmres", 0.02, 1e-9),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_tight_tolerance_solution_and_residual_parity(ctx, name):
    shape, n, k, ncomp, case, jitter, kind, deg, pkind, dt, ntol = CASES[name]
    disc = hdg.Discretization.structured(ctx, shape, n=n, degree=k, n_comp=ncomp, jitter=jitter, seed=12345)
    kw = {"mu": 0.02} if case == "navier_stokes" else {}
    model = hdg.make_case_model(disc, case, **kw)
    state = hdg.make_initial_state(disc, model)
    u0, uh0 = state.u, state.uhat
    oc = port.OraCase(port.tables_from_disc(disc))
    oc.set_model_like(model)
    oc.set("u", u0)
    oc.set("uhat", uh0)
    gtol = 1e-12
    ro = oc.newton(newton_tol=ntol, gmres_tol=gtol, precond=kind, poly_degree=deg, poly_kind=pkind, dt=dt, u_prev=u0)
    tkw = dict(dt=dt, u_prev=u0) if dt else {}
    rep = hdg.newton_solve(disc, model, state, hdg.NewtonConfig(tol=ntol), hdg.GmresConfig(tol=gtol),
                           hdg.PrecondSpec(kind, poly_degree=deg, poly_kind=pkind), **tkw)
    assert rep.converged and ro["converged"], (rep, ro)
    assert rep.n_newton == ro["n_newton"]
    assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_per_newton, ro["gmres_per_newton"])), (rep.gmres_per_newton, ro["gmres_per_newton"])
    assert relerr(state.uhat, oc.get("uhat")) < TOL
    assert relerr(state.u, oc.get("u")) < TOL
    for d in range(disc.dim):
        assert relerr(state.q(d), oc.get(f"q{d}")) < TOL
    # residual norms of the whole Newton history, relative to the initial residual
    h_gpu, h_cpu = np.array(rep.residual_history), np.array(ro["residual_history"])
    assert len(h_gpu) == len(h_cpu)
    assert np.max(np.abs(h_gpu - h_cpu)) <= TOL * h_cpu[0], (h_gpu, h_cpu)
    if deg:
        assert abs(rep.n_inner_prec_ops - ro["n_inner_prec_ops"]) <= 2 * deg * rep.n_newton


def test_config1_tight_vs_compiled_reference(ctx, ref):
    """BASELINE config 1 (2D Poisson, quads, p = 2, BJ) against the UNMODIFIED reference, both at tight tolerances,
    plus a nonlinear case (Burgers, ASM)."""
    for case, k, n, kind in (("poisson2d", 2, 16, "bj"), ("burgers2d", 2, 8, "asm")):
        rc = ref.RefCase(case, k=k, n=n)
        disc = hdg.Discretization.structured(ctx, "quad", n=n, degree=k)
        model = hdg.make_case_model(disc, case)
        state = hdg.make_initial_state(disc, model)
        rr = rc.newton(newton_tol=1e-11, gmres_tol=1e-12, precond=kind)
        rep = hdg.newton_solve(disc, model, state, hdg.NewtonConfig(tol=1e-11), hdg.GmresConfig(tol=1e-12), hdg.PrecondSpec(kind))
        assert rep.converged and rr["converged"] and rep.n_newton == rr["n_newton"]
        assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_per_newton, rr["gmres_per_newton"]))
        assert relerr(state.uhat, rc.get("uhat")) < TOL and relerr(state.u, rc.get("u")) < TOL
        h_gpu, h_cpu = np.array(rep.residual_history), np.array(rr["residual_history"])
        assert np.max(np.abs(h_gpu - h_cpu)) <= TOL * h_cpu[0]


def test_chebyshev_preconditioner_vs_tier_b(ctx):
    """Config 3's named preconditioner: the Chebyshev nodes (spec in DESIGN.md section 6; tier B restates it on the
    reference-pinned harmonic Ritz values) and the polynomial apply on them."""
    disc = hdg.Discretization.structured(ctx, "tri", n=5, degree=4, jitter=0.2, seed=12345)
    model = hdg.make_case_model(disc, "burgers")
    state = hdg.make_initial_state(disc, model)
    oc = port.OraCase(port.tables_from_disc(disc))
    oc.set_model_like(model)
    oc.set("u", state.u)
    oc.set("uhat", state.uhat)
    oc.assemble()
    ops = hdg.assemble_element_operators(disc, model, state)
    K, _ = hdg.assemble_global(disc, ops)
    y = hdg.random_vector(K.n_dof, 9)
    for kind in ("asm", "bj"):
        for pkind, deg in (("gmres", 10), ("chebyshev", 10), ("chebyshev", 5)):
            Pc = hdg.build_preconditioner(hdg.PrecondSpec(kind, poly_degree=deg, poly_kind=pkind), K, ops, disc)
            oc.build_precond(kind, poly_degree=deg, poly_kind=pkind)
            th_gpu, th_cpu = Pc.ritz, oc.ritz
            assert len(th_gpu) == len(th_cpu)
            # harmonic Ritz values: device Arnoldi + Hessenberg-QR vs the oracle's CPU Arnoldi + eigen stand-in
            assert np.max(np.abs(th_gpu - th_cpu)) <= 1e-8 * np.max(np.abs(th_cpu)), (kind, pkind, deg)
            # the apply with each side's own nodes, and with identical nodes injected
            assert relerr(Pc.apply(y), oc.apply_precond(y)) < 1e-7, (kind, pkind, deg)
            oc.set_ritz(th_gpu)
            assert relerr(Pc.apply(y), oc.apply_precond(y)) < 1e-9, (kind, pkind, deg)
