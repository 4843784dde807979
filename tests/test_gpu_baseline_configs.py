"""The five BASELINE.json configurations in miniature (config 1 at full size lives in
tests/test_gpu_golden.py), each solved end to end through the public API and checked against the CPU
oracle / a single-domain run."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg
from oracle import port
from paper_2512_13619_b200 import partition as P
from loopback import Loopback

pytestmark = pytest.mark.gpu


def relerr(a, b):
    return np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b)))


def oracle_for(disc, model, state):
    oc = port.OraCase(port.tables_from_disc(disc))
    oc.set_model_like(model)
    oc.set("u", state.u)
    oc.set("uhat", state.uhat)
    return oc


@pytest.mark.parametrize("kind", ["asm", "ras"])
def test_config2_hex_p3_poisson_additive_schwarz(ctx, kind):
    """configs[1]: 3D Poisson, structured hex, p = 3, (restricted) additive Schwarz GMRES."""
    disc = hdg.Discretization.structured(ctx, "hex", n=3, degree=3)
    model = hdg.make_case_model(disc, "poisson")
    state = hdg.make_initial_state(disc, model)
    oc = oracle_for(disc, model, state)
    ro = oc.newton(precond=kind)
    rep = hdg.newton_solve(disc, model, state, pspec=hdg.PrecondSpec(kind))
    assert rep.converged and rep.n_newton == ro["n_newton"]
    assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_per_newton, ro["gmres_per_newton"]))
    assert relerr(state.uhat, oc.get("uhat")) < 1e-6
    assert abs(rep.final_residual - ro["final_residual"]) < 1e-10 * max(1.0, ro["residual_history"][0])


def test_config3_triangles_p4_burgers_polynomial_preconditioners(ctx):
    """configs[2]: 2D viscous Burgers, (jittered) triangle mesh, p = 4, Newton-GMRES with a polynomial
    preconditioner -- the reference's GMRES (harmonic-Ritz / Leja) polynomial and the Chebyshev variant."""
    disc = hdg.Discretization.structured(ctx, "tri", n=6, degree=4, jitter=0.2, seed=12345)
    model = hdg.make_case_model(disc, "burgers")
    sols, reps = {}, {}
    for name, spec in [("asm", hdg.PrecondSpec("asm")), ("gmres-poly", hdg.PrecondSpec("asm", poly_degree=10)),
                       ("chebyshev", hdg.PrecondSpec("asm", poly_degree=10, poly_kind="chebyshev"))]:
        state = hdg.make_initial_state(disc, model)
        reps[name] = hdg.newton_solve(disc, model, state, pspec=spec)
        sols[name] = state.uhat
        assert reps[name].converged, name
    # the converged trace does not depend on the preconditioner (test_newton.cpp:128-147, 1e-6 max-norm)
    assert np.max(np.abs(sols["gmres-poly"] - sols["asm"])) < 1e-6
    assert np.max(np.abs(sols["chebyshev"] - sols["asm"])) < 1e-6
    # acceptance_main.cpp:415-424 ordering: the polynomial wrapper cuts the outer iteration count
    assert reps["gmres-poly"].n_gmres_total < reps["asm"].n_gmres_total
    assert reps["chebyshev"].n_gmres_total < reps["asm"].n_gmres_total
    assert reps["gmres-poly"].n_inner_prec_ops > 0
    # the polynomial apply itself against the oracle recurrence with identical interpolation nodes
    state = hdg.make_initial_state(disc, model)
    oc = oracle_for(disc, model, state)
    oc.assemble()
    oc.build_precond("asm")
    ops = hdg.assemble_element_operators(disc, model, state)
    K, _ = hdg.assemble_global(disc, ops)
    Pc = hdg.build_preconditioner(hdg.PrecondSpec("asm", poly_degree=8), K, ops, disc)
    oc.set_ritz(Pc.ritz)
    y = hdg.random_vector(K.n_dof, 9)
    assert relerr(Pc.apply(y), oc.apply_precond(y)) < 1e-8


@pytest.mark.parametrize("nr", [2, 4, 8])
def test_config4_tets_p2_elasticity_asm_partitioned(ctx, nr):
    """configs[3]: 3D linear elasticity, tetrahedra, p = 2 (3-component blocks), additive Schwarz,
    partitioned across ranks -- must reproduce the single-domain run."""
    lo, hi = (0, 0, 0), (1, 1, 1)
    d0 = hdg.Discretization.structured(None, "tet", n=2, degree=1)
    gm = P.global_mesh("tet", d0.table("vertex_coords").reshape(-1, 3), d0.table("element_vertices").reshape(d0.ne, 4), lo=lo, hi=hi)
    pspec, gcfg = hdg.PrecondSpec("asm"), hdg.GmresConfig(tol=1e-9)
    one = P.build_local_meshes(gm, np.zeros(gm.ne, dtype=np.int32))[0]
    disc = P.make_discretization(ctx, one, "tet", 2, n_comp=3)
    model = hdg.make_case_model(disc, "elasticity")
    state = hdg.make_initial_state(disc, model)
    oc = oracle_for(disc, model, state)
    rep1 = hdg.newton_solve(disc, model, state, gcfg=gcfg, pspec=pspec)
    ro = oc.newton(precond="asm", gmres_tol=1e-9)
    assert rep1.converged and rep1.n_newton == ro["n_newton"]
    assert all(abs(a - b) <= 1 for a, b in zip(rep1.gmres_per_newton, ro["gmres_per_newton"]))
    uh1 = state.uhat.reshape(gm.nf, -1)
    assert relerr(uh1.ravel(), oc.get("uhat")) < 1e-7
    lms = P.build_local_meshes(gm, P.slab_partition(gm.ne, nr))
    lb = Loopback(lms)

    def work(r, c, lm):
        dl = P.make_discretization(c, lm, "tet", 2, n_comp=3)
        ml = hdg.make_case_model(dl, "elasticity")
        sl = hdg.make_initial_state(dl, ml)
        return hdg.newton_solve(dl, ml, sl, gcfg=gcfg, pspec=pspec), sl.uhat.reshape(len(lm.faces), -1)

    try:
        res = lb.run(work)
    finally:
        lb.close()
    for (rep, uh), lm in zip(res, lms):
        assert rep.converged and rep.n_newton == rep1.n_newton
        assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_per_newton, rep1.gmres_per_newton))
        assert np.max(np.abs(uh[: lm.nf_owned] - uh1[lm.faces[: lm.nf_owned]])) < 1e-7 * max(1.0, np.max(np.abs(uh1)))


@pytest.mark.parametrize("dims,nr", [((2, 2, 2), 2), ((2, 2, 8), 8)])
def test_config5_hex_navier_stokes_bj_partitioned(ctx, dims, nr):
    """configs[4]: 3D compressible Navier-Stokes, hex, 5-component blocks, Newton-GMRES with block-Jacobi,
    one backward-Euler step, partitioned over 2 / 8 ranks (BASELINE: strong scaling 1/2/4/8) vs single domain."""
    lo, hi = (0, 0, 0), (1, 1, 1)
    coords, ev = P.box_hex_mesh(*dims, lo, hi)
    gm = P.global_mesh("hex", coords, ev, lo=lo, hi=hi)
    pspec, gcfg, dt = hdg.PrecondSpec("bj"), hdg.GmresConfig(tol=1e-8), 0.02
    one = P.build_local_meshes(gm, np.zeros(gm.ne, dtype=np.int32))[0]
    disc = P.make_discretization(ctx, one, "hex", 2, n_comp=5)
    model = hdg.make_case_model(disc, "navier_stokes", mu=0.02)
    state = hdg.make_initial_state(disc, model)
    rep1 = hdg.newton_solve(disc, model, state, gcfg=gcfg, pspec=pspec, dt=dt, u_prev=state.u)
    assert rep1.converged
    uh1 = state.uhat.reshape(gm.nf, -1)
    lms = P.build_local_meshes(gm, P.slab_partition(gm.ne, nr))
    lb = Loopback(lms)

    def work(r, c, lm):
        dl = P.make_discretization(c, lm, "hex", 2, n_comp=5)
        ml = hdg.make_case_model(dl, "navier_stokes", mu=0.02)
        sl = hdg.make_initial_state(dl, ml)
        return hdg.newton_solve(dl, ml, sl, gcfg=gcfg, pspec=pspec, dt=dt, u_prev=sl.u), sl.uhat.reshape(len(lm.faces), -1)

    try:
        res = lb.run(work)
    finally:
        lb.close()
    for (rep, uh), lm in zip(res, lms):
        assert rep.converged and rep.n_newton == rep1.n_newton
        assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_per_newton, rep1.gmres_per_newton))
        assert np.max(np.abs(uh[: lm.nf_owned] - uh1[lm.faces[: lm.nf_owned]])) < 1e-7 * max(1.0, np.max(np.abs(uh1)))
