"""Compressible Navier-Stokes (M = D + 2 component blocks: BASELINE config 5 in miniature) against the
tier-B CPU restatement: raw and condensed blocks, block-Jacobi GMRES, one backward-Euler Newton step.
The model has no reference implementation; physics sanity = free-stream
preservation and a Newton iteration that converges at the rate an exact Jacobian gives."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg
from oracle import port

pytestmark = pytest.mark.gpu


def relerr(a, b):
    return np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b)))


def setup(ctx, shape, n, k, mu=0.02):
    D = 3 if shape in ("hex", "tet") else 2
    disc = hdg.Discretization.structured(ctx, shape, n=n, degree=k, n_comp=D + 2)
    model = hdg.make_case_model(disc, "navier_stokes", mu=mu)
    state = hdg.make_initial_state(disc, model)
    oc = port.OraCase(port.tables_from_disc(disc))
    oc.set_model_like(model)
    oc.set("u", state.u)
    oc.set("uhat", state.uhat)
    return disc, model, state, oc


@pytest.mark.parametrize("shape", ["quad", "hex", "tet"])
def test_free_stream_is_preserved(ctx, shape):
    D = 3 if shape in ("hex", "tet") else 2
    disc = hdg.Discretization.structured(ctx, shape, n=2, degree=2, n_comp=D + 2, jitter=0.1)
    gamma = 1.4
    uinf = np.array([1.2] + [0.3, -0.2, 0.1][:D] + [1.0 / (gamma - 1.0) + 0.6 * 0.5 * 1.2], dtype=float)
    const = lambda x: np.broadcast_to(uinf, x.shape[:-1] + (D + 2,))
    model = hdg.Model(disc, "navier_stokes", [gamma, 0.05, 0.71, 3.0], dirichlet=const, initial=const)
    state = hdg.make_initial_state(disc, model)
    tr, it, nrm = hdg.assemble_residual(disc, model, state)
    assert nrm < 1e-11
    assert np.max(np.abs(state.q(0))) < 1e-11            # zero gradient of a constant state


@pytest.mark.parametrize("shape,n,k", [("quad", 3, 2), ("hex", 2, 1), ("hex", 2, 2), ("tet", 1, 2)])
def test_operators_vs_tier_b(ctx, shape, n, k):
    disc, model, state, oc = setup(ctx, shape, n, k)
    u = state.u * (1.0 + 0.01 * hdg.random_vector(disc.npe * disc.ne, 5))
    uh = state.uhat * (1.0 + 0.01 * hdg.random_vector(disc.n_dof, 6))
    state.u, state.uhat = u, uh
    oc.set("u", u)
    oc.set("uhat", uh)
    oc.assemble()
    ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True)
    for nm in ["e_raw", "f_raw", "h_raw", "j_raw", "ru", "ruhat_e"] + [f"d_raw{d}" for d in range(disc.dim)] + \
              [f"g_raw{d}" for d in range(disc.dim)]:
        assert relerr(ops.get(nm), oc.get(nm)) < 1e-11, nm
    for nm in ("kbar", "rbar", "fbar", "hbar"):
        assert relerr(ops.get(nm), oc.get(nm)) < 1e-8, nm
    K, rhs = hdg.assemble_global(disc, ops)
    assert np.array_equal(K.neighbor, oc.neighbor)
    assert relerr(K.blocks, oc.get("blocks")) < 1e-8 and relerr(rhs, oc.get("rhs")) < 1e-8
    x = hdg.random_vector(K.n_dof, 1)
    assert relerr(hdg.block_matvec(K, x), oc.matvec(x)) < 1e-8
    P = hdg.build_preconditioner("bj", K, ops, disc)
    oc.build_precond("bj")
    assert relerr(P.apply_base(x), oc.apply_base(x)) < 1e-7


@pytest.mark.parametrize("shape,n,k", [("quad", 4, 2), ("hex", 2, 2)])
def test_backward_euler_newton_step_vs_tier_b(ctx, shape, n, k):
    disc, model, state, oc = setup(ctx, shape, n, k)
    dt = 0.02
    u0 = state.u
    oc.set_dt(dt, u0)
    ro = oc.newton(precond="bj", gmres_tol=1e-8)
    rep = hdg.newton_solve(disc, model, state, gcfg=hdg.GmresConfig(tol=1e-8), pspec=hdg.PrecondSpec("bj"), dt=dt, u_prev=u0)
    assert rep.converged and ro["converged"]
    assert rep.n_newton == ro["n_newton"]
    assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_per_newton, ro["gmres_per_newton"]))
    assert relerr(state.u, oc.get("u")) < 1e-7 and relerr(state.uhat, oc.get("uhat")) < 1e-7
    # an exact Jacobian: the nonlinear residual collapses by orders of magnitude per step
    h = rep.residual_history
    assert h[1] < 1e-2 * h[0] and h[-1] <= 1e-8
