"""BASELINE.json configurations 2-5 at FULL size on the GPU, checked through size-independent properties (the CPU
oracle cannot run these sizes in seconds; the miniature versions against the oracle are in
test_gpu_baseline_configs.py):
  * structure: neighbour table (slot 0 = self, boundary faces keep -1 in the side-1 slots, adjacency symmetric),
  * assembly consistency: block_matvec(K, x) == face-sum over elements of K-bar^e x^e (face_matrix.cpp:11-61 vs
    local_ops.cpp:408-411) -- the assembled rows are exactly the scattered element blocks,
  * linearity of matvec and preconditioner apply (the condensed system of the reference's flux formulation is
    not symmetric, so no symmetry property is claimed),
  * explicit inverses: (block-Jacobi block)^-1 block = I on sampled blocks,
  * the solve: converged, residual below tolerance, discretisation error at the expected level, and idempotence
    (a second solve from the solution takes zero Newton iterations)."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg

pytestmark = pytest.mark.gpu

FULL = {
    2: dict(shape="hex", n=28, degree=3, n_comp=1, case="poisson", precond="asm", solve=True, jitter=0.0,
            expect=dict(n_newton=2, gmres=(130, 150), l2=(5e-8, 9e-8))),
    3: dict(shape="tri", n=512, degree=4, n_comp=1, case="burgers", precond="asm", solve=False, jitter=0.2),
    4: dict(shape="tet", n=32, degree=2, n_comp=3, case="elasticity", precond="asm", solve=False, jitter=0.2),
    # SURVEY.md section 8 size table: hex 24^3 (K = 24.3 GB, ~100 GB of operators in total; 16^3 was the round-1 smoke size)
    5: dict(shape="hex", n=24, degree=3, n_comp=5, case="navier_stokes", precond="bj", solve=True, jitter=0.0,
            dt=0.01, expect=dict(n_newton=2, gmres=(112, 136))),
}


def setup(ctx, cfg):
    disc = hdg.Discretization.structured(ctx, cfg["shape"], n=cfg["n"], degree=cfg["degree"], n_comp=cfg["n_comp"],
                                         jitter=cfg["jitter"])
    kw = {"mu": 0.02} if cfg["case"] == "navier_stokes" else {}
    model = hdg.make_case_model(disc, cfg["case"], **kw)
    state = hdg.make_initial_state(disc, model)
    return disc, model, state


@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_full_size_operator_properties(ctx, cid):
    cfg = FULL[cid]
    disc, model, state = setup(ctx, cfg)
    tkw = dict(dt=cfg["dt"], u_prev=state.u) if cfg.get("dt") else {}
    ops = hdg.assemble_element_operators(disc, model, state, **tkw)
    K, rhs = hdg.assemble_global(disc, ops)
    nf, ne, mpf, nfl, n_lfe, nb, npe = disc.nf, disc.ne, disc.mpf, disc.nfl, disc.n_lfe, disc.nb, disc.npe
    n = K.n_dof
    assert n == nf * mpf == disc.n_dof

    # ---- structure (bit-exact index work) ----
    nbr = K.neighbor.reshape(nf, nb)
    assert np.array_equal(nbr[:, 0], np.arange(nf))
    f2e = disc.table("face_to_elements").reshape(nf, 2)
    boundary = f2e[:, 1] < 0
    assert np.all(nbr[boundary, n_lfe:] == -1) and np.all(nbr[~boundary] >= 0) and np.all(nbr[:, :n_lfe] >= 0)
    e2f = disc.table("element_to_face").reshape(ne, n_lfe)
    assert np.array_equal(np.sort(np.bincount(e2f.ravel(), minlength=nf)), np.sort(2 - boundary.astype(np.int64)))
    # adjacency is symmetric: g appears in row f as often as f appears in row g
    rows = np.repeat(np.arange(nf), nb - 1)
    cols = nbr[:, 1:].ravel()
    ok = cols >= 0
    fwd = np.sort(rows[ok].astype(np.int64) * nf + cols[ok])
    bwd = np.sort(cols[ok].astype(np.int64) * nf + rows[ok])
    assert np.array_equal(fwd, bwd)

    # ---- assembled rows == scattered element blocks ----
    rng = np.random.default_rng(cid)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    Kx = hdg.block_matvec(K, x)
    xe = hdg.gather_element_trace(disc, x)                                     # (ne, nfl) element-local traces
    ye = hdg.gemv_strided_batch(ctx, ops.ptr("kbar"), nfl, nfl, ne, xe)        # K-bar^e x^e on the device blocks
    acc = np.zeros((nf, mpf))
    np.add.at(acc, e2f.ravel(), ye.reshape(ne * n_lfe, mpf))
    scale = np.max(np.abs(Kx))
    assert np.max(np.abs(acc.ravel() - Kx)) <= 1e-12 * scale

    # ---- linearity ----
    Ky = hdg.block_matvec(K, y)
    assert np.max(np.abs(hdg.block_matvec(K, 2.0 * x - 3.0 * y) - (2.0 * Kx - 3.0 * Ky))) <= 1e-12 * scale
    P = hdg.build_preconditioner(cfg["precond"], K, ops, disc)
    Px, Py = P.apply_base(x), P.apply_base(y)
    pscale = np.max(np.abs(Px))
    assert np.max(np.abs(P.apply_base(2.0 * x - 3.0 * y) - (2.0 * Px - 3.0 * Py))) <= 1e-11 * pscale

    # ---- explicit inverses on sampled blocks ----
    if cfg["precond"] == "bj":
        # (sampled straight from device memory: the whole K is 24 GB at config 5)
        inv = P.get("bj_inv").reshape(nf, mpf, mpf)
        for f in (0, nf // 3, nf - 1):
            blk = np.empty(mpf * mpf)
            ctx.copy(blk, K.blocks_ptr() + 8 * f * mpf * mpf * nb, blk.size)      # slot-0 block of row f, column-major
            d = blk.reshape(mpf, mpf).T
            assert np.max(np.abs(inv[f].T @ d - np.eye(mpf))) <= 1e-9


@pytest.mark.parametrize("cid", [2, 5])
def test_full_size_solve(ctx, cid):
    cfg = FULL[cid]
    disc, model, state = setup(ctx, cfg)
    u0 = state.u
    tkw = dict(dt=cfg["dt"], u_prev=u0) if cfg.get("dt") else {}
    pspec = hdg.PrecondSpec(cfg["precond"])
    rep = hdg.newton_solve(disc, model, state, pspec=pspec, **tkw)
    ex = cfg["expect"]
    assert rep.converged and rep.n_newton == ex["n_newton"] and rep.final_residual <= 1e-8
    assert ex["gmres"][0] <= rep.n_gmres_total <= ex["gmres"][1]
    _, _, nrm = hdg.assemble_residual(disc, model, state, **tkw)
    assert abs(nrm - rep.final_residual) <= 1e-12 + 1e-6 * rep.final_residual
    if "l2" in ex:
        err = disc.l2_error(state.u, model.exact_solution)
        assert ex["l2"][0] <= err <= ex["l2"][1]
    # idempotence: the solution is a fixed point of the solver
    rep2 = hdg.newton_solve(disc, model, state, pspec=pspec, **tkw)
    assert rep2.converged and rep2.n_newton == 0 and rep2.n_gmres_total == 0


def test_full_size_assembly_bitwise_reproducible(ctx):
    """Config 2 at full size, repeated: the condensed operators and the Newton / GMRES trace must not depend on timing.
    (The local kernel's TMA table ring once released a stage while shared-memory loads of it were still queued --
    tma.cuh: ring_release_all -- which corrupted one 8 x 8 tile in ~3e5 elements, only at this scale: 21 952 CTAs, two per SM.)"""
    import hashlib
    cfg = FULL[2]
    disc, model, state = setup(ctx, cfg)
    rng = np.random.default_rng(1)
    state.u = state.u + 0.1 * rng.standard_normal(state.u.shape)
    state.uhat = state.uhat + 0.1 * rng.standard_normal(state.uhat.shape)
    digests = set()
    for _ in range(16):
        ops = hdg.assemble_element_operators(disc, model, state)
        digests.add(hashlib.sha1(ops.get("kbar").tobytes()).hexdigest())
        del ops
    assert len(digests) == 1
    disc, model, state = setup(ctx, cfg)
    u0, uh0 = state.u, state.uhat
    traces = set()
    for _ in range(3):
        state.set("u", u0)
        state.set("uhat", uh0)
        rep = hdg.newton_solve(disc, model, state, hdg.NewtonConfig(), hdg.GmresConfig(), hdg.PrecondSpec(cfg["precond"]))
        traces.add((rep.n_gmres_total, tuple(rep.residual_history)))
    assert len(traces) == 1
