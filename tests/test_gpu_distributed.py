"""Domain-decomposed solver on ONE GPU with several virtual ranks (tests/loopback.py): the partitioned
run must reproduce the single-domain run -- same block rows, same iteration counts (+-1), same
solution on every owned face -- for BJ, ASM and the polynomial wrapper."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg
from paper_2512_13619_b200 import partition as P
from loopback import Loopback

pytestmark = pytest.mark.gpu


def mesh(shape, dims):
    if shape == "hex":
        lo, hi = (0, 0, 0), (1, 1, 1)
        coords, ev = P.box_hex_mesh(*dims, lo, hi)
    else:
        lo, hi = (0, 0), (1, 1)
        coords, ev = P.box_quad_mesh(*dims, lo, hi)
    return P.global_mesh(shape, coords, ev, lo=lo, hi=hi)


def single(ctx, gm, shape, k, case, pspec, gcfg):
    one = P.build_local_meshes(gm, np.zeros(gm.ne, dtype=np.int32))[0]
    disc = P.make_discretization(ctx, one, shape, k)
    model = hdg.make_case_model(disc, case)
    state = hdg.make_initial_state(disc, model)
    rep = hdg.newton_solve(disc, model, state, gcfg=gcfg, pspec=pspec)
    return rep, state.uhat.reshape(gm.nf, -1), state.u.reshape(gm.ne, -1), disc, model


@pytest.mark.parametrize("shape,dims,k,case,kind,deg,nr", [
    ("quad", (6, 6), 2, "poisson", "bj", 0, 2),
    ("quad", (8, 6), 1, "burgers", "asm", 0, 3),
    ("hex", (3, 3, 4), 2, "poisson", "asm", 0, 2),
    ("hex", (2, 2, 6), 1, "poisson", "asm", 4, 3),
    ("quad", (8, 8), 2, "burgers", "bj", 6, 4),
])
def test_partitioned_newton_matches_single_domain(ctx, shape, dims, k, case, kind, deg, nr):
    gm = mesh(shape, dims)
    pspec = hdg.PrecondSpec(kind, poly_degree=deg)
    gcfg = hdg.GmresConfig(tol=1e-9)
    rep1, uh1, u1, _, _ = single(ctx, gm, shape, k, case, pspec, gcfg)
    lms = P.build_local_meshes(gm, P.slab_partition(gm.ne, nr))
    lb = Loopback(lms)

    def work(r, c, lm):
        disc = P.make_discretization(c, lm, shape, k)
        model = hdg.make_case_model(disc, case)
        state = hdg.make_initial_state(disc, model)
        rep = hdg.newton_solve(disc, model, state, gcfg=gcfg, pspec=pspec)
        return rep, state.uhat.reshape(len(lm.faces), -1), state.u.reshape(len(lm.elems), -1)

    try:
        res = lb.run(work)
    finally:
        lb.close()
    for (rep, uh, u), lm in zip(res, lms):
        assert rep.converged and rep.n_newton == rep1.n_newton
        assert all(abs(a - b) <= 1 for a, b in zip(rep.gmres_per_newton, rep1.gmres_per_newton))
        assert abs(rep.final_residual - rep1.final_residual) <= 1e-9 * max(1.0, rep1.residual_history[0])
        scale = max(1.0, np.max(np.abs(uh1)))
        assert np.max(np.abs(uh[: lm.nf_owned] - uh1[lm.faces[: lm.nf_owned]])) < 1e-7 * scale
        # halo faces and ghost elements are kept consistent too (redundant recovery)
        assert np.max(np.abs(uh - uh1[lm.faces])) < 1e-7 * scale
        assert np.max(np.abs(u - u1[lm.elems])) < 1e-7 * max(1.0, np.max(np.abs(u1)))


def test_partitioned_operator_rows_and_preconditioners(ctx):
    shape, k = "hex", 2
    gm = mesh(shape, (3, 2, 4))
    rep1, uh1, u1, d1, m1 = single(ctx, gm, shape, k, "poisson", hdg.PrecondSpec("bj"), hdg.GmresConfig())
    s1 = hdg.make_initial_state(d1, m1)
    ops1 = hdg.assemble_element_operators(d1, m1, s1)
    K1, rhs1 = hdg.assemble_global(d1, ops1)
    B1 = K1.blocks.reshape(gm.nf, -1)
    x = hdg.random_vector(gm.nf * d1.mpf, 3).reshape(gm.nf, -1)
    y1 = hdg.block_matvec(K1, x.ravel()).reshape(gm.nf, -1)
    z1 = {kind: hdg.build_preconditioner(kind, K1, ops1, d1).apply_base(x.ravel()).reshape(gm.nf, -1) for kind in ("bj", "asm")}
    lms = P.build_local_meshes(gm, P.slab_partition(gm.ne, 3))
    lb = Loopback(lms)

    def work(r, c, lm):
        disc = P.make_discretization(c, lm, shape, k)
        model = hdg.make_case_model(disc, "poisson")
        state = hdg.make_initial_state(disc, model)
        ops = hdg.assemble_element_operators(disc, model, state)
        K, rhs = hdg.assemble_global(disc, ops)
        xl = np.full((len(lm.faces), disc.mpf), np.nan)
        xl[: lm.nf_owned] = x[lm.faces[: lm.nf_owned]]          # halo part must come from the exchange
        y = hdg.block_matvec(K, xl.ravel()).reshape(len(lm.faces), -1)
        z = {}
        for kind in ("bj", "asm"):
            Pc = hdg.build_preconditioner(kind, K, ops, disc)
            xl2 = xl.copy()
            z[kind] = Pc.apply_base(xl2.ravel()).reshape(len(lm.faces), -1)
        return K.blocks.reshape(lm.nf_owned, -1), rhs.reshape(len(lm.faces), -1), y, z

    try:
        res = lb.run(work)
    finally:
        lb.close()
    for (B, rhs, y, z), lm in zip(res, lms):
        own = lm.faces[: lm.nf_owned]
        assert np.max(np.abs(B - B1[own])) < 1e-12 * max(1.0, np.max(np.abs(B1)))
        assert np.max(np.abs(rhs[: lm.nf_owned] - rhs1.reshape(gm.nf, -1)[own])) < 1e-12
        assert np.max(np.abs(y[: lm.nf_owned] - y1[own])) < 1e-12 * max(1.0, np.max(np.abs(y1)))
        for kind in ("bj", "asm"):
            assert np.max(np.abs(z[kind][: lm.nf_owned] - z1[kind][own])) < 1e-10 * max(1.0, np.max(np.abs(z1[kind]))), kind


def test_nccl_backend_single_rank(ctx):
    """The NCCL transport itself (dlopen of libnccl.so.2, ncclCommInitRank, all-reduce, empty halo
    plan) on the one GPU this box has: a 1-rank job must reproduce the communicator-free run."""
    import ctypes as C
    from paper_2512_13619_b200 import hdg as H
    gm = mesh("quad", (6, 5))
    lm = P.build_local_meshes(gm, np.zeros(gm.ne, dtype=np.int32))[0]
    c2 = hdg.Context(0)
    try:
        P.install_nccl_comm(c2, lm, None)
        L = H.load_library()
        assert L.hdgb_comm_size(c2._h) == 1 and L.hdgb_comm_rank(c2._h) == 0
        buf = c2.alloc(4)
        c2.copy(buf, np.array([1.0, 2.0, 3.0, 4.0]), 4)
        c2.check(L.hdgb_allreduce_sum(c2._h, buf, 4))
        back = np.empty(4)
        c2.copy(back, buf, 4)
        c2.free(buf)
        assert np.array_equal(back, [1.0, 2.0, 3.0, 4.0])
        out = []
        for cc in (ctx, c2):
            disc = P.make_discretization(cc, lm, "quad", 2)
            model = hdg.make_case_model(disc, "burgers")
            state = hdg.make_initial_state(disc, model)
            rep = hdg.newton_solve(disc, model, state, pspec=hdg.PrecondSpec("asm", poly_degree=4))
            out.append((rep, state.uhat))
        assert out[0][0].gmres_per_newton == out[1][0].gmres_per_newton
        assert np.array_equal(out[0][1], out[1][1])
    finally:
        H.load_library().hdgb_comm_destroy(c2._h)
        c2.close()
