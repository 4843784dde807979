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


def test_overlapped_exchange_equals_blocking_exchange(ctx):
    """Interior rows / elements computed while the halo exchange is in flight (tuning 'overlap_halo') give bit for bit
    the operator applications of the blocking order: same kernels over sub-ranges of the same contiguous rows."""
    shape, k = "hex", 2
    gm = mesh(shape, (3, 3, 9))
    lms = P.build_local_meshes(gm, P.slab_partition(gm.ne, 3))
    assert all(lm.nf_interior > 0 and lm.ne_interior > 0 for lm in lms)
    x = hdg.random_vector(gm.nf * 9, 11).reshape(gm.nf, -1)
    out = {}
    for mode in (1, 0):
        hdg.set_tuning("overlap_halo", mode)
        lb = Loopback(lms)

        def work(r, c, lm):
            disc = P.make_discretization(c, lm, shape, k)
            model = hdg.make_case_model(disc, "poisson")
            state = hdg.make_initial_state(disc, model)
            ops = hdg.assemble_element_operators(disc, model, state)
            K, rhs = hdg.assemble_global(disc, ops)
            xl = np.full((len(lm.faces), disc.mpf), np.nan)
            xl[: lm.nf_owned] = x[lm.faces[: lm.nf_owned]]
            y = hdg.block_matvec(K, xl.ravel().copy()).reshape(len(lm.faces), -1)[: lm.nf_owned]
            Pc = hdg.build_preconditioner("asm", K, ops, disc)
            z = Pc.apply_base(xl.ravel().copy()).reshape(len(lm.faces), -1)[: lm.nf_owned]
            rep = hdg.newton_solve(disc, model, state, pspec=hdg.PrecondSpec("asm"))
            return y, z, rep.gmres_per_newton, state.uhat
        try:
            out[mode] = lb.run(work)
        finally:
            lb.close()
            hdg.set_tuning("overlap_halo", 1)
    for a, b in zip(out[1], out[0]):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert a[2] == b[2] and np.array_equal(a[3], b[3])


def test_nccl_two_stream_exchange_with_self_neighbour():
    """The NCCL exchange on its own stream (halo_begin / halo_end) exercised on ONE GPU: a 1-rank communicator whose
    only neighbour is itself (NCCL supports send / receive to self inside a group).  Owned slices must land in
    the halo part while work enqueued in between on the context's stream touches owned entries only."""
    import ctypes as C
    from paper_2512_13619_b200 import hdg as H
    L = H.load_library()
    c2 = hdg.Context(0)
    try:
        uid = (C.c_char * 128)()
        assert L.hdgb_comm_nccl_unique_id(uid) == 0
        c2.check(L.hdgb_comm_create_nccl(c2._h, bytes(uid.raw), 0, 1))
        nf_owned, n_halo, width = 1000, 37, 9
        ids = np.ascontiguousarray(np.random.default_rng(3).choice(nf_owned, n_halo, replace=False), dtype=np.int32)
        nbr, cnt, off = (np.array([v], dtype=np.int32) for v in (0, n_halo, nf_owned))  # kept alive across the call
        c2.check(L.hdgb_comm_set_halo_plan(c2._h, 1, nbr.ctypes.data, cnt.ctypes.data, ids.ctypes.data,
                                           off.ctypes.data, cnt.ctypes.data))
        vec_h = np.full((nf_owned + n_halo, width), np.nan)
        vec_h[:nf_owned] = hdg.random_vector(nf_owned * width, 8).reshape(nf_owned, width)
        vec = c2.alloc(vec_h.size)
        for rounds in range(3):                    # repeated use of the stream / events / send buffer
            c2.copy(vec, vec_h.ravel(), vec_h.size)
            c2.check(L.hdgb_halo_exchange_begin(c2._h, vec, width))
            c2.check(L.hdgb_halo_exchange_end(c2._h))
            c2.synchronize()
            back = np.empty_like(vec_h)
            c2.copy(back.ravel(), vec, vec_h.size)
            assert np.array_equal(back[:nf_owned], vec_h[:nf_owned])
            assert np.array_equal(back[nf_owned:], vec_h[ids])
            # the blocking form gives the same
            c2.copy(vec, vec_h.ravel(), vec_h.size)
            c2.check(L.hdgb_halo_exchange(c2._h, vec, width))
            c2.copy(back.ravel(), vec, vec_h.size)
            assert np.array_equal(back[nf_owned:], vec_h[ids])
        c2.free(vec)
    finally:
        L.hdgb_comm_destroy(c2._h)
        c2.close()
