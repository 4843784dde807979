"""Host logic of the domain decomposition (partitioner, ghost layer, face ownership, halo plan) on the
CPU: structural invariants in-process, and the N > 1 path with two real processes over gloo."""
import os
import socket

import numpy as np
import pytest

from paper_2512_13619_b200 import hdg as H
from paper_2512_13619_b200 import partition as P


def small_mesh(shape):
    if shape == "hex":
        lo, hi = (0, 0, 0), (1, 1, 1)
        coords, ev = P.box_hex_mesh(3, 2, 4, lo, hi)
    else:
        lo, hi = (0, 0), (1, 1)
        coords, ev = P.box_quad_mesh(5, 6, lo, hi)
    return P.global_mesh(shape, coords, ev, lo=lo, hi=hi)


@pytest.mark.parametrize("shape,nr", [("quad", 2), ("quad", 3), ("hex", 2), ("hex", 4)])
def test_partition_invariants(shape, nr):
    gm = small_mesh(shape)
    part = P.slab_partition(gm.ne, nr)
    lms = P.build_local_meshes(gm, part)
    owned_f = np.concatenate([lm.faces[: lm.nf_owned] for lm in lms])
    assert np.array_equal(np.sort(owned_f), np.arange(gm.nf))               # every face owned exactly once
    owned_e = np.concatenate([lm.elems[: lm.ne_owned] for lm in lms])
    assert np.array_equal(np.sort(owned_e), np.arange(gm.ne))
    for lm in lms:
        # ownership rule: the rank of the side-0 element (mesh.cpp:63-71)
        assert np.all(part[gm.f2e[lm.faces[: lm.nf_owned], 0]] == lm.rank)
        # an owned face finds both adjacent elements, hence its whole block row, locally
        f2e = lm.f2e[: lm.nf_owned]
        assert np.all(f2e[:, 0] >= 0) and np.all(f2e[:, 1] != -2)
        assert np.array_equal(f2e[:, 1] == -1, gm.f2e[lm.faces[: lm.nf_owned], 1] == -1)
        # halo faces are grouped by owner, ascending global id inside a group
        ho, hf = lm.face_owner[lm.nf_owned:], lm.faces[lm.nf_owned:]
        assert np.all(np.diff(ho) >= 0)
        for s in np.unique(ho):
            assert np.all(np.diff(hf[ho == s]) > 0)
        # global orientation flags / local indices survive the cut
        assert np.array_equal(lm.forient, gm.forient[lm.faces])
        assert np.array_equal(lm.tags, gm.tags[lm.faces])
        # send / receive sides of the plan match pairwise
        for k, s in enumerate(lm.nbr_ranks):
            other = lms[int(s)]
            j = list(other.nbr_ranks).index(lm.rank)
            sent_gids = other.faces[other.send_ids[j]]
            recv_gids = lm.faces[lm.recv_off[k]: lm.recv_off[k] + lm.recv_cnt[k]]
            assert np.array_equal(sent_gids, recv_gids)


@pytest.mark.parametrize("shape,dims,nr", [("quad", (8, 9), 2), ("quad", (6, 12), 3), ("hex", (3, 3, 8), 2), ("hex", (2, 3, 12), 3)])
def test_interior_first_numbering_and_overlap_window(shape, dims, nr):
    """The overlap window of the halo exchange: interior elements / faces are numbered first, their rows reference
    owned faces only, and the library (host-only discretisation) finds exactly the partitioner's counts."""
    lo, hi = ((0, 0, 0), (1, 1, 1)) if shape == "hex" else ((0, 0), (1, 1))
    coords, ev = (P.box_hex_mesh if shape == "hex" else P.box_quad_mesh)(*dims, lo, hi)
    gm = P.global_mesh(shape, coords, ev, lo=lo, hi=hi)
    lms = P.build_local_meshes(gm, P.slab_partition(gm.ne, nr))
    for lm in lms:
        assert 0 < lm.ne_interior <= lm.ne_owned and 0 < lm.nf_interior <= lm.nf_owned
        # interior elements touch owned faces only; the first non-interior owned element touches a halo face
        assert np.all(lm.e2f[: lm.ne_interior] < lm.nf_owned)
        if lm.ne_interior < lm.ne_owned:
            assert np.all(np.any(lm.e2f[lm.ne_interior: lm.ne_owned] >= lm.nf_owned, axis=1))
        # the block row of an interior face (all faces of both adjacent elements) stays inside the owned range
        for f in range(lm.nf_owned):
            row = np.concatenate([lm.e2f[e] for e in lm.f2e[f] if e >= 0])
            assert (f < lm.nf_interior) == bool(np.all(row < lm.nf_owned)), f
        # ids ascend inside each group (the single-domain order is kept where it can be)
        for a, b in ((0, lm.nf_interior), (lm.nf_interior, lm.nf_owned)):
            assert np.all(np.diff(lm.faces[a:b]) > 0)
        for a, b in ((0, lm.ne_interior), (lm.ne_interior, lm.ne_owned)):
            assert np.all(np.diff(lm.elems[a:b]) > 0)
        d = P.make_discretization(None, lm, shape, 1)
        assert (d.ne_interior, d.nf_interior) == (lm.ne_interior, lm.nf_interior)
        d.close()
    # one rank: everything is owned, nothing to overlap
    one = P.build_local_meshes(gm, np.zeros(gm.ne, dtype=np.int32))[0]
    d = P.make_discretization(None, one, shape, 1)
    assert (d.ne_interior, d.nf_interior) == (0, 0)
    d.close()


def test_box_tags_match_structured_builder():
    gm = small_mesh("quad")
    d = H.Discretization.structured(None, "quad", n=4, degree=1)
    coords, ev = P.box_quad_mesh(4, 4)
    g4 = P.global_mesh("quad", coords, ev, lo=(0, 0), hi=(1, 1))
    # same faces (as vertex sets) carry the same tags as build_structured_quad's (mesh.cpp:72-73,89-90)
    key = lambda fv: {tuple(sorted(v)): i for i, v in enumerate(fv)}
    a = key(d.table("face_vertices").reshape(-1, 2))
    b = key(g4.fverts)
    ta = d.table("boundary_tag")
    for k, i in a.items():
        assert ta[i] == g4.tags[b[k]]
    assert gm.tags.max() == 4


def test_local_tables_reproduce_global_geometry():
    """Host-only discretisations of the sub-domains: geometry of every local face / element equals the
    global mesh's (same canonical orientation => same quadrature point order, same normals)."""
    gm = small_mesh("hex")
    coords, ev = gm.coords, gm.elem_verts
    # the global tables through the same entry point, as one "rank"
    one = P.build_local_meshes(gm, np.zeros(gm.ne, dtype=np.int32))[0]
    dg = P.make_discretization(None, one, "hex", 2)
    fcg = dg.table("face_coords").reshape(gm.nf, -1)
    fng = dg.table("face_normal").reshape(gm.nf, 2, -1)
    ecg = dg.table("elem_coords").reshape(gm.ne, -1)
    for lm in P.build_local_meshes(gm, P.slab_partition(gm.ne, 3)):
        dl = P.make_discretization(None, lm, "hex", 2)
        assert np.array_equal(dl.table("face_coords").reshape(len(lm.faces), -1), fcg[lm.faces])
        assert np.array_equal(dl.table("elem_coords").reshape(len(lm.elems), -1), ecg[lm.elems])
        fnl = dl.table("face_normal").reshape(len(lm.faces), 2, -1)
        for s in range(2):
            have = lm.f2e[:, s] >= 0
            assert np.array_equal(fnl[have, s], fng[lm.faces[have], s])


def _gloo_worker(rank, world, port, ret):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gm = small_mesh("hex")
        part = P.slab_partition(gm.ne, world)
        lm = P.build_my_local_mesh(gm, part, rank, dist)          # send lists via all_gather_object
        width = 3
        vec = np.full((len(lm.faces), width), np.nan)
        gid = lm.faces[: lm.nf_owned]
        vec[: lm.nf_owned] = gid[:, None] * 10.0 + np.arange(width)[None, :]
        # the halo exchange of the plan, carried by gloo point-to-point messages
        import torch
        reqs, recv_bufs = [], []
        for k, s in enumerate(lm.nbr_ranks):
            if len(lm.send_ids[k]):
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(vec[lm.send_ids[k]])), int(s)))
            if lm.recv_cnt[k]:
                buf = torch.empty(int(lm.recv_cnt[k]), width, dtype=torch.float64)
                recv_bufs.append((k, buf))
                reqs.append(dist.irecv(buf, int(s)))
        for r in reqs:
            r.wait()
        for k, buf in recv_bufs:
            vec[lm.recv_off[k]: lm.recv_off[k] + lm.recv_cnt[k]] = buf.numpy()
        want = lm.faces[:, None] * 10.0 + np.arange(width)[None, :]
        ok = bool(np.array_equal(vec, want))
        # the all-reduce of a Gram-Schmidt pass: owned entries only, so nothing is counted twice
        t = torch.tensor([float(lm.nf_owned), float(np.sum(vec[: lm.nf_owned, 0]))], dtype=torch.float64)
        dist.all_reduce(t)
        ok = ok and t[0].item() == gm.nf and t[1].item() == float(np.sum(np.arange(gm.nf) * 10.0))
        # scatter_local_meshes: rank 0 alone materialises the global mesh; every rank receives the sub-domain
        # (halo plan included) that the redundant construction gives
        calls = []

        def build_global():
            calls.append(rank)
            return small_mesh("hex")
        lm2, nf_global = P.scatter_local_meshes(build_global, world, rank, dist)
        ok = ok and calls == ([0] if rank == 0 else []) and nf_global == gm.nf
        for name in ("elems", "faces", "e2f", "f2e", "flidx", "forient", "fverts", "tags", "nbr_ranks", "recv_off", "recv_cnt"):
            ok = ok and np.array_equal(getattr(lm2, name), getattr(lm, name))
        ok = ok and all(np.array_equal(a, b) for a, b in zip(lm2.send_ids, lm.send_ids))
        ok = ok and (lm2.ne_interior, lm2.nf_interior) == (lm.ne_interior, lm.nf_interior)
        ret[rank] = ok
    finally:
        dist.destroy_process_group()


def test_halo_plan_two_processes_gloo():
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_gloo_worker, args=(world, port, ret), nprocs=world, join=True)
    assert all(ret.get(r) for r in range(world)), dict(ret)
