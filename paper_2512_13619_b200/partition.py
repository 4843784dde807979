"""Domain decomposition of the HDG trace system across the GPUs of one box (north_star item 5).

The reference has no distributed path ("future work"); the design follows SURVEY.md
section 8e: elements are partitioned, a face is owned by the rank owning its side-0 element (the lower
element id, the rule that already fixes the reference's accumulation order, mesh.cpp:63-71), every
rank keeps its owned elements plus ONE layer of ghost elements which it condenses redundantly, and
numbers its faces owned-first, then halo faces grouped by owner.  This module is pure host logic
(numpy): it slices the global connectivity tables into per-rank tables and builds the halo plan.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import hdg as H


@dataclass
class GlobalMesh:
    shape: str
    elem_verts: np.ndarray      # (ne, vpe) int32
    coords: np.ndarray          # (nv, dim)
    e2f: np.ndarray             # (ne, n_lfe)
    f2e: np.ndarray             # (nf, 2), -1 on the boundary
    flidx: np.ndarray           # (nf, 2)
    forient: np.ndarray         # (nf, 2)
    fverts: np.ndarray          # (nf, vpf) canonical corner order
    tags: np.ndarray            # (nf,) 0 interior

    @property
    def ne(self):
        return self.e2f.shape[0]

    @property
    def nf(self):
        return self.f2e.shape[0]


def box_hex_mesh(nx: int, ny: int, nz: int, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)):
    """Vertex coordinates and hexahedra of an nx x ny x nz box mesh, numbered like the structured
    builder of the library (x fastest; v0..v3 bottom CCW, v4..v7 above)."""
    xs = [np.linspace(lo[d], hi[d], n + 1) for d, n in enumerate((nx, ny, nz))]
    Z, Y, X = np.meshgrid(xs[2], xs[1], xs[0], indexing="ij")
    coords = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    vid = lambda i, j, k: (k * (ny + 1) + j) * (nx + 1) + i
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    ev = np.stack([vid(i, j, k), vid(i + 1, j, k), vid(i + 1, j + 1, k), vid(i, j + 1, k),
                   vid(i, j, k + 1), vid(i + 1, j, k + 1), vid(i + 1, j + 1, k + 1), vid(i, j + 1, k + 1)], axis=1)
    return coords, ev.astype(np.int32)


def box_quad_mesh(nx: int, ny: int, lo=(0.0, 0.0), hi=(1.0, 1.0)):
    xs = [np.linspace(lo[d], hi[d], n + 1) for d, n in enumerate((nx, ny))]
    Y, X = np.meshgrid(xs[1], xs[0], indexing="ij")
    coords = np.stack([X.ravel(), Y.ravel()], axis=1)
    vid = lambda i, j: j * (nx + 1) + i
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    i, j = i.ravel(), j.ravel()
    ev = np.stack([vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)], axis=1)
    return coords, ev.astype(np.int32)


def box_boundary_tags(gm_coords, fverts, f2e, lo, hi):
    """Tags of the structured builders: 1 = y-lo, 2 = x-hi, 3 = y-hi, 4 = x-lo, 5 = z-lo, 6 = z-hi."""
    dim = gm_coords.shape[1]
    tags = np.zeros(f2e.shape[0], dtype=np.int32)
    bnd = f2e[:, 1] < 0
    c = gm_coords[fverts]                                  # (nf, vpf, dim)
    tol = 1e-12
    on = lambda d, val: np.all(np.abs(c[:, :, d] - val) < tol, axis=1)
    rules = [(1, 1, lo[1]), (2, 0, hi[0]), (3, 1, hi[1]), (4, 0, lo[0])]
    if dim == 3:
        rules += [(5, 2, lo[2]), (6, 2, hi[2])]
    for tag, d, val in reversed(rules):                    # earlier rules win, like the builder's if-chain
        tags[bnd & on(d, val)] = tag
    tags[bnd & (tags == 0)] = 1
    return tags


def global_mesh(shape: str, coords, elem_verts, tags=None, lo=None, hi=None) -> GlobalMesh:
    """Connectivity of a conforming mesh (host only, no GPU): hdgb_mesh_connectivity."""
    L = H.load_library()
    ev = np.ascontiguousarray(elem_verts, dtype=np.int32)
    xc = np.ascontiguousarray(coords, dtype=np.float64)
    h = C.c_void_p()
    st = L.hdgb_mesh_connectivity(H.SHAPES[shape], ev.shape[0], xc.shape[0], ev.ctypes.data, xc.ctypes.data, C.byref(h))
    if st != 0:
        raise H.InvalidMesh(f"mesh connectivity failed (status {st})")
    d = H.Discretization.__new__(H.Discretization)
    d.ctx, d._h, d._L = None, h, L
    ne = ev.shape[0]
    e2f = d.table("element_to_face").reshape(ne, -1)
    f2e = d.table("face_to_elements").reshape(-1, 2)
    nf = f2e.shape[0]
    gm = GlobalMesh(shape, ev, xc, e2f, f2e, d.table("face_local_index").reshape(nf, 2),
                    d.table("face_orient").reshape(nf, 2), d.table("face_vertices").reshape(nf, -1),
                    d.table("boundary_tag"))
    d.close()
    if tags is not None:
        gm.tags = np.asarray(tags, dtype=np.int32)
    elif lo is not None:
        gm.tags = box_boundary_tags(xc, gm.fverts, gm.f2e, lo, hi)
    return gm


def global_mesh_from_structured(shape: str, n: int, jitter: float = 0.0, seed: int = 12345, lo=None, hi=None) -> GlobalMesh:
    """Connectivity of the library's own structured builder (host-only discretisation, no GPU): the
    partitioned run then cuts exactly the mesh -- element / face numbering, orientation flags, boundary
    tags, jittered vertices -- that Discretization.structured() gives the single-GPU run."""
    d = H.Discretization.structured(None, shape, n=n, degree=1, jitter=jitter, seed=seed, lo=lo, hi=hi)
    ne, nf = d.ne, d.nf
    gm = GlobalMesh(shape, d.table("element_vertices").reshape(ne, -1), d.table("vertex_coords").reshape(-1, d.dim),
                    d.table("element_to_face").reshape(ne, -1), d.table("face_to_elements").reshape(nf, 2),
                    d.table("face_local_index").reshape(nf, 2), d.table("face_orient").reshape(nf, 2),
                    d.table("face_vertices").reshape(nf, -1), d.table("boundary_tag"))
    d.close()
    return gm


def slab_partition(n_elems: int, n_ranks: int) -> np.ndarray:
    """Contiguous element-id ranges (slabs of a structured mesh): rank of every element."""
    return (np.arange(n_elems, dtype=np.int64) * n_ranks // n_elems).astype(np.int32)


@dataclass
class LocalMesh:
    rank: int
    n_ranks: int
    elems: np.ndarray            # global ids of the local elements, owned first
    ne_owned: int
    faces: np.ndarray            # global ids of the local faces: owned, then halo grouped by owner
    nf_owned: int
    face_owner: np.ndarray       # owner rank of every local face
    verts: np.ndarray            # global ids of the local vertices
    elem_verts: np.ndarray
    coords: np.ndarray
    e2f: np.ndarray
    f2e: np.ndarray
    flidx: np.ndarray
    forient: np.ndarray
    fverts: np.ndarray
    tags: np.ndarray
    nf_global: int
    ne_interior: int = 0         # leading owned elements all of whose faces are owned
    nf_interior: int = 0         # leading owned faces whose block row references owned faces only
    # halo plan
    nbr_ranks: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    send_ids: list = field(default_factory=list)       # per neighbour: local ids of owned faces to send
    recv_off: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    recv_cnt: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    needs: dict = field(default_factory=dict)           # owner rank -> global ids this rank receives


def local_mesh(gm: GlobalMesh, part: np.ndarray, rank: int) -> LocalMesh:
    """Per-rank tables: owned elements + one ghost layer; faces owned-first, halo grouped by owner."""
    n_ranks = int(part.max()) + 1
    owned_e = np.flatnonzero(part == rank)
    faces_owned_e = np.unique(gm.e2f[owned_e])
    nbr_e = np.unique(gm.f2e[faces_owned_e].ravel())
    nbr_e = nbr_e[nbr_e >= 0]
    ghost_e = np.setdiff1d(nbr_e, owned_e, assume_unique=True)
    # Overlap window of the halo exchange: an owned element is INTERIOR when this rank owns all its faces, an
    # owned face when both adjacent elements are interior (or absent: domain boundary) -- its block row then
    # references owned faces only.  Interior entities are numbered first (ids ascending within each group), so
    # the library computes them while the exchange is in flight and the interface rest afterwards.
    face_mine = part[gm.f2e[:, 0]] == rank
    e_int = np.all(face_mine[gm.e2f[owned_e]], axis=1)
    owned_e = np.concatenate([owned_e[e_int], owned_e[~e_int]])
    ne_interior = int(np.count_nonzero(e_int))
    elems = np.concatenate([owned_e, ghost_e]).astype(np.int64)
    g2l_e = -np.ones(gm.ne, dtype=np.int64)
    g2l_e[elems] = np.arange(len(elems))

    lf = np.unique(gm.e2f[elems])
    owner = part[gm.f2e[lf, 0]]
    own = lf[owner == rank]
    elem_interior = np.zeros(gm.ne + 1, dtype=bool)      # index -1 (no element) -> slot gm.ne
    elem_interior[owned_e[:ne_interior]] = True
    elem_interior[gm.ne] = True
    f_int = np.all(elem_interior[np.where(gm.f2e[own] < 0, gm.ne, gm.f2e[own])], axis=1)
    own = np.concatenate([own[f_int], own[~f_int]])
    nf_interior = int(np.count_nonzero(f_int))
    halo = lf[owner != rank]
    halo_owner = part[gm.f2e[halo, 0]]
    order = np.lexsort((halo, halo_owner))
    halo, halo_owner = halo[order], halo_owner[order]
    faces = np.concatenate([own, halo]).astype(np.int64)
    g2l_f = -np.ones(gm.nf, dtype=np.int64)
    g2l_f[faces] = np.arange(len(faces))

    verts = np.unique(gm.elem_verts[elems])
    g2l_v = -np.ones(gm.coords.shape[0], dtype=np.int64)
    g2l_v[verts] = np.arange(len(verts))

    f2e_g = gm.f2e[faces]
    f2e_l = np.where(f2e_g < 0, -1, np.where(g2l_e[np.maximum(f2e_g, 0)] >= 0, g2l_e[np.maximum(f2e_g, 0)], -2))
    lm = LocalMesh(rank=rank, n_ranks=n_ranks, elems=elems, ne_owned=len(owned_e), faces=faces, nf_owned=len(own),
                   face_owner=np.concatenate([np.full(len(own), rank), halo_owner]).astype(np.int32), verts=verts,
                   elem_verts=g2l_v[gm.elem_verts[elems]].astype(np.int32), coords=gm.coords[verts],
                   e2f=g2l_f[gm.e2f[elems]].astype(np.int32), f2e=f2e_l.astype(np.int32),
                   flidx=gm.flidx[faces].astype(np.int32), forient=gm.forient[faces].astype(np.int32),
                   fverts=g2l_v[gm.fverts[faces]].astype(np.int32), tags=gm.tags[faces].astype(np.int32),
                   nf_global=gm.nf)
    lm.ne_interior, lm.nf_interior = ne_interior, nf_interior
    nbrs = np.unique(halo_owner)
    lm.needs = {int(s): halo[halo_owner == s] for s in nbrs}
    return lm


def finish_halo_plan(lm: LocalMesh, all_needs: list):
    """all_needs[r] = the `needs` dict of rank r (gathered with all_gather_object, or computed
    redundantly).  Fills the send side: what every other rank expects from this one."""
    g2l_f = {int(g): i for i, g in enumerate(lm.faces[: lm.nf_owned])}
    sends = {}
    for r, nd in enumerate(all_needs):
        if r == lm.rank:
            continue
        want = nd.get(lm.rank)
        if want is not None and len(want):
            sends[r] = np.array([g2l_f[int(g)] for g in want], dtype=np.int32)
    nbrs = sorted(set(sends) | set(lm.needs))
    lm.nbr_ranks = np.array(nbrs, dtype=np.int32)
    lm.send_ids = [sends.get(s, np.zeros(0, np.int32)) for s in nbrs]
    off, cnt = [], []
    halo_owner = lm.face_owner[lm.nf_owned:]
    for s in nbrs:
        idx = np.flatnonzero(halo_owner == s)
        off.append(lm.nf_owned + (int(idx[0]) if len(idx) else 0))
        cnt.append(len(idx))
    lm.recv_off, lm.recv_cnt = np.array(off, dtype=np.int32), np.array(cnt, dtype=np.int32)
    return lm


def build_local_meshes(gm: GlobalMesh, part: np.ndarray):
    """All ranks' local meshes with completed halo plans (single-process use: tests, virtual ranks)."""
    n_ranks = int(part.max()) + 1
    lms = [local_mesh(gm, part, r) for r in range(n_ranks)]
    needs = [lm.needs for lm in lms]
    return [finish_halo_plan(lm, needs) for lm in lms]


def build_my_local_mesh(gm: GlobalMesh, part: np.ndarray, rank: int, dist=None):
    """This rank's local mesh; the send side of the halo plan comes from an all_gather_object of
    every rank's receive lists when torch.distributed is initialised (any backend, gloo included),
    otherwise it is recomputed redundantly."""
    lm = local_mesh(gm, part, rank)
    n_ranks = int(part.max()) + 1
    if dist is not None and dist.is_initialized() and dist.get_world_size() == n_ranks:
        needs = [None] * n_ranks
        dist.all_gather_object(needs, {k: v for k, v in lm.needs.items()})
    else:
        needs = [local_mesh(gm, part, r).needs if r != rank else lm.needs for r in range(n_ranks)]
    return finish_halo_plan(lm, needs)


def scatter_local_meshes(build_global, n_ranks: int, rank: int, dist):
    """Rank 0 alone materialises the global mesh (build_global() -> GlobalMesh), cuts it into the per-rank local
    meshes with completed halo plans and scatters them (torch.distributed object scatter, any backend); the other
    ranks never hold more than their own sub-domain.  Returns (this rank's LocalMesh, global face count)."""
    if dist is None or n_ranks == 1 or not dist.is_initialized():
        gm = build_global()
        return build_local_meshes(gm, slab_partition(gm.ne, n_ranks))[rank], gm.nf
    box = [None]
    if rank == 0:
        gm = build_global()
        lms = build_local_meshes(gm, slab_partition(gm.ne, n_ranks))
        dist.scatter_object_list(box, lms, src=0)
    else:
        dist.scatter_object_list(box, None, src=0)
    return box[0], box[0].nf_global


def make_discretization(ctx, lm: LocalMesh, shape: str, degree: int, n_comp=1, quad_points=0):
    """hdgb_disc_create_from_tables for a local mesh."""
    L = H.load_library()
    h = C.c_void_p()
    arr = lambda a, t: np.ascontiguousarray(a, dtype=t)
    ev, xc = arr(lm.elem_verts, np.int32), arr(lm.coords, np.float64)
    e2f, f2e, fl, fo = arr(lm.e2f, np.int32), arr(lm.f2e, np.int32), arr(lm.flidx, np.int32), arr(lm.forient, np.int32)
    fv, tg, gid = arr(lm.fverts, np.int32), arr(lm.tags, np.int32), arr(lm.faces, np.int64)
    st = L.hdgb_disc_create_from_tables(ctx._h if ctx else None, H.SHAPES[shape], degree, n_comp, quad_points,
                                        ev.shape[0], f2e.shape[0], xc.shape[0], ev.ctypes.data, xc.ctypes.data,
                                        e2f.ctypes.data, f2e.ctypes.data, fl.ctypes.data, fo.ctypes.data, fv.ctypes.data,
                                        tg.ctypes.data, lm.ne_owned, lm.nf_owned, gid.ctypes.data, lm.nf_global, C.byref(h))
    if ctx is not None:
        ctx.check(st)
    elif st != 0:
        raise H.HdgError(f"hdgb_disc_create_from_tables failed (status {st})")
    d = H.Discretization(ctx, h)
    d.ne_owned, d.nf_owned, d.local_mesh = lm.ne_owned, lm.nf_owned, lm
    d.ne_interior, d.nf_interior = (int(v) for v in d.table("interior_counts"))  # as the library sees them
    return d


def install_nccl_comm(ctx, lm: LocalMesh, dist):
    """NCCL communicator + halo plan on this rank's context; the unique id travels over
    torch.distributed (whatever backend the job initialised)."""
    import os
    # one box: keep NCCL's bootstrap on the loopback interface (the container hostname may not resolve,
    # and probing absent NICs can stall communicator creation for minutes)
    os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
    os.environ.setdefault("NCCL_IB_DISABLE", "1")
    L = H.load_library()
    uid = (C.c_char * 128)()
    if lm.rank == 0:
        st = L.hdgb_comm_nccl_unique_id(uid)
        if st != 0:
            raise H.HdgError("ncclGetUniqueId failed")
    box = [bytes(uid.raw)]
    if dist is not None and lm.n_ranks > 1:
        dist.broadcast_object_list(box, src=0)
    ctx.check(L.hdgb_comm_create_nccl(ctx._h, box[0], lm.rank, lm.n_ranks))
    set_halo_plan(ctx, lm)


class HostComm:
    """Host-staged transport over any torch.distributed backend (gloo): the library's callback
    communicator with the halo exchange and the all-reduce carried through host memory.  It exists for
    boxes with fewer GPUs than ranks (several ranks sharing one device, where NCCL refuses to form a
    communicator) and for tests; the production transport is install_nccl_comm."""

    HALO_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int)
    ALLRED_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int)

    def __init__(self, ctx, lm: LocalMesh, dist):
        import torch
        self.ctx, self.lm, self.dist, self.torch = ctx, lm, dist, torch
        self._halo = self.HALO_FN(self.halo)
        self._allred = self.ALLRED_FN(self.allreduce)
        L = H.load_library()
        ctx.check(L.hdgb_comm_set_callbacks(ctx._h, lm.rank, lm.n_ranks, C.cast(self._halo, C.c_void_p),
                                            C.cast(self._allred, C.c_void_p), None))

    def halo(self, user, vec, width):
        try:
            lm, torch, dist = self.lm, self.torch, self.dist
            own = np.empty(lm.nf_owned * width)
            self.ctx.copy(own, vec, own.size)
            own = own.reshape(lm.nf_owned, width)
            reqs, recvs = [], []
            for k, s in enumerate(lm.nbr_ranks):
                if len(lm.send_ids[k]):
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(own[lm.send_ids[k]])), int(s)))
                if lm.recv_cnt[k]:
                    buf = torch.empty(int(lm.recv_cnt[k]) * width, dtype=torch.float64)
                    recvs.append((k, buf))
                    reqs.append(dist.irecv(buf, int(s)))
            for r in reqs:
                r.wait()
            for k, buf in recvs:
                self.ctx.copy(vec + int(lm.recv_off[k]) * width * 8, buf.numpy(), buf.numel())
            return 0
        except Exception as e:  # pragma: no cover
            print("host halo exchange failed:", repr(e), flush=True)
            return 1

    def allreduce(self, user, buf, n):
        try:
            t = self.torch.empty(n, dtype=self.torch.float64)
            self.ctx.copy(t.numpy(), buf, n)
            self.dist.all_reduce(t)
            self.ctx.copy(buf, t.numpy(), n)
            return 0
        except Exception as e:  # pragma: no cover
            print("host all-reduce failed:", repr(e), flush=True)
            return 1


def install_host_comm(ctx, lm: LocalMesh, dist) -> HostComm:
    """Callback communicator carried by torch.distributed point-to-point / all-reduce on host tensors."""
    hc = HostComm(ctx, lm, dist)
    ctx._host_comm = hc  # keep the ctypes thunks alive as long as the context
    return hc


def set_halo_plan(ctx, lm: LocalMesh):
    L = H.load_library()
    nb = np.ascontiguousarray(lm.nbr_ranks, dtype=np.int32)
    sc = np.array([len(s) for s in lm.send_ids], dtype=np.int32)
    sid = np.ascontiguousarray(np.concatenate(lm.send_ids) if len(lm.send_ids) else np.zeros(0), dtype=np.int32)
    ro, rc = np.ascontiguousarray(lm.recv_off, dtype=np.int32), np.ascontiguousarray(lm.recv_cnt, dtype=np.int32)
    ctx.check(L.hdgb_comm_set_halo_plan(ctx._h, len(nb), nb.ctypes.data, sc.ctypes.data, sid.ctypes.data, ro.ctypes.data,
                                        rc.ctypes.data))
