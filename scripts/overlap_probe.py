"""Timing evidence for the overlapped halo exchange on ONE GPU (the box has no second one): rank 0 of a 2-slab
partition of an n x n x 2n hex box (its own n^3 slab + one ghost layer), a 1-rank NCCL communicator and a halo plan
whose only neighbour is the rank itself, so the exchange moves exactly the bytes of the real plan through NCCL's
send / receive kernels (device-local copy instead of NVLink).  The halo VALUES are therefore not the neighbour's --
this script measures time only: block matvec and ASM apply with the exchange (a) blocking on the compute stream,
(b) on its own stream while the interior rows / elements run (tuning "overlap_halo").

  python scripts/overlap_probe.py [--cells 28] [--out gpurun_out/overlap.json]"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=28)
    ap.add_argument("--degree", type=int, default=3)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import paper_2512_13619_b200 as hdg
    from paper_2512_13619_b200 import hdg as H
    from paper_2512_13619_b200 import partition as P
    n = a.cells
    lo, hi = (0.0, 0.0, 0.0), (1.0, 1.0, 2.0)
    coords, ev = P.box_hex_mesh(n, n, 2 * n, lo, hi)
    gm = P.global_mesh("hex", coords, ev, lo=lo, hi=hi)
    lm = P.build_local_meshes(gm, P.slab_partition(gm.ne, 2))[0]
    ctx = hdg.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    L = H.load_library()
    uid = (C.c_char * 128)()
    assert L.hdgb_comm_nccl_unique_id(uid) == 0
    ctx.check(L.hdgb_comm_create_nccl(ctx._h, bytes(uid.raw), 0, 1))
    n_halo = len(lm.faces) - lm.nf_owned
    nbr, cnt, off = (np.array([v], dtype=np.int32) for v in (0, n_halo, lm.nf_owned))
    ids = np.ascontiguousarray(np.arange(lm.nf_owned - n_halo, lm.nf_owned), dtype=np.int32)  # interface faces of this rank
    ctx.check(L.hdgb_comm_set_halo_plan(ctx._h, 1, nbr.ctypes.data, cnt.ctypes.data, ids.ctypes.data, off.ctypes.data, cnt.ctypes.data))
    disc = P.make_discretization(ctx, lm, "hex", a.degree)
    model = hdg.make_case_model(disc, "poisson")
    state = hdg.make_initial_state(disc, model)
    ops = hdg.assemble_element_operators(disc, model, state)
    K, rhs = hdg.assemble_global(disc, ops)
    Pc = hdg.build_preconditioner("asm", K, ops, disc)
    x = torch.randn(disc.n_dof, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)

    def t_us(fn, reps=200):
        for _ in range(10):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return 1e3 * e0.elapsed_time(e1) / reps

    res = {"mesh": f"rank 0 of 2 slabs of hex {n}x{n}x{2 * n}, p={a.degree}", "owned_faces": int(lm.nf_owned),
           "interior_faces": int(lm.nf_interior), "halo_faces": int(n_halo), "owned_elements": int(lm.ne_owned),
           "interior_elements": int(lm.ne_interior), "halo_bytes_per_exchange": int(n_halo * disc.mpf * 8)}
    for mode, name in ((0, "blocking"), (1, "overlapped")):
        hdg.set_tuning("overlap_halo", mode)
        res[f"matvec_us_{name}"] = t_us(lambda: hdg.block_matvec(K, x, y))
        res[f"asm_apply_us_{name}"] = t_us(lambda: Pc.apply_base(x, y))
    hdg.set_tuning("overlap_halo", 1)
    # the exchange alone, and the same operator without a communicator
    vec = x.data_ptr()
    res["exchange_alone_us"] = t_us(lambda: ctx.check(L.hdgb_halo_exchange_begin(ctx._h, vec, disc.mpf)) or ctx.check(L.hdgb_halo_exchange_end(ctx._h)))
    L.hdgb_comm_destroy(ctx._h)
    res["matvec_us_no_comm"] = t_us(lambda: hdg.block_matvec(K, x, y))
    res["asm_apply_us_no_comm"] = t_us(lambda: Pc.apply_base(x, y))
    print(json.dumps(res))
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
