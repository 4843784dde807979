"""Micro-benchmark of orthogonalize (CGS2) on device vectors: streamed three-pass kernels (k_orth.cu) against the
four-pass kernels, per Krylov index.  Bytes: the reference sequence's 8 n (4 j + 6).
  python scripts/bench_orth.py [--n 1091328] [--nvec 1,5,10,25,50]"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1091328)
    ap.add_argument("--nvec", default="1,5,10,25,40,50")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch
    import paper_2512_13619_b200 as hdg
    ctx = hdg.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    L = hdg.load_library()
    n = a.n
    V = torch.randn(51, n, dtype=torch.float64, device="cuda")
    V, _ = torch.linalg.qr(V.T)
    V = V.T.contiguous()
    w0 = torch.randn(n, dtype=torch.float64, device="cuda")
    w = torch.empty_like(w0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    h = np.empty(64)
    for nv in [int(s) for s in a.nvec.split(",")]:
        row = []
        for flag in (0, 1):
            hdg.set_tuning("cgs_stream", flag)
            ts = []
            for r in range(a.reps + 3):
                w.copy_(w0)
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                ctx.check(L.hdgb_orthogonalize(ctx._h, V.data_ptr(), nv, n, w.data_ptr(), 0, h.ctypes.data))
                e1.record(stream)
                torch.cuda.synchronize()
                if r >= 3:
                    ts.append(e0.elapsed_time(e1) * 1e-3)
            t = float(np.median(ts))
            row.append(t)
        by = 8 * n * (4 * nv + 6)
        print(f"nvec {nv:3d}: four-pass {1e6 * row[0]:7.1f} us ({by / row[0] / 1e9:6.0f} GB/s)   streamed {1e6 * row[1]:7.1f} us "
              f"({by / row[1] / 1e9:6.0f} GB/s on the reference's bytes, {8 * n * (3 * nv + 7) / row[1] / 1e9:6.0f} GB/s on its own)")
    hdg.set_tuning("cgs_stream", 1)


if __name__ == "__main__":
    main()
