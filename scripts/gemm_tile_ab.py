"""Same-run A/B of the generic DMMA GEMM's CTA width (tuning keys gemm_wm_cap / gemm_wn_cap: 32-row / 32-column warp tiles per CTA) on the
Schur complement of config 5 in miniature (hex n^3, p = 3, Navier-Stokes, M = 5: 320 x 480 and 480 x 480 products)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2512_13619_b200 as hdg  # noqa: E402

ctx = hdg.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
disc = hdg.Discretization.structured(ctx, "hex", n=n, degree=3, n_comp=5)
model = hdg.make_case_model(disc, "navier_stokes", mu=0.02)
state = hdg.make_initial_state(disc, model)
for rep in range(2):
    for wm, cap in ((4, 4), (4, 2), (4, 1), (3, 1), (2, 2), (2, 1), (1, 2), (1, 1)):
        hdg.set_tuning("gemm_wm_cap", wm)
        hdg.set_tuning("gemm_wn_cap", cap)
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            ops = hdg.assemble_element_operators(disc, model, state, dt=0.01, u_prev=state.u)
            ts.append(time.perf_counter() - t0)
            del ops
        print(f"gemm_wm_cap={wm} gemm_wn_cap={cap} assemble_element_operators min {min(ts[1:]) * 1e3:.2f} ms  (all: {[round(t * 1e3, 2) for t in ts]})", flush=True)
hdg.set_tuning("gemm_wn_cap", 1)
hdg.set_tuning("gemm_wm_cap", 2)
ctx.close()
