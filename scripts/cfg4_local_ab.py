"""Config 4 in miniature (jittered tets 6 x n^3, p = 2, elasticity M = 3): assemble_element_operators with the scalar local
kernel (default for pe < 20) against the DMMA one (tuning key local_dmma_min_pe), same run."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import paper_2512_13619_b200 as hdg  # noqa: E402

ctx = hdg.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
disc = hdg.Discretization.structured(ctx, "tet", n=n, degree=2, n_comp=3, jitter=0.1)
model = hdg.make_case_model(disc, "elasticity")
state = hdg.make_initial_state(disc, model)
print("ne", disc.ne, "pe", disc.pe, "pf", disc.pf, "qe", disc.qe, "qf", disc.qf, "npe", disc.npe, "nfl", disc.nfl, flush=True)
ref = None
for rep in range(2):
    for min_pe, budget in ((20, 216), (8, 216), (8, 96), (8, 48), (20, 96), (20, 48)):
        hdg.set_tuning("local_dmma_min_pe", min_pe)
        hdg.set_tuning("assemble_budget_kb", budget)
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            ops = hdg.assemble_element_operators(disc, model, state)
            ts.append(time.perf_counter() - t0)
            kb = ops.get("kbar") if _ == 3 and rep == 0 else None
            del ops
        if kb is not None:
            if ref is None or budget == 216 and min_pe == 20:
                ref = kb
            else:
                print("   kbar vs scalar kernel: max rel diff", np.max(np.abs(kb - ref)) / np.max(np.abs(ref)))
        print(f"local_dmma_min_pe={min_pe} assemble_budget_kb={budget} assemble_element_operators min {min(ts[1:]) * 1e3:.2f} ms  (all: {[round(t * 1e3, 2) for t in ts]})", flush=True)
hdg.set_tuning("local_dmma_min_pe", 20)
hdg.set_tuning("assemble_budget_kb", 216)
ctx.close()
