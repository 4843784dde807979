"""Repeated Jacobian assemblies of config 2 must give bitwise identical operators (no timing dependence in the streamed
local kernel): prints the number of distinct digests over R runs per tuning mode."""
import hashlib
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2512_13619_b200 as hdg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ctx = hdg.Context(0)
disc = hdg.Discretization.structured(ctx, "hex", n=n, degree=3, jitter=0.1)
model = hdg.make_case_model(disc, "poisson")
state = hdg.make_initial_state(disc, model)
rng = np.random.default_rng(1)
state.u = state.u + 0.1 * rng.standard_normal(state.u.shape)
state.uhat = state.uhat + 0.1 * rng.standard_normal(state.uhat.shape)
ref = None
for mode in (0, 3):
    hdg.set_tuning("local_ed_stream", mode)
    digs = set()
    for r in range(R):
        ops = hdg.assemble_element_operators(disc, model, state)
        kb = ops.get("kbar")
        digs.add(hashlib.sha1(kb.tobytes()).hexdigest())
        if mode == 0 and r == 0:
            ref = kb
        if mode == 3 and r == 0:
            print("rel diff kbar stream vs chunked", np.linalg.norm(kb - ref) / np.linalg.norm(ref), "max abs", np.abs(kb - ref).max())
        del ops
    print("mode", mode, "distinct digests over", R, "runs:", len(digs))
ctx.close()
