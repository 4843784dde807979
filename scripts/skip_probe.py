import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2512_13619_b200 as hdg
cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = hdg.Context(0)
if cfgn == 5:
    disc = hdg.Discretization.structured(ctx, "hex", n=12, degree=3, n_comp=5)
    model = hdg.make_case_model(disc, "navier_stokes", mu=0.02)
else:
    disc = hdg.Discretization.structured(ctx, "hex", n=28, degree=3)
    model = hdg.make_case_model(disc, "poisson")
state = hdg.make_initial_state(disc, model)
kw = dict(dt=0.01, u_prev=state.u) if cfgn == 5 else {}
if len(sys.argv) > 2:
    hdg.set_tuning("local_nt_wide", int(sys.argv[2]))
for skip in (0, 1, 2, 3):
    hdg.set_tuning("local_debug_skip", skip)
    ops = hdg.assemble_element_operators(disc, model, state, **kw)
    del ops
ctx.close()
