import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2512_13619_b200 as hdg
ctx = hdg.Context(0)
disc = hdg.Discretization.structured(ctx, "hex", n=28, degree=3)
model = hdg.make_case_model(disc, "poisson")
state = hdg.State(disc)
z_u = np.zeros(disc.npe*disc.ne); z_uh = np.zeros(disc.n_dof)
ts = []; st = []
for i in range(12):
    state.set("u", z_u); state.set("uhat", z_uh)
    torch.cuda.synchronize(); t = time.perf_counter()
    rep = hdg.newton_solve(disc, model, state, hdg.NewtonConfig(), hdg.GmresConfig(), hdg.PrecondSpec("asm"))
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t); st.append(hdg.hdg.pool_stats())
print(["%.1f" % (1e3*t) for t in ts]); print(st)
