"""A/B of the streamed E / D_d / H / G_d / F / J sweep (local_ed_stream) on config 2: Newton / GMRES trace of one solve each."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2512_13619_b200 as hdg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
ctx = hdg.Context(0)
disc = hdg.Discretization.structured(ctx, "hex", n=n, degree=3)
model = hdg.make_case_model(disc, "poisson")
state = hdg.make_initial_state(disc, model)
u0, uh0 = state.u, state.uhat
res = {}
for flag in (0, 1, 1, 2, 2, 3, 3):
    hdg.set_tuning("local_ed_stream", flag)
    state.set("u", u0)
    state.set("uhat", uh0)
    rep = hdg.newton_solve(disc, model, state, hdg.NewtonConfig(), hdg.GmresConfig(), hdg.PrecondSpec("asm"))
    print(flag, rep.n_newton, rep.n_gmres_total, rep.residual_history, [getattr(rep, k, None) for k in ("gmres_per_newton",)])
    res[flag] = (state.u.copy(), state.uhat.copy())
print("rel diff u", np.linalg.norm(res[0][0] - res[1][0]) / np.linalg.norm(res[0][0]))
ctx.close()
