"""One Jacobian assembly of config 5 in miniature (hex 12^3, p = 3, Navier-Stokes, M = 5) -- ncu target for the wide local kernel."""
import sys
sys.path.insert(0, '/root/repo')
import paper_2512_13619_b200 as hdg
ctx = hdg.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
if len(sys.argv) > 2:
    hdg.set_tuning("local_nt_wide", int(sys.argv[2]))
disc = hdg.Discretization.structured(ctx, "hex", n=n, degree=3, n_comp=5)
model = hdg.make_case_model(disc, "navier_stokes", mu=0.02)
state = hdg.make_initial_state(disc, model)
for _ in range(2):
    ops = hdg.assemble_element_operators(disc, model, state, dt=0.01, u_prev=state.u)
    del ops
ctx.close()
