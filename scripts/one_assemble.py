"""One Jacobian assembly of config 2 (hex 28^3, p = 3, Poisson) -- the ncu target for the local kernel."""
import sys
sys.path.insert(0, '/root/repo')
import paper_2512_13619_b200 as hdg
ctx = hdg.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
disc = hdg.Discretization.structured(ctx, "hex", n=n, degree=3)
model = hdg.make_case_model(disc, "poisson")
state = hdg.make_initial_state(disc, model)
for _ in range(2):
    ops = hdg.assemble_element_operators(disc, model, state)
    del ops
ctx.close()
