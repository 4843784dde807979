import sys, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2512_13619_b200 as hdg
ctx = hdg.Context(0)
stream = torch.cuda.current_stream(); ctx.set_stream(stream.cuda_stream)
disc = hdg.Discretization.structured(ctx, "tri", n=512, degree=4, jitter=0.2)
model = hdg.make_case_model(disc, "burgers")
state = hdg.make_initial_state(disc, model)
ops = hdg.assemble_element_operators(disc, model, state)
K, rhs = hdg.assemble_global(disc, ops)
x = torch.randn(disc.n_dof, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
def t_us(fn, reps=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(stream)
    for _ in range(reps): fn()
    e1.record(stream); torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps
res = {}
P0 = hdg.build_preconditioner("asm", K, ops, disc)
res["matvec"] = t_us(lambda: hdg.block_matvec(K, x, y), 100)
res["asm_base"] = t_us(lambda: P0.apply_base(x, y), 100)
for fused in (1, 0):
    hdg.set_tuning("poly_fused", fused)
    P = hdg.build_preconditioner(hdg.PrecondSpec("asm", poly_degree=10, poly_kind="chebyshev"), K, ops, disc)
    res[f"poly_apply_fused{fused}"] = t_us(lambda: P.apply(x, y))
print(json.dumps(res))
