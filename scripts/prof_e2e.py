import sys, time, cProfile, pstats
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2512_13619_b200 as hdg
ctx = hdg.Context(0)
disc = hdg.Discretization.structured(ctx, "hex", n=28, degree=3)
xq, xf = disc.quad_coords()
sinprod = lambda x: np.prod(np.sin(np.pi * x), axis=-1)
fq = torch.from_numpy(np.ascontiguousarray(3*np.pi**2*sinprod(xq))).pin_memory()
dq = torch.from_numpy(np.ascontiguousarray(sinprod(xf))).pin_memory()
u0 = torch.zeros(disc.npe*disc.ne, dtype=torch.float64).pin_memory(); uh0 = torch.zeros(disc.n_dof, dtype=torch.float64).pin_memory()
uo = torch.empty_like(u0).pin_memory(); uho = torch.empty_like(uh0).pin_memory()
def step():
    m = hdg.Model(disc, "poisson", [1.0], forcing=lambda x: fq.numpy(), dirichlet=lambda x: dq.numpy(), exact=sinprod)
    s = hdg.State(disc); s.set("u", u0.numpy()); s.set("uhat", uh0.numpy())
    rep = hdg.newton_solve(disc, m, s, hdg.NewtonConfig(), hdg.GmresConfig(), hdg.PrecondSpec("asm"))
    ctx.copy(uo.numpy(), s.ptr("u"), uo.numel()); ctx.copy(uho.numpy(), s.ptr("uhat"), uho.numel())
for _ in range(3): step()
torch.cuda.synchronize(); t=time.perf_counter(); step(); torch.cuda.synchronize(); print("e2e step s", time.perf_counter()-t)
pr = cProfile.Profile(); pr.enable(); step(); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
