"""Ad-hoc GPU probe: phase times of one configuration (not a bench; numbers guide tuning)."""
import argparse, time, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2512_13619_b200 as hdg

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="hex"); ap.add_argument("--n", type=int, default=28)
ap.add_argument("--k", type=int, default=3); ap.add_argument("--case", default="poisson")
ap.add_argument("--pc", default="asm"); ap.add_argument("--deg", type=int, default=0)
ap.add_argument("--ncomp", type=int, default=1); ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--tol", type=float, default=1e-6)
a = ap.parse_args()

ctx = hdg.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
t0 = time.time()
disc = hdg.Discretization.structured(ctx, a.shape, n=a.n, degree=a.k, n_comp=a.ncomp)
print(f"setup {time.time()-t0:.2f}s ne={disc.ne} nf={disc.nf} n_dof={disc.n_dof} mpf={disc.mpf} nfl={disc.nfl}", flush=True)
model = hdg.make_case_model(disc, a.case)
state = hdg.make_initial_state(disc, model)

def timed(fn, reps=a.reps, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3

t0 = time.time(); ops = hdg.assemble_element_operators(disc, model, state); ctx.synchronize()
print(f"assemble_element_operators {time.time()-t0:.3f}s", flush=True)
t0 = time.time(); ops = hdg.assemble_element_operators(disc, model, state); ctx.synchronize()
print(f"assemble_element_operators(2nd) {time.time()-t0:.3f}s", flush=True)
t0 = time.time(); K, rhs = hdg.assemble_global(disc, ops); ctx.synchronize()
print(f"assemble_global {time.time()-t0:.3f}s", flush=True)
t0 = time.time(); P = hdg.build_preconditioner(hdg.PrecondSpec(a.pc, poly_degree=a.deg), K, ops, disc); ctx.synchronize()
print(f"build_preconditioner {time.time()-t0:.3f}s", flush=True)
n = K.n_dof
x = torch.randn(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
mpf, nb, nf, ne, nfl = disc.mpf, disc.nb, disc.nf, disc.ne, disc.nfl
t = timed(lambda: hdg.block_matvec(K, x, y)); by = 8*nf*mpf*(mpf*nb+2)+8*nf*nb
print(f"matvec {t*1e6:.1f} us  {by/t/1e9:.0f} GB/s ({by/1e9:.3f} GB)")
t = timed(lambda: P.apply_base(x, y))
by = 8*ne*nfl*nfl+8*(2*ne*nfl+2*nf*mpf) if a.pc in ("asm","ras") else 8*nf*mpf*(mpf+2)
print(f"precond base apply {t*1e6:.1f} us  {by/t/1e9:.0f} GB/s ({by/1e9:.3f} GB)")
ctx.enable_phase_timing(True)
t0 = time.time()
xs, st = hdg.gmres_solve(K, P, rhs, cfg=hdg.GmresConfig(tol=a.tol))
dt = time.time()-t0
print(f"gmres: iters={st.iters} conv={st.converged} rel={st.final_rel_residual:.2e} wall={dt:.3f}s t_mv={st.t_mv:.3f} t_prec={st.t_prec:.3f} t_orth={st.t_orth:.3f}")
ctx.enable_phase_timing(False)
t0 = time.time()
xs, st = hdg.gmres_solve(K, P, rhs, cfg=hdg.GmresConfig(tol=a.tol))
dt = time.time()-t0
print(f"gmres(no phase timing): iters={st.iters} wall={dt:.3f}s  {dt/max(st.iters,1)*1e3:.3f} ms/iter")
state2 = hdg.make_initial_state(disc, model)
t0 = time.time()
rep = hdg.newton_solve(disc, model, state2, gcfg=hdg.GmresConfig(tol=a.tol), pspec=hdg.PrecondSpec(a.pc, poly_degree=a.deg))
dt = time.time()-t0
print(f"newton: {rep} wall={dt:.3f}s t_ass={rep.t_ass:.3f}")
if model.exact_solution is not None:
    print("L2 error:", disc.l2_error(state2.u, model.exact_solution))
