import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2512_13619_b200 as hdg
ctx = hdg.Context(0)
disc = hdg.Discretization.structured(ctx, "hex", n=28, degree=3)
model = hdg.make_case_model(disc, "poisson")
state = hdg.State(disc)
z_u = np.zeros(disc.npe*disc.ne); z_uh = np.zeros(disc.n_dof)
ts = []; st = []; gs = []
import pynvml as nv
nv.nvmlInit(); H = nv.nvmlDeviceGetHandleByIndex(0)
stream = torch.cuda.current_stream(); ctx.set_stream(stream.cuda_stream)
for i in range(12):
    state.set("u", z_u); state.set("uhat", z_uh)
    torch.cuda.synchronize(); t = time.perf_counter(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record(stream)
    rep = hdg.newton_solve(disc, model, state, hdg.NewtonConfig(), hdg.GmresConfig(), hdg.PrecondSpec("asm"))
    e1.record(stream); torch.cuda.synchronize(); ts.append(time.perf_counter() - t); st.append(hdg.hdg.pool_stats())
    gs.append((round(e0.elapsed_time(e1), 1), nv.nvmlDeviceGetPowerUsage(H) // 1000, nv.nvmlDeviceGetClockInfo(H, nv.NVML_CLOCK_SM), hex(nv.nvmlDeviceGetCurrentClocksThrottleReasons(H))))
print(["%.1f" % (1e3*t) for t in ts]); print(st); print(gs)
