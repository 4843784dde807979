import sys, time, threading
sys.path.insert(0, '/root/repo')
import numpy as np, torch, pynvml as nv
import paper_2512_13619_b200 as hdg
nv.nvmlInit(); H = nv.nvmlDeviceGetHandleByIndex(0)
samples = []; stop = False
def samp():
    while not stop:
        samples.append((time.perf_counter(), nv.nvmlDeviceGetClockInfo(H, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetPowerUsage(H)//1000, nv.nvmlDeviceGetCurrentClocksThrottleReasons(H)))
        time.sleep(0.005)
ctx = hdg.Context(0)
disc = hdg.Discretization.structured(ctx, "hex", n=28, degree=3)
model = hdg.make_case_model(disc, "poisson")
state = hdg.State(disc)
z_u = np.zeros(disc.npe*disc.ne); z_uh = np.zeros(disc.n_dof)
th = threading.Thread(target=samp, daemon=True); th.start()
out = []
for i in range(16):
    state.set("u", z_u); state.set("uhat", z_uh)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hdg.newton_solve(disc, model, state, hdg.NewtonConfig(), hdg.GmresConfig(), hdg.PrecondSpec("asm"))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s = [x for x in samples if t0 <= x[0] <= t1]
    out.append((round(1e3*(t1-t0),1), min(x[1] for x in s), max(x[2] for x in s), hex(max(x[3] for x in s)), len(s)))
stop = True
for o in out: print(o)
