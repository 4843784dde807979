#!/usr/bin/env python
"""Benchmark of the HDG solver hot path (BASELINE.json).

Workload at N = 1: BASELINE configs[1] -- 3D Poisson, structured hex mesh 28^3 (1 091 328 trace
DOFs), p = 3, additive Schwarz preconditioned GMRES (the reference's ASM; --precond ras selects the
restricted variant), FP64.  One "step" = one complete
newton_solve of that problem from the zero initial state: residual assembly, quadrature assembly +
static condensation, face-block global assembly, preconditioner build, GMRES to 1e-6, local
recovery, line search.  Metric: trace DOFs solved per second (whole job), plus the per-iteration
GMRES time, the block-matvec / preconditioner-apply GB/s and the Newton solve time BASELINE names.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU implementation of the same path (the tier-B oracle port: the
reference itself is 2D-only and cannot run this 3D configuration) on the host cores, on a bounded
sample (a smaller hex mesh of the same degree / model / preconditioner).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

# stdout carries exactly ONE JSON line: native libraries (NCCL prints its version banner there) and anything
# else that writes to fd 1 during the run are diverted to stderr; emit() writes the line to the real stdout
_REAL_STDOUT = os.dup(1)
os.dup2(2, 1)


def emit(line):
    sys.stdout.flush()
    os.write(_REAL_STDOUT, (json.dumps(line) + "\n").encode())

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "newton_solve_trace_dofs_per_s"
UNIT = "DOF/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cells", dest="n", type=int, default=28, help="hex cells per direction (28 -> 1.09 M trace DOFs)")
    ap.add_argument("--force-dd", action="store_true", help="use the domain-decomposition path even on one rank (testing)")
    ap.add_argument("--degree", type=int, default=3)
    ap.add_argument("--precond", default="asm", choices=["bj", "asm", "ras"])
    ap.add_argument("--cpu-cells", dest="cpu_n", type=int, default=12, help="hex cells per direction of the bounded CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def workload_name(n, k, pc):
    return f"3D Poisson, structured hex {n}^3, p={k}, {pc.upper()}-GMRES(50) tol 1e-6, Newton tol 1e-8, FP64"


# ---- CPU arm: the oracle port on the host cores ----------------------------------------------------
def cpu_sample(n, k, pc, threads):
    """One Newton solve of the bounded CPU sample; returns (seconds, n_dof, report, tables-setup seconds)."""
    from oracle import port
    import paper_2512_13619_b200 as hdg
    hd = hdg.Discretization.structured(None, "hex", n=n, degree=k)  # host-only setup tables (no GPU involved)
    port.set_threads(threads)
    t0 = time.perf_counter()
    oc = port.OraCase(port.tables_from_disc(hd))  # includes precompute_local_factors (setup, not part of the solve)
    t_setup = time.perf_counter() - t0
    xq, xf = hd.quad_coords()
    sinprod = lambda x: np.prod(np.sin(np.pi * x), axis=-1)
    oc.set_model("poisson", [1.0], 3 * np.pi * np.pi * sinprod(xq), sinprod(xf))
    t0 = time.perf_counter()
    rep = oc.newton(precond=pc)
    dt = time.perf_counter() - t0
    return dt, oc.n_dof, rep, t_setup


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    times, rep, n_dof = [], None, 0
    for i in range(a.warmup + a.steps):
        dt, n_dof, rep, _ = cpu_sample(a.cpu_n, a.degree, a.precond, threads)
        if i >= a.warmup:
            times.append(dt)
    total = sum(times)
    value = n_dof * len(times) / total
    sample = (f"hex {a.cpu_n}^3 p={a.degree} ({n_dof} trace DOFs), {rep['n_newton']} Newton / {rep['n_gmres_total']} GMRES "
              f"iterations per solve, {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(a.n, a.degree, a.precond), "bounded_sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gmres_ms_per_iter": 1e3 * (rep["t_mv"] + rep["t_prec"] + rep["t_orth"]) / max(rep["n_gmres_total"], 1),
        "note": "the unmodified reference (oracle/_ref) is 2D/quad-only; this arm is the tier-B restatement "
                "(oracle/hdg_oracle.cpp, bit-identical to the reference on 2D quads) run on all host threads",
    }
    emit(line)


# ---- GPU arm ---------------------------------------------------------------------------------------
class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons DURING the timed region.  NVML in-process (a handful of light queries
    every 200 ms); polling through an `nvidia-smi -lms` child process was measured to add sporadic 20-100 ms stalls
    to individual solves, so it is only the fallback when the NVML binding is missing."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        super().__init__(daemon=True)
        self.device, self.rows, self.stop_flag = device, [], False
        self.proc = None

    def _run_nvml(self):
        import pynvml as nv
        nv.nvmlInit()
        h = None
        try:  # CUDA ordinal -> NVML handle through the UUID (the ordinals differ under CUDA_VISIBLE_DEVICES)
            import torch
            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            h = nv.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU-") else uuid)
        except Exception:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [v for v in vis.split(",") if v.strip().isdigit()]
            h = nv.nvmlDeviceGetHandleByIndex(int(ids[self.device]) if self.device < len(ids) else self.device)
        cmax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
        while not self.stop_flag:
            clk = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            util = float(nv.nvmlDeviceGetUtilizationRates(h).gpu)
            mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.rows.append([clk, cmax, util] + [bool(mask & bits[nm]) for nm in self.NAMES])
            time.sleep(0.2)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits", "-lms", "500"], stdout=subprocess.PIPE, text=True)
        for ln in self.proc.stdout:
            r = [c.strip() for c in ln.split(",")]
            try:
                self.rows.append([float(r[0]), float(r[1]), float(r[2])] + [v.lower().startswith("active") for v in r[3:7]])
            except (ValueError, IndexError):
                pass
            if self.stop_flag:
                break

    def run(self):
        try:
            self._run_nvml()
        except Exception:
            try:
                self._run_smi()
            except Exception:
                pass

    def finish(self):
        self.stop_flag = True
        if self.proc:
            self.proc.terminate()
        sm, mx, reasons = [], 0.0, set()
        for r in self.rows:
            mx = max(mx, r[1])
            if r[2] > 10:
                sm.append(r[0])
            for nm, v in zip(self.NAMES, r[3:7]):
                if v:
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples_under_load": len(sm)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic(a):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the matvec kernel from the committed
    ncu --set full capture of this workload (profiles/traffic.json), or None for other sizes."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        return t.get(f"block_matvec hex {a.n}^3 p={a.degree}")
    except Exception:
        return None


def run_ours(a):
    import torch
    import torch.distributed as dist
    import paper_2512_13619_b200 as hdg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    ctx = hdg.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)  # so torch.cuda.Event sees the launching stream

    if world == 1 and not a.force_dd:
        disc = hdg.Discretization.structured(ctx, "hex", n=a.n, degree=a.degree)
        n_dof_global = disc.n_dof
    else:
        # weak scaling: every rank owns an n^3 slab of an n x n x (n*world) box, partitioned by domain
        # decomposition (one ghost layer, halo exchange + all-reduce over NCCL)
        from paper_2512_13619_b200 import partition as P
        lo, hi = (0.0, 0.0, 0.0), (1.0, 1.0, float(world))
        coords, ev = P.box_hex_mesh(a.n, a.n, a.n * world, lo, hi)
        gm = P.global_mesh("hex", coords, ev, lo=lo, hi=hi)
        lm = P.build_my_local_mesh(gm, P.slab_partition(gm.ne, world), rank, dist if world > 1 else None)
        disc = P.make_discretization(ctx, lm, "hex", a.degree)
        P.install_nccl_comm(ctx, lm, dist if world > 1 else None)
        n_dof_global = gm.nf * disc.mpf
        del gm, coords, ev
    xq, xf = disc.quad_coords()
    pi = np.pi
    sinprod = lambda x: np.prod(np.sin(pi * x), axis=-1)
    # host-side model data and initial state in pinned memory: the step's inputs
    forcing_h = torch.from_numpy(np.ascontiguousarray(3 * pi * pi * sinprod(xq))).pin_memory()
    dirichlet_h = torch.from_numpy(np.ascontiguousarray(sinprod(xf))).pin_memory()
    u0_h = torch.zeros(disc.npe * disc.ne, dtype=torch.float64).pin_memory()
    uh0_h = torch.zeros(disc.n_dof, dtype=torch.float64).pin_memory()
    u_out = torch.empty_like(u0_h).pin_memory()
    uh_out = torch.empty_like(uh0_h).pin_memory()
    h2d = 8 * (forcing_h.numel() + dirichlet_h.numel() + u0_h.numel() + uh0_h.numel())
    d2h = 8 * (u_out.numel() + uh_out.numel())
    pspec = hdg.PrecondSpec(a.precond)
    gcfg, ncfg = hdg.GmresConfig(), hdg.NewtonConfig()

    def make_model(fq, dq):
        return hdg.Model(disc, "poisson", [1.0], forcing=lambda x: fq, dirichlet=lambda x: dq, exact=sinprod)

    # device-resident arm: model tables + state already in HBM
    model = make_model(forcing_h.numpy(), dirichlet_h.numpy())
    state = hdg.State(disc)
    zeros_u = torch.zeros(disc.npe * disc.ne, dtype=torch.float64, device="cuda")
    zeros_uh = torch.zeros(disc.n_dof, dtype=torch.float64, device="cuda")
    reports = []

    def step_resident():
        state.set("u", zeros_u)
        state.set("uhat", zeros_uh)
        reports.append(hdg.newton_solve(disc, model, state, ncfg, gcfg, pspec))

    def step_e2e():
        # the public-API call a user makes with HOST arrays: model data + initial state in, solution out
        m = make_model(forcing_h.numpy(), dirichlet_h.numpy())
        s = hdg.State(disc)
        s.set("u", u0_h.numpy())
        s.set("uhat", uh0_h.numpy())
        rep = hdg.newton_solve(disc, m, s, ncfg, gcfg, pspec)
        ctx.copy(u_out.numpy(), s.ptr("u"), u_out.numel())
        ctx.copy(uh_out.numpy(), s.ptr("uhat"), uh_out.numel())
        return rep

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, count_launches=False):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        if count_launches:
            ctx.reset_launch_count()
        e0.record(stream)
        for _ in range(steps):
            t_dbg = time.perf_counter()
            fn()
            if os.environ.get("BENCH_DEBUG"):
                torch.cuda.synchronize()
                print(f"[bench debug] step {1e3 * (time.perf_counter() - t_dbg):.1f} ms pool {hdg.hdg.pool_stats()}", file=sys.stderr)
        e1.record(stream)
        barrier()
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item()) * 1e-3

    for _ in range(a.warmup):
        step_resident()
    sampler = ClockSampler(local)
    sampler.start()
    reports.clear()
    t_res = timed(step_resident, a.steps, count_launches=True)
    launches = ctx.launch_count
    rep = reports[-1]
    step_e2e()
    t_e2e = timed(step_e2e, a.steps)
    clocks = sampler.finish()

    # ---- dominant-kernel roofline: the fused gather + block GEMV (team_gemv) of block_matvec --------
    mpf, nb, nf, ne, nfl, n_dof = disc.mpf, disc.nb, getattr(disc, 'nf_owned', disc.nf), disc.ne, disc.nfl, disc.n_dof
    ops = hdg.assemble_element_operators(disc, model, state)
    K, rhs = hdg.assemble_global(disc, ops)
    P = hdg.build_preconditioner(pspec, K, ops, disc)
    x = torch.randn(n_dof, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)

    def kernel_time(fn, reps=30):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3 / reps

    # FP64 pipe utilisation of static condensation (north star): one assemble_element_operators call =
    # quadrature assembly of the local blocks + q-elimination + E-bar^-1 + Schur complement, algorithmic flops of
    # SURVEY.md 8(d) against the DMMA peak measured with scripts/micro/fp64_peak.cu on this pool's B200s
    D_, pe_, npe_, qe_, nfp_ = disc.dim, disc.pe, disc.npe, disc.qe, disc.n_lfe * disc.qf
    fl_cond = D_ * (2 * npe_ ** 3 + 4 * npe_ ** 2 * nfl + 2 * npe_ * nfl ** 2) + 2 * npe_ ** 3 + 2 * npe_ ** 2 * nfl + 2 * npe_ * nfl ** 2
    fl_local = 2 * (1 + D_) * npe_ * npe_ * (qe_ + nfp_) + 2 * (1 + D_) * nfl * npe_ * disc.qf + 2 * npe_ * nfl * disc.qf
    t_cond = kernel_time(lambda: hdg.assemble_element_operators(disc, model, state), reps=5)
    t_mv = kernel_time(lambda: hdg.block_matvec(K, x, y))
    t_pc = kernel_time(lambda: P.apply_base(x, y))
    bytes_mv = 8 * nf * mpf * (mpf * nb + 2) + 8 * nf * nb          # K once + x + y + int64 neighbour table
    bytes_pc = (8 * ne * nfl * nfl + 8 * (2 * ne * nfl + 2 * nf * mpf)) if a.precond in ("asm", "ras") \
        else 8 * nf * mpf * (mpf + 2)
    # in-solve averages from one instrumented solve (CUDA events around every phase; adds syncs, so it
    # is NOT part of the timed steps above)
    ctx.enable_phase_timing(True)
    state.set("u", zeros_u)
    state.set("uhat", zeros_uh)
    rep_t = hdg.newton_solve(disc, model, state, ncfg, gcfg, pspec)
    ctx.enable_phase_timing(False)
    n_it = max(rep_t.n_gmres_total, 1)
    n_mv_calls = rep_t.n_gmres_total + 2 * rep_t.n_newton + sum(1 for _ in rep_t.gmres_per_newton)  # + residual evaluations
    peak, peak_src = peaks()
    achieved = bytes_mv / t_mv / 1e9
    err = disc.l2_error(state.u, sinprod)

    if rank == 0:
        line = {
            "metric": METRIC, "value": n_dof_global * a.steps / t_res, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * t_res / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(a.n, a.degree, a.precond), "trace_dofs_per_gpu": n_dof,
                       "elements_per_gpu": ne, "faces_per_gpu": nf,
                       "parallelism": "1 GPU" if world == 1 else
                       f"domain decomposition over {world} GPUs: n x n x (n*{world}) box in z-slabs, one ghost layer, "
                       f"NCCL halo exchange per operator application + all-reduce per Gram-Schmidt pass",
                       "trace_dofs_global": n_dof_global,
                       "l2_policy": "inputs larger than L2 (K = %.2f GB, ASM blocks = %.2f GB vs 126 MB L2)" %
                                    (8e-9 * nf * mpf * mpf * nb, 8e-9 * ne * nfl * nfl)},
            "e2e": {"value": n_dof_global * a.steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": 1e3 * t_e2e / a.steps},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "roofline": {"kernel": "stream_gemv_kernel<2,1> as block_matvec (fused neighbour gather + block-row GEMV, bulk-TMA ring)",
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_source": peak_src, "frac_of_8TBs": achieved / 8000.0,
                         "algorithmic_bytes_per_launch": bytes_mv, "avg_launch_us": 1e6 * t_mv, "traffic": ncu_traffic(a),
                         "in_solve_avg_launch_us": 1e6 * rep_t.t_mv / max(n_mv_calls, 1)},
            "precond_apply": {"kind": a.precond, "GBps": bytes_pc / t_pc / 1e9, "frac": bytes_pc / t_pc / 1e9 / peak,
                              "avg_us": 1e6 * t_pc, "algorithmic_bytes": bytes_pc},
            "condensation": {"what": "assemble_element_operators: local blocks (DMMA) + fused q-elimination + blocked Gauss-Jordan E-bar^-1 + Schur complement",
                             "ms": 1e3 * t_cond, "flops_per_element": fl_cond + fl_local, "achieved": (fl_cond + fl_local) * ne / t_cond / 1e12,
                             "peak": 37.2, "unit": "TFLOP/s", "frac": (fl_cond + fl_local) * ne / t_cond / 1e12 / 37.2,
                             "peak_source": "DMMA m8n8k4 peak measured with scripts/micro/fp64_peak.cu (DFMA pipe: 34.0)"},
            "newton_solve_s": t_res / a.steps, "n_newton": rep.n_newton, "n_gmres_total": rep.n_gmres_total,
            "gmres_ms_per_iter": 1e3 * (rep_t.t_mv + rep_t.t_prec + rep_t.t_orth) / n_it,
            "phase_s": {"t_ass": rep_t.t_ass, "t_mv": rep_t.t_mv, "t_prec": rep_t.t_prec, "t_orth": rep_t.t_orth,
                        "t_total": rep_t.t_total},
            "final_residual": rep.final_residual, "l2_error_vs_exact": err,
        }
        if world == 1 and not a.no_cpu_baseline:
            threads = os.cpu_count() or 1
            dt, nd, rc, _ = cpu_sample(a.cpu_n, a.degree, a.precond, threads)
            line["cpu_baseline"] = {
                "value": nd / dt, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": f"one Newton solve of hex {a.cpu_n}^3 p={a.degree} ({nd} trace DOFs, {rc['n_gmres_total']} GMRES "
                          f"iterations), tier-B oracle port, {dt:.1f} s",
                "gmres_ms_per_iter": 1e3 * (rc["t_mv"] + rc["t_prec"] + rc["t_orth"]) / max(rc["n_gmres_total"], 1)}
        emit(line)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
