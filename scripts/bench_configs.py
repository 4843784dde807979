"""Full-size runs of the five BASELINE.json configurations on one B200 (SURVEY.md section 8 size table):
per config the block-matvec and preconditioner-apply HBM GB/s (algorithmic bytes of SURVEY.md 8(d) / CUDA
event time), operator assembly / preconditioner build time, and one Newton(-GMRES) solve through the public
API.  Prints one JSON line per config and writes them to --out.

  python scripts/bench_configs.py --configs 1,2,3,4,5 --out gpurun_out/configs.json

This is a measurement script (not bench.py's contract line): bench.py stays on configs[1]."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"])
    except Exception:
        return 6650.0


CONFIGS = {
    1: dict(name="2D Poisson, quad 64^2, p=2, BJ-GMRES", shape="quad", n=64, degree=2, n_comp=1, case="poisson2d",
            precond=("bj", 0, "gmres"), dt=None),
    2: dict(name="3D Poisson, hex 28^3, p=3, ASM-GMRES", shape="hex", n=28, degree=3, n_comp=1, case="poisson",
            precond=("asm", 0, "gmres"), dt=None),
    3: dict(name="2D Burgers, jittered tri 2x512^2, p=4, Newton-GMRES, ASM + Chebyshev(10)", shape="tri", n=512, degree=4,
            n_comp=1, case="burgers", precond=("asm", 10, "chebyshev"), dt=None, jitter=0.2),
    4: dict(name="3D elasticity, jittered tet 6x32^3, p=2, M=3, ASM-GMRES", shape="tet", n=32, degree=2, n_comp=3,
            case="elasticity", precond=("asm", 0, "gmres"), dt=None, jitter=0.2),
    5: dict(name="3D compressible Navier-Stokes, hex 24^3, p=3, M=5, Newton-GMRES BJ, one backward-Euler step",
            shape="hex", n=24, degree=3, n_comp=5, case="navier_stokes", precond=("bj", 0, "gmres"), dt=0.01),
}


def run(cfg_id, a):
    import torch
    import paper_2512_13619_b200 as hdg
    cfg = dict(CONFIGS[cfg_id])
    if a.n.get(cfg_id):
        cfg["n"] = a.n[cfg_id]
    ctx = hdg.Context(0)
    for kv in a.tune.split(","):
        if kv:
            k, v = kv.split("=")
            hdg.set_tuning(k, int(v))
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    def ev_time(fn, reps):
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

    def wall(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        return time.perf_counter() - t0, r

    t_setup, disc = wall(lambda: hdg.Discretization.structured(ctx, cfg["shape"], n=cfg["n"], degree=cfg["degree"],
                                                               n_comp=cfg["n_comp"], jitter=cfg.get("jitter", 0.0)))
    kw = {"mu": 0.02} if cfg["case"] == "navier_stokes" else {}
    model = hdg.make_case_model(disc, cfg["case"], **kw)
    state = hdg.make_initial_state(disc, model)
    u0, uh0 = state.u, state.uhat
    dt = cfg["dt"]
    kind, pdeg, pkind = cfg["precond"]
    pspec = hdg.PrecondSpec(kind, poly_degree=pdeg, poly_kind=pkind)
    tkw = dict(dt=dt, u_prev=u0) if dt else {}

    # phases of one Newton iteration, timed separately (second call = warm allocator)
    hdg.assemble_element_operators(disc, model, state, **tkw)
    t_ass, ops = wall(lambda: hdg.assemble_element_operators(disc, model, state, **tkw))
    t_glob, (K, rhs) = wall(lambda: hdg.assemble_global(disc, ops))
    hdg.build_preconditioner(hdg.PrecondSpec(kind), K, ops, disc)
    t_pb, P = wall(lambda: hdg.build_preconditioner(hdg.PrecondSpec(kind), K, ops, disc))
    mpf, nb, nf, ne, nfl, n_dof = disc.mpf, disc.nb, disc.nf, disc.ne, disc.nfl, disc.n_dof
    x = torch.randn(n_dof, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    bytes_mv = 8 * nf * mpf * (mpf * nb + 2) + 8 * nf * nb
    bytes_pc = (8 * ne * nfl * nfl + 8 * (2 * ne * nfl + 2 * nf * mpf)) if kind in ("asm", "ras") else 8 * nf * mpf * (mpf + 2)
    small = bytes_mv < 200e6  # fits L2: report as L2-resident
    reps = 200 if small else 30
    t_mv = ev_time(lambda: hdg.block_matvec(K, x, y), reps)
    t_pc = ev_time(lambda: P.apply_base(x, y), reps)
    peak = peak_gbs()
    del P, K, rhs, ops

    if a.no_solve:
        ctx.close()
        return {"config": cfg_id, "name": cfg["name"], "tuning": a.tune,
                "matvec_GBps": bytes_mv / t_mv / 1e9, "matvec_frac": bytes_mv / t_mv / 1e9 / peak, "matvec_us": 1e6 * t_mv,
                "precond_GBps": bytes_pc / t_pc / 1e9, "precond_frac": bytes_pc / t_pc / 1e9 / peak, "precond_us": 1e6 * t_pc,
                "assemble_element_operators_s": t_ass, "assemble_global_s": t_glob, "precond_build_s": t_pb}
    # one complete solve from the initial state (second run timed: warm allocator, as in bench.py)
    gcfg, ncfg = hdg.GmresConfig(), hdg.NewtonConfig()

    def solve():
        state.set("u", u0)
        state.set("uhat", uh0)
        return hdg.newton_solve(disc, model, state, ncfg, gcfg, pspec, **tkw)

    solve()
    t_solve, rep = wall(solve)
    ctx.enable_phase_timing(True)
    rep_t = solve()
    ctx.enable_phase_timing(False)
    n_it = max(rep_t.n_gmres_total, 1)
    line = {
        "config": cfg_id, "name": cfg["name"], "ne": ne, "nf": nf, "mpf": mpf, "nb": nb, "npe": disc.npe, "nfl": nfl,
        "n_dof": n_dof, "K_GB": 8e-9 * nf * mpf * mpf * nb,
        "matvec": {"us": 1e6 * t_mv, "GBps": bytes_mv / t_mv / 1e9, "frac_of_measured_peak": bytes_mv / t_mv / 1e9 / peak,
                   "algorithmic_bytes": bytes_mv, "l2_resident": small},
        "precond_apply": {"kind": kind, "us": 1e6 * t_pc, "GBps": bytes_pc / t_pc / 1e9,
                          "frac_of_measured_peak": bytes_pc / t_pc / 1e9 / peak, "algorithmic_bytes": bytes_pc},
        "assemble_element_operators_s": t_ass, "assemble_global_s": t_glob, "precond_build_s": t_pb,
        "newton_solve_s": t_solve, "converged": bool(rep.converged), "n_newton": rep.n_newton,
        "n_gmres_total": rep.n_gmres_total, "gmres_per_newton": list(rep.gmres_per_newton),
        "n_inner_prec_ops": rep.n_inner_prec_ops, "final_residual": rep.final_residual,
        "gmres_ms_per_iter": 1e3 * (rep_t.t_mv + rep_t.t_prec + rep_t.t_orth) / n_it,
        "dofs_per_s": n_dof / t_solve,
        "phase_s": {"t_ass": rep_t.t_ass, "t_mv": rep_t.t_mv, "t_prec": rep_t.t_prec, "t_orth": rep_t.t_orth,
                    "t_total": rep_t.t_total},
        "host_setup_s": t_setup, "peak_GBps": peak,
    }
    if model.exact_solution is not None:
        line["l2_error_vs_exact"] = disc.l2_error(state.u, model.exact_solution)
    ctx.close()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--out", default="gpurun_out/configs.json")
    ap.add_argument("--n", default="", help="override mesh sizes, e.g. 5=24,3=256")
    ap.add_argument("--no-solve", action="store_true", help="kernel and phase timings only")
    ap.add_argument("--tune", default="", help="tuning knobs, e.g. stream_packed=0,stream_packed_stage_bytes=4096")
    a = ap.parse_args()
    a.n = {int(k): int(v) for k, v in (kv.split("=") for kv in a.n.split(",") if kv)}
    lines = []
    for c in [int(s) for s in a.configs.split(",")]:
        try:
            ln = run(c, a)
        except Exception as e:  # report and continue with the next config
            ln = {"config": c, "name": CONFIGS[c]["name"], "error": f"{type(e).__name__}: {e}"}
        print(json.dumps(ln), flush=True)
        lines.append(ln)
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text("\n".join(json.dumps(l) for l in lines) + "\n")


if __name__ == "__main__":
    main()
