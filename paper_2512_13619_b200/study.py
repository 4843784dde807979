"""Study harness over the B200 hot path: the reference's CaseSpec / run_case / run_sweep /
convergence_study (proj/include/hdg/study.hpp:14-85, proj/src/study.cpp) with the same CSV schema v1
(study.cpp:139-155) and JSON mirror (:190-221), plus the columns SURVEY.md section 5 asks for
(shape, ngpu).  Control-plane code: thin Python over the C ABI."""
from __future__ import annotations

import csv
import io
import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import hdg as H

CSV_SCHEMA_VERSION = 1
CSV_COLUMNS = ["schema_version", "case", "k", "n", "precond", "poly_degree", "mode", "dt", "steps", "n_newton", "n_gmres",
               "converged", "residual_final", "t_ass", "t_mv", "t_prec", "t_orth", "t_total", "t_total_median", "seed"]
EXTRA_COLUMNS = ["shape", "n_dof", "ngpu"]

_CASE_SHAPE = {"poisson2d": "quad", "convdiff2d": "quad", "burgers2d": "quad", "heat2d": "quad", "poisson3d": "hex"}


@dataclass
class CaseSpec:
    """study.hpp:14-26 (+ shape / n_comp for the configurations the reference cannot run)."""
    case_name: str = "burgers2d"
    k: int = 1
    n: int = 16
    precond: H.PrecondSpec = field(default_factory=H.PrecondSpec)
    gmres: H.GmresConfig = field(default_factory=H.GmresConfig)
    newton: H.NewtonConfig = field(default_factory=H.NewtonConfig)
    dt: float | None = None
    n_steps: int = 1
    tau: float | None = None
    nu: float = 1.0 / 200.0
    kappa: float = 1.0
    velocity: tuple = (0.0, 1.0)
    quad_points: int = 0
    shape: str | None = None

    def resolved_shape(self):
        return self.shape or _CASE_SHAPE.get(self.case_name, "quad")


@dataclass
class CaseResult:
    spec: CaseSpec
    report: object = None
    steps: list = field(default_factory=list)
    state: object = None
    disc: object = None
    model: object = None
    ok: bool = True
    numerical_failure: bool = False
    error: str = ""


_NUMERICAL = (H.SingularBlock, H.NonFiniteState, H.NaNDetected)  # errors.hpp:107-114 is_numerical_failure


class _Totals:
    def __init__(self):
        self.n_newton = self.n_gmres_total = self.n_inner_prec_ops = 0
        self.t_ass = self.t_mv = self.t_prec = self.t_orth = self.t_total = 0.0
        self.final_residual, self.converged = 0.0, False


def make_case_setup(ctx, spec: CaseSpec):
    disc = H.Discretization.structured(ctx, spec.resolved_shape(), n=spec.n, degree=spec.k, quad_points=spec.quad_points)
    model = H.make_case_model(disc, spec.case_name, tau=spec.tau, nu=spec.nu, kappa=spec.kappa, velocity=spec.velocity)
    return disc, model


def run_case_once(ctx, spec: CaseSpec, setup=None) -> CaseResult:
    """run_case_once (study.cpp:96-130): solver errors are captured, not raised."""
    res = CaseResult(spec)
    try:
        disc, model = setup or make_case_setup(ctx, spec)
        res.disc, res.model = disc, model
        state = H.make_initial_state(disc, model)
        res.state = state
        if spec.dt:
            res.steps = H.time_march(disc, model, state, spec.dt, spec.n_steps, spec.newton, spec.gmres, spec.precond)
            tot = _Totals()
            for s in res.steps:
                tot.n_newton += s.n_newton
                tot.n_gmres_total += s.n_gmres_total
                tot.n_inner_prec_ops += s.n_inner_prec_ops
                for nm in ("t_ass", "t_mv", "t_prec", "t_orth", "t_total"):
                    setattr(tot, nm, getattr(tot, nm) + getattr(s, nm))
            tot.converged = bool(res.steps) and all(s.converged for s in res.steps)
            tot.final_residual = res.steps[-1].final_residual if res.steps else 0.0
            res.report = tot
        else:
            res.report = H.newton_solve(disc, model, state, spec.newton, spec.gmres, spec.precond)
    except H.HdgError as e:
        res.ok = False
        res.numerical_failure = isinstance(e, _NUMERICAL)
        res.error = str(e)
        res.report = getattr(e, "report", None) or _Totals()
        res.report.converged = False
    return res


def run_case(ctx, spec: CaseSpec) -> CaseResult:
    return run_case_once(ctx, spec)


def _fmt(v):
    return f"{v:.12g}"


def csv_row(r: CaseResult, t_total_median: float, ngpu=1):
    s, rep = r.spec, r.report
    kind = {0: "none", 1: "bj", 2: "asm", 3: "ras"}[s.precond.kind]
    return [CSV_SCHEMA_VERSION, s.case_name, s.k, s.n, kind, s.precond.poly_degree, "transient" if s.dt else "steady",
            _fmt(s.dt) if s.dt else "", s.n_steps if s.dt else "", rep.n_newton, rep.n_gmres_total,
            "true" if rep.converged else "false", _fmt(rep.final_residual), _fmt(rep.t_ass), _fmt(rep.t_mv), _fmt(rep.t_prec),
            _fmt(rep.t_orth), _fmt(rep.t_total), _fmt(t_total_median), s.precond.ritz_seed,
            s.resolved_shape(), r.disc.n_dof if r.disc is not None else "", ngpu]


def run_sweep(ctx, specs, out, repeat=1, warmup=False):
    """run_sweep (study.cpp:157-188): one CSV row per case, best-of-repeat timings + median total."""
    w = csv.writer(out, lineterminator="\r\n")
    w.writerow(CSV_COLUMNS + EXTRA_COLUMNS)
    ctx.enable_phase_timing(True)
    results = []
    try:
        for spec in specs:
            best, totals = None, []
            try:
                setup = make_case_setup(ctx, spec)
                if warmup:
                    run_case_once(ctx, spec, setup)
                for _ in range(max(1, repeat)):
                    r = run_case_once(ctx, spec, setup)
                    totals.append(r.report.t_total)
                    if best is None or r.report.t_total < best.report.t_total:
                        best = r
            except H.HdgError as e:
                best = CaseResult(spec, report=_Totals(), ok=False, error=str(e))
                totals.append(0.0)
            totals.sort()
            w.writerow(csv_row(best, totals[len(totals) // 2]))
            out.flush()
            results.append(best)
    finally:
        ctx.enable_phase_timing(False)
    return results


def write_json_report(results, path):
    rows = []
    for r in results:
        s, rep = r.spec, r.report
        row = {"schema_version": CSV_SCHEMA_VERSION, "case": s.case_name, "k": s.k, "n": s.n,
               "precond": {0: "none", 1: "bj", 2: "asm", 3: "ras"}[s.precond.kind], "poly_degree": s.precond.poly_degree,
               "mode": "transient" if s.dt else "steady"}
        if s.dt:
            row["dt"], row["steps"] = s.dt, s.n_steps
        row.update(n_newton=rep.n_newton, n_gmres=rep.n_gmres_total, converged=bool(rep.converged),
                   residual_final=rep.final_residual, t_ass=rep.t_ass, t_mv=rep.t_mv, t_prec=rep.t_prec, t_orth=rep.t_orth,
                   t_total=rep.t_total, seed=s.precond.ritz_seed)
        if not r.ok:
            row["error"] = r.error
        rows.append(row)
    with open(path, "w") as f:
        json.dump(rows, f, indent=2)
        f.write("\n")


def convergence_study(ctx, base: CaseSpec, ks, ns):
    """convergence_study (study.cpp:223-261): L2 errors and observed orders with tightened tolerances."""
    rows = []
    for k in ks:
        prev_err, prev_n = 0.0, 0
        for n in ns:
            spec = CaseSpec(**{**base.__dict__, "k": k, "n": n})
            spec.gmres = H.GmresConfig(restart=base.gmres.restart, tol=1e-12, max_iters=base.gmres.max_iters)
            spec.newton = H.NewtonConfig(tol=1e-10, max_newton=base.newton.max_newton, min_alpha=base.newton.min_alpha)
            r = run_case_once(ctx, spec)
            if not r.ok:
                raise H.HdgError("convergence study case failed: " + r.error)
            if r.model.exact_solution is None:
                raise H.HdgError(f"case '{spec.case_name}' has no exact solution")
            err = r.disc.l2_error(r.state.u, r.model.exact_solution)
            order = ""
            if prev_n:
                order = "exact" if (err <= 1e-10 and prev_err <= 1e-10) else _fmt(math.log(prev_err / err) / math.log(n / prev_n))
            rows.append({"k": k, "n": n, "error": err, "order": order})
            prev_err, prev_n = err, n
    return rows
