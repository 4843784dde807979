"""Command-line front end mirroring the reference's `hdgsolve` (proj/src/cli.cpp:186-380): subcommands
solve / sweep / rates / dump, the same option names, the same exit codes (cli.hpp:5-6: 0 ok,
1 usage, 2 not converged, 3 numerical failure).

    python -m paper_2512_13619_b200 solve --case burgers2d --k 2 --n 32 --precond asm --poly-degree 10
"""
from __future__ import annotations

import argparse
import sys

from . import hdg as H
from . import study as S

EXIT_OK, EXIT_USAGE, EXIT_NOT_CONVERGED, EXIT_NUMERICAL = 0, 1, 2, 3


def add_case_options(p, with_kn=True):
    p.add_argument("--case", default="burgers2d", dest="case_name")
    p.add_argument("--shape", default=None, choices=["quad", "hex", "tri", "tet"])
    if with_kn:
        p.add_argument("--k", type=int, default=1)
        p.add_argument("--n", type=int, default=16)
    p.add_argument("--precond", default="bj", choices=["none", "bj", "asm", "ras"])
    p.add_argument("--poly-degree", type=int, default=0)
    p.add_argument("--poly-kind", default="gmres", choices=["gmres", "chebyshev"])
    p.add_argument("--ritz-seed", type=int, default=12345)
    p.add_argument("--ritz-per-restart", action="store_true")
    p.add_argument("--restart", type=int, default=50)
    p.add_argument("--gmres-tol", type=float, default=1e-6)
    p.add_argument("--max-gmres", type=int, default=1000)
    p.add_argument("--orth", default="cgs", choices=["cgs", "mgs"])
    p.add_argument("--newton-tol", type=float, default=1e-8)
    p.add_argument("--max-newton", type=int, default=50)
    p.add_argument("--min-alpha", type=float, default=1.0 / 1024.0)
    p.add_argument("--steady", action="store_true")
    p.add_argument("--dt", type=float, default=None)
    p.add_argument("--steps", type=int, default=1)
    p.add_argument("--tau", type=float, default=None)
    p.add_argument("--nu", type=float, default=1.0 / 200.0)
    p.add_argument("--kappa", type=float, default=1.0)
    p.add_argument("--velocity", default="0,1")
    p.add_argument("--quad-points", type=int, default=0)
    p.add_argument("--device", type=int, default=0)


def to_spec(a, k=None, n=None, precond=None, poly=None):
    if a.dt is not None and a.steady:
        raise SystemExit(EXIT_USAGE)
    return S.CaseSpec(case_name=a.case_name, k=k if k is not None else a.k, n=n if n is not None else a.n,
                      precond=H.PrecondSpec(precond or a.precond, poly_degree=a.poly_degree if poly is None else poly,
                                            ritz_seed=a.ritz_seed, ritz_per_restart=a.ritz_per_restart, poly_kind=a.poly_kind),
                      gmres=H.GmresConfig(restart=a.restart, tol=a.gmres_tol, max_iters=a.max_gmres, orth=a.orth),
                      newton=H.NewtonConfig(tol=a.newton_tol, max_newton=a.max_newton, min_alpha=a.min_alpha),
                      dt=a.dt, n_steps=a.steps, tau=a.tau, nu=a.nu, kappa=a.kappa,
                      velocity=tuple(float(v) for v in a.velocity.split(",")), quad_points=a.quad_points, shape=a.shape)


def print_summary(r):
    s, rep = r.spec, r.report
    kind = {0: "none", 1: "bj", 2: "asm", 3: "ras"}[s.precond.kind]
    print(f"case:           {s.case_name}  k={s.k}  n={s.n}  precond={kind}  poly={s.precond.poly_degree}")
    print("mode:           " + (f"transient dt={s.dt} steps={s.n_steps}" if s.dt else "steady"))
    print(f"converged:      {'yes' if rep.converged else 'no'}")
    print(f"newton iters:   {rep.n_newton}")
    print(f"gmres iters:    {rep.n_gmres_total}")
    if rep.n_inner_prec_ops > 0:
        print(f"poly inner ops: {rep.n_inner_prec_ops}")
    print(f"final residual: {rep.final_residual:.6e}")
    print(f"t_ass={rep.t_ass:.4f}s t_mv={rep.t_mv:.4f}s t_prec={rep.t_prec:.4f}s t_orth={rep.t_orth:.4f}s t_total={rep.t_total:.4f}s")


def exit_code(r):
    if r.ok:
        return EXIT_OK if r.report.converged else EXIT_NOT_CONVERGED
    if r.numerical_failure:
        return EXIT_NUMERICAL
    return EXIT_NOT_CONVERGED if "line search" in r.error else EXIT_USAGE


def main(argv=None):
    ap = argparse.ArgumentParser(prog="hdgsolve-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p_solve = sub.add_parser("solve")
    add_case_options(p_solve)
    p_solve.add_argument("--dump-matrix", default=None)
    p_solve.add_argument("--verbose", action="store_true")
    p_sweep = sub.add_parser("sweep")
    add_case_options(p_sweep, with_kn=False)
    p_sweep.add_argument("--ks", default="1,2")
    p_sweep.add_argument("--ns", default="16,32")
    p_sweep.add_argument("--preconds", default="bj,asm")
    p_sweep.add_argument("--out", default="-")
    p_sweep.add_argument("--json", default=None)
    p_sweep.add_argument("--repeat", type=int, default=1)
    p_sweep.add_argument("--warmup", action="store_true")
    p_rates = sub.add_parser("rates")
    add_case_options(p_rates, with_kn=False)
    p_rates.add_argument("--ks", default="1,2")
    p_rates.add_argument("--ns", default="4,8,16")
    p_dump = sub.add_parser("dump")
    add_case_options(p_dump)
    p_dump.add_argument("--out", required=True)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code not in (0, None) else 0
    try:
        ctx = H.Context(a.device)
    except H.HdgError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    ints = lambda s: [int(v) for v in s.split(",") if v]
    try:
        if a.cmd == "solve":
            ctx.enable_phase_timing(True)
            r = S.run_case(ctx, to_spec(a))
            if not r.ok:
                print(f"error: {r.error}", file=sys.stderr)
            print_summary(r)
            if a.verbose and hasattr(r.report, "residual_history"):
                for i, (res, it) in enumerate(zip(r.report.residual_history[1:], r.report.gmres_per_newton)):
                    print(f"  newton {i}: residual {res:.6e}  gmres {it}", file=sys.stderr)
            if a.dump_matrix and r.ok:
                ops = H.assemble_element_operators(r.disc, r.model, r.state)
                K, rhs = H.assemble_global(r.disc, ops)
                H.write_matrix(a.dump_matrix, K, rhs)
            return exit_code(r)
        if a.cmd == "dump":
            spec = to_spec(a)
            disc, model = S.make_case_setup(ctx, spec)
            state = H.make_initial_state(disc, model)
            ops = H.assemble_element_operators(disc, model, state)
            K, rhs = H.assemble_global(disc, ops)
            H.write_matrix(a.out, K, rhs)
            print(f"wrote {a.out}: nf={K.nf} block={K.block_dim} nb={K.nb}")
            return EXIT_OK
        if a.cmd == "sweep":
            specs = []
            for k in ints(a.ks):
                for n in ints(a.ns):
                    for pc in a.preconds.split(","):
                        base = {"bj-pp": "bj", "asm-pp": "asm", "pp": "none"}.get(pc, pc)
                        poly = (a.poly_degree if a.poly_degree > 0 else 10) if pc.endswith("pp") else 0
                        specs.append(to_spec(a, k=k, n=n, precond=base, poly=poly))
            out = sys.stdout if a.out == "-" else open(a.out, "w", newline="")
            res = S.run_sweep(ctx, specs, out, repeat=a.repeat, warmup=a.warmup)
            if a.json:
                S.write_json_report(res, a.json)
            codes = [exit_code(r) for r in res]
            return max(codes) if codes else EXIT_OK
        if a.cmd == "rates":
            rows = S.convergence_study(ctx, to_spec(a, k=1, n=4), ints(a.ks), ints(a.ns))
            print("k,n,l2_error,order")
            for row in rows:
                print(f"{row['k']},{row['n']},{row['error']:.6e},{row['order']}")
            return EXIT_OK
    except H.HdgError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_NUMERICAL if isinstance(e, S._NUMERICAL) else EXIT_USAGE
    finally:
        ctx.close()
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
