"""One Newton solve of a BASELINE config through the public API (for ncu launch lists / kernel captures):
  python scripts/one_solve.py --config 2 [--warm 1]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from scripts.bench_configs import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--warm", type=int, default=0, help="untimed solves before the last one")
    ap.add_argument("--n", type=int, default=0)
    a = ap.parse_args()
    import paper_2512_13619_b200 as hdg
    cfg = dict(CONFIGS[a.config])
    if a.n:
        cfg["n"] = a.n
    ctx = hdg.Context(0)
    disc = hdg.Discretization.structured(ctx, cfg["shape"], n=cfg["n"], degree=cfg["degree"], n_comp=cfg["n_comp"],
                                         jitter=cfg.get("jitter", 0.0))
    kw = {"mu": 0.02} if cfg["case"] == "navier_stokes" else {}
    model = hdg.make_case_model(disc, cfg["case"], **kw)
    state = hdg.make_initial_state(disc, model)
    u0, uh0 = state.u, state.uhat
    kind, pdeg, pkind = cfg["precond"]
    tkw = dict(dt=cfg["dt"], u_prev=u0) if cfg["dt"] else {}
    for _ in range(a.warm + 1):
        state.set("u", u0)
        state.set("uhat", uh0)
        rep = hdg.newton_solve(disc, model, state, hdg.NewtonConfig(), hdg.GmresConfig(),
                               hdg.PrecondSpec(kind, poly_degree=pdeg, poly_kind=pkind), **tkw)
    print(rep)
    ctx.close()


if __name__ == "__main__":
    main()
