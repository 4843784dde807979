"""Regenerates tests/golden/reference_golden.npz from the UNMODIFIED reference compiled in place
(oracle/_ref; needs /root/reference at build time -- run `make -C oracle ref` first).
Run from the repo root:  python tests/golden/make_golden.py"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, str(ROOT))
from oracle import ref  # noqa: E402

out = {}
rc = ref.RefCase("poisson2d", k=2, n=64)
r = rc.newton(precond="bj")
out["cfg1_n_newton"], out["cfg1_n_gmres"] = r["n_newton"], r["n_gmres_total"]
out["cfg1_final_residual"] = r["final_residual"]
out["cfg1_sum_uhat2"] = np.sum(rc.get("uhat") ** 2)
out["cfg1_uhat_head"] = rc.get("uhat")[:512]
rc = ref.RefCase("poisson2d", k=2, n=64)
r = rc.newton(precond="asm")
out["cfg1_asm_n_newton"], out["cfg1_asm_n_gmres"] = r["n_newton"], r["n_gmres_total"]
for name, nn in [("burgers_k1_n16_bj", "bj"), ("burgers_k1_n16_asm", "asm")]:
    rc = ref.RefCase("burgers2d", k=1, n=16)
    r = rc.newton(precond=nn)
    out[name + "_n_newton"], out[name + "_n_gmres"] = r["n_newton"], r["n_gmres_total"]
    out[name + "_gmres_per_newton"] = r["gmres_per_newton"]
    out[name + "_sum_uhat2"] = np.sum(rc.get("uhat") ** 2)
    out[name + "_uhat"] = rc.get("uhat")
rc = ref.RefCase("burgers2d", k=1, n=16)
r = rc.newton(precond="asm", poly_degree=10)
out["burgers_k1_n16_asmpp10_n_gmres"] = r["n_gmres_total"]
out["burgers_k1_n16_asmpp10_gmres_per_newton"] = r["gmres_per_newton"]
for tag, case, k, n in [("p", "poisson2d", 2, 4), ("b", "burgers2d", 2, 3)]:
    rc = ref.RefCase(case, k=k, n=n)
    rc.perturb(5, 0.1)
    out[f"{tag}_u"], out[f"{tag}_uhat"] = rc.get("u"), rc.get("uhat")
    rc.assemble()
    out[f"{tag}_blocks"], out[f"{tag}_rhs"] = rc.get("k_blocks"), rc.get("rhs")
    out[f"{tag}_neighbor"] = rc.get_i("neighbor")
    out[f"{tag}_kbar"] = rc.get("kbar")
    x = ref.random_vector(rc.n_dof, 42)
    out[f"{tag}_x"], out[f"{tag}_kx"] = x, rc.matvec(x)
    rc.build_precond("bj")
    out[f"{tag}_bj_x"] = rc.apply_base(x)
    rc.build_precond("asm")
    out[f"{tag}_asm_x"] = rc.apply_base(x)
    xs, st = rc.gmres(tol=1e-10, max_iters=300)
    out[f"{tag}_gmres_x"], out[f"{tag}_gmres_iters"] = xs, st["iters"]
np.savez_compressed(ROOT / "tests" / "golden" / "reference_golden.npz", **out)
print({k: (v if np.ndim(v) == 0 else np.shape(v)) for k, v in out.items()})
