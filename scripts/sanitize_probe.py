"""Small invocations of every hand-written kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
the DMMA local-assembly kernel (hex p = 3), fused q-elimination, blocked Gauss-Jordan, the bulk-TMA stream GEMV in
plain and packed mode (forced on for small problems), the TMA-streamed CGS2 passes, the fused polynomial epilogues, the one-kernel Schur complement.

  compute-sanitizer --tool racecheck python scripts/sanitize_probe.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import paper_2512_13619_b200 as hdg  # noqa: E402

ctx = hdg.Context(0)
hdg.set_tuning("stream_min_elems", 0)       # route the small GEMVs through the TMA stream kernel too
cases = [("hex", 3, 3, "poisson", hdg.PrecondSpec("asm")),
         ("hex", 2, 3, "navier_stokes", hdg.PrecondSpec("bj")),       # wide system: records through the L2 scratch, split operand build
         ("hex", 2, 3, "elasticity", hdg.PrecondSpec("asm")),
         ("tri", 6, 4, "burgers", hdg.PrecondSpec("asm", poly_degree=4, poly_kind="chebyshev")),
         ("quad", 6, 2, "burgers", hdg.PrecondSpec("bj", poly_degree=5))]
for shape, n, k, case, pspec in cases:
    ncomp = {"navier_stokes": 5, "elasticity": 3}.get(case, 1)
    disc = hdg.Discretization.structured(ctx, shape, n=n, degree=k, n_comp=ncomp, jitter=0.1 if shape == "tri" else 0.0)
    model = hdg.make_case_model(disc, case, **({"mu": 0.02} if case == "navier_stokes" else {}))
    state = hdg.make_initial_state(disc, model)
    tkw = dict(dt=0.05, u_prev=state.u) if case == "navier_stokes" else {}
    rep = hdg.newton_solve(disc, model, state, pspec=pspec, **tkw)
    assert rep.converged, (shape, rep)
    print(shape, k, case, "newton", rep.n_newton, "gmres", rep.n_gmres_total, "launches", ctx.launch_count)
# the 16-warp variant of the local kernel
hdg.set_tuning("local_nt", 512)
disc = hdg.Discretization.structured(ctx, "hex", n=2, degree=3)
model = hdg.make_case_model(disc, "poisson")
ops = hdg.assemble_element_operators(disc, model, hdg.make_initial_state(disc, model))
hdg.set_tuning("local_nt", 256)
print("16-warp local kernel ok")
# the chunked shared-memory operand builder (the streamed table-ring pipeline is the default for hex p = 3) and the 16-warp streamed sweep of wide systems
for stream, ntw in ((0, 256), (1, 256), (2, 256), (3, 512)):
    hdg.set_tuning("local_ed_stream", stream)
    hdg.set_tuning("local_nt_wide", ntw)
    for case, ncomp in (("poisson", 1), ("navier_stokes", 5)):
        disc = hdg.Discretization.structured(ctx, "hex", n=2, degree=3, n_comp=ncomp)
        model = hdg.make_case_model(disc, case, **({"mu": 0.02} if case == "navier_stokes" else {}))
        st = hdg.make_initial_state(disc, model)
        ops = hdg.assemble_element_operators(disc, model, st, **(dict(dt=0.05, u_prev=st.u) if ncomp > 1 else {}))
hdg.set_tuning("local_ed_stream", 3)
hdg.set_tuning("local_nt_wide", 256)
print("local kernel variants ok")
# the one-kernel Schur complement over its warp counts and both copy widths (npe odd: 8-byte cp.async, k padded)
for shape, k, case, ncomp in (("hex", 2, "poisson", 1), ("tet", 2, "elasticity", 3), ("quad", 3, "elasticity", 2), ("tet", 3, "poisson", 1)):
    disc = hdg.Discretization.structured(ctx, shape, n=2, degree=k, n_comp=ncomp)
    model = hdg.make_case_model(disc, case)
    ops = hdg.assemble_element_operators(disc, model, hdg.make_initial_state(disc, model))
print("fused Schur variants ok")
# the streamed CGS2 passes on a basis long enough for the TMA path
n, nvec = 1 << 16, 6
V, _ = np.linalg.qr(hdg.random_vector(n * nvec, 1).reshape(n, nvec))
h, w = hdg.orthogonalize(ctx, np.ascontiguousarray(V.T), hdg.random_vector(n, 2))
assert abs(np.linalg.norm(w) - 1.0) < 1e-12 and np.max(np.abs(V.T @ w)) < 1e-12
print("cgs ok")
ctx.close()
