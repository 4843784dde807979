"""The FP64 tensor-core (DMMA) paths against the scalar FMA paths they replace, on the same inputs: raw
local blocks (E, D_d, F, G_d, H, J), condensed operators, the assembled block rows and the preconditioner
inverses must agree to rounding for every element shape / model family (the scalar paths are the ones
pinned bit-level against the CPU oracle in the other parity suites)."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg

pytestmark = pytest.mark.gpu

CASES = [("quad", 5, 2, 1, "poisson2d"), ("quad", 4, 3, 1, "burgers"), ("tri", 4, 4, 1, "burgers"), ("hex", 3, 3, 1, "poisson"),
         ("hex", 3, 2, 1, "reaction"), ("tet", 2, 2, 1, "poisson"), ("tet", 2, 2, 3, "elasticity"), ("quad", 4, 2, 2, "elasticity"),
         ("hex", 2, 2, 5, "navier_stokes"), ("quad", 3, 3, 4, "navier_stokes"),
         # element sizes between the tensor-core threshold (pe = 20) and its limit (pe = 64), odd sizes included
         ("quad", 4, 4, 1, "burgers"), ("quad", 3, 5, 1, "poisson2d"), ("tri", 3, 5, 1, "poisson2d"), ("tri", 3, 6, 1, "burgers"),
         ("tet", 2, 3, 1, "poisson"), ("tet", 1, 4, 1, "poisson"), ("quad", 2, 6, 1, "poisson2d"),
         # a wide system whose point records go through the L2 scratch (hex p = 3, three components)
         ("hex", 2, 3, 3, "elasticity")]


def rel(a, b):
    return np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b)))


@pytest.mark.parametrize("shape,n,k,M,case", CASES)
def test_dmma_paths_match_scalar_paths(ctx, shape, n, k, M, case):
    disc = hdg.Discretization.structured(ctx, shape, n=n, degree=k, n_comp=M, jitter=0.15 if shape in ("tri", "tet") else 0.0)
    kw = {"mu": 0.02} if case == "navier_stokes" else {}
    model = hdg.make_case_model(disc, case, **kw)
    state = hdg.make_initial_state(disc, model)
    rng = np.random.default_rng(3)
    state.u = state.u + 0.05 * rng.standard_normal(state.u.shape)       # away from the trivial state
    state.uhat = state.uhat + 0.05 * rng.standard_normal(state.uhat.shape)
    tkw = dict(dt=0.05, u_prev=state.u) if case == "navier_stokes" else {}
    out = {}
    for flag in (0, 1):
        hdg.set_tuning("use_dmma", flag)
        hdg.set_tuning("use_blocked_gj", flag)
        hdg.set_tuning("local_dmma_min_pe", 0)   # small elements too (default: tensor-core path from pe = 20)
        try:
            ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True, **tkw)
            K, rhs = hdg.assemble_global(disc, ops)
            P = hdg.build_preconditioner("asm", K, ops, disc)
            names = ["e_raw", "f_raw", "h_raw", "j_raw"] + [f"d_raw{d}" for d in range(disc.dim)] + \
                    [f"g_raw{d}" for d in range(disc.dim)] + ["kbar", "ebar_inv", "fbar", "hbar", "rbar", "ru"]
            out[flag] = {nm: ops.get(nm) for nm in names}
            out[flag]["K"] = K.blocks
            out[flag]["rhs"] = rhs
            out[flag]["asm_inv"] = P.get("asm_inv")
        finally:
            hdg.set_tuning("use_dmma", 1)
            hdg.set_tuning("use_blocked_gj", 1)
            hdg.set_tuning("local_dmma_min_pe", 20)
    for nm in out[0]:
        a, b = np.asarray(out[1][nm]), np.asarray(out[0][nm])
        tol = 1e-9 if nm in ("asm_inv", "ebar_inv", "kbar", "K", "rbar", "rhs") else 1e-12
        assert rel(a, b) <= tol, (nm, rel(a, b))


def test_point_chunked_sweep_with_tensor_core_blocks(ctx):
    """Wide systems sweep the quadrature points in chunks that accumulate into the blocks; with
    `local_dmma_chunked` the E / D_d part of every chunk runs on the tensor-core path (off by default)."""
    disc = hdg.Discretization.structured(ctx, "hex", n=2, degree=2, n_comp=5)
    model = hdg.make_case_model(disc, "navier_stokes", mu=0.02)
    state = hdg.make_initial_state(disc, model)
    out = {}
    for flag in (0, 1):
        hdg.set_tuning("local_dmma_chunked", flag)
        hdg.set_tuning("local_global_records", 0)   # otherwise the single-launch L2-scratch path takes over
        try:
            ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True, dt=0.05, u_prev=state.u)
            out[flag] = {nm: ops.get(nm) for nm in ["e_raw", "d_raw0", "d_raw1", "d_raw2", "f_raw", "h_raw", "j_raw", "kbar", "ru"]}
        finally:
            hdg.set_tuning("local_dmma_chunked", 0)
            hdg.set_tuning("local_global_records", 1)
    for nm in out[0]:
        assert rel(out[1][nm], out[0][nm]) <= (1e-9 if nm == "kbar" else 1e-12), nm


@pytest.mark.parametrize("nvec,n", [(1, 1000), (7, 12345), (50, 70001), (64, 5000), (65, 3000)])
def test_fused_cgs2_pass_matches_two_kernel_pass(ctx, nvec, n):
    """CGS2 with the first update and the second projection fused into one pass over the basis
    (`fused_cgs`, off by default) against the two-kernel sequence (gmres.cpp:38-57): same Hessenberg
    column and the same normalised vector to rounding; more than 64 vectors falls back transparently."""
    rng = np.random.default_rng(nvec)
    V, _ = np.linalg.qr(rng.standard_normal((n, nvec)))
    w = rng.standard_normal(n)
    out = {}
    for flag in (0, 1):
        hdg.set_tuning("fused_cgs", flag)
        try:
            out[flag] = hdg.orthogonalize(ctx, V.T.copy(), w)
        finally:
            hdg.set_tuning("fused_cgs", 0)
    assert np.max(np.abs(out[1][0] - out[0][0])) <= 1e-12 * np.max(np.abs(out[0][0]))
    assert np.max(np.abs(out[1][1] - out[0][1])) <= 1e-12
    assert np.max(np.abs(V.T @ out[1][1])) <= 1e-12


def test_wide_system_records_in_l2_scratch(ctx):
    """Wide systems (M = 5): point records staged in a global scratch, one launch, E / D_d on DMMA (the default)
    against the scalar point-chunked sweep."""
    disc = hdg.Discretization.structured(ctx, "hex", n=2, degree=2, n_comp=5)
    model = hdg.make_case_model(disc, "navier_stokes", mu=0.02)
    state = hdg.make_initial_state(disc, model)
    out = {}
    for flag in (0, 1):
        hdg.set_tuning("local_global_records", flag)
        try:
            ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True, dt=0.05, u_prev=state.u)
            out[flag] = {nm: ops.get(nm) for nm in ["e_raw", "d_raw0", "d_raw1", "d_raw2", "f_raw", "h_raw", "j_raw", "kbar", "ru", "rbar"]}
        finally:
            hdg.set_tuning("local_global_records", 1)
    for nm in out[0]:
        assert rel(out[1][nm], out[0][nm]) <= (1e-9 if nm in ("kbar", "rbar") else 1e-12), nm


@pytest.mark.parametrize("shape,n,k,M,case", [("hex", 3, 3, 1, "poisson"), ("hex", 2, 2, 1, "burgers"), ("hex", 2, 3, 3, "elasticity"),
                                              ("hex", 2, 2, 5, "navier_stokes")])
def test_sixteen_warp_local_kernel_matches_eight_warp(ctx, shape, n, k, M, case):
    """`local_nt = 512`: one 16-warp CTA per SM, all 1 + D matrices of a scalar system (two component pairs of a wide
    one) per point sweep, two half-warps per quadrature point in the operand builder.  Same products in the same
    order as the default 8-warp kernel: identical raw blocks."""
    disc = hdg.Discretization.structured(ctx, shape, n=n, degree=k, n_comp=M)
    kw = {"mu": 0.02} if case == "navier_stokes" else {}
    model = hdg.make_case_model(disc, case, **kw)
    state = hdg.make_initial_state(disc, model)
    rng = np.random.default_rng(5)
    state.u = state.u + 0.05 * rng.standard_normal(state.u.shape)
    state.uhat = state.uhat + 0.05 * rng.standard_normal(state.uhat.shape)
    tkw = dict(dt=0.05, u_prev=state.u) if case == "navier_stokes" else {}
    out = {}
    try:
        hdg.set_tuning("local_ed_stream", 0)   # both sides on the chunked operand builder
        for nt in (256, 512):
            hdg.set_tuning("local_nt", nt)
            ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True, **tkw)
            names = ["e_raw", "f_raw", "h_raw", "j_raw"] + [f"d_raw{d}" for d in range(disc.dim)] + [f"g_raw{d}" for d in range(disc.dim)]
            out[nt] = {nm: ops.get(nm) for nm in names + ["kbar", "ru"]}
    finally:
        hdg.set_tuning("local_nt", 256)
        hdg.set_tuning("local_ed_stream", 3)
    for nm in out[256]:
        if nm == "ru":   # the residual sweep is split over nt / pe thread groups: another (fixed) summation partition
            assert rel(out[512][nm], out[256][nm]) <= 1e-13, nm
        else:
            assert np.array_equal(out[512][nm], out[256][nm]), nm


@pytest.mark.gpu
@pytest.mark.parametrize("shape,n,case,transient,qp", [("hex", 3, "poisson", False, 0), ("hex", 2, "burgers", True, 0),
                                                       ("hex", 2, "reaction", True, 0), ("hex", 2, "burgers", False, 4),
                                                       ("hex", 2, "burgers", True, 6)])
def test_streamed_ed_sweep_matches_chunked_builder(ctx, shape, n, case, transient, qp):
    """`local_ed_stream` (default on for scalar systems with 64 basis functions per element: hex p = 3): E and
    D_d from the bulk-TMA table ring with fragment-built left operands against the chunked shared-memory operand
    builder and against the scalar (no tensor core) sweep.  Same contraction, the quadrature weight on the other
    operand: equal to rounding.  Jittered meshes, perturbed states, with and without the backward-Euler mass term."""
    # qp: quadrature points per direction (0 = default k + 2 = 5).  4: partial ring stages everywhere (64 volume, 16 face points
    # per face); 6: 216 volume points and 36 > 32 face points per face -- H / G_d / F / J fall back to the staged face kernel
    disc = hdg.Discretization.structured(ctx, shape, n=n, degree=3, jitter=0.15, seed=3, quad_points=qp)
    assert disc.pe == 64
    model = hdg.make_case_model(disc, case)
    state = hdg.make_initial_state(disc, model)
    rng = np.random.default_rng(11)
    state.u = state.u + 0.1 * rng.standard_normal(state.u.shape)
    state.uhat = state.uhat + 0.1 * rng.standard_normal(state.uhat.shape)
    tkw = dict(dt=0.05, u_prev=state.u + 0.01) if transient else {}
    names = ["e_raw"] + [f"d_raw{d}" for d in range(disc.dim)] + ["f_raw", "h_raw", "j_raw", "kbar", "ru"]
    out = {}
    for tag, stream, dmma in (("stream", 3, 1), ("chunked", 0, 1), ("scalar", 0, 0)):
        hdg.set_tuning("local_ed_stream", stream)
        hdg.set_tuning("use_dmma", dmma)
        try:
            ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True, **tkw)
            out[tag] = {nm: ops.get(nm) for nm in names}
        finally:
            hdg.set_tuning("local_ed_stream", 3)
            hdg.set_tuning("use_dmma", 1)
    for nm in names:
        assert np.all(np.isfinite(out["stream"][nm])), nm
        assert rel(out["stream"][nm], out["chunked"][nm]) <= 1e-13, nm
        assert rel(out["stream"][nm], out["scalar"][nm]) <= 1e-12, nm


@pytest.mark.gpu
@pytest.mark.parametrize("case,M,nt", [("navier_stokes", 5, 512), ("navier_stokes", 5, 256), ("elasticity", 3, 512)])
def test_streamed_wide_sweep_matches_chunked_builder(ctx, case, M, nt):
    """Wide systems on hexahedra of degree 3 (config 5's shape): E / D_d one streamed sweep per component pair (table
    ring, coefficient rows gathered into shared memory, 16 or 8 warps) against the chunked operand builder and the
    scalar sweep; backward-Euler mass term on the diagonal pairs."""
    disc = hdg.Discretization.structured(ctx, "hex", n=2, degree=3, n_comp=M, jitter=0.1, seed=4)
    kw = {"mu": 0.02} if case == "navier_stokes" else {}
    model = hdg.make_case_model(disc, case, **kw)
    state = hdg.make_initial_state(disc, model)
    rng = np.random.default_rng(12)
    state.u = state.u + 0.02 * rng.standard_normal(state.u.shape)
    state.uhat = state.uhat + 0.02 * rng.standard_normal(state.uhat.shape)
    tkw = dict(dt=0.05, u_prev=state.u + 0.01)
    names = ["e_raw"] + [f"d_raw{d}" for d in range(3)] + ["f_raw", "h_raw", "j_raw", "kbar", "ru"]
    out = {}
    for tag, stream, dmma in (("stream", 3, 1), ("chunked", 0, 1), ("scalar", 0, 0)):
        hdg.set_tuning("local_ed_stream", stream)
        hdg.set_tuning("local_nt_wide", nt)
        hdg.set_tuning("use_dmma", dmma)
        try:
            ops = hdg.assemble_element_operators(disc, model, state, keep_raw=True, **tkw)
            out[tag] = {nm: ops.get(nm) for nm in names}
        finally:
            hdg.set_tuning("local_ed_stream", 3)
            hdg.set_tuning("local_nt_wide", 256)
            hdg.set_tuning("use_dmma", 1)
    for nm in names:
        assert np.all(np.isfinite(out["stream"][nm])), nm
        assert rel(out["stream"][nm], out["chunked"][nm]) <= 1e-13, nm
        assert rel(out["stream"][nm], out["scalar"][nm]) <= 1e-12, nm
