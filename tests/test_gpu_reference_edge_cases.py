"""The edge cases the reference's own unit tests pin (proj/tests/test_gmres.cpp, test_newton.cpp, test_precond.cpp,
test_face_matrix.cpp), restated one by one against the GPU library through the C ABI: zero right-hand side,
iteration caps, non-finite and singular operators, exact-inverse preconditioning, degenerate Gram-Schmidt input,
line-search damping / failure, Newton caps, per-restart Ritz recomputation, time-marching contracts, harmonic-Ritz
breakdown and argument checks, polynomial telescoping, dense-expansion guard, non-finite state.  Each test names the
reference test it mirrors; tolerances are the reference's."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg

pytestmark = pytest.mark.gpu


def dense_op(ctx, a):
    """y = A x on device vectors through the ABI's strided-batch GEMV (A row-major numpy)."""
    n = a.shape[0]
    dA = ctx.alloc(n * n)
    ctx.copy(dA, np.ascontiguousarray(a.T).ravel(), n * n)

    def op(din, dout, nn):
        ctx.check(ctx._L.hdgb_gemv_strided_batch(ctx._h, n, n, 1, dA, din, dout, 0))
    op.free = lambda: ctx.free(dA)
    return op


def identity_op(ctx):
    def op(din, dout, n):
        ctx.copy(dout, din, n)
    return op


# ---- test_gmres.cpp ------------------------------------------------------------------------------------------------
def test_gmres_zero_rhs_returns_zero(ctx):                      # GmresSolve.ZeroRhsReturnsZero
    rhs = np.zeros(10)
    x, st = hdg.gmres_solve_fn(ctx, 10, identity_op(ctx), identity_op(ctx), rhs, x0=rhs)
    assert st.converged and st.iters == 0 and np.all(x == 0.0)


def test_gmres_identity_converges_in_one_iteration(ctx):        # GmresSolve.IdentityConvergesInOneIteration
    rhs = hdg.random_vector(20, 5)
    x, st = hdg.gmres_solve_fn(ctx, 20, identity_op(ctx), identity_op(ctx), rhs, x0=np.zeros(20))
    assert st.converged and st.iters == 1
    assert np.max(np.abs(x - rhs)) <= 1e-14


def test_gmres_exact_inverse_preconditioner_one_iteration(ctx):  # GmresSolve.ExactInversePreconditionerOneIteration
    n = 12
    a = hdg.random_vector(n * n, 21).reshape(n, n) + 4.0 * np.eye(n)
    mv, pc = dense_op(ctx, a), dense_op(ctx, np.linalg.inv(a))
    rhs = hdg.random_vector(n, 22)
    x, st = hdg.gmres_solve_fn(ctx, n, mv, pc, rhs, x0=np.zeros(n), cfg=hdg.GmresConfig(tol=1e-10))
    mv.free(), pc.free()
    assert st.converged and st.iters == 1
    assert np.max(np.abs(a @ x - rhs)) <= 1e-9


def test_gmres_max_iters_reports_not_converged(ctx):            # GmresSolve.MaxItersReportsNotConverged
    n = 30
    a = np.zeros((n, n))
    for i in range(n):
        a[i, i] = 1.0 + 1e4 * i
        if i + 1 < n:
            a[i, i + 1] = 1e3
    mv = dense_op(ctx, a)
    x, st = hdg.gmres_solve_fn(ctx, n, mv, None, hdg.random_vector(n, 77), x0=np.zeros(n),
                               cfg=hdg.GmresConfig(restart=5, max_iters=8, tol=1e-14))
    mv.free()
    assert not st.converged and st.iters <= 8 and st.final_rel_residual > 1e-14


def test_gmres_nan_operator_throws(ctx):                        # GmresSolve.NaNOperatorThrows
    nan = np.array([np.nan])

    def bad(din, dout, n):
        ctx.copy(dout, din, n)
        ctx.copy(dout, nan, 1)
    with pytest.raises(hdg.NaNDetected):
        hdg.gmres_solve_fn(ctx, 5, bad, identity_op(ctx), hdg.random_vector(5, 1), x0=np.zeros(5))


def test_gmres_singular_operator_throws(ctx):                   # GmresSolve.SingularOperatorThrows
    zeros = np.zeros(8)

    def zero(din, dout, n):
        ctx.copy(dout, zeros, n)
    with pytest.raises(hdg.NaNDetected):
        hdg.gmres_solve_fn(ctx, 8, zero, identity_op(ctx), hdg.random_vector(8, 3), x0=np.zeros(8))


def test_orthogonalize_vector_in_span_reduces_to_noise(ctx):    # Orthogonalize.VectorInSpanReducesToNoise
    v1 = hdg.random_vector(40, 1)
    v1 /= np.linalg.norm(v1)
    h, w = hdg.orthogonalize(ctx, v1[None, :], 3.5 * v1, "cgs")
    assert len(h) == 2 and abs(h[0] - 3.5) <= 1e-12 and h[1] <= 1e-12 * 3.5


def test_orthogonalize_simple_two_vector_case_and_modes_agree(ctx):  # Orthogonalize.SimpleTwoVectorCase / CgsAndMgsAgree
    h, w = hdg.orthogonalize(ctx, np.array([[1.0, 0.0, 0.0]]), np.array([1.0, 1.0, 0.0]), "mgs")
    assert h[0] == 1.0 and h[1] == 1.0 and abs(w[0]) <= 1e-15 and abs(w[1] - 1.0) <= 1e-15
    V, _ = np.linalg.qr(hdg.random_vector(60 * 6, 9).reshape(60, 6))
    y = hdg.random_vector(60, 10)
    hc, wc = hdg.orthogonalize(ctx, np.ascontiguousarray(V.T), y, "cgs")
    hm, wm = hdg.orthogonalize(ctx, np.ascontiguousarray(V.T), y, "mgs")
    assert np.max(np.abs(hc - hm)) <= 1e-12 and np.max(np.abs(wc - wm)) <= 1e-12


# ---- test_newton.cpp -----------------------------------------------------------------------------------------------
def cubic_reaction(ctx, lam):
    """cubic_reaction_model of the reference's tests: -lap u = lambda (8 - u^3), u = 2 on the boundary, on the 2 x 2 mesh
    of poisson_spec(1, 2)."""
    disc = hdg.Discretization.structured(ctx, "quad", n=2, degree=1)
    model = hdg.Model(disc, "reaction", [1.0, lam], forcing=lambda x: np.full(x.shape[:-1], 8.0 * lam),
                      dirichlet=lambda x: np.full(x.shape[:-1], 2.0))
    return disc, model


def test_newton_linear_problem_converges_in_one_iteration(ctx):  # NewtonSolve.LinearProblemConvergesInOneIteration
    disc = hdg.Discretization.structured(ctx, "quad", n=4, degree=2)
    model = hdg.make_case_model(disc, "poisson2d")
    state = hdg.make_initial_state(disc, model)
    rep = hdg.newton_solve(disc, model, state, gcfg=hdg.GmresConfig(tol=1e-10), pspec=hdg.PrecondSpec("asm"))
    assert rep.converged and rep.n_newton == 1 and rep.alpha_history[0] == 1.0 and rep.final_residual <= 1e-8


def test_newton_residual_history_strictly_decreasing(ctx):       # NewtonSolve.ResidualHistoryStrictlyDecreasing
    disc = hdg.Discretization.structured(ctx, "quad", n=8, degree=1)
    model = hdg.make_case_model(disc, "burgers2d")
    state = hdg.make_initial_state(disc, model)
    rep = hdg.newton_solve(disc, model, state, pspec=hdg.PrecondSpec("asm"))
    assert rep.converged and len(rep.residual_history) >= 2
    assert all(b < a for a, b in zip(rep.residual_history, rep.residual_history[1:]))
    assert len(rep.gmres_per_newton) == rep.n_newton


def test_newton_damping_engages_on_overshoot(ctx):               # NewtonSolve.DampingEngagesOnOvershoot
    disc, model = cubic_reaction(ctx, 1.0)
    state = hdg.State(disc)
    state.u = np.full(disc.npe * disc.ne, 0.1)
    state.uhat = np.full(disc.n_dof, 0.1)
    rep = hdg.newton_solve(disc, model, state, gcfg=hdg.GmresConfig(tol=1e-10), pspec=hdg.PrecondSpec("asm"))
    assert rep.converged
    assert min(rep.alpha_history) < 1.0
    assert np.max(np.abs(state.u - 2.0)) <= 1e-6


def test_newton_line_search_failure_throws(ctx):                 # NewtonSolve.LineSearchFailureThrows
    disc, model = cubic_reaction(ctx, 1e6)
    state = hdg.State(disc)
    state.u = np.full(disc.npe * disc.ne, 0.01)
    state.uhat = np.full(disc.n_dof, 0.01)
    u_before = state.u.copy()
    with pytest.raises(hdg.LineSearchFailed) as ei:
        hdg.newton_solve(disc, model, state, ncfg=hdg.NewtonConfig(min_alpha=0.5), pspec=hdg.PrecondSpec("asm"))
    assert ei.value.index == 0                                    # the failing Newton iteration (errors.hpp:92-98)
    assert np.array_equal(state.u, u_before)                      # the last accepted iterate is restored


def test_newton_max_newton_reports_not_converged(ctx):           # NewtonSolve.MaxNewtonReportsNotConverged
    disc = hdg.Discretization.structured(ctx, "quad", n=8, degree=1)
    model = hdg.make_case_model(disc, "burgers2d")
    state = hdg.make_initial_state(disc, model)
    rep = hdg.newton_solve(disc, model, state, ncfg=hdg.NewtonConfig(max_newton=2), pspec=hdg.PrecondSpec("asm"))
    assert not rep.converged and rep.n_newton == 2


def test_newton_per_restart_ritz_recomputation(ctx, ref):        # NewtonSolve.PerRestartRitzRecomputationWorks
    disc = hdg.Discretization.structured(ctx, "quad", n=8, degree=1)
    model = hdg.make_case_model(disc, "burgers2d")
    state = hdg.make_initial_state(disc, model)
    rep = hdg.newton_solve(disc, model, state, gcfg=hdg.GmresConfig(restart=10),
                           pspec=hdg.PrecondSpec("bj", poly_degree=5, ritz_per_restart=True))
    assert rep.converged
    # the same solve without per-restart recomputation reaches the same trace solution (test_newton.cpp:120-141: 1e-6)
    s2 = hdg.make_initial_state(disc, model)
    rep2 = hdg.newton_solve(disc, model, s2, gcfg=hdg.GmresConfig(restart=10), pspec=hdg.PrecondSpec("bj", poly_degree=5))
    assert rep2.converged and np.max(np.abs(state.uhat - s2.uhat)) <= 1e-6
    # per-restart mode rebuilds the polynomial between cycles: more inner operator applications are not required,
    # but the outer iteration counts must stay in the reference's band for this case (acceptance_main.cpp:425-429)
    assert 10 <= rep.n_gmres_total <= 800


def test_time_march_requires_positive_dt(ctx):                   # TimeMarch.RequiresPositiveDt
    disc = hdg.Discretization.structured(ctx, "quad", n=4, degree=1)
    model = hdg.make_case_model(disc, "poisson2d")
    state = hdg.make_initial_state(disc, model)
    for dt in (0.0, -1.0):
        with pytest.raises(hdg.HdgError, match="positive dt"):
            hdg.time_march(disc, model, state, dt, 1)


def test_time_march_huge_step_reproduces_steady_solve(ctx):      # TimeMarch.HugeStepReproducesSteadySolve
    disc = hdg.Discretization.structured(ctx, "quad", n=4, degree=1)
    model = hdg.make_case_model(disc, "poisson2d")
    g, n = hdg.GmresConfig(tol=1e-12), hdg.NewtonConfig(tol=1e-10)
    steady = hdg.make_initial_state(disc, model)
    assert hdg.newton_solve(disc, model, steady, ncfg=n, gcfg=g, pspec=hdg.PrecondSpec("asm")).converged
    marched = hdg.make_initial_state(disc, model)
    reps = hdg.time_march(disc, model, marched, 1e12, 1, ncfg=n, gcfg=g, pspec=hdg.PrecondSpec("asm"))
    assert reps[0].converged
    assert np.max(np.abs(marched.u - steady.u)) <= 1e-6


# ---- test_precond.cpp ----------------------------------------------------------------------------------------------
def test_harmonic_ritz_identity_breaks_down_to_single_value(ctx):  # HarmonicRitz.IdentityBreaksDownToSingleValue
    th = hdg.compute_harmonic_ritz(ctx, identity_op(ctx), 50, 10, seed=42)
    assert len(th) == 1 and abs(th[0].real - 1.0) <= 1e-12 and th[0].imag == 0.0


def test_harmonic_ritz_rejects_degree_above_dimension(ctx):      # HarmonicRitz.RejectsDegreeAboveDimension
    with pytest.raises(hdg.DimensionMismatch):
        hdg.compute_harmonic_ritz(ctx, identity_op(ctx), 3, 4, seed=1)


def test_harmonic_ritz_deterministic_for_fixed_seed(ctx):        # HarmonicRitz.DeterministicForFixedSeed
    a = hdg.random_vector(15 * 15, 3).reshape(15, 15) + 6.0 * np.eye(15)
    op = dense_op(ctx, a)
    t1 = hdg.compute_harmonic_ritz(ctx, op, 15, 6, seed=11)
    t2 = hdg.compute_harmonic_ritz(ctx, op, 15, 6, seed=11)
    t3 = hdg.compute_harmonic_ritz(ctx, op, 15, 6, seed=12)
    op.free()
    assert np.array_equal(t1, t2) and not np.array_equal(t1, t3)


def one_element_system(ctx, identity=False):
    disc = hdg.Discretization.structured(ctx, "quad", n=1 if identity else 2, degree=1)
    model = hdg.make_case_model(disc, "poisson2d")
    state = hdg.make_initial_state(disc, model)
    K, _ = hdg.assemble_global(disc, hdg.assemble_element_operators(disc, model, state))
    if identity:   # K := I, as the reference test overwrites the blocks
        bd, nb = K.block_dim, K.nb
        blocks = np.zeros((K.nf, nb * bd, bd))
        blocks[:, :bd, :] = np.eye(bd)
        K = hdg.FaceBlockMatrix.from_host(ctx, 1, disc.pf, disc.n_lfe, K.nf, K.neighbor, blocks.ravel())
    return disc, K


def test_apply_poly_degree_one_is_scaled_base(ctx):              # ApplyPoly.DegreeOneIsScaledBase
    disc, K = one_element_system(ctx)
    p = hdg.precond_from_host(ctx, "identity", disc.mpf, K.nf, ritz=[4.0], k=K)
    y = hdg.random_vector(K.n_dof, 71)
    z, ops = hdg.apply_poly(p, K, y)
    assert np.array_equal(z, y / 4.0)


def test_apply_poly_telescopes_for_unit_ritz_values_on_identity(ctx):  # ApplyPoly.TelescopesForUnitRitzValuesOnIdentity
    disc, K = one_element_system(ctx, identity=True)
    p = hdg.precond_from_host(ctx, "identity", disc.mpf, K.nf, ritz=[1.0] * 5, k=K)
    y = hdg.random_vector(K.n_dof, 81)
    z, ops = hdg.apply_poly(p, K, y)
    assert ops == 5 and np.max(np.abs(z - y)) <= 1e-12


# ---- test_face_matrix.cpp / test_local_ops.cpp --------------------------------------------------------------------------
def test_to_dense_guards_against_huge_systems(ctx):              # ToDense.GuardsAgainstHugeSystems
    disc, K = one_element_system(ctx)
    with pytest.raises(hdg.TooLargeForDense):
        K.to_dense(limit=K.n_dof - 1)


def test_non_finite_state_is_reported(ctx):                      # local_ops.cpp:33-37 (check_finite: u first, then uhat)
    disc = hdg.Discretization.structured(ctx, "quad", n=3, degree=2)
    model = hdg.make_case_model(disc, "poisson2d")
    state = hdg.make_initial_state(disc, model)
    u = state.u
    u[7] = np.nan
    state.u = u
    with pytest.raises(hdg.NonFiniteState, match="interior"):
        hdg.assemble_element_operators(disc, model, state)
    u[7] = 0.0
    state.u = u
    uh = state.uhat
    uh[3] = np.inf
    state.uhat = uh
    with pytest.raises(hdg.NonFiniteState, match="trace"):
        hdg.assemble_residual(disc, model, state)


# ---- test_dense_batch.cpp -------------------------------------------------------------------------------------------
def test_lu_invert_pivoting_handles_zero_diagonal(ctx):          # LuInvertBatch.PivotingHandlesZeroDiagonal
    a = np.zeros((1, 2, 2))
    a[0, 1, 0] = 1.0   # [b][c][r]: entry (r = 0, c = 1)
    a[0, 0, 1] = 1.0
    inv = hdg.lu_invert_batch(ctx, a.ravel(), 2, 1).reshape(1, 2, 2)
    assert inv[0, 1, 0] == 1.0 and inv[0, 0, 1] == 1.0 and inv[0, 0, 0] == 0.0 and inv[0, 1, 1] == 0.0


def test_lu_invert_identity_diagonal_and_singular_index(ctx):    # LuInvertBatch.IdentityBlocks / DiagonalBlock / SingularBlockNamesIndex
    n, batch = 3, 4
    eye = np.tile(np.eye(n).ravel(), batch)
    assert np.array_equal(hdg.lu_invert_batch(ctx, eye, n, batch), eye)
    d = np.diag([2.0, 4.0, 8.0]).ravel()
    assert np.array_equal(hdg.lu_invert_batch(ctx, d, n, 1), np.diag([0.5, 0.25, 0.125]).ravel())
    a = np.zeros((3, 2, 2))
    a[0] = a[2] = np.eye(2)          # block 1 stays all-zero
    with pytest.raises(hdg.SingularBlock) as ei:
        hdg.lu_invert_batch(ctx, a.ravel(), 2, 3)
    assert ei.value.index == 1


def test_gemv_accumulate_twice_doubles_and_matches_gemm_column(ctx):  # GemvStridedBatch.AccumulateTwiceDoubles / BitIdenticalToGemmSingleColumn
    rows, cols, batch = 6, 4, 7
    a = hdg.random_vector(rows * cols * batch, 51)
    x = hdg.random_vector(cols * batch, 52)
    y = hdg.gemv_strided_batch(ctx, a, rows, cols, batch, x)
    y2 = hdg.gemv_strided_batch(ctx, a, rows, cols, batch, x, y=y.copy(), accumulate=True)
    assert np.array_equal(y2, 2.0 * y)
    c = hdg.gemm_batch(ctx, a, rows, cols, batch, x, cols, 1, batch)
    assert np.max(np.abs(c - y)) <= 1e-15 * max(1.0, np.max(np.abs(y)))


def test_gemm_identity_transpose_broadcast_and_mismatch(ctx):    # GemmBatch.IdentityTimesB / TransposeA / BroadcastMatchesLoopOracle / DimensionMismatch
    n, k, batch = 5, 3, 4
    b = hdg.random_vector(n * k * batch, 7)
    eye = np.eye(n).ravel()
    assert np.array_equal(hdg.gemm_batch(ctx, eye, n, n, 1, b, n, k, batch), b)   # broadcast A = I
    a = hdg.random_vector(n * k * batch, 8)                                         # A_b: n x k, used transposed
    c = hdg.gemm_batch(ctx, a, n, k, batch, b, n, k, batch, transpose_a=True).reshape(batch, k, k)
    A = a.reshape(batch, k, n)   # column-major n x k -> [b][col][row]
    B = b.reshape(batch, k, n)
    want = np.einsum("bir,bjr->bji", A, B)   # (A^T B)[i, j] stored [b][j][i]
    assert np.max(np.abs(c - want)) <= 1e-14
    with pytest.raises(hdg.DimensionMismatch):
        hdg.gemm_batch(ctx, a, n, k, batch, b, n, k, batch)       # inner dimensions k vs n


# ---- test_face_matrix.cpp ------------------------------------------------------------------------------------------
def quad_case(ctx, k, n, case="poisson2d"):
    disc = hdg.Discretization.structured(ctx, "quad", n=n, degree=k)
    model = hdg.make_case_model(disc, case)
    state = hdg.make_initial_state(disc, model)
    ops = hdg.assemble_element_operators(disc, model, state)
    K, rhs = hdg.assemble_global(disc, ops)
    return disc, model, state, ops, K, rhs


def test_gather_extended_scatter_transpose_counts_multiplicity(ctx):  # GatherExtended.ScatterTransposeCountsMultiplicity
    disc, model, state, ops, K, rhs = quad_case(ctx, 1, 3)
    mpf, nb = K.block_dim, K.nb
    gathered = hdg.gather_extended(K, np.ones(K.n_dof)).reshape(K.nf, nb, mpf)
    nbr = K.neighbor.reshape(K.nf, nb)
    counts = np.zeros((K.nf, mpf))
    for f in range(K.nf):
        for s in range(nb):
            if nbr[f, s] >= 0:
                counts[nbr[f, s]] += gathered[f, s]
    boundary = disc.table("face_to_elements").reshape(K.nf, 2)[:, 1] < 0
    assert np.all(counts[boundary] == 4.0) and np.all(counts[~boundary] == 7.0)


def test_assemble_global_structure_properties(ctx):              # AssembleGlobal.NeighborStructureSymmetric / PoissonTraceOperatorSymmetricDefinite / SelfBlocksInvertible
    disc, model, state, ops, K, rhs = quad_case(ctx, 2, 3)
    nbr = K.neighbor.reshape(K.nf, K.nb)
    for f in range(K.nf):
        assert nbr[f, 0] == f
        for g in nbr[f, 1:]:
            if g >= 0:
                assert f in nbr[g]                                  # g lists f back
    # symmetric and (after a sign flip) definite on the flux-continuity rows = interior faces; Dirichlet faces carry
    # the one-sided constraint row uhat = u_D (test_face_matrix.cpp:87-121)
    A = K.to_dense()
    bd = K.block_dim
    interior = np.flatnonzero(disc.table("face_to_elements").reshape(K.nf, 2)[:, 1] >= 0)
    keep = (interior[:, None] * bd + np.arange(bd)[None, :]).ravel()
    sub = -A[np.ix_(keep, keep)]
    assert np.max(np.abs(sub - sub.T)) <= 1e-12 * max(1.0, np.max(np.abs(sub)))
    np.linalg.cholesky(0.5 * (sub + sub.T))                         # raises if not positive definite
    blocks = K.blocks.reshape(K.nf, K.nb, bd, bd)
    assert all(abs(np.linalg.det(blocks[f, 0])) > 1e-12 for f in range(K.nf))


def test_block_matvec_identity_self_blocks_and_linearity(ctx):   # BlockMatvec.IdentitySelfBlocks / Linear
    disc, model, state, ops, K, rhs = quad_case(ctx, 1, 3)
    bd, nb = K.block_dim, K.nb
    blocks = np.zeros((K.nf, nb * bd, bd))
    blocks[:, :bd, :] = np.eye(bd)
    I = hdg.FaceBlockMatrix.from_host(ctx, 1, disc.pf, disc.n_lfe, K.nf, K.neighbor, blocks.ravel())
    x = hdg.random_vector(K.n_dof, 4)
    assert np.array_equal(hdg.block_matvec(I, x), x)
    y = hdg.random_vector(K.n_dof, 5)
    lhs = hdg.block_matvec(K, 2.0 * x - 3.0 * y)
    rhs2 = 2.0 * hdg.block_matvec(K, x) - 3.0 * hdg.block_matvec(K, y)
    assert np.max(np.abs(lhs - rhs2)) <= 1e-12 * max(1.0, np.max(np.abs(rhs2)))


def test_reversed_face_gives_mirrored_coefficients(ctx):         # Orientation.ReversedFaceGivesMirroredCoefficients
    from paper_2512_13619_b200 import partition as P
    k, n = 2, 2
    coords, ev = P.box_quad_mesh(n, n)
    gm = P.global_mesh("quad", coords, ev, lo=(0, 0), hi=(1, 1))

    def solve(flip):
        lm = P.build_local_meshes(gm, np.zeros(gm.ne, dtype=np.int32))[0]
        target = int(np.flatnonzero(lm.f2e[:, 1] >= 0)[0])
        if flip:   # reverse the canonical direction of the first interior face: end vertices swapped, both sides' flags toggled
            lm.fverts[target] = lm.fverts[target][::-1]
            lm.forient[target] = 1 - lm.forient[target]
        disc = P.make_discretization(ctx, lm, "quad", k)
        model = hdg.make_case_model(disc, "poisson2d")
        state = hdg.State(disc)
        K, rhs = hdg.assemble_global(disc, hdg.assemble_element_operators(disc, model, state))
        return np.linalg.solve(K.to_dense(), rhs).reshape(K.nf, -1), target
    ub, target = solve(False)
    uf, _ = solve(True)
    for f in range(ub.shape[0]):
        want = uf[f, ::-1] if f == target else uf[f]
        assert np.max(np.abs(ub[f] - want)) <= 1e-11


# ---- test_precond.cpp (structure / property tests) --------------------------------------------------------------------
def test_build_asm_shared_face_diagonal_sums_and_one_element_exact_solve(ctx):  # BuildAsm.SharedFaceDiagonalSums / ApplyAsm.OneElementIsExactSolve
    disc, model, state, ops, K, rhs = quad_case(ctx, 1, 1)           # one element: ASM block = K-bar, apply = exact solve
    P1 = hdg.build_asm(ops, disc, K)
    y = hdg.random_vector(K.n_dof, 9)
    z = hdg.apply_asm(P1, y)
    assert np.max(np.abs(K.to_dense() @ z - y)) <= 1e-10 * max(1.0, np.max(np.abs(y)))
    # 2 x 2 mesh: the enriched diagonal sub-block of an interior face is the sum of both elements' sub-blocks = K_ff
    disc, model, state, ops, K, rhs = quad_case(ctx, 1, 2)
    P2 = hdg.build_asm(ops, disc, K)
    nfl, pf = disc.nfl, disc.pf
    pbar = np.linalg.inv(P2.get("asm_inv").reshape(disc.ne, nfl, nfl))   # [e][c][r] of the inverse's inverse
    kbar = ops.get("kbar").reshape(disc.ne, nfl, nfl)
    e2f = disc.table("element_to_face").reshape(disc.ne, -1)
    f2e = disc.table("face_to_elements").reshape(disc.nf, 2)
    fli = disc.table("face_local_index").reshape(disc.nf, 2)
    for f in np.flatnonzero(f2e[:, 1] >= 0):
        (e0, e1), (l0, l1) = f2e[f], fli[f]
        s = kbar[e0, l0 * pf:(l0 + 1) * pf, l0 * pf:(l0 + 1) * pf] + kbar[e1, l1 * pf:(l1 + 1) * pf, l1 * pf:(l1 + 1) * pf]
        for e, l in ((e0, l0), (e1, l1)):
            assert np.max(np.abs(pbar[e, l * pf:(l + 1) * pf, l * pf:(l + 1) * pf] - s)) <= 1e-9 * max(1.0, np.max(np.abs(s)))
    assert e2f.shape[1] == 4


def test_preconditioner_applications_are_linear(ctx):            # ApplyPreconditioners.Linearity
    disc, model, state, ops, K, rhs = quad_case(ctx, 2, 3, "burgers2d")
    x, y = hdg.random_vector(K.n_dof, 31), hdg.random_vector(K.n_dof, 32)
    for spec in (hdg.PrecondSpec("bj"), hdg.PrecondSpec("asm"), hdg.PrecondSpec("asm", poly_degree=4)):
        Pc = hdg.build_preconditioner(spec, K, ops, disc)
        lhs = Pc.apply(2.0 * x - 3.0 * y)
        rhs2 = 2.0 * Pc.apply(x) - 3.0 * Pc.apply(y)
        assert np.max(np.abs(lhs - rhs2)) <= 1e-10 * max(1.0, np.max(np.abs(rhs2)))


def test_asm_needs_fewer_iterations_than_bj(ctx):                # PrecondEffectiveness.AsmNeedsFewerIterationsThanBj
    disc, model, state, ops, K, rhs = quad_case(ctx, 2, 8, "burgers2d")
    its = {}
    for kind in ("bj", "asm"):
        Pc = hdg.build_preconditioner(kind, K, ops, disc)
        x, st = hdg.gmres_solve(K, Pc, rhs, cfg=hdg.GmresConfig(tol=1e-8))
        assert st.converged
        its[kind] = st.iters
    assert its["asm"] < its["bj"]
