"""orthogonalize (gmres.cpp:28-59) on the GPU: the three-pass streamed CGS2 (k_orth.cu), the four-pass kernels it
replaces, the domain-decomposed variant (two all-reduces, Pythagorean norm) and long restart lengths -- all against
a numpy restatement of the reference sequence."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg

pytestmark = pytest.mark.gpu


def cgs2_numpy(V, w):
    """The reference sequence: c = V w; w -= c V; then per vector d_i = v_i.w, w -= d_i v_i (interleaved)."""
    w = w.copy()
    c = V @ w
    for i in range(len(V)):
        w -= c[i] * V[i]
    for i in range(len(V)):
        d = V[i] @ w
        c[i] += d
        w -= d * V[i]
    hn = np.sqrt(w @ w)
    return np.concatenate([c, [hn]]), (w / hn if hn > 0 else w)


def basis(nvec, n, seed):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, nvec)))
    return np.ascontiguousarray(q.T), rng.standard_normal(n)


@pytest.mark.parametrize("nvec,n", [(1, 4096), (5, 100000), (33, 50002), (50, 131072), (64, 20000), (7, 128), (3, 1000),
                                    (9, 40001), (70, 30000)])
def test_cgs2_passes_vs_numpy(ctx, nvec, n):
    V, w = basis(nvec, n, nvec + n)
    w = w + 10.0 * V[0] - 3.0 * V[-1]
    want_h, want_w = cgs2_numpy(V, w)
    out = {}
    for flag in (1, 0):
        hdg.set_tuning("cgs_stream", flag)
        try:
            out[flag] = hdg.orthogonalize(ctx, V, w)
            again = hdg.orthogonalize(ctx, V, w)
        finally:
            hdg.set_tuning("cgs_stream", 1)
        h, wn = out[flag]
        scale = np.max(np.abs(want_h))
        assert np.max(np.abs(h - want_h)) <= 1e-13 * scale, flag
        assert np.max(np.abs(wn - want_w)) <= 1e-13, flag
        assert np.max(np.abs(V @ wn)) <= 1e-14 * np.sqrt(n)               # orthogonal to the basis
        assert np.array_equal(again[0], h) and np.array_equal(again[1], wn)   # fixed reduction order: bit-reproducible
    assert np.max(np.abs(out[0][0] - out[1][0])) <= 1e-13 * np.max(np.abs(want_h))


def test_cgs2_nearly_dependent_vector(ctx):
    """w almost in span(V): the second projection matters, and the sub-diagonal entry is tiny."""
    V, w = basis(12, 65536, 3)
    rng = np.random.default_rng(1)
    w = V.T @ rng.standard_normal(12) + 1e-9 * w
    want_h, want_w = cgs2_numpy(V, w)
    h, wn = hdg.orthogonalize(ctx, V, w)
    assert np.max(np.abs(h[:-1] - want_h[:-1])) <= 1e-13 * np.max(np.abs(want_h))
    assert abs(h[-1] - want_h[-1]) <= 1e-6 * want_h[-1]
    assert np.max(np.abs(V @ wn)) <= 1e-9


def test_long_restart_lengths(ctx):
    """GMRES(m) with m far above the default (the reference accepts any restart length, gmres.hpp:15): the projection
    kernels group the basis vectors so that no launch outgrows its shared memory."""
    disc = hdg.Discretization.structured(ctx, "quad", n=12, degree=2)
    model = hdg.make_case_model(disc, "poisson2d")
    state = hdg.make_initial_state(disc, model)
    ops = hdg.assemble_element_operators(disc, model, state)
    K, rhs = hdg.assemble_global(disc, ops)
    rhs = hdg.random_vector(K.n_dof, 11)   # (the manufactured right-hand side converges in three iterations)
    x50, s50 = hdg.gmres_solve(K, None, rhs, cfg=hdg.GmresConfig(restart=50, tol=1e-10, max_iters=4000))
    x900, s900 = hdg.gmres_solve(K, None, rhs, cfg=hdg.GmresConfig(restart=900, tol=1e-10, max_iters=4000))
    assert s900.converged and s900.restarts == 0 and s900.iters > 64
    assert np.max(np.abs(K.to_dense() @ x900 - rhs)) <= 1e-8 * np.max(np.abs(rhs))
    assert s50.converged and np.max(np.abs(x50 - x900)) <= 1e-7 * np.max(np.abs(x900))
    V, w = basis(800, 4000, 5)
    want_h, want_w = cgs2_numpy(V, w)
    h, wn = hdg.orthogonalize(ctx, V, w)
    assert np.max(np.abs(h - want_h)) <= 1e-12 * np.max(np.abs(want_h)) and np.max(np.abs(wn - want_w)) <= 1e-12
