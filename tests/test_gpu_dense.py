"""Batched dense kernels against numpy and the reference's own dense_batch tests
(test_dense_batch.cpp): inverse accuracy, pivoting, lowest singular batch index, broadcast GEMM."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["gj", "gj-copy", "gj-cta", "gj-smem", "tile", "smem"])
def lu_kernel(request):
    """gj: blocked Gauss-Jordan with DMMA rank-16 updates (the default for n > 24; gj-cta: its panel of large
    blocks factored by a 4-warp CTA instead of one warp); tile: register-tiled Gauss-Jordan (n <= 128); smem: one
    block per CTA in shared memory / the global-memory fallback."""
    hdg.set_tuning("use_blocked_gj", 1 if request.param.startswith("gj") else 0)
    hdg.set_tuning("gj_panel_cta", 1 if request.param == "gj-cta" else 0)
    hdg.set_tuning("gj_direct", 0 if request.param == "gj-copy" else 1)   # gj-copy: copy prepass + separate column-permutation pass
    hdg.set_tuning("gj_smem", 1 if request.param == "gj-smem" else 0)   # single kernel, block in shared memory (n <= 128)
    hdg.set_tuning("use_tile_lu", 1 if request.param == "tile" else 0)
    yield request.param
    hdg.set_tuning("use_blocked_gj", 1)
    hdg.set_tuning("gj_panel_cta", 0)
    hdg.set_tuning("gj_direct", 1)
    hdg.set_tuning("gj_smem", 0)
    hdg.set_tuning("use_tile_lu", 1)


@pytest.mark.parametrize("n,batch", [(1, 5), (2, 9), (5, 33), (9, 100), (12, 64), (16, 40), (24, 17), (25, 21), (32, 20),
                                     (40, 11), (64, 9), (70, 5), (96, 7), (100, 3), (128, 2), (150, 2), (33, 300), (200, 3),
                                     (320, 2)])
def test_lu_invert_batch(ctx, lu_kernel, n, batch):
    if not lu_kernel.startswith("gj") and n > 150:
        pytest.skip("the fallback kernels are slow at this size")
    if lu_kernel == "gj-cta" and n <= 128:
        pytest.skip("the CTA panel kernel is for n > 128")
    if lu_kernel == "gj-smem" and (n > 128 or n <= 24):
        pytest.skip("the shared-memory resident variant covers 24 < n <= 128")
    rng = np.random.default_rng(n)
    a = rng.standard_normal((batch, n, n)) + 0.1 * n * np.eye(n)[None]
    a[0] = np.eye(n)[rng.permutation(n)]                       # pure permutation: pivoting (test_dense_batch.cpp:88-96)
    got = hdg.lu_invert_batch(ctx, np.transpose(a, (0, 2, 1)).ravel(), n, batch).reshape(batch, n, n).transpose(0, 2, 1)
    for b in range(batch):
        defect = np.max(np.abs(a[b] @ got[b] - np.eye(n)))
        assert defect <= 1e-10, (b, defect)                    # test_dense_batch.cpp:71-86
    assert np.array_equal(got[0], a[0].T)


@pytest.mark.parametrize("n", [3, 20, 40, 96, 150])
def test_singular_block_reports_lowest_index(ctx, lu_kernel, n):
    rng = np.random.default_rng(7)
    a = rng.standard_normal((6, n, n)) + n * np.eye(n)[None]
    a[4] = 0.0
    a[2, :, 1] = a[2, :, 0]                                    # rank deficient
    with pytest.raises(hdg.SingularBlock) as ei:
        hdg.lu_invert_batch(ctx, np.transpose(a, (0, 2, 1)).ravel(), n, 6)
    assert ei.value.index == 2                                 # lowest bad index (dense_batch.cpp:84-97)
    a[2] = np.eye(n)
    with pytest.raises(hdg.SingularBlock) as ei:
        hdg.lu_invert_batch(ctx, np.transpose(a, (0, 2, 1)).ravel(), n, 6)
    assert ei.value.index == 4
    a[4] = np.nan
    with pytest.raises(hdg.SingularBlock):
        hdg.lu_invert_batch(ctx, np.transpose(a, (0, 2, 1)).ravel(), n, 6)


def test_blocked_gj_large_batch_and_ill_scaled_rows(ctx):
    """More blocks than one grid chunk (65 535) and rows of wildly different scale: the pivot search has to
    pick the large rows first (partial pivoting, dense_batch.cpp:27-36)."""
    n, batch = 26, 66000
    rng = np.random.default_rng(5)
    a = rng.standard_normal((batch, n, n)) + 3.0 * np.eye(n)[None]
    a[:, ::3, :] *= 1e6
    a[65999] = np.eye(n)[::-1]
    got = hdg.lu_invert_batch(ctx, np.transpose(a, (0, 2, 1)).ravel(), n, batch).reshape(batch, n, n).transpose(0, 2, 1)
    for b in (0, 1, 40000, 65535, 65536, 65999):
        assert np.max(np.abs(got[b] @ a[b] - np.eye(n))) <= 1e-9, b
    a[65990] = 0.0
    with pytest.raises(hdg.SingularBlock) as ei:
        hdg.lu_invert_batch(ctx, np.transpose(a, (0, 2, 1)).ravel(), n, batch)
    assert ei.value.index == 65990


@pytest.fixture(params=["dmma", "fma"])
def gemm_kernel(request):
    hdg.set_tuning("use_dmma", 1 if request.param == "dmma" else 0)
    yield request.param
    hdg.set_tuning("use_dmma", 1)


@pytest.mark.parametrize("m,k,n,batch", [(3, 4, 5, 7), (9, 9, 12, 33), (64, 64, 96, 3), (96, 64, 96, 2), (20, 33, 17, 5),
                                         (30, 10, 24, 50), (72, 10, 10, 9), (15, 15, 33, 11), (320, 64, 96, 2),
                                         (130, 70, 129, 2), (16, 16, 24, 70000)])
def test_gemm_batch_and_broadcast(ctx, gemm_kernel, m, k, n, batch):
    if batch > 1000 and gemm_kernel != "dmma":
        pytest.skip("large batch: tensor-core path only")
    rng = np.random.default_rng(m * 7 + n)
    a = rng.standard_normal((batch, k, m))                     # [b][col][row]: column-major m x k
    b = rng.standard_normal((batch, n, k))
    want = np.einsum("bkm,bnk->bnm", a, b)                     # C[b][col n][row m]
    tol = 1e-13 * k * max(1.0, np.max(np.abs(want)))
    got = hdg.gemm_batch(ctx, a.ravel(), m, k, batch, b.ravel(), k, n, batch).reshape(batch, n, m)
    assert np.max(np.abs(got - want)) <= tol
    got = hdg.gemm_batch(ctx, a[0].ravel(), m, k, 1, b.ravel(), k, n, batch).reshape(batch, n, m)   # A broadcast
    assert np.max(np.abs(got - np.einsum("km,bnk->bnm", a[0], b))) <= tol
    at = rng.standard_normal((batch, m, k))                    # stored k x m, used transposed
    got = hdg.gemm_batch(ctx, at.ravel(), k, m, batch, b.ravel(), k, n, batch, transpose_a=True).reshape(batch, n, m)
    assert np.max(np.abs(got - np.einsum("bmk,bnk->bnm", at, b))) <= tol
    with pytest.raises(hdg.DimensionMismatch):
        hdg.gemm_batch(ctx, a.ravel(), m, k, batch, b.ravel(), k + 1, n, batch)


@pytest.mark.parametrize("n,batch", [(16, 30), (40, 50), (64, 33), (96, 21), (128, 5)])
def test_blocked_gj_direct_placement_is_bitwise_the_copy_form(ctx, n, batch):
    """`gj_direct` (default, out-of-place inverses with n <= 128): the first panel reads the input and the last panel and
    update write the inverse's columns at their final places.  Same arithmetic as the form with a copy prepass and a
    separate column-permutation pass: identical bits, including blocks whose pivoting permutes every row."""
    rng = np.random.default_rng(100 + n)
    a = rng.standard_normal((batch, n, n))
    a[1] = np.eye(n)[rng.permutation(n)] * rng.uniform(0.5, 2.0, n)[None, :]
    flat = np.transpose(a, (0, 2, 1)).ravel()
    out = {}
    for flag in (1, 0):
        hdg.set_tuning("gj_direct", flag)
        try:
            out[flag] = hdg.lu_invert_batch(ctx, flat, n, batch)
        finally:
            hdg.set_tuning("gj_direct", 1)
    assert np.array_equal(out[0], out[1])
