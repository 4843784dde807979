"""The two GEMV kernels (team kernel and the TMA stream kernel) against numpy on every block shape
of the BASELINE configurations (and awkward ones: odd rows, odd tails, split items), contiguous and
gathered inputs.  gemv is a sum of `cols` products per entry: tolerance 1e-13 relative to |A||x|."""
import numpy as np
import pytest

import paper_2512_13619_b200 as hdg

pytestmark = pytest.mark.gpu

SHAPES = [(3, 21, 1001), (5, 25, 333), (16, 176, 97), (18, 126, 41), (80, 880, 5), (12, 12, 515), (15, 15, 77),
          (96, 96, 9), (72, 72, 13), (16, 16, 1000), (27, 27, 30), (9, 63, 201), (64, 64, 7), (130, 40, 6), (7, 7, 1),
          # long streams: every warp's TMA ring wraps many times
          (16, 176, 6000), (96, 96, 3000), (3, 21, 150001), (64, 96, 4001), (5, 25, 40003), (18, 126, 5000),
          # packed small-item mode: odd / even rows, odd column counts, items per pass 2 .. 32
          (1, 1, 5000), (2, 3, 70001), (5, 5, 90001), (6, 18, 30000), (10, 30, 20001), (15, 15, 50001), (16, 16, 40000),
          (32, 32, 9001), (4, 31, 12345)]


@pytest.fixture(params=["team", "stream", "stream-unpacked"])
def kernel(request):
    """stream: small items take the packed mode (several items per warp pass); stream-unpacked forces the
    one-item-per-warp mapping for every shape."""
    if request.param.startswith("stream"):
        hdg.set_tuning("use_stream", 1)
        hdg.set_tuning("stream_min_elems", 0)
        hdg.set_tuning("stream_packed", 0 if request.param == "stream-unpacked" else 1)
    else:
        hdg.set_tuning("use_stream", 0)
    yield request.param
    hdg.set_tuning("use_stream", 1)
    hdg.set_tuning("stream_packed", 1)
    hdg.set_tuning("stream_min_elems", 1 << 18)


@pytest.mark.parametrize("rows,cols,batch", SHAPES)
def test_gemv_strided_batch(ctx, kernel, rows, cols, batch):
    rng = np.random.default_rng(rows * 1000 + cols)
    a = rng.standard_normal((batch, cols, rows))        # [b][c][r] = column-major blocks
    x = rng.standard_normal((batch, cols))
    y0 = rng.standard_normal((batch, rows))
    want = np.einsum("bcr,bc->br", a, x)
    bound = 1e-13 * np.einsum("bcr,bc->br", np.abs(a), np.abs(x)).max()
    got = hdg.gemv_strided_batch(ctx, a.ravel(), rows, cols, batch, x.ravel())
    assert np.max(np.abs(got.reshape(batch, rows) - want)) <= bound
    got = hdg.gemv_strided_batch(ctx, a.ravel(), rows, cols, batch, x.ravel(), y=y0.ravel(), accumulate=True)
    assert np.max(np.abs(got.reshape(batch, rows) - (want + y0))) <= bound + 1e-15


@pytest.mark.parametrize("mpf,n_lfe,nf", [(3, 4, 501), (5, 3, 333), (16, 6, 131), (18, 4, 57), (80, 6, 9), (1, 4, 50),
                                          (16, 6, 7000), (3, 4, 120001), (80, 6, 300)])
def test_block_matvec_gather(ctx, kernel, mpf, n_lfe, nf):
    rng = np.random.default_rng(mpf * 100 + nf)
    nb = 2 * n_lfe - 1
    nbr = rng.integers(-1, nf, size=(nf, nb)).astype(np.int64)
    nbr[:, 0] = np.arange(nf)
    blocks = rng.standard_normal((nf, nb, mpf, mpf))     # [f][slot][c][r]
    K = hdg.FaceBlockMatrix.from_host(ctx, 1, mpf, n_lfe, nf, nbr.ravel(), blocks.ravel())
    x = rng.standard_normal(nf * mpf)
    xs = np.where(nbr[..., None] >= 0, x.reshape(nf, mpf)[np.maximum(nbr, 0)], 0.0)   # [f][slot][c]
    want = np.einsum("fscr,fsc->fr", blocks, xs)
    bound = 1e-13 * np.einsum("fscr,fsc->fr", np.abs(blocks), np.abs(xs)).max()
    got = hdg.block_matvec(K, x).reshape(nf, mpf)
    assert np.max(np.abs(got - want)) <= bound
    assert np.array_equal(hdg.gather_extended(K, x).reshape(nf, nb, mpf), xs)


def test_stream_and_team_agree_on_a_real_system(ctx):
    disc = hdg.Discretization.structured(ctx, "hex", n=4, degree=2)
    model = hdg.make_case_model(disc, "poisson")
    state = hdg.make_initial_state(disc, model)
    ops = hdg.assemble_element_operators(disc, model, state)
    K, rhs = hdg.assemble_global(disc, ops)
    P = hdg.build_preconditioner("asm", K, ops, disc)
    x = hdg.random_vector(K.n_dof, 8)
    out = {}
    for name, flag in (("team", 0), ("stream", 1)):
        hdg.set_tuning("use_stream", flag)
        hdg.set_tuning("stream_min_elems", 0)
        out[name] = (hdg.block_matvec(K, x), P.apply_base(x), hdg.gmres_solve(K, P, rhs)[1].iters)
    hdg.set_tuning("use_stream", 1)
    hdg.set_tuning("stream_min_elems", 1 << 18)
    assert np.max(np.abs(out["team"][0] - out["stream"][0])) < 1e-12 * np.max(np.abs(out["team"][0]))
    assert np.max(np.abs(out["team"][1] - out["stream"][1])) < 1e-12 * np.max(np.abs(out["team"][1]))
    assert out["team"][2] == out["stream"][2]
