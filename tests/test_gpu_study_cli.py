"""The study harness and CLI mirror against the reference's own
harness compiled in place: CSV schema v1, iteration counts per sweep row, convergence orders, exit codes
(test_study.cpp / test_cli.cpp), and the .hdgk dump byte format (test_face_matrix.cpp:231-251)."""
import io
import struct

import numpy as np
import pytest

import paper_2512_13619_b200 as hdg
from paper_2512_13619_b200 import study as S
from paper_2512_13619_b200.__main__ import main as cli_main

pytestmark = pytest.mark.gpu


def test_sweep_csv_schema_and_counts(ctx, ref):
    specs = [S.CaseSpec("burgers2d", k=1, n=8, precond=hdg.PrecondSpec(pc, poly_degree=deg))
             for pc, deg in (("bj", 0), ("asm", 0), ("asm", 6))]
    buf = io.StringIO()
    res = S.run_sweep(ctx, specs, buf)
    lines = buf.getvalue().split("\r\n")
    assert lines[0].split(",")[:20] == S.CSV_COLUMNS                      # study.cpp:139-142 header
    for line, r in zip(lines[1:], res):
        cols = line.split(",")
        assert cols[0] == "1" and cols[1] == "burgers2d" and cols[6] == "steady" and cols[11] == "true"
        rc = ref.RefCase("burgers2d", k=1, n=8)
        kind = {1: "bj", 2: "asm"}[r.spec.precond.kind]
        rr = rc.newton(precond=kind, poly_degree=r.spec.precond.poly_degree)
        assert int(cols[9]) == rr["n_newton"]
        assert abs(int(cols[10]) - rr["n_gmres_total"]) <= rr["n_newton"] * (2 if r.spec.precond.poly_degree else 1)
        assert float(cols[13]) > 0 and float(cols[17]) > 0                  # phase timers are filled
    # ASM < BJ and ASM-PP < ASM (acceptance_main.cpp:415-424)
    n = [r.report.n_gmres_total for r in res]
    assert n[1] < n[0] and n[2] < n[1]


def test_convergence_orders(ctx):
    rows = S.convergence_study(ctx, S.CaseSpec("poisson2d", precond=hdg.PrecondSpec("asm")), [1, 2], [4, 8, 16])
    for row in rows:
        if row["order"] not in ("", "exact"):
            assert float(row["order"]) >= row["k"] + 0.5                    # acceptance_main.cpp:392-395


def test_transient_heat_decay(ctx):
    """heat2d: u decays like exp(-2 pi^2 t) (test_newton.cpp:220-248, 10 % band)."""
    spec = S.CaseSpec("heat2d", k=2, n=8, precond=hdg.PrecondSpec("bj"), dt=0.002, n_steps=10)
    r = S.run_case(ctx, spec)
    assert r.ok and r.report.converged
    amp = np.max(np.abs(r.state.u))
    want = np.exp(-2 * np.pi ** 2 * 0.02)
    assert abs(amp - want) < 0.1 * want


def test_cli_exit_codes_and_dump(ctx, tmp_path, capsys):
    assert cli_main(["solve", "--case", "poisson2d", "--k", "2", "--n", "8", "--precond", "bj"]) == 0
    out = capsys.readouterr().out
    assert "converged:      yes" in out and "gmres iters:" in out
    assert cli_main(["solve", "--case", "burgers2d", "--k", "1", "--n", "8", "--max-newton", "1"]) == 2   # not converged
    assert cli_main(["solve", "--case", "poisson2d", "--k", "1", "--n", "4", "--tau", "0"]) == 3          # tau = 0: singular local solve (test_cli.cpp:141-145)
    assert cli_main(["solve", "--case", "nonsense"]) == 1
    path = tmp_path / "k.hdgk"
    assert cli_main(["dump", "--case", "poisson2d", "--k", "2", "--n", "3", "--out", str(path)]) == 0
    raw = path.read_bytes()
    assert raw[:4] == b"HDGK"
    ver, m, pf, n_lfe, nf = struct.unpack("<5I", raw[4:24])
    assert (ver, m, pf, n_lfe, nf) == (1, 1, 3, 4, 24)
    assert len(raw) == 24 + 8 * nf * 7 + 8 * nf * 7 * 9 + 8 * nf * 3


def test_hdgk_round_trip_and_reference_bytes(ctx, ref, tmp_path):
    rc = ref.RefCase("burgers2d", k=2, n=3)
    rc.assemble()
    pr = tmp_path / "ref.hdgk"
    rc.write_matrix(str(pr))
    K, rhs = hdg.read_matrix(ctx, str(pr))                                  # the reference's dump loads
    assert np.array_equal(K.neighbor, rc.get_i("neighbor")) and np.array_equal(K.blocks, rc.get("k_blocks"))
    assert np.array_equal(rhs, rc.get("rhs"))
    po = tmp_path / "ours.hdgk"
    hdg.write_matrix(str(po), K, rhs)
    assert po.read_bytes() == pr.read_bytes()                              # byte-identical round trip
    bad = tmp_path / "bad.hdgk"
    bad.write_bytes(b"NOPE" + pr.read_bytes()[4:])
    with pytest.raises(hdg.IoError):
        hdg.read_matrix(ctx, str(bad))
