"""The multi-rank path with REAL processes: bench.py --gpus 2 starts two ranks itself (torch.distributed.run on
127.0.0.1); on a 1-GPU box they share the device and exchange through the host-staged gloo transport -- the same
domain-decomposed solver code (partitioner, ghost layer, halo plan, overlap window, 2 all-reduces per Arnoldi
step) as over NCCL.  The fixed global mesh cut into two slabs must reproduce the single-rank solve: same Newton
count, GMRES iterations within +-1 per Newton step, same residual."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def run_bench(*args):
    cmd = [sys.executable, str(ROOT / "bench.py"), "--steps", "1", "--warmup", "1", "--no-cpu-baseline", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout          # exactly one JSON line, printed by rank 0
    return json.loads(lines[0])


def test_two_rank_strong_scaling_run_reproduces_single_rank():
    one = run_bench("--gpus", "1", "--cells", "8")
    two = run_bench("--gpus", "2", "--cells", "8", "--scaling", "strong")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["scaling"] == "strong" and "2 ranks" in two["decomposition"]["parallelism"]
    assert two["decomposition"]["trace_dofs_global"] == one["decomposition"]["trace_dofs_global"]
    assert two["decomposition"]["trace_dofs_rank0"] < one["decomposition"]["trace_dofs_rank0"]
    assert two["n_newton"] == one["n_newton"]
    assert abs(two["n_gmres_total"] - one["n_gmres_total"]) <= one["n_newton"]
    assert abs(two["final_residual"] - one["final_residual"]) <= 1e-9
    assert two["gpu_launches"] > 0
