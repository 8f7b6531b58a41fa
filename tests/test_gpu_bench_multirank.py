"""The N > 1 path of bench.py (one process per GPU, placement by rank 0,
broadcast plan, max-over-ranks timing) exercised on a single-GPU box: two
ranks pinned to cuda:0 over gloo (PRISM_BENCH_DEVICE / PRISM_BENCH_BACKEND).
Timings are meaningless here; the test checks the contract: one JSON line
from rank 0, whole-job tokens over both ranks, each rank's models placed by
Algorithm 1 on its own ledger."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_ranks_one_json_line():
    env = dict(os.environ, PRISM_BENCH_BACKEND="gloo", PRISM_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", "--steps", "3",
           "--warmup", "3"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    res = json.loads(lines[0])
    assert res["n_gpus"] == 2 and res["scaling"] == "weak"
    assert res["value"] > 0 and res["e2e"]["value"] > 0
    assert "2 GPU(s)" in res["config"]["parallelism"]
    assert res["gpu_launches"] > 0
