"""bench.py at N > 1 on the 1-GPU test box: `python bench.py --gpus 2` starts
its own two ranks (torch.distributed.run, 127.0.0.1), both ranks share
cuda:0 and gather over gloo (NCCL refuses two ranks on one GPU).  The chunked
gather of (t, distance, segment id) must reassemble, on rank 0, bit for bit
the single projection of both ranks' queries (--verify-gather)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n", [("cfg2", 100_000), ("cfg3", 20_000), ("cfg4", 20_000)])
def test_bench_two_ranks_gather_bitwise(gpu, cfg, n):
    d = _bench("--gpus", "2", "--config", cfg, "--n", str(n), "--steps", "3", "--warmup", "3",
               "--verify-gather", "--no-cpu-baseline")
    assert d["n_gpus"] == 2
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    chk = d["config"]["gather_check"]
    assert chk["queries"] == 2 * n
    assert chk["bitwise_equal"] is True
    assert "gloo" in d["config"]["gather"]
