"""bench.py --gpus N starts N ranks itself (torch.distributed.run over 127.0.0.1) when no
launcher is present; the ranks shard the config's batch and reduce the time with MAX.
CPU-only: --dry-run uses gloo instead of NCCL and skips the device work."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("n", [2, 4])
def test_bench_gpus_flag_forks_ranks(n):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--dry-run"],
                       capture_output=True, text=True, timeout=280, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == n
    assert line["max_elapsed"] == float(n)  # 1 + rank, max over ranks
    assert line["images_total"] == line["global_batch"] == 1024  # C5: global batch 1024 sharded
    assert line["scaling"] == "strong"


def test_bench_single_rank_dry_run():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", "--config", "c2"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["images_total"] == 32 and line["scaling"] == "weak"
