"""The N > 1 path of bench.py (BASELINE config 3: 24 images sharded over the
ranks, batched per GPU): two ranks launched the way the driver launches them
(torch.distributed.run, 127.0.0.1), sharing this pool's one GPU through a gloo
process group (BENCH_SHARED_GPU=1, a code-path check, not a timing)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_bench_two_ranks_print_one_cfg3_line(gpu_lib):
    env = dict(os.environ, BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--images", "4"]
    r = subprocess.run(cmd, env=env, cwd=str(REPO), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["config"]["images_per_gpu"] == 2 and d["config"]["images_total"] == 4
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["costs_finite"]
    assert d["scaling"] == "strong"
