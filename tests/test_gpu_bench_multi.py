"""The multi-GPU arm of bench.py as the driver invokes it (`python bench.py
--gpus N`, no torchrun environment): on a one-GPU lease two ranks share
device 0 (gloo for the barrier and the max over ranks); both run their timed
regions over disjoint stream blocks and rank 0 prints n_gpus 2."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks_on_one_gpu(gpu_lib, scaling):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "4", "--warmup", "3",
                          "--streams", "16", "--scaling", scaling, "--no-extras"],
                         capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    per = 16 if scaling == "weak" else 8
    assert line["n_gpus"] == 2 and line["dist_backend"] == "gloo"
    assert line["config"]["streams_per_gpu"] == per and line["config"]["streams_total"] == 2 * per
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["parity_ok"], line["parity"]  # rank 0's streams against the reference
