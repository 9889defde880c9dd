"""World-size-2 gloo test of the stream-sharded multi-GPU host logic used by
bench.py (paper_2112_13169_b200/multi.py): disjoint stream ownership, the
max-over-ranks timing and the whole-job throughput. CPU only."""
from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2112_13169_b200 import multi

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, r, lr = multi.env()
    owned = list(multi.stream_range(64, r))
    elapsed = 1.0 + r  # rank 1 is slower
    slowest = multi.max_over_ranks(elapsed)
    fps = multi.job_throughput(64 * 10, w, slowest)
    dist.barrier()
    q.put((r, w, lr, owned[0], owned[-1], slowest, fps))
    dist.destroy_process_group()


def test_two_rank_sharding_and_max_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, w0, l0, a0, b0, s0, f0), (r1, w1, l1, a1, b1, s1, f1) = out
    assert (w0, w1) == (2, 2) and (l0, l1) == (0, 1)
    assert (a0, b0, a1, b1) == (0, 63, 64, 127)  # disjoint contiguous stream blocks
    assert s0 == s1 == 2.0                        # both see the slowest rank's time
    assert f0 == f1 == pytest.approx(64 * 10 * 2 / 2.0)


def _bench(*extra):
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in __import__("os").environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--plumbing-only", "--steps", "3", *extra],
                         capture_output=True, text=True, timeout=240, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("scaling,per_rank", [("weak", 64), ("strong", 32)])
def test_bench_relaunches_ranks_for_gpus_flag(scaling, per_rank):
    """`python bench.py --gpus 2` without a torchrun environment spawns two
    ranks itself (gloo here: no GPUs), each owning its own stream block, and
    rank 0 reports n_gpus 2 with the max over ranks of the timed region (rank 1
    sleeps 10 ms in it)."""
    line = _bench("--gpus", "2", "--scaling", scaling)
    assert line["n_gpus"] == 2 and line["backend"] == "gloo"
    assert line["streams_per_rank"] == per_rank
    assert line["owned"] == [[0, per_rank - 1], [per_rank, 2 * per_rank - 1]]
    assert line["max_seconds"] >= 0.01
    assert line["config"]["streams_total"] == 2 * per_rank


def test_bench_single_rank_default():
    line = _bench()
    assert line["n_gpus"] == 1 and line["backend"] is None and line["owned"] == [[0, 63]]
