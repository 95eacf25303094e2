"""Rank plumbing of bench.py at world size 2 over gloo on CPU (no GPU work).

The instance-sharded arms (BASELINE c1-c3) have no data-path collective: rank r
owns the scene seeds [r B, (r + 1) B), the job's time is the slowest rank's
device time (one MAX all-reduce) and rank 0 alone prints.  The reference arm
runs on rank 0 only; the other ranks exit 0 without work or output.
"""

import json
import os
import pathlib
import socket
import subprocess
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    from paper_2503_15259_b200 import scenes
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, r, local = bench.dist_setup(None)
        assert (w, r, local) == (world, rank, rank)
        B = 3
        ids = bench.instance_ids(r, B)
        # each rank draws its own scenes: different seeds give different data
        cfg = scenes.SceneConfig(5, "ml-ud", 24, 6, 8, 3, 4, B)
        first = scenes.make_scene(cfg, ids[0])
        bench.rank_barrier(w)
        ms_local = 10.0 + 5.0 * r                     # rank 1 is the slow one
        ms = bench.max_over_ranks(ms_local, w, torch.device("cpu"))
        q.put((r, ids, ms, bench.whole_job_rate(w, B, 2, ms),
               float(np.abs(first.pilots).sum())))
    finally:
        dist.destroy_process_group()


def test_instance_sharding_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, ids0, ms0, v0, s0), (r1, ids1, ms1, v1, s1) = got
    assert ids0 == [0, 1, 2] and ids1 == [3, 4, 5]            # disjoint, contiguous, complete
    assert ms0 == ms1 == 15.0                                  # the slowest rank's time, on both
    assert v0 == v1 == 2 * 3 * 2 / 15.0e-3                     # whole-job instances / s
    assert s0 != s1                                            # different instances per rank


def test_reference_arm_runs_on_rank_zero_only():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1", MASTER_ADDR="127.0.0.1",
               MASTER_PORT=str(_free_port()))
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], env=env, capture_output=True, text=True,
                       timeout=120)
    assert p.returncode == 0, p.stderr[-1000:]
    assert p.stdout.strip() == ""


def test_single_rank_helpers_need_no_process_group():
    import bench
    assert bench.max_over_ranks(3.5, 1, torch.device("cpu")) == 3.5
    bench.rank_barrier(1)
    assert bench.instance_ids(0, 4) == [0, 1, 2, 3]
    assert json.dumps(bench.whole_job_rate(1, 4096, 5, 1000.0)) == "20480.0"
