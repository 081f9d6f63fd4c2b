"""CPU coverage of the multi-GPU path (bench.py): world_size 2 over gloo.

Frames shard by index with no data-path collective; the only collective is an
all_gather of per-rank stats, and the whole-job rate is all frames divided by the
MAX over ranks of the device time (weak scaling)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = bench.shard_frames(rank, world, 4)
        enc, dec = 10.0 * (rank + 1), 20.0 * (rank + 1)  # rank 1 is the slow one
        st = bench.rank_stats(4, 1000 * (rank + 1), 500, 64 * (rank + 1), enc, dec, True, 50.0 + rank)
        allst = bench.gather_stats(dist, st, "cpu", world)
        q.put((rank, frames, allst.tolist(), bench.aggregate(allst, K=3)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_stats_and_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    res.sort()
    f0, f1 = res[0][1], res[1][1]
    assert not set(f0) & set(f1) and sorted(f0 + f1) == list(range(8))  # disjoint shards
    assert res[0][2] == res[1][2]  # every rank sees the same gathered stats
    agg = res[0][3]
    assert agg["frames"] == 8 * 3
    # max-over-ranks time: rank 1 took (20 + 40) ms per 3 steps in total
    assert agg["t_max_ms"] == pytest.approx(60.0)
    assert agg["value"] == pytest.approx(24 / 0.060)
    assert agg["enc_fps"] == pytest.approx(24 / 0.020) and agg["dec_fps"] == pytest.approx(24 / 0.040)
    assert agg["points"] == 3000 * 3 and agg["mismatch"] == 0 and agg["e2e_ms_max"] == pytest.approx(51.0)


def test_single_rank_aggregate_matches_definition():
    st = bench.rank_stats(64, 8_000_000, 3_600_000, 2_000_000, 8.0, 12.0, True, 30.0)
    agg = bench.aggregate(bench.gather_stats(None, st, "cpu", 1), K=10)
    assert agg["value"] == pytest.approx(640 / 0.020)  # stats carry the summed K-step times
    assert np.isclose(agg["enc_fps"], 640 / 0.008) and np.isclose(agg["dec_fps"], 640 / 0.012)


def test_sequence_shard_covers_every_frame_once():
    """cfg5 (BASELINE configs[4]): the 1000-frame sequence is split by index, frame i on
    rank i mod W, every frame on exactly one rank for W = 1..8."""
    import bench
    for W in range(1, 9):
        parts = [bench.sequence_shard(r, W) for r in range(W)]
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(bench.SEQ_FRAMES))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_default_batch_per_workload():
    """bench defaults: 2048 frames per GPU (4 lanes x 512) up to L = 12, 1024 at L = 13, 256 for
    deeper trees."""
    import bench
    assert bench.default_batch("cfg2") == 2048 and bench.default_batch("cfg2_L13") == 1024
    assert bench.default_batch("cfg2_L14") == 256 and bench.default_batch("cfg3") == 256
    assert bench.default_batch("cfg2_t3") == 2048


def test_bench_gpus2_spawns_two_gloo_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself under
    torch.distributed.run with 2 ranks; here over gloo with the codec-free runner, the
    whole plumbing (process group, shards, barriers, max-over-ranks time, the stats
    all_gather, rank 0's single JSON line) runs on CPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--backend", "gloo",
                        "--plumbing-selftest", "--steps", "3", "--warmup", "3", "--batch", "4"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=300)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout + r.stderr
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["details"]["backend"] == "gloo"
    assert line["config"]["global_batch"] == 8 and line["steps"] == 3
    # rank 1 is the slow one: 4 ms per step -> 24 frames / 12 ms
    assert line["ms_per_step"] == pytest.approx(4.0)
    assert line["value"] == pytest.approx(24 / 0.012)


def test_bench_rejects_world_mismatch():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--plumbing-selftest"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stdout + r.stderr)
