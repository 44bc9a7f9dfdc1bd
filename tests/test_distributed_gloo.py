"""World-size-2 gloo tests of the multi-GPU host logic (run on CPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_10986_b200 import distributed as Dd


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, size, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        # per-image stats of a 10-image job sharded 2 ways
        rng = np.random.default_rng(0)
        full = rng.uniform(0, 1, (10, 4))
        full[:, 2] = 49.0
        a, b = Dd.shard_range(10, rank, size)
        got = Dd.gather_ordered(torch.from_numpy(full[a:b].copy())).numpy()
        # per-trial vector with uneven shards
        trials = np.arange(7, dtype=np.float64) * 0.5
        a2, b2 = Dd.shard_range(7, rank, size)
        counts = [Dd.shard_range(7, r, size)[1] - Dd.shard_range(7, r, size)[0] for r in range(size)]
        pt = Dd.gather_ordered(torch.from_numpy(trials[a2:b2].copy()), counts).numpy()
        mx = Dd.max_over_ranks(float(rank + 3))
        out[rank] = (got.tobytes() == full.tobytes(), pt.tobytes() == trials.tobytes(), mx,
                     Dd.combine_layer_stats(got))
    finally:
        dist.destroy_process_group()


def test_world_size_2_gather_and_max():
    size = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(size, port, out), nprocs=size, join=True)
    ref = Dd.combine_layer_stats(np.random.default_rng(0).uniform(0, 1, (10, 4)) * [1, 1, 0, 1] + [0, 0, 49, 0])
    for r in range(size):
        ok_stats, ok_trials, mx, comb = out[r]
        assert ok_stats and ok_trials and mx == 4.0
        assert comb == ref  # identical, bit for bit, to the single-process result


def test_shard_range_partitions():
    for total in (0, 1, 7, 32, 5000):
        for size in (1, 2, 3, 4, 8):
            spans = [Dd.shard_range(total, r, size) for r in range(size)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(size - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    assert list(Dd.weak_image_indices(32, 3)) == list(range(96, 128))
    with pytest.raises(ValueError):
        Dd.shard_range(10, 2, 2)


def test_layer_shards_cover_outputs_once():
    for N, K in ((8, 64), (3, 70), (1, 5)):
        for size in (1, 2, 4, 8):
            for by in ("batch", "filters"):
                seen = np.zeros((N, K), dtype=int)
                for r in range(size):
                    ni, ki = Dd.layer_shard(N, K, r, size, by)
                    seen[ni, ki] += 1
                assert (seen == 1).all(), (N, K, size, by)
    with pytest.raises(ValueError):
        Dd.layer_shard(4, 4, 0, 2, "pixels")


def _measure_worker(rank, size, port, out):
    import paper_1803_10986_b200 as W
    from oracle import wino_oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        pts = "0,1,-1,1/2,-1/2,inf"
        ts = W.build_transforms(3, 4, W.parse_points(pts))
        trip = O.Triple.from_points(3, 4, pts)
        cfg = W.ConvConfig("fp32", "huffman", "pairwise")

        def local_eval(a, b):  # host stand-in for the device Monte-Carlo kernels
            return O.measure_error(trip, 2, "fp32", "huffman", "pairwise", trials=b - a, seed=3, channels=4,
                                   t0=a)[0]

        rep = Dd.measure_error_sharded(ts, 2, cfg, trials=37, seed=3, channels=4, local_eval=local_eval,
                                       mean=lambda per: float(np.mean(per.numpy())))
        out[rank] = (rep.per_trial.tobytes(), repr(rep.total_l1_mean), rep.trials, rep.per_point_l1_mean)
    finally:
        dist.destroy_process_group()


def test_world_size_2_measure_error_sharded_equals_one_process():
    """The sharded Monte-Carlo measurement (contiguous trial shards, per-trial L1
    gathered in trial order) reproduces the one-process report bit for bit
    (reference harness.py:97-107: draws keyed by (seed, trial))."""
    from oracle import wino_oracle as O
    size = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_measure_worker, args=(size, port, out), nprocs=size, join=True)
    trip = O.Triple.from_points(3, 4, "0,1,-1,1/2,-1/2,inf")
    per, tot, pp = O.measure_error(trip, 2, "fp32", "huffman", "pairwise", trials=37, seed=3, channels=4)
    for r in range(size):
        per_b, tot_r, trials, pp_r = out[r]
        assert per_b == per.tobytes() and tot_r == repr(tot) and trials == 37 and pp_r == tot / 16


def test_bench_launcher_spawns_ranks():
    """`bench.py --gpus 2` with no torchrun environment re-execs itself under
    torch.distributed.run; the --dry-run rehearsal runs the multi-rank plumbing
    (rank env, batch shards, MAX-over-ranks timing, ordered gather of per-image
    error partials) on CPU/gloo and rank 0 prints one JSON line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run",
                          "--vgg-batch", "6", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True
    assert d["shards"] == [[0, 3], [3, 6]]
    assert d["error_images"] == 6 and d["error_equals_one_process"] is True
