"""Multi-GPU sharding: one process per GPU, torch.distributed for plumbing.

The convolution path shards without any exchange (tiles / images / trials are
independent); collectives only combine results:
  * per-image layer error partials and per-trial L1 values are all-gathered
    and reduced in global index order on every rank, so every statistic is
    bit-identical for 1, 2, 4 or 8 GPUs;
  * step times are reduced with MAX (the slowest rank defines the job time).
Works with the NCCL backend on GPUs and with gloo on CPU tensors (tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_range(total: int, rank: int, size: int) -> tuple[int, int]:
    """Contiguous [start, stop) slice of `total` units for `rank` (balanced,
    deterministic; the first total % size ranks get one extra unit)."""
    if size < 1 or not 0 <= rank < size:
        raise ValueError("bad rank / world size")
    base, extra = divmod(total, size)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def layer_shard(N: int, K: int, rank: int, size: int, by: str = "batch") -> tuple[slice, slice]:
    """(image slice, filter slice) of a layer a rank computes.  "batch": a
    contiguous block of images, all filters; "filters": all images, a contiguous
    block of output channels (for batches smaller than the GPU count).  Either
    way every output is computed exactly as on one GPU (outputs are independent),
    and the shards stay on their ranks -- no collective on the convolution path."""
    if by == "batch":
        a, b = shard_range(N, rank, size)
        return slice(a, b), slice(0, K)
    if by == "filters":
        a, b = shard_range(K, rank, size)
        return slice(0, N), slice(a, b)
    raise ValueError("by must be 'batch' or 'filters'")


def conv2d_layer_shard(ts, x, w, cfg, pad: int = 0, by: str = "batch", contraction: str = "exact"):
    """This rank's shard of a layer: y[images, filters] for layer_shard(...);
    x (N, C, H, W) and w (K, C, r, r) are the full tensors (each rank reads only
    what its shard needs)."""
    from .layer import conv2d_layer
    rank, size = world()
    ni, ki = layer_shard(x.shape[0], w.shape[0], rank, size, by)
    return conv2d_layer(ts, x[ni], w[ki], cfg, pad, contraction), (ni, ki)


def weak_image_indices(per_rank: int, rank: int) -> range:
    """Global image indices of a rank in a weak-scaling run (per-rank batch fixed)."""
    return range(rank * per_rank, (rank + 1) * per_rank)


def gather_ordered(local: torch.Tensor, counts: list[int] | None = None) -> torch.Tensor:
    """All-gather variable-length leading-axis chunks and concatenate them in
    rank order (== global index order for contiguous shards)."""
    rank, size = world()
    if size == 1:
        return local
    if counts is None:
        n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
        ns = [torch.zeros_like(n) for _ in range(size)]
        dist.all_gather(ns, n)
        counts = [int(v.item()) for v in ns]
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(size)]
    dist.all_gather(bufs, pad)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)])


def max_over_ranks(value: float, device=None) -> float:
    rank, size = world()
    if size == 1:
        return float(value)
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def combine_layer_stats(stats: np.ndarray) -> dict:
    """stats[N][4] per image (sum|err|, sum|ref|, count, max|err|), already in
    global image order -> job-level error statistics (ordered fp64 sums)."""
    s = np.asarray(stats, dtype=np.float64)
    err = ref = cnt = 0.0
    mx = 0.0
    for row in s:  # fixed global order -> world-size invariant
        err += row[0]
        ref += row[1]
        cnt += row[2]
        mx = max(mx, row[3])
    return {"rel_l1": err / ref if ref else float("nan"), "per_point_l1": err / cnt if cnt else float("nan"),
            "max_abs": mx, "images": int(s.shape[0])}


def trial_counts(trials: int, size: int) -> list[int]:
    """Trials per rank of a contiguous split (shard_range)."""
    return [shard_range(trials, r, size)[1] - shard_range(trials, r, size)[0] for r in range(size)]


def gather_trials(local: torch.Tensor, trials: int) -> torch.Tensor:
    """This rank's per-trial L1 values -> the full per-trial vector in trial order
    (identical on every rank).  Trials are keyed Philox(seed, trial) by the
    reference (harness.py:97-107), so the gathered vector equals the one-process
    vector bit for bit whatever the world size."""
    rank, size = world()
    counts = trial_counts(trials, size)
    if local.shape[0] != counts[rank]:
        raise ValueError("local trial count does not match this rank's shard")
    return gather_ordered(local, counts).contiguous()


def measure_error_sharded(spec, dims, cfg, trials=5000, seed=0, channels=1, local_eval=None, mean=None):
    """measure_error with the trials split across ranks: each rank evaluates a
    contiguous slice, the per-trial L1 values are gathered in trial order and
    the mean is taken over the full vector on every rank -- the report equals
    the single-GPU one bit for bit.

    local_eval(start, stop) -> per-trial L1 (float64) of trials start..stop-1 and
    mean(vector) -> float default to the device paths (libwino Monte-Carlo kernels,
    numpy-ordered device mean); tests substitute host versions to exercise the
    sharding and gather logic on CPU ranks (gloo)."""
    from .harness import ErrorReport

    rank, size = world()
    start, stop = shard_range(trials, rank, size)
    if local_eval is None:
        local_eval = _device_trials(spec, dims, cfg, seed, channels)
        dev = "cuda"
    else:
        dev = "cpu"
    part = local_eval(start, stop) if stop > start else np.zeros(0, dtype=np.float64)
    local = torch.as_tensor(np.ascontiguousarray(part, dtype=np.float64), device=dev)
    per = gather_trials(local, trials)
    total = float(mean(per) if mean is not None else _device_mean(per))
    n_out = spec.n_o ** dims
    return ErrorReport(descriptor=spec.descriptor(), dims=dims, channels=channels,
                       config={"precision": cfg.precision, "dot_order": cfg.dot_order,
                               "channel_sum": cfg.channel_sum},
                       trials=trials, seed=seed, total_l1_mean=total, per_point_l1_mean=total / n_out,
                       n_outputs=n_out, per_trial=per.cpu().numpy())


def _device_trials(spec, dims, cfg, seed, channels):
    from .harness import _measure_variants

    def run(start, stop):
        return _measure_variants(spec, dims, cfg, stop - start, seed, channels, (cfg.channel_sum,),
                                 t0=start)[cfg.channel_sum].per_trial
    return run


def _device_mean(per: torch.Tensor) -> float:
    from . import _native
    from . import device as D
    mean = D.torch.empty(1, dtype=D.torch.float64, device="cuda")
    _native.check(_native.lib().wino_mean_f64(per.shape[0], D.ptr(per), D.ptr(mean), D.stream_handle()), "mean")
    return float(mean.item())
