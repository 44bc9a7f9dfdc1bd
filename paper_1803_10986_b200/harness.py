"""Monte-Carlo error measurement on the GPU (drop-in for the measurement core of
the reference's toomcook.harness, /root/reference/pkg/src/toomcook/harness.py:45-207).

Per trial a fresh kernel and input are drawn uniform(-1, 1) in fp32 from the
Philox stream keyed by (seed, trial) -- generated on the device by the same
Philox4x64-10 numpy uses, so the draws are bit-identical -- and the error is
the L1 distance between the convolution under test and the fp64 direct
reference.  Every stage (draws, fp64 reference, Winograd pipeline, per-trial
L1 in numpy's summation order, the mean) runs in libwino kernels, so the
reported numbers equal the reference's repr for repr.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from . import _native
from . import device as D
from .engine import ConvConfig, _reduce, get_plan


@dataclass(frozen=True)
class DirectSpec:
    """Stands in for a TransformSet when measuring plain direct convolution."""

    n_h: int
    n_o: int

    @property
    def n(self) -> int:
        return self.n_h + self.n_o - 1

    def descriptor(self) -> dict:
        return {"direct": True, "n_h": self.n_h, "n_o": self.n_o, "n": self.n}


@dataclass
class ErrorReport:
    descriptor: dict
    dims: int
    channels: int
    config: dict
    trials: int
    seed: int
    total_l1_mean: float
    per_point_l1_mean: float
    n_outputs: int
    per_trial: np.ndarray | None = field(repr=False, default=None)

    def to_json_dict(self, include_trials: bool = False) -> dict:
        d = {"descriptor": self.descriptor, "dims": self.dims, "channels": self.channels,
             "config": self.config, "trials": self.trials, "seed": self.seed,
             "total_l1_mean": repr(self.total_l1_mean), "per_point_l1_mean": repr(self.per_point_l1_mean),
             "n_outputs": self.n_outputs}
        if include_trials and self.per_trial is not None:
            d["per_trial"] = [repr(float(v)) for v in self.per_trial]
        return d

    def write_json(self, path, include_trials: bool = False) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            json.dump(self.to_json_dict(include_trials), fh, indent=1)
            fh.write("\n")


def _draw(seed, t0, B, dims, n_h, n, channels):
    kshape = (B, channels) + (n_h,) * dims
    xshape = (B, channels) + (n,) * dims
    h = D.empty(kshape, np.float32)
    x = D.empty(xshape, np.float32)
    _native.check(_native.lib().wino_trial_inputs(seed & 0xFFFFFFFFFFFFFFFF, t0, B, dims, n_h, n, channels,
                                                  D.ptr(h), D.ptr(x), D.stream_handle()), "trial_inputs")
    return h, x


def trial_inputs(seed: int, trial: int, dims: int, n_h: int, n: int, channels: int = 1):
    """The (kernel, input) pair of one trial, drawn on the device (harness.py:97-107)."""
    D.require_cuda()
    h, x = _draw(seed, trial, 1, dims, n_h, n, channels)
    return h[0].cpu().numpy(), x[0].cpu().numpy()


def _direct(h, x, dims, dtype_code):
    """direct_products on device tensors -> (B, C, o...)"""
    B, C = h.shape[0], h.shape[1]
    r, n = h.shape[-1], x.shape[-1]
    o = n - r + 1
    out = D.empty((B, C) + (o,) * dims, np.float64 if dtype_code else np.float32)
    _native.check(_native.lib().wino_direct_products(dims, dtype_code, 0, B, C, r, n, D.ptr(h), D.ptr(x),
                                                     D.ptr(out), D.stream_handle()), "direct_products")
    return out


def _chunk_size(trials: int, dims: int, n: int, channels: int) -> int:
    per_trial = channels * n ** dims
    return max(1, min(trials, (64 << 20) // max(per_trial, 1)))


def _measure_variants(spec, dims, cfg, trials, seed, channels, variants, t0=0):
    """Trials t0 .. t0+trials-1 (t0 > 0 when a rank evaluates a shard)."""
    direct = isinstance(spec, DirectSpec)
    n_h, n_o, n = spec.n_h, spec.n_o, spec.n
    n_out = n_o ** dims
    per = {v: D.torch.empty(trials, dtype=D.torch.float64, device="cuda") for v in variants}
    if not direct:
        plan = get_plan(spec, cfg)
    chunk = _chunk_size(trials, dims, n, channels)
    for s in range(0, trials, chunk):
        B = min(trials, s + chunk) - s
        h, x = _draw(seed, t0 + s, B, dims, n_h, n, channels)
        ref = _reduce(_direct(h, x, dims, 1), -(dims + 1), "linear")           # fp64 reference
        if direct:
            prods = _direct(h, x, dims, 1 if cfg.precision == "fp64" else 0)
            outs = {v: _reduce(prods, -(dims + 1), v) for v in variants}
        else:
            if cfg.precision == "fp64":
                h, x = h.double(), x.double()
            zdt = np.float64 if cfg.precision == "fp64" else np.float32
            z = D.empty((B, channels) + (n,) * dims, zdt)
            hfn = _native.lib().wino_tile_hadamard2d if dims == 2 else _native.lib().wino_tile_hadamard1d
            ofn = _native.lib().wino_tile_output2d if dims == 2 else _native.lib().wino_tile_output1d
            _native.check(hfn(plan.handle, B, channels, D.ptr(h), D.ptr(x), D.ptr(z), D.stream_handle()),
                          "hadamard")
            outs = {}
            for v in variants:
                red = _reduce(z, -(dims + 1), v)
                out = D.empty((B,) + (n_o,) * dims, np.float32 if cfg.precision == "fp32" else np.float64)
                _native.check(ofn(plan.handle, B, D.ptr(red), D.ptr(out), D.stream_handle()), "output")
                outs[v] = out
        for v in variants:
            o = outs[v]
            _native.check(_native.lib().wino_trial_l1(B, n_out, 0 if o.dtype == D.torch.float32 else 1, D.ptr(o),
                                                      D.ptr(ref), D.ptr(per[v][s:]), D.stream_handle()), "trial_l1")
    reports = {}
    for v in variants:
        mean = D.torch.empty(1, dtype=D.torch.float64, device="cuda")
        _native.check(_native.lib().wino_mean_f64(trials, D.ptr(per[v]), D.ptr(mean), D.stream_handle()), "mean")
        total = float(mean.item())
        reports[v] = ErrorReport(
            descriptor=spec.descriptor(), dims=dims, channels=channels,
            config={"precision": cfg.precision, "dot_order": cfg.dot_order, "channel_sum": v},
            trials=trials, seed=seed, total_l1_mean=total, per_point_l1_mean=total / n_out,
            n_outputs=n_out, per_trial=per[v].cpu().numpy())
    return reports


def measure_error(spec, dims: int, cfg: ConvConfig = ConvConfig(), trials: int = 5000, seed: int = 0,
                  channels: int = 1, keep_trials: bool = True) -> ErrorReport:
    """Monte-Carlo L1 error of Toom-Cook (or direct) convolution against the fp64
    direct reference (harness.py:172-183)."""
    if trials < 1:
        raise ValueError("trials must be >= 1")
    D.require_cuda()
    rep = _measure_variants(spec, dims, cfg, trials, seed, channels, (cfg.channel_sum,))[cfg.channel_sum]
    if not keep_trials:
        rep.per_trial = None
    return rep


def measure_variants(spec, dims, cfg, trials, seed, channels, variants=("linear", "pairwise")):
    """Several channel-summation variants sharing draws, reference and transforms."""
    D.require_cuda()
    return _measure_variants(spec, dims, cfg, trials, seed, channels, tuple(variants))


@dataclass(frozen=True)
class RatioStats:
    ratio: float
    ci_low: float | None
    ci_high: float | None


def compare_reports(a: ErrorReport, b: ErrorReport, n_boot: int = 1000, boot_seed: int = 0) -> RatioStats:
    """Ratio of per-point means with a bootstrap CI (harness.py:193-207); host
    statistics over two already-measured per-trial vectors."""
    if a.dims != b.dims or a.n_outputs != b.n_outputs or a.trials != b.trials:
        raise ValueError("reports come from mismatched experiments")
    ratio = a.per_point_l1_mean / b.per_point_l1_mean
    if a.per_trial is None or b.per_trial is None:
        return RatioStats(ratio, None, None)
    rng = np.random.default_rng(boot_seed)
    idx = rng.integers(0, a.trials, size=(n_boot, a.trials))
    boots = a.per_trial[idx].mean(axis=1) / b.per_trial[idx].mean(axis=1)
    lo, hi = np.percentile(boots, [2.5, 97.5])
    return RatioStats(ratio, float(lo), float(hi))
