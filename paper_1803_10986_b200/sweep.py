"""The measured columns of the reference's error tables.

The reference regenerates Tables 2-8 with `reproduce_table` (harness.py:636-660):
every measured cell is one `measure_error` / two-variant `_measure_variants`
call on a curated transform set (harness.py:453-494), memoised across tables.
`table_measurements` issues exactly that set of measurements -- same keys,
same curated sets, same trials and seed, same linear/pairwise pairing -- on
the GPU (harness.measure_error / measure_variants, Philox draws, fp64
reference and Winograd path all on device), and returns the per-point L1
means.  The table layout and the published comparison columns stay with the
reference (out of scope).

Which measurements (harness.py:525-611):
  * Tables 2/3: family fp32 / mixed, dims 1 and 2, n in SIZES plus direct
    (n = 0), one channel, linear sum (Table 3's ratios also use the fp32 ones);
  * Tables 4-7: family x dims, output sizes 1..7 (n = 0 or out + 2): one
    channel, and 32 / 64 channels with linear and pairwise sums;
  * Table 8 reuses the 32 / 64-channel pairs of Tables 4-7.
"""
from __future__ import annotations

from .engine import ConvConfig
from .harness import DirectSpec, measure_error, measure_variants
from .pointsets import KERNEL_SIZE, SIZES, curated_transform


def _cfg(family: str, channel_sum: str = "linear") -> ConvConfig:
    return ConvConfig("fp32" if family == "fp32" else "mixed", "huffman", channel_sum)


def key(family: str, dims: int, n: int, channels: int, channel_sum: str) -> str:
    return f"{family}/{dims}d/n{n}/c{channels}/{channel_sum}"


def table_keys(tables=("2", "3", "4", "5", "6", "7", "8"), sizes=SIZES):
    """(family, dims, n, channels, variants) measurement groups, in a fixed order."""
    groups = []
    tables = set(str(t) for t in tables)
    for family, t in (("fp32", "2"), ("mixed", "3")):
        if t in tables or (family == "fp32" and "3" in tables):
            for dims in (1, 2):
                for n in (0,) + tuple(sizes):
                    groups.append((family, dims, n, 1, ("linear",)))
    chan = {("fp32", 1): "4", ("fp32", 2): "5", ("mixed", 1): "6", ("mixed", 2): "7"}
    for (family, dims), t in chan.items():
        if t in tables or "8" in tables:
            for out in range(1, 8):
                n = 0 if out == 1 else out + 2
                groups.append((family, dims, n, 1, ("linear",)))
                for channels in (32, 64):
                    groups.append((family, dims, n, channels, ("linear", "pairwise")))
    seen, out = set(), []
    for g in groups:
        if g not in seen:
            seen.add(g)
            out.append(g)
    return out


def table_measurements(trials: int = 5000, seed: int = 0, tables=("2", "3", "4", "5", "6", "7", "8"),
                       sizes=SIZES) -> dict:
    """{key: per_point_l1_mean} for every measured cell of the chosen tables."""
    res = {}
    for family, dims, n, channels, variants in table_keys(tables, sizes):
        spec = DirectSpec(KERNEL_SIZE, 1) if n == 0 else curated_transform(n, dims, family)
        if len(variants) == 1:
            rep = measure_error(spec, dims, _cfg(family, variants[0]), trials, seed, channels, keep_trials=False)
            res[key(family, dims, n, channels, variants[0])] = rep.per_point_l1_mean
        else:
            reps = measure_variants(spec, dims, _cfg(family), trials, seed, channels, variants)
            for v in variants:
                res[key(family, dims, n, channels, v)] = reps[v].per_point_l1_mean
    return res
