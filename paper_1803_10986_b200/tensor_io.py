"""Tensor files and the `convolve` adapter.

The reference's on-disk interchange for one convolution (toomcook/cli.py):
  * tensor files `load_tensor` / `save_tensor` (cli.py:57-98): JSON
    {"dims": d, "shape": [C, ...], "data": nested} or CSV with a header line
    "shape,C,n[,n]" and one line of flattened values per channel;
  * transform matrices as the transform JSON (transforms.py:126-169, here
    `read_transform_json` / `TransformSet.write_json`);
  * `cmd_convolve` (cli.py:162-176): kernel + input files -> conv_1d / conv_2d
    (or conv_direct with --direct) -> output tensor file.

Same formats and the same error behaviour (ValueError for a shape mismatch, a
missing CSV header, a wrong channel-row count, disagreeing kernel/input dims);
the convolution itself runs through libwino like every other entry point.

    python -m paper_1803_10986_b200 convolve --matrix t.json --kernel h.json --input x.json
"""
from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from .engine import ConvConfig, conv_1d, conv_2d, conv_direct
from .transforms import read_transform_json


def load_tensor(path: str) -> tuple[np.ndarray, int]:
    """Tensor file -> (channel-major float64 array, dims)  (reference cli.py:57-81)."""
    if path.endswith(".json"):
        with open(path, "r", encoding="utf-8") as fh:
            d = json.load(fh)
        arr = np.array(d["data"], dtype=np.float64)
        if list(arr.shape) != list(d["shape"]):
            raise ValueError(f"{path}: data does not match declared shape")
        return arr, int(d["dims"])
    with open(path, "r", encoding="utf-8") as fh:
        lines = [ln.strip() for ln in fh if ln.strip()]
    head = lines[0].split(",") if lines else [""]
    if head[0] != "shape":
        raise ValueError(f"{path}: missing 'shape' header")
    shape = tuple(int(v) for v in head[1:])
    rows = [np.array([float(v) for v in ln.split(",")]) for ln in lines[1:]]
    if len(rows) != shape[0]:
        raise ValueError(f"{path}: expected {shape[0]} channel rows")
    return np.stack(rows).reshape(shape), len(shape) - 1


def save_tensor(path: str | None, arr, dims: int, fmt: str) -> None:
    """(reference cli.py:84-98) values written as float64 reprs; None -> stdout."""
    arr = np.asarray(arr, dtype=np.float64)
    if arr.ndim == dims:
        arr = arr[np.newaxis]
    if fmt == "json":
        text = json.dumps({"dims": dims, "shape": list(arr.shape), "data": arr.tolist()}, indent=1) + "\n"
    else:
        lines = ["shape," + ",".join(str(s) for s in arr.shape)]
        lines += [",".join(repr(float(v)) for v in arr[c].ravel()) for c in range(arr.shape[0])]
        text = "\n".join(lines) + "\n"
    if path is None:
        sys.stdout.write(text)
    else:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)


def convolve(kernel_path: str, input_path: str, cfg: ConvConfig = ConvConfig(), matrix_path: str | None = None,
             direct: bool = False):
    """The reference's `cmd_convolve` computation (cli.py:162-176): returns (out, dims)."""
    h, hdims = load_tensor(kernel_path)
    x, xdims = load_tensor(input_path)
    if hdims != xdims:
        raise ValueError("kernel and input dims disagree")
    if direct:
        return conv_direct(h, x, hdims, precision=cfg.precision, channel_sum=cfg.channel_sum), hdims
    if matrix_path is None:
        raise ValueError("convolve needs --matrix (a transform JSON file) unless --direct")
    ts = read_transform_json(matrix_path)
    return (conv_1d if hdims == 1 else conv_2d)(ts, h, x, cfg), hdims


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1803_10986_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("convolve", help="run one convolution (reference: toomcook convolve)")
    p.add_argument("--matrix", help="transform JSON file")
    p.add_argument("--kernel", required=True, help="kernel tensor file")
    p.add_argument("--input", required=True, help="input tensor file")
    p.add_argument("--direct", action="store_true", help="direct convolution instead of Winograd")
    p.add_argument("--precision", choices=("fp32", "fp64", "mixed"), default="fp32")
    p.add_argument("--dot-order", choices=("linear", "huffman"), default="huffman")
    p.add_argument("--channel-sum", choices=("linear", "pairwise"), default="linear")
    p.add_argument("--format", choices=("json", "csv", "text"), default="text")
    p.add_argument("--out", default=None, help="output file (default stdout)")
    a = ap.parse_args(argv)
    cfg = ConvConfig(precision=a.precision, dot_order=a.dot_order, channel_sum=a.channel_sum)
    out, dims = convolve(a.kernel, a.input, cfg, a.matrix, a.direct)
    save_tensor(a.out, out, dims, "json" if a.format == "json" else "csv")
    return 0
