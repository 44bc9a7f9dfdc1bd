"""Benchmark of the Winograd hot path (BASELINE.json metric:
"Winograd conv direct-equiv TFLOP/s (1/2/4/8 GPU); rel. L1 error vs fp64 direct").

Default workload = BASELINE.json configs[4], the config the metric's 1/2/4/8-GPU
figure is quoted on and that fits one B200: the VGG-16 conv stack (13 3x3 layers,
ReLU, 2x2 max-pools after layers 2/4/7/10), every layer through Winograd
F(6x6,3x3) with the P8 points {0,-1,1,1/2,-1/2,2,-2,inf}, fp32, Huffman-ordered
transforms, pairwise channel sums, exact contraction; global batch 256 of
224x224x3 synthetic U[-1,1] images, He-normal filters (seeded Philox).
A step = one 13-layer forward (38 libwino kernels: layer 1 runs K1+K2 and a fused
K3+K4+ReLU kernel, the other layers K1+K2, K3, K4+ReLU(+pool); input resident in HBM).
Multi-GPU: one process per GPU (`--gpus N` re-execs under torch.distributed.run
when no torchrun environment is set), the global batch sharded by images
(strong scaling); NCCL only reduces timings.  `--impl reference` times the CPU
port of the reference's arithmetic (oracle/) on the host cores on the
BASELINE.md 2-image slice.  `--config cfg1|cfg2|...` selects the single-layer
configs (configs[0..3]) as extra lines.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Winograd conv direct-equiv TFLOP/s"

CONFIGS = {
    # name: (r, m, points, N, C, K, H, pad, x_dist, w_init, precision, dot_order, channel_sum)
    "cfg2": (3, 2, "0,1,-1,inf", 32, 128, 128, 28, 1, "uniform", "he", "fp32", "huffman", "linear"),
    "cfg1": (3, 4, "0,1,-1,1/2,-1/2,inf", 8, 64, 64, 56, 1, "uniform", "uniform", "fp32", "huffman", "linear"),
    "cfg3_m6": (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 64, 256, 256, 28, 1, "uniform", "he", "fp32", "huffman",
                "linear"),
    "cfg3_m6_mixed_pw": (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 64, 256, 256, 28, 1, "uniform", "he", "mixed",
                         "huffman", "pairwise"),
    "cfg4_m4": (5, 4, "0,-1,1,1/2,-1/2,2,-2,inf", 32, 512, 512, 14, 2, "uniform01", "he", "fp32", "huffman",
                "pairwise"),
    "vgg_l5": (3, 6, "0,-1,1,1/2,-1/2,2,-2,inf", 256, 128, 256, 56, 1, "uniform", "he", "fp32", "huffman",
               "pairwise"),
}


def synth(shape, seed, idx, dist):
    g = np.random.Generator(np.random.Philox(key=np.array([seed, idx], dtype=np.uint64)))
    if dist == "uniform":
        return g.random(shape, dtype=np.float32) * np.float32(2) - np.float32(1)
    if dist == "uniform01":
        return g.random(shape, dtype=np.float32)
    return g.standard_normal(shape, dtype=np.float32)


def make_inputs(cfg, rank, seed=2024):
    r, m, pts, N, C, K, H, pad, xd, wi = cfg[:10]
    x = np.stack([synth((C, H, H), seed, rank * N + i, xd) for i in range(N)])
    if wi == "he":
        w = synth((K, C, r, r), seed, 10_000_000, "normal") * np.float32(np.sqrt(2.0 / (r * r * C)))
    else:
        w = synth((K, C, r, r), seed, 10_000_000, "uniform")
    return np.ascontiguousarray(x), np.ascontiguousarray(w.astype(np.float32))


def direct_flops(cfg):
    r, m, pts, N, C, K, H, pad = cfg[:8]
    Ho = H + 2 * pad - r + 1
    return 2 * N * K * C * Ho * Ho * r * r


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------- CPU side
_CPU = {}


def _cpu_worker(span):
    from oracle import wino_oracle as O
    i0, i1 = span
    c = _CPU
    return O.layer_conv2d(c["trip"], c["x"][i0:i1], c["w"], c["pad"], c["prec"], c["order"], c["cs"])


def cpu_layer_time(cfg, x, w, procs):
    """Time the oracle port (the reference's arithmetic on numpy) over images
    x with `procs` worker processes; returns seconds."""
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    from oracle import wino_oracle as O
    r, m, pts, N, C, K, H, pad = cfg[:8]
    _CPU.update(trip=O.Triple.from_points(r, m, pts), x=x, w=w, pad=pad, prec=cfg[10], order=cfg[11], cs=cfg[12])
    n = x.shape[0]
    spans = [(i * n // procs, (i + 1) * n // procs) for i in range(procs)]
    spans = [s for s in spans if s[1] > s[0]]
    ctx = mp.get_context("fork")
    with ProcessPoolExecutor(max_workers=len(spans), mp_context=ctx) as ex:
        list(ex.map(_cpu_worker, [(0, 1)] * len(spans)))  # warm the workers
        t0 = time.perf_counter()
        list(ex.map(_cpu_worker, spans))
        return time.perf_counter() - t0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    """CPU model string of the host (state the core count and the CPU model)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.lower().startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or platform.machine()


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    x, w = make_inputs(cfg, 0)
    procs = min(host_cores(), x.shape[0])
    times = []
    for i in range(args.warmup + args.steps):
        t = cpu_layer_time(cfg, x, w, procs)
        if i >= args.warmup:
            times.append(t)
    ms = 1e3 * float(np.mean(times))
    val = direct_flops(cfg) / (ms * 1e-3) / 1e12
    line = {"metric": METRIC, "value": val, "unit": "TFLOP/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if cfg[10] == "fp32" else "f32/f64",
            "data": "synthetic (seeded Philox U[-1,1] inputs, He-normal filters)",
            "config": config_dict(args, cfg),
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": procs, "cpu_model": cpu_model(), "kind": "port",
                             "sample": f"full batch of {x.shape[0]} images per step, oracle/wino_oracle.py "
                                       f"layer_conv2d (numpy restatement of the reference) over {procs} processes"},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def contraction_note(mode):
    """What a non-exact contraction mode means for parity (stated on every such line)."""
    if mode == "exact":
        return "reference arithmetic: one rounded product and one rounded sum per channel term, bit-identical"
    if mode == "ffma":
        return ("NOT reference arithmetic: fused multiply-add in the channel sum; against the exact output it differs "
                "by 9-127 ulp-scaled units at p99 depending on the config (tests/test_gpu_ffma.py), above "
                "north_star's 4-ulp example; error_vs_fp64 is this mode's own")
    return ("NOT reference arithmetic: U and V rounded to 16 bits, tensor-core FP32 accumulation; error_vs_fp64 is "
            "this mode's own (tc_bf16 at F(6,3): rel. L1 3.9e-2, not a usable Winograd result)")


def config_dict(args, cfg, world=1):
    r, m, pts, N, C, K, H, pad, xd, wi, prec, order, cs = cfg
    return {"workload": args.config, "winograd": f"F({m}x{m},{r}x{r})", "points": pts, "N_per_gpu": N,
            "global_batch": N * world, "C": C, "K": K, "H": H, "W": H, "pad": pad, "precision": prec,
            "dot_order": order, "channel_sum": cs, "contraction": args.contraction,
            "contraction_note": contraction_note(args.contraction), "x_dist": xd, "w_init": wi, "l2": "flushed between timed steps: 256 MiB write, then 256 MiB read of a clean buffer "
                  "(no step data and no dirty lines left in L2)",
            "parallelism": f"dp{world} (independent batches per GPU)"}


# --------------------------------------------------------------------- GPU side
def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1803_10986_b200 as W
    from paper_1803_10986_b200 import _native

    r, m, pts, N, C, K, H, pad, xd, wi, prec, order, cs = cfg
    ts = W.build_transforms(r, m, W.parse_points(pts))
    wcfg = W.ConvConfig(prec, order, cs)
    op = W.layer_op(ts, wcfg, N, C, H, H, K, pad, args.contraction)
    L = op.layout
    x_np, w_np = make_inputs(cfg, rank)
    x = torch.from_numpy(x_np).cuda()
    w = torch.from_numpy(w_np).cuda()
    y = torch.empty(op.out_shape, dtype=torch.float32 if prec == "fp32" else torch.float64, device="cuda")
    uvdt = torch.float64 if prec == "fp64" else torch.float32
    U = torch.empty((L.P, L.Cp, L.Kp), dtype=uvdt, device="cuda")
    V = torch.empty((L.P, L.Cp, L.Tp), dtype=uvdt, device="cuda")
    fused = args.contraction.startswith("tcf_")  # K3t + K4 in one kernel (wino_tcf), no M
    M = torch.empty((1,) if fused else (L.P, L.Kp, L.Tp), dtype=uvdt, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")

    def flush_l2():
        # evict L2: write 256 MiB, then read a clean 256 MiB buffer so the write-back
        # of those dirty lines happens here, not inside the next timed step
        flush.zero_()
        clean.sum()

    lib = _native.lib()
    shp = op.shape
    import ctypes
    sref = ctypes.byref(shp)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    def step(ev=None):
        sh = torch.cuda.current_stream().cuda_stream  # the capture stream inside torch.cuda.graph
        if ev is not None:
            ev[0].record(stream)
        # K1 + K2 in one launch (wino_transforms); the second event pair is empty
        _native.check(lib.wino_transforms(op.plan.handle, sref, _native.as_ptr(x), _native.as_ptr(w),
                                          _native.as_ptr(U), _native.as_ptr(V), sh))
        if ev is not None:
            ev[1].record(stream)
            ev[2].record(stream)
        if fused:
            _native.check(lib.wino_contract_output(op.plan.handle, sref, _native.as_ptr(U), _native.as_ptr(V),
                                                   _native.as_ptr(y), sh))
            if ev is not None:
                ev[3].record(stream)
                ev[4].record(stream)
            return
        _native.check(lib.wino_contract(op.plan.handle, sref, _native.as_ptr(U), _native.as_ptr(V),
                                        _native.as_ptr(M), sh))
        if ev is not None:
            ev[3].record(stream)
        _native.check(lib.wino_output_transform(op.plan.handle, sref, _native.as_ptr(M), _native.as_ptr(y), sh))
        if ev is not None:
            ev[4].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if args.ncu:
        # profiling mode (ncu launch lists / captures): the K steps eagerly, nothing else
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        return

    # The step as a CUDA graph (4 libwino kernel nodes): no CPU launch gaps.
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()

    e_start = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        # keep the GPU busy with the same workload for a while so the clock
        # sampler sees the load the timed region runs under
        t_end = time.perf_counter() + args.soak
        while time.perf_counter() < t_end:
            for _ in range(50):
                graph.replay()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        n0 = _native.launch_count()
        for i in range(args.steps):
            flush_l2()  # evict L2 (outside the timed interval of the step)
            e_start[i].record(stream)
            graph.replay()
            e_end[i].record(stream)
        # instrumented steps: the same four kernels launched eagerly with an
        # event between stages -> per-kernel durations for the roofline
        for i in range(args.steps):
            flush_l2()
            step(evs[i])
        torch.cuda.synchronize()
        n_launch = (2 if fused else 3) * args.steps + (_native.launch_count() - n0)
    if world > 1:
        dist.barrier()
    stage = np.array([[evs[i][j].elapsed_time(evs[i][j + 1]) for j in range(4)] for i in range(args.steps)])
    ms_step = float(np.mean([e_start[i].elapsed_time(e_end[i]) for i in range(args.steps)]))
    ms_stage = stage.mean(axis=0)
    if world > 1:
        t = torch.tensor([ms_step], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    value = direct_flops(cfg) * world / (ms_step * 1e-3) / 1e12

    # ---- end to end through the public API: pinned host x, w in -> pinned host y out,
    # H2D / compute / D2H overlapped over image chunks (W.HostPipeline)
    xh = torch.from_numpy(x_np).pin_memory()
    wh = torch.from_numpy(w_np).pin_memory()
    yh = torch.empty(op.out_shape, dtype=y.dtype).pin_memory()
    chunks = [int(v) for v in args.e2e_chunks.split(",")] if "," in args.e2e_chunks else int(args.e2e_chunks)
    pipe = W.HostPipeline(ts, wcfg, N, C, H, H, K, pad, chunks=chunks, contraction=args.contraction)

    for _ in range(3):
        pipe(xh, wh, yh)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_ms = []
    for _ in range(args.steps):
        flush_l2()
        e0.record(stream)
        pipe(xh, wh, yh)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    # median step: a host-side hiccup (page-cache / driver work on the CPU that issues
    # the copies) can stretch single steps; the mean and every step are reported too
    e2e_mean = float(np.mean(e2e_ms))
    e2e_t = float(np.median(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_t], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_val = direct_flops(cfg) * world / (e2e_t * 1e-3) / 1e12
    y_e2e = yh.clone()

    # ---- error vs fp64 direct (device oracle kernel), per-image partials gathered in image order
    y_ref = op(x, w)
    e2e_same = bool(torch.equal(y_ref.cpu(), y_e2e))
    y64 = W.direct_layer_f64(x, w, pad)
    st = W.layer_error_stats(y_ref, y64)
    if world > 1:
        allst = [torch.empty_like(st) for _ in range(world)]
        dist.all_gather(allst, st)
        st = torch.cat(allst)
    st = st.cpu().numpy()
    err = {"rel_l1": float(st[:, 0].sum() / st[:, 1].sum()), "per_point_l1": float(st[:, 0].sum() / st[:, 2].sum()),
           "max_abs": float(st[:, 3].max()), "images": int(st.shape[0]), "reference": "fp64 direct (device kernel)"}

    # ---- roofline of the dominant kernel (the contraction: FP32 CUDA-core bound)
    peak = measure_peaks(lib, _native, torch)
    flops_c = 2 * L.P * L.T * C * K
    ach = flops_c / (ms_stage[2] * 1e-3) / 1e12
    exact = args.contraction == "exact"
    mp = measured_peaks()
    hbm = mp["hbm_gbs"]
    if fused:
        # wino_tcf: V and U read once (16-bit), y written once; tensor work is ~2 us of it
        fb = 2 * L.P * L.T * C + 2 * L.P * C * K + (4 if prec == "fp32" else 8) * N * K * L.Ho * L.Wo
        gbs = fb / (ms_stage[2] * 1e-3) / 1e9
        roof = {"kernel": "wino_tcf (tcgen05 contraction + output transform, one kernel)", "bound": "hbm",
                "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                "traffic": traffic_of("wino_tcf", args.config, args.contraction),
                "peak_source": mp["source"] + " hbm copy bandwidth", "bytes_per_launch": fb,
                "tensor_tflops": ach, "tensor_frac": ach / mp["bf16_tflops"]}
    elif args.contraction.startswith("tc_"):
        # 2 P T C K flop against 2 P C (T + K) + 4 P K T bytes (16-bit operands read, fp32 M written):
        # <= 256 flop per byte at C = 512, so the unfused tensor-core contraction is bound by moving M
        # (through L2 / HBM), not by the tensor pipe; the tensor-peak fraction is reported beside it
        pk = mp["bf16_tflops"]
        cb = 2 * L.P * C * (L.T + K) + 4 * L.P * K * L.T
        gbs = cb / (ms_stage[2] * 1e-3) / 1e9
        roof = {"kernel": "tc_contract_kernel (tcgen05.mma kind::f16)", "bound": "hbm", "achieved": gbs,
                "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "traffic": None, "bytes_per_launch": cb,
                "peak_source": mp["source"] + " hbm copy bandwidth",
                "bound_note": "algorithmic bytes (U16 + V16 read, fp32 M written); a single small layer's M "
                              "partly stays in the 126 MB L2",
                "tensor_tflops": ach, "frac_of_tensor_peak": ach / pk}
    else:
        pk = max(peak["ffma_tflops"], peak.get("ffma2_tflops", 0.0))  # FP32 pipe peak (scalar or packed FFMA)
        # exact modes: every MAC is a separately rounded multiply and add (scalar
        # FMUL+FADD or packed FFMA2(a, b, -0)+FADD2): the better of the two probes
        xceil = max(peak["fmul_fadd_tflops"], peak.get("fmul_fadd_packed_tflops", 0.0))
        roof = {"kernel": "wino_contract", "bound": "fp32", "bound_note": "FP32 CUDA-core pipe (neither HBM nor tensor cores): the reference rounds every product and sum separately, which tensor-core accumulation cannot reproduce", "achieved": ach, "peak": pk, "unit": "TFLOP/s",
                "frac": ach / pk, "traffic": traffic_of("wino_contract", args.config, args.contraction),
                "peak_source": "measured in this run: libwino wino_peak_probe, max of FFMA and packed FFMA2 (8 chains x 148*8 CTAs); "
                               "MEASURED_PEAKS.json has no FP32 figure",
                "exact_ceiling_tflops": xceil if exact else None,
                "frac_of_exact_ceiling": ach / xceil if exact else None,
                "exact_ceiling_reg_tflops": peak["fmul_fadd_reg_tflops"] if exact else None,
                "frac_of_exact_ceiling_reg": ach / peak["fmul_fadd_reg_tflops"] if exact else None}
    roof.update({"flops_per_launch": flops_c, "share_of_step": float(ms_stage[2] / ms_stage.sum())})
    eb = L.elem_bytes_uv
    mb = 4 if args.contraction.startswith("tc_") else eb  # tensor-core modes: 16-bit U / V (eb = 2), fp32 M
    stage_bytes = [4 * K * C * r * r + eb * L.P * C * K + 4 * N * C * H * H + eb * L.P * L.T * C,
                   None,
                   None,
                   mb * L.P * L.T * K + (4 if prec == "fp32" else 8) * N * K * L.Ho * L.Wo]
    stages = {}
    if fused:
        stage_bytes[2] = roof["bytes_per_launch"]
    for j, name in enumerate(["transforms (K1 input + K2 filter, one launch)", None,
                              "contract + output transform (wino_tcf)" if fused else "contract",
                              None if fused else "output_transform"]):
        if name is None:
            continue
        d = {"ms": float(ms_stage[j])}
        if stage_bytes[j] is not None:
            d["gbs"] = stage_bytes[j] / (ms_stage[j] * 1e-3) / 1e9
            d["frac_hbm"] = d["gbs"] / hbm
        else:
            d["tflops"] = ach
        stages[name] = d

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32" if prec == "fp32" else "f32/f64",
                "data": "synthetic (seeded Philox U[-1,1] inputs, He-normal filters)",
                "config": config_dict(args, cfg, world), "roofline": roof, "stages": stages,
                "error_vs_fp64": err,
                "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": x_np.nbytes + w_np.nbytes,
                        "d2h_bytes_per_step": yh.numel() * yh.element_size(), "ms_per_step": e2e_t,
                        "timing": "median of the K timed steps (CUDA events on the issuing stream)",
                        "ms_per_step_mean": e2e_mean, "ms_steps": [round(v, 4) for v in e2e_ms],
                        "api": f"HostPipeline(chunks={args.e2e_chunks}: H2D | K1-K3-K4 | D2H overlapped on "
                               "3 streams, captured once into a CUDA graph and replayed)",
                        "bitwise_equal_to_device_path": e2e_same},
                "timing": "value/ms_per_step: CUDA-graph replay of the 4-kernel step, events around each "
                          "step, L2 flushed between steps; stages: eager launches with an event between stages",
                "gpu_launches": int(n_launch), "clocks": clk.summary(), "peaks": peak}
        if world == 1 and not args.no_cpu:
            xs = x_np[: args.cpu_images]
            procs = min(host_cores(), xs.shape[0])
            t = cpu_layer_time(cfg, xs, w_np, procs)
            fl = direct_flops(cfg) * xs.shape[0] / N
            line["cpu_baseline"] = {"value": fl / t / 1e12, "unit": "TFLOP/s", "cores": procs, "cpu_model": cpu_model(), "kind": "port",
                                    "sample": f"{xs.shape[0]} of {N} images of the same layer, oracle/wino_oracle.py "
                                              f"layer_conv2d over {procs} processes, {t:.2f} s"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


VGG_POINTS = "0,-1,1,1/2,-1/2,2,-2,inf"


def vgg_inputs(a, b, seed=2024):
    """Synthetic U[-1,1] 3x224x224 images a..b-1, keyed Philox(seed, global image index)."""
    return np.ascontiguousarray(np.stack([synth((3, 224, 224), seed, i, "uniform") for i in range(a, b)]))


def vgg_config(args, n_per_gpu, world):
    return {"workload": "vgg16", "model": "VGG-16 conv stack (13 conv layers, ReLU, 4 max-pools; no FC head)",
            "winograd": "F(6x6,3x3)", "points": VGG_POINTS, "global_batch": args.vgg_batch,
            "batch_per_gpu": n_per_gpu, "image": [3, 224, 224], "precision": "fp32", "dot_order": "huffman",
            "channel_sum": "pairwise", "contraction": args.contraction,
            "contraction_note": contraction_note(args.contraction) + (
                "; layer 1 (C = 3) runs the exact fp32 path (fused K3 + K4 + ReLU): a 3-channel contraction has "
                "nothing for a tensor core" if args.contraction.startswith("tc_") else ""),
            "layers": 13, "pools_after": [2, 4, 7, 10],
            "l2": "no flush needed: inputs and activations >> 126 MB L2 (layer-1 x 154 MB, M 6 GB)",
            "parallelism": f"dp{world} (global batch sharded by images)"}


def vgg_cpu_forward(x, weights, procs):
    """The oracle port of the stack (reference arithmetic, oracle/stack_pool.py) on
    images x over `procs` processes: (seconds, conv outputs, final activation)."""
    from oracle import wino_oracle as O
    from oracle.stack_pool import OraclePool
    from paper_1803_10986_b200.stack import VGG16
    trip = O.Triple.from_points(3, 6, VGG_POINTS)
    with OraclePool(trip, weights, x.shape[0] * 64 * 226 * 226, procs=procs) as pool:
        if procs > 1:
            pool.layer(12, np.zeros((1, 512, 14, 14), np.float32))  # fork + warm the workers
        t0 = time.perf_counter()
        outs, act = pool.stack_forward(x, VGG16)
        return time.perf_counter() - t0, outs, act


def vgg_direct_flops(n):
    from paper_1803_10986_b200.stack import VGG16
    h, tot = 224, 0
    for C, K, pool in VGG16:
        tot += 2 * n * K * C * h * h * 9
        if pool:
            h //= 2
    return tot


def run_reference_vgg(args):
    """--impl reference for vgg16: the reference's arithmetic (oracle port) on the
    host cores; each step = the BASELINE.md 2-image slice through all 13 layers."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from paper_1803_10986_b200.stack import VGG16, he_normal_weights
    x = vgg_inputs(0, args.cpu_vgg_images)
    ws = he_normal_weights(VGG16, 3)
    procs = host_cores()
    from oracle import wino_oracle as O
    from oracle.stack_pool import OraclePool
    trip = O.Triple.from_points(3, 6, VGG_POINTS)
    times = []
    with OraclePool(trip, ws, x.shape[0] * 64 * 226 * 226, procs=procs) as pool:
        pool.layer(12, np.zeros((1, 512, 14, 14), np.float32))
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.stack_forward(x, VGG16, keep=False)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    val = vgg_direct_flops(x.shape[0]) / (ms * 1e-3) / 1e12
    sample = (f"{x.shape[0]} of {args.vgg_batch} images per step through all 13 layers (BASELINE.md 2: 2-image "
              f"slice), oracle/stack_pool.py (oracle/wino_oracle.py layer_conv2d = the reference's per-(filter, tile) "
              f"arithmetic) over {procs} processes")
    line = {"metric": METRIC, "value": val, "unit": "TFLOP/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Philox U[-1,1] 224x224x3 images, He-normal filters)",
            "config": vgg_config(args, args.vgg_batch, 1),
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": procs, "cpu_model": cpu_model(), "kind": "port", "sample": sample},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_vgg(args):
    """BASELINE config 5: VGG-16 conv stack, F(6x6,3x3) P8, pairwise, fp32, global batch
    sharded across ranks (strong scaling); step = one 13-layer forward."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1803_10986_b200 as W
    from paper_1803_10986_b200 import _native
    from paper_1803_10986_b200.distributed import shard_range
    from paper_1803_10986_b200.stack import VGG16, ConvStack, StackPipeline, he_normal_weights

    ts = W.build_transforms(3, 6, W.parse_points(VGG_POINTS))
    wcfg = W.ConvConfig("fp32", "huffman", "pairwise")
    a, b = shard_range(args.vgg_batch, rank, world)
    n = b - a
    st = ConvStack(ts, wcfg, VGG16, n, 224, contraction=args.contraction)
    ws_np = he_normal_weights(VGG16, 3)
    st.set_weights(ws_np)
    x_np = vgg_inputs(a, b)
    x = torch.from_numpy(x_np).cuda()
    for _ in range(max(3, args.warmup)):
        st.forward(x)
    torch.cuda.synchronize()
    if args.ncu:
        for _ in range(args.steps):
            st.forward(x)
        torch.cuda.synchronize()
        return
    if args.traffic:
        # DRAM-traffic capture mode (run under ncu --cache-control none, tools/traffic.py):
        # one forward with an L2 eviction after every libwino kernel -- a read of a clean
        # 256 MiB buffer, whose DRAM writes are exactly the previous kernel's dirty lines
        # still in L2 (the deferred write-back a per-kernel capture would miss)
        clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
        clean.sum()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()  # ncu --profile-from-start off: only this forward is captured
        cur = x
        for i in range(len(st.ops)):
            cur = st.layer_forward(i, cur, after_kernel=lambda: clean.sum())
        clean.sum()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        st.forward(x)
    graph.replay()
    torch.cuda.synchronize()
    es = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stream = torch.cuda.current_stream()
    with ClockSampler(local) as clk:
        t_end = time.perf_counter() + args.soak  # untimed load so the sampler sees the clocks under load
        while time.perf_counter() < t_end:
            graph.replay()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for e0, e1 in es:  # inputs and activations >> L2: no flush needed
            e0.record(stream)
            graph.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    ms_steps = [e0.elapsed_time(e1) for e0, e1 in es]
    ms = float(np.mean(ms_steps))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # whole-job direct-eq flops: every rank's shard (equal or +-1 image)
    gflops = torch.tensor([float(st.direct_flops)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(gflops)
    value = float(gflops.item()) / (ms * 1e-3) / 1e12
    y_dev = st.act[-1].clone()

    # ---- per-layer stage times from an instrumented eager forward (events between stages)
    per_layer, c_ms, c_flops, other_ms, fused_ms, n_contract, c_bytes = [], 0.0, 0, 0.0, 0.0, 0, 0
    mp_ = measured_peaks()
    hbm = mp_["hbm_gbs"]
    cur = x
    if st.fused_act:
        for i, op_ in enumerate(st.ops):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            cur = st.layer_forward(i, cur, events=ev)
            torch.cuda.synchronize()
            C, K, h, w_, pool = st.shapes[i]
            L = op_.layout
            t_x, t_c, t_o = (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]))
            P, T = L.P, L.T
            fused_prev, fused_next = i > 0 and st.fuse_next[i - 1], st.fuse_next[i]
            # x read, V + U written (K2 only when the previous layer's K4 already wrote this layer's V);
            # the tensor-core modes store U and V as 16-bit operands
            uvb = 2 if op_.tensor_core else 4
            b_x = (0 if fused_prev else 4 * n * C * h * w_ + uvb * P * C * T) + 4 * K * C * 9 + uvb * P * C * K
            out_el = n * K * (L.Ho // 2) * (L.Wo // 2) if pool else n * K * L.Ho * L.Wo
            b_o = 4 * P * K * T + 4 * out_el                                             # M read, act written
            if fused_next:  # K4 + act + K1 of the next layer: M read, the next layer's V written
                L2 = st.ops[i + 1].layout
                b_o = 4 * P * K * T + 4 * L2.P * K * L2.T
            if st.smallc[i]:
                # K3 + K4 + activation in one kernel (small C): M never exists; bytes = V read + act written
                b_f = 4 * P * C * T + 4 * P * C * K + 4 * out_el
                per_layer.append({"layer": i + 1, "C": C, "K": K, "H": h, "tile_bm_bn": [L.bm, L.bn],
                                  "transforms_ms": t_x, "transforms_frac_hbm": b_x / (t_x * 1e-3) / 1e9 / hbm,
                                  "fused_contract_output_act_ms": t_c,
                                  "fused_frac_hbm": b_f / (t_c * 1e-3) / 1e9 / hbm,
                                  "contract_ms": 0.0, "output_act_ms": 0.0})
                other_ms += t_x + t_c
                fused_ms += t_c
                continue
            per_layer.append({"layer": i + 1, "C": C, "K": K, "H": h, "tile_bm_bn": [L.bm, L.bn],
                              "transforms_ms": t_x, "transforms_frac_hbm": b_x / (t_x * 1e-3) / 1e9 / hbm,
                              "contract_ms": t_c, "contract_tflops": op_.contraction_flops / (t_c * 1e-3) / 1e12,
                              "output_act_ms": t_o, "output_act_frac_hbm": b_o / (t_o * 1e-3) / 1e9 / hbm,
                              "v_written_by_previous_k4": bool(fused_prev), "k4_fused_with_next_k1": bool(fused_next)})
            if op_.tensor_core:  # U16 + V16 read, fp32 M written: the HBM bytes that bound K3t at alpha = 8
                b_c = 2 * P * C * (T + K) + 4 * P * K * T
                per_layer[-1]["contract_frac_hbm"] = b_c / (t_c * 1e-3) / 1e9 / hbm
                c_bytes += b_c
            c_ms += t_c
            other_ms += t_x + t_o
            c_flops += op_.contraction_flops
            n_contract += 1
    else:
        # tensor-core modes: K1+K2, K3t, K4, then ReLU / pool as its own kernel
        import ctypes
        lib_, D_ = _native.lib(), __import__("paper_1803_10986_b200.device", fromlist=["x"])
        sh_ = D_.stream_handle()
        for i, op_ in enumerate(st.ops):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            C, K, h, w_, pool = st.shapes[i]
            L = op_.layout
            U_, V_, M_ = st._uvm(L)
            sref = ctypes.byref(op_.shape)
            y_ = st.conv_out[i]
            ev[0].record()
            _native.check(lib_.wino_transforms(op_.plan.handle, sref, D_.ptr(cur), D_.ptr(st.weights[i]),
                                               ctypes.c_void_p(U_), ctypes.c_void_p(V_), sh_))
            ev[1].record()
            _native.check(lib_.wino_contract(op_.plan.handle, sref, ctypes.c_void_p(U_), ctypes.c_void_p(V_),
                                             ctypes.c_void_p(M_), sh_))
            ev[2].record()
            _native.check(lib_.wino_output_transform(op_.plan.handle, sref, ctypes.c_void_p(M_), D_.ptr(y_), sh_))
            _native.check(lib_.wino_relu_pool(0, op_.N * K, L.Ho, L.Wo, 1 if pool else 0, D_.ptr(y_),
                                              D_.ptr(st.act[i]), sh_))
            ev[3].record()
            torch.cuda.synchronize()
            t_x, t_c, t_o = (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]))
            per_layer.append({"layer": i + 1, "C": C, "K": K, "H": h, "transforms_ms": t_x, "contract_ms": t_c,
                              "contract_tflops": op_.contraction_flops / (t_c * 1e-3) / 1e12,
                              "output_act_ms": t_o})
            c_ms += t_c
            other_ms += t_x + t_o
            c_flops += op_.contraction_flops
            n_contract += 1
            cur = st.act[i]
    peak = measure_peaks(_native.lib(), _native, torch)
    ach = c_flops / (c_ms * 1e-3) / 1e12 if c_ms else 0.0

    # ---- end to end through the public API: pinned host images in -> pinned host final activation out
    xh = torch.from_numpy(x_np).pin_memory()
    vchunks = [int(v) for v in args.vgg_chunks.split(",")] if "," in str(args.vgg_chunks) else int(args.vgg_chunks)
    pipe = StackPipeline(ts, wcfg, VGG16, n, 224, chunks=vchunks, contraction=args.contraction)
    pipe.set_weights(ws_np)
    yh = torch.empty(pipe.out_shape, dtype=torch.float32).pin_memory()
    for _ in range(2):
        pipe(xh, yh)
    torch.cuda.synchronize()
    e2e_ms = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pipe(xh, yh)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    e2e_t = float(np.median(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_t], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_val = float(gflops.item()) / (e2e_t * 1e-3) / 1e12
    e2e_same = bool(torch.equal(yh, y_dev.cpu()))
    del pipe

    # ---- per-layer isolated error vs fp64 direct (device kernel), unfused forward keeps y per layer
    errs = st.layer_errors(x, images=args.err_images) if not args.no_err else None
    conv_first = [st.conv_out[i][: args.cpu_vgg_images].cpu().numpy() for i in range(len(st.ops))] \
        if (rank == 0 and world == 1 and not args.no_cpu) else None
    st._conv_out = None
    if rank == 0:
        roof = vgg_roof(args, ach, peak, c_ms / (c_ms + other_ms) if c_ms else None,
                        c_bytes / (c_ms * 1e-3) / 1e9 if (c_bytes and c_ms) else None)
        roof.update({"flops_per_forward": c_flops, "launches": n_contract,
                     "kernel": roof["kernel"].replace("13 layers", f"{n_contract} layers"),
                     "achieved_note": f"sum of the {n_contract} contraction launches' algorithmic flops (2 P T C K "
                                      "each) / sum of their CUDA-event durations (instrumented eager forward)"
                                      + ("; layer 1 (C = 3) runs K3 + K4 + ReLU as one kernel and is not counted here"
                                         if fused_ms else "")})
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded Philox U[-1,1] 224x224x3 images, He-normal filters)",
                "config": vgg_config(args, n, world), "roofline": roof,
                "stages": {"contract_ms": c_ms, "transforms_ms": sum(p["transforms_ms"] for p in per_layer),
                           "output_act_ms": sum(p["output_act_ms"] for p in per_layer),
                           "fused_small_c_ms": fused_ms},
                "per_layer_timing": per_layer, "per_layer_error_vs_fp64": errs,
                "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": int(xh.numel() * 4),
                        "d2h_bytes_per_step": int(yh.numel() * 4), "ms_per_step": e2e_t,
                        "ms_steps": [round(v, 3) for v in e2e_ms],
                        "timing": "median of the K timed steps (CUDA events on the issuing stream)",
                        "api": f"StackPipeline(chunks={args.vgg_chunks}): pinned host images -> H2D | 13 layers | "
                               "D2H of the final activation, overlapped on 3 streams; weights resident",
                        "bitwise_equal_to_device_path": e2e_same},
                "timing": f"value/ms_per_step: CUDA-graph replay of the {st.kernels_per_forward}-kernel forward, "
                          "events around each step",
                "ms_steps": [round(v, 3) for v in ms_steps],
                "gpu_launches": st.kernels_per_forward * args.steps, "clocks": clk.summary(), "peaks": peak}
        if world == 1 and not args.no_cpu:
            procs = host_cores()
            xs = x_np[: args.cpu_vgg_images]
            t_all, outs, act = vgg_cpu_forward(xs, ws_np, procs)
            fl = vgg_direct_flops(xs.shape[0])
            line["cpu_baseline"] = {"value": fl / t_all / 1e12, "unit": "TFLOP/s", "cores": procs, "cpu_model": cpu_model(), "kind": "port",
                                    "sample": f"{xs.shape[0]} of {n} images through all 13 layers "
                                              f"(oracle/stack_pool.py over {procs} processes), {t_all:.2f} s"}
            if args.cpu_1core_images > 0:
                x1 = x_np[: args.cpu_1core_images]
                t1, _, _ = vgg_cpu_forward(x1, ws_np, 1)
                line["cpu_baseline_1core"] = {
                    "value": vgg_direct_flops(x1.shape[0]) / t1 / 1e12, "unit": "TFLOP/s", "cores": 1, "cpu_model": cpu_model(),
                    "kind": "port", "sample": f"{x1.shape[0]} image(s) through all 13 layers, one process "
                                              f"(numpy ufuncs are single-threaded), {t1:.2f} s"}
            same = [bool(outs[i].tobytes() == conv_first[i].tobytes()) for i in range(len(outs))]
            line["parity_vs_oracle"] = {"images": int(xs.shape[0]), "layers_bitwise_equal": same,
                                        "final_activation_bitwise_equal": bool(
                                            act.tobytes() == y_dev[: xs.shape[0]].cpu().numpy().tobytes()),
                                        "note": "the cpu_baseline's oracle outputs vs this run's batch-256 outputs "
                                                "of the same images (pre-activation y per layer, final activation)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measured_peaks():
    """Roofline denominators from the driver-written MEASURED_PEAKS.json, else
    the B200_PROFILING.md fallback (6.65 TB/s, 1.59 PFLOP/s bf16)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "source": "MEASURED_PEAKS.json (measured)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "B200_PROFILING.md fallback"}


def traffic_of(kernel, config, contraction):
    """Measured DRAM bytes per launch of `kernel` for a single-layer config.  Only the vgg16
    workload has a committed capture that includes the deferred L2 write-back
    (profiles/traffic_vgg16.json, vgg_traffic); a per-kernel --set full capture of these
    small layers misses most of the writes (they are still dirty in L2), so: None."""
    return None


def vgg_traffic(kernel="wino_contract"):
    """Measured DRAM bytes per launch of `kernel` over one VGG-16 forward, deferred L2
    write-back included (profiles/traffic_vgg16.json from tools/traffic.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_vgg16.json")) as fh:
            rows = [r for r in json.load(fh)["launches"] if r["kernel"] == kernel]
        return float(np.mean([r["traffic"] for r in rows])) if rows else None
    except Exception:
        return None


def vgg_roof(args, ach, peak, share, gbs=None):
    if args.contraction.startswith("tc_"):
        mp = measured_peaks()
        if gbs is not None:
            # 2 P T C K flops against 2 P C (T + K) + 4 P K T bytes: with K = 64..512 the unfused
            # tensor-core contraction at alpha = 8 is bound by writing its fp32 M, not by the tensor pipe
            return {"kernel": "tc_contract_kernel (13 layers)", "bound": "hbm", "achieved": gbs,
                    "peak": mp["hbm_gbs"], "unit": "GB/s", "frac": gbs / mp["hbm_gbs"], "traffic": None,
                    "peak_source": mp["source"] + " HBM copy bandwidth",
                    "bound_note": "U16 + V16 read and the fp32 M written per launch (algorithmic bytes); "
                                  "the same launches as a fraction of the dense bf16 tensor peak: "
                                  f"{ach / mp['bf16_tflops']:.3f} ({ach:.1f} of {mp['bf16_tflops']:.0f} TFLOP/s)",
                    "tensor_tflops": ach, "frac_of_tensor_peak": ach / mp["bf16_tflops"], "share_of_step": share}
        return {"kernel": "tc_contract_kernel (13 layers)", "bound": "tensor", "achieved": ach,
                "peak": mp["bf16_tflops"], "unit": "TFLOP/s", "frac": ach / mp["bf16_tflops"], "traffic": None,
                "peak_source": mp["source"] + " bf16 dense (burst)", "share_of_step": share}
    pk = max(peak["ffma_tflops"], peak.get("ffma2_tflops", 0.0))
    xceil = max(peak["fmul_fadd_tflops"], peak.get("fmul_fadd_packed_tflops", 0.0))
    return {"kernel": "wino_contract (13 layers)", "bound": "fp32", "bound_note": "FP32 CUDA-core pipe (neither HBM nor tensor cores): the reference rounds every product and sum separately, which tensor-core accumulation cannot reproduce", "achieved": ach, "peak": pk,
            "unit": "TFLOP/s", "frac": ach / pk, "traffic": vgg_traffic() if args.contraction == "exact" else None,
            "traffic_note": "mean DRAM bytes per contraction launch over the 13 layers at batch 256, incl. the "
                            "deferred L2 write-back (profiles/traffic_vgg16.json, tools/traffic.py)",
            "peak_source": "measured in this run: libwino wino_peak_probe, max of FFMA and packed FFMA2",
            "exact_ceiling_tflops": xceil, "frac_of_exact_ceiling": ach / xceil, "share_of_step": share}


def measure_peaks(lib, _native, torch):
    import ctypes
    out = torch.zeros(4, dtype=torch.float32, device="cuda")
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = sm * 8, 4096
    res = {}
    for mode, name in ((0, "ffma_tflops"), (1, "fmul_fadd_tflops"), (2, "dfma_tflops"), (3, "dmul_dadd_tflops"),
                       (4, "fmul_fadd_reg_tflops"), (5, "fmul_fadd_packed_tflops"), (6, "ffma2_tflops")):
        it = iters if mode in (0, 1, 4) else iters // 2 if mode in (5, 6) else iters // 8
        for _ in range(2):
            _native.check(lib.wino_peak_probe(mode, blocks, it, ctypes.c_void_p(out.data_ptr()),
                                              torch.cuda.current_stream().cuda_stream))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(lib.wino_peak_probe(mode, blocks, it, ctypes.c_void_p(out.data_ptr()),
                                          torch.cuda.current_stream().cuda_stream))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        # FFMA / DFMA step = 2 flops; FMUL+FADD step = 2 flops (one mul, one add)
        lanes = 2 if mode in (5, 6) else 1  # packed: each chain step is an f32x2 pair
        res[name] = blocks * 256 * 8 * lanes * it * 2 / (ms * 1e-3) / 1e12
    return res


def run_dryrun(args):
    """--dry-run: the multi-rank plumbing of the vgg16 bench on CPU ranks (gloo):
    rank environment, the batch shard of each rank, barrier + MAX-over-ranks step
    time, and the ordered all-gather of per-image error partials -- with the device
    forward replaced by the oracle's first VGG layer on small synthetic images.
    No GPU is touched; used by the launcher test."""
    import torch
    import torch.distributed as dist
    from oracle import wino_oracle as O
    from paper_1803_10986_b200 import distributed as Dd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    a, b = Dd.shard_range(args.vgg_batch, rank, world)
    trip = O.Triple.from_points(3, 6, VGG_POINTS)
    w = O.synthetic((8, 3, 3, 3), 2024, 10_000_000)

    def step(idx):
        x = np.stack([synth((3, 12, 12), 2024, i, "uniform") for i in idx]) if len(idx) else \
            np.zeros((0, 3, 12, 12), np.float32)
        y = O.layer_conv2d(trip, x, w, 1, "fp32", "huffman", "pairwise") if len(idx) else \
            np.zeros((0, 8, 12, 12), np.float32)
        return x, y

    for _ in range(args.warmup):
        step(range(a, b))
    ts = []
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        x, y = step(range(a, b))
        ts.append(time.perf_counter() - t0)
    ms = Dd.max_over_ranks(1e3 * float(np.mean(ts)))
    y64 = O.layer_direct_fp64(x, w, 1) if b > a else np.zeros((0, 8, 12, 12))
    st = np.stack(O.layer_error_stats(y, y64), axis=1).astype(np.float64) if b > a else np.zeros((0, 4))
    allst = Dd.gather_ordered(torch.from_numpy(np.ascontiguousarray(st))).numpy()
    spans = Dd.gather_ordered(torch.tensor([[a, b]], dtype=torch.int64)).tolist()
    err = Dd.combine_layer_stats(allst)
    if rank == 0:
        xa, ya = step(range(args.vgg_batch))  # one-process reference of the same statistics
        one = Dd.combine_layer_stats(np.stack(O.layer_error_stats(ya, O.layer_direct_fp64(xa, w, 1)), axis=1))
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms, "shards": spans,
                          "error_images": err["images"], "error": err, "error_equals_one_process": err == one}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------------------- block-size sweeps
def sweep_variants(which):
    """BASELINE configs[2] / configs[3] as concrete layer variants:
    (label, r, m, points, N, C, K, H, pad, x_dist, precision, dot_order, channel_sum)."""
    from paper_1803_10986_b200.pointsets import canonical_text, curated_text
    out = []
    if which == "sweep_cfg3":
        # F(m,3), m = 2..9, N64 C=K=256 28^2, U[-1,1]: good vs canonical points, Huffman vs
        # linear (the reference's "arbitrary order" baseline), fp32 vs mixed
        for m in range(2, 10):
            n = m + 2
            good, good_mx, canon = curated_text(n, 2, "fp32"), curated_text(n, 2, "mixed"), canonical_text(n)
            for tag, pts, prec, order in (("good", good, "fp32", "huffman"), ("good", good, "fp32", "linear"),
                                          ("canonical", canon, "fp32", "huffman"),
                                          ("good", good_mx, "mixed", "huffman")):
                out.append((f"m{m}-{tag}-{prec}-{order}", 3, m, pts, 64, 256, 256, 28, 1, "uniform", prec, order,
                            "linear"))
    else:
        # F(m,5), m = 2..6, N32 C=K=512 14^2 pad 2: linear vs pairwise channel sums on
        # U[0,1] (post-ReLU-like) and N(0,1) inputs; curated 2D set with n = alpha points
        for m in range(2, 7):
            pts = curated_text(m + 4, 2, "fp32")
            for dist in ("uniform01", "normal"):
                for cs in ("linear", "pairwise"):
                    out.append((f"m{m}-{dist}-{cs}", 5, m, pts, 32, 512, 512, 14, 2, dist, "fp32", "huffman", cs))
    return out


def run_sweep(args):
    """One JSON line per variant (time + error vs fp64 direct), then a summary line
    with the error directions SPEC.md:454 predicts (huffman < linear order, mixed <
    fp32, pairwise < linear channel sum) checked at layer scale."""
    import torch
    import paper_1803_10986_b200 as W
    from paper_1803_10986_b200 import _native
    torch.cuda.set_device(0)
    lines = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for label, r, m, pts, N, C, K, H, pad, xd, prec, order, cs in sweep_variants(args.config):
        ts = W.build_transforms(r, m, W.parse_points(pts))
        cfg = W.ConvConfig(prec, order, cs)
        op = W.layer_op(ts, cfg, N, C, H, H, K, pad, args.contraction)
        x_np = np.stack([synth((C, H, H), 2024, i, xd) for i in range(N)])
        w_np = synth((K, C, r, r), 2024, 10_000_000, "normal") * np.float32(np.sqrt(2.0 / (r * r * C)))
        x, w = torch.from_numpy(x_np).cuda(), torch.from_numpy(w_np).cuda()
        y = torch.empty(op.out_shape, dtype=torch.float32 if prec == "fp32" else torch.float64, device="cuda")
        ws = torch.empty(op.layout.workspace_bytes, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            op(x, w, out=y, workspace=ws)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            op(x, w, out=y, workspace=ws)
        ms = []
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = float(np.median(ms))
        st = W.layer_error_stats(y, W.direct_layer_f64(x, w, pad)).cpu().numpy()
        line = {"metric": METRIC, "workload": args.config, "variant": label, "winograd": f"F({m}x{m},{r}x{r})",
                "points": pts, "N": N, "C": C, "K": K, "H": H, "pad": pad, "x_dist": xd, "precision": prec,
                "dot_order": order, "channel_sum": cs, "contraction": args.contraction, "ms_per_step": t,
                "value": op.direct_flops / (t * 1e-3) / 1e12, "unit": "TFLOP/s",
                "contraction_tflops_note": "whole layer (K1+K2, K3, K4) as a CUDA graph, L2 flushed between steps",
                "error_vs_fp64": {"rel_l1": float(st[:, 0].sum() / st[:, 1].sum()),
                                  "per_point_l1": float(st[:, 0].sum() / st[:, 2].sum()),
                                  "max_abs": float(st[:, 3].max()), "images": int(N)}}
        lines.append(line)
        print(json.dumps(line), flush=True)
        del ws, y, x, w, g
    # error directions, per block size
    err = {ln["variant"]: ln["error_vs_fp64"]["rel_l1"] for ln in lines}
    checks = []

    def check(name, a, b, bound):
        if a in err and b in err:
            ratio = err[a] / err[b]
            checks.append({"check": name, "num": a, "den": b, "ratio": ratio, "bound": bound, "ok": ratio < bound})
    if args.config == "sweep_cfg3":
        for m in range(2, 10):
            check("huffman < linear order (SPEC: >= 5%)", f"m{m}-good-fp32-huffman", f"m{m}-good-fp32-linear", 0.95)
            check("mixed < fp32 (SPEC: ratio < 0.85)", f"m{m}-good-mixed-huffman", f"m{m}-good-fp32-huffman", 0.85)
            check("good < canonical points", f"m{m}-good-fp32-huffman", f"m{m}-canonical-fp32-huffman", 1.0)
    else:
        for m in range(2, 7):
            for dist in ("uniform01", "normal"):
                check("pairwise < linear channel sum (SPEC: ratio < 0.9)", f"m{m}-{dist}-pairwise",
                      f"m{m}-{dist}-linear", 0.9)
    print(json.dumps({"workload": args.config, "summary": True, "lines": len(lines), "direction_checks": checks,
                      "all_ok": all(c["ok"] for c in checks)}), flush=True)


def spawn_ranks(args):
    """`--gpus N` without a torchrun environment: re-exec this script under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous); the ranks'
    rank 0 prints the one JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="vgg16", choices=sorted(CONFIGS) + ["vgg16", "sweep_cfg3", "sweep_cfg4"])
    ap.add_argument("--vgg-batch", type=int, default=256)
    ap.add_argument("--vgg-chunks", default="32,192,32",
                    help="image chunks of the vgg16 e2e pipeline: a count or sizes a,b,... (scaled to the rank's "
                         "batch); small first / last chunks shorten the exposed H2D head and D2H tail "
                         "(69.0 ms vs 69.7 ms for 4 equal chunks)")
    ap.add_argument("--cpu-vgg-images", type=int, default=2, help="vgg16 CPU sample (BASELINE.md: 2-image slice)")
    ap.add_argument("--cpu-1core-images", type=int, default=1, help="vgg16 single-process CPU sample (0: skip)")
    ap.add_argument("--err-images", type=int, default=8)
    ap.add_argument("--no-err", action="store_true")
    ap.add_argument("--contraction", default="exact", choices=["exact", "ffma", "tc_bf16", "tc_fp16", "tcf_bf16", "tcf_fp16"])
    ap.add_argument("--cpu-images", type=int, default=32)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--soak", type=float, default=1.5, help="seconds of untimed load before the timed region")
    ap.add_argument("--e2e-chunks", default="4", help="image chunks of the e2e pipeline: a count or sizes a,b,...")
    ap.add_argument("--ncu", action="store_true", help="profiling mode: warm-up + K eager steps only, no output")
    ap.add_argument("--traffic", action="store_true", help="vgg16: one forward with an L2 eviction after each "
                    "kernel, for the ncu DRAM-traffic capture (tools/traffic.py)")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo rehearsal of the multi-rank plumbing (no GPU)")
    return ap.parse_args(argv)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.dry_run:
        run_dryrun(args)
        return
    if args.config == "vgg16":
        (run_reference_vgg if args.impl == "reference" else run_vgg)(args)
        return
    if args.config.startswith("sweep_"):
        run_sweep(args)
        return
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
