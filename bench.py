"""Benchmark of the Winograd layer hot path (BASELINE.json metric:
"Winograd conv direct-equiv TFLOP/s").

Default workload = BASELINE.json configs[1]: F(2x2, 3x3), points {0,1,-1,inf},
fp32 throughout (huffman transforms, linear channel sum, exact contraction),
N=32 per GPU, C=K=128, H=W=28, pad 1, x ~ U[-1,1], w ~ He-normal, seeded.
A step = filter transform + input transform + channel contraction + output
transform of one batch (the four libwino kernels, inputs resident in HBM).
Multi-GPU: one process per GPU, each rank runs its own batch (global image
indices rank*N .. rank*N+N-1) -> weak scaling; NCCL only reduces timings and
error statistics.  `--impl reference` times the CPU port of the reference's
arithmetic (oracle/) on the host cores for the same workload.
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
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": procs, "kind": "port",
                             "sample": f"full batch of {x.shape[0]} images per step, oracle/wino_oracle.py "
                                       f"layer_conv2d (numpy restatement of the reference) over {procs} processes"},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(args, cfg, world=1):
    r, m, pts, N, C, K, H, pad, xd, wi, prec, order, cs = cfg
    return {"workload": args.config, "winograd": f"F({m}x{m},{r}x{r})", "points": pts, "N_per_gpu": N,
            "global_batch": N * world, "C": C, "K": K, "H": H, "W": H, "pad": pad, "precision": prec,
            "dot_order": order, "channel_sum": cs, "contraction": args.contraction,
            "x_dist": xd, "w_init": wi, "l2": "flushed between timed steps: 256 MiB write, then 256 MiB read of a clean buffer "
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
        pk = mp["bf16_tflops"]
        roof = {"kernel": "tc_contract_kernel (tcgen05.mma kind::f16)", "bound": "tensor", "achieved": ach,
                "peak": pk, "unit": "TFLOP/s", "frac": ach / pk, "traffic": None,
                "peak_source": mp["source"] + " bf16 dense (burst)"}
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
    stage_bytes = [4 * K * C * r * r + eb * L.P * C * K + 4 * N * C * H * H + eb * L.P * L.T * C,
                   None,
                   None,
                   eb * L.P * L.T * K + (4 if prec == "fp32" else 8) * N * K * L.Ho * L.Wo]
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
            line["cpu_baseline"] = {"value": fl / t / 1e12, "unit": "TFLOP/s", "cores": procs, "kind": "port",
                                    "sample": f"{xs.shape[0]} of {N} images of the same layer, oracle/wino_oracle.py "
                                              f"layer_conv2d over {procs} processes, {t:.2f} s"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
    from paper_1803_10986_b200.stack import VGG16, ConvStack, he_normal_weights

    pts = "0,-1,1,1/2,-1/2,2,-2,inf"
    ts = W.build_transforms(3, 6, W.parse_points(pts))
    a, b = shard_range(args.vgg_batch, rank, world)
    n = b - a
    st = ConvStack(ts, W.ConvConfig("fp32", "huffman", "pairwise"), VGG16, n, 224,
                   contraction=args.contraction)
    st.set_weights(he_normal_weights(VGG16, 3))
    x = torch.empty((n, 3, 224, 224), dtype=torch.float32, device="cuda")
    for i in range(n):  # synthetic U[-1,1] images keyed by global image index
        x[i].copy_(torch.from_numpy(synth((3, 224, 224), 2024, a + i, "uniform")))
    for _ in range(max(3, args.warmup)):
        st.forward(x)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        st.forward(x)
    graph.replay()
    torch.cuda.synchronize()
    es = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for e0, e1 in es:  # inputs and activations >> L2: no flush needed
            e0.record()
            graph.replay()
            e1.record()
        torch.cuda.synchronize()
    ms = float(np.mean([e0.elapsed_time(e1) for e0, e1 in es]))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_flops = st.direct_flops * world if world == 1 else None
    flops_all = 0
    for op_ in st.ops:
        flops_all += op_.direct_flops
    # whole-job direct-eq flops: every rank's shard (equal or +-1 image)
    gflops = torch.tensor([float(flops_all)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(gflops)
    value = float(gflops.item()) / (ms * 1e-3) / 1e12
    # per-kernel shares from an instrumented forward (events around each contraction)
    lib = _native.lib()
    import ctypes
    c_ms = 0.0
    c_flops = 0
    other_ms = 0.0
    per_layer = []
    cur = x
    s = torch.cuda.current_stream().cuda_stream
    for i, op_ in enumerate(st.ops):
        L = op_.layout
        ws = st.workspace
        al = lambda v: (v + 255) // 256 * 256
        U = ws.data_ptr()
        V = U + al(L.u_bytes)
        M = V + al(L.v_bytes)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        _native.check(lib.wino_filter_transform(op_.plan.handle, ctypes.byref(op_.shape),
                                                _native.as_ptr(st.weights[i]), ctypes.c_void_p(U), s))
        _native.check(lib.wino_input_transform(op_.plan.handle, ctypes.byref(op_.shape), _native.as_ptr(cur),
                                               ctypes.c_void_p(V), s))
        ev[1].record()
        _native.check(lib.wino_contract(op_.plan.handle, ctypes.byref(op_.shape), ctypes.c_void_p(U),
                                        ctypes.c_void_p(V), ctypes.c_void_p(M), s))
        ev[2].record()
        C, K, h, w_, pool = st.shapes[i]
        if st.fused_act:  # the forward's K4 with ReLU / max-pool fused
            _native.check(lib.wino_output_transform_act(op_.plan.handle, ctypes.byref(op_.shape),
                                                        ctypes.c_void_p(M), _native.as_ptr(st.act[i]),
                                                        1 if pool else 0, s))
        else:
            _native.check(lib.wino_output_transform(op_.plan.handle, ctypes.byref(op_.shape), ctypes.c_void_p(M),
                                                    _native.as_ptr(st.conv_out[i]), s))
            _native.check(lib.wino_relu_pool(0, op_.N * K, L.Ho, L.Wo, 1 if pool else 0,
                                             _native.as_ptr(st.conv_out[i]), _native.as_ptr(st.act[i]), s))
        ev[3].record()
        torch.cuda.synchronize()
        c_ms += ev[1].elapsed_time(ev[2])
        other_ms += ev[0].elapsed_time(ev[1]) + ev[2].elapsed_time(ev[3])
        per_layer.append({"layer": i + 1, "C": C, "K": K, "H": h, "bm_bn": [L.bm, L.bn],
                          "transforms_ms": ev[0].elapsed_time(ev[1]), "contract_ms": ev[1].elapsed_time(ev[2]),
                          "contract_tflops": op_.contraction_flops / (ev[1].elapsed_time(ev[2]) * 1e-3) / 1e12,
                          "output_relu_pool_ms": ev[2].elapsed_time(ev[3])})
        c_flops += op_.contraction_flops
        cur = st.act[i]
    peak = measure_peaks(lib, _native, torch)
    ach = c_flops / (c_ms * 1e-3) / 1e12
    errs = st.layer_errors(x, images=args.err_images) if not args.no_err else None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded Philox U[-1,1] 224x224x3 images, He-normal filters)",
                "config": {"workload": "vgg16", "winograd": "F(6x6,3x3)", "points": pts,
                           "global_batch": args.vgg_batch, "batch_per_gpu": n, "precision": "fp32",
                           "dot_order": "huffman", "channel_sum": "pairwise", "contraction": args.contraction,
                           "layers": 13, "pools_after": [2, 4, 7, 10],
                           "l2": "inputs/activations >> L2 (no flush)",
                           "parallelism": f"dp{world} (batch sharded)"},
                "roofline": vgg_roof(args, ach, peak, c_ms / (c_ms + other_ms)),
                "per_layer_error_vs_fp64": errs, "per_layer_timing": per_layer,
                "gpu_launches": st.kernels_per_forward * args.steps,
                "clocks": clk.summary(), "peaks": peak}
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
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu
    --set full capture summary (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(f"{config}/{contraction}/{kernel}")
    except Exception:
        return None


def vgg_roof(args, ach, peak, share):
    if args.contraction.startswith("tc_"):
        mp = measured_peaks()
        return {"kernel": "tc_contract_kernel (13 layers)", "bound": "tensor", "achieved": ach,
                "peak": mp["bf16_tflops"], "unit": "TFLOP/s", "frac": ach / mp["bf16_tflops"], "traffic": None,
                "peak_source": mp["source"] + " bf16 dense (burst)", "share_of_step": share}
    pk = max(peak["ffma_tflops"], peak.get("ffma2_tflops", 0.0))
    xceil = max(peak["fmul_fadd_tflops"], peak.get("fmul_fadd_packed_tflops", 0.0))
    return {"kernel": "wino_contract (13 layers)", "bound": "fp32", "bound_note": "FP32 CUDA-core pipe (neither HBM nor tensor cores): the reference rounds every product and sum separately, which tensor-core accumulation cannot reproduce", "achieved": ach, "peak": pk,
            "unit": "TFLOP/s", "frac": ach / pk, "traffic": None,
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS) + ["vgg16"])
    ap.add_argument("--vgg-batch", type=int, default=256)
    ap.add_argument("--err-images", type=int, default=8)
    ap.add_argument("--no-err", action="store_true")
    ap.add_argument("--contraction", default="exact", choices=["exact", "ffma", "tc_bf16", "tc_fp16", "tcf_bf16", "tcf_fp16"])
    ap.add_argument("--cpu-images", type=int, default=32)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--soak", type=float, default=1.5, help="seconds of untimed load before the timed region")
    ap.add_argument("--e2e-chunks", default="4", help="image chunks of the e2e pipeline: a count or sizes a,b,...")
    ap.add_argument("--ncu", action="store_true", help="profiling mode: warm-up + K eager steps only, no output")
    args = ap.parse_args()
    if args.config == "vgg16":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "vgg16 CPU reference: use --config cfg2"}))
            return
        run_vgg(args)
        return
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
