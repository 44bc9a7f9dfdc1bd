import ctypes, sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.abspath(__file__)))
import tuning_env  # noqa: E402,F401  (WINO_* env -> libwino tuning keys)
import paper_1803_10986_b200 as W
from paper_1803_10986_b200 import _native
ts = W.build_transforms(3, 2, W.parse_points("0,1,-1,inf"))
op = W.layer_op(ts, W.ConvConfig(), 32, 128, 28, 28, 128, 1)
L = op.layout
x = torch.randn(32, 128, 28, 28, device="cuda"); w = torch.randn(128, 128, 3, 3, device="cuda")
y = torch.empty(op.out_shape, device="cuda")
U = torch.empty((L.P, L.Cp, L.Kp), device="cuda"); V = torch.empty((L.P, L.Cp, L.Tp), device="cuda"); M = torch.empty((L.P, L.Kp, L.Tp), device="cuda")
lib = _native.lib(); sref = ctypes.byref(op.shape); P = _native.as_ptr
def step(evs=None):
    s = torch.cuda.current_stream().cuda_stream
    if evs: evs[0].record()
    lib.wino_filter_transform(op.plan.handle, sref, P(w), P(U), s)
    if evs: evs[1].record()
    lib.wino_input_transform(op.plan.handle, sref, P(x), P(V), s)
    if evs: evs[2].record()
    lib.wino_contract(op.plan.handle, sref, P(U), P(V), P(M), s)
    if evs: evs[3].record()
    lib.wino_output_transform(op.plan.handle, sref, P(M), P(y), s)
    if evs: evs[4].record()
for _ in range(3): step()
torch.cuda.synchronize()
res = {}
# eager with events
evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for _ in range(3): step(evs)
torch.cuda.synchronize()
res["eager_stage_ms"] = [evs[i].elapsed_time(evs[i+1]) for i in range(4)]
# graph with events inside
g = torch.cuda.CUDAGraph()
gevs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(5)]
s = torch.cuda.Stream()
try:
    with torch.cuda.graph(g, stream=s):
        step(gevs)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    res["graph_stage_ms"] = [gevs[i].elapsed_time(gevs[i+1]) for i in range(4)]
    res["graph_total_ms"] = gevs[0].elapsed_time(gevs[4])
except Exception as e:
    res["graph_events_error"] = str(e)[:300]
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2, stream=s):
    step()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3): g2.replay()
torch.cuda.synchronize()
e0.record(); 
for _ in range(20): g2.replay()
e1.record(); torch.cuda.synchronize()
res["graph_replay_ms"] = e0.elapsed_time(e1) / 20
e0.record()
for _ in range(20): step()
e1.record(); torch.cuda.synchronize()
res["eager_ms"] = e0.elapsed_time(e1) / 20
res["launches"] = _native.launch_count()
print(json.dumps(res))
