# compute-sanitizer passes over small instances of every libwino kernel family
set -x
S="compute-sanitizer --print-limit 20 --error-exitcode 9"
$S --tool memcheck python -c "
import sys; sys.path.insert(0, '.')
import numpy as np, paper_1803_10986_b200 as W
from oracle import wino_oracle as O
for (r, m, pts) in [(3, 2, '0,1,-1,inf'), (3, 6, '0,-1,1,1/2,-1/2,2,-2,inf'), (5, 2, '0,-1,1,1/2,-2,inf')]:
    ts = W.build_transforms(r, m, W.parse_points(pts))
    x = O.synthetic((2, 19, 13, 11), 1, 0); w = O.synthetic((21, 19, r, r), 1, 1)
    for cfg in [W.ConvConfig(), W.ConvConfig('mixed', 'huffman', 'pairwise'), W.ConvConfig('fp64', 'linear', 'linear')]:
        W.conv2d_layer(ts, x, w, cfg, pad=1)
    for mode in ['ffma', 'tc_bf16', 'tcf_fp16']:
        if mode == 'tcf_fp16' and m == 6: continue
        W.conv2d_layer(ts, x, w, W.ConvConfig(), pad=1, contraction=mode)
print('memcheck workload done')
"
for tool in racecheck synccheck; do
$S --tool $tool python tools/contract_bench.py --shape 2,40,12,40 --m 2 --reps 1
$S --tool $tool python tools/contract_bench.py --shape 2,70,12,40 --m 4 --cs pairwise --reps 1
done
