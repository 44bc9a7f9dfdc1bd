timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_tc.py -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for c in cfg2; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu --soak 0.3 > gpurun_out/bench_$c.log 2>&1; python bench.py --config $c --contraction tc_bf16 --steps 20 --warmup 5 --no-cpu --soak 0.3 > gpurun_out/bench_${c}_tc.log 2>&1; done
