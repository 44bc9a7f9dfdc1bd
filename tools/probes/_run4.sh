timeout 1500 python -m pytest tests/test_gpu_stack.py tests/test_gpu_layer.py tests/test_gpu_pipeline.py -m gpu -q -x 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu --no-err > gpurun_out/bench_pair.log 2>&1; echo rc=$?
for c in cfg1 cfg2 cfg3_m6 cfg4_m4 cfg3_m6_mixed_pw; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-err --soak 0.3 > gpurun_out/pair_$c.log 2>&1; done
