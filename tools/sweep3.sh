timeout 600 python -m pytest tests/test_gpu_stack.py -x -q > gpurun_out/pt_stack.log 2>&1; tail -3 gpurun_out/pt_stack.log
timeout 600 python bench.py --config vgg16 --steps 5 --warmup 2 > gpurun_out/bench_vgg.log 2>&1; tail -c 2500 gpurun_out/bench_vgg.log
