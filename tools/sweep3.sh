timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pt_tc.log 2>&1; tail -30 gpurun_out/pt_tc.log
python tools/contract_bench.py --shape 32,128,28,128 --m 2 --cs linear --contraction tc_bf16 > gpurun_out/sw_tc.jsonl 2>&1
python tools/contract_bench.py --shape 64,256,28,256 --m 6 --cs linear --contraction tc_bf16 >> gpurun_out/sw_tc.jsonl 2>&1
cat gpurun_out/sw_tc.jsonl
for c in cfg2 cfg3_m6; do python bench.py --config $c --contraction tc_bf16 --steps 20 --warmup 5 --no-cpu --soak 0.3 > gpurun_out/bench_${c}_tc.log 2>&1; done
python bench.py --config vgg16 --steps 5 --warmup 2 --contraction tc_bf16 --no-err > gpurun_out/bench_vgg16_tc.log 2>&1
