python bench.py --steps 20 --warmup 5 --no-cpu --soak 0.5 > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
python tools/contract_bench.py --shape 32,128,28,128 --m 2 --cs linear --variants "8,16,16,8,16,4,0,8;16,8,8,16,16,4,0,8" > gpurun_out/sw_a.jsonl 2>&1
