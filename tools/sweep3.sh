timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_stack.py -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
python tools/contract_bench.py --shape 64,256,28,256 --m 6 --cs pairwise --prec mixed --variants "4,4,8,16,32,4,0,8;4,4,16,16,32,4,0,8;4,4,8,16,32,3,168,8;4,8,8,16,32,3,0,8;8,4,8,16,32,3,0,8;4,4,8,16,16,4,168,8" > gpurun_out/sw_a.jsonl 2>&1
python tools/contract_bench.py --shape 32,512,14,512 --m 4 --r 5 --cs pairwise >> gpurun_out/sw_a.jsonl 2>&1
