python tools/contract_bench.py --shape 32,128,28,128 --m 2 --cs linear --variants "8,8,16,8,16,4,0,8,1;8,8,16,8,16,6,0,8,1;8,8,8,16,16,4,0,8,1;8,8,16,8,32,4,0,8,1" > gpurun_out/sw_a.jsonl 2>&1
python tools/contract_bench.py --shape 64,256,28,256 --m 6 --cs linear --variants "8,8,16,8,16,4,0,8,1;8,8,16,8,16,6,0,8,1" >> gpurun_out/sw_a.jsonl 2>&1
python tools/contract_bench.py --shape 32,128,28,128 --m 2 --cs linear --contraction ffma --variants "8,8,16,8,16,4,0,8,1;8,8,8,16,16,4,0,8,1" >> gpurun_out/sw_a.jsonl 2>&1
python tools/contract_bench.py --shape 64,256,28,256 --m 6 --cs pairwise --prec mixed --variants "4,4,8,16,32,4,168,8,1;4,4,8,16,32,6,168,8,1;4,4,16,16,32,4,0,8,1" >> gpurun_out/sw_a.jsonl 2>&1
