# Packed f32x2 contraction vs scalar: timings + bitwise equality (same_as_default)
set -x
python tools/contract_bench.py --shape 32,128,28,128 --m 2 --cs linear --variants "8,8,16,8,16,4,0,8,0,1;8,8,16,8,32,3,0,8,0,1;8,8,16,8,16,4,0,16,0,1;8,8,8,16,16,4,0,8,0,1;8,16,16,8,16,3,0,8,0,1;16,8,8,16,16,3,0,8,0,1"
python tools/contract_bench.py --shape 32,128,28,128 --m 2 --cs linear --contraction ffma --variants "8,8,16,8,16,4,0,8,0,1;8,16,16,8,16,3,0,8,0,1"
python tools/contract_bench.py --shape 64,256,28,256 --m 6 --cs pairwise --variants "4,4,8,16,32,4,168,8,0,1;4,4,8,16,32,4,0,8,0,1;4,8,8,16,32,4,0,8,0,1;8,4,16,8,32,3,0,8,0,1"
python tools/contract_bench.py --shape 64,256,28,256 --m 6 --cs linear --variants "8,8,16,8,16,4,0,8,0,1"
python tools/contract_bench.py --shape 32,512,14,512 --m 4 --r 5 --cs pairwise --variants "4,4,8,16,32,4,168,8,0,1;4,8,8,16,32,4,0,8,0,1"
