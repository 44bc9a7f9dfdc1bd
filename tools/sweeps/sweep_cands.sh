# Tile-candidate efficiencies (WINO_GEMM forces one config; default = shape-picked)
set -x
python tools/contract_bench.py --shape 8,64,56,64 --m 4 --cs linear --variants "8,8,16,8,16,4,0,16,0,1;8,8,8,16,16,4,0,16,0,1;4,8,16,8,16,4,0,16,0,1"
python tools/contract_bench.py --shape 64,256,28,256 --m 6 --cs linear --variants "8,8,16,8,16,4,0,16,0,1;8,8,8,16,16,4,0,16,0,1;4,8,16,8,16,4,0,16,0,1"
python tools/contract_bench.py --shape 32,64,224,64 --m 6 --cs pairwise --variants "4,4,8,16,32,4,168,8,0,1"
python tools/contract_bench.py --shape 32,3,224,64 --m 6 --cs pairwise --variants "4,4,8,16,32,4,168,8,0,1;4,4,8,16,8,4,168,8,0,1"
python tools/contract_bench.py --shape 32,64,224,64 --m 6 --cs linear --variants "8,8,16,8,16,4,0,16,0,1;8,8,8,16,16,4,0,16,0,1"
python tools/contract_bench.py --shape 32,128,28,128 --m 2 --cs linear --variants "8,8,16,8,16,4,0,16,0,1;4,8,16,8,16,4,0,16,0,1"
