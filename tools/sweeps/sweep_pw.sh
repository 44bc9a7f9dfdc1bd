# Pairwise contraction tile sweep (bitwise equality vs default checked by contract_bench)
python tools/contract_bench.py --shape 64,256,28,256 --m 6 --cs pairwise --variants "4,4,16,16,32,4,168,8,0,1;4,4,8,32,32,4,168,8,0,1;4,4,16,16,32,3,168,8,0,1;4,4,8,16,32,6,168,8,0,1;4,4,16,16,16,6,168,8,0,1;4,4,32,8,32,4,168,8,0,1"
python tools/contract_bench.py --shape 32,512,14,512 --m 4 --r 5 --cs pairwise --variants "4,4,16,16,32,4,168,8,0,1;4,4,8,32,32,4,168,8,0,1"
python tools/contract_bench.py --shape 32,64,224,64 --m 6 --cs pairwise --variants "4,4,16,16,32,4,168,8,0,1;4,4,8,32,32,4,168,8,0,1"
