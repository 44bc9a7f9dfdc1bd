python tools/contract_bench.py --shape 32,128,28,128 --m 2 --cs linear --reps 3 > gpurun_out/p0.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wino_contract -s 3 -c 1 -o gpurun_out/prof_lin2 python tools/contract_bench.py --shape 32,128,28,128 --m 2 --cs linear --reps 3 > gpurun_out/p1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:wino_contract -s 3 -c 1 -o gpurun_out/prof_ffma2 python tools/contract_bench.py --shape 32,128,28,128 --m 2 --cs linear --contraction ffma --reps 3 > gpurun_out/p2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:wino_contract -s 3 -c 1 -o gpurun_out/prof_pw2 python tools/contract_bench.py --shape 64,256,28,256 --m 6 --cs pairwise --prec mixed --reps 3 > gpurun_out/p3.log 2>&1
