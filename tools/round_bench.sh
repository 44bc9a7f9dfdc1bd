# Full bench + launch list + ncu capture of the top kernels (run on the GPU box
# from the repo root:  gpurun -- 'bash tools/round_bench.sh')
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench rc=$?
for c in cfg1 cfg3_m6 cfg3_m6_mixed_pw cfg4_m4; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu --soak 0.5 > gpurun_out/bench_$c.log 2>&1
done
python bench.py --contraction ffma --steps 20 --warmup 5 --no-cpu --soak 0.5 > gpurun_out/bench_cfg2_ffma.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --soak 0 > gpurun_out/b_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --soak 0 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"wino_contract|wino_input_xform|wino_output_xform|wino_filter_xform" -s 4 -c 4 \
    -o gpurun_out/prof_bench python bench.py --steps 2 --warmup 3 --no-cpu --soak 0 > gpurun_out/ncu2.log 2>&1
echo all done
