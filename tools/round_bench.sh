# Full GPU test suite + smoke + benches + launch list + ncu captures (run on the GPU box
# from the repo root:  gpurun -- 'bash tools/round_bench.sh')
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench rc=$?
python bench.py --steps 20 --warmup 5 --e2e-chunks 8 --no-cpu --soak 0.3 > gpurun_out/bench_e2e8.log 2>&1
for c in cfg1 cfg3_m6 cfg3_m6_mixed_pw cfg4_m4; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu --soak 0.5 > gpurun_out/bench_$c.log 2>&1
done
for m in ffma tc_bf16 tc_fp16; do
  python bench.py --contraction $m --steps 20 --warmup 5 --no-cpu --soak 0.5 > gpurun_out/bench_cfg2_$m.log 2>&1
  python bench.py --config cfg3_m6 --contraction $m --steps 20 --warmup 5 --no-cpu --soak 0.5 > gpurun_out/bench_cfg3_m6_$m.log 2>&1
done
for m in tcf_bf16 tcf_fp16; do  # fused K3t+K4 needs alpha^2 <= 32 (cfg2, cfg1)
  python bench.py --contraction $m --steps 20 --warmup 5 --no-cpu --soak 0.5 > gpurun_out/bench_cfg2_$m.log 2>&1
done
python bench.py --config vgg16 --steps 5 --warmup 2 > gpurun_out/bench_vgg16.log 2>&1
python bench.py --config vgg16 --steps 5 --warmup 2 --contraction tc_bf16 --no-err > gpurun_out/bench_vgg16_tc_bf16.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1
python bench.py --ncu --steps 5 --warmup 3 > gpurun_out/b_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --ncu --steps 5 --warmup 3 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"wino_contract|wino_transforms|wino_output" -s 3 -c 3 \
    -o gpurun_out/prof_bench python bench.py --ncu --steps 2 --warmup 3 > gpurun_out/ncu2.log 2>&1
echo all done
