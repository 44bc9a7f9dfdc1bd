# Full GPU test suite + smoke + every bench line + launch list + ncu captures + DRAM traffic
# (run on the GPU box from the repo root:  gpurun -- 'bash tools/round_bench.sh')
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
# headline: BASELINE configs[4] (VGG-16, batch 256) -- the default workload, then the reference arm
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_vgg16.log 2>&1; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_vgg16_reference.log 2>&1; echo reference rc=$?
python bench.py --steps 5 --warmup 3 --contraction tc_bf16 --no-cpu > gpurun_out/bench_vgg16_tc_bf16.log 2>&1
python bench.py --steps 5 --warmup 3 --contraction tc_fp16 --no-cpu > gpurun_out/bench_vgg16_tc_fp16.log 2>&1
python bench.py --steps 5 --warmup 3 --contraction ffma --no-cpu > gpurun_out/bench_vgg16_ffma.log 2>&1
# single-layer configs (extra lines)
for c in cfg1 cfg2 cfg3_m6 cfg3_m6_mixed_pw cfg4_m4; do
  python bench.py --config $c --steps 20 --warmup 5 --soak 0.5 > gpurun_out/bench_$c.log 2>&1
done
for m in ffma tc_bf16 tc_fp16; do
  python bench.py --config cfg2 --contraction $m --steps 20 --warmup 5 --no-cpu --soak 0.5 > gpurun_out/bench_cfg2_$m.log 2>&1
  python bench.py --config cfg3_m6 --contraction $m --steps 20 --warmup 5 --no-cpu --soak 0.5 > gpurun_out/bench_cfg3_m6_$m.log 2>&1
done
for m in tcf_bf16 tcf_fp16; do  # fused K3t+K4 needs alpha^2 <= 32 (cfg2, cfg1)
  python bench.py --config cfg2 --contraction $m --steps 20 --warmup 5 --no-cpu --soak 0.5 > gpurun_out/bench_cfg2_$m.log 2>&1
done
# BASELINE configs[2] / configs[3] sweeps: one line per (m, points, order, precision, sum, input) cell
python bench.py --config sweep_cfg3 --steps 10 --warmup 3 --no-cpu --soak 0.2 > gpurun_out/bench_sweep_cfg3.log 2>&1
python bench.py --config sweep_cfg4 --steps 10 --warmup 3 --no-cpu --soak 0.2 > gpurun_out/bench_sweep_cfg4.log 2>&1
# ncu: launch list of the default command, then --set full of one layer's three kernels (layer 9:
# 3 warm-up forwards x 38 kernels + 2 of layer 1 + 7 layers x 3), then the fused layer-1 kernel
python bench.py --ncu --steps 2 --warmup 3 > gpurun_out/b_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --ncu --steps 2 --warmup 3 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"wino_contract|wino_transforms|wino_output|wino_smallc2" -s 137 -c 3 \
    -o gpurun_out/prof_bench python bench.py --ncu --steps 1 --warmup 3 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"wino_smallc2" -s 3 -c 1 \
    -o gpurun_out/prof_smallc2 python bench.py --ncu --steps 1 --warmup 3 > gpurun_out/ncu3.log 2>&1
# tensor-core mode: the three kernels of a 56 x 56 layer (layer 1 runs the exact path and is not matched: 36 matching kernels per forward)
ncu --set full --clock-control none --import-source on \
    -k regex:"tc_contract_kernel|wino_transforms_tc|wino_output_gather_act" -s 120 -c 3 \
    -o gpurun_out/prof_tc python bench.py --ncu --contraction tc_bf16 --steps 1 --warmup 3 > gpurun_out/ncu4.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/traffic.csv python bench.py --traffic > gpurun_out/traffic_run.log 2>&1
echo all done
