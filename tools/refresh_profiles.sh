# Copy a round_bench.sh run (gpurun_out/) into the tracked profiles/ (round tag $1, default r1)
R=${1:-r1}
cd "$(dirname "$0")/.."
for pair in bench.log:bench bench_cfg1.log:bench_cfg1 bench_cfg2_ffma.log:bench_cfg2_ffma \
    bench_cfg2_tc_bf16.log:bench_cfg2_tc_bf16 bench_cfg2_tc_fp16.log:bench_cfg2_tc_fp16 \
    bench_cfg2_tcf_bf16.log:bench_cfg2_tcf_bf16 bench_cfg2_tcf_fp16.log:bench_cfg2_tcf_fp16 \
    bench_cfg3_m6.log:bench_cfg3_m6 bench_cfg3_m6_ffma.log:bench_cfg3_m6_ffma \
    bench_cfg3_m6_mixed_pw.log:bench_cfg3_m6_mixed_pw bench_cfg3_m6_tc_bf16.log:bench_cfg3_m6_tc_bf16 \
    bench_cfg3_m6_tc_fp16.log:bench_cfg3_m6_tc_fp16 bench_cfg4_m4.log:bench_cfg4_m4 bench_e2e8.log:bench_e2e8 \
    bench_reference.log:bench_reference bench_vgg16.log:bench_vgg16 bench_vgg16_tc_bf16.log:bench_vgg16_tc_bf16; do
  src=gpurun_out/${pair%%:*}; dst=profiles/${R}_${pair##*:}.json
  [ -s "$src" ] && tail -1 "$src" | python -c "import json,sys; json.dump(json.loads(sys.stdin.read()), open('$dst','w'), indent=1)" \
    || echo "skip $src"
done
[ -s gpurun_out/launches.csv ] && python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/${R}_launches.md
[ -s gpurun_out/prof_bench.ncu-rep ] && python tools/ncu_summary.py full gpurun_out/prof_bench.ncu-rep > profiles/${R}_kernels.md
cp gpurun_out/pytest_gpu.log profiles/${R}_pytest_gpu.log 2>/dev/null
echo refreshed
