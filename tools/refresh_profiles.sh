# Copy a round_bench.sh run (gpurun_out/) into the tracked profiles/ (round tag $1, default r2)
R=${1:-r2}
cd "$(dirname "$0")/.."
for f in gpurun_out/bench_*.log; do
  n=$(basename "$f" .log)
  case "$n" in
    bench_sweep_*) grep '^{' "$f" > profiles/${R}_${n}.jsonl || echo "skip $f" ;;
    *) [ -s "$f" ] && grep '^{' "$f" | tail -1 | python -c "import json,sys; json.dump(json.loads(sys.stdin.read()), open('profiles/${R}_${n}.json','w'), indent=1)" \
         || echo "skip $f" ;;
  esac
done
[ -s gpurun_out/launches.csv ] && python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/${R}_launches.md
[ -s gpurun_out/prof_bench.ncu-rep ] && python tools/ncu_summary.py full gpurun_out/prof_bench.ncu-rep > profiles/${R}_kernels.md
[ -s gpurun_out/prof_smallc2.ncu-rep ] && python tools/ncu_summary.py full gpurun_out/prof_smallc2.ncu-rep > profiles/${R}_kernel_smallc2.md
[ -s gpurun_out/prof_tc.ncu-rep ] && python tools/ncu_summary.py full gpurun_out/prof_tc.ncu-rep > profiles/${R}_kernels_tc.md
[ -s gpurun_out/traffic.csv ] && python tools/traffic.py gpurun_out/traffic.csv profiles/traffic_vgg16.json
cp gpurun_out/pytest_gpu.log profiles/${R}_pytest_gpu.log 2>/dev/null
echo refreshed
