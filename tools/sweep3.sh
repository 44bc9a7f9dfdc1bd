timeout 900 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for k in 8 4x8; do
  for sh in "32,128,28,128 --m 2" "8,224,112,224 --m 2" "64,3,224,64 --m 2"; do
    WINO_K1TC=$k python tools/xform_bench.py --contraction tc_bf16 --shape $sh | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', d['shape'], d['m'], 'tr %.1f in %.1f (%.0f GB/s) triv-tr %.1f' % (d['real_transforms_us'], d['real_input_us'], d['real_input_gbs'], d['trivial_transforms_us']))"
  done
done
