timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_stack.py tests/test_gpu_tc.py -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for k in gather staged; do
  for cm in exact tc_bf16; do
  for sh in "32,128,28,128 --m 2" "64,256,28,256 --m 6" "8,64,56,64 --m 4" "32,512,14,512 --m 4" "8,64,224,64 --m 6"; do
    WINO_K4=$k python tools/xform_bench.py --contraction $cm --shape $sh | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k $cm', d['shape'], d['m'], 'out %.1f (%.0f GB/s)' % (d['real_output_us'], d['real_output_gbs']))"
  done
  done
done
