timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_stack.py tests/test_gpu_tile.py -x -q > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for k in gather tile; do
  for sh in "32,128,28,128 --m 2" "64,256,28,256 --m 6" "8,64,56,64 --m 4" "32,512,14,512 --m 4" "8,64,224,64 --m 6"; do
    WINO_K1=$k python tools/xform_bench.py --shape $sh | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', d['shape'], d['m'], 'tr %.1f in %.1f (%.0f GB/s) triv-tr %.1f out %.1f' % (d['real_transforms_us'], d['real_input_us'], d['real_input_gbs'], d['trivial_transforms_us'], d['real_output_us']))"
  done
done
