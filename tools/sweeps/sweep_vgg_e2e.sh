# e2e (StackPipeline) chunk schedules for the VGG-16 batch-256 headline
for c in "32,192,32" "16,224,16" "24,208,24" "16,208,32" "32,96,96,32" "8,240,8"; do
  python bench.py --steps 10 --warmup 3 --no-cpu --no-err --soak 0.2 --vgg-chunks "$c" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']
print('$c', round(e['value'],2), 'TFLOP/s', round(e['ms_per_step'],3), 'ms', e['bitwise_equal_to_device_path'], 'device', round(d['ms_per_step'],3))"
done
