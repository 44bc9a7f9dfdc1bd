# e2e (HostPipeline) chunk schedules for the default bench config
for c in 4 8 "10,8,6,4,2,2" "12,8,6,4,2" "8,8,6,4,3,2,1" "6,6,6,5,4,3,2" "16,8,4,2,1,1" "9,8,7,4,2,1,1"; do
  python bench.py --steps 20 --warmup 5 --no-cpu --soak 0.2 --e2e-chunks "$c" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']
print('$c', round(e['value'],2), 'TFLOP/s', round(e['ms_per_step']*1e3,1), 'us', e['bitwise_equal_to_device_path'])"
done
