for sh in "256,128,112,128 6" "256,64,112,128 6"; do
  set -- $sh
  for k1 in gather bulk bulk120; do
    echo -n "K1=$k1 "; WINO_K1=$k1 python tools/xform_bench.py --shape $1 --m $2 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['shape'], 'm', d['m'], 'K1+K2 %.1f us  K1 %.1f us (%.0f GB/s)  crc %08x' % (d['real_transforms_us'], d['real_input_us'], d['real_input_gbs'], d['V_crc32']))"
  done
done
