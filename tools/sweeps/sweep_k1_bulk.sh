#!/bin/bash
# K1 from bulk-copied image planes in shared memory (WINO_K1=bulk) vs the global-memory gather
for sh in "64,256,28,256 6" "32,128,28,128 2" "32,512,14,512 4" "256,512,14,512 6" "256,512,28,512 6" "256,256,56,256 6" "8,64,56,64 4"; do
  set -- $sh
  for k1 in gather bulk; do
    echo -n "K1=$k1 "; WINO_K1=$k1 python tools/xform_bench.py --shape $1 --m $2 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['shape'], 'm', d['m'], 'K1+K2 %.1f us  K1 %.1f us (%.0f GB/s)  crc %08x' % (d['real_transforms_us'], d['real_input_us'], d['real_input_gbs'], d['V_crc32']))"
  done
done
