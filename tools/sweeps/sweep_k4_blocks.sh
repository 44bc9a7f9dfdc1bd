# minimum blocks per SM (register cap) of the gather K4 kernels (WINO_K4_BLOCKS)
show='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d["shape"], "K4 %.1f us (%.0f GB/s)" % (d["real_output_us"], d["real_output_gbs"]))'
for sh in "256,512,14,512 6" "256,512,28,512 6" "256,256,56,256 6" "256,128,112,128 6" "64,256,28,256 6"; do
  set -- $sh
  for nb in 0 6 7; do
    echo -n "k4_blocks=$nb "; WINO_K4_BLOCKS=$nb python tools/xform_bench.py --shape $1 --m $2 | python -c "$show"
  done
done
