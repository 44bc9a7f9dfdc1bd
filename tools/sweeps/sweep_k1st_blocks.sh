# minimum blocks per SM (register cap) of the K1 kernels: bulk-staged (WINO_K1ST_BLOCKS) and global gather (WINO_K1_BLOCKS)
show='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d["shape"], "K1+K2 %.1f us  K1 %.1f us (%.0f GB/s)  crc %08x" % (d["real_transforms_us"], d["real_input_us"], d["real_input_gbs"], d["V_crc32"]))'
for sh in "256,512,14,512 6" "256,512,28,512 6" "256,256,56,256 6" "64,256,28,256 6" "32,128,28,128 2"; do
  set -- $sh
  for nb in 0 6 7 8; do
    echo -n "k1st_blocks=$nb "; WINO_K1ST_BLOCKS=$nb python tools/xform_bench.py --shape $1 --m $2 | python -c "$show"
  done
done
for sh in "256,128,112,128 6" "256,64,224,64 6"; do
  set -- $sh
  for nb in 0 5 6; do
    echo -n "k1_blocks=$nb "; WINO_K1_BLOCKS=$nb python tools/xform_bench.py --shape $1 --m $2 | python -c "$show"
  done
done
