# K1 channels-per-thread / K4 filters-per-thread sweep (transform micro-benchmark)
for v in 1 2 4 8; do
  echo "== CPT=KPT=$v"
  WINO_CPT=$v WINO_KPT=$v python tools/xform_bench.py --shape 32,128,28,128 --m 2
  WINO_CPT=$v WINO_KPT=$v python tools/xform_bench.py --shape 64,256,28,256 --m 6
  WINO_CPT=$v WINO_KPT=$v python tools/xform_bench.py --shape 8,64,56,64 --m 4
done
