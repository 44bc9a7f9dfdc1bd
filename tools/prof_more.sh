# ncu --set full captures of the non-default kernels (pairwise / tensor-core / fused tcf / VGG layer)
for spec in "cfg3_m6_mixed_pw exact" "cfg3_m6 tc_bf16" "cfg2 tcf_bf16" "cfg3_m6 ffma"; do
  set -- $spec
  python bench.py --config $1 --contraction $2 --ncu --steps 2 --warmup 3 > gpurun_out/ncu_pre_$1_$2.log 2>&1 || continue
  ncu --set full --clock-control none --import-source on -k regex:"wino_contract|tc_contract|wino_tcf|wino_transforms|wino_output" \
      -s 4 -c 3 -o gpurun_out/prof_$1_$2 python bench.py --config $1 --contraction $2 --ncu --steps 2 --warmup 3 \
      > gpurun_out/ncu_$1_$2.log 2>&1
done
echo done
