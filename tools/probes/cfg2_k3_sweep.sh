# cfg2 contraction: tile configs (WINO_GEMM = tm,tn,thm,thn,bk,stages,maxreg,ku,noprod,pack)
for g in default 8,8,16,8,16,4,0,16,0,1 8,8,16,8,16,3,0,16,0,1 8,8,16,8,16,6,0,16,0,1 8,8,8,16,16,4,0,16,0,1 8,8,16,8,32,3,0,16,0,1 8,8,16,16,16,3,0,16,0,1 8,8,16,8,8,8,0,8,0,1 8,8,16,8,16,4,128,16,0,1; do
  if [ $g = default ]; then timeout 300 python tools/probes/cfg2_k3.py; else WINO_GEMM=$g timeout 300 python tools/probes/cfg2_k3.py; fi
done
