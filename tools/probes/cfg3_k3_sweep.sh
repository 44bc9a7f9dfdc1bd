# cfg3 (m=6) linear contraction: tile configs (WINO_GEMM = tm,tn,thm,thn,bk,stages,maxreg,ku,noprod,pack)
for g in default 8,8,16,8,32,2,0,16,0,1 8,8,16,8,32,3,0,16,0,1 8,8,16,8,64,2,0,16,0,1 8,8,16,8,16,3,0,16,0,1 8,8,8,16,32,2,0,16,0,1; do
  if [ $g = default ]; then timeout 300 python tools/probes/cfg3_k3.py; else WINO_GEMM=$g timeout 300 python tools/probes/cfg3_k3.py; fi
done
