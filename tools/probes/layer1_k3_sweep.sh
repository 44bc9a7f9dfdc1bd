# VGG-16 layer-1 contraction: tile configs (WINO_GEMM = tm,tn,thm,thn,bk,stages,maxreg,ku,noprod,pack)
for g in default 4,8,16,16,8,4,0,8,0,1 4,8,16,16,8,4,168,8,0,1 4,8,16,16,8,3,0,8,0,1 4,8,8,32,8,4,0,8,0,1 8,8,8,16,8,4,0,8,0,1 4,16,16,8,8,4,0,8,0,1 4,8,16,16,8,6,0,8,0,1 8,4,8,32,8,4,0,8,0,1; do
  if [ $g = default ]; then timeout 300 python tools/probes/layer1_k3.py; else WINO_GEMM=$g timeout 300 python tools/probes/layer1_k3.py; fi
done
