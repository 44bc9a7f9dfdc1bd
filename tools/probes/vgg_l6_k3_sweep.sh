# VGG-16 layer-6 pairwise contraction: tile configs (WINO_GEMM = tm,tn,thm,thn,bk,stages,maxreg,ku,noprod,pack)
for g in 4,4,16,16,64,2,168,8,0,1 4,4,16,16,64,3,168,8,0,1 4,4,16,16,128,2,168,8,0,1 4,4,16,16,64,2,0,8,0,1 4,4,16,16,64,2,168,16,0,1 4,4,16,16,48,2,168,8,0,1; do
  if [ $g = default ]; then timeout 300 python tools/probes/vgg_l6_k3.py; else WINO_GEMM=$g timeout 300 python tools/probes/vgg_l6_k3.py; fi
done
