nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false -diag-suppress 550 -o gpurun_out/packed_probe tools/probes/packed_probe.cu && ./gpurun_out/packed_probe
