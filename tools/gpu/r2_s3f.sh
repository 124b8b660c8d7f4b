mkdir -p gpurun_out/s3f
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/lp tools/probes/launch_probe.cu && timeout 120 /tmp/lp > gpurun_out/s3f/launch_probe.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/rp tools/probes/read_probe.cu && timeout 300 /tmp/rp 400 4000 > gpurun_out/s3f/read_probe2.log 2>&1
