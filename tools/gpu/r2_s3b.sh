mkdir -p gpurun_out/s3b
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/read_probe tools/probes/read_probe.cu && timeout 300 /tmp/read_probe 8 100 400 1000 4000 > gpurun_out/s3b/read_probe.log 2>&1
timeout 300 python tools/host_breakdown_probe.py > gpurun_out/s3b/host_breakdown.log 2>&1
timeout 300 python tools/host_overhead_probe.py > gpurun_out/s3b/host_overhead.log 2>&1
