mkdir -p gpurun_out/s3i
rm -rf /tmp/hp && mkdir /tmp/hp && cp -r paper_2305_00332_b200 include /tmp/hp/ && rm -f /tmp/hp/paper_2305_00332_b200/libmmlttb.so
(cd /tmp/hp && MMLTTB_NVCC_EXTRA="-DMMLTTB_HOSTPROF" python -c "import sys; sys.path.insert(0,'.'); from paper_2305_00332_b200 import build; build.build(force=True)") > gpurun_out/s3i/build.log 2>&1
nvcc -O3 -std=c++17 -DHOSTPROF -gencode arch=compute_100a,code=sm_100a -I include -o /tmp/chp tools/probes/capi_host_probe.cu -L /tmp/hp/paper_2305_00332_b200 -lmmlttb >> gpurun_out/s3i/build.log 2>&1
MMLTTB_K1_TILES=0 LD_LIBRARY_PATH=/tmp/hp/paper_2305_00332_b200 timeout 120 /tmp/chp > gpurun_out/s3i/capi.log 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/lp tools/probes/launch_probe.cu && timeout 120 /tmp/lp > gpurun_out/s3i/launch_probe.log 2>&1
