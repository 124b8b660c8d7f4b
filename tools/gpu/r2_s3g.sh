mkdir -p gpurun_out/s3g
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -o /tmp/chp tools/probes/capi_host_probe.cu -L paper_2305_00332_b200 -lmmlttb
for v in "1 1" "0 1" "1 0"; do set -- $v
  echo "MMLTTB_K23_PDL=$1 MMLTTB_K1_TILES=0 MMLTTB_K23=$2" >> gpurun_out/s3g/capi.log
  MMLTTB_K23_PDL=$1 MMLTTB_K1_TILES=0 MMLTTB_K23=$2 LD_LIBRARY_PATH=paper_2305_00332_b200 timeout 120 /tmp/chp >> gpurun_out/s3g/capi.log 2>&1
done
