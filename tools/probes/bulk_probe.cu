// Streaming-read throughput of cp.async.bulk (1-D TMA) on B200: persistent
// CTAs stream disjoint contiguous ranges through an NS-slot shared-memory
// ring (full/empty mbarriers); the consumer warps only touch one word per
// slot.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_probe bulk_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ int g_wait_mode;
__device__ __forceinline__ void wait_(unsigned long long* b, unsigned par) {
  const int mode = g_wait_mode;
  if (mode == 0) {
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(su32(b)), "r"(par) : "memory");
  } else if (mode == 1) {
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(su32(b)), "r"(par) : "memory");
  } else {
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n @!p bra W_%=;\n}" ::"r"(su32(b)), "r"(par), "r"(mode) : "memory");
  }
}

__global__ void probe(const char* src, long long per_cta, int T, int NS, unsigned* sink, int SPLIT) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ unsigned long long full[16], empty[16];
  const int NW = blockDim.x / 32, warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const char* base = src + (long long)blockIdx.x * per_cta;
  const long long tiles = per_cta / T;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(NW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long pq = 0;
  // producer role rotates: tile q is issued by lane 0 of warp q % NW (ROT)
  // or always by warp 0 (!ROT)
  auto issue = [&](long long q2) {
    const int st = q2 % NS;
    if (q2 >= NS) wait_(&empty[st], (unsigned)((q2 / NS - 1) & 1));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(T) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(ring + (long long)st * T)), "l"(base + q2 * T), "r"(T), "r"(su32(&full[st])) : "memory");
  };
  auto owner = [&](long long q2) { return SPLIT ? (int)(q2 % NW) : 0; };
  for (long long q2 = 0; q2 < NS && q2 < tiles; ++q2)
    if (warp == owner(q2) && lane == 0) issue(q2);
  unsigned acc = 0;
  for (long long q = 0; q < tiles; ++q) {
    const int st = q % NS;
    wait_(&full[st], (unsigned)((q / NS) & 1));
    acc += ((const unsigned*)(ring + (long long)st * T))[(warp * 32 + lane) % (T / 4)];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
    if (q + NS < tiles && warp == owner(q + NS) && lane == 0) issue(q + NS);
  }
  if (acc == 0x12345678) sink[0] = acc;
}

int main(int argc, char** argv) {
  const long long total = 16LL << 30;
  char* src;
  unsigned* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 4);
  cudaMemset(src, 1, total);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  int Ts[] = {4096, 8192, 16384, 32768};
  int NSs[] = {2, 4, 8};
  int NTs[] = {256};
  int SPs[] = {0, 1};
  int modes[] = {0};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode : modes) {
  cudaMemcpyToSymbol(g_wait_mode, &mode, sizeof(int));
  for (int SP : SPs)
  for (int NT : NTs)
    for (int T : Ts)
      for (int NS : NSs) {
        const long long smem = (long long)T * NS;
        if (smem > 220 * 1024) continue;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, probe, NT, smem);
        if (per_sm < 1) continue;
        for (int cps = 1; cps <= per_sm && cps <= 4; cps *= 2) {
          const int grid = 148 * cps;
          long long per_cta = (total / grid) / T * T;
          probe<<<grid, NT, smem>>>(src, per_cta, T, NS, sink, SP);
          cudaEventRecord(a);
          for (int r = 0; r < 3; ++r) probe<<<grid, NT, smem>>>(src, per_cta, T, NS, sink, SP);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          const double gbs = 3.0 * per_cta * grid / (ms / 1e3) / 1e9;
          printf("mode=%d SPLIT=%2d NT=%d T=%6d NS=%2d ctas/sm=%d inflight/sm=%4lldKB  %7.1f GB/s  %s\n", mode, SP, NT, T, NS, cps,
                 (long long)(NS - 1) * T * cps / 1024, gbs, cudaGetErrorString(cudaGetLastError()));
        }
      }
  }
  return 0;
}
