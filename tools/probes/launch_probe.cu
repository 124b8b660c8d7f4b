// Host-side cost of the launch forms the library uses (per call, back to back,
// no sync): <<<>>>, cudaLaunchKernelEx plain / PDL / cooperative / both,
// cudaMemsetAsync, cudaGraphLaunch of a 3-node graph.  Context for the C1
// per-call overhead (profiles/r02).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o launch_probe launch_probe.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_small(int* p) {
  if (threadIdx.x == 0 && p) atomicAdd(p, 1);
}

template <typename F>
double host_us(F f, int n = 500) {  // issue time on an idle stream (sync between calls)
  for (int i = 0; i < 50; ++i) f();
  cudaDeviceSynchronize();
  double tot = 0;
  for (int i = 0; i < n; ++i) {
    auto t0 = std::chrono::high_resolution_clock::now();
    f();
    auto t1 = std::chrono::high_resolution_clock::now();
    tot += std::chrono::duration<double, std::micro>(t1 - t0).count();
    cudaDeviceSynchronize();
  }
  return tot / n;
}

int main() {
  int* d;
  cudaMalloc(&d, 4096);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto ex = [&](int grid, bool coop, bool pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (coop) { at[na].id = cudaLaunchAttributeCooperative; at[na].val.cooperative = 1; ++na; }
    if (pdl) {
      at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, k_small, d);
  };
  printf("<<<16,256>>>                     %6.2f us\n", host_us([&] { k_small<<<16, 256, 0, st>>>(d); }));
  printf("<<<3000,256>>>                   %6.2f us\n", host_us([&] { k_small<<<3000, 256, 0, st>>>(d); }));
  printf("LaunchKernelEx plain (16)        %6.2f us\n", host_us([&] { ex(16, false, false); }));
  printf("LaunchKernelEx PDL (16)          %6.2f us\n", host_us([&] { ex(16, false, true); }));
  printf("LaunchKernelEx coop (16)         %6.2f us\n", host_us([&] { ex(16, true, false); }));
  printf("LaunchKernelEx coop+PDL (16)     %6.2f us\n", host_us([&] { ex(16, true, true); }));
  printf("cudaMemsetAsync 1 KB             %6.2f us\n", host_us([&] { cudaMemsetAsync(d, 0, 1024, st); }));
  printf("memset + <<<>>> + coop+PDL       %6.2f us\n", host_us([&] {
    cudaMemsetAsync(d, 0, 1024, st);
    k_small<<<3000, 256, 0, st>>>(d);
    ex(16, true, true);
  }));
  cudaGraph_t g;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  cudaMemsetAsync(d, 0, 1024, st);
  k_small<<<3000, 256, 0, st>>>(d);
  ex(16, true, true);
  cudaStreamEndCapture(st, &g);
  cudaGraphExec_t ge;
  cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  printf("graph instantiate: %s\n", cudaGetErrorString(e));
  printf("cudaGraphLaunch (3 nodes)        %6.2f us\n", host_us([&] { cudaGraphLaunch(ge, st); }));
  // device time per call, back to back
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto dev_us = [&](auto f) {
    for (int i = 0; i < 20; ++i) f();
    cudaEventRecord(e0, st);
    for (int i = 0; i < 500; ++i) f();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3 / 500;
  };
  printf("device/call memset+k+coop+PDL    %6.2f us\n", dev_us([&] {
    cudaMemsetAsync(d, 0, 1024, st);
    k_small<<<3000, 256, 0, st>>>(d);
    ex(16, true, true);
  }));
  printf("device/call memset+k+PDL         %6.2f us\n", dev_us([&] {
    cudaMemsetAsync(d, 0, 1024, st);
    k_small<<<3000, 256, 0, st>>>(d);
    ex(16, false, true);
  }));
  printf("device/call k+k                  %6.2f us\n", dev_us([&] {
    k_small<<<3000, 256, 0, st>>>(d);
    k_small<<<16, 256, 0, st>>>(d);
  }));
  printf("device/call graph                %6.2f us\n", dev_us([&] { cudaGraphLaunch(ge, st); }));
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
