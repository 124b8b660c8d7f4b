// Host cost of one mmlttb_minmaxlttb call straight through the C ABI (no
// Python): back-to-back calls on one stream, host time per call and device
// time per call, for the C1 and C3 shapes.  Separates the library's own host
// path from the ctypes/Python layers above it (profiles/r02).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include \
//        -o capi_host_probe tools/probes/capi_host_probe.cu -L paper_2305_00332_b200 -lmmlttb
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include "mmlttb.h"
#ifdef HOSTPROF
extern "C" int mmlttb_hostprof_read(double* acc);
#endif

static void run(long long N, long long n_out, long long r, int ydt) {
  int64_t *x, *out;
  void* y;
  cudaMalloc(&x, N * 8);
  cudaMalloc(&y, N * (ydt == MM_F32 ? 4 : 8));
  cudaMalloc(&out, n_out * 8);
  cudaMemset(y, 0x3c, N * (ydt == MM_F32 ? 4 : 8));
  cudaMemset(x, 0, N * 8);
  const long long wsb = mmlttb_workspace_bytes(MM_OP_MINMAXLTTB, 1, N, n_out, r, ydt);
  void* ws;
  cudaMalloc(&ws, wsb);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto call = [&] {
    int rc = mmlttb_minmaxlttb(x, MM_I64, 0, y, ydt, N, 1, N, n_out, r, out, nullptr, ws, wsb, st);
    if (rc) printf("rc=%d %s\n", rc, mmlttb_last_error());
  };
  for (int i = 0; i < 50; ++i) call();
  cudaStreamSynchronize(st);
  const int n = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto t0 = std::chrono::high_resolution_clock::now();
  cudaEventRecord(e0, st);
  for (int i = 0; i < n; ++i) call();
  auto t1 = std::chrono::high_resolution_clock::now();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("N=%lld n_out=%lld r=%lld %s: host %.2f us/call, device %.2f us/call\n", N, n_out, r,
         ydt == MM_F32 ? "f32" : "f64", std::chrono::duration<double, std::micro>(t1 - t0).count() / n, ms * 1e3 / n);
#ifdef HOSTPROF
  double acc[16];
  mmlttb_hostprof_read(acc);
  printf("   host segments (us/call):");
  for (int i = 1; i < 10; ++i) printf(" %d:%.2f", i, acc[i] / (n + 50));
  printf("\n");
#endif
  // host issue time on an idle stream (sync between calls: no queue back-pressure)
  {
    double tot = 0;
    for (int i = 0; i < 500; ++i) {
      auto a0 = std::chrono::high_resolution_clock::now();
      call();
      auto a1 = std::chrono::high_resolution_clock::now();
      tot += std::chrono::duration<double, std::micro>(a1 - a0).count();
      cudaStreamSynchronize(st);
    }
    printf("   idle-stream host issue %.2f us/call\n", tot / 500);
#ifdef HOSTPROF
    double acc[16];
    mmlttb_hostprof_read(acc);
    printf("   host segments (us/call):");
    for (int i = 1; i < 10; ++i) printf(" %d:%.2f", i, acc[i] / 500);
    printf("\n");
#endif
  }
  // with the deferred status slot armed (the Python path for device inputs)
  mmlttb_status_ring();
  t0 = std::chrono::high_resolution_clock::now();
  cudaEventRecord(e0, st);
  for (int i = 0; i < n; ++i) {
    mmlttb_status_arm();
    call();
  }
  t1 = std::chrono::high_resolution_clock::now();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("   + status_arm: host %.2f us/call, device %.2f us/call\n",
         std::chrono::duration<double, std::micro>(t1 - t0).count() / n, ms * 1e3 / n);
  cudaFree(x); cudaFree(y); cudaFree(out); cudaFree(ws);
}

int main() {
  run(1000000, 1000, 4, MM_F64);
  run(100000000, 2000, 4, MM_F32);
  return 0;
}
