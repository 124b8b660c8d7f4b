// Dependent-chain latency of fp64 add (DADD) and of a shared-memory-fed
// chain on B200.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dadd_probe dadd_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(const double* v, int n, double* out, long long* cyc) {
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, v[i & 1023]);
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}

__global__ void chain_reg(double a, int n, double* out, long long* cyc) {
  double acc = 0.0, b = a * 0.5;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, (i & 1) ? a : b);
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}

__global__ void chain_smem(const double* v, int n, double* out, long long* cyc) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = v[i & 1023];
  __syncthreads();
  if (threadIdx.x) return;
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i + 8 <= n; i += 8) {
    double w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = s[(i + q) & 4095];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, w[q]);
  }
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}

__global__ void chain_many(double a, int n, double* out, long long* cyc) {
  // lanes 0/1 of every warp run a dependent DADD chain, like k_lttb_means_staged
  double acc = 0.0, b = a * 0.5;
  long long t0 = clock64();
  if ((threadIdx.x & 31) < 2) {
#pragma unroll 16
    for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, (i & 1) ? a : b);
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) { out[blockIdx.x] = acc; if (blockIdx.x == 0) cyc[0] = t1 - t0; }
}

int main() {
  double *v, *out;
  long long* cyc;
  cudaMalloc(&v, 1024 * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  cudaMemset(v, 0, 1024 * 8);
  long long c;
  const int n = 5000;
  for (int r = 0; r < 2; ++r) {
    chain_reg<<<1, 1>>>(1.0, n, out, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("register chain: %.2f cycles/add\n", (double)c / n);
    chain_smem<<<1, 128>>>(v, n, out, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("smem-fed chain (8 loads then 8 adds): %.2f cycles/add\n", (double)c / n);
    chain<<<1, 1>>>(v, n, out, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("global-fed chain (L1 hits): %.2f cycles/add\n", (double)c / n);
  }
  double* out2;
  cudaMalloc(&out2, 8 * 8192);
  for (int ctas : {1, 148, 148 * 4, 148 * 8, 148 * 14, 148 * 28}) {
    chain_many<<<ctas, 32>>>(1.0, n, out2, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%5d one-warp CTAs (%.1f warps/SM), lanes 0/1 chain: %.2f cycles/add\n", ctas, ctas / 148.0, (double)c / n);
  }
  return 0;
}
