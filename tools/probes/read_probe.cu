// Read-only HBM stream probe: what a pure read of S bytes costs on this B200 at
// the sizes K1 sees (C3: 400 MB, headline: 4 GB), for the access shapes K1 can
// use.  Context for K1's fixed cost at mid sizes (DESIGN.md §7 item 3).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o read_probe read_probe.cu
//   ./read_probe [MB ...]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldef(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// 32-byte (256-bit) per-thread load, sm_100
struct u8x32 { unsigned a[8]; };
__device__ __forceinline__ u8x32 ld32(const uint4* p) {
  u8x32 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.a[0]), "=r"(r.a[1]), "=r"(r.a[2]), "=r"(r.a[3]), "=r"(r.a[4]), "=r"(r.a[5]),
                 "=r"(r.a[6]), "=r"(r.a[7]) : "l"(p));
  return r;
}

// mode 3: like mode 0 with 32-byte loads (U per lane per round)
template <int U>
__global__ void __launch_bounds__(256) k_range32(const uint4* p, long long nvec, long long per_warp, unsigned* sink) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  long long v0 = w * per_warp, v1 = v0 + per_warp;  // in 32-byte units
  if (v1 > nvec / 2) v1 = nvec / 2;
  unsigned acc = 0;
  for (long long v = v0; v < v1; v += 32 * U) {
    u8x32 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = v + u * 32 + lane;
      if (i < v1) r[u] = ld32(p + 2 * i); else for (int q = 0; q < 8; ++q) r[u].a[q] = 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      for (int q = 0; q < 8; ++q) acc ^= r[u].a[q];
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// mode 0: one contiguous range per warp (K1 flat's shape), U vectors per lane per round
template <int U>
__global__ void __launch_bounds__(256) k_range(const uint4* p, long long nvec, long long per_warp, unsigned* sink) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  long long v0 = w * per_warp, v1 = v0 + per_warp;
  if (v1 > nvec) v1 = nvec;
  unsigned acc = 0;
  for (long long v = v0; v < v1; v += 32 * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = v + u * 32 + lane;
      r[u] = i < v1 ? ldef(p + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// mode 4: static ranges over the first `stat` vectors, then chunks of `chunk`
// vectors handed out by an atomic ticket (tail balancing)
template <int U>
__global__ void __launch_bounds__(256) k_range_dyn(const uint4* p, long long nvec, long long per_warp, long long stat,
                                                   long long chunk, unsigned* ticket, unsigned* sink) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  unsigned acc = 0;
  long long v0 = w * per_warp, v1 = v0 + per_warp;
  if (v1 > stat) v1 = stat;
  for (;;) {
    for (long long v = v0; v < v1; v += 32 * U) {
      uint4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long i = v + u * 32 + lane;
        r[u] = i < v1 ? ldef(p + i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
    }
    unsigned c = 0;
    if (lane == 0) c = atomicAdd(ticket, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    v0 = stat + (long long)c * chunk;
    if (v0 >= nvec) break;
    v1 = v0 + chunk < nvec ? v0 + chunk : nvec;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// mode 1: grid-stride (every round, all warps read one contiguous window)
template <int U>
__global__ void __launch_bounds__(256) k_stride(const uint4* p, long long nvec, unsigned* sink) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long T = (long long)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (long long v = t; v < nvec; v += T * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = v + u * T;
      r[u] = i < nvec ? ldef(p + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// mode 2: one tile per CTA, many CTAs (no persistence)
template <int U>
__global__ void __launch_bounds__(256) k_tiles(const uint4* p, long long nvec, unsigned* sink) {
  const long long v0 = blockIdx.x * (long long)256 * U;
  unsigned acc = 0;
  uint4 r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long i = v0 + u * 256 + threadIdx.x;
    r[u] = i < nvec ? ldef(p + i) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) acc ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
  if (acc == 0x12345678u) sink[0] = acc;
}

int main(int argc, char** argv) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long maxmb = 4000;
  uint4* p;
  unsigned* sink;
  cudaMalloc(&p, maxmb * 1000000LL);
  cudaMalloc(&sink, 64);
  cudaMemset(p, 1, maxmb * 1000000LL);
  void* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  long long sizes[8] = {8, 400, 4000};
  int ns = 3;
  if (argc > 1) { ns = 0; for (int i = 1; i < argc && ns < 8; ++i) sizes[ns++] = atoll(argv[i]); }
  for (int si = 0; si < ns; ++si) {
    const long long bytes = sizes[si] * 1000000LL, nvec = bytes / 16;
    auto run = [&](const char* name, auto launch) {
      float best = 1e30f, sum = 0;
      const int reps = 20;
      for (int r = -3; r < reps; ++r) {
        cudaMemsetAsync(flush, r & 0xff, 256 << 20);  // evict L2
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 0) { sum += ms; if (ms < best) best = ms; }
      }
      cudaError_t e = cudaGetLastError();
      printf("%5lld MB  %-34s mean %8.2f us  best %8.2f us  %7.1f GB/s (mean)  %s\n", sizes[si], name,
             sum / reps * 1e3, best * 1e3, bytes / (sum / reps * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
    };
    for (int wps : {16, 24, 32, 48, 64}) {
      const long long warps = (long long)nsm * wps;
      const long long per = (nvec + warps - 1) / warps;
      char nm[64];
      snprintf(nm, 64, "range U=8 warps/SM=%d", wps);
      run(nm, [&] { k_range<8><<<(unsigned)(warps / 8), 256>>>(p, nvec, per, sink); });
    }
    for (int wps : {24, 32, 64}) {
      const long long warps = (long long)nsm * wps;
      const long long per = (nvec + warps - 1) / warps;
      char nm[64];
      snprintf(nm, 64, "range U=4 warps/SM=%d", wps);
      run(nm, [&] { k_range<4><<<(unsigned)(warps / 8), 256>>>(p, nvec, per, sink); });
    }
    for (int wps : {16, 24, 32}) {
      const long long warps = (long long)nsm * wps;
      const long long per = (nvec / 2 + warps - 1) / warps;
      char nm[64];
      snprintf(nm, 64, "range32B U=4 warps/SM=%d", wps);
      run(nm, [&] { k_range32<4><<<(unsigned)(warps / 8), 256>>>(p, nvec, per, sink); });
      snprintf(nm, 64, "range32B U=8 warps/SM=%d", wps);
      run(nm, [&] { k_range32<8><<<(unsigned)(warps / 8), 256>>>(p, nvec, per, sink); });
    }
    for (int pct : {70, 85, 95}) {
      for (long long ch : {1024LL, 4096LL}) {
        const long long warps = (long long)nsm * 24;
        const long long stat = nvec * pct / 100;
        const long long per = (stat + warps - 1) / warps;
        char nm[64];
        snprintf(nm, 64, "range+dyn %d%% chunk %lldKB", pct, ch * 16 / 1024);
        run(nm, [&] {
          cudaMemsetAsync(sink + 8, 0, 4);
          k_range_dyn<8><<<(unsigned)(warps / 8), 256>>>(p, nvec, per, stat, ch, sink + 8, sink);
        });
      }
    }
    for (int wps : {24, 32, 64}) {
      char nm[64];
      snprintf(nm, 64, "stride U=8 warps/SM=%d", wps);
      run(nm, [&] { k_stride<8><<<(unsigned)(nsm * wps / 8), 256>>>(p, nvec, sink); });
    }
    run("tiles U=8 (32 KB per CTA)", [&] { k_tiles<8><<<(unsigned)((nvec + 2047) / 2048), 256>>>(p, nvec, sink); });
    run("tiles U=16 (64 KB per CTA)", [&] { k_tiles<16><<<(unsigned)((nvec + 4095) / 4096), 256>>>(p, nvec, sink); });
    run("empty launch", [&] { k_tiles<1><<<1, 32>>>(p, 0, sink); });
  }
  return 0;
}
