// Where does the C2 means kernel lose time vs the fp64 add-chain floor?
// 1999 one-warp CTAs, each an in-order sum of 5005 doubles (x and y chains
// on lanes 0/1), like k_lttb_means_staged.  Variants:
//  A: chains on register data only (no memory)
//  B: chains fed from shared memory filled once (no global traffic)
//  C: global -> registers -> shared tile -> chains (the staged kernel's loop)
//  D: C without the y-range fmin/fmax in the stash
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_probe chain_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NB = 1999, LEN = 5005, TILE = 256, PER = TILE / 32;

__device__ __forceinline__ double i2d_fast(long long v) {
  // exact int64 -> double without the conversion unit for |v| < 2^51:
  // (1.5*2^52 + v) is exactly representable; subtracting 1.5*2^52 is exact
  if (v >= -(1LL << 51) && v < (1LL << 51))
    return __dsub_rn(__longlong_as_double(0x4338000000000000LL + v), 6755399441055744.0);
  return __ll2double_rn(v);
}

template <int V>
__global__ void __launch_bounds__(32) kern(const long long* xs, const double* ys, double* out) {
  __shared__ double s_t[2][2][TILE];
  const int lane = threadIdx.x;
  const long long lo = (long long)blockIdx.x * LEN, hi = lo + LEN;
  double acc = 0.0;
  const int which = lane & 1;
  if (V == 0) {
    double a = 1.0 + lane, b = 0.5;
    if (lane < 2) {
#pragma unroll 8
      for (int i = 0; i < LEN; ++i) acc = __dadd_rn(acc, (i & 1) ? a : b);
    }
  } else if (V == 1) {
    for (int i = lane; i < TILE; i += 32) { s_t[0][0][i] = (double)i; s_t[0][1][i] = 0.5 * i; }
    __syncwarp();
    if (lane < 2) {
      const double* src = s_t[0][which];
      for (int t = 0; t < LEN; t += TILE) {
        const int n = LEN - t < TILE ? LEN - t : TILE;
        int i = 0;
        for (; i + 8 <= n; i += 8) {
          double v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = src[i + q];
#pragma unroll
          for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v[q]);
        }
        for (; i < n; ++i) acc = __dadd_rn(acc, src[i]);
      }
    }
  } else if (V == 4) {
    for (int i = lane; i < TILE; i += 32) { s_t[0][0][i] = (double)i; s_t[0][1][i] = 0.5 * i; }
    __syncwarp();
    if (lane < 2) {
      const double* src = s_t[0][which];
      for (int t = 0; t < LEN; t += TILE) {
        const int n = LEN - t < TILE ? LEN - t : TILE;
        int i = 0;
        if (n >= 16) {
          double v0[8], v1[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v0[q] = src[q];
          for (; i + 24 <= n; i += 16) {
#pragma unroll
            for (int q = 0; q < 8; ++q) v1[q] = src[i + 8 + q];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v0[q]);
#pragma unroll
            for (int q = 0; q < 8; ++q) v0[q] = src[i + 16 + q];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v1[q]);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v0[q]);
          i += 8;
        }
        for (; i < n; ++i) acc = __dadd_rn(acc, src[i]);
      }
    }
  } else {
    long long rx[PER];
    double ry[PER];
    double ymn = 1e300, ymx = -1e300;
    auto fetch = [&](long long t0) {
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const long long j = t0 + q * 32 + lane;
        rx[q] = j < hi ? xs[j] : 0;
        ry[q] = j < hi ? ys[j] : 0.0;
      }
    };
    auto stash = [&](int buf, long long t0) {
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        s_t[buf][0][q * 32 + lane] = V == 7 ? i2d_fast(rx[q]) : (double)rx[q];
        s_t[buf][1][q * 32 + lane] = ry[q];
        if (V == 2 && t0 + q * 32 + lane < hi) { ymn = fmin(ymn, ry[q]); ymx = fmax(ymx, ry[q]); }
      }
    };
    fetch(lo);
    stash(0, lo);
    __syncwarp();
    int buf = 0;
    for (long long t0 = lo; t0 < hi; t0 += TILE) {
      const bool more = t0 + TILE < hi;
      if (more) fetch(t0 + TILE);
      if (lane < 2) {
        const int n = (int)(hi - t0 < TILE ? hi - t0 : TILE);
        const double* src = s_t[buf][which];
        int i = 0;
        for (; i + 8 <= n; i += 8) {
          double v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = src[i + q];
#pragma unroll
          for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v[q]);
        }
        for (; i < n; ++i) acc = __dadd_rn(acc, src[i]);
      }
      __syncwarp();
      if (more && V != 6) stash(buf ^ 1, t0 + TILE);
      if (V == 6) { acc += (double)rx[0] * 0.0 + ry[0] * 0.0; }
      __syncwarp();
      buf ^= 1;
    }
    if (V == 2) acc += ymn + ymx;
  }
  if (lane < 2) out[blockIdx.x * 2 + lane] = acc;
}

constexpr int NR = 4;
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bwait(unsigned long long* b, unsigned par) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(su(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void barrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory");
}
// F: warp 1 streams tiles (global -> regs -> shared ring, y range), warp 0's lanes 0/1 run the chains
__global__ void __launch_bounds__(64) kernF(const long long* xs, const double* ys, double* out) {
  __shared__ double ring[NR][2][TILE];
  __shared__ unsigned long long full[NR], empty[NR];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long lo = (long long)blockIdx.x * LEN, hi = lo + LEN;
  const int ntiles = (LEN + TILE - 1) / TILE;
  if (threadIdx.x == 0)
    for (int i = 0; i < NR; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(su(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[i])));
    }
  __syncthreads();
  if (warp == 1) {
    double ymn = 1e300, ymx = -1e300;
    long long rx[PER];
    double ry[PER];
    auto fetch = [&](int t) {
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const long long j = lo + (long long)t * TILE + q * 32 + lane;
        rx[q] = j < hi ? xs[j] : 0;
        ry[q] = j < hi ? ys[j] : 0.0;
      }
    };
    fetch(0);
    for (int t = 0; t < ntiles; ++t) {
      const int st = t % NR;
      if (t >= NR) bwait(&empty[st], (unsigned)((t / NR - 1) & 1));
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        ring[st][0][q * 32 + lane] = (double)rx[q];
        ring[st][1][q * 32 + lane] = ry[q];
        if (lo + (long long)t * TILE + q * 32 + lane < hi) { ymn = fmin(ymn, ry[q]); ymx = fmax(ymx, ry[q]); }
      }
      barrive(&full[st]);  // 32 arrivals complete the phase
      if (t + 1 < ntiles) fetch(t + 1);
    }
    if (lane == 0) out[NB * 2 + blockIdx.x] = ymn + ymx;
  } else if (lane < 2) {
    const int which = lane;
    double acc = 0.0;
    for (int t = 0; t < ntiles; ++t) {
      const int st = t % NR;
      bwait(&full[st], (unsigned)((t / NR) & 1));
      const int n = (int)(hi - lo - (long long)t * TILE < TILE ? hi - lo - (long long)t * TILE : TILE);
      const double* src = ring[st][which];
      int i = 0;
      for (; i + 8 <= n; i += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = src[i + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v[q]);
      }
      for (; i < n; ++i) acc = __dadd_rn(acc, src[i]);
      __syncwarp(0x3u);
      if (lane == 0) barrive(&empty[st]);
    }
    out[blockIdx.x * 2 + which] = acc;
  }
}

// J: cp.async ring NR2 tiles deep (no register staging); chain lanes read the
// raw tiles: lane 0 converts x with the exact magic add, lane 1 reads y
constexpr int NR2 = 4;
__global__ void __launch_bounds__(32) kernJ(const long long* xs, const double* ys, double* out) {
  __shared__ __align__(16) long long sx[NR2][TILE];
  __shared__ __align__(16) double sy[NR2][TILE];
  const int lane = threadIdx.x;
  const long long lo = (long long)blockIdx.x * LEN, hi = lo + LEN;
  const int ntiles = (LEN + TILE - 1) / TILE;
  auto issue = [&](int t) {
    if (t < ntiles) {
      const int st = t % NR2;
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const long long j = lo + (long long)t * TILE + q * 32 + lane;
        if (j < hi) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su(&sx[st][q * 32 + lane])), "l"(xs + j) : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su(&sy[st][q * 32 + lane])), "l"(ys + j) : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int t = 0; t < NR2 - 1; ++t) issue(t);
  double acc = 0.0, ymn = 1e300, ymx = -1e300;
  for (int t = 0; t < ntiles; ++t) {
    issue(t + NR2 - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(NR2 - 1) : "memory");
    __syncwarp();
    const int st = t % NR2;
    const int n = (int)(hi - lo - (long long)t * TILE < TILE ? hi - lo - (long long)t * TILE : TILE);
    if (lane == 0) {
      const long long* src = sx[st];
      int i = 0;
      for (; i + 8 <= n; i += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = i2d_fast(src[i + q]);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v[q]);
      }
      for (; i < n; ++i) acc = __dadd_rn(acc, i2d_fast(src[i]));
    } else if (lane == 1) {
      const double* src = sy[st];
      int i = 0;
      for (; i + 8 <= n; i += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = src[i + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = __dadd_rn(acc, v[q]);
      }
      for (; i < n; ++i) acc = __dadd_rn(acc, src[i]);
    }
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (q * 32 + lane < n) { const double v = sy[st][q * 32 + lane]; ymn = fmin(ymn, v); ymx = fmax(ymx, v); }
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (lane < 2) out[blockIdx.x * 2 + lane] = acc + (ymn + ymx) * 0.0;
}

int main() {
  long long* x;
  double *y, *out;
  cudaMalloc(&x, (size_t)NB * LEN * 8);
  cudaMalloc(&y, (size_t)NB * LEN * 8);
  cudaMalloc(&out, NB * 3 * 8);
  cudaMemset(x, 0, (size_t)NB * LEN * 8);
  cudaMemset(y, 0, (size_t)NB * LEN * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"A register chains", "B smem-fed chains", "C staged (with y range)", "D staged (no y range)",
                         "B2 smem chains, 16 ahead", "F loader warp + chain warp", "H loads, no stash",
                         "G staged, magic int->double", "J cp.async ring, raw tiles"};
  for (int rep = 0; rep < 2; ++rep)
    for (int v = 0; v < 9; ++v) {
      cudaEventRecord(a);
      for (int r = 0; r < 10; ++r) {
        if (v == 0) kern<0><<<NB, 32>>>(x, y, out);
        if (v == 1) kern<1><<<NB, 32>>>(x, y, out);
        if (v == 2) kern<2><<<NB, 32>>>(x, y, out);
        if (v == 3) kern<3><<<NB, 32>>>(x, y, out);
        if (v == 4) kern<4><<<NB, 32>>>(x, y, out);
        if (v == 5) kernF<<<NB, 64>>>(x, y, out);
        if (v == 6) kern<6><<<NB, 32>>>(x, y, out);
        if (v == 7) kern<7><<<NB, 32>>>(x, y, out);
        if (v == 8) kernJ<<<NB, 32>>>(x, y, out);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%-28s %7.1f us per launch (%s)\n", names[v], ms * 100.0f, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
