// fused_launch.cu -- fused one-CTA-per-series MinMaxLTTB kernel launch (batches).
#include "fused_impl.cuh"

namespace mmh {

// ---- fused per-series path (batches of medium series) --------------------

bool fused_ok(int64_t B, int64_t N, int64_t n_out, int64_t r_ps, int ydt) {
  static const bool off = env_i64("MMLTTB_NO_FUSED", 0) != 0;  // A/B knob
  const int64_t k = (n_out - 2) * (r_ps / 2);
  return !off && B >= sm_count() && r_ps >= 2 && r_ps <= 8 && N < (1LL << 31) &&
         fused_smem(k, n_out - 2, 8, esize(ydt)) <= FUSED_SMEM_MAX;
}

// SM count of the current device (cached per device; 148, a B200, when none is present)
int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) { (void)cudaGetLastError(); return 148; }
  if (dev < 64) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) return c;
  }
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    n = 148;
  }
  if (dev < 64) cache[dev].store(n, std::memory_order_relaxed);
  return n;
}

int launch_fused_f32(const FusedArgs& fa, int ydt, cudaStream_t st);
int launch_fused_f64(const FusedArgs& fa, int ydt, cudaStream_t st);
int launch_fused_i64(const FusedArgs& fa, int ydt, cudaStream_t st);
int launch_fused_i32(const FusedArgs& fa, int ydt, cudaStream_t st);

int launch_fused(const FusedArgs& fa, int xdt, int ydt, cudaStream_t st) {
  switch (xdt) {
    case MM_F32: return launch_fused_f32(fa, ydt, st);
    case MM_F64: return launch_fused_f64(fa, ydt, st);
    case MM_I64: return launch_fused_i64(fa, ydt, st);
    default: return launch_fused_i32(fa, ydt, st);
  }
}

}  // namespace mmh
