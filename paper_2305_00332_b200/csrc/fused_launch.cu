// fused_launch.cu -- fused one-CTA-per-series MinMaxLTTB kernel launch (batches).
#include "fused_impl.cuh"

namespace mmh {

// ---- fused per-series path (batches of medium series) --------------------
constexpr int64_t FUSED_MIN_B = 148;

bool fused_ok(int64_t B, int64_t N, int64_t n_out, int64_t r_ps, int ydt) {
  static const bool off = env_i64("MMLTTB_NO_FUSED", 0) != 0;  // A/B knob
  const int64_t k = (n_out - 2) * (r_ps / 2);
  return !off && B >= FUSED_MIN_B && r_ps >= 2 && r_ps <= 8 && N < (1LL << 31) &&
         fused_smem(k, n_out - 2, 8, esize(ydt)) <= FUSED_SMEM_MAX;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
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
