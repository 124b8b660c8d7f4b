// fused_impl.cuh -- launch templates of the fused one-CTA-per-series kernel,
// instantiated per x dtype in fused_x_{f32,f64,i64,i32}.cu; dispatch in fused_launch.cu.
#pragma once
#include "host.cuh"

namespace mmh {

constexpr int64_t FUSED_SMEM_MAX = 110 * 1024;

template <typename XT, typename YT, int SMAX, int NT, int MINB, int U, int LDV = 3, bool KR = true>
int launch_fused_v(const FusedArgs& fa, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  if (int rc = smem_optin(attr, (const void*)k_mmlttb_fused<XT, YT, SMAX, NT, MINB, U, LDV, KR>, (int)FUSED_SMEM_MAX,
                          "k_mmlttb_fused"))
    return rc;
  const int64_t k = (fa.n_out - 2) * (fa.r_ps / 2);
  const size_t smem = (size_t)fused_smem(k, fa.n_out - 2, SMAX, (int)sizeof(YT));
  k_mmlttb_fused<XT, YT, SMAX, NT, MINB, U, LDV, KR><<<(unsigned)fa.B, NT, smem, st>>>(fa);
  return check_launch("k_mmlttb_fused");
}

template <typename XT, typename YT, int SMAX>
int launch_fused_t(const FusedArgs& fa, cudaStream_t st) {
#ifdef MMLTTB_AB  // tuning build only (tools/fused_sweep.sh: MMLTTB_NVCC_EXTRA=-DMMLTTB_AB)
  static const int64_t v = env_i64("MMLTTB_FUSED_VARIANT", 0);
  switch (v) {  // tools/fused_sweep.sh on B200 (variant 0 = default)
    case 1: return launch_fused_v<XT, YT, SMAX, 512, 2, 4>(fa, st);
    case 2: return launch_fused_v<XT, YT, SMAX, 384, 3, 4>(fa, st);
    case 3: return launch_fused_v<XT, YT, SMAX, 256, 4, 4>(fa, st);
    case 4: return launch_fused_v<XT, YT, SMAX, 512, 3, 2>(fa, st);
    case 5: return launch_fused_v<XT, YT, SMAX, 512, 2, 8>(fa, st);
    case 6: return launch_fused_v<XT, YT, SMAX, 512, 3, 4, 2, false>(fa, st);
    case 7: return launch_fused_v<XT, YT, SMAX, 512, 2, 8, 2, true>(fa, st);
    case 8: return launch_fused_v<XT, YT, SMAX, 384, 3, 8, 2, false>(fa, st);
    default: break;
  }
#endif
  // measured best on C4: normal-policy loads, winners re-read from L1/L2
  return launch_fused_v<XT, YT, SMAX, 512, 2, 8, 2, false>(fa, st);
}

template <typename XT, typename YT>
int launch_fused_y(const FusedArgs& fa, cudaStream_t st) {
  return fa.r_ps <= 4 ? launch_fused_t<XT, YT, 4>(fa, st) : launch_fused_t<XT, YT, 8>(fa, st);
}

template <typename XT>
int launch_fused_x(const FusedArgs& fa, int ydt, cudaStream_t st) {
  return ydt == MM_F32 ? launch_fused_y<XT, float>(fa, st) : launch_fused_y<XT, double>(fa, st);
}

}  // namespace mmh
