// fused_impl.cuh -- launch templates of the fused one-CTA-per-series kernel,
// instantiated per x dtype in fused_x_{f32,f64,i64,i32}.cu; dispatch in fused_launch.cu.
#pragma once
#include "host.cuh"

namespace mmh {

constexpr int64_t FUSED_SMEM_MAX = 110 * 1024;

template <typename XT, typename YT, int SMAX, int NT, int MINB, int U, int LDV = 3, bool KR = true>
int launch_fused_v(const FusedArgs& fa, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_mmlttb_fused<XT, YT, SMAX, NT, MINB, U, LDV, KR>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FUSED_SMEM_MAX) != cudaSuccess)
      return fail(MM_ECUDA, "cudaFuncSetAttribute(k_mmlttb_fused)");
    attr = true;
  }
  const int64_t k = (fa.n_out - 2) * (fa.r_ps / 2);
  const size_t smem = (size_t)fused_smem(k, fa.n_out - 2, SMAX, (int)sizeof(YT));
  k_mmlttb_fused<XT, YT, SMAX, NT, MINB, U, LDV, KR><<<(unsigned)fa.B, NT, smem, st>>>(fa);
  return check_launch("k_mmlttb_fused");
}

// TMA-fed persistent fused kernel (fused.cuh): ring of `stages` slots of
// ~MMLTTB_TMA_TILE bytes (whole sub-buckets per slot).  Returns 1 (not
// launched) when the rows are not 16-byte aligned or no CTA fits.
template <typename XT, typename YT, int SMAX, int NT, int MINB, int G>
int launch_fused_tma_v(FusedArgs fa, cudaStream_t st) {
  static const int64_t tile_target = env_i64("MMLTTB_TMA_TILE", 65536);
  static const int64_t stages = std::min<int64_t>(8, std::max<int64_t>(2, env_i64("MMLTTB_TMA_STAGES", 2)));
  constexpr int64_t ys = sizeof(YT);
  if (((uintptr_t)fa.y & 15) || (fa.B > 1 && (fa.y_ld * ys) & 15)) return 1;
  const int64_t k = (fa.n_out - 2) * (fa.r_ps / 2);
  const int64_t maxlen = cdiv(fa.N - 2, k) + 1;
  constexpr int64_t R = NT / G;  // tile = whole multiples of R sub-buckets (one per lane group per round)
  const int64_t tb = std::max<int64_t>(1, std::min<int64_t>(cdiv(k, R), tile_target / (maxlen * ys * R))) * R;
  fa.tile_buckets = tb;
  fa.tile_bytes = cdiv(tb * maxlen * ys + 256, 128) * 128;  // + line widening at both ends
  fa.stages = stages;
  fa.dbg = env_i64("MMLTTB_TMA_DEBUG", 0);
  const int64_t p_bytes = cdiv(fused_smem(k, fa.n_out - 2, SMAX, (int)ys), 128) * 128;
  const int64_t smem = p_bytes + stages * fa.tile_bytes;
  constexpr int64_t SMEM_CAP = 227 * 1024 - 2048;  // opt-in max minus static shared memory
  if (smem > SMEM_CAP) return 1;
  auto kern = k_mmlttb_fused_tma<XT, YT, SMAX, NT, MINB, G>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_CAP) != cudaSuccess)
      return fail(MM_ECUDA, "cudaFuncSetAttribute(k_mmlttb_fused_tma)");
    attr = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, (size_t)smem) != cudaSuccess || per_sm < 1)
    return 1;
  const int64_t grid = std::min<int64_t>(fa.B, (int64_t)per_sm * sm_count());
  kern<<<(unsigned)grid, NT, (size_t)smem, st>>>(fa);
  return check_launch("k_mmlttb_fused_tma");
}

template <typename XT, typename YT, int SMAX>
int launch_fused_t(const FusedArgs& fa, cudaStream_t st) {
  // opt-in (>= 0): the TMA-fed persistent kernel -- streams at 7.4 TB/s on
  // its own but its phase-1 math is latency-bound at the 8 warps that fit
  // beside the ring on C4, so the per-group kernel stays the default
  static const int64_t tv = env_i64("MMLTTB_TMA_VARIANT", -1);
  if (tv >= 0) {
    int rc;
    switch (tv) {
      case 1: rc = launch_fused_tma_v<XT, YT, SMAX, 512, 1, 16>(fa, st); break;
      case 2: rc = launch_fused_tma_v<XT, YT, SMAX, 256, 1, 16>(fa, st); break;
      case 3: rc = launch_fused_tma_v<XT, YT, SMAX, 256, 1, 32>(fa, st); break;
      case 4: rc = launch_fused_tma_v<XT, YT, SMAX, 512, 1, 32>(fa, st); break;
      case 5: rc = launch_fused_tma_v<XT, YT, SMAX, 256, 2, 8>(fa, st); break;
      default: rc = launch_fused_tma_v<XT, YT, SMAX, 256, 1, 8>(fa, st); break;
    }
    if (rc != 1) return rc;
  }
  static const int64_t v = env_i64("MMLTTB_FUSED_VARIANT", 0);  // tuning knob (tools/)
  switch (v) {  // tools/fused_sweep.sh on B200 (variant 0 = default)
    case 1: return launch_fused_v<XT, YT, SMAX, 512, 2, 4>(fa, st);
    case 2: return launch_fused_v<XT, YT, SMAX, 384, 3, 4>(fa, st);
    case 3: return launch_fused_v<XT, YT, SMAX, 256, 4, 4>(fa, st);
    case 4: return launch_fused_v<XT, YT, SMAX, 512, 3, 2>(fa, st);
    case 5: return launch_fused_v<XT, YT, SMAX, 512, 2, 8>(fa, st);
    case 6: return launch_fused_v<XT, YT, SMAX, 512, 3, 4, 2, false>(fa, st);
    case 7: return launch_fused_v<XT, YT, SMAX, 512, 2, 8, 2, true>(fa, st);
    case 8: return launch_fused_v<XT, YT, SMAX, 384, 3, 8, 2, false>(fa, st);
    // measured best on C4: normal-policy loads, winners re-read from L1/L2
    default: return launch_fused_v<XT, YT, SMAX, 512, 2, 8, 2, false>(fa, st);
  }
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
