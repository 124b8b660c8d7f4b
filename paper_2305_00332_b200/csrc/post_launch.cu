// post_launch.cu -- single-CTA K2+K3 (k_post_smem / k_post_fused) and cooperative K2+K3a launch.
#include "host.cuh"

namespace mmh {

// ---- fused K2+K3 (single / few series) -----------------------------------
constexpr int64_t POST_SMEM_MAX = 100 * 1024;
constexpr int64_t POST_SMEM2_MAX = 200 * 1024;

bool post_ok(int64_t k, int64_t n_out, int64_t r_ps) {
  static const bool off = env_i64("MMLTTB_NO_POST_FUSED", 0) != 0;  // A/B knob
  // one CTA's latency chains beat two extra launches only for small k
  // (measured: k = 1996 24 us vs 24 us + a launch; k = 3996 41 us vs 24 us;
  // with the set staged in shared memory, k_post_smem, C1 takes 14.6 us)
  return !off && k <= 2048 && smax_for(r_ps) > 0 && smax_for(r_ps) <= 8 &&
         post_smem(n_out - 2, smax_for(r_ps)) <= POST_SMEM_MAX;
}

template <typename XT, typename YT, int SMAX>
int launch_post_t(const PostArgs& pa, int64_t B, cudaStream_t st) {
  static const bool global_staging = env_i64("MMLTTB_POST_GLOBAL", 0) != 0;  // A/B knob
  const int64_t sm2 = post_smem2(pa.n_out - 2, SMAX, pa.cap);
  if (!global_staging && sm2 <= POST_SMEM2_MAX) {  // preselected set staged in shared memory
    static bool attr2 = false;
    if (!attr2) {
      if (cudaFuncSetAttribute(k_post_smem<XT, YT, SMAX, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)POST_SMEM2_MAX) != cudaSuccess)
        return fail(MM_ECUDA, "cudaFuncSetAttribute(k_post_smem)");
      attr2 = true;
    }
    k_post_smem<XT, YT, SMAX, 1024><<<(unsigned)B, 1024, (size_t)sm2, st>>>(pa);
    return check_launch("k_post_smem");
  }
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_post_fused<XT, YT, SMAX, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)POST_SMEM_MAX) != cudaSuccess)
      return fail(MM_ECUDA, "cudaFuncSetAttribute(k_post_fused)");
    attr = true;
  }
  k_post_fused<XT, YT, SMAX, 1024><<<(unsigned)B, 1024, (size_t)post_smem(pa.n_out - 2, SMAX), st>>>(pa);
  return check_launch("k_post_fused");
}

template <typename XT, typename YT>
int launch_post_y(const PostArgs& pa, int64_t B, int smax, cudaStream_t st) {
  return smax <= 4 ? launch_post_t<XT, YT, 4>(pa, B, st) : launch_post_t<XT, YT, 8>(pa, B, st);
}

int launch_post(const PostArgs& pa, int64_t B, int xdt, int ydt, int smax, cudaStream_t st) {
  const bool y32 = ydt == MM_F32;
  switch (xdt) {
    case MM_F32: return y32 ? launch_post_y<float, float>(pa, B, smax, st) : launch_post_y<float, double>(pa, B, smax, st);
    case MM_F64: return y32 ? launch_post_y<double, float>(pa, B, smax, st) : launch_post_y<double, double>(pa, B, smax, st);
    case MM_I64:
      return y32 ? launch_post_y<long long, float>(pa, B, smax, st) : launch_post_y<long long, double>(pa, B, smax, st);
    default: return y32 ? launch_post_y<int, float>(pa, B, smax, st) : launch_post_y<int, double>(pa, B, smax, st);
  }
}

// ---- cooperative K2+K3a ----------------------------------------------------
template <typename XT, typename YT, int SMAX>
int launch_coop_t(PairArgs pa, LttbArgs la, int64_t B, cudaStream_t st, bool* launched) {
  constexpr int NT = PAIR_NT, IT = PAIR_ITEMS;
  auto fn = k_post_coop<XT, YT, SMAX, NT, IT>;
  static int cap = -1;
  if (cap < 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, NT, 0);
    cap = sms * per;
  }
  int64_t ntiles = std::max<int64_t>(1, cdiv(pa.nb, NT * IT));
  if (ntiles * B > cap || B > 65535) { *launched = false; return MM_OK; }
  *launched = true;
  la.tab_ld = tab_ld(la.n_out - 2, SMAX);
  void* args[] = {(void*)&pa, (void*)&la, (void*)&ntiles};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)fn, dim3((unsigned)ntiles, (unsigned)B), dim3(NT),
                                                    args, 0, st);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (e != cudaSuccess) return fail(MM_ECUDA, "k_post_coop: %s", cudaGetErrorString(e));
  return MM_OK;
}

template <typename XT, typename YT>
int launch_coop_y(PairArgs pa, LttbArgs la, int64_t B, int smax, cudaStream_t st, bool* launched) {
  return smax <= 4 ? launch_coop_t<XT, YT, 4>(pa, la, B, st, launched)
                   : launch_coop_t<XT, YT, 8>(pa, la, B, st, launched);
}

// Try the cooperative K2+K3a; *launched = false when it does not apply.
int launch_coop(PairArgs pa, LttbArgs la, int64_t B, int smax, cudaStream_t st, bool* launched) {
  // opt-in (MMLTTB_COOP=1): measured neutral-to-slower than the separate
  // launches on B200 (c3_1e9 28 vs 26 us, c3 1e8 27 vs 24 us) -- the fixed
  // cost is the phases' dependent memory round trips, not the launches
  static const bool on = env_i64("MMLTTB_COOP", 0) != 0;
  *launched = false;
  if (!on || smax <= 0 || smax > 8) return MM_OK;
  const bool y32 = pa.ydt == MM_F32;
  switch (pa.xdt) {
    case MM_F32:
      return y32 ? launch_coop_y<float, float>(pa, la, B, smax, st, launched)
                 : launch_coop_y<float, double>(pa, la, B, smax, st, launched);
    case MM_F64:
      return y32 ? launch_coop_y<double, float>(pa, la, B, smax, st, launched)
                 : launch_coop_y<double, double>(pa, la, B, smax, st, launched);
    case MM_I64:
      return y32 ? launch_coop_y<long long, float>(pa, la, B, smax, st, launched)
                 : launch_coop_y<long long, double>(pa, la, B, smax, st, launched);
    default:
      return y32 ? launch_coop_y<int, float>(pa, la, B, smax, st, launched)
                 : launch_coop_y<int, double>(pa, la, B, smax, st, launched);
  }
}


}  // namespace mmh
