// post_launch.cu -- single-CTA K2+K3 (k_post_smem / k_post_fused).
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
    static std::atomic<unsigned long long> attr2{0};
    if (int rc = smem_optin(attr2, (const void*)k_post_smem<XT, YT, SMAX, 1024>, (int)POST_SMEM2_MAX, "k_post_smem"))
      return rc;
    k_post_smem<XT, YT, SMAX, 1024><<<(unsigned)B, 1024, (size_t)sm2, st>>>(pa);
    return check_launch("k_post_smem");
  }
  static std::atomic<unsigned long long> attr{0};
  if (int rc = smem_optin(attr, (const void*)k_post_fused<XT, YT, SMAX, 1024>, (int)POST_SMEM_MAX, "k_post_fused"))
    return rc;
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

}  // namespace mmh
