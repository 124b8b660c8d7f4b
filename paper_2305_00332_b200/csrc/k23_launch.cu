// k23_launch.cu -- K23 (k23.cuh): compaction + LTTB of one series' preselected
// points in one cooperative launch; the single-series minmaxlttb tail.
#include "host.cuh"
#include "k23.cuh"

namespace mmh {

unsigned long long* k3s_prof_buffer();  // lttb_launch.cu (tools: MMLTTB_K3S_PROF=1)

// CTAs: enough for the compaction tiles (<= K23_NT * ITEMS sub-buckets each)
// and for the transition-table work (k3 * SMAX^2 area evaluations, ~32 per thread)
inline void k23_plan(int64_t k, int64_t k3, int smax, int nsm, int64_t& G, int& items, int64_t& TS) {
  const int64_t gt = cdiv(k3 * smax * smax, (int64_t)K23_NT * 32);
  G = std::max<int64_t>(cdiv(k, K23_NT), gt);
  G = std::min<int64_t>({G, (int64_t)nsm, k3});
  G = std::max<int64_t>(G, 1);
  TS = cdiv(k, G);
  items = 1;
}

bool k23_ok(int64_t B, int64_t k, int64_t n_out, int64_t r_ps) {
  static const bool on = env_i64("MMLTTB_K23", 1) != 0;  // A/B knob: 0 = K2 + K3a kernels / k_post_smem
  const int smax = smax_for(r_ps);
  return on && B == 1 && smax > 0 && smax <= 32 && n_out - 2 >= 1 && k <= (int64_t)sm_count() * K23_NT;
}

int64_t k23_ws() { return up((int64_t)K23_GMAX * 4) + up((int64_t)K23_GMAX * 32); }  // stat slots + aggregates

template <typename YT, int SMAX>
int launch_k23_t(K23Args a, int64_t r_ps, cudaStream_t st) {
  const int64_t k3 = a.n_out - 2;
  const int64_t maxb = cdiv(k3, a.G) + 1;
  const int64_t np = (maxb + 2) * r_ps + 4;
  const int64_t dyn = 24 * np + 16 * maxb + 2 * maxb * SMAX + 64;
  auto kern = k_k23<YT, SMAX, 1>;
  static std::atomic<unsigned long long> attr{0};
  if (dyn > 48 * 1024) {
    if (int rc = smem_optin(attr, (const void*)kern, (int)std::min<int64_t>(dyn, 200 * 1024), "k_k23")) return rc;
    if (dyn > 200 * 1024) return MM_ENOTSUP;
  }
  a.maxb = (int)maxb;
  a.prof = k3s_prof_buffer();
  if (a.prof) cudaMemsetAsync(a.prof, 0, (size_t)K3S_GMAX * 8 * 8, st);
  // cooperative (grid barriers) and a programmatic dependent of the previous
  // kernel on the stream (K1): K23's CTAs are scheduled as K1's retire and wait
  // in griddepcontrol.wait (A/B knob MMLTTB_K23_PDL=0: plain cooperative launch)
  static const bool pdl = env_i64("MMLTTB_K23_PDL", 1) != 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)a.G);
  cfg.blockDim = dim3(K23_NT);
  cfg.dynamicSmemBytes = (size_t)dyn;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeCooperative;
  attrs[0].val.cooperative = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess && pdl) {  // (PDL with a cooperative launch refused: plain cooperative)
    (void)cudaGetLastError();
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  if (e != cudaSuccess) { (void)cudaGetLastError(); return fail(MM_ECUDA, "k_k23: %s", cudaGetErrorString(e)); }
  return check_launch("k_k23");
}

template <typename YT>
int launch_k23_y(K23Args a, int64_t r_ps, cudaStream_t st) {
  switch (smax_for(r_ps)) {
    case 4: return launch_k23_t<YT, 4>(a, r_ps, st);
    case 8: return launch_k23_t<YT, 8>(a, r_ps, st);
    case 16: return launch_k23_t<YT, 16>(a, r_ps, st);
    default: return launch_k23_t<YT, 32>(a, r_ps, st);
  }
}

// a.sync: K23_STAT zeroed words (the caller merges the zeroing with its own);
// a.stat: k23_ws() bytes of workspace (status slots, then the aggregates)
int launch_k23(K23Args a, int xdt, int ydt, int64_t r_ps, cudaStream_t st) {
  const int64_t k3 = a.n_out - 2;
  int64_t G, TS;
  int items;
  k23_plan(a.k, k3, smax_for(r_ps), sm_count(), G, items, TS);
  a.G = (int)G;
  a.TS = (int)TS;
  a.xdt = xdt;
  a.agg = (unsigned char*)a.stat + up((int64_t)K23_GMAX * 4);
  return ydt == MM_F32 ? launch_k23_y<float>(a, r_ps, st) : launch_k23_y<double>(a, r_ps, st);
}

}  // namespace mmh
