// lttb_impl.cuh -- K3 (LTTB) launch templates, instantiated per x dtype in
// lttb_x_{f32,f64,i64,i32}.cu (parallel compilation); dispatch in lttb_launch.cu.
#pragma once
#include "host.cuh"
#include "k3s.cuh"

namespace mmh {

constexpr int64_t JUMP_SMEM_MAX = 200 * 1024;
// buckets per k_lttb_jump shared-memory segment (two byte tables of seg*SMAX)
inline int64_t jump_seg(int64_t k3, int smax) {
  const int64_t cap = (JUMP_SMEM_MAX / (2 * smax)) / 16 * 16;
  return std::min<int64_t>(cap, (k3 + 15) / 16 * 16);
}

// A/B knobs: points in flight per lane in the flat verification (default 8: 26 vs 29 us on
// C2) and means (default 4: 43 vs 45 us) passes
inline int64_t flat_un(bool verify) {
  static const int64_t uv = env_i64("MMLTTB_K3C_VERIFY_UN", 8), um = env_i64("MMLTTB_K3C_MEANS_UN", 4);
  return verify ? uv : um;
}
// chain resolution over transition maps of width W: one CTA per series scans
// the composed maps (a segmented two-kernel version measured no faster)
template <int W>
int launch_chain_scan(LttbArgs a, cudaStream_t st) {
  k_lttb_scan<W, 512, 4><<<(unsigned)a.B, 512, 0, st>>>(a);
  return check_launch("k_lttb_scan");
}

template <int SMAX> int jump_attr() {
  static std::atomic<unsigned long long> attr{0};
  return smem_optin(attr, (const void*)k_lttb_jump<SMAX>, (int)JUMP_SMEM_MAX, "k_lttb_jump");
}

template <int SMAX>
int launch_jump(LttbArgs a, cudaStream_t st) {
  const int64_t k3 = a.n_out - 2;
  int rc = jump_attr<SMAX>();
  if (rc) return rc;
  a.jump_seg = jump_seg(k3, SMAX);
  k_lttb_jump<SMAX><<<(unsigned)a.B, 1024, (size_t)(2 * a.jump_seg * SMAX), st>>>(a);
  return check_launch("k_lttb_jump");
}

template <typename XT, typename YT, int SMAX>
int launch_tables_jump(LttbArgs a, cudaStream_t st) {
  const int64_t k3 = a.n_out - 2;
  a.tab_ld = tab_ld(k3, SMAX);
  dim3 g((unsigned)cdiv(k3, NBB), (unsigned)a.B);
  constexpr int NT = NBB * SMAX < 1024 ? NBB * SMAX : 1024;
  k_lttb_tables<XT, YT, SMAX, NBB><<<g, NT, 0, st>>>(a);
  int rc = check_launch("k_lttb_tables");
  if (rc) return rc;
  if constexpr (SMAX <= 32) {
    return launch_chain_scan<SMAX>(a, st);
  } else {
    return launch_jump<SMAX>(a, st);
  }
}

// K3s (k3s.cuh): the whole large-bucket LTTB of one series in one cooperative
// launch.  MM_ENOTSUP when the shape does not suit it (too few buckets to fill
// the SMs' warps, or a repair state beyond shared memory; MMLTTB_K3S=0, the
// A/B knob): the caller falls back to the K3c kernels.
unsigned long long* k3s_prof_buffer();

template <typename XT, typename YT>
int launch_k3s(LttbArgs a, void* scratch, int2* gmeta, cudaStream_t st) {
  static const bool on = env_i64("MMLTTB_K3S", 1) != 0;
  if (!on) return MM_ENOTSUP;
  const int64_t k3 = a.n_out - 2;
  int dev = 0, nsm = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(MM_ECUDA, "cudaGetDevice");
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // One warp streams a whole bucket, so with fewer than 8 buckets per SM K3s needs
  // narrow buckets: measured on one box (tools/k3s_check.py, 1e7 points): 10,020-point
  // buckets 109 vs 153 us for the K3c kernels, 33,500-point buckets 205 vs 169 us,
  // 100,000-point buckets 389 vs 240 us (A/B knobs MMLTTB_K3S_MINB4: buckets per SM x 4
  // from which the bucket width is not looked at; MMLTTB_K3S_WIDE: widest such bucket)
  static const int64_t minb4 = env_i64("MMLTTB_K3S_MINB4", 32), wide = env_i64("MMLTTB_K3S_WIDE", 16384);
  if (nsm < 1 || nsm > K3S_GMAX || k3 < 2) return MM_ENOTSUP;
  if (4 * k3 < minb4 * nsm && (a.n - 2) / k3 > wide) return MM_ENOTSUP;
  if (((uintptr_t)a.x & 15) || ((uintptr_t)a.y & 15)) return MM_ENOTSUP;  // 16-byte vector loads  // < 8 busy warps per SM: K3c's flat passes win
  auto kern = k_lttb_k3s<XT, YT>;
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, (const void*)kern) != cudaSuccess) return fail(MM_ECUDA, "cudaFuncGetAttributes(k3s)");
  const int64_t G = std::min<int64_t>(nsm, k3);
  const int64_t maxb = cdiv(k3, G) + 1;
  const int64_t dyn = std::max<int64_t>(std::max<int64_t>(up(maxb * K3S_H) + (maxb + 1) * 8 + maxb * 4 + 32 + (G + 32) * K3S_H, repair_smem_bytes(k3)),
                                        (int64_t)K3S_NW * K3S_STAGE_LD * 8);  // phase 2 stages candidates in the same bytes
  if (dyn + (int64_t)fa.sharedSizeBytes > optin) return MM_ENOTSUP;
  static std::atomic<unsigned long long> attr{0};
  if (int rc = smem_optin(attr, (const void*)kern, (int)(optin - fa.sharedSizeBytes), "k_lttb_k3s")) return rc;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, K3S_NT, (size_t)dyn) != cudaSuccess || occ < 1)
    return MM_ENOTSUP;
  K3sArgs ka{};
  ka.G = (int)G;
  ka.maxb = (int)maxb;
  ka.sync = (unsigned*)scratch;  // K3S_SYNC_WORDS counters / flags (fcount among them)
  a.fcount = (int*)(ka.sync + K3S_FCOUNT);
  ka.agg = (unsigned char*)scratch + up(K3S_SYNC_WORDS * 4);
  ka.cpt = (double2*)(ka.agg + up((int64_t)K3S_GMAX * K3S_H));
  ka.chg = (int*)((unsigned char*)ka.cpt + up(k3 * K3S_H * (int64_t)sizeof(double2)));
  // fixed-point re-verification passes (A/B knobs: MMLTTB_K3S_JMIN / _JMAX; JMAX=0: walks only)
  static const int jmin = (int)env_i64("MMLTTB_K3S_JMIN", 8), jmax = (int)env_i64("MMLTTB_K3S_JMAX", 32);
  ka.jmin = jmin;
  ka.jmax = jmax;
  // group summaries for the pruned candidate search / verification (A/B knob MMLTTB_K3S_PRUNE=0)
  static const bool prune = env_i64("MMLTTB_K3S_PRUNE", 1) != 0;
  ka.gmeta = prune ? gmeta : nullptr;
  ka.prof = k3s_prof_buffer();  // tools only (MMLTTB_K3S_PROF=1)
  if (ka.prof) cudaMemsetAsync(ka.prof, 0, (size_t)(K3S_GMAX * 8 + 64) * 8, st);
  if (cudaMemsetAsync(ka.sync, 0, (size_t)K3S_SYNC_WORDS * 4, st) != cudaSuccess) return fail(MM_ECUDA, "memset(k3s)");
  void* args[] = {(void*)&a, (void*)&ka};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)G), dim3(K3S_NT), args, (size_t)dyn, st);
  if (e != cudaSuccess) { (void)cudaGetLastError(); return fail(MM_ECUDA, "k_lttb_k3s: %s", cudaGetErrorString(e)); }
  return check_launch("k_lttb_k3s");
}

// K3c: large buckets (see kernels.cuh): means, hull candidates, candidate
// tables, jump (positions), verification, repair + output
template <typename XT, typename YT, int H>
int launch_lttb_large(LttbArgs a, cudaStream_t st) {
  const int64_t k3 = a.n_out - 2;
  Carve cv{(char*)a.tables, INT64_MAX / 4};
  a.means = cv.take<double2>(a.B * k3);
  a.means_ld = k3;
  a.cand = cv.take<int64_t>(a.B * k3 * HMAX);
  a.cand_ld = k3 * H;
  a.cand_cnt = cv.take<int>(a.B * k3);
  a.tab_ld = tab_ld(k3, H);
  unsigned char* tabs = cv.take<unsigned char>(a.B * tab_ld(k3, HMAX));
  a.pos = cv.take<int64_t>(a.B * (k3 + 2));
  a.pos_ld = k3 + 2;
  a.best = cv.take<int64_t>(a.B * k3);
  a.flag = cv.take<int>(a.B * k3);
  a.yrange = cv.take<double2>(a.B * k3);
  a.best2 = cv.take<int64_t>(a.B * k3);
  a.flist = cv.take<int>(a.B * k3);
  a.fcount = cv.take<int>(a.B);
  a.merr = cv.take<double2>(a.B * k3);
  // affine-x detection in the means pass (A/B knob MMLTTB_K3C_XAFF=0: always load x)
  static const bool xaff_on = env_i64("MMLTTB_K3C_XAFF", 1) != 0;
  a.xaff = cv.take<XAff>(a.B * k3);
  if (!xaff_on) a.xaff = nullptr;
  a.tables = tabs;
  a.cand_cap = (int)env_i64("MMLTTB_K3C_CAND_CAP", H);  // test knob: a poor heuristic must still be exact
  // flat passes (one series with closed-form buckets; A/B knob MMLTTB_K3C_FLAT=0: per-bucket CTAs)
  static const bool flat_on = env_i64("MMLTTB_K3C_FLAT", 1) != 0;
  const bool flat = flat_on && a.B == 1 && !a.bounds && !a.m_dev;
  a.xrange = cv.take<double2>(a.B * k3);
  FlatArgs fl{}, fl_c{};  // fl_c: the candidate pass (16 resident warps per SM instead of 24)
  unsigned* fcnt = nullptr;
  if (flat) {
    const int64_t L = a.n - 2;
    auto plan = [&](FlatArgs& f, int64_t warps) {
      f.W = std::max<int64_t>(1, std::min<int64_t>(warps, cdiv(L, 256)));
      f.E = cdiv(L, f.W);
      f.W = cdiv(L, f.E);
      f.CP = cdiv(cdiv(L, k3), f.E) + 1;
      return f.CP <= flat_cp_max(k3);
    };
    if (!plan(fl, k3c_flat_warps()) || !plan(fl_c, k3c_flat_warps() * 2 / 3)) return fail(MM_ERANGE, "K3c flat partial slots");
    // arrival counters of the three passes, the failed-certification count, the
    // flagged-bucket count and the fix/verify2 grid barrier: one memset
    fcnt = cv.take<unsigned>(3 * k3 + 3);
    fl.ucount = (int*)(fcnt + 3 * k3);
    a.fcount = (int*)(fcnt + 3 * k3 + 1);
    fl.part = cv.take<unsigned char>(k3 * flat_cp_max(k3) * K3C_FLAT_PART);
    fl.ulist = cv.take<int>(k3);
    fl_c.part = fl.part;
    int2* gmeta = cv.take<int2>(std::min<int64_t>(k3, K3S_K3MAX) * K3S_GCAP);
    const int rk = k3 <= K3S_K3MAX ? launch_k3s<XT, YT>(a, fl.part, gmeta, st) : MM_ENOTSUP;
    if (rk != MM_ENOTSUP) return rk;  // otherwise: the multi-kernel K3c below
    if (cudaMemsetAsync(fcnt, 0, (size_t)(3 * k3 + 3) * sizeof(unsigned), st) != cudaSuccess)
      return fail(MM_ECUDA, "memset");
  }
  const unsigned flat_grid = (unsigned)cdiv(fl.W, 8);
  // any-order means + error bounds (one bandwidth-bound pass; the exact
  // argmaxes certify against the bounds)
  static const int cforce = (int)env_i64("MMLTTB_K3C_CERT_FORCE", 0);  // test knob: every certification fails
  a.cert_force = cforce;
  if (flat) {
    fl.cnt = fcnt;
#ifdef MMLTTB_AB  // tuning build only: points in flight per lane (4: 43 vs 45 us at 8 on C2)
    if (flat_un(false) == 8) k_lttb_means_flat<XT, YT, 8><<<dim3(flat_grid, 1), 256, 0, st>>>(a, fl);
    else
#endif
    k_lttb_means_flat<XT, YT, 4><<<dim3(flat_grid, 1), 256, 0, st>>>(a, fl);
  } else {
    const dim3 g((unsigned)k3, (unsigned)a.B);
#ifdef MMLTTB_AB
    static const int64_t mnt = env_i64("MMLTTB_K3C_MEANS_NT", 256);
    if (mnt == 128) k_lttb_means_approx<XT, YT, 128, 8><<<g, 128, 0, st>>>(a);
    else
#endif
    k_lttb_means_approx<XT, YT, 256, 4><<<g, 256, 0, st>>>(a);
  }
  int rc = check_launch("k_lttb_means");
  if (rc) return rc;
  {
    k_lttb_dircand<XT, YT, H, H / 2, 64><<<dim3((unsigned)k3, (unsigned)a.B), 64, 0, st>>>(a);
    if ((rc = check_launch("k_lttb_dircand"))) return rc;
  }
  k_lttb_ctables<XT, YT, H><<<dim3((unsigned)cdiv(k3, 1024 / H), (unsigned)a.B), 1024, 0, st>>>(a);
  if ((rc = check_launch("k_lttb_ctables"))) return rc;
  if ((rc = launch_chain_scan<H>(a, st))) return rc;
  if (!flat && cudaMemsetAsync(a.fcount, 0, (size_t)a.B * sizeof(int), st) != cudaSuccess)
    return fail(MM_ECUDA, "memset");
  if (flat) {
    fl.cnt = fcnt + 2 * k3;
#ifdef MMLTTB_AB  // (8 in flight: 26 vs 29 us at 4 on C2)
    if (flat_un(true) == 4) k_lttb_verify_flat<XT, YT, 4><<<dim3(flat_grid, 1), 256, 0, st>>>(a, fl);
    else
#endif
    k_lttb_verify_flat<XT, YT, 8><<<dim3(flat_grid, 1), 256, 0, st>>>(a, fl);
    if ((rc = check_launch("k_lttb_verify_flat"))) return rc;
    k_lttb_verify_fix<XT, YT, 256><<<dim3((unsigned)sm_count(), 1), 256, 0, st>>>(a, fl);
    if ((rc = check_launch("k_lttb_verify_fix"))) return rc;
  } else {
#ifdef MMLTTB_AB  // (64 threads per bucket: 30 vs 37.5 us at 256 on C2)
    static const int64_t vnt = env_i64("MMLTTB_K3C_VERIFY_NT", 64);
    if (vnt == 256) k_lttb_verify<XT, YT, 256><<<dim3((unsigned)k3, (unsigned)a.B), 256, 0, st>>>(a);
    else
#endif
    k_lttb_verify<XT, YT, 64><<<dim3((unsigned)k3, (unsigned)a.B), 64, 0, st>>>(a);
    if ((rc = check_launch("k_lttb_verify"))) return rc;
  }
  {
    k_lttb_verify2<XT, YT, 256><<<dim3((unsigned)sm_count(), (unsigned)a.B), 256, 0, st>>>(a);
    if ((rc = check_launch("k_lttb_verify2"))) return rc;
  }
  // chain state staged in shared memory when it fits (A/B knob MMLTTB_K3C_REPAIR_SMEM=0: global)
  static const bool rsm = env_i64("MMLTTB_K3C_REPAIR_SMEM", 1) != 0;
  constexpr int64_t RSMEM_MAX = 200 * 1024;
  const int64_t rbytes = repair_smem_bytes(k3);
  if (rsm && rbytes <= RSMEM_MAX) {
    auto kern = k_lttb_repair_smem<XT, YT, 512>;
    static std::atomic<unsigned long long> attr{0};
    if ((rc = smem_optin(attr, (const void*)kern, (int)RSMEM_MAX, "k_lttb_repair_smem"))) return rc;
    kern<<<(unsigned)a.B, 512, (size_t)rbytes, st>>>(a);
    return check_launch("k_lttb_repair_smem");
  }
#ifdef MMLTTB_AB  // (512 threads: 22.1 vs 24.4 us at 1024 on C2)
  static const int64_t rp = env_i64("MMLTTB_K3C_REPAIR_NT", 512);
  if (rp == 1024) k_lttb_repair<XT, YT, 1024><<<(unsigned)a.B, 1024, 0, st>>>(a);
  else
#endif
  k_lttb_repair<XT, YT, 512><<<(unsigned)a.B, 512, 0, st>>>(a);
  return check_launch("k_lttb_repair");
}

// buckets of <= 64 points (lttb_small_x_*.cu)
template <typename XT, typename YT>
int launch_lttb_small_t(LttbArgs a, int64_t s, cudaStream_t st) {
  if (a.B > 65535) return fail(MM_ERANGE, "batch > 65535 series");
  {
    switch (smax_for(s)) {
      case 4: return launch_tables_jump<XT, YT, 4>(a, st);
      case 8: return launch_tables_jump<XT, YT, 8>(a, st);
      case 16: return launch_tables_jump<XT, YT, 16>(a, st);
      case 32: return launch_tables_jump<XT, YT, 32>(a, st);
      default: return launch_tables_jump<XT, YT, 64>(a, st);
    }
  }
}

template <typename XT>
int launch_lttb_small_x(LttbArgs a, int ydt, int64_t s, cudaStream_t st) {
  if (ydt == MM_F32) return launch_lttb_small_t<XT, float>(a, s, st);
  if (ydt == MM_F64) return launch_lttb_small_t<XT, double>(a, s, st);
  return fail(MM_EINVAL, "y dtype");
}

// larger buckets: K3s / K3c (lttb_x_*.cu)
template <typename XT>
int launch_lttb_large_x(LttbArgs a, int ydt, cudaStream_t st) {
  if (a.B > 65535) return fail(MM_ERANGE, "batch > 65535 series");
  if (ydt == MM_F32) return launch_lttb_large<XT, float, 16>(a, st);
  if (ydt == MM_F64) return launch_lttb_large<XT, double, 16>(a, st);
  return fail(MM_EINVAL, "y dtype");
}

}  // namespace mmh
