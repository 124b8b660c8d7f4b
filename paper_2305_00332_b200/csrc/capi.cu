// capi.cu -- host dispatch behind include/mmlttb.h (extern "C", no torch).
//
// Each entry validates its O(1) arguments defensively (the Python layer has
// already raised the reference's exception classes in the reference's order),
// carves the caller's workspace, and enqueues 1-4 kernels on the caller's
// stream.  Nothing here synchronises the host.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <array>
#include <string>
#include <vector>

#include "../../include/mmlttb.h"
#include "kernels.cuh"
#include "fused.cuh"
#include "raster.cuh"

using namespace mm;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

std::atomic<int64_t> g_launches{0};

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return MM_OK;
}

// Stage timer: events recorded on the caller's stream at K1|K2|K3 boundaries
// of the fused entries (bench.py reads per-kernel device time from these).
struct StageTimer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::array<cudaEvent_t, 4>> calls;
  std::array<cudaEvent_t, 4> cur{};
};
thread_local StageTimer g_timer;

void stage_mark(cudaStream_t st, int i) {
  if (!g_timer.on) return;
  if (g_timer.used == g_timer.pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    g_timer.pool.push_back(e);
  }
  cudaEvent_t e = g_timer.pool[g_timer.used++];
  cudaEventRecord(e, st);
  g_timer.cur[i] = e;
  if (i == 3) g_timer.calls.push_back(g_timer.cur);
}

constexpr int64_t ALIGN = 256;
inline int64_t up(int64_t v) { return (v + ALIGN - 1) / ALIGN * ALIGN; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int esize(int dt) { return (dt == MM_F32 || dt == MM_I32) ? 4 : 8; }
inline bool ydt_ok(int dt) { return dt == MM_F32 || dt == MM_F64; }
inline bool xdt_ok(int dt) { return dt >= MM_F32 && dt <= MM_I32; }

// workspace bump allocator over the caller's buffer
struct Carve {
  char* p;
  int64_t left;
  bool ok = true;
  template <typename T> T* take(int64_t count) {
    const int64_t bytes = up(count * (int64_t)sizeof(T));
    if (bytes > left) { ok = false; return nullptr; }
    T* r = reinterpret_cast<T*>(p);
    p += bytes;
    left -= bytes;
    return r;
  }
};

// ---- K1 planning --------------------------------------------------------
struct ExPlan {
  int64_t C, chunk, Cmax;
  int64_t E = 0, Ws = 0, CP = 0;  // flat mode (E > 0): elements/warp, warps/series, partial stride
};

// Chunks per bucket: enough warps for ~4 waves over 148 SMs x 32 resident
// warps, never a chunk under MIN_CHUNK elements; buckets of <= 4096 points
// are one item each (8-lane groups).  Large buckets of closed-form partitions
// use the flat split (k_extrema_flat): equal element ranges per warp.
constexpr int64_t SMALL_BUCKET = 4096;  // elements: <= this -> one 8-lane group per bucket

int64_t env_i64(const char* name, int64_t dflt) {
  const char* e = getenv(name);  // tuning knobs for tools/*.sh only
  return e ? atoll(e) : dflt;
}

ExPlan plan_extrema(int64_t buckets_total, int64_t max_bucket, int ydt, int64_t B = 0, bool closed_form = false) {
  // tuned on B200 (tools/plan_sweep.sh): ~4 waves of 148 SMs x 32 resident
  // warps, chunks of >= 4096 float32 elements
  static const int64_t want = env_i64("MMLTTB_K1_WANT_WARPS", 148LL * 128);
  static const int64_t minc32 = env_i64("MMLTTB_K1_MIN_CHUNK", 4096);
  // flat split: one wave of 148 SMs x 24 resident warps (80 regs), two for
  // very long series (tools/flat_sweep.sh)
  static const int64_t flat_env = env_i64("MMLTTB_K1_FLAT_WARPS", -1);
  const int64_t min_chunk = ydt == MM_F32 ? minc32 : minc32 / 2;
  ExPlan p;
  const int64_t nb_ = B > 0 ? buckets_total / B : 0;
  const int64_t flat_warps = flat_env >= 0 ? flat_env : (nb_ * max_bucket > 400000000LL ? 148LL * 48 : 148LL * 24);
  if (closed_form && B > 0 && max_bucket > SMALL_BUCKET && flat_warps > 0) {
    const int64_t nb = nb_;
    p.Ws = std::max<int64_t>(1, flat_warps / B);
    p.E = std::max<int64_t>(min_chunk, cdiv(nb * max_bucket, p.Ws));
    p.Ws = cdiv(nb * max_bucket, p.E);
    p.CP = cdiv(max_bucket, p.E) + 1;
    p.C = 1;
    p.chunk = p.E;
    p.Cmax = p.CP;
    return p;
  }
  p.Cmax = std::max<int64_t>(1, std::min<int64_t>(256, cdiv(want, std::max<int64_t>(1, buckets_total))));
  p.C = max_bucket <= SMALL_BUCKET ? 1 : std::max<int64_t>(1, std::min<int64_t>(p.Cmax, cdiv(max_bucket, min_chunk)));
  p.chunk = cdiv(max_bucket, p.C);
  return p;
}

// K1 buffers for nbt = B*nb buckets
int64_t ex_ws(int64_t nbt, const ExPlan& p) {
  int64_t b = up(nbt * (int64_t)sizeof(Ext)) + up(nbt);
  if (p.Cmax > 1) b += up(nbt * p.Cmax * (int64_t)sizeof(Partial)) + up(nbt * 4);
  return b;
}

bool carve_ex(Carve& cv, int64_t nbt, const ExPlan& p, ExArgs& a) {
  a.E = p.E;
  a.Ws = p.Ws;
  a.CP = p.CP;
  a.ext = cv.take<Ext>(nbt);
  a.cnt8 = cv.take<unsigned char>(nbt);
  a.part = nullptr;
  a.arrivals = nullptr;
  if (p.Cmax > 1) {
    a.part = cv.take<Partial>(nbt * p.Cmax);
    a.arrivals = cv.take<unsigned>(nbt);
  }
  return cv.ok;
}

int launch_extrema(const ExArgs& a, int ydt, cudaStream_t st) {
  if (a.E > 0) {  // flat split
    if (cudaMemsetAsync(a.arrivals, 0, (size_t)(a.B * a.nb) * sizeof(unsigned), st) != cudaSuccess)
      return fail(MM_ECUDA, "cudaMemsetAsync(arrivals)");
    const int64_t blocks = cdiv(a.B * a.Ws, 8);
    static const int64_t fv = env_i64("MMLTTB_K1_FLAT_VARIANT", 0);  // A/B knob (tools/flat_sweep.sh)
    if (ydt == MM_F32) {
      switch (fv) {
        case 1: k_extrema_flat<float, 6, 3, 4><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        case 2: k_extrema_flat<float, 4, 3, 4><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        case 3: k_extrema_flat<float, 8, 1, 3><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        case 4: k_extrema_flat<float, 12, 3, 2><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        case 5: k_extrema_flat<float, 16, 3, 2><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        default: k_extrema_flat<float, 8, 3><<<(unsigned)blocks, 256, 0, st>>>(a); break;
      }
    } else {
      k_extrema_flat<double, 8, 3><<<(unsigned)blocks, 256, 0, st>>>(a);
    }
    return check_launch("k_extrema_flat");
  }
  const bool small = a.C == 1 && a.chunk <= SMALL_BUCKET;
  if (small && a.B * a.nb < 16384) {  // few buckets: a whole warp per bucket fills the GPU better
    const int64_t blocks = cdiv(a.B * a.nb, 8);
    if (ydt == MM_F32)
      k_extrema<float, 8, 3, 1, 32><<<(unsigned)blocks, 256, 0, st>>>(a);
    else
      k_extrema<double, 8, 3, 1, 32><<<(unsigned)blocks, 256, 0, st>>>(a);
    return check_launch("k_extrema(warp/bucket)");
  }
  if (small) {
    const int64_t blocks = cdiv(a.B * a.nb, 8 * 4);
    if (blocks > 0x7fffffffLL) return fail(MM_ERANGE, "extrema grid too large");
    if (ydt == MM_F32)
      k_extrema<float, 8, 3, 1, 8><<<(unsigned)blocks, 256, 0, st>>>(a);
    else
      k_extrema<double, 8, 3, 1, 8><<<(unsigned)blocks, 256, 0, st>>>(a);
    return check_launch("k_extrema(small)");
  }
  const int64_t warps = a.B * a.nb * a.C;
  if (a.C > 1 && cudaMemsetAsync(a.arrivals, 0, (size_t)(a.B * a.nb) * sizeof(unsigned), st) != cudaSuccess)
    return fail(MM_ECUDA, "cudaMemsetAsync(arrivals)");
  const int64_t blocks = cdiv(warps, 8);
  if (blocks > 0x7fffffffLL) return fail(MM_ERANGE, "extrema grid too large");
  if (a.chunk >= (1LL << 30)) return fail(MM_ERANGE, "bucket chunk too large");
  static const int variant = [] {
    const char* e = getenv("MMLTTB_K1_VARIANT");  // tuning knob, default = tuned choice
    return e ? atoi(e) : 0;
  }();
  const unsigned g = (unsigned)blocks;
#define MM_K1(T, U, L) k_extrema<T, U, L><<<g, 256, 0, st>>>(a)
#define MM_K1B(T, U, L, MB) k_extrema<T, U, L, MB><<<g, 256, 0, st>>>(a)
  if (ydt == MM_F32) {
    switch (variant) {
      case 1: MM_K1(float, 4, 1); break;
      case 2: MM_K1(float, 4, 2); break;
      case 3: MM_K1(float, 4, 3); break;
      case 4: MM_K1(float, 8, 0); break;
      case 5: MM_K1(float, 8, 1); break;
      case 6: MM_K1(float, 8, 3); break;
      case 7: MM_K1(float, 2, 1); break;
      case 8: MM_K1B(float, 4, 2, 6); break;
      case 9: MM_K1B(float, 4, 3, 6); break;
      case 10: MM_K1B(float, 2, 2, 8); break;
      case 11: MM_K1B(float, 8, 2, 4); break;
      case 12: MM_K1(float, 4, 0); break;
      default: MM_K1(float, 8, 3); break;  // tuned: U=8 vectors in flight, evict-first
    }
  } else {
    switch (variant) {
      case 1: MM_K1(double, 4, 1); break;
      case 4: MM_K1(double, 8, 0); break;
      case 5: MM_K1(double, 8, 1); break;
      case 12: MM_K1(double, 4, 0); break;
      default: MM_K1(double, 8, 3); break;
    }
  }
#undef MM_K1
#undef MM_K1B
  return check_launch("k_extrema");
}

bool mul_ok(int64_t a, int64_t b) { return a == 0 || b <= INT64_MAX / a; }

// ---- K3 planning --------------------------------------------------------
// Buckets of <= 64 points: exact transition tables over all points (K3a).
// Larger buckets: hull-candidate tables + full verification + repair (K3c).
constexpr int NBB = 32;   // buckets per k_lttb_tables block
constexpr int HMAX = 32;  // K3c workspace bound: <= 2 x 16 sampled directions per bucket

int smax_for(int64_t s) {
  if (s <= 4) return 4;
  if (s <= 8) return 8;
  if (s <= 16) return 16;
  if (s <= 32) return 32;
  if (s <= 64) return 64;
  return 0;
}

constexpr int64_t JUMP_SMEM_MAX = 200 * 1024;
// buckets per k_lttb_jump shared-memory segment (two byte tables of seg*SMAX)
int64_t jump_seg(int64_t k3, int smax) {
  const int64_t cap = (JUMP_SMEM_MAX / (2 * smax)) / 16 * 16;
  return std::min<int64_t>(cap, (k3 + 15) / 16 * 16);
}

bool use_tables(int64_t s) { return smax_for(s) > 0; }
bool use_hull() {
  static const bool h = env_i64("MMLTTB_K3C_HULL", 0) != 0;  // A/B knob: hull candidates
  return h;
}
bool use_chain() {
  static const bool c = env_i64("MMLTTB_LTTB_CHAIN", 0) != 0;  // A/B knob: old sequential chain
  return c;
}

int64_t tab_ld(int64_t k3, int smax) { return (k3 * smax + 15) / 16 * 16; }

int64_t lttb_ws(int64_t B, int64_t n_out, int64_t s) {
  const int64_t k3 = n_out - 2;
  if (use_tables(s)) return up(B * tab_ld(k3, smax_for(s)));
  if (use_chain()) return up(B * k3 * (int64_t)sizeof(double2));
  return up(B * k3 * (int64_t)sizeof(double2)) + up(B * k3 * HMAX * 8) + up(B * k3 * 4) + up(B * tab_ld(k3, HMAX)) +
         up(B * (k3 + 2) * 8) + up(B * k3 * 8) + up(B * k3 * 4) + up(B * k3 * (int64_t)sizeof(double2)) +
         up(B * k3 * 8) + up(B * k3 * 4) + up(B * 4);
}

template <int SMAX> int jump_attr() {
  static bool done = false;
  if (!done) {
    if (cudaFuncSetAttribute(k_lttb_jump<SMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)JUMP_SMEM_MAX) != cudaSuccess)
      return fail(MM_ECUDA, "cudaFuncSetAttribute(k_lttb_jump)");
    done = true;
  }
  return MM_OK;
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
    k_lttb_scan<SMAX, 512, 4><<<(unsigned)a.B, 512, 0, st>>>(a);
    return check_launch("k_lttb_scan");
  } else {
    return launch_jump<SMAX>(a, st);
  }
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
  a.tables = tabs;
  a.cand_cap = (int)env_i64("MMLTTB_K3C_CAND_CAP", H);  // test knob: a poor heuristic must still be exact
  // one warp per bucket, 8 KB of tiles each: every bucket's chain resident at once
  // loads two tiles ahead (59 vs 64 us on C2); MMLTTB_K3C_MEANS=1: one tile ahead (A/B knob)
  static const int64_t mv = env_i64("MMLTTB_K3C_MEANS", 0);
  if (mv == 1) k_lttb_means_staged<XT, YT, 256><<<(unsigned)(a.B * (k3 + 1)), 32, 0, st>>>(a);
  else k_lttb_means_staged2<XT, YT, 256><<<(unsigned)(a.B * (k3 + 1)), 32, 0, st>>>(a);
  int rc = check_launch("k_lttb_means");
  if (rc) return rc;
  if (use_hull()) {
    k_lttb_hull<XT, YT, H><<<dim3((unsigned)cdiv(k3, 2), (unsigned)a.B), 64, 0, st>>>(a);
    if ((rc = check_launch("k_lttb_hull"))) return rc;
  } else {
    static const int64_t dnt = env_i64("MMLTTB_K3C_DIRCAND_NT", 64);  // A/B knob (64: 64 vs 68 us at 128 on C2)
    if (dnt == 32) k_lttb_dircand<XT, YT, H, H / 2, 32><<<dim3((unsigned)k3, (unsigned)a.B), 32, 0, st>>>(a);
    else if (dnt == 64) k_lttb_dircand<XT, YT, H, H / 2, 64><<<dim3((unsigned)k3, (unsigned)a.B), 64, 0, st>>>(a);
    else if (dnt == 256) k_lttb_dircand<XT, YT, H, H / 2, 256><<<dim3((unsigned)k3, (unsigned)a.B), 256, 0, st>>>(a);
    else k_lttb_dircand<XT, YT, H, H / 2, 128><<<dim3((unsigned)k3, (unsigned)a.B), 128, 0, st>>>(a);
    if ((rc = check_launch("k_lttb_dircand"))) return rc;
  }
  k_lttb_ctables<XT, YT, H><<<dim3((unsigned)cdiv(k3, 1024 / H), (unsigned)a.B), 1024, 0, st>>>(a);
  if ((rc = check_launch("k_lttb_ctables"))) return rc;
  k_lttb_scan<H, 512, 4><<<(unsigned)a.B, 512, 0, st>>>(a);
  if ((rc = check_launch("k_lttb_scan"))) return rc;
  if (cudaMemsetAsync(a.fcount, 0, (size_t)a.B * sizeof(int), st) != cudaSuccess) return fail(MM_ECUDA, "memset");
  static const int64_t vnt = env_i64("MMLTTB_K3C_VERIFY_NT", 64);  // A/B knob (64: 30 vs 37.5 us at 256 on C2)
  if (vnt == 512) k_lttb_verify<XT, YT, 512><<<dim3((unsigned)k3, (unsigned)a.B), 512, 0, st>>>(a);
  else if (vnt == 128) k_lttb_verify<XT, YT, 128><<<dim3((unsigned)k3, (unsigned)a.B), 128, 0, st>>>(a);
  else if (vnt == 64) k_lttb_verify<XT, YT, 64><<<dim3((unsigned)k3, (unsigned)a.B), 64, 0, st>>>(a);
  else if (vnt == 32) k_lttb_verify<XT, YT, 32><<<dim3((unsigned)k3, (unsigned)a.B), 32, 0, st>>>(a);
  else k_lttb_verify<XT, YT, 256><<<dim3((unsigned)k3, (unsigned)a.B), 256, 0, st>>>(a);
  if ((rc = check_launch("k_lttb_verify"))) return rc;
  static const int64_t v2 = env_i64("MMLTTB_K3C_VERIFY2_NT", 256);  // A/B knob
  if (v2 == 64) k_lttb_verify2<XT, YT, 64><<<dim3(148, (unsigned)a.B), 64, 0, st>>>(a);
  else if (v2 == 128) k_lttb_verify2<XT, YT, 128><<<dim3(148, (unsigned)a.B), 128, 0, st>>>(a);
  else k_lttb_verify2<XT, YT, 256><<<dim3(148, (unsigned)a.B), 256, 0, st>>>(a);
  if ((rc = check_launch("k_lttb_verify2"))) return rc;
  static const int64_t rp = env_i64("MMLTTB_K3C_REPAIR_NT", 512);  // A/B knob (512: 22.1 vs 24.4 us at 1024 on C2)
  if (rp == 256) k_lttb_repair<XT, YT, 256><<<(unsigned)a.B, 256, 0, st>>>(a);
  else if (rp == 512) k_lttb_repair<XT, YT, 512><<<(unsigned)a.B, 512, 0, st>>>(a);
  else k_lttb_repair<XT, YT, 1024><<<(unsigned)a.B, 1024, 0, st>>>(a);
  return check_launch("k_lttb_repair");
}

template <typename XT, typename YT>
int launch_lttb_t(LttbArgs a, int64_t s, cudaStream_t st) {
  const int64_t k3 = a.n_out - 2;
  if (a.B > 65535) return fail(MM_ERANGE, "batch > 65535 series");
  if (use_tables(s)) {
    switch (smax_for(s)) {
      case 4: return launch_tables_jump<XT, YT, 4>(a, st);
      case 8: return launch_tables_jump<XT, YT, 8>(a, st);
      case 16: return launch_tables_jump<XT, YT, 16>(a, st);
      case 32: return launch_tables_jump<XT, YT, 32>(a, st);
      default: return launch_tables_jump<XT, YT, 64>(a, st);
    }
  }
  if (!use_chain()) {
    static const int64_t h = env_i64("MMLTTB_K3C_HMAX", 16);  // A/B knob: 16 or 32 candidates
    return h == 32 ? launch_lttb_large<XT, YT, 32>(a, st) : launch_lttb_large<XT, YT, 16>(a, st);
  }
  a.means = reinterpret_cast<double2*>(a.tables);
  a.means_ld = k3;
  const int64_t n = a.B * k3;
  k_lttb_means<XT, YT><<<(unsigned)cdiv(n, 128), 128, 0, st>>>(a);
  int rc = check_launch("k_lttb_means");
  if (rc) return rc;
  k_lttb_chain<XT, YT, 512><<<(unsigned)a.B, 512, 0, st>>>(a);
  return check_launch("k_lttb_chain");
}

template <typename XT>
int launch_lttb_x(LttbArgs a, int ydt, int64_t s, cudaStream_t st) {
  if (ydt == MM_F32) return launch_lttb_t<XT, float>(a, s, st);
  if (ydt == MM_F64) return launch_lttb_t<XT, double>(a, s, st);
  return fail(MM_EINVAL, "y dtype");
}

// a.tables must point at lttb_ws(B, n_out, s) bytes of workspace
int launch_lttb(LttbArgs a, int xdt, int ydt, int64_t s, cudaStream_t st) {
  switch (xdt) {
    case MM_F32: return launch_lttb_x<float>(a, ydt, s, st);
    case MM_F64: return launch_lttb_x<double>(a, ydt, s, st);
    case MM_I64: return launch_lttb_x<long long>(a, ydt, s, st);
    case MM_I32: return launch_lttb_x<int>(a, ydt, s, st);
  }
  return fail(MM_EINVAL, "x dtype");
}

// ---- shared pieces of the fused entries ----------------------------------
// sizes for minmaxlttb / preselect on B series
int64_t preselect_ws(int64_t B, int64_t N, int64_t n_out, int64_t r_ps, int ydt, bool with_lttb) {
  const int64_t k = (n_out - 2) * (r_ps / 2);
  const int64_t S = cdiv(N - 2, k);
  const ExPlan p = plan_extrema(B * k, S, ydt, B, true);
  const int64_t cap = 2 + 2 * k;
  int64_t bytes = ex_ws(B * k, p) + up(B * 8);
  if (with_lttb) bytes += 3 * up(B * cap * 8) + lttb_ws(B, n_out, r_ps);
  return bytes;
}

constexpr int PAIR_NT = 128, PAIR_ITEMS = 2;

template <typename XT, typename YT>
void pairs_t(const PairArgs& pa, dim3 g, cudaStream_t st) {
  k_compact_pairs<XT, YT, PAIR_NT, PAIR_ITEMS><<<g, PAIR_NT, 0, st>>>(pa);
}

// K2 launch; pa.out_x == null means no gather (x/y dtypes then irrelevant)
int launch_pairs(PairArgs pa, int64_t B, cudaStream_t st) {
  const int64_t tiles = std::max<int64_t>(1, cdiv(pa.nb, PAIR_NT * PAIR_ITEMS));
  if (B > 65535) return fail(MM_ERANGE, "batch > 65535 series");
  const dim3 g((unsigned)tiles, (unsigned)B);
  const bool y32 = pa.ydt == MM_F32;
  if (!pa.out_x) {  // no gather: x unused; y only read for the endpoint finite check
    pa.x = nullptr;
    y32 ? pairs_t<double, float>(pa, g, st) : pairs_t<double, double>(pa, g, st);
    return check_launch("k_compact_pairs");
  }
  switch (pa.xdt) {
    case MM_F32: y32 ? pairs_t<float, float>(pa, g, st) : pairs_t<float, double>(pa, g, st); break;
    case MM_F64: y32 ? pairs_t<double, float>(pa, g, st) : pairs_t<double, double>(pa, g, st); break;
    case MM_I64: y32 ? pairs_t<long long, float>(pa, g, st) : pairs_t<long long, double>(pa, g, st); break;
    default: y32 ? pairs_t<int, float>(pa, g, st) : pairs_t<int, double>(pa, g, st); break;
  }
  return check_launch("k_compact_pairs");
}

// ---- fused per-series path (batches of medium series) --------------------
constexpr int64_t FUSED_SMEM_MAX = 110 * 1024;
constexpr int64_t FUSED_MIN_B = 148;

bool fused_ok(int64_t B, int64_t N, int64_t n_out, int64_t r_ps, int ydt) {
  static const bool off = env_i64("MMLTTB_NO_FUSED", 0) != 0;  // A/B knob
  const int64_t k = (n_out - 2) * (r_ps / 2);
  return !off && B >= FUSED_MIN_B && r_ps >= 2 && r_ps <= 8 && N < (1LL << 31) &&
         fused_smem(k, n_out - 2, 8, esize(ydt)) <= FUSED_SMEM_MAX;
}

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

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
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

int launch_fused(const FusedArgs& fa, int xdt, int ydt, cudaStream_t st) {
  switch (xdt) {
    case MM_F32: return launch_fused_x<float>(fa, ydt, st);
    case MM_F64: return launch_fused_x<double>(fa, ydt, st);
    case MM_I64: return launch_fused_x<long long>(fa, ydt, st);
    default: return launch_fused_x<int>(fa, ydt, st);
  }
}

// First 256 bytes of every fused entry's workspace: status word (bit 0 =
// non-finite y seen), zeroed on the stream at entry.
int* take_status(Carve& cv, cudaStream_t st) {
  int* p = cv.take<int>(1);
  if (p && cudaMemsetAsync(p, 0, sizeof(int), st) != cudaSuccess) return nullptr;
  return p;
}

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

int check_common(const void* y, int ydt, int64_t B, int64_t N, int64_t n_out) {
  if (!y) return fail(MM_EINVAL, "y is null");
  if (!ydt_ok(ydt)) return fail(MM_EINVAL, "y dtype must be f32 or f64");
  if (B < 1 || N < 2) return fail(MM_EINVAL, "need B >= 1 and N >= 2");
  if (n_out < 3 || n_out > N) return fail(MM_EINVAL, "n_out must be in [3, %lld]", (long long)N);
  return MM_OK;
}

}  // namespace

extern "C" {

int mmlttb_version(void) { return 1; }

int64_t mmlttb_launch_count(void) { return g_launches.load(); }

int64_t mmlttb_repair_scans(void) {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, g_repair_scans, sizeof v) != cudaSuccess) return -1;
  return (int64_t)v;
}

int mmlttb_stage_timer(int enable) {
  g_timer.on = enable != 0;
  g_timer.used = 0;
  g_timer.calls.clear();
  return MM_OK;
}

int mmlttb_stage_timer_read(double* ms3, int64_t* calls) {
  for (int i = 0; i < 3; ++i) ms3[i] = 0.0;
  for (auto& c : g_timer.calls) {
    if (cudaEventSynchronize(c[3]) != cudaSuccess) return fail(MM_ECUDA, "cudaEventSynchronize");
    for (int i = 0; i < 3; ++i) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, c[i], c[i + 1]) != cudaSuccess) return fail(MM_ECUDA, "cudaEventElapsedTime");
      ms3[i] += ms;
    }
  }
  *calls = (int64_t)g_timer.calls.size();
  g_timer.used = 0;
  g_timer.calls.clear();
  return MM_OK;
}
const char* mmlttb_last_error(void) { return g_err.c_str(); }

int64_t mmlttb_workspace_bytes(int op, int64_t B, int64_t N, int64_t n_out, int64_t r_ps, int y_dtype) {
  if (B < 1 || N < 3 || n_out < 3 || n_out > N) return 0;
  switch (op) {
    case MM_OP_MINMAXLTTB:
      if (r_ps == 1) return mmlttb_workspace_bytes(MM_OP_MINMAX, B, N, n_out, 0, y_dtype);
      if (r_ps < 2 || r_ps % 2) return 0;
      return ALIGN + preselect_ws(B, N, n_out, r_ps, y_dtype, true);
    case MM_OP_PRESELECT:
      if (r_ps < 2 || r_ps % 2) return 0;
      return ALIGN + preselect_ws(B, N, n_out, r_ps, y_dtype, false);
    case MM_OP_LTTB:
      return lttb_ws(B, n_out, cdiv(N - 2, n_out - 2));
    case MM_OP_MINMAX:
    case MM_OP_M4: {
      const int64_t k = op == MM_OP_MINMAX ? n_out / 2 : n_out / 4;
      if (k < 1) return 0;
      return ALIGN + ex_ws(B * k, plan_extrema(B * k, cdiv(N, k), y_dtype, B, true));
    }
  }
  return 0;
}

int mmlttb_minmax_preselect(const void* y, int y_dtype, int64_t y_ld, int64_t B, int64_t N, int64_t n_out,
                            int64_t r_ps, int64_t* out, int64_t out_ld, int64_t* out_count, void* workspace,
                            int64_t workspace_bytes, void* stream) {
  int rc = check_common(y, y_dtype, B, N, n_out);
  if (rc) return rc;
  if (r_ps < 2 || r_ps % 2) return fail(MM_EINVAL, "r_ps must be even >= 2");
  const int64_t k = (n_out - 2) * (r_ps / 2);
  if (k > N - 2) return fail(MM_EINVAL, "sub-buckets exceed interior");
  if (!mul_ok(k, N)) return fail(MM_ERANGE, "k*N overflows int64");
  if (out_ld < 2 + 2 * k) return fail(MM_EINVAL, "out_ld < 2 + 2k");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t S = cdiv(N - 2, k);
  const ExPlan p = plan_extrema(B * k, S, y_dtype, B, true);
  Carve cv{(char*)workspace, workspace_bytes};
  int* status = take_status(cv, st);
  ExArgs ea{y, y_ld, B, 1, N - 2, k, nullptr, 0, k, p.C, p.chunk};
  if (!carve_ex(cv, B * k, p, ea) || !status) return fail(MM_EWORKSPACE, "workspace too small");
  if ((rc = launch_extrema(ea, y_dtype, st))) return rc;
  PairArgs pa{};
  pa.ext = ea.ext; pa.cnt8 = ea.cnt8; pa.nb = k;
  pa.emit_first = 0; pa.emit_last = N - 1;
  pa.out_idx = out; pa.out_ld = out_ld; pa.out_count = out_count;
  pa.y = y; pa.ydt = y_dtype; pa.y_ld = y_ld; pa.status = status;
  return launch_pairs(pa, B, st);
}

static int minmax_impl(const void* y, int ydt, int64_t y_ld, int64_t B, int64_t N, int64_t n_out, int m4,
                       int64_t force_n_out, int64_t* out, int64_t* out_count, void* ws, int64_t wsb,
                       cudaStream_t st) {
  int rc = check_common(y, ydt, B, N, n_out);
  if (rc) return rc;
  const int64_t k = m4 ? n_out / 4 : n_out / 2;
  if ((m4 && n_out % 4) || (!m4 && n_out % 2)) return fail(MM_EINVAL, "n_out divisibility");
  if (!mul_ok(k + 1, N)) return fail(MM_ERANGE, "k*N overflows int64");
  const ExPlan p = plan_extrema(B * k, cdiv(N, k), ydt, B, true);
  Carve cv{(char*)ws, wsb};
  int* status = take_status(cv, st);
  ExArgs ea{y, y_ld, B, 0, N, k, nullptr, 0, k, p.C, p.chunk};
  if (!carve_ex(cv, B * k, p, ea) || !status) return fail(MM_EWORKSPACE, "workspace too small");
  if ((rc = launch_extrema(ea, ydt, st))) return rc;
  if (!m4 && force_n_out == 0) {
    PairArgs pa{};
    pa.ext = ea.ext; pa.cnt8 = ea.cnt8; pa.nb = k;
    pa.emit_first = -1; pa.emit_last = -1;
    pa.out_idx = out; pa.out_ld = n_out; pa.out_count = out_count;
    pa.y = y; pa.ydt = ydt; pa.y_ld = y_ld; pa.status = status;
    return launch_pairs(pa, B, st);
  }
  CompactArgs ca{};
  ca.ext = ea.ext; ca.nb = k; ca.mode = m4 ? 1 : 0;
  ca.ydt = ydt; ca.status = status;
  ca.emit_first = -1; ca.emit_last = -1; ca.force_n_out = force_n_out; ca.last_index = N - 1;
  ca.start = 0; ca.len = N; ca.k = k; ca.b0 = 0;
  ca.out_idx = out; ca.out_ld = n_out; ca.out_count = out_count;
  k_compact<512><<<(unsigned)B, 512, 0, st>>>(ca);
  return check_launch("k_compact");
}

int mmlttb_minmax(const void* y, int y_dtype, int64_t y_ld, int64_t B, int64_t N, int64_t n_out, int64_t* out,
                  int64_t* out_count, void* workspace, int64_t workspace_bytes, void* stream) {
  return minmax_impl(y, y_dtype, y_ld, B, N, n_out, 0, 0, out, out_count, workspace, workspace_bytes,
                            (cudaStream_t)stream);
}

int mmlttb_m4(const void* y, int y_dtype, int64_t y_ld, int64_t B, int64_t N, int64_t n_out, int64_t* out,
              int64_t* out_count, void* workspace, int64_t workspace_bytes, void* stream) {
  return minmax_impl(y, y_dtype, y_ld, B, N, n_out, 1, 0, out, out_count, workspace, workspace_bytes,
                            (cudaStream_t)stream);
}

int mmlttb_minmaxlttb(const void* x, int x_dtype, int64_t x_ld, const void* y, int y_dtype, int64_t y_ld, int64_t B,
                      int64_t N, int64_t n_out, int64_t r_ps, int64_t* out, int64_t* out_count, void* workspace,
                      int64_t workspace_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (r_ps == 1) {  // downsamplers.py:204-205
    if (n_out % 2) return fail(MM_EINVAL, "r_ps=1 needs an even n_out");
    return minmax_impl(y, y_dtype, y_ld, B, N, n_out, 0, n_out, out, out_count, workspace, workspace_bytes, st);
  }
  int rc = check_common(y, y_dtype, B, N, n_out);
  if (rc) return rc;
  if (!x || !xdt_ok(x_dtype)) return fail(MM_EINVAL, "x missing or bad dtype");
  if (r_ps < 2 || r_ps % 2) return fail(MM_EINVAL, "r_ps must be 1 or even >= 2");
  const int64_t k = (n_out - 2) * (r_ps / 2);
  if (k > N - 2) return fail(MM_EINVAL, "sub-buckets exceed interior");
  if (!mul_ok(k, N)) return fail(MM_ERANGE, "k*N overflows int64");
  Carve cv0{(char*)workspace, workspace_bytes};
  int* status = take_status(cv0, st);
  if (!status) return fail(MM_EWORKSPACE, "workspace too small");
  if (fused_ok(B, N, n_out, r_ps, y_dtype)) {  // one CTA per series, everything on chip
    FusedArgs fa{x, x_ld, y, y_ld, B, N, n_out, r_ps, out, status};
    stage_mark(st, 0);
    if ((rc = launch_fused(fa, x_dtype, y_dtype, st))) return rc;
    stage_mark(st, 1);
    stage_mark(st, 2);
    stage_mark(st, 3);
    if (out_count) {
      k_fill<<<(unsigned)cdiv(B, 256), 256, 0, st>>>(out_count, B, n_out);
      return check_launch("k_fill");
    }
    return MM_OK;
  }
  const int64_t S = cdiv(N - 2, k);
  const ExPlan p = plan_extrema(B * k, S, y_dtype, B, true);
  const int64_t cap = 2 + 2 * k;
  Carve cv = cv0;
  ExArgs ea{y, y_ld, B, 1, N - 2, k, nullptr, 0, k, p.C, p.chunk};
  carve_ex(cv, B * k, p, ea);
  int64_t* cnt = cv.take<int64_t>(B);
  int64_t* pre = cv.take<int64_t>(B * cap);
  double* px = cv.take<double>(B * cap);
  double* py = cv.take<double>(B * cap);
  unsigned char* lt = cv.take<unsigned char>(lttb_ws(B, n_out, r_ps));
  if (!cv.ok) return fail(MM_EWORKSPACE, "workspace too small (%lld bytes)", (long long)workspace_bytes);
  // K1: sub-bucket extrema over partition(1, N-1, k)  (downsamplers.py:149-155)
  stage_mark(st, 0);
  if ((rc = launch_extrema(ea, y_dtype, st))) return rc;
  stage_mark(st, 1);
  if (post_ok(k, n_out, r_ps)) {  // K2 + K3 in one CTA per series
    PostArgs qa{ea.ext, k, x, x_ld, y, y_ld, N, n_out, pre, px, py, cap, out, status};
    if ((rc = launch_post(qa, B, x_dtype, y_dtype, smax_for(r_ps), st))) return rc;
    stage_mark(st, 2);
    stage_mark(st, 3);
    if (out_count) {
      k_fill<<<(unsigned)cdiv(B, 256), 256, 0, st>>>(out_count, B, n_out);
      return check_launch("k_fill");
    }
    return MM_OK;
  }
  // K2: [0] + interleaved pairs + [N-1], gathered as f64 (:156-160, :207)
  PairArgs pa{};
  pa.ext = ea.ext; pa.cnt8 = ea.cnt8; pa.nb = k;
  pa.emit_first = 0; pa.emit_last = N - 1;
  pa.out_idx = pre; pa.out_ld = cap; pa.out_count = cnt;
  pa.x = x; pa.xdt = x_dtype; pa.x_ld = x_ld;
  pa.y = y; pa.ydt = y_dtype; pa.y_ld = y_ld;
  pa.out_x = px; pa.out_y = py; pa.status = status;
  {  // K2 + K3a in one cooperative launch when it fits (small B, r_ps <= 8)
    LttbArgs la{};
    la.x = px; la.x_ld = cap; la.y = py; la.y_ld = cap;
    la.m_dev = cnt; la.n = 0; la.bounds = nullptr; la.map = pre; la.map_ld = cap;
    la.B = B; la.n_out = n_out; la.out = out; la.tables = lt;
    bool launched = false;
    if ((rc = launch_coop(pa, la, B, smax_for(r_ps), st, &launched))) return rc;
    if (launched) {
      stage_mark(st, 2);
      stage_mark(st, 3);
      if (out_count) {
        k_fill<<<(unsigned)cdiv(B, 256), 256, 0, st>>>(out_count, B, n_out);
        return check_launch("k_fill");
      }
      return MM_OK;
    }
  }
  if ((rc = launch_pairs(pa, B, st))) return rc;
  stage_mark(st, 2);
  // K3: LTTB over the compacted sub-series, mapped back (:208-209)
  LttbArgs la{};
  la.x = px; la.x_ld = cap; la.y = py; la.y_ld = cap;
  la.m_dev = cnt; la.n = 0; la.bounds = nullptr; la.map = pre; la.map_ld = cap;
  la.B = B; la.n_out = n_out; la.out = out; la.tables = lt;
  if ((rc = launch_lttb(la, MM_F64, MM_F64, r_ps, st))) return rc;
  stage_mark(st, 3);
  if (out_count) {  // every series yields exactly n_out (P9)
    k_fill<<<(unsigned)cdiv(B, 256), 256, 0, st>>>(out_count, B, n_out);
    return check_launch("k_fill");
  }
  return MM_OK;
}

int mmlttb_lttb(const void* x, int x_dtype, int64_t x_ld, const void* y, int y_dtype, int64_t y_ld, int64_t B,
                int64_t N, int64_t n_out, int64_t* out, void* workspace, int64_t workspace_bytes, void* stream) {
  int rc = check_common(y, y_dtype, B, N, n_out);
  if (rc) return rc;
  if (!x || !xdt_ok(x_dtype)) return fail(MM_EINVAL, "x missing or bad dtype");
  if (!mul_ok(n_out, N)) return fail(MM_ERANGE, "n_out*N overflows int64");
  const int64_t s = cdiv(N - 2, n_out - 2);
  if (workspace_bytes < lttb_ws(B, n_out, s)) return fail(MM_EWORKSPACE, "workspace too small");
  LttbArgs la{};
  la.x = x; la.x_ld = x_ld; la.y = y; la.y_ld = y_ld;
  la.m_dev = nullptr; la.n = N; la.bounds = nullptr; la.map = nullptr;
  la.B = B; la.n_out = n_out; la.out = out; la.tables = (unsigned char*)workspace;
  return launch_lttb(la, x_dtype, y_dtype, s, (cudaStream_t)stream);
}

int mmlttb_every_nth(int64_t N, int64_t n_out, int64_t* out, void* stream) {
  if (n_out < 1 || !mul_ok(n_out, N)) return fail(MM_EINVAL, "bad n_out");
  k_every_nth<<<(unsigned)cdiv(n_out, 256), 256, 0, (cudaStream_t)stream>>>(N, n_out, out);
  return check_launch("k_every_nth");
}

int64_t mmlttb_extrema_workspace_bytes(int64_t k, int64_t max_bucket_len) {
  (void)max_bucket_len;
  return ex_ws(k, plan_extrema(k, 1, MM_F32));
}

int mmlttb_extrema_by_bucket(const void* y, int y_dtype, const int64_t* bounds, int64_t k, int64_t max_bucket_len,
                             int64_t* out_min, int64_t* out_max, void* workspace, int64_t workspace_bytes,
                             void* stream) {
  if (!y || !bounds || !ydt_ok(y_dtype) || k < 1 || max_bucket_len < 1) return fail(MM_EINVAL, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const ExPlan p = plan_extrema(k, max_bucket_len, y_dtype);
  Carve cv{(char*)workspace, workspace_bytes};
  ExArgs ea{y, 0, 1, 0, 1, 1, bounds, 0, k, p.C, p.chunk};
  if (!carve_ex(cv, k, p, ea)) return fail(MM_EWORKSPACE, "workspace too small");
  int rc = launch_extrema(ea, y_dtype, st);
  if (rc) return rc;
  k_finalize_extrema<<<(unsigned)cdiv(k, 256), 256, 0, st>>>(ea.ext, k, out_min, out_max);
  return check_launch("k_finalize_extrema");
}

int64_t mmlttb_lttb_select_workspace_bytes(int64_t n, int64_t nb) {
  (void)n;
  return lttb_ws(1, nb + 1, INT64_MAX / 4);
}

int mmlttb_lttb_select(const void* xs, int x_dtype, const void* ys, int y_dtype, int64_t n, const int64_t* bounds,
                       int64_t nb, int64_t* out, void* workspace, int64_t workspace_bytes, void* stream) {
  if (!xs || !ys || !bounds || !xdt_ok(x_dtype) || !ydt_ok(y_dtype) || nb < 2 || n < 2)
    return fail(MM_EINVAL, "bad arguments");
  if (workspace_bytes < mmlttb_lttb_select_workspace_bytes(n, nb)) return fail(MM_EWORKSPACE, "workspace too small");
  LttbArgs la{};
  la.x = xs; la.y = ys; la.n = n; la.bounds = bounds; la.B = 1; la.n_out = nb + 1; la.out = out;
  la.tables = (unsigned char*)workspace;
  // explicit bounds: bucket sizes are the caller's -> the general (K3c) path
  return launch_lttb(la, x_dtype, y_dtype, INT64_MAX / 4, (cudaStream_t)stream);
}

int64_t mmlttb_shard_workspace_bytes(int64_t N, int64_t n_out, int64_t r_ps, int64_t b0, int64_t b1) {
  const int64_t k = (n_out - 2) * (r_ps / 2);
  if (k < 1 || b1 <= b0) return ALIGN;
  return std::max(ex_ws(b1 - b0, plan_extrema(b1 - b0, cdiv(N - 2, k), MM_F32, 1, true)),
                  ex_ws(b1 - b0, plan_extrema(b1 - b0, cdiv(N - 2, k), MM_F64, 1, true)));
}

int mmlttb_shard_preselect(const void* x_shard, int x_dtype, const void* y_shard, int y_dtype, int64_t lo, int64_t N,
                           int64_t n_out, int64_t r_ps, int64_t b0, int64_t b1, int emit_first, int emit_last,
                           int64_t* out_idx, double* out_x, double* out_y, int64_t* out_count, void* workspace,
                           int64_t workspace_bytes, void* stream) {
  int rc = check_common(y_shard, y_dtype, 1, N, n_out);
  if (rc) return rc;
  if (!x_shard || !xdt_ok(x_dtype)) return fail(MM_EINVAL, "x missing or bad dtype");
  if (r_ps < 2 || r_ps % 2) return fail(MM_EINVAL, "r_ps must be even >= 2");
  const int64_t k = (n_out - 2) * (r_ps / 2);
  if (k > N - 2 || b0 < 0 || b1 > k || b1 < b0) return fail(MM_EINVAL, "bad bucket range");
  if (!mul_ok(k, N)) return fail(MM_ERANGE, "k*N overflows int64");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nb = b1 - b0;
  const ExPlan p = plan_extrema(std::max<int64_t>(nb, 1), cdiv(N - 2, k), y_dtype, 1, true);
  Carve cv{(char*)workspace, workspace_bytes};
  // virtual base: element i of the global series lives at y_shard[i - lo]
  const void* ybase = (const char*)y_shard - lo * esize(y_dtype);
  const void* xbase = (const char*)x_shard - lo * esize(x_dtype);
  ExArgs ea{ybase, 0, 1, 1, N - 2, k, nullptr, b0, nb, p.C, p.chunk};
  if (!carve_ex(cv, std::max<int64_t>(nb, 1), p, ea)) return fail(MM_EWORKSPACE, "workspace too small");
  if (nb > 0 && (rc = launch_extrema(ea, y_dtype, st))) return rc;
  PairArgs pa{};
  pa.ext = ea.ext; pa.cnt8 = ea.cnt8; pa.nb = nb;
  pa.emit_first = emit_first ? 0 : -1; pa.emit_last = emit_last ? N - 1 : -1;
  pa.out_idx = out_idx; pa.out_ld = 0; pa.out_count = out_count;
  pa.x = xbase; pa.xdt = x_dtype; pa.x_ld = 0;
  pa.y = ybase; pa.ydt = y_dtype; pa.y_ld = 0;
  pa.out_x = out_x; pa.out_y = out_y;
  return launch_pairs(pa, 1, st);
}

int mmlttb_merge_shards(const int64_t* idx, const double* xs, const double* ys, const int64_t* counts, int64_t G,
                        int64_t cap, int64_t* out_idx, double* out_x, double* out_y, int64_t* out_m, void* stream) {
  if (G < 1 || cap < 1) return fail(MM_EINVAL, "bad arguments");
  k_merge_shards<<<(unsigned)G, 256, 0, (cudaStream_t)stream>>>(idx, xs, ys, counts, G, cap, out_idx, out_x, out_y,
                                                                 out_m);
  return check_launch("k_merge_shards");
}

int mmlttb_merge_packed(const int64_t* buf, int64_t G, int64_t cap, int64_t* out_idx, double* out_x, double* out_y,
                        int64_t* out_m, void* stream) {
  if (!buf || !out_idx || !out_x || !out_y || !out_m || G < 1 || cap < 1) return fail(MM_EINVAL, "bad arguments");
  k_merge_packed<<<(unsigned)G, 256, 0, (cudaStream_t)stream>>>((const long long*)buf, G, cap, out_idx, out_x, out_y,
                                                                out_m);
  return check_launch("k_merge_packed");
}

int mmlttb_p2p_publish(const int64_t* idx, const double* xs, const double* ys, const int64_t* count, int64_t cap,
                       const uint64_t* peer_bufs, const uint64_t* peer_pads, const uint32_t* own_pad, int64_t G,
                       int64_t rank, uint32_t epoch, void* stream) {
  if (!idx || !xs || !ys || !count || !peer_bufs || !peer_pads || !own_pad || G < 1 || rank < 0 || rank >= G ||
      cap < 1 || epoch == 0)
    return fail(MM_EINVAL, "bad arguments");
  k_p2p_publish<<<(unsigned)G, 256, 0, (cudaStream_t)stream>>>(idx, xs, ys, count, cap,
                                                              (const unsigned long long*)peer_bufs,
                                                              (const unsigned long long*)peer_pads, own_pad, G, rank,
                                                              epoch);
  return check_launch("k_p2p_publish");
}

int mmlttb_p2p_merge(const int64_t* own_buf, const uint32_t* own_pad, const uint64_t* peer_pads, int64_t G,
                     int64_t rank, int64_t cap, uint32_t epoch, int64_t* out_idx, double* out_x, double* out_y,
                     int64_t* out_m, void* stream) {
  if (!own_buf || !own_pad || !peer_pads || !out_idx || !out_x || !out_y || !out_m || G < 1 || cap < 1 || epoch == 0)
    return fail(MM_EINVAL, "bad arguments");
  k_p2p_merge<<<(unsigned)G, 256, 0, (cudaStream_t)stream>>>((const long long*)own_buf, own_pad,
                                                            (const unsigned long long*)peer_pads, G, rank, cap, epoch,
                                                            out_idx, out_x, out_y, out_m);
  return check_launch("k_p2p_merge");
}

int64_t mmlttb_lttb_preselected_workspace_bytes(int64_t B, int64_t n_out, int64_t r_ps) {
  return lttb_ws(B, n_out, r_ps);
}

int mmlttb_lttb_preselected(const int64_t* pre_idx, const double* pre_x, const double* pre_y, const int64_t* m,
                            int64_t B, int64_t ld, int64_t n_out, int64_t r_ps, int64_t* out, void* workspace,
                            int64_t workspace_bytes, void* stream) {
  if (!pre_idx || !pre_x || !pre_y || !m || B < 1 || n_out < 3 || r_ps < 1) return fail(MM_EINVAL, "bad arguments");
  if (workspace_bytes < lttb_ws(B, n_out, r_ps)) return fail(MM_EWORKSPACE, "workspace too small");
  LttbArgs la{};
  la.x = pre_x; la.x_ld = ld; la.y = pre_y; la.y_ld = ld;
  la.m_dev = m; la.map = pre_idx; la.map_ld = ld;
  la.B = B; la.n_out = n_out; la.out = out; la.tables = (unsigned char*)workspace;
  return launch_lttb(la, MM_F64, MM_F64, r_ps, (cudaStream_t)stream);
}

int mmlttb_deinterleave_f64(const void* pairs, int64_t n, double* x, double* y, void* stream) {
  if (!pairs || !x || !y || n < 0) return fail(MM_EINVAL, "bad arguments");
  if (n == 0) return MM_OK;
  if ((uintptr_t)pairs % 16) return fail(MM_EINVAL, "pairs must be 16-byte aligned");
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 32);
  k_deinterleave_f64<<<blocks, 256, 0, (cudaStream_t)stream>>>((const double2*)pairs, x, y, n);
  return check_launch("k_deinterleave_f64");
}

int64_t mmlttb_raster_workspace_bytes(int64_t n, int64_t w, int64_t h) {
  return up(n * 8) * 2 + up(std::max<int64_t>(n - 1, 1) * 16) + up(5 * w * h * 8) + up(cdiv(w * h, 256) * 16) + ALIGN;
}

int mmlttb_rasterize(const void* x, int x_dtype, const void* y, int y_dtype, const int64_t* idx, int64_t n, double x0,
                     double x1, double y0, double y1, int64_t w, int64_t h, uint8_t* pixels, void* workspace,
                     int64_t workspace_bytes, void* stream) {
  if (!x || !y || !pixels || n < 2 || w < 1 || h < 1 || !xdt_ok(x_dtype) || !xdt_ok(y_dtype) ||
      w * h > (int64_t)INT32_MAX)
    return fail(MM_EINVAL, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  Carve cv{(char*)workspace, workspace_bytes};
  RasterCoordArgs a{x, x_dtype, y, y_dtype, idx, n, x0, x1, y0, y1, w, h, nullptr, nullptr, nullptr};
  a.us = cv.take<double>(n);
  a.vs = cv.take<double>(n);
  a.box = cv.take<int>(4 * (n - 1));
  if (!cv.ok) return fail(MM_EWORKSPACE, "workspace too small");
  k_raster_coords<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(a);
  int rc = check_launch("k_raster_coords");
  if (rc) return rc;
  k_raster_boxes<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(a);
  if ((rc = check_launch("k_raster_boxes"))) return rc;
  k_rasterize<<<(unsigned)cdiv(w * h, 256), 256, 0, st>>>(a.us, a.vs, a.box, n, w, h, pixels);
  return check_launch("k_rasterize");
}

int mmlttb_conv_mask(const uint8_t* a, const uint8_t* b, int64_t h, int64_t w, int kernel, uint8_t* mask, void* stream) {
  if (!a || !b || !mask || kernel < 1 || kernel % 2 == 0 || w * h < 1) return fail(MM_EINVAL, "bad arguments");
  k_conv_mask<<<(unsigned)cdiv(w * h, 256), 256, 0, (cudaStream_t)stream>>>(a, b, h, w, kernel, mask);
  return check_launch("k_conv_mask");
}

int mmlttb_pixel_metrics(const uint8_t* a, const uint8_t* b, const uint8_t* mask, int64_t h, int64_t w, int margin,
                         double* out4, void* workspace, int64_t workspace_bytes, void* stream) {
  if (!a || !b || !mask || !out4 || h < 8 || w < 8 || margin < 0 || margin > 255) return fail(MM_EINVAL, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  Carve cv{(char*)workspace, workspace_bytes};
  double* m5 = cv.take<double>(5 * w * h);
  const int64_t nb = cdiv(w * h, 256);
  double* part = cv.take<double>(2 * nb);
  if (!cv.ok) return fail(MM_EWORKSPACE, "workspace too small");
  k_ssim_rows<<<(unsigned)nb, 256, 0, st>>>(a, b, h, w, m5);
  int rc = check_launch("k_ssim_rows");
  if (rc) return rc;
  k_ssim_cols<<<(unsigned)nb, 256, 0, st>>>(a, b, mask, h, w, m5, part);
  if ((rc = check_launch("k_ssim_cols"))) return rc;
  k_metrics_final<<<1, 256, 0, st>>>(a, b, mask, w * h, margin, part, nb, out4);
  return check_launch("k_metrics_final");
}

int mmlttb_validate(const void* x, int x_dtype, const void* y, int y_dtype, int64_t N, int32_t* flags, void* stream) {
  if (!x || !y || !flags || N < 1 || !xdt_ok(x_dtype) || !ydt_ok(y_dtype)) return fail(MM_EINVAL, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(flags, 0, sizeof(int32_t), st) != cudaSuccess) return fail(MM_ECUDA, "memset");
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(N, 256), 148 * 16);
#define MM_V(XT, YT) k_validate<XT, YT><<<blocks, 256, 0, st>>>((const XT*)x, (const YT*)y, N, (int*)flags)
  if (y_dtype == MM_F32) {
    switch (x_dtype) {
      case MM_F32: MM_V(float, float); break;
      case MM_F64: MM_V(double, float); break;
      case MM_I64: MM_V(long long, float); break;
      default: MM_V(int, float); break;
    }
  } else {
    switch (x_dtype) {
      case MM_F32: MM_V(float, double); break;
      case MM_F64: MM_V(double, double); break;
      case MM_I64: MM_V(long long, double); break;
      default: MM_V(int, double); break;
    }
  }
#undef MM_V
  return check_launch("k_validate");
}

}  // extern "C"
