// host.cuh -- host-side helpers shared by the translation units behind
// include/mmlttb.h (capi.cu: the extern "C" entries; k1_launch.cu,
// lttb_launch.cu, fused_launch.cu, post_launch.cu: the kernel launchers,
// compiled in parallel).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <array>
#include <string>
#include <vector>

#include "../../include/mmlttb.h"
#include "kernels.cuh"
#include "fused.cuh"

using namespace mm;
namespace mm { struct K23Args; }

namespace mmh {

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
extern std::atomic<int64_t> g_launches;
int check_launch(const char* what);
void stage_mark(cudaStream_t st, int i);

constexpr int64_t ALIGN = 256;
constexpr int MM_ENOTSUP = -100;  // internal: a fast path declines, the caller falls back (never returned by the C ABI)
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
  int64_t nt = 0;                 // tile mode (nt > 0): tile CTAs per series, partial stride CP
};

// Chunks per bucket: enough warps for ~4 waves over 148 SMs x 32 resident
// warps, never a chunk under MIN_CHUNK elements; buckets of <= 4096 points
// are one item each (8-lane groups).  Large buckets of closed-form partitions
// use the flat split (k_extrema_flat): equal element ranges per warp.
constexpr int64_t SMALL_BUCKET = 4096;  // elements: <= this -> one 8-lane group per bucket

inline int64_t env_i64(const char* name, int64_t dflt) {
  const char* e = getenv(name);  // tuning knobs for tools/*.sh only
  return e ? atoll(e) : dflt;
}

int sm_count();  // of the current device (148 on B200; 148 when no device is present)

inline int64_t dyn_chunk_elems() {
  // measured and not adopted: 4096 / 8192 / 16384-element chunks made C3 K1 93 / 83 / 84 us vs
  // 75 us with one range per warp (each new chunk restarts the load pipeline)
  static const int64_t v = env_i64("MMLTTB_K1_DYN_CHUNK", 0);
  return v;
}
inline ExPlan plan_extrema(int64_t buckets_total, int64_t max_bucket, int ydt, int64_t B = 0, bool closed_form = false,
                           bool dyn = false) {
  // tuned on B200 (tools/plan_sweep.sh): ~4 waves of 148 SMs x 32 resident
  // warps, chunks of >= 4096 float32 elements
  const int64_t nsm = sm_count();
  static const int64_t want_env = env_i64("MMLTTB_K1_WANT_WARPS", -1);
  const int64_t want = want_env >= 0 ? want_env : nsm * 128;
  static const int64_t minc32 = env_i64("MMLTTB_K1_MIN_CHUNK", 4096);
  // flat split: one wave of 148 SMs x 24 resident warps (80 regs), two for
  // very long series (tools/flat_sweep.sh)
  static const int64_t flat_env = env_i64("MMLTTB_K1_FLAT_WARPS", -1);
  // ticketed flat K1 (when the caller provides a zeroed ticket): chunk length in
  // float32-equivalent elements (A/B knob MMLTTB_K1_DYN_CHUNK; 0 = one range per warp)
  const int64_t dyn_chunk = dyn ? dyn_chunk_elems() : 0;
  const int64_t min_chunk = ydt == MM_F32 ? minc32 : minc32 / 2;
  ExPlan p;
  const int64_t nb_ = B > 0 ? buckets_total / B : 0;
  const int64_t flat_warps = flat_env >= 0 ? flat_env : (nb_ * max_bucket > 400000000LL ? nsm * 48 : nsm * 24);
  // flat split above this many elements per bucket (A/B knob MMLTTB_K1_FLAT_MIN; measured on
  // C3 r=32, 3,128-point buckets: 8-lane groups 117.6 us vs flat 126.8 us per call)
  static const int64_t flat_min = env_i64("MMLTTB_K1_FLAT_MIN", SMALL_BUCKET);
#ifdef MMLTTB_AB
  // tile mode (k1_tiles.cuh, tuning build only): 32 KB tile CTAs, sub-buckets of >= one
  // warp's elements (1,024 float32 / 512 float64); knobs MMLTTB_K1_TILES=1,
  // MMLTTB_K1_TILES_MIN (smallest sub-bucket, elements).  Measured and not adopted:
  // C3 K1 124 vs 72 us, 1e9 1.10 vs 0.58 ms -- issue-bound (profiles/r02/k1_tiles.md)
  static const bool tiles_on = env_i64("MMLTTB_K1_TILES", 0) != 0;
  static const int64_t tiles_min = env_i64("MMLTTB_K1_TILES_MIN", SMALL_BUCKET);
  const int64_t vec = ydt == MM_F32 ? 4 : 2, tile_el = 2048 * vec;
  if (closed_form && B > 0 && tiles_on && max_bucket - 1 >= std::max<int64_t>(tiles_min, 256 * vec)) {
    const int64_t nb = nb_;
    p.nt = std::max<int64_t>(1, cdiv(nb * max_bucket / vec, 2048));
    p.CP = cdiv(max_bucket, tile_el) + 2;
    p.C = 1;
    p.chunk = max_bucket;
    p.Cmax = p.CP;
    return p;
  }
#endif
  if (closed_form && B > 0 && max_bucket > flat_min && flat_warps > 0) {
    const int64_t nb = nb_;
    p.Ws = std::max<int64_t>(1, flat_warps / B);
    p.E = std::max<int64_t>(min_chunk, cdiv(nb * max_bucket, p.Ws));
    if (dyn_chunk > 0) p.E = std::min<int64_t>(p.E, dyn_chunk * (ydt == MM_F32 ? 1 : 2) / 2 * 2);  // ticketed chunks
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
inline int64_t ex_ws(int64_t nbt, const ExPlan& p) {
  int64_t b = up(nbt * (int64_t)sizeof(Ext)) + up(nbt);
  if (p.Cmax > 1) b += up(nbt * p.Cmax * (int64_t)sizeof(Partial)) + up(nbt * 4);
  return b;
}

inline bool carve_ex(Carve& cv, int64_t nbt, const ExPlan& p, ExArgs& a) {
  a.E = p.E;
  a.Ws = p.Ws;
  a.CP = p.CP;
  a.nt = p.nt;
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


// Opt a kernel into `bytes` of dynamic shared memory.  The attribute is per
// device (context), so each launch site keeps one bit per device in `mask`.
inline int smem_optin(std::atomic<unsigned long long>& mask, const void* kern, int bytes, const char* what) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(MM_ECUDA, "cudaGetDevice");
  const unsigned long long bit = dev < 64 ? 1ULL << dev : 0ULL;
  if (bit && (mask.load(std::memory_order_acquire) & bit)) return MM_OK;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return fail(MM_ECUDA, "cudaFuncSetAttribute(%s)", what);
  mask.fetch_or(bit, std::memory_order_acq_rel);
  return MM_OK;
}

inline bool mul_ok(int64_t a, int64_t b) { return a == 0 || b <= INT64_MAX / a; }

// ---- K1 (k1_launch.cu) ----
int launch_extrema(const ExArgs& a, int ydt, cudaStream_t st);

// ---- K3 (lttb_launch.cu) ----
// Buckets of <= 64 points: exact transition tables over all points (K3a).
// Larger buckets: candidate tables + full verification + repair (K3c).
constexpr int NBB = 32;   // buckets per k_lttb_tables block
constexpr int HMAX = 32;  // K3c workspace bound: <= 2 x 16 sampled directions per bucket
inline int smax_for(int64_t s) {
  if (s <= 4) return 4;
  if (s <= 8) return 8;
  if (s <= 16) return 16;
  if (s <= 32) return 32;
  if (s <= 64) return 64;
  return 0;
}
inline bool use_tables(int64_t s) { return smax_for(s) > 0; }
inline int64_t tab_ld(int64_t k3, int smax) { return (k3 * smax + 15) / 16 * 16; }
// K3c flat passes (B == 1): one wave of warps, partial slots per bucket
inline int64_t k3c_flat_warps() { return (int64_t)sm_count() * 24; }
constexpr int64_t K3C_FLAT_PART = 256;  // bytes per (bucket, warp) partial, >= every pass's partial
inline int64_t flat_cp_max(int64_t k3) { return (k3c_flat_warps() * 65 / 64 + k3 - 1) / k3 + 3; }
int64_t lttb_ws(int64_t B, int64_t n_out, int64_t s);
int launch_lttb(LttbArgs a, int xdt, int ydt, int64_t s, cudaStream_t st);
int64_t repair_scans_read();

// ---- fused batch kernel (fused_launch.cu) ----
bool fused_ok(int64_t B, int64_t N, int64_t n_out, int64_t r_ps, int ydt);
int launch_fused(const FusedArgs& fa, int xdt, int ydt, cudaStream_t st);

// ---- K2 + K3 of one series in one cooperative launch (k23.cuh, k23_launch.cu) ----
bool k23_ok(int64_t B, int64_t k, int64_t n_out, int64_t r_ps);
int64_t k23_ws();
int launch_k23(K23Args a, int xdt, int ydt, int64_t r_ps, cudaStream_t st);

// ---- K2 + K3 single-CTA (post_launch.cu) ----
constexpr int PAIR_NT = 128, PAIR_ITEMS = 2;
bool post_ok(int64_t k, int64_t n_out, int64_t r_ps);
int launch_post(const PostArgs& pa, int64_t B, int xdt, int ydt, int smax, cudaStream_t st);

}  // namespace mmh

using namespace mmh;
