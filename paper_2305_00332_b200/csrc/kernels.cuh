// kernels.cuh -- sm_100a device code for the MinMaxLTTB path.
//
// K1  k_extrema        streaming first-occurrence argmin/argmax per
//                      (series, sub-bucket, chunk): _kernels.py:22-78
// K2  k_compact        per-series combine of K1 partials, (lo,hi) emission
//                      with dedup, endpoints, exclusive scan, gather of the
//                      preselected (x,y) as f64: downsamplers.py:60-69,
//                      135-161, 164-179, 95-112; core.py:103-105
// K3a k_lttb_tables +  LTTB over small buckets as transition tables
//     k_lttb_jump      T_b[p] = argmax_j area(P_p, P_j, C_{b+1}) built in
//                      parallel, the bucket chain resolved by pointer
//                      jumping in shared memory: _kernels.py:81-119
// K3c k_lttb_means_flat LTTB over large buckets (> 64 points, e.g. full
//     -> dircand ->    `lttb`): certified any-order means, direction-sampled
//     ctables -> scan  candidates, candidate tables + scan, every bucket
//     -> verify_flat   re-scanned exactly (verify), speculative next-bucket
//     -> verify2 ->    picks (verify2) and a repair walk: exact whatever the
//     repair_smem      heuristic (_kernels.py:81-119)
// K3b k_lttb_means +   (A/B knob only) in-order means, then one CTA walks
//     k_lttb_chain     the chain evaluating each bucket's areas
//
// Arithmetic parity: extrema compare IEEE total-order
// integer keys (-0.0 < +0.0; f32 keys order exactly like the f64 keys the
// reference builds); LTTB is strict IEEE fp64 through __dadd_rn / __dsub_rn /
// __dmul_rn / __ddiv_rn (never contracted to FMA), bucket sums in index
// order, strict '>' with lowest index on ties and NaN never winning.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <limits.h>
#include <string.h>

namespace mm {

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------- keys ----
// _kernels.py:22-25 restated for the storage width: bits ^ ((bits>>63)&MAG).
// `b` must be SIGNED so that >> is arithmetic (SURVEY §7 hard part 2).
__device__ __forceinline__ int32_t key32(uint32_t u) {
  const int32_t b = (int32_t)u;
  return b ^ ((b >> 31) & 0x7fffffff);
}
__device__ __forceinline__ long long key64(unsigned long long u) {
  const long long b = (long long)u;
  return b ^ ((b >> 63) & 0x7fffffffffffffffLL);
}

// 16-byte streaming loads; LDV picks the cache policy (tuned on B200, see
// 0 = nc + no L1 allocate + 256B L2 prefetch, 1 = nc + no L1
// allocate, 2 = plain nc (__ldg), 3 = evict-first streaming (__ldcs)).
template <int LDV>
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  if constexpr (LDV == 0) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  } else if constexpr (LDV == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  } else if constexpr (LDV == 2) {
    r = __ldg(p);
  } else {
    r = __ldcs(p);
  }
  return r;
}

template <typename T> struct YTr;
template <> struct YTr<float> {
  typedef int32_t K;
  static constexpr int VEC = 4;
  static __device__ __forceinline__ K kmax() { return 0x7fffffff; }
  static __device__ __forceinline__ K kmin() { return (K)0x80000000; }
  static __device__ __forceinline__ K key(const float* p) { return key32(__float_as_uint(__ldg(p))); }
  static __device__ __forceinline__ void keys(const uint4& v, K* k) {
    k[0] = key32(v.x); k[1] = key32(v.y); k[2] = key32(v.z); k[3] = key32(v.w);
  }
};
template <> struct YTr<double> {
  typedef long long K;
  static constexpr int VEC = 2;
  static __device__ __forceinline__ K kmax() { return 0x7fffffffffffffffLL; }
  static __device__ __forceinline__ K kmin() { return (K)0x8000000000000000ULL; }
  static __device__ __forceinline__ K key(const double* p) {
    return key64((unsigned long long)__double_as_longlong(__ldg(p)));
  }
  static __device__ __forceinline__ void keys(const uint4& v, K* k) {
    k[0] = key64(((unsigned long long)v.y << 32) | v.x);
    k[1] = key64(((unsigned long long)v.w << 32) | v.z);
  }
};

// element -> f64 exactly as np.array(values, dtype=float64) (core.py:49)
template <typename T> __device__ __forceinline__ double to_f64(const T* p, int64_t i);
template <> __device__ __forceinline__ double to_f64<float>(const float* p, int64_t i) { return (double)__ldg(p + i); }
template <> __device__ __forceinline__ double to_f64<double>(const double* p, int64_t i) { return __ldg(p + i); }
template <> __device__ __forceinline__ double to_f64<long long>(const long long* p, int64_t i) {
  return __ll2double_rn(__ldg(p + i));
}
template <> __device__ __forceinline__ double to_f64<int>(const int* p, int64_t i) { return (double)__ldg(p + i); }

// Non-finite detection for free: every NaN/inf maps outside the open key
// interval (key(-inf), key(+inf)), so a bucket holds one iff its min key is
// <= key(-inf) or its max key >= key(+inf) (TimeSeries check, core.py:89-90).
__device__ __forceinline__ bool keys_nonfinite(long long kmin, long long kmax, int ydt) {
  if (ydt == 0) return kmin <= (long long)(int32_t)0x807fffff || kmax >= 0x7f800000LL;
  return kmin <= (long long)0x800fffffffffffffULL || kmax >= 0x7ff0000000000000LL;
}

// ------------------------------------------------------- K1 partials ----
struct Partial {
  long long kmin, kmax;  // total-order keys (sign-extended for f32)
  long long imin, imax;  // element index (INT64_MAX = none)
};

struct Ext;
struct ExArgs {
  const void* y;
  int64_t y_ld;
  int64_t B;
  int64_t start, len, k;   // closed-form partition(start, start+len, k) (core.py:173)
  const int64_t* bounds;   // or explicit bounds (k+1 entries), shared by all series
  int64_t b0, nb;          // buckets [b0, b0+nb) of every series
  int64_t C, chunk;        // chunks per bucket, chunk length (elements)
  Partial* part;           // [B][nb][C]   chunk partials (C > 1 only)
  unsigned* arrivals;      // [B][nb]      zeroed per call (C > 1 only)
  struct Ext* ext;         // [B][nb]      final (imin, imax) per bucket
  unsigned char* cnt8;     // [B][nb]      1 + (imin != imax): K2's scan input
  int64_t E, Ws, CP;       // flat mode: elements per warp, warps per series, partial stride
  int arrivals_zeroed;     // the caller zeroed `arrivals` (merged into its own memset)
  unsigned* ticket;        // flat mode: chunk ticket (zeroed per call) -> persistent warps take
                           // chunks dynamically; null: one static range per warp
  int64_t nt;              // tile mode (k1_tiles.cuh, nt > 0): tile CTAs per series (an upper
                           // bound), partial stride CP
  int64_t e_lo, e_hi;      // tile mode: [pbound(b0), pbound(b0 + nb)) (set by the launcher)
  double rlen, rk;         // tile mode: 1/len, 1/k (division-free bucket arithmetic)
};

struct Ext {
  long long imin, imax;  // first-occurrence argmin / argmax
  long long kmin, kmax;  // their total-order keys: the key map is an involution,
                         // so K2 recovers y[imin], y[imax] without a gather
};

// value of a total-order key (inverse of key32/key64: the same xor)
template <typename T> __device__ __forceinline__ double key_value(long long k);
template <> __device__ __forceinline__ double key_value<float>(long long k) {
  return (double)__int_as_float(key32((uint32_t)(int32_t)k));
}
template <> __device__ __forceinline__ double key_value<double>(long long k) {
  return __longlong_as_double(key64((unsigned long long)k));
}

__device__ __forceinline__ int64_t pbound(int64_t start, int64_t len, int64_t k, int64_t b) {
  return start + (b * len) / k;  // core.py:173 (host guarantees k*len < 2^63)
}

// First-occurrence argmin/argmax (total-order keys) of y[lo, hi) by a group
// of G lanes (lane = index within the group).  Offsets are int32 relative to
// lo (INT_MAX = empty range); results are reduced across the group.  When a
// vector improves the running extreme its raw 16 bytes are kept in
// registers, so the exact element is recovered without re-reading memory (a
// re-read would miss L2 on a long stream and cost extra DRAM traffic).
template <typename T, int U, int LDV, int G, bool KEEPRAW = true, bool PF = false>
__device__ __forceinline__ void group_extrema(const T* y, int64_t lo, int64_t hi, int lane, typename YTr<T>::K& mn,
                                              int& omn, typename YTr<T>::K& mx, int& omx) {
  typedef YTr<T> Tr;
  typedef typename Tr::K K;
  mn = Tr::kmax();
  mx = Tr::kmin();
  omn = INT_MAX;
  omx = INT_MAX;
  bool vmn = false, vmx = false;
  uint4 rmn = make_uint4(0, 0, 0, 0), rmx = make_uint4(0, 0, 0, 0);
  if (lo < hi) {
    const int n = (int)(hi - lo);
    const T* base = y + lo;
    const uintptr_t addr = (uintptr_t)base;
    int head = (int)(((16u - (unsigned)(addr & 15u)) & 15u) / sizeof(T));
    if (head > n) head = n;
    if (lane < head) {
      const K kk = Tr::key(base + lane);
      mn = kk; mx = kk; omn = omx = lane;
    }
    const int nvec = (n - head) / Tr::VEC;
    const uint4* vp = reinterpret_cast<const uint4*>(base + head);
    auto ld_round = [&](uint4 (&r)[U], int v0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * G + lane;
        if (v < nvec) r[u] = ld_stream<LDV>(vp + v);
      }
    };
    auto use_round = [&](const uint4 (&r)[U], int v0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * G + lane;
        if (v < nvec) {
          K kk[Tr::VEC];
          Tr::keys(r[u], kk);
          K vl = kk[0], vh = kk[0];
#pragma unroll
          for (int e = 1; e < Tr::VEC; ++e) { vl = min(vl, kk[e]); vh = max(vh, kk[e]); }
          if (vl < mn) { mn = vl; omn = head + v * Tr::VEC; vmn = true; if (KEEPRAW) rmn = r[u]; }
          if (vh > mx) { mx = vh; omx = head + v * Tr::VEC; vmx = true; if (KEEPRAW) rmx = r[u]; }
        }
      }
    };
    if constexpr (PF) {  // register double buffer: round i+1's loads in flight while round i is reduced
      uint4 ra[U], rb[U];
      if (nvec > 0) ld_round(ra, 0);
      for (int v0 = 0; v0 < nvec; v0 += 2 * G * U) {
        if (v0 + G * U < nvec) ld_round(rb, v0 + G * U);
        use_round(ra, v0);
        if (v0 + 2 * G * U < nvec) ld_round(ra, v0 + 2 * G * U);
        if (v0 + G * U < nvec) use_round(rb, v0 + G * U);
      }
    } else {
      for (int v0 = 0; v0 < nvec; v0 += G * U) {
        uint4 r[U];
        ld_round(r, v0);
        use_round(r, v0);
      }
    }
    if (!KEEPRAW) {  // short ranges read with normal L2 policy: the vectors are still cached
      if (vmn) rmn = __ldg(reinterpret_cast<const uint4*>(base + omn));
      if (vmx) rmx = __ldg(reinterpret_cast<const uint4*>(base + omx));
    }
    const int tp = head + nvec * Tr::VEC + lane;
    if (tp < n) {
      const K kk = Tr::key(base + tp);
      if (kk < mn) { mn = kk; omn = tp; vmn = false; }
      if (kk > mx) { mx = kk; omx = tp; vmx = false; }
    }
    // exact element inside the winning vector: first component with the key
    if (vmn) {
      K kk[Tr::VEC];
      Tr::keys(rmn, kk);
      int e = Tr::VEC - 1;
#pragma unroll
      for (int q = Tr::VEC - 1; q >= 0; --q) if (kk[q] == mn) e = q;
      omn += e;
    }
    if (vmx) {
      K kk[Tr::VEC];
      Tr::keys(rmx, kk);
      int e = Tr::VEC - 1;
#pragma unroll
      for (int q = Tr::VEC - 1; q >= 0; --q) if (kk[q] == mx) e = q;
      omx += e;
    }
  }
#pragma unroll
  for (int off = G / 2; off; off >>= 1) {
    const K omn2 = __shfl_xor_sync(FULL, mn, off);
    const int oo = __shfl_xor_sync(FULL, omn, off);
    if (omn2 < mn || (omn2 == mn && oo < omn)) { mn = omn2; omn = oo; }
    const K omx2 = __shfl_xor_sync(FULL, mx, off);
    const int oq = __shfl_xor_sync(FULL, omx, off);
    if (omx2 > mx || (omx2 == mx && oq < omx)) { mx = omx2; omx = oq; }
  }
}

__device__ __forceinline__ void write_ext(const ExArgs& a, int64_t bkt, int64_t pmn, int64_t pmx, long long kmn,
                                          long long kmx) {
  a.ext[bkt].imin = pmn;
  a.ext[bkt].imax = pmx;
  a.ext[bkt].kmin = kmn;
  a.ext[bkt].kmax = kmx;
  a.cnt8[bkt] = (unsigned char)(pmn != pmx ? 2 : 1);
}

// Partial `slot` (of `target` contributors) of bucket `bkt`: the last warp to
// arrive combines all partials lexicographically and writes the Ext (whole
// warp must call; lane 0 publishes).
__device__ __forceinline__ void publish_partial(const ExArgs& a, int64_t bkt, int64_t slot, int64_t stride,
                                                int64_t target, long long mn, long long mx, int64_t pmn,
                                                int64_t pmx, int lane) {
  if (target == 1) {
    if (lane == 0) write_ext(a, bkt, pmn, pmx, mn, mx);
    return;
  }
  unsigned last = 0;
  if (lane == 0) {
    Partial p;
    p.kmin = mn; p.kmax = mx; p.imin = pmn; p.imax = pmx;
    a.part[bkt * stride + slot] = p;
    __threadfence();
    last = atomicAdd(&a.arrivals[bkt], 1u) == (unsigned)(target - 1);
  }
  last = __shfl_sync(FULL, last, 0);
  if (!last) return;
  __threadfence();
  long long cmn = LLONG_MAX, cmx = LLONG_MIN;
  int64_t cimn = INT64_MAX, cimx = INT64_MAX;
  const Partial* pp = a.part + bkt * stride;
  for (int64_t c2 = lane; c2 < target; c2 += 32) {
    const long long kmn = __ldcg(&pp[c2].kmin), kmx = __ldcg(&pp[c2].kmax);
    const long long qmn = __ldcg(&pp[c2].imin), qmx = __ldcg(&pp[c2].imax);
    if (kmn < cmn || (kmn == cmn && qmn < cimn)) { cmn = kmn; cimn = qmn; }
    if (kmx > cmx || (kmx == cmx && qmx < cimx)) { cmx = kmx; cimx = qmx; }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const long long omn = __shfl_xor_sync(FULL, cmn, off);
    const int64_t oimn = __shfl_xor_sync(FULL, cimn, off);
    if (omn < cmn || (omn == cmn && oimn < cimn)) { cmn = omn; cimn = oimn; }
    const long long omx = __shfl_xor_sync(FULL, cmx, off);
    const int64_t oimx = __shfl_xor_sync(FULL, cimx, off);
    if (omx > cmx || (omx == cmx && oimx < cimx)) { cmx = omx; cimx = oimx; }
  }
  if (lane == 0) {
    write_ext(a, bkt, cimn, cimx, cmn, cmx);
    a.arrivals[bkt] = 0;  // leave the counter reusable
  }
}

// Flat K1 (large buckets): warp w of series s streams the contiguous element
// range [E_lo + w*E, E_lo + (w+1)*E) whatever the bucket edges, so every warp
// does the same work (no last-wave tail); a range spanning bucket edges
// publishes one partial per intersected bucket (slot = w - first warp of the
// bucket), combined by the bucket's last-arriving warp.
template <typename T, int U, int LDV, bool PF = false>
__device__ __forceinline__ void flat_range(const ExArgs& a, int64_t w, int lane) {
  typedef YTr<T> Tr;
  typedef typename Tr::K K;
  const int64_t s = w / a.Ws, wl = w % a.Ws;
  const T* y = (const T*)a.y + s * a.y_ld;
  const int64_t E_lo = pbound(a.start, a.len, a.k, a.b0), E_hi = pbound(a.start, a.len, a.k, a.b0 + a.nb);
  const int64_t e0 = E_lo + wl * a.E;
  const int64_t e1 = min(E_hi, e0 + a.E);
  if (e0 >= e1) return;
  // bucket of e0 in partition(start, start+len, k): floor(((e0-start+1)*k - 1) / len)
  int64_t b = (((e0 - a.start + 1) * a.k) - 1) / a.len;
  for (;;) {
    const int64_t blo = pbound(a.start, a.len, a.k, b), bhi = pbound(a.start, a.len, a.k, b + 1);
    const int64_t lo = max(e0, blo), hi = min(e1, bhi);
    K mn, mx;
    int omn, omx;
    group_extrema<T, U, LDV, 32, true, PF>(y, lo, hi, lane, mn, omn, mx, omx);
    const int64_t pmn = omn == INT_MAX ? INT64_MAX : lo + omn;
    const int64_t pmx = omx == INT_MAX ? INT64_MAX : lo + omx;
    const int64_t wf = (max(blo, E_lo) - E_lo) / a.E;
    const int64_t wt = (min(bhi, E_hi) - 1 - E_lo) / a.E;
    publish_partial(a, s * a.nb + (b - a.b0), wl - wf, a.CP, wt - wf + 1, (long long)mn, (long long)mx, pmn, pmx,
                    lane);
    if (bhi >= e1) break;
    ++b;
  }
}

template <typename T, int U, int LDV, int MINB = 3, bool PF = false, bool DYN = false>
__global__ void __launch_bounds__(256, MINB) k_extrema_flat(ExArgs a) {
  const int lane = threadIdx.x & 31;
  if constexpr (DYN) {  // persistent warps take the next range until none is left (no single-wave tail)
    for (;;) {
      unsigned w = 0;
      if (lane == 0) w = atomicAdd(a.ticket, 1u);
      w = __shfl_sync(FULL, w, 0);
      if ((int64_t)w >= a.B * a.Ws) break;
      flat_range<T, U, LDV, PF>(a, (int64_t)w, lane);
    }
    return;
  }
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= a.B * a.Ws) return;  // warp-uniform
  flat_range<T, U, LDV, PF>(a, w, lane);
}

// One warp per (series, bucket, chunk).  Lanes stream 16-byte vectors
// (U in flight per lane), keep a per-lane running min/max KEY plus the
// position of the vector that first reached it (strict < / >, lane order is
// index order => lane-local first occurrence), recover the exact element
// from that vector at the end, then reduce (key, index) lexicographically
// across the warp -- the same first-occurrence argmin/argmax as
// _argminmax_range (_kernels.py:28-60) independent of evaluation order.
//
// G < 32: a G-lane group per item (small buckets, C == 1): 32/G buckets per
// warp, each group still reading G*16 contiguous bytes per load, so a warp's
// fixed costs (bounds, reduction, stores) are shared by several buckets.
template <typename T, int U, int LDV, int MINB = 1, int G = 32>
__global__ void __launch_bounds__(256, MINB) k_extrema(ExArgs a) {
  typedef YTr<T> Tr;
  typedef typename Tr::K K;
  const int lane = threadIdx.x & (G - 1);  // lane within the item's group
  const int64_t w = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 / G) + (threadIdx.x & 31) / G;
  const int64_t total = a.B * a.nb * a.C;
  const bool live = w < total;
  if (G == 32 && !live) return;  // warp-uniform
  const int64_t c = live ? w % a.C : 0;
  const int64_t t = live ? w / a.C : 0;
  const int64_t b = a.b0 + t % a.nb;
  const int64_t s = t / a.nb;
  int64_t blo, bhi;
  if (a.bounds) {
    blo = a.bounds[b];
    bhi = a.bounds[b + 1];
  } else {
    blo = pbound(a.start, a.len, a.k, b);
    bhi = pbound(a.start, a.len, a.k, b + 1);
  }
  const int64_t lo = blo + c * a.chunk;
  const int64_t hi = live ? min(bhi, lo + a.chunk) : lo;
  const T* y = (const T*)a.y + s * a.y_ld;

  K mn, mx;
  int omn, omx;
  group_extrema<T, U, LDV, G>(y, lo, hi, lane, mn, omn, mx, omx);
  const int64_t pmn = omn == INT_MAX ? INT64_MAX : lo + omn;
  const int64_t pmx = omx == INT_MAX ? INT64_MAX : lo + omx;
  // publish: one chunk per bucket -> final; otherwise the last-arriving warp
  // of the bucket combines all C partials (threadfence-reduction pattern), so
  // no separate combine pass and no single-CTA bottleneck downstream.
  if (G < 32 || a.C == 1) {  // (G < 32 is only launched with C == 1)
    if (lane == 0 && live) write_ext(a, t, pmn, pmx, (long long)mn, (long long)mx);
    return;
  }
  publish_partial(a, t, c, a.C, a.C, (long long)mn, (long long)mx, pmn, pmx, lane);
}

// ---------------------------------------------------- block scan helper --
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int& total, int* sh /* >= NT/32+1 ints */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = lane < NT / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, t, o);
      if (lane >= o) t += y;
    }
    if (lane < NT / 32) sh[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  const int before = wid ? sh[wid - 1] : 0;
  total = sh[NT / 32 - 1];
  __syncthreads();
  return before + x - v;
}

// ---------------------------------------------------------- K2 compact ---
struct CompactArgs {
  const Ext* ext;
  int64_t nb;               // per series: nb buckets
  int mode;                 // 0: minmax pairs, 1: m4 quads
  int64_t emit_first;       // index emitted before everything (-1: none)
  int64_t emit_last;        // index emitted after everything (-1: none)
  int64_t force_n_out;      // > 0: _minmax_with_endpoints (downsamplers.py:164-179)
  int64_t last_index;       // N-1 for force mode
  int64_t start, len, k, b0;  // bucket bounds (m4 first/last)
  int64_t* out_idx;
  int64_t out_ld;
  int64_t* out_count;
  const void* x; int xdt; int64_t x_ld; int64_t x_off;  // gather x[i - x_off] (x may be null)
  const void* y; int ydt; int64_t y_ld; int64_t y_off;
  double* out_x;            // may be null
  double* out_y;
  int* status;              // bit 0: non-finite y seen (may be null)
};

__device__ __forceinline__ double load_any(const void* p, int dt, int64_t i) {
  switch (dt) {
    case 0: return (double)__ldg((const float*)p + i);
    case 1: return __ldg((const double*)p + i);
    case 2: return __ll2double_rn(__ldg((const long long*)p + i));
    default: return (double)__ldg((const int*)p + i);
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) k_compact(CompactArgs a) {
  __shared__ int sh[NT / 32 + 1];
  __shared__ long long s_first, s_last, s_m;
  const int64_t s = blockIdx.x;
  const Ext* ext = a.ext + s * a.nb;
  int64_t* out = a.out_idx + s * a.out_ld;
  double* ox = a.out_x ? a.out_x + s * a.out_ld : nullptr;
  double* oy = a.out_y ? a.out_y + s * a.out_ld : nullptr;
  const void* xs = a.x ? (const void*)((const char*)a.x + s * a.x_ld * (a.xdt == 0 || a.xdt == 3 ? 4 : 8)) : nullptr;
  const void* ys = a.y ? (const void*)((const char*)a.y + s * a.y_ld * (a.ydt == 0 || a.ydt == 3 ? 4 : 8)) : nullptr;

  auto put = [&](int64_t pos, int64_t idx) {
    out[pos] = idx;
    if (ox) ox[pos] = load_any(xs, a.xdt, idx - a.x_off);
    if (oy) oy[pos] = load_any(ys, a.ydt, idx - a.y_off);
  };
  auto items_of = [&](int64_t bl, int64_t* it) -> int {
    const int64_t imin = ext[bl].imin, imax = ext[bl].imax;
    if (a.status && keys_nonfinite(ext[bl].kmin, ext[bl].kmax, a.ydt)) atomicOr(a.status, 1);
    const int64_t lo = min(imin, imax), hi = max(imin, imax);
    if (a.mode == 0) {  // downsamplers.py:60-69
      it[0] = lo; it[1] = hi;
      return hi != lo ? 2 : 1;
    }
    // m4: {first, argmin, argmax, last} sorted, adjacent duplicates dropped (:95-112)
    const int64_t b = a.b0 + bl;
    int64_t q[4] = {pbound(a.start, a.len, a.k, b), lo, hi, pbound(a.start, a.len, a.k, b + 1) - 1};
    // q[0] <= lo <= hi <= q[3] already (extrema lie inside the bucket)
    int n = 0;
    it[n++] = q[0];
#pragma unroll
    for (int i = 1; i < 4; ++i) if (q[i] != q[i - 1]) it[n++] = q[i];
    return n;
  };

  // r_ps == 1 endpoint forcing needs the count before placement
  int prepend = 0, replace_first = 0, append = 0, replace_last = 0;
  int64_t m_total = 0;
  if (a.force_n_out > 0) {
    int64_t acc = 0;
    for (int64_t t0 = 0; t0 < a.nb; t0 += NT) {
      const int64_t bl = t0 + threadIdx.x;
      int cnt = 0;
      if (bl < a.nb) { int64_t it[4]; cnt = items_of(bl, it); }
      int tot;
      block_excl_scan<NT>(cnt, tot, sh);
      acc += tot;
    }
    if (threadIdx.x == 0) {
      int64_t it[4];
      items_of(0, it);
      s_first = it[0];
      const int n = items_of(a.nb - 1, it);
      s_last = it[n - 1];
      s_m = acc;
    }
    __syncthreads();
    m_total = s_m;
    if (s_first != 0) { if (m_total < a.force_n_out) prepend = 1; else replace_first = 1; }
    if (s_last != a.last_index) {
      if (m_total + prepend < a.force_n_out) append = 1; else replace_last = 1;
    }
  }

  int64_t carry = (a.emit_first >= 0 ? 1 : 0) + prepend;
  for (int64_t t0 = 0; t0 < a.nb; t0 += NT) {
    const int64_t bl = t0 + threadIdx.x;
    int64_t it[4];
    int cnt = 0;
    if (bl < a.nb) cnt = items_of(bl, it);
    int tot;
    const int ex = block_excl_scan<NT>(cnt, tot, sh);
    for (int i = 0; i < cnt; ++i) put(carry + ex + i, it[i]);
    carry += tot;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (a.emit_first >= 0) put(0, a.emit_first);
    if (a.emit_last >= 0) put(carry++, a.emit_last);
    if (prepend || replace_first) put(0, 0);
    if (append) put(carry++, a.last_index);
    if (replace_last) put(carry - 1, a.last_index);
    a.out_count[s] = carry;
  }
}

// extrema-only finalize for the _extrema_by_bucket entry point
static __global__ void k_finalize_extrema(const Ext* ext, int64_t k, int64_t* out_min, int64_t* out_max) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= k) return;
  out_min[b] = ext[b].imin;
  out_max[b] = ext[b].imax;
}

// K2 (hot path): multi-CTA compaction of (lo, hi) pairs.  CTA (tile, s)
// owns TB = NT*ITEMS consecutive buckets of series s; its output offset is
// the sum of the previous buckets' 1-byte counts (cnt8, written by K1), so
// there is no inter-CTA handshake.  Each thread gathers its <= 2*ITEMS
// preselected (x, y) values with all loads in flight together.
struct PairArgs {
  const Ext* ext;
  const unsigned char* cnt8;
  int64_t nb;
  int64_t emit_first, emit_last;   // -1: none
  int64_t* out_idx; int64_t out_ld; int64_t* out_count;
  const void* x; int xdt; int64_t x_ld;
  const void* y; int ydt; int64_t y_ld;
  double* out_x; double* out_y;    // may be null (no gather)
  int* status;                     // bit 0: non-finite y seen (may be null)
};

// One tile (TB = NT*ITEMS buckets) of series s; `ntiles` tiles per series.
template <typename XT, typename YT, int NT, int ITEMS>
__device__ __forceinline__ void compact_pairs_tile(const PairArgs& a, int64_t s, int64_t tile, int64_t ntiles) {
  __shared__ int sh[NT / 32 + 1];
  __shared__ long long s_red[NT / 32];
  constexpr int TB = NT * ITEMS;
  const int64_t b_lo = tile * TB;
  const unsigned char* cnt = a.cnt8 + s * a.nb;
  const Ext* ext = a.ext + s * a.nb;
  // this thread's Ext records: loaded first, in flight across the prefix sum
  Ext er[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t bl = b_lo + (int64_t)threadIdx.x * ITEMS + i;
    er[i].imin = er[i].imax = er[i].kmin = er[i].kmax = 0;
    if (bl < a.nb) er[i] = ext[bl];
  }
  // 1. offset of this tile = items of buckets [0, b_lo): the 1-byte counts
  //    are summed as masked 32-bit words (independent loads, no byte chain)
  long long pre = 0;
  {
    const uintptr_t base = (uintptr_t)cnt;
    const uintptr_t wb = base & ~(uintptr_t)3, we = (base + (uintptr_t)b_lo + 3) & ~(uintptr_t)3;
    const int64_t nw = (int64_t)((we - wb) >> 2);
    const uint32_t* words = reinterpret_cast<const uint32_t*>(wb);
    for (int64_t i = threadIdx.x; i < nw; i += NT) {
      uint32_t w = words[i];
      const uintptr_t a0 = wb + 4 * (uintptr_t)i;  // bytes [a0, a0+4)
      if (a0 < base) w &= 0xFFFFFFFFu << (8 * (base - a0));
      const uintptr_t end = base + (uintptr_t)b_lo;
      if (a0 + 4 > end) w &= (end > a0) ? (0xFFFFFFFFu >> (8 * (a0 + 4 - end))) : 0u;
      pre += (w & 0xFFu) + ((w >> 8) & 0xFFu) + ((w >> 16) & 0xFFu) + (w >> 24);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) pre += __shfl_xor_sync(FULL, pre, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = pre;
  __syncthreads();
  long long off = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) off += s_red[w];
  // 2. this thread's buckets: slot 2i = lo, 2i+1 = hi (kept if != lo); all
  //    indexing static so everything stays in registers
  int64_t v[2 * ITEMS];
  long long kv[2 * ITEMS];
  bool keep[2 * ITEMS];
  int n = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t bl = b_lo + (int64_t)threadIdx.x * ITEMS + i;
    const bool ok = bl < a.nb;
    const Ext e = er[i];
    if (ok && a.status && keys_nonfinite(e.kmin, e.kmax, a.ydt)) atomicOr(a.status, 1);
    const bool mfirst = e.imin <= e.imax;
    v[2 * i] = mfirst ? e.imin : e.imax;  // downsamplers.py:60-69
    v[2 * i + 1] = mfirst ? e.imax : e.imin;
    kv[2 * i] = mfirst ? e.kmin : e.kmax;
    kv[2 * i + 1] = mfirst ? e.kmax : e.kmin;
    keep[2 * i] = ok;
    keep[2 * i + 1] = ok && v[2 * i + 1] != v[2 * i];
    n += (int)keep[2 * i] + (int)keep[2 * i + 1];
  }
  int tot;
  const int ex = block_excl_scan<NT>(n, tot, sh);
  const int64_t base = (a.emit_first >= 0 ? 1 : 0) + off + ex;
  int64_t* out = a.out_idx + s * a.out_ld;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  if (a.out_x) {
    // all 4*ITEMS gathers in flight at once (templated types: no per-load switch)
    double gx[2 * ITEMS], gy[2 * ITEMS];
#pragma unroll
    for (int j = 0; j < 2 * ITEMS; ++j) {
      gx[j] = keep[j] ? to_f64(xs, v[j]) : 0.0;
      gy[j] = key_value<YT>(kv[j]);  // exact y[v[j]] from its key: no gather
    }
    int64_t pos = base;
#pragma unroll
    for (int j = 0; j < 2 * ITEMS; ++j)
      if (keep[j]) { a.out_x[s * a.out_ld + pos] = gx[j]; a.out_y[s * a.out_ld + pos] = gy[j]; ++pos; }
  }
  {
    int64_t pos = base;
#pragma unroll
    for (int j = 0; j < 2 * ITEMS; ++j)
      if (keep[j]) out[pos++] = v[j];
  }
  // 3. endpoints (downsamplers.py:157-160) and the count
  if (threadIdx.x == 0) {
    auto emit = [&](int64_t pos, int64_t v) {
      out[pos] = v;
      if (a.out_x) {
        a.out_x[s * a.out_ld + pos] = to_f64(xs, v);
        a.out_y[s * a.out_ld + pos] = to_f64(ys, v);
      }
    };
    if (tile == 0 && a.emit_first >= 0) {
      emit(0, a.emit_first);
      if (a.status && !isfinite(to_f64(ys, a.emit_first))) atomicOr(a.status, 1);
    }
    if (tile == ntiles - 1 && a.emit_last >= 0 && a.status && !isfinite(to_f64(ys, a.emit_last)))
      atomicOr(a.status, 1);
    if (tile == ntiles - 1) {
      int64_t end = (a.emit_first >= 0 ? 1 : 0) + off + tot;
      if (a.emit_last >= 0) emit(end++, a.emit_last);
      if (a.out_count) a.out_count[s] = end;
    }
  }
}

template <typename XT, typename YT, int NT, int ITEMS>
__global__ void __launch_bounds__(NT) k_compact_pairs(PairArgs a) {
  compact_pairs_tile<XT, YT, NT, ITEMS>(a, blockIdx.y, blockIdx.x, gridDim.x);
}


// -------------------------------------------------------------- LTTB -----
// Points of series s: x/y typed (XT/YT), count m (device per series or
// fixed), optional map position -> output index (the preselected indices).
// K3c: a bucket whose x values a closed formula reproduces bit-exactly (an
// arange, or evenly spaced timestamps): later passes compute x_j instead of
// loading it (half the bytes per point)
struct XAff {
  double x0, d;         // float x: x_j = fl(x0 + fl((j - lo) * d))
  long long x0i, di;    // integer x: x_j = (double)(x0i + (j - lo) * di), two's complement
  int ok, pad;
};

template <typename XT> struct XForm {
  static constexpr bool integral = false;
  __device__ __forceinline__ static double at(const XAff& f, int64_t t) { return __dadd_rn(f.x0, __dmul_rn((double)t, f.d)); }
};
template <> struct XForm<long long> {
  static constexpr bool integral = true;
  __device__ __forceinline__ static double at(const XAff& f, int64_t t) {
    return __ll2double_rn((long long)((unsigned long long)f.x0i + (unsigned long long)t * (unsigned long long)f.di));
  }
};
template <> struct XForm<int> {
  static constexpr bool integral = true;
  __device__ __forceinline__ static double at(const XAff& f, int64_t t) {
    return __ll2double_rn((long long)((unsigned long long)f.x0i + (unsigned long long)t * (unsigned long long)f.di));
  }
};

struct LttbArgs {
  const void* x; int64_t x_ld;
  const void* y; int64_t y_ld;
  const int64_t* m_dev; int64_t n;   // m_dev ? m_dev[s] : n
  const int64_t* bounds;             // explicit LTTB bounds (B == 1 only) or null
  const int64_t* map; int64_t map_ld;
  int64_t B, n_out;
  int64_t* out;                      // [B][n_out]
  unsigned char* tables; int64_t tab_ld;  // K3a: [B][k3*SMAX]
  double2* means; int64_t means_ld;       // K3b: [B][k3]
  int64_t jump_seg;                       // buckets per shared-memory segment (k_lttb_jump)
  // K3c (large buckets): hull candidates, verification, repair
  int64_t* cand; int64_t cand_ld;         // [B][k3][HMAX] candidate positions (ascending)
  int* cand_cnt;                          // [B][k3]
  int64_t* pos; int64_t pos_ld;           // [B][k3+2] chosen positions (pre-map)
  int64_t* best;                          // [B][k3] exact argmax given pos[b] (verify)
  int* flag;                              // [B][k3] best != pos[b+1]
  int64_t* best2;                         // [B][k3] exact pick of b given anchor best[b-1] (if flag[b-1])
  int* flist; int* fcount;                // [B][k3] flagged buckets (unordered), [B] their count (zeroed)
  int cand_cap;                           // <= HMAX (tests lower it to force repairs)
  double2* yrange;                        // [B][k3] per-bucket (ymin, ymax) (K3c candidates)
  double2* merr;                          // [B][k3] K3c: |exact - approx| bound of means[b] ((0,0): exact), or null
  int cert_force;                         // test knob: treat every non-exact certification as failed
  XAff* xaff;                             // [B][k3] K3c affine-x buckets, or null
  double2* xrange;                        // [B][k3] K3c flat passes: per-bucket (xmin, xmax)
};

__device__ __forceinline__ double lttb_area(double ax, double ay, double cx, double cy, double xj, double yj) {
  // _kernels.py:114: abs((ax - cx) * (ys[j] - ay) - (ax - xs[j]) * (cy - ay)), every op rounded
  return fabs(__dsub_rn(__dmul_rn(__dsub_rn(ax, cx), __dsub_rn(yj, ay)),
                        __dmul_rn(__dsub_rn(ax, xj), __dsub_rn(cy, ay))));
}

// lttb_area as an ordering key: the bit pattern of |area| (non-negative doubles
// order like their values), NaN -> -1 so it never wins -- the reference's
// `area > best_area` from -1.0 without fp64 compares (DSETP issues on B200's
// narrow XU pipe)
__device__ __forceinline__ long long lttb_area_key(double ax, double ay, double cx, double cy, double xj, double yj) {
  const long long k = __double_as_longlong(__dsub_rn(__dmul_rn(__dsub_rn(ax, cx), __dsub_rn(yj, ay)),
                                                     __dmul_rn(__dsub_rn(ax, xj), __dsub_rn(cy, ay)))) &
                      0x7fffffffffffffffLL;
  return k > 0x7ff0000000000000LL ? -1LL : k;
}

// XU-free element arithmetic for the flat passes.  On B200 the fp64 compares
// (DSETP, behind fmin/fmax and `>` on doubles) and the int64 -> f64 / f64 ->
// f32 conversions issue on the narrow XU pipe, which ncu showed saturated
// (109 %) in a first version of these passes while the fp64 pipe idled.
// Maxima are taken on integer keys instead, and conversions use ALU bit tricks.
// order-preserving int64 key of a double (IEEE total order; the map is an involution)
__device__ __forceinline__ long long dkey(double v) {
  const long long b = __double_as_longlong(v);
  return b ^ ((b >> 63) & 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double dkey_inv(long long k) { return __longlong_as_double(k ^ ((k >> 63) & 0x7fffffffffffffffLL)); }
// exact int64 -> f64 for |x| < 2^51: 1.5 * 2^52 + x has x in its low mantissa bits
__device__ __forceinline__ double i2d_magic(long long x) {
  return __dsub_rn(__longlong_as_double(x + 0x4338000000000000LL), 6755399441055744.0);
}
__device__ __forceinline__ bool i2d_magic_ok(long long x) { return (unsigned long long)(x + (1LL << 51)) < (1ULL << 52); }
// element -> f64 exactly as to_f64 (numpy's conversion)
template <typename T> __device__ __forceinline__ double elem_f64(T v) { return (double)v; }
template <> __device__ __forceinline__ double elem_f64<long long>(long long v) {
  return i2d_magic_ok(v) ? i2d_magic(v) : __ll2double_rn(v);
}
template <> __device__ __forceinline__ double elem_f64<int>(int v) { return i2d_magic((long long)v); }
// f64 -> f32 by truncation (candidate heuristic only): sign, rebased exponent,
// top 23 mantissa bits; underflow -> +-0, overflow -> +-FLT_MAX
__device__ __forceinline__ float d2f_trunc(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned hi = (unsigned)(b >> 32);
  const int e = (int)((hi >> 20) & 0x7ff) - 1023 + 127;
  const unsigned sg = hi & 0x80000000u;
  unsigned r = sg | ((unsigned)e << 23) | (unsigned)((b >> 29) & 0x7fffff);
  r = e <= 0 ? sg : r;
  r = e >= 255 ? (sg | 0x7f7fffffu) : r;
  return __uint_as_float(r);
}
// |T| as a non-negative key; NaN -> -1 (never wins, like the reference's `>`)
__device__ __forceinline__ long long area_key(double t, int& bad) {
  long long k = __double_as_longlong(t) & 0x7fffffffffffffffLL;
  if (k >= 0x7ff0000000000000LL) bad = 1;  // inf or NaN: no certification
  return k > 0x7ff0000000000000LL ? -1LL : k;
}

struct VPart { long long k1, k2, i1; int bad, pad; };

__device__ __forceinline__ void vpart_merge(long long& k1, long long& i1, long long& k2, int& bad, long long o1,
                                            long long oi, long long o2, int ob) {
  const bool take = o1 > k1 || (o1 == k1 && oi < i1);
  const long long lose = take ? k1 : o1;
  k2 = max(max(k2, o2), lose);
  if (take) { k1 = o1; i1 = oi; }
  bad |= ob;
}

__device__ __forceinline__ int64_t lbound(const LttbArgs& a, int64_t m, int64_t b) {
  if (a.bounds) return a.bounds[b];
  return 1 + (b * (m - 2)) / (a.n_out - 2);  // partition(1, m-1, n_out-2), downsamplers.py:129
}

// mean point of bucket b+1 (in-order fp64 sums, _kernels.py:95-104), or the
// last point for the final bucket (:105-107)
template <typename XT, typename YT>
__device__ __forceinline__ double2 lttb_next_mean(const LttbArgs& a, const XT* xs, const YT* ys, int64_t m, int64_t b) {
  const int64_t k3 = a.n_out - 2;
  double2 c;
  if (b + 1 < k3) {
    const int64_t nlo = lbound(a, m, b + 1), nhi = lbound(a, m, b + 2);
    double sx = 0.0, sy = 0.0;
    for (int64_t j = nlo; j < nhi; ++j) {
      sx = __dadd_rn(sx, to_f64(xs, j));
      sy = __dadd_rn(sy, to_f64(ys, j));
    }
    const double cnt = (double)(nhi - nlo);
    c.x = __ddiv_rn(sx, cnt);
    c.y = __ddiv_rn(sy, cnt);
  } else {
    c.x = to_f64(xs, m - 1);
    c.y = to_f64(ys, m - 1);
  }
  return c;
}

// K3a, part 1: T_b[p] for every bucket b and every predecessor candidate p
// (bucket b-1's points; bucket 0's only predecessor is point 0).
// Block = NBB consecutive buckets of one series.
template <typename XT, typename YT, int SMAX, int NBB>
__global__ void __launch_bounds__(NBB * SMAX < 1024 ? NBB * SMAX : 1024) k_lttb_tables(LttbArgs a) {
  // the points of buckets bb-1 .. bb+nbk (anchors, candidates, next-bucket means)
  // are staged in shared memory once, so no thread waits on a chain of loads
  constexpr int PMAX = (NBB + 2) * SMAX + 2;
  __shared__ double s_x[PMAX], s_y[PMAX];
  __shared__ double2 s_mean[NBB];
  __shared__ int64_t s_bnd[NBB + 3];
  const int64_t s = blockIdx.y;
  const int64_t k3 = a.n_out - 2;
  const int64_t bb = (int64_t)blockIdx.x * NBB;
  if (bb >= k3) return;
  const int64_t m = a.m_dev ? a.m_dev[s] : a.n;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  const int nbk = (int)(k3 - bb < NBB ? k3 - bb : (int64_t)NBB);
  // s_bnd[i + 1] = lbound(bb + i), i = -1 .. nbk + 1 (lbound(k3) = m - 1; past it: m)
  for (int i = threadIdx.x; i <= nbk + 2; i += blockDim.x) {
    const int64_t b = bb - 1 + i;
    s_bnd[i] = b < 0 ? 0 : (b <= k3 ? lbound(a, m, b) : m);
  }
  __syncthreads();
  const int64_t lo0 = s_bnd[0];  // anchors of bucket bb (point 0 when bb == 0)
  const int64_t hi0 = bb + nbk >= k3 ? m : s_bnd[nbk + 2];  // through the next bucket, or the last point
  const int np = (int)(hi0 - lo0);
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    s_x[i] = to_f64(xs, lo0 + i);
    s_y[i] = to_f64(ys, lo0 + i);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbk; i += blockDim.x) {  // next-bucket means, in-order fp64 sums (_kernels.py:95-107)
    const int64_t b = bb + i;
    double2 c;
    if (b + 1 < k3) {
      const int64_t nlo = s_bnd[i + 2], nhi = s_bnd[i + 3];
      double sx = 0.0, sy = 0.0;
      for (int64_t jj = nlo; jj < nhi; ++jj) {
        sx = __dadd_rn(sx, s_x[jj - lo0]);
        sy = __dadd_rn(sy, s_y[jj - lo0]);
      }
      const double cnt = (double)(nhi - nlo);
      c = make_double2(__ddiv_rn(sx, cnt), __ddiv_rn(sy, cnt));
    } else {
      c = make_double2(s_x[m - 1 - lo0], s_y[m - 1 - lo0]);
    }
    s_mean[i] = c;
  }
  __syncthreads();
  unsigned char* tab = a.tables + s * a.tab_ld + bb * SMAX;
  for (int it = threadIdx.x; it < nbk * SMAX; it += blockDim.x) {
    const int bi = it / SMAX, p = it % SMAX;
    const int64_t b = bb + bi;
    const int64_t blo = s_bnd[bi + 1], bhi = s_bnd[bi + 2];
    int64_t ap;
    bool valid;
    if (b == 0) { valid = (p == 0); ap = 0; }
    else { const int64_t plo = s_bnd[bi]; valid = p < s_bnd[bi + 1] - plo; ap = plo + p; }
    unsigned char r = 0;
    if (valid) {
      const double ax = s_x[ap - lo0], ay = s_y[ap - lo0];
      const double2 c = s_mean[bi];
      long long best = -1;
      for (int64_t jj = blo; jj < bhi; ++jj) {
        const long long ar = lttb_area_key(ax, ay, c.x, c.y, s_x[jj - lo0], s_y[jj - lo0]);
        if (ar > best) { best = ar; r = (unsigned char)(jj - blo); }  // strict '>' (:115)
      }
    }
    tab[it] = r;
  }
}

// K3a/K3c, part 2: one CTA per series composes the transition tables by
// pointer jumping in shared memory, a segment of `jump_seg` buckets at a
// time: after level w, G_b maps the candidates of bucket (b-w) to bucket b;
// ceil(log2 seg) levels leave G_b mapping the segment's entry domain (the
// previous segment's last pick, carried) to bucket b's pick -- the chain
// out[b+1] = T_b[out[b]] of _kernels.py:108-119 without the sequential walk.
// Output: positions into a.pos (K3c, verified later) or mapped indices into
// a.out.  Candidate mode: local pick -> a.cand[b][pick], else lbound + pick.
template <int SMAX>
__global__ void __launch_bounds__(1024) k_lttb_jump(LttbArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int s_carry;
  const int64_t s = blockIdx.x;
  const int64_t k3 = a.n_out - 2;
  const int64_t m = a.m_dev ? a.m_dev[s] : a.n;
  const int64_t seg = a.jump_seg;
  unsigned char* const A0 = sm;
  unsigned char* const B0 = sm + seg * SMAX;
  const unsigned char* tab = a.tables + s * a.tab_ld;
  int64_t* out = a.out + s * a.n_out;
  int64_t* pos = a.pos ? a.pos + s * a.pos_ld : nullptr;
  const int64_t* map = a.map ? a.map + s * a.map_ld : nullptr;
  const int64_t* cand = a.cand ? a.cand + s * a.cand_ld : nullptr;
  int carry = 0;
  for (int64_t s0 = 0; s0 < k3; s0 += seg) {
    const int64_t len = min(seg, k3 - s0);
    const int64_t nent = len * SMAX;
    unsigned char* A = A0;
    unsigned char* Bf = B0;
    {
      const uint4* src = reinterpret_cast<const uint4*>(tab + s0 * SMAX);
      uint4* dst = reinterpret_cast<uint4*>(A);
      for (int64_t i = threadIdx.x; i < (nent + 15) / 16; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    for (int64_t w = 1; w < len; w <<= 1) {
      for (int64_t it = threadIdx.x; it < nent; it += blockDim.x) {
        const int64_t b = it / SMAX;
        const int p = (int)(it % SMAX);
        unsigned char v = A[it];
        if (b >= w) v = A[b * SMAX + A[(b - w) * SMAX + p]];
        Bf[it] = v;
      }
      __syncthreads();
      unsigned char* t = A; A = Bf; Bf = t;
    }
    for (int64_t bl = threadIdx.x; bl < len; bl += blockDim.x) {
      const int64_t b = s0 + bl;
      const int sel = A[bl * SMAX + carry];
      const int64_t p = cand ? cand[b * SMAX + sel] : lbound(a, m, b) + sel;
      if (pos) pos[b + 1] = p;
      else out[b + 1] = map ? map[p] : p;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_carry = A[(len - 1) * SMAX + carry];
    __syncthreads();
    carry = s_carry;
  }
  if (threadIdx.x == 0) {
    if (pos) {
      pos[0] = 0;
      pos[k3 + 1] = m - 1;
    } else {
      out[0] = map ? map[0] : 0;
      out[k3 + 1] = map ? map[m - 1] : m - 1;
    }
  }
}

// K3a, part 2 for buckets of <= 8 points: each transition table T_b is a
// packed byte map (4 or 8 bytes) and composition is one or two PRMTs, so the
// chain is resolved by a block-wide inclusive scan with the composition
// operator (warp shuffles + one smem level) instead of log2(k3) smem rounds.
// P_b = T_b o ... o T_0; P_b[0] is bucket b's pick (_kernels.py:108-119).
template <int W> struct PMap;
template <> struct PMap<4> {
  uint32_t v;
  static __device__ __forceinline__ PMap ident() { return {0x03020100u}; }
  static __device__ __forceinline__ uint32_t sel(uint32_t f) {
    return (f & 0xFu) | ((f >> 4) & 0xF0u) | ((f >> 8) & 0xF00u) | ((f >> 12) & 0xF000u);
  }
  // (g o f)[p] = g[f[p]]
  static __device__ __forceinline__ PMap comp(PMap g, PMap f) { return {__byte_perm(g.v, 0u, sel(f.v))}; }
  __device__ __forceinline__ int at0() const { return (int)(v & 0xFFu); }
  __device__ __forceinline__ PMap shfl_up(int o) const { return {__shfl_up_sync(FULL, v, o)}; }
  static __device__ __forceinline__ PMap load(const unsigned char* t) { return {*reinterpret_cast<const uint32_t*>(t)}; }
};
template <> struct PMap<8> {
  uint32_t lo, hi;
  static __device__ __forceinline__ PMap ident() { return {0x03020100u, 0x07060504u}; }
  static __device__ __forceinline__ PMap comp(PMap g, PMap f) {
    return {__byte_perm(g.lo, g.hi, PMap<4>::sel(f.lo)), __byte_perm(g.lo, g.hi, PMap<4>::sel(f.hi))};
  }
  __device__ __forceinline__ int at0() const { return (int)(lo & 0xFFu); }
  __device__ __forceinline__ PMap shfl_up(int o) const {
    return {__shfl_up_sync(FULL, lo, o), __shfl_up_sync(FULL, hi, o)};
  }
  static __device__ __forceinline__ PMap load(const unsigned char* t) {
    const uint2 u = *reinterpret_cast<const uint2*>(t);
    return {u.x, u.y};
  }
};

// W = 16 / 32: maps of W bytes; output byte p = g[f[p]] selects among W
// bytes with one PRMT per 8-byte block and a per-byte mux on f's high bits.
template <int W> struct PMapN {
  static constexpr int NW = W / 4;
  uint32_t v[NW];
  static __device__ __forceinline__ PMapN ident() {
    PMapN r;
#pragma unroll
    for (int i = 0; i < NW; ++i) r.v[i] = 0x03020100u + 0x04040404u * (uint32_t)i;
    return r;
  }
  static __device__ __forceinline__ PMapN comp(const PMapN& g, const PMapN& f) {
    PMapN r;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const uint32_t fw = f.v[i];
      const uint32_t sel = PMap<4>::sel(fw & 0x07070707u);
      uint32_t q[W / 8];
#pragma unroll
      for (int k = 0; k < W / 8; ++k) q[k] = __byte_perm(g.v[2 * k], g.v[2 * k + 1], sel);
      uint32_t acc[W / 8];
#pragma unroll
      for (int k = 0; k < W / 8; ++k) acc[k] = q[k];
      int n = W / 8, bit = 3;
#pragma unroll
      while (n > 1) {
        const uint32_t msk = ((fw >> bit) & 0x01010101u) * 0xFFu;
#pragma unroll
        for (int k = 0; k < n / 2; ++k) acc[k] = (acc[2 * k] & ~msk) | (acc[2 * k + 1] & msk);
        n >>= 1;
        ++bit;
      }
      r.v[i] = acc[0];
    }
    return r;
  }
  __device__ __forceinline__ int at0() const { return (int)(v[0] & 0xFFu); }
  __device__ __forceinline__ int at(int p) const { return (int)((v[p >> 2] >> (8 * (p & 3))) & 0xFFu); }
  __device__ __forceinline__ PMapN shfl_up(int o) const {
    PMapN r;
#pragma unroll
    for (int i = 0; i < NW; ++i) r.v[i] = __shfl_up_sync(FULL, v[i], o);
    return r;
  }
  static __device__ __forceinline__ PMapN load(const unsigned char* t) {
    PMapN r;
    const uint4* q = reinterpret_cast<const uint4*>(t);
#pragma unroll
    for (int i = 0; i < NW / 4; ++i) {
      const uint4 u = q[i];
      r.v[4 * i] = u.x; r.v[4 * i + 1] = u.y; r.v[4 * i + 2] = u.z; r.v[4 * i + 3] = u.w;
    }
    return r;
  }
};
template <> struct PMap<16> : PMapN<16> {
  PMap() = default;
  __device__ __forceinline__ PMap(const PMapN<16>& o) : PMapN<16>(o) {}
  static __device__ __forceinline__ PMap ident() { return PMapN<16>::ident(); }
  static __device__ __forceinline__ PMap comp(const PMap& g, const PMap& f) { return PMapN<16>::comp(g, f); }
  __device__ __forceinline__ PMap shfl_up(int o) const { return PMapN<16>::shfl_up(o); }
  static __device__ __forceinline__ PMap load(const unsigned char* t) { return PMapN<16>::load(t); }
};
template <> struct PMap<32> : PMapN<32> {
  PMap() = default;
  __device__ __forceinline__ PMap(const PMapN<32>& o) : PMapN<32>(o) {}
  static __device__ __forceinline__ PMap ident() { return PMapN<32>::ident(); }
  static __device__ __forceinline__ PMap comp(const PMap& g, const PMap& f) { return PMapN<32>::comp(g, f); }
  __device__ __forceinline__ PMap shfl_up(int o) const { return PMapN<32>::shfl_up(o); }
  static __device__ __forceinline__ PMap load(const unsigned char* t) { return PMapN<32>::load(t); }
};

// Resolve the LTTB chain over k3 packed transition maps (tab + b*W) with a
// block-wide inclusive scan under map composition; emit(b, sel) receives
// bucket b's local pick.  All NT threads must call.
template <int W, int NT, int ITEMS, typename Emit>
__device__ __forceinline__ void scan_chain(const unsigned char* tab, int64_t k3, Emit emit) {
  typedef PMap<W> M;
  __shared__ M s_warp[NT / 32];
  __shared__ M s_carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  M carry = M::ident();
  for (int64_t c0 = 0; c0 < k3; c0 += (int64_t)NT * ITEMS) {
    const int64_t b0 = c0 + (int64_t)threadIdx.x * ITEMS;
    M t[ITEMS];
    M agg = M::ident();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      t[i] = (b0 + i < k3) ? M::load(tab + (b0 + i) * W) : M::ident();
      agg = M::comp(t[i], agg);
    }
    // warp inclusive scan of the per-thread aggregates (earlier lanes apply first)
    M inc = agg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const M other = inc.shfl_up(o);
      if (lane >= o) inc = M::comp(inc, other);
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      M w = lane < NT / 32 ? s_warp[lane] : M::ident();
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const M other = w.shfl_up(o);
        if (lane >= o) w = M::comp(w, other);
      }
      if (lane < NT / 32) s_warp[lane] = w;
    }
    __syncthreads();
    // exclusive prefix of this thread = carry, then earlier warps, then earlier lanes
    M pre = carry;
    if (wid > 0) pre = M::comp(s_warp[wid - 1], pre);
    const M lane_prev = inc.shfl_up(1);
    if (lane > 0) pre = M::comp(lane_prev, pre);
    M cur = pre;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      cur = M::comp(t[i], cur);
      if (b0 + i < k3) emit(b0 + i, cur.at0());
    }
    if (threadIdx.x == NT - 1) s_carry = cur;
    __syncthreads();
    carry = s_carry;
    __syncthreads();
  }
}

template <int W, int NT, int ITEMS>
__global__ void __launch_bounds__(NT) k_lttb_scan(LttbArgs a) {
  const int64_t s = blockIdx.x;
  const int64_t k3 = a.n_out - 2;
  const int64_t m = a.m_dev ? a.m_dev[s] : a.n;
  // restrict: the emit's loads (cand, map) never alias its stores (pos, out), so a
  // thread's ITEMS emits can have their loads in flight together
  int64_t* __restrict__ out = a.out + s * a.n_out;
  int64_t* __restrict__ pos = a.pos ? a.pos + s * a.pos_ld : nullptr;
  const int64_t* __restrict__ map = a.map ? a.map + s * a.map_ld : nullptr;
  const int64_t* __restrict__ cand = a.cand ? a.cand + s * a.cand_ld : nullptr;
  scan_chain<W, NT, ITEMS>(a.tables + s * a.tab_ld, k3, [&](int64_t b, int sel) {
    const int64_t p = cand ? cand[b * W + sel] : lbound(a, m, b) + sel;
    if (pos) pos[b + 1] = p;
    else out[b + 1] = map ? map[p] : p;
  });
  if (threadIdx.x == 0) {
    if (pos) {
      pos[0] = 0;
      pos[k3 + 1] = m - 1;
    } else {
      out[0] = map ? map[0] : 0;
      out[k3 + 1] = map ? map[m - 1] : m - 1;
    }
  }
}

// ---------------------------------------------------------------- K3c ----
// LTTB over LARGE buckets (e.g. C2: 1998 buckets of 5005 points), bit-exact.
// area_j = |alpha*(y_j - ay) - (ax - x_j)*beta| is affine in (x_j, y_j), so
// in exact arithmetic each bucket's pick is a vertex of the bucket's convex
// hull whatever the previous pick.  The hull vertices are the candidates:
//   k_lttb_hull     one warp per bucket: per-lane monotone-chain hulls of
//                   32 contiguous segments, merged by lane 0 (a heuristic --
//                   rounding, ties and the HMAX cap can make it miss)
//   k_lttb_ctables  exact reference areas between candidate sets ->
//                   transition tables; k_lttb_jump resolves the chain
//   k_lttb_verify   every bucket re-scanned in full with the exact formula
//                   and tie rule given the previous pick -> flag mismatches
//   k_lttb_repair   one CTA walks from the first mismatch with exact full-
//                   bucket scans until the chain re-joins the candidate
//                   chain (whose later buckets were verified), then writes
//                   the output.  So the result never depends on the heuristic.
// points in flight per thread in the K3c streaming scans (candidate search,
// verification): these kernels are load-latency-bound, not issue-bound
#ifndef K3C_UN_DIR
#define K3C_UN_DIR 8
#endif
#ifndef K3C_UN_VER
#define K3C_UN_VER 8
#endif
#ifndef K3C_QUAD
#define K3C_QUAD 8  // points per min/max group in the direction-candidate scan
#endif

// Direction-sampled candidates (default K3c heuristic; cheaper than hulls).
// Over anchors a in bucket b-1's bounding box and the fixed mean c_b+1, the
// area functional is f(j) = dx*x_j + dy*y_j + const with (dx, dy) = (cy-ay,
// ax-cx) ranging over a rectangle, whose angular span is set by its corners.
// D directions sampled across that span, argmax and argmin of each (the
// maximiser of |f| is one of them) -> <= 2D candidates per bucket.  Exact
// only in the limit; k_lttb_verify / k_lttb_repair make the result exact.
template <typename XT, typename YT, int HMAX, int D, int NT = 128>
__global__ void __launch_bounds__(NT) k_lttb_dircand(LttbArgs a) {
  static_assert(2 * D <= HMAX && 2 * D <= 32, "candidates must fit");
  constexpr int NWC = NT / 32;
  __shared__ float s_v[NWC][2 * D];
  __shared__ int s_i[NWC][2 * D];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t k3 = a.n_out - 2;
  const int64_t s = blockIdx.y, b = blockIdx.x;  // one CTA per bucket
  const int64_t m = a.m_dev ? a.m_dev[s] : a.n;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  const int64_t blo = lbound(a, m, b), bhi = lbound(a, m, b + 1);
  const double2 c = a.means[s * a.means_ld + b];
  // anchor box of bucket b-1 (or the fixed first point)
  double ax0, ax1, ay0, ay1;
  if (b == 0) {
    ax0 = ax1 = to_f64(xs, 0);
    ay0 = ay1 = to_f64(ys, 0);
  } else {
    ax0 = to_f64(xs, lbound(a, m, b - 1));
    ax1 = to_f64(xs, blo - 1);
    const double2 r = a.yrange[s * k3 + b - 1];
    ay0 = r.x;
    ay1 = r.y;
  }
  float th_lo = 1e30f, th_hi = -1e30f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double dxv = c.y - ((q & 1) ? ay1 : ay0);
    const double dyv = ((q & 2) ? ax1 : ax0) - c.x;
    float th = atan2f((float)dyv, (float)dxv);
    if (th > 3.0f) th -= 6.2831853f;  // keep the (x <= c.x) half-plane contiguous
    th_lo = fminf(th_lo, th);
    th_hi = fmaxf(th_hi, th);
  }
  float cs[D], sn[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float th = D > 1 ? th_lo + (th_hi - th_lo) * (float)k / (float)(D - 1) : th_lo;
    sincosf(th, &sn[k], &cs[k]);
  }
  const XT xr = xs[blo];
  const double yr = c.y;
  float vmax[D], vmin[D];
  int imax[D], imin[D];
#pragma unroll
  for (int k = 0; k < D; ++k) { vmax[k] = -INFINITY; vmin[k] = INFINITY; imax[k] = INT_MAX; imin[k] = INT_MAX; }
  // affine-x bucket: X = x_j - x_lo from the index alone (y is the only stream).
  // Conversions avoid the XU pipe (float counter, d2f_trunc): a heuristic, any
  // consistent X, Y works (verify/repair make the result exact)
  const bool aff = a.xaff && a.xaff[s * k3 + b].ok;
  const float fxf = aff ? (float)(XForm<XT>::integral ? (double)a.xaff[s * k3 + b].di : a.xaff[s * k3 + b].d) : 0.f;
  const double xrd = elem_f64(xr);
  const float yrf = (float)yr;
  constexpr int UN = K3C_UN_DIR;
  float of = (float)threadIdx.x;  // running offset from blo (exact below 2^24)
  // Points go in quads (u = 4g..4g+3, offsets o, o+NT, o+2NT, o+3NT): per direction the quad's
  // max / min come from 3 + 3 min/max instructions and only they are compared against the
  // running extremes, which record the quad's first offset; the winning quads are resolved
  // to their element after the CTA reduction.  (5 instead of 8 ALU/FMA ops per point and direction)
  static_assert(UN % K3C_QUAD == 0, "groups");
  constexpr int QG = K3C_QUAD;  // points per group (4: quads, 8: octets)
  for (int64_t j0 = blo + threadIdx.x; j0 < bhi; j0 += NT * UN, of += (float)(NT * UN)) {
    XT rx[UN];
    YT ry[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {  // UN points' loads in flight before any use
      const int64_t j = j0 + NT * u < bhi ? j0 + NT * u : j0;  // out of range: repeat the group's first point
      if (!aff) rx[u] = xs[j];
      ry[u] = ys[j];
    }
#pragma unroll
    for (int g = 0; g < UN / QG; ++g) {
      if (j0 + NT * QG * g < bhi) {
        float X[QG], Y[QG];
#pragma unroll
        for (int t = 0; t < QG; ++t) {
          const int u = QG * g + t;
          const bool in = j0 + NT * u < bhi;
          X[t] = aff ? (in ? of + (float)(NT * u) : of + (float)(NT * QG * g)) * fxf
                     : d2f_trunc(__dsub_rn(elem_f64(rx[u]), xrd));
          if constexpr (sizeof(YT) == 4) Y[t] = __fsub_rn((float)ry[u], yrf);
          else Y[t] = d2f_trunc(__dsub_rn((double)ry[u], yr));
        }
        const int o = (int)(j0 + NT * QG * g - blo);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          float mx = -INFINITY, mn = INFINITY;
#pragma unroll
          for (int t = 0; t < QG; ++t) {
            const float v = fmaf(cs[k], X[t], sn[k] * Y[t]);
            mx = fmaxf(mx, v);
            mn = fminf(mn, v);
          }
          if (mx > vmax[k]) { vmax[k] = mx; imax[k] = o; }
          if (mn < vmin[k]) { vmin[k] = mn; imin[k] = o; }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const float ov = __shfl_xor_sync(FULL, vmax[k], off);
      const int oi = __shfl_xor_sync(FULL, imax[k], off);
      if (ov > vmax[k] || (ov == vmax[k] && oi < imax[k])) { vmax[k] = ov; imax[k] = oi; }
      const float ow = __shfl_xor_sync(FULL, vmin[k], off);
      const int oj = __shfl_xor_sync(FULL, imin[k], off);
      if (ow < vmin[k] || (ow == vmin[k] && oj < imin[k])) { vmin[k] = ow; imin[k] = oj; }
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      s_v[wid][2 * k] = vmax[k]; s_i[wid][2 * k] = imax[k];
      s_v[wid][2 * k + 1] = -vmin[k]; s_i[wid][2 * k + 1] = imin[k];  // both as "max"
    }
  }
  __syncthreads();
  if (wid != 0) return;
  int ci = INT_MAX;
  if (lane < 2 * D) {
    float bv = s_v[0][lane];
    ci = s_i[0][lane];
#pragma unroll
    for (int w = 1; w < NWC; ++w) {
      const float v = s_v[w][lane];
      const int i = s_i[w][lane];
      if (v > bv || (v == bv && i < ci)) { bv = v; ci = i; }
    }
  }
  // resolve each winning quad to its element: recompute the direction's values of the
  // quad's points exactly as in the scan and take the first extreme one
  if (lane < 2 * D && ci != INT_MAX) {
    const int k = lane >> 1;
    const float th = D > 1 ? th_lo + (th_hi - th_lo) * (float)k / (float)(D - 1) : th_lo;
    float snk, csk;
    sincosf(th, &snk, &csk);
    float bestv = -INFINITY;
    int bi = ci;
#pragma unroll
    for (int t = 0; t < K3C_QUAD; ++t) {
      const int o = ci + NT * t;
      if (blo + o < bhi) {
        const float X = aff ? (float)o * fxf : d2f_trunc(__dsub_rn(elem_f64(xs[blo + o]), xrd));
        float Y;
        if constexpr (sizeof(YT) == 4) Y = __fsub_rn((float)ys[blo + o], yrf);
        else Y = d2f_trunc(__dsub_rn((double)ys[blo + o], yr));
        const float v = fmaf(csk, X, snk * Y);
        const float w = (lane & 1) ? -v : v;
        if (w > bestv) { bestv = w; bi = o; }
      }
    }
    ci = bi;
  }
  // sort the <= 32 candidate offsets across the warp (bitonic), then dedup
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int o = __shfl_xor_sync(FULL, ci, j);
      const bool up = ((lane & k) == 0);
      const bool lower = (lane & j) == 0;
      ci = (lower == up) ? min(ci, o) : max(ci, o);
    }
  }
  const int prev = __shfl_up_sync(FULL, ci, 1);
  const bool keep = ci != INT_MAX && (lane == 0 || prev != ci);
  const unsigned km = __ballot_sync(FULL, keep);
  const int rank = __popc(km & ((1u << lane) - 1));
  const int cap = a.cand_cap > 0 && a.cand_cap < HMAX ? a.cand_cap : HMAX;
  int64_t* cand = a.cand + s * a.cand_ld + b * HMAX;
  if (keep && rank < cap) cand[rank] = blo + ci;
  if (lane == 0) {
    const int w = min(__popc(km), cap);
    if (w == 0) cand[0] = blo;
    a.cand_cnt[s * k3 + b] = w ? w : 1;
  }
}

// T_b[p] over candidates: exact reference area (lttb_area), strict '>' in
// ascending index order = lowest index on ties, NaN never wins.
template <typename XT, typename YT, int HMAX>
__global__ void __launch_bounds__(1024) k_lttb_ctables(LttbArgs a) {
  constexpr int NBK = 1024 / HMAX;
  // every thread stages one candidate point of the CTA's buckets (and of the
  // bucket before them, the anchors) in shared memory first: two memory round
  // trips in all instead of a dependent cand -> (x, y) chain per candidate
  __shared__ double2 s_pt[NBK + 1][HMAX];
  __shared__ int s_cnt[NBK + 1];
  const int64_t s = blockIdx.y;
  const int64_t k3 = a.n_out - 2;
  const int bi = threadIdx.x / HMAX, p = threadIdx.x % HMAX;
  const int64_t bb = (int64_t)blockIdx.x * NBK;  // first bucket of the CTA
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  const int64_t* cand = a.cand + s * a.cand_ld;
  const int* cnt = a.cand_cnt + s * k3;
  for (int t = threadIdx.x; t < (NBK + 1) * HMAX; t += 1024) {  // row r = bucket bb - 1 + r
    const int r = t / HMAX, q = t % HMAX;
    const int64_t b = bb - 1 + r;
    if (b >= 0 && b < k3) {
      const int nc = cnt[b];
      if (q == 0) s_cnt[r] = nc;
      if (q < nc) {
        const int64_t jj = cand[b * HMAX + q];
        s_pt[r][q] = make_double2(to_f64(xs, jj), to_f64(ys, jj));
      }
    } else if (q == 0) {
      s_cnt[r] = 0;
    }
  }
  __syncthreads();
  const int64_t b = bb + bi;
  if (b >= k3) return;
  bool valid;
  double ax, ay;
  if (b == 0) { valid = p == 0; ax = to_f64(xs, 0); ay = to_f64(ys, 0); }
  else { valid = p < s_cnt[bi]; ax = valid ? s_pt[bi][p].x : 0.0; ay = valid ? s_pt[bi][p].y : 0.0; }
  unsigned char r = 0;
  if (valid) {
    const double2 c = a.means[s * a.means_ld + b];
    const int nc = s_cnt[bi + 1];
    long long bestv = -1;
    for (int q = 0; q < nc; ++q) {
      const double2 pt = s_pt[bi + 1][q];
      const long long ar = lttb_area_key(ax, ay, c.x, c.y, pt.x, pt.y);
      if (ar > bestv) { bestv = ar; r = (unsigned char)q; }
    }
  }
  a.tables[s * a.tab_ld + b * HMAX + p] = r;
}

// block argmax of the exact area over [lo, hi) given anchor (ax, ay) and mean c
template <typename XT, typename YT, int NT>
__device__ __forceinline__ int64_t block_bucket_argmax(const XT* xs, const YT* ys, int64_t lo, int64_t hi, double ax,
                                                       double ay, double2 c, double* s_a, long long* s_i,
                                                       const XAff* xa = nullptr) {
  // argmax on integer keys of |area| (NaN -> -1, never wins): no fp64
  // compares, which issue on B200's narrow XU pipe
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long bk = -1;
  long long bi = LLONG_MAX;
  constexpr int UN = K3C_UN_VER;
  const bool aff = xa && xa->ok;
  XAff f;
  if (aff) f = *xa;
  const double P = __dsub_rn(ax, c.x), S = __dsub_rn(c.y, ay);
  for (int64_t j0 = lo + threadIdx.x; j0 < hi; j0 += (int64_t)NT * UN) {
    XT rx[UN];
    YT ry[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {  // loads in flight before the area math
      const int64_t j = j0 + (int64_t)NT * u < hi ? j0 + (int64_t)NT * u : lo;
      if (!aff) rx[u] = xs[j];
      ry[u] = ys[j];
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int64_t j = j0 + (int64_t)NT * u;
      if (j < hi) {
        const double xj = aff ? XForm<XT>::at(f, j - lo) : elem_f64(rx[u]);
        // lttb_area: abs((ax - cx) * (y_j - ay) - (ax - x_j) * (cy - ay)), same op order
        const double t = __dsub_rn(__dmul_rn(P, __dsub_rn(elem_f64(ry[u]), ay)), __dmul_rn(__dsub_rn(ax, xj), S));
        long long k = __double_as_longlong(t) & 0x7fffffffffffffffLL;
        k = k > 0x7ff0000000000000LL ? -1LL : k;
        if (k > bk) { bk = k; bi = j; }
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const long long ok = __shfl_xor_sync(FULL, bk, o);
    const long long oi = __shfl_xor_sync(FULL, bi, o);
    if (ok > bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
  }
  if (lane == 0) { s_a[wid] = __longlong_as_double(bk); s_i[wid] = bi; }
  __syncthreads();
  if (wid == 0) {
    bk = lane < NT / 32 ? __double_as_longlong(s_a[lane]) : -1LL;
    bi = lane < NT / 32 ? s_i[lane] : LLONG_MAX;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const long long ok = __shfl_xor_sync(FULL, bk, o);
      const long long oi = __shfl_xor_sync(FULL, bi, o);
      if (ok > bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
    }
    if (lane == 0) s_i[0] = bi == LLONG_MAX ? lo : bi;  // all-NaN bucket keeps bounds[b] (:110)
  }
  __syncthreads();
  const int64_t r = s_i[0];
  __syncthreads();
  return r;
}

// ---- K3c certified means -------------------------------------------------
// The reference's bucket means are in-order fp64 sums (_kernels.py:98-104): a
// dependent chain of ~5,000 DADDs per bucket.  Instead, K3c takes any-order
// (parallel) sums plus a rigorous bound on their distance to the in-order
// result, and every exact argmax (verify / verify2 / repair) CERTIFIES its
// pick against that bound: the runner-up area must trail the winner by more
// than twice the worst-case area error the mean error can cause.  A bucket
// that fails (near-tie, non-finite area) gets its in-order mean computed
// exactly on the spot and is re-scanned, so the output is the reference's
// whatever the data.  A mean is EXACT (bound 0, no certification needed)
// when every partial sum in any order is representable: all values are
// multiples of 2^L (L = lowest set bit over the bucket) and sum|v| < 2^(53+L)
// -- integer x (arange) and float32-origin y usually are.
constexpr double K3C_U = 1.1102230246251565e-16;  // unit roundoff 2^-53

// exponent of the lowest set bit of |v| (zero: +large, it constrains nothing);
// subnormals come out one low, which only makes the exactness test stricter
__device__ __forceinline__ int lsb_exp(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const int e = (int)((b >> 52) & 0x7ff);
  const long long mnt = (long long)((b & 0xfffffffffffffull) | (1ull << 52));
  return v == 0.0 ? 4096 : e - 1075 + (__ffsll(mnt) - 1);
}

// |in-order fp64 mean - fl(S/n)| bound for a bucket of n values with any-order
// sum S, any-order sum of magnitudes A and lowest-bit exponent L; 0 = exact.
__device__ __forceinline__ double mean_err_bound(double S, double A, int L, double n) {
  const double lim = L + 53 > 1100 ? INFINITY : ldexp(1.0, L + 53);
  if (A < lim) return 0.0;  // every partial sum representable: both sums exact
  const double g = n * K3C_U / (1.0 - n * K3C_U);  // gamma_n: |sum_fl - sum| <= gamma_n * sum|v|, any order
  const double c = S / n;
  // |ref - S| <= 2 gamma A; the two divisions add u|c| + u|c'|
  return (2.0 * g * A / n * (1.0 + 4.0 * g) + 2.0 * K3C_U * fabs(c)) * (1.0 + 1e-12) + 1e-300;
}

// Per-bucket stats in one coalesced pass, one CTA per bucket q: (ymin, ymax)
// of bucket q (direction candidates) and, for q >= 1, the approximate mean of
// bucket q with its error bound -> means[q-1], merr[q-1] (the mean bucket q-1
// anchors on).  Bandwidth-bound: no dependent add chain.
template <typename XT, typename YT, int NT, int UN>
__global__ void __launch_bounds__(NT) k_lttb_means_approx(LttbArgs a) {
  constexpr int NW = NT / 32;
  __shared__ double s_d[6][NW];
  __shared__ int s_l[2][NW];
  const int64_t s = blockIdx.y, q = blockIdx.x;
  const int64_t k3 = a.n_out - 2;
  const int64_t m = a.m_dev ? a.m_dev[s] : a.n;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  const int64_t lo = lbound(a, m, q), hi = lbound(a, m, q + 1);
  double sx = 0.0, sy = 0.0, ax = 0.0, ay = 0.0, ymn = INFINITY, ymx = -INFINITY;
  int lx = XForm<XT>::integral ? 0 : 4096, ly = 4096;
  // affine-x candidate from the bucket's first two points (XAff)
  XAff f;
  {
    const XT x0r = xs[lo], x1r = hi - lo > 1 ? xs[lo + 1] : xs[lo];
    f.x0 = (double)x0r;
    f.d = __dsub_rn((double)x1r, (double)x0r);
    f.x0i = (long long)x0r;
    f.di = (long long)((unsigned long long)(long long)x1r - (unsigned long long)(long long)x0r);
  }
  bool aff = true;
  for (int64_t j0 = lo + threadIdx.x; j0 < hi; j0 += (int64_t)NT * UN) {
    XT rx[UN];
    YT ry[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {  // all loads in flight before any use
      const int64_t j = j0 + (int64_t)NT * u < hi ? j0 + (int64_t)NT * u : lo;
      rx[u] = __ldcs(xs + j);  // x streams (evict-first): y stays L2-resident for the later passes
      ry[u] = ys[j];
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      if (j0 + (int64_t)NT * u < hi) {
        const double vx = (double)rx[u], vy = (double)ry[u];
        sx += vx;
        sy += vy;
        ax += fabs(vx);
        ay += fabs(vy);
        ymn = fmin(ymn, vy);
        ymx = fmax(ymx, vy);
        if constexpr (!XForm<XT>::integral) lx = min(lx, lsb_exp(vx));  // integers: lsb >= 2^0
        ly = min(ly, lsb_exp(vy));
        const int64_t t = j0 + (int64_t)NT * u - lo;
        if constexpr (XForm<XT>::integral) aff &= (long long)rx[u] == (long long)((unsigned long long)f.x0i + (unsigned long long)t * (unsigned long long)f.di);
        else aff &= __double_as_longlong(vx) == __double_as_longlong(XForm<XT>::at(f, t));
      }
    }
  }
  aff = __syncthreads_and(aff);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sx += __shfl_xor_sync(FULL, sx, o);
    sy += __shfl_xor_sync(FULL, sy, o);
    ax += __shfl_xor_sync(FULL, ax, o);
    ay += __shfl_xor_sync(FULL, ay, o);
    ymn = fmin(ymn, __shfl_xor_sync(FULL, ymn, o));
    ymx = fmax(ymx, __shfl_xor_sync(FULL, ymx, o));
    lx = min(lx, __shfl_xor_sync(FULL, lx, o));
    ly = min(ly, __shfl_xor_sync(FULL, ly, o));
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (NW > 1) {
    if (lane == 0) {
      s_d[0][wid] = sx; s_d[1][wid] = sy; s_d[2][wid] = ax; s_d[3][wid] = ay; s_d[4][wid] = ymn; s_d[5][wid] = ymx;
      s_l[0][wid] = lx; s_l[1][wid] = ly;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int w = 1; w < NW; ++w) {
      sx += s_d[0][w]; sy += s_d[1][w]; ax += s_d[2][w]; ay += s_d[3][w];
      ymn = fmin(ymn, s_d[4][w]); ymx = fmax(ymx, s_d[5][w]);
      lx = min(lx, s_l[0][w]); ly = min(ly, s_l[1][w]);
    }
  } else if (lane != 0) {
    return;
  }
  a.yrange[s * k3 + q] = make_double2(ymn, ymx);
  if (a.xaff) {
    f.ok = aff;
    f.pad = 0;
    a.xaff[s * k3 + q] = f;
  }
  if (q >= 1) {
    const double n = (double)(hi - lo);
    a.means[s * a.means_ld + q - 1] = make_double2(__ddiv_rn(sx, n), __ddiv_rn(sy, n));
    a.merr[s * k3 + q - 1] = make_double2(mean_err_bound(sx, ax, lx, n), mean_err_bound(sy, ay, ly, n));
  }
  if (q == 0) {  // the last bucket anchors on point m-1 itself (_kernels.py:105-107): exact
    a.means[s * a.means_ld + k3 - 1] = make_double2(to_f64(xs, m - 1), to_f64(ys, m - 1));
    a.merr[s * k3 + k3 - 1] = make_double2(0.0, 0.0);
  }
}

// In-order (reference) mean of bucket b+1, by a whole CTA: tiles staged in
// shared memory, threads 0/1 carry the x/y add chains.  The rare path of a
// failed certification.
template <typename XT, typename YT, int NT>
__device__ double2 block_exact_mean(const LttbArgs& a, const XT* xs, const YT* ys, int64_t m, int64_t b) {
  constexpr int TILE = 512;
  __shared__ double s_t[2][TILE];
  __shared__ double s_c[2];
  const int64_t k3 = a.n_out - 2;
  if (b + 1 >= k3) return make_double2(to_f64(xs, m - 1), to_f64(ys, m - 1));
  const int64_t nlo = lbound(a, m, b + 1), nhi = lbound(a, m, b + 2);
  double acc = 0.0;
  for (int64_t t0 = nlo; t0 < nhi; t0 += TILE) {
    __syncthreads();
    for (int i = threadIdx.x; i < TILE; i += NT) {
      const int64_t j = t0 + i;
      if (j < nhi) { s_t[0][i] = to_f64(xs, j); s_t[1][i] = to_f64(ys, j); }
    }
    __syncthreads();
    if (threadIdx.x < 2) {
      const int n = (int)(nhi - t0 < TILE ? nhi - t0 : (int64_t)TILE);
      const double* src = s_t[threadIdx.x];
      for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, src[i]);  // sx += xs[j] in index order
    }
  }
  const double cnt = (double)(nhi - nlo);
  if (threadIdx.x < 2) s_c[threadIdx.x] = __ddiv_rn(acc, cnt);
  __syncthreads();
  const double2 c = make_double2(s_c[0], s_c[1]);
  __syncthreads();
  return c;
}

// Exact argmax of bucket b given anchor `prev` when means[b] is approximate:
// scan with the approximate mean tracking the winner, the runner-up and the
// magnitudes that bound the area error; certify, else compute the exact mean
// (stored back: merr[b] = 0) and re-scan.
template <typename XT, typename YT, int NT>
__device__ int64_t block_bucket_argmax_cert(const LttbArgs& a, int64_t s, int64_t m, const XT* xs, const YT* ys,
                                            int64_t b, int64_t prev, double* s_a, long long* s_i, bool store = true) {
  const int64_t k3 = a.n_out - 2;
  const int64_t lo = lbound(a, m, b), hi = lbound(a, m, b + 1);
  const double ax = to_f64(xs, prev), ay = to_f64(ys, prev);
  double2* mp = a.means + s * a.means_ld + b;
  double2* ep = a.merr + s * k3 + b;
  const double2 c = *mp;
  const double2 ce = *ep;
  const XAff* xa = a.xaff ? a.xaff + s * k3 + b : nullptr;
  if (ce.x == 0.0 && ce.y == 0.0)  // exact mean: the plain scan IS the reference's
    return block_bucket_argmax<XT, YT, NT>(xs, ys, lo, hi, ax, ay, c, s_a, s_i, xa);
  __shared__ double s_v2[NT / 32], s_q[NT / 32], s_r[NT / 32];
  __shared__ int s_bad[NT / 32];
  __shared__ int s_ok;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double P = __dsub_rn(ax, c.x), S = __dsub_rn(c.y, ay);
  // keys (bit patterns of non-negative doubles order like the values): no fp64 compares
  long long k1 = -1, k2 = -1, kq = 0, kr = 0;
  long long i1 = LLONG_MAX;
  int bad = 0;
  constexpr int UN = K3C_UN_VER;
  const bool aff = xa && xa->ok;
  XAff f;
  if (aff) f = *xa;
  for (int64_t j0 = lo + threadIdx.x; j0 < hi; j0 += (int64_t)NT * UN) {
    XT rx[UN];
    YT ry[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int64_t j = j0 + (int64_t)NT * u < hi ? j0 + (int64_t)NT * u : lo;
      if (!aff) rx[u] = xs[j];
      ry[u] = ys[j];
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int64_t j = j0 + (int64_t)NT * u;
      if (j < hi) {
        const double xj = aff ? XForm<XT>::at(f, j - lo) : elem_f64(rx[u]);
        const double R = __dsub_rn(ax, xj), Q = __dsub_rn(elem_f64(ry[u]), ay);
        const double t = __dsub_rn(__dmul_rn(P, Q), __dmul_rn(R, S));  // lttb_area, same op order
        long long k = __double_as_longlong(t) & 0x7fffffffffffffffLL;
        bad |= (int)(k >> 32) >= 0x7ff00000;  // inf or NaN: no certification
        k = k > 0x7ff0000000000000LL ? -1LL : k;
        kq = max(kq, __double_as_longlong(Q) & 0x7fffffffffffffffLL);
        kr = max(kr, __double_as_longlong(R) & 0x7fffffffffffffffLL);
        if (k > k2) {
          if (k > k1) { k2 = k1; k1 = k; i1 = j; }
          else k2 = k;
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    vpart_merge(k1, i1, k2, bad, __shfl_xor_sync(FULL, k1, o), __shfl_xor_sync(FULL, i1, o),
                __shfl_xor_sync(FULL, k2, o), __shfl_xor_sync(FULL, bad, o));
    kq = max(kq, __shfl_xor_sync(FULL, kq, o));
    kr = max(kr, __shfl_xor_sync(FULL, kr, o));
  }
  if (lane == 0) {
    s_a[wid] = __longlong_as_double(k1); s_i[wid] = i1; s_v2[wid] = __longlong_as_double(k2);
    s_q[wid] = __longlong_as_double(kq); s_r[wid] = __longlong_as_double(kr); s_bad[wid] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NT / 32; ++w) {
      vpart_merge(k1, i1, k2, bad, __double_as_longlong(s_a[w]), s_i[w], __double_as_longlong(s_v2[w]), s_bad[w]);
      kq = max(kq, __double_as_longlong(s_q[w]));
      kr = max(kr, __double_as_longlong(s_r[w]));
    }
    const double v1 = k1 < 0 ? -1.0 : __longlong_as_double(k1), v2 = k2 < 0 ? -1.0 : __longlong_as_double(k2);
    const double qm = __longlong_as_double(kq), rm = __longlong_as_double(kr);
    // area error bound over the bucket (certified means):
    // |P-P'| <= dP, |S-S'| <= dS; |T1-T1'| <= qm (dP + u(2|P'| + dP)), same for T2;
    // |A-A'| <= (dT1 + dT2)(1+u) + 2u max A'
    const double u = K3C_U;
    const double dP = ce.x == 0.0 ? 0.0 : ce.x + u * (2.0 * fabs(P) * (1.0 + 2.0 * u) + ce.x);
    const double dS = ce.y == 0.0 ? 0.0 : ce.y + u * (2.0 * fabs(S) * (1.0 + 2.0 * u) + ce.y);
    const double dT = (dP == 0.0 ? 0.0 : qm * (dP + u * (2.0 * fabs(P) + dP))) +
                      (dS == 0.0 ? 0.0 : rm * (dS + u * (2.0 * fabs(S) + dS)));
    const double E = (dT * (1.0 + 2.0 * u) + 2.0 * u * fmax(v1, 0.0) * (1.0 + 2.0 * u)) * (1.0 + 1e-9) + 1e-300;
    const bool ok = hi - lo == 1 || (!bad && !a.cert_force && __dsub_rn(v1, v2) > 2.0 * E * (1.0 + 1e-9));
    s_ok = ok;
    s_i[0] = i1 == LLONG_MAX ? lo : i1;
  }
  __syncthreads();
  const int ok = s_ok;
  const int64_t r = s_i[0];
  __syncthreads();
  if (ok) return r;
  // failed: the reference's own in-order mean, kept for later scans of bucket b
#ifdef MM_REPAIR_TRACE
  if (threadIdx.x == 0) printf("exact-mean fallback: bucket %lld\n", (long long)b);
#endif
  const double2 ce2 = block_exact_mean<XT, YT, NT>(a, xs, ys, m, b);
  // store=false: other CTAs of a persistent kernel may be reading means/merr[b]
  if (threadIdx.x == 0 && store) { *mp = ce2; *ep = make_double2(0.0, 0.0); }
  return block_bucket_argmax<XT, YT, NT>(xs, ys, lo, hi, ax, ay, ce2, s_a, s_i, xa);
}

template <typename XT, typename YT, int NT>
__device__ __forceinline__ int64_t k3c_argmax(const LttbArgs& a, int64_t s, int64_t m, const XT* xs, const YT* ys,
                                              int64_t b, int64_t prev, double* s_a, long long* s_i) {
  if (a.merr) return block_bucket_argmax_cert<XT, YT, NT>(a, s, m, xs, ys, b, prev, s_a, s_i);
  return block_bucket_argmax<XT, YT, NT>(xs, ys, lbound(a, m, b), lbound(a, m, b + 1), to_f64(xs, prev),
                                         to_f64(ys, prev), a.means[s * a.means_ld + b], s_a, s_i);
}

// ---- K3c flat passes --------------------------------------------------------
// The per-bucket passes above give each bucket one CTA; with ~2,000 buckets of
// ~5,000 points that is 1-2 waves of CTAs each walking its bucket in ~10
// dependent load rounds, so the GPU idles on latency.  The flat passes split
// the series' elements [1, m-1) into equal contiguous ranges, one per warp
// (a single wave), each warp walking the 1-2 bucket segments its range
// intersects; per-(bucket, warp) partials are combined by the bucket's
// last-arriving warp (threadfence reduction), which finalises the bucket.
#ifndef K3C_FLAT_MINB
#define K3C_FLAT_MINB 3  // 3 x 256 threads per SM = 24 warps (host: flat_plan); candidates 2 x 256
#endif
struct FlatArgs {
  int64_t E;                 // elements per warp
  int64_t W;                 // warps per series
  int64_t CP;                // partial slots per bucket (>= warps touching one bucket)
  unsigned* cnt;             // [B][k3] arrival counters (zeroed per call)
  void* part;                // [B][k3][CP] partials
  int* ulist; int* ucount;   // verify: [B][k3] buckets whose certification failed, [B] count (zeroed)
};

// largest b with lbound(b) = 1 + floor(b (m-2) / k3) <= j, for j in [1, m-1)
__device__ __forceinline__ int64_t lttb_bucket_of(int64_t j, int64_t m, int64_t k3) { return (j * k3 - 1) / (m - 2); }

// lane 0: publish this warp's partial, return true if it was the bucket's last
__device__ __forceinline__ bool flat_arrive(unsigned* c, unsigned n) {
  __threadfence();
  const unsigned old = atomicAdd(c, 1u);
  if (old + 1 != n) return false;
  __threadfence();
  return true;
}

// |T_j - T'_j| bound for every j of a bucket (see block_bucket_argmax_cert):
// from the mean error ce and the bucket's |y - ay| / |ax - x| extremes
__device__ __forceinline__ double k3c_area_err(double2 ce, double P, double S, double qmax, double rmax, double v1) {
  const double u = K3C_U;
  const double dP = ce.x == 0.0 ? 0.0 : ce.x + u * (2.0 * fabs(P) * (1.0 + 2.0 * u) + ce.x);
  const double dS = ce.y == 0.0 ? 0.0 : ce.y + u * (2.0 * fabs(S) * (1.0 + 2.0 * u) + ce.y);
  const double dT = (dP == 0.0 ? 0.0 : qmax * (dP + u * (2.0 * fabs(P) + dP))) +
                    (dS == 0.0 ? 0.0 : rmax * (dS + u * (2.0 * fabs(S) + dS)));
  return (dT * (1.0 + 2.0 * u) + 2.0 * u * fmax(v1, 0.0) * (1.0 + 2.0 * u)) * (1.0 + 1e-9) + 1e-300;
}

// One warp's pass over a verification segment [0, n) (offsets from the
// segment start): keys of |T_j| (T_j exactly as lttb_area), top-2 and the
// first index of the top key.  MODE 0: affine integer x from a running f64
// (exact: integers < 2^50); 1: affine x by formula; 2: x loaded.
template <int MODE, typename XT, typename YT, int UN>
__device__ __forceinline__ void verify_scan(const XT* __restrict__ xb, const YT* __restrict__ yb, int n, int lane,
                                            double ax, double ay, double P, double S, double x0d, double dx1,
                                            double dstep, const XAff& f, int64_t t0, long long& k1, long long& k2,
                                            int& i1, int& bad) {
  double xl = MODE == 0 ? __dadd_rn(x0d, __dmul_rn((double)lane, dx1)) : 0.0;  // exact: integer-valued
  for (int i = lane; i < n; i += 32 * UN) {
    XT rx[UN];
    YT ry[UN];
    const bool full = i + 32 * (UN - 1) < n;
    if (full) {  // constant offsets from one pointer: no per-load address arithmetic
      const XT* xp = xb + i;
      const YT* yp = yb + i;
#pragma unroll
      for (int q = 0; q < UN; ++q) {
        if (MODE == 2) rx[q] = xp[32 * q];
        ry[q] = yp[32 * q];
      }
    } else {
#pragma unroll
      for (int q = 0; q < UN; ++q) {
        const int ii = i + 32 * q < n ? i + 32 * q : i;
        if (MODE == 2) rx[q] = xb[ii];
        ry[q] = yb[ii];
      }
    }
#pragma unroll
    for (int q = 0; q < UN; ++q) {
      double xj;
      if (MODE == 0) xj = xl;
      else if (MODE == 1) xj = XForm<XT>::at(f, t0 + i + 32 * q);
      else xj = elem_f64(rx[q]);
      if (MODE == 0) xl = __dadd_rn(xl, dstep);
      if (full || i + 32 * q < n) {
        const double R = __dsub_rn(ax, xj), Q = __dsub_rn(elem_f64(ry[q]), ay);
        const double t = __dsub_rn(__dmul_rn(P, Q), __dmul_rn(R, S));  // lttb_area, same op order
        const long long k = __double_as_longlong(t) & 0x7fffffffffffffffLL;
        bad |= (int)(k >> 32) >= 0x7ff00000;  // inf / NaN: the bucket takes the exact fallback
        if (k > k2) {  // rare after the first few points
          if (k > k1) { k2 = k1; k1 = k; i1 = i + 32 * q; }
          else k2 = k;
        }
      }
    }
  }
}

// Flat verification: every bucket's exact argmax given the candidate chain's
// previous pick, certified against merr (see block_bucket_argmax_cert); a
// bucket that fails certification goes on ulist for k_lttb_verify_fix.
template <typename XT, typename YT, int UN>
__global__ void __launch_bounds__(256, K3C_FLAT_MINB) k_lttb_verify_flat(LttbArgs a, FlatArgs fl) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t s = blockIdx.y;
  const int64_t k3 = a.n_out - 2, m = a.n;
  const int64_t e0 = 1 + gw * fl.E, e1 = min(m - 1, e0 + fl.E);
  if (gw >= fl.W || e0 >= e1) return;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  const int64_t* pos = a.pos + s * a.pos_ld;
  VPart* part = (VPart*)fl.part + s * k3 * fl.CP;
  const double u = K3C_U;
  int64_t b = lttb_bucket_of(e0, m, k3);
  for (int64_t j = e0; j < e1; ++b) {
    const int64_t lo = lbound(a, m, b), hi = lbound(a, m, b + 1);
    const int64_t s1 = min(e1, hi);
    const int n = (int)(s1 - j);  // segment [j, s1), 32-bit offsets
    const int64_t prev = pos[b];
    const double2 c = a.means[s * a.means_ld + b];
    const double2 ce = a.merr ? a.merr[s * k3 + b] : make_double2(0.0, 0.0);
    const double2 yr = a.yrange[s * k3 + b], xr = a.xrange[s * k3 + b];
    const bool aff = a.xaff && a.xaff[s * k3 + b].ok;
    XAff f;
    if (aff) f = a.xaff[s * k3 + b];
    // affine integer x inside the magic range: x_j = i2d_magic(x0 + t d) and
    // consecutive lanes' x step by exact f64 adds (every value an integer < 2^51)
    const bool afi = aff && XForm<XT>::integral && fmax(fabs(xr.x), fabs(xr.y)) < 1125899906842624.0;
    const double dstep = afi ? i2d_magic(32 * f.di) : 0.0;
    const double ax = to_f64(xs, prev), ay = to_f64(ys, prev);
    const double P = __dsub_rn(ax, c.x), S = __dsub_rn(c.y, ay);
    long long k1 = -1, k2 = -1;
    int i1 = INT_MAX, bad = 0;
    const int64_t t0 = j - lo;
    if (afi) {
      const double x0d = i2d_magic((long long)((unsigned long long)f.x0i + (unsigned long long)t0 * (unsigned long long)f.di));
      const double dx1 = i2d_magic(f.di);
      verify_scan<0, XT, YT, UN>(xs + j, ys + j, n, lane, ax, ay, P, S, x0d, dx1, dstep, f, t0, k1, k2, i1, bad);
    } else if (aff) {
      verify_scan<1, XT, YT, UN>(xs + j, ys + j, n, lane, ax, ay, P, S, 0.0, 0.0, 0.0, f, t0, k1, k2, i1, bad);
    } else {
      verify_scan<2, XT, YT, UN>(xs + j, ys + j, n, lane, ax, ay, P, S, 0.0, 0.0, 0.0, f, t0, k1, k2, i1, bad);
    }
    long long i1g = i1 == INT_MAX ? LLONG_MAX : j + i1;
#pragma unroll
    for (int o = 16; o; o >>= 1)
      vpart_merge(k1, i1g, k2, bad, __shfl_xor_sync(FULL, k1, o), __shfl_xor_sync(FULL, i1g, o),
                  __shfl_xor_sync(FULL, k2, o), __shfl_xor_sync(FULL, bad, o));
    const int64_t w0 = (lo - 1) / fl.E;
    const unsigned ns = (unsigned)((hi - 2) / fl.E - w0 + 1);
    bool last = false;
    if (lane == 0) {
      VPart p;
      p.k1 = k1; p.k2 = k2; p.i1 = i1g; p.bad = bad; p.pad = 0;
      part[b * fl.CP + (gw - w0)] = p;
      last = flat_arrive(fl.cnt + s * k3 + b, ns);
    }
    if (__shfl_sync(FULL, (int)last, 0)) {
      k1 = -1; k2 = -1; i1g = LLONG_MAX; bad = 0;
      for (unsigned q = lane; q < ns; q += 32) {
        const VPart* pp = part + b * fl.CP + q;
        vpart_merge(k1, i1g, k2, bad, __ldcg(&pp->k1), __ldcg(&pp->i1), __ldcg(&pp->k2), __ldcg(&pp->bad));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1)
        vpart_merge(k1, i1g, k2, bad, __shfl_xor_sync(FULL, k1, o), __shfl_xor_sync(FULL, i1g, o),
                    __shfl_xor_sync(FULL, k2, o), __shfl_xor_sync(FULL, bad, o));
      if (lane == 0) {
        const bool exact = ce.x == 0.0 && ce.y == 0.0;
        // inf/NaN areas: keys were not remapped in the scan, so the exact block scan decides
        bool ok = !bad && (exact || hi - lo == 1);
        if (!ok && !bad && !a.cert_force) {
          // |Q_j| <= (1+u) max|y - ay| over the bucket's y extremes (likewise R)
          const double qmax = fmax(fabs(__dsub_rn(yr.y, ay)), fabs(__dsub_rn(yr.x, ay))) * (1.0 + 4.0 * u);
          const double rmax = fmax(fabs(__dsub_rn(ax, xr.x)), fabs(__dsub_rn(ax, xr.y))) * (1.0 + 4.0 * u);
          const double v1 = k1 < 0 ? -1.0 : __longlong_as_double(k1), v2 = k2 < 0 ? -1.0 : __longlong_as_double(k2);
          const double E = k3c_area_err(ce, P, S, qmax, rmax, v1);
          ok = __dsub_rn(v1, v2) > 2.0 * E * (1.0 + 1e-9);  // NaN bounds fail
        }
        if (ok) {
          const int64_t r = i1g == LLONG_MAX ? lo : i1g;  // all-NaN bucket keeps bounds[b] (:110)
          a.best[s * k3 + b] = r;
          const bool fg = r != pos[b + 1];
          a.flag[s * k3 + b] = fg;
          if (fg) a.flist[s * k3 + atomicAdd(&a.fcount[s], 1)] = (int)b;
        } else {
          fl.ulist[s * k3 + atomicAdd(&fl.ucount[s], 1)] = (int)b;
        }
      }
    }
    j = s1;
  }
}

// Buckets whose flat certification failed: exact in-order mean, exact re-scan.
template <typename XT, typename YT, int NT>
__global__ void __launch_bounds__(NT) k_lttb_verify_fix(LttbArgs a, FlatArgs fl) {
  __shared__ double s_a[NT / 32];
  __shared__ long long s_i[NT / 32];
  const int64_t s = blockIdx.y;
  const int64_t k3 = a.n_out - 2;
  const int nu = fl.ucount[s];
  const int64_t m = a.m_dev ? a.m_dev[s] : a.n;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  const int64_t* pos = a.pos + s * a.pos_ld;
  for (int q = blockIdx.x; q < nu; q += gridDim.x) {
    const int64_t b = fl.ulist[s * k3 + q];
    const int64_t r = k3c_argmax<XT, YT, NT>(a, s, m, xs, ys, b, pos[b], s_a, s_i);
    if (threadIdx.x == 0) {
      a.best[s * k3 + b] = r;
      const bool fg = r != pos[b + 1];
      a.flag[s * k3 + b] = fg;
      if (fg) a.flist[s * k3 + atomicAdd(&a.fcount[s], 1)] = (int)b;
    }
  }
}

// Flat means pass: per-bucket any-order sums, magnitudes, lowest set bits,
// x / y extremes (integer keys) and the affine-x test, from equal element
// ranges per warp (partials combined by the bucket's last-arriving warp).
struct MPart { double sx, sy, ax, ay; long long kxmn, kxmx, kymn, kymx; int lx, ly, aff, pad; };

__device__ __forceinline__ void mpart_merge(MPart& p, const MPart& o) {
  p.sx += o.sx; p.sy += o.sy; p.ax += o.ax; p.ay += o.ay;
  p.kxmn = min(p.kxmn, o.kxmn); p.kxmx = max(p.kxmx, o.kxmx);
  p.kymn = min(p.kymn, o.kymn); p.kymx = max(p.kymx, o.kymx);
  p.lx = min(p.lx, o.lx); p.ly = min(p.ly, o.ly); p.aff &= o.aff;
}
__device__ __forceinline__ void mpart_shfl(MPart& p, int o) {
  MPart q;
  q.sx = __shfl_xor_sync(FULL, p.sx, o); q.sy = __shfl_xor_sync(FULL, p.sy, o);
  q.ax = __shfl_xor_sync(FULL, p.ax, o); q.ay = __shfl_xor_sync(FULL, p.ay, o);
  q.kxmn = __shfl_xor_sync(FULL, p.kxmn, o); q.kxmx = __shfl_xor_sync(FULL, p.kxmx, o);
  q.kymn = __shfl_xor_sync(FULL, p.kymn, o); q.kymx = __shfl_xor_sync(FULL, p.kymx, o);
  q.lx = __shfl_xor_sync(FULL, p.lx, o); q.ly = __shfl_xor_sync(FULL, p.ly, o);
  q.aff = __shfl_xor_sync(FULL, p.aff, o);
  mpart_merge(p, q);
}
__device__ __forceinline__ void mpart_init(MPart& p, bool integral) {
  p.sx = p.sy = p.ax = p.ay = 0.0;
  p.kxmn = p.kymn = LLONG_MAX; p.kxmx = p.kymx = LLONG_MIN;
  p.lx = integral ? 0 : 4096; p.ly = 4096; p.aff = 1; p.pad = 0;
}

// exponent of |v| (unbiased), for the exactness pre-check
__device__ __forceinline__ int exp_of(double v) { return (int)((__double_as_longlong(v) >> 52) & 0x7ff) - 1023; }

// One warp's pass over a means segment [0, n): any-order sums, magnitudes,
// y extremes (keys), x extremes, lowest set bits (TRYY: y's; float x: x's when
// try_x) and the affine-x test against the bucket's formula.
template <bool TRYY, typename XT, typename YT, int UN>
__device__ __forceinline__ void means_scan(const XT* __restrict__ xb, const YT* __restrict__ yb, int n, int lane,
                                           const XAff& f, int64_t t0, MPart& p, long long& xmn, long long& xmx,
                                           bool try_x) {
  const long long dstep = (long long)((unsigned long long)f.di * 32ull);
  long long xe = (long long)((unsigned long long)f.x0i + (unsigned long long)(t0 + lane) * (unsigned long long)f.di);
  // y extremes on the HIGH word of the total-order key (32-bit min/max, one
  // instruction each): a conservative range, exact to ~2^-20 relative, which is
  // all the direction search and the certification bound need
  int hmn = INT_MAX, hmx = INT_MIN;
  for (int i = lane; i < n; i += 32 * UN) {
    XT rx[UN];
    YT ry[UN];
    const bool full = i + 32 * (UN - 1) < n;
    if (full) {
      const XT* xp = xb + i;
      const YT* yp = yb + i;
#pragma unroll
      for (int q = 0; q < UN; ++q) {
        rx[q] = __ldcs(xp + 32 * q);  // x streams (evict-first): y stays L2-resident for the later passes
        ry[q] = yp[32 * q];
      }
    } else {
#pragma unroll
      for (int q = 0; q < UN; ++q) {
        const int ii = i + 32 * q < n ? i + 32 * q : i;
        rx[q] = __ldcs(xb + ii);
        ry[q] = yb[ii];
      }
    }
#pragma unroll
    for (int q = 0; q < UN; ++q) {
      if (full || i + 32 * q < n) {
        const double vx = elem_f64(rx[q]), vy = elem_f64(ry[q]);
        p.sx = __dadd_rn(p.sx, vx); p.sy = __dadd_rn(p.sy, vy);
        p.ax = __dadd_rn(p.ax, fabs(vx)); p.ay = __dadd_rn(p.ay, fabs(vy));
        const int hy = (int)(__double_as_longlong(vy) >> 32);
        const int hk = hy ^ ((hy >> 31) & 0x7fffffff);  // == dkey(vy) >> 32
        hmn = min(hmn, hk);
        hmx = max(hmx, hk);
        if (TRYY) p.ly = min(p.ly, lsb_exp(vy));
        if constexpr (XForm<XT>::integral) {
          const long long xi = (long long)rx[q];
          if (xi < xmn) xmn = xi;
          if (xi > xmx) xmx = xi;
          p.aff &= xi == xe;
        } else {
          const long long kx = dkey(vx);
          if (kx < p.kxmn) p.kxmn = kx;
          if (kx > p.kxmx) p.kxmx = kx;
          if (try_x) p.lx = min(p.lx, lsb_exp(vx));
          p.aff &= __double_as_longlong(vx) == __double_as_longlong(XForm<XT>::at(f, t0 + i + 32 * q));
        }
      }
      xe = (long long)((unsigned long long)xe + (unsigned long long)dstep);
    }
  }
  if (hmn <= hmx) {
    p.kymn = min(p.kymn, (long long)hmn * 4294967296LL);                  // <= every key
    p.kymx = max(p.kymx, (long long)hmx * 4294967296LL + 4294967295LL);  // >= every key
  }
}

template <typename XT, typename YT, int UN>
__global__ void __launch_bounds__(256, K3C_FLAT_MINB) k_lttb_means_flat(LttbArgs a, FlatArgs fl) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t s = blockIdx.y;
  const int64_t k3 = a.n_out - 2, m = a.n;
  const int64_t e0 = 1 + gw * fl.E, e1 = min(m - 1, e0 + fl.E);
  if (gw >= fl.W || e0 >= e1) return;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  MPart* part = (MPart*)fl.part + s * k3 * fl.CP;
  int64_t b = lttb_bucket_of(e0, m, k3);
  for (int64_t j = e0; j < e1; ++b) {
    const int64_t lo = lbound(a, m, b), hi = lbound(a, m, b + 1);
    const int64_t s1 = min(e1, hi);
    const int n = (int)(s1 - j);
    XAff f;  // affine-x candidate from the bucket's first two points
    {
      const XT x0r = xs[lo], x1r = hi - lo > 1 ? xs[lo + 1] : xs[lo];
      f.x0 = (double)x0r;
      f.d = __dsub_rn((double)x1r, (double)x0r);
      f.x0i = (long long)x0r;
      f.di = (long long)((unsigned long long)(long long)x1r - (unsigned long long)(long long)x0r);
    }
    // exactness is only worth tracking (lowest set bits) when it is plausible:
    // full-mantissa values can never have every partial sum representable, and
    // declaring a mean inexact is always safe (it is then certified)
    const double nb = (double)(hi - lo);
    const double y0 = elem_f64(ys[j]), x0 = elem_f64(xs[j]);
    const bool try_y = y0 == 0.0 || (double)lsb_exp(y0) + 55.0 > (double)exp_of(y0) + log2(nb);
    const bool try_x = !XForm<XT>::integral && (x0 == 0.0 || (double)lsb_exp(x0) + 55.0 > (double)exp_of(x0) + log2(nb));
    const XT* xb = xs + j;
    const YT* yb = ys + j;
    MPart p;
    mpart_init(p, XForm<XT>::integral);
    if (!try_y) p.ly = -4096;
    if (!XForm<XT>::integral && !try_x) p.lx = -4096;
    long long xmn = LLONG_MAX, xmx = LLONG_MIN;  // integer x: extremes on the values themselves
    if (try_y) means_scan<true, XT, YT, UN>(xb, yb, n, lane, f, j - lo, p, xmn, xmx, try_x);
    else means_scan<false, XT, YT, UN>(xb, yb, n, lane, f, j - lo, p, xmn, xmx, try_x);
    if constexpr (XForm<XT>::integral) {  // keys of the (exactly or nearest-) converted extremes
      if (xmn <= xmx) {
        p.kxmn = dkey(elem_f64((XT)xmn));
        p.kxmx = dkey(elem_f64((XT)xmx));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mpart_shfl(p, o);
    const int64_t w0 = (lo - 1) / fl.E;
    const unsigned ns = (unsigned)((hi - 2) / fl.E - w0 + 1);
    bool last = false;
    if (lane == 0) {
      part[b * fl.CP + (gw - w0)] = p;
      last = flat_arrive(fl.cnt + s * k3 + b, ns);
    }
    if (__shfl_sync(FULL, (int)last, 0)) {
      mpart_init(p, true);
      p.lx = 4096;
      for (unsigned q = lane; q < ns; q += 32) {
        const MPart* pp = part + b * fl.CP + q;
        MPart o;
        o.sx = __ldcg(&pp->sx); o.sy = __ldcg(&pp->sy); o.ax = __ldcg(&pp->ax); o.ay = __ldcg(&pp->ay);
        o.kxmn = __ldcg(&pp->kxmn); o.kxmx = __ldcg(&pp->kxmx); o.kymn = __ldcg(&pp->kymn); o.kymx = __ldcg(&pp->kymx);
        o.lx = __ldcg(&pp->lx); o.ly = __ldcg(&pp->ly); o.aff = __ldcg(&pp->aff);
        mpart_merge(p, o);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) mpart_shfl(p, o);
      if (lane == 0) {
        a.yrange[s * k3 + b] = make_double2(dkey_inv(p.kymn), dkey_inv(p.kymx));
        a.xrange[s * k3 + b] = make_double2(dkey_inv(p.kxmn), dkey_inv(p.kxmx));
        if (a.xaff) {
          f.ok = p.aff;
          f.pad = 0;
          a.xaff[s * k3 + b] = f;
        }
        if (b >= 1) {
          a.means[s * a.means_ld + b - 1] = make_double2(__ddiv_rn(p.sx, nb), __ddiv_rn(p.sy, nb));
          a.merr[s * k3 + b - 1] = make_double2(mean_err_bound(p.sx, p.ax, p.lx, nb), mean_err_bound(p.sy, p.ay, p.ly, nb));
        } else {  // the last bucket anchors on point m-1 itself (_kernels.py:105-107): exact
          a.means[s * a.means_ld + k3 - 1] = make_double2(to_f64(xs, m - 1), to_f64(ys, m - 1));
          a.merr[s * k3 + k3 - 1] = make_double2(0.0, 0.0);
        }
      }
    }
    j = s1;
  }
}

template <typename XT, typename YT, int NT>
__global__ void __launch_bounds__(NT) k_lttb_verify(LttbArgs a) {
  __shared__ double s_a[NT / 32];
  __shared__ long long s_i[NT / 32];
  const int64_t s = blockIdx.y;
  const int64_t b = blockIdx.x;
  const int64_t k3 = a.n_out - 2;
  const int64_t m = a.m_dev ? a.m_dev[s] : a.n;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  const int64_t* pos = a.pos + s * a.pos_ld;
  const int64_t prev = pos[b];
  const int64_t r = k3c_argmax<XT, YT, NT>(a, s, m, xs, ys, b, prev, s_a, s_i);
  if (threadIdx.x == 0) {
    a.best[s * k3 + b] = r;
    const bool f = r != pos[b + 1];
    a.flag[s * k3 + b] = f;
    if (f) a.flist[s * k3 + atomicAdd(&a.fcount[s], 1)] = (int)b;
  }
}

// Speculative second step: for every bucket right after a mismatch, the
// exact pick given the EXACT previous pick (best[b-1]) -- in parallel, so an
// isolated mismatch is repaired without any sequential re-scan.
template <typename XT, typename YT, int NT>
__global__ void __launch_bounds__(NT) k_lttb_verify2(LttbArgs a) {
  __shared__ double s_a[NT / 32];
  __shared__ long long s_i[NT / 32];
  const int64_t s = blockIdx.y;
  const int64_t k3 = a.n_out - 2;
  const int nf = a.fcount[s];
  const int64_t m = a.m_dev ? a.m_dev[s] : a.n;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  for (int q = blockIdx.x; q < nf; q += gridDim.x) {  // one flagged bucket f per CTA: bucket f+1
    const int64_t b = (int64_t)a.flist[s * k3 + q] + 1;
    if (b >= k3) continue;
    const int64_t prev = a.best[s * k3 + b - 1];
    const int64_t r = k3c_argmax<XT, YT, NT>(a, s, m, xs, ys, b, prev, s_a, s_i);
    if (threadIdx.x == 0) a.best2[s * k3 + b] = r;
  }
}

static __device__ unsigned long long g_repair_scans;  // exact bucket scans done by k_lttb_repair (stats)

template <typename XT, typename YT, int NT>
__global__ void __launch_bounds__(NT) k_lttb_repair(LttbArgs a) {
  constexpr int LMAX = 2048;  // flagged buckets sorted in shared memory (more: linear search)
  __shared__ double s_a[NT / 32];
  __shared__ long long s_i[NT / 32];
  __shared__ int s_f[LMAX];
  __shared__ long long s_next;
  const int64_t s = blockIdx.x;
  const int64_t k3 = a.n_out - 2;
  const int64_t m = a.m_dev ? a.m_dev[s] : a.n;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  int64_t* pos = a.pos + s * a.pos_ld;
  const int* flag = a.flag + s * k3;
  const int64_t* best = a.best + s * k3;
  const int nf = a.fcount[s];
  const bool listed = nf <= LMAX;
  if (listed) {
    for (int i = threadIdx.x; i < nf; i += NT) s_f[i] = a.flist[s * k3 + i];
    __syncthreads();
    // odd-even transposition sort of the (few) flagged buckets
    for (int ph = 0; ph < nf; ++ph) {
      for (int i = 2 * threadIdx.x + (ph & 1); i + 1 < nf; i += 2 * NT)
        if (s_f[i] > s_f[i + 1]) { const int t = s_f[i]; s_f[i] = s_f[i + 1]; s_f[i + 1] = t; }
      __syncthreads();
    }
  }
  int64_t b = 0;
  int qi = 0;
  while (b < k3) {
    // next verified mismatch at or after b (the chain is synced up to b)
    int64_t nb;
    if (listed) {
      while (qi < nf && s_f[qi] < b) ++qi;
      nb = qi < nf ? s_f[qi] : LLONG_MAX;
    } else {
      if (threadIdx.x == 0) s_next = LLONG_MAX;
      __syncthreads();
      for (int64_t i = b + threadIdx.x; i < k3; i += NT)
        if (flag[i]) atomicMin(&s_next, (long long)i);
      __syncthreads();
      nb = s_next;
      __syncthreads();
    }
    if (nb >= k3) break;
    b = nb;
    __syncthreads();
    if (threadIdx.x == 0) pos[b + 1] = best[b];  // exact: prev pos[b] is on the true chain
    __syncthreads();
    ++b;
    // walk exactly until the chain re-joins the (verified) candidate chain
    while (b < k3) {
      const int64_t prev = pos[b];
      int64_t r;
      if (flag[b - 1] && prev == best[b - 1]) {
        r = a.best2[s * k3 + b];  // precomputed by k_lttb_verify2
      } else {
        r = k3c_argmax<XT, YT, NT>(a, s, m, xs, ys, b, prev, s_a, s_i);
        if (threadIdx.x == 0) atomicAdd(&g_repair_scans, 1ull);
      }
      const int64_t was = pos[b + 1];
      __syncthreads();
      if (threadIdx.x == 0) pos[b + 1] = r;
      __syncthreads();
      ++b;
      if (r == was) break;  // synced: later buckets were verified with this prev
    }
  }
  __syncthreads();
  int64_t* out = a.out + s * a.n_out;
  const int64_t* map = a.map ? a.map + s * a.map_ld : nullptr;
  for (int64_t i = threadIdx.x; i < k3 + 2; i += NT) {
    const int64_t p = pos[i];
    out[i] = map ? map[p] : p;
  }
}

// Same walk with the chain state staged in shared memory (k3 <= ~7,000): the
// positions, verified picks, speculative picks and a next-flagged-bucket
// index (suffix minimum over the flags) live on chip, so each walk step
// costs shared-memory reads instead of dependent global round trips, and no
// flagged-list sort is needed.
__host__ __device__ inline int64_t repair_smem_bytes(int64_t k3) { return 8 * (k3 + 2) + 16 * k3 + 4 * (k3 + 1); }

// (device function: also run by the last CTA of the single-launch K3s kernel,
// which reads state other CTAs wrote in the same launch -- hence the L2 loads)
template <typename XT, typename YT, int NT, typename Pick>
__device__ void repair_walk_smem_p(const LttbArgs& a, int64_t s, unsigned char* dsm, Pick pick) {
  __shared__ double s_a[NT / 32];
  __shared__ long long s_i[NT / 32];
  __shared__ int s_cm[NT];
  const int64_t k3 = a.n_out - 2;
  long long* P = (long long*)dsm;  // chain positions [k3 + 2]
  long long* Bv = P + (k3 + 2);    // verified pick given P[b] [k3]
  long long* B2 = Bv + k3;         // pick given Bv[b-1] (valid where b-1 is flagged) [k3]
  int* Nx = (int*)(B2 + k3);       // smallest flagged bucket >= i, or INT_MAX [k3 + 1]
  const int64_t* pos = a.pos + s * a.pos_ld;
  const int* flag = a.flag + s * k3;
  // coalesced staging (flags into Nx first), 4 rows of loads in flight per thread
  for (int64_t i0 = threadIdx.x; i0 < k3 + 2; i0 += 4 * NT) {
    long long vp[4], vb[4], v2[4];
    int vf[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + q * NT;
      if (i < k3 + 2) vp[q] = __ldcg(pos + i);
      if (i < k3) { vb[q] = __ldcg(a.best + s * k3 + i); v2[q] = __ldcg(a.best2 + s * k3 + i); vf[q] = __ldcg(flag + i); }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + q * NT;
      if (i < k3 + 2) P[i] = vp[q];
      if (i < k3) { Bv[i] = vb[q]; B2[i] = v2[q]; Nx[i] = vf[q]; }
    }
  }
  __syncthreads();
  // next-flagged index: per-thread chunk suffix (shared memory), then a suffix minimum over chunks
  const int64_t C = (k3 + NT - 1) / NT;
  const int64_t c0 = threadIdx.x * C, c1 = min(k3, c0 + C);
  int nxt = INT_MAX;
  for (int64_t i = c1 - 1; i >= c0; --i) {
    if (Nx[i]) nxt = (int)i;
    Nx[i] = nxt;
  }
  s_cm[threadIdx.x] = nxt;
  __syncthreads();
  for (int o = 1; o < NT; o <<= 1) {  // Hillis-Steele suffix minimum
    const int v = threadIdx.x + o < NT ? s_cm[threadIdx.x + o] : INT_MAX;
    __syncthreads();
    s_cm[threadIdx.x] = min(s_cm[threadIdx.x], v);
    __syncthreads();
  }
  const int carry = threadIdx.x + 1 < NT ? s_cm[threadIdx.x + 1] : INT_MAX;
  for (int64_t i = c0; i < c1; ++i)
    if (Nx[i] == INT_MAX) Nx[i] = carry;
  if (threadIdx.x == 0) Nx[k3] = INT_MAX;
  __syncthreads();
  // Thread 0 walks the chain alone (shared-memory state only, no barrier per
  // step) and hands a bucket to the whole CTA only when it needs an exact scan.
#ifdef MM_REPAIR_TRACE
  const long long t_walk0 = clock64();
  long long t_scan = 0;
  int n_scan = 0;
#endif
  __shared__ long long s_rb, s_rp;  // scan request: bucket, previous pick (-1: walk finished)
  int64_t b = 0;                    // thread 0: chain synced up to b
  bool walking = false;             // thread 0: inside a deviation
  int64_t scanned = -1;             // thread 0: result of the last requested scan
  while (true) {
    if (threadIdx.x == 0) {
      s_rb = -1;
      while (true) {
        if (!walking) {
          const int64_t nb = b < k3 ? Nx[b] : INT_MAX;  // next verified mismatch at or after b
          if (nb >= k3) break;
          b = nb;
          P[b + 1] = Bv[b];  // exact: P[b] is on the true chain
          ++b;
          walking = true;
        }
        if (b >= k3) break;
        const int64_t prev = P[b];
        int64_t r;
        if (scanned >= 0) {
          r = scanned;
          scanned = -1;
        } else if (Nx[b - 1] == b - 1 && prev == Bv[b - 1]) {
          r = B2[b];  // precomputed by k_lttb_verify2
        } else {
          s_rb = b;
          s_rp = prev;
          break;
        }
        const int64_t was = P[b + 1];
        P[b + 1] = r;
        ++b;
        if (r == was) walking = false;  // re-joined the verified candidate chain
      }
    }
    __syncthreads();
    const int64_t rb = s_rb;
    if (rb < 0) break;
#ifdef MM_REPAIR_TRACE
    const long long t0s = clock64();
#endif
    const int64_t r = pick(rb, (int64_t)s_rp, s_a, s_i);
    if (threadIdx.x == 0) {
      scanned = r;
      atomicAdd(&g_repair_scans, 1ull);
#ifdef MM_REPAIR_TRACE
      t_scan += clock64() - t0s;
      ++n_scan;
#endif
    }
  }
#ifdef MM_REPAIR_TRACE
  if (threadIdx.x == 0) {
    int nflag = 0;
    for (int64_t i = 0; i < k3; i = Nx[i] + 1) { if (Nx[i] >= k3) break; ++nflag; }
    printf("repair: walk+scans %lld cycles, %d scans %lld cycles, %d flagged\n", clock64() - t_walk0, n_scan, t_scan, nflag);
  }
#endif
  __syncthreads();
  int64_t* out = a.out + s * a.n_out;
  const int64_t* map = a.map ? a.map + s * a.map_ld : nullptr;
  for (int64_t i = threadIdx.x; i < k3 + 2; i += NT) {
    const int64_t p = P[i];
    out[i] = map ? map[p] : p;
  }
}

// the walk with K3c's certified block argmax as the exact re-scan
template <typename XT, typename YT, int NT>
__device__ void repair_walk_smem(const LttbArgs& a, int64_t s, unsigned char* dsm) {
  const int64_t m = a.m_dev ? a.m_dev[s] : a.n;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  repair_walk_smem_p<XT, YT, NT>(a, s, dsm, [&](int64_t b, int64_t prev, double* s_a, long long* s_i) {
    return k3c_argmax<XT, YT, NT>(a, s, m, xs, ys, b, prev, s_a, s_i);
  });
}

template <typename XT, typename YT, int NT>
__global__ void __launch_bounds__(NT) k_lttb_repair_smem(LttbArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  repair_walk_smem<XT, YT, NT>(a, blockIdx.x, dsm);
}

// ----------------------------------------------------------- misc -------
static __global__ void k_fill(int64_t* p, int64_t n, int64_t v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

static __global__ void k_every_nth(int64_t n, int64_t n_out, int64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_out) out[i] = (i * n) / n_out;  // downsamplers.py:44-47
}

// TimeSeries invariants on device (core.py:80-94): bit 0 = a non-finite x or
// y, bit 1 = x decreasing somewhere (np.diff(xs) < 0, i.e. x[i+1] < x[i] in
// value: -0.0 == +0.0).  Integer-domain checks only (finiteness from the
// exponent bits, order on integers or +-0-merged total-order keys): no fp64
// compares or int64 conversions, which issue on B200's narrow XU pipe.  Four
// coalesced elements in flight per thread.
template <typename T> __device__ __forceinline__ bool v_nonfinite(T v) { return false; }
template <> __device__ __forceinline__ bool v_nonfinite<float>(float v) {
  return (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
}
template <> __device__ __forceinline__ bool v_nonfinite<double>(double v) {
  return ((unsigned)(__double_as_longlong(v) >> 32) & 0x7ff00000u) == 0x7ff00000u;
}
template <typename T> __device__ __forceinline__ long long v_order(T v) { return (long long)v; }  // int32: exact
// int64: the reference compares the float64 conversions (equal beyond 2^53 when
// the integers differ by less than the rounding step), so order the conversions
template <> __device__ __forceinline__ long long v_order<long long>(long long v) { return dkey(elem_f64(v)); }
template <> __device__ __forceinline__ long long v_order<float>(float v) {
  const int b = __float_as_int(v) == (int)0x80000000 ? 0 : __float_as_int(v);  // -0.0 -> +0.0
  return (long long)(b ^ ((b >> 31) & 0x7fffffff));
}
template <> __device__ __forceinline__ long long v_order<double>(double v) {
  long long b = __double_as_longlong(v);
  b = b == (long long)0x8000000000000000ULL ? 0 : b;
  return b ^ ((b >> 63) & 0x7fffffffffffffffLL);
}

template <typename T> struct V4 {  // 4 consecutive elements from 16-byte loads
  T v[4];
  __device__ __forceinline__ void load(const T* p) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint4 w[sizeof(T) / 4];
#pragma unroll
    for (int k = 0; k < (int)sizeof(T) / 4; ++k) w[k] = __ldg(q + k);
    memcpy(v, w, 4 * sizeof(T));
  }
};

// Batched: series s (blockIdx.y, grid-strided past 65,535) checks x + s*x_ld
// (x_ld 0: shared x) and y + s*y_ld into flags[s].
template <typename XT, typename YT>
__global__ void __launch_bounds__(256) k_validate(const XT* __restrict__ x0, const YT* __restrict__ y0, int64_t n,
                                                 int64_t x_ld, int64_t y_ld, int64_t B, int* flags) {
  // thread t checks elements [4t, 4t+4) per round (16-byte loads; the host
  // guarantees 16-byte aligned rows of x and y), plus the pair (4t+3, 4t+4)
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = blockIdx.y; s < B; s += gridDim.y) {
    const XT* x = x0 + s * x_ld;
    const YT* y = y0 + s * y_ld;
    int f = 0;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c * 4 < n; c += T) {
      const int64_t i0 = c * 4;
      XT xv[5];
      YT yv[4];
      if (i0 + 4 <= n) {
        V4<XT> a;
        V4<YT> b;
        a.load(x + i0);
        b.load(y + i0);
#pragma unroll
        for (int q = 0; q < 4; ++q) { xv[q] = a.v[q]; yv[q] = b.v[q]; }
        xv[4] = i0 + 4 < n ? x[i0 + 4] : xv[3];
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t i = i0 + q < n ? i0 + q : n - 1;
          xv[q] = x[i];
          yv[q] = y[i];
        }
        xv[4] = xv[3];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (i0 + q < n) {
          if (v_nonfinite(xv[q]) || v_nonfinite(yv[q])) f |= 1;  // core.py:89-90
          const XT nx = i0 + q + 1 < n ? xv[q + 1] : xv[q];
          if (v_order(nx) < v_order(xv[q])) f |= 2;               // core.py:91-92
        }
      }
    }
    f = __reduce_or_sync(FULL, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags + s, f);
  }
}

// unaligned inputs (views): one element per thread per round
template <typename XT, typename YT>
__global__ void __launch_bounds__(256) k_validate_scalar(const XT* __restrict__ x0, const YT* __restrict__ y0,
                                                        int64_t n, int64_t x_ld, int64_t y_ld, int64_t B, int* flags) {
  for (int64_t s = blockIdx.y; s < B; s += gridDim.y) {
    const XT* x = x0 + s * x_ld;
    const YT* y = y0 + s * y_ld;
    int f = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      const XT xv = x[i];
      if (v_nonfinite(xv) || v_nonfinite(y[i])) f |= 1;
      if (i + 1 < n && v_order(x[i + 1]) < v_order(xv)) f |= 2;
    }
    f = __reduce_or_sync(FULL, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(flags + s, f);
  }
}

// TSB1 ingest (seriesio.py:75-95): interleaved little-endian f64 (x, y)
// pairs -> separate x and y arrays on the device.
static __global__ void k_deinterleave_f64(const double2* __restrict__ in, double* __restrict__ x, double* __restrict__ y,
                                   int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = __ldcs(in + i);
    x[i] = v.x;
    y[i] = v.y;
  }
}

// ---- device-initiated exchange over peer memory (replaces the NCCL
// all_gather of the sharded single-series path).  Symmetric
// buffer per rank: int64 [2][G][W] (slot = epoch & 1, row = writer rank,
// W = 3*cap + 1: idx | x bits | y bits | count).  Signal pad (uint32) per
// rank: [g] = last epoch whose row from rank g is complete, [G + g] = last
// epoch rank g has consumed from this rank's rows (ack).
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_until_ge(const unsigned* p, unsigned want) {
  while ((int)(ld_acquire_sys(p) - want) < 0) __nanosleep(64);
}

// CTA g: store this rank's preselected set into peer g's buffer, then raise
// the peer's data flag.  Waits first for peer g's ack of epoch-2 (same slot).
static __global__ void k_p2p_publish(const int64_t* idx, const double* xs, const double* ys, const int64_t* count, int64_t cap,
                              const unsigned long long* peer_bufs, const unsigned long long* peer_pads,
                              const unsigned* own_pad, int64_t G, int64_t rank, unsigned epoch) {
  const int64_t g = blockIdx.x;
  const int64_t W = 3 * cap + 1;
  if (threadIdx.x == 0 && epoch > 2) spin_until_ge(own_pad + G + g, epoch - 2);
  __syncthreads();
  long long* dst = reinterpret_cast<long long*>(peer_bufs[g]) + ((int64_t)(epoch & 1) * G + rank) * W;
  const int64_t n = min(*count, cap);
  constexpr int PER = 4;  // loads in flight per thread before the remote stores
  for (int64_t i0 = threadIdx.x; i0 < n; i0 += (int64_t)blockDim.x * PER) {
    long long vi[PER], vx[PER], vy[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int64_t i = i0 + (int64_t)q * blockDim.x;
      if (i < n) { vi[q] = idx[i]; vx[q] = __double_as_longlong(xs[i]); vy[q] = __double_as_longlong(ys[i]); }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int64_t i = i0 + (int64_t)q * blockDim.x;
      if (i < n) { dst[i] = vi[q]; dst[cap + i] = vx[q]; dst[2 * cap + i] = vy[q]; }
    }
  }
  if (threadIdx.x == 0) dst[3 * cap] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<unsigned*>(peer_pads[g]) + rank, epoch);
  }
}

// CTA g: wait for every row of this epoch, append row g at its offset (rank
// order), then ack rank g.
static __global__ void k_p2p_merge(const long long* own_buf, const unsigned* own_pad, const unsigned long long* peer_pads,
                            int64_t G, int64_t rank, int64_t cap, unsigned epoch, int64_t* oi, double* ox, double* oy,
                            int64_t* om) {
  const int64_t g = blockIdx.x;
  const int64_t W = 3 * cap + 1;
  if (threadIdx.x == 0)
    for (int64_t h = 0; h < G; ++h) spin_until_ge(own_pad + h, epoch);
  __syncthreads();
  const long long* rows = own_buf + (int64_t)(epoch & 1) * G * W;
  int64_t off = 0;
  // rows are written by peers over NVLink: read them at L2 (ld.cg), never
  // from a possibly stale L1 line of this slot's previous use
  for (int64_t h = 0; h < g; ++h) off += __ldcg(rows + h * W + 3 * cap);
  const long long* row = rows + g * W;
  const int64_t n = __ldcg(row + 3 * cap);
  constexpr int PER = 4;  // loads in flight per thread
  for (int64_t i0 = threadIdx.x; i0 < n; i0 += (int64_t)blockDim.x * PER) {
    long long vi[PER], vx[PER], vy[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int64_t i = i0 + (int64_t)q * blockDim.x;
      if (i < n) { vi[q] = __ldcg(row + i); vx[q] = __ldcg(row + cap + i); vy[q] = __ldcg(row + 2 * cap + i); }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int64_t i = i0 + (int64_t)q * blockDim.x;
      if (i < n) { oi[off + i] = vi[q]; ox[off + i] = __longlong_as_double(vx[q]); oy[off + i] = __longlong_as_double(vy[q]); }
    }
  }
  if (g == G - 1 && threadIdx.x == 0) om[0] = off + n;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<unsigned*>(peer_pads[g]) + G + rank, epoch);
  }
}

// Rank-order merge straight from the gathered packed messages ([G][3cap+1]:
// idx | x bits | y bits | count), so no unpacking copies are needed.
// Rank-order merge of the gathered shard messages: grid (tiles, G), each CTA
// copies one tile of MERGE_TILE entries of row g after the counts of rows < g.
// Tiles keep every thread's loads independent (one round trip per tile; a
// single CTA per row looping over 16k entries took 88 us on C5).
constexpr int MERGE_TILE = 1024;
static __global__ void __launch_bounds__(256) k_merge_packed(const long long* __restrict__ buf, int64_t G, int64_t cap,
                                                             int64_t* __restrict__ oi, double* __restrict__ ox,
                                                             double* __restrict__ oy, int64_t* __restrict__ om) {
  const int64_t g = blockIdx.y, W = 3 * cap + 1;
  int64_t off = 0;
  for (int64_t h = 0; h < g; ++h) off += buf[h * W + 3 * cap];
  const long long* row = buf + g * W;
  const int64_t n = row[3 * cap];
  const int64_t t0 = (int64_t)blockIdx.x * MERGE_TILE;
  constexpr int PER = MERGE_TILE / 256;
  long long vi[PER], vx[PER], vy[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int64_t i = t0 + q * 256 + threadIdx.x;
    if (i < n) { vi[q] = row[i]; vx[q] = row[cap + i]; vy[q] = row[2 * cap + i]; }
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int64_t i = t0 + q * 256 + threadIdx.x;
    if (i < n) { oi[off + i] = vi[q]; ox[off + i] = __longlong_as_double(vx[q]); oy[off + i] = __longlong_as_double(vy[q]); }
  }
  if (g == G - 1 && blockIdx.x == 0 && threadIdx.x == 0) om[0] = off + n;
}

static __global__ void __launch_bounds__(256) k_merge_shards(const int64_t* __restrict__ idx,
                                                             const double* __restrict__ xs,
                                                             const double* __restrict__ ys,
                                                             const int64_t* __restrict__ counts, int64_t G, int64_t cap,
                                                             int64_t* __restrict__ oi, double* __restrict__ ox,
                                                             double* __restrict__ oy, int64_t* __restrict__ om) {
  const int64_t g = blockIdx.y;
  int64_t off = 0;
  for (int64_t h = 0; h < g; ++h) off += counts[h];
  const int64_t n = counts[g];
  const int64_t t0 = (int64_t)blockIdx.x * MERGE_TILE;
  constexpr int PER = MERGE_TILE / 256;
  int64_t vi[PER];
  double vx[PER], vy[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int64_t i = t0 + q * 256 + threadIdx.x;
    if (i < n) { vi[q] = idx[g * cap + i]; vx[q] = xs[g * cap + i]; vy[q] = ys[g * cap + i]; }
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int64_t i = t0 + q * 256 + threadIdx.x;
    if (i < n) { oi[off + i] = vi[q]; ox[off + i] = vx[q]; oy[off + i] = vy[q]; }
  }
  if (g == G - 1 && blockIdx.x == 0 && threadIdx.x == 0) om[0] = off + n;
}

}  // namespace mm
