// k1_tiles.cuh -- K1 over large closed-form sub-buckets as many short-lived
// 32 KB tile CTAs (round 2): the per-sub-bucket first-occurrence argmin /
// argmax of _argminmax_range / _extrema_by_bucket (_kernels.py:28-78).
//
// Why tiles: the flat K1 gives every warp one long contiguous range (one
// wave, no tail by construction), but a static split leaves the stream's
// finishing time to the slowest SM and spreads the concurrent reads over
// 3,552 separate DRAM streams.  A read probe (tools/probes/read_probe.cu,
// profiles/r02) shows plain 32 KB tiles -- one CTA loads 2,048 16-byte vectors
// with all eight of each lane's loads in flight, reduces, exits, and the
// block scheduler hands the SM the next tile -- stream 400 MB in 66 us vs
// 73 us for per-warp ranges, and 4 GB at 7.04 vs 6.33 TB/s.
//
// Tile t of a series covers vectors [t*TV, (t+1)*TV) of the 16-byte-aligned
// part of [E_lo, E_hi) (the sub-buckets b0 .. b0+nb-1); the < VEC scalar
// elements before the first aligned vector go to tile 0, the ones after the
// last full vector to the last tile (both on warp 0).  Warp w holds the
// tile's vectors [w*WV, (w+1)*WV) in registers (lane l: vectors l, l+32, ...),
// so a warp whose range crosses a sub-bucket edge re-reduces its registers
// once per sub-bucket (masking by element index) -- nothing is re-read.  The
// warps' (key, index) results meet in shared memory; one warp per sub-bucket
// stores the tile's partial (a sub-bucket inside one tile is final at once),
// and k_extrema_tiles_combine, a programmatic dependent launch, reduces each
// sub-bucket's partials in tile order -- no fences or atomics on the tiles'
// exit path (a last-arriver combine per tile, measured first, made the 4 GB
// stream 1.85x slower: every tile paid a fence and an atomic round trip).
// Ties resolve to the lowest index at every level, so the result is the
// reference's first occurrence whatever order the tiles run in.
#pragma once
#include "kernels.cuh"

namespace mm {

constexpr int K1T_NT = 256;  // threads per tile CTA
constexpr int K1T_U = 8;     // 16-byte vectors per lane (all in flight at once)
constexpr int K1T_NBT = 12;  // sub-buckets per tile bound (host: sub-buckets >= one warp's elements)

// floor(n / d) for 0 <= n < 2^62, 0 < d, quotient < 2^50, from a host-rounded 1/d:
// the fp64 estimate is within 1 of the quotient, one correction step each way
// makes it exact (no 64-bit division subroutine on the tile's critical path)
__device__ __forceinline__ int64_t k1t_div(int64_t n, int64_t d, double rd) {
  int64_t q = __double2ll_rz(__dmul_rn(__ll2double_rn(n), rd));
  if (q * d > n) --q;
  if ((q + 1) * d <= n) ++q;
  return q;
}
__device__ __forceinline__ int64_t k1t_pbound(const ExArgs& a, int64_t b) {
  return a.start + k1t_div(b * a.len, a.k, a.rk);  // core.py:173
}
__device__ __forceinline__ int64_t k1t_bucket(const ExArgs& a, int64_t j) {
  return k1t_div((j - a.start + 1) * a.k - 1, a.len, a.rlen);  // inverse of pbound
}

template <typename K>
__device__ __forceinline__ void lex_min(K& k, int64_t& i, K k2, int64_t i2) {
  if (k2 < k || (k2 == k && i2 < i)) { k = k2; i = i2; }
}
template <typename K>
__device__ __forceinline__ void lex_max(K& k, int64_t& i, K k2, int64_t i2) {
  if (k2 > k || (k2 == k && i2 < i)) { k = k2; i = i2; }
}

template <typename T>
__global__ void __launch_bounds__(K1T_NT, sizeof(T) == 4 ? 4 : 3) k_extrema_tiles(ExArgs a) {
  typedef YTr<T> Tr;
  typedef typename Tr::K K;
  constexpr int VEC = Tr::VEC, U = K1T_U, TV = K1T_NT * U, WV = 32 * U, NW = K1T_NT / 32;
  __shared__ Partial slot[K1T_NBT][NW];
  __shared__ int edge[K1T_NBT + 1];

  const unsigned nt = (unsigned)a.nt;
  const int64_t s = blockIdx.x / nt, t = blockIdx.x % nt;
  const T* y = (const T*)a.y + s * a.y_ld;
  const int64_t E_lo = a.e_lo, E_hi = a.e_hi;
  const uintptr_t addr = (uintptr_t)(y + E_lo);
  const int64_t head = min((int64_t)(((16u - (unsigned)(addr & 15u)) & 15u) / sizeof(T)), E_hi - E_lo);
  const int64_t Ev = E_lo + head;             // first element of vector 0
  const int64_t nvec = (E_hi - Ev) / VEC;     // whole vectors inside [E_lo, E_hi)
  const int64_t ntl = nvec > 0 ? (nvec + TV - 1) / TV : 1;
  if (t >= ntl) return;  // block-uniform (the host grid is an upper bound)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool last = t == ntl - 1;
  asm volatile("griddepcontrol.launch_dependents;");  // the combine grid may be scheduled early

  // tile-local coordinates (int32): element o of the tile is base + o
  const int64_t base = Ev + (int64_t)VEC * t * TV;
  const int nvt = (int)min((int64_t)TV, nvec - (int64_t)t * TV);  // vectors in this tile
  const int wv0 = warp * WV, wv1 = min(nvt, wv0 + WV);          // this warp's vectors
  // every load of the CTA is issued before anything else
  const uint4* vp = reinterpret_cast<const uint4*>(y + base);
  uint4 r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int v = wv0 + u * 32 + lane;
    r[u] = v < wv1 ? ld_stream<3>(vp + v) : make_uint4(0, 0, 0, 0);
  }
  // scalar extras on warp 0: head elements (tile 0) on lanes 0..7, tail elements (last tile) on 8..15
  const int tail0 = VEC * nvt;  // (local) first element after the tile's vectors
  const int ntail = last ? (int)(E_hi - (base + tail0)) : 0;
  int xo = INT_MIN;
  K xk = 0;
  if (warp == 0) {
    if (t == 0 && lane < head) xo = lane - (int)head;
    if (lane >= 8 && lane - 8 < ntail) xo = tail0 + lane - 8;
    if (xo != INT_MIN) xk = Tr::key(y + base + xo);
  }
  if (lane < K1T_NBT) {
    Partial p;
    p.kmin = (long long)Tr::kmax(); p.kmax = (long long)Tr::kmin();
    p.imin = INT64_MAX; p.imax = INT64_MAX;
    slot[lane][warp] = p;
  }
  // the tile's sub-bucket edges in local coordinates, computed once (64-bit divisions) while the loads fly
  const int span_lo = t == 0 ? -(int)head : 0, span_hi = tail0 + ntail;
  const int64_t bt0 = k1t_bucket(a, base + span_lo), bt1 = k1t_bucket(a, base + span_hi - 1);
  const int nbt = (int)(bt1 - bt0 + 1);
  if (nbt > K1T_NBT) __trap();  // host contract: sub-buckets >= one warp's elements
  if (threadIdx.x <= nbt) {
    const int64_t e = k1t_pbound(a, bt0 + threadIdx.x) - base;
    edge[threadIdx.x] = (int)min(max(e, (int64_t)span_lo), (int64_t)span_hi);
  }
  __syncthreads();

  // this warp's element span (warp 0 also owns the extras)
  int wlo = wv0 < wv1 ? VEC * wv0 : INT_MAX, whi = wv0 < wv1 ? VEC * wv1 : INT_MIN;
  const bool extras = warp == 0 && ((t == 0 && head > 0) || ntail > 0);
  if (extras) {
    if (t == 0 && head > 0) wlo = span_lo, whi = max(whi, 0);
    if (ntail > 0) whi = span_hi, wlo = min(wlo, tail0);
  }
  int jw0 = 0, jw1 = -1;  // sub-buckets (tile-relative) meeting the warp's span
  for (int j = 0; j < nbt; ++j) {
    if (edge[j + 1] > wlo && edge[j] < whi) { if (jw1 < 0) jw0 = j; jw1 = j; }
  }
  if (jw0 == jw1 && !extras) {
    // common case: the warp's vectors all lie in one sub-bucket -> reduce the registers
    K mn = Tr::kmax(), mx = Tr::kmin();
    int um = -1, ux = -1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (wv0 + u * 32 + lane < wv1) {
        K kk[VEC];
        Tr::keys(r[u], kk);
        K vl = kk[0], vh = kk[0];
#pragma unroll
        for (int e = 1; e < VEC; ++e) { vl = min(vl, kk[e]); vh = max(vh, kk[e]); }
        if (vl < mn) { mn = vl; um = u; }
        if (vh > mx) { mx = vh; ux = u; }
      }
    }
    int omn = INT_MAX, omx = INT_MAX;  // first component of the winning vector holding the key
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u == um || u == ux) {
        const int o = VEC * (wv0 + u * 32 + lane);
        K kk[VEC];
        Tr::keys(r[u], kk);
#pragma unroll
        for (int e = VEC - 1; e >= 0; --e) {
          if (u == um && kk[e] == mn) omn = o + e;
          if (u == ux && kk[e] == mx) omx = o + e;
        }
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const K k2 = __shfl_xor_sync(FULL, mn, off);
      const int o2 = __shfl_xor_sync(FULL, omn, off);
      if (k2 < mn || (k2 == mn && o2 < omn)) { mn = k2; omn = o2; }
      const K k3 = __shfl_xor_sync(FULL, mx, off);
      const int o3 = __shfl_xor_sync(FULL, omx, off);
      if (k3 > mx || (k3 == mx && o3 < omx)) { mx = k3; omx = o3; }
    }
    if (lane == 0) {
      Partial p;
      p.kmin = (long long)mn; p.kmax = (long long)mx;
      p.imin = omn == INT_MAX ? INT64_MAX : base + omn;
      p.imax = omx == INT_MAX ? INT64_MAX : base + omx;
      slot[jw0][warp] = p;
    }
  } else {
    // a sub-bucket edge (or the scalar extras) inside the warp's span: re-read each
    // piece through L2 (the lines were just fetched; a few warps per tile at most).
    // A superset of the warp's own elements is harmless: (key, index) minima are idempotent.
    for (int j = jw0; j <= jw1; ++j) {
      const int clo = max(wlo, edge[j]), chi = min(whi, edge[j + 1]);
      K mn, mx;
      int omn, omx;
      group_extrema<T, sizeof(T) == 4 ? 4 : 2, 2, 32, false>(y, base + clo, base + chi, lane, mn, omn, mx, omx);
      if (lane == 0) {
        Partial p;
        p.kmin = (long long)mn; p.kmax = (long long)mx;
        p.imin = omn == INT_MAX ? INT64_MAX : base + clo + omn;
        p.imax = omx == INT_MAX ? INT64_MAX : base + clo + omx;
        slot[j][warp] = p;
      }
    }
  }
  __syncthreads();

  // one warp per sub-bucket of the tile: combine the NW warp results, publish the tile's partial
  for (int j = warp; j < nbt; j += NW) {
    long long kmn = LLONG_MAX, kmx = LLONG_MIN;
    int64_t imn = INT64_MAX, imx = INT64_MAX;
    if (lane < NW) {
      const Partial p = slot[j][lane];
      kmn = p.kmin; kmx = p.kmax; imn = p.imin; imx = p.imax;
    }
#pragma unroll
    for (int off = NW / 2; off; off >>= 1) {  // lanes 0..NW-1 (groups of NW never mix)
      const long long k2 = __shfl_xor_sync(FULL, kmn, off);
      const int64_t i2 = __shfl_xor_sync(FULL, imn, off);
      lex_min(kmn, imn, k2, i2);
      const long long k3 = __shfl_xor_sync(FULL, kmx, off);
      const int64_t i3 = __shfl_xor_sync(FULL, imx, off);
      lex_max(kmx, imx, k3, i3);
    }
    const int64_t b = bt0 + j;
    const int64_t blo = max(k1t_pbound(a, b), E_lo);
    const int64_t bhi = min(k1t_pbound(a, b + 1), E_hi);
    const int64_t tf = blo < Ev ? 0 : min((blo - Ev) / ((int64_t)VEC * TV), ntl - 1);
    const int64_t tl = bhi - 1 < Ev ? 0 : min((bhi - 1 - Ev) / ((int64_t)VEC * TV), ntl - 1);
    if (tl == tf) {  // the whole sub-bucket lies in this tile: final
      if (lane == 0) write_ext(a, s * a.nb + (b - a.b0), imn, imx, kmn, kmx);
    } else if (lane == 0) {  // plain store: k_extrema_tiles_combine reduces the slots (no fence, no atomic)
      Partial p;
      p.kmin = kmn; p.kmax = kmx; p.imin = imn; p.imax = imx;
      a.part[(s * a.nb + (b - a.b0)) * a.CP + (t - tf)] = p;
    }
  }
}

// One thread per (series, sub-bucket) spanning several tiles: the lexicographic
// (key, index) reduction of its tiles' partials in tile order (first occurrence),
// written as the sub-bucket's Ext.  Launched as a programmatic dependent of
// k_extrema_tiles: the launch overlaps the stream, griddepcontrol.wait holds the
// reads until every tile's stores are visible.
template <typename T>
__global__ void __launch_bounds__(256) k_extrema_tiles_combine(ExArgs a) {
  constexpr int VEC = YTr<T>::VEC, TV = K1T_NT * K1T_U;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.B * a.nb) return;
  const int64_t s = g / a.nb, b = a.b0 + g % a.nb;
  const T* y = (const T*)a.y + s * a.y_ld;
  const int64_t E_lo = a.e_lo, E_hi = a.e_hi;
  const uintptr_t addr = (uintptr_t)(y + E_lo);
  const int64_t head = min((int64_t)(((16u - (unsigned)(addr & 15u)) & 15u) / sizeof(T)), E_hi - E_lo);
  const int64_t Ev = E_lo + head, nvec = (E_hi - Ev) / VEC;
  const int64_t ntl = nvec > 0 ? (nvec + TV - 1) / TV : 1;
  const int64_t blo = max(k1t_pbound(a, b), E_lo), bhi = min(k1t_pbound(a, b + 1), E_hi);
  const int64_t tf = blo < Ev ? 0 : min((blo - Ev) / ((int64_t)VEC * TV), ntl - 1);
  const int64_t tl = bhi - 1 < Ev ? 0 : min((bhi - 1 - Ev) / ((int64_t)VEC * TV), ntl - 1);
  if (tl == tf) return;  // written by its tile
  const Partial* pp = a.part + g * a.CP;
  long long kmn = LLONG_MAX, kmx = LLONG_MIN;
  int64_t imn = INT64_MAX, imx = INT64_MAX;
  for (int64_t q = 0; q <= tl - tf; ++q) {
    const Partial p = pp[q];
    lex_min(kmn, imn, p.kmin, p.imin);
    lex_max(kmx, imx, p.kmax, p.imax);
  }
  write_ext(a, g, imn, imx, kmn, kmx);
}

}  // namespace mm
