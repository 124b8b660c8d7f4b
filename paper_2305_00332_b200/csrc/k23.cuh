// k23.cuh -- K23: K2 (compaction of the MinMax pairs) + K3 (LTTB over the
// preselected points, buckets of <= SMAX points) of ONE series in a single
// cooperative launch of G small CTAs -- the tail of every single-series
// MinMaxLTTB call (BASELINE C1, C3, C5).
//
//   A  CTA c compacts sub-buckets [c*TS, (c+1)*TS): its output offset is the
//      sum of the earlier 1-byte counts (one vector pass over all counts,
//      which also gives the total m), a block scan places the (lo, hi) pairs
//      (downsamplers.py:60-69, 157-160), x is gathered, y recovered from the
//      K1 keys.                                              | grid sync
//   B  CTA c owns LTTB buckets [B0, B1): their points and both neighbours'
//      are staged in shared memory, the next-bucket means are the reference's
//      in-order sums (_kernels.py:98-107), the transition tables T_b[p] the
//      exact areas with strict '>' (:108-117); the CTA's maps are composed
//      into its aggregate A_c (16-32 bytes)                  | grid sync
//   C  the chain entering CTA c is (A_{c-1} o ... o A_0)(0); a block scan of
//      the CTA's maps from that entry gives every pick, written as the
//      preselected (global) index.
// Replaces k_compact_pairs + k_lttb_tables + k_lttb_scan (3 launches) and the
// single-CTA k_post_smem: the work is tiny, so the cost is latency, which G
// CTAs with every load round-trip batched keep to ~8 dependent steps.
#pragma once
#include "k3s.cuh"

namespace mm {

constexpr int K23_NT = 256;
constexpr int K23_GMAX = 148 * 4;

struct K23Args {
  const Ext* ext;
  const unsigned char* cnt8;  // 16-byte aligned
  int64_t k;                  // sub-buckets
  int64_t N, n_out;
  const void* x; int xdt;     // x gathered at <= 2k + 2 points: any dtype, switched per load
  const void* y;
  int64_t* pre; double* px; double* py;  // preselected set (global index, x, y as f64)
  int64_t* out;
  int* status;                // bit 0: non-finite y seen (overwritten, not ORed: no zeroing needed)
  unsigned long long* mirror; // optional mapped-host slot: gets mtag | status (mmlttb_status_arm)
  unsigned long long mtag;
  unsigned* sync;             // K23_STAT words: barriers 0, 1 (K3S layout: counter 64 i, flag 64 i + 32), zeroed per call
  unsigned* stat;             // [G] per-CTA status bits (written every call)
  unsigned char* agg;         // [G][32] aggregate maps
  int G, TS;                  // CTAs, sub-buckets per CTA (<= K23_NT * ITEMS)
  int maxb;                   // >= LTTB buckets per CTA
  unsigned long long* prof;   // optional [G][8] %globaltimer stamps (tools), or null
};
constexpr int K23_STAT = 64 * 3;  // zeroed words: barriers 0, 1; word 128 = the K1 chunk ticket

// byte-map helpers over the PMap types (W = 4, 8, 16, 32 bytes)
template <int W> struct MapIO;
template <> struct MapIO<4> {
  typedef PMap<4> M;
  static __device__ __forceinline__ M konst(int e) { return {0x01010101u * (unsigned)e}; }
  static __device__ __forceinline__ void store(unsigned char* p, const M& m) { *reinterpret_cast<uint32_t*>(p) = m.v; }
  static __device__ __forceinline__ M shfl_down(const M& m, int o) { return {__shfl_down_sync(FULL, m.v, o)}; }
};
template <> struct MapIO<8> {
  typedef PMap<8> M;
  static __device__ __forceinline__ M konst(int e) { const uint32_t c = 0x01010101u * (unsigned)e; return {c, c}; }
  static __device__ __forceinline__ void store(unsigned char* p, const M& m) { *reinterpret_cast<uint2*>(p) = make_uint2(m.lo, m.hi); }
  static __device__ __forceinline__ M shfl_down(const M& m, int o) {
    return {__shfl_down_sync(FULL, m.lo, o), __shfl_down_sync(FULL, m.hi, o)};
  }
};
template <int W> struct MapION {
  typedef PMap<W> M;
  static __device__ __forceinline__ M konst(int e) {
    M m;
#pragma unroll
    for (int i = 0; i < W / 4; ++i) m.v[i] = 0x01010101u * (unsigned)e;
    return m;
  }
  static __device__ __forceinline__ void store(unsigned char* p, const M& m) {
#pragma unroll
    for (int i = 0; i < W / 16; ++i)
      reinterpret_cast<uint4*>(p)[i] = make_uint4(m.v[4 * i], m.v[4 * i + 1], m.v[4 * i + 2], m.v[4 * i + 3]);
  }
  static __device__ __forceinline__ M shfl_down(const M& m, int o) {
    M r;
#pragma unroll
    for (int i = 0; i < W / 4; ++i) r.v[i] = __shfl_down_sync(FULL, m.v[i], o);
    return r;
  }
};
template <> struct MapIO<16> : MapION<16> {};
template <> struct MapIO<32> : MapION<32> {};

// Block-wide ordered composition of nb maps (tab + i*W, i ascending = applied
// first): emit(i, T_i o ... o T_0 o carry) for each, and the composition of
// all (returned to every thread).
template <int W, int NT, int IT, typename Emit>
__device__ __forceinline__ PMap<W> k23_scan(const unsigned char* tab, int nb, PMap<W> carry, Emit emit) {
  typedef PMap<W> M;
  __shared__ M s_warp[NT / 32];
  __shared__ M s_carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c0 = 0; c0 < nb; c0 += NT * IT) {
    const int b0 = c0 + threadIdx.x * IT;
    M t[IT];
    M agg = M::ident();
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      t[i] = (b0 + i < nb) ? M::load(tab + (b0 + i) * W) : M::ident();
      agg = M::comp(t[i], agg);
    }
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
    M pre = carry;
    if (wid > 0) pre = M::comp(s_warp[wid - 1], pre);
    const M lane_prev = inc.shfl_up(1);
    if (lane > 0) pre = M::comp(lane_prev, pre);
    M cur = pre;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      cur = M::comp(t[i], cur);
      if (b0 + i < nb) emit(b0 + i, cur);
    }
    if (threadIdx.x == NT - 1) s_carry = M::comp(s_warp[NT / 32 - 1], carry);
    __syncthreads();
    carry = s_carry;
    __syncthreads();
  }
  return carry;
}

template <typename YT, int SMAX, int ITEMS>
__global__ void __launch_bounds__(K23_NT) k_k23(K23Args a) {
  constexpr int NT = K23_NT;
  typedef PMap<SMAX> M;
  typedef MapIO<SMAX> IO;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ int sh[NT / 32 + 1];
  __shared__ long long s_red[2][NT / 32];
  __shared__ int s_e;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int c = blockIdx.x;
  const unsigned G = (unsigned)a.G;
  const int64_t k = a.k, N = a.N, k3 = a.n_out - 2;
  const YT* ys = (const YT*)a.y;
  const int ydt = sizeof(YT) == 4 ? 0 : 1;
  int stat = 0;  // this thread's non-finite-y bit
  auto stamp = [&](int i) {
    if (a.prof && t == 0) a.prof[c * 8 + i] = gtimer();
  };
  stamp(0);
  // launched as a programmatic dependent of K1: wait for its grid (and its
  // memory) before reading the extrema (a no-op for an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // ---------------- A: compaction ----------------
  const int64_t b_lo = (int64_t)c * a.TS, b_hi = min(k, b_lo + a.TS);
  // this thread's Ext records (contiguous items), in flight across the count pass
  Ext er[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t bl = b_lo + (int64_t)t * ITEMS + i;
    er[i].imin = er[i].imax = er[i].kmin = er[i].kmax = 0;
    if (bl < b_hi) er[i] = a.ext[bl];
  }
  // counts before the tile and in all: 16 counts per vector load, every load in flight
  long long pre = 0, tot = 0;
  {
    const uint4* cv = reinterpret_cast<const uint4*>(a.cnt8);
    const int64_t nv = (k + 15) / 16;
    for (int64_t v = t; v < nv; v += NT) {
      const uint4 w4 = cv[v];
      const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t j0 = v * 16 + q * 4;  // counts j0 .. j0+3
        uint32_t ww = w[q];
        if (j0 + 4 > k) ww &= k > j0 ? (0xFFFFFFFFu >> (8 * (j0 + 4 - k))) : 0u;
        const uint32_t s = (ww & 0x00FF00FFu) + ((ww >> 8) & 0x00FF00FFu);
        const int sum = (int)((s & 0xFFFFu) + (s >> 16));
        tot += sum;
        if (j0 + 4 <= b_lo) pre += sum;
        else if (j0 < b_lo) {
          const uint32_t wp = ww & (0xFFFFFFFFu >> (8 * (j0 + 4 - b_lo)));
          const uint32_t sp = (wp & 0x00FF00FFu) + ((wp >> 8) & 0x00FF00FFu);
          pre += (sp & 0xFFFFu) + (sp >> 16);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    pre += __shfl_xor_sync(FULL, pre, o);
    tot += __shfl_xor_sync(FULL, tot, o);
  }
  if (lane == 0) { s_red[0][wid] = pre; s_red[1][wid] = tot; }
  __syncthreads();
  pre = 0; tot = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) { pre += s_red[0][w]; tot += s_red[1][w]; }
  const int64_t m = tot + 2;
  {
    int64_t v[2 * ITEMS];
    long long kv[2 * ITEMS];
    bool keep[2 * ITEMS];
    int n = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int64_t bl = b_lo + (int64_t)t * ITEMS + i;
      const bool ok = bl < b_hi;
      const Ext e = er[i];
      if (ok && keys_nonfinite(e.kmin, e.kmax, ydt)) stat = 1;
      const bool mfirst = e.imin <= e.imax;
      v[2 * i] = mfirst ? e.imin : e.imax;  // downsamplers.py:60-69
      v[2 * i + 1] = mfirst ? e.imax : e.imin;
      kv[2 * i] = mfirst ? e.kmin : e.kmax;
      kv[2 * i + 1] = mfirst ? e.kmax : e.kmin;
      keep[2 * i] = ok;
      keep[2 * i + 1] = ok && v[2 * i + 1] != v[2 * i];
      n += (int)keep[2 * i] + (int)keep[2 * i + 1];
    }
    int tt;
    const int ex = block_excl_scan<NT>(n, tt, sh);
    int64_t pos = 1 + pre + ex;
    double gx[2 * ITEMS];
#pragma unroll
    for (int j = 0; j < 2 * ITEMS; ++j) gx[j] = keep[j] ? load_any(a.x, a.xdt, v[j]) : 0.0;  // all gathers in flight
#pragma unroll
    for (int j = 0; j < 2 * ITEMS; ++j)
      if (keep[j]) {
        a.pre[pos] = v[j];
        a.px[pos] = gx[j];
        a.py[pos] = key_value<YT>(kv[j]);  // exact y[v] from its key: no gather
        ++pos;
      }
    if (t == 0 && c == 0) {  // endpoints (downsamplers.py:157-160)
      const double y0 = to_f64(ys, 0), yl = to_f64(ys, N - 1);
      if (!isfinite(y0) || !isfinite(yl)) stat = 1;
      a.pre[0] = 0; a.px[0] = load_any(a.x, a.xdt, 0); a.py[0] = y0;
      a.pre[m - 1] = N - 1; a.px[m - 1] = load_any(a.x, a.xdt, N - 1); a.py[m - 1] = yl;
    }
  }
  stat = __syncthreads_or(stat);
  if (t == 0) a.stat[c] = (unsigned)stat;  // combined after the barrier: no zeroed word needed
  stamp(1);
  k3s_grid_sync(a.sync, 0, G);
  stamp(2);
  if (c == 0 && a.status && wid == 0) {  // the call's status word, overwritten
    unsigned st = 0;
    for (int q = lane; q < (int)G; q += 32) st |= __ldcg(a.stat + q);
    st = __reduce_or_sync(FULL, st);
    if (lane == 0) {
      *a.status = (int)st;
      if (a.mirror) *(volatile unsigned long long*)a.mirror = a.mtag | (st & 1u);
    }
  }
  // ---------------- B: LTTB tables of buckets [B0, B1) ----------------
  const int64_t B0 = (int64_t)c * k3 / G, B1 = (int64_t)(c + 1) * k3 / G;
  const int nb = (int)(B1 - B0);
  auto lb = [&](int64_t b) -> int64_t { return 1 + (b * (m - 2)) / k3; };  // partition(1, m-1, k3)
  const int64_t P0 = B0 == 0 ? 0 : lb(B0 - 1);
  const int64_t P1 = B1 + 1 <= k3 ? lb(B1 + 1) : m;  // exclusive (B1 == k3: through point m-1)
  const int np = (int)(P1 - P0);
  const int npa = (np + 1) & ~1;  // (keeps s_c 16-byte aligned)
  double* s_x = reinterpret_cast<double*>(dsm);
  double* s_y = s_x + npa;
  long long* s_p = reinterpret_cast<long long*>(s_y + npa);  // preselected (global) indices
  double2* s_c = reinterpret_cast<double2*>(s_p + npa);      // next-bucket means [nb]
  unsigned char* s_tab = reinterpret_cast<unsigned char*>(s_c + nb);  // [nb][SMAX]
  unsigned char* s_pm = s_tab + (int64_t)nb * SMAX;  // prefix maps T_b o ... o T_B0 [nb][SMAX]
  for (int i = t; i < np; i += NT) {
    s_x[i] = __ldcg(a.px + P0 + i);
    s_y[i] = __ldcg(a.py + P0 + i);
    s_p[i] = __ldcg(a.pre + P0 + i);
  }
  __syncthreads();
  for (int i = t; i < nb; i += NT) {  // mean of bucket b+1, in order (_kernels.py:98-107)
    const int64_t b = B0 + i;
    double2 cm;
    if (b + 1 < k3) {
      const int64_t nlo = lb(b + 1), nhi = lb(b + 2);
      double sx = 0.0, sy = 0.0;
      for (int64_t j = nlo; j < nhi; ++j) {
        sx = __dadd_rn(sx, s_x[j - P0]);
        sy = __dadd_rn(sy, s_y[j - P0]);
      }
      const double cnt = (double)(nhi - nlo);
      cm = make_double2(__ddiv_rn(sx, cnt), __ddiv_rn(sy, cnt));
    } else {
      cm = make_double2(s_x[m - 1 - P0], s_y[m - 1 - P0]);
    }
    s_c[i] = cm;
  }
  __syncthreads();
  for (int it = t; it < nb * SMAX; it += NT) {  // T_b[p] (anchor p of bucket b-1; bucket 0: point 0)
    const int i = it / SMAX, p = it % SMAX;
    const int64_t b = B0 + i;
    const int64_t blo = lb(b), bhi = lb(b + 1);
    const int64_t alo = b == 0 ? 0 : lb(b - 1);
    const bool valid = b == 0 ? p == 0 : p < blo - alo;
    unsigned char r = 0;
    if (valid) {
      const double ax = s_x[alo + p - P0], ay = s_y[alo + p - P0];
      const double2 cm = s_c[i];
      long long best = -1;
      for (int64_t j = blo; j < bhi; ++j) {
        const long long ar = lttb_area_key(ax, ay, cm.x, cm.y, s_x[j - P0], s_y[j - P0]);
        if (ar > best) { best = ar; r = (unsigned char)(j - blo); }
      }
    }
    s_tab[it] = r;
  }
  __syncthreads();
  // prefix maps of every bucket and the aggregate A_c = T_{B1-1} o ... o T_{B0}
  const M aggm = k23_scan<SMAX, NT, 4>(s_tab, nb, M::ident(), [&](int i, const M& pm) { IO::store(s_pm + (int64_t)i * SMAX, pm); });
  if (t == 0) IO::store(a.agg + (int64_t)c * 32, aggm);
  stamp(3);
  k3s_grid_sync(a.sync, 1, G);
  stamp(4);
  // ---------------- C: chain entry and picks ----------------
  if (wid == 0) {
    int e = 0;
    if (c > 0) {
      const int per = (c + 31) / 32;
      M r = M::ident();
      for (int i = 0; i < per; ++i) {
        const int cc = lane * per + i;
        if (cc < c) r = M::comp(M::load(a.agg + (int64_t)cc * 32), r);  // (L2: written before the sync)
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const M other = IO::shfl_down(r, o);
        if ((lane & (2 * o - 1)) == 0 && lane + o < 32) r = M::comp(other, r);
      }
      e = __shfl_sync(FULL, r.at0(), 0);
    }
    if (lane == 0) s_e = e;
  }
  __syncthreads();
  const int e = s_e;
  for (int i = t; i < nb; i += NT) {  // pick of bucket B0 + i = its prefix map at the entry
    const int64_t b = B0 + i;
    const int sel = s_pm[(int64_t)i * SMAX + e];
    a.out[b + 1] = s_p[lb(b) + sel - P0];
  }
  if (t == 0 && c == 0) a.out[0] = 0;
  if (t == 0 && c == (int)G - 1) a.out[k3 + 1] = N - 1;
  stamp(5);
}

}  // namespace mm
