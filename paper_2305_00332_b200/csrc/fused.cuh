// fused.cuh -- one CTA per series: the whole MinMaxLTTB of a medium series
// (BASELINE C4: 4096 x 1e6 points) without intermediate HBM traffic.
//
//   phase 1  sub-bucket extrema (8-lane groups, group_extrema = K1's scan)
//            -> (lo, hi) offsets and their y values in shared memory
//   phase 2  block scan of the counts, compaction: [0] + (lo, hi)... + [N-1]
//            (downsamplers.py:60-69, 157-160) -> preselected positions and y
//            in shared memory (x is gathered from HBM/L2 on use)
//   phase 3  LTTB over the compacted points (_kernels.py:81-119): means,
//            transition tables and the packed-map block scan, all in shared
//            memory; only the n_out output indices are written to HBM.
// Two CTAs fit per SM (<= ~110 KB shared each), so one CTA's phases 2-3 hide
// behind the other's streaming phase.
#pragma once
#include "kernels.cuh"

namespace mm {

__host__ __device__ inline int64_t k3_of(int64_t n_out) { return n_out - 2; }

struct FusedArgs {
  const void* x; int64_t x_ld;  // x_ld == 0: shared x
  const void* y; int64_t y_ld;
  int64_t B, N, n_out, r_ps;
  int64_t* out;                 // [B][n_out]
  int* status;                  // bit 0: non-finite y seen (may be null)
};

// shared-memory bytes for a series with k sub-buckets (m <= 2k + 2 points);
// y values are kept in their storage type (exact: they are input samples)
__host__ __device__ inline int64_t fused_region1(int64_t k, int64_t k3, int smax, int ysize) {
  const int64_t p1 = k * (2 * ysize + 8);            // phase 1: y lo/hi + offsets lo/hi
  const int64_t p3 = k3 * (16 + smax);               // phase 3 aliases: means + tables
  return ((p1 > p3 ? p1 : p3) + 15) / 16 * 16;
}
// layout: [region1: phase-1 arrays / phase-3 means + tables]
//         [py: m storage type] [pre: m int32]
__host__ __device__ inline int64_t fused_smem(int64_t k, int64_t k3, int smax, int ysize) {
  const int64_t m = 2 * k + 2;
  return fused_region1(k, k3, smax, ysize) + ((m * ysize + 15) / 16) * 16 + ((m * 4 + 15) / 16) * 16;
}

// Phases 2-3 of one series (shared by both fused kernels): compaction of the
// phase-1 results in shared memory, then LTTB; writes the n_out indices.
template <typename XT, typename YT, int SMAX, int NT>
__device__ __forceinline__ void fused_phase23(const FusedArgs& a, int64_t s, unsigned char* sm, int* sh_scan) {
  const int64_t N = a.N;
  const int64_t k = (a.n_out - 2) * (a.r_ps / 2);
  const int64_t mcap = 2 * k + 2;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  YT* s_vlo = reinterpret_cast<YT*>(sm);
  YT* s_vhi = s_vlo + k;
  int* s_lo = reinterpret_cast<int*>(s_vhi + k);
  int* s_hi = s_lo + k;
  const int64_t a1 = fused_region1(k, a.n_out - 2, SMAX, (int)sizeof(YT));
  YT* s_py = reinterpret_cast<YT*>(sm + a1);
  int* s_pre = reinterpret_cast<int*>(sm + a1 + ((mcap * (int64_t)sizeof(YT) + 15) / 16) * 16);
  double2* s_mean = reinterpret_cast<double2*>(sm);
  unsigned char* s_tab = reinterpret_cast<unsigned char*>(s_mean + k3_of(a.n_out));
  // ---- phase 2: compaction (block scan over the k counts) ----
  // (x is gathered lazily in phase 3: staging it here costs 8 B/point of
  // shared memory, i.e. L1 capacity the phase-1 re-reads depend on)
  int64_t carry = 1;  // slot 0 = index 0
  for (int64_t c0 = 0; c0 < k; c0 += NT) {
    const int64_t b = c0 + threadIdx.x;
    int cnt = 0;
    int lo = 0, hi = 0;
    YT vl = 0, vh = 0;
    if (b < k) {
      lo = s_lo[b]; hi = s_hi[b]; vl = s_vlo[b]; vh = s_vhi[b];
      cnt = hi != lo ? 2 : 1;
    }
    int tot;
    const int ex = block_excl_scan<NT>(cnt, tot, sh_scan);
    if (b < k) {
      const int64_t p = carry + ex;
      s_pre[p] = lo; s_py[p] = vl;
      if (cnt == 2) { s_pre[p + 1] = hi; s_py[p + 1] = vh; }
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    if (a.status && (!isfinite((double)ys[0]) || !isfinite((double)ys[N - 1]))) atomicOr(a.status, 1);
    s_pre[0] = 0; s_py[0] = ys[0];
    s_pre[carry] = (int)(N - 1); s_py[carry] = ys[N - 1];
  }
  const int64_t m = carry + 1;
  __syncthreads();
  // ---- phase 3: LTTB over the m preselected points ----
  const int64_t k3 = a.n_out - 2;
  // b * (m - 2) < 2^32 here (m <= 2k + 2 with k bounded by the shared-memory
  // fit), so the bucket bounds use 32-bit division
  const unsigned um = (unsigned)(m - 2), uk3 = (unsigned)k3;
  auto lb = [&](int64_t b) -> int64_t { return 1 + (int64_t)(((unsigned)b * um) / uk3); };
  auto px = [&](int64_t p) -> double { return to_f64(xs, (int64_t)s_pre[p]); };
  for (int64_t b = threadIdx.x; b < k3; b += NT) {  // next-bucket means, in-order sums
    double2 c;
    if (b + 1 < k3) {
      const int64_t nlo = lb(b + 1), nhi = lb(b + 2);
      double sx = 0.0, sy = 0.0;
      for (int64_t j = nlo; j < nhi; ++j) {
        sx = __dadd_rn(sx, px(j));
        sy = __dadd_rn(sy, (double)s_py[j]);
      }
      const double cnt = (double)(nhi - nlo);
      c = make_double2(__ddiv_rn(sx, cnt), __ddiv_rn(sy, cnt));
    } else {
      c = make_double2(px(m - 1), (double)s_py[m - 1]);
    }
    s_mean[b] = c;
  }
  __syncthreads();
  for (int64_t it = threadIdx.x; it < k3 * SMAX; it += NT) {  // transition tables
    const int64_t b = it / SMAX;
    const int p = (int)(it % SMAX);
    const int64_t blo = lb(b), bhi = lb(b + 1);
    int64_t ap = 0;
    bool valid = b == 0 ? p == 0 : p < blo - lb(b - 1);
    if (b > 0) ap = lb(b - 1) + p;
    unsigned char r = 0;
    if (valid) {
      const double ax = px(ap), ay = (double)s_py[ap];
      const double2 c = s_mean[b];
      double best = -1.0;  // fp64 compares here: measured 0.7 % faster on C4 than the integer keys
      for (int64_t j = blo; j < bhi; ++j) {
        const double ar = lttb_area(ax, ay, c.x, c.y, px(j), (double)s_py[j]);
        if (ar > best) { best = ar; r = (unsigned char)(j - blo); }
      }
    }
    s_tab[it] = r;
  }
  __syncthreads();
  // chain: block scan of the packed maps (shared scan_chain)
  int64_t* out = a.out + s * a.n_out;
  scan_chain<SMAX, NT, 1>(s_tab, k3, [&](int64_t b, int sel) { out[b + 1] = s_pre[lb(b) + sel]; });
  if (threadIdx.x == 0) {
    out[0] = 0;
    out[k3 + 1] = N - 1;
  }
}

template <typename XT, typename YT, int SMAX, int NT, int MINB, int U, int LDV = 3, bool KEEPRAW = true>
__global__ void __launch_bounds__(NT, MINB) k_mmlttb_fused(FusedArgs a) {
  typedef YTr<YT> Tr;
  typedef typename Tr::K K;
  constexpr int G = 8, NG = NT / G;
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int sh_scan[NT / 32 + 1];

  const int64_t s = blockIdx.x;
  const int64_t N = a.N;
  const int64_t k = (a.n_out - 2) * (a.r_ps / 2);
  const int64_t L = N - 2;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  // phase-1 arrays: [k] y at lo, y at hi (storage type), lo, hi offsets
  YT* s_vlo = reinterpret_cast<YT*>(sm);
  YT* s_vhi = s_vlo + k;
  int* s_lo = reinterpret_cast<int*>(s_vhi + k);
  int* s_hi = s_lo + k;

  const int lane8 = threadIdx.x & (G - 1);
  const int grp = threadIdx.x / G;
  // ---- phase 1: extrema of every sub-bucket of partition(1, N-1, k) ----
  const int64_t rounds = (k + NG - 1) / NG;  // warp-uniform trip count (group shuffles)
  for (int64_t r = 0; r < rounds; ++r) {
    const int64_t b = r * NG + grp;
    int64_t lo = 0, hi = 0;
    if (b < k) {
      lo = 1 + (b * L) / k;
      hi = 1 + ((b + 1) * L) / k;
    }
    K mn, mx;
    int omn, omx;
    group_extrema<YT, U, LDV, G, KEEPRAW>(ys, lo, hi, lane8, mn, omn, mx, omx);
    if (lane8 == 0 && b < k) {
      if (a.status && keys_nonfinite((long long)mn, (long long)mx, sizeof(YT) == 4 ? 0 : 1)) atomicOr(a.status, 1);
      const bool mfirst = omn <= omx;
      s_lo[b] = (int)(lo + (mfirst ? omn : omx));
      s_hi[b] = (int)(lo + (mfirst ? omx : omn));
      s_vlo[b] = (YT)key_value<YT>((long long)(mfirst ? mn : mx));
      s_vhi[b] = (YT)key_value<YT>((long long)(mfirst ? mx : mn));
    }
  }
  __syncthreads();
  fused_phase23<XT, YT, SMAX, NT>(a, s, sm, sh_scan);
}

// floor(b * L / k) stepped by a fixed number of buckets with adds only
// (quotient + remainder), so the per-bucket bounds of partition(1, N-1, k)
// cost no 64-bit division inside the streaming loop.
struct BoundIter {
  int64_t v, r, dq, dr, k;
  __device__ __forceinline__ void init(int64_t b, int64_t step, int64_t L, int64_t k_) {
    k = k_;
    v = 1 + (b * L) / k;
    r = (b * L) % k;
    dq = (step * L) / k;
    dr = (step * L) % k;
  }
  __device__ __forceinline__ void next() {
    v += dq;
    r += dr;
    if (r >= k) { r -= k; ++v; }
  }
};

}  // namespace mm

namespace mm {

// ---------------------------------------------------------------------------
// K2+K3 in one CTA per series (single / few large series): compaction of the
// K1 bucket extrema, gather, means, transition tables and the chain scan in
// one launch -- removes two kernel boundaries (~20 us of fixed latency) from
// every call.  px/py are written and re-read inside the kernel, so they are
// read with ld.global.cg (never the non-coherent path).
struct PostArgs {
  const Ext* ext;
  int64_t k;                       // sub-buckets per series
  const void* x; int64_t x_ld;
  const void* y; int64_t y_ld;
  int64_t N, n_out;
  int64_t* pre; double* px; double* py; int64_t cap;  // [B][cap] preselected set
  int64_t* out;                    // [B][n_out]
  int* status;
};

__host__ __device__ inline int64_t post_smem(int64_t k3, int smax) {
  return k3 * 16 + ((k3 * smax + 15) / 16) * 16;
}

template <typename XT, typename YT, int SMAX, int NT>
__global__ void __launch_bounds__(NT) k_post_fused(PostArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int sh[NT / 32 + 1];
  __shared__ long long s_m;
  const int64_t s = blockIdx.x;
  const int64_t k = a.k, N = a.N, k3 = a.n_out - 2;
  const Ext* ext = a.ext + s * k;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  int64_t* pre = a.pre + s * a.cap;
  double* px = a.px + s * a.cap;
  double* py = a.py + s * a.cap;
  double2* s_mean = reinterpret_cast<double2*>(sm);
  unsigned char* s_tab = sm + k3 * 16;
  const int ydt = sizeof(YT) == 4 ? 0 : 1;
  // ---- compaction: [0] + (lo, hi)... + [N-1]  (downsamplers.py:60-69, 157-160)
  int64_t carry = 1;
  for (int64_t c0 = 0; c0 < k; c0 += NT) {
    const int64_t b = c0 + threadIdx.x;
    int n = 0;
    int64_t lo = 0, hi = 0;
    long long klo = 0, khi = 0;
    if (b < k) {
      const Ext e = ext[b];
      if (a.status && keys_nonfinite(e.kmin, e.kmax, ydt)) atomicOr(a.status, 1);
      const bool mfirst = e.imin <= e.imax;
      lo = mfirst ? e.imin : e.imax;
      hi = mfirst ? e.imax : e.imin;
      klo = mfirst ? e.kmin : e.kmax;
      khi = mfirst ? e.kmax : e.kmin;
      n = hi != lo ? 2 : 1;
    }
    int tot;
    const int ex = block_excl_scan<NT>(n, tot, sh);
    if (b < k) {
      const int64_t p = carry + ex;
      const double xl = to_f64(xs, lo), xh = n == 2 ? to_f64(xs, hi) : 0.0;  // both gathers in flight
      pre[p] = lo; px[p] = xl; py[p] = key_value<YT>(klo);
      if (n == 2) { pre[p + 1] = hi; px[p + 1] = xh; py[p + 1] = key_value<YT>(khi); }
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    const double y0 = to_f64(ys, 0), yl = to_f64(ys, N - 1);
    if (a.status && (!isfinite(y0) || !isfinite(yl))) atomicOr(a.status, 1);
    pre[0] = 0; px[0] = to_f64(xs, 0); py[0] = y0;
    pre[carry] = N - 1; px[carry] = to_f64(xs, N - 1); py[carry] = yl;
    s_m = carry + 1;
  }
  __syncthreads();
  const int64_t m = s_m;
  auto lb = [&](int64_t b) -> int64_t { return 1 + (b * (m - 2)) / k3; };
  auto X = [&](int64_t p) -> double { return __ldcg(px + p); };
  auto Y = [&](int64_t p) -> double { return __ldcg(py + p); };
  // ---- LTTB over the m points (_kernels.py:81-119): means, tables, chain
  for (int64_t b = threadIdx.x; b < k3; b += NT) {
    double2 c;
    if (b + 1 < k3) {
      const int64_t nlo = lb(b + 1), nhi = lb(b + 2);
      double sx = 0.0, sy = 0.0;
      for (int64_t j = nlo; j < nhi; ++j) {
        sx = __dadd_rn(sx, X(j));
        sy = __dadd_rn(sy, Y(j));
      }
      const double cnt = (double)(nhi - nlo);
      c = make_double2(__ddiv_rn(sx, cnt), __ddiv_rn(sy, cnt));
    } else {
      c = make_double2(X(m - 1), Y(m - 1));
    }
    s_mean[b] = c;
  }
  __syncthreads();
  for (int64_t it = threadIdx.x; it < k3 * SMAX; it += NT) {
    const int64_t b = it / SMAX;
    const int p = (int)(it % SMAX);
    const int64_t blo = lb(b), bhi = lb(b + 1);
    const bool valid = b == 0 ? p == 0 : p < blo - lb(b - 1);
    const int64_t ap = b == 0 ? 0 : lb(b - 1) + p;
    unsigned char r = 0;
    if (valid) {
      const double ax = X(ap), ay = Y(ap);
      const double2 c = s_mean[b];
      long long best = -1;
      for (int64_t j = blo; j < bhi; ++j) {
        const long long ar = lttb_area_key(ax, ay, c.x, c.y, X(j), Y(j));
        if (ar > best) { best = ar; r = (unsigned char)(j - blo); }
      }
    }
    s_tab[it] = r;
  }
  __syncthreads();
  int64_t* out = a.out + s * a.n_out;
  scan_chain<SMAX, NT, 4>(s_tab, k3, [&](int64_t b, int sel) { out[b + 1] = __ldcg(pre + lb(b) + sel); });
  if (threadIdx.x == 0) {
    out[0] = 0;
    out[k3 + 1] = N - 1;
  }
}

// Same as k_post_fused with the preselected set staged in SHARED memory
// (positions, x and y as f64): the LTTB phases then make no global round
// trips -- one L2 gather of x in the compaction, everything else on chip.
__host__ __device__ inline int64_t post_smem2(int64_t k3, int smax, int64_t cap) {
  return k3 * 16 + ((k3 * smax + 15) / 16) * 16 + cap * 24;
}

template <typename XT, typename YT, int SMAX, int NT>
__global__ void __launch_bounds__(NT) k_post_smem(PostArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int sh[NT / 32 + 1];
  const int64_t s = blockIdx.x;
  const int64_t k = a.k, N = a.N, k3 = a.n_out - 2;
  const Ext* ext = a.ext + s * k;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  double2* s_mean = reinterpret_cast<double2*>(sm);
  unsigned char* s_tab = sm + k3 * 16;
  double* s_px = reinterpret_cast<double*>(sm + k3 * 16 + ((k3 * SMAX + 15) / 16) * 16);
  double* s_py = s_px + a.cap;
  long long* s_pre = reinterpret_cast<long long*>(s_py + a.cap);
  const int ydt = sizeof(YT) == 4 ? 0 : 1;
  // ---- compaction: [0] + (lo, hi)... + [N-1]  (downsamplers.py:60-69, 157-160)
  // k <= 2 * NT on this path (post_ok): both rounds' Ext loads, then both rounds'
  // x gathers, are issued before any is consumed (two memory round trips in all)
  static_assert(NT >= 1024, "post_ok bounds k by 2048");
  int n[2];
  int64_t lo[2], hi[2];
  long long klo[2], khi[2];
  double xl[2], xh[2];
  Ext e[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int64_t b = (int64_t)r * NT + threadIdx.x;
    if (b < k) e[r] = ext[b];
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int64_t b = (int64_t)r * NT + threadIdx.x;
    n[r] = 0; lo[r] = hi[r] = 0; klo[r] = khi[r] = 0; xl[r] = xh[r] = 0.0;
    if (b < k) {
      if (a.status && keys_nonfinite(e[r].kmin, e[r].kmax, ydt)) atomicOr(a.status, 1);
      const bool mfirst = e[r].imin <= e[r].imax;
      lo[r] = mfirst ? e[r].imin : e[r].imax;
      hi[r] = mfirst ? e[r].imax : e[r].imin;
      klo[r] = mfirst ? e[r].kmin : e[r].kmax;
      khi[r] = mfirst ? e[r].kmax : e[r].kmin;
      n[r] = hi[r] != lo[r] ? 2 : 1;
      xl[r] = to_f64(xs, lo[r]);  // gathers in flight across the scans
      if (n[r] == 2) xh[r] = to_f64(xs, hi[r]);
    }
  }
  int64_t carry = 1;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if ((int64_t)r * NT >= k) break;  // uniform
    int tot;
    const int ex = block_excl_scan<NT>(n[r], tot, sh);
    if ((int64_t)r * NT + threadIdx.x < k) {
      const int64_t p = carry + ex;
      s_pre[p] = lo[r]; s_px[p] = xl[r]; s_py[p] = key_value<YT>(klo[r]);
      if (n[r] == 2) { s_pre[p + 1] = hi[r]; s_px[p + 1] = xh[r]; s_py[p + 1] = key_value<YT>(khi[r]); }
    }
    carry += tot;
  }
  if (threadIdx.x == 0) {
    const double y0 = to_f64(ys, 0), yl = to_f64(ys, N - 1);
    if (a.status && (!isfinite(y0) || !isfinite(yl))) atomicOr(a.status, 1);
    s_pre[0] = 0; s_px[0] = to_f64(xs, 0); s_py[0] = y0;
    s_pre[carry] = N - 1; s_px[carry] = to_f64(xs, N - 1); s_py[carry] = yl;
  }
  const int64_t m = carry + 1;
  __syncthreads();
  // b * (m - 2) < 2^32 (m <= 2k + 2 and k is small on this path)
  const unsigned um = (unsigned)(m - 2), uk3 = (unsigned)k3;
  auto lb = [&](int64_t b) -> int64_t { return 1 + (int64_t)(((unsigned)b * um) / uk3); };
  // ---- LTTB over the m points (_kernels.py:81-119): means, tables, chain
  for (int64_t b = threadIdx.x; b < k3; b += NT) {
    double2 c;
    if (b + 1 < k3) {
      const int64_t nlo = lb(b + 1), nhi = lb(b + 2);
      double sx = 0.0, sy = 0.0;
      for (int64_t j = nlo; j < nhi; ++j) {
        sx = __dadd_rn(sx, s_px[j]);
        sy = __dadd_rn(sy, s_py[j]);
      }
      const double cnt = (double)(nhi - nlo);
      c = make_double2(__ddiv_rn(sx, cnt), __ddiv_rn(sy, cnt));
    } else {
      c = make_double2(s_px[m - 1], s_py[m - 1]);
    }
    s_mean[b] = c;
  }
  __syncthreads();
  for (int64_t it = threadIdx.x; it < k3 * SMAX; it += NT) {
    const int64_t b = it / SMAX;
    const int p = (int)(it % SMAX);
    const int64_t blo = lb(b), bhi = lb(b + 1);
    const bool valid = b == 0 ? p == 0 : p < blo - lb(b - 1);
    const int64_t ap = b == 0 ? 0 : lb(b - 1) + p;
    unsigned char r = 0;
    if (valid) {
      const double ax = s_px[ap], ay = s_py[ap];
      const double2 c = s_mean[b];
      long long best = -1;
      for (int64_t j = blo; j < bhi; ++j) {
        const long long ar = lttb_area_key(ax, ay, c.x, c.y, s_px[j], s_py[j]);
        if (ar > best) { best = ar; r = (unsigned char)(j - blo); }
      }
    }
    s_tab[it] = r;
  }
  __syncthreads();
  int64_t* out = a.out + s * a.n_out;
  scan_chain<SMAX, NT, 4>(s_tab, k3, [&](int64_t b, int sel) { out[b + 1] = s_pre[lb(b) + sel]; });
  if (threadIdx.x == 0) {
    out[0] = 0;
    out[k3 + 1] = N - 1;
  }
}

}  // namespace mm
