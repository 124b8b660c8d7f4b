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
__host__ __device__ inline int64_t fused_smem(int64_t k, int64_t k3, int smax, int ysize) {
  const int64_t m = 2 * k + 2;
  return fused_region1(k, k3, smax, ysize) + ((m * ysize + 15) / 16) * 16 + ((m * 4 + 15) / 16) * 16;
}

template <typename XT, typename YT, int SMAX, int NT, int MINB, int U>
__global__ void __launch_bounds__(NT, MINB) k_mmlttb_fused(FusedArgs a) {
  typedef YTr<YT> Tr;
  typedef typename Tr::K K;
  typedef PMap<SMAX> M;
  constexpr int G = 8, NG = NT / G;
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int sh_scan[NT / 32 + 1];
  __shared__ M s_warp[NT / 32];
  __shared__ M s_carry;

  const int64_t s = blockIdx.x;
  const int64_t N = a.N;
  const int64_t k = (a.n_out - 2) * (a.r_ps / 2);
  const int64_t L = N - 2;
  const int64_t mcap = 2 * k + 2;
  const YT* ys = (const YT*)a.y + s * a.y_ld;
  const XT* xs = (const XT*)a.x + s * a.x_ld;
  // phase-1 arrays: [k] y at lo, y at hi (storage type), lo, hi offsets
  YT* s_vlo = reinterpret_cast<YT*>(sm);
  YT* s_vhi = s_vlo + k;
  int* s_lo = reinterpret_cast<int*>(s_vhi + k);
  int* s_hi = s_lo + k;
  const int64_t a1 = fused_region1(k, a.n_out - 2, SMAX, (int)sizeof(YT));
  // phase-2 arrays: [mcap] preselected y (storage type) and positions
  YT* s_py = reinterpret_cast<YT*>(sm + a1);
  int* s_pre = reinterpret_cast<int*>(sm + a1 + ((mcap * (int64_t)sizeof(YT) + 15) / 16) * 16);
  // phase-3 aliases over the (dead) phase-1 region
  double2* s_mean = reinterpret_cast<double2*>(sm);                     // [k3]: 16*k3 <= 16*k
  unsigned char* s_tab = reinterpret_cast<unsigned char*>(s_mean + k3_of(a.n_out));  // [k3 * SMAX] after the means

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
    group_extrema<YT, U, 3, G>(ys, lo, hi, lane8, mn, omn, mx, omx);
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
  // ---- phase 2: compaction (block scan over the k counts) ----
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
  auto lb = [&](int64_t b) -> int64_t { return 1 + (b * (m - 2)) / k3; };
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
      double best = -1.0;
      for (int64_t j = blo; j < bhi; ++j) {
        const double ar = lttb_area(ax, ay, c.x, c.y, px(j), (double)s_py[j]);
        if (ar > best) { best = ar; r = (unsigned char)(j - blo); }
      }
    }
    s_tab[it] = r;
  }
  __syncthreads();
  // chain: block scan of the packed maps (as k_lttb_scan), one map per thread
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t* out = a.out + s * a.n_out;
  M cm = M::ident();
  for (int64_t c0 = 0; c0 < k3; c0 += NT) {
    const int64_t b = c0 + threadIdx.x;
    const M t = b < k3 ? M::load(s_tab + b * SMAX) : M::ident();
    M inc = t;
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
    M pre = cm;
    if (wid > 0) pre = M::comp(s_warp[wid - 1], pre);
    const M lane_prev = inc.shfl_up(1);
    if (lane > 0) pre = M::comp(lane_prev, pre);
    const M cur = M::comp(t, pre);
    if (b < k3) out[b + 1] = s_pre[lb(b) + cur.at0()];
    if (threadIdx.x == NT - 1) s_carry = cur;
    __syncthreads();
    cm = s_carry;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = 0;
    out[k3 + 1] = N - 1;
  }
}

}  // namespace mm
