// k3s.cuh -- K3s: exact full LTTB of ONE series with many large buckets
// (BASELINE C2: 1,998 buckets of ~5,005 points) in a SINGLE persistent launch.
//
// Same algorithm and exactness argument as K3c (kernels.cuh: direction
// candidates -> candidate transition tables -> chain -> exact verification
// -> repair), re-organised as one cooperative kernel (one CTA per SM, all
// co-resident).  CTA c owns the contiguous buckets [B0, B1); inside a phase a
// WARP owns a whole bucket, so every reduction is a warp reduction amortised
// over ~150 points per lane and no phase needs more than one pass:
//
//   1 stats   per bucket: any-order sums with rigorous error bounds, x / y
//             ranges, the affine-x test ("certified means") --
//             the only pass that reads HBM (x and y once)            | grid sync
//   2 cand    per bucket: argmax / argmin of Y + lambda*T for D slopes sampled
//             over the anchor box (bucket b-1's ranges) and the mean c_b;
//             points in octets, winners resolved by 16 lanes in parallel | grid sync
//   3 chain   transition tables T_b over the candidate sets (exact areas),
//             CTA aggregate A_c = T_{B1-1} o ... o T_{B0} (16-byte maps), the
//             chain entering CTA c = (A_{c-1} o ... o A_0)(0), then positions
//   4 verify  every bucket re-scanned with the reference's formula, tie rule
//             and (certified) mean given the chain's previous pick; a
//             mismatching bucket's successor gets its exact pick given the
//             exact anchor (verify2)
//   5 repair  the last CTA to finish walks the mismatches (repair_walk_smem)
//             and writes the n_out indices.
//
// The candidate heuristic never affects the result: every bucket is verified
// exactly and every deviation repaired (_kernels.py:81-119 semantics).
#pragma once
#include "kernels.cuh"
#include <type_traits>

namespace mm {

constexpr int K3S_NT = 512;          // 16 warps per CTA
constexpr int K3S_NW = K3S_NT / 32;
#ifndef K3S_DIRS
#define K3S_DIRS 16
#endif
// sampled slopes -> <= 2D candidates per bucket (2D <= 32).  Measured on C2
// (1,998 buckets): 8 slopes leave ~5 buckets per call whose pick is outside
// the candidate set (each costing a whole-CTA walk step after the
// verification), 12 leave ~2, 16 leave none (117 vs 124 us per call); two
// clusters of slopes at the anchor box's y edges instead of an even spread
// are worse (6 misses with 8 or 12)
constexpr int K3S_D = K3S_DIRS;
constexpr int K3S_H = K3S_D <= 8 ? 16 : 32;  // candidate slots per bucket (table width: 16 or 32)
constexpr int K3S_U = 8;             // loads in flight per lane per array
constexpr int K3S_GMAX = 1024;       // CTA bound for the workspace
// Group summaries (round 2, "pruned" phases 2 and 4a): phase 1 also publishes the
// y range of every GROUP of a bucket -- 2^s consecutive warp-wide 16-byte vector
// loads (64 f64 / 128 f32 points for s = 0; s grows so that a bucket has at most
// K3S_GCAP groups).  The candidate search and the verification then bound each
// group's best value from its (y range) x (index range) box and only scan the
// few groups that can matter: on C2 ~5 of 79 groups per bucket for the
// candidates and ~1.1 for the verification (a random walk without spikes: 5.1 / 1.14).
constexpr int K3S_GCAP = 128;
// K3s never runs beyond this many buckets (its repair state must fit shared memory:
// 28 bytes per bucket), so the group summaries are not carved for larger calls
constexpr int64_t K3S_K3MAX = 16384;
// buckets of fewer groups are scanned whole: bounding 12 groups costs what scanning
// them does (6e6 f32 points / n_out 4000, 1,500-point buckets: 122 vs 114 us)
constexpr int K3S_PRUNE_MIN_GROUPS = 24;

struct K3sArgs {
  int G;                 // CTAs, all co-resident (cooperative launch)
  int maxb;              // >= buckets per CTA
  unsigned* sync;        // K3S_SYNC_WORDS counters / flags (zeroed per call); fcount at K3S_FCOUNT
  unsigned char* agg;    // [G][16] aggregate maps
  double2* cpt;          // [k3][16] candidate points (x, y)
  unsigned long long* prof;  // optional [G][8] %globaltimer stamps per phase (tools), or null
  int2* gmeta;           // [k3][K3S_GCAP] per-group (min, max) y keys written by phase 1, or null (no pruning)
  int* chg;              // [k3] re-verification pass in which a bucket's anchor last changed (phase 4j)
  int jmin, jmax;        // phase 4j runs while more than jmin buckets are flagged, for at most jmax passes
};
// sync words: barrier i = counter at 64 i, release flag at 64 i + 32 (separate
// 128-byte lines: the pollers never delay the arrivals); done counter, fcount
constexpr int K3S_DONE = 64 * 4, K3S_FCOUNT = 64 * 4 + 32, K3S_CONFLICT = 64 * 5;
// per-CTA "statistics published" / "candidates published" flags (neighbours wait on them)
constexpr int K3S_FLAGS = 64 * 6, K3S_SYNC_WORDS = 64 * 6 + 2 * K3S_GMAX;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// bounded spin: a protocol bug traps (the launch fails) instead of hanging the GPU
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}
__device__ __forceinline__ void spin_until_set(const unsigned* p, unsigned want) {
  const unsigned long long t0 = gtimer();
  while (ld_acq(p) < want) {
    __nanosleep(32);
    if (gtimer() - t0 > 2000000000ull) __trap();  // 2 s
  }
}
// grid-wide barrier i over the G co-resident CTAs: a release add on the
// counter, then acquire polls of the counter itself (tight; the watchdog clock
// is read every 1,024 polls).  A/B: MMLTTB_BARRIER_FLAG (host) selects the
// earlier variant (last arriver releases a flag on another line).
__device__ __forceinline__ void k3s_grid_sync(unsigned* sync, int i, unsigned G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* ctr = sync + 64 * i;
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    unsigned long long t0 = 0;
    for (unsigned it = 1; ld_acq(ctr) < G; ++it) {
      if ((it & 1023u) == 0) {
        const unsigned long long t = gtimer();
        if (t0 == 0) t0 = t;
        else if (t - t0 > 2000000000ull) __trap();  // 2 s
      }
    }
  }
  __syncthreads();
}

// tool counters (prof mode): [0] verify calls, [1] violations, [2] shared high word, [3] cert fails,
// [4] full-path picks, [5] flagged buckets, [6] 4b picks, [7] repair picks, [8] pruned candidate searches,
// [9] their surviving groups, [10] plain candidate searches, [11] pruned verifications, [12] their
// surviving groups, [13] plain verifications (one warp)
// Compiled in only with -DK3S_PROF (tools; MMLTTB_NVCC_EXTRA): each call reads a
// global pointer the warp then branches on, i.e. an exposed load on the
// latency-bound phases (the phase stamps of `ka.prof` stay: a constant-bank test).
#ifdef K3S_PROF
__device__ unsigned long long* g_k3s_cnt;
__device__ __forceinline__ void k3s_count(int i) {
  if (g_k3s_cnt && (threadIdx.x & 31) == 0 && ((threadIdx.x >> 5) == 0 || i < 0)) atomicAdd(g_k3s_cnt + (i < 0 ? -i : i), 1ull);
}
// tool timeline of one warp (CTA 70, warp 0): slots 32..63
__device__ __forceinline__ void k3s_dbg(int i) {
  if (g_k3s_cnt && blockIdx.x == 70 && threadIdx.x == 0) g_k3s_cnt[32 + i] = gtimer();
}
__device__ __forceinline__ void k3s_cnt_add(int i, int v) {  // (every warp's lane 0)
  if (g_k3s_cnt && (threadIdx.x & 31) == 0) atomicAdd(g_k3s_cnt + i, (unsigned long long)v);
}
#else
__device__ __forceinline__ void k3s_count(int) {}
__device__ __forceinline__ void k3s_dbg(int) {}
__device__ __forceinline__ void k3s_cnt_add(int, int) {}
#endif

// -DK3S_CHECKED (tools/k3s_check.py under a checked build; compute-sanitizer is
// closed on the GPU pool): every index into the round-2 arrays (group
// summaries, survivor lists, the staging buffer, the re-verification stamps)
// and every vector the pruned phases load is range-checked; a violation traps
// (the launch fails).  Compiled out by default.
#ifdef K3S_CHECKED
#define K3S_ASSERT(c) do { if (!(c)) __trap(); } while (0)
#else
#define K3S_ASSERT(c) do { } while (0)
#endif

// reusable grid barrier: the n-th use of counter i waits for n G arrivals
__device__ __forceinline__ void k3s_grid_sync_n(unsigned* sync, int i, unsigned G, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* ctr = sync + 64 * i;
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    unsigned long long t0 = 0;
    for (unsigned it = 1; ld_acq(ctr) < G * n; ++it) {
      if ((it & 1023u) == 0) {
        const unsigned long long t = gtimer();
        if (t0 == 0) t0 = t;
        else if (t - t0 > 2000000000ull) __trap();  // 2 s
      }
    }
  }
  __syncthreads();
}

// float -> int32 key with the same order (IEEE total order)
__device__ __forceinline__ int fkey(float f) {
  const int b = __float_as_int(f);
  return b ^ ((b >> 31) & 0x7fffffff);
}

// sum_{i<n} (x0 + i d) in 128-bit integer arithmetic, rounded once to f64
// (exact whenever the result is below 2^53)
__device__ __forceinline__ double k3s_affine_sum(long long x0, long long d, long long n) {
  const long long tt = n * (n - 1) / 2;
  const unsigned long long lo1 = (unsigned long long)x0 * (unsigned long long)n;
  const long long hi1 = __mul64hi(x0, n);
  const unsigned long long lo2 = (unsigned long long)d * (unsigned long long)tt;
  const long long hi2 = __mul64hi(d, tt);
  const unsigned long long lo = lo1 + lo2;
  const long long hi = hi1 + hi2 + (lo < lo1 ? 1 : 0);
  if (hi == ((long long)lo >> 63)) return (double)(long long)lo;  // fits int64: one rounding
  return __dadd_rn(__dmul_rn((double)hi, 18446744073709551616.0), (double)lo);
}

__device__ __forceinline__ double warp_dsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// ---- 16-byte vector windows --------------------------------------------
// Bucket [lo, hi) of a 16-byte-aligned array of T: full vectors [vf, vl) are
// loaded as uint4 (EV elements each, lane-strided: coalesced 512 B per warp
// load), the < EV head elements [lo, vf*EV) and tail elements [vl*EV, hi)
// individually.
template <typename T> struct Vec {
  static constexpr int EV = 16 / (int)sizeof(T);
  __device__ __forceinline__ static T get(const uint4& v, int e) {
    if constexpr (sizeof(T) == 8) {
      const unsigned long long b = e == 0 ? ((unsigned long long)v.y << 32 | v.x) : ((unsigned long long)v.w << 32 | v.z);
      if constexpr (std::is_same<T, double>::value) return __longlong_as_double((long long)b);
      else return (T)(long long)b;
    } else {
      const unsigned b = e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
      if constexpr (std::is_same<T, float>::value) return __uint_as_float(b);
      else return (T)(int)b;
    }
  }
};
struct VWin {
  int64_t vf, vl;  // full vectors
  int nh, nt;      // head / tail element counts
  int64_t tl;      // first tail element
};
template <typename T>
__device__ __forceinline__ VWin vwin(int64_t lo, int64_t hi) {
  constexpr int EV = Vec<T>::EV;
  VWin w;
  w.vf = (lo + EV - 1) / EV;
  w.vl = hi / EV;
  if (w.vl < w.vf) w.vl = w.vf;
  w.nh = (int)(min(hi, w.vf * EV) - lo);
  w.tl = max(lo, w.vl * EV);
  w.nt = (int)(hi - w.tl);
  if (w.vf * EV >= hi) w.nt = 0;  // no full vector: the head covers everything
  return w;
}
// group geometry of a window: nl warp-loads (32 vectors each), 2^s warp-loads per group, ng groups
struct GGeo { int s, ng; int64_t nl; };
__device__ __forceinline__ GGeo ggeo(const VWin& w) {
  GGeo g;
  g.nl = (w.vl - w.vf + 31) >> 5;
  g.s = 0;
  while (((g.nl + (1LL << g.s) - 1) >> g.s) > K3S_GCAP) ++g.s;
  g.ng = (int)((g.nl + (1LL << g.s) - 1) >> g.s);
  return g;
}
// element index handled by `lane` in the head / tail step (or -1)
__device__ __forceinline__ int64_t vwin_edge(const VWin& w, int64_t lo, int lane) {
  if (lane < w.nh) return lo + lane;
  if (lane >= 16 && lane - 16 < w.nt) return w.tl + (lane - 16);
  return -1;
}

// Lane-strided rounds over a window's full vectors: body(r, v0, cnt, g) gets
// this lane's UV vectors of round g (r[u] = vector v0 + 32u) of which the
// first cnt are in range (cnt == UV in every round but the last, which the
// compiler specialises; out-of-range slots repeat vector v0).
// ALLTAIL: every lane runs the body of the last (partial) round, with cnt = 0
// where it has no vector left (bodies with warp-wide operations).
struct NoMid { __device__ __forceinline__ void operator()() const {} };
template <int UV, bool STREAM, bool PREFETCH, bool ALLTAIL = false, typename F, typename MID = NoMid>
__device__ __forceinline__ void vrounds(const uint4* base, const VWin& w, int L, int NL, F&& body, MID&& mid = NoMid{}) {
  const int64_t nfull = (w.vl - w.vf) / ((int64_t)NL * UV);
  int64_t v0 = w.vf + L;
  const uint4* p = base + v0;
  const int step = NL * UV;
  auto ld = [&](uint4 (&r)[UV], const uint4* q) {
#pragma unroll
    for (int u = 0; u < UV; ++u) r[u] = STREAM ? __ldcs(q + NL * u) : q[NL * u];  // immediate offsets
  };
  int g = 0;
  if constexpr (!PREFETCH) {
    for (; g < nfull; ++g, v0 += step, p += step) {
      uint4 r[UV];
      ld(r, p);
      mid();  // (work that overlaps the loads' latency)
      body(r, v0, UV, g);
    }
  } else {
    // software-pipelined: round g+1's loads are in flight while round g is processed
    uint4 ra[UV], rb[UV];
    if (nfull > 0) ld(ra, p);
    for (; g + 1 < nfull; g += 2) {
      ld(rb, p + step);
      body(ra, v0, UV, g);
      if (g + 2 < nfull) ld(ra, p + 2 * step);
      body(rb, v0 + step, UV, g + 1);
      v0 += 2 * step;
      p += 2 * step;
    }
    if (g < nfull) {
      body(ra, v0, UV, g);
      ++g;
      v0 += step;
      p += step;
    }
  }
  if (ALLTAIL ? (v0 - L < w.vl) : (v0 < w.vl)) {
    const int cnt = v0 < w.vl ? (int)((w.vl - v0 + NL - 1) / NL) : 0;
    if (ALLTAIL && cnt == 0) p = base + w.vf;  // (a valid address; the values are not used)
    uint4 r[UV];
#pragma unroll
    for (int u = 0; u < UV; ++u) r[u] = STREAM ? __ldcs(p + (u < cnt ? NL * u : 0)) : p[u < cnt ? NL * u : 0];
    mid();
    body(r, v0, cnt, g);
  }
}

// ---------------------------------------------------------------- phase 1 --
// One warp: statistics of bucket b = [lo, hi), published for every later phase.
template <typename XT, typename YT>
__device__ __forceinline__ void k3s_stats(const LttbArgs& a, const XT* xs, const YT* ys, int64_t b, int64_t lo,
                                          int64_t hi, int64_t m, int2* gm) {
  constexpr int EY = Vec<YT>::EV, EX = Vec<XT>::EV;
  // elements per lane per round: the same for x and y (they finish together), 8 vectors of the wider type
  constexpr int EPR = 8 * (EX < EY ? EX : EY), UY = EPR / EY;
  const int lane = threadIdx.x & 31;
  const int64_t k3 = a.n_out - 2;
  const int n = (int)(hi - lo);
  const double nb = (double)n;
  XAff f;
  {
    const XT x0r = xs[lo], x1r = n > 1 ? xs[lo + 1] : xs[lo];
    f.x0 = (double)x0r;
    f.d = __dsub_rn((double)x1r, (double)x0r);
    f.x0i = (long long)x0r;
    f.di = (long long)((unsigned long long)(long long)x1r - (unsigned long long)(long long)x0r);
    f.pad = 0;
  }
  const double yfirst = (double)ys[lo];
  const bool try_y = yfirst == 0.0 || (double)lsb_exp(yfirst) + 55.0 > (double)exp_of(yfirst) + log2(nb);
  const double xfirst = (double)xs[lo];
  const bool try_x = !XForm<XT>::integral && (xfirst == 0.0 || (double)lsb_exp(xfirst) + 55.0 > (double)exp_of(xfirst) + log2(nb));
  // ---- y: any-order sum, range keys (f32: exact; f64: high words, conservative), lowest set bit
  double sy = 0.0;
  int kmn = INT_MAX, kmx = INT_MIN, ly = 4096;
  auto ykey = [&](YT y) -> int {
    if constexpr (sizeof(YT) == 4) return fkey((float)y);
    else {
      const int hy = (int)(__double_as_longlong((double)y) >> 32);
      return hy ^ ((hy >> 31) & 0x7fffffff);
    }
  };
  // ---- x: affine test (integral: XOR-accumulated difference from the formula),
  // float x: bit compare + sum, keys, lowest bits
  double sx = 0.0;
  int lx = XForm<XT>::integral ? 0 : 4096, aff = 1;
  long long kxm = LLONG_MAX, kxM = LLONG_MIN;
  unsigned long long dacc = 0;  // integral x: OR of (x ^ formula) over the bucket
  auto xel = [&](XT x, long long xe) {  // xe: integral: the formula's value here; float: the offset j - lo
    if constexpr (XForm<XT>::integral) {
      dacc |= (unsigned long long)((long long)x ^ xe);
    } else {
      const double vx = (double)x;
      aff &= __double_as_longlong(vx) == __double_as_longlong(XForm<XT>::at(f, xe));
      sx = __dadd_rn(sx, vx);
      const long long kk = dkey(vx);
      kxm = min(kxm, kk);
      kxM = max(kxM, kk);
      if (try_x) lx = min(lx, lsb_exp(vx));
    }
  };
  auto xexp = [&](int64_t j) -> long long {
    if constexpr (XForm<XT>::integral) return (long long)((unsigned long long)f.x0i + (unsigned long long)(j - lo) * (unsigned long long)f.di);
    else return (long long)(j - lo);
  };
  const long long xstep = XForm<XT>::integral ? f.di : 1;
  // One merged loop streams y and x: a round's 8 + 8 vector loads per lane are
  // issued together (the pass is bound by rounds x DRAM latency, not by issue).
  // The y loads use a QUAD mapping: in a round of 32 UY vectors, the LS = 32 / UY
  // lanes of set bi = lane / LS load the 32 consecutive vectors of block bi
  // (instruction u: vector 4u + lane % 4 of the lane's 4 UY-vector quad --
  // 64 contiguous bytes per 4 lanes, whole sectors), so a block's (min, max) keys
  // are a lane-local reduction plus log2(LS) shuffle steps per round: the
  // group summaries (2^s blocks per group) cost no warp-wide reduction per load.
  const VWin wy = vwin<YT>(lo, hi);
  const GGeo gg = ggeo(wy);
  {
    const int64_t e = vwin_edge(wy, lo, lane);
    if (e >= 0) {
      const YT y = ys[e];
      sy = __dadd_rn(sy, (double)y);
      const int k = ykey(y);
      kmn = min(kmn, k);
      kmx = max(kmx, k);
      if (try_y) ly = min(ly, lsb_exp((double)y));
    }
    constexpr int LS = 32 / UY;              // lanes per block: 4 (f64) / 8 (f32)
    constexpr int LGU = UY == 8 ? 3 : 2;     // log2(UY)
    const uint4* yv = reinterpret_cast<const uint4*>(ys);
    const int64_t voff = (int64_t)(lane >> 2) * (4 * UY) + (lane & 3);
    int amn = INT_MAX, amx = INT_MIN;        // groups spanning rounds (s > LGU)
    constexpr int UXR = EPR / EX;            // x: lane-strided vectors per lane per round (evict-first)
    const VWin wx = vwin<XT>(lo, hi);
    const uint4* xv = reinterpret_cast<const uint4*>(xs);
    {
      const int64_t ex = vwin_edge(wx, lo, lane);
      if (ex >= 0) xel(xs[ex], xexp(ex));
    }
    const long long vstep = (long long)((unsigned long long)xstep * (unsigned long long)(32 * EX));
    auto run = [&](auto lsb_tag) {
      constexpr bool LSB = decltype(lsb_tag)::value;
      const int nry = (int)((wy.vl - wy.vf + 32 * UY - 1) / (32 * UY)), nrx = (int)((wx.vl - wx.vf + 32 * UXR - 1) / (32 * UXR));
      for (int g = 0; g < max(nry, nrx); ++g) {  // (warp-uniform)
        const int64_t vr = wy.vf + (int64_t)g * (32 * UY), v0 = vr + voff;
        const int64_t x0v = wx.vf + (int64_t)g * (32 * UXR) + lane;
        uint4 r[UY], rx[UXR];
        const bool full = vr + 32 * UY <= wy.vl, fullx = x0v - lane + 32 * UXR <= wx.vl;
        if (full) {
#pragma unroll
          for (int u = 0; u < UY; ++u) r[u] = yv[v0 + 4 * u];
        } else if (g < nry) {
#pragma unroll
          for (int u = 0; u < UY; ++u) r[u] = v0 + 4 * u < wy.vl ? yv[v0 + 4 * u] : make_uint4(0, 0, 0, 0);
        }
        if (fullx) {
#pragma unroll
          for (int u = 0; u < UXR; ++u) rx[u] = __ldcs(xv + x0v + 32 * u);
        } else if (g < nrx) {
#pragma unroll
          for (int u = 0; u < UXR; ++u) rx[u] = x0v + 32 * u < wx.vl ? __ldcs(xv + x0v + 32 * u) : make_uint4(0, 0, 0, 0);
        }
        if (g < nrx) {
          long long xe = xexp(x0v * EX);
#pragma unroll
          for (int u = 0; u < UXR; ++u) {
            if (fullx || x0v + 32 * u < wx.vl) {
#pragma unroll
              for (int q = 0; q < EX; ++q)
                xel(Vec<XT>::get(rx[u], q), (long long)((unsigned long long)xe + (unsigned long long)(q * xstep)));
            }
            xe = (long long)((unsigned long long)xe + (unsigned long long)vstep);
          }
        }
        if (g >= nry) continue;
        int vmn = INT_MAX, vmx = INT_MIN;
#pragma unroll
        for (int u = 0; u < UY; ++u) {
          if (full || v0 + 4 * u < wy.vl) {
#pragma unroll
            for (int q = 0; q < EY; ++q) {
              const YT y = Vec<YT>::get(r[u], q);
              sy = __dadd_rn(sy, (double)y);
              const int k = ykey(y);
              vmn = min(vmn, k);
              vmx = max(vmx, k);
              if (LSB) ly = min(ly, lsb_exp((double)y));
            }
          }
        }
        kmn = min(kmn, vmn);
        kmx = max(kmx, vmx);
        if (gm) {
          // block (LS lanes), then the group's 2^s blocks (or the whole round)
          const int steps = 5 - LGU + min(gg.s, LGU);  // shuffle steps: 1 << i, i < steps
#pragma unroll
          for (int i = 0; i < 5; ++i) {
            if (i < steps) {
              vmn = min(vmn, __shfl_xor_sync(FULL, vmn, 1 << i));
              vmx = max(vmx, __shfl_xor_sync(FULL, vmx, 1 << i));
            }
          }
          if (gg.s <= LGU) {
            const int gi = (int)(((int64_t)g * UY + lane / LS) >> gg.s);
            K3S_ASSERT(gg.ng <= K3S_GCAP);
            if ((lane & ((LS << gg.s) - 1)) == 0 && gi < gg.ng) gm[gi] = make_int2(vmn, vmx);
          } else {
            amn = min(amn, vmn);
            amx = max(amx, vmx);
            const int64_t nblk = (int64_t)(g + 1) * UY;  // blocks so far
            if ((nblk & ((1LL << gg.s) - 1)) == 0 || vr + 32 * UY >= wy.vl) {
              K3S_ASSERT(((nblk - 1) >> gg.s) < gg.ng && gg.ng <= K3S_GCAP);
              if (lane == 0) gm[(int)((nblk - 1) >> gg.s)] = make_int2(amn, amx);
              amn = INT_MAX; amx = INT_MIN;
            }
          }
        }
      }
    };
    if (try_y) run(std::true_type{});
    else run(std::false_type{});
  }
  if constexpr (XForm<XT>::integral) aff = dacc == 0;
  aff = __all_sync(FULL, aff);
  f.ok = aff;
  sy = warp_dsum(sy);
  kmn = __reduce_min_sync(FULL, kmn);
  kmx = __reduce_max_sync(FULL, kmx);
  ly = __reduce_min_sync(FULL, try_y ? ly : -4096);
  double x0, x1, Ax;
  if (XForm<XT>::integral && aff) {  // closed-form sum of the verified arange
    sx = k3s_affine_sum(f.x0i, f.di, n);
    const long long xl = (long long)((unsigned long long)f.x0i + (unsigned long long)(n - 1) * (unsigned long long)f.di);
    x0 = elem_f64((XT)f.x0i);
    x1 = elem_f64((XT)xl);
    if (x1 < x0) { const double tt = x0; x0 = x1; x1 = tt; }
    Ax = __dmul_rn(nb, fmax(fabs(x0), fabs(x1))) * (1.0 + 4.0 * K3C_U);
    lx = 0;
  } else {
    if constexpr (XForm<XT>::integral) {  // (rare) non-affine integer x: second pass
      for (int64_t j = lo + lane; j < hi; j += 32) {
        const double vx = elem_f64(xs[j]);
        sx = __dadd_rn(sx, vx);
        const long long kk = dkey(vx);
        kxm = min(kxm, kk);
        kxM = max(kxM, kk);
      }
    }
    sx = warp_dsum(sx);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      kxm = min(kxm, __shfl_xor_sync(FULL, kxm, o));
      kxM = max(kxM, __shfl_xor_sync(FULL, kxM, o));
    }
    lx = __reduce_min_sync(FULL, XForm<XT>::integral ? 0 : (try_x ? lx : -4096));
    x0 = dkey_inv(kxm);
    x1 = dkey_inv(kxM);
    Ax = __dmul_rn(nb, fmax(fabs(x0), fabs(x1))) * (1.0 + 4.0 * K3C_U);
  }
  if (lane == 0) {
    double y0, y1;
    if constexpr (sizeof(YT) == 4) {
      y0 = (double)__int_as_float(kmn ^ ((kmn >> 31) & 0x7fffffff));
      y1 = (double)__int_as_float(kmx ^ ((kmx >> 31) & 0x7fffffff));
    } else {
      y0 = dkey_inv((long long)kmn * 4294967296LL);                 // <= every value
      y1 = dkey_inv((long long)kmx * 4294967296LL + 4294967295LL);  // >= every value
    }
    const double Ay = __dmul_rn(nb, fmax(fabs(y0), fabs(y1))) * (1.0 + 4.0 * K3C_U);
    a.yrange[b] = make_double2(y0, y1);
    a.xrange[b] = make_double2(x0, x1);
    if (a.xaff) a.xaff[b] = f;
    if (b >= 1) {
      double ex = mean_err_bound(sx, Ax, lx, nb), ey = mean_err_bound(sy, Ay, ly, nb);
      if (!(Ay <= 1.7e308)) ey = INFINITY;  // non-finite y: never certified (the exact path decides)
      if (!(Ax <= 1.7e308)) ex = INFINITY;
      a.means[b - 1] = make_double2(__ddiv_rn(sx, nb), __ddiv_rn(sy, nb));
      a.merr[b - 1] = make_double2(ex, ey);
    }
    if (b == k3 - 1) {  // the last bucket anchors on point m-1 itself (_kernels.py:105-107): exact
      a.means[k3 - 1] = make_double2(to_f64(xs, m - 1), to_f64(ys, m - 1));
      a.merr[k3 - 1] = make_double2(0.0, 0.0);
    }
  }
}

// (min, max) y keys of a group (phase 1) -> rigorous bounds y0 <= every y <= y1 of
// the group (f32: exact; f64: the high words' granules); NaN keys give NaN bounds
template <typename YT>
__device__ __forceinline__ void gkey_bounds(int2 k, double& y0, double& y1) {
  if constexpr (sizeof(YT) == 4) {
    y0 = (double)__int_as_float(k.x ^ ((k.x >> 31) & 0x7fffffff));
    y1 = (double)__int_as_float(k.y ^ ((k.y >> 31) & 0x7fffffff));
  } else {
    y0 = dkey_inv((long long)k.x * 4294967296LL);
    y1 = dkey_inv((long long)k.y * 4294967296LL + 4294967295LL);
  }
}
__device__ __forceinline__ int hw_abs(double v) { return (int)((__double_as_longlong(v) >> 32) & 0x7fffffff); }

// ---------------------------------------------------------------- phase 2 --
// winner lane + group of each of the 2D extremes (warp REDUX on order keys):
// lane e < 2D keeps extreme e's winner
__device__ __forceinline__ void k3s_winners(const float (&vmax)[K3S_D], const float (&vmin)[K3S_D], const int (&gmax)[K3S_D],
                                            const int (&gmin)[K3S_D], int& my_g, int& my_l, int& my_key) {
  constexpr int D = K3S_D;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int e = 0; e < 2 * D; ++e) {
    const int k = e >> 1;
    const int key = (e & 1) ? fkey(-vmin[k]) : fkey(vmax[k]);
    const int wk = __reduce_max_sync(FULL, key);
    const int wl = __ffs(__ballot_sync(FULL, key == wk)) - 1;
    const int wg = __shfl_sync(FULL, (e & 1) ? gmin[k] : gmax[k], wl);
    if (lane == e) { my_g = wg; my_l = wl; my_key = wk; }
  }
}

// lanes' resolved candidate positions `off` (or -1) -> bucket b's sorted,
// de-duplicated candidate set (positions + points)
template <typename XT, typename YT>
__device__ __forceinline__ void k3s_cand_finish(const LttbArgs& a, const K3sArgs& ka, const XT* xs, const YT* ys, int64_t b,
                                                int64_t lo, int64_t off) {
  constexpr int H = K3S_H;
  const int lane = threadIdx.x & 31;
  int o32 = off < 0 ? INT_MAX : (int)(off - lo);
  // sort the <= 2D offsets across the warp (bitonic), de-duplicate, cap
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int o = __shfl_xor_sync(FULL, o32, j);
      const bool up = ((lane & k) == 0);
      const bool lower = (lane & j) == 0;
      o32 = (lower == up) ? min(o32, o) : max(o32, o);
    }
  }
  const int prev = __shfl_up_sync(FULL, o32, 1);
  const bool keep = o32 != INT_MAX && (lane == 0 || prev != o32);
  const unsigned km = __ballot_sync(FULL, keep);
  const int rank = __popc(km & ((1u << lane) - 1));
  const int cap = a.cand_cap > 0 && a.cand_cap < H ? a.cand_cap : H;
  const int cw = max(1, min(__popc(km), cap));
  if (keep && rank < cap) {
    const int64_t p = lo + o32;
    a.cand[b * H + rank] = p;
    ka.cpt[b * H + rank] = make_double2(to_f64(xs, p), to_f64(ys, p));
  }
  if (lane == 0) {
    if (km == 0) { a.cand[b * H] = lo; ka.cpt[b * H] = make_double2(to_f64(xs, lo), to_f64(ys, lo)); }
    a.cand_cnt[b] = cw;
  }
}

// One warp: direction candidates of bucket b = [lo, hi).  D slopes lambda over
// the anchor box (bucket b-1's ranges, or point 0) and the mean c = means[b];
// per slope the argmax and argmin of Y + lambda*T (T: index offset for affine
// x, else x - x_lo) -- in f32, a heuristic (phase 4 makes the result exact).
// A lane's points of a round form one group: per slope the group's max / min
// (3-input min/max trees) meet the running extremes, which remember the
// round; afterwards 2D lanes resolve the 2D winning groups to their points in
// parallel, recomputing the same f32 values.  Affine x: with T = tb + c_p
// (tb the lane's round base, c_p a compile-time offset), a group's extreme is
// fmaf(lambda, tb, max_p fmaf(lambda, c_p, Y_p)) -- one FFMA per point and slope.
template <typename XT, typename YT, bool AFF>
__device__ __forceinline__ void k3s_cand_t(const LttbArgs& a, const K3sArgs& ka, const XT* xs, const YT* ys, int64_t b,
                                           int64_t lo, int64_t hi, const float (&lam)[K3S_D], double xlo) {
  constexpr int D = K3S_D, H = K3S_H;
  constexpr int PR = K3S_D >= 12 ? 8 : 16;  // points per lane per round
  constexpr int EV = Vec<YT>::EV, UV = PR / EV;
  const int lane = threadIdx.x & 31;
  auto tval = [&](int64_t j) -> float { return AFF ? (float)(j - lo) : (float)(elem_f64(xs[j]) - xlo); };
  float vmax[D], vmin[D];
  int gmax[D], gmin[D];
#pragma unroll
  for (int k = 0; k < D; ++k) { vmax[k] = -INFINITY; vmin[k] = INFINITY; gmax[k] = -1; gmin[k] = -1; }
  const VWin w = vwin<YT>(lo, hi);
  const uint4* yv = reinterpret_cast<const uint4*>(ys);
  int ng = 0;
  vrounds<UV, false, false>(yv, w, lane, 32, [&](const uint4 (&r)[UV], int64_t v0, int cnt, int g) {
    ng = g + 1;
    float Y[PR];
#pragma unroll
    for (int u = 0; u < UV; ++u)
#pragma unroll
      for (int q = 0; q < EV; ++q) Y[u * EV + q] = (float)Vec<YT>::get(r[u], q);
    float T[PR];
    if constexpr (!AFF) {
#pragma unroll
      for (int u = 0; u < UV; ++u)
#pragma unroll
        for (int q = 0; q < EV; ++q) T[u * EV + q] = tval((u < cnt ? v0 + 32 * u : v0) * EV + q);
    }
    const float tb = (float)(v0 * EV - lo);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float mx = -INFINITY, mn = INFINITY;
#pragma unroll
      for (int u = 0; u < UV; ++u) {
        if (u < cnt) {
#pragma unroll
          for (int q = 0; q < EV; ++q) {
            const float val = AFF ? fmaf(lam[k], (float)(32 * EV * u + q), Y[u * EV + q]) : fmaf(lam[k], T[u * EV + q], Y[u * EV + q]);
            mx = fmaxf(mx, val);
            mn = fminf(mn, val);
          }
        }
      }
      if (AFF) { mx = fmaf(lam[k], tb, mx); mn = fmaf(lam[k], tb, mn); }
      if (mx > vmax[k]) { vmax[k] = mx; gmax[k] = g; }
      if (mn < vmin[k]) { vmin[k] = mn; gmin[k] = g; }
    }
  });
  ng = __reduce_max_sync(FULL, ng);  // the head / tail group id (lanes without a partial round saw fewer)
  const int64_t ej = vwin_edge(w, lo, lane);
  if (ej >= 0) {  // head / tail elements: group ng
    const float Yj = (float)ys[ej], Tj = tval(ej);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float val = fmaf(lam[k], Tj, Yj);
      if (val > vmax[k]) { vmax[k] = val; gmax[k] = ng; }
      if (val < vmin[k]) { vmin[k] = val; gmin[k] = ng; }
    }
  }
  int my_g = -1, my_l = 0, my_key = 0;  // lane e < 2D keeps extreme e's winner
  k3s_winners(vmax, vmin, gmax, gmin, my_g, my_l, my_key);
  // lanes 0..2D-1 resolve their extreme's group to its first point (parallel re-reads)
  int64_t off = -1;
  if (lane < 2 * D && my_g >= 0) {
    const int k = lane >> 1;
    float lk = lam[0];
#pragma unroll
    for (int q = 1; q < D; ++q) lk = k == q ? lam[q] : lk;
    if (my_g == ng) {
      off = vwin_edge(w, lo, my_l);
    } else {
      const int64_t v0 = w.vf + (int64_t)my_g * 32 * UV + my_l;
      const int cnt = (int)min((int64_t)UV, (w.vl - v0 + 31) / 32);
      const float tb = (float)(v0 * EV - lo);
      uint4 r[UV];
#pragma unroll
      for (int u = 0; u < UV; ++u) r[u] = yv[u < cnt ? v0 + 32 * u : v0];
#pragma unroll
      for (int u = UV - 1; u >= 0; --u) {
        if (u < cnt) {
#pragma unroll
          for (int q = EV - 1; q >= 0; --q) {
            const int64_t j = (v0 + 32 * u) * EV + q;
            const float Yq = (float)Vec<YT>::get(r[u], q);
            const float val = AFF ? fmaf(lk, tb, fmaf(lk, (float)(32 * EV * u + q), Yq)) : fmaf(lk, tval(j), Yq);
            const int kk = (lane & 1) ? fkey(-val) : fkey(val);
            if (kk == my_key) off = j;
          }
        }
      }
    }
  }
  k3s_cand_finish<XT, YT>(a, ka, xs, ys, b, lo, off);
}

// Pruned candidates (affine x; group summaries of phase 1).  For slope lambda
// a group with y range [ymn, ymx] and index offsets [t0, t1] holds a value of
// Y + lambda T of at least ymx + min(lambda t0, lambda t1) and none above
// ymx + max(lambda t0, lambda t1): only groups whose upper bound reaches the
// best lower bound of any group (likewise for the minima) can hold the
// slope's extreme.  The union of those groups over the D slopes (C2: ~5 of 79)
// is staged in shared memory as (Y, T) pairs, and lane l searches slope l % 16
// over half of the staged points (both extremes), so no winner resolution is
// needed: T is the exact index offset (buckets below 2^24 points).  Compact
// code on purpose (rolled loops): a warp runs this once per bucket, and
// straight-line code of that length is bound by instruction fetch.  A heuristic
// like the plain search (phase 4 makes the result exact); returns false when
// the plain search should run instead.
constexpr int K3S_STAGE = 512;  // staged points per warp and chunk (float2 each; + 32 head / tail slots)
constexpr int K3S_STAGE_LD = K3S_STAGE + 32;
template <typename XT, typename YT>
__device__ __noinline__ bool k3s_cand_pruned(const LttbArgs& a, const K3sArgs& ka, const XT* xs, const YT* ys, int64_t b,
                                             int64_t lo, int64_t hi, float lmin, float lmax, unsigned char* slist,
                                             float2* stage, int2 gk0, int2 gk1, int2 gk2, int2 gk3) {
  constexpr int D = K3S_D, NI = K3S_GCAP / 32;
  constexpr int EV = Vec<YT>::EV, CW = K3S_STAGE / (32 * EV);  // warp-loads per chunk
  static_assert(D == 16, "lane l searches slope l % 16");
  const int lane = threadIdx.x & 31;
  k3s_dbg(1);
  const VWin w = vwin<YT>(lo, hi);
  if (hi - lo >= (1 << 24)) return false;  // (T must be exact in f32)
  const GGeo gg = ggeo(w);
  if (gg.ng < K3S_PRUNE_MIN_GROUPS) return false;
  const uint4* yv = reinterpret_cast<const uint4*>(ys);
  // this lane's groups (summaries loaded by the caller, ahead of its own loads):
  // y bounds (outer and inner) and index offsets
  const int2 gk[NI] = {gk0, gk1, gk2, gk3};
  static_assert(NI == 4, "four summaries per lane");
  float yxh[NI], yxl[NI], ynh[NI], ynl[NI], t0[NI], t1[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int gi = lane + 32 * i;
    yxh[i] = yxl[i] = -INFINITY; ynh[i] = ynl[i] = INFINITY; t0[i] = t1[i] = 0.f;
    if (gi < gg.ng) {
      const int2 k = gk[i];
      if constexpr (sizeof(YT) == 4) {
        yxh[i] = yxl[i] = __int_as_float(k.y ^ ((k.y >> 31) & 0x7fffffff));
        ynh[i] = ynl[i] = __int_as_float(k.x ^ ((k.x >> 31) & 0x7fffffff));
      } else {
        yxh[i] = __double2float_ru(dkey_inv((long long)k.y * 4294967296LL + 4294967295LL));
        yxl[i] = __double2float_rd(dkey_inv((long long)k.y * 4294967296LL));
        ynl[i] = __double2float_rd(dkey_inv((long long)k.x * 4294967296LL));
        ynh[i] = __double2float_ru(dkey_inv((long long)k.x * 4294967296LL + 4294967295LL));
      }
      const int64_t v0g = w.vf + ((int64_t)gi << (gg.s + 5)), v1g = min((int64_t)w.vl, (int64_t)(v0g + (32LL << gg.s)));
      t0[i] = (float)(v0g * EV - lo);
      t1[i] = (float)(v1g * EV - 1 - lo);
    }
  }
  k3s_dbg(2);
  const float tspan = (float)(hi - lo), dl = (lmax - lmin) * (1.f / (float)(D - 1));
  bool sv[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) sv[i] = false;
#pragma unroll 4
  for (int k = 0; k < D; ++k) {
    const float l = fmaf(dl, (float)k, lmin);
    float bl = -INFINITY, bs = INFINITY;
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const float p0 = l * t0[i], p1 = l * t1[i];
      bl = fmaxf(bl, yxl[i] + fminf(p0, p1));   // a value of at least this exists
      bs = fminf(bs, ynh[i] + fmaxf(p0, p1));   // a value of at most this exists
    }
    const int kx = __reduce_max_sync(FULL, fkey(bl)), kn = __reduce_max_sync(FULL, fkey(-bs));
    const float tx = __int_as_float(kx ^ ((kx >> 31) & 0x7fffffff)), tn = -__int_as_float(kn ^ ((kn >> 31) & 0x7fffffff));
    const float sl = 2e-6f * (fabsf(l) * tspan);
    const float thx = tx - (sl + 2e-6f * fabsf(tx)), thn = tn + (sl + 2e-6f * fabsf(tn));
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const float p0 = l * t0[i], p1 = l * t1[i];
      sv[i] = sv[i] || (yxh[i] + fmaxf(p0, p1) >= thx) || (ynl[i] + fminf(p0, p1) <= thn);
    }
  }
  k3s_dbg(3);
  int nsurv = 0;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const unsigned wd = __ballot_sync(FULL, sv[i]);
    K3S_ASSERT(!sv[i] || (nsurv + __popc(wd & ((1u << lane) - 1u)) < K3S_GCAP && lane + 32 * i < gg.ng));
    if (sv[i]) slist[nsurv + __popc(wd & ((1u << lane) - 1u))] = (unsigned char)(lane + 32 * i);
    nsurv += __popc(wd);
  }
  __syncwarp();
  const int64_t nun = (int64_t)nsurv << gg.s;  // warp-loads to scan
  if (nsurv == 0 || nun * 2 > gg.nl) return false;
  k3s_cnt_add(8, 1);
  k3s_cnt_add(9, nsurv);
  // lane l: the 4 slopes 4 (l % 4) .. + 3 (8 independent running extremes)
  // over the staged float4s (2 points each) l / 4, l / 4 + 8, ...
  const int sq = lane & 3, ps = lane >> 2;
  float lk[4], bmax[4], bmin[4], tmax[4], tmin[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    lk[j] = fmaf(dl, (float)(4 * sq + j), lmin);
    bmax[j] = -INFINITY; bmin[j] = INFINITY; tmax[j] = -1.f; tmin[j] = -1.f;
  }
  auto search = [&](int np) {  // np: staged points, a multiple of 2
    __syncwarp();
    const float4* s4 = reinterpret_cast<const float4*>(stage);
#pragma unroll 1
    for (int i = ps; i < np / 2; i += 8) {
      const float4 v = s4[i];  // two (Y, T) points
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float a0 = fmaf(lk[j], v.y, v.x), a1 = fmaf(lk[j], v.w, v.z);
        if (a0 > bmax[j]) { bmax[j] = a0; tmax[j] = v.y; }
        if (a0 < bmin[j]) { bmin[j] = a0; tmin[j] = v.y; }
        if (a1 > bmax[j]) { bmax[j] = a1; tmax[j] = v.w; }
        if (a1 < bmin[j]) { bmin[j] = a1; tmin[j] = v.w; }
      }
    }
    __syncwarp();
  };
  k3s_dbg(4);
  const int smask = (1 << gg.s) - 1;
#pragma unroll 1
  for (int64_t q0 = 0; q0 < nun; q0 += CW) {
    uint4 r[CW];
    int64_t vs[CW];
#pragma unroll
    for (int u = 0; u < CW; ++u) {
      vs[u] = -1;
      if (q0 + u < nun) {
        const int64_t q = q0 + u;
        K3S_ASSERT((q >> gg.s) < nsurv && slist[q >> gg.s] < gg.ng);
        const int64_t v = w.vf + 32 * ((((int64_t)slist[q >> gg.s]) << gg.s) + (q & smask)) + lane;
        K3S_ASSERT(v >= w.vf);
        if (v < w.vl) vs[u] = v;
      }
      r[u] = vs[u] >= 0 ? yv[vs[u]] : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < CW; ++u) {
      const float tb = (float)(vs[u] * EV - lo);
#pragma unroll
      for (int e = 0; e < EV; ++e) {
        K3S_ASSERT((u * 32 + lane) * EV + e < K3S_STAGE);
        stage[(u * 32 + lane) * EV + e] = vs[u] >= 0 ? make_float2((float)Vec<YT>::get(r[u], e), tb + (float)e) : make_float2(NAN, 0.f);
      }
    }
    int np = (int)min((int64_t)CW, nun - q0) * 32 * EV;
    if (q0 == 0) {  // head / tail elements ride along (NaN: an empty slot, never wins)
      const int64_t ej = vwin_edge(w, lo, lane);
      K3S_ASSERT(np + lane < K3S_STAGE_LD && (ej < 0 || (ej >= lo && ej < hi)));
      stage[np + lane] = ej >= 0 ? make_float2((float)ys[ej], (float)(ej - lo)) : make_float2(NAN, 0.f);
      np += 32;
    }
    search(np);
  }
  k3s_dbg(5);
  // merge the 8 point subsets (lanes with equal l % 4); lane l then reports
  // extreme l / 4 of its 4 slopes x 2 sides
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float obx = __shfl_xor_sync(FULL, bmax[j], o), otx = __shfl_xor_sync(FULL, tmax[j], o);
      const float obn = __shfl_xor_sync(FULL, bmin[j], o), otn = __shfl_xor_sync(FULL, tmin[j], o);
      if (obx > bmax[j]) { bmax[j] = obx; tmax[j] = otx; }
      if (obn < bmin[j]) { bmin[j] = obn; tmin[j] = otn; }
    }
  }
  float tw = tmax[0];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    tw = ps == 2 * j ? tmax[j] : tw;
    tw = ps == 2 * j + 1 ? tmin[j] : tw;
  }
  const int64_t off = tw >= 0.f ? lo + (int64_t)tw : -1;
  k3s_cand_finish<XT, YT>(a, ka, xs, ys, b, lo, off);
  k3s_dbg(6);
  return true;
}

template <typename XT, typename YT>
__device__ __forceinline__ void k3s_cand(const LttbArgs& a, const K3sArgs& ka, const XT* xs, const YT* ys, int64_t b,
                                         int64_t lo, int64_t hi, unsigned char* slist, float2* stage) {
  constexpr int D = K3S_D;
  k3s_dbg(0);
  int2 gk[4] = {};
  if (ka.gmeta) {
#pragma unroll
    for (int i = 0; i < 4; ++i) gk[i] = __ldcg(ka.gmeta + b * K3S_GCAP + (threadIdx.x & 31) + 32 * i);
  }
  double bx0, bx1, by0, by1;
  if (b == 0) {
    bx0 = bx1 = to_f64(xs, 0);
    by0 = by1 = to_f64(ys, 0);
  } else {
    const double2 xr = __ldcg(a.xrange + b - 1), yr = __ldcg(a.yrange + b - 1);
    bx0 = xr.x; bx1 = xr.y; by0 = yr.x; by1 = yr.y;
  }
  const double2 c = __ldcg(a.means + b);
  XAff f;
  f.ok = 0;
  if (a.xaff) {
    const XAff* fp = a.xaff + b;
    f.d = __ldcg(&fp->d); f.di = __ldcg(&fp->di); f.ok = __ldcg(&fp->ok);
  }
  // area ~ P*Y + S*X with P = ax - cx, S = cy - ay over the anchor box corners;
  // affine x: X = d*T -> extremes of Y + lambda*T with lambda = S*d/P
  const bool aff = f.ok;
  const double dsc = aff ? (XForm<XT>::integral ? (double)f.di : f.d) : 1.0;
  double lmin = INFINITY, lmax = -INFINITY;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double ax = (q & 1) ? bx1 : bx0, ay = (q & 2) ? by1 : by0;
    double l = (c.y - ay) * dsc / (ax - c.x);
    if (l != l) l = 0.0;
    l = fmin(fmax(l, -1e20), 1e20);
    lmin = fmin(lmin, l);
    lmax = fmax(lmax, l);
  }
  if (aff && ka.gmeta && k3s_cand_pruned<XT, YT>(a, ka, xs, ys, b, lo, hi, (float)lmin, (float)lmax, slist, stage, gk[0], gk[1], gk[2], gk[3])) return;
  float lam[D];
#pragma unroll
  for (int k = 0; k < D; ++k) lam[k] = (float)(lmin + (lmax - lmin) * ((double)k / (double)(D - 1)));
  k3s_cnt_add(10, 1);
  if (aff) k3s_cand_t<XT, YT, true>(a, ka, xs, ys, b, lo, hi, lam, 0.0);
  else k3s_cand_t<XT, YT, false>(a, ka, xs, ys, b, lo, hi, lam, elem_f64(xs[lo]));
}

// ---------------------------------------------------------------- phase 3 --
// One warp: T_b[p] = argmax_q exact area(anchor p, candidate q, c_b), strict
// '>' in ascending candidate order (lowest index on ties, NaN never wins).
// Lane l: anchor p = l/2, candidates q in [8(l&1), 8(l&1)+8).
static __device__ __noinline__ void k3s_table(const LttbArgs& a, const K3sArgs& ka, int64_t b, double x0, double y0,
                                          unsigned char* tab) {
  constexpr int H = K3S_H, PL = 32 / H == 2 ? 2 : 1;  // lanes per anchor
  constexpr int QL = H / PL;                           // candidates per lane
  const int lane = threadIdx.x & 31;
  k3s_dbg(8);
  const int p = lane / PL, q0 = (lane % PL) * QL;
  int na = 1;
  double ax = x0, ay = y0;
  if (b > 0) {
    na = __ldcg(a.cand_cnt + b - 1);
    if (p < na) {
      const double2 v = __ldcg(ka.cpt + (b - 1) * H + p);
      ax = v.x; ay = v.y;
    }
  }
  const int nq = __ldcg(a.cand_cnt + b);
  const double2 c = __ldcg(a.means + b);
  long long bk = -2;
  int bq = 0;
  // one coalesced load of the bucket's candidate points, then warp broadcasts
  // (a load per candidate was four dependent L2 round trips)
  double2 mine = make_double2(0.0, 0.0);
  if (lane < nq) mine = __ldcg(ka.cpt + b * H + lane);
  const int nqw = __reduce_max_sync(FULL, nq - q0);  // (warp-uniform trip count)
#pragma unroll 4
  for (int i = 0; i < QL; ++i) {
    if (i >= nqw) break;
    const double px = __shfl_sync(FULL, mine.x, q0 + i), py = __shfl_sync(FULL, mine.y, q0 + i);
    const long long k = lttb_area_key(ax, ay, c.x, c.y, px, py);
    if (q0 + i < nq && k > bk) { bk = k; bq = q0 + i; }
  }
  if (PL == 2) {
    const long long ok = __shfl_xor_sync(FULL, bk, 1);
    const int oq = __shfl_xor_sync(FULL, bq, 1);
    if (ok > bk || (ok == bk && oq < bq)) { bk = ok; bq = oq; }
  }
  if (lane % PL == 0) tab[p] = (unsigned char)(p < na && bk >= -1 ? bq : 0);
  k3s_dbg(9);
}

// ---------------------------------------------------------------- phase 4 --
// In-order fp64 mean of bucket b+1 (_kernels.py:98-104) by lanes 0 / 1 of a warp
// (the rare path of a failed certification), broadcast to the warp.
template <typename XT, typename YT>
__device__ __noinline__ double2 warp_exact_mean(const LttbArgs& a, const XT* xs, const YT* ys, int64_t m, int64_t b) {
  const int lane = threadIdx.x & 31;
  const int64_t k3 = a.n_out - 2;
  if (b + 1 >= k3) return make_double2(to_f64(xs, m - 1), to_f64(ys, m - 1));
  const int64_t nlo = lbound(a, m, b + 1), nhi = lbound(a, m, b + 2);
  double acc = 0.0;
  if (lane < 2) {
    for (int64_t j = nlo; j < nhi; ++j) acc = __dadd_rn(acc, lane == 0 ? to_f64(xs, j) : to_f64(ys, j));
    acc = __ddiv_rn(acc, (double)(nhi - nlo));
  }
  return make_double2(__shfl_sync(FULL, acc, 0), __shfl_sync(FULL, acc, 1));
}

// One warp: exact |area| keys over bucket [lo, hi) given anchor (ax, ay) and
// mean c (lttb_area's op order), every point exactly once: top-2 keys and the
// first index of the top (warp-reduced).
template <typename XT, typename YT>
__device__ __forceinline__ void warp_scan_area(const XT* xs, const YT* ys, int64_t lo, int64_t hi, double ax, double ay,
                                               double2 c, const XAff& f, bool afi, long long& k1, long long& k2,
                                               long long& i1, int& bad) {
  constexpr int EV = Vec<YT>::EV, UV = 16 / EV;
  const int lane = threadIdx.x & 31;
  const double P = __dsub_rn(ax, c.x), S = __dsub_rn(c.y, ay);
  k1 = -1; k2 = -1; bad = 0;
  int64_t il = LLONG_MAX;
  auto xat = [&](int64_t j) -> double {
    return f.ok ? (afi ? i2d_magic((long long)((unsigned long long)f.x0i + (unsigned long long)(j - lo) * (unsigned long long)f.di))
                       : XForm<XT>::at(f, j - lo))
                : elem_f64(xs[j]);
  };
  auto el = [&](double xj, YT y, int64_t j) {
    const double R = __dsub_rn(ax, xj), Q = __dsub_rn((double)y, ay);
    const double tt = __dsub_rn(__dmul_rn(P, Q), __dmul_rn(R, S));  // lttb_area, same op order
    long long k = __double_as_longlong(tt) & 0x7fffffffffffffffLL;
    bad |= (int)(k >> 32) >= 0x7ff00000;      // inf / NaN: no certification
    k = k > 0x7ff0000000000000LL ? -1LL : k;  // NaN never wins
    // (a lane visits its head / tail element BEFORE its vector elements, so an exact tie
    // with the running top must still resolve to the lower index: _kernels.py:114's strict
    // `>` in ascending index order keeps the first of equal areas)
    if (k > k1) { k2 = k1; k1 = k; il = j; }
    else {
      if (k > k2) k2 = k;
      if (k == k1 && k >= 0 && j < il) il = j;
    }
  };
  const VWin w = vwin<YT>(lo, hi);
  {
    const int64_t j = vwin_edge(w, lo, lane);
    if (j >= 0) el(xat(j), ys[j], j);
  }
  const uint4* yv = reinterpret_cast<const uint4*>(ys);
  // affine integer x: exact integer-valued doubles stepped by exact adds
  const double dvec = afi ? i2d_magic(f.di * (32 * EV)) : 0.0, d1 = afi ? i2d_magic(f.di) : 0.0;
  for (int64_t v0 = w.vf + lane; v0 < w.vl; v0 += 32 * UV) {
    uint4 r[UV];
#pragma unroll
    for (int u = 0; u < UV; ++u) r[u] = yv[v0 + 32 * u < w.vl ? v0 + 32 * u : v0];
    double xv = afi ? xat(v0 * EV) : 0.0;
#pragma unroll
    for (int u = 0; u < UV; ++u) {
      const int64_t v = v0 + 32 * u;
      if (v < w.vl) {
        double xq = xv;
#pragma unroll
        for (int q = 0; q < EV; ++q) {
          const int64_t j = v * EV + q;
          el(afi ? xq : xat(j), Vec<YT>::get(r[u], q), j);
          if (afi) xq = __dadd_rn(xq, d1);
        }
      }
      if (afi) xv = __dadd_rn(xv, dvec);
    }
  }
  i1 = il;
#pragma unroll
  for (int o = 16; o; o >>= 1)
    vpart_merge(k1, i1, k2, bad, __shfl_xor_sync(FULL, k1, o), __shfl_xor_sync(FULL, i1, o),
                __shfl_xor_sync(FULL, k2, o), __shfl_xor_sync(FULL, bad, o));
}

// One warp: the reference's pick of bucket b given anchor `prev`, certified
// against the mean's error bound (k3c_area_err); a failed certification takes
// the in-order mean and re-scans.  Never writes means/merr (other warps of the
// launch may be reading them).
template <typename XT, typename YT>
__device__ __noinline__ int64_t warp_pick(const LttbArgs& a, const XT* xs, const YT* ys, int64_t m, int64_t b, int64_t prev) {
  const int64_t lo = lbound(a, m, b), hi = lbound(a, m, b + 1);
  const double ax = to_f64(xs, prev), ay = to_f64(ys, prev);
  const double2 c = __ldcg(a.means + b);
  const double2 ce = __ldcg(a.merr + b);
  const double2 yr = __ldcg(a.yrange + b), xr = __ldcg(a.xrange + b);
  XAff f;
  f.ok = 0;
  if (a.xaff) {
    const XAff* fp = a.xaff + b;
    f.x0 = __ldcg(&fp->x0); f.d = __ldcg(&fp->d); f.x0i = __ldcg(&fp->x0i); f.di = __ldcg(&fp->di);
    f.ok = __ldcg(&fp->ok);
  }
  const bool afi = f.ok && XForm<XT>::integral && fmax(fabs(xr.x), fabs(xr.y)) < 1125899906842624.0 &&
                   fabs((double)f.di) * 128.0 < 1125899906842624.0;
  long long k1, k2, i1;
  int bad;
  warp_scan_area<XT, YT>(xs, ys, lo, hi, ax, ay, c, f, afi, k1, k2, i1, bad);
  const double u = K3C_U;
  bool ok = !bad && ((ce.x == 0.0 && ce.y == 0.0) || hi - lo == 1);
  if (!ok && !bad && !a.cert_force) {
    const double P = __dsub_rn(ax, c.x), S = __dsub_rn(c.y, ay);
    // |Q_j| <= (1+u) max|y - ay| over the bucket's y range (likewise R)
    const double qmax = fmax(fabs(__dsub_rn(yr.y, ay)), fabs(__dsub_rn(yr.x, ay))) * (1.0 + 4.0 * u);
    const double rmax = fmax(fabs(__dsub_rn(ax, xr.x)), fabs(__dsub_rn(ax, xr.y))) * (1.0 + 4.0 * u);
    const double v1 = k1 < 0 ? -1.0 : __longlong_as_double(k1), v2 = k2 < 0 ? -1.0 : __longlong_as_double(k2);
    const double E = k3c_area_err(ce, P, S, qmax, rmax, v1);
    ok = __dsub_rn(v1, v2) > 2.0 * E * (1.0 + 1e-9);  // NaN bounds fail
  }
  if (ok) return i1 == LLONG_MAX ? lo : i1;  // all-NaN bucket keeps bounds[b] (:110)
  const double2 ce2 = warp_exact_mean<XT, YT>(a, xs, ys, m, b);
  warp_scan_area<XT, YT>(xs, ys, lo, hi, ax, ay, ce2, f, afi, k1, k2, i1, bad);
  return i1 == LLONG_MAX ? lo : i1;
}

// Phase 4's common case, for a group of NWG warps (1: one warp per bucket;
// K3S_NW: the whole CTA on one bucket, for the few re-scans of 4b and the
// repair): is r the reference's pick of bucket b given anchor `prev`?  Every
// point's exact |area| key (lttb_area's op order) is compared with r's key Kr
// only -- a point before r must stay below Kr, a point after r must not
// exceed it (lowest index wins ties), one 64-bit compare against a per-vector
// threshold.  The runner-up needed by the certification is bounded by the
// second-largest HIGH word of all keys (32-bit top-2), whose first point is
// also the next guess (*alt) when r is wrong.  Returns false when anything is
// off (violation, inf / NaN, failed certification).
struct GrpRed { int v, m1, m2, j1; };
__device__ __forceinline__ void top2_merge(int& m1, int& m2, int& j1, int om1, int om2, int oj1) {
  m2 = max(max(m2, om2), min(m1, om1));
  j1 = om1 > m1 ? oj1 : (om1 < m1 ? j1 : min(j1, oj1));
  m1 = max(m1, om1);
}

template <int NWG, typename XT, typename YT>
__device__ __noinline__ bool grp_verify(const LttbArgs& a, const XT* xs, const YT* ys, int64_t m, int64_t b, int64_t prev,
                           int64_t r, int64_t* alt, GrpRed* sh, const int2* gm) {
  constexpr int EV = Vec<YT>::EV, UV = 8 / EV, NL = 32 * NWG;
  const int lane = threadIdx.x & 31, wg = NWG == 1 ? 0 : (int)(threadIdx.x >> 5);
  const int L = wg * 32 + lane;
  const int64_t lo = lbound(a, m, b), hi = lbound(a, m, b + 1);
  if (alt) *alt = -1;
  if (NWG == 1) k3s_dbg(16);
  if (r < lo || r >= hi) return false;
  int2 gk[K3S_GCAP / 32] = {};  // group summaries, loaded with the first batch (they only depend on b)
  if constexpr (NWG == 1) {
    if (gm) {
#pragma unroll
      for (int i = 0; i < K3S_GCAP / 32; ++i) gk[i] = __ldcg(gm + lane + 32 * i);
    }
  }
  const double ax = to_f64(xs, prev), ay = to_f64(ys, prev);
  const double2 c = __ldcg(a.means + b);
  const double2 ce = __ldcg(a.merr + b);
  const double2 yr = __ldcg(a.yrange + b), xr = __ldcg(a.xrange + b);
  XAff f;
  f.ok = 0;
  if (a.xaff) {
    const XAff* fp = a.xaff + b;
    f.x0i = __ldcg(&fp->x0i); f.di = __ldcg(&fp->di); f.x0 = __ldcg(&fp->x0); f.d = __ldcg(&fp->d);
    f.ok = __ldcg(&fp->ok);
  }
  // affine integer x, every value (and the anchor's) an integer below 2^50: R_j = ax - x_j is
  // exact, so it is stepped by exact subtractions instead of recomputed
  const bool afi = f.ok && XForm<XT>::integral && fmax(fmax(fabs(xr.x), fabs(xr.y)), fabs(ax)) < 1125899906842624.0 &&
                   fabs((double)f.di) * (4.0 * NL) < 1125899906842624.0;
  const double P = __dsub_rn(ax, c.x), S = __dsub_rn(c.y, ay);
  auto xat = [&](int64_t j) -> double {
    return f.ok ? (afi ? i2d_magic((long long)((unsigned long long)f.x0i + (unsigned long long)(j - lo) * (unsigned long long)f.di))
                       : XForm<XT>::at(f, j - lo))
                : elem_f64(xs[j]);
  };
  auto keyR = [&](double R, double yj) -> long long {
    const double tt = __dsub_rn(__dmul_rn(P, __dsub_rn(yj, ay)), __dmul_rn(R, S));  // lttb_area, same op order
    return __double_as_longlong(tt) & 0x7fffffffffffffffLL;
  };
  const long long Kr = keyR(__dsub_rn(ax, xat(r)), to_f64(ys, r));
  if (Kr >= 0x7ff0000000000000LL) return false;  // inf / NaN pick: the full path decides
  const int hr = (int)(Kr >> 32);
  // 32-bit top-2 of the keys' HIGH words (inf / NaN keys have the largest) and the
  // first point of the top: r is the exact pick iff it holds the top high word alone
  int m1 = -1, m2 = -1, j1 = INT_MAX;
  auto el = [&](double R, double yj, int jr) {
    const int h = (int)(keyR(R, yj) >> 32);
    const bool up = h > m1;
    m2 = max(m2, min(m1, h));
    j1 = up ? jr : j1;
    m1 = max(m1, h);
  };
  const VWin w = vwin<YT>(lo, hi);
  if (NWG == 1 || wg == 0) {  // head / tail elements
    const int64_t j = vwin_edge(w, lo, lane);
    if (j >= 0) el(__dsub_rn(ax, xat(j)), to_f64(ys, j), (int)(j - lo));
  }
  auto run = [&](auto afi_tag) {
    constexpr bool AFI = decltype(afi_tag)::value;
    const double d1 = AFI ? i2d_magic(f.di) : 0.0;
    const double dvec = AFI ? i2d_magic(f.di * (NL * EV)) : 0.0;
    vrounds<UV, false, true>(reinterpret_cast<const uint4*>(ys), w, L, NL, [&](const uint4 (&rr)[UV], int64_t v0, int cnt, int) {
      const int jb = (int)(v0 * EV - lo);
      double Rv = AFI ? __dsub_rn(ax, xat(v0 * EV)) : 0.0;
#pragma unroll
      for (int u = 0; u < UV; ++u) {
        if (u < cnt) {
          double Rq = Rv;
#pragma unroll
          for (int q = 0; q < EV; ++q) {
            const int jr = jb + NL * EV * u + q;
            if constexpr (AFI) {
              el(Rq, (double)Vec<YT>::get(rr[u], q), jr);
              Rq = __dsub_rn(Rq, d1);
            } else {
              el(__dsub_rn(ax, xat(lo + jr)), (double)Vec<YT>::get(rr[u], q), jr);
            }
          }
        }
        if (AFI) Rv = __dsub_rn(Rv, dvec);
      }
    });
  };
  // Pruned scan (one warp, group summaries of phase 1): every fp operation of
  // the area is monotone in its operands, so over a group's box [xa, xb] x [y0, y1]
  // the rounded value tt lies in [fl(Mmin - Nmax), fl(Mmax - Nmin)] with
  // M = fl(P fl(y - ay)) and N = fl(fl(ax - x) S) taken at the box edges -- no
  // error term.  A group whose bound's high word is below r's cannot hold the
  // pick nor share r's high word and is skipped (its bound still feeds the
  // runner-up m2 of the certification); non-finite products keep the group.
  bool scanned = false;
  int mB = -1;
  if (NWG == 1) k3s_dbg(17);
  if constexpr (NWG == 1) {
    // (affine integer x: the bucket's x range comes from the formula's end points,
    // which bound every value only when the formula cannot wrap: else no pruning)
    const bool xnowrap = fabs((double)f.di) * (double)(hi - lo) < 4.0e15 && fmax(fabs(xr.x), fabs(xr.y)) < 4.0e15;
    const GGeo gg = ggeo(w);
    if (gm && gg.ng >= K3S_PRUNE_MIN_GROUPS && (!f.ok || !XForm<XT>::integral || xnowrap)) {
      const bool xexact = f.ok;
      unsigned words[K3S_GCAP / 32];
      int nsurv = 0, mBl = -1;
#pragma unroll
      for (int i = 0; i < K3S_GCAP / 32; ++i) {
        const int gi = lane + 32 * i;
        bool sv = false;
        if (gi < gg.ng) {
          double y0, y1;
          gkey_bounds<YT>(gk[i], y0, y1);
          const int64_t v0g = w.vf + ((int64_t)gi << (gg.s + 5)), v1g = min((int64_t)w.vl, (int64_t)(v0g + (32LL << gg.s)));
          double xa = xr.x, xb = xr.y;
          if (xexact) {
            xa = XForm<XT>::at(f, v0g * EV - lo);
            xb = XForm<XT>::at(f, v1g * EV - 1 - lo);
            if (xb < xa) { const double tt = xa; xa = xb; xb = tt; }
          }
          const double M0 = __dmul_rn(P, __dsub_rn(y0, ay)), M1 = __dmul_rn(P, __dsub_rn(y1, ay));
          const double N0 = __dmul_rn(__dsub_rn(ax, xa), S), N1 = __dmul_rn(__dsub_rn(ax, xb), S);
          const int kfin = max(max(hw_abs(M0), hw_abs(M1)), max(hw_abs(N0), hw_abs(N1)));
          const double tlo = __dsub_rn(fmin(M0, M1), fmax(N0, N1)), thi = __dsub_rn(fmax(M0, M1), fmin(N0, N1));
          const int hb = max(hw_abs(tlo), hw_abs(thi));
          sv = kfin >= 0x7ff00000 || hb >= hr;
          if (!sv) mBl = max(mBl, hb);
        }
        words[i] = __ballot_sync(FULL, sv);
        nsurv += __popc(words[i]);
      }
      if ((((int64_t)nsurv << gg.s) << 1) <= gg.nl) {  // else: the plain scan is cheaper
        scanned = true;
        k3s_cnt_add(11, 1);
        k3s_cnt_add(12, nsurv);
        mB = __reduce_max_sync(FULL, mBl);
        const uint4* yv = reinterpret_cast<const uint4*>(ys);
        const int nsub = 1 << gg.s;
        static_assert(K3S_GCAP == 128, "four ballot words");
#pragma unroll 1
        for (int i = 0; i < K3S_GCAP / 32; ++i) {
          for (unsigned wd = i == 0 ? words[0] : i == 1 ? words[1] : i == 2 ? words[2] : words[3]; wd; wd &= wd - 1) {
            const int gi = 32 * i + __ffs(wd) - 1;
            const int64_t vb = w.vf + ((int64_t)gi << (gg.s + 5)) + lane;
            for (int sub = 0; sub < nsub; sub += 4) {
              uint4 rr[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int64_t v = vb + 32LL * (sub + u);
                K3S_ASSERT(v >= w.vf && gi < gg.ng);
                rr[u] = (sub + u < nsub && v < w.vl) ? yv[v] : make_uint4(0, 0, 0, 0);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int64_t v = vb + 32LL * (sub + u);
                if (sub + u < nsub && v < w.vl) {
#pragma unroll
                  for (int q = 0; q < EV; ++q) {
                    const int64_t j = v * EV + q;
                    el(__dsub_rn(ax, xat(j)), (double)Vec<YT>::get(rr[u], q), (int)(j - lo));
                  }
                }
              }
            }
          }
        }
      }
    }
  }
  if (NWG == 1) k3s_dbg(18);
  if (!scanned) {
    if (NWG == 1) k3s_cnt_add(13, 1);
    if (afi) run(std::true_type{});
    else run(std::false_type{});
  }
  // group reduction
#pragma unroll
  for (int o = 16; o; o >>= 1)
    top2_merge(m1, m2, j1, __shfl_xor_sync(FULL, m1, o), __shfl_xor_sync(FULL, m2, o), __shfl_xor_sync(FULL, j1, o));
  if constexpr (NWG > 1) {
    __syncthreads();
    if (lane == 0) sh[wg] = GrpRed{0, m1, m2, j1};
    __syncthreads();
    m1 = -1; m2 = -1; j1 = INT_MAX;
    for (int q = 0; q < NWG; ++q) {
      const GrpRed g = sh[q];
      top2_merge(m1, m2, j1, g.m1, g.m2, g.j1);
    }
  }
  if (NWG == 1) k3s_dbg(19);
  m2 = max(m2, mB);  // skipped groups: every key's high word <= mB < hr
  if (NWG == 1) k3s_count(-0); else k3s_count(0);
  if (m1 > hr) {  // a point beats r: where the exact pick most likely is
    if (alt && m1 < 0x7ff00000 && j1 != INT_MAX) *alt = lo + j1;
    if (NWG == 1) k3s_count(-1); else k3s_count(1);
    return false;
  }
  if (m2 >= hr) {  // another point shares r's high word: the full comparison decides
    if (NWG == 1) k3s_count(-2); else k3s_count(2);
    return false;
  }
  if ((ce.x == 0.0 && ce.y == 0.0) || hi - lo == 1) return true;  // exact mean: r is the reference's pick
  if (a.cert_force) return false;
  const double u = K3C_U;
  const double qmax = fmax(fabs(__dsub_rn(yr.y, ay)), fabs(__dsub_rn(yr.x, ay))) * (1.0 + 4.0 * u);
  const double rmax = fmax(fabs(__dsub_rn(ax, xr.x)), fabs(__dsub_rn(ax, xr.y))) * (1.0 + 4.0 * u);
  const double v1 = __longlong_as_double(Kr);
  const double v2 = m2 < 0 ? -1.0 : __longlong_as_double(((long long)m2 << 32) | 0xffffffffLL);  // >= every other area
  const double E = k3c_area_err(ce, P, S, qmax, rmax, v1);
  const bool ok = __dsub_rn(v1, v2) > 2.0 * E * (1.0 + 1e-9);
  if (!ok) { if (NWG == 1) k3s_count(-3); else k3s_count(3); }
  return ok;
}

// The reference's pick of bucket b given anchor `prev`, starting from a
// guess: the guess verified (one scan), else the scan's best high-word point
// verified (a second scan), else the full certified top-2 scan (warp: warp_pick;
// CTA: block_bucket_argmax_cert, never storing means back).
template <int NWG, typename XT, typename YT>
__device__ int64_t grp_pick(const LttbArgs& a, const XT* xs, const YT* ys, int64_t m, int64_t b, int64_t prev,
                            int64_t guess, GrpRed* sh, double* s_a, long long* s_i, const int2* gm = nullptr) {
  int64_t alt = -1;
  if (grp_verify<NWG, XT, YT>(a, xs, ys, m, b, prev, guess, &alt, sh, gm)) return guess;
  if (alt >= 0 && alt != guess && grp_verify<NWG, XT, YT>(a, xs, ys, m, b, prev, alt, nullptr, sh, gm)) return alt;
  if (NWG == 1) k3s_count(-4); else k3s_count(4);
  if constexpr (NWG == 1) return warp_pick<XT, YT>(a, xs, ys, m, b, prev);
  else return block_bucket_argmax_cert<XT, YT, 32 * NWG>(a, 0, m, xs, ys, b, prev, s_a, s_i, false);
}

// One warp: argmax of the exact area over bucket b's candidate points given
// anchor `prev` (lowest index on ties): the table's answer for any anchor.
template <typename XT, typename YT>
__device__ __noinline__ int64_t warp_cand_guess(const LttbArgs& a, const K3sArgs& ka, const XT* xs, const YT* ys, int64_t b,
                                   int64_t prev) {
  constexpr int H = K3S_H;
  const int lane = threadIdx.x & 31;
  const double ax = to_f64(xs, prev), ay = to_f64(ys, prev);
  const double2 c = __ldcg(a.means + b);
  const int nq = __ldcg(a.cand_cnt + b);
  long long k = -2;
  if (lane < nq) {
    const double2 p = __ldcg(ka.cpt + b * H + lane);
    k = lttb_area_key(ax, ay, c.x, c.y, p.x, p.y);
  }
  long long bk = k;
  int bq = lane;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const long long ok = __shfl_xor_sync(FULL, bk, o);
    const int oq = __shfl_xor_sync(FULL, bq, o);
    if (ok > bk || (ok == bk && oq < bq)) { bk = ok; bq = oq; }
  }
  return bk >= -1 ? __ldcg(a.cand + b * H + bq) : lbound(a, a.n, b);
}

// ----------------------------------------------------------------- kernel --
template <typename XT, typename YT>
__global__ void __launch_bounds__(K3S_NT, 1) k_lttb_k3s(LttbArgs a, K3sArgs ka) {
  constexpr int NT = K3S_NT, NW = K3S_NW, H = K3S_H;
  extern __shared__ __align__(16) unsigned char dsm[];  // tables [maxb][16] | pos [maxb+1] | entry [maxb]; repair state
  __shared__ int s_e;
  __shared__ int s_last;
  __shared__ unsigned char s_glist[K3S_NW][K3S_GCAP];  // phase 2: surviving groups per warp
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t k3 = a.n_out - 2, m = a.n;
  const int c = blockIdx.x;
  const unsigned G = (unsigned)ka.G;
  const int64_t B0 = (int64_t)c * k3 / G, B1 = (int64_t)(c + 1) * k3 / G;
  const XT* xs = (const XT*)a.x;
  const YT* ys = (const YT*)a.y;
  unsigned char* c_tab = dsm;
  long long* c_pos = reinterpret_cast<long long*>(dsm + ((int64_t)ka.maxb * H + 15) / 16 * 16);
  int* c_e = reinterpret_cast<int*>(c_pos + ka.maxb + 1);
  int* fcount = reinterpret_cast<int*>(ka.sync + K3S_FCOUNT);
  auto stamp = [&](int i) {
    if (ka.prof && t == 0) ka.prof[c * 8 + i] = gtimer();
  };
#ifdef K3S_PROF
  if (t == 0) g_k3s_cnt = ka.prof ? ka.prof + K3S_GMAX * 8 : nullptr;  // (every CTA: same value)
#endif
  __syncthreads();
  stamp(0);

  for (int64_t i = t; i < B1 - B0; i += NT) ka.chg[B0 + i] = 0;
  // ---- 1: statistics (HBM) ----
  for (int64_t b = B0 + wid; b < B1; b += NW) k3s_stats<XT, YT>(a, xs, ys, b, lbound(a, m, b), lbound(a, m, b + 1), m, ka.gmeta ? ka.gmeta + b * K3S_GCAP : nullptr);
  __syncthreads();
  stamp(1);
  // candidates of buckets [B0, B1) need the statistics of B0-1 and B1 (the
  // neighbour CTAs'): wait for those two, not for the whole grid
  if (t == 0) {
    __threadfence();
    st_rel(ka.sync + K3S_FLAGS + c, 1u);
    if (c > 0) spin_until_set(ka.sync + K3S_FLAGS + c - 1, 1u);
    if (c + 1 < (int)G) spin_until_set(ka.sync + K3S_FLAGS + c + 1, 1u);
  }
  __syncthreads();
  k3s_dbg(10);
  // ---- 2: candidates (L2) ----
  for (int64_t b = B0 + wid; b < B1; b += NW) k3s_cand<XT, YT>(a, ka, xs, ys, b, lbound(a, m, b), lbound(a, m, b + 1), s_glist[wid],
                                                         reinterpret_cast<float2*>(dsm) + wid * K3S_STAGE_LD);  // (dsm: free until phase 3)
#ifndef K3S_NO_WARM
  // The first warp without a bucket (C2 has 2-3 of them) runs the verification of the CTA's
  // first bucket once, with an arbitrary anchor and guess, result discarded (the
  // function has no side effects): phase 4a is once-through code bound by
  // instruction fetch (ncu: 49 % of its samples `no_instruction`), and this brings
  // its instructions to the SM while the other warps search candidates.
  // (one warp, and only beside >= 12 searching warps: the discarded scan is a full one -- an arbitrary
  // guess prunes nothing -- and must not outlast the candidate phase; A/B on one box: C2 93.6 vs 95.0 us,
  // 8 buckets per CTA 79.3 vs 77.4 us without this condition)
  if (wid == B1 - B0 && B1 - B0 >= 12 && ka.gmeta) {
    const int64_t wlo = lbound(a, m, B0);
    (void)grp_verify<1, XT, YT>(a, xs, ys, m, B0, wlo - 1, wlo, nullptr, nullptr, ka.gmeta + B0 * K3S_GCAP);
  }
#endif
  __syncthreads();
  stamp(2);
  // the tables of [B0, B1) need CTA c-1's last candidate set
  if (t == 0) {
    __threadfence();
    st_rel(ka.sync + K3S_FLAGS + K3S_GMAX + c, 1u);
    if (c > 0) spin_until_set(ka.sync + K3S_FLAGS + K3S_GMAX + c - 1, 1u);
  }
  __syncthreads();
  k3s_dbg(11);
  // ---- 3: tables, aggregate A_c = T_{B1-1} o ... o T_{B0}, chain entry, positions ----
  const double px0 = to_f64(xs, 0), py0 = to_f64(ys, 0);
  for (int64_t b = B0 + wid; b < B1; b += NW) k3s_table(a, ka, b, px0, py0, c_tab + (b - B0) * H);
  __syncthreads();
  k3s_dbg(12);
  if (wid == 0 && lane < H) {  // lane p walks state p through the CTA's tables (dependent byte lookups)
    int st = lane;
    for (int64_t b = B0; b < B1; ++b) st = c_tab[(b - B0) * H + st];
    ka.agg[(int64_t)c * H + lane] = (unsigned char)st;
  }
  k3s_dbg(13);
  k3s_grid_sync(ka.sync, 2, G);
  stamp(3);
  k3s_dbg(14);
  // entry = (A_{c-1} o ... o A_0)(0).  The predecessors' aggregate maps are staged
  // in shared memory (one L2 round trip); lane l of warp 0 composes its run of
  // maps by byte lookups (32 independent chains), lane 0 then walks the <= 32
  // run maps and the CTA's own tables.
  unsigned char* s_agg = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(c_e + ka.maxb) + 15) & ~(uintptr_t)15);
  unsigned char* s_chk = s_agg + (int64_t)G * H;
  for (int i = t; i < c * (H / 16); i += NT)
    reinterpret_cast<uint4*>(s_agg)[i] = __ldcg(reinterpret_cast<const uint4*>(ka.agg) + i);
  __syncthreads();
  k3s_dbg(23);
  // every thread walks 2 of the 32 x 32 (run, state) pairs through its run of maps;
  // thread 0 then walks the <= 32 run maps and the CTA's own tables
  const int per = (c + 31) / 32;
  {
    const int l = t >> 4, c0 = l * per, c1 = min(c, c0 + per);
    if (c0 < c1) {
#pragma unroll
      for (int q = 0; q < H / 16; ++q) {
        const int p0 = (t & 15) * (H / 16) + q;
        int st = p0;
        for (int cc = c0; cc < c1; ++cc) st = s_agg[cc * H + st];
        s_chk[l * H + p0] = (unsigned char)st;
      }
    }
  }
  __syncthreads();
  k3s_dbg(24);
  if (t == 0) {
    int e = 0;
    for (int l = 0; l * per < c; ++l) e = s_chk[l * H + e];
    s_e = e;
    int ee = e;
    for (int64_t b = B0; b < B1; ++b) {
      ee = c_tab[(b - B0) * H + ee];
      c_e[b - B0] = ee;
    }
  }
  __syncthreads();
  k3s_dbg(25);
  for (int64_t i = t; i <= B1 - B0; i += NT) {
    int64_t p;
    if (i == 0) p = B0 == 0 ? 0 : __ldcg(a.cand + (B0 - 1) * H + s_e);
    else p = __ldcg(a.cand + (B0 + i - 1) * H + c_e[i - 1]);
    c_pos[i] = p;
    a.pos[B0 + i] = p;
  }
  if (t == 0 && B1 == k3) a.pos[k3 + 1] = m - 1;
  k3s_dbg(26);
  __syncthreads();
  stamp(4);
  // ---- 4a: verification (L2), one warp per bucket; the chain's picks go to
  // the output (patched in 4b where a deviation is repaired) ----
  __shared__ GrpRed s_red[NW];
  __shared__ double s_a[NW];
  __shared__ long long s_i[NW];
  int64_t* out = a.out;
  auto omap = [&](int64_t p) -> int64_t { return a.map ? a.map[p] : p; };
  for (int64_t i = t; i < B1 - B0; i += NT) out[B0 + i + 1] = omap(c_pos[i + 1]);
  if (t == 0 && B0 == 0) out[0] = omap(0);
  if (t == 0 && B1 == k3) out[k3 + 1] = omap(m - 1);
  // 4a + 4j.  Pass 0 verifies every bucket.  When many buckets mismatch (smooth
  // data: the pick moves a little with the anchor, so a candidate chain is off
  // almost everywhere), parallel fixed-point passes replace the walks: a pass
  // moves every flagged bucket's exact pick into the chain (pos[b+1] = best[b])
  // and re-verifies -- all at once, pruned -- the buckets whose anchor moved.
  // The invariant best[b] = pick(b | pos[b]), flag[b] = (best[b] != pos[b+1])
  // holds after every pass, so the loop can stop anywhere: no flags left means
  // the chain is the reference's (induction from bucket 0, exact after pass 0;
  // bucket i after pass i at the latest), a few flags left go to 4b, and jmax
  // passes without convergence leave the rest to 4b / the sequential walk.
  {
    int* const fc0 = fcount;
    for (int it = 0;; ++it) {
      for (int64_t b = B0 + wid; b < B1; b += NW) {
        bool fg = false;
        if (it == 0 || __ldcg(ka.chg + b) == it) {
          const int64_t cur = c_pos[b - B0 + 1];
          const int64_t r = grp_pick<1, XT, YT>(a, xs, ys, m, b, c_pos[b - B0], cur, nullptr, nullptr, nullptr,
                                                ka.gmeta ? ka.gmeta + b * K3S_GCAP : nullptr);
          fg = r != cur;
          K3S_ASSERT(r >= lbound(a, m, b) && r < lbound(a, m, b + 1));
          if (lane == 0) {
            a.best[b] = r;
            if (fg) a.flist[atomicAdd(fcount, 1)] = (int)b;
          }
          if (fg) k3s_count(-5);
          if (it) k3s_cnt_add(14, 1);
        }
        if (lane == 0) a.flag[b] = fg;
      }
      if (it == 0) {
        stamp(5);
        k3s_dbg(20);
        k3s_grid_sync(ka.sync, 3, G);
        k3s_dbg(21);
      } else {
        k3s_grid_sync_n(ka.sync, 1, G, 2 * it);
        if (t == 0 && c == 0) k3s_cnt_add(15, 1);
      }
      const int nf = *(volatile int*)fcount;
#ifdef K3S_NO_4J  // (A/B build: no fixed-point passes)
      break;
#endif
      if (nf <= ka.jmin || it >= ka.jmax) break;
      for (int64_t i = t; i < B1 - B0; i += NT) {
        const int64_t b = B0 + i;
        if (__ldcg(a.flag + b)) {
          const int64_t p = __ldcg(a.best + b);
          c_pos[i + 1] = p;
          a.pos[b + 1] = p;
          out[b + 1] = omap(p);
          K3S_ASSERT(b >= 0 && b < k3);
          if (b + 1 < k3) ka.chg[b + 1] = it + 1;
        }
      }
      fcount = fc0 + ((it + 1) & 1);
      if (c == 0 && t == 0) *fcount = 0;
      k3s_grid_sync_n(ka.sync, 1, G, 2 * it + 1);
      if (t == 0 && B0 > 0) c_pos[0] = __ldcg(a.pos + B0);
      __syncthreads();
    }
  }
  // ---- 4b: one CTA per mismatch f: the true pick of bucket f is best[f]; walk
  // on with exact whole-CTA picks (guessed from the candidate sets) until the
  // chain is re-joined, patching the output.  A walk that meets another
  // mismatch (the deviations interact) leaves everything to the sequential
  // repair walk of step 5 ----
  {
    const int nf = *(volatile int*)fcount;
    if (nf == 0) return;  // (grid-uniform) every bucket verified: the output is final, no last-CTA step
    for (int q = c; q < nf; q += (int)G) {
      const int64_t f = __ldcg(a.flist + q);
      int64_t anc = __ldcg(a.best + f);
      if (t == 0) out[f + 1] = omap(anc);
      for (int64_t b = f + 1; b < k3; ++b) {
        const bool dbg = ka.prof && q == 0 && t == 0 && b - f - 1 < 4;
        if (dbg) ka.prof[K3S_GMAX * 8 + 16 + 4 * (b - f - 1)] = gtimer();
        const int64_t guess = warp_cand_guess<XT, YT>(a, ka, xs, ys, b, anc);
        if (dbg) ka.prof[K3S_GMAX * 8 + 16 + 4 * (b - f - 1) + 1] = gtimer();
        // with group summaries every warp takes the pruned pick on its own (the same
        // result, no CTA barrier: a few groups instead of the whole bucket by 512 threads)
        const int64_t r = ka.gmeta ? grp_pick<1, XT, YT>(a, xs, ys, m, b, anc, guess, nullptr, nullptr, nullptr,
                                                         ka.gmeta + b * K3S_GCAP)
                                   : grp_pick<NW, XT, YT>(a, xs, ys, m, b, anc, guess, s_red, s_a, s_i);
        if (dbg) ka.prof[K3S_GMAX * 8 + 16 + 4 * (b - f - 1) + 2] = gtimer();
        if (dbg) ka.prof[K3S_GMAX * 8 + 16 + 4 * (b - f - 1) + 3] = (unsigned long long)(r == guess);
        k3s_count(6);
        if (t == 0 && b == f + 1) a.best2[b] = r;  // (the sequential walk's speculative pick)
        if (__ldcg(a.flag + b)) {
          if (t == 0) atomicOr(ka.sync + K3S_CONFLICT, 1u);
          break;
        }
        if (r == __ldcg(a.pos + b + 1)) break;  // re-joined the verified chain
        if (t == 0) out[b + 1] = omap(r);
        anc = r;
      }
    }
  }
  // ---- 5: the last CTA to finish: only if deviations interacted, the
  // sequential repair walk over all mismatches (rewrites the output) ----
  __syncthreads();
  if (t == 0) {
    __threadfence();
    s_last = atomicAdd(ka.sync + K3S_DONE, 1u) == G - 1;
  }
  __syncthreads();
  k3s_dbg(22);
  if (!s_last) return;
  __threadfence();
  stamp(6);
  if (*(volatile unsigned*)(ka.sync + K3S_CONFLICT)) {
    repair_walk_smem_p<XT, YT, NT>(a, 0, dsm, [&](int64_t b, int64_t prev, double* sa, long long* si) {
      const int64_t guess = warp_cand_guess<XT, YT>(a, ka, xs, ys, b, prev);
      k3s_count(7);
      return grp_pick<NW, XT, YT>(a, xs, ys, m, b, prev, guess, s_red, sa, si);
    });
  }
  __syncthreads();
  stamp(7);
}

}  // namespace mm
