// k1_launch.cu -- K1 (sub-bucket extrema) launch: kernel variant dispatch.
#include "host.cuh"

namespace mmh {

int launch_extrema(const ExArgs& a, int ydt, cudaStream_t st) {
  if (a.E > 0) {  // flat split
    if (!a.arrivals_zeroed && cudaMemsetAsync(a.arrivals, 0, (size_t)(a.B * a.nb) * sizeof(unsigned), st) != cudaSuccess)
      return fail(MM_ECUDA, "cudaMemsetAsync(arrivals)");
    const int64_t blocks = a.ticket ? std::min<int64_t>(cdiv(a.B * a.Ws, 8), (int64_t)sm_count() * 3) : cdiv(a.B * a.Ws, 8);
    if (ydt == MM_F32) {
#ifdef MMLTTB_AB  // tuning build only (tools/flat_sweep.sh)
      static const int64_t fv = env_i64("MMLTTB_K1_FLAT_VARIANT", 0);
      switch (fv) {
        case 1: k_extrema_flat<float, 6, 3, 4><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        case 2: k_extrema_flat<float, 4, 3, 4><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        case 3: k_extrema_flat<float, 8, 1, 3><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        case 4: k_extrema_flat<float, 12, 3, 2><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        case 5: k_extrema_flat<float, 16, 3, 2><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        // register double-buffered rounds (round i+1's loads in flight while round i is reduced):
        // C3 K1 77.1 us at 2 CTAs / SM, 81.8 us with 4-vector rounds at 3, vs 72.9 us; 1e9 611 / 658 vs 575 us
        case 6: k_extrema_flat<float, 8, 3, 2, true><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        case 7: k_extrema_flat<float, 4, 3, 3, true><<<(unsigned)blocks, 256, 0, st>>>(a); break;
        default: k_extrema_flat<float, 8, 3><<<(unsigned)blocks, 256, 0, st>>>(a); break;
      }
#else
      if (a.ticket) k_extrema_flat<float, 8, 3, 3, false, true><<<(unsigned)blocks, 256, 0, st>>>(a);
      else k_extrema_flat<float, 8, 3><<<(unsigned)blocks, 256, 0, st>>>(a);
#endif
    } else {
      if (a.ticket) k_extrema_flat<double, 8, 3, 3, false, true><<<(unsigned)blocks, 256, 0, st>>>(a);
      else k_extrema_flat<double, 8, 3><<<(unsigned)blocks, 256, 0, st>>>(a);
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
  if (a.C > 1 && !a.arrivals_zeroed && cudaMemsetAsync(a.arrivals, 0, (size_t)(a.B * a.nb) * sizeof(unsigned), st) != cudaSuccess)
    return fail(MM_ECUDA, "cudaMemsetAsync(arrivals)");
  const int64_t blocks = cdiv(warps, 8);
  if (blocks > 0x7fffffffLL) return fail(MM_ERANGE, "extrema grid too large");
  if (a.chunk >= (1LL << 30)) return fail(MM_ERANGE, "bucket chunk too large");
  const unsigned g = (unsigned)blocks;
#ifdef MMLTTB_AB  // tuning build only (tools/k1_sweep.sh)
  static const int variant = [] {
    const char* e = getenv("MMLTTB_K1_VARIANT");  // tuning knob, default = tuned choice
    return e ? atoi(e) : 0;
  }();
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
#else
  if (ydt == MM_F32)
    k_extrema<float, 8, 3><<<g, 256, 0, st>>>(a);  // tuned: U=8 vectors in flight, evict-first
  else
    k_extrema<double, 8, 3><<<g, 256, 0, st>>>(a);
#endif
  return check_launch("k_extrema");
}


}  // namespace mmh
