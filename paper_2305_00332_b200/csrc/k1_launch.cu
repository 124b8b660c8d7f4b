// k1_launch.cu -- K1 (sub-bucket extrema) launch: kernel variant dispatch.
#include "host.cuh"
#ifdef MMLTTB_AB
#include "k1_tiles.cuh"
#endif

namespace mmh {

int launch_extrema(const ExArgs& a, int ydt, cudaStream_t st) {
#ifdef MMLTTB_AB
  if (a.nt > 0) {  // tile mode (k1_tiles.cuh; tuning build only)
    const int64_t blocks = a.B * a.nt;
    if (blocks > 0x7fffffffLL) return fail(MM_ERANGE, "extrema grid too large");
    ExArgs t = a;
    t.e_lo = t.start + (t.b0 * t.len) / t.k;  // pbound (core.py:173)
    t.e_hi = t.start + ((t.b0 + t.nb) * t.len) / t.k;
    t.rlen = 1.0 / (double)t.len;
    t.rk = 1.0 / (double)t.k;
    if (ydt == MM_F32)
      k_extrema_tiles<float><<<(unsigned)blocks, K1T_NT, 0, st>>>(t);
    else
      k_extrema_tiles<double><<<(unsigned)blocks, K1T_NT, 0, st>>>(t);
    if (int rc = check_launch("k_extrema_tiles")) return rc;
    // the multi-tile sub-buckets' partials: a programmatic dependent launch
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)cdiv(a.B * a.nb, 256));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = ydt == MM_F32 ? cudaLaunchKernelEx(&cfg, k_extrema_tiles_combine<float>, t)
                                        : cudaLaunchKernelEx(&cfg, k_extrema_tiles_combine<double>, t);
    if (e != cudaSuccess) { (void)cudaGetLastError(); return fail(MM_ECUDA, "k_extrema_tiles_combine: %s", cudaGetErrorString(e)); }
    return check_launch("k_extrema_tiles_combine");
  }
#endif
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
