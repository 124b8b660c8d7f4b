// lttb_x_f32.cu -- K3 launchers for x = float, buckets > 64 points (K3s / K3c; see lttb_impl.cuh)
#include "lttb_impl.cuh"

namespace mmh {

int launch_lttb_small_f32(LttbArgs a, int ydt, int64_t s, cudaStream_t st);  // lttb_small_x_f32.cu

int launch_lttb_f32(LttbArgs a, int ydt, int64_t s, cudaStream_t st) {
  if (use_tables(s)) return launch_lttb_small_f32(a, ydt, s, st);
  return launch_lttb_large_x<float>(a, ydt, st);
}

// k_lttb_repair's counter is a per-translation-unit device variable
int64_t repair_scans_f32() {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, g_repair_scans, sizeof v) != cudaSuccess) return -1;
  return (int64_t)v;
}

}  // namespace mmh
