// lttb_x_i32.cu -- K3 launchers for x = int, buckets > 64 points (K3s / K3c; see lttb_impl.cuh)
#include "lttb_impl.cuh"

namespace mmh {

int launch_lttb_small_i32(LttbArgs a, int ydt, int64_t s, cudaStream_t st);  // lttb_small_x_i32.cu

int launch_lttb_i32(LttbArgs a, int ydt, int64_t s, cudaStream_t st) {
  if (use_tables(s)) return launch_lttb_small_i32(a, ydt, s, st);
  return launch_lttb_large_x<int>(a, ydt, st);
}

// k_lttb_repair's counter is a per-translation-unit device variable
int64_t repair_scans_i32() {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, g_repair_scans, sizeof v) != cudaSuccess) return -1;
  return (int64_t)v;
}

}  // namespace mmh
