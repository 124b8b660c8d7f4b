// lttb_x_i64.cu -- K3 launchers for x = long long (see lttb_impl.cuh)
#include "lttb_impl.cuh"

namespace mmh {

int launch_lttb_i64(LttbArgs a, int ydt, int64_t s, cudaStream_t st) { return launch_lttb_x<long long>(a, ydt, s, st); }

// k_lttb_repair's counter is a per-translation-unit device variable
int64_t repair_scans_i64() {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, g_repair_scans, sizeof v) != cudaSuccess) return -1;
  return (int64_t)v;
}

}  // namespace mmh
