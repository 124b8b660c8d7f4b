// lttb_small_x_i64.cu -- K3a launchers (LTTB buckets <= 64 points) for x = long long
// (a separate translation unit: the build compiles the K3 variants in parallel)
#include "lttb_impl.cuh"

namespace mmh {

int launch_lttb_small_i64(LttbArgs a, int ydt, int64_t s, cudaStream_t st) { return launch_lttb_small_x<long long>(a, ydt, s, st); }

}  // namespace mmh
