// lttb_small_x_f32.cu -- K3a launchers (LTTB buckets <= 64 points) for x = float
// (a separate translation unit: the build compiles the K3 variants in parallel)
#include "lttb_impl.cuh"

namespace mmh {

int launch_lttb_small_f32(LttbArgs a, int ydt, int64_t s, cudaStream_t st) { return launch_lttb_small_x<float>(a, ydt, s, st); }

}  // namespace mmh
