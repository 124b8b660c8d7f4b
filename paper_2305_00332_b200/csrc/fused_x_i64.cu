// fused_x_i64.cu -- fused batch kernel launchers for x = long long (see fused_impl.cuh)
#include "fused_impl.cuh"

namespace mmh {

int launch_fused_i64(const FusedArgs& fa, int ydt, cudaStream_t st) { return launch_fused_x<long long>(fa, ydt, st); }

}  // namespace mmh
