// fused_x_i32.cu -- fused batch kernel launchers for x = int (see fused_impl.cuh)
#include "fused_impl.cuh"

namespace mmh {

int launch_fused_i32(const FusedArgs& fa, int ydt, cudaStream_t st) { return launch_fused_x<int>(fa, ydt, st); }

}  // namespace mmh
