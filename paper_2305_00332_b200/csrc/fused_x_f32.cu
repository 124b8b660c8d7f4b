// fused_x_f32.cu -- fused batch kernel launchers for x = float (see fused_impl.cuh)
#include "fused_impl.cuh"

namespace mmh {

int launch_fused_f32(const FusedArgs& fa, int ydt, cudaStream_t st) { return launch_fused_x<float>(fa, ydt, st); }

}  // namespace mmh
