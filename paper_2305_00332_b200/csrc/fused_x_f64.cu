// fused_x_f64.cu -- fused batch kernel launchers for x = double (see fused_impl.cuh)
#include "fused_impl.cuh"

namespace mmh {

int launch_fused_f64(const FusedArgs& fa, int ydt, cudaStream_t st) { return launch_fused_x<double>(fa, ydt, st); }

}  // namespace mmh
