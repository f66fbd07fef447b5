// sweep_f32_bwd.cu -- explicit instantiation of the fused sweep (float, adjoint).
#include "sweep_impl.cuh"

namespace qfb {

cudaError_t launch_sweep_f32_bwd(const SweepArgs& a, int batch, size_t smem, cudaStream_t s) {
    switch (a.sw.R) {
        case 1: return launch_sweep_t<float, 1, true>(a, batch, smem, s);
        case 2: return launch_sweep_t<float, 2, true>(a, batch, smem, s);
        case 3: return launch_sweep_t<float, 3, true>(a, batch, smem, s);
        case 4: return launch_sweep_t<float, 4, true>(a, batch, smem, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qfb
