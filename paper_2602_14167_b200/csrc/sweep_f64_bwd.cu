// sweep_f64_bwd.cu -- explicit instantiation of the fused sweep (double, adjoint).
#include "sweep_impl.cuh"

namespace qfb {

cudaError_t launch_sweep_f64_bwd(const SweepArgs& a, int batch, size_t smem, cudaStream_t s) {
    switch (a.sw.R) {
        case 1: return launch_sweep_t<double, 1, true>(a, batch, smem, s);
        case 2: return launch_sweep_t<double, 2, true>(a, batch, smem, s);
        case 3: return launch_sweep_t<double, 3, true>(a, batch, smem, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qfb
