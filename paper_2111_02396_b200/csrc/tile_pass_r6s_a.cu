// tile_pass_r6s_a.cu -- K1 tile-pass instantiations, CUDA-core path, 2^6 amplitudes
// per thread for whole-state tiles of n < 12 qubits (T = n) holding 6-qubit fused gates.
#include "tile_pass_kernel.cuh"

namespace qt {

cudaError_t launch_tile_pass_r6s_a(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    switch (a.T) {
        case 6: return launch_tr<6, 6, false>(a, step, ntiles, nslots, s);
        case 7: return launch_tr<7, 6, false>(a, step, ntiles, nslots, s);
        case 8: return launch_tr<8, 6, false>(a, step, ntiles, nslots, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qt
