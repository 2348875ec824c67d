// tile_pass_r6s_b.cu -- K1 tile-pass instantiations, CUDA-core path, 2^6 amplitudes
// per thread for whole-state tiles of n < 12 qubits (T = n) holding 6-qubit fused gates.
#include "tile_pass_kernel.cuh"

namespace qt {

cudaError_t launch_tile_pass_r6s_b(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    switch (a.T) {
        case 9: return launch_tr<9, 6, false>(a, step, ntiles, nslots, s);
        case 10: return launch_tr<10, 6, false>(a, step, ntiles, nslots, s);
        case 11: return launch_tr<11, 6, false>(a, step, ntiles, nslots, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qt
