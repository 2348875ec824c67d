// tile_pass_r5s.cu -- K1 tile-pass instantiations, CUDA-core path, 2^5 amplitudes
// per thread for whole-state tiles of n < 12 qubits (T = n) holding 5-qubit fused gates.
#include "tile_pass_kernel.cuh"

namespace qt {

cudaError_t launch_tile_pass_r5s(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    switch (a.T) {
        case 5: return launch_tr<5, 5, false>(a, step, ntiles, nslots, s);
        case 6: return launch_tr<6, 5, false>(a, step, ntiles, nslots, s);
        case 7: return launch_tr<7, 5, false>(a, step, ntiles, nslots, s);
        case 8: return launch_tr<8, 5, false>(a, step, ntiles, nslots, s);
        case 9: return launch_tr<9, 5, false>(a, step, ntiles, nslots, s);
        case 10: return launch_tr<10, 5, false>(a, step, ntiles, nslots, s);
        case 11: return launch_tr<11, 5, false>(a, step, ntiles, nslots, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qt
