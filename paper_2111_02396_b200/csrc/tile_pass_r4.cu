// tile_pass_r4.cu -- K1 tile-pass instantiations, CUDA-core path, 2^4 amplitudes
// per thread (T = 12) and the whole-state tiles of n < 12 (see tile_pass_kernel.cuh).
#include "tile_pass_kernel.cuh"

namespace qt {

cudaError_t launch_tile_pass_r4(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    switch (a.T) {
        case 1: return launch_tr<1, 1, false>(a, step, ntiles, nslots, s);
        case 2: return launch_tr<2, 2, false>(a, step, ntiles, nslots, s);
        case 3: return launch_tr<3, 3, false>(a, step, ntiles, nslots, s);
        case 4: return launch_tr<4, 4, false>(a, step, ntiles, nslots, s);
        case 5: return launch_tr<5, 4, false>(a, step, ntiles, nslots, s);
        case 6: return launch_tr<6, 4, false>(a, step, ntiles, nslots, s);
        case 7: return launch_tr<7, 4, false>(a, step, ntiles, nslots, s);
        case 8: return launch_tr<8, 4, false>(a, step, ntiles, nslots, s);
        case 9: return launch_tr<9, 4, false>(a, step, ntiles, nslots, s);
        case 10: return launch_tr<10, 4, false>(a, step, ntiles, nslots, s);
        case 11: return launch_tr<11, 4, false>(a, step, ntiles, nslots, s);
        case 12: return launch_tr<12, 4, false>(a, step, ntiles, nslots, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace qt
