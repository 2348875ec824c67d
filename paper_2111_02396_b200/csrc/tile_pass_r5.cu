// tile_pass_r5.cu -- K1 tile-pass instantiation, CUDA-core path, 2^5 amplitudes
// per thread, T = 12 (see tile_pass_kernel.cuh).
#include "tile_pass_kernel.cuh"

namespace qt {

cudaError_t launch_tile_pass_r5(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    return launch_tr<12, 5, false>(a, step, ntiles, nslots, s);
}

}  // namespace qt
