// tile_pass_r5.cu -- instantiations of the K1 tile-pass kernel with 2^5
// amplitudes per thread (see tile_pass.cuh).
#include "tile_pass.cuh"

namespace qt {

cudaError_t launch_tile_pass_r5(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    return launch_tr<12, 5>(a, step, ntiles, nslots, s);
}

}  // namespace qt
