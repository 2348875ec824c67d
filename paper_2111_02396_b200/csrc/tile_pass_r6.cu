// tile_pass_r6.cu -- instantiations of the K1 tile-pass kernel with 2^6
// amplitudes per thread (see tile_pass.cuh).
#include "tile_pass.cuh"

namespace qt {

cudaError_t launch_tile_pass_r6(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    return launch_tr<12, 6>(a, step, ntiles, nslots, s);
}

}  // namespace qt
