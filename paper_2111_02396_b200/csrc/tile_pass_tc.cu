// tile_pass_tc.cu -- K1 tile-pass instantiations, tensor-core path (tcgen05 3xTF32),
// T = 12: R = 4 (256 threads, one subvector per thread, default) and R = 5
// (128 threads, two subvectors per thread).  See tile_pass_kernel.cuh, tc_common.cuh.
#include "tile_pass_kernel.cuh"

namespace qt {

cudaError_t launch_tile_pass_tc(const TileArgs& a, int R, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    if (R == 5) return launch_tr<12, 5, true>(a, step, ntiles, nslots, s);
    return launch_tr<12, 4, true>(a, step, ntiles, nslots, s);
}

}  // namespace qt
