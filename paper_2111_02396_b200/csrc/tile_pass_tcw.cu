// tile_pass_tcw.cu -- K1 tile-pass instantiations for "wide" tensor-core gates:
// fused gates padded to 5 qubits (f = 5; three CTAs per SM) or 6 qubits (f = 6;
// two CTAs per SM, one 64 KB operand buffer), kind::f16 hi / lo GEMMs
// (tc_common.cuh, tile_pass_kernel.cuh apply_tc_wide).
#include "tile_pass_kernel.cuh"

namespace qt {

cudaError_t launch_tile_pass_tcw(const TileArgs& a, int tck, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    if (tck == 6) return launch_tr<12, 5, true, 6>(a, step, ntiles, nslots, s);
    return launch_tr<12, 5, true, 5>(a, step, ntiles, nslots, s);
}

}  // namespace qt
