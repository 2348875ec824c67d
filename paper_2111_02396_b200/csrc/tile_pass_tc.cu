// tile_pass_tc.cu -- K1 tile-pass instantiation, tensor-core path, T = 12, 128
// threads (R = 5): fused gates padded to 4 qubits (f16 runs / 3xTF32 single gates,
// four CTAs per SM); 5- and 6-qubit gates live in tile_pass_tcw.cu.  See
// tile_pass_kernel.cuh and tc_common.cuh.
#include "tile_pass_kernel.cuh"

namespace qt {

cudaError_t launch_tile_pass_tcw(const TileArgs& a, int tck, int step, uint32_t ntiles, int nslots, cudaStream_t s);

cudaError_t launch_tile_pass_tc(const TileArgs& a, int tck, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    if (tck == 5 || tck == 6) return launch_tile_pass_tcw(a, tck, step, ntiles, nslots, s);
    return launch_tr<12, 5, true, 4>(a, step, ntiles, nslots, s);
}

}  // namespace qt

#ifdef QT_TIMING
extern "C" int qt_timing_read(unsigned long long* host16) {
    return (int)cudaMemcpy(host16, qt::timing_buffer(), 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}
#endif
