// kernels.hpp -- launch interface of the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "desc.hpp"

namespace qt {

// Arguments of the tile-pass kernel K1 (+ epilogues K2 rho_Q/choose, K3a block
// sums, K4 Pauli partials).  All pointers are device pointers.
struct TileArgs {
    float2* state;              // batch base; slot b at offset b << n
    int n;                      // qubits
    int T;                      // tile bits
    const PassDesc* passes;
    const int32_t* pass_start;  // per slot
    const int32_t* pass_count;  // per slot
    const PassDesc* step_passes = nullptr;  // grid.y -> this step's pass of an active slot (.slot), or
                                            // nullptr: slot = grid.y, pass via pass_start / pass_count
    const GateDesc* gates;
    float2* pool;               // complex64 matrix pool (read by passes, written by choose)
    const EventDesc* events;
    const ChanDesc* chans;
    const double* chan_data;
    double* rho_part;           // [slot][tile][rho_stride]
    int rho_stride;             // doubles per tile partial (2 * dmax^2)
    int32_t* counters;          // per slot, zero-initialized
    int32_t* records;           // chosen Kraus index of recorded channels
    int32_t* status;            // per slot error code (0 = ok)
    double* blocksum;           // [slot][tile]
    double* obs_part;           // [slot][tile][n_obs]
    int n_obs;
    const ObsDesc* obs;
    uint32_t prefetch;          // L2-prefetch the tile this many CTAs ahead (0 = off; set by the launcher)
    unsigned long long* timing = nullptr;  // -DQT_TIMING builds: clock64 phase sums (diagnostics)
    const void* v3maps = nullptr;          // T = 11 (tile_pass_v3.cu): V3Map per tile layout (PassDesc::pad)
};

// TMA description of one 11-qubit tile layout over a batch buffer (tile_pass_v3.cu):
// 5-D tensor map [qubits 0..3 | up to three runs of tile qubits | rest (16 amplitudes)],
// plus the boxes enumerating the tile qubits outside those runs.
struct alignas(64) V3Map {
    CUtensorMap tm;
    int32_t nops;
    uint32_t op_bytes;
    int32_t op_rest[16];  // rest-coordinate offset of box o
};
bool v3_encode_map(void* state, int n, uint64_t nslots, uint64_t tile_mask, V3Map* out);
cudaError_t launch_tile_pass_v3(const TileArgs& a, const void* maps, int step, uint32_t ntiles, int nslots,
                                cudaStream_t s);

// Largest register width R (amplitudes per thread = 2^R) compiled.
constexpr int kMaxR = 6;
constexpr int kMaxT = 13;

size_t tile_pass_smem_bytes(int T, int R, int tck);
// tck: 0 = CUDA-core fused gates; 4 / 5 / 6 = tensor-core gates padded to tck qubits.
cudaError_t launch_tile_pass(const TileArgs& a, int R, int tck, int step, uint32_t ntiles, int nslots,
                             cudaStream_t s);

// max_k: largest fused-gate arity of the call (threads per gate = 2^max_k)
cudaError_t launch_materialize(const FusedDesc* fused, int n_fused, int max_k, const ConsDesc* cons,
                               const VarDesc* vars, const double* var_data, float2* pool,
                               cudaStream_t s);

cudaError_t launch_finalize_obs(const double* blocksum, const double* obs_part, int ntiles,
                                int n_obs, int nslots, double* out_obs, double* out_norm,
                                cudaStream_t s);

cudaError_t launch_init_states(float2* state, int n, int nslots, cudaStream_t s);

cudaError_t launch_sample(const float2* state, int n, int T, const double* blocksum, int nslots,
                          int shots, uint64_t seed, const uint64_t* traj_ids, const double* p00,
                          const double* p11, uint64_t* out_bits, cudaStream_t s, int n_rng = 0,
                          const int32_t* shot_ids = nullptr, double* heap = nullptr);
// registers with at least 2^kHeapMinLg tiles sample through a block-sum heap (2 x tiles doubles per slot)
constexpr int kHeapMinLg = 10;

// dst[pi(i)] = src[i] where bit b of i moves to bit perm[b] (n <= 24).
cudaError_t launch_permute_qubits(const float2* src, float2* dst, int n, const int* perm, cudaStream_t s);

// rho_Q (2^q x 2^q, q <= 6) of the qubits in qmask over a whole n-qubit state;
// partial: 296 x max(32, 2 * 4^q) doubles scratch; out: 2 * 4^q doubles (device).
cudaError_t launch_rho_reduce(const float2* state, int n, uint64_t qmask, int q, double* partial, double* out,
                              cudaStream_t s);

}  // namespace qt
