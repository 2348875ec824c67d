// desc.hpp -- device descriptors shared by the host planner (plan.cpp) and the
// sm_100a kernels (kernels.cu).  Plain structs, no methods.
#pragma once
#include <stdint.h>

namespace qt {

// Pass flags.
enum : int32_t {
    kPassStore = 1,   // write the tile back to HBM (gate passes)
    kPassRho = 2,     // epilogue: rho_Q partial of a conventional channel + choose
    kPassFinal = 4,   // epilogue: block sums |psi|^2 (tile = low T qubits) for the sampler/norm
    kPassObs = 8,     // epilogue: Pauli-string partial sums
    kPassInit = 16,   // the tile starts as |0...0> (first pass of a trajectory): no HBM load, always stores
};

// One tile pass of one trajectory (Sec. III.A Alg. 1 generalized: every CTA
// owns the 2^T amplitudes spanned by tile_mask for one value of the other bits
// and applies gate_count fused gates to them in shared memory / registers).
struct PassDesc {
    uint64_t tile_mask;   // global qubits of the tile, popcount == T
    int32_t gate_begin;   // into GateDesc[]
    int32_t gate_count;
    int32_t flags;
    int32_t event;        // EventDesc index (kPassRho) or -1
    int32_t obs_begin;    // into ObsDesc[] (kPassObs)
    int32_t obs_count;
    uint8_t tq[16];       // global qubit of tile bit i (ascending), i < T
    int32_t slot;         // batch slot (set by the executor in the per-step launch arrays)
    uint32_t rho_local = 0;  // kPassRho: the channel's qubits as tile-local bits
    int32_t rho_nq = 0;      // kPassRho: channel arity
    int32_t pad = 0;
};
static_assert(sizeof(PassDesc) == 64, "PassDesc layout");

// A fused gate inside a pass and the register layout used to apply it:
// register bit m of a thread's 2^R amplitudes <-> tile-local bit rpos[m]
// (m < k: the gate's qubits ascending, so matrix bit m <-> register bit m;
// m >= k: filler bits), thread-index bit i <-> tile-local bit tpos[i].
// 4 bits per entry.
//
// Tensor-core gates (kGateTC, 4 qubits) form RUNS inside a pass: the first
// gate of a run (kGateRunStart) converts the fp32 tile to the f16 hi/lo GEMM
// operand layout of tc_common.cuh (with a power-of-two tile scale, 2^-shift
// extra headroom for norm-increasing matrices), and every gate of the run
// writes its output directly in the operand layout of the next gate: xu[r]
// is the byte offset, in the next gate's operand layout, of this gate's
// layout role r (r < 4: matrix bit r, r = 4: group bit, r = 5 + i: thread
// bit i).  The last gate of a run writes the fp32 tile back.
struct GateDesc {
    int32_t mat_off;      // complex64 offset into the matrix pool (16-byte aligned)
    int32_t k;            // arity | kGateTC | kGateRunStart | shift << 16
    uint32_t rpos;
    uint32_t tpos;
    uint16_t xu[12];      // TC runs: next-gate operand offsets of this gate's roles
    int32_t pair;         // TC runs: outputs c, c ^ 1 share a 16-byte chunk of the next operand
    uint32_t pad;
};
static_assert(sizeof(GateDesc) == 48, "GateDesc layout");

// Largest number of fused gates in one pass (descriptors staged in smem).
constexpr int kMaxPassGates = 64;

// GateDesc::k / FusedDesc::k flag: a (4- or 5-qubit padded) gate applied on
// tensor cores whose pool entry is the GEMM operand W (tc_common.cuh).
constexpr int32_t kGateTC = 0x100;
constexpr int32_t kGateRunStart = 0x200;  // first gate of a tensor-core run
constexpr int32_t kGateF16 = 0x400;       // 4-qubit gate of a run of >= 2: f16 operands (else 3xTF32)
constexpr int kGateShiftBit = 16;         // bits 16..23: run scale headroom (log2)
// Persistent TMEM kernel (tile_pass_v2.cu, T = 13 tiles, 4-qubit gates):
//   rpos nibbles 0..3 = tile bits of matrix bits 0..3 (config), 4..5 = group bits;
//   tpos nibbles 0..6 = tile bits of TMEM lane bits 0..4 and warp bits 0..1;
//   kGateRunStart: gather the fp32 tile into TMEM operand A (new f16 tile scale);
//   kGateRunEnd: write D back to the fp32 tile; otherwise xu[0..5] = TMEM column
//   offset, in this gate's D, of the next gate's config bits 0..3 / group bits 0..1.
//   The 40 bytes after `k` of a v2 gate are 20 uint16 (v2_units): [0..3] fp32-tile byte
//   offsets of the config bits, [4..5] of the group bits, [6..12] of the row bits
//   (TMEM lane bits 0..4, warp bits 0..1), [13..18] = xu (next-gate source columns).
constexpr int32_t kGateV2 = 0x800;
#ifdef __CUDACC__
#define QT_DESC_HD __host__ __device__
#else
#define QT_DESC_HD
#endif
QT_DESC_HD inline uint16_t* v2_units(GateDesc& g) { return reinterpret_cast<uint16_t*>(&g.rpos); }
QT_DESC_HD inline const uint16_t* v2_units(const GateDesc& g) { return reinterpret_cast<const uint16_t*>(&g.rpos); }
constexpr int32_t kGateRunEnd = 0x1000;
constexpr int32_t kGateXNext = 0x2000;  // v2: the transition to the next gate is an X (16x256b) transposition
// v2: matrix bit 0 is tile bit 0, so configurations c, c ^ 1 are one 16-byte pair of
// the fp32 tile (gather / write-back by 16-byte shared-memory accesses)
constexpr int32_t kGatePair0 = 0x4000;
// Pool bytes of a v2 gate operand: B = 32 rows x [W_hi (32 f16) | W_lo (32 f16)], SWIZZLE_128B.
constexpr int kV2GateBytes = 4096;
// Pool bytes of a tensor-core gate operand padded to k qubits (tc_common.cuh
// gate_bytes): 4 -> f16 B or tf32 hi/lo W (8 KB), 5 -> f16 hi/lo B (16 KB),
// 6 -> f16 hi/lo B in two K-chunks of 256 rows (64 KB).
constexpr int tc_gate_bytes(int k) { return k <= 4 ? 8192 : (k == 5 ? 16384 : 65536); }

// A conventional channel occurrence (Alg. 2 lines 12-21).
struct EventDesc {
    int32_t chan;         // ChanDesc index
    int32_t mat_off;      // pool slot receiving K_i / sqrt(raw p_i) (complex64)
    int32_t record;       // index into the record array, or -1
    int32_t slot;         // batch slot of the trajectory
    double r;             // remaining uniform after the first loop
    int32_t flags;        // kEventNoBounds: conventional algorithm, pbar_i = 0
    int32_t pad;
};
constexpr int32_t kEventNoBounds = 1;

// Channel data for the device choose step (fp64 in chan_data):
//   pbar[n_kraus], then M_i = K_i^dag K_i (2*d*d doubles each), then K_i.
struct ChanDesc {
    uint64_t qmask;       // global qubits of the channel
    int32_t d;
    int32_t n_kraus;
    int32_t off;          // double offset into chan_data
    int32_t nq;
};

// Fused-gate materialization: product of constituents (Sec. III.B).
struct FusedDesc {
    int32_t mat_off;      // complex64 pool offset
    int32_t k;
    int32_t cons_begin;
    int32_t cons_count;
};

// One constituent: variant `var`, its qubits' positions inside the fused
// gate's sorted qubit list (4 bits each), nq in bits 24..27.
struct ConsDesc {
    int32_t var;
    uint32_t pos;
};

struct VarDesc {
    int32_t off;          // complex128 offset into var_data (double2 units)
    int32_t nq;
};

// Pauli observable: phase(L) = i^ny (-1)^popcount(L & zmask), P|L> = phase |L ^ xmask>.
struct ObsDesc {
    uint64_t xmask;
    uint64_t zmask;
    int32_t ny;
    int32_t slot;         // column in the per-trajectory observable array
};

}  // namespace qt
