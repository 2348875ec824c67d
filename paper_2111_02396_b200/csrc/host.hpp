// host.hpp -- host-side data structures of libqtraj (circuit IR, plan,
// per-trajectory programs).  Internal; the public surface is include/qtraj.h.
#pragma once
#include <array>
#include <complex>
#include <cstdint>
#include <string>
#include <memory>
#include <vector>

#include "../../include/qtraj.h"
#include "desc.hpp"
#include <cuda_runtime_api.h>

namespace qt {

using cd = std::complex<double>;

void set_error(const std::string& msg);

// One operation of the circuit, canonicalized: qubits sorted ascending and
// matrices re-indexed so matrix bit m <-> the m-th lowest qubit.
struct HostOp {
    int kind = 0;  // 0 = gate, 1 = channel
    int moment = 0;
    int seq = 0;   // call order
    int nq = 0;
    int q[6] = {0, 0, 0, 0, 0, 0};
    uint64_t mask = 0;
    int n_kraus = 1;       // channel: Kraus operators; gate: parameter sets (1 = plain gate)
    int record = 0;
    std::vector<cd> mats;  // n_kraus * d * d (internal order)
};

const HostOp* circuit_op(const qt_circuit_s* c, int i);
// streaming single-gate pass (gate_stream.cu); cudaErrorNotSupported if n < 7 + max(nq, 4)
cudaError_t gate_stream_apply(cudaStream_t s, void* state, int n, int nq, const int* qs, const cd* U, int repeats,
                              double* kernel_ms);

struct Circuit {
    int n = 0;
    std::vector<HostOp> ops;
    std::vector<double> p00, p11;
    int seq = 0;
    int n_sets = 1;  // parameter sets of sweep gates; trajectory t uses set t mod n_sets
};

// Plan-level operation (canonical order) with channel preprocessing.
struct PlanOp {
    int kind = 0;
    int nq = 0;
    int q[6] = {0, 0, 0, 0, 0, 0};
    uint64_t mask = 0;
    int var_base = 0;   // first variant (gate: its matrix; channel: deferred op i)
    int n_kraus = 1;
    int chan = -1;      // channel ordinal (RNG counter) / ChanDesc index
    int record = -1;    // record column or -1
    bool mixture = false;
    std::vector<double> pbar;
    double s = 0.0;
};

struct Variant {
    int nq = 0;
    bool identity = false;
    double norm = 1.0;  // upper bound on the spectral norm (1 for unitaries and Kraus operators)
};

struct Plan {
    int n = 0;
    int f = 4;          // max fuse size (Sec. III.B)
    int T = 12;         // tile bits
    int CL = 4;         // low qubits always in a tile
    int R = 4;          // register bits (2^R amplitudes / thread)
    bool one_gate = false;
    bool tc = false;    // fused gates padded to tc_k qubits and applied on tcgen05 tensor cores
    int tc_k = 4;       // 4 (f <= 4), 5 (f = 5) or 6 (f = 6)
    bool v3 = false;    // tile_bits = 11: TMA-pipelined kernel (tile_pass_v3.cu), 4-qubit tensor-core gates
    bool v2 = false;    // tc_k == 4 on n >= 13 qubits: T = 13 tiles, persistent TMEM kernel (tile_pass_v2.cu)
    std::vector<PlanOp> ops;
    std::vector<Variant> vars;
    std::vector<VarDesc> var_desc;
    std::vector<double> var_data;   // complex128 interleaved
    std::vector<ChanDesc> chans;
    std::vector<double> chan_data;
    int n_channels = 0;
    int n_recorded = 0;
    int max_conv_d = 1;             // largest d of a non-mixture channel
    int max_chan_d = 1;             // largest d of any channel (conventional mode)
    int n_sets = 1;                 // parameter sets (sweep gates pick variant traj mod n_sets)
    std::vector<double> p00, p11;
    bool has_p00 = false, has_p11 = false;
};

// Switch a plan to the FP32 CUDA-core kernel (4..6-qubit conventional channels, huge norms).
void cuda_core_plan(Plan& P);

// Kraus lower bound sigma_min(K)^2 of a d x d matrix.
double lower_bound(int d, const cd* K);

// ---------------------------------------------------------------------------
// Per-trajectory program produced by the planner (planner.cpp).
// Offsets inside are local to the trajectory; the executor rebases them.
// ---------------------------------------------------------------------------
struct TrajProgram {
    std::vector<PassDesc> passes;
    std::vector<GateDesc> gates;      // mat_off local to the trajectory pool region
    std::vector<FusedDesc> fused;     // mat_off local; cons_begin local
    std::vector<ConsDesc> cons;
    std::vector<EventDesc> events;    // mat_off local; record local column
    std::vector<int32_t> records;     // n_recorded (deferred picks; -1 = conventional, filled on device)
    int32_t pool_size = 0;            // complex64 entries
    uint64_t n_deferred = 0, n_conventional = 0;
    double alg_bytes = 0, alg_flops = 0;
};

struct ObsSpec {
    uint64_t x = 0, z = 0;
    int ny = 0;
};

// Observables grouped by the tile they need: group 0 is evaluated on the
// final pass (tile = low T qubits), group k > 0 on a read-only pass with tile
// masks[k].  ranges[k] = (first, count) into the call's ObsDesc table.
struct ObsGroups {
    std::vector<std::pair<int, int>> ranges;
    std::vector<uint64_t> masks;
    bool final_pass = true;  // false: gate passes only (qt_apply_gate)
};

// Build the program of trajectory `traj` (Alg. 2 first loop on the host,
// fusion, tile passes, epilogues).  Returns QT_OK or an error status.
// mode 0 = Alg. 2 (delayed inner products), 1 = conventional algorithm.
qt_status plan_trajectory(const Plan& P, uint64_t seed, uint64_t traj,
                          const ObsGroups& og, TrajProgram& out, int mode = 0);

// Paper's two-phase fuser on a list of items (exposed for tests).
struct FuseItem {
    uint64_t mask;
    bool fixed;  // never merged (device-chosen conventional op)
};
// Returns fused gates as lists of item indices (time order inside each).
// Two-phase fuser: fused gate j = items flat[offs[j] .. offs[j + 1]) in time order.
void fuse_items(const FuseItem* items, int N, int f, std::vector<int>& flat, std::vector<int>& offs);

}  // namespace qt
