/*
 * qtraj.h -- C ABI of libqtraj, the B200 (sm_100a) noisy quantum-trajectory
 * hot path of arXiv 2111.02396 (qsim + Cirq approximate-noise simulation).
 *
 * Citations: P:N = PAPER.md line N (section / algorithm given alongside).
 *
 * Problem statement (Sec. II; Sec. III.E):
 *   A circuit is an ordered list of moments; a moment holds operations on
 *   disjoint qubits.  An operation is a unitary gate or a quantum
 *   channel given by its Kraus operators {K_i}.  A quantum
 *   trajectory picks one K_i per channel with probability
 *   p_i = <Psi|K_i^dag K_i|Psi>, using the delayed-inner-product
 *   sampler of Alg. 2: lower bounds pbar_i = sigma_min(K_i)^2,
 *   s = sum pbar_i; a uniform r < s picks by the bounds and defers the
 *   operator into gate fusion (Sec. III.B); otherwise all pending
 *   operators are applied and p_i is computed.
 *
 * Conventions:
 *   - qubit q <-> amplitude-index bit q (qubit 0 has stride 1).  State is
 *     complex64, interleaved (re, im), 8 * 2^n bytes.
 *   - every matrix argument is complex128, row-major, interleaved (re, im),
 *     of size 2^nq x 2^nq, in KRONECKER order of the listed qubits:
 *     qubits[0] is the most significant matrix-index bit.
 *   - canonical op order: moments ascending, then call order within a moment.
 *   - bitstrings are uint64 with bit q = qubit q (n <= 63).
 *   - RNG: Philox4x32-10, key = (seed_lo32, seed_hi32), counter =
 *     (ordinal, purpose, traj_lo32, traj_hi32); purpose 1 = channel draw
 *     (ordinal = channel ordinal), 2 = sample, 3 = readout (ordinal =
 *     shot*ceil(n/2) + level/2, half level%2).  Results are a pure function of
 *     (circuit, plan options, seed, trajectory index): independent of batch
 *     size, stream and GPU count.
 *
 * Ownership: inputs are copied at call time.  Handles are library-owned and
 * freed by *_destroy.  State buffers are CALLER-OWNED device memory (e.g. a
 * torch tensor) used on the caller's stream; the library never frees them.
 * Host outputs go into caller-allocated arrays.
 *
 * Errors: functions return a qt_status; negative = failure, with a message
 * available from qt_last_error() (thread-local).  Nothing aborts.
 * The library never falls back to a CPU implementation: without a usable
 * CUDA device every device entry point returns QT_ECUDA.
 */
#ifndef QTRAJ_H
#define QTRAJ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    QT_OK = 0,
    QT_EINVAL = -1,       /* bad argument (null pointer, size, option) */
    QT_EQUBIT = -2,       /* qubit out of range, or duplicated in one moment */
    QT_EARITY = -3,       /* nq > 6, or max_fused outside [2, 6] */
    QT_ENONUNITARY = -4,  /* gate: ||U^dag U - I||_max >= 1e-9 */
    QT_ENONCPTP = -5,     /* channel: ||sum K^dag K - I||_max >= 1e-9 */
    QT_EOOM = -6,         /* device or host allocation failed / buffer too small */
    QT_ECUDA = -7,        /* CUDA runtime error or no device */
    QT_ENCCL = -8,        /* reserved for the multi-GPU layer */
    QT_ELEAK = -9,        /* Alg. 2 second loop fell through with residual > 1e-6 */
    QT_ESTATE = -10       /* zero-norm state */
} qt_status;

typedef struct qt_ctx_s* qt_ctx;
typedef struct qt_circuit_s* qt_circuit;
typedef struct qt_plan_s* qt_plan;

/* Counters of one qt_run_trajectories call (SURVEY 5 "Metrics"). */
typedef struct {
    uint64_t trajectories;
    uint64_t passes;              /* tile passes executed (sum over trajectories) */
    uint64_t fused_gates;         /* fused gates applied (sum over trajectories) */
    uint64_t reductions;          /* rho_Q reductions = conventional channels */
    uint64_t channels_deferred;   /* Alg. 2 first-loop picks */
    uint64_t channels_conventional;
    uint64_t launches;            /* kernels launched by the library */
    double   alg_bytes;           /* algorithmic HBM bytes: 2^(n+4) per gate pass, 2^(n+3) per read-only pass */
    double   alg_flops;           /* 2^(n+k+3) per fused k-qubit gate */
    double   plan_ms;             /* host planning wall time */
    double   device_ms;           /* stream time of the whole call (CUDA events) */
    double   pass_kernel_ms;      /* sum of tile-pass kernel durations (profile mode only) */
    uint64_t pass_launches;       /* tile-pass kernel launches timed in profile mode */
    uint64_t h2d_bytes;           /* host->device bytes copied by the call (tables + programs) */
    uint64_t d2h_bytes;           /* device->host bytes copied by the call (records) */
} qt_stats;

/* ---- context -------------------------------------------------------------
 * device: CUDA ordinal; cuda_stream: a cudaStream_t (NULL = legacy default).
 * All device work of the context is enqueued on that stream. */
qt_status qt_ctx_create(int device, void* cuda_stream, qt_ctx* out);
void qt_ctx_destroy(qt_ctx ctx);
qt_status qt_ctx_set_stream(qt_ctx ctx, void* cuda_stream);

/* ---- circuit upload -------------------------------------------
 * qt_add_gate: U is 2^nq x 2^nq complex128, Kronecker order of qubits[].
 *   Rejects non-unitary input (QT_ENONUNITARY, tolerance 1e-9).
 * qt_add_channel: K holds n_kraus matrices of 2^nq x 2^nq, same layout, in
 *   Kraus-list order (the order Alg. 2 iterates).  Rejects
 *   non-trace-preserving lists (QT_ENONCPTP, 1e-9).  record != 0 makes the
 *   chosen index appear in out_kraus of qt_run_trajectories (measurement key,
 *   P:102).
 * Qubits of the operations of one moment must be disjoint: QT_EQUBIT. */
qt_status qt_circuit_create(int n_qubits, qt_circuit* out);
void qt_circuit_destroy(qt_circuit c);
qt_status qt_add_gate(qt_circuit c, int moment, int nq, const int* qubits, const double* U);
qt_status qt_add_channel(qt_circuit c, int moment, int nq, const int* qubits, int n_kraus,
                         const double* K, int record);
/* Readout errors: p00_err[q] = probability |0> is recorded as 1,
 * p11_err[q] = probability |1> is recorded as 0.  Either may be NULL. */
qt_status qt_set_readout(qt_circuit c, const double* p00_err, const double* p11_err);
/* Parametrized circuits "for many different choices of parameters": a
 * sweep gate carries n_sets unitaries U[s] (n_sets consecutive 2^nq x 2^nq
 * complex128 matrices, layout as qt_add_gate; copied at call time).  Trajectory
 * t of qt_run_trajectories applies U[t mod n_sets], so one call runs every
 * parameter set (interleaved) and each record is a pure function of (circuit,
 * seed, t) as for plain circuits; sweep gates draw no random numbers, so set s
 * of the sweep reproduces trajectories t = s (mod n_sets) of the circuit with
 * U[s] in place of the sweep gate.  All sweep gates of a circuit have the same
 * n_sets (else QT_EINVAL); n_sets = 1 is qt_add_gate.  QT_ENONUNITARY if any
 * U[s] is not unitary (1e-9).  qt_circuit_num_sets returns n_sets (1 without
 * sweep gates). */
qt_status qt_add_gate_sweep(qt_circuit c, int moment, int nq, const int* qubits, int n_sets, const double* U);
int qt_circuit_num_sets(qt_circuit c);
/* Number of channels whose record flag is set (columns of out_kraus). */
int qt_circuit_num_recorded(qt_circuit c);
int qt_circuit_num_channels(qt_circuit c);

/* ---- gate fuser / plan (Sec. III.B) ---------------------------
 * max_fused = f, the paper's maximum fuse size, 2..6 (default 4).
 * The plan snapshots the circuit, canonicalizes every matrix, precomputes the
 * Kraus lower bounds pbar_i = sigma_min(K_i)^2 and s, and flags
 * unitary mixtures (all K_i^dag K_i proportional to I; s = 1). */
qt_status qt_fuse(qt_circuit c, int max_fused, qt_plan* out);

typedef struct {
    int max_fused;    /* f in [2, 6]; 0 = 4 */
    int tile_bits;    /* qubits held per tile; 0 = auto: 13 for n >= 13 with 4-qubit tensor-core
                         gates (persistent TMEM kernel), else 12, or n if n < 12; 12 forces the
                         per-tile kernel; 11 (n >= 12, max_fused <= 4) selects the experimental
                         TMA-pipelined kernel (plans run through qt_run_trajectories only;
                         QT_EINVAL from the stand-alone calls) */
    int low_bits;     /* lowest qubits always in a tile (coalescing); 0 = auto (4) */
    int one_gate_per_pass; /* 1 = every fused gate is its own HBM pass (the paper's GPU scheme) */
    int tensor_cores;      /* 0 = auto (on when n >= 12; fused gates padded to max(f, 4) qubits),
                              1 = on (QT_EINVAL if unsupported),
                              -1 = off: fused gates on FP32 CUDA cores */
} qt_fuse_opts;
qt_status qt_fuse_ex(qt_circuit c, const qt_fuse_opts* opts, qt_plan* out);
void qt_plan_destroy(qt_plan p);

/* ---- trajectories (Alg. 2) -------------------------------------
 * Runs trajectories t_j = traj_begin + j * traj_stride, j < traj_count,
 * `batch` of them concurrently (batch <= state_bytes / (8 * 2^n)).
 * state_dev: caller-owned device buffer; on return it holds the final
 *   (unnormalized: norms are tracked lazily) states of the LAST batch,
 *   trajectory slot b at offset b * 2^n amplitudes.
 * out_bits : host, traj_count * shots_per_traj uint64 (after readout), or NULL.
 * out_kraus: host, traj_count * qt_circuit_num_recorded int32 (chosen Kraus
 *   index of each recorded channel, in canonical order), or NULL.
 * out_obs  : host, traj_count * n_obs doubles: <psi|P|psi>/<psi|psi>, or NULL.
 * mode: 0 = delayed inner product (Alg. 2).  1 = the conventional
 *   trajectory algorithm the paper compares against: no lower bounds,
 *   every channel is a barrier whose p_i are computed on the device (same
 *   draws, same literal subtract loop with pbar_i = 0).  Channels of up to 6 qubits
 *   in both modes: conventional channels of 4..6 qubits run on the CUDA-core kernel
 *   (a tensor-core plan switches to it for such a call; P:203-212 holds for any q). */
typedef struct {
    uint64_t seed;
    uint64_t traj_begin;
    uint64_t traj_stride;   /* 0 = 1 */
    uint64_t traj_count;
    int shots_per_traj;
    int batch;              /* 0 = as many as the state buffer holds (max 256) */
    int mode;
    int profile;            /* 1 = time every tile-pass launch with CUDA events */
    int host_threads;       /* 0 = hardware concurrency */
} qt_run_opts;

/* A Pauli string: paulis[i] in "IXYZ" acts on qubits[i]. */
typedef struct {
    int nq;
    const int* qubits;
    const char* paulis;
} qt_pauli;

qt_status qt_run_trajectories(qt_ctx ctx, qt_plan plan, const qt_run_opts* opts,
                              int n_obs, const qt_pauli* obs,
                              void* state_dev, size_t state_bytes,
                              uint64_t* out_bits, int32_t* out_kraus, double* out_obs,
                              qt_stats* out_stats);

/* ---- stand-alone state operations -----------------------------------------
 * qt_apply_gate: Alg. 1 for one gate on a caller state (in place):
 *   one HBM pass of the streaming kernel (TMA tiles of 128 rows x 2^K amplitudes,
 *   K = max(nq, 5) for n >= 12, max(nq, 4) for n = 11; smaller registers, or gates
 *   wider than the register's tiles allow, run on the trajectory kernels).
 * qt_sample_bitstrings: chain-rule sampling (most significant qubit first)
 *   of `shots` bitstrings from |psi|^2 (norm-invariant), trajectory index
 *   `traj` selects the RNG stream; no readout error is applied.
 * qt_expectation_value: <psi|P|psi>/<psi|psi> for each Pauli string. */
qt_status qt_apply_gate(qt_ctx ctx, void* state_dev, int n, int nq, const int* qubits,
                        const double* U);
/* qt_apply_gate_ex: as qt_apply_gate, applied `repeats` times; if kernel_ms
 * is non-NULL it receives the mean duration of one application (CUDA events
 * on the context stream, first application excluded as warm-up). */
qt_status qt_apply_gate_ex(qt_ctx ctx, void* state_dev, int n, int nq, const int* qubits,
                           const double* U, int repeats, double* kernel_ms);
qt_status qt_sample_bitstrings(qt_ctx ctx, const void* state_dev, int n, uint64_t seed,
                               uint64_t traj, int shots, uint64_t* out);
qt_status qt_expectation_value(qt_ctx ctx, const void* state_dev, int n, int n_obs,
                               const qt_pauli* obs, double* out);

/* ---- building blocks of the distributed-state mode ------------
 * A state of n_total = n + g qubits is split over 2^g processes (global index =
 * rank << n | local index); gates act on local qubits, global qubits are
 * swapped in by an all-to-all (paper_2111_02396_b200/distributed.py).
 * qt_add_matrix: like qt_add_gate without the unitarity check (deferred
 *   non-unitary Kraus operators, K_i / sqrt(p_i) of conventional picks).
 * qt_apply_plan: apply every operation of a gate-only plan to a caller state
 *   (2^n amplitudes, in place); QT_EINVAL if the plan holds channels.
 * qt_reduce_rho: rho_Q[a][b] = sum_rest psi[rest,a] conj(psi[rest,b]) over the
 *   local qubits qubits[0..nq) (nq <= 6), fp64, fixed summation order; out =
 *   2 * 4^nq doubles, row-major interleaved, index bit m <-> m-th lowest qubit.
 * qt_sample_local: the chain-rule levels n-1..0 of shots shot_ids[0..nshots)
 *   of a register of n_total qubits whose high bits were already sampled (RNG
 *   ordinals use n_total); out[i] = the n low bits, no readout error.
 * qt_expectation_partials: <psi|P|psi>/<psi|psi> of the local state and
 *   out_norm = <psi|psi>, so ranks can combine sum_r norm_r * value_r. */
qt_status qt_add_matrix(qt_circuit c, int moment, int nq, const int* qubits, const double* M);
/* qt_permute_qubits: dst[pi(i)] = src[i], bit b of i moved to bit perm[b]
 *   (n <= 40 local qubits; src != dst; device buffers on the context stream). */
qt_status qt_permute_qubits(qt_ctx ctx, const void* src_dev, void* dst_dev, int n, const int* perm);
/* Host-side pieces of Alg. 2 for a driver that owns the state layout:
 * qt_draw: the RNG contract's uniform (purpose 1 channel, 2 sample, 3 readout).
 * qt_channel_first_loop: Alg. 2 lines 2-11 for Kraus list K
 *   (n_kraus matrices, Kronecker order) and uniform u; *pick >= 0: deferred pick
 *   to be applied as K_pick * deferred_scale (1/sqrt(pbar) for unitary
 *   mixtures); *pick = -1: conventional, *r_rest = the remaining uniform.
 *   mode 1 never defers.
 * qt_channel_choose: Alg. 2 lines 13-21 given rho over the
 *   channel's qubits at positions qubits[] (rho in internal order of those
 *   positions, as qt_reduce_rho returns it); *scale = 1/sqrt(raw p_pick). */
double qt_draw(uint64_t seed, uint32_t ordinal, uint32_t purpose, uint64_t traj, int half);
qt_status qt_channel_first_loop(int nq, int n_kraus, const double* K, double u, int mode, int* pick,
                                double* r_rest, double* deferred_scale);
qt_status qt_channel_choose(int nq, int n_kraus, const double* K, const int* qubits, const double* rho,
                            double r, int mode, int* pick, double* scale);
/* qt_readout_flips: readout error (R14) on recorded bitstrings of an
 *   n-qubit register: bits[i] (bit q = qubit q) of shot shot_ids[i] of trajectory
 *   traj; a recorded 0 becomes 1 when u < p00_err[q], a recorded 1 becomes 0 when
 *   u < p11_err[q], u = the READOUT draw of (shot, q) (purpose 3, ordinal
 *   shot * ceil(n/2) + q / 2, half q % 2), one draw per (shot, qubit) whatever the
 *   bit.  p00_err / p11_err: n doubles or NULL.  In place; host only. */
qt_status qt_readout_flips(int n, const double* p00_err, const double* p11_err, uint64_t seed, uint64_t traj,
                           int nshots, const int32_t* shot_ids, uint64_t* bits);
/* Host-side arithmetic of the distributed-state mode (distributed.py orchestrates;
 * these compute).  All host only; inputs are copied / read, outputs caller-owned.
 * qt_rank_sample: the chain-rule levels n_total-1 .. n_local (reading R13) over the
 *   rank bits: level l is held by rank bit level_rank_bit[l - n_local]; the masses
 *   of the two children are sums of rank_mass[r] over the candidate ranks in
 *   ascending r; the SAMPLE draw of (shot_ids[i], l) decides; out_prefix[i] = the
 *   chosen high bits (bit l = logical level l), out_owner[i] = the rank that holds
 *   the chosen slice (it samples the local levels with qt_sample_local).
 *   world = 2^(n_total - n_local).
 * qt_restrict_diagonal: a diagonal operator diag (2^nq complex, Kronecker order of
 *   its listed qubits) on a rank where listed qubit m is global with value fixed[m]
 *   (0 / 1) or local (fixed[m] = -1): out = the 2^k diagonal over the k local
 *   qubits (listed order, Kronecker), *out_k = k (k = 0: a scalar on this rank).
 * qt_embed_rho_diagonal: rho_Q (2^nq x 2^nq complex, internal order: bit m <->
 *   m-th lowest position) of a channel whose K_i^dag K_i are all diagonal (P:204-212
 *   then read only diag rho_Q), on one rank: position m is global with value
 *   global_bit[m] or local (-1); diag_local = the 2^n_loc diagonal of the rank's
 *   reduced rho over its local positions (ascending), or its norm when n_loc = 0.
 * qt_channel_operator: the operator a pick applies, out = K_pick * scale (Alg. 2
 *   line 7 deferred pick / line 16 conventional pick, P:197 / P:207). */
qt_status qt_rank_sample(int world, const double* rank_mass, int n_total, int n_local, const int* level_rank_bit,
                         uint64_t seed, uint64_t traj, int nshots, const int32_t* shot_ids, uint64_t* out_prefix,
                         int32_t* out_owner);
qt_status qt_restrict_diagonal(int nq, const double* diag, const int* fixed, double* out, int* out_k);
qt_status qt_embed_rho_diagonal(int nq, const int* global_bit, int n_loc, const double* diag_local, double* out);
qt_status qt_channel_operator(int nq, int n_kraus, const double* K, int pick, double scale, double* out);
qt_status qt_apply_plan(qt_ctx ctx, qt_plan plan, void* state_dev, size_t state_bytes);
qt_status qt_reduce_rho(qt_ctx ctx, const void* state_dev, int n, int nq, const int* qubits, double* out);
qt_status qt_sample_local(qt_ctx ctx, const void* state_dev, int n, int n_total, uint64_t seed, uint64_t traj,
                          int nshots, const int32_t* shot_ids, uint64_t* out);
qt_status qt_expectation_partials(qt_ctx ctx, const void* state_dev, int n, int n_obs, const qt_pauli* obs,
                                  double* out, double* out_norm);

/* Host-only introspection of the planner (no device work): plans trajectory
 * `traj` exactly as qt_run_trajectories would and reports
 * out[0] tile passes, [1] fused gates, [2] conventional channels (rho_Q
 * reductions), [3] deferred picks, [4] conventional picks, [5] matrix-pool
 * entries, [6] algorithmic bytes, [7] fused-gate constituents, [8] tile bits T,
 * [9] K1 kernel: 0 CUDA cores, 4 / 5 / 6 per-tile tensor-core kernel for gates
 * padded to that many qubits, 13 persistent TMEM kernel (13-qubit tiles).
 * out holds 10 int64. */
qt_status qt_plan_info(qt_plan plan, uint64_t seed, uint64_t traj, int64_t* out);

/* Lower bound used by the sampler, exposed for tests: sigma_min(K)^2 of a
 * d x d complex128 matrix. */
double qt_kraus_lower_bound(int d, const double* K);

const char* qt_last_error(void);
const char* qt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QTRAJ_H */
