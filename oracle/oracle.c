/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the noisy
 * quantum-trajectory hot path of arXiv 2111.02396 ("Simulations of Quantum
 * Circuits with Approximate Noise using qsim and Cirq").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2111_02396_b200/, libqtraj.so) never links, imports
 * or executes anything in oracle/.  This file shares no code, header, table or
 * constant generator with the CUDA path; the Philox generator below is a
 * second, independent implementation of the RNG contract.
 *
 * Precision: complex128 (fp64) throughout.  No blocking, fusion or
 * reordering: every gate is applied on its own with Alg. 1, every channel is
 * sampled with Alg. 2's literal two-loop interval map and applied immediately.
 *
 * Citations: P:N = /root/reference/PAPER.md line N.
 *   Alg. 1 (matrix-vector multiplication)
 *   Alg. 2 (quantum trajectory algorithm)
 *   lower bound = smallest singular value^2
 *   s = 1 for unitary mixtures, always defer
 *   readout p00/p11 naming
 *
 * Readings:
 *   R1 qubit q <-> amplitude index bit q (qubit 0 = stride 1).
 *   R2 gate / Kraus matrices are given in Kronecker order of the listed qubits:
 *      qubits[0] is the MOST significant matrix-index bit.
 *   R6 RNG: Philox4x32-10, key=(seed_lo, seed_hi),
 *      counter=(ordinal, purpose, traj_lo, traj_hi); u53 of (x0,x1) = half 0,
 *      u53 of (x2,x3) = half 1.  CHANNEL draws use ordinal = channel ordinal,
 *      half 0.  SAMPLE/READOUT use ordinal = shot*ceil(n/2) + l/2, half l%2.
 *   R7 literal subtract loop in fp64, strict <, Kraus-list order.
 *   R8 unitary mixture: first loop picks the last operator on fall-through.
 *   R9 second loop weight w_i = max(0, p_i - pbar_i); fall-through picks the
 *      last i with w_i > 0; residual > 1e-6 is an error (ORC_ELEAK).
 *   R13 sampler: chain rule, most significant qubit first, one uniform per
 *      level; bit = 0 iff u*(M0+M1) < M0; M0==0 -> 1; M1==0 -> 0.
 *   R14 readout: a recorded 0 flips to 1 with probability p00[q], a recorded
 *      1 flips to 0 with probability p11[q]; one READOUT draw per (shot,qubit).
 */
#define _POSIX_C_SOURCE 200809L  /* pthread barriers under -std=c11 */
#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

#define ORC_OK 0
#define ORC_EINVAL -1
#define ORC_ELEAK -9
#define ORC_ESTATE -10

enum { PURPOSE_CHANNEL = 1, PURPOSE_SAMPLE = 2, PURPOSE_READOUT = 3 };

/* ------------------------------------------------------------------------ */
/* Fixed index-range decomposition (mode (ii) of BASELINE.md section 3: the  */
/* Alg. 1 outer loop split into disjoint ranges).  Every loop over    */
/* the 2^n amplitudes runs as NCHUNK contiguous ranges, and every fp64 sum   */
/* is the sum of the NCHUNK range sums in range order -- in BOTH modes, so   */
/* results do not depend on the thread count (reading R11: fp64 reductions, */
/* order unspecified by the paper).  With a pool, ranges are spread over     */
/* threads (range r on thread r mod T) and a barrier ends every operation.   */
/* ------------------------------------------------------------------------ */
#define NCHUNK 64

typedef struct pool_s {
    int nthreads; /* including the calling thread */
    pthread_t th[256];
    pthread_barrier_t start, done;
    void (*fn)(void* arg, int chunk);
    void* arg;
    int quit;
} pool_t;

typedef struct { pool_t* P; int tid; } pool_arg_t;

static void* pool_worker(void* a) {
    pool_arg_t* pa = (pool_arg_t*)a;
    pool_t* P = pa->P;
    for (;;) {
        pthread_barrier_wait(&P->start);
        if (P->quit) break;
        for (int c = pa->tid; c < NCHUNK; c += P->nthreads) P->fn(P->arg, c);
        pthread_barrier_wait(&P->done);
    }
    return NULL;
}

/* run fn(arg, c) for c = 0..NCHUNK-1 (in parallel with a pool, serially without) */
static void par_for(pool_t* P, void (*fn)(void*, int), void* arg) {
    if (!P || P->nthreads <= 1) {
        for (int c = 0; c < NCHUNK; ++c) fn(arg, c);
        return;
    }
    P->fn = fn;
    P->arg = arg;
    pthread_barrier_wait(&P->start);
    for (int c = 0; c < NCHUNK; c += P->nthreads) fn(arg, c);
    pthread_barrier_wait(&P->done);
}

static pool_arg_t g_pool_args[256];

static pool_t* pool_create(int nthreads) {
    if (nthreads <= 1) return NULL;
    if (nthreads > 64) nthreads = 64;
    pool_t* P = calloc(1, sizeof(pool_t));
    P->nthreads = nthreads;
    pthread_barrier_init(&P->start, NULL, (unsigned)nthreads);
    pthread_barrier_init(&P->done, NULL, (unsigned)nthreads);
    for (int t = 1; t < nthreads; ++t) {
        g_pool_args[t].P = P;
        g_pool_args[t].tid = t;
        pthread_create(&P->th[t], NULL, pool_worker, &g_pool_args[t]);
    }
    return P;
}

static void pool_destroy(pool_t* P) {
    if (!P) return;
    P->quit = 1;
    pthread_barrier_wait(&P->start);
    for (int t = 1; t < P->nthreads; ++t) pthread_join(P->th[t], NULL);
    pthread_barrier_destroy(&P->start);
    pthread_barrier_destroy(&P->done);
    free(P);
}

static uint64_t chunk_lo(uint64_t dim, int c) { return dim * (uint64_t)c / NCHUNK; }

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), written out plainly.   */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                       uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* u53(a, b) = ((a >> 5) * 2^26 + (b >> 6)) * 2^-53, in [0, 1). */
double orc_u53(uint32_t a, uint32_t b) {
    double hi = (double)(a >> 5);
    double lo = (double)(b >> 6);
    return (hi * 67108864.0 + lo) / 9007199254740992.0;
}

double orc_uniform(uint64_t seed, uint32_t ordinal, uint32_t purpose,
                   uint64_t traj, int half) {
    uint32_t ctr[4] = {ordinal, purpose, (uint32_t)(traj & 0xffffffffu),
                       (uint32_t)(traj >> 32)};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t x[4];
    orc_philox4x32_10(ctr, key, x);
    return half == 0 ? orc_u53(x[0], x[1]) : orc_u53(x[2], x[3]);
}

/* ------------------------------------------------------------------------ */
/* Alg. 1: apply a q-qubit matrix U to the state, one subvector  */
/* at a time.  U is in Kronecker order of qubits[] (qubits[0] = MSB of the   */
/* matrix index).                                                             */
/* ------------------------------------------------------------------------ */
static uint64_t subvector_index(uint64_t base, int nq, const int* qubits,
                                int j) {
    uint64_t idx = base;
    for (int m = 0; m < nq; ++m) {
        int bit = (j >> (nq - 1 - m)) & 1;
        if (bit) idx |= (uint64_t)1 << qubits[m];
    }
    return idx;
}

typedef struct {
    cplx* psi;
    int n, nq;
    const int* qubits;
    const cplx* U;
} apply_arg_t;

/* Alg. 1 over the bases of one index range (the subvectors are disjoint) */
static void apply_chunk(void* a, int c) {
    const apply_arg_t* A = (const apply_arg_t*)a;
    int M = 1 << A->nq;
    uint64_t gate_mask = 0;
    for (int m = 0; m < A->nq; ++m) gate_mask |= (uint64_t)1 << A->qubits[m];
    cplx v[64], w[64];
    uint64_t dim = (uint64_t)1 << A->n;
    for (uint64_t base = chunk_lo(dim, c); base < chunk_lo(dim, c + 1); ++base) {
        if (base & gate_mask) continue; /* one base per subvector */
        for (int k = 0; k < M; ++k) v[k] = A->psi[subvector_index(base, A->nq, A->qubits, k)];
        for (int j = 0; j < M; ++j) {
            cplx acc = 0;
            for (int k = 0; k < M; ++k) acc += A->U[j * M + k] * v[k];
            w[j] = acc;
        }
        for (int j = 0; j < M; ++j) A->psi[subvector_index(base, A->nq, A->qubits, j)] = w[j];
    }
}

static void apply_matrix_p(pool_t* P, cplx* psi, int n, int nq, const int* qubits, const cplx* U) {
    apply_arg_t A = {psi, n, nq, qubits, U};
    par_for(P, apply_chunk, &A);
}

static void apply_matrix(cplx* psi, int n, int nq, const int* qubits, const cplx* U) {
    apply_matrix_p(NULL, psi, n, nq, qubits, U);
}

int orc_apply_gate(double* psi_interleaved, int n, int nq, const int* qubits,
                   const double* U_interleaved) {
    if (n < 1 || n > 40 || nq < 1 || nq > 6) return ORC_EINVAL;
    for (int a = 0; a < nq; ++a) {
        if (qubits[a] < 0 || qubits[a] >= n) return ORC_EINVAL;
        for (int b = 0; b < a; ++b)
            if (qubits[a] == qubits[b]) return ORC_EINVAL;
    }
    apply_matrix((cplx*)psi_interleaved, n, nq, qubits, (const cplx*)U_interleaved);
    return ORC_OK;
}

typedef struct {
    cplx* psi;
    const cplx* src;
    uint64_t dim;
    double a;
    double part[NCHUNK];
    cplx cpart[NCHUNK];
} vec_arg_t;

static void norm_chunk(void* p, int c) {
    vec_arg_t* A = (vec_arg_t*)p;
    double s = 0.0;
    for (uint64_t i = chunk_lo(A->dim, c); i < chunk_lo(A->dim, c + 1); ++i)
        s += creal(A->src[i]) * creal(A->src[i]) + cimag(A->src[i]) * cimag(A->src[i]);
    A->part[c] = s;
}

/* ||psi||^2: range sums, then their sum in range order */
static double norm2_p(pool_t* P, const cplx* psi, int n) {
    vec_arg_t A;
    A.src = psi;
    A.dim = (uint64_t)1 << n;
    par_for(P, norm_chunk, &A);
    double s = 0.0;
    for (int c = 0; c < NCHUNK; ++c) s += A.part[c];
    return s;
}
static double norm2(const cplx* psi, int n) { return norm2_p(NULL, psi, n); }

static void scale_chunk(void* p, int c) {
    vec_arg_t* A = (vec_arg_t*)p;
    for (uint64_t i = chunk_lo(A->dim, c); i < chunk_lo(A->dim, c + 1); ++i) A->psi[i] *= A->a;
}
static void scale_p(pool_t* P, cplx* psi, int n, double a) {
    vec_arg_t A;
    A.psi = psi;
    A.dim = (uint64_t)1 << n;
    A.a = a;
    par_for(P, scale_chunk, &A);
}

static void copy_chunk(void* p, int c) {
    vec_arg_t* A = (vec_arg_t*)p;
    const uint64_t lo = chunk_lo(A->dim, c), hi = chunk_lo(A->dim, c + 1);
    memcpy(A->psi + lo, A->src + lo, sizeof(cplx) * (hi - lo));
}
static void copy_p(pool_t* P, cplx* dst, const cplx* src, int n) {
    vec_arg_t A;
    A.psi = dst;
    A.src = src;
    A.dim = (uint64_t)1 << n;
    par_for(P, copy_chunk, &A);
}

/* sum_i conj(x_i) y_i: range sums in range order */
static void dot_chunk(void* p, int c) {
    vec_arg_t* A = (vec_arg_t*)p;
    cplx s = 0;
    for (uint64_t i = chunk_lo(A->dim, c); i < chunk_lo(A->dim, c + 1); ++i) s += conj(A->src[i]) * A->psi[i];
    A->cpart[c] = s;
}
static cplx dot_p(pool_t* P, const cplx* x, cplx* y, int n) {
    vec_arg_t A;
    A.src = x;
    A.psi = y;
    A.dim = (uint64_t)1 << n;
    par_for(P, dot_chunk, &A);
    cplx s = 0;
    for (int c = 0; c < NCHUNK; ++c) s += A.cpart[c];
    return s;
}

/* ------------------------------------------------------------------------ */
/* Lower bound pbar = sigma_min(K)^2 = smallest eigenvalue of K^dag K */
/* H = K^dag K = A + iB is Hermitian; the real symmetric matrix               */
/* [[A, -B], [B, A]] has the same eigenvalues, each twice.  Cyclic Jacobi.    */
/* ------------------------------------------------------------------------ */
static double jacobi_min_eigenvalue(int N, double* S /* N*N, destroyed */) {
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < N; ++p)
            for (int q = p + 1; q < N; ++q) off += S[p * N + q] * S[p * N + q];
        if (off < 1e-30) break;
        for (int p = 0; p < N; ++p) {
            for (int q = p + 1; q < N; ++q) {
                double apq = S[p * N + q];
                if (fabs(apq) < 1e-300) continue;
                double app = S[p * N + p], aqq = S[q * N + q];
                double theta = (aqq - app) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) /
                           (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < N; ++k) { /* rotate columns p, q */
                    double skp = S[k * N + p], skq = S[k * N + q];
                    S[k * N + p] = c * skp - s * skq;
                    S[k * N + q] = s * skp + c * skq;
                }
                for (int k = 0; k < N; ++k) { /* rotate rows p, q */
                    double spk = S[p * N + k], sqk = S[q * N + k];
                    S[p * N + k] = c * spk - s * sqk;
                    S[q * N + k] = s * spk + c * sqk;
                }
            }
        }
    }
    double m = S[0];
    for (int i = 1; i < N; ++i)
        if (S[i * N + i] < m) m = S[i * N + i];
    return m;
}

static void kdagk(int d, const cplx* K, cplx* H) {
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
            cplx acc = 0;
            for (int k = 0; k < d; ++k) acc += conj(K[k * d + a]) * K[k * d + b];
            H[a * d + b] = acc;
        }
}

double orc_sigma_min_sq(int d, const double* K_interleaved) {
    const cplx* K = (const cplx*)K_interleaved;
    cplx* H = malloc(sizeof(cplx) * d * d);
    kdagk(d, K, H);
    int N = 2 * d;
    double* S = malloc(sizeof(double) * N * N);
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
            double re = creal(H[a * d + b]), im = cimag(H[a * d + b]);
            S[a * N + b] = re;
            S[a * N + (b + d)] = -im;
            S[(a + d) * N + b] = im;
            S[(a + d) * N + (b + d)] = re;
        }
    double lam = jacobi_min_eigenvalue(N, S);
    free(S);
    free(H);
    return lam < 0.0 ? 0.0 : lam;
}

/* K_i^dag K_i = c_i I for every i  ("proportional to unitary"). */
static int is_unitary_mixture(int d, int nk, const cplx* Ks) {
    cplx* H = malloc(sizeof(cplx) * d * d);
    int ok = 1;
    for (int i = 0; i < nk && ok; ++i) {
        kdagk(d, Ks + (size_t)i * d * d, H);
        double c = 0;
        for (int a = 0; a < d; ++a) c += creal(H[a * d + a]);
        c /= d;
        for (int a = 0; a < d && ok; ++a)
            for (int b = 0; b < d; ++b) {
                cplx target = (a == b) ? c : 0;
                if (cabs(H[a * d + b] - target) >= 1e-12) { ok = 0; break; }
            }
    }
    free(H);
    return ok;
}

/* ------------------------------------------------------------------------ */
/* Circuit description (flat arrays, canonical op order).                    */
/* ------------------------------------------------------------------------ */
typedef struct {
    int n;
    int n_ops;
    const int* kind;     /* 0 = gate, 1 = channel */
    const int* nq;
    const int* qubits;   /* n_ops * 6, Kronecker order */
    const int* n_kraus;  /* channels: number of Kraus operators */
    const int64_t* mat_off; /* offset (in complex numbers) into mats */
    const double* mats;  /* interleaved complex128 */
    const double* p00;   /* per qubit, nullable */
    const double* p11;
    int n_obs;
    const char* obs;     /* n_obs * n chars of 'I','X','Y','Z'; char q = qubit q */
    int mode;            /* 0 = Alg. 2 (delayed), 1 = conventional */
} orc_circuit;

typedef struct {
    double* final_state;   /* 2^n complex (interleaved), nullable */
    int32_t* kraus_choice; /* n_channels */
    int8_t* branch;        /* n_channels: 0 deferred (first loop), 1 conventional */
    double* kraus_margin;  /* n_channels: min |r - threshold| over comparisons made */
    uint64_t* bits;        /* shots (after readout) */
    uint64_t* bits_raw;    /* shots (before readout), nullable */
    double* sample_margin; /* shots: min over levels |u*M - M0| / M */
    double* obs_values;    /* n_obs */
} orc_traj_out;

static double min_d(double a, double b) { return a < b ? a : b; }

/* Alg. 2 for one channel; returns status. psi is normalized on entry. */
/* mode 0: Alg. 2 (delayed inner products).  mode 1: the conventional
 * trajectory algorithm of P:181 -- no lower bounds (pbar_i = 0), so every
 * channel computes its p_i = ||K_i psi||^2 and samples with the same literal
 * subtract loop (Alg. 2's second loop with pbar = 0). */
static int sample_channel(pool_t* PL, cplx* psi, int n, int nq, const int* qubits, int nk,
                          const cplx* Ks, double u, int mode, int* chosen, int* branch,
                          double* margin) {
    int d = 1 << nq;
    double pbar[64];
    double s = 0.0;
    for (int i = 0; i < nk; ++i) {
        pbar[i] = orc_sigma_min_sq(d, (const double*)(Ks + (size_t)i * d * d));
        s += pbar[i];
    }
    (void)s;
    int mixture = is_unitary_mixture(d, nk, Ks);
    if (mode == 1) {
        for (int i = 0; i < nk; ++i) pbar[i] = 0.0;
        mixture = 0;
    }
    double r = u;
    double mg = INFINITY;
    /* First loop, Alg. 2 lines 4-11. */
    for (int i = 0; i < nk; ++i) {
        mg = min_d(mg, fabs(r - pbar[i]));
        if (r < pbar[i]) { *chosen = i; *branch = 0; *margin = mg; goto apply_normalized; }
        r -= pbar[i];
    }
    if (mixture) { /* R8: s == 1 mathematically; never enter the second loop */
        *chosen = nk - 1; *branch = 0; *margin = mg;
        goto apply_normalized;
    }
    /* Second loop, Alg. 2 lines 12-21; p_i by applying K_i to a copy. */
    {
        uint64_t dim = (uint64_t)1 << n;
        cplx* tmp = malloc(sizeof(cplx) * dim);
        double p[64], w[64];
        for (int i = 0; i < nk; ++i) {
            copy_p(PL, tmp, psi, n);
            apply_matrix_p(PL, tmp, n, nq, qubits, Ks + (size_t)i * d * d);
            p[i] = norm2_p(PL, tmp, n);
            if (p[i] < pbar[i] - 1e-6) { free(tmp); return ORC_EINVAL; }
            w[i] = p[i] - pbar[i];
            if (w[i] < 0.0) w[i] = 0.0;
        }
        int pick = -1;
        for (int i = 0; i < nk; ++i) {
            mg = min_d(mg, fabs(r - w[i]));
            if (r < w[i]) { pick = i; break; }
            r -= w[i];
        }
        if (pick < 0) { /* R9 fall-through */
            if (r > 1e-6) { free(tmp); return ORC_ELEAK; }
            for (int i = nk - 1; i >= 0; --i)
                if (w[i] > 0.0) { pick = i; break; }
            if (pick < 0) { free(tmp); return ORC_ELEAK; }
        }
        copy_p(PL, tmp, psi, n);
        apply_matrix_p(PL, tmp, n, nq, qubits, Ks + (size_t)pick * d * d);
        /* |Psi> <- (1/sqrt(p_i)) K_i |Psi>  (Alg. 2 line 16) */
        scale_p(PL, tmp, n, 1.0 / sqrt(p[pick]));
        copy_p(PL, psi, tmp, n);
        free(tmp);
        *chosen = pick; *branch = 1; *margin = mg;
        return ORC_OK;
    }
apply_normalized:
    apply_matrix_p(PL, psi, n, nq, qubits, Ks + (size_t)(*chosen) * d * d);
    {
        double nn = norm2_p(PL, psi, n);
        if (!(nn > 0.0)) return ORC_ESTATE;
        scale_p(PL, psi, n, 1.0 / sqrt(nn));
    }
    return ORC_OK;
}

/* Chain-rule sampler (R13): returns the bitstring; margin = min over levels.
 * The masses of the two children of the prefix are range sums (NCHUNK ranges of
 * the 2^l completions, summed in range order). */
typedef struct {
    const cplx* psi;
    uint64_t prefix;
    int l;
    double m0[NCHUNK], m1[NCHUNK];
} mass_arg_t;

static void mass_chunk(void* p, int c) {
    mass_arg_t* A = (mass_arg_t*)p;
    const uint64_t lo_count = (uint64_t)1 << A->l;
    double M0 = 0.0, M1 = 0.0;
    for (uint64_t low = chunk_lo(lo_count, c); low < chunk_lo(lo_count, c + 1); ++low) {
        uint64_t i0 = A->prefix | low;                      /* bit l = 0 */
        uint64_t i1 = A->prefix | ((uint64_t)1 << A->l) | low; /* bit l = 1 */
        M0 += creal(A->psi[i0]) * creal(A->psi[i0]) + cimag(A->psi[i0]) * cimag(A->psi[i0]);
        M1 += creal(A->psi[i1]) * creal(A->psi[i1]) + cimag(A->psi[i1]) * cimag(A->psi[i1]);
    }
    A->m0[c] = M0;
    A->m1[c] = M1;
}

static uint64_t sample_one(pool_t* PL, const cplx* psi, int n, uint64_t seed, uint64_t traj,
                           int shot, double* margin) {
    uint64_t prefix = 0; /* bits above the current level */
    double mg = INFINITY;
    int half_n = (n + 1) / 2;
    mass_arg_t A;
    A.psi = psi;
    for (int l = n - 1; l >= 0; --l) {
        A.prefix = prefix;
        A.l = l;
        par_for(PL, mass_chunk, &A);
        double M0 = 0.0, M1 = 0.0;
        for (int c = 0; c < NCHUNK; ++c) {
            M0 += A.m0[c];
            M1 += A.m1[c];
        }
        double u = orc_uniform(seed, (uint32_t)(shot * half_n + l / 2),
                               PURPOSE_SAMPLE, traj, l % 2);
        int bit;
        if (M0 == 0.0) bit = 1;
        else if (M1 == 0.0) bit = 0;
        else {
            double M = M0 + M1;
            mg = min_d(mg, fabs(u * M - M0) / M);
            bit = (u * M < M0) ? 0 : 1;
        }
        if (bit) prefix |= (uint64_t)1 << l;
    }
    *margin = mg;
    return prefix;
}

static uint64_t readout(uint64_t bits, int n, const double* p00,
                        const double* p11, uint64_t seed, uint64_t traj,
                        int shot) {
    if (!p00 && !p11) return bits;
    int half_n = (n + 1) / 2;
    uint64_t out = bits;
    for (int q = 0; q < n; ++q) {
        double u = orc_uniform(seed, (uint32_t)(shot * half_n + q / 2),
                               PURPOSE_READOUT, traj, q % 2);
        int b = (bits >> q) & 1;
        if (b == 0 && p00 && u < p00[q]) out |= (uint64_t)1 << q;
        if (b == 1 && p11 && u < p11[q]) out &= ~((uint64_t)1 << q);
    }
    return out;
}

/* <psi|P|psi> / <psi|psi> with P = tensor product of single-qubit Paulis,
 * computed by applying each Pauli with Alg. 1 to a copy. */
static double pauli_expectation(pool_t* PL, const cplx* psi, int n, const char* ps) {
    static const cplx X[4] = {0, 1, 1, 0};
    static const cplx Y[4] = {0, -I, I, 0};
    static const cplx Z[4] = {1, 0, 0, -1};
    uint64_t dim = (uint64_t)1 << n;
    cplx* phi = malloc(sizeof(cplx) * dim);
    copy_p(PL, phi, psi, n);
    for (int q = 0; q < n; ++q) {
        const cplx* P = NULL;
        if (ps[q] == 'X') P = X;
        else if (ps[q] == 'Y') P = Y;
        else if (ps[q] == 'Z') P = Z;
        if (P) apply_matrix_p(PL, phi, n, 1, &q, P);
    }
    cplx num = dot_p(PL, psi, phi, n);
    free(phi);
    return creal(num) / norm2_p(PL, psi, n);
}

static int run_one(pool_t* PL, const orc_circuit* c, uint64_t seed, uint64_t traj,
                   int shots, orc_traj_out* o) {
    int n = c->n;
    uint64_t dim = (uint64_t)1 << n;
    cplx* psi = calloc(dim, sizeof(cplx));
    if (!psi) return ORC_EINVAL;
    psi[0] = 1.0; /* |0...0> */
    const cplx* mats = (const cplx*)c->mats;
    int ch = 0;
    int status = ORC_OK;
    for (int op = 0; op < c->n_ops && status == ORC_OK; ++op) {
        const int* qs = c->qubits + 6 * op;
        if (c->kind[op] == 0) {
            apply_matrix_p(PL, psi, n, c->nq[op], qs, mats + c->mat_off[op]);
        } else {
            double u = orc_uniform(seed, (uint32_t)ch, PURPOSE_CHANNEL, traj, 0);
            int chosen = -1, branch = -1;
            double margin = INFINITY;
            status = sample_channel(PL, psi, n, c->nq[op], qs, c->n_kraus[op],
                                    mats + c->mat_off[op], u, c->mode, &chosen, &branch,
                                    &margin);
            if (o->kraus_choice) o->kraus_choice[ch] = chosen;
            if (o->branch) o->branch[ch] = (int8_t)branch;
            if (o->kraus_margin) o->kraus_margin[ch] = margin;
            ++ch;
        }
    }
    if (status == ORC_OK) {
        for (int s = 0; s < shots; ++s) {
            double mg;
            uint64_t b = sample_one(PL, psi, n, seed, traj, s, &mg);
            if (o->bits_raw) o->bits_raw[s] = b;
            if (o->sample_margin) o->sample_margin[s] = mg;
            if (o->bits) o->bits[s] = readout(b, n, c->p00, c->p11, seed, traj, s);
        }
        for (int k = 0; k < c->n_obs; ++k)
            if (o->obs_values) o->obs_values[k] = pauli_expectation(PL, psi, n, c->obs + (size_t)k * n);
        if (o->final_state) memcpy(o->final_state, psi, sizeof(cplx) * dim);
    }
    free(psi);
    return status;
}

/* ------------------------------------------------------------------------ */
/* Public entry: run trajectories traj_begin + stride*j, j < traj_count,     */
/* one trajectory per thread (mode (i) of BASELINE.md section 3).            */
/* Output arrays are indexed by j.                                           */
/* ------------------------------------------------------------------------ */
typedef struct {
    const orc_circuit* c;
    uint64_t seed, traj_begin, stride;
    int64_t traj_count;
    int shots, n_channels;
    double* final_states;
    int32_t* kraus_choice;
    int8_t* branch;
    double* kraus_margin;
    uint64_t* bits;
    uint64_t* bits_raw;
    double* sample_margin;
    double* obs_values;
    int32_t* status;
    int64_t next;
    pthread_mutex_t lock;
    pool_t* pool;  /* mode (ii): range-parallel trajectories, one at a time */
} job_t;

static void* worker(void* arg) {
    job_t* J = (job_t*)arg;
    for (;;) {
        pthread_mutex_lock(&J->lock);
        int64_t j = J->next++;
        pthread_mutex_unlock(&J->lock);
        if (j >= J->traj_count) break;
        uint64_t dim = (uint64_t)1 << J->c->n;
        orc_traj_out o;
        o.final_state = J->final_states ? J->final_states + 2 * dim * j : NULL;
        o.kraus_choice = J->kraus_choice ? J->kraus_choice + (int64_t)J->n_channels * j : NULL;
        o.branch = J->branch ? J->branch + (int64_t)J->n_channels * j : NULL;
        o.kraus_margin = J->kraus_margin ? J->kraus_margin + (int64_t)J->n_channels * j : NULL;
        o.bits = J->bits ? J->bits + (int64_t)J->shots * j : NULL;
        o.bits_raw = J->bits_raw ? J->bits_raw + (int64_t)J->shots * j : NULL;
        o.sample_margin = J->sample_margin ? J->sample_margin + (int64_t)J->shots * j : NULL;
        o.obs_values = J->obs_values ? J->obs_values + (int64_t)J->c->n_obs * j : NULL;
        int st = run_one(J->pool, J->c, J->seed, J->traj_begin + J->stride * (uint64_t)j, J->shots, &o);
        if (J->status) J->status[j] = st;
    }
    return NULL;
}

int orc_run_trajectories(
    int n, int n_ops, const int* kind, const int* nq, const int* qubits,
    const int* n_kraus, const int64_t* mat_off, const double* mats,
    const double* p00, const double* p11, int n_obs, const char* obs,
    uint64_t seed, uint64_t traj_begin, uint64_t stride, int64_t traj_count,
    int shots, int n_threads, int mode, int range_threads,
    double* final_states, int32_t* kraus_choice, int8_t* branch,
    double* kraus_margin, uint64_t* bits, uint64_t* bits_raw,
    double* sample_margin, double* obs_values, int32_t* status) {
    if (n < 1 || n > 34 || n_ops < 0 || shots < 0 || traj_count < 0) return ORC_EINVAL;
    if (mode != 0 && mode != 1) return ORC_EINVAL;
    orc_circuit c = {n, n_ops, kind, nq, qubits, n_kraus, mat_off, mats,
                     p00, p11, n_obs, obs, mode};
    int n_channels = 0;
    for (int i = 0; i < n_ops; ++i) n_channels += (kind[i] == 1);
    job_t J;
    memset(&J, 0, sizeof J);
    J.c = &c; J.seed = seed; J.traj_begin = traj_begin; J.stride = stride ? stride : 1;
    J.traj_count = traj_count; J.shots = shots; J.n_channels = n_channels;
    J.final_states = final_states; J.kraus_choice = kraus_choice; J.branch = branch;
    J.kraus_margin = kraus_margin; J.bits = bits; J.bits_raw = bits_raw;
    J.sample_margin = sample_margin; J.obs_values = obs_values; J.status = status;
    pthread_mutex_init(&J.lock, NULL);
    if (range_threads > 1) {
        /* mode (ii): one trajectory at a time, every pass range-parallel */
        J.pool = pool_create(range_threads);
        worker(&J);
        pool_destroy(J.pool);
    } else {
        /* mode (i): one trajectory per thread */
        if (n_threads < 1) n_threads = 1;
        if (n_threads > 256) n_threads = 256;
        pthread_t th[256];
        for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, worker, &J);
        for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    }
    pthread_mutex_destroy(&J.lock);
    int worst = ORC_OK;
    if (status)
        for (int64_t j = 0; j < traj_count; ++j)
            if (status[j] != ORC_OK) worst = status[j];
    return worst;
}

/* Stand-alone helpers exposed for pins. */
int orc_sample_state(const double* psi_interleaved, int n, uint64_t seed,
                     uint64_t traj, int shots, uint64_t* bits, double* margins) {
    for (int s = 0; s < shots; ++s)
        bits[s] = sample_one(NULL, (const cplx*)psi_interleaved, n, seed, traj, s,
                             margins ? &margins[s] : &(double){0});
    return ORC_OK;
}

double orc_pauli_expectation(const double* psi_interleaved, int n,
                             const char* paulis) {
    return pauli_expectation(NULL, (const cplx*)psi_interleaved, n, paulis);
}

int orc_is_unitary_mixture(int d, int nk, const double* Ks) {
    return is_unitary_mixture(d, nk, (const cplx*)Ks);
}
