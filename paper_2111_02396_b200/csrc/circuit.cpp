// circuit.cpp -- circuit upload, validation, canonicalization and plan
// preprocessing (Sec. II; Kraus lower bounds P:183; unitary
// mixtures P:186).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>

#include "host.hpp"
#include "philox.hpp"

struct qt_circuit_s {
    qt::Circuit c;
    std::map<int, uint64_t> moment_mask;  // qubits used per moment
};
struct qt_plan_s {
    qt::Plan p;
};

namespace qt {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

static qt_status fail(qt_status st, const std::string& msg) {
    set_error(msg);
    return st;
}

// Kronecker-ordered input (qubits[0] = MSB) -> internal order (sorted
// qubits, matrix bit m <-> m-th lowest qubit).
static void canonicalize(int nq, const int* qubits, const double* in, int* q_sorted, cd* out) {
    int order[6];
    for (int i = 0; i < nq; ++i) order[i] = i;
    std::sort(order, order + nq, [&](int a, int b) { return qubits[a] < qubits[b]; });
    for (int m = 0; m < nq; ++m) q_sorted[m] = qubits[order[m]];
    const int d = 1 << nq;
    // internal index a -> Kronecker index: internal bit m is the qubit listed
    // at position order[m], whose Kronecker bit is nq-1-order[m].
    std::vector<int> kidx(d);
    for (int a = 0; a < d; ++a) {
        int k = 0;
        for (int m = 0; m < nq; ++m)
            if ((a >> m) & 1) k |= 1 << (nq - 1 - order[m]);
        kidx[a] = k;
    }
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
            const int ka = kidx[a], kb = kidx[b];
            out[a * d + b] = cd(in[2 * (ka * d + kb)], in[2 * (ka * d + kb) + 1]);
        }
}

// canonical form of operation i (sorted qubits, internal matrix order)
const HostOp* circuit_op(const qt_circuit_s* c, int i) {
    return (c && i >= 0 && i < (int)c->c.ops.size()) ? &c->c.ops[i] : nullptr;
}

static double max_dev_from_identity_of_gram(int d, const cd* const* mats, int count) {
    // || sum_i M_i^dag M_i - I ||_max
    double worst = 0.0;
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
            cd s = 0;
            for (int i = 0; i < count; ++i)
                for (int k = 0; k < d; ++k) s += std::conj(mats[i][k * d + a]) * mats[i][k * d + b];
            const cd target = (a == b) ? cd(1, 0) : cd(0, 0);
            worst = std::max(worst, std::abs(s - target));
        }
    return worst;
}

static qt_status check_qubits(const qt_circuit_s* c, int moment, int nq, const int* qubits, uint64_t* mask_out) {
    if (nq < 1 || nq > 6) return fail(QT_EARITY, "operation arity must be 1..6");
    if (!qubits) return fail(QT_EINVAL, "qubits is NULL");
    if (moment < 0) return fail(QT_EINVAL, "moment must be >= 0");
    uint64_t mask = 0;
    for (int i = 0; i < nq; ++i) {
        if (qubits[i] < 0 || qubits[i] >= c->c.n) return fail(QT_EQUBIT, "qubit out of range");
        const uint64_t bit = 1ull << qubits[i];
        if (mask & bit) return fail(QT_EQUBIT, "duplicate qubit in operation");
        mask |= bit;
    }
    auto it = c->moment_mask.find(moment);
    if (it != c->moment_mask.end() && (it->second & mask))
        return fail(QT_EQUBIT, "qubit used twice in one moment (P:84)");
    *mask_out = mask;
    return QT_OK;
}

// ---------------------------------------------------------------------------
// sigma_min(K)^2 = smallest eigenvalue of the Hermitian H = K^dag K, via
// cyclic Jacobi on the real symmetric 2d x 2d form [[Re H, -Im H],[Im H, Re H]]
// (each eigenvalue of H appears twice).  d = 2 uses the closed form
// lambda_min = (tr - sqrt(tr^2 - 4 det)) / 2 evaluated stably.
// ---------------------------------------------------------------------------
double lower_bound(int d, const cd* K) {
    std::vector<cd> H((size_t)d * d);
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
            cd s = 0;
            for (int k = 0; k < d; ++k) s += std::conj(K[k * d + a]) * K[k * d + b];
            H[a * d + b] = s;
        }
    if (d == 2) {
        const double h00 = H[0].real(), h11 = H[3].real();
        const double off2 = std::norm(H[1]);
        const double tr = h00 + h11;
        const double det = h00 * h11 - off2;
        const double disc = std::sqrt(std::max(0.0, (h00 - h11) * (h00 - h11) + 4.0 * off2));
        const double lmax = 0.5 * (tr + disc);
        const double lmin = lmax > 0 ? det / lmax : 0.0;  // product form avoids cancellation
        return std::max(0.0, lmin);
    }
    const int N = 2 * d;
    std::vector<double> A((size_t)N * N);
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) {
            A[a * N + b] = H[a * d + b].real();
            A[(a + d) * N + (b + d)] = H[a * d + b].real();
            A[a * N + (b + d)] = -H[a * d + b].imag();
            A[(a + d) * N + b] = H[a * d + b].imag();
        }
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0, diag = 0;
        for (int i = 0; i < N; ++i) {
            diag += A[i * N + i] * A[i * N + i];
            for (int j = i + 1; j < N; ++j) off += A[i * N + j] * A[i * N + j];
        }
        if (off <= 1e-32 * std::max(diag, 1e-300)) break;
        for (int p = 0; p < N - 1; ++p)
            for (int q = p + 1; q < N; ++q) {
                const double apq = A[p * N + q];
                if (apq == 0.0) continue;
                const double tau = (A[q * N + q] - A[p * N + p]) / (2.0 * apq);
                const double t = (tau >= 0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
                for (int k = 0; k < N; ++k) {
                    const double akp = A[k * N + p], akq = A[k * N + q];
                    A[k * N + p] = c * akp - s * akq;
                    A[k * N + q] = s * akp + c * akq;
                }
                for (int k = 0; k < N; ++k) {
                    const double apk = A[p * N + k], aqk = A[q * N + k];
                    A[p * N + k] = c * apk - s * aqk;
                    A[q * N + k] = s * apk + c * aqk;
                }
            }
    }
    double m = A[0];
    for (int i = 1; i < N; ++i) m = std::min(m, A[i * N + i]);
    return std::max(0.0, m);
}

}  // namespace qt

using namespace qt;

namespace qt {
// Switch a plan to the FP32 CUDA-core kernel (no tensor cores): T = 12 tiles for n >= 12,
// registers wide enough for every operation and fused gate.
void cuda_core_plan(Plan& P) {
    int max_arity = 1;
    for (const PlanOp& op : P.ops) max_arity = std::max(max_arity, op.nq);
    P.tc = false;
    P.v2 = false;
    if (P.T == 13 || (P.v3 && P.n >= 12)) P.T = 12;
    P.v3 = false;
    if (P.T >= 12) {
        P.R = std::max(P.f <= 4 ? 4 : P.f, max_arity);
    } else {
        P.R = std::min(P.T, std::max(4, std::max(max_arity, P.f)));
    }
    P.f = std::min(P.f, P.R);
}
}  // namespace qt

extern "C" {

const char* qt_last_error(void) { return g_last_error.c_str(); }
const char* qt_version(void) { return "qtraj-b200 0.1 (sm_100a)"; }

double qt_kraus_lower_bound(int d, const double* K) {
    std::vector<cd> k((size_t)d * d);
    for (int i = 0; i < d * d; ++i) k[i] = cd(K[2 * i], K[2 * i + 1]);
    return lower_bound(d, k.data());
}

qt_status qt_circuit_create(int n_qubits, qt_circuit* out) {
    if (!out) return fail(QT_EINVAL, "out is NULL");
    if (n_qubits < 1 || n_qubits > 40) return fail(QT_EINVAL, "n_qubits must be 1..40");
    auto* c = new (std::nothrow) qt_circuit_s();
    if (!c) return fail(QT_EOOM, "host allocation failed");
    c->c.n = n_qubits;
    *out = c;
    return QT_OK;
}

void qt_circuit_destroy(qt_circuit c) { delete c; }

qt_status qt_add_gate(qt_circuit c, int moment, int nq, const int* qubits, const double* U) {
    if (!c || !U) return fail(QT_EINVAL, "NULL argument");
    uint64_t mask;
    qt_status st = check_qubits(c, moment, nq, qubits, &mask);
    if (st != QT_OK) return st;
    HostOp op;
    op.kind = 0;
    op.moment = moment;
    op.seq = c->c.seq++;
    op.nq = nq;
    op.mask = mask;
    op.n_kraus = 1;
    const int d = 1 << nq;
    op.mats.resize((size_t)d * d);
    canonicalize(nq, qubits, U, op.q, op.mats.data());
    const cd* m = op.mats.data();
    if (!(max_dev_from_identity_of_gram(d, &m, 1) < 1e-9))
        return fail(QT_ENONUNITARY, "gate matrix is not unitary (tolerance 1e-9)");
    c->moment_mask[moment] |= mask;
    c->c.ops.push_back(std::move(op));
    return QT_OK;
}

qt_status qt_add_gate_sweep(qt_circuit c, int moment, int nq, const int* qubits, int n_sets, const double* U) {
    if (!c || !U) return fail(QT_EINVAL, "NULL argument");
    if (n_sets < 1 || n_sets > (1 << 20)) return fail(QT_EINVAL, "n_sets must be 1..2^20");
    if (c->c.n_sets > 1 && n_sets > 1 && n_sets != c->c.n_sets)
        return fail(QT_EINVAL, "every sweep gate of a circuit must have the same number of parameter sets");
    uint64_t mask;
    qt_status st = check_qubits(c, moment, nq, qubits, &mask);
    if (st != QT_OK) return st;
    HostOp op;
    op.kind = 0;
    op.moment = moment;
    op.seq = c->c.seq++;
    op.nq = nq;
    op.mask = mask;
    op.n_kraus = n_sets;
    const int d = 1 << nq;
    op.mats.resize((size_t)n_sets * d * d);
    for (int set = 0; set < n_sets; ++set) {
        cd* m = op.mats.data() + (size_t)set * d * d;
        canonicalize(nq, qubits, U + (size_t)set * 2 * d * d, op.q, m);
        const cd* cm = m;
        if (!(max_dev_from_identity_of_gram(d, &cm, 1) < 1e-9))
            return fail(QT_ENONUNITARY, "sweep gate matrix " + std::to_string(set) + " is not unitary (tolerance 1e-9)");
    }
    c->moment_mask[moment] |= mask;
    if (n_sets > 1) c->c.n_sets = n_sets;
    c->c.ops.push_back(std::move(op));
    return QT_OK;
}

int qt_circuit_num_sets(qt_circuit c) { return c ? c->c.n_sets : 0; }

qt_status qt_readout_flips(int n, const double* p00_err, const double* p11_err, uint64_t seed, uint64_t traj,
                           int nshots, const int32_t* shot_ids, uint64_t* bits) {
    if (n < 1 || n > 63 || nshots < 0 || (nshots > 0 && (!shot_ids || !bits)))
        return fail(QT_EINVAL, "qt_readout_flips: bad arguments");
    if (!p00_err && !p11_err) return QT_OK;
    const uint32_t half_n = (uint32_t)(n + 1) / 2;
    for (int i = 0; i < nshots; ++i) {
        const uint64_t b = bits[i];
        uint64_t o = b;
        for (int q = 0; q < n; ++q) {
            const double u = draw(seed, (uint32_t)shot_ids[i] * half_n + (uint32_t)(q / 2), kPurposeReadout, traj, q % 2);
            const int bit = (int)((b >> q) & 1ull);
            if (bit == 0 && p00_err && u < p00_err[q]) o |= 1ull << q;
            if (bit == 1 && p11_err && u < p11_err[q]) o &= ~(1ull << q);
        }
        bits[i] = o;
    }
    return QT_OK;
}

double qt_draw(uint64_t seed, uint32_t ordinal, uint32_t purpose, uint64_t traj, int half) {
    return draw(seed, ordinal, purpose, traj, half);
}

// Alg. 2 lines 2-11 for one channel of nq <= 6 qubits.
qt_status qt_channel_first_loop(int nq, int n_kraus, const double* K, double u, int mode, int* pick,
                                double* r_rest, double* deferred_scale) {
    if (nq < 1 || nq > 6 || n_kraus < 1 || n_kraus > 64 || !K || !pick || !r_rest || !deferred_scale)
        return fail(QT_EINVAL, "bad argument");
    const int d = 1 << nq;
    std::vector<cd> k((size_t)d * d);
    bool mixture = true;
    std::vector<double> pbar(n_kraus);
    for (int i = 0; i < n_kraus; ++i) {
        for (int e = 0; e < d * d; ++e) k[e] = cd(K[2 * ((size_t)i * d * d + e)], K[2 * ((size_t)i * d * d + e) + 1]);
        pbar[i] = lower_bound(d, k.data());
        // K^dag K = c I ?
        double c0 = 0;
        std::vector<cd> H((size_t)d * d);
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) {
                cd s = 0;
                for (int q = 0; q < d; ++q) s += std::conj(k[q * d + a]) * k[q * d + b];
                H[a * d + b] = s;
            }
        for (int a = 0; a < d; ++a) c0 += H[a * d + a].real();
        c0 /= d;
        for (int a = 0; a < d && mixture; ++a)
            for (int b = 0; b < d; ++b)
                if (std::abs(H[a * d + b] - (a == b ? cd(c0, 0) : cd(0, 0))) >= 1e-12) {
                    mixture = false;
                    break;
                }
    }
    double r = u;
    *pick = -1;
    if (mode == 0) {
        for (int i = 0; i < n_kraus; ++i) {
            if (r < pbar[i]) { *pick = i; break; }
            r -= pbar[i];
        }
        if (*pick < 0 && mixture) *pick = n_kraus - 1;  // s == 1
    }
    *r_rest = r;
    *deferred_scale = (*pick >= 0 && mixture && pbar[*pick] > 0) ? 1.0 / std::sqrt(pbar[*pick]) : 1.0;
    return QT_OK;
}

// Alg. 2 lines 13-21 from a reduced density matrix rho over the
// channel's qubits (positions `qubits`, rho in internal order: bit m <-> the
// m-th lowest position).  p_i = Tr(K_i^dag K_i rho) / Tr rho.
qt_status qt_channel_choose(int nq, int n_kraus, const double* K, const int* qubits, const double* rho, double r,
                            int mode, int* pick, double* scale) {
    if (nq < 1 || nq > 6 || n_kraus < 1 || n_kraus > 64 || !K || !qubits || !rho || !pick || !scale)
        return fail(QT_EINVAL, "bad argument");
    const int d = 1 << nq;
    int qs[6];
    std::vector<cd> k((size_t)d * d);
    double tr = 0;
    for (int a = 0; a < d; ++a) tr += rho[2 * (a * d + a)];
    if (!(tr > 0)) return fail(QT_ESTATE, "zero-norm state");
    std::vector<double> raw(n_kraus), w(n_kraus);
    *pick = -1;
    for (int i = 0; i < n_kraus; ++i) {
        canonicalize(nq, qubits, K + (size_t)2 * i * d * d, qs, k.data());
        const double pbar = mode == 1 ? 0.0 : lower_bound(d, k.data());
        double s = 0;  // Re Tr(K^dag K rho)
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) {
                cd m = 0;
                for (int q = 0; q < d; ++q) m += std::conj(k[q * d + a]) * k[q * d + b];
                s += m.real() * rho[2 * (b * d + a)] - m.imag() * rho[2 * (b * d + a) + 1];
            }
        raw[i] = s;
        const double p = s / tr;
        if (p < pbar - 1e-6) return fail(QT_ENONCPTP, "p_i below its lower bound");
        w[i] = std::max(0.0, p - pbar);
        if (r < w[i]) { *pick = i; break; }
        r -= w[i];
    }
    if (*pick < 0) {
        if (r > 1e-6) return fail(QT_ELEAK, "Alg. 2 fall-through residual > 1e-6");
        for (int i = n_kraus - 1; i >= 0; --i)
            if (w[i] > 0) { *pick = i; break; }
        if (*pick < 0) return fail(QT_ELEAK, "no operator with positive weight");
    }
    *scale = 1.0 / std::sqrt(raw[*pick]);
    return QT_OK;
}

qt_status qt_add_matrix(qt_circuit c, int moment, int nq, const int* qubits, const double* M) {
    if (!c || !M) return fail(QT_EINVAL, "NULL argument");
    uint64_t mask;
    qt_status st = check_qubits(c, moment, nq, qubits, &mask);
    if (st != QT_OK) return st;
    HostOp op;
    op.kind = 0;
    op.moment = moment;
    op.seq = c->c.seq++;
    op.nq = nq;
    op.mask = mask;
    op.n_kraus = 1;
    const int d = 1 << nq;
    op.mats.resize((size_t)d * d);
    canonicalize(nq, qubits, M, op.q, op.mats.data());
    for (const cd& x : op.mats)
        if (!std::isfinite(x.real()) || !std::isfinite(x.imag())) return fail(QT_EINVAL, "non-finite matrix entry");
    c->moment_mask[moment] |= mask;
    c->c.ops.push_back(std::move(op));
    return QT_OK;
}

qt_status qt_add_channel(qt_circuit c, int moment, int nq, const int* qubits, int n_kraus,
                         const double* K, int record) {
    if (!c || !K) return fail(QT_EINVAL, "NULL argument");
    if (n_kraus < 1 || n_kraus > 64) return fail(QT_EINVAL, "n_kraus must be 1..64");
    uint64_t mask;
    qt_status st = check_qubits(c, moment, nq, qubits, &mask);
    if (st != QT_OK) return st;
    HostOp op;
    op.kind = 1;
    op.moment = moment;
    op.seq = c->c.seq++;
    op.nq = nq;
    op.mask = mask;
    op.n_kraus = n_kraus;
    op.record = record ? 1 : 0;
    const int d = 1 << nq;
    op.mats.resize((size_t)n_kraus * d * d);
    for (int i = 0; i < n_kraus; ++i)
        canonicalize(nq, qubits, K + (size_t)2 * i * d * d, op.q, op.mats.data() + (size_t)i * d * d);
    std::vector<const cd*> ptrs(n_kraus);
    for (int i = 0; i < n_kraus; ++i) ptrs[i] = op.mats.data() + (size_t)i * d * d;
    if (!(max_dev_from_identity_of_gram(d, ptrs.data(), n_kraus) < 1e-9))
        return fail(QT_ENONCPTP, "Kraus operators are not trace preserving (tolerance 1e-9)");
    c->moment_mask[moment] |= mask;
    c->c.ops.push_back(std::move(op));
    return QT_OK;
}

qt_status qt_set_readout(qt_circuit c, const double* p00_err, const double* p11_err) {
    if (!c) return fail(QT_EINVAL, "NULL circuit");
    const int n = c->c.n;
    for (int q = 0; q < n; ++q) {
        if (p00_err && !(p00_err[q] >= 0.0 && p00_err[q] <= 1.0)) return fail(QT_EINVAL, "p00 outside [0,1]");
        if (p11_err && !(p11_err[q] >= 0.0 && p11_err[q] <= 1.0)) return fail(QT_EINVAL, "p11 outside [0,1]");
    }
    if (p00_err) c->c.p00.assign(p00_err, p00_err + n); else c->c.p00.clear();
    if (p11_err) c->c.p11.assign(p11_err, p11_err + n); else c->c.p11.clear();
    return QT_OK;
}

int qt_circuit_num_recorded(qt_circuit c) {
    if (!c) return 0;
    int k = 0;
    for (auto& op : c->c.ops) k += (op.kind == 1 && op.record);
    return k;
}

int qt_circuit_num_channels(qt_circuit c) {
    if (!c) return 0;
    int k = 0;
    for (auto& op : c->c.ops) k += (op.kind == 1);
    return k;
}

qt_status qt_fuse_ex(qt_circuit c, const qt_fuse_opts* opts, qt_plan* out) {
    if (!c || !out) return fail(QT_EINVAL, "NULL argument");
    qt_fuse_opts o{};
    if (opts) o = *opts;
    const int f = o.max_fused ? o.max_fused : 4;
    if (f < 2 || f > 6) return fail(QT_EARITY, "max_fused must be in [2, 6] (P:143)");
    auto* hp = new (std::nothrow) qt_plan_s();
    if (!hp) return fail(QT_EOOM, "host allocation failed");
    Plan& P = hp->p;
    const Circuit& C = c->c;
    P.n = C.n;
    // register width: 2^R amplitudes per thread; must hold every fused gate
    int max_arity = 1;
    for (auto& op : C.ops) max_arity = std::max(max_arity, op.nq);
    // the persistent TMEM kernel (4-qubit tensor-core gates on 13-qubit tiles) is the
    // default for n >= 13 (tile_bits 0 or 13); tile_bits = 12 selects the per-tile kernel
    const bool v2_ok = C.n >= 13 && o.tensor_cores >= 0 && f <= 4 && max_arity <= f &&
                       (o.tile_bits == 0 || o.tile_bits == 13) && o.low_bits == 0;
    // (QT_TILE13=0 selects the per-tile kernel instead, for A/B measurements)
    const char* env13 = std::getenv("QT_TILE13");
    const bool auto13 = !(env13 && env13[0] == '0');
    // tile_bits = 11: the TMA-pipelined kernel (tile_pass_v3.cu) on 11-qubit tiles
    const bool v3_ok = C.n >= 12 && o.tensor_cores >= 0 && f <= 4 && max_arity <= f && o.low_bits == 0;
    if (o.tile_bits == 11 && C.n >= 12) {
        if (!v3_ok) {
            delete hp;
            return fail(QT_EINVAL, "tile_bits = 11 needs n >= 12, tensor cores and max_fused <= 4");
        }
        P.v3 = true;
    }
    P.T = o.tile_bits ? o.tile_bits : std::min(C.n, (v2_ok && auto13) ? 13 : 12);
    if (P.T == 13 && !v2_ok) {
        delete hp;
        return fail(QT_EINVAL, "tile_bits = 13 needs n >= 13, tensor cores and max_fused <= 4");
    }
    if ((P.T > 12 && P.T != 13) || P.T > C.n || P.T < 1) {
        delete hp;
        return fail(QT_EINVAL, "tile_bits must be <= min(n, 12), or 13");
    }
    if (C.n > 12 && P.T != 12 && P.T != 13 && !P.v3) {
        delete hp;
        return fail(QT_EINVAL, "tile_bits must be 12 or 13 for n > 12 in this build");
    }
    P.CL = std::min(o.low_bits ? o.low_bits : 4, P.T);
    if (P.T >= 12) {
        P.R = std::max(f <= 4 ? 4 : f, max_arity);
    } else {
        // whole-state tiles (n < 12): 2^R amplitudes per thread hold the widest gate
        P.R = std::min(P.T, std::max(4, std::max(max_arity, f)));
    }
    P.f = std::min(f, P.R);
    P.one_gate = o.one_gate_per_pass != 0;
    // tensor cores: every fused gate padded to 4 qubits (f <= 4), T = 12, 128-thread CTAs
    // whose CUDA-core gates use R = 5
    const bool tc_ok = ((P.T == 12 || P.T == 13 || P.v3) && max_arity <= f);
    if (o.tensor_cores > 0 && !tc_ok) {
        delete hp;
        return fail(QT_EINVAL, "tensor_cores needs n >= 12 and gates of <= max_fused qubits");
    }
    P.tc = o.tensor_cores >= 0 && tc_ok;
    if (P.tc) {
        // 128-thread CTAs: f <= 4 -> gates padded to 4 qubits (two 16-amplitude
        // subvectors per thread, 4 CTAs / SM); f = 5 -> padded to 5 qubits (one
        // 32-amplitude subvector per thread, 3 CTAs / SM); f = 6 -> padded to 6
        // qubits (half a 64-amplitude subvector per thread, 2 CTAs / SM)
        P.R = 5;
        P.f = f;
        P.tc_k = f <= 4 ? 4 : f;
        // T = 13: 256 threads per compute warpgroup hold 32 amplitudes each for the
        // CUDA-core gates (device-chosen conventional operators)
        if (P.T == 13) {
            P.v2 = true;
            P.R = 5;
        }
        // T = 11: 128 threads per warpgroup hold 16 amplitudes each (a row of a gate)
        if (P.v3) P.R = 4;
    }
    // canonical order: moment ascending, then call order (stable)
    std::vector<const HostOp*> order;
    for (auto& op : C.ops) order.push_back(&op);
    std::stable_sort(order.begin(), order.end(), [](const HostOp* a, const HostOp* b) {
        return a->moment != b->moment ? a->moment < b->moment : a->seq < b->seq;
    });
    int chan = 0, rec = 0;
    for (const HostOp* hop : order) {
        PlanOp po;
        po.kind = hop->kind;
        po.nq = hop->nq;
        std::memcpy(po.q, hop->q, sizeof po.q);
        po.mask = hop->mask;
        po.n_kraus = hop->n_kraus;
        po.var_base = (int)P.vars.size();
        const int d = 1 << hop->nq;
        if (hop->kind == 1) {
            po.chan = chan++;
            po.record = hop->record ? rec++ : -1;
            // lower bounds and unitary-mixture flag
            po.pbar.resize(hop->n_kraus);
            po.s = 0;
            bool mixture = true;
            for (int i = 0; i < hop->n_kraus; ++i) {
                const cd* K = hop->mats.data() + (size_t)i * d * d;
                po.pbar[i] = lower_bound(d, K);
                po.s += po.pbar[i];
                // K^dag K == c I ?
                double c0 = 0;
                std::vector<cd> H((size_t)d * d);
                for (int a = 0; a < d; ++a)
                    for (int b = 0; b < d; ++b) {
                        cd s = 0;
                        for (int k = 0; k < d; ++k) s += std::conj(K[k * d + a]) * K[k * d + b];
                        H[a * d + b] = s;
                    }
                for (int a = 0; a < d; ++a) c0 += H[a * d + a].real();
                c0 /= d;
                for (int a = 0; a < d && mixture; ++a)
                    for (int b = 0; b < d; ++b)
                        if (std::abs(H[a * d + b] - (a == b ? cd(c0, 0) : cd(0, 0))) >= 1e-12) {
                            mixture = false;
                            break;
                        }
            }
            po.mixture = mixture;
            if (!mixture) P.max_conv_d = std::max(P.max_conv_d, d);
            P.max_chan_d = std::max(P.max_chan_d, d);
            // variants: deferred application of K_i (mixtures: K_i / sqrt(pbar_i), exactly unitary)
            for (int i = 0; i < hop->n_kraus; ++i) {
                const cd* K = hop->mats.data() + (size_t)i * d * d;
                const double sc = (mixture && po.pbar[i] > 0) ? 1.0 / std::sqrt(po.pbar[i]) : 1.0;
                Variant v;
                v.nq = hop->nq;
                bool ident = true;
                VarDesc vd;
                vd.off = (int)(P.var_data.size() / 2);
                vd.nq = hop->nq;
                for (int e = 0; e < d * d; ++e) {
                    const cd x = K[e] * sc;
                    P.var_data.push_back(x.real());
                    P.var_data.push_back(x.imag());
                    const cd target = (e / d == e % d) ? cd(1, 0) : cd(0, 0);
                    if (std::abs(x - target) > 1e-15) ident = false;
                }
                v.identity = ident;
                P.vars.push_back(v);
                P.var_desc.push_back(vd);
            }
            // device channel data: [qmask][pbar][M_i][K_i]
            ChanDesc cdsc;
            cdsc.qmask = hop->mask;
            cdsc.d = d;
            cdsc.n_kraus = hop->n_kraus;
            cdsc.nq = hop->nq;
            cdsc.off = (int)P.chan_data.size();
            for (int i = 0; i < hop->n_kraus; ++i) P.chan_data.push_back(po.pbar[i]);
            for (int i = 0; i < hop->n_kraus; ++i) {
                const cd* K = hop->mats.data() + (size_t)i * d * d;
                for (int a = 0; a < d; ++a)
                    for (int b = 0; b < d; ++b) {
                        cd s = 0;
                        for (int k = 0; k < d; ++k) s += std::conj(K[k * d + a]) * K[k * d + b];
                        P.chan_data.push_back(s.real());
                        P.chan_data.push_back(s.imag());
                    }
            }
            for (int i = 0; i < hop->n_kraus; ++i) {
                const cd* K = hop->mats.data() + (size_t)i * d * d;
                for (int e = 0; e < d * d; ++e) {
                    P.chan_data.push_back(K[e].real());
                    P.chan_data.push_back(K[e].imag());
                }
            }
            P.chans.push_back(cdsc);
        } else {
            // one variant per parameter set (plain gates: one)
            for (int set = 0; set < hop->n_kraus; ++set) {
                const cd* M = hop->mats.data() + (size_t)set * d * d;
                Variant v;
                v.nq = hop->nq;
                VarDesc vd;
                vd.off = (int)(P.var_data.size() / 2);
                vd.nq = hop->nq;
                bool ident = true;
                for (int e = 0; e < d * d; ++e) {
                    P.var_data.push_back(M[e].real());
                    P.var_data.push_back(M[e].imag());
                    const cd target = (e / d == e % d) ? cd(1, 0) : cd(0, 0);
                    if (std::abs(M[e] - target) > 1e-15) ident = false;
                }
                v.identity = ident;
                // qt_add_matrix operations may have any norm: Frobenius bound unless unitary
                if (!(max_dev_from_identity_of_gram(d, &M, 1) < 1e-9)) {
                    double fro = 0;
                    for (int e = 0; e < d * d; ++e) fro += std::norm(M[e]);
                    v.norm = std::max(1.0, std::sqrt(fro));
                }
                P.vars.push_back(v);
                P.var_desc.push_back(vd);
            }
        }
        P.ops.push_back(std::move(po));
    }
    // non-mixture channels on 4..6 qubits: their device-chosen operators (2^q amplitudes
    // per thread) and rho_Q partials run in the CUDA-core kernel
    if (P.tc && P.max_conv_d > 8) {
        if (o.tensor_cores > 0) {
            delete hp;
            return fail(QT_EINVAL, "tensor_cores: non-mixture channels on more than 3 qubits need the CUDA-core path");
        }
        cuda_core_plan(P);
    }
    // the f16 tensor-core operands hold matrix entries below 65504: matrices of
    // huge norm (only possible through qt_add_matrix) use the CUDA-core path
    if (P.tc)
        for (const Variant& v : P.vars)
            if (v.norm > 1e3) {
                if (o.tensor_cores > 0) {
                    delete hp;
                    return fail(QT_EINVAL, "tensor_cores: a matrix of norm > 1e3 does not fit the f16 operands");
                }
                cuda_core_plan(P);
                break;
            }
    P.n_channels = chan;
    P.n_sets = C.n_sets;
    P.n_recorded = rec;
    P.has_p00 = !C.p00.empty();
    P.has_p11 = !C.p11.empty();
    P.p00 = C.p00;
    P.p11 = C.p11;
    *out = hp;
    return QT_OK;
}

qt_status qt_fuse(qt_circuit c, int max_fused, qt_plan* out) {
    qt_fuse_opts o{};
    o.max_fused = max_fused;
    return qt_fuse_ex(c, &o, out);
}

void qt_plan_destroy(qt_plan p) { delete p; }

}  // extern "C"

namespace qt {
const Plan& plan_of(qt_plan p) { return p->p; }
}  // namespace qt
