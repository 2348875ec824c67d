// dist_host.cpp -- host-side method arithmetic of the distributed-state mode
// (SURVEY 8(e) second mode; distributed.py orchestrates, these compute):
//   qt_rank_sample        chain-rule sampling over the rank bits (reading R13) from
//                         the ranks' masses, before the owning rank samples its
//                         local levels (qt_sample_local)
//   qt_restrict_diagonal  a diagonal operator touching global qubits restricted to one
//                         rank's values of those qubits (an operator on its local
//                         qubits, or a scalar)
//   qt_embed_rho_diagonal rho_Q of a channel whose K_i^dag K_i are all diagonal, from
//                         a rank's local diagonal and its global bits (P:204-212 need
//                         only the diagonal then)
//   qt_channel_operator   the operator a pick applies: K_pick * scale (Alg. 2 line 7 /
//                         line 16, P:197 / P:207)
#include <cstdint>
#include <cstring>
#include <vector>

#include "host.hpp"
#include "philox.hpp"

using namespace qt;

namespace {
qt_status fail(qt_status st, const std::string& m) {
    set_error(m);
    return st;
}
}  // namespace

extern "C" {

qt_status qt_rank_sample(int world, const double* rank_mass, int n_total, int n_local, const int* level_rank_bit,
                         uint64_t seed, uint64_t traj, int nshots, const int32_t* shot_ids, uint64_t* out_prefix,
                         int32_t* out_owner) {
    if (world < 1 || (world & (world - 1)) || !rank_mass || n_total < n_local || n_local < 0 || n_total > 63 ||
        nshots < 0 || (nshots > 0 && (!shot_ids || !out_prefix || !out_owner)) ||
        (n_total > n_local && !level_rank_bit))
        return fail(QT_EINVAL, "qt_rank_sample: bad argument");
    const int g = __builtin_ctz((unsigned)world);
    if (n_total - n_local != g) return fail(QT_EINVAL, "qt_rank_sample: n_total - n_local must be log2(world)");
    const int half_n = (n_total + 1) / 2;
    std::vector<int> cand, next;
    for (int sh = 0; sh < nshots; ++sh) {
        cand.resize(world);
        for (int r = 0; r < world; ++r) cand[r] = r;
        uint64_t prefix = 0;
        for (int lvl = n_total - 1; lvl >= n_local; --lvl) {
            const int gb = level_rank_bit[lvl - n_local];
            if (gb < 0 || gb >= g) return fail(QT_EINVAL, "qt_rank_sample: bad rank bit");
            // masses of the two children of the prefix: sums over the candidate ranks in
            // ascending rank order (fixed order)
            double m0 = 0.0, m1 = 0.0;
            for (int r : cand) ((r >> gb) & 1 ? m1 : m0) += rank_mass[r];
            const double u = draw(seed, (uint32_t)(shot_ids[sh] * half_n + lvl / 2), kPurposeSample, traj, lvl & 1);
            int bit;
            if (m0 == 0.0) bit = 1;
            else if (m1 == 0.0) bit = 0;
            else bit = (u * (m0 + m1) < m0) ? 0 : 1;
            next.clear();
            for (int r : cand)
                if (((r >> gb) & 1) == bit) next.push_back(r);
            cand.swap(next);
            prefix |= (uint64_t)bit << lvl;
        }
        out_prefix[sh] = prefix;
        out_owner[sh] = cand.empty() ? -1 : cand[0];
    }
    return QT_OK;
}

qt_status qt_restrict_diagonal(int nq, const double* diag, const int* fixed, double* out, int* out_k) {
    if (nq < 1 || nq > 6 || !diag || !fixed || !out || !out_k) return fail(QT_EINVAL, "qt_restrict_diagonal: bad argument");
    int k = 0;
    for (int m = 0; m < nq; ++m) {
        if (fixed[m] < -1 || fixed[m] > 1) return fail(QT_EINVAL, "qt_restrict_diagonal: fixed[m] must be -1, 0 or 1");
        if (fixed[m] < 0) ++k;
    }
    for (int a = 0; a < (1 << k); ++a) {
        // Kronecker order: listed qubit m is index bit nq - 1 - m; the local qubits
        // keep their listed order in the restricted operator
        int idx = 0;
        for (int m = 0, j = 0; m < nq; ++m) {
            int bit;
            if (fixed[m] >= 0) {
                bit = fixed[m];
            } else {
                bit = (a >> (k - 1 - j)) & 1;
                ++j;
            }
            idx |= bit << (nq - 1 - m);
        }
        out[2 * a] = diag[2 * idx];
        out[2 * a + 1] = diag[2 * idx + 1];
    }
    *out_k = k;
    return QT_OK;
}

qt_status qt_embed_rho_diagonal(int nq, const int* global_bit, int n_loc, const double* diag_local, double* out) {
    if (nq < 1 || nq > 6 || !global_bit || !out || !diag_local || n_loc < 0 || n_loc > nq)
        return fail(QT_EINVAL, "qt_embed_rho_diagonal: bad argument");
    int nl = 0;
    for (int m = 0; m < nq; ++m)
        if (global_bit[m] < 0) ++nl;
    if (nl != n_loc) return fail(QT_EINVAL, "qt_embed_rho_diagonal: n_loc does not match global_bit");
    const int d = 1 << nq;
    std::memset(out, 0, sizeof(double) * 2 * d * d);
    for (int al = 0; al < (1 << n_loc); ++al) {
        // internal order: bit m <-> m-th lowest position; local positions take the
        // local diagonal's index bits in ascending order, global ones this rank's bits
        int a = 0;
        for (int m = 0, j = 0; m < nq; ++m) {
            const int bit = global_bit[m] >= 0 ? global_bit[m] : (al >> j++) & 1;
            a |= bit << m;
        }
        out[2 * (a * d + a)] = diag_local[al];  // n_loc = 0: the rank's norm
    }
    return QT_OK;
}

qt_status qt_channel_operator(int nq, int n_kraus, const double* K, int pick, double scale, double* out) {
    if (nq < 1 || nq > 6 || n_kraus < 1 || !K || !out || pick < 0 || pick >= n_kraus)
        return fail(QT_EINVAL, "qt_channel_operator: bad argument");
    const int dd = 1 << (2 * nq);
    const double* k = K + (size_t)2 * dd * pick;
    for (int e = 0; e < 2 * dd; ++e) out[e] = k[e] * scale;
    return QT_OK;
}

}  // extern "C"
