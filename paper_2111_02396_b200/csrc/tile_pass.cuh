// tile_pass.cuh -- K1 tile-pass kernel template (+ K2/K3a/K4 epilogues) and
// the device helpers shared by the kernel translation units.  Included by
// tile_pass_r4.cu / tile_pass_r5.cu / tile_pass_r6.cu / kernels.cu, which
// instantiate disjoint (T, R) sets so they compile in parallel.
#pragma once
// (from kernels.cu) sm_100a kernels of the noisy-trajectory hot path.
//
//   K1  tile_pass_kernel   Alg. 1 over a whole fused-gate program:
//                          one CTA owns 2^T amplitudes (the qubits of
//                          PassDesc::tile_mask, the 4 lowest always included
//                          so HBM reads are 128-byte runs), keeps them in
//                          shared memory, and applies every fused gate of the
//                          pass in registers (2^R amplitudes per thread); one
//                          shared-memory re-layout per fused gate.
//   K2  (epilogue)         rho_Q partial sums of a conventional channel in fp64
//                          (Alg. 2 line 14 computed in place), then the
//                          last CTA of the trajectory reduces them in a fixed
//                          order and walks Alg. 2 lines 13-21.
//   K3  sample_kernel      chain-rule sampler over fp64 block sums + readout
//                          flips.
//   K4  (epilogue)         Pauli-string partial sums; finalize_obs_kernel.
//   K6  materialize_kernel fused-gate matrices (Sec. III.B) built in
//                          fp64 from their constituents, stored complex64.
//
// Reductions never use floating-point atomics: every sum has a fixed order
// that depends only on n and T, so results are bit-reproducible and
// independent of batch size and GPU count.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.hpp"
#include "philox.hpp"
#include "tc_common.cuh"

namespace qt {

namespace detail {

constexpr int kCL = 4;  // low qubits always inside a tile (128-byte runs)

// CTAs per SM the (T = 12, R = 4) kernel is register-budgeted for.
#ifndef QT_MINB
#define QT_MINB 3
#endif

__device__ __forceinline__ uint32_t swz(uint32_t L) {
    // XOR-fold swizzle of the amplitude slot (linear over GF(2)):
    // bits 0..3 ^= bits 4..7 ^ bits 8..11.
    return L ^ (((L >> 4) ^ (L >> 8)) & 15u);
}

__device__ __forceinline__ uint64_t pdep64(uint64_t x, uint64_t mask) {
    uint64_t r = 0;
    while (mask) {
        const uint64_t low = mask & (~mask + 1);
        if (x & 1) r |= low;
        x >>= 1;
        mask ^= low;
    }
    return r;
}

__device__ __forceinline__ uint32_t pdep32(uint32_t x, uint32_t mask) {
    uint32_t r = 0;
    while (mask) {
        const uint32_t low = mask & (~mask + 1);
        if (x & 1) r |= low;
        x >>= 1;
        mask ^= low;
    }
    return r;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;\n" ::); }

__device__ __forceinline__ void cfma(float2& acc, const float2 u, const float2 v) {
    acc.x = fmaf(u.x, v.x, acc.x);
    acc.x = fmaf(-u.y, v.y, acc.x);
    acc.y = fmaf(u.x, v.y, acc.y);
    acc.y = fmaf(u.y, v.x, acc.y);
}

// Deterministic block reduction of one double (fixed tree; NT compile-time).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
    constexpr int W = NT < 32 ? NT : 32;
    constexpr unsigned mask = W == 32 ? 0xffffffffu : ((1u << W) - 1u);
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
    constexpr int NW = (NT + 31) / 32;
    if constexpr (NW == 1) {
        return v;  // every lane holds the total
    } else {
        const int tid = threadIdx.x;
        __syncthreads();
        if ((tid & 31) == 0) red[tid >> 5] = v;
        __syncthreads();
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += red[w];
        return s;
    }
}

// Block sums of N doubles with one pair of barriers per chunk of 64 / warps
// values (every thread returns the totals in v).  Fixed summation order.
template <int NT, int N>
__device__ __forceinline__ void block_sum_n(double (&v)[N], double* red) {
    constexpr int W = NT < 32 ? NT : 32;
    constexpr unsigned mask = W == 32 ? 0xffffffffu : ((1u << W) - 1u);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) v[i] += __shfl_xor_sync(mask, v[i], o);
    constexpr int NW = (NT + 31) / 32;
    if constexpr (NW > 1) {
        constexpr int C = 64 / NW;  // values per chunk (red holds 64 doubles)
        const int tid = threadIdx.x;
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += C) {
            __syncthreads();
            if ((tid & 31) == 0)
#pragma unroll
                for (int i = c0; i < N && i < c0 + C; ++i) red[(tid >> 5) * C + (i - c0)] = v[i];
            __syncthreads();
#pragma unroll
            for (int i = c0; i < N && i < c0 + C; ++i) {
                double s = 0.0;
#pragma unroll
                for (int w = 0; w < NW; ++w) s += red[w * C + (i - c0)];
                v[i] = s;
            }
        }
    }
}

// w[i] for a block-uniform runtime index (jump table, no local memory).
template <int N>
__device__ __forceinline__ float pick_uniform(const float (&w)[N], int i) {
    float r = 0.f;
#define QT_PICK_CASE(j) \
    case j:             \
        if constexpr (j < N) r = w[j]; \
        break;
    switch (i) {
        QT_PICK_CASE(0) QT_PICK_CASE(1) QT_PICK_CASE(2) QT_PICK_CASE(3) QT_PICK_CASE(4) QT_PICK_CASE(5)
        QT_PICK_CASE(6) QT_PICK_CASE(7) QT_PICK_CASE(8) QT_PICK_CASE(9) QT_PICK_CASE(10) QT_PICK_CASE(11)
        QT_PICK_CASE(12) QT_PICK_CASE(13) QT_PICK_CASE(14) QT_PICK_CASE(15) QT_PICK_CASE(16) QT_PICK_CASE(17)
        QT_PICK_CASE(18) QT_PICK_CASE(19) QT_PICK_CASE(20) QT_PICK_CASE(21) QT_PICK_CASE(22) QT_PICK_CASE(23)
        QT_PICK_CASE(24) QT_PICK_CASE(25) QT_PICK_CASE(26) QT_PICK_CASE(27) QT_PICK_CASE(28) QT_PICK_CASE(29)
        QT_PICK_CASE(30) QT_PICK_CASE(31) QT_PICK_CASE(32) QT_PICK_CASE(33) QT_PICK_CASE(34) QT_PICK_CASE(35)
        QT_PICK_CASE(36) QT_PICK_CASE(37) QT_PICK_CASE(38) QT_PICK_CASE(39) QT_PICK_CASE(40) QT_PICK_CASE(41)
        QT_PICK_CASE(42) QT_PICK_CASE(43) QT_PICK_CASE(44) QT_PICK_CASE(45) QT_PICK_CASE(46) QT_PICK_CASE(47)
        QT_PICK_CASE(48) QT_PICK_CASE(49) QT_PICK_CASE(50) QT_PICK_CASE(51) QT_PICK_CASE(52) QT_PICK_CASE(53)
        QT_PICK_CASE(54) QT_PICK_CASE(55) QT_PICK_CASE(56) QT_PICK_CASE(57) QT_PICK_CASE(58) QT_PICK_CASE(59)
        QT_PICK_CASE(60) QT_PICK_CASE(61) QT_PICK_CASE(62) QT_PICK_CASE(63)
        default: break;
    }
#undef QT_PICK_CASE
    return r;
}

// ---------------------------------------------------------------------------
// Fused-gate application in registers.  The thread holds 2^R amplitudes whose
// register-index bits 0..K-1 are the gate qubits (matrix bit m <-> register
// bit m) and bits K..R-1 are filler tile bits.  Reads the amplitudes from the
// swizzled tile, applies the 2^K x 2^K matrix (shared memory, broadcast), and
// writes the results back to the same slots.
// ---------------------------------------------------------------------------
template <int K, int R>
__device__ __forceinline__ void apply_fused(float2* __restrict__ tile, const float2* __restrict__ M,
                                           const uint32_t pbase, const uint32_t (&unit)[R]) {
    constexpr int D = 1 << K;
    constexpr int NB = 1 << (R - K);
    uint32_t ahi[NB];
    ahi[0] = pbase;
#pragma unroll
    for (int m = 0; m < R - K; ++m)
#pragma unroll
        for (int x = 0; x < (1 << m); ++x) ahi[x + (1 << m)] = ahi[x] ^ unit[K + m];
    // slot of register j = bb * D + r:  ahi[bb] ^ lo(r),  lo(r) = XOR of unit[m] over bits of r
    auto lo = [&](int r) {
        uint32_t x = 0;
#pragma unroll
        for (int m = 0; m < K; ++m)
            if ((r >> m) & 1) x ^= unit[m];
        return x;
    };
    // unit[] / pbase are BYTE offsets: one 3-input XOR (LOP3) per shared access
    char* const tb8 = reinterpret_cast<char*>(tile);
    auto at = [&](uint32_t off) -> float2& { return *reinterpret_cast<float2*>(tb8 + off); };
    float2 a[NB * D];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        const uint32_t l = lo(r);
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) a[bb * D + r] = at(ahi[bb] ^ l);
    }
    const float4* M4 = reinterpret_cast<const float4*>(M);
    // small gates: rows fully unrolled; K >= 5: row loop kept rolled (code size)
#pragma unroll(K >= 5 ? 1 : D)
    for (int r = 0; r < D; ++r) {
        float2 acc[NB];
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) acc[bb] = make_float2(0.f, 0.f);
        if constexpr (D == 1) {
            const float2 u = M[0];
#pragma unroll
            for (int bb = 0; bb < NB; ++bb) cfma(acc[bb], u, a[bb]);
        } else {
#pragma unroll
            for (int m = 0; m < D; m += 2) {
                const float4 u = M4[(r * D + m) >> 1];
#pragma unroll
                for (int bb = 0; bb < NB; ++bb) {
                    cfma(acc[bb], make_float2(u.x, u.y), a[bb * D + m]);
                    cfma(acc[bb], make_float2(u.z, u.w), a[bb * D + m + 1]);
                }
            }
        }
        const uint32_t l = lo(r);
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) at(ahi[bb] ^ l) = acc[bb];
    }
}

// Global qubit mask -> tile-local bit mask (bits of the mask outside the tile dropped).
template <int T>
__device__ __forceinline__ uint32_t to_local(uint64_t m, const PassDesc& P) {
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < T; ++i) r |= (uint32_t)((m >> P.tq[i]) & 1ull) << i;
    return r;
}

template <int R>
__device__ __forceinline__ void dispatch_fused(int k, float2* tile, const float2* M, uint32_t pbase,
                                               const uint32_t (&unit)[R]) {
    switch (k) {
        case 1: if constexpr (R >= 1) apply_fused<1, R>(tile, M, pbase, unit); break;
        case 2: if constexpr (R >= 2) apply_fused<2, R>(tile, M, pbase, unit); break;
        case 3: if constexpr (R >= 3) apply_fused<3, R>(tile, M, pbase, unit); break;
        case 4: if constexpr (R >= 4) apply_fused<4, R>(tile, M, pbase, unit); break;
        case 5: if constexpr (R >= 5) apply_fused<5, R>(tile, M, pbase, unit); break;
        case 6: if constexpr (R >= 6) apply_fused<6, R>(tile, M, pbase, unit); break;
        default: break;
    }
}

// rho_Q partial over the tile for a Q-qubit channel at tile-local positions qp.
template <int Q, int T, int NT>
__device__ __forceinline__ void rho_partial(const float2* tile, uint32_t qlocal, double* out /*2*D*D*/, double* red) {
    constexpr int D = 1 << Q;
    const int tid = threadIdx.x;
    uint32_t qoff[D];
#pragma unroll
    for (int a = 0; a < D; ++a) qoff[a] = pdep32((uint32_t)a, qlocal);
    double acc[2 * D * D];
#pragma unroll
    for (int e = 0; e < 2 * D * D; ++e) acc[e] = 0.0;
    // every slot L with the channel bits clear is the base of one 2^Q group
    for (uint32_t bL = tid; bL < (1u << T); bL += NT) {
        if (bL & qlocal) continue;
        double vr[D], vi[D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const float2 v = tile[swz(bL | qoff[a])];
            vr[a] = v.x;
            vi[a] = v.y;
        }
        // rho[a][b] += psi[a] * conj(psi[b])
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = 0; b < D; ++b) {
                acc[2 * (a * D + b)] += vr[a] * vr[b] + vi[a] * vi[b];
                acc[2 * (a * D + b) + 1] += vi[a] * vr[b] - vr[a] * vi[b];
            }
    }
    block_sum_n<NT, 2 * D * D>(acc, red);
    if (tid == 0)
#pragma unroll
        for (int e = 0; e < 2 * D * D; ++e) out[e] = acc[e];
}

// rho_Q of a Q = 3 qubit channel (8 x 8): one row a at a time (2 D doubles per
// thread in registers), the tile re-read per row; same summation order per entry
// as rho_partial (slots strided over threads, then the fixed block sum).
template <int Q, int T, int NT>
__device__ __forceinline__ void rho_partial_rows(const float2* tile, uint32_t qlocal, double* out /*2*D*D*/,
                                                 double* red) {
    constexpr int D = 1 << Q;
    const int tid = threadIdx.x;
    uint32_t qoff[D];
#pragma unroll
    for (int a = 0; a < D; ++a) qoff[a] = pdep32((uint32_t)a, qlocal);
#pragma unroll 1
    for (int a = 0; a < D; ++a) {
        double acc[2 * D];
#pragma unroll
        for (int e = 0; e < 2 * D; ++e) acc[e] = 0.0;
        for (uint32_t bL = tid; bL < (1u << T); bL += NT) {
            if (bL & qlocal) continue;
            const float2 va = tile[swz(bL | qoff[a])];
            const double ar = va.x, ai = va.y;
#pragma unroll
            for (int b = 0; b < D; ++b) {
                const float2 vb = tile[swz(bL | qoff[b])];
                acc[2 * b] += ar * (double)vb.x + ai * (double)vb.y;
                acc[2 * b + 1] += ai * (double)vb.x - ar * (double)vb.y;
            }
        }
        block_sum_n<NT, 2 * D>(acc, red);
        if (tid == 0)
#pragma unroll
            for (int e = 0; e < 2 * D; ++e) out[2 * D * a + e] = acc[e];
    }
}

// rho_Q partial of a Q = 4..6 qubit channel (D = 2^Q up to 64): every thread owns
// whole entries (a, b) of the D x D matrix and sums them over the tile's 2^(T - Q)
// rows in a fixed order, so no block reduction is needed; entries are written
// straight to `out` (2 D^2 doubles, re / im interleaved, row-major).  A rare path
// (non-mixture channels on many qubits): slow, shared-memory reads only.
template <int T, int NT, typename Swz>
__device__ __forceinline__ void rho_partial_big(const float2* tile, uint32_t qlocal, int nq, double* out, Swz swzf) {
    const int D = 1 << nq;
    const uint32_t rows = 1u << (T - nq);
    const uint32_t rest = ((1u << T) - 1u) & ~qlocal;
    for (int e = threadIdx.x; e < D * D; e += NT) {
        const int a = e / D, b = e % D;
        const uint32_t oa = pdep32((uint32_t)a, qlocal), ob = pdep32((uint32_t)b, qlocal);
        double re = 0.0, im = 0.0;
        for (uint32_t r = 0; r < rows; ++r) {
            const uint32_t bL = pdep32(r, rest);
            const float2 va = tile[swzf(bL | oa)], vb = tile[swzf(bL | ob)];
            // rho[a][b] += psi[a] conj(psi[b])
            re += (double)va.x * vb.x + (double)va.y * vb.y;
            im += (double)va.y * vb.x - (double)va.x * vb.y;
        }
        out[2 * e] = re;
        out[2 * e + 1] = im;
    }
}

// Last tile of a slot, Q >= 4: entry-parallel fixed-order sums of the tile partials,
// written over tile 0's partial (each entry read before it is overwritten by the
// same thread); returns the final rho_Q (global memory).
template <int NT>
__device__ __forceinline__ const double* rho_final_big(double* part, uint32_t ntiles, int stride, int ne) {
    for (int e = threadIdx.x; e < ne; e += NT) {
        double s = 0.0;
        for (uint32_t t = 0; t < ntiles; ++t) s += __ldcg(part + (uint64_t)t * stride + e);
        part[e] = s;
    }
    __threadfence_block();
    return part;
}

// Alg. 2 lines 13-21 for one conventional channel, single thread.
static __device__ __noinline__ void choose_conventional(const EventDesc& E, const ChanDesc& C, const double* cd,
                                    const double* rho /*2*d*d*/, float2* pool, int32_t* records,
                                    int32_t* status) {
    const int d = C.d, nk = C.n_kraus;
    const double* pbar = cd + C.off;
    const double* Mm = pbar + nk;             // M_i = K_i^dag K_i
    const double* Km = Mm + 2 * d * d * nk;   // K_i
    double tr = 0.0;
    for (int a = 0; a < d; ++a) tr += rho[2 * (a * d + a)];
    if (!(tr > 0.0)) { *status = -10; return; }
    double r = E.r;
    double raw[64], w[64];
    int pick = -1;
    for (int i = 0; i < nk; ++i) {
        const double* M = Mm + 2 * d * d * i;
        double s = 0.0;  // Re Tr(M rho) = sum_ab M[a][b] rho[b][a]
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) {
                const double mr = M[2 * (a * d + b)], mi = M[2 * (a * d + b) + 1];
                const double rr = rho[2 * (b * d + a)], ri = rho[2 * (b * d + a) + 1];
                s += mr * rr - mi * ri;
            }
        raw[i] = s;
        const double p = s / tr;
        const double pb = (E.flags & kEventNoBounds) ? 0.0 : pbar[i];  // conventional algorithm: no bounds
        if (p < pb - 1e-6) { *status = -5; return; }
        w[i] = p - pb > 0.0 ? p - pb : 0.0;
        if (r < w[i]) { pick = i; break; }
        r -= w[i];
    }
    if (pick < 0) {
        if (r > 1e-6) { *status = -9; return; }
        for (int i = nk - 1; i >= 0; --i)
            if (w[i] > 0.0) { pick = i; break; }
        if (pick < 0) { *status = -9; return; }
    }
    const double scale = 1.0 / sqrt(raw[pick]);
    const double* K = Km + 2 * d * d * pick;
    for (int e = 0; e < d * d; ++e)
        pool[E.mat_off + e] = make_float2((float)(K[2 * e] * scale), (float)(K[2 * e + 1] * scale));
    if (E.record >= 0) records[E.record] = pick;
}

}  // namespace detail
using namespace detail;

}  // namespace qt

