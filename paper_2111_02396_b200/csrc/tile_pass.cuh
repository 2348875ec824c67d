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
#pragma unroll
    for (int e = 0; e < 2 * D * D; ++e) {
        const double s = block_sum<NT>(acc[e], red);
        if (tid == 0) out[e] = s;
    }
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
        if (p < pbar[i] - 1e-6) { *status = -5; return; }
        w[i] = p - pbar[i] > 0.0 ? p - pbar[i] : 0.0;
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

// ---------------------------------------------------------------------------
// K1 tile pass
// ---------------------------------------------------------------------------
template <int T, int R>
__global__ void __launch_bounds__(1 << (T - R), (R <= 4 && T == 12) ? QT_MINB : 1)
tile_pass_kernel(const TileArgs A, const int step) {
    constexpr int NT = 1 << (T - R);
    constexpr int NA = 1 << R;
    constexpr int TILE = 1 << T;
    constexpr int CL = T < kCL ? T : kCL;
    constexpr int NH = TILE >> CL;
    const int slot = blockIdx.y;
    if (step >= A.pass_count[slot]) return;
    const PassDesc P = A.passes[A.pass_start[slot] + step];

    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* tile = reinterpret_cast<float2*>(smem_raw);
    float2* mbuf = tile + TILE;                                       // 2 x NA*NA
    uint64_t* hoff = reinterpret_cast<uint64_t*>(mbuf + 2 * NA * NA);  // NH (padded to 16 B)
    double* red = reinterpret_cast<double*>(hoff + ((NH + 1) & ~1));  // 64
    GateDesc* gdesc = reinterpret_cast<GateDesc*>(red + 64);          // kMaxPassGates
    __shared__ int s_last;

    const int tid = threadIdx.x;
    const int n = A.n;
    const uint64_t nmask = (n >= 64) ? ~0ull : ((1ull << n) - 1ull);
    const uint64_t base = pdep64((uint64_t)blockIdx.x, nmask & ~P.tile_mask);
    float2* st = A.state + ((uint64_t)slot << n);

    // stage the pass's gate descriptors and the first matrix (async)
    const int ng = P.gate_count;
    for (int c = tid; c < ng; c += NT) cp_async16(gdesc + c, A.gates + P.gate_begin + c);
    cp_async_commit();
    for (int h = tid; h < NH; h += NT) {
        uint64_t o = 0;
#pragma unroll
        for (int i = CL; i < T; ++i) o |= (uint64_t)((h >> (i - CL)) & 1) << P.tq[i];
        hoff[h] = o;
    }
    __syncthreads();
    // HBM -> shared, asynchronous 8-byte copies: 2^CL-amplitude contiguous runs,
    // consecutive threads on consecutive amplitudes
#pragma unroll
    for (int m = 0; m < NA; ++m) {
        const uint32_t L = (uint32_t)(tid + m * NT);
        const uint64_t g = base + hoff[L >> CL] + (L & ((1u << CL) - 1u));
        cp_async8(tile + swz(L), st + g);
    }
    cp_async_commit();
    cp_async_wait_all();  // gate descriptors (the tile may still be in flight for other threads)
    __syncthreads();
    if (ng > 0) {
        const int chunks = (1 << (2 * gdesc[0].k)) >> 1;
        for (int c = tid; c < chunks; c += NT) cp_async16(mbuf + 2 * c, A.pool + gdesc[0].mat_off + 2 * c);
        cp_async_commit();
    }
    for (int gi = 0; gi < ng; ++gi) {
        const GateDesc G = gdesc[gi];
        cp_async_wait_all();
        __syncthreads();  // tile writes of the previous gate + this gate's matrix visible
        if (gi + 1 < ng) {
            const GateDesc Gn = gdesc[gi + 1];
            float2* dst = mbuf + ((gi + 1) & 1) * NA * NA;
            const int chunks = (1 << (2 * Gn.k)) >> 1;
            for (int c = tid; c < chunks; c += NT) cp_async16(dst + 2 * c, A.pool + Gn.mat_off + 2 * c);
            cp_async_commit();
        }
        // register layout (host-computed): register bit m <-> tile bit rpos[m]
        // (bits 0..k-1 = the gate qubits), thread bit i <-> tile bit tpos[i]
        uint32_t unit[R];
#pragma unroll
        for (int m = 0; m < R; ++m) unit[m] = swz(1u << ((G.rpos >> (4 * m)) & 15u)) << 3;
        uint32_t tb = 0;
#pragma unroll
        for (int i = 0; i < T - R; ++i) tb |= (((uint32_t)tid >> i) & 1u) << ((G.tpos >> (4 * i)) & 15u);
        dispatch_fused<R>(G.k, tile, mbuf + (gi & 1) * NA * NA, swz(tb) << 3, unit);
    }
    cp_async_wait_all();  // a pass without gates still has its tile in flight
    __syncthreads();

    // ---- epilogues (read-only on the tile) ----
    const uint32_t ntiles = gridDim.x;
    const uint64_t tile_row = (uint64_t)slot * ntiles + blockIdx.x;
    if (P.flags & kPassRho) {
        const EventDesc E = A.events[P.event];
        const ChanDesc C = A.chans[E.chan];
        const uint64_t qmask = C.qmask;
        const uint32_t ql = to_local<T>(qmask, P);  // channel qubits as tile-local bits
        double* out = A.rho_part + tile_row * A.rho_stride;
        if constexpr (T >= 2) {
            if (C.nq == 1) rho_partial<1, T, NT>(tile, ql, out, red);
            else rho_partial<2, T, NT>(tile, ql, out, red);
        } else {
            rho_partial<1, T, NT>(tile, ql, out, red);
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = (atomicAdd(&A.counters[slot], 1) == (int)ntiles - 1);
        __syncthreads();
        if (s_last) {
            __threadfence();
            const int ne = 2 * C.d * C.d;
            double* fin = red;  // ne <= 32 doubles
            for (int e = tid; e < ne; e += NT) {
                double s = 0.0;
                for (uint32_t t = 0; t < ntiles; ++t)
                    s += __ldcg(A.rho_part + ((uint64_t)slot * ntiles + t) * A.rho_stride + e);
                fin[e] = s;
            }
            __syncthreads();
            if (tid == 0) {
                choose_conventional(E, C, A.chan_data, fin, A.pool, A.records, A.status + slot);
                A.counters[slot] = 0;
            }
        }
    }
    if (P.flags & kPassFinal) {
        double s = 0.0;
#pragma unroll 4
        for (int m = 0; m < NA; ++m) {
            const float2 v = tile[swz((uint32_t)(tid + m * NT))];
            s += (double)v.x * v.x + (double)v.y * v.y;
        }
        s = block_sum<NT>(s, red);
        if (tid == 0) A.blocksum[tile_row] = s;
    }
    if (P.flags & kPassObs) {
        for (int o = 0; o < P.obs_count; ++o) {
            const ObsDesc O = A.obs[P.obs_begin + o];
            const uint64_t xo = O.xmask & ~P.tile_mask;
            const uint32_t xl = to_local<T>(O.xmask, P), zl = to_local<T>(O.zmask, P);
            const int zs = __popcll(base & O.zmask) & 1;
            double s = 0.0;
            if (O.xmask == 0) {  // Z-type string: sum of +-|psi_L|^2 (fp32 per thread, fp64 across)
                float sf = 0.f;
#pragma unroll
                for (int m = 0; m < NA; ++m) {
                    const uint32_t L = (uint32_t)(tid + m * NT);
                    const float2 v = tile[swz(L)];
                    const float p = fmaf(v.x, v.x, v.y * v.y);
                    sf += (__popc(L & zl) & 1) ? -p : p;
                }
                s = zs ? -(double)sf : (double)sf;
            } else
            for (int m = 0; m < NA; ++m) {
                const uint32_t L = (uint32_t)(tid + m * NT);
                const float2 v = tile[swz(L)];
                float2 w;
                if (xo == 0) {
                    w = tile[swz(L ^ xl)];
                } else {  // partner amplitude in another tile (read-only pass only)
                    const uint64_t g = base + hoff[L >> CL] + (L & ((1u << CL) - 1u));
                    w = st[g ^ O.xmask];
                }
                // c = conj(w) * v
                const double cr = (double)w.x * v.x + (double)w.y * v.y;
                const double ci = (double)w.x * v.y - (double)w.y * v.x;
                double t;
                switch (O.ny & 3) {
                    case 0: t = cr; break;
                    case 1: t = -ci; break;
                    case 2: t = -cr; break;
                    default: t = ci; break;
                }
                const int par = (__popc(L & zl) + zs) & 1;
                s += par ? -t : t;
            }
            s = block_sum<NT>(s, red);
            if (tid == 0) A.obs_part[tile_row * A.n_obs + O.slot] = s;
        }
    }

    // ---- shared -> HBM ----
    if (P.flags & kPassStore) {
#pragma unroll
        for (int m = 0; m < NA; ++m) {
            const uint32_t L = (uint32_t)(tid + m * NT);
            const uint64_t g = base + hoff[L >> CL] + (L & ((1u << CL) - 1u));
            st[g] = tile[swz(L)];
        }
    }
}

inline size_t tile_pass_smem_bytes_impl(int T, int R) {
    const int CL = T < kCL ? T : kCL;
    const size_t tile = sizeof(float2) << T;
    const size_t mb = 2 * sizeof(float2) * ((size_t)1 << (2 * R));
    const size_t hoff = sizeof(uint64_t) * ((((size_t)1 << (T - CL)) + 1) & ~(size_t)1);
    return tile + mb + hoff + 64 * sizeof(double) + sizeof(GateDesc) * kMaxPassGates;
}

template <int T, int R>
cudaError_t launch_tr(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    const size_t smem = tile_pass_smem_bytes_impl(T, R);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(tile_pass_kernel<T, R>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid(ntiles, nslots);
    tile_pass_kernel<T, R><<<grid, 1 << (T - R), smem, s>>>(a, step);
    return cudaGetLastError();
}

}  // namespace qt
