// kernels.cu -- sm_100a kernels of the noisy-trajectory hot path.
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
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.hpp"
#include "philox.hpp"
#include "tile_pass_kernel.cuh"

namespace qt {

// Tile-pass instantiations live in tile_pass_{r4,r5,r6,tc}.cu (parallel compile).
cudaError_t launch_tile_pass_r4(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s);
cudaError_t launch_tile_pass_r5(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s);
cudaError_t launch_tile_pass_r5s(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s);
cudaError_t launch_tile_pass_r6s_a(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s);
cudaError_t launch_tile_pass_r6s_b(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s);
cudaError_t launch_tile_pass_r6(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s);
cudaError_t launch_tile_pass_tc(const TileArgs& a, int tck, int step, uint32_t ntiles, int nslots, cudaStream_t s);
cudaError_t launch_tile_pass_v2(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s);

size_t tile_pass_smem_bytes(int T, int R, int tck) { return tile_pass_smem_bytes_impl(T, R, tck != 0, tck ? tck : 4); }

cudaError_t launch_tile_pass(const TileArgs& a, int R, int tck, int step, uint32_t ntiles, int nslots,
                             cudaStream_t s) {
    // Instantiated (T, R): (12, 4), (12, 5), (12, 6), (T, min(T, 4)) for
    // T = 1..11 (the whole state of n < 12 qubits in one CTA) and (T, 5 | 6) for
    // T = R..11 (5- and 6-qubit gates on small registers); tensor cores
    // (tck = 4, 5 or 6 qubits per padded gate): (12, 5).
    if (a.T == 11 && a.v3maps) return tck == 4 ? launch_tile_pass_v3(a, a.v3maps, step, ntiles, nslots, s) : cudaErrorInvalidValue;
    if (a.T == 13) return tck == 4 ? launch_tile_pass_v2(a, step, ntiles, nslots, s) : cudaErrorInvalidValue;
    if (tck) return a.T == 12 && R == 5 ? launch_tile_pass_tc(a, tck, step, ntiles, nslots, s) : cudaErrorInvalidValue;
    if (a.T == 12 && R == 6) return launch_tile_pass_r6(a, step, ntiles, nslots, s);
    if (a.T == 12 && R == 5) return launch_tile_pass_r5(a, step, ntiles, nslots, s);
    if (a.T < 12 && R == 5) return launch_tile_pass_r5s(a, step, ntiles, nslots, s);
    if (a.T < 12 && R == 6) return a.T <= 8 ? launch_tile_pass_r6s_a(a, step, ntiles, nslots, s)
                                            : launch_tile_pass_r6s_b(a, step, ntiles, nslots, s);
    if (R == (a.T < 4 ? a.T : 4)) return launch_tile_pass_r4(a, step, ntiles, nslots, s);
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// K6 fused-matrix materialization (fp64), one CTA per fused gate: the D x D
// product of the constituents (time order) is built in shared memory, one
// thread per matrix element (r, c) per step: V <- (I (x) C_j) V, i.e.
// V'[r][c] = sum_a C_j[r_j][a] V[r with its constituent bits := a][c].
// ---------------------------------------------------------------------------
constexpr int kMatThreads = 256;

__global__ void __launch_bounds__(kMatThreads)
materialize_kernel(const FusedDesc* __restrict__ fused, const ConsDesc* __restrict__ cons,
                   const VarDesc* __restrict__ vars, const double2* __restrict__ var_data,
                   float2* __restrict__ pool) {
    extern __shared__ double2 sm2[];  // two D x D buffers
    const FusedDesc F = fused[blockIdx.x];
    const bool tcm = (F.k & kGateTC) != 0;
    const int k = F.k & 0xff;
    const int D = 1 << k;
    const int DD = D * D;
    double2* v = sm2;
    double2* nv = sm2 + DD;
    for (int e = threadIdx.x; e < DD; e += kMatThreads)
        v[e] = make_double2((e / D) == (e % D) ? 1.0 : 0.0, 0.0);
    __syncthreads();
    for (int j = 0; j < F.cons_count; ++j) {
        const ConsDesc C = cons[F.cons_begin + j];
        const VarDesc Vd = vars[C.var];
        const int q = Vd.nq;
        const int dq = 1 << q;
        uint32_t qm = 0;
        int pos[6];
        for (int m = 0; m < q; ++m) {
            pos[m] = (C.pos >> (4 * m)) & 15;
            qm |= 1u << pos[m];
        }
        const double2* M = var_data + Vd.off;
        for (int e = threadIdx.x; e < DD; e += kMatThreads) {
            const int r = e / D, c = e % D;
            int rl = 0;
            for (int m = 0; m < q; ++m) rl |= ((r >> pos[m]) & 1) << m;
            const int base = r & ~(int)qm;
            double re = 0.0, im = 0.0;
            for (int al = 0; al < dq; ++al) {
                int o = base;
                for (int m = 0; m < q; ++m)
                    if ((al >> m) & 1) o |= 1 << pos[m];
                const double2 u = M[rl * dq + al];
                const double2 x = v[o * D + c];
                re += u.x * x.x - u.y * x.y;
                im += u.x * x.y + u.y * x.x;
            }
            nv[e] = make_double2(re, im);
        }
        __syncthreads();
        double2* t = v;
        v = nv;
        nv = t;
    }
    // element (j, c) of the fused matrix U = v[j * D + c]
    if (!tcm) {
        for (int e = threadIdx.x; e < DD; e += kMatThreads)
            pool[F.mat_off + e] = make_float2((float)v[e].x, (float)v[e].y);
        return;
    }
    if (F.k & kGateV2) {
        // persistent TMEM kernel operand (desc.hpp kV2GateBytes): B row n = 2j + b holds
        // W[n][2c + a] = blk[a][b] of U[j][c] as f16 hi (bytes 0..63) and lo (64..127),
        // SWIZZLE_128B K-major, 32 rows
        __half* B = reinterpret_cast<__half*>(pool + F.mat_off);
        for (int e = threadIdx.x; e < DD; e += kMatThreads) {
            const int jj = e / D, c = e % D;
            const double ur = v[e].x, ui = v[e].y;
            const double blk[2][2] = {{ur, ui}, {-ui, ur}};
            for (int a2 = 0; a2 < 2; ++a2)
                for (int b = 0; b < 2; ++b) {
                    const double w = blk[a2][b];
                    const __half h = __double2half(w);
                    const __half l = __double2half(w - (double)__half2float(h));
                    B[tc::sw128_offset(2 * jj + b, 2 * (2 * c + a2)) >> 1] = h;
                    B[tc::sw128_offset(2 * jj + b, 64 + 2 * (2 * c + a2)) >> 1] = l;
                }
        }
        return;
    }
    if (k == 4 && (F.k & kGateF16)) {
        // kind::f16 operand B (tc_common.cuh): B[2j + b][4c + q] = hi(blk[q & 1][b]),
        // B[32 + 2j + b][4c + q] = lo(blk[q & 1][b]) for q < 2, 0 for q >= 2, with
        // blk the real 2x2 block of U[j][c] (input component a, output component b).
        __half* B = reinterpret_cast<__half*>(pool + F.mat_off);
        for (int e = threadIdx.x; e < DD; e += kMatThreads) {
            const int jj = e / D, c = e % D;
            const double ur = v[e].x, ui = v[e].y;
            const double blk[2][2] = {{ur, ui}, {-ui, ur}};
            for (int b = 0; b < 2; ++b)
                for (int q = 0; q < 4; ++q) {
                    const double w = blk[q & 1][b];
                    const __half h = __double2half(w);
                    const __half l = __double2half(w - (double)__half2float(h));
                    const int kk = 4 * c + q;
                    B[tc::sw128_offset(2 * jj + b, 2 * kk) >> 1] = h;
                    B[tc::sw128_offset(32 + 2 * jj + b, 2 * kk) >> 1] = q < 2 ? l : __float2half(0.f);
                }
        }
        return;
    }
    if (k >= 5) {
        // wide f16 operand B (tc_common.cuh): B[2j + b][2c + a] = blk[a][b] of
        // U[j][c], hi part and lo (remainder) part
        __half* B = reinterpret_cast<__half*>(pool + F.mat_off);
        for (int e = threadIdx.x; e < DD; e += kMatThreads) {
            const int jj = e / D, c = e % D;
            const double ur = v[e].x, ui = v[e].y;
            const double blk[2][2] = {{ur, ui}, {-ui, ur}};
            for (int a2 = 0; a2 < 2; ++a2)
                for (int b = 0; b < 2; ++b) {
                    const double w = blk[a2][b];
                    const __half h = __double2half(w);
                    const __half l = __double2half(w - (double)__half2float(h));
                    B[tc::wide_b_offset(k, 0, 2 * jj + b, 2 * c + a2) >> 1] = h;
                    B[tc::wide_b_offset(k, 1, 2 * jj + b, 2 * c + a2) >> 1] = l;
                }
        }
        return;
    }
    // 3xTF32 operand W (tc_common.cuh; single 4-qubit gates): W[2c + a][2j + b] =
    // real 2x2 block of U[j][c], stored K-major swizzled as hi then lo tf32 parts
    uint32_t* W = reinterpret_cast<uint32_t*>(pool + F.mat_off);
    const uint32_t part = (uint32_t)tc::w_part_bytes(k) >> 2;
    for (int e = threadIdx.x; e < DD; e += kMatThreads) {
        const int jj = e / D, c = e % D;
        const double ur = v[e].x, ui = v[e].y;
        const double blk[2][2] = {{ur, ui}, {-ui, ur}};
        for (int a2 = 0; a2 < 2; ++a2)
            for (int b = 0; b < 2; ++b) {
                const float w = (float)blk[a2][b];
                const uint32_t h = tc::tf32_rna(w);
                const uint32_t l = tc::tf32_rna(w - __uint_as_float(h));
                const uint32_t off = tc::w_offset_bytes_k(k, 2 * jj + b, 2 * c + a2) >> 2;
                W[off] = h;
                W[part + off] = l;
            }
    }
}

cudaError_t launch_materialize(const FusedDesc* fused, int n_fused, int max_k, const ConsDesc* cons,
                               const VarDesc* vars, const double* var_data, float2* pool, cudaStream_t s) {
    if (n_fused <= 0) return cudaSuccess;
    const int kk = max_k < 1 ? 1 : (max_k > 6 ? 6 : max_k);
    const size_t smem = 2 * sizeof(double2) * ((size_t)1 << (2 * kk));
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(materialize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(2 * sizeof(double2) * 64 * 64));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    materialize_kernel<<<n_fused, kMatThreads, smem, s>>>(fused, cons, vars, reinterpret_cast<const double2*>(var_data),
                                                           pool);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K4 finalize: norm = sum of block sums, obs = sum of partials / norm, in a
// fixed order (one CTA per trajectory slot).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
finalize_obs_kernel(const double* __restrict__ blocksum, const double* __restrict__ obs_part,
                    int ntiles, int n_obs, double* __restrict__ out_obs, double* __restrict__ out_norm) {
    __shared__ double red[64];
    const int slot = blockIdx.x;
    const int tid = threadIdx.x;
    double s = 0.0;
    for (int t = tid; t < ntiles; t += 256) s += blocksum[(uint64_t)slot * ntiles + t];
    const double norm = block_sum<256>(s, red);
    if (tid == 0 && out_norm) out_norm[slot] = norm;
    for (int o = 0; o < n_obs; ++o) {
        double p = 0.0;
        for (int t = tid; t < ntiles; t += 256) p += obs_part[((uint64_t)slot * ntiles + t) * n_obs + o];
        const double tot = block_sum<256>(p, red);
        if (tid == 0) out_obs[(uint64_t)slot * n_obs + o] = tot / norm;
    }
}

cudaError_t launch_finalize_obs(const double* blocksum, const double* obs_part, int ntiles,
                                int n_obs, int nslots, double* out_obs, double* out_norm,
                                cudaStream_t s) {
    if (nslots <= 0) return cudaSuccess;
    finalize_obs_kernel<<<nslots, 256, 0, s>>>(blocksum, obs_part, ntiles, n_obs, out_obs, out_norm);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K3 sampler: one warp per (slot, shot).  Chain rule, most significant qubit
// first: bit = 0 iff u * (M0 + M1) < M0; M0 == 0 -> 1; M1 == 0 -> 0.  Levels
// n-1..T use the fp64 block sums of the contiguous 2^T-amplitude tiles, levels
// T-1..0 read the chosen tile.  Then readout flips.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-sum heap of a slot (registers with many tiles): node 1 = the whole state, node i's
// children 2i, 2i + 1 = its lower / upper half, leaves 2^(n-T) + tile = the block sums, so
// the sampler's global levels read two nodes per level instead of re-summing the leaves of
// the current prefix for every shot (pairwise sums, fp64).
__global__ void __launch_bounds__(256) blocksum_heap_kernel(const double* __restrict__ blocksum, int lg,
                                                            double* __restrict__ heap) {
    const uint64_t nt = 1ull << lg;
    const double* bs = blocksum + (uint64_t)blockIdx.x * nt;
    double* h = heap + (uint64_t)blockIdx.x * 2 * nt;
    for (uint64_t i = threadIdx.x; i < nt; i += blockDim.x) h[nt + i] = bs[i];
    __syncthreads();
    for (int d = lg - 1; d >= 0; --d) {
        const uint64_t b = 1ull << d;
        for (uint64_t i = b + threadIdx.x; i < 2 * b; i += blockDim.x) h[i] = h[2 * i] + h[2 * i + 1];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(128)
sample_kernel(const float2* __restrict__ state, int n, int T, const double* __restrict__ blocksum,
              int nslots, int shots, uint64_t seed, const uint64_t* __restrict__ traj_ids,
              const double* __restrict__ p00, const double* __restrict__ p11,
              uint64_t* __restrict__ out_bits, int n_rng, const int32_t* __restrict__ shot_ids,
              const double* __restrict__ heap) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= nslots * shots) return;
    const int slot = gw / shots;
    // distributed-state sampling: shot ids and the RNG's qubit count are the
    // whole register's (the local levels are its low n qubits)
    const int shot = shot_ids ? shot_ids[gw % shots] : gw % shots;
    const uint64_t traj = traj_ids[slot];
    const int half_n = ((n_rng > 0 ? n_rng : n) + 1) / 2;
    const uint64_t ntiles = 1ull << (n - T);
    const double* bs = blocksum + (uint64_t)slot * ntiles;
    uint64_t lo = 0;  // prefix (tile index range [lo, lo + 2^(l-T+1)))
    uint64_t bits = 0;
    for (int l = n - 1; l >= T; --l) {
        const uint64_t half = 1ull << (l - T);
        double m0 = 0.0, m1 = 0.0;
        if (heap) {
            // node of the current prefix at depth n - 1 - l, its two children
            const double* h = heap + (uint64_t)slot * 2 * ntiles;
            const uint64_t node = (1ull << (n - 1 - l)) + (lo >> (l - T + 1));
            m0 = h[2 * node];
            m1 = h[2 * node + 1];
        } else {
            for (uint64_t i = lane; i < half; i += 32) {
                m0 += bs[lo + i];
                m1 += bs[lo + half + i];
            }
            m0 = warp_sum(m0);
            m1 = warp_sum(m1);
        }
        const double u = draw(seed, (uint32_t)(shot * half_n + l / 2), kPurposeSample, traj, l & 1);
        int bit;
        if (m0 == 0.0) bit = 1;
        else if (m1 == 0.0) bit = 0;
        else bit = (u * (m0 + m1) < m0) ? 0 : 1;
        if (bit) {
            lo += half;
            bits |= 1ull << l;
        }
    }
    const float2* tl = state + ((uint64_t)slot << n) + (lo << T);
    uint32_t off = 0;
    for (int l = T - 1; l >= 0; --l) {
        const uint32_t half = 1u << l;
        double m0 = 0.0, m1 = 0.0;
        for (uint32_t i = lane; i < half; i += 32) {
            const float2 a = tl[off + i];
            const float2 b = tl[off + half + i];
            m0 += (double)a.x * a.x + (double)a.y * a.y;
            m1 += (double)b.x * b.x + (double)b.y * b.y;
        }
        m0 = warp_sum(m0);
        m1 = warp_sum(m1);
        const double u = draw(seed, (uint32_t)(shot * half_n + l / 2), kPurposeSample, traj, l & 1);
        int bit;
        if (m0 == 0.0) bit = 1;
        else if (m1 == 0.0) bit = 0;
        else bit = (u * (m0 + m1) < m0) ? 0 : 1;
        if (bit) {
            off += half;
            bits |= 1ull << l;
        }
    }
    if (lane == 0) {
        uint64_t out = bits;
        if (p00 || p11) {
            for (int q = 0; q < n; ++q) {
                const double u = draw(seed, (uint32_t)(shot * half_n + q / 2), kPurposeReadout, traj, q & 1);
                const int b = (int)((bits >> q) & 1);
                if (b == 0 && p00 && u < p00[q]) out |= 1ull << q;
                if (b == 1 && p11 && u < p11[q]) out &= ~(1ull << q);
            }
        }
        out_bits[(uint64_t)slot * shots + (gw % shots)] = out;  // position in the request, not the shot id
    }
}

cudaError_t launch_sample(const float2* state, int n, int T, const double* blocksum, int nslots,
                          int shots, uint64_t seed, const uint64_t* traj_ids, const double* p00,
                          const double* p11, uint64_t* out_bits, cudaStream_t s, int n_rng,
                          const int32_t* shot_ids, double* heap) {
    const long warps = (long)nslots * shots;
    if (warps <= 0) return cudaSuccess;
    if (heap) blocksum_heap_kernel<<<nslots, 256, 0, s>>>(blocksum, n - T, heap);
    const int threads = 128;
    const long blocks = (warps * 32 + threads - 1) / threads;
    sample_kernel<<<(unsigned)blocks, threads, 0, s>>>(state, n, T, blocksum, nslots, shots, seed,
                                                       traj_ids, p00, p11, out_bits, n_rng, shot_ids, heap);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// rho_Q of a few local qubits over a whole state (distributed-state mode): fixed
// grid, fp64 per-block partials, then a fixed-order final sum (deterministic).
// rho[a][b] = sum_rest psi[rest, a] conj(psi[rest, b]), a/b in internal order
// (bit m <-> the m-th lowest qubit of qmask).
// ---------------------------------------------------------------------------
constexpr int kRhoBlocks = 296;

__global__ void __launch_bounds__(256)
rho_reduce_kernel(const float2* __restrict__ state, int n, uint64_t qmask, int q, double* __restrict__ partial) {
    __shared__ double red[8];
    const int d = 1 << q;
    uint64_t qoff[4];
    for (int a = 0; a < d; ++a) {
        uint64_t o = 0, m = qmask;
        int bit = 0;
        while (m) {
            const uint64_t low = m & (~m + 1);
            if ((a >> bit) & 1) o |= low;
            ++bit;
            m ^= low;
        }
        qoff[a] = o;
    }
    double acc[32];
    for (int e = 0; e < 32; ++e) acc[e] = 0.0;
    const uint64_t total = 1ull << n;
    for (uint64_t g = (uint64_t)blockIdx.x * 256 + threadIdx.x; g < total; g += (uint64_t)gridDim.x * 256) {
        if (g & qmask) continue;
        double vr[4], vi[4];
        for (int a = 0; a < d; ++a) {
            const float2 v = state[g | qoff[a]];
            vr[a] = v.x;
            vi[a] = v.y;
        }
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) {
                acc[2 * (a * d + b)] += vr[a] * vr[b] + vi[a] * vi[b];
                acc[2 * (a * d + b) + 1] += vi[a] * vr[b] - vr[a] * vi[b];
            }
    }
    for (int e = 0; e < 2 * d * d; ++e) {
        const double s = block_sum<256>(acc[e], red);
        if (threadIdx.x == 0) partial[(size_t)blockIdx.x * 32 + e] = s;
    }
}

// rho_Q of 3..6 qubits (D = 2^q up to 64): block b owns the fixed range of "rest"
// indices [b R / B, (b + 1) R / B), stages 32 rows of D amplitudes in shared memory
// and every thread accumulates whole entries (a, b) in a fixed order.
__global__ void __launch_bounds__(256)
rho_reduce_big_kernel(const float2* __restrict__ state, int n, uint64_t qmask, int q, double* __restrict__ partial,
                      int stride) {
    extern __shared__ float2 xs[];  // [32][D]
    const int D = 1 << q;
    const uint64_t rows = 1ull << (n - q);
    const uint64_t r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
    int qp[6];
    {
        uint64_t m = qmask;
        for (int j = 0; j < q; ++j) {
            qp[j] = __ffsll((long long)m) - 1;
            m &= m - 1;
        }
    }
    double acc[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) acc[k] = 0.0;
    for (uint64_t rc = r0; rc < r1; rc += 32) {
        const int nr = (int)((r1 - rc) < 32 ? (r1 - rc) : 32);
        for (int idx = threadIdx.x; idx < nr * D; idx += 256) {
            const int r = idx / D, a = idx % D;
            uint64_t g = rc + (uint64_t)r;  // insert the channel bits (ascending positions)
            for (int j = 0; j < q; ++j) {
                const uint64_t low = g & ((1ull << qp[j]) - 1ull);
                g = low | ((g ^ low) << 1) | ((uint64_t)((a >> j) & 1) << qp[j]);
            }
            xs[idx] = state[g];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int e = threadIdx.x + 256 * k;
            if (e < D * D) {
                const int a = e / D, b = e % D;
                double re = acc[2 * k], im = acc[2 * k + 1];
                for (int r = 0; r < nr; ++r) {
                    const float2 va = xs[r * D + a], vb = xs[r * D + b];
                    re += (double)va.x * vb.x + (double)va.y * vb.y;
                    im += (double)va.y * vb.x - (double)va.x * vb.y;
                }
                acc[2 * k] = re;
                acc[2 * k + 1] = im;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int e = threadIdx.x + 256 * k;
        if (e < D * D) {
            partial[(size_t)blockIdx.x * stride + 2 * e] = acc[2 * k];
            partial[(size_t)blockIdx.x * stride + 2 * e + 1] = acc[2 * k + 1];
        }
    }
}

__global__ void rho_final_big_kernel(const double* __restrict__ partial, int ne, int stride, double* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < kRhoBlocks; ++b) s += partial[(size_t)b * stride + e];
        out[e] = s;
    }
}

__global__ void rho_final_kernel(const double* __restrict__ partial, int ne, double* __restrict__ out) {
    const int e = threadIdx.x;
    if (e >= ne) return;
    double s = 0.0;
    for (int b = 0; b < kRhoBlocks; ++b) s += partial[(size_t)b * 32 + e];
    out[e] = s;
}

// Qubit permutation copy: dst[pi(i)] = src[i], bit j of i moves to bit perm[j]
// (distributed-state mode: gathers the swapped local qubits into the top bits).
struct QubitPerm {
    uint8_t p[48];  // destination bit of source bit b
};

// Bits that stay in place are copied with one mask; only moved bits are
// visited, so a swap of the top local bits costs a few operations per element
// and keeps the low bits (coalescing) intact.
__global__ void __launch_bounds__(256)
permute_qubits_kernel(const float2* __restrict__ src, float2* __restrict__ dst, int n, uint64_t fixed_mask,
                      int n_moved, const QubitPerm moved_src, const QubitPerm moved_dst) {
    const uint64_t total = 1ull << n;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < total; i += (uint64_t)gridDim.x * 256) {
        uint64_t j = i & fixed_mask;
        for (int k = 0; k < n_moved; ++k) j |= ((i >> moved_src.p[k]) & 1ull) << moved_dst.p[k];
        dst[j] = src[i];
    }
}

cudaError_t launch_permute_qubits(const float2* src, float2* dst, int n, const int* perm, cudaStream_t s) {
    if (n > 48) return cudaErrorInvalidValue;
    QubitPerm ms{}, md{};
    uint64_t fixed = 0;
    int nm = 0;
    for (int b = 0; b < n; ++b) {
        if (perm[b] == b) {
            fixed |= 1ull << b;
        } else {
            ms.p[nm] = (uint8_t)b;
            md.p[nm] = (uint8_t)perm[b];
            ++nm;
        }
    }
    const uint64_t total = 1ull << n;
    const unsigned blocks = (unsigned)std::min<uint64_t>((total + 255) / 256, 148 * 32);
    permute_qubits_kernel<<<blocks, 256, 0, s>>>(src, dst, n, fixed, nm, ms, md);
    return cudaGetLastError();
}

cudaError_t launch_rho_reduce(const float2* state, int n, uint64_t qmask, int q, double* partial, double* out,
                              cudaStream_t s) {
    if (q >= 3) {
        const int D = 1 << q, stride = 2 * D * D;
        rho_reduce_big_kernel<<<kRhoBlocks, 256, sizeof(float2) * 32 * D, s>>>(state, n, qmask, q, partial, stride);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        rho_final_big_kernel<<<(stride + 255) / 256, 256, 0, s>>>(partial, stride, stride, out);
        return cudaGetLastError();
    }
    rho_reduce_kernel<<<kRhoBlocks, 256, 0, s>>>(state, n, qmask, q, partial);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    rho_final_kernel<<<1, 32, 0, s>>>(partial, 2 << (2 * q), out);
    return cudaGetLastError();
}

}  // namespace qt

namespace qt {

// |0...0> in every slot (after a memset to zero).
__global__ void init_states_kernel(float2* state, int n, int nslots) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nslots) state[(uint64_t)b << n] = make_float2(1.f, 0.f);
}

cudaError_t launch_init_states(float2* state, int n, int nslots, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(state, 0, sizeof(float2) * ((size_t)nslots << n), s);
    if (e != cudaSuccess) return e;
    init_states_kernel<<<(nslots + 127) / 128, 128, 0, s>>>(state, n, nslots);
    return cudaGetLastError();
}

}  // namespace qt
