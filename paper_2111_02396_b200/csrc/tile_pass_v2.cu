// tile_pass_v2.cu -- K1, persistent TMEM kernel: Alg. 1 applied to a
// whole program of fused 4-qubit gates per HBM sweep, for n >= 13 qubits.
//
// One CTA per SM walks the step's (trajectory, tile) items.  A tile = the 2^13
// amplitudes spanned by PassDesc::tile_mask (qubits 0..3 always included, so HBM
// rows are 128-byte runs), 64 KB of complex64 in a swizzled shared-memory buffer.
//   warp 8      loader: 16-byte cp.async of the next tile into a free buffer of
//               three, completing on the buffer's "full" mbarrier.
//   warps 0..3  compute warpgroup 0 }  each owns 256 TMEM columns and processes
//   warps 4..7  compute warpgroup 1 }  every other item: while one waits for its
//               MMAs the other runs its epilogue on the shared tensor core.
// A fused gate U (16 x 16 complex) on a tile is the real GEMM, per group j of
// 128 subvectors (rows = TMEM lanes), D = x_hi W_hi + x_lo W_hi + x_hi W_lo with
// f16 hi / lo splits (~22 significant bits, fp32 accumulate): six M128 N32 K16
// tcgen05.mma with A = [x_hi | x_lo] in TMEM (TS) and B = [W_hi | W_lo] (4 KB,
// bulk-copied) in shared memory.  Gates whose qubits, together, fit in the 6
// thread-local tile bits (4 matrix bits + 2 group bits) form a segment: the next
// gate's A is built from this gate's D inside TMEM (tcgen05.ld of the source
// columns, split, tcgen05.st), so the tile touches shared memory only at the
// segment ends (gather / write back).  Then the K2 / K3a / K4 epilogues and the
// 16-byte stores.  Reductions use fixed orders (no float atomics).
#include <cuda_fp16.h>

#include "tile_pass.cuh"

namespace qt {
namespace v2 {

constexpr int T = 13;
constexpr int TILE = 1 << T;
constexpr uint32_t kTileBytes = TILE * 8;  // 64 KB
constexpr int NBUF = 3;
constexpr int NWG = 2;
constexpr int NT = 128;  // threads per compute warpgroup
constexpr int NA = TILE / NT;  // 64 amplitudes per thread
constexpr int kThreads = (4 * NWG + 1) * 32;
constexpr uint32_t kWOff = NBUF * kTileBytes;
constexpr uint32_t kRedOff = kWOff + NWG * 2 * kV2GateBytes;
constexpr uint32_t kMbarOff = kRedOff + NWG * 64 * 8;
constexpr uint32_t kMiscOff = kMbarOff + 16 * 8;
constexpr size_t kSmemBytes = kMiscOff + 64 + 1024;  // + alignment slack

// fp32 tile slot of amplitude L (8-byte units): bits 1..3 ^= bits 4..6 ^ 7..9 ^ 10..12;
// bit 0 is kept so amplitude pairs stay adjacent and 16-byte aligned (cp.async 16).
__device__ __forceinline__ uint32_t swz(uint32_t L) { return L ^ ((((L >> 4) ^ (L >> 7) ^ (L >> 10)) & 7u) << 1); }

__device__ __forceinline__ void bar_wg(int wg) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + wg), "r"(NT) : "memory");
}

__device__ __forceinline__ void mbar_wait_s(uint32_t a, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a), "r"(phase) : "memory");
}
__device__ __forceinline__ void mbar_init_s(uint32_t a, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t a) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t a) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void cp_async16_s(uint32_t s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void bulk_w(uint32_t dst, const void* src, uint32_t mbar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"((uint32_t)kV2GateBytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"((uint32_t)kV2GateBytes), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
    constexpr uint32_t idesc = tc::idesc_f16_m128(32);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t& a, uint32_t& b) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n" : "=r"(a), "=r"(b) : "r"(taddr) : "memory");
}

// f16 hi / lo split of a scaled complex amplitude: hi = x with the 13 low mantissa
// bits cleared (exact in f16 above 2^-14), lo = the remainder rounded to f16.
__device__ __forceinline__ void split(float re, float im, uint32_t& hi, uint32_t& lo) {
    const float hr = __uint_as_float(__float_as_uint(re) & 0xFFFFE000u);
    const float hm = __uint_as_float(__float_as_uint(im) & 0xFFFFE000u);
    const __half2 h2 = __floats2half2_rn(hr, hm);
    const __half2 l2 = __floats2half2_rn(re - hr, im - hm);
    hi = *reinterpret_cast<const uint32_t*>(&h2);
    lo = *reinterpret_cast<const uint32_t*>(&l2);
}

// Deterministic warpgroup sums (fixed order: lanes by xor tree, then warps 0..3).
template <int N>
__device__ __forceinline__ void wg_sum_n(double (&v)[N], double* red, int wg) {
    const int wtid = threadIdx.x & (NT - 1);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    constexpr int C = 16;  // values per chunk (red: 64 doubles = 4 warps x 16)
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += C) {
        bar_wg(wg);
        if ((wtid & 31) == 0)
#pragma unroll
            for (int i = c0; i < N && i < c0 + C; ++i) red[(wtid >> 5) * C + (i - c0)] = v[i];
        bar_wg(wg);
#pragma unroll
        for (int i = c0; i < N && i < c0 + C; ++i) v[i] = red[i - c0] + red[C + i - c0] + red[2 * C + i - c0] + red[3 * C + i - c0];
    }
}

// rho_Q partial (2^Q x 2^Q, fp64) of the tile for a channel at tile-local bits qlocal.
template <int Q>
__device__ __forceinline__ void rho_partial(const float2* tile, uint32_t qlocal, double* out, double* red, int wg) {
    constexpr int D = 1 << Q;
    const int wtid = threadIdx.x & (NT - 1);
    uint32_t qoff[D];
#pragma unroll
    for (int a = 0; a < D; ++a) qoff[a] = pdep32((uint32_t)a, qlocal);
    double acc[2 * D * D];
#pragma unroll
    for (int e = 0; e < 2 * D * D; ++e) acc[e] = 0.0;
    for (uint32_t bL = wtid; bL < (uint32_t)TILE; bL += NT) {
        if (bL & qlocal) continue;
        double vr[D], vi[D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const float2 v = tile[swz(bL | qoff[a])];
            vr[a] = v.x;
            vi[a] = v.y;
        }
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = 0; b < D; ++b) {
                acc[2 * (a * D + b)] += vr[a] * vr[b] + vi[a] * vi[b];
                acc[2 * (a * D + b) + 1] += vi[a] * vr[b] - vr[a] * vi[b];
            }
    }
    wg_sum_n<2 * D * D>(acc, red, wg);
    if (wtid == 0)
#pragma unroll
        for (int e = 0; e < 2 * D * D; ++e) out[e] = acc[e];
}

// 3-qubit channels: one row of rho_Q at a time.
__device__ __forceinline__ void rho_partial_rows3(const float2* tile, uint32_t qlocal, double* out, double* red,
                                                  int wg) {
    constexpr int D = 8;
    const int wtid = threadIdx.x & (NT - 1);
    uint32_t qoff[D];
#pragma unroll
    for (int a = 0; a < D; ++a) qoff[a] = pdep32((uint32_t)a, qlocal);
#pragma unroll 1
    for (int a = 0; a < D; ++a) {
        double acc[2 * D];
#pragma unroll
        for (int e = 0; e < 2 * D; ++e) acc[e] = 0.0;
        for (uint32_t bL = wtid; bL < (uint32_t)TILE; bL += NT) {
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
        wg_sum_n<2 * D>(acc, red, wg);
        if (wtid == 0)
#pragma unroll
            for (int e = 0; e < 2 * D; ++e) out[2 * D * a + e] = acc[e];
    }
}

struct Item {
    const PassDesc* p;
    int slot;
    uint32_t tile;
};

// Item i of the step: slot index i >> tshift, tile i & (ntiles - 1); nullptr pass =
// the slot has no pass at this step (slot-table launches).
__device__ __forceinline__ Item item_of(const TileArgs& A, int step, uint32_t i, int tshift) {
    Item it;
    const int si = (int)(i >> tshift);
    it.tile = i & ((1u << tshift) - 1u);
    if (A.step_passes) {
        it.p = A.step_passes + si;
        it.slot = it.p->slot;
    } else {
        it.slot = si;
        it.p = step < A.pass_count[si] ? A.passes + A.pass_start[si] + step : nullptr;
    }
    return it;
}

// global base index of a tile: the tile index with a zero inserted at every tile qubit
__device__ __forceinline__ uint64_t tile_base(const PassDesc& P, uint32_t tile) {
    uint64_t base = tile;
#pragma unroll
    for (int i = 0; i < T; ++i) {
        const uint64_t low = base & ((1ull << P.tq[i]) - 1ull);
        base = low | ((base ^ low) << 1);
    }
    return base;
}

__global__ void __launch_bounds__(kThreads, 1) tile_pass_v2_kernel(const TileArgs A, const int step,
                                                                    const uint32_t nitems, const int tshift) {
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw_s = (uint32_t)__cvta_generic_to_shared(smem_raw);
    unsigned char* sm = smem_raw + (((raw_s + 1023u) & ~1023u) - raw_s);
    const uint32_t sm_s = (uint32_t)__cvta_generic_to_shared(sm);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t mb = sm_s + kMbarOff;  // full[3], empty[3], mma[2], wfull[2][2]
    auto full_bar = [&](int b) { return mb + 8u * (uint32_t)b; };
    auto empty_bar = [&](int b) { return mb + 8u * (uint32_t)(3 + b); };
    auto mma_bar = [&](int w) { return mb + 8u * (uint32_t)(6 + w); };
    auto wfull_bar = [&](int w, int i) { return mb + 8u * (uint32_t)(8 + 2 * w + i); };
    uint32_t* misc = reinterpret_cast<uint32_t*>(sm + kMiscOff);  // [0] tmem base, [1..2] last flags
    if (warp == 0) {
        tc::tmem_alloc(misc, 512);
    }
    if (tid == 32) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init_s(full_bar(b), 32);
            mbar_init_s(empty_bar(b), 1);
        }
        for (int w = 0; w < NWG; ++w) {
            mbar_init_s(mma_bar(w), 1);
            mbar_init_s(wfull_bar(w, 0), 1);
            mbar_init_s(wfull_bar(w, 1), 1);
        }
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = misc[0];
    const int n = A.n;
    const uint32_t ntiles = 1u << tshift;

    if (warp == 4 * NWG) {
        // ---------------- loader ----------------
        int j = 0;
        for (uint32_t i = blockIdx.x; i < nitems; i += gridDim.x) {
            const Item it = item_of(A, step, i, tshift);
            if (!it.p) continue;
            const int b = j % NBUF;
            if (j >= NBUF) mbar_wait_s(empty_bar(b), (uint32_t)((j / NBUF - 1) & 1));
            const PassDesc& P = *it.p;
            const uint32_t buf = sm_s + (uint32_t)b * kTileBytes;
            if (P.flags & kPassInit) {
                // first pass of a trajectory: |0...0> (amplitude 0 lives in tile 0, slot 0)
                float4* t4 = reinterpret_cast<float4*>(sm + (size_t)b * kTileBytes);
                for (int k = lane; k < TILE / 2; k += 32) t4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
                __syncwarp();
                if (lane == 0 && it.tile == 0) t4[0] = make_float4(1.f, 0.f, 0.f, 0.f);
                mbar_arrive_s(full_bar(b));
            } else {
                const float2* st = A.state + ((uint64_t)it.slot << n) + tile_base(P, it.tile);
                // lane: pair p = lane & 7 of run h = 4 it + (lane >> 3); h bits 0, 1 fixed
                const int p = lane & 7;
                const uint32_t h0 = (uint32_t)(lane >> 3);
                const uint64_t ofix = ((uint64_t)(h0 & 1u) << P.tq[4]) | ((uint64_t)(h0 >> 1) << P.tq[5]);
                uint64_t M = 0;
#pragma unroll
                for (int q = 6; q < T; ++q) M |= 1ull << P.tq[q];
                uint64_t x = 0;
                const float2* src = st + ofix + 2 * p;
#pragma unroll 4
                for (uint32_t k = 0; k < 128; ++k) {
                    const uint32_t h = 4u * k + h0;
                    const uint32_t L = 16u * h;
                    const uint32_t slot = (L ^ ((((L >> 4) ^ (L >> 7) ^ (L >> 10)) & 7u) << 1)) ^ (2u * (uint32_t)p);
                    cp_async16_s(buf + 8u * slot, src + x);
                    x = (x - M) & M;
                }
                cp_async_arrive_noinc(full_bar(b));
            }
            ++j;
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
    } else {
        // ---------------- compute warpgroups ----------------
        const int wg = warp >> 2;
        const int wtid = tid & (NT - 1);
        const uint32_t tbase = tmem + 256u * (uint32_t)wg;
        const uint32_t lane_off = ((uint32_t)(warp & 3) * 32u) << 16;
        const uint32_t tl = tbase + lane_off;  // this thread's TMEM lane, column 0 of the warpgroup
        double* red = reinterpret_cast<double*>(sm + kRedOff) + 64 * wg;
        const uint32_t wbuf = sm_s + kWOff + (uint32_t)wg * 2u * kV2GateBytes;
        const bool elect = wtid == 0;
        uint32_t mma_phase = 0;
        uint32_t w_issued = 0, w_used = 0;  // bulk W loads issued / consumed (buffer = index & 1)
        int j = 0;
        for (uint32_t i = blockIdx.x; i < nitems; i += gridDim.x) {
            const Item it = item_of(A, step, i, tshift);
            if (!it.p) continue;
            const int b = j++ % NBUF;
            if (((j - 1) & 1) != wg) continue;
            const PassDesc P = *it.p;
            const int slot = it.slot;
            const uint64_t base = tile_base(P, it.tile);
            float2* st = A.state + ((uint64_t)slot << n);
            float2* tile = reinterpret_cast<float2*>(sm + (size_t)b * kTileBytes);
            char* const tb8 = reinterpret_cast<char*>(tile);
            const GateDesc* gates = A.gates + P.gate_begin;
            const int ng = P.gate_count;
            // W of the first tensor-core gate travels with the tile
            int w_next = 0;  // next gate whose W has not been issued
            while (w_next < ng && !(gates[w_next].k & kGateTC)) ++w_next;
            if (elect && w_next < ng) {
                bulk_w(wbuf + (w_issued & 1u) * kV2GateBytes, A.pool + gates[w_next].mat_off,
                       wfull_bar(wg, (int)(w_issued & 1u)));
                ++w_issued;
                ++w_next;
            }
            mbar_wait_s(full_bar(b), (uint32_t)((j - 1) / NBUF & 1));
            float run_scale = 1.f, run_inv = 1.f;
            for (int g = 0; g < ng;) {
                GateDesc G = gates[g];
                if (!(G.k & kGateTC)) {
                    // device-chosen conventional operator (k <= 3) on FP32 CUDA cores, 64 amplitudes per thread
                    uint32_t unit[6];
#pragma unroll
                    for (int m = 0; m < 6; ++m) unit[m] = swz(1u << ((G.rpos >> (4 * m)) & 15u)) << 3;
                    uint32_t tb = 0;
#pragma unroll
                    for (int q = 0; q < 7; ++q) tb |= ((uint32_t)(wtid >> q) & 1u) << ((G.tpos >> (4 * q)) & 15u);
                    const float2* M = A.pool + G.mat_off;
                    const int k = G.k & 0xff;
                    if (k == 1) apply_fused<1, 6>(tile, M, swz(tb) << 3, unit);
                    else if (k == 2) apply_fused<2, 6>(tile, M, swz(tb) << 3, unit);
                    else apply_fused<3, 6>(tile, M, swz(tb) << 3, unit);
                    bar_wg(wg);
                    ++g;
                    continue;
                }
                // ---- segment start: gather the fp32 tile into A (TMEM), new tile scale ----
                {
                    uint32_t ucfg[4], ugrp[2], tb = 0;
#pragma unroll
                    for (int m = 0; m < 4; ++m) ucfg[m] = swz(1u << ((G.rpos >> (4 * m)) & 15u)) << 3;
#pragma unroll
                    for (int a = 0; a < 2; ++a) ugrp[a] = swz(1u << ((G.rpos >> (16 + 4 * a)) & 15u)) << 3;
#pragma unroll
                    for (int q = 0; q < 7; ++q) tb |= ((uint32_t)(wtid >> q) & 1u) << ((G.tpos >> (4 * q)) & 15u);
                    const uint32_t rbase = swz(tb) << 3;
                    float2 v[64];
                    float amax = 0.f;
#pragma unroll
                    for (int jg = 0; jg < 4; ++jg)
#pragma unroll
                        for (int c = 0; c < 16; ++c) {
                            uint32_t o = rbase;
                            if (jg & 1) o ^= ugrp[0];
                            if (jg & 2) o ^= ugrp[1];
#pragma unroll
                            for (int m = 0; m < 4; ++m)
                                if ((c >> m) & 1) o ^= ucfg[m];
                            v[16 * jg + c] = *reinterpret_cast<const float2*>(tb8 + o);
                            amax = fmaxf(amax, fmaxf(fabsf(v[16 * jg + c].x), fabsf(v[16 * jg + c].y)));
                        }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
                    float* redf = reinterpret_cast<float*>(red);
                    if (lane == 0) redf[warp & 3] = amax;
                    bar_wg(wg);
                    amax = fmaxf(fmaxf(redf[0], redf[1]), fmaxf(redf[2], redf[3]));
                    const int shift = (G.k >> kGateShiftBit) & 0xff;
                    int se = 260 - (int)((__float_as_uint(amax) >> 23) & 0xffu) - shift;  // amax 2^(se-127) in [2^6, 2^7)
                    se = min(max(se, 1), 253);
                    run_scale = __uint_as_float((uint32_t)se << 23);
                    run_inv = __uint_as_float((uint32_t)(254 - se) << 23);
#pragma unroll
                    for (int jg = 0; jg < 4; ++jg) {
                        uint32_t a[32];
#pragma unroll
                        for (int c = 0; c < 16; ++c)
                            split(v[16 * jg + c].x * run_scale, v[16 * jg + c].y * run_scale, a[c], a[16 + c]);
                        tc::tmem_st32(tl + 64u * (uint32_t)jg + 32u, a);
                    }
                    tc::tmem_wait_st();
                    tc::fence_before();
                    bar_wg(wg);  // A complete; every fp32 read of this buffer done
                }
                // ---- the segment's gates ----
                for (;;) {
                    if (elect) {
                        // W(g) (issued earlier, in order), then the MMAs of all four groups
                        const uint32_t wi = w_used & 1u;
                        mbar_wait_s(wfull_bar(wg, (int)wi), (w_used >> 1) & 1u);
                        ++w_used;
                        tc::fence_after();
                        const uint32_t wb = wbuf + wi * kV2GateBytes;
                        const uint64_t b0 = tc::smem_desc_sw128(wb), b1 = tc::smem_desc_sw128(wb + 32);
                        const uint64_t b2 = tc::smem_desc_sw128(wb + 64), b3 = tc::smem_desc_sw128(wb + 96);
#pragma unroll
                        for (int jg = 0; jg < 4; ++jg) {
                            const uint32_t d = tbase + 64u * (uint32_t)jg, ah = d + 32u, al = d + 48u;
                            mma_ts(d, ah, b0, 0u);
                            mma_ts(d, ah + 8u, b1, 1u);
                            mma_ts(d, al, b0, 1u);
                            mma_ts(d, al + 8u, b1, 1u);
                            mma_ts(d, ah, b2, 1u);
                            mma_ts(d, ah + 8u, b3, 1u);
                        }
                        tc::mma_commit(reinterpret_cast<uint64_t*>(sm + kMbarOff + 8 * (6 + wg)));
                        // prefetch the next tensor-core gate's W into the other buffer (its
                        // previous user, gate g - 1, has completed)
                        while (w_next < ng && !(gates[w_next].k & kGateTC)) ++w_next;
                        if (w_next < ng && w_issued == w_used) {
                            bulk_w(wbuf + (w_issued & 1u) * kV2GateBytes, A.pool + gates[w_next].mat_off,
                                   wfull_bar(wg, (int)(w_issued & 1u)));
                            ++w_issued;
                            ++w_next;
                        }
                    }
                    __syncwarp();
                    mbar_wait_s(mma_bar(wg), mma_phase);
                    mma_phase ^= 1u;
                    tc::fence_after();
                    if (G.k & kGateRunEnd) {
                        // ---- segment end: D -> fp32 tile ----
                        uint32_t ucfg[4], ugrp[2], tb = 0;
#pragma unroll
                        for (int m = 0; m < 4; ++m) ucfg[m] = swz(1u << ((G.rpos >> (4 * m)) & 15u)) << 3;
#pragma unroll
                        for (int a = 0; a < 2; ++a) ugrp[a] = swz(1u << ((G.rpos >> (16 + 4 * a)) & 15u)) << 3;
#pragma unroll
                        for (int q = 0; q < 7; ++q) tb |= ((uint32_t)(wtid >> q) & 1u) << ((G.tpos >> (4 * q)) & 15u);
                        const uint32_t rbase = swz(tb) << 3;
#pragma unroll
                        for (int jg = 0; jg < 4; ++jg) {
                            uint32_t d[32];
                            tc::tmem_ld32(tl + 64u * (uint32_t)jg, d);
                            tc::tmem_wait_ld();
                            uint32_t o0 = rbase;
                            if (jg & 1) o0 ^= ugrp[0];
                            if (jg & 2) o0 ^= ugrp[1];
#pragma unroll
                            for (int c = 0; c < 16; ++c) {
                                uint32_t o = o0;
#pragma unroll
                                for (int m = 0; m < 4; ++m)
                                    if ((c >> m) & 1) o ^= ucfg[m];
                                *reinterpret_cast<float2*>(tb8 + o) =
                                    make_float2(__uint_as_float(d[2 * c]) * run_inv, __uint_as_float(d[2 * c + 1]) * run_inv);
                            }
                        }
                        tc::fence_before();
                        bar_wg(wg);
                        ++g;
                        break;
                    }
                    // ---- in-TMEM transition to gate g + 1: its A from this gate's D ----
                    {
                        const uint4 x0 = *reinterpret_cast<const uint4*>(&gates[g].xu[0]);
                        const uint32_t xu[6] = {x0.x & 0xffffu, x0.x >> 16, x0.y & 0xffffu,
                                                x0.y >> 16,     x0.z & 0xffffu, x0.z >> 16};
#pragma unroll 1
                        for (int jg = 0; jg < 4; ++jg) {
                            uint32_t cj = tl;
                            if (jg & 1) cj += xu[4];
                            if (jg & 2) cj += xu[5];
                            uint32_t d[32];
#pragma unroll
                            for (int c = 0; c < 16; ++c) {
                                uint32_t col = cj;
#pragma unroll
                                for (int m = 0; m < 4; ++m)
                                    if ((c >> m) & 1) col += xu[m];
                                tmem_ld2(col, d[2 * c], d[2 * c + 1]);
                            }
                            tc::tmem_wait_ld();
                            uint32_t a[32];
#pragma unroll
                            for (int c = 0; c < 16; ++c)
                                split(__uint_as_float(d[2 * c]), __uint_as_float(d[2 * c + 1]), a[c], a[16 + c]);
                            tc::tmem_st32(tl + 64u * (uint32_t)jg + 32u, a);
                        }
                        tc::tmem_wait_st();
                        tc::fence_before();
                        bar_wg(wg);
                    }
                    ++g;
                    G = gates[g];
                }
            }
            // ---------------- epilogues (read-only on the fp32 tile) ----------------
            const uint64_t tile_row = (uint64_t)slot * ntiles + it.tile;
            if (P.flags & kPassRho) {
                const EventDesc E = A.events[P.event];
                const ChanDesc C = A.chans[E.chan];
                const uint32_t ql = to_local<T>(C.qmask, P);
                double* out = A.rho_part + tile_row * A.rho_stride;
                if (C.nq == 1) rho_partial<1>(tile, ql, out, red, wg);
                else if (C.nq == 2) rho_partial<2>(tile, ql, out, red, wg);
                else rho_partial_rows3(tile, ql, out, red, wg);
                __threadfence();
                bar_wg(wg);
                if (wtid == 0) misc[1 + wg] = (atomicAdd(&A.counters[slot], 1) == (int)ntiles - 1);
                bar_wg(wg);
                if (misc[1 + wg]) {
                    // last tile of the slot: sum the tile partials in a fixed order, then choose
                    __threadfence();
                    const int ne = 2 * C.d * C.d;
                    double fin[128];  // ne <= 128 (q <= 3)
                    const double* part = A.rho_part + (uint64_t)slot * ntiles * A.rho_stride;
                    for (int e0 = 0; e0 < ne; e0 += 8) {
                        double acc[8];
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) acc[jj] = 0.0;
                        for (uint32_t t = wtid; t < ntiles; t += NT)
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj)
                                if (e0 + jj < ne) acc[jj] += __ldcg(part + (uint64_t)t * A.rho_stride + e0 + jj);
                        wg_sum_n<8>(acc, red, wg);
                        if (wtid == 0)
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj)
                                if (e0 + jj < ne) fin[e0 + jj] = acc[jj];
                    }
                    if (wtid == 0) {
                        choose_conventional(E, C, A.chan_data, fin, A.pool, A.records, A.status + slot);
                        A.counters[slot] = 0;
                    }
                }
            }
            if (P.flags & kPassFinal) {
                double s[1] = {0.0};
#pragma unroll 8
                for (int m = 0; m < NA; ++m) {
                    const float2 v = tile[swz((uint32_t)(wtid + m * NT))];
                    s[0] += (double)v.x * v.x + (double)v.y * v.y;
                }
                wg_sum_n<1>(s, red, wg);
                if (wtid == 0) A.blocksum[tile_row] = s[0];
            }
            if (P.flags & kPassObs) {
                // Z strings: Walsh-Hadamard transform of |psi(wtid + m NT)|^2 over m
                float w[NA];
#pragma unroll
                for (int m = 0; m < NA; ++m) {
                    const float2 v = tile[swz((uint32_t)(wtid + m * NT))];
                    w[m] = fmaf(v.x, v.x, v.y * v.y);
                }
#pragma unroll
                for (int h = 1; h < NA; h <<= 1)
#pragma unroll
                    for (int m = 0; m < NA; ++m)
                        if (!(m & h)) {
                            const float a = w[m], c = w[m | h];
                            w[m] = a + c;
                            w[m | h] = a - c;
                        }
                for (int o = 0; o < P.obs_count; ++o) {
                    const ObsDesc O = A.obs[P.obs_begin + o];
                    const uint32_t zl = to_local<T>(O.zmask, P);
                    const int zs = __popcll(base & O.zmask) & 1;
                    double part[1];
                    if (O.xmask == 0) {
                        const float vv = pick_uniform<NA>(w, (int)(zl >> 7));
                        const int par = (__popc((uint32_t)wtid & zl & (uint32_t)(NT - 1)) + zs) & 1;
                        part[0] = par ? -(double)vv : (double)vv;
                    } else {
                        const uint64_t xo = O.xmask & ~P.tile_mask;
                        const uint32_t xl = to_local<T>(O.xmask, P);
                        part[0] = 0.0;
#pragma unroll 1
                        for (int m = 0; m < NA; ++m) {
                            const uint32_t L = (uint32_t)(wtid + m * NT);
                            const float2 v = tile[swz(L)];
                            float2 wv;
                            if (xo == 0) {
                                wv = tile[swz(L ^ xl)];
                            } else {  // partner amplitude in another tile (read-only pass only)
                                wv = st[(base + pdep64(L, P.tile_mask)) ^ O.xmask];
                            }
                            const double cr = (double)wv.x * v.x + (double)wv.y * v.y;
                            const double ci = (double)wv.x * v.y - (double)wv.y * v.x;
                            double t;
                            switch (O.ny & 3) {
                                case 0: t = cr; break;
                                case 1: t = -ci; break;
                                case 2: t = -cr; break;
                                default: t = ci; break;
                            }
                            const int par = (__popc(L & zl) + zs) & 1;
                            part[0] += par ? -t : t;
                        }
                    }
                    wg_sum_n<1>(part, red, wg);
                    if (wtid == 0) A.obs_part[tile_row * A.n_obs + O.slot] = part[0];
                }
            }
            // ---------------- shared -> HBM: 16-byte stores of amplitude pairs ----------------
            if (P.flags & kPassStore) {
                // thread: pair p = wtid & 7 of run h = (wtid >> 3) + 16 m
                const int p = wtid & 7;
                const uint32_t hl = (uint32_t)(wtid >> 3);
                uint64_t ofix = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) ofix |= (uint64_t)((hl >> q) & 1u) << P.tq[4 + q];
                uint64_t M = 0;
#pragma unroll
                for (int q = 8; q < T; ++q) M |= 1ull << P.tq[q];
                float4* dst = reinterpret_cast<float4*>(st + base + ofix + 2 * p);
                uint64_t x = 0;
#pragma unroll 4
                for (uint32_t m = 0; m < 32; ++m) {
                    const uint32_t L = 16u * (hl + 16u * m);
                    const uint32_t s2 = (L ^ ((((L >> 4) ^ (L >> 7) ^ (L >> 10)) & 7u) << 1)) ^ (2u * (uint32_t)p);
                    const float4 v = *reinterpret_cast<const float4*>(tb8 + 8u * s2);
                    *reinterpret_cast<float4*>(reinterpret_cast<float2*>(dst) + x) = v;
                    x = (x - M) & M;
                }
            }
            bar_wg(wg);  // every read of the buffer done
            if (elect) mbar_arrive_s(empty_bar(b));
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

}  // namespace v2

size_t tile_pass_v2_smem_bytes() { return v2::kSmemBytes; }

cudaError_t launch_tile_pass_v2(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    static bool configured = false;
    static int sms = 0;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(v2::tile_pass_v2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)v2::kSmemBytes);
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        configured = true;
    }
    int tshift = 0;
    while ((1u << tshift) < ntiles) ++tshift;
    const uint32_t nitems = ntiles * (uint32_t)nslots;
    if (nitems == 0) return cudaSuccess;
    const uint32_t grid = nitems < (uint32_t)sms ? nitems : (uint32_t)sms;
    v2::tile_pass_v2_kernel<<<grid, v2::kThreads, v2::kSmemBytes, s>>>(a, step, nitems, tshift);
    return cudaGetLastError();
}

}  // namespace qt
