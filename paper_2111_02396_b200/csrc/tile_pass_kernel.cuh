// tile_pass_kernel.cuh -- K1 tile-pass kernel (Alg. 1, applied to a whole
// program of fused gates per HBM sweep) with the K2 / K3a / K4 epilogues.
//
//   TC = false: fused gates on FP32 CUDA cores, 2^R amplitudes per thread in
//               registers, one swizzled shared-memory re-layout per gate.
//   TC = true : T = 12, 128 threads.  Fused gates are padded to 4 qubits and
//               applied as the real GEMM of tc_common.cuh on tcgen05 tensor
//               cores: kind::f16 with hi/lo splits, A and B in shared memory,
//               D in TMEM.  A run of consecutive tensor-core gates keeps the
//               tile in the f16 operand layout: each gate's epilogue reads D
//               from TMEM and writes it straight into the next gate's operand
//               layout (one barrier and one MMA round trip per gate, no
//               gather; outputs c, c ^ 1 go out as one 16-byte store when the
//               planner has relabelled the gate's matrix bits, GateDesc::pair).
//               Gates flagged non-TC (the device-chosen operators of
//               conventional channels, k <= 3) use the CUDA-core path with
//               R = 5 on the fp32 tile.  Single 4-qubit gates: 3xTF32 with A in
//               TMEM.  TCK = 5 / 6 (f = 5 / 6 plans): f16 hi/lo GEMMs, one wide
//               gate at a time (apply_tc_wide).
#pragma once
#include <cuda_fp16.h>

#include "tile_pass.cuh"

#ifndef QT_TC4_MINB
#define QT_TC4_MINB 4  // CTAs per SM of the 4-qubit tensor-core K1 (launch bounds)
#endif

namespace qt {

namespace detail {

// Packed fp32 pair arithmetic (sm_100 FADD2 / FMUL2).
__device__ __forceinline__ uint64_t pk2(float x, float y) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ float2 upk2(uint64_t r) {
    float2 o;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
    return o;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// f16 hi / lo split of a (scaled) complex amplitude x (packed pair): hi = x with
// the 13 low mantissa bits cleared (exact in f16 above 2^-14; below, the f16
// rounding error is < 2^-25 absolute against a tile maximum >= 2^6), lo = the
// exact fp32 remainder rounded to f16.  Returns {hi pair, lo pair}.
__device__ __forceinline__ uint2 split_f16(uint64_t x) {
    const float2 xf = upk2(x);
    const float hr = __uint_as_float(__float_as_uint(xf.x) & 0xFFFFE000u);
    const float hi = __uint_as_float(__float_as_uint(xf.y) & 0xFFFFE000u);
    const float2 l = upk2(sub2(x, pk2(hr, hi)));
    const __half2 h2 = __floats2half2_rn(hr, hi);
    const __half2 l2 = __floats2half2_rn(l.x, l.y);
    return make_uint2(*reinterpret_cast<const uint32_t*>(&h2), *reinterpret_cast<const uint32_t*>(&l2));
}

// Byte offset, in the f16 operand layout of a gate, of subvector row s (thread
// bits), group g and configuration c (tc_common.cuh: 8 bytes per amplitude).
__device__ __forceinline__ uint32_t a_offset(uint32_t s, uint32_t g, uint32_t c) {
    return g * (uint32_t)tc::kF16GroupBytes + (s >> 3) * 1024u + (s & 7u) * 128u + ((((c >> 1) ^ s) & 7u) << 4) +
           ((c & 1u) << 3);
}

// fp32 tile layout of a gate (register bit m <-> tile bit rpos[m], thread bit
// i <-> tile bit tpos[i]): byte offsets of the 16 configurations, of the
// group bit, and of this thread's base.
template <int T>
__device__ __forceinline__ void fp32_layout(const GateDesc& G, uint32_t (&lo)[16], uint32_t& grp, uint32_t& base) {
    uint32_t unit[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) unit[m] = swz(1u << ((G.rpos >> (4 * m)) & 15u)) << 3;
    grp = swz(1u << ((G.rpos >> 16) & 15u)) << 3;
    lo[0] = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int x = 0; x < (1 << m); ++x) lo[x + (1 << m)] = lo[x] ^ unit[m];
    uint32_t tb = 0;
#pragma unroll
    for (int i = 0; i < T - 5; ++i) tb |= ((threadIdx.x >> i) & 1u) << ((G.tpos >> (4 * i)) & 15u);
    base = swz(tb) << 3;
}

// 3-qubit device-chosen operators (conventional 3-qubit channels) in the tensor-core
// kernel: an out-of-line call (unit passed through local memory).
template <int R>
__device__ __noinline__ void apply_fused3_outlined(float2* tile, const float2* M, uint32_t pbase,
                                                   const uint32_t (&unit)[R]) {
    apply_fused<3, R>(tile, M, pbase, unit);
}

// A run of tensor-core gates (4 qubits, kind::f16; tc_common.cuh), gates g0..g1
// of the pass (returns g1).  Run start: gather the fp32 tile in the first
// gate's layout, pick the power-of-two tile scale (max |component| -> [2^6,
// 2^7) / 2^shift, so any contraction of the tile stays below 2^13.5 < f16 max)
// and write the hi / lo operand rows in place.  The run's group bit is a tile
// bit no gate touches, so the two 128-row groups are independent pipelines:
// while the MMAs of one group run, the threads read the other group's D rows
// (TMEM lane = thread) and write them straight into the next gate's operand
// layout (byte offsets from G.xu); the last gate writes the fp32 tile back.
template <int T>
__device__ __forceinline__ int tc_run_f16(float2* tile, unsigned char* mbuf, uint32_t mbuf_bytes,
                                          const GateDesc* gdesc, int g0, int ng, const float2* pool, uint32_t tmem,
                                          uint64_t* mbar, uint32_t (&ph)[2], double* red,
                                          unsigned long long* timing = nullptr) {
    using namespace tc;
    constexpr int NT = 128;
#ifdef QT_TIMING
    const bool ts = timing && (blockIdx.x % 32u) == 7u && threadIdx.x == 0;
    const int tw = 0;
    long long tm[7];
#define QT_MARK(i) tm[i] = clock64()
#else
#define QT_MARK(i)
#endif
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    char* const tb8 = reinterpret_cast<char*>(tile);
    const uint32_t tile_s = (uint32_t)__cvta_generic_to_shared(tile);
    const uint32_t mbuf_s = (uint32_t)__cvta_generic_to_shared(mbuf);
    int g1 = g0;
    while (g1 + 1 < ng && (gdesc[g1 + 1].k & (kGateF16 | kGateRunStart)) == kGateF16) ++g1;
    float run_inv;
    {
        const GateDesc& G = gdesc[g0];
        uint32_t lo[16], grp, base;
        fp32_layout<T>(G, lo, grp, base);
        float2 v[32];
        float amax = 0.f;
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                v[16 * g + c] = *reinterpret_cast<const float2*>(tb8 + (base ^ (g ? grp : 0u) ^ lo[c]));
                amax = fmaxf(amax, fmaxf(fabsf(v[16 * g + c].x), fabsf(v[16 * g + c].y)));
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        float* redf = reinterpret_cast<float*>(red);
        if (lane == 0) redf[warp] = amax;
        __syncthreads();  // every fp32 read done (in-place rewrite below) + maxima visible
        amax = fmaxf(fmaxf(redf[0], redf[1]), fmaxf(redf[2], redf[3]));
        const int shift = (G.k >> kGateShiftBit) & 0xff;
        int se = 260 - (int)((__float_as_uint(amax) >> 23) & 0xffu) - shift;  // amax * 2^(se - 127) in [2^6, 2^7)
        se = min(max(se, 1), 253);
        const float run_scale = __uint_as_float((uint32_t)se << 23);
        run_inv = __uint_as_float((uint32_t)(254 - se) << 23);
        const uint64_t sc2 = pk2(run_scale, run_scale);
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int c = 0; c < 16; ++c)
                *reinterpret_cast<uint2*>(tb8 + a_offset(tid, (uint32_t)g, (uint32_t)c)) =
                    split_f16(mul2(pk2(v[16 * g + c].x, v[16 * g + c].y), sc2));
        fence_proxy_async();
        __syncthreads();
    }
    // MMAs of gate g, group grp: D[grp] (TMEM columns 64 grp..) = A[grp] W(g)^T
    auto issue = [&](int g, int grp) {
        fence_after();
        constexpr uint32_t idesc = idesc_f16_m128(64);
        const uint32_t w = mbuf_s + (uint32_t)(g & 1) * mbuf_bytes;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
            mma_f16_ss(tmem + 64 * grp, smem_desc_sw128(tile_s + grp * kF16GroupBytes + ks * 32),
                       smem_desc_sw128(w + ks * 32), idesc, ks > 0);
        mma_commit(mbar + grp);
    };
    if (tid == 0) {
        issue(g0, 0);
        issue(g0, 1);
    }
    __syncwarp();
    const uint32_t lane_off = (warp * 32u) << 16;
    // read D[grp] of this thread's row, write the 16 outputs (split or fp32)
    auto readout = [&](int grp, uint32_t b, const uint32_t (&lo)[16], bool chain, uint64_t inv2, bool pair) {
        uint32_t h0[32], h1[32];
        tmem_ld32(tmem + lane_off + 64 * grp, h0);
        tmem_ld32(tmem + lane_off + 64 * grp + 32, h1);
        tmem_wait_ld();
        if (pair) {  // outputs c, c ^ 1 fill one 16-byte chunk (lo[c ^ 1] = lo[c] ^ 8)
#pragma unroll
            for (int c = 0; c < 16; c += 2) {
                const uint2 x0 = split_f16(add2(pk2(__uint_as_float(h0[2 * c]), __uint_as_float(h0[2 * c + 1])),
                                                pk2(__uint_as_float(h1[2 * c]), __uint_as_float(h1[2 * c + 1]))));
                const uint2 x1 =
                    split_f16(add2(pk2(__uint_as_float(h0[2 * c + 2]), __uint_as_float(h0[2 * c + 3])),
                                   pk2(__uint_as_float(h1[2 * c + 2]), __uint_as_float(h1[2 * c + 3]))));
                *reinterpret_cast<uint4*>(tb8 + (b ^ lo[c])) = make_uint4(x0.x, x0.y, x1.x, x1.y);
            }
            return;
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const uint64_t y = add2(pk2(__uint_as_float(h0[2 * c]), __uint_as_float(h0[2 * c + 1])),
                                    pk2(__uint_as_float(h1[2 * c]), __uint_as_float(h1[2 * c + 1])));
            if (chain)
                *reinterpret_cast<uint2*>(tb8 + (b ^ lo[c])) = split_f16(y);
            else
                *reinterpret_cast<float2*>(tb8 + (b ^ lo[c])) = upk2(mul2(y, inv2));
        }
    };
#pragma unroll 1
    for (int g = g0; g < g1; ++g) {
        const GateDesc& G = gdesc[g];
        // next operand layout: byte offsets of this gate's roles (the group bit is
        // the same tile bit in both gates: group grp stays in region grp)
        const uint4 x0 = *reinterpret_cast<const uint4*>(&G.xu[0]);   // xu[0..7]
        const uint2 x1 = *reinterpret_cast<const uint2*>(&G.xu[8]);   // xu[8..11]
        const uint32_t xu[12] = {x0.x & 0xffffu, x0.x >> 16, x0.y & 0xffffu, x0.y >> 16,
                                 x0.z & 0xffffu, x0.z >> 16, x0.w & 0xffffu, x0.w >> 16,
                                 x1.x & 0xffffu, x1.x >> 16, x1.y & 0xffffu, x1.y >> 16};
        uint32_t obase = 0;
#pragma unroll
        for (int i = 0; i < 7; ++i)
            if ((tid >> i) & 1u) obase ^= xu[5 + i];
        uint32_t lo[16];
        lo[0] = 0;
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int x = 0; x < (1 << m); ++x) lo[x + (1 << m)] = lo[x] ^ xu[m];
        if (xu[4] != (uint32_t)kF16GroupBytes) {
            // the next gate uses another group bit: outputs of either group land in
            // both regions, so both MMAs finish before any write (no overlap)
            mbar_wait(mbar, ph[0]);
            ph[0] ^= 1u;
            mbar_wait(mbar + 1, ph[1]);
            ph[1] ^= 1u;
            fence_after();
            readout(0, obase, lo, true, 0, G.pair != 0);
            readout(1, obase ^ xu[4], lo, true, 0, G.pair != 0);
            if (g + 2 < ng) {  // both MMAs of gate g are done: its W buffer takes W(g + 2)
                const char* src = reinterpret_cast<const char*>(pool + gdesc[g + 2].mat_off);
                unsigned char* dst = mbuf + (g & 1) * mbuf_bytes;
                const int chunks = (gdesc[g + 2].k & kGateTC)
                                       ? (kF16GateBytes >> 4)
                                       : ((int)sizeof(float2) << (2 * (gdesc[g + 2].k & 0xff))) >> 4;
                for (int c = (int)tid; c < chunks; c += NT) cp_async16(dst + 16 * c, src + 16 * c);
                cp_async_commit();
                cp_async_wait_group1();  // W(g + 1) landed (W(g + 2) may be in flight)
            } else {
                cp_async_wait_all();
            }
            fence_proxy_async();
            fence_before();
            __syncthreads();
            if (tid == 0) {
                issue(g + 1, 0);
                issue(g + 1, 1);
            }
            __syncwarp();
            continue;
        }
        // group 0: read D0, write the rows, barrier, then the next gate's group-0
        // MMAs (issued by thread 0) overlap the group-1 readout
        QT_MARK(0);
        mbar_wait(mbar, ph[0]);
        ph[0] ^= 1u;
        fence_after();
        QT_MARK(1);
        readout(0, obase, lo, true, 0, G.pair != 0);
        QT_MARK(2);
        cp_async_wait_all();  // W(g + 1)
        fence_proxy_async();
        fence_before();
        __syncthreads();
        if (tid == 0) issue(g + 1, 0);
        __syncwarp();
        QT_MARK(3);
        // group 1 (issued by thread 64)
        mbar_wait(mbar + 1, ph[1]);
        ph[1] ^= 1u;
        fence_after();
        QT_MARK(4);
        readout(1, obase ^ xu[4], lo, true, 0, G.pair != 0);
        QT_MARK(5);
        if (g + 2 < ng) {  // both MMAs of gate g are done: its W buffer takes W(g + 2)
            const char* src = reinterpret_cast<const char*>(pool + gdesc[g + 2].mat_off);
            unsigned char* dst = mbuf + (g & 1) * mbuf_bytes;
            const int chunks = (gdesc[g + 2].k & kGateTC) ? (kF16GateBytes >> 4)
                                                          : ((int)sizeof(float2) << (2 * (gdesc[g + 2].k & 0xff))) >> 4;
            for (int c = (int)tid; c < chunks; c += NT) cp_async16(dst + 16 * c, src + 16 * c);
            cp_async_commit();
        }
        fence_proxy_async();
        fence_before();
        __syncthreads();
        if (tid == 64) issue(g + 1, 1);
        __syncwarp();
        QT_MARK(6);
#ifdef QT_TIMING
        if (ts) {
            for (int i = 0; i < 6; ++i) atomicAdd(timing + tw + i, (unsigned long long)(tm[i + 1] - tm[i]));
            if (threadIdx.x == 0) atomicAdd(timing + 15, 1ull);
        }
#endif
    }
#undef QT_MARK
    {   // last gate of the run: both groups complete, then the fp32 tile
        uint32_t lo[16], ogrp, obase;
        fp32_layout<T>(gdesc[g1], lo, ogrp, obase);
        mbar_wait(mbar, ph[0]);
        ph[0] ^= 1u;
        mbar_wait(mbar + 1, ph[1]);
        ph[1] ^= 1u;
        fence_after();
        const uint64_t inv2 = pk2(run_inv, run_inv);
#pragma unroll 1
        for (int grp = 0; grp < 2; ++grp) readout(grp, obase ^ (grp ? ogrp : 0u), lo, false, inv2, false);
        fence_before();
    }
    return g1;
}

// Apply one padded 4-qubit gate on tensor cores with 3xTF32 (single-gate runs:
// no operand-layout conversion).  Thread t owns subvectors
// s = t and t + 128 (register bit 4 = the group bit); register j = 16 g + c.
__device__ __forceinline__ void apply_tc_gate(float2* tile, uint32_t w_smem, uint32_t pbase,
                                              const uint32_t (&unit)[5], uint32_t tmem, uint64_t* mbar,
                                              uint32_t& phase) {
    using namespace tc;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    char* const tb8 = reinterpret_cast<char*>(tile);
    uint32_t lo[16];
    lo[0] = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int x = 0; x < (1 << m); ++x) lo[x + (1 << m)] = lo[x] ^ unit[m];
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    // TMEM columns: D0 [0,32), D1 [32,64), A hi [64,96), A lo [96,128).
    // hi = x with the 13 low mantissa bits cleared (exact tf32), lo = x - hi (exact
    // in fp32; the MMA reads its top tf32 bits).
    auto gather = [&](int g, uint32_t (&hi)[32], uint32_t (&lw)[32]) {
        const uint32_t b = pbase ^ (g ? unit[4] : 0u);
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const float2 v = *reinterpret_cast<const float2*>(tb8 + (b ^ lo[c]));
            const uint32_t hx = __float_as_uint(v.x) & 0xFFFFE000u, hy = __float_as_uint(v.y) & 0xFFFFE000u;
            hi[2 * c] = hx;
            hi[2 * c + 1] = hy;
            lw[2 * c] = __float_as_uint(v.x - __uint_as_float(hx));
            lw[2 * c + 1] = __float_as_uint(v.y - __uint_as_float(hy));
        }
    };
    auto issue = [&](int g) {  // A (hi, lo) in TMEM -> D_g ; one elected thread
        tmem_wait_st();
        fence_before();
        __syncthreads();
        if (tid == 0) {
            fence_after();
            const uint32_t d = tmem + 32 * g;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t bh = smem_desc_sw128(w_smem + ks * 32);
                const uint64_t bl = smem_desc_sw128(w_smem + kWBytes + ks * 32);
                mma_tf32_ts(d, tmem + 64 + ks * 8, bh, ks > 0);
                mma_tf32_ts(d, tmem + 96 + ks * 8, bh, 1);
                mma_tf32_ts(d, tmem + 64 + ks * 8, bl, 1);
            }
            mma_commit(mbar);
        }
        __syncwarp();
    };
    auto scatter = [&](int g) {
        const uint32_t b = pbase ^ (g ? unit[4] : 0u);
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + 32 * g, v);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c)
            *reinterpret_cast<float2*>(tb8 + (b ^ lo[c])) =
                make_float2(__uint_as_float(v[2 * c]), __uint_as_float(v[2 * c + 1]));
    };
    {
        uint32_t hi[32], lw[32];
        gather(0, hi, lw);
        tmem_st32(tmem + lane_off + 64, hi);
        tmem_st32(tmem + lane_off + 96, lw);
    }
    issue(0);
    {
        uint32_t hi[32], lw[32];
        gather(1, hi, lw);           // overlaps the group-0 MMAs
        mbar_wait(mbar, phase);      // group 0 done: A columns free, D0 ready
        phase ^= 1u;
        fence_after();
        tmem_st32(tmem + lane_off + 64, hi);
        tmem_st32(tmem + lane_off + 96, lw);
    }
    issue(1);
    scatter(0);                      // overlaps the group-1 MMAs
    mbar_wait(mbar, phase);
    phase ^= 1u;
    fence_after();
    scatter(1);
    fence_before();
}

// Apply one padded K-qubit gate (K = 5, 6) on tensor cores with f16 hi / lo
// operands (tc_common.cuh "wide" gates), 128 threads.  Layout (host-computed,
// R = K): register bits 0..K-1 = the gate bits, thread bits = the other 12 - K
// tile bits.  K = 5: thread t owns subvector t (32 configurations) = MMA row t.
// K = 6: thread t owns configurations 32 h .. 32 h + 31 (h = t >> 6, gate bit
// 5) of subvector s = t & 63; MMA rows s / s + 64 hold its hi / lo parts.  The
// tile is converted in place with a power-of-two tile scale (as a f16 run
// start), the MMAs read A = the tile and B = W from shared memory, and the
// epilogue writes the fp32 tile back.  K = 6 exchanges half of each row's
// outputs through wbuf (free once the MMAs are done).
template <int K>
__device__ __forceinline__ void apply_tc_wide(float2* tile, unsigned char* wbuf, const GateDesc& G, uint32_t tmem,
                                              uint64_t* mbar, uint32_t& phase, double* red) {
    using namespace tc;
    static_assert(K == 5 || K == 6, "wide tensor-core gates are 5 or 6 qubits");
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    char* const tb8 = reinterpret_cast<char*>(tile);
    const uint32_t tile_s = (uint32_t)__cvta_generic_to_shared(tile);
    const uint32_t w_s = (uint32_t)__cvta_generic_to_shared(wbuf);
    uint32_t unit[K];
#pragma unroll
    for (int m = 0; m < K; ++m) unit[m] = swz(1u << ((G.rpos >> (4 * m)) & 15u)) << 3;
    uint32_t tb = 0;
#pragma unroll
    for (int i = 0; i < 12 - K; ++i) tb |= ((tid >> i) & 1u) << ((G.tpos >> (4 * i)) & 15u);
    const uint32_t h = K == 6 ? (tid >> 6) : 0u;
    uint32_t base = swz(tb) << 3;
    if constexpr (K == 6) base ^= h ? unit[K - 1] : 0u;
    uint32_t lo[32];
    lo[0] = 0;
#pragma unroll
    for (int m = 0; m < 5; ++m)
#pragma unroll
        for (int x = 0; x < (1 << m); ++x) lo[x + (1 << m)] = lo[x] ^ unit[m];
    float run_inv;
    {
        float2 v[32];
        float amax = 0.f;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            v[c] = *reinterpret_cast<const float2*>(tb8 + (base ^ lo[c]));
            amax = fmaxf(amax, fmaxf(fabsf(v[c].x), fabsf(v[c].y)));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        float* redf = reinterpret_cast<float*>(red);
        if (lane == 0) redf[warp] = amax;
        __syncthreads();  // every fp32 read done (in-place rewrite below) + maxima visible
        amax = fmaxf(fmaxf(redf[0], redf[1]), fmaxf(redf[2], redf[3]));
        const int shift = (G.k >> kGateShiftBit) & 0xff;
        int se = 260 - (int)((__float_as_uint(amax) >> 23) & 0xffu) - shift;  // amax * 2^(se - 127) in [2^6, 2^7)
        se = min(max(se, 1), 253);
        const float run_scale = __uint_as_float((uint32_t)se << 23);
        run_inv = __uint_as_float((uint32_t)(254 - se) << 23);
        const uint64_t sc2 = pk2(run_scale, run_scale);
        // A rows: K = 5: row t, hi in chunk 0, lo in chunk 1 (16 KB); K = 6: rows
        // s (hi) and s + 64 (lo) of chunk h.  Four configurations per 16-byte store.
        const uint32_t row = K == 5 ? tid : (tid & 63u);
        const uint32_t hi_base = K == 5 ? 0u : h * (uint32_t)kF16GroupBytes;
        const uint32_t lo_base = K == 5 ? (uint32_t)kF16GroupBytes : h * (uint32_t)kF16GroupBytes;
        const uint32_t lo_row = K == 5 ? row : row + 64u;
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint2 sp = split_f16(mul2(pk2(v[4 * c4 + j].x, v[4 * c4 + j].y), sc2));
                hw[j] = sp.x;
                lw[j] = sp.y;
            }
            *reinterpret_cast<uint4*>(tb8 + hi_base + sw128_offset((int)row, 16 * c4)) =
                make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(tb8 + lo_base + sw128_offset((int)lo_row, 16 * c4)) =
                make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
        fence_proxy_async();
        fence_before();
        __syncthreads();
    }
    if (tid == 0) {
        fence_after();
        if constexpr (K == 5) {
            constexpr uint32_t idesc = idesc_f16_m128(64);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t ah = smem_desc_sw128(tile_s + ks * 32);
                const uint64_t al = smem_desc_sw128(tile_s + kF16GroupBytes + ks * 32);
                const uint64_t bh = smem_desc_sw128(w_s + ks * 32);
                const uint64_t bl = smem_desc_sw128(w_s + 8192 + ks * 32);
                mma_f16_ss(tmem, ah, bh, idesc, ks > 0);
                mma_f16_ss(tmem, al, bh, idesc, 1);
                mma_f16_ss(tmem, ah, bl, idesc, 1);
            }
        } else {
            constexpr uint32_t idesc = idesc_f16_m128(256);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const uint32_t off = (uint32_t)((ks & 3) * 32);
                mma_f16_ss(tmem, smem_desc_sw128(tile_s + (ks >> 2) * kF16GroupBytes + off),
                           smem_desc_sw128(w_s + (ks >> 2) * 32768 + off), idesc, ks > 0);
            }
        }
        mma_commit(mbar);
    }
    __syncwarp();
    mbar_wait(mbar, phase);
    phase ^= 1u;
    fence_after();
    const uint32_t lane_off = (warp * 32u) << 16;
    const uint64_t inv2 = pk2(run_inv, run_inv);
    if constexpr (K == 5) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            uint32_t d[32];
            tmem_ld32(tmem + lane_off + 32 * p, d);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 16; ++c)
                *reinterpret_cast<float2*>(tb8 + (base ^ lo[16 * p + c])) =
                    upk2(mul2(pk2(__uint_as_float(d[2 * c]), __uint_as_float(d[2 * c + 1])), inv2));
        }
    } else {
        // row t holds (hi or lo part) x W_hi in columns [0, 128) and x W_lo in
        // [128, 256); output column n = 2 j + b.  Thread t keeps the outputs of its
        // configuration half (columns 64 h ..) and sends the other half to t ^ 64.
        // Rows t >= 64 (warps 2, 3) hold lo parts: their x_lo W_lo columns are the
        // dropped fourth product (as for k <= 5), so those warps read only x_lo W_hi
        // (a quarter less TMEM traffic; tcgen05.ld stays warp-uniform).
        float* xbuf = reinterpret_cast<float*>(wbuf);
        const uint32_t sh = 64u * (h ^ 1u), kh = 64u * h;
        const bool lo_row = h != 0u;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            uint32_t a[32], b[32];
            tmem_ld32(tmem + lane_off + sh + 32 * p, a);
            if (!lo_row) tmem_ld32(tmem + lane_off + 128 + sh + 32 * p, b);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i)
                xbuf[(32 * p + i) * 128 + (tid ^ 64u)] =
                    lo_row ? __uint_as_float(a[i]) : __uint_as_float(a[i]) + __uint_as_float(b[i]);
        }
        __syncthreads();
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            uint32_t a[32], b[32];
            tmem_ld32(tmem + lane_off + kh + 32 * p, a);
            if (!lo_row) tmem_ld32(tmem + lane_off + 128 + kh + 32 * p, b);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const float ar = __uint_as_float(a[2 * c]), ai = __uint_as_float(a[2 * c + 1]);
                const float yr = (lo_row ? ar : ar + __uint_as_float(b[2 * c])) + xbuf[(32 * p + 2 * c) * 128 + tid];
                const float yi =
                    (lo_row ? ai : ai + __uint_as_float(b[2 * c + 1])) + xbuf[(32 * p + 2 * c + 1) * 128 + tid];
                *reinterpret_cast<float2*>(tb8 + (base ^ lo[16 * p + c])) = upk2(mul2(pk2(yr, yi), inv2));
            }
        }
    }
    fence_before();
}

}  // namespace detail

template <int T, int R, bool TC, int TCK = 4>
struct TileCfg {
    static constexpr int NT = 1 << (T - R);
    static constexpr int NA = 1 << R;
    static constexpr int TILE = 1 << T;
    static constexpr int CL = T < detail::kCL ? T : detail::kCL;
    static constexpr int NH = TILE >> CL;
    // shared memory: [W/matrix buffers x2 (x1 for 6-qubit tensor-core gates: 64 KB)]
    // [tile][hoff][red][gdesc][mbar], base 1024-aligned
    static constexpr size_t kMbufBytes = TC ? (size_t)tc::gate_bytes(TCK) : sizeof(float2) * ((size_t)1 << (2 * R));
    static constexpr int kNumMbuf = (TC && TCK == 6) ? 1 : 2;
    static constexpr size_t kTileOff = kNumMbuf * kMbufBytes;
    static constexpr size_t kHoffOff = kTileOff + sizeof(float2) * TILE;
    static constexpr size_t kRedOff = kHoffOff + sizeof(uint64_t) * ((NH + 1) & ~1);
    static constexpr size_t kGdescOff = kRedOff + 64 * sizeof(double);
    static constexpr size_t kMbarOff = kGdescOff + sizeof(GateDesc) * kMaxPassGates;
    static_assert(!TC || TCK != 4 || tc::gate_bytes(4) == tc::kF16GateBytes, "f16 operand size");
    static_assert(!TC || tc::gate_bytes(TCK) == tc_gate_bytes(TCK), "operand size (desc.hpp)");
    static constexpr size_t kBytes = kMbarOff + 16 + 1024;  // 2 mbarriers + alignment slack
};

template <int T, int R, bool TC, int TCK = 4>
__global__ void __launch_bounds__(TileCfg<T, R, TC, TCK>::NT,
                                  TC ? (TCK == 6 ? 2 : (TCK == 5 ? 3 : QT_TC4_MINB)) : ((R <= 4 && T == 12) ? QT_MINB : 1))
tile_pass_kernel(const TileArgs A, const int step) {
    using Cfg = TileCfg<T, R, TC, TCK>;
    // TMEM: TCK = 4: f16 runs use D of both groups (2 x 64 columns), 3xTF32 single
    // gates D0 / D1 / A hi / A lo (4 x 32); TCK = 5: D (64); TCK = 6: D (256)
    constexpr uint32_t kTmemCols = TCK == 6 ? 256 : (TCK == 5 ? 64 : 128);  // CTAs per SM share 512 columns
    constexpr int NT = Cfg::NT;
    constexpr int NA = Cfg::NA;
    constexpr int CL = Cfg::CL;
    constexpr int NH = Cfg::NH;
#ifdef QT_TIMING
    long long kt[6];
    kt[0] = clock64();
#define QT_KMARK(i) kt[i] = clock64()
#else
#define QT_KMARK(i)
#endif
    // this CTA's pass: one load from the per-step array (executor), else via the slot tables
    const PassDesc* Pp;
    if (A.step_passes) {
        Pp = A.step_passes + blockIdx.y;
    } else {
        if (step >= A.pass_count[blockIdx.y]) return;
        Pp = A.passes + A.pass_start[blockIdx.y] + step;
    }
    const PassDesc P = *Pp;
    const int slot = A.step_passes ? P.slot : (int)blockIdx.y;

    extern __shared__ unsigned char smem_raw[];
    // 1024-byte alignment by offsetting smem_raw itself (keeps the pointer in the
    // shared address space: LDS/STS instead of generic LD/ST)
    const uint32_t smem_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    unsigned char* sm = smem_raw + (((smem_base + 1023u) & ~1023u) - smem_base);
    unsigned char* mbuf = sm;  // kNumMbuf x kMbufBytes
    float2* tile = reinterpret_cast<float2*>(sm + Cfg::kTileOff);
    uint64_t* hoff = reinterpret_cast<uint64_t*>(sm + Cfg::kHoffOff);
    double* red = reinterpret_cast<double*>(sm + Cfg::kRedOff);
    GateDesc* gdesc = reinterpret_cast<GateDesc*>(sm + Cfg::kGdescOff);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + Cfg::kMbarOff);
    __shared__ int s_last;
    __shared__ uint32_t s_tmem;

    const int tid = threadIdx.x;
    const int n = A.n;
    const uint64_t nmask = (n >= 64) ? ~0ull : ((1ull << n) - 1ull);
    // tile base index = blockIdx.x with a zero inserted at every tile-qubit
    // position (ascending), i.e. pdep(blockIdx.x, ~tile_mask) in T steps
    uint64_t base = blockIdx.x;
#pragma unroll
    for (int i = 0; i < T; ++i) {
        const uint64_t low = base & ((1ull << P.tq[i]) - 1ull);
        base = low | ((base ^ low) << 1);
    }
    (void)nmask;
    float2* st = A.state + ((uint64_t)slot << n);
    const int ng = P.gate_count;

    uint32_t tmem = 0;
    // mbarrier phases: [0] D group 0 (tf32 gates, f16 group 0), [1] D group 1
    uint32_t ph[2] = {0u, 0u};
    if constexpr (TC) {
        if (ng > 0 && (tid >> 5) == 0) tc::tmem_alloc(&s_tmem, kTmemCols);  // CTAs / SM share 512 columns
        if (tid == 0) {
            tc::mbar_init(mbar, 1);        // D of group 0 ready (tcgen05.commit)
            tc::mbar_init(mbar + 1, 1);    // D of group 1 ready
            tc::fence_mbar_init();
        }
    }

    // stage the pass's gate descriptors (async) and the tile-offset table
    constexpr int kGdChunks = (int)(sizeof(GateDesc) / 16);
    for (int c = tid; c < ng * kGdChunks; c += NT)
        cp_async16(reinterpret_cast<uint4*>(gdesc) + c, reinterpret_cast<const uint4*>(A.gates + P.gate_begin) + c);
    cp_async_commit();
    for (int h = tid; h < NH; h += NT) {
        uint64_t o = 0;
#pragma unroll
        for (int i = CL; i < T; ++i) o |= (uint64_t)((h >> (i - CL)) & 1) << P.tq[i];
        hoff[h] = o;
    }
    if constexpr (TC) tc::fence_before();
    __syncthreads();
    if constexpr (TC) {
        tc::fence_after();
        tmem = s_tmem;
    }
    QT_KMARK(1);
    // HBM -> shared: 8-byte asynchronous copies (the swizzle keeps amplitude pairs
    // adjacent but not 16-byte aligned; register-staged 16-byte loads measured 61%
    // of HBM peak vs 68% for async copies at n = 30).  hoff and swz are linear in
    // the index bits: slot L = tid + m NT has global offset hoff[tid >> CL] +
    // hoff[m NT >> CL] + (tid & (2^CL - 1)) (NT >= 2^CL).
    if (P.flags & kPassInit) {
        // first pass of a trajectory: the tile of |0...0> (amplitude 0 = 1 lives in
        // tile 0 at slot swz(0) = 0), no HBM load
        float4* t4 = reinterpret_cast<float4*>(tile);
        for (int i = tid; i < (1 << T) / 2; i += NT) t4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (tid == 0 && blockIdx.x == 0) t4[0] = make_float4(1.f, 0.f, 0.f, 0.f);
    } else if constexpr (NT >= (1 << CL)) {
        const float2* gsrc = st + base + hoff[tid >> CL] + ((uint32_t)tid & ((1u << CL) - 1u));
        const uint32_t sb = swz((uint32_t)tid);
#pragma unroll 8
        for (int m = 0; m < NA; ++m)
            cp_async8(tile + (sb ^ swz((uint32_t)(m * NT))), gsrc + hoff[(m * NT) >> CL]);
    } else {
#pragma unroll
        for (int m = 0; m < NA; ++m) {
            const uint32_t L = (uint32_t)(tid + m * NT);
            const uint64_t g = base + hoff[L >> CL] + (L & ((1u << CL) - 1u));
            cp_async8(tile + swz(L), st + g);
        }
    }
    cp_async_commit();
    auto mat_bytes = [](const GateDesc& G) -> int {
        return (TC && (G.k & kGateTC)) ? tc::gate_bytes(TCK) : (int)sizeof(float2) * (1 << (2 * (G.k & 0xff)));
    };
    if (ng > 0) {  // the first gate's matrix travels with the tile (descriptor read from global)
        const GateDesc& G0 = A.gates[P.gate_begin];
        const char* src = reinterpret_cast<const char*>(A.pool + G0.mat_off);
        const int chunks = mat_bytes(G0) >> 4;
        for (int c = tid; c < chunks; c += NT) cp_async16(mbuf + 16 * c, src + 16 * c);
        cp_async_commit();
    }
    cp_async_wait_all();  // gate descriptors + tile + W(0)
    __syncthreads();
    QT_KMARK(2);
    // gate matrices: double-buffered, cooperative cp.async (measured faster than
    // one-thread bulk copies completing on an mbarrier)
    auto load_w = [&](int g) {
        unsigned char* dst = mbuf + (Cfg::kNumMbuf == 2 ? (g & 1) * Cfg::kMbufBytes : 0);
        const char* src = reinterpret_cast<const char*>(A.pool + gdesc[g].mat_off);
        const int chunks = mat_bytes(gdesc[g]) >> 4;
        for (int c = tid; c < chunks; c += NT) cp_async16(dst + 16 * c, src + 16 * c);
        cp_async_commit();
    };
    for (int gi = 0; gi < ng; ++gi) {
        const GateDesc& G = gdesc[gi];
        cp_async_wait_all();
        if constexpr (TC) tc::fence_proxy_async();  // cp.async W / st.shared rows -> tensor-core reads
        __syncthreads();  // tile writes of the previous gate visible; W buffer (gi + 1) & 1 free
        if constexpr (Cfg::kNumMbuf == 1) {  // one W buffer: gate gi's matrix is loaded now
            if (gi > 0) {
                load_w(gi);
                cp_async_wait_all();
                tc::fence_proxy_async();
                __syncthreads();
            }
        } else if (gi + 1 < ng) {
            load_w(gi + 1);
        }
        unsigned char* mcur = mbuf + (Cfg::kNumMbuf == 2 ? (gi & 1) * Cfg::kMbufBytes : 0);
        if constexpr (TC && TCK == 4) {
            if (G.k & kGateF16) {  // run start (runs end before any non-f16 gate)
                gi = tc_run_f16<T>(tile, mbuf, (uint32_t)Cfg::kMbufBytes, gdesc, gi, ng, A.pool, tmem, mbar, ph, red,
                                   A.timing);
                continue;
            }
        }
        // register layout (host-computed): register bit m <-> tile bit rpos[m]
        // (bits 0..k-1 = the gate qubits), thread bit i <-> tile bit tpos[i]
        uint32_t unit[R];
#pragma unroll
        for (int m = 0; m < R; ++m) unit[m] = swz(1u << ((G.rpos >> (4 * m)) & 15u)) << 3;
        uint32_t tb = 0;
#pragma unroll
        for (int i = 0; i < T - R; ++i) tb |= (((uint32_t)tid >> i) & 1u) << ((G.tpos >> (4 * i)) & 15u);
        if constexpr (TC) {
            if (G.k & kGateTC) {
                if constexpr (R == 5 && TCK == 4)
                    apply_tc_gate(tile, (uint32_t)__cvta_generic_to_shared(mcur), swz(tb) << 3, unit, tmem, mbar,
                                  ph[0]);
                else if constexpr (R == 5 && (TCK == 5 || TCK == 6))
                    apply_tc_wide<TCK>(tile, mcur, G, tmem, mbar, ph[0], red);
            } else if ((G.k & 0xff) == 1) {  // device-chosen conventional operators (q <= 3)
                apply_fused<1, R>(tile, reinterpret_cast<const float2*>(mcur), swz(tb) << 3, unit);
            } else if ((G.k & 0xff) == 2) {
                apply_fused<2, R>(tile, reinterpret_cast<const float2*>(mcur), swz(tb) << 3, unit);
            } else {  // rare: kept out of line so the tensor-core kernel's hot code is unchanged
                apply_fused3_outlined<R>(tile, reinterpret_cast<const float2*>(mcur), swz(tb) << 3, unit);
            }
            continue;
        }
        dispatch_fused<R>(G.k & 0xff, tile, reinterpret_cast<const float2*>(mcur), swz(tb) << 3, unit);
    }
    cp_async_wait_all();  // a pass without gates still has its tile in flight
    __syncthreads();
    QT_KMARK(3);

    // ---- epilogues (read-only on the tile) ----
    const uint32_t ntiles = gridDim.x;
    const uint64_t tile_row = (uint64_t)slot * ntiles + blockIdx.x;
    if (P.flags & kPassRho) {
        const EventDesc E = A.events[P.event];
        const ChanDesc C = A.chans[E.chan];
        const uint32_t ql = to_local<T>(C.qmask, P);  // channel qubits as tile-local bits
        double* out = A.rho_part + tile_row * A.rho_stride;
        if (C.nq >= 4) {
            rho_partial_big<T, NT>(tile, ql, C.nq, out, [](uint32_t L) { return swz(L); });
        } else if constexpr (T >= 3) {
            if (C.nq == 1) rho_partial<1, T, NT>(tile, ql, out, red);
            else if (C.nq == 2) rho_partial<2, T, NT>(tile, ql, out, red);
            else rho_partial_rows<3, T, NT>(tile, ql, out, red);
        } else if constexpr (T >= 2) {
            if (C.nq == 1) rho_partial<1, T, NT>(tile, ql, out, red);
            else rho_partial<2, T, NT>(tile, ql, out, red);
        } else {
            rho_partial<1, T, NT>(tile, ql, out, red);
        }
        // writers ordered before thread 0 by the barrier; its device-scope fence releases them
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            s_last = (atomicAdd(&A.counters[slot], 1) == (int)ntiles - 1);
        }
        __syncthreads();
        if (s_last) {
            // last CTA of the slot: sum the tile partials with every thread (tiles
            // strided over threads, then a fixed-order block sum), 8 entries at a time
            __threadfence();
            const int ne = 2 * C.d * C.d;
            double* fin = reinterpret_cast<double*>(gdesc);  // ne <= 128 doubles (gate descriptors are done)
            const double* part = A.rho_part + (uint64_t)slot * ntiles * A.rho_stride;
            if (C.nq >= 4) {  // 4..6 qubits: entry-parallel sums in global memory
                const double* rf = rho_final_big<NT>(A.rho_part + (uint64_t)slot * ntiles * A.rho_stride, ntiles,
                                                     A.rho_stride, ne);
                __syncthreads();
                if (tid == 0) {
                    choose_conventional(E, C, A.chan_data, rf, A.pool, A.records, A.status + slot);
                    A.counters[slot] = 0;
                }
            } else
            for (int e0 = 0; e0 < ne; e0 += 8) {
                double acc[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = 0.0;
                for (uint32_t t = tid; t < ntiles; t += NT)
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (e0 + j < ne) acc[j] += __ldcg(part + (uint64_t)t * A.rho_stride + e0 + j);
                block_sum_n<NT, 8>(acc, red);
                if (tid == 0)
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (e0 + j < ne) fin[e0 + j] = acc[j];
            }
            if (C.nq < 4) {
                __syncthreads();
                if (tid == 0) {
                    choose_conventional(E, C, A.chan_data, fin, A.pool, A.records, A.status + slot);
                    A.counters[slot] = 0;
                }
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
        // Z-type strings: p[m] = |psi(tid + m NT)|^2 and its Walsh-Hadamard
        // transform over the register index m, so a string whose tile-local Z
        // bits are zt (thread bits) + zm (register bits) contributes
        // (-1)^{|tid & zt| + |base & z|} w[zm].  fp32 per thread, fp64 across.
        float w[NA];
#pragma unroll
        for (int m = 0; m < NA; ++m) {
            const float2 v = tile[swz((uint32_t)(tid + m * NT))];
            w[m] = fmaf(v.x, v.x, v.y * v.y);
        }
#pragma unroll
        for (int h = 1; h < NA; h <<= 1)
#pragma unroll
            for (int m = 0; m < NA; ++m)
                if (!(m & h)) {
                    const float a = w[m], b = w[m | h];
                    w[m] = a + b;
                    w[m | h] = a - b;
                }
        // one observable at a time (compact code): warp sums parked in red[],
        // flushed with one barrier pair per 64 / warps observables
        constexpr int NW = (NT + 31) / 32;
        constexpr int kFlush = 64 / NW;
        __syncthreads();  // red[] may still be read by a preceding block sum (racecheck)
        for (int o = 0; o < P.obs_count; ++o) {
            const ObsDesc O = A.obs[P.obs_begin + o];
            const uint32_t zl = to_local<T>(O.zmask, P);
            const int zs = __popcll(base & O.zmask) & 1;
            double part;
            if (O.xmask == 0) {
                const float v = pick_uniform<NA>(w, (int)(zl >> (T - R)));
                const int par = (__popc((uint32_t)tid & zl & (uint32_t)(NT - 1)) + zs) & 1;
                part = par ? -(double)v : (double)v;
            } else {
                const uint64_t xo = O.xmask & ~P.tile_mask;
                const uint32_t xl = to_local<T>(O.xmask, P);
                part = 0.0;
#pragma unroll 1
                for (int m = 0; m < NA; ++m) {
                    const uint32_t L = (uint32_t)(tid + m * NT);
                    const float2 v = tile[swz(L)];
                    float2 wv;
                    if (xo == 0) {
                        wv = tile[swz(L ^ xl)];
                    } else {  // partner amplitude in another tile (read-only pass only)
                        const uint64_t g = base + hoff[L >> CL] + (L & ((1u << CL) - 1u));
                        wv = st[g ^ O.xmask];
                    }
                    // c = conj(w) * v, times i^ny, times (-1)^parity
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
                    part += par ? -t : t;
                }
            }
            constexpr int W = NT < 32 ? NT : 32;
            constexpr unsigned mask = W == 32 ? 0xffffffffu : ((1u << W) - 1u);
#pragma unroll
            for (int sh = W / 2; sh > 0; sh >>= 1) part += __shfl_xor_sync(mask, part, sh);
            const int j = o % kFlush;
            if ((tid & 31) == 0) red[j * NW + (tid >> 5)] = part;
            if (j == kFlush - 1 || o + 1 == P.obs_count) {
                __syncthreads();
                for (int jj = tid; jj <= j; jj += NT) {
                    double v = 0.0;
#pragma unroll
                    for (int ww = 0; ww < NW; ++ww) v += red[jj * NW + ww];
                    A.obs_part[tile_row * A.n_obs + A.obs[P.obs_begin + o - j + jj].slot] = v;
                }
                __syncthreads();
            }
        }
    }

    QT_KMARK(4);
    // ---- shared -> HBM: 16-byte stores of amplitude pairs (thread t owns pairs
    // p = t + m NT, lanes cover 8 x 16 B of each 128-byte run) ----
    constexpr bool kWide = (CL == 4) && (NT >= 8) && (NA >= 2) && (NA <= 32);
    if (P.flags & kPassStore) {
        if constexpr (kWide) {
            float4* gdst = reinterpret_cast<float4*>(st + base + hoff[tid >> 3] + 2 * (tid & 7));
            const uint32_t sb = swz(2u * (uint32_t)tid);
#pragma unroll 4
            for (int m = 0; m < NA / 2; ++m) {
                const uint32_t a = sb ^ swz(2u * (uint32_t)(m * NT));  // swz(L + 1) = swz(L) ^ 1
                const float2 a0 = tile[a], a1 = tile[a ^ 1u];
                gdst[hoff[m * (NT / 8)] >> 1] = make_float4(a0.x, a0.y, a1.x, a1.y);
            }
        } else {
#pragma unroll
            for (int m = 0; m < NA; ++m) {
                const uint32_t L = (uint32_t)(tid + m * NT);
                const uint64_t g = base + hoff[L >> CL] + (L & ((1u << CL) - 1u));
                st[g] = tile[swz(L)];
            }
        }
    }
    QT_KMARK(5);
#ifdef QT_TIMING
    if (A.timing && tid == 0 && (blockIdx.x % 32u) == 7u) {
        for (int i = 0; i < 5; ++i) atomicAdd(A.timing + 8 + i, (unsigned long long)(kt[i + 1] - kt[i]));
        atomicAdd(A.timing + 14, 1ull);
    }
#endif
#undef QT_KMARK
    if constexpr (TC) {
        if (ng > 0) {
            tc::fence_before();
            __syncthreads();
            if ((tid >> 5) == 0) tc::tmem_dealloc(tmem, kTmemCols);
        }
    }
}

inline size_t tile_pass_smem_bytes_impl(int T, int R, bool tcm, int tck = 4) {
    const int CL = T < detail::kCL ? T : detail::kCL;
    const size_t mb = tcm ? (size_t)tc::gate_bytes(tck) : sizeof(float2) * ((size_t)1 << (2 * R));
    const size_t nh = ((((size_t)1 << T) >> CL) + 1) & ~(size_t)1;
    return (tcm && tck == 6 ? 1 : 2) * mb + (sizeof(float2) << T) + sizeof(uint64_t) * nh + 64 * sizeof(double) +
           sizeof(GateDesc) * kMaxPassGates + 16 + 1024;
}

#ifdef QT_TIMING
// diagnostics build: phase-sum counters shared by every tile-pass launch
inline unsigned long long* timing_buffer() {
    static unsigned long long* p = nullptr;
    if (!p) {
        cudaMalloc(&p, 16 * sizeof(unsigned long long));
        cudaMemset(p, 0, 16 * sizeof(unsigned long long));
    }
    return p;
}
#endif

template <int T, int R, bool TC, int TCK = 4>
cudaError_t launch_tr(const TileArgs& a, int step, uint32_t ntiles, int nslots, cudaStream_t s) {
    using Cfg = TileCfg<T, R, TC, TCK>;
    const size_t smem = Cfg::kBytes;
    static bool configured = false;
    static uint32_t resident = 0;  // CTAs resident on the whole device
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(tile_pass_kernel<T, R, TC, TCK>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0, dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_pass_kernel<T, R, TC, TCK>, Cfg::NT, smem);
        resident = (uint32_t)(per_sm * sms);
        configured = true;
    }
    TileArgs b = a;
    b.prefetch = 0;  // measured: L2 prefetch of the next wave's tiles did not help (64% vs 66% of HBM)
#ifdef QT_TIMING
    b.timing = timing_buffer();
#endif
    (void)resident;
    dim3 grid(ntiles, nslots);
    tile_pass_kernel<T, R, TC, TCK><<<grid, Cfg::NT, smem, s>>>(b, step);
    return cudaGetLastError();
}

}  // namespace qt
