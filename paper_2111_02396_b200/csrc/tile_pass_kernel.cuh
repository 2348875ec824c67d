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
//               gather).  Gates flagged non-TC (the device-chosen operators of
//               conventional channels, k <= 2) use the CUDA-core path with
//               R = 5 on the fp32 tile.  TCK = 5 (f = 5 plans): 3xTF32 with A
//               in TMEM, one gate at a time.
#pragma once
#include <cuda_fp16.h>

#include "tile_pass.cuh"

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

// One tensor-core gate of a run (4 qubits, kind::f16; tc_common.cuh).  Run start
// (kGateRunStart): gather the fp32 tile in this gate's register layout, pick the
// power-of-two tile scale (max |component| -> [2^6, 2^7) / 2^shift, so any
// contraction of the tile stays below 2^13.5 < f16 max) and write the hi / lo
// operand rows in place.  Then one elected thread issues the 8 MMAs (2 groups
// x 4 K-steps, N = 64) and every thread reads its D rows (TMEM lane = thread)
// and writes the 32 outputs either into the next gate's operand layout (run
// continues: byte offsets from G.xu) or unscaled into the fp32 tile (run end).
template <int T>
__device__ __forceinline__ void tc_gate_f16(float2* tile, uint32_t w_smem, const GateDesc& G, const GateDesc* Gn,
                                            uint32_t tmem, uint64_t* mbar, uint32_t& phase, float& run_scale,
                                            float& run_inv, double* red) {
    using namespace tc;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    char* const tb8 = reinterpret_cast<char*>(tile);
    const uint32_t tile_s = (uint32_t)__cvta_generic_to_shared(tile);
    const int gk = G.k;
    if (gk & kGateRunStart) {
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
        const int shift = (gk >> kGateShiftBit) & 0xff;
        int se = 260 - (int)((__float_as_uint(amax) >> 23) & 0xffu) - shift;  // amax * 2^(se - 127) in [2^6, 2^7)
        se = min(max(se, 1), 253);
        run_scale = __uint_as_float((uint32_t)se << 23);
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
    if (tid == 0) {
        fence_after();
        constexpr uint32_t idesc = idesc_f16_m128(64);
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
                mma_f16_ss(tmem + 64 * g, smem_desc_sw128(tile_s + g * kF16GroupBytes + ks * 32),
                           smem_desc_sw128(w_smem + ks * 32), idesc, ks > 0);
        mma_commit(mbar);
    }
    __syncwarp();
    // output addressing: next operand layout (run continues) or the fp32 tile
    const bool chain = Gn != nullptr && (Gn->k & (kGateTC | kGateRunStart)) == kGateTC;
    uint32_t lo[16], obase, ogrp;
    if (chain) {
        const uint4 x0 = *reinterpret_cast<const uint4*>(&G.xu[0]);   // xu[0..7]
        const uint2 x1 = *reinterpret_cast<const uint2*>(&G.xu[8]);   // xu[8..11]
        const uint32_t xu[12] = {x0.x & 0xffffu, x0.x >> 16, x0.y & 0xffffu, x0.y >> 16,
                                 x0.z & 0xffffu, x0.z >> 16, x0.w & 0xffffu, x0.w >> 16,
                                 x1.x & 0xffffu, x1.x >> 16, x1.y & 0xffffu, x1.y >> 16};
        obase = 0;
#pragma unroll
        for (int i = 0; i < 7; ++i)
            if ((tid >> i) & 1u) obase ^= xu[5 + i];
        ogrp = xu[4];
        lo[0] = 0;
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int x = 0; x < (1 << m); ++x) lo[x + (1 << m)] = lo[x] ^ xu[m];
    } else {
        fp32_layout<T>(G, lo, ogrp, obase);
    }
    mbar_wait(mbar, phase);  // both groups done: the operand rows may be overwritten
    phase ^= 1u;
    fence_after();
    const uint32_t lane_off = (warp * 32u) << 16;
    const uint64_t inv2 = pk2(run_inv, run_inv);
#pragma unroll 1
    for (int g = 0; g < 2; ++g) {
        uint32_t h0[32], h1[32];
        tmem_ld32(tmem + lane_off + 64 * g, h0);
        tmem_ld32(tmem + lane_off + 64 * g + 32, h1);
        tmem_wait_ld();
        const uint32_t b = obase ^ (g ? ogrp : 0u);
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const uint64_t y = add2(pk2(__uint_as_float(h0[2 * c]), __uint_as_float(h0[2 * c + 1])),
                                    pk2(__uint_as_float(h1[2 * c]), __uint_as_float(h1[2 * c + 1])));
            if (chain)
                *reinterpret_cast<uint2*>(tb8 + (b ^ lo[c])) = split_f16(y);
            else
                *reinterpret_cast<float2*>(tb8 + (b ^ lo[c])) = upk2(mul2(y, inv2));
        }
    }
    fence_before();
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

// Apply one padded 5-qubit gate on tensor cores (128 threads): thread t owns
// subvector s = t of 32 amplitudes (register bits 0..4 = the gate bits), TMEM
// lane t.  N = K = 64: TMEM columns D [0,64), A hi [64,128), A lo [128,192);
// W in shared memory as two K-chunks of [64][32] tf32 (hi, then lo at +16 KB).
__device__ __forceinline__ void apply_tc_gate5(float2* tile, uint32_t w_smem, uint32_t pbase,
                                               const uint32_t (&unit)[5], uint32_t tmem, uint64_t* mbar,
                                               uint32_t& phase) {
    using namespace tc;
    const int tid = threadIdx.x;
    char* const tb8 = reinterpret_cast<char*>(tile);
    uint32_t lo[32];
    lo[0] = pbase;
#pragma unroll
    for (int m = 0; m < 5; ++m)
#pragma unroll
        for (int x = 0; x < (1 << m); ++x) lo[x + (1 << m)] = lo[x] ^ unit[m];
    const uint32_t lane = (uint32_t)(tid & 96) << 16;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // configurations 16 h .. 16 h + 15 = A columns 32 h .. 32 h + 31
        uint32_t hi[32], lw[32];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const float2 v = *reinterpret_cast<const float2*>(tb8 + lo[16 * h + c]);
            const uint32_t hx = __float_as_uint(v.x) & 0xFFFFE000u, hy = __float_as_uint(v.y) & 0xFFFFE000u;
            hi[2 * c] = hx;
            hi[2 * c + 1] = hy;
            lw[2 * c] = __float_as_uint(v.x - __uint_as_float(hx));
            lw[2 * c + 1] = __float_as_uint(v.y - __uint_as_float(hy));
        }
        tmem_st32(tmem + lane + 64 + 32 * h, hi);
        tmem_st32(tmem + lane + 128 + 32 * h, lw);
    }
    tmem_wait_st();
    fence_before();
    __syncthreads();
    if (tid == 0) {
        fence_after();
        constexpr uint32_t idesc = idesc_tf32_m128(64);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const uint32_t off = (uint32_t)((ks >> 2) * 8192 + (ks & 3) * 32);
            const uint64_t bh = smem_desc_sw128(w_smem + off);
            const uint64_t bl = smem_desc_sw128(w_smem + (uint32_t)w_part_bytes(5) + off);
            mma_tf32_ts_n(tmem, tmem + 64 + ks * 8, bh, idesc, ks > 0);
            mma_tf32_ts_n(tmem, tmem + 128 + ks * 8, bh, idesc, 1);
            mma_tf32_ts_n(tmem, tmem + 64 + ks * 8, bl, idesc, 1);
        }
        mma_commit(mbar);
    }
    __syncwarp();
    mbar_wait(mbar, phase);
    phase ^= 1u;
    fence_after();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t v[32];
        tmem_ld32(tmem + lane + 32 * h, v);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c)
            *reinterpret_cast<float2*>(tb8 + lo[16 * h + c]) =
                make_float2(__uint_as_float(v[2 * c]), __uint_as_float(v[2 * c + 1]));
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
    // shared memory: [W/matrix buffers x2][tile][hoff][red][gdesc][mbar], base 1024-aligned
    static constexpr size_t kMbufBytes = TC ? (size_t)tc::gate_bytes(TCK) : sizeof(float2) * ((size_t)1 << (2 * R));
    static constexpr size_t kTileOff = 2 * kMbufBytes;
    static constexpr size_t kHoffOff = kTileOff + sizeof(float2) * TILE;
    static constexpr size_t kRedOff = kHoffOff + sizeof(uint64_t) * ((NH + 1) & ~1);
    static constexpr size_t kGdescOff = kRedOff + 64 * sizeof(double);
    static constexpr size_t kMbarOff = kGdescOff + sizeof(GateDesc) * kMaxPassGates;
    static_assert(!TC || TCK != 4 || tc::gate_bytes(4) == tc::kF16GateBytes, "f16 operand size");
    static constexpr size_t kBytes = kMbarOff + 16 + 1024;  // + alignment slack
};

template <int T, int R, bool TC, int TCK = 4>
__global__ void __launch_bounds__(TileCfg<T, R, TC, TCK>::NT,
                                  TC ? (TCK == 5 ? 2 : 4) : ((R <= 4 && T == 12) ? QT_MINB : 1))
tile_pass_kernel(const TileArgs A, const int step) {
    using Cfg = TileCfg<T, R, TC, TCK>;
    // TMEM: TCK = 4: f16 runs use D of both groups (2 x 64 columns), 3xTF32 single
    // gates D0 / D1 / A hi / A lo (4 x 32); TCK = 5: D 64 + A hi/lo 128
    constexpr uint32_t kTmemCols = TCK == 5 ? 256 : 128;  // CTAs per SM share 512 columns
    constexpr int NT = Cfg::NT;
    constexpr int NA = Cfg::NA;
    constexpr int CL = Cfg::CL;
    constexpr int NH = Cfg::NH;
    const int slot = A.slots ? A.slots[blockIdx.y] : (int)blockIdx.y;
    if (step >= A.pass_count[slot]) return;
    const PassDesc P = A.passes[A.pass_start[slot] + step];

    extern __shared__ unsigned char smem_raw[];
    // 1024-byte alignment by offsetting smem_raw itself (keeps the pointer in the
    // shared address space: LDS/STS instead of generic LD/ST)
    const uint32_t smem_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    unsigned char* sm = smem_raw + (((smem_base + 1023u) & ~1023u) - smem_base);
    unsigned char* mbuf = sm;  // 2 x kMbufBytes
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

    uint32_t tmem = 0, phase = 0;
    if constexpr (TC) {
        if (ng > 0 && (tid >> 5) == 0) tc::tmem_alloc(&s_tmem, kTmemCols);  // CTAs / SM share 512 columns
        if (tid == 0) {
            tc::mbar_init(mbar, 1);
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
    // warm L2 with the same-slot tile one resident wave ahead (its CTA will load it soon)
    if (A.prefetch && blockIdx.x + A.prefetch < gridDim.x) {
        const uint64_t nb = pdep64((uint64_t)(blockIdx.x + A.prefetch), nmask & ~P.tile_mask);
        for (int h = tid; h < NH; h += NT)
            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(st + nb + hoff[h]));
    }
    // HBM -> shared.  Wide tiles: 16-byte loads of amplitude pairs (thread t owns
    // pairs p = t + m NT, so lanes cover 8 x 16 B of each 128-byte run), all
    // issued before the swizzled 8-byte shared stores.  hoff is linear in its
    // index bits: hoff[(t >> 3) + m NT / 8] = hoff[t >> 3] | hoff[m NT / 8].
    constexpr bool kWide = (CL == 4) && (NT >= 8) && (NA >= 2) && (NA <= 32);
    // 8-byte asynchronous copies: the swizzle keeps amplitude pairs adjacent but
    // not 16-byte aligned.  (Measured at n = 30: register-staged 16-byte loads
    // 61% of HBM peak vs async 8-byte copies 68%.)
    // hoff and swz are linear in the index bits: slot L = tid + m NT has global
    // offset hoff[tid >> CL] + hoff[m NT >> CL] + (tid & (2^CL - 1)) (NT >= 2^CL)
    if constexpr (NT >= (1 << CL)) {
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
    cp_async_wait_all();  // gate descriptors (the tile may still be in flight for other threads)
    __syncthreads();
    auto mat_bytes = [](const GateDesc& G) -> int {
        return (TC && (G.k & kGateTC)) ? tc::gate_bytes(TCK) : (int)sizeof(float2) * (1 << (2 * (G.k & 0xff)));
    };
    if (ng > 0) {
        const int chunks = mat_bytes(gdesc[0]) >> 4;
        for (int c = tid; c < chunks; c += NT)
            cp_async16(mbuf + 16 * c, reinterpret_cast<const char*>(A.pool + gdesc[0].mat_off) + 16 * c);
        cp_async_commit();
    }
    float run_scale = 1.f, run_inv = 1.f;  // tensor-core run: tile scale (uniform)
    for (int gi = 0; gi < ng; ++gi) {
        const GateDesc& G = gdesc[gi];
        cp_async_wait_all();
        if constexpr (TC) tc::fence_proxy_async();  // cp.async W / st.shared operand -> tensor-core reads
        __syncthreads();  // tile writes of the previous gate + this gate's matrix visible
        if (gi + 1 < ng) {
            const GateDesc& Gn = gdesc[gi + 1];
            unsigned char* dst = mbuf + ((gi + 1) & 1) * Cfg::kMbufBytes;
            const char* src = reinterpret_cast<const char*>(A.pool + Gn.mat_off);
            if (TC && TCK == 4 && (Gn.k & kGateTC)) {
                constexpr int kPer = tc::kF16GateBytes / 16 / NT;
#pragma unroll
                for (int c = 0; c < kPer; ++c) cp_async16(dst + 16 * (tid + c * NT), src + 16 * (tid + c * NT));
            } else {
                const int chunks = mat_bytes(Gn) >> 4;
                for (int c = tid; c < chunks; c += NT) cp_async16(dst + 16 * c, src + 16 * c);
            }
            cp_async_commit();
        }
        unsigned char* mcur = mbuf + (gi & 1) * Cfg::kMbufBytes;
        if constexpr (TC && TCK == 4) {
            if (G.k & kGateF16) {
                tc_gate_f16<T>(tile, (uint32_t)__cvta_generic_to_shared(mcur), G, gi + 1 < ng ? &gdesc[gi + 1] : nullptr,
                               tmem, mbar, phase, run_scale, run_inv, red);
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
                                  phase);
                else if constexpr (R == 5 && TCK == 5)
                    apply_tc_gate5(tile, (uint32_t)__cvta_generic_to_shared(mcur), swz(tb) << 3, unit, tmem, mbar,
                                   phase);
            } else if ((G.k & 0xff) == 1) {  // device-chosen conventional operators (q <= 2)
                apply_fused<1, R>(tile, reinterpret_cast<const float2*>(mcur), swz(tb) << 3, unit);
            } else {
                apply_fused<2, R>(tile, reinterpret_cast<const float2*>(mcur), swz(tb) << 3, unit);
            }
            continue;
        }
        dispatch_fused<R>(G.k & 0xff, tile, reinterpret_cast<const float2*>(mcur), swz(tb) << 3, unit);
    }
    cp_async_wait_all();  // a pass without gates still has its tile in flight
    __syncthreads();

    // ---- epilogues (read-only on the tile) ----
    const uint32_t ntiles = gridDim.x;
    const uint64_t tile_row = (uint64_t)slot * ntiles + blockIdx.x;
    if (P.flags & kPassRho) {
        const EventDesc E = A.events[P.event];
        const ChanDesc C = A.chans[E.chan];
        const uint32_t ql = to_local<T>(C.qmask, P);  // channel qubits as tile-local bits
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

    // ---- shared -> HBM ----
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
    return 2 * mb + (sizeof(float2) << T) + sizeof(uint64_t) * nh + 64 * sizeof(double) +
           sizeof(GateDesc) * kMaxPassGates + 16 + 1024;
}

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
    (void)resident;
    dim3 grid(ntiles, nslots);
    tile_pass_kernel<T, R, TC, TCK><<<grid, Cfg::NT, smem, s>>>(b, step);
    return cudaGetLastError();
}

}  // namespace qt
