// tile_pass_kernel.cuh -- K1 tile-pass kernel (Alg. 1, applied to a whole
// program of fused gates per HBM sweep) with the K2 / K3a / K4 epilogues.
//
//   TC = false: fused gates on FP32 CUDA cores, 2^R amplitudes per thread in
//               registers, one swizzled shared-memory re-layout per gate.
//   TC = true : T = 12, 128 threads.  Fused gates are padded to 4 qubits and
//               applied as the real GEMM of tc_common.cuh on tcgen05 tensor
//               cores (3xTF32, A = amplitudes in TMEM, B = W in shared memory,
//               D in TMEM); gates flagged non-TC (the device-chosen operators of
//               conventional channels, k <= 2) use the CUDA-core path with R = 5.
#pragma once
#include "tile_pass.cuh"

// 1: tensor-core gates issue both M-groups in one MMA batch (256 TMEM columns,
// 2 CTAs / SM); 0: two batches sharing one A buffer (128 columns, 4 CTAs / SM).
#ifndef QT_TC_ONE_ROUND
#define QT_TC_ONE_ROUND 0
#endif

namespace qt {

namespace detail {

// Apply one padded 4-qubit gate on tensor cores.  Thread t owns subvectors
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
#if QT_TC_ONE_ROUND
    // variant: both groups' A in TMEM (A_g hi/lo at [64 + 64 g, 128 + 64 g)),
    // one MMA batch and one round trip per gate; needs 256 TMEM columns
    for (int g = 0; g < 2; ++g) {
        uint32_t hi[32], lw[32];
        gather(g, hi, lw);
        tmem_st32(tmem + lane_off + 64 + 64 * g, hi);
        tmem_st32(tmem + lane_off + 96 + 64 * g, lw);
    }
    tmem_wait_st();
    fence_before();
    __syncthreads();
    if (tid == 0) {
        fence_after();
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            const uint64_t bh = smem_desc_sw128(w_smem + ks * 32);
            const uint64_t bl = smem_desc_sw128(w_smem + kWBytes + ks * 32);
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                mma_tf32_ts(tmem + 32 * g, tmem + 64 + 64 * g + ks * 8, bh, ks > 0);
                mma_tf32_ts(tmem + 32 * g, tmem + 96 + 64 * g + ks * 8, bh, 1);
                mma_tf32_ts(tmem + 32 * g, tmem + 64 + 64 * g + ks * 8, bl, 1);
            }
        }
        mma_commit(mbar);
    }
    __syncwarp();
    mbar_wait(mbar, phase);
    phase ^= 1u;
    fence_after();
    scatter(0);
    scatter(1);
    fence_before();
    return;
#endif
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
    static constexpr size_t kBytes = kMbarOff + 16 + 1024;  // + alignment slack
};

template <int T, int R, bool TC, int TCK = 4>
__global__ void __launch_bounds__(TileCfg<T, R, TC, TCK>::NT,
                                  TC ? ((TCK == 5 || QT_TC_ONE_ROUND) ? 2 : 4) : ((R <= 4 && T == 12) ? QT_MINB : 1))
tile_pass_kernel(const TileArgs A, const int step) {
    using Cfg = TileCfg<T, R, TC, TCK>;
    constexpr uint32_t kTmemCols = (TCK == 5 || QT_TC_ONE_ROUND) ? 256 : 128;  // CTAs per SM share 512 columns
    constexpr int NT = Cfg::NT;
    constexpr int NA = Cfg::NA;
    constexpr int CL = Cfg::CL;
    constexpr int NH = Cfg::NH;
    const int slot = blockIdx.y;
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
    for (int c = tid; c < ng; c += NT) cp_async16(gdesc + c, A.gates + P.gate_begin + c);
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
    // measured (n = 30 single-gate passes): register-staged 16-byte loads 61% of
    // HBM peak vs 8-byte cp.async 68% -> loads stay asynchronous; stores are wide
    constexpr bool kWideLoad = false;
    if constexpr (kWideLoad) {
        const float4* gsrc = reinterpret_cast<const float4*>(st + base + hoff[tid >> 3] + 2 * (tid & 7));
        float4 v[NA / 2];
#pragma unroll
        for (int m = 0; m < NA / 2; ++m) v[m] = __ldcs(gsrc + (hoff[m * (NT / 8)] >> 1));
#pragma unroll
        for (int m = 0; m < NA / 2; ++m) {
            const uint32_t L = 2u * (uint32_t)(tid + m * NT);
            tile[swz(L)] = make_float2(v[m].x, v[m].y);
            tile[swz(L + 1)] = make_float2(v[m].z, v[m].w);
        }
    } else {
        // 8-byte asynchronous copies (small tiles)
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
    for (int gi = 0; gi < ng; ++gi) {
        const GateDesc G = gdesc[gi];
        cp_async_wait_all();
        if constexpr (TC) tc::fence_proxy_async();  // cp.async-written W -> tensor-core reads
        __syncthreads();  // tile writes of the previous gate + this gate's matrix visible
        if (gi + 1 < ng) {
            const GateDesc Gn = gdesc[gi + 1];
            unsigned char* dst = mbuf + ((gi + 1) & 1) * Cfg::kMbufBytes;
            const int chunks = mat_bytes(Gn) >> 4;
            for (int c = tid; c < chunks; c += NT)
                cp_async16(dst + 16 * c, reinterpret_cast<const char*>(A.pool + Gn.mat_off) + 16 * c);
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
        unsigned char* mcur = mbuf + (gi & 1) * Cfg::kMbufBytes;
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
            } else {
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
                    // c = conj(w) * v, times i^ny, times (-1)^parity
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
            }
            s = block_sum<NT>(s, red);
            if (tid == 0) A.obs_part[tile_row * A.n_obs + O.slot] = s;
        }
    }

    // ---- shared -> HBM ----
    if (P.flags & kPassStore) {
        if constexpr (kWide) {
            float4* gdst = reinterpret_cast<float4*>(st + base + hoff[tid >> 3] + 2 * (tid & 7));
#pragma unroll
            for (int m = 0; m < NA / 2; ++m) {
                const uint32_t L = 2u * (uint32_t)(tid + m * NT);
                const float2 a0 = tile[swz(L)], a1 = tile[swz(L + 1)];
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
