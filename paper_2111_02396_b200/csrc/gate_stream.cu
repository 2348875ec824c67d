// gate_stream.cu -- K1 for one fused k-qubit gate per HBM pass (k <= 6): the
// streaming gate-pass kernel behind qt_apply_gate (Alg. 1, one gate;
// the pass cost model of P:135 is exactly one read and one write of the state).
//
// A tile is 128 rows x 2^K configurations (K = max(k, 4); gates of k < 4 qubits
// are padded with the lowest free qubits, identity on them): the row qubits are
// the 7 lowest qubits that are not matrix qubits, the tile spans qubits 0..L-1
// (L = 7 + the matrix qubits below L) plus the matrix qubits above L.  Tiles
// move by TMA: a 5-D tensor map over the state (8-byte elements) with boxes
// [qubits 0..3 | qubits 4..L-1 | up to two high matrix qubits | rest], SWIZZLE_128B
// (16-byte chunk index ^= bits 7..9 of the tile byte offset), several boxes per tile
// when more high matrix qubits remain; TMA stores write the tile back in place.
//
// Roles (one persistent CTA per SM): one producer thread issues the loads into a
// ring of STAGES tiles and, once a tile is computed, its store (the stage is
// reloaded after the store has read it); NWG compute warpgroups take tiles in turn.
// Per tile and warpgroup: every thread owns one row (TMEM lane), gathers its 2^K
// amplitudes, scales them by a power of two (per row: D_row = A_row W, so the scale
// is exact and thread-local), splits them into f16 hi / lo and stores A = [x_hi | x_lo]
// into TMEM; one thread issues the real GEMM D = x_hi W_hi + x_lo W_hi + x_hi W_lo
// (3 x 2^(K-3) tcgen05.mma kind::f16 M128 N2^(K+1) K16, A from TMEM, W from shared
// memory, fp32 accumulate in TMEM; ~22 significant bits as in the trajectory K1);
// every thread reads its D row back (tcgen05.ld), unscales it and writes the
// amplitudes to the tile in place.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tc_common.cuh"

namespace qt {
namespace gs {

struct GsArgs {
    uint64_t tile_mask;     // state qubits of a tile (low run 0..L-1 and the high matrix qubits)
    uint32_t ntiles;        // 2^(n - T)
    int L;                  // low run
    int nops;               // TMA boxes per tile
    uint32_t op_bytes;      // bytes per box
    uint32_t row_basis[7];  // swizzled tile byte offset of row bit j (lane bits 0..4, warp bits 5, 6)
    uint32_t cfg_basis[6];  // swizzled tile byte offset of matrix bit m
    int32_t op_rest[16];    // rest coordinate (units of 2^L amplitudes) of box o
    int pair;               // matrix bit 0 is tile bit 0: configurations 2i, 2i + 1 form one 16-byte pair
    int reps;               // applications per tile (1; > 1 only in the QT_GS_REPS experiment)
};

template <int K>
struct Cfg {
    static constexpr int CFG = 1 << K;
    // STAGES is a multiple of NWG: stage s is always computed by warpgroup s % NWG, so
    // every barrier of a stage is waited on in phase order (a waiter two phases ahead of
    // a barrier would see the parity of an old phase and pass)
    // K = 6: one warpgroup of 256 threads, two per row (configurations 0..31 / 32..63), so
    // that one of the two 64 KB stages is free for loads while the other computes
    static constexpr int SPLIT = K == 6 ? 2 : 1;      // threads per row
    static constexpr int WGT = 128 * SPLIT;            // threads per compute warpgroup
    static constexpr int NWG = K == 6 ? 1 : (K == 5 ? 3 : 4);
    static constexpr uint32_t TILE_BYTES = 128u * CFG * 8u;
    static constexpr int STAGES = K == 4 ? 12 : (K == 5 ? 6 : 2);
    static constexpr int STORE_LAG = STAGES >= 6 ? 1 : 0;
    static constexpr int N = 2 * CFG;                           // real outputs per row
    static constexpr uint32_t W_BYTES = (uint32_t)N * (4 * CFG) * 2;  // N rows x [W_hi (2 CFG) | W_lo (2 CFG)] f16
    static constexpr uint32_t COLS = 4u * CFG;                  // TMEM columns per warpgroup: D (N) + A (2 CFG)
    static constexpr uint32_t TCOLS = NWG * COLS <= 256 ? 256 : 512;  // power of two
    static constexpr int KS = (2 * CFG) / 16;                   // K16 steps per part
    static constexpr uint32_t W_OFF = STAGES * TILE_BYTES;
    static constexpr uint32_t BAR_OFF = W_OFF + W_BYTES;
    static constexpr uint32_t AMX_OFF = BAR_OFF + 512;          // SPLIT > 1: per-thread row maxima
    static constexpr uint32_t SMEM = AMX_OFF + (SPLIT > 1 ? 4 * WGT : 0) + 1024;  // + alignment slack
    static constexpr int THREADS = NWG * WGT + 64;               // + loader warp + storer warp
    static constexpr int MAXREG = (65536 / THREADS) & ~7;
    static_assert(SMEM <= 232448, "shared memory");
    static_assert(STAGES % NWG == 0, "stage -> warpgroup map");
    static_assert(3 * STAGES + NWG + 1 <= 63, "barrier slots");
};

__device__ __forceinline__ bool try_wait(uint32_t a, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok) : "r"(a), "r"(phase) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void wait(uint32_t a, uint32_t phase, const volatile uint32_t* g_dbg_words = nullptr) {
#ifdef QT_GS_WATCHDOG
    long long spins = 0;
    while (!try_wait(a, phase)) {
        if (++spins == (1ll << 25) && (threadIdx.x & 31) == 0) {
            printf("gate_stream watchdog: block %d thread %d barrier %u parity %u\n", blockIdx.x, threadIdx.x, a, phase);
            if (g_dbg_words) {
                const volatile uint32_t* d = g_dbg_words;
                printf("  block %d progress (warp: j*16+step): %u %u %u %u | %u %u %u %u | %u %u %u %u | %u %u %u %u\n",
                       blockIdx.x, d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8], d[9], d[10], d[11], d[12], d[13],
                       d[14], d[15]);
            }
        }
        if (spins == (1ll << 27)) __trap();
    }
#else
    (void)g_dbg_words;
    while (!try_wait(a, phase)) {
    }
#endif
}
__device__ __forceinline__ void bar_init(uint32_t a, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(c) : "memory");
}
__device__ __forceinline__ void arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load(uint32_t dst, const CUtensorMap* tm, int32_t crest, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %2, %2, "
        "%2, %3}], [%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(0), "r"(crest), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* tm, int32_t crest, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %1, %1, %1, %2}], [%3];\n" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(0), "r"(crest), "r"(src)
                 : "memory");
}
template <int NTH = 128>
__device__ __forceinline__ void bar_wg(int wg) { asm volatile("bar.sync %0, %1;\n" ::"r"(1 + wg), "n"(NTH) : "memory"); }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

// f16 hi / lo split of a scaled component: hi = x with its 13 low mantissa bits cleared
// (exact in f16 in the scaled range), lo = the remainder rounded to f16.
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
    const float hx = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    const float hy = __uint_as_float(__float_as_uint(y) & 0xFFFFE000u);
    const __half2 h2 = __floats2half2_rn(hx, hy);
    const __half2 l2 = __floats2half2_rn(x - hx, y - hy);
    hi = *reinterpret_cast<const uint32_t*>(&h2);
    lo = *reinterpret_cast<const uint32_t*>(&l2);
}

template <int K>
__global__ void __launch_bounds__(Cfg<K>::THREADS, 1) __maxnreg__(Cfg<K>::MAXREG)
    gate_stream_kernel(const __grid_constant__ CUtensorMap tm, const GsArgs a, const void* __restrict__ w_glob) {
    using C = Cfg<K>;
    constexpr int CFG = C::CFG;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw_s = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t pad = ((raw_s + 1023u) & ~1023u) - raw_s;
    unsigned char* sm = smem_raw + pad;
    const uint32_t sm_s = raw_s + pad;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t bar = sm_s + C::BAR_OFF;
    // barriers: full[S] (TMA bytes), computed[S] (128 threads), mma[NWG], W, empty[S] (store read)
    const uint32_t w_bar = bar + 8u * (2 * C::STAGES + C::NWG);
    const uint32_t empty_bar = w_bar + 8u;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + C::BAR_OFF + 504);
    volatile uint32_t* dbg = reinterpret_cast<volatile uint32_t*>(sm + C::BAR_OFF + 400);  // watchdog build: progress
#ifdef QT_GS_WATCHDOG
#define GS_PROG(step) \
    if (lane == 0) dbg[warp & 15] = j * 16u + (step);
#else
#define GS_PROG(step)
#endif
    const int producer = C::NWG * C::WGT;
    if (warp == 0) tc::tmem_alloc(tslot, C::TCOLS);
    if (tid == producer) {
        for (int s = 0; s < C::STAGES; ++s) {
            bar_init(bar + 8u * s, 1);                       // full: producer arrive + TMA bytes
            bar_init(bar + 8u * (C::STAGES + s), C::WGT);    // computed: the warpgroup's threads
        }
        for (int w = 0; w < C::NWG; ++w) bar_init(bar + 8u * (2 * C::STAGES + w), 1);  // MMA commit
        bar_init(w_bar, 1);
        for (int s = 0; s < C::STAGES; ++s) bar_init(empty_bar + 8u * s, 1);
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t G = gridDim.x;
    const uint32_t my_tiles = blockIdx.x < a.ntiles ? (a.ntiles - 1u - blockIdx.x) / G + 1u : 0u;

    auto crest_of = [&](uint32_t j) {
        // the tile index with zeros inserted at the high matrix qubits: the tile's first
        // amplitude in units of 2^L (the rest coordinate)
        uint64_t base = (uint64_t)(blockIdx.x + j * G);
        uint64_t hm = a.tile_mask >> a.L;
        while (hm) {
            const int p = __ffsll((long long)hm) - 1;
            hm &= hm - 1;
            base = (base & ((1ull << p) - 1ull)) | ((base >> p) << (p + 1));
        }
        return (int32_t)base;
    };
    if (warp == C::NWG * C::WGT / 32) {
        // ---------------- loader: TMA loads into free stages ----------------
        if (lane == 0) {
            expect_tx(w_bar, C::W_BYTES);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                             sm_s + C::W_OFF),
                         "l"(w_glob), "r"(C::W_BYTES), "r"(w_bar)
                         : "memory");
            for (uint32_t j = 0; j < my_tiles; ++j) {
                const int s = (int)(j % C::STAGES);
                const uint32_t r = j / C::STAGES;
                if (j >= (uint32_t)C::STAGES) wait(empty_bar + 8u * s, (r - 1u) & 1u, dbg);  // previous occupant stored
                expect_tx(bar + 8u * s, C::TILE_BYTES);
                const int32_t cr = crest_of(j);
                const uint32_t st = sm_s + (uint32_t)s * C::TILE_BYTES;
                for (int o = 0; o < a.nops; ++o) tma_load(st + (uint32_t)o * a.op_bytes, &tm, cr + a.op_rest[o], bar + 8u * s);
            }
        }
    } else if (warp == C::NWG * C::WGT / 32 + 1) {
        // ---------------- storer: TMA stores of computed tiles, in order ----------------
        // a stage is released once its store has read it; with many stages one store
        // group stays in flight behind the newest (two reads overlap), with two stages
        // (K = 6) each stage is released as soon as it is read
        if (lane == 0) {
            for (uint32_t j = 0; j < my_tiles; ++j) {
                const int s = (int)(j % C::STAGES);
                wait(bar + 8u * (C::STAGES + s), (j / C::STAGES) & 1u, dbg);
                const int32_t cr = crest_of(j);
                const uint32_t st = sm_s + (uint32_t)s * C::TILE_BYTES;
                for (int o = 0; o < a.nops; ++o) tma_store(&tm, cr + a.op_rest[o], st + (uint32_t)o * a.op_bytes);
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                if (C::STORE_LAG == 0) {
                    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                    arrive(empty_bar + 8u * s);
                } else if (j >= 1) {
                    asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
                    arrive(empty_bar + 8u * ((j - 1) % C::STAGES));
                }
            }
            asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
        }
    } else {
        // ---------------- compute warpgroups ----------------
        constexpr int CPT = CFG / C::SPLIT;  // configurations per thread
        const int wg = warp / (4 * C::SPLIT), wq = warp & 3, hsel = (warp >> 2) & (C::SPLIT - 1);
        const int wtid = tid % C::WGT;
        const int cbase = hsel * CPT;  // this thread's first configuration
        const uint32_t tl = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)wg * C::COLS;  // lane, D column 0
        const uint32_t tA = tl + (uint32_t)C::N;                                          // A: hi, then lo
        uint32_t ro = 0;
        {
            const int r = lane | (wq << 5);
#pragma unroll
            for (int j = 0; j < 7; ++j)
                if ((r >> j) & 1) ro ^= a.row_basis[j];
        }
        uint32_t cb[K];
#pragma unroll
        for (int m = 0; m < K; ++m) cb[m] = a.cfg_basis[m];
        auto cfg_off = [&](int c) {
            uint32_t o = 0;
#pragma unroll
            for (int m = 0; m < K; ++m)
                if ((c >> m) & 1) o ^= cb[m];
            return o;
        };
        const bool pair = a.pair != 0;
        wait(w_bar, 0);
        __syncwarp();
        uint32_t mma_phase = 0;
        for (uint32_t j = (uint32_t)wg; j < my_tiles; j += C::NWG) {
            const int s = (int)(j % C::STAGES);
            GS_PROG(1);
            wait(bar + 8u * s, (j / C::STAGES) & 1u);
            __syncwarp();
            GS_PROG(2);  // the tcgen05 .sync.aligned operations below need converged warps
            unsigned char* tile = sm + (size_t)s * C::TILE_BYTES;
            // (experiment: a.reps > 1 applies the gate reps times per tile -- the cost of
            // several gates per HBM pass in this pipeline; tools/gs_reps.py)
            for (int rep = 0; rep < a.reps; ++rep) {
            if (rep) bar_wg<C::WGT>(wg);  // the previous application's write-backs are visible
            // ---- gather the row's 2^K amplitudes, per-row power-of-two scale ----
            auto load16 = [&](int c0, float2 (&v)[16]) {
                if (pair) {
#pragma unroll
                    for (int c = 0; c < 16; c += 2) {
                        const float4 f = *reinterpret_cast<const float4*>(tile + (ro ^ cfg_off(c0 + c)));
                        v[c] = make_float2(f.x, f.y);
                        v[c + 1] = make_float2(f.z, f.w);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c) v[c] = *reinterpret_cast<const float2*>(tile + (ro ^ cfg_off(c0 + c)));
                }
            };
            // K >= 5: two passes over the tile (amax, then split) so that 32 / 64 amplitudes
            // need not stay in registers; K = 4: one pass
            constexpr int NCH = CPT / 16;
            constexpr int KEEP = (K == 5) ? 1 : NCH;
            float2 v[KEEP][16];
            float amax = 0.f;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                float2(&w)[16] = v[KEEP == 1 ? 0 : ch];
                load16(cbase + 16 * ch, w);
#pragma unroll
                for (int c = 0; c < 16; ++c) amax = fmaxf(amax, fmaxf(fabsf(w[c].x), fabsf(w[c].y)));
            }
            if constexpr (C::SPLIT > 1) {
                // the row's other half: thread wtid ^ 128 (same lane quarter, other warp half)
                float* amx = reinterpret_cast<float*>(sm + C::AMX_OFF);
                amx[wtid] = amax;
                bar_wg<C::WGT>(wg);
                amax = fmaxf(amax, amx[wtid ^ 128]);
            }
            // amax * 2^(se - 127) in [2^6, 2^7): |A| < 2^7, row outputs < 2^7 * 2^(K/2) * ||U||
            int se = 260 - (int)((__float_as_uint(amax) >> 23) & 0xffu);
            se = min(max(se, 1), 253);
            const float scale = __uint_as_float((uint32_t)se << 23);
            const float inv = __uint_as_float((uint32_t)(254 - se) << 23);
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                float2(&w)[16] = v[KEEP == 1 ? 0 : ch];
                if (KEEP == 1) load16(cbase + 16 * ch, w);
                uint32_t hi[16], lo[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) split2(w[c].x * scale, w[c].y * scale, hi[c], lo[c]);
                tmem_st16(tA + (uint32_t)(cbase + 16 * ch), hi);
                tmem_st16(tA + (uint32_t)(CFG + cbase + 16 * ch), lo);
            }
            GS_PROG(3);
            tc::tmem_wait_st();
            GS_PROG(4);
            tc::fence_before();
            bar_wg<C::WGT>(wg);  // A complete; every read of the tile done
            GS_PROG(5);
            if (wtid == 0) {
                tc::fence_after();
                constexpr uint32_t idesc = tc::idesc_f16_m128(C::N);
                const uint32_t d = tmem + (uint32_t)wg * C::COLS;
                const uint32_t ah = d + (uint32_t)C::N, al = ah + (uint32_t)CFG;
                const uint32_t wb = sm_s + C::W_OFF;
                auto bdesc = [&](int step) {
                    return tc::smem_desc_sw128(wb + (uint32_t)(step >> 2) * (uint32_t)(C::N * 128) +
                                               (uint32_t)(step & 3) * 32u);
                };
#pragma unroll
                for (int k = 0; k < C::KS; ++k) mma(d, ah + 8u * k, bdesc(k), idesc, k > 0 ? 1u : 0u);
#pragma unroll
                for (int k = 0; k < C::KS; ++k) mma(d, al + 8u * k, bdesc(k), idesc, 1u);
#pragma unroll
                for (int k = 0; k < C::KS; ++k) mma(d, ah + 8u * k, bdesc(C::KS + k), idesc, 1u);
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                 bar + 8u * (2 * C::STAGES + wg))
                             : "memory");
            }
            GS_PROG(6);
            wait(bar + 8u * (2 * C::STAGES + wg), mma_phase);
            __syncwarp();
            GS_PROG(7);
            mma_phase ^= 1u;
            tc::fence_after();
            // ---- D row -> amplitudes (unscaled) -> tile, in place ----
#pragma unroll
            for (int cc = 0; cc < CPT; cc += 16) {
                const int c0 = cbase + cc;
                uint32_t d[32];
                tc::tmem_ld32(tl + 2u * (uint32_t)c0, d);
                tc::tmem_wait_ld();
                if (pair) {
#pragma unroll
                    for (int c = 0; c < 16; c += 2) {
                        const float4 f = make_float4(__uint_as_float(d[2 * c]) * inv, __uint_as_float(d[2 * c + 1]) * inv,
                                                     __uint_as_float(d[2 * c + 2]) * inv,
                                                     __uint_as_float(d[2 * c + 3]) * inv);
                        *reinterpret_cast<float4*>(tile + (ro ^ cfg_off(c0 + c))) = f;
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        *reinterpret_cast<float2*>(tile + (ro ^ cfg_off(c0 + c))) =
                            make_float2(__uint_as_float(d[2 * c]) * inv, __uint_as_float(d[2 * c + 1]) * inv);
                }
            }
            }  // rep
            tc::fence_before();
            tc::fence_proxy_async();  // generic writes -> the TMA store (async proxy)
            arrive(bar + 8u * (C::STAGES + s));
            GS_PROG(8);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, C::TCOLS);
    }
}

// ---------------------------------------------------------------- host

using cd = std::complex<double>;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

static inline uint32_t swz(uint32_t x) { return x ^ (((x >> 7) & 7u) << 4); }

// shared-memory wavefronts of one warp-wide access (8- or 16-byte per lane) at the
// given lane byte offsets (bank = 4-byte word mod 32; phases of 16 / 8 lanes)
static int wavefronts(const uint32_t* off, int bytes) {
    const int per = bytes == 16 ? 8 : 16;
    int total = 0;
    for (int p0 = 0; p0 < 32; p0 += per) {
        int worst = 0;
        for (int b = 0; b < 32; ++b) {
            uint32_t words[32];
            int nw = 0;
            for (int l = p0; l < p0 + per; ++l)
                for (int w = 0; w < bytes / 4; ++w) {
                    const uint32_t word = off[l] / 4 + (uint32_t)w;
                    if ((int)(word % 32) != b) continue;
                    bool seen = false;
                    for (int i = 0; i < nw; ++i) seen |= words[i] == word;
                    if (!seen) words[nw++] = word;
                }
            worst = std::max(worst, nw);
        }
        total += worst;
    }
    return total;
}

struct GsPlan {
    int K = 0;
    GsArgs a{};
    CUtensorMap tm{};
    std::vector<uint16_t> w;  // W operand image (SW128 K-major f16)
};

static void f16_split(double x, uint16_t& hi, uint16_t& lo) {
    const __half h = __double2half(x);
    const double r = x - (double)__half2float(h);
    const __half l = __double2half(r);
    std::memcpy(&hi, &h, 2);
    std::memcpy(&lo, &l, 2);
}

// Plan one gate (qubits sorted ascending, U in the internal order: matrix bit m <->
// m-th lowest qubit, row-major 2^nq x 2^nq).  false if the register is too small
// (n < 7 + K) or the tensor map cannot be encoded.
static bool plan_gate(void* state, int n, int nq, const int* qs, const cd* U, GsPlan& P) {
    // k <= 4 gates run padded to 5 qubits when the register allows: the 32 KB tiles of the
    // K = 5 kernel stream at 0.94 - 0.96 of HBM for every placement, the 16 KB K = 4 tiles at
    // 0.86 - 0.94 (twice the boxes and barrier round trips per byte)
    const int K = std::max(nq, n >= 12 ? 5 : 4);
    if (n < 7 + K) return false;
    P.K = K;
    // matrix qubits: the gate's plus the lowest free ones as padding
    uint64_t gmask = 0;
    for (int i = 0; i < nq; ++i) gmask |= 1ull << qs[i];
    uint64_t mmask = gmask;
    for (int q = 0; __builtin_popcountll(mmask) < K; ++q) mmask |= 1ull << q;
    int mq[6], nm = 0;
    for (int q = 0; q < n; ++q)
        if ((mmask >> q) & 1) mq[nm++] = q;
    // low run: 7 non-matrix qubits below L
    int L = 7;
    while (L - __builtin_popcountll(mmask & ((1ull << L) - 1ull)) < 7) ++L;
    std::vector<int> high, rowq;
    for (int m = 0; m < K; ++m)
        if (mq[m] >= L) high.push_back(mq[m]);
    for (int q = 0; q < L; ++q)
        if (!((mmask >> q) & 1)) rowq.push_back(q);
    const int T = L + (int)high.size();
    if (T != 7 + K || n < T || n - L > 31) return false;
    GsArgs& a = P.a;
    a.L = L;
    a.tile_mask = ((1ull << L) - 1ull);
    for (int h : high) a.tile_mask |= 1ull << h;
    a.ntiles = (uint32_t)(1ull << (n - T));
    a.pair = (mmask & 1ull) != 0;  // qubit 0 (tile bit 0) is matrix bit 0
    a.reps = getenv("QT_GS_REPS") ? std::max(1, atoi(getenv("QT_GS_REPS"))) : 1;
    // Tile layout in shared memory = the TMA box's dimension order: qubits 0..3 (128-byte
    // rows), then the middle dimensions (runs of consecutive qubits, <= 8 qubits each, at
    // most three), then the boxes of the remaining high matrix qubits.  "natural" keeps the
    // low run in qubit order; "rows first" puts the runs of row qubits right after qubits
    // 0..3 so that they land on the swizzled bank bits (matrix qubits 4, 5, ... otherwise
    // push the row qubits above them and every lane of a quarter-warp hits the same bank
    // group).  The layout with fewer modelled wavefronts wins.
    struct Layout {
        std::vector<std::pair<int, int>> segs;  // middle dims (first qubit, length)
        std::vector<int> ops;                   // high matrix qubits enumerated by boxes
        int pos[64];
        int perm[7];
        int wf = 1 << 30;
        bool ok = false;
    };
    auto build = [&](bool rows_first, Layout& Lo) {
        std::vector<std::pair<int, int>> low;  // runs of qubits 4..L-1 (row runs first if asked)
        for (int pass = 0; pass < (rows_first ? 2 : 1); ++pass)
            for (int q = 4; q < L;) {
                const bool isrow = !((mmask >> q) & 1);
                int e = q + 1;
                while (e < L && (rows_first ? (!((mmask >> e) & 1)) == isrow : true)) ++e;
                if (!rows_first || isrow == (pass == 0)) low.push_back({q, e - q});
                q = e;
            }
        for (auto& r : low)
            for (int q = r.first; q < r.first + r.second; q += 8) Lo.segs.push_back({q, std::min(8, r.first + r.second - q)});
        if (Lo.segs.size() > 3) return;
        size_t hi = 0;
        while (Lo.segs.size() < 3 && hi < high.size()) Lo.segs.push_back({high[hi++], 1});
        for (; hi < high.size(); ++hi) Lo.ops.push_back(high[hi]);
        int p = 0;
        for (int q = 0; q < 4; ++q) Lo.pos[q] = p++;
        for (auto& sg : Lo.segs)
            for (int q = sg.first; q < sg.first + sg.second; ++q) Lo.pos[q] = p++;
        for (int q : Lo.ops) Lo.pos[q] = p++;
        // lane bits: the ordering of the 7 row qubits with the fewest modelled wavefronts
        int perm[7] = {0, 1, 2, 3, 4, 5, 6};
        do {
            uint32_t off[32];
            for (int l = 0; l < 32; ++l) {
                uint32_t o = 0;
                for (int j = 0; j < 5; ++j)
                    if ((l >> j) & 1) o ^= swz(8u << Lo.pos[rowq[perm[j]]]);
                off[l] = o;
            }
            const int w = wavefronts(off, a.pair ? 16 : 8);
            if (w < Lo.wf) {
                Lo.wf = w;
                std::copy(perm, perm + 7, Lo.perm);
            }
        } while (std::next_permutation(perm, perm + 7));
        Lo.ok = true;
    };
    Layout nat, rf;
    build(false, nat);
    build(true, rf);
    const Layout& Lo = (rf.ok && (!nat.ok || rf.wf < nat.wf)) ? rf : nat;
    if (!Lo.ok) return false;
    for (int m = 0; m < K; ++m) a.cfg_basis[m] = swz(8u << Lo.pos[mq[m]]);
    for (int j = 0; j < 7; ++j) a.row_basis[j] = swz(8u << Lo.pos[rowq[Lo.perm[j]]]);
    // tensor map: [0..3] [middle dims] (size-1 fillers) [rest]
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    int nd = 0;
    dims[nd] = 16;
    box[nd++] = 16;
    for (auto& sg : Lo.segs) {
        dims[nd] = 1ull << sg.second;
        strides[nd - 1] = 8ull << sg.first;
        box[nd++] = 1u << sg.second;
    }
    while (nd < 4) {
        dims[nd] = 1;
        strides[nd - 1] = 8ull << L;
        box[nd++] = 1;
    }
    dims[4] = 1ull << (n - L);
    strides[3] = 8ull << L;
    box[4] = 1;
    const int extra = (int)Lo.ops.size();
    a.nops = 1 << extra;
    a.op_bytes = (uint32_t)((128u << K) * 8u) >> extra;
    for (int o = 0; o < a.nops; ++o) {
        int32_t r = 0;
        for (int i = 0; i < extra; ++i)
            if ((o >> i) & 1) r += (int32_t)(1u << (Lo.ops[i] - L));
        a.op_rest[o] = r;
    }
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    if (enc(&P.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, state, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    // padded matrix in matrix-bit order and the W operand image:
    // W[2r + b][part * 2 CFG + 2c + a] = real 2 x 2 block of Up[r][c] (input a, output b)
    const int CFGn = 1 << K, N = 2 * CFGn, KT = 4 * CFGn;
    int gpos[6], npg = 0, ppos[6], npp = 0;
    for (int m = 0; m < K; ++m) {
        if ((gmask >> mq[m]) & 1) gpos[npg++] = m;
        else ppos[npp++] = m;
    }
    const int dq = 1 << nq;
    P.w.assign((size_t)N * KT, 0);
    for (int r = 0; r < CFGn; ++r)
        for (int c = 0; c < CFGn; ++c) {
            bool same = true;
            for (int i = 0; i < npp; ++i) same &= ((r >> ppos[i]) & 1) == ((c >> ppos[i]) & 1);
            cd u = 0;
            if (same) {
                int gr = 0, gc = 0;
                for (int i = 0; i < npg; ++i) {
                    gr |= ((r >> gpos[i]) & 1) << i;
                    gc |= ((c >> gpos[i]) & 1) << i;
                }
                u = U[(size_t)gr * dq + gc];
            }
            const double blk[2][2] = {{u.real(), -u.imag()}, {u.imag(), u.real()}};  // [b][a]
            for (int b = 0; b < 2; ++b)
                for (int ain = 0; ain < 2; ++ain) {
                    uint16_t hi, lo;
                    f16_split(blk[b][ain], hi, lo);
                    const int row = 2 * r + b;
                    for (int part = 0; part < 2; ++part) {
                        const int kk = part * 2 * CFGn + 2 * c + ain;
                        const int atom = kk >> 6, wi = kk & 63;
                        const size_t byte = (size_t)atom * N * 128 + (row >> 3) * 1024 + (row & 7) * 128 +
                                            ((((wi * 2) >> 4) ^ (row & 7)) << 4) + ((wi * 2) & 15);
                        P.w[byte / 2] = part ? lo : hi;
                    }
                }
        }
    return true;
}

template <int K>
static cudaError_t launch_k(const GsPlan& P, const void* w_dev, cudaStream_t s) {
    using C = Cfg<K>;
    // kernel attribute and SM count per device (contexts may live on different GPUs)
    static int sms_of[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    int& sms = sms_of[dev];
    if (!sms) {
        cudaError_t e = cudaFuncSetAttribute(gate_stream_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)C::SMEM);
        if (e != cudaSuccess) return e;
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        sms = n;
    }
    uint32_t grid = std::min<uint32_t>(P.a.ntiles, (uint32_t)sms);
    if (const char* g = getenv("QT_GS_GRID")) grid = std::min<uint32_t>(grid, (uint32_t)std::max(1, atoi(g)));
    gate_stream_kernel<K><<<grid, C::THREADS, C::SMEM, s>>>(P.tm, P.a, w_dev);
    return cudaGetLastError();
}

}  // namespace gs

// One gate applied `repeats` times in place by the streaming kernel.  Returns
// cudaErrorNotSupported when the register is too small for its tiles (the caller
// uses the trajectory kernels instead).  kernel_ms: mean time of one application
// (first one excluded when repeats > 1).
cudaError_t gate_stream_apply(cudaStream_t s, void* state, int n, int nq, const int* qs, const std::complex<double>* U,
                              int repeats, double* kernel_ms) {
    gs::GsPlan P;
    if (!gs::plan_gate(state, n, nq, qs, U, P)) return cudaErrorNotSupported;
    // the W operand lives in a stream-ordered allocation of this call (no state shared
    // between contexts, devices or threads)
    void* w_dev = nullptr;
    cudaError_t e = cudaMallocAsync(&w_dev, P.w.size() * 2, s);
    if (e != cudaSuccess) return e;
    struct Free {
        void* p;
        cudaStream_t s;
        ~Free() { cudaFreeAsync(p, s); }
    } w_free{w_dev, s};
    e = cudaMemcpyAsync(w_dev, P.w.data(), P.w.size() * 2, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // P.w is a local
    if (e != cudaSuccess) return e;
    auto one = [&]() {
        switch (P.K) {
            case 4: return gs::launch_k<4>(P, w_dev, s);
            case 5: return gs::launch_k<5>(P, w_dev, s);
            default: return gs::launch_k<6>(P, w_dev, s);
        }
    };
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (kernel_ms) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
    }
    int timed = repeats;
    if (repeats > 1) {
        if ((e = one()) != cudaSuccess) return e;
        timed = repeats - 1;
    }
    if (kernel_ms) cudaEventRecord(e0, s);
    for (int r = 0; r < timed; ++r)
        if ((e = one()) != cudaSuccess) return e;
    if (kernel_ms) {
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        *kernel_ms = timed > 0 ? ms / timed : 0.0;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    return cudaGetLastError();
}

}  // namespace qt
