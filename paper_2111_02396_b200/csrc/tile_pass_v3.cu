// tile_pass_v3.cu -- K1 on 11-qubit tiles moved by TMA (Alg. 1, every fused gate
// of a pass per HBM sweep; Alg. 2 epilogues): the pipeline of the streaming single-gate
// kernel (gate_stream.cu) applied to trajectory passes.  Selected by tile_bits = 11
// (qt_fuse_opts); experimental: parity-green, but slower than the persistent TMEM kernel on
// C2 (17.1 passes of 11-qubit tiles instead of 12.5 of 13-qubit tiles,
// and a shared-memory gather per gate instead of in-TMEM transitions).
//
// One persistent CTA per SM walks the step's (trajectory, tile) items:
//   loader thread   TMA box loads of item j into stage j % 8 (a tensor map per tile layout
//                   of the batch, over the whole batch buffer), or a bare arrive for a
//                   trajectory's first pass (the tile is built as |0...0> in place);
//   storer thread   TMA box stores of computed items of storing passes, in order, and the
//                   stage's release once the store has read it;
//   4 warpgroups    item j on warpgroup j % 4 (a stage always on the same warpgroup, so its
//                   barriers are waited on in phase order).  A tile is 2^11 amplitudes =
//                   128 rows x 16 configurations of a fused 4-qubit gate: a thread owns a
//                   row (TMEM lane), gathers its 16 amplitudes, scales them by a power of two
//                   from the row's own max, splits them into f16 hi / lo into TMEM; one thread
//                   issues 6 TS tcgen05.mma M128 N32 K16 (D = x_hi W_hi + x_lo W_hi + x_hi W_lo,
//                   W = the persistent kernel's 4 KB operand, bulk-copied one gate ahead); the
//                   row is read back, unscaled and written in place.  Device-chosen operators
//                   (CUDA cores, 16 amplitudes per thread) and the epilogues (rho_Q partials +
//                   the last tile's Alg. 2 choice, block sums, Pauli-string partials) follow.
// Shared-memory tile = the TMA box image with SWIZZLE_128B: byte offset x of amplitude L
// (x = 8 L) lives at x ^ (((x >> 7) & 7) << 4).
#include <cuda.h>
#include <cuda_fp16.h>

#include "tile_pass.cuh"

namespace qt {
namespace v3 {

constexpr int T = 11;
constexpr int TILE = 1 << T;
constexpr uint32_t kTileBytes = TILE * 8;  // 16 KB
constexpr int NWG = 4, NT = 128, NA = TILE / NT;  // 16 amplitudes per thread
constexpr int STAGES = 8;
static_assert(STAGES % NWG == 0, "stage -> warpgroup map");
constexpr uint32_t kWOff = STAGES * kTileBytes;
constexpr uint32_t kRedOff = kWOff + NWG * 2 * kV2GateBytes;
constexpr uint32_t kBarOff = kRedOff + NWG * 256 * 8;
// full[S], computed[S], empty[S], mma[NWG], wfull[NWG][2]
constexpr int kNBar = 3 * STAGES + NWG + 2 * NWG;
constexpr uint32_t kMiscOff = kBarOff + kNBar * 8;
constexpr size_t kSmemBytes = kMiscOff + 64 + 1024;
constexpr int kThreads = NWG * NT + 64;
constexpr uint32_t kTCols = 256;

__device__ __forceinline__ uint32_t swzb(uint32_t L) {  // amplitude index -> swizzled byte offset
    const uint32_t x = L << 3;
    return x ^ (((x >> 7) & 7u) << 4);
}
__device__ __forceinline__ bool try_wait(uint32_t a, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok) : "r"(a), "r"(phase), "r"(1000000u) : "memory");  // suspend (not spin) up to 1 ms
    return ok != 0;
}
__device__ __forceinline__ void wait(uint32_t a, uint32_t phase) {
    while (!try_wait(a, phase)) {
    }
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
#ifdef QT_V3_TIMING
#define V3T(k, t0)                                                                  \
    if (blockIdx.x == 7) {                                                          \
        const long long t1_ = clock64();                                            \
        atomicAdd(A.timing + (k), (unsigned long long)(t1_ - (t0)));                \
        t0 = t1_;                                                                   \
    }
#else
#define V3T(k, t0)
#endif
__device__ __forceinline__ void pf_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];\n" ::"l"(p)); }
__device__ __forceinline__ void bar_wg(int wg) { asm volatile("bar.sync %0, 128;\n" ::"r"(1 + wg) : "memory"); }
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
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
    const float hx = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    const float hy = __uint_as_float(__float_as_uint(y) & 0xFFFFE000u);
    const __half2 h2 = __floats2half2_rn(hx, hy);
    const __half2 l2 = __floats2half2_rn(x - hx, y - hy);
    hi = *reinterpret_cast<const uint32_t*>(&h2);
    lo = *reinterpret_cast<const uint32_t*>(&l2);
}

// Deterministic warpgroup sums (lanes by xor tree, then warps 0..3 in order).
template <int N>
__device__ __forceinline__ void wg_sum(double (&v)[N], double* red, int wg) {
    static_assert(N <= 32, "red holds 4 x 32 doubles");
    const int wtid = threadIdx.x & (NT - 1);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    bar_wg(wg);  // earlier readers of red are done
    if ((wtid & 31) == 0)
#pragma unroll
        for (int i = 0; i < N; ++i) red[(wtid >> 5) * N + i] = v[i];
    bar_wg(wg);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = red[i] + red[N + i] + red[2 * N + i] + red[3 * N + i];
}

// global amplitude index (within the slot) of the tile's amplitude 0
__device__ __forceinline__ uint64_t tile_base(const PassDesc& P, uint32_t tile) {
    uint64_t base = tile;
#pragma unroll
    for (int i = 0; i < T; ++i) {
        const uint64_t low = base & ((1ull << P.tq[i]) - 1ull);
        base = low | ((base ^ low) << 1);
    }
    return base;
}

// rho_Q partial (Q <= 2) of the tile: the upper triangle, D real diagonal entries then
// (re, im) of (a, b), a < b, summed over the complement indices in a fixed order
template <int Q>
__device__ __forceinline__ void rho_partial(const unsigned char* tile, uint32_t ql, double* out, double* red, int wg) {
    constexpr int D = 1 << Q;
    constexpr int NE = D * D;
    const int wtid = threadIdx.x & (NT - 1);
    uint32_t qoff[D];
#pragma unroll
    for (int a = 0; a < D; ++a) qoff[a] = pdep32((uint32_t)a, ql);
    uint32_t qp[Q];
    {
        uint32_t m = ql;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            qp[q] = (uint32_t)__ffs(m) - 1u;
            m &= m - 1u;
        }
    }
    double acc[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] = 0.0;
#pragma unroll
    for (uint32_t k = wtid; k < (uint32_t)(TILE >> Q); k += NT) {
        uint32_t bL = k;
#pragma unroll
        for (int q = 0; q < Q; ++q) bL = (bL & ((1u << qp[q]) - 1u)) | ((bL >> qp[q]) << (qp[q] + 1u));
        double vr[D], vi[D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const float2 v = *reinterpret_cast<const float2*>(tile + swzb(bL | qoff[a]));
            vr[a] = v.x;
            vi[a] = v.y;
        }
        int e = 0;
#pragma unroll
        for (int a = 0; a < D; ++a) acc[e++] += vr[a] * vr[a] + vi[a] * vi[a];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = a + 1; b < D; ++b) {
                acc[e++] += vr[a] * vr[b] + vi[a] * vi[b];
                acc[e++] += vi[a] * vr[b] - vr[a] * vi[b];
            }
    }
    wg_sum<NE>(acc, red, wg);
    if (wtid == 0) {
        int e = 0;
        for (int a = 0; a < D; ++a) {
            out[2 * (a * D + a)] = acc[e++];
            out[2 * (a * D + a) + 1] = 0.0;
        }
        for (int a = 0; a < D; ++a)
            for (int b = a + 1; b < D; ++b) {
                const double re = acc[e++], im = acc[e++];
                out[2 * (a * D + b)] = re;
                out[2 * (a * D + b) + 1] = im;
                out[2 * (b * D + a)] = re;
                out[2 * (b * D + a) + 1] = -im;
            }
    }
}
// 3-qubit channels: one row of rho_Q (16 doubles) at a time
__device__ __forceinline__ void rho_partial_rows3(const unsigned char* tile, uint32_t ql, double* out, double* red,
                                                  int wg) {
    constexpr int D = 8;
    const int wtid = threadIdx.x & (NT - 1);
    uint32_t qoff[D];
#pragma unroll
    for (int a = 0; a < D; ++a) qoff[a] = pdep32((uint32_t)a, ql);
#pragma unroll 1
    for (int a = 0; a < D; ++a) {
        double acc[2 * D];
#pragma unroll
        for (int e = 0; e < 2 * D; ++e) acc[e] = 0.0;
        for (uint32_t bL = wtid; bL < (uint32_t)TILE; bL += NT) {
            if (bL & ql) continue;
            const float2 va = *reinterpret_cast<const float2*>(tile + swzb(bL | qoff[a]));
            const double ar = va.x, ai = va.y;
#pragma unroll
            for (int b = 0; b < D; ++b) {
                const float2 vb = *reinterpret_cast<const float2*>(tile + swzb(bL | qoff[b]));
                acc[2 * b] += ar * (double)vb.x + ai * (double)vb.y;
                acc[2 * b + 1] += ai * (double)vb.x - ar * (double)vb.y;
            }
        }
        wg_sum<2 * D>(acc, red, wg);
        if (wtid == 0)
#pragma unroll
            for (int e = 0; e < 2 * D; ++e) out[2 * D * a + e] = acc[e];
    }
}

// warp reduce-scatter of NE values (NE a power of two <= 32): lane l ends with the warp sum
// of value l >> (5 - log2 NE) (fixed order)
template <int NE>
__device__ __forceinline__ double warp_reduce_scatter(double (&v)[NE], int lane) {
    int o = 16;
#pragma unroll
    for (int h = NE / 2; h >= 1; h >>= 1, o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? v[i] : v[i + h];
            const double keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    double r = v[0];
#pragma unroll
    for (; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    return r;
}

__global__ void __launch_bounds__(kThreads, 1)
    tile_pass_v3_kernel(const TileArgs A, const V3Map* __restrict__ maps, const uint32_t nitems, const int tshift) {
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw_s = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t pad = ((raw_s + 1023u) & ~1023u) - raw_s;
    unsigned char* sm = smem_raw + pad;
    const uint32_t sm_s = raw_s + pad;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t bar = sm_s + kBarOff;
    auto full_b = [&](int s) { return bar + 8u * (uint32_t)s; };
    auto comp_b = [&](int s) { return bar + 8u * (uint32_t)(STAGES + s); };
    auto empty_b = [&](int s) { return bar + 8u * (uint32_t)(2 * STAGES + s); };
    auto mma_b = [&](int w) { return bar + 8u * (uint32_t)(3 * STAGES + w); };
    auto wfull_b = [&](int w, int i) { return bar + 8u * (uint32_t)(3 * STAGES + NWG + 2 * w + i); };
    uint32_t* misc = reinterpret_cast<uint32_t*>(sm + kMiscOff);  // [0] tmem base, [1..4] last flags
    if (warp == 0) tc::tmem_alloc(misc, kTCols);
    if (tid == NWG * NT) {
        for (int s = 0; s < STAGES; ++s) {
            bar_init(full_b(s), 1);
            bar_init(comp_b(s), NT);
            bar_init(empty_b(s), 1);
        }
        for (int w = 0; w < NWG; ++w) {
            bar_init(mma_b(w), 1);
            bar_init(wfull_b(w, 0), 1);
            bar_init(wfull_b(w, 1), 1);
        }
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = misc[0];
    const int n = A.n;
    const uint32_t ntiles = 1u << tshift;
    const uint32_t G = gridDim.x;
    const uint32_t my_items = blockIdx.x < nitems ? (nitems - 1u - blockIdx.x) / G + 1u : 0u;
    auto raw = [&](uint32_t j) { return blockIdx.x + j * G; };
    // rest coordinate (units of 16 amplitudes over the batch buffer) of an item's tile
    auto crest_of = [&](const PassDesc& P, uint32_t tile) {
        return (int32_t)((((uint64_t)P.slot << n) + tile_base(P, tile)) >> 4);
    };

    if (warp == NWG * 4) {
        // ---------------- loader ----------------
        // the whole warp: lane 0 waits for the stage and posts the expected bytes, lane o
        // issues box o (a tile of scattered qubits takes up to 16 boxes)
        for (uint32_t j = 0; j < my_items; ++j) {
            const int s = (int)(j % STAGES);
            if (lane == 0 && j + 4 < my_items) pf_l1(A.step_passes + (raw(j + 4) >> tshift));  // descriptors ahead
#ifdef QT_V3_TIMING
            long long tt = clock64();
#endif
            if (j >= (uint32_t)STAGES) wait(empty_b(s), ((j / STAGES) - 1u) & 1u);
            __syncwarp();
            if (lane == 0) { V3T(10, tt); }
            const uint32_t i = raw(j);
            const PassDesc P = A.step_passes[i >> tshift];
            if (P.flags & kPassInit) {
                if (lane == 0) arrive(full_b(s));  // the warpgroup builds |0...0> in place
                continue;
            }
            const V3Map* M = maps + P.pad;
            if (lane == 0) expect_tx(full_b(s), kTileBytes);
            __syncwarp();
            const int32_t cr = crest_of(P, i & (ntiles - 1u));
            const uint32_t st = sm_s + (uint32_t)s * kTileBytes;
            const int nops = M->nops;
            if (lane < nops) tma_load(st + (uint32_t)lane * M->op_bytes, &M->tm, cr + M->op_rest[lane], full_b(s));
            if (lane == 0) { V3T(11, tt); }
        }
    } else if (warp == NWG * 4 + 1) {
        // ---------------- storer ----------------
        // stores of storing passes, in order; up to kLag store groups stay in flight (a
        // stage is released once its store has read it), read-only items release at once
        if (lane == 0) {
            constexpr int kLag = 3;
            int pend[kLag + 1], np = 0;
            for (uint32_t j = 0; j < my_items; ++j) {
                const int s = (int)(j % STAGES);
                if (j + 4 < my_items) pf_l1(A.step_passes + (raw(j + 4) >> tshift));
#ifdef QT_V3_TIMING
                long long tt = clock64();
#endif
                wait(comp_b(s), (j / STAGES) & 1u);
                V3T(12, tt);
                const uint32_t i = raw(j);
                const PassDesc P = A.step_passes[i >> tshift];
                if (P.flags & (kPassStore | kPassInit)) {
                    const V3Map* M = maps + P.pad;
                    const int32_t cr = crest_of(P, i & (ntiles - 1u));
                    const uint32_t st = sm_s + (uint32_t)s * kTileBytes;
                    for (int o = 0; o < M->nops; ++o) tma_store(&M->tm, cr + M->op_rest[o], st + (uint32_t)o * M->op_bytes);
                    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                    pend[np++] = s;
                    if (np > kLag) {
                        asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(kLag) : "memory");
                        arrive(empty_b(pend[0]));
                        for (int k = 1; k < np; ++k) pend[k - 1] = pend[k];
                        --np;
                    }
                    V3T(13, tt);
                } else {
                    // a read-only item: flush the pending stages too (the loader may be waiting
                    // for one of them, and no later store may come to push it out)
                    if (np) {
                        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                        for (int k = 0; k < np; ++k) arrive(empty_b(pend[k]));
                        np = 0;
                    }
                    arrive(empty_b(s));
                }
            }
            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            for (int k = 0; k < np; ++k) arrive(empty_b(pend[k]));
            asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
        }
    } else {
        // ---------------- compute warpgroups ----------------
        const int wg = warp >> 2, wq = warp & 3;
        const int wtid = tid & (NT - 1);
        const uint32_t tl = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)wg * 64u;  // lane, D column 0
        const uint32_t tA = tl + 32u;                                                 // A: hi, then lo
        double* red = reinterpret_cast<double*>(sm + kRedOff) + 256 * wg;  // [0..127] sums, [128..255] rho_Q
        const uint32_t wbuf = sm_s + kWOff + (uint32_t)wg * 2u * kV2GateBytes;
        uint32_t mma_phase = 0, w_issued = 0, w_used = 0;
        // W operands: a cursor over this warpgroup's items and their tensor-core gates;
        // each call issues the next operand (one 4 KB bulk copy), at most one gate ahead
        // of the MMAs, across item boundaries (the first gate of the next item is in flight
        // while the current item's epilogues run)
        uint32_t wj = (uint32_t)wg;
        int wn = 0, wgb = 0, wgc = -1;
        auto issue_next_w = [&]() {
            while (wj < my_items) {
                if (wgc < 0) {
                    const PassDesc* PW = A.step_passes + (raw(wj) >> tshift);
                    wgb = __ldg(&PW->gate_begin);
                    wgc = __ldg(&PW->gate_count);
                }
                const GateDesc* gl = A.gates + wgb;
                while (wn < wgc && !(__ldg(&gl[wn].k) & kGateTC)) ++wn;
                if (wn < wgc) {
                    if (wtid == 0) {
                        const uint32_t wb = wbuf + (w_issued & 1u) * kV2GateBytes, mb = wfull_b(wg, (int)(w_issued & 1u));
                        expect_tx(mb, kV2GateBytes);
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                                wb),
                            "l"(A.pool + __ldg(&gl[wn].mat_off)), "r"((uint32_t)kV2GateBytes), "r"(mb)
                            : "memory");
                    }
                    ++w_issued;
                    ++wn;
                    return;
                }
                wj += NWG;
                wn = 0;
                wgc = -1;
            }
        };
        issue_next_w();
        if (wtid == 0 && (uint32_t)wg + NWG < my_items) pf_l1(A.step_passes + (raw((uint32_t)wg + NWG) >> tshift));
        for (uint32_t j = (uint32_t)wg; j < my_items; j += NWG) {
            const int s = (int)(j % STAGES);
            const uint32_t i = raw(j);
            // L1 prefetch: the pass descriptor two items ahead, the gate descriptors of the next
            // item (its pass descriptor was prefetched one item ago)
            if (wtid < 32 && j + NWG < my_items) {
                if (lane == 0 && j + 2 * NWG < my_items) pf_l1(A.step_passes + (raw(j + 2 * NWG) >> tshift));
                const PassDesc* PN = A.step_passes + (raw(j + NWG) >> tshift);
                const int nb = (__ldg(&PN->gate_count) * (int)sizeof(GateDesc) + 127) / 128;
                const char* g0 = reinterpret_cast<const char*>(A.gates + __ldg(&PN->gate_begin));
                for (int k = lane; k <= nb; k += 32) pf_l1(g0 + 128 * k);
            }
            const PassDesc P = A.step_passes[i >> tshift];
            const uint32_t tile_idx = i & (ntiles - 1u);
            const int slot = P.slot;
            const uint64_t base = tile_base(P, tile_idx);
            const GateDesc* gds = A.gates + P.gate_begin;
            const int ng = P.gate_count;
#ifdef QT_V3_TIMING
            long long tt = clock64();
            const bool tme = wtid == 0;
#define V3C(k) if (tme) { V3T(k, tt); }
#else
#define V3C(k)
#endif
            V3C(9);
            wait(full_b(s), (j / STAGES) & 1u);
            __syncwarp();
            V3C(0);
            unsigned char* tile = sm + (size_t)s * kTileBytes;
            if (P.flags & kPassInit) {
                // |0...0>: amplitude 0 of the slot lives in tile 0 at tile index 0
                float4* t4 = reinterpret_cast<float4*>(tile);
                for (int k = wtid; k < TILE / 2; k += NT)
                    t4[k] = make_float4((k == 0 && tile_idx == 0) ? 1.f : 0.f, 0.f, 0.f, 0.f);
                bar_wg(wg);
            }
            for (int g = 0; g < ng; ++g) {
                const GateDesc Gd = gds[g];
                if (Gd.k & kGateTC) {
                    issue_next_w();  // the next tensor-core operand (its buffer's MMAs are done)
                    // matrix bits rpos[0..3], row bits tpos[0..6] (lanes 0..4, warps 5..6)
                    // swizzled byte offsets (planner, v3_lanes): xu[0..3] matrix bits, xu[4..10] row bits
                    uint32_t ro = 0;
                    const int r = lane | (wq << 5);
#pragma unroll
                    for (int b = 0; b < 7; ++b)
                        if ((r >> b) & 1) ro ^= Gd.xu[4 + b];
                    uint32_t cb[4];
#pragma unroll
                    for (int m = 0; m < 4; ++m) cb[m] = Gd.xu[m];
                    auto cfg_off = [&](int c) {
                        uint32_t o = 0;
#pragma unroll
                        for (int m = 0; m < 4; ++m)
                            if ((c >> m) & 1) o ^= cb[m];
                        return o;
                    };
                    const bool pair = (Gd.rpos & 15u) == 0u;
                    float2 v[16];
                    if (pair) {
#pragma unroll
                        for (int c = 0; c < 16; c += 2) {
                            const float4 f = *reinterpret_cast<const float4*>(tile + (ro ^ cfg_off(c)));
                            v[c] = make_float2(f.x, f.y);
                            v[c + 1] = make_float2(f.z, f.w);
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < 16; ++c) v[c] = *reinterpret_cast<const float2*>(tile + (ro ^ cfg_off(c)));
                    }
                    float amax = 0.f;
#pragma unroll
                    for (int c = 0; c < 16; ++c) amax = fmaxf(amax, fmaxf(fabsf(v[c].x), fabsf(v[c].y)));
                    int se = 260 - (int)((__float_as_uint(amax) >> 23) & 0xffu);
                    se = min(max(se, 1), 253);
                    const float scale = __uint_as_float((uint32_t)se << 23);
                    const float inv = __uint_as_float((uint32_t)(254 - se) << 23);
                    {
                        uint32_t hi[16], lo[16];
#pragma unroll
                        for (int c = 0; c < 16; ++c) split2(v[c].x * scale, v[c].y * scale, hi[c], lo[c]);
                        tmem_st16(tA, hi);
                        tmem_st16(tA + 16u, lo);
                    }
                    tc::tmem_wait_st();
                    tc::fence_before();
                    bar_wg(wg);  // A complete; every read of the tile for this gate done
                    V3C(1);
                    if (wtid == 0) {
                        wait(wfull_b(wg, (int)(w_used & 1u)), (w_used >> 1) & 1u);
                        tc::fence_after();
                        constexpr uint32_t idesc = tc::idesc_f16_m128(32);
                        const uint32_t d = tmem + (uint32_t)wg * 64u;
                        const uint32_t ah = d + 32u, al = ah + 16u;
                        const uint32_t wb = wbuf + (w_used & 1u) * kV2GateBytes;
#pragma unroll
                        for (int k = 0; k < 2; ++k) mma(d, ah + 8u * k, tc::smem_desc_sw128(wb + 32u * k), idesc, k > 0 ? 1u : 0u);
#pragma unroll
                        for (int k = 0; k < 2; ++k) mma(d, al + 8u * k, tc::smem_desc_sw128(wb + 32u * k), idesc, 1u);
#pragma unroll
                        for (int k = 0; k < 2; ++k) mma(d, ah + 8u * k, tc::smem_desc_sw128(wb + 64u + 32u * k), idesc, 1u);
                        asm volatile(
                            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mma_b(wg))
                            : "memory");
                    }
                    ++w_used;
                    wait(mma_b(wg), mma_phase);
                    __syncwarp();
                    V3C(2);
                    mma_phase ^= 1u;
                    tc::fence_after();
                    {
                        uint32_t d[32];
                        tc::tmem_ld32(tl, d);
                        tc::tmem_wait_ld();
                        if (pair) {
#pragma unroll
                            for (int c = 0; c < 16; c += 2)
                                *reinterpret_cast<float4*>(tile + (ro ^ cfg_off(c))) =
                                    make_float4(__uint_as_float(d[2 * c]) * inv, __uint_as_float(d[2 * c + 1]) * inv,
                                                __uint_as_float(d[2 * c + 2]) * inv, __uint_as_float(d[2 * c + 3]) * inv);
                        } else {
#pragma unroll
                            for (int c = 0; c < 16; ++c)
                                *reinterpret_cast<float2*>(tile + (ro ^ cfg_off(c))) =
                                    make_float2(__uint_as_float(d[2 * c]) * inv, __uint_as_float(d[2 * c + 1]) * inv);
                        }
                    }
                    tc::fence_before();
                    bar_wg(wg);  // the gate's output is in the tile
                    V3C(3);
                } else {
                    // device-chosen operator (CUDA cores): register bits rpos (gate bits first),
                    // thread bits tpos
                    uint32_t unit[4];
#pragma unroll
                    for (int m = 0; m < 4; ++m) unit[m] = Gd.xu[m];
                    uint32_t pb = 0;
#pragma unroll
                    for (int b = 0; b < 7; ++b)
                        if ((wtid >> b) & 1) pb ^= Gd.xu[4 + b];
                    const float2* M = A.pool + Gd.mat_off;
                    const int k = Gd.k & 0xff;
                    float2* tf = reinterpret_cast<float2*>(tile);
                    if (k == 1) apply_fused<1, 4>(tf, M, pb, unit);
                    else if (k == 2) apply_fused<2, 4>(tf, M, pb, unit);
                    else if (k == 3) apply_fused<3, 4>(tf, M, pb, unit);
                    else apply_fused<4, 4>(tf, M, pb, unit);
                    bar_wg(wg);
                    V3C(4);
                }
            }
            V3C(5);
            // ---------------- epilogues (read-only on the tile) ----------------
            const uint64_t tile_row = (uint64_t)slot * ntiles + tile_idx;
            if (P.flags & kPassRho) {
                double* out = A.rho_part + tile_row * A.rho_stride;
                if (P.rho_nq == 1) rho_partial<1>(tile, P.rho_local, out, red, wg);
                else if (P.rho_nq == 2) rho_partial<2>(tile, P.rho_local, out, red, wg);
                else rho_partial_rows3(tile, P.rho_local, out, red, wg);
                bar_wg(wg);
                if (wtid == 0) {
                    __threadfence();
                    misc[1 + wg] = (atomicAdd(&A.counters[slot], 1) == (int)ntiles - 1);
                }
                bar_wg(wg);
                if (misc[1 + wg]) {
                    // last tile of the slot: the tile partials in a fixed order, then Alg. 2's choice
                    __threadfence();
                    const EventDesc E = A.events[P.event];
                    const ChanDesc C = A.chans[E.chan];
                    const int ne = 2 * C.d * C.d;
                    double* fin = red + 128;  // ne <= 128 doubles
                    const double* part = A.rho_part + (uint64_t)slot * ntiles * A.rho_stride;
                    for (int e0 = 0; e0 < ne; e0 += 8) {
                        double acc[8];
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) acc[jj] = 0.0;
                        for (uint32_t t = wtid; t < ntiles; t += NT)
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj)
                                if (e0 + jj < ne) acc[jj] += __ldcg(part + (uint64_t)t * A.rho_stride + e0 + jj);
                        wg_sum<8>(acc, red, wg);  // red[0..31]
                        if (wtid == 0)
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj)
                                if (e0 + jj < ne) fin[e0 + jj] = acc[jj];
                    }
                    if (wtid == 0) {
                        choose_conventional(E, C, A.chan_data, fin, A.pool, A.records, A.status + slot);
                        A.counters[slot] = 0;
                    }
                    bar_wg(wg);
                }
            }
            if (P.flags & kPassFinal) {
                double sum[1] = {0.0};
#pragma unroll
                for (int m = 0; m < NA; ++m) {
                    const float2 v = *reinterpret_cast<const float2*>(tile + swzb((uint32_t)(wtid + m * NT)));
                    sum[0] += (double)v.x * v.x + (double)v.y * v.y;
                }
                wg_sum<1>(sum, red, wg);
                if (wtid == 0) A.blocksum[tile_row] = sum[0];
            }
            if (P.flags & kPassObs) {
                // Z strings: Walsh-Hadamard transform of |psi(wtid + m NT)|^2 over m (tile bits 7..10)
                float w[NA];
#pragma unroll
                for (int m = 0; m < NA; ++m) {
                    const float2 v = *reinterpret_cast<const float2*>(tile + swzb((uint32_t)(wtid + m * NT)));
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
                const float2* st = A.state + ((uint64_t)slot << n);
                double* park = red + 64;  // 4 warps x 16 strings
                for (int o0 = 0; o0 < P.obs_count; o0 += 16) {
                    uint64_t cx = 0, cz = 0;
                    int cny = 0, cslot = 0;
                    if (lane < 16 && o0 + lane < P.obs_count) {
                        const ObsDesc& Ol = A.obs[P.obs_begin + o0 + lane];
                        cx = Ol.xmask;
                        cz = Ol.zmask;
                        cny = Ol.ny;
                        cslot = Ol.slot;
                    }
                    const int oc = min(16, P.obs_count - o0);
                    double pv[16];
#pragma unroll
                    for (int jo = 0; jo < 16; ++jo) {
                        const uint64_t oxm = __shfl_sync(0xffffffffu, cx, jo);
                        const uint64_t ozm = __shfl_sync(0xffffffffu, cz, jo);
                        const int ony = __shfl_sync(0xffffffffu, cny, jo);
                        pv[jo] = 0.0;
                        if (jo < oc) {
                            const uint32_t zl = to_local<T>(ozm, P);
                            const int zs = __popcll(base & ozm) & 1;
                            if (oxm == 0) {
                                const float vv = pick_uniform<NA>(w, (int)(zl >> 7));
                                const int par = (__popc((uint32_t)wtid & zl & (uint32_t)(NT - 1)) + zs) & 1;
                                pv[jo] = par ? -(double)vv : (double)vv;
                            } else {
                                const uint64_t xo = oxm & ~P.tile_mask;
                                const uint32_t xl = to_local<T>(oxm, P);
                                double part = 0.0;
#pragma unroll 1
                                for (int m = 0; m < NA; ++m) {
                                    const uint32_t L = (uint32_t)(wtid + m * NT);
                                    const float2 vv = *reinterpret_cast<const float2*>(tile + swzb(L));
                                    float2 wv;
                                    if (xo == 0) wv = *reinterpret_cast<const float2*>(tile + swzb(L ^ xl));
                                    else wv = st[(base + pdep64(L, P.tile_mask)) ^ oxm];  // read-only pass
                                    const double cr = (double)wv.x * vv.x + (double)wv.y * vv.y;
                                    const double ci = (double)wv.x * vv.y - (double)wv.y * vv.x;
                                    double t;
                                    switch (ony & 3) {
                                        case 0: t = cr; break;
                                        case 1: t = -ci; break;
                                        case 2: t = -cr; break;
                                        default: t = ci; break;
                                    }
                                    const int par = (__popc(L & zl) + zs) & 1;
                                    part += par ? -t : t;
                                }
                                pv[jo] = part;
                            }
                        }
                    }
                    const double rsum = warp_reduce_scatter<16>(pv, lane);
                    bar_wg(wg);  // park's earlier readers are done
                    if ((lane & 1) == 0) park[(wtid >> 5) * 16 + (lane >> 1)] = rsum;
                    bar_wg(wg);
                    if (wtid < oc)  // lane wtid holds string o0 + wtid
                        A.obs_part[tile_row * A.n_obs + cslot] =
                            park[wtid] + park[16 + wtid] + park[32 + wtid] + park[48 + wtid];
                }
            }
            V3C(6);
            tc::fence_before();
            tc::fence_proxy_async();  // generic tile writes -> the TMA store (async proxy)
            arrive(comp_b(s));
#ifdef QT_V3_TIMING
            if (tme && blockIdx.x == 7) atomicAdd(A.timing + 14, 1ull);
#endif
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, kTCols);
    }
}

}  // namespace v3

typedef CUresult (*EncodeTiledFnV3)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Tensor map of the 11-qubit tile layout `tile_mask` (qubits 0..3 included) over a buffer of
// nslots 2^n-amplitude states: box dims [qubits 0..3] [runs of consecutive tile qubits above
// 3, <= 8 qubits each, at most three] [rest = 16-amplitude units, box 1]; tile qubits outside
// those runs are enumerated as boxes (shared-memory image = tile-local index order).
bool v3_encode_map(void* state, int n, uint64_t nslots, uint64_t tile_mask, V3Map* out) {
    static EncodeTiledFnV3 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFnV3>(p);
    }
    if (!fn || (tile_mask & 15ull) != 15ull || __builtin_popcountll(tile_mask) != v3::T) return false;
    if (n - 4 > 31 || (nslots << (n - 4)) > 0x7fffffffull) return false;  // int32 rest coordinates
    int runs_q[16], runs_len[16], nr = 0;
    for (int q = 4; q < n;) {
        if (!((tile_mask >> q) & 1ull)) {
            ++q;
            continue;
        }
        int e = q;
        while (e < n && ((tile_mask >> e) & 1ull) && e - q < 8) ++e;
        runs_q[nr] = q;
        runs_len[nr++] = e - q;
        q = e;
    }
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    dims[0] = 16;
    box[0] = 16;
    const int nd = nr < 3 ? nr : 3;
    for (int d = 0; d < nd; ++d) {
        dims[1 + d] = 1ull << runs_len[d];
        strides[d] = 8ull << runs_q[d];
        box[1 + d] = 1u << runs_len[d];
    }
    for (int d = nd; d < 3; ++d) {
        dims[1 + d] = 1;
        strides[d] = 128;
        box[1 + d] = 1;
    }
    dims[4] = nslots << (n - 4);
    strides[3] = 128;
    box[4] = 1;
    int opq[8], nop = 0;
    for (int r = nd; r < nr; ++r)
        for (int q = runs_q[r]; q < runs_q[r] + runs_len[r]; ++q) opq[nop++] = q;
    if (nop > 4) return false;
    out->nops = 1 << nop;
    out->op_bytes = v3::kTileBytes >> nop;
    for (int o = 0; o < out->nops; ++o) {
        int32_t r = 0;
        for (int b = 0; b < nop; ++b)
            if ((o >> b) & 1) r += (int32_t)(1u << (opq[b] - 4));
        out->op_rest[o] = r;
    }
    for (int o = out->nops; o < 16; ++o) out->op_rest[o] = 0;
    return fn(&out->tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, state, dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#ifdef QT_V3_TIMING
static unsigned long long* g_v3_tbuf = nullptr;
extern "C" void qt_v3_timing_read(unsigned long long* out) {
    cudaDeviceSynchronize();
    if (g_v3_tbuf) cudaMemcpy(out, g_v3_tbuf, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}
#endif

cudaError_t launch_tile_pass_v3(const TileArgs& a, const void* maps, int step, uint32_t ntiles, int nslots,
                                cudaStream_t s) {
    (void)step;
    static bool configured = false;
    static int sms = 0;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(v3::tile_pass_v3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)v3::kSmemBytes);
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
#ifdef QT_V3_TIMING
    static unsigned long long* tb = nullptr;
    if (!tb) {
        cudaMalloc(&tb, 32 * sizeof(unsigned long long));
        cudaMemset(tb, 0, 32 * sizeof(unsigned long long));
    }
    TileArgs b2 = a;
    b2.timing = tb;
    g_v3_tbuf = tb;
    v3::tile_pass_v3_kernel<<<grid, v3::kThreads, v3::kSmemBytes, s>>>(b2, reinterpret_cast<const V3Map*>(maps), nitems,
                                                                       tshift);
#else
    v3::tile_pass_v3_kernel<<<grid, v3::kThreads, v3::kSmemBytes, s>>>(a, reinterpret_cast<const V3Map*>(maps), nitems,
                                                                      tshift);
#endif
    return cudaGetLastError();
}

}  // namespace qt
