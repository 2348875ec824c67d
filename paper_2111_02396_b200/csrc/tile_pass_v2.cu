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
// W operands by one 4 KB bulk copy (async proxy, no proxy fence before the MMAs) instead
// of 16-byte cp.async from every thread (whose consumer fence waits for the issuing
// thread's outstanding tile loads)
#ifndef QT_V2_BULKW
#define QT_V2_BULKW 1
#endif
// L2 prefetch of the tile an item loads when done, at the item's context preparation
// (measured slower on C2: 9380 -> 9069 traj/s; kept off)
// MMA completion: every thread polls the commit mbarrier (1) or one thread polls and a
// warpgroup barrier releases the others (0)
#ifndef QT_V2_ALLWAIT
#define QT_V2_ALLWAIT 1
#endif
#ifndef QT_V2_PICKTREE
#define QT_V2_PICKTREE 1
#endif
#ifndef QT_V2_L2PF
#define QT_V2_L2PF 0
#endif
constexpr int NWG = 2;
constexpr int NT = 256;        // threads per compute warpgroup: 2 warps per TMEM lane quarter
constexpr int NWW = NT / 32;   // warps per warpgroup
constexpr int NA = TILE / NT;  // 32 amplitudes per thread
constexpr int kThreads = NWG * NT;
constexpr uint32_t kWOff = NBUF * kTileBytes;
// per-warpgroup item contexts, double-buffered: item k of a warpgroup uses ctx[k & 1],
// prepared (descriptors, tile bases) while item k - 1 runs
struct alignas(16) Ctx {
    PassDesc p;       // the item's pass
    PassDesc p3;      // pass of the item this warpgroup loads when the item is done
    uint64_t base;    // global index of the tile's amplitude 0
    uint64_t base3;   // same for the item loaded at the end
    GateDesc g[kMaxPassGates];
};
constexpr uint32_t kCtxOff = kWOff + NWG * 2 * kV2GateBytes;
constexpr uint32_t kRedOff = kCtxOff + NWG * 2 * sizeof(Ctx);
constexpr uint32_t kMbarOff = kRedOff + NWG * 256 * 8;
constexpr uint32_t kMiscOff = kMbarOff + 16 * 8;
constexpr size_t kSmemBytes = kMiscOff + 64 + 1024;  // + alignment slack

// fp32 tile slot of amplitude L (8-byte units): bits 1..3 ^= bits 4..6 ^ 7..9 ^ 10..12;
// bit 0 is kept so amplitude pairs stay adjacent and 16-byte aligned (cp.async 16).
__device__ __forceinline__ uint32_t swz(uint32_t L) { return L ^ ((((L >> 4) ^ (L >> 7) ^ (L >> 10)) & 7u) << 1); }

__device__ __forceinline__ void bar_wg(int wg) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + wg), "r"(NT) : "memory");
}

__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok) : "r"(a), "r"(phase) : "memory");
    return ok != 0;
}
// wait with a short sleep between polls (the spinning warps would otherwise take
// issue slots from the other warpgroup)
__device__ __forceinline__ void mbar_wait_s(uint32_t a, uint32_t phase) {
    while (!mbar_try(a, phase)) __nanosleep(64);
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
// One group's gate GEMM, D = x_hi W_hi + x_lo W_hi + x_hi W_lo: six M128 N32 K16 MMAs
// (A = [x_hi | x_lo] at TMEM columns ah .. ah + 31, B = W rows at 32-byte K offsets of
// the SW128 descriptor b0) and the commit, in one asm block: the derived operands are
// formed inside it, so ptxas moves d / ah / b0 into uniform registers once.
__device__ __forceinline__ void mma6_commit(uint32_t d, uint32_t ah, uint64_t b0, uint32_t mbar) {
    constexpr uint32_t idesc = tc::idesc_f16_m128(32);
    asm volatile(
        "{\n\t.reg .pred p0, p1;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t"
        "setp.ne.b32 p0, 0, 0;\n\tsetp.eq.b32 p1, 0, 0;\n\t"
        "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
        "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, p1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], %2, %3, p1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b1, %3, p1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], b2, %3, p1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b3, %3, p1;\n\t"
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}\n" ::"r"(d),
        "r"(ah), "l"(b0), "r"(idesc), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t& a, uint32_t& b) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n" : "=r"(a), "=r"(b) : "r"(taddr) : "memory");
}
// 16 lanes x 256 bits: thread t receives lane base + t/4 (r0, r1) and base + 8 + t/4 (r2,
// r3), columns 2 (t % 4) (r0, r2) and 2 (t % 4) + 1 (r1, r3) -- measured, profiles/r2_tmem_shapes.txt
__device__ __forceinline__ void tmem_ld_16x256(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

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

// f16 hi / lo split of a scaled complex amplitude (packed fp32 pair): hi = x with the
// 13 low mantissa bits cleared (exact in f16 above 2^-14), lo = the remainder rounded.
__device__ __forceinline__ void split(uint64_t x, uint32_t& hi, uint32_t& lo) {
    const float2 xf = upk2(x);
    const float hr = __uint_as_float(__float_as_uint(xf.x) & 0xFFFFE000u);
    const float hm = __uint_as_float(__float_as_uint(xf.y) & 0xFFFFE000u);
    const float2 l = upk2(sub2(x, pk2(hr, hm)));
    const __half2 h2 = __floats2half2_rn(hr, hm);
    const __half2 l2 = __floats2half2_rn(l.x, l.y);
    hi = *reinterpret_cast<const uint32_t*>(&h2);
    lo = *reinterpret_cast<const uint32_t*>(&l2);
}

// Deterministic warpgroup sums (fixed order: lanes by xor tree, then warps 0..7).
template <int N>
__device__ __forceinline__ void wg_sum_n(double (&v)[N], double* red, int wg) {
    const int wtid = threadIdx.x & (NT - 1);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    constexpr int C = 16;  // values per chunk (red: 128 doubles = 8 warps x 16)
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += C) {
        bar_wg(wg);
        if ((wtid & 31) == 0)
#pragma unroll
            for (int i = c0; i < N && i < c0 + C; ++i) red[(wtid >> 5) * C + (i - c0)] = v[i];
        bar_wg(wg);
#pragma unroll
        for (int i = c0; i < N && i < c0 + C; ++i) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NWW; ++w) s += red[w * C + i - c0];
            v[i] = s;
        }
    }
}

// Warp reduce-scatter of NE values (NE a power of two <= 32), fixed order: after
// log2(NE) halving exchanges lane l holds the warp sum of value l >> (5 - log2 NE)
// (the remaining lane bits then reduce by xor pairs, a + b == b + a bit for bit).
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

// rho_Q partial (2^Q x 2^Q, fp64) of the tile for a channel at tile-local bits qlocal
// (rho_Q = sum over the other qubits of psi psi^dag).  Only the upper
// triangle is accumulated -- D real diagonal entries, then (re, im) of (a, b), a < b --
// and the lower one written as its conjugate.  Every thread takes TILE / D / NT
// complementary indices (the tile index with zeros inserted at the channel bits), so
// no thread idles; the warpgroup sum is a reduce-scatter per warp, then a fixed-order
// sum over the 8 warps.
template <int Q>
__device__ __forceinline__ void rho_partial(const float2* tile, uint32_t qlocal, double* out, double* red, int wg) {
    constexpr int D = 1 << Q;
    constexpr int NE = D * D;
    const int wtid = threadIdx.x & (NT - 1), lane = wtid & 31;
    uint32_t qoff[D];
#pragma unroll
    for (int a = 0; a < D; ++a) qoff[a] = pdep32((uint32_t)a, qlocal);
    uint32_t qp[Q];
    {
        uint32_t m = qlocal;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            qp[q] = (uint32_t)__ffs(m) - 1u;
            m &= m - 1u;
        }
    }
    double acc[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] = 0.0;
#pragma unroll 2
    for (uint32_t k = wtid; k < (uint32_t)(TILE >> Q); k += NT) {
        uint32_t bL = k;
#pragma unroll
        for (int q = 0; q < Q; ++q) bL = (bL & ((1u << qp[q]) - 1u)) | ((bL >> qp[q]) << (qp[q] + 1u));
        double vr[D], vi[D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const float2 v = tile[swz(bL | qoff[a])];
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
    const double r = warp_reduce_scatter<NE>(acc, lane);
    bar_wg(wg);  // previous readers of red are done
    if ((lane & (32 / NE - 1)) == 0) red[(wtid >> 5) * NE + (lane / (32 / NE))] = r;
    bar_wg(wg);
    if (wtid < NE) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < NWW; ++w) v += red[w * NE + wtid];
        // entry wtid of the compact order -> (a, b) and its mirror
        if (wtid < D) {
            out[2 * (wtid * D + wtid)] = v;
            out[2 * (wtid * D + wtid) + 1] = 0.0;
        } else {
            int e = D, a = 0, b = 1;
            for (; e + 2 <= wtid; e += 2) {
                if (++b == D) {
                    ++a;
                    b = a + 1;
                }
            }
            if (wtid == e) {
                out[2 * (a * D + b)] = v;
                out[2 * (b * D + a)] = v;
            } else {
                out[2 * (a * D + b) + 1] = v;
                out[2 * (b * D + a) + 1] = -v;
            }
        }
    }
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

// w[i] for a warp-uniform index i (0 <= i < 32) by a branch-free select tree
// (QT_V2_PICKTREE; the default jump table costs an indirect branch per string)
__device__ __forceinline__ float pick_tree32(const float (&w)[32], uint32_t i) {
    float a[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = (i & 1u) ? w[2 * k + 1] : w[2 * k];
    float b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) b[k] = (i & 2u) ? a[2 * k + 1] : a[2 * k];
    float c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = (i & 4u) ? b[2 * k + 1] : b[2 * k];
    const float d0 = (i & 8u) ? c[1] : c[0], d1 = (i & 8u) ? c[3] : c[2];
    return (i & 16u) ? d1 : d0;
}

struct Item {
    const PassDesc* p;
    int slot;
    uint32_t tile;
};

// Item i of the step: the pass of active slot i >> tshift (the executor's per-step
// array), tile i & (ntiles - 1).
__device__ __forceinline__ Item item_of(const TileArgs& A, uint32_t i, int tshift) {
    Item it;
    it.p = A.step_passes + (i >> tshift);
    it.slot = it.p->slot;
    it.tile = i & ((1u << tshift) - 1u);
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

// fp32-tile byte offsets of a gate layout (desc.hpp v2_units): this thread's row
// (lane bits + warp bits) with its group 2h (base0) or 2h + 1 (base1), and the 16
// configurations as base ^ c01[c & 3] ^ c23[c >> 2] (one 3-input XOR per access).
struct Fp32Layout {
    uint32_t base0, base1;
    uint32_t c01[4], c23[4];
};
__device__ __forceinline__ Fp32Layout fp32_layout(const GateDesc& G, int wtid) {
    const uint16_t* u = v2_units(G);
    // (u is 8-byte aligned: GateDesc::rpos sits at offset 8)
    const uint2 w0 = *reinterpret_cast<const uint2*>(u), w1 = *reinterpret_cast<const uint2*>(u + 4);
    const uint2 w2 = *reinterpret_cast<const uint2*>(u + 8), w3 = *reinterpret_cast<const uint2*>(u + 12);
    const uint32_t uc0 = w0.x & 0xffffu, uc1 = w0.x >> 16, uc2 = w0.y & 0xffffu, uc3 = w0.y >> 16;
    const uint32_t ug0 = w1.x & 0xffffu, ug1 = w1.x >> 16;
    const uint32_t ur[7] = {w1.y & 0xffffu, w1.y >> 16, w2.x & 0xffffu, w2.x >> 16, w2.y & 0xffffu, w2.y >> 16,
                            w3.x & 0xffffu};
    Fp32Layout L;
    uint32_t rb = 0;
#pragma unroll
    for (int q = 0; q < 7; ++q)
        if ((wtid >> q) & 1) rb ^= ur[q];
    L.base0 = rb ^ ((wtid >> 7) ? ug1 : 0u);
    L.base1 = L.base0 ^ ug0;
    L.c01[0] = 0;
    L.c01[1] = uc0;
    L.c01[2] = uc1;
    L.c01[3] = uc0 ^ uc1;
    L.c23[0] = 0;
    L.c23[1] = uc2;
    L.c23[2] = uc3;
    L.c23[3] = uc2 ^ uc3;
    return L;
}

__global__ void __launch_bounds__(kThreads, 1) tile_pass_v2_kernel(const TileArgs A, const int step,
                                                                    const uint32_t nitems, const int tshift) {
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw_s = (uint32_t)__cvta_generic_to_shared(smem_raw);
    unsigned char* sm = smem_raw + (((raw_s + 1023u) & ~1023u) - raw_s);
    const uint32_t sm_s = (uint32_t)__cvta_generic_to_shared(sm);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t mb = sm_s + kMbarOff;  // full[3] (use 0), empty[3], mma[2], wfull[2][2], full[3] (use 1)
    // "full" barriers: item jj (buffer jj % 3, warpgroup jj % 2) completes on barrier
    // [jj % 3][(jj / 3) & 1], phase (jj / 6) & 1.  A buffer's successive occupants belong
    // to alternating warpgroups, so with one barrier per buffer a warpgroup could wait for
    // the phase after next while the other warpgroup's load (the phase in between) is
    // still in flight, see the parity of an old phase and read the buffer early (it did:
    // read-only passes of n = 23 registers gave wrong observables).  With two barriers per
    // buffer each one is waited on by a single warpgroup, in phase order.
    auto full_bar = [&](int jj) {
        const int b = jj % NBUF, u = (jj / NBUF) & 1;
        return mb + 8u * (uint32_t)(u ? 12 + b : b);
    };
    auto mma_bar = [&](int w) { return mb + 8u * (uint32_t)(6 + w); };
    auto wfull_bar = [&](int w, int i) { return mb + 8u * (uint32_t)(8 + 2 * w + i); };
    uint32_t* misc = reinterpret_cast<uint32_t*>(sm + kMiscOff);  // [0] tmem base, [1..2] last flags
    if (warp == 0) tc::tmem_alloc(misc, 512);
    if (tid == 32) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init_s(full_bar(b), NT);
            mbar_init_s(full_bar(b + NBUF), NT);
        }
        for (int w = 0; w < NWG; ++w) {
            mbar_init_s(mma_bar(w), 4);  // one commit per issuing warp
            mbar_init_s(wfull_bar(w, 0), QT_V2_BULKW ? 1 : NT);
            mbar_init_s(wfull_bar(w, 1), QT_V2_BULKW ? 1 : NT);
        }
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = misc[0];
    const int n = A.n;
    const uint32_t ntiles = 1u << tshift;

    // Tile loads: the warpgroup that releases a buffer loads its next occupant (item
    // j + NBUF, processed by either warpgroup): 16-byte cp.async per thread, completing
    // on the buffer's "full" mbarrier (NT arrivals).
    auto load_item = [&](int jj, const PassDesc& P, uint32_t tile, uint64_t tbase_g, int wtid) {
        const int b = jj % NBUF;
        const uint32_t buf = sm_s + (uint32_t)b * kTileBytes;
        if (P.flags & kPassInit) {
            // first pass of a trajectory: |0...0> (amplitude 0 lives in tile 0, slot 0)
            float4* t4 = reinterpret_cast<float4*>(sm + (size_t)b * kTileBytes);
            for (int k = wtid; k < TILE / 2; k += NT)
                t4[k] = make_float4((k == 0 && tile == 0) ? 1.f : 0.f, 0.f, 0.f, 0.f);
            mbar_arrive_s(full_bar(jj));
        } else {
            const float2* st = A.state + ((uint64_t)P.slot << n) + tbase_g;
            // thread: pair p = wtid & 7 of run h = 32 k + (wtid >> 3); h bits 0..4 fixed
            const int p = wtid & 7;
            const uint32_t h0 = (uint32_t)(wtid >> 3);
            uint64_t ofix = 0;
#pragma unroll
            for (int q = 0; q < 5; ++q) ofix |= (uint64_t)((h0 >> q) & 1u) << P.tq[4 + q];
            // run offsets of tile bits 9..12 (k bits): sums of four basis offsets
            const float2* src = st + ofix + 2 * p;
            const float2* s1 = src + (1ull << P.tq[9]);
            const uint64_t e1 = 1ull << P.tq[10], e2 = 1ull << P.tq[11], e3 = 1ull << P.tq[12];
#pragma unroll
            for (uint32_t k = 0; k < 16; ++k) {
                const uint32_t L = 16u * (32u * k + h0);
                const uint32_t slot = (L ^ ((((L >> 4) ^ (L >> 7) ^ (L >> 10)) & 7u) << 1)) ^ (2u * (uint32_t)p);
                const uint64_t x = ((k & 2) ? e1 : 0ull) + ((k & 4) ? e2 : 0ull) + ((k & 8) ? e3 : 0ull);
                cp_async16_s(buf + 8u * slot, ((k & 1) ? s1 : src) + x);
            }
            // the loading threads wait for their own copies, then arrive: completion by
            // cp.async.mbarrier.arrive.noinc let consumers pass the phase with part of the
            // tile not yet written (read-only passes of n = 23 registers, about one tile in
            // 4000, measured with QT_DUMP_PARTIALS); waiting here cost nothing measurable
            // on C2 (110.4 vs 110.9 ms per 1024 trajectories)
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            mbar_arrive_s(full_bar(jj));
        }
    };
    {
        // ---------------- compute warpgroups ----------------
        const int wg = warp / NWW;
        const int wtid = tid & (NT - 1);
        const int half = wtid >> 7;  // groups 2 half, 2 half + 1
        const uint32_t tbase = tmem + 256u * (uint32_t)wg;
        const uint32_t lane_off = ((uint32_t)(warp & 3) * 32u) << 16;
        const uint32_t tl = tbase + lane_off;  // this thread's TMEM lane, column 0 of the warpgroup
        const uint32_t tlh = tl + 128u * (uint32_t)half;  // its first group's D
        double* red = reinterpret_cast<double*>(sm + kRedOff) + 256 * wg;
        Ctx* ctxs = reinterpret_cast<Ctx*>(sm + kCtxOff) + 2 * wg;
        const uint32_t wbuf = sm_s + kWOff + (uint32_t)wg * 2u * kV2GateBytes;
        const bool elect = wtid == 0;
        const bool issuer = (wtid & 31) == 0 && wtid < 128;  // MMA issue: lane 0 of warps 0..3 (group = warp)
        const bool prep_warp = (wtid >> 5) == 1;  // warp 1 of the warpgroup prepares the next item's context
        uint32_t mma_phase = 0;
        uint32_t w_issued = 0, w_used = 0;  // bulk W loads issued / consumed (buffer = index & 1)
        // items of this CTA in order (ordinal jj): raw index blockIdx.x + jj gridDim.x;
        // warpgroup w processes the ordinals jj = w (mod 2)
        auto raw = [&](int jj) { return blockIdx.x + (uint32_t)jj * gridDim.x; };
        // context preparation for ordinal jj into c, by the prep warp: stage A loads the
        // pass descriptors (registers), stage B stores them, computes the tile bases and
        // starts the gate-descriptor copies (cp.async group, waited for at the item start)
        uint4 pd_reg = make_uint4(0, 0, 0, 0);
        auto prep_a = [&](int jj) {
            const uint32_t i = raw(jj), i3 = raw(jj + NBUF);
            if (lane < 4 && i < nitems)
                pd_reg = reinterpret_cast<const uint4*>(A.step_passes + (i >> tshift))[lane];
            else if (lane >= 4 && lane < 8 && i3 < nitems)
                pd_reg = reinterpret_cast<const uint4*>(A.step_passes + (i3 >> tshift))[lane - 4];
        };
        auto prep_b = [&](int jj, Ctx* c) {
            const uint32_t i = raw(jj), i3 = raw(jj + NBUF);
            if (i >= nitems) return;
            if (lane < 4) reinterpret_cast<uint4*>(&c->p)[lane] = pd_reg;
            else if (lane < 8 && i3 < nitems) reinterpret_cast<uint4*>(&c->p3)[lane - 4] = pd_reg;
            __syncwarp();
            if (lane == 0) c->base = tile_base(c->p, i & ((1u << tshift) - 1u));
            if (lane == 1 && i3 < nitems) c->base3 = tile_base(c->p3, i3 & ((1u << tshift) - 1u));
            const uint4* src = reinterpret_cast<const uint4*>(A.gates + c->p.gate_begin);
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(c->g);
            const int nch = c->p.gate_count * (int)(sizeof(GateDesc) / 16);
            for (int k = lane; k < nch; k += 32) cp_async16_s(dst + 16u * (uint32_t)k, src + k);
            asm volatile("cp.async.commit_group;\n" ::: "memory");
#if QT_V2_L2PF
            // the tile this item loads when done (ordinal jj + 3, about two items ahead):
            // its 512 runs of 128 B into L2, so the cp.async load later hits L2
            if (i3 < nitems && !(c->p3.flags & kPassInit)) {
                __syncwarp();
                const PassDesc& P3 = c->p3;
                uint64_t ofix = 0;
#pragma unroll
                for (int q = 0; q < 5; ++q) ofix |= (uint64_t)((lane >> q) & 1) << P3.tq[4 + q];
                const float2* s3 = A.state + ((uint64_t)P3.slot << A.n) + c->base3 + ofix;
                const uint64_t e0 = 1ull << P3.tq[9], e1 = 1ull << P3.tq[10], e2 = 1ull << P3.tq[11],
                               e3 = 1ull << P3.tq[12];
#pragma unroll
                for (uint32_t k = 0; k < 16; ++k) {
                    const uint64_t x = ((k & 1) ? e0 : 0ull) + ((k & 2) ? e1 : 0ull) + ((k & 4) ? e2 : 0ull) +
                                       ((k & 8) ? e3 : 0ull);
                    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(s3 + x));
                }
            }
#endif
        };
        // prologue: the first item's context, then the first loads (ordinals 0 and 2 by
        // warpgroup 0, ordinal 1 by warpgroup 1)
        // W operands (4 KB per tensor-core gate, two buffers per warpgroup): every thread
        // copies 16 bytes with cp.async (1-D bulk copies were measured an order of
        // magnitude slower, profiles/r2_ubench_stream.txt).  cp.async.mbarrier.arrive
        // tracks ALL earlier cp.async of the thread, so an item's first two operands are
        // issued at the end of the warpgroup's previous item, before its tile load;
        // later ones as soon as a buffer's MMAs complete.
        auto issue_w_of = [&](const GateDesc* gl, int ngl, int& wn) {
            while (wn < ngl && !(gl[wn].k & kGateTC)) ++wn;
            if (wn < ngl) {
                const uint32_t wi = w_issued & 1u;
#if QT_V2_BULKW
                if (wtid == 32) bulk_w(wbuf + wi * kV2GateBytes, A.pool + gl[wn].mat_off, wfull_bar(wg, (int)wi));
#else
                cp_async16_s(wbuf + wi * kV2GateBytes + 16u * (uint32_t)wtid,
                             reinterpret_cast<const char*>(A.pool + gl[wn].mat_off) + 16 * wtid);
                cp_async_arrive_noinc(wfull_bar(wg, (int)wi));
#endif
                ++w_issued;
                ++wn;
            }
        };
        int w_carry = 0;  // operands of this warpgroup's next item already issued
        if (prep_warp) {
            prep_a(wg);
            prep_b(wg, &ctxs[0]);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        bar_wg(wg);
        if (raw(wg) < nitems) {
            issue_w_of(ctxs[0].g, ctxs[0].p.gate_count, w_carry);
            issue_w_of(ctxs[0].g, ctxs[0].p.gate_count, w_carry);
        }
        for (int jj = 0; jj < NBUF; ++jj) {
            const uint32_t i = raw(jj);
            if (i < nitems && (jj & 1) == wg) {
                const Item it = item_of(A, i, tshift);
                load_item(jj, *it.p, it.tile, tile_base(*it.p, it.tile), wtid);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
#ifdef QT_V2_TIMING
        long long t_prev = clock64();
#define QT_T(k)                                                                              \
    if (wtid == 0 && blockIdx.x == 7) {                                                      \
        const long long t_now = clock64();                                                   \
        atomicAdd(A.timing + (k), (unsigned long long)(t_now - t_prev));                     \
        t_prev = t_now;                                                                      \
    }
#define QT_C(k, v)                                                                           \
    if (wtid == 0 && blockIdx.x == 7) atomicAdd(A.timing + (k), (unsigned long long)(v));
#else
#define QT_T(k)
#define QT_C(k, v)
#endif
        int kk = 0;  // this warpgroup's item count
        for (int jj = wg; raw(jj) < nitems; jj += 2, ++kk) {
            const uint32_t i = raw(jj);
            const uint32_t i3 = raw(jj + NBUF);  // loaded into b by this warpgroup when done
            const int b = jj % NBUF;
            Ctx* cx = &ctxs[kk & 1];  // complete and visible since the previous item's end
            if (prep_warp) prep_a(jj + 2);
            bool prep_pending = prep_warp;
            const PassDesc& P = cx->p;
            const GateDesc* gds = cx->g;
            const int slot = P.slot;
            const uint32_t tile_idx = i & ((1u << tshift) - 1u);
            float2* st = A.state + ((uint64_t)slot << n);
            float2* tile = reinterpret_cast<float2*>(sm + (size_t)b * kTileBytes);
            char* const tb8 = reinterpret_cast<char*>(tile);
            const int ng = P.gate_count;
            int w_next = w_carry;  // next gate whose W has not been issued
            auto issue_w = [&]() { issue_w_of(gds, ng, w_next); };
            const uint64_t base = cx->base, base3 = cx->base3;
            // every thread acquires the tile's "full" phase (the cp.async writes of the
            // loading warpgroup; a single poller + bar.sync would order them too, but
            // compute-sanitizer racecheck only tracks the direct acquire)
            mbar_wait_s(full_bar(jj), (uint32_t)((jj / (2 * NBUF)) & 1));
            QT_T(0);
            QT_C(11, 1);
            float run_inv = 1.f;
            for (int g = 0; g < ng;) {
                if (!(gds[g].k & kGateTC)) {
                    // device-chosen conventional operator (k <= 3) on FP32 CUDA cores, 32 amplitudes per thread
                    const GateDesc& G = gds[g];
                    uint32_t unit[5];
#pragma unroll
                    for (int m = 0; m < 5; ++m) unit[m] = swz(1u << ((G.rpos >> (4 * m)) & 15u)) << 3;
                    uint32_t tb = 0;
#pragma unroll
                    for (int q = 0; q < 8; ++q) tb |= ((uint32_t)(wtid >> q) & 1u) << ((G.tpos >> (4 * q)) & 15u);
                    const float2* M = A.pool + G.mat_off;
                    const int k = G.k & 0xff;
                    if (k == 1) apply_fused<1, 5>(tile, M, swz(tb) << 3, unit);
                    else if (k == 2) apply_fused<2, 5>(tile, M, swz(tb) << 3, unit);
                    else apply_fused<3, 5>(tile, M, swz(tb) << 3, unit);
                    bar_wg(wg);
                    QT_T(16);
                    QT_C(17, 1);
                    ++g;
                    continue;
                }
                // ---- segment start: gather the fp32 tile into A (TMEM), new tile scale ----
                {
                    const Fp32Layout L = fp32_layout(gds[g], wtid);
                    uint64_t v[32];
                    float amax = 0.f;
                    if (gds[g].k & kGatePair0) {
                        // matrix bit 0 = tile bit 0: configurations c, c + 1 are one 16-byte pair
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                            for (int c = 0; c < 16; c += 2) {
                                const uint32_t o = (jj ? L.base1 : L.base0) ^ L.c01[c & 3] ^ L.c23[c >> 2];
                                const float4 f = *reinterpret_cast<const float4*>(tb8 + o);
                                v[16 * jj + c] = pk2(f.x, f.y);
                                v[16 * jj + c + 1] = pk2(f.z, f.w);
                                amax = fmaxf(amax, fmaxf(fmaxf(fabsf(f.x), fabsf(f.y)), fmaxf(fabsf(f.z), fabsf(f.w))));
                            }
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                            for (int c = 0; c < 16; ++c) {
                                const uint32_t o = (jj ? L.base1 : L.base0) ^ L.c01[c & 3] ^ L.c23[c >> 2];
                                const float2 f = *reinterpret_cast<const float2*>(tb8 + o);
                                v[16 * jj + c] = pk2(f.x, f.y);
                                amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
                            }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
                    float* redf = reinterpret_cast<float*>(red);
                    if (lane == 0) redf[wtid >> 5] = amax;
                    bar_wg(wg);
                    amax = redf[0];
#pragma unroll
                    for (int w = 1; w < NWW; ++w) amax = fmaxf(amax, redf[w]);
                    const int shift = (gds[g].k >> kGateShiftBit) & 0xff;
                    int se = 260 - (int)((__float_as_uint(amax) >> 23) & 0xffu) - shift;  // amax 2^(se-127) in [2^6, 2^7)
                    se = min(max(se, 1), 253);
                    const float run_scale = __uint_as_float((uint32_t)se << 23);
                    run_inv = __uint_as_float((uint32_t)(254 - se) << 23);
                    const uint64_t sc2 = pk2(run_scale, run_scale);
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        uint32_t a[32];
#pragma unroll
                        for (int c = 0; c < 16; ++c) split(mul2(v[16 * jj + c], sc2), a[c], a[16 + c]);
                        tc::tmem_st32(tlh + 64u * (uint32_t)jj + 32u, a);
                    }
                    tc::tmem_wait_st();
                    tc::fence_before();
                    bar_wg(wg);  // A complete; every fp32 read of this buffer done
                    QT_T(1);
                    QT_C(13, 1);
                }
                // ---- the segment's gates ----
                for (;;) {
                    if (issuer) {
                        // W(g) (issued earlier, in order), then this issuer's group: four issuing
                        // threads (lane 0 of warps 0..3) keep the tensor pipe fed
                        const uint32_t wi = w_used & 1u;
                        mbar_wait_s(wfull_bar(wg, (int)wi), (w_used >> 1) & 1u);
                        QT_T(22);
#if !QT_V2_BULKW
                        tc::fence_proxy_async();  // cp.async (generic proxy) writes -> tensor-core reads
#endif
                        tc::fence_after();
                        const uint32_t wb = wbuf + wi * kV2GateBytes;
                        const uint32_t d = tbase + 64u * (uint32_t)(wtid >> 5);
                        mma6_commit(d, d + 32u, tc::smem_desc_sw128(wb), mma_bar(wg));
                        QT_T(7);
                    }
                    ++w_used;
                    QT_C(12, 1);
                    const int32_t gk = gds[g].k;
                    __syncwarp();
                    if (prep_pending) {  // in the shadow of the MMAs
                        prep_b(jj + 2, &ctxs[(kk + 1) & 1]);
                        prep_pending = false;
                    }
#if QT_V2_ALLWAIT
                    // every thread acquires the MMAs' completion itself (no barrier round trip)
                    while (!mbar_try(mma_bar(wg), mma_phase)) {
                    }
#else
                    if (elect) mbar_wait_s(mma_bar(wg), mma_phase);
                    tc::fence_before();
                    bar_wg(wg);
#endif
                    QT_T(2);
                    mma_phase ^= 1u;
                    tc::fence_after();
                    issue_w();  // gate g's W buffer is free: the operand of the gate after next
                    if (gk & kGateRunEnd) {
                        // ---- segment end: D -> fp32 tile ----
                        const Fp32Layout L = fp32_layout(gds[g], wtid);
                        const uint64_t inv2 = pk2(run_inv, run_inv);
                        const bool pair = (gk & kGatePair0) != 0;
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            uint32_t d[32];
                            tc::tmem_ld32(tlh + 64u * (uint32_t)jj, d);
                            tc::tmem_wait_ld();
                            const uint32_t o0 = jj ? L.base1 : L.base0;
                            if (pair) {
#pragma unroll
                                for (int c = 0; c < 16; c += 2) {
                                    const uint32_t o = o0 ^ L.c01[c & 3] ^ L.c23[c >> 2];
                                    const float2 a = upk2(
                                        mul2(pk2(__uint_as_float(d[2 * c]), __uint_as_float(d[2 * c + 1])), inv2));
                                    const float2 b = upk2(
                                        mul2(pk2(__uint_as_float(d[2 * c + 2]), __uint_as_float(d[2 * c + 3])), inv2));
                                    *reinterpret_cast<float4*>(tb8 + o) = make_float4(a.x, a.y, b.x, b.y);
                                }
                            } else {
#pragma unroll
                                for (int c = 0; c < 16; ++c) {
                                    const uint32_t o = o0 ^ L.c01[c & 3] ^ L.c23[c >> 2];
                                    *reinterpret_cast<float2*>(tb8 + o) = upk2(
                                        mul2(pk2(__uint_as_float(d[2 * c]), __uint_as_float(d[2 * c + 1])), inv2));
                                }
                            }
                        }
                        tc::fence_before();
                        bar_wg(wg);
                        QT_T(3);
                        ++g;
                        break;
                    }
                    // ---- in-TMEM transition to gate g + 1: its A from this gate's D ----
                    if (gk & kGateXNext) {
                        // X: 16x256b loads transpose lanes and columns (profiles/r2_tmem_shapes.txt):
                        // thread t receives config bits 0, 1 = t & 3 and lane bits 0..2 = t >> 2 of
                        // this gate, plus lane bit 3 as the register pair; the next gate's rows are
                        // (config 0, config 1, lane 0, lane 1, lane 2), its matrix bit 0 is lane bit 3
                        const uint16_t* gu = v2_units(gds[g]) + 14;
                        uint32_t xv[5];
#pragma unroll
                        for (int r = 0; r < 5; ++r) xv[r] = (gu[r] & 0x8000u) ? (16u << 16) : (uint32_t)gu[r];
                        const uint32_t x01[4] = {0u, xv[0], xv[1], xv[0] + xv[1]};
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            const uint32_t ab = tl + (half ? xv[4] : 0u) + (jj ? xv[3] : 0u);
                            uint32_t d[32];
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                uint32_t r4[4];
                                tmem_ld_16x256(ab + x01[q & 3] + ((q & 4) ? xv[2] : 0u), r4);
                                d[4 * q] = r4[0];
                                d[4 * q + 1] = r4[1];
                                d[4 * q + 2] = r4[2];
                                d[4 * q + 3] = r4[3];
                            }
                            tc::tmem_wait_ld();
                            uint32_t a[32];
#pragma unroll
                            for (int c = 0; c < 16; ++c)
                                split(pk2(__uint_as_float(d[2 * c]), __uint_as_float(d[2 * c + 1])), a[c], a[16 + c]);
                            tc::tmem_st32(tlh + 64u * (uint32_t)jj + 32u, a);
                        }
                        tc::tmem_wait_st();
                        tc::fence_before();
                        bar_wg(wg);
                    } else {
                        const uint16_t* gu = v2_units(gds[g]) + 13;
                        const uint32_t xu[6] = {gu[0], gu[1], gu[2], gu[3], gu[4], gu[5]};
                        const uint32_t t01[4] = {0u, xu[0], xu[1], xu[0] + xu[1]};
                        const uint32_t t23[4] = {0u, xu[2], xu[3], xu[2] + xu[3]};
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            // output group 2 half + jj
                            uint32_t cj = tl;
                            if (half) cj += xu[5];
                            if (jj) cj += xu[4];
                            uint32_t d[32];
#pragma unroll
                            for (int c = 0; c < 16; ++c) {
                                tmem_ld2(cj + t01[c & 3] + t23[c >> 2], d[2 * c], d[2 * c + 1]);
                            }
                            tc::tmem_wait_ld();
                            uint32_t a[32];
#pragma unroll
                            for (int c = 0; c < 16; ++c) split(pk2(__uint_as_float(d[2 * c]), __uint_as_float(d[2 * c + 1])), a[c], a[16 + c]);
                            tc::tmem_st32(tlh + 64u * (uint32_t)jj + 32u, a);
                        }
                        tc::tmem_wait_st();
                        tc::fence_before();
                        bar_wg(wg);
                    }
                    QT_T(8);
                    ++g;
                }
            }
            if (prep_pending) {
                prep_b(jj + 2, &ctxs[(kk + 1) & 1]);
                prep_pending = false;
            }
            // ---------------- epilogues (read-only on the fp32 tile) ----------------
            const uint64_t tile_row = (uint64_t)slot * ntiles + tile_idx;
            if (P.flags & kPassRho) {
                const uint32_t ql = P.rho_local;  // channel qubits as tile-local bits (planner)
                double* out = A.rho_part + tile_row * A.rho_stride;
                if (P.rho_nq == 1) rho_partial<1>(tile, ql, out, red, wg);
                else if (P.rho_nq == 2) rho_partial<2>(tile, ql, out, red, wg);
                else rho_partial_rows3(tile, ql, out, red, wg);
                // the partial's writers are ordered before thread 0 by the barrier, and thread
                // 0's device-scope fence before the counter increment releases them
                // cumulatively (one fence per warpgroup instead of one per thread)
                bar_wg(wg);
                if (wtid == 0) {
                    __threadfence();
                    misc[1 + wg] = (atomicAdd(&A.counters[slot], 1) == (int)ntiles - 1);
                }
                bar_wg(wg);
                if (misc[1 + wg]) {
                    // last tile of the slot: sum the tile partials in a fixed order, then choose
                    __threadfence();
                    const EventDesc E = A.events[P.event];
                    const ChanDesc C = A.chans[E.chan];
                    const int ne = 2 * C.d * C.d;
                    double* fin = red + 128;  // ne <= 128 doubles: red[128..255] of this warpgroup
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
                QT_T(9);
                QT_C(14, 1);
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
                QT_T(10);
                QT_C(15, 1);
            }
            QT_T(18);
            if (P.flags & kPassObs) {
                QT_C(19, 1);
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
                // observable descriptors: lane l < 16 of every warp holds string o0 + l of
                // the chunk, broadcast by shuffles (no dependent global load per string)
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
                    if (__all_sync(0xffffffffu, cx == 0)) {
                        // Z strings only: the 16 thread partials side by side, one warp
                        // reduce-scatter, one fixed-order sum over the 8 warps
                        double pv[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const uint64_t ozm = __shfl_sync(0xffffffffu, cz, j);
                            pv[j] = 0.0;
                            if (j < oc) {
                                const uint32_t zl = P.tile_mask == (uint64_t)(TILE - 1) ? (uint32_t)(ozm & (TILE - 1))
                                                                                         : to_local<T>(ozm, P);
                                const int zs = __popcll(base & ozm) & 1;
#if QT_V2_PICKTREE
                                const float vv = pick_tree32(w, zl >> 8);
#else
                                const float vv = pick_uniform<NA>(w, (int)(zl >> 8));
#endif
                                const int par = (__popc((uint32_t)wtid & zl & (uint32_t)(NT - 1)) + zs) & 1;
                                pv[j] = par ? -(double)vv : (double)vv;
                            }
                        }
                        const double r = warp_reduce_scatter<16>(pv, lane);
                        double* park = red + 128;  // 8 warps x 16 strings
                        bar_wg(wg);
                        if ((lane & 1) == 0) park[(wtid >> 5) * 16 + (lane >> 1)] = r;
                        bar_wg(wg);
                        if (wtid < oc) {
                            double v = 0.0;
#pragma unroll
                            for (int w2 = 0; w2 < NWW; ++w2) v += park[w2 * 16 + wtid];
                            A.obs_part[tile_row * A.n_obs + cslot] = v;  // lane wtid holds string o0 + wtid
                        }
                        continue;
                    }
                    bar_wg(wg);  // park's readers of a previous chunk are done
                    for (int j = 0; j < oc; ++j) {
                        const int o = o0 + j;
                        const uint64_t oxm = __shfl_sync(0xffffffffu, cx, j);
                        const uint64_t ozm = __shfl_sync(0xffffffffu, cz, j);
                        const int ony = __shfl_sync(0xffffffffu, cny, j);
                        // tile-local Z bits (the final pass's tile is the low 13 qubits: a mask)
                        const uint32_t zl = P.tile_mask == (uint64_t)(TILE - 1) ? (uint32_t)(ozm & (TILE - 1))
                                                                                 : to_local<T>(ozm, P);
                        const int zs = __popcll(base & ozm) & 1;
                        double part[1];
                        if (oxm == 0) {
                            const float vv = pick_uniform<NA>(w, (int)(zl >> 8));
                            const int par = (__popc((uint32_t)wtid & zl & (uint32_t)(NT - 1)) + zs) & 1;
                            part[0] = par ? -(double)vv : (double)vv;
                        } else {
                            const uint64_t xo = oxm & ~P.tile_mask;
                            const uint32_t xl = to_local<T>(oxm, P);
                            part[0] = 0.0;
#pragma unroll 1
                            for (int m = 0; m < NA; ++m) {
                                const uint32_t L = (uint32_t)(wtid + m * NT);
                                const float2 v = tile[swz(L)];
                                float2 wv;
                                if (xo == 0) {
                                    wv = tile[swz(L ^ xl)];
                                } else {  // partner amplitude in another tile (read-only pass only)
                                    wv = st[(base + pdep64(L, P.tile_mask)) ^ oxm];
                                }
                                const double cr = (double)wv.x * v.x + (double)wv.y * v.y;
                                const double ci = (double)wv.x * v.y - (double)wv.y * v.x;
                                double t;
                                switch (ony & 3) {
                                    case 0: t = cr; break;
                                    case 1: t = -ci; break;
                                    case 2: t = -cr; break;
                                    default: t = ci; break;
                                }
                                const int par = (__popc(L & zl) + zs) & 1;
                                part[0] += par ? -t : t;
                            }
                        }
                        // warp sums parked per (observable, warp); one barrier pair per 16
                        // strings, then a fixed-order sum over the 8 warps
#pragma unroll
                        for (int sh = 16; sh > 0; sh >>= 1) part[0] += __shfl_xor_sync(0xffffffffu, part[0], sh);
                        double* park = red + 128;  // 16 strings x 8 warps
                        const int jo = o & 15;
                        if (lane == 0) park[jo * NWW + (wtid >> 5)] = part[0];
                        if (jo == 15 || o + 1 == P.obs_count) {
                            bar_wg(wg);
                            // column of string o - jo + lane of this chunk
                            const int sl = __shfl_sync(0xffffffffu, cslot, (j - jo + lane) & 15);
                            if (wtid <= jo) {
                                double v = 0.0;
#pragma unroll
                                for (int w2 = 0; w2 < NWW; ++w2) v += park[wtid * NWW + w2];
                                A.obs_part[tile_row * A.n_obs + sl] = v;
                            }
                            bar_wg(wg);
                        }
                    }
                }
            }
            // ---------------- shared -> HBM: 16-byte stores of amplitude pairs ----------------
            QT_T(4);
            if (P.flags & kPassStore) {
                // thread: pair p = wtid & 7 of run h = (wtid >> 3) + 32 m
                const int p = wtid & 7;
                const uint32_t hl = (uint32_t)(wtid >> 3);
                uint64_t ofix = 0;
#pragma unroll
                for (int q = 0; q < 5; ++q) ofix |= (uint64_t)((hl >> q) & 1u) << P.tq[4 + q];
                float2* dst = st + base + ofix + 2 * p;
                float2* d1 = dst + (1ull << P.tq[9]);
                const uint64_t e1 = 1ull << P.tq[10], e2 = 1ull << P.tq[11], e3 = 1ull << P.tq[12];
#pragma unroll
                for (uint32_t m = 0; m < 16; ++m) {
                    const uint32_t L = 16u * (hl + 32u * m);
                    const uint32_t s2 = (L ^ ((((L >> 4) ^ (L >> 7) ^ (L >> 10)) & 7u) << 1)) ^ (2u * (uint32_t)p);
                    const float4 v = *reinterpret_cast<const float4*>(tb8 + 8u * s2);
                    const uint64_t x = ((m & 2) ? e1 : 0ull) + ((m & 4) ? e2 : 0ull) + ((m & 8) ? e3 : 0ull);
                    *reinterpret_cast<float4*>(((m & 1) ? d1 : dst) + x) = v;
                }
            }
            if (prep_warp) asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // next item's context
            bar_wg(wg);  // every read of the buffer and of the staged descriptors done; next context visible
            QT_T(5);
            w_carry = 0;
            if (raw(jj + 2) < nitems) {
                const Ctx* nx = &ctxs[(kk + 1) & 1];
                issue_w_of(nx->g, nx->p.gate_count, w_carry);
                issue_w_of(nx->g, nx->p.gate_count, w_carry);
            }
            if (i3 < nitems) load_item(jj + NBUF, cx->p3, i3 & ((1u << tshift) - 1u), base3, wtid);
            asm volatile("cp.async.commit_group;\n" ::: "memory");
            QT_T(6);
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

}  // namespace v2

size_t tile_pass_v2_smem_bytes() { return v2::kSmemBytes; }
#ifdef QT_V2_TIMING
static unsigned long long* g_v2_tbuf = nullptr;
// diagnostics build: clock64 phase sums of warpgroup leaders of CTA 7 (32 counters)
extern "C" void qt_v2_timing_read(unsigned long long* out) {
    cudaDeviceSynchronize();
    if (g_v2_tbuf) cudaMemcpy(out, g_v2_tbuf, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}
#endif

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
#ifdef QT_V2_TIMING
    if (!g_v2_tbuf) {
        cudaMalloc(&g_v2_tbuf, 32 * sizeof(unsigned long long));
        cudaMemset(g_v2_tbuf, 0, 32 * sizeof(unsigned long long));
    }
    TileArgs b2 = a;
    b2.timing = g_v2_tbuf;
    v2::tile_pass_v2_kernel<<<grid, v2::kThreads, v2::kSmemBytes, s>>>(b2, step, nitems, tshift);
#else
    v2::tile_pass_v2_kernel<<<grid, v2::kThreads, v2::kSmemBytes, s>>>(a, step, nitems, tshift);
#endif
    return cudaGetLastError();
}

}  // namespace qt
