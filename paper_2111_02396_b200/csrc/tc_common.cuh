// tc_common.cuh -- tcgen05 / TMEM / mbarrier primitives (inline PTX, sm_100a) used by
// the tensor-core fused-gate path.
//
// 4-qubit gates (kind::f16, the K1 default): a fused gate U (16 x 16 complex)
// applied to the 256 subvectors x_s of a tile is the real GEMM D = A B^T with
//   A[s][4c + q] = {hi(x_c.re), hi(x_c.im), lo(x_c.re), lo(x_c.im)}[q]   (K = 64 f16)
//   B[n][4c + q]: n = 2j + b   -> hi(W[c][a][b]) for every q   (x_hi + x_lo times W_hi)
//                 n = 32+2j+b  -> lo(W[c][a][b]) for q < 2, 0 otherwise   (x_hi times W_lo)
// with a = q & 1 the input component, b the output component and W[c][a][b] the
// real 2x2 block of U[j][c]; y_j = D[s][2j + b] + D[s][32 + 2j + b].  hi / lo are
// the f16 rounding of a value and of its remainder (22 significant bits; the
// dropped x_lo W_lo term is ~2^-22 relative), the amplitudes carrying a
// power-of-two tile scale that keeps them inside the f16 range.  M = 128 rows
// per MMA (two groups), N = 64, four K-steps of 16: 8 MMAs per gate.  A and B
// both live in shared memory in the SWIZZLE_128B K-major layout (one 128-byte
// row per subvector / output column, 8-row atoms of 1024 B).
//
// 5- and 6-qubit gates (kind::f16, f = 5 / 6 plans; "wide" gates, one gate at
// a time): U (2^k x 2^k complex) applied to the subvectors x_s of a tile is the
// real GEMM Y = X W^T with X[s][2c + a] = component a of x_s[c] and
// W[2j + b][2c + a] = the real 2x2 block of U[j][c] (input component a, output
// component b).  Single precision is kept with f16 hi / lo splits of the
// (tile-scaled) amplitudes and of W:  Y = Xh Wh + Xl Wh + Xh Wl (+ Xl Wl).
//   k = 5: 128 subvectors = M; K = N = 64.  A = [Xh | Xl] as two 16 KB
//          K-chunks, B = [Wh | Wl] as two 8 KB parts; 3 x 4 MMAs M128 N64 K16
//          accumulate into one 64-column D.
//   k = 6: 64 subvectors, K = N = 128.  The MMA rows are (part, subvector):
//          rows 0..63 = Xh, rows 64..127 = Xl; B rows 0..127 = Wh, 128..255 =
//          Wl, so one N = 256 chain (8 K-steps, two 16 KB A chunks / two 32 KB
//          B chunks) gives all four products; the epilogue adds row s and row
//          s + 64 (an exchange through shared memory between threads t, t ^ 64).
#pragma once
#include <stdint.h>

namespace qt {
namespace tc {

// Byte offset of byte `kb` of row `row` in a SWIZZLE_128B K-major operand
// (128-byte rows, 16-byte chunk index ^= row % 8, 8-row atoms of 1024 bytes).
__host__ __device__ __forceinline__ uint32_t sw128_offset(int row, int kb) {
    return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((kb >> 4) ^ row) & 7) << 4) + (kb & 15));
}
// f16 operand of a 4-qubit gate: B = [64 rows][64 f16] (8 KB); A = two groups of
// [128 rows][64 f16] (16 KB each).
constexpr int kF16GateBytes = 64 * 128;
constexpr int kF16GroupBytes = 128 * 128;

// Instruction descriptor: kind::f16 (A, B f16, D f32, both K-major), M = 128, N.
__host__ __device__ constexpr uint32_t idesc_f16_m128(int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
}

// W in shared memory: [N = 32 rows][K = 32 tf32] K-major, 128-byte rows,
// SWIZZLE_128B (16-byte chunk index ^= row % 8), 8-row atoms of 1024 bytes.
__host__ __device__ __forceinline__ uint32_t w_offset_bytes(int n, int k) {
    return (uint32_t)((n >> 3) * 1024 + (n & 7) * 128 + ((((k >> 2) ^ (n & 7)) & 7) << 4) + (k & 3) * 4);
}
constexpr int kWBytes = 32 * 32 * 4;          // one of hi / lo
constexpr int kGateBytes = 2 * kWBytes;       // hi then lo (8 KB)

// tf32 hi / lo W of a 4-qubit gate (3xTF32, single-gate runs): N = K = 32,
// one [N rows][32 tf32] SWIZZLE_128B K-major block per part, hi then lo.
__host__ __device__ __forceinline__ uint32_t w_offset_bytes_k(int k, int n, int kk) {
    const int N = 2 << k;
    return (uint32_t)((kk >> 5) * N * 128) + w_offset_bytes(n, kk & 31);
}
__host__ __device__ constexpr int w_part_bytes(int k) { return (2 << k) * (2 << k) * 4; }
// Pool / shared-memory bytes of a tensor-core gate operand: k = 4: 8 KB (f16
// B or tf32 hi/lo W); k = 5: 2 x [64][64] f16 = 16 KB; k = 6: 2 K-chunks of
// [256][64] f16 = 64 KB.
__host__ __device__ constexpr int gate_bytes(int k) { return k <= 4 ? 2 * w_part_bytes(4) : (k == 5 ? 16384 : 65536); }
// Byte offset of f16 element (row n, K index kk) of a wide-gate B operand.
__host__ __device__ __forceinline__ uint32_t wide_b_offset(int k, int part, int n, int kk) {
    return k == 5 ? (uint32_t)(part * 8192) + sw128_offset(n, 2 * kk)
                  : (uint32_t)((kk >> 6) * 32768) + sw128_offset(part * 128 + n, 2 * (kk & 63));
}

// Instruction descriptor: kind::tf32, D f32, A/B tf32 K-major, M = 128, N.
__host__ __device__ constexpr uint32_t idesc_tf32_m128(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
}

// Shared-memory matrix descriptor (K-major, SWIZZLE_128B, SBO = 1024 B).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);          // start address
    d |= (uint64_t)(1) << 16;                            // LBO (unused for swizzled K-major)
    d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;         // SBO: 8-row atom stride
    d |= (uint64_t)1 << 46;                              // version = 1 (sm100)
    d |= (uint64_t)2 << 61;                              // layout: SWIZZLE_128B
    return d;
}

// Instruction descriptor: kind::tf32, D f32, A/B tf32 K-major, M = 128, N = 32.
constexpr uint32_t kIdescTf32_M128_N32 =
    (1u << 4)            // c_format = F32
    | (2u << 7)          // a_format = TF32
    | (2u << 10)         // b_format = TF32
    | ((32u >> 3) << 17) // n_dim
    | ((128u >> 4) << 24);  // m_dim

__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
        ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(kIdescTf32_M128_N32), "r"(accumulate),
          "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

__device__ __forceinline__ void mma_tf32_ts_n(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
        ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate),
          "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

// D (TMEM) (+)= A (smem desc) * B (smem desc)^T, kind::f16.
__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(a)
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a), "r"(phase) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}

// One-thread bulk copy global -> shared completing on an mbarrier (expect_tx).
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* mbar) {
    const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(m), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(d), "l"(gsrc), "r"(bytes), "r"(m) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

// TMEM allocation (one warp), columns = power of two >= 32.
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t cols) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(a), "r"(cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(cols) : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread (lane) i <-> TMEM lane (warp base + i).
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n"
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
          "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
          "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
          "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ uint32_t tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return r;
}

}  // namespace tc
}  // namespace qt
