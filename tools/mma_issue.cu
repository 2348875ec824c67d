// mma_issue.cu -- cycles to ISSUE the 24 tcgen05.mma (kind::f16, TS, M128 N32 K16) of
// one v2 gate (4 groups x 6) under different issue styles:
//   0: one thread (tid % 128 == 0) issues per-MMA asm statements (compiler "waterfall" loops)
//   1: the whole warp runs the issue code, operands made warp-uniform with __shfl_sync,
//      each MMA predicated on elect.sync inside the asm
//   2: one asm block with all 24 MMAs (elect.sync predicate), addresses as asm operands
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_issue.bin tools/mma_issue.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include "../paper_2111_02396_b200/csrc/tc_common.cuh"
using namespace qt::tc;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
    constexpr uint32_t idesc = idesc_f16_m128(32);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
// elect one lane of the (converged) warp inside the asm
__device__ __forceinline__ void mma_ts_e(uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
    constexpr uint32_t idesc = idesc_f16_m128(32);
    asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "elect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void gate24(uint32_t tbase, uint64_t b0, uint64_t b1, uint64_t b2, uint64_t b3) {
    constexpr uint32_t idesc = idesc_f16_m128(32);
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b32 d, ah, al;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "mov.b32 d, %0;\n\t"
#define QT_G(OFF)                                                                  \
        "add.u32 d, %0, " #OFF ";\n\tadd.u32 ah, d, 32;\n\tadd.u32 al, d, 48;\n\t"  \
        "@e tcgen05.mma.cta_group::1.kind::f16 [d], [ah], %1, %5, 0;\n\t"          \
        "add.u32 ah, ah, 8;\n\t"                                                   \
        "@e tcgen05.mma.cta_group::1.kind::f16 [d], [ah], %2, %5, 1;\n\t"          \
        "@e tcgen05.mma.cta_group::1.kind::f16 [d], [al], %1, %5, 1;\n\t"          \
        "add.u32 al, al, 8;\n\t"                                                   \
        "@e tcgen05.mma.cta_group::1.kind::f16 [d], [al], %2, %5, 1;\n\t"          \
        "add.u32 ah, ah, -8;\n\t"                                                  \
        "@e tcgen05.mma.cta_group::1.kind::f16 [d], [ah], %3, %5, 1;\n\t"          \
        "add.u32 ah, ah, 8;\n\t"                                                   \
        "@e tcgen05.mma.cta_group::1.kind::f16 [d], [ah], %4, %5, 1;\n\t"
        QT_G(0) QT_G(64) QT_G(128) QT_G(192)
#undef QT_G
        "}\n" ::"r"(tbase), "l"(b0), "l"(b1), "l"(b2), "l"(b3), "r"(idesc));
}

__global__ void __launch_bounds__(256, 1) k(long long* out, int mode, int reps) {
    __shared__ __align__(1024) unsigned char wb[2][4096];
    __shared__ uint64_t mbar[2];
    __shared__ uint32_t tb;
    const int tid = threadIdx.x, warp = tid >> 5, wg = warp >> 2;
    for (int i = tid; i < 2 * 4096 / 4; i += 256) reinterpret_cast<uint32_t*>(wb)[i] = 0x3c003c00u;
    if (warp == 0) tmem_alloc(&tb, 512);
    if (tid == 0) { mbar_init(&mbar[0], mode == 4 ? 4 : 1); mbar_init(&mbar[1], mode == 4 ? 4 : 1); fence_mbar_init(); }
    fence_proxy_async();
    fence_before(); __syncthreads(); fence_after();
    long long ti = 0;
    uint32_t ph = 0;
    const bool issuer = mode == 0 ? (tid & 127) == 0 : (mode == 4 ? (tid & 31) == 0 : (tid & 127) < 32);
    if (issuer) {
        uint32_t tbase = tb + 256u * wg;
        uint32_t w = (uint32_t)__cvta_generic_to_shared(wb[wg]);
        if (mode != 0 && mode != 4) {
            tbase = __shfl_sync(0xffffffffu, tbase, 0);
            w = __shfl_sync(0xffffffffu, w, 0);
        }
        if (mode == 3) {
            // the CTA owns all 512 columns: the allocation starts at column 0 (checked)
            if (tb != 0) asm volatile("trap;");
            tbase = wg ? 256u : 0u;
            w = (uint32_t)__cvta_generic_to_shared(wb[0]) + (wg ? 4096u : 0u);
        }
        const uint64_t b0 = smem_desc_sw128(w), b1 = smem_desc_sw128(w + 32), b2 = smem_desc_sw128(w + 64), b3 = smem_desc_sw128(w + 96);
        for (int r = 0; r < reps; ++r) {
            const long long t0 = clock64();
            if (mode == 4) {
                const uint32_t jg = (uint32_t)(warp & 3);
                const uint32_t d = tbase + 64u * jg, ah = d + 32u, al = d + 48u;
                mma_ts(d, ah, b0, 0u); mma_ts(d, ah + 8u, b1, 1u); mma_ts(d, al, b0, 1u);
                mma_ts(d, al + 8u, b1, 1u); mma_ts(d, ah, b2, 1u); mma_ts(d, ah + 8u, b3, 1u);
            } else if (mode == 3) {
                if (wg == 0) {
                    const uint32_t w0 = (uint32_t)__cvta_generic_to_shared(wb[0]);
                    gate24(0u, smem_desc_sw128(w0), smem_desc_sw128(w0 + 32), smem_desc_sw128(w0 + 64), smem_desc_sw128(w0 + 96));
                } else {
                    const uint32_t w1 = (uint32_t)__cvta_generic_to_shared(wb[1]);
                    gate24(256u, smem_desc_sw128(w1), smem_desc_sw128(w1 + 32), smem_desc_sw128(w1 + 64), smem_desc_sw128(w1 + 96));
                }
            } else if (mode == 2) {
                gate24(tbase, b0, b1, b2, b3);
            } else {
                for (int jg = 0; jg < 4; ++jg) {
                    const uint32_t d = tbase + 64u * jg, ah = d + 32u, al = d + 48u;
                    if (mode == 0) {
                        mma_ts(d, ah, b0, 0u); mma_ts(d, ah + 8u, b1, 1u); mma_ts(d, al, b0, 1u);
                        mma_ts(d, al + 8u, b1, 1u); mma_ts(d, ah, b2, 1u); mma_ts(d, ah + 8u, b3, 1u);
                    } else {
                        mma_ts_e(d, ah, b0, 0u); mma_ts_e(d, ah + 8u, b1, 1u); mma_ts_e(d, al, b0, 1u);
                        mma_ts_e(d, al + 8u, b1, 1u); mma_ts_e(d, ah, b2, 1u); mma_ts_e(d, ah + 8u, b3, 1u);
                    }
                }
            }
            if (mode == 0 || (tid & 31) == 0) mma_commit(&mbar[wg]);
            __syncwarp((mode == 0 || mode == 4) ? 1u : 0xffffffffu);
            const long long t1 = clock64();
            mbar_wait(&mbar[wg], ph);
            ph ^= 1;
            if (r >= 4) ti += t1 - t0;
        }
        if (blockIdx.x == 0 && (tid & 127) == 0) out[wg] = ti / (reps - 4);
        if (mode == 4 && blockIdx.x == 0 && (tid & 127) == 96) out[2 + wg] = ti / (reps - 4);
    }
    fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

int main() {
    long long* d; cudaMalloc(&d, 64);
    for (int mode = 0; mode < 5; ++mode) {
        cudaMemset(d, 0, 64);
        k<<<148, 256>>>(d, mode, 68);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("mode %d: issue of 24 MMAs: wg0 %lld cyc, wg1 %lld cyc (mode 4, warp 3: %lld / %lld)\n", mode, h[0], h[1], h[2], h[3]);
    }
    return 0;
}
