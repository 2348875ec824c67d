// tc_rate2.cu -- tcgen05.mma issue->complete cycles per MMA (one CTA, M = 128):
// kind::tf32 (K = 8) vs kind::f16 (K = 16), TS vs SS, N = 16..256, with
// nacc independent accumulators, and 1..4 concurrent CTAs on one SM.
#include <cuda_runtime.h>
#include <stdio.h>
#include "../paper_2111_02396_b200/csrc/tc_common.cuh"
using namespace qt::tc;

template <bool F16>
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if (F16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
                     ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
                     ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}
template <bool F16>
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if (F16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

template <bool F16, int N, int SS, int NMMA, int NACC>
__global__ void __launch_bounds__(128) rate(long long* out, int cols) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    unsigned char* sm = dsm + ((1024 - ((uint32_t)__cvta_generic_to_shared(dsm) & 1023)) & 1023);
    uint32_t* bsm = reinterpret_cast<uint32_t*>(sm);             // 256 rows x 128 B
    uint32_t* asm_ = reinterpret_cast<uint32_t*>(sm + 32768);    // 128 rows x 128 B
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t one = F16 ? 0x3c003c00u : 0x3f800000u;
    for (int i = tid; i < 256 * 32; i += 128) bsm[i] = one;
    for (int i = tid; i < 128 * 32; i += 128) asm_[i] = one;
    if (warp == 0) tmem_alloc(&tbase, cols);
    if (tid == 0) { mbar_init(&mbar, 1); fence_mbar_init(); }
    fence_proxy_async();
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tb = tbase;
    const uint32_t fmt = F16 ? 0u : 2u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const int dcols = N;  // accumulator columns
    uint32_t phase = 0;
    long long acc = 0;
    for (int it = 0; it < 12; ++it) {
        __syncthreads();
        long long t0 = clock64();
        if (tid == 0) {
            const uint32_t sb = (uint32_t)__cvta_generic_to_shared(bsm);
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(asm_);
#pragma unroll
            for (int k = 0; k < NMMA; ++k) {
                const uint32_t d = tb + (k % NACC) * dcols;
                if (SS) mma_ss<F16>(d, smem_desc_sw128(sa + (k & 3) * 32), smem_desc_sw128(sb + (k & 3) * 32), idesc, k >= NACC);
                else mma_ts<F16>(d, tb + NACC * dcols + (k & 3) * 8, smem_desc_sw128(sb + (k & 3) * 32), idesc, k >= NACC);
            }
            mma_commit(&mbar);
        }
        __syncwarp();
        mbar_wait(&mbar, phase);
        phase ^= 1;
        long long t1 = clock64();
        if (it >= 4) acc += t1 - t0;
    }
    if (tid == 0) out[blockIdx.x] = acc / 8;
    fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc(tb, cols);
}

template <bool F16, int N, int ss, int nacc>
void run(const char* name, long long* d, int ctas) {
    int cols = 32;
    while (cols < nacc * N + (ss ? 0 : 32)) cols *= 2;
    if (cols * ctas > 512) return;
    const size_t smem = 32768 + 16384 + 1024;
    cudaFuncSetAttribute(rate<F16, N, ss, 8, nacc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(rate<F16, N, ss, 40, nacc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long h1[4], h2[4];
    rate<F16, N, ss, 8, nacc><<<ctas, 128, smem>>>(d, cols); cudaDeviceSynchronize(); cudaMemcpy(h1, d, 8 * ctas, cudaMemcpyDeviceToHost);
    rate<F16, N, ss, 40, nacc><<<ctas, 128, smem>>>(d, cols);
    cudaError_t e = cudaDeviceSynchronize(); cudaMemcpy(h2, d, 8 * ctas, cudaMemcpyDeviceToHost);
    if (e) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
    const double per = (h2[0] - h1[0]) / 32.0;
    const int K = F16 ? 16 : 8;
    printf("%-5s %s nacc=%d N=%3d ctas=%d: latency(8)=%5lld  per-MMA=%6.1f cyc  => %5.0f MAC/clk (per CTA)\n", name,
           ss ? "SS" : "TS", nacc, N, ctas, h1[0], per, 128.0 * N * K / per);
}

int main() {
    long long* d; cudaMalloc(&d, 64);
    // co-residence on one SM is not guaranteed for ctas > 1 (grid spread over SMs);
    // ctas > 1 uses cluster-free launches and is only indicative
#define R2(SS, N, NACC) run<false, N, SS, NACC>("tf32", d, 1); run<true, N, SS, NACC>("f16", d, 1);
#define RN(SS, NACC) R2(SS, 16, NACC) R2(SS, 32, NACC) R2(SS, 64, NACC) R2(SS, 128, NACC) R2(SS, 256, NACC)
    RN(0, 1) RN(0, 2) RN(1, 1) RN(1, 2)
    return 0;
}
