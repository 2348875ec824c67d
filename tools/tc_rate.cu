// tc_rate.cu -- tcgen05.mma kind::tf32 issue->complete cycles vs N (TS mode, M = 128, K = 8).
#include <cuda_runtime.h>
#include <stdio.h>
#include "../paper_2111_02396_b200/csrc/tc_common.cuh"
using namespace qt::tc;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
                 ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

__global__ void __launch_bounds__(128) rate(long long* out, int N, int ss, int nmma, int nacc) {
    __shared__ __align__(1024) uint32_t bsm[128 * 32];
    __shared__ __align__(1024) uint32_t asm_[128 * 32];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 32; i += 128) bsm[i] = 0x3f800000u;
    for (int i = tid; i < 128 * 32; i += 128) asm_[i] = 0x3f800000u;
    if (warp == 0) tmem_alloc(&tbase, 512);
    if (tid == 0) { mbar_init(&mbar, 1); fence_mbar_init(); }
    fence_proxy_async();
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tb = tbase;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    uint32_t phase = 0;
    long long acc = 0;
    for (int it = 0; it < 12; ++it) {
        __syncthreads();
        long long t0 = clock64();
        if (tid == 0) {
            const uint32_t sb = (uint32_t)__cvta_generic_to_shared(bsm);
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(asm_);
            for (int k = 0; k < nmma; ++k) {
                if (ss) mma_ss(tb, smem_desc_sw128(sa + (k & 3) * 32), smem_desc_sw128(sb + (k & 3) * 32), idesc, k > 0);
                else mma_ts(tb + (k % nacc) * 64, tb + 256 + (k & 3) * 8, smem_desc_sw128(sb + (k & 3) * 32), idesc, k >= nacc);
            }
            mma_commit(&mbar);
        }
        __syncwarp();
        mbar_wait(&mbar, phase);
        phase ^= 1;
        long long t1 = clock64();
        if (it >= 4) acc += t1 - t0;
    }
    if (tid == 0) out[0] = acc / 8;
    fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 512);
}

int main() {
    long long* d; cudaMalloc(&d, 64);
    for (int nacc : {1, 2, 4})
        for (int N : {32, 64}) {
            long long h1, h2;
            rate<<<1, 128>>>(d, N, 0, 8, nacc); cudaDeviceSynchronize(); cudaMemcpy(&h1, d, 8, cudaMemcpyDeviceToHost);
            rate<<<1, 128>>>(d, N, 0, 40, nacc); cudaError_t e = cudaDeviceSynchronize(); cudaMemcpy(&h2, d, 8, cudaMemcpyDeviceToHost);
            if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            const double per = (h2 - h1) / 32.0;
            printf("TS nacc=%d N=%3d: latency(8)=%lld  per-MMA=%.1f cyc  => %.0f tf32 MAC/clk/SM\n", nacc, N, h1, per, 128.0 * N * 8 / per);
        }
    return 0;
}
