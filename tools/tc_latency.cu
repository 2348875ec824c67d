// tc_latency.cu -- clock64 timing of the tcgen05 fused-gate chain pieces (one CTA).
#include <cuda_runtime.h>
#include <stdio.h>
#include "../paper_2111_02396_b200/csrc/tc_common.cuh"
using namespace qt::tc;

__global__ void __launch_bounds__(128) lat(long long* out, int nmma) {
    __shared__ __align__(1024) uint32_t wsm[2 * 32 * 32];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 2 * 32 * 32; i += 128) wsm[i] = 0x3f800000u;
    if (warp == 0) tmem_alloc(&tbase, 128);
    if (tid == 0) { mbar_init(&mbar, 1); fence_mbar_init(); }
    fence_before(); __syncthreads(); fence_after();
    const uint32_t tb = tbase, lane_off = (uint32_t)(warp * 32) << 16;
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = 0x3f800000u;
    fence_proxy_async();
    uint32_t phase = 0;
    long long t_st = 0, t_mma = 0, t_ld = 0, t_sync = 0;
    for (int it = 0; it < 20; ++it) {
        long long t0 = clock64();
        tmem_st32(tb + lane_off + 64, v);
        tmem_st32(tb + lane_off + 96, v);
        tmem_wait_st();
        long long t1 = clock64();
        fence_before();
        __syncthreads();
        long long t2 = clock64();
        if (tid == 0) {
            fence_after();
            const uint32_t sb = (uint32_t)__cvta_generic_to_shared(wsm);
            for (int k = 0; k < nmma; ++k)
                mma_tf32_ts(tb, tb + 64 + (k & 3) * 8, smem_desc_sw128(sb + (k & 3) * 32), k > 0);
            mma_commit(&mbar);
        }
        __syncwarp();
        mbar_wait(&mbar, phase);
        phase ^= 1;
        fence_after();
        long long t3 = clock64();
        tmem_ld32(tb + lane_off, v);
        tmem_wait_ld();
        long long t4 = clock64();
        if (it >= 4) { t_st += t1 - t0; t_sync += t2 - t1; t_mma += t3 - t2; t_ld += t4 - t3; }
        for (int i = 0; i < 32; ++i) v[i] = (v[i] & 0x7fffffffu) | 0x3f800000u;
    }
    if (tid == 0) { out[0] = t_st / 16; out[1] = t_sync / 16; out[2] = t_mma / 16; out[3] = t_ld / 16; }
    fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 128);
}

int main() {
    long long* d; cudaMalloc(&d, 64);
    for (int nmma : {1, 3, 6, 12, 24, 48}) {
        lat<<<1, 128>>>(d, nmma);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("nmma=%2d  tmem_st(2x x32)+wait=%lld  bar=%lld  issue->mbar=%lld  tmem_ld(x32)+wait=%lld cycles\n", nmma, h[0], h[1], h[2], h[3]);
    }
    return 0;
}
