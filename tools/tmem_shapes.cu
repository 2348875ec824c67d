// tmem_shapes.cu -- which (TMEM lane, column) each thread of a warp reads with the
// tcgen05.ld shapes 16x64b / 16x128b / 16x256b / 16x32bx2 (written with 32x32b,
// value = lane << 16 | column), and the throughput of a 32x32b-store /
// 16x256b-load round trip (a lane <-> register transpose inside TMEM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tmem_shapes.bin tools/tmem_shapes.cu
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2111_02396_b200/csrc/tc_common.cuh"
using namespace qt::tc;

__global__ void shapes(uint32_t* out) {
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tmem_alloc(&tbase, 64);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tb = tbase;
    const uint32_t lo = ((uint32_t)warp * 32u) << 16;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = ((uint32_t)(warp * 32 + lane) << 16) | (uint32_t)c;
    tmem_st32(tb + lo, v);
    for (int c = 0; c < 32; ++c) v[c] = ((uint32_t)(warp * 32 + lane) << 16) | (uint32_t)(32 + c);
    tmem_st32(tb + lo + 32, v);
    tmem_wait_st();
    __syncwarp();
    if (warp == 0) {
        uint32_t r[8];
        // 16x64b.x1: 1 register
        asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];\n" : "=r"(r[0]) : "r"(tb));
        tmem_wait_ld();
        out[0 * 32 + lane] = r[0];
        asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0, %1}, [%2];\n" : "=r"(r[0]), "=r"(r[1]) : "r"(tb));
        tmem_wait_ld();
        out[1 * 32 + lane] = r[0];
        out[2 * 32 + lane] = r[1];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tb));
        tmem_wait_ld();
        for (int i = 0; i < 4; ++i) out[(3 + i) * 32 + lane] = r[i];
        asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x1.b32 {%0}, [%1], 4;\n" : "=r"(r[0]) : "r"(tb));
        tmem_wait_ld();
        out[7 * 32 + lane] = r[0];
        // lane offset 16 (second half of the subpartition)
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tb + (16u << 16)));
        tmem_wait_ld();
        for (int i = 0; i < 4; ++i) out[(8 + i) * 32 + lane] = r[i];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tb));
        tmem_wait_ld();
        for (int i = 0; i < 8; ++i) out[(12 + i) * 32 + lane] = r[i];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 64);
}

// SHFL throughput alone and mixed with STS.128 / LDS.64 (do they share the shared-memory data path?)
template <int MODE>
__global__ void __launch_bounds__(256) shfl_bw(uint32_t* sink, int iters) {
    __shared__ __align__(16) uint32_t sm[8192];
    const int tid = threadIdx.x;
    uint32_t a0 = tid, a1 = tid * 3, a2 = tid * 5, a3 = tid * 7;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 2) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                a0 = __shfl_xor_sync(0xffffffffu, a0, 1 + (j & 15));
                a1 = __shfl_xor_sync(0xffffffffu, a1, 2);
                a2 = __shfl_xor_sync(0xffffffffu, a2, 4);
                a3 = __shfl_xor_sync(0xffffffffu, a3, 8);
            }
        }
        if (MODE == 1 || MODE == 2) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                reinterpret_cast<uint4*>(sm)[(tid + 256 * (j & 7)) & 2047] = make_uint4(a0 + it, a1, a2 + j, a3);
        }
    }
    if ((a0 ^ a1 ^ a2 ^ a3) == 0x12345u) sink[0] = a0 + sm[tid];
}

int main_bw() {
    uint32_t* sink;
    cudaMalloc(&sink, 64);
    const int iters = 4096;
    const char* nm[3] = {"shfl only", "sts.128 only", "shfl + sts.128"};
    for (int m = 0; m < 3; ++m) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (m == 0) shfl_bw<0><<<148 * 4, 256>>>(sink, iters);
            if (m == 1) shfl_bw<1><<<148 * 4, 256>>>(sink, iters);
            if (m == 2) shfl_bw<2><<<148 * 4, 256>>>(sink, iters);
            cudaEventRecord(b);
            cudaDeviceSynchronize();
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double clk = 1.965e9 * ms * 1e-3;
        const double warps = 148.0 * 4 * 8;
        const double shfl = (m != 1) ? warps * iters * 32 / clk / 148 : 0;   // warp-shfl per clk per SM
        const double sts = (m != 0) ? warps * iters * 8 * 512 / clk / 148 : 0;  // bytes per clk per SM
        printf("%-16s %.3f ms: shfl %.2f warp-instr/clk/SM (%.0f B/clk), sts %.1f B/clk/SM\n", nm[m], ms, shfl,
               shfl * 128, sts);
    }
    return 0;
}

int main() {
    main_bw();
    uint32_t* d;
    cudaMalloc(&d, 20 * 32 * 4);
    cudaMemset(d, 0xff, 20 * 32 * 4);
    shapes<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) {
        printf("err %s\n", cudaGetErrorString(e));
        return 1;
    }
    uint32_t h[20 * 32];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[20] = {"16x64b r0", "16x128b r0", "16x128b r1", "16x256b r0", "16x256b r1", "16x256b r2",
                             "16x256b r3", "16x32bx2(off4) r0", "16x256b@lane16 r0", "@16 r1", "@16 r2", "@16 r3",
                             "16x256b.x2 r0", "r1", "r2", "r3", "r4", "r5", "r6", "r7"};
    for (int s = 0; s < 20; ++s) {
        printf("%-20s", names[s]);
        for (int t = 0; t < 32; ++t) printf(" %d:%d", h[s * 32 + t] >> 16, h[s * 32 + t] & 0xffff);
        printf("\n");
    }
    return 0;
}
