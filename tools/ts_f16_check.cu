// ts_f16_check.cu -- layout check of tcgen05.mma kind::f16 with A in TMEM (TS):
// A[128][64] f16 stored with tcgen05.st 32x32b (thread = row, column k/2 holds the
// f16 pair (k even: low half)), B[32][64] f16 K-major SWIZZLE_128B in shared
// memory, D[128][32] = A B^T (f32) via four K16 steps (A columns 8 ks.., B bytes
// 32 ks..).  Also the 3-product scheme used by K1 (x_hi W_hi + x_lo W_hi + x_hi
// W_lo with A = [x_hi (16 cols) | x_lo (16 cols)], B row = [W_hi (64 B) | W_lo]).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ts_f16_check.bin tools/ts_f16_check.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2111_02396_b200/csrc/tc_common.cuh"
using namespace qt::tc;

__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

// mode 0: plain D = A B^T (K = 64); mode 1: 3-product scheme
__global__ void check(const __half* A, const __half* B, float* D, int mode) {
    __shared__ __align__(1024) unsigned char bs[32 * 128];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    // B: row n (128 bytes = 64 f16), 16-byte chunk index ^= n & 7, 8-row atoms of 1024 B
    for (int i = tid; i < 32 * 64; i += 128) {
        const int n = i / 64, k = i % 64;
        *reinterpret_cast<__half*>(bs + sw128_offset(n, 2 * k)) = B[i];
    }
    if (warp == 0) tmem_alloc(&tbase, 64);
    if (tid == 0) {
        mbar_init(&mbar, 1);
        fence_mbar_init();
    }
    fence_proxy_async();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tb = tbase;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) {
        const __half lo = A[tid * 64 + 2 * c], hi = A[tid * 64 + 2 * c + 1];
        v[c] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
    }
    tmem_st32(tb + ((uint32_t)(warp * 32) << 16) + 32, v);  // A at columns 32..63
    tmem_wait_st();
    fence_before();
    __syncthreads();
    if (tid == 0) {
        fence_after();
        const uint32_t idesc = idesc_f16_m128(32);
        const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(bs);
        if (mode == 0) {
            for (int ks = 0; ks < 4; ++ks)
                mma_f16_ts(tb, tb + 32 + 8 * ks, smem_desc_sw128(b0 + 32 * ks), idesc, ks > 0);
        } else {
            // A cols 32..47 = x_hi (K 0..31), 48..63 = x_lo; B bytes 0..63 = W_hi, 64..127 = W_lo
            for (int ks = 0; ks < 2; ++ks) mma_f16_ts(tb, tb + 32 + 8 * ks, smem_desc_sw128(b0 + 32 * ks), idesc, ks > 0);
            for (int ks = 0; ks < 2; ++ks) mma_f16_ts(tb, tb + 48 + 8 * ks, smem_desc_sw128(b0 + 32 * ks), idesc, 1);
            for (int ks = 0; ks < 2; ++ks) mma_f16_ts(tb, tb + 32 + 8 * ks, smem_desc_sw128(b0 + 64 + 32 * ks), idesc, 1);
        }
        mma_commit(&mbar);
    }
    __syncwarp();
    mbar_wait(&mbar, 0);
    fence_after();
    tmem_ld32(tb + ((uint32_t)(warp * 32) << 16), v);
    tmem_wait_ld();
    for (int c = 0; c < 32; ++c) D[tid * 32 + c] = __uint_as_float(v[c]);
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 64);
}

int main() {
    __half *hA = new __half[128 * 64], *hB = new __half[32 * 64];
    float* hD = new float[128 * 32];
    srand(7);
    for (int i = 0; i < 128 * 64; ++i) hA[i] = __float2half((rand() % 17 - 8) / 8.0f);
    for (int i = 0; i < 32 * 64; ++i) hB[i] = __float2half((rand() % 13 - 6) / 4.0f);
    __half *dA, *dB;
    float* dD;
    cudaMalloc(&dA, sizeof(__half) * 128 * 64);
    cudaMalloc(&dB, sizeof(__half) * 32 * 64);
    cudaMalloc(&dD, sizeof(float) * 128 * 32);
    cudaMemcpy(dA, hA, sizeof(__half) * 128 * 64, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(__half) * 32 * 64, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
        check<<<1, 128>>>(dA, dB, dD, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) {
            printf("err %s\n", cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(hD, dD, sizeof(float) * 128 * 32, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 32; ++n) {
                double s = 0;
                if (mode == 0) {
                    for (int k = 0; k < 64; ++k) s += (double)__half2float(hA[m * 64 + k]) * __half2float(hB[n * 64 + k]);
                } else {
                    for (int k = 0; k < 32; ++k) {
                        const double xh = __half2float(hA[m * 64 + k]), xl = __half2float(hA[m * 64 + 32 + k]);
                        const double wh = __half2float(hB[n * 64 + k]), wl = __half2float(hB[n * 64 + 32 + k]);
                        s += xh * wh + xl * wh + xh * wl;
                    }
                }
                maxerr = fmax(maxerr, fabs(s - hD[m * 32 + n]));
            }
        printf("mode %d (%s): max |D - ref| = %g  (D[0][0] = %g)\n", mode, mode ? "3-product" : "plain K64", maxerr,
               hD[0]);
    }
    return 0;
}
