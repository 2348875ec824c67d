// ubench_sm.cu -- per-SM throughput of the operations a chained tensor-core gate
// is built from, measured on the whole B200 (grid = 148 x C CTAs, C resident per
// SM), timed with CUDA events:
//   ldtm   : tcgen05.ld 32x32b.x{16,32} + wait::ld loops (TMEM -> registers)
//   sts    : st.shared.v4 loops (conflict-free)
//   mma    : tcgen05.mma kind::f16 M128 N{32,64,128} K16, SS (A, B in smem) or
//            TS (A in TMEM), one issuing thread per CTA, commit per 8 MMAs
//   mix    : mma (SS, N64) issued by thread 0 while all warps run ldtm + sts
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_sm.bin tools/ubench_sm.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2111_02396_b200/csrc/tc_common.cuh"
using namespace qt::tc;

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

constexpr int kIters = 2048;

// mode: 0 ldtm x32, 1 ldtm x16, 2 sts, 3 mma SS, 4 mma TS, 5 mix (mma SS + ldtm + sts)
template <int MODE, int N>
__global__ void __launch_bounds__(256) bench(unsigned* sink, int warps_active) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    unsigned char* sm = dsm + ((1024 - ((uint32_t)__cvta_generic_to_shared(dsm) & 1023)) & 1023);
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (48 << 10) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    constexpr uint32_t kCols = (MODE == 4 && N >= 64) ? 256u : ((MODE == 3 && N == 256) ? 256u : 128u);
    if (warp == 0) tmem_alloc(&tbase, kCols);
    if (tid == 0) {
        mbar_init(&mbar, 1);
        fence_mbar_init();
    }
    fence_proxy_async();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tb = tbase;
    unsigned acc = 0;
    const uint32_t lane_off = ((uint32_t)(warp & 3) * 32u) << 16;
    const bool active = warp < warps_active;
    if (MODE == 0 || MODE == 1 || MODE == 5) {
        if (active) {
            for (int it = 0; it < kIters; ++it) {
                if (MODE == 1) {
                    uint32_t v[16];
                    tmem_ld16(tb + lane_off + 16 * (it & 3), v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc += v[j];
                } else {
                    uint32_t v[32];
                    tmem_ld32(tb + lane_off + (MODE == 5 ? 64 : 32 * (it & 3)), v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) acc ^= v[j];
                    if (MODE == 5) {  // 8 B per amplitude written back: 16 amps x 8 B = 128 B per thread
                        uint4* p = reinterpret_cast<uint4*>(sm + 16384 + ((tid * 16) & 16383));
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            p[(j * 256) & 1023] = make_uint4(v[4 * j] ^ acc, v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                        }
                    }
                }
            }
        }
    }
    if (MODE == 2 && active) {
        uint4* p = reinterpret_cast<uint4*>(sm) + tid;
        for (int it = 0; it < kIters; ++it) {
#pragma unroll
            for (int j = 0; j < 8; ++j) p[(j * 256 + it) & 2047] = make_uint4(it, j, tid, acc);
        }
    }
    if ((MODE == 3 || MODE == 4 || MODE == 5) && tid == 0) {
        const uint32_t idesc = idesc_f16_m128(N);
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm);
        const uint32_t sb = sa + 16384;
        uint32_t phase = 0;
        const int nmma = MODE == 5 ? kIters / 2 : kIters;
        for (int it = 0; it < nmma; it += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (MODE == 4)
                    mma_f16_ts(tb, tb + (N >= 64 ? 128 : 64) + (k & 3) * 8, smem_desc_sw128(sb + (k & 3) * 32), idesc, k > 0);
                else
                    mma_f16_ss(tb, smem_desc_sw128(sa + (k & 3) * 32), smem_desc_sw128(sb + (k & 3) * 32), idesc,
                               k > 0);
            }
            mma_commit(&mbar);
            mbar_wait(&mbar, phase);
            phase ^= 1u;
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, kCols);
    if (acc == 0x12345678u) sink[0] = acc;
}

template <int MODE, int N>
void run(const char* name, int ctas_per_sm, int threads, int warps_active) {
    const int cols = (MODE == 4 && N >= 64) ? 256 : ((MODE == 3 && N == 256) ? 256 : 128);
    if (cols * ctas_per_sm > 512) return;
    const int sms = 148;
    const size_t smem = (48 << 10) + 1024;
    cudaFuncSetAttribute(bench<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned* sink;
    cudaMalloc(&sink, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    bench<MODE, N><<<sms * ctas_per_sm, threads, smem>>>(sink, warps_active);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) bench<MODE, N><<<sms * ctas_per_sm, threads, smem>>>(sink, warps_active);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        exit(1);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double clk = 1.965e9 * ms * 1e-3 / reps;  // SM cycles per launch (at max clock)
    double per_sm = 0;
    const char* unit = "";
    if (MODE == 0) per_sm = (double)ctas_per_sm * warps_active * kIters * 32 * 32 * 4 / clk, unit = "B/clk/SM TMEM read";
    if (MODE == 1) per_sm = (double)ctas_per_sm * warps_active * kIters * 32 * 16 * 4 / clk, unit = "B/clk/SM TMEM read";
    if (MODE == 2) per_sm = (double)ctas_per_sm * warps_active * 32 * kIters * 8 * 16 / clk, unit = "B/clk/SM STS";
    if (MODE == 3 || MODE == 4)
        per_sm = (double)ctas_per_sm * kIters * 128.0 * N * 16 / clk, unit = "MAC/clk/SM";
    if (MODE == 5)
        per_sm = (double)ctas_per_sm * (kIters / 2) * 128.0 * N * 16 / clk, unit = "MAC/clk/SM (mma part)";
    printf("%-28s ctas/SM=%d thr=%3d warps=%d : %8.1f %s   (%.3f ms)\n", name, ctas_per_sm, threads, warps_active,
           per_sm, unit, ms / reps);
    if (MODE == 5) {
        const double tm = (double)ctas_per_sm * warps_active * kIters * 32 * 32 * 4 / clk;
        printf("%-28s   ... + TMEM read %.1f B/clk/SM + STS %.1f B/clk/SM\n", "", tm, tm);
    }
    cudaFree(sink);
}

int main() {
    for (int c = 1; c <= 4; c *= 2) {
        run<0, 64>("ldtm x32", c, 128, 4);
        run<0, 64>("ldtm x32 (8 warps)", c, 256, 8);
        run<1, 64>("ldtm x16", c, 128, 4);
        run<2, 64>("sts.128", c, 128, 4);
        run<2, 64>("sts.128 (8 warps)", c, 256, 8);
        run<3, 32>("mma SS N32", c, 128, 0);
        run<3, 64>("mma SS N64", c, 128, 0);
        run<3, 128>("mma SS N128", c, 128, 0);
        run<3, 256>("mma SS N256", c, 128, 0);
        run<4, 32>("mma TS N32", c, 128, 0);
        run<4, 64>("mma TS N64", c, 128, 0);
        run<4, 128>("mma TS N128", c, 128, 0);
        run<5, 64>("mix SS N64 + ldtm + sts", c, 128, 4);
    }
    return 0;
}
