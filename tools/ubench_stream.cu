// ubench_stream.cu -- in-place tile streaming through shared memory with 1-D bulk
// copies (cp.async.bulk, UBLKCP): the HBM side of a K1 pass without the gates.
// A tile = 2^TB amplitudes (complex64) spanned by qubits 0..3 (128-byte runs) plus
// TB - 4 higher qubits spread over the register; a persistent CTA per SM walks
// its tiles with S shared-memory stages: warp 0 issues the loads of tile i + S - 1
// and the stores of tile i (each lane 1/32 of the runs; one mbarrier per stage
// completes on the transferred bytes; bulk groups track the stores' shared reads).
// Runs are placed at a 144-byte stride (16-byte skew per run, the bank rotation the
// gate gathers need).  Reports GB/s = 2 x 8 x 2^n / time.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_stream.bin tools/ubench_stream.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

struct Args {
    float2* state;
    int n;
    uint8_t tq[16];  // high tile qubits (tile bits 4..TB-1)
    uint32_t ntiles;
};

template <int TB, int S, int STRIDE, int RUNQ>
__global__ void __launch_bounds__(128, 1) stream(const Args A) {
    constexpr int NR = 1 << (TB - RUNQ);        // runs per tile
    constexpr int RB = 8 << RUNQ;               // bytes per run
    constexpr int STAGE = NR * STRIDE;
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[S];
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t fb = (uint32_t)__cvta_generic_to_shared(full);
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(fb + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (tid >= 32) return;
    // tiles of this CTA: blockIdx.x, + gridDim.x, ...
    auto tile_base = [&](uint32_t t) -> uint64_t {
        uint64_t b = t;
        // insert zeros at qubits 0..RUNQ-1 and at every high tile qubit (ascending)
        b <<= RUNQ;
        for (int i = 0; i < TB - RUNQ; ++i) {
            const uint64_t low = b & ((1ull << A.tq[i]) - 1ull);
            b = low | ((b ^ low) << 1);
        }
        return b;
    };
    auto run_off = [&](int r) -> uint64_t {
        uint64_t o = 0;
        for (int i = 0; i < TB - RUNQ; ++i) o |= (uint64_t)((r >> i) & 1) << A.tq[i];
        return o;
    };
    const int my = (int)((A.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
    auto load = [&](int j) {
        const int s = j % S;
        const uint64_t b = tile_base(blockIdx.x + (uint32_t)j * gridDim.x);
        if (lane == 0) mbar_expect(fb + 8 * s, (uint32_t)(NR * RB));
        __syncwarp();
        for (int r = lane; r < NR; r += 32)
            bulk_g2s(sbase + s * STAGE + r * STRIDE, A.state + b + run_off(r), RB, fb + 8 * s);
    };
    for (int j = 0; j < S - 1 && j < my; ++j) load(j);
    for (int j = 0; j < my; ++j) {
        const int s = j % S;
        mbar_wait(fb + 8 * s, (uint32_t)((j / S) & 1));
        const uint64_t b = tile_base(blockIdx.x + (uint32_t)j * gridDim.x);
        for (int r = lane; r < NR; r += 32) bulk_s2g(A.state + b + run_off(r), sbase + s * STAGE + r * STRIDE, RB);
        bulk_commit();
        bulk_wait_read<1>();  // the stores of tile j - 1 have left stage (j - 1) % S
        __syncwarp();
        if (j + S - 1 < my) load(j + S - 1);
    }
    bulk_wait_all();
}

template <int TB, int S, int STRIDE, int RUNQ>
void run(float2* st, int n, const char* name) {
    Args a;
    a.state = st;
    a.n = n;
    // high tile qubits: spread over RUNQ..n-1
    const int nh = TB - RUNQ;
    for (int i = 0; i < nh; ++i) a.tq[i] = (uint8_t)(RUNQ + (i * (n - RUNQ)) / nh);
    a.ntiles = 1u << (n - TB);
    constexpr int NR = 1 << (TB - RUNQ);
    const size_t smem = (size_t)S * NR * STRIDE;
    cudaFuncSetAttribute(stream<TB, S, STRIDE, RUNQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms = 148;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    stream<TB, S, STRIDE, RUNQ><<<sms, 128, smem>>>(a);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) stream<TB, S, STRIDE, RUNQ><<<sms, 128, smem>>>(a);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        exit(1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double gbs = 2.0 * 8.0 * (double)(1ull << n) / (ms * 1e-3) / 1e9;
    printf("%-34s TB=%d S=%d stride=%d runq=%d smem=%zu KB: %.3f ms  %.0f GB/s  (%.1f%% of 6535)\n", name, TB, S,
           STRIDE, RUNQ, smem >> 10, ms, gbs, 100.0 * gbs / 6534.8);
}

int main() {
    const int n = 30;
    float2* st;
    if (cudaMalloc(&st, (sizeof(float2) << n))) return 1;
    cudaMemset(st, 0, sizeof(float2) << n);
    run<12, 4, 144, 4>(st, n, "12q tile, 4 stages");
    run<12, 6, 144, 4>(st, n, "12q tile, 6 stages");
    run<13, 2, 144, 4>(st, n, "13q tile, 2 stages");
    run<13, 3, 144, 4>(st, n, "13q tile, 3 stages");
    run<13, 3, 128, 4>(st, n, "13q tile, 3 stages, no skew");
    run<12, 3, 144, 4>(st, n, "12q tile, 3 stages");
    run<12, 6, 272, 5>(st, n, "12q tile, 6 stages, 256B runs");
    run<13, 3, 272, 5>(st, n, "13q tile, 3 stages, 256B runs");
    return 0;
}
