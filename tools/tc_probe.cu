// tc_probe.cu -- standalone check of the tcgen05 3xTF32 fused-gate mechanics
// (tc_common.cuh): Y[s] = U x[s] for 256 subvectors of 16 complex amplitudes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tc_probe.cu -o /tmp/tc_probe
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>
#include <complex>

#include "../paper_2111_02396_b200/csrc/tc_common.cuh"

using namespace qt::tc;

__global__ void __launch_bounds__(128) probe(const float2* __restrict__ X, const uint32_t* __restrict__ Wg,
                                             float2* __restrict__ Y, int variant) {
    __shared__ __align__(1024) uint32_t wsm[2 * 32 * 32];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 2 * 32 * 32; i += 128) wsm[i] = Wg[i];
    if (warp == 0) tmem_alloc(&tbase, 256);
    if (tid == 0) { mbar_init(&mbar, 1); fence_mbar_init(); }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tb = tbase;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    // A rows: row = tid (group 0) and tid + 128 (group 1)
    for (int g = 0; g < 2; ++g) {
        uint32_t hi[32], lo[32];
        for (int c = 0; c < 16; ++c) {
            float2 v = X[(g * 128 + tid) * 16 + c];
            float vv[2] = {v.x, v.y};
            for (int a = 0; a < 2; ++a) {
                uint32_t h = tf32_rna(vv[a]);
                float l = vv[a] - __uint_as_float(h);
                hi[2 * c + a] = h;
                lo[2 * c + a] = tf32_rna(l);
            }
        }
        tmem_st32(tb + lane_off + 64 + 32 * g, hi);   // Ahi_g at cols 64 + 32 g
        tmem_st32(tb + lane_off + 128 + 32 * g, lo);  // Alo_g at cols 128 + 32 g
    }
    tmem_wait_st();
    fence_proxy_async();
    fence_before();
    __syncthreads();
    if (tid == 0) {
        fence_after();
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(wsm);
        for (int g = 0; g < 2; ++g) {
            const uint32_t d = tb + 32 * g;
            for (int ks = 0; ks < 4; ++ks) {
                const uint64_t bh = smem_desc_sw128(sb + ks * 32);
                const uint64_t bl = smem_desc_sw128(sb + kWBytes + ks * 32);
                mma_tf32_ts(d, tb + 64 + 32 * g + ks * 8, bh, ks > 0);
                if (variant >= 1) mma_tf32_ts(d, tb + 128 + 32 * g + ks * 8, bh, 1);
                if (variant >= 2) mma_tf32_ts(d, tb + 64 + 32 * g + ks * 8, bl, 1);
            }
        }
        mma_commit(&mbar);
    }
    __syncwarp();
    mbar_wait(&mbar, 0);
    fence_after();
    for (int g = 0; g < 2; ++g) {
        uint32_t v[32];
        tmem_ld32(tb + lane_off + 32 * g, v);
        tmem_wait_ld();
        for (int j = 0; j < 16; ++j)
            Y[(g * 128 + tid) * 16 + j] = make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tb, 256);
}

static uint32_t tf32_host(float x) {  // round to nearest (ties away) at 13 dropped bits
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x1000u) & ~0x1FFFu;
    return u;
}

int main() {
    srand(7);
    auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
    std::vector<std::complex<double>> U(256);
    for (auto& u : U) u = {rnd() * 0.25, rnd() * 0.25};
    std::vector<float2> X(256 * 16);
    for (auto& x : X) x = make_float2(rnd(), rnd());
    // W[k = 2c + a][n = 2j + b]: real 2x2 block of U[j][c]
    std::vector<uint32_t> W(2 * 32 * 32, 0);
    for (int c = 0; c < 16; ++c)
        for (int j = 0; j < 16; ++j) {
            const double ur = U[j * 16 + c].real(), ui = U[j * 16 + c].imag();
            const double blk[2][2] = {{ur, ui}, {-ui, ur}};  // [a][b]: (re_in,re_out) ur, (re_in,im_out) ui, (im_in,re_out) -ui, (im_in,im_out) ur
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b) {
                    const int k = 2 * c + a, n = 2 * j + b;
                    const float w = (float)blk[a][b];
                    const uint32_t h = tf32_host(w);
                    float hf;
                    memcpy(&hf, &h, 4);
                    const uint32_t l = tf32_host(w - hf);
                    W[w_offset_bytes(n, k) / 4] = h;
                    W[(kWBytes + w_offset_bytes(n, k)) / 4] = l;
                }
        }
    float2 *dX, *dY;
    uint32_t* dW;
    cudaMalloc(&dX, X.size() * 8);
    cudaMalloc(&dY, X.size() * 8);
    cudaMalloc(&dW, W.size() * 4);
    cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 3; ++variant) {
        cudaMemset(dY, 0, X.size() * 8);
        probe<<<1, 128>>>(dX, dW, dY, variant);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<float2> Y(X.size());
        cudaMemcpy(Y.data(), dY, Y.size() * 8, cudaMemcpyDeviceToHost);
        double num = 0, den = 0, mx = 0;
        for (int s = 0; s < 256; ++s)
            for (int j = 0; j < 16; ++j) {
                std::complex<double> acc = 0;
                for (int c = 0; c < 16; ++c)
                    acc += U[j * 16 + c] * std::complex<double>(X[s * 16 + c].x, X[s * 16 + c].y);
                std::complex<double> got(Y[s * 16 + j].x, Y[s * 16 + j].y);
                num += std::norm(got - acc);
                den += std::norm(acc);
                mx = fmax(mx, std::abs(got - acc));
            }
        printf("variant %d (1=+XlWh, 2=+XhWl): rel-L2 %.3e  max abs %.3e\n", variant, sqrt(num / den), mx);
    }
    return 0;
}
