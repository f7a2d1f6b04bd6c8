// Random-row gather ceiling on B200: rows of 256 B from two 1 GiB tensors (K, V) at the sampled
// density of C3 (3.3% of keys, ascending per unit), vs contiguous rows.  nvcc -O3 -arch=sm_100a.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void gather_ld(const uint4* __restrict__ K, const uint4* __restrict__ V, const int* __restrict__ idx,
                          int nrows, uint4* __restrict__ out) {
    // each half-warp copies one row (16 lanes x 16 B); K and V rows of the same key
    const int lane = threadIdx.x & 31;
    const int hw = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
    const int nhw = (gridDim.x * blockDim.x) >> 4;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int r = hw; r < nrows; r += nhw) {
        const long long row = idx[r];
        const uint4 a = __ldcs(K + row * 16 + (lane & 15));
        const uint4 b = __ldcs(V + row * 16 + (lane & 15));
        acc.x ^= a.x ^ b.x; acc.y ^= a.y ^ b.y; acc.z ^= a.z ^ b.z; acc.w ^= a.w ^ b.w;
    }
    if (acc.x == 0x12345678u) out[0] = acc;
}

template <int UNROLL>
__global__ void gather_ld_u(const uint4* __restrict__ K, const uint4* __restrict__ V, const int* __restrict__ idx,
                            int nrows, uint4* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int hw = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
    const int nhw = (gridDim.x * blockDim.x) >> 4;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int r0 = hw; r0 < nrows; r0 += nhw * UNROLL) {
        uint4 a[UNROLL], b[UNROLL];
#pragma unroll
        for (int j = 0; j < UNROLL; j++) {
            const int r = r0 + j * nhw;
            const long long row = r < nrows ? idx[r] : 0;
            a[j] = __ldcs(K + row * 16 + (lane & 15));
            b[j] = __ldcs(V + row * 16 + (lane & 15));
        }
#pragma unroll
        for (int j = 0; j < UNROLL; j++) {
            acc.x ^= a[j].x ^ b[j].x; acc.y ^= a[j].y ^ b[j].y; acc.z ^= a[j].z ^ b[j].z; acc.w ^= a[j].w ^ b[j].w;
        }
    }
    if (acc.x == 0x12345678u) out[0] = acc;
}

int main() {
    const long long units = 64, n = 65536, rows = units * n;
    const size_t bytes = rows * 256;
    uint4 *K, *V, *out;
    cudaMalloc(&K, bytes); cudaMalloc(&V, bytes); cudaMalloc(&out, 64);
    cudaMemset(K, 1, bytes); cudaMemset(V, 2, bytes);
    std::mt19937_64 rng(1);
    for (double dens : {0.033, 0.1, 0.3, 1.0}) {
        std::vector<int> idx;
        for (long long u = 0; u < units; u++)
            for (long long i = 0; i < n; i++)
                if (dens >= 1.0 || (rng() % 1000000) < dens * 1e6) idx.push_back((int)(u * n + i));
        int* d_idx;
        cudaMalloc(&d_idx, idx.size() * 4);
        cudaMemcpy(d_idx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
        const int nr = (int)idx.size();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int variant = 0; variant < 3; variant++) {
            for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
                auto run = [&]() {
                    if (variant == 0) gather_ld<<<blocks, 256>>>(K, V, d_idx, nr, out);
                    else if (variant == 1) gather_ld_u<4><<<blocks, 256>>>(K, V, d_idx, nr, out);
                    else gather_ld_u<8><<<blocks, 256>>>(K, V, d_idx, nr, out);
                };
                run();
                cudaEventRecord(e0);
                for (int it = 0; it < 10; it++) run();
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double us = ms * 1e3 / 10;
                printf("density %.3f rows %d variant %d blocks %d: %.1f us  %.2f TB/s\n", dens, nr, variant, blocks, us,
                       nr * 512.0 / us / 1e6);
            }
        }
        cudaFree(d_idx);
    }
    return 0;
}
