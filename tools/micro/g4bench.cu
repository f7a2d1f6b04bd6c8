// Throughput of random-row gathers into shared memory on B200: TMA gather4 (box 64 cols x 1 row, 128B
// swizzle, 4 rows per instruction) vs 1-D cp.async.bulk of whole 256-B rows.  One CTA per SM, one warp
// issuing, NS stages of 128 rows x 256 B; rows drawn at random (3% density, sorted) from a 1 GiB tensor.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o g4bench g4bench.cu
#include <cuda.h>
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>

#include "../../paper_2410_16179_b200/csrc/common.cuh"

using namespace mp;

constexpr int TR = 128, NS = 3;

__device__ __forceinline__ void tma_gather4(const CUtensorMap* map, uint32_t dst, uint64_t* bar, int col, int r0,
                                            int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7];" ::"r"(dst),
        "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_prefetch4(const CUtensorMap* map, int col, int r0, int r1, int r2, int r3) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile::gather4 [%0, {%1, %2, %3, %4, %5}];" ::"l"(map),
                 "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                 : "memory");
}
__device__ __forceinline__ void bulk_prefetch(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

// MODE 2: cp.async 16 B (LSU path) into the 128B-swizzled tile; WARPS warps issue, 32*WARPS arrivals per stage
template <int WARPS, int PF = 0>
__global__ void __launch_bounds__(32 * WARPS, 1) gbench_cp(const uint16_t* base, const int* idx, int tiles_per_cta,
                                                           unsigned* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NS * 32768);
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid < NS) mbar_init(&bar[tid], 32 * WARPS);
    fence_mbar_init();
    __syncthreads();
    const int* my = idx + (size_t)blockIdx.x * tiles_per_cta * TR;
    unsigned acc = 0;
    for (int t = 0; t < tiles_per_cta + NS; t++) {
        if (t >= NS) {
            const int s = (t - NS) % NS;
            mbar_wait(&bar[s], (uint32_t)(((t - NS) / NS) & 1));
            acc += reinterpret_cast<unsigned*>(sm + s * 32768)[lane];
        }
        if (PF > 0 && t + PF < tiles_per_cta) {  // L2 prefetch (LSU path) of the rows PF tiles ahead
            const int* r = my + (t + PF) * TR;
            for (int c = tid; c < TR * 2; c += 32 * WARPS)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (size_t)r[c >> 1] * 128 + (c & 1) * 64));
        }
        if (t < tiles_per_cta) {
            const int s = t % NS;
            const uint32_t dst = smem_u32(sm + s * 32768);
            const int* r = my + t * TR;
            // 128 rows x 16 chunks; thread handles chunks tid, tid + 32*WARPS, ...
            for (int c = tid; c < TR * 16; c += 32 * WARPS) {
                const int row = c >> 4, j = c & 15, h = j >> 3, jl = j & 7;
                const uint32_t d = dst + h * 16384 + row * 128 + ((jl ^ (row & 7)) << 4);
                cp16(d, base + (size_t)r[row] * 128 + j * 8);
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar[s])) : "memory");
        }
    }
    if (acc == 0x12345u) sink[0] = acc;
}

template <int MODE, int PF>
__global__ void __launch_bounds__(32, 1) gbench(const __grid_constant__ CUtensorMap map, const uint16_t* base,
                                                const int* idx, int tiles_per_cta, unsigned* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NS * 32768);
    const int lane = threadIdx.x;
    if (lane < NS) mbar_init(&bar[lane], 1);
    fence_mbar_init();
    __syncwarp();
    const int* my = idx + (size_t)blockIdx.x * tiles_per_cta * TR;
    unsigned acc = 0;
    for (int t = 0; t < tiles_per_cta + NS; t++) {
        if (t >= NS) {  // consume tile t - NS
            const int s = (t - NS) % NS;
            mbar_wait(&bar[s], (uint32_t)(((t - NS) / NS) & 1));
            acc += reinterpret_cast<unsigned*>(sm + s * 32768)[lane];
            __syncwarp();
        }
        if (PF > 0 && t + PF < tiles_per_cta) {  // L2 prefetch PF tiles ahead
            const int* r = my + (t + PF) * TR;
            if (MODE == 0) {
                tma_prefetch4(&map, 0, r[4 * lane], r[4 * lane + 1], r[4 * lane + 2], r[4 * lane + 3]);
                tma_prefetch4(&map, 64, r[4 * lane], r[4 * lane + 1], r[4 * lane + 2], r[4 * lane + 3]);
            } else {
                for (int i = 0; i < 4; i++) bulk_prefetch(base + (size_t)r[lane * 4 + i] * 128, 256);
            }
        }
        if (t < tiles_per_cta) {
            const int s = t % NS;
            const uint32_t dst = smem_u32(sm + s * 32768);
            const int* r = my + t * TR;
            if (lane == 0) mbar_arrive_expect_tx(&bar[s], TR * 256);
            __syncwarp();
            if (MODE == 0) {  // gather4: lane = row group of 4, both halves
                tma_gather4(&map, dst + lane * 512, &bar[s], 0, r[4 * lane], r[4 * lane + 1], r[4 * lane + 2],
                            r[4 * lane + 3]);
                tma_gather4(&map, dst + 16384 + lane * 512, &bar[s], 64, r[4 * lane], r[4 * lane + 1], r[4 * lane + 2],
                            r[4 * lane + 3]);
            } else {  // 1-D bulk copy of whole rows: 4 per lane
                for (int i = 0; i < 4; i++)
                    bulk_g2s(sm + s * 32768 + (lane * 4 + i) * 256, base + (size_t)r[lane * 4 + i] * 128, 256, &bar[s]);
            }
        }
    }
    if (acc == 0x12345u) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const long long rows = 4LL << 20;  // 64 units x 65536 keys x 256 B = 1 GiB (C3 K cache)
    uint16_t* base;
    cudaMalloc(&base, rows * 256);
    cudaMemset(base, 1, rows * 256);
    const int tiles = 24;
    const int nc = 148;
    std::mt19937_64 rng(3);
    // C3-like sample: 3.3% of the keys of every unit, ascending, concatenated; CTA c takes a contiguous range
    std::vector<int> all;
    for (long long r = 0; r < rows; r++)
        if (rng() % 1000 < 33) all.push_back((int)r);
    std::vector<int> idx((size_t)nc * tiles * TR);
    for (size_t i = 0; i < idx.size(); i++) idx[i] = all[i % all.size()];
    int* didx;
    unsigned* sink;
    cudaMalloc(&didx, idx.size() * 4);
    cudaMalloc(&sink, 64);
    cudaMemcpy(didx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
    CUtensorMap m;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows}, strides[1] = {256};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = NS * 32768 + 64;
    cudaFuncSetAttribute(gbench<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gbench<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gbench<0, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gbench<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gbench<0, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaFuncSetAttribute(gbench_cp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gbench_cp<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gbench_cp<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gbench_cp<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gbench_cp<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gbench_cp<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[11] = {"gather4", "bulk256", "gather4+pf4", "bulk256+pf4", "gather4+pf8", "cp16 x1 warp",
                            "cp16 x4 warps", "cp16 x8 warps", "cp16 x8 +pf2", "cp16 x8 +pf4", "cp16 x4 +pf4"};
    for (int mode = 5; mode < 11; mode++) {
        for (int rep = 0; rep < 3; rep++) {
            cudaMemset(base, rep, 256 << 20);  // evict L2
            cudaEventRecord(e0);
            if (mode == 0) gbench<0, 0><<<nc, 32, smem>>>(m, base, didx, tiles, sink);
            else if (mode == 1) gbench<1, 0><<<nc, 32, smem>>>(m, base, didx, tiles, sink);
            else if (mode == 2) gbench<0, 4><<<nc, 32, smem>>>(m, base, didx, tiles, sink);
            else if (mode == 3) gbench<1, 4><<<nc, 32, smem>>>(m, base, didx, tiles, sink);
            else if (mode == 4) gbench<0, 8><<<nc, 32, smem>>>(m, base, didx, tiles, sink);
            else if (mode == 5) gbench_cp<1><<<nc, 32, smem>>>(base, didx, tiles, sink);
            else if (mode == 6) gbench_cp<4><<<nc, 128, smem>>>(base, didx, tiles, sink);
            else if (mode == 7) gbench_cp<8><<<nc, 256, smem>>>(base, didx, tiles, sink);
            else if (mode == 8) gbench_cp<8, 2><<<nc, 256, smem>>>(base, didx, tiles, sink);
            else if (mode == 9) gbench_cp<8, 4><<<nc, 256, smem>>>(base, didx, tiles, sink);
            else gbench_cp<4, 4><<<nc, 128, smem>>>(base, didx, tiles, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = (double)nc * tiles * TR * 256;
            printf("%s rep %d: %.1f us  %.2f TB/s  (%s)\n", names[mode], rep, ms * 1e3,
                   bytes / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
