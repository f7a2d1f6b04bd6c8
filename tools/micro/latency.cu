// pointer-chase latency probe: L1, L2 (same/cross die unknown), DRAM; and
// a store-then-load-from-another-SM pattern like the decode's partials.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void chase(const uint32_t* __restrict__ p, int n, int iters, long long* out, uint32_t* sink, int mode) {
    uint32_t j = 0;
    // warm-up pass
    for (int i = 0; i < n; i++) j = mode == 0 ? p[j] : __ldcg(p + j);
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) j = mode == 0 ? p[j] : __ldcg(p + j);
    long long t1 = clock64();
    out[0] = (t1 - t0) / iters;
    sink[0] = j;
}
__global__ void chase_cold(const uint32_t* __restrict__ p, int iters, long long* out, uint32_t* sink) {
    uint32_t j = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) j = __ldcg(p + j);
    long long t1 = clock64();
    out[0] = (t1 - t0) / iters;
    sink[0] = j;
}
__global__ void writer(uint32_t* p, int n, uint32_t stride) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += gridDim.x * blockDim.x) p[i] = (uint32_t)((i + stride) % n);
}
int main() {
    const int N = 1 << 26;  // 256 MB
    uint32_t *p, *sink;
    long long* out;
    cudaMalloc(&p, (size_t)N * 4);
    cudaMalloc(&sink, 64);
    cudaMalloc(&out, 64);
    long long h;
    for (int ws : {4096, 1 << 16, 1 << 20, 1 << 22, 1 << 24, 1 << 26}) {
        uint32_t stride = 64 * 32 + 17;  // jump > 1 line
        writer<<<148, 256>>>(p, ws, stride);
        cudaDeviceSynchronize();
        chase<<<1, 1>>>(p, ws / 64 > 100000 ? 100000 : ws / 64, 20000, out, sink, 1);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("working set %9d B: ldcg latency %lld cycles\n", ws * 4, h);
    }
    // freshly written by many SMs, read by one SM, L2-resident set of 1 MB
    writer<<<148, 256>>>(p, 1 << 18, 4111);
    cudaDeviceSynchronize();
    chase_cold<<<1, 1>>>(p, 5000, out, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("fresh-written 1 MB, first touch by another SM: %lld cycles\n", h);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock %d kHz\n", clk);
    return 0;
}
