// Building-block check for the tcgen05 estimator (estimate8): TMA gather4 of 128 random K / V rows into
// 128B-swizzled tiles, logits MMA (K-major SW128 A), in-place xbar transform, hashed-dot MMA, PV MMA with
// V^T as an MN-major SW128 A operand and the weights as an MN-major B operand; compared with the CPU.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../include -o tc8 tc8.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <random>
#include <vector>

#include "../../paper_2410_16179_b200/csrc/common.cuh"

using namespace mp;

constexpr int NR = 4096;  // rows in K / V
constexpr int TR = 128;   // rows per tile

struct Args {
    const uint16_t* q;   // [16][128] bf16 (heads padded to 16)
    const float* c;      // [128]
    const uint16_t* w;   // [128 rows][16] bf16 weights
    const int* idx;      // [128]
    float* out_l;        // [128][16]
    float* out_x;        // [128][16]
    float* out_pv;       // [128 d][16]
};

__device__ __forceinline__ void tma_gather4(const CUtensorMap* map, void* dst, uint64_t* bar, int col, int r0, int r1,
                                            int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}

__global__ void __launch_bounds__(192, 1) tc8_kernel(const __grid_constant__ CUtensorMap mapK,
                                                     const __grid_constant__ CUtensorMap mapV, Args a) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* Kt = sm;                 // 2 halves x 16 KB
    uint8_t* Vt = sm + 32768;         // 2 halves x 16 KB
    uint8_t* Qt = sm + 65536;         // 4 KB, K-major no-swizzle
    uint8_t* Wt = sm + 69632;         // 4 KB, MN-major no-swizzle
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 73728);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);
    uint64_t *b_full = bars, *b_l = bars + 1, *b_x = bars + 2, *b_h = bars + 3, *b_w = bars + 4, *b_pv = bars + 5;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        mbar_init(b_full, 1);
        mbar_init(b_l, 1);
        mbar_init(b_x, 1);
        mbar_init(b_h, 1);
        mbar_init(b_w, 1);
        mbar_init(b_pv, 1);
        fence_mbar_init();
    }
    // q tile: (n, k) at (n/8)*2048 + (k/8)*128 + (n%8)*16 + (k%8)*2
    for (int e = tid; e < 16 * 128; e += 192) {
        const int n = e / 128, k = e % 128;
        *reinterpret_cast<uint16_t*>(Qt + (n / 8) * 2048 + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) = a.q[e];
    }
    if (warp == 1) {
        tmem_alloc(tslot, 64);
        tmem_relinquish();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t idesc_kk = umma_idesc_bf16(128, 16);
    const uint32_t idesc_mnmn = umma_idesc_bf16(128, 16) | (1u << 15) | (1u << 16);
    if (warp == 0 && lane == 0) {
        mbar_arrive_expect_tx(b_full, TR * 512);
        for (int g = 0; g < TR / 4; g++) {
            const int* r = a.idx + 4 * g;
            for (int h = 0; h < 2; h++) {
                tma_gather4(&mapK, Kt + h * 16384 + g * 512, b_full, h * 64, r[0], r[1], r[2], r[3]);
                tma_gather4(&mapV, Vt + h * 16384 + g * 512, b_full, h * 64, r[0], r[1], r[2], r[3]);
            }
        }
    } else if (warp == 1 && lane == 0) {
        mbar_wait(b_full, 0);
        tc_fence_after();
        const uint32_t kb = smem_u32(Kt), qb = smem_u32(Qt), vb = smem_u32(Vt), wb = smem_u32(Wt);
        for (int kk = 0; kk < 8; kk++) {  // logits: D0[128 rows][16] = K . Q^T
            const uint64_t ad = desc_sw128(kb + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
            const uint64_t bd = umma_desc(qb + kk * 256, 128, 2048);
            umma_bf16(tmem + 0, ad, bd, idesc_kk, kk > 0);
        }
        umma_commit(b_l);
        mbar_wait(b_x, 0);
        tc_fence_after();
        for (int kk = 0; kk < 8; kk++) {  // hashed dots: D1 = X . Q^T (X in place of K)
            const uint64_t ad = desc_sw128(kb + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024);
            const uint64_t bd = umma_desc(qb + kk * 256, 128, 2048);
            umma_bf16(tmem + 16, ad, bd, idesc_kk, kk > 0);
        }
        umma_commit(b_h);
        mbar_wait(b_w, 0);
        tc_fence_after();
        for (int kk = 0; kk < 8; kk++) {  // PV: D2[128 d][16] = V^T . W  (A MN-major SW128, B MN-major)
            const uint64_t ad = desc_sw128(vb + kk * 2048, 16384, 1024);
            const uint64_t bd = umma_desc(wb + kk * 256, 128, 2048);
            umma_bf16(tmem + 32, ad, bd, idesc_mnmn, kk > 0);
        }
        umma_commit(b_pv);
    } else if (warp >= 2) {
        const int ct = tid - 64;                  // compute thread 0..127
        const int quad = warp & 3;                // TMEM lane quadrant of this warp
        const int row = quad * 32 + lane;         // TMEM lane = tile row (logits) / d (PV)
        const uint32_t tq = tmem + ((uint32_t)(quad * 32) << 16);
        mbar_wait(b_l, 0);
        tc_fence_after();
        float v[16];
        tmem_ld16(tq + 0, v);
        for (int n = 0; n < 16; n++) a.out_l[row * 16 + n] = v[n];
        // in-place xbar = bf16(fl32(k - c)): 16-B chunk j of row r holds logical chunk j ^ (r % 8)
        for (int ch = ct; ch < 2048; ch += 128) {
            const int h = ch / 1024, o = (ch % 1024) * 16, r = o / 128, js = (o % 128) / 16, jl = js ^ (r % 8);
            const int d0 = h * 64 + jl * 8;
            uint4* p = reinterpret_cast<uint4*>(Kt + h * 16384 + o);
            uint4 x = *p;
            uint32_t* w4 = reinterpret_cast<uint32_t*>(&x);
            for (int i = 0; i < 4; i++) {
                const float lo = __uint_as_float(w4[i] << 16) - a.c[d0 + 2 * i];
                const float hi = __uint_as_float(w4[i] & 0xffff0000u) - a.c[d0 + 2 * i + 1];
                const __nv_bfloat162 b2 = __floats2bfloat162_rn(lo, hi);
                w4[i] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            *p = x;
        }
        // W tile (MN-major, no swizzle): (n, k) at (n/8)*2048 + (k/8)*128 + (k%8)*16 + (n%8)*2; k = key row
        for (int e = ct; e < 128 * 16; e += 128) {
            const int k = e / 16, n = e % 16;
            *reinterpret_cast<uint16_t*>(Wt + (n / 8) * 2048 + (k / 8) * 128 + (k % 8) * 16 + (n % 8) * 2) =
                a.w[k * 16 + n];
        }
        fence_proxy_async();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (ct == 0) {
            mbar_arrive(b_x);
            mbar_arrive(b_w);
        }
        mbar_wait(b_h, 0);
        tc_fence_after();
        tmem_ld16(tq + 16, v);
        for (int n = 0; n < 16; n++) a.out_x[row * 16 + n] = v[n];
        mbar_wait(b_pv, 0);
        tc_fence_after();
        tmem_ld16(tq + 32, v);
        for (int n = 0; n < 16; n++) a.out_pv[row * 16 + n] = v[n];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 64);
}

static uint16_t f2bf(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7FFF + ((u >> 16) & 1);
    return (uint16_t)(u >> 16);
}
static float bf2f_h(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    std::mt19937 rng(7);
    std::normal_distribution<float> nd;
    std::vector<uint16_t> K(NR * 128), V(NR * 128), q(16 * 128, 0), w(128 * 16);
    std::vector<float> c(128);
    for (auto& x : K) x = f2bf(nd(rng));
    for (auto& x : V) x = f2bf(nd(rng));
    for (int n = 0; n < 4; n++)
        for (int k = 0; k < 128; k++) q[n * 128 + k] = f2bf(1.5f * nd(rng));
    for (auto& x : c) x = 0.05f * nd(rng);
    for (int r = 0; r < 128; r++)
        for (int n = 0; n < 16; n++) w[r * 16 + n] = n < 8 ? f2bf(std::fabs(nd(rng))) : 0;
    std::vector<int> idx(128);
    for (auto& x : idx) x = rng() % NR;
    uint16_t *dK, *dV, *dq, *dw;
    float *dc, *ol, *ox, *opv;
    int* didx;
    cudaMalloc(&dK, NR * 256);
    cudaMalloc(&dV, NR * 256);
    cudaMalloc(&dq, 16 * 256);
    cudaMalloc(&dw, 128 * 32);
    cudaMalloc(&dc, 512);
    cudaMalloc(&didx, 512);
    cudaMalloc(&ol, 128 * 64);
    cudaMalloc(&ox, 128 * 64);
    cudaMalloc(&opv, 128 * 64);
    cudaMemcpy(dK, K.data(), NR * 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dV, V.data(), NR * 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, q.data(), 16 * 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dw, w.data(), 128 * 32, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, c.data(), 512, cudaMemcpyHostToDevice);
    cudaMemcpy(didx, idx.data(), 512, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
    if (!enc) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    CUtensorMap mK, mV;
    cuuint64_t dims[2] = {128, NR}, strides[1] = {256};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult r1 = enc(&mK, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dK, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(&mV, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dV, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d %d\n", (int)r1, (int)r2);
    Args a{dq, dc, dw, didx, ol, ox, opv};
    const int smem = 73728 + 128;
    cudaFuncSetAttribute(tc8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tc8_kernel<<<1, 192, smem>>>(mK, mV, a);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<float> hl(128 * 16), hx(128 * 16), hpv(128 * 16);
    cudaMemcpy(hl.data(), ol, 128 * 64, cudaMemcpyDeviceToHost);
    cudaMemcpy(hx.data(), ox, 128 * 64, cudaMemcpyDeviceToHost);
    cudaMemcpy(hpv.data(), opv, 128 * 64, cudaMemcpyDeviceToHost);
    double el = 0, ex = 0, epv = 0, ml = 0, mx = 0, mpv = 0;
    for (int r = 0; r < 128; r++)
        for (int n = 0; n < 4; n++) {
            double sl = 0, sx = 0;
            for (int k = 0; k < 128; k++) {
                const float kv = bf2f_h(K[idx[r] * 128 + k]);
                const float xv = bf2f_h(f2bf(kv - c[k]));
                sl += (double)kv * bf2f_h(q[n * 128 + k]);
                sx += (double)xv * bf2f_h(q[n * 128 + k]);
            }
            el = std::max(el, std::fabs(sl - hl[r * 16 + n]));
            ex = std::max(ex, std::fabs(sx - hx[r * 16 + n]));
            ml = std::max(ml, std::fabs(sl));
            mx = std::max(mx, std::fabs(sx));
        }
    for (int d = 0; d < 128; d++)
        for (int n = 0; n < 8; n++) {
            double s = 0;
            for (int r = 0; r < 128; r++) s += (double)bf2f_h(V[idx[r] * 128 + d]) * bf2f_h(w[r * 16 + n]);
            epv = std::max(epv, std::fabs(s - hpv[d * 16 + n]));
            mpv = std::max(mpv, std::fabs(s));
        }
    printf("logits max err %.3g (max %.3g); hashed %.3g (max %.3g); pv %.3g (max %.3g)\n", el, ml, ex, mx, epv, mpv);
    printf("sample logits gpu %f cpu-row0: ", hl[0]);
    double s0 = 0;
    for (int k = 0; k < 128; k++) s0 += (double)bf2f_h(K[idx[0] * 128 + k]) * bf2f_h(q[k]);
    printf("%f\n", s0);
    return (el < 1e-3 * ml && ex < 1e-3 * mx && epv < 1e-3 * mpv) ? 0 : 2;
}
