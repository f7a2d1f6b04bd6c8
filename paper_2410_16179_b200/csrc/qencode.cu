// qencode.cu -- query SimHash, Alg. 1 "q_code = Encode(q, W)".
// qbar = [q, 0] (reading R4): only the first 128 rows of W meet non-zero
// query entries.  Bit j = [exact(q . W_j) > 0] (R6).
//
// fp32 accumulation of exact bf16 x bf16 products with a certified sign test,
// fp64 and exact-integer fallbacks for the rare near-zero dots (see kernel).
#include "common.cuh"
#include "kernels.cuh"

namespace mp {

constexpr int QE_COLS = 32;   // columns per CTA (one warp-wide ballot word)
constexpr int QE_HPB = 8;     // query heads per CTA
constexpr int QE_THREADS = 256;

// CTA = 32 columns x 8 heads; warp w: heads 4*(w%2) .. +3, d-quarter w/2; lane = column.
// fp32 products are exact (bf16 x bf16); fp32 sums certify the sign when
// |acc| > 2^-16 sum|q_d W_dj| (error <= 65 * 2^-24 * sum|.|); otherwise the
// warp recomputes that dot in fp64 (certified at 2^-44) and, failing that, in
// exact integers.
__global__ void __launch_bounds__(QE_THREADS) qencode_kernel(const uint16_t* __restrict__ q, int64_t BHq,
                                                             const float* __restrict__ W, int KL, int KLw,
                                                             uint32_t* __restrict__ qbits, uint32_t* status) {
    // let the dependent decode kernel launch now: it streams codes while we encode
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ float ws[HD][QE_COLS];
    __shared__ __align__(16) float qs[HD][QE_HPB];
    __shared__ __align__(16) float qa[HD][QE_HPB];
    __shared__ float pacc[3][QE_HPB][QE_COLS], pbnd[3][QE_HPB][QE_COLS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j0 = blockIdx.x * QE_COLS;
    const int64_t h0 = (int64_t)blockIdx.y * QE_HPB;
    {   // all loads in flight before any store (16 W values + 8 q values per thread)
        constexpr int NW = HD * QE_COLS / QE_THREADS, NQ = HD * QE_HPB / QE_THREADS;
        float wv[NW];
        uint16_t qv[NQ];
#pragma unroll
        for (int i = 0; i < NW; i++) {
            const int e = tid + i * QE_THREADS, d = e / QE_COLS, c = e % QE_COLS;
            wv[i] = (j0 + c < KL) ? __ldg(W + (int64_t)d * KL + j0 + c) : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < NQ; i++) {
            const int e = tid + i * QE_THREADS, h = e / HD, d = e % HD;
            qv[i] = (h0 + h < BHq) ? __ldg(q + (h0 + h) * HD + d) : (uint16_t)0;
        }
#pragma unroll
        for (int i = 0; i < NW; i++) {
            const int e = tid + i * QE_THREADS;
            ws[e / QE_COLS][e % QE_COLS] = wv[i];
        }
#pragma unroll
        for (int i = 0; i < NQ; i++) {
            const int e = tid + i * QE_THREADS, h = e / HD, d = e % HD;
            const float f = bf2f(qv[i]);
            qs[d][h] = f;
            qa[d][h] = fabsf(f);
        }
    }
    __syncthreads();
    const int hs = warp & 1, dq = warp >> 1;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f}, bnd[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 16
    for (int dd = 0; dd < HD / 4; dd++) {
        const int d = dq * (HD / 4) + dd;
        const float w = ws[d][lane];
        const float wa = fabsf(w);
        const float4 q4 = *reinterpret_cast<const float4*>(&qs[d][hs * 4]);
        const float4 a4 = *reinterpret_cast<const float4*>(&qa[d][hs * 4]);
        acc[0] = fmaf(q4.x, w, acc[0]);
        acc[1] = fmaf(q4.y, w, acc[1]);
        acc[2] = fmaf(q4.z, w, acc[2]);
        acc[3] = fmaf(q4.w, w, acc[3]);
        bnd[0] = fmaf(a4.x, wa, bnd[0]);
        bnd[1] = fmaf(a4.y, wa, bnd[1]);
        bnd[2] = fmaf(a4.z, wa, bnd[2]);
        bnd[3] = fmaf(a4.w, wa, bnd[3]);
    }
    if (dq > 0) {
#pragma unroll
        for (int t = 0; t < 4; t++) {
            pacc[dq - 1][hs * 4 + t][lane] = acc[t];
            pbnd[dq - 1][hs * 4 + t][lane] = bnd[t];
        }
    }
    __syncthreads();
    if (dq > 0) return;
    const int j = j0 + lane;
    const bool live = j < KL;
#pragma unroll
    for (int t = 0; t < 4; t++) {
        const int h = hs * 4 + t;
        const float s = ((acc[t] + pacc[0][h][lane]) + pacc[1][h][lane]) + pacc[2][h][lane];
        const float bb = ((bnd[t] + pbnd[0][h][lane]) + pbnd[1][h][lane]) + pbnd[2][h][lane];
        int bit = s > 0.0f;
        const bool unsure = live && (h0 + h < BHq) && !(fabsf(s) > 0x1p-16f * bb);
        uint32_t um = __ballot_sync(0xffffffffu, unsure);
        while (um) {  // rare: warp-cooperative fp64 recomputation of column (j0 + src)
            const int src = __ffs(um) - 1;
            um &= um - 1;
            double sd = 0.0, bd = 0.0;
#pragma unroll
            for (int r = 0; r < HD / 32; r++) {
                const int d = lane + 32 * r;
                const double pq = (double)qs[d][h] * (double)ws[d][src];
                sd += pq;
                bd += fabs(pq);
            }
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) {
                sd += __shfl_xor_sync(0xffffffffu, sd, m);
                bd += __shfl_xor_sync(0xffffffffu, bd, m);
            }
            int b2;
            if (fabs(sd) > 0x1p-44 * bd) {
                b2 = sd > 0.0;
            } else {
                b2 = 0;
                if (lane == 0) {
                    uint16_t xa[HD], wb[HD];
                    for (int d = 0; d < HD; d++) {
                        xa[d] = q[(h0 + h) * HD + d];
                        wb[d] = (uint16_t)(__float_as_uint(ws[d][src]) >> 16);
                    }
                    b2 = exact_dot_sign_bf16(xa, wb, HD, status) > 0;
                }
                b2 = __shfl_sync(0xffffffffu, b2, 0);
            }
            if (lane == src) bit = b2;
        }
        const uint32_t word = __ballot_sync(0xffffffffu, bit && live);
        if (lane == 0 && h0 + h < BHq && (j0 >> 5) < KLw) qbits[(h0 + h) * KLw + (j0 >> 5)] = word;
    }
}

int launch_qencode(const uint16_t* q, int64_t BHq, const float* W, int KL, int KLw, uint32_t* qbits,
                   uint32_t* status, cudaStream_t st) {
    dim3 grid((unsigned)((KL + QE_COLS - 1) / QE_COLS), (unsigned)((BHq + QE_HPB - 1) / QE_HPB));
    qencode_kernel<<<grid, QE_THREADS, 0, st>>>(q, BHq, W, KL, KLw, qbits, status);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

}  // namespace mp
