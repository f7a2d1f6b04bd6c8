// qencode.cu -- query SimHash, Alg. 1 "q_code = Encode(q, W)".
// qbar = [q, 0] (reading R4): only the first 128 rows of W meet non-zero
// query entries.  Bit j = [exact(q . W_j) > 0] (R6).
//
// fp64 accumulation of exact bf16 x bf16 products; the sign is certified when
// |acc| > 2^-44 * sum|q_d W_dj| (the fp64 summation error bound is
// 127 * 2^-53 * sum|.|); otherwise (never observed in practice) an exact
// integer dot decides.  Thread = one column j, 8 query heads per CTA.
#include "common.cuh"
#include "kernels.cuh"

namespace mp {

constexpr int QE_HEADS = 4;

__global__ void __launch_bounds__(128) qencode_kernel(const uint16_t* __restrict__ q, int64_t BHq,
                                                      const float* __restrict__ W, int KL, int KLw,
                                                      uint32_t* __restrict__ qbits, uint32_t* status) {
    __shared__ double qd[HD][QE_HEADS];
    __shared__ float qa[HD][QE_HEADS];
    const int tid = threadIdx.x;
    const int j = blockIdx.x * 128 + tid;
    const int64_t h0 = (int64_t)blockIdx.y * QE_HEADS;
    for (int e = tid; e < HD * QE_HEADS; e += 128) {
        int h = e / HD, d = e % HD;
        float f = (h0 + h < BHq) ? bf2f(q[(h0 + h) * HD + d]) : 0.0f;
        qd[d][h] = (double)f;
        qa[d][h] = fabsf(f);
    }
    __syncthreads();
    double acc[QE_HEADS];
    float bnd[QE_HEADS];
#pragma unroll
    for (int h = 0; h < QE_HEADS; h++) {
        acc[h] = 0.0;
        bnd[h] = 0.0f;
    }
    const bool live = j < KL;
    const float* wp = W + (live ? j : 0);
#pragma unroll 8
    for (int d = 0; d < HD; d++) {
        const float w = live ? __ldg(wp + (int64_t)d * KL) : 0.0f;
        const double2 q01 = *reinterpret_cast<const double2*>(&qd[d][0]);
        const double2 q23 = *reinterpret_cast<const double2*>(&qd[d][2]);
        const float4 aq = *reinterpret_cast<const float4*>(&qa[d][0]);
        const double wd = (double)w;
        const float wa = fabsf(w);
        acc[0] = fma(q01.x, wd, acc[0]);
        acc[1] = fma(q01.y, wd, acc[1]);
        acc[2] = fma(q23.x, wd, acc[2]);
        acc[3] = fma(q23.y, wd, acc[3]);
        bnd[0] = fmaf(aq.x, wa, bnd[0]);
        bnd[1] = fmaf(aq.y, wa, bnd[1]);
        bnd[2] = fmaf(aq.z, wa, bnd[2]);
        bnd[3] = fmaf(aq.w, wa, bnd[3]);
    }
#pragma unroll
    for (int h = 0; h < QE_HEADS; h++) {
        int bit;
        if (fabs(acc[h]) > 0x1p-44 * (double)bnd[h]) {
            bit = acc[h] > 0.0;
        } else if (!live || h0 + h >= BHq) {
            bit = 0;
        } else {
            uint16_t a[HD], b[HD];
            for (int d = 0; d < HD; d++) {
                a[d] = q[(h0 + h) * HD + d];
                b[d] = (uint16_t)(__float_as_uint(W[(int64_t)d * KL + j]) >> 16);
            }
            bit = exact_dot_sign_bf16(a, b, HD, status) > 0;
        }
        uint32_t word = __ballot_sync(0xffffffffu, bit);
        if ((tid & 31) == 0 && h0 + h < BHq && (j >> 5) < KLw) qbits[(h0 + h) * KLw + (j >> 5)] = word;
    }
}

int launch_qencode(const uint16_t* q, int64_t BHq, const float* W, int KL, int KLw, uint32_t* qbits,
                   uint32_t* status, cudaStream_t st) {
    dim3 grid((unsigned)((KL + 127) / 128), (unsigned)((BHq + QE_HEADS - 1) / QE_HEADS));
    qencode_kernel<<<grid, 128, 0, st>>>(q, BHq, W, KL, KLw, qbits, status);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

}  // namespace mp
