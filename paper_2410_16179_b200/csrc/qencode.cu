// qencode.cu -- query SimHash, Alg. 1 "q_code = Encode(q, W)".
// qbar = [q, 0] (reading R4): only the first 128 rows of W meet non-zero
// query entries.  Bit j = [exact(q . W_j) > 0] (R6).
//
// fp64 accumulation of exact bf16 x bf16 products; the sign is certified when
// |acc| > 2^-44 * sum|q_d W_dj| (the fp64 summation error bound is
// 127 * 2^-53 * sum|.|); otherwise (never observed in practice) an exact
// integer dot decides.
#include "common.cuh"
#include "kernels.cuh"

namespace mp {

constexpr int QE_HEADS = 4;
constexpr int QE_COLS = 128;

// CTA = 128 columns x 4 query heads, 256 threads: thread (column c, half hf)
// accumulates d in [64 hf, 64 hf + 64) from a W tile staged in shared memory.
__global__ void __launch_bounds__(256) qencode_kernel(const uint16_t* __restrict__ q, int64_t BHq,
                                                      const float* __restrict__ W, int KL, int KLw,
                                                      uint32_t* __restrict__ qbits, uint32_t* status) {
    // let the dependent decode kernel launch now: it streams codes while we encode
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ __align__(16) float ws[];  // [HD][QE_COLS]
    __shared__ double qd[HD][QE_HEADS];
    __shared__ float qa[HD][QE_HEADS];
    __shared__ double pacc[QE_COLS][QE_HEADS];
    __shared__ float pbnd[QE_COLS][QE_HEADS];
    const int tid = threadIdx.x;
    const int j0 = blockIdx.x * QE_COLS;
    const int64_t h0 = (int64_t)blockIdx.y * QE_HEADS;
    // stage W[:, j0 : j0+128] (zero beyond KL)
    if ((KL & 3) == 0 && j0 + QE_COLS <= KL) {
        for (int e = tid; e < HD * QE_COLS / 4; e += 256) {
            const int d = e / (QE_COLS / 4), c4 = e % (QE_COLS / 4);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(ws + d * QE_COLS + c4 * 4)),
                         "l"(W + (int64_t)d * KL + j0 + c4 * 4)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    } else {
        for (int e = tid; e < HD * QE_COLS; e += 256) {
            const int d = e / QE_COLS, c = e % QE_COLS;
            ws[e] = (j0 + c < KL) ? __ldg(W + (int64_t)d * KL + j0 + c) : 0.0f;
        }
    }
    for (int e = tid; e < HD * QE_HEADS; e += 256) {
        const int h = e / HD, d = e % HD;
        const float f = (h0 + h < BHq) ? bf2f(q[(h0 + h) * HD + d]) : 0.0f;
        qd[d][h] = (double)f;
        qa[d][h] = fabsf(f);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int c = tid & (QE_COLS - 1), hf = tid >> 7;
    double acc[QE_HEADS] = {0.0, 0.0, 0.0, 0.0};
    float bnd[QE_HEADS] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 8
    for (int dd = 0; dd < HD / 2; dd++) {
        const int d = hf * (HD / 2) + dd;
        const float w = ws[d * QE_COLS + c];
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
    if (hf == 1) {
#pragma unroll
        for (int h = 0; h < QE_HEADS; h++) {
            pacc[c][h] = acc[h];
            pbnd[c][h] = bnd[h];
        }
    }
    __syncthreads();
    if (hf == 1) return;
    const int j = j0 + c;
    const bool live = j < KL;
#pragma unroll
    for (int h = 0; h < QE_HEADS; h++) {
        const double s = acc[h] + pacc[c][h];
        const float bb = bnd[h] + pbnd[c][h];
        int bit;
        // |error| <= 127 * 2^-53 * sum|q_d W_dj| < 2^-44 * bnd (bnd in fp32, rel. err < 2^-16)
        if (fabs(s) > 0x1p-44 * (double)bb) {
            bit = s > 0.0;
        } else if (!live || h0 + h >= BHq) {
            bit = 0;
        } else {
            uint16_t xa[HD], wb[HD];
            for (int d = 0; d < HD; d++) {
                xa[d] = q[(h0 + h) * HD + d];
                wb[d] = (uint16_t)(__float_as_uint(W[(int64_t)d * KL + j]) >> 16);
            }
            bit = exact_dot_sign_bf16(xa, wb, HD, status) > 0;
        }
        const uint32_t word = __ballot_sync(0xffffffffu, bit);
        if ((tid & 31) == 0 && h0 + h < BHq && (j >> 5) < KLw) qbits[(h0 + h) * KLw + (j >> 5)] = word;
    }
}

int launch_qencode(const uint16_t* q, int64_t BHq, const float* W, int KL, int KLw, uint32_t* qbits,
                   uint32_t* status, cudaStream_t st) {
    const size_t smem = (size_t)HD * QE_COLS * 4;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(qencode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return MAGICPIG_ECUDA;
        attr = true;
    }
    dim3 grid((unsigned)((KL + QE_COLS - 1) / QE_COLS), (unsigned)((BHq + QE_HEADS - 1) / QE_HEADS));
    qencode_kernel<<<grid, 256, smem, st>>>(q, BHq, W, KL, KLw, qbits, status);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

}  // namespace mp
