// qencode.cu -- query SimHash, Alg. 1 "q_code = Encode(q, W)".
// qbar = [q, 0] (reading R4): only the first 128 rows of W meet non-zero
// query entries.  Bit j = [exact(q . W_j) > 0] (R6).
//
// A small dense contraction Q [B*Hq][128] x W [128][K*L] on tensor cores
// (mma.sync bf16: every product q_d W_dj is exact, fp32 accumulate).  The same
// contraction of |q| and |W| bounds sum_d |q_d W_dj|; a sign is certified when
// |acc| > 2^-16 * bound (the fp32 tensor-core accumulation error over 8 k-steps
// is below 2^-19 of the bound), otherwise the thread recomputes that dot in
// fp64 (certified at 2^-44) and, failing that, in exact integers.
//
// CTA = 32 columns (one packed query-code word) x 128 query heads; warp w owns
// heads 16w .. 16w+15 (one m16 tile) and all 4 n8 tiles.  W is read once per
// CTA (fp32 -> bf16, exact by the bf16-representable contract) and staged
// column-major in shared memory; q fragments come straight from global memory.
#include "common.cuh"
#include "kernels.cuh"

namespace mp {

constexpr int QE_COLS = 32;    // columns per CTA = one qbits word
constexpr int QE_HEADS = 128;  // query heads per CTA
constexpr int QE_THREADS = 256;
constexpr int QE_WP = HD + 8;  // smem pitch (bf16) of a staged W column: conflict-free fragment loads

__device__ __forceinline__ void qe_mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// rare: the dot recomputed in fp64 (certified at 2^-44), then exactly; out of line so that the hot path of
// the encode stays small in the instruction cache
__device__ __noinline__ int qe_slow_sign(const uint16_t* __restrict__ qh, const uint16_t* wcol, uint32_t* status) {
    double sd = 0.0, bd = 0.0;
    for (int d = 0; d < HD; d++) {
        const double pq = (double)bf2f(qh[d]) * (double)bf2f(wcol[d]);
        sd += pq;
        bd += fabs(pq);
    }
    if (fabs(sd) > 0x1p-44 * bd) return sd > 0.0;
    uint16_t xa[HD], wv[HD];
    for (int d = 0; d < HD; d++) {
        xa[d] = qh[d];
        wv[d] = wcol[d];
    }
    return exact_dot_sign_bf16(xa, wv, HD, status) > 0;
}
// the ln u table (once per (K, L, min_collisions)), out of line for the same reason
__device__ __noinline__ void qe_fill_lut(float* lutab, int K, int L, int minc) {
    const int nb = gridDim.x * gridDim.y, bid = blockIdx.y * gridDim.x + blockIdx.x;
    for (int i = bid * QE_THREADS + threadIdx.x; i <= LUT_N; i += nb * QE_THREADS)
        lutab[i] = (float)log_sampling_prob_d((double)LUT_P0 + (double)i * (1.0 - (double)LUT_P0) / LUT_N, K, L, minc);
}

__global__ void __launch_bounds__(QE_THREADS) qencode_kernel(const uint16_t* __restrict__ q, int64_t BHq,
                                                             const float* __restrict__ W, int KL, int KLw,
                                                             uint32_t* __restrict__ qbits, uint32_t* status,
                                                             int K, int L, int minc, float* __restrict__ lutab) {
    // let the dependent Query kernel launch now (it waits for the codes with griddepcontrol.wait)
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ __align__(16) uint16_t wsm[QE_COLS][QE_WP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j0 = blockIdx.x * QE_COLS;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int64_t hbase = (int64_t)blockIdx.y * QE_HEADS + warp * 16;
    const int64_t ha = hbase + g4, hb = hbase + g4 + 8;
    const uint32_t* qa = reinterpret_cast<const uint32_t*>(q + (ha < BHq ? ha : 0) * HD);
    const uint32_t* qb = reinterpret_cast<const uint32_t*>(q + (hb < BHq ? hb : 0) * HD);
    uint32_t af[8][4];
    {   // W[d][j0 .. j0+31] -> bf16, column-major in smem (all 16 loads per thread in flight first)
        constexpr int NL = HD * QE_COLS / QE_THREADS;
        float wv[NL];
#pragma unroll
        for (int i = 0; i < NL; i++) {
            const int e = tid + i * QE_THREADS, d = e / QE_COLS, c = e % QE_COLS;
            wv[i] = (j0 + c < KL) ? __ldg(W + (int64_t)d * KL + j0 + c) : 0.0f;
        }
        // q fragments: loads in flight together with W's (one global latency)
#pragma unroll
        for (int ks = 0; ks < 8; ks++) {
            const int w0 = (16 * ks + 2 * t4) >> 1;
            af[ks][0] = ha < BHq ? __ldg(qa + w0) : 0u;
            af[ks][1] = hb < BHq ? __ldg(qb + w0) : 0u;
            af[ks][2] = ha < BHq ? __ldg(qa + w0 + 4) : 0u;
            af[ks][3] = hb < BHq ? __ldg(qb + w0 + 4) : 0u;
        }
#pragma unroll
        for (int i = 0; i < NL; i++) {
            const int e = tid + i * QE_THREADS, d = e / QE_COLS, c = e % QE_COLS;
            wsm[c][d] = (uint16_t)(__float_as_uint(wv[i]) >> 16);  // exact: W is bf16-representable
        }
    }
    __syncthreads();
    float acc[4][4], bnd[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; nt++)
#pragma unroll
        for (int i = 0; i < 4; i++) acc[nt][i] = bnd[nt][i] = 0.0f;
#pragma unroll
    for (int ks = 0; ks < 8; ks++) {
        uint32_t aa[4];
#pragma unroll
        for (int i = 0; i < 4; i++) aa[i] = af[ks][i] & 0x7fff7fffu;  // |q| (exact)
#pragma unroll
        for (int nt = 0; nt < 4; nt++) {
            const uint16_t* wc = &wsm[nt * 8 + g4][16 * ks + 2 * t4];
            const uint32_t b0 = *reinterpret_cast<const uint32_t*>(wc);
            const uint32_t b1 = *reinterpret_cast<const uint32_t*>(wc + 8);
            qe_mma(acc[nt], af[ks], b0, b1);
            qe_mma(bnd[nt], aa, b0 & 0x7fff7fffu, b1 & 0x7fff7fffu);
        }
    }
    // bits: element (row, col) = (g4 | g4 + 8, nt * 8 + 2 t4 + i) in acc[nt][(row >= 8) * 2 + i]
    uint32_t wa = 0u, wb = 0u;
#pragma unroll
    for (int nt = 0; nt < 4; nt++) {
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const int col = nt * 8 + 2 * t4 + (e & 1);
            const int64_t h = (e >> 1) ? hb : ha;
            const bool live = j0 + col < KL && h < BHq;
            const float s = acc[nt][e];
            int bit = s > 0.0f;
#ifndef MP_QE_CERT
#define MP_QE_CERT 0x1p-16f
#endif
            if (live && !(fabsf(s) > MP_QE_CERT * bnd[nt][e])) {
                bit = qe_slow_sign(q + h * HD, wsm[col], status);
            }
            if (bit && live) {
                if (e >> 1) wb |= 1u << col;
                else wa |= 1u << col;
            }
        }
    }
    wa |= __shfl_xor_sync(0xffffffffu, wa, 1);
    wa |= __shfl_xor_sync(0xffffffffu, wa, 2);
    wb |= __shfl_xor_sync(0xffffffffu, wb, 1);
    wb |= __shfl_xor_sync(0xffffffffu, wb, 2);
    if (t4 == 0) {
        if (ha < BHq) qbits[ha * KLw + (j0 >> 5)] = wa;
        if (hb < BHq) qbits[hb * KLw + (j0 >> 5)] = wb;
    }
    __shared__ int lut_todo;
    // the previous grid in the stream must be complete before this one is (see launch_qencode)
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifndef MP_QE_LUTCHK
#define MP_QE_LUTCHK 1
#endif
    if (lutab && (MP_QE_LUTCHK || (blockIdx.x == 0 && blockIdx.y == 0))) {  // after the codes: off the Query kernel's critical path until this grid completes
        // the estimator's ln u(p) table (Eq.) in fp64, spread over the CTAs; kept in the workspace
        // and refilled only when (K, L, min_collisions) change: header word = key, next word = arrivals
        uint32_t* hdr = reinterpret_cast<uint32_t*>(lutab + LUT_N + 2);
        const uint32_t want = 1u + (((uint32_t)K * 2048u + (uint32_t)L) << 1) + (uint32_t)(minc - 1);
        if (threadIdx.x == 0) lut_todo = __ldcg(hdr) != want;
        __syncthreads();
        if (lut_todo) {
            const int nb = gridDim.x * gridDim.y;
            qe_fill_lut(lutab, K, L, minc);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                if (atomicAdd(hdr + 1, 1u) == (uint32_t)nb - 1) {  // last CTA: the table is complete
                    hdr[1] = 0u;
                    __threadfence();
                    atomicExch(hdr, want);
                }
            }
        }
    }
}

#ifndef MP_QE_PDL
#define MP_QE_PDL 0
#endif
int launch_qencode(const uint16_t* q, int64_t BHq, const float* W, int KL, int KLw, uint32_t* qbits,
                   uint32_t* status, cudaStream_t st, int K, int L, int minc, float* lutab) {
    // PDL: the encode may start while the previous kernel in the stream (the previous decode's merge) runs;
    // it touches nothing that kernel reads, and it waits for that grid before it completes, so everything
    // after the encode stays ordered after the previous decode
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)KLw, (unsigned)((BHq + QE_HEADS - 1) / QE_HEADS));
    cfg.blockDim = dim3(QE_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = MP_QE_PDL;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, qencode_kernel, q, BHq, W, KL, KLw, qbits, status, K, L, minc, lutab);
    count_launch(1);
    return e == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

}  // namespace mp
