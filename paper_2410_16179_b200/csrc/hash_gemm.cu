// hash_gemm.cu -- key SimHash as a dense contraction on the 5th-gen tensor
// cores ("projected on K directions, only the sign of the
// projection is kept"; Alg. 1 input HT).
//
//   acc[i][j] = xbar_i . W_j   (bf16 x bf16 -> fp32 in TMEM, tcgen05.mma)
//   bit[i][j] = acc > 0, packed by __ballot_sync into bit-plane words
//   |acc| <= eps |xbar_i| max_j |W_j|  ->  (i, j) appended to a fix-up list and
//   recomputed exactly in integers (fixup kernel), so every bit is the sign of
//   the EXACT dot product (reading R6).
//
// CTA = GM_R M=128 key tiles (A operand resident in shared memory) x all K*L columns streamed in
// N = GM_N chunks (bulk-copy ring).  Default GM_N = 128, GM_R = 2 (measured at C3: N = 64 x 4 tiles
// 3908 us, N = 128 x 2 tiles 3266 us).  Warp roles:
//   warp 0: bulk-copy producer (cp.async.bulk + mbarrier complete_tx)
//   warp 1: TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..: epilogue (tcgen05.ld 32x32b -> sign/filter -> ballot -> STG.128),
//              HG_EW / 4 warps per TMEM lane quarter, HG_CW columns each (16 warps x 16 columns
//              by default: the epilogue, not the tensor pipe, paced the 8-warp version)
// TMEM: 2 accumulator stages x (GM_R tiles x GM_N columns) = 512 columns (4 x 64, or 2 x 128 with
// MP_HG_N=128).
#include "common.cuh"
#include "kernels.cuh"

namespace mp {

constexpr int GM_R = HG_R;
constexpr int GM_N = HG_N;
constexpr int GM_STAGES = GM_N >= 256 ? 2 : 3;  // W chunk ring (shared memory: A tiles + stages <= 227 KB)
#ifndef MP_HG_EW
#define MP_HG_EW 16
#endif
constexpr int HG_EW = MP_HG_EW;              // epilogue warps: HG_EW / 4 per TMEM lane quarter
constexpr int HG_CW = GM_N / (HG_EW / 4);    // columns of a chunk per epilogue warp (32 or 16)
constexpr int GM_THREADS = 64 + 32 * HG_EW;  // producer, MMA, epilogue warps
constexpr int HG_SUBW = HG_CW > 16 ? 16 : HG_CW;  // columns per TMEM load (bounds the registers)
constexpr int HG_NSUB = HG_CW / HG_SUBW;
#ifndef MP_HG_RTU
#define MP_HG_RTU 1
#endif
constexpr int HG_RTU = MP_HG_RTU;  // epilogue unroll over the 4 key tiles (code size vs the i-cache)  // producer, MMA, 8 epilogue warps (2 per TMEM lane quarter)

__device__ __forceinline__ void tmem_ldn(uint32_t ta, uint32_t (&v)[32]) { tmem_ld32(ta, v); }
__device__ __forceinline__ void tmem_ldn(uint32_t ta, uint32_t (&v)[16]) { tmem_ld16(ta, v); }

struct GemmParams {
    const uint8_t* xt;
    const uint8_t* wt;
    const float* xnorm;
    const float* wmax;
    uint32_t* codes;
    uint2* fix_list;
    uint32_t* fix_count;
    uint32_t fix_cap;
    int64_t n_local, n_pad, nchunks;
    int KD, KL, NT, KLq;
    uint32_t* status;
    float* dbg_acc;  // debug: raw accumulators of tile 0 of CTA (0,0), [128][KL]
};

size_t gemm_smem_bytes(int KD) {
    return (size_t)GM_R * 128 * KD * 2 + (size_t)GM_STAGES * GM_N * KD * 2 + 256;
}

__global__ void __launch_bounds__(GM_THREADS, 1) hash_gemm_kernel(GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int KD = p.KD;
    const uint32_t a_tile = 128u * KD * 2u;
    const uint32_t b_tile = (uint32_t)GM_N * KD * 2u;
    uint8_t* sA = smem;
    uint8_t* sB = smem + GM_R * a_tile;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + GM_STAGES * b_tile);
    uint64_t* a_full = bars;
    uint64_t* b_full = bars + 1;
    uint64_t* b_empty = bars + 1 + GM_STAGES;
    uint64_t* t_full = bars + 1 + 2 * GM_STAGES;
    uint64_t* t_empty = bars + 3 + 2 * GM_STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5 + 2 * GM_STAGES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t unit = blockIdx.y;
    const int64_t m0 = (int64_t)blockIdx.x * (GM_R * 128);

    if (warp == 0 && lane == 0) {
        mbar_init(a_full, 1);
        for (int s = 0; s < GM_STAGES; s++) {
            mbar_init(b_full + s, 1);
            mbar_init(b_empty + s, 1);
        }
        for (int s = 0; s < 2; s++) {
            mbar_init(t_full + s, 1);
            mbar_init(t_empty + s, HG_EW);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // A: the 4 key tiles of this CTA (consecutive in global memory)
            mbar_arrive_expect_tx(a_full, GM_R * a_tile);
            const uint8_t* asrc = p.xt + (unit * (p.n_pad >> 7) + (m0 >> 7)) * (int64_t)a_tile;
            for (int rt = 0; rt < GM_R; rt++) bulk_g2s(sA + rt * a_tile, asrc + rt * a_tile, a_tile, a_full);
            for (int c = 0; c < p.NT; c++) {
                int s = c % GM_STAGES;
                if (c >= GM_STAGES) mbar_wait(b_empty + s, ((c / GM_STAGES) - 1) & 1);
                mbar_arrive_expect_tx(b_full + s, b_tile);
                bulk_g2s(sB + s * b_tile, p.wt + (int64_t)c * b_tile, b_tile, b_full + s);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = umma_idesc_bf16(128, GM_N);
            const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
            mbar_wait(a_full, 0);
            tc_fence_after();
            for (int c = 0; c < p.NT; c++) {
                int s = c % GM_STAGES, ts = c & 1;
                mbar_wait(b_full + s, (c / GM_STAGES) & 1);
                if (c >= 2) mbar_wait(t_empty + ts, ((c >> 1) - 1) & 1);
                tc_fence_after();
                for (int rt = 0; rt < GM_R; rt++) {
                    for (int ks = 0; ks < KD / 16; ks++) {
                        uint64_t ad = umma_desc(a_base + rt * a_tile + ks * 2 * (16 * 128), 16 * 128, 128);
                        uint64_t bd = umma_desc(b_base + s * b_tile + ks * 2 * ((GM_N / 8) * 128), (GM_N / 8) * 128, 128);
                        umma_bf16(tmem + ts * (GM_R * GM_N) + rt * GM_N, ad, bd, idesc, ks > 0 ? 1u : 0u);
                    }
                }
                umma_commit(b_empty + s);
                umma_commit(t_full + ts);
            }
        }
    } else {
        // ---------------- epilogue ----------------
        const int q = warp & 3;            // TMEM lane quarter this warp may access
        const int h = (warp - 2) >> 2;     // which HG_CW of the GM_N columns of a chunk
        const float wmax = *p.wmax;
        const bool dbg = p.dbg_acc && blockIdx.x == 0 && blockIdx.y == 0;
        float thr[GM_R];
#pragma unroll
        for (int rt = 0; rt < GM_R; rt++) {
            int64_t m = m0 + rt * 128 + q * 32 + lane;
            float xn = m < p.n_pad ? p.xnorm[unit * p.n_pad + m] : -1.0f;
            thr[rt] = xn * (HASH_EPS * wmax);  // negative for padding rows: never flagged
        }
        for (int c = 0; c < p.NT; c++) {
            const int ts = c & 1;
            mbar_wait(t_full + ts, (c >> 1) & 1);
            tc_fence_after();
#pragma unroll HG_RTU
            for (int rs = 0; rs < GM_R * HG_NSUB; rs++) {
                const int rt = rs / HG_NSUB, sc = rs % HG_NSUB;  // key tile, 16-column piece of this warp's share
                const int64_t kb = (m0 + rt * 128 + q * 32) >> 5;  // key block of this warp
                const int64_t kchunk = kb >> 5;
                const int lin = (int)(kb & 31);
                uint4* cw = reinterpret_cast<uint4*>(p.codes) + ((unit * p.nchunks + kchunk) * p.KLq) * 32 + lin;
                {
                    uint32_t v[HG_SUBW];
                    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + ts * (GM_R * GM_N) + rt * GM_N + h * HG_CW +
                                        sc * HG_SUBW;
                    tmem_ldn(ta, v);
                    tmem_wait_ld();
                    const int j0 = c * GM_N + h * HG_CW + sc * HG_SUBW;
                    uint32_t w[HG_SUBW];
                    float mn = 3.0e38f;
                    constexpr int NQ = HG_SUBW / 4;  // uint4 stores (4 column words each)
                    if (j0 + HG_SUBW <= p.KL && (j0 >> 2) + NQ <= p.KLq) {
                        // interior columns (all but the last chunk): no per-column bounds
#pragma unroll
                        for (int cc = 0; cc < HG_SUBW; cc++) {
                            const float a = __uint_as_float(v[cc]);
                            w[cc] = __ballot_sync(0xffffffffu, a > 0.0f);
                            mn = fminf(mn, fabsf(a));
                        }
                        // the ballot words are warp-uniform: one lane stores them (no per-lane selects)
                        if (lane == 0) {
#pragma unroll
                            for (int qd = 0; qd < NQ; qd++)
                                cw[(int64_t)((j0 >> 2) + qd) * 32] =
                                    make_uint4(w[4 * qd], w[4 * qd + 1], w[4 * qd + 2], w[4 * qd + 3]);
                        }
                    } else {
#pragma unroll
                        for (int cc = 0; cc < HG_SUBW; cc++) {
                            float a = __uint_as_float(v[cc]);
                            w[cc] = __ballot_sync(0xffffffffu, a > 0.0f);
                            if (j0 + cc < p.KL) mn = fminf(mn, fabsf(a));
                        }
#pragma unroll
                        for (int qd = 0; qd < NQ; qd++) {
                            int jq = (j0 >> 2) + qd;
                            if (lane == qd && jq < p.KLq)
                                cw[(int64_t)jq * 32] = make_uint4(w[4 * qd], w[4 * qd + 1], w[4 * qd + 2], w[4 * qd + 3]);
                        }
                    }
                    float th = thr[0];
#pragma unroll
                    for (int k = 1; k < GM_R; k++)
                        if (rt == k) th = thr[k];
                    if (__any_sync(0xffffffffu, mn <= th)) {
                        const int64_t m = m0 + rt * 128 + q * 32 + lane;
                        for (int cc = 0; cc < HG_SUBW; cc++) {
                            float a = __uint_as_float(v[cc]);
                            bool f = fabsf(a) <= th && (j0 + cc) < p.KL;
                            uint32_t fm = __ballot_sync(0xffffffffu, f);
                            if (fm) {
                                uint32_t base = 0;
                                if (lane == 0) base = atomicAdd(p.fix_count, (uint32_t)__popc(fm));
                                base = __shfl_sync(0xffffffffu, base, 0);
                                if (f) {
                                    uint32_t slot = base + __popc(fm & ((1u << lane) - 1u));
                                    if (slot < p.fix_cap)
                                        p.fix_list[slot] = make_uint2((uint32_t)(unit * p.n_pad + m), (uint32_t)(j0 + cc));
                                    else
                                        atomicOr(p.status, MAGICPIG_STATUS_OVERFLOW);
                                }
                            }
                        }
                    }
                    if (dbg && rt == 0) {  // (every piece sc of tile 0)
                        for (int cc = 0; cc < HG_SUBW; cc++)
                            if (j0 + cc < p.KL) p.dbg_acc[(int64_t)(q * 32 + lane) * p.KL + j0 + cc] = __uint_as_float(v[cc]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(t_empty + ts);
        }
    }
    __syncwarp();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// Exact recomputation of flagged dots; patches the code bit.
__global__ void __launch_bounds__(128) hash_fixup_kernel(const uint2* __restrict__ list,
                                                         const uint32_t* __restrict__ count, uint32_t cap,
                                                         const uint8_t* __restrict__ xt,
                                                         const uint8_t* __restrict__ wt, int64_t n_pad,
                                                         int64_t nchunks, int KD, int KLq,
                                                         uint32_t* __restrict__ codes, uint32_t* status) {
    uint32_t n = min(*count, cap);
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
        uint2 e = list[idx];
        int64_t unit = (int64_t)e.x / n_pad, m = (int64_t)e.x % n_pad;
        int j = (int)e.y;
        uint16_t xa[144], wa[144];
        const uint8_t* xb = xt + (unit * (n_pad >> 7) + (m >> 7)) * (int64_t)(128 * KD * 2);
        const int r = (int)(m & 127);
        const uint8_t* wb = wt + (int64_t)(j / HG_N) * (HG_N * KD * 2);
        const int cidx = j % HG_N;
        for (int kc = 0; kc < KD / 8; kc++) {
            uint4 xv = *reinterpret_cast<const uint4*>(xb + (kc * 16 + (r >> 3)) * 128 + (r & 7) * 16);
            uint4 wv = *reinterpret_cast<const uint4*>(wb + (kc * (HG_N / 8) + (cidx >> 3)) * 128 + (cidx & 7) * 16);
            const uint32_t xs[4] = {xv.x, xv.y, xv.z, xv.w}, ws[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int t = 0; t < 4; t++) {
                xa[kc * 8 + 2 * t] = (uint16_t)(xs[t] & 0xFFFF);
                xa[kc * 8 + 2 * t + 1] = (uint16_t)(xs[t] >> 16);
                wa[kc * 8 + 2 * t] = (uint16_t)(ws[t] & 0xFFFF);
                wa[kc * 8 + 2 * t + 1] = (uint16_t)(ws[t] >> 16);
            }
        }
        int sg = exact_dot_sign_bf16(xa, wa, KD, status);
        int64_t kb = m >> 5;
        int64_t widx = ((((unit * nchunks + (kb >> 5)) * KLq + (j >> 2)) * 32 + (kb & 31)) << 2) + (j & 3);
        uint32_t bit = 1u << (m & 31);
        if ((j >> 2) < KLq) {
            if (sg > 0) atomicOr(codes + widx, bit);
            else atomicAnd(codes + widx, ~bit);
        }
    }
}

int launch_hash_gemm(const uint8_t* xt, const uint8_t* wt, const float* xnorm, const float* wmax,
                     uint32_t* codes, uint2* fix_list, uint32_t* fix_count, uint32_t fix_cap, int64_t units,
                     int64_t n_local, int64_t n_pad, int64_t nchunks, int KD, int KL, int NT, int KLq,
                     uint32_t* status, float* dbg_acc, cudaStream_t st) {
    GemmParams p;
    p.xt = xt;
    p.wt = wt;
    p.xnorm = xnorm;
    p.wmax = wmax;
    p.codes = codes;
    p.fix_list = fix_list;
    p.fix_count = fix_count;
    p.fix_cap = fix_cap;
    p.n_local = n_local;
    p.n_pad = n_pad;
    p.nchunks = nchunks;
    p.KD = KD;
    p.KL = KL;
    p.NT = NT;
    p.KLq = KLq;
    p.status = status;
    p.dbg_acc = dbg_acc;
    size_t smem = gemm_smem_bytes(KD);
    cudaFuncSetAttribute(hash_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)(n_pad / (GM_R * 128)), (unsigned)units);
    if (dbg_acc) grid = dim3(1, 1);
    hash_gemm_kernel<<<grid, GM_THREADS, smem, st>>>(p);
    count_launch(1);
    if (!dbg_acc) {
        hash_fixup_kernel<<<4 * 148, 128, 0, st>>>(fix_list, fix_count, fix_cap, xt, wt, n_pad, nchunks, KD, KLq,
                                                   codes, status);
        count_launch(1);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

}  // namespace mp
