// decode.cu -- MagicPIG decode step (Algorithm 1).
//
// One CTA = one 1024-key chunk of one (sequence, kv head) unit, or a 1/tsplit
// share of its tables when there are too few chunks to fill the GPU.
//
//  scan     Query(HT, q_code) over bit-plane codes: lane = 32-key block,
//           128-bit coalesced loads; per table and query head one LOP3 per bit
//           (m &= P_b ^ QX_b) and a saturating counter (seen1/seen2) gives the
//           ">= 2 tables match" rule for 32 keys at once.
//  combine  warps -> CTA via shared memory; CTAs of one chunk via atomicOr
//           (exact: (a1,a2)+(b1,b2) = (a1|b1, a2|b2|(a1&b1))), last CTA goes on.
//  compact  S_g (sampled, per query head) U T (sink/local) -> ascending
//           list of chunk offsets (ballot/popc prefix sums).
//  gather   warp per listed key: k, v rows (256 B each) -> logits q.k/sqrt(d)
//           (P:109), for i in S_g: cos of the hashed vectors (R5), p, log u
//           (fp64) and z = logit - log u; online softmax.
//  merge    chunk partial (m, s, a) -> last CTA of the unit merges all chunks
//           in fixed order (log-sum-exp, "recursive attention" P:171).
#include "common.cuh"
#include "kernels.cuh"

namespace mp {

constexpr int NWARP = DEC_THREADS / 32;
constexpr float INV_SQRT_D = 0.08838834764831845f;  // 1/sqrt(128)

// bits r of a 32-key block [base, base+32) whose local index lies in [lo, hi)
__device__ __forceinline__ uint32_t range_mask(int64_t base, int64_t lo, int64_t hi) {
    int64_t a = lo - base, b = hi - base;
    a = a < 0 ? 0 : (a > 32 ? 32 : a);
    b = b < 0 ? 0 : (b > 32 ? 32 : b);
    if (b <= a) return 0u;
    uint32_t hiMask = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
    uint32_t loMask = a >= 32 ? 0xffffffffu : ((1u << a) - 1u);
    return hiMask & ~loMask;
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <int G>
__device__ __forceinline__ void load_masks(const uint32_t* p, uint32_t (&q)[G]) {
    if constexpr (G % 4 == 0) {
#pragma unroll
        for (int t = 0; t < G / 4; t++) {
            uint4 v = reinterpret_cast<const uint4*>(p)[t];
            q[4 * t] = v.x;
            q[4 * t + 1] = v.y;
            q[4 * t + 2] = v.z;
            q[4 * t + 3] = v.w;
        }
    } else if constexpr (G == 2) {
        uint2 v = *reinterpret_cast<const uint2*>(p);
        q[0] = v.x;
        q[1] = v.y;
    } else {
        q[0] = p[0];
    }
}

template <int K, int G>
__global__ void __launch_bounds__(DEC_THREADS) decode_kernel(DecodeArgs a) {
    constexpr int TG = tg_of(K), QG = qg_of(K);
    extern __shared__ __align__(16) uint32_t qx[];  // [ncols][G] match masks
    __shared__ uint32_t s_part[NWARP][G][2][32];
    __shared__ uint32_t s_sel[G][32];
    __shared__ uint32_t s_tm[32];
    __shared__ uint16_t s_list[KCHUNK];
    __shared__ int s_nsel;
    __shared__ uint32_t s_flag;
    __shared__ float s_m[NWARP][G], s_s[NWARP][G];
    __shared__ float s_a[NWARP][HD];
    __shared__ float s_q[G][HD];
    __shared__ float s_qn[G];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t cg = blockIdx.x / a.tsplit;  // global chunk = unit * nchunks + chunk
    const int part = blockIdx.x % a.tsplit;
    const int64_t unit = cg / a.nchunks, chunk = cg % a.nchunks;
    const int64_t b = unit / a.Hkv, hkv = unit % a.Hkv;
    const int64_t qh0 = b * a.Hq + hkv * G;  // first query head (row of q) of this unit
    const int g0 = (int)((int64_t)part * a.ngroups / a.tsplit);
    const int g1 = (int)((int64_t)(part + 1) * a.ngroups / a.tsplit);
    const int col0 = g0 * TG * K;
    const int ncols = (g1 - g0) * TG * K;

    // ---- query masks: QX[c][g] = qbit ? 0 : ~0, so  P ^ QX = 1 where the key bit equals qbit
    for (int e = tid; e < ncols * G; e += DEC_THREADS) {
        int c = e / G, g = e % G;
        int col = col0 + c;
        uint32_t bit = 0;
        if (col < a.KL) bit = (a.qbits[(qh0 + g) * a.KLw + (col >> 5)] >> (col & 31)) & 1u;
        qx[e] = bit ? 0u : 0xffffffffu;
    }
    __syncthreads();

    // ---- scan
    uint32_t s1[G], s2[G];
#pragma unroll
    for (int g = 0; g < G; g++) s1[g] = s2[g] = 0u;
    const uint4* cp = reinterpret_cast<const uint4*>(a.codes) + (cg * a.KLq) * 32 + lane;
    int grp = g0 + warp;
    uint4 P[QG];
    if (grp < g1) {
#pragma unroll
        for (int t = 0; t < QG; t++) P[t] = ldg_stream(cp + (int64_t)(grp * QG + t) * 32);
    }
    while (grp < g1) {
        const int nxt = grp + NWARP;
        uint4 Pn[QG];
        if (nxt < g1) {
#pragma unroll
            for (int t = 0; t < QG; t++) Pn[t] = ldg_stream(cp + (int64_t)(nxt * QG + t) * 32);
        }
        const uint32_t* wv = reinterpret_cast<const uint32_t*>(P);
        const uint32_t* qrow = qx + (size_t)(grp - g0) * TG * K * G;
#pragma unroll
        for (int tt = 0; tt < TG; tt++) {
            if (grp * TG + tt < a.L) {
                uint32_t m[G];
#pragma unroll
                for (int g = 0; g < G; g++) m[g] = 0xffffffffu;
#pragma unroll
                for (int bb = 0; bb < K; bb++) {
                    const uint32_t w = wv[tt * K + bb];
                    uint32_t qq[G];
                    load_masks<G>(qrow + (tt * K + bb) * G, qq);
#pragma unroll
                    for (int g = 0; g < G; g++) m[g] &= w ^ qq[g];
                }
#pragma unroll
                for (int g = 0; g < G; g++) {
                    s2[g] |= s1[g] & m[g];
                    s1[g] |= m[g];
                }
            }
        }
#pragma unroll
        for (int t = 0; t < QG; t++) P[t] = Pn[t];
        grp = nxt;
    }

    // ---- combine warps
#pragma unroll
    for (int g = 0; g < G; g++) {
        s_part[warp][g][0][lane] = s1[g];
        s_part[warp][g][1][lane] = s2[g];
    }
    __syncthreads();
    if (tid < G * 32) {
        const int g = tid >> 5;
        uint32_t a1 = 0, a2 = 0;
        for (int w = 0; w < NWARP; w++) {
            uint32_t b1 = s_part[w][g][0][lane], b2 = s_part[w][g][1][lane];
            a2 |= b2 | (a1 & b1);
            a1 |= b1;
        }
        if (a.tsplit > 1) {
            uint32_t* sg = a.seen + ((cg * G + g) * 2) * 32 + lane;
            uint32_t old1 = atomicOr(sg, a1);
            atomicOr(sg + 32, a2 | (old1 & a1));
        }
        s_part[0][g][0][lane] = a1;
        s_part[0][g][1][lane] = a2;
    }
    if (a.tsplit > 1) {
        __threadfence();
        __syncthreads();
        if (tid == 0) s_flag = atomicAdd(a.chunk_ctr + cg, 1u) == (uint32_t)(a.tsplit - 1);
        __syncthreads();
        if (!s_flag) return;
        __threadfence();
        if (tid < G * 32) {
            const int g = tid >> 5;
            uint32_t* sg = a.seen + ((cg * G + g) * 2) * 32 + lane;
            s_part[0][g][0][lane] = atomicExch(sg, 0u);
            s_part[0][g][1][lane] = atomicExch(sg + 32, 0u);
        }
        if (tid == 0) a.chunk_ctr[cg] = 0u;
    }
    __syncthreads();

    // ---- final masks: S_g = count >= min_collisions, restricted to D; T = static keys
    const int64_t cbase = chunk * KCHUNK;  // local index of the chunk's first key
    if (tid < 32) {
        const int64_t base = cbase + lane * 32;
        uint32_t valid = range_mask(base, 0, a.n_local);
        uint32_t tm = (range_mask(base, -a.seq_offset, (int64_t)a.sink - a.seq_offset) |
                       range_mask(base, a.n_global - a.local - a.seq_offset, a.n_global - a.seq_offset)) &
                      valid;
        s_tm[lane] = tm;
    }
    __syncthreads();
    if (tid < G * 32) {
        const int g = tid >> 5;
        uint32_t v = (a.minc == 1 ? s_part[0][g][0][lane] : s_part[0][g][1][lane]);
        const int64_t base = cbase + lane * 32;
        v &= range_mask(base, 0, a.n_local) & ~s_tm[lane];
        s_sel[g][lane] = v;
        int cnt = __popc(v);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
        if (lane == 0) a.chunk_cnt[cg * G + g] = cnt;
        if (a.s_mask) {
            int64_t nw = (a.n_local + 31) >> 5;
            int64_t widx = chunk * 32 + lane;
            if (widx < nw) a.s_mask[(qh0 + g) * nw + widx] = v;
        }
    }
    // query vectors for the gather
    for (int e = tid; e < G * HD; e += DEC_THREADS) s_q[e / HD][e % HD] = bf2f(a.q[(qh0 + e / HD) * HD + e % HD]);
    __syncthreads();
    if (tid < G * 32) {
        const int g = tid >> 5;
        float x0 = s_q[g][lane * 4], x1 = s_q[g][lane * 4 + 1], x2 = s_q[g][lane * 4 + 2], x3 = s_q[g][lane * 4 + 3];
        float nn = warp_sum_f(x0 * x0 + x1 * x1 + x2 * x2 + x3 * x3);
        if (lane == 0) s_qn[g] = sqrtf(nn);
    }
    // ---- compaction (ascending order) of U = (union_g S_g) U T
    if (warp == 0) {
        uint32_t u = s_tm[lane];
#pragma unroll
        for (int g = 0; g < G; g++) u |= s_sel[g][lane];
        int c = __popc(u);
        int incl = c;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, incl, m);
            if (lane >= m) incl += t;
        }
        int pos = incl - c;
        while (u) {
            int r = __ffs(u) - 1;
            u &= u - 1;
            s_list[pos++] = (uint16_t)(lane * 32 + r);
        }
        if (lane == 31) s_nsel = incl;
    }
    __syncthreads();

    // ---- gather + estimator (warp per key, lane = 4 dims)
    float m_run[G], s_run[G], acc[G][4];
#pragma unroll
    for (int g = 0; g < G; g++) {
        m_run[g] = -INFINITY;
        s_run[g] = 0.0f;
        acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.0f;
    }
    float qv[G][4];
#pragma unroll
    for (int g = 0; g < G; g++) {
        qv[g][0] = s_q[g][lane * 4];
        qv[g][1] = s_q[g][lane * 4 + 1];
        qv[g][2] = s_q[g][lane * 4 + 2];
        qv[g][3] = s_q[g][lane * 4 + 3];
    }
    const float4 cvec = reinterpret_cast<const float4*>(a.center + unit * HD)[lane];
    const float* knorm = a.key_norm + unit * a.n_local;
    const uint16_t* kbase = a.k + unit * a.n_local * HD;
    const uint16_t* vbase = a.v + unit * a.n_local * HD;
    const int nsel = s_nsel;
    for (int e = warp; e < nsel; e += NWARP) {
        const int off = s_list[e];
        const int64_t i = cbase + off;
        const uint32_t bitm = 1u << (off & 31);
        const bool is_t = (s_tm[off >> 5] & bitm) != 0;
        uint32_t inS = 0;
#pragma unroll
        for (int g = 0; g < G; g++) inS |= ((s_sel[g][off >> 5] & bitm) ? 1u : 0u) << g;
        const uint2 kr = __ldg(reinterpret_cast<const uint2*>(kbase + i * HD) + lane);
        const uint2 vr = __ldg(reinterpret_cast<const uint2*>(vbase + i * HD) + lane);
        const float k0 = __uint_as_float(kr.x << 16), k1 = __uint_as_float(kr.x & 0xffff0000u);
        const float k2 = __uint_as_float(kr.y << 16), k3 = __uint_as_float(kr.y & 0xffff0000u);
        const float v0 = __uint_as_float(vr.x << 16), v1 = __uint_as_float(vr.x & 0xffff0000u);
        const float v2 = __uint_as_float(vr.y << 16), v3 = __uint_as_float(vr.y & 0xffff0000u);
        float logit[G];
#pragma unroll
        for (int g = 0; g < G; g++) logit[g] = warp_sum_f(qv[g][0] * k0 + qv[g][1] * k1 + qv[g][2] * k2 + qv[g][3] * k3) * INV_SQRT_D;
        float lu[G];
#pragma unroll
        for (int g = 0; g < G; g++) lu[g] = 0.0f;
        if (inS) {
            // the hashed key vector xbar_i (same arithmetic as the build); |xbar_i| from the index
            const float x0 = bf2f(f2bf_rn(__fsub_rn(k0, cvec.x))), x1 = bf2f(f2bf_rn(__fsub_rn(k1, cvec.y)));
            const float x2 = bf2f(f2bf_rn(__fsub_rn(k2, cvec.z))), x3 = bf2f(f2bf_rn(__fsub_rn(k3, cvec.w)));
            const float xnorm = __ldg(knorm + i);
#pragma unroll
            for (int g = 0; g < G; g++) {
                if (inS & (1u << g)) {
                    float dq = warp_sum_f(qv[g][0] * x0 + qv[g][1] * x1 + qv[g][2] * x2 + qv[g][3] * x3);
                    float den = s_qn[g] * xnorm;
                    float cs = den > 0.0f ? dq / den : 0.0f;
                    cs = fminf(1.0f, fmaxf(-1.0f, cs));
                    const float p = 1.0f - acosf(cs) * 0.3183098861837907f;
                    lu[g] = log_sampling_prob(p, K, a.L, a.minc);
                }
            }
        }
#pragma unroll
        for (int g = 0; g < G; g++) {
            if (is_t || (inS & (1u << g))) {
                const float z = logit[g] - lu[g];
                if (z > m_run[g]) {
                    const float sc = __expf(m_run[g] - z);
                    s_run[g] = s_run[g] * sc + 1.0f;
                    acc[g][0] = acc[g][0] * sc + v0;
                    acc[g][1] = acc[g][1] * sc + v1;
                    acc[g][2] = acc[g][2] * sc + v2;
                    acc[g][3] = acc[g][3] * sc + v3;
                    m_run[g] = z;
                } else {
                    const float w = __expf(z - m_run[g]);
                    s_run[g] += w;
                    acc[g][0] += w * v0;
                    acc[g][1] += w * v1;
                    acc[g][2] += w * v2;
                    acc[g][3] += w * v3;
                }
            }
        }
    }
    // ---- combine warp states -> chunk partial (one head at a time)
    float* pc = a.parts + cg * G * PART;
#pragma unroll
    for (int g = 0; g < G; g++) {
        if (lane == 0) {
            s_m[warp][g] = m_run[g];
            s_s[warp][g] = s_run[g];
        }
        s_a[warp][lane * 4] = acc[g][0];
        s_a[warp][lane * 4 + 1] = acc[g][1];
        s_a[warp][lane * 4 + 2] = acc[g][2];
        s_a[warp][lane * 4 + 3] = acc[g][3];
        __syncthreads();
        if (tid < HD) {
            const int d = tid;
            float M = -INFINITY;
            for (int w = 0; w < NWARP; w++) M = fmaxf(M, s_m[w][g]);
            float S = 0.0f, A = 0.0f;
            if (M != -INFINITY) {
                for (int w = 0; w < NWARP; w++) {
                    if (s_m[w][g] == -INFINITY) continue;
                    const float f = __expf(s_m[w][g] - M);
                    S += s_s[w][g] * f;
                    A += s_a[w][d] * f;
                }
            }
            pc[g * PART + 2 + d] = A;
            if (d == 0) {
                pc[g * PART] = M;
                pc[g * PART + 1] = S;
            }
        }
        __syncthreads();
    }
    // ---- last chunk of the unit merges all chunks (fixed order)
    __threadfence();
    __syncthreads();
    if (tid == 0) s_flag = atomicAdd(a.unit_ctr + unit, 1u) == (uint32_t)(a.nchunks - 1);
    __syncthreads();
    if (!s_flag) return;
    __threadfence();
    const float* pu = a.parts + unit * a.nchunks * G * PART;
    for (int e = tid; e < G * HD; e += DEC_THREADS) {
        const int g = e / HD, d = e % HD;
        float M = -INFINITY;
        for (int64_t c = 0; c < a.nchunks; c++) M = fmaxf(M, __ldcg(pu + (c * G + g) * PART));
        float S = 0.0f, A = 0.0f;
        if (M != -INFINITY) {
            for (int64_t c = 0; c < a.nchunks; c++) {
                const float mc = __ldcg(pu + (c * G + g) * PART);
                if (mc == -INFINITY) continue;
                const float f = __expf(mc - M);
                S += __ldcg(pu + (c * G + g) * PART + 1) * f;
                A += __ldcg(pu + (c * G + g) * PART + 2 + d) * f;
            }
        }
        const int64_t row = qh0 + g;
        if (a.out) a.out[row * HD + d] = S > 0.0f ? A / S : 0.0f;
        if (a.partial) {
            a.partial[row * PART + 2 + d] = A;
            if (d == 0) {
                a.partial[row * PART] = M;
                a.partial[row * PART + 1] = S;
            }
        }
        if (d == 0) {
            if (!(S > 0.0f) && a.out) atomicOr(a.status, MAGICPIG_STATUS_DEGENERATE);
            if (a.s_count) {
                int tot = 0;
                for (int64_t c = 0; c < a.nchunks; c++) tot += __ldcg(a.chunk_cnt + (unit * a.nchunks + c) * G + g);
                a.s_count[row] = tot;
            }
        }
    }
    if (tid == 0) a.unit_ctr[unit] = 0u;
}

// P-way merge of partial states (sequence shards): parts [P][BH][130]
__global__ void merge_partials_kernel(const float* __restrict__ parts, int P, int64_t BH, float* __restrict__ out) {
    const int64_t row = blockIdx.x;
    const int d = threadIdx.x;
    float M = -INFINITY;
    for (int p = 0; p < P; p++) M = fmaxf(M, parts[((int64_t)p * BH + row) * PART]);
    float S = 0.0f, A = 0.0f;
    if (M != -INFINITY) {
        for (int p = 0; p < P; p++) {
            const float* pp = parts + ((int64_t)p * BH + row) * PART;
            if (pp[0] == -INFINITY) continue;
            const float f = __expf(pp[0] - M);
            S += pp[1] * f;
            A += pp[2 + d] * f;
        }
    }
    out[row * HD + d] = S > 0.0f ? A / S : 0.0f;
}

__global__ void empty_partial_kernel(float* __restrict__ partial, int64_t BH) {
    const int64_t row = blockIdx.x;
    for (int d = threadIdx.x; d < PART; d += blockDim.x) partial[row * PART + d] = d == 0 ? -INFINITY : 0.0f;
}

int launch_empty_partial(float* partial, int64_t BH, cudaStream_t st) {
    empty_partial_kernel<<<(unsigned)BH, 128, 0, st>>>(partial, BH);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

template <int K, int G>
static int launch_kg(const DecodeArgs& a, cudaStream_t st) {
    constexpr int TG = tg_of(K);
    int maxg = (a.ngroups + a.tsplit - 1) / a.tsplit + 1;
    size_t smem = (size_t)maxg * TG * K * G * 4;
    auto kern = decode_kernel<K, G>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int64_t nblk = a.B * a.Hkv * a.nchunks * a.tsplit;
    kern<<<(unsigned)nblk, DEC_THREADS, smem, st>>>(a);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

template <int K>
static int launch_k(const DecodeArgs& a, int G, cudaStream_t st) {
    switch (G) {
        case 1: return launch_kg<K, 1>(a, st);
        case 2: return launch_kg<K, 2>(a, st);
        case 4: return launch_kg<K, 4>(a, st);
        case 8: return launch_kg<K, 8>(a, st);
    }
    return MAGICPIG_EINVAL;
}

int launch_decode(const DecodeArgs& a, cudaStream_t st) {
    const int G = (int)(a.Hq / a.Hkv);
    switch (a.K) {
#define MPK(k) \
    case k: return launch_k<k>(a, G, st);
        MPK(1) MPK(2) MPK(3) MPK(4) MPK(5) MPK(6) MPK(7) MPK(8)
        MPK(9) MPK(10) MPK(11) MPK(12) MPK(13) MPK(14) MPK(15) MPK(16)
#undef MPK
    }
    return MAGICPIG_EINVAL;
}

int launch_merge(const float* parts, int P, int64_t BH, float* out, cudaStream_t st) {
    merge_partials_kernel<<<(unsigned)BH, HD, 0, st>>>(parts, P, BH, out);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

}  // namespace mp
