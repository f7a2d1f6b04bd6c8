// decode.cu -- MagicPIG decode step (Algorithm 1).
//
// Grid: one thread-block CLUSTER of CS CTAs per 1024-key chunk of one
// (sequence, kv head) unit; CTA r of the cluster scans table groups
// [r*ng/CS, (r+1)*ng/CS).  8 warps per CTA; lane = 32-key block.
//
//  stream   each warp streams its table groups (QG*512 contiguous bytes each)
//           into a private shared-memory ring with cp.async.bulk + mbarrier;
//           the first copies are issued BEFORE griddepcontrol.wait, so the
//           code stream overlaps the query-encode kernel (PDL).
//  scan     Query(HT, q_code): per table and query head one LOP3 per
//           bit (m &= P_b ^ QX_b) and a saturating counter (seen1/seen2) gives
//           the ">= 2 tables match" rule for 32 keys at once.
//  combine  warps -> CTA via shared memory, CTAs -> cluster via DSMEM:
//           (a1,a2)+(b1,b2) = (a1|b1, a2|b2|(a1&b1)); every CTA ends with the
//           same S_g and the same ascending list of S U T (P:171 static keys).
//  gather   CTA r takes list entries r, r+CS, ...; K/V rows (256 B each) and
//           |xbar_i| staged by cp.async in double-buffered batches; warp per
//           key: logits q.k/sqrt(d), cos of the hashed vectors (R5),
//           p, log u (fp32, R11), z = logit - log u,
//           online softmax.
//  merge    CTA partials -> rank 0 via DSMEM -> chunk partial; the last chunk
//           of a unit merges all chunks in fixed order (log-sum-exp,
//           "recursive attention" P:171).  Counters self-clean (graph-safe).
#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cgr = cooperative_groups;

namespace mp {

constexpr int NWARP = DEC_THREADS / 32;
constexpr int RB = 32;                   // rows (keys) per gather batch
constexpr int XS = 272;                  // bytes per row of the bf16 xbar tile (16-B aligned, conflict-free ldmatrix)
constexpr int QBS = 272;                 // bytes per row of the bf16 query tile
constexpr int ROWB = 2 * HD * 2 + 16;    // k row + v row + norm (padded) bytes
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

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
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

// online-softmax update of one head's running state with score z and value row
__device__ __forceinline__ void osm_update(float z, float& m, float& s, float (&acc)[4], float v0, float v1,
                                           float v2, float v3) {
    if (z > m) {
        const float sc = __expf(m - z);
        s = s * sc + 1.0f;
        acc[0] = acc[0] * sc + v0;
        acc[1] = acc[1] * sc + v1;
        acc[2] = acc[2] * sc + v2;
        acc[3] = acc[3] * sc + v3;
        m = z;
    } else {
        const float w = __expf(z - m);
        s += w;
        acc[0] += w * v0;
        acc[1] += w * v1;
        acc[2] += w * v2;
        acc[3] += w * v3;
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ long long clk64() { return clock64(); }
#define MP_ACC(ph, t0)                                  \
    do {                                                 \
        if (a.timeline && threadIdx.x == 0) {            \
            long long t1_ = clk64();                     \
            tacc[(ph) - 11] += (t1_ - (t0));             \
            t0 = t1_;                                    \
        }                                                \
    } while (0)
// debug timeline: slot 0 = %globaltimer at CTA start (ns); slots 1..10 = SM cycles
// since the CTA start (clock64 of thread 0), +1 so that 0 means "not reached"
#define MP_STAMP(ph)                                                                                   \
    do {                                                                                                \
        if (a.timeline && threadIdx.x == 0) {                                                           \
            if ((ph) == 0) {                                                                            \
                a.timeline[(size_t)blockIdx.x * 32] = gtimer();                                         \
                mp_t0 = clk64();                                                                        \
            } else {                                                                                    \
                a.timeline[(size_t)blockIdx.x * 32 + (ph)] = (unsigned long long)(clk64() - mp_t0 + 1); \
            }                                                                                           \
        }                                                                                               \
    } while (0)

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t (&r)[2], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}
// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D, fp32 accumulate (exact products)
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// D(16x8 fp32) = A(16x8 tf32, row) * B(8x8 tf32, col) + C
__device__ __forceinline__ void mma1688_tf32(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// Per-CTA working set of the batched gather (static shared memory).
template <int G>
struct __align__(16) GatherShared {
    int keys[KCHUNK];            // local key index of every entry this CTA gathers
    uint16_t bits[KCHUNK];       // bit g: key in S_g; bit 8: static (u = 1)
    __align__(16) uint8_t qb16[8 * QBS];  // query heads as bf16 rows (mma B operand), zero padded
    float c[HD];                 // centering vector
    float qn[G];                 // |q_g|
    float zl[RB][8], zd[RB][8], w[RB][8];
    float mrun[G], srun[G], scale[G];
    float xn[RB];
    uint16_t sbits[RB];
    uint64_t rbar[2];            // row-buffer mbarriers (bulk copies of K/V rows)
};

// Batched gather + estimator over n entries (keys[], bits[]) of one unit
// (PAPER.md:109-115): K/V rows and |xbar| staged by cp.async, logits K Q^T and
// hashed-vector dots X Q^T on tensor cores (mma.sync m16n8k16, bf16 in, fp32
// accumulate), one thread per (key, head) for z = logit - log u, then an online
// softmax whose state (m, s per head; a per (head, dim pair)) is thread-parallel.
// acc: this warp's two 16x8 tf32-MMA accumulator tiles of a[g][d] (rows = heads g,
// columns = dims 16*warp .. 16*warp+15); c0,c1 = (g = lane/4, d = 2*(lane%4) + {0,1}).
template <int K, int G>
__device__ __forceinline__ void gather_batched(const DecodeArgs& a, GatherShared<G>& sh, uint8_t* region,
                                               int n, int64_t unit, float (&acc)[2][4]) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint8_t* rows = region;                  // [2][RB][ROWB]
    uint8_t* xt = region + 2 * RB * ROWB;    // [RB][XS]
    const float* knorm = a.key_norm + unit * a.n_local;
    const uint16_t* kbase = a.k + unit * a.n_local * HD;
    const uint16_t* vbase = a.v + unit * a.n_local * HD;
    const int nbatch = (n + RB - 1) / RB;
    // K/V rows by bulk copy (lane r of warp 0 copies row r), |xbar| by cp.async (warp 1)
    if (tid == 0) {
        mbar_init(&sh.rbar[0], 1);
        mbar_init(&sh.rbar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto stage = [&](int bt) {
        uint8_t* buf = rows + (bt & 1) * RB * ROWB;
        const int nbt = min(RB, n - bt * RB);
        if (warp == 0) {
            if (lane == 0) {
                fence_proxy_async();
                mbar_arrive_expect_tx(&sh.rbar[bt & 1], (uint32_t)nbt * 512u);
            }
            __syncwarp();
            if (lane < nbt) {
                const int64_t i = sh.keys[bt * RB + lane];
                bulk_g2s(buf + lane * ROWB, kbase + i * HD, 256, &sh.rbar[bt & 1]);
                bulk_g2s(buf + lane * ROWB + 256, vbase + i * HD, 256, &sh.rbar[bt & 1]);
            }
        } else if (warp == 1 && lane < nbt) {
            cp_async4(buf + lane * ROWB + 512, knorm + sh.keys[bt * RB + lane]);
        }
        cp_async_commit();
    };
    if (nbatch > 0) stage(0);
    long long tcl = clk64();
    long long tacc[4] = {0, 0, 0, 0};
    for (int bt = 0; bt < nbatch; bt++) {
        if (bt + 1 < nbatch) {
            stage(bt + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        mbar_wait(&sh.rbar[bt & 1], (uint32_t)((bt >> 1) & 1));
        __syncthreads();
        MP_ACC(11, tcl);
        const uint8_t* buf = rows + (bt & 1) * RB * ROWB;
        const int nb = min(RB, n - bt * RB);
        // (a) xbar = bf16(fl32(k - c)) for the batch rows (cvt.rn.bf16x2.f32), all warps
#pragma unroll
        for (int t = 0; t < RB * (HD / 8) / DEC_THREADS; t++) {
            const int e = tid + DEC_THREADS * t;
            const int rr = e / (HD / 8), dg = e % (HD / 8);
            const uint4 kv = *reinterpret_cast<const uint4*>(buf + rr * ROWB + dg * 16);
            const float4 c0 = *reinterpret_cast<const float4*>(&sh.c[dg * 8]);
            const float4 c1 = *reinterpret_cast<const float4*>(&sh.c[dg * 8 + 4]);
            const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            const uint32_t kw[4] = {kv.x, kv.y, kv.z, kv.w};
            uint32_t xw[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const __nv_bfloat162 xb = __floats2bfloat162_rn(__fsub_rn(__uint_as_float(kw[u] << 16), cc[2 * u]),
                                                                __fsub_rn(__uint_as_float(kw[u] & 0xffff0000u), cc[2 * u + 1]));
                xw[u] = *reinterpret_cast<const uint32_t*>(&xb);
            }
            *reinterpret_cast<uint4*>(xt + rr * XS + dg * 16) = make_uint4(xw[0], xw[1], xw[2], xw[3]);
        }
        __syncthreads();
        // (b) tensor cores: warp (mt, which) = 16 rows x {raw keys -> logits, xbar -> cos}
        if (warp < 2 * (RB / 16)) {
            const int mt = warp & 1, which = warp >> 1;
            const uint8_t* abase = which == 0 ? buf : xt;
            const int astride = which == 0 ? ROWB : XS;
            float d4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            const int arow = mt * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
            const uint32_t a_addr = smem_u32(abase + arow * astride + 16 * (lane >> 4));
            const uint32_t b_addr = smem_u32(sh.qb16 + (lane & 7) * QBS + 16 * ((lane >> 3) & 1));
#pragma unroll
            for (int ks = 0; ks < HD / 16; ks++) {
                uint32_t af[4], bfr[2];
                ldsm_x4(af, a_addr + ks * 32);
                ldsm_x2(bfr, b_addr + ks * 32);
                mma16816(d4, af, bfr);
            }
            float(*dst)[8] = which == 0 ? sh.zl : sh.zd;
            const int r0 = mt * 16 + (lane >> 2), c0 = (lane & 3) * 2;
            dst[r0][c0] = d4[0];
            dst[r0][c0 + 1] = d4[1];
            dst[r0 + 8][c0] = d4[2];
            dst[r0 + 8][c0 + 1] = d4[3];
        }
        __syncthreads();
        MP_ACC(12, tcl);
        // (c+d) warp g = head g, lane = row: z = q.k/sqrt(d) - log u (u from the hashed
        // vectors' angle R5), then the batch max, rescale factor and weights of the online softmax
        if (warp < G) {
            const int g = warp, rr = lane;  // RB == 32
            float z = -INFINITY;
            if (rr < nb) {
                const uint32_t sb = sh.bits[bt * RB + rr];
                const float logit = sh.zl[rr][g] * INV_SQRT_D;
                if (sb & 0x100u) {
                    z = logit;
                } else if (sb & (1u << g)) {
                    const float xn = *reinterpret_cast<const float*>(buf + rr * ROWB + 512);
                    const float den = sh.qn[g] * xn;
                    float cs = den > 0.0f ? __fdividef(sh.zd[rr][g], den) : 0.0f;
                    cs = fminf(1.0f, fmaxf(-1.0f, cs));
                    const float p = 1.0f - acosf(cs) * 0.3183098861837907f;
                    z = logit - log_sampling_prob(p, K, a.L, a.minc);
                }
            }
            float mb = z;
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, m));
            const float mo = sh.mrun[g];
            const float mn = fmaxf(mo, mb);
            const float sc = (mo == -INFINITY) ? 0.0f : __expf(mo - mn);
            // weights rounded to tf32 (the accumulation MMA's input); the normaliser uses
            // the same rounded weights, so the estimate stays a convex combination
            const float w = (z == -INFINITY) ? 0.0f : to_tf32(__expf(z - mn));
            const float wsum = warp_sum_f(w);
            sh.w[rr][g] = w;
            if (lane == 0) {
                sh.scale[g] = sc;
                sh.srun[g] = sh.srun[g] * sc + wsum;
                sh.mrun[g] = mn;
            }
        }
        __syncthreads();
        MP_ACC(13, tcl);
        // (e) a[g][d] = a * scale + sum_rows w * v on tensor cores (tf32 m16n8k8, fp32 accumulate):
        // A = weights [heads x rows], B = V [rows x dims]; warp w owns dims 16w .. 16w+15
        {
            const int g = lane >> 2;
            const float sc = g < G ? sh.scale[g] : 0.0f;
#pragma unroll
            for (int nt = 0; nt < 2; nt++) {
                acc[nt][0] *= sc;
                acc[nt][1] *= sc;
            }
#pragma unroll
            for (int ks = 0; ks < RB / 8; ks++) {
                const int k0 = ks * 8 + (lane & 3), k1 = k0 + 4;
                const uint32_t a0 = g < G ? __float_as_uint(sh.w[k0][g]) : 0u;
                const uint32_t a2 = g < G ? __float_as_uint(sh.w[k1][g]) : 0u;
#pragma unroll
                for (int nt = 0; nt < 2; nt++) {
                    const int dcol = warp * 16 + nt * 8 + (lane >> 2);
                    const uint32_t v0 = k0 < nb ? (uint32_t)*reinterpret_cast<const uint16_t*>(buf + k0 * ROWB + 256 + dcol * 2) << 16 : 0u;
                    const uint32_t v1 = k1 < nb ? (uint32_t)*reinterpret_cast<const uint16_t*>(buf + k1 * ROWB + 256 + dcol * 2) << 16 : 0u;
                    mma1688_tf32(acc[nt], a0, a2, v0, v1);
                }
            }
        }
        __syncthreads();  // buffer (bt & 1) is refilled by stage(bt + 2); w reused
        MP_ACC(14, tcl);
    }
    if (a.timeline && threadIdx.x == 0)
        for (int t = 0; t < 4; t++) a.timeline[(size_t)blockIdx.x * 32 + 11 + t] = (unsigned long long)tacc[t];
}

template <int K, int G>
__global__ void __launch_bounds__(DEC_THREADS) decode_kernel(DecodeArgs a) {
    constexpr int TG = tg_of(K), QG = qg_of(K);
    constexpr uint32_t GB = QG * 512;  // bytes of one table group of one chunk
    extern __shared__ __align__(128) uint8_t dsm[];
    uint32_t* qx = reinterpret_cast<uint32_t*>(dsm);  // [ncols][G] match masks
    uint8_t* ring = dsm + a.qx_bytes;                  // scan: [NWARP][depth][GB]; gather: rows + x tile
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + a.ring_bytes);  // [NWARP][depth]
    uint32_t* qb = reinterpret_cast<uint32_t*>(bars + NWARP * a.depth);  // [G][KLw] packed query bits

    __shared__ uint32_t s_part[NWARP][G][2][32];
    __shared__ uint32_t s_sel[G][32];
    __shared__ uint32_t s_tm[32];
    __shared__ int s_base[32];
    __shared__ int s_n;
    __shared__ uint32_t s_flag;
    __shared__ GatherShared<G> sh;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int CS = a.tsplit;  // power of two
    const int lcs = __ffs(CS) - 1;
    cgr::cluster_group cluster = cgr::this_cluster();
    const int rank = CS > 1 ? (int)cluster.block_rank() : 0;
    const int64_t per_unit = a.nchunks + a.nstatic;  // clusters per unit: chunk scans + static pieces
    const int64_t cid = blockIdx.x / CS;
    const int64_t unit = cid / per_unit, slot = cid % per_unit;
    const bool is_static = slot >= a.nchunks;
    const int64_t chunk = slot;
    const int64_t cgid = unit * a.nchunks + chunk;  // global chunk (valid if !is_static)
    const int64_t b = unit / a.Hkv, hkv = unit % a.Hkv;
    const int64_t qh0 = b * a.Hq + hkv * G;  // first query head (row of q) of this unit
    const int g0 = (int)((int64_t)rank * a.ngroups / CS);
    const int g1 = (int)((int64_t)(rank + 1) * a.ngroups / CS);
    const int col0 = g0 * TG * K;
    const int ncols = (g1 - g0) * TG * K;
    const int depth = a.depth;
    long long mp_t0 = 0;
    MP_STAMP(0);

    const uint8_t* csrc = reinterpret_cast<const uint8_t*>(a.codes) + (size_t)cgid * a.KLq * 512;
    uint8_t* myring = ring + (size_t)warp * depth * GB;
    uint64_t* mybar = bars + warp * depth;
    const int n_my = (!is_static && g1 - g0 > warp) ? (g1 - g0 - warp + NWARP - 1) / NWARP : 0;
    if (!is_static) {
        // ---- 1. stream this CTA's code groups: whole range -> L2 now, ring refills from L2
        if (tid == 0 && g1 > g0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(csrc + (size_t)g0 * GB),
                         "r"((uint32_t)((g1 - g0) * GB))
                         : "memory");
        if (lane == 0) {
            for (int s = 0; s < depth; s++) mbar_init(mybar + s, 1);
            fence_mbar_init();
            for (int k = 0; k < depth && k < n_my; k++) {
                const int grp = g0 + warp + k * NWARP;
                mbar_arrive_expect_tx(mybar + k, GB);
                bulk_g2s(myring + k * GB, csrc + (size_t)grp * GB, GB, mybar + k);
            }
        }
    }
    // query rows (bf16 mma operand, heads >= G zero), |q_g|, centering vector: no dependency on the encode
    for (int e = tid; e < 8 * (HD / 2); e += DEC_THREADS) {
        const int g = e / (HD / 2), dp = e % (HD / 2);
        uint32_t v = 0;
        if (g < G) v = __ldg(reinterpret_cast<const uint32_t*>(a.q + (qh0 + g) * HD) + dp);
        *reinterpret_cast<uint32_t*>(sh.qb16 + g * QBS + dp * 4) = v;
    }
    if (tid < HD) sh.c[tid] = __ldg(a.center + unit * HD + tid);
    if (tid < G) {
        sh.mrun[tid] = -INFINITY;
        sh.srun[tid] = 0.0f;
    }
    __syncthreads();
    if (tid < G * 32) {
        const int g = tid >> 5;
        const uint2 qq = *reinterpret_cast<const uint2*>(sh.qb16 + g * QBS + lane * 8);
        const float x0 = __uint_as_float(qq.x << 16), x1 = __uint_as_float(qq.x & 0xffff0000u);
        const float x2 = __uint_as_float(qq.y << 16), x3 = __uint_as_float(qq.y & 0xffff0000u);
        const float nn = warp_sum_f(x0 * x0 + x1 * x1 + x2 * x2 + x3 * x3);
        if (lane == 0) sh.qn[g] = sqrtf(nn);
    }

    if (is_static) {
        // ---- static piece: keys of T = [0,sink) U [n-local,n) (global positions) on this shard,
        // u = 1 (P:115 log [u, 1_t]); no dependency on the query codes
        const int64_t off = a.seq_offset, nl = a.n_local;
        const int64_t lo1 = max((int64_t)0, -off), hi1 = min(nl, (int64_t)a.sink - off);
        const int64_t len1 = hi1 > lo1 ? hi1 - lo1 : 0;
        int64_t lo2 = max((int64_t)0, a.n_global - a.local - off), hi2 = min(nl, a.n_global - off);
        if (len1 > 0 && lo2 < hi1) lo2 = hi1;
        const int64_t len2 = hi2 > lo2 ? hi2 - lo2 : 0;
        const int64_t p0 = (slot - a.nchunks) * (int64_t)KCHUNK;  // this piece's first T entry
        const int64_t nT = len1 + len2;
        const int64_t cnt = nT > p0 ? min((int64_t)KCHUNK, nT - p0) : 0;
        const int nmine = cnt > rank ? (int)((cnt - rank + CS - 1) / CS) : 0;
        for (int j = tid; j < nmine; j += DEC_THREADS) {
            const int64_t t = p0 + rank + (int64_t)j * CS;
            sh.keys[j] = (int)(t < len1 ? lo1 + t : lo2 + (t - len1));
            sh.bits[j] = 0x100u;
        }
        if (tid == 0) s_n = nmine;
        __syncthreads();
    } else {
        // ---- 2. wait for the query-encode kernel (programmatic dependent launch)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        MP_STAMP(1);
        // ---- 3. query masks: QX[c][g] = qbit ? 0 : ~0, so  P ^ QX = 1 where the key bit equals qbit
        for (int e = tid; e < G * a.KLw; e += DEC_THREADS) qb[e] = __ldcg(a.qbits + qh0 * a.KLw + e);
        __syncthreads();
        // thread per (head, 32 columns): one funnel-shifted word of query bits -> 32 masks
        for (int e = tid; e < G * ((ncols + 31) >> 5); e += DEC_THREADS) {
            const int g = e % G, c0 = (e / G) * 32;
            const int col = col0 + c0, wi = col >> 5, sft = col & 31;
            const uint32_t* qw = qb + g * a.KLw;
            uint32_t bits = qw[wi] >> sft;
            if (sft && wi + 1 < a.KLw) bits |= qw[wi + 1] << (32 - sft);
            const int nc = min(32, ncols - c0);
            for (int t = 0; t < nc; t++)
                qx[(c0 + t) * G + g] = (col + t < a.KL && ((bits >> t) & 1u)) ? 0u : 0xffffffffu;
        }
        __syncthreads();
        MP_STAMP(2);

        // ---- 4. scan
        uint32_t s1[G], s2[G];
#pragma unroll
        for (int g = 0; g < G; g++) s1[g] = s2[g] = 0u;
        for (int k = 0; k < n_my; k++) {
            const int sl = k % depth;
            const int grp = g0 + warp + k * NWARP;
            mbar_wait(mybar + sl, (uint32_t)((k / depth) & 1));
            uint4 P[QG];
            const uint4* src = reinterpret_cast<const uint4*>(myring + sl * GB) + lane;
#pragma unroll
            for (int t = 0; t < QG; t++) P[t] = src[t * 32];
            __syncwarp();
            if (lane == 0 && k + depth < n_my) {
                fence_proxy_async();
                const int ng = grp + depth * NWARP;
                mbar_arrive_expect_tx(mybar + sl, GB);
                bulk_g2s(myring + sl * GB, csrc + (size_t)ng * GB, GB, mybar + sl);
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
        }

        // ---- 5. combine: warps -> CTA (shared), CTAs -> cluster (DSMEM)
#pragma unroll
        for (int g = 0; g < G; g++) {
            s_part[warp][g][0][lane] = s1[g];
            s_part[warp][g][1][lane] = s2[g];
        }
        __syncthreads();
        MP_STAMP(3);
        uint32_t f1 = 0, f2 = 0;  // valid in threads tid < G*32: (g = tid/32, block = lane)
        if (tid < G * 32) {
            const int g = tid >> 5;
            for (int w = 0; w < NWARP; w++) {
                const uint32_t b1 = s_part[w][g][0][lane], b2 = s_part[w][g][1][lane];
                f2 |= b2 | (f1 & b1);
                f1 |= b1;
            }
        }
        __syncthreads();
        if (tid < G * 32) {
            s_part[0][tid >> 5][0][lane] = f1;
            s_part[0][tid >> 5][1][lane] = f2;
        }
        if (CS > 1) {
            cluster.sync();
            if (tid < G * 32) {
                const int g = tid >> 5;
                f1 = f2 = 0;
                for (int r = 0; r < CS; r++) {
                    const uint32_t* rp = cluster.map_shared_rank(&s_part[0][g][0][0], r);
                    const uint32_t b1 = rp[lane], b2 = rp[32 + lane];
                    f2 |= b2 | (f1 & b1);
                    f1 |= b1;
                }
            }
        }
        MP_STAMP(4);

        // ---- 6. final masks: S_g = count >= min_collisions restricted to D (T excluded)
        const int64_t cbase = chunk * KCHUNK;  // local index of the chunk's first key
        if (tid < 32) {
            const int64_t base = cbase + lane * 32;
            const uint32_t valid = range_mask(base, 0, a.n_local);
            s_tm[lane] = (range_mask(base, -a.seq_offset, (int64_t)a.sink - a.seq_offset) |
                          range_mask(base, a.n_global - a.local - a.seq_offset, a.n_global - a.seq_offset)) &
                         valid;
        }
        __syncthreads();
        if (tid < G * 32) {
            const int g = tid >> 5;
            uint32_t v = (a.minc == 1 ? f1 : f2);
            const int64_t base = cbase + lane * 32;
            v &= range_mask(base, 0, a.n_local) & ~s_tm[lane];
            s_sel[g][lane] = v;
            if (rank == 0) {
                int cnt = __popc(v);
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
                if (lane == 0) a.chunk_cnt[cgid * G + g] = cnt;
                if (a.s_mask) {
                    const int64_t nw = (a.n_local + 31) >> 5;
                    const int64_t widx = chunk * 32 + lane;
                    if (widx < nw) a.s_mask[(qh0 + g) * nw + widx] = v;
                }
            }
        }
        __syncthreads();
        // ---- 7. compaction (ascending) of union_g S_g; entry e goes to cluster rank e % CS.
        // warp 0: exclusive scan of the 32 block counts; then warp w emits blocks w, w+8, ..
        // (lane = key of the block, position = block base + popc of the lower set bits)
        if (warp == 0) {
            uint32_t u = 0;
#pragma unroll
            for (int g = 0; g < G; g++) u |= s_sel[g][lane];
            const int c = __popc(u);
            int incl = c;
#pragma unroll
            for (int m = 1; m < 32; m <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, m);
                if (lane >= m) incl += t;
            }
            s_base[lane] = incl - c;
            if (lane == 31) s_n = incl > rank ? (incl - rank + CS - 1) >> lcs : 0;
        }
        __syncthreads();
        for (int bl = warp; bl < 32; bl += NWARP) {
            uint32_t u = 0, sg[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                sg[g] = s_sel[g][bl];
                u |= sg[g];
            }
            if ((u >> lane) & 1u) {
                const int pos = s_base[bl] + __popc(u & ((1u << lane) - 1u));
                if ((pos & (CS - 1)) == rank) {
                    uint32_t bits = 0;
#pragma unroll
                    for (int g = 0; g < G; g++) bits |= ((sg[g] >> lane) & 1u) << g;
                    sh.keys[pos >> lcs] = (int)(cbase + bl * 32 + lane);
                    sh.bits[pos >> lcs] = (uint16_t)bits;
                }
            }
        }
        // remote s_part reads are done: let the cluster peers go on (we wait before exiting)
        if (CS > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        __syncthreads();
    }
    MP_STAMP(5);

    // ---- 8. gather + estimator over this CTA's entries
    float acc[2][4] = {{0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f}};
    gather_batched<K, G>(a, sh, ring, s_n, unit, acc);
    MP_STAMP(6);

    // ---- 9. this CTA's partial state (m, s, a) -> global parts[unit][slot*CS + rank]
    const int np = (int)per_unit * CS;
    float* pc = a.parts + (unit * np + slot * CS + rank) * G * PART;
    if ((lane >> 2) < G) {
#pragma unroll
        for (int nt = 0; nt < 2; nt++) {
            const int d0 = warp * 16 + nt * 8 + 2 * (lane & 3);
            *reinterpret_cast<float2*>(pc + (lane >> 2) * PART + 2 + d0) = make_float2(acc[nt][0], acc[nt][1]);
        }
    }
    if (tid < G) {
        pc[tid * PART] = sh.mrun[tid];
        pc[tid * PART + 1] = sh.srun[tid];
    }
    MP_STAMP(7);
    if (CS > 1 && !is_static) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    MP_STAMP(8);
    // static pieces touch shared global state (parts / counters) only after the
    // preceding grids' writes are visible
    if (is_static) asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---- 10. the last CTA of the unit merges all of its np partials (fixed order)
    __threadfence();
    __syncthreads();
    if (tid == 0) s_flag = atomicAdd(a.unit_ctr + unit, 1u) == (uint32_t)(np - 1);
    __syncthreads();
    if (!s_flag) return;
    __threadfence();
    MP_STAMP(9);
    long long tm0 = clk64();
    // The unit's partial block (np x G x PART floats, contiguous) comes into shared
    // memory by bulk copies -- one L2 round trip when it fits -- and every thread
    // (head g, dim pair dp) folds the partials in fixed order with an online
    // log-sum-exp merge ("recursive attention").
    __shared__ int s_cnt[G];
    __shared__ __align__(8) uint64_t s_mbar[2];
    const float* pu = a.parts + unit * (int64_t)np * G * PART;
    constexpr uint32_t PROW = G * PART * 4;  // bytes of one partial (all G heads)
    const int per_buf = max(1, (int)((uint32_t)a.dyn_bytes / 2u / PROW));
    const int nblk = (np + per_buf - 1) / per_buf;
    float* mbuf0 = reinterpret_cast<float*>(dsm);
    float* mbuf1 = mbuf0 + (size_t)per_buf * G * PART;
    auto issue = [&](int j) {  // block j -> buffer j & 1
        const int c0 = j * per_buf, cnt = min(per_buf, np - c0);
        mbar_arrive_expect_tx(&s_mbar[j & 1], (uint32_t)cnt * PROW);
        bulk_g2s((j & 1) ? mbuf1 : mbuf0, pu + (size_t)c0 * G * PART, (uint32_t)cnt * PROW, &s_mbar[j & 1]);
    };
    if (tid == 0) {
        mbar_init(&s_mbar[0], 1);
        mbar_init(&s_mbar[1], 1);
        fence_mbar_init();
        // other CTAs' generic-proxy writes (made visible by the counter) are read by the async proxy;
        // this CTA's own generic accesses to the buffers precede the bulk writes
        asm volatile("fence.proxy.async;" ::: "memory");
        for (int j = 0; j < 2 && j < nblk; j++) issue(j);
    }
    if (warp < G) {  // |S_g| summed over the unit's chunks
        int cnt = 0;
        for (int c = lane; c < (int)a.nchunks; c += 32) cnt += __ldcg(a.chunk_cnt + (unit * a.nchunks + c) * G + warp);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
        if (lane == 0) s_cnt[warp] = cnt;
    }
    __syncthreads();  // mbarrier inits visible before any wait
    constexpr int NI = (G * (HD / 2) + DEC_THREADS - 1) / DEC_THREADS;
    float Mx[NI], Sx[NI], A0[NI], A1[NI];
#pragma unroll
    for (int t = 0; t < NI; t++) Mx[t] = -INFINITY, Sx[t] = A0[t] = A1[t] = 0.0f;
    for (int j = 0; j < nblk; j++) {
        mbar_wait(&s_mbar[j & 1], (uint32_t)((j >> 1) & 1));
        const float* buf = (j & 1) ? mbuf1 : mbuf0;
        const int cnt = min(per_buf, np - j * per_buf);
        if (a.timeline && tid == 0 && j == 0) a.timeline[(size_t)blockIdx.x * 32 + 17] = (unsigned long long)(clk64() - tm0);
#pragma unroll
        for (int t = 0; t < NI; t++) {
            const int e = tid + t * DEC_THREADS;
            if (e < G * (HD / 2)) {
                const int g = e / (HD / 2), dp = e % (HD / 2);
                const float* pg = buf + (size_t)g * PART;
                float Mb = -INFINITY;  // block max, then one rescale of the running state
                for (int c = 0; c < cnt; c++) Mb = fmaxf(Mb, pg[(size_t)c * G * PART]);
                const float Mn = fmaxf(Mx[t], Mb);
                if (Mn != -INFINITY) {
                    const float fo = Mx[t] == -INFINITY ? 0.0f : __expf(Mx[t] - Mn);
                    float s_ = Sx[t] * fo, a0 = A0[t] * fo, a1 = A1[t] * fo;
#pragma unroll 4
                    for (int c = 0; c < cnt; c++) {
                        const float* pp = pg + (size_t)c * G * PART;
                        const float mc = pp[0];
                        const float f = mc == -INFINITY ? 0.0f : __expf(mc - Mn);
                        const float2 av = *reinterpret_cast<const float2*>(pp + 2 + 2 * dp);
                        s_ = fmaf(f, pp[1], s_);
                        a0 = fmaf(f, av.x, a0);
                        a1 = fmaf(f, av.y, a1);
                    }
                    Mx[t] = Mn, Sx[t] = s_, A0[t] = a0, A1[t] = a1;
                }
            }
        }
        if (j + 2 < nblk) {
            __syncthreads();  // buffer j & 1 fully read
            if (tid == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(j + 2);
            }
        }
    }
    if (a.timeline && tid == 0) a.timeline[(size_t)blockIdx.x * 32 + 18] = (unsigned long long)(clk64() - tm0);
#pragma unroll
    for (int t = 0; t < NI; t++) {
        const int e = tid + t * DEC_THREADS;
        if (e >= G * (HD / 2)) continue;
        const int g = e / (HD / 2), dp = e % (HD / 2);
        const float M = Mx[t], S = Sx[t];
        const int64_t row = qh0 + g;
        if (a.out)
            *reinterpret_cast<float2*>(a.out + row * HD + 2 * dp) =
                S > 0.0f ? make_float2(A0[t] / S, A1[t] / S) : make_float2(0.0f, 0.0f);
        if (a.partial) {
            *reinterpret_cast<float2*>(a.partial + row * PART + 2 + 2 * dp) = make_float2(A0[t], A1[t]);
            if (dp == 0) {
                a.partial[row * PART] = M;
                a.partial[row * PART + 1] = S;
            }
        }
        if (dp == 0 && !(S > 0.0f) && a.out) atomicOr(a.status, MAGICPIG_STATUS_DEGENERATE);
    }
    if (a.timeline && tid == 0) a.timeline[(size_t)blockIdx.x * 32 + 19] = (unsigned long long)(clk64() - tm0);
    if (tid < G && a.s_count) a.s_count[qh0 + tid] = s_cnt[tid];
    if (tid == 0) a.unit_ctr[unit] = 0u;
    MP_STAMP(10);
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

static size_t ring_bytes(int K, int depth) {
    size_t scan = (size_t)NWARP * depth * qg_of(K) * 512;
    size_t gath = 2 * RB * ROWB + RB * XS;
    return (scan > gath ? scan : gath + 127) & ~(size_t)127;
}

size_t decode_dyn_smem(int K, int G, int ncols_max, int depth, int KLw) {
    size_t qxb = ((size_t)ncols_max * G * 4 + 127) & ~(size_t)127;
    return qxb + ring_bytes(K, depth) + (size_t)NWARP * depth * 8 + (size_t)G * KLw * 4;
}

template <int K, int G>
static int launch_kg(DecodeArgs a, cudaStream_t st) {
    constexpr int TG = tg_of(K);
    const int maxg = (a.ngroups + a.tsplit - 1) / a.tsplit;
    const int ncols_max = maxg * TG * K;
    a.qx_bytes = (int)(((size_t)ncols_max * G * 4 + 127) & ~(size_t)127);
    a.depth = 3;
    if (decode_dyn_smem(K, G, ncols_max, 3, a.KLw) > 96 * 1024) a.depth = 2;
    a.ring_bytes = (int)ring_bytes(K, a.depth);
    size_t smem = decode_dyn_smem(K, G, ncols_max, a.depth, a.KLw);
    a.dyn_bytes = (int)smem;
    auto kern = decode_kernel<K, G>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MAGICPIG_ECUDA;
    const int64_t nblk = a.B * a.Hkv * (a.nchunks + a.nstatic) * a.tsplit;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nblk);
    cfg.blockDim = dim3(DEC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[2];
    int na = 0;
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    na++;
    if (a.tsplit > 1) {
        attrs[na].id = cudaLaunchAttributeClusterDimension;
        attrs[na].val.clusterDim.x = (unsigned)a.tsplit;
        attrs[na].val.clusterDim.y = 1;
        attrs[na].val.clusterDim.z = 1;
        na++;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
    count_launch(1);
    return e == cudaSuccess ? 0 : MAGICPIG_ECUDA;
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
