// decode5.cu -- MagicPIG decode step (Algorithm 1) as ONE
// persistent, warp-specialised kernel: one CTA per SM walks a contiguous range
// of tiles, a tile being either a 1024-key code chunk of a (sequence, kv head)
// unit or a piece (<= 1024 keys) of its static set T.
//
//   8 scan warps    each streams its own table groups (group j of every chunk tile
//                   goes to warp j % 8) through a private D-slot shared-memory
//                   ring with cp.async (16 B per lane, one commit group per table
//                   group, refilled as soon as a slot is read), starting before
//                   the query codes exist, so the stream overlaps the query-encode
//                   kernel (PDL).  (1-D cp.async.bulk copies and a single producer
//                   warp were both measured far below HBM rate: per-warp
//                   memory-level parallelism is what the stream needs.)
//                   Query(HT, q_code): per table and query head one LOP3
//                   per bit and a saturating counter -> the ">= 2 tables match"
//                   rule for 32 keys per lane; warps combine in shared
//                   memory; S_g restricted to D; ascending compaction of
//                   union_g S_g into one of two tile descriptors.
//   4 gather warps  per descriptor: K/V rows + |xbar_i| of the listed keys staged
//                   by bulk copies (3-deep), logits q.k/sqrt(d) and the
//                   hashed-vector dots on tensor cores (mma.sync bf16), p, log u
//                   (R5, R11), z = logit - log u, an online
//                   softmax whose a[g][d] accumulates on tensor cores (tf32 hi + lo weights).
//                   When the unit changes they flush the unit's partial state
//                   (m, s, |S|, a) and the last CTA of a unit merges its partials
//                   in fixed order (log-sum-exp, "recursive attention" P:171).
//
// Bucket mode (a.sbits != NULL, buckets.cu): S_g arrives as per-head bitmaps from the
// bucketed hash-table query; the scan warps skip the code stream and only compact.
// The unit merge keeps the records in registers (warp per head, lane = 4 dims, up to
// 24 records per load round) and the arrival is one acq_rel atomic (no full fences).
//
// Tiles of a unit: nstatic static pieces, then nchunks code chunks.  CTA i owns
// tiles [i*T/P, (i+1)*T/P), so the CTAs touching unit u are contiguous and the
// partial of (u, i) lives at record u + i: the records of a unit are contiguous.
// Counters self-clean (CUDA-graph replayable).
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.cuh"

namespace mp {
namespace v5 {

constexpr int NSW = 8;                          // scan warps
constexpr int NGW = 4;                          // gather warps
constexpr int THREADS = (NSW + NGW) * 32;       // 384
constexpr int GT0 = NSW * 32;                   // first gather thread
constexpr int RB = 32;                          // rows per gather batch
constexpr int NSTAGE = 3;                       // row stages in flight
constexpr int ROWB = 528;                       // k row | v row | |xbar| (+pad)
constexpr int XS = 272;                         // bf16 xbar tile row stride (bytes)
constexpr int QBS = 272;                        // bf16 query tile row stride (bytes)
constexpr int PREC = PREC5;                     // record per head: m, s, |S_g|, 0, a[128]
constexpr float INV_SQRT_D = 0.08838834764831845f;
constexpr int MB = 24;                          // unit merge: records loaded per round (<= 32)

// per-warp ring depth (table groups in flight per scan warp): ~104 KB of codes per CTA
__host__ __device__ constexpr int ring_depth(int QG) {
    return (104 * 1024) / (NSW * QG * 512) < 2 ? 2 : ((104 * 1024) / (NSW * QG * 512) > 16 ? 16 : (104 * 1024) / (NSW * QG * 512));
}

struct Desc {
    int keys[KCHUNK];      // local key index
    uint16_t bits[KCHUNK]; // bit g: key in S_g; 0x100: static (u = 1)
    int unit, n;
    int cnt[8];            // |S_g| of this tile
};

// per-CTA shared state that is not sized by the problem
struct __align__(16) Fixed {
    Desc desc[2];
    __align__(16) uint8_t qb16[8 * QBS];  // query rows of the gather's current unit (bf16, heads >= G zero)
    float c[HD];
    float qn[8], mrun[8], srun[8], scale[8], cnt[8];
    float Mm[8], Sm[8], Cm[8], fo[8];  // unit merge: running max, sum, |S|, block rescale
    float zl[RB][8], zd[RB][8], w[RB][8];
    uint32_t s_sel[8][32];
    uint32_t s_tm[32];
    int s_base[32];
    int s_cnt[8];
    int s_n;
    int flag;
    uint64_t dfull[2], dempty[2], rowbar[NSTAGE];
};

// mbarrier wait for long waits: try_wait without a suspend hint, backing off with nanosleep so
// that waiting warps do not take issue slots from the scan warps of the same SM
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    uint32_t ns = 32;
    while (!ok) {
        __nanosleep(ns);
        ns = ns < 512 ? ns * 2 : 512;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void bar_named(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t range_mask(int64_t base, int64_t lo, int64_t hi) {
    int64_t a = lo - base, b = hi - base;
    a = a < 0 ? 0 : (a > 32 ? 32 : a);
    b = b < 0 ? 0 : (b > 32 ? 32 : b);
    if (b <= a) return 0u;
    const uint32_t hiMask = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
    const uint32_t loMask = a >= 32 ? 0xffffffffu : ((1u << a) - 1u);
    return hiMask & ~loMask;
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}
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
// D(16x8 fp32) = A(16x8 tf32; rows 8..15 zero) * B(8x8 tf32) + D
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
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// first CTA whose tile range contains tile t (CTA i owns [i*T/P, (i+1)*T/P))
__device__ __forceinline__ int64_t owner_of(int64_t t, int64_t T, int64_t P) { return ((t + 1) * P - 1) / T; }

// static keys T of this shard (global positions [0,sink) U [n_global-local, n_global)) -> local ranges
struct StaticRanges {
    int64_t lo1, len1, lo2, len2;
};
__device__ __forceinline__ StaticRanges static_ranges(const DecodeArgs& a) {
    StaticRanges r;
    const int64_t off = a.seq_offset, nl = a.n_local;
    r.lo1 = max((int64_t)0, -off);
    const int64_t hi1 = min(nl, (int64_t)a.sink - off);
    r.len1 = hi1 > r.lo1 ? hi1 - r.lo1 : 0;
    r.lo2 = max((int64_t)0, a.n_global - a.local - off);
    const int64_t hi2 = min(nl, a.n_global - off);
    if (r.len1 > 0 && r.lo2 < hi1) r.lo2 = hi1;
    r.len2 = hi2 > r.lo2 ? hi2 - r.lo2 : 0;
    return r;
}

#define V5_STAMP(slot)                                                                                  \
    do {                                                                                                 \
        if (a.timeline) a.timeline[(size_t)blockIdx.x * 32 + (slot)] = (unsigned long long)(clock64() - t_start + 1); \
    } while (0)

template <int K, int G>
__global__ void __launch_bounds__(THREADS, 1) decode5_kernel(DecodeArgs a) {
    constexpr int TG = tg_of(K), QG = qg_of(K);
    constexpr uint32_t GB = QG * 512;  // bytes of one table group of one chunk
    extern __shared__ __align__(128) uint8_t dsm[];
    uint8_t* ring = dsm;                                                    // [NSW][D][GB]
    uint32_t* qx = reinterpret_cast<uint32_t*>(dsm + a.v5_off_qx);          // [ncolsP][G] match masks
    uint32_t* qbw = reinterpret_cast<uint32_t*>(dsm + a.v5_off_qbw);        // [G][KLw] packed query bits
    uint32_t* s_part = reinterpret_cast<uint32_t*>(dsm + a.v5_off_part);    // [NSW][G][2][32]
    uint8_t* rows = dsm + a.v5_off_rows;                                    // [NSTAGE][RB][ROWB]
    uint8_t* xt = dsm + a.v5_off_xt;                                        // [RB][XS]
    Fixed& f = *reinterpret_cast<Fixed*>(dsm + a.v5_off_fixed);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t T = a.v5_tiles, P = gridDim.x, tpu = a.nstatic + a.nchunks;
    const int64_t t0 = (int64_t)blockIdx.x * T / P, t1 = ((int64_t)blockIdx.x + 1) * T / P;
    const long long t_start = clock64();
    if (a.timeline && tid == 0) a.timeline[(size_t)blockIdx.x * 32] = gtimer();

    if (tid == 0) {
        mbar_init(&f.dfull[0], 1);
        mbar_init(&f.dfull[1], 1);
        mbar_init(&f.dempty[0], 1);
        mbar_init(&f.dempty[1], 1);
        for (int s = 0; s < NSTAGE; s++) mbar_init(&f.rowbar[s], NGW * 32);
        fence_mbar_init();
    }
    for (int e = tid; e < 8 * QBS / 4; e += THREADS) reinterpret_cast<uint32_t*>(f.qb16)[e] = 0u;
    __syncthreads();

    if (warp < NSW) {
        // ===================== scan warps
        constexpr int D = ring_depth(QG);
        uint8_t* myring = ring + (size_t)warp * D * GB;
        // this CTA's chunk tiles are the consecutive global chunks [gc0, gc1) (chunk tiles of a unit
        // follow its static pieces, chunks of consecutive units are adjacent in memory)
        auto chunks_before = [&](int64_t t) { return (t / tpu) * a.nchunks + max(t % tpu - a.nstatic, (int64_t)0); };
        const int64_t gc1 = chunks_before(t1);
        const size_t CB = (size_t)a.KLq * 512;  // code bytes per chunk
        const uint8_t* codes_b = reinterpret_cast<const uint8_t*>(a.codes);
        // issue iterator over this warp's (chunk, group) sequence: a source pointer that steps by
        // NSW groups and jumps to the next chunk; ring write/read pointers rotate (no divisions)
        int64_t it_c = chunks_before(t0);
        int it_j = warp;
        const bool has_groups = warp < a.ngroups;
        const uint8_t* it_src = codes_b + (size_t)it_c * CB + (size_t)warp * GB + lane * 16;
        uint8_t* const ring_end = myring + (size_t)D * GB;
        uint8_t* wr = myring + lane * 16;
        const uint8_t* rd = myring + lane * 16;
        auto issue = [&]() {
            if (has_groups && it_c < gc1) {
#pragma unroll
                for (int q = 0; q < QG; q++) cp_async16(wr + q * 512, it_src + q * 512);
                it_j += NSW;
                if (it_j >= a.ngroups) {
                    it_j = warp;
                    it_c++;
                    it_src = codes_b + (size_t)it_c * CB + (size_t)warp * GB + lane * 16;
                } else {
                    it_src += NSW * GB;
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            wr += GB;
            if (wr >= ring_end) wr -= (size_t)D * GB;
        };
        // bucket mode (a.sbits != NULL): S comes from the bucketed hash-table query (buckets.cu) as
        // per-head bitmaps; the scan warps only read them and compact (no code stream)
        const bool dense = a.sbits == nullptr;
        if (dense) {
#pragma unroll 1
            for (int k = 0; k < D; k++) issue();
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");  // query codes of the encode kernel
        const StaticRanges sr = static_ranges(a);
        const int ncolsP = a.ngroups * TG * K;
        int64_t cur_u = -1;
        int di = 0;
        long long acc_wait = 0, acc_desc = 0;
        for (int64_t t = t0; t < t1; t++, di++) {
            const int64_t u = t / tpu, r = t % tpu;
            const bool is_static = r < a.nstatic;
            const int64_t b = u / a.Hkv, hkv = u % a.Hkv;
            const int64_t qh0 = b * a.Hq + hkv * G;
            if (!is_static) {
                const int64_t chunk = r - a.nstatic;
                const int64_t cbase = chunk * KCHUNK;
                if (dense) {
                if (u != cur_u) {  // query masks of unit u: QX[c][g] = qbit ? 0 : ~0 (P ^ QX = 1 where bits agree)
                    bar_named(1, NSW * 32);
                    for (int e = tid; e < G * a.KLw; e += NSW * 32) qbw[e] = __ldcg(a.qbits + qh0 * a.KLw + e);
                    bar_named(1, NSW * 32);
                    for (int e = tid; e < ncolsP * G; e += NSW * 32) {
                        const int c = e / G, g = e % G;
                        qx[e] = (c < a.KL && ((qbw[g * a.KLw + (c >> 5)] >> (c & 31)) & 1u)) ? 0u : 0xffffffffu;
                    }
                    bar_named(1, NSW * 32);
                    cur_u = u;
                    if (tid == 0 && t == t0) V5_STAMP(1);
                }
                uint32_t s1[G], s2[G];
#pragma unroll
                for (int g = 0; g < G; g++) s1[g] = s2[g] = 0u;
                for (int j = warp; j < a.ngroups; j += NSW) {
                    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
                    __syncwarp();
                    uint4 Pw[QG];
#pragma unroll
                    for (int q = 0; q < QG; q++) Pw[q] = *reinterpret_cast<const uint4*>(rd + q * 512);
                    rd += GB;
                    if (rd >= ring_end) rd -= (size_t)D * GB;
                    __syncwarp();
                    issue();  // refill the slot just read
                    const uint32_t* wv = reinterpret_cast<const uint32_t*>(Pw);
                    const uint32_t* qrow = qx + (size_t)j * TG * K * G;
#pragma unroll
                    for (int tt = 0; tt < TG; tt++) {
                        if (TG == 1 || tt == 0 || j * TG + tt < a.L) {
                            uint32_t m[G];
#pragma unroll
                            for (int g = 0; g < G; g++) m[g] = 0xffffffffu;
#pragma unroll
                            for (int bb = 0; bb < K; bb++) {
                                const uint32_t w = wv[tt * K + bb];
                                const uint32_t* qp = qrow + (tt * K + bb) * G;
                                if constexpr (G % 4 == 0) {
#pragma unroll
                                    for (int g4 = 0; g4 < G / 4; g4++) {
                                        const uint4 qq = reinterpret_cast<const uint4*>(qp)[g4];
                                        m[4 * g4] &= w ^ qq.x;
                                        m[4 * g4 + 1] &= w ^ qq.y;
                                        m[4 * g4 + 2] &= w ^ qq.z;
                                        m[4 * g4 + 3] &= w ^ qq.w;
                                    }
                                } else {
#pragma unroll
                                    for (int g = 0; g < G; g++) m[g] &= w ^ qp[g];
                                }
                            }
#pragma unroll
                            for (int g = 0; g < G; g++) {
                                s2[g] |= s1[g] & m[g];
                                s1[g] |= m[g];
                            }
                        }
                    }
                }
                if (t == t0 && lane == 0) V5_STAMP(11 + warp);
#pragma unroll
                for (int g = 0; g < G; g++) {
                    s_part[((warp * G + g) * 2 + 0) * 32 + lane] = s1[g];
                    s_part[((warp * G + g) * 2 + 1) * 32 + lane] = s2[g];
                }
                }  // dense
                if (tid < 32) {
                    const int64_t base = cbase + lane * 32;
                    f.s_tm[lane] = (range_mask(base, -a.seq_offset, (int64_t)a.sink - a.seq_offset) |
                                    range_mask(base, a.n_global - a.local - a.seq_offset, a.n_global - a.seq_offset)) &
                                   range_mask(base, 0, a.n_local);
                }
                bar_named(1, NSW * 32);
                // warps -> CTA: (a1,a2)+(b1,b2) = (a1|b1, a2|b2|(a1&b1)); S_g = count >= minc on D
                if (tid < G * 32) {
                    const int g = tid >> 5;
                    uint32_t sel;
                    if (dense) {
                        uint32_t f1 = 0, f2 = 0;
#pragma unroll
                        for (int w = 0; w < NSW; w++) {
                            const uint32_t b1 = s_part[((w * G + g) * 2 + 0) * 32 + lane];
                            const uint32_t b2 = s_part[((w * G + g) * 2 + 1) * 32 + lane];
                            f2 |= b2 | (f1 & b1);
                            f1 |= b1;
                        }
                        sel = a.minc == 1 ? f1 : f2;
                    } else {
                        const int64_t nwb = (a.n_local + 31) >> 5, wi = chunk * 32 + lane;
                        sel = wi < nwb ? __ldcg(a.sbits + (qh0 + g) * nwb + wi) : 0u;
                    }
                    const int64_t base = cbase + lane * 32;
                    uint32_t v = sel & range_mask(base, 0, a.n_local) & ~f.s_tm[lane];
                    f.s_sel[g][lane] = v;
                    int cnt = __popc(v);
#pragma unroll
                    for (int m = 16; m >= 1; m >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
                    if (lane == 0) f.s_cnt[g] = cnt;
                    if (a.s_mask) {
                        const int64_t nw = (a.n_local + 31) >> 5;
                        const int64_t widx = chunk * 32 + lane;
                        if (widx < nw) a.s_mask[(qh0 + g) * nw + widx] = v;
                    }
                }
                bar_named(1, NSW * 32);
                if (warp == 0) {  // exclusive scan of the 32 block counts of union_g S_g
                    uint32_t uu = 0;
#pragma unroll
                    for (int g = 0; g < G; g++) uu |= f.s_sel[g][lane];
                    const int c = __popc(uu);
                    int incl = c;
#pragma unroll
                    for (int m = 1; m < 32; m <<= 1) {
                        const int tq = __shfl_up_sync(0xffffffffu, incl, m);
                        if (lane >= m) incl += tq;
                    }
                    f.s_base[lane] = incl - c;
                    if (lane == 31) f.s_n = incl;
                }
            }
            // descriptor slot free?  (consumed by the gather warps two tiles ago)
            long long td0 = clock64();
            if (di >= 2) mbar_wait_sleep(&f.dempty[di & 1], (uint32_t)(((di >> 1) - 1) & 1));
            acc_desc += clock64() - td0;
            bar_named(1, NSW * 32);
            Desc& D = f.desc[di & 1];
            if (is_static) {
                const int64_t p0 = r * (int64_t)KCHUNK, nT = sr.len1 + sr.len2;
                const int cnt = nT > p0 ? (int)min((int64_t)KCHUNK, nT - p0) : 0;
                for (int j = tid; j < cnt; j += NSW * 32) {
                    const int64_t tt = p0 + j;
                    D.keys[j] = (int)(tt < sr.len1 ? sr.lo1 + tt : sr.lo2 + (tt - sr.len1));
                    D.bits[j] = 0x100u;
                }
                if (tid == 0) {
                    D.n = cnt;
                    for (int g = 0; g < 8; g++) D.cnt[g] = 0;
                }
            } else {
                const int64_t cbase = (r - a.nstatic) * KCHUNK;
                for (int bl = warp; bl < 32; bl += NSW) {
                    uint32_t uu = 0, sg[G];
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        sg[g] = f.s_sel[g][bl];
                        uu |= sg[g];
                    }
                    if ((uu >> lane) & 1u) {
                        const int pos = f.s_base[bl] + __popc(uu & ((1u << lane) - 1u));
                        uint32_t bits = 0;
#pragma unroll
                        for (int g = 0; g < G; g++) bits |= ((sg[g] >> lane) & 1u) << g;
                        D.keys[pos] = (int)(cbase + bl * 32 + lane);
                        D.bits[pos] = (uint16_t)bits;
                    }
                }
                if (tid == 0) {
                    D.n = f.s_n;
                    for (int g = 0; g < 8; g++) D.cnt[g] = g < G ? f.s_cnt[g] : 0;
                }
            }
            if (tid == 0) D.unit = (int)u;
            bar_named(1, NSW * 32);
            if (tid == 0) {
                mbar_arrive(&f.dfull[di & 1]);
                if (t == t0) V5_STAMP(2);
            }
        }
        if (a.timeline && tid == 0) {
            a.timeline[(size_t)blockIdx.x * 32 + 23] = (unsigned long long)acc_wait;
            a.timeline[(size_t)blockIdx.x * 32 + 24] = (unsigned long long)acc_desc;
            a.timeline[(size_t)blockIdx.x * 32 + 25] = (unsigned long long)(clock64() - t_start);
        }
        return;
    }

    // ===================== gather warps (threads GT0 .. GT0 + 127)
    const int gtid = tid - GT0, gw = warp - NSW;
    float acc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; nt++) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.0f;
    int64_t cur_u = -1;
    uint32_t rseq = 0;      // row stages issued (buffer rseq % NSTAGE)
    const float* knorm_all = a.key_norm;

    // ---- flush the partial state of unit u; the last CTA of the unit merges all of its records
    auto flush = [&](int64_t u) {
        const int64_t tu0 = u * tpu, tu1 = tu0 + tpu - 1;
        const int64_t ilo = owner_of(tu0, T, P), ihi = owner_of(tu1, T, P);
        const int np = (int)(ihi - ilo + 1);
        float* rec = a.parts + (size_t)(u + blockIdx.x) * G * PREC;
        if (gtid == 0) V5_STAMP(21);
        {
            const int g = lane >> 2;
            if (g < G) {
#pragma unroll
                for (int nt = 0; nt < 4; nt++) {
                    const int d0 = gw * 32 + nt * 8 + 2 * (lane & 3);
                    *reinterpret_cast<float2*>(rec + g * PREC + 4 + d0) = make_float2(acc[nt][0], acc[nt][1]);
                }
            }
            if (gtid < G) {
                *reinterpret_cast<float4*>(rec + gtid * PREC) = make_float4(f.mrun[gtid], f.srun[gtid], f.cnt[gtid], 0.0f);
            }
        }
        // arrival: the named barrier orders the group's record stores before thread 0's acq_rel atomic
        // (release is cumulative), whose acquire half orders the merging CTA's loads after the other
        // CTAs' releases -- no full memory fences
        bar_named(2, NGW * 32);
        if (gtid == 0) {
            uint32_t old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.unit_ctr + u) : "memory");
            f.flag = old == (uint32_t)(np - 1);
        }
        bar_named(2, NGW * 32);
        if (gtid == 0) V5_STAMP(22);
        if (!f.flag) return;
        V5_STAMP(4);
        // warp per head, lane = 4 dims: the unit's records in fixed order, MB per round, all loads of a
        // round in flight together (record headers one per lane, broadcast by shuffles); running
        // log-sum-exp rescale between rounds
        const float* pu = a.parts + (size_t)(u + ilo) * G * PREC;
        const int64_t b = u / a.Hkv, hkv = u % a.Hkv;
        const int64_t qh0 = b * a.Hq + hkv * G;
#pragma unroll 1
        for (int g = gw; g < G; g += NGW) {
            float M = -INFINITY, S = 0.0f, C = 0.0f;
            float4 A = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll 1
            for (int c0 = 0; c0 < np; c0 += MB) {
                const int nr = min(MB, np - c0);
                float4 av[MB];
#pragma unroll
                for (int j = 0; j < MB; j++)
                    av[j] = j < nr ? __ldcg(reinterpret_cast<const float4*>(pu + ((size_t)(c0 + j) * G + g) * PREC + 4) + lane)
                                   : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                const float4 hd = lane < nr ? __ldcg(reinterpret_cast<const float4*>(pu + ((size_t)(c0 + lane) * G + g) * PREC))
                                            : make_float4(-INFINITY, 0.0f, 0.0f, 0.0f);
                float Mn = hd.x;
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) Mn = fmaxf(Mn, __shfl_xor_sync(0xffffffffu, Mn, m));
                Mn = fmaxf(Mn, M);
                const float fo = M == -INFINITY ? 0.0f : __expf(M - Mn);
                const float fc = hd.x == -INFINITY ? 0.0f : __expf(hd.x - Mn);
                S = S * fo + warp_sum_f(fc * hd.y);
                C += warp_sum_f(hd.z);
                A.x *= fo, A.y *= fo, A.z *= fo, A.w *= fo;
#pragma unroll
                for (int j = 0; j < MB; j++) {
                    const float fj = __shfl_sync(0xffffffffu, fc, j);
                    A.x = fmaf(fj, av[j].x, A.x);
                    A.y = fmaf(fj, av[j].y, A.y);
                    A.z = fmaf(fj, av[j].z, A.z);
                    A.w = fmaf(fj, av[j].w, A.w);
                }
                M = Mn;
            }
            if (gtid == 0 && g == 0) V5_STAMP(20);
            const int64_t row = qh0 + g;
            if (a.out) {
                const float inv = S > 0.0f ? 1.0f / S : 0.0f;
                *reinterpret_cast<float4*>(a.out + row * HD + 4 * lane) =
                    make_float4(A.x * inv, A.y * inv, A.z * inv, A.w * inv);
            }
            if (a.partial) {
                float* pp = a.partial + row * PART;
                *reinterpret_cast<float2*>(pp + 2 + 4 * lane) = make_float2(A.x, A.y);
                *reinterpret_cast<float2*>(pp + 4 + 4 * lane) = make_float2(A.z, A.w);
                if (lane == 0) pp[0] = M, pp[1] = S;
            }
            if (lane == 0) {
                if (a.s_count) a.s_count[row] = (int32_t)C;
                if (!(S > 0.0f) && a.out) atomicOr(a.status, MAGICPIG_STATUS_DEGENERATE);
            }
        }
        if (gtid == 0) a.unit_ctr[u] = 0u;
        bar_named(2, NGW * 32);  // merge buffer (row stages) free again
        V5_STAMP(5);
    };

    // ---- stage k: K/V rows and |xbar| of entries e0 .. e0+nb by cp.async (16 B pieces; a warp
    // moves one 256-B K row and one V row per step), completion counted on the stage's mbarrier
    auto stage = [&](const Desc& D, int e0, int nb, int64_t unit) {
        const uint32_t k = rseq++;
        uint8_t* buf = rows + (size_t)(k % NSTAGE) * RB * ROWB;
        uint64_t* bar = &f.rowbar[k % NSTAGE];
        const int part = lane;  // 16-B piece: 0..15 K row, 16..31 V row
#pragma unroll
        for (int it = 0; it < RB / NGW; it++) {
            const int rr = gw + NGW * it;
            if (rr < nb) {
                const int64_t i = D.keys[e0 + rr];
                const uint16_t* src = (part < 16 ? a.k : a.v) + (unit * a.n_local + i) * HD + (part & 15) * 8;
                cp_async16(buf + rr * ROWB + part * 16, src);
            }
        }
        if (gtid < nb) cp_async4(buf + gtid * ROWB + 512, knorm_all + unit * a.n_local + D.keys[e0 + gtid]);
        cp_async_mbar_arrive(bar);
    };

    // ---- query rows, |q_g|, centering vector of unit u; running state reset
    auto load_unit = [&](int64_t u) {
            const int64_t b = u / a.Hkv, hkv = u % a.Hkv;
            const int64_t qh0 = b * a.Hq + hkv * G;
            for (int e = gtid; e < G * (HD / 2); e += NGW * 32) {
                const int g = e / (HD / 2), dp = e % (HD / 2);
                *reinterpret_cast<uint32_t*>(f.qb16 + g * QBS + dp * 4) =
                    __ldg(reinterpret_cast<const uint32_t*>(a.q + (qh0 + g) * HD) + dp);
            }
            f.c[gtid] = __ldg(a.center + u * HD + gtid);
            if (gtid < G) {
                f.mrun[gtid] = -INFINITY;
                f.srun[gtid] = 0.0f;
                f.cnt[gtid] = 0.0f;
            }
            bar_named(2, NGW * 32);
            for (int g = gw; g < G; g += NGW) {  // |q_g|, warp per head
                const uint2 qq = *reinterpret_cast<const uint2*>(f.qb16 + g * QBS + lane * 8);
                const float x0 = __uint_as_float(qq.x << 16), x1 = __uint_as_float(qq.x & 0xffff0000u);
                const float x2 = __uint_as_float(qq.y << 16), x3 = __uint_as_float(qq.y & 0xffff0000u);
                const float nn = warp_sum_f(x0 * x0 + x1 * x1 + x2 * x2 + x3 * x3);
                if (lane == 0) f.qn[g] = sqrtf(nn);
            }
            bar_named(2, NGW * 32);
    };

    int di = 0;
    bool first_batch = true;
    long long acc_df = 0, acc_rw = 0;
    if (t0 < t1) {  // the first unit's data while the scan warps work
        cur_u = t0 / tpu;
        load_unit(cur_u);
    }
    for (int64_t t = t0; t < t1; t++, di++) {
        long long tg0 = clock64();
        mbar_wait_sleep(&f.dfull[di & 1], (uint32_t)((di >> 1) & 1));
        acc_df += clock64() - tg0;
        const Desc& D = f.desc[di & 1];
        const int64_t u = D.unit;
        if (u != cur_u) {
            flush(cur_u);
#pragma unroll
            for (int nt = 0; nt < 4; nt++) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.0f;
            load_unit(u);
            cur_u = u;
        }
        if (gtid < G) f.cnt[gtid] += (float)D.cnt[gtid];
        const int n = D.n;
        const int nbatch = (n + RB - 1) / RB;
        const uint32_t rbase = rseq;
        for (int bt = 0; bt < 2 && bt < nbatch; bt++) stage(D, bt * RB, min(RB, n - bt * RB), u);
        for (int bt = 0; bt < nbatch; bt++) {
            if (bt + 2 < nbatch) stage(D, (bt + 2) * RB, min(RB, n - (bt + 2) * RB), u);
            const uint32_t k = rbase + bt;
            const uint8_t* buf = rows + (size_t)(k % NSTAGE) * RB * ROWB;
            long long tr0 = clock64();
            mbar_wait_sleep(&f.rowbar[k % NSTAGE], (k / NSTAGE) & 1);
            acc_rw += clock64() - tr0;
            const int nb = min(RB, n - bt * RB);
            // (a) xbar = bf16(fl32(k - c)) of the batch rows (cvt.rn.bf16x2.f32)
#pragma unroll
            for (int it = 0; it < RB * (HD / 8) / (NGW * 32); it++) {
                const int e = gtid + NGW * 32 * it;
                const int rr = e / (HD / 8), dg = e % (HD / 8);
                const uint4 kv = *reinterpret_cast<const uint4*>(buf + rr * ROWB + dg * 16);
                const float4 c0 = *reinterpret_cast<const float4*>(&f.c[dg * 8]);
                const float4 c1 = *reinterpret_cast<const float4*>(&f.c[dg * 8 + 4]);
                const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
                const uint32_t kw[4] = {kv.x, kv.y, kv.z, kv.w};
                uint32_t xw[4];
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const __nv_bfloat162 xb =
                        __floats2bfloat162_rn(__fsub_rn(__uint_as_float(kw[q] << 16), cc[2 * q]),
                                              __fsub_rn(__uint_as_float(kw[q] & 0xffff0000u), cc[2 * q + 1]));
                    xw[q] = *reinterpret_cast<const uint32_t*>(&xb);
                }
                *reinterpret_cast<uint4*>(xt + rr * XS + dg * 16) = make_uint4(xw[0], xw[1], xw[2], xw[3]);
            }
            bar_named(2, NGW * 32);
            // (b) tensor cores: warp (mt, which) = 16 rows x {raw keys -> logits, xbar -> hashed dots}
            {
                const int mt = gw & 1, which = gw >> 1;
                const uint8_t* abase = which == 0 ? buf : xt;
                const int astride = which == 0 ? ROWB : XS;
                float d4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                const int arow = mt * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
                const uint32_t a_addr = smem_u32(abase + arow * astride + 16 * (lane >> 4));
                const uint32_t b_addr = smem_u32(f.qb16 + (lane & 7) * QBS + 16 * ((lane >> 3) & 1));
#pragma unroll
                for (int ks = 0; ks < HD / 16; ks++) {
                    uint32_t af[4], bfr[2];
                    ldsm_x4(af, a_addr + ks * 32);
                    ldsm_x2(bfr, b_addr + ks * 32);
                    mma16816(d4, af, bfr);
                }
                float(*dst)[8] = which == 0 ? f.zl : f.zd;
                const int r0 = mt * 16 + (lane >> 2), c0 = (lane & 3) * 2;
                dst[r0][c0] = d4[0];
                dst[r0][c0 + 1] = d4[1];
                dst[r0 + 8][c0] = d4[2];
                dst[r0 + 8][c0 + 1] = d4[3];
            }
            bar_named(2, NGW * 32);
            // (c) warp = head, lane = row: z = q.k/sqrt(d) - log u (u from the hashed vectors'
            // angle, R5), batch max, rescale factor and tf32 weights of the online softmax
#pragma unroll
            for (int g = gw; g < G; g += NGW) {
                const int rr = lane;
                float z = -INFINITY;
                if (rr < nb) {
                    const uint32_t sb = D.bits[bt * RB + rr];
                    const float logit = f.zl[rr][g] * INV_SQRT_D;
                    if (sb & 0x100u) {
                        z = logit;
                    } else if (sb & (1u << g)) {
                        const float xn = *reinterpret_cast<const float*>(buf + rr * ROWB + 512);
                        const float den = f.qn[g] * xn;
                        float cs = den > 0.0f ? __fdividef(f.zd[rr][g], den) : 0.0f;
                        cs = fminf(1.0f, fmaxf(-1.0f, cs));
                        const float p = 1.0f - acosf(cs) * 0.3183098861837907f;
                        z = logit - log_sampling_prob(p, K, a.L, a.minc);
                    }
                }
                float mb = z;
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, m));
                const float mo = f.mrun[g];
                const float mn = fmaxf(mo, mb);
                const float sc = (mo == -INFINITY) ? 0.0f : __expf(mo - mn);
                // fp32 weights; the P.V MMA takes them as tf32 hi + lo parts (two MMAs, ~2^-21 relative
                // per weight), so heavy cancellation in the value rows (|o| << |v|) stays accurate
                const float w = (z == -INFINITY) ? 0.0f : __expf(z - mn);
                const float wsum = warp_sum_f(w);
                f.w[rr][g] = w;
                __syncwarp();  // every lane has read f.mrun[g] before lane 0 replaces it
                if (lane == 0) {
                    f.scale[g] = sc;
                    f.srun[g] = f.srun[g] * sc + wsum;
                    f.mrun[g] = mn;
                }
            }
            bar_named(2, NGW * 32);
            // (d) a[g][d] = a * scale + sum_rows w * v on tensor cores (tf32 m16n8k8, fp32 accumulate):
            // A = weights [heads x rows], B = V [rows x dims]; warp gw owns dims 32 gw .. 32 gw + 31
            {
                const int g = lane >> 2;
                const float sc = g < G ? f.scale[g] : 0.0f;
#pragma unroll
                for (int nt = 0; nt < 4; nt++) {
                    acc[nt][0] *= sc;
                    acc[nt][1] *= sc;
                }
#pragma unroll
                for (int ks = 0; ks < RB / 8; ks++) {
                    const int k0 = ks * 8 + (lane & 3), k1 = k0 + 4;
                    const float w0 = g < G ? f.w[k0][g] : 0.0f, w1 = g < G ? f.w[k1][g] : 0.0f;
                    const float h0 = to_tf32(w0), h1 = to_tf32(w1);
                    const uint32_t a0 = __float_as_uint(h0), a2 = __float_as_uint(h1);
                    const uint32_t l0 = __float_as_uint(to_tf32(w0 - h0)), l2 = __float_as_uint(to_tf32(w1 - h1));
#pragma unroll
                    for (int nt = 0; nt < 4; nt++) {
                        const int dcol = gw * 32 + nt * 8 + (lane >> 2);
                        const uint32_t v0 =
                            k0 < nb ? (uint32_t)*reinterpret_cast<const uint16_t*>(buf + k0 * ROWB + 256 + dcol * 2) << 16 : 0u;
                        const uint32_t v1 =
                            k1 < nb ? (uint32_t)*reinterpret_cast<const uint16_t*>(buf + k1 * ROWB + 256 + dcol * 2) << 16 : 0u;
                        mma1688_tf32(acc[nt], a0, a2, v0, v1);
                        mma1688_tf32(acc[nt], l0, l2, v0, v1);
                    }
                }
            }
            bar_named(2, NGW * 32);  // stage buffer and weights reused
            if (first_batch && gtid == 0) {
                V5_STAMP(3);
                first_batch = false;
            }
        }
        if (gtid == 0) mbar_arrive(&f.dempty[di & 1]);
    }
    if (cur_u >= 0) flush(cur_u);
    if (gtid == 0) V5_STAMP(6);
    if (a.timeline && gtid == 0) {
        a.timeline[(size_t)blockIdx.x * 32 + 26] = (unsigned long long)acc_df;
        a.timeline[(size_t)blockIdx.x * 32 + 27] = (unsigned long long)acc_rw;
        a.timeline[(size_t)blockIdx.x * 32 + 28] = (unsigned long long)(clock64() - t_start);
    }
}

}  // namespace v5

// ---- host: shared-memory layout and launch
static size_t al128(size_t x) { return (x + 127) & ~(size_t)127; }


// fills the v5 layout fields of a; returns the dynamic smem bytes, or 0 if v5 does not fit
size_t decode5_layout(DecodeArgs& a, int G, int max_smem) {
    const int TG = tg_of(a.K), QG = qg_of(a.K);
    const size_t GB = (size_t)QG * 512;
    const int ncolsP = a.ngroups * TG * a.K;
    size_t fixed = al128((size_t)ncolsP * G * 4);  // qx
    const size_t o_qbw = fixed;
    fixed += al128((size_t)G * a.KLw * 4);
    const size_t o_part = fixed;
    fixed += al128((size_t)v5::NSW * G * 2 * 32 * 4);
    const size_t o_rows = fixed;
    fixed += al128((size_t)v5::NSTAGE * v5::RB * v5::ROWB);
    const size_t o_xt = fixed;
    fixed += al128((size_t)v5::RB * v5::XS);
    const size_t o_fixed = fixed;
    fixed += al128(sizeof(v5::Fixed));
    const size_t budget = (size_t)max_smem - 256;
    const size_t ring = al128((size_t)v5::NSW * v5::ring_depth(QG) * GB);
    if (ring + fixed > budget) return 0;
    a.v5_ns = v5::ring_depth(QG);
    a.v5_off_qx = (int)ring;
    a.v5_off_qbw = (int)(ring + o_qbw);
    a.v5_off_part = (int)(ring + o_part);
    a.v5_off_rows = (int)(ring + o_rows);
    a.v5_off_xt = (int)(ring + o_xt);
    a.v5_off_fixed = (int)(ring + o_fixed);
    a.v5_off_bars = (int)(ring + fixed);
    return ring + fixed;
}

template <int K, int G>
static int launch5_kg(DecodeArgs a, int nsm, int max_smem, cudaStream_t st) {
    const size_t smem = decode5_layout(a, G, max_smem);
    if (!smem) return MAGICPIG_EINVAL;
    auto kern = v5::decode5_kernel<K, G>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MAGICPIG_ECUDA;
    a.v5_hs = 1;
    a.v5_tiles = a.B * a.Hkv * (a.nstatic + a.nchunks);
    const int64_t P = a.v5_tiles < nsm ? a.v5_tiles : nsm;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)P);
    cfg.blockDim = dim3(v5::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
    count_launch(1);
    return e == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

template <int K>
static int launch5_k(const DecodeArgs& a, int G, int nsm, int max_smem, cudaStream_t st) {
    switch (G) {
        case 1: return launch5_kg<K, 1>(a, nsm, max_smem, st);
        case 2: return launch5_kg<K, 2>(a, nsm, max_smem, st);
        case 4: return launch5_kg<K, 4>(a, nsm, max_smem, st);
        case 8: return launch5_kg<K, 8>(a, nsm, max_smem, st);
    }
    return MAGICPIG_EINVAL;
}

int launch_decode5(const DecodeArgs& a, int nsm, int max_smem, cudaStream_t st) {
    const int G = (int)(a.Hq / a.Hkv);
    switch (a.K) {
#define MPK(k) \
    case k: return launch5_k<k>(a, G, nsm, max_smem, st);
        MPK(1) MPK(2) MPK(3) MPK(4) MPK(5) MPK(6) MPK(7) MPK(8)
        MPK(9) MPK(10) MPK(11) MPK(12) MPK(13) MPK(14) MPK(15) MPK(16)
#undef MPK
    }
    return MAGICPIG_EINVAL;
}

}  // namespace mp
