// estimate.cu -- the sampling-and-estimation half of a MagicPIG decode step
// (Algorithm 1), after the Query step has produced per-head
// S bitmaps (dense code scan, scan6.cu, or the bucketed tables, buckets.cu):
//
//   select_kernel    CTA per (sequence, kv head) unit: S_g restricted to the
//                    dynamic keys D (P:171 static cache excluded), the union over
//                    the G query heads of the unit, compacted in ascending key
//                    order into one list per unit (entry = key | head bits << 24),
//                    plus |S_g| per head and the list length.
//   estimate_kernel  the self-normalised importance-sampling estimator
//                        o_g = sum_{i in S_g u T} e^{z_i} v_i / sum e^{z_i},
//                        z_i = q_g.k_i / sqrt(d) - ln u_i      (u_i = 1 on T)
//                    with u_i the closed-form sampling probability (Eq. P:86-91)
//                    at the angle between the hashed vectors (reading R5).
//                    The unit lists (each preceded by the unit's static keys T,
//                    P:619) are concatenated; every warp of the persistent grid
//                    owns one contiguous range of that sequence (perfect balance,
//                    no producer warp), cut into 16-row slabs at unit boundaries.
//                    Per slab: K and V rows by one 256-B bulk copy each
//                    (cp.async.bulk, completion on a per-stage mbarrier, two
//                    stages per warp, entries of the next slab prefetched),
//                    logits q.k and hashed dots qbar.xbar on tensor cores
//                    (mma.sync bf16, xbar = bf16(fl32(k - c)) formed in the A
//                    fragments), ln u for the (row, head) items in S only
//                    (compacted over the warp), online softmax (rescale skipped
//                    when no running max moves), a[g][d] += w v on tensor cores
//                    with w split into bf16 hi + lo (fp32-accurate).
//                    When a warp leaves a unit it writes its record (m, s, a) to
//                    parts[u + warp]; the last warp of the unit (acq_rel counter)
//                    merges the unit's records in warp order (log-sum-exp,
//                    "recursive attention").  Counters self-clean, so the
//                    step is CUDA-graph replayable.
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.cuh"
#include "pieces.cuh"

namespace mp {
namespace v7 {

constexpr int NW = EST_WARPS;  // estimator warps per CTA
constexpr int SR = 16;         // rows per slab (mma M)
constexpr int NST = 2;         // row stages per warp
constexpr int SPW = 2;         // minimum slabs per active warp
constexpr int RP = 272;        // shared-memory row pitch (256 B + 16: ldmatrix conflict-free)
constexpr int PREC = PREC5;    // record per head: m, s, 0, 0, a[128]
constexpr int MB = 16;         // unit merge: records per load round
constexpr float INV_SQRT_D = 0.08838834764831845f;

struct __align__(128) WBuf {
    uint8_t k[NST][SR * RP];  // K rows
    uint8_t v[NST][SR * RP];  // V rows
    float xn[NST][SR];        // |xbar_i|
    float c[HD];              // -c: negated centering vector of the warp's current unit (16-B aligned)
    float items[SR * 8];      // compacted (row, head) items: cos in, ln u out
    uint16_t wt[16 * SR];     // PV B operand: [column n][row] bf16 (hi | lo weights)
    int key[NST][SR];         // local key index of each row
    uint32_t bits[NST][SR];   // bit g: key in S_g; 0x100: static (u = 1)
    uint64_t bar[NST];        // stage barriers: bulk-copy bytes + the lanes' cp.async (norms)
    long long su[NST];        // unit of the slab in the stage
    int snr[NST];             // rows of the slab
};
static_assert(offsetof(WBuf, c) % 16 == 0 && offsetof(WBuf, wt) % 16 == 0 && offsetof(WBuf, bar) % 8 == 0,
              "WBuf alignment");

__device__ __forceinline__ void cp4z(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_mbar_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
// D(16x8 fp32) += A(16x16 bf16, row) * B(16x8 bf16, col): exact products, fp32 accumulate
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// bf16 pair (lo = element d, hi = element d+1) -> bf16(fl32(k - c)) pair: one packed fp32 add (FADD2) of
// the negated centering vector, one cvt.rn.bf16x2
__device__ __forceinline__ uint32_t xbar_pair(uint32_t kw, float2 nc) {
    const float2 x = __fadd2_rn(make_float2(__uint_as_float(kw << 16), __uint_as_float(kw & 0xffff0000u)), nc);
    const __nv_bfloat162 xb = __floats2bfloat162_rn(x.x, x.y);
    return *reinterpret_cast<const uint32_t*>(&xb);
}
// ============================================================================ select
// One warp per piece = (unit, 1024-key chunk): S_g restricted to D for the unit's G heads (lane = 32-key
// word), the union compacted in ascending key order into the piece's list (capacity 1024), the list
// length and |S_g| of the piece.  Pieces are independent (no cross-chunk order is needed: the estimator
// concatenates them through a prefix over the piece lengths).
constexpr int SEL_WPB = 8;  // warps (pieces) per CTA

template <int G>
__global__ void __launch_bounds__(SEL_WPB * 32) select_kernel(EstArgs a) {
    asm volatile("griddepcontrol.launch_dependents;");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t pid = (int64_t)blockIdx.x * SEL_WPB + warp;
    if (pid >= a.B * a.Hkv * a.nchunks) return;
    const int64_t u = pid / a.nchunks, c = pid % a.nchunks;
    const int64_t b = u / a.Hkv, hkv = u % a.Hkv, qh0 = b * a.Hq + hkv * G;
    const int64_t nwb = (a.n_local + 31) >> 5;
    const StaticRanges sr = static_ranges(a);
    const int64_t wi = c * 32 + lane;
    const bool ok = wi < nwb;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // S bitmaps of the Query kernel
    uint32_t sg[G];
    if (a.sparts <= 1) {
#pragma unroll
        for (int g = 0; g < G; g++) sg[g] = ok ? __ldcg(a.sbits + (qh0 + g) * nwb + wi) : 0u;
    } else {
        // combine the id slices' (seen once, seen twice) words: (a1, a2) + (b1, b2) = (a1|b1, a2|b2|(a1&b1))
        const int P = a.sparts;
        uint32_t w1[G][BM_PARTS], w2[G][BM_PARTS];
#pragma unroll
        for (int g = 0; g < G; g++)
#pragma unroll
            for (int p = 0; p < BM_PARTS; p++) {
                const uint32_t* base = a.sbits + (((qh0 + g) * P + p) * 2) * nwb + wi;
                w1[g][p] = (ok && p < P) ? __ldcg(base) : 0u;
                w2[g][p] = (ok && p < P) ? __ldcg(base + nwb) : 0u;
            }
#pragma unroll
        for (int g = 0; g < G; g++) {
            uint32_t f1 = 0u, f2 = 0u;
#pragma unroll
            for (int p = 0; p < BM_PARTS; p++) {
                f2 |= w2[g][p] | (f1 & w1[g][p]);
                f1 |= w1[g][p];
            }
            sg[g] = a.minc > 1 ? f2 : f1;
        }
    }
    emit_piece<G>(a, sr, u, c, qh0, lane, sg);
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ============================================================================ estimate
// owner warp of entry e when E entries are split into W contiguous ranges [k E / W, (k+1) E / W)
__device__ __forceinline__ int64_t owner_of(int64_t e, int64_t E, int64_t W) { return ((e + 1) * W - 1) / E; }

template <int G>
__global__ void __launch_bounds__(NW * 32, 1) estimate_kernel(EstArgs a) {
    constexpr int NT = (2 * G + 7) / 8;  // PV n-tiles: columns [hi heads | lo heads | pad]
    extern __shared__ __align__(128) uint8_t dsm[];
    // pref[p] = first entry of piece p in the concatenation; piece u * P = unit u's static keys, piece
    // u * P + 1 + c = the list of chunk c of unit u (P = nchunks + 1)
    int* pref = reinterpret_cast<int*>(dsm);
    __shared__ int wsum[NW];
    WBuf* wbuf = reinterpret_cast<WBuf*>(dsm + a.off_wbuf);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t units = a.B * a.Hkv;
    const int64_t nwb = (a.n_local + 31) >> 5;
    const StaticRanges sr = static_ranges(a);
    const int nT = (int)(sr.len1 + sr.len2);
    const int P = (int)a.nchunks + 1;
    const int NP = (int)units * P;
    WBuf& wb = wbuf[warp];
    unsigned long long* tl = a.timeline ? a.timeline + ((size_t)blockIdx.x * NW + warp) * 16 : nullptr;
    auto stamp = [&](int i) {
        if (tl && lane == 0) tl[i] = gtimer();
    };
    stamp(0);

    if (lane < NST) mbar_init(&wb.bar[lane], 33);  // 1 expect_tx + 32 noinc arrivals
    // rows a slab does not load must hold finite values (0 * stale = 0); pad columns of the PV weights stay 0
    for (int e = lane; e < (int)offsetof(WBuf, c) / 16; e += 32)
        reinterpret_cast<uint4*>(&wb)[e] = make_uint4(0u, 0u, 0u, 0u);
    for (int e = lane; e < 8 * SR; e += 32) reinterpret_cast<uint32_t*>(wb.wt)[e] = 0u;
    fence_mbar_init();
    fence_proxy_async();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // lists of the select step
    stamp(1);

    {   // block exclusive scan of the piece lengths (coalesced loads into smem, then per-thread segments)
        for (int pp = tid; pp < NP; pp += NW * 32) {
            const int u = pp / P, cc = pp - u * P;
            pref[pp] = cc == 0 ? nT : __ldcg(a.pcnt + (int64_t)u * a.nchunks + cc - 1);
        }
        __syncthreads();
        const int per = (NP + NW * 32 - 1) / (NW * 32);
        const int p0 = min(NP, tid * per), p1 = min(NP, p0 + per);
        int sum = 0;
        for (int pp = p0; pp < p1; pp++) sum += pref[pp];
        const int incl = warp_incl_scan(sum, lane);
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int run = 0;
        for (int w = 0; w < warp; w++) run += wsum[w];
        run += incl - sum;
        for (int pp = p0; pp < p1; pp++) {
            const int len = pref[pp];
            pref[pp] = run;
            run += len;
        }
        if (tid == NW * 32 - 1) pref[NP] = run;
        __syncthreads();
    }
    const int64_t E = pref[NP];
    stamp(2);
    const int64_t Wt = (int64_t)gridDim.x * NW;
    int64_t Wa = (E + SR * SPW - 1) / (SR * SPW);
    Wa = Wa < 1 ? 1 : (Wa > Wt ? Wt : Wa);
    // record table for the merge kernel: unit u's records are parts[u + k], k = k_lo .. k_lo + np - 1
    if (blockIdx.x == 0) {
        for (int64_t u = tid; u < units; u += NW * 32) {
            int2 r = make_int2(0, 0);
            const int64_t e0 = pref[u * P], e1 = pref[(u + 1) * P];
            if (e1 > e0) {
                const int64_t k_lo = owner_of(e0, E, Wa), k_hi = owner_of(e1 - 1, E, Wa);
                r = make_int2((int)k_lo, (int)(k_hi - k_lo + 1));
            }
            a.urec[u] = r;
        }
    }
    asm volatile("griddepcontrol.launch_dependents;");
    if (E == 0) return;
    const int64_t kw = (int64_t)warp * gridDim.x + blockIdx.x;  // active warps spread over the CTAs first
    if (kw >= Wa) return;
    const int64_t e_lo = kw * E / Wa, e_hi = (kw + 1) * E / Wa;
    if (e_lo >= e_hi) return;

    // ---------------------------------------------------------------- per-warp pipeline
    const int g4 = lane >> 2, t4 = lane & 3;
    const int h0 = 2 * t4, h1 = 2 * t4 + 1;  // logit-side heads of this thread (columns of the m16n8 D)
    auto pv_head = [&](int nt, int i) {
        const int n = nt * 8 + 2 * t4 + i;
        return n < G ? n : (n < 2 * G ? n - G : -1);
    };
    auto find_piece = [&](int64_t e) {  // last piece p with pref[p] <= e (pref nondecreasing, pref[0] = 0)
        int lo = 0, hi = NP;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pref[mid] <= e) lo = mid;
            else hi = mid;
        }
        return lo;
    };

    // plans of the next two slabs to issue (unit, rows, this lane's entry), so the entry loads of a slab
    // are in flight one whole slab before its row copies are issued
    struct Plan {
        int64_t u;
        int nr, key;
        uint32_t bits;
    };
    int ps = find_piece(e_lo);  // piece holding the plan cursor
    int64_t pcur = e_lo;
    auto plan_next = [&](Plan& PL) {
        PL.nr = 0;
        PL.key = 0;
        PL.bits = 0u;
        if (pcur >= e_hi) return;
        while (pref[ps + 1] <= pcur) ps++;
        const int u = ps / P;
        const int64_t uend = min(e_hi, (int64_t)pref[(u + 1) * P]);
        PL.u = u;
        PL.nr = (int)min((int64_t)SR, uend - pcur);
        const int r = lane & 15;
        if (r < PL.nr) {
            const int e = (int)(pcur + r);
            int pi = ps;
            while (pref[pi + 1] <= e) pi++;
            const int j = e - pref[pi], cc = pi - u * P;
            if (cc == 0) {
                PL.key = (int)(j < sr.len1 ? sr.lo1 + j : sr.lo2 + (j - sr.len1));
                PL.bits = 0x100u | ((1u << G) - 1u);
            } else {
                const uint32_t ent = __ldcg(a.ents + ((int64_t)u * a.nchunks + cc - 1) * KCHUNK + j);
                PL.key = (int)(ent & 0xffffffu);
                PL.bits = ent >> 24;
            }
        }
        pcur += PL.nr;
    };
    Plan P0, P1;
    int issued = 0, computed = 0;
    auto issue = [&]() {
        if (P0.nr == 0) return;
        const int st = issued % NST;
        const int r = lane & 15;
        const int nr = P0.nr;
        if (lane < 16) {
            wb.key[st][r] = P0.key;
            wb.bits[st][r] = P0.bits;
        }
        if (lane == 0) {
            wb.su[st] = P0.u;
            wb.snr[st] = nr;
        }
        uint64_t* bar = &wb.bar[st];
        fence_proxy_async();  // this stage's earlier ldmatrix reads before the async-proxy refill
        if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)nr * 512u);
        __syncwarp();
        if (r < nr) {
            const int64_t row = P0.u * a.n_local + P0.key;
            if (lane < 16) {
                bulk_g2s(wb.k[st] + r * RP, a.k + row * HD, 256, bar);
                cp4z(&wb.xn[st][r], a.key_norm + row, true);
            } else {
                bulk_g2s(wb.v[st] + r * RP, a.v + row * HD, 256, bar);
            }
        }
        cp_mbar_arrive_noinc(bar);
        issued++;
        P0 = P1;
        plan_next(P1);
    };

    float acc[8][NT][4];
    float m0 = -INFINITY, m1 = -INFINITY, s0 = 0.0f, s1 = 0.0f;
    uint32_t qf[8][2];
    float qn0 = 0.0f, qn1 = 0.0f;
    auto reset_state = [&]() {
#pragma unroll
        for (int dt = 0; dt < 8; dt++)
#pragma unroll
            for (int nt = 0; nt < NT; nt++)
                acc[dt][nt][0] = acc[dt][nt][1] = acc[dt][nt][2] = acc[dt][nt][3] = 0.0f;
        m0 = m1 = -INFINITY;
        s0 = s1 = 0.0f;
    };
    auto load_unit = [&](int64_t u) {
        const int64_t b = u / a.Hkv, hkv = u % a.Hkv;
        const int64_t qh0 = b * a.Hq + hkv * G;
        float sq = 0.0f;
#pragma unroll
        for (int ks = 0; ks < 8; ks++) {
            const int d0 = 16 * ks + 2 * t4;
            if (g4 < G) {
                const uint32_t* qr = reinterpret_cast<const uint32_t*>(a.q + (qh0 + g4) * HD);
                qf[ks][0] = __ldg(qr + d0 / 2);
                qf[ks][1] = __ldg(qr + d0 / 2 + 4);
            } else {
                qf[ks][0] = qf[ks][1] = 0u;
            }
#pragma unroll
            for (int i = 0; i < 2; i++) {
                const float lo = __uint_as_float(qf[ks][i] << 16), hi = __uint_as_float(qf[ks][i] & 0xffff0000u);
                sq = fmaf(lo, lo, fmaf(hi, hi, sq));
            }
        }
        __syncwarp();  // the previous unit's readers of wb.c are done
        const float4 cv = __ldg(reinterpret_cast<const float4*>(a.center + u * HD) + lane);
        *reinterpret_cast<float4*>(&wb.c[4 * lane]) = make_float4(-cv.x, -cv.y, -cv.z, -cv.w);
        __syncwarp();
        // |q_g|^2: lanes 4g .. 4g+3 hold head g's 128 elements
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
        const float qn = sqrtf(sq);
        qn0 = __shfl_sync(0xffffffffu, qn, 4 * h0);
        qn1 = __shfl_sync(0xffffffffu, qn, 4 * (h1 & 7));
    };

    // leave unit u: record (m, s, a) of this warp -> parts[u + kw] (merged by merge_kernel)
    auto flush = [&](int64_t u) {
        float* rec = a.parts + (size_t)(u + kw) * G * PREC;
#pragma unroll
        for (int dt = 0; dt < 8; dt++) {
#pragma unroll
            for (int i = 0; i < 2; i++) {
                // hi column of head h at (nt = 0, i); its lo column G + h
                float hiA = acc[dt][0][i], hiB = acc[dt][0][2 + i], loA, loB;
                if constexpr (G == 8) {
                    loA = acc[dt][NT - 1][i];
                    loB = acc[dt][NT - 1][2 + i];
                } else if constexpr (G == 4) {
                    loA = __shfl_down_sync(0xffffffffu, hiA, 2);
                    loB = __shfl_down_sync(0xffffffffu, hiB, 2);
                } else if constexpr (G == 2) {
                    loA = __shfl_down_sync(0xffffffffu, hiA, 1);
                    loB = __shfl_down_sync(0xffffffffu, hiB, 1);
                } else {
                    loA = acc[dt][0][1];
                    loB = acc[dt][0][3];
                }
                const int h = 2 * t4 + i;
                const bool own = (G == 1) ? (t4 == 0 && i == 0) : (h < G);
                if (own) {
                    __stcg(rec + h * PREC + 4 + dt * 16 + g4, hiA + loA);
                    __stcg(rec + h * PREC + 4 + dt * 16 + g4 + 8, hiB + loB);
                }
            }
        }
        if (g4 == 0) {
            if (h0 < G) __stcg(reinterpret_cast<float2*>(rec + h0 * PREC), make_float2(m0, s0));
            if (h1 < G) __stcg(reinterpret_cast<float2*>(rec + h1 * PREC), make_float2(m1, s1));
        }
    };

    plan_next(P0);
    plan_next(P1);
    stamp(3);
#pragma unroll 1
    for (int i = 0; i < NST; i++) issue();
    stamp(4);
    int64_t cur_u = -1;
    reset_state();
#pragma unroll 1
    while (computed < issued) {
        const int st = computed % NST;
        const int64_t su = wb.su[st];
        const int nr = wb.snr[st];
        if (su != cur_u) {
            if (cur_u >= 0) {
                flush(cur_u);
                reset_state();
            }
            cur_u = su;
            load_unit(su);
        }
        mbar_wait(&wb.bar[st], (uint32_t)((computed / NST) & 1));
        if (computed == 0) stamp(5);
        const uint8_t* Kt = wb.k[st];
        const uint8_t* Vt = wb.v[st];

        // (1) logits l = q.k and hashed dots qbar.xbar (mma.sync bf16, fp32 accumulate)
        float dl[4] = {0.0f, 0.0f, 0.0f, 0.0f}, dx[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        {
            const int mi = lane >> 3, rr = lane & 7;
            const int row = (mi & 1) * 8 + rr;
            const uint32_t kbase = smem_u32(Kt + row * RP + (mi >> 1) * 16);
#pragma unroll
            for (int ks = 0; ks < 8; ks++) {
                uint32_t af[4];
                ldsm_x4(af, kbase + ks * 32);
                mma16816(dl, af, qf[ks][0], qf[ks][1]);
                const float2 ca = *reinterpret_cast<const float2*>(&wb.c[16 * ks + 2 * t4]);
                const float2 cb = *reinterpret_cast<const float2*>(&wb.c[16 * ks + 2 * t4 + 8]);
                uint32_t xf[4];
                xf[0] = xbar_pair(af[0], ca);
                xf[1] = xbar_pair(af[1], ca);
                xf[2] = xbar_pair(af[2], cb);
                xf[3] = xbar_pair(af[3], cb);
                mma16816(dx, xf, qf[ks][0], qf[ks][1]);
            }
        }
        // (2) items (row, head): ra = g4 (dl[0], dl[1]), rb = g4 + 8 (dl[2], dl[3]); heads h0, h1
        const uint32_t ba = wb.bits[st][g4], bb = wb.bits[st][g4 + 8];
        const float xna = wb.xn[st][g4], xnb = wb.xn[st][g4 + 8];
        const uint32_t bt[4] = {ba, ba, bb, bb};
        const int hh[4] = {h0, h1, h0, h1};
        bool need[4];
        float cs[4];
        {
            const float qn[4] = {qn0, qn1, qn0, qn1};
            const float xn[4] = {xna, xna, xnb, xnb};
#pragma unroll
            for (int i = 0; i < 4; i++) {
                need[i] = hh[i] < G && !(bt[i] & 0x100u) && ((bt[i] >> hh[i]) & 1u);
                const float den = qn[i] * xn[i];
                const float c = den > 0.0f ? __fdividef(dx[i], den) : 0.0f;
                cs[i] = fminf(1.0f, fmaxf(-1.0f, c));
            }
        }
        // ln u of the items that need it, compacted over the warp (one MUFU chain per lane per round)
        float lu[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        {
            int base = 0, pos[4];
            const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const uint32_t bal = __ballot_sync(0xffffffffu, need[i]);
                pos[i] = base + __popc(bal & lt);
                base += __popc(bal);
                if (need[i]) wb.items[pos[i]] = cs[i];
            }
            __syncwarp();
            for (int e = lane; e < base; e += 32) {
                const float p = 1.0f - acosf(wb.items[e]) * 0.3183098861837907f;
                wb.items[e] = log_sampling_prob_lut(a.lutab, p, a.K, a.L, a.minc);
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; i++)
                if (need[i]) lu[i] = wb.items[pos[i]];
        }
        float z[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const float l = dl[i] * INV_SQRT_D;
            z[i] = (hh[i] < G && (bt[i] & 0x100u)) ? l : (need[i] ? l - lu[i] : -INFINITY);
        }
        if (a.weighted) {
            const int64_t b = cur_u / a.Hkv, hkv = cur_u % a.Hkv, qh0 = b * a.Hq + hkv * G;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int r = (i >> 1) ? g4 + 8 : g4;
                if (z[i] != -INFINITY && r < nr) {
                    const int key = wb.key[st][r];
                    atomicOr(a.weighted + (qh0 + hh[i]) * nwb + (key >> 5), 1u << (key & 31));
                }
            }
        }
        // (3) online softmax per head (rows of head h are spread over the 8 lanes with the same t4)
        float mx0 = fmaxf(z[0], z[2]), mx1 = fmaxf(z[1], z[3]);
#pragma unroll
        for (int m = 4; m <= 16; m <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, m));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, m));
        }
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const bool moved = __any_sync(0xffffffffu, mn0 != m0 || mn1 != m1);
        const float al0 = m0 == -INFINITY ? 0.0f : __expf(m0 - mn0);
        const float al1 = m1 == -INFINITY ? 0.0f : __expf(m1 - mn1);
        const float mnn[4] = {mn0, mn1, mn0, mn1};
        __nv_bfloat16 whi[4], wlo[4];
        float wsum0 = 0.0f, wsum1 = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const float w = z[i] == -INFINITY ? 0.0f : __expf(z[i] - mnn[i]);
            whi[i] = __float2bfloat16_rn(w);
            wlo[i] = __float2bfloat16_rn(w - __bfloat162float(whi[i]));
            const float we = __bfloat162float(whi[i]) + __bfloat162float(wlo[i]);
            if (i & 1) wsum1 += we;
            else wsum0 += we;
        }
#pragma unroll
        for (int m = 4; m <= 16; m <<= 1) {
            wsum0 += __shfl_xor_sync(0xffffffffu, wsum0, m);
            wsum1 += __shfl_xor_sync(0xffffffffu, wsum1, m);
        }
        s0 = s0 * al0 + wsum0;
        s1 = s1 * al1 + wsum1;
        m0 = mn0;
        m1 = mn1;
        // weights -> PV B operand [n][row]: hi in column h, lo in column G + h
        {
            __nv_bfloat16* wt = reinterpret_cast<__nv_bfloat16*>(wb.wt);
            const int rows[4] = {g4, g4, g4 + 8, g4 + 8};
#pragma unroll
            for (int i = 0; i < 4; i++) {
                if (hh[i] < G) {
                    wt[hh[i] * SR + rows[i]] = whi[i];
                    wt[(G + hh[i]) * SR + rows[i]] = wlo[i];
                }
            }
        }
        __syncwarp();
        // (4) rescale the running a (per PV column: the head's alpha from the lane that holds it)
        if (moved) {
#pragma unroll
            for (int nt = 0; nt < NT; nt++)
#pragma unroll
                for (int i = 0; i < 2; i++) {
                    const int h = pv_head(nt, i);
                    const int src = (lane & ~3) | ((h < 0 ? 0 : h) >> 1);
                    const float x0 = __shfl_sync(0xffffffffu, al0, src);
                    const float x1 = __shfl_sync(0xffffffffu, al1, src);
                    const float al = h < 0 ? 0.0f : ((h & 1) ? x1 : x0);
#pragma unroll
                    for (int dt = 0; dt < 8; dt++) {
                        acc[dt][nt][i] *= al;
                        acc[dt][nt][2 + i] *= al;
                    }
                }
        }
        // (5) a[d][n] += V^T[d][rows] W[rows][n] on tensor cores (V^T fragments by ldmatrix.trans)
        {
            uint32_t bw[NT][2];
            const uint32_t* wt32 = reinterpret_cast<const uint32_t*>(wb.wt);
#pragma unroll
            for (int nt = 0; nt < NT; nt++) {
                bw[nt][0] = wt32[((nt * 8 + g4) * SR + 2 * t4) >> 1];
                bw[nt][1] = wt32[((nt * 8 + g4) * SR + 2 * t4 + 8) >> 1];
            }
            const int mi = lane >> 3, rr = lane & 7;
            const int row = (mi >> 1) * 8 + rr;
            const uint32_t vbase = smem_u32(Vt + row * RP + (mi & 1) * 16);
#pragma unroll
            for (int dt = 0; dt < 8; dt++) {
                uint32_t af[4];
                ldsm_x4_t(af, vbase + dt * 32);
#pragma unroll
                for (int nt = 0; nt < NT; nt++) mma16816(acc[dt][nt], af, bw[nt][0], bw[nt][1]);
            }
        }
        __syncwarp();  // stage buffer, weight tile and items free
        computed++;
        issue();  // refill the stage just consumed
    }
    stamp(6);
    if (tl && lane == 0) tl[11] = (unsigned long long)computed;
    stamp(7);
    if (cur_u >= 0) flush(cur_u);
    stamp(10);
}

// ============================================================================ merge
// CTA per (sequence, query head), thread per dimension: the log-sum-exp merge of the unit's warp records
// in record order ("recursive attention"): M = max m_j, S = sum s_j e^{m_j - M},
// A = sum a_j e^{m_j - M}, o = A / S.  PDL: waits for the estimator grid.
// MS slices of HD threads: slice z merges records j = z, z + MS, ... (RB per load round), then slice 0
// combines the MS partial states from shared memory in slice order (long contexts at small batch give a
// unit hundreds of records: B=1 128K, 12 warps/SM -> 222 per unit)
constexpr int MS = 4;
template <int G>
__global__ void __launch_bounds__(HD * MS) merge_kernel(EstArgs a) {
    constexpr int RB = 16;  // records per load round (all loads of a round in flight together)
    __shared__ int hsum[HD / 32];
    __shared__ float pm[MS][HD], ps[MS][HD], pa[MS][HD];
    const int64_t row = blockIdx.x, b = row / a.Hq, hq = row % a.Hq;
    const int64_t g = hq % G, u = b * a.Hkv + hq / G;
    const int d = threadIdx.x % HD, z = threadIdx.x / HD, lane = threadIdx.x & 31;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");  // the next step's encode (touches nothing read here)
    if (z == 0) {  // |S_g| = sum over the unit's pieces (select step)
        int hc = 0;
        for (int64_t c = d; c < a.nchunks; c += HD) hc += __ldcg(a.hpc + row * a.nchunks + c);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) hc += __shfl_xor_sync(0xffffffffu, hc, m);
        if (lane == 0) hsum[d >> 5] = hc;
    }
    const int2 rr = __ldcg(a.urec + u);
    const float* base = a.parts + ((size_t)(u + rr.x) * G + g) * PREC;
    const size_t stride = (size_t)G * PREC;
    const int np = rr.y;
    float M = -INFINITY, S = 0.0f, A = 0.0f;
#pragma unroll 1
    for (int j0 = z; j0 < np; j0 += RB * MS) {
        float mj[RB], sj[RB], aj[RB];
#pragma unroll
        for (int j = 0; j < RB; j++) {
            const int jj = j0 + j * MS;
            const bool ok = jj < np;
            const float* rp = base + (size_t)jj * stride;
            mj[j] = ok ? __ldcg(rp) : -INFINITY;
            sj[j] = ok ? __ldcg(rp + 1) : 0.0f;
            aj[j] = ok ? __ldcg(rp + 4 + d) : 0.0f;
        }
        float Mn = M;
#pragma unroll
        for (int j = 0; j < RB; j++) Mn = fmaxf(Mn, mj[j]);
        const float fo = M == -INFINITY ? 0.0f : __expf(M - Mn);
        S *= fo;
        A *= fo;
#pragma unroll
        for (int j = 0; j < RB; j++) {
            const float f = mj[j] == -INFINITY ? 0.0f : __expf(mj[j] - Mn);
            S = fmaf(f, sj[j], S);
            A = fmaf(f, aj[j], A);
        }
        M = Mn;
    }
    pm[z][d] = M, ps[z][d] = S, pa[z][d] = A;
    __syncthreads();
    if (z != 0) return;
    M = pm[0][d], S = ps[0][d], A = pa[0][d];
#pragma unroll
    for (int y = 1; y < MS; y++) {
        const float My = pm[y][d];
        const float Mn = fmaxf(M, My);
        if (Mn == -INFINITY) continue;
        const float f0 = M == -INFINITY ? 0.0f : __expf(M - Mn), f1 = My == -INFINITY ? 0.0f : __expf(My - Mn);
        S = S * f0 + ps[y][d] * f1;
        A = A * f0 + pa[y][d] * f1;
        M = Mn;
    }
    if (a.out) a.out[row * HD + d] = S > 0.0f ? A * (1.0f / S) : 0.0f;
    if (a.partial) {
        float* pp = a.partial + row * PART;
        pp[2 + d] = A;
        if (d == 0) pp[0] = M, pp[1] = S;
    }
    if (d == 0) {
        if (a.s_count) a.s_count[row] = hsum[0] + hsum[1] + hsum[2] + hsum[3];
        if (!(S > 0.0f) && a.out) atomicOr(a.status, MAGICPIG_STATUS_DEGENERATE);
    }
}

}  // namespace v7

// ---- host
static size_t al128e(size_t x) { return (x + 127) & ~(size_t)127; }

size_t estimate_layout(EstArgs& a, int G) {
    (void)G;
    const size_t pieces = (size_t)(a.B * a.Hkv * (a.nchunks + 1));
    a.off_wbuf = (int)al128e((pieces + 1) * 4);
    return a.off_wbuf + sizeof(v7::WBuf) * v7::NW;
}

template <int G>
static int launch_select_g(const EstArgs& a, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    const int64_t pieces = a.B * a.Hkv * a.nchunks;
    cfg.gridDim = dim3((unsigned)((pieces + v7::SEL_WPB - 1) / v7::SEL_WPB));
    cfg.blockDim = dim3(v7::SEL_WPB * 32);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, v7::select_kernel<G>, a);
    count_launch(1);
    return e == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

int launch_select(const EstArgs& a, cudaStream_t st) {
    switch ((int)(a.Hq / a.Hkv)) {
        case 1: return launch_select_g<1>(a, st);
        case 2: return launch_select_g<2>(a, st);
        case 4: return launch_select_g<4>(a, st);
        case 8: return launch_select_g<8>(a, st);
    }
    return MAGICPIG_EINVAL;
}

template <int G>
static int launch_estimate_g(EstArgs a, int nsm, int max_smem, cudaStream_t st) {
    const size_t smem = estimate_layout(a, G);
    if (smem > (size_t)max_smem) return MAGICPIG_EINVAL;
    auto kern = v7::estimate_kernel<G>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MAGICPIG_ECUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nsm);
    cfg.blockDim = dim3(v7::NW * 32);
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

template <int G>
static int launch_merge_g(const EstArgs& a, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.B * a.Hq));
    cfg.blockDim = dim3(HD * v7::MS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, v7::merge_kernel<G>, a);
    count_launch(1);
    return e == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

int launch_est_merge(const EstArgs& a, cudaStream_t st) {
    switch ((int)(a.Hq / a.Hkv)) {
        case 1: return launch_merge_g<1>(a, st);
        case 2: return launch_merge_g<2>(a, st);
        case 4: return launch_merge_g<4>(a, st);
        case 8: return launch_merge_g<8>(a, st);
    }
    return MAGICPIG_EINVAL;
}

int launch_estimate(const EstArgs& a, int nsm, int max_smem, cudaStream_t st) {
    if (a.B * a.Hkv * (a.nchunks + 1) > EST_MAX_PIECES || a.n_local >= (1 << 24)) return MAGICPIG_EINVAL;
    switch ((int)(a.Hq / a.Hkv)) {
        case 1: return launch_estimate_g<1>(a, nsm, max_smem, st);
        case 2: return launch_estimate_g<2>(a, nsm, max_smem, st);
        case 4: return launch_estimate_g<4>(a, nsm, max_smem, st);
        case 8: return launch_estimate_g<8>(a, nsm, max_smem, st);
    }
    return MAGICPIG_EINVAL;
}

}  // namespace mp
