// estimate9.cu -- kernel 9: the balanced estimator of kernel 7 (estimate.cu: same piece lists, same contiguous
// per-warp ranges, same records for merge_kernel) with the K/V gather moved off the async/bulk-copy path and
// onto plain 16-byte global loads straight into the mma.sync fragments.
//
// Why: the round-2 micro-benchmarks of random-row gathers on B200 put 256-B bulk copies at
// ~1.0 TB/s and plain ld.global gathers from many warps at 5.5-6 TB/s; kernel 7 (bulk copies, 8 warps/SM)
// reached 2.17 TB/s at C3.  Here no K/V byte touches shared memory:
//
//   logits / hashed dots  D[row][head] = sum_k A[row][k] B[k][head] (m16n8k16).  The sum over k is
//       order-free, so the k axis is permuted: lane (g, t) holds A[row g][*] and A[row g+8][*] as the 64
//       contiguous bytes {64 j + 16 t .. +16 : j = 0..3} of each row (4 LDG.128 per row; one warp
//       instruction reads 64 contiguous bytes of 8 rows), k-step ks = 2 j + h takes components 2h, 2h+1 of
//       the j-th load; q (B operand) and the centering vector c are read with the same permutation.
//   P.V                    a[d][n] += sum_rows V^T[d][row] W[row][n] (m16n8k16, A = V^T).  Lane (g, t)
//       needs V^T at rows {2t, 2t+1, 2t+8, 2t+9}; the output dimension d is permuted so that lane g's
//       dimensions are {8g .. 8g+7} u {64+8g .. 64+8g+7}: two LDG.128 per row (one warp instruction reads
//       4 rows x 128 contiguous bytes), pairs (row r, row r+1) built with one PRMT per A register.
//       Accumulator (dt, i) <-> d = 8g + dt (rows g) and 64 + 8g + dt (rows g+8).
//
// Per warp the slab s+1 loads are issued right after slab s consumed the registers they overwrite (K after
// the logits, V after P.V), so each load has the rest of a slab's compute to land, and 12 warps per SM
// (1 CTA, <= 168 registers) interleave.  Everything else (prefix over the pieces, ln u for the (row, head)
// items in S only, online softmax, hi/lo bf16 weights, unit records) follows kernel 7 (see estimate.cu and
// PAPER.md:107-116, Eq. P:86-91).
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.cuh"
#include "pieces.cuh"

namespace mp {
namespace v9 {

using v7::StaticRanges;
using v7::static_ranges;
using v7::warp_incl_scan;

// estimator warps per CTA: G = 8 carries two PV n-tiles (64 accumulator registers) -> 8 warps, <= 255 regs
template <int G>
__host__ __device__ constexpr int nwarps() { return G == 8 ? 8 : EST9_WARPS; }
constexpr int SR = 16;          // rows per slab (mma M)
constexpr int SPW = 2;          // minimum slabs per active warp
constexpr int PREC = PREC5;
constexpr float INV_SQRT_D = 0.08838834764831845f;

struct __align__(16) WBuf {
    uint2 qf[8][32];       // q_g as the logits' B fragments: [k-step][lane] (unit's G heads, permuted k)
    float c[HD];           // -c of the warp's current unit
    float items[SR * 8];   // compacted (row, head) items: cos in, ln u out
    uint16_t wt[16 * SR];  // PV B operand: [column n][row] bf16 (hi | lo weights)
};

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// bf16 pair (lo = element d, hi = element d+1) -> bf16(fl32(k - c)) pair: two mixed-precision adds
// (add.rn.f32.bf16: the bf16 operand widened exactly, one fp32 rounding) and one cvt.rn.bf16x2
__device__ __forceinline__ uint32_t xbar_pair(uint32_t kw, float2 nc) {
    float x0, x1;
    uint32_t r;
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
        "add.rn.f32.bf16 %0, l, %3;\n\tadd.rn.f32.bf16 %1, h, %4;\n\t}"
        : "=f"(x0), "=f"(x1)
        : "r"(kw), "f"(nc.x), "f"(nc.y));
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x1), "f"(x0));
    return r;
}
// one-use 16-B gather load: no L1 allocation, the rest of the 256-B row prefetched into L2
__device__ __forceinline__ uint4 ldg_row16(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t comp(const uint4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}
__device__ __forceinline__ uint32_t prmt(uint32_t x, uint32_t y, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(y), "r"(sel));
    return r;
}

__device__ __forceinline__ void prefetch_l2_row(const void* p) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], 256;" ::"l"(p) : "memory");
}
// the same 256-B row by two plain L2 prefetches (LSU path, no TMA issue)
__device__ __forceinline__ void prefetch_l2_row2(const uint16_t* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p) : "memory");
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 64) : "memory");
}
// ln u(p) from the CTA's shared-memory copy of the table (see log_sampling_prob_lut)
__device__ __forceinline__ float lnu_smem(const float* tab, float p, int K, int L, int minc) {
    if (p >= 1.0f) return 0.0f;
    if (!(p >= LUT_P0)) return log_sampling_prob(p, K, L, minc);
    const float x = (p - LUT_P0) * LUT_INV_H;
    const int i = min((int)x, LUT_N - 1);
    const float f = x - (float)i;
    const float t0 = tab[i], t1 = tab[i + 1];
    return fmaf(f, t1 - t0, t0);
}

// owner warp of entry e when E entries are split into W contiguous ranges [k E / W, (k+1) E / W)
__device__ __forceinline__ int64_t owner_of(int64_t e, int64_t E, int64_t W) { return ((e + 1) * W - 1) / E; }

// DBG: the weighted-set debug export (a.weighted) -- a separate instantiation, so the timed kernel carries no
// per-row key registers for it
template <int G, bool DBG>
__global__ void __launch_bounds__(nwarps<G>() * 32, 1) estimate9_kernel(EstArgs a) {
    constexpr int NW = nwarps<G>();
    constexpr int NT = (2 * G + 7) / 8;  // PV n-tiles: columns [hi heads | lo heads | pad]
    extern __shared__ __align__(128) uint8_t dsm[];
    int* pref = reinterpret_cast<int*>(dsm);
    __shared__ int wsum[32];
    WBuf* wbuf = reinterpret_cast<WBuf*>(dsm + a.off_wbuf);
    float* lut = reinterpret_cast<float*>(dsm + a.off_wbuf + NW * sizeof(WBuf));

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t units = a.B * a.Hkv;
    const int64_t nwb = (a.n_local + 31) >> 5;
    const StaticRanges sr = static_ranges(a);
    const int nT = (int)(sr.len1 + sr.len2);
    const int P = (int)a.nchunks + 1;
    const int NP = (int)units * P;
    WBuf& wb = wbuf[warp];
    for (int e = lane; e < 8 * SR; e += 32) reinterpret_cast<uint32_t*>(wb.wt)[e] = 0u;  // pad columns stay 0
    asm volatile("griddepcontrol.wait;" ::: "memory");  // lists of the select step

    for (int i = tid; i <= LUT_N; i += NW * 32) lut[i] = __ldg(a.lutab + i);
    {   // block exclusive scan of the piece lengths
        // piece lengths: pcnt [units][nchunks] -> pref[u * P + 1 + c]; warp per unit, lane per chunk, four
        // units (eight loads) in flight per lane, no integer division
        const int nch = (int)a.nchunks;
        for (int c0 = 0; c0 < nch; c0 += 64)
            for (int u0 = warp; u0 < (int)units; u0 += NW * 4) {
                int v[4][2];
#pragma unroll
                for (int k = 0; k < 4; k++)
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int u = u0 + k * NW, cc = c0 + lane + 32 * h;
                        v[k][h] = (u < (int)units && cc < nch) ? __ldcg(a.pcnt + (int64_t)u * nch + cc) : 0;
                    }
#pragma unroll
                for (int k = 0; k < 4; k++)
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int u = u0 + k * NW, cc = c0 + lane + 32 * h;
                        if (u < (int)units && cc < nch) pref[u * P + 1 + cc] = v[k][h];
                    }
            }
        for (int u = tid; u < (int)units; u += NW * 32) pref[u * P] = nT;
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
    const int64_t Wt = (int64_t)gridDim.x * NW;
    int64_t Wa = (E + SR * SPW - 1) / (SR * SPW);
    Wa = Wa < 1 ? 1 : (Wa > Wt ? Wt : Wa);
    if (blockIdx.x == 0) {  // record table for the merge kernel
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

    const int g4 = lane >> 2, t4 = lane & 3;
    const int h0 = 2 * t4, h1 = 2 * t4 + 1;  // logit-side heads of this thread (columns of the m16n8 D)
    auto pv_head = [&](int nt, int i) {
        const int n = nt * 8 + 2 * t4 + i;
        return n < G ? n : (n < 2 * G ? n - G : -1);
    };
    auto find_piece = [&](int64_t e) {
        int lo = 0, hi = NP;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pref[mid] <= e) lo = mid;
            else hi = mid;
        }
        return lo;
    };
    // plan of a slab: unit, rows, and (lanes r and r + 16) the raw list entry of row r (key | head bits << 24,
    // or a static key with stat = 1).  Entries are loaded three slabs before their rows are issued and
    // decoded only at issue time, so the entry load is off the row loads' dependency chain.
    struct Plan {
        int u, nr;
        uint32_t ent;
        int stat;
    };
    int ps = find_piece(e_lo);
    int pu = ps / P, pu_end = (pu + 1) * P;  // unit of piece ps and its end piece
    int64_t pcur = e_lo;
    auto plan_next = [&](Plan& PL) {
        PL.nr = 0;
        PL.ent = 0u;
        PL.stat = 0;
        PL.u = 0;
        if (pcur >= e_hi) return;
        while (pref[ps + 1] <= pcur) ps++;
        while (ps >= pu_end) pu++, pu_end += P;
        const int u = pu;
        const int64_t uend = min(e_hi, (int64_t)pref[pu_end]);
        PL.u = u;
        PL.nr = (int)min((int64_t)SR, uend - pcur);
        const int r = lane & 15;
        if (r < PL.nr) {
            const int e = (int)(pcur + r);
            int pi = ps;
            while (pref[pi + 1] <= e) pi++;
            const int j = e - pref[pi], cc = pi - (pu_end - P);
            if (cc == 0) {
                PL.ent = (uint32_t)(j < sr.len1 ? sr.lo1 + j : sr.lo2 + (j - sr.len1));
                PL.stat = 1;
            } else {
                PL.ent = __ldcg(a.ents + ((int64_t)u * a.nchunks + cc - 1) * KCHUNK + j);
            }
        }
        pcur += PL.nr;
    };
    auto plan_key = [&](const Plan& PL) { return (int)(PL.ent & 0xffffffu); };
    auto plan_bits = [&](const Plan& PL) { return PL.stat ? (0x100u | ((1u << G) - 1u)) : PL.ent >> 24; };

    // registers of the slab in flight: K rows g4 (kr[0..3]) and g4 + 8 (kr[4..7]); V rows 2t, 2t+1, 2t+8, 2t+9
    // (vr[2i]: bytes 16 g4 .., vr[2i+1]: bytes 128 + 16 g4 ..)
    uint4 kr[8], vr[8];
    float xn0 = 0.0f, xn1 = 0.0f;  // |xbar| of rows g4, g4 + 8
    uint32_t bt0 = 0u, bt1 = 0u;   // head bits of rows g4, g4 + 8
    int key0 = 0, key1 = 0;        // (debug export) keys of rows g4, g4 + 8
    auto issue_k = [&](const Plan& PL, float& nx0, float& nx1, uint32_t& nb0, uint32_t& nb1, int& nk0, int& nk1) {
        const int key = plan_key(PL);
        const uint32_t bits = plan_bits(PL);
        const int k0 = __shfl_sync(0xffffffffu, key, g4);
        const int k1 = __shfl_sync(0xffffffffu, key, g4 + 8);
        if (DBG) nk0 = k0, nk1 = k1;
        nb0 = __shfl_sync(0xffffffffu, bits, g4);
        nb1 = __shfl_sync(0xffffffffu, bits, g4 + 8);
        const int64_t base = (int64_t)PL.u * a.n_local;
        const bool ok0 = g4 < PL.nr, ok1 = g4 + 8 < PL.nr;
        const uint4* r0 = reinterpret_cast<const uint4*>(a.k + (base + k0) * HD) + t4;
        const uint4* r1 = reinterpret_cast<const uint4*>(a.k + (base + k1) * HD) + t4;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            kr[j] = ok0 ? ldg_row16(r0 + 4 * j) : make_uint4(0u, 0u, 0u, 0u);
            kr[4 + j] = ok1 ? ldg_row16(r1 + 4 * j) : make_uint4(0u, 0u, 0u, 0u);
        }
        nx0 = ok0 ? __ldg(a.key_norm + base + k0) : 0.0f;
        nx1 = ok1 ? __ldg(a.key_norm + base + k1) : 0.0f;
    };
    auto issue_v = [&](const Plan& PL) {
        const int64_t base = (int64_t)PL.u * a.n_local;
        const int mykey = plan_key(PL);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int r = 2 * t4 + (i & 1) + (i >> 1) * 8;
            const int key = __shfl_sync(0xffffffffu, mykey, r);
            const bool ok = r < PL.nr;
            const uint4* vp = reinterpret_cast<const uint4*>(a.v + (base + key) * HD) + g4;
            vr[2 * i] = ok ? ldg_row16(vp) : make_uint4(0u, 0u, 0u, 0u);
            vr[2 * i + 1] = ok ? ldg_row16(vp + 8) : make_uint4(0u, 0u, 0u, 0u);
        }
    };

    float acc[8][NT][4];
    float m0 = -INFINITY, m1 = -INFINITY, s0 = 0.0f, s1 = 0.0f;
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
        uint2 qv[8];
#pragma unroll
        for (int ks = 0; ks < 8; ks++) {
            // k-step ks = 2 j + h: elements 32 j + 8 t + 4 h .. + 3 (see the header)
            const int d0 = 32 * (ks >> 1) + 8 * t4 + 4 * (ks & 1);
            if (g4 < G) {
                qv[ks] = __ldg(reinterpret_cast<const uint2*>(a.q + (qh0 + g4) * HD + d0));
            } else {
                qv[ks] = make_uint2(0u, 0u);
            }
            const uint32_t qw[2] = {qv[ks].x, qv[ks].y};
#pragma unroll
            for (int i = 0; i < 2; i++) {
                const float lo = __uint_as_float(qw[i] << 16), hi = __uint_as_float(qw[i] & 0xffff0000u);
                sq = fmaf(lo, lo, fmaf(hi, hi, sq));
            }
        }
        __syncwarp();  // the previous unit's readers of wb.c / wb.qf are done
#pragma unroll
        for (int ks = 0; ks < 8; ks++) wb.qf[ks][lane] = qv[ks];
        const float4 cv = __ldg(reinterpret_cast<const float4*>(a.center + u * HD) + lane);
        *reinterpret_cast<float4*>(&wb.c[4 * lane]) = make_float4(-cv.x, -cv.y, -cv.z, -cv.w);
        __syncwarp();
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
        const float qn = sqrtf(sq);
        if constexpr (G <= 4) {  // compact items: heads 2 (t4 & 1), 2 (t4 & 1) + 1
            qn0 = __shfl_sync(0xffffffffu, qn, 4 * (2 * (t4 & 1)));
            qn1 = __shfl_sync(0xffffffffu, qn, 4 * (2 * (t4 & 1) + 1));
        } else {
            qn0 = __shfl_sync(0xffffffffu, qn, 4 * h0);
            qn1 = __shfl_sync(0xffffffffu, qn, 4 * (h1 & 7));
        }
    };
    // leave unit u: record (m, s, a) of this warp -> parts[u + kw]; accumulator (dt, i) of rows g4 is
    // dimension 8 g4 + dt, of rows g4 + 8 dimension 64 + 8 g4 + dt
    auto flush = [&](int64_t u) {
        float* rec = a.parts + (size_t)(u + kw) * G * PREC;
#pragma unroll
        for (int i = 0; i < 2; i++) {
            float va[8], vb[8];
#pragma unroll
            for (int dt = 0; dt < 8; dt++) {
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
                va[dt] = hiA + loA;
                vb[dt] = hiB + loB;
            }
            const int h = 2 * t4 + i;
            const bool own = (G == 1) ? (t4 == 0 && i == 0) : (h < G);
            if (own) {
                float4* pa = reinterpret_cast<float4*>(rec + h * PREC + 4 + 8 * g4);
                float4* pb = reinterpret_cast<float4*>(rec + h * PREC + 4 + 64 + 8 * g4);
                __stcg(pa, make_float4(va[0], va[1], va[2], va[3]));
                __stcg(pa + 1, make_float4(va[4], va[5], va[6], va[7]));
                __stcg(pb, make_float4(vb[0], vb[1], vb[2], vb[3]));
                __stcg(pb + 1, make_float4(vb[4], vb[5], vb[6], vb[7]));
            }
        }
        if (g4 == 0) {
            if (h0 < G) __stcg(reinterpret_cast<float2*>(rec + h0 * PREC), make_float2(m0, s0));
            if (h1 < G) __stcg(reinterpret_cast<float2*>(rec + h1 * PREC), make_float2(m1, s1));
        }
    };

#ifndef MP_E9_PF
#define MP_E9_PF 0
#endif
    // MP_E9_PF 2: the rows of the plan's slab into L2 by plain prefetches (lane r < 16: K row r, lane
    // 16 + r: V row r), for the two slabs after the first at the start (a warp with few slabs would otherwise
    // wait for each slab's rows in turn) and (3) also for slab s + 3 in every iteration
    auto prefetch_plan = [&](const Plan& PL) {
        const int r = lane & 15;
        const int key = __shfl_sync(0xffffffffu, plan_key(PL), r);
        if (r < PL.nr) prefetch_l2_row2((lane < 16 ? a.k : a.v) + ((int64_t)PL.u * a.n_local + key) * HD);
    };
    Plan P0, P1, P2;
    plan_next(P0);
    plan_next(P1);
    plan_next(P2);
    if (MP_E9_PF >= 2) {
        prefetch_plan(P1);
        prefetch_plan(P2);
    }
    int cu = P0.u, cnr = P0.nr;
    issue_k(P0, xn0, xn1, bt0, bt1, key0, key1);
    issue_v(P0);
    P0 = P1;
    P1 = P2;
    plan_next(P2);
    int64_t cur_u = -1;
    reset_state();
#pragma unroll 1
    while (cnr > 0) {
        if (cu != cur_u) {
            if (cur_u >= 0) {
                flush(cur_u);
                reset_state();
            }
            cur_u = cu;
            load_unit(cu);
        }
        // (1) logits q.k and hashed dots qbar.xbar from the K registers
        float dl[4] = {0.0f, 0.0f, 0.0f, 0.0f}, dx[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int ks = 0; ks < 8; ks++) {
            const int j = ks >> 1, h = ks & 1;
            uint32_t af[4];
            af[0] = comp(kr[j], 2 * h);
            af[1] = comp(kr[4 + j], 2 * h);
            af[2] = comp(kr[j], 2 * h + 1);
            af[3] = comp(kr[4 + j], 2 * h + 1);
            const uint2 qb = wb.qf[ks][lane];
            mma16816(dl, af, qb.x, qb.y);
            const float4 cc = *reinterpret_cast<const float4*>(&wb.c[32 * j + 8 * t4 + 4 * h]);
            const float2 ca = make_float2(cc.x, cc.y), cb = make_float2(cc.z, cc.w);
            uint32_t xf[4];
            xf[0] = xbar_pair(af[0], ca);
            xf[1] = xbar_pair(af[1], ca);
            xf[2] = xbar_pair(af[2], cb);
            xf[3] = xbar_pair(af[3], cb);
            mma16816(dx, xf, qb.x, qb.y);
        }
        // the next slab's K rows (and norms, head bits) into the registers just consumed
        float nxn0 = 0.0f, nxn1 = 0.0f;
        uint32_t nbt0 = 0u, nbt1 = 0u;
        int nk0 = 0, nk1 = 0;
        const int nu = P0.u, nnr = P0.nr;
        issue_k(P0, nxn0, nxn1, nbt0, nbt1, nk0, nk1);  // nr = 0: every load predicated off

        // (2) items (row, head).  G = 8: every lane's four mma outputs, rows g4 (dl[0], dl[1]) and g4 + 8
        // (dl[2], dl[3]), heads h0, h1.  G <= 4 (compact): columns 4..7 of the logits tile are empty, so lane
        // t4 >= 2 takes over row g4 + 8 of lane t4 - 2 (xor 2) and every lane has two items, one row, heads
        // 2 (t4 & 1) and 2 (t4 & 1) + 1; the per-head reductions then run over xor 2, 4, 8, 16.
        constexpr bool CMP = G <= 4;
        constexpr int NI = CMP ? 2 : 4;
        const bool hirow = CMP && t4 >= 2;
        float dlv[NI], dxv[NI];
        uint32_t bt[NI];
        int hh[NI], rows[NI];
        float qnv[NI], xnv[NI];
        if constexpr (CMP) {
            const float sl2 = __shfl_xor_sync(0xffffffffu, dl[2], 2), sl3 = __shfl_xor_sync(0xffffffffu, dl[3], 2);
            const float sx2 = __shfl_xor_sync(0xffffffffu, dx[2], 2), sx3 = __shfl_xor_sync(0xffffffffu, dx[3], 2);
            dlv[0] = hirow ? sl2 : dl[0];
            dlv[1] = hirow ? sl3 : dl[1];
            dxv[0] = hirow ? sx2 : dx[0];
            dxv[1] = hirow ? sx3 : dx[1];
#pragma unroll
            for (int i = 0; i < 2; i++) {
                bt[i] = hirow ? bt1 : bt0;
                hh[i] = 2 * (t4 & 1) + i;
                rows[i] = hirow ? g4 + 8 : g4;
                xnv[i] = hirow ? xn1 : xn0;
            }
            qnv[0] = qn0, qnv[1] = qn1;
        } else {
#pragma unroll
            for (int i = 0; i < 4; i++) {
                dlv[i] = dl[i], dxv[i] = dx[i];
                bt[i] = (i >> 1) ? bt1 : bt0;
                hh[i] = (i & 1) ? h1 : h0;
                rows[i] = (i >> 1) ? g4 + 8 : g4;
                xnv[i] = (i >> 1) ? xn1 : xn0;
                qnv[i] = (i & 1) ? qn1 : qn0;
            }
        }
        bool need[NI];
        float cs[NI];
#pragma unroll
        for (int i = 0; i < NI; i++) {
            need[i] = hh[i] < G && !(bt[i] & 0x100u) && ((bt[i] >> hh[i]) & 1u);
            const float den = qnv[i] * xnv[i];
            const float c = den > 0.0f ? __fdividef(dxv[i], den) : 0.0f;
            cs[i] = fminf(1.0f, fmaxf(-1.0f, c));
        }
        float lu[NI];
        {
            int base = 0, pos[NI];
            const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
            for (int i = 0; i < NI; i++) {
                lu[i] = 0.0f;
                const uint32_t bal = __ballot_sync(0xffffffffu, need[i]);
                pos[i] = base + __popc(bal & lt);
                base += __popc(bal);
                if (need[i]) wb.items[pos[i]] = cs[i];
            }
            __syncwarp();
            for (int e = lane; e < base; e += 32) {
                const float p = 1.0f - acosf(wb.items[e]) * 0.3183098861837907f;
#ifndef MP_E9_SLUT
#define MP_E9_SLUT 1
#endif
                wb.items[e] = MP_E9_SLUT ? lnu_smem(lut, p, a.K, a.L, a.minc)
                                         : log_sampling_prob_lut(a.lutab, p, a.K, a.L, a.minc);
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < NI; i++)
                if (need[i]) lu[i] = wb.items[pos[i]];
        }
        float z[NI];
#pragma unroll
        for (int i = 0; i < NI; i++) {
            const float l = dlv[i] * INV_SQRT_D;
            z[i] = (hh[i] < G && (bt[i] & 0x100u)) ? l : (need[i] ? l - lu[i] : -INFINITY);
        }
        if (DBG) {
            const int64_t b = cur_u / a.Hkv, hkv = cur_u % a.Hkv, qh0 = b * a.Hq + hkv * G;
#pragma unroll
            for (int i = 0; i < NI; i++) {
                if (z[i] != -INFINITY && rows[i] < cnr) {
                    const int key = rows[i] >= 8 ? key1 : key0;
                    atomicOr(a.weighted + (qh0 + hh[i]) * nwb + (key >> 5), 1u << (key & 31));
                }
            }
        }
        // (3) online softmax per head (rows of head h are spread over the lanes with the same t4 (G = 8) or
        // t4 & 1 (compact))
        constexpr int MLO = CMP ? 2 : 4;
        float mx0 = CMP ? z[0] : fmaxf(z[0], z[NI > 2 ? 2 : 0]);
        float mx1 = CMP ? z[1] : fmaxf(z[1], z[NI > 2 ? 3 : 1]);
#pragma unroll
        for (int m = MLO; m <= 16; m <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, m));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, m));
        }
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const bool moved = __any_sync(0xffffffffu, mn0 != m0 || mn1 != m1);
        const float al0 = m0 == -INFINITY ? 0.0f : __expf(m0 - mn0);
        const float al1 = m1 == -INFINITY ? 0.0f : __expf(m1 - mn1);
        __nv_bfloat16 whi[NI], wlo[NI];
        float wsum0 = 0.0f, wsum1 = 0.0f;
#pragma unroll
        for (int i = 0; i < NI; i++) {
            const float mni = (i & 1) ? mn1 : mn0;
            const float w = z[i] == -INFINITY ? 0.0f : __expf(z[i] - mni);
            whi[i] = __float2bfloat16_rn(w);
            wlo[i] = __float2bfloat16_rn(w - __bfloat162float(whi[i]));
            const float we = __bfloat162float(whi[i]) + __bfloat162float(wlo[i]);
            if (i & 1) wsum1 += we;
            else wsum0 += we;
        }
#pragma unroll
        for (int m = MLO; m <= 16; m <<= 1) {
            wsum0 += __shfl_xor_sync(0xffffffffu, wsum0, m);
            wsum1 += __shfl_xor_sync(0xffffffffu, wsum1, m);
        }
        s0 = s0 * al0 + wsum0;
        s1 = s1 * al1 + wsum1;
        m0 = mn0;
        m1 = mn1;
        {
            __nv_bfloat16* wt = reinterpret_cast<__nv_bfloat16*>(wb.wt);
#pragma unroll
            for (int i = 0; i < NI; i++) {
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
        // (5) a[d][n] += V^T[d][rows] W[rows][n]: V^T fragments from the row registers by PRMT
        {
            uint32_t bw[NT][2];
            const uint32_t* wt32 = reinterpret_cast<const uint32_t*>(wb.wt);
#pragma unroll
            for (int nt = 0; nt < NT; nt++) {
                bw[nt][0] = wt32[((nt * 8 + g4) * SR + 2 * t4) >> 1];
                bw[nt][1] = wt32[((nt * 8 + g4) * SR + 2 * t4 + 8) >> 1];
            }
#pragma unroll
            for (int dt = 0; dt < 8; dt++) {
                const int w = dt >> 1;
                const uint32_t sel = (dt & 1) ? 0x7632u : 0x5410u;
                uint32_t af[4];
                af[0] = prmt(comp(vr[0], w), comp(vr[2], w), sel);  // rows 2t, 2t+1; d = 8 g4 + dt
                af[1] = prmt(comp(vr[1], w), comp(vr[3], w), sel);  // rows 2t, 2t+1; d = 64 + 8 g4 + dt
                af[2] = prmt(comp(vr[4], w), comp(vr[6], w), sel);  // rows 2t+8, 2t+9
                af[3] = prmt(comp(vr[5], w), comp(vr[7], w), sel);
#pragma unroll
                for (int nt = 0; nt < NT; nt++) mma16816(acc[dt][nt], af, bw[nt][0], bw[nt][1]);
            }
        }
        __syncwarp();  // weight tile and items free
        issue_v(P0);
        cu = nu;
        cnr = nnr;
        xn0 = nxn0, xn1 = nxn1, bt0 = nbt0, bt1 = nbt1, key0 = nk0, key1 = nk1;
        P0 = P1;
        P1 = P2;
        plan_next(P2);
        if (MP_E9_PF == 1) {   // rows of slab s + 3 into L2 (their registers are loaded two slabs later)
            const int r = lane & 15;
            const int key = __shfl_sync(0xffffffffu, plan_key(P1), r);
            if (r < P1.nr) {
                const int64_t row = (int64_t)P1.u * a.n_local + key;
                prefetch_l2_row((lane < 16 ? a.k : a.v) + row * HD);
            }
        }
        if (MP_E9_PF >= 3) prefetch_plan(P1);
    }
    if (cur_u >= 0) flush(cur_u);
}

}  // namespace v9

static size_t al128e9(size_t x) { return (x + 127) & ~(size_t)127; }

template <int G>
static int launch_estimate9_g(EstArgs a, int nsm, int max_smem, cudaStream_t st) {
    const size_t pieces = (size_t)(a.B * a.Hkv * (a.nchunks + 1));
    a.off_wbuf = (int)al128e9((pieces + 1) * 4);
    const size_t smem = a.off_wbuf + sizeof(v9::WBuf) * v9::nwarps<G>() + (LUT_N + 4) * 4;
    if (smem > (size_t)max_smem) return MAGICPIG_EINVAL;
    auto kern = a.weighted ? v9::estimate9_kernel<G, true> : v9::estimate9_kernel<G, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MAGICPIG_ECUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nsm);
    cfg.blockDim = dim3(v9::nwarps<G>() * 32);
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

int launch_estimate9(const EstArgs& a, int nsm, int max_smem, cudaStream_t st) {
    if (a.B * a.Hkv * (a.nchunks + 1) > EST_MAX_PIECES || a.n_local >= (1 << 24)) return MAGICPIG_EINVAL;
    switch ((int)(a.Hq / a.Hkv)) {
        case 1: return launch_estimate9_g<1>(a, nsm, max_smem, st);
        case 2: return launch_estimate9_g<2>(a, nsm, max_smem, st);
        case 4: return launch_estimate9_g<4>(a, nsm, max_smem, st);
        case 8: return launch_estimate9_g<8>(a, nsm, max_smem, st);
    }
    return MAGICPIG_EINVAL;
}

}  // namespace mp
