// attend.cu -- the estimator half of a MagicPIG decode step (Algorithm 1,
// PAPER.md:109-116): for every (sequence, query head) the sampled set S_g
// (given as per-head bitmaps by the Query step: the dense code scan in
// scan6.cu or the bucketed hash tables in buckets.cu) plus the static set T
// is gathered from the KV cache and reduced with the
// self-normalised importance-sampling estimator
//     o_g = sum_{i in S_g u T} e^{z_i} v_i / sum e^{z_i},
//     z_i = q_g.k_i/sqrt(d) - ln u_i   (u_i = 1 on T)
// where u_i is the closed-form sampling probability (Eq. P:86-91) at the angle
// between the hashed vectors (reading R5), p_i = 1 - theta_i/pi.
//
// One persistent CTA per SM walks a contiguous range of tiles (a tile is the
// static piece or one 1024-key chunk of a (sequence, kv head) unit, as in
// decode5.cu), so the CTAs touching a unit are contiguous.
//
//   producer warp   per tile: the G head bitmaps (cp.async, PRE tiles ahead),
//                   S_g = bitmap & D, union over heads, ascending compaction
//                   into a shared-memory descriptor (<= 1024 entries of one
//                   unit: key index + head bits; static keys carry bit 8)
//                   in a 4096-entry ring, published as soon as it holds >= 128
//                   entries (32 descriptors in flight, released in order).
//   8 consumer      every warp owns every 8th 16-row "slab" of the CTA's
//   warps           descriptor stream and works on it alone: K and V rows by
//                   one 256-B bulk copy each (cp.async.bulk, completion on a
//                   per-stage mbarrier; |xbar_i| by cp.async; 2 slabs in flight
//                   per warp; 272-B row pitch), logits q.k and hashed dots
//                   qbar.xbar on tensor cores (mma.sync bf16, xbar =
//                   bf16(fl32(k - c)) formed in the A fragments), ln u only for
//                   the (row, head) items in S (compacted over the warp),
//                   online softmax, and a[g][d] += w v on tensor cores with the
//                   weights split into bf16 hi + lo parts (w = hi + lo to
//                   2^-17 relative), so the estimate is fp32-accurate.
//   unit end        the 8 warp states are combined in shared memory (fixed
//                   order), the CTA's record (m, s, |S_g|, a) goes to
//                   parts[u + cta]; the last CTA of the unit (acq_rel counter)
//                   merges the unit's records in fixed order (log-sum-exp,
//                   "recursive attention") and writes out / partial /
//                   s_count.  Counters self-clean (CUDA-graph replayable).
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.cuh"

namespace mp {
namespace v6 {

constexpr int NC = 8;                      // consumer warps
constexpr int THREADS = (NC + 1) * 32;     // + 1 producer warp
constexpr int SR = 16;                     // rows per slab (mma M)
constexpr int DCAP = 1024;                 // entries per descriptor (max)
constexpr int DMIN = 128;                  // a descriptor is published once it holds >= DMIN entries
constexpr int ERING = 4096;                // entry ring (power of two)
constexpr int NDESC = 32;                  // descriptor (header) ring
constexpr int NST = 2;                     // row stages per consumer warp
constexpr int PRE = 4;                     // bitmap tiles prefetched by the producer
constexpr int QEV = 16;                    // per-warp event queue
constexpr int PREC = PREC5;                // record per head: m, s, |S_g|, 0, a[128]
constexpr float INV_SQRT_D = 0.08838834764831845f;
constexpr int MB = 16;                     // unit merge: records per load round

// a descriptor = n consecutive entries of the entry ring starting at e0 (mod ERING), all of one unit
struct Desc {
    long long e0;          // first entry (monotone position; ring index = e0 & (ERING - 1))
    int n, unit, slab0, nslab, unit_end;
    int cnt[8];            // sum over the descriptor of |S_g|
};

constexpr int RP = 272;                    // shared-memory row pitch (256 B + 16: ldmatrix conflict-free)

struct __align__(128) WarpBuf {
    uint8_t k[NST][SR * RP];    // K rows (one 256-B bulk copy each)
    uint8_t v[NST][SR * RP];    // V rows
    float xn[NST][SR];          // |xbar_i|
    uint64_t bar[NST];          // stage barriers: bulk-copy bytes + the lanes' cp.async (norms)
    uint16_t wt[16 * SR];       // PV B operand: [column n][row] bf16 (hi | lo weights)
    float c[HD];                // centering vector of the warp's current unit
    float items[SR * 8];        // compacted (row, head) items: cos in, ln u out
};

struct Shared {
    int keys[ERING];        // entry ring: local key index
    uint16_t bits[ERING];   //             bit g: key in S_g; 0x100: static (u = 1)
    Desc desc[NDESC];
    uint32_t bmp[PRE][8][32];
    uint64_t full[NDESC], empty[NDESC];
    float ucnt[8];
    int flag;
};

__device__ __forceinline__ void bar_named(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// 16-B / 4-B async copies with zero fill (src_size 0 -> zeros)
__device__ __forceinline__ void cp16z(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp4z(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_mbar_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
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
// bf16 pair (lo = element c, hi = element c+1) -> bf16(fl32(k - c)) pair (cvt.rn.bf16x2)
__device__ __forceinline__ uint32_t xbar_pair(uint32_t kw, float c0, float c1) {
    const __nv_bfloat162 xb = __floats2bfloat162_rn(__fsub_rn(__uint_as_float(kw << 16), c0),
                                                    __fsub_rn(__uint_as_float(kw & 0xffff0000u), c1));
    return *reinterpret_cast<const uint32_t*>(&xb);
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
__device__ __forceinline__ int64_t owner_of(int64_t t, int64_t T, int64_t P) { return ((t + 1) * P - 1) / T; }

struct StaticRanges {
    int64_t lo1, len1, lo2, len2;
};
__device__ __forceinline__ StaticRanges static_ranges(const AttendArgs& a) {
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

template <int G>
__global__ void __launch_bounds__(THREADS, 1) attend_kernel(AttendArgs a) {
    constexpr int NT = (2 * G + 7) / 8;  // PV n-tiles: columns [hi heads | lo heads | pad]
    extern __shared__ __align__(128) uint8_t dsm[];
    Shared& sh = *reinterpret_cast<Shared*>(dsm);
    WarpBuf* wbuf = reinterpret_cast<WarpBuf*>(dsm + a.off_wbuf);
    float* comb = reinterpret_cast<float*>(dsm + a.off_comb);  // [NC][G][132]: m, s, a[128] (+2 pad)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t T = a.tiles, P = gridDim.x, tpu = a.nstatic + a.nchunks;
    const int64_t t0 = (int64_t)blockIdx.x * T / P, t1 = ((int64_t)blockIdx.x + 1) * T / P;
    const int64_t nwb = (a.n_local + 31) >> 5;

    if (tid == 0) {
        for (int i = 0; i < NDESC; i++) {
            mbar_init(&sh.full[i], 1);
            mbar_init(&sh.empty[i], NC);
        }
        fence_mbar_init();
    }
    if (tid < NC * NST) mbar_init(&wbuf[tid / NST].bar[tid % NST], 33);  // 1 expect_tx + 32 noinc arrivals
    if (tid < 8) sh.ucnt[tid] = 0.0f;
    // zero the warp buffers: rows a slab does not load must hold finite values (0 * stale = 0), and the
    // pad columns of the PV weight tiles stay 0
    for (int e = tid; e < NC * (int)offsetof(WarpBuf, bar) / 16; e += THREADS) {
        const int w = e / ((int)offsetof(WarpBuf, bar) / 16), o = e % ((int)offsetof(WarpBuf, bar) / 16);
        reinterpret_cast<uint4*>(&wbuf[w])[o] = make_uint4(0u, 0u, 0u, 0u);
    }
    for (int e = tid; e < NC * 16 * SR / 2; e += THREADS)
        reinterpret_cast<uint32_t*>(wbuf[e / (8 * SR)].wt)[e % (8 * SR)] = 0u;
    fence_proxy_async();
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // S bitmaps of the Query kernel

    if (warp == NC) {
        // ============================================================ producer
        const StaticRanges sr = static_ranges(a);
        int64_t tp = t0;  // next tile to prefetch
        auto prefetch = [&]() {
            const int slot = (int)((tp - t0) % PRE);
            if (tp < t1) {
                const int64_t u = tp / tpu, r = tp % tpu;
                if (r >= a.nstatic) {
                    const int64_t chunk = r - a.nstatic, b = u / a.Hkv, hkv = u % a.Hkv;
                    const int64_t qh0 = b * a.Hq + hkv * G, wi = chunk * 32 + lane;
                    const bool ok = wi < nwb;
#pragma unroll
                    for (int g = 0; g < G; g++)
                        cp4z(&sh.bmp[slot][g][lane], a.sbits + (ok ? (qh0 + g) * nwb + wi : 0), ok);
                }
            }
            cp_commit();
            tp++;
        };
#pragma unroll 1
        for (int i = 0; i < PRE - 1; i++) prefetch();

        int di = 0, dn = 0, slab_base = 0;
        int64_t ewr = 0, e_free = ERING;  // entry write position; entries below e_free may be written
        int hrel = 0;                     // descriptors < hrel are released by all consumers
        int cntg[G];
#pragma unroll
        for (int g = 0; g < G; g++) cntg[g] = 0;
        int64_t cur_u = t0 / tpu;
        // wait for the oldest outstanding descriptor's release (consumers release in order)
        auto release_one = [&]() {
            mbar_wait(&sh.empty[hrel % NDESC], (uint32_t)((hrel / NDESC) & 1));
            const Desc& R = sh.desc[hrel % NDESC];
            e_free = (int64_t)R.e0 + R.n + ERING;
            hrel++;
        };
        auto ensure = [&](int cnt) {  // room for cnt more entries of the open descriptor
            while (ewr + cnt > e_free) {
                if (hrel >= di) break;  // cannot happen: an open descriptor holds <= DCAP < ERING entries
                release_one();
            }
        };
        auto close_desc = [&](int unit_end) {
            int c8[G];
#pragma unroll
            for (int g = 0; g < G; g++) {
                int c = cntg[g];
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
                c8[g] = c;
                cntg[g] = 0;
            }
            if (lane == 0) {
                Desc* D = &sh.desc[di % NDESC];
                D->e0 = (long long)(ewr - dn);
                D->n = dn;
                D->unit = (int)cur_u;
                D->slab0 = slab_base;
                D->nslab = (dn + SR - 1) / SR;
                D->unit_end = unit_end;
#pragma unroll
                for (int g = 0; g < 8; g++) D->cnt[g] = g < G ? c8[g] : 0;
            }
            slab_base += (dn + SR - 1) / SR;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh.full[di % NDESC]);
            di++;
            while (hrel <= di - NDESC) release_one();  // header slot of descriptor di free
            dn = 0;
        };
#pragma unroll 1
        for (int64_t t = t0; t < t1; t++) {
            prefetch();
            const int64_t u = t / tpu, r = t % tpu;
            if (u != cur_u) {
                close_desc(1);
                cur_u = u;
            }
            const int64_t b = u / a.Hkv, hkv = u % a.Hkv;
            const int64_t qh0 = b * a.Hq + hkv * G;
            if (r < a.nstatic) {
                const int64_t p0 = r * (int64_t)KCHUNK, nT = sr.len1 + sr.len2;
                const int cnt = nT > p0 ? (int)min((int64_t)KCHUNK, nT - p0) : 0;
                if (dn + cnt > DCAP) close_desc(0);
                ensure(cnt);
                for (int j = lane; j < cnt; j += 32) {
                    const int64_t tt = p0 + j;
                    const int e = (int)((ewr + j) & (ERING - 1));
                    sh.keys[e] = (int)(tt < sr.len1 ? sr.lo1 + tt : sr.lo2 + (tt - sr.len1));
                    sh.bits[e] = 0x100u;
                }
                dn += cnt;
                ewr += cnt;
                cp_wait<PRE - 1>();  // keep the group accounting aligned with the chunk path
            } else {
                const int64_t chunk = r - a.nstatic;
                const int slot = (int)((t - t0) % PRE);
                cp_wait<PRE - 1>();
                __syncwarp();
                const int64_t base = chunk * KCHUNK + lane * 32;
                const uint32_t dmask =
                    range_mask(base, 0, a.n_local) &
                    ~(range_mask(base, -a.seq_offset, (int64_t)a.sink - a.seq_offset) |
                      range_mask(base, a.n_global - a.local - a.seq_offset, a.n_global - a.seq_offset));
                uint32_t sg[G], un = 0u;
#pragma unroll
                for (int g = 0; g < G; g++) {
                    sg[g] = sh.bmp[slot][g][lane] & dmask;
                    un |= sg[g];
                    cntg[g] += __popc(sg[g]);
                }
                if (a.s_mask && chunk * 32 + lane < nwb) {
#pragma unroll
                    for (int g = 0; g < G; g++) a.s_mask[(qh0 + g) * nwb + chunk * 32 + lane] = sg[g];
                }
                const int c = __popc(un);
                int incl = c;
#pragma unroll
                for (int m = 1; m < 32; m <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, m);
                    if (lane >= m) incl += v;
                }
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                if (dn + total > DCAP) close_desc(0);
                ensure(total);
                int64_t pos = ewr + incl - c;
                uint32_t rem = un;
                while (rem) {
                    const int bit = __ffs(rem) - 1;
                    rem &= rem - 1u;
                    uint32_t hb = 0;
#pragma unroll
                    for (int g = 0; g < G; g++) hb |= ((sg[g] >> bit) & 1u) << g;
                    sh.keys[pos & (ERING - 1)] = (int)(base + bit);
                    sh.bits[pos & (ERING - 1)] = (uint16_t)hb;
                    pos++;
                }
                dn += total;
                ewr += total;
            }
            __syncwarp();
            // publish early so the consumers start (and stay busy) while the rest of the unit is compacted
            if (dn >= DMIN && t + 1 < t1 && (t + 1) / tpu == cur_u) close_desc(0);
        }
        close_desc(1);
        cp_wait<0>();
        return;
    }

    // ================================================================ consumers
    WarpBuf& wb = wbuf[warp];
    const int g4 = lane >> 2, t4 = lane & 3;
    const int h0 = 2 * t4, h1 = 2 * t4 + 1;  // logit-side heads of this thread (columns of the m16n8 D)
    // PV-side columns n = nt*8 + 2*t4 + i: head (hi for n < G, lo for G <= n < 2G, -1 = pad); the softmax
    // state of head h lives in the lanes with t4 = h / 2
    auto pv_head = [&](int nt, int i) {
        const int n = nt * 8 + 2 * t4 + i;
        return n < G ? n : (n < 2 * G ? n - G : -1);
    };
    float acc[8][NT][4];
#pragma unroll
    for (int dt = 0; dt < 8; dt++)
#pragma unroll
        for (int nt = 0; nt < NT; nt++) acc[dt][nt][0] = acc[dt][nt][1] = acc[dt][nt][2] = acc[dt][nt][3] = 0.0f;
    float m0 = -INFINITY, m1 = -INFINITY, s0 = 0.0f, s1 = 0.0f;
    uint32_t qf[8][2];
    float qn0 = 0.0f, qn1 = 0.0f;
    int64_t cur_u = -1;

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
        *reinterpret_cast<float4*>(&wb.c[4 * lane]) = __ldg(reinterpret_cast<const float4*>(a.center + u * HD) + lane);
        __syncwarp();
        // |q_g|^2: lanes 4g .. 4g+3 hold head g's 128 elements
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
        const float qn = sqrtf(sq);
        qn0 = __shfl_sync(0xffffffffu, qn, 4 * h0);
        qn1 = __shfl_sync(0xffffffffu, qn, 4 * (h1 & 7));
    };

    // ---- event queue: the issue cursor walks the descriptors in order; per descriptor it queues this warp's
    // slabs (after issuing their row copies) and an end marker.  The compute side pops them in order.
    int q_d[QEV], q_j[QEV];  // j >= 0: slab; j < 0: end of descriptor q_d
    int qh = 0, qt = 0;      // head / tail (monotone)
    int issued = 0, computed = 0;  // slabs
    int idi = 0;             // descriptor the issue cursor is in
    int ij = warp;           // next slab index (CTA stream) of this warp
    bool idesc_ready = false, done_issue = false;
    uint32_t* const items = reinterpret_cast<uint32_t*>(wb.items);
    (void)items;

    auto issue_slab = [&](const Desc& D, int j) {
        const int st = issued % NST;
        const int e0 = (j - D.slab0) * SR;
        const int nr = min(SR, D.n - e0);
        const int64_t ubase = (int64_t)D.unit * a.n_local;
        const int r = lane & 15;
        uint64_t* bar = &wb.bar[st];
        fence_proxy_async();  // this stage's earlier ldmatrix reads before the async-proxy refill
        if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)nr * 512u);
        __syncwarp();
        if (r < nr) {
            const int64_t key = sh.keys[(int)(D.e0 + e0 + r) & (ERING - 1)];
            if (lane < 16) bulk_g2s(wb.k[st] + r * RP, a.k + (ubase + key) * HD, 256, bar);
            else bulk_g2s(wb.v[st] + r * RP, a.v + (ubase + key) * HD, 256, bar);
            if (lane < 16) cp4z(&wb.xn[st][r], a.key_norm + ubase + key, true);
        }
        cp_mbar_arrive_noinc(bar);
        issued++;
    };

    // advance the issue cursor: issue while stage buffers are free and descriptors are published
    auto pump = [&](bool block) {
        while (!done_issue && issued - computed < NST && qt - qh < QEV - 1) {
            if (!idesc_ready) {
                const uint32_t par = (uint32_t)((idi / NDESC) & 1);
                if (!mbar_test(&sh.full[idi % NDESC], par)) {
                    if (!(block && qt == qh)) return;
                    mbar_wait(&sh.full[idi % NDESC], par);
                }
                idesc_ready = true;
            }
            const Desc& D = sh.desc[idi % NDESC];
            if (ij < D.slab0 + D.nslab) {
                issue_slab(D, ij);
                q_d[qt % QEV] = idi;
                q_j[qt % QEV] = ij;
                qt++;
                ij += NC;
            } else {
                q_d[qt % QEV] = idi;
                q_j[qt % QEV] = -1;
                qt++;
                const bool last = D.unit_end && (D.unit == (int)((t1 - 1) / tpu));
                idi++;
                idesc_ready = false;
                if (last) done_issue = true;
            }
        }
    };

    const int ctid = tid;  // consumer thread id 0 .. NC*32-1
#pragma unroll 1
    while (true) {
        pump(true);
        if (qh == qt) break;
        const int d = q_d[qh % QEV], j = q_j[qh % QEV];
        qh++;
        const Desc& D = sh.desc[d % NDESC];
        if (j < 0) {
            // ---- end of descriptor d
            if (warp == 0 && lane < G) sh.ucnt[lane] += (float)D.cnt[lane];
            const int unit_end = D.unit_end, unit = D.unit;
            __syncwarp();
            if (unit_end) {
                // combine the NC warp states of this unit (fixed order) -> record parts[u + cta]
                const int64_t u = unit;
                float* cw = comb + (size_t)warp * G * 132;
                // pass 1: hi columns (and m, s); pass 2: lo columns added
#pragma unroll
                for (int pass = 0; pass < 2; pass++) {
#pragma unroll
                    for (int nt = 0; nt < NT; nt++)
#pragma unroll
                        for (int i = 0; i < 2; i++) {
                            const int n = nt * 8 + 2 * t4 + i, h = pv_head(nt, i);
                            if (h < 0 || (pass == 0) != (n < G)) continue;
#pragma unroll
                            for (int dt = 0; dt < 8; dt++) {
                                float* p0 = cw + h * 132 + 2 + dt * 16 + g4;
                                if (pass == 0) {
                                    p0[0] = acc[dt][nt][i];
                                    p0[8] = acc[dt][nt][2 + i];
                                } else {
                                    p0[0] += acc[dt][nt][i];
                                    p0[8] += acc[dt][nt][2 + i];
                                }
                            }
                        }
                    if (pass == 0 && g4 == 0) {
                        if (h0 < G) cw[h0 * 132] = m0, cw[h0 * 132 + 1] = s0;
                        if (h1 < G) cw[h1 * 132] = m1, cw[h1 * 132 + 1] = s1;
                    }
                    __syncwarp();
                }
                // this warp's state is in the combine area: reset it for the next unit
#pragma unroll
                for (int dt = 0; dt < 8; dt++)
#pragma unroll
                    for (int nt = 0; nt < NT; nt++)
                        acc[dt][nt][0] = acc[dt][nt][1] = acc[dt][nt][2] = acc[dt][nt][3] = 0.0f;
                m0 = m1 = -INFINITY;
                s0 = s1 = 0.0f;
                cur_u = -1;
                bar_named(1, NC * 32);
                float* rec = a.parts + (size_t)(u + blockIdx.x) * G * PREC;
                for (int e = ctid; e < G * HD; e += NC * 32) {
                    const int h = e / HD, dd = e % HD;
                    float M = -INFINITY;
#pragma unroll
                    for (int w = 0; w < NC; w++) M = fmaxf(M, comb[(w * G + h) * 132]);
                    float A = 0.0f;
#pragma unroll
                    for (int w = 0; w < NC; w++) {
                        const float mw = comb[(w * G + h) * 132];
                        if (mw != -INFINITY) A = fmaf(comb[(w * G + h) * 132 + 2 + dd], __expf(mw - M), A);
                    }
                    rec[h * PREC + 4 + dd] = A;
                }
                if (ctid < G) {
                    const int h = ctid;
                    float M = -INFINITY, S = 0.0f;
#pragma unroll
                    for (int w = 0; w < NC; w++) M = fmaxf(M, comb[(w * G + h) * 132]);
#pragma unroll
                    for (int w = 0; w < NC; w++) {
                        const float mw = comb[(w * G + h) * 132];
                        if (mw != -INFINITY) S = fmaf(comb[(w * G + h) * 132 + 1], __expf(mw - M), S);
                    }
                    *reinterpret_cast<float4*>(rec + h * PREC) = make_float4(M, S, sh.ucnt[h], 0.0f);
                }
                const int64_t tu0 = u * tpu, tu1 = tu0 + tpu - 1;
                const int64_t ilo = owner_of(tu0, T, P), ihi = owner_of(tu1, T, P);
                const int np = (int)(ihi - ilo + 1);
                bar_named(1, NC * 32);
                if (ctid == 0) {
                    uint32_t old;
                    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                                 : "=r"(old)
                                 : "l"(a.unit_ctr + u)
                                 : "memory");
                    sh.flag = old == (uint32_t)(np - 1);
                    for (int h = 0; h < 8; h++) sh.ucnt[h] = 0.0f;
                }
                bar_named(1, NC * 32);
                if (sh.flag) {
                    // last CTA of the unit: merge its records u + ilo .. u + ihi in fixed order, warp per head
                    const float* pu = a.parts + (size_t)(u + ilo) * G * PREC;
                    const int64_t b = u / a.Hkv, hkv = u % a.Hkv;
                    const int64_t qh0 = b * a.Hq + hkv * G;
#pragma unroll 1
                    for (int g = warp; g < G; g += NC) {
                        float M = -INFINITY, S = 0.0f, C = 0.0f;
                        float4 A = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll 1
                        for (int c0 = 0; c0 < np; c0 += MB) {
                            const int nr = min(MB, np - c0);
                            float4 av[MB];
#pragma unroll
                            for (int jj = 0; jj < MB; jj++)
                                av[jj] = jj < nr ? __ldcg(reinterpret_cast<const float4*>(
                                                           pu + ((size_t)(c0 + jj) * G + g) * PREC + 4) +
                                                       lane)
                                                 : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                            const float4 hd =
                                lane < nr ? __ldcg(reinterpret_cast<const float4*>(pu + ((size_t)(c0 + lane) * G + g) * PREC))
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
                            for (int jj = 0; jj < MB; jj++) {
                                const float fj = __shfl_sync(0xffffffffu, fc, jj);
                                A.x = fmaf(fj, av[jj].x, A.x);
                                A.y = fmaf(fj, av[jj].y, A.y);
                                A.z = fmaf(fj, av[jj].z, A.z);
                                A.w = fmaf(fj, av[jj].w, A.w);
                            }
                            M = Mn;
                        }
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
                    if (ctid == 0) a.unit_ctr[u] = 0u;
                }
                bar_named(1, NC * 32);  // combine area reusable
            }
            if (lane == 0) mbar_arrive(&sh.empty[d % NDESC]);
            continue;
        }

        // ---- slab j of descriptor d
        if (D.unit != cur_u) {
            cur_u = D.unit;
            load_unit(cur_u);
        }
        const int st = computed % NST;
        mbar_wait(&wb.bar[st], (uint32_t)((computed / NST) & 1));
        const int e0 = (j - D.slab0) * SR;
        const int nr = min(SR, D.n - e0);
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
                xf[0] = xbar_pair(af[0], ca.x, ca.y);
                xf[1] = xbar_pair(af[1], ca.x, ca.y);
                xf[2] = xbar_pair(af[2], cb.x, cb.y);
                xf[3] = xbar_pair(af[3], cb.x, cb.y);
                mma16816(dx, xf, qf[ks][0], qf[ks][1]);
            }
        }
        // (2) items (row, head): ra = g4 (dl[0], dl[1]), rb = g4 + 8 (dl[2], dl[3]); heads h0, h1
        const uint32_t ba = g4 < nr ? sh.bits[(int)(D.e0 + e0 + g4) & (ERING - 1)] : 0u;
        const uint32_t bb = g4 + 8 < nr ? sh.bits[(int)(D.e0 + e0 + g4 + 8) & (ERING - 1)] : 0u;
        const float xna = wb.xn[st][g4], xnb = wb.xn[st][g4 + 8];
        bool need[4];
        float cs[4];
        {
            const uint32_t bt[4] = {ba, ba, bb, bb};
            const int hh[4] = {h0, h1, h0, h1};
            const float qn[4] = {qn0, qn1, qn0, qn1};
            const float xn[4] = {xna, xna, xnb, xnb};
#pragma unroll
            for (int i = 0; i < 4; i++) {
                need[i] = hh[i] < G && !(bt[i] & 0x100u) && ((bt[i] >> hh[i]) & 1u);
                const float den = qn[i] * xn[i];
                float c = den > 0.0f ? __fdividef(dx[i], den) : 0.0f;
                cs[i] = fminf(1.0f, fmaxf(-1.0f, c));
            }
        }
        // compact the items that need ln u over the warp (one MUFU chain per lane per round)
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
                wb.items[e] = log_sampling_prob(p, a.K, a.L, a.minc);
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; i++)
                if (need[i]) lu[i] = wb.items[pos[i]];
        }
        float z[4];
        {
            const uint32_t bt[4] = {ba, ba, bb, bb};
            const int hh[4] = {h0, h1, h0, h1};
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const float l = dl[i] * INV_SQRT_D;
                z[i] = (hh[i] < G && (bt[i] & 0x100u)) ? l : (need[i] ? l - lu[i] : -INFINITY);
            }
        }
        if (a.weighted) {
            const uint32_t bt[2] = {ba, bb};
            const int64_t b = cur_u / a.Hkv, hkv = cur_u % a.Hkv;
            const int64_t qh0 = b * a.Hq + hkv * G;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int r = (i >> 1) ? g4 + 8 : g4;
                const int h = (i & 1) ? h1 : h0;
                if (z[i] != -INFINITY && r < nr) {
                    (void)bt;
                    const int key = sh.keys[(int)(D.e0 + e0 + r) & (ERING - 1)];
                    atomicOr(a.weighted + (qh0 + h) * nwb + (key >> 5), 1u << (key & 31));
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
            const int hh[4] = {h0, h1, h0, h1};
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
        __syncwarp();  // stage buffer and weight tile free
        computed++;
    }
}

}  // namespace v6

// ---- host: shared-memory layout and launch
static size_t al128(size_t x) { return (x + 127) & ~(size_t)127; }

size_t attend_layout(AttendArgs& a, int G) {
    size_t off = al128(sizeof(v6::Shared));
    a.off_wbuf = (int)off;
    off += al128(sizeof(v6::WarpBuf) * v6::NC);
    a.off_comb = (int)off;
    off += al128((size_t)v6::NC * G * 132 * 4);
    return off;
}

template <int G>
static int launch6_g(AttendArgs a, int nsm, int max_smem, cudaStream_t st) {
    const size_t smem = attend_layout(a, G);
    if (smem > (size_t)max_smem) return MAGICPIG_EINVAL;
    auto kern = v6::attend_kernel<G>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MAGICPIG_ECUDA;
    const int64_t P = a.tiles < nsm ? a.tiles : nsm;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)P);
    cfg.blockDim = dim3(v6::THREADS);
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

int launch_attend(const AttendArgs& a, int nsm, int max_smem, cudaStream_t st) {
    const int G = (int)(a.Hq / a.Hkv);
    switch (G) {
        case 1: return launch6_g<1>(a, nsm, max_smem, st);
        case 2: return launch6_g<2>(a, nsm, max_smem, st);
        case 4: return launch6_g<4>(a, nsm, max_smem, st);
        case 8: return launch6_g<8>(a, nsm, max_smem, st);
    }
    return MAGICPIG_EINVAL;
}

}  // namespace mp
