// estimate8.cu -- the self-normalised importance-sampling estimator of a MagicPIG
// decode step (Algorithm 1) on the 5th-generation tensor cores:
//     o_g = sum_{i in S_g u T} e^{z_i} v_i / sum e^{z_i},
//     z_i = q_g.k_i / sqrt(d) - ln u_i     (u_i = 1 on the static set T)
// with u_i the closed-form sampling probability (Eq. P:86-91) at the angle between
// the hashed vectors xbar_i = [bf16(fl32(k_i - c)), s_i] and qbar = [q, 0] (R5).
//
// Input: the per-piece union lists of the select step (pieces.cuh).  The unit
// lists (each preceded by the unit's static keys) are concatenated; CTA i of
// the persistent grid owns the contiguous range [i E / P, (i+1) E / P) of that
// sequence, cut into tiles of <= 128 rows at unit boundaries.  Per CTA:
//
//   warp 0  producer  per tile: entries -> rows; row head bits and |xbar_i|,
//                     the unit's q tile (UMMA K-major operand), -c and |q_g|
//                     into the stage's info area; K and V rows by TMA gather4
//                     (cp.async.bulk.tensor ... tile::gather4, 4 rows x 64
//                     columns per instruction, 128B-swizzled) into two stages.
//   warp 1  MMA       one thread issues tcgen05.mma (bf16, fp32 accumulate in
//                     TMEM, double-buffered per tile):
//                       logits  L[128 rows][16]  = K . Q^T   (A: K-major SW128)
//                       hashed  H[128 rows][16]  = X . Q^T   (X = xbar in place of K)
//                       PV      A[128 d][16]     = V^T . W   (A: V tile as an
//                                                 MN-major SW128 operand; B: weights)
//   warps 2-9 compute (TMEM lane quadrant = warp % 4; heads split in two halves)
//                     in-place K -> X (x = bf16(fl32(k - c)), swizzle-aware), then
//                     one thread per row: cos -> p -> ln u (table) -> z for the
//                     (row, head) items in S, tile max / weights (hi + lo bf16
//                     parts: fp32-accurate) / tile sum, the weight tile W; then one
//                     thread per dimension d combines the tile's PV accumulator into
//                     the running (m, s, a) of the unit (log-sum-exp).
// When the CTA leaves a unit it writes its record (m, s, a) to parts[u + cta]; the
// v7 merge kernel reduces the records of each unit in CTA order ("recursive
// attention").
#include <cuda_bf16.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"
#include "pieces.cuh"

namespace mp {
namespace v8 {

using v7::StaticRanges;
using v7::static_ranges;
using v7::warp_incl_scan;

constexpr int TR = 128;                      // rows per tile (UMMA M)
constexpr int NSK = 3;                       // K stages (freed after the hashed-dot MMA)
constexpr int NSV = 2;                       // V stages (freed after the PV MMA)
constexpr int NI = 4;                        // tile-info ring (the producer runs up to NI tiles ahead)
constexpr int NLW = 4;                       // loader warps (cp.async of the K / V rows)
constexpr int NLT = NLW * 32;
constexpr int NCW = 8;                       // compute warps
constexpr int NCT = NCW * 32;
constexpr int CW0 = 2 + NLW;                 // first compute warp
constexpr int THREADS = (2 + NLW + NCW) * 32;
constexpr int PREC = PREC5;                  // record per head: m, s, 0, 0, a[128]
constexpr float INV_SQRT_D = 0.08838834764831845f;

// shared memory layout
constexpr int TILE = 32768;                  // one K or V tile: 2 x 16 KB halves, SW128
constexpr int OFF_V = NSK * TILE;
constexpr int OFF_INFO = OFF_V + NSV * TILE;
constexpr int INFO_QT = 0;                   // q tile: K-major no-swizzle, (n, k) at (n/8)*2048 + (k/8)*128 + (n%8)*16 + (k%8)*2
constexpr int INFO_C = 4096;                 // -c [128] f32
constexpr int INFO_BITS = 4608;              // head bits per row [128] u32 (0x100: static)
constexpr int INFO_KEY = 5120;               // local key per row [128] i32
constexpr int INFO_QN = 5632;                // |q_g| [16] f32
constexpr int INFO_BYTES = 6144;
constexpr int OFF_W = OFF_INFO + NI * INFO_BYTES;  // 2 weight tiles (MN-major no-swizzle) x 4 KB
constexpr int OFF_RED = OFF_W + 2 * 4096;    // tile max / sum per (quadrant, head): [2][4][8] f32
constexpr int OFF_BAR = OFF_RED + 256;
constexpr int NBAR = 2 * NSK + 2 * NSV + 2 * NI + 5 * 2;
constexpr int OFF_PREF = OFF_BAR + NBAR * 8 + 16;  // + tmem slot; piece prefix follows
static_assert(OFF_V % 1024 == 0 && OFF_INFO % 1024 == 0, "stage alignment (SWIZZLE_128B atoms)");

struct Est8Args {
    EstArgs e;
    int P;  // pieces per unit
};

// UMMA shared-memory descriptor with 128-byte swizzle (atoms of 8 rows x 128 B, 1024-B aligned)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return umma_desc(saddr, lbo, sbo) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// named barrier of the compute warps; the two head halves reach it from different instantiations (code
// addresses) of the compute loop, hence the non-.aligned form
__device__ __forceinline__ void bar_cw() { asm volatile("barrier.sync 1, %0;" ::"n"(NCT) : "memory"); }
__device__ __forceinline__ int64_t owner_of(int64_t e, int64_t E, int64_t W) { return ((e + 1) * W - 1) / E; }

template <int G>
__global__ void __launch_bounds__(THREADS, 1) estimate8_kernel(const Est8Args A8) {
    constexpr int HP = (G + 1) / 2;  // heads per compute half
    extern __shared__ __align__(1024) uint8_t sm[];
    const EstArgs& a = A8.e;
    const int P = A8.P;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
    uint64_t* fullK = bars;            // [NSK] K rows landed (cp.async arrivals of the loader threads)
    uint64_t* kfree = fullK + NSK;     // [NSK] K region read for the last time (hashed MMA done)
    uint64_t* fullV = kfree + NSK;     // [NSV] V rows landed
    uint64_t* vfree = fullV + NSV;     // [NSV] V region read for the last time (PV MMA done)
    uint64_t* meta = vfree + NSV;      // [NI] tile info written (producer lanes)
    uint64_t* ifree = meta + NI;       // [NI] tile info consumed
    uint64_t* lbar = ifree + NI;       // [2] logits done
    uint64_t* xbar = lbar + 2;         // [2] X written
    uint64_t* hbar = xbar + 2;         // [2] hashed dots done
    uint64_t* wbar = hbar + 2;         // [2] weight tile written
    uint64_t* pvbar = wbar + 2;        // [2] PV done
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + NBAR);
    int* pref = reinterpret_cast<int*>(sm + OFF_PREF);
    float* red = reinterpret_cast<float*>(sm + OFF_RED);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t units = a.B * a.Hkv;
    const StaticRanges sr = static_ranges(a);
    const int nT = (int)(sr.len1 + sr.len2);
    const int NP = (int)units * P;
    // debug timeline (one row of 16 per CTA): 0 start, 1 prefix done, 2/3 producer first/last tile info,
    // 4 first logits issued, 5 compute first logits ready, 6 compute loop end, 7 end; 8 tiles;
    // 9..12 compute-thread-0 wait time (ns) on K rows / logits / hashed / PV
    unsigned long long* tl = a.timeline ? a.timeline + (size_t)blockIdx.x * 16 : nullptr;
    auto stamp = [&](int i) {
        if (tl) tl[i] = gtime();
    };
    if (tid == 0) stamp(0);

    if (tid == 0) {
        for (int s = 0; s < NSK; s++) {
            mbar_init(&fullK[s], NLT);
            mbar_init(&kfree[s], 1);
        }
        for (int s = 0; s < NSV; s++) {
            mbar_init(&fullV[s], NLT);
            mbar_init(&vfree[s], 1);
        }
        for (int i = 0; i < NI; i++) {
            mbar_init(&meta[i], 32);
            mbar_init(&ifree[i], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&lbar[b], 1);
            mbar_init(&xbar[b], 1);
            mbar_init(&hbar[b], 1);
            mbar_init(&wbar[b], 1);
            mbar_init(&pvbar[b], 1);
        }
        fence_mbar_init();
    }
    // zero the q tiles (rows >= G stay 0) and the weight tiles (columns >= 2G stay 0)
    for (int e = tid; e < NI * 1024; e += THREADS)
        reinterpret_cast<uint32_t*>(sm + OFF_INFO + (e / 1024) * INFO_BYTES + INFO_QT)[e % 1024] = 0u;
    for (int e = tid; e < 2 * 1024; e += THREADS) reinterpret_cast<uint32_t*>(sm + OFF_W)[e] = 0u;
    if (warp == 1) {
        tmem_alloc(tslot, 128);
        tmem_relinquish();
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // lists of the select step
    // ---- piece prefix (as v7): piece u*P = unit u's static keys, u*P + 1 + c = the list of chunk c
    {
        __shared__ int wsum[THREADS / 32];
        for (int p0 = tid; p0 < NP; p0 += 8 * THREADS) {  // 8 loads in flight per thread, then the stores
            int v[8];
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const int pp = p0 + k * THREADS;
                const int u = pp / P, cc = pp - u * P;
                v[k] = pp >= NP ? 0 : (cc == 0 ? nT : __ldcg(a.pcnt + (int64_t)u * a.nchunks + cc - 1));
            }
#pragma unroll
            for (int k = 0; k < 8; k++)
                if (p0 + k * THREADS < NP) pref[p0 + k * THREADS] = v[k];
        }
        __syncthreads();
        const int per = (NP + THREADS - 1) / THREADS;
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
        if (tid == THREADS - 1) pref[NP] = run;
    }
    fence_proxy_async();  // zeroed q / weight tiles before the tensor core reads them
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const int64_t E = pref[NP];
    if (tid == 0) stamp(1);
    const int64_t Pc = gridDim.x;
    if (blockIdx.x == 0) {  // record table for the merge kernel
        for (int64_t u = tid; u < units; u += THREADS) {
            int2 r = make_int2(0, 0);
            const int64_t e0 = pref[u * P], e1 = pref[(u + 1) * P];
            if (e1 > e0) {
                const int64_t k_lo = owner_of(e0, E, Pc), k_hi = owner_of(e1 - 1, E, Pc);
                r = make_int2((int)k_lo, (int)(k_hi - k_lo + 1));
            }
            a.urec[u] = r;
        }
    }
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t e_lo = E > 0 ? (int64_t)blockIdx.x * E / Pc : 0, e_hi = E > 0 ? ((int64_t)blockIdx.x + 1) * E / Pc : 0;
    // tile sequence of this CTA (every role walks it identically): tile = <= 128 entries of one unit
    const int u_lo = [&]() {  // unit of the CTA's first entry
        int lo = 0, hi = (int)units;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pref[mid * P] <= e_lo) lo = mid;
            else hi = mid;
        }
        return lo;
    }();
    auto next_tile = [&](int64_t cur, int& u, int& nr) {
        while (pref[(u + 1) * P] <= cur) u++;
        const int64_t uend = min(e_hi, (int64_t)pref[(u + 1) * P]);
        nr = (int)min((int64_t)TR, uend - cur);
    };

    if (warp == 0) {
        // ============================================================ producer: tile info + L2 prefetch
        int u = u_lo, nr = 0, t = 0;
        int ps = 0;  // piece holding the cursor
        {
            int lo = 0, hi = NP;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (pref[mid] <= e_lo) lo = mid;
                else hi = mid;
            }
            ps = lo;
        }
#pragma unroll 1
        for (int64_t cur = e_lo; cur < e_hi; cur += nr, t++) {
            next_tile(cur, u, nr);
            const int i = t % NI;
            if (t >= NI) mbar_wait(&ifree[i], (uint32_t)(((t / NI) - 1) & 1));
            uint8_t* info = sm + OFF_INFO + i * INFO_BYTES;
            uint32_t* rbits = reinterpret_cast<uint32_t*>(info + INFO_BITS);
            int* rkey = reinterpret_cast<int*>(info + INFO_KEY);
            while (pref[ps + 1] <= cur) ps++;
            // rows r = lane + 32 j: entry cur + r (pad rows: the tile's first row, weight 0)
            uint32_t ent[4];
            int jv[4], cv[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int r = lane + 32 * j;
                const int e = (int)cur + (r < nr ? r : 0);
                int pi = ps;
                while (pref[pi + 1] <= e) pi++;
                jv[j] = e - pref[pi];
                cv[j] = pi - u * P;
                ent[j] = cv[j] > 0 ? __ldcg(a.ents + ((int64_t)u * a.nchunks + cv[j] - 1) * KCHUNK + jv[j]) : 0u;
            }
            const int64_t b = u / a.Hkv, hkv = u % a.Hkv, qh0 = b * a.Hq + hkv * G;
            uint2 qv[G];
#pragma unroll
            for (int g = 0; g < G; g++) qv[g] = __ldg(reinterpret_cast<const uint2*>(a.q + (qh0 + g) * HD) + lane);
            const float4 cvec = __ldg(reinterpret_cast<const float4*>(a.center + (int64_t)u * HD) + lane);
            const int64_t rb = (int64_t)u * a.n_local;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int r = lane + 32 * j;
                int key;
                uint32_t bits;
                if (cv[j] == 0) {
                    key = (int)(jv[j] < sr.len1 ? sr.lo1 + jv[j] : sr.lo2 + (jv[j] - sr.len1));
                    bits = 0x100u | ((1u << G) - 1u);
                } else {
                    key = (int)(ent[j] & 0xffffffu);
                    bits = ent[j] >> 24;
                }
                rbits[r] = r < nr ? bits : 0u;
                rkey[r] = key;
                // the rows' K and V lines into L2 now: the compute warps' copies of this tile, NI tiles later at
                // most, then hit L2
                const uint16_t* kr = a.k + (rb + key) * HD;
                const uint16_t* vr = a.v + (rb + key) * HD;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(kr));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(kr + 64));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(vr));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(vr + 64));
            }
            uint8_t* qt = info + INFO_QT;
#pragma unroll
            for (int g = 0; g < G; g++) {
                const int k = 4 * lane;  // this lane's 4 elements of q_g
                *reinterpret_cast<uint2*>(qt + (g / 8) * 2048 + (k / 8) * 128 + (g % 8) * 16 + (k % 8) * 2) = qv[g];
                float sq = 0.0f;
                const uint32_t w2[2] = {qv[g].x, qv[g].y};
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const float lo = __uint_as_float(w2[h] << 16), hi = __uint_as_float(w2[h] & 0xffff0000u);
                    sq = fmaf(lo, lo, fmaf(hi, hi, sq));
                }
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, m);
                if (lane == 0) reinterpret_cast<float*>(info + INFO_QN)[g] = sqrtf(sq);
            }
            reinterpret_cast<float4*>(info + INFO_C)[lane] = make_float4(-cvec.x, -cvec.y, -cvec.z, -cvec.w);
            fence_proxy_async();  // q tile (generic writes) before the tensor core reads it
            mbar_arrive(&meta[i]);
            if (lane == 0) stamp(t == 0 ? 2 : 3);
        }
    } else if (warp == 1) {
        // ============================================================ MMA issuer
        if (lane == 0) {
            const uint32_t idesc_k = umma_idesc_bf16(TR, 16);
            const uint32_t idesc_mn = umma_idesc_bf16(TR, 16) | (1u << 15) | (1u << 16);  // A, B MN-major
            // logits of tile t + 1 are issued right after the hashed dots of tile t (before waiting for tile t's
            // weights), so the compute warps find them ready when they finish tile t
            auto logits = [&](int t) {
                const int sk = t % NSK, b = t & 1, i = t % NI;
                mbar_wait(&meta[i], (uint32_t)((t / NI) & 1));
                mbar_wait(&fullK[sk], (uint32_t)((t / NSK) & 1));
                fence_proxy_async();  // the K rows were written by cp.async (generic proxy): visible to the MMA
                tc_fence_after();
                const uint32_t kb = smem_u32(sm + sk * TILE);
                const uint32_t qb = smem_u32(sm + OFF_INFO + i * INFO_BYTES + INFO_QT);
#pragma unroll
                for (int kk = 0; kk < 8; kk++)
                    umma_bf16(tmem + b * 48, desc_sw128(kb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                              umma_desc(qb + kk * 256, 128, 2048), idesc_k, kk > 0);
                umma_commit(&lbar[b]);
                if (t == 0) stamp(4);
            };
            int u = u_lo, nr = 0, t = 0;
            if (e_lo < e_hi) logits(0);
#pragma unroll 1
            for (int64_t cur = e_lo; cur < e_hi; cur += nr, t++) {
                next_tile(cur, u, nr);
                const int sk = t % NSK, sv = t % NSV, b = t & 1, i = t % NI;
                const uint32_t ph = (uint32_t)((t >> 1) & 1);
                const uint32_t kb = smem_u32(sm + sk * TILE), vb = smem_u32(sm + OFF_V + sv * TILE);
                const uint32_t qb = smem_u32(sm + OFF_INFO + i * INFO_BYTES + INFO_QT);
                const uint32_t wb = smem_u32(sm + OFF_W + b * 4096);
                const uint32_t tb = tmem + b * 48;
                mbar_wait(&xbar[b], ph);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; kk++)
                    umma_bf16(tb + 16, desc_sw128(kb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                              umma_desc(qb + kk * 256, 128, 2048), idesc_k, kk > 0);
                umma_commit(&hbar[b]);
                umma_commit(&kfree[sk]);
                // TMEM buffer (t + 1) & 1 was last read by the compute warps for tile t - 1, before wbar(t - 1)
                if (cur + nr < e_hi) logits(t + 1);
                mbar_wait(&wbar[b], ph);
                mbar_wait(&fullV[sv], (uint32_t)((t / NSV) & 1));
                fence_proxy_async();
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; kk++)
                    umma_bf16(tb + 32, desc_sw128(vb + kk * 2048, 16384, 1024), umma_desc(wb + kk * 256, 128, 2048),
                              idesc_mn, kk > 0);
                umma_commit(&pvbar[b]);
                umma_commit(&vfree[sv]);
            }
        }
    } else if (warp < CW0) {
        // ============================================================ loaders: K / V rows by cp.async (LSU path)
        const int lt = tid - 64;
        int u = u_lo, nr = 0, t = 0;
#pragma unroll 1
        for (int64_t cur = e_lo; cur < e_hi; cur += nr, t++) {
            next_tile(cur, u, nr);
            const int sk = t % NSK, sv = t % NSV;
            mbar_wait(&meta[t % NI], (uint32_t)((t / NI) & 1));
            const int* rkey = reinterpret_cast<const int*>(sm + OFF_INFO + (t % NI) * INFO_BYTES + INFO_KEY);
            // thread's 16 chunks per tensor: rows r0 + 8 k, 16-B column j (constant), swizzled position
            const int cj = lt & 15, cr0 = lt >> 4;
            const uint32_t coff = (uint32_t)((cj >> 3) * 16384 + cr0 * 128 + (((cj & 7) ^ (cr0 & 7)) << 4));
            int key[16];
#pragma unroll
            for (int k = 0; k < 16; k++) key[k] = rkey[cr0 + 8 * k];
            const int64_t ub = (int64_t)u * a.n_local;
            const uint16_t* kb = a.k + ub * HD + cj * 8;
            const uint16_t* vb = a.v + ub * HD + cj * 8;
            const uint32_t dk = smem_u32(sm + sk * TILE) + coff, dv = smem_u32(sm + OFF_V + sv * TILE) + coff;
            if (t >= NSK) mbar_wait(&kfree[sk], (uint32_t)(((t / NSK) - 1) & 1));
#pragma unroll
            for (int k = 0; k < 16; k++) cp16(dk + k * 1024, kb + (int64_t)key[k] * HD);
            cp_arrive_noinc(&fullK[sk]);
            if (t >= NSV) mbar_wait(&vfree[sv], (uint32_t)(((t / NSV) - 1) & 1));
#pragma unroll
            for (int k = 0; k < 16; k++) cp16(dv + k * 1024, vb + (int64_t)key[k] * HD);
            cp_arrive_noinc(&fullV[sv]);
        }
    } else {
        // ============================================================ compute warps
        const int cw = warp - CW0, ct = tid - CW0 * 32, quad = warp & 3, half = cw >> 2;
        const int row = quad * 32 + lane;  // TMEM lane: tile row (logits / dots) and dimension d (PV)
        const uint32_t tq = tmem + ((uint32_t)(quad * 32) << 16);
        // the two halves of the compute warps handle heads [HALF * HP, ...): compile-time head indices keep
        // the TMEM rows in registers (no dynamic indexing)
        auto run = [&](auto half_c) {
        constexpr int h_lo = decltype(half_c)::value * HP, h_hi = G < h_lo + HP ? G : h_lo + HP;
        float Mr[HP], Sr[HP], Ar[HP];  // running state of the current unit (heads h_lo..); Ar for dimension row
        float mt[HP], st[HP];          // the previous tile's max / sum (for its PV combine)
        int cur_u = -1, prev_u = -1;
#pragma unroll
        for (int j = 0; j < HP; j++) Mr[j] = -INFINITY, Sr[j] = 0.0f, Ar[j] = 0.0f, mt[j] = -INFINITY, st[j] = 0.0f;
        // K or V rows of tile tn (unit un) into stage tn % NS: 16-B chunks to their 128B-swizzled places
        auto flush = [&](int u) {
            float* rec = a.parts + (size_t)(u + blockIdx.x) * G * PREC;
#pragma unroll
            for (int j = 0; j < HP; j++) {
                const int h = h_lo + j;
                if (h < h_hi) {
                    __stcg(rec + h * PREC + 4 + row, Ar[j]);
                    if (row == 0) __stcg(reinterpret_cast<float2*>(rec + h * PREC), make_float2(Mr[j], Sr[j]));
                }
                Mr[j] = -INFINITY, Sr[j] = 0.0f, Ar[j] = 0.0f;
            }
        };
        auto combine_prev = [&](int tp) {  // PV accumulator of tile tp -> running state of its unit
            const int bp = tp & 1;
            const unsigned long long w4 = (tl && ct == 0) ? gtime() : 0ull;
            mbar_wait(&pvbar[bp], (uint32_t)((tp >> 1) & 1));
            if (tl && ct == 0) tl[12] += gtime() - w4;
            tc_fence_after();
            float pv[16];
            tmem_ld16(tq + bp * 48 + 32, pv);
            if (prev_u != cur_u) {
                if (cur_u >= 0) flush(cur_u);
                cur_u = prev_u;
            }
#pragma unroll
            for (int j = 0; j < HP; j++) {
                const int h = h_lo + j;
                if (h < h_hi && st[j] > 0.0f) {
                    const float at = pv[h] + pv[G + h];
                    const float Mn = fmaxf(Mr[j], mt[j]);
                    const float fo = Mr[j] == -INFINITY ? 0.0f : __expf(Mr[j] - Mn);
                    const float fn = __expf(mt[j] - Mn);
                    Ar[j] = Ar[j] * fo + at * fn;
                    Sr[j] = Sr[j] * fo + st[j] * fn;
                    Mr[j] = Mn;
                }
            }
        };
        int u = u_lo, nr = 0, t = 0;
#pragma unroll 1
        for (int64_t cur = e_lo; cur < e_hi; cur += nr, t++) {
            next_tile(cur, u, nr);
            const int sk = t % NSK, b = t & 1, i = t % NI;
            const uint32_t ph = (uint32_t)((t >> 1) & 1);
            uint8_t* kt = sm + sk * TILE;
            const uint8_t* info = sm + OFF_INFO + i * INFO_BYTES;
            const unsigned long long q0 = (tl && ct == 0) ? gtime() : 0ull;
            mbar_wait(&meta[i], (uint32_t)((t / NI) & 1));
            // |xbar| of this thread's row (used in (c); the load is in flight during (a) and (b))
            const float xn = __ldg(a.key_norm + (int64_t)u * a.n_local + reinterpret_cast<const int*>(info + INFO_KEY)[row]);
            const unsigned long long w0 = (tl && ct == 0) ? gtime() : 0ull;
            mbar_wait(&fullK[sk], (uint32_t)((t / NSK) & 1));  // every loader thread's K copies landed
            const unsigned long long w1 = (tl && ct == 0) ? gtime() : 0ull;
            mbar_wait(&lbar[b], ph);
            if (tl && ct == 0) {
                const unsigned long long w2 = gtime();
                tl[9] += w1 - w0;
                tl[10] += w2 - w1;
                if (t == 0) tl[5] = w2;
            }
            tc_fence_after();
            float lv[16];
            tmem_ld16(tq + b * 48, lv);
            const unsigned long long q1 = (tl && ct == 0) ? gtime() : 0ull;
            // (a) in-place xbar = bf16(fl32(k - c)); 16-B chunk js of row r holds logical chunk js ^ (r % 8).
            // This thread's chunks: ct + 256 k -> half k / 4, rows (ct / 8) + 32 (k % 4), chunk ct % 8: the
            // logical column block is the same for all of them within a half.
            {
                const float* nc = reinterpret_cast<const float*>(info + INFO_C);
                const int dblk = ((ct & 7) ^ ((ct >> 3) & 7)) << 3;
                float2 cc[2][4];
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    const float4 c0 = *reinterpret_cast<const float4*>(nc + hh * 64 + dblk);
                    const float4 c1 = *reinterpret_cast<const float4*>(nc + hh * 64 + dblk + 4);
                    cc[hh][0] = make_float2(c0.x, c0.y), cc[hh][1] = make_float2(c0.z, c0.w);
                    cc[hh][2] = make_float2(c1.x, c1.y), cc[hh][3] = make_float2(c1.z, c1.w);
                }
                uint4* p0 = reinterpret_cast<uint4*>(kt + ct * 16);
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    uint4* p = p0 + (k >> 2) * 1024 + (k & 3) * 256;  // + half * 16 KB + 32 rows per step
                    uint4 x = *p;
                    uint32_t* w4 = reinterpret_cast<uint32_t*>(&x);
#pragma unroll
                    for (int k2 = 0; k2 < 4; k2++) {
                        const float2 xv = __fadd2_rn(
                            make_float2(__uint_as_float(w4[k2] << 16), __uint_as_float(w4[k2] & 0xffff0000u)),
                            cc[k >> 2][k2]);
                        const __nv_bfloat162 xb = __floats2bfloat162_rn(xv.x, xv.y);
                        w4[k2] = *reinterpret_cast<const uint32_t*>(&xb);
                    }
                    *p = x;
                }
            }
            fence_proxy_async();
            bar_cw();
            if (ct == 0) mbar_arrive(&xbar[b]);
            const unsigned long long q2 = (tl && ct == 0) ? gtime() : 0ull;
            // (b) the previous tile's PV accumulator; then its stage's V region is free for the next tile
            if (t > 0) combine_prev(t - 1);
            // (c) softmax of this tile: one thread per row, heads h_lo .. h_hi
            const unsigned long long w3 = (tl && ct == 0) ? gtime() : 0ull;
            mbar_wait(&hbar[b], ph);
            if (tl && ct == 0) tl[11] += gtime() - w3;
            tc_fence_after();
            float hv[16];
            tmem_ld16(tq + b * 48 + 16, hv);
            const uint32_t bits = reinterpret_cast<const uint32_t*>(info + INFO_BITS)[row];
            const float* qn = reinterpret_cast<const float*>(info + INFO_QN);
            float z[HP];
#pragma unroll
            for (int j = 0; j < HP; j++) {
                const int h = h_lo + j;
                z[j] = -INFINITY;
                if (h < h_hi) {
                    const float l = lv[h] * INV_SQRT_D;
                    if (bits & 0x100u) {
                        z[j] = l;
                    } else if ((bits >> h) & 1u) {
                        const float den = qn[h] * xn;
                        const float cs = fminf(1.0f, fmaxf(-1.0f, den > 0.0f ? __fdividef(hv[h], den) : 0.0f));
                        const float p = 1.0f - acosf(cs) * 0.3183098861837907f;
                        z[j] = l - log_sampling_prob_lut(a.lutab, p, a.K, a.L, a.minc);
                    }
                }
            }
            if (a.weighted) {
                const int64_t bb = u / a.Hkv, hkv = u % a.Hkv, qh0 = bb * a.Hq + hkv * G;
                const int64_t nwb = (a.n_local + 31) >> 5;
                const int key = reinterpret_cast<const int*>(info + INFO_KEY)[row];
#pragma unroll
                for (int j = 0; j < HP; j++)
                    if (z[j] != -INFINITY && row < nr)
                        atomicOr(a.weighted + (qh0 + h_lo + j) * nwb + (key >> 5), 1u << (key & 31));
            }
            // tile max per head over the 128 rows
#pragma unroll
            for (int j = 0; j < HP; j++) {
                float m = z[j];
#pragma unroll
                for (int k = 16; k >= 1; k >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, k));
                if (lane == 0) red[quad * 8 + h_lo + j] = m;
            }
            bar_cw();
            uint16_t* wt = reinterpret_cast<uint16_t*>(sm + OFF_W + b * 4096);
#pragma unroll
            for (int j = 0; j < HP; j++) {
                const int h = h_lo + j;
                const float m = fmaxf(fmaxf(red[h], red[8 + h]), fmaxf(red[16 + h], red[24 + h]));
                mt[j] = m;
                const float w = (z[j] == -INFINITY) ? 0.0f : __expf(z[j] - m);
                const __nv_bfloat16 whi = __float2bfloat16_rn(w);
                const __nv_bfloat16 wlo = __float2bfloat16_rn(w - __bfloat162float(whi));
                if (h < h_hi) {
                    // W (MN-major, no swizzle): (n, k = row) at (n/8)*2048 + (k/8)*128 + (k%8)*16 + (n%8)*2
                    const int n1 = h, n2 = G + h;
                    wt[((n1 >> 3) * 2048 + (row >> 3) * 128 + (row & 7) * 16 + (n1 & 7) * 2) >> 1] =
                        *reinterpret_cast<const uint16_t*>(&whi);
                    wt[((n2 >> 3) * 2048 + (row >> 3) * 128 + (row & 7) * 16 + (n2 & 7) * 2) >> 1] =
                        *reinterpret_cast<const uint16_t*>(&wlo);
                }
                float sv = __bfloat162float(whi) + __bfloat162float(wlo);
#pragma unroll
                for (int k = 16; k >= 1; k >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, k);
                if (lane == 0) red[32 + quad * 8 + h] = sv;
            }
            fence_proxy_async();
            bar_cw();
            if (ct == 0) {
                mbar_arrive(&wbar[b]);
                mbar_arrive(&ifree[i]);  // this tile's info (q tile, bits, keys, -c, |q|) is no longer read
            }
#pragma unroll
            for (int j = 0; j < HP; j++) {
                const int h = h_lo + j;
                st[j] = (red[32 + h] + red[32 + 8 + h]) + (red[32 + 16 + h] + red[32 + 24 + h]);
            }
            bar_cw();  // red reusable
            prev_u = u;
            if (tl && ct == 0) {
                const unsigned long long q3 = gtime();
                tl[13] += q1 - q0;
                tl[14] += q2 - q1;
                tl[15] += q3 - q2;
            }
        }
        if (t > 0) combine_prev(t - 1);
        if (cur_u >= 0) flush(cur_u);
        if (ct == 0) {
            stamp(6);
            if (tl) tl[8] = (unsigned long long)t;
        }
            };
        if (half == 0) run(std::integral_constant<int, 0>{});
        else run(std::integral_constant<int, 1>{});
    }

    tc_fence_before();
    __syncthreads();
    if (tid == 0) stamp(7);
    if (warp == 1) tmem_dealloc(tmem, 128);
}

}  // namespace v8

// ---- host
size_t estimate8_smem(const EstArgs& a) {
    const int64_t NP = a.B * a.Hkv * (a.nchunks + 1);
    return (size_t)v8::OFF_PREF + (size_t)(NP + 1) * 4;
}

template <int G>
static int launch8_g(const EstArgs& a, int nsm, int max_smem, cudaStream_t st) {
    const size_t smem = estimate8_smem(a);
    if (smem > (size_t)max_smem) return MAGICPIG_EINVAL;
    auto kern = v8::estimate8_kernel<G>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MAGICPIG_ECUDA;
    v8::Est8Args a8;
    a8.e = a;
    a8.P = (int)a.nchunks + 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nsm);
    cfg.blockDim = dim3(v8::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a8);
    count_launch(1);
    return e == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

bool estimate8_ok(const EstArgs& a, int max_smem) {
    return estimate8_smem(a) <= (size_t)max_smem && a.n_local < (1 << 24);
}

int launch_estimate8(const EstArgs& a, int nsm, int max_smem, cudaStream_t st) {
    switch ((int)(a.Hq / a.Hkv)) {
        case 1: return launch8_g<1>(a, nsm, max_smem, st);
        case 2: return launch8_g<2>(a, nsm, max_smem, st);
        case 4: return launch8_g<4>(a, nsm, max_smem, st);
        case 8: return launch8_g<8>(a, nsm, max_smem, st);
    }
    return MAGICPIG_EINVAL;
}

}  // namespace mp
