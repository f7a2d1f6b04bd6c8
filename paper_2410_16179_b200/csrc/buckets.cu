// buckets.cu -- the paper's hash tables HT as inverted lists:
// for every (sequence, kv head) unit and table t, the keys sorted by their K-bit
// code, so that Query(HT, q_code) (Alg. 1) reads only the L buckets
// the query falls into ("negligible computationally", P:446-456
// table sizes) instead of streaming every key's codes.
//
//   bucket_build_kernel  CTA per (unit, table): codes of the table from the bit
//                        planes -> shared-memory histogram over 2^K buckets ->
//                        exclusive scan -> offsets; scatter of key ids (shared-memory atomics:
//                        a bucket's ids are deterministic as a set, not in order; S is a
//                        bitmap, so the Query result does not depend on the order).
//   bucket_mark_kernel   CTA per (unit, query head): for each table the ids of
//                        the query's bucket -> two shared-memory bitmaps
//                        (seen >= 1, seen >= 2; a key is in exactly one bucket
//                        per table, so "seen twice" = matched in >= 2 tables,
//                        the P:84 rule) -> S bitmap in global memory, consumed
//                        by the decode kernel in place of the code scan.
// S is the same set as the dense scan computes (oracle pin P10 proves the two
// forms equal in the oracle; the GPU parity tests check both against it).
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace mp {
namespace cgr = cooperative_groups;

constexpr int BK_THREADS = 512;
constexpr int BM_THREADS = 512;

// key ids are stored as 16-bit words when every local index fits (n_local <= 65536: the paper's int16
// table entries), else as int32.  Per unit: L*(2^K+1) int32 offsets, then the L*n_local ids.
__host__ __device__ __forceinline__ bool ids16(int64_t n_local) { return n_local <= 65536; }
__host__ __device__ __forceinline__ size_t unit_words(int L, int nb, int64_t n_local) {
    const size_t ne = (size_t)L * (size_t)n_local;
    return (size_t)L * ((size_t)nb + 1) + (ids16(n_local) ? (ne + 1) / 2 : ne);
}
// id number idx of a unit's id array (ids0 = the unit's first id word)
__device__ __forceinline__ int load_id(const int32_t* __restrict__ ids0, size_t idx, bool narrow) {
    return narrow ? (int)__ldg(reinterpret_cast<const unsigned short*>(ids0) + idx) : __ldg(ids0 + idx);
}

// code of table t for the 32 keys of block blk (bit r of word b = column t*K+b of key 32*blk+r)
__device__ __forceinline__ void table_words(const uint32_t* __restrict__ cu, int KLq, int K, int t, int64_t blk,
                                            uint32_t (&w)[16]) {
    const int64_t chunk = blk >> 5, l = blk & 31;
#pragma unroll
    for (int b = 0; b < 16; b++) {
        if (b < K) {
            const int col = t * K + b;
            w[b] = __ldg(cu + ((chunk * KLq + (col >> 2)) * 32 + l) * 4 + (col & 3));
        }
    }
}
__device__ __forceinline__ uint32_t key_code(const uint32_t (&w)[16], int K, int r) {
    uint32_t c = 0;
#pragma unroll
    for (int b = 0; b < 16; b++)
        if (b < K) c |= ((w[b] >> r) & 1u) << b;
    return c;
}

// block-wide exclusive scan of hist[0..nb) in place; returns the total (all threads)
__device__ int block_exclusive_scan(int* hist, int nb, int* warp_tot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
    const int per = (nb + nt - 1) / nt, b0 = min(nb, tid * per), b1 = min(nb, b0 + per);
    int s = 0;
    for (int b = b0; b < b1; b++) s += hist[b];
    int incl = s;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, m);
        if (lane >= m) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = nt >> 5;
        int v = lane < nw ? warp_tot[lane] : 0, iv = v;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, iv, m);
            if (lane >= m) iv += u;
        }
        if (lane < nw) warp_tot[lane] = iv - v;
        if (lane == 31) warp_tot[32] = iv;
    }
    __syncthreads();
    int run = warp_tot[warp] + incl - s;
    for (int b = b0; b < b1; b++) {
        const int h = hist[b];
        hist[b] = run;
        run += h;
    }
    const int total = warp_tot[32];
    __syncthreads();
    return total;
}

// grid (L, units); dynamic smem = 2^K ints
__global__ void __launch_bounds__(BK_THREADS) bucket_build_kernel(const uint32_t* __restrict__ codes, int64_t n_local,
                                                                   int K, int L, int KLq, int64_t nchunks,
                                                                   int32_t* __restrict__ tables) {
    extern __shared__ int hist[];
    __shared__ int warp_tot[33];
    const int t = blockIdx.x;
    const int64_t u = blockIdx.y;
    const int nb = 1 << K;
    const uint32_t* cu = codes + (size_t)u * nchunks * KLq * 128;
    int32_t* tu = tables + (size_t)u * unit_words(L, nb, n_local);
    int32_t* offs = tu + (size_t)t * (nb + 1);
    const bool narrow = ids16(n_local);
    int32_t* ids = tu + (size_t)L * (nb + 1) + (narrow ? 0 : (size_t)t * n_local);
    uint16_t* ids_h = reinterpret_cast<uint16_t*>(tu + (size_t)L * (nb + 1)) + (size_t)t * n_local;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const int64_t nblk = (n_local + 31) >> 5;
    for (int64_t blk = threadIdx.x; blk < nblk; blk += blockDim.x) {
        uint32_t w[16];
        table_words(cu, KLq, K, t, blk, w);
        const int nr = (int)min((int64_t)32, n_local - blk * 32);
        for (int r = 0; r < nr; r++) atomicAdd(&hist[key_code(w, K, r)], 1);
    }
    __syncthreads();
    const int total = block_exclusive_scan(hist, nb, warp_tot);
    for (int b = threadIdx.x; b < nb; b += blockDim.x) offs[b] = hist[b];
    if (threadIdx.x == 0) offs[nb] = total;
    __syncthreads();
    for (int64_t blk = threadIdx.x; blk < nblk; blk += blockDim.x) {
        uint32_t w[16];
        table_words(cu, KLq, K, t, blk, w);
        const int nr = (int)min((int64_t)32, n_local - blk * 32);
        for (int r = 0; r < nr; r++) {
            const int pos = atomicAdd(&hist[key_code(w, K, r)], 1);
            if (narrow) ids_h[pos] = (uint16_t)(blk * 32 + r);
            else ids[pos] = (int32_t)(blk * 32 + r);
        }
    }
}

// grid (Hq, B); dynamic smem = 2 * nw words + 2 * L + 1 ints.  qbits [B][Hq][KLw] (bit j = column j of q_g).
// Latency structure: one round for every table's bucket range (thread per table), a block scan of the
// bucket sizes, then the ids of all L buckets as one flattened array split over the CTA in runs of BM_RUN
// consecutive entries per thread (one binary search per run, then a forward walk over the tables), all
// loads of a run in flight before the shared-memory atomics.  Bucket sizes are very skewed (the query's
// bucket can hold thousands of keys), so the split is over entries, not over tables.
constexpr int BM_RUN = 8;
// parts > 1 (grid.z = parts): CTA z handles the z-th slice of the head's flattened ids and writes its own
// (seen once, seen twice) bitmaps, sbits[B][Hq][parts][2][nw]; the select step combines the parts with the
// same saturating counter (P:84 rule).  Bucket sizes are skewed, so slicing by ids balances the CTAs.
__global__ void __launch_bounds__(BM_THREADS) bucket_mark_kernel(const uint32_t* __restrict__ qbits,
                                                                  const int32_t* __restrict__ tables, int64_t Hq,
                                                                  int64_t Hkv, int64_t n_local, int K, int L, int KLw,
                                                                  int minc, uint32_t* __restrict__ sbits) {
    const int parts = gridDim.z, part = blockIdx.z;
    asm volatile("griddepcontrol.launch_dependents;");  // the estimator kernel may start its prologue
    extern __shared__ uint32_t seen[];  // seen1[nw], seen2[nw], lo[L], start[L + 1]
    __shared__ int warp_tot[33];
    const int64_t hq = blockIdx.x, b = blockIdx.y;
    const int64_t G = Hq / Hkv, u = b * Hkv + hq / G;
    const int nb = 1 << K;
    const int64_t nw = (n_local + 31) >> 5;
    uint32_t* seen1 = seen;
    uint32_t* seen2 = seen + nw;
    int* lo_s = reinterpret_cast<int*>(seen + 2 * nw);
    int* start = lo_s + L;
    const int tid = threadIdx.x;
    const int32_t* tu = tables + (size_t)u * unit_words(L, nb, n_local);
    const bool narrow = ids16(n_local);
    for (int64_t w = tid; w < 2 * nw; w += blockDim.x) seen[w] = 0u;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // query codes of the encode kernel
    const uint32_t* qb = qbits + (b * Hq + hq) * KLw;
    for (int t = tid; t < L; t += blockDim.x) {
        // query code of table t: columns t*K .. t*K+K-1 (little endian, R7)
        const int c0 = t * K;
        const uint64_t two = (uint64_t)__ldcg(qb + (c0 >> 5)) |
                             ((c0 >> 5) + 1 < KLw ? (uint64_t)__ldcg(qb + (c0 >> 5) + 1) << 32 : 0ull);
        const int qc = (int)((two >> (c0 & 31)) & (uint64_t)(nb - 1));
        const int32_t* offs = tu + (size_t)t * (nb + 1);
        const int lo = __ldg(offs + qc), hi = __ldg(offs + qc + 1);
        lo_s[t] = lo;
        start[t] = hi - lo;
    }
    __syncthreads();
    const int total = block_exclusive_scan(start, L, warp_tot);  // start[t] = first flat index of table t
    if (tid == 0) start[L] = total;
    __syncthreads();
    const int32_t* ids0 = tu + (size_t)L * (nb + 1);
    const int e_beg = (int)((int64_t)total * part / parts), e_end = (int)((int64_t)total * (part + 1) / parts);
    for (int e0 = e_beg + tid * BM_RUN; e0 < e_end; e0 += blockDim.x * BM_RUN) {
        int lo = 0, hi = L;  // table of flat index e0: last t with start[t] <= e0
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (start[mid] <= e0) lo = mid;
            else hi = mid;
        }
        int t = lo, tnext = start[t + 1];
        int ids[BM_RUN];
#pragma unroll
        for (int j = 0; j < BM_RUN; j++) {
            const int e = e0 + j;
            ids[j] = -1;
            if (e < e_end) {
                while (e >= tnext) tnext = start[++t + 1];
                ids[j] = load_id(ids0, (size_t)t * n_local + lo_s[t] + (e - start[t]), narrow);
            }
        }
#pragma unroll
        for (int j = 0; j < BM_RUN; j++) {
            if (ids[j] >= 0) {
                const int i = ids[j];
                const uint32_t bit = 1u << (i & 31);
                const uint32_t old = atomicOr(&seen1[i >> 5], bit);
                if (minc > 1 && (old & bit)) atomicOr(&seen2[i >> 5], bit);
            }
        }
    }
    __syncthreads();
    if (parts == 1) {
        const uint32_t* src = minc > 1 ? seen2 : seen1;
        uint32_t* dst = sbits + (b * Hq + hq) * nw;
        for (int64_t w = tid; w < nw; w += blockDim.x) dst[w] = src[w];
    } else {
        uint32_t* dst = sbits + ((b * Hq + hq) * parts + part) * 2 * nw;
        for (int64_t w = tid; w < 2 * nw; w += blockDim.x) dst[w] = seen[w];
    }
}

// v2 (parts == 1): the same S, with the L bucket ranges cut into 32-id chunks (prefix over the chunk counts)
// and the chunks dealt to the warps, BM2_UNROLL chunks per warp in flight: one coalesced 128-B load per
// chunk, the chunk's table found once per round (binary search, then a forward walk), no per-id address
// search.  1024 threads per CTA: the heaviest query head (about twice the mean, C3) sets the kernel time.
constexpr int BM2_THREADS = 1024;
constexpr int BM2_UNROLL = 4;
__global__ void __launch_bounds__(BM2_THREADS) bucket_mark2_kernel(const uint32_t* __restrict__ qbits,
                                                                    const int32_t* __restrict__ tables, int64_t Hq,
                                                                    int64_t Hkv, int64_t n_local, int K, int L,
                                                                    int KLw, int minc, uint32_t* __restrict__ sbits) {
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ uint32_t seen[];  // seen1[nw], seen2[nw], lo[L], len[L], cstart[L + 1]
    __shared__ int warp_tot[33];
    const int64_t hq = blockIdx.x, b = blockIdx.y;
    const int64_t G = Hq / Hkv, u = b * Hkv + hq / G;
    const int nb = 1 << K;
    const int nw = (int)((n_local + 31) >> 5);
    uint32_t* seen1 = seen;
    uint32_t* seen2 = seen + nw;
    int* lo_s = reinterpret_cast<int*>(seen + 2 * nw);
    int* len_s = lo_s + L;
    int* cstart = len_s + L;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t* tu = tables + (size_t)u * unit_words(L, nb, n_local);
    const bool narrow = ids16(n_local);
    for (int w = tid; w < 2 * nw; w += BM2_THREADS) seen[w] = 0u;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // query codes of the encode kernel
    const uint32_t* qb = qbits + (b * Hq + hq) * KLw;
    for (int t = tid; t < L; t += BM2_THREADS) {
        const int c0 = t * K;  // query code of table t: columns t*K .. t*K+K-1 (little endian, R7)
        const uint64_t two = (uint64_t)__ldcg(qb + (c0 >> 5)) |
                             ((c0 >> 5) + 1 < KLw ? (uint64_t)__ldcg(qb + (c0 >> 5) + 1) << 32 : 0ull);
        const int qc = (int)((two >> (c0 & 31)) & (uint64_t)(nb - 1));
        const int32_t* offs = tu + (size_t)t * (nb + 1);
        const int lo = __ldg(offs + qc), hi = __ldg(offs + qc + 1);
        lo_s[t] = lo;
        len_s[t] = hi - lo;
        cstart[t] = (hi - lo + 31) >> 5;
    }
    __syncthreads();
    const int C = block_exclusive_scan(cstart, L, warp_tot);  // cstart[t] = first chunk of table t
    if (tid == 0) cstart[L] = C;
    __syncthreads();
    const int32_t* ids0 = tu + (size_t)L * (nb + 1);
    constexpr int NWP = BM2_THREADS / 32;
    for (int c0 = warp * BM2_UNROLL; c0 < C; c0 += NWP * BM2_UNROLL) {
        int lo = 0, hi = L;  // table of chunk c0: last t with cstart[t] <= c0 (warp-uniform)
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (cstart[mid] <= c0) lo = mid;
            else hi = mid;
        }
        int t = lo;
        int ids[BM2_UNROLL];
#pragma unroll
        for (int j = 0; j < BM2_UNROLL; j++) {
            const int c = c0 + j;
            ids[j] = -1;
            if (c < C) {
                while (c >= cstart[t + 1]) t++;
                const int off = ((c - cstart[t]) << 5) + lane;
                if (off < len_s[t]) ids[j] = load_id(ids0, (size_t)t * n_local + lo_s[t] + off, narrow);
            }
        }
#pragma unroll
        for (int j = 0; j < BM2_UNROLL; j++) {
            if (ids[j] >= 0) {
                const int i = ids[j];
                const uint32_t bit = 1u << (i & 31);
                const uint32_t old = atomicOr(&seen1[i >> 5], bit);
                if (minc > 1 && (old & bit)) atomicOr(&seen2[i >> 5], bit);
            }
        }
    }
    __syncthreads();
    const uint32_t* src = minc > 1 ? seen2 : seen1;
    uint32_t* dst = sbits + (b * Hq + hq) * nw;
    for (int w = tid; w < nw; w += BM2_THREADS) dst[w] = src[w];
}

// v3 (parts == 1, the default): a cluster of BM3_CS CTAs per (sequence, query head).  The head's bucket ranges
// are cut into 32-id chunks; CTA r of the cluster takes the r-th contiguous share of the chunks, warp w of the
// CTA the w-th contiguous share of that (one binary search per warp, then a forward walk over the tables),
// BM3_UNROLL chunks (one coalesced 128-B load each) in flight per warp.  Each CTA marks its own seen-once /
// seen-twice bitmaps; after a cluster barrier CTA 0 combines them through distributed shared memory with the
// same saturating counter, (a1, a2) + (b1, b2) = (a1 | b1, a2 | b2 | (a1 & b1)), and writes S.  Splitting a
// head over two SMs halves the heaviest head's time (the C3 heads' id counts are skewed: max ~1.9x the mean).
#ifndef MP_BM3_THREADS
#define MP_BM3_THREADS 512
#endif
#ifndef MP_BM3_UNROLL
#define MP_BM3_UNROLL 4
#endif
constexpr int BM3_THREADS = MP_BM3_THREADS;
constexpr int BM3_UNROLL = MP_BM3_UNROLL;
#ifndef MP_BM3_CS
#define MP_BM3_CS 2
#endif
constexpr int BM3_CS = MP_BM3_CS;
template <bool NARROW>  // NARROW: 16-bit ids (n_local <= 65536), a compile-time load width
__global__ void __launch_bounds__(BM3_THREADS) bucket_mark3_kernel(const uint32_t* __restrict__ qbits,
                                                                    const int32_t* __restrict__ tables, int64_t Hq,
                                                                    int64_t Hkv, int64_t n_local, int K, int L,
                                                                    int KLw, int minc, uint32_t* __restrict__ sbits) {
    #ifndef MP_BM3_LD_END
#define MP_BM3_LD_END 1
#endif
    if (!MP_BM3_LD_END) asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ uint32_t seen[];  // seen1[nw], seen2[nw], base[L], len[L], cstart[L + 1]
    __shared__ int warp_tot[33];
    cgr::cluster_group cluster = cgr::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int64_t hq = blockIdx.x / BM3_CS, b = blockIdx.y;
    const int64_t G = Hq / Hkv, u = b * Hkv + hq / G;
    const int nb = 1 << K;
    const int nw = (int)((n_local + 31) >> 5);
    uint32_t* seen1 = seen;
    uint32_t* seen2 = seen + nw;
    int* base_s = reinterpret_cast<int*>(seen + 2 * nw);
    int* len_s = base_s + L;
    int* cstart = len_s + L;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t* tu = tables + (size_t)u * unit_words(L, nb, n_local);
    constexpr bool narrow = NARROW;
#ifndef MP_BM3_PAIR
#define MP_BM3_PAIR 0
#endif
    // 16-bit ids two per lane per load: parity-green but measured slower at C3 (Query 16.97 vs 15.77 us), off
    constexpr bool PAIR = NARROW && MP_BM3_PAIR;
    for (int w = tid; w < 2 * nw; w += BM3_THREADS) seen[w] = 0u;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // query codes of the encode kernel
    const uint32_t* qb = qbits + (b * Hq + hq) * KLw;
    for (int t = tid; t < L; t += BM3_THREADS) {
        const int c0 = t * K;  // query code of table t: columns t*K .. t*K+K-1 (little endian, R7)
        const uint64_t two = (uint64_t)__ldcg(qb + (c0 >> 5)) |
                             ((c0 >> 5) + 1 < KLw ? (uint64_t)__ldcg(qb + (c0 >> 5) + 1) << 32 : 0ull);
        const int qc = (int)((two >> (c0 & 31)) & (uint64_t)(nb - 1));
        const int32_t* offs = tu + (size_t)t * (nb + 1);
        const int lo = __ldg(offs + qc), hi = __ldg(offs + qc + 1);
        base_s[t] = (int)((int64_t)t * n_local + lo);  // < L * n_local (checked on the host)
        len_s[t] = hi - lo;
        // PAIR: 64-id chunks of aligned 32-bit id pairs (the range widened to an even start)
        cstart[t] = PAIR ? (hi > lo ? (hi - lo + (base_s[t] & 1) + 63) >> 6 : 0) : (hi - lo + 31) >> 5;
    }
    __syncthreads();
    const int C = block_exclusive_scan(cstart, L, warp_tot);  // cstart[t] = first chunk of table t
    if (tid == 0) cstart[L] = C;
    __syncthreads();
    const int32_t* ids0 = tu + (size_t)L * (nb + 1);
    constexpr int NWP = BM3_THREADS / 32;
    const int cr0 = (int)((int64_t)C * rank / BM3_CS), cr1 = (int)((int64_t)C * (rank + 1) / BM3_CS);
    const int cw0 = cr0 + (int)((int64_t)(cr1 - cr0) * warp / NWP);
    const int cw1 = cr0 + (int)((int64_t)(cr1 - cr0) * (warp + 1) / NWP);
    int t = 0;
    if (cw0 < cw1) {  // table of chunk cw0: last t with cstart[t] <= cw0
        int lo = 0, hi = L;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (cstart[mid] <= cw0) lo = mid;
            else hi = mid;
        }
        t = lo;
    }
    for (int c0 = cw0; c0 < cw1; c0 += BM3_UNROLL) {
        int ids[BM3_UNROLL][PAIR ? 2 : 1];
#pragma unroll
        for (int j = 0; j < BM3_UNROLL; j++) {
            const int c = c0 + j;
#pragma unroll
            for (int h = 0; h < (PAIR ? 2 : 1); h++) ids[j][h] = -1;
            if (c < cw1) {
                while (c >= cstart[t + 1]) t++;
                if constexpr (PAIR) {
                    // id elements e, e + 1 of the unit's array in one aligned 32-bit load (little endian)
                    const int b = base_s[t], end = b + len_s[t];
                    const int e = (b & ~1) + ((c - cstart[t]) << 6) + 2 * lane;
                    if (e + 1 >= b && e < end) {
                        const uint32_t w =
                            __ldg(reinterpret_cast<const unsigned int*>(reinterpret_cast<const uint16_t*>(ids0) + e));
                        if (e >= b) ids[j][0] = (int)(w & 0xffffu);
                        if (e + 1 < end) ids[j][1] = (int)(w >> 16);
                    }
                } else {
                    const int off = ((c - cstart[t]) << 5) + lane;
                    if (off < len_s[t]) ids[j][0] = load_id(ids0, (size_t)base_s[t] + off, narrow);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < BM3_UNROLL; j++) {
#pragma unroll
            for (int h = 0; h < (PAIR ? 2 : 1); h++) {
                if (ids[j][h] >= 0) {
                    const int i = ids[j][h];
                    const uint32_t bit = 1u << (i & 31);
                    const uint32_t old = atomicOr(&seen1[i >> 5], bit);
                    if (minc > 1 && (old & bit)) atomicOr(&seen2[i >> 5], bit);
                }
            }
        }
    }
    cluster.sync();  // every CTA's bitmaps complete
    if (rank == 0) {
        uint32_t* dst = sbits + (b * Hq + hq) * nw;
        for (int w = tid; w < nw; w += BM3_THREADS) {
            uint32_t f1 = seen1[w], f2 = seen2[w];
#pragma unroll
            for (int r = 1; r < BM3_CS; r++) {
                const uint32_t* rs = cluster.map_shared_rank(seen, r);
                const uint32_t b1 = rs[w], b2 = rs[nw + w];
                f2 |= b2 | (f1 & b1);
                f1 |= b1;
            }
            dst[w] = minc > 1 ? f2 : f1;
        }
    }
    cluster.sync();  // the other CTAs' shared memory stays alive until CTA 0 has read it
    if (MP_BM3_LD_END) asm volatile("griddepcontrol.launch_dependents;");
}

size_t bucket_tables_words(int K, int L, int64_t units, int64_t n_local) {
    return (size_t)units * unit_words(L, 1 << K, n_local);
}

int launch_bucket_build(const uint32_t* codes, int64_t units, int64_t n_local, int K, int L, int KLq,
                        int64_t nchunks, int32_t* tables, cudaStream_t st) {
    if (units < 1 || n_local < 1) return 0;
    const size_t smem = ((size_t)1 << K) * 4;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(bucket_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return MAGICPIG_ECUDA;
    bucket_build_kernel<<<dim3((unsigned)L, (unsigned)units), BK_THREADS, smem, st>>>(codes, n_local, K, L, KLq,
                                                                                     nchunks, tables);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

#ifndef MP_BM2
#define MP_BM2 3
#endif
int launch_bucket_mark(const uint32_t* qbits, const int32_t* tables, int64_t B, int64_t Hq, int64_t Hkv,
                       int64_t n_local, int K, int L, int KLw, int minc, uint32_t* sbits, cudaStream_t st, int parts) {
    if (MP_BM2 == 3 && parts == 1 && (int64_t)L * n_local < (1ll << 31)) {
        const size_t smem3 = (size_t)((n_local + 31) >> 5) * 8 + (size_t)(3 * L + 1) * 4;
        if (smem3 <= 208 * 1024) {
            auto kern = ids16(n_local) ? bucket_mark3_kernel<true> : bucket_mark3_kernel<false>;
            if (smem3 > 48 * 1024 &&
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3) != cudaSuccess)
                return MAGICPIG_ECUDA;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(Hq * BM3_CS), (unsigned)B, 1u);
            cfg.blockDim = dim3(BM3_THREADS);
            cfg.dynamicSmemBytes = smem3;
            cfg.stream = st;
            cudaLaunchAttribute attr[2];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            attr[1].id = cudaLaunchAttributeClusterDimension;
            attr[1].val.clusterDim.x = BM3_CS;
            attr[1].val.clusterDim.y = 1;
            attr[1].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 2;
            cudaError_t e = cudaLaunchKernelEx(&cfg, kern, qbits, tables, Hq, Hkv, n_local, K, L, KLw,
                                               minc, sbits);
            count_launch(1);
            return e == cudaSuccess ? 0 : MAGICPIG_ECUDA;
        }
    }
    if (MP_BM2 == 2 && parts == 1) {
        const size_t smem2 = (size_t)((n_local + 31) >> 5) * 8 + (size_t)(3 * L + 1) * 4;
        if (smem2 <= 208 * 1024) {
            if (smem2 > 48 * 1024 && cudaFuncSetAttribute(bucket_mark2_kernel,
                                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                          (int)smem2) != cudaSuccess)
                return MAGICPIG_ECUDA;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)Hq, (unsigned)B, 1u);
            cfg.blockDim = dim3(BM2_THREADS);
            cfg.dynamicSmemBytes = smem2;
            cfg.stream = st;
            cudaLaunchAttribute attr;
            attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr.val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = &attr;
            cfg.numAttrs = 1;
            cudaError_t e = cudaLaunchKernelEx(&cfg, bucket_mark2_kernel, qbits, tables, Hq, Hkv, n_local, K, L, KLw,
                                               minc, sbits);
            count_launch(1);
            return e == cudaSuccess ? 0 : MAGICPIG_ECUDA;
        }
    }
    const size_t smem = (size_t)((n_local + 31) >> 5) * 8 + (size_t)(2 * L + 1) * 4;
    if (smem > 208 * 1024) return MAGICPIG_EINVAL;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(bucket_mark_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return MAGICPIG_ECUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)Hq, (unsigned)B, (unsigned)parts);
    cfg.blockDim = dim3(BM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, bucket_mark_kernel, qbits, tables, Hq, Hkv, n_local, K, L, KLw, minc,
                                       sbits);
    count_launch(1);
    return e == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

}  // namespace mp
