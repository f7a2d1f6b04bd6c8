// pieces.cuh -- device helpers shared by the Query kernels that emit the v7 piece lists (scan6.cu) and the
// select / estimator kernels (estimate.cu): the dynamic-key mask D (P:171, P:619 static cache excluded),
// and the ordered union list of one piece = (unit, 1024-key chunk).
#pragma once
#include "common.cuh"
#include "kernels.cuh"

namespace mp {
namespace v7 {

__device__ __forceinline__ uint32_t range_mask(int64_t base, int64_t lo, int64_t hi) {
    int64_t x = lo - base, y = hi - base;
    x = x < 0 ? 0 : (x > 32 ? 32 : x);
    y = y < 0 ? 0 : (y > 32 ? 32 : y);
    if (y <= x) return 0u;
    const uint32_t hiMask = y >= 32 ? 0xffffffffu : ((1u << y) - 1u);
    const uint32_t loMask = x >= 32 ? 0xffffffffu : ((1u << x) - 1u);
    return hiMask & ~loMask;
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}
__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, v, m);
        if (lane >= m) v += x;
    }
    return v;
}

// static keys T on this shard (sink tokens at global [0, sink), local window at [n - local, n)),
// as local index ranges [lo1, lo1 + len1) u [lo2, lo2 + len2)
struct StaticRanges {
    int64_t lo1, len1, lo2, len2;
};
__device__ __forceinline__ StaticRanges static_ranges(const EstArgs& a) {
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

// S_g words of one piece (lane = 32-key word) -> D mask, |S_g| of the piece, the ordered union list
template <int G>
__device__ __forceinline__ void emit_piece(const EstArgs& a, const StaticRanges& sr, int64_t u, int64_t c,
                                           int64_t qh0, int lane, uint32_t (&sg)[G]) {
    const int64_t nwb = (a.n_local + 31) >> 5;
    const int64_t wi = c * 32 + lane, base = wi * 32;
    const uint32_t dmask = range_mask(base, 0, a.n_local) &
                           ~(range_mask(base, sr.lo1, sr.lo1 + sr.len1) | range_mask(base, sr.lo2, sr.lo2 + sr.len2));
    uint32_t un = 0u;
#pragma unroll
    for (int g = 0; g < G; g++) {
        sg[g] &= dmask;
        un |= sg[g];
        int h = __popc(sg[g]);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) h += __shfl_xor_sync(0xffffffffu, h, m);
        if (lane == 0) a.hpc[(qh0 + g) * a.nchunks + c] = h;
        if (a.s_mask && wi < nwb) a.s_mask[(qh0 + g) * nwb + wi] = sg[g];
    }
    const int cnt = __popc(un);
    const int incl = warp_incl_scan(cnt, lane);
    uint32_t* list = a.ents + (u * a.nchunks + c) * KCHUNK;
    int pos = incl - cnt;
    while (un) {
        const int bit = __ffs(un) - 1;
        un &= un - 1u;
        uint32_t hb = 0u;
#pragma unroll
        for (int g = 0; g < G; g++) hb |= ((sg[g] >> bit) & 1u) << g;
        list[pos++] = (uint32_t)(base + bit) | (hb << 24);
    }
    if (lane == 31) a.pcnt[u * a.nchunks + c] = incl;
}


}  // namespace v7
}  // namespace mp
