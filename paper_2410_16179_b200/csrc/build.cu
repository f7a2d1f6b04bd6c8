// build.cu -- key statistics, centering, MIPS transform and operand
// preparation for the hash GEMM (PAPER.md:124-127 centering, P:49-55 MIPS).
//
// All bandwidth-bound (one pass over K per phase): 128-bit loads of key rows,
// exact integer (fixed-point 2^-64) accumulation so that every reduction is
// order-independent and bit-reproducible (reading R2b).
#include "common.cuh"
#include "kernels.cuh"

namespace mp {

constexpr float ABS_LIMIT = 134217728.0f;  // 2^27

// is global position `pos` static (sink / local window)? (R12)
__device__ __forceinline__ bool is_static_pos(int64_t pos, int64_t n_global, int sink, int local) {
    return pos < (int64_t)sink || pos >= n_global - (int64_t)local;
}

// q64 accumulation of bf16 values in two int64 words, total = hi * 2^40 + lo: the same integers as summing
// q64_of_bf16 (value * 2^64 = M * 2^s, s = e - 70, truncated toward zero for s < 0), without 128-bit shifts.
// |k| < 2^27 gives s <= 83, so a term is < 2^52 in hi (s >= 40) or < 2^48 in lo; a lane adds at most
// STATS_SPLIT / 8 = 128 terms per split, so neither word can overflow.
__device__ __forceinline__ void q64_acc_bf16(long long& hi, long long& lo, uint16_t h) {
    const int E = (h >> 7) & 0xFF;
    const long long M = (long long)((h & 0x7Fu) | (E ? 0x80u : 0u));
    const int s = (E ? E : 1) - 70;
    long long vhi = 0, vlo = 0;
    if (s >= 40) vhi = M << (s - 40);
    else if (s >= 0) vlo = M << s;
    else if (s > -8) vlo = M >> (-s);
    if (h & 0x8000u) vhi = -vhi, vlo = -vlo;
    hi += vhi;
    lo += vlo;
}

// ---------------------------------------------------------------------------
// Phase 1: per (unit, split, dim) partial sums of q64(k) over dynamic keys.
// grid (nsplit, units), block 256: warp per key (stride 8), lane = 4 dims,
// per-lane int128 accumulators; warps combined through shared memory.
__global__ void __launch_bounds__(256) key_stats_partial_kernel(
    const uint16_t* __restrict__ k, int64_t n_local, int64_t seq_offset, int64_t n_global, int sink,
    int local, int64_t* __restrict__ part_sum, int64_t* __restrict__ part_cnt, uint32_t* status) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t unit = blockIdx.y;
    const int split = blockIdx.x, nsplit = gridDim.x;
    const int64_t i0 = (int64_t)split * STATS_SPLIT;
    const int64_t i1 = min(i0 + (int64_t)STATS_SPLIT, n_local);
    const uint16_t* kp = k + unit * n_local * HD;
    long long ahi[4] = {0, 0, 0, 0}, alo[4] = {0, 0, 0, 0};
    int cnt = 0;
    bool bad = false;
    constexpr int UN = 4;  // keys in flight per warp (all loads issued before the accumulation)
    for (int64_t i = i0 + warp; i < i1; i += 8 * UN) {
        uint2 kr[UN];
        bool ok[UN];
#pragma unroll
        for (int u = 0; u < UN; u++) {
            const int64_t ii = i + 8 * u;
            ok[u] = ii < i1 && !is_static_pos(seq_offset + ii, n_global, sink, local);
            kr[u] = ok[u] ? __ldg(reinterpret_cast<const uint2*>(kp + ii * HD) + lane) : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < UN; u++) {
            if (!ok[u]) continue;
            const uint16_t h[4] = {(uint16_t)(kr[u].x & 0xFFFF), (uint16_t)(kr[u].x >> 16),
                                   (uint16_t)(kr[u].y & 0xFFFF), (uint16_t)(kr[u].y >> 16)};
#pragma unroll
            for (int t = 0; t < 4; t++) {
                bad |= fabsf(bf2f(h[t])) >= ABS_LIMIT;
                q64_acc_bf16(ahi[t], alo[t], h[t]);
            }
            cnt++;
        }
    }
    if (bad) atomicOr(status, MAGICPIG_STATUS_INEXACT);
    __shared__ unsigned long long sm[8][HD][2];
    __shared__ int scnt[8];
#pragma unroll
    for (int t = 0; t < 4; t++) {
        const u128 u = (u128)(((i128)ahi[t] << 40) + (i128)alo[t]);
        sm[warp][lane * 4 + t][0] = (unsigned long long)u;
        sm[warp][lane * 4 + t][1] = (unsigned long long)(u >> 64);
    }
    if (lane == 0) scnt[warp] = cnt;
    __syncthreads();
    if (threadIdx.x < HD) {
        const int d = threadIdx.x;
        i128 tot = 0;
        for (int w = 0; w < 8; w++) tot += (i128)(((u128)sm[w][d][1] << 64) | (u128)sm[w][d][0]);
        st_q64(part_sum + ((unit * nsplit + split) * HD + d) * 2, tot);
    }
    if (threadIdx.x == 0) {
        int c = 0;
        for (int w = 0; w < 8; w++) c += scnt[w];
        part_cnt[unit * nsplit + split] = c;
    }
}

// Sum of P partial copies: out[u][d] = sum_p part[u][p][d]  (fixed order)
// grid (units), block 128
__global__ void __launch_bounds__(128) sum_parts_kernel(const int64_t* __restrict__ part_sum,
                                                        const int64_t* __restrict__ part_cnt, int nsplit,
                                                        int64_t* __restrict__ key_sum,
                                                        int64_t* __restrict__ count) {
    const int d = threadIdx.x;
    const int64_t unit = blockIdx.x;
    i128 acc = 0;
    int64_t c = 0;
    for (int p = 0; p < nsplit; p++) {
        acc += ld_q64(part_sum + ((unit * nsplit + p) * HD + d) * 2);
        c += part_cnt[unit * nsplit + p];
    }
    st_q64(key_sum + (unit * HD + d) * 2, acc);
    if (d == 0) count[unit] = c;
}

// Shard reduction (after an all-gather): mode 0 sum of key sums and counts,
// mode 1 max of r2.  grid (ceil(units*128/256)), block 256.
__global__ void reduce_shards_kernel(int mode, const int64_t* __restrict__ parts_sum,
                                     const int64_t* __restrict__ parts_cnt, int P, int64_t units,
                                     int64_t* __restrict__ out_sum, int64_t* __restrict__ out_cnt) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (mode == 0) {
        int64_t nel = units * HD;
        if (idx < nel) {
            i128 acc = 0;
            for (int p = 0; p < P; p++) acc += ld_q64(parts_sum + ((int64_t)p * nel + idx) * 2);
            st_q64(out_sum + idx * 2, acc);
        }
        if (idx < units) {
            int64_t c = 0;
            for (int p = 0; p < P; p++) c += parts_cnt[(int64_t)p * units + idx];
            out_cnt[idx] = c;
        }
    } else {
        if (idx < units) {
            i128 m = 0;
            for (int p = 0; p < P; p++) {
                i128 v = ld_q64(parts_sum + ((int64_t)p * units + idx) * 2);
                m = v > m ? v : m;
            }
            st_q64(out_sum + idx * 2, m);
        }
    }
}

// ---------------------------------------------------------------------------
// Phase 2a: centering vector c = fl32(fl64(fl64(sum 2^-64) / count)).
// grid (units), block 128
__global__ void __launch_bounds__(128) center_kernel(const int64_t* __restrict__ key_sum,
                                                     const int64_t* __restrict__ count, int do_center,
                                                     float* __restrict__ center) {
    const int d = threadIdx.x;
    const int64_t unit = blockIdx.x;
    float c = 0.0f;
    int64_t n = count[unit];
    if (do_center && n > 0) {
        double s = q64_to_double(ld_q64(key_sum + (unit * HD + d) * 2));
        c = (float)(s / (double)n);
    }
    center[unit * HD + d] = c;
}

// x = bf16(fl32(k - c)) for the 4 dims of this lane; returns q64 sum of x^2
__device__ __forceinline__ u128 transform4(uint2 kraw, float4 c, uint32_t& x01, uint32_t& x23,
                                           bool& bad) {
    float k0 = __uint_as_float(kraw.x << 16), k1 = __uint_as_float(kraw.x & 0xFFFF0000u);
    float k2 = __uint_as_float(kraw.y << 16), k3 = __uint_as_float(kraw.y & 0xFFFF0000u);
    uint16_t b0 = f2bf_rn(__fsub_rn(k0, c.x)), b1 = f2bf_rn(__fsub_rn(k1, c.y));
    uint16_t b2 = f2bf_rn(__fsub_rn(k2, c.z)), b3 = f2bf_rn(__fsub_rn(k3, c.w));
    float f0 = bf2f(b0), f1 = bf2f(b1), f2 = bf2f(b2), f3 = bf2f(b3);
    bad |= fabsf(f0) >= ABS_LIMIT || fabsf(f1) >= ABS_LIMIT || fabsf(f2) >= ABS_LIMIT ||
           fabsf(f3) >= ABS_LIMIT;
    x01 = (uint32_t)b0 | ((uint32_t)b1 << 16);
    x23 = (uint32_t)b2 | ((uint32_t)b3 << 16);
    // squares of bf16 values are exact in fp32 (16 significant bits)
    return q64_of_f32(__fmul_rn(f0, f0)) + q64_of_f32(__fmul_rn(f1, f1)) + q64_of_f32(__fmul_rn(f2, f2)) +
           q64_of_f32(__fmul_rn(f3, f3));
}

__device__ __forceinline__ u128 warp_sum_u128(u128 v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += shfl_xor_u128(v, m);
    return v;
}

// Phase 2b: per (unit, split) partial max of n2q over dynamic keys.
// grid (nsplit, units), block 256 (8 warps; warp per key, lane = 4 dims)
__global__ void __launch_bounds__(256) r2_partial_kernel(const uint16_t* __restrict__ k, int64_t n_local,
                                                         int64_t seq_offset, int64_t n_global, int sink,
                                                         int local, const float* __restrict__ center,
                                                         int64_t* __restrict__ part_r2, uint32_t* status) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t unit = blockIdx.y;
    const int split = blockIdx.x, nsplit = gridDim.x;
    const int64_t i0 = (int64_t)split * STATS_SPLIT;
    const int64_t i1 = min(i0 + (int64_t)STATS_SPLIT, n_local);
    const float4 c = reinterpret_cast<const float4*>(center + unit * HD)[lane];
    const uint16_t* kp = k + unit * n_local * HD;
    u128 best = 0;
    bool bad = false;
    constexpr int UN = 4;  // keys in flight per warp
    for (int64_t i = i0 + warp; i < i1; i += 8 * UN) {
        uint2 kr[UN];
        bool ok[UN];
#pragma unroll
        for (int u = 0; u < UN; u++) {
            const int64_t ii = i + 8 * u;
            ok[u] = ii < i1 && !is_static_pos(seq_offset + ii, n_global, sink, local);
            kr[u] = ok[u] ? __ldg(reinterpret_cast<const uint2*>(kp + ii * HD) + lane) : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < UN; u++) {
            if (!ok[u]) continue;  // warp-uniform
            uint32_t a, b;
            u128 s = warp_sum_u128(transform4(kr[u], c, a, b, bad));
            best = s > best ? s : best;
        }
    }
    if (bad) atomicOr(status, MAGICPIG_STATUS_INEXACT);
    __shared__ unsigned long long sm[8][2];
    if (lane == 0) {
        sm[warp][0] = (unsigned long long)best;
        sm[warp][1] = (unsigned long long)(best >> 64);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u128 m = 0;
        for (int w = 0; w < 8; w++) {
            u128 v = ((u128)sm[w][1] << 64) | (u128)sm[w][0];
            m = v > m ? v : m;
        }
        st_q64(part_r2 + (unit * nsplit + split) * 2, (i128)m);
    }
}

// ---------------------------------------------------------------------------
// Lane-per-key forms of phases 2b and 3a (the same integers as the warp-per-key forms above, without the
// per-key 128-bit warp reductions): a thread reads its key's whole row (16 x 16 B), forms
// x = bf16(fl32(k - c)) element by element, and sums q64(x^2) exactly in three int64 words.
// x = +-m 2^(Ex - 134) (m <= 255 incl. the implicit bit) -> q64(x^2) = trunc(m^2 2^s), s = 2 Ex - 204 (the
// fp32 square of a bf16 value is exact, and q64_of_f32 truncates the same product); |x| < 2^27 gives
// s <= 102.  Words: hi (scale 2^64, s >= 64), mid (2^32, 32 <= s < 64), lo (s < 32); every term is below
// 2^54 and a row adds 128 of them, so no word overflows.
struct N2Acc {
    unsigned long long hi, mid, lo;
};
__device__ __forceinline__ void n2_add(N2Acc& a, uint16_t xb) {
    const int E = (xb >> 7) & 0xFF;
    const unsigned long long m = (xb & 0x7Fu) | (E ? 0x80u : 0u);
    const unsigned long long m2 = m * m;
    const int sx = 2 * (E ? E : 1) - 204;
    if (sx >= 64) a.hi += m2 << (sx - 64);
    else if (sx >= 32) a.mid += m2 << (sx - 32);
    else if (sx >= 0) a.lo += m2 << sx;
    else if (sx > -16) a.lo += m2 >> (-sx);
}
__device__ __forceinline__ u128 n2_total(const N2Acc& a) {
    return ((u128)a.hi << 64) + ((u128)a.mid << 32) + (u128)a.lo;
}
// one key row: x pairs (xw[w] = bf16 pair of dims 2w, 2w+1) and the exact q64 |x|^2; c from shared memory
__device__ __forceinline__ u128 row_xbar(const uint16_t* __restrict__ krow, const float* __restrict__ cs,
                                         uint32_t (&xw)[64], bool& bad) {
    N2Acc acc = {0ull, 0ull, 0ull};
#pragma unroll
    for (int q = 0; q < 16; q++) {
        const uint4 kv = __ldg(reinterpret_cast<const uint4*>(krow) + q);
        const uint32_t kk[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const int d = 8 * q + 2 * t;
            const uint16_t b0 = f2bf_rn(__fsub_rn(__uint_as_float(kk[t] << 16), cs[d]));
            const uint16_t b1 = f2bf_rn(__fsub_rn(__uint_as_float(kk[t] & 0xFFFF0000u), cs[d + 1]));
            bad |= fabsf(bf2f(b0)) >= ABS_LIMIT || fabsf(bf2f(b1)) >= ABS_LIMIT;
            n2_add(acc, b0);
            n2_add(acc, b1);
            xw[4 * q + t] = (uint32_t)b0 | ((uint32_t)b1 << 16);
        }
    }
    return n2_total(acc);
}

// Phase 2b, lane per key: grid (nsplit, units), block 256; thread t of split s takes keys s*1024 + t + 256 j
__global__ void __launch_bounds__(256) r2_partial2_kernel(const uint16_t* __restrict__ k, int64_t n_local,
                                                          int64_t seq_offset, int64_t n_global, int sink,
                                                          int local, const float* __restrict__ center,
                                                          int64_t* __restrict__ part_r2, uint32_t* status) {
    __shared__ float cs[HD];
    __shared__ unsigned long long sm[8][2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t unit = blockIdx.y;
    const int split = blockIdx.x, nsplit = gridDim.x;
    if (tid < HD) cs[tid] = center[unit * HD + tid];
    __syncthreads();
    const int64_t i0 = (int64_t)split * STATS_SPLIT;
    const int64_t i1 = min(i0 + (int64_t)STATS_SPLIT, n_local);
    const uint16_t* kp = k + unit * n_local * HD;
    u128 best = 0;
    bool bad = false;
    for (int64_t i = i0 + tid; i < i1; i += 256) {
        if (is_static_pos(seq_offset + i, n_global, sink, local)) continue;
        uint32_t xw[64];
        const u128 n2 = row_xbar(kp + i * HD, cs, xw, bad);
        best = n2 > best ? n2 : best;
    }
    if (bad) atomicOr(status, MAGICPIG_STATUS_INEXACT);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        const u128 o = shfl_xor_u128(best, m);
        best = o > best ? o : best;
    }
    if (lane == 0) {
        sm[warp][0] = (unsigned long long)best;
        sm[warp][1] = (unsigned long long)(best >> 64);
    }
    __syncthreads();
    if (tid == 0) {
        u128 m = 0;
        for (int w = 0; w < 8; w++) {
            u128 v = ((u128)sm[w][1] << 64) | (u128)sm[w][0];
            m = v > m ? v : m;
        }
        st_q64(part_r2 + (unit * nsplit + split) * 2, (i128)m);
    }
}

// Phase 3a, lane per key: grid (n_pad / 256, units), block 256 (thread = key i = 256 blockIdx.x + t).
// Row r of tile i/128 in the UMMA canonical K-major layout: 16-B chunk kc of row r at
// (kc*16 + r/8)*128 + (r%8)*16 -- 32 consecutive threads write 512 contiguous bytes per chunk.
__global__ void __launch_bounds__(256) prep_x2_kernel(const uint16_t* __restrict__ k, int64_t n_local,
                                                      int64_t n_pad, int mips, int KD,
                                                      const float* __restrict__ center,
                                                      const int64_t* __restrict__ r2, uint8_t* __restrict__ xt,
                                                      float* __restrict__ xnorm, float* __restrict__ key_norm,
                                                      uint32_t* status) {
    __shared__ float cs[HD];
    const int tid = threadIdx.x;
    const int64_t unit = blockIdx.y;
    if (tid < HD) cs[tid] = center[unit * HD + tid];
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * 256 + tid;
    if (i >= n_pad) return;
    const int r = (int)(i & 127);
    uint8_t* tbase = xt + (unit * (n_pad >> 7) + (i >> 7)) * (int64_t)(128 * KD * 2) + (r >> 3) * 128 + (r & 7) * 16;
    uint32_t xw[64];
    bool bad = false;
    u128 n2 = 0;
    if (i < n_local) {
        n2 = row_xbar(k + (unit * n_local + i) * HD, cs, xw, bad);
    } else {
#pragma unroll
        for (int w = 0; w < 64; w++) xw[w] = 0u;
    }
    if (bad) atomicOr(status, MAGICPIG_STATUS_INEXACT);
#pragma unroll
    for (int kc = 0; kc < 16; kc++)
        *reinterpret_cast<uint4*>(tbase + kc * 16 * 128) =
            make_uint4(xw[4 * kc], xw[4 * kc + 1], xw[4 * kc + 2], xw[4 * kc + 3]);
    const double n2d = q64_to_double((i128)n2);
    if (KD > HD) {
        uint16_t sv = 0;
        if (mips && i < n_local) {
            const i128 diff = ld_q64(r2 + unit * 2) - (i128)n2;
            sv = diff > 0 ? d2bf_rn_pos(sqrt(q64_to_double(diff))) : (uint16_t)0;
        }
        for (int kc = 16; kc < KD / 8; kc++)
            *reinterpret_cast<uint4*>(tbase + kc * 16 * 128) = make_uint4(kc == 16 ? (uint32_t)sv : 0u, 0u, 0u, 0u);
        const float sf = bf2f(sv);
        const float nr = (float)sqrt(n2d + (double)sf * (double)sf);
        xnorm[unit * n_pad + i] = i < n_local ? nr : -1.0f;
        if (i < n_local) key_norm[unit * n_local + i] = nr;
    } else {
        const float nr = (float)sqrt(n2d);
        xnorm[unit * n_pad + i] = i < n_local ? nr : -1.0f;
        if (i < n_local) key_norm[unit * n_local + i] = nr;
    }
}

// max over splits -> r2[unit]; grid (ceil(units/128)), block 128
__global__ void max_parts_kernel(const int64_t* __restrict__ part_r2, int nsplit, int64_t units,
                                 int64_t* __restrict__ r2) {
    int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= units) return;
    i128 m = 0;
    for (int p = 0; p < nsplit; p++) {
        i128 v = ld_q64(part_r2 + (u * nsplit + p) * 2);
        m = v > m ? v : m;
    }
    st_q64(r2 + u * 2, m);
}

// ---------------------------------------------------------------------------
// Phase 3a: hashed key vectors xbar_i = [bf16(fl32(k - c)), s_i, 0...] written
// straight into the UMMA canonical K-major no-swizzle layout, one 128-row tile
// per 128*KD*2 bytes: element (r, kk) at ((kk/8)*16 + r/8)*128 + (r%8)*16 + (kk%8)*2.
// Also |xbar_i| (fp32, for the filter threshold; -1 for padding rows).
// grid (ceil(n_pad/(8*PX_KEYS)), units), block 256 (warp per PX_KEYS consecutive keys)
constexpr int PX_KEYS = 8;
__global__ void __launch_bounds__(256) prep_x_kernel(const uint16_t* __restrict__ k, int64_t n_local,
                                                     int64_t n_pad, int mips, int KD,
                                                     const float* __restrict__ center,
                                                     const int64_t* __restrict__ r2,
                                                     uint8_t* __restrict__ xt, float* __restrict__ xnorm,
                                                     float* __restrict__ key_norm, uint32_t* status) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t unit = blockIdx.y;
    const int64_t ib = ((int64_t)blockIdx.x * 8 + warp) * PX_KEYS;  // this warp's PX_KEYS consecutive keys
    if (ib >= n_pad) return;
    const float4 c = reinterpret_cast<const float4*>(center + unit * HD)[lane];
    uint2 kr[PX_KEYS];
#pragma unroll
    for (int u = 0; u < PX_KEYS; u++) {  // every row load in flight before the transforms
        const int64_t i = ib + u;
        kr[u] = i < n_local ? __ldg(reinterpret_cast<const uint2*>(k + (unit * n_local + i) * HD) + lane)
                            : make_uint2(0u, 0u);
    }
    bool bad = false;
    i128 rr = 0;
    if (mips) rr = ld_q64(r2 + unit * 2);
#pragma unroll
    for (int u = 0; u < PX_KEYS; u++) {
        const int64_t i = ib + u;
        if (i >= n_pad) break;
        const int64_t tile = i >> 7;
        const int r = (int)(i & 127);
        uint8_t* tbase = xt + (unit * (n_pad >> 7) + tile) * (int64_t)(128 * KD * 2);
        const int rowoff = (r >> 3) * 128 + (r & 7) * 16;
        uint32_t a = 0, b = 0;
        u128 n2 = 0;
        if (i < n_local) n2 = warp_sum_u128(transform4(kr[u], c, a, b, bad));
        // dims kk = 4*lane .. 4*lane+3: chunk kk/8 = lane/2, offset (lane&1)*8 bytes
        *reinterpret_cast<uint2*>(tbase + (lane >> 1) * 16 * 128 + rowoff + (lane & 1) * 8) = make_uint2(a, b);
        if (lane < (KD - HD) / 8) {
            uint16_t sv = 0;
            double n2d = q64_to_double((i128)n2);
            if (mips && lane == 0 && i < n_local) {
                i128 diff = rr - (i128)n2;
                sv = diff > 0 ? d2bf_rn_pos(sqrt(q64_to_double(diff))) : (uint16_t)0;
            }
            uint4 v = make_uint4((uint32_t)sv, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(tbase + (16 + lane) * 16 * 128 + rowoff) = v;
            if (lane == 0) {
                float sf = bf2f(sv);
                float nr = (float)sqrt(n2d + (double)sf * (double)sf);
                xnorm[unit * n_pad + i] = i < n_local ? nr : -1.0f;
                if (i < n_local) key_norm[unit * n_local + i] = nr;
            }
        } else if (KD == HD && lane == 0) {
            float nr = (float)sqrt(q64_to_double((i128)n2));
            xnorm[unit * n_pad + i] = i < n_local ? nr : -1.0f;
            if (i < n_local) key_norm[unit * n_local + i] = nr;
        }
    }
    if (bad) atomicOr(status, MAGICPIG_STATUS_INEXACT);
}

// Phase 3b: projections W [dp][KL] fp32 -> bf16 tiles of HG_N columns in the
// same canonical layout (element (c, kk) at ((kk/8)*(HG_N/8) + c/8)*128 + (c%8)*16 +
// (kk%8)*2), zero padded to KD rows and NT*HG_N columns; wmax = max_j |W_j|.
// grid (NT), block HG_N (thread = column)
__global__ void __launch_bounds__(HG_N) prep_w_kernel(const float* __restrict__ W, int dp, int KL, int KD,
                                                    uint8_t* __restrict__ wt, float* __restrict__ wmax,
                                                    uint32_t* status) {
    const int c = threadIdx.x;
    const int j = blockIdx.x * HG_N + c;
    uint8_t* tbase = wt + (int64_t)blockIdx.x * (HG_N * KD * 2);
    const int rowoff = (c >> 3) * 128 + (c & 7) * 16;
    float nrm = 0.0f;
    bool notrepr = false;
    for (int kc = 0; kc < KD / 8; kc++) {
        uint32_t h[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
            uint32_t lo = 0, hi = 0;
            int kk = kc * 8 + 2 * t;
            if (j < KL && kk < dp) {
                uint32_t u = __float_as_uint(W[(int64_t)kk * KL + j]);
                notrepr |= (u & 0xFFFFu) != 0;
                lo = u >> 16;
                float f = bf2f((uint16_t)lo);
                nrm = fmaf(f, f, nrm);
            }
            if (j < KL && kk + 1 < dp) {
                uint32_t u = __float_as_uint(W[(int64_t)(kk + 1) * KL + j]);
                notrepr |= (u & 0xFFFFu) != 0;
                hi = u >> 16;
                float f = bf2f((uint16_t)hi);
                nrm = fmaf(f, f, nrm);
            }
            h[t] = lo | (hi << 16);
        }
        *reinterpret_cast<uint4*>(tbase + kc * (HG_N / 8) * 128 + rowoff) = make_uint4(h[0], h[1], h[2], h[3]);
    }
    if (notrepr) atomicOr(status, MAGICPIG_STATUS_NOTREPR);
    // positive floats order like their bit patterns
    float nr = sqrtf(nrm) * (1.0f + 0x1p-10f);
    atomicMax(reinterpret_cast<unsigned int*>(wmax), __float_as_uint(nr));
}

// ---------------------------------------------------------------------------
// launchers
int launch_key_stats(const uint16_t* k, int64_t units, int64_t n_local, int64_t seq_offset,
                     int64_t n_global, int sink, int local, int64_t* part_sum, int64_t* part_cnt,
                     int64_t* key_sum, int64_t* count, uint32_t* status, cudaStream_t st) {
    int nsplit = (int)((n_local + STATS_SPLIT - 1) / STATS_SPLIT);
    if (nsplit < 1) nsplit = 1;
    key_stats_partial_kernel<<<dim3(nsplit, (unsigned)units), 256, 0, st>>>(
        k, n_local, seq_offset, n_global, sink, local, part_sum, part_cnt, status);
    sum_parts_kernel<<<(unsigned)units, 128, 0, st>>>(part_sum, part_cnt, nsplit, key_sum, count);
    count_launch(2);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

int launch_key_norms(const uint16_t* k, int64_t units, int64_t n_local, int64_t seq_offset,
                     int64_t n_global, int sink, int local, int do_center, const int64_t* key_sum,
                     const int64_t* count, float* center, int64_t* part_r2, int64_t* r2, uint32_t* status,
                     cudaStream_t st) {
    int nsplit = (int)((n_local + STATS_SPLIT - 1) / STATS_SPLIT);
    if (nsplit < 1) nsplit = 1;
    center_kernel<<<(unsigned)units, 128, 0, st>>>(key_sum, count, do_center, center);
#ifndef MP_LANE_PER_KEY
#define MP_LANE_PER_KEY 1
#endif
    if (MP_LANE_PER_KEY)
        r2_partial2_kernel<<<dim3(nsplit, (unsigned)units), 256, 0, st>>>(k, n_local, seq_offset, n_global, sink,
                                                                          local, center, part_r2, status);
    else
        r2_partial_kernel<<<dim3(nsplit, (unsigned)units), 256, 0, st>>>(k, n_local, seq_offset, n_global, sink,
                                                                         local, center, part_r2, status);
    max_parts_kernel<<<(unsigned)((units + 127) / 128), 128, 0, st>>>(part_r2, nsplit, units, r2);
    count_launch(3);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

int launch_reduce_shards(int mode, const int64_t* parts_sum, const int64_t* parts_cnt, int P, int64_t units,
                         int64_t* out_sum, int64_t* out_cnt, cudaStream_t st) {
    int64_t n = mode == 0 ? units * HD : units;
    reduce_shards_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(mode, parts_sum, parts_cnt, P, units,
                                                                      out_sum, out_cnt);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

int launch_prep(const uint16_t* k, int64_t units, int64_t n_local, int64_t n_pad, int mips, int KD,
                const float* center, const int64_t* r2, uint8_t* xt, float* xnorm, float* key_norm, const float* W,
                int KL, int NT, uint8_t* wt, float* wmax, uint32_t* status, cudaStream_t st) {
    cudaMemsetAsync(wmax, 0, sizeof(float), st);
    if (MP_LANE_PER_KEY)
        prep_x2_kernel<<<dim3((unsigned)((n_pad + 255) / 256), (unsigned)units), 256, 0, st>>>(
            k, n_local, n_pad, mips, KD, center, r2, xt, xnorm, key_norm, status);
    else
        prep_x_kernel<<<dim3((unsigned)((n_pad + 8 * PX_KEYS - 1) / (8 * PX_KEYS)), (unsigned)units), 256, 0, st>>>(
            k, n_local, n_pad, mips, KD, center, r2, xt, xnorm, key_norm, status);
    prep_w_kernel<<<NT, HG_N, 0, st>>>(W, HD + (mips ? 1 : 0), KL, KD, wt, wmax, status);
    count_launch(2);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

// ---------------------------------------------------------------------------
// Decode-time append: keys n_old .. n_old + m - 1 of every unit hashed with the index's
// frozen c and r^2 (reading R3; s = 0 when |x|^2 > r^2), exactly as the build does: xbar, |xbar| (key_norm),
// and one bit per projection column, bit = [exact xbar . W_j > 0] (R6) written into the bit-plane
// codes (layout for n_old + m keys).  CTA per (new key, unit): warp 0 forms xbar in shared memory; then
// thread per column: fp64 sum of the exact bf16 x bf16 products, certified when |sum| > 2^-44 sum |.|
// (the fp64 error over 129 terms is below 2^-45 of it), else the exact integer sign.
__global__ void __launch_bounds__(256) append_keys_kernel(const uint16_t* __restrict__ k_new, int64_t m,
                                                          int64_t n_old, int mips, const float* __restrict__ W,
                                                          int KL, int KLq, int64_t nchunks,
                                                          const float* __restrict__ center,
                                                          const int64_t* __restrict__ r2, uint32_t* __restrict__ codes,
                                                          float* __restrict__ key_norm, uint32_t* status) {
    __shared__ uint16_t xs[HD + 8];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t i = blockIdx.x, unit = blockIdx.y;
    const int64_t n_new = n_old + m, pos = n_old + i;
    const int dp = HD + (mips ? 1 : 0);
    if (tid < 32) {
        const float4 c = reinterpret_cast<const float4*>(center + unit * HD)[lane];
        const uint2 kr = reinterpret_cast<const uint2*>(k_new + (unit * m + i) * HD)[lane];
        uint32_t a = 0, b = 0;
        bool bad = false;
        const u128 n2 = warp_sum_u128(transform4(kr, c, a, b, bad));
        if (bad) atomicOr(status, MAGICPIG_STATUS_INEXACT);
        reinterpret_cast<uint2*>(xs)[lane] = make_uint2(a, b);
        if (lane == 0) {
            uint16_t sv = 0;
            if (mips) {
                const i128 diff = ld_q64(r2 + unit * 2) - (i128)n2;
                sv = diff > 0 ? d2bf_rn_pos(sqrt(q64_to_double(diff))) : (uint16_t)0;
            }
            xs[HD] = sv;
            const float sf = bf2f(sv);
            key_norm[unit * n_new + pos] = (float)sqrt(q64_to_double((i128)n2) + (double)sf * (double)sf);
        }
    }
    __syncthreads();
    const int64_t chunk = pos >> 10, blk = (pos >> 5) & 31;
    const uint32_t bit = 1u << (pos & 31);
    uint32_t* cu = codes + (unit * nchunks + chunk) * (int64_t)KLq * 128;
    for (int j = tid; j < KLq * 4; j += blockDim.x) {
        int sg = 0;
        if (j < KL) {
            double s = 0.0, sa = 0.0;
            for (int d = 0; d < dp; d++) {
                const double pr = (double)bf2f(xs[d]) * (double)__ldg(W + (int64_t)d * KL + j);
                s += pr;
                sa += fabs(pr);
            }
            if (fabs(s) > 0x1p-44 * sa) {
                sg = s > 0.0;
            } else {
                uint16_t wv[HD + 1];
                for (int d = 0; d < dp; d++) wv[d] = (uint16_t)(__float_as_uint(__ldg(W + (int64_t)d * KL + j)) >> 16);
                sg = exact_dot_sign_bf16(xs, wv, dp, status) > 0;
            }
        }
        uint32_t* w = cu + (((int64_t)(j >> 2)) * 32 + blk) * 4 + (j & 3);
        if (sg) atomicOr(w, bit);
        else atomicAnd(w, ~bit);
    }
}

int launch_append_keys(const uint16_t* k_new, int64_t m, int64_t units, int64_t n_old, int mips, const float* W,
                       int KL, int KLq, int64_t nchunks, const float* center, const int64_t* r2, uint32_t* codes,
                       float* key_norm, uint32_t* status, cudaStream_t st) {
    if (m < 1 || units < 1) return 0;
    append_keys_kernel<<<dim3((unsigned)m, (unsigned)units), 256, 0, st>>>(k_new, m, n_old, mips, W, KL, KLq, nchunks,
                                                                          center, r2, codes, key_norm, status);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

}  // namespace mp
