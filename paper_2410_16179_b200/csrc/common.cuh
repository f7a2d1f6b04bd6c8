// common.cuh -- shared device helpers of the sm_100a MagicPIG library.
// (CUDA path only; nothing here is shared with oracle/.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/magicpig.h"

namespace mp {

constexpr int HD = 128;          // head dim (only 128 supported)
constexpr int KCHUNK = 1024;     // keys per code chunk (32 blocks of 32 keys)
constexpr int PART = HD + 2;     // (m, s, a[128]) partial softmax state
constexpr int PREC5 = HD + 4;    // persistent decode record per head: (m, s, |S_g|, 0, a[128])
constexpr float HASH_EPS = 0x1p-19f;  // tensor-core filter: |acc| <= eps*|x||W_j| -> exact fix-up
                                      // (measured tcgen05 error 2^-23.5 |x||W_j|: 22x margin)

typedef __int128 i128;
typedef unsigned __int128 u128;

// --------------------------------------------------------------------------
// table grouping: a "group" is TG tables = QG 4-column quads (lcm(K, 4) columns)
__host__ __device__ constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }
__host__ __device__ constexpr int tg_of(int K) { return 4 / gcd_c(K, 4); }
__host__ __device__ constexpr int qg_of(int K) { return K / gcd_c(K, 4); }

struct Geom {
    int K, L, KL;
    int TG, QG;        // tables / quads per group
    int ngroups;       // ceil(L / TG)
    int KLq;           // quads per key chunk row = ngroups * QG
    int KLw;           // 32-bit words of a packed query code = ceil(KL / 32)
    int64_t nchunks;   // ceil(n_local / 1024)
};

__host__ __device__ inline Geom make_geom(int K, int L, int64_t n_local) {
    Geom g;
    g.K = K;
    g.L = L;
    g.KL = K * L;
    g.TG = tg_of(K);
    g.QG = qg_of(K);
    g.ngroups = (L + g.TG - 1) / g.TG;
    g.KLq = g.ngroups * g.QG;
    g.KLw = (g.KL + 31) / 32;
    g.nchunks = (n_local + KCHUNK - 1) / KCHUNK;
    return g;
}

// --------------------------------------------------------------------------
// bf16 helpers
__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float(uint32_t(h) << 16); }

// fp32 -> bf16, round to nearest even (finite inputs)
__device__ __forceinline__ uint16_t f2bf_rn(float f) {
    uint32_t u = __float_as_uint(f);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

// non-negative double -> bf16, ONE round-to-nearest-even step
__device__ __forceinline__ uint16_t d2bf_rn_pos(double v) {
    if (!(v > 0.0)) return 0;
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    int e = (int)((b >> 52) & 0x7FF) - 1023;
    if (e >= -126) {
        unsigned long long rem = b & ((1ull << 45) - 1ull);
        unsigned long long t = b >> 45;
        const unsigned long long half = 1ull << 44;
        if (rem > half || (rem == half && (t & 1ull))) t += 1ull;
        double r = __longlong_as_double((long long)(t << 45));
        return (uint16_t)(__float_as_uint((float)r) >> 16);  // exact conversion
    }
    // bf16 subnormal: f * 2^-133
    long long f = __double2ll_rn(v * 0x1p133);
    return (uint16_t)f;
}

// --------------------------------------------------------------------------
// fixed point, units of 2^-64 (reading R2b)
// trunc(k * 2^64) for a bf16 value k (|k| < 2^27 assumed, checked by caller)
__device__ __forceinline__ i128 q64_of_bf16(uint16_t h) {
    int E = (h >> 7) & 0xFF;
    uint32_t M = (h & 0x7Fu) | (E ? 0x80u : 0u);
    int e = E ? E : 1;
    // value = M * 2^(e - 134); * 2^64 -> M * 2^(e - 70)
    u128 mag;
    if (e >= 70) mag = ((u128)M) << (e - 70);
    else mag = (70 - e >= 32) ? (u128)0 : (u128)(M >> (70 - e));
    return (h & 0x8000u) ? -(i128)mag : (i128)mag;
}

// trunc(x2 * 2^64) for a non-negative exactly representable fp32 value
__device__ __forceinline__ u128 q64_of_f32(float x2) {
    uint32_t b = __float_as_uint(x2);
    int E = (b >> 23) & 0xFF;
    uint32_t M = (b & 0x7FFFFFu) | (E ? 0x800000u : 0u);
    int e = E ? E : 1;
    // value = M * 2^(e - 150); * 2^64 -> M * 2^(e - 86)
    if (e >= 86) return ((u128)M) << (e - 86);
    int sh = 86 - e;
    return sh >= 32 ? (u128)0 : (u128)(M >> sh);
}

// round-to-nearest-even int128 -> double, then * 2^-64
__device__ __forceinline__ double q64_to_double(i128 v) {
    if (v == 0) return 0.0;
    bool neg = v < 0;
    u128 a = neg ? (u128)0 - (u128)v : (u128)v;
    unsigned long long hi = (unsigned long long)(a >> 64), lo = (unsigned long long)a;
    int msb = hi ? 127 - __clzll((long long)hi) : 63 - __clzll((long long)lo);
    double r;
    if (msb <= 52) {
        r = (double)lo;
    } else {
        int sh = msb - 52;
        u128 m = a >> sh;
        u128 rem = a - (m << sh);
        u128 half = ((u128)1) << (sh - 1);
        if (rem > half || (rem == half && ((unsigned long long)m & 1ull))) m += 1;
        r = ldexp((double)(unsigned long long)m, sh);
    }
    r = ldexp(r, -64);
    return neg ? -r : r;
}

__device__ __forceinline__ i128 ld_q64(const int64_t* p) {
    u128 lo = (u128)(unsigned long long)p[0];
    u128 hi = (u128)(unsigned long long)p[1];
    return (i128)(lo | (hi << 64));
}
__device__ __forceinline__ void st_q64(int64_t* p, i128 v) {
    u128 u = (u128)v;
    p[0] = (int64_t)(unsigned long long)u;
    p[1] = (int64_t)(unsigned long long)(u >> 64);
}

__device__ __forceinline__ u128 shfl_xor_u128(u128 v, int m) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
    lo = __shfl_xor_sync(0xffffffffu, lo, m);
    hi = __shfl_xor_sync(0xffffffffu, hi, m);
    return ((u128)hi << 64) | (u128)lo;
}

// --------------------------------------------------------------------------
// exact sign of sum_t a_t * b_t for bf16 a, b (both given as bf16 bit
// patterns).  Integer accumulation aligned to the largest product exponent;
// products more than 100 binades below it are dropped, and the result is
// flagged (STATUS_INEXACT) only if they could have changed the sign.
__device__ inline int exact_dot_sign_bf16(const uint16_t* a, const uint16_t* b, int n,
                                          uint32_t* status) {
    int emax = -1;
    for (int t = 0; t < n; t++) {
        uint16_t x = a[t], y = b[t];
        if ((x & 0x7FFF) == 0 || (y & 0x7FFF) == 0) continue;
        int ex = (x >> 7) & 0xFF, ey = (y >> 7) & 0xFF;
        int e = (ex ? ex : 1) + (ey ? ey : 1);
        emax = e > emax ? e : emax;
    }
    if (emax < 0) return 0;
    const int base = emax - 100;
    i128 acc = 0;
    bool dropped = false;
    for (int t = 0; t < n; t++) {
        uint16_t x = a[t], y = b[t];
        if ((x & 0x7FFF) == 0 || (y & 0x7FFF) == 0) continue;
        int ex = (x >> 7) & 0xFF, ey = (y >> 7) & 0xFF;
        uint32_t mx = (x & 0x7Fu) | (ex ? 0x80u : 0u);
        uint32_t my = (y & 0x7Fu) | (ey ? 0x80u : 0u);
        int e = (ex ? ex : 1) + (ey ? ey : 1);
        uint32_t m = mx * my;
        if (e < base) {
            dropped = true;
            continue;
        }
        i128 term = ((i128)m) << (e - base);
        acc += ((x ^ y) & 0x8000u) ? -term : term;
    }
    if (dropped) {
        i128 lim = ((i128)n) << 16;
        if (acc < lim && acc > -lim) atomicOr(status, MAGICPIG_STATUS_INEXACT);
    }
    return (acc > 0) - (acc < 0);
}

// --------------------------------------------------------------------------
// log of the sampling probability (Eq. LSH sampling probability):
//   x = p^K;  min 2: u = P[Binomial(L, x) >= 2] = 1-(1-x)^L-Lx(1-x)^(L-1)
//             min 1: u = 1-(1-x)^L
// fp32 and cancellation-free (R11):
//   y = (L-1) x <= 1:  ln u = ln C(L,2) + 2 ln x + (L-2) ln(1-x) + ln(1 + s),
//                      s = sum_{j>=3} t_j/t_2 (Horner; t_{j+1}/t_j = (L-j)/(j+1) * x/(1-x))
//   y > 1:             ln u = ln(-expm1((L-1) ln(1-x) + ln(1+y)))   (u >= 0.26)
// floored at ln(1e-300).
constexpr float LOG_U_FLOOR = -690.7755279f;

__device__ __forceinline__ float log_sampling_prob(float p, int K, int L, int minc) {
    // hardware log2/exp2 (MUFU, ~2 ulp): |error in ln u| < 1e-5, far below the
    // 2e-3 output tolerance; the chain stays short because this runs once per
    // (sampled key, head) on the critical path of the decode.
    if (!(p > 0.0f)) return LOG_U_FLOOR;
    if (p >= 1.0f) return 0.0f;
    const float lnx = (float)K * __logf(p);
    const float x = __expf(lnx);
    const float l1mx = __logf(1.0f - x);  // ln(1 - x); x <= 1 - 2^-24 here
    float lu;
    if (minc == 1) {
        const float Lx = (float)L * x;
        if (Lx < 1e-3f) lu = lnx + __logf((float)L) - 0.5f * (float)(L - 1) * x;
        else lu = __logf(-expm1f((float)L * l1mx));
    } else {
        const float y = (float)(L - 1) * x;
        if (y <= 1.0f) {
            const float r = __fdividef(x, 1.0f - x);
            float s = 0.0f;
#pragma unroll
            for (int j = 11; j >= 2; j--) {
                // s_j = (L-j)/(j+1) r (1 + s_{j+1}); terms beyond L vanish; truncation < y^10/11! ~ 3e-8
                const float c = (float)(L - j) * (1.0f / (float)(j + 1));
                s = (L - j > 0) ? c * r * (1.0f + s) : 0.0f;
            }
            lu = __logf(0.5f * (float)L * (float)(L - 1)) + 2.0f * lnx + (float)(L - 2) * l1mx + __logf(1.0f + s);
        } else {
            lu = __logf(-expm1f((float)(L - 1) * l1mx + __logf(1.0f + y)));
        }
    }
    return fmaxf(lu, LOG_U_FLOOR);
}

// double-precision evaluation of the same cancellation-free form (fills the ln u table)
__device__ inline double log_sampling_prob_d(double p, int K, int L, int minc) {
    if (!(p > 0.0)) return (double)LOG_U_FLOOR;
    if (p >= 1.0) return 0.0;
    const double lnx = (double)K * log(p);
    const double x = exp(lnx);
    const double l1mx = log1p(-x);
    double lu;
    if (minc == 1) {
        lu = log(-expm1((double)L * l1mx));
    } else {
        const double y = (double)(L - 1) * x;
        if (y <= 1.0) {
            const double r = x / (1.0 - x);
            double s = 0.0;
            for (int j = 24; j >= 2; j--) s = (L - j > 0) ? (double)(L - j) / (double)(j + 1) * r * (1.0 + s) : 0.0;
            lu = log(0.5 * (double)L * (double)(L - 1)) + 2.0 * lnx + (double)(L - 2) * l1mx + log1p(s);
        } else {
            lu = log(-expm1((double)(L - 1) * l1mx + log1p(y)));
        }
    }
    return lu > (double)LOG_U_FLOOR ? lu : (double)LOG_U_FLOOR;
}

// ln u(p) table over p in [LUT_P0, 1]: LUT_N intervals, linear interpolation (|error| < 4e-6 in ln u,
// d^2 ln u / dp^2 <= ~600 on this range); below LUT_P0 (u < 1e-5 at K >= 7: such keys are essentially
// never sampled) the fp32 closed form is evaluated directly.
constexpr int LUT_N = 4096;
constexpr float LUT_P0 = 0.125f;
constexpr float LUT_INV_H = (float)LUT_N / (1.0f - LUT_P0);
constexpr int LUT_WORDS = LUT_N + 8;
__device__ __forceinline__ float log_sampling_prob_lut(const float* __restrict__ tab, float p, int K, int L,
                                                       int minc) {
    if (p >= 1.0f) return 0.0f;
    if (!(p >= LUT_P0)) return log_sampling_prob(p, K, L, minc);
    const float x = (p - LUT_P0) * LUT_INV_H;
    const int i = min((int)x, LUT_N - 1);
    const float f = x - (float)i;
    const float t0 = __ldg(tab + i), t1 = __ldg(tab + i + 1);
    return fmaf(f, t1 - t0, t0);
}

// --------------------------------------------------------------------------
// PTX wrappers: mbarrier, bulk copy, tcgen05
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: the waiting warp sleeps in hardware until the
// phase completes (or the hint expires) instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MPWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra MPWAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x100000u)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate (kind::f16)
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 columns of 32-bit: thread t gets lane (base lane + t), cols c..c+31
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle ("interleaved" canonical
// layout): core matrix = 8 rows x 16 bytes contiguous; LBO = byte distance
// between core matrices adjacent in K; SBO = between 8-row groups.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, layout type 0 = SWIZZLE_NONE
}

// instruction descriptor, kind::f16: A,B = bf16 K-major, D = f32
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

}  // namespace mp
