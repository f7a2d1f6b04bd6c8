/*
 * magicpig_oracle.c -- plain, slow, double-precision CPU ORACLE for MagicPIG's
 * decode-time hot path (arXiv 2410.16179).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_2410_16179_b200/csrc); neither side includes or links the other.
 *
 * Citations "P:<line>" refer to /root/reference/PAPER.md (the paper's LaTeX
 * source).  Readings of the paper where it is silent or ambiguous are the ones
 * listed in DESIGN.md section "Readings" (R1..R20) and SURVEY.md 8(c) C-3.
 *
 * Everything is written as plain loops in the paper's order, in IEEE double,
 * compiled with -O2 -ffp-contract=off (no FMA contraction, no reassociation).
 * bf16 inputs are passed as their raw 16-bit patterns and decoded here.
 *
 * Exactness contract:
 *   - products of two bf16-representable values are exact in double;
 *   - every accumulation that must be exact is done with TwoSum and an
 *     "inexact" flag; sign decisions that would be affected fall back to an
 *     exact (Shewchuk) floating-point expansion, so every hash bit is the sign
 *     of the EXACT real dot product, with sign(0) -> bit 0.
 *
 * Parity status: every function below is pinned by a -m "not gpu" test
 * (tests/test_oracle_pins.py); see the per-function comments.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_EINEXACT (-2)    /* an accumulation that the contract requires exact was not */
#define OR_ENOTREPR (-3)    /* W value not bf16-representable */
#define OR_EDEGENERATE (-4) /* S and T both empty for some head */

/* ------------------------------------------------------------------------- */
/* bf16 helpers (encoding defined by the bfloat16 format, not by the paper).  */

double oracle_bf16_to_double(uint16_t h) {
    /* bf16 = upper 16 bits of an IEEE binary32 */
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* Round a double to the nearest bf16 (ties to even), ONE rounding step.
 * Used for x_i = bf16_rn(.) and s_i = bf16_rn(sqrt(.)). */
uint16_t oracle_bf16_from_double(double v) {
    uint16_t sign = signbit(v) ? 0x8000u : 0u;
    double a = fabs(v);
    if (a == 0.0) return sign;
    if (isinf(a) || isnan(a)) return (uint16_t)(sign | 0x7F80u | (isnan(a) ? 0x40u : 0u));
    int e;
    double m = frexp(a, &e); /* a = m * 2^e, 0.5 <= m < 1 */
    /* normal bf16: value = (1.f) * 2^(E-127), 8 significant bits */
    int E = e - 1 + 127; /* biased exponent of a */
    if (E >= 1) {
        double t = ldexp(m, 8);      /* in [128, 256): 8 significant bits + fraction */
        double r = nearbyint(t);     /* round half to even (default rounding mode) */
        if (r == 256.0) { r = 128.0; E += 1; }
        if (E >= 255) return (uint16_t)(sign | 0x7F80u); /* overflow -> inf */
        return (uint16_t)(sign | ((uint32_t)E << 7) | ((uint32_t)r - 128u));
    }
    /* subnormal bf16: value = f * 2^-133, f in [0,128) */
    double t = ldexp(a, 133);
    double r = nearbyint(t); /* r <= 128; 128 encodes the smallest normal */
    return (uint16_t)(sign | (uint32_t)r);
}

/* fp32 round-to-nearest-even of an exact pair value hi+lo (|lo| <= ulp(hi)/2).
 * Avoids double rounding when hi alone sits on an fp32 midpoint. */
static float f32_round_pair(double hi, double lo) {
    float f = (float)hi;
    if (lo == 0.0) return f;
    double d = hi - (double)f; /* exact */
    if (d > 0.0) {
        float up = nextafterf(f, INFINITY);
        double mid = 0.5 * ((double)f + (double)up);
        if (hi == mid && lo > 0.0) f = up;
    } else if (d < 0.0) {
        float dn = nextafterf(f, -INFINITY);
        double mid = 0.5 * ((double)f + (double)dn);
        if (hi == mid && lo < 0.0) f = dn;
    }
    return f;
}

/* Knuth TwoSum: s + e == a + b exactly. */
static void two_sum(double a, double b, double *s, double *e) {
    double x = a + b;
    double bv = x - a;
    double av = x - bv;
    *e = (a - av) + (b - bv);
    *s = x;
}

/* Shewchuk grow-expansion with zero elimination: e[0..m) nonoverlapping,
 * increasing magnitude; adds b exactly.  Returns the new length. */
static int grow_expansion(double *e, int m, double b) {
    double q = b;
    int k = 0;
    for (int i = 0; i < m; i++) {
        double s, h;
        two_sum(q, e[i], &s, &h);
        if (h != 0.0) e[k++] = h;
        q = s;
    }
    if (q != 0.0) e[k++] = q;
    return k;
}

/* Sign of the EXACT real value of sum_t a[t]*b[t] where each product is exact
 * in double (bf16 x bf16).  Fast path: sequential double sum, exact when no
 * TwoSum error term appears; otherwise an exact expansion decides.
 * Returns -1, 0, +1.  (SimHash sign of the projection; sign(0)->0 is
 * reading R6.) */
int oracle_exact_dot_sign(const double *a, const double *b, int m) {
    double s = 0.0;
    int inexact = 0;
    for (int t = 0; t < m; t++) {
        double p = a[t] * b[t];
        double e;
        two_sum(s, p, &s, &e);
        if (e != 0.0) inexact = 1;
    }
    if (!inexact) return (s > 0.0) - (s < 0.0);
    double *ex = (double *)malloc(sizeof(double) * (size_t)(m + 1));
    int len = 0;
    for (int t = 0; t < m; t++) len = grow_expansion(ex, len, a[t] * b[t]);
    int sg = 0;
    if (len > 0) sg = (ex[len - 1] > 0.0) - (ex[len - 1] < 0.0);
    free(ex);
    return sg;
}

/* ------------------------------------------------------------------------- */
/* Static / dynamic partition (P:171 on-device cache; "initial 4 tokens
 * and local 64"; reading R12): T = [0,sink) U [n-local, n), D = the rest.     */

int oracle_is_static(int64_t pos, int64_t n, int sink, int local) {
    return pos < (int64_t)sink || pos >= n - (int64_t)local;
}

/* ------------------------------------------------------------------------- */
/* Fixed-point exact sums (reading R2b).  A double sum of bf16 values or of
 * their squares is NOT exact in general (the spread of binades exceeds 53
 * bits for N(0,1) data), so the key statistics are accumulated exactly as
 * integers in units of 2^-64:  q(v) = trunc(v * 2^64)  (exact for |v| >= 2^-57
 * when v is a bf16 value or a square of one), summed in 128-bit integers, and
 * converted back with one round-to-nearest-even step.                        */
typedef __int128 i128;

#define FIX_SHIFT 64
#define ABS_LIMIT 134217728.0 /* 2^27: |k|, |x| must stay below it (no overflow) */

static i128 fix_of(double v) { /* trunc(v * 2^64), v exactly a double */
    return (i128)ldexp(v, FIX_SHIFT);
}

/* round-to-nearest-even conversion of an int128 to double, then * 2^-64 */
double oracle_fix_to_double(i128 v) {
    if (v == 0) return 0.0;
    int neg = v < 0;
    unsigned __int128 a = neg ? (unsigned __int128)(-(v + 1)) + 1u : (unsigned __int128)v;
    int msb = 127;
    while (!((a >> msb) & 1u)) msb--;
    double r;
    if (msb <= 52) {
        r = (double)(uint64_t)a;
    } else {
        int sh = msb - 52;
        unsigned __int128 m = a >> sh;
        unsigned __int128 rem = a & ((((unsigned __int128)1) << sh) - 1u);
        unsigned __int128 half = ((unsigned __int128)1) << (sh - 1);
        if (rem > half || (rem == half && (m & 1u))) m += 1u;
        r = ldexp((double)(uint64_t)m, sh);
    }
    r = ldexp(r, -FIX_SHIFT);
    return neg ? -r : r;
}

static void put_i128(uint64_t *dst, i128 v) {
    unsigned __int128 u = (unsigned __int128)v;
    dst[0] = (uint64_t)u;
    dst[1] = (uint64_t)(u >> 64);
}

/* ------------------------------------------------------------------------- */
/* Data pre-processing: centering then the MIPS transform
 * (Eq. data transform), per (sequence, kv head).
 *
 *   ksum_d = sum_{i in D} q(k_{i,d})                     (exact integer)
 *   c_d    = fl32( fl64( fl64(ksum_d 2^-64) / |D| ) )     (R2, R3)
 *   x_i    = bf16_rn( fl32(k_i - c) )          for all n keys   (R16)
 *   n2q_i  = sum_d q(x_{i,d}^2)                           (exact integer)
 *   r2q    = max_{i in D} n2q_i                           (P:50 r = max|k_i|)
 *   s_i    = bf16_rn( sqrt_rn( fl64((r2q - n2q_i) 2^-64) ) ), 0 if r2q <= n2q_i
 *   xbar_i = [x_i, s_i] if mips else x_i
 * center=0 -> c = 0.  |D| = 0 -> c = 0 and r2q = 0.
 * Outputs: c[d] (float), xbar[n][d+mips] (bf16 bits), n2[n] = fl64(n2q 2^-64),
 * *r2 = fl64(r2q 2^-64); optional exact integers as (lo, hi) uint64 pairs:
 * ksum_q[d][2], r2_q[2], n2_q[n][2].  Returns OR_EINEXACT if some |k| or |x|
 * reaches 2^27 (outside the exact range).                                  */
int oracle_key_transform(int n, int d, const uint16_t *k, int sink, int local,
                         int center, int mips, float *c, uint16_t *xbar,
                         double *n2, double *r2_out, uint64_t *ksum_q, uint64_t *r2_q,
                         uint64_t *n2_q) {
    if (n < 0 || d <= 0) return OR_EINVAL;
    int inexact = 0;
    int dp = d + (mips ? 1 : 0);
    int64_t nD = 0;
    for (int i = 0; i < n; i++)
        if (!oracle_is_static(i, n, sink, local)) nD++;
    /* centering vector (k_i - (1/n) sum k_i, taken over the sampled set D) */
    for (int j = 0; j < d; j++) {
        i128 sum = 0;
        for (int i = 0; i < n; i++) {
            if (oracle_is_static(i, n, sink, local)) continue;
            double kv = oracle_bf16_to_double(k[(size_t)i * d + j]);
            if (fabs(kv) >= ABS_LIMIT) inexact = 1;
            sum += fix_of(kv);
        }
        if (ksum_q) put_i128(ksum_q + 2 * (size_t)j, sum);
        if (center && nD > 0) {
            double mean = oracle_fix_to_double(sum) / (double)nD;
            c[j] = (float)mean;
        } else {
            c[j] = 0.0f;
        }
    }
    /* transformed keys and exact squared norms */
    i128 *nq = (i128 *)malloc(sizeof(i128) * (size_t)(n > 0 ? n : 1));
    i128 r2q = 0;
    for (int i = 0; i < n; i++) {
        i128 acc = 0;
        for (int j = 0; j < d; j++) {
            double kv = oracle_bf16_to_double(k[(size_t)i * d + j]);
            double hi, lo;
            two_sum(kv, -(double)c[j], &hi, &lo);
            float diff = f32_round_pair(hi, lo); /* fl32(k - c) */
            uint16_t xb = oracle_bf16_from_double((double)diff);
            xbar[(size_t)i * dp + j] = xb;
            double xv = oracle_bf16_to_double(xb);
            if (fabs(xv) >= ABS_LIMIT) inexact = 1;
            acc += fix_of(xv * xv); /* square of a bf16 value: exact in double */
        }
        nq[i] = acc;
        n2[i] = oracle_fix_to_double(acc);
        if (n2_q) put_i128(n2_q + 2 * (size_t)i, acc);
        if (!oracle_is_static(i, n, sink, local) && acc > r2q) r2q = acc;
    }
    if (mips) {
        for (int i = 0; i < n; i++) {
            double diff = r2q > nq[i] ? oracle_fix_to_double(r2q - nq[i]) : 0.0;
            xbar[(size_t)i * dp + d] = oracle_bf16_from_double(sqrt(diff));
        }
    }
    free(nq);
    *r2_out = oracle_fix_to_double(r2q);
    if (r2_q) put_i128(r2_q, r2q);
    return inexact ? OR_EINEXACT : OR_OK;
}

/* Check that every W value is exactly bf16-representable (R8). */
int oracle_check_w(const float *W, int64_t count) {
    for (int64_t t = 0; t < count; t++) {
        uint32_t u;
        memcpy(&u, &W[t], 4);
        if ((u & 0xFFFFu) != 0u) return OR_ENOTREPR;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* SimHash Encode ("projected on K directions, only the sign of the
 * projection is kept"; Alg. 1 Encode).
 * vec: dp values (double); W: [dp][K*L] row-major float (bf16-representable).
 * Table t uses columns [tK, tK+K); code bit b = [exact(vec . W[:,tK+b]) > 0]
 * (R6, R7).  codes: L uint16 (K <= 16).                                      */
static double *transpose_w(const float *W, int dp, int KL) {
    double *Wt = (double *)malloc(sizeof(double) * (size_t)dp * KL);
    for (int r = 0; r < dp; r++)
        for (int j = 0; j < KL; j++) Wt[(size_t)j * dp + r] = (double)W[(size_t)r * KL + j];
    return Wt;
}

static void encode_with_wt(const double *vec, int dp, const double *Wt, int K, int L,
                           uint16_t *codes) {
    for (int t = 0; t < L; t++) {
        uint32_t code = 0;
        for (int b = 0; b < K; b++) {
            int j = t * K + b;
            if (oracle_exact_dot_sign(vec, Wt + (size_t)j * dp, dp) > 0) code |= (1u << b);
        }
        codes[t] = (uint16_t)code;
    }
}

void oracle_encode_vec(const double *vec, int dp, const float *W, int K, int L,
                       uint16_t *codes) {
    double *Wt = transpose_w(W, dp, K * L);
    encode_with_wt(vec, dp, Wt, K, L, codes);
    free(Wt);
}

/* Encode keys: xbar [n][dp] bf16 bits -> codes [n][L]. */
void oracle_encode_keys(int n, int dp, const uint16_t *xbar, const float *W, int K,
                        int L, uint16_t *codes) {
    double *vec = (double *)malloc(sizeof(double) * (size_t)dp);
    double *Wt = transpose_w(W, dp, K * L);
    for (int i = 0; i < n; i++) {
        for (int r = 0; r < dp; r++) vec[r] = oracle_bf16_to_double(xbar[(size_t)i * dp + r]);
        encode_with_wt(vec, dp, Wt, K, L, codes + (size_t)i * L);
    }
    free(Wt);
    free(vec);
}

/* Encode a query: qbar = [q, 0] (R4: query is not centered).  Only the
 * first d rows of W meet non-zero query entries. */
void oracle_encode_query(int d, int mips, const uint16_t *q, const float *W, int K,
                         int L, uint16_t *codes) {
    int dp = d + (mips ? 1 : 0);
    double *vec = (double *)malloc(sizeof(double) * (size_t)dp);
    for (int r = 0; r < d; r++) vec[r] = oracle_bf16_to_double(q[r]);
    if (mips) vec[d] = 0.0;
    oracle_encode_vec(vec, dp, W, K, L, codes);
    free(vec);
}

/* ------------------------------------------------------------------------- */
/* Query (Alg. 1; two-table rule P:84 footnote): number of tables in
 * which key i shares the query's K-bit code. */
void oracle_collision_counts(int n, int L, const uint16_t *codes, const uint16_t *qcode,
                             int32_t *cnt) {
    for (int i = 0; i < n; i++) {
        int c = 0;
        for (int t = 0; t < L; t++)
            if (codes[(size_t)i * L + t] == qcode[t]) c++;
        cnt[i] = c;
    }
}

/* Bucketed hash tables (the paper's HT): for each table a list
 * of key ids grouped by code; Query = look up the query's bucket in each table
 * and count hits per key.  A second, independent way to get the counts (pin
 * P10).  counts must be zero-initialised by the caller. */
void oracle_bucket_query(int n, int K, int L, const uint16_t *codes, const uint16_t *qcode,
                         int32_t *counts) {
    int nb = 1 << K;
    int32_t *start = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nb + 1));
    int32_t *ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    for (int t = 0; t < L; t++) {
        /* counting sort of key ids by code: HT_t */
        for (int b = 0; b <= nb; b++) start[b] = 0;
        for (int i = 0; i < n; i++) start[codes[(size_t)i * L + t] + 1]++;
        for (int b = 0; b < nb; b++) start[b + 1] += start[b];
        int32_t *fill = (int32_t *)malloc(sizeof(int32_t) * (size_t)nb);
        for (int b = 0; b < nb; b++) fill[b] = start[b];
        for (int i = 0; i < n; i++) ids[fill[codes[(size_t)i * L + t]]++] = i;
        free(fill);
        /* lookup */
        int b = qcode[t];
        for (int p = start[b]; p < start[b + 1]; p++) counts[ids[p]]++;
    }
    free(start);
    free(ids);
}

/* ------------------------------------------------------------------------- */
/* Eq. (LSH sampling probability), P:86-91 / Alg. 1 P:111-113:
 *   p = 1 - arccos(cos)/pi
 *   u = 1 - (1-p^K)^L - L p^K (1-p^K)^(L-1)         (min_collisions = 2)
 *   u = 1 - (1-p^K)^L                               (min_collisions = 1)
 * The printed form cancels catastrophically in double for small p (it even
 * goes negative), so it is evaluated in an algebraically identical form
 * (reading R11): with x = p^K and y = (L-1) x,
 *   min 2, y <= 1 : u = sum_{j=2}^{L} C(L,j) x^j (1-x)^(L-j)   (binomial tail,
 *                   all terms positive; "at least two of L independent tables
 *                   match", each with probability x)
 *   min 2, y >  1 : u = -expm1( (L-1) log1p(-x) + log1p(y) )
 *   min 1         : u = -expm1( L log1p(-x) )                              */
double oracle_collision_prob(double cosv) {
    if (cosv > 1.0) cosv = 1.0;
    if (cosv < -1.0) cosv = -1.0;
    return 1.0 - acos(cosv) / M_PI;
}

double oracle_sampling_prob(double p, int K, int L, int min_collisions) {
    double x = pow(p, (double)K);
    if (min_collisions == 1) return -expm1((double)L * log1p(-x));
    if (x >= 1.0) return 1.0;
    if (x <= 0.0) return 0.0;
    double y = (double)(L - 1) * x;
    if (y > 1.0) return -expm1((double)(L - 1) * log1p(-x) + log1p(y));
    /* binomial tail, term by term */
    double t = 0.5 * (double)L * (double)(L - 1) * x * x * exp((double)(L - 2) * log1p(-x));
    double sum = 0.0;
    for (int j = 2; j <= L; j++) {
        sum += t;
        if (t <= 1e-18 * sum) break;
        t = t * (double)(L - j) / (double)(j + 1) * (x / (1.0 - x));
    }
    return sum;
}

/* The formula exactly as printed, for comparison in tests. */
double oracle_sampling_prob_naive(double p, int K, int L) {
    double x = pow(p, (double)K);
    return 1.0 - pow(1.0 - x, (double)L) - (double)L * x * pow(1.0 - x, (double)(L - 1));
}

/* Eq. (budget): expected sampled fraction at p = 0.5. */
double oracle_expected_budget(int K, int L, int min_collisions) {
    return oracle_sampling_prob(0.5, K, L, min_collisions);
}

/* ------------------------------------------------------------------------- */
/* Exact attention: o = Softmax(q K^T / sqrt(d)) V.  Reference
 * semantics for pins P4, P5, P9.  k, v: [n][d] bf16; q: [d] bf16. */
void oracle_exact_attention(int n, int d, const uint16_t *q, const uint16_t *k,
                            const uint16_t *v, double *out) {
    double *l = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double m = -INFINITY;
    double scale = 1.0 / sqrt((double)d);
    for (int i = 0; i < n; i++) {
        double s = 0.0;
        for (int j = 0; j < d; j++)
            s += oracle_bf16_to_double(q[j]) * oracle_bf16_to_double(k[(size_t)i * d + j]);
        l[i] = s * scale;
        if (l[i] > m) m = l[i];
    }
    double z = 0.0;
    for (int j = 0; j < d; j++) out[j] = 0.0;
    for (int i = 0; i < n; i++) {
        double w = exp(l[i] - m);
        z += w;
        for (int j = 0; j < d; j++) out[j] += w * oracle_bf16_to_double(v[(size_t)i * d + j]);
    }
    for (int j = 0; j < d; j++) out[j] /= z;
    free(l);
}

/* Exact attention with raw fp64 keys (used for the centering-invariance pin
 * P9, where the keys are centered in double). */
void oracle_exact_attention_f64(int n, int d, const double *q, const double *k,
                                const double *v, double *out) {
    double *l = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double m = -INFINITY;
    double scale = 1.0 / sqrt((double)d);
    for (int i = 0; i < n; i++) {
        double s = 0.0;
        for (int j = 0; j < d; j++) s += q[j] * k[(size_t)i * d + j];
        l[i] = s * scale;
        if (l[i] > m) m = l[i];
    }
    double z = 0.0;
    for (int j = 0; j < d; j++) out[j] = 0.0;
    for (int i = 0; i < n; i++) {
        double w = exp(l[i] - m);
        z += w;
        for (int j = 0; j < d; j++) out[j] += w * v[(size_t)i * d + j];
    }
    for (int j = 0; j < d; j++) out[j] /= z;
    free(l);
}

/* ------------------------------------------------------------------------- */
/* The estimator for a FIXED candidate set (Eq. importance sampling
 * unnormalized P:74-79 == Eq. close form P:133-139, Alg. 1 line P:115):
 *   z_i = q k_i^T / sqrt(d) - log u_i   (i in S),   z_i = q k_i^T/sqrt(d) (i in T)
 *   o   = sum_i e^{z_i - m} v_i / sum_i e^{z_i - m}
 * sel[i]: 0 = not used, 1 = sampled (in S, weight 1/u_i), 2 = static (u = 1).
 * logu[i] used only where sel[i] == 1.  Returns the partial state (m, s, a)
 * too (the "recursive attention" merge state).  Returns 0 if nothing
 * is selected (out = 0, m = -inf, s = 0).                                   */
int oracle_estimate(int n, int d, const uint16_t *q, const uint16_t *k, const uint16_t *v,
                    const uint8_t *sel, const double *logu, double *out, double *m_out,
                    double *s_out, double *a_out) {
    double scale = 1.0 / sqrt((double)d);
    double m = -INFINITY;
    int any = 0;
    double *z = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; i++) {
        if (!sel[i]) continue;
        double s = 0.0;
        for (int j = 0; j < d; j++)
            s += oracle_bf16_to_double(q[j]) * oracle_bf16_to_double(k[(size_t)i * d + j]);
        z[i] = s * scale - (sel[i] == 1 ? logu[i] : 0.0);
        if (z[i] > m) m = z[i];
        any = 1;
    }
    double den = 0.0;
    double *a = (double *)calloc((size_t)d, sizeof(double));
    if (any) {
        for (int i = 0; i < n; i++) {
            if (!sel[i]) continue;
            double w = exp(z[i] - m);
            den += w;
            for (int j = 0; j < d; j++) a[j] += w * oracle_bf16_to_double(v[(size_t)i * d + j]);
        }
    }
    for (int j = 0; j < d; j++) {
        if (out) out[j] = any ? a[j] / den : 0.0;
        if (a_out) a_out[j] = a[j];
    }
    if (m_out) *m_out = m;
    if (s_out) *s_out = den;
    free(a);
    free(z);
    return any;
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1 (MagicPIG Decoding) for one (sequence, kv head) unit
 * and its G query heads (GQA: tables per kv head P:446, S per query head R15).
 *
 * Inputs: k, v [n][d] bf16; q [G][d] bf16; W [(d+mips)][K*L] float.
 * Config: K, L, center, mips, min_collisions, sink, local.
 * Steps:  pre-process keys -> Encode keys (HT build)
 *         -> Encode q -> Query: counts, S = {i in D : cnt >= 2} (P:107,
 *         P:84) -> p, u from the angle between the hashed vectors (P:111-113,
 *         R5) -> estimator over S U T.
 * Outputs (any may be NULL): out [G][d]; partial [G][d+2] = (m, s, a[d]);
 *   s_count [G] (= |S_g|); counts [G][n]; in_s [G][n] (0/1/2 as sel);
 *   codes [n][L]; qcodes [G][L]; c [d]; r2; logu [G][n] (only where in S).
 * Returns OR_OK, OR_EINEXACT (contract violated), OR_ENOTREPR,
 * OR_EDEGENERATE (some head with S and T both empty; its out row is 0).    */
/* Build half of Algorithm 1 (the hash tables HT): pre-processing
 * then Encode of every key.  Outputs xbar
 * [n][d+mips], n2 [n], codes [n][L], c [d], r2.  Returns the transform status. */
int oracle_build_unit(int n, int d, int K, int L, int center, int mips, int sink, int local,
                      const uint16_t *k, const float *W, uint16_t *xbar, double *n2,
                      uint16_t *codes, float *c, double *r2) {
    if (n < 0 || d <= 0 || K < 1 || K > 16 || L < 1) return OR_EINVAL;
    int dp = d + (mips ? 1 : 0);
    int rc = oracle_check_w(W, (int64_t)dp * K * L);
    if (rc) return rc;
    int status = oracle_key_transform(n, d, k, sink, local, center, mips, c, xbar, n2, r2,
                                      NULL, NULL, NULL);
    oracle_encode_keys(n, dp, xbar, W, K, L, codes);
    return status;
}

/* Decode half of Algorithm 1 given the unit's index (xbar, n2,
 * codes from oracle_build_unit) for G query heads.  Outputs as in
 * oracle_decode_unit below.  Returns OR_OK or OR_EDEGENERATE. */
int oracle_decode_indexed(int n, int d, int G, int K, int L, int mips, int min_collisions,
                          int sink, int local, const uint16_t *k, const uint16_t *v,
                          const uint16_t *q, const float *W, const uint16_t *xbar,
                          const double *n2, const uint16_t *codes, double *out, double *partial,
                          int32_t *s_count, int32_t *counts_out, uint8_t *in_s_out,
                          uint16_t *qcodes_out, double *logu_out) {
    if (n < 0 || d <= 0 || G <= 0 || K < 1 || K > 16 || L < 1) return OR_EINVAL;
    if (min_collisions < 1 || min_collisions > L) return OR_EINVAL;
    int dp = d + (mips ? 1 : 0);
    uint16_t *qc = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)L);
    int32_t *cnt = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    uint8_t *sel = (uint8_t *)malloc((size_t)(n > 0 ? n : 1));
    double *logu = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *o = (double *)malloc(sizeof(double) * (size_t)d);
    double *a = (double *)malloc(sizeof(double) * (size_t)d);
    int degenerate = 0;
    for (int g = 0; g < G; g++) {
        const uint16_t *qg = q + (size_t)g * d;
        oracle_encode_query(d, mips, qg, W, K, L, qc);
        oracle_collision_counts(n, L, codes, qc, cnt);
        double qn2 = 0.0;
        for (int j = 0; j < d; j++) qn2 += oracle_bf16_to_double(qg[j]) * oracle_bf16_to_double(qg[j]);
        double qnorm = sqrt(qn2);
        int ns = 0;
        for (int i = 0; i < n; i++) {
            logu[i] = 0.0;
            if (oracle_is_static(i, n, sink, local)) { sel[i] = 2; continue; }
            if (cnt[i] < min_collisions) { sel[i] = 0; continue; }
            sel[i] = 1;
            ns++;
            /* cos between the vectors actually hashed: qbar = [q,0], xbar_i (R5) */
            double dot = 0.0;
            for (int j = 0; j < d; j++)
                dot += oracle_bf16_to_double(qg[j]) * oracle_bf16_to_double(xbar[(size_t)i * dp + j]);
            double xn2 = n2[i];
            if (mips) {
                double s = oracle_bf16_to_double(xbar[(size_t)i * dp + d]);
                xn2 += s * s;
            }
            double den = qnorm * sqrt(xn2);
            double cosv = den > 0.0 ? dot / den : 0.0; /* zero vector: p = 1/2 (R13b) */
            double p = oracle_collision_prob(cosv);
            double u = oracle_sampling_prob(p, K, L, min_collisions);
            if (u < 1e-300) u = 1e-300; /* S:333 floor */
            logu[i] = log(u);
        }
        double m = -INFINITY, s = 0.0;
        int any = oracle_estimate(n, d, qg, k, v, sel, logu, o, &m, &s, a);
        if (!any) degenerate = 1;
        if (out) memcpy(out + (size_t)g * d, o, sizeof(double) * (size_t)d);
        if (partial) {
            partial[(size_t)g * (d + 2) + 0] = m;
            partial[(size_t)g * (d + 2) + 1] = s;
            memcpy(partial + (size_t)g * (d + 2) + 2, a, sizeof(double) * (size_t)d);
        }
        if (s_count) s_count[g] = ns;
        if (counts_out) memcpy(counts_out + (size_t)g * n, cnt, sizeof(int32_t) * (size_t)n);
        if (in_s_out) memcpy(in_s_out + (size_t)g * n, sel, (size_t)n);
        if (qcodes_out) memcpy(qcodes_out + (size_t)g * L, qc, sizeof(uint16_t) * (size_t)L);
        if (logu_out) memcpy(logu_out + (size_t)g * n, logu, sizeof(double) * (size_t)n);
    }
    free(qc); free(cnt); free(sel); free(logu); free(o); free(a);
    return degenerate ? OR_EDEGENERATE : OR_OK;
}

/* Algorithm 1 end to end for one unit: oracle_build_unit + oracle_decode_indexed. */
int oracle_decode_unit(int n, int d, int G, int K, int L, int center, int mips,
                       int min_collisions, int sink, int local, const uint16_t *k,
                       const uint16_t *v, const uint16_t *q, const float *W, double *out,
                       double *partial, int32_t *s_count, int32_t *counts_out,
                       uint8_t *in_s_out, uint16_t *codes_out, uint16_t *qcodes_out,
                       float *c_out, double *r2_out, double *logu_out) {
    if (n < 0 || d <= 0 || G <= 0 || K < 1 || K > 16 || L < 1) return OR_EINVAL;
    if (min_collisions < 1 || min_collisions > L) return OR_EINVAL;
    int dp = d + (mips ? 1 : 0);
    float *c = (float *)malloc(sizeof(float) * (size_t)d);
    uint16_t *xbar = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(n > 0 ? n : 1) * dp);
    double *n2 = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    uint16_t *codes = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(n > 0 ? n : 1) * L);
    double r2 = 0.0;
    int status = oracle_build_unit(n, d, K, L, center, mips, sink, local, k, W, xbar, n2, codes, c, &r2);
    if (status == OR_ENOTREPR || status == OR_EINVAL) {
        free(c); free(xbar); free(n2); free(codes);
        return status;
    }
    int rc = oracle_decode_indexed(n, d, G, K, L, mips, min_collisions, sink, local, k, v, q, W,
                                   xbar, n2, codes, out, partial, s_count, counts_out, in_s_out,
                                   qcodes_out, logu_out);
    if (codes_out) memcpy(codes_out, codes, sizeof(uint16_t) * (size_t)n * L);
    if (c_out) memcpy(c_out, c, sizeof(float) * (size_t)d);
    if (r2_out) *r2_out = r2;
    free(c); free(xbar); free(n2); free(codes);
    if (status) return status;
    return rc;
}

/* Merge of partial softmax states ("recursive attention"):
 *   M = max_j m_j, S = sum_j s_j e^{m_j - M}, A = sum_j a_j e^{m_j - M}, o = A/S.
 * parts: [P][d+2]; out: [d].  Returns 0 if all parts are empty. */
int oracle_merge_partials(int P, int d, const double *parts, double *out) {
    double M = -INFINITY;
    for (int j = 0; j < P; j++)
        if (parts[(size_t)j * (d + 2)] > M) M = parts[(size_t)j * (d + 2)];
    for (int t = 0; t < d; t++) out[t] = 0.0;
    if (M == -INFINITY) return 0;
    double S = 0.0;
    for (int j = 0; j < P; j++) {
        double mj = parts[(size_t)j * (d + 2)];
        if (mj == -INFINITY) continue;
        double f = exp(mj - M);
        S += parts[(size_t)j * (d + 2) + 1] * f;
        for (int t = 0; t < d; t++) out[t] += parts[(size_t)j * (d + 2) + 2 + t] * f;
    }
    for (int t = 0; t < d; t++) out[t] /= S;
    return 1;
}

/* ------------------------------------------------------------------------- */
/* Estimator-quality harness: the estimators the paper
 * compares, over a normalized attention distribution w [n] (sum 1) and values
 * v [n][d], all in double (o = wV).                               */

/* w = Softmax(x). */
void oracle_softmax_f64(int n, const double *x, double *w) {
    double m = -INFINITY, z = 0.0;
    for (int i = 0; i < n; i++)
        if (x[i] > m) m = x[i];
    for (int i = 0; i < n; i++) {
        w[i] = exp(x[i] - m);
        z += w[i];
    }
    for (int i = 0; i < n; i++) w[i] /= z;
}

/* Exact output o = wV. */
void oracle_expectation(int n, int d, const double *w, const double *v, double *out) {
    for (int j = 0; j < d; j++) out[j] = 0.0;
    for (int i = 0; i < n; i++)
        for (int j = 0; j < d; j++) out[j] += w[i] * v[(size_t)i * d + j];
}

/* TopK attention: the m indices r_1..r_m with the largest w (ties:
 * lower index first), o = sum_j w_{r_j} v_{r_j} / sum_j w_{r_j}.  Returns m. */
int oracle_topk_estimate(int n, int d, const double *w, const double *v, int m, double *out) {
    if (m > n) m = n;
    if (m < 0) m = 0;
    unsigned char *taken = (unsigned char *)calloc((size_t)(n > 0 ? n : 1), 1);
    double den = 0.0;
    for (int j = 0; j < d; j++) out[j] = 0.0;
    for (int r = 0; r < m; r++) { /* plain selection: the largest untaken weight */
        int best = -1;
        for (int i = 0; i < n; i++)
            if (!taken[i] && (best < 0 || w[i] > w[best])) best = i;
        taken[best] = 1;
        den += w[best];
        for (int j = 0; j < d; j++) out[j] += w[best] * v[(size_t)best * d + j];
    }
    for (int j = 0; j < d; j++) out[j] = den > 0.0 ? out[j] / den : 0.0;
    free(taken);
    return m;
}

/* Oracle sampling estimation (Definition): B indices drawn iid from
 * w -- draw j is the first index whose cumulative weight exceeds uniforms[j]
 * (uniforms in [0, 1), supplied by the caller) -- and o = (1/B) sum_j v_{i_j}
 * = sum_{i in S} (f_i / B) v_i.  Returns |S| (unique draws). */
int oracle_oracle_sampling(int n, int d, const double *w, const double *v, int B, const double *uniforms,
                           double *out) {
    double *cdf = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int *f = (int *)calloc((size_t)(n > 0 ? n : 1), sizeof(int));
    double c = 0.0;
    for (int i = 0; i < n; i++) {
        c += w[i];
        cdf[i] = c;
    }
    for (int b = 0; b < B; b++) {
        int lo = 0, hi = n - 1; /* first i with cdf[i] > u (the last index if rounding leaves u >= cdf) */
        while (lo < hi) {
            int mid = (lo + hi) / 2;
            if (cdf[mid] > uniforms[b]) hi = mid;
            else lo = mid + 1;
        }
        f[lo]++;
    }
    int uniq = 0;
    for (int j = 0; j < d; j++) out[j] = 0.0;
    for (int i = 0; i < n; i++) {
        if (!f[i]) continue;
        uniq++;
        for (int j = 0; j < d; j++) out[j] += ((double)f[i] / (double)B) * v[(size_t)i * d + j];
    }
    free(cdf);
    free(f);
    return uniq;
}

/* Theorem 1: the oracle-sampling estimate is unbiased with per-
 * coordinate variance Var_w(v_j) / B; std[j] = sqrt((E_w[v_j^2] - E_w[v_j]^2) / B). */
void oracle_oracle_sampling_std(int n, int d, const double *w, const double *v, int B, double *std) {
    for (int j = 0; j < d; j++) {
        double m1 = 0.0, m2 = 0.0;
        for (int i = 0; i < n; i++) {
            const double x = v[(size_t)i * d + j];
            m1 += w[i] * x;
            m2 += w[i] * x * x;
        }
        const double var = m2 - m1 * m1;
        std[j] = sqrt((var > 0.0 ? var : 0.0) / (double)B);
    }
}

/* Theorem 2: E|S| = sum_i (1 - (1 - w_i)^B) (each index is absent
 * from B iid draws with probability (1 - w_i)^B), bounded by 1 + B (1 - max_i w_i). */
double oracle_expected_unique(int n, const double *w, int B) {
    double e = 0.0;
    for (int i = 0; i < n; i++) e += -expm1((double)B * log1p(-w[i]));
    return e;
}

/* ------------------------------------------------------------------------- */
/* Decode-time append (P:171 on-device local window, P:619
 * 64 local tokens): a new key is hashed with the index's FROZEN centering
 * vector c and MIPS radius r^2 (reading R3: c and r are taken over D at build
 * time; an appended key with |x|^2 > r^2 gets s = 0, i.e. r^2 - n2 clamped at
 * 0), exactly as oracle_key_transform + oracle_encode_keys do for built keys:
 *   x = bf16_rn(fl32(k - c)),  n2q = sum_d q(x_d^2),
 *   s = bf16_rn(sqrt_rn(fl64(max(r2q - n2q, 0) 2^-64)))   (mips),
 *   codes = SimHash of xbar = [x, s].
 * r2_q: the frozen radius as the (lo, hi) int128 pair of oracle_key_transform.
 * Outputs xbar [m][d+mips], n2 [m] (= fl64(n2q 2^-64)), codes [m][L].  The
 * token leaving the local window becomes a dynamic key by position alone
 * (oracle_is_static with the new n), its code already exists (R16).        */
int oracle_append_keys(int m, int d, int K, int L, int mips, const uint16_t *k_new, const float *W,
                       const float *c, const uint64_t *r2_q, uint16_t *xbar, double *n2, uint16_t *codes) {
    if (m < 0 || d <= 0 || K < 1 || K > 16 || L < 1) return OR_EINVAL;
    int dp = d + (mips ? 1 : 0);
    int rc = oracle_check_w(W, (int64_t)dp * K * L);
    if (rc) return rc;
    const i128 r2q = (i128)(((unsigned __int128)r2_q[1] << 64) | (unsigned __int128)r2_q[0]);
    int inexact = 0;
    for (int i = 0; i < m; i++) {
        i128 acc = 0;
        for (int j = 0; j < d; j++) {
            double kv = oracle_bf16_to_double(k_new[(size_t)i * d + j]);
            if (fabs(kv) >= ABS_LIMIT) inexact = 1;
            double hi, lo;
            two_sum(kv, -(double)c[j], &hi, &lo);
            uint16_t xb = oracle_bf16_from_double((double)f32_round_pair(hi, lo));
            xbar[(size_t)i * dp + j] = xb;
            double xv = oracle_bf16_to_double(xb);
            if (fabs(xv) >= ABS_LIMIT) inexact = 1;
            acc += fix_of(xv * xv);
        }
        n2[i] = oracle_fix_to_double(acc);
        if (mips) {
            double diff = r2q > acc ? oracle_fix_to_double(r2q - acc) : 0.0;
            xbar[(size_t)i * dp + d] = oracle_bf16_from_double(sqrt(diff));
        }
    }
    oracle_encode_keys(m, dp, xbar, W, K, L, codes);
    return inexact ? OR_EINEXACT : OR_OK;
}
