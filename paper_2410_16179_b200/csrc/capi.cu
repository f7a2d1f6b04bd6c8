// capi.cu -- the C ABI (include/magicpig.h): validation, workspace layout,
// launch sequencing.  No allocation; process-wide state: a launch counter and the debug kernel selector.
#include <atomic>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

namespace mp {

static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

static inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

static int max_smem_optin() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || n <= 0)
            n = 227 * 1024;
    }
    return n;
}

// decode kernel selection (debug knob, magicpig_debug_set_decode_kernel; see magicpig.h): 0 = automatic
// (5 for small decodes, else 7), 4..8 = a specific kernel generation (A/B arms); all compute the same S
// bit for bit.
static std::atomic<int> g_decode_kernel{0};
// the auto choice for decodes larger than two chunk tiles per SM (A/B-selected on B200)
constexpr int LARGE_KVER = 9;

static bool cfg_ok(const magicpig_config* c) {
    if (!c) return false;
    if (c->head_dim != HD) return false;
    if (c->K < 1 || c->K > 16) return false;
    if (c->L < 1 || c->L > 1024) return false;
    if (c->min_collisions < 1 || c->min_collisions > 2 || c->L < c->min_collisions) return false;
    if (c->center < 0 || c->center > 1 || c->mips < 0 || c->mips > 1) return false;
    if (c->sink < 0 || c->local < 0) return false;
    return true;
}

// bucketed tables: 2^K-entry histogram in shared memory, n-bit seen bitmaps per head in shared memory
static bool buckets_ok(const magicpig_config* c, int64_t n_local) {
    return cfg_ok(c) && c->K <= 14 && (size_t)((n_local + 31) / 32) * 8 <= 200 * 1024;
}

static bool shape_ok(int64_t B, int64_t Hkv, int64_t n_local, int64_t seq_offset, int64_t n_global) {
    if (B < 1 || Hkv < 1 || n_local < 0 || seq_offset < 0) return false;
    if (seq_offset + n_local > n_global) return false;
    if (n_local > ((int64_t)1 << 31) - KCHUNK) return false;
    return true;
}

// ---------------------------------------------------------------- layouts
struct BuildWs {
    uint32_t* status;
    float* wmax;
    uint32_t* fix_count;
    int64_t* part_sum;
    int64_t* part_cnt;
    int64_t* part_r2;
    uint8_t* xt;
    float* xnorm;
    uint8_t* wt;
    uint2* fix_list;
    uint32_t fix_cap;
    int64_t n_pad;
    int nsplit, KD, NT;
    size_t bytes;
};

static BuildWs build_layout(const magicpig_config* c, int64_t B, int64_t Hkv, int64_t n_local, void* base) {
    BuildWs w;
    memset(&w, 0, sizeof(w));
    const Geom g = make_geom(c->K, c->L, n_local);
    const int64_t units = B * Hkv;
    w.n_pad = ((n_local + KCHUNK - 1) / KCHUNK) * KCHUNK;
    w.nsplit = (int)((n_local + STATS_SPLIT - 1) / STATS_SPLIT);
    if (w.nsplit < 1) w.nsplit = 1;
    w.KD = c->mips ? 144 : 128;
    int cols = g.KL > g.KLq * 4 ? g.KL : g.KLq * 4;
    w.NT = (cols + HG_N - 1) / HG_N;
    int64_t dots = units * w.n_pad * (int64_t)w.NT * HG_N;
    int64_t cap = dots / 512;
    if (cap < 65536) cap = 65536;
    if (cap > 0x7fffffffLL) cap = 0x7fffffffLL;
    w.fix_cap = (uint32_t)cap;
    uint8_t* p = (uint8_t*)base;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* r = p ? p + off : nullptr;
        off += align256(bytes);
        return r;
    };
    uint8_t* hdr = take(256);
    w.status = (uint32_t*)hdr;
    w.wmax = hdr ? (float*)(hdr + 4) : nullptr;
    w.fix_count = hdr ? (uint32_t*)(hdr + 8) : nullptr;
    w.part_sum = (int64_t*)take((size_t)units * w.nsplit * HD * 16);
    w.part_cnt = (int64_t*)take((size_t)units * w.nsplit * 8);
    w.part_r2 = (int64_t*)take((size_t)units * w.nsplit * 16);
    w.xt = take((size_t)units * w.n_pad * w.KD * 2);
    w.xnorm = (float*)take((size_t)units * w.n_pad * 4);
    w.wt = take((size_t)w.NT * HG_N * w.KD * 2);
    w.fix_list = (uint2*)take((size_t)w.fix_cap * 8);
    w.bytes = off;
    return w;
}

struct DecodeWs {
    uint32_t* status;
    float* lutab;
    uint32_t* qbits;
    uint32_t* unit_ctr;
    float* parts;
    int32_t* chunk_cnt;
    uint32_t* sbits;
    uint32_t* ents;
    int32_t* pcnt;
    int32_t* hpc;
    int2* urec;
    uint16_t* qstage;  // magicpig_decode_host: q copied from the host
    float* ostage;     //                       out before the copy to the host
    size_t bytes;
};

static DecodeWs decode_layout(const magicpig_config* c, int64_t B, int64_t Hq, int64_t Hkv, int64_t n_local,
                              void* base) {
    DecodeWs w;
    memset(&w, 0, sizeof(w));
    const Geom g = make_geom(c->K, c->L, n_local);
    const int64_t units = B * Hkv;
    const int64_t G = Hq / Hkv;
    const int64_t nch = g.nchunks > 0 ? g.nchunks : 1;
    uint8_t* p = (uint8_t*)base;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        uint8_t* r = p ? p + off : nullptr;
        off += align256(bytes);
        return r;
    };
    w.status = (uint32_t*)take(256);
    w.lutab = (float*)take((size_t)LUT_WORDS * 4);
    w.qbits = (uint32_t*)take((size_t)B * Hq * g.KLw * 4);
    w.unit_ctr = (uint32_t*)take((size_t)units * 4);
    const int64_t nT = n_local < (int64_t)c->sink + c->local ? n_local : (int64_t)c->sink + c->local;
    const int64_t nst = nT > 0 ? (nT + KCHUNK - 1) / KCHUNK : 1;
    const size_t parts4 = (size_t)units * (nch + nst) * 8 * G * PART * 4;      // up to 8 CTAs per cluster
    const size_t parts5 = (size_t)(units + (int64_t)num_sms() * EST_MAX_WARPS) * G * PREC5 * 4;  // record u + warp
    w.parts = (float*)take(parts4 > parts5 ? parts4 : parts5);
    w.chunk_cnt = (int32_t*)take((size_t)units * nch * G * 4);
    w.sbits = (uint32_t*)take((size_t)B * Hq * ((n_local + 31) / 32) * 4 * 2 * BM_PARTS);  // Query step output
    w.ents = (uint32_t*)take((size_t)units * nch * KCHUNK * 4);  // v7 piece lists
    w.pcnt = (int32_t*)take((size_t)units * nch * 4);
    w.hpc = (int32_t*)take((size_t)B * Hq * nch * 4);
    w.urec = (int2*)take((size_t)units * 8);
    w.qstage = (uint16_t*)take((size_t)B * Hq * HD * 2);
    w.ostage = (float*)take((size_t)B * Hq * HD * 4);
    w.bytes = off;
    return w;
}

static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

}  // namespace mp

using namespace mp;

extern "C" {

int magicpig_validate_config(const magicpig_config* cfg) { return cfg_ok(cfg) ? MAGICPIG_OK : MAGICPIG_EINVAL; }

size_t magicpig_codes_words(const magicpig_config* cfg, int64_t B, int64_t Hkv, int64_t n_local) {
    if (!cfg_ok(cfg) || B < 1 || Hkv < 1 || n_local < 0) return 0;
    const Geom g = make_geom(cfg->K, cfg->L, n_local);
    return (size_t)(B * Hkv) * (size_t)g.nchunks * (size_t)g.KLq * 128;
}

size_t magicpig_build_workspace_bytes(const magicpig_config* cfg, int64_t B, int64_t Hkv, int64_t n_local) {
    if (!cfg_ok(cfg) || B < 1 || Hkv < 1 || n_local < 0) return 0;
    return build_layout(cfg, B, Hkv, n_local, nullptr).bytes;
}

size_t magicpig_decode_workspace_bytes(const magicpig_config* cfg, int64_t B, int64_t Hq, int64_t Hkv,
                                       int64_t n_local) {
    if (!cfg_ok(cfg) || B < 1 || Hkv < 1 || Hq < Hkv || Hq % Hkv || n_local < 0) return 0;
    return decode_layout(cfg, B, Hq, Hkv, n_local, nullptr).bytes;
}

int magicpig_workspace_init(void* ws, size_t ws_bytes, void* stream) {
    if (!ws) return MAGICPIG_EINVAL;
    return cudaMemsetAsync(ws, 0, ws_bytes, S(stream)) == cudaSuccess ? MAGICPIG_OK : MAGICPIG_ECUDA;
}

int magicpig_workspace_status(void* ws, uint32_t* status, void* stream) {
    if (!ws || !status) return MAGICPIG_EINVAL;
    if (cudaMemcpyAsync(status, ws, 4, cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess) return MAGICPIG_ECUDA;
    if (cudaMemsetAsync(ws, 0, 4, S(stream)) != cudaSuccess) return MAGICPIG_ECUDA;
    return cudaStreamSynchronize(S(stream)) == cudaSuccess ? MAGICPIG_OK : MAGICPIG_ECUDA;
}

int magicpig_key_stats(const magicpig_config* cfg, const uint16_t* k, int64_t B, int64_t Hkv, int64_t n_local,
                       int64_t seq_offset, int64_t n_global, int64_t* key_sum, int64_t* count, void* ws,
                       size_t ws_bytes, void* stream) {
    if (!cfg_ok(cfg) || !shape_ok(B, Hkv, n_local, seq_offset, n_global)) return MAGICPIG_EINVAL;
    if (!key_sum || !count || !ws || (n_local > 0 && !k)) return MAGICPIG_EINVAL;
    BuildWs w = build_layout(cfg, B, Hkv, n_local, ws);
    if (ws_bytes < w.bytes) return MAGICPIG_EWORKSPACE;
    return launch_key_stats(k, B * Hkv, n_local, seq_offset, n_global, cfg->sink, cfg->local, w.part_sum,
                            w.part_cnt, key_sum, count, w.status, S(stream));
}

int magicpig_key_norms(const magicpig_config* cfg, const uint16_t* k, int64_t B, int64_t Hkv, int64_t n_local,
                       int64_t seq_offset, int64_t n_global, const int64_t* key_sum, const int64_t* count,
                       float* center, int64_t* r2, void* ws, size_t ws_bytes, void* stream) {
    if (!cfg_ok(cfg) || !shape_ok(B, Hkv, n_local, seq_offset, n_global)) return MAGICPIG_EINVAL;
    if (!key_sum || !count || !center || !r2 || !ws || (n_local > 0 && !k)) return MAGICPIG_EINVAL;
    BuildWs w = build_layout(cfg, B, Hkv, n_local, ws);
    if (ws_bytes < w.bytes) return MAGICPIG_EWORKSPACE;
    return launch_key_norms(k, B * Hkv, n_local, seq_offset, n_global, cfg->sink, cfg->local, cfg->center, key_sum,
                            count, center, w.part_r2, r2, w.status, S(stream));
}

int magicpig_reduce_stats(int mode, const int64_t* parts_sum, const int64_t* parts_cnt, int P, int64_t B,
                          int64_t Hkv, int64_t* out_sum, int64_t* out_cnt, void* stream) {
    if ((mode != 0 && mode != 1) || P < 1 || B < 1 || Hkv < 1 || !parts_sum || !out_sum) return MAGICPIG_EINVAL;
    if (mode == 0 && (!parts_cnt || !out_cnt)) return MAGICPIG_EINVAL;
    return launch_reduce_shards(mode, parts_sum, parts_cnt, P, B * Hkv, out_sum, out_cnt, S(stream));
}

int magicpig_build_tables(const magicpig_config* cfg, const uint16_t* k, int64_t B, int64_t Hkv, int64_t n_local,
                          int64_t seq_offset, int64_t n_global, const float* W, const float* center,
                          const int64_t* r2, uint32_t* codes, float* key_norm, void* ws, size_t ws_bytes,
                          void* stream) {
    if (!cfg_ok(cfg) || !shape_ok(B, Hkv, n_local, seq_offset, n_global)) return MAGICPIG_EINVAL;
    if (!W || !center || !r2 || !codes || !ws || (n_local > 0 && (!k || !key_norm))) return MAGICPIG_EINVAL;
    BuildWs w = build_layout(cfg, B, Hkv, n_local, ws);
    if (ws_bytes < w.bytes) return MAGICPIG_EWORKSPACE;
    if (n_local == 0) return MAGICPIG_OK;
    const Geom g = make_geom(cfg->K, cfg->L, n_local);
    cudaStream_t st = S(stream);
    if (cudaMemsetAsync(w.fix_count, 0, 4, st) != cudaSuccess) return MAGICPIG_ECUDA;
    int rc = launch_prep(k, B * Hkv, n_local, w.n_pad, cfg->mips, w.KD, center, r2, w.xt, w.xnorm, key_norm, W,
                         g.KL, w.NT, w.wt, w.wmax, w.status, st);
    if (rc) return rc;
    return launch_hash_gemm(w.xt, w.wt, w.xnorm, w.wmax, codes, w.fix_list, w.fix_count, w.fix_cap, B * Hkv,
                            n_local, w.n_pad, g.nchunks, w.KD, g.KL, w.NT, g.KLq, w.status, nullptr, st);
}

int magicpig_append_keys(const magicpig_config* cfg, const uint16_t* k_new, int64_t m, int64_t B, int64_t Hkv,
                         int64_t n_old, const float* W, const float* center, const int64_t* r2, uint32_t* codes,
                         float* key_norm, void* ws, size_t ws_bytes, void* stream) {
    if (!cfg_ok(cfg) || m < 0 || B < 1 || Hkv < 1 || n_old < 0 || !shape_ok(B, Hkv, n_old + m, 0, n_old + m))
        return MAGICPIG_EINVAL;
    if (m > 0 && (!k_new || !W || !center || !r2 || !codes || !key_norm || !ws || ws_bytes < 4)) return MAGICPIG_EINVAL;
    const Geom g = make_geom(cfg->K, cfg->L, n_old + m);
    return launch_append_keys(k_new, m, B * Hkv, n_old, cfg->mips, W, g.KL, g.KLq, g.nchunks, center, r2, codes,
                              key_norm, (uint32_t*)ws, S(stream));
}

int magicpig_build_index(const magicpig_config* cfg, const uint16_t* k, int64_t B, int64_t Hkv, int64_t n,
                         const float* W, float* center, int64_t* r2, uint32_t* codes, float* key_norm,
                         int64_t* key_sum, int64_t* count, void* ws, size_t ws_bytes, void* stream) {
    int rc = magicpig_key_stats(cfg, k, B, Hkv, n, 0, n, key_sum, count, ws, ws_bytes, stream);
    if (rc) return rc;
    rc = magicpig_key_norms(cfg, k, B, Hkv, n, 0, n, key_sum, count, center, r2, ws, ws_bytes, stream);
    if (rc) return rc;
    return magicpig_build_tables(cfg, k, B, Hkv, n, 0, n, W, center, r2, codes, key_norm, ws, ws_bytes, stream);
}

int magicpig_encode_queries(const magicpig_config* cfg, const uint16_t* q, int64_t B, int64_t Hq, const float* W,
                            void* ws, size_t ws_bytes, void* stream) {
    if (!cfg_ok(cfg) || B < 1 || Hq < 1 || !q || !W || !ws) return MAGICPIG_EINVAL;
    // the query-code region sits at the same offset in every decode workspace
    DecodeWs w = decode_layout(cfg, B, Hq, 1, 0, ws);
    const Geom g = make_geom(cfg->K, cfg->L, 0);
    if (ws_bytes < (size_t)((uint8_t*)w.qbits - (uint8_t*)ws) + (size_t)B * Hq * g.KLw * 4) return MAGICPIG_EWORKSPACE;
    return launch_qencode(q, B * Hq, W, g.KL, g.KLw, w.qbits, w.status, S(stream), cfg->K, cfg->L,
                          cfg->min_collisions, w.lutab);
}

static int decode_impl(const magicpig_config* cfg, const uint16_t* q, int64_t Hq, const uint32_t* codes,
                       const float* center, const float* key_norm, const uint16_t* k, const uint16_t* v, int64_t B,
                       int64_t Hkv, int64_t n_local, int64_t seq_offset, int64_t n_global, float* out,
                       float* partial, int32_t* s_count, uint32_t* s_mask, void* ws, size_t ws_bytes,
                       void* stream, unsigned long long* timeline, int64_t timeline_len, int64_t* grid_out,
                       const int32_t* tables = nullptr, uint32_t* weighted = nullptr, int stages = 7,
                       int force_kver = -1) {
    if (!cfg_ok(cfg) || !shape_ok(B, Hkv, n_local, seq_offset, n_global)) return MAGICPIG_EINVAL;
    if (Hq < Hkv || Hq % Hkv) return MAGICPIG_EINVAL;
    const int64_t G = Hq / Hkv;
    if (G != 1 && G != 2 && G != 4 && G != 8) return MAGICPIG_EINVAL;
    if (!q || !center || !ws) return MAGICPIG_EINVAL;
    if (n_local > 0 && !key_norm) return MAGICPIG_EINVAL;
    if (n_local > 0 && ((!codes && !tables) || !k || !v)) return MAGICPIG_EINVAL;
    if (tables && !buckets_ok(cfg, n_local)) return MAGICPIG_EINVAL;
    DecodeWs w = decode_layout(cfg, B, Hq, Hkv, n_local, ws);
    if (ws_bytes < w.bytes) return MAGICPIG_EWORKSPACE;
    cudaStream_t st = S(stream);
    const Geom g = make_geom(cfg->K, cfg->L, n_local);
    if (n_local == 0) {
        // nothing on this shard: empty partial states, zero outputs
        if (partial) {
            int rc0 = launch_empty_partial(partial, B * Hq, st);
            if (rc0) return rc0;
        }
        if (out && cudaMemsetAsync(out, 0, (size_t)B * Hq * HD * 4, st) != cudaSuccess) return MAGICPIG_ECUDA;
        if (s_count && cudaMemsetAsync(s_count, 0, (size_t)B * Hq * 4, st) != cudaSuccess) return MAGICPIG_ECUDA;
        return MAGICPIG_OK;
    }
    DecodeArgs a;
    memset(&a, 0, sizeof(a));
    a.q = q;
    a.qbits = w.qbits;
    a.codes = codes;
    a.center = center;
    a.key_norm = key_norm;
    a.k = k;
    a.v = v;
    a.B = B;
    a.Hkv = Hkv;
    a.Hq = Hq;
    a.n_local = n_local;
    a.seq_offset = seq_offset;
    a.n_global = n_global;
    a.K = cfg->K;
    a.L = cfg->L;
    a.KL = g.KL;
    a.KLw = g.KLw;
    a.KLq = g.KLq;
    a.ngroups = g.ngroups;
    a.TG = g.TG;
    a.QG = g.QG;
    a.nchunks = g.nchunks;
    {   // static keys T on this shard -> pieces of <= 1024 keys, one cluster each
        const int64_t lo1 = 0 > -seq_offset ? 0 : -seq_offset;
        const int64_t hi1 = n_local < (int64_t)cfg->sink - seq_offset ? n_local : (int64_t)cfg->sink - seq_offset;
        int64_t lo2 = n_global - cfg->local - seq_offset;
        if (lo2 < 0) lo2 = 0;
        const int64_t hi2 = n_local < n_global - seq_offset ? n_local : n_global - seq_offset;
        const int64_t len1 = hi1 > lo1 ? hi1 - lo1 : 0;
        if (len1 > 0 && lo2 < hi1) lo2 = hi1;
        const int64_t len2 = hi2 > lo2 ? hi2 - lo2 : 0;
        const int64_t nT = len1 + len2;
        a.nstatic = nT > 0 ? (nT + KCHUNK - 1) / KCHUNK : 1;
    }
    // cluster size: smallest power of two (<= 8) giving >= 1.5 CTAs per SM, with
    // at least 8 table groups (one per warp) per CTA
    const int64_t total = B * Hkv * g.nchunks;
    int ts = 1;
    while (ts < 8 && total * ts * 2 < 3 * (int64_t)num_sms() && g.ngroups / (2 * ts) >= DEC_THREADS / 32) ts *= 2;
    a.tsplit = ts;
    a.sink = cfg->sink;
    a.local = cfg->local;
    a.minc = cfg->min_collisions;
    a.out = out;
    a.partial = partial;
    a.s_count = s_count;
    a.s_mask = s_mask;
    a.unit_ctr = w.unit_ctr;
    a.parts = w.parts;
    a.chunk_cnt = w.chunk_cnt;
    a.status = w.status;
    int kver = force_kver >= 0 ? force_kver : g_decode_kernel.load();
    if (kver == 0) {
        // auto (default): small decodes (at most two 1024-key chunk tiles per SM) are latency-bound -> the
        // persistent fused kernel 5 (one launch after the encode); larger ones -> kernel 7 (Query kernel,
        // select, the balanced estimator, the unit merge), which scales with the sampled rows
        DecodeArgs t = a;
        const bool small = B * Hkv * g.nchunks <= 2 * (int64_t)num_sms() && decode5_layout(t, (int)G, max_smem_optin());
        kver = small ? 5 : LARGE_KVER;
    }
    if (kver % 10 == 9 && timeline) kver = 7;  // kernel 9 keeps no timeline
    if ((kver % 10 == 6 && !timeline) || kver % 10 == 7 || kver % 10 == 8 || kver % 10 == 9) {
        const bool v7 = (kver % 10 == 7 || kver % 10 == 8 || kver % 10 == 9) && B * Hkv * (g.nchunks + 1) <= EST_MAX_PIECES &&
                        n_local < (1 << 24);
        EstArgs ea;
        memset(&ea, 0, sizeof(ea));
        ea.q = q, ea.center = center, ea.key_norm = key_norm, ea.k = k, ea.v = v, ea.sbits = w.sbits;
        ea.B = B, ea.Hkv = Hkv, ea.Hq = Hq, ea.n_local = n_local, ea.seq_offset = seq_offset;
        ea.n_global = n_global, ea.nchunks = g.nchunks;
        ea.K = cfg->K, ea.L = cfg->L, ea.minc = cfg->min_collisions, ea.sink = cfg->sink, ea.local = cfg->local;
        ea.ents = w.ents, ea.pcnt = w.pcnt, ea.hpc = w.hpc, ea.s_mask = s_mask, ea.weighted = weighted;
        ea.out = out, ea.partial = partial, ea.s_count = s_count;
        ea.unit_ctr = w.unit_ctr, ea.parts = w.parts, ea.status = w.status, ea.urec = w.urec;
        ea.lutab = w.lutab;
        ea.sparts = (v7 && tables) ? BM_PARTS : 1;
        const bool fused = v7 && !tables;  // the dense scan emits the piece lists itself
        // Query(HT, q_code) -> S bitmaps: bucketed tables or the dense code scan (PDL after the encode)
        int rc = 0;
        if (!(stages & 1)) {
        } else if (tables) {
            rc = launch_bucket_mark(w.qbits, tables, B, Hq, Hkv, n_local, cfg->K, cfg->L, g.KLw,
                                    cfg->min_collisions, w.sbits, st, v7 ? BM_PARTS : 1);
        } else {
            ScanArgs sa;
            memset(&sa, 0, sizeof(sa));
            sa.qbits = w.qbits;
            sa.codes = codes;
            sa.sbits = w.sbits;
            sa.B = B, sa.Hkv = Hkv, sa.Hq = Hq, sa.n_local = n_local, sa.nchunks = g.nchunks;
            sa.tiles = B * Hkv * g.nchunks;
            sa.K = cfg->K, sa.L = cfg->L, sa.KL = g.KL, sa.KLw = g.KLw, sa.KLq = g.KLq, sa.ngroups = g.ngroups;
            sa.minc = cfg->min_collisions;
            if (fused) sa.fuse = 1, sa.est = ea;
            rc = launch_scan6(sa, num_sms(), max_smem_optin(), st);
        }
        if (rc || !(stages & 6)) return rc;
        if (v7) {
            // ordered S_g u ... lists per unit, then the balanced estimator and the unit merge
            if (grid_out) *grid_out = (int64_t)num_sms() * EST_WARPS;  // timeline rows (one per warp)
            if (timeline) {
                const size_t rows = (size_t)num_sms() * EST_WARPS;
                if (timeline_len < (int64_t)rows * 16) return MAGICPIG_EINVAL;
                if (cudaMemsetAsync(timeline, 0, rows * 16 * 8, st) != cudaSuccess) return MAGICPIG_ECUDA;
                ea.timeline = timeline;
            }
            if ((stages & 2) && !fused) rc = launch_select(ea, st);
            if (rc || !(stages & 4)) return rc;
            // kernel 8: the tcgen05 estimator (TMA gather4 tiles) when its layout fits, else kernel 7's
            if (kver % 10 == 8 && estimate8_ok(ea, max_smem_optin())) {
                if (grid_out) *grid_out = num_sms();  // timeline rows (one per CTA)
                rc = launch_estimate8(ea, num_sms(), max_smem_optin(), st);
            } else if (kver % 10 == 9) {
                rc = launch_estimate9(ea, num_sms(), max_smem_optin(), st);
            } else {
                rc = launch_estimate(ea, num_sms(), max_smem_optin(), st);
            }
            return rc ? rc : launch_est_merge(ea, st);
        }
        // estimator over S_g u T
        AttendArgs aa;
        memset(&aa, 0, sizeof(aa));
        aa.q = q, aa.center = center, aa.key_norm = key_norm, aa.k = k, aa.v = v, aa.sbits = w.sbits;
        aa.B = B, aa.Hkv = Hkv, aa.Hq = Hq, aa.n_local = n_local, aa.seq_offset = seq_offset;
        aa.n_global = n_global, aa.nchunks = g.nchunks, aa.nstatic = a.nstatic;
        aa.tiles = B * Hkv * (g.nchunks + a.nstatic);
        aa.K = cfg->K, aa.L = cfg->L, aa.minc = cfg->min_collisions, aa.sink = cfg->sink, aa.local = cfg->local;
        aa.out = out, aa.partial = partial, aa.s_count = s_count, aa.s_mask = s_mask, aa.weighted = weighted;
        aa.unit_ctr = w.unit_ctr, aa.parts = w.parts, aa.status = w.status;
        if (grid_out) *grid_out = aa.tiles < num_sms() ? aa.tiles : num_sms();
        return launch_attend(aa, num_sms(), max_smem_optin(), st);
    }
    if (weighted || stages != 7) return MAGICPIG_EINVAL;  // v6 / v7 paths only
    bool v5 = kver % 10 == 5 || tables;  // bucket mode runs on the persistent kernel only
    a.dbg = kver / 10;
    if (v5) {
        DecodeArgs t = a;
        v5 = decode5_layout(t, (int)G, max_smem_optin()) != 0;
        if (!v5 && tables) return MAGICPIG_EINVAL;
    }
    if (tables) {  // Query(HT, q_code) on the bucketed tables -> S bitmaps (PDL after the encode)
        int rc = launch_bucket_mark(w.qbits, tables, B, Hq, Hkv, n_local, cfg->K, cfg->L, g.KLw,
                                    cfg->min_collisions, w.sbits, st);
        if (rc) return rc;
        a.sbits = w.sbits;
    }
    const int64_t tiles = B * Hkv * (g.nchunks + a.nstatic);  // one tile per 1024-key chunk
    const int64_t grid = v5 ? (tiles < num_sms() ? tiles : num_sms()) : tiles * a.tsplit;
    if (grid_out) *grid_out = grid;
    if (timeline) {
        if (timeline_len < grid * 32) return MAGICPIG_EINVAL;
        if (cudaMemsetAsync(timeline, 0, (size_t)grid * 32 * 8, st) != cudaSuccess) return MAGICPIG_ECUDA;
        a.timeline = timeline;
    }
    return v5 ? launch_decode5(a, num_sms(), max_smem_optin(), st) : launch_decode(a, st);
}

extern "C" int magicpig_debug_decode_kernel_choice(const magicpig_config* cfg, int64_t B, int64_t Hq, int64_t Hkv,
                                                   int64_t n_local, int buckets) {
    if (!cfg_ok(cfg) || B < 1 || Hkv < 1 || Hq < Hkv || Hq % Hkv || n_local < 1) return MAGICPIG_EINVAL;
    int kver = g_decode_kernel.load();
    const Geom g = make_geom(cfg->K, cfg->L, n_local);
    const int64_t G = Hq / Hkv;
    if (kver == 0) {
        DecodeArgs t;
        memset(&t, 0, sizeof(t));
        t.K = cfg->K, t.L = cfg->L, t.KL = g.KL, t.KLw = g.KLw, t.KLq = g.KLq, t.ngroups = g.ngroups;
        t.TG = g.TG, t.QG = g.QG, t.nchunks = g.nchunks, t.B = B, t.Hkv = Hkv, t.Hq = Hq, t.n_local = n_local;
        const bool small = B * Hkv * g.nchunks <= 2 * (int64_t)num_sms() && decode5_layout(t, (int)G, max_smem_optin());
        kver = small ? 5 : LARGE_KVER;
    }
    (void)buckets;
    return kver % 10;
}

extern "C" int magicpig_debug_set_decode_kernel(int version) {
    if (version != 0 && (version % 10 < 4 || version % 10 > 9)) return MAGICPIG_EINVAL;
    g_decode_kernel.store(version);
    return MAGICPIG_OK;
}

extern "C" int magicpig_decode_encoded(const magicpig_config* cfg, const uint16_t* q, int64_t Hq,
                                       const uint32_t* codes, const float* center, const float* key_norm,
                                       const uint16_t* k, const uint16_t* v, int64_t B, int64_t Hkv, int64_t n_local,
                                       int64_t seq_offset, int64_t n_global, float* out, float* partial,
                                       int32_t* s_count, uint32_t* s_mask, void* ws, size_t ws_bytes, void* stream) {
    return decode_impl(cfg, q, Hq, codes, center, key_norm, k, v, B, Hkv, n_local, seq_offset, n_global, out,
                       partial, s_count, s_mask, ws, ws_bytes, stream, nullptr, 0, nullptr);
}

extern "C" int64_t magicpig_debug_decode_timeline(const magicpig_config* cfg, const uint16_t* q, int64_t Hq,
                                                  const uint32_t* codes, const float* center, const float* key_norm,
                                                  const uint16_t* k, const uint16_t* v, int64_t B, int64_t Hkv,
                                                  int64_t n_local, const float* W, float* out,
                                                  unsigned long long* timeline, int64_t timeline_len, void* ws,
                                                  size_t ws_bytes, void* stream) {
    if (!timeline) return MAGICPIG_EINVAL;
    int rc = magicpig_encode_queries(cfg, q, B, Hq, W, ws, ws_bytes, stream);
    if (rc) return rc;
    int64_t grid = 0;
    rc = decode_impl(cfg, q, Hq, codes, center, key_norm, k, v, B, Hkv, n_local, 0, n_local, out, nullptr, nullptr,
                     nullptr, ws, ws_bytes, stream, timeline, timeline_len, &grid);
    return rc ? rc : grid;
}

extern "C" int64_t magicpig_debug_decode_timeline_buckets(const magicpig_config* cfg, const uint16_t* q, int64_t Hq,
                                                          const int32_t* tables, const float* center,
                                                          const float* key_norm, const uint16_t* k, const uint16_t* v,
                                                          int64_t B, int64_t Hkv, int64_t n_local, const float* W,
                                                          float* out, unsigned long long* timeline,
                                                          int64_t timeline_len, void* ws, size_t ws_bytes,
                                                          void* stream) {
    if (!timeline || !tables || !buckets_ok(cfg, n_local)) return MAGICPIG_EINVAL;
    int rc = magicpig_encode_queries(cfg, q, B, Hq, W, ws, ws_bytes, stream);
    if (rc) return rc;
    int64_t grid = 0;
    rc = decode_impl(cfg, q, Hq, nullptr, center, key_norm, k, v, B, Hkv, n_local, 0, n_local, out, nullptr, nullptr,
                     nullptr, ws, ws_bytes, stream, timeline, timeline_len, &grid, tables);
    return rc ? rc : grid;
}

int magicpig_decode(const magicpig_config* cfg, const uint16_t* q, int64_t Hq, const uint32_t* codes,
                    const float* center, const float* key_norm, const uint16_t* k, const uint16_t* v, int64_t B,
                    int64_t Hkv, int64_t n_local, int64_t seq_offset, int64_t n_global, const float* W, float* out,
                    float* partial, int32_t* s_count, uint32_t* s_mask, void* ws, size_t ws_bytes, void* stream) {
    if (!W) return MAGICPIG_EINVAL;
    if (n_local > 0) {
        int rc = magicpig_encode_queries(cfg, q, B, Hq, W, ws, ws_bytes, stream);
        if (rc) return rc;
    }
    return magicpig_decode_encoded(cfg, q, Hq, codes, center, key_norm, k, v, B, Hkv, n_local, seq_offset, n_global, out,
                                   partial, s_count, s_mask, ws, ws_bytes, stream);
}

size_t magicpig_bucket_tables_words(const magicpig_config* cfg, int64_t B, int64_t Hkv, int64_t n_local) {
    if (!buckets_ok(cfg, n_local) || B < 1 || Hkv < 1 || n_local < 0) return 0;
    return bucket_tables_words(cfg->K, cfg->L, B * Hkv, n_local);
}

int magicpig_build_buckets(const magicpig_config* cfg, const uint32_t* codes, int64_t B, int64_t Hkv,
                           int64_t n_local, int32_t* tables, void* stream) {
    if (!buckets_ok(cfg, n_local) || B < 1 || Hkv < 1 || n_local < 0 || !codes || !tables) return MAGICPIG_EINVAL;
    const Geom g = make_geom(cfg->K, cfg->L, n_local);
    return launch_bucket_build(codes, B * Hkv, n_local, cfg->K, cfg->L, g.KLq, g.nchunks, tables, S(stream));
}

int magicpig_decode_buckets(const magicpig_config* cfg, const uint16_t* q, int64_t Hq, const int32_t* tables,
                            const float* center, const float* key_norm, const uint16_t* k, const uint16_t* v,
                            int64_t B, int64_t Hkv, int64_t n_local, int64_t seq_offset, int64_t n_global,
                            const float* W, float* out, float* partial, int32_t* s_count, uint32_t* s_mask,
                            void* ws, size_t ws_bytes, void* stream) {
    if (!W || (n_local > 0 && !tables)) return MAGICPIG_EINVAL;
    if (n_local > 0) {
        int rc = magicpig_encode_queries(cfg, q, B, Hq, W, ws, ws_bytes, stream);
        if (rc) return rc;
    }
    return decode_impl(cfg, q, Hq, nullptr, center, key_norm, k, v, B, Hkv, n_local, seq_offset, n_global, out,
                       partial, s_count, s_mask, ws, ws_bytes, stream, nullptr, 0, nullptr, tables);
}

int magicpig_decode_buckets_encoded(const magicpig_config* cfg, const uint16_t* q, int64_t Hq,
                                    const int32_t* tables, const float* center, const float* key_norm,
                                    const uint16_t* k, const uint16_t* v, int64_t B, int64_t Hkv, int64_t n_local,
                                    int64_t seq_offset, int64_t n_global, float* out, float* partial,
                                    int32_t* s_count, uint32_t* s_mask, void* ws, size_t ws_bytes, void* stream) {
    if (n_local > 0 && !tables) return MAGICPIG_EINVAL;
    return decode_impl(cfg, q, Hq, nullptr, center, key_norm, k, v, B, Hkv, n_local, seq_offset, n_global, out,
                       partial, s_count, s_mask, ws, ws_bytes, stream, nullptr, 0, nullptr, tables);
}

int magicpig_debug_decode_sets(const magicpig_config* cfg, const uint16_t* q, int64_t Hq, const uint32_t* codes,
                               const int32_t* tables, const float* center, const float* key_norm, const uint16_t* k,
                               const uint16_t* v, int64_t B, int64_t Hkv, int64_t n_local, int64_t seq_offset,
                               int64_t n_global, const float* W, float* out, uint32_t* s_mask, uint32_t* weighted,
                               void* ws, size_t ws_bytes, void* stream) {
    if (!W || !weighted || (n_local > 0 && !codes && !tables) || n_local < 1) return MAGICPIG_EINVAL;
    if (!cfg_ok(cfg) || Hq < Hkv || Hkv < 1 || B < 1 || Hq % Hkv) return MAGICPIG_EINVAL;
    const int kv = g_decode_kernel.load();
    if (kv != 0 && kv % 10 < 6) return MAGICPIG_EINVAL;  // the weighted-set export exists on kernels 6-8
    if (cudaMemsetAsync(weighted, 0, (size_t)B * Hq * ((n_local + 31) / 32) * 4, S(stream)) != cudaSuccess)
        return MAGICPIG_ECUDA;
    int rc = magicpig_encode_queries(cfg, q, B, Hq, W, ws, ws_bytes, stream);
    if (rc) return rc;
    return decode_impl(cfg, q, Hq, codes, center, key_norm, k, v, B, Hkv, n_local, seq_offset, n_global, out,
                       nullptr, nullptr, s_mask, ws, ws_bytes, stream, nullptr, 0, nullptr, tables, weighted, 7,
                       kv == 0 ? LARGE_KVER : kv);
}

int magicpig_decode_host(const magicpig_config* cfg, const uint16_t* q_host, int64_t Hq, const uint32_t* codes,
                         const int32_t* tables, const float* center, const float* key_norm, const uint16_t* k,
                         const uint16_t* v, int64_t B, int64_t Hkv, int64_t n_local, const float* W, float* out_host,
                         void* ws, size_t ws_bytes, void* stream) {
    if (!cfg_ok(cfg) || !q_host || !out_host || !W || !ws || B < 1 || Hkv < 1 || Hq < Hkv || Hq % Hkv || n_local < 0)
        return MAGICPIG_EINVAL;
    if (tables && !buckets_ok(cfg, n_local)) return MAGICPIG_EINVAL;
    DecodeWs w = decode_layout(cfg, B, Hq, Hkv, n_local, ws);
    if (ws_bytes < w.bytes) return MAGICPIG_EWORKSPACE;
    cudaStream_t st = S(stream);
    if (cudaMemcpyAsync(w.qstage, q_host, (size_t)B * Hq * HD * 2, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return MAGICPIG_ECUDA;
    int rc = MAGICPIG_OK;
    if (n_local > 0) rc = magicpig_encode_queries(cfg, w.qstage, B, Hq, W, ws, ws_bytes, stream);
    if (rc) return rc;
    rc = decode_impl(cfg, w.qstage, Hq, tables ? nullptr : codes, center, key_norm, k, v, B, Hkv, n_local, 0, n_local,
                     w.ostage, nullptr, nullptr, nullptr, ws, ws_bytes, stream, nullptr, 0, nullptr, tables);
    if (rc) return rc;
    if (cudaMemcpyAsync(out_host, w.ostage, (size_t)B * Hq * HD * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return MAGICPIG_ECUDA;
    return cudaStreamSynchronize(st) == cudaSuccess ? MAGICPIG_OK : MAGICPIG_ECUDA;
}

int magicpig_debug_decode_stage(const magicpig_config* cfg, int stage, const uint16_t* q, int64_t Hq,
                                const uint32_t* codes, const int32_t* tables, const float* center,
                                const float* key_norm, const uint16_t* k, const uint16_t* v, int64_t B, int64_t Hkv,
                                int64_t n_local, float* out, void* ws, size_t ws_bytes, void* stream) {
    if (stage < 1 || stage > 7) return MAGICPIG_EINVAL;
    const int kv = g_decode_kernel.load();
    if ((kv != 0 && kv % 10 < 6) || n_local < 1) return MAGICPIG_EINVAL;
    return decode_impl(cfg, q, Hq, codes, center, key_norm, k, v, B, Hkv, n_local, 0, n_local, out, nullptr, nullptr,
                       nullptr, ws, ws_bytes, stream, nullptr, 0, nullptr, tables, nullptr, stage, kv == 0 ? LARGE_KVER : kv);
}

int magicpig_debug_build_phases(const magicpig_config* cfg, const uint16_t* k, int64_t B, int64_t Hkv, int64_t n,
                                const float* W, float* center, int64_t* r2, uint32_t* codes, float* key_norm,
                                int64_t* key_sum, int64_t* count, void* ws, size_t ws_bytes, void* stream,
                                void* const* events) {
    if (!events || n < 1) return MAGICPIG_EINVAL;
    for (int i = 0; i < 5; i++)
        if (!events[i]) return MAGICPIG_EINVAL;
    cudaStream_t st = S(stream);
    auto rec = [&](int i) { return cudaEventRecord((cudaEvent_t)events[i], st) == cudaSuccess; };
    if (!rec(0)) return MAGICPIG_ECUDA;
    int rc = magicpig_key_stats(cfg, k, B, Hkv, n, 0, n, key_sum, count, ws, ws_bytes, stream);
    if (rc) return rc;
    if (!rec(1)) return MAGICPIG_ECUDA;
    rc = magicpig_key_norms(cfg, k, B, Hkv, n, 0, n, key_sum, count, center, r2, ws, ws_bytes, stream);
    if (rc) return rc;
    if (!rec(2)) return MAGICPIG_ECUDA;
    if (!cfg_ok(cfg) || !W || !codes || !key_norm) return MAGICPIG_EINVAL;
    BuildWs w = build_layout(cfg, B, Hkv, n, ws);
    if (ws_bytes < w.bytes) return MAGICPIG_EWORKSPACE;
    const Geom g = make_geom(cfg->K, cfg->L, n);
    if (cudaMemsetAsync(w.fix_count, 0, 4, st) != cudaSuccess) return MAGICPIG_ECUDA;
    rc = launch_prep(k, B * Hkv, n, w.n_pad, cfg->mips, w.KD, center, r2, w.xt, w.xnorm, key_norm, W, g.KL, w.NT,
                     w.wt, w.wmax, w.status, st);
    if (rc) return rc;
    if (!rec(3)) return MAGICPIG_ECUDA;
    rc = launch_hash_gemm(w.xt, w.wt, w.xnorm, w.wmax, codes, w.fix_list, w.fix_count, w.fix_cap, B * Hkv, n, w.n_pad,
                          g.nchunks, w.KD, g.KL, w.NT, g.KLq, w.status, nullptr, st);
    if (rc) return rc;
    return rec(4) ? MAGICPIG_OK : MAGICPIG_ECUDA;
}

int magicpig_merge_partials(const float* parts, int P, int64_t BH, float* out, void* stream) {
    if (!parts || !out || P < 1 || BH < 1) return MAGICPIG_EINVAL;
    return launch_merge(parts, P, BH, out, S(stream));
}

int magicpig_export_codes(const magicpig_config* cfg, const uint32_t* codes, int64_t B, int64_t Hkv,
                          int64_t n_local, uint16_t* canonical, void* stream) {
    if (!cfg_ok(cfg) || B < 1 || Hkv < 1 || n_local < 0 || (n_local > 0 && (!codes || !canonical)))
        return MAGICPIG_EINVAL;
    const Geom g = make_geom(cfg->K, cfg->L, n_local);
    return launch_export_codes(codes, B * Hkv, n_local, cfg->K, cfg->L, g.KLq, g.nchunks, canonical, S(stream));
}

int magicpig_import_codes(const magicpig_config* cfg, const uint16_t* canonical, int64_t B, int64_t Hkv,
                          int64_t n_local, uint32_t* codes, void* stream) {
    if (!cfg_ok(cfg) || B < 1 || Hkv < 1 || n_local < 0 || (n_local > 0 && (!codes || !canonical)))
        return MAGICPIG_EINVAL;
    const Geom g = make_geom(cfg->K, cfg->L, n_local);
    return launch_import_codes(canonical, B * Hkv, n_local, cfg->K, cfg->L, g.KLq, g.nchunks, codes, S(stream));
}

int magicpig_query_codes(const magicpig_config* cfg, const uint16_t* q, int64_t B, int64_t Hq, const float* W,
                         uint16_t* qcodes, void* ws, size_t ws_bytes, void* stream) {
    if (!cfg_ok(cfg) || B < 1 || Hq < 1 || !q || !W || !qcodes || !ws) return MAGICPIG_EINVAL;
    DecodeWs w = decode_layout(cfg, B, Hq, 1, 0, ws);
    const Geom g = make_geom(cfg->K, cfg->L, 0);
    if (ws_bytes < (size_t)((uint8_t*)w.qbits - (uint8_t*)ws) + (size_t)B * Hq * g.KLw * 4) return MAGICPIG_EWORKSPACE;
    int rc = launch_qencode(q, B * Hq, W, g.KL, g.KLw, w.qbits, w.status, S(stream));
    if (rc) return rc;
    return launch_qbits_to_canonical(w.qbits, B * Hq, cfg->K, cfg->L, g.KLw, qcodes, S(stream));
}

int magicpig_collision_counts(const magicpig_config* cfg, const uint16_t* q, int64_t Hq, const uint32_t* codes,
                              int64_t B, int64_t Hkv, int64_t n_local, const float* W, uint16_t* counts, void* ws,
                              size_t ws_bytes, void* stream) {
    if (!cfg_ok(cfg) || B < 1 || Hkv < 1 || Hq < Hkv || Hq % Hkv || n_local < 0) return MAGICPIG_EINVAL;
    if (!q || !W || !ws || (n_local > 0 && (!codes || !counts))) return MAGICPIG_EINVAL;
    DecodeWs w = decode_layout(cfg, B, Hq, Hkv, n_local, ws);
    if (ws_bytes < w.bytes) return MAGICPIG_EWORKSPACE;
    const Geom g = make_geom(cfg->K, cfg->L, n_local);
    int rc = launch_qencode(q, B * Hq, W, g.KL, g.KLw, w.qbits, w.status, S(stream));
    if (rc) return rc;
    return launch_collision_counts(w.qbits, codes, B, Hkv, Hq, n_local, cfg->K, cfg->L, g.KLw, g.KLq, g.nchunks,
                                   counts, S(stream));
}

int magicpig_debug_hash_acc(const magicpig_config* cfg, const uint16_t* k, int64_t n_local, const float* W,
                            const float* center, const int64_t* r2, float* acc, void* ws, size_t ws_bytes,
                            void* stream) {
    if (!cfg_ok(cfg) || n_local < 1 || !k || !W || !center || !r2 || !acc || !ws) return MAGICPIG_EINVAL;
    BuildWs w = build_layout(cfg, 1, 1, n_local, ws);
    const Geom g = make_geom(cfg->K, cfg->L, n_local);
    size_t codes_bytes = (size_t)g.nchunks * g.KLq * 128 * 4;
    if (ws_bytes < w.bytes + align256(codes_bytes) + align256((size_t)n_local * 4)) return MAGICPIG_EWORKSPACE;
    uint32_t* scratch_codes = (uint32_t*)((uint8_t*)ws + w.bytes);
    cudaStream_t st = S(stream);
    if (cudaMemsetAsync(w.fix_count, 0, 4, st) != cudaSuccess) return MAGICPIG_ECUDA;
    float* scratch_norm = (float*)((uint8_t*)ws + w.bytes + align256(codes_bytes));
    int rc = launch_prep(k, 1, n_local, w.n_pad, cfg->mips, w.KD, center, r2, w.xt, w.xnorm, scratch_norm, W, g.KL,
                         w.NT, w.wt, w.wmax, w.status, st);
    if (rc) return rc;
    return launch_hash_gemm(w.xt, w.wt, w.xnorm, w.wmax, scratch_codes, w.fix_list, w.fix_count, w.fix_cap, 1,
                            n_local, w.n_pad, g.nchunks, w.KD, g.KL, w.NT, g.KLq, w.status, acc, st);
}

const char* magicpig_strerror(int err) {
    switch (err) {
        case MAGICPIG_OK: return "ok";
        case MAGICPIG_EINVAL: return "invalid argument (shape, range or NULL pointer)";
        case MAGICPIG_ENOTREPR: return "projection value not bf16-representable";
        case MAGICPIG_EDEGENERATE: return "a head had neither sampled nor static keys";
        case MAGICPIG_ECUDA: return "CUDA error";
        case MAGICPIG_EWORKSPACE: return "workspace too small";
        case MAGICPIG_EINEXACT: return "value outside the exact fixed-point range (|k| >= 2^27)";
        case MAGICPIG_EOVERFLOW: return "hash fix-up list overflow";
    }
    return "unknown error";
}

const char* magicpig_version(void) { return "magicpig-b200 0.1 (sm_100a)"; }

uint64_t magicpig_launch_count(void) { return g_launches.load(); }

}  // extern "C"
