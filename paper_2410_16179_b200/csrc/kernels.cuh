// kernels.cuh -- internal launcher declarations (CUDA path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mp {

constexpr int STATS_SPLIT = 1024;
#ifndef MP_HG_N
#define MP_HG_N 128
#endif
constexpr int HG_N = MP_HG_N;              // hash GEMM: columns per W tile / MMA N (64, 128 or 256)
constexpr int HG_R = 256 / HG_N;           // hash GEMM: 128-key tiles per CTA (TMEM: 2 stages x HG_R x HG_N = 512)  // keys per partial-statistics CTA
constexpr int DEC_THREADS = 256;   // decode CTA (8 warps)

void count_launch(int n);
size_t gemm_smem_bytes(int KD);

int launch_key_stats(const uint16_t* k, int64_t units, int64_t n_local, int64_t seq_offset, int64_t n_global,
                     int sink, int local, int64_t* part_sum, int64_t* part_cnt, int64_t* key_sum,
                     int64_t* count, uint32_t* status, cudaStream_t st);
int launch_key_norms(const uint16_t* k, int64_t units, int64_t n_local, int64_t seq_offset, int64_t n_global,
                     int sink, int local, int do_center, const int64_t* key_sum, const int64_t* count,
                     float* center, int64_t* part_r2, int64_t* r2, uint32_t* status, cudaStream_t st);
int launch_reduce_shards(int mode, const int64_t* parts_sum, const int64_t* parts_cnt, int P, int64_t units,
                         int64_t* out_sum, int64_t* out_cnt, cudaStream_t st);
int launch_prep(const uint16_t* k, int64_t units, int64_t n_local, int64_t n_pad, int mips, int KD,
                const float* center, const int64_t* r2, uint8_t* xt, float* xnorm, float* key_norm, const float* W,
                int KL, int NT, uint8_t* wt, float* wmax, uint32_t* status, cudaStream_t st);
int launch_hash_gemm(const uint8_t* xt, const uint8_t* wt, const float* xnorm, const float* wmax,
                     uint32_t* codes, uint2* fix_list, uint32_t* fix_count, uint32_t fix_cap, int64_t units,
                     int64_t n_local, int64_t n_pad, int64_t nchunks, int KD, int KL, int NT, int KLq,
                     uint32_t* status, float* dbg_acc, cudaStream_t st);

int launch_append_keys(const uint16_t* k_new, int64_t m, int64_t units, int64_t n_old, int mips, const float* W,
                       int KL, int KLq, int64_t nchunks, const float* center, const int64_t* r2, uint32_t* codes,
                       float* key_norm, uint32_t* status, cudaStream_t st);
int launch_qencode(const uint16_t* q, int64_t BHq, const float* W, int KL, int KLw, uint32_t* qbits,
                   uint32_t* status, cudaStream_t st, int K = 0, int L = 0, int minc = 2, float* lutab = nullptr);

struct DecodeArgs {
    const uint16_t* q;
    const uint32_t* qbits;
    const uint32_t* codes;
    const float* center;
    const float* key_norm;
    const uint16_t* k;
    const uint16_t* v;
    int64_t B, Hkv, Hq, n_local, seq_offset, n_global;
    int K, L, KL, KLw, KLq, ngroups, TG, QG;
    int64_t nchunks;
    int64_t nstatic;  // static-key pieces (clusters) per unit
    int tsplit, sink, local, minc;
    int qx_bytes, depth, ring_bytes;  // set by the launcher
    int dyn_bytes;                    // dynamic shared memory per CTA (set by the launcher)
    // persistent kernel (decode5.cu): ring slots, shared-memory offsets, tile count
    int v5_ns, v5_off_qx, v5_off_qbw, v5_off_part, v5_off_rows, v5_off_xt, v5_off_fixed, v5_off_bars;
    int64_t v5_tiles;
    int v5_hs;                        // chunk tiles per 1024-key chunk (1 or 2)
    int dbg;                          // debug flags (kernel 5: bit 0 = no L2 prefetch)
    unsigned long long* timeline;  // debug: [grid][16] globaltimer stamps, or NULL
    float* out;
    float* partial;
    int32_t* s_count;
    uint32_t* s_mask;
    const uint32_t* sbits;           // bucket mode: S bitmaps [B][Hq][ceil(n/32)] (NULL = dense scan)
    uint32_t* unit_ctr;
    float* parts;
    int32_t* chunk_cnt;
    uint32_t* status;
};
int launch_decode(const DecodeArgs& a, cudaStream_t st);
size_t decode5_layout(DecodeArgs& a, int G, int max_smem);
int launch_decode5(const DecodeArgs& a, int nsm, int max_smem, cudaStream_t st);
size_t bucket_tables_words(int K, int L, int64_t units, int64_t n_local);
int launch_bucket_build(const uint32_t* codes, int64_t units, int64_t n_local, int K, int L, int KLq,
                        int64_t nchunks, int32_t* tables, cudaStream_t st);
#ifndef MP_BM_PARTS
#define MP_BM_PARTS 1
#endif
constexpr int BM_PARTS = MP_BM_PARTS;  // id slices per (sequence, query head) in the v7 bucketed Query
                                        // (A/B on B200: 1 = 84.8 us C3 step, 2 = 88.6, 4 = 91.9)
int launch_bucket_mark(const uint32_t* qbits, const int32_t* tables, int64_t B, int64_t Hq, int64_t Hkv,
                       int64_t n_local, int K, int L, int KLw, int minc, uint32_t* sbits, cudaStream_t st,
                       int parts = 1);
int launch_merge(const float* parts, int P, int64_t BH, float* out, cudaStream_t st);
int launch_empty_partial(float* partial, int64_t BH, cudaStream_t st);

int launch_export_codes(const uint32_t* codes, int64_t units, int64_t n_local, int K, int L, int KLq,
                        int64_t nchunks, uint16_t* canonical, cudaStream_t st);
int launch_import_codes(const uint16_t* canonical, int64_t units, int64_t n_local, int K, int L, int KLq,
                        int64_t nchunks, uint32_t* codes, cudaStream_t st);
int launch_qbits_to_canonical(const uint32_t* qbits, int64_t BHq, int K, int L, int KLw, uint16_t* out,
                              cudaStream_t st);
int launch_collision_counts(const uint32_t* qbits, const uint32_t* codes, int64_t B, int64_t Hkv, int64_t Hq,
                            int64_t n_local, int K, int L, int KLw, int KLq, int64_t nchunks, uint16_t* counts,
                            cudaStream_t st);


struct AttendArgs {
    const uint16_t* q;
    const float* center;
    const float* key_norm;
    const uint16_t* k;
    const uint16_t* v;
    const uint32_t* sbits;        // [B][Hq][ceil(n/32)]
    int64_t B, Hkv, Hq, n_local, seq_offset, n_global;
    int64_t nchunks, nstatic, tiles;
    int K, L, minc, sink, local;
    int off_wbuf, off_comb;       // set by attend_layout
    float* out;
    float* partial;
    int32_t* s_count;
    uint32_t* s_mask;             // debug: S_g restricted to D
    uint32_t* weighted;           // debug: (head, key) pairs that received a finite weight (S_g u T)
    uint32_t* unit_ctr;
    float* parts;
    uint32_t* status;
};
size_t attend_layout(AttendArgs& a, int G);
int launch_attend(const AttendArgs& a, int nsm, int max_smem, cudaStream_t st);

// ---- decode v7: Query (scan6 | bucket_mark) -> S bitmaps -> select (ordered S_g u ... lists per unit)
//      -> estimate (every warp a contiguous range of the concatenated lists)
struct EstArgs {
    const uint16_t* q;
    const float* center;
    const float* key_norm;
    const uint16_t* k;
    const uint16_t* v;
    const uint32_t* sbits;        // [B][Hq][ceil(n/32)] S bitmaps of the Query step, or with sparts > 1
                                  // [B][Hq][sparts][2][ceil(n/32)] (seen once, seen twice) per id slice
    int sparts;
    int64_t B, Hkv, Hq, n_local, seq_offset, n_global, nchunks;
    int K, L, minc, sink, local;
    int off_wbuf;                 // set by estimate_layout
    uint32_t* ents;               // [units][nchunks][1024] per piece: key | head bits << 24 (union_g S_g)
    int32_t* pcnt;                // [units][nchunks] entries of each piece (D only)
    int32_t* hpc;                 // [B*Hq][nchunks] |S_g| of each piece
    uint32_t* s_mask;             // debug: S_g restricted to D
    uint32_t* weighted;           // debug: (head, key) pairs that received a finite weight
    float* out;
    float* partial;
    int32_t* s_count;
    uint32_t* unit_ctr;
    float* parts;
    uint32_t* status;
    unsigned long long* timeline;  // debug: [grid * EST_WARPS][16] %globaltimer stamps per warp, or NULL
    int2* urec;                    // [units] (first record slot k_lo, record count) for the merge kernel
    const float* lutab;            // ln u(p) table (LUT_N + 1 entries over [LUT_P0, 1]), filled by the encode
};
#ifndef MP_EST_WARPS
#define MP_EST_WARPS 8
#endif
constexpr int EST_WARPS = MP_EST_WARPS;  // warps per estimator CTA
#ifndef MP_EST9_WARPS
#define MP_EST9_WARPS 12
#endif
constexpr int EST9_WARPS = MP_EST9_WARPS;  // warps per kernel-9 estimator CTA
constexpr int EST_MAX_WARPS = EST_WARPS > EST9_WARPS ? EST_WARPS : EST9_WARPS;
constexpr int EST_MAX_PIECES = 12288;  // units * (chunks + 1): the estimator's piece prefix in smem
int launch_select(const EstArgs& a, cudaStream_t st);
size_t estimate_layout(EstArgs& a, int G);
int launch_estimate(const EstArgs& a, int nsm, int max_smem, cudaStream_t st);
int launch_est_merge(const EstArgs& a, cudaStream_t st);
bool estimate8_ok(const EstArgs& a, int max_smem);
int launch_estimate8(const EstArgs& a, int nsm, int max_smem, cudaStream_t st);
int launch_estimate9(const EstArgs& a, int nsm, int max_smem, cudaStream_t st);

// ---- decode v6: Query (dense scan6 or bucketed bucket_mark) -> S bitmaps -> estimator (attend)
struct ScanArgs {
    const uint32_t* qbits;
    const uint32_t* codes;
    uint32_t* sbits;              // [B][Hq][ceil(n/32)]
    int64_t B, Hkv, Hq, n_local, nchunks, tiles;
    int K, L, KL, KLw, KLq, ngroups, minc;
    int nsw, depth, off_qx, off_qbw, off_part;  // set by scan6_layout
    int fuse;                     // 1: also emit the v7 piece lists (select fused into the scan)
    EstArgs est;                  //    ... with these outputs
};
size_t scan6_layout(ScanArgs& a, int G, int max_smem);
int launch_scan6(const ScanArgs& a, int nsm, int max_smem, cudaStream_t st);




}  // namespace mp
