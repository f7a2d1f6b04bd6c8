// codes_io.cu -- conversions between the bit-plane code layout and the
// canonical per-key codes (debug / interchange), and an exact per-key
// collision count (debug path of Alg. 1 Query).
#include "common.cuh"
#include "kernels.cuh"

namespace mp {

__device__ __forceinline__ int64_t plane_word(int64_t unit, int64_t nchunks, int KLq, int64_t key, int j) {
    const int64_t kb = key >> 5;
    return ((((unit * nchunks + (kb >> 5)) * KLq + (j >> 2)) * 32 + (kb & 31)) << 2) + (j & 3);
}

// canonical[u][i][t] = sum_b bit(i, tK+b) << b.  grid (ceil(n*L/256), units)
__global__ void export_codes_kernel(const uint32_t* __restrict__ codes, int64_t n_local, int K, int L, int KLq,
                                    int64_t nchunks, uint16_t* __restrict__ canonical) {
    const int64_t unit = blockIdx.y;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_local * L) return;
    const int64_t i = e / L;
    const int t = (int)(e % L);
    uint32_t c = 0;
    for (int b = 0; b < K; b++) {
        uint32_t w = codes[plane_word(unit, nchunks, KLq, i, t * K + b)];
        c |= ((w >> (i & 31)) & 1u) << b;
    }
    canonical[(unit * n_local + i) * L + t] = (uint16_t)c;
}

// one thread per (32-key block, column) word, including padding (written 0)
__global__ void import_codes_kernel(const uint16_t* __restrict__ canonical, int64_t n_local, int K, int L,
                                    int KLq, int64_t nchunks, uint32_t* __restrict__ codes) {
    const int64_t unit = blockIdx.y;
    const int64_t nwords_unit = nchunks * (int64_t)KLq * 128;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nwords_unit) return;
    // decode the word position
    const int w = (int)(e & 3);
    const int64_t r1 = e >> 2;
    const int lin = (int)(r1 & 31);
    const int64_t r2 = r1 >> 5;
    const int jq = (int)(r2 % KLq);
    const int64_t chunk = r2 / KLq;
    const int j = jq * 4 + w;
    const int t = j / K, b = j % K;
    const int64_t key0 = chunk * KCHUNK + lin * 32;
    uint32_t word = 0;
    if (t < L) {
        for (int r = 0; r < 32; r++) {
            int64_t i = key0 + r;
            if (i < n_local) word |= ((uint32_t)(canonical[(unit * n_local + i) * L + t] >> b) & 1u) << r;
        }
    }
    codes[unit * nwords_unit + e] = word;
}

// packed query bits [BHq][KLw] -> canonical [BHq][L]
__global__ void qbits_canonical_kernel(const uint32_t* __restrict__ qbits, int64_t BHq, int K, int L, int KLw,
                                       uint16_t* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= BHq * L) return;
    const int64_t h = e / L;
    const int t = (int)(e % L);
    uint32_t c = 0;
    for (int b = 0; b < K; b++) {
        int j = t * K + b;
        c |= ((qbits[h * KLw + (j >> 5)] >> (j & 31)) & 1u) << b;
    }
    out[e] = (uint16_t)c;
}

// exact count of tables whose K-bit code equals the query's: thread per (key, q head)
__global__ void collision_counts_kernel(const uint32_t* __restrict__ qbits, const uint32_t* __restrict__ codes,
                                        int64_t Hkv, int64_t Hq, int64_t n_local, int K, int L, int KLw, int KLq,
                                        int64_t nchunks, uint16_t* __restrict__ counts) {
    const int64_t row = blockIdx.y;  // b * Hq + hq
    const int64_t b = row / Hq, hq = row % Hq;
    const int64_t G = Hq / Hkv;
    const int64_t unit = b * Hkv + hq / G;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_local) return;
    int cnt = 0;
    for (int t = 0; t < L; t++) {
        bool eq = true;
        for (int bb = 0; bb < K; bb++) {
            int j = t * K + bb;
            uint32_t kbit = (codes[plane_word(unit, nchunks, KLq, i, j)] >> (i & 31)) & 1u;
            uint32_t qbit = (qbits[row * KLw + (j >> 5)] >> (j & 31)) & 1u;
            eq &= kbit == qbit;
        }
        cnt += eq;
    }
    counts[row * n_local + i] = (uint16_t)cnt;
}

int launch_export_codes(const uint32_t* codes, int64_t units, int64_t n_local, int K, int L, int KLq,
                        int64_t nchunks, uint16_t* canonical, cudaStream_t st) {
    int64_t n = n_local * L;
    if (n == 0) return 0;
    export_codes_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)units), 256, 0, st>>>(codes, n_local, K, L, KLq,
                                                                                         nchunks, canonical);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

int launch_import_codes(const uint16_t* canonical, int64_t units, int64_t n_local, int K, int L, int KLq,
                        int64_t nchunks, uint32_t* codes, cudaStream_t st) {
    int64_t n = nchunks * (int64_t)KLq * 128;
    if (n == 0) return 0;
    import_codes_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)units), 256, 0, st>>>(canonical, n_local, K, L, KLq,
                                                                                         nchunks, codes);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

int launch_qbits_to_canonical(const uint32_t* qbits, int64_t BHq, int K, int L, int KLw, uint16_t* out,
                              cudaStream_t st) {
    int64_t n = BHq * L;
    qbits_canonical_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(qbits, BHq, K, L, KLw, out);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

int launch_collision_counts(const uint32_t* qbits, const uint32_t* codes, int64_t B, int64_t Hkv, int64_t Hq,
                            int64_t n_local, int K, int L, int KLw, int KLq, int64_t nchunks, uint16_t* counts,
                            cudaStream_t st) {
    if (n_local == 0) return 0;
    collision_counts_kernel<<<dim3((unsigned)((n_local + 127) / 128), (unsigned)(B * Hq)), 128, 0, st>>>(
        qbits, codes, Hkv, Hq, n_local, K, L, KLw, KLq, nchunks, counts);
    count_launch(1);
    return cudaGetLastError() == cudaSuccess ? 0 : MAGICPIG_ECUDA;
}

}  // namespace mp
