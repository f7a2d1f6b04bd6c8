// scan6.cu -- Query(HT, q_code) of Algorithm 1 on the dense
// bit-plane codes: for every key and query head, the number of tables whose
// K-bit code equals the query's, and the ">= 2 tables match" rule
// -> per-head S bitmaps sbits[B][Hq][ceil(n/32)] (bit r of word w = key 32w+r
// has count >= min_collisions; the estimator kernel, attend.cu, restricts it
// to the dynamic keys D).  Bandwidth kernel: the codes are the only large
// input (|D| K L / 8 bytes per unit).
//
// One persistent CTA per SM over a contiguous range of 1024-key chunks.  Each
// of the NSW warps owns table group j (TG tables = QG 4-column quads, 512 B
// per quad per chunk) of every chunk for j = warp (mod NSW) and streams its
// groups through a private shared-memory ring with cp.async (16 B per lane, a
// commit group per table group, refilled as soon as a slot is read), starting
// before the query codes exist (PDL overlap with the encode kernel).  Per table
// and query head: one LOP3 per code bit (m &= P_b ^ QX_b, QX = 0 / ~0 from the
// query bit) and a saturating counter (seen1 / seen2); the warps' counters are
// combined per chunk in shared memory (one barrier per chunk, double-buffered).
#include "common.cuh"
#include "kernels.cuh"
#include "pieces.cuh"

namespace mp {
namespace v6 {

constexpr int NSW_MAX = 16;              // scan warps (runtime: 16, or 8 when the rings do not fit)
constexpr int SC_THREADS = NSW_MAX * 32;
constexpr int RING_BUDGET = 176 * 1024;  // bytes of code rings per CTA (depth chosen at launch)

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// wait until at most n commit groups of this thread are pending (n < 16, warp-uniform)
__device__ __forceinline__ void cp_wait_dyn(int n) {
    switch (n) {
#define W_(k) \
    case k: asm volatile("cp.async.wait_group " #k ";" ::: "memory"); break;
        W_(0) W_(1) W_(2) W_(3) W_(4) W_(5) W_(6) W_(7) W_(8) W_(9) W_(10) W_(11) W_(12) W_(13) W_(14)
        default: asm volatile("cp.async.wait_group 15;" ::: "memory"); break;
#undef W_
    }
}

template <int K, int G>
__global__ void __launch_bounds__(SC_THREADS, 1) scan6_kernel(ScanArgs a) {
    constexpr int TG = tg_of(K), QG = qg_of(K);
    constexpr uint32_t GB = QG * 512;  // bytes of one table group of one chunk
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ __align__(128) uint8_t dsm[];
    const int D = a.depth;
    uint8_t* ring = dsm;                                                  // [NSW][D][GB]
    uint32_t* qx = reinterpret_cast<uint32_t*>(dsm + a.off_qx);           // [ncolsP][G] match masks
    uint32_t* qbw = reinterpret_cast<uint32_t*>(dsm + a.off_qbw);         // [G][KLw] packed query bits
    uint32_t* s_part = reinterpret_cast<uint32_t*>(dsm + a.off_part);     // [2][nsw][G][2][32]
    __shared__ uint32_t s_fin[2][8][32];                                   // fused select: S_g words per chunk

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NSW = a.nsw, NTH = NSW * 32;
    const int64_t T = a.tiles, P = gridDim.x;
    const int64_t c0 = (int64_t)blockIdx.x * T / P, c1 = ((int64_t)blockIdx.x + 1) * T / P;  // global chunks
    const size_t CB = (size_t)a.KLq * 512;  // code bytes per chunk
    const uint8_t* codes_b = reinterpret_cast<const uint8_t*>(a.codes);
    uint8_t* myring = ring + (size_t)warp * D * GB;
    uint8_t* const ring_end = myring + (size_t)D * GB;

    // issue iterator over this warp's (chunk, group) sequence
    int64_t it_c = c0;
    int it_j = warp;
    const bool has_groups = warp < a.ngroups;
    const uint8_t* it_src = codes_b + (size_t)it_c * CB + (size_t)warp * GB + lane * 16;
    uint8_t* wr = myring + lane * 16;
    const uint8_t* rd = myring + lane * 16;
    auto issue = [&]() {
        if (has_groups && it_c < c1) {
#pragma unroll
            for (int q = 0; q < QG; q++) cp_async16(wr + q * 512, it_src + q * 512);
            it_j += NSW;
            if (it_j >= a.ngroups) {
                it_j = warp;
                it_c++;
                it_src = codes_b + (size_t)it_c * CB + (size_t)warp * GB + lane * 16;
            } else {
                it_src += NSW * GB;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        wr += GB;
        if (wr >= ring_end) wr -= (size_t)D * GB;
    };
#pragma unroll 1
    for (int k = 0; k < D; k++) issue();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // query codes of the encode kernel

    const int ncolsP = a.ngroups * TG * K;
    const int64_t nwb = (a.n_local + 31) >> 5;
    int64_t cur_u = -1;
    int par = 0;
#pragma unroll 1
    for (int64_t c = c0; c < c1; c++, par ^= 1) {
        const int64_t u = c / a.nchunks, chunk = c % a.nchunks;
        const int64_t b = u / a.Hkv, hkv = u % a.Hkv;
        const int64_t qh0 = b * a.Hq + hkv * G;
        if (u != cur_u) {  // query masks of unit u: QX[c][g] = qbit ? 0 : ~0 (P ^ QX = 1 where bits agree)
            __syncthreads();
            for (int e = tid; e < G * a.KLw; e += NTH) qbw[e] = __ldcg(a.qbits + qh0 * a.KLw + e);
            __syncthreads();
            for (int e = tid; e < ncolsP * G; e += NTH) {
                const int cc = e / G, g = e % G;
                qx[e] = (cc < a.KL && ((qbw[g * a.KLw + (cc >> 5)] >> (cc & 31)) & 1u)) ? 0u : 0xffffffffu;
            }
            __syncthreads();
            cur_u = u;
        }
        uint32_t s1[G], s2[G];
#pragma unroll
        for (int g = 0; g < G; g++) s1[g] = s2[g] = 0u;
#pragma unroll 1
        for (int j = warp; j < a.ngroups; j += NSW) {
            cp_wait_dyn(D - 1);
            __syncwarp();
            uint4 Pw[QG];
#pragma unroll
            for (int q = 0; q < QG; q++) Pw[q] = *reinterpret_cast<const uint4*>(rd + q * 512);
            rd += GB;
            if (rd >= ring_end) rd -= (size_t)D * GB;
            __syncwarp();
            issue();  // refill the slot just read
            const uint32_t* wv = reinterpret_cast<const uint32_t*>(Pw);
            const uint32_t* qrow = qx + (size_t)j * TG * K * G;
#pragma unroll
            for (int tt = 0; tt < TG; tt++) {
                if (TG == 1 || tt == 0 || j * TG + tt < a.L) {
                    uint32_t m[G];
#pragma unroll
                    for (int g = 0; g < G; g++) m[g] = 0xffffffffu;
#pragma unroll
                    for (int bb = 0; bb < K; bb++) {
                        const uint32_t w = wv[tt * K + bb];
                        const uint32_t* qp = qrow + (tt * K + bb) * G;
                        if constexpr (G % 4 == 0) {
#pragma unroll
                            for (int g4 = 0; g4 < G / 4; g4++) {
                                const uint4 qq = reinterpret_cast<const uint4*>(qp)[g4];
                                m[4 * g4] &= w ^ qq.x;
                                m[4 * g4 + 1] &= w ^ qq.y;
                                m[4 * g4 + 2] &= w ^ qq.z;
                                m[4 * g4 + 3] &= w ^ qq.w;
                            }
                        } else {
#pragma unroll
                            for (int g = 0; g < G; g++) m[g] &= w ^ qp[g];
                        }
                    }
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        s2[g] |= s1[g] & m[g];
                        s1[g] |= m[g];
                    }
                }
            }
        }
        uint32_t* sp = s_part + (size_t)par * NSW * G * 64;
#pragma unroll
        for (int g = 0; g < G; g++) {
            sp[((warp * G + g) * 2 + 0) * 32 + lane] = s1[g];
            sp[((warp * G + g) * 2 + 1) * 32 + lane] = s2[g];
        }
        __syncthreads();
        // warps -> CTA: (a1,a2)+(b1,b2) = (a1|b1, a2|b2|(a1&b1)); S_g = count >= minc
        if (warp < G) {
            const int g = warp;
            uint32_t f1 = 0, f2 = 0;
#pragma unroll 4
            for (int w = 0; w < NSW; w++) {
                const uint32_t b1 = sp[((w * G + g) * 2 + 0) * 32 + lane];
                const uint32_t b2 = sp[((w * G + g) * 2 + 1) * 32 + lane];
                f2 |= b2 | (f1 & b1);
                f1 |= b1;
            }
            const int64_t wi = chunk * 32 + lane;
            if (a.fuse) s_fin[par][g][lane] = a.minc == 1 ? f1 : f2;
            else if (wi < nwb) a.sbits[(qh0 + g) * nwb + wi] = a.minc == 1 ? f1 : f2;
        }
        if (a.fuse && warp < G) {
            // select fused into the scan: the union of the unit's heads over this chunk -> its piece list
            if (G > 1) asm volatile("bar.sync 1, %0;" ::"r"(G * 32) : "memory");
            if (warp == 0) {
                uint32_t sg[G];
#pragma unroll
                for (int g = 0; g < G; g++) sg[g] = s_fin[par][g][lane];
                v7::emit_piece<G>(a.est, v7::static_ranges(a.est), u, chunk, qh0, lane, sg);
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

}  // namespace v6

static size_t al128s(size_t x) { return (x + 127) & ~(size_t)127; }

// fills the layout fields of a; returns the dynamic smem bytes (0 if it does not fit)
size_t scan6_layout(ScanArgs& a, int G, int max_smem) {
    const int TG = tg_of(a.K), QG = qg_of(a.K);
    const size_t GB = (size_t)QG * 512;
    const int ncolsP = a.ngroups * TG * a.K;
    size_t fixed = al128s((size_t)ncolsP * G * 4);  // qx
    const size_t o_qbw = fixed;
    fixed += al128s((size_t)G * a.KLw * 4);
    const size_t o_part = fixed;
    fixed += al128s((size_t)2 * v6::NSW_MAX * G * 2 * 32 * 4);
    const size_t budget = (size_t)max_smem - 256 - 2048;  // static smem of the kernel (s_fin)
    if (fixed >= budget) return 0;
    size_t avail = budget - fixed;
    if (avail > (size_t)v6::RING_BUDGET) avail = v6::RING_BUDGET;
    // 16 warps with >= 3 ring slots each, else 8 warps with >= 2 (large K*L / G = 8)
    int nsw = 16, depth = (int)(avail / (16 * GB));
    if (depth < 3) {
        nsw = 8;
        depth = (int)(avail / (8 * GB));
    }
    if (depth > 16) depth = 16;
    if (depth < 2) return 0;
    a.nsw = nsw;
    a.depth = depth;
    const size_t ring = al128s((size_t)nsw * depth * GB);
    a.off_qx = (int)ring;
    a.off_qbw = (int)(ring + o_qbw);
    a.off_part = (int)(ring + o_part);
    return ring + fixed;
}

template <int K, int G>
static int launch_scan_kg(ScanArgs a, int nsm, int max_smem, cudaStream_t st) {
    const size_t smem = scan6_layout(a, G, max_smem);
    if (!smem) return MAGICPIG_EINVAL;
    auto kern = v6::scan6_kernel<K, G>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return MAGICPIG_ECUDA;
    const int64_t P = a.tiles < nsm ? a.tiles : nsm;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)P);
    cfg.blockDim = dim3((unsigned)(a.nsw * 32));
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

template <int K>
static int launch_scan_k(const ScanArgs& a, int G, int nsm, int max_smem, cudaStream_t st) {
    switch (G) {
        case 1: return launch_scan_kg<K, 1>(a, nsm, max_smem, st);
        case 2: return launch_scan_kg<K, 2>(a, nsm, max_smem, st);
        case 4: return launch_scan_kg<K, 4>(a, nsm, max_smem, st);
        case 8: return launch_scan_kg<K, 8>(a, nsm, max_smem, st);
    }
    return MAGICPIG_EINVAL;
}

int launch_scan6(const ScanArgs& a, int nsm, int max_smem, cudaStream_t st) {
    const int G = (int)(a.Hq / a.Hkv);
    switch (a.K) {
#define MPK(k) \
    case k: return launch_scan_k<k>(a, G, nsm, max_smem, st);
        MPK(1) MPK(2) MPK(3) MPK(4) MPK(5) MPK(6) MPK(7) MPK(8)
        MPK(9) MPK(10) MPK(11) MPK(12) MPK(13) MPK(14) MPK(15) MPK(16)
#undef MPK
    }
    return MAGICPIG_EINVAL;
}

}  // namespace mp
