// pdl_kernels.cu -- sm_100a kernels for the PolyDL hot path:
//   * tile_mma_kernel: warp-specialised implicit-GEMM engine shared by the
//     blocked convolution (Fig. 9 nest) and the row-major
//     GEMM (Fig. 1).  TMA stages operand tiles into 64/128B
//     swizzled shared memory, one elected thread issues tcgen05.mma kind::tf32
//     with the fp32 accumulator in TMEM, and four epilogue warps drain TMEM
//     through registers, applying the fused bias + ReLU (Alg. 3, PAPER.md:
//     566-596) before the only store of the output.
//   * 3xTF32: four "split" warps turn every landed fp32 tile x into
//     hi = tf32(x) (in place) and lo = x - hi (second buffer); the MMA warp
//     issues hi*hi + hi*lo + lo*hi.  Conv weights are split once at prepack.
//   * simt kernels: exact-fp32 CUDA-core GEMM / conv (PDL_MODE_FP32, and the
//     GEMM path for leading dimensions TMA cannot describe), the unfused
//     bias+ReLU pass, and the weight prepack.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/pdl.h"
#include "pdl_sm100.cuh"

namespace pdl {

enum { KIND_GEMM = 0, KIND_CONV = 1 };

// Geometry / epilogue parameters (by value, param space).
struct TileParams {
    // common
    int num_kb;       // pipeline k-blocks per tile
    int n_out;        // output columns (GEMM N / conv K)
    unsigned flags;   // PDL_BIAS | PDL_RELU
    const float *bias;
    float *out;
    // GEMM
    int M, ldc;
    float alpha, beta;
    // conv
    int nimg, P, Q, KT, R, S, pad, stride, CT;
    int BW, BH, BNI;       // box of output pixels per tile
    int tiles_w, tiles_h;  // tile grid over (Q, P); images fastest-after
    int m_tiles;           // number of M tiles
    int raster;            // 0: blockIdx.x -> M tile, 1: -> N tile
    int seg_kb;            // k-blocks per TMEM accumulation segment
};

struct TmaMaps {
    CUtensorMap a[4];  // conv: one per (row, col) parity for stride 2; GEMM: a[0]
    CUtensorMap b;
};

template <int KIND, int BN, int CG>
struct Geo {
    static constexpr int BM = 128;
    // GEMM: A [128 rows][32 fp32] SW128, B [BN/32 chunks][32 k][32 n] SW128 (MN-major)
    // CONV: A [CG][128 rows][16 fp32] SW64, B [CG][BN rows][16 fp32] SW64 (K-major)
    static constexpr int A_SUB = KIND == KIND_GEMM ? BM * 128 : BM * 64;
    static constexpr int B_SUB = KIND == KIND_GEMM ? BN * 128 : BN * 64;
    static constexpr int NSUB = KIND == KIND_GEMM ? 1 : CG;
    static constexpr int A_BYTES = A_SUB * NSUB;
    static constexpr int B_BYTES = B_SUB * NSUB;
    static constexpr int KK = KIND == KIND_GEMM ? 4 : 2;  // K=8 MMAs per sub-tile
};

template <int KIND, int BN, int CG, bool SPLIT3>
struct Smem {
    using G = Geo<KIND, BN, CG>;
    static constexpr int STAGE = (G::A_BYTES + G::B_BYTES) * (SPLIT3 ? 2 : 1);
    static constexpr int BUDGET = 200 * 1024;
    static constexpr int STAGES = (BUDGET / STAGE) > 8 ? 8 : (BUDGET / STAGE);
    static constexpr int A_HI = 0;
    static constexpr int A_LO = G::A_BYTES;
    static constexpr int B_HI = SPLIT3 ? 2 * G::A_BYTES : G::A_BYTES;
    static constexpr int B_LO = B_HI + G::B_BYTES;
    static constexpr int BAR_OFF = STAGES * STAGE;
    static constexpr int TOTAL = BAR_OFF + 512 + 1024;  // barriers + alignment slack
    static_assert(STAGES >= 2, "tile too large for a 2-stage pipeline");
};

__device__ __forceinline__ float4 split_hi(float4 v) {
    float4 h;
    h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    return h;
}

// In-place hi + separate lo over `bytes` of shared memory (layout-agnostic:
// the transform is element-wise, so the swizzled tile stays swizzled).
__device__ __forceinline__ void split_tile(uint8_t *hi, uint8_t *lo, int bytes, int tid,
                                           int nthreads) {
    float4 *h4 = reinterpret_cast<float4 *>(hi);
    float4 *l4 = reinterpret_cast<float4 *>(lo);
    const int n = bytes >> 4;
#pragma unroll 4
    for (int i = tid; i < n; i += nthreads) {
        float4 v = h4[i];
        float4 h = split_hi(v);
        float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        h4[i] = h;
        l4[i] = l;
    }
}

// Epilogue for 16 consecutive output columns [col0, col0+16) of one row.
template <int KIND>
__device__ __forceinline__ void store16(const TileParams &p, float *dst, int col0,
                                        const float *v) {
    const bool has_bias = (p.flags & PDL_BIAS) && p.bias;
    const bool relu = p.flags & PDL_RELU;
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
        const int col = col0 + q4 * 4;
        if (KIND == KIND_GEMM && col >= p.n_out) break;
        float4 r = make_float4(v[q4 * 4 + 0], v[q4 * 4 + 1], v[q4 * 4 + 2], v[q4 * 4 + 3]);
        if (KIND == KIND_GEMM) {
            r.x *= p.alpha; r.y *= p.alpha; r.z *= p.alpha; r.w *= p.alpha;
            if (p.beta != 0.f) {
                const float4 c = *reinterpret_cast<const float4 *>(dst + q4 * 4);
                r.x += p.beta * c.x; r.y += p.beta * c.y;
                r.z += p.beta * c.z; r.w += p.beta * c.w;
            }
        }
        if (has_bias) {
            const float4 b = __ldg(reinterpret_cast<const float4 *>(p.bias + col));
            r.x += b.x; r.y += b.y; r.z += b.z; r.w += b.w;
        }
        if (relu) {  // Python max(v, 0.0): keep v unless 0 > v
            r.x = (0.f > r.x) ? 0.f : r.x;
            r.y = (0.f > r.y) ? 0.f : r.y;
            r.z = (0.f > r.z) ? 0.f : r.z;
            r.w = (0.f > r.w) ? 0.f : r.w;
        }
        *reinterpret_cast<float4 *>(dst + q4 * 4) = r;
    }
}

// Implicit-GEMM tile engine.  One CTA = one 128 x BN output tile.
//   warp 0      TMA producer (one lane)
//   warp 1      tcgen05.mma issuer (one lane)
//   warp 2      TMEM allocator
//   warps 4-7   3xTF32 split of each landed stage, then TMEM drain + epilogue
// The reduction is cut into segments of p.seg_kb k-blocks; each segment is
// accumulated in one of two TMEM buffers (ping-pong) and drained into fp32
// registers with round-to-nearest adds.  The tensor core's accumulator
// truncates, so an unsegmented K=4096 sum drifts to ~3e-5 relative error;
// 256-element segments keep it near 3e-6 at any K.
template <int KIND, int BN, int CG, bool SPLIT3>
__global__ void __launch_bounds__(256, 1)
    tile_mma_kernel(const __grid_constant__ TmaMaps maps, const TileParams p) {
    using G = Geo<KIND, BN, CG>;
    using L = Smem<KIND, BN, CG, SPLIT3>;
    constexpr int STAGES = L::STAGES;
    constexpr bool SEGMENTED = BN <= 128;  // register budget for the running sums
    constexpr uint32_t TMEM_COLS = SEGMENTED ? 2 * BN : BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem =
        reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);
    uint64_t *ready = full + STAGES;
    uint64_t *empty = ready + STAGES;
    uint64_t *tmem_full = empty + STAGES;  // [2]
    uint64_t *tmem_empty = tmem_full + 2;  // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int m_tile = p.raster ? blockIdx.y : blockIdx.x;
    const int n_tile = p.raster ? blockIdx.x : blockIdx.y;
    const int n0 = n_tile * BN;
    const int seg_kb = SEGMENTED ? p.seg_kb : p.num_kb;
    const int nseg = (p.num_kb + seg_kb - 1) / seg_kb;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&maps.b);
        tma_prefetch(&maps.a[0]);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&ready[s], 128);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tmem_full[b], 1);
            mbar_init(&tmem_empty[b], 128);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // Conv tile origin (shared by producer and epilogue).
    int q0 = 0, p0 = 0, i0 = 0, m0 = 0;
    if (KIND == KIND_CONV) {
        int t = m_tile;
        const int tw = t % p.tiles_w;
        t /= p.tiles_w;
        const int th = t % p.tiles_h;
        t /= p.tiles_h;
        q0 = tw * p.BW;
        p0 = th * p.BH;
        i0 = t * p.BNI;
    } else {
        m0 = m_tile * G::BM;
    }

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint32_t tx =
                KIND == KIND_GEMM
                    ? (uint32_t)(G::BM * 32 * 4 + BN * 32 * 4)
                    : (uint32_t)(CG * 64 * p.BW * p.BH * p.BNI + CG * BN * 64 * (SPLIT3 ? 2 : 1));
            int s = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t *st = smem + s * L::STAGE;
                mbar_arrive_expect_tx(&full[s], tx);
                if (KIND == KIND_GEMM) {
                    tma_load_2d(st + L::A_HI, &maps.a[0], &full[s], kb * 32, m0);
#pragma unroll
                    for (int c = 0; c < BN / 32; ++c)
                        tma_load_2d(st + L::B_HI + c * 4096, &maps.b, &full[s], n0 + c * 32,
                                    kb * 32);
                } else {
                    const int rs_n = p.R * p.S;
                    const int ctg = kb / rs_n;
                    const int rs = kb - ctg * rs_n;
                    const int r = rs / p.S;
                    const int sx = rs - r * p.S;
                    int dh = r - p.pad, dw = sx - p.pad, mi = 0;
                    if (p.stride == 2) {
                        const int ph2 = dh & 1, pw2 = dw & 1;
                        mi = ph2 * 2 + pw2;
                        dh = (dh - ph2) >> 1;
                        dw = (dw - pw2) >> 1;
                    }
#pragma unroll
                    for (int c = 0; c < CG; ++c)
                        tma_load_5d(st + L::A_HI + c * G::A_SUB, &maps.a[mi], &full[s], 0,
                                    q0 + dw, p0 + dh, ctg * CG + c, i0);
                    tma_load_5d(st + L::B_HI, &maps.b, &full[s], 0, n0, rs, ctg * CG, 0);
                }
                if (++s == STAGES) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (one thread) =====================
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(128, BN, KIND == KIND_GEMM ? 1 : 0);
            const uint32_t layout = KIND == KIND_GEMM ? LAYOUT_SW128 : LAYOUT_SW64;
            const uint32_t a_sbo = KIND == KIND_GEMM ? 1024 : 512;
            const uint32_t smem0 = smem_u32(smem);
            int s = 0;
            uint32_t ph = 0;
            int g = 0, in_seg = 0;
            uint32_t d_tmem = tmem_base;
            for (int kb = 0; kb < p.num_kb; ++kb) {
                if (in_seg == 0) {  // new segment: wait for its TMEM buffer to be drained
                    mbar_wait(&tmem_empty[g & 1], ((g >> 1) & 1) ^ 1);
                    tc_fence_after();
                    d_tmem = tmem_base + (SEGMENTED ? (uint32_t)((g & 1) * BN) : 0u);
                }
                mbar_wait(SPLIT3 ? &ready[s] : &full[s], ph);
                tc_fence_after();
                const uint32_t st = smem0 + s * L::STAGE;
#pragma unroll
                for (int c = 0; c < G::NSUB; ++c) {
#pragma unroll
                    for (int kk = 0; kk < G::KK; ++kk) {
                        const uint32_t a_off = c * G::A_SUB + kk * 32;
                        const uint64_t ahi = smem_desc(st + L::A_HI + a_off, 16, a_sbo, layout);
                        const uint64_t alo = smem_desc(st + L::A_LO + a_off, 16, a_sbo, layout);
                        uint64_t bhi, blo;
                        if (KIND == KIND_GEMM) {
                            // MN-major tf32 operand: 128B rows of 32 n-values, 32B-atom
                            // swizzle (layout SWIZZLE_128B_BASE32B); 4-row k-groups at
                            // SBO = 512B, 32-col chunks at LBO = 32 rows * 128B.
                            bhi = smem_desc(st + L::B_HI + kk * 1024, 4096, 512, LAYOUT_SW128_B32);
                            blo = smem_desc(st + L::B_LO + kk * 1024, 4096, 512, LAYOUT_SW128_B32);
                        } else {
                            const uint32_t b_off = c * G::B_SUB + kk * 32;
                            bhi = smem_desc(st + L::B_HI + b_off, 16, 512, LAYOUT_SW64);
                            blo = smem_desc(st + L::B_LO + b_off, 16, 512, LAYOUT_SW64);
                        }
                        const uint32_t acc = (in_seg | c | kk) != 0;
                        mma_tf32(d_tmem, ahi, bhi, idesc, acc);
                        if (SPLIT3) {
                            mma_tf32(d_tmem, ahi, blo, idesc, 1);
                            mma_tf32(d_tmem, alo, bhi, idesc, 1);
                        }
                    }
                }
                mma_commit(&empty[s]);
                if (++s == STAGES) { s = 0; ph ^= 1; }
                if (++in_seg == seg_kb || kb + 1 == p.num_kb) {
                    mma_commit(&tmem_full[g & 1]);
                    in_seg = 0;
                    ++g;
                }
            }
        }
    } else if (warp >= 4) {
        const int tid = threadIdx.x - 128;
        const int quarter = warp - 4;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        float sum[SEGMENTED ? BN : 1];
        if (SEGMENTED) {
#pragma unroll
            for (int i = 0; i < (SEGMENTED ? BN : 1); ++i) sum[i] = 0.f;
        }
        int drained = 0;
        auto drain = [&](int g) {
            mbar_wait(&tmem_full[g & 1], (g >> 1) & 1);
            tc_fence_after();
            if (SEGMENTED) {
                const uint32_t base = tmem_base + lane_off + (uint32_t)((g & 1) * BN);
#pragma unroll
                for (int j = 0; j < BN / 16; ++j) {
                    float v[16];
                    tmem_ld16(base + j * 16, v);
#pragma unroll
                    for (int i = 0; i < 16; ++i) sum[(SEGMENTED ? j * 16 + i : 0)] += v[i];
                }
                tc_fence_before();
                mbar_arrive(&tmem_empty[g & 1]);
            }
        };
        const int a_valid = KIND == KIND_GEMM ? G::A_SUB : 64 * p.BW * p.BH * p.BNI;
        {
            int s = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < p.num_kb; ++kb) {
                if (SPLIT3) {
                    // ===================== 3xTF32 split =====================
                    mbar_wait(&full[s], ph);
                    uint8_t *st = smem + s * L::STAGE;
#pragma unroll
                    for (int c = 0; c < G::NSUB; ++c)
                        split_tile(st + L::A_HI + c * G::A_SUB, st + L::A_LO + c * G::A_SUB,
                                   a_valid, tid, 128);
                    if (KIND == KIND_GEMM)
                        split_tile(st + L::B_HI, st + L::B_LO, G::B_BYTES, tid, 128);
                    fence_proxy_async_smem();
                    mbar_arrive(&ready[s]);
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
                // drain segments that finished at least one k-block ago
                if (SEGMENTED && drained < nseg - 1 && kb >= (drained + 1) * seg_kb) drain(drained++);
            }
        }
        // ===================== epilogue =====================
        bool valid;
        float *obase = nullptr;
        size_t cstride = 0;
        if (KIND == KIND_GEMM) {
            const int gm = m0 + row;
            valid = gm < p.M;
            obase = p.out + (size_t)(valid ? gm : 0) * p.ldc;
        } else {
            const int per_img = p.BW * p.BH;
            const int il = row / per_img;
            const int rem = row - il * per_img;
            const int hl = rem / p.BW;
            const int wl = rem - hl * p.BW;
            const int img = i0 + il, pp = p0 + hl, qq = q0 + wl;
            valid = il < p.BNI && img < p.nimg && pp < p.P && qq < p.Q;
            const size_t plane = (size_t)p.P * p.Q * 16;
            obase = p.out + ((size_t)(valid ? img : 0) * p.KT) * plane +
                    ((size_t)(valid ? pp : 0) * p.Q + (valid ? qq : 0)) * 16;
            cstride = plane;  // next 16-channel block kt
        }
        if (SEGMENTED) {
            while (drained < nseg) drain(drained++);
            if (valid) {
#pragma unroll
                for (int j = 0; j < BN / 16; ++j) {
                    const int col0 = n0 + j * 16;
                    if (col0 < p.n_out) {
                        float *dst = KIND == KIND_GEMM ? obase + col0 : obase + (size_t)(col0 >> 4) * cstride;
                        store16<KIND>(p, dst, col0, &sum[SEGMENTED ? j * 16 : 0]);
                    }
                }
            }
        } else {
            drain(0);
#pragma unroll 1
            for (int j = 0; j < BN / 16; ++j) {
                float v[16];
                tmem_ld16(tmem_base + lane_off + j * 16, v);
                const int col0 = n0 + j * 16;
                if (!valid || col0 >= p.n_out) continue;
                float *dst = KIND == KIND_GEMM ? obase + col0 : obase + (size_t)(col0 >> 4) * cstride;
                store16<KIND>(p, dst, col0, v);
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}

// ------------------------------------------------------------------ SIMT kernels

// Exact fp32 GEMM on CUDA cores: 64x64 tile, 256 threads, 4x4 per thread.
__global__ void __launch_bounds__(256) simt_gemm_kernel(const float *__restrict__ A,
                                                        const float *__restrict__ B,
                                                        float *__restrict__ C, int M, int N,
                                                        int K, int lda, int ldb, int ldc,
                                                        float alpha, float beta,
                                                        const float *__restrict__ bias,
                                                        unsigned flags) {
    __shared__ float As[16][64 + 1];
    __shared__ float Bs[16][64];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int mb = blockIdx.y * 64, nb = blockIdx.x * 64;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += 16) {
        for (int i = threadIdx.x; i < 16 * 64; i += 256) {
            const int mm = i >> 4, kk = i & 15;  // A tile: 64 rows x 16 k
            const int gm = mb + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < K) ? A[(size_t)gm * lda + gk] : 0.f;
            const int kr = i >> 6, nn = i & 63;  // B tile: 16 k x 64 cols
            const int gk2 = k0 + kr, gn = nb + nn;
            Bs[kr][nn] = (gk2 < K && gn < N) ? B[(size_t)gk2 * ldb + gn] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = mb + ty * 4 + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = nb + tx * 4 + j;
            if (gn >= N) continue;
            float r = alpha * acc[i][j];
            if (beta != 0.f) r += beta * C[(size_t)gm * ldc + gn];
            if ((flags & PDL_BIAS) && bias) r += bias[gn];
            if ((flags & PDL_RELU) && 0.f > r) r = 0.f;
            C[(size_t)gm * ldc + gn] = r;
        }
    }
}

// Exact fp32 direct conv on CUDA cores: one thread = one output pixel x 16 channels.
__global__ void __launch_bounds__(128) simt_conv_kernel(const float *__restrict__ x,
                                                        const float *__restrict__ w,
                                                        const float *__restrict__ bias,
                                                        float *__restrict__ y, int N, int CT,
                                                        int KT, int H, int W, int R, int S,
                                                        int stride, int pad, int P, int Q,
                                                        unsigned flags) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = (long long)N * KT * P * Q;
    if (idx >= total) return;
    const int q = idx % Q;
    const int pp = (idx / Q) % P;
    const int kt = (idx / ((long long)Q * P)) % KT;
    const int n = idx / ((long long)Q * P * KT);
    float acc[16] = {};
    for (int ct = 0; ct < CT; ++ct)
        for (int r = 0; r < R; ++r) {
            const int ih = pp * stride + r - pad;
            if (ih < 0 || ih >= H) continue;
            for (int s = 0; s < S; ++s) {
                const int iw = q * stride + s - pad;
                if (iw < 0 || iw >= W) continue;
                const float *xi = x + ((((size_t)n * CT + ct) * H + ih) * W + iw) * 16;
                const float *wb = w + ((((size_t)kt * CT + ct) * R + r) * S + s) * 256;
                for (int c = 0; c < 16; ++c) {
                    const float a = xi[c];
#pragma unroll
                    for (int k = 0; k < 16; ++k) acc[k] = fmaf(__ldg(wb + c * 16 + k), a, acc[k]);
                }
            }
        }
    float *yo = y + ((((size_t)n * KT + kt) * P + pp) * Q + q) * 16;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        float r = acc[k];
        if ((flags & PDL_BIAS) && bias) r += bias[kt * 16 + k];
        if ((flags & PDL_RELU) && 0.f > r) r = 0.f;
        yo[k] = r;
    }
}

// Unfused element-wise pass y = max(y + b, 0) over nKhw16k (float4 vectorised).
__global__ void bias_relu_kernel(float4 *__restrict__ y, const float4 *__restrict__ bias,
                                 long long n4, int pq, int KT, unsigned flags) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
        float4 v = y[i];
        if ((flags & PDL_BIAS) && bias) {
            const int kt = (int)((i / (4LL * pq)) % KT);
            const float4 b = __ldg(bias + kt * 4 + (int)(i & 3));
            v.x += b.x; v.y += b.y; v.z += b.z; v.w += b.w;
        }
        if (flags & PDL_RELU) {
            v.x = (0.f > v.x) ? 0.f : v.x;
            v.y = (0.f > v.y) ? 0.f : v.y;
            v.z = (0.f > v.z) ? 0.f : v.z;
            v.w = (0.f > v.w) ? 0.f : v.w;
        }
        y[i] = v;
    }
}

// Weight prepack KCRS16c16k -> packed[plane][ct][r*S+s][k][c] (K-major rows of
// 16 input channels per output channel k); plane 0 = hi (or raw for TF32),
// plane 1 = lo = w - tf32(w) for 3xTF32.
__global__ void prepack_weights_kernel(const float *__restrict__ w, float *__restrict__ out,
                                       int CT, int KT, int RS, int split) {
    const long long total = (long long)KT * CT * RS * 256;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        // source index order: kt, ct, rs, c, k
        const int k = i & 15;
        const int c = (i >> 4) & 15;
        long long t = i >> 8;
        const int rs = t % RS;
        t /= RS;
        const int ct = t % CT;
        const int kt = (int)(t / CT);
        const float v = w[i];
        const size_t dst = ((((size_t)ct * RS + rs) * (KT * 16)) + (size_t)kt * 16 + k) * 16 + c;
        if (split) {
            const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
            out[dst] = h;
            out[dst + total] = v - h;
        } else {
            out[dst] = v;
        }
    }
}

}  // namespace pdl
