// pdl_kernels.cu -- sm_100a kernels for the PolyDL hot path:
//   * tile_mma_kernel: warp-specialised implicit-GEMM engine shared by the
//     blocked convolution (Fig. 9 nest) and the row-major
//     GEMM (Fig. 1).  TMA stages operand tiles into 64/128B
//     swizzled shared memory, one elected thread issues tcgen05.mma kind::tf32
//     with the fp32 accumulator in TMEM, and eight epilogue warps drain TMEM
//     through registers, applying the fused bias + ReLU (Alg. 3, PAPER.md:
//     566-596) before the only store of the output (TMA box stores).
//   * 3xTF32: four staging warps copy each landed A row into TMEM as
//     hi = x (the tensor core truncates to tf32) and lo = x - tf32(x); the MMA
//     warp issues hi*hi + hi*lo + lo*hi with A read from TMEM.  Conv weights
//     are split once at prepack; the GEMM's B lo is formed in shared memory.
//   * stem (C <= 4 real channels, e.g. ResNet's 3->64 7x7/2): the whole input
//     halo of a 16x8-pixel tile is one stage (even / odd input columns as two
//     boxes for stride 2); the staging warps gather tap-aligned 16-value chunks;
//     3xTF32 issues fused-B MMAs (Ahi x [Bhi | Blo] at N=128, Alo x Bhi at N=64).
//   * persistent work units: (M tile, N tile[, split-K range]); segment tiles
//     stack 128-byte-aligned row boxes spanning images for small 1x1 maps;
//     programmatic dependent launch (griddepcontrol) overlaps the prologue with
//     the previous kernel on the stream.
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

enum { KIND_GEMM = 0, KIND_CONV = 1, KIND_STEM = 2 };

// Diagnostic switches (flags bits >= 8): results are WRONG when set; used only to
// attribute time between pipeline roles (scripts/probe_*roles*.py).  Compiled in only
// with -DPDL_DIAG (PDL_DIAG=1 python -m paper_2006_02230_b200.build): the product
// library has no such branches and rejects the bits.
enum : unsigned {
    DBG_NO_A_TMA = 1u << 8,     // producer skips the A loads
    DBG_NO_STAGE_ST = 1u << 9,  // staging warps skip the tcgen05.st into TMEM
    DBG_NO_EPI_STORE = 1u << 10,  // epilogue skips the global stores
    DBG_NO_MMA = 1u << 11,        // MMA warp commits without issuing the MMAs
    DBG_NO_GATHER = 1u << 12      // stem staging skips the halo reads (stores zeros)
};
constexpr unsigned kDiagBits = 0x1f00u;
#ifdef PDL_DIAG
#define PDL_DBG(p, bit) (((p).flags & (bit)) != 0)
#else
#define PDL_DBG(p, bit) false
#endif

// Division by a runtime constant without the ~100-cycle integer divide: q = umulhi(x, mul) >> shr
// (mul = ceil(2^(31 + ceil(log2 d)) / d); exact for 0 <= x < 2^31).  The tile decode of every role
// divides by the tile-grid extents once per work unit; with hardware divides one decode is ~700
// cycles, on the critical path of short tiles' epilogues.
struct FastDiv {
    unsigned mul, shr;
    int d;
};
inline FastDiv make_fastdiv(int d) {
    FastDiv f{0u, 0u, d > 0 ? d : 1};
    if (f.d > 1) {
        unsigned a = 0;
        while ((1u << a) < (unsigned)f.d) ++a;  // ceil(log2 d)
        const unsigned p = 31 + a;
        f.mul = (unsigned)(((1ull << p) + (unsigned)f.d - 1) / (unsigned)f.d);
        f.shr = p - 32;
    }
    return f;
}
__device__ __forceinline__ int fdiv(int x, const FastDiv &f) {
    return f.d == 1 ? x : (int)(__umulhi((unsigned)x, f.mul) >> f.shr);
}

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
    int box_w, box_h;      // stem: halo tile (input pixels x input rows) of one output tile
    int halo_odd;          // packed stride-2 stem: byte offset of the odd-column halo region
                           // (0: one contiguous halo box)
    // segment tiles (conv, small maps): an M tile is seg_tile consecutive "bands" of the
    // (image group, output row) sequence -- a band is one output row of seg_imgs images
    // (1 for even Q, 2 for odd Q, so a band is a multiple of 128 bytes) -- loaded as up to
    // three exact-height boxes {Q, h rows, seg_imgs images} stacked at 128-byte-aligned smem
    // offsets (TMA swizzles by absolute smem address, so the stack is the canonical SW64
    // tile; the epilogue stores the same boxes).  seg_mode 0: box tiles.
    int seg_mode, seg_tile, seg_bytes, seg_imgs;
    int res_bytes;         // resident-weight conv: bytes of one weight plane of the N-tile
    int m_tiles;           // number of M tiles
    int n_tiles;           // number of N tiles
    int raster;            // bit 0: M-tiles fastest tile order (see tile_coord)
    int seg_kb;            // k-blocks per TMEM accumulation segment
    // split-K: every tile's reduction is cut into `split` ranges of kb_per k-blocks,
    // computed as separate work units; each writes its fp32 partial to part, and the
    // last of a tile's units to arrive (ctr[tile], self-resetting) sums the partials in
    // split order and runs the epilogue.  split == 1: no workspace is touched.
    int split, kb_per;
    float *part;
    int *ctr;
    unsigned long long *trace;  // PDL_TRACE builds: per-event clock64 stamps of block 0
    // divisors of the tile decode (filled by launch_tile from the fields above)
    FastDiv fd_n_tiles, fd_m_tiles, fd_tiles_w, fd_tiles_h, fd_split, fd_P, fd_rs, fd_S, fd_seg;
};

// Timeline tracing (PDL_TRACE builds only): block 0 stamps clock64 at each
// pipeline hand-off; slot = event * kTraceN + index.
constexpr int kTraceN = 4096;
enum TraceEv {
    TR_P_ISSUE = 0,   // producer: stage free, issuing TMA for k-block i
    TR_S_FULL,        // staging: data of k-block i landed
    TR_S_TFREE,       // staging: TMEM slot free
    TR_S_DONE,        // staging: A slot ready (tready arrived)
    TR_M_READY,       // MMA: k-block i ready
    TR_M_ISSUED,      // MMA: k-block i issued + committed
    TR_E_FULL,        // epilogue: segment g landed in TMEM
    TR_E_DRAINED,     // epilogue: segment g drained
    TR_E_STORED,      // epilogue: tile j stored
    TR_M_WAITED,      // MMA: barrier observed (before tcgen05.fence::after_thread_sync)
    TR_M_LOOP,        // MMA: top of k-block loop
    TR_KERNEL,        // [0] kernel entry, [1] prologue done (barriers, TMEM), [2] after griddepcontrol.wait,
                      // [3] before the final CTA sync (warp 8 lane 0), [4] after TMEM dealloc, [5] producer entered,
                      // [6] its first tile decoded, [7] before its first stage wait
    TR_SPLIT,         // split-K, per unit j: [2j] partial written + counter bumped, [2j+1] reduction read back
    TR_COUNT
};
__device__ __forceinline__ void trace_ev(const TileParams &p, int ev, int i) {
#ifdef PDL_TRACE
    if (p.trace && blockIdx.x == 0 && i < kTraceN) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
        p.trace[ev * kTraceN + i] = t;
    }
#else
    (void)p; (void)ev; (void)i;
#endif
}

constexpr int kSegMaxRows = 10;  // segment tiles: one box map per row count 1..10
struct TmaMaps {
    // conv box tiles: a[parity] ((row, col) parity map for stride 2, a[0] for stride 1);
    // conv segment tiles: a[h - 1] = box of h output rows; GEMM / stem: a[0..1]
    CUtensorMap a[kSegMaxRows];
    CUtensorMap b;
    CUtensorMap y[kSegMaxRows];  // conv / stem output [N][KT][P][Q][16] (TMA-stored epilogue)
};

// Shared-memory tiles of one pipeline stage.
//   GEMM: A [128 rows][32 fp32]   SW128 K-major        B [BN/32][32 k][32 n] SW128_B32 MN-major
//   CONV: A [CG][128 rows][16]    SW64  K-major        B [CG/2][BN rows][32] SW128 K-major
//                                                      (CG = 1: B [BN rows][16] SW64)
//   STEM: A halo tile [rows][px][4 fp32], no swizzle   B resident: [plane][chunk][BN][4]
constexpr int kStemHaloBytes = 16384;
#ifndef PDL_EPI_BUFS
#define PDL_EPI_BUFS 2
#endif
// output-box ring depth for the output-heavy resident-weight 1x1 convs: their epilogue
// is the bottleneck -- a 16-channel box store takes ~1000 cycles to
// release its smem (traces: ResNet layers 4/8 spend 4100-4300 cycles per tile storing)
#ifndef PDL_STEM_WIDE_EPI
#define PDL_STEM_WIDE_EPI 0
#endif
#ifndef PDL_EPI_BUFS_WIDE
#define PDL_EPI_BUFS_WIDE 4
#endif  // stem halo tile: box_w * box_h * 16 B
// For KIND_STEM the CG template parameter selects the reduction packing:
//   CG = 1: k-block = one kernel row, K = 8 taps x 4 channels = 32 (any C <= 4, S <= 8)
//   CG = kStemPackedCG: K = (r, s, c) dense for C = 3, 7x7 (147 -> 160), two k-blocks of
//           80 per tile (one TMEM slot each): 29% fewer MMAs and 5 MMA-warp passes -> 2
constexpr int kStemPackedCG = 5;

// PAIR: the tile is computed by a CTA pair with cta_group::2 MMAs (M = 256): each
// CTA stages its own 128 A rows and holds BN/2 rows of B.
template <int KIND, int BN, int CG, bool PAIR = false>
struct Geo {
    static constexpr int BM = 128;
    // stem: one stage = the whole input halo of a tile, 4 channels (16 B) per pixel
    static constexpr int A_SUB = KIND == KIND_GEMM ? BM * 128 : KIND == KIND_CONV ? BM * 64 : kStemHaloBytes;
    // conv weights: 128-byte rows (32 input channels, SW128) whenever CG >= 2 -- 64-byte
    // SW64 rows make every tensor-core B read 2-way bank conflicted
    static constexpr int B_ROW = (KIND == KIND_CONV && CG == 1) ? 64 : 128;
    static constexpr int NB = KIND == KIND_CONV ? (CG >= 2 ? CG / 2 : 1) : 1;
    static constexpr int B_SUB = KIND == KIND_STEM ? BN * 128 : (PAIR ? BN / 2 : BN) * B_ROW;
    static constexpr int NSUB = KIND == KIND_CONV ? CG : 1;
    static constexpr int A_BYTES = A_SUB * NSUB;
    static constexpr int B_BYTES = B_SUB * NB;
    static constexpr int KK = KIND == KIND_CONV ? 2 : 4;  // K=8 MMAs per sub-tile
    static constexpr bool STEM_PACKED = KIND == KIND_STEM && CG == kStemPackedCG;
    static constexpr int KS = KIND == KIND_CONV ? 16 * CG : STEM_PACKED ? 80 : 32;  // K per k-block
    static constexpr int NK = KS / 8;                                // K=8 MMA steps per stage
    // B-descriptor advance (16-byte units) of K=8 step j within a stage
    __host__ __device__ static constexpr uint32_t boff(int j) {
        return KIND == KIND_GEMM ? (uint32_t)(j * 64)                   // 8 k-rows x 128 B
             : KIND == KIND_CONV ? (uint32_t)(((j * 32) / B_ROW * B_SUB + (j * 32) % B_ROW) / 16)
                                 : (uint32_t)(j * 2 * BN);             // stem: 2 chunks x BN x 16 B
    }
};

constexpr int kStemMaxR = 7;  // resident stem weights: R <= 7 kernel rows

// one plane of the stem's resident weights: (k-blocks x KS/4 chunks) x BN x 16 B
template <int BN, int CG>
struct StemW {
    static constexpr int CHUNKS = CG == kStemPackedCG ? 2 * 20 : kStemMaxR * 8;
    static constexpr int PLANE_BYTES = CHUNKS * BN * 16;
};

// TS = A operand staged in TMEM by the split warps (3xTF32, and the stem's tap gather).
// SMEM stages (TMA ring) and TMEM A slots (split -> MMA ring) are separate rings.
// RESW (1x1 conv): the N-tile's whole weight slice stays resident in smem (RESW
// bytes reserved per plane), loaded once per CTA; stages then carry A only.
// HALO (3xTF32 spatial conv, stride 1): the input halo of a tile -- (BW+S-1) x (BH+R-1)
// pixels of CG 16-channel sub-tiles -- is loaded once per channel group into one of two
// halo buffers, and the staging warps read every tap's shifted window from it; stages
// then carry B only (the per-tap A boxes re-read every input pixel R*S times).
constexpr int kHaloSub = 16384;  // bytes per 16-channel sub-tile of a halo buffer (<= 256 px)

template <int KIND, int BN, int CG, bool SPLIT3, bool PAIR = false, int RESW = 0, bool HALO = false>
struct Smem {
    using G = Geo<KIND, BN, CG, PAIR>;
    // A staged in TMEM (TS MMAs): 3xTF32, the stem, and halo convs (TF32 too: the shifted
    // tap windows are read by the staging warps, not by the tensor core)
    static constexpr bool TS = SPLIT3 || KIND == KIND_STEM || HALO;
    static constexpr int PLANES = SPLIT3 ? 2 : 1;  // B planes resident in a stage (hi, lo)
    // B planes loaded by TMA: conv / stem weights carry both (prepacked once); the
    // GEMM loads B itself and the staging warps form lo = B - tf32(B) in smem.
    // (Forming the conv weights' lo on chip too was measured 5-12% slower: the
    // staging warps' smem traffic costs more than the TMA bytes it saves.)
    static constexpr int LOAD_PLANES = KIND == KIND_GEMM ? 1 : PLANES;
    // stem weights stay resident for the whole kernel (one N-tile per CTA)
    static constexpr int W_BYTES = KIND == KIND_STEM ? PLANES * StemW<BN, CG>::PLANE_BYTES : PLANES * RESW;
    static constexpr int STAGE = HALO ? G::B_BYTES * PLANES
                                 : (KIND == KIND_STEM || RESW) ? G::A_BYTES : G::A_BYTES + G::B_BYTES * PLANES;
    static constexpr int HALO_BUF = CG * kHaloSub;
    // two halo buffers (the next channel group's halo loads during this one's taps), one
    // for 64-channel k-blocks (two 64 KB buffers would leave two weight stages)
    static constexpr int HALO_NBUF = CG >= 4 ? 1 : 2;
    static constexpr int HALO_BYTES = HALO ? HALO_NBUF * HALO_BUF : 0;
    // conv / stem epilogue: one 128-row x 16-channel (8 KB, SW64) TMA-store buffer
    // per column half of the epilogue warps
    // two output-box buffers per column half: a box is filled while the previous
    // one drains (one buffer serialised the epilogue on each TMA store's smem read)
    // (only where smem keeps >= 4 stages: with 64 KB weight planes a 4-deep ring leaves
    // 2 stages and layer 5 ran 28% slower; the stem measured no change)
    // (batched 4-deep rings on every BN=128 layer cost those layers a stage: 3-15% slower)
    static constexpr int EPI_BUFS = ((RESW > 0 && RESW <= 32768) || (KIND == KIND_STEM && PDL_STEM_WIDE_EPI))
                                        ? PDL_EPI_BUFS_WIDE : PDL_EPI_BUFS;
    static constexpr int EPI_BYTES = KIND == KIND_GEMM ? 0 : 2 * EPI_BUFS * 8192;
    // 227 KB opt-in dynamic smem per CTA, minus 2 KB for barriers + base alignment
    static constexpr int BUDGET = 232448 - 2048 - W_BYTES - EPI_BYTES - HALO_BYTES;
    static constexpr int S0 = BUDGET / STAGE;
    static constexpr int STAGES = S0 > 16 ? 16 : S0;
    static constexpr int SLOT_COLS = SPLIT3 ? 2 * G::KS : G::KS;  // TMEM columns per A slot
    // 3xTF32 with 256 columns: ONE 256-column accumulator (two would fill TMEM and leave no A slots);
    // the epilogue drains it at every segment end while the MMAs wait
    static constexpr bool ONE_ACC = SPLIT3 && BN > 128;
    static constexpr int A_SLOT0 = ONE_ACC ? BN : 2 * BN;         // after the accumulator(s)
    static constexpr int T0 = TS ? (512 - A_SLOT0) / SLOT_COLS : 1;
    static constexpr int TSLOTS = T0 > 8 ? 8 : T0;
    static constexpr int A_OFF = 0;
    static constexpr int B_HI = HALO ? 0 : G::A_BYTES;
    static constexpr int B_LO = B_HI + G::B_BYTES;
    static constexpr int HALO_OFF = STAGES * STAGE;   // halo buffers (HALO)
    static constexpr int W_OFF = HALO_OFF + HALO_BYTES;  // stem / resident weights
    static constexpr int EPI_OFF = W_OFF + W_BYTES;
    static constexpr int BAR_OFF = EPI_OFF + EPI_BYTES;
    static constexpr int TOTAL = BAR_OFF + 1024 + 1024;  // barriers + alignment slack
    static_assert(TOTAL <= 232448, "shared memory over the 227 KB per-CTA limit");
    static constexpr uint32_t TMEM_COLS = TS ? 512 : 2 * BN;
    static_assert(STAGES >= 2, "tile too large for a 2-stage pipeline");
    static_assert(!TS || TSLOTS >= 2, "not enough TMEM for two A slots");
};

__device__ __forceinline__ float tf32_lo(float x) {
    // the tensor core truncates fp32 operands to tf32 (probed on B200), so the
    // hi part is x itself and lo = x - trunc_tf32(x), exact in fp32
    return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ float4 lds128(uint32_t saddr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(saddr));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t saddr, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// lo = x - tf32(x) for `bytes` of shared memory (element-wise, layout-agnostic).
__device__ __forceinline__ void split_lo_smem(uint32_t src, uint32_t lo, int bytes, int tid,
                                              int nthreads) {
    const int n = bytes >> 4;
#pragma unroll 4
    for (int i = tid; i < n; i += nthreads) {
        const float4 v = lds128(src + i * 16);
        sts128(lo + i * 16, make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w)));
    }
}

// Fused element-wise epilogue of Alg. 3 on output column(s) from
// `col`, in the reference's order of operations: PDL_SCALE multiplies by scale[k]
// (batch-norm inference affine, scale stored after the K shifts in `bias`), PDL_BIAS
// adds bias[k], PDL_RELU is Python's max(v, 0.0) (keep v unless 0 > v), PDL_RELU6 is
// min(max(v, 0.0), 6.0) (keep v unless 6 < v).  Columns >= n_out read nothing.
__device__ __forceinline__ float epi_relu(unsigned f, float v) {
    if (f & (PDL_RELU | PDL_RELU6)) v = (0.f > v) ? 0.f : v;
    if (f & PDL_RELU6) v = (6.f < v) ? 6.f : v;
    return v;
}
__device__ __forceinline__ float epilogue1(unsigned f, const float *bias, int n_out, int col, float v) {
    if (bias && col < n_out) {
        if (f & PDL_SCALE) v = __fmul_rn(v, __ldg(bias + n_out + col));
        if (f & PDL_BIAS) v = __fadd_rn(v, __ldg(bias + col));
    }
    return epi_relu(f, v);
}
// FULL = false: bias + ReLU only.  The tile kernels compile it into their default
// instances and get the scale / ReLU6 form only in separate EPIX instances: even
// one extra select per element in the epilogue loop moved the output-heavy layers
// (stem, 2, 4, 8) by 4-16% (register allocation / code layout of the big kernel),
// measured with scripts/ab_libs.sh.
template <bool FULL>
__device__ __forceinline__ float4 epilogue4(unsigned f, const float *bias, int n_out, int col, float4 r) {
    if constexpr (FULL) {
        if (bias && col < n_out) {
            if (f & PDL_SCALE) {
                const float4 s = __ldg(reinterpret_cast<const float4 *>(bias + n_out + col));
                r.x = __fmul_rn(r.x, s.x); r.y = __fmul_rn(r.y, s.y);
                r.z = __fmul_rn(r.z, s.z); r.w = __fmul_rn(r.w, s.w);
            }
            if (f & PDL_BIAS) {
                const float4 b = __ldg(reinterpret_cast<const float4 *>(bias + col));
                r.x = __fadd_rn(r.x, b.x); r.y = __fadd_rn(r.y, b.y);
                r.z = __fadd_rn(r.z, b.z); r.w = __fadd_rn(r.w, b.w);
            }
        }
        r.x = epi_relu(f, r.x); r.y = epi_relu(f, r.y); r.z = epi_relu(f, r.z); r.w = epi_relu(f, r.w);
    } else {
        if ((f & PDL_BIAS) && bias && col < n_out) {
            const float4 b = __ldg(reinterpret_cast<const float4 *>(bias + col));
            r.x += b.x; r.y += b.y; r.z += b.z; r.w += b.w;
        }
        if (f & PDL_RELU) {
            r.x = (0.f > r.x) ? 0.f : r.x;
            r.y = (0.f > r.y) ? 0.f : r.y;
            r.z = (0.f > r.z) ? 0.f : r.z;
            r.w = (0.f > r.w) ? 0.f : r.w;
        }
    }
    return r;
}

// Epilogue for 16 consecutive output columns [col0, col0+16) of one row.
template <int KIND, bool EPIX>
__device__ __forceinline__ void store16(const TileParams &p, float *dst, int col0,
                                        const float *v) {
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
        r = epilogue4<EPIX>(p.flags, p.bias, p.n_out, col, r);
        *reinterpret_cast<float4 *>(dst + q4 * 4) = r;
    }
}

// Persistent implicit-GEMM tile engine.  gridDim.x CTAs (<= #SMs, a multiple of
// the N-tile count so every CTA keeps one N-tile), one per SM; CTA b processes
// tiles b, b + gridDim.x, ... (N-tiles fastest: concurrent CTAs share
// activation rows through L2).
//   warp 0       TMA producer (one lane), runs ahead across tile boundaries
//   warp 1       tcgen05.mma issuer (one lane)
//   warp 2       TMEM allocator
//   warps 4-7    A staging (TS modes): thread = tile row = TMEM lane; reads its
//                row of the landed tile (stem: gathers the taps), writes hi (= x,
//                the tensor core truncates) and lo = x - tf32(x) into a TMEM A
//                slot with tcgen05.st; the GEMM also forms B's lo in smem
//   warps 8-15   TMEM drain + epilogue; warp 8+e owns TMEM lanes 32*(e%4).. and
//                output columns [(e/4)*BN/2, (e/4+1)*BN/2)
// Rings: SMEM stages  full[s] (TMA -> staging) / empty[s] (staging [+ MMA] -> TMA);
//        TMEM A slots tready[t] (staging -> MMA) / tfree[t] (MMA -> staging);
//        accumulators tmem_full[b] (MMA -> epilogue) / tmem_empty[b] (epilogue -> MMA).
// 3xTF32 issues hi*hi + hi*lo + lo*hi per K=8 step.  The reduction of every tile
// is cut into segments of p.seg_kb k-blocks; each segment accumulates in one of
// two TMEM buffers (ping-pong, continuing across tiles) and is drained into
// fp32 registers with round-to-nearest adds.  The tensor core's accumulator
// truncates, so an unsegmented K=4096 sum drifts to ~3e-5 relative error;
// 256-element segments keep it near 3e-6 at any K.  The ping-pong also lets
// tile i's epilogue overlap tile i+1's first segment.
constexpr int kThreads = 512;
constexpr int kSplitWarp0 = 4;
constexpr int kEpiWarp0 = 8;
constexpr int kEpiThreads = 256;

struct TileCoord {
    int n0;          // first output column
    int m0;          // GEMM: first row
    int q0, p0, i0;  // conv: first output col / row / image of the pixel box
};

template <int KIND, int BN>
__device__ __forceinline__ TileCoord tile_coord(const TileParams &p, int tile) {
    TileCoord c;
    // raster bit 0: M-tiles fastest (consecutive CTAs share a weight N-tile through L2);
    // default N-tiles fastest (they share activation rows).  The host clears the bit for
    // the stem, resident-weight tiles and clusters (one N-tile per CTA / cluster lockstep).
    int mt, nt;
    if (p.raster & 1) {
        nt = fdiv(tile, p.fd_m_tiles);
        mt = tile - nt * p.m_tiles;
    } else {
        mt = fdiv(tile, p.fd_n_tiles);
        nt = tile - mt * p.n_tiles;
    }
    c.n0 = nt * BN;
    c.m0 = 0;
    c.q0 = 0;
    c.p0 = 0;
    c.i0 = 0;
    if (KIND == KIND_GEMM) {
        c.m0 = mt * 128;
    } else if (p.seg_mode) {
        // segment tiles: bands [mt * seg_tile, +seg_tile); i0 = image group, p0 = first row
        const int g0 = mt * p.seg_tile;
        c.i0 = fdiv(g0, p.fd_P);
        c.p0 = g0 - c.i0 * p.P;
    } else {
        int t = mt;
        const int t1 = fdiv(t, p.fd_tiles_w);
        const int tw = t - t1 * p.tiles_w;
        t = fdiv(t1, p.fd_tiles_h);
        const int th = t1 - t * p.tiles_h;
        c.q0 = tw * p.BW;
        c.p0 = th * p.BH;
        c.i0 = t * p.BNI;
    }
    return c;
}

// Packed ResNet-stem gather (C=3, R=S=7), tap-aligned: reduction chunk CH (0..9)
// of 16 values holds taps 5*CH .. 5*CH+4 (tap = r*7 + s, 3 channels each) and a
// zero, so every tap is read from the halo exactly once per tile (147 real
// values of 160).  col[s] = byte offset of tap column s for this thread (the
// stride-2 halo is split into even / odd input-column regions, so the 16-byte
// pixels a warp reads for one tap are contiguous: 4 smem wavefronts, not 8).
template <int CH>
__device__ __forceinline__ void stem_gather_chunk(uint32_t sa, uint32_t row_step, const uint32_t (&col)[7],
                                                  bool live, float (&x)[16]) {
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int tap = 5 * CH + i;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (tap < 49 && live) v = lds128(sa + (uint32_t)(tap / 7) * row_step + col[tap % 7]);
        x[3 * i] = v.x;
        x[3 * i + 1] = v.y;
        x[3 * i + 2] = v.z;
    }
    x[15] = 0.f;
}
// chunk c (0..4) of packed k-block KB (5 chunks = 80 values each)
template <int KB>
__device__ __forceinline__ void stem_gather_kb(int c, uint32_t sa, uint32_t row_step, const uint32_t (&col)[7],
                                               bool live, float (&x)[16]) {
    switch (c) {
        case 0: stem_gather_chunk<KB * 5 + 0>(sa, row_step, col, live, x); break;
        case 1: stem_gather_chunk<KB * 5 + 1>(sa, row_step, col, live, x); break;
        case 2: stem_gather_chunk<KB * 5 + 2>(sa, row_step, col, live, x); break;
        case 3: stem_gather_chunk<KB * 5 + 3>(sa, row_step, col, live, x); break;
        default: stem_gather_chunk<KB * 5 + 4>(sa, row_step, col, live, x); break;
    }
}

// EPIX: the extended fused epilogue (PDL_SCALE, PDL_RELU6) -- separate instances, see epilogue4
template <int KIND, int BN, int CG, bool SPLIT3, int CL, bool PAIR = false, int RESW = 0, bool HALO = false,
          bool EPIX = false>
__global__ void __launch_bounds__(kThreads, 1)
    tile_mma_kernel(const __grid_constant__ TmaMaps maps, const TileParams p) {
    static_assert(CL == 1 || KIND != KIND_STEM, "the stem keeps its weights resident");
    static_assert(!PAIR || (CL == 2 && KIND == KIND_CONV && SPLIT3), "pairs: 3xTF32 conv, cluster 2");
    static_assert(!RESW || (KIND == KIND_CONV && CL == 1 && !PAIR && SPLIT3), "resident weights: 3xTF32 conv");
    static_assert(!HALO || (KIND == KIND_CONV && CL == 1 && !PAIR && !RESW), "halo: conv, cluster 1");
    static_assert(BN <= 128 || (KIND == KIND_CONV && !HALO && !RESW && CL == 1 && !PAIR),
                  "BN=256: conv, cluster 1");
    using G = Geo<KIND, BN, CG, PAIR>;
    using L = Smem<KIND, BN, CG, SPLIT3, PAIR, RESW, HALO>;
    constexpr bool TS = L::TS;
    constexpr int STAGES = L::STAGES;
    // fused-B stem (3xTF32, packed): one accumulator of 2*BN columns ([AhBh + AlBh | AhBl]),
    // so no accumulator double-buffering (the epilogue drains it in ~150 cycles)
    constexpr bool FUSED = KIND == KIND_STEM && G::STEM_PACKED && SPLIT3;
    constexpr int PL = SPLIT3 ? 2 : 1;  // stem weight planes, layout [kb][chunk][plane][BN][4]
    // accumulator buffer / mbarrier parity of TMEM segment g
    constexpr bool ONE_ACC = FUSED || L::ONE_ACC;
    // 3xTF32 at 256 columns: the epilogue threads sum 128 columns of segments in registers, past
    // the 128 registers a 512-thread CTA gives each thread -- the warpgroups trade registers
    // (setmaxnreg): warps 0-3 (TMA, MMA) 48, the staging warps 80, the epilogue warps 192
    constexpr bool REGTRADE = L::ONE_ACC;
    auto acc_buf = [](int g) { return ONE_ACC ? 0 : (g & 1); };
    auto acc_par = [](int g) { return (uint32_t)(ONE_ACC ? (g & 1) : ((g >> 1) & 1)); };
    constexpr int TSLOTS = L::TSLOTS;
    constexpr int HALF = BN / 2;  // columns per epilogue warp
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem =
        reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);
    uint64_t *empty = full + STAGES;
    uint64_t *tready = empty + STAGES;
    uint64_t *tfree = tready + 8;
    uint64_t *tmem_full = tfree + 8;       // [2]
    uint64_t *tmem_empty = tmem_full + 2;  // [2]
    uint64_t *wfull = tmem_empty + 2;      // stem weights landed
    uint64_t *hfull = wfull + 1;           // [2] halo buffer landed (HALO)
    uint64_t *hempty = hfull + 2;          // [2] halo buffer read by every tap (HALO)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(hempty + 2);
    volatile uint32_t *split_flag = tmem_slot + 1;  // split-K: "this CTA reduces the tile"

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) trace_ev(p, TR_KERNEL, 0);
    const int num_tiles = p.m_tiles * p.n_tiles;
    const int seg_kb = p.seg_kb;
    // Cluster of CL CTAs = CL consecutive M-tiles of one N-tile ("super-tile"),
    // processed in lockstep; each CTA loads 1/CL of the B tile and multicasts it.
    const int rank = CL > 1 ? (int)cluster_ctarank() : 0;
    const int cid = blockIdx.x / CL;
    const int ncl = gridDim.x / CL;
    const int num_super = ((p.m_tiles + CL - 1) / CL) * p.n_tiles;
    const int SPL = p.split;                 // 1 unless split-K
    const int num_units = num_super * SPL;   // work unit u = (super-tile u / SPL, split u % SPL)
    const uint16_t cl_mask = (uint16_t)((1u << CL) - 1);
    auto tile_of = [&](int st) {  // M-tile may exceed m_tiles (phantom: loads OOB zeros, stores masked)
        const int mg = fdiv(st, p.fd_n_tiles);
        const int nt = st - mg * p.n_tiles;
        return (mg * CL + rank) * p.n_tiles + nt;
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch(&maps.b);
        tma_prefetch(&maps.a[0]);
        if (KIND == KIND_CONV && p.stride == 2 && !p.seg_mode) {
            tma_prefetch(&maps.a[1]);
            tma_prefetch(&maps.a[2]);
            tma_prefetch(&maps.a[3]);
        }
        // stem: only the staging warps read a stage; conv/GEMM: staging (A) + the MMA
        // commits of all CL CTAs (B is multicast into every CTA of the cluster)
        // pairs: the leader's one multicast commit per k-block reaches both CTAs;
        // tready / tmem_empty of the leader count both CTAs' staging / epilogue
        const uint32_t empty_count = HALO ? 1 : (KIND == KIND_STEM || RESW) ? 128 : PAIR ? 129 : (TS ? 128 : 0) + CL;
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], empty_count);
        }
        for (int t = 0; t < TSLOTS; ++t) {
            mbar_init(&tready[t], PAIR ? 256 : 128);
            mbar_init(&tfree[t], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tmem_full[b], 1);
            mbar_init(&tmem_empty[b], PAIR ? 2 * kEpiThreads : kEpiThreads);
        }
        mbar_init(wfull, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&hfull[b], 1);
            mbar_init(&hempty[b], 128);
        }
        fence_mbar_init();
    }
    // The producer decodes its first unit here, while warp 2 allocates TMEM and the CTA syncs
    // (timelines of short launches: ~0.7 us between the end of the prologue and the first TMA
    // issue went into this decode)
    TileCoord tc_first = {};
    if (warp == 0 && lane == 0 && KIND != KIND_STEM && cid < num_units)
        tc_first = tile_coord<KIND, BN>(p, tile_of(fdiv(cid, p.fd_split)));
    if (warp == 2) {
        if constexpr (PAIR) tmem_alloc2<L::TMEM_COLS>(tmem_slot);
        else tmem_alloc<L::TMEM_COLS>(tmem_slot);
    }
    tc_fence_before();
    if (CL > 1) cluster_sync();  // peers multicast into our barriers: they must exist
    else __syncthreads();
    tc_fence_after();
    // programmatic dependent launch: let the next kernel on the stream start its own
    // prologue now, and touch global memory only once the previous grid has finished
    // (a no-op when launched without the attribute)
    if (threadIdx.x == 0) trace_ev(p, TR_KERNEL, 1);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) trace_ev(p, TR_KERNEL, 2);
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t smem0 = smem_u32(smem);
    // REGTRADE: per-warpgroup register budgets (64 + 88 + 2 x 176 registers x 128 threads = 64 K), each
    // set at the top of the warpgroup's own branch so that the code it dominates is allocated to it
    if (warp < kSplitWarp0) {
    if constexpr (REGTRADE) asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            trace_ev(p, TR_KERNEL, 5);
            uint32_t tx;
            if (KIND == KIND_GEMM) tx = (uint32_t)(G::BM * 32 * 4 + BN * 32 * 4);
            else if (KIND == KIND_CONV)
                tx = (uint32_t)((PDL_DBG(p, DBG_NO_A_TMA) || HALO ? 0 : CG * 64 * p.BW * p.BH * p.BNI) +
                                (RESW ? 0 : G::B_BYTES * L::LOAD_PLANES));
            else tx = (uint32_t)(16 * p.box_w * p.box_h * (p.halo_odd ? 2 : 1));
            // HALO: one box of (box_w x box_h x BNI) pixels per 16-channel sub-tile
            const uint32_t htx = (uint32_t)(CG * 64 * p.box_w * p.box_h * p.BNI);
            int hb = 0;
            uint32_t hph = 0;
            if (RESW && blockIdx.x < num_tiles) {
                // the grid is a multiple of n_tiles: this CTA keeps one N-tile throughout
                const int n0 = (blockIdx.x % p.n_tiles) * BN;
                mbar_arrive_expect_tx(wfull, (uint32_t)(L::PLANES * p.res_bytes));
                for (int pl = 0; pl < L::PLANES; ++pl)
                    tma_load_5d(smem + L::W_OFF + pl * RESW, &maps.b, wfull, 0, n0, 0, 0, pl);
            }
            if (KIND == KIND_STEM && blockIdx.x < num_tiles) {  // CL == 1 here
                // resident weights of this CTA's N-tile: [plane][kb][KS/4 chunks][BN][4]
                const int n0 = (blockIdx.x % p.n_tiles) * BN;
                // [kb][chunk][plane][BN][4]: one box covers both planes of every chunk
                mbar_arrive_expect_tx(wfull, (uint32_t)(L::PLANES * p.num_kb * (G::KS / 4) * BN * 16));
                tma_load_5d(smem + L::W_OFF, &maps.b, wfull, 0, n0, 0, 0, 0);
            }
            int s = 0;
            uint32_t ph = 0;
            int kglob = 0;
            if (KIND == KIND_STEM) {
                // one stage = the input halo of a whole output tile; its R k-blocks
                // (kernel rows) are all staged from it
                for (int st = cid; st < num_super; st += ncl, ++kglob) {
                    const TileCoord tc = tile_coord<KIND, BN>(p, tile_of(st));
                    mbar_wait(&empty[s], ph ^ 1);
                    trace_ev(p, TR_P_ISSUE, kglob);
                    mbar_arrive_expect_tx(&full[s], tx);
                    const int c0 = tc.q0 * p.stride - p.pad;  // first input column of the halo
                    if (p.halo_odd) {
                        // stride 2: even and odd input columns as two dense boxes
                        // (a[0] / a[1] index columns 2k / 2k+1)
                        tma_load_5d(smem + s * L::STAGE + L::A_OFF, &maps.a[0], &full[s], 0,
                                    (c0 + (c0 & 1)) / 2, tc.p0 * p.stride - p.pad, 0, tc.i0);
                        tma_load_5d(smem + s * L::STAGE + L::A_OFF + p.halo_odd, &maps.a[1], &full[s], 0,
                                    (c0 - (c0 & 1)) / 2, tc.p0 * p.stride - p.pad, 0, tc.i0);
                    } else {
                        tma_load_5d(smem + s * L::STAGE + L::A_OFF, &maps.a[0], &full[s], 0, c0,
                                    tc.p0 * p.stride - p.pad, 0, tc.i0);
                    }
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
            }
            for (int u = cid; KIND != KIND_STEM && u < num_units; u += ncl) {
                const int st = fdiv(u, p.fd_split);
                const int kb0 = (u - st * SPL) * p.kb_per, kb1 = min(p.num_kb, kb0 + p.kb_per);
                const TileCoord tc = u == cid ? tc_first : tile_coord<KIND, BN>(p, tile_of(st));
                if (u == cid) trace_ev(p, TR_KERNEL, 6);
                for (int kb = kb0; kb < kb1; ++kb, ++kglob) {
                    if constexpr (HALO) {
                        // new channel group (or the first k-block of this unit): its halo
                        const int rs_n = p.R * p.S;
                        const int ctg = fdiv(kb, p.fd_rs);
                        if (kb - ctg * rs_n == 0 || kb == kb0) {
                            mbar_wait(&hempty[hb], hph ^ 1);
                            mbar_arrive_expect_tx(&hfull[hb], htx);
                            uint8_t *hbuf = smem + L::HALO_OFF + hb * L::HALO_BUF;
#pragma unroll
                            for (int c = 0; c < CG; ++c)
                                tma_load_5d(hbuf + c * kHaloSub, &maps.a[0], &hfull[hb], 0, tc.q0 - p.pad,
                                            tc.p0 - p.pad, ctg * CG + c, tc.i0);
                            if (++hb == L::HALO_NBUF) { hb = 0; hph ^= 1; }
                        }
                    }
                    if (kglob == 0) trace_ev(p, TR_KERNEL, 7);
                    mbar_wait(&empty[s], ph ^ 1);
                    trace_ev(p, TR_P_ISSUE, kglob);
                    uint8_t *sp = smem + s * L::STAGE;
                    mbar_arrive_expect_tx(&full[s], tx);
                    if (KIND == KIND_GEMM) {
                        tma_load_2d(sp + L::A_OFF, &maps.a[0], &full[s], kb * 32, tc.m0);
                        for (int c = rank; c < BN / 32; c += CL) {
                            if (CL == 1)
                                tma_load_2d(sp + L::B_HI + c * 4096, &maps.b, &full[s],
                                            tc.n0 + c * 32, kb * 32);
                            else
                                tma_load_2d_mc(sp + L::B_HI + c * 4096, &maps.b, &full[s],
                                               tc.n0 + c * 32, kb * 32, cl_mask);
                        }
                    } else if (KIND == KIND_CONV) {
                        const int rs_n = p.R * p.S;
                        const int ctg = fdiv(kb, p.fd_rs);
                        const int rs = kb - ctg * rs_n;
                        const int r = fdiv(rs, p.fd_S);
                        const int sx = rs - r * p.S;
                        int dh = r - p.pad, dw = sx - p.pad, mi = 0;
                        if (p.stride == 2) {
                            const int ph2 = dh & 1, pw2 = dw & 1;
                            mi = ph2 * 2 + pw2;
                            dh = (dh - ph2) >> 1;
                            dw = (dw - pw2) >> 1;
                        }
                        if (PDL_DBG(p, DBG_NO_A_TMA) || HALO) {
                        } else if (p.seg_mode) {
                            // bands p0.. of image group i0, then the next group(s) from row 0
                            int grp = tc.i0, r = tc.p0, left = p.seg_tile, off = 0;
                            while (left > 0) {
                                const int h = min(left, p.P - r);
#pragma unroll
                                for (int c = 0; c < CG; ++c)
                                    tma_load_5d(sp + L::A_OFF + c * G::A_SUB + off, &maps.a[h - 1], &full[s], 0,
                                                dw, r + dh, ctg * CG + c, grp * p.seg_imgs);
                                off += h * p.seg_bytes;
                                left -= h;
                                ++grp;
                                r = 0;
                            }
                        } else {
#pragma unroll
                            for (int c = 0; c < CG; ++c)
                                tma_load_5d(sp + L::A_OFF + c * G::A_SUB, &maps.a[mi], &full[s], 0,
                                            tc.q0 + dw, tc.p0 + dh, ctg * CG + c, tc.i0);
                        }
                        if (RESW) {
                        } else if (CL == 1 || PAIR) {
                            // pair: this CTA's BN/2 rows of B (the MMA reads both halves)
                            tma_load_5d(sp + L::B_HI, &maps.b, &full[s], 0, tc.n0 + (PAIR ? rank * (BN / 2) : 0),
                                        rs, ctg * G::NB, 0);
                        } else {
                            // this CTA's slice: rows [rank*BN/CL, +BN/CL) of every (plane, nb) sub-tile
                            constexpr int SL = BN / CL;
#pragma unroll
                            for (int pl = 0; pl < L::LOAD_PLANES; ++pl)
#pragma unroll
                                for (int nb = 0; nb < G::NB; ++nb)
                                    tma_load_5d_mc(sp + L::B_HI + pl * G::B_BYTES + nb * G::B_SUB +
                                                       rank * SL * G::B_ROW,
                                                   &maps.b, &full[s], 0, tc.n0 + rank * SL, rs,
                                                   ctg * G::NB + nb, pl, cl_mask);
                        }
                    }
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (whole warp, one elected lane issues) ============
        {
            constexpr uint32_t idesc = idesc_tf32(PAIR ? 256 : 128, BN, KIND == KIND_GEMM ? 1 : 0);
            if ((KIND == KIND_STEM || RESW) && blockIdx.x < num_tiles) {  // CL == 1 here
                mbar_wait(wfull, 0);
                tc_fence_after();
            }
            int s = 0, t = 0;
            uint32_t ph = 0, tph = 0;
            int g = 0, kglob = 0;
            const int num_kb = p.num_kb;
            // pairs: only the leader CTA issues (its MMAs drive both CTAs' tensor cores)
            for (int u = cid; u < num_units && (!PAIR || rank == 0); u += ncl) {
                const int kb0 = (u - fdiv(u, p.fd_split) * SPL) * p.kb_per, kb1 = min(num_kb, kb0 + p.kb_per);
                int in_seg = 0;
                uint32_t d_tmem = tmem_base;
                for (int kb = kb0; kb < kb1; ++kb, ++kglob) {
                    if (in_seg == 0) {  // new segment: wait for its TMEM buffer to be drained
                        if (PAIR) mbar_wait_cluster(&tmem_empty[acc_buf(g)], acc_par(g) ^ 1);
                        else mbar_wait(&tmem_empty[acc_buf(g)], acc_par(g) ^ 1);
                        tc_fence_after();
                        d_tmem = tmem_base + (uint32_t)(acc_buf(g) * BN);
                    }
                    if (lane == 0) trace_ev(p, TR_M_LOOP, kglob);
                    if (PAIR) mbar_wait_cluster(&tready[t], tph);
                    else if (TS) mbar_wait(&tready[t], tph);
                    else mbar_wait(&full[s], ph);
                    if (lane == 0) trace_ev(p, TR_M_WAITED, kglob);
                    tc_fence_after();
                    if (lane == 0) trace_ev(p, TR_M_READY, kglob);
                    const uint32_t st = smem0 + s * L::STAGE;
                    const uint32_t a_t = tmem_base + L::A_SLOT0 + t * L::SLOT_COLS;
                    if constexpr (TS) {
                        // k-block base descriptors (step offsets are immediates in the asm)
                        uint64_t bhi, blo;
                        if (KIND == KIND_GEMM) {
                            // MN-major tf32 operand: 128B rows of 32 n-values, 32B-atom swizzle
                            // (SWIZZLE_128B_BASE32B); 4-row k-groups at SBO = 512B, 32-col
                            // chunks at LBO = 32 rows * 128B.
                            bhi = smem_desc(st + L::B_HI, 4096, 512, LAYOUT_SW128_B32);
                            blo = smem_desc(st + L::B_LO, 4096, 512, LAYOUT_SW128_B32);
                        } else if (KIND == KIND_CONV && RESW) {
                            // resident [plane][channel group][BN rows][G]: k-block kb = NB groups
                            const uint32_t lay = G::B_ROW == 128 ? LAYOUT_SW128 : LAYOUT_SW64;
                            const uint32_t w = smem0 + L::W_OFF + (uint32_t)(kb * G::B_BYTES);
                            bhi = smem_desc(w, 16, 8 * G::B_ROW, lay);
                            blo = smem_desc(w + RESW, 16, 8 * G::B_ROW, lay);
                        } else if (KIND == KIND_CONV) {
                            const uint32_t lay = G::B_ROW == 128 ? LAYOUT_SW128 : LAYOUT_SW64;
                            bhi = smem_desc(st + L::B_HI, 16, 8 * G::B_ROW, lay);
                            blo = smem_desc(st + L::B_LO, 16, 8 * G::B_ROW, lay);
                        } else {
                            // resident no-swizzle K-major weights [kb][chunk][plane][BN][4]: 8-row x
                            // 16B core matrices; 4-value chunks are PL*BN*16 B apart, the lo plane
                            // of a chunk sits BN*16 B after its hi plane (so [hi | lo] is one
                            // 2*BN-row operand for the fused MMA)
                            const uint32_t w = smem0 + L::W_OFF + (uint32_t)(kb * (G::KS / 4) * PL * BN * 16);
                            bhi = smem_desc(w, PL * BN * 16, 128, 0);
                            blo = smem_desc(w + BN * 16, PL * BN * 16, 128, 0);
                        }
                        if (PDL_DBG(p, DBG_NO_MMA)) {
                        } else if constexpr (PAIR) {
                            mma_ts_block2<G::NK, SPLIT3, G::KS, G::boff(0), G::boff(1), G::boff(2),
                                          G::boff(3), G::boff(4), G::boff(5), G::boff(6), G::boff(7)>(
                                d_tmem, a_t, bhi, blo, idesc, in_seg != 0);
                        } else if constexpr (FUSED) {  // packed stem, fused B: 8 + 2 k-steps
                            constexpr uint32_t i2n = idesc_tf32(128, 2 * BN, 0);
                            constexpr uint32_t SB = 2 * PL * BN;  // 16-byte units per K=8 step
                            mma_ts_block_fused<8, G::KS, 0, SB, 2 * SB, 3 * SB, 4 * SB, 5 * SB, 6 * SB, 7 * SB>(
                                d_tmem, a_t, bhi, i2n, idesc, in_seg != 0);
                            mma_ts_block_fused<2, G::KS, 0, SB>(d_tmem, a_t + 64, bhi + 8 * SB, i2n, idesc, 1u);
                        } else if constexpr (KIND == KIND_STEM) {
                            constexpr uint32_t SB = 2 * PL * BN;  // 16-byte units per K=8 step
                            if constexpr (G::NK == 10) {  // packed stem: 8 + 2 k-steps
                                mma_ts_block<8, SPLIT3, G::KS, 0, SB, 2 * SB, 3 * SB, 4 * SB, 5 * SB, 6 * SB, 7 * SB>(
                                    d_tmem, a_t, bhi, blo, idesc, in_seg != 0);
                                mma_ts_block<2, SPLIT3, G::KS, 0, SB, 0, 0>(d_tmem, a_t + 64, bhi + 8 * SB,
                                                                            blo + 8 * SB, idesc, 1u);
                            } else {
                                mma_ts_block<G::NK, SPLIT3, G::KS, 0, SB, 2 * SB, 3 * SB, 4 * SB, 5 * SB, 6 * SB,
                                             7 * SB>(d_tmem, a_t, bhi, blo, idesc, in_seg != 0);
                            }
                        } else {
                            mma_ts_block<G::NK, SPLIT3, G::KS, G::boff(0), G::boff(1), G::boff(2),
                                         G::boff(3), G::boff(4), G::boff(5), G::boff(6), G::boff(7)>(
                                d_tmem, a_t, bhi, blo, idesc, in_seg != 0);
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < G::NSUB; ++c) {
#pragma unroll
                            for (int kk = 0; kk < G::KK; ++kk) {
                                uint64_t bhi;
                                if (KIND == KIND_GEMM) {
                                    bhi = smem_desc(st + L::B_HI + kk * 1024, 4096, 512, LAYOUT_SW128_B32);
                                } else {
                                    const uint32_t kbyte = (c * G::KK + kk) * 32;  // K=8 step -> 32 B
                                    const uint32_t b_off = (kbyte / G::B_ROW) * G::B_SUB + kbyte % G::B_ROW;
                                    const uint32_t lay = G::B_ROW == 128 ? LAYOUT_SW128 : LAYOUT_SW64;
                                    bhi = smem_desc(st + L::B_HI + b_off, 16, 8 * G::B_ROW, lay);
                                }
                                const uint32_t acc = (in_seg | c | kk) != 0;
                                const uint32_t layout = KIND == KIND_GEMM ? LAYOUT_SW128 : LAYOUT_SW64;
                                const uint32_t a_sbo = KIND == KIND_GEMM ? 1024 : 512;
                                const uint32_t a_off = c * G::A_SUB + kk * 32;
                                const uint64_t ahi = smem_desc(st + L::A_OFF + a_off, 16, a_sbo, layout);
                                mma1_ss_elect(d_tmem, ahi, bhi, idesc, acc);
                            }
                        }
                    }
                    // release the stage (B, and SS-mode A; in every CTA of the cluster)
                    // and the TMEM A slot
                    if constexpr (PAIR) {
                        mma_commit_pair_elect(&empty[s]);
                        mma_commit_pair_elect(&tfree[t]);
                    } else if (RESW) {
                        mma_commit_elect(&tfree[t]);  // the stage held only A (read by staging)
                    } else if (KIND != KIND_STEM && TS && CL == 1) {
                        mma_commit2_elect(&empty[s], &tfree[t]);
                    } else {
                        if (KIND != KIND_STEM) {
                            if (CL == 1) mma_commit_elect(&empty[s]);
                            else mma_commit_mc_elect(&empty[s], cl_mask);
                        }
                        if (TS) mma_commit_elect(&tfree[t]);
                    }
                    if (lane == 0) trace_ev(p, TR_M_ISSUED, kglob);
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                    if (++t == TSLOTS) { t = 0; tph ^= 1; }
                    if (++in_seg == seg_kb || kb + 1 == kb1) {
                        if constexpr (PAIR) mma_commit_pair_elect(&tmem_full[acc_buf(g)]);
                        else mma_commit_elect(&tmem_full[acc_buf(g)]);
                        in_seg = 0;
                        ++g;
                    }
                }
            }
        }
    }
    } else if (warp < kEpiWarp0) {
        // ===================== A staging into TMEM (hi / lo) =====================
        if constexpr (REGTRADE) asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
        if constexpr (KIND == KIND_STEM) {
            // thread = output pixel (ph, pw) of the BW x BH tile; k-block = kernel row r:
            // gather taps 0..7 (4 channels each) of input row ph*stride + r from the
            // tile's halo stage, split hi/lo, store to the TMEM A slot
            const int tid = threadIdx.x - kSplitWarp0 * 32;
            const int quarter = warp - kSplitWarp0;
            const int row = quarter * 32 + lane;
            const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
            const bool live = row < p.BW * p.BH;
            const int ph_ = live ? row / p.BW : 0;
            const int pw_ = live ? row - ph_ * p.BW : 0;
            uint32_t pix0 = (uint32_t)((ph_ * p.stride) * p.box_w + pw_ * p.stride) * 16;
            const uint32_t row_step = (uint32_t)p.box_w * 16;
            // packed stem: byte offset of tap column s (see stem_gather_chunk)
            uint32_t col[7];
            if (p.halo_odd) {
                pix0 = (uint32_t)((ph_ * 2) * p.box_w + pw_) * 16;
                const int c0 = -p.pad;  // column parity pattern is the same for every tile
                const int e0 = (c0 + (c0 & 1)) / 2, o0 = (c0 - (c0 & 1)) / 2;
#pragma unroll
                for (int sx = 0; sx < 7; ++sx) {
                    const int cc = c0 + sx;
                    col[sx] = (cc & 1) ? (uint32_t)p.halo_odd + (uint32_t)((cc - 1) / 2 - o0) * 16
                                       : (uint32_t)(cc / 2 - e0) * 16;
                }
            } else {
#pragma unroll
                for (int sx = 0; sx < 7; ++sx) col[sx] = (uint32_t)sx * 16;
            }
            int s = 0, t = 0;
            uint32_t ph = 0, tph = 0;
            int kglob = 0;
            const bool tr = tid == 0;
            for (int st_i = cid; st_i < num_super; st_i += ncl) {
                mbar_wait(&full[s], ph);
                const uint32_t sa = smem0 + s * L::STAGE + L::A_OFF + pix0;
                for (int kb = 0; kb < p.num_kb; ++kb, ++kglob) {
                    if (tr) trace_ev(p, TR_S_FULL, kglob);
                    if constexpr (G::STEM_PACKED) {
                        // 80 packed reduction values = 5 chunks of 16, gathered and stored
                        // chunk by chunk (registers stay at 2 x 16)
                        mbar_wait(&tfree[t], tph ^ 1);
                        if (tr) trace_ev(p, TR_S_TFREE, kglob);
                        tc_fence_after();
                        const uint32_t t_hi = tmem_base + lane_off + L::A_SLOT0 + t * L::SLOT_COLS;
#pragma unroll
                        for (int c = 0; c < 5; ++c) {
                            float x[16], lo[16];
                            const bool lv = live && !PDL_DBG(p, DBG_NO_GATHER);
                            if (kb == 0) stem_gather_kb<0>(c, sa, row_step, col, lv, x);
                            else stem_gather_kb<1>(c, sa, row_step, col, lv, x);
#pragma unroll
                            for (int i = 0; i < 16; ++i) lo[i] = tf32_lo(x[i]);
                            if (!PDL_DBG(p, DBG_NO_STAGE_ST)) {
                                tmem_st16(t_hi + c * 16, x);
                                if (SPLIT3) tmem_st16(t_hi + G::KS + c * 16, lo);
                            }
                        }
                        if (kb + 1 == p.num_kb) {  // halo tile consumed
                            fence_proxy_async_smem();
                            mbar_arrive(&empty[s]);
                        }
                        tmem_wait_st();
                        tc_fence_before();
                        mbar_arrive(&tready[t]);
                        if (tr) trace_ev(p, TR_S_DONE, kglob);
                        if (++t == TSLOTS) { t = 0; tph ^= 1; }
                        continue;
                    }
                    float x[32], lo[32];
#pragma unroll
                    for (int tp = 0; tp < 8; ++tp) {
                        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (live && tp < p.S) v = lds128(sa + kb * row_step + tp * 16);
                        x[4 * tp] = v.x; x[4 * tp + 1] = v.y; x[4 * tp + 2] = v.z; x[4 * tp + 3] = v.w;
                    }
                    if (kb + 1 == p.num_kb) {  // halo tile consumed
                        fence_proxy_async_smem();
                        mbar_arrive(&empty[s]);
                    }
#pragma unroll
                    for (int i = 0; i < 32; ++i) lo[i] = tf32_lo(x[i]);
                    mbar_wait(&tfree[t], tph ^ 1);
                    if (tr) trace_ev(p, TR_S_TFREE, kglob);
                    tc_fence_after();
                    const uint32_t t_hi = tmem_base + lane_off + L::A_SLOT0 + t * L::SLOT_COLS;
                    if (!PDL_DBG(p, DBG_NO_STAGE_ST)) {
                        tmem_st32(t_hi, x);
                        if (SPLIT3) tmem_st32(t_hi + G::KS, lo);
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive(&tready[t]);
                    if (tr) trace_ev(p, TR_S_DONE, kglob);
                    if (++t == TSLOTS) { t = 0; tph ^= 1; }
                }
                if (++s == STAGES) { s = 0; ph ^= 1; }
            }
        } else if (TS) {
            const int tid = threadIdx.x - kSplitWarp0 * 32;
            const int quarter = warp - kSplitWarp0;
            const int row = quarter * 32 + lane;
            const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
            int s = 0, t = 0;
            uint32_t ph = 0, tph = 0;
            int kglob = 0;
            const bool tr = tid == 0;
            // HALO: halo-buffer ring, and this row's halo pixel index at tap (0, 0)
            int hb = 0;
            uint32_t hph = 0;
            int hrow0 = 0;
            if constexpr (HALO) {
                const int per_img = p.BW * p.BH;
                if (row < per_img * p.BNI) {
                    const int il = row / per_img, rem = row - il * per_img;
                    const int ph_ = rem / p.BW, pw_ = rem - ph_ * p.BW;
                    hrow0 = (il * p.box_h + ph_) * p.box_w + pw_;
                }
            }
            for (int u = cid; u < num_units; u += ncl) {
                const int kb0 = (u - fdiv(u, p.fd_split) * SPL) * p.kb_per, kb1 = min(p.num_kb, kb0 + p.kb_per);
                for (int kb = kb0; kb < kb1; ++kb, ++kglob) {
                    int hrow = 0;
                    bool group_end = false;
                    // the stage's B (and A, without HALO) landed: tready below is what the MMA
                    // warp waits on, so it must imply B is in shared memory
                    mbar_wait(&full[s], ph);
                    if constexpr (HALO) {
                        const int rs_n = p.R * p.S;
                        const int rs = kb - fdiv(kb, p.fd_rs) * rs_n;
                        if (rs == 0 || kb == kb0) mbar_wait(&hfull[hb], hph);
                        const int r = fdiv(rs, p.fd_S);
                        hrow = hrow0 + r * p.box_w + (rs - r * p.S);
                        group_end = rs == rs_n - 1 || kb + 1 == kb1;
                    }
                    if (tr) trace_ev(p, TR_S_FULL, kglob);
                    const uint32_t sa = smem0 + s * L::STAGE + L::A_OFF;
                    const uint32_t t_hi = tmem_base + lane_off + L::A_SLOT0 + t * L::SLOT_COLS;
                    if (KIND == KIND_GEMM) {
                        float x[32], lo[32];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const float4 v = lds128(sa + row * 128 + ((j ^ (row & 7)) << 4));
                            x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
                        }
                        split_lo_smem(smem0 + s * L::STAGE + L::B_HI, smem0 + s * L::STAGE + L::B_LO,
                                      G::B_BYTES, tid, 128);
                        fence_proxy_async_smem();
                        mbar_arrive(&empty[s]);  // A rows read (B_lo written before MMA's commit)
#pragma unroll
                        for (int i = 0; i < 32; ++i) lo[i] = tf32_lo(x[i]);
                        mbar_wait(&tfree[t], tph ^ 1);
                        tc_fence_after();
                        tmem_st32(t_hi, x);
                        tmem_st32(t_hi + G::KS, lo);
                    } else if (KIND == KIND_CONV) {
                        float x[16 * CG];
                        if constexpr (HALO) {
                            // this tap's shifted window of the halo (SW64 by absolute address)
                            const uint32_t hbuf = smem0 + L::HALO_OFF + hb * L::HALO_BUF + hrow * 64;
#pragma unroll
                            for (int c = 0; c < CG; ++c)
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    const float4 v = lds128(hbuf + c * kHaloSub + ((j ^ ((hrow >> 1) & 3)) << 4));
                                    x[16 * c + 4 * j] = v.x; x[16 * c + 4 * j + 1] = v.y;
                                    x[16 * c + 4 * j + 2] = v.z; x[16 * c + 4 * j + 3] = v.w;
                                }
                            if (group_end) {  // every tap of this channel group has been read
                                // the next TMA (async proxy) write of this buffer must not
                                // overtake these generic-proxy reads (measured: without the
                                // fence, halo + short split-K ranges read a reloaded buffer)
                                fence_proxy_async_smem();
                                mbar_arrive(&hempty[hb]);
                                if (++hb == L::HALO_NBUF) { hb = 0; hph ^= 1; }
                            }
                        } else {
#pragma unroll
                            for (int c = 0; c < CG; ++c)
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    const float4 v =
                                        lds128(sa + c * G::A_SUB + row * 64 + ((j ^ ((row >> 1) & 3)) << 4));
                                    x[16 * c + 4 * j] = v.x; x[16 * c + 4 * j + 1] = v.y;
                                    x[16 * c + 4 * j + 2] = v.z; x[16 * c + 4 * j + 3] = v.w;
                                }
                            fence_proxy_async_smem();  // generic reads before the stage's next TMA write
                            mbar_arrive(&empty[s]);  // A rows read
                        }
                        mbar_wait(&tfree[t], tph ^ 1);
                        if (tr) trace_ev(p, TR_S_TFREE, kglob);
                        tc_fence_after();
                        if (!PDL_DBG(p, DBG_NO_STAGE_ST)) {
                            // fully unrolled: x[] must stay in registers and the warp-collective
                            // tcgen05.st must not sit in a data-dependent loop
#pragma unroll
                            for (int c = 0; c < CG; ++c) {
                                float hi[16], lo[16];
#pragma unroll
                                for (int i = 0; i < 16; ++i) {
                                    hi[i] = x[16 * c + i];
                                    lo[i] = tf32_lo(hi[i]);
                                }
                                tmem_st16(t_hi + c * 16, hi);
                                if (SPLIT3) tmem_st16(t_hi + G::KS + c * 16, lo);
                            }
                        }
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    if (PAIR) mbar_arrive_on(&tready[t], 0);  // the leader issues for both CTAs
                    else mbar_arrive(&tready[t]);
                    if (tr) trace_ev(p, TR_S_DONE, kglob);
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                    if (++t == TSLOTS) { t = 0; tph ^= 1; }
                }
            }
        }
    } else {
        // ===================== TMEM drain + epilogue =====================
        if constexpr (REGTRADE) asm volatile("setmaxnreg.inc.sync.aligned.u32 176;");
        const int e = warp - kEpiWarp0;
        const int quarter = e & 3;
        const int half = e >> 2;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const bool tr = e == 0 && lane == 0;
        int g = 0, jt = 0;
        uint32_t eblk = 0;  // output boxes issued by this half (epilogue buffer ring)
        for (int u = cid; u < num_units; u += ncl, ++jt) {
            const int st_i = fdiv(u, p.fd_split), sp = u - st_i * SPL;
            const int kb0 = sp * p.kb_per, kb1 = min(p.num_kb, kb0 + p.kb_per);
            const int nseg = fdiv(kb1 - kb0 + seg_kb - 1, p.fd_seg);
            const TileCoord tc = tile_coord<KIND, BN>(p, tile_of(st_i));
            if constexpr (KIND == KIND_CONV && BN > 128 && !SPLIT3) {
                // ---- streaming epilogue (TF32, BN=256: 128 columns per thread do not fit
                // in registers): one segment per tile (the host sets seg_kb = num_kb, no
                // split-K); each 16-column block goes TMEM -> registers -> smem box -> TMA
                // store, and the accumulator is released after its last block is read
                mbar_wait(&tmem_full[acc_buf(g)], acc_par(g));
                tc_fence_after();
                const uint32_t base = tmem_base + lane_off + (uint32_t)(acc_buf(g) * BN + half * HALF);
                const uint32_t ebase = smem0 + L::EPI_OFF + half * L::EPI_BUFS * 8192;
                const bool in_box = row < p.BW * p.BH * p.BNI;
                const bool leader = quarter == 0 && lane == 0;
#pragma unroll 1
                for (int j = 0; j < HALF / 16; ++j) {
                    float v[16];
                    tmem_ld16_nowait(base + j * 16, v);
                    tmem_wait_ld();
                    if (j == HALF / 16 - 1) {
                        tc_fence_before();
                        mbar_arrive(&tmem_empty[acc_buf(g)]);
                    }
                    const int col0 = tc.n0 + half * HALF + j * 16;
                    const uint32_t ebuf = ebase + (uint32_t)(eblk % L::EPI_BUFS) * 8192;
                    ++eblk;
                    if (leader) bulk_wait_read<L::EPI_BUFS - 1>();
                    named_bar_sync(2 + half, 128);
                    if (in_box) {
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            float4 r = make_float4(v[q4 * 4], v[q4 * 4 + 1], v[q4 * 4 + 2], v[q4 * 4 + 3]);
                            r = epilogue4<EPIX>(p.flags, p.bias, p.n_out, col0 + q4 * 4, r);
                            sts128(ebuf + row * 64 + ((q4 ^ ((row >> 1) & 3)) << 4), r);
                        }
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(2 + half, 128);
                    if (leader) {
                        if (col0 < p.n_out && !PDL_DBG(p, DBG_NO_EPI_STORE)) {
                            if (p.seg_mode) {
                                int grp = tc.i0, r = tc.p0, left = p.seg_tile;
                                uint32_t off = 0;
                                while (left > 0) {
                                    const int h = min(left, p.P - r);
                                    tma_store_5d(&maps.y[h - 1], ebuf + off, 0, 0, r, col0 >> 4, grp * p.seg_imgs);
                                    off += (uint32_t)(h * p.seg_bytes);
                                    left -= h;
                                    ++grp;
                                    r = 0;
                                }
                            } else {
                                tma_store_5d(&maps.y[0], ebuf, 0, tc.q0, tc.p0, col0 >> 4, tc.i0);
                            }
                        }
                        bulk_commit();
                    }
                }
                ++g;
                if (tr) trace_ev(p, TR_E_STORED, jt);
                continue;
            }
            float sum[HALF];
            for (int sg = 0; sg < nseg; ++sg, ++g) {
                mbar_wait(&tmem_full[acc_buf(g)], acc_par(g));
                tc_fence_after();
                if (tr) trace_ev(p, TR_E_FULL, g);
                const uint32_t base = tmem_base + lane_off + (uint32_t)(acc_buf(g) * BN + half * HALF);
                if constexpr (FUSED) {
                    // [AhBh + AlBh | AhBl]: add the two column halves of this segment
#pragma unroll
                    for (int j = 0; j < HALF / 16; ++j) {
                        float v0[16], v1[16];
                        tmem_ld16_nowait(base + j * 16, v0);
                        tmem_ld16_nowait(base + BN + j * 16, v1);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            sum[j * 16 + i] = sg == 0 ? v0[i] + v1[i] : sum[j * 16 + i] + (v0[i] + v1[i]);
                    }
                } else if (sg == 0) {
                    // first segment: load straight into the sums (all loads in flight, one wait)
#pragma unroll
                    for (int j = 0; j < HALF / 16; ++j) tmem_ld16_nowait(base + j * 16, &sum[j * 16]);
                    tmem_wait_ld();
                } else {
#pragma unroll
                    for (int j = 0; j < HALF / 32; ++j) {
                        float v[32];
                        tmem_ld16_nowait(base + j * 32, &v[0]);
                        tmem_ld16_nowait(base + j * 32 + 16, &v[16]);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) sum[j * 32 + i] += v[i];
                    }
                }
                tc_fence_before();
                if (PAIR) mbar_arrive_on(&tmem_empty[acc_buf(g)], 0);
                else mbar_arrive(&tmem_empty[acc_buf(g)]);
                if (tr) trace_ev(p, TR_E_DRAINED, g);
            }
            if (SPL > 1) {
                // ---- split-K: publish this unit's partial; the tile's last unit reduces.
                // (A fixed reducer per tile, sp == tile % SPL, was tried: its waits for late
                // parts cost what spreading the reductions saved -- L18 at 32 images, 4-way
                // split: 122.9 us vs 122.1 with this rule -- so the simpler rule stays.
                // Splits pay only for long ranges; plan_split asks for >= 16 k-blocks.)
                const int tile = tile_of(st_i);
                // partial layout [16-column block][float4 of the block][128 rows][4]: a warp's 32
                // rows of one float4 are 512 contiguous bytes, for the write and the read back
                auto poff = [&](int j, int q4) { return (((half * (HALF / 16) + j) * 4 + q4) * 128 + row) * 4; };
                float *mine = p.part + ((size_t)tile * SPL + sp) * (128 * BN);
#pragma unroll
                for (int j = 0; j < HALF / 16; ++j)
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4)
                        *reinterpret_cast<float4 *>(mine + poff(j, q4)) =
                            make_float4(sum[j * 16 + q4 * 4], sum[j * 16 + q4 * 4 + 1], sum[j * 16 + q4 * 4 + 2],
                                        sum[j * 16 + q4 * 4 + 3]);
                __threadfence();
                named_bar_sync(4, kEpiThreads);
                if (e == 0 && lane == 0) {
                    const int prev = atomicAdd(p.ctr + tile, 1);
                    const uint32_t last = prev == SPL - 1;
                    if (last) p.ctr[tile] = 0;  // ready for the next launch
                    *split_flag = last;
                }
                named_bar_sync(4, kEpiThreads);
                if (tr) trace_ev(p, TR_SPLIT, 2 * jt);
                if (!*split_flag) continue;
                __threadfence();
                const float *tp = p.part + (size_t)tile * SPL * (128 * BN);
                if (SPL == 2) {
                    // two ranges: p0 + p1 is the same sum whichever unit arrives last, so the
                    // reducer keeps its own range in registers and reads only the other one
                    // (fp32 addition commutes exactly, so the result is bitwise the general path's)
                    const float *src = tp + (size_t)(sp ^ 1) * (128 * BN);
#pragma unroll
                    for (int j0 = 0; j0 < HALF / 16; j0 += 2) {
                        float4 w4[2][4];
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                            for (int q4 = 0; q4 < 4; ++q4)
                                w4[jj][q4] = (j0 + jj < HALF / 16)
                                                 ? __ldcg(reinterpret_cast<const float4 *>(src + poff(j0 + jj, q4)))
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            if (j0 + jj >= HALF / 16) break;
#pragma unroll
                            for (int q4 = 0; q4 < 4; ++q4) {
                                float *d = &sum[(j0 + jj) * 16 + q4 * 4];
                                d[0] += w4[jj][q4].x; d[1] += w4[jj][q4].y;
                                d[2] += w4[jj][q4].z; d[3] += w4[jj][q4].w;
                            }
                        }
                    }
                } else {
                    // fixed split order (independent of arrival order): ((p0 + p1) + p2) + ...;
                    // this unit's own partial is read back too.  Loads are batched (all of p0, then
                    // 8 float4 of each later partial at a time): one dependent L2 round trip per
                    // batch, not per 16 columns and partial (L18 at 32 images: 4-way split
                    // 131.8 -> 122.1 us, 8-way 530 -> 432 us)
#pragma unroll
                    for (int j = 0; j < HALF / 16; ++j)
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            const float4 v4 = __ldcg(reinterpret_cast<const float4 *>(tp + poff(j, q4)));
                            sum[j * 16 + q4 * 4] = v4.x; sum[j * 16 + q4 * 4 + 1] = v4.y;
                            sum[j * 16 + q4 * 4 + 2] = v4.z; sum[j * 16 + q4 * 4 + 3] = v4.w;
                        }
#pragma unroll 1
                    for (int q = 1; q < SPL; ++q) {
                        const float *src = tp + (size_t)q * (128 * BN);
#pragma unroll
                        for (int j0 = 0; j0 < HALF / 16; j0 += 2) {
                            float4 w4[2][4];
#pragma unroll
                            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                                for (int q4 = 0; q4 < 4; ++q4)
                                    w4[jj][q4] = (j0 + jj < HALF / 16)
                                                     ? __ldcg(reinterpret_cast<const float4 *>(src + poff(j0 + jj, q4)))
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                            for (int jj = 0; jj < 2; ++jj) {
                                if (j0 + jj >= HALF / 16) break;
#pragma unroll
                                for (int q4 = 0; q4 < 4; ++q4) {
                                    float *d = &sum[(j0 + jj) * 16 + q4 * 4];
                                    d[0] += w4[jj][q4].x; d[1] += w4[jj][q4].y;
                                    d[2] += w4[jj][q4].z; d[3] += w4[jj][q4].w;
                                }
                            }
                        }
                    }
                }
            }
            if (SPL > 1 && tr) trace_ev(p, TR_SPLIT, 2 * jt + 1);
            if constexpr (KIND != KIND_GEMM) {
                // ---- store via TMA (bias + ReLU fused): per 16-channel block, the half's
                // 128 threads write their pixel's 64 bytes into a SW64 smem image of the
                // output box, one thread stores the box; TMA clips pixels outside P x Q
                const uint32_t ebase = smem0 + L::EPI_OFF + half * L::EPI_BUFS * 8192;
                const bool in_box = row < p.BW * p.BH * p.BNI;
                const bool leader = quarter == 0 && lane == 0;
                // one 16-channel output box of this tile from smem buffer `ebuf`
                auto store_box = [&](uint32_t ebuf, int col0) {
                    if (col0 >= p.n_out || PDL_DBG(p, DBG_NO_EPI_STORE)) {
                    } else if (p.seg_mode) {
                        int grp = tc.i0, r = tc.p0, left = p.seg_tile;
                        uint32_t off = 0;
                        while (left > 0) {
                            const int h = min(left, p.P - r);
                            tma_store_5d(&maps.y[h - 1], ebuf + off, 0, 0, r, col0 >> 4, grp * p.seg_imgs);
                            off += (uint32_t)(h * p.seg_bytes);
                            left -= h;
                            ++grp;
                            r = 0;
                        }
                    } else {
                        tma_store_5d(&maps.y[0], ebuf, 0, tc.q0, tc.p0, col0 >> 4, tc.i0);
                    }
                };
                auto write_box = [&](uint32_t ebuf, int j, int col0) {
                    if (!in_box) return;
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        float4 r = make_float4(sum[j * 16 + q4 * 4], sum[j * 16 + q4 * 4 + 1],
                                               sum[j * 16 + q4 * 4 + 2], sum[j * 16 + q4 * 4 + 3]);
                        r = epilogue4<EPIX>(p.flags, p.bias, p.n_out, col0 + q4 * 4, r);
                        sts128(ebuf + row * 64 + ((q4 ^ ((row >> 1) & 3)) << 4), r);
                    }
                };
                if constexpr (L::EPI_BUFS >= HALF / 16 && (RESW || KIND == KIND_STEM)) {
                    // output-heavy tiles with a buffer per box: write every box of the tile,
                    // then store them all (2 barriers per tile instead of 2 per box; stem
                    // -6%, layers 2/4 -5/-11%; compute-bound BN=64 layer 3 keeps the ring)
                    if (leader) bulk_wait_read<0>();  // the previous tile's boxes left smem
                    named_bar_sync(2 + half, 128);
#pragma unroll
                    for (int j = 0; j < HALF / 16; ++j)
                        write_box(ebase + (uint32_t)j * 8192, j, tc.n0 + half * HALF + j * 16);
                    fence_proxy_async_smem();
                    named_bar_sync(2 + half, 128);
                    if (leader) {
#pragma unroll
                        for (int j = 0; j < HALF / 16; ++j)
                            store_box(ebase + (uint32_t)j * 8192, tc.n0 + half * HALF + j * 16);
                        bulk_commit();
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < HALF / 16; ++j) {
                        const int col0 = tc.n0 + half * HALF + j * 16;
                        const uint32_t ebuf = ebase + (uint32_t)(eblk % L::EPI_BUFS) * 8192;
                        ++eblk;
                        if (leader) bulk_wait_read<L::EPI_BUFS - 1>();  // this buffer's last box left
                        named_bar_sync(2 + half, 128);
                        write_box(ebuf, j, col0);
                        fence_proxy_async_smem();
                        named_bar_sync(2 + half, 128);
                        if (leader) {
                            store_box(ebuf, col0);
                            bulk_commit();  // one group per block (possibly empty): uniform ring
                        }
                    }
                }
                if (tr) trace_ev(p, TR_E_STORED, jt);
                continue;
            }
            // ---- store (bias + ReLU fused) ----
            bool valid;
            float *obase;
            size_t cstride = 0;
            if (KIND == KIND_GEMM) {
                const int gm = tc.m0 + row;
                valid = gm < p.M;
                obase = p.out + (size_t)(valid ? gm : 0) * p.ldc;
            } else {
                const int per_img = p.BW * p.BH;
                const int il = row / per_img;
                const int rem = row - il * per_img;
                const int hl = rem / p.BW;
                const int wl = rem - hl * p.BW;
                const int img = tc.i0 + il, pp = tc.p0 + hl, qq = tc.q0 + wl;
                valid = il < p.BNI && img < p.nimg && pp < p.P && qq < p.Q;
                const size_t plane = (size_t)p.P * p.Q * 16;
                obase = p.out + ((size_t)(valid ? img : 0) * p.KT) * plane +
                        ((size_t)(valid ? pp : 0) * p.Q + (valid ? qq : 0)) * 16;
                cstride = plane;  // next 16-channel block kt
            }
            if (valid && !PDL_DBG(p, DBG_NO_EPI_STORE)) {
#pragma unroll
                for (int j = 0; j < HALF / 16; ++j) {
                    const int col0 = tc.n0 + half * HALF + j * 16;
                    if (col0 < p.n_out) {
                        float *dst = KIND == KIND_GEMM ? obase + col0
                                                       : obase + (size_t)(col0 >> 4) * cstride;
                        store16<KIND, EPIX>(p, dst, col0, &sum[j * 16]);
                    }
                }
            }
            if (tr) trace_ev(p, TR_E_STORED, jt);
        }
    }
    if (KIND != KIND_GEMM && warp >= kEpiWarp0 && ((warp - kEpiWarp0) & 3) == 0 && lane == 0)
        bulk_wait<0>();  // output boxes written before the CTA retires
    __syncwarp();
    if (threadIdx.x == kEpiWarp0 * 32) trace_ev(p, TR_KERNEL, 3);
    tc_fence_before();
    if (CL > 1) cluster_sync();  // no CTA leaves while peers may still multicast into it
    else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if constexpr (PAIR) tmem_dealloc2<L::TMEM_COLS>(tmem_base);
        else tmem_dealloc<L::TMEM_COLS>(tmem_base);
        if (lane == 0) trace_ev(p, TR_KERNEL, 4);
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
            C[(size_t)gm * ldc + gn] = epilogue1(flags, bias, N, gn, r);
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
                                                        unsigned flags, int C_real) {
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
                    if (ct * 16 + c >= C_real) break;
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
        yo[k] = epilogue1(flags, bias, KT * 16, kt * 16 + k, r);
    }
}

// Unfused element-wise pass over nKhw16k (float4 vectorised): the same epilogue as the
// fused kernels (scale, bias, ReLU / ReLU6).
__global__ void bias_relu_kernel(float4 *__restrict__ y, const float *__restrict__ bias,
                                 long long n4, int pq, int KT, unsigned flags) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
        const int kt = (int)((i / (4LL * pq)) % KT);
        y[i] = epilogue4<true>(flags, bias, KT * 16, kt * 16 + (int)(i & 3) * 4, y[i]);
    }
}

// `+=` of a conv result onto non-zero incoming output contents, then the epilogue:
// y = act((y + y0) * scale + bias) over nKhw16k (the executor's accumulating nests).
__global__ void accumulate_epilogue_kernel(float4 *__restrict__ y, const float4 *__restrict__ y0,
                                           const float *__restrict__ bias, long long n4, int pq, int KT,
                                           unsigned flags) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
        const int kt = (int)((i / (4LL * pq)) % KT);
        float4 v = y[i];
        const float4 a = y0[i];
        v.x = __fadd_rn(v.x, a.x); v.y = __fadd_rn(v.y, a.y);
        v.z = __fadd_rn(v.z, a.z); v.w = __fadd_rn(v.w, a.w);
        y[i] = epilogue4<true>(flags, bias, KT * 16, kt * 16 + (int)(i & 3) * 4, v);
    }
}

// Weight prepack KCRS16c16k -> packed[plane][C/G][r*S+s][k][G] (K-major rows of G
// input channels per output channel k; G = 32 when the channel-block count is
// even, else 16); plane 0 = w (the tensor core truncates to tf32), plane 1 =
// lo = w - tf32(w) for 3xTF32.  Input channels >= C_real are zeroed (nChw16c
// pads C to a multiple of 16).
__global__ void prepack_weights_kernel(const float *__restrict__ w, float *__restrict__ out,
                                       int CT, int KT, int RS, int split, int C_real, int G) {
    const long long total = (long long)KT * CT * RS * 256;
    const int K = KT * 16;
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
        const int cin = ct * 16 + c;
        const float v = (cin < C_real) ? w[i] : 0.f;
        const size_t dst = ((((size_t)(cin / G) * RS + rs) * K) + (size_t)kt * 16 + k) * G + cin % G;
        out[dst] = v;
        if (split) out[dst + total] = v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    }
}

// Stem prepack: KCRS16c16k (CT = 1, C_real <= 4) -> packed[kchunk][plane][k][4]
// (no-swizzle K-major core matrices, 4 reduction values per 16-byte chunk).
// Unpacked: chunk = r*8 + tap, value = channel (taps >= S and channels >= C_real
// zero).  Packed (C=3, 7x7): reduction index q = 4kc + j sits in tap-aligned
// 16-value group q/16 = taps 5*(q/16) .. +4, three channels each, value 15 zero.
__global__ void prepack_stem_weights_kernel(const float *__restrict__ w, float *__restrict__ out,
                                            int K, int R, int S, int split, int C_real, int nchunks,
                                            int packed) {
    const long long plane = (long long)nchunks * K * 4;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < plane;
         i += (long long)gridDim.x * blockDim.x) {
        const int j = i & 3;
        long long t = i >> 2;
        const int k = t % K;
        const int kc = (int)(t / K);
        int r, tap, c;
        bool ok;
        if (packed) {
            // tap-aligned chunks of 16: value jj of chunk ch = tap 5*ch + jj/3, channel
            // jj%3 (jj = 15 and taps >= R*S are zero) -- matches stem_gather_chunk
            const int q = kc * 4 + j;
            const int ch = q >> 4, jj = q & 15;
            const int t = 5 * ch + jj / 3;
            c = jj % 3;
            ok = jj < 15 && t < R * S && c < C_real;
            r = t / S;
            tap = t - r * S;
        } else {
            r = kc / 8;
            tap = kc % 8;
            c = j;
            ok = tap < S && c < C_real;
        }
        float v = 0.f;
        if (ok) v = w[((((size_t)(k >> 4) * R + r) * S + tap) * 16 + c) * 16 + (k & 15)];
        // layout [kchunk][plane][k][4]: the lo plane of a chunk follows its hi plane
        const int planes = split ? 2 : 1;
        const size_t o = ((size_t)kc * planes * K + k) * 4 + j;
        out[o] = v;
        if (split) out[o + (size_t)K * 4] = v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    }
}

}  // namespace pdl
