/*
 * pdl.h -- C ABI of libpdl.so, the B200 (sm_100a) implementation of the hot
 * path of PolyDL (arXiv 2006.02230) as exposed by the reference `looprank`
 * package.  Plain pointers and sizes only; every tensor pointer is a
 * caller-owned DEVICE pointer, every call is stream-ordered and asynchronous,
 * no call allocates device memory.  Return 0 on success, a negative PDL_E*
 * code otherwise; pdl_last_error() gives a thread-local message.
 *
 * What each entry point replaces in the reference (/root/reference):
 *
 *   pdl_conv2d_fwd_nchw16c  -- simcache.interpret (pkg/src/looprank/simcache.py:89-204)
 *       executing the Fig. 9 blocked convolution nest
 *       whose innermost band is the `#pragma microkernel gemm(...)` region
 *       (loopdsl.py:250, 502-514; substitute_microkernel loopdsl.py:747-760).
 *       Layouts are the nest's array declarations: input nChw16c, filter
 *       KCRS16c16k, output nKhw16k.  Unlike the .pdl nest (which cannot express
 *       padding), x is UNPADDED and the kernel zero-fills the
 *       halo; pad = R/2 in every BASELINE config.
 *   pdl_conv2d_fwd_prepacked / pdl_conv2d_prepack_weights -- the same call
 *       split in two: a one-time weight reorder (+ hi/lo TF32 split for 3xTF32)
 *       and the per-batch convolution.  This mirrors how the paper's CPU
 *       implementation keeps KCRS16c16k weights in a blocked format prepared
 *       once per layer.
 *   PDL_BIAS | PDL_RELU flags -- the conv -> bias+ReLU program (two nests in
 *       one .pdl Program) fused per Alg. 3 (
 *       SPEC.md:531-591): the element-wise op is applied to the fully reduced
 *       accumulator before the single store.
 *   pdl_gemm_f32            -- interpret on the Fig. 1 / Fig. 12 GEMM nest
 *       C[i][j] += A[i][k]*B[k][j] in its
 *       beta*C + alpha*A*B form, row-major.
 *   pdl_bias_relu_nchw16c   -- the stand-alone element-wise nest
 *       `output = max(output + bias, 0.0)` (the unfused GPU baseline).
 *
 * Numerics: PDL_MODE_3XTF32 (default) splits every fp32 operand x into
 * hi = tf32(x) and lo = x - hi and accumulates hi*hi + hi*lo + lo*hi in fp32
 * on the tcgen05 tensor cores (max-rel <= 1e-5 vs the float64 oracle);
 * PDL_MODE_TF32 is one tensor pass (<= 1e-2); PDL_MODE_FP32 runs exact fp32
 * FMAs on the CUDA cores (also the path for shapes TMA cannot describe).
 */
#ifndef PDL_H_
#define PDL_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDL_ABI_VERSION 1

/* Schedule knobs chosen by the ranker (paper_2006_02230_b200/rank.py);
 * NULL or zero fields = library default.  bm is fixed at 128 (tcgen05 M). */
typedef struct pdl_tile_cfg {
    int bm;        /* output rows (pixels / GEMM M) per CTA tile: 128          */
    int bn;        /* output columns (K channels / GEMM N) per tile: 64|128, conv also 256
                      (TF32 default for K % 256 == 0; 3xTF32 with bk = 32, opt-in)           */
    int bk;        /* reduction elements per pipeline stage (16*cg for conv)    */
    int stages;    /* smem pipeline depth                                       */
    int cluster_m; /* CTAs per cluster sharing (TMA-multicasting) a weight tile: 1|2|4 */
    int cluster_n; /* 2: CTA-pair tiles, cta_group::2 MMAs with M = 256 (3xTF32 conv) */
    int split_k;   /* 0: auto (split the reduction when the tiles leave SMs idle
                      and a workspace is given), 1: off, >1: that many ranges   */
    int raster;    /* bit 0 (PDL_RASTER_M_FASTEST): tile order with output-pixel tiles
                      fastest (consecutive CTAs share weights; default: output-channel
                      tiles fastest, they share activations; ignored with clusters,
                      CTA pairs, the stem and resident weights); bit 1 (PDL_RASTER_BOX_TILES):
                      box tiles only -- no multi-image segment tiles for small maps;
                      bit 2 (PDL_RASTER_SEG_TILES): segment tiles whenever the shape
                      allows, even if they do not remove a wave of tiles; bits 3, 4,
                      6 and the tile box in bits 8-30 below; any other bit: PDL_EUNSUPPORTED              */
} pdl_tile_cfg;

#define PDL_RASTER_M_FASTEST 1
#define PDL_RASTER_BOX_TILES 2
#define PDL_RASTER_SEG_TILES 4
#define PDL_RASTER_SINGLE_IMAGE_TILES 8 /* box tiles hold several images only when a whole image
                                          fits (the round-1 geometry); default: the box search
                                          over (pixels wide, pixels high, images) that fills the
                                          128 tensor-core rows best */
#define PDL_RASTER_NO_HALO 16  /* 3x3 convs: one A box per tap instead of one halo per channel group */
#define PDL_RASTER_HALO_CG4 64 /* 3xTF32 halo mode with 64-channel k-blocks (one halo buffer) */
/* explicit conv tile box: w x h output pixels of n consecutive images, w*h*n <= 128 */
#define PDL_RASTER_TILE(w, h, n) (((w) & 0xff) << 8 | ((h) & 0xff) << 16 | ((n) & 0x7f) << 24)
#define PDL_RASTER_TILE_MASK 0x7fffff00

enum {
    PDL_BIAS = 1,             /* y += bias[k]                                  */
    PDL_RELU = 2,             /* y = max(y, 0)   (after bias)                  */
    PDL_RELU6 = 1 << 2,       /* y = min(max(y, 0), 6)   (after bias; ReLU6 of
                                 PAPER.md:1233-1234)                           */
    PDL_SCALE = 1 << 3,       /* y *= scale[k] before the bias (batch-norm
                                 inference affine): `bias`
                                 then holds 2*K floats, shift[K] then scale[K];
                                 the shift is added only with PDL_BIAS         */
    PDL_MODE_3XTF32 = 0 << 4, /* default                                       */
    PDL_MODE_TF32 = 1 << 4,
    PDL_MODE_FP32 = 2 << 4,
    PDL_MODE_MASK = 3 << 4,
    PDL_HOST_X_READY = 1 << 6,/* pdl_conv2d_fwd_host: x_host, packed_w and bias are
                                 final at call time (not written by work still pending
                                 on the stream) and y_host is not read by such work, so
                                 this call's copies in and convolutions may overlap an
                                 earlier call's copies out                      */
    PDL_NO_SIMT = 1 << 7,     /* GEMM: fail with PDL_EUNSUPPORTED instead of running
                                 the CUDA-core kernel when the operands cannot take the
                                 tensor-core path (unaligned pointers, K = 0, or N /
                                 lda / ldb / ldc not multiples of 4)            */
    PDL_X_NCHW4C = 1 << 13    /* conv, narrow-channel path only (C <= 4, the ResNet
                                 stem): x is [N][H][W][4] fp32 (nChw4c with one channel
                                 block; channels >= C must be finite, their weights are
                                 zero) instead of nChw16c.  nChw16c stores the stem's 3
                                 channels in 64-byte pixels and HBM / PCIe move all 64;
                                 this layout moves the 16 the kernel reads.  Same
                                 arithmetic in the same order: results are bitwise equal
                                 to the nChw16c call.  Weights, bias and y are unchanged.
                                 pdl_pack_nchw4c() produces it from NCHW.        */
};
/* Every entry point rejects flag bits it does not implement (PDL_EUNSUPPORTED). */

enum {
    PDL_OK = 0,
    PDL_EINVAL = -1,     /* bad shape / argument                                */
    PDL_EALIGN = -2,     /* pointer or stride not 16-byte aligned               */
    PDL_EDEVICE = -3,    /* no sm_100 device                                    */
    PDL_ELAUNCH = -4,    /* CUDA launch / driver failure                        */
    PDL_EWORKSPACE = -5, /* workspace missing or too small                      */
    PDL_EUNSUPPORTED = -6
};

enum { PDL_OP_CONV2D = 1, PDL_OP_GEMM = 2 };

/* Convolution, raw KCRS16c16k weights.  Needs a workspace of
 * pdl_workspace_bytes(PDL_OP_CONV2D, dims, cfg) bytes (the prepacked weights,
 * then -- 256-byte aligned -- the split-K area when the schedule splits; that
 * area must be zero on first use), dims = {N, C, K, H, W, R, S, stride, pad, flags}. */
int pdl_conv2d_fwd_nchw16c(const float *x, const float *w, const float *bias, float *y,
                           int N, int C, int K, int H, int W, int R, int S, int stride,
                           int pad, unsigned flags, const pdl_tile_cfg *cfg, void *workspace,
                           size_t ws_bytes, void *stream);

/* One-time weight reorder KCRS16c16k -> tensor-core operand image (and hi/lo
 * split for 3xTF32).  `packed` must hold pdl_conv2d_packed_bytes(...) bytes. */
size_t pdl_conv2d_packed_bytes(int C, int K, int R, int S, unsigned flags);
int pdl_conv2d_prepack_weights(const float *w, void *packed, int C, int K, int R, int S,
                               unsigned flags, void *stream);
int pdl_conv2d_fwd_prepacked(const float *x, const void *packed_w, const float *bias,
                             float *y, int N, int C, int K, int H, int W, int R, int S,
                             int stride, int pad, unsigned flags, const pdl_tile_cfg *cfg,
                             void *stream);

/* Split-K (small batches: a 7x7 layer at 32 images has 64 tiles for 148 SMs):
 * the same call with a workspace, so the library may cut each tile's reduction
 * into ranges computed by different CTAs.  Partials meet in the workspace; the
 * last CTA of a tile sums them in range order (deterministic, independent of
 * arrival order) and runs the fused epilogue.  The workspace (256-byte aligned,
 * pdl_conv2d_splitk_workspace_bytes(...) bytes, 0 = this shape does not split)
 * starts with a fixed 1 KB block of tile counters that must be ZERO before its
 * first use; the counters reset themselves, so one workspace can serve later
 * calls of any shape on the same stream (not concurrent streams). */
size_t pdl_conv2d_splitk_workspace_bytes(int N, int C, int K, int H, int W, int R, int S,
                                         int stride, int pad, unsigned flags,
                                         const pdl_tile_cfg *cfg);
int pdl_conv2d_fwd_prepacked_ws(const float *x, const void *packed_w, const float *bias,
                                float *y, int N, int C, int K, int H, int W, int R, int S,
                                int stride, int pad, unsigned flags, const pdl_tile_cfg *cfg,
                                void *workspace, size_t ws_bytes, void *stream);

/* Host-buffer convolution -- the reference's interpret() contract (host arrays
 * in, fresh host arrays out: simcache.py:89-204, inputs copied at :110).
 * x_host [N][C/16][H][W][16] and y_host [N][K/16][P][Q][16] are HOST pointers
 * (pinned -- cudaHostAlloc / cudaHostRegister -- or the copies serialise);
 * packed_w / bias / workspace are device pointers.  The minibatch is cut into
 * chunks of `chunk` images (0 = library default, ~64 MB of x per chunk, at
 * least 4 chunks when the batch allows); each chunk's host->device copy,
 * convolution and device->host copy run on three internal streams (one set per
 * device and workspace) through 3 staging slots, so both PCIe directions and the
 * tensor cores overlap.  Ordered after prior work on `stream`; with
 * PDL_HOST_X_READY and a previous call on the same workspace (any thread), only
 * after that call's convolutions: the copies in and convolutions may run while
 * its copies out are still going, and the copies out are NOT ordered after other
 * work pending on `stream` (see PDL_HOST_X_READY).  Work enqueued on `stream`
 * after the call sees y_host complete; on an error return, `stream` still waits
 * for whatever the call had enqueued.  workspace must hold pdl_conv2d_host_workspace_bytes(...)
 * bytes (same chunk): an x third written by copies in (3 chunk slots) and two y
 * thirds (each the call's whole output) read by copies out, used by alternate
 * calls. */
size_t pdl_conv2d_host_workspace_bytes(int N, int C, int K, int H, int W, int R, int S,
                                       int stride, int pad, int chunk);
int pdl_conv2d_fwd_host(const float *x_host, const void *packed_w, const float *bias,
                        float *y_host, int N, int C, int K, int H, int W, int R, int S,
                        int stride, int pad, unsigned flags, const pdl_tile_cfg *cfg, int chunk,
                        void *workspace, size_t ws_bytes, void *stream);

/* C = act(alpha * A B + beta * C), row-major with leading dimensions lda/ldb/ldc;
 * act = PDL_RELU / PDL_RELU6 / none.  workspace: optional split-K area (same rules
 * as pdl_conv2d_fwd_prepacked_ws), pdl_workspace_bytes(PDL_OP_GEMM, {M, N, K, flags},
 * cfg) bytes; NULL = no split.  PDL_BIAS / PDL_SCALE need pdl_gemm_f32_epilogue
 * (EINVAL here).  Operands TMA cannot describe (see PDL_NO_SIMT) run on the CUDA
 * cores in exact fp32. */
int pdl_gemm_f32(const float *A, const float *B, float *C, int M, int N, int K, int lda,
                 int ldb, int ldc, float alpha, float beta, unsigned flags,
                 const pdl_tile_cfg *cfg, void *workspace, size_t ws_bytes, void *stream);

/* The GEMM with the full fused epilogue of Alg. 3 (the fused
 * GEMM + batch-norm / bias + ReLU programs): per output column n,
 *   C = act((alpha * A B + beta * C) * scale[n] + shift[n])
 * bias = shift[N] (PDL_BIAS), or shift[N] then scale[N] (PDL_SCALE; the shift is
 * added only with PDL_BIAS); 16-byte aligned device pointer, may be NULL without
 * those flags.  Same rules as pdl_gemm_f32 otherwise. */
int pdl_gemm_f32_epilogue(const float *A, const float *B, float *C, const float *bias, int M,
                          int N, int K, int lda, int ldb, int ldc, float alpha, float beta,
                          unsigned flags, const pdl_tile_cfg *cfg, void *workspace,
                          size_t ws_bytes, void *stream);

/* Unfused element-wise pass over y[N][K/16][P][Q][16] (the GPU baseline). */
int pdl_bias_relu_nchw16c(float *y, const float *bias, int N, int K, int P, int Q,
                          unsigned flags, void *stream);

/* `+=` onto incoming output contents (the nest's output was not zero): y = the
 * convolution result, y0 = the incoming contents; y = act((y + y0) * scale + bias)
 * with the same flags / bias layout as the fused epilogue. */
int pdl_accumulate_epilogue_nchw16c(float *y, const float *y0, const float *bias, int N, int K,
                                    int P, int Q, unsigned flags, void *stream);

/* Layout conversion on either side of the path (device to device):
 *   NCHW [N][C][H][W]      <-> nChw16c [N][ceil(C/16)][H][W][16] (pad channels zero)
 *   OIHW [K][C][R][S]       -> KCRS16c16k [K/16][ceil(C/16)][R][S][16c][16k]
 * The reference keeps tensors blocked throughout; these are
 * the pack/unpack steps a PyTorch-layout caller needs before/after it. */
int pdl_pack_nchw16c(const float *src, float *dst, int N, int C, int H, int W, void *stream);
/* NCHW (C <= 4) -> [N][H][W][4], channels >= C zero: the PDL_X_NCHW4C input layout */
int pdl_pack_nchw4c(const float *src, float *dst, int N, int C, int H, int W, void *stream);
int pdl_unpack_nchw16c(const float *src, float *dst, int N, int C, int H, int W, void *stream);
int pdl_pack_kcrs16c16k(const float *src, float *dst, int K, int C, int R, int S, void *stream);

size_t pdl_workspace_bytes(int op, const int *dims, const pdl_tile_cfg *cfg);

/* The schedule the library will run for a call (after its own rules: resident
 * weights, halo mode, segment tiles, split-K planning, 256-column TF32 tiles) --
 * what the ranker reasons about.  Pure host computation; no device work. */
typedef struct pdl_schedule {
    int kind;        /* 1: tile-engine conv, 2: narrow-channel stem conv, 3: GEMM        */
    int bn, bk;      /* output columns per tile; reduction elements per k-block          */
    int cluster;     /* CTAs per cluster (2 with a CTA pair)                              */
    int tile_w, tile_h, tile_images; /* output pixels per M tile (GEMM: 128 x 1 x 1)     */
    int seg_rows;    /* > 0: segment tiles of that many output rows (bands)               */
    int m_tiles, n_tiles;
    int num_kb;      /* k-blocks per tile                                                 */
    int split, kb_per; /* split-K ranges per tile, k-blocks per range                     */
    int halo;        /* input halo loaded once per channel group (stem: whole-tile halo)  */
    int resident;    /* weights of the N-tile resident in shared memory                   */
    int pair;        /* CTA pair (cta_group::2, M = 256)                                  */
    int order;       /* 1: output-pixel tiles fastest                                     */
    int flat;        /* 1x1 / stride 1 / pad 0 map flattened to one row                   */
    size_t splitk_workspace_bytes;
} pdl_schedule;
/* with_workspace != 0: the call will pass a split-K workspace (auto split may engage). */
int pdl_conv2d_schedule(int N, int C, int K, int H, int W, int R, int S, int stride, int pad,
                        unsigned flags, const pdl_tile_cfg *cfg, int with_workspace,
                        pdl_schedule *out);
int pdl_gemm_schedule(int M, int N, int K, unsigned flags, const pdl_tile_cfg *cfg,
                      int with_workspace, pdl_schedule *out);

/* Tile config the library would pick for a conv / GEMM (for the ranker and
 * the bench's roofline report).  Writes *cfg, returns 0. */
int pdl_default_cfg(int op, const int *dims, pdl_tile_cfg *cfg);

/* Number of kernel launches the last successful call on this thread issued. */
int pdl_last_launch_count(void);

const char *pdl_last_error(void);
int pdl_abi_version(void);
/* 0 if the current device is sm_100 (B200), PDL_EDEVICE otherwise. */
int pdl_device_check(void);

#ifdef __cplusplus
}
#endif
#endif /* PDL_H_ */
