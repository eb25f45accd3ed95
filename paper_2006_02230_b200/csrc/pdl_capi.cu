// pdl_capi.cu -- the extern "C" boundary of libpdl.so (include/pdl.h): argument
// validation, tile-config selection, TMA tensor-map encoding and kernel launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/pdl.h"
#include "pdl_layout.cuh"
#include "pdl_kernels.cuh"

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PDL_ELAUNCH, "%s: %s", what, cudaGetErrorString(e));
    return PDL_OK;
}

// ---------------------------------------------------------------- driver entry
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

int get_encode() {
    std::call_once(g_encode_once, [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<EncodeTiledFn>(fn);
    });
    if (!g_encode) return fail(PDL_EDEVICE, "cuTensorMapEncodeTiled unavailable");
    return PDL_OK;
}

int encode(CUtensorMap *m, const void *base, int rank, const cuuint64_t *dims,
           const cuuint64_t *strides_bytes, const cuuint32_t *box, CUtensorMapSwizzle sw,
           const char *what,
           CUtensorMapL2promotion l2 = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void *>(base),
                          dims, strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, l2,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PDL_EINVAL, "tensor map encode failed (%s, rc=%d)", what, (int)r);
    return PDL_OK;
}

// ---------------------------------------------------------------- device check
// Per-device state (a process may drive several GPUs, e.g. one host thread per
// device): the sm_100 check and the SM count, each initialised once per device.
constexpr int kMaxDevices = 16;
struct DevInfo {
    std::once_flag once;
    int ok = 0;
    int sms = 148;
};
DevInfo g_dev[kMaxDevices];

int cur_dev() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return -1;
    return dev;
}

DevInfo *dev_info() {
    const int dev = cur_dev();
    if (dev < 0) return nullptr;
    DevInfo &d = g_dev[dev];
    std::call_once(d.once, [&] {
        int major = 0, minor = 0, sms = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
            d.sms = sms;
        d.ok = (major == 10 && minor == 0) ? 1 : 0;
        cudaGetLastError();
    });
    return &d;
}

// SM count of the current device (148 on B200; the planners size grids by it)
int sms() {
    const DevInfo *d = dev_info();
    return d ? d->sms : 148;
}

int device_check() {
    const DevInfo *d = dev_info();
    if (!d || d->ok != 1) return fail(PDL_EDEVICE, "libpdl requires an sm_100 (B200) device");
    return PDL_OK;
}

// PDL_TRACE builds: device buffer receiving block 0's event stamps (see pdl_trace_buffer).
unsigned long long *g_trace = nullptr;

// Programmatic dependent launch of the tile engine (PDL_NO_PDL=1 in the
// environment turns it off, for A/B measurements).
const bool g_pdl = [] {
    const char *e = std::getenv("PDL_NO_PDL");
    return !(e && e[0] == '1');
}();

// Reduction elements accumulated in TMEM before an fp32 round-to-nearest drain.
constexpr int kSegElems = 256;
// CTAs per cluster sharing (multicasting) each weight tile.
// conv: no weight multicast by default.  Round 1i A/B on one box (256 images, CUDA-graph
// suite): cluster 1 beats cluster 2 on layers 3/7/9/10 (-9/-4/-6/-3%) and ties elsewhere,
// suite +1.5% (profiles/cluster_ab_r1i.json)
constexpr int kDefaultConvCluster = 1;

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Flag bits each entry point accepts; anything else is rejected rather than ignored.
// The diagnostic bits (pdl::kDiagBits) exist only in -DPDL_DIAG builds.
#ifdef PDL_DIAG
constexpr unsigned kDiag = pdl::kDiagBits;
#else
constexpr unsigned kDiag = 0;
#endif
constexpr unsigned kEpiFlags = PDL_BIAS | PDL_RELU | PDL_RELU6 | PDL_SCALE;
constexpr unsigned kConvFlags = kEpiFlags | PDL_MODE_MASK;
// entry points that read x: the compact narrow-channel layout is theirs alone
constexpr unsigned kConvXFlags = kConvFlags | PDL_X_NCHW4C;
constexpr unsigned kGemmFlags = kEpiFlags | PDL_MODE_MASK | PDL_NO_SIMT;
constexpr int kRasterBits = PDL_RASTER_M_FASTEST | PDL_RASTER_BOX_TILES | PDL_RASTER_SEG_TILES | PDL_RASTER_NO_HALO |
                            PDL_RASTER_HALO_CG4 | PDL_RASTER_SINGLE_IMAGE_TILES | PDL_RASTER_TILE_MASK;

int check_flags(unsigned flags, unsigned allowed, const char *what) {
    const unsigned bad = flags & ~(allowed | kDiag);
    if (bad) return fail(PDL_EUNSUPPORTED, "%s: unsupported flag bits 0x%x", what, bad);
    if ((flags & PDL_MODE_MASK) == PDL_MODE_MASK) return fail(PDL_EINVAL, "%s: invalid mode bits", what);
    return PDL_OK;
}

// ---------------------------------------------------------------- launch helpers
// Persistent launch: grid = as many CTAs (clusters of CL) as can be co-resident,
// capped by the work.  Clusters of 4 cannot use every SM (GPC granularity), so
// the co-resident count comes from cudaOccupancyMaxActiveClusters.
template <int KIND, int BN, int CG, bool SPLIT3, int CL, bool PAIR = false, int RESW = 0, bool HALO = false,
          bool EPIX = false>
int launch_tile(const pdl::TmaMaps &maps, const pdl::TileParams &p, int work_ctas, cudaStream_t s) {
    using L = pdl::Smem<KIND, BN, CG, SPLIT3, PAIR, RESW, HALO>;
    auto kern = pdl::tile_mma_kernel<KIND, BN, CG, SPLIT3, CL, PAIR, RESW, HALO, EPIX>;
    // the dynamic-smem attribute and the co-resident CTA count are per device
    static std::once_flag once[kMaxDevices];
    static cudaError_t attr_err[kMaxDevices];
    static int max_ctas[kMaxDevices];
    const int dev = cur_dev();
    if (dev < 0) return fail(PDL_EDEVICE, "tile_mma_kernel: no current device");
    const int sm_count = sms();
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    // programmatic dependent launch: this grid may start (barrier init, TMEM
    // alloc, descriptor prefetch) while the previous kernel on the stream drains;
    // it reads / writes global memory only after griddepcontrol.wait
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    lc.blockDim = dim3(pdl::kThreads);
    lc.dynamicSmemBytes = L::TOTAL;
    lc.stream = s;
    lc.attrs = at;
    lc.numAttrs = 2;
    std::call_once(once[dev], [&] {
        attr_err[dev] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
        if (attr_err[dev] != cudaSuccess) return;
        int ncl = 0;
        lc.gridDim = dim3(CL * 64);
        if (cudaOccupancyMaxActiveClusters(&ncl, kern, &lc) != cudaSuccess || ncl <= 0)
            ncl = sm_count / CL;
        cudaGetLastError();
        max_ctas[dev] = std::min(ncl * CL, sm_count / CL * CL);
    });
    if (attr_err[dev] != cudaSuccess)
        return fail(PDL_ELAUNCH, "cudaFuncSetAttribute: %s", cudaGetErrorString(attr_err[dev]));
    int grid = std::min(max_ctas[dev], (work_ctas + CL - 1) / CL * CL);
    if (KIND == pdl::KIND_STEM || RESW) grid = std::max(p.n_tiles, grid / p.n_tiles * p.n_tiles);
    lc.gridDim = dim3(grid);
    pdl::TileParams pt = p;
    pt.trace = g_trace;
    if (pt.split <= 1) {
        pt.split = 1;
        pt.kb_per = pt.num_kb;
    }
    pt.fd_n_tiles = pdl::make_fastdiv(pt.n_tiles);
    pt.fd_m_tiles = pdl::make_fastdiv(pt.m_tiles);
    pt.fd_tiles_w = pdl::make_fastdiv(pt.tiles_w);
    pt.fd_tiles_h = pdl::make_fastdiv(pt.tiles_h);
    pt.fd_split = pdl::make_fastdiv(pt.split);
    pt.fd_P = pdl::make_fastdiv(pt.P);
    pt.fd_rs = pdl::make_fastdiv(pt.R * pt.S);
    pt.fd_S = pdl::make_fastdiv(pt.S);
    pt.fd_seg = pdl::make_fastdiv(pt.seg_kb);
    cudaError_t e = cudaLaunchKernelEx(&lc, kern, maps, pt);
    if (e != cudaSuccess) return fail(PDL_ELAUNCH, "tile_mma_kernel launch: %s", cudaGetErrorString(e));
    ++g_launches;
    return check_launch("tile_mma_kernel");
}

template <int KIND, bool SPLIT3, int CL>
int dispatch_bn(int bn, int cg, const pdl::TmaMaps &maps, const pdl::TileParams &p, int work,
                cudaStream_t s) {
    if constexpr (KIND == pdl::KIND_STEM) {
        if (bn == 64 && CL == 1 && cg == 1) return launch_tile<KIND, 64, 1, SPLIT3, 1>(maps, p, work, s);
        if (bn == 64 && CL == 1 && cg == pdl::kStemPackedCG)
            return launch_tile<KIND, 64, pdl::kStemPackedCG, SPLIT3, 1>(maps, p, work, s);
    } else if constexpr (KIND == pdl::KIND_GEMM) {
        switch (bn) {
            case 64: return launch_tile<KIND, 64, 1, SPLIT3, CL>(maps, p, work, s);
            case 128: return launch_tile<KIND, 128, 1, SPLIT3, CL>(maps, p, work, s);
        }
    } else {
        if (bn == 64 && cg == 1) return launch_tile<KIND, 64, 1, SPLIT3, CL>(maps, p, work, s);
        if (bn == 64 && cg == 2) return launch_tile<KIND, 64, 2, SPLIT3, CL>(maps, p, work, s);
        if (bn == 64 && cg == 4) return launch_tile<KIND, 64, 4, SPLIT3, CL>(maps, p, work, s);
        if (bn == 128 && cg == 1) return launch_tile<KIND, 128, 1, SPLIT3, CL>(maps, p, work, s);
        if (bn == 128 && cg == 2) return launch_tile<KIND, 128, 2, SPLIT3, CL>(maps, p, work, s);
        if (bn == 128 && cg == 4 && (!SPLIT3 || CL == 1)) return launch_tile<KIND, 128, 4, SPLIT3, CL>(maps, p, work, s);
        if constexpr (!SPLIT3 && CL == 1) {
            if (bn == 256 && cg == 2) return launch_tile<KIND, 256, 2, false, 1>(maps, p, work, s);
            if (bn == 256 && cg == 4) return launch_tile<KIND, 256, 4, false, 1>(maps, p, work, s);
        }
        if constexpr (SPLIT3 && CL == 1) {
            // 3xTF32 at 256 columns: one accumulator, register-traded epilogue (see the kernel)
            if (bn == 256 && cg == 2) return launch_tile<KIND, 256, 2, true, 1>(maps, p, work, s);
        }
    }
    return fail(PDL_EUNSUPPORTED, "no kernel instance for bn=%d cg=%d cluster=%d", bn, cg, CL);
}

// Extended-epilogue instances (PDL_SCALE / PDL_RELU6): cluster 1, no pairs, resident
// weights, halo or 256-column tiles (the host picks a plain schedule for these calls)
template <int KIND, bool SPLIT3>
int dispatch_epix(int bn, int cg, const pdl::TmaMaps &maps, const pdl::TileParams &p, cudaStream_t s) {
    const int work = p.m_tiles * p.n_tiles * std::max(1, p.split);
    if constexpr (KIND == pdl::KIND_STEM) {
        if (bn == 64 && cg == 1) return launch_tile<KIND, 64, 1, SPLIT3, 1, false, 0, false, true>(maps, p, work, s);
        if (bn == 64 && cg == pdl::kStemPackedCG)
            return launch_tile<KIND, 64, pdl::kStemPackedCG, SPLIT3, 1, false, 0, false, true>(maps, p, work, s);
    } else if constexpr (KIND == pdl::KIND_GEMM) {
        if (bn == 64) return launch_tile<KIND, 64, 1, SPLIT3, 1, false, 0, false, true>(maps, p, work, s);
        if (bn == 128) return launch_tile<KIND, 128, 1, SPLIT3, 1, false, 0, false, true>(maps, p, work, s);
    } else {
        if (bn == 64 && cg == 1) return launch_tile<KIND, 64, 1, SPLIT3, 1, false, 0, false, true>(maps, p, work, s);
        if (bn == 64 && cg == 2) return launch_tile<KIND, 64, 2, SPLIT3, 1, false, 0, false, true>(maps, p, work, s);
        if (bn == 64 && cg == 4) return launch_tile<KIND, 64, 4, SPLIT3, 1, false, 0, false, true>(maps, p, work, s);
        if (bn == 128 && cg == 1) return launch_tile<KIND, 128, 1, SPLIT3, 1, false, 0, false, true>(maps, p, work, s);
        if (bn == 128 && cg == 2) return launch_tile<KIND, 128, 2, SPLIT3, 1, false, 0, false, true>(maps, p, work, s);
        if (bn == 128 && cg == 4) return launch_tile<KIND, 128, 4, SPLIT3, 1, false, 0, false, true>(maps, p, work, s);
    }
    return fail(PDL_EUNSUPPORTED, "no extended-epilogue instance for bn=%d cg=%d", bn, cg);
}

// Resident-weight 1x1 conv instances (3xTF32, cluster 1): RESW bytes per plane
int dispatch_resident(int bn, int cg, int plane_bytes, const pdl::TmaMaps &maps,
                      const pdl::TileParams &p, cudaStream_t s) {
    const int work = p.m_tiles * p.n_tiles;
    if (cg == 2 && plane_bytes <= 32768) {
        if (bn == 128) return launch_tile<pdl::KIND_CONV, 128, 2, true, 1, false, 32768>(maps, p, work, s);
        if (bn == 64) return launch_tile<pdl::KIND_CONV, 64, 2, true, 1, false, 32768>(maps, p, work, s);
    }
    if (cg == 2 && plane_bytes <= 65536) {
        if (bn == 128) return launch_tile<pdl::KIND_CONV, 128, 2, true, 1, false, 65536>(maps, p, work, s);
        if (bn == 64) return launch_tile<pdl::KIND_CONV, 64, 2, true, 1, false, 65536>(maps, p, work, s);
    }
    return fail(PDL_EUNSUPPORTED, "no resident-weight instance for bn=%d cg=%d (%d B)", bn, cg, plane_bytes);
}

// Halo conv instances (stride 1, R*S > 1, cluster 1): input halo loaded once per channel
// group, every tap read from it by the staging warps (TS MMAs in both modes)
template <bool SPLIT3>
int dispatch_halo(int bn, int cg, const pdl::TmaMaps &maps, const pdl::TileParams &p, cudaStream_t s) {
    const int work = p.m_tiles * p.n_tiles * std::max(1, p.split);
    if (bn == 64 && cg == 1) return launch_tile<pdl::KIND_CONV, 64, 1, SPLIT3, 1, false, 0, true>(maps, p, work, s);
    if (bn == 64 && cg == 2) return launch_tile<pdl::KIND_CONV, 64, 2, SPLIT3, 1, false, 0, true>(maps, p, work, s);
    if (bn == 64 && cg == 4) return launch_tile<pdl::KIND_CONV, 64, 4, SPLIT3, 1, false, 0, true>(maps, p, work, s);
    if (bn == 128 && cg == 1) return launch_tile<pdl::KIND_CONV, 128, 1, SPLIT3, 1, false, 0, true>(maps, p, work, s);
    if (bn == 128 && cg == 2) return launch_tile<pdl::KIND_CONV, 128, 2, SPLIT3, 1, false, 0, true>(maps, p, work, s);
    // TF32: 64-channel k-blocks at BN=128 (one halo buffer, one weight plane per stage)
    if (bn == 128 && cg == 4) return launch_tile<pdl::KIND_CONV, 128, 4, SPLIT3, 1, false, 0, true>(maps, p, work, s);
    return fail(PDL_EUNSUPPORTED, "no halo instance for bn=%d cg=%d", bn, cg);
}

// CTA-pair (cta_group::2) conv instances: 3xTF32, cluster of 2
int dispatch_pair(int bn, int cg, const pdl::TmaMaps &maps, const pdl::TileParams &p, cudaStream_t s) {
    const int work = ((p.m_tiles + 1) / 2) * 2 * p.n_tiles;
    if (bn == 128 && cg == 2) return launch_tile<pdl::KIND_CONV, 128, 2, true, 2, true>(maps, p, work, s);
    if (bn == 64 && cg == 2) return launch_tile<pdl::KIND_CONV, 64, 2, true, 2, true>(maps, p, work, s);
    if (bn == 64 && cg == 4) return launch_tile<pdl::KIND_CONV, 64, 4, true, 2, true>(maps, p, work, s);
    return fail(PDL_EUNSUPPORTED, "no CTA-pair instance for bn=%d cg=%d", bn, cg);
}

template <int KIND, bool SPLIT3>
int dispatch_tile(int bn, int cg, int cl, const pdl::TmaMaps &maps, const pdl::TileParams &p,
                  cudaStream_t s) {
    // work in CTAs: one per (M-tile, N-tile[, split]), rounded up to whole clusters per N-tile
    const int work = ((p.m_tiles + cl - 1) / cl) * cl * p.n_tiles * std::max(1, p.split);
    if constexpr (KIND == pdl::KIND_STEM) return dispatch_bn<KIND, SPLIT3, 1>(bn, cg, maps, p, work, s);
    else {
        switch (cl) {
            case 1: return dispatch_bn<KIND, SPLIT3, 1>(bn, cg, maps, p, work, s);
            case 2: return dispatch_bn<KIND, SPLIT3, 2>(bn, cg, maps, p, work, s);
            case 4: return dispatch_bn<KIND, SPLIT3, 4>(bn, cg, maps, p, work, s);
        }
    }
    return fail(PDL_EUNSUPPORTED, "cluster size %d not in {1,2,4}", cl);
}

// ---------------------------------------------------------------- split-K
size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Split-K plan: when a layer's tiles leave persistent CTAs idle (small per-GPU
// batches: 7x7 maps at 32 images fill 64 of 148 SMs), each tile's reduction is
// cut into `split` ranges run as separate units; partials meet in the workspace
// [ctr: kSplitMaxTiles ints][part: tiles x split x 128 x BN fp32].  The counter
// block has a FIXED size so that the partials of one plan never land on the
// counters of another (a workspace reused across shapes keeps zero counters).
// req: cfg->split_k (0 = auto, 1 = off, > 1 = forced).
constexpr int kSplitMaxTiles = 256;
constexpr size_t kSplitCtrBytes = kSplitMaxTiles * sizeof(int);
struct SplitPlan {
    int split = 1, kb_per = 0;
    size_t bytes = 0;
};

SplitPlan plan_split(int m_tiles, int n_tiles, int cl, int bn, int num_kb, int seg_kb, int req) {
    const int sm_count = sms();
    SplitPlan sp;
    sp.kb_per = num_kb;
    const int tiles = (m_tiles + cl - 1) / cl * cl * n_tiles;
    int S = 1;
    if (req > 1) {
        S = std::min(req, num_kb);
    } else if (req == 0 && tiles < sm_count) {
        // cost ~ waves x (k-blocks per unit + fixed per-unit overhead of ~8 k-blocks:
        // first-load latency, TMEM drain, partial write/read; small GEMMs measured
        // slower with a 4-k-block model)
        constexpr double kOverheadKb = 8.0;
        // a split must win by > 15% under the model (marginal wins measured as losses:
        // ResNet layer 12 at 32 images, 100 tiles, x4 predicted 1% faster, ran 1.6x slower)
        double best = 0.85 * (double)((tiles + sm_count - 1) / sm_count) * (num_kb + kOverheadKb);
        for (int s = 2; s <= 16; ++s) {
            const int kps = (num_kb + s - 1) / s;
            if (kps < 16) break;  // shorter ranges lose to the partial exchange (512^3 GEMM)
            // the split units must fit one wave: a second wave of units waits for the first one's
            // reductions (ResNet layer 17 at 28 / 32 images, 56 tiles: x5 in two waves ran 74-76 us
            // against 57 us for x2 in one wave, where this model had predicted 75 vs 80)
            if ((long long)tiles * s > sm_count) break;
            const double c = (double)((tiles * s + sm_count - 1) / sm_count) * (kps + kOverheadKb) + 0.25 * s;
            if (c < best - 1e-9) {
                best = c;
                S = s;
            }
        }
    }
    if (tiles > kSplitMaxTiles) S = 1;  // only small grids split (auto: tiles < #SMs)
    if (S > 1) {
        int kps = (num_kb + S - 1) / S;
        if (kps > seg_kb) {  // ranges on segment edges, unless that unbalances the last range
            const int r = (kps + seg_kb - 1) / seg_kb * seg_kb;
            if (num_kb - r * (S - 1) >= r / 2) kps = r;
        }
        const int split = (num_kb + kps - 1) / kps;
        if (split > 1) {
            sp.split = split;
            sp.kb_per = kps;
            sp.bytes = kSplitCtrBytes + (size_t)tiles * split * 128 * bn * sizeof(float);
        }
    }
    return sp;
}

// Bind a split plan to the caller's workspace (NULL workspace + auto = no split).
int bind_split(pdl::TileParams &p, const SplitPlan &sp, void *ws, size_t ws_bytes, int cl) {
    p.split = sp.split;
    p.kb_per = sp.kb_per;
    if (sp.split == 1) return PDL_OK;
    if (!ws || ws_bytes < sp.bytes)
        return fail(PDL_EWORKSPACE, "split-K x%d needs a zero-initialised workspace of %zu bytes", sp.split, sp.bytes);
    if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(PDL_EALIGN, "split-K workspace must be 256-byte aligned");
    p.ctr = reinterpret_cast<int *>(ws);
    p.part = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(ws) + kSplitCtrBytes);
    return PDL_OK;
}

// GEMM tile choice (shared by the launch and the workspace query).
void gemm_cfg(int M, int N, const pdl_tile_cfg *cfg_in, int *bn, int *cl, int *raster) {
    const int sm_count = sms();
    // cluster 1 (no B multicast): equal at 4096^3, 3-10% faster below (r1j A/B)
    // 64-column tiles when 128-column tiles would not fill one wave: small GEMMs are
    // latency-bound chains per tile, and twice the CTAs halve the chain (graph-replayed
    // 256^3 / 512^3 / 1024^3: 9.5 / 16.5 / 21.5 -> 7.3 / 11.9 / 16.6 us; 2048^3 keeps 128)
    const long long tiles128 = (long long)((M + 127) / 128) * ((N + 127) / 128);
    *bn = (N <= 64 || tiles128 < sm_count) ? 64 : 128;
    *raster = 0;
    *cl = 1;
    if (cfg_in) {
        if (cfg_in->bn) *bn = cfg_in->bn;
        if (cfg_in->cluster_m) *cl = cfg_in->cluster_m;
        *raster = cfg_in->raster;
    }
}

size_t gemm_split_bytes(int M, int N, int K, unsigned flags, const pdl_tile_cfg *cfg_in) {
    if (M <= 0 || N <= 0 || K <= 0 || (flags & PDL_MODE_MASK) == PDL_MODE_FP32) return 0;
    int bn, cl, raster;
    gemm_cfg(M, N, cfg_in, &bn, &cl, &raster);
    if (flags & (PDL_RELU6 | PDL_SCALE)) cl = 1;  // extended-epilogue instances are cluster 1
    if (cl != 1 && cl != 2 && cl != 4) return 0;
    return plan_split((M + 127) / 128, (N + bn - 1) / bn, cl, bn, (K + 31) / 32, kSegElems / 32,
                      cfg_in ? cfg_in->split_k : 0).bytes;
}

// ---------------------------------------------------------------- conv geometry
struct ConvGeom {
    int P, Q;        // true output extents
    int Hg, Wg;      // geometry extents (flattened for 1x1/s1/p0)
    int Pg, Qg;
    bool flat;
    int BW, BH, BNI, tiles_w, tiles_h, tiles_n;
    int m_tiles;
    // segment tiles (see TileParams): 0 = box tiles
    int seg_mode = 0, seg_tile = 0, seg_imgs = 1;
};

// Box tile search.  A tile is a box of BW x BH output pixels of BNI consecutive images
// (one TMA box per 16-channel sub-tile, any BNI: the image is just the box's outermost
// dimension), BW * BH * BNI <= 128 rows.  Round 1 only packed several images into a tile
// when a whole image fit (7x7 maps), so 28x28 maps filled 112 of 128 MMA rows, 14x14 box
// tiles 98 and 7x7 maps 98: 12-23% of every tensor-core pass multiplied zero rows.  The
// search first finds the fewest waves of the persistent grid (tiles x n_tiles work units
// over the SMs -- at small batches the wave count is what the time follows), then takes the
// widest box (longest contiguous run: BW pixels x 64 B per row and image) among the shapes
// within kTileSlack of that, then the fewest tiles, then the taller box.  Runs shorter than
// kMinRunPx pixels are not considered unless the map itself is narrower.
//   halo_r / halo_s >= 0: the tile's input halo (BW + halo_s) x (BH + halo_r) x BNI pixels
//   must fit one halo buffer (kHaloSub bytes per 16-channel sub-tile), see HALO.
// Measured on the 20 ResNet-50 layers at 256 images (scripts/probe_tile_shapes.py,
// profiles/tile_shapes_r2f.log): the pick is the fastest or within 2% of the fastest
// explicit box on every layer; suite 157.6 -> 170.9 TFLOP/s same box.
constexpr int kMinRunPx = 4;
constexpr double kTileSlack = 1.04;
struct BoxShape {
    int bw = 0, bh = 0, bni = 0;
    long long tiles = 0, waves = 0;
};
BoxShape pick_box_search(int N, int Pg, int Qg, int n_tiles, int halo_r, int halo_s, long long wave);

// The search costs 5-15 us of host time; its result only depends on the arguments, so calls
// repeat it from a table (eager launches of 20-us layers would otherwise wait for the host).
BoxShape pick_box(int N, int Pg, int Qg, int n_tiles, int halo_r, int halo_s) {
    struct Key {
        int v[7];
        bool operator<(const Key &o) const { return std::lexicographical_compare(v, v + 7, o.v, o.v + 7); }
    };
    static std::mutex mu;
    static std::map<Key, BoxShape> table;
    const int wave = sms();
    const Key k{{N, Pg, Qg, n_tiles, halo_r, halo_s, wave}};
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = table.find(k);
        if (it != table.end()) return it->second;
    }
    const BoxShape b = pick_box_search(N, Pg, Qg, n_tiles, halo_r, halo_s, wave);
    std::lock_guard<std::mutex> lock(mu);
    if (table.size() > 4096) table.clear();
    table[k] = b;
    return b;
}

BoxShape pick_box_search(int N, int Pg, int Qg, int n_tiles, int halo_r, int halo_s, long long wave) {
    const int halo_px = pdl::kHaloSub / 64;
    BoxShape best;
    for (int pass = 0; pass < 2; ++pass) {
        // pass 0: the fewest waves (then tiles); pass 1: the widest box within the slack of it
        const long long wlimit = pass ? (long long)(best.waves * kTileSlack) : 0;
        BoxShape pick;
        for (int bw = std::min(Qg, 128); bw >= 1; --bw) {
            if (bw < std::min(Qg, kMinRunPx)) break;
            for (int bh = std::min(Pg, 128 / bw); bh >= 1; --bh) {
                int bni = std::min(N, 128 / (bw * bh));
                if (halo_r >= 0) bni = std::min(bni, halo_px / ((bw + halo_s) * (bh + halo_r)));
                if (bni < 1) continue;
                const long long tiles =
                    (long long)((Qg + bw - 1) / bw) * ((Pg + bh - 1) / bh) * ((N + bni - 1) / bni);
                const long long waves = (tiles * n_tiles + wave - 1) / wave;
                const BoxShape c{bw, bh, bni, tiles, waves};
                if (pass == 0) {
                    if (!pick.bw || waves < pick.waves || (waves == pick.waves && tiles < pick.tiles)) pick = c;
                } else if (waves <= wlimit) {
                    if (!pick.bw || (bw == pick.bw && tiles < pick.tiles)) pick = c;
                }
            }
            if (pass == 1 && pick.bw) break;  // widest box found
        }
        best = pick;
        if (!best.bw) break;
    }
    return best;
}
// a beats b by more than the slack (waves first, then tiles)
bool box_wins(const BoxShape &a, const BoxShape &b) {
    if (!a.bw) return false;
    if (!b.bw) return true;
    return a.waves < b.waves || (a.waves == b.waves && (long long)(a.tiles * kTileSlack) < b.tiles);
}

// n_tiles: output-channel tiles (segment tiles only pay when they cut whole waves).
// single_image: the round-1 geometry (PDL_RASTER_SINGLE_IMAGE_TILES): a tile holds several
// images only when a whole image fits.  halo_r / halo_s: see pick_box (-1: no halo limit).
// tile_w/h/n > 0: the caller's explicit box (PDL_RASTER_TILE), in image coordinates.
ConvGeom conv_geom(int N, int H, int W, int R, int S, int stride, int pad, bool allow_seg = true,
                   int n_tiles = 1, bool force_seg = false, bool single_image = false, int halo_r = -1,
                   int halo_s = -1, int tile_w = 0, int tile_h = 0, int tile_n = 0) {
    ConvGeom g{};
    g.P = (H + 2 * pad - R) / stride + 1;
    g.Q = (W + 2 * pad - S) / stride + 1;
    g.flat = (R == 1 && S == 1 && stride == 1 && pad == 0);
    g.Hg = g.flat ? 1 : H;
    g.Wg = g.flat ? H * W : W;
    g.Pg = g.flat ? 1 : g.P;
    g.Qg = g.flat ? g.P * g.Q : g.Q;
    g.BW = std::min(g.Qg, 128);
    g.BH = std::min(g.Pg, 128 / g.BW);
    g.BNI = (g.BH == g.Pg) ? std::max(1, std::min(N, 128 / (g.BW * g.BH))) : 1;
    if (tile_w > 0) {
        g.flat = false;
        g.Hg = H; g.Wg = W; g.Pg = g.P; g.Qg = g.Q;
        g.BW = tile_w; g.BH = tile_h; g.BNI = tile_n;
    } else if (!single_image) {
        const long long legacy = (long long)((g.Qg + g.BW - 1) / g.BW) * ((g.Pg + g.BH - 1) / g.BH) *
                                 ((N + g.BNI - 1) / g.BNI);
        BoxShape b = pick_box(N, g.Pg, g.Qg, n_tiles, halo_r, halo_s);
        if (halo_r >= 0) {
            // halo mode saves 3-4% on a 3x3 layer; a box that does not fit a halo buffer but
            // fills the rows better saves more (ResNet layer 17: 7x1 pixels x 18 images with
            // per-tap boxes 247 us, 7x7 x 2 images with the halo 335 us; layers 7 / 12: 4% / 3%)
            const BoxShape free_box = pick_box(N, g.Pg, g.Qg, n_tiles, -1, -1);
            if (box_wins(free_box, b)) b = free_box;
        }
        bool unflat = false;
        if (g.flat) {  // 1x1/s1/p0: also boxes of the unflattened map (rows of several images)
            // (the flattened map has the longer runs: it stays unless the boxes win by the slack)
            const BoxShape b2 = pick_box(N, g.P, g.Q, n_tiles, -1, -1);
            if (box_wins(b2, b)) { b = b2; unflat = true; }
        }
        if (b.bw && b.tiles < legacy) {
            if (unflat) { g.flat = false; g.Hg = H; g.Wg = W; g.Pg = g.P; g.Qg = g.Q; }
            g.BW = b.bw; g.BH = b.bh; g.BNI = b.bni;
        }
    }
    g.tiles_w = (g.Qg + g.BW - 1) / g.BW;
    g.tiles_h = (g.Pg + g.BH - 1) / g.BH;
    g.tiles_n = (N + g.BNI - 1) / g.BNI;
    g.m_tiles = g.tiles_w * g.tiles_h * g.tiles_n;
    // Segment tiles: small maps waste rows in box tiles (14x14: 126 + 70 of 256 rows per
    // image; 7x7: 98 of 128).  A segment tile is T consecutive bands of the (image group,
    // output row) sequence; a band is one output row of one image (Q even) or of two images
    // (Q odd), so every band is a whole number of 128-byte smem rows.  The tile loads as up
    // to three exact-height boxes {Q, h, images}, so tiles span images and fill T bands of
    // up to 128 pixels.  Only the parity-0 map is used (stride 1, or 1x1 / pad 0 stride 2),
    // and T <= kSegMaxRows box heights.
    // Odd widths (two-image bands, 7x7) are implemented but only used when forced
    // (PDL_RASTER_SEG_TILES): on ResNet's 7x7 layers they tie box tiles at best and lose
    // 9-13% on layers 18/19 (many short tiles: 2-3 boxes per load and store).
    if (g.Q % 2 && !force_seg) allow_seg = false;
    // 3x3 layers: the two boxes per tap and k-block cost what the fuller tiles save (ResNet
    // layer 12: segment 0.326-0.331 ms vs box 0.323 ms, ncu tensor pipe 64% vs 82%); 1x1
    // layers gain 4-5% (layers 13/14).  Segment tiles only for 1x1 unless forced.
    if ((R != 1 || S != 1) && !force_seg) allow_seg = false;
    {
        const int gi = (g.Q % 2) ? 2 : 1;     // images per band
        const int band = gi * g.Q;            // pixels per band
        const int T = band <= 128 ? 128 / band : 0;
        if (allow_seg && T >= 2 && T <= pdl::kSegMaxRows && (stride == 1 || (R == 1 && S == 1 && pad == 0))) {
            const long long bands = (long long)((N + gi - 1) / gi) * g.P;
            const long long mt = (bands + T - 1) / T;
            // only when it removes whole waves of the persistent grid: within one wave the
            // per-tile latency is what counts, and a tile spanning images issues 2-3 boxes
            // per k-block (measured 2-6% slower at 32-64 images when the wave count is unchanged)
            const long long wave = sms();
            const long long w_box = ((long long)g.m_tiles * n_tiles + wave - 1) / wave;
            const long long w_seg = (mt * n_tiles + wave - 1) / wave;
            // (round 2: with multi-image boxes the segment tiles lose on every ResNet layer at 256
            // and 32 images -- layers 13 / 14 at 256: 150 / 275 us against 126 / 224 us -- so they
            // are only taken when forced)
            (void)w_seg; (void)w_box;
            if (force_seg && mt < (1ll << 30)) {
                g.seg_mode = 1;
                g.seg_tile = T;
                g.seg_imgs = gi;
                g.m_tiles = (int)mt;
                g.flat = false;
                g.Hg = H;
                g.Wg = W;
                g.Pg = g.P;
                g.Qg = g.Q;
                g.BW = band;  // epilogue / transaction bytes: T bands of `band` pixels
                g.BH = T;
                g.BNI = 1;
            }
        }
    }
    return g;
}

// Narrow-channel path (ResNet stem): <= 4 real input channels, <= 8 taps per row.
bool is_stem(int C, int R, int S, int stride) {
    return C <= 4 && S <= 8 && R <= pdl::kStemMaxR && (stride == 1 || stride == 2);
}

int ceil16(int c) { return (c + 15) / 16; }

// ResNet stem (C=3, 7x7): the reduction is packed (r, s, c)-dense, 147 -> 160
// values in two k-blocks of 80 (20 four-value chunks each) instead of one
// k-block of 8 taps x 4 channels per kernel row (7 x 32 = 224): 29% fewer MMAs
// and 2 instead of 7 MMA-warp passes per tile.  Other narrow shapes keep rows.
bool stem_packed(int C, int R, int S) { return C == 3 && R == 7 && S == 7; }
int stem_kblocks(int C, int R, int S) { return stem_packed(C, R, S) ? 2 : R; }
int stem_chunks_per_kb(int C, int R, int S) { return stem_packed(C, R, S) ? 20 : 8; }

// Input channels per packed weight row: 32 (128-byte SW128 rows) when the number
// of 16-channel blocks is even, else 16 (64-byte SW64 rows).
int weight_group(int C) { return ceil16(C) % 2 == 0 ? 32 : 16; }

void conv_default_cfg(int C, int K, int R, int S, pdl_tile_cfg *c, unsigned flags = 0, bool wide = true) {
    const int CT = ceil16(C);
    c->bm = 128;
    c->bn = K >= 128 ? 128 : 64;
    int cg = (CT % 2 == 0) ? 2 : 1;
    // BN=64 spatial convs: 64-channel k-blocks halve the MMA-warp passes per tile
    // (the 12 N=64 MMAs of a 32-channel block do not cover the pass overhead;
    // measured 0.39 -> 0.345 ms on ResNet layer 3, profiles/sweep_r1.json)
    if (c->bn == 64 && R * S > 1 && CT % 4 == 0) cg = 4;
    // ... and BN=64 1x1 convs with >= 128 input channels (round-2 sweep, profiles/sweep_r2n_b256.json:
    // ResNet layer 5, c256 -> k64: 0.196 ms against 0.224-0.235 ms with resident weights and
    // 32-channel k-blocks; layer 2, c64 -> k64, would have one k-block per tile and keeps them)
    if (c->bn == 64 && R * S == 1 && CT % 4 == 0 && CT >= 8 && (flags & PDL_MODE_MASK) == PDL_MODE_3XTF32) cg = 4;
    // TF32: 64-channel k-blocks everywhere the channels allow (one weight plane per stage
    // leaves room).  A 32-channel TF32 k-block is 4 MMAs against the fixed per-k-block
    // hand-off; doubling it made the 1x1 layers 25-35% faster (layer 13: 122.8 -> 88.9 us,
    // layer 19: 207.8 -> 137.8 us) and the halo 3x3 layers 5% faster.
    // (1x1 layers with <= 128 input channels keep 32-channel blocks: with only 1-2
    // k-blocks per tile they lose the k-loop pipelining -- layers 2/4/8 were 3-4% slower)
    if ((flags & PDL_MODE_MASK) == PDL_MODE_TF32 && CT % 4 == 0 && (R * S > 1 || CT >= 16)) cg = 4;
    // TF32 convs with K % 256 == 0: 256-column tiles (one N=256 MMA per K step, half the A
    // fill per flop; streaming epilogue), 32-channel k-blocks (48 KB stages), no halo mode
    // (its TS MMAs need TMEM columns the two 256-column accumulators use).  1x1 layers
    // 10-21% faster in the suite; 3x3 layers 12/17 151 -> 135 / 168 -> 132 us isolated.
    // (not when the caller asks for a multicast cluster or split-K, which 256 tiles lack)
    // (64-channel k-blocks at 256 columns -- two 96 KB stages -- helped the spatial layers 12 / 17 by
    // 6-8% while the tile decode still divided (profiles/tf32_bn256_bk64_r2q.log); with the divide-free
    // decode 32-channel k-blocks win again, layer 12: 96 vs 117 us, profiles/sweep_r2z_b256.json)
    if (wide && (flags & PDL_MODE_MASK) == PDL_MODE_TF32 && K % 256 == 0 && CT % 2 == 0) {
        c->bn = 256;
        cg = 2;
    }
    c->bk = 16 * cg;
    c->stages = 0;
    c->cluster_m = kDefaultConvCluster;
    c->cluster_n = c->split_k = 1;
    c->raster = 0;
}

// The default schedule of a call: conv_default_cfg, except that 256-column tiles (which cannot
// split the reduction) give way to the 128-column schedule when they would leave SMs idle --
// small batches: ResNet layer 17 at 32 images is 28 tiles of 256 columns (TF32 82 -> 46 us).
void conv_auto_cfg(int N, int C, int K, int H, int W, int R, int S, int stride, int pad, unsigned flags,
                   const pdl_tile_cfg *cfg_in, pdl_tile_cfg *cfg) {
    const bool wide = !(cfg_in && (cfg_in->cluster_m > 1 || cfg_in->split_k > 1));
    conv_default_cfg(C, K, R, S, cfg, flags, wide);
    // 3xTF32 at 256 columns (one accumulator, register-traded epilogue; results bitwise those of the
    // 128-column tiles; cfg bn = 256, bk = 32) is NOT a default.  Before the tile decode lost its integer
    // divides it was 3-9% faster on the 1x1 layers with >= 512 output channels (half as many tile
    // decodes per flop: profiles/bn256_3xtf32_r2y.log); with the divide-free decode the 128-column
    // tiles win by 5-10% on layers 9 / 14 / 18 / 19 and tie on 8 / 13 (profiles/bn256_vs_128_r2z.log):
    // two 80 KB stages and an un-overlapped accumulator drain against four stages and two accumulators.
    if (cfg->bn == 256 && !(cfg_in && (cfg_in->bn || cfg_in->bk))) {
        const ConvGeom g0 = conv_geom(N, H, W, R, S, stride, pad, false, K / 256, false,
                                      cfg_in && (cfg_in->raster & PDL_RASTER_SINGLE_IMAGE_TILES));
        // (only when the twice as many 128-column tiles still fit one wave: 112 tiles of 256 columns
        // -- layers 18 / 19 at 32 images -- beat 224 of 128 in two waves by 6-15%)
        if (2ll * g0.m_tiles * (K / 256) <= sms()) conv_default_cfg(C, K, R, S, cfg, flags, false);
    }
}

// Output map of the TMA-stored epilogue: y [N][KT][Pg][Qg][16] in the tile
// geometry (flattened for 1x1/s1/p0), box = one 16-channel block of a tile.
int encode_y(CUtensorMap *m, float *y, int N, int KT, int Pg, int Qg, int BW, int BH, int BNI) {
    const cuuint64_t dims[5] = {16, (cuuint64_t)Qg, (cuuint64_t)Pg, (cuuint64_t)KT, (cuuint64_t)N};
    const cuuint64_t str[4] = {64, (cuuint64_t)Qg * 64, (cuuint64_t)Pg * Qg * 64,
                               (cuuint64_t)KT * Pg * Qg * 64};
    const cuuint32_t box[5] = {16, (cuuint32_t)BW, (cuuint32_t)BH, 1, (cuuint32_t)BNI};
    return encode(m, y, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B, "conv y");
}

int conv_check(const float *x, const float *y, int N, int C, int K, int H, int W, int R, int S,
               int stride, int pad) {
    if (N <= 0 || C <= 0 || K <= 0 || H <= 0 || W <= 0 || R <= 0 || S <= 0)
        return fail(PDL_EINVAL, "conv: non-positive dimension");
    if (K % 16) return fail(PDL_EINVAL, "conv: K must be a multiple of 16 (got %d)", K);
    if (stride != 1 && stride != 2) return fail(PDL_EUNSUPPORTED, "conv: stride must be 1 or 2");
    if (pad < 0 || pad >= R || pad >= S) return fail(PDL_EINVAL, "conv: bad padding %d", pad);
    if ((H + 2 * pad - R) < 0 || (W + 2 * pad - S) < 0) return fail(PDL_EINVAL, "conv: empty output");
    if (!aligned16(x) || !aligned16(y)) return fail(PDL_EALIGN, "conv: x / y must be 16-byte aligned");
    return PDL_OK;
}

// Stem tile = BW x BH output pixels (<= 128); its input halo (box_w x box_h pixels,
// 16 B each) is one TMA box and one pipeline stage.  Per tile the engine spends
// ~R x 700 cycles on MMAs and the TMA ~4.4 cycles per 16-byte halo element (both
// measured on B200, profiles/trace_*); pick the shape minimising tiles x max(the two).
bool stem_tile(int P, int Q, int R, int S, int stride, int *BWo, int *BHo) {
    constexpr double kMmaPerRow = 700.0, kTmaPerElem = 4.4;
    double best = 1e30;
    int BW = 0, BH = 0;
    for (int bw = std::min(Q, 128); bw >= 1; --bw) {
        const int bh = std::min(P, 128 / bw);
        const int bxw = (bw - 1) * stride + S, bxh = (bh - 1) * stride + R;
        if (bxw > 256 || bxh > 256 || 16 * bxw * bxh > pdl::kStemHaloBytes) continue;
        const double tiles = (double)((Q + bw - 1) / bw) * ((P + bh - 1) / bh);
        const double cost = tiles * std::max(R * kMmaPerRow, kTmaPerElem * bxw * bxh);
        if (cost < best - 1e-9) { best = cost; BW = bw; BH = bh; }
    }
    *BWo = BW;
    *BHo = BH;
    return BW > 0;
}

int conv_fwd_stem(const float *x, const float *wp, const float *bias, float *y, int N, int C,
                  int K, int H, int W, int R, int S, int stride, int pad, unsigned flags,
                  const pdl_tile_cfg *cfg_in, cudaStream_t st) {
    int rc;
    const bool split = (flags & PDL_MODE_MASK) == PDL_MODE_3XTF32;
    const int bn = 64;  // resident weights: 2 planes x 7 rows x 8 taps x 64 x 16 B = 112 KB
    (void)cfg_in;
    const int P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
    // tile = BW x BH output pixels (<= 128); its input halo (box_w x box_h pixels,
    // 16 B each) is one TMA box and one pipeline stage.  Per tile the engine spends
    // ~R x 700 cycles on MMAs and the TMA ~4.4 cycles per 16-byte halo element
    // (both measured on B200, profiles/trace_*); pick the shape minimising
    // tiles x max(the two).
    int BW = 0, BH = 0;
    if (!stem_tile(P, Q, R, S, stride, &BW, &BH))
        return fail(PDL_EUNSUPPORTED, "stem: no halo tile fits (S=%d R=%d)", S, R);
    int box_w = (BW - 1) * stride + S;
    const int box_h = (BH - 1) * stride + R;
    // packed stride-2 stem: the halo is loaded as two dense boxes, even and odd input
    // columns (BW + (S+1)/2 - 1 pixels each), so one tap's pixels are contiguous in smem
    const bool parity = stem_packed(C, R, S) && stride == 2;
    int halo_odd = 0;
    if (parity) {
        box_w = BW - 1 + (S + 1) / 2;
        halo_odd = (box_w * box_h * 16 + 127) / 128 * 128;
        if (2 * halo_odd > pdl::kStemHaloBytes) return fail(PDL_EUNSUPPORTED, "stem: halo too large");
    }
    pdl::TmaMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    // pixel = 16 channels (nChw16c, 64 B, of which the kernel reads the first 16 B) or,
    // with PDL_X_NCHW4C, exactly the 4 channels it reads (16 B: a quarter of the HBM
    // and PCIe bytes -- the padded layout makes HBM return the whole 64-byte pixel)
    const bool compact = (flags & PDL_X_NCHW4C) != 0;
    const cuuint64_t px = compact ? 16 : 64;  // bytes per pixel
    const cuuint64_t pc = px / 4;             // floats per pixel
    if (parity) {
        for (int par = 0; par < 2; ++par) {
            const cuuint64_t dims[5] = {pc, (cuuint64_t)((W - par + 1) / 2), (cuuint64_t)H, 1, (cuuint64_t)N};
            const cuuint64_t str[4] = {2 * px, (cuuint64_t)W * px, (cuuint64_t)H * W * px, (cuuint64_t)H * W * px};
            const cuuint32_t box[5] = {4, (cuuint32_t)box_w, (cuuint32_t)box_h, 1, 1};
            if ((rc = encode(&maps.a[par], x + par * pc, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE,
                             "stem x parity", CU_TENSOR_MAP_L2_PROMOTION_NONE)))
                return rc;
        }
    } else {
        const cuuint64_t dims[5] = {pc, (cuuint64_t)W, (cuuint64_t)H, 1, (cuuint64_t)N};
        const cuuint64_t str[4] = {px, (cuuint64_t)W * px, (cuuint64_t)H * W * px, (cuuint64_t)H * W * px};
        const cuuint32_t box[5] = {4, (cuuint32_t)box_w, (cuuint32_t)box_h, 1, 1};
        // nChw16c: only 16 of every 64 bytes are used, do not promote to 256B L2 fills;
        // compact rows are dense
        if ((rc = encode(&maps.a[0], x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE, "stem x",
                         compact ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE)))
            return rc;
    }
    {
        const int planes = split ? 2 : 1;
        const int nkb = stem_kblocks(C, R, S), cpk = stem_chunks_per_kb(C, R, S);
        // [kb][chunk][plane][K][4] (the lo plane of a chunk follows its hi plane)
        const cuuint64_t dims[5] = {4, (cuuint64_t)K, (cuuint64_t)planes, (cuuint64_t)cpk, (cuuint64_t)nkb};
        const cuuint64_t str[4] = {16, (cuuint64_t)K * 16, (cuuint64_t)planes * K * 16,
                                   (cuuint64_t)cpk * planes * K * 16};
        const cuuint32_t box[5] = {4, (cuuint32_t)bn, (cuuint32_t)planes, (cuuint32_t)cpk, (cuuint32_t)nkb};  // resident
        if ((rc = encode(&maps.b, wp, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE, "stem w")))
            return rc;
    }
    if ((rc = encode_y(&maps.y[0], y, N, K / 16, P, Q, BW, BH, 1))) return rc;
    pdl::TileParams p{};
    p.num_kb = stem_kblocks(C, R, S);
    p.seg_kb = std::max(1, kSegElems / (4 * stem_chunks_per_kb(C, R, S)));
    p.n_out = K;
    p.flags = flags & ~(unsigned)PDL_X_NCHW4C;
    p.bias = bias;
    p.out = y;
    p.nimg = N;
    p.P = P;
    p.Q = Q;
    p.KT = K / 16;
    p.R = R;
    p.S = S;
    p.pad = pad;
    p.stride = stride;
    p.CT = 1;
    p.BW = BW;
    p.BH = BH;
    p.BNI = 1;
    p.box_w = box_w;
    p.box_h = box_h;
    p.halo_odd = halo_odd;
    p.tiles_w = (Q + BW - 1) / BW;
    p.tiles_h = (P + BH - 1) / BH;
    p.m_tiles = p.tiles_w * p.tiles_h * N;
    p.n_tiles = (K + bn - 1) / bn;
    // the grid is a multiple of n_tiles: every CTA keeps one N-tile (resident weights)
    const int scg = stem_packed(C, R, S) ? pdl::kStemPackedCG : 1;
    if (flags & (PDL_SCALE | PDL_RELU6))
        return split ? dispatch_epix<pdl::KIND_STEM, true>(bn, scg, maps, p, st)
                     : dispatch_epix<pdl::KIND_STEM, false>(bn, scg, maps, p, st);
    if (split) return dispatch_tile<pdl::KIND_STEM, true>(bn, scg, 1, maps, p, st);
    return dispatch_tile<pdl::KIND_STEM, false>(bn, scg, 1, maps, p, st);
}

// ws / ws_bytes: split-K workspace (may be NULL: no split unless cfg forces one).
// query != NULL: only store the split-K workspace bytes this call would need.
int conv_fwd_tc(const float *x, const float *wp, const float *bias, float *y, int N, int C, int K,
                int H, int W, int R, int S, int stride, int pad, unsigned flags,
                const pdl_tile_cfg *cfg_in, cudaStream_t st, void *ws = nullptr, size_t ws_bytes = 0,
                size_t *query = nullptr, pdl_schedule *sched = nullptr) {
    int rc;
    if (stride == 2 && (H < 2 || W < 2)) return fail(PDL_EUNSUPPORTED, "conv: stride 2 needs H,W >= 2");
    if ((flags & PDL_X_NCHW4C) && !is_stem(C, R, S, stride))
        return fail(PDL_EUNSUPPORTED, "conv: PDL_X_NCHW4C (compact 4-channel x) is the narrow-channel "
                    "path's layout: C <= 4, S <= 8, R <= %d (got C=%d R=%d S=%d)", pdl::kStemMaxR, C, R, S);
    if (is_stem(C, R, S, stride)) {
        if (query) {
            *query = 0;
            return PDL_OK;
        }
        if (sched) {
            const int P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
            int BW, BH;
            if (!stem_tile(P, Q, R, S, stride, &BW, &BH)) return fail(PDL_EUNSUPPORTED, "stem: no halo tile fits");
            std::memset(sched, 0, sizeof(*sched));
            sched->kind = 2;
            sched->bn = 64;
            sched->bk = 4 * stem_chunks_per_kb(C, R, S);
            sched->cluster = 1;
            sched->tile_w = BW;
            sched->tile_h = BH;
            sched->tile_images = 1;
            sched->m_tiles = ((Q + BW - 1) / BW) * ((P + BH - 1) / BH) * N;
            sched->n_tiles = (K + 63) / 64;
            sched->num_kb = sched->kb_per = stem_kblocks(C, R, S);
            sched->split = 1;
            sched->resident = 1;
            sched->halo = 1;
            return PDL_OK;
        }
        if ((rc = get_encode())) return rc;
        return conv_fwd_stem(x, wp, bias, y, N, C, K, H, W, R, S, stride, pad, flags, cfg_in, st);
    }
    if (cfg_in && (cfg_in->raster & ~kRasterBits))
        return fail(PDL_EUNSUPPORTED, "conv: unsupported raster bits 0x%x", cfg_in->raster & ~kRasterBits);
    const bool split = (flags & PDL_MODE_MASK) == PDL_MODE_3XTF32;
    pdl_tile_cfg cfg;
    conv_auto_cfg(N, C, K, H, W, R, S, stride, pad, flags, cfg_in, &cfg);
    if (cfg_in) {
        if (cfg_in->bn) cfg.bn = cfg_in->bn;
        if (cfg_in->bk) cfg.bk = cfg_in->bk;
        if (cfg_in->cluster_m) cfg.cluster_m = cfg_in->cluster_m;
        if (cfg_in->cluster_n) cfg.cluster_n = cfg_in->cluster_n;
        cfg.raster = cfg_in->raster;
    }
    // scale / ReLU6 epilogue: the plain schedule of the EPIX instances (cluster 1, at most
    // 128 columns; no pairs, resident weights or halo)
    const bool epix = flags & (PDL_SCALE | PDL_RELU6);
    if (epix) {
        if (cfg.bn > 128) cfg.bn = 128;
        cfg.cluster_m = cfg.cluster_n = 1;
    }
    // cluster_n == 2: the tile is computed by a CTA pair with cta_group::2 MMAs
    // (M = 256, each CTA holds half of B); 3xTF32 only
    const bool pair = cfg.cluster_n == 2 && split;
    if (pair) cfg.cluster_m = 2;
    // 1x1 convs whose N-tile weight slice fits in 64 KB per plane keep it resident
    // (loaded once per CTA; stages carry A only) unless a multicast cluster is asked for
    const int res_plane = ceil16(C) * 16 * cfg.bn * 4;
    const bool resident = split && !pair && !epix && R == 1 && S == 1 && cfg.bk == 32 && res_plane <= 65536 &&
                          cfg.bn <= 128 &&
                          (!cfg_in || cfg_in->cluster_m <= 1);
    if (resident) cfg.cluster_m = 1;
    const int CT = ceil16(C), KT = K / 16, cg = cfg.bk / 16;
    int cl = cfg.cluster_m;
    const int G = weight_group(C);
    if ((G == 32) != (cg >= 2)) return fail(PDL_EINVAL, "conv: bk=%d incompatible with C=%d", cfg.bk, C);
    if (cl != 1 && cl != 2 && cl != 4) return fail(PDL_EINVAL, "conv: cluster_m must be 1, 2 or 4");
    if (cfg.bn % (8 * cl)) return fail(PDL_EINVAL, "conv: bn=%d not divisible into %d slices", cfg.bn, cl);
    if (cg < 1 || CT % cg) return fail(PDL_EINVAL, "conv: bk=%d does not divide C=%d", cfg.bk, C);
    // halo mode wanted (decided before the tile shape: the shape must fit a halo buffer)
    const bool halo_cg4 = (cfg_in && (cfg_in->raster & PDL_RASTER_HALO_CG4)) || cfg.bn == 64;
    const bool want_halo = !pair && !resident && !epix && stride == 1 && R * S > 1 && cl == 1 && cfg.bn <= 128 &&
                           (cg <= 2 || (!split && cg == 4) || halo_cg4 || cfg.bn == 128) &&
                           !(cfg_in && (cfg_in->raster & PDL_RASTER_NO_HALO));
    // explicit tile box (PDL_RASTER_TILE): bits 8-15 BW, 16-23 BH, 24-30 BNI
    const int tile_w = cfg_in ? (cfg_in->raster >> 8) & 0xff : 0, tile_h = cfg_in ? (cfg_in->raster >> 16) & 0xff : 0,
              tile_n = cfg_in ? (cfg_in->raster >> 24) & 0x7f : 0;
    if (tile_w || tile_h || tile_n) {
        const int Pq = (H + 2 * pad - R) / stride + 1, Qq = (W + 2 * pad - S) / stride + 1;
        if (tile_w < 1 || tile_h < 1 || tile_n < 1 || tile_w * tile_h * tile_n > 128 || tile_w > Qq || tile_h > Pq ||
            tile_n > N || pair)
            return fail(PDL_EINVAL, "conv: tile box %d x %d pixels x %d images must be 1..128 rows inside the "
                        "%d x %d map and the batch", tile_w, tile_h, tile_n, Qq, Pq);
    }
    const ConvGeom g = conv_geom(N, H, W, R, S, stride, pad,
                                 !pair && !tile_w && !(cfg_in && (cfg_in->raster & PDL_RASTER_BOX_TILES)),
                                 (K + cfg.bn - 1) / cfg.bn, cfg_in && (cfg_in->raster & PDL_RASTER_SEG_TILES),
                                 pair || (cfg_in && (cfg_in->raster & PDL_RASTER_SINGLE_IMAGE_TILES)),
                                 want_halo ? R - 1 : -1, want_halo ? S - 1 : -1, tile_w, tile_h, tile_n);
    // segment tiles: no weight multicast by default (pairs of CTAs in lockstep wait for
    // the one whose tile spans two images; cluster 1 measured 4-9% faster on ResNet
    // layers 12/13/15 at 256 images)
    if ((g.seg_mode && !(cfg_in && cfg_in->cluster_m)) || epix) cl = 1;
    const int m_tiles = g.m_tiles, n_tiles = (K + cfg.bn - 1) / cfg.bn;
    const int num_kb = (CT / cg) * R * S;
    // BN=256 (TF32): one accumulation segment per tile, never split (streaming epilogue)
    // BN=256: TF32 streams one accumulation segment per tile; 3xTF32 keeps the 256-element segments
    const int seg_kb = (cfg.bn > 128 && !split) ? num_kb : std::max(1, kSegElems / (16 * cg));
    SplitPlan spl;
    spl.kb_per = num_kb;
    if (!pair && !resident && cfg.bn <= 128) {
        const int req = cfg_in ? cfg_in->split_k : 0;
        spl = plan_split(m_tiles, n_tiles, cl, cfg.bn, num_kb, seg_kb, (ws || query) ? req : (req > 1 ? req : 1));
    }
    if (query) {
        *query = spl.bytes;
        return PDL_OK;
    }
    // halo mode (3xTF32, stride 1, spatial filter): one box of the tile's whole input halo
    // per channel group instead of one box per tap
    // 3xTF32 64-channel k-blocks at BN=64 (layer 3) take halo mode with one halo buffer:
    // 333 vs 340 us isolated in round 1p (a tie in round 1l); PDL_RASTER_HALO_CG4 forces it
    // (3xTF32: not with 64-channel k-blocks at BN=128 -- two 64 KB halo buffers leave 2 weight
    // stages; BN=128 3x3 layers 7/12/17 run 4-6% faster isolated.  TF32 stages carry one
    // weight plane, so 64-channel k-blocks keep 4 stages.)
    const int halo_w = g.BW + S - 1, halo_h = g.BH + R - 1;
    const bool halo = want_halo && !g.seg_mode && halo_w <= 256 && halo_h <= 256 &&
                      halo_w * halo_h * g.BNI * 64 <= pdl::kHaloSub;
    if (sched) {
        std::memset(sched, 0, sizeof(*sched));
        sched->kind = 1;
        sched->bn = cfg.bn;
        sched->bk = cfg.bk;
        sched->cluster = pair ? 2 : cl;
        sched->tile_w = g.seg_mode ? g.Q * g.seg_imgs : g.BW;
        sched->tile_h = g.seg_mode ? g.seg_tile : g.BH;
        sched->tile_images = g.seg_mode ? g.seg_imgs : g.BNI;
        sched->seg_rows = g.seg_mode ? g.seg_tile : 0;
        sched->m_tiles = m_tiles;
        sched->n_tiles = n_tiles;
        sched->num_kb = num_kb;
        sched->split = spl.split;
        sched->kb_per = spl.kb_per;
        sched->halo = halo ? 1 : 0;
        sched->resident = resident ? 1 : 0;
        sched->pair = pair ? 1 : 0;
        sched->order = (cl == 1 && !pair && !resident) ? (cfg.raster & 1) : 0;
        sched->flat = g.flat ? 1 : 0;
        sched->splitk_workspace_bytes = spl.bytes;
        return PDL_OK;
    }
    if ((rc = get_encode())) return rc;

    pdl::TmaMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    cuuint32_t abox[5] = {16, (cuuint32_t)g.BW, (cuuint32_t)g.BH, 1, (cuuint32_t)g.BNI};
    if (halo) {
        abox[1] = (cuuint32_t)halo_w;
        abox[2] = (cuuint32_t)halo_h;
    }
    if (g.seg_mode) {
        // one A map and one y map per box height 1..T (parity-0 view for stride 2)
        const int Wv = stride == 1 ? W : (W + 1) / 2, Hv = stride == 1 ? H : (H + 1) / 2;
        const cuuint64_t cs = stride == 1 ? 64 : 128, rs = stride == 1 ? (cuuint64_t)W * 64 : (cuuint64_t)W * 128;
        const cuuint64_t dims[5] = {16, (cuuint64_t)Wv, (cuuint64_t)Hv, (cuuint64_t)CT, (cuuint64_t)N};
        const cuuint64_t str[4] = {cs, rs, (cuuint64_t)H * W * 64, (cuuint64_t)CT * H * W * 64};
        // stride 2 reads every other 64-byte pixel: no 256-byte L2 promotion (it would
        // fetch the skipped odd pixels too)
        const CUtensorMapL2promotion l2 = stride == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                      : CU_TENSOR_MAP_L2_PROMOTION_NONE;
        for (int h = 1; h <= std::min(g.seg_tile, g.P); ++h) {
            const cuuint32_t box[5] = {16, (cuuint32_t)g.Q, (cuuint32_t)h, 1, (cuuint32_t)g.seg_imgs};
            if ((rc = encode(&maps.a[h - 1], x, 5, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B, "conv x rows",
                             l2)))
                return rc;
            if ((rc = encode_y(&maps.y[h - 1], y, N, KT, g.P, g.Q, g.Q, h, g.seg_imgs))) return rc;
        }
    } else if (stride == 1) {
        const cuuint64_t dims[5] = {16, (cuuint64_t)g.Wg, (cuuint64_t)g.Hg, (cuuint64_t)CT, (cuuint64_t)N};
        const cuuint64_t str[4] = {64, (cuuint64_t)g.Wg * 64, (cuuint64_t)g.Hg * g.Wg * 64,
                                   (cuuint64_t)CT * g.Hg * g.Wg * 64};
        if ((rc = encode(&maps.a[0], x, 5, dims, str, abox, CU_TENSOR_MAP_SWIZZLE_64B, "conv x")))
            return rc;
    } else {
        // 1-wide filters never read the odd input columns, so a parity map's 64-byte
        // pixels sit 128 bytes apart and nothing else reads the gaps: 256-byte L2
        // promotion would fetch every skipped pixel as well (ncu: 1.6x the algorithmic
        // DRAM bytes on ResNet layers 6/11/16).  Wider filters read the odd columns
        // through the other parity maps, so the promoted lines are used.
        const CUtensorMapL2promotion l2 = S == 1 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                                 : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
        for (int ph = 0; ph < 2; ++ph)
            for (int pw = 0; pw < 2; ++pw) {
                const cuuint64_t dims[5] = {16, (cuuint64_t)((W - pw + 1) / 2),
                                            (cuuint64_t)((H - ph + 1) / 2), (cuuint64_t)CT,
                                            (cuuint64_t)N};
                const cuuint64_t str[4] = {128, (cuuint64_t)W * 128, (cuuint64_t)H * W * 64,
                                           (cuuint64_t)CT * H * W * 64};
                const float *base = x + ((size_t)ph * W + pw) * 16;
                if ((rc = encode(&maps.a[ph * 2 + pw], base, 5, dims, str, abox,
                                 CU_TENSOR_MAP_SWIZZLE_64B, "conv x parity", l2)))
                    return rc;
            }
    }
    {
        const int planes = split ? 2 : 1;
        const int NB = cg >= 2 ? cg / 2 : 1;
        const cuuint64_t rowb = (cuuint64_t)G * 4;
        const cuuint64_t dims[5] = {(cuuint64_t)G, (cuuint64_t)K, (cuuint64_t)(R * S),
                                    (cuuint64_t)(CT * 16 / G), (cuuint64_t)planes};
        const cuuint64_t str[4] = {rowb, (cuuint64_t)K * rowb, (cuuint64_t)R * S * K * rowb,
                                   (cuuint64_t)(CT * 16 / G) * R * S * K * rowb};
        // cluster: each CTA multicasts a BN/cl-row slice of one (plane, nb) sub-tile per op
        // pair: each CTA loads its BN/2 rows of every (plane, nb) sub-tile itself;
        // resident: one box = the N-tile's whole slice of one plane
        const bool whole = cl == 1 || pair;
        cuuint32_t bbox[5] = {(cuuint32_t)G, (cuuint32_t)(pair ? cfg.bn / 2 : cfg.bn / cl), 1,
                              (cuuint32_t)(whole ? NB : 1), (cuuint32_t)(whole ? planes : 1)};
        if (resident) {
            bbox[1] = (cuuint32_t)cfg.bn;
            bbox[3] = (cuuint32_t)(CT * 16 / G);
            bbox[4] = 1;
        }
        if ((rc = encode(&maps.b, wp, 5, dims, str, bbox,
                         G == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, "conv w")))
            return rc;
    }
    if (!g.seg_mode && (rc = encode_y(&maps.y[0], y, N, KT, g.Pg, g.Qg, g.BW, g.BH, g.BNI))) return rc;
    pdl::TileParams p{};
    p.num_kb = num_kb;
    p.seg_kb = seg_kb;
    p.n_out = K;
    p.flags = flags;
    p.bias = bias;
    p.out = y;
    p.nimg = N;
    p.P = g.Pg;
    p.Q = g.Qg;
    p.KT = KT;
    p.R = R;
    p.S = S;
    p.pad = pad;
    p.stride = stride;
    p.CT = CT;
    p.BW = g.BW;
    p.BH = g.BH;
    p.BNI = g.BNI;
    p.tiles_w = g.tiles_w;
    p.tiles_h = g.tiles_h;
    p.seg_mode = g.seg_mode;
    p.seg_tile = g.seg_tile;
    p.seg_bytes = g.Q * g.seg_imgs * 64;
    p.seg_imgs = g.seg_imgs;
    p.m_tiles = m_tiles;
    // tile order (raster bit 0) only where CTAs do not pin an N-tile: no clusters, pairs,
    // resident weights
    p.raster = (cl == 1 && !pair && !resident) ? (cfg.raster & 1) : 0;
    p.n_tiles = n_tiles;
    if ((rc = bind_split(p, spl, ws, ws_bytes, cl))) return rc;
    if (halo) {
        p.box_w = halo_w;
        p.box_h = halo_h;
        return split ? dispatch_halo<true>(cfg.bn, cg, maps, p, st) : dispatch_halo<false>(cfg.bn, cg, maps, p, st);
    }
    if (pair) return dispatch_pair(cfg.bn, cg, maps, p, st);
    if (resident) {
        p.res_bytes = res_plane;
        return dispatch_resident(cfg.bn, cg, res_plane, maps, p, st);
    }
    if (epix)
        return split ? dispatch_epix<pdl::KIND_CONV, true>(cfg.bn, cg, maps, p, st)
                     : dispatch_epix<pdl::KIND_CONV, false>(cfg.bn, cg, maps, p, st);
    if (split) return dispatch_tile<pdl::KIND_CONV, true>(cfg.bn, cg, cl, maps, p, st);
    return dispatch_tile<pdl::KIND_CONV, false>(cfg.bn, cg, cl, maps, p, st);
}

// ---------------------------------------------------------------- host-buffer pipeline
// Copy streams and slot events of pdl_conv2d_fwd_host, one set per (device,
// workspace), in a process-wide table: the relaxed (PDL_HOST_X_READY) ordering
// depends on the previous call that used the same workspace, whichever thread made
// it.  The table mutex is held while a call enqueues its work, so calls sharing a
// workspace from several threads see each other's events in a consistent order.
constexpr int kHostSlots = 3;     // device staging slots (x and y) in flight
struct HostPipe {
    bool ready = false;
    cudaStream_t h2d = nullptr, d2h = nullptr, cs = nullptr;  // copies in / out, convolutions
    cudaEvent_t entry = nullptr, x_in[kHostSlots], done[kHostSlots], y_done[2];
    cudaEvent_t x_free = nullptr;     // last conv of the previous call (x area no longer read)
    bool used = false;                // a previous call completed its enqueue on this workspace
    size_t last_ws_bytes = 0;
    int parity = 0;                   // y area half of the next call
};
std::mutex g_pipe_mu;
std::map<std::pair<int, const void *>, HostPipe> g_pipes;

// caller holds g_pipe_mu
int host_pipe(const void *ws, HostPipe **out) {
    const int dev = cur_dev();
    if (dev < 0) return fail(PDL_EDEVICE, "conv host: no current device");
    HostPipe &hp = g_pipes[{dev, ws}];
    if (!hp.ready) {
        const unsigned ef = cudaEventDisableTiming;
        bool ok = cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&hp.cs, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaEventCreateWithFlags(&hp.entry, ef) == cudaSuccess &&
                  cudaEventCreateWithFlags(&hp.x_free, ef) == cudaSuccess;
        for (int i = 0; ok && i < kHostSlots; ++i)
            ok = cudaEventCreateWithFlags(&hp.x_in[i], ef) == cudaSuccess &&
                 cudaEventCreateWithFlags(&hp.done[i], ef) == cudaSuccess;
        for (int q = 0; ok && q < 2; ++q)
            ok = cudaEventCreateWithFlags(&hp.y_done[q], ef) == cudaSuccess &&
                 cudaEventRecord(hp.y_done[q], hp.d2h) == cudaSuccess;
        if (!ok) return fail(PDL_ELAUNCH, "conv host: stream/event creation failed");
        hp.ready = true;
    }
    *out = &hp;
    return PDL_OK;
}

// x bytes per host-pipeline copy.  e2e A/B on the 256-image suite (scripts/ab_e2e.sh,
// profiles/e2e_chunk_ab_r1o.log): 8 MB 138.8 ms/step, 16 MB 130.8, 32 MB 127.6, 64 MB 126.8
#ifndef PDL_HOST_CHUNK_MB
#define PDL_HOST_CHUNK_MB 64
#endif
// Images per pipeline chunk: ~64 MB of x per copy (PCIe-efficient transfers), at
// least 4 chunks when the batch allows (so both copy directions overlap).
int host_chunk(int N, size_t x_img) {
    const size_t target = (size_t)PDL_HOST_CHUNK_MB << 20;
    int c = (int)std::max<size_t>(1, target / std::max<size_t>(x_img, 1));
    return std::max(1, std::min(c, (N + 3) / 4));
}

}  // namespace

extern "C" {

int pdl_abi_version(void) { return PDL_ABI_VERSION; }

// Diagnostics (not in pdl.h): route tile-engine timeline stamps of block 0 to a
// caller-owned device buffer of TR_COUNT * 4096 uint64 (PDL_TRACE builds only).
void pdl_debug_set_trace(void *dev_buffer) {
    g_trace = reinterpret_cast<unsigned long long *>(dev_buffer);
}
const char *pdl_last_error(void) { return g_err.c_str(); }
int pdl_last_launch_count(void) { return g_launches; }
int pdl_device_check(void) { return device_check(); }

size_t pdl_conv2d_packed_bytes(int C, int K, int R, int S, unsigned flags) {
    const int planes = (flags & PDL_MODE_MASK) == PDL_MODE_3XTF32 ? 2 : 1;
    if (is_stem(C, R, S, 1))
        return (size_t)planes * stem_kblocks(C, R, S) * stem_chunks_per_kb(C, R, S) * K * 4 * sizeof(float);
    return (size_t)planes * ceil16(C) * 16 * K * R * S * sizeof(float);
}

int pdl_conv2d_prepack_weights(const float *w, void *packed, int C, int K, int R, int S,
                               unsigned flags, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = device_check())) return rc;
    if ((rc = check_flags(flags, kConvFlags, "prepack"))) return rc;
    if (C <= 0 || K % 16 || K <= 0 || R <= 0 || S <= 0) return fail(PDL_EINVAL, "prepack: bad shape");
    if (!aligned16(w) || !aligned16(packed)) return fail(PDL_EALIGN, "prepack: unaligned pointer");
    const int split = (flags & PDL_MODE_MASK) == PDL_MODE_3XTF32;
    if (is_stem(C, R, S, 1)) {
        const int nch = stem_kblocks(C, R, S) * stem_chunks_per_kb(C, R, S);
        const long long plane = (long long)nch * K * 4;
        const int blocks = (int)std::min<long long>((plane + 255) / 256, 148LL * 16);
        pdl::prepack_stem_weights_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
            w, reinterpret_cast<float *>(packed), K, R, S, split, C, nch, stem_packed(C, R, S));
    } else {
        const long long total = (long long)K * ceil16(C) * 16 * R * S;
        const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
        pdl::prepack_weights_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
            w, reinterpret_cast<float *>(packed), ceil16(C), K / 16, R * S, split, C,
            weight_group(C));
    }
    ++g_launches;
    return check_launch("prepack_weights_kernel");
}

int pdl_conv2d_fwd_prepacked(const float *x, const void *packed_w, const float *bias, float *y,
                             int N, int C, int K, int H, int W, int R, int S, int stride, int pad,
                             unsigned flags, const pdl_tile_cfg *cfg, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = device_check())) return rc;
    if ((rc = check_flags(flags, kConvXFlags, "conv"))) return rc;
    if ((rc = conv_check(x, y, N, C, K, H, W, R, S, stride, pad))) return rc;
    if ((flags & (PDL_BIAS | PDL_SCALE)) && (!bias || !aligned16(bias)))
        return fail(PDL_EALIGN, "conv: PDL_BIAS / PDL_SCALE need a 16-byte aligned bias");
    if ((flags & PDL_MODE_MASK) == PDL_MODE_FP32)
        return fail(PDL_EUNSUPPORTED, "conv: PDL_MODE_FP32 takes raw weights (pdl_conv2d_fwd_nchw16c)");
    if (!aligned16(packed_w)) return fail(PDL_EALIGN, "conv: packed weights unaligned");
    return conv_fwd_tc(x, reinterpret_cast<const float *>(packed_w), bias, y, N, C, K, H, W, R, S,
                       stride, pad, flags, cfg, (cudaStream_t)stream);
}

size_t pdl_conv2d_splitk_workspace_bytes(int N, int C, int K, int H, int W, int R, int S, int stride,
                                         int pad, unsigned flags, const pdl_tile_cfg *cfg) {
    if ((flags & PDL_MODE_MASK) == PDL_MODE_FP32) return 0;
    size_t need = 0;
    if (conv_check(nullptr, nullptr, N, C, K, H, W, R, S, stride, pad)) return 0;
    if (conv_fwd_tc(nullptr, nullptr, nullptr, nullptr, N, C, K, H, W, R, S, stride, pad, flags, cfg,
                    nullptr, nullptr, 0, &need))
        return 0;
    return need;
}

int pdl_conv2d_fwd_prepacked_ws(const float *x, const void *packed_w, const float *bias, float *y,
                                int N, int C, int K, int H, int W, int R, int S, int stride, int pad,
                                unsigned flags, const pdl_tile_cfg *cfg, void *workspace,
                                size_t ws_bytes, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = device_check())) return rc;
    if ((rc = check_flags(flags, kConvXFlags, "conv"))) return rc;
    if ((rc = conv_check(x, y, N, C, K, H, W, R, S, stride, pad))) return rc;
    if ((flags & (PDL_BIAS | PDL_SCALE)) && (!bias || !aligned16(bias)))
        return fail(PDL_EALIGN, "conv: PDL_BIAS / PDL_SCALE need a 16-byte aligned bias");
    if ((flags & PDL_MODE_MASK) == PDL_MODE_FP32)
        return fail(PDL_EUNSUPPORTED, "conv: PDL_MODE_FP32 takes raw weights (pdl_conv2d_fwd_nchw16c)");
    if (!aligned16(packed_w)) return fail(PDL_EALIGN, "conv: packed weights unaligned");
    return conv_fwd_tc(x, reinterpret_cast<const float *>(packed_w), bias, y, N, C, K, H, W, R, S,
                       stride, pad, flags, cfg, (cudaStream_t)stream, workspace, ws_bytes);
}

int pdl_conv2d_schedule(int N, int C, int K, int H, int W, int R, int S, int stride, int pad,
                        unsigned flags, const pdl_tile_cfg *cfg, int with_workspace, pdl_schedule *out) {
    int rc;
    if (!out) return fail(PDL_EINVAL, "schedule: null output");
    if ((rc = check_flags(flags, kConvXFlags, "schedule"))) return rc;
    if ((rc = conv_check(nullptr, nullptr, N, C, K, H, W, R, S, stride, pad))) return rc;
    // a non-null stand-in workspace: auto split-K may engage
    static char ws_token;
    return conv_fwd_tc(nullptr, nullptr, nullptr, nullptr, N, C, K, H, W, R, S, stride, pad, flags, cfg,
                       nullptr, with_workspace ? &ws_token : nullptr, 0, nullptr, out);
}

size_t pdl_conv2d_host_workspace_bytes(int N, int C, int K, int H, int W, int R, int S, int stride,
                                       int pad, int chunk) {
    if (N <= 0 || C <= 0 || K <= 0 || H <= 0 || W <= 0 || stride <= 0) return 0;
    const int P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
    if (P <= 0 || Q <= 0) return 0;
    const size_t x_img = (size_t)ceil16(C) * H * W * 64, y_img = (size_t)(K / 16) * P * Q * 64;
    const int c = chunk > 0 ? std::min(chunk, N) : host_chunk(N, x_img);
    // [x area | y area 0 | y area 1], equal thirds: copies in only write the x area (3 chunk
    // slots), a y area holds the call's whole output (the convolutions never wait for copies
    // out), and consecutive calls alternate y areas, so a call's H2D and convolutions never
    // wait for the previous call's D2H
    return 3 * align256(std::max((size_t)kHostSlots * align256(c * x_img), (size_t)N * y_img));
}

int pdl_conv2d_fwd_host(const float *x_host, const void *packed_w, const float *bias,
                        float *y_host, int N, int C, int K, int H, int W, int R, int S,
                        int stride, int pad, unsigned flags, const pdl_tile_cfg *cfg, int chunk,
                        void *workspace, size_t ws_bytes, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = device_check())) return rc;
    if ((rc = check_flags(flags, kConvXFlags | PDL_HOST_X_READY, "conv host"))) return rc;
    if (!x_host || !y_host) return fail(PDL_EINVAL, "conv host: null host buffer");
    if (chunk < 0) return fail(PDL_EINVAL, "conv host: negative chunk");
    if ((flags & PDL_MODE_MASK) == PDL_MODE_FP32)
        return fail(PDL_EUNSUPPORTED, "conv host: PDL_MODE_FP32 takes raw weights (pdl_conv2d_fwd_nchw16c)");
    if ((flags & (PDL_BIAS | PDL_SCALE)) && (!bias || !aligned16(bias)))
        return fail(PDL_EALIGN, "conv: PDL_BIAS / PDL_SCALE need a 16-byte aligned bias");
    if (!aligned16(packed_w) || !aligned16(workspace))
        return fail(PDL_EALIGN, "conv host: packed weights / workspace unaligned");
    // shape checks before anything is enqueued (workspace stands in for x / y)
    if ((rc = conv_check((const float *)workspace, (const float *)workspace, N, C, K, H, W, R, S,
                         stride, pad)))
        return rc;
    const size_t need = pdl_conv2d_host_workspace_bytes(N, C, K, H, W, R, S, stride, pad, chunk);
    if (!workspace || ws_bytes < need)
        return fail(PDL_EWORKSPACE, "conv host: workspace of %zu bytes required", need);
    std::lock_guard<std::mutex> lock(g_pipe_mu);
    HostPipe *hp;
    if ((rc = host_pipe(workspace, &hp))) return rc;
    const int P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
    if ((flags & PDL_X_NCHW4C) && !is_stem(C, R, S, stride))
        return fail(PDL_EUNSUPPORTED, "conv host: PDL_X_NCHW4C needs the narrow-channel path (C <= 4)");
    // x_host is nChw16c, or [N][H][W][4] with PDL_X_NCHW4C (a quarter of the H2D bytes)
    const size_t x_img = (flags & PDL_X_NCHW4C) ? (size_t)H * W * 16 : (size_t)ceil16(C) * H * W * 64;
    const size_t y_img = (size_t)(K / 16) * P * Q * 64;
    uint8_t *ws = reinterpret_cast<uint8_t *>(workspace);
    const size_t third = ws_bytes / 3 & ~(size_t)255;
    int c = chunk > 0 ? std::min(chunk, N) : host_chunk(N, x_img);
    // (the workspace was sized for nChw16c chunks: the compact layout's larger automatic
    // chunks must still fit the three x slots)
    c = (int)std::max<size_t>(1, std::min<size_t>(c, third / kHostSlots / x_img));
    const size_t xs = align256(c * x_img);
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned cflags = flags & ~(unsigned)PDL_HOST_X_READY;
    // Three internal streams; chunk i uses x slot i % kHostSlots and its own images' place
    // in this call's y area q (the whole output):
    //   h2d: [slot's previous conv done] copy x  -> x_in
    //   cs : [x_in] conv -> done
    //   d2h: [done] copy y;  after the last chunk -> y_done[q]
    // Default: everything is ordered after prior work on `stream` (entry event).  With
    // PDL_HOST_X_READY (x_host, packed_w and bias are final at call time, and y_host is
    // not read by work still pending on `stream`) and a previous call on this workspace,
    // the copies in only wait for that call's last convolution to release the x area and
    // the convolutions only for their own y area (the previous call used the other one),
    // so the previous call's copies out overlap this call's copies in AND convolutions:
    // both PCIe directions stay busy across layers.  `stream` waits for this call's
    // copies out before any later work.
    if (cudaEventRecord(hp->entry, st) != cudaSuccess)
        return fail(PDL_ELAUNCH, "conv host: entry event");
    const bool relaxed = (flags & PDL_HOST_X_READY) && hp->used && hp->last_ws_bytes == ws_bytes;
    if (!relaxed) hp->parity = 0;
    const int q = hp->parity;
    uint8_t *ws_y = ws + (size_t)(1 + q) * third;
    // A failure after work was enqueued: join what was enqueued into `stream` (later work
    // on it, and a later call on this workspace, stay ordered after it) and forget the
    // relaxed-ordering state.
    auto abort_call = [&](int code) {
        cudaEventRecord(hp->x_free, hp->cs);
        cudaEventRecord(hp->y_done[q], hp->d2h);
        cudaStreamWaitEvent(st, hp->x_free, 0);
        cudaStreamWaitEvent(st, hp->y_done[q], 0);
        cudaEventRecord(hp->y_done[q ^ 1], hp->d2h);
        hp->used = false;
        return code;
    };
    if (cudaStreamWaitEvent(hp->h2d, relaxed ? hp->x_free : hp->entry, 0) != cudaSuccess ||
        (!relaxed && cudaStreamWaitEvent(hp->cs, hp->entry, 0) != cudaSuccess))
        return abort_call(fail(PDL_ELAUNCH, "conv host: entry wait"));
    // this y area's previous user (two calls back) must have copied all of it out
    if (cudaStreamWaitEvent(hp->cs, hp->y_done[q], 0) != cudaSuccess)
        return abort_call(fail(PDL_ELAUNCH, "conv host: y area wait"));
    const int nchunks = (N + c - 1) / c;
    int launches = 0;
    for (int i = 0; i < nchunks; ++i) {
        const int b = i % kHostSlots;
        const int n0 = i * c, n = std::min(c, N - n0);
        float *xd = reinterpret_cast<float *>(ws + b * xs);
        float *yd = reinterpret_cast<float *>(ws_y + n0 * y_img);
        if (i >= kHostSlots && cudaStreamWaitEvent(hp->h2d, hp->done[b], 0) != cudaSuccess)
            return abort_call(fail(PDL_ELAUNCH, "conv host: wait"));
        if (cudaMemcpyAsync(xd, reinterpret_cast<const uint8_t *>(x_host) + n0 * x_img, n * x_img,
                            cudaMemcpyHostToDevice, hp->h2d) != cudaSuccess ||
            cudaEventRecord(hp->x_in[b], hp->h2d) != cudaSuccess)
            return abort_call(fail(PDL_ELAUNCH, "conv host: H2D copy: %s", cudaGetErrorString(cudaGetLastError())));
        if (cudaStreamWaitEvent(hp->cs, hp->x_in[b], 0) != cudaSuccess)
            return abort_call(fail(PDL_ELAUNCH, "conv host: wait"));
        if ((rc = conv_fwd_tc(xd, reinterpret_cast<const float *>(packed_w), bias, yd, n, C, K, H, W,
                              R, S, stride, pad, cflags, cfg, hp->cs)))
            return abort_call(rc);
        launches += g_launches;
        if (cudaEventRecord(hp->done[b], hp->cs) != cudaSuccess ||
            cudaStreamWaitEvent(hp->d2h, hp->done[b], 0) != cudaSuccess ||
            cudaMemcpyAsync(reinterpret_cast<uint8_t *>(y_host) + n0 * y_img, yd, n * y_img,
                            cudaMemcpyDeviceToHost, hp->d2h) != cudaSuccess)
            return abort_call(fail(PDL_ELAUNCH, "conv host: D2H copy: %s", cudaGetErrorString(cudaGetLastError())));
    }
    // the x area is free once the last convolution has run (next call's copies in)
    if (cudaEventRecord(hp->x_free, hp->cs) != cudaSuccess)
        return abort_call(fail(PDL_ELAUNCH, "conv host: x_free"));
    // later work on `stream` sees every y copy (and so every convolution) done
    if (cudaEventRecord(hp->y_done[q], hp->d2h) != cudaSuccess ||
        cudaStreamWaitEvent(st, hp->y_done[q], 0) != cudaSuccess)
        return abort_call(fail(PDL_ELAUNCH, "conv host: exit wait"));
    hp->used = true;
    hp->last_ws_bytes = ws_bytes;
    hp->parity = q ^ 1;
    g_launches = launches;
    return PDL_OK;
}

int pdl_conv2d_fwd_nchw16c(const float *x, const float *w, const float *bias, float *y, int N,
                           int C, int K, int H, int W, int R, int S, int stride, int pad,
                           unsigned flags, const pdl_tile_cfg *cfg, void *workspace,
                           size_t ws_bytes, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = device_check())) return rc;
    if ((rc = check_flags(flags, kConvXFlags, "conv"))) return rc;
    if ((rc = conv_check(x, y, N, C, K, H, W, R, S, stride, pad))) return rc;
    if ((flags & (PDL_BIAS | PDL_SCALE)) && (!bias || !aligned16(bias)))
        return fail(PDL_EALIGN, "conv: PDL_BIAS / PDL_SCALE need a 16-byte aligned bias");
    cudaStream_t st = (cudaStream_t)stream;
    if ((flags & PDL_MODE_MASK) == PDL_MODE_FP32) {
        if (flags & PDL_X_NCHW4C)
            return fail(PDL_EUNSUPPORTED, "conv: PDL_MODE_FP32 reads nChw16c (no PDL_X_NCHW4C)");
        const int P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
        const long long total = (long long)N * (K / 16) * P * Q;
        pdl::simt_conv_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(
            x, w, bias, y, N, ceil16(C), K / 16, H, W, R, S, stride, pad, P, Q, flags, C);
        ++g_launches;
        return check_launch("simt_conv_kernel");
    }
    // workspace = [prepacked weights][split-K area, when the plan splits]
    const size_t packed = pdl_conv2d_packed_bytes(C, K, R, S, flags);
    if (!workspace || ws_bytes < packed)
        return fail(PDL_EWORKSPACE, "conv: workspace of %zu bytes required", packed);
    const unsigned wflags = flags & ~(unsigned)PDL_X_NCHW4C;  // the weight image does not depend on x's layout
    const size_t off = align256(packed);
    void *split_ws = ws_bytes > off ? reinterpret_cast<uint8_t *>(workspace) + off : nullptr;
    const size_t split_bytes = ws_bytes > off ? ws_bytes - off : 0;
    if ((rc = pdl_conv2d_prepack_weights(w, workspace, C, K, R, S, wflags, stream))) return rc;
    rc = conv_fwd_tc(x, reinterpret_cast<const float *>(workspace), bias, y, N, C, K, H, W, R, S,
                     stride, pad, flags, cfg, st, split_ws, split_bytes);
    if (rc == PDL_OK) g_launches = 2;
    return rc;
}

int pdl_gemm_f32_epilogue(const float *A, const float *B, float *C, const float *bias, int M, int N, int K,
                          int lda, int ldb, int ldc, float alpha, float beta, unsigned flags,
                          const pdl_tile_cfg *cfg_in, void *workspace, size_t ws_bytes, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = device_check())) return rc;
    if ((rc = check_flags(flags, kGemmFlags, "gemm"))) return rc;
    if (M < 0 || N < 0 || K < 0) return fail(PDL_EINVAL, "gemm: negative dimension");
    if (lda < std::max(K, 1) || ldb < std::max(N, 1) || ldc < std::max(N, 1))
        return fail(PDL_EINVAL, "gemm: leading dimension too small");
    if ((flags & (PDL_BIAS | PDL_SCALE)) && (!bias || !aligned16(bias)))
        return fail(PDL_EALIGN, "gemm: PDL_BIAS / PDL_SCALE need a 16-byte aligned bias[N] (shift[N] | scale[N])");
    if (M == 0 || N == 0) return PDL_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned mode = flags & PDL_MODE_MASK;
    const unsigned eflags = flags & (kEpiFlags | kDiag);
    const float *ebias = (flags & (PDL_BIAS | PDL_SCALE)) ? bias : nullptr;
    // TMA describes the operands only with 16-byte aligned bases and row strides
    const bool tma_ok = K > 0 && aligned16(A) && aligned16(B) && aligned16(C) && lda % 4 == 0 &&
                        ldb % 4 == 0 && ldc % 4 == 0 && N % 4 == 0;
    if (mode != PDL_MODE_FP32 && !tma_ok && (flags & PDL_NO_SIMT))
        return fail(PDL_EUNSUPPORTED, "gemm: tensor-core path needs K > 0, 16-byte aligned A/B/C and "
                    "N, lda, ldb, ldc multiples of 4 (PDL_NO_SIMT forbids the CUDA-core path)");
    if (mode == PDL_MODE_FP32 || !tma_ok) {
        dim3 grid((N + 63) / 64, (M + 63) / 64);
        pdl::simt_gemm_kernel<<<grid, 256, 0, st>>>(A, B, C, M, N, K, lda, ldb, ldc, alpha, beta, ebias,
                                                    eflags);
        ++g_launches;
        return check_launch("simt_gemm_kernel");
    }
    if ((rc = get_encode())) return rc;
    int bn, cl, raster;
    gemm_cfg(M, N, cfg_in, &bn, &cl, &raster);
    const bool epix = flags & (PDL_RELU6 | PDL_SCALE);  // extended-epilogue instances are cluster 1
    if (epix) cl = 1;
    if (cl != 1 && cl != 2 && cl != 4) return fail(PDL_EINVAL, "gemm: cluster_m must be 1, 2 or 4");
    pdl::TmaMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    {
        const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
        const cuuint64_t str[1] = {(cuuint64_t)lda * 4};
        const cuuint32_t box[2] = {32, 128};
        if ((rc = encode(&maps.a[0], A, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B, "gemm A"))) return rc;
    }
    {
        const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
        const cuuint64_t str[1] = {(cuuint64_t)ldb * 4};
        const cuuint32_t box[2] = {32, 32};
        if ((rc = encode(&maps.b, B, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, "gemm B"))) return rc;
    }
    pdl::TileParams p{};
    p.num_kb = (K + 31) / 32;
    p.seg_kb = kSegElems / 32;
    p.n_out = N;
    p.flags = eflags;
    p.bias = ebias;
    p.out = C;
    p.M = M;
    p.ldc = ldc;
    p.alpha = alpha;
    p.beta = beta;
    p.raster = cl == 1 ? (raster & 1) : 0;
    p.m_tiles = (M + 127) / 128;
    p.n_tiles = (N + bn - 1) / bn;
    {
        const int req = cfg_in ? cfg_in->split_k : 0;
        const SplitPlan spl = plan_split(p.m_tiles, p.n_tiles, cl, bn, p.num_kb, p.seg_kb,
                                         workspace ? req : (req > 1 ? req : 1));
        if ((rc = bind_split(p, spl, workspace, ws_bytes, cl))) return rc;
    }
    if (epix)
        return mode == PDL_MODE_3XTF32 ? dispatch_epix<pdl::KIND_GEMM, true>(bn, 1, maps, p, st)
                                       : dispatch_epix<pdl::KIND_GEMM, false>(bn, 1, maps, p, st);
    if (mode == PDL_MODE_3XTF32) return dispatch_tile<pdl::KIND_GEMM, true>(bn, 1, cl, maps, p, st);
    return dispatch_tile<pdl::KIND_GEMM, false>(bn, 1, cl, maps, p, st);
}

int pdl_gemm_schedule(int M, int N, int K, unsigned flags, const pdl_tile_cfg *cfg_in, int with_workspace,
                      pdl_schedule *out) {
    int rc;
    if (!out) return fail(PDL_EINVAL, "schedule: null output");
    if ((rc = check_flags(flags, kGemmFlags, "schedule"))) return rc;
    if (M <= 0 || N <= 0 || K <= 0) return fail(PDL_EINVAL, "schedule: non-positive GEMM dimension");
    int bn, cl, raster;
    gemm_cfg(M, N, cfg_in, &bn, &cl, &raster);
    if (flags & (PDL_RELU6 | PDL_SCALE)) cl = 1;
    std::memset(out, 0, sizeof(*out));
    out->kind = 3;
    out->bn = bn;
    out->bk = 32;
    out->cluster = cl;
    out->tile_w = 128;
    out->tile_h = out->tile_images = 1;
    out->m_tiles = (M + 127) / 128;
    out->n_tiles = (N + bn - 1) / bn;
    out->num_kb = (K + 31) / 32;
    const int req = cfg_in ? cfg_in->split_k : 0;
    const SplitPlan spl = plan_split(out->m_tiles, out->n_tiles, cl, bn, out->num_kb, kSegElems / 32,
                                     with_workspace ? req : (req > 1 ? req : 1));
    out->split = spl.split;
    out->kb_per = spl.kb_per;
    out->order = cl == 1 ? (raster & 1) : 0;
    out->flat = 1;
    out->splitk_workspace_bytes = spl.bytes;
    return PDL_OK;
}

int pdl_gemm_f32(const float *A, const float *B, float *C, int M, int N, int K, int lda, int ldb,
                 int ldc, float alpha, float beta, unsigned flags, const pdl_tile_cfg *cfg_in,
                 void *workspace, size_t ws_bytes, void *stream) {
    if (flags & (PDL_BIAS | PDL_SCALE)) {
        g_launches = 0;
        return fail(PDL_EINVAL, "gemm: PDL_BIAS / PDL_SCALE take a bias vector: use pdl_gemm_f32_epilogue");
    }
    return pdl_gemm_f32_epilogue(A, B, C, nullptr, M, N, K, lda, ldb, ldc, alpha, beta, flags, cfg_in,
                                 workspace, ws_bytes, stream);
}

int pdl_bias_relu_nchw16c(float *y, const float *bias, int N, int K, int P, int Q, unsigned flags,
                          void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = device_check())) return rc;
    if ((rc = check_flags(flags, kConvFlags, "bias_relu"))) return rc;
    if (K % 16 || N < 0 || P < 0 || Q < 0) return fail(PDL_EINVAL, "bias_relu: bad shape");
    if (!aligned16(y) || ((flags & (PDL_BIAS | PDL_SCALE)) && (!bias || !aligned16(bias))))
        return fail(PDL_EALIGN, "bias_relu: unaligned pointer");
    const long long n4 = (long long)N * K * P * Q / 4;
    if (n4 == 0) return PDL_OK;
    const int blocks = (int)std::min<long long>((n4 + 255) / 256, 148LL * 8);
    pdl::bias_relu_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<float4 *>(y), bias, n4, P * Q, K / 16, flags);
    ++g_launches;
    return check_launch("bias_relu_kernel");
}

int pdl_accumulate_epilogue_nchw16c(float *y, const float *y0, const float *bias, int N, int K, int P,
                                    int Q, unsigned flags, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = device_check())) return rc;
    if ((rc = check_flags(flags, kConvFlags, "accumulate"))) return rc;
    if (K % 16 || N < 0 || P < 0 || Q < 0) return fail(PDL_EINVAL, "accumulate: bad shape");
    if (!y0) return fail(PDL_EINVAL, "accumulate: null addend");
    if (!aligned16(y) || !aligned16(y0) || ((flags & (PDL_BIAS | PDL_SCALE)) && (!bias || !aligned16(bias))))
        return fail(PDL_EALIGN, "accumulate: unaligned pointer");
    const long long n4 = (long long)N * K * P * Q / 4;
    if (n4 == 0) return PDL_OK;
    const int blocks = (int)std::min<long long>((n4 + 255) / 256, 148LL * 8);
    pdl::accumulate_epilogue_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<float4 *>(y), reinterpret_cast<const float4 *>(y0), bias, n4, P * Q, K / 16, flags);
    ++g_launches;
    return check_launch("accumulate_epilogue_kernel");
}

static int layout_check(const void *a, const void *b, long long n) {
    int rc;
    if ((rc = device_check())) return rc;
    if (n < 0) return fail(PDL_EINVAL, "layout: negative dimension");
    if (!a || !b) return fail(PDL_EINVAL, "layout: null pointer");
    return PDL_OK;
}

int pdl_pack_nchw16c(const float *src, float *dst, int N, int C, int H, int W, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = layout_check(src, dst, (long long)N | C | H | W))) return rc;
    if (N <= 0 || C <= 0 || H <= 0 || W <= 0) return fail(PDL_EINVAL, "pack: empty tensor");
    if (!aligned16(dst)) return fail(PDL_EALIGN, "pack: dst must be 16-byte aligned");
    const long long planes = (long long)N * ceil16(C), hw = (long long)H * W;
    if (planes > 65535 || (hw + 255) / 256 > 0x7fffffffLL)
        return fail(PDL_EUNSUPPORTED, "pack: tensor too large");
    const dim3 grid((unsigned)((hw + pdl::kLayoutThreads - 1) / pdl::kLayoutThreads), (unsigned)planes);
    pdl::pack_nchw16c_kernel<<<grid, pdl::kLayoutThreads, 0, (cudaStream_t)stream>>>(src, dst, N, C, H, W);
    ++g_launches;
    return check_launch("pack_nchw16c_kernel");
}

int pdl_pack_nchw4c(const float *src, float *dst, int N, int C, int H, int W, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = layout_check(src, dst, (long long)N | C | H | W))) return rc;
    if (N <= 0 || C <= 0 || H <= 0 || W <= 0) return fail(PDL_EINVAL, "pack: empty tensor");
    if (C > 4) return fail(PDL_EINVAL, "pack_nchw4c: C must be <= 4 (got %d)", C);
    if (!aligned16(dst)) return fail(PDL_EALIGN, "pack: dst must be 16-byte aligned");
    const long long hw = (long long)H * W;
    if (N > 65535 || (hw + 255) / 256 > 0x7fffffffLL) return fail(PDL_EUNSUPPORTED, "pack: tensor too large");
    const dim3 grid((unsigned)((hw + pdl::kLayoutThreads - 1) / pdl::kLayoutThreads), (unsigned)N);
    pdl::pack_nchw4c_kernel<<<grid, pdl::kLayoutThreads, 0, (cudaStream_t)stream>>>(
        src, reinterpret_cast<float4 *>(dst), N, C, H, W);
    ++g_launches;
    return check_launch("pack_nchw4c_kernel");
}

int pdl_unpack_nchw16c(const float *src, float *dst, int N, int C, int H, int W, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = layout_check(src, dst, (long long)N | C | H | W))) return rc;
    if (N <= 0 || C <= 0 || H <= 0 || W <= 0) return fail(PDL_EINVAL, "unpack: empty tensor");
    if (!aligned16(src)) return fail(PDL_EALIGN, "unpack: src must be 16-byte aligned");
    const long long planes = (long long)N * ceil16(C), hw = (long long)H * W;
    if (planes > 65535 || (hw + 255) / 256 > 0x7fffffffLL)
        return fail(PDL_EUNSUPPORTED, "unpack: tensor too large");
    const dim3 grid((unsigned)((hw + pdl::kLayoutThreads - 1) / pdl::kLayoutThreads), (unsigned)planes);
    pdl::unpack_nchw16c_kernel<<<grid, pdl::kLayoutThreads, 0, (cudaStream_t)stream>>>(src, dst, N, C, H, W);
    ++g_launches;
    return check_launch("unpack_nchw16c_kernel");
}

int pdl_pack_kcrs16c16k(const float *src, float *dst, int K, int C, int R, int S, void *stream) {
    g_launches = 0;
    int rc;
    if ((rc = layout_check(src, dst, (long long)K | C | R | S))) return rc;
    if (K <= 0 || K % 16 || C <= 0 || R <= 0 || S <= 0)
        return fail(PDL_EINVAL, "pack weights: K must be a positive multiple of 16");
    const long long total = (long long)K * ceil16(C) * 16 * R * S;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    pdl::pack_kcrs16c16k_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(src, dst, K, C, R, S);
    ++g_launches;
    return check_launch("pack_kcrs16c16k_kernel");
}

size_t pdl_workspace_bytes(int op, const int *dims, const pdl_tile_cfg *cfg) {
    (void)cfg;
    if (op == PDL_OP_CONV2D && dims) {
        // dims = {N, C, K, H, W, R, S, stride, pad, flags}: prepacked weights + split-K area
        const size_t split = pdl_conv2d_splitk_workspace_bytes(dims[0], dims[1], dims[2], dims[3], dims[4],
                                                               dims[5], dims[6], dims[7], dims[8],
                                                               (unsigned)dims[9], cfg);
        const size_t packed = pdl_conv2d_packed_bytes(dims[1], dims[2], dims[5], dims[6], (unsigned)dims[9]);
        return split ? align256(packed) + split : packed;
    }
    if (op == PDL_OP_GEMM && dims) {
        // dims = {M, N, K, flags}: split-K area (0 when the GEMM fills the GPU)
        return gemm_split_bytes(dims[0], dims[1], dims[2], (unsigned)dims[3], cfg);
    }
    return 0;
}

int pdl_default_cfg(int op, const int *dims, pdl_tile_cfg *cfg) {
    if (!cfg || !dims) return fail(PDL_EINVAL, "default_cfg: null argument");
    if (op == PDL_OP_CONV2D) {
        // dims = {N, C, K, H, W, R, S, stride, pad, flags}
        if (dims[0] <= 0 || dims[3] <= 0 || dims[4] <= 0 || (dims[7] != 1 && dims[7] != 2) ||
            dims[3] + 2 * dims[8] < dims[5] || dims[4] + 2 * dims[8] < dims[6])
            conv_default_cfg(dims[1], dims[2], dims[5], dims[6], cfg, (unsigned)dims[9]);
        else
            conv_auto_cfg(dims[0], dims[1], dims[2], dims[3], dims[4], dims[5], dims[6], dims[7], dims[8],
                          (unsigned)dims[9], nullptr, cfg);
        return PDL_OK;
    }
    if (op == PDL_OP_GEMM) {
        // dims = {M, N, K}
        int bn, cl, raster;
        gemm_cfg(dims[0], dims[1], nullptr, &bn, &cl, &raster);
        cfg->bm = 128;
        cfg->bn = bn;
        cfg->bk = 32;
        cfg->stages = 0;
        cfg->cluster_m = cl;
        cfg->cluster_n = cfg->split_k = 1;
        cfg->raster = 0;
        return PDL_OK;
    }
    return fail(PDL_EINVAL, "default_cfg: unknown op %d", op);
}

}  // extern "C"
