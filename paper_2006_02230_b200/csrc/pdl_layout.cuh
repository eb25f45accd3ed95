// Layout conversion kernels: the data path on either side of the conv
// (SURVEY 8(f)4).  PyTorch-native NCHW / OIHW <-> the reference nest's blocked
// nChw16c / KCRS16c16k (PAPER.md:740-763 array declarations).  HBM-bound
// transposes of a [16][H*W] channel slab into [H*W][16].
#pragma once
#include <cuda_runtime.h>

namespace pdl {

// One thread per pixel of one (image, 16-channel block) plane: 16 channel
// loads, each coalesced across the warp (consecutive pixels), and 4 float4
// stores of the pixel's 64-byte group (the warp covers 2 KB contiguous) --
// no shared memory, 16 independent loads in flight per thread.
constexpr int kLayoutThreads = 256;

// src NCHW [N][C][H][W] -> dst nChw16c [N][ceil(C/16)][H][W][16], channels >= C zero
__global__ void __launch_bounds__(kLayoutThreads) pack_nchw16c_kernel(const float *__restrict__ src,
                                                                      float *__restrict__ dst, int N,
                                                                      int C, int H, int W) {
    const long long hw = (long long)H * W;
    const int CB = (C + 15) / 16;
    const long long pix = (long long)blockIdx.x * kLayoutThreads + threadIdx.x;
    const int cb = blockIdx.y % CB;
    const int n = blockIdx.y / CB;
    if (pix >= hw) return;
    const float *in = src + ((size_t)n * C + cb * 16) * hw + pix;
    float v[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] = (cb * 16 + c < C) ? __ldg(in + (size_t)c * hw) : 0.f;
    float4 *out = reinterpret_cast<float4 *>(dst + (((size_t)n * CB + cb) * hw + pix) * 16);
#pragma unroll
    for (int j = 0; j < 4; ++j) out[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}

// src NCHW [N][C][H][W] (C <= 4) -> dst [N][H][W][4] (nChw4c, one channel block),
// channels >= C zero: the compact input of the narrow-channel conv (PDL_X_NCHW4C).
// One thread per pixel: C coalesced loads, one float4 store.
__global__ void __launch_bounds__(kLayoutThreads) pack_nchw4c_kernel(const float *__restrict__ src,
                                                                     float4 *__restrict__ dst, int N,
                                                                     int C, int H, int W) {
    const long long hw = (long long)H * W;
    const long long pix = (long long)blockIdx.x * kLayoutThreads + threadIdx.x;
    const int n = blockIdx.y;
    if (pix >= hw) return;
    const float *in = src + (size_t)n * C * hw + pix;
    float v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = c < C ? __ldg(in + (size_t)c * hw) : 0.f;
    dst[(size_t)n * hw + pix] = make_float4(v[0], v[1], v[2], v[3]);
}

// src nChw16c [N][ceil(C/16)][H][W][16] -> dst NCHW [N][C][H][W] (padding channels dropped)
__global__ void __launch_bounds__(kLayoutThreads) unpack_nchw16c_kernel(const float *__restrict__ src,
                                                                        float *__restrict__ dst, int N,
                                                                        int C, int H, int W) {
    const long long hw = (long long)H * W;
    const int CB = (C + 15) / 16;
    const long long pix = (long long)blockIdx.x * kLayoutThreads + threadIdx.x;
    const int cb = blockIdx.y % CB;
    const int n = blockIdx.y / CB;
    if (pix >= hw) return;
    const float4 *in = reinterpret_cast<const float4 *>(src + (((size_t)n * CB + cb) * hw + pix) * 16);
    float v[16];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float4 t = __ldg(in + j);
        v[4 * j] = t.x; v[4 * j + 1] = t.y; v[4 * j + 2] = t.z; v[4 * j + 3] = t.w;
    }
    float *out = dst + ((size_t)n * C + cb * 16) * hw + pix;
#pragma unroll
    for (int c = 0; c < 16; ++c)
        if (cb * 16 + c < C) out[(size_t)c * hw] = v[c];
}

// OIHW [K][C][R][S] -> KCRS16c16k [K/16][ceil(C/16)][R][S][16c][16k], channels >= C zero
__global__ void pack_kcrs16c16k_kernel(const float *__restrict__ src, float *__restrict__ dst, int K,
                                       int C, int R, int S) {
    const int CB = (C + 15) / 16;
    const long long total = (long long)K * CB * 16 * R * S;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int k16 = (int)(i & 15);
        long long t = i >> 4;
        const int c16 = (int)(t & 15);
        t >>= 4;
        const int s = (int)(t % S);
        t /= S;
        const int r = (int)(t % R);
        t /= R;
        const int cb = (int)(t % CB);
        const int kb = (int)(t / CB);
        const int k = kb * 16 + k16, c = cb * 16 + c16;
        dst[i] = c < C ? __ldg(src + (((size_t)k * C + c) * R + r) * S + s) : 0.f;
    }
}

}  // namespace pdl
