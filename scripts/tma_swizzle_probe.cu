// tma_swizzle_probe.cu -- does a SWIZZLE_64B TMA box written at a smem offset that
// is 128-byte but not 512-byte aligned land in the layout defined by the ABSOLUTE
// smem address bits (16-byte chunk j of a 64-byte row at address A goes to chunk
// j ^ ((A >> 7) & 3))?  If so, an M tile can be assembled from several row boxes
// (e.g. 9 rows of 14 pixels spanning two images) in the canonical SW64 layout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/tma_swizzle_probe.cu -o scripts/tma_swizzle_probe.bin
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2006_02230_b200/csrc/pdl_sm100.cuh"

using namespace pdl;

__global__ void probe(const __grid_constant__ CUtensorMap m, int dst_off, float *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 16384);
    float *f = reinterpret_cast<float *>(smem);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) f[i] = -1.f;
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(bar, 14 * 64);
        tma_load_2d(smem + dst_off, &m, bar, 0, 0);
        mbar_wait(bar, 0);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = f[i];
}

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    // global: 14 rows x 16 floats, value = row * 16 + col
    std::vector<float> h(14 * 16);
    for (int i = 0; i < 14 * 16; ++i) h[i] = (float)i;
    float *g, *out;
    cudaMalloc(&g, h.size() * 4);
    cudaMemcpy(g, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 4096 * 4);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
    CUtensorMap m;
    const cuuint64_t dims[2] = {16, 14};
    const cuuint64_t str[1] = {64};
    const cuuint32_t box[2] = {16, 14}, es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", (int)r); return 1; }
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 2048);
    for (int off : {0, 128, 512, 896, 2688, 448, 64, 192}) {
        probe<<<1, 128, 16384 + 2048>>>(m, off, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("off %4d: %s\n", off, cudaGetErrorString(e)); return 0; }
        std::vector<float> o(4096);
        cudaMemcpy(o.data(), out, 4096 * 4, cudaMemcpyDeviceToHost);
        int abs_ok = 1, rel_ok = 1;
        for (int row = 0; row < 14; ++row)
            for (int j = 0; j < 4; ++j) {
                const int A = off + row * 64;                 // byte address of the row
                const int ja = j ^ ((A >> 7) & 3);            // absolute-address swizzle
                const int jr = j ^ (((row * 64) >> 7) & 3);   // swizzle relative to the box start
                for (int k = 0; k < 4; ++k) {
                    const float want = (float)(row * 16 + j * 4 + k);
                    if (o[(A + ja * 16) / 4 + k] != want) abs_ok = 0;
                    if (o[(off + row * 64 + jr * 16) / 4 + k] != want) rel_ok = 0;
                }
            }
        printf("off %4d: absolute-address swizzle %s, box-relative swizzle %s\n", off, abs_ok ? "MATCH" : "no",
               rel_ok ? "MATCH" : "no");
    }
    return 0;
}
