// tma_store_probe.cu -- throughput of TMA box STORES from shared memory, the output
// path of the conv epilogue.  148 CTAs each store NB boxes of 8 KB (16 channels x
// 128 pixels, 64-byte rows, SWIZZLE_64B, like one 16-channel block of a 1x1 conv tile)
// to distinct places of a [N][KT][HW][16] fp32 tensor, keeping DEPTH stores in flight
// (cp.async.bulk.wait_group.read DEPTH-1 before reusing a buffer), issued by one
// thread or round-robin by two threads (two bulk-group queues).  Reports cycles per
// 8 KB store (max CTA) and the aggregate write bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/tma_store_probe.cu -o scripts/tma_store_probe.bin
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2006_02230_b200/csrc/pdl_sm100.cuh"

using namespace pdl;
constexpr int N = 256, KT = 16, HW = 3136, NB = 600;

template <int DEPTH, int ISSUERS, int BOX_KT>
__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap m, unsigned long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < DEPTH * ISSUERS * 2048 * BOX_KT; i += blockDim.x)
        reinterpret_cast<float *>(smem)[i] = 1.f;
    fence_proxy_async_smem();
    __syncthreads();
    const unsigned long long t0 = clock64();
    const int who = threadIdx.x / 32;
    if ((threadIdx.x & 31) == 0 && who < ISSUERS) {
        for (int i = who; i < NB / BOX_KT; i += ISSUERS) {
            const int box = blockIdx.x * (NB / BOX_KT) + i;      // distinct boxes per CTA
            const int px_tiles = HW / 128;                       // 24 full 128-px tiles per image block
            const int kt = (box * BOX_KT) % KT, rest = box * BOX_KT / KT;
            const int pt = rest % px_tiles, img = (rest / px_tiles) % N;
            const int slot = (i / ISSUERS) % DEPTH;
            if (i / ISSUERS >= DEPTH) bulk_wait_read<DEPTH - 1>();
            tma_store_5d(&m, smem_u32(smem + (who * DEPTH + slot) * 8192 * BOX_KT), 0, pt * 128, 0, kt, img);
            bulk_commit();
        }
        bulk_wait<0>();
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int DEPTH, int ISSUERS, int BOX_KT>
void run(EncodeFn enc, float *y, unsigned long long *cyc) {
    CUtensorMap m;
    const cuuint64_t dims[5] = {16, HW, 1, KT, N};
    const cuuint64_t str[4] = {64, (cuuint64_t)HW * 64, (cuuint64_t)HW * 64, (cuuint64_t)KT * HW * 64};
    const cuuint32_t box[5] = {16, 128, 1, BOX_KT, 1}, es[5] = {1, 1, 1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, y, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto k = probe<DEPTH, ISSUERS, BOX_KT>;
    const int sm = DEPTH * ISSUERS * 8192 * BOX_KT + 2048;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    float best = 1e9;
    unsigned long long mx = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<148, 64, sm>>>(m, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
        std::vector<unsigned long long> h(148);
        cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
        mx = 0;
        for (auto c : h) mx = c > mx ? c : mx;
    }
    const double bytes = 148.0 * NB * 8192;
    printf("depth %d issuers %d box %2d KB: %6.0f cycles per 8 KB store, %.0f GB/s (%s)\n", DEPTH, ISSUERS,
           8 * BOX_KT, (double)mx / NB, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float *y;
    cudaMalloc(&y, (size_t)N * KT * HW * 64);
    unsigned long long *cyc;
    cudaMalloc(&cyc, 148 * 8);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
    run<1, 1, 1>(enc, y, cyc);
    run<2, 1, 1>(enc, y, cyc);
    run<4, 1, 1>(enc, y, cyc);
    run<8, 1, 1>(enc, y, cyc);
    run<2, 2, 1>(enc, y, cyc);
    run<4, 2, 1>(enc, y, cyc);
    run<2, 1, 2>(enc, y, cyc);
    run<4, 1, 2>(enc, y, cyc);
    return 0;
}
