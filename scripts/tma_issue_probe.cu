// tma_issue_probe.cu -- cost of TMA box count vs box size for conv A tiles.
// x = [64 img][16 ct][14][14][16] fp32 (12.8 MB, L2-resident after the first pass).
// Per "k-block" one producer thread loads 16 KB of A in one of three ways:
//   A: 2 boxes {16, 14, 9, 1, 1} (two 126-px tiles of 8 KB, like box tiles)
//   B: 18 boxes {16, 14, 1, 1, 1} (896 B each: one output row per box)
//   C: 4 boxes {16, 14, 9, 1, 1} (two-box windows: 2 x 8 KB per 16-channel sub)
// 148 CTAs x 2000 k-blocks; reports cycles per k-block (max CTA).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2006_02230_b200/csrc/pdl_sm100.cuh"

using namespace pdl;
constexpr int NIMG = 64, CT = 16, HW = 14, STAGES = 4, STAGE = 36 * 1024, KB = 2000;

template <int V>
__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap m9, const __grid_constant__ CUtensorMap m1,
                                               unsigned long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE), *empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int k = 0; k < KB; ++k) {
            const int img = (blockIdx.x * 7 + k) % NIMG, ct = k % CT, r0 = k % 6;
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t *d = smem + s * STAGE;
            if (V == 0) {
                mbar_arrive_expect_tx(&full[s], 2 * 8064);
                tma_load_5d(d, &m9, &full[s], 0, 0, r0, ct, img);
                tma_load_5d(d + 8192, &m9, &full[s], 0, 0, r0, (ct + 1) % CT, img);
            } else if (V == 1) {
                mbar_arrive_expect_tx(&full[s], 18 * 896);
                for (int j = 0; j < 9; ++j)
                    for (int c = 0; c < 2; ++c)
                        tma_load_5d(d + c * 8192 + j * 896, &m1, &full[s], 0, 0, (r0 + j) % HW, (ct + c) % CT, img);
            } else {
                mbar_arrive_expect_tx(&full[s], 4 * 8064);
                for (int c = 0; c < 2; ++c) {
                    tma_load_5d(d + c * 16384, &m9, &full[s], 0, 0, r0 + 5, (ct + c) % CT, img);
                    tma_load_5d(d + c * 16384 + 8192, &m9, &full[s], 0, 0, r0 + 5 - HW, (ct + c) % CT, (img + 1) % NIMG);
                }
            }
            if (++s == STAGES) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int s = 0;
        uint32_t ph = 0;
        for (int k = 0; k < KB; ++k) {
            mbar_wait(&full[s], ph);
            mbar_arrive(&empty[s]);
            if (++s == STAGES) { s = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    float *x;
    const size_t bytes = (size_t)NIMG * CT * HW * HW * 64;
    cudaMalloc(&x, bytes);
    cudaMemset(x, 0, bytes);
    unsigned long long *cyc;
    cudaMalloc(&cyc, 148 * 8);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
    CUtensorMap m9, m1;
    const cuuint64_t dims[5] = {16, HW, HW, CT, NIMG};
    const cuuint64_t str[4] = {64, HW * 64, HW * HW * 64, (cuuint64_t)CT * HW * HW * 64};
    const cuuint32_t b9[5] = {16, HW, 9, 1, 1}, b1[5] = {16, HW, 1, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    enc(&m9, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, x, dims, str, b9, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&m1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, x, dims, str, b1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const char *names[3] = {"A 2 boxes of 9 rows (16 KB)", "B 18 boxes of 1 row (16 KB)", "C 4 boxes of 9 rows (32 KB, half OOB)"};
    for (int grid : {148, 74, 16}) {
        for (int v = 0; v < 3; ++v) {
            auto k = v == 0 ? probe<0> : v == 1 ? probe<1> : probe<2>;
            const int sm = STAGES * STAGE + 2048;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            for (int rep = 0; rep < 3; ++rep) {
                k<<<grid, 64, sm>>>(m9, m1, cyc);
                cudaError_t e = cudaDeviceSynchronize();
                std::vector<unsigned long long> h(grid);
                cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
                unsigned long long mx = 0;
                for (auto c : h) mx = c > mx ? c : mx;
                if (rep == 2)
                    printf("grid %3d %-40s %s %.0f cycles per k-block\n", grid, names[v], cudaGetErrorString(e),
                           (double)mx / KB);
            }
        }
    }
    return 0;
}
