// tma_probe.cu -- how fast can one SM's TMA bring in the ResNet stem's input
// halo?  The stem tile (16 x 8 outputs, 7x7 stride 2) needs a 37 x 21 pixel
// halo of the nChw16c input (C = 3 real channels in a 64-byte pixel).  Each
// variant below streams one halo per "tile" through a ring of smem stages
// (one producer thread, one consumer thread re-arming the ring) on 148 CTAs,
// 169 tiles each (the N=256 stem), and reports cycles per tile:
//   A  box {4 ch, 37 px, 21 rows}: 777 rows of 16 B (the current kernel)
//   B  box {16 ch, 37 px, 21 rows}: 777 rows of 64 B (whole pixels)
//   C  3-D view [N][H][W*16] floats, box {128 floats = 8 px, 21 rows} x 5 loads (1 KB rows)
//   D  box {4 ch, 19 px, 21 rows} on even + odd column maps (parity split), 2 loads
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda scripts/tma_probe.cu -o /tmp/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2006_02230_b200/csrc/pdl_sm100.cuh"

using namespace pdl;

constexpr int N = 256, H = 224, W = 224;
constexpr int TILES_PER_IMG = 7 * 14;  // 112 / 16 x 112 / 8
constexpr int STAGE_BYTES = 54 * 1024;
constexpr int STAGES = 3;

struct Maps {
    CUtensorMap m0, m1;
};

template <int V>
__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ Maps maps, int tiles, unsigned long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int i = 0; i < tiles; ++i) {
            const int t = blockIdx.x + i * gridDim.x;
            const int img = (t / TILES_PER_IMG) % N, tt = t % TILES_PER_IMG;
            const int q0 = (tt % 7) * 16, p0 = (tt / 7) * 8;
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t *dst = smem + s * STAGE_BYTES;
            if (V == 0) {
                mbar_arrive_expect_tx(&full[s], 37 * 21 * 16);
                tma_load_5d(dst, &maps.m0, &full[s], 0, 2 * q0 - 3, 2 * p0 - 3, 0, img);
            } else if (V == 1) {
                mbar_arrive_expect_tx(&full[s], 37 * 21 * 64);
                tma_load_5d(dst, &maps.m0, &full[s], 0, 2 * q0 - 3, 2 * p0 - 3, 0, img);
            } else if (V == 2) {
                mbar_arrive_expect_tx(&full[s], 5 * 21 * 512);
                for (int j = 0; j < 5; ++j)
                    tma_load_5d(dst + j * 21 * 512, &maps.m0, &full[s], (2 * q0 - 3) * 16 + j * 128, 2 * p0 - 3, img, 0, 0);
            } else {
                mbar_arrive_expect_tx(&full[s], (19 + 19) * 21 * 16);
                // even input columns 2q0-2.. (q0-1 + k), odd 2q0-3.. -> both 19 wide
                tma_load_5d(dst, &maps.m0, &full[s], 0, q0 - 1, 2 * p0 - 3, 0, img);
                tma_load_5d(dst + 19 * 21 * 16, &maps.m1, &full[s], 0, q0 - 2, 2 * p0 - 3, 0, img);
            }
            if (++s == STAGES) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int s = 0;
        uint32_t ph = 0;
        for (int i = 0; i < tiles; ++i) {
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
    const size_t bytes = (size_t)N * H * W * 64;
    cudaMalloc(&x, bytes);
    cudaMemset(x, 0, bytes);
    unsigned long long *cyc;
    cudaMalloc(&cyc, 148 * sizeof(unsigned long long));
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    const int tiles = (N * TILES_PER_IMG + 147) / 148;
    const char *names[4] = {"A box{4ch,37px,21} 777x16B", "B box{16ch,37px,21} 777x64B",
                            "C [N][H][W*16] box{128,21} x5 (105x512B)", "D parity box{4ch,19px,21} x2"};
    for (int v = 0; v < 4; ++v) {
        Maps m;
        CUresult r;
        if (v == 0 || v == 1) {
            const cuuint64_t dims[5] = {16, W, H, 1, N};
            const cuuint64_t str[4] = {64, (cuuint64_t)W * 64, (cuuint64_t)H * W * 64, (cuuint64_t)H * W * 64};
            const cuuint32_t box[5] = {(cuuint32_t)(v == 0 ? 4 : 16), 37, 21, 1, 1};
            r = enc(&m.m0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            m.m1 = m.m0;
        } else if (v == 2) {
            const cuuint64_t dims[5] = {(cuuint64_t)W * 16, H, N, 1, 1};
            const cuuint64_t str[4] = {(cuuint64_t)W * 64, (cuuint64_t)H * W * 64, bytes, bytes};
            const cuuint32_t box[5] = {128, 21, 1, 1, 1};
            r = enc(&m.m0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            m.m1 = m.m0;
        } else {
            for (int par = 0; par < 2; ++par) {
                const cuuint64_t dims[5] = {16, (cuuint64_t)(W - par + 1) / 2, H, 1, N};
                const cuuint64_t str[4] = {128, (cuuint64_t)W * 64, (cuuint64_t)H * W * 64, (cuuint64_t)H * W * 64};
                const cuuint32_t box[5] = {4, 19, 21, 1, 1};
                r = enc(par ? &m.m1 : &m.m0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, x + par * 16, dims, str, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r) break;
            }
        }
        if (r != CUDA_SUCCESS) {
            printf("%s: encode failed %d\n", names[v], (int)r);
            continue;
        }
        auto k = v == 0 ? probe<0> : v == 1 ? probe<1> : v == 2 ? probe<2> : probe<3>;
        const int sm = STAGES * STAGE_BYTES + 2048;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k<<<148, 64, sm>>>(m, tiles, cyc);
            cudaEventRecord(e1);
            cudaError_t err = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<unsigned long long> h(148);
            cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
            unsigned long long mx = 0;
            for (auto c : h) mx = c > mx ? c : mx;
            if (rep == 2)
                printf("%-45s %s  %.4f ms  %.0f cycles/tile (max CTA)\n", names[v], cudaGetErrorString(err), ms,
                       (double)mx / tiles);
        }
    }
    return 0;
}
