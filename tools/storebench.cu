// tools/storebench.cu -- store-path ceilings on B200 for the fused kernels' output patterns
// (DESIGN.md §4.3): per-thread 8-byte stores touching 64 bytes of each of 4 lines per warp
// instruction (fused7's c stores), 8-byte stores covering 2 whole lines, 16-byte stores
// covering 4 whole lines, and TMA (cp.async.bulk.tensor) stores of 32 KB smem tiles.
// Each writes `bytes` to a buffer (DRAM-bound for 8 GB, L2-resident for 64 MB x reps).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

// view: rows of 512 complex (4 KB); a "tile" = 8 (or 16) columns x 512 rows
// (a) fused7 c-store pattern: lane (s8 = tid & 7, h8 = tid >> 3), 16 values per round, row h8 + 16 k
__global__ void k_st64_half(float2* out, int64_t tiles, int reps) {
    const int tid = threadIdx.x, s8 = tid & 7, h8 = tid >> 3;
    for (int r = 0; r < reps; ++r)
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            float2* base = out + (t / 64) * 512 * 512 + (t % 64) * 8;   // 64 tiles of 8 columns per 512x512 block
#pragma unroll 8
            for (int k = 0; k < 32; ++k) __stcs(base + (int64_t)(h8 + 16 * k) * 512 + s8, make_float2(k, r));
        }
}
// (b) 16-column tiles, lane (s16 = tid & 15, h16 = tid >> 4) with 128 threads covering 8 rows: 2 whole lines / instr
__global__ void k_st64_full(float2* out, int64_t tiles, int reps) {
    const int tid = threadIdx.x, s16 = tid & 15, h16 = tid >> 4;
    for (int r = 0; r < reps; ++r)
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            float2* base = out + (t / 32) * 512 * 512 + (t % 32) * 16;
#pragma unroll 8
            for (int k = 0; k < 64; ++k) __stcs(base + (int64_t)(h16 + 8 * k) * 512 + s16, make_float2(k, r));
        }
}
// (c) 16-byte stores, 4 whole lines per warp instruction
__global__ void k_st128(float4* out, int64_t tiles, int reps) {
    const int tid = threadIdx.x, s8 = tid & 7, h8 = tid >> 3;
    for (int r = 0; r < reps; ++r)
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            float4* base = out + (t / 32) * 512 * 256 + (t % 32) * 8;
#pragma unroll 8
            for (int k = 0; k < 32; ++k) __stcs(base + (int64_t)(h8 + 16 * k) * 256 + s8, make_float4(k, r, 0, 1));
        }
}
// (d) TMA stores: each CTA fills a 32 KB smem tile (8 columns x 512 rows) once and stores it
// as two 8 x 256 boxes per tile
__global__ void k_tma_store(const __grid_constant__ CUtensorMap map, int64_t tiles, int reps) {
    extern __shared__ __align__(128) float2 sm[];
    for (int i = threadIdx.x; i < 8 * 512; i += blockDim.x) sm[i] = make_float2(i, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int r = 0; r < reps; ++r)
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int x = (int)(t % 64) * 8, y = (int)(t / 64) * 512;
                for (int h = 0; h < 2; ++h) {
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&map),
                                 "r"(x), "r"(y + 256 * h), "r"((uint32_t)__cvta_generic_to_shared(sm + 256 * 8 * h))
                                 : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
            }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

template <typename F>
float timeit(F f, int reps = 3) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    const size_t big = (size_t)8 << 30;   // 8 GiB: DRAM-bound
    float2* buf;
    CK(cudaMalloc(&buf, big));
    CK(cudaFuncSetAttribute(k_tma_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    for (int pass = 0; pass < 2; ++pass) {
        const size_t bytes = pass == 0 ? big : ((size_t)64 << 20);
        const int reps = pass == 0 ? 1 : 64;
        const char* tag = pass == 0 ? "dram_8GiB" : "l2_64MiB_x64";
        const int64_t tiles8 = bytes / (8 * 512 * 8), tiles16 = bytes / (16 * 512 * 8);
        const double total = (double)bytes * reps;
        for (int ctas : {3, 4}) {
            const int grid = sms * ctas;
            float ms = timeit([&] { k_st64_half<<<grid, 128>>>(buf, tiles8, reps); });
            printf("{\"case\": \"%s\", \"ctas_per_sm\": %d, \"pattern\": \"st64 64B/line (fused7 c)\", \"GBs\": %.0f}\n", tag, ctas, total / (ms * 1e-3) / 1e9);
            ms = timeit([&] { k_st64_full<<<grid, 128>>>(buf, tiles16, reps); });
            printf("{\"case\": \"%s\", \"ctas_per_sm\": %d, \"pattern\": \"st64 whole lines\", \"GBs\": %.0f}\n", tag, ctas, total / (ms * 1e-3) / 1e9);
            ms = timeit([&] { k_st128<<<grid, 128>>>((float4*)buf, tiles16, reps); });
            printf("{\"case\": \"%s\", \"ctas_per_sm\": %d, \"pattern\": \"st128 whole lines\", \"GBs\": %.0f}\n", tag, ctas, total / (ms * 1e-3) / 1e9);
        }
        CUtensorMap map;
        cuuint64_t dims[2] = {512, (cuuint64_t)(bytes / 4096)};
        cuuint64_t strides[1] = {4096};
        cuuint32_t box[2] = {8, 256}, es[2] = {1, 1};
        if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            return 1;
        }
        for (int ctas : {1, 3, 6}) {
            float ms = timeit([&] { k_tma_store<<<sms * ctas, 128, 32768>>>(map, tiles8, reps); });
            printf("{\"case\": \"%s\", \"ctas_per_sm\": %d, \"pattern\": \"tma store 8x256 boxes\", \"GBs\": %.0f}\n", tag, ctas, total / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
