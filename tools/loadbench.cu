// tools/loadbench.cu -- tile-load ceilings for the fused kernels' input path.
// Each CTA streams 32 KB tiles (8 columns x 512 rows of a row-major array with 4 KB rows, the
// shape of an f tile or a ring tile) from an L2-resident 80 MB buffer and does `work` dummy FMA
// per value, two ways:
//   ldg: 128 threads, lane (s8, h8) loads rows h8 + 16 k (k < 32) of column s8 into registers,
//        the next tile's loads issued before the current tile's work (register prefetch)
//   tma: thread 0 copies the next tile (two 8 x 256 boxes) into one of NB shared buffers while
//        the threads read the current one from shared memory (mbarrier per buffer)
// Reports GB/s of tile data delivered for several CTAs/SM and work amounts.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ROWS = 512, COLS = 512;   // a 2 MB "signal" block: 512 rows of 512 complex

__device__ __forceinline__ float2 ldg2(const float2* p) {
    float2 r;
    asm volatile("ld.global.cg.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
    return r;
}

__global__ void __launch_bounds__(128, 3) k_ldg(const float2* buf, int64_t ntile, int tiles_per_cta, int work, float* sink) {
    const int tid = threadIdx.x, s8 = tid & 7, h8 = tid >> 3;
    float2 pre[32];
    float acc = 0.f;
    int64_t t = blockIdx.x;
    auto load = [&](int64_t tile) {
        const int64_t tt = tile % ntile;
        const float2* b = buf + (tt / 64) * ROWS * COLS + (tt % 64) * 8 + s8;
#pragma unroll
        for (int k = 0; k < 32; ++k) pre[k] = ldg2(b + (int64_t)(h8 + 16 * k) * COLS);
    };
    load(t);
    for (int i = 0; i < tiles_per_cta; ++i) {
        float2 v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = pre[k];
        load(t + (int64_t)gridDim.x * (i + 1));
        for (int w = 0; w < work; ++w)
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k].x = fmaf(v[k].x, 1.0001f, v[k].y);
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += v[k].x;
        __syncthreads();
    }
    if (acc == 1234.5f) sink[0] = acc;
}

template <int NB, bool WIDE = false>
__global__ void __launch_bounds__(128, 3) k_tma(const __grid_constant__ CUtensorMap map, int64_t ntile, int tiles_per_cta,
                                                int work, float* sink) {
    extern __shared__ __align__(128) float2 sm[];
    __shared__ __align__(8) uint64_t bar[NB];
    const int tid = threadIdx.x, s8 = tid & 7, h8 = tid >> 3;
    auto sa = [](const void* p) { return (uint32_t)__cvta_generic_to_shared(p); };
    if (tid == 0) {
        for (int b = 0; b < NB; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[b])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int i) {
        const int64_t tt = ((int64_t)blockIdx.x + (int64_t)gridDim.x * i) % ntile;
        const int b = i % NB;
        float2* dst = sm + b * 8 * ROWS;
        asm volatile("fence.proxy.async;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[b])), "r"(8 * ROWS * 8) : "memory");
        const int x = WIDE ? (int)((tt / 2) % 32) * 16 : (int)(tt % 64) * 8;
        const int y = WIDE ? (int)((tt / 2) / 32) * ROWS + (int)(tt & 1) * 256 : (int)(tt / 64) * ROWS;
        for (int h = 0; h < (WIDE ? 1 : 2); ++h)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                             sa(dst + h * 256 * 8)),
                         "l"(&map), "r"(x), "r"(y + 256 * h), "r"(sa(&bar[b]))
                         : "memory");
    };
    if (tid == 0)
        for (int i = 0; i < NB - 1 && i < tiles_per_cta; ++i) issue(i);
    float acc = 0.f;
    for (int i = 0; i < tiles_per_cta; ++i) {
        const int b = i % NB;
        const uint32_t parity = (i / NB) & 1;
        uint32_t done = 0;
        do {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(sa(&bar[b])), "r"(parity) : "memory");
        } while (!done);
        float2 v[32];
        const float2* src = sm + b * 8 * ROWS;
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = src[(h8 + 16 * k) * 8 + s8];
        __syncthreads();   // buffer (i - 1) % NB fully read: refill it
        if (tid == 0 && i + NB - 1 < tiles_per_cta) issue(i + NB - 1);
        for (int w = 0; w < work; ++w)
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k].x = fmaf(v[k].x, 1.0001f, v[k].y);
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += v[k].x;
    }
    if (acc == 1234.5f) sink[0] = acc;
}


// cp.async (LDGSTS, .cg: L2 only) of the tile into shared memory, double-buffered
__global__ void __launch_bounds__(128, 3) k_cpasync(const float2* buf, int64_t ntile, int tiles_per_cta, int work, float* sink) {
    extern __shared__ __align__(128) float2 sm[];
    const int tid = threadIdx.x, s8 = tid & 7, h8 = tid >> 3;
    auto issue = [&](int i) {
        const int64_t tt = ((int64_t)blockIdx.x + (int64_t)gridDim.x * i) % ntile;
        const float2* b = buf + (tt / 64) * ROWS * COLS + (tt % 64) * 8;
        float2* dst = sm + (i & 1) * 8 * ROWS;
        // 16-byte chunks: 512 rows x 4 chunks; thread tid takes chunks tid, tid + 128, ...
        for (int c = tid; c < ROWS * 4; c += 128) {
            const int row = c >> 2, q = c & 3;
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + row * 8 + 2 * q);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(b + (int64_t)row * COLS + 2 * q) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0);
    float acc = 0.f;
    for (int i = 0; i < tiles_per_cta; ++i) {
        if (i + 1 < tiles_per_cta) {
            issue(i + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        float2 v[32];
        const float2* src = sm + (i & 1) * 8 * ROWS;
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = src[(h8 + 16 * k) * 8 + s8];
        __syncthreads();
        for (int w = 0; w < work; ++w)
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k].x = fmaf(v[k].x, 1.0001f, v[k].y);
#pragma unroll
        for (int k = 0; k < 32; ++k) acc += v[k].x;
    }
    if (acc == 1234.5f) sink[0] = acc;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
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
    const size_t bytes = (size_t)80 << 20;   // L2-resident like the ring
    float2* buf;
    float* sink;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMalloc(&sink, 64));
    CK(cudaMemset(buf, 0, bytes));
    const int64_t ntile = bytes / (8 * ROWS * 8);
    CUtensorMap map;
    cuuint64_t dims[2] = {COLS, bytes / (COLS * 8)};
    cuuint64_t strides[1] = {COLS * 8};
    cuuint32_t box[2] = {8, 256}, es[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return 1;
    }
    CK(cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 32768));
    CK(cudaFuncSetAttribute(k_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768));
    CK(cudaFuncSetAttribute(k_tma<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768));
    CK(cudaFuncSetAttribute(k_tma<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768));
    const int tiles = 200;
    CK(cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, 56 * 1024));
    CK(cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 32768));
    // wide boxes: 16 columns (128-byte rows), 256 rows, one 32 KB box per "tile pair"
    CUtensorMap mapw;
    {
        cuuint32_t boxw[2] = {16, 256};
        if (enc(&mapw, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, buf, dims, strides, boxw, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            return 1;
        }
    }
    for (int work : {0, 8}) {
        for (int ballast : {0, 56}) {
            const int grid = sms * 3;
            const double total = (double)grid * tiles * 32768;
            float ms = timeit([&] { k_ldg<<<grid, 128, ballast * 1024>>>(buf, ntile, tiles, work, sink); });
            printf("{\"method\": \"ldg regs + %d KB smem ballast\", \"ctas_per_sm\": 3, \"work\": %d, \"GBs\": %.0f, \"cycles_per_tile\": %.0f}\n",
                   ballast, work, total / (ms * 1e-3) / 1e9, ms * 1e-3 * 1.965e9 / tiles);
        }
        const int grid = sms * 3;
        const double total = (double)grid * tiles * 32768;
        float ms = timeit([&] { k_cpasync<<<grid, 128, 2 * 32768>>>(buf, ntile, tiles, work, sink); });
        printf("{\"method\": \"cp.async.cg double-buffered\", \"ctas_per_sm\": 3, \"work\": %d, \"GBs\": %.0f, \"cycles_per_tile\": %.0f}\n", work,
               total / (ms * 1e-3) / 1e9, ms * 1e-3 * 1.965e9 / tiles);
        // TMA, 16-column boxes: each copy brings 2 tiles' worth (32 KB = 16 x 256 rows x 8 B):
        // counted as half a tile pair -- use the 8-column kernel with the wide map on 2 CTAs
        ms = timeit([&] { k_tma<3, true><<<sms * 2, 128, 3 * 32768>>>(mapw, ntile, tiles, work, sink); });
        printf("{\"method\": \"tma 16-col boxes 3 buffers\", \"ctas_per_sm\": 2, \"work\": %d, \"GBs\": %.0f}\n", work,
               (double)sms * 2 * tiles * 32768 / (ms * 1e-3) / 1e9);
    }
    for (int work : {0, 8, 32}) {
        for (int ctas : {2, 3}) {
            const int grid = sms * ctas;
            const double total = (double)grid * tiles * 32768;
            float ms = timeit([&] { k_ldg<<<grid, 128>>>(buf, ntile, tiles, work, sink); });
            printf("{\"method\": \"ldg regs\", \"ctas_per_sm\": %d, \"work\": %d, \"GBs\": %.0f, \"cycles_per_tile\": %.0f}\n", ctas, work,
                   total / (ms * 1e-3) / 1e9, ms * 1e-3 * 1.965e9 / tiles);
            ms = timeit([&] { k_tma<2><<<grid, 128, 2 * 32768>>>(map, ntile, tiles, work, sink); });
            printf("{\"method\": \"tma 2 buffers\", \"ctas_per_sm\": %d, \"work\": %d, \"GBs\": %.0f, \"cycles_per_tile\": %.0f}\n", ctas,
                   work, total / (ms * 1e-3) / 1e9, ms * 1e-3 * 1.965e9 / tiles);
            if (ctas == 2) {
                ms = timeit([&] { k_tma<3><<<grid, 128, 3 * 32768>>>(map, ntile, tiles, work, sink); });
                printf("{\"method\": \"tma 3 buffers\", \"ctas_per_sm\": %d, \"work\": %d, \"GBs\": %.0f, \"cycles_per_tile\": %.0f}\n",
                       ctas, work, total / (ms * 1e-3) / 1e9, ms * 1e-3 * 1.965e9 / tiles);
            }
        }
        {
            const int grid = sms;
            const double total = (double)grid * tiles * 32768;
            float ms = timeit([&] { k_tma<6><<<grid, 128, 6 * 32768>>>(map, ntile, tiles, work, sink); });
            printf("{\"method\": \"tma 6 buffers\", \"ctas_per_sm\": 1, \"work\": %d, \"GBs\": %.0f, \"cycles_per_tile\": %.0f}\n", work,
                   total / (ms * 1e-3) / 1e9, ms * 1e-3 * 1.965e9 / tiles);
        }
    }
    return 0;
}
