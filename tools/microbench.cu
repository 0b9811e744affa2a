// tools/microbench.cu -- measures the B200 ceilings DESIGN.md uses: FP32/FP64 FMA and FADD
// issue rates, L2-resident read/write bandwidth, HBM copy bandwidth, shared-memory bandwidth.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <typename T>
__global__ void k_ffma(T* out, int iters, T a, T b) {
    T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
            x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
// 3-register FFMA: multiplicand from a register that varies (not an immediate/constant)
template <typename T>
__global__ void k_ffma3(T* out, int iters, T a0) {
    T a = a0 + threadIdx.x * (T)1e-7, b = a * (T)0.5;
    T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, b, a); x2 = fma(x2, a, x0); x3 = fma(x3, b, x1);
            x4 = fma(x4, a, x2); x5 = fma(x5, b, x3); x6 = fma(x6, a, x4); x7 = fma(x7, b, x5);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
template <typename T>
__global__ void k_fadd(T* out, int iters) {
    T a = threadIdx.x * (T)1e-7, b = a * (T)0.5;
    T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x0 = x0 + a; x1 = x1 + b; x2 = x2 + x0; x3 = x3 + x1;
            x4 = x4 + x2; x5 = x5 + x3; x6 = x6 + x4; x7 = x7 + x5;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_read(const float4* __restrict__ in, size_t n, int reps, float4* out) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            float4 v = in[i];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    if (acc.x == 1234.5f) out[0] = acc;
}
__global__ void k_write(float4* out, size_t n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
            out[i] = make_float4(r, i, 0, 1);
}
__global__ void k_copy(const float4* __restrict__ in, float4* out, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) out[i] = in[i];
}
__global__ void k_smem(float* out, int iters) {
    __shared__ float2 buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = make_float2(i, i);
    __syncthreads();
    float2 acc = make_float2(0, 0);
    int idx = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float2 v = buf[(idx + k * 256) & 4095];
            acc.x += v.x; acc.y += v.y;
        }
        idx += 32;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
}

template <typename F>
float timeit(F f, int reps = 5) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    printf("{\"sms\": %d, \"clock_khz\": %d, \"l2_bytes\": %d", sms, clk, l2);
    float* fo; double* dout; CK(cudaMalloc(&fo, 1 << 26)); CK(cudaMalloc(&dout, 1 << 27));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    double ops = (double)blocks * threads * iters * 64;  // 8 chains x 8 unrolled
    float ms = timeit([&] { k_ffma<float><<<blocks, threads>>>(fo, iters, 1.0000001f, 1e-7f); });
    printf(", \"fp32_ffma_imm_Tinstr_s\": %.3f", ops / (ms * 1e-3) / 1e12);
    ms = timeit([&] { k_ffma3<float><<<blocks, threads>>>(fo, iters, 1.0000001f); });
    printf(", \"fp32_ffma_reg_Tinstr_s\": %.3f", ops / (ms * 1e-3) / 1e12);
    ms = timeit([&] { k_fadd<float><<<blocks, threads>>>(fo, iters); });
    printf(", \"fp32_fadd_Tinstr_s\": %.3f", ops / (ms * 1e-3) / 1e12);
    ms = timeit([&] { k_ffma3<double><<<blocks, threads>>>(dout, iters / 4, 1.0000001); });
    printf(", \"fp64_dfma_reg_Tinstr_s\": %.3f", ops / 4 / (ms * 1e-3) / 1e12);
    ms = timeit([&] { k_fadd<double><<<blocks, threads>>>(dout, iters / 4); });
    printf(", \"fp64_dadd_Tinstr_s\": %.3f", ops / 4 / (ms * 1e-3) / 1e12);
    // L2-resident read / write bandwidth at several footprints
    float4* buf; size_t big = (size_t)4 << 30; CK(cudaMalloc(&buf, big)); float4* buf2; CK(cudaMalloc(&buf2, big));
    cudaMemset(buf, 0, big);
    for (size_t mb : {16, 32, 64, 96}) {
        size_t n = mb * (1 << 20) / 16;
        int reps = 20;
        ms = timeit([&] { k_read<<<sms * 4, 512>>>(buf, n, reps, buf2); });
        printf(", \"l2_read_%zuMB_GBs\": %.0f", mb, (double)n * 16 * reps / (ms * 1e-3) / 1e9);
        ms = timeit([&] { k_write<<<sms * 4, 512>>>(buf, n, reps); });
        printf(", \"l2_write_%zuMB_GBs\": %.0f", mb, (double)n * 16 * reps / (ms * 1e-3) / 1e9);
    }
    size_t n = big / 16;
    ms = timeit([&] { k_read<<<sms * 4, 512>>>(buf, n, 1, buf2); });
    printf(", \"hbm_read_GBs\": %.0f", (double)n * 16 / (ms * 1e-3) / 1e9);
    ms = timeit([&] { k_write<<<sms * 4, 512>>>(buf, n, 1); });
    printf(", \"hbm_write_GBs\": %.0f", (double)n * 16 / (ms * 1e-3) / 1e9);
    ms = timeit([&] { k_copy<<<sms * 4, 512>>>(buf, buf2, n); });
    printf(", \"hbm_copy_GBs\": %.0f", (double)n * 32 / (ms * 1e-3) / 1e9);
    ms = timeit([&] { k_smem<<<sms * 4, 256>>>(fo, 4096); });
    printf(", \"smem_read_B_per_clk_per_sm\": %.1f", (double)sms * 4 * 256 * 4096 * 8 * 8 / (ms * 1e-3) / (clk * 1e3) / sms);
    printf("}\n");
    return 0;
}
