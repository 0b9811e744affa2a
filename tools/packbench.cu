// packed FP32x2 (FFMA2/FADD2) vs scalar FFMA/FADD issue throughput on sm_100a
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){ u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ u64 add2(u64 a, u64 b){ u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__global__ void k_fma2(u64* out, int iters, u64 a, u64 b) {
    u64 x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) { x[0]=fma2(x[0],a,b); x[1]=fma2(x[1],a,b); x[2]=fma2(x[2],a,b); x[3]=fma2(x[3],a,b);
                                       x[4]=fma2(x[4],a,b); x[5]=fma2(x[5],a,b); x[6]=fma2(x[6],a,b); x[7]=fma2(x[7],a,b);}
    }
    u64 s = 0; for (int k = 0; k < 8; ++k) s ^= x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_add2(u64* out, int iters, u64 a) {
    u64 x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) { x[0]=add2(x[0],a); x[1]=add2(x[1],a); x[2]=add2(x[2],a); x[3]=add2(x[3],a);
                                       x[4]=add2(x[4],a); x[5]=add2(x[5],a); x[6]=add2(x[6],a); x[7]=add2(x[7],a);}
    }
    u64 s = 0; for (int k = 0; k < 8; ++k) s ^= x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed: FADD2 interleaved with independent LDS/SHFL (does packed math co-issue with MIO?)
__global__ void k_ffma(float* out, int iters, float a, float b) {
    float x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) { for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b); }
    }
    float s = 0; for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_shfl(float* out, int iters) {
    float x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) { for (int j = 0; j < 8; ++j) x[j] = __shfl_xor_sync(0xffffffffu, x[j], 16) + 1.0f; }
    }
    float s = 0; for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_lds64(float* out, int iters) {
    __shared__ float2 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float2(i, i);
    __syncthreads();
    float2 acc[4] = {};
    int idx = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) { float2 v = buf[(idx + k * 64) & 2047]; acc[k&3].x += v.x; acc[k&3].y += v.y; }
        idx = (idx + 32) & 2047;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0].x + acc[1].y + acc[2].x + acc[3].y;
}
__global__ void k_lds128(float* out, int iters) {
    __shared__ float4 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
    __syncthreads();
    float4 acc[4] = {};
    int idx = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) { float4 v = buf[(idx + k * 64) & 1023]; acc[k&3].x += v.x; acc[k&3].w += v.w; }
        idx = (idx + 32) & 1023;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0].x + acc[1].w + acc[2].x + acc[3].w;
}
template <typename F> float timeit(F f) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
    return best;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    void* o; cudaMalloc(&o, 1 << 26);
    const int blocks = sms * 8, thr = 256, it = 2048;
    double n = (double)blocks * thr * it * 64;  // thread-instructions
    double cyc = clk * 1e3 * sms;
    float ms;
    ms = timeit([&] { k_ffma<<<blocks, thr>>>((float*)o, it, 1.0000001f, 1e-7f); });
    printf("FFMA   warp-instr/clk/SM %.2f\n", n / 32 / (ms * 1e-3) / cyc);
    u64 a2 = 0x3f8000013f800001ull, b2 = 0x3400000034000000ull;
    ms = timeit([&] { k_fma2<<<blocks, thr>>>((u64*)o, it, a2, b2); });
    printf("FFMA2  warp-instr/clk/SM %.2f  (x2 lanes)\n", n / 32 / (ms * 1e-3) / cyc);
    ms = timeit([&] { k_add2<<<blocks, thr>>>((u64*)o, it, b2); });
    printf("FADD2  warp-instr/clk/SM %.2f  (x2 lanes)\n", n / 32 / (ms * 1e-3) / cyc);
    ms = timeit([&] { k_shfl<<<blocks, thr>>>((float*)o, it / 4); });
    printf("SHFL(+FADD) warp-shfl/clk/SM %.2f\n", n / 4 / 32 / (ms * 1e-3) / cyc);
    ms = timeit([&] { k_lds64<<<blocks, thr>>>((float*)o, it / 4); });
    printf("LDS.64 warp-instr/clk/SM %.2f\n", (double)blocks * thr * (it / 4) * 16 / 32 / (ms * 1e-3) / cyc);
    ms = timeit([&] { k_lds128<<<blocks, thr>>>((float*)o, it / 4); });
    printf("LDS.128 warp-instr/clk/SM %.2f\n", (double)blocks * thr * (it / 4) * 16 / 32 / (ms * 1e-3) / cyc);
    return 0;
}
