// tools/fftbench.cu -- throughput of the warp FFT alone (no global memory in the loop).
#include <cstdio>
#include "../paper_1307_4569_b200/csrc/fast_kernels.cuh"
using namespace nsdgt;

template <int E, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_fft(float2* io, int iters) {
    __shared__ float2 scr_all[WARPS * WarpFftShape<E>::SCRATCH];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float2* scr = scr_all + warp * WarpFftShape<E>::SCRATCH;
    WarpFft<float, E> f;
    f.init(lane);
    float2 v[E];
    const int base = (blockIdx.x * WARPS + warp) * 32 * E;
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = io[base + lane + 32 * k];
    for (int it = 0; it < iters; ++it) {
        f.run(v, scr, lane);
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = make_float2(v[k].x * 0.03125f, v[k].y * 0.03125f);
    }
#pragma unroll
    for (int k = 0; k < E; ++k) io[base + lane + 32 * k] = v[k];
}

template <int E, int WARPS, int MINB>
void run(const char* name, int blocks) {
    float2* io; cudaMalloc(&io, sizeof(float2) * blocks * WARPS * 32 * E);
    cudaMemset(io, 0, sizeof(float2) * blocks * WARPS * 32 * E);
    const int iters = 200;
    k_fft<E, WARPS, MINB><<<blocks, WARPS * 32>>>(io, 2);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k_fft<E, WARPS, MINB><<<blocks, WARPS * 32>>>(io, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double ffts = (double)blocks * WARPS * iters;
    const double pts = ffts * 32 * E;
    printf("%-28s blocks=%d: %.3f ms, %.1f G-FFT/s, %.2f ns per 1k points, %s\n", name, blocks, ms, ffts / (ms * 1e-3) / 1e9,
           ms * 1e6 / (pts / 1000), cudaGetErrorString(cudaGetLastError()));
    cudaFree(io);
}

int main() {
    run<16, 8, 2>("E16 (512) 2x8 warps/SM", 296);
    run<16, 8, 1>("E16 (512) 1x8 warps/SM", 148);
    run<16, 4, 4>("E16 (512) 4x4 warps/SM", 592);
    run<8, 8, 4>("E8 (256) 4x8 warps/SM", 592);
    run<8, 8, 2>("E8 (256) 2x8 warps/SM", 296);
    return 0;
}
