/*
 * examples/dgt_c_example.c -- the C ABI used from plain C (no Python, no torch):
 * plan config 1's lattice (L = 240, a = 8, M = 12, lambda = 1/2, complex128), transform one
 * signal through dgt_execute_host (host buffers), compute the canonical dual window, build a
 * synthesis plan with it and reconstruct the signal through device buffers and
 * dgt_execute_inverse.  Prints the relative reconstruction error (expected ~1e-15).
 *
 *   gcc -O2 -I include examples/dgt_c_example.c -L paper_1307_4569_b200 -lnsdgt \
 *       -Wl,-rpath,$PWD/paper_1307_4569_b200 -L/usr/local/cuda/lib64 -lcudart -lm
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "nsdgt.h"

#define CHECK(call)                                                                     \
    do {                                                                                \
        int _s = (call);                                                                \
        if (_s != DGT_OK) {                                                             \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, dgt_strerror(_s), dgt_last_error()); \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

int main(void) {
    const int64_t L = 240, a = 8, M = 12, l1 = 1, l2 = 2, N = L / a;
    double* g = malloc(sizeof(double) * 2 * L);
    double* f = malloc(sizeof(double) * 2 * L);
    double* c = malloc(sizeof(double) * 2 * M * N);
    double* gd = malloc(sizeof(double) * 2 * L);
    double* fr = malloc(sizeof(double) * 2 * L);
    /* periodised Gaussian window (tfr = a M / L), unit norm; a deterministic test signal */
    double nrm = 0.0;
    for (int64_t l = 0; l < L; ++l) {
        double v = 0.0;
        for (int k = -3; k <= 3; ++k) {
            const double x = (double)(l + k * L);
            v += exp(-M_PI * x * x / ((double)a * M));
        }
        g[2 * l] = v;
        g[2 * l + 1] = 0.0;
        nrm += v * v;
        f[2 * l] = sin(0.3 * l) + 0.5 * cos(0.07 * l * l);
        f[2 * l + 1] = 0.25 * sin(1.1 * l);
    }
    for (int64_t l = 0; l < L; ++l) g[2 * l] /= sqrt(nrm);

    dgt_plan_t plan = NULL, synth = NULL;
    CHECK(dgt_plan(&plan, L, a, M, l1, l2, g, DGT_C128, DGT_G_ON_HOST, 0, 0, 0, 0, NULL));
    dgt_lattice_info info;
    CHECK(dgt_plan_query(plan, &info));
    printf("branch %d shear (%lld, %lld) inner M'=%lld d=%lld p=%lld q=%lld\n", (int)info.branch,
           (long long)info.s0, (long long)info.s1, (long long)info.iM, (long long)info.d, (long long)info.p,
           (long long)info.q);
    CHECK(dgt_execute_host(plan, f, c, 1, NULL));                   /* c = DGT(f) */
    CHECK(dgt_window_dual(plan, 0, gd, DGT_G_ON_HOST, NULL));        /* gamma = S^-1 g */
    CHECK(dgt_plan(&synth, L, a, M, l1, l2, gd, DGT_C128, DGT_G_ON_HOST, 0, 0, 0, 0, NULL));

    void *c_dev = NULL, *f_dev = NULL;
    if (cudaMalloc(&c_dev, sizeof(double) * 2 * M * N) != cudaSuccess || cudaMalloc(&f_dev, sizeof(double) * 2 * L) != cudaSuccess)
        return 1;
    cudaMemcpy(c_dev, c, sizeof(double) * 2 * M * N, cudaMemcpyHostToDevice);
    CHECK(dgt_execute_inverse(synth, c_dev, f_dev, 1, NULL));        /* f = sum c gamma_{m,n} */
    cudaMemcpy(fr, f_dev, sizeof(double) * 2 * L, cudaMemcpyDeviceToHost);

    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < 2 * L; ++i) {
        num += (fr[i] - f[i]) * (fr[i] - f[i]);
        den += f[i] * f[i];
    }
    printf("reconstruction rel_err %.3e\n", sqrt(num / den));
    cudaFree(c_dev);
    cudaFree(f_dev);
    dgt_destroy(synth);
    dgt_destroy(plan);
    free(g); free(f); free(c); free(gd); free(fr);
    return sqrt(num / den) < 1e-10 ? 0 : 2;
}
