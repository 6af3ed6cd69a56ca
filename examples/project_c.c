/*
 * project_c.c — the library used from plain C (no Python, no torch): the random projection
 * Y = A . Omega of PAPER.md Eq 1 through include/shgemm.h only.
 *
 *   gcc -O2 -I include examples/project_c.c -o project_c \
 *       -L paper_2304_04612_b200 -lshgemm -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,...
 *   ./project_c m k n seed  > Y.bin         (prints a summary line on stderr)
 *
 * A is filled on the device by shg_synth_f32 (Gaussian, OMEGA_SPEC §6, seed `seed`, stream 0x100),
 * Omega by gen_omega_f16 (seed 0), Y = A . Omega by shgemm; Y (m x n FP32, row-major) is written to
 * stdout as raw little-endian floats so a test can compare it with the Python binding's result.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "shgemm.h"

#define CHECK_CUDA(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 2; } } while (0)
#define CHECK_SHG(x) do { shg_status_t s_ = (x); if (s_ != SHG_OK) { \
    fprintf(stderr, "%s: status %d %s\n", #x, (int)s_, shg_last_error()); return 3; } } while (0)

int main(int argc, char **argv) {
    if (argc != 5) {
        fprintf(stderr, "usage: %s m k n seed\n", argv[0]);
        return 1;
    }
    const int64_t m = atoll(argv[1]), k = atoll(argv[2]), n = atoll(argv[3]);
    const uint64_t seed = strtoull(argv[4], NULL, 10);
    if (!shg_device_supported()) {
        fprintf(stderr, "no sm_100 device\n");
        return 4;
    }
    /* SURVEY §8(b) layouts: A row-major (lda >= k), Omega row-major (ldo >= n), Y row-major */
    const int64_t lda = (k + 3) / 4 * 4, ldo = n;
    float *A = NULL, *Y = NULL;
    uint16_t *Om = NULL;
    CHECK_CUDA(cudaMalloc((void **)&A, (size_t)(m * lda) * sizeof(float)));
    CHECK_CUDA(cudaMalloc((void **)&Om, (size_t)(k * ldo) * sizeof(uint16_t)));
    CHECK_CUDA(cudaMalloc((void **)&Y, (size_t)(m * n) * sizeof(float)));
    cudaStream_t st;
    CHECK_CUDA(cudaStreamCreate(&st));
    shg_stream_t s = (shg_stream_t)st;
    CHECK_SHG(shg_synth_f32(0, seed, 0x100u, m, k, 0, A, lda, s));
    CHECK_SHG(gen_omega_f16(k, n, 0, SHG_DIST_GAUSSIAN, Om, ldo, s));
    CHECK_SHG(shgemm(m, n, k, A, lda, Om, ldo, Y, n, s));
    CHECK_CUDA(cudaStreamSynchronize(st));
    float *h = (float *)malloc((size_t)(m * n) * sizeof(float));
    CHECK_CUDA(cudaMemcpy(h, Y, (size_t)(m * n) * sizeof(float), cudaMemcpyDeviceToHost));
    fwrite(h, sizeof(float), (size_t)(m * n), stdout);
    double sum = 0.0;
    for (int64_t i = 0; i < m * n; ++i) sum += h[i];
    fprintf(stderr, "%s: Y = A . Omega, %lld x %lld x %lld, sum %.9g, %llu kernels\n", shg_version(), (long long)m,
            (long long)k, (long long)n, sum, (unsigned long long)shg_launch_count());
    free(h);
    cudaFree(A);
    cudaFree(Om);
    cudaFree(Y);
    cudaStreamDestroy(st);
    return 0;
}
