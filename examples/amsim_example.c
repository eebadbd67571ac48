/*
 * Standalone use of the C ABI (include/amsim.h) without Python or PyTorch:
 * build an Alg. 1 table from a user-supplied functional model, run one
 * approximate GEMM on the GPU and compare a few outputs with a host
 * evaluation of the same model.
 *
 *   gcc -O2 -I include -I $CUDA_HOME/include examples/amsim_example.c \
 *       -L paper_2209_04161_b200 -lamsim -L $CUDA_HOME/lib64 -lcudart -lm -o amsim_example
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "amsim.h"

/* a user multiplier model: the exact product, i.e. bfloat16 by
 * truncation at m = 7 (the library truncates the operands before calling it) */
static float my_model(float a, float b) { return a * b; }

static float trunc7(float x)
{
    unsigned u;
    memcpy(&u, &x, 4);
    u &= 0xFFFF0000u;
    memcpy(&x, &u, 4);
    return x;
}

#define CHECK(call)                                                                            \
    do {                                                                                       \
        amsim_status s_ = (call);                                                              \
        if (s_ != AMSIM_OK) {                                                                  \
            fprintf(stderr, "%s failed: %d (%s)\n", #call, (int)s_, amsim_last_error());       \
            return 1;                                                                          \
        }                                                                                      \
    } while (0)

int main(void)
{
    const int M = 64, N = 48, K = 80;
    amsim_lut *lut = NULL;
    CHECK(amsim_lut_build(my_model, 7, &lut));
    float *hA = malloc(sizeof(float) * M * K), *hB = malloc(sizeof(float) * K * N), *hC = malloc(sizeof(float) * M * N);
    srand(1);
    for (int i = 0; i < M * K; i++) hA[i] = (float)rand() / RAND_MAX - 0.5f;
    for (int i = 0; i < K * N; i++) hB[i] = (float)rand() / RAND_MAX - 0.5f;
    float *dA, *dB, *dC;
    if (cudaMalloc((void **)&dA, sizeof(float) * M * K) != cudaSuccess ||
        cudaMalloc((void **)&dB, sizeof(float) * K * N) != cudaSuccess ||
        cudaMalloc((void **)&dC, sizeof(float) * M * N) != cudaSuccess) {
        fprintf(stderr, "no CUDA device\n");
        return 2;
    }
    cudaMemcpy(dA, hA, sizeof(float) * M * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(float) * K * N, cudaMemcpyHostToDevice);
    CHECK(amsim_set_path_policy(2)); /* no split-K: sequential FP32 order, comparable bit for bit */
    CHECK(amsim_gemm(lut, 0, 0, M, N, K, dA, K, dB, N, dC, N, 0, NULL));
    cudaMemcpy(hC, dC, sizeof(float) * M * N, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M; i += 7)
        for (int j = 0; j < N; j += 5) {
            float acc = 0.0f;
            for (int t = 0; t < K; t++) acc += trunc7(hA[i * K + t]) * trunc7(hB[t * N + j]);
            if (acc != hC[i * N + j]) bad++;
        }
    printf("amsim_example: %s (%d mismatches), %llu kernel launches\n", bad ? "FAIL" : "ok", bad,
           (unsigned long long)amsim_launch_count());
    amsim_lut_destroy(lut);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
    free(hA);
    free(hB);
    free(hC);
    return bad ? 1 : 0;
}
