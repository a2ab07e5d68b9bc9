// cuFFT timings for the inverse 2048^2 x 32 FFT2 split by axis (layout study).
#include <cufft.h>
#include <cstdio>
#include <cuda_runtime.h>
static float timeit(cufftHandle p, cufftComplex* d, int reps = 20) {
    for (int i = 0; i < 3; ++i) cufftExecC2C(p, d, d, CUFFT_INVERSE);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) cufftExecC2C(p, d, d, CUFFT_INVERSE);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}
int main() {
    const int B = 32, Y = 2048, X = 2048;
    cufftComplex* d; cudaMalloc(&d, sizeof(cufftComplex) * (size_t)B * X * Y);
    cudaMemset(d, 0, sizeof(cufftComplex) * (size_t)B * X * Y);
    cufftHandle p2, py, px, pyb;
    int n2[2] = {Y, X};
    cufftPlanMany(&p2, 2, n2, nullptr, 1, X * Y, nullptr, 1, X * Y, CUFFT_C2C, B);
    printf("2-D [b][y][x]                 %.3f ms\n", timeit(p2, d));
    int n1[1] = {Y}, emb[1] = {Y};
    cufftPlanMany(&py, 1, n1, emb, B * X, 1, emb, B * X, 1, CUFFT_C2C, B * X);
    printf("1-D along y, [y][b][x]        %.3f ms\n", timeit(py, d));
    int nx[1] = {X};
    cufftPlanMany(&px, 1, nx, nullptr, 1, X, nullptr, 1, X, CUFFT_C2C, B * Y);
    printf("1-D along x, rows             %.3f ms\n", timeit(px, d));
    cufftPlanMany(&pyb, 1, n1, emb, X, 1, emb, X, 1, CUFFT_C2C, X);  // one plane [y][x]
    float t = 0;
    for (int i = 0; i < 3; ++i) cufftExecC2C(pyb, d, d, CUFFT_INVERSE);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) for (int i = 0; i < B; ++i) cufftExecC2C(pyb, d + (size_t)i * X * Y, d + (size_t)i * X * Y, CUFFT_INVERSE);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t, a, b);
    printf("1-D along y, per plane x32    %.3f ms\n", t / 10);
    return 0;
}
