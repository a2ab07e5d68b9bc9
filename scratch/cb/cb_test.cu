#include <cufftXt.h>
#include <cstdio>
#include <vector>
#include <fstream>
#include <iterator>
#include <algorithm>
#include <random>
#include <ctime>
#include <cstdlib>
struct CbInfo { const float* in; int n_slices, T, P, B; const int* perm; float2* q; };
__global__ void pack(const float* in, int n, int T, int P, int B, float2* out) { // [b][t][p]
    size_t N = (size_t)B * T * P;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < N; i += (size_t)gridDim.x * blockDim.x) {
        size_t b = i / ((size_t)T * P), r = i % ((size_t)T * P);
        float2 v; v.x = 2*b < n ? in[2*b*(size_t)T*P + r] : 0; v.y = 2*b+1 < n ? in[(2*b+1)*(size_t)T*P + r] : 0; out[i] = v; }
}
__global__ void permk(const float2* in, const int* perm, int B, size_t N, float2* q) { // [b][s] -> [perm s][b]
    __shared__ float2 t[64][33];
    size_t s0 = (size_t)blockIdx.x * 32; int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int b = ty; b < B; b += 8) { size_t s = s0 + tx; if (s < N) t[b][tx] = in[b * N + s]; }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) { size_t s = s0 + i; if (s >= N) break; size_t row = (size_t)perm[s] * B; for (int b = tx; b < B; b += 32) q[row + b] = t[b][i]; }
}
#define CK(x) do { auto r = (x); if ((int)r) { printf("%s -> %d line %d\n", #x, (int)r, __LINE__); return 1; } } while (0)
int main() {
    const int T = 1536, P = 2048, B = 32, n = 64;
    const size_t N = (size_t)T * P;
    float* in; float2 *work, *q1, *q2; int* perm;
    CK(cudaMalloc(&in, 4 * N * n)); CK(cudaMalloc(&work, 8 * N * B)); CK(cudaMalloc(&q1, 8 * N * B)); CK(cudaMalloc(&q2, 8 * N * B)); CK(cudaMalloc(&perm, 4 * N));
    std::vector<float> h(N * n); std::mt19937 g(1); std::uniform_real_distribution<float> U(-1, 1); for (auto& v : h) v = U(g);
    CK(cudaMemcpy(in, h.data(), 4 * N * n, cudaMemcpyHostToDevice));
    std::vector<int> hp(N); for (size_t i = 0; i < N; ++i) hp[i] = (int)i; std::shuffle(hp.begin() + 0, hp.end(), g);
    // keep perm local-ish: shuffle within blocks of 4096 like patch grouping
    for (size_t i = 0; i < N; ++i) hp[i] = (int)i; for (size_t b0 = 0; b0 < N; b0 += 4096) std::shuffle(hp.begin() + b0, hp.begin() + std::min(N, b0 + 4096), g);
    CK(cudaMemcpy(perm, hp.data(), 4 * N, cudaMemcpyHostToDevice));
    // reference path: pack [b][t][p] -> cuFFT batch B*T -> perm
    cufftHandle p0; CK(cufftPlan1d(&p0, P, CUFFT_C2C, B * T));
    // callback path: layout [t][b][p]
    const char* fn = getenv("FB") ? getenv("FB") : "cb_dev.fatbin"; std::ifstream f(fn, std::ios::binary); std::vector<char> fb((std::istreambuf_iterator<char>(f)), {});
    printf("fatbin %zu bytes\n", fb.size());
    cufftHandle p1; CK(cufftCreate(&p1));
    CbInfo hci{in, n, T, P, B, perm, q2}; CbInfo* dci; CK(cudaMalloc(&dci, sizeof(CbInfo))); CK(cudaMemcpy(dci, &hci, sizeof(hci), cudaMemcpyHostToDevice));
    void* info = dci;
    CK(cufftXtSetJITCallback(p1, "cb_load_pack", fb.data(), fb.size(), CUFFT_CB_LD_COMPLEX, &info));
    CK(cufftXtSetJITCallback(p1, "cb_store_perm", fb.data(), fb.size(), CUFFT_CB_ST_COMPLEX, &info));
    size_t ws; auto tp0 = clock(); CK(cufftMakePlan1d(p1, P, CUFFT_C2C, B * T, &ws)); printf("plan %.1f s cpu\n", (clock() - tp0) / (double)CLOCKS_PER_SEC);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        pack<<<148 * 16, 256>>>(in, n, T, P, B, work); CK(cufftExecC2C(p0, work, work, CUFFT_FORWARD)); permk<<<(N + 31) / 32, 256>>>(work, perm, B, N, q1);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); printf("ref path %.3f ms\n", ms);
        cudaEventRecord(e0);
        CK(cufftExecC2C(p1, work, work, CUFFT_FORWARD));
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); printf("callback path %.3f ms\n", ms);
    }
    CK(cudaDeviceSynchronize());
    std::vector<float2> a(N * B), b(N * B); cudaMemcpy(a.data(), q1, 8 * N * B, cudaMemcpyDeviceToHost); cudaMemcpy(b.data(), q2, 8 * N * B, cudaMemcpyDeviceToHost);
    double d = 0, m = 0; for (size_t i = 0; i < a.size(); ++i) { d = std::max(d, (double)fabs(a[i].x - b[i].x) + fabs(a[i].y - b[i].y)); m = std::max(m, (double)fabs(a[i].x)); }
    printf("max diff %g (max %g)\n", d, m);
}
