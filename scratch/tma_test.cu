// standalone check of the 3-D TMA box load used by k_sh_tma
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
__global__ void k(const __grid_constant__ CUtensorMap tmap, int x0, int y0, unsigned long long* out, int n) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar;
    unsigned sbar = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sbar));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sbar), "r"(n * 8) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
            ::"r"((unsigned)__cvta_generic_to_shared(sm)), "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(x0), "r"(y0), "r"(0), "r"(sbar) : "memory");
    }
    __syncthreads();
    asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(sbar) : "memory");
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = ((unsigned long long*)sm)[i];
}
int main(int argc, char** argv) {
    int X = 64, Y = 64, B = argc > 1 ? atoi(argv[1]) : 1; int bx = argc > 2 ? atoi(argv[2]) : 10; int fl = argc > 3 ? atoi(argv[3]) : 0; int x0 = argc > 4 ? atoi(argv[4]) : -1; int y0 = argc > 5 ? atoi(argv[5]) : x0;
    std::vector<unsigned long long> h((size_t)X * Y * B);
    for (size_t i = 0; i < h.size(); ++i) h[i] = i + 1;
    unsigned long long *d, *o;
    cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 1 << 20);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void* f = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    CUtensorMap tm;
    int m = fl ? 2 : 1;
    cuuint64_t dims[3] = {(cuuint64_t)X * m, (cuuint64_t)Y, (cuuint64_t)B};
    cuuint64_t str[2] = {(cuuint64_t)X * 8, (cuuint64_t)X * Y * 8};
    cuuint32_t box[3] = {(cuuint32_t)(bx * m), 11, (cuuint32_t)B}, es[3] = {1, 1, 1};
    CUresult r = enc(&tm, fl ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d (q %d)\n", (int)r, (int)q);
    int n = bx * 11 * B;
    k<<<1, 128, n * 8>>>(tm, x0 * m, y0, o, n);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<unsigned long long> ho(n);
    cudaMemcpy(ho.data(), o, n * 8, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 12; ++i) printf("%llu ", ho[i]);
    printf("\n");
}
