// Micro-benchmark: TMA tile::gather4 of 256-byte rows (the S operand X[s][32]
// complex64) in the CSR order of S, vs per-lane LDG.128 gathers.  Built as a
// standalone .so (scratch/g4/build.sh) and driven from scratch/g4/g4.py.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

constexpr int STAGES = 4;
constexpr int CH = 64;  // rows per chunk (16 gather4)

__device__ __forceinline__ void wait_par(unsigned bar, unsigned par) {
    asm volatile("{\n .reg .pred p;\nW1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W1;\n}\n" ::"r"(bar), "r"(par) : "memory");
}

__global__ void __launch_bounds__(256) k_g4(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                            long long n, float* out) {
    extern __shared__ __align__(1024) unsigned char smem[];
    float4* buf = reinterpret_cast<float4*>(smem);  // [STAGES][CH][16]
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + STAGES * CH * 256);
    const long long nch = n / CH;
    const long long c0 = nch * blockIdx.x / gridDim.x, c1 = nch * (blockIdx.x + 1) / gridDim.x;
    unsigned bar[STAGES];
    for (int s = 0; s < STAGES; ++s) bar[s] = (unsigned)__cvta_generic_to_shared(bars + s);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar[s]));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](long long c, int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar[s]), "r"(CH * 256) : "memory");
        const int* ix = idx + c * CH;
        for (int g = 0; g < CH / 4; ++g) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(buf + (s * CH + g * 4) * 16);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
                "l"(reinterpret_cast<unsigned long long>(&tm)), "r"(0), "r"(ix[4 * g]), "r"(ix[4 * g + 1]), "r"(ix[4 * g + 2]),
                "r"(ix[4 * g + 3]), "r"(bar[s])
                : "memory");
        }
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES - 1 && c0 + s < c1; ++s) issue(c0 + s, s);
    float acc = 0.f;
    unsigned par = 0;
    for (long long c = c0; c < c1; ++c) {
        const int s = (int)((c - c0) % STAGES);
        if (threadIdx.x == 0 && c + STAGES - 1 < c1) issue(c + STAGES - 1, (s + STAGES - 1) % STAGES);
        wait_par(bar[s], (par >> s) & 1);
        par ^= 1u << s;
        const float4* b = buf + s * CH * 16;
        for (int k = threadIdx.x; k < CH * 16; k += 256) {
            const float4 v = b[k];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncthreads();
    }
    if (acc == 12345.f) out[0] = acc;
}

__global__ void __launch_bounds__(256) k_ldg(const float4* __restrict__ x, const int* __restrict__ idx, long long n,
                                             float* out) {
    const int h = threadIdx.x >> 4, l = threadIdx.x & 15;
    float acc = 0.f;
    const long long halves = (long long)gridDim.x * 16;
    for (long long j0 = (blockIdx.x * 16LL + h) * 8; j0 < n; j0 += halves * 8) {
        float4 q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) q[u] = j0 + u < n ? __ldg(x + (size_t)idx[j0 + u] * 16 + l) : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += q[u].x + q[u].y + q[u].z + q[u].w;
    }
    if (acc == 12345.f) out[0] = acc;
}

// warp per row: each LDG touches one 128-byte line (LDG.32, 2 per row) or two (LDG.64, 1 per row)
template <int MODE>
__global__ void __launch_bounds__(256) k_ldgw(const float* __restrict__ x, const int* __restrict__ idx, long long n,
                                              float* out) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * 8, w0 = blockIdx.x * 8LL + (threadIdx.x >> 5);
    float acc = 0.f;
    for (long long j0 = w0 * 8; j0 < n; j0 += warps * 8) {
        if (MODE == 0) {
            float a[8], b[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const float* r = x + (size_t)idx[j0 + u] * 64;
                a[u] = __ldg(r + lane);
                b[u] = __ldg(r + 32 + lane);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += a[u] + b[u];
        } else {
            float2 a[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u] = __ldg(reinterpret_cast<const float2*>(x + (size_t)idx[j0 + u] * 64) + lane);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += a[u].x + a[u].y;
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

extern "C" int g4_run(const void* x, long long nrows, const int* idx, long long n, int mode, int grid, float* ms) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess) return -1;
        enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    }
    CUtensorMap tm;
    cuuint64_t dims[2] = {32, (cuuint64_t)nrows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {32, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(x), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return -2;
    float* out;
    cudaMalloc(&out, 4);
    const int sm = STAGES * CH * 256 + STAGES * 8;
    cudaFuncSetAttribute(k_g4, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k_g4<<<grid, 256, sm>>>(tm, idx, n, out);
        else if (mode == 1) k_ldg<<<grid, 256>>>((const float4*)x, idx, n, out);
        else if (mode == 2) k_ldgw<0><<<grid, 256>>>((const float*)x, idx, n, out);
        else k_ldgw<1><<<grid, 256>>>((const float*)x, idx, n, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    cudaFree(out);
    return e == cudaSuccess ? 0 : (int)e;
}
