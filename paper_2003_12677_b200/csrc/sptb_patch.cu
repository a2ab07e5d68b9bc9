// Patch-grouped S^H SpMM (radon direction) and the permuting transposes of
// the sample axis.
//
// Q[s'][b] = (sub ? sub - : ) sum_k v_k X[b][m_k]: every sample s' of a work
// item is centred in one PATCH_W x PATCH_W grid patch, so all its nonzeros
// fall in the patch box (patch + halo).  A CTA stages that box -- read
// directly from the batch-outer FFT2 output [b][y][x], no transpose pass --
// into shared memory as [b][cell] planes (odd plane stride: the lane-per-batch
// reads below are bank-conflict free), then a warp per sample accumulates its
// (cell, value) records from shared memory and writes the 8B-byte output row.
// Each grid value is fetched once per patch instead of once per touching
// nonzero (~5x fewer L2->SM bytes than a per-row gather), which is what lets
// the forward SpMM approach the HBM roofline.  Deterministic: the entry order
// within a row is the CSR order of gridding.py:179.
#include "sptb_internal.cuh"

#include <algorithm>

namespace sptb {

template <typename R> struct PCplx;
template <> struct PCplx<float> { using T = float2; };
template <> struct PCplx<double> { using T = double2; };

template <typename R>
struct alignas(16) PRec {
    unsigned cell, pad;
    typename PCplx<R>::T v;
};

constexpr int PT = 256;  // threads per CTA

__device__ __forceinline__ void pcp8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void pcp16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void pcp_wait() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// acc(lo, hi) += (s, s) * x(lo, hi): sm_100 packed FP32x2 FMA, scalar broadcast
__device__ __forceinline__ void ffma2s(unsigned long long& acc, float s, unsigned long long x) {
    asm("{\n .reg .b64 t;\n mov.b64 t, {%1, %1};\n fma.rn.f32x2 %0, t, %2, %0;\n}"
        : "+l"(acc) : "f"(s), "l"(x));
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
    return make_float2(__uint_as_float((unsigned)v), __uint_as_float((unsigned)(v >> 32)));
}

// G lanes per sample row, lane owns batch columns lig + G*q (q < CPL)
template <typename R, int G, int CPL, bool SUB>
__global__ void __launch_bounds__(PT)
k_sh_patch(const int4* __restrict__ items, const int* __restrict__ rp,
           const PRec<R>* __restrict__ meta, int npx, int bw, int halo, int X, int Y,
           long long M, const typename PCplx<R>::T* __restrict__ x,
           typename PCplx<R>::T* __restrict__ y, const typename PCplx<R>::T* __restrict__ sub) {
    using C = typename PCplx<R>::T;
    constexpr int BB = G * CPL, NG = PT / G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int cells = bw * bw;
    const int ps = cells | 1;  // odd plane stride
    C* xs = reinterpret_cast<C*>(smem_raw);                                      // [BB][ps]
    PRec<R>* s_meta = reinterpret_cast<PRec<R>*>(xs + ((BB * ps + 1) & ~1));     // [ne]
    __shared__ int s_rp[PATCH_ITEM_ROWS + 1];

    const int tid = threadIdx.x;
    const int4 it = items[blockIdx.x];
    const int pid = it.x, r0 = it.y, r1 = it.z, e0 = it.w;
    const int nr = r1 - r0;
    const int bx0 = (pid % npx) * PATCH_W - halo, by0 = (pid / npx) * PATCH_W - halo;

    // grid box -> shared memory: a warp walks planes b, its lanes walk the box
    // cells (coalesced along x).  Cell coordinates are computed once per lane.
    {
        constexpr int MAXI = 8;  // cells <= 256 (kernel width <= 9)
        const int warp = tid >> 5, lane = tid & 31;
        long long goff[MAXI];
        int soff[MAXI];
        unsigned inb = 0;
        const int ni = (cells + 31) >> 5;
#pragma unroll
        for (int i = 0; i < MAXI; ++i) {
            const int c = lane + 32 * i;
            const int ly = c / bw, lx = c - ly * bw;
            const int gx = bx0 + lx, gy = by0 + ly;
            soff[i] = c;
            goff[i] = (long long)gy * X + gx;
            if (i < ni && c < cells && gx >= 0 && gx < X && gy >= 0 && gy < Y) inb |= 1u << i;
        }
        for (int b = warp; b < BB; b += PT / 32) {
            const C* src = x + (size_t)b * M;
            C* dst = xs + b * ps;
#pragma unroll
            for (int i = 0; i < MAXI; ++i) {
                if (i >= ni) break;
                if (inb & (1u << i)) {
                    if (sizeof(C) == 8) pcp8(dst + soff[i], src + goff[i]);
                    else pcp16(dst + soff[i], src + goff[i]);
                } else if (soff[i] < cells) {
                    dst[soff[i]].x = 0;
                    dst[soff[i]].y = 0;
                }
            }
        }
    }
    for (int i = tid; i <= nr; i += PT) s_rp[i] = __ldg(rp + r0 + i) - e0;
    __syncthreads();
    const int ne = s_rp[nr];
    {   // (cell, value) records: contiguous, 16-byte chunks
        constexpr int RC = (int)sizeof(PRec<R>) / 16;
        const char* src = reinterpret_cast<const char*>(meta + e0);
        char* dst = reinterpret_cast<char*>(s_meta);
        for (int i = tid; i < ne * RC; i += PT) pcp16(dst + 16 * i, src + 16 * i);
    }
    pcp_wait();
    __syncthreads();

    const int g = tid / G, lig = tid % G;
    for (int r = g; r < nr; r += NG) {
        C acc[CPL];
        const int end = s_rp[r + 1];
        if constexpr (sizeof(C) == 8) {
            // complex64: records {byte offset, re, im, 0}; packed FP32x2 FMAs with
            // the value broadcast as a scalar operand (FFMA2 R.F32): re-part and
            // im-part accumulators, combined once per row
            const char* xl = reinterpret_cast<const char*>(xs) + (size_t)lig * ps * 8;
            const float4* m4 = reinterpret_cast<const float4*>(s_meta);
            unsigned long long arr[CPL], aii[CPL];
#pragma unroll
            for (int q = 0; q < CPL; ++q) arr[q] = aii[q] = 0ull;
#pragma unroll 3
            for (int k = s_rp[r]; k < end; ++k) {
                const float4 m = m4[k];
                const unsigned off = __float_as_uint(m.x);
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const unsigned long long xv =
                        *reinterpret_cast<const unsigned long long*>(xl + (size_t)q * G * ps * 8 + off);
                    ffma2s(arr[q], m.y, xv);
                    ffma2s(aii[q], m.z, xv);
                }
            }
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const float2 a = unpack2(arr[q]), b = unpack2(aii[q]);
                acc[q].x = a.x - b.y;
                acc[q].y = a.y + b.x;
            }
        } else {
#pragma unroll
            for (int q = 0; q < CPL; ++q) acc[q].x = acc[q].y = 0;
#pragma unroll 4
            for (int k = s_rp[r]; k < end; ++k) {
                const PRec<R> m = s_meta[k];
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    const C v = xs[(lig + G * q) * ps + m.cell];
                    acc[q].x = fma(m.v.x, v.x, acc[q].x);
                    acc[q].x = fma(-m.v.y, v.y, acc[q].x);
                    acc[q].y = fma(m.v.x, v.y, acc[q].y);
                    acc[q].y = fma(m.v.y, v.x, acc[q].y);
                }
            }
        }
        const size_t o = (size_t)(r0 + r) * BB;
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
            C out = acc[q];
            if (SUB) {
                const C sv = sub[o + lig + G * q];
                out.x = sv.x - out.x;
                out.y = sv.y - out.y;
            }
            y[o + lig + G * q] = out;
        }
    }
}

template <typename R, int G, int CPL>
static int sh_patch_dispatch(const sptb_plan* p, const void* x, void* y, const void* sub,
                             cudaStream_t st) {
    using C = typename PCplx<R>::T;
    const PatchSH& sp = p->shp;
    if (sp.n_items == 0) return SPTB_OK;
    constexpr int BB = G * CPL;
    const int cells = sp.bw * sp.bw, ps = cells | 1;
    const size_t sm = sizeof(C) * (size_t)((BB * ps + 1) & ~1) + sizeof(PRec<R>) * (size_t)sp.max_item_nnz;
    auto run = [&](auto kern) -> int {
        SPTB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        kern<<<(unsigned)sp.n_items, PT, sm, st>>>(sp.items, sp.rp, (const PRec<R>*)sp.meta, sp.npx,
                                                   sp.bw, sp.halo, p->X, p->Y, p->M, (const C*)x,
                                                   (C*)y, (const C*)sub);
        SPTB_LAUNCHED();
        return SPTB_OK;
    };
    if (sub) return run(k_sh_patch<R, G, CPL, true>);
    return run(k_sh_patch<R, G, CPL, false>);
}

template <typename R>
int launch_spmm_sh_patch(const sptb_plan* p, const void* x_bm, void* y_sb, int B, const void* sub,
                         cudaStream_t st) {
    switch (B) {
        case 1: return sh_patch_dispatch<R, 1, 1>(p, x_bm, y_sb, sub, st);
        case 2: return sh_patch_dispatch<R, 2, 1>(p, x_bm, y_sb, sub, st);
        case 4: return sh_patch_dispatch<R, 4, 1>(p, x_bm, y_sb, sub, st);
        case 8: return sh_patch_dispatch<R, 8, 1>(p, x_bm, y_sb, sub, st);
        case 16: return sh_patch_dispatch<R, 16, 1>(p, x_bm, y_sb, sub, st);
        case 32: return sh_patch_dispatch<R, 16, 2>(p, x_bm, y_sb, sub, st);
        case 64: return sh_patch_dispatch<R, 16, 4>(p, x_bm, y_sb, sub, st);
    }
    return fail(SPTB_ERR_ARG, "patch spmm: batch must be a power of two <= 64");
}
template int launch_spmm_sh_patch<float>(const sptb_plan*, const void*, void*, int, const void*, cudaStream_t);
template int launch_spmm_sh_patch<double>(const sptb_plan*, const void*, void*, int, const void*, cudaStream_t);

// ---------------------------------------------------------------------------
// Sample-axis transposes with the patch renumbering:
//   permute:   [b][s] -> [perm[s]][b]     (FFT1 output -> SpMM operand)
//   unpermute: [s'][b] -> [b][order[s']]  (SpMM output -> IFFT1 input)
// 32 samples x B columns per tile through shared memory; the scattered side
// moves whole B*sizeof(complex) rows.
// ---------------------------------------------------------------------------
template <typename C>
__global__ void __launch_bounds__(256) k_perm_bs_sb(const C* __restrict__ in, C* __restrict__ out,
                                                   const int* __restrict__ perm, int B, long long N) {
    __shared__ C t[64][33];
    const long long s0 = (long long)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int b = ty; b < B; b += 8) {
        const long long s = s0 + tx;
        if (s < N) t[b][tx] = in[(size_t)b * N + s];
    }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
        const long long s = s0 + i;
        if (s >= N) break;
        const size_t row = (size_t)perm[s] * B;
        for (int b = tx; b < B; b += 32) out[row + b] = t[b][i];
    }
}

template <typename C>
__global__ void __launch_bounds__(256) k_unperm_sb_bs(const C* __restrict__ in, C* __restrict__ out,
                                                     const int* __restrict__ order, int B, long long N) {
    __shared__ C t[64][33];
    const long long s0 = (long long)blockIdx.x * 32;  // s' tile
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int i = ty; i < 32; i += 8) {
        const long long s = s0 + i;
        if (s >= N) break;
        for (int b = tx; b < B; b += 32) t[b][i] = in[(size_t)s * B + b];
    }
    __syncthreads();
    for (int b = ty; b < B; b += 8) {
        const long long s = s0 + tx;
        if (s < N) out[(size_t)b * N + order[s]] = t[b][tx];
    }
}

template <typename R>
int launch_transpose_permute(const void* in_bs, void* out_sb, const int* perm, int B, int64_t N,
                             cudaStream_t st) {
    using C = typename PCplx<R>::T;
    if (B > 64) return fail(SPTB_ERR_ARG, "transpose: B > 64");
    k_perm_bs_sb<C><<<(unsigned)((N + 31) / 32), 256, 0, st>>>((const C*)in_bs, (C*)out_sb, perm, B, N);
    SPTB_LAUNCHED();
    return SPTB_OK;
}
template <typename R>
int launch_transpose_unpermute(const void* in_sb, void* out_bs, const int* order, int B, int64_t N,
                               cudaStream_t st) {
    using C = typename PCplx<R>::T;
    if (B > 64) return fail(SPTB_ERR_ARG, "transpose: B > 64");
    k_unperm_sb_bs<C><<<(unsigned)((N + 31) / 32), 256, 0, st>>>((const C*)in_sb, (C*)out_bs, order, B, N);
    SPTB_LAUNCHED();
    return SPTB_OK;
}
template int launch_transpose_permute<float>(const void*, void*, const int*, int, int64_t, cudaStream_t);
template int launch_transpose_permute<double>(const void*, void*, const int*, int, int64_t, cudaStream_t);
template int launch_transpose_unpermute<float>(const void*, void*, const int*, int, int64_t, cudaStream_t);
template int launch_transpose_unpermute<double>(const void*, void*, const int*, int, int64_t, cudaStream_t);

}  // namespace sptb
