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

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

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

__device__ __forceinline__ void pcp16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// acc(lo, hi) += (s, s) * x(lo, hi): sm_100 packed FP32x2 FMA, scalar broadcast
__device__ __forceinline__ void ffma2s(unsigned long long& acc, float s, unsigned long long x) {
    asm("{\n .reg .b64 t;\n mov.b64 t, {%1, %1};\n fma.rn.f32x2 %0, t, %2, %0;\n}"
        : "+l"(acc) : "f"(s), "l"(x));
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
    return make_float2(__uint_as_float((unsigned)v), __uint_as_float((unsigned)(v >> 32)));
}

__device__ __forceinline__ void pcp4(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void pcp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void pcp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Shared-memory stage of one work item: box planes [BB][ps] | records | row pointers
struct PatchStage {
    int meta_off, rp_off, bytes;
};
template <typename R>
__host__ __device__ inline PatchStage patch_stage(int BB, int bw, int max_item_nnz) {
    using C = typename PCplx<R>::T;
    const int ps = (bw * bw) | 1;
    PatchStage s;
    s.meta_off = (int)(((size_t)BB * ps * sizeof(C) + 15) & ~(size_t)15);
    s.rp_off = s.meta_off + (int)sizeof(PRec<R>) * max_item_nnz;
    s.bytes = (s.rp_off + 4 * (PATCH_ITEM_ROWS + 1) + 127) & ~127;
    return s;
}

template <int SZ>
__device__ __forceinline__ void pcp_el(unsigned dst, const void* src) {
    if constexpr (SZ == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src));
    else
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}

// Persistent CTAs walk the work items with a two-stage cp.async pipeline: the
// box, records and row pointers of item i+1 are in flight while item i is
// computed (one item per CTA and a single stage when the grid covers all
// items).  G lanes per sample row, lane owns batch columns lig + G*q.  BWT is
// the box width when known at compile time (10 for the width-3 kernel), else 0.
template <typename R, int G, int CPL, bool SUB, int BWT>
__global__ void __launch_bounds__(PT)
k_sh_patch(const int4* __restrict__ items, int n_items, const int* __restrict__ rp,
           const PRec<R>* __restrict__ meta, int npx, int bw_rt, int halo, int X, int Y,
           long long M, const typename PCplx<R>::T* __restrict__ x,
           typename PCplx<R>::T* __restrict__ y, const typename PCplx<R>::T* __restrict__ sub,
           PatchStage sg) {
    using C = typename PCplx<R>::T;
    constexpr int BB = G * CPL, NG = PT / G, NW = PT / 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int bw = BWT > 0 ? BWT : bw_rt;
    const int cells = bw * bw;
    const int ps = cells | 1;  // odd plane stride: lane-per-plane reads are conflict free
    const int nsl = (cells + 31) >> 5;  // 32-cell slots of the box
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // stage one item.  Box cells outside the grid are never referenced by a
    // record (the matrix has no entries there), so their coordinates are just
    // clamped.  Each warp takes (slot, plane group) units: a lane copies its
    // cell of PGS planes.
    auto issue = [&](const int4 d, const int e1, unsigned char* st) {
        constexpr int PGS = BB < 8 ? BB : 8, NPG = BB / PGS;
        const unsigned xs0 = (unsigned)__cvta_generic_to_shared(st);
        const int bx0 = (d.x % npx) * PATCH_W - halo, by0 = (d.x / npx) * PATCH_W - halo;
        for (int u = warp; u < nsl * NPG; u += NW) {
            const int pg = u / nsl, sl = u - pg * nsl;
            const int c = sl * 32 + lane;
            if (c < cells) {
                const int ly = c / bw, lx = c - ly * bw;
                const int gx = min(max(bx0 + lx, 0), X - 1), gy = min(max(by0 + ly, 0), Y - 1);
                const C* src = x + (size_t)(pg * PGS) * M + ((size_t)gy * X + gx);
                const unsigned dst = xs0 + (unsigned)(((pg * PGS) * ps + c) * (int)sizeof(C));
#pragma unroll
                for (int j = 0; j < PGS; ++j)
                    pcp_el<sizeof(C)>(dst + (unsigned)(j * ps * (int)sizeof(C)), src + (size_t)j * M);
            }
        }
        int* srp = reinterpret_cast<int*>(st + sg.rp_off);
        const int nr = d.z - d.y;
        for (int i = tid; i <= nr; i += PT) pcp4(srp + i, rp + d.y + i);
        constexpr int RC = (int)sizeof(PRec<R>) / 16;
        const char* msrc = reinterpret_cast<const char*>(meta + d.w);
        char* mdst = reinterpret_cast<char*>(st + sg.meta_off);
        const int nc = (e1 - d.w) * RC;
        for (int i = tid; i < nc; i += PT) pcp16(mdst + 16 * i, msrc + 16 * i);
    };

    int it = blockIdx.x;
    if (it >= n_items) return;
    int4 d = items[it];
    int e1 = __ldg(rp + d.z);
    issue(d, e1, smem_raw);
    pcp_commit();
    int nx = it + gridDim.x;
    int4 dn = make_int4(0, 0, 0, 0);
    int e1n = 0;
    if (nx < n_items) {
        dn = items[nx];
        e1n = __ldg(rp + dn.z);
    }
    int s = 0;
    const int g = tid / G, lig = tid % G;
    while (true) {
        if (nx < n_items) issue(dn, e1n, smem_raw + (s ^ 1) * sg.bytes);
        pcp_commit();
        const int nn = nx + gridDim.x;
        int4 dnn = make_int4(0, 0, 0, 0);
        int e1nn = 0;
        if (nn < n_items) {
            dnn = items[nn];
            e1nn = __ldg(rp + dnn.z);
        }
        pcp_wait1();
        __syncthreads();

        unsigned char* st = smem_raw + s * sg.bytes;
        const C* xs = reinterpret_cast<const C*>(st);
        const int* srp = reinterpret_cast<const int*>(st + sg.rp_off);
        const int r0 = d.y, nr = d.z - d.y, e0 = d.w;
        for (int r = g; r < nr; r += NG) {
            C acc[CPL];
            const int beg = srp[r] - e0, n = srp[r + 1] - e0 - beg;
            if constexpr (sizeof(C) == 8) {
                // complex64: records {byte offset, re, im, 0}; packed FP32x2 FMAs
                // (FFMA2 with the value broadcast): re-part and im-part
                // accumulators, combined once per row
                const char* xq[CPL];
#pragma unroll
                for (int q = 0; q < CPL; ++q)
                    xq[q] = reinterpret_cast<const char*>(xs + (lig + q * G) * ps);
                const float4* m4 = reinterpret_cast<const float4*>(st + sg.meta_off) + beg;
                float2 arr[CPL], aii[CPL];
#pragma unroll
                for (int q = 0; q < CPL; ++q) arr[q] = aii[q] = make_float2(0.f, 0.f);
                auto step = [&](const float4 m) {
                    const unsigned off = __float_as_uint(m.x);
#pragma unroll
                    for (int q = 0; q < CPL; ++q) {
                        const float2 xv = *reinterpret_cast<const float2*>(xq[q] + off);
                        arr[q] = __ffma2_rn(make_float2(m.y, m.y), xv, arr[q]);
                        aii[q] = __ffma2_rn(make_float2(m.z, m.z), xv, aii[q]);
                    }
                };
                if (n <= 9) {
                    // a 3x3 stencil row (every row of the width-3 kernel): fully
                    // unrolled, record loads issued up front
                    float4 mm[9];
#pragma unroll
                    for (int k = 0; k < 9; ++k)
                        if (k < n) mm[k] = m4[k];
#pragma unroll
                    for (int k = 0; k < 9; ++k)
                        if (k < n) step(mm[k]);
                } else {
#pragma unroll 3
                    for (int k = 0; k < n; ++k) step(m4[k]);
                }
#pragma unroll
                for (int q = 0; q < CPL; ++q) {
                    acc[q].x = arr[q].x - aii[q].y;
                    acc[q].y = arr[q].y + aii[q].x;
                }
            } else {
                const PRec<R>* sm = reinterpret_cast<const PRec<R>*>(st + sg.meta_off) + beg;
#pragma unroll
                for (int q = 0; q < CPL; ++q) acc[q].x = acc[q].y = 0;
#pragma unroll 4
                for (int k = 0; k < n; ++k) {
                    const PRec<R> m = sm[k];
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
        if (nx >= n_items) break;
        __syncthreads();  // stage s is refilled by the next iteration's issue
        it = nx;
        nx = nn;
        d = dn;
        e1 = e1n;
        dn = dnn;
        e1n = e1nn;
        s ^= 1;
    }
}

// ---------------------------------------------------------------------------
// Slot-mode S^H (kernel width 3): one CTA per work item (<= PATCH_ITEM_ROWS
// samples of one patch).  Stage the 10x10 box of all BB planes and the
// items's rows (9 value slots + base cell, 80 B per row for complex64), then a
// group of G lanes per row accumulates the 9 slots: the box cell of slot k is
// base + (k / 3) * 10 + k % 3, an immediate offset from the row's base.
// Per nonzero and batch column that is one shared-memory read of the grid
// value and a broadcast of the slot value -- 3 shared wavefronts per
// row-nonzero (vs 4 with per-nonzero index records) and 8 B per nonzero from
// HBM for the matrix.
// ---------------------------------------------------------------------------
constexpr int SLOT_BW = PATCH_W + 2;
constexpr int SLOT_PS = SLOT_BW * SLOT_BW + 1;  // odd plane stride

#ifndef SPTB_SH_MINB
#define SPTB_SH_MINB 4
#endif
template <typename R, int G, int CPL, bool SUB>
__global__ void __launch_bounds__(PT, SPTB_SH_MINB)
k_sh_slot(const int4* __restrict__ items, int n_items, const typename PCplx<R>::T* __restrict__ sval,
          int npx, int X, int Y, long long M, const typename PCplx<R>::T* __restrict__ x,
          typename PCplx<R>::T* __restrict__ y, const typename PCplx<R>::T* __restrict__ sub,
          int stage_bytes) {
    using C = typename PCplx<R>::T;
    constexpr int BB = G * CPL, NG = PT / G, NW = PT / 32;
    constexpr int CELLS = SLOT_BW * SLOT_BW, NSL = (CELLS + 31) / 32;
    constexpr int XS_BYTES = (BB * SLOT_PS * (int)sizeof(C) + 15) & ~15;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // stage an item: the box through (slot, plane group) units per warp (cells
    // outside the grid are clamped: no slot of a regular row points at them
    // with a nonzero), the rows as contiguous 16-byte chunks
    auto issue = [&](const int4 d, unsigned char* st) {
        constexpr int PGS = BB < 8 ? BB : 8, NPG = BB / PGS;
        const unsigned xs0 = (unsigned)__cvta_generic_to_shared(st);
        const int bx0 = (d.x % npx) * PATCH_W, by0 = (d.x / npx) * PATCH_W - 1;  // slot-mode patch origin
#pragma unroll
        for (int u = warp; u < NSL * NPG; u += NW) {
            const int pg = u / NSL, sl = u - pg * NSL;
            const int c = sl * 32 + lane;
            if (c < CELLS) {
                const int ly = c / SLOT_BW, lx = c - ly * SLOT_BW;
                const int gx = min(max(bx0 + lx, 0), X - 1), gy = min(max(by0 + ly, 0), Y - 1);
                const C* src = x + (size_t)(pg * PGS) * M + ((size_t)gy * X + gx);
                const unsigned dst = xs0 + (unsigned)(((pg * PGS) * SLOT_PS + c) * (int)sizeof(C));
#pragma unroll
                for (int j = 0; j < PGS; ++j)
                    pcp_el<sizeof(C)>(dst + (unsigned)(j * SLOT_PS * (int)sizeof(C)), src + (size_t)j * M);
            }
        }
        const char* s8 = reinterpret_cast<const char*>(sval + (size_t)d.y * SLOT_STRIDE);
        char* d8 = reinterpret_cast<char*>(st + XS_BYTES);
        const int nc = (d.z - d.y) * SLOT_STRIDE * (int)sizeof(C) / 16;
        for (int i = tid; i < nc; i += PT) pcp16(d8 + 16 * i, s8 + 16 * i);
    };

    int it = blockIdx.x;
    if (it >= n_items) return;
    int4 d = items[it];
    issue(d, smem_raw);
    pcp_commit();
    int nx = it + gridDim.x;
    int4 dn = make_int4(0, 0, 0, 0);
    if (nx < n_items) dn = items[nx];
    int s = 0;
    const int g = tid / G, lig = tid % G;
    while (true) {
        if (nx < n_items) issue(dn, smem_raw + (s ^ 1) * stage_bytes);
        pcp_commit();
        const int nn = nx + gridDim.x;
        int4 dnn = make_int4(0, 0, 0, 0);
        if (nn < n_items) dnn = items[nn];
        pcp_wait1();
        __syncthreads();
        const unsigned char* stg = smem_raw + s * stage_bytes;
        const C* xs = reinterpret_cast<const C*>(stg);
        const C* rows = reinterpret_cast<const C*>(stg + XS_BYTES);
        const int r0 = d.y, nr = d.z - d.y;
    for (int r = g; r < nr; r += NG) {
        const C* rv = rows + r * SLOT_STRIDE;
        C acc[CPL];
        if constexpr (sizeof(C) == 8) {
            const float4* r4 = reinterpret_cast<const float4*>(rv);
            const float4 v89 = r4[4];
            const int base = __float_as_int(v89.z);  // slot 9 .x
            float4 vv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) vv[i] = r4[i];
            const float vre[9] = {vv[0].x, vv[0].z, vv[1].x, vv[1].z, vv[2].x, vv[2].z, vv[3].x, vv[3].z, v89.x};
            const float vim[9] = {vv[0].y, vv[0].w, vv[1].y, vv[1].w, vv[2].y, vv[2].w, vv[3].y, vv[3].w, v89.y};
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const float2* xq = reinterpret_cast<const float2*>(xs + (lig + q * G) * SLOT_PS + base);
                float2 arr = make_float2(0.f, 0.f), aii = make_float2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    const float2 xv = xq[(k / 3) * SLOT_BW + k % 3];
                    arr = __ffma2_rn(make_float2(vre[k], vre[k]), xv, arr);
                    aii = __ffma2_rn(make_float2(vim[k], vim[k]), xv, aii);
                }
                acc[q].x = arr.x - aii.y;
                acc[q].y = arr.y + aii.x;
            }
        } else {
            const int base = (int)__double_as_longlong(rv[9].x);
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const C* xq = xs + (lig + q * G) * SLOT_PS + base;
                C a;
                a.x = a.y = 0;
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    const C v = rv[k], xv = xq[(k / 3) * SLOT_BW + k % 3];
                    a.x = fma(v.x, xv.x, a.x);
                    a.x = fma(-v.y, xv.y, a.x);
                    a.y = fma(v.x, xv.y, a.y);
                    a.y = fma(v.y, xv.x, a.y);
                }
                acc[q] = a;
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
        if (nx >= n_items) break;
        __syncthreads();  // stage s is refilled by the next iteration's issue
        nx = nn;
        d = dn;
        dn = dnn;
        s ^= 1;
    }
}

// irregular slot-mode rows [r_begin, N): direct gathers from the batch-outer
// grid through the original S^H CSR (a handful of rows whose stencil centre
// lies outside the grid)
template <typename R, bool SUB>
__global__ void __launch_bounds__(256)
k_sh_rows(const int* __restrict__ order, const int* __restrict__ rp, const int* __restrict__ col,
          const typename PCplx<R>::T* __restrict__ val, long long r_begin, long long N, int B,
          long long M, const typename PCplx<R>::T* __restrict__ x,
          typename PCplx<R>::T* __restrict__ y, const typename PCplx<R>::T* __restrict__ sub,
          int sample_order) {
    using C = typename PCplx<R>::T;
    const long long n = (N - r_begin) * B;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const long long r = r_begin + e / B;
        const int b = (int)(e % B);
        const int s = order[r];
        C a;
        a.x = a.y = 0;
        for (int k = rp[s]; k < rp[s + 1]; ++k) {
            const C v = val[k], xv = x[(size_t)b * M + col[k]];
            a.x = fma(v.x, xv.x, a.x);
            a.x = fma(-v.y, xv.y, a.x);
            a.y = fma(v.x, xv.y, a.y);
            a.y = fma(v.y, xv.x, a.y);
        }
        const size_t o = (size_t)(sample_order ? s : r) * B + b;
        if (SUB) {
            const C sv = sub[o];
            a.x = sv.x - a.x;
            a.y = sv.y - a.y;
        }
        y[o] = a;
    }
}

// ---------------------------------------------------------------------------
// TMA slot-mode S^H.  One elected thread stages the item with two bulk
// copies completing on one mbarrier: the 10 x 11 x BB box of the batch-outer
// grid through a 3-D tensor map (zero fill outside the grid) and the item's
// slot rows (contiguous).  No per-lane copy instructions (LDGSTS held the MIO
// queue for ~1/3 of the kernel).  The dense box has an even plane stride
// (110 cells), so lanes read planes lig + 8q with G = 8 lanes per row, and the
// build alternates block-origin parity between the two rows that share a
// half-warp: their cells differ in parity, which makes the 16 reads of a
// half-warp hit 16 distinct 8-byte bank pairs.
// ---------------------------------------------------------------------------
static_assert(PATCH_ITEM_ROWS % 16 == 0 && PATCH_ITEM_ROWS <= 256, "item rows: u8 hand-out order, 16-byte copies");
constexpr int TMA_BY = SLOT_BW + 1;             // box rows (one spare)
constexpr int TMA_PS = SLOT_BW * TMA_BY;        // plane stride in cells

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}

#ifndef SPTB_TMA_MINB
#define SPTB_TMA_MINB 5
#endif
template <typename R, int G, int CPL, bool SUB>
__global__ void __launch_bounds__(PT, SPTB_TMA_MINB)
k_sh_tma(const __grid_constant__ CUtensorMap tmap, const int4* __restrict__ items,
         const unsigned char* __restrict__ item_perm, const typename PCplx<R>::T* __restrict__ sval, int npx,
         typename PCplx<R>::T* __restrict__ y, const typename PCplx<R>::T* __restrict__ sub,
         const int* __restrict__ rowmap) {
    using C = typename PCplx<R>::T;
    constexpr int BB = G * CPL, NG = PT / G;
    constexpr int XS_BYTES = (BB * TMA_PS * (int)sizeof(C) + 127) & ~127;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) unsigned long long bar;
    const C* xs = reinterpret_cast<const C*>(smem_raw);
    const C* rows = reinterpret_cast<const C*>(smem_raw + XS_BYTES);
    const unsigned char* sperm = smem_raw + XS_BYTES + PATCH_ITEM_ROWS * SLOT_STRIDE * (int)sizeof(C);
    const int tid = threadIdx.x;
    const int4 d = items[blockIdx.x];
    const int r0 = d.y, nr = d.z - d.y;
    const unsigned sbar = (unsigned)__cvta_generic_to_shared(&bar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sbar));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        const unsigned box_bytes = BB * TMA_PS * (unsigned)sizeof(C);
        const unsigned row_bytes = (unsigned)(nr * SLOT_STRIDE * (int)sizeof(C));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sbar),
                     "r"(box_bytes + row_bytes + PATCH_ITEM_ROWS) : "memory");
        const int bx0 = (d.x % npx) * PATCH_W, by0 = (d.x / npx) * PATCH_W - 1;  // slot-mode patch origin
        const int ex = (int)sizeof(C) / 8;  // 8-byte tensor elements per complex
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(smem_raw)),
            "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(bx0 * ex), "r"(by0), "r"(0), "r"(sbar)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                (unsigned)__cvta_generic_to_shared(smem_raw + XS_BYTES)),
            "l"(sval + (size_t)r0 * SLOT_STRIDE), "r"(row_bytes), "r"(sbar)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                (unsigned)__cvta_generic_to_shared(sperm)),
            "l"(item_perm + (size_t)blockIdx.x * PATCH_ITEM_ROWS), "r"(PATCH_ITEM_ROWS), "r"(sbar)
            : "memory");
    }
    __syncthreads();
    mbar_wait(sbar, 0);

    const int g = tid / G, lig = tid % G;
    for (int rr = g; rr < nr; rr += NG) {
        const int r = sperm[rr];
        const C* rv = rows + r * SLOT_STRIDE;
        C acc[CPL];
        if constexpr (sizeof(C) == 8) {
            const float4* r4 = reinterpret_cast<const float4*>(rv);
            const float4 v89 = r4[4];
            const int base = __float_as_int(v89.z);  // slot 9 .x (row-major cell in a 10-wide box)
            float4 vv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) vv[i] = r4[i];
            const float vre[9] = {vv[0].x, vv[0].z, vv[1].x, vv[1].z, vv[2].x, vv[2].z, vv[3].x, vv[3].z, v89.x};
            const float vim[9] = {vv[0].y, vv[0].w, vv[1].y, vv[1].w, vv[2].y, vv[2].w, vv[3].y, vv[3].w, v89.y};
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const float2* xq = reinterpret_cast<const float2*>(xs + (lig + q * G) * TMA_PS + base);
                float2 arr = make_float2(0.f, 0.f), aii = make_float2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    const float2 xv = xq[(k / 3) * SLOT_BW + k % 3];
                    arr = __ffma2_rn(make_float2(vre[k], vre[k]), xv, arr);
                    aii = __ffma2_rn(make_float2(vim[k], vim[k]), xv, aii);
                }
                acc[q].x = arr.x - aii.y;
                acc[q].y = arr.y + aii.x;
            }
        } else {
            const int base = (int)__double_as_longlong(rv[9].x);
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const C* xq = xs + (lig + q * G) * TMA_PS + base;
                C a;
                a.x = a.y = 0;
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    const C v = rv[k], xv = xq[(k / 3) * SLOT_BW + k % 3];
                    a.x = fma(v.x, xv.x, a.x);
                    a.x = fma(-v.y, xv.y, a.x);
                    a.y = fma(v.x, xv.y, a.y);
                    a.y = fma(v.y, xv.x, a.y);
                }
                acc[q] = a;
            }
        }
        // rowmap (order: s' -> s): rows in sample order for the fused inverse FFT1
        const size_t o = (size_t)(rowmap ? __ldg(rowmap + r0 + r) : r0 + r) * BB;
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

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {  // shared with sptb_fft.cu
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)f;
    }();
    return fn;
}

// TMA path usable: 16-byte aligned operand and row/plane strides
bool tma_ok(const sptb_plan* p, const void* x) {
    const size_t cs = p->csize;
    return p->shp.slot_mode && tmap_encoder() != nullptr && ((uintptr_t)x % 16) == 0 &&
           ((size_t)p->X * cs) % 16 == 0 && ((size_t)p->M * cs) % 16 == 0 && !switches().no_tma;
}

template <typename R, int G, int CPL>
static int sh_tma_dispatch(const sptb_plan* p, const void* x, void* y, const void* sub, cudaStream_t st,
                           bool sample_order) {
    using C = typename PCplx<R>::T;
    const PatchSH& sp = p->shp;
    constexpr int BB = G * CPL;
    constexpr int XS_BYTES = (BB * TMA_PS * (int)sizeof(C) + 127) & ~127;
    const size_t sm = XS_BYTES + (size_t)PATCH_ITEM_ROWS * SLOT_STRIDE * sizeof(C) + PATCH_ITEM_ROWS;
    if (sp.n_items > 0) {
        const int ex = (int)sizeof(C) / 8;
        CUtensorMap tm;
        const cuuint64_t dims[3] = {(cuuint64_t)p->X * ex, (cuuint64_t)p->Y, (cuuint64_t)BB};
        const cuuint64_t strides[2] = {(cuuint64_t)p->X * sizeof(C), (cuuint64_t)p->M * sizeof(C)};
        const cuuint32_t box[3] = {(cuuint32_t)(SLOT_BW * ex), (cuuint32_t)TMA_BY, (cuuint32_t)BB};
        const cuuint32_t es[3] = {1, 1, 1};
        const CUresult cr = tmap_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(x), dims,
                                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return fail(SPTB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
        auto run = [&](auto kern) -> int {
            SPTB_CUDA(set_smem_once((const void*)kern, (int)sm));
            kern<<<(unsigned)sp.n_items, PT, sm, st>>>(tm, sp.items, sp.item_perm, (const C*)sp.sval, sp.npx,
                                                       (C*)y, (const C*)sub, sample_order ? sp.order : nullptr);
            SPTB_LAUNCHED();
            return SPTB_OK;
        };
        if (sub) SPTB_TRY(run(k_sh_tma<R, G, CPL, true>));
        else SPTB_TRY(run(k_sh_tma<R, G, CPL, false>));
    }
    if (sp.n_reg < p->N) {
        const long long n = (p->N - sp.n_reg) * BB;
        const unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 8);
        if (sub)
            k_sh_rows<R, true><<<grid, 256, 0, st>>>(sp.order, p->SH.row_ptr, p->SH.col, (const C*)p->SH.val,
                                                     sp.n_reg, p->N, BB, p->M, (const C*)x, (C*)y, (const C*)sub, sample_order ? 1 : 0);
        else
            k_sh_rows<R, false><<<grid, 256, 0, st>>>(sp.order, p->SH.row_ptr, p->SH.col, (const C*)p->SH.val,
                                                      sp.n_reg, p->N, BB, p->M, (const C*)x, (C*)y, (const C*)sub, sample_order ? 1 : 0);
        SPTB_LAUNCHED();
    }
    return SPTB_OK;
}

template <typename R, int G, int CPL>
static int sh_slot_dispatch(const sptb_plan* p, const void* x, void* y, const void* sub,
                            cudaStream_t st) {
    using C = typename PCplx<R>::T;
    const PatchSH& sp = p->shp;
    constexpr int BB = G * CPL;
    constexpr int XS_BYTES = (BB * SLOT_PS * (int)sizeof(C) + 15) & ~15;
    const size_t sm = XS_BYTES + (size_t)PATCH_ITEM_ROWS * SLOT_STRIDE * sizeof(C);
    if (sp.n_items > 0) {
        // one item per CTA (measured faster here than a persistent two-stage pipeline)
        constexpr bool one_per_cta = true;
        const int stage = (int)((sm + 127) & ~(size_t)127);
        const size_t smt = one_per_cta ? sm : 2 * (size_t)stage;
        auto run = [&](auto kern) -> int {
            SPTB_CUDA(set_smem_once((const void*)kern, (int)smt));
            int per_sm = 1, nsm = 148;
            SPTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PT, smt));
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device);
            const long long grid = one_per_cta ? sp.n_items
                                               : std::min<long long>(sp.n_items, (long long)nsm * std::max(per_sm, 1));
            kern<<<(unsigned)grid, PT, smt, st>>>(sp.items, (int)sp.n_items, (const C*)sp.sval, sp.npx, p->X,
                                                  p->Y, p->M, (const C*)x, (C*)y, (const C*)sub, stage);
            SPTB_LAUNCHED();
            return SPTB_OK;
        };
        if (sub) SPTB_TRY(run(k_sh_slot<R, G, CPL, true>));
        else SPTB_TRY(run(k_sh_slot<R, G, CPL, false>));
    }
    if (sp.n_reg < p->N) {
        const long long n = (p->N - sp.n_reg) * BB;
        const unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 8);
        if (sub)
            k_sh_rows<R, true><<<grid, 256, 0, st>>>(sp.order, p->SH.row_ptr, p->SH.col, (const C*)p->SH.val,
                                                     sp.n_reg, p->N, BB, p->M, (const C*)x, (C*)y, (const C*)sub, 0);
        else
            k_sh_rows<R, false><<<grid, 256, 0, st>>>(sp.order, p->SH.row_ptr, p->SH.col, (const C*)p->SH.val,
                                                      sp.n_reg, p->N, BB, p->M, (const C*)x, (C*)y, (const C*)sub, 0);
        SPTB_LAUNCHED();
    }
    return SPTB_OK;
}

template <typename R, int G, int CPL>
static int sh_patch_dispatch(const sptb_plan* p, const void* x, void* y, const void* sub,
                             cudaStream_t st) {
    using C = typename PCplx<R>::T;
    const PatchSH& sp = p->shp;
    if (sp.n_items == 0) return SPTB_OK;
    constexpr int BB = G * CPL;
    const PatchStage sg = patch_stage<R>(BB, sp.bw, sp.max_item_nnz);
    // persistent two-stage pipeline
    constexpr bool one_per_cta = false;
    const size_t sm = (one_per_cta ? 1 : 2) * (size_t)sg.bytes;
    auto run = [&](auto kern) -> int {
        static int dev_cached = -1, per_sm = 0;
        static size_t sm_cached = 0;
        if (dev_cached != p->device || sm_cached != sm) {
            SPTB_CUDA(set_smem_once((const void*)kern, (int)sm));
            SPTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PT, sm));
            dev_cached = p->device;
            sm_cached = sm;
        }
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device);
        const long long grid = one_per_cta ? sp.n_items
                                           : std::min<long long>(sp.n_items, (long long)nsm * std::max(per_sm, 1));
        kern<<<(unsigned)grid, PT, sm, st>>>(sp.items, (int)sp.n_items, sp.rp, (const PRec<R>*)sp.meta,
                                             sp.npx, sp.bw, sp.halo, p->X, p->Y, p->M, (const C*)x,
                                             (C*)y, (const C*)sub, sg);
        SPTB_LAUNCHED();
        return SPTB_OK;
    };
    if (sp.bw == 10) {
        if (sub) return run(k_sh_patch<R, G, CPL, true, 10>);
        return run(k_sh_patch<R, G, CPL, false, 10>);
    }
    if (sub) return run(k_sh_patch<R, G, CPL, true, 0>);
    return run(k_sh_patch<R, G, CPL, false, 0>);
}
template <typename R>
int launch_spmm_sh_patch(const sptb_plan* p, const void* x_bm, void* y_sb, int B, const void* sub,
                         cudaStream_t st, bool sample_order) {
    if (sample_order && (sub || !tma_ok(p, x_bm)))
        return fail(SPTB_ERR_STATE, "patch spmm: sample-order output needs the TMA path");
    if (tma_ok(p, x_bm)) switch (B) {
        case 1: return sh_tma_dispatch<R, 1, 1>(p, x_bm, y_sb, sub, st, sample_order);
        case 2: return sh_tma_dispatch<R, 2, 1>(p, x_bm, y_sb, sub, st, sample_order);
        case 4: return sh_tma_dispatch<R, 4, 1>(p, x_bm, y_sb, sub, st, sample_order);
        case 8: return sh_tma_dispatch<R, 8, 1>(p, x_bm, y_sb, sub, st, sample_order);
        case 16: return sh_tma_dispatch<R, 8, 2>(p, x_bm, y_sb, sub, st, sample_order);
        case 32: return sh_tma_dispatch<R, 8, 4>(p, x_bm, y_sb, sub, st, sample_order);
        case 64: return sh_tma_dispatch<R, 8, 8>(p, x_bm, y_sb, sub, st, sample_order);
        default: return fail(SPTB_ERR_ARG, "patch spmm: batch must be a power of two <= 64");
    }
    if (p->shp.slot_mode) switch (B) {
        case 1: return sh_slot_dispatch<R, 1, 1>(p, x_bm, y_sb, sub, st);
        case 2: return sh_slot_dispatch<R, 2, 1>(p, x_bm, y_sb, sub, st);
        case 4: return sh_slot_dispatch<R, 4, 1>(p, x_bm, y_sb, sub, st);
        case 8: return sh_slot_dispatch<R, 8, 1>(p, x_bm, y_sb, sub, st);
        case 16: return sh_slot_dispatch<R, 16, 1>(p, x_bm, y_sb, sub, st);
        case 32: return sh_slot_dispatch<R, 16, 2>(p, x_bm, y_sb, sub, st);
        case 64: return sh_slot_dispatch<R, 16, 4>(p, x_bm, y_sb, sub, st);
        default: return fail(SPTB_ERR_ARG, "patch spmm: batch must be a power of two <= 64");
    }
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
template int launch_spmm_sh_patch<float>(const sptb_plan*, const void*, void*, int, const void*, cudaStream_t, bool);
template int launch_spmm_sh_patch<double>(const sptb_plan*, const void*, void*, int, const void*, cudaStream_t, bool);

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
