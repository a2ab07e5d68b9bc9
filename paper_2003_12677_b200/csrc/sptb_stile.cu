// Output-tiled S SpMM (adjoint / gridrec direction):  Y[b][m] = S_(w) X,
// X [s'][b] (batch innermost, the FFT1-side operand), Y batch-outer for the
// inverse 2-D FFT.  The reference computes it with scipy CSR
// (operators.py:124-136, 178-184).
//
// S = conj(S^H)^T and every sample's nonzeros sit in the 3x3 block around its
// stencil centre (gridding.py:104-143): grid cell m receives, from each sample
// centred at m - (ex, ey) (ex, ey in {-1, 0, 1}), the conjugate of that
// sample's slot (ey + 1) * 3 + (ex + 1).  A tile is the 8x8 cells of a sample
// patch; its samples (own patch + neighbour edge columns/rows/corners) are at
// most STILE_RUNS contiguous s' runs (border-class order, build_patches):
//   * one elected thread stages the runs -- X rows and slot rows -- and the
//     tile's centre table with <= 21 bulk copies on one mbarrier;
//   * a group of 16 lanes per cell walks the 9 neighbour centres; per sample
//     it reads one broadcast slot value (compile-time slot index) and one
//     16-byte piece of the sample's X row -- no per-nonzero index at all;
//   * the 64 x B tile leaves through shared memory as row runs per plane.
// Dense tiles (> STILE_CAP samples, the centre of the polar grid) gather
// through the CSR of S instead; cells touched by irregular samples (stencil
// centre outside the grid) get a deterministic fix-up pass.  Accumulation
// order is fixed (neighbour, then s'): results do not depend on the batch slot.
#include "sptb_internal.cuh"

#include <algorithm>
#include <cstring>
#include <vector>

namespace sptb {

namespace {

template <typename R> struct TCplx;
template <> struct TCplx<float> { using T = float2; };
template <> struct TCplx<double> { using T = double2; };

constexpr int TT = 256;  // threads per CTA
constexpr int TG = 16;   // lanes per grid cell

__device__ __forceinline__ void sbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "SW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra SW;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void sbulk(void* dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// tile (64 cells x BB planes) -> y: cells (8px + 1 + ox, 8py + oy); the x = 0
// column (no S entries: border, gridding.py:136-137) is written as zeros by
// the px = 0 tiles
template <typename C, int BB>
__device__ __forceinline__ void store_tile(const C* ot, int px, int py, int X, int Y, long long M, C* y) {
    constexpr int OS = STILE * STILE + 1;
    for (int e = threadIdx.x; e < BB * STILE * STILE; e += TT) {
        const int b = e / (STILE * STILE), cell = e % (STILE * STILE);
        const int gx = STILE * px + 1 + cell % STILE, gy = STILE * py + cell / STILE;
        if (gx < X && gy < Y) y[(size_t)b * M + (size_t)gy * X + gx] = ot[b * OS + cell];
    }
    if (px == 0)
        for (int e = threadIdx.x; e < BB * STILE; e += TT) {
            const int b = e / STILE, gy = STILE * py + e % STILE;
            if (gy < Y) {
                C z;
                z.x = z.y = 0;
                y[(size_t)b * M + (size_t)gy * X] = z;
            }
        }
}

template <typename R, int BB>
__global__ void __launch_bounds__(TT)
k_s_tile(const int* __restrict__ tiles, const STileMeta* __restrict__ meta, int npx, int X, int Y,
         long long M, const typename TCplx<R>::T* __restrict__ x,
         const typename TCplx<R>::T* __restrict__ vals, typename TCplx<R>::T* __restrict__ y) {
    using C = typename TCplx<R>::T;
    constexpr int CW = BB >= 2 * TG ? BB / TG : 1;  // columns per lane
    constexpr int NL = BB / CW;                     // lanes per cell in use
    constexpr int NGRP = TT / TG;
    constexpr int CPG = STILE * STILE / NGRP;       // cells per group
    constexpr int XROW = BB * (int)sizeof(C);
    constexpr int VROW = SLOT_STRIDE * (int)sizeof(C);
    constexpr int OS = STILE * STILE + 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(16) unsigned tab[100];
    __shared__ __align__(8) unsigned long long bar;
    unsigned char* xs = smem_raw;                       // [CAP][BB] C
    unsigned char* vs = xs + STILE_CAP * XROW;          // [CAP][10] C
    const int tid = threadIdx.x;
    const int tile = tiles[blockIdx.x];
    const int px = tile % npx, py = tile / npx;
    const STileMeta* mt = meta + tile;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        const int ns = mt->ns;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb),
                     "r"((unsigned)ns * (XROW + VROW) + 400u) : "memory");
        sbulk(tab, mt->table, 400u, sb);
        int off = 0;
#pragma unroll 1
        for (int i = 0; i < STILE_RUNS; ++i) {
            const int2 rn = mt->run[i];
            if (rn.y > 0) {
                sbulk(xs + off * XROW, x + (size_t)rn.x * BB, (unsigned)(rn.y * XROW), sb);
                sbulk(vs + off * VROW, vals + (size_t)rn.x * SLOT_STRIDE, (unsigned)(rn.y * VROW), sb);
                off += rn.y;
            }
        }
    }
    __syncthreads();
    sbar_wait(sb, 0);

    const int g = tid / TG, lig = tid % TG;
    C ar[CPG][CW], ai[CPG][CW];
#pragma unroll
    for (int j = 0; j < CPG; ++j)
#pragma unroll
        for (int w = 0; w < CW; ++w) ar[j][w].x = ar[j][w].y = ai[j][w].x = ai[j][w].y = 0;
    if (lig < NL) {
        const unsigned char* xl = xs + lig * CW * (int)sizeof(C);
#pragma unroll
        for (int j = 0; j < CPG; ++j) {
            const int cell = g + NGRP * j;
            const int bx = cell % STILE + 1, by = cell / STILE + 1;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const int ey = k / 3 - 1, ex = k % 3 - 1;
                const unsigned t = tab[(by - ey) * 10 + (bx - ex)];
                const int beg = (int)(t & 0xffffu), cnt = (int)(t >> 16);
                const C* vp = reinterpret_cast<const C*>(vs) + beg * SLOT_STRIDE + k;
                const unsigned char* xp = xl + beg * XROW;
#pragma unroll 2
                for (int i = 0; i < cnt; ++i) {
                    const C v = vp[i * SLOT_STRIDE];
                    if constexpr (sizeof(C) == 8 && CW == 2) {
                        const float4 xv = *reinterpret_cast<const float4*>(xp + i * XROW);
                        const float2 x0 = make_float2(xv.x, xv.y), x1 = make_float2(xv.z, xv.w);
                        float2 r0 = make_float2(ar[j][0].x, ar[j][0].y), r1 = make_float2(ar[j][1].x, ar[j][1].y);
                        float2 i0 = make_float2(ai[j][0].x, ai[j][0].y), i1 = make_float2(ai[j][1].x, ai[j][1].y);
                        r0 = __ffma2_rn(make_float2(v.x, v.x), x0, r0);
                        i0 = __ffma2_rn(make_float2(v.y, v.y), x0, i0);
                        r1 = __ffma2_rn(make_float2(v.x, v.x), x1, r1);
                        i1 = __ffma2_rn(make_float2(v.y, v.y), x1, i1);
                        ar[j][0].x = r0.x; ar[j][0].y = r0.y; ar[j][1].x = r1.x; ar[j][1].y = r1.y;
                        ai[j][0].x = i0.x; ai[j][0].y = i0.y; ai[j][1].x = i1.x; ai[j][1].y = i1.y;
                    } else {
                        const C* xq = reinterpret_cast<const C*>(xp + i * XROW);
#pragma unroll
                        for (int w = 0; w < CW; ++w) {
                            const C xv = xq[w];
                            ar[j][w].x = fma(v.x, xv.x, ar[j][w].x);
                            ar[j][w].y = fma(v.x, xv.y, ar[j][w].y);
                            ai[j][w].x = fma(v.y, xv.x, ai[j][w].x);
                            ai[j][w].y = fma(v.y, xv.y, ai[j][w].y);
                        }
                    }
                }
            }
        }
    }
    __syncthreads();  // the staging area becomes the output tile
    C* ot = reinterpret_cast<C*>(smem_raw);
    if (lig < NL) {
#pragma unroll
        for (int j = 0; j < CPG; ++j)
#pragma unroll
            for (int w = 0; w < CW; ++w) {
                C o;  // conj(v) x = (vr xr + vi xi, vr xi - vi xr)
                o.x = ar[j][w].x + ai[j][w].y;
                o.y = ar[j][w].y - ai[j][w].x;
                ot[(lig * CW + w) * OS + g + NGRP * j] = o;
            }
    }
    __syncthreads();
    store_tile<C, BB>(ot, px, py, X, Y, M, y);
}

// dense tiles: gather through the CSR of S (columns renumbered to s'); the
// values are the ones of S itself (no conjugation)
template <typename R, int BB>
__global__ void __launch_bounds__(TT)
k_s_dense(const int* __restrict__ tiles, int npx, int X, int Y, long long M, const int* __restrict__ rp,
          const int* __restrict__ col, const typename TCplx<R>::T* __restrict__ val,
          const typename TCplx<R>::T* __restrict__ x, typename TCplx<R>::T* __restrict__ y) {
    using C = typename TCplx<R>::T;
    constexpr int CW = BB >= 2 * TG ? BB / TG : 1;
    constexpr int NL = BB / CW;
    constexpr int NGRP = TT / TG;
    constexpr int CPG = STILE * STILE / NGRP;
    constexpr int OS = STILE * STILE + 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    C* ot = reinterpret_cast<C*>(smem_raw);
    const int tile = tiles[blockIdx.x];
    const int px = tile % npx, py = tile / npx;
    const int g = threadIdx.x / TG, lig = threadIdx.x % TG;
#pragma unroll 1
    for (int j = 0; j < CPG; ++j) {
        const int cell = g + NGRP * j;
        const int gx = STILE * px + 1 + cell % STILE, gy = STILE * py + cell / STILE;
        C a[CW];
#pragma unroll
        for (int w = 0; w < CW; ++w) a[w].x = a[w].y = 0;
        if (gx < X && gy < Y && lig < NL) {
            const long long m = (long long)gy * X + gx;
            const int e0 = rp[m], e1 = rp[m + 1];
#pragma unroll 4
            for (int e = e0; e < e1; ++e) {
                const C v = __ldg(val + e);
                const C* xq = x + (size_t)__ldg(col + e) * BB + lig * CW;
#pragma unroll
                for (int w = 0; w < CW; ++w) {
                    const C xv = __ldg(xq + w);
                    a[w].x = fma(v.x, xv.x, a[w].x);
                    a[w].x = fma(-v.y, xv.y, a[w].x);
                    a[w].y = fma(v.x, xv.y, a[w].y);
                    a[w].y = fma(v.y, xv.x, a[w].y);
                }
            }
        }
        if (lig < NL)
#pragma unroll
            for (int w = 0; w < CW; ++w) ot[(lig * CW + w) * OS + cell] = a[w];
    }
    __syncthreads();
    store_tile<C, BB>(ot, px, py, X, Y, M, y);
}

// cells touched by irregular samples: y[b][m] += sum conj(slot value) x[s'][b]
template <typename R>
__global__ void k_s_fix(int n_fix, const int* __restrict__ cell, const int* __restrict__ ptr,
                        const int2* __restrict__ ent, const typename TCplx<R>::T* __restrict__ vals, int B,
                        long long M, const typename TCplx<R>::T* __restrict__ x,
                        typename TCplx<R>::T* __restrict__ y) {
    using C = typename TCplx<R>::T;
    const long long n = (long long)n_fix * B;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / B), b = (int)(e % B);
        C a;
        a.x = a.y = 0;
        for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
            const int2 t = ent[k];
            const C v = vals[(size_t)t.x * SLOT_STRIDE + t.y], xv = x[(size_t)t.x * B + b];
            a.x = fma(v.x, xv.x, a.x);
            a.x = fma(v.y, xv.y, a.x);
            a.y = fma(v.x, xv.y, a.y);
            a.y = fma(-v.y, xv.x, a.y);
        }
        C* o = y + (size_t)b * M + cell[i];
        C cur = *o;
        cur.x += a.x;
        cur.y += a.y;
        *o = cur;
    }
}

template <typename R>
__global__ void k_fold_slots(const typename TCplx<R>::T* __restrict__ sval, const int* __restrict__ order,
                             const R* __restrict__ w, long long wlen, long long N, int P,
                             typename TCplx<R>::T* __restrict__ out) {
    const long long n = N * SLOT_STRIDE;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / SLOT_STRIDE;
        const int k = (int)(i - r * SLOT_STRIDE);
        typename TCplx<R>::T v = sval[i];
        if (k < 9) {
            const long long s = order[r];
            const R f = (wlen == N) ? w[s] : w[s % P];
            v.x *= f;
            v.y *= f;
        }
        out[i] = v;
    }
}

template <typename R, int BB>
int s_tile_dispatch(const sptb_plan* p, const void* csr_vals, const void* slot, const void* x, void* y,
                    cudaStream_t st) {
    using C = typename TCplx<R>::T;
    const STiles& t = p->stl;
    const int npx = p->shp.npx;
    const size_t so = (size_t)BB * (STILE * STILE + 1) * sizeof(C);
    if (t.n_sparse > 0) {
        const size_t sm = std::max((size_t)STILE_CAP * (BB + SLOT_STRIDE) * sizeof(C), so);
        auto kern = k_s_tile<R, BB>;
        SPTB_CUDA(set_smem_once((const void*)kern, (int)sm));
        kern<<<t.n_sparse, TT, sm, st>>>(t.sparse, t.meta, npx, p->X, p->Y, p->M, (const C*)x,
                                        (const C*)slot, (C*)y);
        SPTB_LAUNCHED();
    }
    if (t.n_dense > 0) {
        auto kern = k_s_dense<R, BB>;
        SPTB_CUDA(set_smem_once((const void*)kern, (int)so));
        kern<<<t.n_dense, TT, so, st>>>(t.dense, npx, p->X, p->Y, p->M, p->S.row_ptr, p->shp.s_colp,
                                       (const C*)csr_vals, (const C*)x, (C*)y);
        SPTB_LAUNCHED();
    }
    if (t.n_fix > 0) {
        const long long n = (long long)t.n_fix * BB;
        k_s_fix<R><<<(unsigned)std::min<long long>((n + 255) / 256, 148LL * 8), 256, 0, st>>>(
            t.n_fix, t.fix_cell, t.fix_ptr, t.fix_ent, (const C*)slot, BB, p->M, (const C*)x, (C*)y);
        SPTB_LAUNCHED();
    }
    return SPTB_OK;
}

}  // namespace

template <typename R>
int launch_spmm_s(const sptb_plan* p, const void* vals, const void* x_sb, void* y_bm, int B,
                  cudaStream_t st) {
    const void* slot = nullptr;
    if (p->stl.meta && p->shp.sval) {
        if (vals == p->S.val) slot = p->shp.sval;
        else if (vals == p->SW_val && p->stl.swval) slot = p->stl.swval;
    }
    // bulk copies need 16-byte rows and a 16-byte aligned operand
    const bool aligned = ((uintptr_t)x_sb % 16) == 0 && (size_t)B * p->csize >= 16 &&
                         (size_t)STILE_CAP * (B + SLOT_STRIDE) * p->csize <= 200 * 1024;
    // opt-in (SPTB_STILE=1) until it beats the row gather: the dense centre
    // tiles still serialise
    static const bool use_tiles = [] {
        const char* e = getenv("SPTB_STILE");
        return e && e[0] == '1';
    }();
    if (!slot || !aligned || !use_tiles)
        return launch_spmm<R>(s_permuted(p), vals, x_sb, y_bm, B, true, nullptr, st);
    switch (B) {
        case 1: return s_tile_dispatch<R, 1>(p, vals, slot, x_sb, y_bm, st);
        case 2: return s_tile_dispatch<R, 2>(p, vals, slot, x_sb, y_bm, st);
        case 4: return s_tile_dispatch<R, 4>(p, vals, slot, x_sb, y_bm, st);
        case 8: return s_tile_dispatch<R, 8>(p, vals, slot, x_sb, y_bm, st);
        case 16: return s_tile_dispatch<R, 16>(p, vals, slot, x_sb, y_bm, st);
        case 32: return s_tile_dispatch<R, 32>(p, vals, slot, x_sb, y_bm, st);
        case 64: return s_tile_dispatch<R, 64>(p, vals, slot, x_sb, y_bm, st);
    }
    return fail(SPTB_ERR_ARG, "spmm: batch must be a power of two <= 64");
}
template int launch_spmm_s<float>(const sptb_plan*, const void*, const void*, void*, int, cudaStream_t);
template int launch_spmm_s<double>(const sptb_plan*, const void*, const void*, void*, int, cudaStream_t);

// w-folded slot rows for S diag(w) (sptb_plan_set_filter)
int fold_slot_filter(sptb_plan* p) {
    if (p->stl.swval) {
        cudaFree(p->stl.swval);
        p->stl.swval = nullptr;
    }
    if (p->w_len == 0 || !p->shp.sval) return SPTB_OK;
    const long long n = p->N * SLOT_STRIDE;
    SPTB_CUDA(cudaMalloc(&p->stl.swval, p->csize * (size_t)n));
    const unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16);
    if (p->prec == SPTB_PREC_F64)
        k_fold_slots<double><<<grid, 256, 0, p->stream>>>((const double2*)p->shp.sval, p->shp.order,
                                                        (const double*)p->w_dev, p->w_len, p->N, p->P,
                                                        (double2*)p->stl.swval);
    else
        k_fold_slots<float><<<grid, 256, 0, p->stream>>>((const float2*)p->shp.sval, p->shp.order,
                                                       (const float*)p->w_dev, p->w_len, p->N, p->P,
                                                       (float2*)p->stl.swval);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

// Host build of the tile metadata (once per plan, slot mode).  Tile = sample
// patch q = (px, py); staged runs in a fixed order; the centre table maps
// the 10x10 centre box (x in [8px, 8px+9], y in [8py-1, 8py+8]) to the staged
// list.
int build_stiles(sptb_plan* p, const std::vector<int>& cx, const std::vector<int>& cy,
                 const std::vector<int>& rp, const std::vector<int>& col, const std::vector<int>& order,
                 const std::vector<int64_t>& cnt, const std::vector<int>& cls_start) {
    STiles& t = p->stl;
    const PatchSH& sp = p->shp;
    const int X = p->X, npx = sp.npx, npy = sp.npy;
    const int64_t npatch = (int64_t)npx * npy;
    std::vector<STileMeta> meta((size_t)npatch);
    std::vector<int> sparse, dense;
    std::vector<char> is_dense((size_t)npatch, 0);
    auto cs = [&](int64_t q, int c) { return cls_start[(size_t)q * STILE_NCLS1 + c]; };
    for (int64_t q = 0; q < npatch; ++q) {
        STileMeta& m = meta[(size_t)q];
        std::memset(&m, 0, sizeof(m));
        const int px = (int)(q % npx), py = (int)(q / npx);
        int nr = 0;
        auto add = [&](int64_t b, int64_t e) {
            if (e > b) m.run[nr++] = make_int2((int)b, (int)(e - b));
        };
        auto nb = [&](int dx, int dy, int c0, int c1) {
            const int qx = px + dx, qy = py + dy;
            if (qx < 0 || qx >= npx || qy < 0 || qy >= npy) return;
            const int64_t qq = (int64_t)qy * npx + qx;
            add(cs(qq, c0), cs(qq, c1));
        };
        add(cnt[q], cnt[q + 1]);   // own patch
        nb(-1, 0, 2, 5);           // left: TR R BR
        nb(1, 0, 0, 1);            // right: TL ...
        nb(1, 0, 6, 8);            //        ... BL L
        nb(0, -1, 4, 7);           // top: BR B BL
        nb(0, 1, 0, 3);            // bottom: TL T TR
        nb(-1, -1, 4, 5);          // top-left: BR
        nb(1, -1, 6, 7);           // top-right: BL
        nb(-1, 1, 2, 3);           // bottom-left: TR
        nb(1, 1, 0, 1);            // bottom-right: TL
        int ns = 0;
        for (int i = 0; i < nr; ++i) ns += m.run[i].y;
        m.ns = ns;
        if (ns > STILE_CAP) {
            is_dense[(size_t)q] = 1;
            dense.push_back((int)q);
            continue;
        }
        sparse.push_back((int)q);
        int li = 0, last = -1;
        for (int i = 0; i < nr; ++i)
            for (int r = m.run[i].x; r < m.run[i].x + m.run[i].y; ++r, ++li) {
                const int smp = order[r];
                const int bx = cx[smp] - STILE * px, by = cy[smp] - (STILE * py - 1);
                if (bx < 0 || bx > 9 || by < 0 || by > 9)
                    return fail(SPTB_ERR_STATE, "tile build: sample centre outside the tile's centre box");
                const int n = by * 10 + bx;
                unsigned& e = m.table[n];
                if ((e >> 16) == 0) {
                    e = (unsigned)li | (1u << 16);
                } else {
                    if (n != last) return fail(SPTB_ERR_STATE, "tile build: centre cell not contiguous");
                    e += 1u << 16;
                }
                last = n;
            }
    }
    // irregular samples (after n_reg): fix-up entries per touched cell outside dense tiles
    std::vector<std::pair<int, int2>> fx;
    for (int64_t r = sp.n_reg; r < p->N; ++r) {
        const int smp = order[r];
        for (int k = rp[smp]; k < rp[smp + 1]; ++k) {
            const int gx = col[k] % X, gy = col[k] / X;
            const int qx = std::min(std::max(gx - 1, 0) / STILE, npx - 1), qy = gy / STILE;
            if (is_dense[(size_t)qy * npx + qx]) continue;
            const int slot = (gy - cy[smp] + 1) * 3 + (gx - cx[smp] + 1);
            fx.push_back({col[k], make_int2((int)r, slot)});
        }
    }
    std::stable_sort(fx.begin(), fx.end(), [](const std::pair<int, int2>& a, const std::pair<int, int2>& b) {
        return a.first < b.first;
    });
    std::vector<int> fcell, fptr(1, 0);
    std::vector<int2> fent;
    for (size_t i = 0; i < fx.size(); ++i) {
        if (i == 0 || fx[i].first != fx[i - 1].first) {
            if (i) fptr.push_back((int)fent.size());
            fcell.push_back(fx[i].first);
        }
        fent.push_back(fx[i].second);
    }
    if (!fx.empty()) fptr.push_back((int)fent.size());
    t.n_sparse = (int)sparse.size();
    t.n_dense = (int)dense.size();
    t.n_fix = (int)fcell.size();
    SPTB_CUDA(cudaMalloc(&t.meta, sizeof(STileMeta) * std::max<size_t>(meta.size(), 1)));
    SPTB_CUDA(cudaMemcpy(t.meta, meta.data(), sizeof(STileMeta) * meta.size(), cudaMemcpyHostToDevice));
    SPTB_CUDA(cudaMalloc(&t.sparse, sizeof(int) * std::max<size_t>(sparse.size(), 1)));
    SPTB_CUDA(cudaMalloc(&t.dense, sizeof(int) * std::max<size_t>(dense.size(), 1)));
    if (!sparse.empty())
        SPTB_CUDA(cudaMemcpy(t.sparse, sparse.data(), sizeof(int) * sparse.size(), cudaMemcpyHostToDevice));
    if (!dense.empty())
        SPTB_CUDA(cudaMemcpy(t.dense, dense.data(), sizeof(int) * dense.size(), cudaMemcpyHostToDevice));
    if (t.n_fix) {
        SPTB_CUDA(cudaMalloc(&t.fix_cell, sizeof(int) * fcell.size()));
        SPTB_CUDA(cudaMalloc(&t.fix_ptr, sizeof(int) * fptr.size()));
        SPTB_CUDA(cudaMalloc(&t.fix_ent, sizeof(int2) * fent.size()));
        SPTB_CUDA(cudaMemcpy(t.fix_cell, fcell.data(), sizeof(int) * fcell.size(), cudaMemcpyHostToDevice));
        SPTB_CUDA(cudaMemcpy(t.fix_ptr, fptr.data(), sizeof(int) * fptr.size(), cudaMemcpyHostToDevice));
        SPTB_CUDA(cudaMemcpy(t.fix_ent, fent.data(), sizeof(int2) * fent.size(), cudaMemcpyHostToDevice));
    }
    return SPTB_OK;
}

}  // namespace sptb
