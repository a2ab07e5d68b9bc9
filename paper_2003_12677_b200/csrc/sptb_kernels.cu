// Hot-path kernels: gridding SpMM (K1/K2), layout transposes, pack/unpack
// (K3-K6 elementwise stages).  sm_100a, no tensor cores: every kernel here is
// HBM/L2-bound.
#include "sptb_internal.cuh"

#include <algorithm>

namespace sptb {

template <typename R> struct Cplx;
template <> struct Cplx<float> { using T = float2; };
template <> struct Cplx<double> { using T = double2; };

// 8- or 16-byte lane chunk holding CW complex values
template <typename R, int CW> struct Chunk;
template <> struct Chunk<float, 1> {
    using T = float2;
    static __device__ __forceinline__ void ld(const void* p, float2 (&c)[1]) {
        c[0] = __ldg(reinterpret_cast<const float2*>(p));
    }
};
template <> struct Chunk<float, 2> {
    using T = float4;
    static __device__ __forceinline__ void ld(const void* p, float2 (&c)[2]) {
        float4 v = __ldg(reinterpret_cast<const float4*>(p));
        c[0] = make_float2(v.x, v.y);
        c[1] = make_float2(v.z, v.w);
    }
};
template <> struct Chunk<double, 1> {
    using T = double2;
    static __device__ __forceinline__ void ld(const void* p, double2 (&c)[1]) {
        c[0] = __ldg(reinterpret_cast<const double2*>(p));
    }
};

template <typename C>
__device__ __forceinline__ void cmac(C& acc, const C& a, const C& b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}

// ---------------------------------------------------------------------------
// CSR SpMM over a batch-innermost dense operand.
//
// One CTA owns TILE consecutive rows.  The tile's row pointers and, when they
// fit (<= CAP entries), its column indices and values are staged in shared
// memory with coalesced loads, so the gather loop issues only the 8/16-byte
// lane loads of x (one contiguous BB*sizeof(C) run per nonzero) plus FMAs.
// A "group" of G lanes computes one row for all BB = G*CPL*CW columns.
// Rows longer than LMAX nonzeros (the skewed centre of S: up to 4852 at
// 2048^2 x 1536) are flagged with a warp ballot and split into NCH fixed
// chunks shared by all groups of the CTA, combined in chunk order -- results
// are deterministic and independent of which group ran which chunk.
// TRANS: the tile is staged in shared memory and written [b][row] (the
// batch-outer layout cuFFT wants): the layout transpose is fused into the
// epilogue.  SUB: y = sub - A x  ([row][b]).
// ---------------------------------------------------------------------------
constexpr int SPMM_THREADS = 256;
constexpr int LMAX = 64;
constexpr int NCH = 16;
#ifndef SPTB_UNR
#define SPTB_UNR 8
#endif
constexpr int UNR = SPTB_UNR;
constexpr int CAP = 1024;  // staged nonzeros per tile

template <typename R, int G, int CPL, int CW>
struct SpmmCfg {
    static constexpr int BB = G * CPL * CW;
    static constexpr int NG = SPMM_THREADS / G;
    static constexpr int TILE = (4 * NG < 64) ? 64 : (4 * NG > 256 ? 256 : 4 * NG);
};

// acc += sum_k val[k] * x[col[k]]  over k in [beg, end), metadata from smem
// (STAGED) or global memory; UNR gathers issued before their FMAs.
template <typename R, int G, int CPL, int CW, bool STAGED>
__device__ __forceinline__ void row_accumulate(
    const int* __restrict__ ci, const typename Cplx<R>::T* __restrict__ cv,
    const typename Cplx<R>::T* __restrict__ x, int beg, int end, int lig,
    typename Cplx<R>::T (&acc)[CPL][CW]) {
    using C = typename Cplx<R>::T;
    constexpr int BB = G * CPL * CW;
    const C* xl = x + (size_t)lig * CW;
    // every chunk issues all of its (predicated) gathers before any FMA, so a
    // typical row (<= UNR nonzeros) costs one memory round trip
    for (int k = beg; k < end; k += UNR) {
        int cc[UNR];
        C vv[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const bool ok = k + u < end;
            cc[u] = ok ? (STAGED ? ci[k + u] : __ldg(ci + k + u)) : -1;
            C z;
            z.x = z.y = 0;
            vv[u] = ok ? cv[k + u] : z;
        }
        C xs[UNR][CPL][CW];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                if (cc[u] >= 0) {
                    Chunk<R, CW>::ld(xl + (size_t)cc[u] * BB + (size_t)q * G * CW, xs[u][q]);
                } else {
#pragma unroll
                    for (int w = 0; w < CW; ++w) xs[u][q][w].x = xs[u][q][w].y = 0;
                }
            }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int q = 0; q < CPL; ++q)
#pragma unroll
                for (int w = 0; w < CW; ++w) cmac(acc[q][w], vv[u], xs[u][q][w]);
    }
}

template <typename R, int G, int CPL, int CW, bool TRANS, bool SUB>
__global__ void __launch_bounds__(SPMM_THREADS)
k_spmm(const int* __restrict__ rp, const int* __restrict__ ci,
       const typename Cplx<R>::T* __restrict__ cv,
       const typename Cplx<R>::T* __restrict__ x, typename Cplx<R>::T* __restrict__ y,
       const typename Cplx<R>::T* __restrict__ sub, int rows) {
    using C = typename Cplx<R>::T;
    using Cfg = SpmmCfg<R, G, CPL, CW>;
    constexpr int BB = Cfg::BB, NG = Cfg::NG, TILE = Cfg::TILE;
    constexpr int LD = BB + 1;  // padded smem row (bank spread)
    constexpr int NW = TILE / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* s_val = reinterpret_cast<C*>(smem_raw);          // [CAP]
    C* part = s_val + CAP;                              // [NCH][BB]
    C* tile = part + NCH * BB;                          // [TILE][LD] (TRANS only)
    __shared__ int s_rp[TILE + 1];
    __shared__ int s_col[CAP];
    __shared__ unsigned s_long[NW];

    const int tid = threadIdx.x;
    const int g = tid / G, lig = tid % G;
    const int row0 = blockIdx.x * TILE;
    const int nrows = min(TILE, rows - row0);
    for (int i = tid; i <= nrows; i += SPMM_THREADS) s_rp[i] = rp[row0 + i];
    __syncthreads();
    const int e0 = s_rp[0], ne = s_rp[nrows] - e0;
    const bool staged = ne <= CAP;
    if (staged) {
        for (int i = tid; i < ne; i += SPMM_THREADS) {
            s_col[i] = __ldg(ci + e0 + i);
            s_val[i] = cv[e0 + i];
        }
    }
    for (int r = tid; r < NW * 32; r += SPMM_THREADS) {
        const bool lng = r < nrows && (s_rp[r + 1] - s_rp[r]) > LMAX;
        const unsigned m = __ballot_sync(0xffffffffu, lng);
        if ((r & 31) == 0) s_long[r >> 5] = m;
    }
    __syncthreads();

    auto emit = [&](int r, const C (&a)[CPL][CW]) {
#pragma unroll
        for (int q = 0; q < CPL; ++q)
#pragma unroll
            for (int w = 0; w < CW; ++w) {
                const int b = (q * G + lig) * CW + w;
                if (TRANS) {
                    tile[r * LD + b] = a[q][w];
                } else {
                    const size_t o = (size_t)(row0 + r) * BB + b;
                    C v = a[q][w];
                    if (SUB) {
                        const C s = sub[o];
                        v.x = s.x - v.x;
                        v.y = s.y - v.y;
                    }
                    y[o] = v;
                }
            }
    };

    // short rows: one group per row
    for (int r = g; r < nrows; r += NG) {
        const int beg = s_rp[r] - e0, end = s_rp[r + 1] - e0;
        if (end - beg > LMAX) continue;
        C acc[CPL][CW];
#pragma unroll
        for (int q = 0; q < CPL; ++q)
#pragma unroll
            for (int w = 0; w < CW; ++w) acc[q][w].x = acc[q][w].y = 0;
        if (staged)
            row_accumulate<R, G, CPL, CW, true>(s_col, s_val, x, beg, end, lig, acc);
        else
            row_accumulate<R, G, CPL, CW, false>(ci + e0, cv + e0, x, beg, end, lig, acc);
        emit(r, acc);
    }

    // long rows (ballot mask, ascending): NCH chunks over all groups
    for (int wd = 0; wd < NW; ++wd) {
        unsigned m = s_long[wd];
        while (m) {
            const int r = wd * 32 + __ffs(m) - 1;
            m &= m - 1;
            const int beg = s_rp[r] - e0, len = s_rp[r + 1] - s_rp[r];
            for (int c = g; c < NCH; c += NG) {
                const int cb = beg + (int)(((long long)len * c) / NCH);
                const int ce = beg + (int)(((long long)len * (c + 1)) / NCH);
                C acc[CPL][CW];
#pragma unroll
                for (int q = 0; q < CPL; ++q)
#pragma unroll
                    for (int w = 0; w < CW; ++w) acc[q][w].x = acc[q][w].y = 0;
                if (staged)
                    row_accumulate<R, G, CPL, CW, true>(s_col, s_val, x, cb, ce, lig, acc);
                else
                    row_accumulate<R, G, CPL, CW, false>(ci + e0, cv + e0, x, cb, ce, lig, acc);
#pragma unroll
                for (int q = 0; q < CPL; ++q)
#pragma unroll
                    for (int w = 0; w < CW; ++w) part[c * BB + (q * G + lig) * CW + w] = acc[q][w];
            }
            __syncthreads();
            for (int b = tid; b < BB; b += SPMM_THREADS) {
                C s = part[b];
                for (int c = 1; c < NCH; ++c) {
                    s.x += part[c * BB + b].x;
                    s.y += part[c * BB + b].y;
                }
                if (TRANS) {
                    tile[r * LD + b] = s;
                } else {
                    const size_t o = (size_t)(row0 + r) * BB + b;
                    if (SUB) {
                        const C t = sub[o];
                        s.x = t.x - s.x;
                        s.y = t.y - s.y;
                    }
                    y[o] = s;
                }
            }
            __syncthreads();
        }
    }

    if (TRANS) {
        __syncthreads();
        // y[b][row0 + i]: consecutive threads -> consecutive rows
#pragma unroll 4
        for (int e = tid; e < BB * TILE; e += SPMM_THREADS) {
            const int b = e / TILE, i = e % TILE;
            if (i < nrows) y[(size_t)b * rows + row0 + i] = tile[i * LD + b];
        }
    }
}

template <typename R, int G, int CPL, int CW>
static int spmm_dispatch(const DevCSR& A, const void* val, const void* x, void* y,
                         bool trans, const void* sub, cudaStream_t st) {
    using C = typename Cplx<R>::T;
    using Cfg = SpmmCfg<R, G, CPL, CW>;
    const int rows = (int)A.rows;
    if (rows == 0) return SPTB_OK;
    const int grid = (rows + Cfg::TILE - 1) / Cfg::TILE;
    size_t sm = (size_t)(CAP + NCH * Cfg::BB) * sizeof(C);
    if (trans) sm += (size_t)Cfg::TILE * (Cfg::BB + 1) * sizeof(C);
    auto run = [&](auto kern) -> int {
        // the row gather lives on L1 hits of gathered rows: leave the carveout to
        // the driver (forcing 100% smem cost 5%, 0-25% tripled the time)
        SPTB_CUDA(set_smem_once((const void*)kern, (int)sm, -1));
        kern<<<grid, SPMM_THREADS, sm, st>>>(A.row_ptr, A.col, (const C*)val, (const C*)x,
                                             (C*)y, (const C*)sub, rows);
        SPTB_LAUNCHED();
        return SPTB_OK;
    };
    if (trans) return run(k_spmm<R, G, CPL, CW, true, false>);
    if (sub) return run(k_spmm<R, G, CPL, CW, false, true>);
    return run(k_spmm<R, G, CPL, CW, false, false>);
}

template <>
int launch_spmm<float>(const DevCSR& A, const void* val, const void* x, void* y, int B,
                       bool trans, const void* sub, cudaStream_t st) {
    if (trans && sub) return fail(SPTB_ERR_ARG, "spmm: trans+sub unsupported");
    switch (B) {
        case 1: return spmm_dispatch<float, 1, 1, 1>(A, val, x, y, trans, sub, st);
        case 2: return spmm_dispatch<float, 1, 1, 2>(A, val, x, y, trans, sub, st);
        case 4: return spmm_dispatch<float, 2, 1, 2>(A, val, x, y, trans, sub, st);
        case 8: return spmm_dispatch<float, 4, 1, 2>(A, val, x, y, trans, sub, st);
        case 16: return spmm_dispatch<float, 8, 1, 2>(A, val, x, y, trans, sub, st);
#ifndef SPTB_S32_G
#define SPTB_S32_G 16
#endif
        case 32: return spmm_dispatch<float, SPTB_S32_G, 16 / SPTB_S32_G, 2>(A, val, x, y, trans, sub, st);
        case 64: return spmm_dispatch<float, 32, 1, 2>(A, val, x, y, trans, sub, st);
    }
    return fail(SPTB_ERR_ARG, "spmm: batch must be a power of two <= 64");
}

template <>
int launch_spmm<double>(const DevCSR& A, const void* val, const void* x, void* y, int B,
                        bool trans, const void* sub, cudaStream_t st) {
    if (trans && sub) return fail(SPTB_ERR_ARG, "spmm: trans+sub unsupported");
    switch (B) {
        case 1: return spmm_dispatch<double, 1, 1, 1>(A, val, x, y, trans, sub, st);
        case 2: return spmm_dispatch<double, 2, 1, 1>(A, val, x, y, trans, sub, st);
        case 4: return spmm_dispatch<double, 4, 1, 1>(A, val, x, y, trans, sub, st);
        case 8: return spmm_dispatch<double, 8, 1, 1>(A, val, x, y, trans, sub, st);
        case 16: return spmm_dispatch<double, 16, 1, 1>(A, val, x, y, trans, sub, st);
        case 32: return spmm_dispatch<double, 32, 1, 1>(A, val, x, y, trans, sub, st);
        case 64: return spmm_dispatch<double, 32, 2, 1>(A, val, x, y, trans, sub, st);
    }
    return fail(SPTB_ERR_ARG, "spmm: batch must be a power of two <= 64");
}

// ---------------------------------------------------------------------------
// [b][m] -> [m][b] tiled transpose (B <= 64): 32 m x B tile through smem.
// ---------------------------------------------------------------------------
template <typename C>
__global__ void __launch_bounds__(256) k_transpose_bm_mb(const C* __restrict__ in,
                                                         C* __restrict__ out, int B,
                                                         long long M) {
    __shared__ C t[64][33];
    const long long m0 = (long long)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int b = ty; b < B; b += 8) {
        const long long m = m0 + tx;
        if (m < M) t[b][tx] = in[(size_t)b * M + m];
    }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
        const long long m = m0 + i;
        if (m >= M) break;
        for (int b = tx; b < B; b += 32) out[(size_t)m * B + b] = t[b][i];
    }
}

template <typename R>
int launch_transpose_bm_to_mb(const void* in, void* out, int B, int64_t M, cudaStream_t st) {
    using C = typename Cplx<R>::T;
    if (B > 64) return fail(SPTB_ERR_ARG, "transpose: B > 64");
    const int grid = (int)((M + 31) / 32);
    k_transpose_bm_mb<C><<<grid, 256, 0, st>>>((const C*)in, (C*)out, B, M);
    SPTB_LAUNCHED();
    return SPTB_OK;
}
template int launch_transpose_bm_to_mb<float>(const void*, void*, int, int64_t, cudaStream_t);
template int launch_transpose_bm_to_mb<double>(const void*, void*, int, int64_t, cudaStream_t);

// ---------------------------------------------------------------------------
// pack / unpack between caller slices and complex [b][len]
// (pairing a + ib of slices (2k, 2k+1): pipeline.py:122-159)
// gridDim = (nblk, B): block-uniform unit b, each thread handles 4 elements
// of the plane with independent loads issued before any store.
// ---------------------------------------------------------------------------
constexpr int PK = 4;

template <typename TI, typename R>
__global__ void __launch_bounds__(256)
k_pack(const TI* __restrict__ in, bool cplx, long long n, long long u0, int nb, long long len,
       const R* __restrict__ plane, typename Cplx<R>::T* __restrict__ out) {
    using C = typename Cplx<R>::T;
    const int b = blockIdx.y;
    C* dst = out + (size_t)b * len;
    const long long u = u0 + b;
    const TI* pa = nullptr;
    const TI* pb = nullptr;
    long long es = 1;
    if (b < nb) {
        if (cplx) {
            pa = in + u * len * 2;
            pb = pa + 1;
            es = 2;
        } else {
            pa = in + (2 * u) * len;
            pb = (2 * u + 1 < n) ? in + (2 * u + 1) * len : nullptr;
        }
    }
    const long long stride = (long long)gridDim.x * blockDim.x * PK;
    for (long long i0 = (long long)blockIdx.x * blockDim.x * PK + threadIdx.x; i0 < len; i0 += stride) {
        R re[PK], im[PK], d[PK];
#pragma unroll
        for (int k = 0; k < PK; ++k) {
            const long long i = i0 + (long long)k * blockDim.x;
            re[k] = im[k] = (R)0;
            d[k] = (R)1;
            if (i < len && pa) {
                re[k] = (R)pa[i * es];
                if (pb) im[k] = (R)pb[i * es];
                if (plane) d[k] = plane[i];
            }
        }
#pragma unroll
        for (int k = 0; k < PK; ++k) {
            const long long i = i0 + (long long)k * blockDim.x;
            if (i < len) {
                C v;
                v.x = re[k] * d[k];
                v.y = im[k] * d[k];
                dst[i] = v;
            }
        }
    }
}

template <typename TO, typename R>
__global__ void __launch_bounds__(256)
k_unpack(const typename Cplx<R>::T* __restrict__ z, long long len, const R* __restrict__ plane,
         R scale, TO* __restrict__ out, bool cplx, long long n, long long u0) {
    using C = typename Cplx<R>::T;
    const int b = blockIdx.y;
    const C* src = z + (size_t)b * len;
    const long long u = u0 + b;
    TO* pa;
    TO* pb;
    long long es = 1;
    if (cplx) {
        pa = out + u * len * 2;
        pb = pa + 1;
        es = 2;
    } else {
        pa = out + (2 * u) * len;
        pb = (2 * u + 1 < n) ? out + (2 * u + 1) * len : nullptr;
    }
    const long long stride = (long long)gridDim.x * blockDim.x * PK;
    for (long long i0 = (long long)blockIdx.x * blockDim.x * PK + threadIdx.x; i0 < len; i0 += stride) {
        C v[PK];
        R f[PK];
#pragma unroll
        for (int k = 0; k < PK; ++k) {
            const long long i = i0 + (long long)k * blockDim.x;
            if (i < len) {
                v[k] = src[i];
                f[k] = plane ? plane[i] * scale : scale;
            }
        }
#pragma unroll
        for (int k = 0; k < PK; ++k) {
            const long long i = i0 + (long long)k * blockDim.x;
            if (i < len) {
                pa[i * es] = (TO)(v[k].x * f[k]);
                if (pb) pb[i * es] = (TO)(v[k].y * f[k]);
            }
        }
    }
}

// f32 real pairs, 4 consecutive elements per thread: 128-bit loads and stores
// (the scalar kernels above reach ~55% of HBM bandwidth on 2048^2 planes)
__global__ void __launch_bounds__(256)
k_unpack4(const float4* __restrict__ z, long long len4, const float4* __restrict__ plane, float scale,
          float4* __restrict__ out, long long n, long long u0) {
    const int b = blockIdx.y;
    const long long u = u0 + b;
    const float4* src = z + (size_t)b * len4 * 2;
    float4* pa = out + (size_t)(2 * u) * len4;
    float4* pb = (2 * u + 1 < n) ? out + (size_t)(2 * u + 1) * len4 : nullptr;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len4;
         i += (long long)gridDim.x * blockDim.x) {
        const float4 v0 = __ldcs(src + 2 * i), v1 = __ldcs(src + 2 * i + 1);
        float4 f = make_float4(scale, scale, scale, scale);
        if (plane) {
            const float4 d = __ldg(plane + i);
            f = make_float4(d.x * scale, d.y * scale, d.z * scale, d.w * scale);
        }
        __stcs(pa + i, make_float4(v0.x * f.x, v0.z * f.y, v1.x * f.z, v1.z * f.w));
        if (pb) __stcs(pb + i, make_float4(v0.y * f.x, v0.w * f.y, v1.y * f.z, v1.w * f.w));
    }
}

__global__ void __launch_bounds__(256)
k_pack4(const float4* __restrict__ in, long long len4, const float4* __restrict__ plane, long long n,
        long long u0, int nb, float4* __restrict__ out) {
    const int b = blockIdx.y;
    const long long u = u0 + b;
    float4* dst = out + (size_t)b * len4 * 2;
    const float4* pa = b < nb ? in + (size_t)(2 * u) * len4 : nullptr;
    const float4* pb = (b < nb && 2 * u + 1 < n) ? in + (size_t)(2 * u + 1) * len4 : nullptr;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len4;
         i += (long long)gridDim.x * blockDim.x) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), c = a;
        if (pa) a = __ldcs(pa + i);
        if (pb) c = __ldcs(pb + i);
        if (plane) {
            const float4 d = __ldg(plane + i);
            a = make_float4(a.x * d.x, a.y * d.y, a.z * d.z, a.w * d.w);
            c = make_float4(c.x * d.x, c.y * d.y, c.z * d.z, c.w * d.w);
        }
        dst[2 * i] = make_float4(a.x, c.x, a.y, c.y);
        dst[2 * i + 1] = make_float4(a.z, c.z, a.w, c.w);
    }
}

static bool vec4_ok(const void* a, const void* b, long long len) {
    return len % 4 == 0 && ((uintptr_t)a % 16) == 0 && ((uintptr_t)b % 16) == 0;
}

static dim3 vec_grid(long long len4, int nplanes) {
    const long long per = (len4 + 255) / 256;
    const long long cap = std::max<long long>(1, 148LL * 32 / std::max(1, nplanes));
    return dim3((unsigned)std::max<long long>(1, std::min(per, cap)), (unsigned)nplanes);
}

static int grid_for(long long total) {
    long long g = (total + 255) / 256;
    return (int)std::min<long long>(g, 148LL * 32);
}

static dim3 plane_grid(long long len, int nplanes) {
    long long per = (len + 256LL * PK - 1) / (256LL * PK);
    const long long cap = std::max<long long>(1, 148LL * 16 / std::max(1, nplanes));
    return dim3((unsigned)std::max<long long>(1, std::min(per, std::max<long long>(cap, 1))),
                (unsigned)nplanes);
}

template <typename R>
int launch_pack(const void* in, int fmt, int64_t n, int64_t u0, int nb, int B, int64_t len,
                const void* plane, void* out, cudaStream_t st) {
    using C = typename Cplx<R>::T;
    const bool cplx = fmt & SPTB_FMT_COMPLEX;
    if constexpr (sizeof(R) == 4) {
        if (!cplx && !(fmt & SPTB_FMT_F64) && vec4_ok(in, out, len) && ((uintptr_t)plane % 16) == 0) {
            k_pack4<<<vec_grid(len / 4, B), 256, 0, st>>>((const float4*)in, len / 4, (const float4*)plane, n,
                                                         u0, nb, (float4*)out);
            SPTB_LAUNCHED();
            return SPTB_OK;
        }
    }
    const dim3 grid = plane_grid(len, B);
    if (fmt & SPTB_FMT_F64)
        k_pack<double, R><<<grid, 256, 0, st>>>((const double*)in, cplx, n, u0, nb, len,
                                                (const R*)plane, (C*)out);
    else
        k_pack<float, R><<<grid, 256, 0, st>>>((const float*)in, cplx, n, u0, nb, len,
                                               (const R*)plane, (C*)out);
    SPTB_LAUNCHED();
    return SPTB_OK;
}
template int launch_pack<float>(const void*, int, int64_t, int64_t, int, int, int64_t, const void*, void*, cudaStream_t);
template int launch_pack<double>(const void*, int, int64_t, int64_t, int, int, int64_t, const void*, void*, cudaStream_t);

template <typename R>
int launch_unpack(const void* in, int64_t len, const void* plane, double scale, void* out,
                  int fmt, int64_t n, int64_t u0, int nb, cudaStream_t st) {
    using C = typename Cplx<R>::T;
    const bool cplx = fmt & SPTB_FMT_COMPLEX;
    if constexpr (sizeof(R) == 4) {
        if (!cplx && !(fmt & SPTB_FMT_F64) && vec4_ok(in, out, len) && ((uintptr_t)plane % 16) == 0) {
            k_unpack4<<<vec_grid(len / 4, nb), 256, 0, st>>>((const float4*)in, len / 4, (const float4*)plane,
                                                            (float)scale, (float4*)out, n, u0);
            SPTB_LAUNCHED();
            return SPTB_OK;
        }
    }
    const dim3 grid = plane_grid(len, nb);
    if (fmt & SPTB_FMT_F64)
        k_unpack<double, R><<<grid, 256, 0, st>>>((const C*)in, len, (const R*)plane, (R)scale,
                                                  (double*)out, cplx, n, u0);
    else
        k_unpack<float, R><<<grid, 256, 0, st>>>((const C*)in, len, (const R*)plane, (R)scale,
                                                 (float*)out, cplx, n, u0);
    SPTB_LAUNCHED();
    return SPTB_OK;
}
template int launch_unpack<float>(const void*, int64_t, const void*, double, void*, int, int64_t, int64_t, int, cudaStream_t);
template int launch_unpack<double>(const void*, int64_t, const void*, double, void*, int, int64_t, int64_t, int, cudaStream_t);

// z[b][t][p] *= w[p] (wlen == P) or w[t*P+p] (wlen == N)
template <typename R>
__global__ void k_weight_sino(typename Cplx<R>::T* __restrict__ z, const R* __restrict__ w,
                              long long wlen, int P, long long N, int B) {
    const long long total = (long long)B * N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long s = e % N;
        const R f = (wlen == N) ? w[s] : w[s % P];
        auto v = z[e];
        v.x *= f;
        v.y *= f;
        z[e] = v;
    }
}

template <typename R>
int launch_weight_sino(void* z, const void* w, int64_t wlen, int P, int64_t N, int B,
                       cudaStream_t st) {
    using C = typename Cplx<R>::T;
    k_weight_sino<R><<<grid_for((long long)B * N), 256, 0, st>>>((C*)z, (const R*)w, wlen, P, N, B);
    SPTB_LAUNCHED();
    return SPTB_OK;
}
template int launch_weight_sino<float>(void*, const void*, int64_t, int, int64_t, int, cudaStream_t);
template int launch_weight_sino<double>(void*, const void*, int64_t, int, int64_t, int, cudaStream_t);

// F-order grid rows (gx*Y+gy) <-> C-order rows (gy*X+gx), B complex per row
template <typename C>
__global__ void k_permute_grid(const C* __restrict__ in, C* __restrict__ out, int X, int Y,
                               int B, bool f_to_c) {
    const long long total = (long long)X * Y * B;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long mc = e / B;
        const int b = (int)(e - mc * B);
        const long long gy = mc / X, gx = mc - gy * X;
        const long long mf = gx * Y + gy;
        if (f_to_c)
            out[e] = in[mf * B + b];
        else
            out[mf * B + b] = in[e];
    }
}

template <typename R>
int launch_permute_grid(const void* in, void* out, int X, int Y, int B, bool f_to_c,
                        cudaStream_t st) {
    using C = typename Cplx<R>::T;
    k_permute_grid<C><<<grid_for((long long)X * Y * B), 256, 0, st>>>((const C*)in, (C*)out, X, Y,
                                                                       B, f_to_c);
    SPTB_LAUNCHED();
    return SPTB_OK;
}
template int launch_permute_grid<float>(const void*, void*, int, int, int, bool, cudaStream_t);
template int launch_permute_grid<double>(const void*, void*, int, int, int, bool, cudaStream_t);

}  // namespace sptb
