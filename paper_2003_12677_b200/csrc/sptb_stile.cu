// Output-tiled S SpMM (adjoint / gridrec direction):  Y[b][m] = S_(w) X,
// X [s'][b] (batch innermost, the FFT1-side operand), Y batch-outer for the
// inverse 2-D FFT.
//
// S = conj(S^H)^T, and every sample's nonzeros sit in the 3x3 block around its
// stencil centre (gridding.py:104-143), so the nonzeros of an 8x8 tile of grid
// cells come from the samples whose block touches the tile.  One CTA per tile:
//   * cp.async stages, per needed sample, its X row (B complex, contiguous)
//     and its slot row (9 values + base, the S^H slot layout of sptb_patch.cu),
//     plus the chunk's u32 metadata (cell pointers, entries); per-row bulk
//     (TMA) copies measured 3x slower here: ~150 requests of 80-256 B per tile;
//   * a group of 16 lanes per grid cell accumulates conj(v) * X[s] over the
//     cell's entries (lanes own batch columns 2*lig, 2*lig+1: LDS.128 of the
//     staged row, conflict free); tiles touched by more than STILE_CHUNK samples
//     loop over chunks, accumulating in registers (entry order is ascending
//     (s', slot): deterministic and independent of the batch slot);
//   * the 64 x B tile goes through shared memory and leaves as 64-byte row runs
//     of each batch plane.  Tiles without samples write zeros (the grid outside
//     the disk is part of the inverse FFT input).
// The reference computes the same product with scipy CSR (operators.py:124-136,
// 178-184); no per-nonzero column index or value is stored here: an entry is
// 2 bytes (local sample, slot), the values are the slot rows shared with S^H.
#include "sptb_internal.cuh"

#include <algorithm>
#include <vector>

namespace sptb {

namespace {

template <typename R> struct TCplx;
template <> struct TCplx<float> { using T = float2; };
template <> struct TCplx<double> { using T = double2; };

constexpr int TT = 256;  // threads per CTA
constexpr int TG = 16;   // lanes per grid cell

__device__ __forceinline__ void tcp16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem));
}

// BB batch columns; lane lig of a cell group owns columns [CW*lig, CW*lig+CW)
template <typename R, int BB>
__global__ void __launch_bounds__(TT)
k_s_tile(const int* __restrict__ tile_chunk, const int4* __restrict__ chunks,
         const int* __restrict__ samp, const unsigned* __restrict__ meta,
         const typename TCplx<R>::T* __restrict__ vals, int ntx, int X, int Y, long long M,
         const typename TCplx<R>::T* __restrict__ x, typename TCplx<R>::T* __restrict__ y) {
    using C = typename TCplx<R>::T;
    constexpr int CW = BB >= 2 * TG ? BB / TG : 1;    // columns per lane
    constexpr int NL = BB / CW;                       // lanes per cell actually used
    constexpr int NGRP = TT / TG;                     // cell groups per CTA
    constexpr int CPG = STILE * STILE / NGRP;         // cells per group
    constexpr int XROW = BB * (int)sizeof(C);         // staged X row bytes (power of two)
    constexpr int VROW = SLOT_STRIDE * (int)sizeof(C);
    constexpr int UX = XROW / 16, UV = VROW / 16, US = UX + UV;  // 16-byte units per sample
    constexpr int NW = TT / 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ int s_ids[STILE_CHUNK];
    unsigned char* xs = smem_raw;                                   // [CHUNK][BB] C
    unsigned char* vs = xs + STILE_CHUNK * XROW;                    // [CHUNK][10] C
    unsigned* ms = reinterpret_cast<unsigned*>(vs + STILE_CHUNK * VROW);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tile = blockIdx.x;
    const int c0 = tile_chunk[tile], c1 = tile_chunk[tile + 1];
    const int g = tid / TG, lig = tid % TG;

    // accumulators: acc += v * x split as (vr * x) and (vi * x), conj applied at the end
    C ar[CPG][CW], ai[CPG][CW];
#pragma unroll
    for (int j = 0; j < CPG; ++j)
#pragma unroll
        for (int w = 0; w < CW; ++w) ar[j][w].x = ar[j][w].y = ai[j][w].x = ai[j][w].y = 0;

    for (int c = c0; c < c1; ++c) {
        const int4 ch = chunks[c];  // {tile, sample begin, n samples, meta offset (u32 units)}
        const int ns = ch.z;
        const unsigned* mg = meta + ch.w;
        // stage: a warp per sample, lane u < US copies 16-byte unit u of the
        // sample's X row (u < UX) or slot row; then the metadata block
        if (tid < ns) s_ids[tid] = samp[ch.y + tid];
        __syncthreads();
        for (int i = warp; i < ns; i += NW) {
            const long long sm = s_ids[i];
            if (lane < UX)
                tcp16(xs + i * XROW + 16 * lane, reinterpret_cast<const char*>(x + sm * BB) + 16 * lane);
            else if (lane < US)
                tcp16(vs + i * VROW + 16 * (lane - UX),
                      reinterpret_cast<const char*>(vals + sm * SLOT_STRIDE) + 16 * (lane - UX));
        }
        const int mu = (((int)__ldg(mg + STILE * STILE) + STILE * STILE + 1 + 3) & ~3) / 4;
        for (int u = tid; u < mu; u += TT) tcp16(ms + 4 * u, mg + 4 * u);
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();

        if (lig < NL) {
            const unsigned char* xl = xs + lig * CW * (int)sizeof(C);
            const unsigned* ent = ms + STILE * STILE + 1;
#pragma unroll
            for (int j = 0; j < CPG; ++j) {
                const int cell = g + NGRP * j;
                const int e0 = ms[cell], e1 = ms[cell + 1];
#pragma unroll 4
                for (int e = e0; e < e1; ++e) {
                    const unsigned rec = ent[e];  // (local sample << 16) | (local * 10 + slot)
                    const C v = reinterpret_cast<const C*>(vs)[rec & 0xffffu];
                    const C* xp = reinterpret_cast<const C*>(xl + (rec >> 16) * XROW);
                    if constexpr (sizeof(C) == 8 && CW == 2) {
                        const float4 xv = *reinterpret_cast<const float4*>(xp);
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
#pragma unroll
                        for (int w = 0; w < CW; ++w) {
                            const C xv = xp[w];
                            ar[j][w].x = fma(v.x, xv.x, ar[j][w].x);
                            ar[j][w].y = fma(v.x, xv.y, ar[j][w].y);
                            ai[j][w].x = fma(v.y, xv.x, ai[j][w].x);
                            ai[j][w].y = fma(v.y, xv.y, ai[j][w].y);
                        }
                    }
                }
            }
        }
        __syncthreads();  // the stage is refilled by the next chunk
    }

    // conj(v) * x = (vr xr + vi xi, vr xi - vi xr); tile -> shared [b][65]
    C* ot = reinterpret_cast<C*>(smem_raw);
    constexpr int OS = STILE * STILE + 1;
    if (lig < NL) {
#pragma unroll
        for (int j = 0; j < CPG; ++j)
#pragma unroll
            for (int w = 0; w < CW; ++w) {
                C o;
                o.x = ar[j][w].x + ai[j][w].y;
                o.y = ar[j][w].y - ai[j][w].x;
                ot[(lig * CW + w) * OS + g + NGRP * j] = o;
            }
    }
    __syncthreads();
    // cell pairs: thread -> (pair p = tid % 32, plane b = tid / 32 + 8 k)
    const int tx0 = (tile % ntx) * STILE, ty0 = (tile / ntx) * STILE;
    const int pr = tid & 31;
    const int cell = 2 * pr, gx = tx0 + cell % STILE, gy = ty0 + cell / STILE;
    if (gy < Y) {
        C* yo = y + (size_t)gy * X + gx;
#pragma unroll 4
        for (int b = tid >> 5; b < BB; b += NW) {
            const C v0 = ot[b * OS + cell], v1 = ot[b * OS + cell + 1];
            if (gx + 1 < X) {
                yo[(size_t)b * M] = v0;
                yo[(size_t)b * M + 1] = v1;
            } else if (gx < X) {
                yo[(size_t)b * M] = v0;
            }
        }
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
int s_tile_dispatch(const sptb_plan* p, const void* vals, const void* x, void* y, cudaStream_t st) {
    using C = typename TCplx<R>::T;
    const STiles& t = p->stl;
    const int ntiles = t.ntx * t.nty;
    const size_t sm = (size_t)STILE_CHUNK * (BB + SLOT_STRIDE) * sizeof(C) + 4 * (size_t)t.max_meta + 16;
    const size_t smo = (size_t)BB * (STILE * STILE + 1) * sizeof(C);
    const size_t smt = std::max(sm, smo);
    auto kern = k_s_tile<R, BB>;
    SPTB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smt));
    SPTB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    kern<<<ntiles, TT, smt, st>>>(t.tile_chunk, t.chunks, t.samp, t.meta, (const C*)vals, t.ntx, p->X, p->Y,
                                  p->M, (const C*)x, (C*)y);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

}  // namespace

template <typename R>
int launch_spmm_s(const sptb_plan* p, const void* vals, const void* x_sb, void* y_bm, int B,
                  cudaStream_t st) {
    const void* slot = nullptr;
    if (p->stl.tile_chunk && p->shp.sval) {
        if (vals == p->S.val) slot = p->shp.sval;
        else if (vals == p->SW_val && p->stl.swval) slot = p->stl.swval;
    }
    // bulk copies need 16-byte rows and a 16-byte aligned operand
    const bool aligned = ((uintptr_t)x_sb % 16) == 0 && (size_t)B * p->csize >= 16;
    // the tiled kernel is opt-in (SPTB_STILE=1) until it beats the row gather
    static const bool use_tiles = [] {
        const char* e = getenv("SPTB_STILE");
        return e && e[0] == '1';
    }();
    if (!slot || !aligned || !use_tiles)
        return launch_spmm<R>(s_permuted(p), vals, x_sb, y_bm, B, true, nullptr, st);
    switch (B) {
        case 1: return s_tile_dispatch<R, 1>(p, slot, x_sb, y_bm, st);
        case 2: return s_tile_dispatch<R, 2>(p, slot, x_sb, y_bm, st);
        case 4: return s_tile_dispatch<R, 4>(p, slot, x_sb, y_bm, st);
        case 8: return s_tile_dispatch<R, 8>(p, slot, x_sb, y_bm, st);
        case 16: return s_tile_dispatch<R, 16>(p, slot, x_sb, y_bm, st);
        case 32: return s_tile_dispatch<R, 32>(p, slot, x_sb, y_bm, st);
        case 64: return s_tile_dispatch<R, 64>(p, slot, x_sb, y_bm, st);
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

// Host build of the tile lists (once per plan).  Entry (s', slot) of tile t
// for grid cell m = (cy + ey) * X + (cx + ex), slot = (ey + 1) * 3 + (ex + 1).
int build_stiles(sptb_plan* p, const std::vector<int>& cx, const std::vector<int>& cy,
                 const std::vector<int>& rp, const std::vector<int>& col, const std::vector<int>& order) {
    STiles& t = p->stl;
    const int X = p->X, Y = p->Y;
    const int64_t N = p->N;
    t.ntx = (X + STILE - 1) / STILE;
    t.nty = (Y + STILE - 1) / STILE;
    const int64_t ntiles = (int64_t)t.ntx * t.nty;
    std::vector<int64_t> cnt(ntiles + 1, 0);
    for (int64_t r = 0; r < N; ++r) {
        const int s = order[r];
        for (int k = rp[s]; k < rp[s + 1]; ++k) {
            const int gx = col[k] % X, gy = col[k] / X;
            cnt[(gy / STILE) * t.ntx + gx / STILE + 1]++;
        }
    }
    for (int64_t i = 0; i < ntiles; ++i) cnt[i + 1] += cnt[i];
    // entry key within a tile: cell (6 bits) | s' (31 bits) | slot (4 bits), in s' order
    std::vector<uint64_t> ent((size_t)std::max<int64_t>(cnt[ntiles], 1));
    {
        std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
        for (int64_t r = 0; r < N; ++r) {
            const int s = order[r];
            for (int k = rp[s]; k < rp[s + 1]; ++k) {
                const int gx = col[k] % X, gy = col[k] / X;
                const int ti = (gy / STILE) * t.ntx + gx / STILE;
                const int cell = (gy % STILE) * STILE + gx % STILE;
                const int slot = (gy - cy[s] + 1) * 3 + (gx - cx[s] + 1);
                ent[fill[ti]++] = ((uint64_t)cell << 40) | ((uint64_t)r << 4) | (uint64_t)slot;
            }
        }
    }
    std::vector<int> tile_chunk(ntiles + 1, 0), samp;
    std::vector<int4> chunks;
    std::vector<unsigned> meta;
    std::vector<int> smp;
    std::vector<int> cellcnt(STILE * STILE + 1);
    for (int64_t ti = 0; ti < ntiles; ++ti) {
        tile_chunk[ti] = (int)chunks.size();
        const int64_t a = cnt[ti], b = cnt[ti + 1];
        if (a == b) continue;
        smp.clear();
        for (int64_t i = a; i < b; ++i) smp.push_back((int)((ent[i] >> 4) & 0x7fffffffULL));
        std::sort(smp.begin(), smp.end());
        smp.erase(std::unique(smp.begin(), smp.end()), smp.end());
        // entries sorted by (s', slot) within the tile; stable by cell later
        std::sort(ent.begin() + a, ent.begin() + b, [](uint64_t u, uint64_t v) {
            return (u & 0xffffffffffULL) < (v & 0xffffffffffULL);
        });
        const int ns = (int)smp.size();
        int64_t ei = a;
        for (int s0 = 0; s0 < ns; s0 += STILE_CHUNK) {
            const int s1 = std::min(ns, s0 + STILE_CHUNK);
            const int last = smp[s1 - 1];
            int64_t ej = ei;
            while (ej < b && (int)((ent[ej] >> 4) & 0x7fffffffULL) <= last) ++ej;
            std::fill(cellcnt.begin(), cellcnt.end(), 0);
            for (int64_t i = ei; i < ej; ++i) cellcnt[(int)(ent[i] >> 40) + 1]++;
            for (int i = 0; i < STILE * STILE; ++i) cellcnt[i + 1] += cellcnt[i];
            const int nent = (int)(ej - ei);
            const size_t moff = meta.size();
            const int mlen = (nent + STILE * STILE + 1 + 3) & ~3;
            meta.resize(moff + mlen, 0);
            for (int i = 0; i <= STILE * STILE; ++i) meta[moff + i] = (unsigned)cellcnt[i];
            std::vector<int> pos(cellcnt.begin(), cellcnt.end() - 1);
            int li = s0;
            for (int64_t i = ei; i < ej; ++i) {  // ascending (s', slot): per-cell order preserved
                const int sp = (int)((ent[i] >> 4) & 0x7fffffffULL);
                while (smp[li] != sp) ++li;
                const int cell = (int)(ent[i] >> 40);
                meta[moff + STILE * STILE + 1 + pos[cell]++] =
                    ((unsigned)(li - s0) << 16) | (unsigned)((li - s0) * SLOT_STRIDE + (int)(ent[i] & 15));
            }
            t.max_meta = std::max(t.max_meta, mlen);
            chunks.push_back(make_int4((int)ti, (int)samp.size(), s1 - s0, (int)moff));
            samp.insert(samp.end(), smp.begin() + s0, smp.begin() + s1);
            ei = ej;
        }
    }
    tile_chunk[ntiles] = (int)chunks.size();
    if (meta.size() >= (size_t)INT32_MAX) return fail(SPTB_ERR_STATE, "tile metadata too large");
    t.n_chunks = (int64_t)chunks.size();
    SPTB_CUDA(cudaMalloc(&t.tile_chunk, sizeof(int) * tile_chunk.size()));
    SPTB_CUDA(cudaMalloc(&t.chunks, sizeof(int4) * std::max<size_t>(chunks.size(), 1)));
    SPTB_CUDA(cudaMalloc(&t.samp, sizeof(int) * std::max<size_t>(samp.size(), 1)));
    SPTB_CUDA(cudaMalloc(&t.meta, sizeof(unsigned) * std::max<size_t>(meta.size(), 4)));
    SPTB_CUDA(cudaMemcpy(t.tile_chunk, tile_chunk.data(), sizeof(int) * tile_chunk.size(), cudaMemcpyHostToDevice));
    if (!chunks.empty()) {
        SPTB_CUDA(cudaMemcpy(t.chunks, chunks.data(), sizeof(int4) * chunks.size(), cudaMemcpyHostToDevice));
        SPTB_CUDA(cudaMemcpy(t.samp, samp.data(), sizeof(int) * samp.size(), cudaMemcpyHostToDevice));
        SPTB_CUDA(cudaMemcpy(t.meta, meta.data(), sizeof(unsigned) * meta.size(), cudaMemcpyHostToDevice));
    }
    return SPTB_OK;
}

}  // namespace sptb
