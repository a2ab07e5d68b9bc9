// S SpMM (adjoint / gridrec direction):  Y[b][m] = S_(w) X,  X [s][b] (batch
// innermost, the FFT1-side operand), Y batch-outer for the inverse 2-D FFT.
// The reference computes it with scipy CSR (operators.py:124-136, 178-184).
//
// Row-segment kernel for complex64 and a 32-vector batch (the production
// gridrec / solver launch):
//   * a TILE is a run of consecutive rows with <= SEG_W nonzeros and <= SEG_TR
//     rows (host-built once per plan from row_ptr); its row pointers, column
//     indices and values are staged in shared memory;
//   * the 16 half-warps of the CTA split the tile's nonzeros evenly at row
//     boundaries; a half-warp walks its nonzeros as one flat stream, lane l
//     owning complex columns 2l, 2l+1 (one 16-byte load per nonzero: the
//     half-warp reads the whole 256-byte X row), SEG_UNR gathers in flight
//     before their packed FP32x2 FMAs; a finished row is written once to the
//     shared output tile -- no per-row unrolled slots, no predicated waste;
//   * the tile leaves through shared memory as 256-byte runs of [b][m]
//     (XOR-swizzled 16-byte slots: conflict-free both ways);
//   * rows longer than SEG_LONG nonzeros (the centre of the polar grid, up to
//     4,852) get one CTA each: 16 fixed contiguous pieces summed in piece
//     order.
// Every row's sum has a fixed order that depends only on the matrix: results
// are deterministic and independent of a vector's batch slot.
#include "sptb_internal.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace sptb {

namespace {

constexpr int SEG_THREADS = 256;  // 8 warps = 16 half-warps
constexpr int SEG_HALVES = SEG_THREADS / 16;
#ifndef SEG_TR_
#define SEG_TR_ 128
#endif
#ifndef SEG_W_
#define SEG_W_ 1024
#endif
#ifndef SEG_EXACT_
#define SEG_EXACT_ 9  // measured 9: 0.649, 10: 0.657, 8: 0.651, 6: 0.676 ms at c2
#endif
#ifndef SEG_MINB_
#define SEG_MINB_ 4
#endif
constexpr int SEG_TR = SEG_TR_;   // rows per tile (shared output tile)
constexpr int SEG_W = SEG_W_;     // nonzeros per tile (staged metadata)
constexpr int SEG_LONG = 128;     // longer rows: one CTA per row
#ifndef SEG_ALIGN2
#define SEG_ALIGN2 1                 // rows laid out on even entries (padded copy of S)
#endif
#ifndef SEG_UNR_
#define SEG_UNR_ 8
#endif
constexpr int SEG_UNR = SEG_UNR_;  // gathers in flight per half-warp (long rows)
constexpr int SEG_EXACT = SEG_EXACT_;  // row lengths with an exactly unrolled body
static_assert(!SEG_ALIGN2 || SEG_EXACT >= 8 || SEG_EXACT % 2 == 0,
              "exact chunks of longer rows must start on even entries (paired loads)");
constexpr int SEG_BB = 32;        // complex columns (batch) of this kernel

// shared memory: out tile [SEG_TR][16] float4 | cols [SEG_W] | vals [SEG_W] float2 | pair records
constexpr int SEG_OUT_BYTES = SEG_TR * (SEG_BB / 2) * 16;
// staged arrays carry 16-byte slack: the bulk copies start at the 16-byte
// boundary below the tile's first entry
constexpr int SEG_COLB = (SEG_W + 4) * 4, SEG_VALB = (SEG_W + 2) * 8, SEG_PAIRB = ((SEG_TR / 2 + 1) * 8 + 31) & ~15;
constexpr int SEG_SMEM = SEG_OUT_BYTES + SEG_COLB + SEG_VALB + SEG_PAIRB;

__device__ __forceinline__ float4 ldg_nc4(const float4* p) { return __ldg(p); }

__device__ __forceinline__ void seg_bulk(void* dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void seg_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\nSW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra SW;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// acc1 += (v.x, v.x) * q,  acc2 += (v.y, v.y) * q   for the lane's two columns;
// the complex product is re = acc1.x - acc2.y, im = acc1.y + acc2.x
struct Acc {
    float2 a1[2], a2[2];
    __device__ __forceinline__ void zero() {
        a1[0] = a1[1] = a2[0] = a2[1] = make_float2(0.f, 0.f);
    }
    __device__ __forceinline__ void mac(float2 v, float4 q) {
        const float2 q0 = make_float2(q.x, q.y), q1 = make_float2(q.z, q.w);
        const float2 vx = make_float2(v.x, v.x), vy = make_float2(v.y, v.y);
        a1[0] = __ffma2_rn(vx, q0, a1[0]);
        a1[1] = __ffma2_rn(vx, q1, a1[1]);
        a2[0] = __ffma2_rn(vy, q0, a2[0]);
        a2[1] = __ffma2_rn(vy, q1, a2[1]);
    }
    // K nonzeros at staged positions j0 .. j0+K-1: all loads first
    // (values are read from shared memory at use: only the K gathers hold
    // registers while in flight)
    template <int K>
    __device__ __forceinline__ void exact(const int* s_col, const float2* s_val, const float4* xl, int j0) {
        float4 q[K];
#if SEG_ALIGN2
        // rows start on even entries: columns two per 8-byte load, values two per 16-byte load
#pragma unroll
        for (int u = 0; u < K; u += 2) {
            const int2 c = *reinterpret_cast<const int2*>(s_col + j0 + u);
            q[u] = ldg_nc4(xl + (size_t)c.x * (SEG_BB / 2));
            if (u + 1 < K) q[u + 1] = ldg_nc4(xl + (size_t)c.y * (SEG_BB / 2));
        }
#pragma unroll
        for (int u = 0; u < K; u += 2) {
            const float4 v = *reinterpret_cast<const float4*>(s_val + j0 + u);
            mac(make_float2(v.x, v.y), q[u]);
            if (u + 1 < K) mac(make_float2(v.z, v.w), q[u + 1]);
        }
#else
#pragma unroll
        for (int u = 0; u < K; ++u) q[u] = ldg_nc4(xl + (size_t)s_col[j0 + u] * (SEG_BB / 2));
#pragma unroll
        for (int u = 0; u < K; ++u) mac(s_val[j0 + u], q[u]);
#endif
    }
    // the first n (< K possible, <= 0 allowed) of K positions; the others load
    // staged entry 0 with weight 0
    template <int K>
    __device__ __forceinline__ void pred(const int* s_col, const float2* s_val, const float4* xl, int j0, int n) {
        float4 q[K];
#pragma unroll
        for (int u = 0; u < K; ++u) q[u] = ldg_nc4(xl + (size_t)s_col[u < n ? j0 + u : 0] * (SEG_BB / 2));
#pragma unroll
        for (int u = 0; u < K; ++u) mac(u < n ? s_val[j0 + u] : make_float2(0.f, 0.f), q[u]);
    }
    __device__ __forceinline__ float4 result() const {
        return make_float4(a1[0].x - a2[0].y, a1[0].y + a2[0].x, a1[1].x - a2[1].y, a1[1].y + a2[1].x);
    }
};

// output tile: row r, 16-byte slot cp (columns 2cp, 2cp+1) at r*16 + (cp ^ (r & 7))
__device__ __forceinline__ int oslot(int r, int cp) { return r * (SEG_BB / 2) + (cp ^ (r & 7)); }

// Rows in length order, in pairs (host-built records); warp w takes pairs
// w, w + 8, ...: half 0 the first row of the pair, half 1 the second.  The
// two rows of a pair almost always have the same length, so both halves run
// the same exactly-unrolled body: K loads in flight, then K packed FMA pairs.
__device__ __forceinline__ void seg_pairs(int np_, const unsigned long long* s_pair, const int* s_col,
                                          const float2* s_val, const float4* xl, float4* out, int tid) {
    const int l = tid & 15;
    const int w = tid >> 5, h2 = (tid >> 4) & 1;
    for (int pi = w; pi < np_; pi += SEG_THREADS / 32) {
        const unsigned long long rec = s_pair[pi];
        const int la = (int)((rec >> 35) & 255), lb = (int)((rec >> 43) & 255);
        const bool has = h2 ? ((rec >> 14) & 1) : true;
        const int my = h2 ? (int)((rec >> 7) & 127) : (int)(rec & 127);
        const int mybeg = h2 ? (int)((rec >> 25) & 1023) : (int)((rec >> 15) & 1023);
        const int mylen = h2 ? lb : la;
        Acc acc;
        acc.zero();
        if (la == lb) {
            int k = 0, n = la;
            if (n > SEG_EXACT) {
                constexpr int CK = SEG_EXACT < 8 ? SEG_EXACT : 8;
                for (; n > SEG_EXACT + CK; k += CK, n -= CK) acc.exact<CK>(s_col, s_val, xl, mybeg + k);
                if (n > SEG_EXACT) {  // two exact pieces
                    acc.exact<CK>(s_col, s_val, xl, mybeg + k);
                    k += CK;
                    n -= CK;
                }
            }
            switch (n) {
#define SEG_CASE(K) \
    case K: acc.exact<K>(s_col, s_val, xl, mybeg + k); break;
                SEG_CASE(1) SEG_CASE(2) SEG_CASE(3) SEG_CASE(4) SEG_CASE(5) SEG_CASE(6)
#if SEG_EXACT_ >= 7
                SEG_CASE(7)
#endif
#if SEG_EXACT_ >= 8
                SEG_CASE(8)
#endif
#if SEG_EXACT_ >= 9
                SEG_CASE(9)
#endif
#if SEG_EXACT_ >= 10
                SEG_CASE(10)
#endif
#undef SEG_CASE
                default: break;
            }
        } else {
            const int nmin = min(la, lb), nmax = max(la, lb);
            int k = 0;
            constexpr int CK = SEG_EXACT < 8 ? SEG_EXACT : 8;
            for (; k + CK <= nmin; k += CK) acc.exact<CK>(s_col, s_val, xl, mybeg + k);
            for (; k < nmax; k += CK) acc.pred<CK>(s_col, s_val, xl, mybeg + k, mylen - k);
        }
        if (has) out[oslot(my, l)] = acc.result();
    }
}

// Y[b][r0 + r] from the shared output tile; warp w takes 16-byte column slots
// cp, lanes consecutive rows (256-byte runs per column)
__device__ __forceinline__ void seg_epilogue(const float4* out, float2* y, long long M, int r0, int nr, int tid) {
    const int w = tid >> 5;
    const int lane = tid & 31;
    for (int cp = w; cp < SEG_BB / 2; cp += SEG_THREADS / 32) {
        float2* yb = y + (size_t)(2 * cp) * M + r0;
        for (int r = lane; r < nr; r += 32) {
            const float4 v = out[oslot(r, cp)];
            yb[r] = make_float2(v.x, v.y);
            yb[r + M] = make_float2(v.z, v.w);
        }
    }
}

__global__ void __launch_bounds__(SEG_THREADS, SEG_MINB_)
k_spmm_seg(const int* __restrict__ row_ptr, const int* __restrict__ col, const float2* __restrict__ val,
           const float2* __restrict__ x, float2* __restrict__ y, long long M,
           const int4* __restrict__ tiles, const unsigned long long* __restrict__ pairs,
           const int* __restrict__ longs, int n_long, const int4* __restrict__ tile_e, int n_tiles, int pf,
           const int* __restrict__ prp) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) unsigned long long stage_bar;
    float4* out = reinterpret_cast<float4*>(smem);
    int* s_col = reinterpret_cast<int*>(smem + SEG_OUT_BYTES);
    float2* s_val = reinterpret_cast<float2*>(smem + SEG_OUT_BYTES + SEG_COLB);
    unsigned long long* s_pair = reinterpret_cast<unsigned long long*>(smem + SEG_OUT_BYTES + SEG_COLB + SEG_VALB);

    const int tid = threadIdx.x, h = tid >> 4, l = tid & 15;
    const float4* xl = reinterpret_cast<const float4*>(x) + l;  // lane's 16 bytes of a 256-byte row

    if ((int)blockIdx.x < n_long) {
        // ---- one long row: 16 contiguous pieces, summed in piece order
        const int r = longs[blockIdx.x];
        const int e0 = prp[r], len = row_ptr[r + 1] - row_ptr[r];
        const int pb = e0 + (int)(((long long)len * h) / SEG_HALVES);
        const int pe = e0 + (int)(((long long)len * (h + 1)) / SEG_HALVES);
        Acc acc;
        acc.zero();
        for (int j = pb; j < pe; j += SEG_UNR) {
            float4 q[SEG_UNR];
#pragma unroll
            for (int u = 0; u < SEG_UNR; ++u)
                if (j + u < pe) q[u] = ldg_nc4(xl + (size_t)__ldg(col + j + u) * (SEG_BB / 2));
#pragma unroll
            for (int u = 0; u < SEG_UNR; ++u)
                if (j + u < pe) acc.mac(__ldg(val + j + u), q[u]);
        }
        out[h * (SEG_BB / 2) + l] = acc.result();
        __syncthreads();
        if (tid < SEG_BB) {
            const int cp = tid >> 1, odd = tid & 1;
            float2 s = make_float2(0.f, 0.f);
            for (int k = 0; k < SEG_HALVES; ++k) {
                const float4 t = out[k * (SEG_BB / 2) + cp];
                s.x += odd ? t.z : t.x;
                s.y += odd ? t.w : t.y;
            }
            y[(size_t)tid * M + r] = s;
        }
        return;
    }

    // ---- a tile of short rows
    // two independent loads (no row_ptr round trip before the staging loads)
    const int4 t = tiles[blockIdx.x - n_long];             // {row begin, row end, pair begin, pairs}
    const int4 te = __ldg(tile_e + (blockIdx.x - n_long));  // {first entry, entries, ...}
    const int r0 = t.x, nr = t.y - t.x, np_ = t.w;
    const int e0 = te.x, ne = te.y;
    // staging by three bulk copies on one mbarrier (16-byte aligned sources:
    // the arrays start at the boundary below e0 / the first pair record)
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&stage_bar);
    const int oc = e0 & 3, ov = e0 & 1, op = t.z & 1;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        const unsigned cb = ((unsigned)(oc + ne) * 4u + 15u) & ~15u, vb = ((unsigned)(ov + ne) * 8u + 15u) & ~15u;
        const unsigned pb = ((unsigned)(op + np_) * 8u + 15u) & ~15u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb), "r"(cb + vb + pb) : "memory");
        seg_bulk(s_col, col + (e0 - oc), cb, sb);
        seg_bulk(s_val, val + (e0 - ov), vb, sb);
        seg_bulk(s_pair, pairs + (t.z - op), pb, sb);
    }
    __syncthreads();  // the mbarrier is initialised
    seg_wait(sb, 0);
    s_col += oc;
    s_val += ov;
    s_pair += op;

    seg_pairs(np_, s_pair, s_col, s_val, xl, out, tid);
    if (pf && tid == 0) {
        // the tile pf launches ahead: pull its columns, values and pair
        // records into L2 so that CTA's staging does not wait on DRAM
        // (measured: 0.750 -> 0.734 ms at c2)
        const int nt = (int)blockIdx.x - n_long + pf;
        if (nt < n_tiles) {
            const int4 te = __ldg(tile_e + nt);
            const unsigned long long ca = reinterpret_cast<unsigned long long>(col + te.x) & ~15ull;
            const unsigned long long va = reinterpret_cast<unsigned long long>(val + te.x) & ~15ull;
            const unsigned long long pa = reinterpret_cast<unsigned long long>(pairs + te.z) & ~15ull;
            const unsigned cb = ((unsigned)te.y * 4u + 31u) & ~15u, vb = ((unsigned)te.y * 8u + 31u) & ~15u;
            const unsigned pbytes = ((unsigned)te.w * 8u + 31u) & ~15u;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(ca), "r"(cb) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(va), "r"(vb) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(pa), "r"(pbytes) : "memory");
        }
        // and the tile records of the CTAs pf + 8 .. pf + 15 ahead (one 128-byte line each)
        const int nt2 = nt + 8;
        if ((nt2 & 7) == 0 && nt2 < n_tiles) {
            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(tiles + nt2) : "memory");
            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(tile_e + nt2) : "memory");
        }
    }
    __syncthreads();
    seg_epilogue(out, y, M, r0, nr, tid);
}

// Host schedule (once per plan, from S's structure): tiles of short rows and the list of long rows (longest first)
int build_seg(sptb_plan* p) {
    SSeg& s = p->sseg;
    if (s.built) return SPTB_OK;
    const int64_t M = p->S.rows;
    std::vector<int> rp0(M + 1), rp(M + 1);
    SPTB_CUDA(cudaMemcpy(rp0.data(), p->S.row_ptr, sizeof(int) * (M + 1), cudaMemcpyDeviceToHost));
    // rp: row pointers of the copy of S the kernel reads (rows on even entries when SEG_ALIGN2)
    rp[0] = 0;
    for (int64_t q = 0; q < M; ++q) {
        const int ln = rp0[q + 1] - rp0[q];
        rp[q + 1] = rp[q] + (SEG_ALIGN2 ? ((ln + 1) & ~1) : ln);
    }
    if ((int64_t)rp[M] < (int64_t)rp0[M]) return fail(SPTB_ERR_STATE, "padded S overflows int32");
    std::vector<int4> tiles;
    std::vector<std::pair<int, int>> longs;
    std::vector<unsigned long long> pairs;
    std::vector<int4> tile_e;  // per tile {first entry, entries, first pair record, pair records}
    int64_t r = 0;
    while (r < M) {
        const int len = rp0[r + 1] - rp0[r];
        if (len > SEG_LONG) {
            longs.push_back({-len, (int)r});
            ++r;
            continue;
        }
        const int64_t r0 = r;
        int nnz = 0;
        while (r < M && r - r0 < SEG_TR) {
            const int ln = rp0[r + 1] - rp0[r], pl = rp[r + 1] - rp[r];
            if (ln > SEG_LONG || nnz + pl > SEG_W) break;
            nnz += pl;
            ++r;
        }
        // the tile's rows by length (stable), paired: record = row a | row b
        // << 7 | has b << 14 | begin a << 15 | begin b << 25 | len a << 35 |
        // len b << 43 (rows, begins tile-local)
        std::vector<std::pair<int, int>> lr;
        for (int64_t q = r0; q < r; ++q) lr.push_back({rp0[q + 1] - rp0[q], (int)(q - r0)});
        std::stable_sort(lr.begin(), lr.end(),
                         [](const std::pair<int, int>& x, const std::pair<int, int>& y) { return x.first < y.first; });
        const int pb = (int)pairs.size();
        for (size_t i = 0; i < lr.size(); i += 2) {
            const int ra = lr[i].second, la = lr[i].first;
            const bool hb = i + 1 < lr.size();
            const int rb = hb ? lr[i + 1].second : 0, lb = hb ? lr[i + 1].first : 0;
            const unsigned long long ba = (unsigned long long)(rp[r0 + ra] - rp[r0]);
            const unsigned long long bb = hb ? (unsigned long long)(rp[r0 + rb] - rp[r0]) : 0ull;
            pairs.push_back((unsigned long long)ra | ((unsigned long long)rb << 7) |
                            ((unsigned long long)hb << 14) | (ba << 15) | (bb << 25) |
                            ((unsigned long long)la << 35) | ((unsigned long long)lb << 43));
        }
        tiles.push_back(make_int4((int)r0, (int)r, pb, (int)pairs.size() - pb));
        tile_e.push_back(make_int4(rp[r0], rp[r] - rp[r0], pb, (int)pairs.size() - pb));
    }
    std::sort(longs.begin(), longs.end());
    std::vector<int> lr(longs.size());
    for (size_t i = 0; i < longs.size(); ++i) lr[i] = longs[i].second;
    s.n_tiles = (int)tiles.size();
    s.n_long = (int)lr.size();
    s.pnnz = rp[M];
    SPTB_CUDA(cudaMalloc(&s.prp, sizeof(int) * (M + 1)));
    SPTB_CUDA(cudaMemcpy(s.prp, rp.data(), sizeof(int) * (M + 1), cudaMemcpyHostToDevice));
    SPTB_CUDA(cudaMalloc(&s.tiles, sizeof(int4) * std::max<size_t>(1, tiles.size())));
    SPTB_CUDA(cudaMalloc(&s.tile_e, sizeof(int4) * std::max<size_t>(1, tile_e.size())));
    if (!tile_e.empty())
        SPTB_CUDA(cudaMemcpy(s.tile_e, tile_e.data(), sizeof(int4) * tile_e.size(), cudaMemcpyHostToDevice));
    SPTB_CUDA(cudaMalloc(&s.longs, sizeof(int) * std::max<size_t>(1, lr.size())));
    SPTB_CUDA(cudaMalloc(&s.pairs, sizeof(unsigned long long) * (std::max<size_t>(1, pairs.size()) + 2)));
    if (!pairs.empty())
        SPTB_CUDA(cudaMemcpy(s.pairs, pairs.data(), sizeof(unsigned long long) * pairs.size(),
                             cudaMemcpyHostToDevice));
    if (!tiles.empty())
        SPTB_CUDA(cudaMemcpy(s.tiles, tiles.data(), sizeof(int4) * tiles.size(), cudaMemcpyHostToDevice));
    if (!lr.empty())
        SPTB_CUDA(cudaMemcpy(s.longs, lr.data(), sizeof(int) * lr.size(), cudaMemcpyHostToDevice));
    s.built = true;
    return SPTB_OK;
}

// row r's entries rp0[r] .. rp0[r+1]-1 -> positions prp[r] ..; pad slots stay zero
template <typename T>
__global__ void k_pad_rows(const int* __restrict__ rp0, const int* __restrict__ prp, const T* __restrict__ src,
                           T* __restrict__ dst, long long M) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < M;
         r += (long long)gridDim.x * blockDim.x) {
        const int b = rp0[r], n = rp0[r + 1] - b, d = prp[r];
        for (int k = 0; k < n; ++k) dst[d + k] = src[b + k];
    }
}

// the kernel's copies of A's columns ([0] S.col, [1] the s' renumbering) and
// values ([0] S.val, [1] SW_val) in the padded row layout, built on first use
int ensure_padded(sptb_plan* p, const DevCSR& A, const void* vals, const int** pc, const float2** pv,
                  cudaStream_t st) {
    SSeg& s = p->sseg;
    if (!SEG_ALIGN2) {
        *pc = A.col;
        *pv = (const float2*)vals;
        return SPTB_OK;
    }
    const int ci = A.col == p->S.col ? 0 : (A.col == p->shp.s_colp ? 1 : -1);
    const int vi = vals == p->S.val ? 0 : (vals == p->SW_val ? 1 : -1);
    if (ci < 0 || vi < 0) return fail(SPTB_ERR_STATE, "S kernel: unknown column or value array");
    const size_t n = (size_t)std::max<int64_t>(s.pnnz, 1) + 4;  // +4: bulk-copy slack
    const unsigned grid = (unsigned)std::min<long long>((p->M + 255) / 256, 148 * 16);
    if (!s.pcol_ok[ci]) {
        if (!s.pcol[ci]) SPTB_CUDA(cudaMalloc(&s.pcol[ci], sizeof(int) * n));
        SPTB_CUDA(cudaMemsetAsync(s.pcol[ci], 0, sizeof(int) * n, st));
        k_pad_rows<int><<<grid, 256, 0, st>>>(A.row_ptr, s.prp, A.col, s.pcol[ci], p->M);
        SPTB_LAUNCHED();
        s.pcol_ok[ci] = true;
    }
    if (!s.pval_ok[vi]) {
        if (!s.pval[vi]) SPTB_CUDA(cudaMalloc(&s.pval[vi], sizeof(float2) * n));
        SPTB_CUDA(cudaMemsetAsync(s.pval[vi], 0, sizeof(float2) * n, st));
        k_pad_rows<float2><<<grid, 256, 0, st>>>(A.row_ptr, s.prp, (const float2*)vals, (float2*)s.pval[vi], p->M);
        SPTB_LAUNCHED();
        s.pval_ok[vi] = true;
    }
    *pc = s.pcol[ci];
    *pv = (const float2*)s.pval[vi];
    return SPTB_OK;
}

}  // namespace

bool spmm_seg_ok(const sptb_plan* p, const void* x, const void* y, int B) {
    return p->prec == SPTB_PREC_F32 && B == SEG_BB && ((uintptr_t)x % 16) == 0 && ((uintptr_t)y % 8) == 0 &&
           p->S.rows < (1LL << 31) && !switches().spmm_rows;
}

int launch_spmm_seg(sptb_plan* p, const DevCSR& A, const void* vals, const void* x, void* y,
                    cudaStream_t st) {
    SPTB_TRY(build_seg(p));
    const SSeg& s = p->sseg;
    const unsigned grid = (unsigned)(s.n_long + s.n_tiles);
    if (grid == 0) return SPTB_OK;
    SPTB_CUDA(set_smem_once((const void*)k_spmm_seg, SEG_SMEM, -1));
    // L2 prefetch distance in tiles (6 waves of 148 SMs; SPTB_SEG_PF overrides, 0: off)
    static const int pf = [] {
        const char* e = getenv("SPTB_SEG_PF");
        return e ? std::max(0, atoi(e)) : 888;
    }();
    const int* pc = nullptr;
    const float2* pv = nullptr;
    SPTB_TRY(ensure_padded(p, A, vals, &pc, &pv, st));
    k_spmm_seg<<<grid, SEG_THREADS, SEG_SMEM, st>>>(A.row_ptr, pc, pv, (const float2*)x, (float2*)y, p->M, s.tiles,
                                                  s.pairs, s.longs, s.n_long, s.tile_e, s.n_tiles, pf, s.prp);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

// Y[b][m] = S_(w) X for X in the patch order s' (solver residuals, S^H side)
template <typename R>
int launch_spmm_s(sptb_plan* p, const void* vals, const void* x_sb, void* y_bm, int B, cudaStream_t st) {
    const DevCSR A = s_permuted(p);
    if (spmm_seg_ok(p, x_sb, y_bm, B)) return launch_spmm_seg(p, A, vals, x_sb, y_bm, st);
    return launch_spmm<R>(A, vals, x_sb, y_bm, B, true, nullptr, st);
}
template int launch_spmm_s<float>(sptb_plan*, const void*, const void*, void*, int, cudaStream_t);
template int launch_spmm_s<double>(sptb_plan*, const void*, const void*, void*, int, cudaStream_t);

// Y[b][m] = S_(w) X for X in sample order s (gridrec after the fused FFT1)
template <typename R>
int launch_spmm_s_sample(sptb_plan* p, const void* vals, const void* x_sb, void* y_bm, int B,
                         cudaStream_t st) {
    if (spmm_seg_ok(p, x_sb, y_bm, B)) return launch_spmm_seg(p, p->S, vals, x_sb, y_bm, st);
    return launch_spmm<R>(p->S, vals, x_sb, y_bm, B, true, nullptr, st);
}
template int launch_spmm_s_sample<float>(sptb_plan*, const void*, const void*, void*, int, cudaStream_t);
template int launch_spmm_s_sample<double>(sptb_plan*, const void*, const void*, void*, int, cudaStream_t);

}  // namespace sptb
