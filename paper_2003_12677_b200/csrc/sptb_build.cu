// Device build of the gridding matrices (K12) and host-side deapodization.
//
// Restates gridding.py:84-195 (build_coo -> prune -> coo_to_csr) and
// geometry.py:146-272 (kernel, kernel transform, deapodization) for the
// device index convention (row-major grid m = gy*n_x + gx, sample
// s = t*n_p + j).  Structural decisions (rint ties, kernel support, border,
// Nyquist ring, in-bounds) are evaluated in IEEE double with explicit
// round-to-nearest intrinsics so they reproduce the reference's numpy
// evaluation exactly; S^H comes out in sample order with stencil-ordered
// columns, S is obtained by a stable radix sort on the grid row.
#include "sptb_internal.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

namespace sptb {

namespace {

struct BuildArgs {
    int P, T, X, Y, W, family;
    double beta, sigma, i0beta, thr;
    const double* ct;     // cos(theta), device
    const double* st;     // sin(theta), device
    const double2* ramp;  // per detector bin phase (mirrored bins conjugated)
};

__device__ __forceinline__ double signed_freq(int j, int P) {
    const int h = P / 2;
    return (double)(((j + h) % P) - h);
}

// kernel_eval (geometry.py:146-161)
__device__ double kern(const BuildArgs& a, double t) {
    const double half = a.W * 0.5;
    if (!(fabs(t) < half)) return 0.0;
    if (a.family == SPTB_KERNEL_KB) {
        const double q = __ddiv_rn(__dmul_rn(2.0, t), (double)a.W);
        const double r = fmax(__dsub_rn(1.0, __dmul_rn(q, q)), 0.0);
        return cyl_bessel_i0(a.beta * sqrt(r)) / a.i0beta;
    }
    const double z = t / a.sigma;
    return exp(-0.5 * z * z);
}

// nearest node + fractional offset with negative-frequency mirroring
// (gridding.py:100-121; polar_coords geometry.py:202-215)
__device__ void sample_base(const BuildArgs& a, int t, int j, double& rx, double& ry,
                            double& fx, double& fy) {
    const double pj = signed_freq(j, a.P);
    const bool nyq = (a.P % 2 == 0) && (j == a.P / 2);
    const bool neg = pj < 0 && !nyq;
    const int jj = neg ? (a.P - j) % a.P : j;
    const double p = signed_freq(jj, a.P);
    const double px = __dadd_rn(__dmul_rn(a.ct[t], p), a.X / 2.0);
    const double py = __dadd_rn(__dmul_rn(a.st[t], p), a.Y / 2.0);
    rx = rint(px);
    ry = rint(py);
    fx = __dsub_rn(px, rx);
    fy = __dsub_rn(py, ry);
    if (neg) {
        rx = __dsub_rn((double)a.X, rx);
        ry = __dsub_rn((double)a.Y, ry);
        fx = -fx;
        fy = -fy;
    }
}

// One stencil entry: returns true when kept; sets grid row (C order) and value.
__device__ bool entry(const BuildArgs& a, int t, int j, double rx, double ry, double fx,
                      double fy, int si, int sj, int& m, double2& v) {
    const int h = a.W / 2;
    const int sx = si - h, sy = sj - h;
    const long long gx = (long long)rx + sx, gy = (long long)ry + sy;
    if (gx < 0 || gx >= a.X || gy < 0 || gy >= a.Y) return false;
    if (gx == 0 || gy == 0) return false;                      // border (:136-137)
    if ((a.P % 2 == 0) && j == a.P / 2) return false;           // Nyquist (:138-140)
    const double kx = kern(a, __dsub_rn(fx, (double)sx));
    const double ky = kern(a, __dsub_rn(fy, (double)sy));
    const double wgt = kx * ky * ((((gx + gy) % 2) == 0) ? 1.0 : -1.0);
    const double2 r = a.ramp[j];
    v = make_double2(wgt * r.x, wgt * r.y);
    if (!(hypot(v.x, v.y) > a.thr)) return false;               // prune (:159-163)
    m = (int)(gy * a.X + gx);
    return true;
}

__global__ void k_count(BuildArgs a, int* cnt) {
    const long long N = (long long)a.T * a.P;
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < N;
         s += (long long)gridDim.x * blockDim.x) {
        const int t = (int)(s / a.P), j = (int)(s % a.P);
        double rx, ry, fx, fy;
        sample_base(a, t, j, rx, ry, fx, fy);
        int c = 0;
        for (int si = 0; si < a.W; ++si)
            for (int sj = 0; sj < a.W; ++sj) {
                int m;
                double2 v;
                c += entry(a, t, j, rx, ry, fx, fy, si, sj, m, v) ? 1 : 0;
            }
        cnt[s] = c;
    }
}

// S^H row s: columns m (stencil order), values conj(v)  (gridding.py:179)
template <typename C>
__global__ void k_fill(BuildArgs a, const int* rp, int* col, C* val, int* ent_s) {
    const long long N = (long long)a.T * a.P;
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < N;
         s += (long long)gridDim.x * blockDim.x) {
        const int t = (int)(s / a.P), j = (int)(s % a.P);
        double rx, ry, fx, fy;
        sample_base(a, t, j, rx, ry, fx, fy);
        int o = rp[s];
        for (int si = 0; si < a.W; ++si)
            for (int sj = 0; sj < a.W; ++sj) {
                int m;
                double2 v;
                if (entry(a, t, j, rx, ry, fx, fy, si, sj, m, v)) {
                    col[o] = m;
                    C c;
                    c.x = v.x;
                    c.y = -v.y;
                    val[o] = c;
                    ent_s[o] = (int)s;
                    ++o;
                }
            }
    }
}

__global__ void k_iota(int* v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        v[i] = (int)i;
}

__global__ void k_row_hist(const int* keys, long long n, int* cnt) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        atomicAdd(cnt + keys[i], 1);
}

template <typename C>
__global__ void k_gather_S(const int* perm, const int* ent_s, const C* shv, int* col, C* val,
                           long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int k = perm[i];
        col[i] = ent_s[k];
        C v = shv[k];
        v.y = -v.y;
        val[i] = v;
    }
}

int grid_of(long long n) {
    long long g = (n + 255) / 256;
    return (int)(g < 148LL * 64 ? (g > 0 ? g : 1) : 148LL * 64);
}


template <typename C>
int build_typed(sptb_plan* p, const BuildArgs& a) {
    cudaStream_t st = p->stream;
    const long long N = p->N, M = p->M;
    int* cnt = nullptr;
    SPTB_CUDA(cudaMalloc(&cnt, sizeof(int) * (N + 1)));
    SPTB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * (N + 1), st));
    k_count<<<grid_of(N), 256, 0, st>>>(a, cnt);
    SPTB_LAUNCHED();

    DevCSR& SH = p->SH;
    SH.rows = N;
    SH.cols = M;
    SPTB_CUDA(cudaMalloc(&SH.row_ptr, sizeof(int) * (N + 1)));
    size_t tmp_bytes = 0;
    SPTB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, SH.row_ptr, (int)(N + 1), st));
    void* tmp = nullptr;
    SPTB_CUDA(cudaMalloc(&tmp, tmp_bytes));
    SPTB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, SH.row_ptr, (int)(N + 1), st));
    SPTB_CUDA(cudaFree(tmp));
    int nnz = 0;
    SPTB_CUDA(cudaMemcpyAsync(&nnz, SH.row_ptr + N, sizeof(int), cudaMemcpyDeviceToHost, st));
    SPTB_CUDA(cudaStreamSynchronize(st));
    SH.nnz = nnz;
    SH.max_row = a.W * a.W;

    const size_t nn = nnz > 0 ? (size_t)nnz : 1;
    int* ent_s = nullptr;
    SPTB_CUDA(cudaMalloc(&SH.col, sizeof(int) * nn));
    SPTB_CUDA(cudaMalloc(&SH.val, sizeof(C) * nn));
    SPTB_CUDA(cudaMalloc(&ent_s, sizeof(int) * nn));
    k_fill<C><<<grid_of(N), 256, 0, st>>>(a, SH.row_ptr, SH.col, (C*)SH.val, ent_s);
    SPTB_LAUNCHED();

    // S = (S^H)^H : stable radix sort of entries by grid row
    DevCSR& S = p->S;
    S.rows = M;
    S.cols = N;
    S.nnz = nnz;
    SPTB_CUDA(cudaMalloc(&S.row_ptr, sizeof(int) * (M + 1)));
    SPTB_CUDA(cudaMalloc(&S.col, sizeof(int) * (nn + 4)));  // +4: 16-byte bulk-copy slack (S kernel staging)
    SPTB_CUDA(cudaMalloc(&S.val, sizeof(C) * (nn + 4)));
    int *keys_out = nullptr, *idx_in = nullptr, *idx_out = nullptr, *rcnt = nullptr;
    SPTB_CUDA(cudaMalloc(&keys_out, sizeof(int) * nn));
    SPTB_CUDA(cudaMalloc(&idx_in, sizeof(int) * nn));
    SPTB_CUDA(cudaMalloc(&idx_out, sizeof(int) * nn));
    SPTB_CUDA(cudaMalloc(&rcnt, sizeof(int) * (M + 1)));
    k_iota<<<grid_of(nnz), 256, 0, st>>>(idx_in, nnz);
    SPTB_LAUNCHED();
    int end_bit = 1;
    while ((1LL << end_bit) < M) ++end_bit;
    tmp_bytes = 0;
    SPTB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, SH.col, keys_out, idx_in,
                                              idx_out, nnz, 0, end_bit, st));
    SPTB_CUDA(cudaMalloc(&tmp, tmp_bytes));
    SPTB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, SH.col, keys_out, idx_in, idx_out,
                                              nnz, 0, end_bit, st));
    SPTB_CUDA(cudaFree(tmp));
    SPTB_CUDA(cudaMemsetAsync(rcnt, 0, sizeof(int) * (M + 1), st));
    k_row_hist<<<grid_of(nnz), 256, 0, st>>>(keys_out, nnz, rcnt);
    SPTB_LAUNCHED();
    tmp_bytes = 0;
    SPTB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, rcnt, S.row_ptr, (int)(M + 1), st));
    SPTB_CUDA(cudaMalloc(&tmp, tmp_bytes));
    SPTB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, rcnt, S.row_ptr, (int)(M + 1), st));
    int* dmax = nullptr;
    SPTB_CUDA(cudaMalloc(&dmax, sizeof(int)));
    size_t tb2 = 0;
    SPTB_CUDA(cub::DeviceReduce::Max(nullptr, tb2, rcnt, dmax, (int)M, st));
    void* tmp2 = nullptr;
    SPTB_CUDA(cudaMalloc(&tmp2, tb2));
    SPTB_CUDA(cub::DeviceReduce::Max(tmp2, tb2, rcnt, dmax, (int)M, st));
    k_gather_S<C><<<grid_of(nnz), 256, 0, st>>>(idx_out, ent_s, (const C*)SH.val, S.col,
                                                 (C*)S.val, nnz);
    SPTB_LAUNCHED();
    int mx = 0;
    SPTB_CUDA(cudaMemcpyAsync(&mx, dmax, sizeof(int), cudaMemcpyDeviceToHost, st));
    SPTB_CUDA(cudaStreamSynchronize(st));
    S.max_row = mx;
    for (void* q : {(void*)tmp, tmp2, (void*)dmax, (void*)keys_out, (void*)idx_in,
                    (void*)idx_out, (void*)rcnt, (void*)ent_s, (void*)cnt})
        SPTB_CUDA(cudaFree(q));
    return SPTB_OK;
}

// ---------------------------------------------------------------- patch grouping of S^H

__global__ void k_centers(BuildArgs a, int* cx, int* cy) {
    const long long N = (long long)a.T * a.P;
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < N;
         s += (long long)gridDim.x * blockDim.x) {
        double rx, ry, fx, fy;
        sample_base(a, (int)(s / a.P), (int)(s % a.P), rx, ry, fx, fy);
        cx[s] = (int)rx;
        cy[s] = (int)ry;
    }
}

// complex64 records {byte offset of the cell in a box plane, re, im, 0} (16 B);
// complex128 records {cell, 0, re, im} (32 B)  -- see sptb_patch.cu PRec
__global__ void k_patch_meta_f32(const int* emap, const unsigned* cell, const float2* val,
                                 void* meta, long long n) {
    float4* out = reinterpret_cast<float4*>(meta);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float2 v = val[emap[i]];
        out[i] = make_float4(__uint_as_float(cell[i] * 8u), v.x, v.y, 0.f);
    }
}
__global__ void k_patch_meta_f64(const int* emap, const unsigned* cell, const double2* val,
                                 void* meta, long long n) {
    struct alignas(16) Rec { unsigned cell, pad; double2 v; };
    Rec* out = reinterpret_cast<Rec*>(meta);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        Rec r;
        r.cell = cell[i];
        r.pad = 0;
        r.v = val[emap[i]];
        out[i] = r;
    }
}

__global__ void k_map_cols(const int* col, const int* perm, int* out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = perm[col[i]];
}

// slot-mode rows: sval[r][k] = S^H value of entry src[r*10+k] (zero when < 0);
// slot 9 carries the box cell of the block origin in .x
template <typename C>
__global__ void k_slot_vals(const int* src, const int* base, const C* val, C* out, long long nrows) {
    const long long n = nrows * SLOT_STRIDE;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / SLOT_STRIDE;
        const int k = (int)(i - r * SLOT_STRIDE);
        C v;
        v.x = 0;
        v.y = 0;
        if (k == 9) {
            if (sizeof(v.x) == 4) v.x = __int_as_float(base[r]);
            else v.x = __longlong_as_double((long long)base[r]);
        } else if (src[i] >= 0) {
            v = val[src[i]];
        }
        out[i] = v;
    }
}

// Group S^H rows by the PATCH_W x PATCH_W grid patch of their stencil centre
// (the rint node of the polar sample, gridding.py:104-121).  Slot mode (kernel
// width 3) stores each regular row as 9 fixed slots; record mode stores every
// nonzero by its cell in the patch box.  Host-side bookkeeping, once per plan.
int build_patches(sptb_plan* p, const BuildArgs& a) {
    PatchSH& sp = p->shp;
    const int X = p->X, Y = p->Y;
    const int64_t N = p->N, nnz = p->SH.nnz;
    sp.halo = a.W / 2;
    sp.bw = PATCH_W + 2 * sp.halo;
    sp.npx = (X + PATCH_W - 1) / PATCH_W;
    sp.npy = (Y + PATCH_W - 1) / PATCH_W;
    sp.slot_mode = (a.W == 3) ? 1 : 0;
    int *dcx = nullptr, *dcy = nullptr;
    SPTB_CUDA(cudaMalloc(&dcx, sizeof(int) * N));
    SPTB_CUDA(cudaMalloc(&dcy, sizeof(int) * N));
    k_centers<<<grid_of(N), 256, 0, p->stream>>>(a, dcx, dcy);
    SPTB_LAUNCHED();
    std::vector<int> cx(N), cy(N), rp(N + 1), col(nnz > 0 ? nnz : 1);
    SPTB_CUDA(cudaMemcpy(cx.data(), dcx, sizeof(int) * N, cudaMemcpyDeviceToHost));
    SPTB_CUDA(cudaMemcpy(cy.data(), dcy, sizeof(int) * N, cudaMemcpyDeviceToHost));
    SPTB_CUDA(cudaMemcpy(rp.data(), p->SH.row_ptr, sizeof(int) * (N + 1), cudaMemcpyDeviceToHost));
    if (nnz) SPTB_CUDA(cudaMemcpy(col.data(), p->SH.col, sizeof(int) * nnz, cudaMemcpyDeviceToHost));
    cudaFree(dcx);
    cudaFree(dcy);
    const int64_t npatch = (int64_t)sp.npx * sp.npy;
    std::vector<int> pid(N);
    std::vector<int> base(sp.slot_mode ? N : 0);
    std::vector<int64_t> cnt(npatch + 2, 0);  // last bucket: irregular rows
    for (int64_t s = 0; s < N; ++s) {
        const int gx = std::min(std::max(cx[s], 0), X - 1), gy = std::min(std::max(cy[s], 0), Y - 1);
        int q = (gy / PATCH_W) * sp.npx + gx / PATCH_W;
        if (sp.slot_mode) {
            // slot-mode patches are shifted one cell in x (patch px covers x in
            // [8px+1, 8px+8], box origin 8px): the TMA box origin must sit on a
            // 16-byte boundary of the grid row
            const int px = std::min(std::max(gx - 1, 0) / PATCH_W, sp.npx - 1);
            q = (gy / PATCH_W) * sp.npx + px;
            const int bx0 = px * PATCH_W, by0 = (q / sp.npx) * PATCH_W - sp.halo;
            const int lx0 = cx[s] - 1 - bx0, ly0 = cy[s] - 1 - by0;
            const bool reg = lx0 >= 0 && lx0 + 2 < sp.bw && ly0 >= 0 && ly0 + 2 < sp.bw;
            for (int k = rp[s]; k < rp[s + 1]; ++k) {
                const int ex = col[k] % X - cx[s], ey = col[k] / X - cy[s];
                if (ex < -1 || ex > 1 || ey < -1 || ey > 1)
                    return fail(SPTB_ERR_STATE, "slot build: stencil entry outside the 3x3 block");
            }
            if (!reg) q = (int)npatch;
            base[s] = reg ? ly0 * sp.bw + lx0 : 0;
        }
        pid[s] = q;
        cnt[q + 1]++;
    }
    for (int64_t q = 0; q <= npatch; ++q) cnt[q + 1] += cnt[q];
    std::vector<int> order(N), perm(N);
    {
        std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
        for (int64_t s = 0; s < N; ++s) {  // stable counting sort by patch
            const int64_t d = fill[pid[s]]++;
            order[d] = (int)s;
            perm[s] = (int)d;
        }
    }
    sp.n_reg = sp.slot_mode ? cnt[npatch] : N;
#ifndef SPTB_CLASS_ORDER
#define SPTB_CLASS_ORDER 1
#endif
    if (sp.slot_mode && SPTB_CLASS_ORDER) {
        // within a patch: border class (TL, T, TR, R, BR, B, BL, L, interior),
        // then stencil-centre cell, then sample: each neighbour of the patch
        // finds the samples it shares with it in at most two contiguous runs
        std::vector<std::pair<uint64_t, int>> key;
        for (int64_t q = 0; q < npatch; ++q) {
            key.clear();
            const int px = (int)(q % sp.npx), py = (int)(q / sp.npx);
            for (int64_t r = cnt[q]; r < cnt[q + 1]; ++r) {
                const int sm = order[r];
                const int lx = cx[sm] - PATCH_W * px - 1, ly = cy[sm] - PATCH_W * py;
                const int c = border_class(lx, ly);
                key.push_back({((uint64_t)c << 40) | ((uint64_t)(ly * PATCH_W + lx) << 32) | (uint64_t)sm, sm});
            }
            std::sort(key.begin(), key.end());
            int64_t r = cnt[q];
            for (auto& kv : key) {
                order[r] = kv.second;
                perm[kv.second] = (int)r;
                ++r;
            }
        }
    }
    std::vector<int4> items;
    std::vector<unsigned char> item_perm;
    std::vector<int> rpn, emap, slot_src, base_r;
    std::vector<unsigned> cell;
    if (sp.slot_mode) {
        // slot rows for every sample (irregular rows too: the output-tiled S
        // reads them; their base is unused)
        slot_src.assign((size_t)std::max<int64_t>(N, 1) * SLOT_STRIDE, -1);
        base_r.assign(std::max<int64_t>(N, 1), 0);
        for (int64_t r = 0; r < N; ++r) {
            const int s = order[r];
            base_r[r] = base[s];
            for (int k = rp[s]; k < rp[s + 1]; ++k) {
                const int ex = col[k] % X - cx[s], ey = col[k] / X - cy[s];
                slot_src[(size_t)r * SLOT_STRIDE + (ey + 1) * 3 + (ex + 1)] = k;
            }
        }
        for (int64_t q = 0; q < npatch; ++q)
            for (int64_t r0 = cnt[q]; r0 < cnt[q + 1]; r0 += PATCH_ITEM_ROWS)
                items.push_back(make_int4((int)q, (int)r0, (int)std::min<int64_t>(cnt[q + 1], r0 + PATCH_ITEM_ROWS), 0));
        // full items (the dense centre) launch first so the long CTAs do not
        // form the tail; spatial order is kept within both groups (L2 reuse of halos)
        std::stable_partition(items.begin(), items.end(),
                              [](const int4& it) { return it.z - it.y == PATCH_ITEM_ROWS; });
        // per item, the order in which its rows are handed to lane groups: rows
        // whose block origins differ in x parity alternate, so the two rows of a
        // half-warp read cells of opposite parity (conflict-free box reads in
        // the TMA kernel, whose plane stride is even)
        item_perm.assign(items.size() * PATCH_ITEM_ROWS, 0);
        std::vector<int> ev, od;
        for (size_t it = 0; it < items.size(); ++it) {
            ev.clear();
            od.clear();
            for (int r = items[it].y; r < items[it].z; ++r) ((base_r[r] & 1) ? od : ev).push_back(r - items[it].y);
            size_t ie = 0, io = 0;
            for (int k = 0; k < items[it].z - items[it].y; ++k) {
                const bool take_even = ie < ev.size() && (k % 2 == 0 || io >= od.size());
                item_perm[it * PATCH_ITEM_ROWS + k] = (unsigned char)(take_even ? ev[ie++] : od[io++]);
            }
        }
        int *dsrc = nullptr, *dbase = nullptr;
        SPTB_CUDA(cudaMalloc(&dsrc, sizeof(int) * slot_src.size()));
        SPTB_CUDA(cudaMalloc(&dbase, sizeof(int) * base_r.size()));
        SPTB_CUDA(cudaMalloc(&sp.sval, p->csize * slot_src.size()));
        SPTB_CUDA(cudaMemcpy(dsrc, slot_src.data(), sizeof(int) * slot_src.size(), cudaMemcpyHostToDevice));
        SPTB_CUDA(cudaMemcpy(dbase, base_r.data(), sizeof(int) * base_r.size(), cudaMemcpyHostToDevice));
        if (p->prec == SPTB_PREC_F64)
            k_slot_vals<double2><<<grid_of((long long)slot_src.size()), 256, 0, p->stream>>>(
                dsrc, dbase, (const double2*)p->SH.val, (double2*)sp.sval, N);
        else
            k_slot_vals<float2><<<grid_of((long long)slot_src.size()), 256, 0, p->stream>>>(
                dsrc, dbase, (const float2*)p->SH.val, (float2*)sp.sval, N);
        SPTB_LAUNCHED();
        SPTB_CUDA(cudaStreamSynchronize(p->stream));
        cudaFree(dsrc);
        cudaFree(dbase);
    } else {
        rpn.assign(N + 1, 0);
        emap.assign(nnz > 0 ? nnz : 1, 0);
        cell.assign(nnz > 0 ? nnz : 1, 0);
        int64_t e = 0;
        for (int64_t q = 0; q < npatch; ++q) {
            const int bx0 = (int)(q % sp.npx) * PATCH_W - sp.halo, by0 = (int)(q / sp.npx) * PATCH_W - sp.halo;
            for (int64_t r0 = cnt[q]; r0 < cnt[q + 1]; r0 += PATCH_ITEM_ROWS) {
                const int64_t r1 = std::min<int64_t>(cnt[q + 1], r0 + PATCH_ITEM_ROWS);
                const int64_t ebeg = e;
                for (int64_t r = r0; r < r1; ++r) {
                    const int s = order[r];
                    for (int k = rp[s]; k < rp[s + 1]; ++k) {
                        const int gx = col[k] % X, gy = col[k] / X;
                        const int lx = gx - bx0, ly = gy - by0;
                        if (lx < 0 || lx >= sp.bw || ly < 0 || ly >= sp.bw)
                            return fail(SPTB_ERR_STATE, "patch build: stencil outside its box");
                        cell[e] = (unsigned)(ly * sp.bw + lx);
                        emap[e] = k;
                        ++e;
                    }
                    rpn[r + 1] = (int)e;
                }
                sp.max_item_nnz = std::max<int>(sp.max_item_nnz, (int)(e - ebeg));
                items.push_back(make_int4((int)q, (int)r0, (int)r1, (int)ebeg));
            }
        }
    }
    sp.n_items = (int64_t)items.size();
    SPTB_CUDA(cudaMalloc(&sp.items, sizeof(int4) * std::max<size_t>(items.size(), 1)));
    SPTB_CUDA(cudaMalloc(&sp.perm, sizeof(int) * N));
    SPTB_CUDA(cudaMalloc(&sp.order, sizeof(int) * N));
    SPTB_CUDA(cudaMalloc(&sp.s_colp, sizeof(int) * (std::max<int64_t>(nnz, 1) + 4)));
    if (!items.empty())
        SPTB_CUDA(cudaMemcpy(sp.items, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice));
    if (!item_perm.empty()) {
        SPTB_CUDA(cudaMalloc(&sp.item_perm, item_perm.size()));
        SPTB_CUDA(cudaMemcpy(sp.item_perm, item_perm.data(), item_perm.size(), cudaMemcpyHostToDevice));
    }
    SPTB_CUDA(cudaMemcpy(sp.perm, perm.data(), sizeof(int) * N, cudaMemcpyHostToDevice));
    SPTB_CUDA(cudaMemcpy(sp.order, order.data(), sizeof(int) * N, cudaMemcpyHostToDevice));
    if (!sp.slot_mode) {
        const size_t rec = p->csize == 16 ? 32 : 16;
        int* demap = nullptr;
        unsigned* dcell = nullptr;
        SPTB_CUDA(cudaMalloc(&sp.rp, sizeof(int) * (N + 1)));
        SPTB_CUDA(cudaMalloc(&sp.meta, rec * std::max<int64_t>(nnz, 1)));
        SPTB_CUDA(cudaMalloc(&demap, sizeof(int) * std::max<int64_t>(nnz, 1)));
        SPTB_CUDA(cudaMalloc(&dcell, sizeof(unsigned) * std::max<int64_t>(nnz, 1)));
        SPTB_CUDA(cudaMemcpy(sp.rp, rpn.data(), sizeof(int) * (N + 1), cudaMemcpyHostToDevice));
        if (nnz) {
            SPTB_CUDA(cudaMemcpy(demap, emap.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));
            SPTB_CUDA(cudaMemcpy(dcell, cell.data(), sizeof(unsigned) * nnz, cudaMemcpyHostToDevice));
            if (p->prec == SPTB_PREC_F64)
                k_patch_meta_f64<<<grid_of(nnz), 256, 0, p->stream>>>(demap, dcell, (const double2*)p->SH.val, sp.meta, nnz);
            else
                k_patch_meta_f32<<<grid_of(nnz), 256, 0, p->stream>>>(demap, dcell, (const float2*)p->SH.val, sp.meta, nnz);
            SPTB_LAUNCHED();
        }
        SPTB_CUDA(cudaStreamSynchronize(p->stream));
        cudaFree(demap);
        cudaFree(dcell);
    }
    if (nnz) {
        k_map_cols<<<grid_of(nnz), 256, 0, p->stream>>>(p->S.col, sp.perm, sp.s_colp, nnz);
        SPTB_LAUNCHED();
    }
    SPTB_CUDA(cudaStreamSynchronize(p->stream));
    return SPTB_OK;
}

// ---------------------------------------------------------------- host math

double bessel_i0(double x) {
    // power series sum_k ((x/2)^k / k!)^2, converges for all x
    const double q = 0.25 * x * x;
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 1000; ++k) {
        term *= q / ((double)k * (double)k);
        sum += term;
        if (term < 1e-18 * sum) break;
    }
    return sum;
}

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
    x.assign(n, 0.0);
    w.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        double dp = 0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = 0.0;
            for (int k = 1; k <= n; ++k) {
                const double p2 = p1;
                p1 = p0;
                p0 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p2) / k;
            }
            dp = n * (z * p0 - p1) / (z * z - 1.0);
            const double dz = p0 / dp;
            z -= dz;
            if (std::fabs(dz) < 1e-16) break;
        }
        x[i] = -z;
        w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
}

// kernel_transform (geometry.py:164-191)
double kernel_ft(const sptb_kernel& k, double nu) {
    if (k.family == SPTB_KERNEL_KB) {
        const double w = k.width;
        const double z2 = k.beta * k.beta - (M_PI * w * nu) * (M_PI * w * nu);
        double out;
        if (z2 > 0) {
            const double z = std::sqrt(z2);
            out = std::sinh(z) / z;
        } else {
            const double z = std::sqrt(-z2);
            out = (std::fabs(z) < 1e-12) ? 1.0 : std::sin(z) / z;
        }
        return out * (w / bessel_i0(k.beta));
    }
    static thread_local std::vector<double> gx, gw;
    if (gx.size() != 64) gauss_legendre(64, gx, gw);
    const double half = k.width / 2.0;
    double s = 0;
    for (int i = 0; i < 64; ++i) {
        const double t = gx[i] * half;
        s += std::cos(2.0 * M_PI * nu * t) * std::exp(-0.5 * (t / k.sigma) * (t / k.sigma)) *
             gw[i] * half;
    }
    return s;
}

}  // namespace

int build_deapo(sptb_plan* p, const sptb_kernel* k) {
    const int X = p->X, Y = p->Y;
    std::vector<double> ax(X), ay(Y);
    for (int i = 0; i < X; ++i) ax[i] = kernel_ft(*k, (i - X / 2.0) / X);
    for (int i = 0; i < Y; ++i) ay[i] = kernel_ft(*k, (i - Y / 2.0) / Y);
    double mx = 0;
    for (double a : ay)
        for (double b : ax) mx = std::max(mx, std::fabs(a * b));
    const double eps = 1e-6 * mx;
    const double r = std::min(X, Y) / 2.0;
    p->deapo_host.assign((size_t)X * Y, 0.0);
    long long bad = 0;
    for (int y = 0; y < Y; ++y) {
        const double dy = y - Y / 2.0;
        for (int x = 0; x < X; ++x) {
            const double dx = x - X / 2.0;
            if (!(dy * dy + dx * dx < r * r)) continue;
            const double apod = ay[y] * ax[x];
            if (std::fabs(apod) < eps) {
                ++bad;
                continue;
            }
            const long long sgn = ((x - X / 2) + (y - Y / 2)) % 2;
            p->deapo_host[(size_t)y * X + x] = (sgn == 0 ? 1.0 : -1.0) / apod;
        }
    }
    if (bad)
        return fail(SPTB_ERR_NEAR_ZERO, "kernel transform vanishes at " + std::to_string(bad) +
                                            " supported grid points; narrow the kernel");
    // separable form for the fused FFT2 kernels: deapo = [dx^2 + dy^2 < r^2] * fx[x] * fy[y]
    std::vector<float> fxy((size_t)X + Y);
    for (int x = 0; x < X; ++x) fxy[x] = (float)((((x - X / 2) % 2) == 0 ? 1.0 : -1.0) / ax[x]);
    for (int y = 0; y < Y; ++y) fxy[(size_t)X + y] = (float)((((y - Y / 2) % 2) == 0 ? 1.0 : -1.0) / ay[y]);
    SPTB_CUDA(cudaMalloc(&p->deapo_xy, fxy.size() * sizeof(float)));
    SPTB_CUDA(cudaMemcpy(p->deapo_xy, fxy.data(), fxy.size() * sizeof(float), cudaMemcpyHostToDevice));
    const size_t n = (size_t)X * Y;
    if (p->prec == SPTB_PREC_F64) {
        SPTB_CUDA(cudaMalloc(&p->deapo, n * sizeof(double)));
        SPTB_CUDA(cudaMemcpy(p->deapo, p->deapo_host.data(), n * sizeof(double),
                             cudaMemcpyHostToDevice));
    } else {
        std::vector<float> f(n);
        for (size_t i = 0; i < n; ++i) f[i] = (float)p->deapo_host[i];
        SPTB_CUDA(cudaMalloc(&p->deapo, n * sizeof(float)));
        SPTB_CUDA(cudaMemcpy(p->deapo, f.data(), n * sizeof(float), cudaMemcpyHostToDevice));
    }
    return SPTB_OK;
}

int build_matrices(sptb_plan* p, const sptb_geometry* g, const sptb_kernel* k) {
    const int P = p->P, T = p->T;
    std::vector<double2> ramp(P);
    std::vector<char> neg(P, 0);
    const int h = P / 2;
    for (int j = 0; j < P; ++j) {
        const double pj = (double)(((j + h) % P) - h);
        neg[j] = pj < 0 && !((P % 2 == 0) && j == P / 2);
        const double th = ((2.0 * M_PI) * p->center) * pj / P;
        ramp[j] = make_double2(std::cos(th), std::sin(th));
    }
    for (int j = 0; j < P; ++j)
        if (neg[j]) {
            const double2 m = ramp[(P - j) % P];
            ramp[j] = make_double2(m.x, -m.y);  // gridding.py:130-131
        }
    double *dct = nullptr, *dst = nullptr;
    double2* dramp = nullptr;
    SPTB_CUDA(cudaMalloc(&dct, sizeof(double) * T));
    SPTB_CUDA(cudaMalloc(&dst, sizeof(double) * T));
    SPTB_CUDA(cudaMalloc(&dramp, sizeof(double2) * P));
    SPTB_CUDA(cudaMemcpy(dct, g->cos_theta, sizeof(double) * T, cudaMemcpyHostToDevice));
    SPTB_CUDA(cudaMemcpy(dst, g->sin_theta, sizeof(double) * T, cudaMemcpyHostToDevice));
    SPTB_CUDA(cudaMemcpy(dramp, ramp.data(), sizeof(double2) * P, cudaMemcpyHostToDevice));
    BuildArgs a;
    a.P = P;
    a.T = T;
    a.X = p->X;
    a.Y = p->Y;
    a.W = k->width;
    a.family = k->family;
    a.beta = k->beta;
    a.sigma = k->sigma;
    a.i0beta = bessel_i0(k->beta);
    a.thr = p->threshold;
    a.ct = dct;
    a.st = dst;
    a.ramp = dramp;
    int rc = (p->prec == SPTB_PREC_F64) ? build_typed<double2>(p, a) : build_typed<float2>(p, a);
    if (rc == SPTB_OK) rc = build_patches(p, a);
    cudaFree(dct);
    cudaFree(dst);
    cudaFree(dramp);
    if (rc != SPTB_OK) return rc;
    return build_deapo(p, k);
}

// ---------------------------------------------------------------- filter fold

// S diag(w) on S's pattern; with threshold > 0 the folded entries with
// |w v| <= threshold are zeroed, as the reference prunes its weighted build
// (gridding.py:146-163)
template <typename C, typename R>
__global__ void k_fold(const int* col, const C* v, C* out, const R* w, long long wlen,
                       long long N, int P, long long nnz, double thr) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nnz;
         i += (long long)gridDim.x * blockDim.x) {
        const long long s = col[i];
        const R f = (wlen == N) ? w[s] : w[s % P];
        C c = v[i];
        c.x *= f;
        c.y *= f;
        if (thr > 0 && !(hypot((double)c.x, (double)c.y) > thr)) c.x = c.y = 0;
        out[i] = c;
    }
}

// w_host -> w_dev (plan precision)
int upload_weights(sptb_plan* p) {
    if (p->w_dev) {
        cudaFree(p->w_dev);
        p->w_dev = nullptr;
    }
    p->w_len = (int64_t)p->w_host.size();
    if (p->w_len == 0) return SPTB_OK;
    const size_t rs = p->csize / 2;
    SPTB_CUDA(cudaMalloc(&p->w_dev, rs * p->w_len));
    if (p->prec == SPTB_PREC_F64) {
        SPTB_CUDA(cudaMemcpy(p->w_dev, p->w_host.data(), rs * p->w_len, cudaMemcpyHostToDevice));
    } else {
        std::vector<float> f(p->w_len);
        for (int64_t i = 0; i < p->w_len; ++i) f[i] = (float)p->w_host[i];
        SPTB_CUDA(cudaMemcpy(p->w_dev, f.data(), rs * p->w_len, cudaMemcpyHostToDevice));
    }
    return SPTB_OK;
}

int fold_filter(sptb_plan* p) {
    const long long nnz = p->S.nnz;
    const size_t cs = p->csize;
    if (p->SW_val) {
        cudaFree(p->SW_val);
        p->SW_val = nullptr;
    }
    p->sseg.pval_ok[1] = false;  // the S kernel's padded copy of S diag(w) is stale
    SPTB_TRY(upload_weights(p));
    if (p->w_len == 0) return SPTB_OK;
    SPTB_CUDA(cudaMalloc(&p->SW_val, cs * ((nnz > 0 ? nnz : 1) + 4)));
    if (nnz == 0) return SPTB_OK;
    // weights multiply in double like the reference's folded build (gridding.py:146-152)
    // -- float plans round the folded value once.
    if (p->prec == SPTB_PREC_F64)
        k_fold<double2, double><<<grid_of(nnz), 256, 0, p->stream>>>(
            p->S.col, (const double2*)p->S.val, (double2*)p->SW_val, (const double*)p->w_dev,
            p->w_len, p->N, p->P, nnz, p->threshold);
    else
        k_fold<float2, float><<<grid_of(nnz), 256, 0, p->stream>>>(
            p->S.col, (const float2*)p->S.val, (float2*)p->SW_val, (const float*)p->w_dev,
            p->w_len, p->N, p->P, nnz, p->threshold);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

}  // namespace sptb
