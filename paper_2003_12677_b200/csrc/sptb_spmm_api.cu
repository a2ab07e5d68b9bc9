// sptb_spmm: the reference's free spmv/spmm (operators.py:124-136) in the
// reference's own index convention (F-order grid rows, sample rows in
// (theta, p) order, nrhs innermost), plus the SpMM benchmark hook.
#include "sptb_internal.cuh"

#include <algorithm>
#include <vector>

namespace sptb {

template <typename R> struct CplxT;
template <> struct CplxT<float> { using T = float2; };
template <> struct CplxT<double> { using T = double2; };

// caller row of device row r: grid rows map C-order -> F-order (X > 0), sample
// rows map s' -> order[s'] (rowmap), otherwise identity
__device__ __forceinline__ long long caller_row(long long r, int X, int Y, const int* rowmap) {
    if (rowmap) return rowmap[r];
    if (X == 0) return r;
    const long long gy = r / X, gx = r - gy * X;
    return gx * Y + gy;
}

// caller (rows, nrhs) columns [c0, c0+nb) -> device [row][B] (BATCH_OUTER: [b][row])
template <typename TI, typename R, bool BATCH_OUTER>
__global__ void k_gather_cols(const TI* __restrict__ in, long long rows, long long nrhs,
                              long long c0, int nb, int B, int X, int Y, const int* rowmap,
                              typename CplxT<R>::T* __restrict__ out) {
    const long long total = rows * B;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        long long r;
        int b;
        if (BATCH_OUTER) {
            b = (int)(e / rows);
            r = e - (long long)b * rows;
        } else {
            r = e / B;
            b = (int)(e - r * B);
        }
        typename CplxT<R>::T v;
        v.x = 0;
        v.y = 0;
        if (b < nb) {
            const long long o = (caller_row(r, X, Y, rowmap) * nrhs + c0 + b) * 2;
            v.x = (R)in[o];
            v.y = (R)in[o + 1];
        }
        out[e] = v;
    }
}

template <typename TO, typename R>
__global__ void k_scatter_cols(const typename CplxT<R>::T* __restrict__ in, long long rows,
                               long long nrhs, long long c0, int nb, int B, int X, int Y,
                               const int* rowmap, TO* __restrict__ out) {
    const long long total = rows * nb;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long r = e / nb;
        const int b = (int)(e - r * nb);
        const auto v = in[r * B + b];
        const long long o = (caller_row(r, X, Y, rowmap) * nrhs + c0 + b) * 2;
        out[o] = (TO)v.x;
        out[o + 1] = (TO)v.y;
    }
}

static int gridn(long long n) {
    long long g = (n + 255) / 256;
    return (int)std::min<long long>(std::max<long long>(g, 1), 148LL * 32);
}

template <typename R>
int spmm_ref(sptb_plan* p, int which, const void* x, void* y, int64_t nrhs, int fmt) {
    using C = typename CplxT<R>::T;
    const bool adjoint = which == SPTB_MAT_SH;
    const void* vals = p->S.val;
    if (which == SPTB_MAT_SW) {
        if (!p->SW_val) return fail(SPTB_ERR_STATE, "no filter set");
        vals = p->SW_val;
    }
    const int64_t in_rows = adjoint ? p->M : p->N, out_rows = adjoint ? p->N : p->M;
    cudaStream_t st = p->stream;
    const size_t eb = (fmt & SPTB_FMT_F64) ? 8 : 4;
    bool dx = true, dy = true;
    is_device_ptr(x, &dx);
    is_device_ptr(y, &dy);
    const void* xs = x;
    void* ys = y;
    const size_t xbytes = eb * 2 * (size_t)in_rows * nrhs, ybytes = eb * 2 * (size_t)out_rows * nrhs;
    if (!dx) {
        SPTB_TRY(ensure_stage(&p->stage_in, &p->stage_in_bytes, xbytes));
        SPTB_CUDA(cudaMemcpyAsync(p->stage_in, x, xbytes, cudaMemcpyHostToDevice, st));
        xs = p->stage_in;
    }
    if (!dy) {
        SPTB_TRY(ensure_stage(&p->stage_out, &p->stage_out_bytes, ybytes));
        ys = p->stage_out;
    }
    int Bw = 1;
    while (Bw < std::min<int64_t>(p->max_batch, nrhs)) Bw <<= 1;
    SPTB_TRY(ensure_work(p, Bw));
    const bool f64 = fmt & SPTB_FMT_F64;
    for (int64_t c0 = 0; c0 < nrhs; c0 += p->max_batch) {
        const int nb = (int)std::min<int64_t>(p->max_batch, nrhs - c0);
        int B = 1;
        while (B < nb) B <<= 1;
        if (adjoint) {
            // grid operand batch-outer [b][m] -> patch S^H -> [s'][b] -> caller (theta, p) rows
            C* xin = (C*)p->G0;
            C* yout = (C*)p->S1;
            if (f64)
                k_gather_cols<double, R, true><<<gridn(in_rows * B), 256, 0, st>>>(
                    (const double*)xs, in_rows, nrhs, c0, nb, B, p->X, p->Y, nullptr, xin);
            else
                k_gather_cols<float, R, true><<<gridn(in_rows * B), 256, 0, st>>>(
                    (const float*)xs, in_rows, nrhs, c0, nb, B, p->X, p->Y, nullptr, xin);
            SPTB_LAUNCHED();
            SPTB_TRY(launch_spmm_sh_patch<R>(p, xin, yout, B, nullptr, st));
            if (f64)
                k_scatter_cols<double, R><<<gridn(out_rows * nb), 256, 0, st>>>(
                    yout, out_rows, nrhs, c0, nb, B, 0, 0, p->shp.order, (double*)ys);
            else
                k_scatter_cols<float, R><<<gridn(out_rows * nb), 256, 0, st>>>(
                    yout, out_rows, nrhs, c0, nb, B, 0, 0, p->shp.order, (float*)ys);
            SPTB_LAUNCHED();
        } else {
            // sample operand [s'][b] -> S (columns renumbered) -> [m][b] -> caller F-order rows
            C* xin = (C*)p->S1;
            C* yout = (C*)p->G1;
            if (f64)
                k_gather_cols<double, R, false><<<gridn(in_rows * B), 256, 0, st>>>(
                    (const double*)xs, in_rows, nrhs, c0, nb, B, 0, 0, p->shp.order, xin);
            else
                k_gather_cols<float, R, false><<<gridn(in_rows * B), 256, 0, st>>>(
                    (const float*)xs, in_rows, nrhs, c0, nb, B, 0, 0, p->shp.order, xin);
            SPTB_LAUNCHED();
            SPTB_TRY(launch_spmm<R>(s_permuted(p), vals, xin, yout, B, false, nullptr, st));
            if (f64)
                k_scatter_cols<double, R><<<gridn(out_rows * nb), 256, 0, st>>>(
                    yout, out_rows, nrhs, c0, nb, B, p->X, p->Y, nullptr, (double*)ys);
            else
                k_scatter_cols<float, R><<<gridn(out_rows * nb), 256, 0, st>>>(
                    yout, out_rows, nrhs, c0, nb, B, p->X, p->Y, nullptr, (float*)ys);
            SPTB_LAUNCHED();
        }
    }
    if (!dy) SPTB_CUDA(cudaMemcpyAsync(y, ys, ybytes, cudaMemcpyDeviceToHost, st));
    SPTB_CUDA(cudaStreamSynchronize(st));
    return SPTB_OK;
}

// ---------------------------------------------------------------- benchmark hook

template <typename C>
__global__ void k_fill_pattern(C* x, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned h = (unsigned)(i * 2654435761u);
        C v;
        v.x = (float)((h & 0xffff) * (1.0 / 65536.0) - 0.5);
        v.y = (float)((h >> 16) * (1.0 / 65536.0) - 0.5);
        x[i] = v;
    }
}

// exactly the launches gridrec / radon issue: S^H = patch kernel over [b][m]
// with rows written in sample order (radon's TMA inverse FFT1 reads them);
// S / S diag(w) = the S kernel over [s][b] (sample order, after the fused
// FFT1) -> [b][m]
template <typename R>
int time_spmm(sptb_plan* p, int which, int B, int reps, double* ms) {
    using C = typename CplxT<R>::T;
    const bool adjoint = which == SPTB_MAT_SH;
    const void* vals = p->S.val;
    if (which == SPTB_MAT_SW) {
        if (!p->SW_val) return fail(SPTB_ERR_STATE, "no filter set");
        vals = p->SW_val;
    }
    SPTB_TRY(ensure_work(p, B));
    C* x = (C*)(adjoint ? p->G0 : p->S1);
    C* y = (C*)(adjoint ? p->S1 : p->G0);
    const long long nx = (long long)B * (adjoint ? p->M : p->N);
    k_fill_pattern<C><<<gridn(nx), 256, 0, p->stream>>>(x, nx);
    SPTB_LAUNCHED();
    auto launch = [&]() -> int {
        if (adjoint) return launch_spmm_sh_patch<R>(p, x, y, B, nullptr, p->stream, tma_ok(p, x));
        return launch_spmm_s_sample<R>(p, vals, x, y, B, p->stream);
    };
    for (int w = 0; w < 2; ++w) SPTB_TRY(launch());
    cudaEvent_t e0, e1;
    SPTB_CUDA(cudaEventCreate(&e0));
    SPTB_CUDA(cudaEventCreate(&e1));
    SPTB_CUDA(cudaEventRecord(e0, p->stream));
    for (int r = 0; r < reps; ++r) SPTB_TRY(launch());
    SPTB_CUDA(cudaEventRecord(e1, p->stream));
    SPTB_CUDA(cudaEventSynchronize(e1));
    float t = 0;
    SPTB_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms = (double)t / reps;
    return SPTB_OK;
}

}  // namespace sptb

using namespace sptb;

extern "C" int sptb_spmm(sptb_plan* p, int32_t which, const void* x, void* y, int64_t nrhs,
                         int32_t fmt) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    if (!(fmt & SPTB_FMT_COMPLEX)) return fail(SPTB_ERR_ARG, "spmm operands are complex");
    if (nrhs < 1) return fail(SPTB_ERR_ARG, "nrhs must be >= 1");
    if (which != SPTB_MAT_S && which != SPTB_MAT_SH && which != SPTB_MAT_SW)
        return fail(SPTB_ERR_ARG, "unknown matrix");
    cudaSetDevice(p->device);
    return p->prec == SPTB_PREC_F64 ? spmm_ref<double>(p, which, x, y, nrhs, fmt)
                                    : spmm_ref<float>(p, which, x, y, nrhs, fmt);
}

extern "C" int sptb_time_spmm(sptb_plan* p, int32_t which, int32_t B, int32_t reps,
                              double* ms_per_launch, int64_t* distinct_inputs) {
    if (!p || !ms_per_launch) return fail(SPTB_ERR_ARG, "null argument");
    if (B < 1 || B > 64 || (B & (B - 1))) return fail(SPTB_ERR_ARG, "B must be a power of two <= 64");
    if (reps < 1) return fail(SPTB_ERR_ARG, "reps must be >= 1");
    if (which != SPTB_MAT_S && which != SPTB_MAT_SH && which != SPTB_MAT_SW)
        return fail(SPTB_ERR_ARG, "unknown matrix");
    cudaSetDevice(p->device);
    if (distinct_inputs) {
        // input rows of S are samples (rows of S^H) and vice versa: count non-empty ones
        const DevCSR& other = (which == SPTB_MAT_SH) ? p->S : p->SH;
        std::vector<int> rp(other.rows + 1);
        SPTB_CUDA(cudaMemcpy(rp.data(), other.row_ptr, sizeof(int) * rp.size(), cudaMemcpyDeviceToHost));
        int64_t c = 0;
        for (int64_t i = 0; i < other.rows; ++i) c += rp[i + 1] > rp[i];
        *distinct_inputs = c;
    }
    return p->prec == SPTB_PREC_F64 ? time_spmm<double>(p, which, B, reps, ms_per_launch)
                                    : time_spmm<float>(p, which, B, reps, ms_per_launch);
}
