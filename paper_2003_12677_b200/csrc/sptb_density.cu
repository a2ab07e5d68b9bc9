// Density-compensation weights on the device: density_filter_solve
// (operators.py:189-236).  CGLS on || |S| d - 1 ||_2 over per-sample weights d
// (the entry magnitudes carry the sampling density; the phases are unit
// modulus), then clamp >= 0 and symmetrise d(theta, p) = d(theta, -p) so the
// folded operator stays real-to-real (operators.py:227-232).
//
// |S| and |S|^T are applied straight from the plan's CSR pair (S rows = grid
// cells, S^H rows = samples) with the magnitude taken on the fly; vectors are
// float64 like the reference; reductions are fixed-shape two-pass trees, so
// the weights are bitwise reproducible run to run.
#include "sptb_internal.cuh"

#include <cmath>
#include <vector>

namespace sptb {

namespace {

constexpr int DT = 256;
constexpr int DRED = 1024;  // first-pass partial sums

// y[r] = sum_k |v_k| x[col_k]; one warp per row (rows of S reach 4852 entries)
template <typename C>
__global__ void k_abs_spmv(const int* __restrict__ rp, const int* __restrict__ col, const C* __restrict__ val,
                           const double* __restrict__ x, double* __restrict__ y, long long rows) {
    const int lane = threadIdx.x & 31;
    const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = w0; r < rows; r += nw) {
        double a = 0;
        for (int k = rp[r] + lane; k < rp[r + 1]; k += 32) {
            const C v = val[k];
            a += sqrt((double)v.x * (double)v.x + (double)v.y * (double)v.y) * x[col[k]];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) y[r] = a;
    }
}

// partial[b] = sum over a fixed slice of i of a[i] * c[i]   (c == nullptr: a[i]^2)
__global__ void k_dot_partial(const double* __restrict__ a, const double* __restrict__ c, long long n,
                              double* __restrict__ partial) {
    __shared__ double sh[DT];
    double s = 0;
    const long long per = (n + DRED - 1) / DRED;
    const long long i0 = blockIdx.x * per, i1 = min(n, i0 + per);
    for (long long i = i0 + threadIdx.x; i < i1; i += DT) s += c ? a[i] * c[i] : a[i] * a[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = DT / 2; o; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}
__global__ void k_dot_final(const double* __restrict__ partial, double* __restrict__ out) {
    __shared__ double sh[DRED];
    for (int i = threadIdx.x; i < DRED; i += blockDim.x) sh[i] = partial[i];
    __syncthreads();
    for (int o = DRED / 2; o; o >>= 1) {
        for (int i = threadIdx.x; i < o; i += blockDim.x) sh[i] += sh[i + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// y = a * x + b * y  (elementwise)
__global__ void k_axpby(double a, const double* __restrict__ x, double b, double* __restrict__ y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = a * x[i] + b * y[i];
}
__global__ void k_fill(double v, double* __restrict__ y, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = v;
}
// d = max(x, 0) symmetrised in p:  0.5 (d[t][j] + d[t][(P - j) % P])
__global__ void k_clamp_sym(const double* __restrict__ x, double* __restrict__ d, int T, int P) {
    const long long n = (long long)T * P;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long t = i / P;
        const int j = (int)(i - t * P);
        const double a = fmax(x[i], 0.0), b = fmax(x[t * P + (P - j) % P], 0.0);
        d[i] = 0.5 * (a + b);
    }
}

unsigned gridn(long long n) { return (unsigned)std::min<long long>((n + DT - 1) / DT, 148LL * 32); }

template <typename C>
int density_solve(sptb_plan* p, int max_iter, double tol, double* w_out, double* hist, int* n_hist,
                  int* converged, double* final_res) {
    const long long M = p->M, N = p->N;
    cudaStream_t st = p->stream;
    double *x = nullptr, *r = nullptr, *s = nullptr, *pp = nullptr, *q = nullptr, *part = nullptr, *sc = nullptr;
    std::vector<void*> bufs;
    auto alloc = [&](double** b, long long n) -> int {
        SPTB_CUDA(cudaMalloc(b, sizeof(double) * std::max<long long>(n, 1)));
        bufs.push_back(*b);
        return SPTB_OK;
    };
    struct Free {
        std::vector<void*>& b;
        ~Free() {
            for (void* v : b) cudaFree(v);
        }
    } fr{bufs};
    SPTB_TRY(alloc(&x, N));
    SPTB_TRY(alloc(&r, M));
    SPTB_TRY(alloc(&s, N));
    SPTB_TRY(alloc(&pp, N));
    SPTB_TRY(alloc(&q, M));
    SPTB_TRY(alloc(&part, DRED));
    SPTB_TRY(alloc(&sc, 1));
    auto spmv_S = [&](const double* in, double* out) -> int {  // |S| in : N -> M
        k_abs_spmv<C><<<gridn(M * 32), DT, 0, st>>>(p->S.row_ptr, p->S.col, (const C*)p->S.val, in, out, M);
        SPTB_LAUNCHED();
        return SPTB_OK;
    };
    auto spmv_SH = [&](const double* in, double* out) -> int {  // |S|^T in : M -> N
        k_abs_spmv<C><<<gridn(N * 32), DT, 0, st>>>(p->SH.row_ptr, p->SH.col, (const C*)p->SH.val, in, out, N);
        SPTB_LAUNCHED();
        return SPTB_OK;
    };
    auto dot = [&](const double* a, const double* c, long long n, double* out) -> int {
        k_dot_partial<<<DRED, DT, 0, st>>>(a, c, n, part);
        SPTB_LAUNCHED();
        k_dot_final<<<1, DT, 0, st>>>(part, sc);
        SPTB_LAUNCHED();
        SPTB_CUDA(cudaMemcpyAsync(out, sc, sizeof(double), cudaMemcpyDeviceToHost, st));
        SPTB_CUDA(cudaStreamSynchronize(st));
        return SPTB_OK;
    };
    k_fill<<<gridn(N), DT, 0, st>>>(0.0, x, N);
    SPTB_LAUNCHED();
    k_fill<<<gridn(M), DT, 0, st>>>(1.0, r, M);  // r = b = 1
    SPTB_LAUNCHED();
    SPTB_TRY(spmv_SH(r, s));
    SPTB_CUDA(cudaMemcpyAsync(pp, s, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
    double gamma = 0, rr = 0;
    SPTB_TRY(dot(s, nullptr, N, &gamma));
    SPTB_TRY(dot(r, nullptr, M, &rr));
    int nh = 0;
    hist[nh++] = std::sqrt(rr);
    *converged = 0;
    for (int it = 0; it < max_iter; ++it) {
        SPTB_TRY(spmv_S(pp, q));
        double qq = 0;
        SPTB_TRY(dot(q, nullptr, M, &qq));
        if (qq <= 0 || gamma <= 0) break;
        const double alpha = gamma / qq;
        k_axpby<<<gridn(N), DT, 0, st>>>(alpha, pp, 1.0, x, N);
        SPTB_LAUNCHED();
        k_axpby<<<gridn(M), DT, 0, st>>>(-alpha, q, 1.0, r, M);
        SPTB_LAUNCHED();
        SPTB_TRY(dot(r, nullptr, M, &rr));
        hist[nh++] = std::sqrt(rr);
        if (hist[nh - 1] <= tol * hist[0]) {
            *converged = 1;
            break;
        }
        SPTB_TRY(spmv_SH(r, s));
        double gnew = 0;
        SPTB_TRY(dot(s, nullptr, N, &gnew));
        k_axpby<<<gridn(N), DT, 0, st>>>(1.0, s, gnew / gamma, pp, N);  // p = s + (gnew/gamma) p
        SPTB_LAUNCHED();
        gamma = gnew;
    }
    *n_hist = nh;
    k_clamp_sym<<<gridn(N), DT, 0, st>>>(x, s, p->T, p->P);
    SPTB_LAUNCHED();
    SPTB_TRY(spmv_S(s, q));
    k_fill<<<gridn(M), DT, 0, st>>>(1.0, r, M);
    SPTB_LAUNCHED();
    k_axpby<<<gridn(M), DT, 0, st>>>(1.0, q, -1.0, r, M);  // r = q - 1
    SPTB_LAUNCHED();
    double fr2 = 0;
    SPTB_TRY(dot(r, nullptr, M, &fr2));
    *final_res = std::sqrt(fr2);
    SPTB_CUDA(cudaMemcpyAsync(w_out, s, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
    SPTB_CUDA(cudaStreamSynchronize(st));
    return SPTB_OK;
}

}  // namespace

}  // namespace sptb

using namespace sptb;

extern "C" int sptb_density_filter(sptb_plan* p, int32_t max_iter, double tol, double* weights_out,
                                   double* residual_history, int32_t* n_history, int32_t* converged,
                                   double* final_residual) {
    if (!p || !weights_out || !residual_history || !n_history || !converged || !final_residual)
        return fail(SPTB_ERR_ARG, "null argument");
    if (max_iter < 0) return fail(SPTB_ERR_ARG, "max_iter must be >= 0");
    cudaSetDevice(p->device);
    int nh = 0, cv = 0;
    const int rc = p->prec == SPTB_PREC_F64
                       ? density_solve<double2>(p, max_iter, tol, weights_out, residual_history, &nh, &cv,
                                                final_residual)
                       : density_solve<float2>(p, max_iter, tol, weights_out, residual_history, &nh, &cv,
                                               final_residual);
    *n_history = nh;
    *converged = cv;
    return rc;
}
