// Device-resident batched solvers: FBP, SIRT (BB steps), CGLS, split-Bregman TV.
//
// Restates solvers.py:122-460 for a batch of B complex units (each = two real
// slices = two channels, solvers.py:1-10).  Formulation choices:
//  * Sinogram-space vectors live in the detector-frequency domain in the
//    batch-innermost layout [s][b]:  Rhat = FFT1(r).  Because
//    FFT1(radon(v)) = S^H FFT2(deapo v) exactly (unnormalised FFTs, the
//    reference's gamma collapses to 1/n_p -- SURVEY Appendix A.2), the 1D FFT
//    pair of every "r = b - A u" / "A^H W r" step cancels: an iteration costs
//    one FFT2 + one IFFT2 + two SpMMs.
//  * Per-channel weighted norms come from one complex spectrum by the
//    Hermitian split |F(re)|^2, |F(im)|^2 = (A +- C)/(2 n_p), with
//    A = sum w|R_k|^2, C = sum w Re(R_k R_-k)  (needs symmetric w, which
//    every radial filter is).  Per-channel scaling of a spectral vector mixes
//    bins k and -k (mirror kernel below).
//  * Every scalar of the reference (alpha, beta, gamma, delta, mu, tol,
//    divergence, activity) is computed on the device per unit and channel;
//    reductions are fixed-shape two-stage trees (deterministic, independent
//    of a unit's position in the batch).  The host only polls a lagged
//    "units still active" counter to stop early.
//  * Precision: the operators (SpMM, cuFFT, their fused epilogues) run in the
//    plan precision R.  SIRT recomputes r = b - A u every iteration, so its
//    iterates stay in R.  The Krylov recurrences of CGLS and TV (u, p, r,
//    and TV's d / b / grad residuals) are carried in float64 -- exactly the
//    "fp32 operator outputs, fp64 vectors" regime the survey measured
//    against the 1e-3 solver bar (hard part 6).
#include "sptb_internal.cuh"
#include "sptb_fftcore.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

namespace sptb {

template <typename R> struct CT;
template <> struct CT<float> { using T = float2; };
template <> struct CT<double> { using T = double2; };
using D2 = double2;

enum UnitStatus { RUNNING = 0, ST_CONVERGED = 1, ST_DIVERGED = 2, ST_NONFINITE = 3,
                  ST_ZERO = 4, ST_STOPPED = 5, ST_PAD = 6 };

struct Unit {
    double alpha[2], alpha0[2], beta[2], gamma[2], gamma0[2], bnorm[2];
    double mu[2], lam[2];
    double kap[2];  // TV shrink threshold 1 / lam
    double min_res;
    int act[2];      // per-channel activity of the current CG step
    int status;      // UnitStatus
    int active;      // still iterating (outer loop)
    int stepped;     // took a step this iteration
    int iters;
    int single;      // real input: channel 1 absent
    int converged;
    int inner_stop;  // TV inner CGLS: break flag
    int pad_;
};

struct Global {
    int n_active;
};

// ------------------------------------------------------------------ reductions

constexpr int RT = 256;

template <int K, bool MAX>
__device__ __forceinline__ void block_reduce_store(double (&acc)[K], double* out) {
    __shared__ double sh[K > 0 ? K : 1][RT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double v = acc[k];
        for (int o = 16; o > 0; o >>= 1) {
            const double t = __shfl_down_sync(0xffffffffu, v, o);
            v = MAX ? fmax(v, t) : v + t;
        }
        if (lane == 0) sh[k][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double s = MAX ? 0.0 : 0.0;
        for (int w = 0; w < RT / 32; ++w) s = MAX ? fmax(s, sh[threadIdx.x][w]) : s + sh[threadIdx.x][w];
        out[threadIdx.x] = s;
    }
}

// partial[(blk*B + b)*K + k] -> sums[b*K + k]: one FT-thread block per
// output, threads take blk = t, t + FT, ... and a fixed shuffle + shared
// tree combines them (deterministic).  (One warp per output, 8 blocks for
// 64 sums, left a k_spec finish -- 6144 partials per output -- as 192
// dependent L2 round trips per lane on 8 SMs.)
constexpr int FT = 128;
__global__ void __launch_bounds__(FT) k_finish(const double* __restrict__ part, int nblk, int B, int K, int is_max,
                                              double* __restrict__ sums) {
    __shared__ double sh[FT / 32];
    const int w = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = w / K, k = w % K;
    double s = 0;
#pragma unroll 4
    for (int blk = threadIdx.x; blk < nblk; blk += FT) {
        const double v = part[((size_t)blk * B + b) * K + k];
        s = is_max ? fmax(s, v) : s + v;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_down_sync(0xffffffffu, s, o);
        s = is_max ? fmax(s, t) : s + t;
    }
    if (lane == 0) sh[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = sh[0];
        for (int u = 1; u < FT / 32; ++u) t = is_max ? fmax(t, sh[u]) : t + sh[u];
        sums[w] = t;
    }
}

// grid kernels: gridDim = (nblk, B); block-uniform unit b; element (b, m)
struct GridIdx {
    int X, Y;
};

// elements per thread per k_grid round: 4, or Op::kUnroll for register-heavy
// fp64 stencil ops (TV: 124-136 registers at 4 left one 256-thread CTA per SM)
template <class Op, class = void>
struct OpUnroll {
    static constexpr int value = 4;
};
template <class Op>
struct OpUnroll<Op, std::void_t<decltype(Op::kUnroll)>> {
    static constexpr int value = Op::kUnroll;
};
// elements in flight per thread in k_tv_rowfft: Op::kRowUnroll, else as k_grid
template <class Op, class = void>
struct OpRowUnroll {
    static constexpr int value = OpUnroll<Op>::value;
};
template <class Op>
struct OpRowUnroll<Op, std::void_t<decltype(Op::kRowUnroll)>> {
    static constexpr int value = Op::kRowUnroll;
};

#ifndef TV_UNROLL
#define TV_UNROLL 2
#endif
// ops whose value() result is not a W element (reductions only): k_tv_rowfft
// stores nothing for them
template <class Op, class = void>
struct OpStoresW {
    static constexpr bool value = true;
};
template <class Op>
struct OpStoresW<Op, std::void_t<decltype(Op::kNoW)>> {
    static constexpr bool value = !Op::kNoW;
};
// ops that take the grid coordinates directly (no index split per element)
template <class Op, class = void>
struct OpLoadXY {
    static constexpr bool value = false;
};
template <class Op>
struct OpLoadXY<Op, std::void_t<decltype(&Op::load_xy)>> {
    static constexpr bool value = true;
};
template <class Op, class = void>
struct OpLoadNwXY {
    static constexpr bool value = false;
};
template <class Op>
struct OpLoadNwXY<Op, std::void_t<decltype(&Op::load_nw_xy)>> {
    static constexpr bool value = true;
};
template <int K, bool MAX, class Op>
__global__ void __launch_bounds__(RT) k_grid(Op op, long long M, double* part) {
    const int b = blockIdx.y;
    double acc[K > 0 ? K : 1];
#pragma unroll
    for (int k = 0; k < (K > 0 ? K : 1); ++k) acc[k] = 0;
    if (op.enabled(b)) {
        constexpr int U = OpUnroll<Op>::value;
        using In = typename Op::In;
        const long long stride = (long long)gridDim.x * RT * U;
        for (long long m0 = blockIdx.x * (long long)RT * U + threadIdx.x; m0 < M; m0 += stride) {
            In v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long m = m0 + (long long)u * RT;
                if (m < M) v[u] = op.load(b, (size_t)b * M + m, m);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long m = m0 + (long long)u * RT;
                if (m < M) op.apply(b, (size_t)b * M + m, m, v[u], acc);
            }
        }
    }
    if constexpr (K > 0) block_reduce_store<K, MAX>(acc, part + ((size_t)blockIdx.x * gridDim.y + b) * K);
}

// ------------------------------------------------------------------ helpers

template <typename T>
__device__ __forceinline__ T pos_(T v) { return v > (T)0 ? v : (T)0; }

__device__ __forceinline__ bool finite2(double x, double y) { return isfinite(x) && isfinite(y); }

__device__ __forceinline__ double safe_div(double num, double den, double fb) {
    return den > 0 ? num / den : fb;
}

template <typename C>
__device__ __forceinline__ D2 d2(const C& c) { return make_double2((double)c.x, (double)c.y); }

template <typename R>
__device__ __forceinline__ typename CT<R>::T rc(double x, double y) {
    typename CT<R>::T c;
    c.x = (R)x;
    c.y = (R)y;
    return c;
}

// forward differences (solvers.py:308-314): last column / row zero.  V is
// the storage type of the TV state (the plan's complex type); arithmetic is
// fp64
// grid point m -> (x, y) in 32-bit float-reciprocal arithmetic with a +-1
// fix-up (exact for m < 2^24): the 64-bit m % X and m / X these stencil
// helpers used cost ~90 instructions per element and made the TV passes
// instruction-bound (ncu: 382 M instructions for one gradient-norm pass)
__device__ __forceinline__ void split_m(long long m, int X, int& x, int& y) {
    if (m >= (1LL << 24)) {  // grids beyond 4096^2: exact integer division
        x = (int)(m % X);
        y = (int)(m / X);
        return;
    }
    const int mi = (int)m;
    int q = __float2int_rz(__int2float_rn(mi) * __frcp_rn((float)X));
    int r = mi - q * X;
    if (r < 0) {
        q -= 1;
        r += X;
    } else if (r >= X) {
        q += 1;
        r -= X;
    }
    x = r;
    y = q;
}

template <typename V>
__device__ __forceinline__ D2 grad_x(const V* v, size_t i, long long m, int X) {
    int x, y;
    split_m(m, X, x, y);
    if (x == X - 1) return make_double2(0, 0);
    const D2 a = d2(v[i]), b = d2(v[i + 1]);
    return make_double2(b.x - a.x, b.y - a.y);
}
template <typename V>
__device__ __forceinline__ D2 grad_y(const V* v, size_t i, long long m, int X, int Y) {
    int x, y;
    split_m(m, X, x, y);
    if (y == Y - 1) return make_double2(0, 0);
    const D2 a = d2(v[i]), b = d2(v[i + X]);
    return make_double2(b.x - a.x, b.y - a.y);
}
// -div2d(vx, vy) (solvers.py:317-327), i.e. grad^T
template <typename V>
__device__ __forceinline__ D2 grad_t(const V* vx, const V* vy, size_t i, long long m, int X, int Y) {
    // div2d(vx,vy)[y][x] = vx[x] (x<X-1) - vx[x-1] (x>0) + same along y; return its negative
    int x, y;
    split_m(m, X, x, y);
    double re = 0, im = 0;
    if (x < X - 1) { re += (double)vx[i].x; im += (double)vx[i].y; }
    if (x > 0) { re -= (double)vx[i - 1].x; im -= (double)vx[i - 1].y; }
    if (y < Y - 1) { re += (double)vy[i].x; im += (double)vy[i].y; }
    if (y > 0) { re -= (double)vy[i - X].x; im -= (double)vy[i - X].y; }
    return make_double2(-re, -im);
}
template <typename V>
__device__ __forceinline__ V tv_store(double x, double y) {
    V v;
    v.x = x;
    v.y = y;
    return v;
}

// Raw stencil neighbours, loaded in an op's load() phase and differenced in
// apply(): the loads of all of a thread's elements are then in flight
// together (differencing inside load() serialised each element's loads
// behind the previous element's conversions: ncu long-scoreboard).  The TV
// element arithmetic runs in the storage type's precision (fp32 for the
// complex64 build, fp64 for the complex128 build); reductions accumulate in
// fp64.  (fp64 differencing and shrink made these passes fp64-issue-bound:
// 1.66 G instructions, "wait" stalls, for one shrink pass.)
template <typename V> struct Sc;
template <> struct Sc<float2> { using T = float; };
template <> struct Sc<double2> { using T = double; };
template <typename V>
__device__ __forceinline__ V mk(typename Sc<V>::T x, typename Sc<V>::T y) {
    V v;
    v.x = x;
    v.y = y;
    return v;
}

template <typename V>
struct Fwd {  // centre, right (x+1), down (y+1); forward differences
    V c, r, d;
    bool hr, hd;
    __device__ __forceinline__ V gx() const { return hr ? mk<V>(r.x - c.x, r.y - c.y) : mk<V>(0, 0); }
    __device__ __forceinline__ V gy() const { return hd ? mk<V>(d.x - c.x, d.y - c.y) : mk<V>(0, 0); }
};
template <typename V>
__device__ __forceinline__ Fwd<V> load_fwd_xy(const V* v, size_t i, int x, int y, int X, int Y) {
    Fwd<V> f;
    f.hr = x < X - 1;
    f.hd = y < Y - 1;
    f.c = v[i];
    f.r = v[f.hr ? i + 1 : i];
    f.d = v[f.hd ? i + X : i];
    return f;
}
template <typename V>
__device__ __forceinline__ Fwd<V> load_fwd(const V* v, size_t i, long long m, int X, int Y) {
    int x, y;
    split_m(m, X, x, y);
    return load_fwd_xy(v, i, x, y, X, Y);
}
template <typename V>
struct Bwd {  // grad^T = -div: vx at x and x-1, vy at y and y-1
    V xc, xl, yc, yu;
    bool hxc, hxl, hyc, hyu;
    __device__ __forceinline__ V gt() const {
        typename Sc<V>::T re = 0, im = 0;
        if (hxc) { re += xc.x; im += xc.y; }
        if (hxl) { re -= xl.x; im -= xl.y; }
        if (hyc) { re += yc.x; im += yc.y; }
        if (hyu) { re -= yu.x; im -= yu.y; }
        return mk<V>(-re, -im);
    }
};
template <typename V>
__device__ __forceinline__ Bwd<V> load_bwd_xy(const V* vx, const V* vy, size_t i, int x, int y, int X, int Y) {
    Bwd<V> b;
    b.hxc = x < X - 1;
    b.hxl = x > 0;
    b.hyc = y < Y - 1;
    b.hyu = y > 0;
    b.xc = vx[i];
    b.xl = vx[b.hxl ? i - 1 : i];
    b.yc = vy[i];
    b.yu = vy[b.hyu ? i - X : i];
    return b;
}
template <typename V>
__device__ __forceinline__ Bwd<V> load_bwd(const V* vx, const V* vy, size_t i, long long m, int X, int Y) {
    int x, y;
    split_m(m, X, x, y);
    return load_bwd_xy(vx, vy, i, x, y, X, Y);
}

// ------------------------------------------------------------------ grid ops
// Two-phase element ops: load() gathers every input of element i (and its
// stencil neighbours) into registers, apply() computes, stores and
// accumulates.  k_grid issues the loads of U elements before any store, so
// the (always element-local) read-write pairs cannot serialise the loop on
// memory latency through conservative aliasing.

template <typename R>
struct OpSirtUpdate {  // u += alpha g; [nonneg]; W = deapo u; count non-finite u
    using C = typename CT<R>::T;
    C* u;
    const C* g;
    C* w;
    const R* deapo;
    const Unit* us;
    int nonneg;
    struct In { C x, g; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int b, size_t i, long long m) const {
        In v;
        v.x = u[i];
        v.g = us[b].active ? g[i] : C{};
        v.d = deapo[m];
        return v;
    }
    __device__ void apply(int b, size_t i, long long, const In& v, double (&acc)[1]) const {
        C x = v.x;
        const Unit& un = us[b];
        if (un.active) {
            x.x = (R)((double)x.x + un.alpha[0] * (double)v.g.x);
            x.y = (R)((double)x.y + un.alpha[1] * (double)v.g.y);
            if (nonneg) {
                x.x = pos_(x.x);
                x.y = pos_(x.y);
            }
            u[i] = x;
        }
        if (!finite2(x.x, x.y)) acc[0] += 1.0;
        w[i] = rc<R>(x.x * v.d, x.y * v.d);
    }
};

// OpSirtUpdate fused with the x pass of the forward FFT2 of W (complex64,
// X = 2^LOGN): 4 grid rows per CTA, lane j owns x = j + TP r.  u += alpha g
// (fp64 arithmetic as OpSirtUpdate), [nonneg], W row = FFT_x(deapo u); the
// per-unit non-finite count is an integer, accumulated with atomics (exact,
// order independent).  The y pass follows (launch_fft2_cols); together they
// replace OpSirtUpdate + the 2-D FFT and skip writing and re-reading W.
template <int LOGN>
__global__ void __launch_bounds__(4 * (1 << LOGN) / 16, 1024 / (4 * (1 << LOGN) / 16))
k_sirt_update_rowfft(float2* __restrict__ u, const float2* __restrict__ g, float2* __restrict__ w,
                     const float* __restrict__ deapo, const Unit* __restrict__ us, int nonneg, long long M, int Y,
                     const float2* __restrict__ tw, double* __restrict__ bad_count) {
    using namespace fftcore;
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3;
    extern __shared__ __align__(16) float2 sirt_fbuf[];
    const int rb = threadIdx.x / TP, j = threadIdx.x % TP;
    const long long gr = (long long)blockIdx.x * 4 + rb;  // b * Y + y
    const int b = (int)(gr / Y), y = (int)(gr - (long long)b * Y);
    const size_t base = (size_t)b * M + (size_t)y * N;
    const Unit& un = us[b];
    const bool act = un.active;
    const double a0 = un.alpha[0], a1 = un.alpha[1];
    float2 v[16];
    int bad = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int i = j + TP * r;
        float2 x = u[base + i];
        if (act) {
            const float2 gv = g[base + i];
            x.x = (float)((double)x.x + a0 * (double)gv.x);
            x.y = (float)((double)x.y + a1 * (double)gv.y);
            if (nonneg) {
                x.x = pos_(x.x);
                x.y = pos_(x.y);
            }
            u[base + i] = x;
        }
        if (!finite2(x.x, x.y)) ++bad;
        const float d = deapo[(size_t)y * N + i];
        v[r] = make_float2(x.x * d, x.y * d);
    }
    dft16<false>(v);
    fft16_stages_tab<LOGN, false>(v, sirt_fbuf + rb * N, j, tw);
#pragma unroll
    for (int q = 0; q < NB3; ++q)
#pragma unroll
        for (int r = 0; r < R3; ++r) w[base + j + TP * q + 256 * r] = v[q * R3 + r];
#pragma unroll
    for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(bad_count + b, (double)bad);
}

// Inverse-FFT2 x pass fused with OpAdjPost<float, true> (SIRT's gradient):
// W row -> IFFT_x -> g_new = deapo * scale * row; BB dots against the old g
// (<go,go>, <go, go - gn> per channel) reduced per CTA in a fixed order and
// written as part[(y0 / 4 * B + b) * 4 + k] for k_finish: deterministic.
template <int LOGN>
__global__ void __launch_bounds__(4 * (1 << LOGN) / 16, 1024 / (4 * (1 << LOGN) / 16))
k_sirt_adjpost_rowfft(const float2* __restrict__ w, float2* __restrict__ g, const float* __restrict__ deapo,
                      double scale, long long M, int Y, int B, const float2* __restrict__ tw,
                      double* __restrict__ part) {
    using namespace fftcore;
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3, NT = 4 * TP;
    extern __shared__ __align__(16) float2 sirt_fbuf[];
    __shared__ double red[4][NT / 32];
    const int rb = threadIdx.x / TP, j = threadIdx.x % TP;
    const long long gr0 = (long long)blockIdx.x * 4;
    const int b = (int)(gr0 / Y), y0 = (int)(gr0 - (long long)b * Y), y = y0 + rb;
    const size_t base = (size_t)b * M + (size_t)y * N;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = w[base + j + TP * r];
    dft16<true>(v);
    fft16_stages_tab<LOGN, true>(v, sirt_fbuf + rb * N, j, tw);
    double acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < NB3; ++q)
#pragma unroll
        for (int r = 0; r < R3; ++r) {
            const int x = j + TP * q + 256 * r;
            const double d = (double)deapo[(size_t)y * N + x] * scale;
            const float2 z = v[q * R3 + r];
            const float2 gn = make_float2((float)(z.x * d), (float)(z.y * d));
            const float2 go = g[base + x];
            acc[0] += (double)go.x * go.x;
            acc[1] += (double)go.y * go.y;
            acc[2] += (double)go.x * ((double)go.x - (double)gn.x);
            acc[3] += (double)go.y * ((double)go.y - (double)gn.y);
            g[base + x] = gn;
        }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double t = acc[k];
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
        if (lane == 0) red[k][warp] = t;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double t = 0;
        for (int i = 0; i < NT / 32; ++i) t += red[threadIdx.x][i];
        part[((size_t)(y0 / 4) * B + b) * 4 + threadIdx.x] = t;
    }
}

// A TV element pass fused with the x passes of the FFT2 around it (complex64,
// X = 2^LOGN, 4 grid rows of one unit per CTA): INV_IN: W row -> IFFT_x ->
// the op's y (the inverse y pass ran before); FWD_OUT: the op's W values ->
// FFT_x -> W row (the forward y pass follows), else the values are stored.
// Replaces IFFT_x + op + FFT_x (three passes over W) by one.  The row lives
// in the CTA's shared row buffer between the transforms, so the element
// loop holds no FFT registers: lane j takes x = j + TP k (coalesced), the
// op's loads of Op::kUnroll elements in flight together, as in k_grid (a
// first version kept the 16 transform values in registers: 128 registers,
// one element's stencil loads in flight per thread, 3.5 ms per outer
// iteration slower than the unfused passes).  The op's K sums are reduced
// per CTA in a fixed order into part[(y0 / 4 * B + b) * K + k] for k_finish
// (deterministic).
template <int LOGN, bool INV_IN, bool FWD_OUT, int K, class Op>
// (no transform: no row buffer, 32 registers, 4 CTAs of 16 warps per SM --
// the gradient norm 259 -> 232 us)
__global__ void __launch_bounds__(4 * (1 << LOGN) / 16,
                                  ((INV_IN || FWD_OUT) ? 1024 : 2048) / (4 * (1 << LOGN) / 16))
k_tv_rowfft(Op op, float2* __restrict__ w, long long M, int Y, int B, const float2* __restrict__ tw,
            double* __restrict__ part) {
    using namespace fftcore;
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3, NT = 4 * TP;
    constexpr int U = OpRowUnroll<Op>::value;
    static_assert(16 % U == 0, "unroll divides 16");
    extern __shared__ __align__(16) float2 tv_fbuf[];
    __shared__ double red[K][NT / 32];
    const int rb = threadIdx.x / TP, j = threadIdx.x % TP;
    const long long gr0 = (long long)blockIdx.x * 4;
    const int b = (int)(gr0 / Y), y0 = (int)(gr0 - (long long)b * Y), y = y0 + rb;
    const size_t base = (size_t)b * M + (size_t)y * N;
    float2* row = tv_fbuf + rb * N;
    const bool en = op.enabled(b);  // CTA-uniform
    if constexpr (INV_IN) {
        float2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = w[base + j + TP * r];
        dft16<true>(v);
        fft16_stages_tab<LOGN, true>(v, row, j, tw);
        __syncthreads();  // stage 3 read other lanes' slots
#pragma unroll
        for (int q = 0; q < NB3; ++q)
#pragma unroll
            for (int r = 0; r < R3; ++r) row[j + TP * q + 256 * r] = v[q * R3 + r];
        // lane j reads back only its own slots x = j + TP k: no barrier
    }
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0;
#pragma unroll 1
    for (int k0 = 0; k0 < 16; k0 += U) {
        typename Op::In in[U];
        if (en) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int x = j + TP * (k0 + u);
                if constexpr (INV_IN) {
                    if constexpr (OpLoadNwXY<Op>::value) in[u] = op.load_nw_xy(b, base + x, x, y);
                    else in[u] = op.load_nw(b, base + x, (long long)y * N + x);
                    in[u].y = row[x];
                } else if constexpr (OpLoadXY<Op>::value) {
                    in[u] = op.load_xy(b, base + x, x, y);
                } else {
                    in[u] = op.load(b, base + x, (long long)y * N + x);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int x = j + TP * (k0 + u);
            float2 val;
            if (en) val = op.value(b, base + x, (long long)y * N + x, in[u], acc);
            else if constexpr (INV_IN) val = row[x];
            else val = w[base + x];
            if constexpr (FWD_OUT) row[x] = val;
            else if constexpr (OpStoresW<Op>::value) w[base + x] = val;
        }
    }
    if constexpr (FWD_OUT) {
        float2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = row[j + TP * r];  // own slots
        __syncthreads();  // fft16_stages overwrites other lanes' slots
        dft16<false>(v);
        fft16_stages_tab<LOGN, false>(v, row, j, tw);
#pragma unroll
        for (int q = 0; q < NB3; ++q)
#pragma unroll
            for (int r = 0; r < R3; ++r) w[base + j + TP * q + 256 * r] = v[q * R3 + r];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double t = acc[k];
#pragma unroll
        for (int s = 16; s; s >>= 1) t += __shfl_down_sync(0xffffffffu, t, s);
        if (lane == 0) red[k][warp] = t;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double t = 0;
        for (int u = 0; u < NT / 32; ++u) t += red[threadIdx.x][u];
        part[((size_t)(y0 / 4) * B + b) * K + threadIdx.x] = t;
    }
}

template <typename R, typename V>
struct OpDeapo {  // w = deapo * v * scale  (v of any precision, w of plan precision)
    using C = typename CT<R>::T;
    const V* v;
    C* w;
    const R* deapo;
    double scale;
    struct In { V x; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const { return In{v[i], deapo[m]}; }
    __device__ void apply(int, size_t i, long long, const In& q, double (&)[1]) const {
        const double d = (double)q.d * scale;
        w[i] = rc<R>(q.x.x * d, q.x.y * d);
    }
};

template <typename R, typename V>
struct OpStore {  // out = deapo * y * scale  (V precision)
    using C = typename CT<R>::T;
    const C* y;
    V* out;
    const R* deapo;
    double scale;
    struct In { C y; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const { return In{y[i], deapo[m]}; }
    __device__ void apply(int, size_t i, long long, const In& q, double (&)[1]) const {
        const double d = (double)q.d * scale;
        V o;
        o.x = q.y.x * d;
        o.y = q.y.y * d;
        out[i] = o;
    }
};

// g = deapo*y*scale (adjoint post-IFFT2); acc <g,g> per channel; with BB the
// dots vs the previous g: <du,du> = a^2 <g,g>, <du, g - g_new> = a <g, g - g_new>
template <typename R, bool BB>
struct OpAdjPost {
    using C = typename CT<R>::T;
    const C* y;
    C* g;
    const R* deapo;
    double scale;
    struct In { C y, go; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const {
        In v;
        v.y = y[i];
        v.go = BB ? g[i] : C{};
        v.d = deapo[m];
        return v;
    }
    __device__ void apply(int, size_t i, long long, const In& v, double (&acc)[BB ? 4 : 2]) const {
        const double d = (double)v.d * scale;
        const C gn = rc<R>(v.y.x * d, v.y.y * d);
        if (BB) {
            acc[0] += (double)v.go.x * v.go.x;
            acc[1] += (double)v.go.y * v.go.y;
            acc[2] += (double)v.go.x * ((double)v.go.x - (double)gn.x);
            acc[3] += (double)v.go.y * ((double)v.go.y - (double)gn.y);
        } else {
            acc[0] += (double)gn.x * gn.x;
            acc[1] += (double)gn.y * gn.y;
        }
        g[i] = gn;
    }
};

template <typename V>
struct OpNonfinite {
    const V* u;
    struct In { V x; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long) const { return In{u[i]}; }
    __device__ void apply(int, size_t, long long, const In& v, double (&acc)[1]) const {
        if (!finite2(v.x.x, v.x.y)) acc[0] += 1.0;
    }
};

template <typename V>
struct OpNonneg {
    V* u;
    const Unit* us;
    struct In { V x; };
    __device__ bool enabled(int b) const { return us[b].status != ST_PAD; }
    __device__ In load(int, size_t i, long long) const { return In{u[i]}; }
    __device__ void apply(int, size_t i, long long, const In& v, double (&)[1]) const {
        V x = v.x;
        x.x = pos_(x.x);
        x.y = pos_(x.y);
        u[i] = x;
    }
};

// The last inner CGLS step of a TV outer iteration (solvers.py:450-459): only
// u += alpha p survives it -- s = adj(r), gamma, beta and p are never read
// again (u is returned, the next outer restarts from r = b - fwd(u)), so
// that step is this one pass (+ the nonneg projection of solvers.py:414),
// with the arithmetic of OpTvStepS's u update.
template <typename V>
struct OpTvAxpy {
    V* u;
    const V* p;
    const Unit* us;
    int nonneg;
    struct In { V x, pp; };
    __device__ bool enabled(int b) const { return us[b].status != ST_PAD; }
    __device__ In load(int, size_t i, long long) const { return In{u[i], p[i]}; }
    __device__ void apply(int b, size_t i, long long, const In& v, double (&)[1]) const {
        using T = typename Sc<V>::T;
        const Unit& un = us[b];
        V x = v.x;
        if (un.stepped) x = mk<V>(x.x + (T)un.alpha[0] * v.pp.x, x.y + (T)un.alpha[1] * v.pp.y);
        if (nonneg) {
            x.x = pos_(x.x);
            x.y = pos_(x.y);
        }
        if (un.stepped || nonneg) u[i] = x;
    }
};

template <typename R>
struct OpAbsMax {  // per-channel max |deapo*y*scale| (TV default mu, solvers.py:364-372)
    using C = typename CT<R>::T;
    const C* y;
    const R* deapo;
    double scale;
    struct In { C y; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const { return In{y[i], deapo[m]}; }
    __device__ void apply(int, size_t, long long, const In& v, double (&acc)[2]) const {
        const double d = (double)v.d * scale;
        acc[0] = fmax(acc[0], fabs((double)(R)(v.y.x * d)));
        acc[1] = fmax(acc[1], fabs((double)(R)(v.y.y * d)));
    }
};

// ------------------------------------------------------------------ grid ops (CGLS, fp64 vectors)

template <typename R, typename V = D2>
struct OpCglsInit {  // p = s = deapo*y*scale ; <s,s> ; W = deapo p
    using C = typename CT<R>::T;
    C* w;
    V* p;
    const R* deapo;
    double scale;
    struct In { C y; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load_nw(int, size_t, long long m) const {
        In v;
        v.d = deapo[m];
        return v;
    }
    __device__ In load(int, size_t i, long long m) const { return In{w[i], deapo[m]}; }
    __device__ C value(int, size_t i, long long, const In& v, double (&acc)[2]) const {
        const double d = (double)v.d;
        const D2 s = make_double2(v.y.x * d * scale, v.y.y * d * scale);
        acc[0] += s.x * s.x;
        acc[1] += s.y * s.y;
        p[i] = tv_store<V>(s.x, s.y);
        return rc<R>(s.x * d, s.y * d);
    }
    __device__ void apply(int b, size_t i, long long m, const In& v, double (&acc)[2]) const {
        w[i] = value(b, i, m, v, acc);
    }
};

template <typename R>
struct OpDotS {  // <s,s>, s = deapo*y*scale
    using C = typename CT<R>::T;
    const C* y;
    const R* deapo;
    double scale;
    struct In { C y; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load_nw(int, size_t, long long m) const {
        In v;
        v.d = deapo[m];
        return v;
    }
    __device__ In load(int, size_t i, long long m) const { return In{y[i], deapo[m]}; }
    // fused after the inverse x pass: the row y is stored unchanged
    __device__ C value(int, size_t, long long, const In& v, double (&acc)[2]) const {
        const double d = (double)v.d * scale;
        const double sx = v.y.x * d, sy = v.y.y * d;
        acc[0] += sx * sx;
        acc[1] += sy * sy;
        return v.y;
    }
    __device__ void apply(int b, size_t i, long long m, const In& v, double (&acc)[2]) const {
        (void)value(b, i, m, v, acc);
    }
};

template <typename R, typename V = D2>
struct OpCglsTail {  // u += alpha p ; p = s + beta p ; W = deapo p_new ; non-finite u
    using C = typename CT<R>::T;
    V* u;
    V* p;
    C* w;  // in: y (IFFT2 output), out: deapo * p
    const R* deapo;
    double scale;
    const Unit* us;
    struct In { V x, pp; C y; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const { return In{u[i], p[i], w[i], deapo[m]}; }
    __device__ void apply(int b, size_t i, long long m, const In& v, double (&acc)[1]) const {
        w[i] = value(b, i, m, v, acc);
    }
    __device__ C value(int b, size_t i, long long, const In& v, double (&acc)[1]) const {
        const Unit& un = us[b];
        D2 x = d2(v.x);
        D2 pp = d2(v.pp);
        const double d = (double)v.d;
        if (un.stepped) {
            x.x += un.alpha[0] * pp.x;
            x.y += un.alpha[1] * pp.y;
            u[i] = tv_store<V>(x.x, x.y);
            if (un.active) {
                pp.x = v.y.x * d * scale + un.beta[0] * pp.x;
                pp.y = v.y.y * d * scale + un.beta[1] * pp.y;
                p[i] = tv_store<V>(pp.x, pp.y);
            }
        }
        if (!finite2(x.x, x.y)) acc[0] += 1.0;
        return rc<R>(pp.x * d, pp.y * d);
    }
};

// ------------------------------------------------------------------ grid ops (CGS, fp64 vectors)
// Conjugate gradient squared on A^H W A u = A^H W b (solvers.py:262-305):
// r, shadow, p, q, h, v are grid vectors; "step" = q + h is never stored.

template <typename R>
struct OpCgsInit {  // c = deapo*y*scale ; r = shadow = p = q = c ; rho = <c,c> ; W = deapo p
    using C = typename CT<R>::T;
    C* w;
    D2 *r, *sh, *p, *q;
    const R* deapo;
    double scale;
    struct In { C y; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const { return In{w[i], deapo[m]}; }
    __device__ void apply(int, size_t i, long long, const In& v, double (&acc)[2]) const {
        const double d = (double)v.d;
        const D2 c = make_double2(v.y.x * d * scale, v.y.y * d * scale);
        acc[0] += c.x * c.x;
        acc[1] += c.y * c.y;
        r[i] = c;
        sh[i] = c;
        p[i] = c;
        q[i] = c;
        w[i] = rc<R>(c.x * d, c.y * d);
    }
};

template <typename R>
struct OpCgsV {  // v = deapo*y*scale (= M p) ; sigma = <shadow, v>
    using C = typename CT<R>::T;
    const C* w;
    const D2* sh;
    D2* v;
    const R* deapo;
    double scale;
    struct In { C y; D2 s; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const { return In{w[i], sh[i], deapo[m]}; }
    __device__ void apply(int, size_t i, long long, const In& x, double (&acc)[2]) const {
        const double d = (double)x.d * scale;
        const D2 vv = make_double2(x.y.x * d, x.y.y * d);
        acc[0] += x.s.x * vv.x;
        acc[1] += x.s.y * vv.y;
        v[i] = vv;
    }
};

template <typename R>
struct OpCgsStep {  // h = q - alpha v ; u += alpha (q + h) ; W = deapo (q + h) ; non-finite u
    using C = typename CT<R>::T;
    D2 *u, *h;
    const D2 *q, *v;
    C* w;
    const R* deapo;
    const Unit* us;
    struct In { D2 x, qq, vv; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const { return In{u[i], q[i], v[i], deapo[m]}; }
    __device__ void apply(int b, size_t i, long long, const In& e, double (&acc)[1]) const {
        const Unit& un = us[b];
        const double d = (double)e.d;
        D2 x = e.x, st = make_double2(0, 0);
        if (un.stepped) {
            const D2 hh = make_double2(e.qq.x - un.alpha[0] * e.vv.x, e.qq.y - un.alpha[1] * e.vv.y);
            st = make_double2(e.qq.x + hh.x, e.qq.y + hh.y);
            x.x += un.alpha[0] * st.x;
            x.y += un.alpha[1] * st.y;
            h[i] = hh;
            u[i] = x;
        }
        if (!finite2(x.x, x.y)) acc[0] += 1.0;
        w[i] = rc<R>(st.x * d, st.y * d);
    }
};

template <typename R>
struct OpCgsResid {  // r -= alpha deapo*y*scale (= M step) ; rho_new = <shadow, r> ; W = deapo u
    using C = typename CT<R>::T;
    C* w;
    D2* r;
    const D2 *sh, *u;
    const R* deapo;
    double scale;
    const Unit* us;
    struct In { C y; D2 rr, s, x; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const { return In{w[i], r[i], sh[i], u[i], deapo[m]}; }
    __device__ void apply(int b, size_t i, long long, const In& e, double (&acc)[2]) const {
        const Unit& un = us[b];
        const double d = (double)e.d;
        D2 rr = e.rr;
        if (un.stepped) {
            rr.x -= un.alpha[0] * (e.y.x * d * scale);
            rr.y -= un.alpha[1] * (e.y.y * d * scale);
            r[i] = rr;
        }
        acc[0] += e.s.x * rr.x;
        acc[1] += e.s.y * rr.y;
        w[i] = rc<R>(e.x.x * d, e.x.y * d);
    }
};

template <typename R>
struct OpCgsDir {  // q = r + beta h ; p = q + beta (h + beta p) ; W = deapo p
    using C = typename CT<R>::T;
    const D2 *r, *h;
    D2 *q, *p;
    C* w;
    const R* deapo;
    const Unit* us;
    struct In { D2 rr, hh, pp; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const { return In{r[i], h[i], p[i], deapo[m]}; }
    __device__ void apply(int b, size_t i, long long, const In& e, double (&)[1]) const {
        const Unit& un = us[b];
        D2 pp = e.pp;
        if (un.active) {
            const double b0 = un.beta[0], b1 = un.beta[1];
            const D2 qq = make_double2(e.rr.x + b0 * e.hh.x, e.rr.y + b1 * e.hh.y);
            pp = make_double2(qq.x + b0 * (e.hh.x + b0 * pp.x), qq.y + b1 * (e.hh.y + b1 * pp.y));
            q[i] = qq;
            p[i] = pp;
        }
        const double d = (double)e.d;
        w[i] = rc<R>(pp.x * d, pp.y * d);
    }
};

// ------------------------------------------------------------------ grid ops (TV)

// s = mu (deapo y scale) + lam grad^T(rho)   (adj(), solvers.py:397-399)
// MODE 0: p = s, W = deapo p, acc <s,s>;  1: acc <s,s>, W = s (in place);
// 2: W holds s (MODE 1's): p = s + beta p, W = deapo p
template <typename R, int MODE, typename V>
struct OpTvS {
    static constexpr int kUnroll = MODE == 2 ? 4 : TV_UNROLL;  // MODE 2: 3 loads per element
    using C = typename CT<R>::T;
    C* w;
    V* p;
    const V *rx, *ry;
    const R* deapo;
    double scale;
    const Unit* us;
    int X, Y;
    struct In { C y; Bwd<V> g; V pp; R d; };
    __device__ bool enabled(int b) const { return MODE == 1 || us[b].active; }
    // every input but y (the fused x passes supply y from registers)
    __device__ In load_nw(int, size_t i, long long m) const {
        In v;
        if (MODE != 2) v.g = load_bwd(rx, ry, i, m, X, Y);
        if (MODE == 2) v.pp = p[i];
        v.d = deapo[m];
        return v;
    }
    __device__ In load_nw_xy(int, size_t i, int x, int y) const {
        In v;
        if (MODE != 2) v.g = load_bwd_xy(rx, ry, i, x, y, X, Y);
        if (MODE == 2) v.pp = p[i];
        v.d = deapo[(size_t)y * X + x];
        return v;
    }
    __device__ In load(int b, size_t i, long long m) const {
        In v = load_nw(b, i, m);
        v.y = w[i];
        return v;
    }
    // the new W element (stored by apply(), or fed to a fused forward x pass)
    __device__ C value(int b, size_t i, long long, const In& v, double (&acc)[2]) const {
        using T = typename Sc<V>::T;
        const Unit& un = us[b];
        const T d = (T)v.d;
        if (MODE == 2) {
            V pp = v.pp;
            if (!un.inner_stop) {
                pp.x = (T)v.y.x + (T)un.beta[0] * pp.x;
                pp.y = (T)v.y.y + (T)un.beta[1] * pp.y;
                p[i] = pp;
            }
            return rc<R>(pp.x * d, pp.y * d);
        }
        const T ds = (T)(v.d * scale);
        const V gt = v.g.gt();
        const V s = mk<V>((T)un.mu[0] * ((T)v.y.x * ds) + (T)un.lam[0] * gt.x,
                          (T)un.mu[1] * ((T)v.y.y * ds) + (T)un.lam[1] * gt.y);
        acc[0] += (double)s.x * (double)s.x;
        acc[1] += (double)s.y * (double)s.y;
        if (MODE == 0) {
            p[i] = s;
            return rc<R>(s.x * d, s.y * d);
        }
        return rc<R>(s.x, s.y);
    }
    __device__ void apply(int b, size_t i, long long m, const In& v, double (&acc)[2]) const {
        w[i] = value(b, i, m, v, acc);
    }
};

template <typename V>
struct OpTvGradNorm {  // ||grad p||^2 per channel
    static constexpr bool kNoW = true;
    const V* p;
    const Unit* us;
    int X, Y;
    struct In { Fwd<V> f; };
    __device__ bool enabled(int b) const { return us[b].active; }
    __device__ In load(int, size_t i, long long m) const { return In{load_fwd(p, i, m, X, Y)}; }
    __device__ In load_xy(int, size_t i, int x, int y) const { return In{load_fwd_xy(p, i, x, y, X, Y)}; }
    __device__ void apply(int, size_t, long long, const In& v, double (&acc)[2]) const {
        const V gx = v.f.gx(), gy = v.f.gy();
        acc[0] += (double)(gx.x * gx.x + gy.x * gy.x);
        acc[1] += (double)(gx.y * gx.y + gy.y * gy.y);
    }
    __device__ float2 value(int b, size_t i, long long m, const In& v, double (&acc)[2]) const {
        apply(b, i, m, v, acc);
        return make_float2(0.f, 0.f);
    }
};

// The CGLS step fused into the beta pass (solvers.py:401-413): u += alpha p,
// rho_new = rho - alpha grad p, and s = mu (deapo y scale) + lam grad^T(rho_new)
// with <s,s> -- rho_new at x-1 and y-1 is recomputed from the old rho and p
// (a 5-point stencil of p), so rho is read from one buffer and written to
// the other (neighbours still read the old values).  W (y) becomes s.
template <typename R, typename V>
struct OpTvStepS {
    static constexpr int kUnroll = TV_UNROLL;
    using C = typename CT<R>::T;
    C* w;
    V* u;
    const V *p, *rx, *ry;  // rho (old)
    V *nx, *ny;            // rho (new)
    const R* deapo;
    double scale;
    const Unit* us;
    int X, Y;
    struct In { C y; V pc, pr, pd, pl, pu, xc, xl, yc, yu, uu; R d; bool hr, hd, hl, hu; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int b, size_t i, long long m) const {
        In v = load_nw(b, i, m);
        v.y = w[i];
        return v;
    }
    __device__ In load_nw(int b, size_t i, long long m) const {
        int x, y;
        split_m(m, X, x, y);
        return load_nw_xy(b, i, x, y);
    }
    __device__ In load_nw_xy(int, size_t i, int x, int y) const {
        const long long m = (long long)y * X + x;
        In v;
        v.hr = x < X - 1;
        v.hd = y < Y - 1;
        v.hl = x > 0;
        v.hu = y > 0;
        v.pc = p[i];
        v.pr = p[v.hr ? i + 1 : i];
        v.pd = p[v.hd ? i + X : i];
        v.pl = p[v.hl ? i - 1 : i];
        v.pu = p[v.hu ? i - X : i];
        v.xc = rx[i];
        v.xl = rx[v.hl ? i - 1 : i];
        v.yc = ry[i];
        v.yu = ry[v.hu ? i - X : i];
        v.uu = u[i];
        v.d = deapo[m];
        return v;
    }
    __device__ void apply(int b, size_t i, long long m, const In& v, double (&acc)[2]) const {
        w[i] = value(b, i, m, v, acc);
    }
    __device__ C value(int b, size_t i, long long, const In& v, double (&acc)[2]) const {
        using T = typename Sc<V>::T;
        const Unit& un = us[b];
        const bool st = un.stepped;
        const T a0 = st ? (T)un.alpha[0] : (T)0, a1 = st ? (T)un.alpha[1] : (T)0;
        // grad p at i, and the x / y differences ending at i (grad at x-1 / y-1)
        const V gx = v.hr ? mk<V>(v.pr.x - v.pc.x, v.pr.y - v.pc.y) : mk<V>(0, 0);
        const V gy = v.hd ? mk<V>(v.pd.x - v.pc.x, v.pd.y - v.pc.y) : mk<V>(0, 0);
        const V gxl = mk<V>(v.pc.x - v.pl.x, v.pc.y - v.pl.y);
        const V gyu = mk<V>(v.pc.x - v.pu.x, v.pc.y - v.pu.y);
        const V xc = mk<V>(v.xc.x - a0 * gx.x, v.xc.y - a1 * gx.y);
        const V yc = mk<V>(v.yc.x - a0 * gy.x, v.yc.y - a1 * gy.y);
        const V xl = mk<V>(v.xl.x - a0 * gxl.x, v.xl.y - a1 * gxl.y);
        const V yu = mk<V>(v.yu.x - a0 * gyu.x, v.yu.y - a1 * gyu.y);
        if (st) u[i] = mk<V>(v.uu.x + a0 * v.pc.x, v.uu.y + a1 * v.pc.y);
        nx[i] = xc;
        ny[i] = yc;
        T re = 0, im = 0;  // -grad^T(rho_new)
        if (v.hr) { re += xc.x; im += xc.y; }
        if (v.hl) { re -= xl.x; im -= xl.y; }
        if (v.hd) { re += yc.x; im += yc.y; }
        if (v.hu) { re -= yu.x; im -= yu.y; }
        const T ds = (T)(v.d * scale);
        const V s = mk<V>((T)un.mu[0] * ((T)v.y.x * ds) - (T)un.lam[0] * re,
                          (T)un.mu[1] * ((T)v.y.y * ds) - (T)un.lam[1] * im);
        acc[0] += (double)s.x * (double)s.x;
        acc[1] += (double)s.y * (double)s.y;
        return rc<R>(s.x, s.y);
    }
};

// isotropic shrink + Bregman update (solvers.py:418-421, 330-341); W = deapo u.
// Fused with the next outer iteration's stacked target (solvers.py:410-411):
// d is used only there, so the pass writes rho = (d - b) - grad u (u is the
// same) instead of d -- one fp64 grid pass less per outer iteration, and no d.
template <typename R, typename V>
struct OpTvShrink {
    static constexpr int kUnroll = TV_UNROLL;
    // in the fused x pass 4 elements' loads in flight (1.82 -> 1.71 ms, 56 registers)
    static constexpr int kRowUnroll = 4;
    using C = typename CT<R>::T;
    const V* u;
    V *rx, *ry, *bx, *by;
    C* w;
    const R* deapo;
    const Unit* us;
    int X, Y;
    struct In { Fwd<V> f; V bx, by; R d; };
    __device__ bool enabled(int) const { return true; }
    __device__ In load(int, size_t i, long long m) const {
        return In{load_fwd(u, i, m, X, Y), bx[i], by[i], deapo[m]};
    }
    __device__ In load_xy(int, size_t i, int x, int y) const {
        return In{load_fwd_xy(u, i, x, y, X, Y), bx[i], by[i], deapo[(size_t)y * X + x]};
    }
    __device__ void apply(int b, size_t i, long long m, const In& in, double (&acc)[1]) const {
        w[i] = value(b, i, m, in, acc);
    }
    __device__ C value(int b, size_t i, long long, const In& in, double (&acc)[1]) const {
        using T = typename Sc<V>::T;
        const Unit& un = us[b];
        const V x = in.f.c, gx = in.f.gx(), gy = in.f.gy();
        if (!(isfinite(x.x) && isfinite(x.y))) acc[0] += 1.0;
        const T d = (T)in.d;
        const C wv = rc<R>(x.x * d, x.y * d);
        if (!un.active) return wv;
        const T vx[2] = {gx.x + in.bx.x, gx.y + in.bx.y};
        const T vy[2] = {gy.x + in.by.x, gy.y + in.by.y};
        T ox[2], oy[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const T kap = (T)un.kap[c];  // 1 / lam (k_tv_mu)
            const T mag = sqrt(vx[c] * vx[c] + vy[c] * vy[c]);
            const T f = (mag - kap > (T)0 ? mag - kap : (T)0) / (mag > (T)0 ? mag : (T)1);
            ox[c] = vx[c] * f;
            oy[c] = vy[c] * f;
        }
        const V nbx = mk<V>(in.bx.x + gx.x - ox[0], in.bx.y + gx.y - ox[1]);
        const V nby = mk<V>(in.by.x + gy.x - oy[0], in.by.y + gy.y - oy[1]);
        bx[i] = nbx;
        by[i] = nby;
        rx[i] = mk<V>(ox[0] - nbx.x - gx.x, ox[1] - nbx.y - gx.y);
        ry[i] = mk<V>(oy[0] - nby.x - gy.x, oy[1] - nby.y - gy.y);
        return wv;
    }
};

// ------------------------------------------------------------------ spectral kernels
// Pairs (t, jh) with its mirror (t, (P-jh) mod P), all b.  UPDATE: Rhat -=
// chan_scale(alpha, Qhat) through the mirror mix (stepped units only); then the
// A, C partial sums of the (updated) Rhat.  RV = storage of Rhat; rf = optional
// plan-precision copy of Rhat for the next SpMM.
constexpr int SPEC_Q = 4;  // work items per detector row in k_spec
#ifndef SPEC_U_
#define SPEC_U_ 1
#endif
constexpr int SPEC_U = SPEC_U_;  // bins per thread in flight

template <typename R, typename RV, bool UPDATE>
__global__ void __launch_bounds__(RT)
k_spec(RV* __restrict__ rh, const typename CT<R>::T* __restrict__ qh,
       typename CT<R>::T* __restrict__ rf, const int* __restrict__ perm,
       const R* __restrict__ w, long long wlen, int T, int P,
       int B, const Unit* __restrict__ us, double* __restrict__ part) {
    const int H = P / 2 + 1;
    double a = 0, c = 0;
    const int lgB = __ffs(B) - 1;  // B is a power of two dividing RT
    const int b = threadIdx.x & (B - 1);
    const bool step = UPDATE ? (us[b].stepped != 0) : false;
    double ap = 0, am = 0;
    if (UPDATE) {
        ap = 0.5 * (us[b].alpha[0] + us[b].alpha[1]);
        am = 0.5 * (us[b].alpha[0] - us[b].alpha[1]);
    }
    // work item = (detector row t, quarter q of its bins jh): 4T items for a
    // grid of 4T blocks (whole rows per block left a 1.3-wave tail: T = 1536
    // rows on 1184 blocks); a thread keeps its unit b and steps jh by RT / B
    // (the flat (jh, b) index with a runtime divide by B cost ~100
    // instructions per pair: ncu 68% SM throughput at 47% of HBM)
    for (int item = blockIdx.x; item < T * SPEC_Q; item += gridDim.x) {
    const int t = item / SPEC_Q, q = item - t * SPEC_Q;
    const int j_end = H * (q + 1) / SPEC_Q;
    const int* prow = perm + (size_t)t * P;
    // SPEC_U bins per round, all index loads, then all spectrum (and Q) loads,
    // then the arithmetic (per-thread accumulation order unchanged).  Measured
    // (ncu, CGLS at c2, B = 32): norms 181 us with the loads interleaved in the
    // arithmetic, 168 at SPEC_U = 1, 161 at 4; the update pass 435 / 413 / 456
    // us -- 1 is the default
    const int stp = RT >> lgB;
    for (int jh0 = H * q / SPEC_Q + (threadIdx.x >> lgB); jh0 < j_end; jh0 += SPEC_U * stp) {
        size_t s1[SPEC_U], s2[SPEC_U];
        RV r1v[SPEC_U], r2v[SPEC_U];
        typename CT<R>::T q1v[SPEC_U], q2v[SPEC_U];
#pragma unroll
        for (int u = 0; u < SPEC_U; ++u) {
            const int jh = jh0 + u * stp;
            const int j2 = jh ? P - jh : 0;  // jh < H: j2 >= jh, each pair once
            s1[u] = (size_t)prow[jh < j_end ? jh : 0];
            s2[u] = (size_t)prow[jh < j_end ? j2 : 0];
        }
#pragma unroll
        for (int u = 0; u < SPEC_U; ++u) {
            r1v[u] = rh[s1[u] * B + b];
            r2v[u] = rh[s2[u] * B + b];
            if (UPDATE && step) {
                q1v[u] = qh[s1[u] * B + b];
                q2v[u] = qh[s2[u] * B + b];
            }
        }
#pragma unroll
        for (int u = 0; u < SPEC_U; ++u) {
        const int jh = jh0 + u * stp;
        if (jh >= j_end) break;
        const int j1 = jh, j2 = jh ? P - jh : 0;
        const double wt = w ? (double)(wlen == P ? w[j1] : w[(size_t)t * P + j1]) : 1.0;
        D2 r1 = d2(r1v[u]);
        D2 r2 = d2(r2v[u]);
        if (UPDATE && step) {
            const D2 q1 = d2(q1v[u]), q2 = d2(q2v[u]);
            const D2 n1 = make_double2(r1.x - (ap * q1.x + am * q2.x), r1.y - (ap * q1.y - am * q2.y));
            const D2 n2 = make_double2(r2.x - (ap * q2.x + am * q1.x), r2.y - (ap * q2.y - am * q1.y));
            r1 = n1;
            r2 = n2;
            RV o1, o2;
            o1.x = r1.x; o1.y = r1.y;
            o2.x = r2.x; o2.y = r2.y;
            rh[s1[u] * B + b] = o1;
            if (j2 != j1) rh[s2[u] * B + b] = o2;
        }
        if (rf) {
            rf[s1[u] * B + b] = rc<R>(r1.x, r1.y);
            if (j2 != j1) rf[s2[u] * B + b] = rc<R>(r2.x, r2.y);
        }
        if (j1 == j2) {
            a += wt * (r1.x * r1.x + r1.y * r1.y);
            c += wt * (r1.x * r1.x - r1.y * r1.y);
        } else {
            a += wt * (r1.x * r1.x + r1.y * r1.y + r2.x * r2.x + r2.y * r2.y);
            c += 2.0 * wt * (r1.x * r2.x - r1.y * r2.y);
        }
        }
    }
    }
    // reduce threads sharing b (tid = b + B*k), fixed order
    __shared__ double sa[RT], sc[RT];
    sa[threadIdx.x] = a;
    sc[threadIdx.x] = c;
    __syncthreads();
    if (threadIdx.x < B) {
        double ta = 0, tc = 0;
        for (int k = threadIdx.x; k < RT; k += B) {
            ta += sa[k];
            tc += sc[k];
        }
        double* o = part + ((size_t)blockIdx.x * B + threadIdx.x) * 2;
        o[0] = ta;
        o[1] = tc;
    }
}

// ------------------------------------------------------------------ scalar kernels
// A, C -> per-channel squared weighted norms
// (clamps rounding negatives to 0 but lets NaN through, like the reference's sums)
__device__ __forceinline__ double clamp0(double v) { return v < 0.0 ? 0.0 : v; }
__device__ __forceinline__ void chan_norm2(const double* ac, int P, const Unit& un, double* n2) {
    n2[0] = clamp0((ac[0] + ac[1]) / (2.0 * P));
    n2[1] = un.single ? 0.0 : clamp0((ac[0] - ac[1]) / (2.0 * P));
}

__global__ void k_init_units(Unit* us, int nb, int B, int single_last, Global* gl) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit u;
    memset(&u, 0, sizeof(Unit));
    u.min_res = INFINITY;
    u.status = b < nb ? RUNNING : ST_PAD;
    u.active = b < nb;
    u.single = (single_last && b == nb - 1) ? 1 : 0;
    us[b] = u;
    if (b == 0) gl->n_active = 0;
}

// b_norm per channel; zero right-hand side -> converged, 0 iterations
__global__ void k_bnorm(Unit* us, const double* ac, int P, int B) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    if (un.status == ST_PAD) return;
    double n2[2];
    chan_norm2(ac + 2 * b, P, un, n2);
    un.bnorm[0] = sqrt(n2[0]);
    un.bnorm[1] = sqrt(n2[1]);
    if (sqrt(n2[0] + n2[1]) == 0.0) {
        un.status = ST_ZERO;
        un.active = 0;
        un.converged = 1;
    }
}

// residual bookkeeping shared by FBP / SIRT / CGLS / TV
// (solvers.py:127-129, 164-176, 214-221, 422-428)
__device__ void record_residual(Unit& un, const double* ac, int P, int it, int B, int b,
                                double* hist, bool nonfinite, bool divergence, double tol,
                                bool tol_only_positive) {
    double n2[2];
    chan_norm2(ac, P, un, n2);
    const double r0 = sqrt(n2[0]), r1 = sqrt(n2[1]);
    const double res = sqrt(n2[0] + n2[1]);
    // the unit's own count: an active unit has run every iteration so far, and
    // the kernel's arguments stay the same from iteration to iteration (the
    // iteration bodies are replayed as CUDA graphs)
    (void)it;
    hist[(size_t)un.iters * B + b] = res;
    un.iters += 1;
    if (nonfinite) {
        un.status = ST_NONFINITE;
        un.active = 0;
        un.converged = 0;
        return;
    }
    if (divergence) {
        if (res < un.min_res) un.min_res = res;  // python min(): NaN never wins
        if (res > 10.0 * un.min_res) {
            un.status = ST_DIVERGED;
            un.active = 0;
            return;
        }
    }
    const double rel = fmax(safe_div(r0, un.bnorm[0], 0.0), safe_div(r1, un.bnorm[1], 0.0));
    if ((!tol_only_positive || tol > 0) && rel <= tol) {
        un.status = ST_CONVERGED;
        un.converged = 1;
        un.active = 0;
    }
}

__global__ void k_count_active(const Unit* us, int B, Global* gl) {
    __shared__ int n;
    if (threadIdx.x == 0) n = 0;
    __syncthreads();
    if (threadIdx.x < B && us[threadIdx.x].active) atomicAdd(&n, 1);
    __syncthreads();
    if (threadIdx.x == 0) gl->n_active = n;
}

__global__ void k_fbp_check(Unit* us, const double* ac, const double* nf, int P, int B,
                            double* hist) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    if (un.status == ST_PAD) return;
    record_residual(un, ac + 2 * b, P, 0, B, b, hist, nf[b] > 0, false, -1.0, false);
    if (un.status != ST_NONFINITE) {
        un.status = ST_CONVERGED;
        un.converged = 1;
    }
}

// SIRT: alpha0 = <g,g> / ||A g||_w^2  (solvers.py:152-156)
__global__ void k_sirt_alpha0(Unit* us, const double* gg, const double* ac, int P, int B) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    double n2[2];
    chan_norm2(ac + 2 * b, P, un, n2);
    for (int c = 0; c < 2; ++c) {
        const double a0 = (un.single && c == 1) ? 0.0 : safe_div(gg[2 * b + c], n2[c], 0.0);
        un.alpha0[c] = a0;
        un.alpha[c] = un.active ? a0 : 0.0;
    }
}

__global__ void k_sirt_check(Unit* us, const double* ac, const double* nf, int P, int it, int B,
                             double* hist, double tol) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    if (!un.active) return;
    record_residual(un, ac + 2 * b, P, it, B, b, hist, nf[b] > 0, true, tol, false);
}

// BB1 step with safeguarded fallback (solvers.py:177-184)
__global__ void k_sirt_alpha(Unit* us, const double* dots, int B, int bb) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    for (int c = 0; c < 2; ++c) {
        double a = un.alpha0[c];
        if (bb && !(un.single && c == 1)) {
            const double al = un.alpha[c];
            const double dd = al * al * dots[4 * b + c];
            const double ddg = al * dots[4 * b + 2 + c];
            a = safe_div(dd, ddg, un.alpha0[c]);
            if (!(a > 0)) a = un.alpha0[c];
        }
        if (un.single && c == 1) a = 0.0;
        un.alpha[c] = un.active ? a : 0.0;
    }
}

// CGLS (solvers.py:197-226)
__global__ void k_cgls_init(Unit* us, const double* ss, int B) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    for (int c = 0; c < 2; ++c) {
        un.gamma[c] = ss[2 * b + c];
        un.gamma0[c] = un.gamma[c];
    }
}

// delta = ||q||^2 per channel.  tv != 0: stacked TV delta = mu ||A p||_w^2 +
// lam ||grad p||^2 (solvers.py:401-403,444-451), non-finite guard, no gamma floor.
__global__ void k_cgls_alpha(Unit* us, const double* ac, const double* gnorm, int P, int B, int tv) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    un.stepped = 0;
    const bool live = tv ? (un.active && !un.inner_stop) : un.active;
    un.alpha[0] = un.alpha[1] = 0.0;
    if (!live) return;
    double dl[2];
    chan_norm2(ac + 2 * b, P, un, dl);
    if (tv)
        for (int c = 0; c < 2; ++c)
            dl[c] = (un.single && c == 1) ? 0.0 : un.mu[c] * dl[c] + un.lam[c] * gnorm[2 * b + c];
    if (tv && !(isfinite(dl[0]) && isfinite(dl[1]) && isfinite(un.gamma[0]) &&
                isfinite(un.gamma[1]))) {
        un.status = ST_NONFINITE;
        un.active = 0;
        return;
    }
    const double eps2 = 2.220446049250313e-16 * 2.220446049250313e-16;
    bool any = false;
    for (int c = 0; c < 2; ++c) {
        bool a = dl[c] > 0;
        if (!tv) a = a && (un.gamma[c] > eps2 * un.gamma0[c]);
        if (un.single && c == 1) a = false;
        un.act[c] = a;
        any = any || a;
    }
    if (!any) {
        if (tv) {
            un.inner_stop = 1;
        } else {
            un.status = ST_STOPPED;  // breakdown / stagnation: flagged, not thrown
            un.active = 0;
        }
        return;
    }
    for (int c = 0; c < 2; ++c) un.alpha[c] = un.act[c] ? safe_div(un.gamma[c], dl[c], 0.0) : 0.0;
    un.stepped = 1;
}

__global__ void k_cgls_check(Unit* us, const double* ac, int P, int it, int B, double* hist,
                             double tol) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    if (!un.stepped) return;
    record_residual(un, ac + 2 * b, P, it, B, b, hist, false, false, tol, false);
}

__global__ void k_cgls_beta(Unit* us, const double* ss, int B, int tv) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    if (!un.stepped) {
        un.beta[0] = un.beta[1] = 0.0;
        return;
    }
    for (int c = 0; c < 2; ++c) {
        un.beta[c] = un.act[c] ? safe_div(ss[2 * b + c], un.gamma[c], 0.0) : 0.0;
        un.gamma[c] = ss[2 * b + c];
    }
    (void)tv;
}

// CGS (solvers.py:280-291): sigma = <shadow, M p>; any channel |sigma| > 0
// steps with alpha = rho / sigma (safe division), else the unit stops
// (breakdown: converged = False, not thrown)
__global__ void k_cgs_alpha(Unit* us, const double* sig, int B) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    un.stepped = 0;
    un.alpha[0] = un.alpha[1] = 0.0;
    if (!un.active) return;
    bool any = false;
    for (int c = 0; c < 2; ++c) {
        const bool a = !(un.single && c == 1) && fabs(sig[2 * b + c]) > 0;
        un.act[c] = a;
        any = any || a;
    }
    if (!any) {
        un.status = ST_STOPPED;
        un.active = 0;
        un.converged = 0;
        return;
    }
    for (int c = 0; c < 2; ++c) un.alpha[c] = un.act[c] ? safe_div(un.gamma[c], sig[2 * b + c], 0.0) : 0.0;
    un.stepped = 1;
}

// residual of b - A u (history, non-finite u, tol), then rho_new / beta
// (solvers.py:292-304)
__global__ void k_cgs_check(Unit* us, const double* ac, const double* nf, const double* rho_new,
                            int P, int it, int B, double* hist, double tol) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    un.beta[0] = un.beta[1] = 0.0;
    if (!un.stepped) return;
    record_residual(un, ac + 2 * b, P, it, B, b, hist, nf[b] > 0, false, tol, false);
    if (!un.active) return;
    bool any = false;
    for (int c = 0; c < 2; ++c) any = any || (!(un.single && c == 1) && fabs(rho_new[2 * b + c]) > 0);
    if (!any) {
        un.status = ST_STOPPED;
        un.active = 0;
        un.converged = 0;
        return;
    }
    for (int c = 0; c < 2; ++c) {
        un.beta[c] = (un.single && c == 1) ? 0.0 : safe_div(rho_new[2 * b + c], un.gamma[c], 0.0);
        un.gamma[c] = rho_new[2 * b + c];
    }
}

// non-finite u after a step overrides the tol decision (solvers.py:217 precedes :219)
__global__ void k_flag_nonfinite(Unit* us, const double* nf, int B, int only_stepped) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    if (un.status == ST_PAD) return;
    if (only_stepped && !un.stepped) return;
    if (nf[b] > 0 && un.status != ST_NONFINITE) {
        un.status = ST_NONFINITE;
        un.active = 0;
        un.converged = 0;
    }
}

// TV: mu per channel (cfg or 0.1 max|A^H b|), lam = 2 mu  (solvers.py:364-375)
__global__ void k_tv_mu(Unit* us, const double* mx, double cfg_mu, int B) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    for (int c = 0; c < 2; ++c) {
        double mu = cfg_mu > 0 ? cfg_mu : 0.1 * mx[2 * b + c];
        if (!(mu > 0)) mu = 1.0;
        if (un.single && c == 1) mu = cfg_mu > 0 ? cfg_mu : un.mu[0];
        un.mu[c] = mu;
        un.lam[c] = 2.0 * mu;
    }
    if (un.single && cfg_mu <= 0) {  // channel 1 copies channel 0 (kappa[-1], solvers.py:338)
        un.mu[1] = un.mu[0];
        un.lam[1] = un.lam[0];
    }
    for (int c = 0; c < 2; ++c) un.kap[c] = 1.0 / un.lam[c];
}

__global__ void k_tv_inner_begin(Unit* us, const double* ss, int B) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    un.inner_stop = 0;
    un.gamma[0] = ss[2 * b];
    un.gamma[1] = ss[2 * b + 1];
}

__global__ void k_tv_check(Unit* us, const double* ac, const double* nf, int P, int it, int B,
                           double* hist, double tol) {
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    if (!un.active) return;
    if (nf[b] > 0) {  // _check_finite(u, "tv") precedes the residual (solvers.py:417)
        un.status = ST_NONFINITE;
        un.active = 0;
        return;
    }
    record_residual(un, ac + 2 * b, P, it, B, b, hist, false, false, tol, true);
}

__global__ void k_tv_finish(Unit* us, int B) {  // for/else: full run counts as converged
    const int b = threadIdx.x;
    if (b >= B) return;
    Unit& un = us[b];
    if (un.status == RUNNING) {
        un.status = ST_CONVERGED;
        un.converged = 1;
        un.active = 0;
    }
}

// ------------------------------------------------------------------ host driver

template <typename R>
struct Solver {
    using C = typename CT<R>::T;
    sptb_plan* p;
    int B;
    cudaStream_t st;
    int nblk_grid = 0, nblk_spec = 0;
    // plan precision
    C *U = nullptr, *G = nullptr, *W = nullptr, *BH = nullptr, *RH = nullptr, *QH = nullptr;
    // float64 Krylov state (CGLS / TV)
    D2 *Ud = nullptr, *Pd = nullptr;  // CGS iterate and direction (fp64)
    C *bx = nullptr, *by = nullptr, *rx = nullptr, *ry = nullptr;  // TV: Bregman b, stacked target rho
    C *rx2 = nullptr, *ry2 = nullptr;  // TV: the other rho buffer of the fused step
    D2 *Rg = nullptr, *SHg = nullptr, *Qg = nullptr, *Hg = nullptr, *Vg = nullptr;  // CGS
    double *part = nullptr, *sums = nullptr, *sums2 = nullptr, *sums3 = nullptr, *hist = nullptr;
    Unit* us = nullptr;
    Global* gl = nullptr;
    int* pinned = nullptr;
    static constexpr int LAG = 2;  // the host runs up to LAG iterations ahead of the device
    cudaEvent_t ev[LAG + 1] = {};
    std::vector<std::pair<size_t, void*>> owned;
    // iteration bodies after the first are captured once and replayed as a
    // CUDA graph: one launch per iteration instead of 10-40 (the small
    // per-slice scalar kernels made launch overhead dominate at config-1 size)
    cudaGraphExec_t gexec = nullptr;
    long long gkernels = 0;
    bool gfail = false;

    template <class F>
    int iterate(int it, F&& body) {
        if (it == 0 || gfail || switches().no_graph) return body();
        if (!gexec) {
            const long long l0 = sptb_launch_count();
            if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
                cudaGetLastError();
                gfail = true;
                return body();
            }
            const int rc = body();
            cudaGraph_t g = nullptr;
            const cudaError_t e = cudaStreamEndCapture(st, &g);
            gkernels = sptb_launch_count() - l0;
            count_launch((int)-gkernels);  // captured, not run
            if (rc != SPTB_OK || e != cudaSuccess || !g) {
                if (g) cudaGraphDestroy(g);
                cudaGetLastError();
                gfail = true;
                return rc != SPTB_OK ? rc : body();
            }
            const cudaError_t ei = cudaGraphInstantiate(&gexec, g, 0);
            cudaGraphDestroy(g);
            if (ei != cudaSuccess) {
                cudaGetLastError();
                gexec = nullptr;
                gfail = true;
                return body();
            }
        }
        SPTB_CUDA(cudaGraphLaunch(gexec, st));
        count_launch((int)gkernels);
        return SPTB_OK;
    }

    // buffers come from / return to the plan's pool (best fit within 2x)
    int alloc(void** ptr, size_t bytes) {
        auto& pool = p->pool;
        int best = -1;
        for (int i = 0; i < (int)pool.size(); ++i)
            if (pool[i].first >= bytes && pool[i].first <= 2 * bytes &&
                (best < 0 || pool[i].first < pool[best].first))
                best = i;
        if (best >= 0) {
            owned.push_back(pool[best]);
            *ptr = pool[best].second;
            pool.erase(pool.begin() + best);
            return SPTB_OK;
        }
        if (cudaMalloc(ptr, bytes) != cudaSuccess) {
            cudaGetLastError();
            for (auto& kv : pool) cudaFree(kv.second);  // retry after dropping the cache
            pool.clear();
            if (cudaMalloc(ptr, bytes) != cudaSuccess) {
                cudaGetLastError();
                return fail(SPTB_ERR_OOM, "solver buffers: out of device memory");
            }
        }
        owned.push_back({bytes, *ptr});
        return SPTB_OK;
    }
    ~Solver() {
        if (gexec) cudaGraphExecDestroy(gexec);
        // stream-ordered reuse: the next solve runs on the same stream
        for (auto& kv : owned) p->pool.push_back(kv);
    }

    int init(int algo, int max_iter, bool cgs) {
        st = p->stream;
        SPTB_TRY(ensure_work(p, B));
        const size_t gb = sizeof(C) * (size_t)B * p->M, sb = sizeof(C) * (size_t)B * p->N;
        const size_t gd = sizeof(D2) * (size_t)B * p->M;
        W = (C*)p->G0;
        SPTB_TRY(alloc((void**)&BH, sb));
        SPTB_TRY(alloc((void**)&RH, sb));
        SPTB_TRY(alloc((void**)&QH, sb));
        if (algo == SPTB_ALGO_CGLS && cgs) {  // CGS: fp64 grid vectors
            SPTB_TRY(alloc((void**)&Ud, gd));
            SPTB_TRY(alloc((void**)&Pd, gd));
        } else {  // FBP / SIRT / CGLS / TV: iterate (and p) in the plan's type
            SPTB_TRY(alloc((void**)&U, gb));
            SPTB_TRY(alloc((void**)&G, gb));
        }
        if (algo == SPTB_ALGO_TV) {
            for (C** q : {&bx, &by, &rx, &ry, &rx2, &ry2}) SPTB_TRY(alloc((void**)q, gb));
        }
        if (algo == SPTB_ALGO_CGLS && cgs) {
            for (D2** q : {&Rg, &SHg, &Qg, &Hg, &Vg}) SPTB_TRY(alloc((void**)q, gd));
        }
        nblk_grid = std::max(1, 1184 / B);
        nblk_spec = p->T * SPEC_Q;
        // partial sums: k_grid (nblk_grid blocks), k_spec (nblk_spec) and the
        // fused x passes (Y / 4 row groups), up to 4 sums per unit
        const size_t np = (size_t)std::max({nblk_grid, nblk_spec, (int)(p->Y / 4)}) * B * 4;
        SPTB_TRY(alloc((void**)&part, sizeof(double) * np));
        SPTB_TRY(alloc((void**)&sums, sizeof(double) * B * 4));
        SPTB_TRY(alloc((void**)&sums2, sizeof(double) * B * 4));
        SPTB_TRY(alloc((void**)&sums3, sizeof(double) * B * 4));
        SPTB_TRY(alloc((void**)&hist, sizeof(double) * (size_t)std::max(max_iter, 1) * B));
        SPTB_TRY(alloc((void**)&us, sizeof(Unit) * B));
        SPTB_TRY(alloc((void**)&gl, sizeof(Global)));
        static_assert(LAG + 1 <= 4, "plan keeps 4 early-exit events");
        if (!p->solver_pinned) {
            SPTB_CUDA(cudaHostAlloc((void**)&p->solver_pinned, sizeof(int) * 4, cudaHostAllocDefault));
            for (auto& e : p->solver_ev) SPTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        pinned = p->solver_pinned;
        for (int i = 0; i <= LAG; ++i) ev[i] = p->solver_ev[i];
        return SPTB_OK;
    }

    int zero_state(int algo) {
        const size_t gb = sizeof(C) * (size_t)B * p->M, gd = sizeof(D2) * (size_t)B * p->M;
        if (U) SPTB_CUDA(cudaMemsetAsync(U, 0, gb, st));
        if (Ud) SPTB_CUDA(cudaMemsetAsync(Ud, 0, gd, st));
        if (algo == SPTB_ALGO_TV)
            for (C* q : {bx, by, rx, ry}) SPTB_CUDA(cudaMemsetAsync(q, 0, gb, st));  // u = d = b = 0: rho = 0
        return SPTB_OK;
    }

    template <int K, bool MAX = false, class Op>
    int grid(const Op& op, double* out_sums) {
        dim3 g(nblk_grid, B);
        k_grid<K, MAX, Op><<<g, RT, 0, st>>>(op, p->M, part);
        SPTB_LAUNCHED();
        if (K > 0 && out_sums) {
            k_finish<<<B * K, FT, 0, st>>>(part, nblk_grid, B, K, MAX ? 1 : 0,
                                                          out_sums);
            SPTB_LAUNCHED();
        }
        return SPTB_OK;
    }

    template <bool UPDATE, typename RV>
    int spec(RV* rh, const C* qh, C* rf, double* out_sums) {
        k_spec<R, RV, UPDATE><<<nblk_spec, RT, 0, st>>>(rh, qh, rf, p->shp.perm, (const R*)p->w_dev, p->w_len,
                                                        p->T, p->P, B, us, part);
        SPTB_LAUNCHED();
        k_finish<<<B * 2, FT, 0, st>>>(part, nblk_spec, B, 2, 0, out_sums);
        SPTB_LAUNCHED();
        return SPTB_OK;
    }

    int fft(cufftHandle h, void* z, int dir) {
        if (z == (void*)W && fft2_inplace_ok(p, z))  // the grid FFT2: fused column + row passes
            return launch_fft2_inplace(p, z, B, dir == CUFFT_INVERSE, st);
        count_fft();
        if (sizeof(R) == 8)
            SPTB_CUFFT(cufftExecZ2Z(h, (cufftDoubleComplex*)z, (cufftDoubleComplex*)z, dir));
        else
            SPTB_CUFFT(cufftExecC2C(h, (cufftComplex*)z, (cufftComplex*)z, dir));
        return SPTB_OK;
    }

    // fused SIRT update + x pass (complex64, fused FFT2 usable, S^H via TMA)
    bool sirt_fused_ok() const {
        return sizeof(R) == 4 && fft2_inplace_ok(p, W) && tma_ok(p, W) && !switches().sirt_unfused;
    }
    int sirt_update_forward(int nonneg) {
        if constexpr (sizeof(R) == 4) {
            const int L = fft2_log2(p->X);
            const float2* tw = fft2_twiddles(p, L);
            if (!tw) return fail(SPTB_ERR_CUDA, "fft2: twiddle table");
            SPTB_CUDA(cudaMemsetAsync(sums2, 0, sizeof(double) * B, st));
            const unsigned grid = (unsigned)((long long)B * p->Y / 4);
            auto run = [&](auto kern, int logn) -> int {
                const int nt = 4 * (1 << logn) / 16, sm = (int)(sizeof(float2) * 4 * (1 << logn));
                SPTB_CUDA(set_smem_once((const void*)kern, sm, -1));
                kern<<<grid, nt, sm, st>>>((float2*)U, (const float2*)G, (float2*)W, (const float*)p->deapo, us,
                                           nonneg, p->M, p->Y, tw, sums2);
                SPTB_LAUNCHED();
                return SPTB_OK;
            };
            switch (L) {
                case 9: SPTB_TRY(run(k_sirt_update_rowfft<9>, 9)); break;
                case 10: SPTB_TRY(run(k_sirt_update_rowfft<10>, 10)); break;
                case 11: SPTB_TRY(run(k_sirt_update_rowfft<11>, 11)); break;
                case 12: SPTB_TRY(run(k_sirt_update_rowfft<12>, 12)); break;
                default: return fail(SPTB_ERR_ARG, "sirt fused pass: unsupported n_x");
            }
            SPTB_TRY(launch_fft2_cols(p, W, B, false, st));
            return launch_spmm_sh_patch<R>(p, W, RH, B, BH, st);
        } else {
            (void)nonneg;
            return fail(SPTB_ERR_STATE, "sirt fused pass: complex64 only");
        }
    }

    // S_(w) RH -> W, y pass, then the x pass fused with OpAdjPost<R, true> -> G, sums3
    int sirt_adjoint_post(double scale) {
        if constexpr (sizeof(R) == 4) {
            const int L = fft2_log2(p->X);
            const float2* tw = fft2_twiddles(p, L);
            if (!tw) return fail(SPTB_ERR_CUDA, "fft2: twiddle table");
            const void* vals = p->SW_val ? p->SW_val : p->S.val;
            SPTB_TRY(launch_spmm_s<R>(p, vals, RH, W, B, st));
            SPTB_TRY(launch_fft2_cols(p, W, B, true, st));
            const unsigned grid = (unsigned)((long long)B * p->Y / 4);
            auto run = [&](auto kern, int logn) -> int {
                const int nt = 4 * (1 << logn) / 16, sm = (int)(sizeof(float2) * 4 * (1 << logn));
                SPTB_CUDA(set_smem_once((const void*)kern, sm, -1));
                kern<<<grid, nt, sm, st>>>((const float2*)W, (float2*)G, (const float*)p->deapo, scale, p->M, p->Y,
                                           B, tw, part);
                SPTB_LAUNCHED();
                return SPTB_OK;
            };
            switch (L) {
                case 9: SPTB_TRY(run(k_sirt_adjpost_rowfft<9>, 9)); break;
                case 10: SPTB_TRY(run(k_sirt_adjpost_rowfft<10>, 10)); break;
                case 11: SPTB_TRY(run(k_sirt_adjpost_rowfft<11>, 11)); break;
                case 12: SPTB_TRY(run(k_sirt_adjpost_rowfft<12>, 12)); break;
                default: return fail(SPTB_ERR_ARG, "sirt fused pass: unsupported n_x");
            }
            k_finish<<<B * 4, FT, 0, st>>>(part, p->Y / 4, B, 4, 0, sums3);
            SPTB_LAUNCHED();
            return SPTB_OK;
        } else {
            (void)scale;
            return fail(SPTB_ERR_STATE, "sirt fused pass: complex64 only");
        }
    }

    // TV element passes fused with the FFT2 x passes (k_tv_rowfft)
    bool tv_fused_ok() const {
        return sizeof(R) == 4 && fft2_inplace_ok(p, W) && p->Y % 4 == 0 && !switches().xpass_unfused;
    }
    template <bool INV_IN, bool FWD_OUT, int K, class Op>
    int tv_row(const Op& op, double* out_sums) {
        if constexpr (sizeof(R) == 4) {
            const int L = fft2_log2(p->X);
            const float2* tw = fft2_twiddles(p, L);
            if (!tw) return fail(SPTB_ERR_CUDA, "fft2: twiddle table");
            const unsigned grid = (unsigned)((long long)B * p->Y / 4);
            auto run = [&](auto kern, int logn) -> int {
                const int nt = 4 * (1 << logn) / 16;
                const int sm = (INV_IN || FWD_OUT) ? (int)(sizeof(float2) * 4 * (1 << logn)) : 0;
                if (sm) SPTB_CUDA(set_smem_once((const void*)kern, sm, -1));
                kern<<<grid, nt, sm, st>>>(op, (float2*)W, p->M, p->Y, B, tw, part);
                SPTB_LAUNCHED();
                return SPTB_OK;
            };
            switch (L) {
                case 9: SPTB_TRY(run(k_tv_rowfft<9, INV_IN, FWD_OUT, K, Op>, 9)); break;
                case 10: SPTB_TRY(run(k_tv_rowfft<10, INV_IN, FWD_OUT, K, Op>, 10)); break;
                case 11: SPTB_TRY(run(k_tv_rowfft<11, INV_IN, FWD_OUT, K, Op>, 11)); break;
                case 12: SPTB_TRY(run(k_tv_rowfft<12, INV_IN, FWD_OUT, K, Op>, 12)); break;
                default: return fail(SPTB_ERR_ARG, "tv fused pass: unsupported n_x");
            }
            if (out_sums) {
                k_finish<<<B * K, FT, 0, st>>>(part, p->Y / 4, B, K, 0, out_sums);
                SPTB_LAUNCHED();
            }
            return SPTB_OK;
        } else {
            (void)op;
            (void)out_sums;
            return fail(SPTB_ERR_STATE, "tv fused pass: complex64 only");
        }
    }
    // S_(w) rh -> W and the inverse y pass (the x pass is fused into the next op)
    int adjoint_cols(const C* rh) {
        const void* vals = p->SW_val ? p->SW_val : p->S.val;
        SPTB_TRY(launch_spmm_s<R>(p, vals, rh, W, B, st));
        return launch_fft2_cols(p, W, B, true, st);
    }
    // the forward y pass of W (x pass done) and S^H: out = (sub -) S^H W
    int forward_cols(C* out, const C* sub) {
        SPTB_TRY(launch_fft2_cols(p, W, B, false, st));
        return launch_spmm_sh_patch<R>(p, W, out, B, sub, st);
    }

    // out[s][b] = (sub ? sub - : ) S^H FFT2(W)    (W holds deapo*v, [b][m]; clobbered)
    int forward_spec(C* out, const C* sub) {
        FFTPlans* f;
        SPTB_TRY(get_fft(p, B, &f));
        SPTB_TRY(fft(f->fft2, W, CUFFT_FORWARD));
        // patch-grouped S^H reads the batch-outer FFT2 output directly
        return launch_spmm_sh_patch<R>(p, W, out, B, sub, st);
    }

    // W[b][m] = IFFT2(S_(w) rh)   (caller applies deapo/P)
    int adjoint_grid(const C* rh, bool filtered) {
        FFTPlans* f;
        SPTB_TRY(get_fft(p, B, &f));
        const void* vals = (filtered && p->SW_val) ? p->SW_val : p->S.val;
        SPTB_TRY(launch_spmm_s<R>(p, vals, rh, W, B, st));
        return fft(f->fft2, W, CUFFT_INVERSE);
    }

    // BH = FFT1(sino) in [s][b]; units from caller slices
    int load_sino(const void* in, int fmt, int64_t n, int64_t u0, int nb) {
        FFTPlans* f;
        SPTB_TRY(get_fft(p, B, &f));
        SPTB_TRY(launch_pack<R>(in, fmt, n, u0, nb, B, p->N, nullptr, p->S0, st));
        SPTB_TRY(fft(f->fft1, p->S0, CUFFT_FORWARD));
        return launch_transpose_permute<R>(p->S0, BH, p->shp.perm, B, p->N, st);
    }

    int unit_kernel_done() {
        SPTB_LAUNCHED();
        return SPTB_OK;
    }

    // lagged early exit: true when every unit had stopped LAG iterations ago
    int poll(int it, bool* stop) {
        *stop = false;
        k_count_active<<<1, 64, 0, st>>>(us, B, gl);
        SPTB_LAUNCHED();
        SPTB_CUDA(cudaMemcpyAsync(pinned + it % (LAG + 1), &gl->n_active, sizeof(int),
                                  cudaMemcpyDeviceToHost, st));
        SPTB_CUDA(cudaEventRecord(ev[it % (LAG + 1)], st));
        if (it >= LAG) {
            SPTB_CUDA(cudaEventSynchronize(ev[(it - LAG) % (LAG + 1)]));
            if (pinned[(it - LAG) % (LAG + 1)] == 0) *stop = true;
        }
        return SPTB_OK;
    }

    const R* deapo() const { return (const R*)p->deapo; }

    // ---------------------------------------------------------------- FBP
    int run_fbp() {
        const bool filt = p->SW_val != nullptr;
        const double scale = (filt ? p->calib : 1.0) / p->P;
        SPTB_TRY(adjoint_grid(BH, filt));
        SPTB_TRY(grid<0>(OpStore<R, C>{W, U, deapo(), scale}, nullptr));
        // weighted residual of the reprojection (solvers.py:125-128)
        SPTB_TRY(grid<0>(OpDeapo<R, C>{U, W, deapo(), 1.0}, nullptr));
        SPTB_TRY(forward_spec(RH, BH));
        SPTB_TRY(grid<1>(OpNonfinite<C>{U}, sums2));
        SPTB_TRY(spec<false>(RH, (const C*)nullptr, (C*)nullptr, sums));
        k_fbp_check<<<1, 64, 0, st>>>(us, sums, sums2, p->P, B, hist);
        return unit_kernel_done();
    }

    // ---------------------------------------------------------------- SIRT
    int run_sirt(const sptb_solver_config& cfg) {
        const double invP = 1.0 / p->P;
        // g = A^H W b ; alpha0 from ||A g||_w  (solvers.py:151-156)
        SPTB_TRY(adjoint_grid(BH, true));
        SPTB_TRY(grid<2>(OpAdjPost<R, false>{W, G, deapo(), invP}, sums2));
        SPTB_TRY(grid<0>(OpDeapo<R, C>{G, W, deapo(), 1.0}, nullptr));
        SPTB_TRY(forward_spec(QH, nullptr));
        SPTB_TRY(spec<false>(QH, (const C*)nullptr, (C*)nullptr, sums));
        k_sirt_alpha0<<<1, 64, 0, st>>>(us, sums2, sums, p->P, B);
        SPTB_TRY(unit_kernel_done());
        for (int it = 0; it < cfg.max_iter; ++it) {
            bool stop;
            SPTB_TRY(poll(it, &stop));
            if (stop) break;
            SPTB_TRY(iterate(it, [&]() -> int {
            // u += alpha g ; W = deapo u ; non-finite count ; Rhat = Bhat - F(u)
            if (sirt_fused_ok()) {
                SPTB_TRY(sirt_update_forward(cfg.nonneg));
            } else {
                SPTB_TRY(grid<1>(OpSirtUpdate<R>{U, G, W, deapo(), us, cfg.nonneg}, sums2));
                SPTB_TRY(forward_spec(RH, BH));
            }
            SPTB_TRY(spec<false>(RH, (const C*)nullptr, (C*)nullptr, sums));
            k_sirt_check<<<1, 64, 0, st>>>(us, sums, sums2, p->P, it, B, hist, cfg.tol);
            SPTB_TRY(unit_kernel_done());
            // g_new = A^H W r ; BB dots against the previous g
            if (sirt_fused_ok()) {
                SPTB_TRY(sirt_adjoint_post(invP));
            } else {
                SPTB_TRY(adjoint_grid(RH, true));
                SPTB_TRY(grid<4>(OpAdjPost<R, true>{W, G, deapo(), invP}, sums3));
            }
            k_sirt_alpha<<<1, 64, 0, st>>>(us, sums3, B, cfg.bb_enabled);
            return unit_kernel_done();
            }));
        }
        return SPTB_OK;
    }


    // ---------------------------------------------------------------- CGLS
    int run_cgls(const sptb_solver_config& cfg) {
        const double invP = 1.0 / p->P;
        // r = b (u0 = 0); s = A^H W r; p = s; gamma = <s,s>  (solvers.py:197-203).
        // u, p and the spectral residual are stored in the plan's type (the
        // passes are HBM-bound), the recurrence arithmetic is fp64
        SPTB_CUDA(cudaMemcpyAsync(RH, BH, sizeof(C) * (size_t)B * p->N, cudaMemcpyDeviceToDevice, st));
        // fused: the element passes share the FFT2 x passes (k_tv_rowfft), W
        // leaves every iteration x-transformed for the next forward y pass
        const bool fused = tv_fused_ok();
        if (fused) {
            SPTB_TRY(adjoint_cols(BH));
            SPTB_TRY((tv_row<true, true, 2>(OpCglsInit<R, C>{W, G, deapo(), invP}, sums2)));
        } else {
            SPTB_TRY(adjoint_grid(BH, true));
            SPTB_TRY(grid<2>(OpCglsInit<R, C>{W, G, deapo(), invP}, sums2));
        }
        k_cgls_init<<<1, 64, 0, st>>>(us, sums2, B);
        SPTB_TRY(unit_kernel_done());
        for (int it = 0; it < cfg.max_iter; ++it) {
            bool stop;
            SPTB_TRY(poll(it, &stop));
            if (stop) break;
            if (fused) {
                SPTB_TRY(iterate(it, [&]() -> int {
                SPTB_TRY(forward_cols(QH, nullptr));
                SPTB_TRY(spec<false>(QH, (const C*)nullptr, (C*)nullptr, sums));
                k_cgls_alpha<<<1, 64, 0, st>>>(us, sums, nullptr, p->P, B, 0);
                SPTB_TRY(unit_kernel_done());
                SPTB_TRY(spec<true>(RH, QH, (C*)nullptr, sums));
                k_cgls_check<<<1, 64, 0, st>>>(us, sums, p->P, it, B, hist, cfg.tol);
                SPTB_TRY(unit_kernel_done());
                // s = A^H W r: IFFT_x + gamma_new
                SPTB_TRY(adjoint_cols(RH));
                SPTB_TRY((tv_row<true, false, 2>(OpDotS<R>{W, deapo(), invP}, sums2)));
                k_cgls_beta<<<1, 64, 0, st>>>(us, sums2, B, 0);
                SPTB_TRY(unit_kernel_done());
                // u += alpha p ; p = s + beta p ; FFT_x(deapo p_new)
                SPTB_TRY((tv_row<false, true, 1>(OpCglsTail<R, C>{U, G, W, deapo(), invP, us}, sums3)));
                k_flag_nonfinite<<<1, 64, 0, st>>>(us, sums3, B, 1);
                return unit_kernel_done();
                }));
                continue;
            }
            SPTB_TRY(iterate(it, [&]() -> int {
            // q = A p  -> delta, alpha, activity
            SPTB_TRY(forward_spec(QH, nullptr));
            SPTB_TRY(spec<false>(QH, (const C*)nullptr, (C*)nullptr, sums));
            k_cgls_alpha<<<1, 64, 0, st>>>(us, sums, nullptr, p->P, B, 0);
            SPTB_TRY(unit_kernel_done());
            // r -= alpha q (mirror mix, fp64 arithmetic, in place) and ||r||_w
            SPTB_TRY(spec<true>(RH, QH, (C*)nullptr, sums));
            k_cgls_check<<<1, 64, 0, st>>>(us, sums, p->P, it, B, hist, cfg.tol);
            SPTB_TRY(unit_kernel_done());
            // s = A^H W r ; gamma_new ; beta
            SPTB_TRY(adjoint_grid(RH, true));
            SPTB_TRY(grid<2>(OpDotS<R>{W, deapo(), invP}, sums2));
            k_cgls_beta<<<1, 64, 0, st>>>(us, sums2, B, 0);
            SPTB_TRY(unit_kernel_done());
            // u += alpha p ; p = s + beta p ; W = deapo p_new
            SPTB_TRY(grid<1>(OpCglsTail<R, C>{U, G, W, deapo(), invP, us}, sums3));
            k_flag_nonfinite<<<1, 64, 0, st>>>(us, sums3, B, 1);
            return unit_kernel_done();
            }));
        }
        if (cfg.nonneg) SPTB_TRY(grid<0>(OpNonneg<C>{U, us}, nullptr));
        return SPTB_OK;
    }

    // ---------------------------------------------------------------- CGS
    // cgs_mode of solve_cgls (solvers.py:262-305).  M v = A^H W A v costs one
    // forward and one adjoint application; an iteration applies M twice and
    // A once more for the reported residual b - A u.
    int normal_apply() {  // W holds deapo*v on entry, IFFT2(S_w F(v)) on exit
        SPTB_TRY(forward_spec(QH, nullptr));
        return adjoint_grid(QH, true);
    }

    int run_cgs(const sptb_solver_config& cfg) {
        const double invP = 1.0 / p->P;
        // c = A^H W b ; r = shadow = p = q = c ; rho = <shadow, r>
        SPTB_TRY(adjoint_grid(BH, true));
        SPTB_TRY(grid<2>(OpCgsInit<R>{W, Rg, SHg, Pd, Qg, deapo(), invP}, sums2));
        k_cgls_init<<<1, 64, 0, st>>>(us, sums2, B);  // gamma := rho
        SPTB_TRY(unit_kernel_done());
        for (int it = 0; it < cfg.max_iter; ++it) {
            bool stop;
            SPTB_TRY(poll(it, &stop));
            if (stop) break;
            SPTB_TRY(iterate(it, [&]() -> int {
            // v = M p ; sigma ; alpha
            SPTB_TRY(normal_apply());
            SPTB_TRY(grid<2>(OpCgsV<R>{W, SHg, Vg, deapo(), invP}, sums2));
            k_cgs_alpha<<<1, 64, 0, st>>>(us, sums2, B);
            SPTB_TRY(unit_kernel_done());
            // h = q - alpha v ; u += alpha (q + h) ; r -= alpha M (q + h)
            SPTB_TRY(grid<1>(OpCgsStep<R>{Ud, Hg, Qg, Vg, W, deapo(), us}, sums3));
            SPTB_TRY(normal_apply());
            SPTB_TRY(grid<2>(OpCgsResid<R>{W, Rg, SHg, Ud, deapo(), invP, us}, sums2));
            // reported residual b - A u ; tol ; rho_new ; beta
            SPTB_TRY(forward_spec(RH, BH));
            SPTB_TRY(spec<false>(RH, (const C*)nullptr, (C*)nullptr, sums));
            k_cgs_check<<<1, 64, 0, st>>>(us, sums, sums3, sums2, p->P, it, B, hist, cfg.tol);
            SPTB_TRY(unit_kernel_done());
            // q = r + beta h ; p = q + beta (h + beta p) ; W = deapo p
            return grid<0>(OpCgsDir<R>{Rg, Hg, Qg, Pd, W, deapo(), us}, nullptr);
            }));
        }
        if (cfg.nonneg) SPTB_TRY(grid<0>(OpNonneg<D2>{Ud, us}, nullptr));
        return SPTB_OK;
    }

    // ---------------------------------------------------------------- TV
    // One outer iteration with the element passes fused into the FFT2 x
    // passes (same algorithm and arithmetic as the unfused body in run_tv;
    // the sums are reduced per grid row group instead of per k_grid block)
    int tv_outer_fused(int inner, double invP, int it, int nonneg, double tol) {
        const int X = p->X, Y = p->Y;
        // r = target - fwd(u), s = adj(r), p = s: IFFT_x + OpTvS<0> + FFT_x
        SPTB_TRY(adjoint_cols(RH));
        SPTB_TRY((tv_row<true, true, 2>(OpTvS<R, 0, C>{W, G, rx, ry, deapo(), invP, us, X, Y}, sums2)));
        k_tv_inner_begin<<<1, 64, 0, st>>>(us, sums2, B);
        SPTB_TRY(unit_kernel_done());
        C *ra = rx, *rb = ry, *wa = rx2, *wb = ry2;
        for (int j = 0; j < inner; ++j) {
            SPTB_TRY(forward_cols(QH, nullptr));  // Qhat = F(p) (x pass done)
            SPTB_TRY(spec<false>(QH, (const C*)nullptr, (C*)nullptr, sums));
            // ||grad p||^2 in 4-row groups (x, y known per lane)
            SPTB_TRY((tv_row<false, false, 2>(OpTvGradNorm<C>{G, us, X, Y}, sums2)));
            k_cgls_alpha<<<1, 64, 0, st>>>(us, sums, sums2, p->P, B, 1);
            SPTB_TRY(unit_kernel_done());
            if (j == inner - 1) {
                SPTB_TRY(grid<0>(OpTvAxpy<C>{U, G, us, nonneg}, nullptr));
                break;
            }
            SPTB_TRY(spec<true>(RH, QH, (C*)nullptr, sums));
            SPTB_TRY(adjoint_cols(RH));
            // IFFT_x + the step (u, rho) + s -> W
            SPTB_TRY((tv_row<true, false, 2>(OpTvStepS<R, C>{W, U, G, ra, rb, wa, wb, deapo(), invP, us, X, Y},
                                             sums2)));
            std::swap(ra, wa);
            std::swap(rb, wb);
            k_cgls_beta<<<1, 64, 0, st>>>(us, sums2, B, 1);
            SPTB_TRY(unit_kernel_done());
            // p = s + beta p ; FFT_x(deapo p)
            SPTB_TRY((tv_row<false, true, 2>(OpTvS<R, 2, C>{W, G, ra, rb, deapo(), invP, us, X, Y}, nullptr)));
        }
        // shrink + Bregman + next target; FFT_x(deapo u); residual b - A u
        SPTB_TRY((tv_row<false, true, 1>(OpTvShrink<R, C>{U, rx, ry, bx, by, W, deapo(), us, X, Y}, sums3)));
        SPTB_TRY(forward_cols(RH, BH));
        SPTB_TRY(spec<false>(RH, (const C*)nullptr, (C*)nullptr, sums));
        k_tv_check<<<1, 64, 0, st>>>(us, sums, sums3, p->P, it, B, hist, tol);
        return unit_kernel_done();
    }

    int run_tv(const sptb_solver_config& cfg) {
        const double invP = 1.0 / p->P;
        const int X = p->X, Y = p->Y;
        // mu: cfg or 0.1 max |A^H b| per channel (unfiltered adjoint)
        if (cfg.mu > 0) {
            k_tv_mu<<<1, 64, 0, st>>>(us, sums3, cfg.mu, B);
        } else {
            SPTB_TRY(adjoint_grid(BH, false));
            SPTB_TRY((grid<2, true>(OpAbsMax<R>{W, deapo(), invP}, sums3)));
            k_tv_mu<<<1, 64, 0, st>>>(us, sums3, 0.0, B);
        }
        SPTB_TRY(unit_kernel_done());
        // u0 = 0 -> rho_a = b.  The TV state (u = U, p = G, rho, b and the
        // spectral residual RH) is stored in the plan's complex type with fp64
        // arithmetic in every pass: the element passes are HBM-bound, and the
        // stacked CGLS restarts every outer iteration after 2 steps
        SPTB_CUDA(cudaMemcpyAsync(RH, BH, sizeof(C) * (size_t)B * p->N, cudaMemcpyDeviceToDevice, st));
        const int inner = std::max(1, cfg.tv_inner_iter);
        const bool fused = tv_fused_ok();
        for (int it = 0; it < cfg.max_iter; ++it) {
            bool stop;
            SPTB_TRY(poll(it, &stop));
            if (stop) break;
            if (fused) {
                SPTB_TRY(iterate(it, [&]() -> int { return tv_outer_fused(inner, invP, it, cfg.nonneg, cfg.tol); }));
                continue;
            }
            SPTB_TRY(iterate(it, [&]() -> int {
            // stacked CGLS on (sqrt(mu) A; sqrt(lam) grad) u = (sqrt(mu) b; sqrt(lam)(d - b));
            // rho = (d - b) - grad u comes from the previous shrink pass (0 at u = 0)
            SPTB_TRY(adjoint_grid(RH, true));
            SPTB_TRY(grid<2>(OpTvS<R, 0, C>{W, G, rx, ry, deapo(), invP, us, X, Y}, sums2));
            k_tv_inner_begin<<<1, 64, 0, st>>>(us, sums2, B);
            SPTB_TRY(unit_kernel_done());
            // rho ping-pongs between (rx, ry) and (rx2, ry2) through the fused
            // step passes; S0 reads and the shrink pass writes (rx, ry)
            C *ra = rx, *rb = ry, *wa = rx2, *wb = ry2;
            for (int j = 0; j < inner; ++j) {
                SPTB_TRY(forward_spec(QH, nullptr));                // Qhat = F(p)
                SPTB_TRY(spec<false>(QH, (const C*)nullptr, (C*)nullptr, sums));
                SPTB_TRY(grid<2>(OpTvGradNorm<C>{G, us, X, Y}, sums2));
                k_cgls_alpha<<<1, 64, 0, st>>>(us, sums, sums2, p->P, B, 1);
                SPTB_TRY(unit_kernel_done());
                if (j == inner - 1) {  // only u += alpha p is live (OpTvAxpy)
                    SPTB_TRY(grid<0>(OpTvAxpy<C>{U, G, us, cfg.nonneg ? 1 : 0}, nullptr));
                    break;
                }
                SPTB_TRY(spec<true>(RH, QH, (C*)nullptr, sums));     // rho_a -= alpha A p (in place)
                SPTB_TRY(adjoint_grid(RH, true));
                // u += alpha p ; rho -= alpha grad p ; s ; <s,s>  (W = s)
                SPTB_TRY(grid<2>(OpTvStepS<R, C>{W, U, G, ra, rb, wa, wb, deapo(), invP, us, X, Y}, sums2));
                std::swap(ra, wa);
                std::swap(rb, wb);
                k_cgls_beta<<<1, 64, 0, st>>>(us, sums2, B, 1);
                SPTB_TRY(unit_kernel_done());
                SPTB_TRY(grid<2>(OpTvS<R, 2, C>{W, G, ra, rb, deapo(), invP, us, X, Y}, nullptr));
            }
            // shrink + Bregman + the next stacked target; W = deapo u; non-finite u
            SPTB_TRY(grid<1>(OpTvShrink<R, C>{U, rx, ry, bx, by, W, deapo(), us, X, Y}, sums3));
            // residual b - A u (reused as the next outer rho_a: same u)
            SPTB_TRY(forward_spec(RH, BH));
            SPTB_TRY(spec<false>(RH, (const C*)nullptr, (C*)nullptr, sums));
            k_tv_check<<<1, 64, 0, st>>>(us, sums, sums3, p->P, it, B, hist, cfg.tol);
            return unit_kernel_done();
            }));
        }
        k_tv_finish<<<1, 64, 0, st>>>(us, B);
        return unit_kernel_done();
    }
};

template <typename R>
int solve_typed(sptb_plan* p, const sptb_solver_config& cfg, const void* sino, int in_fmt,
                void* rec, int out_fmt, int64_t n, double* hist, int32_t* iters,
                int32_t* converged, int32_t* status) {
    using C = typename CT<R>::T;
    const bool cplx = in_fmt & SPTB_FMT_COMPLEX;
    const int64_t units = cplx ? n : (n + 1) / 2;
    const int iters_cap = cfg.algorithm == SPTB_ALGO_FBP ? 1 : cfg.max_iter;
    int first_fail = SPTB_OK;
    bool din = true, dout = true;
    is_device_ptr(sino, &din);
    is_device_ptr(rec, &dout);
    const size_t eb = (in_fmt & SPTB_FMT_F64) ? 8 : 4, ebo = (out_fmt & SPTB_FMT_F64) ? 8 : 4;
    const size_t per_in = eb * p->N * (cplx ? 2 : 1), per_out = ebo * p->M * (cplx ? 2 : 1);
    const void* src = sino;
    void* dst = rec;
    if (!din) {
        SPTB_TRY(ensure_stage(&p->stage_in, &p->stage_in_bytes, per_in * n));
        SPTB_CUDA(cudaMemcpyAsync(p->stage_in, sino, per_in * n, cudaMemcpyHostToDevice, p->stream));
        src = p->stage_in;
    }
    if (!dout) {
        SPTB_TRY(ensure_stage(&p->stage_out, &p->stage_out_bytes, per_out * n));
        dst = p->stage_out;
    }
    int Bmax = 1;
    while (Bmax < std::min<int64_t>(units, p->max_batch)) Bmax <<= 1;
    Solver<R> sv;
    sv.p = p;
    sv.B = Bmax;
    SPTB_TRY(sv.init(cfg.algorithm, iters_cap, cfg.cgs_mode != 0));
    std::vector<double> hbuf((size_t)iters_cap * Bmax);
    std::vector<Unit> ubuf(Bmax);
    for (int64_t u0 = 0; u0 < units; u0 += Bmax) {
        const int nb = (int)std::min<int64_t>(Bmax, units - u0);
        const bool single_last = !cplx && (2 * (u0 + nb) > n);
        cudaStream_t st = p->stream;
        k_init_units<<<1, 64, 0, st>>>(sv.us, nb, Bmax, single_last ? 1 : 0, sv.gl);
        SPTB_LAUNCHED();
        SPTB_TRY(sv.zero_state(cfg.algorithm));
        SPTB_CUDA(cudaMemsetAsync(sv.hist, 0, sizeof(double) * (size_t)iters_cap * Bmax, st));
        SPTB_TRY(sv.load_sino(src, in_fmt, n, u0, nb));
        if (cfg.algorithm != SPTB_ALGO_FBP) {  // solve_fbp has no zero-rhs shortcut
            SPTB_TRY(sv.template spec<false>(sv.BH, (const C*)nullptr, (C*)nullptr, sv.sums));
            k_bnorm<<<1, 64, 0, st>>>(sv.us, sv.sums, p->P, Bmax);
            SPTB_LAUNCHED();
        }
        switch (cfg.algorithm) {
            case SPTB_ALGO_FBP: SPTB_TRY(sv.run_fbp()); break;
            case SPTB_ALGO_SIRT: SPTB_TRY(sv.run_sirt(cfg)); break;
            case SPTB_ALGO_CGLS:
                SPTB_TRY(cfg.cgs_mode ? sv.run_cgs(cfg) : sv.run_cgls(cfg));
                break;
            case SPTB_ALGO_TV: SPTB_TRY(sv.run_tv(cfg)); break;
            default: return fail(SPTB_ERR_ARG, "unknown algorithm");
        }
        if (sv.Ud)
            SPTB_TRY(launch_unpack<double>(sv.Ud, p->M, nullptr, 1.0, dst, out_fmt, n, u0, nb, st));
        else
            SPTB_TRY(launch_unpack<R>(sv.U, p->M, nullptr, 1.0, dst, out_fmt, n, u0, nb, st));
        SPTB_CUDA(cudaMemcpyAsync(hbuf.data(), sv.hist, sizeof(double) * hbuf.size(),
                                  cudaMemcpyDeviceToHost, st));
        SPTB_CUDA(cudaMemcpyAsync(ubuf.data(), sv.us, sizeof(Unit) * Bmax, cudaMemcpyDeviceToHost, st));
        SPTB_CUDA(cudaStreamSynchronize(st));
        for (int b = 0; b < nb; ++b) {
            const int64_t u = u0 + b;
            const Unit& un = ubuf[b];
            if (iters) iters[u] = un.iters;
            if (converged) converged[u] = un.converged;
            int s = SPTB_OK;
            if (un.status == ST_DIVERGED) s = SPTB_ERR_DIVERGENCE;
            if (un.status == ST_NONFINITE) s = SPTB_ERR_NONFINITE;
            if (status) status[u] = s;
            if (s != SPTB_OK && first_fail == SPTB_OK) {
                first_fail = s;
                fail(s, std::string(s == SPTB_ERR_DIVERGENCE ? "residual exceeds 10x its minimum"
                                                             : "produced non-finite values") +
                            " (unit " + std::to_string(u) + ")");
            }
            if (hist)
                for (int k = 0; k < iters_cap; ++k)
                    hist[u * iters_cap + k] = k < un.iters ? hbuf[(size_t)k * Bmax + b] : 0.0;
        }
    }
    if (!dout) {
        SPTB_CUDA(cudaMemcpyAsync(rec, dst, per_out * n, cudaMemcpyDeviceToHost, p->stream));
        SPTB_CUDA(cudaStreamSynchronize(p->stream));
    }
    return first_fail;
}

}  // namespace sptb

using namespace sptb;

// Every solver grid pass multiplies by the deapodization plane (M reals),
// re-read once per unit: 32 x 16.8 MB per pass at 2048^2 when the streaming
// W / u / g traffic evicts it from L2 between units.  Pin it in the L2
// persisting carve-out for the solver stream's kernels (captured into the
// iteration graphs with the launches).  SPTB_NO_L2_PERSIST: off (A/B).
static void persist_deapo(sptb_plan* p) {
    const char* off = getenv("SPTB_NO_L2_PERSIST");
    if ((off && off[0] && off[0] != '0') || !p->deapo) return;
    int maxp = 0, maxw = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, p->device);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, p->device);
    const size_t bytes = (size_t)p->M * (p->csize / 2);
    if (maxp <= 0 || maxw <= 0) return;
    const size_t win = std::min(bytes, (size_t)maxw);
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    const size_t want = std::min(win, (size_t)maxp);
    if (cur < want && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    cudaStreamAttrValue a = {};
    a.accessPolicyWindow.base_ptr = p->deapo;
    a.accessPolicyWindow.num_bytes = win;
    a.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)std::max(cur, want) / (double)win);
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(p->solver_stream, cudaStreamAttributeAccessPolicyWindow, &a) != cudaSuccess)
        cudaGetLastError();
}

extern "C" int sptb_solve(sptb_plan* p, const sptb_solver_config* cfg, const void* sino,
                          int32_t in_fmt, void* rec, int32_t out_fmt, int64_t n, double* hist,
                          int32_t* iters, int32_t* converged, int32_t* status) {
    if (!p || !cfg) return fail(SPTB_ERR_ARG, "null argument");
    if ((in_fmt & SPTB_FMT_COMPLEX) != (out_fmt & SPTB_FMT_COMPLEX))
        return fail(SPTB_ERR_ARG, "output kind (real/complex) must match the input's");
    if (cfg->max_iter < 1) return fail(SPTB_ERR_ARG, "max_iter must be >= 1");
    if (cfg->algorithm < SPTB_ALGO_FBP || cfg->algorithm > SPTB_ALGO_TV)
        return fail(SPTB_ERR_ARG, "unknown algorithm");
    if (n <= 0) return SPTB_OK;
    cudaSetDevice(p->device);
    // the solve runs on a plan-owned stream joined to the caller's by events:
    // a capturable stream (the iteration graphs) even when the caller uses
    // the legacy default stream
    if (!p->solver_stream) {
        SPTB_CUDA(cudaStreamCreateWithFlags(&p->solver_stream, cudaStreamNonBlocking));
        for (auto& e : p->solver_join) SPTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        persist_deapo(p);
    }
    cudaStream_t caller = p->stream;
    SPTB_CUDA(cudaEventRecord(p->solver_join[0], caller));
    SPTB_CUDA(cudaStreamWaitEvent(p->solver_stream, p->solver_join[0], 0));
    SPTB_TRY(sptb_plan_set_stream(p, p->solver_stream));  // also rebinds the cuFFT plans
    const int rc = p->prec == SPTB_PREC_F64
                       ? solve_typed<double>(p, *cfg, sino, in_fmt, rec, out_fmt, n, hist, iters, converged,
                                             status)
                       : solve_typed<float>(p, *cfg, sino, in_fmt, rec, out_fmt, n, hist, iters, converged,
                                            status);
    SPTB_TRY(sptb_plan_set_stream(p, caller));
    SPTB_CUDA(cudaEventRecord(p->solver_join[1], p->solver_stream));
    SPTB_CUDA(cudaStreamWaitEvent(caller, p->solver_join[1], 0));
    return rc;
}
