// Radix-16 register FFT building blocks shared by the fused FFT kernels
// (sptb_fft.cu) and the solver's fused grid passes (sptb_solvers.cu):
// complex helpers, DFTs of size 2/4/8/16, twiddle powers from a per-plan
// table (tw[k] = exp(-2 pi i k / N), INV conjugates) and the two exchange
// stages of an N = 2^LOGN transform held 16 points per thread.
#pragma once

#include <cuda_runtime.h>

namespace sptb {
namespace fftcore {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 mul_mi(float2 a) {
    return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft2(float2* v) {
    const float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}
template <bool INV>
__device__ __forceinline__ void dft4(float2* v) {  // in natural order, out natural order
    const float2 d0 = cadd(v[0], v[2]), d1 = csub(v[0], v[2]);
    const float2 d2 = cadd(v[1], v[3]), d3 = mul_mi<INV>(csub(v[1], v[3]));
    v[0] = cadd(d0, d2);
    v[2] = csub(d0, d2);
    v[1] = cadd(d1, d3);
    v[3] = csub(d1, d3);
}
template <bool INV>
__device__ __forceinline__ void dft8(float2* v) {
    constexpr float h = 0.70710678118654752440f;
    float2 e[4], o[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        e[r] = cadd(v[r], v[r + 4]);
        o[r] = csub(v[r], v[r + 4]);
    }
    // o[r] *= w8^r, w8 = exp(-+ i pi / 4)
    o[1] = INV ? make_float2(h * (o[1].x - o[1].y), h * (o[1].x + o[1].y))
               : make_float2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
    o[2] = mul_mi<INV>(o[2]);
    o[3] = INV ? make_float2(-h * (o[3].x + o[3].y), h * (o[3].x - o[3].y))
               : make_float2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
    dft4<INV>(e);
    dft4<INV>(o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[2 * k] = e[k];
        v[2 * k + 1] = o[k];
    }
}

// ---------------------------------------------------------------------------
// Register-resident variant for n_p = 2^LOGN, 512 <= n_p <= 4096: 16 points
// per thread, n_p / 16 threads per transform, three stages of radix 16, 16
// and n_p / 256 computed in registers (the radix-16 DFT as 4 x 4 with
// constant twiddles), two shared-memory exchanges between them.  The XOR
// swizzle i ^ ((i >> 4) & 15) makes every exchange pattern conflict free.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int swz4(int i) { return i ^ ((i >> 4) & 15); }

template <bool INV>
__device__ __forceinline__ float2 tw16(int m) {  // W16^m, m in [0, 16)
    constexpr float c[16] = {1.f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                             0.f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                             -1.f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f,
                             0.f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
    // sin(2 pi m / 16) = cos(2 pi (m - 4) / 16)
    const float sn = c[(m + 12) & 15];
    return make_float2(c[m & 15], INV ? sn : -sn);
}

template <bool INV>
__device__ __forceinline__ void dft16(float2* v) {
    float2 a[4][4];  // a[r1][k0]
#pragma unroll
    for (int r1 = 0; r1 < 4; ++r1) {
        float2 t[4] = {v[r1], v[r1 + 4], v[r1 + 8], v[r1 + 12]};
        dft4<INV>(t);
#pragma unroll
        for (int k0 = 0; k0 < 4; ++k0) a[r1][k0] = (r1 * k0) ? cmul(t[k0], tw16<INV>(r1 * k0)) : t[k0];
    }
#pragma unroll
    for (int k0 = 0; k0 < 4; ++k0) {
        float2 t[4] = {a[0][k0], a[1][k0], a[2][k0], a[3][k0]};
        dft4<INV>(t);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) v[k0 + 4 * k1] = t[k1];
    }
}

template <int R, bool INV>
__device__ __forceinline__ void dft_r(float2* v) {
    if constexpr (R == 16) dft16<INV>(v);
    else if constexpr (R == 8) dft8<INV>(v);
    else if constexpr (R == 4) dft4<INV>(v);
    else dft2<INV>(v);
}

// w[r] = W_N^(m r) for r < R (w[0] unused): W_N^m and W_N^(2m) from the
// table, the rest by products -- each power at most 3 multiplications deep
template <int R, bool INV>
__device__ __forceinline__ void twiddle_powers(float2* w, const float2* __restrict__ tw, int m) {
    float2 w1 = __ldg(tw + m);
    if (INV) w1.y = -w1.y;
    w[1] = w1;
    if constexpr (R > 2) {
        float2 w2 = __ldg(tw + 2 * m);
        if (INV) w2.y = -w2.y;
        w[2] = w2;
        w[3] = cmul(w2, w1);
    }
    if constexpr (R > 4) {
        const float2 w4 = cmul(w[2], w[2]);
        w[4] = w4;
        w[5] = cmul(w4, w[1]);
        w[6] = cmul(w4, w[2]);
        w[7] = cmul(w4, w[3]);
    }
    if constexpr (R > 8) {
        const float2 w8 = cmul(w[4], w[4]);
        w[8] = w8;
#pragma unroll
        for (int r = 9; r < 16; ++r) w[r] = cmul(w8, w[r - 8]);
    }
}

// stages 2 and 3 on one transform held in buf (swizzled); the 16 values of
// stage 1 are in v; on return buf holds the natural-order transform (when
// STORE_SMEM) or v holds X[j + n/R3 * r ... ] for the caller (two butterflies
// of R3 when R3 < 16: v[c * R3 + r] = X[(j + c * T) + 256 * r]).
template <int LOGN, bool INV>
__device__ __forceinline__ void fft16_stages(float2* v, float2* buf, int j, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, T = N / 16, R3 = N / 256, NB3 = 16 / R3;
    // stage 1 output y[16 j + r]
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[swz4(16 * j + r)] = v[r];
    __syncthreads();
    // stage 2: Ns = 16, radix 16; twiddles w^r, w = W_256^(j % 16), built by
    // products of one table load (<= 4 roundings deep)
    {
        float2 w[16];
        twiddle_powers<16, INV>(w, tw, (j & 15) * (N / 256));
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float2 x = buf[swz4(j + T * r)];
            v[r] = r ? cmul(x, w[r]) : x;
        }
    }
    dft16<INV>(v);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[swz4((j >> 4) * 256 + (j & 15) + 16 * r)] = v[r];
    __syncthreads();
    // stage 3: Ns = 256, radix R3, NB3 butterflies per thread (jj = j + c T)
#pragma unroll
    for (int c = 0; c < NB3; ++c) {
        const int jj = j + c * T;
        float2 w[R3];
        twiddle_powers<R3, INV>(w, tw, jj & 255);
#pragma unroll
        for (int r = 0; r < R3; ++r) {
            const float2 x = buf[swz4(jj + (N / R3) * r)];
            v[c * R3 + r] = r ? cmul(x, w[r]) : x;
        }
        dft_r<R3, INV>(v + c * R3);
    }
}



// The twiddles of stages 2 and 3 depend only on the lane (j), not on the
// transform: persistent kernels compute them once and keep them in registers
// (15 + NB3 (R3 - 1) complex values) instead of two table loads and ~30
// complex products per transform.
template <int LOGN, bool INV>
struct StageTwiddles {
    static constexpr int N = 1 << LOGN, T = N / 16, R3 = N / 256, NB3 = 16 / R3;
    float2 w2[16];
    float2 w3[NB3][R3];
    __device__ __forceinline__ StageTwiddles(const float2* __restrict__ tw, int j) {
        twiddle_powers<16, INV>(w2, tw, (j & 15) * (N / 256));
#pragma unroll
        for (int c = 0; c < NB3; ++c) twiddle_powers<R3, INV>(w3[c], tw, (j + c * T) & 255);
    }
};

// fft16_stages with precomputed twiddles (same arithmetic, same results)
template <int LOGN, bool INV>
__device__ __forceinline__ void fft16_stages_pre(float2* v, float2* buf, int j, const StageTwiddles<LOGN, INV>& tw) {
    constexpr int N = 1 << LOGN, T = N / 16, R3 = N / 256, NB3 = 16 / R3;
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[swz4(16 * j + r)] = v[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const float2 x = buf[swz4(j + T * r)];
        v[r] = r ? cmul(x, tw.w2[r]) : x;
    }
    dft16<INV>(v);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[swz4((j >> 4) * 256 + (j & 15) + 16 * r)] = v[r];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NB3; ++c) {
        const int jj = j + c * T;
#pragma unroll
        for (int r = 0; r < R3; ++r) {
            const float2 x = buf[swz4(jj + (N / R3) * r)];
            v[c * R3 + r] = r ? cmul(x, tw.w3[c][r]) : x;
        }
        dft_r<R3, INV>(v + c * R3);
    }
}

// fft16_stages with the stage-2/3 twiddle powers read from the plan's
// per-LOGN tables instead of built by products (one-pass kernels that cannot
// keep StageTwiddles in registers): tw + N holds T2[r][m] = W_N^(m (N/256) r)
// (16 x 16, r-major: a warp's lanes read 16 consecutive entries) and
// tw + N + 256 holds T3[r][m] = W_N^(m r) (R3 x 256), rounded from double.
// Measured against the products: SIRT's update pass 0.881 -> 0.854 ms, the
// TV passes within 1% (the one-pass kernels are bound by memory latency and
// the exchange barriers, not by the twiddle arithmetic)
template <int LOGN, bool INV>
__device__ __forceinline__ void fft16_stages_tab(float2* v, float2* buf, int j, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, T = N / 16, R3 = N / 256, NB3 = 16 / R3;
    const float2* t2 = tw + N;
    const float2* t3 = tw + N + 256;
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[swz4(16 * j + r)] = v[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const float2 x = buf[swz4(j + T * r)];
        if (r) {
            float2 w = __ldg(t2 + r * 16 + (j & 15));
            if (INV) w.y = -w.y;
            v[r] = cmul(x, w);
        } else {
            v[r] = x;
        }
    }
    dft16<INV>(v);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[swz4((j >> 4) * 256 + (j & 15) + 16 * r)] = v[r];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NB3; ++c) {
        const int jj = j + c * T;
#pragma unroll
        for (int r = 0; r < R3; ++r) {
            const float2 x = buf[swz4(jj + (N / R3) * r)];
            if (r) {
                float2 w = __ldg(t3 + r * 256 + (jj & 255));
                if (INV) w.y = -w.y;
                v[c * R3 + r] = cmul(x, w);
            } else {
                v[c * R3 + r] = x;
            }
        }
        dft_r<R3, INV>(v + c * R3);
    }
}

}  // namespace fftcore
}  // namespace sptb
