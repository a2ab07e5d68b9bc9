// Fused detector-axis FFT kernels (complex64, n_p = 2^k, 128 <= n_p <= 4096).
//
// The reference applies fft_P (ortho) to every projection row before S and
// ifft_P after S^H (operators.py:162-165, 178-182).  With cuFFT the device path
// was pack (caller slices -> complex [b][t][p]) + FFT1 + a permuting transpose
// to the SpMM operand layout [s'][b] -- three passes over the sinogram batch.
// These kernels do it in one: a CTA owns one angle t and BG batch columns,
// reads the caller's real slice pairs (or complex slices) straight from the
// input, runs the FFT in shared memory (Stockham autosort, radix 8 then 4/2,
// XOR-swizzled buffer: every stage's reads and writes are bank-conflict free)
// and writes each frequency p as a BG * 8-byte run of row perm[t * n_p + p].
// The inverse kernel is the mirror: gather rows [s'][b], inverse FFT, scale
// by 1/n_p and write the caller's real pairs (or complex slices).
// Twiddles come from a per-plan table computed in double on the host.
#include "sptb_internal.cuh"
#include "sptb_fftcore.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <vector>

#ifndef SPTB_FFT_CARVEOUT
#define SPTB_FFT_CARVEOUT -1
#endif

namespace sptb {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder();  // sptb_patch.cu

namespace {

using namespace fftcore;

constexpr int FT = 256;   // threads per CTA
constexpr int FBG = 4;    // batch columns per CTA (32-byte output runs)

__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 3) & 15); }

// One in-place Stockham stage (sub-transform length Ns = 2^LNS, radix 2^LR)
// of FBG transforms of length N = 2^LOGN held in buf[b * N + swz(i)], then the
// remaining stages.  tw[k] = exp(-2 pi i k / N).
template <int LOGN, int LNS, bool INV>
__device__ __forceinline__ void fft_stage(float2* buf, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, NS = 1 << LNS;
    constexpr int LR = (LOGN - LNS) >= 3 ? 3 : (LOGN - LNS);
    constexpr int R = 1 << LR, NBF = N >> LR;
    constexpr int NB = (NBF * FBG + FT - 1) / FT;  // butterflies per thread
    float2 v[NB][R];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        const int g = threadIdx.x + q * FT;
        if (g < NBF * FBG) {
            const int b = g / NBF, j = g - b * NBF;
            const float2* src = buf + b * N;
            const int ts = (j & (NS - 1)) * (N / (NS * R));  // twiddle step
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 x = src[swz(j + r * NBF)];
                if (NS > 1 && r > 0) {
                    float2 w = __ldg(tw + ((r * ts) & (N - 1)));
                    if (INV) w.y = -w.y;
                    x = cmul(x, w);
                }
                v[q][r] = x;
            }
            if constexpr (LR == 3) dft8<INV>(v[q]);
            else if constexpr (LR == 2) dft4<INV>(v[q]);
            else dft2<INV>(v[q]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        const int g = threadIdx.x + q * FT;
        if (g < NBF * FBG) {
            const int b = g / NBF, j = g - b * NBF;
            float2* dst = buf + b * N;
            const int k = j & (NS - 1);
            const int o = (j - k) * R + k;
#pragma unroll
            for (int r = 0; r < R; ++r) dst[swz(o + r * NS)] = v[q][r];
        }
    }
    __syncthreads();
    if constexpr (LNS + LR < LOGN) fft_stage<LOGN, LNS + LR, INV>(buf, tw);
}

template <int LOGN, bool INV>
__device__ __forceinline__ void fft_smem(float2* buf, const float2* __restrict__ tw) {
    fft_stage<LOGN, 0, INV>(buf, tw);
}

// caller slices -> FFT along p -> q[perm[t * N + p]][b]
template <int LOGN>
__global__ void __launch_bounds__(FT, 3)
k_fft1_fwd(const float* __restrict__ in, int cplx, long long n, long long u0, int nb, int T,
           const int* __restrict__ perm, const float2* __restrict__ tw, float2* __restrict__ q, int B) {
    constexpr int N = 1 << LOGN;
    extern __shared__ __align__(16) float2 fbuf[];
    const int t = blockIdx.y, b0 = blockIdx.x * FBG;  // batch groups of one angle run back to back
    const long long plane = (long long)T * N;
    // all loads of the CTA in flight before the first shared-memory store
    constexpr int PER = (N + FT - 1) / FT;
    float2 z[FBG][PER];
#pragma unroll
    for (int b = 0; b < FBG; ++b) {
        const long long u = u0 + b0 + b;
        const float* pa = nullptr;
        const float* pb = nullptr;
        if (b0 + b < nb) {
            if (cplx) {
                pa = in + (u * plane + (long long)t * N) * 2;
            } else {
                pa = in + (2 * u) * plane + (long long)t * N;
                pb = (2 * u + 1 < n) ? in + (2 * u + 1) * plane + (long long)t * N : nullptr;
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = threadIdx.x + k * FT;
            z[b][k] = make_float2(0.f, 0.f);
            if (pa && i < N) {
                if (cplx) {
                    z[b][k] = __ldg(reinterpret_cast<const float2*>(pa) + i);
                } else {
                    z[b][k].x = __ldg(pa + i);
                    if (pb) z[b][k].y = __ldg(pb + i);
                }
            }
        }
    }
#pragma unroll
    for (int b = 0; b < FBG; ++b)
#pragma unroll
        for (int k = 0; k < PER; ++k)
            if (threadIdx.x + k * FT < N) fbuf[b * N + swz(threadIdx.x + k * FT)] = z[b][k];
    __syncthreads();
    fft_smem<LOGN, false>(fbuf, tw);
    const int* pr = perm ? perm + (long long)t * N : nullptr;
    for (int i = threadIdx.x; i < N; i += FT) {
        float2* dst = q + (size_t)(pr ? __ldg(pr + i) : t * N + i) * B + b0;
        const int si = swz(i);
        const float4 lo = make_float4(fbuf[si].x, fbuf[si].y, fbuf[N + si].x, fbuf[N + si].y);
        const float4 hi = make_float4(fbuf[2 * N + si].x, fbuf[2 * N + si].y, fbuf[3 * N + si].x, fbuf[3 * N + si].y);
        reinterpret_cast<float4*>(dst)[0] = lo;
        reinterpret_cast<float4*>(dst)[1] = hi;
    }
}

// q[perm[t * N + p]][b] -> inverse FFT along p, * scale -> caller slices
template <int LOGN>
__global__ void __launch_bounds__(FT, 3)
k_fft1_inv(const float2* __restrict__ q, int B, const int* __restrict__ perm, const float2* __restrict__ tw,
           float scale, float* __restrict__ out, int cplx, long long n, long long u0, int nb, int T) {
    constexpr int N = 1 << LOGN;
    extern __shared__ __align__(16) float2 fbuf[];
    const int t = blockIdx.y, b0 = blockIdx.x * FBG;  // batch groups of one angle run back to back
    const int* pr = perm + (long long)t * N;
    for (int i = threadIdx.x; i < N; i += FT) {
        const float4* src = reinterpret_cast<const float4*>(q + (size_t)__ldg(pr + i) * B + b0);
        const float4 lo = __ldg(src), hi = __ldg(src + 1);
        const int si = swz(i);
        fbuf[si] = make_float2(lo.x, lo.y);
        fbuf[N + si] = make_float2(lo.z, lo.w);
        fbuf[2 * N + si] = make_float2(hi.x, hi.y);
        fbuf[3 * N + si] = make_float2(hi.z, hi.w);
    }
    __syncthreads();
    fft_smem<LOGN, true>(fbuf, tw);
    const long long plane = (long long)T * N;
    for (int b = 0; b < FBG; ++b) {
        if (b0 + b >= nb) break;
        const long long u = u0 + b0 + b;
        float* pa;
        float* pb = nullptr;
        if (cplx) {
            pa = out + (u * plane + (long long)t * N) * 2;
        } else {
            pa = out + (2 * u) * plane + (long long)t * N;
            if (2 * u + 1 < n) pb = out + (2 * u + 1) * plane + (long long)t * N;
        }
        for (int i = threadIdx.x; i < N; i += FT) {
            const float2 z = fbuf[b * N + swz(i)];
            if (cplx) {
                reinterpret_cast<float2*>(pa)[i] = make_float2(z.x * scale, z.y * scale);
            } else {
                pa[i] = z.x * scale;
                if (pb) pb[i] = z.y * scale;
            }
        }
    }
}

// caller slices -> FFT along p -> q[perm[t * N + p]][b]; BG transforms per CTA
// (BG batch columns: each frequency leaves as one 8 BG-byte run)
// mbarrier wait and 1-D bulk copies (cp.async.bulk) shared by the kernels below
__device__ __forceinline__ void fbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "FW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra FW;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
                 "r"((unsigned)__cvta_generic_to_shared(src)), "r"(bytes)
                 : "memory");
}

template <int LOGN, int BG, bool BULK = false>
__global__ void __launch_bounds__(BG * (1 << LOGN) / 16, 1024 / (BG * (1 << LOGN) / 16))
k_fft1r_fwd(const float* __restrict__ in, int cplx, long long n, long long u0, int nb, int T,
            const int* __restrict__ perm, const float2* __restrict__ tw, float2* __restrict__ q, int B) {
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3;
    extern __shared__ __align__(16) float2 fbuf[];
    const int t = blockIdx.y, b0 = blockIdx.x * BG;
    const int b = threadIdx.x / TP, j = threadIdx.x % TP;
    float2* buf = fbuf + b * N;
    const long long plane = (long long)T * N;
    const long long u = u0 + b0 + b;
    float2 v[16];
    if constexpr (BULK) {
        // real pairs: the CTA's 2 BG rows (slices 2u, 2u + 1 at angle t) land in
        // the exchange buffer by bulk copies (the per-lane scalar loads were
        // LSU-throttled); slice 2(b0 + b) + h row at fbuf floats [(2 b + h) N]
        float* raw = reinterpret_cast<float*>(fbuf);
        __shared__ __align__(8) unsigned long long bar;
        const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb));
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            unsigned bytes = 0;
            for (int k = 0; k < 2 * BG; ++k) {
                const long long sl = 2 * (u0 + b0) + k;
                if (b0 + k / 2 < nb && sl < n) bytes += N * 4u;
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb), "r"(bytes) : "memory");
            for (int k = 0; k < 2 * BG; ++k) {
                const long long sl = 2 * (u0 + b0) + k;
                if (b0 + k / 2 < nb && sl < n) bulk_g2s(raw + k * N, in + sl * plane + (long long)t * N, N * 4u, sb);
            }
        }
        __syncthreads();
        fbar_wait(sb, 0);
        const bool ha = b0 + b < nb, hb = ha && 2 * u + 1 < n;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int i = j + TP * r;
            v[r] = make_float2(ha ? raw[2 * b * N + i] : 0.f, hb ? raw[(2 * b + 1) * N + i] : 0.f);
        }
        __syncthreads();  // staged rows consumed before the exchange overwrites them
    } else {
        const float* pa = nullptr;
        const float* pb = nullptr;
        if (b0 + b < nb) {
            if (cplx) {
                pa = in + (u * plane + (long long)t * N) * 2;
            } else {
                pa = in + (2 * u) * plane + (long long)t * N;
                pb = (2 * u + 1 < n) ? in + (2 * u + 1) * plane + (long long)t * N : nullptr;
            }
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int i = j + TP * r;
            float2 z = make_float2(0.f, 0.f);
            if (pa) {
                if (cplx) z = __ldg(reinterpret_cast<const float2*>(pa) + i);
                else {
                    z.x = __ldg(pa + i);
                    if (pb) z.y = __ldg(pb + i);
                }
            }
            v[r] = z;
        }
    }
    dft16<false>(v);
    fft16_stages<LOGN, false>(v, buf, j, tw);
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NB3; ++c)
#pragma unroll
        for (int r = 0; r < R3; ++r) buf[swz4(j + c * TP + 256 * r)] = v[c * R3 + r];
    __syncthreads();
    const int* pr = perm ? perm + (long long)t * N : nullptr;
    constexpr int NI = N / (BG * TP);  // = 4: all row indices loaded before any store
    int rowi[NI];
#pragma unroll
    for (int k = 0; k < NI; ++k) {
        const int i = threadIdx.x + k * BG * TP;
        rowi[k] = perm ? __ldg(pr + i) : t * N + i;  // no perm: sample order (S with original columns)
    }
#pragma unroll
    for (int k = 0; k < NI; ++k) {
        const int i = threadIdx.x + k * BG * TP;
        float4* dst = reinterpret_cast<float4*>(q + (size_t)rowi[k] * B + b0);
        const int si = swz4(i);
#pragma unroll
        for (int h = 0; h < BG / 2; ++h)
            dst[h] = make_float4(fbuf[2 * h * N + si].x, fbuf[2 * h * N + si].y, fbuf[(2 * h + 1) * N + si].x,
                                 fbuf[(2 * h + 1) * N + si].y);
    }
}

// ---------------------------------------------------------------------------
// 2-D inverse FFT of the gridded batch G [b][y][x] (after S) fused with the
// deapodization and the unpack to the caller's real slice pairs.  cuFFT's
// 2-D plan makes two passes (strided y, contiguous x) and the unpack a third;
// here the y pass runs in place and the x pass writes the caller's slices:
//   k_fft2_col: a CTA owns CW = 4 adjacent columns of one plane; lane
//     (c, j) = (tid % CW, tid / CW) loads rows j + TP r of column c, so each
//     warp load is 8 rows x 32 contiguous bytes; the radix-16 register FFT
//     exchanges through a per-column buffer of stride N + 4 (the XOR swizzle
//     keeps 4 consecutive j in an aligned block of 4 slots, the +4 stride
//     moves the 4 columns onto disjoint blocks: conflict-free); outputs land
//     in the same (j + TP q) rows, written straight back.
//   k_fft2_row: RB rows per CTA, inverse FFT along x, times deapo(y, x) *
//     scale, real part to slice 2u and imaginary part to slice 2u + 1.
// ---------------------------------------------------------------------------
#ifndef SPTB_FFT2_CW
#define SPTB_FFT2_CW 4
#endif
constexpr int CW2 = SPTB_FFT2_CW;  // columns per CTA in the y pass
constexpr int RB2 = 4;             // rows per CTA in the x pass

template <int LOGN, bool INV>
__global__ void __launch_bounds__(CW2 * (1 << LOGN) / 16, 1024 / (CW2 * (1 << LOGN) / 16))
k_fft2_col(float2* __restrict__ g, int X, long long M, int strips, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3, LD = N + 16 / CW2;
    extern __shared__ __align__(16) float2 fbuf[];
    // column base recomputed after the FFT (keeps it out of the register budget)
    auto colp = [&]() {
        const int c = threadIdx.x % CW2, j = threadIdx.x / CW2;
        const int b = blockIdx.x / strips, x0 = (blockIdx.x - b * strips) * CW2;
        return g + (size_t)b * M + (size_t)j * X + x0 + c;
    };
    const int step = TP * X;  // rows j + TP r, r = 0..15 (< 2^24 elements)
    float2 v[16];
    {
        const float2* pp = colp();
#pragma unroll
        for (int r = 0; r < 16; ++r, pp += step) v[r] = *pp;
    }
    dft16<INV>(v);
    fft16_stages<LOGN, INV>(v, fbuf + (threadIdx.x % CW2) * LD, threadIdx.x / CW2, tw);
    // output j + TP q + 256 r = j + TP (q + NB3 r) sits in v[q R3 + r]; the
    // base goes through an opaque move so the compiler recomputes the 16 row
    // addresses instead of keeping the load addresses live (it spilled them)
    float2* pp = colp();
    asm volatile("mov.b64 %0, %0;" : "+l"(pp));
#pragma unroll
    for (int m = 0; m < 16; ++m, pp += step) *pp = v[(m % NB3) * R3 + m / NB3];
}

template <int LOGN>
__global__ void __launch_bounds__(RB2 * (1 << LOGN) / 16, 1024 / (RB2 * (1 << LOGN) / 16))
k_fft2_row_unpack(const float2* __restrict__ g, long long M, int Y, const float* __restrict__ plane, float scale,
                  float* __restrict__ out, long long n, long long u0, int nb, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3;
    extern __shared__ __align__(16) float2 fbuf[];
    const int rb = threadIdx.x / TP, j = threadIdx.x % TP;
    const long long gr = (long long)blockIdx.x * RB2 + rb;  // b * Y + y
    const int b = (int)(gr / Y), y = (int)(gr - (long long)b * Y);
    const float2* row = g + (size_t)b * M + (size_t)y * N;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = __ldcs(row + j + TP * r);
    dft16<true>(v);
    fft16_stages<LOGN, true>(v, fbuf + rb * N, j, tw);
    if (b >= nb) return;
    const long long u = u0 + b;
    float* pa = out + (size_t)(2 * u) * M + (size_t)y * N;
    float* pb = (2 * u + 1 < n) ? out + (size_t)(2 * u + 1) * M + (size_t)y * N : nullptr;
    const float* pl = plane ? plane + (size_t)y * N : nullptr;
#pragma unroll
    for (int q = 0; q < NB3; ++q)
#pragma unroll
        for (int r = 0; r < R3; ++r) {
            const int x = j + TP * q + 256 * r;
            const float f = pl ? __ldg(pl + x) * scale : scale;
            const float2 z = v[q * R3 + r];
            __stcs(pa + x, z.x * f);
            if (pb) __stcs(pb + x, z.y * f);
        }
}

// y pass with the strip staged by TMA: N / 256 boxes of 256 rows x CW2
// columns land in [row][c] order on one mbarrier (no per-lane loads: the LSU
// queue throttled the LDG version), L2 promotion 256 B so the neighbouring
// strips' sectors come from the same DRAM bursts

#ifndef SPTB_FFT2_TSTORE
#define SPTB_FFT2_TSTORE 1
#endif
template <int LOGN, bool INV, bool TSTORE = SPTB_FFT2_TSTORE>
__global__ void __launch_bounds__(CW2 * (1 << LOGN) / 16, 1024 / (CW2 * (1 << LOGN) / 16))
k_fft2_col_tma(const __grid_constant__ CUtensorMap tmap, float2* __restrict__ g, int X, long long M, int strips,
               const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, LD = N + 16 / CW2, R3 = N / 256, NB3 = 16 / R3;
    // own name: an extern array shares the alignment of its first declaration
    // (16 for fbuf) and the TMA destination needs 128
    extern __shared__ __align__(128) unsigned char colbuf_raw[];
    float2* fbuf = reinterpret_cast<float2*>(colbuf_raw);
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        const int b = blockIdx.x / strips, x0 = (blockIdx.x - b * strips) * CW2;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb),
                     "r"((unsigned)(N * CW2 * sizeof(float2))) : "memory");
#pragma unroll 1
        for (int k = 0; k < N / 256; ++k)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(fbuf + k * 256 * CW2)),
                "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(x0), "r"(256 * k), "r"(b), "r"(sb)
                : "memory");
    }
    __syncthreads();
    fbar_wait(sb, 0);
    const int c = threadIdx.x % CW2, j = threadIdx.x / CW2;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = fbuf[(j + TP * r) * CW2 + c];
    __syncthreads();  // staged strip consumed before the exchange buffers overwrite it
    dft16<INV>(v);
    fft16_stages<LOGN, INV>(v, fbuf + c * LD, j, tw);
    if constexpr (TSTORE) {
        // the strip leaves the way it came: [row][c] in shared memory, N / 256 TMA stores
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 16; ++m) fbuf[(j + TP * m) * CW2 + c] = v[(m % NB3) * R3 + m / NB3];
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const int b = blockIdx.x / strips, x0 = (blockIdx.x - b * strips) * CW2;
#pragma unroll 1
            for (int k = 0; k < N / 256; ++k)
                asm volatile(
                    "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                        reinterpret_cast<unsigned long long>(&tmap)),
                    "r"(x0), "r"(256 * k), "r"(b), "r"((unsigned)__cvta_generic_to_shared(fbuf + k * 256 * CW2))
                    : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        }
    } else {
        float2* pp;
        {
            const int b = blockIdx.x / strips, x0 = (blockIdx.x - b * strips) * CW2;
            pp = g + (size_t)b * M + (size_t)j * X + x0 + c;
        }
        const int step = TP * X;
#pragma unroll
        for (int m = 0; m < 16; ++m, pp += step) *pp = v[(m % NB3) * R3 + m / NB3];
    }
}

// Persistent y pass: one 512-thread CTA per SM walks strips blockIdx.x,
// + gridDim.x, ... with three strip buffers: while strip k is transformed in
// buffer k % 3, strip k + 1 is already loading into the next buffer and
// strip k - 1's TMA store drains from the previous one (ncu: the per-strip
// kernel spent ~50% of its warps' time waiting for its own load).
constexpr int COLP_BUFS = 3;
template <int LOGN, bool INV>
__global__ void __launch_bounds__(CW2 * (1 << LOGN) / 16, 1)
k_fft2_col_pers(const __grid_constant__ CUtensorMap tmap, int strips, int nstrip, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, LD = N + 16 / CW2, R3 = N / 256, NB3 = 16 / R3;
    constexpr int BUF = CW2 * LD;  // float2 per buffer (>= N * CW2 staging)
    extern __shared__ __align__(128) unsigned char colpbuf_raw[];
    float2* base = reinterpret_cast<float2*>(colpbuf_raw);
    __shared__ __align__(8) unsigned long long bar[COLP_BUFS];
    const int c = threadIdx.x % CW2, j = threadIdx.x / CW2;
    auto load = [&](int s, int k) {  // tid 0: strip s into buffer k % 3
        const int b = s / strips, x0 = (s - b * strips) * CW2;
        const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar[k % COLP_BUFS]);
        float2* dst = base + (k % COLP_BUFS) * BUF;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb),
                     "r"((unsigned)(N * CW2 * sizeof(float2))) : "memory");
#pragma unroll 1
        for (int q = 0; q < N / 256; ++q)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst + q * 256 * CW2)),
                "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(x0), "r"(256 * q), "r"(b), "r"(sb)
                : "memory");
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < COLP_BUFS; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if ((int)blockIdx.x < nstrip) load(blockIdx.x, 0);
    }
    __syncthreads();
    const StageTwiddles<LOGN, INV> stw(tw, threadIdx.x / CW2);
    int k = 0;
    for (int s = blockIdx.x; s < nstrip; s += gridDim.x, ++k) {
        float2* fbuf = base + (k % COLP_BUFS) * BUF;
        if (threadIdx.x == 0 && s + (int)gridDim.x < nstrip) {
            // buffer (k + 1) % 3 last held strip k - 2: its store must have been read out
            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            load(s + gridDim.x, k + 1);
        }
        fbar_wait((unsigned)__cvta_generic_to_shared(&bar[k % COLP_BUFS]), (unsigned)((k / COLP_BUFS) & 1));
        float2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = fbuf[(j + TP * r) * CW2 + c];
        __syncthreads();
        dft16<INV>(v);
        fft16_stages_pre<LOGN, INV>(v, fbuf + c * LD, j, stw);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 16; ++m) fbuf[(j + TP * m) * CW2 + c] = v[(m % NB3) * R3 + m / NB3];
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const int b = s / strips, x0 = (s - b * strips) * CW2;
#pragma unroll 1
            for (int q = 0; q < N / 256; ++q)
                asm volatile(
                    "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                        reinterpret_cast<unsigned long long>(&tmap)),
                    "r"(x0), "r"(256 * q), "r"(b), "r"((unsigned)__cvta_generic_to_shared(fbuf + q * 256 * CW2))
                    : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// Inverse FFT1 for radon with S^H rows in sample order: for angle t the P
// rows t P + p of Q [s][b] are a P x B matrix whose columns are the batch
// units, i.e. the y pass again with plane = angle and X = B.  N/256 TMA boxes
// (4 columns x 256 rows) in, the column FFT, then the two real rows of each
// unit (slices 2u, 2u + 1 at angle t, scaled by 1/P) leave by bulk stores from
// a [2 c + h][P + 4] staging area (the +4 row pad spreads the 4 columns over
// distinct banks).
template <int LOGN>
__global__ void __launch_bounds__(CW2 * (1 << LOGN) / 16, 1024 / (CW2 * (1 << LOGN) / 16))
k_fft1_inv_col(const __grid_constant__ CUtensorMap tmap, int T, float scale, float* __restrict__ out, long long n,
               long long u0, int nb, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, LD = N + 16 / CW2, R3 = N / 256, NB3 = 16 / R3, RS = N + 4;
    extern __shared__ __align__(128) unsigned char colbuf_raw[];
    float2* fbuf = reinterpret_cast<float2*>(colbuf_raw);
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    const int b0 = blockIdx.x * CW2, t = blockIdx.y;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb),
                     "r"((unsigned)(N * CW2 * sizeof(float2))) : "memory");
#pragma unroll 1
        for (int k = 0; k < N / 256; ++k)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];\n" ::"r"((unsigned)__cvta_generic_to_shared(fbuf + k * 256 * CW2)),
                "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(b0), "r"(t * N + 256 * k), "r"(sb)
                : "memory");
    }
    __syncthreads();
    fbar_wait(sb, 0);
    const int c = threadIdx.x % CW2, j = threadIdx.x / CW2;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = fbuf[(j + TP * r) * CW2 + c];
    __syncthreads();
    dft16<true>(v);
    fft16_stages<LOGN, true>(v, fbuf + c * LD, j, tw);
    __syncthreads();
    float* stg = reinterpret_cast<float*>(fbuf);  // [2 CW2][RS]
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const int pidx = j + TP * m;
        const float2 z = v[(m % NB3) * R3 + m / NB3];
        stg[(2 * c) * RS + pidx] = z.x * scale;
        stg[(2 * c + 1) * RS + pidx] = z.y * scale;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const long long plane = (long long)T * N;
        for (int cc = 0; cc < CW2; ++cc) {
            if (b0 + cc >= nb) break;
            const long long u = u0 + b0 + cc;
            bulk_s2g(out + (2 * u) * plane + (long long)t * N, stg + (2 * cc) * RS, N * 4u);
            if (2 * u + 1 < n) bulk_s2g(out + (2 * u + 1) * plane + (long long)t * N, stg + (2 * cc + 1) * RS, N * 4u);
        }
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
}

// Forward FFT1 for gridrec as a column pass: for angle t, the 2 CW2 real rows
// (slices 2u, 2u + 1 of units b0..b0+3) come in by bulk copies into a
// [2 c + h][P + 4] staging area, lane (c, j) runs the column FFT of unit
// b0 + c, and Q rows t P + p (sample order) leave as N/256 TMA boxes of
// 4 columns x 256 rows from [p][c] staging (the per-row 32-byte STG runs of
// k_fft1r_fwd were its bottleneck).
template <int LOGN>
__global__ void __launch_bounds__(CW2 * (1 << LOGN) / 16, 1024 / (CW2 * (1 << LOGN) / 16))
k_fft1_fwd_col(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ in, int T, long long n,
               long long u0, int nb, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, LD = N + 16 / CW2, R3 = N / 256, NB3 = 16 / R3, RS = N + 4;
    extern __shared__ __align__(128) unsigned char colbuf_raw[];
    float2* fbuf = reinterpret_cast<float2*>(colbuf_raw);
    float* stg = reinterpret_cast<float*>(fbuf);  // [2 CW2][RS]
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    const int b0 = blockIdx.x * CW2, t = blockIdx.y;
    const long long plane = (long long)T * N;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        unsigned bytes = 0;
        for (int k = 0; k < 2 * CW2; ++k)
            if (b0 + k / 2 < nb && 2 * (u0 + b0) + k < n) bytes += N * 4u;
        if (bytes) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb), "r"(bytes) : "memory");
            for (int k = 0; k < 2 * CW2; ++k) {
                const long long sl = 2 * (u0 + b0) + k;
                if (b0 + k / 2 < nb && sl < n) bulk_g2s(stg + k * RS, in + sl * plane + (long long)t * N, N * 4u, sb);
            }
        }
    }
    __syncthreads();
    if (b0 < nb) fbar_wait(sb, 0);  // some row was requested iff unit b0 is valid
    const int c = threadIdx.x % CW2, j = threadIdx.x / CW2;
    const long long u = u0 + b0 + c;
    const bool ha = b0 + c < nb, hb = ha && 2 * u + 1 < n;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int i = j + TP * r;
        v[r] = make_float2(ha ? stg[(2 * c) * RS + i] : 0.f, hb ? stg[(2 * c + 1) * RS + i] : 0.f);
    }
    __syncthreads();
    dft16<false>(v);
    fft16_stages<LOGN, false>(v, fbuf + c * LD, j, tw);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; ++m) fbuf[(j + TP * m) * CW2 + c] = v[(m % NB3) * R3 + m / NB3];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll 1
        for (int k = 0; k < N / 256; ++k)
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                    reinterpret_cast<unsigned long long>(&tmap)),
                "r"(b0), "r"(t * N + 256 * k), "r"((unsigned)__cvta_generic_to_shared(fbuf + k * 256 * CW2))
                : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
}

// Persistent version of k_fft1_fwd_col (same triple-buffer scheme as
// k_fft2_col_pers): strip s = (angle t, unit group bg), bg fastest.
template <int LOGN>
__global__ void __launch_bounds__(CW2 * (1 << LOGN) / 16, 1)
k_fft1_fwd_pers(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ in, int T, int ngrp,
                long long n, long long u0, int nb, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, LD = N + 16 / CW2, R3 = N / 256, NB3 = 16 / R3, RS = N + 4;
    constexpr int BUF = CW2 * LD;
    extern __shared__ __align__(128) unsigned char colpbuf_raw[];
    float2* base = reinterpret_cast<float2*>(colpbuf_raw);
    __shared__ __align__(8) unsigned long long bar[COLP_BUFS];
    const long long plane = (long long)T * N;
    const int nstrip = ngrp * T;
    const int c = threadIdx.x % CW2, j = threadIdx.x / CW2;
    auto load = [&](int s, int k) {  // tid 0: rows of strip s into buffer k % 3 (only valid units)
        const int bg = s % ngrp, t = s / ngrp, b0 = bg * CW2;
        float* stg = reinterpret_cast<float*>(base + (k % COLP_BUFS) * BUF);
        const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar[k % COLP_BUFS]);
        if (b0 >= nb) {  // nothing to load: still complete the phase (parity is counted per use)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sb) : "memory");
            return;
        }
        unsigned bytes = 0;
        for (int q = 0; q < 2 * CW2; ++q)
            if (b0 + q / 2 < nb && 2 * (u0 + b0) + q < n) bytes += N * 4u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb), "r"(bytes) : "memory");
        for (int q = 0; q < 2 * CW2; ++q) {
            const long long sl = 2 * (u0 + b0) + q;
            if (b0 + q / 2 < nb && sl < n) bulk_g2s(stg + q * RS, in + sl * plane + (long long)t * N, N * 4u, sb);
        }
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < COLP_BUFS; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if ((int)blockIdx.x < nstrip) load(blockIdx.x, 0);
    }
    __syncthreads();
    const StageTwiddles<LOGN, false> stw(tw, threadIdx.x / CW2);
    int k = 0;
    for (int s = blockIdx.x; s < nstrip; s += gridDim.x, ++k) {
        float2* fbuf = base + (k % COLP_BUFS) * BUF;
        float* stg = reinterpret_cast<float*>(fbuf);
        const int bg = s % ngrp, t = s / ngrp, b0 = bg * CW2;
        if (threadIdx.x == 0 && s + (int)gridDim.x < nstrip) {
            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            load(s + gridDim.x, k + 1);
        }
        fbar_wait((unsigned)__cvta_generic_to_shared(&bar[k % COLP_BUFS]), (unsigned)((k / COLP_BUFS) & 1));
        const long long u = u0 + b0 + c;
        const bool ha = b0 + c < nb, hb = ha && 2 * u + 1 < n;
        float2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int i = j + TP * r;
            v[r] = make_float2(ha ? stg[(2 * c) * RS + i] : 0.f, hb ? stg[(2 * c + 1) * RS + i] : 0.f);
        }
        __syncthreads();
        dft16<false>(v);
        fft16_stages_pre<LOGN, false>(v, fbuf + c * LD, j, stw);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 16; ++m) fbuf[(j + TP * m) * CW2 + c] = v[(m % NB3) * R3 + m / NB3];
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll 1
            for (int q = 0; q < N / 256; ++q)
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                        reinterpret_cast<unsigned long long>(&tmap)),
                    "r"(b0), "r"(t * N + 256 * q), "r"((unsigned)__cvta_generic_to_shared(fbuf + q * 256 * CW2))
                    : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// radon side: caller real pairs (slices 2u, 2u + 1) times deapo(y, x) ->
// forward FFT along x -> G row (planes b >= nb are zero-filled: the S^H
// kernel reads all B planes)
template <int LOGN>
__global__ void __launch_bounds__(RB2 * (1 << LOGN) / 16, 1024 / (RB2 * (1 << LOGN) / 16))
k_fft2_row_pack(const float* __restrict__ in, long long M, int Y, const float* __restrict__ plane, long long n,
                long long u0, int nb, float2* __restrict__ g, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3;
    extern __shared__ __align__(16) float2 fbuf[];
    const int rb = threadIdx.x / TP, j = threadIdx.x % TP;
    const long long gr = (long long)blockIdx.x * RB2 + rb;  // b * Y + y
    const int b = (int)(gr / Y), y = (int)(gr - (long long)b * Y);
    const long long u = u0 + b;
    const float* pa = b < nb ? in + (size_t)(2 * u) * M + (size_t)y * N : nullptr;
    const float* pb = (b < nb && 2 * u + 1 < n) ? in + (size_t)(2 * u + 1) * M + (size_t)y * N : nullptr;
    const float* pl = plane ? plane + (size_t)y * N : nullptr;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int x = j + TP * r;
        const float d = pl ? __ldg(pl + x) : 1.f;
        v[r] = make_float2(pa ? __ldcs(pa + x) * d : 0.f, pb ? __ldcs(pb + x) * d : 0.f);
    }
    dft16<false>(v);
    fft16_stages<LOGN, false>(v, fbuf + rb * N, j, tw);
    float2* row = g + (size_t)b * M + (size_t)y * N;
#pragma unroll
    for (int q = 0; q < NB3; ++q)
#pragma unroll
        for (int r = 0; r < R3; ++r) row[j + TP * q + 256 * r] = v[q * R3 + r];
}

// Bulk-copy versions of the two row kernels: the RB2 rows of a CTA are
// contiguous (Y % RB2 == 0), so the input, the deapodization rows and the
// output each move as one cp.async.bulk per CTA (no per-lane global loads or
// scalar stores; the LDG/STG versions were LSU-bound).
// deapodization weight of row y from the separable factors (build_deapo):
// [dx^2 + dy^2 < r^2] * fx[x] * fy[y] * scale, r = min(X, Y) / 2; dxy == nullptr: scale
struct Deapo {
    const float* fx;
    float fy, s;
    int dy2, r2, hx;
    // fx_s: shared copy of the X factors (nullptr when dxy is)
    __device__ __forceinline__ Deapo(const float* dxy, const float* fx_s, int X, int Y, int y, float scale)
        : fx(dxy ? fx_s : nullptr), s(scale) {
        hx = X / 2;
        const int dy = y - Y / 2, r = min(X, Y) / 2;
        dy2 = dy * dy;
        r2 = r * r;
        fy = dxy ? __ldg(dxy + X + y) * scale : scale;
    }
    __device__ __forceinline__ float operator()(int x) const {
        if (!fx) return s;
        const int dx = x - hx;
        return dx * dx + dy2 < r2 ? fx[x] * fy : 0.f;
    }
};


template <int LOGN>
__global__ void __launch_bounds__(RB2 * (1 << LOGN) / 16, 1024 / (RB2 * (1 << LOGN) / 16))
k_fft2_row_unpack_b(const float2* __restrict__ g, long long M, int Y, const float* __restrict__ dxy, float scale,
                    float* __restrict__ out, long long n, long long u0, int nb, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3;
    extern __shared__ __align__(128) unsigned char rowbuf_raw[];
    float2* fbuf = reinterpret_cast<float2*>(rowbuf_raw);  // [RB2][N]
    float* fxs = reinterpret_cast<float*>(fbuf + RB2 * N);  // [N] x factors of the deapodization
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    const long long gr0 = (long long)blockIdx.x * RB2;
    const int b = (int)(gr0 / Y), y0 = (int)(gr0 - (long long)b * Y);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb),
                     "r"(RB2 * N * 8u + (dxy ? N * 4u : 0u))
                     : "memory");
        bulk_g2s(fbuf, g + (size_t)b * M + (size_t)y0 * N, RB2 * N * 8u, sb);
        if (dxy) bulk_g2s(fxs, dxy, N * 4u, sb);
    }
    __syncthreads();
    fbar_wait(sb, 0);
    const int rb = threadIdx.x / TP, j = threadIdx.x % TP;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = fbuf[rb * N + j + TP * r];
    __syncthreads();
    dft16<true>(v);
    fft16_stages<LOGN, true>(v, fbuf + rb * N, j, tw);
    if (b >= nb) return;  // uniform over the CTA
    __syncthreads();
    float* sa = reinterpret_cast<float*>(fbuf);  // [RB2][N] real parts, then [RB2][N] imaginary parts
    float* sbm = sa + RB2 * N;
    const Deapo dp(dxy, fxs, N, Y, y0 + rb, scale);
#pragma unroll
    for (int q = 0; q < NB3; ++q)
#pragma unroll
        for (int r = 0; r < R3; ++r) {
            const int x = j + TP * q + 256 * r;
            const float f = dp(x);
            const float2 z = v[q * R3 + r];
            sa[rb * N + x] = z.x * f;
            sbm[rb * N + x] = z.y * f;
        }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const long long u = u0 + b;
        bulk_s2g(out + (size_t)(2 * u) * M + (size_t)y0 * N, sa, RB2 * N * 4u);
        if (2 * u + 1 < n) bulk_s2g(out + (size_t)(2 * u + 1) * M + (size_t)y0 * N, sbm, RB2 * N * 4u);
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
}

template <int LOGN>
__global__ void __launch_bounds__(RB2 * (1 << LOGN) / 16, 1024 / (RB2 * (1 << LOGN) / 16))
k_fft2_row_pack_b(const float* __restrict__ in, long long M, int Y, const float* __restrict__ dxy, long long n,
                  long long u0, int nb, float2* __restrict__ g, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3;
    extern __shared__ __align__(128) unsigned char rowbuf_raw[];
    float2* fbuf = reinterpret_cast<float2*>(rowbuf_raw);
    float* sa = reinterpret_cast<float*>(fbuf);   // [RB2][N] slice 2u rows
    float* sbm = sa + RB2 * N;                    // [RB2][N] slice 2u + 1 rows
    float* fxs = reinterpret_cast<float*>(fbuf + RB2 * N);  // [N] x factors of the deapodization
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    const long long gr0 = (long long)blockIdx.x * RB2;
    const int b = (int)(gr0 / Y), y0 = (int)(gr0 - (long long)b * Y);
    const long long u = u0 + b;
    const bool ha = b < nb, hb = b < nb && 2 * u + 1 < n;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        const unsigned bytes = (ha ? RB2 * N * 4u : 0u) + (hb ? RB2 * N * 4u : 0u) + (ha && dxy ? N * 4u : 0u);
        if (bytes) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb), "r"(bytes) : "memory");
            if (ha) bulk_g2s(sa, in + (size_t)(2 * u) * M + (size_t)y0 * N, RB2 * N * 4u, sb);
            if (hb) bulk_g2s(sbm, in + (size_t)(2 * u + 1) * M + (size_t)y0 * N, RB2 * N * 4u, sb);
            if (ha && dxy) bulk_g2s(fxs, dxy, N * 4u, sb);
        }
    }
    __syncthreads();
    if (ha) fbar_wait(sb, 0);
    const int rb = threadIdx.x / TP, j = threadIdx.x % TP;
    float2 v[16];
    const Deapo dp(dxy, fxs, N, Y, y0 + rb, 1.f);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int x = j + TP * r;
        const float d = dp(x);
        v[r] = make_float2(ha ? sa[rb * N + x] * d : 0.f, hb ? sbm[rb * N + x] * d : 0.f);
    }
    __syncthreads();
    dft16<false>(v);
    fft16_stages<LOGN, false>(v, fbuf + rb * N, j, tw);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NB3; ++q)
#pragma unroll
        for (int r = 0; r < R3; ++r) fbuf[rb * N + j + TP * q + 256 * r] = v[q * R3 + r];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        bulk_s2g(g + (size_t)b * M + (size_t)y0 * N, fbuf, RB2 * N * 8u);
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
}

// in-place x pass (solver grids): RB2 contiguous rows in, FFT, back out
template <int LOGN, bool INV>
__global__ void __launch_bounds__(RB2 * (1 << LOGN) / 16, 1024 / (RB2 * (1 << LOGN) / 16))
k_fft2_row_b(float2* __restrict__ g, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3;
    extern __shared__ __align__(128) unsigned char rowbuf_raw[];
    float2* fbuf = reinterpret_cast<float2*>(rowbuf_raw);
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    float2* rows = g + (size_t)blockIdx.x * RB2 * N;  // planes are whole rows: row index b * Y + y
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb), "r"(RB2 * N * 8u)
                     : "memory");
        bulk_g2s(fbuf, rows, RB2 * N * 8u, sb);
    }
    __syncthreads();
    fbar_wait(sb, 0);
    const int rb = threadIdx.x / TP, j = threadIdx.x % TP;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = fbuf[rb * N + j + TP * r];
    __syncthreads();
    dft16<INV>(v);
    fft16_stages<LOGN, INV>(v, fbuf + rb * N, j, tw);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NB3; ++q)
#pragma unroll
        for (int r = 0; r < R3; ++r) fbuf[rb * N + j + TP * q + 256 * r] = v[q * R3 + r];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        bulk_s2g(rows, fbuf, RB2 * N * 8u);
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
}

// Persistent version of k_fft2_row_unpack_b: one 512-thread CTA per SM walks
// 4-row strips with three 64 KB buffers (next strip's bulk load and the
// previous strip's two bulk stores overlap the current FFT); the deapo x
// factors are staged once.
template <int LOGN>
__global__ void __launch_bounds__(RB2 * (1 << LOGN) / 16, 1)
k_fft2_row_unpack_pers(const float2* __restrict__ g, long long M, int Y, const float* __restrict__ dxy, float scale,
                       float* __restrict__ out, long long n, long long u0, int nstrip, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3, BUF = RB2 * N;
    extern __shared__ __align__(128) unsigned char rowpbuf_raw[];
    float2* base = reinterpret_cast<float2*>(rowpbuf_raw);
    float* fxs = reinterpret_cast<float*>(base + COLP_BUFS * BUF);
    __shared__ __align__(8) unsigned long long bar[COLP_BUFS + 1];
    auto load = [&](int s, int k) {
        const long long gr0 = (long long)s * RB2;
        const int b = (int)(gr0 / Y), y0 = (int)(gr0 - (long long)b * Y);
        const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar[k % COLP_BUFS]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb), "r"(BUF * 8u) : "memory");
        bulk_g2s(base + (k % COLP_BUFS) * BUF, g + (size_t)b * M + (size_t)y0 * N, BUF * 8u, sb);
    };
    const unsigned fb = (unsigned)__cvta_generic_to_shared(&bar[COLP_BUFS]);
    if (threadIdx.x == 0) {
        for (int i = 0; i <= COLP_BUFS; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if (dxy) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb), "r"(N * 4u) : "memory");
            bulk_g2s(fxs, dxy, N * 4u, fb);
        }
        if ((int)blockIdx.x < nstrip) load(blockIdx.x, 0);
    }
    __syncthreads();
    if (dxy) fbar_wait(fb, 0);
    const int rb = threadIdx.x / TP, j = threadIdx.x % TP;
    const StageTwiddles<LOGN, true> stw(tw, threadIdx.x % (N / 16));
    int k = 0;
    for (int s = blockIdx.x; s < nstrip; s += gridDim.x, ++k) {
        float2* fbuf = base + (k % COLP_BUFS) * BUF;
        const long long gr0 = (long long)s * RB2;
        const int b = (int)(gr0 / Y), y0 = (int)(gr0 - (long long)b * Y);
        if (threadIdx.x == 0 && s + (int)gridDim.x < nstrip) {
            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            load(s + gridDim.x, k + 1);
        }
        fbar_wait((unsigned)__cvta_generic_to_shared(&bar[k % COLP_BUFS]), (unsigned)((k / COLP_BUFS) & 1));
        float2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = fbuf[rb * N + j + TP * r];
        __syncthreads();
        dft16<true>(v);
        fft16_stages_pre<LOGN, true>(v, fbuf + rb * N, j, stw);
        __syncthreads();
        float* sa = reinterpret_cast<float*>(fbuf);
        float* sbm = sa + RB2 * N;
        const Deapo dp(dxy, fxs, N, Y, y0 + rb, scale);
#pragma unroll
        for (int q = 0; q < NB3; ++q)
#pragma unroll
            for (int r = 0; r < R3; ++r) {
                const int x = j + TP * q + 256 * r;
                const float f = dp(x);
                const float2 z = v[q * R3 + r];
                sa[rb * N + x] = z.x * f;
                sbm[rb * N + x] = z.y * f;
            }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const long long u = u0 + b;
            bulk_s2g(out + (size_t)(2 * u) * M + (size_t)y0 * N, sa, RB2 * N * 4u);
            if (2 * u + 1 < n) bulk_s2g(out + (size_t)(2 * u + 1) * M + (size_t)y0 * N, sbm, RB2 * N * 4u);
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// Persistent version of k_fft1_inv_col: strip s = (angle t, group bg of
// CW2 units with at least one valid unit), bg fastest; triple-buffered like
// k_fft2_col_pers (TMA loads of Q boxes, bulk stores of the slice rows).
template <int LOGN>
__global__ void __launch_bounds__(CW2 * (1 << LOGN) / 16, 1)
k_fft1_inv_pers(const __grid_constant__ CUtensorMap tmap, int T, int ngrp, float scale, float* __restrict__ out,
                long long n, long long u0, int nb, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, LD = N + 16 / CW2, R3 = N / 256, NB3 = 16 / R3, RS = N + 4;
    constexpr int BUF = CW2 * LD;
    extern __shared__ __align__(128) unsigned char colpbuf_raw[];
    float2* base = reinterpret_cast<float2*>(colpbuf_raw);
    __shared__ __align__(8) unsigned long long bar[COLP_BUFS];
    const int nstrip = ngrp * T;
    const int c = threadIdx.x % CW2, j = threadIdx.x / CW2;
    auto load = [&](int s, int k) {
        const int bg = s % ngrp, t = s / ngrp;
        const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar[k % COLP_BUFS]);
        float2* dst = base + (k % COLP_BUFS) * BUF;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb),
                     "r"((unsigned)(N * CW2 * sizeof(float2))) : "memory");
#pragma unroll 1
        for (int q = 0; q < N / 256; ++q)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst + q * 256 * CW2)),
                "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(bg * CW2), "r"(t * N + 256 * q), "r"(sb)
                : "memory");
    };
    if (threadIdx.x == 0) {
        for (int i = 0; i < COLP_BUFS; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if ((int)blockIdx.x < nstrip) load(blockIdx.x, 0);
    }
    __syncthreads();
    const long long plane = (long long)T * N;
    const StageTwiddles<LOGN, true> stw(tw, threadIdx.x / CW2);
    int k = 0;
    for (int s = blockIdx.x; s < nstrip; s += gridDim.x, ++k) {
        float2* fbuf = base + (k % COLP_BUFS) * BUF;
        const int bg = s % ngrp, t = s / ngrp, b0 = bg * CW2;
        if (threadIdx.x == 0 && s + (int)gridDim.x < nstrip) {
            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            load(s + gridDim.x, k + 1);
        }
        fbar_wait((unsigned)__cvta_generic_to_shared(&bar[k % COLP_BUFS]), (unsigned)((k / COLP_BUFS) & 1));
        float2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = fbuf[(j + TP * r) * CW2 + c];
        __syncthreads();
        dft16<true>(v);
        fft16_stages_pre<LOGN, true>(v, fbuf + c * LD, j, stw);
        __syncthreads();
        float* stg = reinterpret_cast<float*>(fbuf);
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int pidx = j + TP * m;
            const float2 z = v[(m % NB3) * R3 + m / NB3];
            stg[(2 * c) * RS + pidx] = z.x * scale;
            stg[(2 * c + 1) * RS + pidx] = z.y * scale;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int cc = 0; cc < CW2; ++cc) {
                if (b0 + cc >= nb) break;
                const long long u = u0 + b0 + cc;
                bulk_s2g(out + (2 * u) * plane + (long long)t * N, stg + (2 * cc) * RS, N * 4u);
                if (2 * u + 1 < n)
                    bulk_s2g(out + (2 * u + 1) * plane + (long long)t * N, stg + (2 * cc + 1) * RS, N * 4u);
            }
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// Persistent version of k_fft2_row_pack_b (radon): strips of 4 rows over
// all B planes, triple-buffered, stage twiddles in registers.  Planes >= nb
// load nothing (zeros) but still complete their buffer's mbarrier phase.
template <int LOGN>
__global__ void __launch_bounds__(RB2 * (1 << LOGN) / 16, 1)
k_fft2_row_pack_pers(const float* __restrict__ in, long long M, int Y, const float* __restrict__ dxy, long long n,
                     long long u0, int nb, float2* __restrict__ g, int nstrip, const float2* __restrict__ tw) {
    constexpr int N = 1 << LOGN, TP = N / 16, R3 = N / 256, NB3 = 16 / R3, BUF = RB2 * N;
    extern __shared__ __align__(128) unsigned char rowpbuf_raw[];
    float2* base = reinterpret_cast<float2*>(rowpbuf_raw);
    float* fxs = reinterpret_cast<float*>(base + COLP_BUFS * BUF);
    __shared__ __align__(8) unsigned long long bar[COLP_BUFS + 1];
    auto load = [&](int s, int k) {
        const long long gr0 = (long long)s * RB2;
        const int b = (int)(gr0 / Y), y0 = (int)(gr0 - (long long)b * Y);
        const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar[k % COLP_BUFS]);
        if (b >= nb) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sb) : "memory");
            return;
        }
        const long long u = u0 + b;
        const bool hb = 2 * u + 1 < n;
        float* sa = reinterpret_cast<float*>(base + (k % COLP_BUFS) * BUF);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb),
                     "r"(RB2 * N * 4u * (hb ? 2u : 1u)) : "memory");
        bulk_g2s(sa, in + (size_t)(2 * u) * M + (size_t)y0 * N, RB2 * N * 4u, sb);
        if (hb) bulk_g2s(sa + RB2 * N, in + (size_t)(2 * u + 1) * M + (size_t)y0 * N, RB2 * N * 4u, sb);
    };
    const unsigned fb = (unsigned)__cvta_generic_to_shared(&bar[COLP_BUFS]);
    if (threadIdx.x == 0) {
        for (int i = 0; i <= COLP_BUFS; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if (dxy) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb), "r"(N * 4u) : "memory");
            bulk_g2s(fxs, dxy, N * 4u, fb);
        }
        if ((int)blockIdx.x < nstrip) load(blockIdx.x, 0);
    }
    __syncthreads();
    if (dxy) fbar_wait(fb, 0);
    const int rb = threadIdx.x / TP, j = threadIdx.x % TP;
    const StageTwiddles<LOGN, false> stw(tw, j);
    int k = 0;
    for (int s = blockIdx.x; s < nstrip; s += gridDim.x, ++k) {
        float2* fbuf = base + (k % COLP_BUFS) * BUF;
        const long long gr0 = (long long)s * RB2;
        const int b = (int)(gr0 / Y), y0 = (int)(gr0 - (long long)b * Y);
        if (threadIdx.x == 0 && s + (int)gridDim.x < nstrip) {
            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            load(s + gridDim.x, k + 1);
        }
        fbar_wait((unsigned)__cvta_generic_to_shared(&bar[k % COLP_BUFS]), (unsigned)((k / COLP_BUFS) & 1));
        const bool ha = b < nb, hb = ha && 2 * (u0 + b) + 1 < n;
        const float* sa = reinterpret_cast<const float*>(fbuf);
        const float* sbm = sa + RB2 * N;
        const Deapo dp(dxy, fxs, N, Y, y0 + rb, 1.f);
        float2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int x = j + TP * r;
            const float d = dp(x);
            v[r] = make_float2(ha ? sa[rb * N + x] * d : 0.f, hb ? sbm[rb * N + x] * d : 0.f);
        }
        __syncthreads();
        dft16<false>(v);
        fft16_stages_pre<LOGN, false>(v, fbuf + rb * N, j, stw);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NB3; ++q)
#pragma unroll
            for (int r = 0; r < R3; ++r) fbuf[rb * N + j + TP * q + 256 * r] = v[q * R3 + r];
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            bulk_s2g(g + (size_t)b * M + (size_t)y0 * N, fbuf, RB2 * N * 8u);
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

int log2_fft(long long n) {
    if (n < 512 || n > 4096 || (n & (n - 1))) return 0;
    int l = 0;
    while ((1LL << l) < n) ++l;
    return l;
}

// W_n^k for k < n, then (n >= 256) the stage tables of fft16_stages_tab:
// T2[r][m] = W_n^(m (n/256) r) (16 x 16) and T3[r][m] = W_n^(m r) (n/256 x 256)
const float2* twiddles(sptb_plan* p, int logn) {
    if (!p->twn[logn]) {
        const int n = 1 << logn;
        auto w = [n](long long k) {
            const double a = -2.0 * M_PI * (double)(k % n) / (double)n;
            return make_float2((float)std::cos(a), (float)std::sin(a));
        };
        std::vector<float2> h(n);
        for (int k = 0; k < n; ++k) h[k] = w(k);
        if (n >= 256) {
            const int r3 = n / 256;
            for (int r = 0; r < 16; ++r)
                for (int m = 0; m < 16; ++m) h.push_back(w((long long)m * (n / 256) * r));
            for (int r = 0; r < r3; ++r)
                for (int m = 0; m < 256; ++m) h.push_back(w((long long)m * r));
        }
        if (cudaMalloc(&p->twn[logn], sizeof(float2) * h.size()) != cudaSuccess) return nullptr;
        if (cudaMemcpy(p->twn[logn], h.data(), sizeof(float2) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess)
            return nullptr;
    }
    return (const float2*)p->twn[logn];
}

bool col_tma_ok(const void* g) {
    return tmap_encoder() != nullptr && ((uintptr_t)g % 16) == 0 && !switches().no_tma;
}

// G [b][y][x] complex64 as a 3-D tensor of 8-byte elements; box CW2 x 256 x 1
int col_tmap(const sptb_plan* p, const void* g, int planes, CUtensorMap* tm) {
    const cuuint64_t dims[3] = {(cuuint64_t)p->X, (cuuint64_t)p->Y, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)p->X * 8, (cuuint64_t)p->M * 8};
    const cuuint32_t box[3] = {(cuuint32_t)CW2, 256u, 1u};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult cr = tmap_encoder()(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(g), dims, strides,
                                       box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(SPTB_ERR_CUDA, "cuTensorMapEncodeTiled (fft2) failed: " + std::to_string((int)cr));
    return SPTB_OK;
}

int sm_count() {
    static int n = [] {
        int d = 0, v = 148;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
        return v;
    }();
    return n;
}

// y pass over nb planes: persistent triple-buffered kernel (default) or one CTA per strip
template <int LOGN, bool INV>
int run_col(const CUtensorMap& tm, float2* g, int X, long long M, int strips, int nb, const float2* tw,
            cudaStream_t st) {
    constexpr int NT = CW2 * (1 << LOGN) / 16;
    const int nstrip = nb * strips;
    const size_t buf = sizeof(float2) * CW2 * ((1 << LOGN) + 16 / CW2);
    if (COLP_BUFS * buf <= 227 * 1024 && !switches().fft2_no_persist) {
        const int sm = (int)(COLP_BUFS * buf);
        SPTB_CUDA(set_smem_once((const void*)k_fft2_col_pers<LOGN, INV>, sm, SPTB_FFT_CARVEOUT));
        k_fft2_col_pers<LOGN, INV><<<(unsigned)std::min(nstrip, sm_count()), NT, sm, st>>>(tm, strips, nstrip, tw);
        SPTB_LAUNCHED();
        return SPTB_OK;
    }
    SPTB_CUDA(set_smem_once((const void*)k_fft2_col_tma<LOGN, INV>, (int)buf, SPTB_FFT_CARVEOUT));
    k_fft2_col_tma<LOGN, INV><<<(unsigned)nstrip, NT, (int)buf, st>>>(tm, g, X, M, strips, tw);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

template <int LOGN>
int col_launch(sptb_plan* p, float2* g, int nb, cudaStream_t st) {
    const float2* tw = twiddles(p, LOGN);
    if (!tw) return fail(SPTB_ERR_CUDA, "fft2: twiddle table");
    constexpr int NT = CW2 * (1 << LOGN) / 16;
    const int sm = (int)(sizeof(float2) * CW2 * ((1 << LOGN) + 16 / CW2));
    const int strips = p->X / CW2;
    if (col_tma_ok(g)) {
        CUtensorMap tm;
        SPTB_TRY(col_tmap(p, g, nb, &tm));
        return run_col<LOGN, true>(tm, g, p->X, p->M, strips, nb, tw, st);
    }
    SPTB_CUDA(set_smem_once((const void*)k_fft2_col<LOGN, true>, sm, SPTB_FFT_CARVEOUT));
    k_fft2_col<LOGN, true><<<(unsigned)(nb * strips), NT, sm, st>>>(g, p->X, p->M, strips, tw);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

template <int LOGN>
int col_launch_fwd(sptb_plan* p, float2* g, int nb, cudaStream_t st) {
    const float2* tw = twiddles(p, LOGN);
    if (!tw) return fail(SPTB_ERR_CUDA, "fft2: twiddle table");
    constexpr int NT = CW2 * (1 << LOGN) / 16;
    const int sm = (int)(sizeof(float2) * CW2 * ((1 << LOGN) + 16 / CW2));
    const int strips = p->X / CW2;
    if (col_tma_ok(g)) {
        CUtensorMap tm;
        SPTB_TRY(col_tmap(p, g, nb, &tm));
        return run_col<LOGN, false>(tm, g, p->X, p->M, strips, nb, tw, st);
    }
    SPTB_CUDA(set_smem_once((const void*)k_fft2_col<LOGN, false>, sm, SPTB_FFT_CARVEOUT));
    k_fft2_col<LOGN, false><<<(unsigned)(nb * strips), NT, sm, st>>>(g, p->X, p->M, strips, tw);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

// bulk copies: 16-byte aligned caller slices and G (rows are 4 N or 8 N bytes);
// the deapodization plane is applied from its separable factors (plan->deapo_xy)
bool row_bulk_ok(const void* a, const void* g) {
    return ((uintptr_t)a % 16) == 0 && ((uintptr_t)g % 16) == 0 &&
           !switches().fft2_no_bulk;
}

template <int LOGN, bool INV>
int col_launch_dir(sptb_plan* p, float2* g, int nb, cudaStream_t st) {
    const float2* tw = twiddles(p, LOGN);
    if (!tw) return fail(SPTB_ERR_CUDA, "fft2: twiddle table");
    constexpr int NT = CW2 * (1 << LOGN) / 16;
    const int sm = (int)(sizeof(float2) * CW2 * ((1 << LOGN) + 16 / CW2));
    const int strips = p->X / CW2;
    CUtensorMap tm;
    SPTB_TRY(col_tmap(p, g, nb, &tm));
    return run_col<LOGN, INV>(tm, g, p->X, p->M, strips, nb, tw, st);
}

template <int LOGN, bool INV>
int row_launch_dir(sptb_plan* p, float2* g, int nb, cudaStream_t st) {
    const float2* tw = twiddles(p, LOGN);
    if (!tw) return fail(SPTB_ERR_CUDA, "fft2: twiddle table");
    constexpr int NT = RB2 * (1 << LOGN) / 16;
    const int sm = (int)(8 * RB2 * (1 << LOGN));
    SPTB_CUDA(set_smem_once((const void*)k_fft2_row_b<LOGN, INV>, sm, SPTB_FFT_CARVEOUT));
    k_fft2_row_b<LOGN, INV><<<(unsigned)((long long)nb * p->Y / RB2), NT, sm, st>>>(g, tw);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

template <bool INV>
int fft2_inplace(sptb_plan* p, float2* g, int nb, cudaStream_t st) {
    switch (log2_fft(p->Y)) {
        case 9: SPTB_TRY((col_launch_dir<9, INV>(p, g, nb, st))); break;
        case 10: SPTB_TRY((col_launch_dir<10, INV>(p, g, nb, st))); break;
        case 11: SPTB_TRY((col_launch_dir<11, INV>(p, g, nb, st))); break;
        case 12: SPTB_TRY((col_launch_dir<12, INV>(p, g, nb, st))); break;
        default: return fail(SPTB_ERR_ARG, "fused FFT2: unsupported n_y");
    }
    switch (log2_fft(p->X)) {
        case 9: return row_launch_dir<9, INV>(p, g, nb, st);
        case 10: return row_launch_dir<10, INV>(p, g, nb, st);
        case 11: return row_launch_dir<11, INV>(p, g, nb, st);
        case 12: return row_launch_dir<12, INV>(p, g, nb, st);
    }
    return fail(SPTB_ERR_ARG, "fused FFT2: unsupported n_x");
}

template <int LOGN>
int row_pack_launch(sptb_plan* p, const float* in, const float* plane, int64_t n, int64_t u0, int nb, int B,
                    float2* g, cudaStream_t st) {
    const float2* tw = twiddles(p, LOGN);
    if (!tw) return fail(SPTB_ERR_CUDA, "fft2: twiddle table");
    constexpr int NT = RB2 * (1 << LOGN) / 16;
    if (row_bulk_ok(in, g)) {
        const int smp = (int)((COLP_BUFS * 8 * RB2 + 4) * (1 << LOGN));
        if (smp <= 227 * 1024 && !switches().fft2_no_persist) {
            const int nstrip = (int)((long long)B * p->Y / RB2);
            SPTB_CUDA(set_smem_once((const void*)k_fft2_row_pack_pers<LOGN>, smp, SPTB_FFT_CARVEOUT));
            k_fft2_row_pack_pers<LOGN><<<(unsigned)std::min(nstrip, sm_count()), NT, smp, st>>>(
                in, p->M, p->Y, plane ? p->deapo_xy : nullptr, n, u0, nb, g, nstrip, tw);
            SPTB_LAUNCHED();
            return SPTB_OK;
        }
        const int smb = (int)((8 * RB2 + 4) * (1 << LOGN));
        SPTB_CUDA(set_smem_once((const void*)k_fft2_row_pack_b<LOGN>, smb, SPTB_FFT_CARVEOUT));
        k_fft2_row_pack_b<LOGN><<<(unsigned)((long long)B * p->Y / RB2), NT, smb, st>>>(
            in, p->M, p->Y, plane ? p->deapo_xy : nullptr, n, u0, nb, g, tw);
        SPTB_LAUNCHED();
        return SPTB_OK;
    }
    const int sm = (int)(sizeof(float2) * RB2 * (1 << LOGN));
    SPTB_CUDA(set_smem_once((const void*)k_fft2_row_pack<LOGN>, sm, SPTB_FFT_CARVEOUT));
    k_fft2_row_pack<LOGN><<<(unsigned)(((long long)B * p->Y + RB2 - 1) / RB2), NT, sm, st>>>(
        in, p->M, p->Y, plane, n, u0, nb, g, tw);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

template <int LOGN>
int row_launch(sptb_plan* p, const float2* g, const float* plane, float scale, float* out, int64_t n, int64_t u0,
               int nb, cudaStream_t st) {
    const float2* tw = twiddles(p, LOGN);
    if (!tw) return fail(SPTB_ERR_CUDA, "fft2: twiddle table");
    constexpr int NT = RB2 * (1 << LOGN) / 16;
    if (row_bulk_ok(out, g)) {
        const int smp = (int)((COLP_BUFS * 8 * RB2 + 4) * (1 << LOGN));
        if (smp <= 227 * 1024 && !switches().fft2_no_persist) {
            const int nstrip = (int)((long long)nb * p->Y / RB2);
            SPTB_CUDA(set_smem_once((const void*)k_fft2_row_unpack_pers<LOGN>, smp, SPTB_FFT_CARVEOUT));
            k_fft2_row_unpack_pers<LOGN><<<(unsigned)std::min(nstrip, sm_count()), NT, smp, st>>>(
                g, p->M, p->Y, plane ? p->deapo_xy : nullptr, scale, out, n, u0, nstrip, tw);
            SPTB_LAUNCHED();
            return SPTB_OK;
        }
        const int smb = (int)((8 * RB2 + 4) * (1 << LOGN));
        SPTB_CUDA(set_smem_once((const void*)k_fft2_row_unpack_b<LOGN>, smb, SPTB_FFT_CARVEOUT));
        k_fft2_row_unpack_b<LOGN><<<(unsigned)((long long)nb * p->Y / RB2), NT, smb, st>>>(
            g, p->M, p->Y, plane ? p->deapo_xy : nullptr, scale, out, n, u0, nb, tw);
        SPTB_LAUNCHED();
        return SPTB_OK;
    }
    const int sm = (int)(sizeof(float2) * RB2 * (1 << LOGN));
    SPTB_CUDA(set_smem_once((const void*)k_fft2_row_unpack<LOGN>, sm, SPTB_FFT_CARVEOUT));
    k_fft2_row_unpack<LOGN><<<(unsigned)(((long long)nb * p->Y + RB2 - 1) / RB2), NT, sm, st>>>(
        g, p->M, p->Y, plane, scale, out, n, u0, nb, tw);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

const int* g_fwd_perm = nullptr;  // row map of the current forward launch (nullptr: sample order)

int fft1_log2(const sptb_plan* p) {
    const int P = p->P;
    if (P < 128 || P > 4096 || (P & (P - 1))) return 0;
    int l = 0;
    while ((1 << l) < P) ++l;
    return l;
}

int ensure_tw(sptb_plan* p) {
    if (p->tw1) return SPTB_OK;
    std::vector<float2> h(p->P);
    for (int k = 0; k < p->P; ++k) {
        const double a = -2.0 * M_PI * (double)k / (double)p->P;
        h[k] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    SPTB_CUDA(cudaMalloc(&p->tw1, sizeof(float2) * p->P));
    SPTB_CUDA(cudaMemcpy(p->tw1, h.data(), sizeof(float2) * p->P, cudaMemcpyHostToDevice));
    return SPTB_OK;
}

template <int LOGN>
int fwd_launch(sptb_plan* p, const void* in, int fmt, int64_t n, int64_t u0, int nb, int B, void* q,
               cudaStream_t st) {
    const size_t sm = sizeof(float2) * FBG * (1 << LOGN);
    if constexpr (LOGN >= 9) {
        if (!switches().fft1_stockham) {
#ifndef SPTB_FFT1_BG
#define SPTB_FFT1_BG 4
#endif
            // batch columns per CTA: 4 (32-byte row runs); 8 (64-byte runs, 1024-thread CTAs) measured 0.94 vs 0.70 ms
            constexpr int BG = (SPTB_FFT1_BG * (1 << LOGN) / 16 <= 1024) ? SPTB_FFT1_BG : FBG;
            if (B % BG == 0) {
                constexpr int NT = BG * (1 << LOGN) / 16;
                const size_t smb = sizeof(float2) * BG * (1 << LOGN);
                if (!(fmt & SPTB_FMT_COMPLEX) && ((uintptr_t)in % 16) == 0 && !switches().fft1_no_bulk) {
                    SPTB_CUDA(set_smem_once((const void*)k_fft1r_fwd<LOGN, BG, true>, (int)smb));
                    k_fft1r_fwd<LOGN, BG, true><<<dim3((unsigned)(B / BG), (unsigned)p->T), NT, smb, st>>>(
                        (const float*)in, 0, n, u0, nb, p->T, g_fwd_perm, (const float2*)p->tw1, (float2*)q, B);
                    SPTB_LAUNCHED();
                    return SPTB_OK;
                }
                SPTB_CUDA(set_smem_once((const void*)k_fft1r_fwd<LOGN, BG>, (int)smb));
                k_fft1r_fwd<LOGN, BG><<<dim3((unsigned)(B / BG), (unsigned)p->T), NT, smb, st>>>(
                    (const float*)in, (fmt & SPTB_FMT_COMPLEX) ? 1 : 0, n, u0, nb, p->T, g_fwd_perm,
                    (const float2*)p->tw1, (float2*)q, B);
            } else {
                constexpr int NT = FBG * (1 << LOGN) / 16;
                SPTB_CUDA(set_smem_once((const void*)k_fft1r_fwd<LOGN, FBG>, (int)sm));
                k_fft1r_fwd<LOGN, FBG><<<dim3((unsigned)(B / FBG), (unsigned)p->T), NT, sm, st>>>(
                    (const float*)in, (fmt & SPTB_FMT_COMPLEX) ? 1 : 0, n, u0, nb, p->T, g_fwd_perm,
                    (const float2*)p->tw1, (float2*)q, B);
            }
            SPTB_LAUNCHED();
            return SPTB_OK;
        }
    }
    SPTB_CUDA(set_smem_once((const void*)k_fft1_fwd<LOGN>, (int)sm, SPTB_FFT_CARVEOUT));
    k_fft1_fwd<LOGN><<<dim3((unsigned)(B / FBG), (unsigned)p->T), FT, sm, st>>>(
        (const float*)in, (fmt & SPTB_FMT_COMPLEX) ? 1 : 0, n, u0, nb, p->T, g_fwd_perm,
        (const float2*)p->tw1, (float2*)q, B);
    SPTB_LAUNCHED();
    return SPTB_OK;
}
template <int LOGN>
int inv_launch(sptb_plan* p, const void* q, int B, void* out, int fmt, int64_t n, int64_t u0, int nb,
               cudaStream_t st) {
    // (a register radix-16 inverse, as the forward, measured slower than the
    // Stockham kernel on the gathered input and was removed)
    const size_t sm = sizeof(float2) * FBG * (1 << LOGN);
    SPTB_CUDA(set_smem_once((const void*)k_fft1_inv<LOGN>, (int)sm, SPTB_FFT_CARVEOUT));
    k_fft1_inv<LOGN><<<dim3((unsigned)((nb + FBG - 1) / FBG), (unsigned)p->T), FT, sm, st>>>(
        (const float2*)q, B, p->shp.perm, (const float2*)p->tw1, 1.0f / (float)p->P, (float*)out,
        (fmt & SPTB_FMT_COMPLEX) ? 1 : 0, n, u0, nb, p->T);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

}  // namespace

// usable: complex64 plan, f32 caller data, n_p = 2^k in [128, 4096], B a multiple of FBG
bool fft1_fused_ok(const sptb_plan* p, int fmt, int B) {
    return p->prec == SPTB_PREC_F32 && !(fmt & SPTB_FMT_F64) && fft1_log2(p) > 0 && B % FBG == 0 &&
           !switches().no_fused_fft1;
}

int launch_fft1_fwd(sptb_plan* p, const void* in, int fmt, int64_t n, int64_t u0, int nb, int B, void* q,
                    cudaStream_t st, bool permute) {
    SPTB_TRY(ensure_tw(p));
    g_fwd_perm = permute ? p->shp.perm : nullptr;
    switch (fft1_log2(p)) {
        case 7: return fwd_launch<7>(p, in, fmt, n, u0, nb, B, q, st);
        case 8: return fwd_launch<8>(p, in, fmt, n, u0, nb, B, q, st);
        case 9: return fwd_launch<9>(p, in, fmt, n, u0, nb, B, q, st);
        case 10: return fwd_launch<10>(p, in, fmt, n, u0, nb, B, q, st);
        case 11: return fwd_launch<11>(p, in, fmt, n, u0, nb, B, q, st);
        case 12: return fwd_launch<12>(p, in, fmt, n, u0, nb, B, q, st);
    }
    return fail(SPTB_ERR_ARG, "fused FFT1: unsupported n_p");
}

int launch_fft1_inv(sptb_plan* p, const void* q, int B, void* out, int fmt, int64_t n, int64_t u0, int nb,
                    cudaStream_t st) {
    SPTB_TRY(ensure_tw(p));
    switch (fft1_log2(p)) {
        case 7: return inv_launch<7>(p, q, B, out, fmt, n, u0, nb, st);
        case 8: return inv_launch<8>(p, q, B, out, fmt, n, u0, nb, st);
        case 9: return inv_launch<9>(p, q, B, out, fmt, n, u0, nb, st);
        case 10: return inv_launch<10>(p, q, B, out, fmt, n, u0, nb, st);
        case 11: return inv_launch<11>(p, q, B, out, fmt, n, u0, nb, st);
        case 12: return inv_launch<12>(p, q, B, out, fmt, n, u0, nb, st);
    }
    return fail(SPTB_ERR_ARG, "fused FFT1: unsupported n_p");
}

// usable: complex64 plan, real f32 caller slices, X and Y powers of two in
// [512, 4096] (the row kernel owns whole rows: Y * nb a multiple of RB2)
bool fft2_fused_ok(const sptb_plan* p, int fmt) {
    return p->prec == SPTB_PREC_F32 && !(fmt & (SPTB_FMT_F64 | SPTB_FMT_COMPLEX)) && log2_fft(p->X) > 0 &&
           log2_fft(p->Y) > 0 && !switches().no_fused_fft2;
}

int launch_fft2_inv_unpack(sptb_plan* p, void* g, const void* plane, double scale, void* out, int64_t n,
                           int64_t u0, int nb, cudaStream_t st) {
    float2* G = (float2*)g;
    int rc;
    switch (log2_fft(p->Y)) {
        case 9: rc = col_launch<9>(p, G, nb, st); break;
        case 10: rc = col_launch<10>(p, G, nb, st); break;
        case 11: rc = col_launch<11>(p, G, nb, st); break;
        case 12: rc = col_launch<12>(p, G, nb, st); break;
        default: return fail(SPTB_ERR_ARG, "fused FFT2: unsupported n_y");
    }
    if (rc != SPTB_OK) return rc;
    const float* pl = (const float*)plane;
    const float sc = (float)scale;
    switch (log2_fft(p->X)) {
        case 9: return row_launch<9>(p, G, pl, sc, (float*)out, n, u0, nb, st);
        case 10: return row_launch<10>(p, G, pl, sc, (float*)out, n, u0, nb, st);
        case 11: return row_launch<11>(p, G, pl, sc, (float*)out, n, u0, nb, st);
        case 12: return row_launch<12>(p, G, pl, sc, (float*)out, n, u0, nb, st);
    }
    return fail(SPTB_ERR_ARG, "fused FFT2: unsupported n_x");
}

int launch_fft2_pack_fwd(sptb_plan* p, const void* in, const void* plane, int64_t n, int64_t u0, int nb, int B,
                         void* g, cudaStream_t st) {
    float2* G = (float2*)g;
    const float* pl = (const float*)plane;
    int rc;
    switch (log2_fft(p->X)) {
        case 9: rc = row_pack_launch<9>(p, (const float*)in, pl, n, u0, nb, B, G, st); break;
        case 10: rc = row_pack_launch<10>(p, (const float*)in, pl, n, u0, nb, B, G, st); break;
        case 11: rc = row_pack_launch<11>(p, (const float*)in, pl, n, u0, nb, B, G, st); break;
        case 12: rc = row_pack_launch<12>(p, (const float*)in, pl, n, u0, nb, B, G, st); break;
        default: return fail(SPTB_ERR_ARG, "fused FFT2: unsupported n_x");
    }
    if (rc != SPTB_OK) return rc;
    switch (log2_fft(p->Y)) {  // zero planes stay zero: only the nb filled planes need the y pass
        case 9: return col_launch_fwd<9>(p, G, nb, st);
        case 10: return col_launch_fwd<10>(p, G, nb, st);
        case 11: return col_launch_fwd<11>(p, G, nb, st);
        case 12: return col_launch_fwd<12>(p, G, nb, st);
    }
    return fail(SPTB_ERR_ARG, "fused FFT2: unsupported n_y");
}

// in-place unnormalised 2-D FFT of nb planes [b][y][x] (cuFFT's sign convention)
bool fft2_inplace_ok(const sptb_plan* p, const void* g) {
    return p->prec == SPTB_PREC_F32 && log2_fft(p->X) > 0 && log2_fft(p->Y) > 0 && col_tma_ok(g) &&
           !switches().no_fused_fft2;
}

int launch_fft2_inplace(sptb_plan* p, void* g, int nb, bool inverse, cudaStream_t st) {
    return inverse ? fft2_inplace<true>(p, (float2*)g, nb, st) : fft2_inplace<false>(p, (float2*)g, nb, st);
}

bool fft1_inv_tma_ok(const sptb_plan* p, const void* q, const void* out, int fmt, int B) {
    return p->prec == SPTB_PREC_F32 && !(fmt & (SPTB_FMT_F64 | SPTB_FMT_COMPLEX)) && log2_fft(p->P) > 0 &&
           B % CW2 == 0 && col_tma_ok(q) && ((uintptr_t)out % 16) == 0 &&
           !switches().no_fused_fft1 && !switches().fft1_inv_gather;
}

// Q [s][b] complex64 (s in sample order) as a 2-D tensor of 8-byte elements;
// box CW2 columns x 256 rows
int q_tmap(const sptb_plan* p, const void* q, int B, CUtensorMap* tm) {
    const cuuint64_t dims[2] = {(cuuint64_t)B, (cuuint64_t)p->N};
    const cuuint64_t strides[1] = {(cuuint64_t)B * 8};
    const cuuint32_t box[2] = {(cuuint32_t)CW2, 256u};
    const cuuint32_t es[2] = {1, 1};
    const CUresult cr = tmap_encoder()(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(q), dims, strides, box,
                                       es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(SPTB_ERR_CUDA, "cuTensorMapEncodeTiled (fft1) failed: " + std::to_string((int)cr));
    return SPTB_OK;
}

template <int LOGN>
int fwd_col_launch(sptb_plan* p, const void* in, int64_t n, int64_t u0, int nb, int B, void* q, cudaStream_t st) {
    const float2* tw = twiddles(p, LOGN);
    if (!tw) return fail(SPTB_ERR_CUDA, "fft1: twiddle table");
    CUtensorMap tm;
    SPTB_TRY(q_tmap(p, q, B, &tm));
    constexpr int NT = CW2 * (1 << LOGN) / 16;
    const int sm = (int)(sizeof(float2) * CW2 * ((1 << LOGN) + 16 / CW2));
    if (COLP_BUFS * sm <= 227 * 1024 && !switches().fft2_no_persist) {
        const int smp = COLP_BUFS * sm, nstrip = (B / CW2) * p->T;
        SPTB_CUDA(set_smem_once((const void*)k_fft1_fwd_pers<LOGN>, smp, SPTB_FFT_CARVEOUT));
        k_fft1_fwd_pers<LOGN><<<(unsigned)std::min(nstrip, sm_count()), NT, smp, st>>>(
            tm, (const float*)in, p->T, B / CW2, n, u0, nb, tw);
        SPTB_LAUNCHED();
        return SPTB_OK;
    }
    SPTB_CUDA(set_smem_once((const void*)k_fft1_fwd_col<LOGN>, sm, SPTB_FFT_CARVEOUT));
    k_fft1_fwd_col<LOGN><<<dim3((unsigned)(B / CW2), (unsigned)p->T), NT, sm, st>>>(tm, (const float*)in, p->T, n, u0,
                                                                                   nb, tw);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

int launch_fft1_fwd_tma(sptb_plan* p, const void* in, int64_t n, int64_t u0, int nb, int B, void* q,
                        cudaStream_t st) {
    switch (log2_fft(p->P)) {
        case 9: return fwd_col_launch<9>(p, in, n, u0, nb, B, q, st);
        case 10: return fwd_col_launch<10>(p, in, n, u0, nb, B, q, st);
        case 11: return fwd_col_launch<11>(p, in, n, u0, nb, B, q, st);
        case 12: return fwd_col_launch<12>(p, in, n, u0, nb, B, q, st);
    }
    return fail(SPTB_ERR_ARG, "fft1 (TMA): unsupported n_p");
}

bool fft1_fwd_tma_ok(const sptb_plan* p, const void* in, const void* q, int fmt, int B) {
    return p->prec == SPTB_PREC_F32 && !(fmt & (SPTB_FMT_F64 | SPTB_FMT_COMPLEX)) && log2_fft(p->P) > 0 &&
           B % CW2 == 0 && col_tma_ok(q) && ((uintptr_t)in % 16) == 0 && !switches().no_fused_fft1 &&
           !switches().fft1_fwd_rows;
}

template <int LOGN>
int inv_col_launch(sptb_plan* p, const void* q, int B, void* out, int64_t n, int64_t u0, int nb, cudaStream_t st) {
    const float2* tw = twiddles(p, LOGN);
    if (!tw) return fail(SPTB_ERR_CUDA, "fft1: twiddle table");
    CUtensorMap tm;
    SPTB_TRY(q_tmap(p, q, B, &tm));
    constexpr int NT = CW2 * (1 << LOGN) / 16;
    const int sm = (int)(sizeof(float2) * CW2 * ((1 << LOGN) + 16 / CW2));
    if (COLP_BUFS * sm <= 227 * 1024 && !switches().fft2_no_persist) {
        const int smp = COLP_BUFS * sm, ngrp = (nb + CW2 - 1) / CW2, nstrip = ngrp * p->T;
        SPTB_CUDA(set_smem_once((const void*)k_fft1_inv_pers<LOGN>, smp, SPTB_FFT_CARVEOUT));
        k_fft1_inv_pers<LOGN><<<(unsigned)std::min(nstrip, sm_count()), NT, smp, st>>>(
            tm, p->T, ngrp, 1.0f / (float)p->P, (float*)out, n, u0, nb, tw);
        SPTB_LAUNCHED();
        return SPTB_OK;
    }
    SPTB_CUDA(set_smem_once((const void*)k_fft1_inv_col<LOGN>, sm, SPTB_FFT_CARVEOUT));
    k_fft1_inv_col<LOGN><<<dim3((unsigned)((nb + CW2 - 1) / CW2), (unsigned)p->T), NT, sm, st>>>(
        tm, p->T, 1.0f / (float)p->P, (float*)out, n, u0, nb, tw);
    SPTB_LAUNCHED();
    return SPTB_OK;
}

int launch_fft1_inv_tma(sptb_plan* p, const void* q, int B, void* out, int64_t n, int64_t u0, int nb,
                        cudaStream_t st) {
    switch (log2_fft(p->P)) {
        case 9: return inv_col_launch<9>(p, q, B, out, n, u0, nb, st);
        case 10: return inv_col_launch<10>(p, q, B, out, n, u0, nb, st);
        case 11: return inv_col_launch<11>(p, q, B, out, n, u0, nb, st);
        case 12: return inv_col_launch<12>(p, q, B, out, n, u0, nb, st);
    }
    return fail(SPTB_ERR_ARG, "fft1 (TMA): unsupported n_p");
}

const float2* fft2_twiddles(sptb_plan* p, int logn) { return twiddles(p, logn); }

int fft2_log2(long long n) { return log2_fft(n); }

// y pass only, in place over nb planes (the solver's fused row passes do the x pass)
int launch_fft2_cols(sptb_plan* p, void* g, int nb, bool inverse, cudaStream_t st) {
    float2* G = (float2*)g;
    switch (log2_fft(p->Y)) {
        case 9: return inverse ? col_launch_dir<9, true>(p, G, nb, st) : col_launch_dir<9, false>(p, G, nb, st);
        case 10: return inverse ? col_launch_dir<10, true>(p, G, nb, st) : col_launch_dir<10, false>(p, G, nb, st);
        case 11: return inverse ? col_launch_dir<11, true>(p, G, nb, st) : col_launch_dir<11, false>(p, G, nb, st);
        case 12: return inverse ? col_launch_dir<12, true>(p, G, nb, st) : col_launch_dir<12, false>(p, G, nb, st);
    }
    return fail(SPTB_ERR_ARG, "fused FFT2: unsupported n_y");
}

}  // namespace sptb
