// Internal declarations shared by the sptb translation units.
//
// Device data layout (per plan, B = complex vectors in one launch):
//   grid vectors, real space   : [b][y][x]   ("G" buffers, cuFFT 2D native)
//   grid vectors, SpMM operand : [m][b]      m = y*n_x + x (batch innermost)
//   sino vectors, real space   : [b][t][p]   ("S" buffers, cuFFT 1D native)
//   sino vectors, SpMM side    : [s][b]      s = t*n_p + p
// The batch-innermost layouts give every gathered nonzero a contiguous
// B*sizeof(complex) run (128-bit lane loads); the batch-outer layouts keep
// cuFFT on its fast contiguous path (measured: batch-inner 2D cuFFT is 11x
// slower on B200, profiles/r01_fftprobe.txt).  Transposes between the two are
// fused into SpMM epilogues where the SpMM writes, and are standalone tiled
// transposes where it reads.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/sptb.h"

namespace sptb {

// Raise a kernel's dynamic shared-memory limit (and set the preferred smem
// carveout in percent; < 0 leaves the driver's choice, e.g. for gather
// kernels that live on L1 hits) once per function: cudaFuncSetAttribute is not free, and the hot
// launch paths call this every time.
cudaError_t set_smem_once(const void* func, int bytes, int carveout = 100);

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
void count_launch(int n = 1);
void count_fft(int n = 1);

#define SPTB_CUDA(expr)                                                     \
    do {                                                                    \
        cudaError_t _e = (expr);                                            \
        if (_e != cudaSuccess)                                              \
            return ::sptb::fail(SPTB_ERR_CUDA, std::string(#expr) + ": " +  \
                                cudaGetErrorString(_e));                    \
    } while (0)

#define SPTB_CUFFT(expr)                                                    \
    do {                                                                    \
        cufftResult _r = (expr);                                            \
        if (_r != CUFFT_SUCCESS)                                            \
            return ::sptb::fail(SPTB_ERR_CUFFT, std::string(#expr) +        \
                                " -> cufftResult " + std::to_string((int)_r)); \
    } while (0)

#define SPTB_TRY(expr)                                                      \
    do {                                                                    \
        int _s = (expr);                                                    \
        if (_s != SPTB_OK) return _s;                                       \
    } while (0)

#define SPTB_LAUNCHED()                                                     \
    do {                                                                    \
        ::sptb::count_launch();                                             \
        cudaError_t _e = cudaGetLastError();                                \
        if (_e != cudaSuccess)                                              \
            return ::sptb::fail(SPTB_ERR_CUDA, std::string("launch: ") +    \
                                cudaGetErrorString(_e));                    \
    } while (0)

// CSR matrix on the device (int32 indices, complex values of plan precision)
struct DevCSR {
    int64_t rows = 0, cols = 0, nnz = 0;
    int* row_ptr = nullptr;   // rows + 1
    int* col = nullptr;       // nnz
    void* val = nullptr;      // nnz complex (float2 or double2)
    int max_row = 0;          // longest row
};

// S^H regrouped by grid patch: every sample is assigned to the PATCH_W x
// PATCH_W grid patch holding its stencil centre, so all of its nonzeros fall in
// the patch's box (patch + halo of width/2 cells).  Samples are renumbered
// s' (patch-major, stable); work items cover <= PATCH_ITEM_ROWS samples of one
// patch.  Nonzeros are stored as (box-local cell, value) records.
constexpr int PATCH_W = 8;
#ifndef SPTB_ITEM_ROWS
#define SPTB_ITEM_ROWS 192
#endif
constexpr int PATCH_ITEM_ROWS = SPTB_ITEM_ROWS;

// Slot mode (kernel width 3): a sample's nonzeros all lie in the 3x3 block
// around its stencil centre, so a row is stored as 9 fixed slots (pruned
// entries are zero) plus the box cell of the block origin in a tenth slot:
// no per-nonzero index, and the cell offsets of the slots are compile-time
// constants.  Rows whose block leaves their patch box ("irregular": centre
// outside the grid) are numbered last and handled by a direct-gather kernel.
constexpr int SLOT_STRIDE = 10;  // complex elements per slot-mode row

struct PatchSH {
    int halo = 1, bw = 10, npx = 0, npy = 0;
    int slot_mode = 0;        // 1: sval/irregular layout, 0: records (meta/rp)
    int64_t n_items = 0;
    int64_t n_reg = 0;        // slot mode: rows [0, n_reg) are in items, the rest irregular
    int max_item_nnz = 0;
    int4* items = nullptr;    // {patch id, row begin (s'), row end, entry begin}
    int* rp = nullptr;        // N + 1, row pointers in s' order (record mode)
    void* meta = nullptr;     // nnz records {u32 cell, u32 pad, complex val} (record mode)
    void* sval = nullptr;     // slot mode: [N][SLOT_STRIDE] complex, slot 9 .x = base cell bits
    unsigned char* item_perm = nullptr;  // slot mode: [n_items][PATCH_ITEM_ROWS] row hand-out order
    int* perm = nullptr;      // perm[s] = s'
    int* order = nullptr;     // order[s'] = s
    int* s_colp = nullptr;    // S column indices renumbered to s'
};

// Sample border class inside its patch (TL T TR R BR B BL L interior): the
// within-patch sample order of build_patches groups samples by it.
constexpr int PATCH_NCLS = 9;
inline int border_class(int lx, int ly) {
    const bool l = lx == 0, r = lx == PATCH_W - 1, t = ly == 0, b = ly == PATCH_W - 1;
    if (t) return l ? 0 : (r ? 2 : 1);
    if (b) return r ? 4 : (l ? 6 : 5);
    if (r) return 3;
    if (l) return 7;
    return 8;
}

// Schedule of the row-segment S kernel (sptb_spmm_s.cu), built once per plan
// from S's row pointers: tiles of short rows and the long rows.
struct SSeg {
    bool built = false;
    int n_tiles = 0, n_long = 0;
    int4* tiles = nullptr;  // {row begin, row end, first pair record, pair records}
    int* longs = nullptr;   // long row ids, longest first
    unsigned long long* pairs = nullptr;  // per tile, its rows by length in pairs (packed)
    int4* tile_e = nullptr;  // per tile {first entry, entries, first pair, pairs} (L2 prefetch of a later tile)
    // the copy of S the kernel reads: rows start on even entries (zero pads),
    // columns [0] sample order / [1] s', values [0] S / [1] S diag(w)
    int* prp = nullptr;
    int64_t pnnz = 0;
    int* pcol[2] = {nullptr, nullptr};
    void* pval[2] = {nullptr, nullptr};
    bool pcol_ok[2] = {false, false}, pval_ok[2] = {false, false};
};

// Path-selection switches (tests and A/B measurements only): read from the
// environment once, and again on sptb_reload_switches().
struct Switches {
    bool no_tma = false, no_fused_fft1 = false, no_fused_fft2 = false;
    bool fft2_no_persist = false, fft2_no_bulk = false;
    bool fft1_stockham = false, fft1_no_bulk = false;
    bool fft1_inv_gather = false, fft1_fwd_rows = false, fft1_perm = false;
    bool sirt_unfused = false, xpass_unfused = false, spmm_rows = false, no_graph = false;
    int pipe_chunks = 0;   // host pipeline chunks per call (0: default)
    std::vector<int> pipe_sizes;  // explicit host pipeline chunk sizes in units (A/B)
};
const Switches& switches();
void reload_switches();

struct FFTPlans {
    cufftHandle fft2 = 0;   // Y x X, batch B, [b][y][x]
    cufftHandle fft1 = 0;   // n_p,   batch B*T, [b][t][p]
};

}  // namespace sptb

struct sptb_plan {
    int device = 0;
    int prec = SPTB_PREC_F32;
    int P = 0, T = 0, X = 0, Y = 0;
    int64_t M = 0, N = 0;
    double center = 0;
    int max_batch = 1;
    double threshold = 0;
    cudaStream_t stream = nullptr;
    size_t csize = 8;          // bytes per complex element

    sptb::DevCSR S, SH;        // S: M x N rows=grid, SH: N x M rows=samples
    sptb::PatchSH shp;         // patch-grouped S^H (the production forward SpMM)
    sptb::SSeg sseg;           // row-segment S schedule (the production adjoint SpMM)
    void* SW_val = nullptr;    // S values with the filter folded (nullptr: none)
    std::vector<double> w_host;  // filter weights (n_p or N), empty = none
    void* w_dev = nullptr;       // real weights of plan precision (n_p or N)
    int64_t w_len = 0;
    double calib = 1.0;
    void* wspec_dev = nullptr;          // sptb_spectral_apply weights (N entries, plan precision)
    std::vector<double> wspec_host;     // what wspec_dev holds
    std::vector<float> wspec_f32;       // complex64 plans: upload staging

    void* deapo = nullptr;     // M real (plan precision), row-major [y][x]
    float* deapo_xy = nullptr; // separable factors: (-1)^(x-X/2)/kx(x) [X], then (-1)^(y-Y/2)/ky(y) [Y]
    std::vector<double> deapo_host;

    // work buffers (max_batch complex vectors each)
    void* G0 = nullptr;  // grid [b][m]  (FFT2 in place)
    void* G1 = nullptr;  // grid [m][b]
    void* G2 = nullptr;  // extra grid buffers for solvers
    void* S0 = nullptr;  // sino [b][s]  (FFT1 in place)
    void* S1 = nullptr;  // sino [s][b]
    int work_B = 0;      // batch the work buffers are sized for
    // caller-format staging for host pointers
    void* stage_in = nullptr;
    size_t stage_in_bytes = 0;
    void* stage_out = nullptr;
    size_t stage_out_bytes = 0;
    // pipelined host I/O (drive(): H2D / compute / D2H of successive chunks overlap)
    static constexpr int NPIPE = 3;
    cudaStream_t io_in = nullptr, io_out = nullptr;
    cudaEvent_t ev_in[NPIPE] = {}, ev_comp[NPIPE] = {}, ev_out[NPIPE] = {}, ev_start = nullptr;
    void* pin[NPIPE] = {};
    void* pout[NPIPE] = {};
    size_t pin_bytes[NPIPE] = {}, pout_bytes[NPIPE] = {};
    void* tw1 = nullptr;       // fused FFT1 twiddles exp(-2 pi i k / n_p), complex64
    void* twn[13] = {};        // fused FFT2 twiddles exp(-2 pi i k / 2^L), indexed by L
    // reduction scratch
    double* red = nullptr;
    size_t red_len = 0;

    std::map<int, sptb::FFTPlans> ffts;  // keyed by batch
    void* fft_work = nullptr;
    size_t fft_work_bytes = 0;

    std::vector<void*> extra;            // solver-owned device buffers
    // device buffers returned by finished solves, reused by the next one
    // (cudaMalloc/cudaFree per solve stalled the stream and varied by ms)
    std::vector<std::pair<size_t, void*>> pool;
    int* solver_pinned = nullptr;        // lagged early-exit counters
    cudaStream_t solver_stream = nullptr;  // solves run here (capturable: not the legacy stream)
    cudaEvent_t solver_join[2] = {};
    cudaEvent_t solver_ev[4] = {};
};

namespace sptb {

// ---------------------------------------------------------------- helpers
int get_fft(sptb_plan* p, int B, FFTPlans** out);
int ensure_work(sptb_plan* p, int B);
int ensure_stage(void** buf, size_t* have, size_t need);
int is_device_ptr(const void* ptr, bool* dev);

// ---------------------------------------------------------------- matrix build
int build_matrices(sptb_plan* p, const sptb_geometry* g, const sptb_kernel* k);
int fold_filter(sptb_plan* p);
int upload_weights(sptb_plan* p);

// ---------------------------------------------------------------- kernels (templated on precision)
// SpMM  y = A x, x: [col][B]; trans_out: y written [b][row] (else [row][b]);
// sub != nullptr: y = sub - A x  ([row][b], non-transposed only)
template <typename R>
int launch_spmm(const DevCSR& A, const void* val, const void* x, void* y, int B,
                bool trans_out, const void* sub, cudaStream_t st);

template <typename R>
int launch_transpose_bm_to_mb(const void* in, void* out, int B, int64_t M, cudaStream_t st);

// patch-grouped S^H: x [b][m] (batch-outer) -> y [s'][b]; sub: y = sub - S^H x;
// sample_order: rows written at order[s'] = s instead (TMA path, no sub)
template <typename R>
int launch_spmm_sh_patch(const sptb_plan* p, const void* x_bm, void* y_sb, int B, const void* sub,
                         cudaStream_t st, bool sample_order = false);
bool tma_ok(const sptb_plan* p, const void* x);  // the TMA S^H path is usable for operand x
// [b][s] -> [perm[s]][b]   and   [s'][b] -> [b][order[s']]
template <typename R>
int launch_transpose_permute(const void* in_bs, void* out_sb, const int* perm, int B, int64_t N,
                             cudaStream_t st);
template <typename R>
int launch_transpose_unpermute(const void* in_sb, void* out_bs, const int* order, int B, int64_t N,
                               cudaStream_t st);
// Y[b][m] = S_(w) X (vals = S.val or SW_val): the row-segment kernel for a
// complex64 32-vector batch, else the row-gather kernel.  X [s'][b] (patch
// order, columns renumbered) or, for _sample, X [s][b] (sample order).
template <typename R>
int launch_spmm_s(sptb_plan* p, const void* vals, const void* x_sb, void* y_bm, int B, cudaStream_t st);
template <typename R>
int launch_spmm_s_sample(sptb_plan* p, const void* vals, const void* x_sb, void* y_bm, int B,
                         cudaStream_t st);
// S with columns renumbered to the patch order s'
inline DevCSR s_permuted(const sptb_plan* p) {
    DevCSR A = p->S;
    A.col = p->shp.s_colp;
    return A;
}

// fused detector-axis FFTs (sptb_fft.cu): caller slices -> FFT1 -> [s'][b], and back
bool fft1_fused_ok(const sptb_plan* p, int fmt, int B);
// permute: rows perm[s] (the patch order s') for S with renumbered columns;
// false: rows in sample order s for S with its original columns
int launch_fft1_fwd(sptb_plan* p, const void* in, int fmt, int64_t n, int64_t u0, int nb, int B, void* q,
                    cudaStream_t st, bool permute = true);
int launch_fft1_inv(sptb_plan* p, const void* q, int B, void* out, int fmt, int64_t n, int64_t u0, int nb,
                    cudaStream_t st);
// forward FFT1 of caller real pairs -> q [s][b] (sample order) by TMA stores
bool fft1_fwd_tma_ok(const sptb_plan* p, const void* in, const void* q, int fmt, int B);
int launch_fft1_fwd_tma(sptb_plan* p, const void* in, int64_t n, int64_t u0, int nb, int B, void* q,
                        cudaStream_t st);
// inverse FFT1 of rows in sample order (q [s][b]) staged by TMA -> caller real pairs
bool fft1_inv_tma_ok(const sptb_plan* p, const void* q, const void* out, int fmt, int B);
int launch_fft1_inv_tma(sptb_plan* p, const void* q, int B, void* out, int64_t n, int64_t u0, int nb,
                        cudaStream_t st);
// 2-D inverse FFT of G [b][y][x] (in place along y) fused with the
// deapodization and unpack to caller real slice pairs (sptb_fft.cu)
bool fft2_fused_ok(const sptb_plan* p, int fmt);
int launch_fft2_inv_unpack(sptb_plan* p, void* g, const void* plane, double scale, void* out, int64_t n,
                           int64_t u0, int nb, cudaStream_t st);
// in-place unnormalised 2-D FFT of nb planes (solver grids), complex64 only
bool fft2_inplace_ok(const sptb_plan* p, const void* g);
const float2* fft2_twiddles(sptb_plan* p, int logn);
int fft2_log2(long long n);  // log2 n for 512 <= n = 2^k <= 4096, else 0
int launch_fft2_cols(sptb_plan* p, void* g, int nb, bool inverse, cudaStream_t st);
int launch_fft2_inplace(sptb_plan* p, void* g, int nb, bool inverse, cudaStream_t st);
// caller real pairs times plane -> forward 2-D FFT -> G [b][y][x], B planes
int launch_fft2_pack_fwd(sptb_plan* p, const void* in, const void* plane, int64_t n, int64_t u0, int nb, int B,
                         void* g, cudaStream_t st);
// pack caller slices -> complex [b][len] (optionally times a real plane)
// unpack complex [b][len] -> caller slices, times plane (optional) * scale
template <typename R>
int launch_pack(const void* in, int fmt, int64_t n, int64_t u0, int nb, int B,
                int64_t len, const void* plane, void* out, cudaStream_t st);
template <typename R>
int launch_unpack(const void* in, int64_t len, const void* plane, double scale,
                  void* out, int fmt, int64_t n, int64_t u0, int nb, cudaStream_t st);
// multiply [b][t][p] by real weights indexed p (len P) or s (len T*P)
template <typename R>
int launch_weight_sino(void* z, const void* w, int64_t wlen, int P, int64_t N, int B,
                       cudaStream_t st);
template <typename R>
int launch_permute_grid(const void* in, void* out, int X, int Y, int B, bool f_to_c,
                        cudaStream_t st);

}  // namespace sptb
