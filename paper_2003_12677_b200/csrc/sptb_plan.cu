// Plan lifecycle and the operator entry points of the C ABI (include/sptb.h).
#include "sptb_internal.cuh"

#include <cstdlib>
#include <mutex>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <vector>

namespace sptb {

// ---------------------------------------------------------------- switches
namespace {
Switches g_switches;
bool g_switches_read = false;
bool env_on(const char* name) {
    const char* e = getenv(name);
    return e && e[0] && e[0] != '0';
}
int env_int(const char* name) {
    const char* e = getenv(name);
    return e ? atoi(e) : 0;
}
}  // namespace

void reload_switches() {
    Switches s;
    s.no_tma = env_on("SPTB_NO_TMA");
    s.no_fused_fft1 = env_on("SPTB_NO_FUSED_FFT1");
    s.no_fused_fft2 = env_on("SPTB_NO_FUSED_FFT2");
    s.fft2_no_persist = env_on("SPTB_FFT2_NO_PERSIST");
    s.fft2_no_bulk = env_on("SPTB_FFT2_NO_BULK");
    s.fft1_stockham = env_on("SPTB_FFT1_STOCKHAM");
    s.fft1_no_bulk = env_on("SPTB_FFT1_NO_BULK");
    s.fft1_inv_gather = env_on("SPTB_FFT1_INV_GATHER");
    s.fft1_fwd_rows = env_on("SPTB_FFT1_FWD_ROWS");
    s.fft1_perm = env_on("SPTB_FFT1_PERM");
    s.sirt_unfused = env_on("SPTB_SIRT_UNFUSED");
    s.xpass_unfused = env_on("SPTB_XPASS_UNFUSED");
    s.spmm_rows = env_on("SPTB_SPMM_ROWS");
    s.no_graph = env_on("SPTB_NO_GRAPH");
    s.pipe_chunks = std::max(0, env_int("SPTB_PIPE_CHUNKS"));
    if (const char* e = getenv("SPTB_PIPE_SIZES")) {  // "1,2,4,..." (the last size repeats)
        for (const char* q = e; *q;) {
            const int v = atoi(q);
            if (v > 0) s.pipe_sizes.push_back(v);
            while (*q && *q != ',') ++q;
            if (*q == ',') ++q;
        }
    }
    g_switches = s;
    g_switches_read = true;
}

const Switches& switches() {
    if (!g_switches_read) reload_switches();
    return g_switches;
}


static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};
static std::atomic<long long> g_ffts{0};
void count_fft(int n) { g_ffts += n; }

void set_error(const std::string& m) { g_err = m; }
int fail(int code, const std::string& m) {
    g_err = m;
    return code;
}
void count_launch(int n) { g_launches += n; }

int is_device_ptr(const void* ptr, bool* dev) {
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *dev = false;
        return SPTB_OK;
    }
    *dev = (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
    return SPTB_OK;
}

cudaError_t set_smem_once(const void* func, int bytes, int carveout) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    static std::map<const void*, int> done;
    auto it = done.find(func);
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && carveout >= 0)
        e = cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
    if (e == cudaSuccess) done[func] = bytes;
    return e;
}

int ensure_stage(void** buf, size_t* have, size_t need) {
    if (*have >= need) return SPTB_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *have = 0;
    SPTB_CUDA(cudaMalloc(buf, need));
    *have = need;
    return SPTB_OK;
}

// Operator work buffers sized for B complex vectors; grown on demand.
int ensure_work(sptb_plan* p, int B) {
    if (p->work_B >= B) return SPTB_OK;
    for (void** b : {&p->G0, &p->G1, &p->S0, &p->S1}) {
        if (*b) cudaFree(*b);
        *b = nullptr;
    }
    p->work_B = 0;
    const size_t gb = p->csize * (size_t)B * p->M;
    const size_t sb = p->csize * (size_t)B * p->N;
    if (cudaMalloc(&p->G0, gb) != cudaSuccess || cudaMalloc(&p->G1, gb) != cudaSuccess ||
        cudaMalloc(&p->S0, sb) != cudaSuccess || cudaMalloc(&p->S1, sb) != cudaSuccess) {
        cudaGetLastError();
        return fail(SPTB_ERR_OOM, "work buffers: out of device memory");
    }
    p->work_B = B;
    return SPTB_OK;
}

int get_fft(sptb_plan* p, int B, FFTPlans** out) {
    auto it = p->ffts.find(B);
    if (it != p->ffts.end()) {
        *out = &it->second;
        return SPTB_OK;
    }
    FFTPlans f;
    const cufftType ty = p->prec == SPTB_PREC_F64 ? CUFFT_Z2Z : CUFFT_C2C;
    int n2[2] = {p->Y, p->X};
    SPTB_CUFFT(cufftCreate(&f.fft2));
    size_t ws = 0;
    SPTB_CUFFT(cufftMakePlanMany(f.fft2, 2, n2, nullptr, 1, (int)p->M, nullptr, 1, (int)p->M, ty,
                                 B, &ws));
    SPTB_CUFFT(cufftSetStream(f.fft2, p->stream));
    int n1[1] = {p->P};
    SPTB_CUFFT(cufftCreate(&f.fft1));
    SPTB_CUFFT(cufftMakePlanMany(f.fft1, 1, n1, nullptr, 1, p->P, nullptr, 1, p->P, ty,
                                 B * p->T, &ws));
    SPTB_CUFFT(cufftSetStream(f.fft1, p->stream));
    p->ffts[B] = f;
    *out = &p->ffts[B];
    return SPTB_OK;
}

static int exec_fft(sptb_plan* p, cufftHandle h, void* z, int dir) {
    count_fft();
    if (p->prec == SPTB_PREC_F64)
        SPTB_CUFFT(cufftExecZ2Z(h, (cufftDoubleComplex*)z, (cufftDoubleComplex*)z, dir));
    else
        SPTB_CUFFT(cufftExecC2C(h, (cufftComplex*)z, (cufftComplex*)z, dir));
    return SPTB_OK;
}

static int pow2_at_least(int n) {
    int b = 1;
    while (b < n) b <<= 1;
    return b;
}

// ------------------------------------------------------------------ batching
// A call covers `units` complex vectors; REAL input pairs slices (2k, 2k+1).
struct Batch {
    int64_t u0;
    int nb, B;
};

static int64_t n_units(int fmt, int64_t n) { return (fmt & SPTB_FMT_COMPLEX) ? n : (n + 1) / 2; }

static size_t elem_bytes(int fmt) { return (fmt & SPTB_FMT_F64) ? 8 : 4; }

// caller slices covered by units [u0, u0+nb): first slice index and count
static void slice_range(int fmt, int64_t n, int64_t u0, int nb, int64_t* first, int64_t* cnt) {
    if (fmt & SPTB_FMT_COMPLEX) {
        *first = u0;
        *cnt = nb;
    } else {
        *first = 2 * u0;
        *cnt = std::min<int64_t>(2 * (u0 + nb), n) - 2 * u0;
    }
}
static size_t slice_bytes(int fmt, int64_t len) {
    return elem_bytes(fmt) * len * ((fmt & SPTB_FMT_COMPLEX) ? 2 : 1);
}

// Generic driver: host pointers are staged per batch through device buffers.
static int ensure_pipe(sptb_plan* p) {
    if (p->io_in) return SPTB_OK;
    SPTB_CUDA(cudaStreamCreateWithFlags(&p->io_in, cudaStreamNonBlocking));
    SPTB_CUDA(cudaStreamCreateWithFlags(&p->io_out, cudaStreamNonBlocking));
    for (int k = 0; k < sptb_plan::NPIPE; ++k) {
        SPTB_CUDA(cudaEventCreateWithFlags(&p->ev_in[k], cudaEventDisableTiming));
        SPTB_CUDA(cudaEventCreateWithFlags(&p->ev_comp[k], cudaEventDisableTiming));
        SPTB_CUDA(cudaEventCreateWithFlags(&p->ev_out[k], cudaEventDisableTiming));
    }
    SPTB_CUDA(cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming));
    return SPTB_OK;
}

// Generic driver over batches of `units` (complex vectors).  Device pointers:
// one pass per max_batch units on the plan stream.  Host pointers: the units
// are cut into >= 8 chunks and run as a three-stage pipeline -- H2D of chunk
// i+1 (io_in stream), compute of chunk i (plan stream), D2H of chunk i-1
// (io_out stream) -- through NPIPE rotating staging buffers, so the PCIe
// transfers in both directions overlap each other and the kernels.
template <typename F>
static int drive(sptb_plan* p, const void* in, int in_fmt, int64_t in_len, void* out,
                 int out_fmt, int64_t out_len, int64_t n, F&& body) {
    if ((in_fmt & SPTB_FMT_COMPLEX) != (out_fmt & SPTB_FMT_COMPLEX))
        return fail(SPTB_ERR_ARG, "output kind (real/complex) must match the input's");
    if (n < 0) return fail(SPTB_ERR_ARG, "negative slice count");
    if (n == 0) return SPTB_OK;
    bool din = true, dout = true;
    is_device_ptr(in, &din);
    is_device_ptr(out, &dout);
    const int64_t units = n_units(in_fmt, n);
    int64_t chunk = p->max_batch;
    std::vector<int64_t> sizes;  // host buffers: pipeline chunk sizes in units
    if (!din || !dout) {
        // split into pipeline chunks so H2D, kernels and D2H overlap.  The
        // first chunk's H2D and the last one's D2H stay exposed, so those two
        // are single units; the rest go in chunks of 4 units, the smallest
        // batch the fused FFT passes take (B % 4 == 0).  SPTB_PIPE_CHUNKS=k
        // overrides with k equal chunks.
        if (!switches().pipe_sizes.empty()) {
            const auto& ps = switches().pipe_sizes;
            for (int64_t u = 0, i = 0; u < units; ++i) {
                const int64_t c = std::min<int64_t>(std::min<int64_t>(ps[std::min<size_t>(i, ps.size() - 1)],
                                                                      p->max_batch), units - u);
                sizes.push_back(c);
                u += c;
            }
        } else if (switches().pipe_chunks > 0) {
            const int64_t c = std::max<int64_t>(1, std::min<int64_t>(
                p->max_batch, (units + switches().pipe_chunks - 1) / switches().pipe_chunks));
            for (int64_t u = 0; u < units; u += c) sizes.push_back(std::min(c, units - u));
        } else if (units >= 8 && p->max_batch >= 2) {
            // two single units, 2-unit chunks, three single units: PCIe-bound,
            // the finer grain keeps both copy directions busy (measured 22.55
            // ms per 64-slice step vs 23.29 with 4-unit chunks and the fused
            // B % 4 passes, scratch/e2e_sweep.sh)
            sizes = {1, 1};
            int64_t mid = units - 5;
            for (; mid >= 2; mid -= 2) sizes.push_back(2);
            if (mid) sizes.push_back(1);
            sizes.insert(sizes.end(), {1, 1, 1});
        } else {
            for (int64_t u = 0; u < units; ++u) sizes.push_back(1);
        }
        chunk = *std::max_element(sizes.begin(), sizes.end());
    }
    SPTB_TRY(ensure_work(p, pow2_at_least((int)std::min<int64_t>(chunk, units))));
    if (din && dout) {
        for (int64_t u0 = 0; u0 < units; u0 += chunk) {
            const int nb = (int)std::min<int64_t>(chunk, units - u0);
            SPTB_TRY(body(in, n, u0, out, n, u0, nb, pow2_at_least(nb)));
        }
        return SPTB_OK;
    }
    SPTB_TRY(ensure_pipe(p));
    const size_t sbi = slice_bytes(in_fmt, in_len), sbo = slice_bytes(out_fmt, out_len);
    SPTB_CUDA(cudaEventRecord(p->ev_start, p->stream));  // after earlier work on the plan stream
    SPTB_CUDA(cudaStreamWaitEvent(p->io_in, p->ev_start, 0));
    int64_t u0 = 0;
    for (size_t i = 0; i < sizes.size(); u0 += sizes[i], ++i) {
        const int k = (int)(i % sptb_plan::NPIPE);
        const int nb = (int)sizes[i];
        int64_t first, cnt;
        slice_range(in_fmt, n, u0, nb, &first, &cnt);
        const void* src = in;
        int64_t n_loc = n, u_loc = u0;
        if (!din) {
            SPTB_TRY(ensure_stage(&p->pin[k], &p->pin_bytes[k], sbi * cnt));
            if (i >= sptb_plan::NPIPE) SPTB_CUDA(cudaStreamWaitEvent(p->io_in, p->ev_comp[k], 0));
            SPTB_CUDA(cudaMemcpyAsync(p->pin[k], (const char*)in + sbi * first, sbi * cnt,
                                      cudaMemcpyHostToDevice, p->io_in));
            SPTB_CUDA(cudaEventRecord(p->ev_in[k], p->io_in));
            SPTB_CUDA(cudaStreamWaitEvent(p->stream, p->ev_in[k], 0));
            src = p->pin[k];
            n_loc = cnt;
            u_loc = 0;
        }
        void* dst = out;
        int64_t on_loc = n, ou_loc = u0;
        if (!dout) {
            SPTB_TRY(ensure_stage(&p->pout[k], &p->pout_bytes[k], sbo * cnt));
            if (i >= sptb_plan::NPIPE) SPTB_CUDA(cudaStreamWaitEvent(p->stream, p->ev_out[k], 0));
            dst = p->pout[k];
            on_loc = cnt;
            ou_loc = 0;
        }
        SPTB_TRY(body(src, n_loc, u_loc, dst, on_loc, ou_loc, nb, pow2_at_least(nb)));
        SPTB_CUDA(cudaEventRecord(p->ev_comp[k], p->stream));
        if (!dout) {
            SPTB_CUDA(cudaStreamWaitEvent(p->io_out, p->ev_comp[k], 0));
            SPTB_CUDA(cudaMemcpyAsync((char*)out + sbo * first, p->pout[k], sbo * cnt,
                                      cudaMemcpyDeviceToHost, p->io_out));
            SPTB_CUDA(cudaEventRecord(p->ev_out[k], p->io_out));
        }
    }
    SPTB_CUDA(cudaStreamSynchronize(p->stream));
    SPTB_CUDA(cudaStreamSynchronize(p->io_out));
    SPTB_CUDA(cudaStreamSynchronize(p->io_in));
    return SPTB_OK;
}

// ------------------------------------------------------------------ operators (typed)
template <typename R>
int radon_batch(sptb_plan* p, const void* in, int in_fmt, int64_t n, int64_t u0, int nb, int B,
                void* out, int out_fmt, int64_t on, int64_t ou0) {
    FFTPlans* f;
    SPTB_TRY(get_fft(p, B, &f));
    cudaStream_t st = p->stream;
    if (fft2_fused_ok(p, in_fmt)) {
        SPTB_TRY(launch_fft2_pack_fwd(p, in, p->deapo, n, u0, nb, B, p->G0, st));
    } else {
        SPTB_TRY(launch_pack<R>(in, in_fmt, n, u0, nb, B, p->M, p->deapo, p->G0, st));
        SPTB_TRY(exec_fft(p, f->fft2, p->G0, CUFFT_FORWARD));
    }
    // patch SpMM reads the batch-outer FFT2 output directly -> [s'][b], or
    // [s][b] (sample order) for the TMA-staged inverse FFT1
    const bool so = tma_ok(p, p->G0) && fft1_inv_tma_ok(p, p->S1, out, out_fmt, B);
    SPTB_TRY(launch_spmm_sh_patch<R>(p, p->G0, p->S1, B, nullptr, st, so));
    if (so) return launch_fft1_inv_tma(p, p->S1, B, out, on, ou0, nb, st);
    if (fft1_fused_ok(p, out_fmt, B))  // gather [s'][b] + IFFT1 + unpack in one pass
        return launch_fft1_inv(p, p->S1, B, out, out_fmt, on, ou0, nb, st);
    SPTB_TRY(launch_transpose_unpermute<R>(p->S1, p->S0, p->shp.order, B, p->N, st));
    SPTB_TRY(exec_fft(p, f->fft1, p->S0, CUFFT_INVERSE));
    return launch_unpack<R>(p->S0, p->N, nullptr, 1.0 / p->P, out, out_fmt, on, ou0, nb, st);
}

template <typename R>
int iradon_batch(sptb_plan* p, bool filtered, double scale, const void* in, int in_fmt,
                 int64_t n, int64_t u0, int nb, int B, void* out, int out_fmt, int64_t on,
                 int64_t ou0) {
    FFTPlans* f;
    SPTB_TRY(get_fft(p, B, &f));
    cudaStream_t st = p->stream;
    const void* vals = (filtered && p->SW_val) ? p->SW_val : p->S.val;
    if (fft1_fused_ok(p, in_fmt, B) && !switches().fft1_perm) {
        // pack + FFT1 in one pass, rows left in sample order: the row gather
        // of S reads them through its original column indices (no permutation)
        if (fft1_fwd_tma_ok(p, in, p->S1, in_fmt, B))
            SPTB_TRY(launch_fft1_fwd_tma(p, in, n, u0, nb, B, p->S1, st));
        else
            SPTB_TRY(launch_fft1_fwd(p, in, in_fmt, n, u0, nb, B, p->S1, st, false));
        SPTB_TRY(launch_spmm_s_sample<R>(p, vals, p->S1, p->G0, B, st));
    } else {
        if (fft1_fused_ok(p, in_fmt, B)) {  // pack + FFT1 + permute in one pass
            SPTB_TRY(launch_fft1_fwd(p, in, in_fmt, n, u0, nb, B, p->S1, st));
        } else {
            SPTB_TRY(launch_pack<R>(in, in_fmt, n, u0, nb, B, p->N, nullptr, p->S0, st));
            SPTB_TRY(exec_fft(p, f->fft1, p->S0, CUFFT_FORWARD));
            SPTB_TRY(launch_transpose_permute<R>(p->S0, p->S1, p->shp.perm, B, p->N, st));
        }
        SPTB_TRY(launch_spmm_s<R>(p, vals, p->S1, p->G0, B, st));
    }
    if (fft2_fused_ok(p, out_fmt))
        return launch_fft2_inv_unpack(p, p->G0, p->deapo, scale / p->P, out, on, ou0, nb, st);
    SPTB_TRY(exec_fft(p, f->fft2, p->G0, CUFFT_INVERSE));
    return launch_unpack<R>(p->G0, p->M, p->deapo, scale / p->P, out, out_fmt, on, ou0, nb, st);
}

template <typename R>
int weights_batch(sptb_plan* p, const void* w, int64_t wlen, const void* in, int in_fmt, int64_t n,
                  int64_t u0, int nb, int B, void* out, int out_fmt, int64_t on, int64_t ou0) {
    FFTPlans* f;
    SPTB_TRY(get_fft(p, B, &f));
    cudaStream_t st = p->stream;
    SPTB_TRY(launch_pack<R>(in, in_fmt, n, u0, nb, B, p->N, nullptr, p->S0, st));
    SPTB_TRY(exec_fft(p, f->fft1, p->S0, CUFFT_FORWARD));
    if (wlen) SPTB_TRY(launch_weight_sino<R>(p->S0, w, wlen, p->P, p->N, B, st));
    SPTB_TRY(exec_fft(p, f->fft1, p->S0, CUFFT_INVERSE));
    return launch_unpack<R>(p->S0, p->N, nullptr, 1.0 / p->P, out, out_fmt, on, ou0, nb, st);
}

#define DISPATCH(p, fn, ...) \
    ((p)->prec == SPTB_PREC_F64 ? fn<double>(__VA_ARGS__) : fn<float>(__VA_ARGS__))

int op_radon(sptb_plan* p, const void* in, int in_fmt, void* out, int out_fmt, int64_t n) {
    return drive(p, in, in_fmt, p->M, out, out_fmt, p->N, n,
                 [&](const void* s, int64_t nl, int64_t ul, void* d, int64_t onl, int64_t oul,
                     int nb, int B) {
                     return DISPATCH(p, radon_batch, p, s, in_fmt, nl, ul, nb, B, d, out_fmt, onl, oul);
                 });
}

int op_iradon(sptb_plan* p, bool filtered, double scale, const void* in, int in_fmt, void* out,
              int out_fmt, int64_t n) {
    return drive(p, in, in_fmt, p->N, out, out_fmt, p->M, n,
                 [&](const void* s, int64_t nl, int64_t ul, void* d, int64_t onl, int64_t oul,
                     int nb, int B) {
                     return DISPATCH(p, iradon_batch, p, filtered, scale, s, in_fmt, nl, ul, nb, B,
                                     d, out_fmt, onl, oul);
                 });
}

}  // namespace sptb

using namespace sptb;

extern "C" {

const char* sptb_last_error(void) { return g_err.c_str(); }
int32_t sptb_version(void) { return 1; }
int64_t sptb_launch_count(void) { return g_launches.load(); }
int64_t sptb_fft_count(void) { return g_ffts.load(); }

int sptb_plan_create(sptb_plan** out, const sptb_geometry* g, const sptb_kernel* k,
                     int32_t precision, int32_t max_batch, int32_t device, double threshold) {
    if (!out || !g || !k) return fail(SPTB_ERR_ARG, "null argument");
    *out = nullptr;
    if (g->n_p < 2 || g->n_theta < 1 || g->n_x < 2 || g->n_y < 2)
        return fail(SPTB_ERR_ARG, "invalid geometry sizes");
    if (!g->cos_theta || !g->sin_theta) return fail(SPTB_ERR_ARG, "missing angle tables");
    if (k->width < 1 || k->width % 2 == 0) return fail(SPTB_ERR_ARG, "kernel width must be odd");
    if (k->family != SPTB_KERNEL_KB && k->family != SPTB_KERNEL_GAUSS)
        return fail(SPTB_ERR_ARG, "unknown kernel family");
    if (precision != SPTB_PREC_F32 && precision != SPTB_PREC_F64)
        return fail(SPTB_ERR_ARG, "precision must be SPTB_PREC_F32 or SPTB_PREC_F64");
    if (max_batch < 1 || max_batch > 64 || (max_batch & (max_batch - 1)))
        return fail(SPTB_ERR_ARG, "max_batch must be a power of two in [1, 64]");
    const long long M = (long long)g->n_x * g->n_y, N = (long long)g->n_theta * g->n_p;
    if (M * 64 >= (1LL << 31) * 64 || N >= (1LL << 31) || M * k->width * k->width >= (1LL << 31))
        return fail(SPTB_ERR_ARG, "geometry exceeds int32 indexing");
    SPTB_CUDA(cudaSetDevice(device));
    sptb_plan* p = new sptb_plan();
    p->device = device;
    p->prec = precision;
    p->csize = precision == SPTB_PREC_F64 ? 16 : 8;
    p->P = g->n_p;
    p->T = g->n_theta;
    p->X = g->n_x;
    p->Y = g->n_y;
    p->M = M;
    p->N = N;
    p->center = g->center;
    p->max_batch = max_batch;
    p->threshold = threshold;
    int rc = build_matrices(p, g, k);
    if (rc != SPTB_OK) {
        std::string m = g_err;
        sptb_plan_destroy(p);
        return fail(rc, m);
    }
    *out = p;
    return SPTB_OK;
}

int sptb_reload_switches(void) {
    sptb::reload_switches();
    return SPTB_OK;
}

int sptb_plan_destroy(sptb_plan* p) {
    if (!p) return SPTB_OK;
    cudaSetDevice(p->device);
    for (auto& kv : p->ffts) {
        if (kv.second.fft2) cufftDestroy(kv.second.fft2);
        if (kv.second.fft1) cufftDestroy(kv.second.fft1);
    }
    void* bufs[] = {p->S.row_ptr, p->S.col, p->S.val, p->SH.row_ptr, p->SH.col, p->SH.val,
                    p->SW_val, p->w_dev, p->deapo, p->deapo_xy, p->G0, p->G1, p->G2, p->S0, p->S1,
                    p->stage_in, p->stage_out, p->red, p->fft_work,
                    p->shp.items, p->shp.rp, p->shp.meta, p->shp.perm, p->shp.order,
                    p->shp.s_colp, p->shp.sval, p->shp.item_perm, p->sseg.tiles,
                    p->sseg.longs, p->sseg.pairs, p->sseg.tile_e, p->sseg.prp, p->sseg.pcol[0], p->sseg.pcol[1],
                    p->sseg.pval[0], p->sseg.pval[1], p->wspec_dev, p->tw1};
    for (void* b : bufs)
        if (b) cudaFree(b);
    for (void* b : p->twn)
        if (b) cudaFree(b);
    for (int k = 0; k < sptb_plan::NPIPE; ++k) {
        if (p->pin[k]) cudaFree(p->pin[k]);
        if (p->pout[k]) cudaFree(p->pout[k]);
        if (p->ev_in[k]) cudaEventDestroy(p->ev_in[k]);
        if (p->ev_comp[k]) cudaEventDestroy(p->ev_comp[k]);
        if (p->ev_out[k]) cudaEventDestroy(p->ev_out[k]);
    }
    if (p->ev_start) cudaEventDestroy(p->ev_start);
    if (p->io_in) cudaStreamDestroy(p->io_in);
    if (p->io_out) cudaStreamDestroy(p->io_out);
    for (void* b : p->extra)
        if (b) cudaFree(b);
    for (auto& kv : p->pool) cudaFree(kv.second);
    if (p->solver_pinned) cudaFreeHost(p->solver_pinned);
    for (auto& e : p->solver_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : p->solver_join)
        if (e) cudaEventDestroy(e);
    if (p->solver_stream) cudaStreamDestroy(p->solver_stream);
    delete p;
    return SPTB_OK;
}

int sptb_plan_set_stream(sptb_plan* p, void* stream) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    p->stream = (cudaStream_t)stream;
    for (auto& kv : p->ffts) {
        SPTB_CUFFT(cufftSetStream(kv.second.fft2, p->stream));
        SPTB_CUFFT(cufftSetStream(kv.second.fft1, p->stream));
    }
    return SPTB_OK;
}

int sptb_plan_set_filter(sptb_plan* p, const double* w, int64_t nw) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    if (nw != 0 && nw != p->P && nw != p->N)
        return fail(SPTB_ERR_SHAPE, "filter weights fit neither (n_p,) nor (N,)");
    for (int64_t i = 0; i < nw; ++i)
        if (!(w[i] >= 0) || !std::isfinite(w[i]))
            return fail(SPTB_ERR_ARG, "filter weights must be finite and >= 0");
    cudaSetDevice(p->device);
    p->w_host.assign(w, w + nw);
    p->calib = 1.0;
    return fold_filter(p);
}

int sptb_plan_set_calibration(sptb_plan* p, double c) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    p->calib = c;
    return SPTB_OK;
}

int sptb_plan_calibrate(sptb_plan* p, double* out) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    cudaSetDevice(p->device);
    // flat disk -> radon -> filtered iradon (scale 1) -> mean over the disk
    const int X = p->X, Y = p->Y;
    const double r = std::min(X, Y) / 2.0;
    std::vector<double> disk((size_t)X * Y, 0.0);
    std::vector<char> mask((size_t)X * Y, 0);
    for (int y = 0; y < Y; ++y)
        for (int x = 0; x < X; ++x) {
            const double dy = y - Y / 2.0, dx = x - X / 2.0;
            if (dy * dy + dx * dx < r * r) {
                disk[(size_t)y * X + x] = 1.0;
                mask[(size_t)y * X + x] = 1;
            }
        }
    std::vector<double> sino((size_t)p->N), rec((size_t)p->M);
    SPTB_TRY(op_radon(p, disk.data(), SPTB_FMT_F64 | SPTB_FMT_REAL, sino.data(),
                      SPTB_FMT_F64 | SPTB_FMT_REAL, 1));
    SPTB_TRY(op_iradon(p, true, 1.0, sino.data(), SPTB_FMT_F64 | SPTB_FMT_REAL, rec.data(),
                       SPTB_FMT_F64 | SPTB_FMT_REAL, 1));
    double s = 0;
    long long c = 0;
    for (size_t i = 0; i < rec.size(); ++i)
        if (mask[i]) {
            s += rec[i];
            ++c;
        }
    const double mean = c ? s / c : 0.0;
    p->calib = (mean == 0.0) ? 1.0 : 1.0 / mean;
    if (out) *out = p->calib;
    return SPTB_OK;
}

int sptb_plan_matrix_info(sptb_plan* p, int32_t which, int64_t* rows, int64_t* cols,
                          int64_t* nnz) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    const DevCSR& A = (which == SPTB_MAT_SH) ? p->SH : p->S;
    if (rows) *rows = A.rows;
    if (cols) *cols = A.cols;
    if (nnz) *nnz = A.nnz;
    return SPTB_OK;
}

int sptb_plan_matrix_copy(sptb_plan* p, int32_t which, int32_t* rp, int32_t* ci, double* v) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    cudaSetDevice(p->device);
    const DevCSR& A = (which == SPTB_MAT_SH) ? p->SH : p->S;
    const void* vals = A.val;
    if (which == SPTB_MAT_SW) {
        if (!p->SW_val) return fail(SPTB_ERR_STATE, "no filter set");
        vals = p->SW_val;
    }
    SPTB_CUDA(cudaStreamSynchronize(p->stream));
    if (rp) SPTB_CUDA(cudaMemcpy(rp, A.row_ptr, sizeof(int) * (A.rows + 1), cudaMemcpyDeviceToHost));
    if (ci && A.nnz) SPTB_CUDA(cudaMemcpy(ci, A.col, sizeof(int) * A.nnz, cudaMemcpyDeviceToHost));
    if (v && A.nnz) {
        if (p->prec == SPTB_PREC_F64) {
            SPTB_CUDA(cudaMemcpy(v, vals, 16 * A.nnz, cudaMemcpyDeviceToHost));
        } else {
            std::vector<float> f(2 * A.nnz);
            SPTB_CUDA(cudaMemcpy(f.data(), vals, 8 * A.nnz, cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < f.size(); ++i) v[i] = f[i];
        }
    }
    return SPTB_OK;
}

int sptb_plan_deapo_copy(sptb_plan* p, double* out) {
    if (!p || !out) return fail(SPTB_ERR_ARG, "null argument");
    std::memcpy(out, p->deapo_host.data(), sizeof(double) * p->deapo_host.size());
    return SPTB_OK;
}

int sptb_radon(sptb_plan* p, const void* in, int32_t in_fmt, void* out, int32_t out_fmt,
               int64_t n) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    cudaSetDevice(p->device);
    return op_radon(p, in, in_fmt, out, out_fmt, n);
}

int sptb_radon_adjoint(sptb_plan* p, const void* in, int32_t in_fmt, void* out, int32_t out_fmt,
                       int64_t n) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    cudaSetDevice(p->device);
    return op_iradon(p, false, 1.0, in, in_fmt, out, out_fmt, n);
}

int sptb_iradon(sptb_plan* p, const void* in, int32_t in_fmt, void* out, int32_t out_fmt,
                int64_t n) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    cudaSetDevice(p->device);
    if (!p->SW_val) return op_iradon(p, false, 1.0, in, in_fmt, out, out_fmt, n);
    return op_iradon(p, true, p->calib, in, in_fmt, out, out_fmt, n);
}

int sptb_backproject(sptb_plan* p, int32_t filtered, double scale, const void* in,
                     int32_t in_fmt, void* out, int32_t out_fmt, int64_t n) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    if (filtered && !p->SW_val) return fail(SPTB_ERR_STATE, "plan has no filter");
    cudaSetDevice(p->device);
    return op_iradon(p, filtered != 0, scale, in, in_fmt, out, out_fmt, n);
}

int sptb_spectral_apply(sptb_plan* p, const double* w, int64_t nw, const void* in,
                        int32_t in_fmt, void* out, int32_t out_fmt, int64_t n) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    if (nw != p->P && nw != p->N)
        return fail(SPTB_ERR_SHAPE, "weights fit neither (n_p,) nor (N,)");
    cudaSetDevice(p->device);
    // the caller's weights go to a plan-owned buffer (sized once for N
    // entries, re-uploaded only when they change): no allocation per call
    const size_t rs = p->prec == SPTB_PREC_F64 ? 8 : 4;
    if (!p->wspec_dev) SPTB_CUDA(cudaMalloc(&p->wspec_dev, rs * (size_t)p->N));
    if (p->wspec_host.size() != (size_t)nw || !std::equal(w, w + nw, p->wspec_host.begin())) {
        p->wspec_host.assign(w, w + nw);
        if (rs == 8) {
            SPTB_CUDA(cudaMemcpyAsync(p->wspec_dev, p->wspec_host.data(), 8 * nw, cudaMemcpyHostToDevice,
                                      p->stream));
        } else {
            p->wspec_f32.resize(nw);
            for (int64_t i = 0; i < nw; ++i) p->wspec_f32[i] = (float)w[i];
            SPTB_CUDA(cudaMemcpyAsync(p->wspec_dev, p->wspec_f32.data(), 4 * nw, cudaMemcpyHostToDevice,
                                      p->stream));
        }
    }
    return drive(p, in, in_fmt, p->N, out, out_fmt, p->N, n,
                 [&](const void* s, int64_t nl, int64_t ul, void* d, int64_t onl, int64_t oul,
                     int nb, int B) {
                     return DISPATCH(p, weights_batch, p, p->wspec_dev, nw, s, in_fmt, nl, ul, nb, B, d,
                                     out_fmt, onl, oul);
                 });
}

int sptb_apply_weights(sptb_plan* p, const void* in, int32_t in_fmt, void* out, int32_t out_fmt,
                       int64_t n) {
    if (!p) return fail(SPTB_ERR_ARG, "null plan");
    cudaSetDevice(p->device);
    return drive(p, in, in_fmt, p->N, out, out_fmt, p->N, n,
                 [&](const void* s, int64_t nl, int64_t ul, void* d, int64_t onl, int64_t oul,
                     int nb, int B) {
                     return DISPATCH(p, weights_batch, p, p->w_dev, p->w_len, s, in_fmt, nl, ul, nb, B,
                                     d, out_fmt, onl, oul);
                 });
}

}  // extern "C"
