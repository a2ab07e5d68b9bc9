#include <cufftXt.h>
struct CbInfo {
    const float* in;      // caller real slices [slice][T][P]
    int n_slices, T, P, B;
    const int* perm;      // s -> s'
    float2* q;            // [s'][B]
};
// input layout seen by cuFFT: [t][b][p]
extern "C" __device__ cufftComplex cb_load_pack(void* dataIn, unsigned long long offset, void* callerInfo, void* sp) {
    const CbInfo* ci = (const CbInfo*)callerInfo;
    const unsigned o = (unsigned)offset;
    const unsigned P = ci->P, B = ci->B;
    const unsigned p = o % P, tb = o / P, b = tb % B, t = tb / B;
    const size_t plane = (size_t)ci->T * P;
    const size_t rel = (size_t)t * P + p;
    cufftComplex v;
    const int s0 = 2 * b;
    v.x = s0 < ci->n_slices ? ci->in[s0 * plane + rel] : 0.f;
    v.y = s0 + 1 < ci->n_slices ? ci->in[(s0 + 1) * plane + rel] : 0.f;
    return v;
}
extern "C" __device__ void cb_store_perm(void* dataOut, unsigned long long offset, cufftComplex e, void* callerInfo, void* sp) {
    const CbInfo* ci = (const CbInfo*)callerInfo;
    const unsigned o = (unsigned)offset;
    const unsigned P = ci->P, B = ci->B;
    const unsigned p = o % P, tb = o / P, b = tb % B, t = tb / B;
    const int sp2 = ci->perm[t * P + p];
    ci->q[(size_t)sp2 * B + b] = make_float2(e.x, e.y);
}
