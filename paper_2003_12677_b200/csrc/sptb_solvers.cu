// Device-resident solvers (placeholder until the fused solver kernels land).
#include "sptb_internal.cuh"

using namespace sptb;

extern "C" int sptb_solve(sptb_plan* p, const sptb_solver_config* cfg, const void* sino,
                          int32_t in_fmt, void* rec, int32_t out_fmt, int64_t n, double* hist,
                          int32_t* iters, int32_t* converged, int32_t* status) {
    (void)p; (void)cfg; (void)sino; (void)in_fmt; (void)rec; (void)out_fmt; (void)n;
    (void)hist; (void)iters; (void)converged; (void)status;
    return fail(SPTB_ERR_STATE, "sptb_solve: not implemented yet");
}
