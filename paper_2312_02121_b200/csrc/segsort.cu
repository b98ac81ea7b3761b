// segsort.cu -- the per-tile sort of the scatter-binned lists as its own
// kernel (one CTA per tile; segsort.cuh).  The frame path normally runs the
// same code fused into the top of the raster forward instead
// (gs_set_option("fuse_sort", 0) selects this kernel).
#include "internal.cuh"
#include "segsort.cuh"

namespace gs {

__global__ void __launch_bounds__(WS_THREADS) segsort_kernel(const uint2* __restrict__ ranges,
                                                             const uint32_t* __restrict__ dkeys,
                                                             uint32_t* __restrict__ vals,
                                                             uint32_t* __restrict__ alt) {
    griddep_wait();
    __shared__ SegsortShared sh;
    segsort_tile(sh, ranges[blockIdx.x], dkeys, vals, alt);
}

int launch_segsort(const uint2* ranges, int n_tiles, const uint32_t* dkeys, uint32_t* vals, uint32_t* alt,
                   cudaStream_t s) {
    if (n_tiles <= 0) return 0;
    launch_k(segsort_kernel, dim3((unsigned)n_tiles), dim3(WS_THREADS), 0, s, ranges, dkeys, vals, alt);
    return check_launch("segsort_kernel");
}

}  // namespace gs
