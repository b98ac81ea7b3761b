// common.cuh -- constants, camera parameters and the shared per-(pixel,
// splat) evaluation used by BOTH the forward and backward rasterizers.
//
// The backward pass replays the forward's skip/clamp decisions
// (sg/raster_backward.py:64-71 mirrors sg/raster_forward.py:130-137), so the
// sigma/alpha arithmetic lives in exactly one function here, written with
// explicit round-to-nearest intrinsics so nvcc cannot contract it
// differently in the two kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/splat_b200.h"

namespace gs {

constexpr int TILE = GS_TILE_SIZE;             // sg/binning.py:8
constexpr int TILE_PIX = TILE * TILE;
constexpr float DILATION = 0.3f;               // sg/projection.py:17
constexpr float ALPHA_MIN = 1.0f / 255.0f;     // sg/raster_forward.py:21
constexpr float ALPHA_MAX = 0.999f;            // sg/raster_forward.py:22
constexpr float T_MIN = 1e-4f;                 // sg/raster_forward.py:25
constexpr float SIGMA_CUT = 4.5f;              // sg/raster_forward.py:30
constexpr float QUAT_EPS = 1e-12f;             // sg/core.py:13
constexpr double QUAT_EPS_D = 1e-12;           // (float64 helpers, ops64.cu)
constexpr double DILATION_D = 0.3;
constexpr float NEG_LOG2E = -1.4426950408889634f;
constexpr int MAX_RADIUS = 1 << 24;            // clamp so int math cannot overflow

// Kernel-side camera: rotation/translation split out of the 4x4 view.
struct CamK {
    float R[9];  // row-major R_cw
    float t[3];
    float fx, fy, cx, cy;
    int W, H;
    float near_plane, far_plane;
    int tiles_x, tiles_y;
};

inline CamK make_camk(const gs_camera& c) {
    CamK k;
    for (int r = 0; r < 3; ++r) {
        for (int q = 0; q < 3; ++q) k.R[3 * r + q] = c.view[4 * r + q];
        k.t[r] = c.view[4 * r + 3];
    }
    k.fx = c.fx; k.fy = c.fy; k.cx = c.cx; k.cy = c.cy;
    k.W = c.width; k.H = c.height;
    k.near_plane = c.near_plane; k.far_plane = c.far_plane;
    k.tiles_x = (c.width + TILE - 1) / TILE;
    k.tiles_y = (c.height + TILE - 1) / TILE;
    return k;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// sigma = 0.5*(A dx^2 + C dy^2) + B dx dy   (sg/raster_forward.py:132-135)
// evaluated as (hC*dy + B*dx)*dy + (hA*dx)*dx with hA = A/2, hC = C/2
// (exact halvings), every op rounded explicitly.  The packed form computes
// (hA*dx, B*dx) with one FMUL2 from the staged (hA, B) pair.
__device__ __forceinline__ float splat_sigma(float dx, float dy, float hA, float B, float hC) {
    const float t = __fmaf_rn(hC, dy, __fmul_rn(dx, B));
    return __fmaf_rn(t, dy, __fmul_rn(__fmul_rn(dx, hA), dx));
}

// Same expression with hA*dx hoisted (pixels sharing a column share dx):
// bit-identical to splat_sigma(dx, dy, hA, B, hC) when hAdx == dx*hA.
__device__ __forceinline__ float splat_sigma_h(float dx, float hAdx, float dy, float B, float hC) {
    return __fmaf_rn(__fmaf_rn(hC, dy, __fmul_rn(dx, B)), dy, __fmul_rn(hAdx, dx));
}

// ---- packed fp32 pairs (sm_100a FFMA2/FMUL2/FADD2) ----------------------
// Two pixels of one column are evaluated with one f32x2 instruction per op;
// a scalar operand is broadcast for free.  Per lane the rounding is that of
// the scalar op, so splat_sigma2 == (splat_sigma_h(lo), splat_sigma_h(hi))
// bit for bit.
typedef unsigned long long f32x2;

__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(f32x2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 bc2(float v) { return pk2(v, v); }
__device__ __forceinline__ float lo2(f32x2 v) {
    float a, b;
    upk2(v, a, b);
    return a;
}
__device__ __forceinline__ float hi2(f32x2 v) {
    float a, b;
    upk2(v, a, b);
    return b;
}
__device__ __forceinline__ f32x2 sel2(bool plo, bool phi, f32x2 a, f32x2 b) {  // per lane: p ? a : b
    float alo, ahi, blo, bhi;
    upk2(a, alo, ahi);
    upk2(b, blo, bhi);
    return pk2(plo ? alo : blo, phi ? ahi : bhi);
}
__device__ __forceinline__ f32x2 pin2(f32x2 x) {
    asm volatile("" : "+l"(x));
    return x;
}

// (hA*dx, B*dx) for a column: one FMUL2 from the staged (hA, B) pair.
__device__ __forceinline__ f32x2 sigma_base(float dx, float hA, float B) { return mul2(pk2(dx, dx), pk2(hA, B)); }

// sigma for the pixel pair dy = (dy_lo, dy_hi) sharing dx, from
// base = sigma_base(dx, hA, B): per lane bit-identical to splat_sigma.
__device__ __forceinline__ f32x2 splat_sigma2(float dx, f32x2 base, f32x2 dy, float hC, f32x2* t_out = nullptr) {
    const f32x2 t = fma2(pk2(hC, hC), dy, pk2(hi2(base), hi2(base)));
    if (t_out) *t_out = t;
    const float c0 = __fmul_rn(lo2(base), dx);
    return fma2(t, dy, pk2(c0, c0));
}

// det of the 2d covariance and its inverse terms (A, B, C)
// (sg/raster_forward.py:86-92), shared by the projection kernel and the
// per-pixel API so both produce the same conic bit for bit.
__device__ __forceinline__ float cov2d_det(float ca, float cb, float cc) {
    return __fmaf_rn(ca, cc, -__fmul_rn(cb, cb));
}
__device__ __forceinline__ float4 conic_of(float ca, float cb, float cc, float det, float opacity) {
    const float idet = __fdiv_rn(1.f, det);
    return make_float4(__fmul_rn(cc, idet), -__fmul_rn(cb, idet), __fmul_rn(ca, idet), opacity);
}

// exp(-sigma) shared by forward and backward (sg/raster_forward.py:136,
// sg/raster_backward.py:68).
__device__ __forceinline__ float splat_exp_neg(float sigma) {
    return ex2_approx(__fmul_rn(sigma, NEG_LOG2E));
}

// Tile rectangle of a splat's closed bbox square, sg/binning.py:35-46.
// floor((m -/+ r)/16) is computed exactly as floor_div(floor(m) -/+ r, 16):
// m is fp32, r an integer, so no rounding can move a tile edge.
__device__ __forceinline__ void tile_rect(float mx, float my, int r, int tiles_x, int tiles_y,
                                          int& tx0, int& tx1, int& ty0, int& ty1) {
    const int fx = (int)floorf(mx), fy = (int)floorf(my);
    tx0 = max(0, (fx - r) >> 4);
    tx1 = min(tiles_x - 1, (fx + r) >> 4);
    ty0 = max(0, (fy - r) >> 4);
    ty1 = min(tiles_y - 1, (fy + r) >> 4);
}

// Warp-cooperative walk over 32 consecutive Gaussians' tile rects (lane =
// one Gaussian, rect tx0..tx1 x ty0..ty1, empty when tx1 < tx0): the warp
// takes the rects' tiles 32 at a time, each lane finding its entry's owner
// by binary search over the lanes' exclusive prefix and decoding the tile
// row-major; f(tiles[UNROLL], gaussians[UNROLL]) per step, tile 0xFFFFFFFF
// for no entry.
// TCOUNT_REPL replicas of the scatter binning's per-tile counters: Gaussian
// g counts (and later takes its slots) in replica (g >> 5) % TCOUNT_REPL, so
// the hot tiles' atomics spread over several L2 lines.
constexpr int TCOUNT_REPL = 8;
__device__ __forceinline__ uint32_t tcount_replica(uint32_t g) { return (g >> 5) & (TCOUNT_REPL - 1); }
// direct binning: slot-counter replicas per tile (<= TCOUNT_REPL), chosen per warp of Gaussians
#ifndef DIRECT_REPL
#define DIRECT_REPL 8
#endif
constexpr int DREPL = DIRECT_REPL;
__device__ __forceinline__ uint32_t direct_replica(uint32_t g) { return (g >> 5) & (DREPL - 1); }

// Per entry f(tile, gaussian); UNROLL entries per lane per step (independent
// atomics in flight).
template <int UNROLL = 1, typename F>
__device__ __forceinline__ void walk_tile_rects(int lane, uint32_t g, int tx0, int tx1, int ty0, int ty1,
                                                int tiles_x, F&& f) {
    const int w = tx1 - tx0 + 1;
    const uint32_t cnt = (uint32_t)(w * (ty1 - ty0 + 1));
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const float rw = w > 0 ? 1.f / (float)w : 0.f;
    for (uint32_t t0 = 0; t0 < total; t0 += 32 * UNROLL) {
        uint32_t tl[UNROLL], gl[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const uint32_t t = t0 + 32 * u + lane;
            int L = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t e = __shfl_sync(0xffffffffu, excl, L + step);
                if (e <= t) L += step;
            }
            const uint32_t j = t - __shfl_sync(0xffffffffu, excl, L);
            const int ow = __shfl_sync(0xffffffffu, w, L);
            const float orw = __shfl_sync(0xffffffffu, rw, L);
            const int otx0 = __shfl_sync(0xffffffffu, tx0, L), oty0 = __shfl_sync(0xffffffffu, ty0, L);
            gl[u] = __shfl_sync(0xffffffffu, g, L);
            int row = (int)((float)j * orw);
            if (row * ow > (int)j) --row;
            if ((row + 1) * ow <= (int)j) ++row;
            tl[u] = t < total ? (uint32_t)((oty0 + row) * tiles_x + otx0 + ((int)j - row * ow)) : 0xFFFFFFFFu;
        }
        f(tl, gl);
    }
}

__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}

// Shared-memory histogram update for one digit per lane: when every valid
// lane of the warp holds the same digit (typical for high key bytes) one
// lane adds the count, otherwise each valid lane adds 1 (cheaper than
// match_any aggregation on sm_100a).
__device__ __forceinline__ void warp_hist_add(uint32_t* h, uint32_t d, bool valid) {
    const uint32_t vm = __ballot_sync(0xffffffffu, valid);
    if (!vm) return;
    const int leader = __ffs(vm) - 1;
    const uint32_t d0 = __shfl_sync(0xffffffffu, d, leader);
    if (__all_sync(0xffffffffu, !valid || d == d0)) {
        if ((int)(threadIdx.x & 31) == leader) atomicAdd(&h[d0], (uint32_t)__popc(vm));
    } else if (valid) {
        atomicAdd(&h[d], 1u);
    }
}

// The same update aggregated with match_any: one atomic per distinct digit
// of the warp (for concentrated digits, where per-lane atomics serialise on
// a few addresses).
__device__ __forceinline__ void warp_hist_add_match(uint32_t* h, uint32_t d, bool valid) {
    const uint32_t peers = __match_any_sync(0xffffffffu, valid ? d : 0xFFFFFFFFu);
    if (valid && (peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0u) atomicAdd(&h[d], (uint32_t)__popc(peers));
}

// Shared-memory access through 32-bit shared-window addresses computed once
// (keeps nvcc from re-deriving generic->shared conversions in hot loops).
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a)
                 : "memory");
    return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace gs

// error plumbing shared by the extern "C" entry points (defined in abi.cu)
namespace gs {
int set_error(const char* fmt, ...);
int check_launch(const char* what);

// Programmatic dependent launch: the frame path's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization so a kernel's CTAs can
// be scheduled while its predecessor drains; each such kernel starts with
// griddep_wait() (griddepcontrol.wait: returns once the predecessor grid
// has completed and its memory is visible; a no-op for a normal launch).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();  // GS_PDL=0 disables (abi.cu)

// Buffers a kernel clears for the kernels after it (16-byte units), so a
// frame needs no memset nodes (they would break the launch chain).
struct ZeroJobs {
    uint4* p[3];
    unsigned long long n16[3];
    // job 2 runs only when *cond2 != 0 (null: always) -- the frame path's
    // backward accumulators, zeroed only when the workspace is not known clean
    const unsigned long long* cond2;
};

__device__ __forceinline__ void run_zero_jobs(const ZeroJobs& zj) {
    const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        if (j == 2 && zj.cond2 && *zj.cond2 == 0ull) continue;
        for (unsigned long long k = tid; k < zj.n16[j]; k += stride) zj.p[j][k] = make_uint4(0u, 0u, 0u, 0u);
    }
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
}  // namespace gs
