// project.cu -- stage 1 (projection forward) and stage 5 (projection
// backward).  One thread per Gaussian; both kernels are HBM-bound
// (80 B/Gaussian forward, 104 B/Gaussian backward).
#include <cstdlib>

#include "common.cuh"
#include "internal.cuh"

namespace gs {

// sg/core.py:146-171 quat_to_rotmat (normalised, (w,x,y,z) order).
// Explicit roundings (no contraction left to the compiler): every kernel that
// forms R -- per view or once for all views -- gets the same bits.
__device__ __forceinline__ void quat_rot(float w, float x, float y, float z, float R[9]) {
    const float xx = __fmul_rn(x, x), yy = __fmul_rn(y, y), xy = __fmul_rn(x, y), xz = __fmul_rn(x, z),
                yz = __fmul_rn(y, z);
    R[0] = __fsub_rn(1.f, 2.f * __fmaf_rn(z, z, yy));
    R[1] = 2.f * __fmaf_rn(-w, z, xy);
    R[2] = 2.f * __fmaf_rn(w, y, xz);
    R[3] = 2.f * __fmaf_rn(w, z, xy);
    R[4] = __fsub_rn(1.f, 2.f * __fmaf_rn(z, z, xx));
    R[5] = 2.f * __fmaf_rn(-w, x, yz);
    R[6] = 2.f * __fmaf_rn(-w, y, xz);
    R[7] = 2.f * __fmaf_rn(w, x, yz);
    R[8] = __fsub_rn(1.f, 2.f * __fmaf_rn(y, y, xx));
}

// |q| with one fixed rounding sequence
__device__ __forceinline__ float quat_norm(float4 q) {
    return sqrtf(__fmaf_rn(q.w, q.w, __fmaf_rn(q.z, q.z, __fmaf_rn(q.y, q.y, __fmul_rn(q.x, q.x)))));
}

// a0 b0 + a1 b1 + a2 b2 with one fixed rounding sequence (no contraction
// left to the compiler, so every kernel computing it gets the same bits)
__device__ __forceinline__ float dot3_rn(float a0, float b0, float a1, float b1, float a2, float b2) {
    return __fmaf_rn(a2, b2, __fmaf_rn(a1, b1, __fmul_rn(a0, b0)));
}

__device__ __forceinline__ void report(unsigned long long* status, int i, int code) {
    atomicMin(status, ((unsigned long long)(unsigned)i << 8) | (unsigned long long)code);
}

// The projection split into its view-independent part and the per-view rest
// for the multi-view kernel (which reads and prepares a Gaussian once and
// runs the rest for every view).  project_fwd_kernel keeps the same
// operations inline (the split costs it register spills at its 32-register
// budget); the roundings that the compiler could otherwise contract
// differently in the two contexts are explicit (dot3_rn), so both give the
// same bits.
// View-independent part (sg/core.py:146-195): the scale / quaternion validity
// and M = R(q / |q|) diag(s).
struct FwdPrep {
    int err;  // 0, GS_ERR_SCALE or GS_ERR_QUAT
    float M[9];
};
__device__ __forceinline__ FwdPrep proj_fwd_prep(float4 q, float sx, float sy, float sz) {
    FwdPrep P;
    const float qn = quat_norm(q);
    P.err = (sx <= 0.f || sy <= 0.f || sz <= 0.f) ? GS_ERR_SCALE : (qn <= QUAT_EPS ? GS_ERR_QUAT : 0);
    if (P.err == 0) {
        const float inv = 1.f / qn;
        float R[9];
        quat_rot(q.x * inv, q.y * inv, q.z * inv, q.w * inv, R);
        // M = R diag(s)
        P.M[0] = R[0] * sx, P.M[1] = R[1] * sy, P.M[2] = R[2] * sz;
        P.M[3] = R[3] * sx, P.M[4] = R[4] * sy, P.M[5] = R[5] * sz;
        P.M[6] = R[6] * sx, P.M[7] = R[7] * sy, P.M[8] = R[8] * sz;
    }
    return P;
}

// The rest of sg/projection.py:115-145 for a Gaussian not culled by depth
// (camera-space mean t): errors -> Sigma' + 0.3 I -> pixel -> radius ->
// off-screen cull, plus the conic and the tile rect.
__device__ __forceinline__ void proj_fwd_core(const CamK& cam, int i, float tx, float ty, float tz, const FwdPrep& P,
                                              float op, unsigned long long* status, float4& o_xydr, float4& o_con,
                                              uint32_t& nt, float& ca, float& cb, float& cc, int& tx0, int& tx1,
                                              int& ty0, int& ty1) {
    if (P.err) {
        report(status, i, P.err);
        return;
    }
    const float* Rc = cam.R;
    const float* M = P.M;
    // T = J R_cw, J = [[fx/tz, 0, -fx tx/tz^2], [0, fy/tz, -fy ty/tz^2]]
    const float iz = 1.f / tz;
    const float j00 = cam.fx * iz, j02 = -cam.fx * tx * iz * iz;
    const float j11 = cam.fy * iz, j12 = -cam.fy * ty * iz * iz;
    float T0[3], T1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        T0[k] = __fmaf_rn(j02, Rc[6 + k], __fmul_rn(j00, Rc[k]));
        T1[k] = __fmaf_rn(j12, Rc[6 + k], __fmul_rn(j11, Rc[3 + k]));
    }
    // V = T M; Sigma' = V V^T + 0.3 I  (T Sigma T^T with Sigma = M M^T)
    float V0[3], V1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        V0[c] = dot3_rn(T0[0], M[c], T0[1], M[3 + c], T0[2], M[6 + c]);
        V1[c] = dot3_rn(T1[0], M[c], T1[1], M[3 + c], T1[2], M[6 + c]);
    }
    ca = __fadd_rn(dot3_rn(V0[0], V0[0], V0[1], V0[1], V0[2], V0[2]), DILATION);
    cb = dot3_rn(V0[0], V1[0], V0[1], V1[1], V0[2], V1[2]);
    cc = __fadd_rn(dot3_rn(V1[0], V1[0], V1[1], V1[1], V1[2], V1[2]), DILATION);
    if (fabsf(tz) < 1e-12f) {
        report(status, i, GS_ERR_HOMOG);
        return;
    }
    const float px = (cam.fx * (tx / tz) + 0.5f) + cam.cx;
    const float py = (cam.fy * (ty / tz) + 0.5f) + cam.cy;
    const float det = cov2d_det(ca, cb, cc);
    if (!(det > 0.f && ca + cc > 0.f)) {
        report(status, i, GS_ERR_COV2D);
        return;
    }
    const float mid = 0.5f * (ca + cc);
    const float lam = __fadd_rn(mid, sqrtf(__fmaf_rn(cb, cb, __fmul_rn(__fmul_rn(0.25f, ca - cc), ca - cc))));
    const float rf = ceilf(3.f * sqrtf(lam));
    const int r = rf < (float)MAX_RADIUS ? (int)rf : MAX_RADIUS;
    const float fr = (float)r;
    const bool off = (px + fr < 0.f) || (px - fr >= (float)cam.W) || (py + fr < 0.f) || (py - fr >= (float)cam.H);
    o_xydr = make_float4(px, py, tz, __int_as_float(off ? 0 : r));
    if (!off) {
        o_con = conic_of(ca, cb, cc, det, op);
        tile_rect(px, py, r, cam.tiles_x, cam.tiles_y, tx0, tx1, ty0, ty1);
        nt = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
    }
}

// sg/projection.py:115-145 project_gaussian for every Gaussian, in the
// reference's order of checks: depth cull (:124-125) -> scale/quat errors
// (sg/core.py:189-192) -> J (:64-82) -> Sigma' + 0.3 I (:85-96) -> pixel map
// through P (:45-61; equals fx*tx/tz + 0.5 + cx) -> radius (:99-112) ->
// off-screen cull (:131-137).  Plus the conic (sg/raster_forward.py:86-92)
// and the tile count of the bbox square (sg/binning.py:35-46).
// MODE 1 / 2 (frame path): also write the depth sort key of every Gaussian
// (float bits of the camera depth for visible ones, 0xFFFFFFFF for culled
// ones).  MODE 1 (depth-first binning) reduces the range [kmin, kmax] of the
// visible keys into meta[5] / meta[6] for the depth sort that follows
// (sort.cu: keys relative to kmin, culled ones dropped); MODE 2 (scatter binning) counts
// every tile's intersections instead (tcount, one red.add per pair); MODE 3
// (direct binning) takes a slot in the tile's fixed-stride bin for every
// pair (atomicAdd with return on one of the tile's DREPL counters, 4
// in flight per lane) and writes the Gaussian id there:
// bins[tile * kstride + replica * kr + slot], kr = kstride / DREPL
// (slots past kr are dropped; the raster forward reports the overflow).
#ifndef DIRECT_UNROLL
#define DIRECT_UNROLL 4  // slot atomics in flight per lane (direct binning)
#endif
#ifndef PFWD_MINB
#define PFWD_MINB 8  // 32 registers, 8 resident CTAs per SM (config 4 projection 165 -> 160 us)
#endif
// MODE 1 also histograms the depth keys' low byte: 40 registers (6 CTAs per
// SM) instead of a spill at 32
constexpr int pfwd_minb(int mode) { return mode == 1 ? 6 : PFWD_MINB; }
template <int MODE>
__global__ void __launch_bounds__(256, pfwd_minb(MODE)) project_fwd_kernel(
    const float* __restrict__ means, const float* __restrict__ scales, const float4* __restrict__ quats,
    const float* __restrict__ opac, int n, CamK cam, float4* __restrict__ xydr, float4* __restrict__ conic,
    uint32_t* __restrict__ tiles, float* __restrict__ cov_out, unsigned long long* __restrict__ status,
    uint32_t* __restrict__ dkeys, uint32_t* __restrict__ dhist, ZeroJobs zj, uint32_t* __restrict__ tcount,
    uint32_t* __restrict__ bins, uint32_t kstride) {
    constexpr bool DKEY = MODE != 0;
    griddep_wait();
    run_zero_jobs(zj);  // frame path: clear the later stages' counters / accumulators
    // MODE 1: the histogram of the visible depth keys' low byte (the depth
    // sort's first pass rotates it by the minimum's low byte: sort.cu)
    __shared__ uint32_t s_lo[MODE == 1 ? 256 : 1];
    if (MODE == 1) {
        for (int k = threadIdx.x; k < 256; k += blockDim.x) s_lo[k] = 0u;
        __syncthreads();
    }
    // MODE 1: the range [kmin, kmax] of the visible depth keys, so the depth
    // sort ranks keys relative to kmin and skips the passes above its width
    uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
    // grid-stride over Gaussians (warps stay converged for the histogram
    // vote); the shared histograms are flushed once per CTA
    const int n_round = (n + 31) & ~31;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += gridDim.x * blockDim.x) {
    uint32_t dkey = 0xFFFFFFFFu;
    int tx0 = 0, tx1 = -1, ty0 = 0, ty1 = -1;  // tile rect (MODE 2 / 3 walk it)
    if (i < n) {
    const float mx = means[3 * i], my = means[3 * i + 1], mz = means[3 * i + 2];
    // every input load is issued up front (one memory round trip; the culled
    // Gaussians' scale / quat / opacity reads are the price)
    const float sx = scales[3 * i], sy = scales[3 * i + 1], sz = scales[3 * i + 2];
    const float4 q = quats[i];
    const float op = opac[i];
    const float* Rc = cam.R;
    const float tx = Rc[0] * mx + Rc[1] * my + Rc[2] * mz + cam.t[0];
    const float ty = Rc[3] * mx + Rc[4] * my + Rc[5] * mz + cam.t[1];
    const float tz = Rc[6] * mx + Rc[7] * my + Rc[8] * mz + cam.t[2];
    float4 o_xydr = make_float4(0.f, 0.f, tz, __int_as_float(0));
    float4 o_con = make_float4(0.f, 0.f, 0.f, 0.f);
    float ca = 0.f, cb = 0.f, cc = 0.f;
    uint32_t nt = 0;
    const bool depth_culled = (tz <= cam.near_plane) || (tz >= cam.far_plane);
    if (!depth_culled) {
        const float qn = quat_norm(q);
        if (sx <= 0.f || sy <= 0.f || sz <= 0.f) {
            report(status, i, GS_ERR_SCALE);
        } else if (qn <= QUAT_EPS) {
            report(status, i, GS_ERR_QUAT);
        } else {
            const float inv = 1.f / qn;
            float R[9];
            quat_rot(q.x * inv, q.y * inv, q.z * inv, q.w * inv, R);
            // M = R diag(s)
            const float M[9] = {R[0] * sx, R[1] * sy, R[2] * sz, R[3] * sx, R[4] * sy,
                                R[5] * sz, R[6] * sx, R[7] * sy, R[8] * sz};
            // T = J R_cw, J = [[fx/tz, 0, -fx tx/tz^2], [0, fy/tz, -fy ty/tz^2]]
            const float iz = 1.f / tz;
            const float j00 = cam.fx * iz, j02 = -cam.fx * tx * iz * iz;
            const float j11 = cam.fy * iz, j12 = -cam.fy * ty * iz * iz;
            float T0[3], T1[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                T0[k] = __fmaf_rn(j02, Rc[6 + k], __fmul_rn(j00, Rc[k]));
                T1[k] = __fmaf_rn(j12, Rc[6 + k], __fmul_rn(j11, Rc[3 + k]));
            }
            // V = T M; Sigma' = V V^T + 0.3 I  (T Sigma T^T with Sigma = M M^T)
            float V0[3], V1[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                V0[c] = dot3_rn(T0[0], M[c], T0[1], M[3 + c], T0[2], M[6 + c]);
                V1[c] = dot3_rn(T1[0], M[c], T1[1], M[3 + c], T1[2], M[6 + c]);
            }
            ca = __fadd_rn(dot3_rn(V0[0], V0[0], V0[1], V0[1], V0[2], V0[2]), DILATION);
            cb = dot3_rn(V0[0], V1[0], V0[1], V1[1], V0[2], V1[2]);
            cc = __fadd_rn(dot3_rn(V1[0], V1[0], V1[1], V1[1], V1[2], V1[2]), DILATION);
            if (fabsf(tz) < 1e-12f) {
                report(status, i, GS_ERR_HOMOG);
            } else {
                const float px = (cam.fx * (tx / tz) + 0.5f) + cam.cx;
                const float py = (cam.fy * (ty / tz) + 0.5f) + cam.cy;
                const float det = cov2d_det(ca, cb, cc);
                if (!(det > 0.f && ca + cc > 0.f)) {
                    report(status, i, GS_ERR_COV2D);
                } else {
                    const float mid = 0.5f * (ca + cc);
                    const float lam = __fadd_rn(mid, sqrtf(__fmaf_rn(cb, cb, __fmul_rn(__fmul_rn(0.25f, ca - cc), ca - cc))));
                    const float rf = ceilf(3.f * sqrtf(lam));
                    const int r = rf < (float)MAX_RADIUS ? (int)rf : MAX_RADIUS;
                    const float fr = (float)r;
                    const bool off = (px + fr < 0.f) || (px - fr >= (float)cam.W) || (py + fr < 0.f) ||
                                     (py - fr >= (float)cam.H);
                    o_xydr = make_float4(px, py, tz, __int_as_float(off ? 0 : r));
                    if (!off) {
                        o_con = conic_of(ca, cb, cc, det, op);
                        tile_rect(px, py, r, cam.tiles_x, cam.tiles_y, tx0, tx1, ty0, ty1);
                        nt = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
                    }
                }
            }
        }
    }
    xydr[i] = o_xydr;
    conic[i] = o_con;
    tiles[i] = nt;
    if (cov_out) {
        cov_out[3 * i] = ca;
        cov_out[3 * i + 1] = cb;
        cov_out[3 * i + 2] = cc;
    }
    if (DKEY) {
        dkey = nt ? __float_as_uint(tz) : 0xFFFFFFFFu;
        dkeys[i] = dkey;
    }
    }  // i < n
    if (MODE == 3) {
        // replica r of every tile: counter tcount[r * tiles + tile], slots
        // [r * kr, (r + 1) * kr) of the tile's bin (a warp's Gaussians share
        // r; spreading the slot atomics over DREPL addresses per tile
        // cuts their same-address serialisation in L2)
        const uint32_t r = direct_replica((uint32_t)i), kr = kstride / DREPL;
        uint32_t* tc = tcount + (size_t)r * (cam.tiles_x * cam.tiles_y);
        walk_tile_rects<DIRECT_UNROLL>(threadIdx.x & 31, (uint32_t)i, tx0, tx1, ty0, ty1, cam.tiles_x,
                           [&](const uint32_t* tl, const uint32_t* gl) {
                               uint32_t slot[DIRECT_UNROLL];
#pragma unroll
                               for (int u = 0; u < DIRECT_UNROLL; ++u)
                                   slot[u] = tl[u] != 0xFFFFFFFFu ? atomicAdd(&tc[tl[u]], 1u) : kr;
#pragma unroll
                               for (int u = 0; u < DIRECT_UNROLL; ++u)
                                   if (slot[u] < kr) bins[(size_t)tl[u] * kstride + r * kr + slot[u]] = gl[u];
                           });
    }
    if (MODE == 2) {
        uint32_t* tc = tcount + (size_t)tcount_replica((uint32_t)i) * (cam.tiles_x * cam.tiles_y);
        walk_tile_rects(threadIdx.x & 31, 0u, tx0, tx1, ty0, ty1, cam.tiles_x,
                        [&](const uint32_t* tl, const uint32_t*) {
                            if (tl[0] != 0xFFFFFFFFu) atomicAdd(&tc[tl[0]], 1u);
                        });
    }
    if (MODE == 1 && dkey != 0xFFFFFFFFu) {
        kmin = min(kmin, dkey);
        kmax = max(kmax, dkey);
    }
    if (MODE == 1) warp_hist_add(s_lo, dkey & 255u, dkey != 0xFFFFFFFFu);
    }  // grid-stride
    if (MODE == 1) {  // one atomic pair per warp (meta[5] / meta[6], reset by frame_init_kernel)
        kmin = __reduce_min_sync(0xffffffffu, kmin);
        kmax = __reduce_max_sync(0xffffffffu, kmax);
        if ((threadIdx.x & 31) == 0 && kmin <= kmax) {
            atomicMin(reinterpret_cast<unsigned long long*>(status) + 5, (unsigned long long)kmin);
            atomicMax(reinterpret_cast<unsigned long long*>(status) + 6, (unsigned long long)kmax);
        }
        __syncthreads();
        for (int k = threadIdx.x; k < 256; k += blockDim.x)
            if (s_lo[k]) atomicAdd(&dhist[k], s_lo[k]);
    }
}

// View-independent part of sg/proj_backward.py:139-175 for one Gaussian:
// the unit quaternion (and 1/|q|), R, M = R diag(s) and Sigma = M M^T.
struct BwdPrep {
    float qw, qx, qy, qz, inv;
    float R[9], M[9], Sg[9];
};
// M = R diag(s) and Sigma = M M^T of a prepared Gaussian (P.R set)
__device__ __forceinline__ void bwd_prep_ms(BwdPrep& P, const float s[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) P.M[3 * a + b] = P.R[3 * a + b] * s[b];
    // Sigma = M M^T
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            P.Sg[3 * a + b] = P.M[3 * a] * P.M[3 * b] + P.M[3 * a + 1] * P.M[3 * b + 1] + P.M[3 * a + 2] * P.M[3 * b + 2];
}
__device__ __forceinline__ BwdPrep proj_bwd_prep(float4 q, const float s[3]) {
    BwdPrep P;
    const float qn = quat_norm(q);
    P.inv = 1.f / qn;
    P.qw = q.x * P.inv, P.qx = q.y * P.inv, P.qy = q.z * P.inv, P.qz = q.w * P.inv;
    quat_rot(P.qw, P.qx, P.qy, P.qz, P.R);
    bwd_prep_ms(P, s);
    return P;
}

// Per-view body of sg/proj_backward.py:200-222 for one visible Gaussian and
// the view's screen-space gradients (gg = d_mean2d x, y, d_cov00, d_cov01;
// g11 = d_cov11): d_mean, d_scale, d_quat and the 12 d_view terms.
__device__ __forceinline__ void proj_bwd_view(const CamK& cam, float mx, float my, float mz, const float s[3],
                                              const BwdPrep& P, float4 gg, float g11, float& dmx, float& dmy,
                                              float& dmz, float& dsx, float& dsy, float& dsz, float4& dq,
                                              float dv[12]) {
    const float qw = P.qw, qx = P.qx, qy = P.qy, qz = P.qz, inv = P.inv;
    const float* R = P.R;
    const float* M = P.M;
    const float* Sg = P.Sg;
    const float* Rc = cam.R;
    const float tx = Rc[0] * mx + Rc[1] * my + Rc[2] * mz + cam.t[0];
    const float ty = Rc[3] * mx + Rc[4] * my + Rc[5] * mz + cam.t[1];
    const float tz = Rc[6] * mx + Rc[7] * my + Rc[8] * mz + cam.t[2];
    const float iz = 1.f / tz, iz2 = iz * iz;
    const float j00 = cam.fx * iz, j02 = -cam.fx * tx * iz2;
    const float j11 = cam.fy * iz, j12 = -cam.fy * ty * iz2;
    float T0[3], T1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        T0[k] = j00 * Rc[k] + j02 * Rc[6 + k];
        T1[k] = j11 * Rc[3 + k] + j12 * Rc[6 + k];
    }
    const float gx = gg.x, gy = gg.y, g00 = gg.z, g01 = gg.w;
    // mean2d_backward (:53-77) == J^T d_mean2d with dt_w = 0
    float dt0 = cam.fx * gx * iz;
    float dt1 = cam.fy * gy * iz;
    float dt2 = -(cam.fx * gx * tx + cam.fy * gy * ty) * iz2;
    // cov2d_backward (:88-121)
    float GT0[3], GT1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        GT0[k] = g00 * T0[k] + g01 * T1[k];
        GT1[k] = g01 * T0[k] + g11 * T1[k];
    }
    float dS[9];  // T^T G T
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) dS[3 * a + b] = T0[a] * GT0[b] + T1[a] * GT1[b];
    // _cov_transform_grad (:80-85): G T Sigma^T + G^T T Sigma = 2 (G T) Sigma
    float dT0[3], dT1[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        dT0[b] = 2.f * (GT0[0] * Sg[b] + GT0[1] * Sg[3 + b] + GT0[2] * Sg[6 + b]);
        dT1[b] = 2.f * (GT1[0] * Sg[b] + GT1[1] * Sg[3 + b] + GT1[2] * Sg[6 + b]);
    }
    // dJ = dT R_cw^T (only the structurally non-zero entries of J matter)
    const float dJ00 = dT0[0] * Rc[0] + dT0[1] * Rc[1] + dT0[2] * Rc[2];
    const float dJ02 = dT0[0] * Rc[6] + dT0[1] * Rc[7] + dT0[2] * Rc[8];
    const float dJ11 = dT1[0] * Rc[3] + dT1[1] * Rc[4] + dT1[2] * Rc[5];
    const float dJ12 = dT1[0] * Rc[6] + dT1[1] * Rc[7] + dT1[2] * Rc[8];
    const float iz3 = iz2 * iz;
    dt0 += -cam.fx * iz2 * dJ02;
    dt1 += -cam.fy * iz2 * dJ12;
    dt2 += -cam.fx * iz2 * dJ00 + 2.f * cam.fx * tx * iz3 * dJ02 - cam.fy * iz2 * dJ11 +
           2.f * cam.fy * ty * iz3 * dJ12;
    // world_backward (:124-136)
    dmx = Rc[0] * dt0 + Rc[3] * dt1 + Rc[6] * dt2;
    dmy = Rc[1] * dt0 + Rc[4] * dt1 + Rc[7] * dt2;
    dmz = Rc[2] * dt0 + Rc[5] * dt1 + Rc[8] * dt2;
    const float dtv[3] = {dt0, dt1, dt2};
    const float hm[4] = {mx, my, mz, 1.f};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dv[4 * a + b] = dtv[a] * hm[b];
    // view rotation path (:218-222): d_view[:3,:3] += J^T dT
    const float J0[3] = {j00, 0.f, j02}, J1[3] = {0.f, j11, j12};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) dv[4 * a + b] += J0[a] * dT0[b] + J1[a] * dT1[b];
    // covariance3d_backward (:151-175): dM = (dS + dS^T) M = 2 dS M
    float dM[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            dM[3 * a + b] = 2.f * (dS[3 * a] * M[b] + dS[3 * a + 1] * M[3 + b] + dS[3 * a + 2] * M[6 + b]);
    float dR[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) dR[3 * a + b] = dM[3 * a + b] * s[b];
    dsx = R[0] * dM[0] + R[3] * dM[3] + R[6] * dM[6];
    dsy = R[1] * dM[1] + R[4] * dM[4] + R[7] * dM[7];
    dsz = R[2] * dM[2] + R[5] * dM[5] + R[8] * dM[8];
    // <dR, dR/dq_k> with the Jacobians of :139-148
    const float gw = 2.f * (-qz * dR[1] + qy * dR[2] + qz * dR[3] - qx * dR[5] - qy * dR[6] + qx * dR[7]);
    const float gxq = 2.f * (qy * dR[1] + qz * dR[2] + qy * dR[3] - 2.f * qx * dR[4] - qw * dR[5] +
                             qz * dR[6] + qw * dR[7] - 2.f * qx * dR[8]);
    const float gyq = 2.f * (-2.f * qy * dR[0] + qx * dR[1] + qw * dR[2] + qx * dR[3] + qz * dR[5] -
                             qw * dR[6] + qz * dR[7] - 2.f * qy * dR[8]);
    const float gzq = 2.f * (-2.f * qz * dR[0] - qw * dR[1] + qx * dR[2] + qw * dR[3] - 2.f * qz * dR[4] +
                             qy * dR[5] + qx * dR[6] + qy * dR[7]);
    // normalisation chain: (dq_hat - q_hat (q_hat . dq_hat)) / |q|
    const float dot = qw * gw + qx * gxq + qy * gyq + qz * gzq;
    dq = make_float4((gw - qw * dot) * inv, (gxq - qx * dot) * inv, (gyq - qy * dot) * inv,
                     (gzq - qz * dot) * inv);
}

constexpr int PBWD_THREADS = 256;

// Per-Gaussian loop body of sg/proj_backward.py:200-222.
#ifndef PBWD_RGBO_EARLY
#define PBWD_RGBO_EARLY 1  // measured: config 3 1042 -> 1057 frames/s (project bwd itself 4.38 -> 4.54 ms)
#endif
#ifndef PBWD_TWO_PHASE
#define PBWD_TWO_PHASE 0  // 1: read the visibility word first, the rest only for visible Gaussians
#endif
#ifndef PBWD_LASTBLOCK
#define PBWD_LASTBLOCK 0  // 1: the last block to finish reduces d_view (else view_reduce_kernel)
#endif
#ifndef PBWD_MINB
#define PBWD_MINB 4  // 64 registers: 4 CTAs per SM (config 4: 264 -> 239 us)
#endif
__global__ void __launch_bounds__(PBWD_THREADS, PBWD_MINB) project_bwd_kernel(
    const float* __restrict__ means, const float* __restrict__ scales, const float4* __restrict__ quats,
    int n, CamK cam, const uint32_t* __restrict__ tiles, float4* __restrict__ d_geo,
    float* __restrict__ d_c11, float* __restrict__ d_means, float* __restrict__ d_scales,
    float4* __restrict__ d_quats, float* __restrict__ view_partials, bool accumulate, int gstride,
    float4* __restrict__ rgbo_in, float4* __restrict__ rgbo_out, unsigned int* __restrict__ done_counter,
    float* __restrict__ d_view16, unsigned long long* __restrict__ clean_word, unsigned long long clean_sig,
    bool clear_accum, bool vis_from_grads) {
    griddep_wait();
    // grid-stride over Gaussians (resident blocks): d_view is accumulated per
    // thread over its Gaussians and reduced once per block, so the fixed-order
    // reduction of the block partials (view_reduce_kernel) stays short
    float dva[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) dva[k] = 0.f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    // the visibility word first: a culled Gaussian's gradient is exactly
    // zero (sg/proj_backward.py:200-203 loops over `projected` only), so its
    // parameters and (never touched) accumulator rows are not read at all
    const bool in = i < n;
    const uint32_t nt = in ? tiles[i] : 0u;
    bool vis = in && nt != 0u;
    float4 v_rgbo = make_float4(0.f, 0.f, 0.f, 0.f), gg = make_float4(0.f, 0.f, 0.f, 0.f);
    float g11 = 0.f;
    float mx = 0.f, my = 0.f, mz = 0.f, s[3] = {1.f, 1.f, 1.f};
    float4 q = make_float4(1.f, 0.f, 0.f, 0.f);
    float om[3] = {0.f, 0.f, 0.f}, os[3] = {0.f, 0.f, 0.f};  // accumulate: the caller's running sums
    float4 oq = make_float4(0.f, 0.f, 0.f, 0.f), orgbo = make_float4(0.f, 0.f, 0.f, 0.f);
#if PBWD_TWO_PHASE
    if (vis) {
#else
    if (in) {  // every load issued up front, ahead of the visibility test (one memory round trip)
#endif
        if (rgbo_in) v_rgbo = rgbo_in[(size_t)i * gstride];
        gg = d_geo[(size_t)i * gstride];
        g11 = d_c11[i];
        mx = means[3 * i], my = means[3 * i + 1], mz = means[3 * i + 2];
        s[0] = scales[3 * i], s[1] = scales[3 * i + 1], s[2] = scales[3 * i + 2];
        q = quats[i];
        if (accumulate) {
            om[0] = d_means[3 * i], om[1] = d_means[3 * i + 1], om[2] = d_means[3 * i + 2];
            os[0] = d_scales[3 * i], os[1] = d_scales[3 * i + 1], os[2] = d_scales[3 * i + 2];
            oq = d_quats[i];
            if (rgbo_in && !PBWD_RGBO_EARLY) orgbo = rgbo_out[i];
        }
    }
    // tile bands (dist.py): the screen-space gradients were summed over the
    // ranks' bands, so a Gaussian culled from this rank's band may carry
    // another band's gradient; only non-zero rows can (a Gaussian culled by
    // depth has none anywhere, so its undefined projection is never touched)
    if (vis_from_grads && in && !vis)
        vis = gg.x != 0.f || gg.y != 0.f || gg.z != 0.f || gg.w != 0.f || g11 != 0.f || v_rgbo.x != 0.f ||
              v_rgbo.y != 0.f || v_rgbo.z != 0.f || v_rgbo.w != 0.f;
    if (PBWD_RGBO_EARLY && rgbo_in && in && (vis || !accumulate)) {
        if (accumulate) {
            const float4 o = rgbo_out[i];
            rgbo_out[i] = make_float4(o.x + v_rgbo.x, o.y + v_rgbo.y, o.z + v_rgbo.z, o.w + v_rgbo.w);
        } else {
            rgbo_out[i] = v_rgbo;
        }
    }
    float dv[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) dv[k] = 0.f;
    if (in) {
        float dmx = 0.f, dmy = 0.f, dmz = 0.f, dsx = 0.f, dsy = 0.f, dsz = 0.f;
        float4 dq = make_float4(0.f, 0.f, 0.f, 0.f);
        if (vis) {
            const BwdPrep P = proj_bwd_prep(q, s);
            proj_bwd_view(cam, mx, my, mz, s, P, gg, g11, dmx, dmy, dmz, dsx, dsy, dsz, dq, dv);
        }
        if (accumulate) {  // sum over views into the caller's gradient (culled: nothing to add)
            if (vis) {
            d_means[3 * i] = om[0] + dmx; d_means[3 * i + 1] = om[1] + dmy; d_means[3 * i + 2] = om[2] + dmz;
            d_scales[3 * i] = os[0] + dsx; d_scales[3 * i + 1] = os[1] + dsy; d_scales[3 * i + 2] = os[2] + dsz;
            d_quats[i] = make_float4(oq.x + dq.x, oq.y + dq.y, oq.z + dq.z, oq.w + dq.w);
            }
        } else {
            d_means[3 * i] = dmx; d_means[3 * i + 1] = dmy; d_means[3 * i + 2] = dmz;
            d_scales[3 * i] = dsx; d_scales[3 * i + 1] = dsy; d_scales[3 * i + 2] = dsz;
            d_quats[i] = dq;
        }
    }
    // frame path: the d_color / d_opacity row of the interleaved buffer
    // (accumulating: a culled Gaussian adds exact zeros -- skip its row); all
    // read-modify-writes store at the end, well behind their loads
    if (!PBWD_RGBO_EARLY && rgbo_in && in && (vis || !accumulate))
        rgbo_out[i] = accumulate ? make_float4(orgbo.x + v_rgbo.x, orgbo.y + v_rgbo.y, orgbo.z + v_rgbo.z,
                                               orgbo.w + v_rgbo.w)
                                 : v_rgbo;
    if (clear_accum && vis) {
        // leave the accumulators zero for the next frame (culled rows were
        // never touched).  After the outputs, with streaming stores: issued
        // right behind the loads of the same rows, these stores made the
        // kernel 2.2x slower at config 3 (the loads' sectors stall them)
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        if (rgbo_in) __stcs(rgbo_in + (size_t)i * gstride, z);
        __stcs(d_geo + (size_t)i * gstride, z);
        __stcs(d_c11 + i, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 12; ++k) dva[k] += dv[k];
    }  // grid-stride
    // block partial of d_view (deterministic: fixed shuffle tree + fixed warp
    // order).  Transposed warp reduction of the 12 values padded to 16: each
    // level exchanges half of the values, so 16 shuffles instead of 60.
    __shared__ float red[PBWD_THREADS / 32][12];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {
        float v16[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v16[k] = k < 12 ? dva[k] : 0.f;
#pragma unroll
        for (int h = 8, m = 16; h >= 1; h >>= 1, m >>= 1) {  // lane bit m selects the kept half
            const bool up = lane & m;
#pragma unroll
            for (int j = 0; j < h; ++j) {
                const float send = up ? v16[j] : v16[j + h];
                const float keep = up ? v16[j + h] : v16[j];
                v16[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
            }
        }
        // v16[0] of lane L: value index (L >> 1), summed over the 16 lanes sharing (L & 1)
        const float tot = v16[0] + __shfl_xor_sync(0xffffffffu, v16[0], 1);
        const int k = lane >> 1;
        if ((lane & 1) == 0 && k < 12) red[warp][k] = tot;
    }
    __syncthreads();
    if (threadIdx.x < 12) {
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < PBWD_THREADS / 32; ++w) v += red[w][threadIdx.x];
        view_partials[blockIdx.x * 12 + threadIdx.x] = v;
        if (done_counter) __threadfence();  // the writers' fence, before the last-block vote
    }
    if (!done_counter) return;  // a separate view_reduce_kernel finishes d_view
    // frame path: the last block to finish sums the partials (fixed order,
    // same tree as view_reduce_kernel) -- no extra kernel launch
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(done_counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int k = warp; k < 12; k += PBWD_THREADS / 32) {
        float v = 0.f;
        for (int b = lane; b < (int)gridDim.x; b += 32) v += ((volatile float*)view_partials)[b * 12 + k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) d_view16[k] = v;
    }
    if (threadIdx.x < 4) d_view16[12 + threadIdx.x] = 0.f;
    if (threadIdx.x == 0) {
        *done_counter = 0u;
        if (clean_word) *clean_word = clear_accum ? clean_sig : 0ull;
    }
}

// Fixed-order sum of the per-block d_view partials -> 4x4 (bottom row 0,
// sg/proj_backward.py:31-32).
__global__ void __launch_bounds__(384) view_reduce_kernel(const float* __restrict__ partials, int nblocks,
                                                          float* __restrict__ d_view16,
                                                          unsigned long long* __restrict__ clean_word,
                                                          unsigned long long clean_stamp, bool add) {
    griddep_wait();
    if (clean_word && threadIdx.x == 0) *clean_word = clean_stamp;
    const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float v = 0.f;
    for (int b = lane; b < nblocks; b += 32) v += partials[b * 12 + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) d_view16[k] = add ? d_view16[k] + v : v;
    if (threadIdx.x < 4) d_view16[12 + threadIdx.x] = 0.f;
}

// Frame start: status word = all ones (no error), intersection total and the
// depth-digit histograms = 0 (the projection accumulates into them).
// Frame reset ahead of the projection: meta, the depth histograms and (scatter
// binning) the per-tile intersection counts the projection accumulates.
// meta[4] = 1 when the backward accumulators must be zeroed this frame: the
// workspace's clean word does not carry this layout's signature (fresh or
// re-laid-out workspace, or the last backward kept its screen-space
// gradients); the word is then stamped (the projection zeroes them).
__global__ void __launch_bounds__(256) frame_init_kernel(unsigned long long* __restrict__ meta,
                                                         uint32_t* __restrict__ dhist, uint32_t* __restrict__ tcount,
                                                         int n_counts, unsigned long long* __restrict__ clean_word,
                                                         unsigned long long clean_sig) {
    griddep_wait();
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0) {
            meta[0] = ~0ull;
            meta[1] = 0ull;
            meta[2] = 0ull;
            meta[3] = 0ull;
            if (clean_word) {
                meta[4] = *clean_word != clean_sig ? 1ull : 0ull;
                *clean_word = clean_sig;
            }
            meta[5] = 0xFFFFFFFFull;  // visible depth-key range (depth-first binning)
            meta[6] = 0ull;
            meta[7] = 0ull;           // visible Gaussians (the depth sort's first pass)
            meta[8] = 4ull;           // depth-sort passes
        }
        for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x) dhist[k] = 0u;
    }
    if (tcount)
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_counts; k += gridDim.x * blockDim.x) tcount[k] = 0u;
}

int launch_project_fwd_dkey(const float* means3, const float* scales3, const float* quats4, const float* opac,
                            int64_t n, const CamK& k, float* xydr4, float* conic4, uint32_t* tiles, float* cov3,
                            unsigned long long* status, uint32_t* dkeys, uint32_t* dhist, cudaStream_t s,
                            const ZeroJobs& zj, uint32_t* tcount, uint32_t* bins, uint32_t kstride,
                            unsigned long long* clean_word, unsigned long long clean_sig) {
    const int n_tiles = k.tiles_x * k.tiles_y;
    const int init_blocks = tcount ? (TCOUNT_REPL * n_tiles + 2047) / 2048 : 1;
    launch_k(frame_init_kernel, dim3((unsigned)init_blocks), dim3(256), 0, s, status, dhist, tcount,
             TCOUNT_REPL * n_tiles, clean_word, clean_sig);
    if (check_launch("frame_init_kernel")) return -1;
    int64_t blocks = (n + 255) / 256;
    if (blocks < 1) blocks = 1;  // the zero jobs run even for an empty scene
    const int64_t cap = (int64_t)sort_sm_count() * (tcount ? PFWD_MINB : pfwd_minb(1));  // resident CTAs
    if (blocks > cap) blocks = cap;
    if (tcount && bins)
        launch_k(project_fwd_kernel<3>, dim3((unsigned)blocks), dim3(256), 0, s, means3, scales3,
                 (const float4*)quats4, opac, (int)n, k, (float4*)xydr4, (float4*)conic4, tiles, cov3, status, dkeys,
                 dhist, zj, tcount, bins, kstride);
    else if (tcount)
        launch_k(project_fwd_kernel<2>, dim3((unsigned)blocks), dim3(256), 0, s, means3, scales3,
                 (const float4*)quats4, opac, (int)n, k, (float4*)xydr4, (float4*)conic4, tiles, cov3, status, dkeys,
                 dhist, zj, tcount, (uint32_t*)nullptr, 0u);
    else
        launch_k(project_fwd_kernel<1>, dim3((unsigned)blocks), dim3(256), 0, s, means3, scales3,
                 (const float4*)quats4, opac, (int)n, k, (float4*)xydr4, (float4*)conic4, tiles, cov3, status, dkeys,
                 dhist, zj, (uint32_t*)nullptr, (uint32_t*)nullptr, 0u);
    return check_launch("project_fwd_kernel<dkey>");
}

// ---------------------------------------------------------------- all views at once
// The projection backward of a multi-view step (sg/proj_backward.py:178-223
// for every view, summed): one pass over the Gaussians, each thread loading
// its Gaussian's parameters once, deriving the view-independent part (unit
// quaternion, R, M, Sigma) once, then for every view reading the view's
// screen-space gradient rows (its own workspace), adding the view's
// contribution to registers and clearing the rows it read; the parameter
// gradients are written once.  Against one projection backward per view,
// which re-reads the parameters and read-modify-writes the running sums for
// every view (~224 B per visible Gaussian and view), this moves ~76 B per
// visible Gaussian and view.  A Gaussian is visible in a view iff its rows are
// non-zero: a culled one's rows are never written, and a visible one with
// zero rows contributes exactly zero (the backward is linear in them), so the
// visibility word is not read.  d_view per view: the 12 terms are warp-
// reduced per view (transposed shuffle tree, fixed order), summed per warp in
// shared memory, per block into the view's own partials, then by
// views_reduce_kernel in a fixed order -- deterministic.
__global__ void __launch_bounds__(PBWD_THREADS, 2) views_project_bwd_kernel(
    const float* __restrict__ means, const float* __restrict__ scales, const float4* __restrict__ quats, int n,
    const MvArgs args, float* __restrict__ d_means, float* __restrict__ d_scales, float4* __restrict__ d_quats,
    float4* __restrict__ d_rgbo, bool accumulate, bool clear_rows) {
    griddep_wait();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ float s_dv[PBWD_THREADS / 32][MV_MAX][12];  // per-warp d_view sums (each warp owns its row)
    for (int k = lane; k < MV_MAX * 12; k += 32) (&s_dv[warp][0][0])[k] = 0.f;
    __syncwarp();
    const int nv = args.nv;
    const int n_round = (n + 31) & ~31;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += gridDim.x * blockDim.x) {
        const bool in = i < n;
        float mx = 0.f, my = 0.f, mz = 0.f, s[3] = {1.f, 1.f, 1.f};
        float4 q = make_float4(1.f, 0.f, 0.f, 0.f);
        if (in) {
            mx = means[3 * i], my = means[3 * i + 1], mz = means[3 * i + 2];
            s[0] = scales[3 * i], s[1] = scales[3 * i + 1], s[2] = scales[3 * i + 2];
            q = quats[i];
        }
        BwdPrep P;
        bool prepped = false;
        // accumulate: the running sums start from the rows' current values, so
        // views split over several calls sum in exactly the one-call order
        float am[3] = {0.f, 0.f, 0.f}, as[3] = {0.f, 0.f, 0.f};
        float4 aq = make_float4(0.f, 0.f, 0.f, 0.f), argbo = make_float4(0.f, 0.f, 0.f, 0.f);
        if (in && accumulate) {
            am[0] = d_means[3 * i], am[1] = d_means[3 * i + 1], am[2] = d_means[3 * i + 2];
            as[0] = d_scales[3 * i], as[1] = d_scales[3 * i + 1], as[2] = d_scales[3 * i + 2];
            aq = d_quats[i];
            argbo = d_rgbo[i];
        }
        // the next view's rows are loaded while this view's are processed
        float4 nrg = make_float4(0.f, 0.f, 0.f, 0.f), ngg = nrg;
        float ng11 = 0.f;
        if (in && nv > 0) {
            nrg = args.v[0].g8[2 * (size_t)i];
            ngg = args.v[0].g8[2 * (size_t)i + 1];
            ng11 = args.v[0].d_c11[i];
        }
        for (int v = 0; v < nv; ++v) {
            const MvView& V = args.v[v];
            const float4 rg = nrg, gg = ngg;
            const float g11 = ng11;
            if (in && v + 1 < nv) {
                const MvView& N = args.v[v + 1];
                nrg = N.g8[2 * (size_t)i];
                ngg = N.g8[2 * (size_t)i + 1];
                ng11 = N.d_c11[i];
            }
            const bool vis = gg.x != 0.f || gg.y != 0.f || gg.z != 0.f || gg.w != 0.f || g11 != 0.f ||
                             rg.x != 0.f || rg.y != 0.f || rg.z != 0.f || rg.w != 0.f;
            float dv[12];
#pragma unroll
            for (int k = 0; k < 12; ++k) dv[k] = 0.f;
            if (vis) {
                if (!prepped) {
                    P = proj_bwd_prep(q, s);
                    prepped = true;
                }
                float dmx, dmy, dmz, dsx, dsy, dsz;
                float4 dq;
                proj_bwd_view(V.cam, mx, my, mz, s, P, gg, g11, dmx, dmy, dmz, dsx, dsy, dsz, dq, dv);
                am[0] += dmx, am[1] += dmy, am[2] += dmz;
                as[0] += dsx, as[1] += dsy, as[2] += dsz;
                aq.x += dq.x, aq.y += dq.y, aq.z += dq.z, aq.w += dq.w;
                argbo.x += rg.x, argbo.y += rg.y, argbo.z += rg.z, argbo.w += rg.w;
                if (clear_rows) {  // the accumulators stay zero for the view's next frame
                    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                    __stcs(V.g8 + 2 * (size_t)i, z);
                    __stcs(V.g8 + 2 * (size_t)i + 1, z);
                    __stcs(V.d_c11 + i, 0.f);
                }
            }
            if (__any_sync(0xffffffffu, vis)) {
                // transposed warp reduction of the 12 terms (padded to 16)
                float v16[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) v16[k] = k < 12 ? dv[k] : 0.f;
#pragma unroll
                for (int h = 8, m = 16; h >= 1; h >>= 1, m >>= 1) {
                    const bool up = lane & m;
#pragma unroll
                    for (int j = 0; j < h; ++j) {
                        const float send = up ? v16[j] : v16[j + h];
                        const float keep = up ? v16[j + h] : v16[j];
                        v16[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                    }
                }
                const float tot = v16[0] + __shfl_xor_sync(0xffffffffu, v16[0], 1);
                const int k = lane >> 1;
                if ((lane & 1) == 0 && k < 12) s_dv[warp][v][k] += tot;
            }
        }
        if (in) {
            d_means[3 * i] = am[0], d_means[3 * i + 1] = am[1], d_means[3 * i + 2] = am[2];
            d_scales[3 * i] = as[0], d_scales[3 * i + 1] = as[1], d_scales[3 * i + 2] = as[2];
            d_quats[i] = aq;
            d_rgbo[i] = argbo;
        }
    }
    __syncthreads();
    // block partials: per view, the warps' sums in warp order
    for (int k = threadIdx.x; k < nv * 12; k += blockDim.x) {
        const int v = k / 12, c = k - 12 * v;
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < PBWD_THREADS / 32; ++w) acc += s_dv[w][v][c];
        args.v[v].partials[blockIdx.x * 12 + c] = acc;
    }
}

// The same projection backward with the per-view work compacted.  Only
// ~9 % of a config-3 step's (Gaussian, view) rows are non-zero (early
// termination hides most in-frustum Gaussians), so in the kernel above a
// warp runs the ~400-instruction per-view body for nearly every (warp, view)
// with a few lanes live, and reads every row to find the non-zero ones.
// Here the raster backward marks every Gaussian it adds to (one bit per
// Gaussian and view, gs_frame_view.touched, cleared by the forward), and each
// warp owns 32 Gaussians per iteration: lane v reads view v's 32 marks, the
// marked (view, Gaussian) pairs become a view-major item list in shared
// memory (a warp prefix sum over the lanes' counts), the view-independent
// part of each Gaussian (mean, scale, unit quaternion, R) goes to shared
// memory, and the per-view body runs on 32 items at a time, one per lane --
// its rows loaded a batch ahead and cleared after use.  The items' d_mean /
// d_scale / d_quat / d_rgbo go through shared memory back to their owner
// lanes, which add them in item order, i.e. in view order (the order of the
// kernel above).  d_view: a segmented scan over the batch's view runs (fixed
// order), the run totals into the warp's per-view sums, then block partials
// and views_reduce_kernel as above -- deterministic.  Config 3: 1.61 ->
// 0.57 ms per step; reading every row and queueing the non-zero ones instead
// took 1.14 ms (bound by the 3.5 GB of rows), a per-view walk with the marks
// 0.86 ms (~100 instructions per (warp, view)); clearing a row right after
// loading it (store behind the load of the same address) took 4.7 ms.
constexpr int VG = 20;    // per-Gaussian fields: mean 3, scale 3, qw qx qy qz inv, R 9 (M, Sigma per item)
constexpr int VCAM = 15;  // per-view camera fields (R 9, t 3, fx, fy; odd stride)
struct VbWarp {
    float g[VG][32];              // the warp's 32 Gaussians (SoA)
    uint16_t items[MV_MAX * 32];  // the marked (view, Gaussian) pairs, view-major: view << 5 | lane
    float out[14][32];            // a batch's d_mean 3, d_scale 3, d_quat 4, d_rgbo 4 per item
    uint32_t own[32];             // per owner lane: its items in the batch (bit mask)
    float dv[MV_MAX][12];         // per-view d_view sums
};
struct VbShared {
    float cam[MV_MAX][VCAM];
    float4* g8[MV_MAX];
    float* c11[MV_MAX];
    VbWarp w[PBWD_THREADS / 32];
};

// One batch of up to 32 items, one per lane: the item's rows (cleared after
// reading), the per-view body, the results to shared memory for their
// owners, d_view by a segmented scan over the batch's view runs.
// An item's rows (loaded a batch ahead).
struct VbRow {
    float4 rg, gg;
    float g11;
};
__device__ __forceinline__ VbRow vb_load(const VbShared& sh, const VbWarp& W, int lane, int i0, int b0, int total) {
    VbRow r;
    r.rg = r.gg = make_float4(0.f, 0.f, 0.f, 0.f);
    r.g11 = 0.f;
    if (b0 + lane < total) {
        const uint32_t it = W.items[b0 + lane];
        const size_t gi = (size_t)(i0 + (int)(it & 31u));
        const float4* g8 = sh.g8[it >> 5] + 2 * gi;
        r.rg = g8[0], r.gg = g8[1];
        r.g11 = sh.c11[it >> 5][gi];
    }
    return r;
}

__device__ __forceinline__ void vb_process(VbShared& sh, VbWarp& W, int lane, int i0, int b0, int count,
                                           bool clear_rows, const VbRow& row) {
    const bool act = lane < count;
    const uint32_t it = act ? W.items[b0 + lane] : 0u;
    const int j = (int)(it & 31u);
    const int v = act ? (int)(it >> 5) : 0x10000 + lane;  // (inactive lanes: runs of their own)
    float dvv[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) dvv[k] = 0.f;
    if (act) {
        const size_t gi = (size_t)(i0 + j);
        float4* g8 = sh.g8[v] + 2 * gi;
        float* c11 = sh.c11[v] + gi;
        const float4 rg = row.rg, gg = row.gg;
        const float g11 = row.g11;
        CamK cam;
        const float* c = sh.cam[v];
#pragma unroll
        for (int k = 0; k < 9; ++k) cam.R[k] = c[k];
        cam.t[0] = c[9], cam.t[1] = c[10], cam.t[2] = c[11];
        cam.fx = c[12], cam.fy = c[13];
        const float sc[3] = {W.g[3][j], W.g[4][j], W.g[5][j]};
        BwdPrep P;
        P.qw = W.g[6][j], P.qx = W.g[7][j], P.qy = W.g[8][j], P.qz = W.g[9][j], P.inv = W.g[10][j];
#pragma unroll
        for (int k = 0; k < 9; ++k) P.R[k] = W.g[11 + k][j];
        bwd_prep_ms(P, sc);
        float dmx, dmy, dmz, dsx, dsy, dsz;
        float4 dq;
        proj_bwd_view(cam, W.g[0][j], W.g[1][j], W.g[2][j], sc, P, gg, g11, dmx, dmy, dmz, dsx, dsy, dsz, dq, dvv);
        W.out[0][lane] = dmx, W.out[1][lane] = dmy, W.out[2][lane] = dmz;
        W.out[3][lane] = dsx, W.out[4][lane] = dsy, W.out[5][lane] = dsz;
        W.out[6][lane] = dq.x, W.out[7][lane] = dq.y, W.out[8][lane] = dq.z, W.out[9][lane] = dq.w;
        W.out[10][lane] = rg.x, W.out[11][lane] = rg.y, W.out[12][lane] = rg.z, W.out[13][lane] = rg.w;
        // the accumulators stay zero for the view's next frame (cleared well
        // after the loads: a store right behind the load of the same row stalls
        // the warp for tens of microseconds)
        if (clear_rows) {
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            __stcs(g8, z);
            __stcs(g8 + 1, z);
            __stcs(c11, 0.f);
        }
    }
    // d_view: inclusive scan within each run of equal views (the items are
    // view-major, so a view's items are contiguous); the run's last lane adds
    // the total to the warp's sum for the view
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int vo = __shfl_up_sync(0xffffffffu, v, off);
        const bool take = lane >= off && vo == v;
#pragma unroll
        for (int k = 0; k < 12; ++k) {
            const float t = __shfl_up_sync(0xffffffffu, dvv[k], off);
            if (take) dvv[k] = __fadd_rn(t, dvv[k]);
        }
    }
    const int vn = __shfl_down_sync(0xffffffffu, v, 1);
    if (act && (lane == count - 1 || vn != v)) {
#pragma unroll
        for (int k = 0; k < 12; ++k) W.dv[v][k] = __fadd_rn(W.dv[v][k], dvv[k]);
    }
    // owners: each item's lane set per owner (lowest lane publishes it)
    const uint32_t same = __match_any_sync(0xffffffffu, act ? j : 32 + lane);
    if (act && lane == __ffs(same) - 1) W.own[j] = same;
    __syncwarp();
}

__global__ void __launch_bounds__(PBWD_THREADS, 2) views_project_bwd_compact_kernel(
    const float* __restrict__ means, const float* __restrict__ scales, const float4* __restrict__ quats, int n,
    const MvArgs args, float* __restrict__ d_means, float* __restrict__ d_scales, float4* __restrict__ d_quats,
    float4* __restrict__ d_rgbo, bool accumulate, bool clear_rows) {
    griddep_wait();
    extern __shared__ __align__(16) unsigned char vb_raw[];
    VbShared& sh = *reinterpret_cast<VbShared*>(vb_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    VbWarp& W = sh.w[warp];
    const int nv = args.nv;
    for (int k = threadIdx.x; k < nv * VCAM; k += blockDim.x) {
        const int v = k / VCAM, f = k - v * VCAM;
        const CamK& c = args.v[v].cam;
        sh.cam[v][f] = f < 9 ? c.R[f] : f < 12 ? c.t[f - 9] : f == 12 ? c.fx : f == 13 ? c.fy : 0.f;
    }
    if (threadIdx.x < nv) sh.g8[threadIdx.x] = args.v[threadIdx.x].g8, sh.c11[threadIdx.x] = args.v[threadIdx.x].d_c11;
    for (int k = lane; k < MV_MAX * 12; k += 32) (&W.dv[0][0])[k] = 0.f;
    W.own[lane] = 0u;
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    const int n_round = (n + 31) & ~31;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += gridDim.x * blockDim.x) {
        const bool in = i < n;
        const int i0 = i - lane;  // the warp's first Gaussian
        // lane v: view v's marks of the warp's 32 Gaussians (the raster backward
        // marked every Gaussian it added to; unmarked rows are zero)
        uint32_t vmark = 0u;
        if (lane < nv) {
            vmark = 0xFFFFFFFFu;
            if (args.v[lane].touched) {
                const uint32_t a = (uint32_t)(args.v[lane].tbase + i0);
                const uint32_t* t = args.v[lane].touched + (a >> 5);
                const uint32_t sh5 = a & 31u;
                vmark = t[0] >> sh5;
                if (sh5 && i0 + 32 - (int)sh5 < n) vmark |= t[1] << (32u - sh5);
            }
            if (n - i0 < 32) vmark &= (1u << (n - i0)) - 1u;
        }
        // the items, view-major: lane v writes its marked Gaussians after the lower views'
        const uint32_t cnt = (uint32_t)__popc(vmark);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = (int)__shfl_sync(0xffffffffu, incl, 31);
        {
            uint32_t m = vmark, k = incl - cnt;
            while (m) {
                const uint32_t jj = (uint32_t)(__ffs(m) - 1);
                m &= m - 1u;
                W.items[k++] = (uint16_t)(((uint32_t)lane << 5) | jj);
            }
        }
        {
            float mx = 0.f, my = 0.f, mz = 0.f, sc[3] = {1.f, 1.f, 1.f};
            float4 q = make_float4(1.f, 0.f, 0.f, 0.f);
            if (in) {
                mx = means[3 * i], my = means[3 * i + 1], mz = means[3 * i + 2];
                sc[0] = scales[3 * i], sc[1] = scales[3 * i + 1], sc[2] = scales[3 * i + 2];
                q = quats[i];
            }
            const BwdPrep P = proj_bwd_prep(q, sc);
            W.g[0][lane] = mx, W.g[1][lane] = my, W.g[2][lane] = mz;
            W.g[3][lane] = sc[0], W.g[4][lane] = sc[1], W.g[5][lane] = sc[2];
            W.g[6][lane] = P.qw, W.g[7][lane] = P.qx, W.g[8][lane] = P.qy, W.g[9][lane] = P.qz;
            W.g[10][lane] = P.inv;
#pragma unroll
            for (int k = 0; k < 9; ++k) W.g[11 + k][lane] = P.R[k];
        }
        float acc[14];  // d_mean 3, d_scale 3, d_quat 4, d_rgbo 4
#pragma unroll
        for (int c = 0; c < 14; ++c) acc[c] = 0.f;
        if (in && accumulate) {
            acc[0] = d_means[3 * i], acc[1] = d_means[3 * i + 1], acc[2] = d_means[3 * i + 2];
            acc[3] = d_scales[3 * i], acc[4] = d_scales[3 * i + 1], acc[5] = d_scales[3 * i + 2];
            const float4 o = d_quats[i], r = d_rgbo[i];
            acc[6] = o.x, acc[7] = o.y, acc[8] = o.z, acc[9] = o.w;
            acc[10] = r.x, acc[11] = r.y, acc[12] = r.z, acc[13] = r.w;
        }
        __syncwarp();
        VbRow row = vb_load(sh, W, lane, i0, 0, total);
        for (int b0 = 0; b0 < total; b0 += 32) {
            const VbRow cur = row;
            if (b0 + 32 < total) row = vb_load(sh, W, lane, i0, b0 + 32, total);  // the next batch's rows in flight
            vb_process(sh, W, lane, i0, b0, min(32, total - b0), clear_rows, cur);
            // an owner adds its items of the batch in item (= view) order
            uint32_t mm = W.own[lane];
            if (mm) W.own[lane] = 0u;
            while (mm) {
                const int k = __ffs(mm) - 1;
                mm &= mm - 1u;
#pragma unroll
                for (int c = 0; c < 14; ++c) acc[c] = __fadd_rn(acc[c], W.out[c][k]);
            }
            __syncwarp();
        }
        if (in) {
            d_means[3 * i] = acc[0], d_means[3 * i + 1] = acc[1], d_means[3 * i + 2] = acc[2];
            d_scales[3 * i] = acc[3], d_scales[3 * i + 1] = acc[4], d_scales[3 * i + 2] = acc[5];
            d_quats[i] = make_float4(acc[6], acc[7], acc[8], acc[9]);
            d_rgbo[i] = make_float4(acc[10], acc[11], acc[12], acc[13]);
        }
        __syncwarp();  // the warp's Gaussian fields and items are rewritten next iteration
    }
    (void)lt;
    __syncthreads();
    for (int k = threadIdx.x; k < nv * 12; k += blockDim.x) {
        const int v = k / 12, c = k - 12 * v;
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < PBWD_THREADS / 32; ++w) acc += sh.w[w].dv[v][c];
        args.v[v].partials[blockIdx.x * 12 + c] = acc;
    }
}

// Per view (one CTA each): the fixed-order sum of its block partials ->
// d_views16[v] (bottom row 0), and its workspace stamped clean (or not).
__global__ void __launch_bounds__(384) views_reduce_kernel(const MvArgs args, int nblocks, float* __restrict__ d_views16,
                                                           bool add) {
    griddep_wait();
    const int v = blockIdx.x;
    const MvView& V = args.v[v];
    if (threadIdx.x == 0 && V.clean_word) *V.clean_word = V.clean_stamp;
    const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float acc = 0.f;
    for (int b = lane; b < nblocks; b += 32) acc += V.partials[b * 12 + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    float* dv = d_views16 + 16 * v;
    if (lane == 0) dv[k] = add ? dv[k] + acc : acc;
    if (threadIdx.x < 4) dv[12 + threadIdx.x] = 0.f;
}

int launch_views_project_bwd(const float* means3, const float* scales3, const float* quats4, int64_t n,
                             const MvArgs& a, float* d_means3, float* d_scales3, float* d_quats4, float* d_rgbo4,
                             float* d_views16, bool accumulate, bool clear_rows, bool add_view, cudaStream_t s) {
    if (a.nv <= 0) return 0;
    int blocks = (int)((n + PBWD_THREADS - 1) / PBWD_THREADS);
    const int resident = sort_sm_count() * 2;
    if (blocks > resident) blocks = resident;
    if (blocks < 1) blocks = 1;
    static const bool compact = [] {
        const char* e = getenv("GS_PBWD_COMPACT");
        return !(e && e[0] == '0');
    }();
    if (compact) {
        static const bool attr = [] {
            cudaFuncSetAttribute(views_project_bwd_compact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(VbShared));
            return true;
        }();
        (void)attr;
        launch_k(views_project_bwd_compact_kernel, dim3(blocks), dim3(PBWD_THREADS), sizeof(VbShared), s, means3,
                 scales3, (const float4*)quats4, (int)n, a, d_means3, d_scales3, (float4*)d_quats4,
                 (float4*)d_rgbo4, accumulate, clear_rows);
        if (check_launch("views_project_bwd_compact_kernel")) return -1;
    } else {
        launch_k(views_project_bwd_kernel, dim3(blocks), dim3(PBWD_THREADS), 0, s, means3, scales3,
                 (const float4*)quats4, (int)n, a, d_means3, d_scales3, (float4*)d_quats4, (float4*)d_rgbo4,
                 accumulate, clear_rows);
        if (check_launch("views_project_bwd_kernel")) return -1;
    }
    launch_k(views_reduce_kernel, dim3(a.nv), dim3(384), 0, s, a, blocks, d_views16, add_view);
    return check_launch("views_reduce_kernel");
}

// ---------------------------------------------------------------- all views at once (forward)
// The depth-first frame's projection (project_fwd_kernel<1>) for every view
// of a multi-view step in one pass: each Gaussian's parameters are read once
// (44 B) and its M = R diag(s) formed once; per view the camera-space mean,
// the depth cull and the rest of sg/projection.py:115-145 write the view's
// xydr / conic / tiles / depth key (40 B) into its own workspace.  Each
// view's visible depth-key range is reduced per warp, per block in shared
// memory and once per block into the view's meta[5] / meta[6].  Against one
// projection per view: 40 + 44/views instead of 84 B per Gaussian and view.
__global__ void __launch_bounds__(256) views_init_kernel(const MvFwdArgs a) {
    griddep_wait();
    const MvFwdView& V = a.v[blockIdx.x];
    if (threadIdx.x == 0) {
        unsigned long long* meta = V.meta;
        meta[0] = ~0ull;
        meta[1] = 0ull;
        meta[2] = 0ull;
        meta[3] = 0ull;
        meta[4] = *V.clean_word != V.clean_sig ? 1ull : 0ull;
        *V.clean_word = V.clean_sig;
        meta[5] = 0xFFFFFFFFull;
        meta[6] = 0ull;
        meta[7] = 0ull;
        meta[8] = 4ull;
    }
    for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x) V.dhist[k] = 0u;
}

__global__ void __launch_bounds__(256, 4) views_project_fwd_kernel(const float* __restrict__ means,
                                                                   const float* __restrict__ scales,
                                                                   const float4* __restrict__ quats,
                                                                   const float* __restrict__ opac, int n,
                                                                   const MvFwdArgs a) {
    griddep_wait();
    const int nv = a.nv;
    for (int v = 0; v < nv; ++v) run_zero_jobs(a.v[v].zj);
    __shared__ uint32_t s_kmin[MV_MAX], s_kmax[MV_MAX];
    __shared__ uint32_t s_lo[MV_MAX][256];  // per view: the visible keys' low-byte histogram (sort.cu)
    // per view: the camera and the output pointers in shared memory (the view
    // loop's reads are then shared loads, not register-indexed constant loads)
    struct Hot {
        CamK cam;
        float4* xydr;
        float4* conic;
        uint32_t* tiles;
        uint32_t* dkeys;
        unsigned long long* meta;
    };
    __shared__ Hot s_v[MV_MAX];
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        s_v[v].cam = a.v[v].cam;
        s_v[v].xydr = a.v[v].xydr, s_v[v].conic = a.v[v].conic, s_v[v].tiles = a.v[v].tiles;
        s_v[v].dkeys = a.v[v].dkeys, s_v[v].meta = a.v[v].meta;
    }
    for (int v = threadIdx.x; v < MV_MAX; v += blockDim.x) s_kmin[v] = 0xFFFFFFFFu, s_kmax[v] = 0u;
    for (int k = threadIdx.x; k < MV_MAX * 256; k += blockDim.x) (&s_lo[0][0])[k] = 0u;
    __syncthreads();
    const int n_round = (n + 31) & ~31;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += gridDim.x * blockDim.x) {
        const bool in = i < n;
        float mx = 0.f, my = 0.f, mz = 0.f, sx = 1.f, sy = 1.f, sz = 1.f, op = 0.f;
        float4 q = make_float4(1.f, 0.f, 0.f, 0.f);
        if (in) {
            mx = means[3 * i], my = means[3 * i + 1], mz = means[3 * i + 2];
            sx = scales[3 * i], sy = scales[3 * i + 1], sz = scales[3 * i + 2];
            q = quats[i];
            op = opac[i];
        }
        const FwdPrep P = proj_fwd_prep(q, sx, sy, sz);
        for (int v = 0; v < nv; ++v) {
            const Hot& V = s_v[v];
            const CamK& cam = V.cam;
            uint32_t dkey = 0xFFFFFFFFu;
            if (in) {
                const float* Rc = cam.R;
                const float tx = Rc[0] * mx + Rc[1] * my + Rc[2] * mz + cam.t[0];
                const float ty = Rc[3] * mx + Rc[4] * my + Rc[5] * mz + cam.t[1];
                const float tz = Rc[6] * mx + Rc[7] * my + Rc[8] * mz + cam.t[2];
                float4 o_xydr = make_float4(0.f, 0.f, tz, __int_as_float(0));
                float4 o_con = make_float4(0.f, 0.f, 0.f, 0.f);
                float ca = 0.f, cb = 0.f, cc = 0.f;
                int tx0 = 0, tx1 = -1, ty0 = 0, ty1 = -1;
                uint32_t nt = 0;
                if (!((tz <= cam.near_plane) || (tz >= cam.far_plane)))
                    proj_fwd_core(cam, i, tx, ty, tz, P, op, V.meta, o_xydr, o_con, nt, ca, cb, cc, tx0, tx1, ty0,
                                  ty1);
                V.xydr[i] = o_xydr;
                V.conic[i] = o_con;
                V.tiles[i] = nt;
                dkey = nt ? __float_as_uint(tz) : 0xFFFFFFFFu;
                V.dkeys[i] = dkey;
            }
            warp_hist_add(s_lo[v], dkey & 255u, dkey != 0xFFFFFFFFu);
            const uint32_t kmin = __reduce_min_sync(0xffffffffu, dkey);
            const uint32_t kmax = __reduce_max_sync(0xffffffffu, dkey != 0xFFFFFFFFu ? dkey : 0u);
            if ((threadIdx.x & 31) == 0 && kmin != 0xFFFFFFFFu) {
                atomicMin(&s_kmin[v], kmin);
                atomicMax(&s_kmax[v], kmax);
            }
        }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < nv; v += blockDim.x)
        if (s_kmin[v] <= s_kmax[v]) {
            atomicMin(a.v[v].meta + 5, (unsigned long long)s_kmin[v]);
            atomicMax(a.v[v].meta + 6, (unsigned long long)s_kmax[v]);
        }
    for (int k = threadIdx.x; k < nv * 256; k += blockDim.x) {
        const uint32_t c = (&s_lo[0][0])[k];
        if (c) atomicAdd(&a.v[k >> 8].dhist[k & 255], c);
    }
}

int launch_views_project_fwd(const float* means3, const float* scales3, const float* quats4, const float* opac,
                             int64_t n, const MvFwdArgs& a, cudaStream_t s) {
    if (a.nv <= 0) return 0;
    launch_k(views_init_kernel, dim3(a.nv), dim3(256), 0, s, a);
    if (check_launch("views_init_kernel")) return -1;
    int64_t blocks = (n + 255) / 256;
    if (blocks < 1) blocks = 1;  // the zero jobs run even for an empty scene
    const int64_t cap = (int64_t)sort_sm_count() * 4;
    if (blocks > cap) blocks = cap;
    launch_k(views_project_fwd_kernel, dim3((unsigned)blocks), dim3(256), 0, s, means3, scales3,
             (const float4*)quats4, opac, (int)n, a);
    return check_launch("views_project_fwd_kernel");
}

int launch_project_bwd(const float* means3, const float* scales3, const float* quats4, int64_t n, const CamK& k,
                       const uint32_t* tiles, const float* d_geo4, const float* d_c11, float* d_means3,
                       float* d_scales3, float* d_quats4, float* d_view16, float* partials, cudaStream_t s,
                       bool accumulate, int gstride, const float* rgbo_in, float* rgbo_out,
                       unsigned int* done_counter, unsigned long long* clean_word, unsigned long long clean_sig,
                       bool clear_accum, bool add_view, bool vis_from_grads) {
    int blocks = (int)((n + PBWD_THREADS - 1) / PBWD_THREADS);
    const int resident = sort_sm_count() * PBWD_MINB;
    if (blocks > resident) blocks = resident;
    if (blocks > 0) {
        launch_k(project_bwd_kernel, dim3(blocks), dim3(PBWD_THREADS), 0, s, means3, scales3, (const float4*)quats4,
                 (int)n, k, tiles, (float4*)d_geo4, const_cast<float*>(d_c11), d_means3, d_scales3,
                 (float4*)d_quats4, partials, accumulate, gstride, (float4*)rgbo_in, (float4*)rgbo_out,
                 PBWD_LASTBLOCK ? done_counter : nullptr, d_view16, clean_word, clean_sig, clear_accum,
                 vis_from_grads);
        done_counter = PBWD_LASTBLOCK ? done_counter : nullptr;
        if (check_launch("project_bwd_kernel")) return -1;
        if (done_counter) return 0;  // the last block wrote d_view
    }
    launch_k(view_reduce_kernel, dim3(1), dim3(384), 0, s, (const float*)partials, blocks, d_view16, clean_word,
             clear_accum ? clean_sig : 0ull, add_view);
    return check_launch("view_reduce_kernel");
}

}  // namespace gs

using namespace gs;

extern "C" {

int gs_project_fwd(const float* means3, const float* scales3, const float* quats4, const float* opacities,
                   int64_t n, const gs_camera* cam, float* out_xydr4, float* out_conic4, uint32_t* out_tiles,
                   float* out_cov3, unsigned long long* status, gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_project_fwd: n=%lld out of range", (long long)n);
    if (!cam) return set_error("gs_project_fwd: null camera");
    if (n == 0) return 0;
    const CamK k = make_camk(*cam);
    const int blocks = (int)((n + 255) / 256);
    project_fwd_kernel<0><<<blocks, 256, 0, (cudaStream_t)stream>>>(
        means3, scales3, (const float4*)quats4, opacities, (int)n, k, (float4*)out_xydr4, (float4*)out_conic4,
        out_tiles, out_cov3, status, nullptr, nullptr, ZeroJobs{}, nullptr, nullptr, 0u);
    return check_launch("project_fwd_kernel");
}

size_t gs_project_bwd_workspace_bytes(int64_t n) {
    const int64_t blocks = (n + PBWD_THREADS - 1) / PBWD_THREADS;
    return (size_t)(blocks > 0 ? blocks : 1) * 12 * sizeof(float);
}

int gs_project_bwd(const float* means3, const float* scales3, const float* quats4, int64_t n,
                   const gs_camera* cam, const uint32_t* tiles, const float* d_geo4, const float* d_c11,
                   float* d_means3, float* d_scales3, float* d_quats4, float* d_view16, void* ws,
                   size_t ws_bytes, gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_project_bwd: n=%lld out of range", (long long)n);
    if (!cam) return set_error("gs_project_bwd: null camera");
    if (ws_bytes < gs_project_bwd_workspace_bytes(n)) return set_error("gs_project_bwd: workspace too small");
    const CamK k = make_camk(*cam);
    const int blocks = (int)((n + PBWD_THREADS - 1) / PBWD_THREADS);
    if (blocks > 0) {
        project_bwd_kernel<<<blocks, PBWD_THREADS, 0, (cudaStream_t)stream>>>(
            means3, scales3, (const float4*)quats4, (int)n, k, tiles, (float4*)d_geo4, const_cast<float*>(d_c11),
            d_means3, d_scales3, (float4*)d_quats4, (float*)ws, false, 1, nullptr, nullptr, nullptr, d_view16,
            nullptr, 0ull, false, false);
        if (check_launch("project_bwd_kernel")) return -1;
    }
    view_reduce_kernel<<<1, 384, 0, (cudaStream_t)stream>>>((const float*)ws, blocks, d_view16, nullptr, 0ull, false);
    return check_launch("view_reduce_kernel");
}

}  // extern "C"
