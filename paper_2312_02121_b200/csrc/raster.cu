// raster.cu -- stage 3 (front-to-back compositing forward) and stage 4
// (back-to-front replay backward).  One CTA per 16x16 tile, one pixel per
// thread; splat records of the tile's sorted list are staged in shared
// memory a batch at a time.  Bound: FP32 issue (DESIGN.md roofline).
#include "common.cuh"

namespace gs {

constexpr int RB = TILE_PIX;  // batch size == threads per CTA == 256

struct SplatSmem {
    float4 a[RB];  // x, y, hA = A/2, B
    float4 b[RB];  // hC = C/2, opacity, r, g
    float c[RB];   // b (blue)
    uint32_t id[RB];
};

__device__ __forceinline__ void stage_splat(SplatSmem& s, int k, uint32_t id, const float4* __restrict__ xydr,
                                            const float4* __restrict__ conic, const float* __restrict__ colors) {
    const float4 g = xydr[id];
    const float4 q = conic[id];
    const float r = colors[3 * id], gg = colors[3 * id + 1], bb = colors[3 * id + 2];
    s.a[k] = make_float4(g.x, g.y, 0.5f * q.x, q.y);
    s.b[k] = make_float4(0.5f * q.z, q.w, r, gg);
    s.c[k] = bb;
    s.id[k] = id;
}

// sg/raster_forward.py:116-154 _composite_tile for one tile, per pixel:
//   sigma -> alpha = min(o e^-sigma, 0.999) -> visible = sigma<=4.5 & alpha>=1/255
//   -> nT = T(1-alpha); ET: nT < 1e-4 stops WITHOUT compositing -> else
//   C += alpha T c, T = nT, n_contrib = pos + 1; finally C += bg T.
template <bool ET, bool COUNT>
__global__ void __launch_bounds__(RB) raster_fwd_kernel(const uint2* __restrict__ ranges,
                                                        const uint32_t* __restrict__ sorted_vals,
                                                        const float4* __restrict__ xydr,
                                                        const float4* __restrict__ conic,
                                                        const float* __restrict__ colors, float3 bg, int W, int H,
                                                        int tiles_x, float* __restrict__ out_img,
                                                        float* __restrict__ out_T, int* __restrict__ out_nc,
                                                        unsigned long long* __restrict__ counts) {
    __shared__ SplatSmem s;
    const int tile = blockIdx.x;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int col = tx * TILE + (threadIdx.x & (TILE - 1));
    const int row = ty * TILE + (threadIdx.x >> 4);
    const bool inside = col < W && row < H;
    const float px = (float)col + 0.5f, py = (float)row + 0.5f;
    const uint2 rg = ranges[tile];
    const int start = (int)rg.x, end = (int)rg.y;

    float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f;
    int nc = 0;
    bool done = !inside;
    unsigned long long e_f = 0, e_s = 0, e_a = 0, e_c = 0;
    for (int b0 = start; b0 < end; b0 += RB) {
        if (__syncthreads_count(!done) == 0) break;
        const int j = b0 + (int)threadIdx.x;
        if (j < end) stage_splat(s, threadIdx.x, sorted_vals[j], xydr, conic, colors);
        __syncthreads();
        const int cnt = min(RB, end - b0);
        if (!done) {
            for (int k = 0; k < cnt; ++k) {
                const float4 a = s.a[k];
                const float hC = s.b[k].x;
                const float dx = __fsub_rn(px, a.x), dy = __fsub_rn(py, a.y);
                const float sigma = splat_sigma(dx, dy, a.z, a.w, hC);
                if (COUNT) ++e_f;
                if (sigma <= SIGMA_CUT) {
                    const float4 bq = s.b[k];
                    const float e = splat_exp_neg(sigma);
                    const float alpha = fminf(__fmul_rn(bq.y, e), ALPHA_MAX);
                    if (COUNT) ++e_s;
                    if (alpha >= ALPHA_MIN) {
                        if (COUNT) ++e_a;
                        const float nT = __fmul_rn(T, __fsub_rn(1.f, alpha));
                        if (ET && nT < T_MIN) {
                            done = true;
                            break;
                        }
                        if (COUNT) ++e_c;
                        const float w = __fmul_rn(alpha, T);
                        cr = __fmaf_rn(w, bq.z, cr);
                        cg = __fmaf_rn(w, bq.w, cg);
                        cb = __fmaf_rn(w, s.c[k], cb);
                        T = nT;
                        nc = b0 - start + k + 1;
                    }
                }
            }
        }
    }
    if (inside) {
        const int p = row * W + col;
        out_img[3 * p] = __fmaf_rn(bg.x, T, cr);
        out_img[3 * p + 1] = __fmaf_rn(bg.y, T, cg);
        out_img[3 * p + 2] = __fmaf_rn(bg.z, T, cb);
        out_T[p] = T;
        out_nc[p] = nc;
    }
    if (COUNT) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            e_f += __shfl_xor_sync(0xffffffffu, e_f, o);
            e_s += __shfl_xor_sync(0xffffffffu, e_s, o);
            e_a += __shfl_xor_sync(0xffffffffu, e_a, o);
            e_c += __shfl_xor_sync(0xffffffffu, e_c, o);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&counts[0], e_f);
            atomicAdd(&counts[1], e_s);
            atomicAdd(&counts[2], e_a);
            atomicAdd(&counts[3], e_c);
        }
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// sg/raster_backward.py:47-108 _backward_tile for one tile, per pixel:
// seed T = final_T, S = bg final_T; walk pos = max(n_contrib)-1 .. 0, replay
// the forward's contrib decision, T_here = T/(1-alpha), accumulate dc, d_alpha,
// live = contrib & alpha_raw < 0.999 -> d_opacity, d_sigma -> d_mean2d and
// the full-matrix d_cov2d; S += w c; T = T_here.  Per splat, the 9 gradient
// values are warp-shuffle reduced and ONE lane per warp adds them to global
// memory with vector reductions (red.global.add.v4.f32).
template <bool COUNT>
__global__ void __launch_bounds__(RB) raster_bwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ sorted_vals, const float4* __restrict__ xydr,
    const float4* __restrict__ conic, const float* __restrict__ colors, float3 bg, int W, int H, int tiles_x,
    const float* __restrict__ final_T, const int* __restrict__ n_contrib, const float* __restrict__ d_img,
    float4* __restrict__ d_rgbo, float4* __restrict__ d_geo, float* __restrict__ d_c11,
    unsigned long long* __restrict__ counts) {
    __shared__ SplatSmem s;
    __shared__ int s_max[RB / 32];
    const int tile = blockIdx.x;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int col = tx * TILE + (threadIdx.x & (TILE - 1));
    const int row = ty * TILE + (threadIdx.x >> 4);
    const bool inside = col < W && row < H;
    const float px = (float)col + 0.5f, py = (float)row + 0.5f;
    const uint2 rg = ranges[tile];
    const int start = (int)rg.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    float T = 1.f, g0 = 0.f, g1 = 0.f, g2 = 0.f;
    int nc = 0;
    if (inside) {
        const int p = row * W + col;
        T = final_T[p];
        nc = n_contrib[p];
        g0 = d_img[3 * p];
        g1 = d_img[3 * p + 1];
        g2 = d_img[3 * p + 2];
    }
    float S0 = bg.x * T, S1 = bg.y * T, S2 = bg.z * T;
    const int wmax = __reduce_max_sync(0xffffffffu, nc);
    if (lane == 0) s_max[warp] = wmax;
    __syncthreads();
    int max_nc = 0;
#pragma unroll
    for (int w = 0; w < RB / 32; ++w) max_nc = max(max_nc, s_max[w]);
    unsigned long long e_s = 0, e_c = 0;

    for (int bend = max_nc; bend > 0; bend -= RB) {
        const int bstart = max(0, bend - RB);
        __syncthreads();
        const int k0 = (int)threadIdx.x;
        if (bstart + k0 < bend) stage_splat(s, k0, sorted_vals[start + bstart + k0], xydr, conic, colors);
        __syncthreads();
        for (int k = bend - bstart - 1; k >= 0; --k) {
            const int pos = bstart + k;
            const float4 a = s.a[k];
            const float4 bq = s.b[k];
            const float dx = __fsub_rn(px, a.x), dy = __fsub_rn(py, a.y);
            const float sigma = splat_sigma(dx, dy, a.z, a.w, bq.x);
            const float e = splat_exp_neg(sigma);
            const float araw = __fmul_rn(bq.y, e);
            const float alpha = fminf(araw, ALPHA_MAX);
            const bool act = pos < nc;
            const bool sig_ok = act && sigma <= SIGMA_CUT;
            const bool contrib = sig_ok && alpha >= ALPHA_MIN;
            if (COUNT) {
                e_s += sig_ok;
                e_c += contrib;
            }
            if (!__any_sync(0xffffffffu, contrib)) continue;
            float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, v4 = 0.f, v5 = 0.f, v6 = 0.f, v7 = 0.f, v8 = 0.f;
            if (contrib) {
                const float cb = s.c[k];
                const float inv = __frcp_rn(1.f - alpha);
                const float th = T * inv;
                const float w = alpha * th;
                v0 = w * g0;
                v1 = w * g1;
                v2 = w * g2;
                const float da = th * (bq.z * g0 + bq.w * g1 + cb * g2) - inv * (S0 * g0 + S1 * g1 + S2 * g2);
                if (araw < ALPHA_MAX) {
                    v3 = da * e;
                    const float m = araw * da;  // = -d_sigma
                    const float y0 = 2.f * a.z * dx + a.w * dy;
                    const float y1 = a.w * dx + 2.f * bq.x * dy;
                    v4 = m * y0;
                    v5 = m * y1;
                    const float hm = 0.5f * m;
                    v6 = hm * y0 * y0;
                    v7 = hm * y0 * y1;
                    v8 = hm * y1 * y1;
                }
                S0 += w * bq.z;
                S1 += w * bq.w;
                S2 += w * cb;
                T = th;
            }
            v0 = warp_sum(v0); v1 = warp_sum(v1); v2 = warp_sum(v2);
            v3 = warp_sum(v3); v4 = warp_sum(v4); v5 = warp_sum(v5);
            v6 = warp_sum(v6); v7 = warp_sum(v7); v8 = warp_sum(v8);
            if (lane == 0) {
                const uint32_t id = s.id[k];
                red_add_v4(&d_rgbo[id], v0, v1, v2, v3);
                red_add_v4(&d_geo[id], v4, v5, v6, v7);
                atomicAdd(&d_c11[id], v8);
            }
        }
    }
    if (COUNT) {
        unsigned long long e_b = (unsigned long long)nc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            e_b += __shfl_xor_sync(0xffffffffu, e_b, o);
            e_s += __shfl_xor_sync(0xffffffffu, e_s, o);
            e_c += __shfl_xor_sync(0xffffffffu, e_c, o);
        }
        if (lane == 0) {
            atomicAdd(&counts[0], e_b);
            atomicAdd(&counts[1], e_s);
            atomicAdd(&counts[2], e_c);
        }
    }
}

}  // namespace gs

using namespace gs;

extern "C" {

int gs_raster_fwd(const uint32_t* ranges2, const uint32_t* sorted_vals, const float* xydr4, const float* conic4,
                  const float* colors3, const float* background3, int32_t width, int32_t height,
                  int early_termination, float* out_image, float* out_final_T, int32_t* out_n_contrib,
                  unsigned long long* counts, gs_stream_t stream) {
    if (width < 1 || height < 1) return set_error("gs_raster_fwd: bad image size %dx%d", width, height);
    const int tiles_x = (width + TILE - 1) / TILE, tiles_y = (height + TILE - 1) / TILE;
    const float3 bg = make_float3(background3[0], background3[1], background3[2]);
    const unsigned nt = (unsigned)(tiles_x * tiles_y);
    cudaStream_t s = (cudaStream_t)stream;
#define GS_LAUNCH_FWD(ET, CNT)                                                                                 \
    raster_fwd_kernel<ET, CNT><<<nt, RB, 0, s>>>((const uint2*)ranges2, sorted_vals, (const float4*)xydr4,    \
                                                 (const float4*)conic4, colors3, bg, width, height, tiles_x, \
                                                 out_image, out_final_T, out_n_contrib, counts)
    if (early_termination) {
        if (counts) GS_LAUNCH_FWD(true, true); else GS_LAUNCH_FWD(true, false);
    } else {
        if (counts) GS_LAUNCH_FWD(false, true); else GS_LAUNCH_FWD(false, false);
    }
#undef GS_LAUNCH_FWD
    return check_launch("raster_fwd_kernel");
}

int gs_raster_bwd(const uint32_t* ranges2, const uint32_t* sorted_vals, const float* xydr4, const float* conic4,
                  const float* colors3, const float* background3, int32_t width, int32_t height,
                  const float* final_T, const int32_t* n_contrib, const float* d_image, float* d_rgbo4,
                  float* d_geo4, float* d_c11, unsigned long long* counts, gs_stream_t stream) {
    if (width < 1 || height < 1) return set_error("gs_raster_bwd: bad image size %dx%d", width, height);
    const int tiles_x = (width + TILE - 1) / TILE, tiles_y = (height + TILE - 1) / TILE;
    const float3 bg = make_float3(background3[0], background3[1], background3[2]);
    const unsigned nt = (unsigned)(tiles_x * tiles_y);
    cudaStream_t s = (cudaStream_t)stream;
    if (counts)
        raster_bwd_kernel<true><<<nt, RB, 0, s>>>((const uint2*)ranges2, sorted_vals, (const float4*)xydr4,
                                                  (const float4*)conic4, colors3, bg, width, height, tiles_x,
                                                  final_T, n_contrib, d_image, (float4*)d_rgbo4, (float4*)d_geo4,
                                                  d_c11, counts);
    else
        raster_bwd_kernel<false><<<nt, RB, 0, s>>>((const uint2*)ranges2, sorted_vals, (const float4*)xydr4,
                                                   (const float4*)conic4, colors3, bg, width, height, tiles_x,
                                                   final_T, n_contrib, d_image, (float4*)d_rgbo4,
                                                   (float4*)d_geo4, d_c11, counts);
    return check_launch("raster_bwd_kernel");
}

}  // extern "C"
