// raster.cu -- stage 3 (front-to-back compositing forward) and stage 4
// (back-to-front replay backward).
//
// Layout: one CTA per 16x16 tile, 128 threads.  Warp w owns the 8x8 quadrant
// (w&1, w>>1) of the tile; lane l owns the two pixels (l&7, l>>3) and
// (l&7, (l>>3)+4) of that quadrant, so the two pixels share a column (and the
// dx of every splat) and a warp covers a compact 8x8 block (good early-stop
// coherence forward, dense contributions backward).  The tile's sorted splat
// records are staged in shared memory 128 at a time.  Bound: FP32 issue.
#include "common.cuh"

namespace gs {

constexpr int RT = 128;  // threads per CTA == splats per staged batch

struct SplatSmem {
    float4 a[RT];  // x, y, hA = A/2, B
    float4 b[RT];  // hC = C/2, opacity, r, g
    float c[RT];   // blue
    uint32_t id[RT];
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

struct PixMap {
    int col, row0, row1;
};

__device__ __forceinline__ PixMap pixel_map(int tile, int tiles_x) {
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    PixMap m;
    m.col = tx * TILE + (warp & 1) * 8 + (lane & 7);
    m.row0 = ty * TILE + (warp >> 1) * 8 + (lane >> 3);
    m.row1 = m.row0 + 4;
    return m;
}

struct FwdPix {
    float T, cr, cg, cb;
    int nc;
    bool done;
};

// One visible-candidate evaluation of sg/raster_forward.py:136-150 for one
// pixel; sigma already passed the cut.
template <bool ET>
__device__ __forceinline__ void fwd_commit(FwdPix& p, float sigma, const float4& bq, float blue, int pos1,
                                           unsigned long long& e_a, unsigned long long& e_c, bool count) {
    const float e = splat_exp_neg(sigma);
    const float alpha = fminf(__fmul_rn(bq.y, e), ALPHA_MAX);
    if (alpha >= ALPHA_MIN) {
        if (count) ++e_a;
        const float nT = __fmul_rn(p.T, __fsub_rn(1.f, alpha));
        if (ET && nT < T_MIN) {
            p.done = true;  // the stopping splat is not composited (:141-144)
            return;
        }
        if (count) ++e_c;
        const float w = __fmul_rn(alpha, p.T);
        p.cr = __fmaf_rn(w, bq.z, p.cr);
        p.cg = __fmaf_rn(w, bq.w, p.cg);
        p.cb = __fmaf_rn(w, blue, p.cb);
        p.T = nT;
        p.nc = pos1;
    }
}

// sg/raster_forward.py:116-154 _composite_tile for one tile.
template <bool ET, bool COUNT>
__global__ void __launch_bounds__(RT) raster_fwd_kernel(const uint2* __restrict__ ranges,
                                                        const uint32_t* __restrict__ sorted_vals,
                                                        const float4* __restrict__ xydr,
                                                        const float4* __restrict__ conic,
                                                        const float* __restrict__ colors, float3 bg, int W, int H,
                                                        int tiles_x, float* __restrict__ out_img,
                                                        float* __restrict__ out_T, int* __restrict__ out_nc,
                                                        unsigned long long* __restrict__ counts) {
    __shared__ SplatSmem s;
    const int tile = blockIdx.x;
    const PixMap pm = pixel_map(tile, tiles_x);
    const bool in0 = pm.col < W && pm.row0 < H;
    const bool in1 = pm.col < W && pm.row1 < H;
    const float px = (float)pm.col + 0.5f;
    const float py0 = (float)pm.row0 + 0.5f, py1 = (float)pm.row1 + 0.5f;
    const uint2 rg = ranges[tile];
    const int start = (int)rg.x, end = (int)rg.y;

    FwdPix p0{1.f, 0.f, 0.f, 0.f, 0, !in0};
    FwdPix p1{1.f, 0.f, 0.f, 0.f, 0, !in1};
    unsigned long long e_f = 0, e_s = 0, e_a = 0, e_c = 0;
    for (int b0 = start; b0 < end; b0 += RT) {
        if (__syncthreads_count(!(p0.done && p1.done)) == 0) break;
        const int j = b0 + (int)threadIdx.x;
        if (j < end) stage_splat(s, threadIdx.x, sorted_vals[j], xydr, conic, colors);
        __syncthreads();
        const int cnt = min(RT, end - b0);
        const int pos_base = b0 - start + 1;
        for (int k = 0; k < cnt; ++k) {
            if (p0.done && p1.done) break;
            const float4 a = s.a[k];
            const float hC = s.b[k].x;
            const float dx = __fsub_rn(px, a.x);
            const float hAdx = __fmul_rn(a.z, dx);
            const float dy0 = __fsub_rn(py0, a.y);
            const float dy1 = __fsub_rn(py1, a.y);
            const float s0 = splat_sigma_h(dx, hAdx, dy0, a.w, hC);
            const float s1 = splat_sigma_h(dx, hAdx, dy1, a.w, hC);
            const bool v0 = !p0.done && s0 <= SIGMA_CUT;
            const bool v1 = !p1.done && s1 <= SIGMA_CUT;
            if (COUNT) {
                e_f += (!p0.done) + (!p1.done);
                e_s += v0 + v1;
            }
            if (v0 || v1) {
                const float4 bq = s.b[k];
                const float blue = s.c[k];
                if (v0) fwd_commit<ET>(p0, s0, bq, blue, pos_base + k, e_a, e_c, COUNT);
                if (v1) fwd_commit<ET>(p1, s1, bq, blue, pos_base + k, e_a, e_c, COUNT);
            }
        }
    }
    if (in0) {
        const int p = pm.row0 * W + pm.col;
        out_img[3 * p] = __fmaf_rn(bg.x, p0.T, p0.cr);
        out_img[3 * p + 1] = __fmaf_rn(bg.y, p0.T, p0.cg);
        out_img[3 * p + 2] = __fmaf_rn(bg.z, p0.T, p0.cb);
        out_T[p] = p0.T;
        out_nc[p] = p0.nc;
    }
    if (in1) {
        const int p = pm.row1 * W + pm.col;
        out_img[3 * p] = __fmaf_rn(bg.x, p1.T, p1.cr);
        out_img[3 * p + 1] = __fmaf_rn(bg.y, p1.T, p1.cg);
        out_img[3 * p + 2] = __fmaf_rn(bg.z, p1.T, p1.cb);
        out_T[p] = p1.T;
        out_nc[p] = p1.nc;
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

struct BwdPix {
    float T, S0, S1, S2, g0, g1, g2;
    int nc;
};

// Accumulators of the 9 per-splat gradient values of one lane.
struct Acc9 {
    float v[9];
};

// sg/raster_backward.py:62-108 for one pixel and one splat whose sigma passed
// the cut and which is active (pos < n_contrib).
__device__ __forceinline__ bool bwd_pixel(BwdPix& p, float sigma, float dx, float dy, const float4& a,
                                          const float4& bq, float blue, Acc9& acc) {
    const float e = splat_exp_neg(sigma);
    const float araw = __fmul_rn(bq.y, e);
    const float alpha = fminf(araw, ALPHA_MAX);
    if (!(alpha >= ALPHA_MIN)) return false;
    const float inv = __frcp_rn(1.f - alpha);
    const float th = p.T * inv;  // T before this splat (:75)
    const float w = alpha * th;
    acc.v[0] = fmaf(w, p.g0, acc.v[0]);
    acc.v[1] = fmaf(w, p.g1, acc.v[1]);
    acc.v[2] = fmaf(w, p.g2, acc.v[2]);
    // d alpha = sum_k (c_k T_here - S_k / (1 - alpha)) g_k  (:86-90)
    const float da = th * (bq.z * p.g0 + bq.w * p.g1 + blue * p.g2) - inv * (p.S0 * p.g0 + p.S1 * p.g1 + p.S2 * p.g2);
    if (araw < ALPHA_MAX) {  // live (:91)
        acc.v[3] = fmaf(da, e, acc.v[3]);
        const float m = araw * da;  // = -d_sigma
        const float y0 = 2.f * a.z * dx + a.w * dy;
        const float y1 = a.w * dx + 2.f * bq.x * dy;
        acc.v[4] = fmaf(m, y0, acc.v[4]);   // d mean2d = -d_sigma * y  (:97-98)
        acc.v[5] = fmaf(m, y1, acc.v[5]);
        const float hm = 0.5f * m;           // d cov2d = -1/2 d_sigma y y^T (:99-105)
        acc.v[6] = fmaf(hm * y0, y0, acc.v[6]);
        acc.v[7] = fmaf(hm * y0, y1, acc.v[7]);
        acc.v[8] = fmaf(hm * y1, y1, acc.v[8]);
    }
    p.S0 = fmaf(w, bq.z, p.S0);
    p.S1 = fmaf(w, bq.w, p.S1);
    p.S2 = fmaf(w, blue, p.S2);
    p.T = th;
    return true;
}

// Transposed warp reduction of 8 values: after it, lane L with (L & 3) == 0
// holds the warp total of value index L >> 2.  9 shuffles instead of 40.
__device__ __forceinline__ float warp_reduce8(const float* v, int lane) {
    float r4[4], r2[2];
    const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float send = b16 ? v[j] : v[j + 4];
        const float keep = b16 ? v[j + 4] : v[j];
        r4[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const float send = b8 ? r4[j] : r4[j + 2];
        const float keep = b8 ? r4[j + 2] : r4[j];
        r2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const float send = b4 ? r2[0] : r2[1];
    const float keep = b4 ? r2[1] : r2[0];
    float r = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    return r;
}

// sg/raster_backward.py:47-108 _backward_tile for one tile.  Per splat the
// 9 gradient values of the warp's 64 pixels are summed per lane, transposed-
// reduced across the warp, and 8 lanes (+1 for d_cov11) issue one vector of
// global reductions per warp per Gaussian.
template <bool COUNT>
__global__ void __launch_bounds__(RT) raster_bwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ sorted_vals, const float4* __restrict__ xydr,
    const float4* __restrict__ conic, const float* __restrict__ colors, float3 bg, int W, int H, int tiles_x,
    const float* __restrict__ final_T, const int* __restrict__ n_contrib, const float* __restrict__ d_img,
    float4* __restrict__ d_rgbo, float4* __restrict__ d_geo, float* __restrict__ d_c11,
    unsigned long long* __restrict__ counts) {
    __shared__ SplatSmem s;
    __shared__ int s_max[RT / 32];
    const int tile = blockIdx.x;
    const PixMap pm = pixel_map(tile, tiles_x);
    const bool in0 = pm.col < W && pm.row0 < H;
    const bool in1 = pm.col < W && pm.row1 < H;
    const float px = (float)pm.col + 0.5f;
    const float py0 = (float)pm.row0 + 0.5f, py1 = (float)pm.row1 + 0.5f;
    const uint2 rg = ranges[tile];
    const int start = (int)rg.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    BwdPix p0{1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0};
    BwdPix p1{1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0};
    if (in0) {
        const int p = pm.row0 * W + pm.col;
        p0.T = final_T[p];
        p0.nc = n_contrib[p];
        p0.g0 = d_img[3 * p]; p0.g1 = d_img[3 * p + 1]; p0.g2 = d_img[3 * p + 2];
    }
    if (in1) {
        const int p = pm.row1 * W + pm.col;
        p1.T = final_T[p];
        p1.nc = n_contrib[p];
        p1.g0 = d_img[3 * p]; p1.g1 = d_img[3 * p + 1]; p1.g2 = d_img[3 * p + 2];
    }
    p0.S0 = bg.x * p0.T; p0.S1 = bg.y * p0.T; p0.S2 = bg.z * p0.T;
    p1.S0 = bg.x * p1.T; p1.S1 = bg.y * p1.T; p1.S2 = bg.z * p1.T;
    const int warp_max = __reduce_max_sync(0xffffffffu, max(p0.nc, p1.nc));
    if (lane == 0) s_max[warp] = warp_max;
    __syncthreads();
    int max_nc = 0;
#pragma unroll
    for (int w = 0; w < RT / 32; ++w) max_nc = max(max_nc, s_max[w]);
    unsigned long long e_s = 0, e_c = 0;

    for (int bend = max_nc; bend > 0; bend -= RT) {
        const int bstart = max(0, bend - RT);
        __syncthreads();
        const int k0 = (int)threadIdx.x;
        if (bstart + k0 < bend) stage_splat(s, k0, sorted_vals[start + bstart + k0], xydr, conic, colors);
        __syncthreads();
        const int kmax = min(bend, warp_max) - bstart;  // positions >= warp_max are inactive for this warp
        for (int k = kmax - 1; k >= 0; --k) {
            const int pos = bstart + k;
            const float4 a = s.a[k];
            const float hC = s.b[k].x;
            const float dx = __fsub_rn(px, a.x);
            const float hAdx = __fmul_rn(a.z, dx);
            const float dy0 = __fsub_rn(py0, a.y);
            const float dy1 = __fsub_rn(py1, a.y);
            const float s0 = splat_sigma_h(dx, hAdx, dy0, a.w, hC);
            const float s1 = splat_sigma_h(dx, hAdx, dy1, a.w, hC);
            const bool v0 = pos < p0.nc && s0 <= SIGMA_CUT;
            const bool v1 = pos < p1.nc && s1 <= SIGMA_CUT;
            if (COUNT) e_s += v0 + v1;
            if (!__any_sync(0xffffffffu, v0 || v1)) continue;
            const float4 bq = s.b[k];
            const float blue = s.c[k];
            Acc9 acc;
#pragma unroll
            for (int q = 0; q < 9; ++q) acc.v[q] = 0.f;
            bool c0 = false, c1 = false;
            if (v0) c0 = bwd_pixel(p0, s0, dx, dy0, a, bq, blue, acc);
            if (v1) c1 = bwd_pixel(p1, s1, dx, dy1, a, bq, blue, acc);
            if (COUNT) e_c += c0 + c1;
            if (!__any_sync(0xffffffffu, c0 || c1)) continue;
            const float r = warp_reduce8(acc.v, lane);
            float c11 = acc.v[8];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c11 += __shfl_xor_sync(0xffffffffu, c11, o);
            const uint32_t id = s.id[k];
            if ((lane & 3) == 0) {
                const int idx = lane >> 2;
                float* dst = idx < 4 ? reinterpret_cast<float*>(&d_rgbo[id]) + idx
                                     : reinterpret_cast<float*>(&d_geo[id]) + (idx - 4);
                atomicAdd(dst, r);
            }
            if (lane == 0) atomicAdd(&d_c11[id], c11);
        }
    }
    if (COUNT) {
        unsigned long long e_b = (unsigned long long)(p0.nc + p1.nc);
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
    raster_fwd_kernel<ET, CNT><<<nt, RT, 0, s>>>((const uint2*)ranges2, sorted_vals, (const float4*)xydr4,    \
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
        raster_bwd_kernel<true><<<nt, RT, 0, s>>>((const uint2*)ranges2, sorted_vals, (const float4*)xydr4,
                                                  (const float4*)conic4, colors3, bg, width, height, tiles_x,
                                                  final_T, n_contrib, d_image, (float4*)d_rgbo4, (float4*)d_geo4,
                                                  d_c11, counts);
    else
        raster_bwd_kernel<false><<<nt, RT, 0, s>>>((const uint2*)ranges2, sorted_vals, (const float4*)xydr4,
                                                   (const float4*)conic4, colors3, bg, width, height, tiles_x,
                                                   final_T, n_contrib, d_image, (float4*)d_rgbo4,
                                                   (float4*)d_geo4, d_c11, counts);
    return check_launch("raster_bwd_kernel");
}

}  // extern "C"
