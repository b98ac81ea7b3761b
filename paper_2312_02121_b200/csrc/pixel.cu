// pixel.cu -- the per-pixel API on the device:
//   gs_conic_from_cov        sg/raster_forward.py:86-92  _cov2d_inverse_terms
//   gs_eval_alpha            sg/raster_forward.py:175-196 eval_alpha
//   gs_composite_pixels      sg/raster_forward.py:199-219 composite_pixel
//   gs_composite_pixels_bwd  sg/raster_backward.py:111-163 composite_pixel_backward
//                            and transmittance_replay
//
// Each query is one pixel centre with its own depth-ordered bin (CSR over
// indices into the splat arrays).  One thread per query walks its bin with
// exactly the arithmetic of the tile rasterizers (same splat_sigma_h /
// splat_exp_neg / rcp_approx sequence, every op explicitly rounded), so a
// query at a rendered pixel's centre with that pixel's tile bin reproduces
// the frame's image / final_T / n_contrib bit for bit and the backward's
// per-pixel contributions up to summation order.  These are diagnostics
// and test hooks: one thread per query is the right shape (bins are short,
// queries independent); the frame path never calls them.
#include "common.cuh"

namespace gs {

struct SplatView {
    float x, y, hA, B, hC, opacity, r, g, b;
};

__device__ __forceinline__ SplatView load_splat(const float4* __restrict__ xydr, const float4* __restrict__ conic,
                                                const float* __restrict__ colors, int j) {
    const float4 a = xydr[j];
    const float4 q = conic[j];
    SplatView s;
    s.x = a.x; s.y = a.y;
    s.hA = 0.5f * q.x; s.B = q.y; s.hC = 0.5f * q.z; s.opacity = q.w;
    s.r = colors[3 * j]; s.g = colors[3 * j + 1]; s.b = colors[3 * j + 2];
    return s;
}

// sigma at (px, py), the rasterizers' evaluation order (splat_sigma2 per lane)
__device__ __forceinline__ float query_sigma(const SplatView& s, float px, float py, float& dx, float& dy) {
    dx = __fsub_rn(px, s.x);
    dy = __fsub_rn(py, s.y);
    return splat_sigma_h(dx, __fmul_rn(s.hA, dx), dy, s.B, s.hC);
}

__global__ void __launch_bounds__(256) conic_kernel(const float* __restrict__ cov3, const float* __restrict__ opac,
                                                    float4* __restrict__ conic, int n,
                                                    unsigned long long* __restrict__ status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float ca = cov3[3 * i], cb = cov3[3 * i + 1], cc = cov3[3 * i + 2];
    const float det = cov2d_det(ca, cb, cc);
    if (!(det > 0.f)) {  // sg/raster_forward.py:89-90
        atomicMin(status, ((unsigned long long)i << 8) | (unsigned long long)GS_ERR_COV2D);
        conic[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    conic[i] = conic_of(ca, cb, cc, det, opac[i]);
}

// alpha (0 when skipped), delta, sigma per (splat, pixel) query
__global__ void __launch_bounds__(256) eval_alpha_kernel(const float4* __restrict__ xydr,
                                                         const float4* __restrict__ conic,
                                                         const int32_t* __restrict__ splat,
                                                         const float2* __restrict__ pix, int n,
                                                         float* __restrict__ out_alpha, float2* __restrict__ out_delta,
                                                         float* __restrict__ out_sigma) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int j = splat[q];
    const float4 a = xydr[j];
    const float4 c = conic[j];
    SplatView s;
    s.x = a.x; s.y = a.y; s.hA = 0.5f * c.x; s.B = c.y; s.hC = 0.5f * c.z;
    const float2 p = pix[q];
    float dx, dy;
    const float sg = query_sigma(s, p.x, p.y, dx, dy);
    const float al = fminf(__fmul_rn(c.w, splat_exp_neg(sg)), ALPHA_MAX);
    out_alpha[q] = (sg <= SIGMA_CUT && al >= ALPHA_MIN) ? al : 0.f;  // sg/raster_forward.py:193-195
    out_delta[q] = make_float2(dx, dy);
    out_sigma[q] = sg;
}

// sg/raster_forward.py:116-154 _composite_tile for one pixel per thread
__global__ void __launch_bounds__(128) composite_kernel(const float4* __restrict__ xydr,
                                                        const float4* __restrict__ conic,
                                                        const float* __restrict__ colors,
                                                        const int64_t* __restrict__ bin_ptr,
                                                        const int32_t* __restrict__ bin_idx,
                                                        const float2* __restrict__ pix, int n, float3 bg, bool et,
                                                        float* __restrict__ out_color, float* __restrict__ out_T,
                                                        int32_t* __restrict__ out_nc) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const float2 p = pix[q];
    const int64_t b0 = bin_ptr[q], len = bin_ptr[q + 1] - b0;
    float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f;
    int nc = 0;
    for (int64_t pos = 0; pos < len; ++pos) {
        const SplatView s = load_splat(xydr, conic, colors, bin_idx[b0 + pos]);
        float dx, dy;
        const float sg = query_sigma(s, p.x, p.y, dx, dy);
        if (!(sg <= SIGMA_CUT)) continue;
        const float al = fminf(__fmul_rn(s.opacity, splat_exp_neg(sg)), ALPHA_MAX);
        if (al < ALPHA_MIN) continue;                       // skipped, not counted (:136-139)
        const float ntr = __fmul_rn(T, __fsub_rn(1.f, al));
        if (et && ntr < T_MIN) break;                       // stop without compositing (:141-144)
        const float w = __fmul_rn(al, T);
        cr = __fmaf_rn(w, s.r, cr);
        cg = __fmaf_rn(w, s.g, cg);
        cb = __fmaf_rn(w, s.b, cb);
        T = ntr;
        nc = (int)pos + 1;
    }
    out_color[3 * q] = __fmaf_rn(bg.x, T, cr);              // background term (:153)
    out_color[3 * q + 1] = __fmaf_rn(bg.y, T, cg);
    out_color[3 * q + 2] = __fmaf_rn(bg.z, T, cb);
    out_T[q] = T;
    out_nc[q] = nc;
}

// sg/raster_backward.py:47-108 _backward_tile for one pixel per thread,
// the tile backward's per-pixel arithmetic.  Gradients accumulate
// atomically into per-splat rows (d_rgbo4, d_geo4, d_c11 as gs_raster_bwd);
// t_log (optional, sized like bin_idx) receives the replayed T before each
// contributing entry, NaN elsewhere (transmittance_replay, :138-163).
__global__ void __launch_bounds__(128) composite_bwd_kernel(
    const float4* __restrict__ xydr, const float4* __restrict__ conic, const float* __restrict__ colors,
    const int64_t* __restrict__ bin_ptr, const int32_t* __restrict__ bin_idx, const float2* __restrict__ pix, int n,
    float3 bg, const float* __restrict__ final_T, const int32_t* __restrict__ n_contrib,
    const float* __restrict__ d_pix, float4* __restrict__ d_rgbo, float4* __restrict__ d_geo,
    float* __restrict__ d_c11, float* __restrict__ t_log) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const float2 p = pix[q];
    const int64_t b0 = bin_ptr[q], len = bin_ptr[q + 1] - b0;
    if (t_log) {
        for (int64_t pos = 0; pos < len; ++pos) t_log[b0 + pos] = __int_as_float(0x7fc00000);
    }
    float T = final_T[q];
    const int nc = min((int64_t)n_contrib[q], len);
    const float g0 = d_pix[3 * q], g1 = d_pix[3 * q + 1], g2 = d_pix[3 * q + 2];
    float s0 = __fmul_rn(bg.x, T), s1 = __fmul_rn(bg.y, T), s2 = __fmul_rn(bg.z, T);  // (:58)
    for (int pos = nc - 1; pos >= 0; --pos) {
        const int j = bin_idx[b0 + pos];
        const SplatView s = load_splat(xydr, conic, colors, j);
        float dx, dy;
        const float sg = query_sigma(s, p.x, p.y, dx, dy);
        if (!(sg <= SIGMA_CUT)) continue;
        const float E = splat_exp_neg(sg);
        const float araw = __fmul_rn(s.opacity, E);
        const float al = fminf(araw, ALPHA_MAX);
        if (al < ALPHA_MIN) continue;
        const float inv = rcp_approx(__fsub_rn(1.f, al));
        const float th = __fmul_rn(T, inv);                 // T before this splat (:75)
        if (t_log) t_log[b0 + pos] = th;
        const float w = __fmul_rn(al, th);
        const float cdot = __fmaf_rn(s.b, g2, __fmaf_rn(s.g, g1, __fmul_rn(s.r, g0)));
        const float sdot = __fmaf_rn(s2, g2, __fmaf_rn(s1, g1, __fmul_rn(s0, g0)));
        const float da = __fsub_rn(__fmul_rn(th, cdot), __fmul_rn(inv, sdot));
        const float dal = araw < ALPHA_MAX ? da : 0.f;      // clamped alpha has no opacity/geometry path (:91)
        const float m = __fmul_rn(araw, dal);               // = -d_sigma
        const float y0 = __fmaf_rn(s.B, dy, __fmul_rn(2.f * s.hA, dx));
        const float y1 = __fmaf_rn(2.f * s.hC, dy, __fmul_rn(s.B, dx));
        const float hm = __fmul_rn(0.5f, m);
        const float hy0 = __fmul_rn(hm, y0), hy1 = __fmul_rn(hm, y1);
        atomicAdd(&d_rgbo[j].x, __fmul_rn(w, g0));
        atomicAdd(&d_rgbo[j].y, __fmul_rn(w, g1));
        atomicAdd(&d_rgbo[j].z, __fmul_rn(w, g2));
        atomicAdd(&d_rgbo[j].w, __fmul_rn(dal, E));
        atomicAdd(&d_geo[j].x, __fmul_rn(m, y0));
        atomicAdd(&d_geo[j].y, __fmul_rn(m, y1));
        atomicAdd(&d_geo[j].z, __fmul_rn(hy0, y0));
        atomicAdd(&d_geo[j].w, __fmul_rn(hy0, y1));
        atomicAdd(&d_c11[j], __fmul_rn(hy1, y1));
        s0 = __fmaf_rn(w, s.r, s0);
        s1 = __fmaf_rn(w, s.g, s1);
        s2 = __fmaf_rn(w, s.b, s2);
        T = th;
    }
}

static unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

}  // namespace gs

using namespace gs;

extern "C" {

int gs_conic_from_cov(const float* cov3, const float* opacities, int64_t n, float* out_conic4,
                      unsigned long long* status, gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_conic_from_cov: n out of range");
    if (n == 0) return 0;
    conic_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(cov3, opacities, (float4*)out_conic4, (int)n,
                                                                       status);
    return check_launch("conic_kernel");
}

int gs_eval_alpha(const float* xydr4, const float* conic4, const int32_t* splat, const float* pix2, int64_t n,
                  float* out_alpha, float* out_delta2, float* out_sigma, gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_eval_alpha: n out of range");
    if (n == 0) return 0;
    eval_alpha_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        (const float4*)xydr4, (const float4*)conic4, splat, (const float2*)pix2, (int)n, out_alpha,
        (float2*)out_delta2, out_sigma);
    return check_launch("eval_alpha_kernel");
}

int gs_composite_pixels(const float* xydr4, const float* conic4, const float* colors3, const int64_t* bin_ptr,
                        const int32_t* bin_idx, const float* pix2, int64_t n, const float* background3,
                        int early_termination, float* out_color3, float* out_final_T, int32_t* out_n_contrib,
                        gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_composite_pixels: n out of range");
    if (n == 0) return 0;
    const float3 bg = make_float3(background3[0], background3[1], background3[2]);
    composite_kernel<<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
        (const float4*)xydr4, (const float4*)conic4, colors3, bin_ptr, bin_idx, (const float2*)pix2, (int)n, bg,
        early_termination != 0, out_color3, out_final_T, out_n_contrib);
    return check_launch("composite_kernel");
}

int gs_composite_pixels_bwd(const float* xydr4, const float* conic4, const float* colors3, const int64_t* bin_ptr,
                            const int32_t* bin_idx, const float* pix2, int64_t n, const float* background3,
                            const float* final_T, const int32_t* n_contrib, const float* d_pixels3, float* d_rgbo4,
                            float* d_geo4, float* d_c11, float* t_log, gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_composite_pixels_bwd: n out of range");
    if (n == 0) return 0;
    const float3 bg = make_float3(background3[0], background3[1], background3[2]);
    composite_bwd_kernel<<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
        (const float4*)xydr4, (const float4*)conic4, colors3, bin_ptr, bin_idx, (const float2*)pix2, (int)n, bg,
        final_T, n_contrib, d_pixels3, (float4*)d_rgbo4, (float4*)d_geo4, d_c11, t_log);
    return check_launch("composite_bwd_kernel");
}

}  // extern "C"
