// raster.cu -- stage 3 (front-to-back compositing forward) and stage 4
// (back-to-front replay backward).
//
// Layout: one CTA per 16x16 tile, 256/PX threads, PX pixels per thread.
//   PX = 2: 4 warps, each an 8x8 quadrant of the tile;
//   PX = 4: 2 warps, each 8 columns x 16 rows;
//   PX = 8: 1 warp for the whole tile.
// A thread's PX pixels share one column (hence dx and hA*dx of every splat).
// The tile's sorted splat records are staged in shared memory RB = 128 at a
// time.  Bound: FP32 issue (DESIGN.md roofline).
//
// Region masks: while staging, every splat's bounding square (radius r, the
// square sg/binning.py:35-46 bins by), grown by one pixel, is tested against
// each warp's pixel region; a warp then walks only the set bits of its own
// mask.  A skipped (pixel, splat) pair lies more than one pixel outside the
// 3-sigma square, so sigma > 4.5 there with a wide margin: the skip never
// changes a decision, and forward and backward (same PX, same test) replay
// identical evaluation sequences.
//
// Retired pixels (forward: out of the image or early-terminated) get
// py = +inf, so their sigma is inf/NaN and fails the cut: the hot loop needs
// no per-pixel "done" test.
#include <cstdlib>

#include "common.cuh"
#include "internal.cuh"

namespace gs {

constexpr int RB = 128;       // splats per staged batch
constexpr int MW = RB / 32;   // mask words per warp region

struct SplatSmem {
    float4 a[RB];  // x, y, hA = A/2, B
    float4 b[RB];  // hC = C/2, opacity, r, g
    float c[RB];   // blue
    uint32_t id[RB];
};

// Keep a loop-invariant value in a register (stops ptxas from
// rematerialising it inside the hot loop).
__device__ __forceinline__ float pin(float x) {
    asm volatile("" : "+f"(x));
    return x;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int PX>
struct TileGeom {
    static constexpr int THREADS = TILE_PIX / PX;
    static constexpr int NW = THREADS / 32;
    static constexpr int LC = NW >= 2 ? 8 : 16;    // columns covered by one warp
    static constexpr int RS = 32 / LC;             // row stride between a thread's pixels
    static constexpr int WROWS = NW == 4 ? 8 : 16;  // rows covered by one warp
    int col;
    int row[PX];
    __device__ __forceinline__ TileGeom(int tile, int tiles_x) {
        const int tx = tile % tiles_x, ty = tile / tiles_x;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        col = tx * TILE + (NW >= 2 ? (warp & 1) * 8 : 0) + (lane % LC);
        const int base = NW == 4 ? (warp >> 1) * 8 : 0;
#pragma unroll
        for (int k = 0; k < PX; ++k) row[k] = ty * TILE + base + (lane / LC) + RS * k;
    }
    // pixel-centre bounds of warp w's region
    __device__ __forceinline__ static void region(int tile, int tiles_x, int w, float& x0, float& x1, float& y0,
                                                  float& y1) {
        const int tx = tile % tiles_x, ty = tile / tiles_x;
        const int c0 = tx * TILE + (NW >= 2 ? (w & 1) * 8 : 0);
        const int r0 = ty * TILE + (NW == 4 ? (w >> 1) * 8 : 0);
        x0 = (float)c0 + 0.5f;
        x1 = (float)(c0 + LC - 1) + 0.5f;
        y0 = (float)r0 + 0.5f;
        y1 = (float)(r0 + WROWS - 1) + 0.5f;
    }
};

// Stage splat k of the batch and publish, per warp region, whether its
// (grown) bounding square reaches that region.
template <int PX>
__device__ __forceinline__ void stage_batch(SplatSmem& s, uint32_t (*s_mask)[MW], int tile, int tiles_x,
                                            const uint32_t* __restrict__ ids, int first, int count,
                                            const float4* __restrict__ xydr, const float4* __restrict__ conic,
                                            const float* __restrict__ colors) {
    using G = TileGeom<PX>;
    constexpr int NT = G::THREADS, PER = RB / NT;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int k = u * NT + (int)threadIdx.x;
        const bool valid = k < count;
        float x = 0.f, y = 0.f, r = -1e30f;
        if (valid) {
            const uint32_t id = ids[first + k];
            const float4 g = xydr[id];
            const float4 q = conic[id];
            s.a[k] = make_float4(g.x, g.y, 0.5f * q.x, q.y);
            s.b[k] = make_float4(0.5f * q.z, q.w, colors[3 * id], colors[3 * id + 1]);
            s.c[k] = colors[3 * id + 2];
            s.id[k] = id;
            x = g.x;
            y = g.y;
            r = (float)__float_as_int(g.w) + 1.f;
        }
#pragma unroll
        for (int w = 0; w < G::NW; ++w) {
            float x0, x1, y0, y1;
            G::region(tile, tiles_x, w, x0, x1, y0, y1);
            const bool ov = valid && x + r >= x0 && x - r <= x1 && y + r >= y0 && y - r <= y1;
            const uint32_t m = __ballot_sync(0xffffffffu, ov);
            if (lane == 0) s_mask[w][u * G::NW + warp] = m;
        }
    }
}

// ============================================================ forward
// sg/raster_forward.py:116-154 _composite_tile for one tile.
template <int PX, bool ET, bool COUNT>
__global__ void __launch_bounds__(TileGeom<PX>::THREADS) raster_fwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ sorted_vals, const float4* __restrict__ xydr,
    const float4* __restrict__ conic, const float* __restrict__ colors, float3 bg, int W, int H, int tiles_x,
    float* __restrict__ out_img, float* __restrict__ out_T, int* __restrict__ out_nc,
    unsigned long long* __restrict__ counts) {
    using G = TileGeom<PX>;
    __shared__ SplatSmem s;
    __shared__ uint32_t s_mask[G::NW][MW];
    const int tile = blockIdx.x;
    const int warp = threadIdx.x >> 5;
    const G geo(tile, tiles_x);
    const float INF = __int_as_float(0x7f800000);
    static_assert(PX % 2 == 0, "pixels are evaluated in f32x2 pairs");
    constexpr int NP = PX / 2;
    const float px = pin((float)geo.col + 0.5f);
    float py[PX], T[PX], cr[PX], cg[PX], cb[PX];
    int nc[PX], stop[PX];
    f32x2 PY[NP];
    unsigned done = 0;
#pragma unroll
    for (int q = 0; q < PX; ++q) {
        const bool in = geo.col < W && geo.row[q] < H;
        py[q] = in ? (float)geo.row[q] + 0.5f : INF;
        done |= in ? 0u : (1u << q);
        T[q] = 1.f; cr[q] = 0.f; cg[q] = 0.f; cb[q] = 0.f; nc[q] = 0; stop[q] = -1;
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) PY[j] = pin2(pk2(py[2 * j], py[2 * j + 1]));
    constexpr unsigned ALL = (1u << PX) - 1u;
    const uint2 rg = ranges[tile];
    const int start = (int)rg.x, end = (int)rg.y;
    unsigned long long e_s = 0, e_a = 0, e_c = 0;

    for (int b0 = start; b0 < end; b0 += RB) {
        if (__syncthreads_count(done != ALL) == 0) break;
        stage_batch<PX>(s, s_mask, tile, tiles_x, sorted_vals, b0, min(RB, end - b0), xydr, conic, colors);
        __syncthreads();
        if (__all_sync(0xffffffffu, done == ALL)) continue;  // whole warp finished: only help staging
        const int pos_base = b0 - start + 1;
        bool warp_done = false;
        // composite splat k (sigma already evaluated) into the visible pixels
        auto slow = [&](int k, const float* sg, const bool* vis) {
            const float4 bq = s.b[k];
            const float blue = s.c[k];
#pragma unroll
            for (int q = 0; q < PX; ++q) {
                if (!vis[q]) continue;
                const float e = splat_exp_neg(sg[q]);
                const float alpha = fminf(__fmul_rn(bq.y, e), ALPHA_MAX);
                if (!(alpha >= ALPHA_MIN)) continue;
                if (COUNT) ++e_a;
                const float nT = __fmul_rn(T[q], __fsub_rn(1.f, alpha));
                if (ET && nT < T_MIN) {  // stop WITHOUT compositing (:141-144)
                    py[q] = INF;
                    PY[q / 2] = pk2(py[q & ~1], py[q | 1]);
                    done |= 1u << q;
                    stop[q] = pos_base + k;
                    continue;
                }
                if (COUNT) ++e_c;
                const float w = __fmul_rn(alpha, T[q]);
                cr[q] = __fmaf_rn(w, bq.z, cr[q]);
                cg[q] = __fmaf_rn(w, bq.w, cg[q]);
                cb[q] = __fmaf_rn(w, blue, cb[q]);
                T[q] = nT;
                nc[q] = pos_base + k;
            }
        };
#pragma unroll 1
        for (int j = 0; j < MW && !warp_done; ++j) {
            uint32_t m = s_mask[warp][j];
            while (m) {
                // two splats per iteration: independent sigma chains (ILP),
                // compositing still strictly in list order
                const int k0 = j * 32 + (__ffs(m) - 1);
                m &= m - 1;
                const bool has1 = m != 0;
                const int k1 = has1 ? j * 32 + (__ffs(m) - 1) : k0;
                m &= m - 1;
                const float4 a0 = s.a[k0], a1 = s.a[k1];
                const float hC0 = s.b[k0].x, hC1 = s.b[k1].x;
                const float dx0 = __fsub_rn(px, a0.x), dx1 = __fsub_rn(px, a1.x);
                const float hAdx0 = __fmul_rn(a0.z, dx0), hAdx1 = __fmul_rn(a1.z, dx1);
                float sg0[PX], sg1[PX];
                bool vis0[PX], vis1[PX];
                bool any0 = false, any1 = false;
#pragma unroll
                for (int t = 0; t < NP; ++t) {
                    upk2(splat_sigma2(dx0, hAdx0, sub2(PY[t], pk2(a0.y, a0.y)), a0.w, hC0), sg0[2 * t],
                         sg0[2 * t + 1]);
                    upk2(splat_sigma2(dx1, hAdx1, sub2(PY[t], pk2(a1.y, a1.y)), a1.w, hC1), sg1[2 * t],
                         sg1[2 * t + 1]);
                }
#pragma unroll
                for (int q = 0; q < PX; ++q) {
                    vis0[q] = sg0[q] <= SIGMA_CUT;  // false for retired pixels (py = inf)
                    vis1[q] = has1 && sg1[q] <= SIGMA_CUT;
                    any0 |= vis0[q];
                    any1 |= vis1[q];
                }
                const uint32_t v0 = __ballot_sync(0xffffffffu, any0);
                const uint32_t v1 = __ballot_sync(0xffffffffu, any1);
                if (COUNT) {
#pragma unroll
                    for (int q = 0; q < PX; ++q) e_s += vis0[q];
                }
                if (v0) slow(k0, sg0, vis0);
                if (v1) {
#pragma unroll
                    for (int q = 0; q < PX; ++q) vis1[q] = vis1[q] && !((done >> q) & 1u);  // retired at k0
                    if (COUNT) {
#pragma unroll
                        for (int q = 0; q < PX; ++q) e_s += vis1[q];
                    }
                    slow(k1, sg1, vis1);
                } else if (COUNT && has1) {
#pragma unroll
                    for (int q = 0; q < PX; ++q) e_s += vis1[q] && !((done >> q) & 1u);
                }
                if (ET && (v0 | v1) && __all_sync(0xffffffffu, done == ALL)) {
                    warp_done = true;
                    break;
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < PX; ++q) {
        if (geo.col < W && geo.row[q] < H) {
            const int p = geo.row[q] * W + geo.col;
            out_img[3 * p] = __fmaf_rn(bg.x, T[q], cr[q]);
            out_img[3 * p + 1] = __fmaf_rn(bg.y, T[q], cg[q]);
            out_img[3 * p + 2] = __fmaf_rn(bg.z, T[q], cb[q]);
            out_T[p] = T[q];
            out_nc[p] = nc[q];
        }
    }
    if (COUNT) {
        // E_f: (pixel, entry) pairs the reference visits while not done =
        // entries up to and including the stopping one, else the whole list
        unsigned long long e_f = 0;
#pragma unroll
        for (int q = 0; q < PX; ++q)
            if (geo.col < W && geo.row[q] < H) e_f += (unsigned long long)(stop[q] >= 0 ? stop[q] : end - start);
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

// ============================================================ backward

// Transposed warp reduction of 8 values: afterwards lane L with (L & 3) == 0
// holds the warp total of value index L >> 2 (9 shuffles instead of 40).
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

// sg/raster_backward.py:47-108 _backward_tile for one tile: seed T = final_T,
// S = bg * final_T; walk pos = max(n_contrib)-1 .. 0 replaying the forward's
// decisions (same sigma/exp code, same region masks); contrib ->
// T_here = T/(1-alpha), w = alpha T_here, dc += w g,
// d_alpha = T_here c.g - S.g/(1-alpha); live (alpha_raw < 0.999) ->
// d_opacity += d_alpha e^-sigma, d_sigma = -alpha_raw d_alpha,
// d_mean2d += -d_sigma y, d_cov2d += -d_sigma/2 y y^T with y = conic * delta
// (full-matrix convention, :99-105); S += w c; T = T_here.  Per splat the
// warp's 9 sums are transposed-reduced and 8 (+1) lanes issue one global
// reduction each: one atomic per warp per Gaussian value.
template <int PX, bool COUNT>
__global__ void __launch_bounds__(TileGeom<PX>::THREADS) raster_bwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ sorted_vals, const float4* __restrict__ xydr,
    const float4* __restrict__ conic, const float* __restrict__ colors, float3 bg, int W, int H, int tiles_x,
    const float* __restrict__ final_T, const int* __restrict__ n_contrib, const float* __restrict__ d_img,
    float4* __restrict__ d_rgbo, float4* __restrict__ d_geo, float* __restrict__ d_c11,
    unsigned long long* __restrict__ counts) {
    using G = TileGeom<PX>;
    constexpr int NW = G::NW;
    __shared__ SplatSmem s;
    __shared__ uint32_t s_mask[NW][MW];
    __shared__ int s_max[NW];
    const int tile = blockIdx.x;
    const G geo(tile, tiles_x);
    static_assert(PX % 2 == 0, "pixels are evaluated in f32x2 pairs");
    constexpr int NP = PX / 2;
    const float px = pin((float)geo.col + 0.5f);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float py[PX], T[PX], S0[PX], S1[PX], S2[PX], g0[PX], g1[PX], g2[PX];
    int nc[PX];
    int my_max = 0;
#pragma unroll
    for (int q = 0; q < PX; ++q) {
        const bool in = geo.col < W && geo.row[q] < H;
        py[q] = (float)geo.row[q] + 0.5f;
        T[q] = 1.f; nc[q] = 0; g0[q] = 0.f; g1[q] = 0.f; g2[q] = 0.f;
        if (in) {
            const int p = geo.row[q] * W + geo.col;
            T[q] = final_T[p];
            nc[q] = n_contrib[p];
            g0[q] = d_img[3 * p]; g1[q] = d_img[3 * p + 1]; g2[q] = d_img[3 * p + 2];
        }
        S0[q] = bg.x * T[q]; S1[q] = bg.y * T[q]; S2[q] = bg.z * T[q];
        my_max = max(my_max, nc[q]);
    }
    f32x2 PY[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) PY[j] = pin2(pk2(py[2 * j], py[2 * j + 1]));
    const int warp_max = __reduce_max_sync(0xffffffffu, my_max);
    if (lane == 0) s_max[warp] = warp_max;
    const uint2 rg = ranges[tile];
    const int start = (int)rg.x;
    __syncthreads();
    int max_nc = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) max_nc = max(max_nc, s_max[w]);
    unsigned long long e_s = 0, e_c = 0;

    for (int bend = max_nc; bend > 0; bend -= RB) {
        const int bstart = max(0, bend - RB);
        __syncthreads();
        stage_batch<PX>(s, s_mask, tile, tiles_x, sorted_vals, start + bstart, bend - bstart, xydr, conic, colors);
        __syncthreads();
        const int kmax = min(bend, warp_max) - bstart;  // positions >= warp_max are inactive for this warp
#pragma unroll 1
        for (int j = MW - 1; j >= 0; --j) {
            const int lim = kmax - 32 * j;
            if (lim <= 0) continue;
            uint32_t m = s_mask[warp][j] & (lim >= 32 ? 0xffffffffu : ((1u << lim) - 1u));
            while (m) {
                const int b = 31 - __clz(m);
                m &= ~(1u << b);
                const int k = 32 * j + b;
                const int pos = bstart + k;
                const float4 a = s.a[k];
                const float hC = s.b[k].x;
                const float dx = __fsub_rn(px, a.x);
                const float hAdx = __fmul_rn(a.z, dx);
                float sg[PX], dy[PX];
                bool v[PX];
                bool any = false;
#pragma unroll
                for (int j = 0; j < NP; ++j) {
                    const f32x2 DY = sub2(PY[j], pk2(a.y, a.y));
                    upk2(DY, dy[2 * j], dy[2 * j + 1]);
                    upk2(splat_sigma2(dx, hAdx, DY, a.w, hC), sg[2 * j], sg[2 * j + 1]);
                }
#pragma unroll
                for (int q = 0; q < PX; ++q) {
                    v[q] = pos < nc[q] && sg[q] <= SIGMA_CUT;
                    any |= v[q];
                }
                if (COUNT) {
#pragma unroll
                    for (int q = 0; q < PX; ++q) e_s += v[q];
                }
                if (!__any_sync(0xffffffffu, any)) continue;
                const float4 bq = s.b[k];
                const float blue = s.c[k];
                const float A2 = 2.f * a.z, C2 = 2.f * bq.x;
                float acc[9];
#pragma unroll
                for (int t = 0; t < 9; ++t) acc[t] = 0.f;
                bool anyc = false;
#pragma unroll
                for (int q = 0; q < PX; ++q) {
                    if (!v[q]) continue;
                    const float e = splat_exp_neg(sg[q]);
                    const float araw = __fmul_rn(bq.y, e);
                    const float alpha = fminf(araw, ALPHA_MAX);
                    if (!(alpha >= ALPHA_MIN)) continue;
                    anyc = true;
                    if (COUNT) ++e_c;
                    const float inv = rcp_approx(1.f - alpha);
                    const float th = T[q] * inv;  // T before this splat (:75)
                    const float w = alpha * th;
                    acc[0] = fmaf(w, g0[q], acc[0]);
                    acc[1] = fmaf(w, g1[q], acc[1]);
                    acc[2] = fmaf(w, g2[q], acc[2]);
                    const float cdot = bq.z * g0[q] + bq.w * g1[q] + blue * g2[q];
                    const float sdot = S0[q] * g0[q] + S1[q] * g1[q] + S2[q] * g2[q];
                    const float da = th * cdot - inv * sdot;
                    if (araw < ALPHA_MAX) {  // live (:91)
                        acc[3] = fmaf(da, e, acc[3]);
                        const float mm = araw * da;  // = -d_sigma
                        const float y0 = A2 * dx + a.w * dy[q];
                        const float y1 = a.w * dx + C2 * dy[q];
                        const float hm = 0.5f * mm;
                        acc[4] = fmaf(mm, y0, acc[4]);
                        acc[5] = fmaf(mm, y1, acc[5]);
                        acc[6] = fmaf(hm * y0, y0, acc[6]);
                        acc[7] = fmaf(hm * y0, y1, acc[7]);
                        acc[8] = fmaf(hm * y1, y1, acc[8]);
                    }
                    S0[q] = fmaf(w, bq.z, S0[q]);
                    S1[q] = fmaf(w, bq.w, S1[q]);
                    S2[q] = fmaf(w, blue, S2[q]);
                    T[q] = th;
                }
                const uint32_t cmask = __ballot_sync(0xffffffffu, anyc);
                if (!cmask) continue;
                const uint32_t id = s.id[k];
                if (__popc(cmask) <= 3) {
                    // few contributing lanes: their own vector reductions are
                    // cheaper than a 9-value warp reduction (same or fewer
                    // atomic lane-ops, ~45 fewer instructions)
                    if (anyc) {
                        red_add_v4(&d_rgbo[id], acc[0], acc[1], acc[2], acc[3]);
                        red_add_v4(&d_geo[id], acc[4], acc[5], acc[6], acc[7]);
                        atomicAdd(&d_c11[id], acc[8]);
                    }
                    continue;
                }
                const float r = warp_reduce8(acc, lane);
                float c11 = acc[8];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c11 += __shfl_xor_sync(0xffffffffu, c11, o);
                if ((lane & 3) == 0) {
                    const int idx = lane >> 2;
                    float* dst = idx < 4 ? reinterpret_cast<float*>(&d_rgbo[id]) + idx
                                         : reinterpret_cast<float*>(&d_geo[id]) + (idx - 4);
                    atomicAdd(dst, r);
                }
                if (lane == 0) atomicAdd(&d_c11[id], c11);
            }
        }
    }
    if (COUNT) {
        unsigned long long e_b = 0;
#pragma unroll
        for (int q = 0; q < PX; ++q) e_b += (unsigned long long)nc[q];
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

// Pixels per thread, shared by forward and backward (they must replay the
// same evaluation sequence).  GS_RASTER_PX=2|4|8 overrides for experiments.
static int raster_px() {
    static int v = -1;
    if (v < 0) {
        v = 2;
        const char* e = getenv("GS_RASTER_PX");
        if (e && (atoi(e) == 2 || atoi(e) == 4 || atoi(e) == 8)) v = atoi(e);
    }
    return v;
}

template <int PX>
static void launch_fwd(bool et, bool cnt, unsigned nt, cudaStream_t s, const uint2* ranges, const uint32_t* vals,
                       const float4* xydr, const float4* conic, const float* colors, float3 bg, int W, int H,
                       int tiles_x, float* img, float* T, int* nc, unsigned long long* counts) {
    constexpr int NT = TileGeom<PX>::THREADS;
    if (et) {
        if (cnt) raster_fwd_kernel<PX, true, true><<<nt, NT, 0, s>>>(ranges, vals, xydr, conic, colors, bg, W, H, tiles_x, img, T, nc, counts);
        else raster_fwd_kernel<PX, true, false><<<nt, NT, 0, s>>>(ranges, vals, xydr, conic, colors, bg, W, H, tiles_x, img, T, nc, counts);
    } else {
        if (cnt) raster_fwd_kernel<PX, false, true><<<nt, NT, 0, s>>>(ranges, vals, xydr, conic, colors, bg, W, H, tiles_x, img, T, nc, counts);
        else raster_fwd_kernel<PX, false, false><<<nt, NT, 0, s>>>(ranges, vals, xydr, conic, colors, bg, W, H, tiles_x, img, T, nc, counts);
    }
}

template <int PX>
static void launch_bwd(bool cnt, unsigned nt, cudaStream_t s, const uint2* ranges, const uint32_t* vals,
                       const float4* xydr, const float4* conic, const float* colors, float3 bg, int W, int H,
                       int tiles_x, const float* fT, const int* nc, const float* dimg, float4* d_rgbo,
                       float4* d_geo, float* d_c11, unsigned long long* counts) {
    constexpr int NT = TileGeom<PX>::THREADS;
    if (cnt)
        raster_bwd_kernel<PX, true><<<nt, NT, 0, s>>>(ranges, vals, xydr, conic, colors, bg, W, H, tiles_x, fT, nc, dimg, d_rgbo, d_geo, d_c11, counts);
    else
        raster_bwd_kernel<PX, false><<<nt, NT, 0, s>>>(ranges, vals, xydr, conic, colors, bg, W, H, tiles_x, fT, nc, dimg, d_rgbo, d_geo, d_c11, counts);
}

int launch_raster_fwd(const uint2* ranges, const uint32_t* vals, const float* xydr4, const float* conic4,
                      const float* colors3, float3 bg, int W, int H, bool et, float* img, float* T, int* nc,
                      unsigned long long* counts, cudaStream_t s) {
    const int tiles_x = (W + TILE - 1) / TILE, tiles_y = (H + TILE - 1) / TILE;
    const unsigned nt = (unsigned)(tiles_x * tiles_y);
    const int px = raster_px();
    auto f = px == 2 ? launch_fwd<2> : px == 8 ? launch_fwd<8> : launch_fwd<4>;
    f(et, counts != nullptr, nt, s, ranges, vals, (const float4*)xydr4, (const float4*)conic4, colors3, bg, W, H,
      tiles_x, img, T, nc, counts);
    return check_launch("raster_fwd_kernel");
}

int launch_raster_bwd(const uint2* ranges, const uint32_t* vals, const float* xydr4, const float* conic4,
                      const float* colors3, float3 bg, int W, int H, const float* fT, const int* nc,
                      const float* dimg, float* d_rgbo4, float* d_geo4, float* d_c11, unsigned long long* counts,
                      cudaStream_t s) {
    const int tiles_x = (W + TILE - 1) / TILE, tiles_y = (H + TILE - 1) / TILE;
    const unsigned nt = (unsigned)(tiles_x * tiles_y);
    const int px = raster_px();
    auto f = px == 2 ? launch_bwd<2> : px == 8 ? launch_bwd<8> : launch_bwd<4>;
    f(counts != nullptr, nt, s, ranges, vals, (const float4*)xydr4, (const float4*)conic4, colors3, bg, W, H,
      tiles_x, fT, nc, dimg, (float4*)d_rgbo4, (float4*)d_geo4, d_c11, counts);
    return check_launch("raster_bwd_kernel");
}

}  // namespace gs

using namespace gs;

extern "C" {

int gs_raster_fwd(const uint32_t* ranges2, const uint32_t* sorted_vals, const float* xydr4, const float* conic4,
                  const float* colors3, const float* background3, int32_t width, int32_t height,
                  int early_termination, float* out_image, float* out_final_T, int32_t* out_n_contrib,
                  unsigned long long* counts, gs_stream_t stream) {
    if (width < 1 || height < 1) return set_error("gs_raster_fwd: bad image size %dx%d", width, height);
    const float3 bg = make_float3(background3[0], background3[1], background3[2]);
    return launch_raster_fwd((const uint2*)ranges2, sorted_vals, xydr4, conic4, colors3, bg, width, height,
                             early_termination != 0, out_image, out_final_T, out_n_contrib, counts,
                             (cudaStream_t)stream);
}

int gs_raster_bwd(const uint32_t* ranges2, const uint32_t* sorted_vals, const float* xydr4, const float* conic4,
                  const float* colors3, const float* background3, int32_t width, int32_t height,
                  const float* final_T, const int32_t* n_contrib, const float* d_image, float* d_rgbo4,
                  float* d_geo4, float* d_c11, unsigned long long* counts, gs_stream_t stream) {
    if (width < 1 || height < 1) return set_error("gs_raster_bwd: bad image size %dx%d", width, height);
    const float3 bg = make_float3(background3[0], background3[1], background3[2]);
    return launch_raster_bwd((const uint2*)ranges2, sorted_vals, xydr4, conic4, colors3, bg, width, height, final_T,
                             n_contrib, d_image, d_rgbo4, d_geo4, d_c11, counts, (cudaStream_t)stream);
}

}  // extern "C"
