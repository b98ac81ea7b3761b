// raster.cu -- stage 3 (front-to-back compositing forward) and stage 4
// (back-to-front replay backward).
//
// Layout: one CTA of 128 threads per 16x16 tile.  Warp w owns the 8x8
// quadrant (w&1, w>>1); lane l owns the pixel pair (l&7, l>>3) and
// (l&7, (l>>3)+4) of that quadrant.  The pair shares a column, so every
// per-pixel quantity is one packed f32x2 value and every op one sm_100a
// FFMA2/FMUL2/FADD2 (scalar splat parameters are broadcast for free).
// Bound: FP32 issue (DESIGN.md roofline).
//
// Staging: the tile's sorted splat records are loaded RB = 128 at a time
// into shared memory.  Each staged splat's sigma <= 4.5 ellipse (slightly
// inflated, see stage_batch) is intersected exactly with the four quadrants
// and every warp gets a compacted, order-preserving list of the batch
// entries that can reach it (a third fewer than the ellipse's bounding box
// admits).  A skipped (pixel, splat) pair has sigma > 4.5 with margin, so the
// skip never changes a decision, and forward and backward (same lists) replay
// identical evaluation sequences.
//
// The per-pixel work after the sigma cut is straight-line predicated code on
// the pair (no per-pixel branches); the forward processes two list entries
// per iteration (independent sigma chains) but composites strictly in order.
//
// Retired pixels (forward: out of the image or early-terminated) get
// py = +inf, so sigma is inf/NaN and fails the cut.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "internal.cuh"
#include "segsort.cuh"

namespace gs {

constexpr int NW = 4;    // warps (quadrants, forward)
#ifndef GS_FWD_UNROLL
#define GS_FWD_UNROLL 1  // unrolling of the forward's entry-pair loop (A/B knob)
#endif
constexpr int FWD_UNROLL = GS_FWD_UNROLL;
#ifndef GS_FWD_DONE_EVERY
// Entry pairs between the forward's "whole warp retired" votes (a power of two).  1 = after every
// pair, unconditionally: measured best at config 3 (raster forward 6.57 ms per step; every 2nd /
// 4th / 8th pair 6.67 / 6.70 / 6.72 -- most warps leave their list early, and late exits cost more
// than the votes; the earlier vote guarded by "some pixel passed the sigma cut" 6.78).
#define GS_FWD_DONE_EVERY 1
#endif
constexpr int FWD_DONE_EVERY = GS_FWD_DONE_EVERY;
#ifndef GS_RB
#define GS_RB 128
#endif
constexpr int RB = GS_RB;  // splats per staged batch (A/B knob: 128 or 256)
// compacted-list entry index (the sentinel is RB)
using ListIdx = std::conditional_t<(RB < 255), uint8_t, uint16_t>;

// Warp regions: NWR = 4 -> four 8x8 quadrants (one pixel pair per lane);
// NWR = 2 -> two 8-column x 16-row halves (two pixel pairs per lane).
template <int NWR>
struct BatchT {
    // per staged entry, one 48-byte record (one base address for all of its
    // loads): a = (x, y, hA = A/2, B), b = (hC = C/2, opacity, r, g),
    // c = (blue, splat id bits, -, -); [RB] = sentinel: x = +inf, never visible
    struct Ent {
        float4 a, b, c;
    } e[RB + 1];
    uint32_t mask[NWR][RB / 32];  // region reach bits per group of 32 entries
    __align__(4) ListIdx list[NWR][RB + 2];  // compacted entry indices per region (+ sentinel pad)
    // forward records of this batch (entry indices, one byte each, per region): written over the
    // region's own list -- record j is stored only after the list entries up to j were read (the
    // records are a subsequence of the list, and the sigma votes order a pair's reads before its
    // stores) -- so the batch is 6784 B and 8 CTAs fit a 64 KB carve-out (192 KB of L1)
    __device__ __forceinline__ uint8_t* rbuf(int w) { return reinterpret_cast<uint8_t*>(list[w]); }
    __device__ __forceinline__ const uint8_t* rbuf(int w) const { return reinterpret_cast<const uint8_t*>(list[w]); }
};
using Batch = BatchT<NW>;

__device__ __forceinline__ float pin(float x) {
    asm volatile("" : "+f"(x));
    return x;
}

struct Quad {
    int col, row0;  // this thread's pixel column and first row (second = row0 + 4)
    __device__ __forceinline__ Quad(int tile, int tiles_x) {
        const int tx = tile % tiles_x, ty = tile / tiles_x;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        col = tx * TILE + (warp & 1) * 8 + (lane & 7);
        row0 = ty * TILE + (warp >> 1) * 8 + (lane >> 3);
    }
};

// Stage `count` entries starting at ids[first] and build the warp-region
// lists.  Returns this warp's list length.  Ends with the CTA synchronized.
template <int NWR>
__device__ __forceinline__ int stage_batch(BatchT<NWR>& s, int tile, int tiles_x, const uint32_t* ids,
                                           int first, int count, const float4* __restrict__ xydr,
                                           const float4* __restrict__ conic, const float* __restrict__ colors) {
    constexpr int NTR = 32 * NWR;
    constexpr int NB = NWR == 4 ? 2 : 1;           // row bands of the tile (8 or 16 rows)
    constexpr float RH = NWR == 4 ? 7.f : 15.f;  // band height - 1 (pixel rows)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
#pragma unroll
    for (int u = 0; u < RB / NTR; ++u) {
        const int k = u * NTR + (int)threadIdx.x;
        const bool valid = k < count;
        // per row band: the ellipse's x-interval [x + xl, x + xr] inside the band
        float x = 0.f, xl[NB], xr[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) xl[j] = 1e30f, xr[j] = -1e30f;
        if (valid) {
            const uint32_t id = ids[first + k];
            const float4 g = xydr[id];
            const float4 q = conic[id];
            s.e[k].a = make_float4(g.x, g.y, 0.5f * q.x, q.y);
            s.e[k].b = make_float4(0.5f * q.z, q.w, colors[3 * id], colors[3 * id + 1]);
            s.e[k].c = make_float4(colors[3 * id + 2], __uint_as_float(id), 0.f, 0.f);
            x = g.x;
            // Exact reach of the sigma <= 4.5 ellipse {d : d^T Q d <= 9} of
            // the conic Q = [A B; B C] in each band dy in [lo, hi]: x extends
            // to (-B dy +- sqrt(K A - det dy^2)) / A, concave / convex in dy,
            // so the extremes sit at dy = -+ B sqrt(K / (C det)) clamped to
            // the band.  K = 9 (1 + 0.4%) absorbs the fp32 rounding of both
            // this test and the pixels' sigma, which is bounded by ~8 eps 9
            // / (1 - |rho|) for the conic's correlation rho: entries with
            // 1 - rho^2 < 1e-3 (needle-thin) use the axis-aligned box grown
            // by one pixel instead; the band extents get a 0.01 px + 0.2%
            // pad for their own rounding.  Either way the skip never drops a pair
            // the sigma cut would keep.  The circle radius (the binning
            // bound, sg/binning.py:35-46) caps both.
            const float A = q.x, B = q.y, Cq = q.z;
            const float det = __fmaf_rn(A, Cq, -__fmul_rn(B, B));
            const float r = (float)__float_as_int(g.w) + 1.f;
            const float idq = rcp_approx(det);
            if (det > 1e-3f * A * Cq) {
                constexpr float K = 9.036f;
                const float rx = fminf(r, sqrt_approx(K * Cq * idq));
                const float ry = fminf(r, sqrt_approx(K * A * idq));
                const float iA = rcp_approx(A);
                const float ds = -B * sqrt_approx(K * idq * rcp_approx(Cq));  // dy of the max-x point
                // sqrt(K A - det dy^2) near the band's tangent rows loses up to
                // sqrt(4 eps K A) / A <= 5e-4 rx (as 1/sqrt(A) <= rx/3)
                const float pad = __fmaf_rn(2e-3f, rx, 0.01f);
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                    const float lo = fmaxf((float)(ty * TILE + 8 * j) + 0.5f - g.y, -ry);
                    const float hi = fminf((float)(ty * TILE + 8 * j) + 0.5f + RH - g.y, ry);
                    if (lo <= hi) {
                        const float d1 = fminf(fmaxf(ds, lo), hi), d2 = fminf(fmaxf(-ds, lo), hi);
                        const float s1 = sqrt_approx(fmaxf(__fmaf_rn(-det, d1 * d1, K * A), 0.f));
                        const float s2 = sqrt_approx(fmaxf(__fmaf_rn(-det, d2 * d2, K * A), 0.f));
                        xr[j] = fminf((s1 - B * d1) * iA, rx) + pad;
                        xl[j] = fmaxf((-s2 - B * d2) * iA, -rx) - pad;
                    }
                }
            } else {
                const float rx = fminf(r, __fmaf_rn(3.003f, sqrt_approx(Cq * idq), 1.f));
                const float ry = fminf(r, __fmaf_rn(3.003f, sqrt_approx(A * idq), 1.f));
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                    const float y0 = (float)(ty * TILE + 8 * j) + 0.5f;
                    if (g.y + ry >= y0 && g.y - ry <= y0 + RH) xl[j] = -rx, xr[j] = rx;
                }
            }
        }
#pragma unroll
        for (int w = 0; w < NWR; ++w) {
            const int j = NB == 2 ? (w >> 1) : 0;
            const float x0 = (float)(tx * TILE + (w & 1) * 8) + 0.5f;
            const bool ov = x + xr[j] >= x0 && x + xl[j] <= x0 + 7.f;
            const uint32_t m = __ballot_sync(0xffffffffu, ov);
            if (lane == 0) s.mask[w][u * NWR + warp] = m;
        }
    }
    __syncthreads();
    // each warp compacts its own quadrant list (order preserved)
    int n = 0;
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < RB / 32; ++j) {
        const uint32_t m = s.mask[warp][j];
        if ((m >> lane) & 1u) s.list[warp][n + __popc(m & lt)] = (ListIdx)(32 * j + lane);
        n += __popc(m);
    }
    if (lane == 0) s.list[warp][n] = (ListIdx)RB;  // pad odd lists with the sentinel
    __syncwarp();
    return n;
}

// ============================================================ forward

struct FwdPair {
    f32x2 T, CR, CG, CB, PY;
    int nc0, nc1, stop0, stop1;
    unsigned done;  // bit0 / bit1: pixel retired
};

// One list entry (sigma pair already evaluated) composited into the pair:
// sg/raster_forward.py:136-150, straight-line and predicated.
template <bool ET, bool COUNT>
__device__ __forceinline__ void fwd_commit(FwdPair& p, f32x2 SG, bool vis0, bool vis1, const float4& bq, float blue,
                                           int pos1, unsigned long long& e_a, unsigned long long& e_c) {
    const float INF = __int_as_float(0x7f800000);
    const f32x2 SL = mul2(SG, bc2(NEG_LOG2E));
    const f32x2 E = pk2(ex2_approx(lo2(SL)), ex2_approx(hi2(SL)));
    const f32x2 ARAW = mul2(bc2(bq.y), E);
    const float al0 = fminf(lo2(ARAW), ALPHA_MAX), al1 = fminf(hi2(ARAW), ALPHA_MAX);
    const bool ok0 = vis0 && al0 >= ALPHA_MIN, ok1 = vis1 && al1 >= ALPHA_MIN;
    const f32x2 AL = pk2(al0, al1);
    const f32x2 NTr = mul2(p.T, sub2(bc2(1.f), AL));
    const bool st0 = ET && ok0 && lo2(NTr) < T_MIN, st1 = ET && ok1 && hi2(NTr) < T_MIN;
    const bool cm0 = ok0 && !st0, cm1 = ok1 && !st1;
    const f32x2 Wt = mul2(AL, p.T);
    const f32x2 WC = pk2(cm0 ? lo2(Wt) : 0.f, cm1 ? hi2(Wt) : 0.f);
    p.CR = fma2(WC, bc2(bq.z), p.CR);
    p.CG = fma2(WC, bc2(bq.w), p.CG);
    p.CB = fma2(WC, bc2(blue), p.CB);
    p.T = sel2(cm0, cm1, NTr, p.T);
    p.nc0 = cm0 ? pos1 : p.nc0;
    p.nc1 = cm1 ? pos1 : p.nc1;
    if (ET && (st0 || st1)) {  // stop WITHOUT compositing (:141-144)
        p.PY = pk2(st0 ? INF : lo2(p.PY), st1 ? INF : hi2(p.PY));
        p.done |= (st0 ? 1u : 0u) | (st1 ? 2u : 0u);
        p.stop0 = st0 ? pos1 : p.stop0;
        p.stop1 = st1 ? pos1 : p.stop1;
    }
    if (COUNT) {
        e_a += (unsigned)ok0 + (unsigned)ok1;
        e_c += (unsigned)cm0 + (unsigned)cm1;
    }
}

// Records of (warp, list entry) for the backward: the splat id and its
// 0-based position in the tile list, for every entry whose commit step this
// warp ran (some pixel of the quadrant passed the sigma cut) -- a
// warp-uniform condition the forward already has, so recording costs no
// extra vote.  The backward replays exactly these entries, back to front.
// Per entry one byte goes to the warp's shared buffer; the batch's records
// are written out coalesced when the warp leaves the batch.
// rcur: the warp's shared cursor (32-bit shared address of its next byte in
// rbuf), so a record costs one STS.U8 and one add (every lane stores the
// same byte to the same address: no lane test).
__device__ __forceinline__ void fwd_record(uint32_t& rcur, int k) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(rcur), "r"(k) : "memory");
    ++rcur;
}
template <int NWR>
__device__ __forceinline__ void fwd_record_flush(const BatchT<NWR>& s, int warp, int lane, uint32_t& rcur,
                                                 uint32_t rbase_w, uint2*& rp, int pos0) {
    __syncwarp();
    const int nrec = (int)(rcur - rbase_w);
    for (int j = lane; j < nrec; j += 32) {
        const int k = s.rbuf(warp)[j];
        rp[j] = make_uint2(__float_as_uint(s.e[k].c.y), (uint32_t)(pos0 + k));
    }
    rp += nrec;
    rcur = rbase_w;
}

// sg/raster_forward.py:116-154 _composite_tile for one tile.
// NWR = 4: 128 threads, one pixel pair per lane, two list entries per
// iteration (independent sigma chains); NWR = 2: 64 threads, two pixel pairs
// per lane (8x16 halves), one entry per iteration.
// Shared memory of the forward: the staged batch, or (SORT) its union with
// the per-tile sort that runs first.
template <int NWR, bool SORT>
struct FwdShared {
    BatchT<NWR> b;
};
template <int NWR>
struct FwdShared<NWR, true> {
    union {
        BatchT<NWR> b;
        SegsortShared srt;
    };
};

// Out of line, so the sorts' register allocation stays out of the raster loop's.
static __device__ __noinline__ void fwd_sort_segments(SegsortShared& sh, uint32_t base, uint32_t kr,
                                                      const uint32_t (&cnt)[DREPL],
                                                      const uint32_t* __restrict__ dkeys, uint32_t* vals,
                                                      uint32_t* __restrict__ alt) {
    segsort_tile_segments<DREPL>(sh, base, kr, cnt, dkeys, vals, alt);
}
static __device__ __noinline__ void fwd_sort_tile(SegsortShared& sh, uint2 rg, const uint32_t* __restrict__ dkeys,
                                                  uint32_t* vals, uint32_t* __restrict__ alt) {
    segsort_tile(sh, rg, dkeys, vals, alt);
}

template <int NWR, bool ET, bool COUNT, bool REC>
__device__ __noinline__ void raster_fwd_body(BatchT<NWR>& s, int tile, const uint2 rg,
                                                              const uint32_t* sorted_vals,
                                                              const float4* __restrict__ xydr,
                                                              const float4* __restrict__ conic,
                                                              const float* __restrict__ colors, float3 bg, int W,
                                                              int H, int tiles_x, float* __restrict__ out_img,
                                                              float* __restrict__ out_T, int* __restrict__ out_nc,
                                                              unsigned long long* __restrict__ counts,
                                                              uint2* __restrict__ rec,
                                                              uint32_t* __restrict__ rec_count,
                                                              const uint32_t* __restrict__ tile_order) {
    constexpr int NPR = 4 / NWR;
    static_assert(!REC || NWR == 4, "records are per 8x8 quadrant");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int col = tx * TILE + (warp & 1) * 8 + (lane & 7);
    const int rbase = ty * TILE + (NWR == 4 ? (warp >> 1) * 8 : 0) + (lane >> 3);
    const float INF = __int_as_float(0x7f800000);
    const float px = pin((float)col + 0.5f);
    FwdPair p[NPR];
    bool inb[2 * NPR];
#pragma unroll
    for (int j = 0; j < NPR; ++j) {
        const int r0 = rbase + 8 * j;
        inb[2 * j] = col < W && r0 < H;
        inb[2 * j + 1] = col < W && r0 + 4 < H;
        p[j].T = bc2(1.f);
        p[j].CR = p[j].CG = p[j].CB = bc2(0.f);
        p[j].PY = pk2(inb[2 * j] ? (float)r0 + 0.5f : INF, inb[2 * j + 1] ? (float)r0 + 4.5f : INF);
        p[j].nc0 = p[j].nc1 = 0;
        p[j].stop0 = p[j].stop1 = -1;
        p[j].done = (inb[2 * j] ? 0u : 1u) | (inb[2 * j + 1] ? 0u : 2u);
    }
    auto all_done = [&]() {
        bool d = true;
#pragma unroll
        for (int j = 0; j < NPR; ++j) d = d && p[j].done == 3u;
        return d;
    };
    const int start = (int)rg.x, end = (int)rg.y;
    unsigned long long e_s = 0, e_a = 0, e_c = 0;
    // this warp's record region: 4 * start + warp * len (no atomics)
    uint2* rp = REC ? rec + 4 * (int64_t)start + (int64_t)warp * (end - start) : nullptr;
    const uint32_t rbuf_w = smem_addr(s.rbuf(warp));
    uint32_t rcur = rbuf_w;
    if (threadIdx.x == 0) {  // sentinel entry: dx = -inf -> sigma NaN -> never visible
        s.e[RB].a = make_float4(INF, 0.f, 0.f, 0.f);
        s.e[RB].b = make_float4(0.f, 0.f, 0.f, 0.f);
        s.e[RB].c = make_float4(0.f, 0.f, 0.f, 0.f);
    }

    for (int b0 = start; b0 < end; b0 += RB) {
        if (__syncthreads_count(!all_done()) == 0) break;
        const int n = stage_batch<NWR>(s, tile, tiles_x, sorted_vals, b0, min(RB, end - b0), xydr, conic, colors);
        if (__all_sync(0xffffffffu, all_done())) continue;  // whole warp finished: only help staging
        const int pos_base = b0 - start + 1;
        if constexpr (NPR == 1) {
            using Pair = std::conditional_t<sizeof(ListIdx) == 1, uint16_t, uint32_t>;
            constexpr int IB = 8 * sizeof(ListIdx);
            const Pair* lst2 = reinterpret_cast<const Pair*>(s.list[warp]);
#pragma unroll FWD_UNROLL
            for (int i = 0; i < n; i += 2) {
                const uint32_t kk = lst2[i >> 1];
                const int k0 = kk & ((1u << IB) - 1u), k1 = kk >> IB;  // k1 may be the sentinel
                const float4 a0 = s.e[k0].a, a1 = s.e[k1].a;
                const float hC0 = s.e[k0].b.x, hC1 = s.e[k1].b.x;
                const float dx0 = __fsub_rn(px, a0.x), dx1 = __fsub_rn(px, a1.x);
                const f32x2 SG0 = splat_sigma2(dx0, sigma_base(dx0, a0.z, a0.w), sub2(p[0].PY, bc2(a0.y)), hC0);
                const f32x2 SG1 = splat_sigma2(dx1, sigma_base(dx1, a1.z, a1.w), sub2(p[0].PY, bc2(a1.y)), hC1);
                const bool v00 = lo2(SG0) <= SIGMA_CUT, v01 = hi2(SG0) <= SIGMA_CUT;  // false when retired
                bool v10 = lo2(SG1) <= SIGMA_CUT, v11 = hi2(SG1) <= SIGMA_CUT;
                const uint32_t b0m = __ballot_sync(0xffffffffu, v00 || v01);
                const uint32_t b1m = __ballot_sync(0xffffffffu, v10 || v11);
                if (COUNT) e_s += (unsigned)v00 + (unsigned)v01;
                if (b0m) {
                    fwd_commit<ET, COUNT>(p[0], SG0, v00, v01, s.e[k0].b, s.e[k0].c.x, pos_base + k0, e_a, e_c);
                    if (REC) fwd_record(rcur, k0);
                }
                v10 = v10 && !(p[0].done & 1u);  // retired at k0
                v11 = v11 && !(p[0].done & 2u);
                if (COUNT) e_s += (unsigned)v10 + (unsigned)v11;
                if (b1m) {  // never the sentinel (its sigma is NaN)
                    fwd_commit<ET, COUNT>(p[0], SG1, v10, v11, s.e[k1].b, s.e[k1].c.x, pos_base + k1, e_a, e_c);
                    if (REC) fwd_record(rcur, k1);
                }
                // all pixels retired: leave the batch.  Voted on every FWD_DONE_EVERY-th pair only -- a
                // retired pixel's PY is +inf, so the pairs evaluated before the vote fires commit nothing
                if (ET && (i & (2 * FWD_DONE_EVERY - 2)) == (2 * FWD_DONE_EVERY - 2) &&
                    __all_sync(0xffffffffu, p[0].done == 3u))
                    break;
            }
            if (REC) fwd_record_flush(s, warp, lane, rcur, rbuf_w, rp, pos_base - 1);
        } else {
            const ListIdx* lst = s.list[warp];
#pragma unroll 1
            for (int i = 0; i < n; ++i) {
                const int k = lst[i];
                const float4 a = s.e[k].a;
                const float hC = s.e[k].b.x;
                const float dx = __fsub_rn(px, a.x);
                const f32x2 base = sigma_base(dx, a.z, a.w);
                f32x2 SG[NPR];
                bool v[2 * NPR];
                bool any = false;
#pragma unroll
                for (int j = 0; j < NPR; ++j) {
                    SG[j] = splat_sigma2(dx, base, sub2(p[j].PY, bc2(a.y)), hC);
                    v[2 * j] = lo2(SG[j]) <= SIGMA_CUT;
                    v[2 * j + 1] = hi2(SG[j]) <= SIGMA_CUT;
                    any = any || v[2 * j] || v[2 * j + 1];
                }
                if (COUNT) {
#pragma unroll
                    for (int q = 0; q < 2 * NPR; ++q) e_s += (unsigned)v[q];
                }
                if (!__any_sync(0xffffffffu, any)) continue;
                const float4 bq = s.e[k].b;
                const float blue = s.e[k].c.x;
#pragma unroll
                for (int j = 0; j < NPR; ++j)
                    if (__any_sync(0xffffffffu, v[2 * j] || v[2 * j + 1]))
                        fwd_commit<ET, COUNT>(p[j], SG[j], v[2 * j], v[2 * j + 1], bq, blue, pos_base + k, e_a, e_c);
                if (ET && __all_sync(0xffffffffu, all_done())) break;
            }
        }
    }
    if (REC && lane == 0) {
        rec_count[(size_t)tile * 4 + warp] =
            (uint32_t)(rp - (rec + 4 * (int64_t)rg.x + (int64_t)warp * (rg.y - rg.x)));
    }
#pragma unroll
    for (int j = 0; j < NPR; ++j) {
        float T0, T1, r0, r1, g0, g1, bb0, bb1;
        upk2(p[j].T, T0, T1);
        upk2(p[j].CR, r0, r1);
        upk2(p[j].CG, g0, g1);
        upk2(p[j].CB, bb0, bb1);
        const int row0 = rbase + 8 * j;
        if (inb[2 * j]) {
            const int q = row0 * W + col;
            out_img[3 * q] = __fmaf_rn(bg.x, T0, r0);
            out_img[3 * q + 1] = __fmaf_rn(bg.y, T0, g0);
            out_img[3 * q + 2] = __fmaf_rn(bg.z, T0, bb0);
            out_T[q] = T0;
            out_nc[q] = p[j].nc0;
        }
        if (inb[2 * j + 1]) {
            const int q = (row0 + 4) * W + col;
            out_img[3 * q] = __fmaf_rn(bg.x, T1, r1);
            out_img[3 * q + 1] = __fmaf_rn(bg.y, T1, g1);
            out_img[3 * q + 2] = __fmaf_rn(bg.z, T1, bb1);
            out_T[q] = T1;
            out_nc[q] = p[j].nc1;
        }
    }
    if (COUNT) {
        // E_f: (pixel, entry) pairs the reference visits while not done =
        // entries up to and including the stopping one, else the whole list
        unsigned long long e_f = 0;
#pragma unroll
        for (int j = 0; j < NPR; ++j) {
            if (inb[2 * j]) e_f += (unsigned long long)(p[j].stop0 >= 0 ? p[j].stop0 : end - start);
            if (inb[2 * j + 1]) e_f += (unsigned long long)(p[j].stop1 >= 0 ? p[j].stop1 : end - start);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            e_f += __shfl_xor_sync(0xffffffffu, e_f, o);
            e_s += __shfl_xor_sync(0xffffffffu, e_s, o);
            e_a += __shfl_xor_sync(0xffffffffu, e_a, o);
            e_c += __shfl_xor_sync(0xffffffffu, e_c, o);
        }
        if (lane == 0) {
            atomicAdd(&counts[0], e_f);
            atomicAdd(&counts[1], e_s);
            atomicAdd(&counts[2], e_a);
            atomicAdd(&counts[3], e_c);
        }
    }
}

// SORT (frame path, scatter / direct binning): the CTA first sorts its
// tile's range of sorted_vals in place by (depth, index) (segsort.cuh) --
// the per-tile sort fused into the raster, so a tile's sort overlaps other
// tiles' compositing on the same SM instead of being a latency-bound kernel
// of its own.  Direct binning (direct_counts != nullptr): the tile's list is
// bins[tile * kstride, + count) as the projection left it; the CTA writes
// the tile's range, adds its count to meta[1] (total intersections) and
// raises meta[2] (capacity needed = tiles * DREPL * the longest replica
// segment); a segment over kstride / DREPL leaves the tile
// unrastered (the caller re-runs with a larger capacity).
// meta[3] = kstride tells readers of the bins that they are strided.
template <int NWR, bool ET, bool COUNT, bool REC, int MINB = (NWR == 4 ? 10 : 16), bool SORT = false>
__global__ void __launch_bounds__(32 * NWR, MINB) raster_fwd_kernel(
    const uint2* ranges, const uint32_t* sorted_vals, const float4* __restrict__ xydr,
    const float4* __restrict__ conic, const float* __restrict__ colors, float3 bg, int W, int H, int tiles_x,
    float* __restrict__ out_img, float* __restrict__ out_T, int* __restrict__ out_nc,
    unsigned long long* __restrict__ counts, uint2* __restrict__ rec, uint32_t* __restrict__ rec_count,
    const uint32_t* __restrict__ tile_order, const uint32_t* __restrict__ dkeys, uint32_t* __restrict__ sort_alt,
    const uint32_t* __restrict__ direct_counts, uint32_t kstride, unsigned long long* __restrict__ meta) {
    griddep_wait();
    __shared__ FwdShared<NWR, SORT> sh;
    const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
    uint2 rg;
    if constexpr (SORT) {
      if (direct_counts) {
        // the tile's DREPL replica segments (project.cu MODE 3)
        const uint32_t kr = kstride / DREPL, b = (uint32_t)tile * kstride;
        uint32_t cnt[DREPL], c = 0, mx = 0;
#pragma unroll
        for (int r = 0; r < DREPL; ++r) {
            cnt[r] = direct_counts[(size_t)r * gridDim.x + tile];
            c += cnt[r];
            mx = max(mx, cnt[r]);
        }
        rg = mx <= kr ? make_uint2(b, b + c) : make_uint2(b, b);
        if (threadIdx.x == 0) {
            if (blockIdx.x == 0) meta[3] = kstride;
            const_cast<uint2*>(ranges)[tile] = rg;
            if (c) {
                atomicAdd(&meta[1], (unsigned long long)c);
                atomicMax(&meta[2], (unsigned long long)mx * DREPL * (unsigned long long)(gridDim.x));
            }
        }
        if (mx <= kr) fwd_sort_segments(sh.srt, b, kr, cnt, dkeys, const_cast<uint32_t*>(sorted_vals), sort_alt);
      } else {
        rg = ranges[tile];
        fwd_sort_tile(sh.srt, rg, dkeys, const_cast<uint32_t*>(sorted_vals), sort_alt);
      }
    } else {
        rg = ranges[tile];
    }
    raster_fwd_body<NWR, ET, COUNT, REC>(sh.b, tile, rg, sorted_vals, xydr, conic, colors, bg, W, H, tiles_x,
                                         out_img, out_T, out_nc, counts, rec, rec_count, tile_order);
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

// sigma of one list entry for this lane's pixel pairs (backward replay)
template <int NPR>
struct BwdEvalT {
    float dx;
    f32x2 DY[NPR], SG[NPR];
    bool v[2 * NPR];
    bool any;
    unsigned n_vis;
};
template <int NPR, int NWR>
__device__ __forceinline__ void bwd_eval(const BatchT<NWR>& s, int k, int pos, float px, const f32x2 (&PY)[NPR],
                                         const int (&nc)[2 * NPR], BwdEvalT<NPR>& e) {
    const float4 a = s.e[k].a;
    const float hC = s.e[k].b.x;
    e.dx = __fsub_rn(px, a.x);
    const f32x2 base = sigma_base(e.dx, a.z, a.w);
    e.any = false;
    e.n_vis = 0;
#pragma unroll
    for (int j = 0; j < NPR; ++j) {
        e.DY[j] = sub2(PY[j], bc2(a.y));
        e.SG[j] = splat_sigma2(e.dx, base, e.DY[j], hC);
        e.v[2 * j] = pos < nc[2 * j] && lo2(e.SG[j]) <= SIGMA_CUT;
        e.v[2 * j + 1] = pos < nc[2 * j + 1] && hi2(e.SG[j]) <= SIGMA_CUT;
        e.any = e.any || e.v[2 * j] || e.v[2 * j + 1];
        e.n_vis += (unsigned)e.v[2 * j] + (unsigned)e.v[2 * j + 1];
    }
}

// Replay + gradient of one entry on the lane's pairs (sg/raster_backward.py
// :64-107), then the per-warp accumulation into the splat's gradient rows.
template <int NPR, bool COUNT, int NWR>
__device__ __forceinline__ void bwd_commit(const BatchT<NWR>& s, int k, const BwdEvalT<NPR>& e, int lane, f32x2 (&T)[NPR],
                                           const f32x2 (&G0)[NPR], const f32x2 (&G1)[NPR], const f32x2 (&G2)[NPR],
                                           f32x2 (&S0)[NPR], f32x2 (&S1)[NPR], f32x2 (&S2)[NPR],
                                           float4* __restrict__ d_rgbo, float4* __restrict__ d_geo,
                                           float* __restrict__ d_c11, int gstride, unsigned long long& e_c) {
    const float4 a = s.e[k].a;
    const float4 bq = s.e[k].b;
    const float blue = s.e[k].c.x;
    const float hC = bq.x;
    const float dx = e.dx;
    float acc[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) acc[t] = 0.f;  // dead for NPR == 1 (first pair assigns)
    bool anyc = false;
#pragma unroll
    for (int j = 0; j < NPR; ++j) {
        // replay of the forward decisions on the pair
        const f32x2 SL = mul2(e.SG[j], bc2(NEG_LOG2E));
        const f32x2 E = pk2(ex2_approx(lo2(SL)), ex2_approx(hi2(SL)));
        const f32x2 ARAW = mul2(bc2(bq.y), E);
        const float al0 = fminf(lo2(ARAW), ALPHA_MAX), al1 = fminf(hi2(ARAW), ALPHA_MAX);
        const bool c0 = e.v[2 * j] && al0 >= ALPHA_MIN, c1 = e.v[2 * j + 1] && al1 >= ALPHA_MIN;
        if (COUNT) e_c += (unsigned)c0 + (unsigned)c1;
        if (NPR > 1 && !__any_sync(0xffffffffu, c0 || c1)) continue;
        anyc = anyc || c0 || c1;
        const f32x2 AL = pk2(al0, al1);
        const f32x2 OM = sub2(bc2(1.f), AL);
        const f32x2 INV = pk2(rcp_approx(lo2(OM)), rcp_approx(hi2(OM)));
        const f32x2 TH = mul2(T[j], INV);  // T before this splat (:75)
        const f32x2 Wt = mul2(AL, TH);
        const f32x2 WC = pk2(c0 ? lo2(Wt) : 0.f, c1 ? hi2(Wt) : 0.f);
        const f32x2 CDOT = fma2(bc2(blue), G2[j], fma2(bc2(bq.w), G1[j], mul2(bc2(bq.z), G0[j])));
        const f32x2 SDOT = fma2(S2[j], G2[j], fma2(S1[j], G1[j], mul2(S0[j], G0[j])));
        const f32x2 DA = sub2(mul2(TH, CDOT), mul2(INV, SDOT));
        // live (:91): contributing and not clamped
        const bool l0 = c0 && lo2(ARAW) < ALPHA_MAX, l1 = c1 && hi2(ARAW) < ALPHA_MAX;
        const f32x2 DAL = pk2(l0 ? lo2(DA) : 0.f, l1 ? hi2(DA) : 0.f);
        const f32x2 M = mul2(ARAW, DAL);  // = -d_sigma
        const f32x2 Y0 = fma2(bc2(a.w), e.DY[j], bc2(2.f * a.z * dx));
        const f32x2 Y1 = fma2(bc2(2.f * hC), e.DY[j], bc2(a.w * dx));
        const f32x2 HM = mul2(bc2(0.5f), M);
        const f32x2 HY0 = mul2(HM, Y0), HY1 = mul2(HM, Y1);
        const f32x2 D[9] = {mul2(WC, G0[j]), mul2(WC, G1[j]), mul2(WC, G2[j]), mul2(DAL, E), mul2(M, Y0),
                            mul2(M, Y1),     mul2(HY0, Y0),   mul2(HY0, Y1),   mul2(HY1, Y1)};
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const float v = lo2(D[t]) + hi2(D[t]);
            acc[t] = NPR == 1 ? v : acc[t] + v;
        }
        S0[j] = fma2(WC, bc2(bq.z), S0[j]);
        S1[j] = fma2(WC, bc2(bq.w), S1[j]);
        S2[j] = fma2(WC, bc2(blue), S2[j]);
        T[j] = sel2(c0, c1, TH, T[j]);
    }
    const uint32_t cmask = __ballot_sync(0xffffffffu, anyc);
    if (!cmask) return;
    const uint32_t id = __float_as_uint(s.e[k].c.y);
    if (__popc(cmask) <= 3) {
        // few contributing lanes: their own vector reductions are cheaper
        // than a 9-value warp reduction
        if (anyc) {
            red_add_v4(&d_rgbo[(size_t)id * gstride], acc[0], acc[1], acc[2], acc[3]);
            red_add_v4(&d_geo[(size_t)id * gstride], acc[4], acc[5], acc[6], acc[7]);
            atomicAdd(&d_c11[id], acc[8]);
        }
        return;
    }
    const float r = warp_reduce8(acc, lane);
    float c11 = acc[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c11 += __shfl_xor_sync(0xffffffffu, c11, o);
    if ((lane & 3) == 0) {
        const int idx = lane >> 2;
        float* dst = idx < 4 ? reinterpret_cast<float*>(&d_rgbo[(size_t)id * gstride]) + idx
                             : reinterpret_cast<float*>(&d_geo[(size_t)id * gstride]) + (idx - 4);
        atomicAdd(dst, r);
    }
    if (lane == 0) atomicAdd(&d_c11[id], c11);
}

// sg/raster_backward.py:47-108 _backward_tile for one tile: seed T = final_T,
// S = bg * final_T; walk pos = max(n_contrib)-1 .. 0 replaying the forward's
// decisions (same sigma/exp code, same quadrant lists); contrib ->
// T_here = T/(1-alpha), w = alpha T_here, dc += w g,
// d_alpha = T_here c.g - S.g/(1-alpha); live (alpha_raw < 0.999) ->
// d_opacity += d_alpha e^-sigma, d_sigma = -alpha_raw d_alpha,
// d_mean2d += -d_sigma y, d_cov2d += -d_sigma/2 y y^T with y = conic * delta
// (full-matrix convention, :99-105); S += w c; T = T_here.  Per splat the
// warp's 9 sums are transposed-reduced and 8 (+1) lanes issue one global
// reduction each (one atomic per warp per Gaussian value); when at most 3
// lanes contribute they add their own sums directly instead.
template <int NWR, bool COUNT>
__global__ void __launch_bounds__(32 * NWR, NWR == 4 ? 8 : 4) raster_bwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ sorted_vals, const float4* __restrict__ xydr,
    const float4* __restrict__ conic, const float* __restrict__ colors, float3 bg, int W, int H, int tiles_x,
    const float* __restrict__ final_T, const int* __restrict__ n_contrib, const float* __restrict__ d_img,
    float4* __restrict__ d_rgbo, float4* __restrict__ d_geo, float* __restrict__ d_c11, int gstride,
    unsigned long long* __restrict__ counts) {
    constexpr int NPR = 4 / NWR;  // pixel pairs per lane
    __shared__ BatchT<NWR> s;
    __shared__ int s_max[NWR];
    const int tile = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int col = tx * TILE + (warp & 1) * 8 + (lane & 7);
    const int rbase = ty * TILE + (NWR == 4 ? (warp >> 1) * 8 : 0) + (lane >> 3);
    const float px = pin((float)col + 0.5f);
    f32x2 T[NPR], G0[NPR], G1[NPR], G2[NPR], S0[NPR], S1[NPR], S2[NPR], PY[NPR];
    int nc[2 * NPR];
    int my_max = 0;
#pragma unroll
    for (int j = 0; j < NPR; ++j) {
        float t[2] = {1.f, 1.f}, ga[2] = {0.f, 0.f}, gb[2] = {0.f, 0.f}, gc[2] = {0.f, 0.f};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int row = rbase + 8 * j + 4 * h;
            nc[2 * j + h] = 0;
            if (col < W && row < H) {
                const int q = row * W + col;
                t[h] = final_T[q];
                nc[2 * j + h] = n_contrib[q];
                ga[h] = d_img[3 * q]; gb[h] = d_img[3 * q + 1]; gc[h] = d_img[3 * q + 2];
            }
            my_max = max(my_max, nc[2 * j + h]);
        }
        T[j] = pk2(t[0], t[1]);
        G0[j] = pk2(ga[0], ga[1]); G1[j] = pk2(gb[0], gb[1]); G2[j] = pk2(gc[0], gc[1]);
        S0[j] = mul2(bc2(bg.x), T[j]); S1[j] = mul2(bc2(bg.y), T[j]); S2[j] = mul2(bc2(bg.z), T[j]);
        PY[j] = pin2(pk2((float)(rbase + 8 * j) + 0.5f, (float)(rbase + 8 * j) + 4.5f));
    }
    const int warp_max = __reduce_max_sync(0xffffffffu, my_max);
    if (lane == 0) s_max[warp] = warp_max;
    const uint2 rg = ranges[tile];
    const int start = (int)rg.x;
    __syncthreads();
    int max_nc = 0;
#pragma unroll
    for (int w = 0; w < NWR; ++w) max_nc = max(max_nc, s_max[w]);
    unsigned long long e_s = 0, e_c = 0;
    if (threadIdx.x == 0) {  // sentinel entry: dx = -inf -> sigma NaN -> never visible
        s.e[RB].a = make_float4(__int_as_float(0x7f800000), 0.f, 0.f, 0.f);
        s.e[RB].b = make_float4(0.f, 0.f, 0.f, 0.f);
        s.e[RB].c = make_float4(0.f, 0.f, 0.f, 0.f);
    }

    for (int bend = max_nc; bend > 0; bend -= RB) {
        const int bstart = max(0, bend - RB);
        __syncthreads();
        int n = stage_batch<NWR>(s, tile, tiles_x, sorted_vals, start + bstart, bend - bstart, xydr, conic, colors);
        const ListIdx* lst = s.list[warp];
        const int kmax = min(bend, warp_max) - bstart;  // positions >= warp_max are inactive for this warp
        while (n > 0 && (int)lst[n - 1] >= kmax) --n;
        // two entries per iteration (independent sigma chains), committed
        // strictly back to front; an odd list's last pair uses the sentinel
#pragma unroll 1
        for (int i = n - 1; i >= 0; i -= 2) {
            const int k0 = lst[i];
            const int k1 = i > 0 ? (int)lst[i - 1] : RB;
            BwdEvalT<NPR> e0, e1;
            bwd_eval<NPR>(s, k0, bstart + k0, px, PY, nc, e0);
            bwd_eval<NPR>(s, k1, bstart + k1, px, PY, nc, e1);
            const bool a0 = __any_sync(0xffffffffu, e0.any), a1 = __any_sync(0xffffffffu, e1.any);
            if (COUNT) e_s += e0.n_vis + e1.n_vis;
            if (a0)
                bwd_commit<NPR, COUNT>(s, k0, e0, lane, T, G0, G1, G2, S0, S1, S2, d_rgbo, d_geo, d_c11, gstride,
                                       e_c);
            if (a1)
                bwd_commit<NPR, COUNT>(s, k1, e1, lane, T, G0, G1, G2, S0, S1, S2, d_rgbo, d_geo, d_c11, gstride,
                                       e_c);
        }
    }
    if (COUNT) {
        unsigned long long e_b = 0;
#pragma unroll
        for (int q = 0; q < 2 * NPR; ++q) e_b += (unsigned long long)nc[q];
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

// Record-driven backward (frame path): each warp replays, back to front,
// only the list entries its forward ran the commit step for (records of
// (splat id, list position)) -- no list staging, no sigma vote over entries
// the warp never composited, no CTA barriers.  Decisions are replayed with
// the forward's arithmetic (sigma cut, alpha >= 1/255, position < n_contrib).
//
// Accumulation: instead of a shuffle reduction per contributing record,
// each lane parks its 9 per-record partial sums (already summed over its
// pixel pair) in a per-warp shared-memory batch laid out [slot][value][lane]
// (rows of 32 lanes, stride 36 words so row reads are conflict-free 128-bit
// loads); every RBS records the warp sums the 9 * RBS rows -- one row per
// lane, 8 LDS.128 + adds -- and issues one atomic per row.  About half the
// instructions of a 9-value shuffle reduction per record.  A slot's splat
// id rides in the padding word of its first row, so a batch may span
// staging chunks.
constexpr int RBS = 3;        // records per reduction batch (9 * RBS <= 32 rows: one row per lane)
constexpr int RROW = 36;      // row stride (words): 32 lanes + pad

// A staged record: the splat's (x, y, A/2, B), (C/2, opacity, r, g),
// (b, list position, splat id, -) -- one base address, three LDS.128.
struct __align__(16) RecStage {
    float4 a, b, c;
};
constexpr uint32_t REC_BYTES = sizeof(RecStage);

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}

// Sum the batch's 9 * nslot rows (one per lane) and add each to its
// splat's gradient slot.  red: this warp's batch (32-bit shared address);
// each slot's splat id sits in the padding word (lane 32) of its first row.
// The conic rows (6..8) were accumulated without their factor 1/2, applied
// here (exact).
// GS_BWD_V4=1: two red.global.add.v4.f32 + one scalar red per (warp, record)
// instead of 9 scalar reds (3 L2 requests instead of 9).  Measured at config 3:
// raster backward 9.03 -> 9.54 ms per 32 views (the 3 shuffles + the extra
// predicated branch cost more issue slots than the L2 requests saved; the
// kernel is issue-bound, not L2-atomic-bound: 19 G reds/s), so it is off.
#ifndef GS_BWD_V4
#define GS_BWD_V4 0
#endif
// ids: 0 = each slot's splat id rides in the padding word of its first row; otherwise the shared
// address of slot 0's staged record id, slot k's one record (REC_BYTES) below it (GS_BWD_IDS).
__device__ __forceinline__ void bwd_flush(uint32_t red, int nslot, int lane, float* __restrict__ g8,
                                          float* __restrict__ d_c11, uint32_t ids = 0u) {
    const int k = lane / 9, t = lane - 9 * k;
    float sum = 0.f;
    if (lane < 9 * nslot) {
        const uint32_t row = red + (uint32_t)lane * (RROW * 4);
        const float4 a = lds_f4(row);
        f32x2 s01 = pk2(a.x, a.y), s23 = pk2(a.z, a.w);
#pragma unroll
        for (int j = 1; j < 8; ++j) {
            const float4 b = lds_f4(row + 16 * j);
            s01 = add2(s01, pk2(b.x, b.y));
            s23 = add2(s23, pk2(b.z, b.w));
        }
        const f32x2 s2 = add2(s01, s23);
        sum = lo2(s2) + hi2(s2);
        if (t >= 6) sum *= 0.5f;
    }
#if GS_BWD_V4
    // rows 0-3 (d_rgbo) and 4-7 (d_geo) of a slot are one 16-byte gradient
    // row each: lanes 9k and 9k+4 gather their 3 neighbours' sums and issue
    // one red.global.add.v4.f32 each, lane 9k+8 adds d_c11 (3 L2 requests
    // per (warp, record) instead of 9)
    const float s1 = __shfl_down_sync(0xffffffffu, sum, 1);
    const float s2v = __shfl_down_sync(0xffffffffu, sum, 2);
    const float s3 = __shfl_down_sync(0xffffffffu, sum, 3);
    if (lane < 9 * nslot && (t == 0 || t == 4 || t == 8)) {
        const uint32_t id = lds_u32(ids ? ids - (uint32_t)k * REC_BYTES : red + (uint32_t)k * (9 * RROW * 4) + 32 * 4);
        if (t == 8)
            atomicAdd(d_c11 + id, sum);
        else
            red_add_v4(reinterpret_cast<float4*>(g8 + 8 * (size_t)id + t), sum, s1, s2v, s3);
    }
#else
    if (lane < 9 * nslot) {
        const uint32_t id = lds_u32(ids ? ids - (uint32_t)k * REC_BYTES : red + (uint32_t)k * (9 * RROW * 4) + 32 * 4);
        atomicAdd(t < 8 ? g8 + 8 * (size_t)id + t : d_c11 + id, sum);
    }
#endif
}

#ifndef GS_BWD_WPC
#define GS_BWD_WPC 4
#endif
constexpr int BWD_WPC = GS_BWD_WPC;  // warps per CTA of the record backward (4 or 1)
// resident record-backward CTAs per SM the registers are budgeted for: 7 (68 registers, nothing
// spilled or rematerialised) measured a little faster than 8 (64) -- config 3 raster backward
// 8.69 -> 8.63 ms per step and 1453 -> 1457 frames/s, config 1 +0.6 %, configs 2 / 4 +-0.2 %
#ifndef GS_BWD_MINB
#define GS_BWD_MINB (GS_BWD_WPC == 4 ? 7 : 32)
#endif
#ifndef GS_BWD_UNROLL
#define GS_BWD_UNROLL 1
#endif
[[maybe_unused]] constexpr int BWD_UNROLL = GS_BWD_UNROLL;
// Record loop in groups of RBS records with compile-time batch slots and an unconditional flush
// per group (staging chunks of 30 records, a whole number of groups) instead of a running slot
// counter tested after every record: config 3 raster backward 9.11 -> 8.73 ms per step
// (0 restores the counted loop, whose 2x / 4x unrolling gave 9.00).
#ifndef GS_BWD_G3
#define GS_BWD_G3 1
#endif
// Grouped loop: the flush takes each slot's splat id from the staged record (a group never leaves its
// chunk) instead of a copy lane 0 parks in the row padding per record: config 3 raster backward
// 8.63 -> 8.42 ms per step, 1457 -> 1472 frames/s (0: the parked copy, which the counted loop needs).
#ifndef GS_BWD_IDS
#define GS_BWD_IDS 1
#endif
// Alpha zeroed for the pixels a record does not contribute to, instead of selects on the weight and on
// T (rcp.approx.ftz(1.0) is exactly 1.0 -- checked on the device, tools/ab_r2g.sh -- so T * 1 keeps T
// bit for bit): config 3 raster backward 8.42 -> 8.17 ms per step, 1472 -> 1488 frames/s.
#ifndef GS_BWD_AZ
#define GS_BWD_AZ 1
#endif
#ifndef GS_BWD_CH
#define GS_BWD_CH (GS_BWD_G3 ? 30 : 32)
#endif
constexpr int BWD_CH = GS_BWD_CH;  // records staged per chunk (<= 32; 16: 18.7 KB of shared memory per CTA)
__global__ void __launch_bounds__(32 * BWD_WPC, GS_BWD_MINB) raster_bwd_rec_kernel(
    const uint2* __restrict__ ranges, const uint2* __restrict__ rec, const uint32_t* __restrict__ rec_count,
    const float4* __restrict__ xydr, const float4* __restrict__ conic, const float* __restrict__ colors, float3 bg,
    int W, int H, int tiles_x, const float* __restrict__ final_T, const int* __restrict__ n_contrib,
    const float* __restrict__ d_img, float* __restrict__ g8, float* __restrict__ d_c11,
    const uint32_t* __restrict__ tile_order, const unsigned long long* __restrict__ meta,
    uint32_t* __restrict__ touched) {
    griddep_wait();
    // BWD_WPC warps per CTA: 4 (one CTA per tile) or 1 (one CTA per 8x8
    // quadrant: a warp that finishes frees its slot without waiting for
    // its tile's slowest quadrant; the warps never synchronise anyway).
    // Measured: 1 is 3 % slower at config 1 and 5 % at config 2 -- a tile's
    // four warps gather the same splats, so they share L1 lines.
    __shared__ RecStage s_rec[BWD_WPC][BWD_CH];
    __shared__ __align__(16) float s_red[BWD_WPC][RBS][9][RROW];
    const int job = (int)blockIdx.x / (4 / BWD_WPC);
    // the forward's raster order exists unless it binned directly (meta[3] = bin stride)
    const int tile = tile_order && meta[3] == 0 ? (int)tile_order[job] : job;
    const int lane = threadIdx.x & 31, wslot = threadIdx.x >> 5;
    const int warp = BWD_WPC == 4 ? wslot : (int)blockIdx.x % 4;  // quadrant
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int col = tx * TILE + (warp & 1) * 8 + (lane & 7);
    const int rbase = ty * TILE + (warp >> 1) * 8 + (lane >> 3);
    const float px = pin((float)col + 0.5f);
    float t[2] = {1.f, 1.f}, ga[2] = {0.f, 0.f}, gb[2] = {0.f, 0.f}, gc[2] = {0.f, 0.f};
    int nc[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int row = rbase + 4 * h;
        if (col < W && row < H) {
            const int q = row * W + col;
            t[h] = final_T[q];
            nc[h] = n_contrib[q];
            ga[h] = d_img[3 * q]; gb[h] = d_img[3 * q + 1]; gc[h] = d_img[3 * q + 2];
        }
    }
    f32x2 T = pk2(t[0], t[1]);
    const f32x2 G0 = pk2(ga[0], ga[1]), G1 = pk2(gb[0], gb[1]), G2 = pk2(gc[0], gc[1]);
    // the backward's running sum S (sg/raster_backward.py:58,107: S = bg T_final + sum w c over the
    // entries behind) enters the gradient only through S . g, so the pixel keeps SDOT = S . g:
    // seeded (bg . g) T_final, advanced by w (c . g) = w CDOT per contributing entry (1 FFMA2
    // instead of 3 S updates + a 3-term dot per record)
    f32x2 SDOT = mul2(fma2(bc2(bg.z), G2, fma2(bc2(bg.y), G1, mul2(bc2(bg.x), G0))), T);
    const f32x2 PY = pin2(pk2((float)rbase + 0.5f, (float)rbase + 4.5f));
    const uint2 rg = ranges[tile];
    const int64_t rb = 4 * (int64_t)rg.x + (int64_t)warp * (rg.y - rg.x);
    const int count = (int)rec_count[(size_t)tile * 4 + warp];
    const uint32_t red_w = smem_addr(&s_red[wslot][0][0][0]);
    const uint32_t stage_w = smem_addr(&s_rec[wslot][0]);
    int nslot = 0;
    [[maybe_unused]] uint32_t tail_ids = 0u;
    for (int hi = count; hi > 0; hi -= BWD_CH) {
        const int lo = hi > BWD_CH ? hi - BWD_CH : 0;
        const int nb = hi - lo;
        if (lane < nb) {  // stage up to BWD_CH records and their splats (independent gathers)
            const uint2 r = rec[rb + lo + lane];
            // the splat's screen-space rows get added to: mark it for the projection backward
            if (touched) atomicOr(touched + (r.x >> 5), 1u << (r.x & 31u));
            const float4 g = xydr[r.x];
            const float4 q = conic[r.x];
            RecStage& st = s_rec[wslot][lane];
            st.a = make_float4(g.x, g.y, 0.5f * q.x, q.y);
            st.b = make_float4(0.5f * q.z, q.w, colors[3 * r.x], colors[3 * r.x + 1]);
            st.c = make_float4(colors[3 * r.x + 2], __int_as_float((int)r.y), __int_as_float((int)r.x), 0.f);
        }
        __syncwarp();
        // one record: its 9 partial sums parked in the batch slot at `slot` (this lane's word of
        // the slot's first row)
        auto record = [&](int k, uint32_t slot) {
            const uint32_t sk = stage_w + (uint32_t)k * REC_BYTES;
            const float4 cq = lds_f4(sk + 32);
            const int pos = __float_as_int(cq.y);
            const float4 a = lds_f4(sk);
            const float4 bq = lds_f4(sk + 16);
            const float blue = cq.x;
            const float hC = bq.x;
            const float dx = __fsub_rn(px, a.x);
            const f32x2 base = sigma_base(dx, a.z, a.w);  // (A/2 dx, B dx)
            const f32x2 DY = sub2(PY, bc2(a.y));
            f32x2 T1;  // C/2 dy + B dx
            const f32x2 SG = splat_sigma2(dx, base, DY, hC, &T1);
            const f32x2 SL = mul2(SG, bc2(NEG_LOG2E));
            const f32x2 E = pk2(ex2_approx(lo2(SL)), ex2_approx(hi2(SL)));
            const f32x2 ARAW = mul2(bc2(bq.y), E);
            const float al0 = fminf(lo2(ARAW), ALPHA_MAX), al1 = fminf(hi2(ARAW), ALPHA_MAX);
            const bool c0 = pos < nc[0] && lo2(SG) <= SIGMA_CUT && al0 >= ALPHA_MIN;
            const bool c1 = pos < nc[1] && hi2(SG) <= SIGMA_CUT && al1 >= ALPHA_MIN;
            // no vote: ~98 % of records contribute to some pixel of the warp;
            // a record that does not adds zero rows (WC = DAL = 0, T kept)
#if GS_BWD_AZ
            // a pixel the record does not contribute to gets alpha 0: 1 - alpha = 1, its reciprocal
            // (rcp.approx of 1.0) is exactly 1, so TH = T, the weight is 0 and neither needs a select
            const f32x2 AL = pk2(c0 ? al0 : 0.f, c1 ? al1 : 0.f);
            const f32x2 OM = sub2(bc2(1.f), AL);
            const f32x2 INV = pk2(rcp_approx(lo2(OM)), rcp_approx(hi2(OM)));
            const f32x2 TH = mul2(T, INV);
            const f32x2 WC = mul2(AL, TH);
#else
            const f32x2 AL = pk2(al0, al1);
            const f32x2 OM = sub2(bc2(1.f), AL);
            const f32x2 INV = pk2(rcp_approx(lo2(OM)), rcp_approx(hi2(OM)));
            const f32x2 TH = mul2(T, INV);
            const f32x2 Wt = mul2(AL, TH);
            const f32x2 WC = pk2(c0 ? lo2(Wt) : 0.f, c1 ? hi2(Wt) : 0.f);
#endif
            const f32x2 CDOT = fma2(bc2(blue), G2, fma2(bc2(bq.w), G1, mul2(bc2(bq.z), G0)));
            const f32x2 DA = sub2(mul2(TH, CDOT), mul2(INV, SDOT));
            const bool l0 = c0 && lo2(ARAW) < ALPHA_MAX, l1 = c1 && hi2(ARAW) < ALPHA_MAX;
            const f32x2 DAL = pk2(l0 ? lo2(DA) : 0.f, l1 ? hi2(DA) : 0.f);
            const f32x2 M = mul2(ARAW, DAL);
            const f32x2 Y0 = fma2(bc2(a.w), DY, bc2(lo2(base) + lo2(base)));  // A dx + B dy
            const f32x2 Y1 = fma2(bc2(hC), DY, T1);                           // B dx + C dy
            const f32x2 MY0 = mul2(M, Y0), MY1 = mul2(M, Y1);
            // rows 6..8 are M Y Y without the 1/2 of d sigma / d conic (bwd_flush applies it)
            const f32x2 D[9] = {mul2(WC, G0), mul2(WC, G1), mul2(WC, G2), mul2(DAL, E), MY0,
                                MY1,          mul2(MY0, Y0), mul2(MY0, Y1), mul2(MY1, Y1)};
#pragma unroll
            for (int u = 0; u < 9; ++u) sts_f32(slot + u * (RROW * 4), lo2(D[u]) + hi2(D[u]));
#if !(GS_BWD_G3 && GS_BWD_IDS)
            if (lane == 0) sts_u32(slot + 32 * 4, __float_as_uint(cq.z));  // splat id -> row padding
#endif
            SDOT = fma2(WC, CDOT, SDOT);
#if GS_BWD_AZ
            T = TH;
#else
            T = sel2(c0, c1, TH, T);
#endif
        };
#if GS_BWD_G3
        // groups of RBS records with compile-time slots and an unconditional flush (a chunk
        // holds a whole number of groups, so only the last chunk -- lo == 0 -- has a remainder)
        int k = nb - 1;
        for (; k >= RBS - 1; k -= RBS) {
#pragma unroll
            for (int j = 0; j < RBS; ++j) record(k - j, red_w + (uint32_t)j * (9 * RROW * 4) + 4 * lane);
            __syncwarp();
            // (a group never leaves its chunk: the flush reads the ids from the staged records)
            bwd_flush(red_w, RBS, lane, g8, d_c11, GS_BWD_IDS ? stage_w + (uint32_t)k * REC_BYTES + 40u : 0u);
            __syncwarp();
        }
        if (k >= 0) tail_ids = stage_w + (uint32_t)k * REC_BYTES + 40u;  // (last chunk: stays staged)
        for (; k >= 0; --k) {
            record(k, red_w + (uint32_t)nslot * (9 * RROW * 4) + 4 * lane);
            ++nslot;
        }
#else
#pragma unroll BWD_UNROLL
        for (int k = nb - 1; k >= 0; --k) {
            record(k, red_w + (uint32_t)nslot * (9 * RROW * 4) + 4 * lane);
            if (++nslot == RBS) {
                __syncwarp();
                bwd_flush(red_w, RBS, lane, g8, d_c11);
                __syncwarp();
                nslot = 0;
            }
        }
#endif
        __syncwarp();  // the next chunk restages s_rec (the batch keeps its own ids)
    }
    if (nslot) {
        __syncwarp();
        bwd_flush(red_w, nslot, lane, g8, d_c11, (GS_BWD_G3 && GS_BWD_IDS) ? tail_ids : 0u);
    }
}

// Warp regions of the backward: 2 (8x16 halves) or 4 (8x8 quadrants).  The
// region geometry never changes a decision (skipped pairs are far outside
// the 3-sigma square), so it is free to differ from the forward's.
static int bwd_regions() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GS_BWD_REGIONS");
        v = (e && atoi(e) == 2) ? 2 : 4;
    }
    return v;
}

static int fwd_regions() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GS_FWD_REGIONS");
        v = (e && atoi(e) == 2) ? 2 : 4;
    }
    return v;
}

#ifndef GS_FWD_FRAME_MINB
#define GS_FWD_FRAME_MINB 9  // resident forward CTAs per SM the frame path's registers are budgeted for
#endif

// A/B knobs: GS_FWD_PAD / GS_BWD_PAD = bytes of (unused) dynamic shared memory added to the frame
// path's raster launches (caps their resident CTAs per SM below the register limit);
// GS_FWD_CARVE / GS_BWD_CARVE = preferred shared-memory carve-out in percent of the maximum
// (cudaFuncAttributePreferredSharedMemoryCarveout; the rest of the 256 KB is L1).
static size_t pad_env(const char* name) {
    const char* e = getenv(name);
    const long v = e ? atol(e) : 0;
    return v > 0 && v <= 200 * 1024 ? (size_t)v : 0;
}
template <typename F>
static void carve_env(const char* name, F* kernel, int dflt = -1) {
    const char* e = getenv(name);
    const int v = e ? atoi(e) : dflt;
    if (v >= 0 && v <= 100) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, v);
}
// The frame path's forward asks for the 64 KB carve-out (25 % of 228 KB; a hint the driver may
// ignore) and pads its 6.8 KB batch to > 7 KB per CTA, so 7 CTAs sit in it (instead of 9 in
// 100 KB): alone it runs as fast (192 KB of L1 for the gathers make up for the occupancy), and in
// a multi-view step the registers it leaves free let other views' latency-bound binning kernels
// sit beside it (config 3: 1405 -> 1420 frames/s; 8 CTAs 1409, 6 CTAs 1363).
constexpr int FWD_FRAME_CARVE = 25;
constexpr size_t FWD_FRAME_PAD = 512;

int launch_raster_fwd(const uint2* ranges, const uint32_t* vals, const float* xydr4, const float* conic4,
                      const float* colors3, float3 bg, int W, int H, bool et, float* img, float* T, int* nc,
                      unsigned long long* counts, cudaStream_t s, uint2* rec, uint32_t* rec_count,
                      const uint32_t* tile_order, const uint32_t* dkeys, uint32_t* sort_alt,
                      const uint32_t* direct_counts, uint32_t kstride, unsigned long long* meta) {
    const int tiles_x = (W + TILE - 1) / TILE, tiles_y = (H + TILE - 1) / TILE;
    const unsigned nt = (unsigned)(tiles_x * tiles_y);
    const float4* g = (const float4*)xydr4;
    const float4* q = (const float4*)conic4;
    uint32_t* dk = nullptr;
#define GS_FWD_R(NWR, ET, CNT, REC)                                                                          \
    raster_fwd_kernel<NWR, ET, CNT, REC><<<nt, 32 * NWR, 0, s>>>(ranges, vals, g, q, colors3, bg, W, H, tiles_x, \
                                                                 img, T, nc, counts, rec, rec_count, tile_order, \
                                                                 dk, dk, dk, 0u, nullptr)
#define GS_FWD(NWR, ET, CNT) GS_FWD_R(NWR, ET, CNT, false)
    const bool cnt = counts != nullptr;
    // frame path: 8x8 quadrants with commit records, 9 CTAs/SM (measured best
    // against 8 and 10), optionally with the per-tile sort fused in front
    static const size_t fwd_pad = getenv("GS_FWD_PAD") ? pad_env("GS_FWD_PAD") : FWD_FRAME_PAD;
#define GS_FWD_M(ET, SORT)                                                                                     \
    {                                                                                                          \
        static bool once = false;                                                                              \
        if (!once) {                                                                                           \
            once = true;                                                                                       \
            carve_env("GS_FWD_CARVE", raster_fwd_kernel<4, ET, false, true, GS_FWD_FRAME_MINB, SORT>,         \
                      SORT ? -1 : FWD_FRAME_CARVE); /* (the fused sort's 16 KB want the default) */           \
            if (fwd_pad > 40 * 1024)                                                                           \
                cudaFuncSetAttribute(raster_fwd_kernel<4, ET, false, true, GS_FWD_FRAME_MINB, SORT>,           \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_pad);               \
        }                                                                                                      \
    }                                                                                                          \
    launch_k(raster_fwd_kernel<4, ET, false, true, GS_FWD_FRAME_MINB, SORT>, dim3(nt), dim3(128),              \
             (SORT && !getenv("GS_FWD_PAD")) ? 0 : fwd_pad, s, ranges, vals, g, q,                             \
             colors3, bg, W, H, tiles_x, img, T, nc, counts, rec, rec_count, tile_order, dkeys, sort_alt,        \
             direct_counts, kstride, meta)
    if (dkeys && !(rec && !cnt)) return set_error("raster_fwd: the fused tile sort needs the frame path");
    if (direct_counts && (!dkeys || !meta)) return set_error("raster_fwd: direct binning needs the fused sort");
    if (rec && !cnt) {
        if (dkeys) { if (et) { GS_FWD_M(true, true); } else { GS_FWD_M(false, true); } }
        else { if (et) { GS_FWD_M(true, false); } else { GS_FWD_M(false, false); } }
    } else if (rec) {
        if (et) GS_FWD_R(4, true, true, true); else GS_FWD_R(4, false, true, true);
    } else if (fwd_regions() == 2) {
        if (et) { if (cnt) GS_FWD(2, true, true); else GS_FWD(2, true, false); }
        else { if (cnt) GS_FWD(2, false, true); else GS_FWD(2, false, false); }
    } else {
        if (et) { if (cnt) GS_FWD(4, true, true); else GS_FWD(4, true, false); }
        else { if (cnt) GS_FWD(4, false, true); else GS_FWD(4, false, false); }
    }
#undef GS_FWD
#undef GS_FWD_R
#undef GS_FWD_M
    return check_launch("raster_fwd_kernel");
}

int launch_raster_bwd(const uint2* ranges, const uint32_t* vals, const float* xydr4, const float* conic4,
                      const float* colors3, float3 bg, int W, int H, const float* fT, const int* nc,
                      const float* dimg, float* d_rgbo4, float* d_geo4, float* d_c11, unsigned long long* counts,
                      cudaStream_t s, int gstride) {
    const int tiles_x = (W + TILE - 1) / TILE, tiles_y = (H + TILE - 1) / TILE;
    const unsigned nt = (unsigned)(tiles_x * tiles_y);
    const float4* g = (const float4*)xydr4;
    const float4* q = (const float4*)conic4;
#define GS_BWD(NWR, CNT)                                                                                 \
    raster_bwd_kernel<NWR, CNT><<<nt, 32 * NWR, 0, s>>>(ranges, vals, g, q, colors3, bg, W, H, tiles_x, fT, nc, \
                                                        dimg, (float4*)d_rgbo4, (float4*)d_geo4, d_c11, gstride, \
                                                        counts)
    if (bwd_regions() == 4) {
        if (counts) GS_BWD(4, true); else GS_BWD(4, false);
    } else {
        if (counts) GS_BWD(2, true); else GS_BWD(2, false);
    }
#undef GS_BWD
    return check_launch("raster_bwd_kernel");
}

int launch_raster_bwd_rec(const uint2* ranges, const uint2* rec, const uint32_t* rec_count, const float* xydr4,
                          const float* conic4, const float* colors3, float3 bg, int W, int H, const float* fT,
                          const int* nc, const float* dimg, float* g8, float* d_c11, cudaStream_t s,
                          const uint32_t* tile_order, const unsigned long long* meta, uint32_t* touched) {
    const int tiles_x = (W + TILE - 1) / TILE, tiles_y = (H + TILE - 1) / TILE;
    if (tile_order && !meta) return set_error("raster_bwd_rec: a raster order needs the frame meta");
    static const size_t bwd_pad = pad_env("GS_BWD_PAD");
    static bool once = false;
    if (!once) {
        once = true;
        carve_env("GS_BWD_CARVE", raster_bwd_rec_kernel);
    }
    launch_k(raster_bwd_rec_kernel, dim3((unsigned)(tiles_x * tiles_y * (4 / BWD_WPC))), dim3(32 * BWD_WPC), bwd_pad, s,
             ranges, rec, rec_count,
             (const float4*)xydr4, (const float4*)conic4, colors3, bg, W, H, tiles_x, fT, nc, dimg, g8, d_c11,
             tile_order, meta, touched);
    return check_launch("raster_bwd_rec_kernel");
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
                             n_contrib, d_image, d_rgbo4, d_geo4, d_c11, counts, (cudaStream_t)stream, 1);
}

}  // extern "C"
