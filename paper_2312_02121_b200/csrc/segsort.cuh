#pragma once
// segsort.cuh -- per-tile sort of the scatter-binned lists (small scenes),
// as CTA-wide device code: run by segsort_kernel (segsort.cu) or fused into
// the top of the raster forward (raster.cu), one tile per CTA of 128 threads.
//
// sg/binning.py:27-65 wants every tile's list in (depth, source_index)
// order.  The depth-first path (frame.cu) gets it from a global stable sort
// of the N depth keys (4 onesweep passes) before emission.  For small scenes
// those passes are latency-bound, so the scatter path writes every tile's
// pairs straight into its range in arbitrary order (binning.cu) and sorts
// each range here: a stable LSD radix sort by the Gaussians' depth keys,
// then a check for equal depths next to each other.  Ties (rare: exactly
// equal float depths) re-sort the range by source index first and by depth
// second, which is the (depth, index) order whatever the input order was.
//
// Key bytes that are constant over a range are skipped (depths within a
// tile usually share their top byte); a range whose depths are all equal
// is one tie run and gets the index passes only.

#include "common.cuh"

namespace gs {

constexpr int SEG_THREADS = 128;
constexpr int SEG_WARPS = SEG_THREADS / 32;
constexpr int SEG_ITEMS = 4;
constexpr int SEG_CHUNK = SEG_THREADS * SEG_ITEMS;

// Short lists (the common case, len <= WS_MAX): one CTA of 4 warps per
// tile, 4 items per thread in registers (input order = (warp, item, lane)),
// everything else in shared memory.  Each varying key byte is one stable
// pass: per-warp peer-mask ranking (shared atomic OR; the lowest peer adds
// the group to the warp's digit count), a CTA scan of the digits' per-warp
// counts, a scatter to the digit start + warp offset + rank and a gather
// back into registers.  Four items per lane keep the per-pass dependency
// chain short (the ranking is the latency-bound part).
constexpr int WS_WARPS = 4;
constexpr int WS_THREADS = 32 * WS_WARPS;
constexpr int WS_ITEMS = 4;
constexpr int WS_MAX = WS_THREADS * WS_ITEMS;  // 512 entries

struct SmallShared {
    uint32_t peers[WS_WARPS][2][256];
    uint32_t whist[WS_WARPS][256];  // per-warp digit counts, then their output offsets
    uint32_t key[WS_MAX], val[WS_MAX];
    uint32_t tmp[WS_WARPS];
    uint32_t red[4];  // key or / and, index or / and
    uint32_t tie;
};

// load(idx): the input value at list position idx (all loads happen before
// any write to gv, so the input may live inside gv's range).
template <typename Load>
__device__ __forceinline__ void small_sort(SmallShared& sh, const uint32_t* __restrict__ dkeys, uint32_t* gv,
                                           int len, Load load) {
    auto& s_peers = sh.peers;
    auto& s_whist = sh.whist;
    auto& s_key = sh.key;
    auto& s_val = sh.val;
    auto& s_tmp = sh.tmp;
    auto& s_red = sh.red;
    auto& s_tie = sh.tie;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ibase = warp * (32 * WS_ITEMS) + lane;  // item i at ibase + 32 i
    uint32_t k[WS_ITEMS], v[WS_ITEMS];
    if (tid == 0) {
        s_red[0] = 0u;
        s_red[1] = ~0u;
        s_red[2] = 0u;
        s_red[3] = ~0u;
        s_tie = 0u;
    }
#pragma unroll
    for (int i = 0; i < WS_ITEMS; ++i) v[i] = ibase + 32 * i < len ? load(ibase + 32 * i) : 0u;
    uint32_t ko = 0u, ka = ~0u, vo = 0u, va = ~0u;
#pragma unroll
    for (int i = 0; i < WS_ITEMS; ++i) {
        const bool in = ibase + 32 * i < len;
        k[i] = in ? dkeys[v[i]] : 0u;
        if (in) {
            ko |= k[i];
            ka &= k[i];
            vo |= v[i];
            va &= v[i];
        }
    }
    for (int j = lane; j < 2 * 256; j += 32) (&s_peers[warp][0][0])[j] = 0u;
    __syncthreads();
    ko = __reduce_or_sync(0xffffffffu, ko);
    ka = __reduce_and_sync(0xffffffffu, ka);
    vo = __reduce_or_sync(0xffffffffu, vo);
    va = __reduce_and_sync(0xffffffffu, va);
    if (lane == 0) {
        atomicOr(&s_red[0], ko);
        atomicAnd(&s_red[1], ka);
        atomicOr(&s_red[2], vo);
        atomicAnd(&s_red[3], va);
    }
    __syncthreads();
    const uint32_t kvary = s_red[0] ^ s_red[1], vvary = s_red[2] ^ s_red[3];
    const uint32_t lt = lanemask_lt();
    // one stable pass over byte `shift` of the depth keys (by_id false) or
    // of the source indices (by_id true)
    auto pass = [&](bool by_id, int shift) {
        for (int j = lane; j < 256; j += 32) s_whist[warp][j] = 0u;
        __syncwarp();
        uint32_t rank[WS_ITEMS], dg[WS_ITEMS];
#pragma unroll
        for (int i = 0; i < WS_ITEMS; ++i) {
            const bool valid = ibase + 32 * i < len;
            const uint32_t d = ((by_id ? v[i] : k[i]) >> shift) & 255u;
            dg[i] = d;
            uint32_t* pm = &s_peers[warp][i & 1][d];
            if (valid) atomicOr(pm, 1u << lane);
            __syncwarp();
            const uint32_t peers = valid ? *pm : 0u;
            const uint32_t old = valid ? s_whist[warp][d] : 0u;
            __syncwarp();
            if (valid && (peers & lt) == 0u) {
                s_whist[warp][d] = old + (uint32_t)__popc(peers);
                *pm = 0u;
            }
            rank[i] = old + (uint32_t)__popc(peers & lt);
        }
        __syncthreads();
        {  // digits DPT tid ..: CTA exclusive scan of the totals, then per-warp offsets
            constexpr int DPT = 256 / WS_THREADS;
            uint32_t c[DPT][WS_WARPS], mine = 0u;
#pragma unroll
            for (int h = 0; h < DPT; ++h) {
#pragma unroll
                for (int w = 0; w < WS_WARPS; ++w) {
                    c[h][w] = s_whist[w][DPT * tid + h];
                    mine += c[h][w];
                }
            }
            uint32_t incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_tmp[warp] = incl;
            __syncthreads();
            uint32_t run = incl - mine;
            for (int w = 0; w < warp; ++w) run += s_tmp[w];
#pragma unroll
            for (int h = 0; h < DPT; ++h)
#pragma unroll
                for (int w = 0; w < WS_WARPS; ++w) {
                    s_whist[w][DPT * tid + h] = run;
                    run += c[h][w];
                }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < WS_ITEMS; ++i)
            if (ibase + 32 * i < len) {
                const uint32_t pos = s_whist[warp][dg[i]] + rank[i];
                s_key[pos] = k[i];
                s_val[pos] = v[i];
            }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < WS_ITEMS; ++i)
            if (ibase + 32 * i < len) {
                k[i] = s_key[ibase + 32 * i];
                v[i] = s_val[ibase + 32 * i];
            }
        __syncthreads();
    };
    bool tie = kvary == 0u;  // all depths equal: one tie run
    if (!tie) {
        for (int b = 0; b < 4; ++b)
            if ((kvary >> (8 * b)) & 255u) pass(false, 8 * b);
        // s_key holds the depth-sorted keys: any equal neighbours?
        bool t = false;
#pragma unroll
        for (int i = 0; i < WS_ITEMS; ++i) {
            const int idx = ibase + 32 * i;
            if (idx > 0 && idx < len) t = t || s_key[idx] == s_key[idx - 1];
        }
        if (__any_sync(0xffffffffu, t) && lane == 0) s_tie = 1u;
        __syncthreads();
        tie = s_tie != 0u;
    }
    if (tie) {  // (depth, index) order: index bytes first, then depth bytes
        for (int b = 0; b < 4; ++b)
            if ((vvary >> (8 * b)) & 255u) pass(true, 8 * b);
        for (int b = 0; b < 4; ++b)
            if ((kvary >> (8 * b)) & 255u) pass(false, 8 * b);
    }
#pragma unroll
    for (int i = 0; i < WS_ITEMS; ++i)
        if (ibase + 32 * i < len) gv[ibase + 32 * i] = v[i];
}

// Long lists (len > WS_MAX): the CTA sorts its range with chunked passes
// through L2 (ping-pong between the range and its alternate buffer).  One
// read pass builds the per-byte histograms of the key (depth key, or source
// index when by_id) and finds its constant bytes; each varying byte is then
// one stable pass: SEG_CHUNK entries at a time with the onesweep ranking
// (per-warp peer masks built with shared atomic OR, input order = (warp,
// item, lane)).  Ends with the sorted range back in `seg`.
struct SegShared {
    uint32_t hist[4][256];            // per byte, then running digit starts
    uint32_t whist[SEG_WARPS][256];   // per-warp digit counts of the chunk
    uint32_t peers[SEG_WARPS][2][256];  // peer-mask banks
    uint32_t vor, vand, flag;
    uint32_t tmp[SEG_WARPS];
};

__device__ __forceinline__ uint32_t seg_key(const uint32_t* __restrict__ dkeys, uint32_t v, bool by_id) {
    return by_id ? v : dkeys[v];
}

static __device__ __noinline__ void cta_radix(SegShared& sh, const uint32_t* __restrict__ dkeys, uint32_t* seg,
                                              uint32_t* alt, int len, bool by_id) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int k = tid; k < 4 * 256; k += SEG_THREADS) (&sh.hist[0][0])[k] = 0u;
    for (int k = tid; k < SEG_WARPS * 2 * 256; k += SEG_THREADS) (&sh.peers[0][0][0])[k] = 0u;
    if (tid == 0) {
        sh.vor = 0u;
        sh.vand = ~0u;
    }
    __syncthreads();
    // 1. per-byte histograms + which bytes vary
    uint32_t o = 0u, a = ~0u;
    for (int i = tid; i < len; i += SEG_THREADS) {
        const uint32_t key = seg_key(dkeys, seg[i], by_id);
        o |= key;
        a &= key;
#pragma unroll
        for (int b = 0; b < 4; ++b) atomicAdd(&sh.hist[b][(key >> (8 * b)) & 255u], 1u);
    }
    o = __reduce_or_sync(0xffffffffu, o);
    a = __reduce_and_sync(0xffffffffu, a);
    if (lane == 0) {
        atomicOr(&sh.vor, o);
        atomicAnd(&sh.vand, a);
    }
    __syncthreads();
    const uint32_t vary = sh.vor ^ sh.vand;
    // exclusive digit starts per byte (thread = DPT consecutive digits)
    constexpr int DPT = 256 / SEG_THREADS;
#pragma unroll 1
    for (int b = 0; b < 4; ++b) {
        uint32_t c[DPT], mine = 0u;
#pragma unroll
        for (int h = 0; h < DPT; ++h) {
            c[h] = sh.hist[b][DPT * tid + h];
            mine += c[h];
        }
        uint32_t incl = mine;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        if (lane == 31) sh.tmp[warp] = incl;
        __syncthreads();
        uint32_t base = incl - mine;
        for (int w = 0; w < warp; ++w) base += sh.tmp[w];
        __syncthreads();
#pragma unroll
        for (int h = 0; h < DPT; ++h) {
            sh.hist[b][DPT * tid + h] = base;
            base += c[h];
        }
    }
    __syncthreads();
    // 2. one stable scatter pass per varying byte
    uint32_t* src = seg;
    uint32_t* dst = alt;
    const uint32_t lt = lanemask_lt();
    for (int b = 0; b < 4; ++b) {
        if (((vary >> (8 * b)) & 255u) == 0u) continue;  // constant byte: identity pass
        const int shift = 8 * b;
        for (int c0 = 0; c0 < len; c0 += SEG_CHUNK) {
            const int wbase = c0 + warp * (SEG_ITEMS * 32);
            uint32_t v[SEG_ITEMS], d[SEG_ITEMS], rank[SEG_ITEMS];
#pragma unroll
            for (int i = 0; i < SEG_ITEMS; ++i) {
                const int idx = wbase + i * 32 + lane;
                v[i] = idx < len ? src[idx] : 0u;
                d[i] = idx < len ? (seg_key(dkeys, v[i], by_id) >> shift) & 255u : 256u;
            }
            for (int k = tid; k < SEG_WARPS * 256; k += SEG_THREADS) (&sh.whist[0][0])[k] = 0u;
            __syncthreads();
#pragma unroll
            for (int i = 0; i < SEG_ITEMS; ++i) {
                const bool valid = d[i] < 256u;
                uint32_t* pm = &sh.peers[warp][i & 1][valid ? d[i] : 0];
                if (valid) atomicOr(pm, 1u << lane);
                __syncwarp();
                const uint32_t peers = valid ? *pm : 0u;
                const uint32_t old = valid ? sh.whist[warp][d[i]] : 0u;
                __syncwarp();
                if (valid && (peers & lt) == 0u) {
                    sh.whist[warp][d[i]] = old + (uint32_t)__popc(peers);
                    *pm = 0u;
                }
                rank[i] = old + (uint32_t)__popc(peers & lt);
            }
            __syncthreads();
            // per digit: warp offsets within the chunk, then advance the digit start
            for (int dd = tid; dd < 256; dd += SEG_THREADS) {
                uint32_t run = sh.hist[b][dd];
#pragma unroll
                for (int w = 0; w < SEG_WARPS; ++w) {
                    const uint32_t cnt = sh.whist[w][dd];
                    sh.whist[w][dd] = run;
                    run += cnt;
                }
                sh.hist[b][dd] = run;
            }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < SEG_ITEMS; ++i)
                if (d[i] < 256u) dst[sh.whist[warp][d[i]] + rank[i]] = v[i];
            __syncthreads();
        }
        uint32_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != seg) {  // odd number of passes: copy back
        for (int i = tid; i < len; i += SEG_THREADS) seg[i] = src[i];
    }
    __syncthreads();
}

// Shared memory of one tile sort (either strategy).
union SegsortShared {
    SmallShared small;
    SegShared large;
};

// Sort one tile's range rg of vals by (depth key, index): short lists in
// shared memory (small_sort), long ones with chunked passes through L2
// (cta_radix) plus the tie repair.  Called by all 128 threads of the CTA;
// ends with the CTA synchronized and the sorted range visible to it.
__device__ __forceinline__ void segsort_tile(SegsortShared& sh, uint2 rg, const uint32_t* __restrict__ dkeys,
                                             uint32_t* __restrict__ vals, uint32_t* __restrict__ alt) {
    const int len = (int)(rg.y - rg.x);
    if (len <= 1) return;
    uint32_t* seg = vals + rg.x;
    if (len <= WS_MAX) {
        small_sort(sh.small, dkeys, seg, len, [&](int i) { return seg[i]; });
        __syncthreads();
        return;
    }
    cta_radix(sh.large, dkeys, seg, alt + rg.x, len, false);
    // equal depths next to each other?  then (index, then depth) passes
    if (threadIdx.x == 0) sh.large.flag = 0u;
    __syncthreads();
    bool t = false;
    for (int i = 1 + (int)threadIdx.x; i < len; i += SEG_THREADS) t = t || dkeys[seg[i]] == dkeys[seg[i - 1]];
    if (__any_sync(0xffffffffu, t) && (threadIdx.x & 31) == 0) sh.large.flag = 1u;
    __syncthreads();
    if (sh.large.flag) {
        cta_radix(sh.large, dkeys, seg, alt + rg.x, len, true);
        cta_radix(sh.large, dkeys, seg, alt + rg.x, len, false);
    }
}

// Direct binning with replicated slot counters: the tile's list is NR
// segments, segment j at vals[base + j * kr, + cnt[j]).  Sorted by
// (depth, index) into vals[base, + sum cnt) (the NR segments are gathered
// first; the first segment's data is already in place).
template <int NR>
__device__ __forceinline__ void segsort_tile_segments(SegsortShared& sh, uint32_t base, uint32_t kr,
                                                      const uint32_t (&cnt)[NR],
                                                      const uint32_t* __restrict__ dkeys,
                                                      uint32_t* __restrict__ vals, uint32_t* __restrict__ alt) {
    uint32_t pre[NR + 1];
    pre[0] = 0;
#pragma unroll
    for (int j = 0; j < NR; ++j) pre[j + 1] = pre[j] + cnt[j];
    const int len = (int)pre[NR];
    uint32_t* seg = vals + base;
    auto load = [&](int i) {  // list position -> segment value
        int j = 0;
#pragma unroll
        for (int q = 1; q < NR; ++q) j += (uint32_t)i >= pre[q] ? 1 : 0;
        return seg[(uint32_t)j * kr + ((uint32_t)i - pre[j])];
    };
    if (len <= WS_MAX) {
        if (len == 1) {
            if (threadIdx.x == 0) seg[0] = load(0);
            __syncthreads();
            return;
        }
        if (len > 1) small_sort(sh.small, dkeys, seg, len, load);
        __syncthreads();
        return;
    }
    // long list: gather into alt, copy back contiguous, then the in-place path
    uint32_t* tmp = alt + base;
    for (int i = threadIdx.x; i < len; i += SEG_THREADS) tmp[i] = load(i);
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += SEG_THREADS) seg[i] = tmp[i];
    __syncthreads();
    segsort_tile(sh, make_uint2(base, base + (uint32_t)len), dkeys, vals, alt);
    __syncthreads();
}

}  // namespace gs
