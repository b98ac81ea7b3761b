// segsort.cu -- per-tile depth sort (segment binning for small scenes).
//
// sg/binning.py:27-65 wants every tile's list in (depth, source_index)
// order.  The depth-first path (frame.cu) gets it from a global stable sort
// of the N depth keys (4 onesweep passes) before emission.  For small scenes
// those passes are latency-bound (~8 us each at N = 1e5), so the segment
// path instead emits in Gaussian-index order, stably sorts by tile id, and
// then sorts each tile's list here, stably by the depth key of its
// Gaussians: stable on an index-ordered list = (depth, index) order.
//
// One CTA per tile.  The list is processed in chunks of SEG_CHUNK entries
// with the onesweep ranking (per-warp peer masks built with shared atomic
// OR, input order = (warp, item, lane)); digit starts come from the
// segment's own per-byte histograms (one read pass, which also finds the
// key bytes that are constant over the segment -- those passes are
// skipped; depths within a tile usually share their top byte).  Passes
// ping-pong between the list and its alternate buffer through L2; keys are
// re-gathered from the per-Gaussian key array every pass.
#include "common.cuh"
#include "internal.cuh"

namespace gs {

constexpr int SEG_THREADS = 256;
constexpr int SEG_WARPS = SEG_THREADS / 32;
constexpr int SEG_ITEMS = 4;
constexpr int SEG_CHUNK = SEG_THREADS * SEG_ITEMS;

// Short lists (the common case): one warp per tile, the whole list in
// registers (WS_ITEMS per lane, input order = (item, lane)).  One read of
// the list builds the warp's per-byte digit histograms (and finds the key
// bytes that are constant over the list -- skipped); each varying byte is
// then one stable peer-mask ranking pass that scatters every item to its
// final slot as soon as it is ranked (digit starts known up front, so no
// per-item rank registers), no CTA barriers.  Sized to stay at <= 96
// registers so a frame's tiles fit one wave (5 CTAs of 4 warps per SM).
// Longer lists are left to segsort_kernel below.
constexpr int WS_ITEMS = 16;
constexpr int WS_MAX = 32 * WS_ITEMS;  // 512 entries
constexpr int WS_WARPS = 4;

__global__ void __launch_bounds__(32 * WS_WARPS, 5) segsort_warp_kernel(const uint2* __restrict__ ranges, int n_tiles,
                                                                       const uint32_t* __restrict__ dkeys,
                                                                       uint32_t* __restrict__ vals) {
    griddep_wait();
    __shared__ uint32_t s_peers[WS_WARPS][2][256];
    __shared__ uint32_t s_hist[WS_WARPS][4][256];  // digit counts, then running digit slots
    __shared__ uint32_t s_key[WS_WARPS][WS_MAX], s_val[WS_WARPS][WS_MAX];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.x * WS_WARPS + warp;
    if (tile >= n_tiles) return;
    const uint2 rg = ranges[tile];
    const int len = (int)(rg.y - rg.x);
    if (len <= 1 || len > WS_MAX) return;
    uint32_t* gv = vals + rg.x;
    uint32_t k[WS_ITEMS], v[WS_ITEMS];
    uint32_t o = 0u, a = ~0u;
#pragma unroll
    for (int i = 0; i < WS_ITEMS; ++i) {
        const int idx = i * 32 + lane;
        v[i] = idx < len ? gv[idx] : 0u;
    }
#pragma unroll
    for (int i = 0; i < WS_ITEMS; ++i) {
        const int idx = i * 32 + lane;
        k[i] = idx < len ? dkeys[v[i]] : 0u;
        if (idx < len) {
            o |= k[i];
            a &= k[i];
        }
    }
    const uint32_t vary = __reduce_or_sync(0xffffffffu, o) ^ __reduce_and_sync(0xffffffffu, a);
    if (vary == 0u) return;  // all keys equal: the index order already is the answer
    {
        uint4* z = reinterpret_cast<uint4*>(&s_peers[warp][0][0]);
        for (int j = lane; j < 2 * 256 / 4; j += 32) z[j] = make_uint4(0u, 0u, 0u, 0u);
        z = reinterpret_cast<uint4*>(&s_hist[warp][0][0]);
        for (int j = lane; j < 4 * 256 / 4; j += 32) z[j] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < WS_ITEMS; ++i) {
        if (i * 32 + lane < len) {
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if ((vary >> (8 * b)) & 255u) atomicAdd(&s_hist[warp][b][(k[i] >> (8 * b)) & 255u], 1u);
        }
    }
    __syncwarp();
    const uint32_t lt = lanemask_lt();
    for (int b = 0; b < 4; ++b) {
        if (((vary >> (8 * b)) & 255u) == 0u) continue;
        const int shift = 8 * b;
        uint32_t* cnt = s_hist[warp][b];
        {  // exclusive scan of the 256 digit counts: 8 per lane + warp scan
            uint32_t c8[8], run = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c8[j] = cnt[lane * 8 + j];
                run += c8[j];
            }
            uint32_t incl = run;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            uint32_t base = incl - run;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                cnt[lane * 8 + j] = base;
                base += c8[j];
            }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < WS_ITEMS; ++i) {
            const bool valid = i * 32 + lane < len;
            const uint32_t d = (k[i] >> shift) & 255u;
            uint32_t* pm = &s_peers[warp][i & 1][d];
            if (valid) atomicOr(pm, 1u << lane);
            __syncwarp();
            const uint32_t peers = valid ? *pm : 0u;
            const uint32_t old = valid ? cnt[d] : 0u;
            __syncwarp();
            if (valid) {
                if ((peers & lt) == 0u) {
                    cnt[d] = old + (uint32_t)__popc(peers);
                    *pm = 0u;
                }
                const uint32_t pos = old + (uint32_t)__popc(peers & lt);
                s_key[warp][pos] = k[i];
                s_val[warp][pos] = v[i];
            }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < WS_ITEMS; ++i) {
            const int idx = i * 32 + lane;
            if (idx < len) {
                k[i] = s_key[warp][idx];
                v[i] = s_val[warp][idx];
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < WS_ITEMS; ++i) {
        const int idx = i * 32 + lane;
        if (idx < len) gv[idx] = v[i];
    }
}

// Long lists (len > WS_MAX): one CTA per tile, chunked passes through L2.
// A few CTAs stride over the tiles (long lists are rare) instead of one CTA
// per tile that mostly exits at once.
__global__ void __launch_bounds__(SEG_THREADS) segsort_kernel(const uint2* __restrict__ ranges, int n_tiles,
                                                              const uint32_t* __restrict__ dkeys,
                                                              uint32_t* __restrict__ vals,
                                                              uint32_t* __restrict__ alt) {
    griddep_wait();
    __shared__ uint32_t s_hist[4][256];                 // per byte, then running digit starts
    __shared__ uint32_t s_whist[SEG_WARPS][256];        // per-warp digit counts of the chunk
    __shared__ uint32_t s_peers[SEG_WARPS][2][256];     // peer-mask banks
    __shared__ uint32_t s_or, s_and;
    __shared__ uint32_t s_tmp[SEG_WARPS];
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint2 rg = ranges[tile];
        const int start = (int)rg.x, len = (int)(rg.y - rg.x);
        if (len <= WS_MAX) continue;  // segsort_warp_kernel's
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        for (int k = tid; k < 4 * 256; k += SEG_THREADS) (&s_hist[0][0])[k] = 0u;
        for (int k = tid; k < SEG_WARPS * 2 * 256; k += SEG_THREADS) (&s_peers[0][0][0])[k] = 0u;
        if (tid == 0) {
            s_or = 0u;
            s_and = ~0u;
        }
        __syncthreads();
        // 1. per-byte histograms + which bytes vary
        uint32_t o = 0u, a = ~0u;
        for (int i = tid; i < len; i += SEG_THREADS) {
            const uint32_t key = dkeys[vals[start + i]];
            o |= key;
            a &= key;
    #pragma unroll
            for (int b = 0; b < 4; ++b) atomicAdd(&s_hist[b][(key >> (8 * b)) & 255u], 1u);
        }
        o = __reduce_or_sync(0xffffffffu, o);
        a = __reduce_and_sync(0xffffffffu, a);
        if (lane == 0) {
            atomicOr(&s_or, o);
            atomicAnd(&s_and, a);
        }
        __syncthreads();
        const uint32_t vary = s_or ^ s_and;
        // exclusive digit starts per byte (thread = digit)
    #pragma unroll 1
        for (int b = 0; b < 4; ++b) {
            const uint32_t c = s_hist[b][tid];
            uint32_t incl = c;
    #pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            if (lane == 31) s_tmp[warp] = incl;
            __syncthreads();
            uint32_t base = 0;
            for (int w = 0; w < warp; ++w) base += s_tmp[w];
            __syncthreads();
            s_hist[b][tid] = base + incl - c;
        }
        __syncthreads();
        // 2. one stable scatter pass per varying byte
        uint32_t* src = vals + start;
        uint32_t* dst = alt + start;
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
                    d[i] = idx < len ? (dkeys[v[i]] >> shift) & 255u : 256u;
                }
    #pragma unroll
                for (int k = 0; k < SEG_WARPS; ++k) s_whist[k][tid] = 0u;
                __syncthreads();
    #pragma unroll
                for (int i = 0; i < SEG_ITEMS; ++i) {
                    const bool valid = d[i] < 256u;
                    uint32_t* pm = &s_peers[warp][i & 1][valid ? d[i] : 0];
                    if (valid) atomicOr(pm, 1u << lane);
                    __syncwarp();
                    const uint32_t peers = valid ? *pm : 0u;
                    const uint32_t old = valid ? s_whist[warp][d[i]] : 0u;
                    __syncwarp();
                    if (valid && (peers & lt) == 0u) {
                        s_whist[warp][d[i]] = old + (uint32_t)__popc(peers);
                        *pm = 0u;
                    }
                    rank[i] = old + (uint32_t)__popc(peers & lt);
                }
                __syncthreads();
                // per digit: warp offsets within the chunk, then advance the digit start
                {
                    uint32_t run = s_hist[b][tid];
    #pragma unroll
                    for (int w = 0; w < SEG_WARPS; ++w) {
                        const uint32_t cnt = s_whist[w][tid];
                        s_whist[w][tid] = run;
                        run += cnt;
                    }
                    s_hist[b][tid] = run;
                }
                __syncthreads();
    #pragma unroll
                for (int i = 0; i < SEG_ITEMS; ++i)
                    if (d[i] < 256u) dst[s_whist[warp][d[i]] + rank[i]] = v[i];
                __syncthreads();
            }
            uint32_t* t = src;
            src = dst;
            dst = t;
        }
        if (src != vals + start) {  // odd number of passes: copy back
            for (int i = tid; i < len; i += SEG_THREADS) vals[start + i] = src[i];
        }
        __syncthreads();  // shared state is reset for the next tile
    }
}

int launch_segsort(const uint2* ranges, int n_tiles, const uint32_t* dkeys, uint32_t* vals, uint32_t* alt,
                   cudaStream_t s) {
    if (n_tiles <= 0) return 0;
    static const bool carve = [] {  // 5 CTAs x 41 KB: ask for the full shared-memory carveout
        return cudaFuncSetAttribute(segsort_warp_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    (int)cudaSharedmemCarveoutMaxShared) == cudaSuccess;
    }();
    (void)carve;
    launch_k(segsort_warp_kernel, dim3((unsigned)((n_tiles + WS_WARPS - 1) / WS_WARPS)), dim3(32 * WS_WARPS), 0, s,
             ranges, n_tiles, dkeys, vals);
    if (check_launch("segsort_warp_kernel")) return -1;
    launch_k(segsort_kernel, dim3((unsigned)min(n_tiles, 2 * 148)), dim3(SEG_THREADS), 0, s, ranges, n_tiles, dkeys,
             vals, alt);
    return check_launch("segsort_kernel");
}

}  // namespace gs
