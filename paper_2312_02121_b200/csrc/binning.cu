// binning.cu -- stage 2 around the sort: exclusive scan of the per-Gaussian
// tile counts (single-pass decoupled look-back), key emission and per-tile
// range detection.  Together with sort.cu these replace sg/binning.py:27-65
// (assign_tiles + sort_bins).  All HBM-bound.
#include <cstdlib>

#include "common.cuh"
#include "internal.cuh"

namespace gs {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;  // 4096 counts per CTA
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;
constexpr unsigned long long FLAG_AGG = 1ull << 62;
constexpr unsigned long long FLAG_PRE = 2ull << 62;
constexpr unsigned long long VAL_MASK = (1ull << 62) - 1;

// look-back status words (flag and value in one 64-bit word): GPU-scope
// relaxed accesses (volatile would make them system-scope)
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ws layout: [0] tile counter (u32, padded to 16 B), then u64 status[ctas].
// gather != nullptr: scans in[gather[p]] (counts in depth-sorted order).
__global__ void __launch_bounds__(SCAN_THREADS) scan_kernel(const uint32_t* __restrict__ in,
                                                           const uint32_t* __restrict__ gather,
                                                           uint32_t* __restrict__ out, int64_t n,
                                                           unsigned int* __restrict__ tile_counter,
                                                           unsigned long long* __restrict__ status,
                                                           unsigned long long* __restrict__ total) {
    griddep_wait();
    __shared__ unsigned int s_tile;
    __shared__ unsigned long long s_warp[SCAN_THREADS / 32];
    __shared__ unsigned long long s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const unsigned int tile = s_tile;
    const int64_t base = (int64_t)tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
    if (gather) {
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) v[k] = (base + k < n) ? in[gather[base + k]] : 0u;
    } else if (base + SCAN_ITEMS <= n && ((reinterpret_cast<uintptr_t>(in + base) & 15) == 0)) {
        const uint4* p = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS / 4; ++k) {
            const uint4 q = p[k];
            v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) v[k] = (base + k < n) ? in[base + k] : 0u;
    }
    unsigned long long sum = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) sum += v[k];
    // block exclusive scan of the per-thread sums
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    unsigned long long warp_off = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < SCAN_THREADS / 32; ++w) {
        const unsigned long long s = s_warp[w];
        if (w < warp) warp_off += s;
        agg += s;
    }
    // decoupled look-back (one thread)
    if (threadIdx.x == 0) {
        unsigned long long prefix = 0;
        if (tile == 0) {
            st_volatile(&status[0], FLAG_PRE | agg);
        } else {
            st_volatile(&status[tile], FLAG_AGG | agg);
            __threadfence();
            int p = (int)tile - 1;
            while (true) {
                const unsigned long long s = ld_volatile(&status[p]);
                const unsigned long long f = s & ~VAL_MASK;
                if (f == 0) continue;
                prefix += s & VAL_MASK;
                if (f == FLAG_PRE) break;
                --p;
            }
            st_volatile(&status[tile], FLAG_PRE | (prefix + agg));
        }
        s_prefix = prefix;
        if ((int64_t)(tile + 1) * SCAN_TILE >= n) *total = prefix + agg;
    }
    __syncthreads();
    unsigned long long run = s_prefix + warp_off + (incl - sum);
    uint32_t o[SCAN_ITEMS];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        o[k] = (uint32_t)run;
        run += v[k];
    }
    if (base + SCAN_ITEMS <= n && ((reinterpret_cast<uintptr_t>(out + base) & 15) == 0)) {
        uint4* p = reinterpret_cast<uint4*>(out + base);
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS / 4; ++k) p[k] = make_uint4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k)
            if (base + k < n) out[base + k] = o[k];
    }
}

// sg/binning.py:35-46: one (tile, gaussian) pair per tile of the rectangle,
// row-major within a Gaussian, Gaussians in index order.
__global__ void __launch_bounds__(256) emit_kernel(const float4* __restrict__ xydr,
                                                   const uint32_t* __restrict__ offsets,
                                                   const uint32_t* __restrict__ tiles, int n, int tiles_x,
                                                   int tiles_y, unsigned long long* __restrict__ keys,
                                                   uint32_t* __restrict__ vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (tiles[i] == 0u) return;
    const float4 g = xydr[i];
    const int r = __float_as_int(g.w);
    int tx0, tx1, ty0, ty1;
    tile_rect(g.x, g.y, r, tiles_x, tiles_y, tx0, tx1, ty0, ty1);
    const unsigned long long dbits = (unsigned long long)__float_as_uint(g.z);
    uint32_t off = offsets[i];
    for (int ty = ty0; ty <= ty1; ++ty) {
        for (int tx = tx0; tx <= tx1; ++tx) {
            keys[off] = ((unsigned long long)(ty * tiles_x + tx) << 32) | dbits;
            vals[off] = (uint32_t)i;
            ++off;
        }
    }
}

// Tiles touched by an arbitrary (mean2d, radius) square (radius < 0 counts
// 0), clamped to the grid like sg/binning.py:38-43 -- an off-image square
// yields an empty rectangle.
__global__ void __launch_bounds__(256) tile_counts_kernel(const float4* __restrict__ xydr, int n, int tiles_x,
                                                          int tiles_y, uint32_t* __restrict__ tiles) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 g = xydr[i];
    const int r = __float_as_int(g.w);
    uint32_t c = 0;
    if (r >= 0 && fabsf(g.x) < 1.6e7f && fabsf(g.y) < 1.6e7f) {
        int tx0, tx1, ty0, ty1;
        tile_rect(g.x, g.y, min(r, MAX_RADIUS), tiles_x, tiles_y, tx0, tx1, ty0, ty1);
        c = (uint32_t)(max(0, tx1 - tx0 + 1) * max(0, ty1 - ty0 + 1));
    }
    tiles[i] = c;
}

__global__ void __launch_bounds__(256) ranges_kernel(const unsigned long long* __restrict__ keys, int64_t n,
                                                     uint2* __restrict__ ranges) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = (uint32_t)(keys[i] >> 32);
    if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != t) ranges[t].x = (uint32_t)i;
    if (i == n - 1 || (uint32_t)(keys[i + 1] >> 32) != t) ranges[t].y = (uint32_t)(i + 1);
}

// Depth-first emission: thread p handles the p-th Gaussian in (depth, index)
// order (order[] from the depth sort) and writes one (tile id, gaussian id)
// pair per tile of its rectangle, row-major, at offsets[p] + k.  A STABLE
// sort on the tile id then yields per-tile lists in (depth, source_index)
// order -- sg/binning.py:50-65 -- with 32-bit keys and 1-2 passes.  The
// digit histograms of that sort are accumulated here (warp-aggregated).
// Pairs at or beyond `capacity` are dropped (the caller re-runs with a
// larger buffer when the reported total exceeds it).
__global__ void __launch_bounds__(256) emit_sorted_kernel(const uint32_t* __restrict__ order,
                                                          const float4* __restrict__ xydr,
                                                          const uint32_t* __restrict__ offsets, int n, int tiles_x,
                                                          int tiles_y, int64_t capacity,
                                                          uint32_t* __restrict__ tile_keys,
                                                          uint32_t* __restrict__ vals,
                                                          uint32_t* __restrict__ tile_hist, int tile_passes) {
    griddep_wait();
    __shared__ uint32_t sh[2 * 256];
    for (int k = threadIdx.x; k < 2 * 256; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    // grid-stride over Gaussians (whole warps per trip); the shared tile-digit
    // histograms are flushed once per CTA
    const int n_round = (n + 31) & ~31;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n_round; p += gridDim.x * blockDim.x) {
    int tx0 = 0, tx1 = -1, ty0 = 0, ty1 = -1;
    uint32_t g = 0, off = 0;
    if (p < n) {
        g = order ? order[p] : (uint32_t)p;  // order == nullptr: Gaussian-index order
        off = offsets[p];
        const float4 gx = xydr[g];
        const int r = __float_as_int(gx.w);
        if (r > 0) tile_rect(gx.x, gx.y, r, tiles_x, tiles_y, tx0, tx1, ty0, ty1);
    }
    // The warp's 32 Gaussians own the contiguous output range
    // [off(lane 0), off(lane 0) + total): the warp walks it 32 entries at a
    // time (coalesced stores); each entry finds its owner lane by a binary
    // search over the lanes' exclusive prefix and decodes its tile row-major.
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
    const uint32_t base = __shfl_sync(0xffffffffu, off, 0);
    const float rw = w > 0 ? 1.f / (float)w : 0.f;
    for (uint32_t t0 = 0; t0 < total; t0 += 32) {
        const uint32_t t = t0 + lane;
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
        const uint32_t og = __shfl_sync(0xffffffffu, g, L);
        int row = (int)((float)j * orw);
        if (row * ow > (int)j) --row;
        if ((row + 1) * ow <= (int)j) ++row;
        const uint32_t tile = (uint32_t)((oty0 + row) * tiles_x + otx0 + ((int)j - row * ow));
        const bool valid = t < total && (int64_t)(base + t) < capacity;
        if (valid) {
            tile_keys[base + t] = tile;
            vals[base + t] = og;
            atomicAdd(&sh[tile & 255u], 1u);
        }
        if (tile_passes > 1) warp_hist_add(sh + 256, (tile >> 8) & 255u, valid);  // high digit: few distinct values
    }
    }  // grid-stride
    __syncthreads();
    for (int k = threadIdx.x; k < tile_passes * 256; k += blockDim.x) {
        const uint32_t v = sh[k];
        if (v) atomicAdd(&tile_hist[k], v);
    }
}

// Warp-cooperative emission of 32 consecutive Gaussians' pairs (lane = one
// Gaussian, off = its output offset, rect given): the warp owns the
// contiguous range [off(lane 0), off(lane 0) + total) and walks it 32 entries
// at a time (coalesced stores), each entry finding its owner lane by binary
// search over the lanes' exclusive prefix and decoding its tile row-major.
__device__ __forceinline__ void emit_warp(int lane, uint32_t g, uint32_t base, int tx0, int tx1, int ty0, int ty1,
                                          int tiles_x, int64_t capacity, uint32_t* __restrict__ tile_keys,
                                          uint32_t* __restrict__ vals, uint32_t* sh, int tile_passes) {
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
    for (uint32_t t0 = 0; t0 < total; t0 += 32) {
        const uint32_t t = t0 + lane;
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
        const uint32_t og = __shfl_sync(0xffffffffu, g, L);
        int row = (int)((float)j * orw);
        if (row * ow > (int)j) --row;
        if ((row + 1) * ow <= (int)j) ++row;
        const uint32_t tile = (uint32_t)((oty0 + row) * tiles_x + otx0 + ((int)j - row * ow));
        const bool valid = t < total && (int64_t)(base + t) < capacity;
        if (valid) {
            tile_keys[base + t] = tile;
            vals[base + t] = og;
            atomicAdd(&sh[tile & 255u], 1u);
        }
        if (tile_passes > 1) warp_hist_add(sh + 256, (tile >> 8) & 255u, valid);  // high digit: few distinct values
    }
}

// Fused scan + emission (frame path): persistent CTAs take chunks of
// ES_CHUNK consecutive Gaussians (in depth order, or index order when order
// == nullptr) from a counter, scan their tile counts (the projection's
// per-Gaussian counts), get the chunk's output base by decoupled look-back
// and emit the pairs directly -- no offsets array, no separate scan kernel.
// Chunk layout: round r, warp w, lane -> Gaussian r * 256 + w * 32 + lane,
// so each warp emits 32 consecutive Gaussians per round.  The last chunk's
// CTA writes the intersection total.
constexpr int ES_THREADS = 256;

size_t emit_scan_ws_bytes(int64_t n) {
    const int64_t chunks = (n + ES_THREADS - 1) / ES_THREADS;  // sized for the 1-round variant
    return 16 + (size_t)(chunks > 0 ? chunks : 1) * sizeof(unsigned long long);
}

template <int ES_ROUNDS>
__global__ void __launch_bounds__(ES_THREADS) emit_scan_kernel(
    const uint32_t* __restrict__ order, const float4* __restrict__ xydr, const uint32_t* __restrict__ counts, int n,
    int tiles_x, int tiles_y, int64_t capacity, uint32_t* __restrict__ tile_keys, uint32_t* __restrict__ vals,
    uint32_t* __restrict__ tile_hist, int tile_passes, unsigned int* __restrict__ chunk_counter,
    unsigned long long* __restrict__ status, unsigned long long* __restrict__ total,
    const uint32_t* __restrict__ order_alt, const unsigned long long* __restrict__ sort_meta) {
    griddep_wait();
    if (sort_meta) {  // depth-first frame: meta[7] visible Gaussians sorted, in order_alt after an odd pass count
        if (sort_meta[1] & 1ull) order = order_alt;
        n = min(n, (int)sort_meta[0]);
    }
    constexpr int ES_CHUNK = ES_THREADS * ES_ROUNDS;
    __shared__ uint32_t sh[2 * 256];
    __shared__ uint32_t s_wsum[ES_ROUNDS][ES_THREADS / 32];
    __shared__ unsigned int s_chunk;
    __shared__ unsigned long long s_prefix;
    for (int k = threadIdx.x; k < 2 * 256; k += blockDim.x) sh[k] = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n_chunks = (n + ES_CHUNK - 1) / ES_CHUNK;
    while (true) {
        __syncthreads();  // s_chunk / s_wsum reuse
        if (threadIdx.x == 0) s_chunk = atomicAdd(chunk_counter, 1u);
        __syncthreads();
        const int chunk = (int)s_chunk;
        if (chunk >= n_chunks) break;
        uint32_t g[ES_ROUNDS], cnt[ES_ROUNDS];
#pragma unroll
        for (int r = 0; r < ES_ROUNDS; ++r) {
            const int p = chunk * ES_CHUNK + r * ES_THREADS + (int)threadIdx.x;
            g[r] = p < n ? (order ? order[p] : (uint32_t)p) : 0u;
            cnt[r] = p < n ? counts[g[r]] : 0u;
        }
#pragma unroll
        for (int r = 0; r < ES_ROUNDS; ++r) {
            uint32_t incl = cnt[r];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) s_wsum[r][warp] = incl;
        }
        __syncthreads();
        // the chunk's aggregate and this warp's base in every round
        unsigned long long agg = 0;
        uint32_t wbase[ES_ROUNDS];
#pragma unroll
        for (int r = 0; r < ES_ROUNDS; ++r) {
            uint32_t before = 0, rt = 0;
#pragma unroll
            for (int w = 0; w < ES_THREADS / 32; ++w) {
                const uint32_t v = s_wsum[r][w];
                if (w < warp) before += v;
                rt += v;
            }
            wbase[r] = (uint32_t)agg + before;
            agg += rt;
        }
        if (threadIdx.x == 0) {  // decoupled look-back
            unsigned long long prefix = 0;
            if (chunk == 0) {
                st_volatile(&status[0], FLAG_PRE | agg);
            } else {
                st_volatile(&status[chunk], FLAG_AGG | agg);
                __threadfence();
                // look-back: the immediate predecessor first (usually already
                // inclusive when chunks are processed in waves), then windows
                // of LB predecessor statuses per round trip
                constexpr int LB = 8;
                int q = chunk - 1;
                bool found = false;
                {
                    unsigned long long sv = ld_volatile(&status[q]);
                    while ((sv & ~VAL_MASK) == 0) sv = ld_volatile(&status[q]);
                    prefix += sv & VAL_MASK;
                    found = (sv & ~VAL_MASK) == FLAG_PRE;
                    --q;
                }
                while (!found) {
                    unsigned long long wv[LB];
#pragma unroll
                    for (int j = 0; j < LB; ++j) wv[j] = q - j >= 0 ? ld_volatile(&status[q - j]) : FLAG_PRE;
#pragma unroll
                    for (int j = 0; j < LB; ++j) {
                        if (!found) {
                            unsigned long long sv = wv[j];
                            while ((sv & ~VAL_MASK) == 0) sv = ld_volatile(&status[q - j]);
                            prefix += sv & VAL_MASK;
                            found = (sv & ~VAL_MASK) == FLAG_PRE;
                        }
                    }
                    q -= LB;
                }
                st_volatile(&status[chunk], FLAG_PRE | (prefix + agg));
            }
            s_prefix = prefix;
            if (chunk == n_chunks - 1) *total = prefix + agg;
        }
        __syncthreads();
        const uint32_t prefix = (uint32_t)s_prefix;
#pragma unroll
        for (int r = 0; r < ES_ROUNDS; ++r) {
            int tx0 = 0, tx1 = -1, ty0 = 0, ty1 = -1;
            if (cnt[r]) {
                const float4 gx = xydr[g[r]];
                tile_rect(gx.x, gx.y, __float_as_int(gx.w), tiles_x, tiles_y, tx0, tx1, ty0, ty1);
            }
            emit_warp(lane, g[r], prefix + wbase[r], tx0, tx1, ty0, ty1, tiles_x, capacity, tile_keys, vals, sh,
                      tile_passes);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < tile_passes * 256; k += blockDim.x) {
        const uint32_t v = sh[k];
        if (v) atomicAdd(&tile_hist[k], v);
    }
}

int launch_emit_scan(const uint32_t* order, const float* xydr4, const uint32_t* counts, int64_t n, int tiles_x,
                     int tiles_y, int64_t capacity, uint32_t* tile_keys, uint32_t* vals, uint32_t* tile_hist,
                     int tile_passes, void* ws, unsigned long long* total, cudaStream_t s, const uint32_t* order_alt,
                     const unsigned long long* sort_meta) {
    // small scenes: one Gaussian per thread per chunk (more CTAs in flight);
    // large: 4 rounds per chunk (fewer look-backs)
    const int rounds = n <= (1 << 18) ? 1 : 4;
    const int64_t chunks = (n + ES_THREADS * rounds - 1) / (ES_THREADS * rounds);
    const int64_t resident = (int64_t)sort_sm_count() * 8;
    int64_t grid = chunks < resident ? chunks : resident;
    if (grid < 1) grid = 1;
    unsigned int* counter = (unsigned int*)ws;
    unsigned long long* status = (unsigned long long*)((char*)ws + 16);
    if (rounds == 1)
        launch_k(emit_scan_kernel<1>, dim3((unsigned)grid), dim3(ES_THREADS), 0, s, order, (const float4*)xydr4,
                 counts, (int)n, tiles_x, tiles_y, capacity, tile_keys, vals, tile_hist, tile_passes, counter, status,
                 total, order_alt, sort_meta);
    else
        launch_k(emit_scan_kernel<4>, dim3((unsigned)grid), dim3(ES_THREADS), 0, s, order, (const float4*)xydr4,
                 counts, (int)n, tiles_x, tiles_y, capacity, tile_keys, vals, tile_hist, tile_passes, counter, status,
                 total, order_alt, sort_meta);
    return check_launch("emit_scan_kernel");
}

// ---------------------------------------------------------------- tile-sorted emission
// Depth-first binning without a global sort by tile (frame.cu, <= 10240
// tiles): every (tile, gaussian) pair is written straight to its final slot
//     start(tile) + #{pairs of the same tile emitted earlier}
// where "earlier" is the emission order of sg/binning.py:35-46 over the
// Gaussians in (depth, index) order -- exactly the stable order of
// sg/binning.py:50-65.  A stable counting sort whose digit is the whole tile
// id, over chunks of ET_CHUNK consecutive Gaussians of the depth order:
//   et_expand_kernel   walks each chunk's pairs once, in emission order,
//                      writing them as (chunk-local Gaussian << 16 | tile)
//                      words (every warp's run contiguous, placed by a
//                      decoupled look-back over the chunks' pair totals) and
//                      the chunk's per-tile counts (one u16 row)
//   et_colsum_kernel   per tile, the column sums of those counts over 32
//                      segments of chunks and the tile's total -> tcount
//   (tile_scan_kernel  the totals -> ranges, raster order, starts)
//   et_colscan_kernel  per (chunk, tile): start(tile) + the pairs of all
//                      earlier chunks (u32 rows)
//   et_place_kernel    per chunk: its row of bases and its Gaussian ids bulk-
//                      copied (TMA) into shared memory; its pair words
//                      streamed twice -- per-(warp, tile) counts, then, with
//                      the per-warp offsets, each step's 32 pairs ranked in
//                      lane (= emission) order and the Gaussian ids written.
// Replaces emission (8 B / pair written) + 2 onesweep passes over the pairs
// (2 x 16 B / pair) + range detection (4 B / pair) by 4 B / pair written
// and read twice, 4 B / pair of output and 12 B / (chunk, tile) of tables.
// What did not work: a decoupled look-back over the 4346 tile digits per
// chunk in one kernel (320 us per config-3 view: the first wave's chunks all
// look back to chunk 0 together); walking the rects in the placement kernel
// itself, twice (154 us against 116 + 28 for the expansion; the placement is
// latency-bound on its loads, hence the bulk copies and the 8-step batches of
// pair words); 4-, 6-, 12- and 16-warp chunks (per-chunk overheads or
// occupancy); match_any on every step, even with the 8 steps' matches
// issued together (3.70 -> 4.43 ms per config-3 step: match_any is slow on
// sm_100a, the returning atomic + duplicate check needs it on ~1 step in 4).  The sorted tile keys are not written (the ranges imply them).
#ifndef GS_ET_WARPS
#define GS_ET_WARPS 8  // warps per chunk (A/B knob)
#endif
#ifndef GS_ET_MINB
#define GS_ET_MINB 2  // resident placement CTAs per SM the registers are budgeted for
#endif
constexpr int ET_WARPS = GS_ET_WARPS;
#ifndef GS_ET_ROUNDS
#define GS_ET_ROUNDS 8
#endif
constexpr int ET_ROUNDS = GS_ET_ROUNDS;  // 32-Gaussian rounds per warp (u16 counts and offsets)
constexpr int ET_THREADS = ET_WARPS * 32;
constexpr int ET_CHUNK = ET_THREADS * ET_ROUNDS;  // Gaussians per chunk (2048: u16 chunk counts, 11-bit locals)
constexpr int ES_WARPS = 32;                      // chunk segments of the column sums

// row stride (tiles) of the per-(chunk, tile) tables and the shared tables: a
// multiple of 8, so every u16 and u32 row starts 16-byte aligned (bulk copies)
__host__ __device__ inline int et_stride(int n_tiles) { return (n_tiles + 7) & ~7; }
// placement shared memory: per-warp u16 offsets + the bases + the chunk's Gaussian ids
size_t emit_tiles_smem(int n_tiles) {
    return (size_t)ET_WARPS * et_stride(n_tiles) * 2 + (size_t)et_stride(n_tiles) * 4 + (size_t)ET_CHUNK * 4;
}
bool emit_tiles_fits(int n_tiles) { return n_tiles >= 1 && emit_tiles_smem(n_tiles) <= 200 * 1024; }  // <= 9856 tiles
// tables: u32 bases [chunk][tile], u16 counts [chunk][tile], u32 segment sums
// [32][tile], u32 per-(chunk, warp) pair offsets
struct EtTables {
    uint32_t* bases;
    unsigned short* counts;
    uint32_t* segs;
    uint32_t* wbases;
};
static size_t et_chunks(int64_t n) {
    const int64_t c = (n + ET_CHUNK - 1) / ET_CHUNK;
    return (size_t)(c > 0 ? c : 1);
}
static size_t et_layout(int64_t n, int n_tiles, char* table, EtTables* t) {
    const size_t hs = (size_t)et_stride(n_tiles), C = et_chunks(n);
    const size_t o_counts = C * hs * 4, o_segs = o_counts + C * hs * 2, o_wb = o_segs + ES_WARPS * hs * 4;
    const size_t total = o_wb + (C * (ET_WARPS + 1) * 4 + 15) / 16 * 16;
    if (t) {
        t->bases = reinterpret_cast<uint32_t*>(table);
        t->counts = reinterpret_cast<unsigned short*>(table + o_counts);
        t->segs = reinterpret_cast<uint32_t*>(table + o_segs);
        t->wbases = reinterpret_cast<uint32_t*>(table + o_wb);
    }
    return total;
}
size_t emit_tiles_table_bytes(int64_t n, int n_tiles) { return et_layout(n, n_tiles, nullptr, nullptr); }

// The chunk's Gaussians (depth-order positions p0 + 32 r, one per lane and
// round) and their tile rects; rounds past the visible count are empty.
struct EtRound {
    uint32_t g;
    int tx0, ty0, w, h;
};
__device__ __forceinline__ void et_load(const uint32_t* __restrict__ order, const float4* __restrict__ xydr, int p0,
                                        int V, int tiles_x, int tiles_y, EtRound (&rd)[ET_ROUNDS]) {
#pragma unroll
    for (int r = 0; r < ET_ROUNDS; ++r) rd[r].g = p0 + 32 * r < V ? order[p0 + 32 * r] : 0xFFFFFFFFu;
#pragma unroll
    for (int r = 0; r < ET_ROUNDS; ++r) {
        int tx0 = 0, tx1 = -1, ty0 = 0, ty1 = -1;
        if (rd[r].g != 0xFFFFFFFFu) {
            const float4 q = xydr[rd[r].g];
            tile_rect(q.x, q.y, __float_as_int(q.w), tiles_x, tiles_y, tx0, tx1, ty0, ty1);
        }
        rd[r].tx0 = tx0, rd[r].ty0 = ty0, rd[r].w = tx1 - tx0 + 1, rd[r].h = ty1 - ty0 + 1;
    }
}

// Walk the pairs of one round's 32 Gaussians in emission order, 32 per step:
// f(tile or 0xFFFFFFFF, gaussian).  Empty rects may only trail the non-empty
// ones (the depth order holds visible Gaussians only; rounds past the visible
// count are empty).  The owner of step lane j is the owner of the step's
// first pair (the last lane whose segment starts at or before it: one
// ballot) plus the segments starting inside the step up to j (a bit mask of
// the in-step start positions, one warp OR-reduction): ~35 instructions per
// step instead of a 5-level binary search over the lanes' offsets (80).
template <typename F>
__device__ __forceinline__ void et_walk(int lane, const EtRound& rd, int tiles_x, F&& f) {
    const uint32_t cnt = (uint32_t)(rd.w * rd.h);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - cnt, total = __shfl_sync(0xffffffffu, incl, 31);
    const float rw = rd.w > 0 ? 1.f / (float)rd.w : 0.f;
    const int tb = rd.ty0 * tiles_x + rd.tx0;  // the tile of the lane's first pair
    const uint32_t le = lanemask_lt() | (1u << lane);
    for (uint32_t t0 = 0; t0 < total; t0 += 32) {
        const uint32_t first = __ballot_sync(0xffffffffu, cnt != 0u && excl <= t0);
        const uint32_t sp = excl - t0;  // start position in the step (when inside)
        const uint32_t starts = __reduce_or_sync(0xffffffffu, (cnt != 0u && excl > t0 && sp < 32u) ? 1u << sp : 0u);
        const int L = (31 - __clz((int)first)) + __popc(starts & le);
        const uint32_t t = t0 + lane;
        const int j = (int)(t - __shfl_sync(0xffffffffu, excl, L));
        const int ow = __shfl_sync(0xffffffffu, rd.w, L);
        const float orw = __shfl_sync(0xffffffffu, rw, L);
        const int otb = __shfl_sync(0xffffffffu, tb, L);
        const uint32_t og = __shfl_sync(0xffffffffu, rd.g, L);
        int row = (int)((float)j * orw);
        if (row * ow > j) --row;
        if ((row + 1) * ow <= j) ++row;
        f(t < total ? (uint32_t)(otb + row * (tiles_x - ow) + j) : 0xFFFFFFFFu, og, t, L);
    }
}

// Every tile of the lane's own rect, row-major (order-free uses: counts).
// Divergent, so a warp runs as long as its largest rect, but ~5 instructions
// per tile against the walk's ~45 per step of 32.
// depth-first frame: meta[7] visible Gaussians sorted, in order_alt after an odd pass count (meta[8])
__device__ __forceinline__ const uint32_t* et_order(const uint32_t* order, const uint32_t* order_alt,
                                                    const unsigned long long* meta) {
    return (meta[8] & 1ull) ? order_alt : order;
}

// Expansion: the chunk's pairs walked once, in emission order, and written
// out as (chunk-local Gaussian index << 16 | tile) words -- every warp's
// pairs contiguous at a global offset obtained by a decoupled look-back over
// the chunks' pair totals (one status word per chunk, chunks taken in order
// from a counter) -- together with the chunk's per-tile counts.
__global__ void __launch_bounds__(ET_THREADS) et_expand_kernel(
    const uint32_t* __restrict__ order, const uint32_t* __restrict__ order_alt, const float4* __restrict__ xydr,
    int n, int tiles_x, int tiles_y, int64_t capacity, unsigned short* __restrict__ counts,
    uint32_t* __restrict__ pairs, uint32_t* __restrict__ wbases, unsigned int* __restrict__ chunk_counter,
    unsigned long long* __restrict__ status, const unsigned long long* __restrict__ meta) {
    griddep_wait();
    const int V = min(n, (int)meta[7]);
    order = et_order(order, order_alt, meta);
    const int n_tiles = tiles_x * tiles_y, hs = et_stride(n_tiles);
    const int n_chunks = (V + ET_CHUNK - 1) / ET_CHUNK;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem);  // [tile] (u32: shared atomics)
    __shared__ unsigned int s_chunk;
    __shared__ uint32_t s_wt[ET_WARPS];
    __shared__ unsigned long long s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_chunk = atomicAdd(chunk_counter, 1u);  // chunks in launch order: look-back progress
    for (int t = tid; t < hs; t += ET_THREADS) s_cnt[t] = 0u;
    __syncthreads();
    const int chunk = (int)s_chunk;
    if (chunk >= n_chunks) return;
    EtRound rd[ET_ROUNDS];
    et_load(order, xydr, chunk * ET_CHUNK + warp * (32 * ET_ROUNDS) + lane, V, tiles_x, tiles_y, rd);
    uint32_t rtot[ET_ROUNDS], wsum = 0;  // pairs per round of this warp, and in all
#pragma unroll
    for (int r = 0; r < ET_ROUNDS; ++r) {
        rtot[r] = __reduce_add_sync(0xffffffffu, (uint32_t)(rd[r].w * rd[r].h));
        wsum += rtot[r];
    }
    if (lane == 0) s_wt[warp] = wsum;
    __syncthreads();
    if (warp == 0) {  // the chunk's global pair offset: decoupled look-back over the chunks' totals
        unsigned long long agg = 0;
        for (int w = 0; w < ET_WARPS; ++w) agg += s_wt[w];
        unsigned long long prefix = 0;
        if (chunk == 0) {
            if (lane == 0) st_volatile(&status[0], FLAG_PRE | agg);
        } else {
            if (lane == 0) st_volatile(&status[chunk], FLAG_AGG | agg);
            // warp-wide: lane l reads predecessor q - l; the nearest inclusive
            // prefix (PRE) ends the window, the aggregates up to it are summed
            int q = chunk - 1;
            while (true) {
                const int pq = q - lane;
                unsigned long long sv = pq >= 0 ? ld_volatile(&status[pq]) : FLAG_PRE;
                while (__any_sync(0xffffffffu, (sv & ~VAL_MASK) == 0)) {
                    if ((sv & ~VAL_MASK) == 0) sv = ld_volatile(&status[pq]);
                }
                const uint32_t pre = __ballot_sync(0xffffffffu, (sv & ~VAL_MASK) == FLAG_PRE);
                const int stop = pre ? __ffs(pre) - 1 : 32;  // lanes [0, stop] count
                unsigned long long v = lane <= stop ? (sv & VAL_MASK) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                prefix += v;
                if (pre) break;
                q -= 32;
            }
            if (lane == 0) st_volatile(&status[chunk], FLAG_PRE | (prefix + agg));
        }
        if (lane == 0) s_base = prefix;
        if (lane == 0) {
            unsigned long long b = prefix;
            for (int w = 0; w < ET_WARPS; ++w) {
                wbases[(size_t)chunk * (ET_WARPS + 1) + w] = (uint32_t)b;
                b += s_wt[w];
            }
            wbases[(size_t)chunk * (ET_WARPS + 1) + ET_WARPS] = (uint32_t)b;
        }
    }
    __syncthreads();
    unsigned long long out = s_base;
    for (int w = 0; w < warp; ++w) out += s_wt[w];
#pragma unroll
    for (int r = 0; r < ET_ROUNDS; ++r) {
        const uint32_t loc0 = (uint32_t)(warp * (32 * ET_ROUNDS) + 32 * r) << 16;  // the round's first local index
        et_walk(lane, rd[r], tiles_x, [&](uint32_t tile, uint32_t, uint32_t t, int L) {
            if (tile != 0xFFFFFFFFu) {
                atomicAdd(&s_cnt[tile], 1u);
                const unsigned long long pos = out + t;
                if ((int64_t)pos < capacity) pairs[pos] = (loc0 + ((uint32_t)L << 16)) | tile;
            }
        });
        out += rtot[r];
    }
    __syncthreads();
    uint32_t* row = reinterpret_cast<uint32_t*>(counts + (size_t)chunk * hs);  // two u16 per word
    for (int k = tid; k < hs / 2; k += ET_THREADS) row[k] = s_cnt[2 * k] | (s_cnt[2 * k + 1] << 16);
}

// One CTA per 32 tiles (lane = tile), 32 warps over consecutive runs of
// chunks: each warp's column sums (segs) and the tiles' totals (tcount).
__global__ void __launch_bounds__(ES_WARPS * 32) et_colsum_kernel(const unsigned short* __restrict__ counts,
                                                                  uint32_t* __restrict__ segs, int n, int n_tiles,
                                                                  uint32_t* __restrict__ totals,
                                                                  const unsigned long long* __restrict__ meta) {
    griddep_wait();
    const int V = min(n, (int)meta[7]);
    const int chunks = (V + ET_CHUNK - 1) / ET_CHUNK;
    const int hs = et_stride(n_tiles);
    __shared__ uint32_t s_sum[ES_WARPS][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    const bool in = t < n_tiles;
    const int per = (chunks + ES_WARPS - 1) / ES_WARPS;
    const int c0 = min(chunks, warp * per), c1 = min(chunks, c0 + per);
    uint32_t sum = 0;
    if (in) {
        int c = c0;
        for (; c + 8 <= c1; c += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = counts[(size_t)(c + u) * hs + t];
#pragma unroll
            for (int u = 0; u < 8; ++u) sum += v[u];
        }
        for (; c < c1; ++c) sum += counts[(size_t)c * hs + t];
        segs[(size_t)warp * hs + t] = sum;
    }
    s_sum[warp][lane] = sum;
    __syncthreads();
    if (warp == 0 && in) {
        uint32_t tot = 0;
        for (int w = 0; w < ES_WARPS; ++w) tot += s_sum[w][lane];
        totals[t] = tot;
    }
}

// The same CTAs after the tile scan (tcount = every tile's start): per
// (chunk, tile) the absolute slot of the chunk's first pair of the tile,
// start + the column sums of the earlier segments + the running sum.
__global__ void __launch_bounds__(ES_WARPS * 32) et_colscan_kernel(const unsigned short* __restrict__ counts,
                                                                   const uint32_t* __restrict__ segs,
                                                                   const uint32_t* __restrict__ starts,
                                                                   uint32_t* __restrict__ bases, int n, int n_tiles,
                                                                   int64_t capacity,
                                                                   const unsigned long long* __restrict__ meta) {
    griddep_wait();
    if ((int64_t)meta[1] > capacity) return;  // over capacity: nothing is placed
    const int V = min(n, (int)meta[7]);
    const int chunks = (V + ET_CHUNK - 1) / ET_CHUNK;
    const int hs = et_stride(n_tiles);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    if (t >= n_tiles) return;
    const int per = (chunks + ES_WARPS - 1) / ES_WARPS;
    const int c0 = min(chunks, warp * per), c1 = min(chunks, c0 + per);
    uint32_t run = starts[t];
    for (int w = 0; w < warp; ++w) run += segs[(size_t)w * hs + t];
    int c = c0;
    for (; c + 8 <= c1; c += 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = counts[(size_t)(c + u) * hs + t];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            bases[(size_t)(c + u) * hs + t] = run;
            run += v[u];
        }
    }
    for (; c < c1; ++c) {
        const uint32_t v = counts[(size_t)c * hs + t];
        bases[(size_t)c * hs + t] = run;
        run += v;
    }
}

// 1D bulk (TMA) copy global -> shared completing on an mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

// Placement (see the section head).  Over capacity (meta[1]) nothing is
// written and the host re-runs with more room.
__global__ void __launch_bounds__(ET_THREADS, GS_ET_MINB) et_place_kernel(
    const uint32_t* __restrict__ order, const uint32_t* __restrict__ order_alt, int n, int n_tiles,
    int64_t capacity, const uint32_t* __restrict__ bases, const uint32_t* __restrict__ pairs,
    const uint32_t* __restrict__ wbases, uint32_t* __restrict__ vals, const unsigned long long* __restrict__ meta) {
    griddep_wait();
    if ((int64_t)meta[1] > capacity) return;
    const int V = min(n, (int)meta[7]);
    const int chunk = blockIdx.x;
    if (chunk * ET_CHUNK >= V) return;
    order = et_order(order, order_alt, meta);
    const int hs = et_stride(n_tiles);
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned short* s_hist = reinterpret_cast<unsigned short*>(smem);                // [warp][tile]
    uint32_t* s_base = reinterpret_cast<uint32_t*>(smem + (size_t)ET_WARPS * hs * 2);  // [tile]
    uint32_t* s_gid = s_base + hs;                                                    // [local Gaussian]
    __shared__ __align__(8) uint64_t s_bar;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {  // the chunk's row of bases and its Gaussian ids, by the bulk-copy engine
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t row = (uint32_t)hs * 4, ids = (uint32_t)ET_CHUNK * 4;
        mbar_expect_tx(&s_bar, row + ids);
        bulk_g2s(s_base, bases + (size_t)chunk * hs, row, &s_bar);
        bulk_g2s(s_gid, order + (size_t)chunk * ET_CHUNK, ids, &s_bar);  // (ids past V are never referenced)
    }
    {
        uint4* z = reinterpret_cast<uint4*>(smem);
        const int n16 = (ET_WARPS * hs * 2 + 15) / 16;
        for (int k = tid; k < n16; k += ET_THREADS) z[k] = make_uint4(0u, 0u, 0u, 0u);
    }
    const uint32_t wb = wbases[(size_t)chunk * (ET_WARPS + 1) + warp];
    const uint32_t we = min(wbases[(size_t)chunk * (ET_WARPS + 1) + warp + 1], (uint32_t)capacity);
    __syncthreads();
    // 1. per-(warp, tile) pair counts (PF steps of 32 pair words in flight)
    constexpr int PF = 8;
    uint32_t* h32 = reinterpret_cast<uint32_t*>(s_hist + warp * hs);
    for (uint32_t p0 = wb; p0 < we; p0 += 32 * PF) {
        uint32_t wv[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const uint32_t p = p0 + 32 * u + lane;
            wv[u] = p < we ? pairs[p] : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const uint32_t tile = wv[u] & 0xFFFFu;
            if (wv[u] != 0xFFFFFFFFu) atomicAdd(&h32[tile >> 1], 1u << ((tile & 1u) * 16));
        }
    }
    __syncthreads();
    // 2. per tile: exclusive offsets over the warps
    for (int t = tid; t < n_tiles; t += ET_THREADS) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < ET_WARPS; ++w) {
            const uint32_t c = s_hist[w * hs + t];
            s_hist[w * hs + t] = (unsigned short)run;
            run += c;
        }
    }
    mbar_wait(&s_bar, 0);
    __syncthreads();
    // 3. the pairs again, in order (PF steps at a time).  Each pair takes its
    //    warp's offset of its tile with a returning shared atomic; when no two
    //    lanes of the step share a tile (after - old == 1 everywhere) that is
    //    its slot, otherwise the lanes of each shared tile re-rank in lane
    //    order over the group's range [after - k, after) (match_any)
    const uint32_t lt = lanemask_lt();
    for (uint32_t q0 = wb; q0 < we; q0 += 32 * PF) {
        uint32_t wv[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const uint32_t p = q0 + 32 * u + lane;
            wv[u] = p < we ? pairs[p] : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            if (q0 + 32 * u >= we) break;  // (warp-uniform)
            const bool valid = wv[u] != 0xFFFFFFFFu;
            uint32_t tile = 0xFFFFFFFFu, og = 0u, sh = 0u, old = 0u, base = 0u;
            if (valid) {
                tile = wv[u] & 0xFFFFu;
                og = s_gid[wv[u] >> 16];
                sh = (tile & 1u) * 16;
                base = s_base[tile];
                old = (atomicAdd(&h32[tile >> 1], 1u << sh) >> sh) & 0xFFFFu;
            }
            __syncwarp();
            const uint32_t after = valid ? (h32[tile >> 1] >> sh) & 0xFFFFu : 0u;
            if (__any_sync(0xffffffffu, after - old > 1u)) {
                const uint32_t peers = __match_any_sync(0xffffffffu, tile);
                old = after - (uint32_t)__popc(peers) + (uint32_t)__popc(peers & lt);
            }
            if (valid) vals[base + old] = og;
            __syncwarp();  // the next step's atomics after every lane's read
        }
    }
}

static int et_attr(const void* k, size_t smem, size_t& done) {
    if (smem > 48 * 1024 && smem > done) {
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return check_launch("emit_tiles smem attribute");
        done = smem;
    }
    return 0;
}

int launch_emit_tiles_count(const uint32_t* order, const uint32_t* order_alt, const float* xydr4, int64_t n,
                            int tiles_x, int tiles_y, int64_t capacity, void* table, uint32_t* totals,
                            uint32_t* pairs, void* scan_ws, const unsigned long long* meta, cudaStream_t s) {
    const int n_tiles = tiles_x * tiles_y;
    if (!emit_tiles_fits(n_tiles)) return set_error("emit_tiles: %d tiles do not fit shared memory", n_tiles);
    if (n <= 0) return 0;
    EtTables tb;
    et_layout(n, n_tiles, static_cast<char*>(table), &tb);
    const int64_t chunks = (n + ET_CHUNK - 1) / ET_CHUNK;  // capacity-sized grids: fewer visible -> early exit
    const size_t smem_x = (size_t)et_stride(n_tiles) * 4;
    static size_t done_x = 0;
    if (et_attr((const void*)et_expand_kernel, smem_x, done_x)) return -1;
    launch_k(et_expand_kernel, dim3((unsigned)chunks), dim3(ET_THREADS), smem_x, s, order, order_alt,
             (const float4*)xydr4, (int)n, tiles_x, tiles_y, capacity, tb.counts, pairs, tb.wbases,
             (unsigned int*)scan_ws, (unsigned long long*)((char*)scan_ws + 16), meta);
    if (check_launch("et_expand_kernel")) return -1;
    launch_k(et_colsum_kernel, dim3((unsigned)((n_tiles + 31) / 32)), dim3(ES_WARPS * 32), 0, s,
             (const unsigned short*)tb.counts, tb.segs, (int)n, n_tiles, totals, meta);
    return check_launch("et_colsum_kernel");
}

int launch_emit_tiles(const uint32_t* order, const uint32_t* order_alt, int64_t n, int tiles_x, int tiles_y,
                      int64_t capacity, const uint32_t* starts, void* table, const uint32_t* pairs, uint32_t* vals,
                      const unsigned long long* meta, cudaStream_t s) {
    const int n_tiles = tiles_x * tiles_y;
    if (!emit_tiles_fits(n_tiles)) return set_error("emit_tiles: %d tiles do not fit shared memory", n_tiles);
    if (n <= 0) return 0;
    EtTables tb;
    et_layout(n, n_tiles, static_cast<char*>(table), &tb);
    launch_k(et_colscan_kernel, dim3((unsigned)((n_tiles + 31) / 32)), dim3(ES_WARPS * 32), 0, s,
             (const unsigned short*)tb.counts, (const uint32_t*)tb.segs, starts, tb.bases, (int)n, n_tiles, capacity,
             meta);
    if (check_launch("et_colscan_kernel")) return -1;
    const int64_t chunks = (n + ET_CHUNK - 1) / ET_CHUNK;
    const size_t smem_p = emit_tiles_smem(n_tiles);
    static size_t done_p = 0;
    if (et_attr((const void*)et_place_kernel, smem_p, done_p)) return -1;
    launch_k(et_place_kernel, dim3((unsigned)chunks), dim3(ET_THREADS), smem_p, s, order, order_alt, (int)n, n_tiles,
             capacity, (const uint32_t*)tb.bases, pairs, (const uint32_t*)tb.wbases, vals, meta);
    return check_launch("et_place_kernel");
}

// ---------------------------------------------------------------- scatter binning
// Small scenes (frame.cu): the projection counts every tile's intersections
// (project_fwd_kernel<2>); one CTA scans those counts into the tile ranges
// and per-tile write cursors; every pair is then written straight into its
// tile's range through an atomic cursor -- no global sort by tile.  The
// order inside a range is arbitrary; segsort.cu sorts each range by
// (depth, source index) afterwards.

// One CTA of 1024 threads (n_tiles <= 65536): exclusive scan of the tile
// counts (TCOUNT_REPL replicas, summed) -> ranges and per-replica cursors
// (tcount is overwritten in place), total -> *total.  Warp w owns a
// contiguous chunk of tiles and walks it 32 tiles at a time (coalesced
// replica reads): one sweep for the chunk total, a block scan over the 32
// chunk totals, a second sweep that writes.  Over capacity: every range
// empty and every cursor at capacity (the scatter then writes nothing; the
// host reruns with more room).  order != nullptr: also the heaviest-first
// raster launch order (tile_order_kernel's bucketing).
template <int REPL>
__global__ void __launch_bounds__(1024) tile_scan_kernel(uint32_t* __restrict__ tcount, int n_tiles,
                                                         int64_t capacity, uint2* __restrict__ ranges,
                                                         unsigned long long* __restrict__ total,
                                                         uint32_t* __restrict__ order) {
    griddep_wait();
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_bucket[34];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int chunk = (((n_tiles + 31) >> 5) + 31) & ~31;  // tiles per warp, a multiple of 32
    const int c0 = warp * chunk, c1 = min(n_tiles, c0 + chunk);
    if (tid < 34) s_bucket[tid] = 0u;
    auto tile_count = [&](int t) {
        uint32_t c = 0;
#pragma unroll
        for (int r = 0; r < REPL; ++r) c += tcount[(size_t)r * n_tiles + t];
        return c;
    };
    uint32_t sum = 0;
    for (int t = c0 + lane; t < c1; t += 32) sum += tile_count(t);
    sum = __reduce_add_sync(0xffffffffu, sum);
    if (lane == 0) s_warp[warp] = sum;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = s_warp[lane];
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        s_warp[lane] = wi - w;  // exclusive chunk offsets
        if (lane == 31) {
            *total = (unsigned long long)wi;
            s_bucket[33] = wi;
        }
    }
    __syncthreads();
    const bool over = (int64_t)s_bucket[33] > capacity;
    uint32_t run = s_warp[warp];
    for (int tb = c0; tb < c1; tb += 32) {
        const int t = tb + lane;
        const bool in = t < c1;
        uint32_t cr[REPL], c = 0;
#pragma unroll
        for (int r = 0; r < REPL; ++r) {
            cr[r] = in ? tcount[(size_t)r * n_tiles + t] : 0u;
            c += cr[r];
        }
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t start = run + incl - c;
        run += __shfl_sync(0xffffffffu, incl, 31);
        if (in) {
            uint32_t cur = start;
#pragma unroll
            for (int r = 0; r < REPL; ++r) {  // replica r's cursor: the tile start + earlier replicas
                tcount[(size_t)r * n_tiles + t] = over ? (uint32_t)capacity : cur;
                cur += cr[r];
            }
            if (over) c = 0;
            ranges[t] = c ? make_uint2(start, start + c) : make_uint2(0u, 0u);  // empty tiles: (0, 0)
            if (order) atomicAdd(&s_bucket[__clz(c)], 1u);  // clz: 0 = longest bucket ... 32 = empty
        }
    }
    if (!order) return;
    __syncthreads();
    if (tid == 0) {
        uint32_t b_run = 0;
        for (int b = 0; b < 33; ++b) {
            const uint32_t c = s_bucket[b];
            s_bucket[b] = b_run;
            b_run += c;
        }
    }
    __syncthreads();
    for (int t = c0 + lane; t < c1; t += 32) {
        const uint2 r = ranges[t];  // this thread's own writes
        order[atomicAdd(&s_bucket[__clz(r.y - r.x)], 1u)] = (uint32_t)t;
    }
}

int launch_tile_scan(uint32_t* tcount, int n_tiles, int64_t capacity, uint2* ranges, unsigned long long* total,
                     uint32_t* order, cudaStream_t s, int replicas) {
    if (n_tiles <= 0 || n_tiles > 65536) return set_error("tile_scan: %d tiles out of range", n_tiles);
    if (replicas == 1)
        launch_k(tile_scan_kernel<1>, dim3(1), dim3(1024), 0, s, tcount, n_tiles, capacity, ranges, total, order);
    else
        launch_k(tile_scan_kernel<TCOUNT_REPL>, dim3(1), dim3(1024), 0, s, tcount, n_tiles, capacity, ranges, total,
                 order);
    return check_launch("tile_scan_kernel");
}

// Every visible Gaussian's (tile, gaussian) pairs into the tiles' ranges
// through the atomic cursors; warps walk 32 Gaussians' rects together,
// SCATTER_UNROLL cursor atomics in flight per lane.
#ifndef SCATTER_UNROLL
#define SCATTER_UNROLL 4
#endif
__global__ void __launch_bounds__(256) scatter_pairs_kernel(const float4* __restrict__ xydr,
                                                            const uint32_t* __restrict__ counts, int n, int tiles_x,
                                                            int tiles_y, uint32_t capacity,
                                                            uint32_t* __restrict__ cursors,
                                                            uint32_t* __restrict__ tile_keys,
                                                            uint32_t* __restrict__ vals) {
    griddep_wait();
    const int n_round = (n + 31) & ~31;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += gridDim.x * blockDim.x) {
        int tx0 = 0, tx1 = -1, ty0 = 0, ty1 = -1;
        if (i < n && counts[i]) {
            const float4 g = xydr[i];
            tile_rect(g.x, g.y, __float_as_int(g.w), tiles_x, tiles_y, tx0, tx1, ty0, ty1);
        }
        uint32_t* cur = cursors + (size_t)tcount_replica((uint32_t)i) * (tiles_x * tiles_y);
        walk_tile_rects<SCATTER_UNROLL>(threadIdx.x & 31, (uint32_t)i, tx0, tx1, ty0, ty1, tiles_x,
                           [&](const uint32_t* tl, const uint32_t* gl) {
                               uint32_t slot[SCATTER_UNROLL];
#pragma unroll
                               for (int u = 0; u < SCATTER_UNROLL; ++u)
                                   slot[u] = tl[u] != 0xFFFFFFFFu ? atomicAdd(&cur[tl[u]], 1u) : capacity;
#pragma unroll
                               for (int u = 0; u < SCATTER_UNROLL; ++u)
                                   if (slot[u] < capacity) {
                                       tile_keys[slot[u]] = tl[u];
                                       vals[slot[u]] = gl[u];
                                   }
                           });
    }
}

int launch_scatter_pairs(const float* xydr4, const uint32_t* counts, int64_t n, int tiles_x, int tiles_y,
                         int64_t capacity, uint32_t* cursors, uint32_t* tile_keys, uint32_t* vals, cudaStream_t s) {
    int64_t blocks = (n + 255) / 256;
    const int64_t cap = (int64_t)sort_sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) return 0;
    launch_k(scatter_pairs_kernel, dim3((unsigned)blocks), dim3(256), 0, s, (const float4*)xydr4, counts, (int)n,
             tiles_x, tiles_y, (uint32_t)capacity, cursors, tile_keys, vals);
    return check_launch("scatter_pairs_kernel");
}

// Raster launch order: heaviest tile lists first, so the rasterizers' last
// CTAs are short ones (uneven scenes otherwise end on a few long tiles).
// Tiles are bucketed by floor(log2(list length)), buckets descending; order
// within a bucket is arbitrary.  One CTA (n_tiles <= 65536).
__global__ void __launch_bounds__(1024) tile_order_kernel(const uint2* __restrict__ ranges, int n_tiles,
                                                          uint32_t* __restrict__ order) {
    griddep_wait();
    __shared__ uint32_t s_cnt[34];
    if (threadIdx.x < 34) s_cnt[threadIdx.x] = 0u;
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
        const uint2 r = ranges[t];
        const uint32_t len = r.y - r.x;
        atomicAdd(&s_cnt[__clz(len)], 1u);  // clz: 0 = longest bucket ... 32 = empty
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int b = 0; b < 33; ++b) {
            const uint32_t c = s_cnt[b];
            s_cnt[b] = run;
            run += c;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
        const uint2 r = ranges[t];
        order[atomicAdd(&s_cnt[__clz(r.y - r.x)], 1u)] = (uint32_t)t;
    }
}

int launch_tile_order(const uint2* ranges, int n_tiles, uint32_t* order, cudaStream_t s) {
    if (n_tiles <= 0) return 0;
    launch_k(tile_order_kernel, dim3(1), dim3(1024), 0, s, ranges, n_tiles, order);
    return check_launch("tile_order_kernel");
}

__global__ void __launch_bounds__(256) ranges_u32_kernel(const uint32_t* __restrict__ keys, int64_t n_cap,
                                                         const unsigned long long* __restrict__ n_dev,
                                                         uint2* __restrict__ ranges) {
    griddep_wait();
    // 4 sorted keys per thread (one 16-byte load when aligned and in range)
    const int64_t n = n_dev ? min((int64_t)*n_dev, n_cap) : n_cap;
    const int64_t i0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (i0 >= n) return;
    uint32_t k[4];
    if (i0 + 4 <= n) {
        const uint4 v = *reinterpret_cast<const uint4*>(keys + i0);
        k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) k[j] = i0 + j < n ? keys[i0 + j] : 0xFFFFFFFFu;
    }
    uint32_t prev = i0 > 0 ? keys[i0 - 1] : 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t i = i0 + j;
        if (i >= n) break;
        const uint32_t t = k[j];
        if (i == 0 || prev != t) ranges[t].x = (uint32_t)i;
        const uint32_t next = j < 3 ? (i + 1 < n ? k[j + 1] : 0xFFFFFFFFu) : (i + 1 < n ? keys[i + 1] : 0xFFFFFFFFu);
        if (i == n - 1 || next != t) ranges[t].y = (uint32_t)(i + 1);
        prev = t;
    }
}

size_t scan_ws_bytes(int64_t n) {
    const int64_t ctas = (n + SCAN_TILE - 1) / SCAN_TILE;
    return 16 + (size_t)(ctas > 0 ? ctas : 1) * sizeof(unsigned long long);
}

int launch_scan(const uint32_t* in, const uint32_t* gather, uint32_t* out, int64_t n, void* ws,
                unsigned long long* total, cudaStream_t s) {
    if (n == 0) return 0;
    const int64_t ctas = (n + SCAN_TILE - 1) / SCAN_TILE;
    launch_k(scan_kernel, dim3((unsigned)ctas), dim3(SCAN_THREADS), 0, s, in, gather, out, n, (unsigned int*)ws,
                                                       (unsigned long long*)((char*)ws + 16), total);
    return check_launch("scan_kernel");
}

int launch_emit_sorted(const uint32_t* order, const float* xydr4, const uint32_t* offsets, int64_t n, int tiles_x,
                       int tiles_y, int64_t capacity, uint32_t* tile_keys, uint32_t* vals, uint32_t* tile_hist,
                       int tile_passes, cudaStream_t s) {
    if (n == 0) return 0;
    int64_t blocks = (n + 255) / 256;
    const int64_t cap = (int64_t)sort_sm_count() * 8;  // resident CTAs
    if (blocks > cap) blocks = cap;
    launch_k(emit_sorted_kernel, dim3((unsigned)blocks), dim3(256), 0, s, order, (const float4*)xydr4, offsets, (int)n,
                                                                  tiles_x, tiles_y, capacity, tile_keys, vals,
                                                                  tile_hist, tile_passes);
    return check_launch("emit_sorted_kernel");
}

int launch_ranges_u64(const unsigned long long* sorted_keys, int64_t n, uint2* ranges, cudaStream_t s) {
    if (n == 0) return 0;
    ranges_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sorted_keys, n, ranges);
    return check_launch("ranges_kernel");
}

int launch_ranges_u32(const uint32_t* sorted_tile_keys, int64_t n_cap, const unsigned long long* n_dev,
                      uint2* ranges, cudaStream_t s) {
    if (n_cap == 0) return 0;
    launch_k(ranges_u32_kernel, dim3((unsigned)((n_cap + 1023) / 1024)), dim3(256), 0, s, sorted_tile_keys, n_cap,
             n_dev, ranges);
    return check_launch("ranges_u32_kernel");
}

}  // namespace gs

using namespace gs;

extern "C" {

size_t gs_scan_workspace_bytes(int64_t n) {
    const int64_t ctas = (n + SCAN_TILE - 1) / SCAN_TILE;
    return 16 + (size_t)(ctas > 0 ? ctas : 1) * sizeof(unsigned long long);
}

int gs_scan_tiles(const uint32_t* tiles, uint32_t* offsets, int64_t n, void* ws, size_t ws_bytes,
                  unsigned long long* total, gs_stream_t stream) {
    if (n < 0) return set_error("gs_scan_tiles: negative n");
    if (ws_bytes < gs_scan_workspace_bytes(n)) return set_error("gs_scan_tiles: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        if (cudaMemsetAsync(total, 0, sizeof(unsigned long long), s) != cudaSuccess)
            return check_launch("gs_scan_tiles memset");
        return 0;
    }
    const int64_t ctas = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (cudaMemsetAsync(ws, 0, gs_scan_workspace_bytes(n), s) != cudaSuccess) return check_launch("scan memset");
    unsigned int* counter = (unsigned int*)ws;
    unsigned long long* status = (unsigned long long*)((char*)ws + 16);
    scan_kernel<<<(unsigned)ctas, SCAN_THREADS, 0, s>>>(tiles, nullptr, offsets, n, counter, status, total);
    return check_launch("scan_kernel");
}

int gs_emit_keys(const float* xydr4, const uint32_t* offsets, const uint32_t* tiles, int64_t n, int32_t width,
                 int32_t height, unsigned long long* keys, uint32_t* vals, gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_emit_keys: n out of range");
    if (n == 0) return 0;
    const int tiles_x = (width + TILE - 1) / TILE, tiles_y = (height + TILE - 1) / TILE;
    emit_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        (const float4*)xydr4, offsets, tiles, (int)n, tiles_x, tiles_y, keys, vals);
    return check_launch("emit_kernel");
}

int gs_tile_counts(const float* xydr4, int64_t n, int32_t width, int32_t height, uint32_t* out_tiles,
                   gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_tile_counts: n out of range");
    if (n == 0) return 0;
    const int tiles_x = (width + TILE - 1) / TILE, tiles_y = (height + TILE - 1) / TILE;
    tile_counts_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        (const float4*)xydr4, (int)n, tiles_x, tiles_y, out_tiles);
    return check_launch("tile_counts_kernel");
}

int gs_tile_ranges(const unsigned long long* sorted_keys, int64_t n, uint32_t* ranges2, int32_t n_tiles,
                   gs_stream_t stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(ranges2, 0, (size_t)n_tiles * 2 * sizeof(uint32_t), s) != cudaSuccess)
        return check_launch("ranges memset");
    if (n == 0) return 0;
    ranges_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sorted_keys, n, (uint2*)ranges2);
    return check_launch("ranges_kernel");
}

}  // extern "C"
