// sort.cu -- hand-written stable LSD radix sort of (key, uint32 value) pairs
// in the "onesweep" style: the digit histograms of every pass are produced
// up front (by sort_hist_kernel, or fused into the producer kernel), then
// one kernel per 8-bit pass ranks a tile of keys with per-warp peer masks,
// obtains the tile's global digit offsets through a decoupled look-back
// chained scan, and scatters through shared memory so the global writes are
// runs of consecutive addresses.
//
// Stability is what reproduces sg/binning.py:50-65's (depth, source_index)
// order: keys are emitted in Gaussian-index order, equal keys keep it.
// Keys: uint32 (depth-first binning, frame.cu) or uint64 (the general
// (tile << 32 | depth bits) C-ABI sort, gs_sort_pairs).
#include <cstdlib>

#include "common.cuh"
#include "internal.cuh"

// decoupled look-back window (status loads in flight per round trip; 4 beat
// 1, 8 and 16 at configs 2 and 4)
#ifndef GS_SORT_LB
#define GS_SORT_LB 4
#endif

namespace gs {

constexpr int SORT_THREADS = 256;
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr int RADIX = 256;
constexpr int MAX_PASSES = 8;
constexpr uint32_t ST_AGG = 1u << 30;
constexpr uint32_t ST_PRE = 2u << 30;
constexpr uint32_t ST_MASK = (1u << 30) - 1;

// Items per thread: the large tile amortises the look-back for big inputs;
// the small one (4 items) gives 4x more CTAs when the input would otherwise
// fill less than two waves (latency-bound passes at N ~ 1e5).
template <typename K>
struct SortCfg;
template <>
struct SortCfg<uint32_t> {
    static constexpr int ITEMS = 16;
};
template <>
struct SortCfg<unsigned long long> {
    static constexpr int ITEMS = 15;
};
constexpr int SMALL_ITEMS = 4;

template <typename K, int ITEMS>
constexpr int sort_tile() { return SORT_THREADS * ITEMS; }

// The peer-mask banks (ranking) and the key / value staging (scatter) are
// live at different times: they share memory when the staging is the larger.
template <typename K, int ITEMS>
constexpr bool sort_peers_alias() {
    return (size_t)sort_tile<K, ITEMS>() * (sizeof(K) + 4) >= (size_t)SORT_WARPS * 2 * RADIX * 4;
}
template <typename K, int ITEMS>
constexpr size_t sort_smem() {
    return (size_t)sort_tile<K, ITEMS>() * (sizeof(K) + 4) + (size_t)SORT_WARPS * RADIX * 4 + 2 * RADIX * 4 +
           (sort_peers_alias<K, ITEMS>() ? 0 : (size_t)SORT_WARPS * 2 * RADIX * 4) +  // peer-mask banks (RANK_OR)
           RADIX * 4;                            // the next digit's histogram (depth sort)
}

// look-back status words: GPU-scope relaxed accesses (flag and value share
// one 32-bit word, so no further ordering is needed); volatile would make
// them system-scope
__device__ __forceinline__ uint32_t ldv(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void stv(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// shared-memory reductions / volatile loads through 32-bit shared addresses (the ranking loop)
__device__ __forceinline__ void red_shared_or(uint32_t a, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_shared_add(uint32_t a, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32v(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}

__device__ __forceinline__ int64_t resolve_n(const unsigned long long* n_dev, int64_t n_cap) {
    if (!n_dev) return n_cap;
    const int64_t v = (int64_t)*n_dev;
    return v < n_cap ? v : n_cap;
}

template <typename K>
__global__ void __launch_bounds__(256) sort_hist_kernel(const K* __restrict__ keys, int64_t n_cap,
                                                        const unsigned long long* __restrict__ n_dev, int passes,
                                                        uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[MAX_PASSES * RADIX];
    for (int k = threadIdx.x; k < passes * RADIX; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    const int64_t n = resolve_n(n_dev, n_cap);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_round = (n + 31) / 32 * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
        const bool valid = i < n;
        const K key = valid ? keys[i] : (K)0;
        for (int p = 0; p < passes; ++p)
            warp_hist_add(sh + p * RADIX, (uint32_t)((key >> (8 * p)) & (K)255), valid);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < passes * RADIX; k += blockDim.x) {
        const uint32_t v = sh[k];
        if (v) atomicAdd(&hist[k], v);
    }
}

// Inclusive scan over the 256 threads of the CTA (one value per thread).
__device__ __forceinline__ uint32_t block_incl_scan256(uint32_t v, uint32_t* s_tmp /*8*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_tmp[warp] = v;
    __syncthreads();
    uint32_t off = 0;
#pragma unroll
    for (int w = 0; w < SORT_WARPS; ++w)
        if (w < warp) off += s_tmp[w];
    __syncthreads();
    return v + off;
}

// One 8-bit pass.  vin == nullptr means value = input index (identity).
template <typename K, int ITEMS>
constexpr int sort_minb() {
#ifndef GS_SORT_MINB16
#define GS_SORT_MINB16 4  // 64 registers (a 12-byte spill): with the peer masks over the staging (43 KB of
                          // shared memory) 4 CTAs per SM -- config 3 depth sort 4.16 -> 3.75 ms per step
#endif
    if (sizeof(K) == 4 && ITEMS == 16) return GS_SORT_MINB16;
    return sizeof(K) == 4 ? (ITEMS <= 8 ? 5 : (ITEMS <= 12 ? 4 : (ITEMS <= 16 ? 3 : 2))) : 2;
}

// rel_min (uint32 keys, depth sort pass 0): keys are taken relative to
// *rel_min and 0xFFFFFFFF keys (culled Gaussians) are dropped -- the output
// holds only the valid items, in order.  npass_dev: the pass is skipped
// entirely when `pass` >= *npass_dev (the relative keys are narrower).
// The depth sort has no histogram kernel: pass 0's digit histogram is the
// projection's histogram of the visible keys' ABSOLUTE low byte, rotated by
// the minimum's low byte ((key - min) mod 256 = (key mod 256 - min mod 256)
// mod 256); pass 0 also writes the pass count (meta[8], from the key range
// meta[5..6] = rel_min[0..1]) and the visible count (meta[7] = the
// histogram's total), and every pass adds the next digit's histogram of its
// keys into next_hist (the passes are latency-bound: the extra shared
// atomics are nearly free).
template <typename K, int ITEMS, bool RANK_OR>
__global__ void __launch_bounds__(SORT_THREADS, (sort_minb<K, ITEMS>())) onesweep_kernel(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n_cap, const unsigned long long* __restrict__ n_dev, int shift,
    const uint32_t* __restrict__ hist, uint32_t* __restrict__ status, uint32_t* __restrict__ counter,
    const unsigned long long* __restrict__ rel_min, const unsigned long long* __restrict__ npass_dev, int pass,
    uint32_t* __restrict__ next_hist, unsigned long long* __restrict__ meta_out) {
    griddep_wait();
    if (npass_dev && pass >= (int)*npass_dev) return;
    constexpr int TILE_N = sort_tile<K, ITEMS>();
    extern __shared__ __align__(16) unsigned char smem[];
    K* s_keys = reinterpret_cast<K*>(smem);
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + TILE_N);
    uint32_t* s_whist = s_vals + TILE_N;               // [warp][digit]
    uint32_t* s_gbase = s_whist + SORT_WARPS * RADIX;  // global dst of local slot 0 per digit
    uint32_t* s_lstart = s_gbase + RADIX;              // local start of each digit in the tile
    constexpr bool ALIAS = sort_peers_alias<K, ITEMS>();
    // [warp][2][digit] peer masks (RANK_OR), over the staging when it is the larger
    uint32_t* s_peers = ALIAS ? reinterpret_cast<uint32_t*>(smem) : s_lstart + RADIX;
    uint32_t* s_next = ALIAS ? s_lstart + RADIX : s_peers + SORT_WARPS * 2 * RADIX;  // [digit] next digit's counts
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_tmp[SORT_WARPS];
    __shared__ uint32_t s_total;

    const int64_t n = resolve_n(n_dev, n_cap);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(counter, 1u);
#pragma unroll
    for (int k = 0; k < SORT_WARPS; ++k) s_whist[k * RADIX + tid] = 0;
    if (RANK_OR) {
#pragma unroll
        for (int k = 0; k < 2 * SORT_WARPS; ++k) s_peers[k * RADIX + tid] = 0;
    }
    if (next_hist) s_next[tid] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    if ((int64_t)tile * TILE_N >= n) return;  // capacity-sized grid, fewer items this frame
    const int64_t wbase = (int64_t)tile * TILE_N + (int64_t)warp * (ITEMS * 32);

    K key[ITEMS];
    uint32_t val[ITEMS];
    uint32_t rank[ITEMS];
    uint32_t okm = 0;  // valid items (bit i)
    const K kmin = rel_min ? (K)*rel_min : (K)0;
    constexpr uint32_t ALL_OK = ITEMS >= 32 ? 0xffffffffu : ((1u << ITEMS) - 1u);
    if (wbase + ITEMS * 32 <= n) {
        // a full warp slice (all but the last tile's): plain loads at constant offsets from one base
        const K* kp = kin + wbase + lane;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) key[i] = kp[i * 32];
        if (vin) {
            const uint32_t* vp = vin + wbase + lane;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) val[i] = vp[i * 32];
        } else {
            const uint32_t v0 = (uint32_t)(wbase + lane);
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) val[i] = v0 + (uint32_t)(i * 32);
        }
        okm = ALL_OK;
        if (rel_min) {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                if (key[i] == (K)0xFFFFFFFFu) okm &= ~(1u << i);
                key[i] -= kmin;
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int64_t idx = wbase + i * 32 + lane;
            key[i] = idx < n ? kin[idx] : (K)0;
            val[i] = idx < n ? (vin ? vin[idx] : (uint32_t)idx) : 0u;
            bool ok = idx < n;
            if (rel_min) {
                ok = ok && key[i] != (K)0xFFFFFFFFu;
                key[i] -= kmin;
            }
            okm |= ok ? (1u << i) : 0u;
        }
    }
    const bool warp_all_ok = __all_sync(0xffffffffu, okm == ALL_OK);
    if (next_hist) {  // the next pass's digit of this tile's keys
        const uint32_t next_w = smem_addr(s_next);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const bool valid = (okm >> i) & 1u;
            const uint32_t d4 = ((uint32_t)(key[i] >> (shift + 8)) & 255u) * 4u;
            int same;
            __match_all_sync(0xffffffffu, valid ? d4 : 0xffffffffu, &same);
            // one digit in the whole warp (typical for the high bytes): lane 0 adds 32
            if (valid && (!same || lane == 0)) red_shared_add(next_w + d4, same ? 32u : 1u);
        }
    }
    // warp-local stable ranking: items in (i, lane) order = input order
    const uint32_t lt = lanemask_lt();
    if (RANK_OR) {
        // peer masks built with shared atomic OR (two alternating mask
        // banks, so a bank is cleared while the other is being filled);
        // 32-bit shared addresses, and a predicate-free body when every item
        // of the warp is valid (all passes but the compacting first one)
        const uint32_t peer_w = smem_addr(s_peers + warp * 2 * RADIX);
        const uint32_t whist_w = smem_addr(s_whist + warp * RADIX);
        const uint32_t lbit = 1u << lane;
        if (warp_all_ok) {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const uint32_t d4 = ((uint32_t)(key[i] >> shift) & 255u) * 4u;
                const uint32_t pm = peer_w + (uint32_t)((i & 1) * RADIX * 4) + d4;
                const uint32_t wh = whist_w + d4;
                red_shared_or(pm, lbit);
                __syncwarp();
                const uint32_t peers = lds_u32v(pm);
                const uint32_t old = lds_u32v(wh);
                __syncwarp();
                if ((peers & lt) == 0) {  // lowest peer: bump the count, clear the mask
                    sts_u32(wh, old + (uint32_t)__popc(peers));
                    sts_u32(pm, 0u);
                }
                rank[i] = old + (uint32_t)__popc(peers & lt);
            }
        } else {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const bool valid = (okm >> i) & 1u;
                const uint32_t d4 = ((uint32_t)(key[i] >> shift) & 255u) * 4u;
                const uint32_t pm = peer_w + (uint32_t)((i & 1) * RADIX * 4) + d4;
                const uint32_t wh = whist_w + d4;
                if (valid) red_shared_or(pm, lbit);
                __syncwarp();
                const uint32_t peers = valid ? lds_u32v(pm) : 0u;
                const uint32_t old = valid ? lds_u32v(wh) : 0u;
                __syncwarp();
                if (valid && (peers & lt) == 0) {
                    sts_u32(wh, old + (uint32_t)__popc(peers));
                    sts_u32(pm, 0u);
                }
                rank[i] = old + (uint32_t)__popc(peers & lt);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const bool valid = (okm >> i) & 1u;
            const uint32_t d = valid ? (uint32_t)(key[i] >> shift) & 255u : 256u;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const int leader = __ffs(peers) - 1;
            uint32_t old = 0;
            if (valid && lane == leader) old = atomicAdd(&s_whist[warp * RADIX + d], (uint32_t)__popc(peers));
            old = __shfl_sync(0xffffffffu, old, leader);
            rank[i] = old + (uint32_t)__popc(peers & lt);
        }
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, tile total, chained scan
    const uint32_t d = (uint32_t)tid;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < SORT_WARPS; ++w) {
        const uint32_t c = s_whist[w * RADIX + d];
        s_whist[w * RADIX + d] = run;
        run += c;
    }
    uint32_t* st = status + (size_t)tile * RADIX + d;
    uint32_t excl = 0;
    if (tile == 0) {
        stv(st, ST_PRE | run);
    } else {
        stv(st, ST_AGG | run);
        // decoupled look-back over windows of LB predecessors: the LB status
        // loads of a window are in flight together (one L2 round trip per
        // window instead of per predecessor); a not-yet-posted entry is
        // re-polled in place
        constexpr int LB = GS_SORT_LB;
        int p = (int)tile - 1;
        bool found = false;
        while (!found) {
            uint32_t w[LB];
#pragma unroll
            for (int j = 0; j < LB; ++j) w[j] = p - j >= 0 ? ldv(status + (size_t)(p - j) * RADIX + d) : ST_PRE;
#pragma unroll
            for (int j = 0; j < LB; ++j) {
                if (!found) {
                    uint32_t v = w[j];
                    while ((v & ~ST_MASK) == 0) v = ldv(status + (size_t)(p - j) * RADIX + d);
                    excl += v & ST_MASK;
                    found = (v & ~ST_MASK) == ST_PRE;
                }
            }
            p -= LB;
        }
        stv(st, ST_PRE | (excl + run));
    }
    // depth sort pass 0: the projection's absolute low-byte histogram, rotated
    const uint32_t h = rel_min ? hist[(d + (uint32_t)*rel_min) & 255u] : hist[d];
    const uint32_t lincl = block_incl_scan256(run, s_tmp);
    const uint32_t hincl = block_incl_scan256(h, s_tmp);
    if (meta_out && tile == 0 && d == RADIX - 1) {  // visible count and pass count (read by the later kernels)
        const uint32_t kmin = (uint32_t)rel_min[0], kmax = (uint32_t)rel_min[1];
        const uint32_t range = kmin <= kmax ? kmax - kmin : 0u;
        meta_out[7] = (unsigned long long)hincl;
        meta_out[8] = (unsigned long long)(range == 0u ? 1 : (32 - __clz((int)range) + 7) / 8);
    }
    const uint32_t lstart = lincl - run;
    if (d == RADIX - 1) s_total = lincl;  // valid items of the tile
    s_lstart[d] = lstart;
    s_gbase[d] = (hincl - h) + excl - lstart;  // mod 2^32; dst = gbase + local slot
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        if ((okm >> i) & 1u) {
            const uint32_t dd = (uint32_t)(key[i] >> shift) & 255u;
            const uint32_t pos = s_lstart[dd] + s_whist[warp * RADIX + dd] + rank[i];
            s_keys[pos] = key[i];
            s_vals[pos] = val[i];
        }
    }
    __syncthreads();
    const int cnt = (int)s_total;
    for (int j = tid; j < cnt; j += SORT_THREADS) {
        const K k = s_keys[j];
        const uint32_t dd = (uint32_t)(k >> shift) & 255u;
        const uint32_t dst = s_gbase[dd] + (uint32_t)j;
        kout[dst] = k;
        vout[dst] = s_vals[j];
    }
    if (next_hist) {
        const uint32_t c = s_next[tid];  // (the scatter loop's barrier ordered the counts)
        if (c) atomicAdd(&next_hist[tid], c);
    }
}

template <typename K, int ITEMS, bool RANK_OR>
static int set_sort_attr() {
    static bool done = false;
    if (!done) {
        if (cudaFuncSetAttribute(onesweep_kernel<K, ITEMS, RANK_OR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sort_smem<K, ITEMS>()) != cudaSuccess)
            return check_launch("onesweep smem attribute");
        done = true;
    }
    return 0;
}

int sort_sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    return sms;
}

// Sized for the small tile (the most CTAs either variant can launch).
template <typename K>
size_t onesweep_status_bytes(int64_t n_cap, int passes) {
    const int64_t tiles = (n_cap + sort_tile<K, SMALL_ITEMS>() - 1) / sort_tile<K, SMALL_ITEMS>();
    return (size_t)passes * (size_t)(tiles > 0 ? tiles : 1) * RADIX * 4;
}
template size_t onesweep_status_bytes<uint32_t>(int64_t, int);
template size_t onesweep_status_bytes<unsigned long long>(int64_t, int);

// Runs `passes` onesweep passes from bit 0.  hist: passes x 256 digit counts
// (already accumulated), status: zeroed onesweep_status_bytes, counters:
// `passes` zeroed uint32.  identity_vals: the first pass ignores v0's
// contents and uses the input index as value (v0 is still the ping-pong
// scratch).  Result lands in (k1, v1) when passes is odd, else (k0, v0).
// Warp ranking flavour: shared atomic-OR peer masks (default) or match_any
// (GS_SORT_RANK=match).
static bool rank_or() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GS_SORT_RANK");
        v = (e && e[0] == 'm') ? 0 : 1;
    }
    return v == 1;
}

struct PassOpts {  // depth sort: pass 0 relative + compacting, later passes on the compacted count
    const unsigned long long* n_dev_rest = nullptr;
    const unsigned long long* rel_min0 = nullptr;
    const unsigned long long* npass_dev = nullptr;
    bool next_hist = false;             // every pass but the last adds the next digit's histogram
    unsigned long long* meta = nullptr;  // pass 0 writes meta[7] (visible) and meta[8] (passes)
};

template <typename K, int ITEMS, bool RANK_OR>
static int run_passes_t(K* k0, uint32_t* v0, K* k1, uint32_t* v1, int64_t n_cap, const unsigned long long* n_dev,
                        int passes, const uint32_t* hist, uint32_t* status, uint32_t* counters, cudaStream_t s,
                        bool identity_vals, const PassOpts& po = PassOpts()) {
    if (set_sort_attr<K, ITEMS, RANK_OR>()) return -1;
    const int64_t tiles = (n_cap + sort_tile<K, ITEMS>() - 1) / sort_tile<K, ITEMS>();
    K* kin = k0;
    K* kout = k1;
    uint32_t* vin = v0;
    uint32_t* vout = v1;
    for (int p = 0; p < passes; ++p) {
        launch_k(onesweep_kernel<K, ITEMS, RANK_OR>, dim3((unsigned)tiles), dim3(SORT_THREADS),
                 sort_smem<K, ITEMS>(), s, (const K*)kin, (const uint32_t*)((p == 0 && identity_vals) ? nullptr : vin),
                 kout, vout, n_cap, (p > 0 && po.n_dev_rest) ? po.n_dev_rest : n_dev, 8 * p,
                 (const uint32_t*)(hist + p * RADIX), status + (size_t)p * tiles * RADIX, counters + p,
                 p == 0 ? po.rel_min0 : nullptr, po.npass_dev, p,
                 po.next_hist && p + 1 < passes ? const_cast<uint32_t*>(hist) + (p + 1) * RADIX : nullptr,
                 p == 0 ? po.meta : nullptr);
        if (check_launch("onesweep_kernel")) return -1;
        K* tk = kin; kin = kout; kout = tk;
        uint32_t* tv = vin; vin = vout; vout = tv;
    }
    return 0;
}

template <typename K, int ITEMS>
static int run_passes(K* k0, uint32_t* v0, K* k1, uint32_t* v1, int64_t n_cap, const unsigned long long* n_dev,
                      int passes, const uint32_t* hist, uint32_t* status, uint32_t* counters, cudaStream_t s,
                      bool identity_vals, const PassOpts& po = PassOpts()) {
    if (rank_or())
        return run_passes_t<K, ITEMS, true>(k0, v0, k1, v1, n_cap, n_dev, passes, hist, status, counters, s,
                                            identity_vals, po);
    return run_passes_t<K, ITEMS, false>(k0, v0, k1, v1, n_cap, n_dev, passes, hist, status, counters, s,
                                         identity_vals, po);
}

template <typename K>
int run_onesweep(K* k0, uint32_t* v0, K* k1, uint32_t* v1, int64_t n_cap, const unsigned long long* n_dev,
                 int passes, const uint32_t* hist, uint32_t* status, uint32_t* counters, cudaStream_t s,
                 bool identity_vals) {
    if (n_cap <= 0) return 0;
    constexpr int BIG = SortCfg<K>::ITEMS;
    const int64_t big_tiles = (n_cap + sort_tile<K, BIG>() - 1) / sort_tile<K, BIG>();
    static int small_env = -2;
    if (small_env == -2) {
        const char* e = getenv("GS_SORT_SMALL");
        small_env = e ? atoi(e) : -1;
    }
    const bool small = small_env >= 0 ? small_env != 0 : big_tiles < 64;
    if (small)
        return run_passes<K, SMALL_ITEMS>(k0, v0, k1, v1, n_cap, n_dev, passes, hist, status, counters, s,
                                          identity_vals);
    if constexpr (sizeof(K) == 4) {  // A/B switch: GS_SORT_ITEMS=8|12 (default SortCfg)
        static int items_env = -2;
        if (items_env == -2) {
            const char* e = getenv("GS_SORT_ITEMS");
            items_env = e ? atoi(e) : -1;
        }
        if (items_env == 8)
            return run_passes<K, 8>(k0, v0, k1, v1, n_cap, n_dev, passes, hist, status, counters, s, identity_vals);
        if (items_env == 12)
            return run_passes<K, 12>(k0, v0, k1, v1, n_cap, n_dev, passes, hist, status, counters, s, identity_vals);
        if (items_env == 20)
            return run_passes<K, 20>(k0, v0, k1, v1, n_cap, n_dev, passes, hist, status, counters, s, identity_vals);
        if (items_env == 24)
            return run_passes<K, 24>(k0, v0, k1, v1, n_cap, n_dev, passes, hist, status, counters, s, identity_vals);
    }
    return run_passes<K, BIG>(k0, v0, k1, v1, n_cap, n_dev, passes, hist, status, counters, s, identity_vals);
}
template int run_onesweep<uint32_t>(uint32_t*, uint32_t*, uint32_t*, uint32_t*, int64_t,
                                    const unsigned long long*, int, const uint32_t*, uint32_t*, uint32_t*,
                                    cudaStream_t, bool);
template int run_onesweep<unsigned long long>(unsigned long long*, uint32_t*, unsigned long long*, uint32_t*,
                                              int64_t, const unsigned long long*, int, const uint32_t*,
                                              uint32_t*, uint32_t*, cudaStream_t, bool);

// Look-back status the depth sort of n keys uses (its pass variant, 4 passes).
size_t depth_sort_status_bytes(int64_t n) {
    constexpr int BIG = SortCfg<uint32_t>::ITEMS;
    const int64_t big_tiles = (n + sort_tile<uint32_t, BIG>() - 1) / sort_tile<uint32_t, BIG>();
    const int items = big_tiles < 64 ? SMALL_ITEMS : BIG;
    const int64_t tiles = (n + (int64_t)SORT_THREADS * items - 1) / ((int64_t)SORT_THREADS * items);
    return (size_t)4 * (size_t)(tiles > 0 ? tiles : 1) * RADIX * 4;
}

// Stable sort of the visible Gaussians by depth (frame.cu): hist holds the
// projection's histogram of the visible keys' absolute low byte (rows 1-3
// zeroed; the passes fill them in turn), meta[5..6] the key range.
int run_depth_sort(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, int64_t n_cap,
                   unsigned long long* meta, uint32_t* hist, uint32_t* status, uint32_t* counters, cudaStream_t s) {
    if (n_cap <= 0) return 0;
    PassOpts po;
    po.n_dev_rest = meta + 7;
    po.rel_min0 = meta + 5;
    po.npass_dev = meta + 8;
    po.next_hist = true;
    po.meta = meta;
    constexpr int BIG = SortCfg<uint32_t>::ITEMS;
    const int64_t big_tiles = (n_cap + sort_tile<uint32_t, BIG>() - 1) / sort_tile<uint32_t, BIG>();
    if (big_tiles < 64)
        return run_passes<uint32_t, SMALL_ITEMS>(k0, v0, k1, v1, n_cap, nullptr, 4, hist, status, counters, s, true,
                                                 po);
    return run_passes<uint32_t, BIG>(k0, v0, k1, v1, n_cap, nullptr, 4, hist, status, counters, s, true, po);
}

template <typename K>
int launch_sort_hist(const K* keys, int64_t n_cap, const unsigned long long* n_dev, int passes, uint32_t* hist,
                     cudaStream_t s) {
    int64_t hb = (n_cap + 255) / 256;
    const int64_t lim = (int64_t)sort_sm_count() * 4;
    if (hb > lim) hb = lim;
    if (hb < 1) hb = 1;
    sort_hist_kernel<K><<<(unsigned)hb, 256, 0, s>>>(keys, n_cap, n_dev, passes, hist);
    return check_launch("sort_hist_kernel");
}
template int launch_sort_hist<uint32_t>(const uint32_t*, int64_t, const unsigned long long*, int, uint32_t*,
                                        cudaStream_t);
template int launch_sort_hist<unsigned long long>(const unsigned long long*, int64_t, const unsigned long long*,
                                                  int, uint32_t*, cudaStream_t);

}  // namespace gs

using namespace gs;

extern "C" {

size_t gs_sort_workspace_bytes(int64_t n, int end_bit) {
    const int passes = (end_bit + 7) / 8;
    return (size_t)MAX_PASSES * RADIX * 4 + 64 + onesweep_status_bytes<unsigned long long>(n, passes);
}

int gs_sort_pairs(unsigned long long* keys, unsigned long long* keys_alt, uint32_t* vals, uint32_t* vals_alt,
                  int64_t n, int end_bit, void* ws, size_t ws_bytes, int* selector, gs_stream_t stream) {
    if (end_bit < 1 || end_bit > 64) return set_error("gs_sort_pairs: end_bit %d out of range", end_bit);
    if (n < 0 || n >= (int64_t)ST_MASK) return set_error("gs_sort_pairs: n=%lld out of range", (long long)n);
    if (ws_bytes < gs_sort_workspace_bytes(n, end_bit)) return set_error("gs_sort_pairs: workspace too small");
    const int passes = (end_bit + 7) / 8;
    *selector = 0;
    if (n == 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t* hist = (uint32_t*)ws;
    uint32_t* counters = hist + MAX_PASSES * RADIX;
    uint32_t* status = counters + 16;
    if (cudaMemsetAsync(ws, 0, gs_sort_workspace_bytes(n, end_bit), s) != cudaSuccess)
        return check_launch("sort memset");
    if (launch_sort_hist<unsigned long long>(keys, n, nullptr, passes, hist, s)) return -1;
    if (run_onesweep<unsigned long long>(keys, vals, keys_alt, vals_alt, n, nullptr, passes, hist, status, counters,
                                         s, false))
        return -1;
    *selector = passes & 1;
    return 0;
}

}  // extern "C"
