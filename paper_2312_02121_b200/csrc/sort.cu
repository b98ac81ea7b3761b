// sort.cu -- hand-written stable LSD radix sort of (uint64 key, uint32 value)
// pairs in the "onesweep" style (one upfront histogram of every digit pass,
// then one kernel per 8-bit pass that ranks a tile of keys, obtains its
// global digit offsets through a decoupled look-back chained scan and
// scatters).  Stability is what makes (tile << 32 | depth bits) keys emitted
// in Gaussian-index order reproduce sg/binning.py:50-65's
// (depth, source_index) order.
#include "common.cuh"

namespace gs {

constexpr int SORT_THREADS = 256;
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr int SORT_ITEMS = 15;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;  // 3840 pairs per CTA
constexpr int RADIX = 256;
constexpr int MAX_PASSES = 8;
constexpr uint32_t ST_AGG = 1u << 30;
constexpr uint32_t ST_PRE = 2u << 30;
constexpr uint32_t ST_MASK = (1u << 30) - 1;
constexpr size_t SORT_SMEM = (size_t)SORT_TILE * 8 + (size_t)SORT_TILE * 4 + (size_t)SORT_WARPS * RADIX * 4 +
                             2 * RADIX * 4;

__device__ __forceinline__ uint32_t ldv(const uint32_t* p) { return *(const volatile uint32_t*)p; }
__device__ __forceinline__ void stv(uint32_t* p, uint32_t v) { *(volatile uint32_t*)p = v; }

__global__ void __launch_bounds__(256) sort_hist_kernel(const unsigned long long* __restrict__ keys, int64_t n,
                                                        int passes, uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[MAX_PASSES * RADIX];
    for (int k = threadIdx.x; k < passes * RADIX; k += blockDim.x) sh[k] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&sh[p * RADIX + (int)((key >> (8 * p)) & 255ull)], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < passes * RADIX; k += blockDim.x) {
        const uint32_t v = sh[k];
        if (v) atomicAdd(&hist[k], v);
    }
}

// Inclusive block scan over 256 threads (one value per thread).
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

__global__ void __launch_bounds__(SORT_THREADS, 2) onesweep_kernel(
    const unsigned long long* __restrict__ kin, const uint32_t* __restrict__ vin,
    unsigned long long* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n, int shift,
    const uint32_t* __restrict__ hist, uint32_t* __restrict__ status, uint32_t* __restrict__ counter) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* s_keys = reinterpret_cast<unsigned long long*>(smem);
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + SORT_TILE);
    uint32_t* s_whist = s_vals + SORT_TILE;       // [warp][digit]
    uint32_t* s_gbase = s_whist + SORT_WARPS * RADIX;  // global dst of local slot 0 per digit
    uint32_t* s_lstart = s_gbase + RADIX;         // local start of each digit in the tile
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_tmp[SORT_WARPS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(counter, 1u);
#pragma unroll
    for (int k = 0; k < SORT_WARPS; ++k) s_whist[k * RADIX + tid] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const int64_t wbase = (int64_t)tile * SORT_TILE + (int64_t)warp * (SORT_ITEMS * 32);

    unsigned long long key[SORT_ITEMS];
    uint32_t val[SORT_ITEMS];
    uint32_t rank[SORT_ITEMS];
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        const int64_t idx = wbase + i * 32 + lane;
        key[i] = idx < n ? kin[idx] : ~0ull;
        val[i] = idx < n ? vin[idx] : 0u;
    }
    // warp-local stable ranking: items in (i, lane) order = input order
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        const int64_t idx = wbase + i * 32 + lane;
        const bool valid = idx < n;
        const uint32_t d = (uint32_t)(key[i] >> shift) & 255u;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        rank[i] = 0;
        if (valid) {
            const uint32_t peers = __match_any_sync(vmask, d);
            const int leader = __ffs(peers) - 1;
            uint32_t old = 0;
            if (lane == leader) old = atomicAdd(&s_whist[warp * RADIX + d], (uint32_t)__popc(peers));
            old = __shfl_sync(peers, old, leader);
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
        int p = (int)tile - 1;
        while (true) {
            const uint32_t s = ldv(status + (size_t)p * RADIX + d);
            const uint32_t f = s & ~ST_MASK;
            if (f == 0) continue;
            excl += s & ST_MASK;
            if (f == ST_PRE) break;
            --p;
        }
        stv(st, ST_PRE | (excl + run));
    }
    const uint32_t h = hist[d];
    const uint32_t lincl = block_incl_scan256(run, s_tmp);
    const uint32_t hincl = block_incl_scan256(h, s_tmp);
    const uint32_t lstart = lincl - run;
    s_lstart[d] = lstart;
    s_gbase[d] = (hincl - h) + excl - lstart;  // mod 2^32; dst = gbase + local slot
    __syncthreads();
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        const int64_t idx = wbase + i * 32 + lane;
        if (idx < n) {
            const uint32_t dd = (uint32_t)(key[i] >> shift) & 255u;
            const uint32_t pos = s_lstart[dd] + s_whist[warp * RADIX + dd] + rank[i];
            s_keys[pos] = key[i];
            s_vals[pos] = val[i];
        }
    }
    __syncthreads();
    const int64_t rem = n - (int64_t)tile * SORT_TILE;
    const int cnt = rem < SORT_TILE ? (int)rem : SORT_TILE;
    for (int j = tid; j < cnt; j += SORT_THREADS) {
        const unsigned long long k = s_keys[j];
        const uint32_t dd = (uint32_t)(k >> shift) & 255u;
        const uint32_t dst = s_gbase[dd] + (uint32_t)j;
        kout[dst] = k;
        vout[dst] = s_vals[j];
    }
}

static bool g_sort_attr_set = false;

}  // namespace gs

using namespace gs;

extern "C" {

size_t gs_sort_workspace_bytes(int64_t n, int end_bit) {
    const int passes = (end_bit + 7) / 8;
    const int64_t tiles = (n + SORT_TILE - 1) / SORT_TILE;
    return (size_t)MAX_PASSES * RADIX * 4 + 64 + (size_t)passes * (size_t)(tiles > 0 ? tiles : 1) * RADIX * 4;
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
    if (!g_sort_attr_set) {
        if (cudaFuncSetAttribute(onesweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SORT_SMEM) !=
            cudaSuccess)
            return check_launch("onesweep smem attribute");
        g_sort_attr_set = true;
    }
    const int64_t tiles = (n + SORT_TILE - 1) / SORT_TILE;
    uint32_t* hist = (uint32_t*)ws;
    uint32_t* counters = hist + MAX_PASSES * RADIX;
    uint32_t* status = counters + 16;
    const size_t status_bytes = (size_t)passes * (size_t)tiles * RADIX * 4;
    if (cudaMemsetAsync(ws, 0, (size_t)MAX_PASSES * RADIX * 4 + 64 + status_bytes, s) != cudaSuccess)
        return check_launch("sort memset");
    int sms = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int64_t hb = (n + 255) / 256;
    if (hb > (int64_t)sms * 4) hb = (int64_t)sms * 4;
    sort_hist_kernel<<<(unsigned)hb, 256, 0, s>>>(keys, n, passes, hist);
    if (check_launch("sort_hist_kernel")) return -1;
    unsigned long long* kin = keys;
    unsigned long long* kout = keys_alt;
    uint32_t* vin = vals;
    uint32_t* vout = vals_alt;
    for (int p = 0; p < passes; ++p) {
        onesweep_kernel<<<(unsigned)tiles, SORT_THREADS, SORT_SMEM, s>>>(
            kin, vin, kout, vout, n, 8 * p, hist + p * RADIX, status + (size_t)p * tiles * RADIX, counters + p);
        if (check_launch("onesweep_kernel")) return -1;
        unsigned long long* tk = kin; kin = kout; kout = tk;
        uint32_t* tv = vin; vin = vout; vout = tv;
    }
    *selector = passes & 1;
    return 0;
}

}  // extern "C"
