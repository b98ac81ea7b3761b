// internal.cuh -- host-side launchers shared between translation units
// (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace gs {

// project.cu
int launch_project_fwd_dkey(const float* means3, const float* scales3, const float* quats4, const float* opac,
                            int64_t n, const CamK& k, float* xydr4, float* conic4, uint32_t* tiles, float* cov3,
                            unsigned long long* status, uint32_t* dkeys, uint32_t* dhist, cudaStream_t s,
                            const ZeroJobs& zj, uint32_t* tcount = nullptr, uint32_t* bins = nullptr,
                            uint32_t kstride = 0, unsigned long long* clean_word = nullptr,
                            unsigned long long clean_sig = 0);  // also resets meta (status, total, need), dhist and
                            // (scatter / direct binning: per-tile intersection counts) tcount first;
                            // bins != nullptr: direct binning into bins[tile * kstride + slot]
int launch_project_bwd(const float* means3, const float* scales3, const float* quats4, int64_t n, const CamK& k,
                       const uint32_t* tiles, const float* d_geo4, const float* d_c11, float* d_means3,
                       float* d_scales3, float* d_quats4, float* d_view16, float* partials, cudaStream_t s,
                       bool accumulate = false, int gstride = 1, const float* rgbo_in = nullptr,
                       float* rgbo_out = nullptr, unsigned int* done_counter = nullptr,
                       unsigned long long* clean_word = nullptr, unsigned long long clean_sig = 0,
                       bool clear_accum = false, bool add_view = false, bool vis_from_grads = false);
// clear_accum (frame path): every visible Gaussian's screen-space accumulator
// row (d_geo4 row + d_rgbo row + d_c11) is zeroed after it is read, and the
// last block stamps *clean_word = clean_sig (0 when not clearing), which the
// next gs_frame_forward checks instead of zeroing the accumulators itself.
// gstride 2: d_geo4 rows interleaved with d_rgbo rows (g8 layout); with
// rgbo_in, each Gaussian's d_rgbo row is copied (or added) to rgbo_out.
constexpr int PBWD_BLOCK = 256;
// all views of a step at once (project.cu): per view its camera, its
// workspace's screen-space gradient rows ([d_rgbo4 | d_geo4] per Gaussian,
// d_c11), its d_view partials (>= blocks x 12 floats) and its clean word
constexpr int MV_MAX = 32;
struct MvView {
    CamK cam;
    float4* g8;
    float* d_c11;
    // bit (tbase + i) of touched clear: Gaussian i's rows are zero (the raster
    // backward marks every Gaussian it adds to; nullptr: read every row)
    const uint32_t* touched;
    int tbase;
    float* partials;
    unsigned long long* clean_word;
    unsigned long long clean_stamp;
};
struct MvArgs {
    int nv;
    MvView v[MV_MAX];
};
// the depth-first projection of every view of a step (views_init_kernel +
// views_project_fwd_kernel, project.cu): per view its camera, its
// workspace's outputs, meta, depth histograms, clean word and zero jobs
struct MvFwdView {
    CamK cam;
    float4* xydr;
    float4* conic;
    uint32_t* tiles;
    uint32_t* dkeys;
    uint32_t* dhist;
    unsigned long long* meta;
    unsigned long long* clean_word;
    unsigned long long clean_sig;
    ZeroJobs zj;
};
struct MvFwdArgs {
    int nv;
    MvFwdView v[MV_MAX];
};
int launch_views_project_fwd(const float* means3, const float* scales3, const float* quats4, const float* opac,
                             int64_t n, const MvFwdArgs& a, cudaStream_t s);
int launch_views_project_bwd(const float* means3, const float* scales3, const float* quats4, int64_t n,
                             const MvArgs& a, float* d_means3, float* d_scales3, float* d_quats4, float* d_rgbo4,
                             float* d_views16, bool accumulate, bool clear_rows, bool add_view, cudaStream_t s);

// sort.cu
int sort_sm_count();
template <typename K>
size_t onesweep_status_bytes(int64_t n_cap, int passes);
size_t depth_sort_status_bytes(int64_t n);  // the part of onesweep_status_bytes(n, 4) the depth sort uses
template <typename K>
int run_onesweep(K* k0, uint32_t* v0, K* k1, uint32_t* v1, int64_t n_cap, const unsigned long long* n_dev,
                 int passes, const uint32_t* hist, uint32_t* status, uint32_t* counters, cudaStream_t s,
                 bool identity_vals);
// Stable sort of the visible Gaussians by depth (frame.cu, depth-first
// binning): keys relative to meta[5], culled (0xFFFFFFFF) ones dropped by the
// first pass, later passes over meta[7] items, passes beyond meta[8] skipped.
// The (keys, ids) end in (k1, v1) when meta[8] is odd, else in (k0, v0).
int run_depth_sort(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, int64_t n_cap,
                   unsigned long long* meta, uint32_t* hist, uint32_t* status, uint32_t* counters, cudaStream_t s);
template <typename K>
int launch_sort_hist(const K* keys, int64_t n_cap, const unsigned long long* n_dev, int passes, uint32_t* hist,
                     cudaStream_t s);

// binning.cu
size_t scan_ws_bytes(int64_t n);
int launch_scan(const uint32_t* in, const uint32_t* gather, uint32_t* out, int64_t n, void* ws,
                unsigned long long* total, cudaStream_t s);  // ws must be zeroed
int launch_emit_sorted(const uint32_t* order, const float* xydr4, const uint32_t* offsets, int64_t n,
                       int tiles_x, int tiles_y, int64_t capacity, uint32_t* tile_keys, uint32_t* vals,
                       uint32_t* tile_hist, int tile_passes, cudaStream_t s);
// fused scan of the projection's tile counts + pair emission (frame path);
// ws (emit_scan_ws_bytes(n), zeroed): chunk counter + look-back status
size_t emit_scan_ws_bytes(int64_t n);
int launch_emit_scan(const uint32_t* order, const float* xydr4, const uint32_t* counts, int64_t n, int tiles_x,
                     int tiles_y, int64_t capacity, uint32_t* tile_keys, uint32_t* vals, uint32_t* tile_hist,
                     int tile_passes, void* ws, unsigned long long* total, cudaStream_t s,
                     const uint32_t* order_alt = nullptr, const unsigned long long* sort_meta = nullptr);
// sort_meta (depth-first frame, = meta + 7): [0] the number of sorted (visible)
// Gaussians, [1] the depth-sort pass count (odd: the order is in order_alt)
// depth-first binning, tile-sorted emission (binning.cu): the expanded pairs
// (pairs: capacity u32 scratch), the per-(chunk, tile) counts and their
// column sums (table: emit_tiles_table_bytes, no zeroing needed; scan_ws:
// emit_scan_ws_bytes, zeroed) and every tile's total into totals; then
// (launch_tile_scan(totals, ..., replicas 1) makes the ranges and leaves the
// starts in totals) the bases of every (chunk, tile) and the placement
size_t emit_tiles_smem(int n_tiles);
bool emit_tiles_fits(int n_tiles);
size_t emit_tiles_table_bytes(int64_t n, int n_tiles);
int launch_emit_tiles_count(const uint32_t* order, const uint32_t* order_alt, const float* xydr4, int64_t n,
                            int tiles_x, int tiles_y, int64_t capacity, void* table, uint32_t* totals,
                            uint32_t* pairs, void* scan_ws, const unsigned long long* meta, cudaStream_t s);
int launch_emit_tiles(const uint32_t* order, const uint32_t* order_alt, int64_t n, int tiles_x, int tiles_y,
                      int64_t capacity, const uint32_t* starts, void* table, const uint32_t* pairs, uint32_t* vals,
                      const unsigned long long* meta, cudaStream_t s);
// option "tile_emit" (abi.cu): 1 (default) tile-sorted emission where it fits, 0 emission + onesweep by tile
bool tile_emit();
// scatter binning: tile scan (ranges, cursors, total, optional raster order)
// and the unordered scatter of the (tile, gaussian) pairs
int launch_tile_scan(uint32_t* tcount, int n_tiles, int64_t capacity, uint2* ranges, unsigned long long* total,
                     uint32_t* order, cudaStream_t s, int replicas = TCOUNT_REPL);
int launch_scatter_pairs(const float* xydr4, const uint32_t* counts, int64_t n, int tiles_x, int tiles_y,
                         int64_t capacity, uint32_t* cursors, uint32_t* tile_keys, uint32_t* vals, cudaStream_t s);
// heaviest-first raster launch order of the tiles (one CTA)
int launch_tile_order(const uint2* ranges, int n_tiles, uint32_t* order, cudaStream_t s);
int launch_ranges_u64(const unsigned long long* sorted_keys, int64_t n, uint2* ranges,
                      cudaStream_t s);  // ranges must be zeroed
int launch_ranges_u32(const uint32_t* sorted_tile_keys, int64_t n_cap, const unsigned long long* n_dev,
                      uint2* ranges, cudaStream_t s);  // ranges must be zeroed

// segsort.cu: per-tile stable sort of each tile's list by depth key
int launch_segsort(const uint2* ranges, int n_tiles, const uint32_t* dkeys, uint32_t* vals, uint32_t* alt,
                   cudaStream_t s);
// binning strategy of the frame path (abi.cu): 0 auto, 1 depth-first, 2 scatter
int binning_mode();
// frame path with scatter binning: tile sort fused into the raster forward (1) or its own kernel (0)
bool fuse_sort();

// raster.cu
int launch_raster_fwd(const uint2* ranges, const uint32_t* vals, const float* xydr4, const float* conic4,
                      const float* colors3, float3 bg, int W, int H, bool et, float* img, float* T, int* nc,
                      unsigned long long* counts, cudaStream_t s, uint2* rec = nullptr,
                      uint32_t* rec_count = nullptr, const uint32_t* tile_order = nullptr,
                      const uint32_t* dkeys = nullptr, uint32_t* sort_alt = nullptr,  // dkeys: fused tile sort
                      const uint32_t* direct_counts = nullptr, uint32_t kstride = 0,    // direct binning
                      unsigned long long* meta = nullptr);
// record-driven backward of the frame path (records written by the forward)
int launch_raster_bwd_rec(const uint2* ranges, const uint2* rec, const uint32_t* rec_count, const float* xydr4,
                          const float* conic4, const float* colors3, float3 bg, int W, int H, const float* fT,
                          const int* nc, const float* dimg, float* g8, float* d_c11, cudaStream_t s,
                          const uint32_t* tile_order = nullptr, const unsigned long long* meta = nullptr,
                          uint32_t* touched = nullptr);
int launch_raster_bwd(const uint2* ranges, const uint32_t* vals, const float* xydr4, const float* conic4,
                      const float* colors3, float3 bg, int W, int H, const float* fT, const int* nc,
                      const float* dimg, float* d_rgbo4, float* d_geo4, float* d_c11, unsigned long long* counts,
                      cudaStream_t s, int gstride);  // gstride: float4 rows between splats (1, or 2 interleaved)

}  // namespace gs
