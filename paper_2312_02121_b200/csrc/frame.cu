// frame.cu -- one differentiable render as two sync-free entry points.
//
// gs_frame_forward, depth-first binning (large scenes):
//   project (+ depth keys and their digit histograms)
//   -> 4-pass onesweep sort of the Gaussians by depth (stable, index order)
//   -> scan of tile counts in depth order -> emission of (tile, gaussian)
//   pairs in depth order (+ tile-digit histograms) -> 1-2 pass stable sort by
//   tile id -> per-tile ranges (+ raster order) -> raster forward.
//   With the tile-sorted emission (option tile_emit, <= 9800 tiles), the
//   emission and the sort by tile are one stable counting pass instead:
//   per-(chunk, tile) pair counts -> column prefixes + tile totals -> tile
//   scan (ranges, raster order) -> every pair written to its final slot.
// gs_frame_forward, scatter binning (N <= 400k):
//   project (+ depth keys and per-tile intersection counts) -> tile scan
//   (ranges, cursors, raster order) -> pair scatter -> per-tile (depth,
//   index) sort (segsort.cu) -> raster forward.
// gs_frame_backward: raster backward (atomic per-warp accumulation of the
//   screen-space gradients) -> projection backward (+ fixed-order d_view).
//
// Nothing here synchronizes with the host or allocates: intersections are
// written into a caller-sized capacity and the true total is reported in
// meta[1]; a caller that sees total > capacity re-runs with a larger
// workspace.  That makes a whole training step capturable in a CUDA graph.
//
// The depth-first binning is equivalent to sorting (tile << 32 | depth bits)
// keys emitted in Gaussian order (gs_emit_keys + gs_sort_pairs): both give
// every tile's list in (depth, source_index) order -- sg/binning.py:50-65 --
// but the 64-bit variant sorts I pairs over 5-6 passes while this sorts N
// 32-bit keys over 4 passes plus I 32-bit keys over 1-2 passes.
#include <cstring>

#include "common.cuh"
#include "internal.cuh"

namespace gs {

namespace {

constexpr size_t ALIGN = 256;

inline size_t up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

int tile_passes_for(int n_tiles) { return n_tiles <= 256 ? 1 : 2; }

// Heaviest-first tile order pays only when the raster grid is more than one
// wave (148 SMs x 8 resident CTAs); GS_TILE_ORDER=0 disables it (A/B switch).
bool tile_order_enabled(int n_tiles) {
    static const bool on = [] {
        const char* e = getenv("GS_TILE_ORDER");
        return !(e && e[0] == '0');
    }();
    return on && n_tiles > 148 * 8;
}

// Binning strategy (gs_set_option("binning"): 0 auto, 1 depth-first,
// 2 scatter, 3 direct).  Auto: direct for small scenes on up to 4096 tiles,
// scatter for other small scenes, depth-first for N > 400k.
enum Binning { DEPTH_FIRST = 1, SCATTER = 2, DIRECT = 3 };
Binning binning_for(int64_t n, int n_tiles) {
    const int bmode = binning_mode();
    if (bmode >= 1 && bmode <= 3) return (Binning)bmode;
    if (n > 400000) return DEPTH_FIRST;
    return n_tiles <= 4096 ? DIRECT : SCATTER;
}
bool scatter_binning(int64_t n, int n_tiles) { return binning_for(n, n_tiles) != DEPTH_FIRST; }

// Direct binning: every tile owns kstride = capacity / tiles pair slots.
int64_t direct_stride(int64_t cap, int n_tiles) { return n_tiles > 0 ? cap / n_tiles : 0; }

// Every binning leaves the frame's tile-sorted (keys, vals) in the primary
// buffers (the depth-first emission targets the alternates when it sorts an
// odd number of tile passes), so readers never depend on the options.

struct Layout {
    // persistent (written each frame)
    size_t xydr, conic, tiles, dkeys, dkeys_alt, order, order_alt, offsets;
    size_t tkeys, tkeys_alt, tvals, tvals_alt, ranges, rec, rec_count, tile_order, tcount, clean;
    // zeroed region
    size_t zero_begin, meta, dhist, thist, counters, scan_ws, touched, dstatus, tstatus, zero_end;
    // backward
    size_t etable;  // tile-sorted emission: per-(chunk, tile) counts and prefixes
    size_t d_geo, d_c11, pbwd_done, partials;
    size_t total;
};

Layout layout(int64_t n, int64_t cap, int W, int H) {
    const int64_t nt = (int64_t)((W + TILE - 1) / TILE) * ((H + TILE - 1) / TILE);
    const int tp = tile_passes_for((int)nt);
    Layout L;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o += up(bytes > 0 ? bytes : 1);
        return at;
    };
    // the clean word sits at offset 0 for every layout, so a frame of any
    // other layout run on the same workspace always overwrites it
    L.clean = take(16);  // layout signature while the backward accumulators are known zero
    L.xydr = take(16 * n);
    L.conic = take(16 * n);
    L.tiles = take(4 * n);
    L.dkeys = take(4 * n);
    L.dkeys_alt = take(4 * n);
    L.order = take(4 * n);
    L.order_alt = take(4 * n);
    L.offsets = take(4 * n);
    L.tkeys = take(4 * cap);
    L.tkeys_alt = take(4 * cap);
    L.tvals = take(4 * cap);
    L.tvals_alt = take(4 * cap);
    L.rec = take(8 * 4 * cap);    // forward commit records, 4 warp regions per tile list
    L.rec_count = take(16 * nt);  // records per (tile, warp)
    L.tile_order = take(4 * nt);  // raster launch order (heaviest lists first)
    L.tcount = take(4 * TCOUNT_REPL * nt);  // scatter binning: tile counts, then write cursors
    L.zero_begin = o;
    L.meta = take(128);  // [0] status [1] total intersections [2] capacity needed [3] direct-binning
                         // tile stride [4] accumulators-to-zero flag [5,6] visible depth-key min / max
                         // [7] visible Gaussians [8] depth-sort passes
    L.dhist = take(4 * 256 * 4);
    L.thist = take(4 * 256 * 2);
    L.counters = take(64);
    L.scan_ws = take(emit_scan_ws_bytes(n));
    L.ranges = take(8 * nt);
    L.touched = take(4 * ((n + 31) / 32));  // Gaussians the raster backward added to (bit per Gaussian)
    L.dstatus = take(onesweep_status_bytes<uint32_t>(n, 4));  // sized for either pass variant; the used part is zeroed
    L.zero_end = o;
    L.tstatus = take(onesweep_status_bytes<uint32_t>(cap, tp));  // tile passes (depth-first without the tile emission)
    L.etable = take(emit_tiles_fits((int)nt) ? emit_tiles_table_bytes(n, (int)nt) : 0);
    L.d_geo = take(32 * n);  // interleaved screen-space gradients: [d_rgbo 4 | d_geo 4] per Gaussian
    L.d_c11 = take(4 * n);
    L.pbwd_done = take(16);  // last-block counter of the projection backward (zeroed with the accumulators)
    L.partials = take(12 * 4 * ((n + PBWD_BLOCK - 1) / PBWD_BLOCK + 1));
    L.total = o;
    return L;
}

void mark(void* const* ev, int k, cudaStream_t s) {
    if (!ev || !ev[k]) return;
    // inside stream capture an External record becomes a real event-record node
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags((cudaEvent_t)ev[k], s, cudaEventRecordExternal);
    else
        cudaEventRecord((cudaEvent_t)ev[k], s);
}

template <typename T>
T* at(void* ws, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

// Signature of a workspace layout (stamped in the clean word while the
// backward accumulators hold zeros).
unsigned long long clean_sig(int64_t n, int64_t cap, int W, int H) {
    unsigned long long h = 0x9e3779b97f4a7c15ull;
    for (unsigned long long v : {(unsigned long long)n, (unsigned long long)cap, (unsigned long long)W,
                                 (unsigned long long)H}) {
        h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
        h *= 0xbf58476d1ce4e5b9ull;
    }
    return h | 1ull;  // never 0 (0 = "not clean")
}

// Buffers the frame's projection clears for the later stages (no memset
// nodes): the counters, tile ranges and the part of the depth sort's
// look-back status its pass variant uses; the tile passes' status only for
// the depth-first binning without the tile-sorted emission; and -- only when
// the workspace is not known clean (meta[4]) -- the backward's screen-space
// accumulators.
ZeroJobs frame_zero_jobs(const Layout& L, void* ws, int64_t n, int n_tiles, bool tile_passes) {
    ZeroJobs zj;
    zj.p[0] = at<uint4>(ws, L.thist);
    zj.n16[0] = (L.dstatus + depth_sort_status_bytes(n) - L.thist + 15) / 16;
    zj.p[1] = at<uint4>(ws, L.tstatus);
    zj.n16[1] = tile_passes ? (L.etable - L.tstatus) / 16 : 0;
    zj.p[2] = at<uint4>(ws, L.d_geo);
    zj.n16[2] = (L.partials - L.d_geo) / 16;
    zj.cond2 = at<unsigned long long>(ws, L.meta) + 4;
    return zj;
}

bool uses_tile_emit(int64_t n, int n_tiles) {
    return binning_for(n, n_tiles) == DEPTH_FIRST && tile_emit() && emit_tiles_fits(n_tiles);
}

int frame_forward_impl(const float* means3, const float* scales3, const float* quats4, const float* opacities,
                       const float* colors3, int64_t n, const gs_camera* cam, const float* background3,
                       int early_termination, int64_t isect_capacity, void* ws, size_t ws_bytes, float* out_image,
                       float* out_final_T, int32_t* out_n_contrib, unsigned long long* counts4,
                       void* const* stage_events, gs_stream_t stream, bool projected);

}  // namespace

}  // namespace gs

using namespace gs;

extern "C" {

int gs_frame_binning(int64_t n, int32_t width, int32_t height) {
    return (int)binning_for(n, ((width + TILE - 1) / TILE) * ((height + TILE - 1) / TILE));
}

int gs_frame_tile_emit(int64_t n, int32_t width, int32_t height) {
    const int nt = ((width + TILE - 1) / TILE) * ((height + TILE - 1) / TILE);
    return binning_for(n, nt) == DEPTH_FIRST && tile_emit() && emit_tiles_fits(nt) ? 1 : 0;
}

size_t gs_frame_workspace_bytes(int64_t n, int64_t isect_capacity, int32_t width, int32_t height) {
    return layout(n, isect_capacity, width, height).total;
}

int gs_frame_workspace_init(int64_t n, int64_t isect_capacity, int32_t width, int32_t height, void* ws,
                            gs_stream_t stream) {
    const Layout L = layout(n, isect_capacity, width, height);
    if (cudaMemsetAsync(at<char>(ws, L.clean), 0, 16, (cudaStream_t)stream) != cudaSuccess)
        return check_launch("gs_frame_workspace_init");
    return 0;
}

int gs_frame_view_of(int64_t n, int64_t isect_capacity, int32_t width, int32_t height, void* ws,
                     gs_frame_view* out) {
    const Layout L = layout(n, isect_capacity, width, height);
    out->xydr4 = at<float>(ws, L.xydr);
    out->conic4 = at<float>(ws, L.conic);
    out->tiles = at<uint32_t>(ws, L.tiles);
    out->depth_order = at<uint32_t>(ws, L.order);
    out->depth_order_alt = at<uint32_t>(ws, L.order_alt);
    out->sorted_tile_keys = at<uint32_t>(ws, L.tkeys);
    out->sorted_vals = at<uint32_t>(ws, L.tvals);
    out->ranges2 = at<uint32_t>(ws, L.ranges);
    out->meta = at<unsigned long long>(ws, L.meta);
    out->d_geo4 = at<float>(ws, L.d_geo) + 4;  // rows of 8 floats: [d_rgbo 4 | d_geo 4]
    out->d_c11 = at<float>(ws, L.d_c11);
    out->bwd_accum = at<char>(ws, L.d_geo);
    out->bwd_accum_bytes = L.partials - L.d_geo;
    out->rec_count = at<uint32_t>(ws, L.rec_count);
    out->touched = at<uint32_t>(ws, L.touched);
    return 0;
}

int gs_frame_forward(const float* means3, const float* scales3, const float* quats4, const float* opacities,
                     const float* colors3, int64_t n, const gs_camera* cam, const float* background3,
                     int early_termination, int64_t isect_capacity, void* ws, size_t ws_bytes, float* out_image,
                     float* out_final_T, int32_t* out_n_contrib, unsigned long long* counts4, void* const* stage_events,
                     gs_stream_t stream) {
    return frame_forward_impl(means3, scales3, quats4, opacities, colors3, n, cam, background3, early_termination,
                              isect_capacity, ws, ws_bytes, out_image, out_final_T, out_n_contrib, counts4,
                              stage_events, stream, false);
}

int gs_frame_forward_projected(const float* means3, const float* scales3, const float* quats4,
                               const float* opacities, const float* colors3, int64_t n, const gs_camera* cam,
                               const float* background3, int early_termination, int64_t isect_capacity, void* ws,
                               size_t ws_bytes, float* out_image, float* out_final_T, int32_t* out_n_contrib,
                               void* const* stage_events, gs_stream_t stream) {
    if (cam && binning_for(n, ((cam->width + TILE - 1) / TILE) * ((cam->height + TILE - 1) / TILE)) != DEPTH_FIRST)
        return set_error("gs_frame_forward_projected: the view does not use depth-first binning");
    return frame_forward_impl(means3, scales3, quats4, opacities, colors3, n, cam, background3, early_termination,
                              isect_capacity, ws, ws_bytes, out_image, out_final_T, out_n_contrib, nullptr,
                              stage_events, stream, true);
}

int gs_frames_project(const float* means3, const float* scales3, const float* quats4, const float* opacities,
                      int64_t n, int32_t n_views, const gs_camera* cams, const int64_t* capacities,
                      void* const* workspaces, const size_t* ws_bytes, gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_frames_project: n=%lld out of range", (long long)n);
    if (n_views < 0 || (n_views > 0 && (!cams || !capacities || !workspaces || !ws_bytes)))
        return set_error("gs_frames_project: bad view arrays");
    cudaStream_t s = (cudaStream_t)stream;
    for (int v0 = 0; v0 < n_views; v0 += MV_MAX) {
        MvFwdArgs a;
        a.nv = n_views - v0 < MV_MAX ? n_views - v0 : MV_MAX;
        for (int j = 0; j < a.nv; ++j) {
            const gs_camera& c = cams[v0 + j];
            if (c.width < 1 || c.height < 1) return set_error("gs_frames_project: bad image size");
            const int nt = ((c.width + TILE - 1) / TILE) * ((c.height + TILE - 1) / TILE);
            if (nt > 65536) return set_error("gs_frames_project: more than 65536 tiles");
            if (binning_for(n, nt) != DEPTH_FIRST)
                return set_error("gs_frames_project: view %d does not use depth-first binning", v0 + j);
            if (capacities[v0 + j] < 0 || capacities[v0 + j] >= (1ll << 30))
                return set_error("gs_frames_project: capacity out of range");
            const Layout L = layout(n, capacities[v0 + j], c.width, c.height);
            if (ws_bytes[v0 + j] < L.total) return set_error("gs_frames_project: workspace %d too small", v0 + j);
            void* ws = workspaces[v0 + j];
            MvFwdView& V = a.v[j];
            V.cam = make_camk(c);
            V.xydr = at<float4>(ws, L.xydr);
            V.conic = at<float4>(ws, L.conic);
            V.tiles = at<uint32_t>(ws, L.tiles);
            V.dkeys = at<uint32_t>(ws, L.dkeys);
            V.dhist = at<uint32_t>(ws, L.dhist);
            V.meta = at<unsigned long long>(ws, L.meta);
            V.clean_word = at<unsigned long long>(ws, L.clean);
            V.clean_sig = clean_sig(n, capacities[v0 + j], c.width, c.height);
            V.zj = frame_zero_jobs(L, ws, n, nt, !uses_tile_emit(n, nt));
        }
        if (launch_views_project_fwd(means3, scales3, quats4, opacities, n, a, s)) return -1;
    }
    return 0;
}

}  // extern "C"

namespace gs {
namespace {

int frame_forward_impl(const float* means3, const float* scales3, const float* quats4, const float* opacities,
                       const float* colors3, int64_t n, const gs_camera* cam, const float* background3,
                       int early_termination, int64_t isect_capacity, void* ws, size_t ws_bytes, float* out_image,
                       float* out_final_T, int32_t* out_n_contrib, unsigned long long* counts4,
                       void* const* stage_events, gs_stream_t stream, bool projected) {
    if (!cam || !background3) return set_error("gs_frame_forward: null camera/background");
    if (n < 0 || n > 0x7fffffff) return set_error("gs_frame_forward: n=%lld out of range", (long long)n);
    if (isect_capacity < 0 || isect_capacity >= (1ll << 30))
        return set_error("gs_frame_forward: capacity %lld out of range", (long long)isect_capacity);
    if (cam->width < 1 || cam->height < 1) return set_error("gs_frame_forward: bad image size");
    const int W = cam->width, H = cam->height;
    const int tiles_x = (W + TILE - 1) / TILE, tiles_y = (H + TILE - 1) / TILE;
    if ((int64_t)tiles_x * tiles_y > 65536) return set_error("gs_frame_forward: more than 65536 tiles");
    const Layout L = layout(n, isect_capacity, W, H);
    if (ws_bytes < L.total) return set_error("gs_frame_forward: workspace %zu < %zu", ws_bytes, L.total);
    cudaStream_t s = (cudaStream_t)stream;
    const CamK k = make_camk(*cam);
    const int tp = tile_passes_for(tiles_x * tiles_y);
    unsigned long long* meta = at<unsigned long long>(ws, L.meta);
    uint32_t* counters = at<uint32_t>(ws, L.counters);

    mark(stage_events, 0, s);
    // 1. projection + depth keys.  No memset nodes: a one-CTA init kernel
    // resets meta and the depth histograms, and the projection kernel clears
    // the later stages' counters / look-back status / tile ranges and the
    // backward's screen-space accumulators (zeroed here, once per forward).
    const int n_tiles = tiles_x * tiles_y;
    const Binning binning = binning_for(n, n_tiles);
    // depth-first binning with the tile-sorted emission (no global sort by tile)
    const bool etiles = uses_tile_emit(n, n_tiles);
    const ZeroJobs zj = frame_zero_jobs(L, ws, n, n_tiles, binning == DEPTH_FIRST && !etiles);
    const bool scatter = binning == SCATTER;
    const bool direct = binning == DIRECT && counts4 == nullptr;  // the counted pass bins by scatter
    const int64_t kstride = direct_stride(isect_capacity, n_tiles);
    const uint32_t* t_order = !direct && tile_order_enabled(n_tiles) ? at<uint32_t>(ws, L.tile_order) : nullptr;
    // projected: gs_frames_project already projected this view (with every other view of the step)
    if (!projected &&
        launch_project_fwd_dkey(means3, scales3, quats4, opacities, n, k, at<float>(ws, L.xydr),
                                at<float>(ws, L.conic), at<uint32_t>(ws, L.tiles), nullptr, meta,
                                at<uint32_t>(ws, L.dkeys), at<uint32_t>(ws, L.dhist), s, zj,
                                binning != DEPTH_FIRST ? at<uint32_t>(ws, L.tcount) : nullptr,
                                direct ? at<uint32_t>(ws, L.tvals) : nullptr, (uint32_t)kstride,
                                at<unsigned long long>(ws, L.clean), clean_sig(n, isect_capacity, W, H)))
        return -1;
    mark(stage_events, 1, s);
    const float3 bg = make_float3(background3[0], background3[1], background3[2]);
    if (direct) {
        // 2-6. direct binning: the projection wrote every pair into its
        //      tile's fixed-stride bin; the raster forward sorts each bin
        //      by (depth, index) first and reports the counts
        mark(stage_events, 2, s);
        mark(stage_events, 3, s);
        mark(stage_events, 4, s);
        if (launch_raster_fwd(at<uint2>(ws, L.ranges), at<uint32_t>(ws, L.tvals), at<float>(ws, L.xydr),
                              at<float>(ws, L.conic), colors3, bg, W, H, early_termination != 0, out_image,
                              out_final_T, out_n_contrib, nullptr, s, at<uint2>(ws, L.rec),
                              at<uint32_t>(ws, L.rec_count), nullptr, at<uint32_t>(ws, L.dkeys),
                              at<uint32_t>(ws, L.tvals_alt), at<uint32_t>(ws, L.tcount), (uint32_t)kstride, meta))
            return -1;
        mark(stage_events, 5, s);
        return 0;
    }
    if (binning != DEPTH_FIRST) {
        // 2-6. scatter binning: the projection counted every tile's pairs;
        //      scan -> ranges + cursors (+ raster order), scatter the pairs
        //      into their ranges, sort each range by (depth, index)
        mark(stage_events, 2, s);
        uint32_t* tcount = at<uint32_t>(ws, L.tcount);
        if (launch_tile_scan(tcount, n_tiles, isect_capacity, at<uint2>(ws, L.ranges), meta + 1,
                             const_cast<uint32_t*>(t_order), s))
            return -1;
        if (launch_scatter_pairs(at<float>(ws, L.xydr), at<uint32_t>(ws, L.tiles), n, tiles_x, tiles_y,
                                 isect_capacity, tcount, at<uint32_t>(ws, L.tkeys), at<uint32_t>(ws, L.tvals), s))
            return -1;
        mark(stage_events, 3, s);
        // per-tile sort at the top of the raster forward (the counted pass keeps the separate kernel)
        const bool fused = fuse_sort() && counts4 == nullptr;
        if (!fused && launch_segsort(at<uint2>(ws, L.ranges), n_tiles, at<uint32_t>(ws, L.dkeys),
                                     at<uint32_t>(ws, L.tvals), at<uint32_t>(ws, L.tvals_alt), s))
            return -1;
        mark(stage_events, 4, s);
        if (launch_raster_fwd(at<uint2>(ws, L.ranges), at<uint32_t>(ws, L.tvals), at<float>(ws, L.xydr),
                              at<float>(ws, L.conic), colors3, bg, W, H, early_termination != 0, out_image,
                              out_final_T, out_n_contrib, counts4, s, at<uint2>(ws, L.rec),
                              at<uint32_t>(ws, L.rec_count), t_order, fused ? at<uint32_t>(ws, L.dkeys) : nullptr,
                              fused ? at<uint32_t>(ws, L.tvals_alt) : nullptr))
            return -1;
        mark(stage_events, 5, s);
        return 0;
    }
    // 2. depth-first: stable depth sort of the visible Gaussians (keys relative
    //    to the visible minimum, culled ones dropped by the first pass, only the
    //    passes the key width needs; the order ends in `order_alt` after an odd
    //    pass count, meta[8])
    if (run_depth_sort(at<uint32_t>(ws, L.dkeys), at<uint32_t>(ws, L.order), at<uint32_t>(ws, L.dkeys_alt),
                       at<uint32_t>(ws, L.order_alt), n, meta, at<uint32_t>(ws, L.dhist), at<uint32_t>(ws, L.dstatus),
                       counters, s))
        return -1;
    const uint32_t* order = at<uint32_t>(ws, L.order);
    mark(stage_events, 2, s);
    if (etiles) {
        // 3. per-(chunk of the depth order, tile) pair counts, their column
        //    prefixes and the tiles' totals -> ranges (+ total -> meta[1],
        //    raster order)
        uint32_t* totals = at<uint32_t>(ws, L.tcount);
        if (launch_emit_tiles_count(order, at<uint32_t>(ws, L.order_alt), at<float>(ws, L.xydr), n, tiles_x, tiles_y,
                                    isect_capacity, at<char>(ws, L.etable), totals, at<uint32_t>(ws, L.tkeys),
                                    at<char>(ws, L.scan_ws), meta, s))
            return -1;
        if (launch_tile_scan(totals, n_tiles, isect_capacity, at<uint2>(ws, L.ranges), meta + 1,
                             const_cast<uint32_t*>(t_order), s, 1))
            return -1;
        mark(stage_events, 3, s);
        // 4. every pair straight to its slot, tile lists in (depth, index) order
        if (launch_emit_tiles(order, at<uint32_t>(ws, L.order_alt), n, tiles_x, tiles_y, isect_capacity, totals,
                              at<char>(ws, L.etable), at<uint32_t>(ws, L.tkeys), at<uint32_t>(ws, L.tvals), meta, s))
            return -1;
        mark(stage_events, 4, s);
        if (launch_raster_fwd(at<uint2>(ws, L.ranges), at<uint32_t>(ws, L.tvals), at<float>(ws, L.xydr),
                              at<float>(ws, L.conic), colors3, bg, W, H, early_termination != 0, out_image,
                              out_final_T, out_n_contrib, counts4, s, at<uint2>(ws, L.rec),
                              at<uint32_t>(ws, L.rec_count), t_order))
            return -1;
        mark(stage_events, 5, s);
        return 0;
    }
    // 3+4. fused: scan of the tile counts (in depth order), total ->
    //      meta[1], emission of the (tile, gaussian) pairs + tile-digit histograms
    // (an odd number of tile passes starts from the alternate buffers, so the
    // sorted pairs always end in the primary ones)
    const bool odd = tp & 1;
    uint32_t* k0 = at<uint32_t>(ws, odd ? L.tkeys_alt : L.tkeys);
    uint32_t* v0 = at<uint32_t>(ws, odd ? L.tvals_alt : L.tvals);
    uint32_t* k1 = at<uint32_t>(ws, odd ? L.tkeys : L.tkeys_alt);
    uint32_t* v1 = at<uint32_t>(ws, odd ? L.tvals : L.tvals_alt);
    if (launch_emit_scan(order, at<float>(ws, L.xydr), at<uint32_t>(ws, L.tiles), n, tiles_x, tiles_y,
                         isect_capacity, k0, v0, at<uint32_t>(ws, L.thist), tp, at<char>(ws, L.scan_ws), meta + 1, s,
                         at<uint32_t>(ws, L.order_alt), meta + 7))
        return -1;
    mark(stage_events, 3, s);
    // 5. stable sort by tile id (bits [0, 8*tp))
    if (run_onesweep<uint32_t>(k0, v0, k1, v1, isect_capacity, meta + 1, tp, at<uint32_t>(ws, L.thist),
                               at<uint32_t>(ws, L.tstatus), counters + 4, s, false))
        return -1;
    const uint32_t* skeys = at<uint32_t>(ws, L.tkeys);
    const uint32_t* svals = at<uint32_t>(ws, L.tvals);
    // 6. per-tile ranges
    if (launch_ranges_u32(skeys, isect_capacity, meta + 1, at<uint2>(ws, L.ranges), s)) return -1;
    // 6b. heaviest-first raster launch order
    if (t_order && launch_tile_order(at<uint2>(ws, L.ranges), n_tiles, at<uint32_t>(ws, L.tile_order), s))
        return -1;
    mark(stage_events, 4, s);
    // 7. raster forward
    if (launch_raster_fwd(at<uint2>(ws, L.ranges), svals, at<float>(ws, L.xydr), at<float>(ws, L.conic), colors3,
                          bg, W, H, early_termination != 0, out_image, out_final_T, out_n_contrib, counts4, s,
                          at<uint2>(ws, L.rec), at<uint32_t>(ws, L.rec_count), t_order))
        return -1;
    mark(stage_events, 5, s);
    return 0;
}

}  // namespace
}  // namespace gs

extern "C" {

int gs_frame_backward(const float* means3, const float* scales3, const float* quats4, const float* colors3,
                      int64_t n, const gs_camera* cam, const float* background3, int64_t isect_capacity, void* ws,
                      size_t ws_bytes, const float* final_T, const int32_t* n_contrib, const float* d_image,
                      float* d_means3, float* d_scales3, float* d_quats4, float* d_rgbo4, float* d_view16,
                      int accumulate, unsigned long long* counts3, void* const* stage_events, gs_stream_t stream) {
    if (!cam || !background3) return set_error("gs_frame_backward: null camera/background");
    const int W = cam->width, H = cam->height;
    const Layout L = layout(n, isect_capacity, W, H);
    if (ws_bytes < L.total) return set_error("gs_frame_backward: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const CamK k = make_camk(*cam);
    const int tiles_x = (W + TILE - 1) / TILE, tiles_y = (H + TILE - 1) / TILE;
    const uint32_t* svals = at<uint32_t>(ws, L.tvals);
    mark(stage_events, 0, s);
    // the screen-space accumulators are zero here: the previous backward's
    // projection backward cleared the rows it read, or gs_frame_forward zeroed
    // them (meta[4]) when the workspace was not stamped clean for this layout
    const float3 bg = make_float3(background3[0], background3[1], background3[2]);
    float* g8 = at<float>(ws, L.d_geo);
    if (counts3) {  // counted pass (roofline numerators): the list-walking backward counts evaluations
        if (launch_raster_bwd(at<uint2>(ws, L.ranges), svals, at<float>(ws, L.xydr), at<float>(ws, L.conic),
                              colors3, bg, W, H, final_T, n_contrib, d_image, g8, g8 + 4, at<float>(ws, L.d_c11),
                              counts3, s, 2))
            return -1;
        // the list-walking backward does not mark the Gaussians it adds to: all count as touched
        if (cudaMemsetAsync(at<uint32_t>(ws, L.touched), 0xFF, 4 * ((n + 31) / 32), s) != cudaSuccess)
            return set_error("gs_frame_backward: memset failed");
    } else if (launch_raster_bwd_rec(at<uint2>(ws, L.ranges), at<uint2>(ws, L.rec), at<uint32_t>(ws, L.rec_count),
                                     at<float>(ws, L.xydr), at<float>(ws, L.conic), colors3, bg, W, H, final_T,
                                     n_contrib, d_image, g8, at<float>(ws, L.d_c11), s,
                                     tile_order_enabled(tiles_x * tiles_y) ? at<uint32_t>(ws, L.tile_order) : nullptr,
                                     at<unsigned long long>(ws, L.meta), at<uint32_t>(ws, L.touched))) {
        return -1;
    }
    mark(stage_events, 1, s);
    // accumulate bit 0: add into the outputs; bit 1: keep the screen-space
    // gradients in the workspace (gs_frame_view.d_geo4 / d_c11) -- the next
    // forward then re-zeroes them; bit 2: stage_events[3] is an event this
    // stream waits on before the projection backward -- a multi-view step
    // orders only the views' read-modify-write accumulation, so one view's
    // raster backward (its own workspace) overlaps the previous view's
    // projection backward
    const bool keep = (accumulate & 2) != 0;
    if (accumulate & 8) {
        // raster backward only: the screen-space gradients stay in the
        // workspace for a reduction across ranks (tile bands) and
        // gs_frame_project_backward; until then the accumulators are dirty
        if (cudaMemsetAsync(at<char>(ws, L.clean), 0, 8, s) != cudaSuccess)
            return check_launch("gs_frame_backward: clean word");
        mark(stage_events, 2, s);
        return 0;
    }
    if ((accumulate & 4) && stage_events && stage_events[3] &&
        cudaStreamWaitEvent(s, (cudaEvent_t)stage_events[3], 0) != cudaSuccess)
        return check_launch("gs_frame_backward: wait event");
    if (launch_project_bwd(means3, scales3, quats4, n, k, at<uint32_t>(ws, L.tiles), g8 + 4,
                           at<float>(ws, L.d_c11), d_means3, d_scales3, d_quats4, d_view16, at<float>(ws, L.partials),
                           s, (accumulate & 1) != 0, 2, g8, d_rgbo4, at<unsigned int>(ws, L.pbwd_done),
                           at<unsigned long long>(ws, L.clean), clean_sig(n, isect_capacity, W, H), !keep))
        return -1;
    mark(stage_events, 2, s);
    return 0;
}

int gs_frame_project_backward(const float* means3, const float* scales3, const float* quats4, int64_t n,
                              const gs_camera* cam, int64_t isect_capacity, void* ws, size_t ws_bytes, int64_t begin,
                              int64_t end, float* d_means3, float* d_scales3, float* d_quats4, float* d_rgbo4,
                              float* d_view16, int flags, gs_stream_t stream) {
    if (!cam) return set_error("gs_frame_project_backward: null camera");
    if (begin < 0 || end > n || begin > end)
        return set_error("gs_frame_project_backward: range [%lld, %lld) outside [0, %lld)", (long long)begin,
                         (long long)end, (long long)n);
    const int W = cam->width, H = cam->height;
    const Layout L = layout(n, isect_capacity, W, H);
    if (ws_bytes < L.total) return set_error("gs_frame_project_backward: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const CamK k = make_camk(*cam);
    float* g8 = at<float>(ws, L.d_geo) + 8 * begin;
    const bool keep = (flags & 2) != 0;
    return launch_project_bwd(means3 + 3 * begin, scales3 + 3 * begin, quats4 + 4 * begin, end - begin, k,
                              at<uint32_t>(ws, L.tiles) + begin, g8 + 4, at<float>(ws, L.d_c11) + begin,
                              d_means3 + 3 * begin, d_scales3 + 3 * begin, d_quats4 + 4 * begin, d_view16,
                              at<float>(ws, L.partials), s, (flags & 1) != 0, 2, g8, d_rgbo4 + 4 * begin, nullptr,
                              at<unsigned long long>(ws, L.clean), clean_sig(n, isect_capacity, W, H), !keep,
                              (flags & 16) != 0, (flags & 32) != 0);
}

int gs_frame_views_project_backward(const float* means3, const float* scales3, const float* quats4, int64_t n,
                                    int32_t n_views, const gs_camera* cams, const int64_t* capacities,
                                    void* const* workspaces, const size_t* ws_bytes, int64_t begin, int64_t end,
                                    float* d_means3, float* d_scales3, float* d_quats4, float* d_rgbo4,
                                    float* d_views16, int flags, gs_stream_t stream) {
    if (n_views < 0 || (n_views > 0 && (!cams || !capacities || !workspaces || !ws_bytes)))
        return set_error("gs_frame_views_project_backward: bad view arrays");
    if (begin < 0 || end > n || begin > end)
        return set_error("gs_frame_views_project_backward: range [%lld, %lld) outside [0, %lld)", (long long)begin,
                         (long long)end, (long long)n);
    cudaStream_t s = (cudaStream_t)stream;
    const bool keep = (flags & 2) != 0;
    for (int v0 = 0; v0 < n_views; v0 += MV_MAX) {
        MvArgs a;
        a.nv = n_views - v0 < MV_MAX ? n_views - v0 : MV_MAX;
        for (int j = 0; j < a.nv; ++j) {
            const gs_camera& c = cams[v0 + j];
            const Layout L = layout(n, capacities[v0 + j], c.width, c.height);
            if (ws_bytes[v0 + j] < L.total)
                return set_error("gs_frame_views_project_backward: workspace %d too small", v0 + j);
            void* ws = workspaces[v0 + j];
            MvView& V = a.v[j];
            V.cam = make_camk(c);
            V.g8 = at<float4>(ws, L.d_geo) + 2 * begin;
            V.d_c11 = at<float>(ws, L.d_c11) + begin;
            V.touched = at<uint32_t>(ws, L.touched);
            V.tbase = (int)begin;
            V.partials = at<float>(ws, L.partials);
            // the call whose range ends at n declares the workspace's rows clear (the
            // earlier ranges' calls cleared theirs) or, keeping its rows, dirty
            V.clean_word = end == n ? at<unsigned long long>(ws, L.clean) : nullptr;
            V.clean_stamp = keep ? 0ull : clean_sig(n, capacities[v0 + j], c.width, c.height);
        }
        if (launch_views_project_bwd(means3 + 3 * begin, scales3 + 3 * begin, quats4 + 4 * begin, end - begin, a,
                                     d_means3 + 3 * begin, d_scales3 + 3 * begin, d_quats4 + 4 * begin,
                                     d_rgbo4 + 4 * begin, d_views16 + 16 * v0, (flags & 1) != 0 || v0 > 0, !keep,
                                     (flags & 16) != 0, s))
            return -1;
    }
    return 0;
}

}  // extern "C"
