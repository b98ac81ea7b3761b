// abi.cu -- error plumbing and device queries of the C ABI.
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <cstdio>

#include "common.cuh"

namespace gs {

static thread_local char g_last_error[512] = "";

int set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
    return -1;
}

bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GS_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

static int g_binning = -1;  // -1: not set (env GS_BINNING, else auto)

int binning_mode() {
    if (g_binning < 0) {
        const char* e = getenv("GS_BINNING");
        g_binning = e ? atoi(e) : 0;
    }
    return g_binning;
}

static int g_fuse_sort = -1;  // -1: not set (env GS_FUSE_SORT, else on)

bool fuse_sort() {
    if (g_fuse_sort < 0) {
        const char* e = getenv("GS_FUSE_SORT");
        g_fuse_sort = (e && e[0] == '0') ? 0 : 1;
    }
    return g_fuse_sort == 1;
}

static int g_tile_emit = -1;  // -1: not set (env GS_TILE_EMIT, else on)

bool tile_emit() {
    if (g_tile_emit < 0) {
        const char* e = getenv("GS_TILE_EMIT");
        g_tile_emit = (e && e[0] == '0') ? 0 : 1;
    }
    return g_tile_emit == 1;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error("%s: %s", what, cudaGetErrorString(e));
    return 0;
}

}  // namespace gs

extern "C" {

const char* gs_last_error(void) { return gs::g_last_error; }

int gs_version(void) { return 1; }

int gs_set_option(const char* name, int value) {
    if (!name) return gs::set_error("gs_set_option: null name");
    if (strcmp(name, "binning") == 0) {
        if (value < 0 || value > 3) return gs::set_error("gs_set_option: binning must be 0 (auto), 1, 2 or 3");
        gs::g_binning = value;
        return 0;
    }
    if (strcmp(name, "fuse_sort") == 0) {
        if (value < 0 || value > 1) return gs::set_error("gs_set_option: fuse_sort must be 0 or 1");
        gs::g_fuse_sort = value;
        return 0;
    }
    if (strcmp(name, "tile_emit") == 0) {
        if (value < 0 || value > 1) return gs::set_error("gs_set_option: tile_emit must be 0 or 1");
        gs::g_tile_emit = value;
        return 0;
    }
    return gs::set_error("gs_set_option: unknown option %s", name);
}

int gs_get_option(const char* name) {
    if (!name) return gs::set_error("gs_get_option: null name");
    if (strcmp(name, "binning") == 0) return gs::binning_mode();
    if (strcmp(name, "fuse_sort") == 0) return gs::fuse_sort() ? 1 : 0;
    if (strcmp(name, "tile_emit") == 0) return gs::tile_emit() ? 1 : 0;
    return gs::set_error("gs_get_option: unknown option %s", name);
}

int gs_device_sm_count(void) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return sms;
}

}  // extern "C"
