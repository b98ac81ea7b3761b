/*
 * splat_oracle.c -- fp64 CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_2312_02121_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links or calls it.
 *
 * It restates, in plain C and float64 like the reference, the
 * algorithm of the `splatgrad` package under /root/reference/pkg/src/splatgrad
 * (abbreviated sg/ below).  Every function cites the reference lines it
 * follows.  It is pinned against golden vectors produced by running the
 * reference itself (tests/golden/make_golden.py writes tests/golden/NAME.npz, checked
 * by tests/test_oracle_golden.py).
 *
 * Parallelism: OpenMP over Gaussians (projection, projection backward) and
 * over tiles (raster forward/backward).  Backward accumulators are private per
 * thread and merged in thread order, so a run is deterministic for a given
 * thread count (the reference is single-threaded, sg/raster_backward.py:176).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_TILE 16                    /* sg/binning.py:8 */
#define ORC_DILATION 0.3               /* sg/projection.py:17 */
#define ORC_ALPHA_MIN (1.0 / 255.0)    /* sg/raster_forward.py:21 */
#define ORC_ALPHA_MAX 0.999            /* sg/raster_forward.py:22 */
#define ORC_T_MIN 1e-4                 /* sg/raster_forward.py:25 */
#define ORC_SIGMA_CUT 4.5              /* sg/raster_forward.py:30 */
#define ORC_QUAT_EPS 1e-12             /* sg/core.py:13 */

/* error codes shared with the CUDA status word (include/splat_b200.h) */
#define ORC_OK 0
#define ORC_ERR_SCALE 1   /* sg/core.py:189-191  "scale components must be positive" */
#define ORC_ERR_QUAT 2    /* sg/core.py:160-163  "quaternion norm is too small ..." */
#define ORC_ERR_HOMOG 3   /* sg/projection.py:54-55 "degenerate projection" */
#define ORC_ERR_COV2D 4   /* sg/projection.py:108-109 "2d covariance must be positive definite" */

typedef struct orc_camera {
    double view[16]; /* row-major world->camera, sg/core.py:59-129 */
    double fx, fy, cx, cy;
    int64_t width, height;
    double near_plane, far_plane;
} orc_camera;

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* sg/core.py:146-171 quat_to_rotmat on the normalised quaternion (w,x,y,z). */
static int quat_to_rotmat(const double q[4], double R[9], double qhat[4], double* norm_out) {
    double norm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (norm <= ORC_QUAT_EPS) return ORC_ERR_QUAT;
    double w = q[0] / norm, x = q[1] / norm, y = q[2] / norm, z = q[3] / norm;
    R[0] = 1.0 - 2.0 * (y * y + z * z); R[1] = 2.0 * (x * y - w * z); R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z); R[4] = 1.0 - 2.0 * (x * x + z * z); R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y); R[7] = 2.0 * (y * z + w * x); R[8] = 1.0 - 2.0 * (x * x + y * y);
    if (qhat) { qhat[0] = w; qhat[1] = x; qhat[2] = y; qhat[3] = z; }
    if (norm_out) *norm_out = norm;
    return ORC_OK;
}

/* sg/core.py:174-195 compose_covariance_3d: M = R diag(s), Sigma = M M^T.
 * The scale check precedes the quaternion check (sg/core.py:189-192). */
static int compose_cov3d(const double q[4], const double s[3], double R[9], double M[9], double Sig[9],
                         double qhat[4], double* qnorm) {
    /* np.any(s <= 0.0): NaN passes, like the reference */
    if (s[0] <= 0.0 || s[1] <= 0.0 || s[2] <= 0.0) return ORC_ERR_SCALE;
    int e = quat_to_rotmat(q, R, qhat, qnorm);
    if (e) return e;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) M[3 * i + j] = R[3 * i + j] * s[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            Sig[3 * i + j] = M[3 * i + 0] * M[3 * j + 0] + M[3 * i + 1] * M[3 * j + 1] + M[3 * i + 2] * M[3 * j + 2];
    return ORC_OK;
}

/* sg/projection.py:64-82 projection_jacobian (2x3, row-major). */
static void jacobian(const double t[4], const orc_camera* c, double J[6]) {
    double tx = t[0], ty = t[1], tz = t[2];
    J[0] = c->fx / tz; J[1] = 0.0; J[2] = -c->fx * tx / (tz * tz);
    J[3] = 0.0; J[4] = c->fy / tz; J[5] = -c->fy * ty / (tz * tz);
}

/* sg/core.py:97-111 projection_matrix (4x4 row-major). */
static void proj_matrix(const orc_camera* c, double P[16]) {
    double n = c->near_plane, f = c->far_plane;
    memset(P, 0, 16 * sizeof(double));
    P[0] = 2.0 * c->fx / (double)c->width;
    P[5] = 2.0 * c->fy / (double)c->height;
    P[10] = (f + n) / (f - n);
    P[11] = -2.0 * f * n / (f - n);
    P[14] = 1.0;
}

/*
 * sg/projection.py:115-145 project_gaussian, batched like
 * sg/raster_forward.py:246-252 _project_scene (visible[i] = 1 for the
 * members of the compacted `projected` list, in source order).
 * Outputs per scene Gaussian: t_cam(4), mean2d(2), cov2d (a, b, c) of the
 * symmetric 2x2, depth, radius.  Returns the first error code in source
 * order (the reference raises at the first offending Gaussian) and its index.
 */
int orc_project(int64_t n, const double* means, const double* scales, const double* quats,
                const orc_camera* cam, int8_t* visible, double* t_cam, double* mean2d, double* cov2d,
                double* depth, int64_t* radius, int64_t* err_index, int nthreads) {
    set_threads(nthreads);
    int64_t first_err = n;
    int first_code = ORC_OK;
    double P[16];
    proj_matrix(cam, P);
    const double* V = cam->view;
#pragma omp parallel
    {
        int64_t my_err = n;
        int my_code = ORC_OK;
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            const double* m = means + 3 * i;
            double t[4];
            /* sg/projection.py:36-42 world_to_camera */
            for (int r = 0; r < 4; ++r) t[r] = V[4 * r + 0] * m[0] + V[4 * r + 1] * m[1] + V[4 * r + 2] * m[2] + V[4 * r + 3];
            visible[i] = 0;
            radius[i] = 0;
            for (int r = 0; r < 4; ++r) t_cam[4 * i + r] = t[r];
            double d = t[2];
            depth[i] = d;
            mean2d[2 * i] = mean2d[2 * i + 1] = 0.0;
            cov2d[3 * i] = cov2d[3 * i + 1] = cov2d[3 * i + 2] = 0.0;
            if (d <= cam->near_plane || d >= cam->far_plane) continue; /* :124-125 */
            double R[9], M[9], S[9];
            int e = compose_cov3d(quats + 4 * i, scales + 3 * i, R, M, S, NULL, NULL);
            if (e) { if (i < my_err) { my_err = i; my_code = e; } continue; }
            double J[6];
            jacobian(t, cam, J);
            /* sg/projection.py:85-96 project_covariance: T = J R_cw */
            double T[6];
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 3; ++b)
                    T[3 * a + b] = J[3 * a + 0] * V[0 * 4 + b] + J[3 * a + 1] * V[1 * 4 + b] + J[3 * a + 2] * V[2 * 4 + b];
            double TS[6];
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 3; ++b)
                    TS[3 * a + b] = T[3 * a + 0] * S[0 * 3 + b] + T[3 * a + 1] * S[1 * 3 + b] + T[3 * a + 2] * S[2 * 3 + b];
            double c00 = TS[0] * T[0] + TS[1] * T[1] + TS[2] * T[2];
            double c01 = TS[0] * T[3] + TS[1] * T[4] + TS[2] * T[5];
            double c11 = TS[3] * T[3] + TS[4] * T[4] + TS[5] * T[5];
            c00 += ORC_DILATION;
            c11 += ORC_DILATION;
            /* sg/projection.py:45-61 camera_to_pixel through P */
            double tp[4];
            for (int r = 0; r < 4; ++r) tp[r] = P[4 * r + 0] * t[0] + P[4 * r + 1] * t[1] + P[4 * r + 2] * t[2] + P[4 * r + 3] * t[3];
            double tw = tp[3];
            if (fabs(tw) < 1e-12) { if (i < my_err) { my_err = i; my_code = ORC_ERR_HOMOG; } continue; }
            double mx = ((double)cam->width * tp[0] / tw + 1.0) / 2.0 + cam->cx;
            double my = ((double)cam->height * tp[1] / tw + 1.0) / 2.0 + cam->cy;
            /* sg/projection.py:99-112 bounding_radius */
            double det = c00 * c11 - c01 * c01;
            if (!(det > 0.0 && c00 + c11 > 0.0)) { if (i < my_err) { my_err = i; my_code = ORC_ERR_COV2D; } continue; }
            double mid = 0.5 * (c00 + c11);
            double lam = mid + sqrt(0.25 * (c00 - c11) * (c00 - c11) + c01 * c01);
            int64_t r = (int64_t)ceil(3.0 * sqrt(lam));
            mean2d[2 * i] = mx;
            mean2d[2 * i + 1] = my;
            cov2d[3 * i] = c00; cov2d[3 * i + 1] = c01; cov2d[3 * i + 2] = c11;
            radius[i] = r;
            /* sg/projection.py:131-137 off-screen cull */
            if (mx + (double)r < 0.0 || mx - (double)r >= (double)cam->width ||
                my + (double)r < 0.0 || my - (double)r >= (double)cam->height)
                continue;
            visible[i] = 1;
        }
#pragma omp critical
        {
            if (my_err < first_err) { first_err = my_err; first_code = my_code; }
        }
    }
    *err_index = first_err < n ? first_err : -1;
    return first_code;
}

/* sg/binning.py:35-46 tile rectangle of one splat (closed square vs
 * half-open tiles).  floor((m -/+ r)/16) in fp64 exactly like the reference. */
static void tile_rect(double mx, double my, int64_t r, int64_t tiles_x, int64_t tiles_y,
                      int64_t* tx0, int64_t* tx1, int64_t* ty0, int64_t* ty1) {
    int64_t a = (int64_t)floor((mx - (double)r) / ORC_TILE);
    int64_t b = (int64_t)floor((mx + (double)r) / ORC_TILE);
    int64_t c = (int64_t)floor((my - (double)r) / ORC_TILE);
    int64_t d = (int64_t)floor((my + (double)r) / ORC_TILE);
    *tx0 = a < 0 ? 0 : a;
    *tx1 = b > tiles_x - 1 ? tiles_x - 1 : b;
    *ty0 = c < 0 ? 0 : c;
    *ty1 = d > tiles_y - 1 ? tiles_y - 1 : d;
}

/* Count pass of sg/binning.py:27-47 assign_tiles: bin_count[tile]. Returns I. */
int64_t orc_bin_count(int64_t n, const int8_t* visible, const double* mean2d, const int64_t* radius,
                      int64_t width, int64_t height, int64_t* bin_count) {
    int64_t tiles_x = (width + ORC_TILE - 1) / ORC_TILE, tiles_y = (height + ORC_TILE - 1) / ORC_TILE;
    memset(bin_count, 0, (size_t)(tiles_x * tiles_y) * sizeof(int64_t));
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!visible[i]) continue;
        int64_t tx0, tx1, ty0, ty1;
        tile_rect(mean2d[2 * i], mean2d[2 * i + 1], radius[i], tiles_x, tiles_y, &tx0, &tx1, &ty0, &ty1);
        for (int64_t ty = ty0; ty <= ty1; ++ty)
            for (int64_t tx = tx0; tx <= tx1; ++tx) { bin_count[ty * tiles_x + tx]++; total++; }
    }
    return total;
}

static const double* g_sort_depth;
static int cmp_depth_index(const void* pa, const void* pb) {
    int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    double da = g_sort_depth[a], db = g_sort_depth[b];
    if (da < db) return -1;
    if (da > db) return 1;
    return (a > b) - (a < b);
}

/*
 * sg/binning.py:27-47 assign_tiles (append order = source order) followed by
 * sg/binning.py:50-65 sort_bins (key (depth, source_index)) when `sort` != 0.
 * Bins are CSR: bin_ptr[tiles+1], bin_idx[I] holding SCENE indices.
 */
void orc_bin_fill(int64_t n, const int8_t* visible, const double* mean2d, const int64_t* radius,
                  const double* depth, int64_t width, int64_t height, const int64_t* bin_count,
                  int64_t* bin_ptr, int64_t* bin_idx, int sort) {
    int64_t tiles_x = (width + ORC_TILE - 1) / ORC_TILE, tiles_y = (height + ORC_TILE - 1) / ORC_TILE;
    int64_t nt = tiles_x * tiles_y;
    bin_ptr[0] = 0;
    for (int64_t t = 0; t < nt; ++t) bin_ptr[t + 1] = bin_ptr[t] + bin_count[t];
    int64_t* fill = (int64_t*)calloc((size_t)nt, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        if (!visible[i]) continue;
        int64_t tx0, tx1, ty0, ty1;
        tile_rect(mean2d[2 * i], mean2d[2 * i + 1], radius[i], tiles_x, tiles_y, &tx0, &tx1, &ty0, &ty1);
        for (int64_t ty = ty0; ty <= ty1; ++ty)
            for (int64_t tx = tx0; tx <= tx1; ++tx) {
                int64_t b = ty * tiles_x + tx;
                bin_idx[bin_ptr[b] + fill[b]++] = i;
            }
    }
    free(fill);
    if (sort) {
        g_sort_depth = depth;
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t t = 0; t < nt; ++t)
            qsort(bin_idx + bin_ptr[t], (size_t)(bin_ptr[t + 1] - bin_ptr[t]), sizeof(int64_t), cmp_depth_index);
    }
}

/* sg/raster_forward.py:86-92 _cov2d_inverse_terms. */
static void conic_of(const double* cov, double* A, double* B, double* C) {
    double a = cov[0], b = cov[1], c = cov[2];
    double det = a * c - b * b;
    *A = c / det; *B = -b / det; *C = a / det;
}

static inline double rel_margin(double v, double thr) { return fabs(v - thr) / fabs(thr); }

/*
 * sg/raster_forward.py:116-154 _composite_tile over every tile
 * (sg/raster_forward.py:157-172 _iter_tiles, :222-243 _render_with_grid).
 * mean2d/cov2d/opac/colors are indexed by SCENE index (bins hold scene ids).
 * Optional outputs:
 *   margin[H*W]  -- minimum relative distance of any decision this pixel
 *                   evaluated (sigma<=4.5, alpha>=1/255, o*e^-s vs 0.999,
 *                   nT<1e-4) to its threshold; a pixel whose GPU fp32 value
 *                   disagrees AND whose margin is tiny is a branch-flip case.
 *   margin_pos[H*W] -- bin position of that decision, margin_kind[H*W] which.
 *   counts[4]    -- E_f, E_f_sigma, E_f_alpha, E_f_commit.
 */
void orc_raster_fwd(int64_t width, int64_t height, const int64_t* bin_ptr, const int64_t* bin_idx,
                    const double* mean2d, const double* cov2d, const double* opac, const double* colors,
                    const double* bg, int early_termination, double* image, double* final_T,
                    int64_t* n_contrib, double* margin, int64_t* margin_pos, int8_t* margin_kind,
                    int64_t* counts, int nthreads) {
    set_threads(nthreads);
    int64_t tiles_x = (width + ORC_TILE - 1) / ORC_TILE, tiles_y = (height + ORC_TILE - 1) / ORC_TILE;
    int64_t nt = tiles_x * tiles_y;
    int64_t c_f = 0, c_s = 0, c_a = 0, c_c = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : c_f, c_s, c_a, c_c)
    for (int64_t tile = 0; tile < nt; ++tile) {
        int64_t ty = tile / tiles_x, tx = tile % tiles_x;
        int64_t r0 = ty * ORC_TILE, r1 = r0 + ORC_TILE < height ? r0 + ORC_TILE : height;
        int64_t q0 = tx * ORC_TILE, q1 = q0 + ORC_TILE < width ? q0 + ORC_TILE : width;
        const int64_t* order = bin_idx + bin_ptr[tile];
        int64_t len = bin_ptr[tile + 1] - bin_ptr[tile];
        for (int64_t row = r0; row < r1; ++row) {
            for (int64_t col = q0; col < q1; ++col) {
                double px = (double)col + 0.5, py = (double)row + 0.5;
                double cr = 0, cg = 0, cb = 0, T = 1.0;
                int64_t nc = 0;
                double mg = INFINITY;
                int64_t mpos = -1;
                int8_t mkind = 0;
                for (int64_t pos = 0; pos < len; ++pos) {
                    int64_t j = order[pos];
                    double A, B, C;
                    conic_of(cov2d + 3 * j, &A, &B, &C);
                    double dx = px - mean2d[2 * j], dy = py - mean2d[2 * j + 1];
                    double sigma = 0.5 * (A * dx * dx + C * dy * dy) + B * dx * dy;
                    double araw = opac[j] * exp(-sigma);
                    double alpha = araw < ORC_ALPHA_MAX ? araw : ORC_ALPHA_MAX;
                    c_f++;
                    double m = rel_margin(sigma, ORC_SIGMA_CUT);
                    if (m < mg) { mg = m; mpos = pos; mkind = 1; }
                    if (!(sigma <= ORC_SIGMA_CUT)) continue;
                    c_s++;
                    m = rel_margin(alpha, ORC_ALPHA_MIN);
                    if (m < mg) { mg = m; mpos = pos; mkind = 2; }
                    m = rel_margin(araw, ORC_ALPHA_MAX);
                    if (m < mg) { mg = m; mpos = pos; mkind = 3; }
                    if (!(alpha >= ORC_ALPHA_MIN)) continue;
                    c_a++;
                    double nT = T * (1.0 - alpha);
                    if (early_termination) {
                        m = rel_margin(nT, ORC_T_MIN);
                        if (m < mg) { mg = m; mpos = pos; mkind = 4; }
                        if (nT < ORC_T_MIN) break; /* :141-144, the stopping splat is not composited */
                    }
                    c_c++;
                    double w = alpha * T;
                    cr += w * colors[3 * j]; cg += w * colors[3 * j + 1]; cb += w * colors[3 * j + 2];
                    T = nT;
                    nc = pos + 1;
                }
                int64_t p = row * width + col;
                image[3 * p] = cr + bg[0] * T;
                image[3 * p + 1] = cg + bg[1] * T;
                image[3 * p + 2] = cb + bg[2] * T;
                final_T[p] = T;
                n_contrib[p] = nc;
                if (margin) margin[p] = mg;
                if (margin_pos) margin_pos[p] = mpos;
                if (margin_kind) margin_kind[p] = mkind;
            }
        }
    }
    if (counts) { counts[0] = c_f; counts[1] = c_s; counts[2] = c_a; counts[3] = c_c; }
}

/*
 * sg/raster_backward.py:47-108 _backward_tile over every tile, summed like
 * sg/raster_backward.py:166-205 accumulate_image_backward.  Outputs per
 * SCENE Gaussian: d_color(3), d_opacity, d_mean2d(2), d_cov2d as the full
 * 2x2 (4, both off-diagonals = c01, sg/raster_backward.py:99-105).
 * Per (tile, splat) the pixel sum is formed first, then added to the
 * accumulator, like the reference's np.sum-then-+= (:81, :92, :97-105).
 * counts[3] = E_b (sum n_contrib), E_b_sigma, E_b_contrib.
 */
void orc_raster_bwd(int64_t width, int64_t height, const int64_t* bin_ptr, const int64_t* bin_idx,
                    const double* mean2d, const double* cov2d, const double* opac, const double* colors,
                    const double* bg, const double* final_T, const int64_t* n_contrib, const double* d_image,
                    int64_t n_gauss, double* d_color, double* d_opacity, double* d_mean2d, double* d_cov2d,
                    int64_t* counts, int nthreads) {
    set_threads(nthreads);
    int64_t tiles_x = (width + ORC_TILE - 1) / ORC_TILE, tiles_y = (height + ORC_TILE - 1) / ORC_TILE;
    int64_t nt = tiles_x * tiles_y;
    int nth = 1;
#ifdef _OPENMP
    nth = omp_get_max_threads();
#endif
    /* private accumulators: 9 doubles per Gaussian per thread */
    double* acc = (double*)calloc((size_t)nth * (size_t)n_gauss * 9, sizeof(double));
    int64_t c_b = 0, c_s = 0, c_c = 0;
#pragma omp parallel reduction(+ : c_b, c_s, c_c)
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double* my = acc + (size_t)tid * (size_t)n_gauss * 9;
        double Tp[ORC_TILE * ORC_TILE], S[ORC_TILE * ORC_TILE][3];
#pragma omp for schedule(dynamic, 1)
        for (int64_t tile = 0; tile < nt; ++tile) {
            int64_t ty = tile / tiles_x, tx = tile % tiles_x;
            int64_t r0 = ty * ORC_TILE, r1 = r0 + ORC_TILE < height ? r0 + ORC_TILE : height;
            int64_t q0 = tx * ORC_TILE, q1 = q0 + ORC_TILE < width ? q0 + ORC_TILE : width;
            const int64_t* order = bin_idx + bin_ptr[tile];
            int64_t len = bin_ptr[tile + 1] - bin_ptr[tile];
            if (len == 0) continue;
            int64_t npx = (r1 - r0) * (q1 - q0);
            int64_t max_n = 0;
            for (int64_t k = 0; k < npx; ++k) {
                int64_t row = r0 + k / (q1 - q0), col = q0 + k % (q1 - q0);
                int64_t p = row * width + col;
                if (n_contrib[p] > max_n) max_n = n_contrib[p];
                Tp[k] = final_T[p];
                for (int c = 0; c < 3; ++c) S[k][c] = bg[c] * Tp[k];
                c_b += n_contrib[p];
            }
            for (int64_t pos = max_n - 1; pos >= 0; --pos) {
                int64_t j = order[pos];
                double A, B, C;
                conic_of(cov2d + 3 * j, &A, &B, &C);
                double sdc0 = 0, sdc1 = 0, sdc2 = 0, sdo = 0, sm0 = 0, sm1 = 0, s00 = 0, s01 = 0, s11 = 0;
                int any = 0;
                for (int64_t k = 0; k < npx; ++k) {
                    int64_t row = r0 + k / (q1 - q0), col = q0 + k % (q1 - q0);
                    int64_t p = row * width + col;
                    if (!(n_contrib[p] > pos)) continue;
                    double px = (double)col + 0.5, py = (double)row + 0.5;
                    double dx = px - mean2d[2 * j], dy = py - mean2d[2 * j + 1];
                    double sigma = 0.5 * (A * dx * dx + C * dy * dy) + B * dx * dy;
                    double e = exp(-sigma);
                    double araw = opac[j] * e;
                    double alpha = araw < ORC_ALPHA_MAX ? araw : ORC_ALPHA_MAX;
                    if (!(sigma <= ORC_SIGMA_CUT)) continue;
                    c_s++;
                    if (!(alpha >= ORC_ALPHA_MIN)) continue;
                    c_c++;
                    any = 1;
                    double om = 1.0 - alpha;
                    double th = Tp[k] / om;
                    double w = alpha * th;
                    const double* g = d_image + 3 * p;
                    sdc0 += w * g[0]; sdc1 += w * g[1]; sdc2 += w * g[2];
                    const double* col3 = colors + 3 * j;
                    double da = (col3[0] * th - S[k][0] / om) * g[0] + (col3[1] * th - S[k][1] / om) * g[1] +
                                (col3[2] * th - S[k][2] / om) * g[2];
                    if (araw < ORC_ALPHA_MAX) { /* live, :91-93 */
                        sdo += da * e;
                        double dsig = -araw * da;
                        double y0 = A * dx + B * dy, y1 = B * dx + C * dy;
                        sm0 += -dsig * y0; sm1 += -dsig * y1;
                        s00 += -0.5 * dsig * y0 * y0; s01 += -0.5 * dsig * y0 * y1; s11 += -0.5 * dsig * y1 * y1;
                    }
                    for (int c = 0; c < 3; ++c) S[k][c] += w * col3[c];
                    Tp[k] = th;
                }
                if (!any) continue;
                double* a = my + 9 * j;
                a[0] += sdc0; a[1] += sdc1; a[2] += sdc2; a[3] += sdo;
                a[4] += sm0; a[5] += sm1; a[6] += s00; a[7] += s01; a[8] += s11;
            }
        }
    }
    memset(d_color, 0, (size_t)n_gauss * 3 * sizeof(double));
    memset(d_opacity, 0, (size_t)n_gauss * sizeof(double));
    memset(d_mean2d, 0, (size_t)n_gauss * 2 * sizeof(double));
    memset(d_cov2d, 0, (size_t)n_gauss * 4 * sizeof(double));
    for (int t = 0; t < nth; ++t) {
        const double* a = acc + (size_t)t * (size_t)n_gauss * 9;
        for (int64_t j = 0; j < n_gauss; ++j) {
            const double* v = a + 9 * j;
            d_color[3 * j] += v[0]; d_color[3 * j + 1] += v[1]; d_color[3 * j + 2] += v[2];
            d_opacity[j] += v[3];
            d_mean2d[2 * j] += v[4]; d_mean2d[2 * j + 1] += v[5];
            d_cov2d[4 * j] += v[6]; d_cov2d[4 * j + 1] += v[7]; d_cov2d[4 * j + 2] += v[7]; d_cov2d[4 * j + 3] += v[8];
        }
    }
    free(acc);
    if (counts) { counts[0] = c_b; counts[1] = c_s; counts[2] = c_c; }
}

/*
 * Per-pixel API.  Splat arrays are indexed by the
 * query bins' own indices (the reference's `projected` list order);
 * opac/colors are per splat (the scene rows already gathered).
 *
 * sg/raster_forward.py:86-92,175-196 eval_alpha for n (splat, pixel) pairs:
 * out4[q] = (alpha, dx, dy, sigma), alpha 0 when skipped.
 */
void orc_eval_alpha(int64_t n, const int64_t* splat, const double* pix, const double* mean2d, const double* cov2d,
                    const double* opac, double* out4) {
    for (int64_t q = 0; q < n; ++q) {
        int64_t j = splat[q];
        double A, B, C;
        conic_of(cov2d + 3 * j, &A, &B, &C);
        double dx = pix[2 * q] - mean2d[2 * j], dy = pix[2 * q + 1] - mean2d[2 * j + 1];
        double sigma = 0.5 * (A * dx * dx + C * dy * dy) + B * dx * dy;
        double alpha = opac[j] * exp(-sigma);
        if (alpha > ORC_ALPHA_MAX) alpha = ORC_ALPHA_MAX;
        if (sigma > ORC_SIGMA_CUT || alpha < ORC_ALPHA_MIN) alpha = 0.0;
        out4[4 * q] = alpha; out4[4 * q + 1] = dx; out4[4 * q + 2] = dy; out4[4 * q + 3] = sigma;
    }
}

/*
 * sg/raster_forward.py:199-219 composite_pixel (the :116-154 loop for one
 * pixel) for n queries, each with its own bin and early-termination flag.
 * margin/margin_kind as orc_raster_fwd (optional).
 */
void orc_composite_pixels(int64_t n, const int64_t* bin_ptr, const int64_t* bin_idx, const double* pix,
                          const int8_t* et, const double* mean2d, const double* cov2d, const double* opac,
                          const double* colors, const double* bg, double* color, double* final_T, int64_t* n_contrib,
                          double* margin, int8_t* margin_kind) {
    for (int64_t q = 0; q < n; ++q) {
        double px = pix[2 * q], py = pix[2 * q + 1];
        double cr = 0, cg = 0, cb = 0, T = 1.0, mg = INFINITY;
        int64_t nc = 0;
        int8_t mkind = 0;
        for (int64_t pos = 0; pos < bin_ptr[q + 1] - bin_ptr[q]; ++pos) {
            int64_t j = bin_idx[bin_ptr[q] + pos];
            double A, B, C;
            conic_of(cov2d + 3 * j, &A, &B, &C);
            double dx = px - mean2d[2 * j], dy = py - mean2d[2 * j + 1];
            double sigma = 0.5 * (A * dx * dx + C * dy * dy) + B * dx * dy;
            double araw = opac[j] * exp(-sigma);
            double alpha = araw < ORC_ALPHA_MAX ? araw : ORC_ALPHA_MAX;
            double m = rel_margin(sigma, ORC_SIGMA_CUT);
            if (m < mg) { mg = m; mkind = 1; }
            if (!(sigma <= ORC_SIGMA_CUT)) continue;
            m = rel_margin(alpha, ORC_ALPHA_MIN);
            if (m < mg) { mg = m; mkind = 2; }
            m = rel_margin(araw, ORC_ALPHA_MAX);
            if (m < mg) { mg = m; mkind = 3; }
            if (!(alpha >= ORC_ALPHA_MIN)) continue;
            double nT = T * (1.0 - alpha);
            if (et[q]) {
                m = rel_margin(nT, ORC_T_MIN);
                if (m < mg) { mg = m; mkind = 4; }
                if (nT < ORC_T_MIN) break;
            }
            double w = alpha * T;
            cr += w * colors[3 * j]; cg += w * colors[3 * j + 1]; cb += w * colors[3 * j + 2];
            T = nT;
            nc = pos + 1;
        }
        color[3 * q] = cr + bg[0] * T;
        color[3 * q + 1] = cg + bg[1] * T;
        color[3 * q + 2] = cb + bg[2] * T;
        final_T[q] = T;
        n_contrib[q] = nc;
        if (margin) margin[q] = mg;
        if (margin_kind) margin_kind[q] = mkind;
    }
}

/*
 * sg/raster_backward.py:111-163 composite_pixel_backward /
 * transmittance_replay (the :47-108 walk for one pixel) for n queries.
 * Gradients accumulate into per-splat rows: d9[j] = d_color 3, d_opacity,
 * d_mean2d 2, d_cov2d 00, 01 (= 10), 11.  t_log (optional, sized like
 * bin_idx): replayed T before each contributing entry, NaN elsewhere.
 */
void orc_composite_pixels_bwd(int64_t n, const int64_t* bin_ptr, const int64_t* bin_idx, const double* pix,
                              const double* mean2d, const double* cov2d, const double* opac, const double* colors,
                              const double* bg, const double* final_T, const int64_t* n_contrib,
                              const double* d_pix, double* d9, double* t_log) {
    for (int64_t q = 0; q < n; ++q) {
        const int64_t b0 = bin_ptr[q], len = bin_ptr[q + 1] - b0;
        if (t_log)
            for (int64_t pos = 0; pos < len; ++pos) t_log[b0 + pos] = NAN;
        double px = pix[2 * q], py = pix[2 * q + 1];
        double T = final_T[q];
        double S[3] = {bg[0] * T, bg[1] * T, bg[2] * T};
        const double* g = d_pix + 3 * q;
        int64_t nc = n_contrib[q] < len ? n_contrib[q] : len;
        for (int64_t pos = nc - 1; pos >= 0; --pos) {
            int64_t j = bin_idx[b0 + pos];
            double A, B, C;
            conic_of(cov2d + 3 * j, &A, &B, &C);
            double dx = px - mean2d[2 * j], dy = py - mean2d[2 * j + 1];
            double sigma = 0.5 * (A * dx * dx + C * dy * dy) + B * dx * dy;
            double e = exp(-sigma);
            double araw = opac[j] * e;
            double alpha = araw < ORC_ALPHA_MAX ? araw : ORC_ALPHA_MAX;
            if (!(sigma <= ORC_SIGMA_CUT) || !(alpha >= ORC_ALPHA_MIN)) continue;
            double om = 1.0 - alpha, th = T / om, w = alpha * th;
            if (t_log) t_log[b0 + pos] = th;
            const double* col3 = colors + 3 * j;
            double* a = d9 + 9 * j;
            a[0] += w * g[0]; a[1] += w * g[1]; a[2] += w * g[2];
            double da = (col3[0] * th - S[0] / om) * g[0] + (col3[1] * th - S[1] / om) * g[1] +
                        (col3[2] * th - S[2] / om) * g[2];
            if (araw < ORC_ALPHA_MAX) {
                a[3] += da * e;
                double dsig = -araw * da;
                double y0 = A * dx + B * dy, y1 = B * dx + C * dy;
                a[4] += -dsig * y0; a[5] += -dsig * y1;
                a[6] += -0.5 * dsig * y0 * y0; a[7] += -0.5 * dsig * y0 * y1; a[8] += -0.5 * dsig * y1 * y1;
            }
            for (int c = 0; c < 3; ++c) S[c] += w * col3[c];
            T = th;
        }
    }
}

/* sg/proj_backward.py:139-148 dR/d(w,x,y,z) for a unit quaternion. */
static void rotmat_quat_jacobians(double w, double x, double y, double z, double Jq[4][9]) {
    double t[4][9] = {
        {0.0, -z, y, z, 0.0, -x, -y, x, 0.0},
        {0.0, y, z, y, -2.0 * x, -w, z, w, -2.0 * x},
        {-2.0 * y, x, w, x, 0.0, z, -w, z, -2.0 * y},
        {-2.0 * z, -w, x, w, -2.0 * z, y, x, y, 0.0},
    };
    for (int k = 0; k < 4; ++k)
        for (int e = 0; e < 9; ++e) Jq[k][e] = 2.0 * t[k][e];
}

/*
 * sg/proj_backward.py:178-223 scene_backward, per visible Gaussian (loop body
 * :200-222), composed of mean2d_backward (:53-77), cov2d_backward (:88-121),
 * _cov_transform_grad (:80-85), world_backward (:124-136) and
 * covariance3d_backward (:151-175).  Inputs d_mean2d (n,2) and d_cov2d (n,4)
 * are the screen-space gradients of orc_raster_bwd.  Culled rows stay 0.
 * d_view is the 4x4 sum over Gaussians (fixed order: per-thread partials in
 * thread order).
 */
int orc_project_bwd(int64_t n, const double* means, const double* scales, const double* quats,
                    const orc_camera* cam, const int8_t* visible, const double* t_cam_all,
                    const double* d_mean2d, const double* d_cov2d, double* d_mean, double* d_scale,
                    double* d_quat, double* d_view, int nthreads) {
    set_threads(nthreads);
    double P[16];
    proj_matrix(cam, P);
    const double* V = cam->view;
    int nth = 1;
#ifdef _OPENMP
    nth = omp_get_max_threads();
#endif
    double* dv_part = (double*)calloc((size_t)nth * 16, sizeof(double));
    int err = 0;
#pragma omp parallel
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double* dv = dv_part + 16 * tid;
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            double* dm = d_mean + 3 * i; double* ds = d_scale + 3 * i; double* dq = d_quat + 4 * i;
            dm[0] = dm[1] = dm[2] = 0.0; ds[0] = ds[1] = ds[2] = 0.0; dq[0] = dq[1] = dq[2] = dq[3] = 0.0;
            if (!visible[i]) continue;
            const double* t = t_cam_all + 4 * i;
            double R[9], M[9], Sig[9], qhat[4], qn;
            if (compose_cov3d(quats + 4 * i, scales + 3 * i, R, M, Sig, qhat, &qn)) { err = 1; continue; }
            double J[6];
            jacobian(t, cam, J);
            double T[6];
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 3; ++b)
                    T[3 * a + b] = J[3 * a + 0] * V[0 * 4 + b] + J[3 * a + 1] * V[1 * 4 + b] + J[3 * a + 2] * V[2 * 4 + b];
            /* mean2d_backward :53-77 */
            double tp[4];
            for (int r = 0; r < 4; ++r) tp[r] = P[4 * r + 0] * t[0] + P[4 * r + 1] * t[1] + P[4 * r + 2] * t[2] + P[4 * r + 3] * t[3];
            double tw = tp[3];
            double wdx = (double)cam->width * d_mean2d[2 * i], hdy = (double)cam->height * d_mean2d[2 * i + 1];
            double dtp[4] = {0.5 * wdx / tw, 0.5 * hdy / tw, 0.0, -0.5 * (wdx * tp[0] + hdy * tp[1]) / (tw * tw)};
            double dt_m[4];
            for (int c = 0; c < 4; ++c) dt_m[c] = P[0 * 4 + c] * dtp[0] + P[1 * 4 + c] * dtp[1] + P[2 * 4 + c] * dtp[2] + P[3 * 4 + c] * dtp[3];
            /* cov2d_backward :88-121 with G the full 2x2 d_cov2d */
            const double* G = d_cov2d + 4 * i;
            double GT[6], GtT[6];
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 3; ++b) {
                    GT[3 * a + b] = G[2 * a + 0] * T[b] + G[2 * a + 1] * T[3 + b];
                    GtT[3 * a + b] = G[0 * 2 + a] * T[b] + G[1 * 2 + a] * T[3 + b];
                }
            double dSig[9];
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) dSig[3 * a + b] = T[a] * GT[b] + T[3 + a] * GT[3 + b];
            /* _cov_transform_grad :80-85: dT = G T Sig^T + G^T T Sig */
            double dT[6];
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 3; ++b) {
                    double s = 0.0;
                    for (int k = 0; k < 3; ++k) s += GT[3 * a + k] * Sig[3 * b + k] + GtT[3 * a + k] * Sig[3 * k + b];
                    dT[3 * a + b] = s;
                }
            double dJ[6];
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 3; ++b)
                    dJ[3 * a + b] = dT[3 * a + 0] * V[4 * b + 0] + dT[3 * a + 1] * V[4 * b + 1] + dT[3 * a + 2] * V[4 * b + 2];
            double tx = t[0], ty = t[1], tz = t[2], fx = cam->fx, fy = cam->fy;
            double tz2 = tz * tz, tz3 = tz2 * tz;
            double dt_c[4] = {-fx / tz2 * dJ[2], -fy / tz2 * dJ[5],
                              -fx / tz2 * dJ[0] + 2.0 * fx * tx / tz3 * dJ[2] - fy / tz2 * dJ[4] + 2.0 * fy * ty / tz3 * dJ[5],
                              0.0};
            double dt[4];
            for (int c = 0; c < 4; ++c) dt[c] = dt_m[c] + dt_c[c];
            /* world_backward :124-136 */
            const double* m = means + 3 * i;
            double q4[4] = {m[0], m[1], m[2], 1.0};
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) dv[4 * a + b] += dt[a] * q4[b];
            for (int c = 0; c < 3; ++c) dm[c] = V[0 * 4 + c] * dt[0] + V[1 * 4 + c] * dt[1] + V[2 * 4 + c] * dt[2];
            /* covariance3d_backward :151-175 */
            double dM[9];
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) {
                    double s = 0.0;
                    for (int k = 0; k < 3; ++k) s += dSig[3 * a + k] * M[3 * k + b] + dSig[3 * k + a] * M[3 * k + b];
                    dM[3 * a + b] = s;
                }
            const double* sc = scales + 3 * i;
            double dR[9];
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) dR[3 * a + b] = dM[3 * a + b] * sc[b];
            for (int b = 0; b < 3; ++b) ds[b] = R[0 * 3 + b] * dM[0 * 3 + b] + R[1 * 3 + b] * dM[1 * 3 + b] + R[2 * 3 + b] * dM[2 * 3 + b];
            double Jq[4][9];
            rotmat_quat_jacobians(qhat[0], qhat[1], qhat[2], qhat[3], Jq);
            double dqh[4];
            for (int k = 0; k < 4; ++k) {
                double s = 0.0;
                for (int e = 0; e < 9; ++e) s += dR[e] * Jq[k][e];
                dqh[k] = s;
            }
            double dot = qhat[0] * dqh[0] + qhat[1] * dqh[1] + qhat[2] * dqh[2] + qhat[3] * dqh[3];
            for (int k = 0; k < 4; ++k) dq[k] = (dqh[k] - qhat[k] * dot) / qn;
            /* rotation path :218-222: d_view[:3,:3] += J^T dT */
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) dv[4 * a + b] += J[a] * dT[b] + J[3 + a] * dT[3 + b];
        }
    }
    memset(d_view, 0, 16 * sizeof(double));
    for (int t = 0; t < nth; ++t)
        for (int e = 0; e < 16; ++e) d_view[e] += dv_part[16 * t + e];
    free(dv_part);
    return err;
}
