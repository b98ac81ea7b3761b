// ops64.cu -- the reference's per-splat helper functions in float64 on the
// device, batched (one thread per item): the scalar building blocks the
// fused kernels inline, exposed one by one so the drop-in API offers every
// name of sg/__init__.py:64-119.  One C entry point, gs_op64(op, ...):
//
//   GS_OP_QUAT_TO_ROTMAT       sg/core.py:146-171          q(4)            -> R(9)
//   GS_OP_COMPOSE_COV3D        sg/core.py:174-195          q(4), s(3)      -> R(9), S(9), M(9), sigma(9)
//   GS_OP_FROBENIUS            sg/core.py:198-204          x(k), y(k)      -> sum x*y   (n rows of k = cols)
//   GS_OP_WORLD_TO_CAMERA      sg/projection.py:36-42      mean(3)         -> t(4)
//   GS_OP_CAMERA_TO_PIXEL      sg/projection.py:45-61      t(4)            -> mean2d(2)
//   GS_OP_PROJECTION_JACOBIAN  sg/projection.py:64-82      t(4)            -> J(6)
//   GS_OP_PROJECT_COVARIANCE   sg/projection.py:85-96      J(6), Rcw(9), sigma(9) -> cov2d(4)
//   GS_OP_BOUNDING_RADIUS      sg/projection.py:99-112     cov2d(4)        -> r(1, integral)
//   GS_OP_MEAN2D_BACKWARD      sg/proj_backward.py:53-77   dm(2), t(4)     -> dt(4)
//   GS_OP_COV2D_BACKWARD       sg/proj_backward.py:88-121  G(4), T(6), sigma(9), J(6), Rcw(9), t(4)
//                                                          -> dsigma(9), dt(4)
//   GS_OP_WORLD_BACKWARD       sg/proj_backward.py:124-136 dt(4), mean(3)  -> dmean(3), dview(16)
//   GS_OP_COV3D_BACKWARD       sg/proj_backward.py:151-175 dsigma(9), R(9), S(9), M(9), q(4), s(3)
//                                                          -> dq(4), ds(3)
//
// Matrices are row-major.  Errors go to the status word (atomicMin of
// index << 8 | code) like the rest of the library; the Python layer raises
// the reference's ValueError.
#include "common.cuh"
#include "internal.cuh"

namespace gs {

namespace {

struct Op64Args {
    const double* in[6];
    double* out[4];
    double view[16];
    double fx, fy, cx, cy, near_plane, far_plane;
    int W, H, cols;
};

__device__ __forceinline__ void err64(unsigned long long* status, long long i, int code) {
    if (status) atomicMin(status, ((unsigned long long)i << 8) | (unsigned long long)code);
}

// sg/core.py:146-171 (q normalised first; (w, x, y, z))
__device__ bool rotmat64(const double* q, double R[9], unsigned long long* status, long long i) {
    const double nq = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(nq > QUAT_EPS_D)) {
        err64(status, i, GS_ERR_QUAT);
        return false;
    }
    const double w = q[0] / nq, x = q[1] / nq, y = q[2] / nq, z = q[3] / nq;
    R[0] = 1.0 - 2.0 * (y * y + z * z); R[1] = 2.0 * (x * y - w * z); R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z); R[4] = 1.0 - 2.0 * (x * x + z * z); R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y); R[7] = 2.0 * (y * z + w * x); R[8] = 1.0 - 2.0 * (x * x + y * y);
    return true;
}

// P = projection matrix (sg/core.py:98-111); t' = P t
__device__ void proj_apply(const Op64Args& a, const double* t, double tp[4]) {
    const double n = a.near_plane, f = a.far_plane;
    tp[0] = 2.0 * a.fx / a.W * t[0];
    tp[1] = 2.0 * a.fy / a.H * t[1];
    tp[2] = (f + n) / (f - n) * t[2] - 2.0 * f * n / (f - n) * t[3];
    tp[3] = t[2];
}

__global__ void __launch_bounds__(128) op64_kernel(int op, long long n, Op64Args a, unsigned long long* status) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    switch (op) {
        case GS_OP_QUAT_TO_ROTMAT: {
            double R[9];
            if (rotmat64(a.in[0] + 4 * i, R, status, i))
                for (int k = 0; k < 9; ++k) a.out[0][9 * i + k] = R[k];
            break;
        }
        case GS_OP_COMPOSE_COV3D: {
            const double* s = a.in[1] + 3 * i;
            if (!(s[0] > 0.0 && s[1] > 0.0 && s[2] > 0.0)) {  // checked before the quaternion (:187-190)
                err64(status, i, GS_ERR_SCALE);
                break;
            }
            double R[9];
            if (!rotmat64(a.in[0] + 4 * i, R, status, i)) break;
            double M[9];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) M[3 * r + c] = R[3 * r + c] * s[c];
            for (int k = 0; k < 9; ++k) {
                a.out[0][9 * i + k] = R[k];
                a.out[1][9 * i + k] = (k % 4 == 0) ? s[k / 4] : 0.0;
                a.out[2][9 * i + k] = M[k];
            }
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c)
                    a.out[3][9 * i + 3 * r + c] = M[3 * r] * M[3 * c] + M[3 * r + 1] * M[3 * c + 1] +
                                                  M[3 * r + 2] * M[3 * c + 2];
            break;
        }
        case GS_OP_FROBENIUS: {
            const double* x = a.in[0] + (long long)a.cols * i;
            const double* y = a.in[1] + (long long)a.cols * i;
            double acc = 0.0;
            for (int k = 0; k < a.cols; ++k) acc += x[k] * y[k];
            a.out[0][i] = acc;
            break;
        }
        case GS_OP_WORLD_TO_CAMERA: {
            const double* m = a.in[0] + 3 * i;
            for (int r = 0; r < 4; ++r)
                a.out[0][4 * i + r] = a.view[4 * r] * m[0] + a.view[4 * r + 1] * m[1] + a.view[4 * r + 2] * m[2] +
                                      a.view[4 * r + 3];
            break;
        }
        case GS_OP_CAMERA_TO_PIXEL: {
            double tp[4];
            proj_apply(a, a.in[0] + 4 * i, tp);
            if (fabs(tp[3]) < 1e-12) {
                err64(status, i, GS_ERR_HOMOG);
                break;
            }
            a.out[0][2 * i] = (a.W * tp[0] / tp[3] + 1.0) / 2.0 + a.cx;
            a.out[0][2 * i + 1] = (a.H * tp[1] / tp[3] + 1.0) / 2.0 + a.cy;
            break;
        }
        case GS_OP_PROJECTION_JACOBIAN: {
            const double* t = a.in[0] + 4 * i;
            if (!(t[2] > 0.0)) {
                err64(status, i, GS_ERR_BEHIND);
                break;
            }
            const double tz = t[2];
            double* J = a.out[0] + 6 * i;
            J[0] = a.fx / tz; J[1] = 0.0; J[2] = -a.fx * t[0] / (tz * tz);
            J[3] = 0.0; J[4] = a.fy / tz; J[5] = -a.fy * t[1] / (tz * tz);
            break;
        }
        case GS_OP_PROJECT_COVARIANCE: {
            const double* J = a.in[0] + 6 * i;
            const double* R = a.in[1] + 9 * i;
            const double* S = a.in[2] + 9 * i;
            double T[6], TS[6];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 3; ++c) T[3 * r + c] = J[3 * r] * R[c] + J[3 * r + 1] * R[3 + c] + J[3 * r + 2] * R[6 + c];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 3; ++c) TS[3 * r + c] = T[3 * r] * S[c] + T[3 * r + 1] * S[3 + c] + T[3 * r + 2] * S[6 + c];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c)
                    a.out[0][4 * i + 2 * r + c] = TS[3 * r] * T[3 * c] + TS[3 * r + 1] * T[3 * c + 1] +
                                                  TS[3 * r + 2] * T[3 * c + 2] + (r == c ? DILATION_D : 0.0);
            break;
        }
        case GS_OP_BOUNDING_RADIUS: {
            const double* c2 = a.in[0] + 4 * i;
            const double ca = c2[0], cb = c2[1], cc = c2[3];
            const double det = ca * cc - cb * cb;
            if (!(det > 0.0 && ca + cc > 0.0)) {
                err64(status, i, GS_ERR_COV2D);
                break;
            }
            const double mid = 0.5 * (ca + cc);
            const double lam = mid + sqrt(0.25 * (ca - cc) * (ca - cc) + cb * cb);
            a.out[0][i] = ceil(3.0 * sqrt(lam));
            break;
        }
        case GS_OP_MEAN2D_BACKWARD: {
            const double* g = a.in[0] + 2 * i;
            double tp[4];
            proj_apply(a, a.in[1] + 4 * i, tp);
            if (fabs(tp[3]) < 1e-12) {
                err64(status, i, GS_ERR_HOMOG);
                break;
            }
            const double wdx = a.W * g[0], hdy = a.H * g[1];
            const double d0 = 0.5 * wdx / tp[3], d1 = 0.5 * hdy / tp[3];
            const double d3 = -0.5 * (wdx * tp[0] + hdy * tp[1]) / (tp[3] * tp[3]);
            // P^T d_t' (P is zero except [0,0], [1,1], [2,2], [2,3], [3,2] = 1; d_t'[2] = 0)
            const double n_ = a.near_plane, f = a.far_plane;
            double* dt = a.out[0] + 4 * i;
            dt[0] = 2.0 * a.fx / a.W * d0;
            dt[1] = 2.0 * a.fy / a.H * d1;
            dt[2] = (f + n_) / (f - n_) * 0.0 + d3;
            dt[3] = -2.0 * f * n_ / (f - n_) * 0.0;
            break;
        }
        case GS_OP_COV2D_BACKWARD: {
            const double* G = a.in[0] + 4 * i;
            const double* T = a.in[1] + 6 * i;
            const double* S = a.in[2] + 9 * i;
            const double* R = a.in[4] + 9 * i;
            const double* t = a.in[5] + 4 * i;
            // d_sigma = T^T G T
            double GT[6];  // G T (2x3)
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 3; ++c) GT[3 * r + c] = G[2 * r] * T[c] + G[2 * r + 1] * T[3 + c];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) a.out[0][9 * i + 3 * r + c] = T[r] * GT[c] + T[3 + r] * GT[3 + c];
            // d_T = G T sigma^T + G^T T sigma (:80-85)
            double GtT[6];  // G^T T
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 3; ++c) GtT[3 * r + c] = G[r] * T[c] + G[2 + r] * T[3 + c];
            double dT[6];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 3; ++c) {
                    double v = 0.0;
                    for (int k = 0; k < 3; ++k) v += GT[3 * r + k] * S[3 * c + k] + GtT[3 * r + k] * S[3 * k + c];
                    dT[3 * r + c] = v;
                }
            // d_J = d_T R_cw^T
            double dJ[6];
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 3; ++c)
                    dJ[3 * r + c] = dT[3 * r] * R[3 * c] + dT[3 * r + 1] * R[3 * c + 1] + dT[3 * r + 2] * R[3 * c + 2];
            const double tx = t[0], ty = t[1], tz = t[2], tz2 = tz * tz, tz3 = tz2 * tz;
            double* dt = a.out[1] + 4 * i;
            dt[0] = -a.fx / tz2 * dJ[2];
            dt[1] = -a.fy / tz2 * dJ[5];
            dt[2] = -a.fx / tz2 * dJ[0] + 2.0 * a.fx * tx / tz3 * dJ[2] - a.fy / tz2 * dJ[4] +
                    2.0 * a.fy * ty / tz3 * dJ[5];
            dt[3] = 0.0;
            break;
        }
        case GS_OP_WORLD_BACKWARD: {
            const double* dt = a.in[0] + 4 * i;
            const double* m = a.in[1] + 3 * i;
            const double q[4] = {m[0], m[1], m[2], 1.0};
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c) a.out[1][16 * i + 4 * r + c] = dt[r] * q[c];
            for (int c = 0; c < 3; ++c)  // R^T dt[:3]
                a.out[0][3 * i + c] = a.view[c] * dt[0] + a.view[4 + c] * dt[1] + a.view[8 + c] * dt[2];
            break;
        }
        case GS_OP_COV3D_BACKWARD: {
            const double* g = a.in[0] + 9 * i;
            const double* R = a.in[1] + 9 * i;
            const double* S = a.in[2] + 9 * i;
            const double* M = a.in[3] + 9 * i;
            const double* q = a.in[4] + 4 * i;
            double dM[9];  // g M + g^T M
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) {
                    double v = 0.0;
                    for (int k = 0; k < 3; ++k) v += (g[3 * r + k] + g[3 * k + r]) * M[3 * k + c];
                    dM[3 * r + c] = v;
                }
            double dR[9];  // dM S^T
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c)
                    dR[3 * r + c] = dM[3 * r] * S[3 * c] + dM[3 * r + 1] * S[3 * c + 1] + dM[3 * r + 2] * S[3 * c + 2];
            for (int c = 0; c < 3; ++c)  // diag(R^T dM)
                a.out[1][3 * i + c] = R[c] * dM[c] + R[3 + c] * dM[3 + c] + R[6 + c] * dM[6 + c];
            const double nq = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
            if (!(nq > QUAT_EPS_D)) {
                err64(status, i, GS_ERR_QUAT);
                break;
            }
            const double w = q[0] / nq, x = q[1] / nq, y = q[2] / nq, z = q[3] / nq;
            // <dR, dR/dq_k> with the printed Jacobians (:139-148)
            const double J[4][9] = {{0.0, -z, y, z, 0.0, -x, -y, x, 0.0},
                                    {0.0, y, z, y, -2.0 * x, -w, z, w, -2.0 * x},
                                    {-2.0 * y, x, w, x, 0.0, z, -w, z, -2.0 * y},
                                    {-2.0 * z, -w, x, w, -2.0 * z, y, x, y, 0.0}};
            double dqh[4];
            for (int k = 0; k < 4; ++k) {
                double v = 0.0;
                for (int e = 0; e < 9; ++e) v += dR[e] * 2.0 * J[k][e];
                dqh[k] = v;
            }
            const double qh[4] = {w, x, y, z};
            const double dot = qh[0] * dqh[0] + qh[1] * dqh[1] + qh[2] * dqh[2] + qh[3] * dqh[3];
            for (int k = 0; k < 4; ++k) a.out[0][4 * i + k] = (dqh[k] - qh[k] * dot) / nq;
            break;
        }
        default:
            break;
    }
}

}  // namespace

}  // namespace gs

using namespace gs;

extern "C" {

int gs_op64(int op, int64_t n, const double* const* in /*[host] array of device pointers*/,
            double* const* out /*[host]*/, int32_t cols, const gs_camera64* cam /*[host], nullable*/,
            unsigned long long* status, gs_stream_t stream) {
    if (op < GS_OP_QUAT_TO_ROTMAT || op > GS_OP_COV3D_BACKWARD) return set_error("gs_op64: unknown op %d", op);
    if (n < 0) return set_error("gs_op64: n=%lld", (long long)n);
    if (n == 0) return 0;
    Op64Args a = {};
    static const int n_in[] = {0, 1, 2, 2, 1, 1, 1, 3, 1, 2, 6, 2, 5};
    static const int n_out[] = {0, 1, 4, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2};
    for (int k = 0; k < n_in[op]; ++k) {
        if (!in || !in[k]) return set_error("gs_op64: op %d input %d is null", op, k);
        a.in[k] = in[k];
    }
    for (int k = 0; k < n_out[op]; ++k) {
        if (!out || !out[k]) return set_error("gs_op64: op %d output %d is null", op, k);
        a.out[k] = out[k];
    }
    const bool needs_cam = op >= GS_OP_WORLD_TO_CAMERA && op != GS_OP_PROJECT_COVARIANCE &&
                           op != GS_OP_BOUNDING_RADIUS && op != GS_OP_COV3D_BACKWARD;
    if (needs_cam && !cam) return set_error("gs_op64: op %d needs a camera", op);
    if (cam) {
        for (int k = 0; k < 16; ++k) a.view[k] = cam->view[k];
        a.fx = cam->fx; a.fy = cam->fy; a.cx = cam->cx; a.cy = cam->cy;
        a.W = cam->width; a.H = cam->height;
        a.near_plane = cam->near_plane; a.far_plane = cam->far_plane;
    }
    a.cols = cols;
    const int blocks = (int)((n + 127) / 128);
    op64_kernel<<<blocks, 128, 0, (cudaStream_t)stream>>>(op, (long long)n, a, status);
    return check_launch("op64_kernel");
}

}  // extern "C"
