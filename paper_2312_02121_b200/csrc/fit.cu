// fit.cu -- the training step around the hot path:
// sg/optimize.py:96-190 fit, one iteration =
//   activate (exp / sigmoid, :144-145) -> render -> L2 loss + d_image
//   (:157-158, :163 passes 2 * resid) -> scene backward -> chain to log /
//   logit space (:167, :172) -> Adam per parameter class (:84-89) ->
//   clip colours (:176).
// gs_loss_l2 and gs_adam_step are the two fused kernels; with the frame
// entry points an iteration is capturable in one CUDA graph (no host sync:
// the loss goes to a device array).
#include "common.cuh"

namespace gs {

// d_image = 2 (image - target); loss[0] += sum (image - target)^2 (fp64).
__global__ void __launch_bounds__(256) loss_l2_kernel(const float* __restrict__ img, const float* __restrict__ tgt,
                                                      int64_t n, float* __restrict__ d_img,
                                                      double* __restrict__ loss) {
    __shared__ double s_part[8];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float r = img[i] - tgt[i];
        d_img[i] = 2.f * r;
        acc += (double)r * (double)r;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_part[w];
        atomicAdd(loss, t);
    }
}

struct AdamHyper {
    float lr_mean, lr_scale, lr_quat, lr_opacity, lr_color;
    float beta1, beta2, eps;
    float bc1, bc2;  // 1 - beta^step
};

__device__ __forceinline__ float adam_update(float p, float g, float& m, float& v, float lr, const AdamHyper& h) {
    m = h.beta1 * m + (1.f - h.beta1) * g;
    v = h.beta2 * v + (1.f - h.beta2) * g * g;
    const float mh = m / h.bc1, vh = v / h.bc2;
    return p - lr * mh / (sqrtf(vh) + h.eps);
}

// One Adam step for every Gaussian (sg/optimize.py:84-89,165-176) and the
// activated parameters for the next render.  grads: d_mean (n,3),
// d_scale (n,3), d_quat (n,4), d_rgbo (n,4) = d_color, d_opacity.
// State m, v: (n,14) each, column order mean 3 | log_scale 3 | quat 4 |
// logit 1 | color 3.
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ means, float* __restrict__ log_scales,
                                                   float* __restrict__ quats, float* __restrict__ logits,
                                                   float* __restrict__ colors, float* __restrict__ scales,
                                                   float* __restrict__ opac, const float* __restrict__ d_mean,
                                                   const float* __restrict__ d_scale, const float* __restrict__ d_quat,
                                                   const float4* __restrict__ d_rgbo, float* __restrict__ m,
                                                   float* __restrict__ v, int n, AdamHyper h) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float* mi = m + 14 * (size_t)i;
    float* vi = v + 14 * (size_t)i;
#pragma unroll
    for (int c = 0; c < 3; ++c) means[3 * i + c] = adam_update(means[3 * i + c], d_mean[3 * i + c], mi[c], vi[c],
                                                               h.lr_mean, h);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        // d/d log s = s * d/d s (:167), s the scale of this iteration's render
        const float g = d_scale[3 * i + c] * scales[3 * i + c];
        const float ls = adam_update(log_scales[3 * i + c], g, mi[3 + c], vi[3 + c], h.lr_scale, h);
        log_scales[3 * i + c] = ls;
        scales[3 * i + c] = expf(ls);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) quats[4 * i + c] = adam_update(quats[4 * i + c], d_quat[4 * i + c], mi[6 + c],
                                                               vi[6 + c], h.lr_quat, h);
    const float4 dr = d_rgbo[i];
    {
        const float o = opac[i];
        const float g = dr.w * o * (1.f - o);  // logit chain (:172)
        const float lg = adam_update(logits[i], g, mi[10], vi[10], h.lr_opacity, h);
        logits[i] = lg;
        opac[i] = 1.f / (1.f + expf(-lg));
    }
    const float dc[3] = {dr.x, dr.y, dr.z};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float col = adam_update(colors[3 * i + c], dc[c], mi[11 + c], vi[11 + c], h.lr_color, h);
        colors[3 * i + c] = fminf(fmaxf(col, 0.f), 1.f);  // clip (:176)
    }
}

// scales = exp(log_scales), opac = sigmoid(logits) (sg/optimize.py:144-145)
__global__ void __launch_bounds__(256) activate_kernel(const float* __restrict__ log_scales,
                                                       const float* __restrict__ logits, float* __restrict__ scales,
                                                       float* __restrict__ opac, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    scales[3 * i] = expf(log_scales[3 * i]);
    scales[3 * i + 1] = expf(log_scales[3 * i + 1]);
    scales[3 * i + 2] = expf(log_scales[3 * i + 2]);
    opac[i] = 1.f / (1.f + expf(-logits[i]));
}

}  // namespace gs

using namespace gs;

extern "C" {

int gs_loss_l2(const float* image, const float* target, int64_t n, float* d_image, double* loss,
               gs_stream_t stream) {
    if (n < 0) return set_error("gs_loss_l2: negative n");
    if (n == 0) return 0;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    loss_l2_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(image, target, n, d_image, loss);
    return check_launch("loss_l2_kernel");
}

int gs_activate(const float* log_scales3, const float* logits, float* scales3, float* opacities, int64_t n,
                gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_activate: n out of range");
    if (n == 0) return 0;
    activate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(log_scales3, logits, scales3,
                                                                                  opacities, (int)n);
    return check_launch("activate_kernel");
}

int gs_adam_step(float* means3, float* log_scales3, float* quats4, float* logits, float* colors3, float* scales3,
                 float* opacities, const float* d_means3, const float* d_scales3, const float* d_quats4,
                 const float* d_rgbo4, float* adam_m14, float* adam_v14, int64_t n, int step, const float* lrs5,
                 float beta1, float beta2, float eps, gs_stream_t stream) {
    if (n < 0 || n > 0x7fffffff) return set_error("gs_adam_step: n out of range");
    if (step < 1) return set_error("gs_adam_step: step must be >= 1");
    if (n == 0) return 0;
    AdamHyper h;
    h.lr_mean = lrs5[0]; h.lr_scale = lrs5[1]; h.lr_quat = lrs5[2]; h.lr_opacity = lrs5[3]; h.lr_color = lrs5[4];
    h.beta1 = beta1; h.beta2 = beta2; h.eps = eps;
    h.bc1 = (float)(1.0 - pow((double)beta1, (double)step));
    h.bc2 = (float)(1.0 - pow((double)beta2, (double)step));
    adam_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        means3, log_scales3, quats4, logits, colors3, scales3, opacities, d_means3, d_scales3, d_quats4,
        (const float4*)d_rgbo4, adam_m14, adam_v14, (int)n, h);
    return check_launch("adam_kernel");
}

}  // extern "C"
