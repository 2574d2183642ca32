// the paper's two-pass foveated baseline (App. A).
// Pass 1 renders the fovea rectangle plus its transition band at full
// resolution through a cropped camera (tight frustum); pass 2 renders the
// whole view at half resolution honouring the visibility mask; both passes
// of all views go through ONE vrs render call (vrs_api.cu).  This file holds
// the two pieces that are specific to the baseline:
//   k_mask_half          visibility mask for pass 2: a half-resolution pixel
//                        is visible iff any of its (up to) 2x2 pixels is;
//   k_two_pass_combine   bilinear upsampling of pass 2 (pixel-centre aligned:
//                        full-res pixel i samples pass-2 coordinate (i-0.5)/2,
//                        edge-clamped -- the NPP resize convention of P:765)
//                        and the blend w*P1 + (1-w)*up(P2) with the same
//                        continuous fovea weight as the single-pass hybrid
//                        ramp, per channel of RGBA and depth.
#include <algorithm>

#include "vrs_internal.cuh"

namespace vrs {

__global__ void k_mask_half(const uint8_t* __restrict__ src, int W, int H, uint8_t* __restrict__ dst, int W2, int H2) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (int64_t)W2 * H2) return;
    const int i2 = (int)(k % W2), j2 = (int)(k / W2);
    uint8_t m = 0;
    for (int b = 0; b < 2; b++)
        for (int a = 0; a < 2; a++) {
            const int i = 2 * i2 + a, j = 2 * j2 + b;
            if (i < W && j < H) m |= src[(size_t)j * W + i];
        }
    dst[k] = m ? 1 : 0;
}

__global__ void k_two_pass_combine(TwoPassParams tp, const float4* __restrict__ prgba, const float* __restrict__ pdepth,
                                   float* __restrict__ rgba, float* __restrict__ depth, int64_t total) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        int vi = 0;
        while (vi + 1 < tp.n && k >= tp.v[vi + 1].out_off) vi++;
        const TwoPassView& t = tp.v[vi];
        const int64_t loc = k - t.out_off;
        const int i = (int)(loc % t.W), j = (int)(loc / t.W);
        // bilinear pass-2 sample
        const float u = ((float)i - 0.5f) * 0.5f, w = ((float)j - 0.5f) * 0.5f;
        const float fu = floorf(u), fw = floorf(w);
        const float ax = u - fu, ay = w - fw;
        const int xa = min(max((int)fu, 0), t.W2 - 1), xb = min(max((int)fu + 1, 0), t.W2 - 1);
        const int ya = min(max((int)fw, 0), t.H2 - 1), yb = min(max((int)fw + 1, 0), t.H2 - 1);
        const int64_t r0 = t.p2_off + (int64_t)ya * t.W2, r1 = t.p2_off + (int64_t)yb * t.W2;
        const float w00 = (1.0f - ax) * (1.0f - ay), w10 = ax * (1.0f - ay), w01 = (1.0f - ax) * ay, w11 = ax * ay;
        const float4 c00 = prgba[r0 + xa], c10 = prgba[r0 + xb], c01 = prgba[r1 + xa], c11 = prgba[r1 + xb];
        float4 c;
        c.x = w00 * c00.x + w10 * c10.x + w01 * c01.x + w11 * c11.x;
        c.y = w00 * c00.y + w10 * c10.y + w01 * c01.y + w11 * c11.y;
        c.z = w00 * c00.z + w10 * c10.z + w01 * c01.z + w11 * c11.z;
        c.w = w00 * c00.w + w10 * c10.w + w01 * c01.w + w11 * c11.w;
        float d = w00 * pdepth[r0 + xa] + w10 * pdepth[r0 + xb] + w01 * pdepth[r1 + xa] + w11 * pdepth[r1 + xb];
        // fovea weight (the single-pass ramp), pass 1 inside its rectangle
        const int ci = i - t.i0, cj = j - t.j0;
        if (ci >= 0 && cj >= 0 && ci < t.w1 && cj < t.h1) {
            ViewParams fv;
            fv.gx = t.gx; fv.gy = t.gy; fv.rx = t.rx; fv.ry = t.ry; fv.ramp = t.ramp;
            const float wf = fovea_weight(fv, (float)i + 0.5f, (float)j + 0.5f);
            if (wf > 0.0f) {
                const int64_t p1 = t.p1_off + (int64_t)cj * t.w1 + ci;
                const float4 a = prgba[p1];
                const float ad = pdepth[p1];
                const float wb = 1.0f - wf;
                c = make_float4(wf * a.x + wb * c.x, wf * a.y + wb * c.y, wf * a.z + wb * c.z, wf * a.w + wb * c.w);
                d = wf * ad + wb * d;
            }
        }
        store_pixel(tp.out_fmt, rgba, depth, (size_t)k, c, d);
    }
}

void launch_mask_half(const uint8_t* src, int W, int H, uint8_t* dst, int W2, int H2, cudaStream_t st) {
    const int64_t n = (int64_t)W2 * H2;
    if (n == 0) return;
    k_mask_half<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, W, H, dst, W2, H2);
}

void launch_two_pass_combine(const TwoPassParams& tp, const float4* prgba, const float* pdepth, float* rgba,
                             float* depth, int64_t total, cudaStream_t st) {
    if (total == 0) return;
    const int sms = device_sms();
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sms * 16);
    k_two_pass_combine<<<(unsigned)blocks, 256, 0, st>>>(tp, prgba, pdepth, rgba, depth, total);
}

}  // namespace vrs
