// backward pass of the training-mode render (non-foveated,
// full-rate items, per-sample K = 16 window, Optimal Projection): the
// gradient of L = sum_px g_rgba . RGBA + g_depth * Depth with respect to the
// raw 3DGS parameters (means, quaternions, log-scales, opacity logits, SH),
// the differentiable rasterizer the paper fine-tunes with (P:106, P:164-165,
// P:311-316).  The blend order and the blended set are those of the forward
// frame (piecewise constant in the parameters); clamps contribute zero.
//
//   k_blend_bwd      one thread per pixel replays the forward (same staging,
//                    same window, same exact decisions) and, at every blend of
//                    entry k, forms dL/d alpha_k, dL/d tau_k, dL/d rgb_k from
//                    the prefix sums and the forward's outputs
//                    (d RGB / d alpha_k = rgb_k T_k - (RGB - C_<=k) / (1 - alpha_k),
//                    d A / d alpha_k = T / (1 - alpha_k), likewise for depth),
//                    chains them through q = num / s^2 and tau = d^T b / d^T A d
//                    to the splat record's coefficients and adds them into a
//                    per-(view, Gaussian) gradient record of 24 floats;
//   k_preproc_bwd    one thread per (view, Gaussian) with a non-zero record
//                    re-runs the activation + Optimal Projection (O1-O5) in
//                    forward-mode dual numbers over the 10 geometric inputs
//                    (mean 3, log-scale 3, raw quaternion 4), contracts with the
//                    record, and adds the SH, opacity and geometry gradients
//                    into the per-Gaussian outputs (views summed by atomics).
// The oracle is oracle/grad.py (plain PyTorch fp64 autograd over the C++
// oracle's blend orders), pinned by tests/test_grad_pins.py.
#include "k_blend_common.cuh"

namespace vrs {

namespace {

constexpr int kGB = 80;  // staged records per batch (as k_blend)
// Gradient arithmetic needs no bit-exactness (the replayed forward decisions
// do, and keep the R9 forms): its divisions use the fast MUFU reciprocal
// (relative error ~1e-7 against the 2e-3 gradient tolerance) instead of the
// IEEE division sequence.
#ifndef VRS_BWD_FASTDIV
#define VRS_BWD_FASTDIV 1
#endif
#if VRS_BWD_FASTDIV
#define GDIV(a, b) __fdividef((a), (b))
#else
#define GDIV(a, b) ((a) / (b))
#endif
// at most 2^VRS_BWD_STEPS lanes of a group are summed by shuffles before one of them adds
// (C9 backward: 15.9 ms with pairs (1), 16.4 with quads (2), 18.3 with octets (3), 20.7 with
// whole groups (5), 22.4 with every lane adding its own record: the shuffles, not the L2
// atomics, are the limit)
#ifndef VRS_BWD_STEPS
#define VRS_BWD_STEPS 1
#endif

// gradient record layout per (view, Gaussian)
enum : int { kGRgb = 0, kGSigma = 3, kGU = 4, kGE1x = 7, kGE1z = 8, kGE2 = 9, kGC = 12, kGA = 15, kGB3 = 21 };

struct BwdSmem {
    float4 r0[kGB], r1[kGB], r2[kGB], r3[kGB], r4[kGB], r5[kGB];
    uint32_t mask[kGB];
    float4 wblock[8];
    unsigned long long w_key[kWindow][256];
    float w_a[kWindow][256];
};

constexpr uint32_t kBSlot = 256 * 8;
constexpr uint32_t kBRing = (kWindow - 1) * kBSlot;

}  // namespace

__global__ void __launch_bounds__(256) k_blend_bwd(FrameParams fp, FrameBufs fb, const float* __restrict__ f_rgba,
                                                   const float* __restrict__ f_depth,
                                                   const float* __restrict__ g_rgba,
                                                   const float* __restrict__ g_depth, float* __restrict__ gbuf) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BwdSmem& S = *reinterpret_cast<BwdSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int vi = 0;
    const int item = blockIdx.x;
    while (vi + 1 < fp.n_views && item >= fp.v[vi + 1].item_off) vi++;
    const ViewParams& v = fp.v[vi];
    const uint32_t it = v.items[item - v.item_off];
    const int tile = (int)(it & 0xfffffu), sub = (int)((it >> 20) & 3u);
    const int T = fp.T;
    const int tx = tile % v.tw, ty = tile / v.tw;
    const int ox = tx * T + (T == 32 ? 16 * (sub & 1) : 0), oy = ty * T + (T == 32 ? 16 * (sub >> 1) : 0);
    const int px = ox + (warp & 1) * 8 + (lane & 7), py = oy + (warp >> 1) * 4 + (lane >> 3);
    const bool in_img = px < v.W && py < v.H;
    const float x = ((float)px + 0.5f - v.cx) / v.fx;
    const float y = ((float)py + 0.5f - v.cy) / v.fy;
    const float dn = sqrtf(fmaf(x, x, fmaf(y, y, 1.0f)));
    const uint32_t rb = fb.ranges[2 * (size_t)(v.tile_base + tile)];
    const uint32_t re = fb.ranges[2 * (size_t)(v.tile_base + tile) + 1];
    const float4* __restrict__ recv = fb.rec + (size_t)vi * fp.N * kRecF4;
    const float4* __restrict__ colv = fb.col + (size_t)vi * fp.N;
    float* __restrict__ gview = gbuf + (size_t)vi * fp.N * 24;
    // forward outputs and incoming gradients at this pixel
    float4 fo = make_float4(0.f, 0.f, 0.f, 0.f), go = fo;
    float fd = 0.0f, gd = 0.0f;
    if (in_img) {
        const size_t pi = (size_t)v.pix_off + (size_t)py * v.W + px;
        fo = reinterpret_cast<const float4*>(f_rgba)[pi];
        go = reinterpret_cast<const float4*>(g_rgba)[pi];
        fd = f_depth[pi];
        gd = g_depth[pi];
    }
    const float Tfin = 1.0f - fo.w;
    if (tid < 8) {  // per-warp sample extent (the forward's conservative footprint skip)
        const int wwx = (tid & 1) * 8, wwy = (tid >> 1) * 4;
        S.wblock[tid] = make_float4((float)(ox + wwx + 4), (float)(oy + wwy + 2), 3.5f, 1.5f);  // centre, half-extent
    }
    char* const wkb = reinterpret_cast<char*>(&S.w_key[0][tid]);
    char* const wab = reinterpret_cast<char*>(&S.w_a[0][tid]);
#define WK(off) (*reinterpret_cast<unsigned long long*>(wkb + (off)))
#define WA(off) (*reinterpret_cast<float*>(wab + ((off) >> 1)))
#pragma unroll
    for (int k = 0; k < kWindow; k++) {
        WK(k * kBSlot) = kSentinelKey;
        WA(k * kBSlot) = 0.0f;
    }
    float Tr = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f, Dd = 0.0f;
    bool done = !in_img;
    uint32_t hk = 0;

    // one blend of the forward, with its gradient contributions
    auto blend_bwd = [&](unsigned long long key, float a) {
        const uint32_t g = (uint32_t)key;
        const float tau = key_tau(key);
        const float Tk = Tr;
        const float wgt = a * Tk;
        if (a > 0.0f) {  // sentinels (alpha 0) blend nothing and have no gradient
            const float4 col = __ldg(colv + g);
            Cr = fmaf(col.x, wgt, Cr);
            Cg = fmaf(col.y, wgt, Cg);
            Cb = fmaf(col.z, wgt, Cb);
            Dd = fmaf(tau, wgt, Dd);
            const float inv1a = GDIV(1.0f, 1.0f - a);
            float ga = go.x * (col.x * Tk - (fo.x - Cr) * inv1a) + go.y * (col.y * Tk - (fo.y - Cg) * inv1a) +
                       go.z * (col.z * Tk - (fo.z - Cb) * inv1a) + go.w * Tfin * inv1a +
                       gd * (tau * dn * Tk - (fd - Dd * dn) * inv1a);
            const float4* rp = recv + (size_t)g * kRecF4;
            const float4 a0 = __ldg(rp + 0), a1 = __ldg(rp + 1), a2 = __ldg(rp + 2), a3 = __ldg(rp + 3),
                         a4 = __ldg(rp + 4), a5 = __ldg(rp + 5);
            // the 24 gradient components of this blend, added with six vector reductions
            float gv[24];
#pragma unroll
            for (int k = 0; k < 24; k++) gv[k] = 0.0f;
            gv[kGRgb + 0] = go.x * wgt;
            gv[kGRgb + 1] = go.y * wgt;
            gv[kGRgb + 2] = go.z * wgt;
            if (a < kAlphaMax) {  // alpha = sigma exp(-q/2) unclamped
                const float s = fmaf(a0.x, x, fmaf(a0.y, y, a0.z));
                const float ex = fmaf(a1.x, x, a1.y);
                const float ey = fmaf(a1.z, x, fmaf(a1.w, y, a2.x));
                const float num = fmaf(ex, fmaf(a2.y, ex, a2.z * ey), ey * fmaf(a2.z, ex, a2.w * ey));
                const float is = GDIV(1.0f, s);
                const float q = num * is * is;
                const float sigma = a5.y;
                gv[kGSigma] = ga * GDIV(a, sigma);
                const float gq = -0.5f * ga * a;
                const float gnum = gq * is * is, gs = -2.0f * gq * q * is;
                gv[kGC + 0] = gnum * ex * ex;
                gv[kGC + 1] = gnum * 2.0f * ex * ey;
                gv[kGC + 2] = gnum * ey * ey;
                const float gex = 2.0f * gnum * fmaf(a2.y, ex, a2.z * ey);
                const float gey = 2.0f * gnum * fmaf(a2.z, ex, a2.w * ey);
                gv[kGE1x] = gex * x;
                gv[kGE1z] = gex;
                gv[kGE2 + 0] = gey * x;
                gv[kGE2 + 1] = gey * y;
                gv[kGE2 + 2] = gey;
                gv[kGU + 0] = gs * x;
                gv[kGU + 1] = gs * y;
                gv[kGU + 2] = gs;
            }
            if (tau > fp.near_plane) {  // tau = dtb / den unclamped
                const float den = quad3z1(a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, x, y);
                const float gt = gd * dn * wgt;
                const float rden = GDIV(1.0f, den);
                const float gdtb = gt * rden, gden = -gt * tau * rden;
                gv[kGB3 + 0] = gdtb * x;
                gv[kGB3 + 1] = gdtb * y;
                gv[kGB3 + 2] = gdtb;
                gv[kGA + 0] = gden * x * x;
                gv[kGA + 1] = gden * 2.0f * x * y;
                gv[kGA + 2] = gden * 2.0f * x;
                gv[kGA + 3] = gden * y * y;
                gv[kGA + 4] = gden * 2.0f * y;
                gv[kGA + 5] = gden;
            }
            float* gr = gview + (size_t)g * 24;
#ifndef VRS_BWD_NO_AGG
            // lanes blending the same Gaussian at this instant sum their records first:
            // suffix sums along the group's lanes by pointer jumping (each lane links to
            // the next lane of its group; every step doubles the links): after s steps
            // the lane of group rank r holds ranks r .. r + 2^s - 1, and the lanes of rank
            // 0 mod 2^s add them
            const unsigned act = __activemask();
            const unsigned peers = __match_any_sync(act, g);
            const int nmax = min((int)__reduce_max_sync(act, (unsigned)__popc(peers)), 1 << VRS_BWD_STEPS);
            const unsigned above = peers & ~((2u << lane) - 1u);  // (lane 31: 2u << 31 = 0 -> none)
            int nxt = above ? __ffs(above) - 1 : -1;
            for (int st = 1; st < nmax; st <<= 1) {
                const int src = nxt >= 0 ? nxt : lane;
#pragma unroll
                for (int k = 0; k < 24; k++) {
                    const float o = __shfl_sync(act, gv[k], src);
                    gv[k] += nxt >= 0 ? o : 0.0f;
                }
                const int nn = __shfl_sync(act, nxt, src);
                nxt = nxt >= 0 ? nn : -1;
            }
            if ((__popc(peers & ((1u << lane) - 1u)) & ((1 << VRS_BWD_STEPS) - 1)) == 0)
#endif
#pragma unroll
            for (int k = 0; k < 24; k += 4)  // (skipping all-zero vectors measured slower: the tests cost more)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(gr + k), "f"(gv[k]),
                             "f"(gv[k + 1]), "f"(gv[k + 2]), "f"(gv[k + 3])
                             : "memory");
        }
        Tr = Tr * (1.0f - a);
        done = Tr < kTmin;
    };
    auto contribute = [&](const unsigned long long key, const float alpha) {
        const unsigned long long kh = WK(hk);
        const bool direct = key < kh;
        const float ah = WA(hk);
        blend_bwd(direct ? key : kh, direct ? alpha : ah);
        if (direct || done) return;
        hk = (hk + kBSlot) & kBRing;
        uint32_t jo = (hk + (kWindow - 2) * kBSlot) & kBRing;
        uint32_t dst = (jo + kBSlot) & kBRing;
        unsigned long long kj = WK(jo);
        int left = kWindow - 1;
#pragma unroll 1
        while (kj > key) {
            WK(dst) = kj;
            WA(dst) = WA(jo);
            dst = jo;
            if (--left == 0) break;
            jo = (jo - kBSlot) & kBRing;
            kj = WK(jo);
        }
        WK(dst) = key;
        WA(dst) = alpha;
    };

    for (uint32_t base = rb; base < re; base += kGB) {
        __syncthreads();
        const uint32_t idx = base + tid;
        if (tid < kGB && idx < re) {
            uint32_t g = __ldg(fb.vals + idx);
            g = (g < (uint32_t)fp.N) ? g : 0u;
            const float4* rp = recv + (size_t)g * kRecF4;
            S.r0[tid] = __ldg(rp + 0);
            S.r1[tid] = __ldg(rp + 1);
            S.r2[tid] = __ldg(rp + 2);
            S.r3[tid] = __ldg(rp + 3);
            S.r4[tid] = __ldg(rp + 4);
            const float4 a5 = __ldg(rp + 5), a7 = __ldg(rp + 7);
            S.r5[tid] = make_float4(a5.x, a5.y, __uint_as_float(g), 0.0f);
            S.mask[tid] = footprint_mask<8>(a7, S.wblock);
        }
        if (__syncthreads_count(!done) == 0) break;
        const int nb = min((int)(re - base), kGB);
        for (int c = 0; c < nb; c += 32) {
          if (__all_sync(0xffffffffu, done)) break;
          unsigned bits = __ballot_sync(0xffffffffu, (c + lane < nb) && ((S.mask[c + lane] >> warp) & 1u));
          while (bits) {
            const int j = c + __ffs(bits) - 1;
            bits &= bits - 1;
            if (done) continue;
            const float4 a0 = S.r0[j], a1 = S.r1[j], a2 = S.r2[j];
            const float s = fmaf(a0.x, x, fmaf(a0.y, y, a0.z));
            const float ex = fmaf(a1.x, x, a1.y);
            const float ey = fmaf(a1.z, x, fmaf(a1.w, y, a2.x));
            const float cx = fmaf(a2.y, ex, a2.z * ey), cy = fmaf(a2.z, ex, a2.w * ey);
            const float num = fmaf(ex, cx, ey * cy);
            const float ss = s * s;
            if (!(s > 0.0f) || !(num <= a0.w * ss)) continue;
            const float4 a3 = S.r3[j], a4 = S.r4[j], t = S.r5[j];
            const float den = quad3z1(a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, x, y);
            const float dtb = fmaf(a4.z, x, fmaf(a4.w, y, t.x));
            float tau;
            const float alpha = alpha_tau(num, ss, den, dtb, t.y, tau);
            contribute(order_key(tau, __float_as_uint(t.z), fp.near_plane), alpha);
          }
        }
    }
#pragma unroll 1
    for (int k = 0; k < kWindow && !done; k++) {
        blend_bwd(WK(hk), WA(hk));
        hk = (hk + kBSlot) & kBRing;
    }
#undef WK
#undef WA
}

// ------------------------------------------------------------------ dual numbers
namespace {

constexpr int kND = 10;  // mean 3, log-scale 3, raw quaternion 4
struct Dl {
    float v;
    float d[kND];
};
__device__ __forceinline__ Dl dconst(float c) {
    Dl r;
    r.v = c;
#pragma unroll
    for (int i = 0; i < kND; i++) r.d[i] = 0.0f;
    return r;
}
__device__ __forceinline__ Dl operator+(const Dl& a, const Dl& b) {
    Dl r;
    r.v = a.v + b.v;
#pragma unroll
    for (int i = 0; i < kND; i++) r.d[i] = a.d[i] + b.d[i];
    return r;
}
__device__ __forceinline__ Dl operator-(const Dl& a, const Dl& b) {
    Dl r;
    r.v = a.v - b.v;
#pragma unroll
    for (int i = 0; i < kND; i++) r.d[i] = a.d[i] - b.d[i];
    return r;
}
__device__ __forceinline__ Dl operator*(const Dl& a, const Dl& b) {
    Dl r;
    r.v = a.v * b.v;
#pragma unroll
    for (int i = 0; i < kND; i++) r.d[i] = fmaf(a.d[i], b.v, a.v * b.d[i]);
    return r;
}
__device__ __forceinline__ Dl operator*(const Dl& a, float c) {
    Dl r;
    r.v = a.v * c;
#pragma unroll
    for (int i = 0; i < kND; i++) r.d[i] = a.d[i] * c;
    return r;
}
__device__ __forceinline__ Dl operator*(float c, const Dl& a) { return a * c; }
__device__ __forceinline__ Dl operator+(const Dl& a, float c) {
    Dl r = a;
    r.v += c;
    return r;
}
__device__ __forceinline__ Dl operator-(const Dl& a) { return a * -1.0f; }
__device__ __forceinline__ Dl dinv(const Dl& a) {
    Dl r;
    r.v = 1.0f / a.v;
    const float k = -r.v * r.v;
#pragma unroll
    for (int i = 0; i < kND; i++) r.d[i] = a.d[i] * k;
    return r;
}
__device__ __forceinline__ Dl operator/(const Dl& a, const Dl& b) { return a * dinv(b); }
__device__ __forceinline__ Dl dsqrt(const Dl& a) {
    Dl r;
    r.v = sqrtf(a.v);
    const float k = 0.5f / r.v;
#pragma unroll
    for (int i = 0; i < kND; i++) r.d[i] = a.d[i] * k;
    return r;
}
__device__ __forceinline__ Dl dexp(const Dl& a) {
    Dl r;
    r.v = expf(a.v);
#pragma unroll
    for (int i = 0; i < kND; i++) r.d[i] = a.d[i] * r.v;
    return r;
}

}  // namespace

// SH basis (3DGS convention, as k_color) at unit direction (x, y, z) in duals
__device__ __forceinline__ int sh_basis_d(const Dl& x, const Dl& y, const Dl& z, int deg, Dl* B) {
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    int n = 0;
    B[n++] = dconst(C0);
    if (deg > 0) {
        B[n++] = y * -C1;
        B[n++] = z * C1;
        B[n++] = x * -C1;
    }
    if (deg > 1) {
        const Dl xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
        B[n++] = xy * 1.0925484305920792f;
        B[n++] = yz * -1.0925484305920792f;
        B[n++] = (zz * 2.0f - xx - yy) * 0.31539156525252005f;
        B[n++] = xz * -1.0925484305920792f;
        B[n++] = (xx - yy) * 0.5462742152960396f;
        if (deg > 2) {
            B[n++] = y * (xx * 3.0f - yy) * -0.5900435899266435f;
            B[n++] = xy * z * 2.890611442640554f;
            B[n++] = y * (zz * 4.0f - xx - yy) * -0.4570457994644658f;
            B[n++] = z * (zz * 2.0f - xx * 3.0f - yy * 3.0f) * 0.3731763325901154f;
            B[n++] = x * (zz * 4.0f - xx - yy) * -0.4570457994644658f;
            B[n++] = z * (xx - yy) * 1.445305721320277f;
            B[n++] = x * (xx - yy * 3.0f) * -0.5900435899266435f;
        }
    }
    return n;
}

__global__ void __launch_bounds__(128) k_preproc_bwd(FrameParams fp, const float4* __restrict__ mu4,
                                                     const float4* __restrict__ raw, const float* __restrict__ sh,
                                                     int sh_stride, const float* __restrict__ gbuf,
                                                     float* __restrict__ g_means, float* __restrict__ g_quats,
                                                     float* __restrict__ g_ls, float* __restrict__ g_logits,
                                                     float* __restrict__ g_sh, int64_t total) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int vi = (int)(t / fp.N);
    const int64_t g = t - (int64_t)vi * fp.N;
    const float* G = gbuf + (size_t)t * 24;
    float Gv[24];
    bool any = false;
#pragma unroll
    for (int k = 0; k < 24; k++) {
        Gv[k] = G[k];
        any = any || Gv[k] != 0.0f;
    }
    if (!any) return;
    const ViewParams& v = fp.v[vi];
    // inputs with their seeds
    const float4 m4 = mu4[g], q4 = raw[2 * g], l4 = raw[2 * g + 1];
    Dl m[3], ls[3], q[4];
    const float mv[3] = {m4.x, m4.y, m4.z}, lv[3] = {l4.x, l4.y, l4.z}, qv[4] = {q4.x, q4.y, q4.z, q4.w};
    for (int i = 0; i < 3; i++) {
        m[i] = dconst(mv[i]);
        m[i].d[i] = 1.0f;
        ls[i] = dconst(lv[i]);
        ls[i].d[3 + i] = 1.0f;
    }
    for (int i = 0; i < 4; i++) {
        q[i] = dconst(qv[i]);
        q[i].d[6 + i] = 1.0f;
    }
    // activation (L1): normalised quaternion, R, Sigma = R S^2 R^T, Sigma^-1 = R S^-2 R^T
    const Dl qi = dinv(dsqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]));
    const Dl w = q[0] * qi, x = q[1] * qi, y = q[2] * qi, z = q[3] * qi;
    Dl R[3][3];
    R[0][0] = dconst(1.0f) - (y * y + z * z) * 2.0f;
    R[0][1] = (x * y - w * z) * 2.0f;
    R[0][2] = (x * z + w * y) * 2.0f;
    R[1][0] = (x * y + w * z) * 2.0f;
    R[1][1] = dconst(1.0f) - (x * x + z * z) * 2.0f;
    R[1][2] = (y * z - w * x) * 2.0f;
    R[2][0] = (x * z - w * y) * 2.0f;
    R[2][1] = (y * z + w * x) * 2.0f;
    R[2][2] = dconst(1.0f) - (x * x + y * y) * 2.0f;
    Dl s2[3], is2[3];
    for (int k = 0; k < 3; k++) {
        s2[k] = dexp(ls[k] * 2.0f);
        is2[k] = dinv(s2[k]);
    }
    // Sigma_c = W Sigma W^T with Sigma = sum_k s2_k r_k r_k^T (r_k = column k of R): P = W R
    float Wm[3][3];
    for (int i = 0; i < 9; i++) Wm[i / 3][i % 3] = v.R[i];
    Dl P[3][3];
    for (int i = 0; i < 3; i++)
        for (int k = 0; k < 3; k++) P[i][k] = R[0][k] * Wm[i][0] + R[1][k] * Wm[i][1] + R[2][k] * Wm[i][2];
    // camera-frame mean, optimal-plane frame
    Dl vv[3], mc[3];
    for (int i = 0; i < 3; i++) vv[i] = m[i] + (-v.o[i]);
    for (int i = 0; i < 3; i++) mc[i] = vv[0] * Wm[i][0] + vv[1] * Wm[i][1] + vv[2] * Wm[i][2];
    const Dl r = dsqrt(mc[0] * mc[0] + mc[1] * mc[1] + mc[2] * mc[2]);
    const Dl ir = dinv(r);
    Dl u[3];
    for (int i = 0; i < 3; i++) u[i] = mc[i] * ir;
    const Dl ih = dinv(dsqrt(u[2] * u[2] + u[0] * u[0]));
    Dl e1[3], e2[3];
    e1[0] = u[2] * ih;
    e1[1] = dconst(0.0f);
    e1[2] = -(u[0] * ih);
    e2[0] = u[1] * e1[2];
    e2[1] = u[2] * e1[0] - u[0] * e1[2];
    e2[2] = -(u[1] * e1[0]);
    // Sigma_2 = E^T Sigma_c E / r^2 + dilation: with pe_k = P^T e (per column k), e^T Sigma_c f = sum_k s2_k pe_k pf_k
    Dl p1[3], p2[3];
    for (int k = 0; k < 3; k++) {
        p1[k] = P[0][k] * e1[0] + P[2][k] * e1[2];  // e1.y = 0
        p2[k] = P[0][k] * e2[0] + P[1][k] * e2[1] + P[2][k] * e2[2];
    }
    const Dl ir2 = ir * ir;
    Dl s00 = (s2[0] * p1[0] * p1[0] + s2[1] * p1[1] * p1[1] + s2[2] * p1[2] * p1[2]) * ir2;
    Dl s01 = (s2[0] * p1[0] * p2[0] + s2[1] * p1[1] * p2[1] + s2[2] * p1[2] * p2[2]) * ir2;
    Dl s11 = (s2[0] * p2[0] * p2[0] + s2[1] * p2[1] * p2[1] + s2[2] * p2[2] * p2[2]) * ir2;
    const Dl jx = u[2] * (1.0f / v.fx), jy = u[2] * (1.0f / v.fy);
    const Dl J00 = e1[0] * jx, J10 = e2[0] * jx, J11 = e2[1] * jy;  // J01 = e1.y jy = 0
    s00 = s00 + J00 * J00 * 0.3f;
    s01 = s01 + J00 * J10 * 0.3f;
    s11 = s11 + (J10 * J10 + J11 * J11) * 0.3f;
    const Dl idet = dinv(s00 * s11 - s01 * s01);
    const Dl C00 = s11 * idet, C01 = -(s01 * idet), C11 = s00 * idet;
    // A = W Sigma^-1 W^T = sum_k is2_k P_k P_k^T, b = A mu_c
    Dl A[6];
    const int I[6] = {0, 0, 0, 1, 1, 2}, J[6] = {0, 1, 2, 1, 2, 2};
    for (int e = 0; e < 6; e++)
        A[e] = is2[0] * P[I[e]][0] * P[J[e]][0] + is2[1] * P[I[e]][1] * P[J[e]][1] + is2[2] * P[I[e]][2] * P[J[e]][2];
    Dl bvec[3];
    bvec[0] = A[0] * mc[0] + A[1] * mc[1] + A[2] * mc[2];
    bvec[1] = A[1] * mc[0] + A[3] * mc[1] + A[4] * mc[2];
    bvec[2] = A[2] * mc[0] + A[4] * mc[1] + A[5] * mc[2];
    // contraction with the gradient record (order: rgb 3, sigma, u 3, e1x, e1z, e2 3, C 3, A 6, b 3)
    float acc[kND];
    for (int i = 0; i < kND; i++) acc[i] = 0.0f;
    auto add = [&](const Dl& o, float gk) {
        if (gk == 0.0f) return;
        for (int i = 0; i < kND; i++) acc[i] = fmaf(gk, o.d[i], acc[i]);
    };
    for (int i = 0; i < 3; i++) add(u[i], Gv[kGU + i]);
    add(e1[0], Gv[kGE1x]);
    add(e1[2], Gv[kGE1z]);
    for (int i = 0; i < 3; i++) add(e2[i], Gv[kGE2 + i]);
    add(C00, Gv[kGC + 0]);
    add(C01, Gv[kGC + 1]);
    add(C11, Gv[kGC + 2]);
    for (int e = 0; e < 6; e++) add(A[e], Gv[kGA + e]);
    for (int i = 0; i < 3; i++) add(bvec[i], Gv[kGB3 + i]);
    // colour: rgb_c = max(0, sum_k Y_k(dir) sh_kc + 0.5), dir = (mu - o) / |mu - o| (world frame)
    const Dl iv = dinv(dsqrt(vv[0] * vv[0] + vv[1] * vv[1] + vv[2] * vv[2]));
    Dl B[16];
    const int nb = sh_basis_d(vv[0] * iv, vv[1] * iv, vv[2] * iv, fp.sh_coeffs == 1 ? 0 : (fp.sh_coeffs == 4 ? 1 :
                              (fp.sh_coeffs == 9 ? 2 : 3)), B);
    const int ncoef = fp.sh_coeffs;
    const float* shg = sh + (size_t)g * sh_stride;  // device layout: [N][chunks] float4, coefficient-major RGB
    float* gsh = g_sh + (size_t)g * ncoef * 3;
    for (int c = 0; c < 3; c++) {
        const float gc = Gv[kGRgb + c];
        if (gc == 0.0f) continue;
        Dl val = dconst(0.5f);
        for (int k = 0; k < nb; k++) val = val + B[k] * shg[k * 3 + c];
        if (!(val.v > 0.0f)) continue;  // clamped colour: no gradient
        add(val, gc);
        for (int k = 0; k < nb; k++) atomicAdd(gsh + k * 3 + c, gc * B[k].v);
    }
    // opacity: sigma = sigmoid(logit)
    if (Gv[kGSigma] != 0.0f) {
        const float sg = 1.0f / (1.0f + expf(-l4.w));
        atomicAdd(g_logits + g, Gv[kGSigma] * sg * (1.0f - sg));
    }
    for (int i = 0; i < 3; i++) atomicAdd(g_means + 3 * g + i, acc[i]);
    for (int i = 0; i < 3; i++) atomicAdd(g_ls + 3 * g + i, acc[3 + i]);
    for (int i = 0; i < 4; i++) atomicAdd(g_quats + 4 * g + i, acc[6 + i]);
}

void launch_backward(const FrameParams& fp, FrameBufs fb, int total_items, const float4* mu4, const float4* raw,
                     const float* sh, int sh_stride, const float* f_rgba, const float* f_depth, const float* g_rgba,
                     const float* g_depth, float* gbuf, float* g_means, float* g_quats, float* g_ls,
                     float* g_logits, float* g_sh, cudaStream_t st) {
    if (total_items > 0) {
        const size_t smem = sizeof(BwdSmem);
        ensure_smem_attr((const void*)k_blend_bwd, (int)smem);
        k_blend_bwd<<<(unsigned)total_items, 256, smem, st>>>(fp, fb, f_rgba, f_depth, g_rgba, g_depth, gbuf);
    }
    const int64_t total = (int64_t)fp.n_views * fp.N;
    if (total > 0)
        k_preproc_bwd<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(fp, mu4, raw, sh, sh_stride, gbuf, g_means,
                                                                       g_quats, g_ls, g_logits, g_sh, total);
}

}  // namespace vrs
