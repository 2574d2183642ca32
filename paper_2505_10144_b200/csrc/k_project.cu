// Per-Gaussian stage and Gaussian/tile
// instantiation (step 3): Optimal Projection, SH colour,
// conservative footprint, exact per-tile culling with Eq.4 on the optimal
// plane, StopThePop per-tile depth at the back-projected maximum
// point and visibility-mask skipping through the SAT.
//
// k_cull: one thread per Gaussian tests every view's frustum cone (the
// Gaussian's attributes read once for all views: stereo fusion of the
// per-Gaussian stage, the "fusion of stereo rendering passes" of P:735) and
// appends the surviving (view, Gaussian) candidates; k_preprocess projects
// them and expands their footprint tiles into the test list; k_color
// evaluates the SH colour of the visible ones (on the side stream);
// k_tiletest_direct runs one Eq.4 test per (Gaussian, tile) candidate.
#include <algorithm>

#include "vrs_internal.cuh"

namespace vrs {

struct Proj {
    int valid;
    float muc[3], u[3], e1[3], e2[3];
    float S2[3], C[3], eps;
    float A[6], bv[3];
    float sigma, qcut;
    int rect[4];
    float bbox[4];
    float m2[2], Cp[3];  // EWA baseline: pixel mean and conic
    uint32_t foot[4];    // record slot 7: packed conservative footprint (vrs_internal.cuh Footprint)
};

// Record slot 7 (vrs_internal.cuh footprint_of): the bounding box rounded
// outward to int16, and -- for an ellipse, ax = {minor-axis unit vector (2),
// centre z0 (2), r^2, Q00, Q01, Q11, det} of the pixel-space conic
// (z - z0)^T M (z - z0) <= r^2, M = [[Q00, Q01], [Q01, Q11]] -- a separating
// axis: n rounded to binary16, the centre's offset d from the box centre
// along n and the half-width r sqrt(n^T M^-1 n) + |d rounding| + 1 px,
// rounded up; else (have_ax false) n = 0 and an infinite half-width: box only.
#ifndef VRS_FOOT_MARGIN
#define VRS_FOOT_MARGIN 1.0
#endif
__device__ __forceinline__ void pack_footprint(Proj& p, const bool have_ax, const double ax0 = 0.0, const double ax1 = 0.0,
                                               const double ax2 = 0.0, const double ax3 = 0.0, const double ax4 = 0.0,
                                               const double ax5 = 0.0, const double ax6 = 0.0, const double ax7 = 0.0,
                                               const double ax8 = 0.0) {
    const double ax[9] = {ax0, ax1, ax2, ax3, ax4, ax5, ax6, ax7, ax8};
    auto i16 = [](double v) { return (uint32_t)(uint16_t)(int16_t)fmin(fmax(v, -32768.0), 32767.0); };
    const double bx0 = floor((double)p.bbox[0]), bx1 = ceil((double)p.bbox[1]);
    const double by0 = floor((double)p.bbox[2]), by1 = ceil((double)p.bbox[3]);
    p.foot[0] = i16(bx0) | (i16(bx1) << 16);
    p.foot[1] = i16(by0) | (i16(by1) << 16);
    __half2 n = __floats2half2_rn(0.0f, 0.0f);
    __half2 dh = __halves2half2(__float2half_rn(0.0f), __ushort_as_half((unsigned short)0x7c00u));  // (0, +inf)
    if (have_ax && bx0 > -32768.0 && bx1 < 32767.0 && by0 > -32768.0 && by1 < 32767.0) {
        const __half hx = __double2half(ax[0]), hy = __double2half(ax[1]);
        const double nx = (double)__half2float(hx), ny = (double)__half2float(hy);
        const double q = nx * nx * ax[7] - 2.0 * nx * ny * ax[6] + ny * ny * ax[5];  // det * n^T M^-1 n
        const double ext = sqrt(ax[4] * q / ax[8]);
        const double d = nx * (ax[2] - 0.5 * (bx0 + bx1)) + ny * (ax[3] - 0.5 * (by0 + by1));
        const __half d16 = __double2half(d);
        const double hw = ext + fabs(d - (double)__half2float(d16)) + VRS_FOOT_MARGIN;
        if (isfinite(hw) && q >= 0.0) {
            n = __halves2half2(hx, hy);
            dh = __halves2half2(d16, __float2half_ru(__double2float_ru(hw)));
        }
    }
    p.foot[2] = *reinterpret_cast<const uint32_t*>(&n);
    p.foot[3] = *reinterpret_cast<const uint32_t*>(&dh);
}

__device__ __forceinline__ void set_rect(const ViewParams& v, int T, double xmin, double xmax, double ymin,
                                         double ymax, Proj& p) {
    const double W = v.W, H = v.H;
    p.bbox[0] = (float)fmax(xmin, -2.0); p.bbox[1] = (float)fmin(xmax, W + 2.0);
    p.bbox[2] = (float)fmax(ymin, -2.0); p.bbox[3] = (float)fmin(ymax, H + 2.0);
    if (xmax < 0.0 || ymax < 0.0 || xmin > W || ymin > H) return;
    const double it = (T == 32) ? 0.03125 : 0.0625;  // 1/T, exact (T is 16 or 32)
    p.rect[0] = max(0, (int)floor(fmax(xmin, 0.0) * it));
    p.rect[1] = max(0, (int)floor(fmax(ymin, 0.0) * it));
    p.rect[2] = min(v.tw - 1, (int)floor(fmin(xmax, W) * it));
    p.rect[3] = min(v.th - 1, (int)floor(fmin(ymax, H) * it));
}

// Sigma_c = W Sigma W^T (T = W*Sigma, then T*W^T, each entry a dot3)
__device__ __forceinline__ void conj3(const ViewParams& v, float4 a, float4 b, float Sc[3][3]) {
    const float S[3][3] = {{a.x, a.y, a.z}, {a.y, a.w, b.x}, {a.z, b.x, b.y}};
    float Tm[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) Tm[i][j] = dot3(v.R[3 * i], v.R[3 * i + 1], v.R[3 * i + 2], S[0][j], S[1][j], S[2][j]);
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = i; j < 3; j++) Sc[i][j] = dot3(Tm[i][0], Tm[i][1], Tm[i][2], v.R[3 * j], v.R[3 * j + 1], v.R[3 * j + 2]);
    Sc[1][0] = Sc[0][1]; Sc[2][0] = Sc[0][2]; Sc[2][1] = Sc[1][2];
}

// EWA baseline (Eq.3; 3DGS computeCov2D with its 1.3 tan(fov/2)
// clamp, SURVEY "EWA mode", config C5): pixel-space conic from the local-affine
// Jacobian at the clamped mean, + 0.3 px^2, screen-space footprint.
__device__ void project_splat_ewa(const ViewParams& v, float4 m4, float4 c0, float4 c1, float4 i0, float4 i1,
                                  int T, float near_plane, Proj& p) {
    p.valid = 0;
    p.rect[0] = 0; p.rect[1] = 0; p.rect[2] = -1; p.rect[3] = -1;
    p.qcut = m4.w;
    p.sigma = c1.z;
    const float vx = m4.x - v.o[0], vy = m4.y - v.o[1], vz = m4.z - v.o[2];
    p.muc[0] = dot3(v.R[0], v.R[1], v.R[2], vx, vy, vz);
    p.muc[1] = dot3(v.R[3], v.R[4], v.R[5], vx, vy, vz);
    p.muc[2] = dot3(v.R[6], v.R[7], v.R[8], vx, vy, vz);
    if (!(p.muc[2] > near_plane) || p.qcut < 0.0f) return;
    float Sc[3][3];
    conj3(v, c0, c1, Sc);
    const float z = p.muc[2];
    const float limx = 1.3f * ((0.5f * (float)v.W) / v.fx), limy = 1.3f * ((0.5f * (float)v.H) / v.fy);
    const float txtz = p.muc[0] / z, tytz = p.muc[1] / z;
    const float tx = fminf(limx, fmaxf(-limx, txtz)) * z;
    const float ty = fminf(limy, fmaxf(-limy, tytz)) * z;
    const float zz = z * z;
    const float J00 = v.fx / z, J02 = -(v.fx * tx) / zz, J11 = v.fy / z, J12 = -(v.fy * ty) / zz;
    const float a0 = fmaf(J00, Sc[0][0], J02 * Sc[0][2]), a1 = fmaf(J00, Sc[0][1], J02 * Sc[1][2]),
                a2 = fmaf(J00, Sc[0][2], J02 * Sc[2][2]);
    const float b1 = fmaf(J11, Sc[1][1], J12 * Sc[1][2]), b2 = fmaf(J11, Sc[1][2], J12 * Sc[2][2]);
    float c00 = fmaf(a0, J00, a2 * J02), c01 = fmaf(a1, J11, a2 * J12), c11 = fmaf(b1, J11, b2 * J12);
    c00 = c00 + 0.3f;
    c11 = c11 + 0.3f;
    p.S2[0] = c00; p.S2[1] = c01; p.S2[2] = c11;
    const float det = fmaf(c00, c11, -(c01 * c01));
    if (!(det > 0.0f)) return;
    const float idet = 1.0f / det;
    p.Cp[0] = c11 * idet; p.Cp[1] = -c01 * idet; p.Cp[2] = c00 * idet;
    p.m2[0] = fmaf(v.fx, p.muc[0] / z, v.cx);
    p.m2[1] = fmaf(v.fy, p.muc[1] / z, v.cy);
    float Ai[3][3];
    conj3(v, i0, i1, Ai);
    p.A[0] = Ai[0][0]; p.A[1] = 2.0f * Ai[0][1]; p.A[2] = Ai[1][1];
    p.A[3] = 2.0f * Ai[0][2]; p.A[4] = 2.0f * Ai[1][2]; p.A[5] = Ai[2][2];
#pragma unroll
    for (int i = 0; i < 3; i++) p.bv[i] = dot3(Ai[i][0], Ai[i][1], Ai[i][2], p.muc[0], p.muc[1], p.muc[2]);
    p.valid = 1;
    const double rx = sqrt((double)p.qcut * c00), ry = sqrt((double)p.qcut * c11);
    set_rect(v, T, p.m2[0] - rx - 1.0, p.m2[0] + rx + 1.0, p.m2[1] - ry - 1.0, p.m2[1] + ry + 1.0, p);
    pack_footprint(p, false);
}

// O1-O6 (DESIGN "Numerics contract"): view transform and near cull,
// optimal-plane frame, projected covariance with pixel-mapped dilation,
// conic, depth coefficients, cone-vs-frustum cull and conic footprint.
__device__ void project_splat(const ViewParams& v, float4 m4, float4 c0, float4 c1, float4 i0, float4 i1, int T,
                              float near_plane, Proj& p) {
    p.valid = 0;
    p.rect[0] = 0; p.rect[1] = 0; p.rect[2] = -1; p.rect[3] = -1;
    p.qcut = m4.w;
    p.sigma = c1.z;
    const float vx = m4.x - v.o[0], vy = m4.y - v.o[1], vz = m4.z - v.o[2];
    p.muc[0] = dot3(v.R[0], v.R[1], v.R[2], vx, vy, vz);
    p.muc[1] = dot3(v.R[3], v.R[4], v.R[5], vx, vy, vz);
    p.muc[2] = dot3(v.R[6], v.R[7], v.R[8], vx, vy, vz);
    if (!(p.muc[2] > near_plane) || p.qcut < 0.0f) return;
    // optimal plane frame
    const float r2 = dot3(p.muc[0], p.muc[1], p.muc[2], p.muc[0], p.muc[1], p.muc[2]);
    const float r = sqrtf(r2);
    const float inv_r = 1.0f / r;
    p.u[0] = p.muc[0] * inv_r; p.u[1] = p.muc[1] * inv_r; p.u[2] = p.muc[2] * inv_r;
    const float h = sqrtf(fmaf(p.u[2], p.u[2], p.u[0] * p.u[0]));
    const float ih = 1.0f / h;
    p.e1[0] = p.u[2] * ih; p.e1[1] = 0.0f; p.e1[2] = -(p.u[0] * ih);
    p.e2[0] = p.u[1] * p.e1[2];
    p.e2[1] = fmaf(p.u[2], p.e1[0], -(p.u[0] * p.e1[2]));
    p.e2[2] = -(p.u[1] * p.e1[0]);
    // Sigma_c = W Sigma_w W^T: T = W*Sigma (row i of W dot column j), then T*W^T
    const float S[3][3] = {{c0.x, c0.y, c0.z}, {c0.y, c0.w, c1.x}, {c0.z, c1.x, c1.y}};
    float Tm[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) Tm[i][j] = dot3(v.R[3 * i], v.R[3 * i + 1], v.R[3 * i + 2], S[0][j], S[1][j], S[2][j]);
    float Sc[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = i; j < 3; j++) Sc[i][j] = dot3(Tm[i][0], Tm[i][1], Tm[i][2], v.R[3 * j], v.R[3 * j + 1], v.R[3 * j + 2]);
    Sc[1][0] = Sc[0][1]; Sc[2][0] = Sc[0][2]; Sc[2][1] = Sc[1][2];
    float P1[3], P2[3];
#pragma unroll
    for (int i = 0; i < 3; i++) {
        P1[i] = dot3(Sc[i][0], Sc[i][1], Sc[i][2], p.e1[0], p.e1[1], p.e1[2]);
        P2[i] = dot3(Sc[i][0], Sc[i][1], Sc[i][2], p.e2[0], p.e2[1], p.e2[2]);
    }
    const float ir2 = inv_r * inv_r;
    float s00 = dot3(p.e1[0], p.e1[1], p.e1[2], P1[0], P1[1], P1[2]) * ir2;
    float s01 = dot3(p.e1[0], p.e1[1], p.e1[2], P2[0], P2[1], P2[2]) * ir2;
    float s11 = dot3(p.e2[0], p.e2[1], p.e2[2], P2[0], P2[1], P2[2]) * ir2;
    // pixel-mapped dilation (+0.3 px^2 at the mean's image position)
    const float jx = p.u[2] / v.fx, jy = p.u[2] / v.fy;
    const float J00 = p.e1[0] * jx, J01 = p.e1[1] * jy, J10 = p.e2[0] * jx, J11 = p.e2[1] * jy;
    const float d00 = fmaf(J00, J00, J01 * J01), d01 = fmaf(J00, J10, J01 * J11), d11 = fmaf(J10, J10, J11 * J11);
    s00 = fmaf(0.3f, d00, s00);
    s01 = fmaf(0.3f, d01, s01);
    s11 = fmaf(0.3f, d11, s11);
    p.S2[0] = s00; p.S2[1] = s01; p.S2[2] = s11;
    const float det = fmaf(s00, s11, -(s01 * s01));
    if (!(det > 0.0f)) return;
    const float idet = 1.0f / det;
    p.C[0] = s11 * idet; p.C[1] = -s01 * idet; p.C[2] = s00 * idet;
    p.eps = 0.5f / sqrtf(fmaf(p.qcut, s00 + s11, 1.0f));
    // depth coefficients: A = W Sigma_w^-1 W^T (same product order), b = A mu_c
    const float Si[3][3] = {{i0.x, i0.y, i0.z}, {i0.y, i0.w, i1.x}, {i0.z, i1.x, i1.y}};
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) Tm[i][j] = dot3(v.R[3 * i], v.R[3 * i + 1], v.R[3 * i + 2], Si[0][j], Si[1][j], Si[2][j]);
    float Ai[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = i; j < 3; j++) Ai[i][j] = dot3(Tm[i][0], Tm[i][1], Tm[i][2], v.R[3 * j], v.R[3 * j + 1], v.R[3 * j + 2]);
    Ai[1][0] = Ai[0][1]; Ai[2][0] = Ai[0][2]; Ai[2][1] = Ai[1][2];
    p.A[0] = Ai[0][0]; p.A[1] = 2.0f * Ai[0][1]; p.A[2] = Ai[1][1];
    p.A[3] = 2.0f * Ai[0][2]; p.A[4] = 2.0f * Ai[1][2]; p.A[5] = Ai[2][2];
#pragma unroll
    for (int i = 0; i < 3; i++) p.bv[i] = dot3(Ai[i][0], Ai[i][1], Ai[i][2], p.muc[0], p.muc[1], p.muc[2]);
    // O6(a) cone vs frustum side planes (double, conservative margin)
    const double S00 = s00, S01 = s01, S11 = s11;
    const double lmax = 0.5 * (S00 + S11) + sqrt(0.25 * (S00 - S11) * (S00 - S11) + S01 * S01);
    const double t2 = (double)p.qcut * lmax;
    const double sinb = sqrt(t2 / (1.0 + t2));
    const double ud0 = p.u[0], ud1 = p.u[1], ud2 = p.u[2];
    {   // unit normals precomputed per view in double (the oracle divides by |n| here; a
        // rounding apart, which the 1e-4 margin covers: the test only has to be conservative)
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const double nu = v.dplane[k][0] * ud0 + v.dplane[k][1] * ud1 + v.dplane[k][2] * ud2;
            if (nu < -(sinb + 1e-4)) return;
        }
    }
    p.valid = 1;
    // O6(b,c) conic bounding box on the image plane (double), whole-screen fallback
    const double W = v.W, H = v.H;
    if (ud2 > sinb + 1e-3) {
        const double e1d[3] = {p.e1[0], p.e1[1], p.e1[2]}, e2d[3] = {p.e2[0], p.e2[1], p.e2[2]};
        const double ud[3] = {ud0, ud1, ud2};
        double G[3][3];
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) {
                double mf = (double)p.C[0] * e1d[i] * e1d[j] + (double)p.C[1] * (e1d[i] * e2d[j] + e2d[i] * e1d[j]) +
                            (double)p.C[2] * e2d[i] * e2d[j];
                G[i][j] = mf - (double)p.qcut * ud[i] * ud[j];
            }
        const double Ki[3][3] = {{v.kinv[0], 0.0, v.kinv[2]}, {0.0, v.kinv[1], v.kinv[3]}, {0.0, 0.0, 1.0}};
        double Tq[3][3], Q[3][3];
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < 3; k++) acc += G[i][k] * Ki[k][j];
                Tq[i][j] = acc;
            }
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k < 3; k++) acc += Ki[k][i] * Tq[k][j];
                Q[i][j] = acc;
            }
        const double a00 = Q[1][1] * Q[2][2] - Q[1][2] * Q[1][2];
        const double a11 = Q[0][0] * Q[2][2] - Q[0][2] * Q[0][2];
        const double a22 = Q[0][0] * Q[1][1] - Q[0][1] * Q[0][1];
        const double a02 = Q[0][1] * Q[1][2] - Q[0][2] * Q[1][1];
        const double a12 = Q[0][1] * Q[0][2] - Q[0][0] * Q[1][2];
        const double dx = a02 * a02 - a00 * a22, dy = a12 * a12 - a11 * a22;
        if (a22 != 0.0 && dx >= 0.0 && dy >= 0.0 && isfinite(dx) && isfinite(dy)) {
            const double sx = sqrt(dx), sy = sqrt(dy), ia = 1.0 / a22;
            const double xa = (a02 - sx) * ia, xb = (a02 + sx) * ia;
            const double ya = (a12 - sy) * ia, yb = (a12 + sy) * ia;
            set_rect(v, T, fmin(xa, xb) - 1.0, fmax(xa, xb) + 1.0, fmin(ya, yb) - 1.0, fmax(ya, yb) + 1.0, p);
            // separating axis for the blend's per-warp footprint skip: the minor axis
            // of the ellipse (M positive definite), r^2 = -det Q / det M
            const double detQ = Q[0][0] * a00 + Q[0][1] * (Q[0][2] * Q[1][2] - Q[0][1] * Q[2][2]) + Q[0][2] * a02;
            const double r2 = -detQ * ia;
            if (a22 > 0.0 && Q[0][0] > 0.0 && r2 >= 0.0 && isfinite(r2)) {
                const double hm = 0.5 * (Q[0][0] + Q[1][1]), dm = 0.5 * (Q[0][0] - Q[1][1]);
                const double lmax = hm + sqrt(dm * dm + Q[0][1] * Q[0][1]);
                // eigenvector of lmax: the longer of (Q01, lmax - Q00) and (lmax - Q11, Q01)
                double nx = Q[0][1], ny = lmax - Q[0][0];
                const double mx = lmax - Q[1][1], my = Q[0][1];
                if (mx * mx + my * my > nx * nx + ny * ny) { nx = mx; ny = my; }
                const double nn = sqrt(nx * nx + ny * ny);
                if (nn > 0.0) {
                    pack_footprint(p, true, nx / nn, ny / nn, a02 * ia, a12 * ia, r2, Q[0][0], Q[0][1], Q[1][1], a22);
                    return;
                }
            }
            pack_footprint(p, false);
            return;
        }
    }
    // whole-screen fallback
    set_rect(v, T, -2.0, W + 2.0, -2.0, H + 2.0, p);
    pack_footprint(p, false);
}

// Splat fields needed by the tile test and the key.
struct TileSplat {
    float ux, uy, uz, e1x, e1z, e2x, e2y, e2z, C0, C1, C2, qcut, eps;
    float A[6], bx, by, bz;
};

// Eq.4 on one polygon edge p -> p + d with t clamped to [0,1];
// keeps the running minimum (strictly smaller q wins: earlier edge on ties).
__device__ __forceinline__ void eq4_edge(const TileSplat& s, float ppx, float ppy, float qx, float qy, float& qmin,
                                         float& hx, float& hy) {
    const float ddx = qx - ppx, ddy = qy - ppy;
    const float cdx = fmaf(s.C0, ddx, s.C1 * ddy), cdy = fmaf(s.C1, ddx, s.C2 * ddy);
    const float den = fmaf(ddx, cdx, ddy * cdy);
    const float nmr = -fmaf(ppx, cdx, ppy * cdy);
    float t;
    if (nmr <= 0.0f || !(den > 0.0f)) t = 0.0f;
    else if (nmr >= den) t = 1.0f;
    else t = nmr / den;
    const float X = fmaf(t, ddx, ppx), Y = fmaf(t, ddy, ppy);
    const float cX = fmaf(s.C0, X, s.C1 * Y), cY = fmaf(s.C1, X, s.C2 * Y);
    const float q = fmaf(X, cX, Y * cY);
    if (q < qmin) { qmin = q; hx = X; hy = Y; }
}

// Minimum of X^T C X over a quad (vertices relative to the mean): 0 if the
// mean is inside, else Eq.4 on the four edges.
__device__ __forceinline__ void quad_min(const TileSplat& s, const float yx[4], const float yy[4], float& qmin,
                                         float& hx, float& hy) {
    int npos = 0, nneg = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int k1 = (k + 1) & 3;
        const float ddx = yx[k1] - yx[k], ddy = yy[k1] - yy[k];
        const float cr = fmaf(ddy, yx[k], -(ddx * yy[k]));
        npos += (cr >= 0.0f) ? 1 : 0;
        nneg += (cr <= 0.0f) ? 1 : 0;
    }
    if (npos == 4 || nneg == 4) {
        qmin = 0.0f;
    } else {
        qmin = __int_as_float(0x7f800000);
#pragma unroll
        for (int k = 0; k < 4; k++) eq4_edge(s, yx[k], yy[k], yx[(k + 1) & 3], yy[(k + 1) & 3], qmin, hx, hy);
    }
}

// EWA baseline O7: StopThePop's screen-space tile test: the tile
// rectangle relative to the projected mean, Eq.4 in pixel units (C = pixel
// conic, stored in C0..C2; mean in ux, uy); key ray through x_hat.
__device__ bool tile_test_ewa(const TileSplat& s, const ViewParams& v, int x0, int y0, int x1, int y1, float& dhx,
                              float& dhy, float& dhz) {
    const float ax = (float)x0 - s.ux, bx = (float)x1 - s.ux, ay = (float)y0 - s.uy, by = (float)y1 - s.uy;
    const float yx[4] = {ax, bx, bx, ax}, yy[4] = {ay, ay, by, by};
    float hx = 0.0f, hy = 0.0f, qmin;
    quad_min(s, yx, yy, qmin, hx, hy);
    dhx = ((s.ux + hx) - v.cx) / v.fx;
    dhy = ((s.uy + hy) - v.cy) / v.fy;
    dhz = 1.0f;
    return qmin <= s.qcut * kO7Margin;
}

// O7: Eq.4 on the optimal-plane polygon of the tile, corner
// rays clipped at s >= eps (DESIGN R8); returns keep and d_hat.
// Fast path: all four corners in front (the common case) -> unrolled quad.
// ax, bx, ay, by: the tile's corner rays ((float)x0 - cx) / fx etc. (per-view tables, k_cull)
__device__ bool tile_test(const TileSplat& s, float ax, float bx, float ay, float by, float& dhx, float& dhy,
                          float& dhz) {
    float dx[4] = {ax, bx, bx, ax}, dy[4] = {ay, ay, by, by}, sv[4];
    int nin = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        sv[k] = fmaf(s.ux, dx[k], fmaf(s.uy, dy[k], s.uz));
        nin += (sv[k] >= s.eps) ? 1 : 0;
    }
    if (nin == 0) return false;
    float hx = 0.0f, hy = 0.0f, qmin;
    if (nin == 4) {
        float yx[4], yy[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const float is = 1.0f / dot3(s.ux, s.uy, s.uz, dx[k], dy[k], 1.0f);
            yx[k] = dot3(s.e1x, 0.0f, s.e1z, dx[k], dy[k], 1.0f) * is;
            yy[k] = dot3(s.e2x, s.e2y, s.e2z, dx[k], dy[k], 1.0f) * is;
        }
        quad_min(s, yx, yy, qmin, hx, hy);
    } else {
        // partially behind the clip level: Sutherland-Hodgman against s >= eps
        float px[5], py[5];
        int n = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int k1 = (k + 1) & 3;
            const bool ia = sv[k] >= s.eps, ib = sv[k1] >= s.eps;
            if (ia) { px[n] = dx[k]; py[n] = dy[k]; n++; }
            if (ia != ib) {
                const int a = ia ? k : k1, b = ia ? k1 : k;
                const float t = (sv[a] - s.eps) / (sv[a] - sv[b]);
                px[n] = fmaf(t, dx[b] - dx[a], dx[a]);
                py[n] = fmaf(t, dy[b] - dy[a], dy[a]);
                n++;
            }
        }
        float yx[5], yy[5];
        for (int k = 0; k < n; k++) {
            const float is = 1.0f / dot3(s.ux, s.uy, s.uz, px[k], py[k], 1.0f);
            yx[k] = dot3(s.e1x, 0.0f, s.e1z, px[k], py[k], 1.0f) * is;
            yy[k] = dot3(s.e2x, s.e2y, s.e2z, px[k], py[k], 1.0f) * is;
        }
        int npos = 0, nneg = 0;
        for (int k = 0; k < n; k++) {
            const int k1 = (k + 1 == n) ? 0 : k + 1;
            const float ddx = yx[k1] - yx[k], ddy = yy[k1] - yy[k];
            const float cr = fmaf(ddy, yx[k], -(ddx * yy[k]));
            npos += (cr >= 0.0f) ? 1 : 0;
            nneg += (cr <= 0.0f) ? 1 : 0;
        }
        if (npos == n || nneg == n) {
            qmin = 0.0f;
        } else {
            qmin = __int_as_float(0x7f800000);
            for (int k = 0; k < n; k++) {
                const int k1 = (k + 1 == n) ? 0 : k + 1;
                eq4_edge(s, yx[k], yy[k], yx[k1], yy[k1], qmin, hx, hy);
            }
        }
    }
    dhx = fmaf(hy, s.e2x, fmaf(hx, s.e1x, s.ux));
    dhy = fmaf(hy, s.e2y, fmaf(hx, 0.0f, s.uy));
    dhz = fmaf(hy, s.e2z, fmaf(hx, s.e1z, s.uz));
    return qmin <= s.qcut * kO7Margin;
}

// O8: StopThePop per-tile depth on the unit ray through x_hat.
__device__ __forceinline__ float tile_depth(const TileSplat& s, float x, float y, float z, float near_plane) {
    const float dAd = quad3(s.A[0], s.A[1], s.A[2], s.A[3], s.A[4], s.A[5], x, y, z);
    const float db = fmaf(s.bx, x, fmaf(s.by, y, s.bz * z));
    const float nd = sqrtf(dot3(x, y, z, x, y, z));
    const float t = nd * (db / dAd);
    return (t > near_plane) ? t : near_plane;
}

__device__ __forceinline__ uint32_t sat_count(const uint32_t* sat, int S, int x0, int y0, int x1, int y1) {
    // read-only for the whole frame (k_setup wrote it before): through the
    // non-coherent path, so the per-view table stays in L1
    return __ldg(sat + (y1 + 1) * S + x1 + 1) - __ldg(sat + y0 * S + x1 + 1) - __ldg(sat + (y1 + 1) * S + x0) +
           __ldg(sat + y0 * S + x0);
}

__device__ __forceinline__ void proj_to_tilesplat(const Proj& p, TileSplat& s) {
    s.ux = p.u[0]; s.uy = p.u[1]; s.uz = p.u[2];
    s.e1x = p.e1[0]; s.e1z = p.e1[2]; s.e2x = p.e2[0]; s.e2y = p.e2[1]; s.e2z = p.e2[2];
    s.C0 = p.C[0]; s.C1 = p.C[1]; s.C2 = p.C[2]; s.qcut = p.qcut; s.eps = p.eps;
#pragma unroll
    for (int i = 0; i < 6; i++) s.A[i] = p.A[i];
    s.bx = p.bv[0]; s.by = p.bv[1]; s.bz = p.bv[2];
}

// View-dependent colour: real SH through degree 3 (3DGS basis), +0.5, >= 0.
// The coefficients come either from memory (src) or, already loaded, from q.
__device__ __forceinline__ void sh_color_q(const float4 q4[12], int chunks, int ncoef, float dx, float dy, float dz,
                                           float out[3]);
__device__ void sh_color(const SceneDev& sc, int64_t g, int64_t N, int ncoef, float dx, float dy, float dz,
                         float out[3]) {
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    float basis[16];
    basis[0] = C0;
    if (ncoef > 1) {
        basis[1] = -C1 * dy; basis[2] = C1 * dz; basis[3] = -C1 * dx;
    }
    if (ncoef > 4) {
        const float xx = dx * dx, yy = dy * dy, zz = dz * dz, xy = dx * dy, yz = dy * dz, xz = dx * dz;
        basis[4] = 1.0925484305920792f * xy;
        basis[5] = -1.0925484305920792f * yz;
        basis[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
        basis[7] = -1.0925484305920792f * xz;
        basis[8] = 0.5462742152960396f * (xx - yy);
        if (ncoef > 9) {
            basis[9] = -0.5900435899266435f * dy * (3.0f * xx - yy);
            basis[10] = 2.890611442640554f * xy * dz;
            basis[11] = -0.4570457994644658f * dy * (4.0f * zz - xx - yy);
            basis[12] = 0.3731763325901154f * dz * (2.0f * zz - 3.0f * xx - 3.0f * yy);
            basis[13] = -0.4570457994644658f * dx * (4.0f * zz - xx - yy);
            basis[14] = 1.445305721320277f * dz * (xx - yy);
            basis[15] = -0.5900435899266435f * dx * (xx - 3.0f * yy);
        }
    }
    // accumulate chunk by chunk (4 floats of the coefficient-major RGB array at
    // a time; all indices compile-time: no local memory, few live registers)
    const float4* src = sc.sh + (size_t)g * sc.sh_chunks;
    float acc[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int c4 = 0; c4 < 12; c4++) {
        if (c4 < sc.sh_chunks) {
            const float4 q = __ldg(src + c4);
            const float qv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int f = 4 * c4 + k;  // coefficient f / 3, channel f % 3
                if (f / 3 < ncoef) acc[f % 3] = fmaf(basis[f / 3], qv[k], acc[f % 3]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < 3; c++) {
        const float r = acc[c] + 0.5f;
        out[c] = r > 0.0f ? r : 0.0f;
    }
}

__device__ __forceinline__ void load_gauss(const SceneDev& sc, int64_t g, int64_t N, float4& m4, float4& c0,
                                           float4& c1, float4& i0, float4& i1) {
    m4 = __ldg(&sc.mu[g]);
    (void)N;
    c0 = __ldg(&sc.geo[4 * g + 0]);
    c1 = __ldg(&sc.geo[4 * g + 1]);
    i0 = __ldg(&sc.geo[4 * g + 2]);
    i1 = __ldg(&sc.geo[4 * g + 3]);
}

// Step 1a: cheap conservative cull over all Gaussians and views.  The
// footprint of a Gaussian lies in the cone of half-angle beta' around u with
// tan^2 beta' = q_cut (s_max^2 / r^2 + 0.3 / f_min^2) >= q_cut lambda_max(Sigma_2)
// (lambda_max(E^T Sigma_c E) <= s_max^2, dilation <= 0.3/f^2), so a view whose
// frustum misses that (inflated) cone is also culled by the exact O6(a) test:
// culling here never changes results, it only compacts the work of step 1b.
__global__ void __launch_bounds__(256) k_cull(SceneDev sc, FrameParams fp, FrameBufs fb) {
    if (blockIdx.x == 0) {
        // per-view tile-corner ray tables for the tile test: xr[k] = ((float)min(kT, W) - cx) / fx,
        // yr[k] likewise (the O7 corner rays, the same operations as the oracle's)
        for (int vi = 0; vi < fp.n_views; vi++) {
            const ViewParams& v = fp.v[vi];
            for (int k = threadIdx.x; k <= v.tw; k += blockDim.x)
                v.xr[k] = ((float)min(k * fp.T, v.W) - v.cx) / v.fx;
            for (int k = threadIdx.x; k <= v.th; k += blockDim.x)
                v.yr[k] = ((float)min(k * fp.T, v.H) - v.cy) / v.fy;
        }
    }
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t N = fp.N;
    const bool in = g < N;
    float4 m4 = make_float4(0.f, 0.f, 0.f, -1.0f);
    float smax = 0.0f;
    if (in) {
        m4 = __ldg(&sc.mu[g]);
        smax = __ldg(&sc.smax[g]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t s_wcnt[32];
    __shared__ uint32_t s_base;
    bool any = false;
    for (int vi = 0; vi < fp.n_views; vi++) {
        const ViewParams& v = fp.v[vi];
        bool pass = false;
        if (in && m4.w >= 0.0f) {
            const float vx = m4.x - v.o[0], vy = m4.y - v.o[1], vz = m4.z - v.o[2];
            const float mx = dot3(v.R[0], v.R[1], v.R[2], vx, vy, vz);
            const float my = dot3(v.R[3], v.R[4], v.R[5], vx, vy, vz);
            const float mz = dot3(v.R[6], v.R[7], v.R[8], vx, vy, vz);
            if (mz > fp.near_plane && fp.ewa) {
                pass = true;  // EWA baseline: screen-space footprint decides (no cone)
            } else if (mz > fp.near_plane) {
                const float r2 = dot3(mx, my, mz, mx, my, mz);
                const float tan2 = m4.w * (smax * smax / r2 + v.dil);
                const float sinb = sqrtf(tan2 / (1.0f + tan2)) * 1.01f + 2e-3f;
                const float ir = rsqrtf(r2);
                const float ux = mx * ir, uy = my * ir, uz = mz * ir;
                pass = true;
#pragma unroll
                for (int k = 0; k < 4; k++)
                    pass = pass && (v.plane[k][0] * ux + v.plane[k][1] * uy + v.plane[k][2] * uz >= -sinb);
            }
        }
        // block-aggregated append of (view, g) to the work list: one global
        // atomic per block and view (a single hot counter serialises otherwise)
        const unsigned m = __ballot_sync(0xffffffffu, pass);
        if (lane == 0) s_wcnt[warp] = (uint32_t)__popc(m);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
                const uint32_t c = s_wcnt[w];
                s_wcnt[w] = tot;
                tot += c;
            }
            s_base = tot ? atomicAdd(fb.cand_count, tot) : 0u;
        }
        __syncthreads();
        if (pass)
            fb.cand[s_base + s_wcnt[warp] + __popc(m & ((1u << lane) - 1u))] = (uint32_t)((int64_t)vi * N + g);
        any = any || pass;
        __syncthreads();
    }
    const int nany = __syncthreads_count(any);  // Gaussians read by step 1b (statistic, one atomic per block)
    if (threadIdx.x == 0 && nany) atomicAdd(fb.frustum_count, (uint32_t)nany);
}

// Step 1b: exact per-(view, Gaussian) preprocess of the compacted candidates:
// projection, footprint, candidate tile count and splat record (the SH colour
// runs in k_color on the side stream).
// Step 2 (fused): each warp takes 32 consecutive candidates per iteration,
// scans their tile counts with shuffles and writes the expansion (splat
// view*N+g | rect-local tile index << 32) itself, every output slot finding
// its owner lane by a binary search over the warp's prefix sums -- no block
// barrier, so warps do not wait for each other.  The slices of the test list
// and of the visible-splat list are reserved with one 64-bit atomic per warp
// iteration (reserving for several iterations at once measured no faster).
// The list order is arbitrary: the binned sort makes the final pair order
// independent of it.
// Input staging: every lane copies its next candidate's 80 input bytes (mu
// and the 64-B geometry record) into the warp's shared-memory double buffer
// with cp.async while it projects the current one; the candidate index itself
// is read two iterations ahead.
#ifndef VRS_PP_MINB
#define VRS_PP_MINB 2
#endif
#ifndef VRS_PP_GRID
#define VRS_PP_GRID 2
#endif
#ifndef VRS_TT_GRID
#define VRS_TT_GRID 8
#endif
#ifndef VRS_TT_MINB
#define VRS_TT_MINB 4
#endif
namespace {
constexpr int kPPWarps = 8;
struct PPStage {
    float4 in[2][5][32];  // [buffer][mu, geo0..geo3][lane]: conflict-free LDS.128 / cp.async
};
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
}  // namespace

__global__ void __launch_bounds__(256, VRS_PP_MINB) k_preprocess(SceneDev sc, FrameParams fp, FrameBufs fb, int64_t test_cap) {
    const int lane = threadIdx.x & 31;
    const int64_t N = fp.N;
    const uint32_t nc = *fb.cand_count;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const unsigned lt = (1u << lane) - 1u;
    auto view_of = [&](uint32_t s) {  // view = number of view blocks of N below s (no 64-bit division)
        int vi = 0;
        while (vi + 1 < fp.n_views && (int64_t)s >= (int64_t)(vi + 1) * N) vi++;
        return vi;
    };
    __shared__ PPStage s_pp[kPPWarps];
    PPStage& stg = s_pp[threadIdx.x >> 5];
    // issue the copies of candidate s into buffer b (nothing if out of range); always one group
    auto stage_in = [&](uint32_t ci, uint32_t s, int b) {
        if (ci < nc) {
            const int64_t g = (int64_t)s - (int64_t)view_of(s) * N;
            cp_async16(&stg.in[b][0][lane], sc.mu + g);
#pragma unroll
            for (int k = 0; k < 4; k++) cp_async16(&stg.in[b][1 + k][lane], sc.geo + 4 * g + k);
        }
        cp_async_commit();
    };
    const uint32_t first = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32u + (uint32_t)lane;
    uint32_t s_cur = first < nc ? __ldg(fb.cand + first) : 0u;
    uint32_t s_nxt = first + nw * 32u < nc ? __ldg(fb.cand + first + nw * 32u) : 0u;
    stage_in(first, s_cur, 0);
    int buf = 0;
    for (uint32_t b0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32u; b0 < nc; b0 += nw * 32u) {
        const uint32_t i = b0 + lane;
        const uint32_t sidx_in = s_cur;
        {
            const uint32_t inext = i + nw * 32u, inn = inext + nw * 32u;
            stage_in(inext, s_nxt, buf ^ 1);
            s_cur = s_nxt;
            s_nxt = inn < nc ? __ldg(fb.cand + inn) : 0u;
            cp_async_wait1();  // this lane's copies of candidate i have landed
        }
        uint32_t cnt = 0, sidx = 0;
        if (i < nc) {
            sidx = sidx_in;
            const int vi = view_of(sidx);
            const ViewParams& v = fp.v[vi];
            const float4 m4 = stg.in[buf][0][lane];
            const float4 c0 = stg.in[buf][1][lane], c1 = stg.in[buf][2][lane];
            const float4 i0 = stg.in[buf][3][lane], i1 = stg.in[buf][4][lane];
            Proj p;
            if (fp.ewa) project_splat_ewa(v, m4, c0, c1, i0, i1, fp.T, fp.near_plane, p);
            else project_splat(v, m4, c0, c1, i0, i1, fp.T, fp.near_plane, p);
            // number of (Gaussian, tile) candidates = rect area, 0 if the rect holds no
            // visible tile (SAT); the exact Eq.4 tests run load-balanced in k_tiletest
            // (a view without invisible tiles skips the table: every tile counts)
            if (p.valid && p.rect[0] <= p.rect[2] && p.rect[1] <= p.rect[3] &&
                (v.n_inv == 0 || sat_count(v.sat, v.tw + 1, p.rect[0], p.rect[1], p.rect[2], p.rect[3]) > 0))
                cnt = (uint32_t)((p.rect[2] - p.rect[0] + 1) * (p.rect[3] - p.rect[1] + 1));
            if (cnt) {
                float4* rec = fb.rec + (size_t)sidx * kRecF4;
                const uint32_t r01 = (uint32_t)p.rect[0] | ((uint32_t)p.rect[1] << 16);
                const uint32_t r23 = (uint32_t)p.rect[2] | ((uint32_t)p.rect[3] << 16);
                if (fp.ewa) {
                    rec[0] = make_float4(p.m2[0], p.m2[1], p.qcut, p.Cp[0]);
                    rec[1] = make_float4(p.Cp[1], p.Cp[2], 0.0f, 0.0f);
                    rec[2] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                    p.eps = 0.0f;
                } else {
                    rec[0] = make_float4(p.u[0], p.u[1], p.u[2], p.qcut);
                    rec[1] = make_float4(p.e1[0], p.e1[2], p.e2[0], p.e2[1]);
                    rec[2] = make_float4(p.e2[2], p.C[0], p.C[1], p.C[2]);
                }
                rec[3] = make_float4(p.A[0], p.A[1], p.A[2], p.A[3]);
                rec[4] = make_float4(p.A[4], p.A[5], p.bv[0], p.bv[1]);
                rec[5] = make_float4(p.bv[2], p.sigma, p.eps, __uint_as_float(r01));
                // rec[6] = (global-sort key depth (N3: view-space z or |mu - o|), -, -, rect23)
                float* r6 = reinterpret_cast<float*>(rec + 6);
                r6[0] = (fp.sort_mode == VRS_SORT_Z) ? p.muc[2]
                                                     : sqrtf(dot3(p.muc[0], p.muc[1], p.muc[2], p.muc[0], p.muc[1],
                                                                  p.muc[2]));
                r6[3] = __uint_as_float(r23);
                rec[7] = make_float4(__uint_as_float(p.foot[0]), __uint_as_float(p.foot[1]),
                                     __uint_as_float(p.foot[2]), __uint_as_float(p.foot[3]));
            }
        }
        // warp inclusive scan of the counts; visible splats (cnt > 0) listed alongside
        uint32_t inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
        const unsigned vb = __ballot_sync(0xffffffffu, cnt != 0u);
        // one 64-bit atomic reserves both slices: tests in bits 0-35, visible splats in 36-63
        unsigned long long old = 0;
        if (lane == 0 && (tot | vb))
            old = atomicAdd(fb.tv, ((unsigned long long)__popc(vb) << kTvShift) | (unsigned long long)tot);
        old = __shfl_sync(0xffffffffu, old, 0);
        const uint32_t base = (uint32_t)min(old & kTvMask, 0xffffffffull), vbase = (uint32_t)(old >> kTvShift);
        if (cnt) fb.vis_list[vbase + __popc(vb & lt)] = sidx;
        for (uint32_t o0 = 0; o0 < tot; o0 += 32u) {
            const uint32_t o = o0 + (uint32_t)lane;
            int lo = 0;  // owner: first lane e with inc_e > o
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, inc, lo + step - 1);
                if (v <= o) lo += step;
            }
            const uint32_t e_inc = __shfl_sync(0xffffffffu, inc, lo);
            const uint32_t e_cnt = __shfl_sync(0xffffffffu, cnt, lo);
            const uint32_t e_sidx = __shfl_sync(0xffffffffu, sidx, lo);
            const int64_t pos = (int64_t)base + o;
            if (o < tot && pos < test_cap)
                fb.sidk[pos] = (unsigned long long)e_sidx | ((unsigned long long)(o - (e_inc - e_cnt)) << 32);
        }
        buf ^= 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}


// Step 3 (fused): one thread per (Gaussian, candidate tile): Eq.4 test (O7)
// and key (O8), then stream compaction of the kept candidates (blocks take
// 512-candidate tiles from a counter and reserve their output with one
// atomic; the emission order is therefore arbitrary, and irrelevant: the
// binned sort orders by (tile, depth, g)).  When tile_cnt is given, every
// written pair also takes its rank inside its tile from a per-tile counter
// (its bucket slot, k_binsort.cu).  Candidates come from the expansion the
// preprocess wrote (sidk: splat | rect-local tile index << 32).
namespace {
constexpr int kTT = 256;           // threads per block
#ifndef VRS_TT_ITEMS
#define VRS_TT_ITEMS 2
#endif
constexpr int kTTItems = VRS_TT_ITEMS;  // candidates per thread (independent: ILP)

constexpr int kTTTile = kTT * kTTItems;
static_assert(kTT / 32 * kTTItems <= 32, "k_tiletest's single-warp scan covers at most 32 warp-slots");
}  // namespace

__device__ __forceinline__ bool test_candidate(const FrameParams& fp, const FrameBufs& fb, unsigned long long sk,
                                               uint64_t& key, uint32_t& gout) {
    const uint32_t sidx = (uint32_t)sk, l = (uint32_t)(sk >> 32);
    int vi = 0;
    while (vi + 1 < fp.n_views && (int64_t)sidx >= (int64_t)(vi + 1) * fp.N) vi++;
    const ViewParams& v = fp.v[vi];
    const float4* rec = fb.rec + (size_t)sidx * kRecF4;
    const float4 r0 = __ldg(rec + 0), r1 = __ldg(rec + 1), r2 = __ldg(rec + 2), r5 = __ldg(rec + 5);
    // rect23 only: k_color writes the colour into rec[6].xyz concurrently (side stream)
    const float r6w = __ldg(reinterpret_cast<const float*>(rec + 6) + 3);
    const uint32_t r01 = __float_as_uint(r5.w), r23 = __float_as_uint(r6w);
    const int tx0 = r01 & 0xffff, ty0 = r01 >> 16, tx1 = r23 & 0xffff;
    const int rw = tx1 - tx0 + 1;
    const int tx = tx0 + (int)(l % (uint32_t)rw), ty = ty0 + (int)(l / (uint32_t)rw);
    if (v.n_inv != 0 && !v.vis[ty * v.tw + tx]) return false;  // (no table read when every tile is visible)
    TileSplat s;
    const int T = fp.T, x0 = tx * T, y0 = ty * T;
    float hx, hy, hz;
    if (fp.ewa) {  // record: (m.x, m.y, q_cut, Cp0) (Cp1, Cp2, -, -)
        s.ux = r0.x; s.uy = r0.y; s.qcut = r0.z; s.C0 = r0.w; s.C1 = r1.x; s.C2 = r1.y;
        if (!tile_test_ewa(s, v, x0, y0, min(x0 + T, v.W), min(y0 + T, v.H), hx, hy, hz)) return false;
    } else {
        s.ux = r0.x; s.uy = r0.y; s.uz = r0.z; s.qcut = r0.w;
        s.e1x = r1.x; s.e1z = r1.y; s.e2x = r1.z; s.e2y = r1.w;
        s.e2z = r2.x; s.C0 = r2.y; s.C1 = r2.z; s.C2 = r2.w;
        s.eps = r5.z;
        if (!tile_test(s, __ldg(v.xr + tx), __ldg(v.xr + tx + 1), __ldg(v.yr + ty), __ldg(v.yr + ty + 1), hx, hy, hz))
            return false;
    }
    const float4 r3 = __ldg(rec + 3), r4 = __ldg(rec + 4);  // only for kept pairs
    s.A[0] = r3.x; s.A[1] = r3.y; s.A[2] = r3.z; s.A[3] = r3.w;
    s.A[4] = r4.x; s.A[5] = r4.y; s.bx = r4.z; s.by = r4.w; s.bz = r5.x;
    // StopThePop per-tile depth at x_hat (O8), or the global-sort baselines' per-Gaussian depth (N3)
    const float td = (fp.sort_mode == VRS_SORT_STOPTHEPOP) ? tile_depth(s, hx, hy, hz, fp.near_plane)
                                                            : __ldg(reinterpret_cast<const float*>(rec + 6));
    const uint64_t tile = (uint64_t)(v.tile_base + ty * v.tw + tx);
    key = (tile << 32) | (uint64_t)__float_as_uint(td);
    gout = (uint32_t)((int64_t)sidx - (int64_t)vi * fp.N);
    return true;
}

// Frame path: every kept pair takes its arrival rank in its tile's counter
// and goes straight into the tile's bucket slot (tile * kTileCap + rank), or,
// past kTileCap, onto the overflow list (k_ovf_bucket places those once the
// tile offsets are known).  No compaction, no block synchronisation.
__global__ void __launch_bounds__(kTT, VRS_TT_MINB) k_tiletest_direct(FrameParams fp, FrameBufs fb, int64_t test_cap,
                                                                      BinScratch bs) {
    const int64_t total = min(fb_tests(fb), test_cap);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < total; t0 += stride * kTTItems) {
        uint64_t key[kTTItems];
        uint32_t gv[kTTItems];
        bool keep[kTTItems];
#pragma unroll
        for (int it = 0; it < kTTItems; it++) {
            const int64_t t = t0 + it * stride;
            keep[it] = false;
            key[it] = 0;
            gv[it] = 0;
            if (t < total) keep[it] = test_candidate(fp, fb, fb.sidk[t], key[it], gv[it]);
        }
#pragma unroll
        for (int it = 0; it < kTTItems; it++) {
            if (!keep[it]) continue;
            const uint32_t tl = (uint32_t)(key[it] >> 32);
            const uint32_t r = atomicAdd(&bs.tile_cnt[tl], 1u);
            if (r < kTileCap) {
                bs.tbucket[(size_t)tl * kTileCap + r] = (key[it] << 32) | gv[it];
            } else {
                const uint32_t o = atomicAdd(bs.ovf_count, 1u);
                if (o < fp.pair_cap) {
                    fb.keys_alt[o] = key[it];
                    fb.vals_alt[o] = gv[it];
                    bs.rank[o] = r;
                }
            }
        }
    }
}

// Parity hook path (vrs_debug_pairs sorted=0): the kept pairs compacted into
// (keys, vals) by one atomic per 512-candidate block tile.
__global__ void __launch_bounds__(kTT, VRS_TT_MINB) k_tiletest(FrameParams fp, FrameBufs fb, int64_t test_cap, uint64_t* keys,
                                                  uint32_t* vals, uint32_t* counter) {
    __shared__ uint32_t s_wc[kTT / 32 * kTTItems];
    __shared__ uint32_t s_tile, s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t total = min(fb_tests(fb), test_cap);
    const int64_t ntiles = (total + kTTTile - 1) / kTTTile;
    while (true) {
        if (tid == 0) s_tile = atomicAdd(counter, 1u);
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= ntiles) break;
        uint64_t key[kTTItems];
        uint32_t gv[kTTItems];
        bool keep[kTTItems];
#pragma unroll
        for (int it = 0; it < kTTItems; it++) {
            const int64_t t = tile * kTTTile + it * kTT + tid;
            keep[it] = false;
            key[it] = 0;
            gv[it] = 0;
            if (t < total) keep[it] = test_candidate(fp, fb, fb.sidk[t], key[it], gv[it]);
        }
        uint32_t wbits[kTTItems];
#pragma unroll
        for (int it = 0; it < kTTItems; it++) {
            wbits[it] = __ballot_sync(0xffffffffu, keep[it]);
            if (lane == 0) s_wc[it * (kTT / 32) + warp] = __popc(wbits[it]);
        }
        __syncthreads();
        if (warp == 0) {
            constexpr int nw = kTT / 32 * kTTItems;  // warp-slots (<= 32, static_assert above)
            const uint32_t c = (lane < nw) ? s_wc[lane] : 0u;
            uint32_t inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const uint32_t agg = __shfl_sync(0xffffffffu, inc, 31);
            if (lane < nw) s_wc[lane] = inc - c;
            if (lane == 0) s_base = agg ? atomicAdd(fb.total, agg) : 0u;
        }
        __syncthreads();
        const uint32_t base = s_base;
#pragma unroll
        for (int it = 0; it < kTTItems; it++) {
            if (keep[it]) {
                const uint32_t pos = base + s_wc[it * (kTT / 32) + warp] + __popc(wbits[it] & lt);
                if (pos < fp.pair_cap) {
                    keys[pos] = key[it];
                    vals[pos] = gv[it];
                }
            }
        }
    }
}

// Exact per-(view, g) pair counts (parity hook / statistics only): the
// pairs of a splat are contiguous in emission order, so its count is the
// number of emitted pairs whose candidate falls in its candidate range;
// computed by a binary search of the splat range in the candidate->pair map.
__global__ void k_counts(FrameParams fp, FrameBufs fb, int64_t test_cap) {
    const int64_t total = min(fb_tests(fb), test_cap);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key;
        uint32_t g;
        const unsigned long long sk = fb.sidk[t];
        if (test_candidate(fp, fb, sk, key, g)) atomicAdd(&fb.counts[(uint32_t)sk], 1u);
    }
}

// Parity hook: the oracle's 48-float semantic splat layout.
__global__ void k_debug_splats(SceneDev sc, FrameParams fp, FrameBufs fb, int vi, float* out) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t N = fp.N;
    if (g >= N) return;
    float4 m4, c0, c1, i0, i1;
    load_gauss(sc, g, N, m4, c0, c1, i0, i1);
    const ViewParams& v = fp.v[vi];
    Proj p;
    for (int i = 0; i < 3; i++) { p.u[i] = p.e1[i] = p.e2[i] = p.S2[i] = p.C[i] = p.bv[i] = 0.0f; }
    for (int i = 0; i < 6; i++) p.A[i] = 0.0f;
    for (int i = 0; i < 4; i++) p.bbox[i] = 0.0f;
    p.eps = 0.0f;
    p.m2[0] = p.m2[1] = p.Cp[0] = p.Cp[1] = p.Cp[2] = 0.0f;
    if (fp.ewa) project_splat_ewa(v, m4, c0, c1, i0, i1, fp.T, fp.near_plane, p);
    else project_splat(v, m4, c0, c1, i0, i1, fp.T, fp.near_plane, p);
    float* o = out + g * 48;
    for (int i = 0; i < 48; i++) o[i] = 0.0f;
    o[0] = (float)p.valid;
    for (int i = 0; i < 3; i++) {
        o[1 + i] = p.muc[i]; o[4 + i] = p.u[i]; o[7 + i] = p.e1[i]; o[10 + i] = p.e2[i];
        o[13 + i] = p.S2[i]; o[16 + i] = p.C[i]; o[31 + i] = p.bv[i];
    }
    o[19] = p.eps;
    o[20] = p.m2[0]; o[21] = p.m2[1]; o[22] = p.Cp[0]; o[23] = p.Cp[1]; o[24] = p.Cp[2];
    for (int i = 0; i < 6; i++) o[25 + i] = p.A[i];
    o[37] = p.sigma; o[38] = p.qcut;
    for (int i = 0; i < 4; i++) { o[39 + i] = (float)p.rect[i]; o[43 + i] = p.bbox[i]; }
    const uint32_t cnt = fb.counts[(size_t)vi * N + g];
    o[47] = (float)cnt;
    if (p.valid) {
        const float dx = m4.x - v.o[0], dy = m4.y - v.o[1], dz = m4.z - v.o[2];
        const float inv = 1.0f / sqrtf(dot3(dx, dy, dz, dx, dy, dz));
        float rgb[3];
        sh_color(sc, g, N, fp.sh_coeffs, dx * inv, dy * inv, dz * inv, rgb);
        o[34] = rgb[0]; o[35] = rgb[1]; o[36] = rgb[2];
    }
}

__device__ __forceinline__ void sh_color_q(const float4 q4[12], int chunks, int ncoef, float dx, float dy, float dz,
                                           float out[3]) {
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    float basis[16];
    basis[0] = C0;
    if (ncoef > 1) {
        basis[1] = -C1 * dy; basis[2] = C1 * dz; basis[3] = -C1 * dx;
    }
    if (ncoef > 4) {
        const float xx = dx * dx, yy = dy * dy, zz = dz * dz, xy = dx * dy, yz = dy * dz, xz = dx * dz;
        basis[4] = 1.0925484305920792f * xy;
        basis[5] = -1.0925484305920792f * yz;
        basis[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
        basis[7] = -1.0925484305920792f * xz;
        basis[8] = 0.5462742152960396f * (xx - yy);
        if (ncoef > 9) {
            basis[9] = -0.5900435899266435f * dy * (3.0f * xx - yy);
            basis[10] = 2.890611442640554f * xy * dz;
            basis[11] = -0.4570457994644658f * dy * (4.0f * zz - xx - yy);
            basis[12] = 0.3731763325901154f * dz * (2.0f * zz - 3.0f * xx - 3.0f * yy);
            basis[13] = -0.4570457994644658f * dx * (4.0f * zz - xx - yy);
            basis[14] = 1.445305721320277f * dz * (xx - yy);
            basis[15] = -0.5900435899266435f * dx * (xx - 3.0f * yy);
        }
    }
    float acc[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int c4 = 0; c4 < 12; c4++) {
        if (c4 < chunks) {
            const float qv[4] = {q4[c4].x, q4[c4].y, q4[c4].z, q4[c4].w};
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int f = 4 * c4 + k;
                if (f / 3 < ncoef) acc[f % 3] = fmaf(basis[f / 3], qv[k], acc[f % 3]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < 3; c++) {
        const float r = acc[c] + 0.5f;
        out[c] = r > 0.0f ? r : 0.0f;
    }
}

// Step 1c: view-dependent SH colour (Eq.2 colour term) of the
// splats with at least one candidate tile, a streaming pass over the list the
// preprocess appended them to (kept out of k_preprocess so its block scan
// does not wait on the 192 B SH fetches).
__global__ void __launch_bounds__(256) k_color(SceneDev sc, FrameParams fp, FrameBufs fb) {
    const int64_t N = fp.N;
    const uint32_t n = fb_visible(fb);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t sidx = fb.vis_list[i];
        int vi = 0;
        while (vi + 1 < fp.n_views && (int64_t)sidx >= (int64_t)(vi + 1) * N) vi++;
        const int64_t g = (int64_t)sidx - (int64_t)vi * N;
        const ViewParams& v = fp.v[vi];
        // all loads first (the mean and every SH chunk are independent)
        const float4 m4 = __ldg(&sc.mu[g]);
        const float4* src = sc.sh + (size_t)g * sc.sh_chunks;
        float4 q[12];
#pragma unroll
        for (int c4 = 0; c4 < 12; c4++) q[c4] = c4 < sc.sh_chunks ? __ldg(src + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float dx = m4.x - v.o[0], dy = m4.y - v.o[1], dz = m4.z - v.o[2];
        const float inv = 1.0f / sqrtf(dot3(dx, dy, dz, dx, dy, dz));
        float rgb[3];
        sh_color_q(q, sc.sh_chunks, fp.sh_coeffs, dx * inv, dy * inv, dz * inv, rgb);
        fb.col[sidx] = make_float4(rgb[0], rgb[1], rgb[2], 0.0f);
    }
}


void launch_preprocess(const SceneDev& sc, const FrameParams& fp, FrameBufs fb, int64_t test_cap, cudaStream_t st) {
    cudaMemsetAsync(fb.tv, 0, 8, st);
    cudaMemsetAsync(fb.cand_count, 0, 4, st);
    cudaMemsetAsync(fb.frustum_count, 0, 4, st);
    if (fp.N == 0) return;
    constexpr int B = 256;
    k_cull<<<(unsigned)((fp.N + B - 1) / B), B, 0, st>>>(sc, fp, fb);
    const int sms = device_sms();
    static_assert(B == 32 * kPPWarps, "one staging buffer per warp");
    k_preprocess<<<sms * VRS_PP_GRID, B, 0, st>>>(sc, fp, fb, test_cap);
}

void launch_color(const SceneDev& sc, const FrameParams& fp, FrameBufs fb, cudaStream_t st) {
    if (fp.N == 0) return;
    k_color<<<device_sms() * 8, 256, 0, st>>>(sc, fp, fb);
}

static int sm_count() {
    return device_sms();
}

void launch_tiletest(const FrameParams& fp, FrameBufs fb, int64_t test_cap, uint64_t* keys, uint32_t* vals,
                     uint32_t* counter, cudaStream_t st) {
    cudaMemsetAsync(fb.total, 0, 4, st);  // pair total: block atomics below
    if ((int64_t)fp.n_views * fp.N == 0) return;
    cudaMemsetAsync(counter, 0, 4, st);
    k_tiletest<<<sm_count() * 8, kTT, 0, st>>>(fp, fb, test_cap, keys, vals, counter);
}

void launch_tiletest_direct(const FrameParams& fp, FrameBufs fb, int64_t test_cap, const BinScratch& bs,
                            cudaStream_t st) {
    cudaMemsetAsync(bs.ovf_count, 0, 4, st);
    if ((int64_t)fp.n_views * fp.N == 0) return;
    k_tiletest_direct<<<sm_count() * VRS_TT_GRID, kTT, 0, st>>>(fp, fb, test_cap, bs);
}

void launch_counts(const FrameParams& fp, FrameBufs fb, int64_t test_cap, cudaStream_t st) {
    const int64_t n = (int64_t)fp.n_views * fp.N;
    if (n == 0) return;
    cudaMemsetAsync(fb.counts, 0, sizeof(uint32_t) * n, st);
    k_counts<<<sm_count() * 8, 256, 0, st>>>(fp, fb, test_cap);
}

void launch_debug_splats(const SceneDev& sc, const FrameParams& fp, FrameBufs fb, int view, float* out,
                         cudaStream_t st) {
    if (fp.N == 0) return;
    k_debug_splats<<<(unsigned)((fp.N + 127) / 128), 128, 0, st>>>(sc, fp, fb, view, out);
}

}  // namespace vrs
