/*
 * VRSplat render-path ORACLE (test infrastructure only; see oracle.h).
 *
 * Plain CPU implementation of SURVEY.md §8(c) steps O0-O12, written from the
 * paper (/root/reference/PAPER.md, cited as P:line) and the DESIGN.md
 * "Numerics contract".  Decision quantities (everything that decides culling,
 * tile membership, sort keys, per-sample membership and per-sample order) are
 * IEEE binary32 in the exact operation order of the contract (explicit fmaf,
 * IEEE / and sqrt; built with -ffp-contract=off).  Tolerance-only quantities
 * (alpha, colour, transmittance, accumulated RGB/A/D) are computed in double.
 * Conservative-only quantities (frustum-cone cull, footprint rectangle) are
 * computed in double with explicit safety margins.
 *
 * No blocking, fusion or reordering beyond the algorithm: one stage after the
 * other, std::stable_sort for the global sort, plain loops for the rest;
 * threads only across independent output samples.
 *
 * Every function is pinned (tests/test_oracle_pins*.py):
 * the readings of DESIGN.md (L5 dilation, L12/L13/L17 periphery, R4 tau
 * clamp) are contract choices, and the oracle's implementation of each is
 * checked against closed forms, limits or an independent reconstruction.
 */
#include "oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <thread>
#include <vector>

namespace {

/* ------------------------------------------------------------------ scene */

struct Scene {
    int64_t n = 0;
    int deg = 0;
    int ncoef = 1;
    std::vector<float> mu, cov, icov, sigma, qcut, sh;  // activated, compacted
    std::map<int, std::vector<uint8_t>> masks;          // slot -> W*H bytes
    std::map<int, std::pair<int, int>> mask_dims;
};

/* O0 / SURVEY §8a step 0 / L1: activation of raw 3DGS attributes on the host
 * in double, rounded once to float.  Sigma = R S S^T R^T (Eq.1);
 * its inverse R S^-2 R^T; sigma = sigmoid(logit); q_cut = 2 ln(255 sigma)
 * (alpha >= 1/255 <=> q <= q_cut).  Non-finite records are dropped and
 * counted; the quaternion is normalised silently. */
static bool activate_one(const float* m, const float* q, const float* ls, float logit, const float* shc,
                         int ncoef, float* mu, float* cov, float* icov, float* sig, float* qc) {
    for (int i = 0; i < 3; i++) if (!std::isfinite(m[i]) || !std::isfinite(ls[i])) return false;
    for (int i = 0; i < 4; i++) if (!std::isfinite(q[i])) return false;
    if (!std::isfinite(logit)) return false;
    for (int i = 0; i < ncoef * 3; i++) if (!std::isfinite(shc[i])) return false;
    double w = q[0], x = q[1], y = q[2], z = q[3];
    double nrm = std::sqrt(w * w + x * x + y * y + z * z);
    if (!(nrm > 0.0)) return false;
    w /= nrm; x /= nrm; y /= nrm; z /= nrm;
    double R[3][3] = {{1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)},
                      {2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)},
                      {2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)}};
    double s2[3], is2[3];
    for (int k = 0; k < 3; k++) {
        double s = std::exp((double)ls[k]);
        s2[k] = s * s;
        is2[k] = 1.0 / s2[k];
    }
    const int I[6] = {0, 0, 0, 1, 1, 2}, J[6] = {0, 1, 2, 1, 2, 2};
    for (int e = 0; e < 6; e++) {
        int i = I[e], j = J[e];
        double c = (R[i][0] * R[j][0]) * s2[0] + (R[i][1] * R[j][1]) * s2[1] + (R[i][2] * R[j][2]) * s2[2];
        double ic = (R[i][0] * R[j][0]) * is2[0] + (R[i][1] * R[j][1]) * is2[1] + (R[i][2] * R[j][2]) * is2[2];
        cov[e] = (float)c;
        icov[e] = (float)ic;
        if (!std::isfinite(cov[e]) || !std::isfinite(icov[e])) return false;
    }
    double sg = 1.0 / (1.0 + std::exp(-(double)logit));
    float sgf = (float)sg;
    *sig = sgf;
    *qc = (float)(2.0 * std::log(255.0 * (double)sgf));
    for (int i = 0; i < 3; i++) mu[i] = m[i];
    return true;
}

/* ------------------------------------------------------------- per view */

// Splat record for one (view, gaussian): SURVEY §8(c) O1-O6.
struct Splat {
    int valid = 0;
    float muc[3] = {0, 0, 0}, u[3] = {0, 0, 0}, e1[3] = {0, 0, 0}, e2[3] = {0, 0, 0};
    float S2[3] = {0, 0, 0}, C[3] = {0, 0, 0}, eps = 0, A[6] = {0, 0, 0, 0, 0, 0};
    float bv[3] = {0, 0, 0}, rgb[3] = {0, 0, 0}, sigma = 0, qcut = 0;
    int rect[4] = {0, 0, -1, -1};  // tx0, ty0, tx1, ty1 (inclusive); empty if tx0 > tx1
    float bbox[4] = {0, 0, 0, 0};  // conservative pixel extent xmin, xmax, ymin, ymax
    uint32_t count = 0;
    // EWA baseline (projection = 1, config C5): pixel-space mean and conic
    float m2[2] = {0, 0}, Cp[3] = {0, 0, 0};
};

enum { CLS_HIGH = 0, CLS_LOW = 1, CLS_HYBRID = 2, CLS_INVIS = 3 };

struct ViewState {
    orc_view v;
    int tw = 0, th = 0;        // coarse (assignment) tile grid
    int64_t tile_base = 0;     // global tile id offset
    std::vector<int32_t> vis;  // per tile visibility bit
    std::vector<uint32_t> sat; // summed-area table
    std::vector<int32_t> cls;  // per tile class
    std::vector<Splat> splats;
};

struct Oracle {
    Scene sc;
    orc_params p{};
    std::vector<ViewState> views;
    std::vector<uint32_t> counts;       // [view][g]
    std::vector<uint64_t> keys_unsorted, keys;
    std::vector<uint32_t> vals_unsorted, vals;
    std::vector<uint32_t> ranges;       // [global tile][2]
    int64_t ntiles = 0;
    int64_t stats[ORC_STATS] = {0};
};

/* DESIGN "Numerics contract" R6: dot3(a,b) = fmaf(a.x,b.x, fmaf(a.y,b.y, a.z*b.z)). */
static inline float dot3(const float* a, const float* b) {
    return std::fmaf(a[0], b[0], std::fmaf(a[1], b[1], a[2] * b[2]));
}
/* Quadratic form d^T Q d for the stored pre-doubled coefficients
 * (a=Q00, b=2Q01, c=Q11, p=2Q02, e=2Q12, f=Q22); R6 "per-sample quadratic",
 * generalised to d.z != 1 (the z = 1 case reduces exactly to the R6 form). */
static inline float quad3(const float* Q, float x, float y, float z) {
    return std::fmaf(std::fmaf(Q[0], x, std::fmaf(Q[1], y, Q[3] * z)), x,
                     std::fmaf(std::fmaf(Q[2], y, Q[4] * z), y, (Q[5] * z) * z));
}

/* Homogeneous chart quadratic of a ray d (R6 "per-sample quadratic"):
 * ex = e1.d, ey = e2.d (the ray's chart point times s = u.d),
 * num = [ex ey] C [ex ey]^T = q * s^2.  Membership is num <= q_cut*s^2 (R3). */
static inline float chart_num(const float* e1, const float* e2, const float* C, const float* d) {
    float ex = std::fmaf(e1[0], d[0], std::fmaf(e1[1], d[1], e1[2] * d[2]));
    float ey = std::fmaf(e2[0], d[0], std::fmaf(e2[1], d[1], e2[2] * d[2]));
    float cx = std::fmaf(C[0], ex, C[1] * ey), cy = std::fmaf(C[1], ex, C[2] * ey);
    return std::fmaf(ex, cx, ey * cy);
}

/* Per-sample alpha and depth in the contract's binary32 form (DESIGN R9):
 * one IEEE reciprocal r = 1/(s^2 * den) serves both quotients,
 *   x   = (num * -0.5 log2 e) * (den * r)      (= -q/2 log2 e, q = num/s^2)
 *   tau = dtb * (s^2 * r)                       (= dtb / den, StopThePop depth)
 * alpha = min(0.99, sigma * 2^x), 2^x = 2^n * p(f), n = floor x,
 * p a fixed degree-5 polynomial (relative error 1.5e-7), scaled exactly.  All
 * implementations therefore produce identical alpha and transmittance
 * T_k = T_{k-1} * (1 - alpha_k), so the T < 1e-4 stop is an exact decision. */
struct SampleAT { float alpha, tau; };
static inline float alpha_of_x(float x, float sigma) {
    float fl = std::floor(x);
    float f = x - fl;
    float p = 0.00187757565f;
    p = std::fmaf(p, f, 0.00898934249f);
    p = std::fmaf(p, f, 0.0558263175f);
    p = std::fmaf(p, f, 0.240153611f);
    p = std::fmaf(p, f, 0.693153083f);
    p = std::fmaf(p, f, 0.99999994f);
    float e = std::ldexp(p, (int)fl);
    float a = sigma * e;
    return a < 0.99f ? a : 0.99f;
}
/* r = 1/v in IEEE binary32 with v clamped to [2^-100, 2^100] (R9; the clamp
 * never binds for a visible splat and lets the GPU skip rcp.rn's slow path). */
static inline float rcp_clamped(float v) {
    return 1.0f / std::fmin(std::fmax(v, 0x1p-100f), 0x1p100f);
}
static inline SampleAT sample_alpha_tau(float num, float ss, float den, float dtb, float sigma, float near_plane) {
    float r = rcp_clamped(ss * den);
    float x = std::fmax((num * -0.72134752f) * (den * r), -64.0f);  // NaN/-inf guard
    SampleAT o;
    o.alpha = alpha_of_x(x, sigma);
    o.tau = std::fmax(dtb * (ss * r), near_plane);  // clamped >= near like the tile key (O8, R4); NaN -> near
    return o;
}
/* EWA baseline per sample (q directly in pixels; one IEEE division for tau). */
static inline SampleAT sample_alpha_tau_ewa(float q, float den, float dtb, float sigma, float near_plane) {
    SampleAT o;
    o.alpha = alpha_of_x(std::fmax(q * -0.72134752f, -64.0f), sigma);
    o.tau = std::fmax(dtb / den, near_plane);
    return o;
}
static inline float ewa_q(const float* C, float dx, float dy) {
    return std::fmaf(dx, std::fmaf(C[0], dx, C[1] * dy), dy * std::fmaf(C[1], dx, C[2] * dy));
}

/* 3x3 symmetric (xx,xy,xz,yy,yz,zz) conjugation W S W^T, R6 "3x3 products":
 * T = W*S first, then T*W^T, each entry a dot3. */
static void conj3(const float* W, const float* S6, float* out6) {
    float S[3][3] = {{S6[0], S6[1], S6[2]}, {S6[1], S6[3], S6[4]}, {S6[2], S6[4], S6[5]}};
    float T[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            float col[3] = {S[0][j], S[1][j], S[2][j]};
            T[i][j] = dot3(&W[3 * i], col);
        }
    const int I[6] = {0, 0, 0, 1, 1, 2}, J[6] = {0, 1, 2, 1, 2, 2};
    for (int e = 0; e < 6; e++) out6[e] = dot3(T[I[e]], &W[3 * J[e]]);
}

/* View-dependent colour, real SH basis through degree 3 with the 3DGS
 * constants (SURVEY O5 [ext]), +0.5, clamped at 0.  Tolerance-only:
 * double. */
static void sh_color(const float* shc, int deg, const double dir[3], float out[3]) {
    const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                          0.5462742152960396};
    const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                          -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
    double x = dir[0], y = dir[1], z = dir[2];
    for (int c = 0; c < 3; c++) {
        auto S = [&](int k) { return (double)shc[k * 3 + c]; };
        double r = C0 * S(0);
        if (deg > 0) r = r - C1 * y * S(1) + C1 * z * S(2) - C1 * x * S(3);
        if (deg > 1) {
            double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
            r += C2[0] * xy * S(4) + C2[1] * yz * S(5) + C2[2] * (2.0 * zz - xx - yy) * S(6) + C2[3] * xz * S(7) +
                 C2[4] * (xx - yy) * S(8);
            if (deg > 2) {
                r += C3[0] * y * (3.0 * xx - yy) * S(9) + C3[1] * xy * z * S(10) +
                     C3[2] * y * (4.0 * zz - xx - yy) * S(11) + C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy) * S(12) +
                     C3[4] * x * (4.0 * zz - xx - yy) * S(13) + C3[5] * z * (xx - yy) * S(14) +
                     C3[6] * x * (xx - 3.0 * yy) * S(15);
            }
        }
        r += 0.5;
        out[c] = (float)(r > 0.0 ? r : 0.0);
    }
}

/* Shared tail of O5/O6 for both projections: depth coefficients and colour. */
static void depth_and_colour(const Scene& S, const orc_view& v, int64_t g, Splat& sp) {
    const float* mu = &S.mu[3 * g];
    float Ai[6];
    conj3(v.R, &S.icov[6 * g], Ai);  // A = W Sigma_w^-1 W^T = Sigma_c^-1
    sp.A[0] = Ai[0];
    sp.A[1] = 2.0f * Ai[1];
    sp.A[2] = Ai[3];
    sp.A[3] = 2.0f * Ai[2];
    sp.A[4] = 2.0f * Ai[4];
    sp.A[5] = Ai[5];
    float Am[3][3] = {{Ai[0], Ai[1], Ai[2]}, {Ai[1], Ai[3], Ai[4]}, {Ai[2], Ai[4], Ai[5]}};
    for (int i = 0; i < 3; i++) sp.bv[i] = dot3(Am[i], sp.muc);
    double d[3] = {(double)mu[0] - v.o[0], (double)mu[1] - v.o[1], (double)mu[2] - v.o[2]};
    double nd = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int i = 0; i < 3; i++) d[i] /= nd;
    sh_color(&S.sh[(size_t)g * S.ncoef * 3], S.deg, d, sp.rgb);
}

/* Pixel bbox [xmin,xmax]x[ymin,ymax] (already expanded) -> bbox + tile rect (O6d). */
static void set_rect(const Oracle& O, const ViewState& vs, double xmin, double xmax, double ymin, double ymax,
                     Splat& sp) {
    const double W = vs.v.width, H = vs.v.height;
    sp.bbox[0] = (float)std::max(xmin, -2.0); sp.bbox[1] = (float)std::min(xmax, W + 2.0);
    sp.bbox[2] = (float)std::max(ymin, -2.0); sp.bbox[3] = (float)std::min(ymax, H + 2.0);
    const int T_a = O.p.assign_tile;
    if (xmax < 0.0 || ymax < 0.0 || xmin > W || ymin > H) return;  // empty rect
    sp.rect[0] = std::max(0, (int)std::floor(std::max(xmin, 0.0) / T_a));
    sp.rect[1] = std::max(0, (int)std::floor(std::max(ymin, 0.0) / T_a));
    sp.rect[2] = std::min(vs.tw - 1, (int)std::floor(std::min(xmax, W) / T_a));
    sp.rect[3] = std::min(vs.th - 1, (int)std::floor(std::min(ymax, H) / T_a));
}

/* EWA baseline (Eq.3; SURVEY "EWA mode", config C5): the 3DGS
 * local-affine projection Sigma_2D = J W Sigma W^T J^T + 0.3 I in pixels
 * ([ext] 3DGS computeCov2D, with its 1.3 tan(fov/2) clamp of the Jacobian
 * point), per-sample q = D^T C D from the projected mean, tiles tested in
 * screen space (StopThePop's original tile culling). */
static void preprocess_ewa(const Oracle& O, const ViewState& vs, int64_t g, Splat& sp) {
    const Scene& S = O.sc;
    const orc_view& v = vs.v;
    float Sc[6];
    conj3(v.R, &S.cov[6 * g], Sc);
    const float z = sp.muc[2];
    const float limx = 1.3f * ((0.5f * (float)v.width) / v.fx), limy = 1.3f * ((0.5f * (float)v.height) / v.fy);
    const float txtz = sp.muc[0] / z, tytz = sp.muc[1] / z;
    const float tx = std::fmin(limx, std::fmax(-limx, txtz)) * z;
    const float ty = std::fmin(limy, std::fmax(-limy, tytz)) * z;
    const float zz = z * z;
    const float J00 = v.fx / z, J02 = -(v.fx * tx) / zz, J11 = v.fy / z, J12 = -(v.fy * ty) / zz;
    // rows of J Sigma_c (Sigma_c = xx,xy,xz,yy,yz,zz)
    const float a0 = std::fmaf(J00, Sc[0], J02 * Sc[2]), a1 = std::fmaf(J00, Sc[1], J02 * Sc[4]),
                a2 = std::fmaf(J00, Sc[2], J02 * Sc[5]);
    const float b1 = std::fmaf(J11, Sc[3], J12 * Sc[4]), b2 = std::fmaf(J11, Sc[4], J12 * Sc[5]);
    float c00 = std::fmaf(a0, J00, a2 * J02), c01 = std::fmaf(a1, J11, a2 * J12), c11 = std::fmaf(b1, J11, b2 * J12);
    c00 = c00 + 0.3f;
    c11 = c11 + 0.3f;
    sp.S2[0] = c00; sp.S2[1] = c01; sp.S2[2] = c11;
    const float det = std::fmaf(c00, c11, -(c01 * c01));
    if (!(det > 0.0f)) return;
    const float idet = 1.0f / det;
    sp.Cp[0] = c11 * idet;
    sp.Cp[1] = -c01 * idet;
    sp.Cp[2] = c00 * idet;
    sp.m2[0] = std::fmaf(v.fx, sp.muc[0] / z, v.cx);
    sp.m2[1] = std::fmaf(v.fy, sp.muc[1] / z, v.cy);
    depth_and_colour(S, v, g, sp);
    sp.valid = 1;
    // footprint: axis extents of D^T C D <= q_cut are sqrt(q_cut Sigma_ii), + 1 px
    const double rx = std::sqrt((double)sp.qcut * c00), ry = std::sqrt((double)sp.qcut * c11);
    set_rect(O, vs, sp.m2[0] - rx - 1.0, sp.m2[0] + rx + 1.0, sp.m2[1] - ry - 1.0, sp.m2[1] + ry + 1.0, sp);
}

/* O1-O6 for one Gaussian in one view. */
static void preprocess_one(const Oracle& O, const ViewState& vs, int64_t g, Splat& sp) {
    const Scene& S = O.sc;
    const orc_view& v = vs.v;
    const float* mu = &S.mu[3 * g];
    sp = Splat();
    // O1 view transform and near cull; never-contributing (q_cut < 0).
    float vv[3] = {mu[0] - v.o[0], mu[1] - v.o[1], mu[2] - v.o[2]};
    for (int i = 0; i < 3; i++) sp.muc[i] = dot3(&v.R[3 * i], vv);
    sp.qcut = S.qcut[g];
    sp.sigma = S.sigma[g];
    if (!(sp.muc[2] > O.p.near_plane) || sp.qcut < 0.0f) return;
    if (O.p.projection == 1) {
        preprocess_ewa(O, vs, g, sp);
        return;
    }
    // O2 optimal plane: tangent plane of the unit sphere at o, perpendicular
    // to o->mu.  u = mu_c / r, basis e1, e2.
    float r2 = dot3(sp.muc, sp.muc);
    float r = std::sqrt(r2);
    float inv_r = 1.0f / r;
    for (int i = 0; i < 3; i++) sp.u[i] = sp.muc[i] * inv_r;
    float h = std::sqrt(std::fmaf(sp.u[2], sp.u[2], sp.u[0] * sp.u[0]));
    float ih = 1.0f / h;
    sp.e1[0] = sp.u[2] * ih;
    sp.e1[1] = 0.0f;
    sp.e1[2] = -(sp.u[0] * ih);
    sp.e2[0] = sp.u[1] * sp.e1[2];
    sp.e2[1] = std::fmaf(sp.u[2], sp.e1[0], -(sp.u[0] * sp.e1[2]));
    sp.e2[2] = -(sp.u[1] * sp.e1[0]);
    // O3 projected covariance Sigma_2 = (1/r^2) E^T Sigma_c E, Sigma_c = W Sigma_w W^T.
    float Sc[6];
    conj3(v.R, &S.cov[6 * g], Sc);
    float Scm[3][3] = {{Sc[0], Sc[1], Sc[2]}, {Sc[1], Sc[3], Sc[4]}, {Sc[2], Sc[4], Sc[5]}};
    float P1[3], P2[3];
    for (int i = 0; i < 3; i++) {
        P1[i] = dot3(Scm[i], sp.e1);
        P2[i] = dot3(Scm[i], sp.e2);
    }
    float ir2 = inv_r * inv_r;
    float s00 = dot3(sp.e1, P1) * ir2, s01 = dot3(sp.e1, P2) * ir2, s11 = dot3(sp.e2, P2) * ir2;
    // O4 pixel-mapped dilation (+0.3 px^2 at the mean's image position, L5).
    float jx = sp.u[2] / v.fx, jy = sp.u[2] / v.fy;
    float J00 = sp.e1[0] * jx, J01 = sp.e1[1] * jy, J10 = sp.e2[0] * jx, J11 = sp.e2[1] * jy;
    float d00 = std::fmaf(J00, J00, J01 * J01), d01 = std::fmaf(J00, J10, J01 * J11),
          d11 = std::fmaf(J10, J10, J11 * J11);
    s00 = std::fmaf(0.3f, d00, s00);
    s01 = std::fmaf(0.3f, d01, s01);
    s11 = std::fmaf(0.3f, d11, s11);
    sp.S2[0] = s00; sp.S2[1] = s01; sp.S2[2] = s11;
    // O5 conic C = Sigma_2^-1, depth coefficients.
    float det = std::fmaf(s00, s11, -(s01 * s01));
    if (!(det > 0.0f)) return;
    float idet = 1.0f / det;
    sp.C[0] = s11 * idet;
    sp.C[1] = -s01 * idet;
    sp.C[2] = s00 * idet;
    // clip level for O7: rays with 0 < u.d < eps have tan^2(angle to u) >
    // (1-eps^2)/eps^2 >= 4 (1 + q_cut tr(Sigma_2)) - 1 > q_cut * lambda_max / lambda... i.e.
    // q >= tan^2 / lambda_max(Sigma_2) > q_cut (tr >= lambda_max), DESIGN R8.
    sp.eps = 0.5f / std::sqrt(std::fmaf(sp.qcut, s00 + s11, 1.0f));
    depth_and_colour(S, v, g, sp);
    // O6(a) cone vs frustum side planes (conservative, double, margin 1e-4).
    double S00 = s00, S01 = s01, S11 = s11;
    double lmax = 0.5 * (S00 + S11) + std::sqrt(0.25 * (S00 - S11) * (S00 - S11) + S01 * S01);
    double t2 = (double)sp.qcut * lmax;
    double sinb = std::sqrt(t2 / (1.0 + t2));
    double ud[3] = {sp.u[0], sp.u[1], sp.u[2]};
    {
        double xl = (0.0 - v.cx) / v.fx, xr = ((double)v.width - v.cx) / v.fx;
        double yt = (0.0 - v.cy) / v.fy, yb = ((double)v.height - v.cy) / v.fy;
        double N[4][3] = {{1.0, 0.0, -xl}, {-1.0, 0.0, xr}, {0.0, 1.0, -yt}, {0.0, -1.0, yb}};
        for (int k = 0; k < 4; k++) {
            double nn = std::sqrt(N[k][0] * N[k][0] + N[k][1] * N[k][1] + N[k][2] * N[k][2]);
            double nu = (N[k][0] * ud[0] + N[k][1] * ud[1] + N[k][2] * ud[2]) / nn;
            if (nu < -(sinb + 1e-4)) return;  // cone entirely outside this plane
        }
    }
    sp.valid = 1;
    // O6(b) conic bbox on the image plane, (c) whole-screen fallback.
    const double W = v.width, H = v.height;
    double xmin = -1e30, xmax = 1e30, ymin = -1e30, ymax = 1e30;
    bool whole = !(ud[2] > sinb + 1e-3);
    if (!whole) {
        // ray conic M = E C E^T rebuilt in double from the float frame and conic
        double Mf[3][3];
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++)
                Mf[i][j] = (double)sp.C[0] * sp.e1[i] * sp.e1[j] + (double)sp.C[1] * (sp.e1[i] * (double)sp.e2[j] +
                           sp.e2[i] * (double)sp.e1[j]) + (double)sp.C[2] * sp.e2[i] * sp.e2[j];
        double G[3][3];
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) G[i][j] = Mf[i][j] - (double)sp.qcut * ud[i] * ud[j];
        double Ki[3][3] = {{1.0 / v.fx, 0.0, -(double)v.cx / v.fx}, {0.0, 1.0 / v.fy, -(double)v.cy / v.fy},
                           {0.0, 0.0, 1.0}};
        double T[3][3], Q[3][3];
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) {
                T[i][j] = 0.0;
                for (int k = 0; k < 3; k++) T[i][j] += G[i][k] * Ki[k][j];
            }
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) {
                Q[i][j] = 0.0;
                for (int k = 0; k < 3; k++) Q[i][j] += Ki[k][i] * T[k][j];
            }
        double a00 = Q[1][1] * Q[2][2] - Q[1][2] * Q[1][2];
        double a11 = Q[0][0] * Q[2][2] - Q[0][2] * Q[0][2];
        double a22 = Q[0][0] * Q[1][1] - Q[0][1] * Q[0][1];
        double a02 = Q[0][1] * Q[1][2] - Q[0][2] * Q[1][1];
        double a12 = Q[0][1] * Q[0][2] - Q[0][0] * Q[1][2];
        double dx = a02 * a02 - a00 * a22, dy = a12 * a12 - a11 * a22;
        if (a22 != 0.0 && dx >= 0.0 && dy >= 0.0 && std::isfinite(dx) && std::isfinite(dy)) {
            double sx = std::sqrt(dx), sy = std::sqrt(dy);
            double xa = (a02 - sx) / a22, xb = (a02 + sx) / a22;
            double ya = (a12 - sy) / a22, yb = (a12 + sy) / a22;
            xmin = std::min(xa, xb); xmax = std::max(xa, xb);
            ymin = std::min(ya, yb); ymax = std::max(ya, yb);
        } else {
            whole = true;
        }
    }
    if (whole) { xmin = -1.0; xmax = W + 1.0; ymin = -1.0; ymax = H + 1.0; }
    // O6(d) expand by 1 px, inclusive coarse-tile rect, clamp.
    set_rect(O, vs, xmin - 1.0, xmax + 1.0, ymin - 1.0, ymax + 1.0, sp);
}

/* Minimum of the 2D quadratic X^T C X over a convex polygon (vertices relative
 * to the Gaussian's mean): 0 if the mean (origin) is inside (all edge cross
 * products share a sign), else Eq.4 on every edge with t
 * clamped to [0,1], strictly smaller q wins (earlier edge on ties). */
static void poly_min(const float* C, const float* yx, const float* yy, int n, float* qmin_out, float* hx_out,
                     float* hy_out) {
    // mean (chart origin) inside the convex polygon: all edge cross products share a sign
    int npos = 0, nneg = 0;
    for (int k = 0; k < n; k++) {
        int k1 = (k + 1 == n) ? 0 : k + 1;
        float ddx = yx[k1] - yx[k], ddy = yy[k1] - yy[k];
        float cr = std::fmaf(ddy, yx[k], -(ddx * yy[k]));
        if (cr >= 0.0f) npos++;
        if (cr <= 0.0f) nneg++;
    }
    float hx, hy, qmin;
    if (npos == n || nneg == n) {
        hx = 0.0f; hy = 0.0f; qmin = 0.0f;  // x_hat = mu_2D
    } else {
        qmin = INFINITY; hx = 0.0f; hy = 0.0f;
        for (int k = 0; k < n; k++) {  // Eq.4 on every edge, t clamped to [0,1]
            int k1 = (k + 1 == n) ? 0 : k + 1;
            float ppx = yx[k], ppy = yy[k];
            float ddx = yx[k1] - yx[k], ddy = yy[k1] - yy[k];
            float cdx = std::fmaf(C[0], ddx, C[1] * ddy), cdy = std::fmaf(C[1], ddx, C[2] * ddy);
            float den = std::fmaf(ddx, cdx, ddy * cdy);
            float nmr = -std::fmaf(ppx, cdx, ppy * cdy);  // d^T C (mu2D - p), mu2D = 0
            float t;
            if (nmr <= 0.0f || !(den > 0.0f)) t = 0.0f;
            else if (nmr >= den) t = 1.0f;
            else t = nmr / den;
            float X = std::fmaf(t, ddx, ppx), Y = std::fmaf(t, ddy, ppy);
            float cX = std::fmaf(C[0], X, C[1] * Y), cY = std::fmaf(C[1], X, C[2] * Y);
            float q = std::fmaf(X, cX, Y * cY);
            if (q < qmin) { qmin = q; hx = X; hy = Y; }
        }
    }
    *qmin_out = qmin;
    *hx_out = hx;
    *hy_out = hy;
}

/* O7 (Eq.4) on the Gaussian's optimal plane; returns keep and
 * the ray d_hat through the maximum point x_hat.  Tile = closed
 * pixel-edge rectangle [x0,x1]x[y0,y1] (L8).  Projecting the tile onto the
 * optimal plane gives a convex polygon.  Corner rays are first
 * clipped to s = u.d >= eps (rays with 0 < s < eps provably have
 * q > q_cut: DESIGN reading R8 / L20), so the polygon is bounded; the mean
 * (chart origin) inside it gives x_hat = mu_2D, otherwise Eq.4 runs on
 * every polygon edge with t clamped to [0,1].  Keep iff
 * q_min <= q_cut * 1.001 (conservative prefilter, DESIGN reading R7). */
static bool tile_test(const Splat& sp, const orc_view& v, int x0, int y0, int x1, int y1, float* qmin_out,
                      float dhat[3]) {
    const int cx_[4] = {x0, x1, x1, x0}, cy_[4] = {y0, y0, y1, y1};  // TL, TR, BR, BL
    float dx[4], dy[4], s[4];
    int nin = 0;
    for (int k = 0; k < 4; k++) {
        dx[k] = ((float)cx_[k] - v.cx) / v.fx;
        dy[k] = ((float)cy_[k] - v.cy) / v.fy;
        s[k] = std::fmaf(sp.u[0], dx[k], std::fmaf(sp.u[1], dy[k], sp.u[2]));
        if (s[k] >= sp.eps) nin++;
    }
    *qmin_out = INFINITY;
    if (nin == 0) return false;  // tile entirely at s < eps: no contribution (L20)
    // polygon on the image plane z = 1 (Sutherland-Hodgman against s >= eps)
    float px[5], py[5];
    int n = 0;
    for (int k = 0; k < 4; k++) {
        int k1 = (k + 1) & 3;
        bool ia = s[k] >= sp.eps, ib = s[k1] >= sp.eps;
        if (ia) { px[n] = dx[k]; py[n] = dy[k]; n++; }
        if (ia != ib) {  // crossing, interpolated from the inside vertex
            int a = ia ? k : k1, b = ia ? k1 : k;
            float t = (s[a] - sp.eps) / (s[a] - s[b]);
            px[n] = std::fmaf(t, dx[b] - dx[a], dx[a]);
            py[n] = std::fmaf(t, dy[b] - dy[a], dy[a]);
            n++;
        }
    }
    float yx[5], yy[5];
    for (int k = 0; k < n; k++) {
        float d[3] = {px[k], py[k], 1.0f};
        float is = 1.0f / dot3(sp.u, d);  // chart point = (e1.d, e2.d) / (u.d)  (R6: one IEEE reciprocal)
        yx[k] = dot3(sp.e1, d) * is;
        yy[k] = dot3(sp.e2, d) * is;
    }
    float hx, hy, qmin;
    poly_min(sp.C, yx, yy, n, &qmin, &hx, &hy);
    *qmin_out = qmin;
    for (int i = 0; i < 3; i++) dhat[i] = std::fmaf(hy, sp.e2[i], std::fmaf(hx, sp.e1[i], sp.u[i]));
    return qmin <= sp.qcut * 1.001f;
}

/* EWA baseline O7: StopThePop's screen-space tile test: the tile's
 * pixel-edge rectangle relative to the projected mean, the same polygon
 * minimum in pixel units; the ray through x_hat gives the key depth. */
static bool tile_test_ewa(const Splat& sp, const orc_view& v, int x0, int y0, int x1, int y1, float* qmin_out,
                          float dhat[3]) {
    const int cx_[4] = {x0, x1, x1, x0}, cy_[4] = {y0, y0, y1, y1};
    float yx[4], yy[4];
    for (int k = 0; k < 4; k++) {
        yx[k] = (float)cx_[k] - sp.m2[0];
        yy[k] = (float)cy_[k] - sp.m2[1];
    }
    float hx, hy, qmin;
    poly_min(sp.Cp, yx, yy, 4, &qmin, &hx, &hy);
    *qmin_out = qmin;
    dhat[0] = ((sp.m2[0] + hx) - v.cx) / v.fx;
    dhat[1] = ((sp.m2[1] + hy) - v.cy) / v.fy;
    dhat[2] = 1.0f;
    return qmin <= sp.qcut * 1.001f;
}

/* O8 key depth: StopThePop per-tile depth = distance of the max-density
 * point along the unit ray through x_hat, clamped >= near. */
static float tile_depth(const Splat& sp, const float d[3], float near_plane) {
    float dAd = quad3(sp.A, d[0], d[1], d[2]);
    float db = std::fmaf(sp.bv[0], d[0], std::fmaf(sp.bv[1], d[1], sp.bv[2] * d[2]));
    float nd = std::sqrt(dot3(d, d));
    float t = nd * (db / dAd);
    return (t > near_plane) ? t : near_plane;
}

/* Global-sort baselines (N3): one depth per (view, Gaussian)
 * for every tile -- Mini-Splatting (z): the view-space z of mu (the 3DGS sort
 * order, "given by the z-coordinate of mu in view-space");
 * Mini-Splatting (Dist): |mu - o| = sqrt(mu_c . mu_c).  Both
 * exceed near (O1 culls mu_c.z <= near, and |mu_c| >= mu_c.z). */
static float global_depth(const Splat& sp, int mode) {
    if (mode == 1) return sp.muc[2];
    return std::sqrt(dot3(sp.muc, sp.muc));
}

static inline uint32_t fbits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}

/* Per-pixel blend weight of the fovea ramp (L12): 1 inside the full-rate
 * rect, linear to 0 over ramp*(2*radius) outside, at pixel centres. */
static float fovea_weight(const orc_view& v, float px, float py) {
    float ax = std::fabs(px - v.fovea_center[0]) - v.fovea_radius[0];
    float ay = std::fabs(py - v.fovea_center[1]) - v.fovea_radius[1];
    ax = ax > 0.0f ? ax : 0.0f;
    ay = ay > 0.0f ? ay : 0.0f;
    float dxn = v.fovea_ramp * (2.0f * v.fovea_radius[0]);
    float dyn = v.fovea_ramp * (2.0f * v.fovea_radius[1]);
    float wx = dxn > 0.0f ? ax / dxn : (ax > 0.0f ? 1.0f : 0.0f);
    float wy = dyn > 0.0f ? ay / dyn : (ay > 0.0f ? 1.0f : 0.0f);
    float m = wx > wy ? wx : wy;
    float w = 1.0f - m;
    return w < 0.0f ? 0.0f : (w > 1.0f ? 1.0f : w);
}

/* Per-view static setup: visibility bitfield, SAT,
 * tile classes. */
static void setup_view(Oracle& O, ViewState& vs) {
    const orc_view& v = vs.v;
    const int T = O.p.assign_tile;
    vs.tw = (v.width + T - 1) / T;
    vs.th = (v.height + T - 1) / T;
    vs.vis.assign((size_t)vs.tw * vs.th, 1);
    const uint8_t* mask = nullptr;
    auto it = O.sc.masks.find(v.mask_slot);
    if (v.mask_slot >= 0 && it != O.sc.masks.end()) mask = it->second.data();
    if (mask) {
        for (int ty = 0; ty < vs.th; ty++)
            for (int tx = 0; tx < vs.tw; tx++) {
                int any = 0;
                for (int y = ty * T; y < std::min((ty + 1) * T, v.height) && !any; y++)
                    for (int x = tx * T; x < std::min((tx + 1) * T, v.width); x++)
                        if (mask[(size_t)y * v.width + x] > 0) { any = 1; break; }
                vs.vis[(size_t)ty * vs.tw + tx] = any;
            }
    }
    vs.sat.assign((size_t)(vs.tw + 1) * (vs.th + 1), 0);
    for (int ty = 0; ty < vs.th; ty++)
        for (int tx = 0; tx < vs.tw; tx++)
            vs.sat[(size_t)(ty + 1) * (vs.tw + 1) + tx + 1] = vs.sat[(size_t)ty * (vs.tw + 1) + tx + 1] +
                                                              vs.sat[(size_t)(ty + 1) * (vs.tw + 1) + tx] -
                                                              vs.sat[(size_t)ty * (vs.tw + 1) + tx] +
                                                              (uint32_t)vs.vis[(size_t)ty * vs.tw + tx];
    vs.cls.assign((size_t)vs.tw * vs.th, CLS_HIGH);
    for (int ty = 0; ty < vs.th; ty++)
        for (int tx = 0; tx < vs.tw; tx++) {
            size_t t = (size_t)ty * vs.tw + tx;
            if (!vs.vis[t]) { vs.cls[t] = CLS_INVIS; continue; }
            if (!v.fovea_enabled) { vs.cls[t] = CLS_HIGH; continue; }
            bool all1 = true, all0 = true;
            for (int y = ty * T; y < std::min((ty + 1) * T, v.height); y++)
                for (int x = tx * T; x < std::min((tx + 1) * T, v.width); x++) {
                    float w = fovea_weight(v, (float)x + 0.5f, (float)y + 0.5f);
                    if (w != 1.0f) all1 = false;
                    if (w != 0.0f) all0 = false;
                }
            vs.cls[t] = all1 ? CLS_HIGH : (all0 ? CLS_LOW : CLS_HYBRID);
        }
}

static inline int64_t sat_count(const ViewState& vs, int x0, int y0, int x1, int y1) {
    const int S = vs.tw + 1;
    return (int64_t)vs.sat[(size_t)(y1 + 1) * S + x1 + 1] - vs.sat[(size_t)y0 * S + x1 + 1] -
           vs.sat[(size_t)(y1 + 1) * S + x0] + vs.sat[(size_t)y0 * S + x0];
}

/* Walk a splat's rect in row-major order, skipping invisible tiles, running
 * O7; calls f(tx, ty, dhat) for every kept tile. */
template <class F>
static void for_kept_tiles(const Oracle& O, const ViewState& vs, const Splat& sp, F&& f) {
    if (!sp.valid || sp.rect[0] > sp.rect[2] || sp.rect[1] > sp.rect[3]) return;
    if (sat_count(vs, sp.rect[0], sp.rect[1], sp.rect[2], sp.rect[3]) == 0) return;
    const int T = O.p.assign_tile;
    for (int ty = sp.rect[1]; ty <= sp.rect[3]; ty++)
        for (int tx = sp.rect[0]; tx <= sp.rect[2]; tx++) {
            if (!vs.vis[(size_t)ty * vs.tw + tx]) continue;
            int x0 = tx * T, y0 = ty * T, x1 = std::min(x0 + T, vs.v.width), y1 = std::min(y0 + T, vs.v.height);
            float qmin, dh[3];
            const bool keep = (O.p.projection == 1) ? tile_test_ewa(sp, vs.v, x0, y0, x1, y1, &qmin, dh)
                                                     : tile_test(sp, vs.v, x0, y0, x1, y1, &qmin, dh);
            if (keep) f(tx, ty, dh);
        }
}

/* ------------------------------------------------------------ rendering */

struct Px { double r, g, b, a, d; };

struct SampleStats { int64_t evals = 0, contribs = 0, overflow = 0, term = 0; };

/* O10-O11: one sample (ray through image point (xs, ys) in pixel-edge
 * coordinates) streams its tile list in key order through a K-entry window
 * sorted by (tau, g); overflow pops the minimum and blends it
 * front-to-back (Eq.2 with product transmittance, L2); stop once T < 1e-4,
 * checked after blending (L11); drain at stream end. */
struct WEnt { float tau; uint32_t g; float alpha; };

static Px render_sample(const Oracle& O, int view, int64_t gtile, float xs, float ys, SampleStats& st,
                        std::vector<uint32_t>* order = nullptr) {
    const ViewState& vs = O.views[view];
    const orc_view& v = vs.v;
    const float x = (xs - v.cx) / v.fx, y = (ys - v.cy) / v.fy;
    const float dray[3] = {x, y, 1.0f};
    const double dn = std::sqrt((double)x * x + (double)y * y + 1.0);
    // global-sort baselines (N3) have no per-sample window: every contribution
    // is blended in list order (K = 0: insert, then pop the same entry)
    const bool global = O.p.sort_mode != 0;
    const int K = global ? 0 : O.p.window_k;
    // tau clamp at near (R4) unless the pin hook asks for the unclamped reading
    const float tau_floor = O.p.tau_unclamped ? -INFINITY : O.p.near_plane;
    uint32_t b = O.ranges[2 * gtile], e = O.ranges[2 * gtile + 1];
    std::vector<WEnt> win;
    float T = 1.0f;  // transmittance: binary32 product (exact decision, R9)
    double C[3] = {0, 0, 0}, D = 0.0;
    bool done = false, overflowed = false;
    auto blend = [&](const WEnt& w) {
        const Splat& sp = vs.splats[w.g];
        if (order) order->push_back(w.g);
        double wt = (double)w.alpha * (double)T;
        for (int c = 0; c < 3; c++) C[c] += (double)sp.rgb[c] * wt;
        D += (double)w.tau * dn * wt;
        T = T * (1.0f - w.alpha);
        if (T < 1e-4f) done = true;
    };
    for (uint32_t i = b; i < e && !done; i++) {
        st.evals++;
        uint32_t g = O.vals[i];
        const Splat& sp = vs.splats[g];
        SampleAT at;
        if (O.p.projection == 1) {  // EWA baseline: q from the projected mean in pixels
            float q = ewa_q(sp.Cp, xs - sp.m2[0], ys - sp.m2[1]);
            if (!(q <= sp.qcut)) continue;
            at = sample_alpha_tau_ewa(q, quad3(sp.A, x, y, 1.0f),
                                      std::fmaf(sp.bv[0], x, std::fmaf(sp.bv[1], y, sp.bv[2])), sp.sigma,
                                      tau_floor);
        } else {
            float s = std::fmaf(sp.u[0], x, std::fmaf(sp.u[1], y, sp.u[2]));
            if (!(s > 0.0f)) continue;
            float num = chart_num(sp.e1, sp.e2, sp.C, dray);
            float ss = s * s;
            if (!(num <= sp.qcut * ss)) continue;  // alpha < 1/255, division-free (R3)
            float den = quad3(sp.A, x, y, 1.0f);
            float dtb = std::fmaf(sp.bv[0], x, std::fmaf(sp.bv[1], y, sp.bv[2]));
            at = sample_alpha_tau(num, ss, den, dtb, sp.sigma, tau_floor);  // P:254, L10, R9
        }
        float alpha = at.alpha;
        float tau = at.tau;  // depth of max density along this pixel's ray (O10)
        st.contribs++;
        WEnt ent{tau, g, alpha};
        auto pos = std::upper_bound(win.begin(), win.end(), ent, [](const WEnt& a, const WEnt& c) {
            return a.tau < c.tau || (a.tau == c.tau && a.g < c.g);
        });
        win.insert(pos, ent);
        if ((int)win.size() > K) {
            overflowed = !global;
            WEnt m = win.front();
            win.erase(win.begin());
            blend(m);
        }
    }
    for (size_t i = 0; i < win.size() && !done; i++) blend(win[i]);
    if (overflowed) st.overflow++;
    if (done) st.term++;
    Px out;
    out.r = C[0] + (double)T * O.p.background[0];
    out.g = C[1] + (double)T * O.p.background[1];
    out.b = C[2] + (double)T * O.p.background[2];
    out.a = 1.0 - (double)T;
    out.d = D;
    return out;
}

/* SURVEY N2 / DESIGN "N2 hierarchical resort": StopThePop's hierarchy
 * ("hierarchical per-pixel resorting") with a block level ahead
 * of the per-sample window.  The 16 samples of one 4x4 sample block (4x4
 * pixels of a full-rate item, 4x4 2x2-group samples of a LowRes item) stream
 * their tile's list in key order together:
 *   1. entry g is ADMITTED to the block iff at least one not-yet-terminated
 *      in-image sample of the block passes the per-sample membership test
 *      (R3, exactly as O10); the set of such samples is kept with it;
 *   2. admitted entries wait in a block queue Q sorted by (tau_B, g), tau_B =
 *      max(dtb/den, near) on the ray through the block centre (the R4/R6
 *      forms, one IEEE division);  when |Q| > K_B the minimum is RELEASED;
 *   3. a release gives every sample of its set that has not terminated the
 *      entry's per-sample alpha and tau (R9) and inserts it into that
 *      sample's window (K_P = window_k entries, ordered by (tau, g)); window
 *      overflow pops and blends the minimum exactly as O10-O11;
 *   4. at stream end Q releases in order, then every window drains (O11).
 * K_B = 0 releases every entry at admission, i.e. the flat per-sample mode
 * with K = K_P (pin H1); K_B, K_P >= list length gives the full per-sample
 * sort (pin H2).  Evaluations count list entries visited before the sample's
 * termination (the entry whose processing released the terminating blend). */
struct HEnt { float tauB; uint32_t g; uint32_t mask; uint32_t idx; };

/* Block-level list entry with everything its samples need (computed by
 * render_block_hier from the geometry, or given directly to the pin H3). */
struct HIn {
    float tauB;           // block-centre depth (R4 form)
    float tauG[4];        // 2x2-group-centre depths (R4 form), group q = (row / 2) * 2 + col / 2
    uint32_t g;           // Gaussian index (tie-break, R4)
    uint32_t member;      // bit s: sample s passes the membership test (R3)
    float tau[16], alpha[16];  // per-sample depth and alpha (R9), where member
    float rgb[3];         // colour (O5)
};

/* The two-level queue mechanics of N2 on one block's stream (steps 1-4
 * above); valid[s] = sample s is in the image; dn[s] = |d| of its ray. */
static void hier_core(const std::vector<HIn>& in, int KB, int KG, int KP, const bool* valid, const double* dn,
                      const float* bg, Px* out, SampleStats* st) {
    const uint32_t n = (uint32_t)in.size();
    float T[16];
    double C[16][3], D[16];
    bool done[16], ovf[16];
    uint32_t stop[16];
    std::vector<WEnt> win[16];
    for (int s = 0; s < 16; s++) {
        T[s] = 1.0f;
        C[s][0] = C[s][1] = C[s][2] = 0.0;
        D[s] = 0.0;
        done[s] = !valid[s];
        ovf[s] = false;
        stop[s] = n ? n - 1 : 0;
    }
    std::vector<uint32_t> colour_of;  // WEnt.g holds the entry index; colours by index
    auto blend = [&](int s, const WEnt& w, uint32_t pos) {
        const HIn& h = in[w.g];
        double wt = (double)w.alpha * (double)T[s];
        for (int c = 0; c < 3; c++) C[s][c] += (double)h.rgb[c] * wt;
        D[s] += (double)w.tau * dn[s] * wt;
        T[s] = T[s] * (1.0f - w.alpha);
        if (T[s] < 1e-4f) { done[s] = true; stop[s] = pos; }
    };
    auto release_samples = [&](const HEnt& e, uint32_t pos) {
        const HIn& h = in[e.idx];
        for (int s = 0; s < 16; s++) {
            if (!((e.mask >> s) & 1u) || done[s]) continue;
            st[s].contribs++;
            WEnt ent{h.tau[s], e.idx, h.alpha[s]};  // .g = entry index; order by (tau, Gaussian g)
            auto it = std::upper_bound(win[s].begin(), win[s].end(), ent, [&](const WEnt& a, const WEnt& c) {
                return a.tau < c.tau || (a.tau == c.tau && in[a.g].g < in[c.g].g);
            });
            win[s].insert(it, ent);
            if ((int)win[s].size() > KP) {
                ovf[s] = true;
                WEnt m = win[s].front();
                win[s].erase(win[s].begin());
                blend(s, m, pos);
            }
        }
    };
    // 2x2 group level: a block release enters the queue of every group holding a
    // not-terminated member sample (members restricted to the group), ordered by
    // the group-centre depth; group overflow releases the minimum to its samples
    std::vector<HEnt> QG[4];
    auto release = [&](const HEnt& e, uint32_t pos) {
        for (int q = 0; q < 4; q++) {
            uint32_t gm = 0;
            for (int s = 0; s < 16; s++) {
                const int row = s >> 2, col = s & 3;
                if (((row >> 1) * 2 + (col >> 1)) == q && ((e.mask >> s) & 1u) && !done[s]) gm |= 1u << s;
            }
            if (!gm) continue;
            HEnt h{in[e.idx].tauG[q], e.g, gm, e.idx};
            auto it = std::upper_bound(QG[q].begin(), QG[q].end(), h, [](const HEnt& a, const HEnt& c) {
                return a.tauB < c.tauB || (a.tauB == c.tauB && a.g < c.g);
            });
            QG[q].insert(it, h);
            if ((int)QG[q].size() > KG) {
                HEnt m = QG[q].front();
                QG[q].erase(QG[q].begin());
                release_samples(m, pos);
            }
        }
    };
    std::vector<HEnt> Q;
    for (uint32_t i = 0; i < n; i++) {
        bool all = true;
        for (int s = 0; s < 16; s++) all = all && done[s];
        if (all) break;
        uint32_t mask = 0;
        for (int s = 0; s < 16; s++)
            if (!done[s] && ((in[i].member >> s) & 1u)) mask |= 1u << s;
        if (!mask) continue;
        HEnt h{in[i].tauB, in[i].g, mask, i};
        auto it = std::upper_bound(Q.begin(), Q.end(), h, [](const HEnt& a, const HEnt& c) {
            return a.tauB < c.tauB || (a.tauB == c.tauB && a.g < c.g);
        });
        Q.insert(it, h);
        if ((int)Q.size() > KB) {
            HEnt m = Q.front();
            Q.erase(Q.begin());
            release(m, i);
        }
    }
    for (const HEnt& h : Q) release(h, n ? n - 1 : 0);
    for (int q = 0; q < 4; q++)
        for (const HEnt& h : QG[q]) release_samples(h, n ? n - 1 : 0);
    for (int s = 0; s < 16; s++) {
        for (size_t k = 0; k < win[s].size() && !done[s]; k++) blend(s, win[s][k], n ? n - 1 : 0);
        if (valid[s]) {
            st[s].evals += n ? (int64_t)stop[s] + 1 : 0;
            if (ovf[s]) st[s].overflow++;
            if (done[s]) st[s].term++;
        }
        out[s].r = C[s][0] + (double)T[s] * bg[0];
        out[s].g = C[s][1] + (double)T[s] * bg[1];
        out[s].b = C[s][2] + (double)T[s] * bg[2];
        out[s].a = 1.0 - (double)T[s];
        out[s].d = D[s];
    }
}

static void render_block_hier(const Oracle& O, int view, int64_t gtile, const float* xs, const float* ys,
                              const bool* valid, float xc, float yc, const float* xgc, const float* ygc, Px* out,
                              SampleStats* st) {
    const ViewState& vs = O.views[view];
    const orc_view& v = vs.v;
    const uint32_t b = O.ranges[2 * gtile], e = O.ranges[2 * gtile + 1];
    float x[16], y[16];
    double dn[16];
    for (int s = 0; s < 16; s++) {
        x[s] = (xs[s] - v.cx) / v.fx;
        y[s] = (ys[s] - v.cy) / v.fy;
        dn[s] = std::sqrt((double)x[s] * x[s] + (double)y[s] * y[s] + 1.0);
    }
    const float xB = (xc - v.cx) / v.fx, yB = (yc - v.cy) / v.fy;  // block-centre ray (R6 sample form)
    std::vector<HIn> in(e - b);
    for (uint32_t i = b; i < e; i++) {
        HIn& h = in[i - b];
        h.g = O.vals[i];
        const Splat& sp = vs.splats[h.g];
        float den = quad3(sp.A, xB, yB, 1.0f);
        float dtb = std::fmaf(sp.bv[0], xB, std::fmaf(sp.bv[1], yB, sp.bv[2]));
        h.tauB = std::fmax(dtb / den, O.p.near_plane);  // tau_B (R4 form; NaN -> near)
        for (int q = 0; q < 4; q++) {  // tau_G on the group-centre rays (same forms)
            const float xq = (xgc[q] - v.cx) / v.fx, yq = (ygc[q] - v.cy) / v.fy;
            const float dq = quad3(sp.A, xq, yq, 1.0f);
            const float tq = std::fmaf(sp.bv[0], xq, std::fmaf(sp.bv[1], yq, sp.bv[2]));
            h.tauG[q] = std::fmax(tq / dq, O.p.near_plane);
        }
        h.member = 0;
        for (int c = 0; c < 3; c++) h.rgb[c] = sp.rgb[c];
        for (int s = 0; s < 16; s++) {
            h.tau[s] = h.alpha[s] = 0.0f;
            float sv = std::fmaf(sp.u[0], x[s], std::fmaf(sp.u[1], y[s], sp.u[2]));
            if (!(sv > 0.0f)) continue;
            float dray[3] = {x[s], y[s], 1.0f};
            float num = chart_num(sp.e1, sp.e2, sp.C, dray);
            float ss = sv * sv;
            if (!(num <= sp.qcut * ss)) continue;  // alpha < 1/255 (R3)
            h.member |= 1u << s;
            float dens = quad3(sp.A, x[s], y[s], 1.0f);
            float dtbs = std::fmaf(sp.bv[0], x[s], std::fmaf(sp.bv[1], y[s], sp.bv[2]));
            SampleAT at = sample_alpha_tau(num, ss, dens, dtbs, sp.sigma, O.p.near_plane);
            h.tau[s] = at.tau;
            h.alpha[s] = at.alpha;
        }
    }
    hier_core(in, O.p.block_queue, O.p.group_queue, O.p.window_k, valid, dn, O.p.background, out, st);
}

/* The 4x4 sample block containing full-rate sample (i, j) or LowRes group
 * (i, j) (pixel of the group origin) of coarse tile (tx, ty): sample points,
 * in-image flags and the block centre (mean of its 16 sample points). */
static void hier_block(const ViewState& vs, int T, bool low, int i, int j, int* bx0, int* by0, float* xs,
                       float* ys, bool* valid, float* xc, float* yc, float* xgc, float* ygc) {
    const int W = vs.v.width, H = vs.v.height;
    if (low) {  // blocks of 4x4 groups = 8x8 pixels, aligned inside the tile
        int x0 = (i / T) * T, y0 = (j / T) * T;
        int gx0 = ((i - x0) / 2) & ~3, gy0 = ((j - y0) / 2) & ~3;
        *bx0 = x0 + 2 * gx0;
        *by0 = y0 + 2 * gy0;
        for (int k = 0; k < 16; k++) {
            int px = *bx0 + 2 * (k & 3), py = *by0 + 2 * (k >> 2);
            xs[k] = (float)(px + 1);
            ys[k] = (float)(py + 1);
            valid[k] = px < W && py < H;
        }
        *xc = (float)(*bx0 + 4);
        *yc = (float)(*by0 + 4);
        for (int q = 0; q < 4; q++) {  // group q: samples (2(q&1).., 2(q>>1)..) -> centre 4 px further per step
            xgc[q] = (float)(*bx0 + 4 * (q & 1) + 2);
            ygc[q] = (float)(*by0 + 4 * (q >> 1) + 2);
        }
    } else {
        *bx0 = i & ~3;
        *by0 = j & ~3;
        for (int k = 0; k < 16; k++) {
            int px = *bx0 + (k & 3), py = *by0 + (k >> 2);
            xs[k] = (float)px + 0.5f;
            ys[k] = (float)py + 0.5f;
            valid[k] = px < W && py < H;
        }
        *xc = (float)(*bx0 + 2);
        *yc = (float)(*by0 + 2);
        for (int q = 0; q < 4; q++) {
            xgc[q] = (float)(*bx0 + 2 * (q & 1) + 1);
            ygc[q] = (float)(*by0 + 2 * (q >> 1) + 1);
        }
    }
}

struct FrameCtx {
    const Oracle* O;
    int view;
    // memo of samples: key -> Px  (key = kind<<62 | y<<31 | x)
    std::map<uint64_t, Px> memo;
    SampleStats st;
    // optional precomputed sample planes (orc_render): full-rate samples at
    // pixel centres (stride We) and 2x2-group samples (stride We/2)
    const std::vector<Px>* full = nullptr;
    const std::vector<Px>* low = nullptr;
    int We = 0;
};

/* Sample value used by pixel (i,j): full-rate pixel-centre sample (HighRes,
 * Hybrid, non-foveated) or the 2x2-group centre sample (LowRes). */
static Px pixel_sample(FrameCtx& F, int i, int j, bool low) {
    const ViewState& vs = F.O->views[F.view];
    const int T = F.O->p.assign_tile;
    int tx = i / T, ty = j / T;
    int64_t gt = vs.tile_base + (int64_t)ty * vs.tw + tx;
    if (low && F.low) return (*F.low)[(size_t)(j / 2) * (F.We / 2) + (i / 2)];
    if (!low && F.full) return (*F.full)[(size_t)j * F.We + i];
    float xs, ys;
    uint64_t key;
    if (low) {
        int x0 = tx * T, y0 = ty * T;
        int gx = (i - x0) / 2, gy = (j - y0) / 2;
        xs = (float)(x0 + 2 * gx + 1);
        ys = (float)(y0 + 2 * gy + 1);
        key = (1ull << 62) | ((uint64_t)(y0 + 2 * gy) << 31) | (uint64_t)(x0 + 2 * gx);
    } else {
        xs = (float)i + 0.5f;
        ys = (float)j + 0.5f;
        key = ((uint64_t)j << 31) | (uint64_t)i;
    }
    auto it = F.memo.find(key);
    if (it != F.memo.end()) return it->second;
    if (F.O->p.resort == 1) {  // the whole 4x4 block renders together (N2)
        int bx0, by0;
        float bxs[16], bys[16], xc, yc, xgc[4], ygc[4];
        bool valid[16];
        hier_block(vs, T, low, i, j, &bx0, &by0, bxs, bys, valid, &xc, &yc, xgc, ygc);
        Px outs[16];
        SampleStats sts[16];
        render_block_hier(*F.O, F.view, gt, bxs, bys, valid, xc, yc, xgc, ygc, outs, sts);
        for (int k = 0; k < 16; k++) {
            uint64_t kk = low ? ((1ull << 62) | ((uint64_t)(by0 + 2 * (k >> 2)) << 31) | (uint64_t)(bx0 + 2 * (k & 3)))
                              : (((uint64_t)(by0 + (k >> 2)) << 31) | (uint64_t)(bx0 + (k & 3)));
            F.memo[kk] = outs[k];
        }
        return F.memo[key];
    }
    Px p = render_sample(*F.O, F.view, gt, xs, ys, F.st);
    F.memo[key] = p;
    return p;
}

static inline int tile_class(const ViewState& vs, int T, int i, int j) {
    return vs.cls[(size_t)(j / T) * vs.tw + (i / T)];
}

/* O12 compose for output pixel (i,j). */
static Px pixel_out(FrameCtx& F, int i, int j) {
    const Oracle& O = *F.O;
    const ViewState& vs = O.views[F.view];
    const orc_view& v = vs.v;
    const int T = O.p.assign_tile;
    int cls = tile_class(vs, T, i, j);
    if (cls == CLS_INVIS) return Px{O.p.background[0], O.p.background[1], O.p.background[2], 0.0, 0.0};
    if (cls == CLS_HIGH) return pixel_sample(F, i, j, false);
    if (cls == CLS_HYBRID) {  // w*P + (1-w)*avg_2x2(P)
        int i0 = i & ~1, j0 = j & ~1;
        Px p00 = pixel_sample(F, i0, j0, false), p01 = pixel_sample(F, i0 + 1, j0, false);
        Px p10 = pixel_sample(F, i0, j0 + 1, false), p11 = pixel_sample(F, i0 + 1, j0 + 1, false);
        Px p = pixel_sample(F, i, j, false);
        double w = fovea_weight(v, (float)i + 0.5f, (float)j + 0.5f);
        auto mix = [&](double P, double a, double b, double c, double d) {
            double avg = ((a + b) + (c + d)) * 0.25;
            return w * P + (1.0 - w) * avg;
        };
        return Px{mix(p.r, p00.r, p01.r, p10.r, p11.r), mix(p.g, p00.g, p01.g, p10.g, p11.g),
                  mix(p.b, p00.b, p01.b, p10.b, p11.b), mix(p.a, p00.a, p01.a, p10.a, p11.a),
                  mix(p.d, p00.d, p01.d, p10.d, p11.d)};
    }
    // LowRes: nearest-neighbour upsample + 3x3 (1,2,1)x(1,2,1) blur over
    // LowRes-class in-image neighbours, renormalised.
    double acc[5] = {0, 0, 0, 0, 0}, wsum = 0.0;
    for (int dj = -1; dj <= 1; dj++)
        for (int di = -1; di <= 1; di++) {
            int ii = i + di, jj = j + dj;
            if (ii < 0 || jj < 0 || ii >= v.width || jj >= v.height) continue;
            if (tile_class(vs, T, ii, jj) != CLS_LOW) continue;
            double w = (double)((2 - std::abs(di)) * (2 - std::abs(dj)));
            Px p = pixel_sample(F, ii, jj, true);
            acc[0] += w * p.r; acc[1] += w * p.g; acc[2] += w * p.b; acc[3] += w * p.a; acc[4] += w * p.d;
            wsum += w;
        }
    return Px{acc[0] / wsum, acc[1] / wsum, acc[2] / wsum, acc[3] / wsum, acc[4] / wsum};
}

static int nthreads(const Oracle& O) {
    int t = O.p.threads;
    if (t <= 0) t = (int)std::thread::hardware_concurrency();
    return t < 1 ? 1 : t;
}

}  // namespace

/* ======================================================================= API */

extern "C" {

void* orc_create(int64_t n, int sh_degree, const float* means, const float* quats, const float* log_scales,
                 const float* logits, const float* sh, int64_t* n_rejected) {
    if (n < 0 || sh_degree < 0 || sh_degree > 3) return nullptr;
    Oracle* O = new Oracle();
    Scene& S = O->sc;
    S.deg = sh_degree;
    S.ncoef = (sh_degree + 1) * (sh_degree + 1);
    S.mu.reserve(3 * n); S.cov.reserve(6 * n); S.icov.reserve(6 * n);
    S.sigma.reserve(n); S.qcut.reserve(n); S.sh.reserve((size_t)n * S.ncoef * 3);
    int64_t rej = 0;
    for (int64_t i = 0; i < n; i++) {
        float mu[3], cov[6], icov[6], sg, qc;
        const float* shc = sh + (size_t)i * S.ncoef * 3;
        if (!activate_one(means + 3 * i, quats + 4 * i, log_scales + 3 * i, logits[i], shc, S.ncoef, mu, cov, icov,
                          &sg, &qc)) {
            rej++;
            continue;
        }
        S.mu.insert(S.mu.end(), mu, mu + 3);
        S.cov.insert(S.cov.end(), cov, cov + 6);
        S.icov.insert(S.icov.end(), icov, icov + 6);
        S.sigma.push_back(sg);
        S.qcut.push_back(qc);
        S.sh.insert(S.sh.end(), shc, shc + S.ncoef * 3);
    }
    S.n = n - rej;
    if (n_rejected) *n_rejected = rej;
    return O;
}

void orc_destroy(void* h) { delete (Oracle*)h; }

int64_t orc_num_gaussians(void* h) { return ((Oracle*)h)->sc.n; }

void orc_get_activated(void* h, float* mu, float* cov, float* icov, float* sigma, float* qcut) {
    Scene& S = ((Oracle*)h)->sc;
    std::memcpy(mu, S.mu.data(), 4 * S.mu.size());
    std::memcpy(cov, S.cov.data(), 4 * S.cov.size());
    std::memcpy(icov, S.icov.data(), 4 * S.icov.size());
    std::memcpy(sigma, S.sigma.data(), 4 * S.sigma.size());
    std::memcpy(qcut, S.qcut.data(), 4 * S.qcut.size());
}

int orc_set_mask(void* h, int slot, int w, int hgt, const uint8_t* mask) {
    Scene& S = ((Oracle*)h)->sc;
    if (!mask) { S.masks.erase(slot); S.mask_dims.erase(slot); return 0; }
    S.masks[slot] = std::vector<uint8_t>(mask, mask + (size_t)w * hgt);
    S.mask_dims[slot] = {w, hgt};
    return 0;
}

/* Stages O1-O8 + ranges for all views (instantiate, sort, ranges). */
int orc_prepare(void* h, int n_views, const orc_view* views, const orc_params* p) {
    Oracle& O = *(Oracle*)h;
    O.p = *p;
    if (O.p.assign_tile != 16 && O.p.assign_tile != 32) return 1;
    if (O.p.projection != 0 && O.p.projection != 1) return 4;
    if (O.p.sort_mode < 0 || O.p.sort_mode > 2 || (O.p.sort_mode != 0 && O.p.resort != 0)) return 5;
    O.views.assign(n_views, ViewState());
    O.ntiles = 0;
    for (int v = 0; v < n_views; v++) {
        O.views[v].v = views[v];
        if (views[v].fovea_enabled && O.p.assign_tile != 32) return 2;
        auto md = O.sc.mask_dims.find(views[v].mask_slot);
        if (views[v].mask_slot >= 0 && md != O.sc.mask_dims.end() &&
            (md->second.first != views[v].width || md->second.second != views[v].height))
            return 3;
        setup_view(O, O.views[v]);
        O.views[v].tile_base = O.ntiles;
        O.ntiles += (int64_t)O.views[v].tw * O.views[v].th;
    }
    const int64_t N = O.sc.n;
    // O1-O6 per (view, g), then exact counts
    O.counts.assign((size_t)n_views * N, 0);
    for (int v = 0; v < n_views; v++) {
        ViewState& vs = O.views[v];
        vs.splats.assign(N, Splat());
        int nt = nthreads(O);
        std::vector<std::thread> th;
        for (int t = 0; t < nt; t++)
            th.emplace_back([&, t]() {
                for (int64_t g = t; g < N; g += nt) {
                    preprocess_one(O, vs, g, vs.splats[g]);
                    uint32_t c = 0;
                    for_kept_tiles(O, vs, vs.splats[g], [&](int, int, const float*) { c++; });
                    vs.splats[g].count = c;
                }
            });
        for (auto& x : th) x.join();
        for (int64_t g = 0; g < N; g++) O.counts[(size_t)v * N + g] = vs.splats[g].count;
    }
    // exclusive scan -> instance ranges; duplicate in (view, g, tile row-major) order
    int64_t P = 0;
    for (uint32_t c : O.counts) P += c;
    O.keys_unsorted.assign(P, 0);
    O.vals_unsorted.assign(P, 0);
    int64_t off = 0;
    for (int v = 0; v < n_views; v++) {
        const ViewState& vs = O.views[v];
        for (int64_t g = 0; g < N; g++) {
            for_kept_tiles(O, vs, vs.splats[g], [&](int tx, int ty, const float* dh) {
                uint64_t tile = (uint64_t)(vs.tile_base + (int64_t)ty * vs.tw + tx);
                float td = O.p.sort_mode == 0 ? tile_depth(vs.splats[g], dh, O.p.near_plane)
                                              : global_depth(vs.splats[g], O.p.sort_mode);
                O.keys_unsorted[off] = (tile << 32) | fbits(td);
                O.vals_unsorted[off] = (uint32_t)g;
                off++;
            });
        }
    }
    // global stable sort by key
    std::vector<int64_t> idx(P);
    for (int64_t i = 0; i < P; i++) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(),
                     [&](int64_t a, int64_t b) { return O.keys_unsorted[a] < O.keys_unsorted[b]; });
    O.keys.resize(P);
    O.vals.resize(P);
    for (int64_t i = 0; i < P; i++) { O.keys[i] = O.keys_unsorted[idx[i]]; O.vals[i] = O.vals_unsorted[idx[i]]; }
    // per-tile ranges
    O.ranges.assign(2 * O.ntiles, 0);
    for (int64_t i = 0; i < P; i++) {
        uint64_t t = O.keys[i] >> 32;
        if (i == 0 || (O.keys[i - 1] >> 32) != t) O.ranges[2 * t] = (uint32_t)i;
        if (i == P - 1 || (O.keys[i + 1] >> 32) != t) O.ranges[2 * t + 1] = (uint32_t)(i + 1);
    }
    std::memset(O.stats, 0, sizeof(O.stats));
    O.stats[0] = P;
    for (int v = 0; v < n_views; v++) {
        const ViewState& vs = O.views[v];
        for (int32_t c : vs.cls) O.stats[6 + c]++;
        for (size_t t = 0; t < vs.cls.size(); t++) {
            int ty = (int)(t / vs.tw), tx = (int)(t % vs.tw);
            int c = vs.cls[t];
            if (c == CLS_LOW) O.stats[10] += 1;
            else if (c != CLS_INVIS) {
                int T = O.p.assign_tile;
                if (T == 16) O.stats[10] += 1;
                else
                    for (int sub = 0; sub < 4; sub++)
                        if (tx * T + 16 * (sub & 1) < vs.v.width && ty * T + 16 * (sub >> 1) < vs.v.height)
                            O.stats[10] += 1;
            }
        }
        for (int64_t g = 0; g < N; g++) O.stats[11] += vs.splats[g].count > 0;
    }
    return 0;
}

int64_t orc_num_pairs(void* h) { return (int64_t)((Oracle*)h)->keys.size(); }

void orc_get_counts(void* h, uint32_t* out) {
    Oracle& O = *(Oracle*)h;
    std::memcpy(out, O.counts.data(), 4 * O.counts.size());
}

void orc_get_pairs(void* h, int sorted, uint64_t* keys, uint32_t* vals) {
    Oracle& O = *(Oracle*)h;
    const auto& K = sorted ? O.keys : O.keys_unsorted;
    const auto& V = sorted ? O.vals : O.vals_unsorted;
    std::memcpy(keys, K.data(), 8 * K.size());
    std::memcpy(vals, V.data(), 4 * V.size());
}

int64_t orc_num_tiles(void* h) { return ((Oracle*)h)->ntiles; }

void orc_get_ranges(void* h, uint32_t* out) {
    Oracle& O = *(Oracle*)h;
    std::memcpy(out, O.ranges.data(), 4 * O.ranges.size());
}

int orc_get_tile_info(void* h, int view, int32_t* cls, int32_t* vis) {
    Oracle& O = *(Oracle*)h;
    const ViewState& vs = O.views[view];
    if (cls) std::memcpy(cls, vs.cls.data(), 4 * vs.cls.size());
    if (vis) std::memcpy(vis, vs.vis.data(), 4 * vs.vis.size());
    return vs.tw * 65536 + vs.th;
}

void orc_get_splats(void* h, int view, float* out) {
    Oracle& O = *(Oracle*)h;
    const ViewState& vs = O.views[view];
    for (size_t g = 0; g < vs.splats.size(); g++) {
        const Splat& s = vs.splats[g];
        float* o = out + g * ORC_SPLAT_FLOATS;
        o[0] = (float)s.valid;
        for (int i = 0; i < 3; i++) {
            o[1 + i] = s.muc[i]; o[4 + i] = s.u[i]; o[7 + i] = s.e1[i]; o[10 + i] = s.e2[i];
            o[13 + i] = s.S2[i]; o[16 + i] = s.C[i]; o[31 + i] = s.bv[i]; o[34 + i] = s.rgb[i];
        }
        o[19] = s.eps;
        o[20] = s.m2[0]; o[21] = s.m2[1]; o[22] = s.Cp[0]; o[23] = s.Cp[1]; o[24] = s.Cp[2];
        for (int i = 0; i < 6; i++) o[25 + i] = s.A[i];
        o[37] = s.sigma; o[38] = s.qcut;
        for (int i = 0; i < 4; i++) { o[39 + i] = (float)s.rect[i]; o[43 + i] = s.bbox[i]; }
        o[47] = (float)s.count;
    }
}

/* Full frames for every view (O9-O12).  Phase A renders every sample once
 * (threads over coarse tiles); phase B composes every output pixel. */
int orc_render(void* h, float* rgba, float* depth) {
    Oracle& O = *(Oracle*)h;
    O.stats[1] = O.stats[2] = O.stats[3] = O.stats[4] = O.stats[5] = 0;
    size_t pix_off = 0;
    for (int v = 0; v < (int)O.views.size(); v++) {
        const ViewState& vs = O.views[v];
        const int W = vs.v.width, H = vs.v.height, T = O.p.assign_tile;
        const int We = W + (W & 1), He = H + (H & 1);  // even extents: 2x2 groups at odd borders
        std::vector<Px> full((size_t)We * He), low_((size_t)(We / 2) * (He / 2));
        int nt = nthreads(O);
        std::atomic<int64_t> next(0);
        std::vector<SampleStats> sts(nt);
        std::vector<int64_t> nsamp(nt, 0);
        std::vector<std::thread> th;
        const int64_t ntile = (int64_t)vs.tw * vs.th;
        for (int t = 0; t < nt; t++)
            th.emplace_back([&, t]() {
                for (;;) {
                    int64_t tt = next.fetch_add(1);
                    if (tt >= ntile) break;
                    int ty = (int)(tt / vs.tw), tx = (int)(tt % vs.tw);
                    int c = vs.cls[tt];
                    if (c == CLS_INVIS) continue;
                    int64_t gt = vs.tile_base + tt;
                    int x0 = tx * T, y0 = ty * T;
                    if (O.p.resort == 1) {  // N2: 4x4 sample blocks render together
                        const bool low = c == CLS_LOW;
                        const int span = low ? 8 : 4;
                        for (int by = y0; by < std::min(y0 + T, He); by += span)
                            for (int bx = x0; bx < std::min(x0 + T, We); bx += span) {
                                int bx0, by0;
                                float bxs[16], bys[16], xc, yc, xgc[4], ygc[4];
                                bool valid[16];
                                hier_block(vs, T, low, bx, by, &bx0, &by0, bxs, bys, valid, &xc, &yc, xgc, ygc);
                                Px outs[16];
                                SampleStats bst[16];
                                render_block_hier(O, v, gt, bxs, bys, valid, xc, yc, xgc, ygc, outs, bst);
                                for (int k = 0; k < 16; k++) {
                                    int px = low ? bx0 + 2 * (k & 3) : bx0 + (k & 3);
                                    int py = low ? by0 + 2 * (k >> 2) : by0 + (k >> 2);
                                    if (px >= We || py >= He) continue;
                                    if (low) low_[(size_t)(py / 2) * (We / 2) + px / 2] = outs[k];
                                    else full[(size_t)py * We + px] = outs[k];
                                    if (valid[k]) {
                                        nsamp[t]++;
                                        sts[t].evals += bst[k].evals; sts[t].contribs += bst[k].contribs;
                                        sts[t].overflow += bst[k].overflow; sts[t].term += bst[k].term;
                                    }
                                }
                            }
                        continue;
                    }
                    if (c == CLS_LOW) {
                        for (int gy = 0; 2 * gy < std::min(T, He - y0); gy++)
                            for (int gx = 0; 2 * gx < std::min(T, We - x0); gx++) {
                                bool in = x0 + 2 * gx < W && y0 + 2 * gy < H;
                                SampleStats dummy;
                                low_[(size_t)(y0 / 2 + gy) * (We / 2) + x0 / 2 + gx] =
                                    render_sample(O, v, gt, (float)(x0 + 2 * gx + 1), (float)(y0 + 2 * gy + 1),
                                                  in ? sts[t] : dummy);
                                nsamp[t] += in;
                            }
                    } else {
                        for (int y = y0; y < std::min(y0 + T, He); y++)
                            for (int x = x0; x < std::min(x0 + T, We); x++) {
                                bool in = x < W && y < H;
                                SampleStats dummy;
                                full[(size_t)y * We + x] =
                                    render_sample(O, v, gt, (float)x + 0.5f, (float)y + 0.5f, in ? sts[t] : dummy);
                                nsamp[t] += in;
                            }
                    }
                }
            });
        for (auto& x : th) x.join();
        for (int t = 0; t < nt; t++) {
            O.stats[1] += nsamp[t]; O.stats[2] += sts[t].evals; O.stats[3] += sts[t].contribs;
            O.stats[4] += sts[t].overflow; O.stats[5] += sts[t].term;
        }
        th.clear();
        std::atomic<int> nextrow(0);
        for (int t = 0; t < nt; t++)
            th.emplace_back([&]() {
                FrameCtx F{&O, v, {}, {}, &full, &low_, We};
                for (;;) {
                    int j = nextrow.fetch_add(1);
                    if (j >= H) break;
                    for (int i = 0; i < W; i++) {
                        Px p = pixel_out(F, i, j);
                        size_t k = pix_off + (size_t)j * W + i;
                        rgba[4 * k + 0] = (float)p.r; rgba[4 * k + 1] = (float)p.g;
                        rgba[4 * k + 2] = (float)p.b; rgba[4 * k + 3] = (float)p.a;
                        depth[k] = (float)p.d;
                    }
                }
            });
        for (auto& x : th) x.join();
        pix_off += (size_t)W * H;
    }
    return 0;
}

/* Final output values at listed pixels only (for parity sampling at full
 * sizes); vxy = (view, x, y) triples. */
int orc_render_pixels(void* h, int64_t n, const int32_t* vxy, float* rgba, float* depth) {
    Oracle& O = *(Oracle*)h;
    int nt = nthreads(O);
    std::atomic<int64_t> next(0);
    std::vector<std::thread> th;
    for (int t = 0; t < nt; t++)
        th.emplace_back([&]() {
            for (;;) {
                int64_t k = next.fetch_add(1);
                if (k >= n) break;
                FrameCtx F{&O, vxy[3 * k], {}, {}, nullptr, nullptr, 0};
                Px p = pixel_out(F, vxy[3 * k + 1], vxy[3 * k + 2]);
                rgba[4 * k + 0] = (float)p.r; rgba[4 * k + 1] = (float)p.g;
                rgba[4 * k + 2] = (float)p.b; rgba[4 * k + 3] = (float)p.a;
                depth[k] = (float)p.d;
            }
        });
    for (auto& x : th) x.join();
    return 0;
}

void orc_get_stats(void* h, int64_t* out) { std::memcpy(out, ((Oracle*)h)->stats, sizeof(int64_t) * ORC_STATS); }

/* Brute force (pin P9): every pixel centre, ALL Gaussians with q <= q_cut at
 * that sample (no tiles, no window), full sort by (tau, g), front-to-back
 * blend with the same termination rule. */
int orc_render_bruteforce(void* h, int view, float* rgba, float* depth) {
    Oracle& O = *(Oracle*)h;
    const ViewState& vs = O.views[view];
    const orc_view& v = vs.v;
    const int64_t N = O.sc.n;
    for (int j = 0; j < v.height; j++)
        for (int i = 0; i < v.width; i++) {
            float x = ((float)i + 0.5f - v.cx) / v.fx, y = ((float)j + 0.5f - v.cy) / v.fy;
            double dn = std::sqrt((double)x * x + (double)y * y + 1.0);
            std::vector<WEnt> all;
            for (int64_t g = 0; g < N; g++) {
                const Splat& sp = vs.splats[g];
                if (!sp.valid) continue;
                float den = quad3(sp.A, x, y, 1.0f);
                float dtb = std::fmaf(sp.bv[0], x, std::fmaf(sp.bv[1], y, sp.bv[2]));
                SampleAT at;
                if (O.p.projection == 1) {
                    float q = ewa_q(sp.Cp, ((float)i + 0.5f) - sp.m2[0], ((float)j + 0.5f) - sp.m2[1]);
                    if (!(q <= sp.qcut)) continue;
                    at = sample_alpha_tau_ewa(q, den, dtb, sp.sigma, O.p.near_plane);
                } else {
                    float s = std::fmaf(sp.u[0], x, std::fmaf(sp.u[1], y, sp.u[2]));
                    if (!(s > 0.0f)) continue;
                    float dray[3] = {x, y, 1.0f};
                    float num = chart_num(sp.e1, sp.e2, sp.C, dray);
                    if (!(num <= sp.qcut * (s * s))) continue;
                    at = sample_alpha_tau(num, s * s, den, dtb, sp.sigma, O.p.near_plane);
                }
                all.push_back(WEnt{at.tau, (uint32_t)g, at.alpha});
            }
            if (O.p.sort_mode == 0) {
                std::stable_sort(all.begin(), all.end(), [](const WEnt& a, const WEnt& c) {
                    return a.tau < c.tau || (a.tau == c.tau && a.g < c.g);
                });
            } else {  // global-sort baselines: one depth per Gaussian, ties by g
                std::stable_sort(all.begin(), all.end(), [&](const WEnt& a, const WEnt& c) {
                    float ka = global_depth(vs.splats[a.g], O.p.sort_mode);
                    float kc = global_depth(vs.splats[c.g], O.p.sort_mode);
                    return ka < kc || (ka == kc && a.g < c.g);
                });
            }
            float T = 1.0f;
            double C[3] = {0, 0, 0}, D = 0.0;
            for (const WEnt& w : all) {
                const Splat& sp = vs.splats[w.g];
                double wt = (double)w.alpha * (double)T;
                for (int c = 0; c < 3; c++) C[c] += (double)sp.rgb[c] * wt;
                D += (double)w.tau * dn * wt;
                T = T * (1.0f - w.alpha);
                if (T < 1e-4f) break;
            }
            size_t k = (size_t)j * v.width + i;
            rgba[4 * k + 0] = (float)(C[0] + (double)T * O.p.background[0]);
            rgba[4 * k + 1] = (float)(C[1] + (double)T * O.p.background[1]);
            rgba[4 * k + 2] = (float)(C[2] + (double)T * O.p.background[2]);
            rgba[4 * k + 3] = (float)(1.0 - (double)T);
            depth[k] = (float)D;
        }
    return 0;
}

int orc_tile_test(void* h, int view, int64_t g, int x0, int y0, int x1, int y1, float* out) {
    Oracle& O = *(Oracle*)h;
    const ViewState& vs = O.views[view];
    const Splat& sp = vs.splats[g];
    if (!sp.valid) { out[0] = -1.0f; return 0; }
    float qmin = 0.0f, dh[3] = {0, 0, 0};
    bool keep = (O.p.projection == 1) ? tile_test_ewa(sp, vs.v, x0, y0, x1, y1, &qmin, dh)
                                       : tile_test(sp, vs.v, x0, y0, x1, y1, &qmin, dh);
    out[0] = keep ? 1.0f : 0.0f;
    out[1] = qmin;
    out[2] = tile_depth(sp, dh, O.p.near_plane);
    out[3] = dh[0]; out[4] = dh[1]; out[5] = dh[2];
    return 0;
}

void orc_sat(int tw, int th, const uint8_t* bits, uint32_t* sat) {
    const int S = tw + 1;
    for (int i = 0; i < S; i++) sat[i] = 0;
    for (int y = 0; y < th; y++) {
        sat[(size_t)(y + 1) * S] = 0;
        for (int x = 0; x < tw; x++)
            sat[(size_t)(y + 1) * S + x + 1] = sat[(size_t)y * S + x + 1] + sat[(size_t)(y + 1) * S + x] -
                                               sat[(size_t)y * S + x] + (bits[(size_t)y * tw + x] ? 1u : 0u);
    }
}

int64_t orc_sat_count(int tw, const uint32_t* sat, int x0, int y0, int x1, int y1) {
    const int S = tw + 1;
    if (x0 > x1 || y0 > y1) return 0;
    return (int64_t)sat[(size_t)(y1 + 1) * S + x1 + 1] - sat[(size_t)y0 * S + x1 + 1] - sat[(size_t)(y1 + 1) * S + x0] +
           sat[(size_t)y0 * S + x0];
}

/* Eq.4 for one edge p + t d, chart-origin mean, conic C; clamped t. */
float orc_eq4_edge(const float* C, const float* p, const float* d, float* xhat) {
    float cdx = std::fmaf(C[0], d[0], C[1] * d[1]), cdy = std::fmaf(C[1], d[0], C[2] * d[1]);
    float den = std::fmaf(d[0], cdx, d[1] * cdy);
    float nmr = -std::fmaf(p[0], cdx, p[1] * cdy);
    float t;
    if (nmr <= 0.0f || !(den > 0.0f)) t = 0.0f;
    else if (nmr >= den) t = 1.0f;
    else t = nmr / den;
    xhat[0] = std::fmaf(t, d[0], p[0]);
    xhat[1] = std::fmaf(t, d[1], p[1]);
    float cX = std::fmaf(C[0], xhat[0], C[1] * xhat[1]), cY = std::fmaf(C[1], xhat[0], C[2] * xhat[1]);
    return std::fmaf(xhat[0], cX, xhat[1] * cY);
}

/* N4 hook (test infrastructure): the blend order of every pixel of a
 * full-rate (non-foveated) view -- the Gaussians each pixel blended, front to
 * back, as O10-O11 decide them.  counts[W*H]; seq gets the concatenated lists
 * (up to cap entries); returns the total length (or -1 for a foveated view). */
int64_t orc_blend_orders(void* h, int view, int32_t* counts, uint32_t* seq, int64_t cap) {
    Oracle& O = *(Oracle*)h;
    const ViewState& vs = O.views[view];
    if (vs.v.fovea_enabled) return -1;
    const int W = vs.v.width, H = vs.v.height, T = O.p.assign_tile;
    int64_t tot = 0;
    for (int j = 0; j < H; j++)
        for (int i = 0; i < W; i++) {
            if (vs.cls[(size_t)(j / T) * vs.tw + (i / T)] == CLS_INVIS) {
                counts[(size_t)j * W + i] = 0;
                continue;
            }
            const int64_t gt = vs.tile_base + (int64_t)(j / T) * vs.tw + (i / T);
            std::vector<uint32_t> order;
            SampleStats st;
            render_sample(O, view, gt, (float)i + 0.5f, (float)j + 0.5f, st, &order);
            counts[(size_t)j * W + i] = (int32_t)order.size();
            for (uint32_t g : order) {
                if (tot < cap) seq[tot] = g;
                tot++;
            }
        }
    return tot;
}

/* Pin H3 hook: the N2 queue mechanics on a given stream of n block entries
 * (tauB[n], tauG[n*4], g[n], member[n], tau[n*16], alpha[n*16], rgb[n*3]); all 16
 * samples in the image, |d| = 1; out = 16 x (r, g, b, a, depth). */
int orc_hier_core(int64_t n, int kb, int kg, int kp, const float* tauB, const float* tauG, const uint32_t* g,
                  const uint32_t* member, const float* tau, const float* alpha, const float* rgb, double* out,
                  int64_t* stats) {
    std::vector<HIn> in((size_t)n);
    for (int64_t i = 0; i < n; i++) {
        in[i].tauB = tauB[i];
        for (int q = 0; q < 4; q++) in[i].tauG[q] = tauG[4 * i + q];
        in[i].g = g[i];
        in[i].member = member[i];
        for (int s = 0; s < 16; s++) {
            in[i].tau[s] = tau[16 * i + s];
            in[i].alpha[s] = alpha[16 * i + s];
        }
        for (int c = 0; c < 3; c++) in[i].rgb[c] = rgb[3 * i + c];
    }
    bool valid[16];
    double dn[16];
    for (int s = 0; s < 16; s++) { valid[s] = true; dn[s] = 1.0; }
    const float bg[3] = {0.0f, 0.0f, 0.0f};
    Px px[16];
    SampleStats st[16];
    hier_core(in, kb, kg, kp, valid, dn, bg, px, st);
    for (int s = 0; s < 16; s++) {
        out[5 * s + 0] = px[s].r; out[5 * s + 1] = px[s].g; out[5 * s + 2] = px[s].b;
        out[5 * s + 3] = px[s].a; out[5 * s + 4] = px[s].d;
        stats[4 * s + 0] = st[s].evals; stats[4 * s + 1] = st[s].contribs;
        stats[4 * s + 2] = st[s].overflow; stats[4 * s + 3] = st[s].term;
    }
    return 0;
}

/* Per-sample depth tau (O10) of Gaussian g at image point (x, y) (pixel
 * coordinates), for the ray-march pin P5. */
/* Pin hook: the contract's per-sample alpha and tau (DESIGN R9) on given inputs. */
void orc_sample_alpha_tau(int64_t n, const float* num, const float* ss, const float* den, const float* dtb,
                          const float* sigma, float near_plane, float* alpha, float* tau) {
    for (int64_t i = 0; i < n; i++) {
        SampleAT at = sample_alpha_tau(num[i], ss[i], den[i], dtb[i], sigma[i], near_plane);
        alpha[i] = at.alpha;
        tau[i] = at.tau;
    }
}

float orc_sample_depth(void* h, int view, int64_t g, float xs, float ys) {
    Oracle& O = *(Oracle*)h;
    const ViewState& vs = O.views[view];
    const Splat& sp = vs.splats[g];
    float x = (xs - vs.v.cx) / vs.v.fx, y = (ys - vs.v.cy) / vs.v.fy;
    float den = quad3(sp.A, x, y, 1.0f);
    float dtb = std::fmaf(sp.bv[0], x, std::fmaf(sp.bv[1], y, sp.bv[2]));
    float s = std::fmaf(sp.u[0], x, std::fmaf(sp.u[1], y, sp.u[2]));
    float d[3] = {x, y, 1.0f};
    return sample_alpha_tau(chart_num(sp.e1, sp.e2, sp.C, d), s * s, den, dtb, sp.sigma, O.p.near_plane).tau;
}

}  // extern "C"
