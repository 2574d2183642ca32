// hierarchical resort mode of the single foveated blend launch
// (StopThePop's "hierarchical per-pixel resorting", with the
// hierarchical culling of P:431), selected by vrs_set_resort_mode(ctx, 1).
//
// The items, samples, staging and warp-block culling are those of k_blend
// (k_blend.cu).  The 16 samples of each 4x4 sample block (one half-warp:
// lanes with (lane >> 2) & 1 equal) stream their tile list together:
//   admission  an entry enters the block queue iff a not-terminated in-image
//              sample of the block passes the per-sample membership test
//              (R3, as O10); the set of such samples (a lane mask) goes with it;
//   queue      K_B = 8 entries ordered by (tau_B, g), tau_B = max(dtb/den, near)
//              on the block-centre ray (one IEEE division, R4 form), held in
//              registers: lane k of the half-warp holds entry k, so insertion
//              and removal are one ballot + shuffles; the entries' splat
//              records are copied to a per-block shared-memory cache
//              (K_B + 1 slots) because they outlive their staging batch;
//   release    when the queue exceeds K_B its minimum is released: each of its
//              samples that has not terminated computes alpha and tau (R9) and
//              inserts into its own window of K_P = 8 (the k_blend ring), where
//              overflow pops and blends the minimum (O10-O11);
//   drain      at stream end the queue releases in order, then the windows drain.
// The oracle's render_block_hier / hier_core (oracle/oracle.cpp) is the
// specification; parity is bit-exact in every decision (membership, orders,
// T < 1e-4 stops) and within tolerance in colour and depth.
#include "k_blend_common.cuh"

namespace vrs {

namespace {

constexpr int kHT = 256;          // threads per block: one 16x16 item
constexpr int kHW = kHT / 32;
constexpr int kHBatch = 80;       // staged records per batch
constexpr int kHP = kHierWindow;  // per-sample window K_P
constexpr int kHB = kHierQueue;   // block queue K_B (+1 slot for the incoming entry)
constexpr int kHG = kHierGroup;   // 2x2 group queue K_G (the 4 lanes of a group hold one entry each)
static_assert(kHG <= 4, "the group queue lives in the 4 lanes of a 2x2 group");
static_assert(kHB + 1 <= 16, "the block queue lives in the 16 lanes of a half-warp");
static_assert((kHP & (kHP - 1)) == 0, "ring needs a power-of-two window");

struct HierSmem {
    float4 r[6][kHBatch];        // staged records (k_blend layout r0..r5)
    uint32_t mask[kHBatch];
    float4 wblock[kHW];
    float4 cache[2 * kHW][kHB + 1][6];  // per 4x4 block: records of queued entries
    unsigned long long w_key[kHP][kHT];
    float w_a[kHP][kHT];
    unsigned long long cnt[4];
};

constexpr uint32_t kHSlot = kHT * 8;
constexpr uint32_t kHRing = kHP * kHSlot - 1u;  // wraps the slot bits, keeps the column bits

}  // namespace

#ifndef VRS_HIER_MINB
#define VRS_HIER_MINB 4
#endif
template <bool kCounters>
__global__ void __launch_bounds__(kHT, VRS_HIER_MINB) k_blend_hier(FrameParams fp, FrameBufs fb, float* __restrict__ rgba,
                                                      float* __restrict__ depth) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    HierSmem& S = *reinterpret_cast<HierSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int vi = 0;
    const int item = blockIdx.x;
    while (vi + 1 < fp.n_views && item >= fp.v[vi + 1].item_off) vi++;
    const ViewParams& v = fp.v[vi];
    const uint32_t it = v.items[item - v.item_off];
    const int tile = (int)(it & 0xfffffu), sub = (int)((it >> 20) & 3u), kind = (int)(it >> 22);
    const int T = fp.T;
    const int tx = tile % v.tw, ty = tile / v.tw;
    const int x0 = tx * T, y0 = ty * T;
    const int lx = lane & 7, ly = lane >> 3, wx = (warp & 1) * 8, wy = (warp >> 1) * 4;
    const int sx = wx + lx, sy = wy + ly;
    // 4x4 block of this lane: half-warp hb, queue index kq inside it
    const int hb = (lane >> 2) & 1, kq = ly * 4 + (lane & 3), blk = warp * 2 + hb;
    const unsigned hmask = 0x0F0F0F0Fu << (4 * hb);
    auto lane_of = [&](int k) { return (k >> 2) * 8 + hb * 4 + (k & 3); };
    const bool low = kind == kItemLow;
    const int ox = low ? x0 : x0 + (T == 32 ? 16 * (sub & 1) : 0);
    const int oy = low ? y0 : y0 + (T == 32 ? 16 * (sub >> 1) : 0);
    int px, py;
    float xs, ys, xc, yc;  // sample point; block centre (mean of its 16 sample points)
    if (low) {
        px = x0 + 2 * sx;
        py = y0 + 2 * sy;
        xs = (float)(px + 1);
        ys = (float)(py + 1);
        xc = (float)(x0 + 2 * (wx + 4 * hb) + 4);
        yc = (float)(y0 + 2 * wy + 4);
    } else {
        px = ox + sx;
        py = oy + sy;
        xs = (float)px + 0.5f;
        ys = (float)py + 0.5f;
        xc = (float)(ox + wx + 4 * hb + 2);
        yc = (float)(oy + wy + 2);
    }
    const bool in_img = px < v.W && py < v.H;
    // 2x2 group of this lane (lanes l0, l0|1, l0|8, l0|9), its rank inside it and its centre
    const int grk = ((lane >> 3) & 1) * 2 + (lane & 1);
    const unsigned glanes = 0x303u << (lane & ~9);
    auto lane_of_g = [&](int r) { return (lane & ~9) | (r & 1) | ((r >> 1) << 3); };
    float xgc, ygc;
    if (low) {
        xgc = (float)(x0 + 2 * (wx + 4 * hb) + 4 * ((lane & 3) >> 1) + 2);
        ygc = (float)(y0 + 2 * wy + 4 * (ly >> 1) + 2);
    } else {
        xgc = (float)(ox + wx + 4 * hb + 2 * ((lane & 3) >> 1) + 1);
        ygc = (float)(oy + wy + 2 * (ly >> 1) + 1);
    }
    if (tid < kHW) {
        const int wwx = (tid & 1) * 8, wwy = (tid >> 1) * 4;
        float4 b;
        if (low)  // centre, half-extent of the warp's samples (k_blend layout)
            b = make_float4((float)(x0 + 2 * wwx + 8), (float)(y0 + 2 * wwy + 4), 7.0f, 3.0f);
        else
            b = make_float4((float)(ox + wwx + 4), (float)(oy + wwy + 2), 3.5f, 1.5f);
        S.wblock[tid] = b;
    }
    if (kCounters && tid < 4) S.cnt[tid] = 0ull;
    const float x = (xs - v.cx) / v.fx;
    const float y = (ys - v.cy) / v.fy;
    const float xB = (xc - v.cx) / v.fx;
    const float yB = (yc - v.cy) / v.fy;
    const float xG = (xgc - v.cx) / v.fx;
    const float yG = (ygc - v.cy) / v.fy;
    const float dn = sqrtf(fmaf(x, x, fmaf(y, y, 1.0f)));
    const uint32_t rb = fb.ranges[2 * (size_t)(v.tile_base + tile)];
    const uint32_t re = fb.ranges[2 * (size_t)(v.tile_base + tile) + 1];
    const float4* __restrict__ recv = fb.rec + (size_t)vi * fp.N * kRecF4;
    const float4* __restrict__ colv = fb.col + (size_t)vi * fp.N;
    // ring offsets carry the thread's column (tid * 8), so window addresses are the
    // arrays' block-uniform bases plus one offset (k_blend.cu)
    char* const wkb = reinterpret_cast<char*>(&S.w_key[0][0]);
    char* const wab = reinterpret_cast<char*>(&S.w_a[0][0]);
#define WK(off) (*reinterpret_cast<unsigned long long*>(wkb + (off)))
#define WA(off) (*reinterpret_cast<float*>(wab + ((off) >> 1)))
#pragma unroll
    for (int k = 0; k < kHP; k++) {
        WK(k * kHSlot + 8u * tid) = kSentinelKey;
        WA(k * kHSlot + 8u * tid) = 0.0f;
    }
    float Tr = 1.0f, Cr = 0.0f, Cg = 0.0f, Cb = 0.0f, Dd = 0.0f;
    bool done = !in_img;  // samples outside the image take no part (oracle: valid[s])
    uint32_t hk = 8u * tid;  // ring head: slot * slot bytes + the thread's column
    uint32_t n_contrib = 0, stop_pos = re - 1;
    // block queue: this lane's entry kq (valid when kq < qn), count and free cache slot (uniform per half)
    unsigned long long qkey = ~0ull;
    uint32_t qmask = 0, qslot = 0;
    int qn = 0, fslot = 0;
    // group queue: this lane's entry grk (valid when grk < gn), count (uniform per group)
    unsigned long long gkey = ~0ull;
    uint32_t gmask = 0;
    int gn = 0;

    auto blend_one = [&](unsigned long long key, float a) {
        const float4* cp;
        asm("mad.wide.u32 %0, %1, 16, %2;" : "=l"(cp) : "r"((uint32_t)key), "l"(colv));
        const float4 col = __ldg(cp);
        const float wgt = a * Tr;
        Cr = fmaf(col.x, wgt, Cr);
        Cg = fmaf(col.y, wgt, Cg);
        Cb = fmaf(col.z, wgt, Cb);
        Dd = fmaf(key_tau(key), wgt, Dd);
        Tr = Tr * (1.0f - a);
        done = Tr < kTmin;
    };
    // per-sample window (K_P ring, sentinel-prefilled; k_blend's insertion)
    auto contribute = [&](const unsigned long long key, const float alpha, const uint32_t pos) {
        if (kCounters) n_contrib++;
        const unsigned long long kh = WK(hk);
        const bool direct = key < kh;
        const float ah = WA(hk);
        blend_one(direct ? key : kh, direct ? alpha : ah);
        if (kCounters && done) stop_pos = pos;
        if (direct || done) return;
        hk = (hk + kHSlot) & kHRing;
        uint32_t jo = (hk + (kHP - 2) * kHSlot) & kHRing;
        uint32_t dst = (jo + kHSlot) & kHRing;
        unsigned long long kj = WK(jo);
        int left = kHP - 1;
#pragma unroll 1
        while (kj > key) {
            WK(dst) = kj;
            WA(dst) = WA(jo);
            dst = jo;
            if (--left == 0) break;
            jo = (jo - kHSlot) & kHRing;
            kj = WK(jo);
        }
        WK(dst) = key;
        WA(dst) = alpha;
    };
    // release of a queued entry to this lane's sample (record from the block cache)
    auto release = [&](const int slot, const uint32_t pos) {
        const float4* rc = S.cache[blk][slot];
        const float4 a0 = rc[0], a1 = rc[1], a2 = rc[2];
        const float s = fmaf(a0.x, x, fmaf(a0.y, y, a0.z));
        const float ex = fmaf(a1.x, x, a1.y);
        const float ey = fmaf(a1.z, x, fmaf(a1.w, y, a2.x));
        const float cx = fmaf(a2.y, ex, a2.z * ey), cy = fmaf(a2.z, ex, a2.w * ey);
        const float num = fmaf(ex, cx, ey * cy);
        const float ss = s * s;
        const float4 a3 = rc[3], a4 = rc[4], t5 = rc[5];
        const float den = quad3z1(a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, x, y);
        const float dtb = fmaf(a4.z, x, fmaf(a4.w, y, t5.x));
        float tau;
        const float alpha = alpha_tau(num, ss, den, dtb, t5.y, tau);
        contribute(order_key(tau, __float_as_uint(t5.z), fp.near_plane), alpha, pos);
    };
    // release of entry g to this lane's sample with the record read from global memory
    // (a group-queue entry outlives its block-queue cache slot)
    auto release_global = [&](const uint32_t g, const uint32_t pos) {
        const float4* rp = recv + (size_t)g * kRecF4;
        const float4 a0 = __ldg(rp + 0), a1 = __ldg(rp + 1), a2 = __ldg(rp + 2);
        const float s = fmaf(a0.x, x, fmaf(a0.y, y, a0.z));
        const float ex = fmaf(a1.x, x, a1.y);
        const float ey = fmaf(a1.z, x, fmaf(a1.w, y, a2.x));
        const float cx = fmaf(a2.y, ex, a2.z * ey), cy = fmaf(a2.z, ex, a2.w * ey);
        const float num = fmaf(ex, cx, ey * cy);
        const float ss = s * s;
        const float4 a3 = __ldg(rp + 3), a4 = __ldg(rp + 4), t5 = __ldg(rp + 5);
        const float den = quad3z1(a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, x, y);
        const float dtb = fmaf(a4.z, x, fmaf(a4.w, y, t5.x));
        float tau;
        const float alpha = alpha_tau(num, ss, den, dtb, t5.y, tau);
        contribute(order_key(tau, g, fp.near_plane), alpha, pos);
    };
    // the 2x2 group level: a block release (key ek, member lanes em, cache slot es; valid per
    // half) enters the queue of every group with a not-terminated member, ordered by the
    // group-centre depth; a full group queue releases its minimum (possibly the new entry)
    auto group_stage = [&](const bool valid, const unsigned long long ek, const uint32_t em, const int es,
                           const uint32_t pos) {
        const unsigned notdone = __ballot_sync(0xffffffffu, !done);
        const uint32_t gm = valid ? (em & glanes & notdone) : 0u;
        const bool ins = gm != 0u;
        if (!__any_sync(0xffffffffu, ins)) return;
        unsigned long long kg = ~0ull;
        if (ins) {  // tau_G (R4 form, one IEEE division) from the entry's cached record
            const float4* rc = S.cache[blk][es];
            const float4 a3 = rc[3], a4 = rc[4], t5 = rc[5];
            const float denG = quad3z1(a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, xG, yG);
            const float dtbG = fmaf(a4.z, xG, fmaf(a4.w, yG, t5.x));
            const float tauG = fmaxf(__fdiv_rn(dtbG, denG), fp.near_plane);
            kg = ((unsigned long long)__float_as_uint(tauG) << 32) | (uint32_t)ek;
        }
        const int pg = __popc(__ballot_sync(0xffffffffu, grk < gn && gkey < kg) & glanes);
        const int su = lane_of_g(grk > 0 ? grk - 1 : 0), sd = lane_of_g(grk < 3 ? grk + 1 : 3);
        const unsigned long long ku = __shfl_sync(0xffffffffu, gkey, su), kd = __shfl_sync(0xffffffffu, gkey, sd),
                                 k0 = __shfl_sync(0xffffffffu, gkey, lane_of_g(0));
        const uint32_t mu = __shfl_sync(0xffffffffu, gmask, su), md = __shfl_sync(0xffffffffu, gmask, sd),
                       m0 = __shfl_sync(0xffffffffu, gmask, lane_of_g(0));
        unsigned long long rk = 0;
        uint32_t rm = 0;
        if (ins) {
            if (gn < kHG) {  // room: insert at pg
                if (grk > pg) {
                    gkey = ku;
                    gmask = mu;
                } else if (grk == pg) {
                    gkey = kg;
                    gmask = gm;
                }
                gn++;
            } else if (pg == 0) {  // full, the new entry is the minimum: released at once
                rk = kg;
                rm = gm;
            } else {  // full: release the minimum, the new entry takes rank pg - 1
                rk = k0;
                rm = m0;
                if (grk < pg - 1) {
                    gkey = kd;
                    gmask = md;
                } else if (grk == pg - 1) {
                    gkey = kg;
                    gmask = gm;
                }
            }
        }
        if (((rm >> lane) & 1u) && !done) release_global((uint32_t)rk, pos);
        __syncwarp();
    };
    // pop the minimum of each half whose flag is set; release it to its samples
    auto pop_release = [&](const bool pop, const uint32_t pos) {
        const unsigned long long ek = __shfl_sync(0xffffffffu, qkey, lane_of(0));
        const uint32_t em = __shfl_sync(0xffffffffu, qmask, lane_of(0));
        const int es = __shfl_sync(0xffffffffu, (int)qslot, lane_of(0));
        const int up = lane_of(kq < 15 ? kq + 1 : 15);
        const unsigned long long nk = __shfl_sync(0xffffffffu, qkey, up);
        const uint32_t nm = __shfl_sync(0xffffffffu, qmask, up);
        const uint32_t ns = __shfl_sync(0xffffffffu, qslot, up);
        if (pop) {
            qkey = (kq + 1 < qn) ? nk : ~0ull;
            qmask = nm;
            qslot = ns;
            qn--;
            fslot = es;
        }
        if (kHG == 0) {
            if (pop && ((em >> lane) & 1u) && !done) release(es, pos);
        } else {
            group_stage(pop, ek, em, es, pos);
        }
    };

    for (uint32_t base = rb; base < re; base += kHBatch) {
        __syncthreads();
        const uint32_t idx = base + tid;
        if (tid < kHBatch && idx < re) {
            uint32_t g = __ldg(fb.vals + idx);
            g = (g < (uint32_t)fp.N) ? g : 0u;
            const float4* rp = recv + (size_t)g * kRecF4;
            const float4 a5 = __ldg(rp + 5), a7 = __ldg(rp + 7);
            S.r[0][tid] = __ldg(rp + 0);
            S.r[1][tid] = __ldg(rp + 1);
            S.r[2][tid] = __ldg(rp + 2);
            S.r[3][tid] = __ldg(rp + 3);
            S.r[4][tid] = __ldg(rp + 4);
            S.r[5][tid] = make_float4(a5.x, a5.y, __uint_as_float(g), 0.0f);
            const uint32_t m = footprint_mask<kHW>(a7, S.wblock);
            S.mask[tid] = fp.no_cull ? 0xffu : m;
        }
        if (__syncthreads_count(!done) == 0) break;
        const int nb = min((int)(re - base), kHBatch);
        for (int c = 0; c < nb; c += 32) {
            if (__all_sync(0xffffffffu, done)) break;
            const bool rel = (c + lane < nb) && ((S.mask[c + lane] >> warp) & 1u);
            unsigned bits = __ballot_sync(0xffffffffu, rel);
            while (bits) {
                const int j = c + __ffs(bits) - 1;
                bits &= bits - 1;
                // admission: per-sample membership (R3), ballot per half
                const float4 a0 = S.r[0][j], a1 = S.r[1][j], a2 = S.r[2][j];
                const float s = fmaf(a0.x, x, fmaf(a0.y, y, a0.z));
                const float ex = fmaf(a1.x, x, a1.y);
                const float ey = fmaf(a1.z, x, fmaf(a1.w, y, a2.x));
                const float cx = fmaf(a2.y, ex, a2.z * ey), cy = fmaf(a2.z, ex, a2.w * ey);
                const float num = fmaf(ex, cx, ey * cy);
                const bool m = !done && (s > 0.0f) && (num <= a0.w * (s * s));
                const unsigned mb = __ballot_sync(0xffffffffu, m) & hmask;
                const bool admit = mb != 0u;
                if (!__any_sync(0xffffffffu, admit)) continue;
                // block-centre depth tau_B and the new key
                const float4 a3 = S.r[3][j], a4 = S.r[4][j], t5 = S.r[5][j];
                const float denB = quad3z1(a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, xB, yB);
                const float dtbB = fmaf(a4.z, xB, fmaf(a4.w, yB, t5.x));
                const float tauB = fmaxf(__fdiv_rn(dtbB, denB), fp.near_plane);
                const unsigned long long nkey =
                    ((unsigned long long)__float_as_uint(tauB) << 32) | __float_as_uint(t5.z);
                const int pos = __popc(__ballot_sync(0xffffffffu, kq < qn && qkey < nkey) & hmask);
                if (admit && kq < 6) S.cache[blk][fslot][kq] = S.r[kq][j];
                const int dn_src = lane_of(kq > 0 ? kq - 1 : 0);
                const unsigned long long pk = __shfl_sync(0xffffffffu, qkey, dn_src);
                const uint32_t pm = __shfl_sync(0xffffffffu, qmask, dn_src);
                const uint32_t ps = __shfl_sync(0xffffffffu, qslot, dn_src);
                if (admit) {
                    if (kq > pos) {
                        qkey = pk;
                        qmask = pm;
                        qslot = ps;
                    } else if (kq == pos) {
                        qkey = nkey;
                        qmask = mb;
                        qslot = (uint32_t)fslot;
                    }
                    qn++;
                    fslot = qn;  // before the first pop, slots are taken in order
                }
                __syncwarp();
                const bool pop = admit && qn > kHB;
                if (__any_sync(0xffffffffu, pop)) pop_release(pop, base + (uint32_t)j);
                __syncwarp();  // the released slot's cache reads precede its reuse (memory order, not just execution)
            }
        }
    }
    // stream end: the queues release in order, then the windows drain
    while (__any_sync(0xffffffffu, qn > 0)) pop_release(qn > 0, re - 1);
    // then the group queues release in order
    while (__any_sync(0xffffffffu, gn > 0)) {
        const bool has = gn > 0;
        const unsigned long long k0 = __shfl_sync(0xffffffffu, gkey, lane_of_g(0));
        const uint32_t m0 = __shfl_sync(0xffffffffu, gmask, lane_of_g(0));
        const int sd = lane_of_g(grk < 3 ? grk + 1 : 3);
        const unsigned long long kd = __shfl_sync(0xffffffffu, gkey, sd);
        const uint32_t md = __shfl_sync(0xffffffffu, gmask, sd);
        if (has) {
            gkey = (grk + 1 < gn) ? kd : ~0ull;
            gmask = md;
            gn--;
            if (((m0 >> lane) & 1u) && !done) release_global((uint32_t)k0, re - 1);
        }
        __syncwarp();
    }
#pragma unroll 1
    for (int k = 0; k < kHP && !done; k++) {
        blend_one(WK(hk), WA(hk));
        hk = (hk + kHSlot) & kHRing;
    }
#undef WK
#undef WA
    Dd = Dd * dn;
    const float oR = Cr + Tr * fp.bg[0], oG = Cg + Tr * fp.bg[1], oB = Cb + Tr * fp.bg[2], oA = 1.0f - Tr;
    if (low) {
        if (in_img) {
            const size_t li = (size_t)v.low_off + (size_t)(py >> 1) * v.low_w + (px >> 1);
            fb.low_rgba[li] = make_float4(oR, oG, oB, oA);
            fb.low_depth[li] = Dd;
        }
    } else if (kind == kItemHybrid) {
        const int l0 = lane & ~9;
        float vals[5] = {oR, oG, oB, oA, Dd};
        float outv[5];
        const float wgt = fovea_weight(v, (float)px + 0.5f, (float)py + 0.5f);
#pragma unroll
        for (int c = 0; c < 5; c++) {
            const float p00 = __shfl_sync(0xffffffffu, vals[c], l0);
            const float p01 = __shfl_sync(0xffffffffu, vals[c], l0 | 1);
            const float p10 = __shfl_sync(0xffffffffu, vals[c], l0 | 8);
            const float p11 = __shfl_sync(0xffffffffu, vals[c], l0 | 9);
            const float avg = ((p00 + p01) + (p10 + p11)) * 0.25f;
            outv[c] = fmaf(wgt, vals[c] - avg, avg);
        }
        if (in_img) {
            const size_t pi = (size_t)v.pix_off + (size_t)py * v.W + px;
            store_pixel(fp.out_fmt, rgba, depth, pi, make_float4(outv[0], outv[1], outv[2], outv[3]), outv[4]);
        }
    } else if (in_img) {
        const size_t pi = (size_t)v.pix_off + (size_t)py * v.W + px;
        store_pixel(fp.out_fmt, rgba, depth, pi, make_float4(oR, oG, oB, oA), Dd);
    }
    if (kCounters) {
        const unsigned long long ev = in_img ? (unsigned long long)(stop_pos - rb + 1) : 0ull;
        const bool overflowed = n_contrib > (uint32_t)kHP;
        unsigned long long c0 = rb < re ? ev : 0ull, c1 = in_img ? n_contrib : 0u,
                           c2 = (in_img && overflowed) ? 1u : 0u, c3 = (in_img && done) ? 1u : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            c0 += __shfl_xor_sync(0xffffffffu, c0, o);
            c1 += __shfl_xor_sync(0xffffffffu, c1, o);
            c2 += __shfl_xor_sync(0xffffffffu, c2, o);
            c3 += __shfl_xor_sync(0xffffffffu, c3, o);
        }
        __syncthreads();
        if (lane == 0) {
            atomicAdd(&S.cnt[0], c0);
            atomicAdd(&S.cnt[1], c1);
            atomicAdd(&S.cnt[2], c2);
            atomicAdd(&S.cnt[3], c3);
        }
        __syncthreads();
        if (tid == 0) {
            atomicAdd(&fb.stats[0], S.cnt[0]);
            atomicAdd(&fb.stats[1], S.cnt[1]);
            atomicAdd(&fb.stats[2], S.cnt[2]);
            atomicAdd(&fb.stats[3], S.cnt[3]);
        }
    }
}

void launch_blend_hier(const FrameParams& fp, FrameBufs fb, int total_items, float* rgba, float* depth,
                       cudaStream_t st) {
    if (total_items <= 0) return;
    const size_t smem = sizeof(HierSmem);
    ensure_smem_attr((const void*)k_blend_hier<true>, (int)smem);
    ensure_smem_attr((const void*)k_blend_hier<false>, (int)smem);
    if (fp.counters) k_blend_hier<true><<<(unsigned)total_items, kHT, smem, st>>>(fp, fb, rgba, depth);
    else k_blend_hier<false><<<(unsigned)total_items, kHT, smem, st>>>(fp, fb, rgba, depth);
}

}  // namespace vrs
