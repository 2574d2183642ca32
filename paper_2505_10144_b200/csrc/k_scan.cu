// Step 2: exclusive prefix sum of the per-(view, Gaussian) pair
// counts -> each Gaussian's instance range in the global sort buffer (P:446
// "compute the range of each Gaussian's instances inside this buffer").
// Single pass, decoupled look-back: each 4096-element tile publishes its
// aggregate, then its inclusive prefix, in one 64-bit status word.
#include <algorithm>

#include "vrs_internal.cuh"

namespace vrs {

namespace {
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kFlagAgg = 1ull << 32, kFlagPre = 2ull << 32;

// Status words are self-contained (flag + value): relaxed GPU-scope
// accesses suffice and avoid the L1 invalidation an acquire load implies.
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
}  // namespace

// scratch[0] low word: tile counter; scratch[1 + t]: status of tile t.
// Persistent: blocks take tiles in order from the counter until n (read on the
// device, so the scanned length need not be known on the host) is covered.
__global__ void __launch_bounds__(kScanThreads) k_scan(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                       uint32_t* total, const uint32_t* __restrict__ n_dev,
                                                       int64_t cap, unsigned long long* scratch,
                                                       unsigned long long* __restrict__ expand, int64_t expand_cap) {
    __shared__ uint32_t s_tile, s_excl;
    __shared__ uint32_t s_warp[kScanThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = n_dev ? min((int64_t)*n_dev, cap) : cap;
    const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
    if (n == 0) {
        if (blockIdx.x == 0 && tid == 0) *total = 0;
        return;
    }
    unsigned long long* status = scratch + 1;
    while (true) {
        if (tid == 0) s_tile = atomicAdd(reinterpret_cast<unsigned int*>(scratch), 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if ((int64_t)tile >= ntiles) break;
        const int64_t base = (int64_t)tile * kScanTile + (int64_t)tid * kScanItems;
        uint32_t v[kScanItems];
        if (base + kScanItems <= n && ((reinterpret_cast<uintptr_t>(in + base) & 15) == 0)) {
            const uint4* p = reinterpret_cast<const uint4*>(in + base);
#pragma unroll
            for (int k = 0; k < kScanItems / 4; k++) {
                uint4 q = __ldcs(p + k);
                v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < kScanItems; k++) v[k] = (base + k < n) ? in[base + k] : 0u;
        }
        uint32_t tsum = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; k++) tsum += v[k];
        uint32_t inc = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        uint32_t wpre = 0, agg = 0;
#pragma unroll
        for (int w = 0; w < kScanThreads / 32; w++) {
            if (w < warp) wpre += s_warp[w];
            agg += s_warp[w];
        }
        if (warp == 0) {
            uint32_t excl = 0;
            if (tile == 0) {
                if (lane == 0) st_release(&status[0], kFlagPre | agg);
            } else {
                if (lane == 0) st_release(&status[tile], kFlagAgg | agg);
                int64_t j = (int64_t)tile - 1;
                while (true) {
                    const int64_t jj = j - lane;
                    unsigned long long st = 0;
                    if (jj >= 0) {
                        do { st = ld_acquire(&status[jj]); } while ((st >> 32) == 0);
                    } else {
                        st = kFlagPre;
                    }
                    const unsigned pre_mask = __ballot_sync(0xffffffffu, (st >> 32) == 2);
                    const int stop = pre_mask ? (__ffs(pre_mask) - 1) : 31;
                    uint32_t val = (lane <= stop) ? (uint32_t)st : 0u;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                    excl += val;
                    if (pre_mask) break;
                    j -= 32;
                }
                if (lane == 0) st_release(&status[tile], kFlagPre | (excl + agg));
            }
            if (lane == 0) s_excl = excl;
        }
        __syncthreads();
        uint32_t run = s_excl + wpre + inc - tsum;
        if (expand) {  // candidate -> (element, local index) map
            uint32_t o = run;
#pragma unroll 1
            for (int k = 0; k < kScanItems; k++) {
                const unsigned long long e = (unsigned long long)(base + k);
                for (uint32_t j = 0; j < v[k] && (int64_t)o + j < expand_cap; j++)
                    expand[o + j] = e | ((unsigned long long)j << 32);
                o += v[k];
            }
        }
        if (!out) {
        } else if (base + kScanItems <= n && ((reinterpret_cast<uintptr_t>(out + base) & 15) == 0)) {
            uint4* p = reinterpret_cast<uint4*>(out + base);
#pragma unroll
            for (int k = 0; k < kScanItems / 4; k++) {
                uint4 q;
                q.x = run; run += v[4 * k];
                q.y = run; run += v[4 * k + 1];
                q.z = run; run += v[4 * k + 2];
                q.w = run; run += v[4 * k + 3];
                p[k] = q;
            }
        } else {
#pragma unroll
            for (int k = 0; k < kScanItems; k++) {
                if (base + k < n) out[base + k] = run;
                run += v[k];
            }
        }
        if (tid == 0 && (int64_t)tile == ntiles - 1) *total = s_excl + agg;
        __syncthreads();
    }
}

size_t scan_scratch_words(int64_t n) { return (size_t)((n + kScanTile - 1) / kScanTile) + 2; }

void launch_scan(const uint32_t* in, uint32_t* out, uint32_t* total, const uint32_t* n_dev, int64_t cap,
                 uint32_t* scratch32, cudaStream_t st, unsigned long long* expand, int64_t expand_cap) {
    unsigned long long* scratch = reinterpret_cast<unsigned long long*>(scratch32);
    if (cap <= 0) {
        cudaMemsetAsync(total, 0, 4, st);
        return;
    }
    const int sms = device_sms();
    const int64_t tiles = (cap + kScanTile - 1) / kScanTile;
    cudaMemsetAsync(scratch, 0, (size_t)(tiles + 1) * 8, st);
    const int64_t grid = std::min<int64_t>(tiles, (int64_t)sms * 4);
    k_scan<<<(unsigned)grid, kScanThreads, 0, st>>>(in, out, total, n_dev, cap, scratch, expand, expand_cap);
}

}  // namespace vrs
