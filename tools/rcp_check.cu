// Exhaustive check of the blend's clamped reciprocal (DESIGN R9): for every
// binary32 v in [2^-100, 2^100], MUFU estimate + one Newton step == __frcp_rn(v).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o rcp_check tools/rcp_check.cu
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t lo, uint32_t hi, unsigned long long* bad, uint32_t* first) {
    for (uint64_t b = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= hi;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const float v = __uint_as_float((uint32_t)b);
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
        const float e = fmaf(-v, r, 1.0f);
        r = fmaf(r, e, r);
        if (__float_as_uint(r) != __float_as_uint(__frcp_rn(v))) {
            atomicAdd(bad, 1ull);
            atomicMin(first, (uint32_t)b);
        }
    }
}
int main() {
    unsigned long long* bad;
    uint32_t* first;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&first, 4);
    *bad = 0;
    *first = 0xffffffffu;
    const float lo = 0x1p-100f, hi = 0x1p100f;
    k<<<148 * 16, 256>>>(*(const uint32_t*)&lo, *(const uint32_t*)&hi, bad, first);
    cudaError_t err = cudaDeviceSynchronize();
    printf("{\"range\": \"[2^-100, 2^100]\", \"values\": %u, \"mismatches\": %llu, \"first_bad_bits\": %u, \"cuda\": \"%s\"}\n",
           *(const uint32_t*)&hi - *(const uint32_t*)&lo + 1, *bad, *first, cudaGetErrorString(err));
    return (err == cudaSuccess && *bad == 0) ? 0 : 1;
}
