// Does compute-sanitizer racecheck model mbarrier hand-offs?  mode 0: producer
// warp writes shared memory, arrives on an mbarrier; consumer warp try_waits and
// reads.  mode 1: consumer reads, then (fence + atomic) hands the buffer back and
// the producer overwrites after observing the count (WAR through an atomic).
// mode 2: WAR through an "empty" mbarrier (consumer arrives, producer waits).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ void init(unsigned long long* b, uint32_t n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ void arrive(unsigned long long* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ bool tw(unsigned long long* b, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
    return ok;
}
__global__ void k(int mode, int* out) {
    __shared__ int buf[32];
    __shared__ unsigned long long full, empty;
    __shared__ unsigned cnt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { init(&full, 1); init(&empty, 1); cnt = 0; }
    __syncthreads();
    if (mode == 0) {
        if (warp == 0) { buf[lane] = lane; __syncwarp(); if (lane == 0) arrive(&full); }
        else { while (!tw(&full, 0)) {} out[lane] = buf[lane]; }
    } else if (mode == 1) {
        if (warp == 1) { out[lane] = buf[lane]; __syncwarp(); if (lane == 0) { __threadfence_block(); atomicAdd(&cnt, 1u); } }
        else { if (lane == 0) { while (atomicAdd(&cnt, 0u) == 0u) {} __threadfence_block(); } __syncwarp(); buf[lane] = 7; }
    } else {
        if (warp == 1) { out[lane] = buf[lane]; __syncwarp(); if (lane == 0) arrive(&empty); }
        else { while (!tw(&empty, 0)) {} buf[lane] = 7; }
    }
}
int main() {
    int* o; cudaMalloc(&o, 128);
    for (int m = 0; m < 3; m++) { k<<<1, 64>>>(m, o); cudaDeviceSynchronize(); printf("mode %d done\n", m); }
    return 0;
}
