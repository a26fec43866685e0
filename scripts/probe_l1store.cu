// Does a global store keep (update) the line in L1, or does the next load of the
// line go to L2?  One warp, dependent chains over a 4 KB footprint.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_l1store scripts/probe_l1store.cu
#include <cstdio>
#include <cstdint>
#define N 2048
__device__ __forceinline__ uint32_t ld(const uint16_t* p) {
    uint16_t v;
    asm volatile("ld.global.ca.u16 %0, [%1];" : "=h"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st(uint16_t* p, uint32_t v) {
    asm volatile("st.global.u16 [%0], %1;" ::"l"(p), "h"(static_cast<uint16_t>(v)) : "memory");
}
template <int kMode>
__global__ void probe(uint16_t* buf, long long* out) {
    const uint32_t lane = threadIdx.x;
    long long best = 1ll << 60;
    uint32_t acc = 0, sink = 0;
    for (int rep = 0; rep < 3; ++rep) {
        acc = lane;
        __syncwarp();
        const long long t0 = clock64();
        for (int i = 0; i < N; ++i) {
            const uint32_t a = (acc * 7 + lane) & 2047;
            const uint32_t v = ld(buf + a);
            if (kMode == 1) st(buf + a, v);       // same value: the chain stays reproducible
            __syncwarp();
            acc = kMode == 2 ? v : ld(buf + ((v + 1) & 2047)) & 2047;  // mode 2: one load per link
        }
        const long long t1 = clock64();
        if (t1 - t0 < best) best = t1 - t0;
        sink ^= acc;
    }
    if (lane == 0) out[kMode] = best;
    out[8 + kMode * 32 + lane] = sink;  // keeps the loads alive
}
int main() {
    uint16_t* buf; long long* d;
    cudaMalloc(&buf, 4096); cudaMalloc(&d, 2048);
    uint16_t h[2048]; for (int i = 0; i < 2048; ++i) h[i] = (uint16_t)((i * 13 + 5) & 2047);
    cudaMemcpy(buf, h, 4096, cudaMemcpyHostToDevice);
    probe<0><<<1, 32>>>(buf, d); probe<1><<<1, 32>>>(buf, d); probe<2><<<1, 32>>>(buf, d);
    long long o[8]; cudaMemcpy(o, d, 64, cudaMemcpyDeviceToHost);
    printf("ld -> ld (dependent)            %.1f cycles/iter\nld -> st same line -> ld        %.1f cycles/iter\nld only                         %.1f cycles/iter\n",
           (double)o[0] / N, (double)o[1] / N, (double)o[2] / N);
    return 0;
}
