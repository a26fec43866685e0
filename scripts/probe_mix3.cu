// Does the FP64 pipe overlap with the integer work of a counter-based RNG?
// Groups of independent chains per warp, 16 warps per SMSP; prints cycles per
// group per warp per SMSP.  (nvcc -arch=sm_100a -O3 -o probe_mix3 probe_mix3.cu)
#include <cstdio>
#include <cuda_runtime.h>
template <int MIX>
__global__ void __launch_bounds__(256) mix_kernel(int iters, unsigned s0, unsigned s1, double d0, unsigned* sink) {
    unsigned a[8], g[8], b = s1 | 1u, c = s0 ^ 0x9E3779B9u;
    unsigned long long w[8];
    double f[8], h[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { a[k] = s0 + k * 31u + threadIdx.x; g[k] = a[k] * 3u; w[k] = a[k]; f[k] = d0 + k + threadIdx.x * 1e-3; h[k] = f[k] * 0.5; }
    const double fm = d0 * 0.999, fc = d0 * 1e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const bool dfma = MIX == 0 || MIX == 1 || MIX == 2 || MIX == 4 || MIX == 5 || MIX == 6 || MIX == 7 || MIX == 8;
            const bool dfma2 = MIX == 4 || MIX == 8;
            const bool wide = MIX == 1 || MIX == 2 || MIX == 3 || MIX == 4;
            const bool lop = MIX == 2 || MIX == 3 || MIX == 4 || MIX == 6 || MIX == 8;
            const bool hi_lo = MIX == 5 || MIX == 6 || MIX == 8;
            const bool lop_only = MIX == 7;
            if (dfma) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[k]) : "d"(fm), "d"(fc));
            if (dfma2) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(h[k]) : "d"(fm), "d"(fc));
            if (wide) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[k]) : "r"(g[k]), "r"(b));
            if (lop || lop_only) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(b), "r"(c));
            if (hi_lo) { unsigned hi; asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(g[k]), "r"(b)); asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(g[k]) : "r"(b)); a[k] ^= hi; }
        }
    }
    unsigned t = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t ^= a[k] ^ g[k] ^ (unsigned)w[k] ^ (unsigned)(w[k] >> 32) ^ (unsigned)__double2loint(f[k]) ^ (unsigned)__double2loint(h[k]);
    if (t == 0x12345u) sink[0] = t;
}
template <int MIX>
void run(const char* name) {
    unsigned* sink; cudaMalloc(&sink, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        mix_kernel<MIX><<<148 * 8, 256>>>(20000, 12345u, 777u, 1.0, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
    }
    printf("%-44s %.3f ms  %.2f cycles per group per warp per SMSP\n", name, best, best * 1e-3 * 1.965e9 / (20000.0 * 16.0));
    cudaFree(sink);
}
int main() {
    run<0>("8 dfma"); run<1>("8 dfma + 8 wide"); run<2>("8 dfma + 8 wide + 8 lop3"); run<3>("8 wide + 8 lop3");
    run<4>("16 dfma + 8 wide + 8 lop3"); run<5>("8 dfma + 8 (mul.hi + mul.lo + xor)"); run<6>("8 dfma + 8 (mul.hi + mul.lo + xor) + 8 lop3");
    run<7>("8 dfma + 8 lop3"); run<8>("16 dfma + 8 (hi+lo+xor) + 8 lop3");
    return 0;
}
