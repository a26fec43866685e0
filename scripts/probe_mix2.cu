// Which pipes does IMAD.WIDE occupy?  Pairs of instruction classes, 8+8
// independent chains per warp, 16 warps per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
template <int MIX>
__global__ void __launch_bounds__(256) mix_kernel(int iters, unsigned s0, unsigned s1, double d0, unsigned* sink) {
    unsigned a[8], g[8], b = s1 | 1u, c = s0 ^ 0x9E3779B9u;
    unsigned long long w[8];
    double f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { a[k] = s0 + k * 31u + threadIdx.x; g[k] = a[k] * 3u; w[k] = a[k]; f[k] = d0 + k + threadIdx.x * 1e-3; }
    const double fm = d0 * 0.999, fc = d0 * 1e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (MIX == 0 || MIX == 1 || MIX == 2 || MIX == 6) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[k]) : "r"(g[k]), "r"(b));
            if (MIX == 1 || MIX == 3 || MIX == 5) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(b), "r"(c));
            if (MIX == 3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(g[k]) : "r"(b), "r"(c));
            if (MIX == 2) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[k]) : "r"(b));
            if (MIX == 4 || MIX == 5 || MIX == 6) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(g[k]) : "r"(b), "r"(c));
            if (MIX == 4) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
            if (MIX == 7) { asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c)); asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(g[k]) : "r"(b), "r"(c)); }
            if (MIX == 8) { asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[k]) : "d"(fm), "d"(fc)); asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c)); asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(g[k]) : "r"(b), "r"(c)); }
            if (MIX == 9) { asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[k]) : "d"(fm), "d"(fc)); asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[k]) : "r"(b)); }
        }
    }
    unsigned t = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t ^= a[k] ^ g[k] ^ (unsigned)w[k] ^ (unsigned)(w[k] >> 32) ^ (unsigned)__double2loint(f[k]);
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
    printf("%-34s %.3f ms  %.2f cycles per group per warp per SMSP\n", name, best, best * 1e-3 * 1.965e9 / (20000.0 * 16.0));
    cudaFree(sink);
}
int main() {
    run<0>("8 wide"); run<1>("8 wide + 8 lop3"); run<2>("8 wide + 8 iadd"); run<3>("16 lop3"); run<4>("16 ffma");
    run<5>("8 lop3 + 8 ffma"); run<6>("8 wide + 8 ffma"); run<7>("8 imad.lo + 8 lop3"); run<8>("8 dfma + 8 imad.lo + 8 lop3"); run<9>("8 dfma + 8 mul.hi");
    return 0;
}
