// Reciprocal throughput (cycles per warp instruction per SMSP) of the
// instructions the RNG and simulators are made of, on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
template <int OP>
__global__ void __launch_bounds__(256) rt_kernel(int iters, unsigned s0, unsigned s1, double d0, unsigned* sink) {
    unsigned a[CHAINS], b = s1 | 1u, c = s0 ^ 0x9E3779B9u;
    unsigned long long w[CHAINS];
    double f[CHAINS];
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) { a[k] = s0 + k * 31u + threadIdx.x; w[k] = a[k]; f[k] = d0 + k + threadIdx.x * 1e-3; }
    const double fm = d0 * 0.999, fc = d0 * 1e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CHAINS; ++k) {
            if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
            if (OP == 1) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[k]) : "r"(b));
            if (OP == 2) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[k]) : "r"(a[k]), "r"(b));
            if (OP == 3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(b), "r"(c));
            if (OP == 4) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[k]) : "r"(b));
            if (OP == 5) asm volatile("shf.l.wrap.b32 %0, %0, %0, 7;" : "+r"(a[k]));
            if (OP == 6) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[k]) : "d"(fm), "d"(fc));
            if (OP == 7) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(f[k]) : "d"(fc));
            if (OP == 8) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(f[k]) : "d"(fm));
            if (OP == 9) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
            if (OP == 10) asm volatile("mul.lo.u64 %0, %0, %1;" : "+l"(w[k]) : "l"((unsigned long long)b * 0x10001ull));
            if (OP == 11) asm volatile("mul.hi.u64 %0, %0, %1;" : "+l"(w[k]) : "l"(0xD2B74407B1CE6E93ull));
        }
    }
    unsigned t = 0;
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) t ^= a[k] ^ (unsigned)w[k] ^ (unsigned)(w[k] >> 32) ^ (unsigned)__double2loint(f[k]);
    if (t == 0x12345u) sink[0] = t;
}

template <int OP>
void run(const char* name) {
    unsigned* sink; cudaMalloc(&sink, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000, blocks = 148 * 8;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cudaEventRecord(e0);
        rt_kernel<OP><<<blocks, 256>>>(iters, 12345u, 777u, 1.0, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
    }
    const double cyc = best * 1e-3 * 1.965e9 / (double(iters) * CHAINS * 16.0);
    printf("%-14s %.3f ms  rt = %.2f cycles per warp instruction per SMSP\n", name, best, cyc);
    cudaFree(sink);
}

int main() {
    run<0>("mad.lo.u32"); run<1>("mul.hi.u32"); run<2>("mad.wide.u32"); run<3>("lop3.b32");
    run<4>("add.u32"); run<5>("shf.l.wrap"); run<6>("fma.f64"); run<7>("add.f64"); run<8>("mul.f64");
    run<9>("fma.f32"); run<10>("mul.lo.u64"); run<11>("mul.hi.u64");
    return 0;
}
