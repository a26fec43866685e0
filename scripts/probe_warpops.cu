// Dependent-chain latencies (cycles per link, one warp) of the warp-level and
// conversion ops the TB Gillespie kernel's lookup is built from.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_warpops scripts/probe_warpops.cu
#include <cstdio>
#include <cstdint>
#define N 4096
__global__ void probe(long long* out, uint32_t seed, double dseed) {
    const uint32_t lane = threadIdx.x;
    __shared__ uint16_t tab[1024];
    for (int i = lane; i < 1024; i += 32) tab[i] = (uint16_t)((i & 31) * 3 + 1);
    __syncwarp();
    long long t0, t1;
    uint32_t x = seed + lane, acc = 0;
    // 1: ballot + ffs + shfl
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        const uint32_t m = __ballot_sync(0xffffffffu, x > (acc & 15));
        const uint32_t o = __ffs(m) - 1;
        acc += __shfl_sync(0xffffffffu, x, o & 31);
    }
    t1 = clock64();
    if (lane == 0) out[0] = (t1 - t0) / N;
    // 2: redux max
    uint32_t acc2 = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        const bool own = (x & 31) == (acc2 & 31);
        acc2 += __reduce_max_sync(0xffffffffu, own ? (lane << 16 | (x & 0xffff)) : 0u);
    }
    t1 = clock64();
    if (lane == 0) out[1] = (t1 - t0) / N;
    // 3: F2I
    double d = dseed;
    uint32_t acc3 = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        acc3 = static_cast<uint32_t>(d);
        d = __hiloint2double(0x40200000 + (acc3 & 7), 0);
    }
    t1 = clock64();
    if (lane == 0) out[2] = (t1 - t0) / N;
    // 4: magic-add floor
    uint32_t acc4 = 0;
    d = dseed;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        acc4 = __double2loint(__dadd_rd(d, 0x1p52));
        d = __hiloint2double(0x40200000 + (acc4 & 7), 0);
    }
    t1 = clock64();
    if (lane == 0) out[3] = (t1 - t0) / N;
    // 5: LDS dependent
    uint32_t idx = lane;
    t0 = clock64();
    for (int i = 0; i < N; ++i) idx = tab[(idx * 7 + lane) & 1023];
    t1 = clock64();
    if (lane == 0) out[4] = (t1 - t0) / N;
    // 6: ballot + popc
    uint32_t acc6 = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        const uint32_t m = __ballot_sync(0xffffffffu, x > (acc6 & 15));
        acc6 += __popc(m);
    }
    t1 = clock64();
    if (lane == 0) out[5] = (t1 - t0) / N;
    // 7: ballot only (+ dependent LOP)
    uint32_t acc7 = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        const uint32_t m = __ballot_sync(0xffffffffu, x > (acc7 & 15));
        acc7 ^= m;
    }
    t1 = clock64();
    if (lane == 0) out[6] = (t1 - t0) / N;
    // 8: shfl only
    uint32_t acc8 = x;
    t0 = clock64();
    for (int i = 0; i < N; ++i) acc8 = __shfl_sync(0xffffffffu, acc8 + 1, (acc8 + lane) & 31);
    t1 = clock64();
    if (lane == 0) out[7] = (t1 - t0) / N;
    // 9: DFMA chain
    double e = dseed;
    t0 = clock64();
    for (int i = 0; i < N; ++i) e = fma(e, 1.0000001, 1e-9);
    t1 = clock64();
    if (lane == 0) out[8] = (t1 - t0) / N;
    // 10: IEEE division chain
    double q = dseed;
    t0 = clock64();
    for (int i = 0; i < N; ++i) q = __ddiv_rn(dseed + 3.0, q + 1.5);
    t1 = clock64();
    if (lane == 0) out[9] = (t1 - t0) / N;
    // 11: match_any
    uint32_t acc11 = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) acc11 += __match_any_sync(0xffffffffu, (x + acc11) & 3);
    t1 = clock64();
    if (lane == 0) out[10] = (t1 - t0) / N;
    // 12: uniform branch on a predicate
    uint32_t acc12 = x;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        if (__any_sync(0xffffffffu, acc12 == 0xdeadbeef)) break;
        acc12 = acc12 * 3 + 1;
    }
    t1 = clock64();
    if (lane == 0) out[11] = (t1 - t0) / N;
    if (acc + acc2 + acc3 + acc4 + idx + acc6 + acc7 + acc8 + acc11 + acc12 == 12345 && e + q == 1.0) out[15] = 1;
}
int main() {
    long long* d;
    cudaMalloc(&d, 16 * 8);
    probe<<<1, 32>>>(d, 5, 9.5);
    probe<<<1, 32>>>(d, 5, 9.5);
    long long h[16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[] = {"ballot+ffs+shfl", "redux.max(+select)", "F2I.U32.F64 (+I2D bits)", "dadd_rd magic (+bits)",
                           "LDS.U16 dependent", "ballot+popc", "ballot+xor", "shfl", "DFMA", "ddiv_rn(+2 dadd)",
                           "match_any", "any+branch+imad"};
    for (int i = 0; i < 12; ++i) printf("%-28s %lld cycles/link\n", names[i], h[i]);
    return 0;
}
