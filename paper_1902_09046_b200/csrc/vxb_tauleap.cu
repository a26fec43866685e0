// vxb_tauleap.cu -- multilevel Monte Carlo with coupled Poisson tau-leaping on
// the Michaelis-Menten network (config 4): S+E->C (k1), C->S+E (k2), C->E+P (k3).
//
// Not in the reference (tau-leap is out of scope there; rng.cpp
// has no Poisson sampler).  The scheme is defined by oracle/vxb_oracle.cpp
// (vxo_mlmc_level) in the style of tb_model.cpp:39-116 and reproduced here
// bit-for-bit:
//  * Poisson(lam) by CDF inversion from ONE uniform: p0 = exp(-lam) through the
//    reference's exp2_clamped (fastmath.hpp:57-79), p_k = (p_{k-1} lam)(1/k),
//    at most 1023 terms; the reciprocals 1/k come from a shared-memory table; the
//    outcome k = 0 is decided from 1 - lam where that is safe (see poisson_inv);
//  * propensities from max(X,0): a1 = (k1 S) E, a2 = k2 C, a3 = k3 C;
//  * level 0: plain tau-leap; step s reads stream positions 4s + r;
//  * level l>=1: Anderson-Higham coupling of a fine path (tau_l) with a coarse
//    path (M tau_l) whose propensities are frozen over the coarse step; per fine
//    step and reaction r: m = min(af, ac), P1~Poi(m tau), P2~Poi((af-m) tau),
//    P3~Poi((ac-m) tau); reaction r of fine step s owns Philox block 3s + r
//    (position 6s+2r drives P1, position 6s+2r+1 the residual -- at most one of
//    P2, P3 has a positive rate, so they share it); fine fires P1+P2, coarse P1+P3;
//  * path i of level l owns RngStream(derive_seed(seed,{l}), i).
// Quiet steps: on the fine levels rate * tau ~ 1e-3, so in most steps nothing fires and
// neither the state nor the propensities change.  The coupled loop keeps the six
// thresholds "uniform <= thr => k = 0" in registers, refreshes them only after an event
// (or when a new coarse step finds a changed coarse state), and decides a quiet step
// with six compares and one branch; the three (throughput generator: two) Philox
// blocks of the step are drawn before that branch so that their round chains
// interleave.  The decisions are those of the plain loop, so the exact instance stays
// bit-identical to the oracle.  The throughput instances draw the six uniforms of a
// fine step from TWO Philox4x32 blocks (42 bits each in fp64, 23-bit midpoints in fp32).
// One path per thread, integer state in registers; only four 64-bit sums (and
// optionally Y per path) leave the device, so the level sums are exact integers
// and identical for any sharding.

#include <cmath>
#include <vector>

#include "vxb_common.cuh"
#include "vxb_rng.cuh"

#ifndef VXB_TL_MINB
#define VXB_TL_MINB 4  // swept 1, 4, 6, 8: config 4 exact 1.01 / 0.94 / 0.99 / 0.99 s
#endif

namespace vxb {

constexpr int kTlBlock = 128;
constexpr int kMaxPoisson = 1023;

struct TauParams {
    uint64_t first, count;
    uint64_t seed_hash;  // splitmix64(derive_seed(seed,{level}))
    FastKeys fast;       // VXB_RNG_FAST: Philox4x32 round keys of the seed
    uint64_t n_fine;     // fine steps
    uint32_t level, refine;
    double tau;
    double rate[3];
    int32_t init[4];
    long long* sums;  // 4
    int32_t* y_out;
};

struct MM {
    int32_t s, e, c, p;
    __device__ __forceinline__ void fire(int k1, int k2, int k3) {
        s += -k1 + k2;
        e += -k1 + k2 + k3;
        c += k1 - k2 - k3;
        p += k3;
    }
    __device__ __forceinline__ void prop(const double* k, double* a) const {
        const double ds = static_cast<double>(s > 0 ? s : 0);
        const double de = static_cast<double>(e > 0 ? e : 0);
        const double dc = static_cast<double>(c > 0 ? c : 0);
        a[0] = __dmul_rn(__dmul_rn(k[0], ds), de);
        a[1] = __dmul_rn(k[1], dc);
        a[2] = __dmul_rn(k[2], dc);
    }
};

template <class A>
__device__ __forceinline__ int poisson_inv(double lam, double u, const double* __restrict__ inv,
                                           long long& iters) {
    if (!(lam > 0.0)) return 0;
    // The inversion returns 0 iff u <= p0 = exp(-lam).  exp(-lam) >= 1 - lam, and the
    // computed p0 is within 2^-49 (relative) of exp(-lam), so u <= (1 - lam) - 2^-48
    // already decides k = 0 -- without evaluating the exponential.  On the fine levels
    // (lam = rate * tau ~ 1e-3) that is the outcome of >99% of the draws, and a warp
    // whose 32 lanes all take it skips the polynomial altogether.  Same k, same
    // iteration count: results stay bit-identical to the oracle.
    const double one_m = __dsub_rn(1.0, lam);
    if (u <= __dsub_rn(one_m, 0x1p-48)) return 0;
    // Second shortcut, same argument one term further: exp(-lam) <= 1 - lam + lam^2/2, so
    // u above that (plus the margin) is beyond the computed p0: k >= 1; and the CDF after
    // one term, exp(-lam)(1 + lam), is >= 1 - lam^2 (its computed value within 2^-48 of
    // that), so u <= (1 - lam^2) - 2^-47 ends the oracle's loop at k = 1, after exactly one
    // iteration.  The exponential is then needed only in two windows of width ~lam^2/2
    // instead of for every draw above 1 - lam: on the fine levels once in ~1e6 draws
    // instead of once in ~1e3, and a warp rarely has a lane on the slow path.
    if (lam < 0.5) {
        const double l2 = __dmul_rn(lam, lam);
        if (u > __dadd_rn(__dadd_rn(one_m, __dmul_rn(0.5, l2)), 0x1p-48) &&
            u <= __dsub_rn(__dsub_rn(1.0, l2), 0x1p-47)) {
            ++iters;
            return 1;
        }
    }
    double p = exp2_clamped<A>(A::mul(-lam, kInvLn2));
    double cdf = p;
    int k = 0;
    while (u > cdf && k < kMaxPoisson) {
        ++k;
        p = A::mul(A::mul(p, lam), inv[k]);
        cdf = A::add(cdf, p);
        ++iters;
    }
    return k;
}

// ---- fp32 throughput instance (VXB_F32 + VXB_RNG_FAST): propensities, rates and the
// CDF inversion in float, p0 = 2^(-lam log2 e) by ONE MUFU (ex2.approx), 23-bit uniforms
// from mantissa bits.  Statistically validated against the fp64 instances
// (tests/test_gpu_workloads.py); the state is integer in every instance, so the
// conservation laws hold exactly here too.
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// (m + 1/2) 2^-23 for a 23-bit m: the MIDPOINT of the bucket, exact in float (no int->float
// conversion).  With the bucket's lower edge P(u <= p0) would be too large by up to 2^-23
// for every draw -- at event probabilities of 1e-3 per step a -6e-5 relative bias of the
// firing rate, visible in E[P(T)] at 1e8 paths; midpoints make the error symmetric.
__device__ __forceinline__ float unit_f32(uint32_t w) {
    return __uint_as_float(0x3F800000u | (w >> 9)) - (1.0f - 0x1p-24f);
}
// Inversion on the SURVIVAL side: v uniform, k = 0 iff v >= q0 = 1 - exp(-lam), then
// k = 1 iff v >= q0 - p1, ...  On the fine levels lam ~ 1e-3, so an event has probability
// ~lam and a float CDF near 1 resolves it to 6e-8 ABSOLUTE = 1e-4 relative (the first
// version of this instance inverted the CDF and came out 7e-5 high in E[P(T)] at 4e7 paths,
// chi2 43 on 24 dof); q0 itself is small and carries float RELATIVE precision: for
// lam < 1/8 from the series lam (1 - lam/2 (1 - lam/3 (1 - lam/4 (1 - lam/5)))) (truncation
// < 5e-8 relative), above from one MUFU ex2.
__device__ __forceinline__ int poisson_inv_f32(float lam, float v, const float* __restrict__ inv,
                                               long long& iters) {
    if (!(lam > 0.0f)) return 0;
    if (v >= lam) return 0;  // q0 = 1 - exp(-lam) <= lam (and so is the computed q0): k = 0, no series
    float q0, p;
    if (lam < 0.125f) {
        q0 = lam * (1.0f - 0.5f * lam * (1.0f - (1.0f / 3.0f) * lam * (1.0f - 0.25f * lam * (1.0f - 0.2f * lam))));
        p = 1.0f - q0;
    } else {
        p = ex2_approx(-1.4426950408889634f * lam);
        q0 = 1.0f - p;
    }
    if (v >= q0) return 0;
    float tail = q0;
    int k = 0;
    while (v < tail && k < kMaxPoisson) {
        ++k;
        p = p * lam * inv[k];
        const float next = tail - p;
        ++iters;
        if (next == tail) break;  // the terms have dropped below the float resolution of the tail
        tail = next;
    }
    return k;
}
// 21 bits made of the low 11 bits of two Philox words (the fifth and sixth field of a block)
__device__ __forceinline__ uint32_t low_field(uint32_t x, uint32_t y) {  // 21 bits of two words' low 11
    return ((x & 0x7FFu) << 10) | ((y & 0x7FFu) >> 1);
}
// The 23-bit uniform m (midpoint (m + 1/2) 2^-23) decides k = 0 for rate lam iff
// m >= Tm = ceil(lam 2^23 - 1/2) (the pre-test v >= lam of poisson_inv_f32; all exact in
// float).  The quiet test sees only the leading 21 bits t of m: t >= ceil(Tm / 4) implies it.
// Returns that bound on t, or 2^21 when no t can decide (lam too large).
__device__ __forceinline__ uint32_t quiet_bound_f32(float lam) {
    const float tm = ceilf(lam * 8388608.0f - 0.5f);
    if (!(tm > 0.0f)) return 0u;               // lam <= 2^-24 (or not positive): every uniform
    if (!(tm < 8388608.0f)) return 1u << 21;   // lam > 1 - 2^-24: none
    return (static_cast<uint32_t>(tm) + 3u) >> 2;
}
struct MMf {  // propensities in float from the integer state
    __device__ __forceinline__ static void prop(const MM& x, const float* k, float* a) {
        const float ds = static_cast<float>(x.s > 0 ? x.s : 0);
        const float de = static_cast<float>(x.e > 0 ? x.e : 0);
        const float dc = static_cast<float>(x.c > 0 ? x.c : 0);
        a[0] = k[0] * ds * de;
        a[1] = k[1] * dc;
        a[2] = k[2] * dc;
    }
};

__global__ void __launch_bounds__(kTlBlock, VXB_TL_MINB) tauleap_f32_kernel(const __grid_constant__ TauParams p) {
    __shared__ float s_inv[kMaxPoisson + 1];
    __shared__ long long s_sum[4];
    for (int k = threadIdx.x; k <= kMaxPoisson; k += kTlBlock) s_inv[k] = k ? 1.0f / static_cast<float>(k) : 0.0f;
    if (threadIdx.x < 4) s_sum[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * kTlBlock + threadIdx.x;
    long long sy = 0, sy2 = 0, sp = 0, it = 0;
    if (r < p.count) {
        const uint64_t path = p.first + r;
        const uint32_t pl = static_cast<uint32_t>(path), ph = static_cast<uint32_t>(path >> 32);
        const float tau = static_cast<float>(p.tau);
        const float rate[3] = {static_cast<float>(p.rate[0]), static_cast<float>(p.rate[1]),
                               static_cast<float>(p.rate[2])};
        // the fp32 instance draws from its own domain (bit 7 of the domain word)
        const uint32_t dom = kDomNoise | 0x80u | (p.level << 8);
        MM f{p.init[0], p.init[1], p.init[2], p.init[3]};
        MM c = f;
        float af[3], ac[3];
        if (p.level == 0) {
            for (uint64_t st = 0; st < p.n_fine; ++st) {
                MMf::prop(f, rate, af);
                const Words32 w = philox4x32(p.fast, static_cast<uint32_t>(st),
                                             dom | (static_cast<uint32_t>(st >> 32) << 16), pl, ph);
                const int k0 = poisson_inv_f32(af[0] * tau, unit_f32(w.a), s_inv, it);
                const int k1 = poisson_inv_f32(af[1] * tau, unit_f32(w.b), s_inv, it);
                const int k2 = poisson_inv_f32(af[2] * tau, unit_f32(w.c), s_inv, it);
                f.fire(k0, k1, k2);
            }
        } else {
            // as in tauleap_kernel: the bounds above which a draw decides k = 0 stay in
            // registers and are refreshed only after an event; a quiet step is ONE Philox
            // block (the leading 21 bits of the six uniforms, fields as in
            // StepBits<VXB_RNG_FAST>), six compares and one branch; a step that is not quiet
            // draws the second block for the two trailing bits of the 23-bit uniforms
            uint32_t phase = 0;
            bool stale = true, coarse_moved = true;
            uint32_t bound_c[3], bound_r[3];  // reactions 0, 1: on the word (shifted by 11); 2: on the field
            bool loud = false;  // some rate is too large for any uniform to decide k = 0 up front
            for (uint64_t st = 0; st < p.n_fine; ++st) {
                if (phase == 0 && coarse_moved) {
                    MMf::prop(c, rate, ac);
                    coarse_moved = false;
                    stale = true;
                }
                if (++phase == p.refine) phase = 0;
                if (stale) {
                    MMf::prop(f, rate, af);
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const float mn = af[q] < ac[q] ? af[q] : ac[q];
                        const float mx = af[q] > ac[q] ? af[q] : ac[q];
                        bound_c[q] = quiet_bound_f32(mn * tau);
                        bound_r[q] = quiet_bound_f32((mx - mn) * tau);
                    }
                    loud = ((bound_c[0] | bound_c[1] | bound_c[2] | bound_r[0] | bound_r[1] | bound_r[2]) >> 21) != 0;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        bound_c[q] <<= 11;
                        bound_r[q] <<= 11;
                    }
                    stale = false;
                }
                const uint32_t hi = dom | (static_cast<uint32_t>((2 * st) >> 32) << 16);
                const Words32 w0 = philox4x32(p.fast, static_cast<uint32_t>(2 * st), hi, pl, ph);
                const uint32_t t4 = low_field(w0.a, w0.b), t5 = low_field(w0.c, w0.d);
                const bool quiet = !loud & (w0.a >= bound_c[0]) & (w0.b >= bound_r[0]) & (w0.c >= bound_c[1]) &
                                   (w0.d >= bound_r[1]) & (t4 >= bound_c[2]) & (t5 >= bound_r[2]);
                if (quiet) continue;
                // the full 23-bit uniforms, left-aligned as unit_f32 takes them: 21 leading
                // bits, then two bits of the second block
                const Words32 w1 = philox4x32(p.fast, static_cast<uint32_t>(2 * st + 1), hi, pl, ph);
                const uint32_t word[6] = {(w0.a & ~0x7FFu) | ((w1.a >> 30) << 9),  (w0.b & ~0x7FFu) | ((w1.b >> 30) << 9),
                                          (w0.c & ~0x7FFu) | ((w1.c >> 30) << 9),  (w0.d & ~0x7FFu) | ((w1.d >> 30) << 9),
                                          (t4 << 11) | (((w1.a >> 28) & 3u) << 9), (t5 << 11) | (((w1.b >> 28) & 3u) << 9)};
                int kf[3], kc[3];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const bool fine_larger = af[q] > ac[q];
                    const float mn = af[q] < ac[q] ? af[q] : ac[q];
                    const float mx = fine_larger ? af[q] : ac[q];
                    const int p1 = poisson_inv_f32(mn * tau, unit_f32(word[2 * q]), s_inv, it);
                    const int pr = poisson_inv_f32((mx - mn) * tau, unit_f32(word[2 * q + 1]), s_inv, it);
                    kf[q] = p1 + (fine_larger ? pr : 0);
                    kc[q] = p1 + (fine_larger ? 0 : pr);
                }
                f.fire(kf[0], kf[1], kf[2]);
                c.fire(kc[0], kc[1], kc[2]);
                // the bounds follow the fine state at once, the frozen coarse rates at the next coarse step
                stale = (kf[0] | kf[1] | kf[2]) != 0;
                coarse_moved = coarse_moved | ((kc[0] | kc[1] | kc[2]) != 0);
            }
        }
        const int32_t y = p.level == 0 ? f.p : f.p - c.p;
        if (p.y_out) p.y_out[r] = y;
        sy = y;
        sy2 = static_cast<long long>(y) * y;
        sp = f.p;
    }
    for (int o = 16; o; o >>= 1) {
        sy += __shfl_down_sync(0xffffffffu, sy, o);
        sy2 += __shfl_down_sync(0xffffffffu, sy2, o);
        sp += __shfl_down_sync(0xffffffffu, sp, o);
        it += __shfl_down_sync(0xffffffffu, it, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[0]), static_cast<unsigned long long>(sy));
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[1]), static_cast<unsigned long long>(sy2));
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[2]), static_cast<unsigned long long>(sp));
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[3]), static_cast<unsigned long long>(it));
    }
    __syncthreads();
    if (threadIdx.x < 4)
        atomicAdd(reinterpret_cast<unsigned long long*>(&p.sums[threadIdx.x]),
                  static_cast<unsigned long long>(s_sum[threadIdx.x]));
}

// Two uniforms of random block `block` of this path: the reference stream's pair
// block (positions 2*block, 2*block+1) or, for the throughput generator, the
// Philox4x32 block (block, level domain, path).
template <int kRng>
__device__ __forceinline__ void draw_pair(const TauParams& p, uint64_t key, uint64_t path,
                                          uint64_t block, double& u0, double& u1) {
    if (kRng == VXB_RNG_REF) {
        const Words w = philox2x64(key, block);
        u0 = to_unit(w.w0);
        u1 = to_unit(w.w1);
    } else {
        const Words32 w = philox4x32(p.fast, static_cast<uint32_t>(block),
                                     kDomNoise | (p.level << 8) | (static_cast<uint32_t>(block >> 32) << 16),
                                     static_cast<uint32_t>(path), static_cast<uint32_t>(path >> 32));
        u0 = fast_unit(w.a, w.b);
        u1 = fast_unit(w.c, w.d);
    }
}

// The random bits of one coupled fine step, and the quiet test on them.  A uniform is
// only ever COMPARED on the common path, so the test is done on the leading 32 bits of
// the raw word against an integer bound (quiet_bound): `top < bound` implies
// u <= (1 - lam) - 2^-48, i.e. k = 0 by the first shortcut of poisson_inv.  The bound is
// conservative by less than one unit of 2^-32: a draw that falls in that sliver (or any
// draw that fires) takes the full path, which converts the words to doubles and runs the
// oracle's inversion -- the results are those of the plain loop, bit for bit.
template <int kRng> struct StepBits;
template <> struct StepBits<VXB_RNG_REF> {
    Words w[3];  // reaction q of fine step st owns Philox2x64 block 3 st + q
    __device__ __forceinline__ void draw(const TauParams&, uint64_t key, uint64_t, uint64_t st) {
#pragma unroll
        for (int q = 0; q < 3; ++q) w[q] = philox2x64(key, 3 * st + q);
    }
    __device__ __forceinline__ uint32_t top_common(int q) const { return static_cast<uint32_t>(w[q].w0 >> 32); }
    __device__ __forceinline__ uint32_t top_residual(int q) const { return static_cast<uint32_t>(w[q].w1 >> 32); }
    __device__ __forceinline__ double common(int q) const { return to_unit(w[q].w0); }
    __device__ __forceinline__ double residual(int q) const { return to_unit(w[q].w1); }
    // top < bound  =>  x < T 2^11  =>  (x >> 11) < T = floor(thr 2^53)  =>  to_unit(x) <= thr
    __device__ __forceinline__ void complete(const TauParams&) {}
    __device__ __forceinline__ static uint32_t bound(double lam, int) {
        if (!(lam > 0.0)) return 0xFFFFFFFFu;  // never fires (the sliver still takes the full path)
        const double thr = __dsub_rn(__dsub_rn(1.0, lam), 0x1p-48);
        if (!(thr > 0.0)) return 0u;           // lam >= 1: always the full path
        return static_cast<uint32_t>((__double2ull_rd(thr * 0x1p53) << 11) >> 32);
    }
};
// Throughput generator: ONE Philox4x32 block (2 st) carries the leading 21 bits of the six
// uniforms of a fine step -- the leading 21 bits of its four words and two fields made of
// their low 11 bits -- and decides a quiet step; only a step that is not quiet draws the
// second block (2 st + 1) for the trailing 21 bits of the 42-bit uniforms.  Field order:
// (common, residual) of reaction 0, of reaction 1 (words a b c d), of reaction 2 (low bits).
template <> struct StepBits<VXB_RNG_FAST> {
    Words32 a, b;
    uint32_t hi, pl, ph, ctr;
    __device__ __forceinline__ void draw(const TauParams& p, uint64_t, uint64_t path, uint64_t st) {
        hi = kDomNoise | (p.level << 8) | (static_cast<uint32_t>((2 * st) >> 32) << 16);
        pl = static_cast<uint32_t>(path);
        ph = static_cast<uint32_t>(path >> 32);
        ctr = static_cast<uint32_t>(2 * st);
        a = philox4x32(p.fast, ctr, hi, pl, ph);
    }
    // leading bits in the form the bounds are stored in: the whole word for reactions 0 and 1
    // (bound shifted left by 11), the 21-bit field for reaction 2
    __device__ __forceinline__ uint32_t top_common(int q) const { return q == 0 ? a.a : q == 1 ? a.c : low_field(a.a, a.b); }
    __device__ __forceinline__ uint32_t top_residual(int q) const { return q == 0 ? a.b : q == 1 ? a.d : low_field(a.c, a.d); }
    // top21 < floor(thr 2^21)  =>  the 42-bit mantissa is below thr 2^42  =>  u < thr
    __device__ __forceinline__ static uint32_t bound(double lam, int q) {
        const uint32_t all = q == 2 ? 0x1FFFFFu : 0xFFFFFFFFu;
        if (!(lam > 0.0)) return all;
        const double thr = __dsub_rn(__dsub_rn(1.0, lam), 0x1p-48);
        if (!(thr > 0.0)) return 0u;
        const uint32_t b21 = __double2uint_rd(thr * 0x1p21);
        return q == 2 ? b21 : b21 << 11;
    }
    __device__ __forceinline__ void complete(const TauParams& p) { b = philox4x32(p.fast, ctr + 1, hi, pl, ph); }
    // 42-bit uniform from leading and trailing 21 bits: 1.m - 1 with m = top : low : 0...
    __device__ __forceinline__ static double unit42(uint32_t top, uint32_t low) {
        return __dsub_rn(__hiloint2double(0x3FF00000u | (top >> 1), (top << 31) | (low << 10)), 1.0);
    }
    __device__ __forceinline__ double common(int q) const {
        return q == 0 ? unit42(a.a >> 11, b.a >> 11) : q == 1 ? unit42(a.c >> 11, b.c >> 11)
                                                             : unit42(low_field(a.a, a.b), low_field(b.a, b.b));
    }
    __device__ __forceinline__ double residual(int q) const {
        return q == 0 ? unit42(a.b >> 11, b.b >> 11) : q == 1 ? unit42(a.d >> 11, b.d >> 11)
                                                             : unit42(low_field(a.c, a.d), low_field(b.c, b.d));
    }
};

template <int kRng>
__global__ void __launch_bounds__(kTlBlock, VXB_TL_MINB) tauleap_kernel(const __grid_constant__ TauParams p) {
    using PA = typename std::conditional<kRng == VXB_RNG_REF, Exact, Fused>::type;
    __shared__ double s_inv[kMaxPoisson + 1];
    __shared__ long long s_sum[4];
    for (int k = threadIdx.x; k <= kMaxPoisson; k += kTlBlock)
        s_inv[k] = k ? __ddiv_rn(1.0, static_cast<double>(k)) : 0.0;
    if (threadIdx.x < 4) s_sum[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * kTlBlock + threadIdx.x;
    long long sy = 0, sy2 = 0, sp = 0, it = 0;
    if (r < p.count) {
        const uint64_t path = p.first + r;
        const uint64_t key = stream_key(p.seed_hash, path);
        MM f{p.init[0], p.init[1], p.init[2], p.init[3]};
        MM c = f;
        double af[3], ac[3];
        if (p.level == 0) {
            for (uint64_t st = 0; st < p.n_fine; ++st) {
                f.prop(p.rate, af);
                double ua, ub, uc, ud;
                draw_pair<kRng>(p, key, path, 2 * st, ua, ub);      // positions 4s, 4s+1
                draw_pair<kRng>(p, key, path, 2 * st + 1, uc, ud);  // position 4s+2
                const int k0 = poisson_inv<PA>(__dmul_rn(af[0], p.tau), ua, s_inv, it);
                const int k1 = poisson_inv<PA>(__dmul_rn(af[1], p.tau), ub, s_inv, it);
                const int k2 = poisson_inv<PA>(__dmul_rn(af[2], p.tau), uc, s_inv, it);
                f.fire(k0, k1, k2);
            }
        } else {
            // On the fine levels (rate * tau ~ 1e-3) a step in which NOTHING fires is the
            // rule, and then neither state nor propensities change.  The bounds below
            // which a draw decides k = 0 (first shortcut of poisson_inv, see StepBits) are
            // therefore kept in registers and refreshed only after an event or a new
            // coarse step with a changed coarse state; a quiet step is the step's Philox
            // blocks, six 32-bit compares and ONE branch.  Same decisions as the oracle's
            // loop, bit for bit.
            uint32_t phase = 0;
            bool stale = true, coarse_moved = true;
            uint32_t bound_c[3], bound_r[3];  // leading word below it: the common / residual Poisson is 0
            for (uint64_t st = 0; st < p.n_fine; ++st) {
                if (phase == 0 && coarse_moved) {
                    c.prop(p.rate, ac);
                    coarse_moved = false;
                    stale = true;
                }
                if (++phase == p.refine) phase = 0;
                if (stale) {
                    f.prop(p.rate, af);
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const double mn = af[q] < ac[q] ? af[q] : ac[q];
                        const double mx = af[q] > ac[q] ? af[q] : ac[q];
                        bound_c[q] = StepBits<kRng>::bound(__dmul_rn(mn, p.tau), q);
                        bound_r[q] = StepBits<kRng>::bound(__dmul_rn(__dsub_rn(mx, mn), p.tau), q);
                    }
                    stale = false;
                }
                int kf[3], kc[3];
                // reaction q of fine step st owns Philox block 3 st + q: word 0 drives the
                // common Poisson, word 1 the residual one.  The three blocks are drawn
                // BEFORE the inversions: their round chains are independent and interleave
                // in one basic block, whereas the branches of an inversion fence off a
                // block drawn after it
                StepBits<kRng> bits;
                bits.draw(p, key, path, st);
                bool quiet = true;
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    quiet = quiet & (bits.top_common(q) < bound_c[q]) & (bits.top_residual(q) < bound_r[q]);
                if (quiet) continue;
                bits.complete(p);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const bool fine_larger = af[q] > ac[q];
                    const double mn = af[q] < ac[q] ? af[q] : ac[q];
                    const double mx = fine_larger ? af[q] : ac[q];
                    // a draw that is quiet by itself is 0 without being converted (the few lanes
                    // of a warp that are here rarely have more than one draw that is not)
                    int p1 = 0, pr = 0;
                    if (!(bits.top_common(q) < bound_c[q]))
                        p1 = poisson_inv<PA>(__dmul_rn(mn, p.tau), bits.common(q), s_inv, it);
                    // at most one of (af - m), (ac - m) is positive: one inversion serves both
                    if (!(bits.top_residual(q) < bound_r[q]))
                        pr = poisson_inv<PA>(__dmul_rn(__dsub_rn(mx, mn), p.tau), bits.residual(q), s_inv, it);
                    kf[q] = p1 + (fine_larger ? pr : 0);
                    kc[q] = p1 + (fine_larger ? 0 : pr);
                }
                f.fire(kf[0], kf[1], kf[2]);
                c.fire(kc[0], kc[1], kc[2]);
                // the bounds follow the fine state at once, the frozen coarse rates at the next coarse step
                stale = (kf[0] | kf[1] | kf[2]) != 0;
                coarse_moved = coarse_moved | ((kc[0] | kc[1] | kc[2]) != 0);
            }
        }
        const int32_t y = p.level == 0 ? f.p : f.p - c.p;
        if (p.y_out) p.y_out[r] = y;
        sy = y;
        sy2 = static_cast<long long>(y) * y;
        sp = f.p;
    }
    for (int o = 16; o; o >>= 1) {
        sy += __shfl_down_sync(0xffffffffu, sy, o);
        sy2 += __shfl_down_sync(0xffffffffu, sy2, o);
        sp += __shfl_down_sync(0xffffffffu, sp, o);
        it += __shfl_down_sync(0xffffffffu, it, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[0]), static_cast<unsigned long long>(sy));
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[1]), static_cast<unsigned long long>(sy2));
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[2]), static_cast<unsigned long long>(sp));
        atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[3]), static_cast<unsigned long long>(it));
    }
    __syncthreads();
    if (threadIdx.x < 4)
        atomicAdd(reinterpret_cast<unsigned long long*>(&p.sums[threadIdx.x]),
                  static_cast<unsigned long long>(s_sum[threadIdx.x]));
}

static uint64_t level_steps(const vxb_mlmc_cfg& cfg, uint32_t level) {
    require(cfg.tau0 > 0.0 && cfg.t_end > 0.0, "invalid-horizon", "need a positive horizon");
    uint64_t nf = static_cast<uint64_t>(std::llround(cfg.t_end / cfg.tau0));
    require(nf >= 1, "invalid-horizon", "need at least one step");
    for (uint32_t l = 0; l < level; ++l) nf *= cfg.refine;
    return nf;
}

void mlmc_level_device(vxb_ctx* ctx, const vxb_model& model, const vxb_mlmc_cfg& cfg,
                       uint32_t level, uint64_t first, uint64_t count, int64_t* sums_host,
                       int32_t* y_dev) {
    require(model.model == VXB_MODEL_MM_TAULEAP, "invalid-argument", "not the tau-leap model");
    require(cfg.refine >= 2 && level < cfg.levels, "invalid-argument", "bad level");
    TauParams p{};
    p.first = first;
    p.count = count;
    const uint64_t lv = level;
    p.seed_hash = splitmix64(vxb_derive_seed(cfg.seed, &lv, 1));
    p.fast = make_fast_keys(splitmix64(cfg.seed));
    require(model.rng == VXB_RNG_REF || model.rng == VXB_RNG_FAST, "invalid-argument", "bad rng mode");
    require(model.precision == VXB_F64 || (model.precision == VXB_F32 && model.rng == VXB_RNG_FAST),
            "invalid-argument", "the fp32 tau-leap instance exists for the throughput generator only");
    p.n_fine = level_steps(cfg, level);
    p.level = level;
    p.refine = cfg.refine;
    p.tau = cfg.t_end / static_cast<double>(p.n_fine);
    for (int k = 0; k < 3; ++k) p.rate[k] = model.consts[4 + k];
    for (int k = 0; k < 4; ++k) p.init[k] = static_cast<int32_t>(model.consts[k]);
    Scratch d_sums(ctx, 4 * sizeof(long long));
    VXB_CUDA(cudaMemsetAsync(d_sums.as<void>(), 0, 4 * sizeof(long long), ctx->stream));
    p.sums = d_sums.as<long long>();
    p.y_out = y_dev;
    if (count) {
        LaunchScope scope(ctx, VXB_K_TAULEAP);
        if (model.precision == VXB_F32)
            tauleap_f32_kernel<<<grid_for(count, kTlBlock), kTlBlock, 0, ctx->stream>>>(p);
        else if (model.rng == VXB_RNG_FAST)
            tauleap_kernel<VXB_RNG_FAST><<<grid_for(count, kTlBlock), kTlBlock, 0, ctx->stream>>>(p);
        else
            tauleap_kernel<VXB_RNG_REF><<<grid_for(count, kTlBlock), kTlBlock, 0, ctx->stream>>>(p);
        check_launch("tauleap_kernel");
    }
    long long h[4];
    VXB_CUDA(cudaMemcpyAsync(h, p.sums, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < 4; ++k) sums_host[k] = h[k];
}

}  // namespace vxb

using namespace vxb;

extern "C" int vxb_mlmc_level(vxb_ctx* ctx, const vxb_model* model, const vxb_mlmc_cfg* cfg,
                              uint32_t level, uint64_t first, uint64_t count, int64_t* sums,
                              int32_t* y_out) {
    return guarded([&] {
        use(ctx);
        require(model && cfg && sums, "invalid-argument", "null argument");
        Staged d_y(ctx, y_out, count * sizeof(int32_t), false, true);
        int64_t h[4];
        mlmc_level_device(ctx, *model, *cfg, level, first, count, h, d_y.as<int32_t>());
        if (is_device_pointer(sums))
            VXB_CUDA(cudaMemcpy(sums, h, sizeof(h), cudaMemcpyHostToDevice));
        else
            for (int k = 0; k < 4; ++k) sums[k] = h[k];
        d_y.finish();
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// Estimator (vxo_mlmc_tauleap): sum of the level means; variance = sum var_l / paths.
extern "C" int vxb_mlmc_tauleap(vxb_ctx* ctx, const vxb_model* model, const vxb_mlmc_cfg* cfg,
                                vxb_mlmc_out* out) {
    return guarded([&] {
        use(ctx);
        require(model && cfg && out, "invalid-argument", "null argument");
        require(cfg->paths >= 2, "insufficient-data", "variance needs at least two values");
        double est = 0.0, var = 0.0;
        uint64_t steps = level_steps(*cfg, 0);
        for (uint32_t l = 0; l < cfg->levels; ++l) {
            int64_t sums[4];
            mlmc_level_device(ctx, *model, *cfg, l, 0, cfg->paths, sums, nullptr);
            const double n = static_cast<double>(cfg->paths);
            const double mean = static_cast<double>(sums[0]) / n;
            const double v =
                (static_cast<double>(sums[1]) - static_cast<double>(sums[0]) * mean) / (n - 1.0);
            if (out->level_mean) out->level_mean[l] = mean;
            if (out->level_var) out->level_var[l] = v;
            if (out->level_cost)
                out->level_cost[l] =
                    static_cast<double>(l == 0 ? steps : steps + steps / cfg->refine);
            est += mean;
            var += v / n;
            steps *= cfg->refine;
        }
        out->estimate = est;
        out->std_error = std::sqrt(var);
    });
}
