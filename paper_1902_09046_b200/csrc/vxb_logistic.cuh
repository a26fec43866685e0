// vxb_logistic.cuh -- device side of the logistic-growth SDE simulator
// (kernels 2+3 of the hot path): keying, prior draw, Euler-Maruyama path with
// the summary/distance evaluation fused into the step loop.
//
// The model follows the pattern of toggle_switch.cpp: prior box map (:17-22),
// explicit operation order in the update (:46-62), variates addressed by a
// canonical layout in counter space (toggle_switch.hpp:52-57).  Relative to a
// row's base position: positions 0..2 are the prior uniforms, the counter is
// aligned to even (abc.cpp:53), and position 4+j is the normal of step j+1.
#pragma once

#include <cmath>

#include "vxb_rng.cuh"

#define VXB_MAX_SUMMARY 128

namespace vxb {

enum { kKeyParticle = 0, kKeyWorker = 1, kKeyFixed = 2 };

struct Keying {
    int mode;
    uint64_t seed_hash;    // splitmix64(seed)
    uint64_t fixed_key;    // kKeyFixed
    uint64_t fixed_pos;    // kKeyFixed
    uint64_t base_blocks;  // worker mode: blocks per worker (blocked.cpp:46-47)
    uint64_t extra_blocks;
    uint64_t width;       // V
    uint64_t row_stride;  // stream positions one row consumes
    FastKeys fast;        // VXB_RNG_FAST: Philox4x32 round keys of the seed
};

struct LogisticModel {
    uint32_t steps, obs_stride, n_obs;
    double dt, sqdt, x0;
    double lo[3], hi[3];
};

// Stream key and base counter position of global row `row`.
__device__ __forceinline__ void locate_row(const Keying& k, uint64_t row, uint64_t& key,
                                           uint64_t& base) {
    if (k.mode == kKeyParticle) {
        key = stream_key(k.seed_hash, row);
        base = 0;
    } else if (k.mode == kKeyWorker) {
        // inverse of partition(n, P, V) (blocked.cpp:34-63): the first `extra`
        // workers own base+1 blocks of V rows, the rest own base blocks.
        const uint64_t b = row / k.width;
        const uint64_t big = k.extra_blocks * (k.base_blocks + 1);
        uint64_t w, first_block;
        if (b < big) {
            w = b / (k.base_blocks + 1);
            first_block = w * (k.base_blocks + 1);
        } else {
            w = k.extra_blocks + (b - big) / k.base_blocks;
            first_block = big + (w - k.extra_blocks) * k.base_blocks;
        }
        key = stream_key(k.seed_hash, w);
        base = (row - first_block * k.width) * k.row_stride;
    } else {
        key = k.fixed_key;
        base = k.fixed_pos;
    }
}

// Prior draw (reference RNG): three uniforms at positions base..base+2 mapped
// onto the box as lo + u*(hi-lo).  base is even.
__device__ __forceinline__ void draw_prior_ref(const LogisticModel& m, uint64_t key, uint64_t base,
                                               double* theta) {
    const Words a = philox2x64(key, base >> 1);
    const Words b = philox2x64(key, (base >> 1) + 1);
    const double u0 = to_unit(a.w0), u1 = to_unit(a.w1), u2 = to_unit(b.w0);
    theta[0] = __dadd_rn(m.lo[0], __dmul_rn(u0, __dsub_rn(m.hi[0], m.lo[0])));
    theta[1] = __dadd_rn(m.lo[1], __dmul_rn(u1, __dsub_rn(m.hi[1], m.lo[1])));
    theta[2] = __dadd_rn(m.lo[2], __dmul_rn(u2, __dsub_rn(m.hi[2], m.lo[2])));
}
// Prior draw of the throughput generator: counter (0..1, kDomPrior, row).
__device__ __forceinline__ void draw_prior_fast(const LogisticModel& m, const FastKeys& fk,
                                                uint64_t row, double* theta) {
    const uint32_t rl = static_cast<uint32_t>(row), rh = static_cast<uint32_t>(row >> 32);
    const Words32 a = philox4x32(fk, 0u, kDomPrior, rl, rh);
    const Words32 b = philox4x32(fk, 1u, kDomPrior, rl, rh);
    const double u0 = fast_unit(a.a, a.b), u1 = fast_unit(a.c, a.d), u2 = fast_unit(b.a, b.b);
    theta[0] = m.lo[0] + u0 * (m.hi[0] - m.lo[0]);
    theta[1] = m.lo[1] + u1 * (m.hi[1] - m.lo[1]);
    theta[2] = m.lo[2] + u2 * (m.hi[2] - m.lo[2]);
}

// ------------------------------------------------------------ noise sources
// next(z) yields the next kBatch standard normals of the row.
//
// The counter-based generators run ONE BATCH AHEAD: next() turns the random bits
// drawn during the previous call into normals and draws the bits of the
// following batch.  The two halves are independent, so the integer Philox
// rounds (FMA-heavy/ALU pipes) and the FP64 Box-Muller + SDE steps of a warp
// sit in the same basic block and are interleaved by the instruction
// scheduler.  Without this every warp alternates between an all-integer and an
// all-FP64 phase, the warps of an SM sub-partition fall into step, and the
// pipes are used one after the other instead of side by side (measured: the
// step time was the SUM of the integer and FP64 pipe times).
template <class Real>
struct RefNoise {  // bit-identical to RngStream::fill_gaussian (rng.cpp:142-164)
    static constexpr int kBatch = 2;
    uint64_t key, pair;
    Words ahead;
    __device__ __forceinline__ RefNoise(uint64_t key_, uint64_t first_pair)
        : key(key_), pair(first_pair + 1), ahead(philox2x64(key_, first_pair)) {}
    __device__ __forceinline__ void next(Real* z) {
        const Words w = ahead;
        ahead = philox2x64(key, pair++);
        double ze, zo;
        box_muller<Exact>(w, ze, zo);
        z[0] = static_cast<Real>(ze);
        z[1] = static_cast<Real>(zo);
    }
};
struct FastNoise64 {
    // eight normals from three Philox blocks (fast_box_muller_x4); batch q of the
    // row uses blocks 3q, 3q+1, 3q+2 of its (domain, row) counter space
    static constexpr int kBatch = 8;
    const FastKeys& fk;
    const double2* tbl;
    uint32_t row_lo, row_hi, block, domain;
    Words32 ahead0, ahead1, ahead2;
    __device__ __forceinline__ FastNoise64(const FastKeys& fk_, const double2* tbl_, uint32_t rl,
                                           uint32_t rh, uint32_t first_block,
                                           uint32_t domain_ = kDomNoise)
        : fk(fk_), tbl(tbl_), row_lo(rl), row_hi(rh), block(first_block), domain(domain_) {
        draw();
    }
    __device__ __forceinline__ void draw() {
        ahead0 = philox4x32(fk, block, domain, row_lo, row_hi);
        ahead1 = philox4x32(fk, block + 1, domain, row_lo, row_hi);
        ahead2 = philox4x32(fk, block + 2, domain, row_lo, row_hi);
        block += 3;
    }
    __device__ __forceinline__ void next(double* z) {
        const Words32 u = ahead0, v = ahead1, w = ahead2;
        draw();
        fast_box_muller_x4(u, v, w, tbl, z);
    }
};
struct FastNoise32 {
    // sixteen normals from three Philox blocks (box_muller_f32_x8)
    static constexpr int kBatch = 16;
    const FastKeys& fk;
    uint32_t row_lo, row_hi, block;
    Words32 ahead0, ahead1, ahead2;
    __device__ __forceinline__ FastNoise32(const FastKeys& fk_, uint32_t rl, uint32_t rh,
                                           uint32_t first_block)
        : fk(fk_), row_lo(rl), row_hi(rh), block(first_block) {
        draw();
    }
    __device__ __forceinline__ void draw() {
        ahead0 = philox4x32(fk, block, kDomNoise, row_lo, row_hi);
        ahead1 = philox4x32(fk, block + 1, kDomNoise, row_lo, row_hi);
        ahead2 = philox4x32(fk, block + 2, kDomNoise, row_lo, row_hi);
        block += 3;
    }
    __device__ __forceinline__ void next(float* z) {
        const Words32 u = ahead0, v = ahead1, w = ahead2;
        draw();
        box_muller_f32_x8(u, v, w, z);
    }
};
template <class Real>
struct ExternalNoise {
    static constexpr int kBatch = 2;
    const Real* row;
    uint32_t j, steps;
    __device__ __forceinline__ void next(Real* z) {
        z[0] = j < steps ? row[j] : Real(0);
        z[1] = j + 1 < steps ? row[j + 1] : Real(0);
        j += 2;
    }
};

// One Euler-Maruyama step:  x + (a x)(1 - x/K) + (c x) z  with a = r dt,
// c = sigma sqrt(dt), 1/K hoisted; evaluated ((x + drift) + diffusion) in the
// exact mode; four FMAs in the FMA parity mode; fp64 throughput mode: the same
// polynomial as x (A + B x + c z) with A = 1 + a and B = -a/K hoisted (two FMAs
// and a multiply).
template <class Real, class A>
__device__ __forceinline__ Real logistic_step(Real x, Real a, Real c, Real inv_k, Real z, Real a1,
                                              Real bk) {
    if (A::kExact) {
        const Real drift = A::mul(A::mul(a, x), A::sub(Real(1), A::mul(x, inv_k)));
        const Real diff = A::mul(A::mul(c, x), z);
        return A::add(A::add(x, drift), diff);
    } else if (A::kCompactStep) {
        return x * A::mad(c, z, A::mad(bk, x, a1));
    } else {
        // x (1 + a (1 - x/K) + c z): same polynomial, four FMAs
        const Real sat = A::mad(-x, inv_k, Real(1));
        const Real g = A::mad(c, z, A::mul(a, sat));
        return A::mad(x, g, x);
    }
}

// Runs observations [obs_begin, obs_end) of one path: steps obs_begin * stride up to
// obs_end * stride (up to the last step when obs_end == n_obs), from state x and partial
// squared distance ss, both updated in place.  Summaries are handed to `emit(k, value)` as
// they are produced, so the trajectory never leaves registers; the squared distance
// accumulates left to right in observation order (abc.cpp:16-24).  `bad` is set when an
// observed state is not finite.  The noise source must stand at the batch that holds step
// obs_begin * stride.
// ss_bound (early rejection, vxb_abc_reject with VXB_OPT_EARLY_REJECT; +inf otherwise): the
// squared distance only grows, so a row whose partial sum exceeds the bound can no longer
// come out with rho <= epsilon; the segment stops at the first observation at which that
// holds for every row of the warp (observations fall on the same step in every row).
template <class Real, class A, class Noise, class Emit>
__device__ __forceinline__ void logistic_segment(const LogisticModel& m, const double* theta,
                                                 const double* __restrict__ observed, Noise& noise,
                                                 Emit&& emit, bool& bad, Real ss_bound,
                                                 uint32_t obs_begin, uint32_t obs_end, Real& x_io,
                                                 Real& ss_io) {
    const Real r = static_cast<Real>(theta[0]);
    const Real k = static_cast<Real>(theta[1]);
    const Real sigma = static_cast<Real>(theta[2]);
    const Real a = Exact::mul(r, static_cast<Real>(m.dt));
    const Real c = Exact::mul(sigma, static_cast<Real>(m.sqdt));
    const Real inv_k = Exact::div(Real(1), k);
    const Real a1 = Real(1) + a, bk = -a * inv_k;  // throughput-mode form of the step
    Real x = x_io;
    Real ss = ss_io;
    uint32_t next = obs_begin, since = 0;
    bool stop = false;
    const bool early = isfinite(ss_bound);
    bad = false;
    constexpr uint32_t kB = Noise::kBatch;
    const uint32_t stride = m.obs_stride;
    const uint32_t steps = obs_end >= m.n_obs ? m.steps : obs_end * stride;
    auto observe = [&] {
        since = 0;
        if (next < m.n_obs) {
            const Real d = A::sub(x, static_cast<Real>(observed[next]));
            ss = A::mad(d, d, ss);
            bad = bad || !isfinite(x);
            emit(next, x);
            ++next;
            if (early) stop = __all_sync(__activemask(), !(ss <= ss_bound)) != 0;
        }
    };
    if (stride % kB == 0 && m.steps == stride * m.n_obs) {
        // observation stride a multiple of the batch (e.g. the exact instance, batch 2,
        // on the BASELINE grid of 100): whole batches between observations, no per-step
        // bookkeeping.  The throughput instances on the BASELINE grid (100 = 12 x 8 + 4 =
        // 6 x 16 + 4) take the general loop below -- measured on B200 it is no slower
        // (fp64: 70.8 ms per 2e7 rows at stride 100 against 71.9-72.3 ms at strides 80 /
        // 200 / 400, which come through here; profiles/r2_stride_probe.json)
        const uint32_t per = stride / kB;
        const uint32_t last = obs_end < m.n_obs ? obs_end : m.n_obs;
        for (uint32_t o = obs_begin; o < last; ++o) {
            for (uint32_t i = 0; i < per; ++i) {
                Real z[kB];
                noise.next(z);
#pragma unroll
                for (uint32_t q = 0; q < kB; ++q) x = logistic_step<Real, A>(x, a, c, inv_k, z[q], a1, bk);
            }
            observe();
            if (stop) break;
        }
        x_io = x;
        ss_io = ss;
        return;
    }
    uint32_t j = obs_begin * stride;
    if (const uint32_t skip = j % kB) {
        // a segment that begins inside a noise batch (the source stands at the batch that
        // holds step j): the first skip normals belong to the previous segment
        Real z[kB];
        noise.next(z);
        for (uint32_t q = skip; q < kB && j < steps; ++q, ++j) {
            x = logistic_step<Real, A>(x, a, c, inv_k, z[q], a1, bk);
            if (++since == stride) observe();
        }
    }
    for (; j + kB <= steps && !stop; j += kB) {
        Real z[kB];
        noise.next(z);
        if (since + kB < stride) {  // no observation inside this batch (warp-uniform)
#pragma unroll
            for (uint32_t q = 0; q < kB; ++q) x = logistic_step<Real, A>(x, a, c, inv_k, z[q], a1, bk);
            since += kB;
        } else {
#pragma unroll
            for (uint32_t q = 0; q < kB; ++q) {
                x = logistic_step<Real, A>(x, a, c, inv_k, z[q], a1, bk);
                if (++since == stride) observe();
            }
        }
    }
    if (j < steps && !stop) {  // ragged tail: fewer than kBatch steps left
        Real z[kB];
        noise.next(z);
        for (uint32_t q = 0; j + q < steps; ++q) {
            x = logistic_step<Real, A>(x, a, c, inv_k, z[q], a1, bk);
            if (++since == stride) observe();
        }
    }
    x_io = x;
    ss_io = ss;
}

// Runs one whole path; returns rho.
template <class Real, class A, class Noise, class Emit>
__device__ __forceinline__ Real logistic_path(const LogisticModel& m, const double* theta,
                                              const double* __restrict__ observed, Noise& noise,
                                              Emit&& emit, bool& bad) {
    Real x = static_cast<Real>(m.x0), ss = 0;
    logistic_segment<Real, A>(m, theta, observed, noise, emit, bad, static_cast<Real>(INFINITY), 0u, m.n_obs, x, ss);
    return Exact::sqrt(ss);
}

}  // namespace vxb
