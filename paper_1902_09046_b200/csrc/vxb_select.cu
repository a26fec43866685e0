// vxb_select.cu -- epsilon selection and accepted-row compaction (kernel 4).
//
// Replaces the single-threaded tail of the reference ABC sampler,
// abc::select_epsilon (abc.cpp:75-97): std::sort of all discrepancies, type-7
// quantile (numeric.cpp:20-30), ceil(q n) guard, ascending scan for rho <= eps.
// On the device no sort is needed:
//   * the two or three order statistics the quantile rule reads are found by a
//     most-significant-digit radix select (11-bit digits, shared-memory
//     histograms, digit choice on the device so the passes queue without host
//     round trips) -- exact, so epsilon is bit-identical to the sorted answer;
//   * accepted rows are compacted by warp ballot + block prefix sums with the
//     block offsets taken from a scan (not from atomics), which yields the
//     ascending row order of abc.cpp:93-95 deterministically.
// Both are HBM-bound streaming passes over rho (8 B/row per pass).

#include <cmath>
#include <limits>

#include "vxb_internal.cuh"

namespace vxb {

constexpr int kDigitBits = 11;
constexpr int kBins = 1 << kDigitBits;
constexpr int kMaxRanks = 4;
constexpr int kSelBlock = 256;
constexpr int kSelItems = 16;  // rows per thread per block tile

// Monotone map of a real to an unsigned key (total order of the reals).
__device__ __forceinline__ uint64_t order_key(double v) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ uint64_t order_key(float v) {
    const uint32_t b = __float_as_uint(v);
    const uint32_t k = (b >> 31) ? ~b : (b | 0x80000000u);
    return static_cast<uint64_t>(k) << 32;  // high half so the digit schedule is shared
}
__host__ inline double key_to_double(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
    double v;
    memcpy(&v, &b, 8);
    return v;
}
__host__ inline float key_to_float(uint64_t k64) {
    const uint32_t k = static_cast<uint32_t>(k64 >> 32);
    const uint32_t b = (k >> 31) ? (k & 0x7FFFFFFFu) : ~k;
    float v;
    memcpy(&v, &b, 4);
    return v;
}

// flag and value are loaded unconditionally (two independent loads, no
// short-circuit between them)
template <class Real>
__device__ __forceinline__ bool row_valid(const Real* rho, const uint8_t* failed, uint64_t i,
                                          Real& value) {
    const uint8_t flag = failed ? __ldg(failed + i) : uint8_t(0);
    value = __ldg(rho + i);
    return (flag == 0) & !isnan(value);
}

struct SelectState {
    uint64_t prefix[kMaxRanks];     // digits fixed so far (high bits)
    uint64_t remaining[kMaxRanks];  // rank inside the current bucket
    uint64_t n_valid;
};

// out[0]: valid rows; out[1]: rows excluded by their flag alone (flag set, value not
// NaN).  When out[1] is zero the flags carry no information beyond the NaNs and the
// digit passes need not read them (8 instead of 9 bytes per row).
template <class Real>
__global__ void __launch_bounds__(256, 8)
count_valid_kernel(const Real* __restrict__ rho, const uint8_t* __restrict__ failed, uint64_t n,
                   unsigned long long* out) {
    uint64_t c = 0, only_flag = 0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t first = 0;
    if (sizeof(Real) == 8 && failed && (reinterpret_cast<uintptr_t>(rho) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(failed) & 3) == 0) {
        // aligned fp64 rows with flags: four rows per step as two 16-byte loads and one
        // 4-byte load of their flags (a byte load per row wastes most of its sector)
        const double2* r2 = reinterpret_cast<const double2*>(rho);
        const uint32_t* f4 = reinterpret_cast<const uint32_t*>(failed);
        const uint64_t groups = n / 4;
        constexpr int kInFlight = 4;
        for (uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g0 < groups;
             g0 += kInFlight * stride) {
            double2 a[kInFlight], b[kInFlight];
            uint32_t f[kInFlight];
            bool in[kInFlight];
#pragma unroll
            for (int u = 0; u < kInFlight; ++u) {
                const uint64_t g = g0 + static_cast<uint64_t>(u) * stride;
                in[u] = g < groups;
                const uint64_t gg = in[u] ? g : 0;
                a[u] = __ldg(r2 + 2 * gg);
                b[u] = __ldg(r2 + 2 * gg + 1);
                f[u] = __ldg(f4 + gg);
            }
#pragma unroll
            for (int u = 0; u < kInFlight; ++u) {
                const double v[4] = {a[u].x, a[u].y, b[u].x, b[u].y};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const bool flagged = (f[u] >> (8 * e)) & 0xFFu;
                    const bool number = !isnan(v[e]);
                    c += (in[u] && number && !flagged) ? 1 : 0;
                    only_flag += (in[u] && number && flagged) ? 1 : 0;
                }
            }
        }
        first = groups * 4;
    }
    for (uint64_t i0 = first + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n;
         i0 += 16 * stride) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {  // sixteen independent loads per trip
            const uint64_t i = i0 + static_cast<uint64_t>(u) * stride;
            Real v = Real(0);
            const bool inside = i < n;
            const bool ok = inside && row_valid(rho, failed, i, v);
            c += ok ? 1 : 0;
            only_flag += (inside && !ok && !isnan(v)) ? 1 : 0;
        }
    }
    for (int o = 16; o; o >>= 1) {
        c += __shfl_down_sync(0xffffffffu, c, o);
        only_flag += __shfl_down_sync(0xffffffffu, only_flag, o);
    }
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, static_cast<unsigned long long>(c));
    if ((threadIdx.x & 31) == 0 && only_flag) atomicAdd(out + 1, static_cast<unsigned long long>(only_flag));
}

#ifndef VXB_HIST_INFLIGHT
#define VXB_HIST_INFLIGHT 4
#endif
// 16-byte vectors of the row type (the flag-free stream reads rho through them)
template <class Real> struct RowVec;
template <> struct RowVec<double> {
    using type = double2;
    static constexpr int kLanes = 2;
    static __device__ __forceinline__ double at(const double2& v, int e) { return e ? v.y : v.x; }
};
template <> struct RowVec<float> {
    using type = float4;
    static constexpr int kLanes = 4;
    static __device__ __forceinline__ float at(const float4& v, int e) {
        return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
    }
};

template <int kDistinct>
__device__ __forceinline__ void hist_one(uint64_t key, bool ok, int shift, bool all, uint64_t limit,
                                         const uint64_t* pref, unsigned int* sh) {
#pragma unroll
    for (int a = 0; a < kDistinct; ++a) {
        const uint64_t x = key ^ pref[a];
        if (ok && (all || x < limit)) atomicAdd(&sh[a * kBins + static_cast<unsigned>(x >> shift)], 1u);
    }
}

// the row stream of one digit pass for kDistinct different prefixes
template <class Real, bool kFlags, int kDistinct>
__device__ __forceinline__ void hist_rows(const Real* __restrict__ rho, const uint8_t* __restrict__ failed,
                                          uint64_t n, int shift, bool all, uint64_t limit,
                                          const uint64_t* pref, unsigned int* sh) {
    constexpr int kInFlight = VXB_HIST_INFLIGHT;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kSelBlock;
    uint64_t first = 0;  // rows below `first` were taken by the vector loop
    if (!kFlags && (reinterpret_cast<uintptr_t>(rho) & 15) == 0) {
        // no flags to read and an aligned base: 16-byte loads, half (a quarter) of the
        // load instructions and address arithmetic per row
        using V = RowVec<Real>;
        const typename V::type* r = reinterpret_cast<const typename V::type*>(rho);
        const uint64_t nv = n / V::kLanes;
        constexpr int kVecInFlight = kInFlight > 1 ? kInFlight / 2 : 1;
        for (uint64_t j0 = static_cast<uint64_t>(blockIdx.x) * kSelBlock + threadIdx.x; j0 < nv;
             j0 += stride * kVecInFlight) {
            typename V::type v[kVecInFlight];
            bool in[kVecInFlight];
#pragma unroll
            for (int u = 0; u < kVecInFlight; ++u) {
                const uint64_t j = j0 + static_cast<uint64_t>(u) * stride;
                in[u] = j < nv;
                v[u] = __ldg(r + (in[u] ? j : 0));
            }
#pragma unroll
            for (int u = 0; u < kVecInFlight; ++u)
#pragma unroll
                for (int e = 0; e < V::kLanes; ++e) {
                    const Real x = V::at(v[u], e);
                    hist_one<kDistinct>(order_key(x), in[u] & !isnan(x), shift, all, limit, pref, sh);
                }
        }
        first = nv * V::kLanes;
    }
    for (uint64_t i0 = first + static_cast<uint64_t>(blockIdx.x) * kSelBlock + threadIdx.x; i0 < n;
         i0 += stride * kInFlight) {
        Real v[kInFlight];
        bool ok[kInFlight];
#pragma unroll
        for (int u = 0; u < kInFlight; ++u) {  // the loads of a trip are issued together
            const uint64_t i = i0 + static_cast<uint64_t>(u) * stride;
            const bool inside = i < n;
            v[u] = inside ? __ldg(rho + i) : Real(0);
            const uint8_t flag = (kFlags && inside) ? __ldg(failed + i) : uint8_t(0);
            ok[u] = inside & (flag == 0) & !isnan(v[u]);
        }
#pragma unroll
        for (int u = 0; u < kInFlight; ++u)
            hist_one<kDistinct>(order_key(v[u]), ok[u], shift, all, limit, pref, sh);
    }
}

#ifndef VXB_HIST_CTAS
#define VXB_HIST_CTAS 8  // swept 4 / 6 / 8 CTAs per SM at 1e8 rows: 3.05 / 2.24 / 1.98 ms for the six passes
#endif
template <class Real, bool kFlags>
__global__ void __launch_bounds__(kSelBlock, VXB_HIST_CTAS)
radix_hist_kernel(const Real* __restrict__ rho, const uint8_t* __restrict__ failed, uint64_t n,
                  int shift, int bits, int n_ranks, const SelectState* __restrict__ state,
                  unsigned int* __restrict__ hist /* n_ranks x kBins */) {
    extern __shared__ unsigned int sh[];  // n_ranks x kBins
    for (int i = threadIdx.x; i < n_ranks * kBins; i += kSelBlock) sh[i] = 0;
    __syncthreads();
    const int hi_shift = shift + bits;  // bits above the current digit
    // x < limit  <=>  the digits above the current one equal the prefix
    const bool all = hi_shift >= 64;
    const uint64_t limit = all ? ~0ull : (1ull << hi_shift);
    // distinct prefixes among the ranks, compacted (warp-uniform bookkeeping)
    uint64_t pref[kMaxRanks];  // distinct prefix a
    int slot[kMaxRanks];       // rank q counts in histogram slot[q]
    int n_distinct = 0;
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q) pref[q] = 0;
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q) {
        slot[q] = 0;
        if (q >= n_ranks) continue;
        const uint64_t mine = state->prefix[q];
        int found = -1;
#pragma unroll
        for (int a = 0; a < kMaxRanks; ++a)
            if (a < n_distinct && pref[a] == mine && found < 0) found = a;
        if (found < 0) {
            found = n_distinct;
#pragma unroll
            for (int a = 0; a < kMaxRanks; ++a)
                if (a == n_distinct) pref[a] = mine;
            ++n_distinct;
        }
        slot[q] = found;
    }
    switch (n_distinct) {
        case 1: hist_rows<Real, kFlags, 1>(rho, failed, n, shift, all, limit, pref, sh); break;
        case 2: hist_rows<Real, kFlags, 2>(rho, failed, n, shift, all, limit, pref, sh); break;
        case 3: hist_rows<Real, kFlags, 3>(rho, failed, n, shift, all, limit, pref, sh); break;
        default: hist_rows<Real, kFlags, 4>(rho, failed, n, shift, all, limit, pref, sh); break;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kMaxRanks; ++q) {
        if (q >= n_ranks) break;
        for (int i = threadIdx.x; i < kBins; i += kSelBlock) {
            const unsigned int c = sh[slot[q] * kBins + i];
            if (c) atomicAdd(&hist[q * kBins + i], c);
        }
    }
}

// Picks, for every rank, the bucket holding it; clears the histogram.
__global__ void radix_pick_kernel(int shift, int bits, int n_ranks, SelectState* state,
                                  unsigned int* hist) {
    const int q = blockIdx.x;
    if (q >= n_ranks) return;
    __shared__ unsigned int bins[kBins];
    const int nb = 1 << bits;
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) {
        bins[i] = i < nb ? hist[q * kBins + i] : 0;
        hist[q * kBins + i] = 0;
    }
    __syncthreads();
    // block-wide exclusive scan: 256 threads x 8 consecutive bins
    constexpr int kPer = kBins / 256;
    __shared__ unsigned long long warp_tot[8];
    unsigned long long local = 0;
    for (int j = 0; j < kPer; ++j) local += bins[threadIdx.x * kPer + j];
    unsigned long long incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((threadIdx.x & 31) >= o) incl += t;
    }
    if ((threadIdx.x & 31) == 31) warp_tot[threadIdx.x >> 5] = incl;
    __syncthreads();
    unsigned long long before = incl - local;
    for (int w = 0; w < static_cast<int>(threadIdx.x >> 5); ++w) before += warp_tot[w];
    // exactly one thread owns the bucket that holds rank k (k < total by contract)
    const unsigned long long k = state->remaining[q];
    __syncthreads();
    if (k >= before && k < before + local) {
        unsigned long long run = before;
        int chosen = threadIdx.x * kPer;
        for (int j = 0; j < kPer; ++j) {
            const unsigned c = bins[threadIdx.x * kPer + j];
            if (k < run + c) {
                chosen = threadIdx.x * kPer + j;
                break;
            }
            run += c;
        }
        state->remaining[q] = k - run;
        state->prefix[q] |= static_cast<uint64_t>(chosen) << shift;
    }
}

// ---- compaction: tile = kSelBlock*kSelItems consecutive rows per block ----
template <class Real>
__device__ __forceinline__ bool row_accepted(const Real* rho, const uint8_t* failed, uint64_t i,
                                             uint64_t n, double eps) {
    // compared in double so that an fp32 rho is tested against the unrounded
    // epsilon, as the host rule does; NaN compares false.  Both loads are issued
    // unconditionally (no short-circuit between them): a streaming pass wants every
    // load of a thread in flight at once, not a flag load followed by a dependent
    // value load.
    const bool inside = i < n;
    const uint8_t flag = (inside && failed) ? __ldg(failed + i) : uint8_t(0);
    const Real value = inside ? __ldg(rho + i) : Real(0);
    return inside & (flag == 0) & (static_cast<double>(value) <= eps);
}

// Row of (warp, bit s, lane) inside a block tile: every warp owns 32*kSelItems
// consecutive rows and sweeps them in kSelItems/4 groups of 128 rows; in a group a lane
// owns FOUR consecutive rows (bits 4g .. 4g+3), so that aligned fp64 rows are read as
// two 16-byte loads and their flags as one 4-byte load (a byte load per row wastes most
// of its 32-byte sector).  Ascending row order inside a warp is (group, lane, bit).
static_assert(kSelItems % 4 == 0, "rows are taken four at a time");
__device__ __forceinline__ uint64_t tile_row(uint64_t tile0, unsigned warp, int s, unsigned lane) {
    return tile0 + static_cast<uint64_t>(warp) * (32 * kSelItems) + static_cast<uint64_t>(s >> 2) * 128 +
           lane * 4 + (s & 3);
}

// Pass 1 (the only pass over rho): per-block accept counts, and every thread's
// accept flags (bit s = row tile_row(.., s, lane); one bit per row, n/8 bytes) so that
// the write pass never has to read the 8-9 B/row again.
template <class Real>
__global__ void __launch_bounds__(kSelBlock, 8)
accept_count_kernel(const Real* __restrict__ rho, const uint8_t* __restrict__ failed, uint64_t n,
                    double eps, unsigned int* __restrict__ block_counts,
                    unsigned short* __restrict__ thread_flags /* n_blocks x kSelBlock, optional */) {
    static_assert(kSelItems <= 16, "flags are stored as 16 bits per thread");
    const uint64_t tile0 = static_cast<uint64_t>(blockIdx.x) * kSelBlock * kSelItems;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned flags = 0;
    const bool whole = tile0 + static_cast<uint64_t>(kSelBlock) * kSelItems <= n;
    if (sizeof(Real) == 8 && whole && (reinterpret_cast<uintptr_t>(rho) & 15) == 0 &&
        (!failed || (reinterpret_cast<uintptr_t>(failed) & 3) == 0)) {
        // whole tile, aligned fp64: all 16-byte loads (and the 4-byte flag words) of the
        // thread are issued before anything depends on them
        constexpr int kGroups = kSelItems / 4;
        double2 a[kGroups], b[kGroups];
        uint32_t f[kGroups];
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
            const uint64_t row = tile_row(tile0, warp, 4 * g, lane);
            const double2* src = reinterpret_cast<const double2*>(rho + row);
            a[g] = __ldg(src);
            b[g] = __ldg(src + 1);
            f[g] = failed ? __ldg(reinterpret_cast<const uint32_t*>(failed + row)) : 0u;
        }
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
            const double v[4] = {static_cast<double>(a[g].x), static_cast<double>(a[g].y),
                                 static_cast<double>(b[g].x), static_cast<double>(b[g].y)};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                flags |= ((((f[g] >> (8 * e)) & 0xFFu) == 0) & (v[e] <= eps) ? 1u : 0u) << (4 * g + e);
        }
    } else {
#pragma unroll
        for (int s = 0; s < kSelItems; ++s)  // all loads of the thread in flight together
            flags |= (row_accepted(rho, failed, tile_row(tile0, warp, s, lane), n, eps) ? 1u : 0u) << s;
    }
    if (thread_flags)
        thread_flags[static_cast<uint64_t>(blockIdx.x) * kSelBlock + threadIdx.x] =
            static_cast<unsigned short>(flags);
    unsigned c = __popc(flags);
    for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    __shared__ unsigned int warp_sum[kSelBlock / 32];
    if (lane == 0) warp_sum[warp] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = 0;
        for (int w = 0; w < kSelBlock / 32; ++w) t += warp_sum[w];
        block_counts[blockIdx.x] = t;
    }
}

// Exclusive scan of the block counts (one CTA, serial over chunks of 1024).
__global__ void __launch_bounds__(1024)
scan_blocks_kernel(const unsigned int* __restrict__ counts, uint64_t n_blocks,
                   unsigned long long* __restrict__ offsets, unsigned long long* total) {
    __shared__ unsigned long long warp_tot[32];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t c0 = 0; c0 < n_blocks; c0 += 1024) {
        const uint64_t i = c0 + threadIdx.x;
        const unsigned long long v = i < n_blocks ? counts[i] : 0;
        unsigned long long incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
            if ((threadIdx.x & 31) >= o) incl += t;
        }
        if ((threadIdx.x & 31) == 31) warp_tot[threadIdx.x >> 5] = incl;
        __syncthreads();
        if (threadIdx.x < 32) {
            unsigned long long w = warp_tot[threadIdx.x];
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long t = __shfl_up_sync(0xffffffffu, w, o);
                if (threadIdx.x >= o) w += t;
            }
            warp_tot[threadIdx.x] = w;  // inclusive over warps
        }
        __syncthreads();
        const unsigned long long warp_off = (threadIdx.x >> 5) ? warp_tot[(threadIdx.x >> 5) - 1] : 0;
        const unsigned long long base = carry;
        if (i < n_blocks) offsets[i] = base + warp_off + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry = base + warp_off + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

// Pass 2: ascending indices of the accepted rows from the stored flags (n/8 bytes
// read) and the scanned block offsets: the ballots of a group's four bits give the
// order (group, lane, bit) inside a warp.
__global__ void __launch_bounds__(kSelBlock)
accept_write_kernel(const unsigned short* __restrict__ thread_flags,
                    const unsigned long long* __restrict__ offsets, uint64_t index_base, uint64_t cap,
                    uint64_t* __restrict__ idx) {
    __shared__ unsigned int warp_cnt[kSelBlock / 32];
    const uint64_t tile0 = static_cast<uint64_t>(blockIdx.x) * kSelBlock * kSelItems;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned flags = thread_flags[static_cast<uint64_t>(blockIdx.x) * kSelBlock + threadIdx.x];
    unsigned mine = __popc(flags);
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0) warp_cnt[warp] = mine;
    __syncthreads();
    if (mine == 0) return;  // nothing accepted in this warp's rows (the common case)
    unsigned long long dst = offsets[blockIdx.x];
    for (unsigned w = 0; w < warp; ++w) dst += warp_cnt[w];
    const unsigned below = (1u << lane) - 1;
#pragma unroll
    for (int g = 0; g < kSelItems / 4; ++g) {  // ascending rows: (group, lane, bit)
        const unsigned nib = (flags >> (4 * g)) & 0xFu;
        unsigned before = 0, all = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const unsigned ballot = __ballot_sync(0xffffffffu, (nib >> e) & 1u);
            before += __popc(ballot & below);
            all += __popc(ballot);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if ((nib >> e) & 1u) {
                const unsigned long long at = dst + before + __popc(nib & ((1u << e) - 1));
                if (at < cap) idx[at] = tile_row(tile0, warp, 4 * g + e, lane) + index_base;
            }
        dst += all;
    }
}

template <class Real>
void order_statistics_device(vxb_ctx* ctx, const Real* rho, const uint8_t* failed, uint64_t n,
                             const uint64_t* ranks, int n_ranks, double* values, vxb_comm* comm) {
    // comm (several ranks, each holding n rows of one long vector): the per-digit
    // histograms are integer counts, so their all-reduce between the counting and the
    // picking kernel makes every rank walk the digits of the WHOLE vector's order
    // statistics -- 6 (fp64) or 3 (fp32) all-reduces of n_ranks x 2048 counters, and no
    // distance ever leaves its device.  n may be zero on a rank.
    const bool shared = comm != nullptr;  // a one-rank communicator runs its collectives too (tests)
    require(n_ranks >= 1 && n_ranks <= kMaxRanks, "invalid-argument", "too many ranks");
    Scratch d_state(ctx, sizeof(SelectState));
    Scratch d_hist(ctx, sizeof(unsigned int) * kMaxRanks * kBins);
    SelectState init{};
    for (int q = 0; q < n_ranks; ++q) init.remaining[q] = ranks[q];
    VXB_CUDA(cudaMemcpyAsync(d_state.as<void>(), &init, sizeof(init), cudaMemcpyHostToDevice,
                             ctx->stream));
    VXB_CUDA(cudaMemsetAsync(d_hist.as<void>(), 0, sizeof(unsigned int) * kMaxRanks * kBins,
                             ctx->stream));
    const int key_bits = sizeof(Real) == 8 ? 64 : 32;
    const int low = 64 - key_bits;  // float keys live in the high half
    // persistent grid of exactly the CTAs that are resident at once (a second wave
    // takes as long as the first); the shared-memory histogram is sized for the ranks
    // in use, so the register budget of the launch bounds decides the residency
    const size_t hist_smem = static_cast<size_t>(n_ranks) * kBins * sizeof(unsigned int);
    int per_sm = 0;
    auto kernel = failed ? radix_hist_kernel<Real, true> : radix_hist_kernel<Real, false>;
    VXB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kSelBlock, hist_smem));
    require(per_sm >= 1, "internal", "the histogram kernel does not fit on an SM");
    const unsigned grid = static_cast<unsigned>(
        std::min<uint64_t>((n + kSelBlock - 1) / kSelBlock,
                           static_cast<uint64_t>(ctx->prop.multiProcessorCount) * per_sm));
    int top = 64;
    while (top > low) {
        const int bits = std::min(kDigitBits, top - low);
        const int shift = top - bits;
        if (grid) {
            LaunchScope scope(ctx, VXB_K_SELECT);
            kernel<<<grid, kSelBlock, hist_smem, ctx->stream>>>(
                rho, failed, n, shift, bits, n_ranks, d_state.as<SelectState>(),
                d_hist.as<unsigned int>());
            check_launch("radix_hist_kernel");
        }
        if (shared)
            comm_allreduce_sum_u32(comm, d_hist.as<unsigned int>(), static_cast<size_t>(n_ranks) * kBins);
        {
            LaunchScope scope(ctx, VXB_K_SELECT);
            radix_pick_kernel<<<n_ranks, 256, 0, ctx->stream>>>(shift, bits, n_ranks,
                                                                d_state.as<SelectState>(),
                                                                d_hist.as<unsigned int>());
            check_launch("radix_pick_kernel");
        }
        top = shift;
    }
    SelectState fin{};
    VXB_CUDA(cudaMemcpyAsync(&fin, d_state.as<void>(), sizeof(fin), cudaMemcpyDeviceToHost,
                             ctx->stream));
    VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int q = 0; q < n_ranks; ++q)
        values[q] = sizeof(Real) == 8 ? key_to_double(fin.prefix[q])
                                      : static_cast<double>(key_to_float(fin.prefix[q]));
}

template <class Real>
uint64_t count_valid_device(vxb_ctx* ctx, const Real* rho, const uint8_t* failed, uint64_t n,
                            uint64_t* only_flag, vxb_comm* comm) {
    Scratch d_cnt(ctx, 2 * sizeof(unsigned long long));
    VXB_CUDA(cudaMemsetAsync(d_cnt.as<void>(), 0, 2 * sizeof(unsigned long long), ctx->stream));
    const unsigned grid = static_cast<unsigned>(
        std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(ctx->prop.multiProcessorCount) * 8));
    if (grid) {
        LaunchScope scope(ctx, VXB_K_SELECT);
        count_valid_kernel<Real><<<grid, 256, 0, ctx->stream>>>(rho, failed, n,
                                                               d_cnt.as<unsigned long long>());
        check_launch("count_valid_kernel");
    }
    // several ranks: both counts are those of the whole vector (every rank must take the
    // same with / without flags decision, and the same ranks)
    if (comm) comm_allreduce_sum_i64(comm, d_cnt.as<long long>(), 2);
    unsigned long long c[2] = {0, 0};
    VXB_CUDA(cudaMemcpyAsync(c, d_cnt.as<void>(), sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
    VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (only_flag) *only_flag = c[1];
    return c[0];
}

template <class Real>
void compact_device_t(vxb_ctx* ctx, const Real* rho, const uint8_t* failed, uint64_t n, double eps,
                      uint64_t index_base, uint64_t cap, uint64_t* n_accepted_host,
                      uint64_t* idx_dev) {
    const uint64_t tile = static_cast<uint64_t>(kSelBlock) * kSelItems;
    const uint64_t n_blocks = (n + tile - 1) / tile;
    if (n_blocks == 0) {
        if (is_device_pointer(n_accepted_host))
            VXB_CUDA(cudaMemsetAsync(n_accepted_host, 0, sizeof(uint64_t), ctx->stream));
        else
            *n_accepted_host = 0;
        return;
    }
    Scratch d_counts(ctx, n_blocks * sizeof(unsigned int));
    Scratch d_offsets(ctx, n_blocks * sizeof(unsigned long long));
    const bool want_idx = idx_dev && cap;
    Scratch d_flags(ctx, want_idx ? n_blocks * kSelBlock * sizeof(unsigned short) : 0);
    Scratch d_total(ctx, sizeof(unsigned long long));
    {
        LaunchScope scope(ctx, VXB_K_COMPACT);
        accept_count_kernel<Real><<<static_cast<unsigned>(n_blocks), kSelBlock, 0, ctx->stream>>>(
            rho, failed, n, eps, d_counts.as<unsigned int>(),
            want_idx ? d_flags.as<unsigned short>() : nullptr);
        check_launch("accept_count_kernel");
    }
    {
        LaunchScope scope(ctx, VXB_K_COMPACT);
        scan_blocks_kernel<<<1, 1024, 0, ctx->stream>>>(d_counts.as<unsigned int>(), n_blocks,
                                                        d_offsets.as<unsigned long long>(),
                                                        d_total.as<unsigned long long>());
        check_launch("scan_blocks_kernel");
    }
    if (want_idx) {
        LaunchScope scope(ctx, VXB_K_COMPACT);
        accept_write_kernel<<<static_cast<unsigned>(n_blocks), kSelBlock, 0, ctx->stream>>>(
            d_flags.as<unsigned short>(), d_offsets.as<unsigned long long>(), index_base, cap, idx_dev);
        check_launch("accept_write_kernel");
    }
    if (is_device_pointer(n_accepted_host)) {
        // device-resident count: the call stays asynchronous (no host round trip)
        VXB_CUDA(cudaMemcpyAsync(n_accepted_host, d_total.as<void>(), sizeof(unsigned long long),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
        return;
    }
    unsigned long long total = 0;
    VXB_CUDA(cudaMemcpyAsync(&total, d_total.as<void>(), sizeof(total), cudaMemcpyDeviceToHost,
                             ctx->stream));
    VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    *n_accepted_host = total;
}

void compact_accepted_device(vxb_ctx* ctx, int precision, const void* rho_dev,
                             const uint8_t* failed_dev, uint64_t n, double epsilon,
                             uint64_t index_base, uint64_t cap, uint64_t* n_accepted_host,
                             uint64_t* idx_dev) {
    if (precision == VXB_F32)
        compact_device_t<float>(ctx, static_cast<const float*>(rho_dev), failed_dev, n, epsilon,
                                index_base, cap, n_accepted_host, idx_dev);
    else
        compact_device_t<double>(ctx, static_cast<const double*>(rho_dev), failed_dev, n, epsilon,
                                 index_base, cap, n_accepted_host, idx_dev);
}

void order_statistics_any(vxb_ctx* ctx, int precision, const void* rho_dev,
                          const uint8_t* failed_dev, uint64_t n, const uint64_t* ranks,
                          int n_ranks, double* values, vxb_comm* comm) {
    if (precision == VXB_F32)
        order_statistics_device<float>(ctx, static_cast<const float*>(rho_dev), failed_dev, n,
                                       ranks, n_ranks, values, comm);
    else
        order_statistics_device<double>(ctx, static_cast<const double*>(rho_dev), failed_dev, n,
                                        ranks, n_ranks, values, comm);
}

// only_flag (optional): rows that their flag alone excludes; zero means the digit
// passes may be run without the flags
uint64_t count_valid_any(vxb_ctx* ctx, int precision, const void* rho_dev,
                         const uint8_t* failed_dev, uint64_t n, uint64_t* only_flag, vxb_comm* comm) {
    return precision == VXB_F32
               ? count_valid_device<float>(ctx, static_cast<const float*>(rho_dev), failed_dev, n, only_flag, comm)
               : count_valid_device<double>(ctx, static_cast<const double*>(rho_dev), failed_dev, n, only_flag, comm);
}

// The quantile rule of select_epsilon (abc.cpp:85-89 with numeric.cpp:20-30)
// evaluated on exact order statistics: same operations in the same order as
// the reference performs on its sorted array.
double epsilon_from_order_statistics(vxb_ctx* ctx, int precision, const void* rho_dev,
                                     const uint8_t* failed_dev, uint64_t n, double q,
                                     vxb_comm* comm = nullptr) {
    require(q > 0.0 && q <= 1.0, "invalid-argument", "accept fraction must lie in (0, 1]");
    uint64_t only_flag = 0;
    const uint64_t nv = count_valid_any(ctx, precision, rho_dev, failed_dev, n, &only_flag, comm);
    // the digit counters are 32 bits wide: one device cannot hold that many rows, several can
    require(nv < (1ull << 32), "invalid-shape", "the radix select counts at most 2^32 - 1 valid rows");
    require(nv >= 1, "empty-set", "every prior predictive row failed");
    if (only_flag == 0) failed_dev = nullptr;  // every failed row is a NaN: the digit passes skip the flags
    uint64_t ranks[3];
    int nr = 0;
    double eps;
    const uint64_t min_accept = static_cast<uint64_t>(std::ceil(q * static_cast<double>(nv)));
    // quantile_sorted
    uint64_t lo = 0;
    double frac = 0.0;
    int mode;  // 0: single element, 1: last element, 2: interpolate
    if (nv == 1) {
        mode = 0;
        ranks[nr++] = 0;
    } else {
        const double h = static_cast<double>(nv - 1) * q;
        lo = static_cast<uint64_t>(h);
        if (lo + 1 >= nv) {
            mode = 1;
            ranks[nr++] = nv - 1;
        } else {
            mode = 2;
            frac = h - static_cast<double>(lo);
            ranks[nr++] = lo;
            ranks[nr++] = lo + 1;
        }
    }
    const int guard_slot = nr;
    if (min_accept >= 1) ranks[nr++] = min_accept - 1;
    double v[3];
    order_statistics_any(ctx, precision, rho_dev, failed_dev, n, ranks, nr, v, comm);
    if (mode == 2)
        eps = v[0] + frac * (v[1] - v[0]);
    else
        eps = v[0];
    if (min_accept >= 1 && eps < v[guard_slot]) eps = v[guard_slot];
    return eps;
}

// quantile (numeric.cpp:20-36) of n device-resident finite values.
double quantile_device(vxb_ctx* ctx, const double* values_dev, uint64_t n, double level) {
    require(n >= 1, "insufficient-data", "quantile of an empty sample");
    require(level >= 0.0 && level <= 1.0, "invalid-argument", "quantile level outside [0,1]");
    uint64_t ranks[2] = {0, 0};
    double v[2];
    if (n == 1) {
        order_statistics_any(ctx, VXB_F64, values_dev, nullptr, n, ranks, 1, v);
        return v[0];
    }
    const double h = static_cast<double>(n - 1) * level;
    const uint64_t lo = static_cast<uint64_t>(h);
    if (lo + 1 >= n) {
        ranks[0] = n - 1;
        order_statistics_any(ctx, VXB_F64, values_dev, nullptr, n, ranks, 1, v);
        return v[0];
    }
    const double frac = h - static_cast<double>(lo);
    ranks[0] = lo;
    ranks[1] = lo + 1;
    order_statistics_any(ctx, VXB_F64, values_dev, nullptr, n, ranks, 2, v);
    return v[0] + frac * (v[1] - v[0]);
}

}  // namespace vxb

using namespace vxb;

extern "C" int vxb_order_statistics(vxb_ctx* ctx, int precision, const void* rho,
                                    const uint8_t* failed, uint64_t n, const uint64_t* ranks,
                                    uint32_t n_ranks, double* values, uint64_t* n_valid) {
    return guarded([&] {
        use(ctx);
        require(rho && ranks && values, "invalid-argument", "null argument");
        require(n >= 1, "insufficient-data", "order statistic of an empty sample");
        const size_t real = precision == VXB_F32 ? 4 : 8;
        Staged d_rho(ctx, rho, n * real, true, false);
        Staged d_failed(ctx, failed, n, true, false);
        uint64_t only_flag = 0;
        const uint64_t nv = count_valid_any(ctx, precision, d_rho.ptr(), d_failed.as<uint8_t>(), n, &only_flag);
        const uint8_t* flags = only_flag ? d_failed.as<uint8_t>() : nullptr;
        if (n_valid) *n_valid = nv;
        for (uint32_t q = 0; q < n_ranks; ++q)
            require(ranks[q] < nv, "invalid-argument", "rank exceeds the number of valid rows");
        for (uint32_t q0 = 0; q0 < n_ranks; q0 += kMaxRanks) {
            const int nr = static_cast<int>(std::min<uint32_t>(kMaxRanks, n_ranks - q0));
            order_statistics_any(ctx, precision, d_rho.ptr(), flags, n, ranks + q0, nr, values + q0);
        }
    });
}

extern "C" int vxb_compact_accepted(vxb_ctx* ctx, int precision, const void* rho,
                                    const uint8_t* failed, uint64_t n, double epsilon,
                                    uint64_t index_base, uint64_t cap, uint64_t* n_accepted,
                                    uint64_t* idx) {
    return guarded([&] {
        use(ctx);
        require(rho && n_accepted, "invalid-argument", "null argument");
        const size_t real = precision == VXB_F32 ? 4 : 8;
        Staged d_rho(ctx, rho, n * real, true, false);
        Staged d_failed(ctx, failed, n, true, false);
        Staged d_idx(ctx, idx, cap * sizeof(uint64_t), false, true);
        uint64_t total = 0;
        compact_accepted_device(ctx, precision, d_rho.ptr(), d_failed.as<uint8_t>(), n, epsilon,
                                index_base, cap, &total, d_idx.as<uint64_t>());
        *n_accepted = total;
        d_idx.finish(std::min(total, cap) * sizeof(uint64_t));
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

extern "C" int vxb_select_epsilon(vxb_ctx* ctx, int precision, const void* rho,
                                  const uint8_t* failed, uint64_t n, double accept_fraction,
                                  double* epsilon, uint64_t cap, uint64_t* n_accepted,
                                  uint64_t* idx) {
    return guarded([&] {
        use(ctx);
        require(rho && epsilon && n_accepted, "invalid-argument", "null argument");
        require(accept_fraction > 0.0 && accept_fraction <= 1.0, "invalid-argument",
                "accept fraction must lie in (0, 1]");
        require(n >= 1, "empty-set", "every prior predictive row failed");
        const size_t real = precision == VXB_F32 ? 4 : 8;
        Staged d_rho(ctx, rho, n * real, true, false);
        Staged d_failed(ctx, failed, n, true, false);
        const double eps = epsilon_from_order_statistics(ctx, precision, d_rho.ptr(),
                                                         d_failed.as<uint8_t>(), n, accept_fraction);
        *epsilon = eps;
        Staged d_idx(ctx, idx, cap * sizeof(uint64_t), false, true);
        uint64_t total = 0;
        compact_accepted_device(ctx, precision, d_rho.ptr(), d_failed.as<uint8_t>(), n, eps, 0, cap,
                                &total, d_idx.as<uint64_t>());
        *n_accepted = total;
        d_idx.finish(std::min(total, cap) * sizeof(uint64_t));
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// Distributed form of vxb_select_epsilon: see the header.  Every rank returns the same
// epsilon (same integer histograms, same host arithmetic) and compacts its own rows
// under global indices; the index blocks travel in one all-gather.
extern "C" int vxb_sharded_select_epsilon(vxb_ctx* ctx, vxb_comm* comm, int precision,
                                          const void* rho_local, const uint8_t* failed_local,
                                          uint64_t n_local, uint64_t first_row,
                                          double accept_fraction, double* epsilon,
                                          uint64_t* n_accepted, uint64_t cap, void* block_local,
                                          void* blocks_all) {
    return guarded([&] {
        use(ctx);
        require(epsilon && n_accepted, "invalid-argument", "null argument");
        require(n_local == 0 || rho_local, "invalid-argument", "null distances");
        require(accept_fraction > 0.0 && accept_fraction <= 1.0, "invalid-argument",
                "accept fraction must lie in (0, 1]");
        require(cap == 0 || (block_local && is_device_pointer(block_local)), "invalid-argument",
                "block_local is a device buffer of VXB_INDEX_BLOCK_BYTES(cap)");
        require(cap == 0 || !comm || (blocks_all && is_device_pointer(blocks_all)), "invalid-argument",
                "blocks_all is a device buffer of n_ranks blocks");
        const size_t real = precision == VXB_F32 ? 4 : 8;
        Staged d_rho(ctx, rho_local, n_local * real, true, false);
        Staged d_failed(ctx, failed_local, n_local, true, false);
        const double eps = epsilon_from_order_statistics(ctx, precision, d_rho.ptr(), d_failed.as<uint8_t>(),
                                                         n_local, accept_fraction, comm);
        *epsilon = eps;
        const size_t block = VXB_INDEX_BLOCK_BYTES(cap);
        Scratch d_count(ctx, 2 * sizeof(uint64_t));
        uint64_t* count_dev = cap ? static_cast<uint64_t*>(block_local) : d_count.as<uint64_t>();
        if (cap) VXB_CUDA(cudaMemsetAsync(block_local, 0, 16, ctx->stream));
        compact_accepted_device(ctx, precision, d_rho.ptr(), d_failed.as<uint8_t>(), n_local, eps, first_row,
                                cap, count_dev, cap ? reinterpret_cast<uint64_t*>(static_cast<char*>(block_local) + 16)
                                                    : nullptr);
        if (cap && comm)
            comm_allgather(comm, block_local, blocks_all, block);
        else if (cap && blocks_all && blocks_all != block_local)
            VXB_CUDA(cudaMemcpyAsync(blocks_all, block_local, block, cudaMemcpyDeviceToDevice, ctx->stream));
        uint64_t* total_dev = d_count.as<uint64_t>() + 1;
        VXB_CUDA(cudaMemcpyAsync(total_dev, count_dev, sizeof(uint64_t), cudaMemcpyDeviceToDevice, ctx->stream));
        if (comm) comm_allreduce_sum_i64(comm, reinterpret_cast<long long*>(total_dev), 1);
        uint64_t total = 0;
        VXB_CUDA(cudaMemcpyAsync(&total, total_dev, sizeof(total), cudaMemcpyDeviceToHost, ctx->stream));
        VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        *n_accepted = total;
    });
}
