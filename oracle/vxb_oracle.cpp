// oracle/vxb_oracle.cpp -- TEST INFRASTRUCTURE (the parity oracle), not product.
//
// A self-contained CPU restatement of the hot path of the vexbayes reference,
// written against the reference's published algorithm; every function cites the
// reference location it follows (paths relative to /root/reference/proj/core/).
// It has NO dependency on /root/reference, so it travels to the GPU box.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm may load it.  Build: oracle/Makefile (g++ -O2 -ffp-contract=off, the
// reference's flags, proj/CMakeLists.txt:15-18 -- per-operation IEEE rounding,
// no FMA contraction).
//
// Pinning (tests/test_oracle_pins.py, tests/test_anneal.py): the RNG, fastmath,
// numeric, partition, ABC sampler, epsilon selection, resampling, ESS, p-value
// counting, the toggle-switch model, the bioassay model with the likelihood-
// annealed sampler (smc::run_smc) and run_weak_info_test, and the TB Gillespie
// model are checked bit-for-bit against oracle/_ref (the unmodified reference
// compiled from /root/reference) where that library is present, and everywhere
// against the golden vectors it generated (tests/golden/, scripts
// tests/golden/make_golden*.py).
// Workloads the reference does not contain -- ABC-SMC generation loop, weighted
// covariance, Poisson variates, tau-leap and its MLMC coupling -- are
// "parity unpinned": they are defined HERE and anchored by
// analytic checks only.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "../include/vexbayes_cuda.h"  // vxb_model / vxb_keying / cfg structs only

namespace {

thread_local std::string g_err;

struct OracleError {
    std::string text;
};
[[noreturn]] void raise(const char* code, const char* msg) {
    throw OracleError{std::string(code) + ": " + msg};  // errors.hpp:11-28 "code: message"
}
void require(bool ok, const char* code, const char* msg) {
    if (!ok) raise(code, msg);
}
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const OracleError& e) {
        g_err = e.text;
        return 1;
    }
}

template <class To, class From>
To bit_cast(const From& v) {
    To out;
    static_assert(sizeof(To) == sizeof(From));
    std::memcpy(&out, &v, sizeof(To));
    return out;
}

template <class F>
void parallel_for(std::uint64_t n, unsigned threads, F&& body) {
    if (threads <= 1 || n < 2) {
        for (std::uint64_t i = 0; i < n; ++i) body(i);
        return;
    }
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            for (std::uint64_t i = t; i < n; i += threads) body(i);
        });
    for (auto& th : pool) th.join();
}

// ===================================================================== RNG
// splitmix64: rng.cpp:22-27
std::uint64_t splitmix64(std::uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
// derive_seed: rng.cpp:29-35
std::uint64_t derive_seed(std::uint64_t seed, const std::uint64_t* path, std::size_t n) {
    std::uint64_t h = splitmix64(seed);
    for (std::size_t i = 0; i < n; ++i) h = splitmix64(h ^ path[i]);
    return h;
}
std::uint64_t derive_seed1(std::uint64_t seed, std::uint64_t a) { return derive_seed(seed, &a, 1); }

// key derivation: rng.cpp:37-40.  stream_id is 32-bit in the reference; the
// oracle takes 64 bits (identical for ids < 2^32).
std::uint64_t stream_key(std::uint64_t seed, std::uint64_t stream_id) {
    return splitmix64(splitmix64(seed) ^ stream_id);
}

struct Block {
    std::uint64_t w0, w1;
};
// Philox2x64-10 on the 128-bit pair index: rng.cpp:12-14 (constants), 65-78.
Block philox_block(std::uint64_t key, std::uint64_t idx_lo, std::uint64_t idx_hi) {
    std::uint64_t c0 = idx_lo, c1 = idx_hi, k = key;
    for (int round = 0; round < 10; ++round) {
        const unsigned __int128 prod = static_cast<unsigned __int128>(0xD2B74407B1CE6E93ULL) * c0;
        const std::uint64_t hi = static_cast<std::uint64_t>(prod >> 64);
        const std::uint64_t lo = static_cast<std::uint64_t>(prod);
        c0 = hi ^ k ^ c1;
        c1 = lo;
        k += 0x9E3779B97F4A7C15ULL;
    }
    return {c0, c1};
}
// to_unit: rng.cpp:16-18
double to_unit(std::uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }

// ================================================================ fastmath
// The reference's libm-free elementary functions (fastmath.hpp:23-128) restated
// as coefficient tables + one Horner routine.  Every step is a separately
// rounded multiply followed by a separately rounded add (this file is compiled
// with -ffp-contract=off), in the reference's order, so results are identical
// bit for bit (pinned in tests/test_oracle_pins.py).
constexpr double kLn2 = 0x1.62e42fefa39efp-1;     // fastmath.hpp:19
constexpr double kInvLn2 = 0x1.71547652b82fep+0;  // fastmath.hpp:20
constexpr double kRoundMagic = 0x1.8p52;          // (x + M) - M rounds x to an integer

template <std::size_t N>
double horner(const double (&coef)[N], double x) {
    double acc = coef[0];
    for (std::size_t i = 1; i < N; ++i) acc = acc * x + coef[i];
    return acc;
}
// 2 atanh(t) / (2 t) series in s = t^2: sum_{k} s^k / (2k+1), highest power first (:40-50)
constexpr double kAtanhSeries[11] = {1.0 / 21.0, 1.0 / 19.0, 1.0 / 17.0, 1.0 / 15.0, 1.0 / 13.0, 1.0 / 11.0,
                                     1.0 / 9.0,  1.0 / 7.0,  1.0 / 5.0,  1.0 / 3.0,  1.0};
// exp(w) Taylor coefficients 1/13! ... 1/0! (:63-76)
constexpr double kExpSeries[14] = {1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
                                   1.0 / 362880.0,     1.0 / 40320.0,     1.0 / 5040.0,     1.0 / 720.0,
                                   1.0 / 120.0,        1.0 / 24.0,        1.0 / 6.0,        0.5,
                                   1.0,                1.0};
// sin(s)/s in s^2: 1/21! ... alternating (:90-100); cos(s) in s^2: -1/22! ... (:113-124)
constexpr double kSinSeries[11] = {1.0 / 51090942171709440000.0, -1.0 / 121645100408832000.0,
                                   1.0 / 355687428096000.0,      -1.0 / 1307674368000.0,
                                   1.0 / 6227020800.0,           -1.0 / 39916800.0,
                                   1.0 / 362880.0,               -1.0 / 5040.0,
                                   1.0 / 120.0,                  -1.0 / 6.0,
                                   1.0};
constexpr double kCosSeries[12] = {-1.0 / 1124000727777607680000.0, 1.0 / 2432902008176640000.0,
                                   -1.0 / 6402373705728000.0,       1.0 / 20922789888000.0,
                                   -1.0 / 87178291200.0,            1.0 / 479001600.0,
                                   -1.0 / 3628800.0,                1.0 / 40320.0,
                                   -1.0 / 720.0,                    1.0 / 24.0,
                                   -1.0 / 2.0,                      1.0};

// log2 of a finite positive double (fastmath.hpp:23-51): split into exponent and
// mantissa, fold the mantissa into [sqrt(1/2), sqrt 2), then the atanh series of
// t = (m-1)/(m+1).
double log2_pos(double x) {
    std::uint64_t raw = bit_cast<std::uint64_t>(x);
    std::int64_t expo = static_cast<std::int64_t>((raw >> 52) & 0x7FF);
    if (expo == 0) {  // subnormal: scale into the normal range first
        raw = bit_cast<std::uint64_t>(x * 0x1p64);
        expo = static_cast<std::int64_t>((raw >> 52) & 0x7FF) - 64;
    }
    double mant = bit_cast<double>((raw & 0xFFFFFFFFFFFFFULL) | 0x3FF0000000000000ULL);
    const bool fold = mant > 1.4142135623730951;
    if (fold) mant = 0.5 * mant;
    const double expo_d = static_cast<double>(expo - 1023 + (fold ? 1 : 0));
    const double t = (mant - 1.0) / (mant + 1.0);
    const double series = horner(kAtanhSeries, t * t);
    return expo_d + (2.0 * kInvLn2) * t * series;
}
double ln_pos(double x) { return log2_pos(x) * kLn2; }  // fastmath.hpp:54

// 2^z with z clamped to the normal exponent range (fastmath.hpp:57-79)
double exp2_clamped(double z) {
    if (z < -1022.0) z = -1022.0;
    if (z > 1023.0) z = 1023.0;
    const double whole = (z + kRoundMagic) - kRoundMagic;
    const double frac = (z - whole) * kLn2;  // |frac| <= ln2/2
    const double series = horner(kExpSeries, frac);
    const std::uint64_t biased = static_cast<std::uint64_t>(static_cast<std::int64_t>(whole) + 1023);
    return series * bit_cast<double>(biased << 52);
}
double pow_pos(double x, double y) { return exp2_clamped(y * log2_pos(x)); }  // fastmath.hpp:82

// sin(pi a) and cos(pi a) (fastmath.hpp:85-128): reduce a to r in [-1/2, 1/2] around
// the nearest integer n, evaluate at s = pi r, flip the sign for odd n.
struct PiReduced {
    double s, s2, sign;
};
PiReduced reduce_pi(double a) {
    const double whole = (a + kRoundMagic) - kRoundMagic;
    const double s = (a - whole) * 3.141592653589793238462643383279502884;
    const bool odd = (static_cast<std::int64_t>(whole) & 1) != 0;
    return {s, s * s, odd ? -1.0 : 1.0};
}
double sinpi(double a) {
    const PiReduced r = reduce_pi(a);
    const double base = r.s * horner(kSinSeries, r.s2);
    return r.sign * base;
}
double cospi(double a) {
    const PiReduced r = reduce_pi(a);
    return r.sign * horner(kCosSeries, r.s2);
}

// Random-access view of RngStream(seed, stream_id): every output is a pure
// function of the counter position (rng.hpp:18-28).  64-bit positions.
struct Stream {
    std::uint64_t key;
    std::uint64_t pos = 0;
    std::uint64_t cache_idx = ~0ULL;
    Block cache{0, 0};
    Stream(std::uint64_t seed, std::uint64_t id) : key(stream_key(seed, id)) {}
    const Block& block_of(std::uint64_t p) {  // current_pair_block: rng.cpp:80-90
        const std::uint64_t idx = p >> 1;
        if (idx != cache_idx) {
            cache = philox_block(key, idx, 0);
            cache_idx = idx;
        }
        return cache;
    }
    void align_even() { pos += pos & 1; }  // rng.cpp:57-59
    std::uint64_t next_u64() {             // rng.cpp:92-97
        const Block& b = block_of(pos);
        const std::uint64_t w = (pos & 1) ? b.w1 : b.w0;
        ++pos;
        return w;
    }
    double next_unit() { return to_unit(next_u64()); }  // rng.cpp:99
    // next_uniform / fill_uniform: rng.cpp:101-110, 125-140
    double next_uniform(double a, double b) {
        require(a <= b, "invalid-range", "uniform lower bound exceeds upper bound");
        if (a == b) {
            next_u64();
            return a;
        }
        const double top = std::nextafter(b, a);
        const double r = a + next_unit() * (b - a);
        return r < a ? a : (r > top ? top : r);
    }
    // next_gaussian: rng.cpp:112-123 (pair m = pos/2, cos branch at even pos)
    double next_gaussian(double mu, double sigma) {
        require(sigma >= 0.0, "invalid-scale", "gaussian sigma must be nonnegative");
        const bool odd = (pos & 1) != 0;
        const Block& b = block_of(pos);
        const double u1 = to_unit(b.w0);
        const double u2 = to_unit(b.w1);
        const double r = std::sqrt(-2.0 * ln_pos(1.0 - u1));
        const double ang = 2.0 * u2;
        const double z = odd ? r * sinpi(ang) : r * cospi(ang);
        ++pos;
        return mu + sigma * z;
    }
};

// ================================================================= numeric
// quantile_sorted: numeric.cpp:20-30 (type-7)
double quantile_sorted(const double* sorted, std::size_t n, double level) {
    require(n > 0, "insufficient-data", "quantile of an empty sample");
    require(level >= 0.0 && level <= 1.0, "invalid-argument", "quantile level outside [0,1]");
    if (n == 1) return sorted[0];
    const double h = static_cast<double>(n - 1) * level;
    const std::size_t lo = static_cast<std::size_t>(h);
    if (lo + 1 >= n) return sorted[n - 1];
    const double frac = h - static_cast<double>(lo);
    return sorted[lo] + frac * (sorted[lo + 1] - sorted[lo]);
}
// quantile: numeric.cpp:32-36
double quantile(const double* sample, std::size_t n, double level) {
    std::vector<double> copy(sample, sample + n);
    std::sort(copy.begin(), copy.end());
    return quantile_sorted(copy.data(), n, level);
}
// logsumexp: numeric.cpp:11-18
double logsumexp(const double* x, std::size_t n) {
    double m = -std::numeric_limits<double>::infinity();
    for (std::size_t i = 0; i < n; ++i) m = std::max(m, x[i]);
    if (!std::isfinite(m)) return m;
    double s = 0.0;
    for (std::size_t i = 0; i < n; ++i) s += std::exp(x[i] - m);
    return m + std::log(s);
}
// sample_covariance: numeric.cpp:55-79
void sample_covariance(const double* data, std::size_t rows, std::size_t dim, double* cov) {
    require(rows >= 2, "insufficient-data", "covariance needs at least two rows");
    std::vector<double> mu(dim, 0.0);
    for (std::size_t r = 0; r < rows; ++r)
        for (std::size_t k = 0; k < dim; ++k) mu[k] += data[r * dim + k];
    for (double& v : mu) v /= static_cast<double>(rows);
    std::fill(cov, cov + dim * dim, 0.0);
    for (std::size_t r = 0; r < rows; ++r)
        for (std::size_t i = 0; i < dim; ++i) {
            const double di = data[r * dim + i] - mu[i];
            for (std::size_t j = 0; j <= i; ++j) cov[i * dim + j] += di * (data[r * dim + j] - mu[j]);
        }
    const double norm = 1.0 / static_cast<double>(rows - 1);
    for (std::size_t i = 0; i < dim; ++i)
        for (std::size_t j = 0; j <= i; ++j) {
            cov[i * dim + j] *= norm;
            cov[j * dim + i] = cov[i * dim + j];
        }
}
// cholesky: numeric.cpp:81-96
bool cholesky(double* a, std::size_t dim) {
    for (std::size_t j = 0; j < dim; ++j) {
        double d = a[j * dim + j];
        for (std::size_t k = 0; k < j; ++k) d -= a[j * dim + k] * a[j * dim + k];
        if (!(d > 0.0)) return false;
        const double ljj = std::sqrt(d);
        a[j * dim + j] = ljj;
        for (std::size_t i = j + 1; i < dim; ++i) {
            double s = a[i * dim + j];
            for (std::size_t k = 0; k < j; ++k) s -= a[i * dim + k] * a[j * dim + k];
            a[i * dim + j] = s / ljj;
        }
        for (std::size_t i = 0; i < j; ++i) a[i * dim + j] = 0.0;
    }
    return true;
}
// partition: blocked.cpp:34-63
void partition(std::uint64_t total, std::uint64_t workers, std::uint64_t width,
               std::uint64_t* ranges) {
    require(total >= 1, "invalid-shape", "partition needs at least one item");
    require(workers >= 1, "invalid-shape", "partition needs at least one worker");
    require(width >= 1, "invalid-shape", "partition needs a positive block width");
    const std::uint64_t blocks = (total + width - 1) / width;
    const std::uint64_t base = blocks / workers, extra = blocks % workers;
    std::uint64_t begin_block = 0;
    for (std::uint64_t w = 0; w < workers; ++w) {
        const std::uint64_t nb = base + (w < extra ? 1 : 0);
        const std::uint64_t begin = begin_block * width;
        std::uint64_t end = (begin_block + nb) * width;
        if (end > total) end = total;
        if (begin > total) {
            ranges[2 * w] = total;
            ranges[2 * w + 1] = total;
        } else {
            ranges[2 * w] = begin;
            ranges[2 * w + 1] = end;
        }
        begin_block += nb;
    }
}
bool supported_width(std::uint64_t v) {  // blocked.cpp:10-12
    return v == 1 || v == 2 || v == 4 || v == 8 || v == 16;
}

// Canonical two-level summation used by every reduction the reference leaves
// to a serial coordinator loop and that the GPU must reproduce bit-for-bit
// independent of its launch shape: elements are summed left-to-right inside
// consecutive chunks of kChunk, then the chunk totals left-to-right.
constexpr std::size_t kChunk = 256;
template <class Get>
double canon_sum(std::size_t n, Get&& get) {
    double total = 0.0;
    for (std::size_t c0 = 0; c0 < n; c0 += kChunk) {
        const std::size_t c1 = std::min(n, c0 + kChunk);
        double part = 0.0;
        for (std::size_t i = c0; i < c1; ++i) part += get(i);
        total += part;
    }
    return total;
}
// Canonical two-level inclusive scan: cum[i] = offset(chunk) + local prefix.
void canon_cumsum(const double* w, std::size_t n, double* cum) {
    double offset = 0.0;
    for (std::size_t c0 = 0; c0 < n; c0 += kChunk) {
        const std::size_t c1 = std::min(n, c0 + kChunk);
        double run = 0.0;
        for (std::size_t i = c0; i < c1; ++i) {
            run += w[i];
            cum[i] = offset + run;
        }
        offset = offset + run;
    }
}
std::size_t upper_bound_idx(const double* cum, std::size_t n, double target) {
    // std::upper_bound of smc.cpp:287, clamped as smc.cpp:289
    std::size_t lo = 0, hi = n;
    while (lo < hi) {
        const std::size_t mid = lo + (hi - lo) / 2;
        if (target < cum[mid]) hi = mid; else lo = mid + 1;
    }
    return lo >= n ? n - 1 : lo;
}

// ======================================================= logistic SDE model
// Model in the mould of toggle_switch.cpp: prior box map (:17-22), Euler-
// Maruyama with explicit operation order (:46-62), variates addressed by a
// canonical layout in counter space (toggle_switch.hpp:52-57): relative to the
// row's base position, positions 0..dim-1 are the prior uniforms, the counter
// is aligned to even (abc.cpp:53), then position dim_e + j is the standard
// normal of step j+1.
struct Logistic {
    std::uint32_t steps, stride, n_obs;
    double dt, sqdt, x0;
    double lo[3], hi[3];
    explicit Logistic(const vxb_model& m)
        : steps(m.steps), stride(m.obs_stride), n_obs(m.obs_stride ? m.steps / m.obs_stride : 0),
          dt(m.dt), sqdt(m.consts[0]), x0(m.x0) {
        require(m.model == VXB_MODEL_LOGISTIC_SDE, "invalid-argument", "not a logistic model");
        require(m.dim == 3, "invalid-shape", "logistic model has three parameters");
        require(m.steps >= 1 && m.obs_stride >= 1, "invalid-horizon", "need at least one step");
        require(m.summary_dim == n_obs && n_obs >= 1, "invalid-summary",
                "summary_dim must equal steps / obs_stride");
        for (int k = 0; k < 3; ++k) {
            lo[k] = m.prior_lo[k];
            hi[k] = m.prior_hi[k];
            require(lo[k] <= hi[k], "invalid-range", "uniform lower bound exceeds upper bound");
        }
    }
    std::uint64_t row_stride() const {  // positions one row consumes in a worker stream
        return 4 + steps + (steps & 1);
    }
    void sample_prior(Stream& s, double* theta) const {
        double unit[3];
        for (int k = 0; k < 3; ++k) unit[k] = s.next_uniform(0.0, 1.0);
        for (int k = 0; k < 3; ++k) theta[k] = lo[k] + unit[k] * (hi[k] - lo[k]);
    }
    // returns false when the state left the reals (the reference would throw
    // and abc.cpp:57-60 flags the row)
    template <class Real, class Noise>
    bool simulate(const double* theta, Noise&& noise, double* summary) const {
        const Real r = static_cast<Real>(theta[0]);
        const Real k = static_cast<Real>(theta[1]);
        const Real sigma = static_cast<Real>(theta[2]);
        const Real a = r * static_cast<Real>(dt);
        const Real c = sigma * static_cast<Real>(sqdt);
        const Real inv_k = Real(1) / k;
        Real x = static_cast<Real>(x0);
        std::uint32_t next = 0, since = 0;
        for (std::uint32_t j = 0; j < steps; ++j) {
            const Real z = static_cast<Real>(noise(j));
            const Real drift = (a * x) * (Real(1) - x * inv_k);
            const Real diff = (c * x) * z;
            x = (x + drift) + diff;
            if (++since == stride) {
                since = 0;
                if (next < n_obs) summary[next++] = static_cast<double>(x);
            }
        }
        for (std::uint32_t i = 0; i < n_obs; ++i)
            if (!std::isfinite(summary[i])) return false;
        return true;
    }
};

// discrepancy: abc.cpp:16-24 (left-to-right accumulation), in Real
template <class Real>
double discrepancy(const double* sim, const double* obs, std::size_t n) {
    Real ss = 0;
    for (std::size_t i = 0; i < n; ++i) {
        const Real d = static_cast<Real>(sim[i]) - static_cast<Real>(obs[i]);
        ss += d * d;
    }
    return static_cast<double>(std::sqrt(ss));
}

template <class Real>
void abc_row(const Logistic& lg, Stream& s, const double* observed, const double* ext_noise,
             double* theta, double* summary, double* rho, std::uint8_t* failed) {
    lg.sample_prior(s, theta);
    if (sizeof(Real) == 4)
        for (int k = 0; k < 3; ++k) theta[k] = static_cast<double>(static_cast<float>(theta[k]));
    s.align_even();  // abc.cpp:53
    bool ok;
    if (ext_noise) {
        ok = lg.simulate<Real>(theta, [&](std::uint32_t j) { return ext_noise[j]; }, summary);
        s.pos += lg.steps + (lg.steps & 1);
    } else {
        ok = lg.simulate<Real>(theta, [&](std::uint32_t) { return s.next_gaussian(0.0, 1.0); },
                               summary);
        s.pos += lg.steps & 1;  // fill_gaussian consumes an even count
    }
    if (ok) {
        *rho = discrepancy<Real>(summary, observed, lg.n_obs);
        *failed = 0;
    } else {  // abc.cpp:57-60
        *rho = std::numeric_limits<double>::quiet_NaN();
        *failed = 1;
        std::fill(summary, summary + lg.n_obs, 0.0);
    }
}

// ===================================================== toggle-switch model
// The reference's own SDE (toggle_switch.cpp), restated: prior box map
// (:17-22), per-cell canonical variate layout cell_stride = 2T
// (toggle_switch.hpp:52-57): relative to the aligned call position, cell c owns
// positions [c*2T, (c+1)*2T); positions 2(j-1), 2(j-1)+1 are step j's (u, v)
// increments, position 2(T-1) the observation normal, the last one padding.
// Euler-Maruyama update with previous-step powers and floor at 1 (:46-62),
// noisy observation (:64-69), 19 type-7 quantiles of the sorted observations
// (:123-133).
struct Toggle {
    std::uint32_t steps, cells;
    double lo[7], hi[7];
    explicit Toggle(const vxb_model& m) : steps(m.steps), cells(static_cast<std::uint32_t>(m.consts[1])) {
        require(m.model == VXB_MODEL_TOGGLE, "invalid-argument", "not the toggle-switch model");
        require(m.dim == 7 && m.summary_dim == 19, "invalid-shape",
                "toggle model has 7 parameters and 19 summaries");
        require(cells >= 1, "invalid-shape", "toggle simulation needs at least one cell");
        for (int k = 0; k < 7; ++k) {
            lo[k] = m.prior_lo[k];
            hi[k] = m.prior_hi[k];
            require(lo[k] <= hi[k], "invalid-range", "uniform lower bound exceeds upper bound");
        }
    }
    std::uint64_t padded(std::uint64_t v) const { return (cells + v - 1) / v * v; }
    // stream positions one row consumes: 7 uniforms, align, padded cells x 2T
    std::uint64_t row_stride(std::uint64_t v) const { return 8 + padded(v) * 2 * steps; }
    void sample_prior(Stream& s, double* theta) const {
        double unit[7];
        for (int k = 0; k < 7; ++k) unit[k] = s.next_uniform(0.0, 1.0);
        for (int k = 0; k < 7; ++k) theta[k] = lo[k] + unit[k] * (hi[k] - lo[k]);
    }
    // y[cells] for one parameter vector; s.pos must be the aligned call position
    void simulate(const double* th, Stream& s, std::uint64_t v, double* y) const {
        const double mu = th[0], sigma = th[1], gamma = th[2];
        const double alpha_u = th[3], alpha_v = th[4], beta_u = th[5], beta_v = th[6];
        const std::uint64_t b0 = s.pos;
        for (std::uint64_t c = 0; c < cells; ++c) {
            s.pos = b0 + c * 2 * steps;
            double u = 10.0, w = 10.0;
            for (std::uint32_t j = 1; j < steps; ++j) {
                const double zu = s.next_gaussian(0.0, 1.0);
                const double zv = s.next_gaussian(0.0, 1.0);
                const double p_u = pow_pos(w, beta_u);
                const double p_v = pow_pos(u, beta_v);
                double ut = u * 0.97;
                ut += alpha_u / (1.0 + p_u) - 1.0;
                double vt = w * 0.97;
                vt += alpha_v / (1.0 + p_v) - 1.0;
                ut += 0.5 * zu;
                vt += 0.5 * zv;
                u = ut >= 1.0 ? ut : 1.0;
                w = vt >= 1.0 ? vt : 1.0;
            }
            const double eta = s.next_gaussian(0.0, 1.0);
            const double obs = u + mu + sigma * mu * eta / pow_pos(u, gamma);
            y[c] = obs >= 1.0 ? obs : 1.0;
        }
        s.pos = b0 + padded(v) * 2 * steps;
    }
    // returns false for the rows the reference would flag (Error inside simulate)
    bool summaries(const double* th, Stream& s, std::uint64_t v, double* q) const {
        if (steps < 2 || cells < 19) return false;  // invalid-horizon / insufficient-data
        std::vector<double> y(cells);
        simulate(th, s, v, y.data());
        std::sort(y.begin(), y.end());
        for (int k = 0; k < 19; ++k) q[k] = quantile_sorted(y.data(), cells, 0.05 * static_cast<double>(k + 1));
        return true;
    }
};

void toggle_prior_predictive(const vxb_model* m, const vxb_keying* key, std::uint64_t n_total,
                             std::uint64_t first, std::uint64_t count, const double* observed,
                             double* params, double* summaries, double* rho, std::uint8_t* failed,
                             unsigned threads) {
    const Toggle tg(*m);
    require(m->precision == VXB_F64, "invalid-argument", "the toggle model is fp64");
    std::vector<std::uint64_t> ranges;
    std::uint64_t v = 1;
    if (key->mode == VXB_KEY_WORKER) {
        require(key->workers >= 1, "invalid-shape", "need at least one worker");
        require(supported_width(key->block_width), "invalid-shape", "unsupported block width");
        v = key->block_width;
        ranges.resize(2 * key->workers);
        partition(n_total, key->workers, v, ranges.data());
    }
    parallel_for(count, threads, [&](std::uint64_t r) {
        const std::uint64_t row = first + r;
        std::uint64_t id = row, base = 0;
        if (key->mode == VXB_KEY_WORKER) {
            std::uint64_t w = 0;
            while (!(row >= ranges[2 * w] && row < ranges[2 * w + 1])) ++w;
            id = w;
            base = (row - ranges[2 * w]) * tg.row_stride(v);
        }
        Stream s(key->seed, id);
        s.pos = base;
        double theta[7], q[19];
        tg.sample_prior(s, theta);
        s.align_even();
        double dist = std::numeric_limits<double>::quiet_NaN();
        std::uint8_t bad = 0;
        if (tg.summaries(theta, s, v, q)) {
            dist = discrepancy<double>(q, observed, 19);
        } else {
            bad = 1;
            std::fill(q, q + 19, 0.0);
        }
        if (params) std::copy(theta, theta + 7, params + r * 7);
        if (summaries) std::copy(q, q + 19, summaries + r * 19);
        if (rho) rho[r] = dist;
        if (failed) failed[r] = bad;
    });
}

}  // namespace

extern "C" {

const char* vxo_last_error() { return g_err.c_str(); }

// --------------------------------------------------------------- substrate
std::uint64_t vxo_splitmix64(std::uint64_t z) { return splitmix64(z); }
std::uint64_t vxo_derive_seed(std::uint64_t seed, const std::uint64_t* path, std::size_t n) {
    return derive_seed(seed, path, n);
}
int vxo_stream_u64(std::uint64_t seed, std::uint64_t id, std::uint64_t pos, std::uint64_t n,
                   std::uint64_t* out) {
    return guarded([&] {
        Stream s(seed, id);
        s.pos = pos;
        for (std::uint64_t i = 0; i < n; ++i) out[i] = s.next_u64();
    });
}
int vxo_fill_uniform(std::uint64_t seed, std::uint64_t id, std::uint64_t pos, std::uint64_t n,
                     double a, double b, double* out) {
    return guarded([&] {
        require(a <= b, "invalid-range", "uniform lower bound exceeds upper bound");
        Stream s(seed, id);
        s.pos = pos;
        for (std::uint64_t i = 0; i < n; ++i) out[i] = s.next_uniform(a, b);
    });
}
int vxo_fill_gaussian(std::uint64_t seed, std::uint64_t id, std::uint64_t pos, std::uint64_t n,
                      double mu, double sigma, double* out) {
    return guarded([&] {
        require(sigma >= 0.0, "invalid-scale", "gaussian sigma must be nonnegative");
        Stream s(seed, id);
        s.pos = pos;
        for (std::uint64_t i = 0; i < n; ++i) out[i] = s.next_gaussian(mu, sigma);
    });
}
int vxo_fastmath(int fn, const double* x, const double* y, std::uint64_t n, double* out) {
    return guarded([&] {
        for (std::uint64_t i = 0; i < n; ++i) switch (fn) {
                case 0: out[i] = log2_pos(x[i]); break;
                case 1: out[i] = ln_pos(x[i]); break;
                case 2: out[i] = exp2_clamped(x[i]); break;
                case 3: out[i] = sinpi(x[i]); break;
                case 4: out[i] = cospi(x[i]); break;
                case 5: out[i] = pow_pos(x[i], y[i]); break;
                default: raise("invalid-argument", "unknown fastmath function");
            }
    });
}
int vxo_quantile(const double* sample, std::uint64_t n, double level, double* out) {
    return guarded([&] { *out = quantile(sample, n, level); });
}
int vxo_logsumexp(const double* x, std::uint64_t n, double* out) {
    return guarded([&] { *out = logsumexp(x, n); });
}
int vxo_sample_covariance(const double* data, std::uint64_t rows, std::uint64_t dim, double* cov) {
    return guarded([&] { sample_covariance(data, rows, dim, cov); });
}
int vxo_cholesky(double* a, std::uint64_t dim) { return cholesky(a, dim) ? 0 : 1; }
int vxo_partition(std::uint64_t total, std::uint64_t workers, std::uint64_t width,
                  std::uint64_t* ranges) {
    return guarded([&] { partition(total, workers, width, ranges); });
}
double vxo_discrepancy(const double* sim, const double* obs, std::uint64_t n) {
    return discrepancy<double>(sim, obs, n);
}

// --------------------------------------------------------------- ABC (C0/C1)
// run_prior_predictive: abc.cpp:26-73, rows [first, first+count) of n_total.
// key->mode VXB_KEY_WORKER reproduces the reference keying; VXB_KEY_PARTICLE
// gives row i the stream (seed, i).  external_noise: count x steps doubles.
int vxo_abc_prior_predictive(const vxb_model* m, const vxb_keying* key, std::uint64_t n_total,
                             std::uint64_t first, std::uint64_t count, const double* observed,
                             double* params, double* summaries, double* rho, std::uint8_t* failed,
                             const double* external_noise, unsigned threads) {
    return guarded([&] {
        require(n_total >= 1, "invalid-shape", "need at least one prior predictive sample");
        require(first + count <= n_total, "invalid-shape", "row range exceeds the job");
        if (m->model == VXB_MODEL_TOGGLE) {
            toggle_prior_predictive(m, key, n_total, first, count, observed, params, summaries, rho,
                                    failed, threads);
            return;
        }
        const Logistic lg(*m);
        const std::size_t sd = lg.n_obs;
        std::vector<double> obs(observed, observed + sd);
        const bool f32 = m->precision == VXB_F32;
        if (f32)
            for (double& v : obs) v = static_cast<double>(static_cast<float>(v));
        std::vector<std::uint64_t> ranges;
        if (key->mode == VXB_KEY_WORKER) {
            require(key->workers >= 1, "invalid-shape", "need at least one worker");
            require(supported_width(key->block_width), "invalid-shape", "unsupported block width");
            ranges.resize(2 * key->workers);
            partition(n_total, key->workers, key->block_width, ranges.data());
        }
        parallel_for(count, threads, [&](std::uint64_t r) {
            const std::uint64_t row = first + r;
            std::uint64_t id = row, base = 0;
            if (key->mode == VXB_KEY_WORKER) {
                std::uint64_t w = 0;
                while (!(row >= ranges[2 * w] && row < ranges[2 * w + 1])) ++w;
                id = w;
                base = (row - ranges[2 * w]) * lg.row_stride();
            }
            Stream s(key->seed, id);
            s.pos = base;
            double theta[3], dist;
            std::uint8_t bad;
            std::vector<double> summary(sd);
            const double* ext = external_noise ? external_noise + r * lg.steps : nullptr;
            if (f32)
                abc_row<float>(lg, s, obs.data(), ext, theta, summary.data(), &dist, &bad);
            else
                abc_row<double>(lg, s, obs.data(), ext, theta, summary.data(), &dist, &bad);
            if (params) std::copy(theta, theta + 3, params + r * 3);
            if (summaries) std::copy(summary.begin(), summary.end(), summaries + r * sd);
            if (rho) rho[r] = dist;
            if (failed) failed[r] = bad;
        });
    });
}

int vxo_simulate_at(const vxb_model* m, const double* theta, std::uint64_t seed, std::uint64_t id,
                    std::uint64_t pos, double* summary) {
    return guarded([&] {
        if (m->model == VXB_MODEL_TOGGLE) {  // bench.cpp:69-77 (block width 1: no padding)
            const Toggle tg(*m);
            require(tg.steps >= 2, "invalid-horizon", "toggle simulation needs at least two time points");
            require(tg.cells >= 19, "insufficient-data", "need at least 19 observations for the quantile summary");
            Stream st(seed, id);
            st.pos = pos;
            st.align_even();
            tg.summaries(theta, st, 1, summary);
            return;
        }
        const Logistic lg(*m);
        Stream s(seed, id);
        s.pos = pos;
        s.align_even();
        double th[3] = {theta[0], theta[1], theta[2]};
        bool ok;
        if (m->precision == VXB_F32) {
            for (double& v : th) v = static_cast<double>(static_cast<float>(v));
            ok = lg.simulate<float>(th, [&](std::uint32_t) { return s.next_gaussian(0.0, 1.0); },
                                    summary);
        } else {
            ok = lg.simulate<double>(th, [&](std::uint32_t) { return s.next_gaussian(0.0, 1.0); },
                                     summary);
        }
        require(ok, "invalid-state", "state left the reals");
    });
}

// select_epsilon: abc.cpp:75-97
int vxo_select_epsilon(const double* rho, const std::uint8_t* failed, std::uint64_t n, double q,
                       double* eps, std::uint64_t cap, std::uint64_t* n_acc, std::uint64_t* idx) {
    return guarded([&] {
        require(q > 0.0 && q <= 1.0, "invalid-argument", "accept fraction must lie in (0, 1]");
        std::vector<double> v;
        v.reserve(n);
        for (std::uint64_t r = 0; r < n; ++r)
            if (!(failed && failed[r])) v.push_back(rho[r]);
        require(!v.empty(), "empty-set", "every prior predictive row failed");
        std::sort(v.begin(), v.end());
        double e = quantile_sorted(v.data(), v.size(), q);
        const std::size_t min_accept =
            static_cast<std::size_t>(std::ceil(q * static_cast<double>(v.size())));
        if (min_accept >= 1 && e < v[min_accept - 1]) e = v[min_accept - 1];
        *eps = e;
        std::uint64_t k = 0;
        for (std::uint64_t r = 0; r < n; ++r)
            if (!(failed && failed[r]) && rho[r] <= e) {
                if (idx && k < cap) idx[k] = r;
                ++k;
            }
        *n_acc = k;
    });
}

// ------------------------------------------------------------ p-values (C2)
// Draw order of weak_info.cpp:82-106 (align_even; Gaussian prior draw taking
// one pair; then the data) and the counting rule of estimate_pvalues,
// weak_info.cpp:108-120 (value <= observed, ties count).
int vxo_ppp_pvalues(const vxb_model* m, const double* lambda, const double* log_norm,
                    std::uint32_t n_lambda, std::uint64_t m_total, std::uint64_t first,
                    std::uint64_t count, std::uint64_t seed, double ybar_obs,
                    std::uint64_t* counts, double* pvalues, double* ybar_out, unsigned threads) {
    return guarded([&] {
        require(m->model == VXB_MODEL_NORMAL_MEAN, "invalid-argument", "not the normal-mean model");
        require(m->steps >= 1, "insufficient-data", "need at least one observation per dataset");
        require(n_lambda >= 1 && m_total >= 1 && first + count <= m_total, "invalid-shape",
                "bad lambda grid or dataset range");
        const std::uint64_t n = m->steps;
        const double dn = static_cast<double>(n);
        for (std::uint32_t k = 0; k < n_lambda; ++k) {
            require(lambda[k] >= 0.0, "invalid-argument", "prior scales must be nonnegative");
            const double v = lambda[k] * lambda[k] + 1.0 / dn;
            const double logm_obs = log_norm[k] - ((0.5 * ybar_obs) * ybar_obs) / v;
            const std::uint64_t sk = derive_seed1(seed, k);
            std::vector<std::uint64_t> part(std::max(1u, threads), 0);
            const unsigned nt = std::max(1u, threads);
            std::vector<std::thread> pool;
            auto body = [&](unsigned t) {
                std::uint64_t c = 0;
                for (std::uint64_t j = t; j < count; j += nt) {
                    Stream s(sk, first + j);
                    s.align_even();
                    const double theta = lambda[k] * s.next_gaussian(0.0, 1.0);
                    s.pos = 2;  // second half of the prior pair is discarded
                    double sum = 0.0;
                    for (std::uint64_t i = 0; i < n; ++i) sum += theta + s.next_gaussian(0.0, 1.0);
                    const double ybar = sum / dn;
                    if (ybar_out) ybar_out[static_cast<std::uint64_t>(k) * count + j] = ybar;
                    const double logm = log_norm[k] - ((0.5 * ybar) * ybar) / v;
                    if (logm <= logm_obs) ++c;
                }
                part[t] = c;
            };
            if (nt == 1) {
                body(0);
            } else {
                for (unsigned t = 0; t < nt; ++t) pool.emplace_back(body, t);
                for (auto& th : pool) th.join();
            }
            std::uint64_t c = 0;
            for (std::uint64_t v2 : part) c += v2;
            counts[k] = c;
            if (pvalues) pvalues[k] = static_cast<double>(c) / static_cast<double>(m_total);
        }
    });
}

// estimate_pvalues: weak_info.cpp:108-120; compute_cutoff: :122-125
int vxo_estimate_pvalues(const double* base, std::uint64_t nb, const double* k, std::uint64_t nk,
                         double* out) {
    return guarded([&] {
        require(nk >= 1, "invalid-argument", "need at least one comparison evidence");
        std::vector<double> sorted(k, k + nk);
        std::sort(sorted.begin(), sorted.end());
        for (std::uint64_t i = 0; i < nb; ++i) {
            const auto it = std::upper_bound(sorted.begin(), sorted.end(), base[i]);
            out[i] = static_cast<double>(it - sorted.begin()) / static_cast<double>(nk);
        }
    });
}
int vxo_compute_cutoff(const double* p, std::uint64_t n, double alpha, double* out) {
    return guarded([&] {
        require(alpha > 0.0 && alpha < 1.0, "invalid-argument", "alpha must lie in (0, 1)");
        *out = quantile(p, n, alpha);
    });
}

// ------------------------------------------------ libm exp, restated
// std::exp is what the reference's weight algebra calls (smc.cpp:214,278,299,
// numeric.cpp:16-17).  The oracle itself keeps calling std::exp; this restatement of
// the algorithm behind it (glibc >= 2.28: N = 128 table, degree-5 polynomial, the
// multiply-adds contracted as the x86-64 FMA build evaluates them) exists so that the
// device copy of the same algorithm (csrc/vxb_libmexp.cuh) can be pinned: restated ==
// std::exp on this machine (tests/test_oracle_pins.py), device == restated == std::exp
// on the GPU box (tests/test_gpu_workloads.py).
struct ExpEntry {
    std::uint64_t tail, sbits;
};
static const ExpEntry kExpTable[128] = {
#define VXB_EXP_PAIR(a, b) {a, b}
#include "../paper_1902_09046_b200/csrc/vxb_libm_exp_entries.inc"
#undef VXB_EXP_PAIR
};
// fused = true: the FMA build of the library (a*b + c contracted where the x86-64 FMA
// build contracts it); fused = false: its plain build (this file is compiled with
// -ffp-contract=off, so a * b + c rounds twice).
static double exp_mad(bool fused, double a, double b, double c) {
    return fused ? std::fma(a, b, c) : a * b + c;
}
static double exp_restated_special(bool fused, double tmp, std::uint64_t sbits, std::uint64_t ki) {
    if ((ki & 0x80000000ULL) == 0) {
        sbits -= 1009ULL << 52;
        const double scale = bit_cast<double>(sbits);
        return 0x1p1009 * exp_mad(fused, scale, tmp, scale);
    }
    sbits += 1022ULL << 52;
    const double scale = bit_cast<double>(sbits);
    const double m = scale * tmp;
    double y = scale + m;
    if (y < 1.0) {
        const double hi = 1.0 + y;
        const double lo = (scale - y) + m;
        double t = (1.0 - hi) + y;
        t = t + lo;
        y = (t + hi) - 1.0;
        if (y == 0.0) y = 0.0;
    }
    return 0x1p-1022 * y;
}
static double exp_restated(double x, bool fused = true) {
    const std::uint32_t abstop = static_cast<std::uint32_t>(bit_cast<std::uint64_t>(x) >> 52) & 0x7ffu;
    bool special = false;
    if (abstop - 0x3c9u >= 0x3fu) {
        if (static_cast<std::int32_t>(abstop - 0x3c9u) < 0) return 1.0 + x;
        if (abstop >= 0x409u) {
            if (bit_cast<std::uint64_t>(x) == 0xfff0000000000000ULL) return 0.0;
            if (abstop >= 0x7ffu) return 1.0 + x;
            return x < 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
        }
        special = true;
    }
    double kd = exp_mad(fused, x, 0x1.71547652b82fep+7, 0x1.8p+52);
    const std::uint64_t ki = bit_cast<std::uint64_t>(kd);
    kd -= 0x1.8p+52;
    double r = exp_mad(fused, kd, -0x1.62e42fefa0000p-8, x);
    r = exp_mad(fused, kd, -0x1.cf79abc9e3b3ap-47, r);
    const ExpEntry e = kExpTable[ki & 127u];
    const std::uint64_t sbits = e.sbits + (ki << 45);
    const double tail = bit_cast<double>(e.tail);
    const double r2 = r * r;
    const double p23 = exp_mad(fused, 0x1.555555555543cp-3, r, 0x1.ffffffffffdbdp-2);
    const double t1 = tail + r;
    const double p45 = exp_mad(fused, r, 0x1.1111167a4d017p-7, 0x1.55555cf172b91p-5);
    const double t2 = exp_mad(fused, p23, r2, t1);
    const double tmp = exp_mad(fused, r2 * r2, p45, t2);
    if (special) return exp_restated_special(fused, tmp, sbits, ki);
    const double scale = bit_cast<double>(sbits);
    return exp_mad(fused, scale, tmp, scale);
}

// libm exp restatement: out[i] = exp_restated(x[i]); libm[i] = std::exp(x[i]) (optional)
int vxo_exp_restated(const double* x, std::uint64_t n, double* out, double* libm, int plain_build) {
    return guarded([&] {
        for (std::uint64_t i = 0; i < n; ++i) {
            out[i] = exp_restated(x[i], plain_build == 0);
            if (libm) libm[i] = std::exp(x[i]);
        }
    });
}
// n pseudo-random arguments (splitmix64 of seed + i mapped to [lo, hi)): how many
// differ between the restatement and the live std::exp (bitwise; NaN never occurs);
// *first_bad receives the first offending argument.
int vxo_exp_restated_sweep(std::uint64_t seed, std::uint64_t n, double lo, double hi,
                           unsigned threads, std::uint64_t* mismatches, double* first_bad,
                           int plain_build) {
    return guarded([&] {
        if (threads == 0) threads = 1;
        std::vector<std::uint64_t> bad(threads, 0);
        std::vector<double> firsts(threads, std::numeric_limits<double>::quiet_NaN());
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                for (std::uint64_t i = t; i < n; i += threads) {
                    const double u = static_cast<double>(splitmix64(seed + i) >> 11) * 0x1p-53;
                    const double x = lo + u * (hi - lo);
                    const double a = exp_restated(x, plain_build == 0), b = std::exp(x);
                    if (bit_cast<std::uint64_t>(a) != bit_cast<std::uint64_t>(b)) {
                        if (bad[t]++ == 0) firsts[t] = x;
                    }
                }
            });
        for (auto& th : pool) th.join();
        *mismatches = 0;
        for (unsigned t = 0; t < threads; ++t) {
            *mismatches += bad[t];
            if (bad[t] && std::isnan(*first_bad)) *first_bad = firsts[t];
        }
    });
}
// -------------------------------------------------------------- SMC pieces
// ess: smc.cpp:208-219
int vxo_ess(const double* lw, std::uint64_t n, double* out) {
    return guarded([&] {
        double m = -std::numeric_limits<double>::infinity();
        for (std::uint64_t i = 0; i < n; ++i) m = std::max(m, lw[i]);
        require(m > -std::numeric_limits<double>::infinity(), "degenerate-ensemble",
                "all weights are zero");
        double s1 = 0.0, s2 = 0.0;
        for (std::uint64_t i = 0; i < n; ++i) {
            const double e = std::exp(lw[i] - m);
            s1 += e;
            s2 += e * e;
        }
        *out = s1 * s1 / s2;
    });
}
// resample_multinomial: smc.cpp:268-300 (draw i = position i of the stream)
int vxo_resample_multinomial(std::uint64_t n, std::uint32_t dim, const double* log_w,
                             const double* particles, std::uint64_t seed, std::uint64_t id,
                             double* particles_out, std::uint64_t* ancestors) {
    return guarded([&] {
        double m = -std::numeric_limits<double>::infinity();
        for (std::uint64_t i = 0; i < n; ++i) m = std::max(m, log_w[i]);
        require(m > -std::numeric_limits<double>::infinity(), "degenerate-ensemble",
                "all weights are zero");
        std::vector<double> cum(n);
        double run = 0.0;
        for (std::uint64_t i = 0; i < n; ++i) {
            run += std::exp(log_w[i] - m);
            cum[i] = run;
        }
        require(std::isfinite(run) && run > 0.0, "degenerate-ensemble", "weight sum is not finite");
        Stream s(seed, id);
        for (std::uint64_t i = 0; i < n; ++i) {
            const double target = s.next_unit() * run;
            const std::uint64_t a = upper_bound_idx(cum.data(), n, target);
            if (ancestors) ancestors[i] = a;
            if (particles_out)
                std::copy_n(particles + a * dim, dim, particles_out + i * dim);
        }
    });
}

// ----------------------------------------------------------- ABC-SMC (C3)
// NOT IN THE REFERENCE (SPEC.md:353 lists ABC-SMC as a non-goal): the scheme
// below is this repository's definition, assembled
// from reference pieces: inverse-CDF ancestors (smc.cpp:286-290), proposal
// theta + L z with inc_k = sum_{m<=k} L[k][m] z_m (smc.cpp:115-119), Cholesky +
// jitter (numeric.cpp:81-96, smc.cpp:318-323), type-7 quantile
// (numeric.cpp:20-36), zero prior density => reject (smc.cpp:131).

// Weighted moments with the canonical two-level sums.  w is normalised.
// cov = sum w d d^T / (1 - sum w^2)  (equals the n-1 divisor for equal weights,
// numeric.cpp:55-79).  Returns sum w^2.
double vxo_weighted_moments_impl(const double* theta, const double* w, std::size_t n,
                                 std::size_t dim, double* mean, double* cov) {
    for (std::size_t a = 0; a < dim; ++a)
        mean[a] = canon_sum(n, [&](std::size_t i) { return w[i] * theta[i * dim + a]; });
    const double s2 = canon_sum(n, [&](std::size_t i) { return w[i] * w[i]; });
    const double denom = 1.0 - s2;
    for (std::size_t a = 0; a < dim; ++a)
        for (std::size_t b = 0; b <= a; ++b) {
            const double c = canon_sum(n, [&](std::size_t i) {
                return (w[i] * (theta[i * dim + a] - mean[a])) * (theta[i * dim + b] - mean[b]);
            });
            cov[a * dim + b] = c / denom;
            cov[b * dim + a] = cov[a * dim + b];
        }
    return s2;
}
int vxo_weighted_moments(const double* theta, const double* w, std::uint64_t n, std::uint32_t dim,
                         double* mean, double* cov, double* sum_w2) {
    return guarded([&] {
        require(n >= 2, "insufficient-data", "covariance needs at least two rows");
        const double s2 = vxo_weighted_moments_impl(theta, w, n, dim, mean, cov);
        if (sum_w2) *sum_w2 = s2;
    });
}
int vxo_canon_cumsum(const double* w, std::uint64_t n, double* cum) {
    return guarded([&] { canon_cumsum(w, n, cum); });
}
double vxo_canon_sum(const double* w, std::uint64_t n) {
    return canon_sum(n, [&](std::size_t i) { return w[i]; });
}

// kernel factor: scale * cov, Cholesky, jitter on failure (smc.cpp:311-325)
int vxo_make_kernel(const double* cov, std::uint32_t dim, double scale, double jitter,
                    double* chol) {
    return guarded([&] {
        std::vector<double> c(cov, cov + dim * dim);
        for (double& v : c) v = scale * v;
        std::copy(c.begin(), c.end(), chol);
        if (!cholesky(chol, dim)) {
            for (std::uint32_t k = 0; k < dim; ++k) c[k * dim + k] += jitter;
            std::copy(c.begin(), c.end(), chol);
            require(cholesky(chol, dim), "degenerate-ensemble",
                    "covariance is rank deficient beyond jitter");
        }
    });
}

// One proposal p of generation gen >= 1; stream RngStream(derive_seed(seed,{gen}), p):
//   position 0       ancestor uniform (inverse CDF over cum_prev)
//   positions 2..2+d_e-1   the d Gaussian increments (pair aligned, d_e = d + d%2)
//   position 2+d_e+j standard normal of simulation step j+1
// flag: 1 accepted, 0 rejected by distance, 2 outside the prior box, 3 failed.
int vxo_abcsmc_propose(const vxb_model* m, std::uint64_t seed, std::uint32_t gen,
                       std::uint64_t first, std::uint64_t count, std::uint64_t n_prev,
                       const double* theta_prev, const double* cum_prev, const double* chol,
                       const double* observed, double epsilon, double* theta_out, double* rho_out,
                       std::uint8_t* flag_out, unsigned threads) {
    return guarded([&] {
        const Logistic lg(*m);
        require(gen >= 1, "invalid-argument", "generation 0 is the prior predictive set");
        require(n_prev >= 1, "insufficient-data", "empty previous population");
        const std::uint64_t sg = derive_seed1(seed, gen);
        const std::size_t d = 3, de = 4;
        parallel_for(count, threads, [&](std::uint64_t r) {
            Stream s(sg, first + r);
            const double target = s.next_unit() * cum_prev[n_prev - 1];
            const std::size_t a = upper_bound_idx(cum_prev, n_prev, target);
            s.align_even();
            double z[4];
            for (std::size_t k = 0; k < de; ++k) z[k] = s.next_gaussian(0.0, 1.0);
            double th[3];
            bool inside = true;
            for (std::size_t k = 0; k < d; ++k) {
                double inc = 0.0;
                for (std::size_t q = 0; q <= k; ++q) inc += chol[k * d + q] * z[q];
                th[k] = theta_prev[a * d + k] + inc;
                inside = inside && th[k] >= lg.lo[k] && th[k] < lg.hi[k];
            }
            std::uint8_t flag;
            double dist = std::numeric_limits<double>::quiet_NaN();
            if (!inside) {
                flag = 2;
            } else {
                std::vector<double> summary(lg.n_obs);
                const bool ok = lg.simulate<double>(
                    th, [&](std::uint32_t) { return s.next_gaussian(0.0, 1.0); }, summary.data());
                if (!ok) {
                    flag = 3;
                } else {
                    dist = discrepancy<double>(summary.data(), observed, lg.n_obs);
                    flag = dist <= epsilon ? 1 : 0;
                }
            }
            std::copy(th, th + d, theta_out + r * d);
            rho_out[r] = dist;
            flag_out[r] = flag;
        });
    });
}

// Unnormalised importance weight of new particle i: 1 / sum_j w_j exp(-q_ij/2),
// q = |L^-1 (theta_i - theta_j)|^2 by forward substitution with reciprocal
// pivots, exp through exp2_clamped (fastmath.hpp:57-79); j summed in index order.
int vxo_abcsmc_weights(std::uint32_t dim, std::uint64_t count, const double* theta_new, std::uint64_t n_prev, const double* theta_prev,
                       const double* w_prev, const double* chol, double* w_out, unsigned threads) {
    return guarded([&] {
        require(dim >= 1 && dim <= 8, "invalid-shape", "dimension out of range");
        double invd[8];
        for (std::uint32_t k = 0; k < dim; ++k) invd[k] = 1.0 / chol[k * dim + k];
        parallel_for(count, threads, [&](std::uint64_t r) {
            const double* ti = theta_new + r * dim;
            double sum = 0.0;
            for (std::uint64_t j = 0; j < n_prev; ++j) {
                double y[8];
                double q = 0.0;
                for (std::uint32_t k = 0; k < dim; ++k) {
                    double v = ti[k] - theta_prev[j * dim + k];
                    for (std::uint32_t c = 0; c < k; ++c) v -= chol[k * dim + c] * y[c];
                    y[k] = v * invd[k];
                    q += y[k] * y[k];
                }
                sum += w_prev[j] * exp2_clamped((-0.5 * q) * kInvLn2);
            }
            w_out[r] = 1.0 / sum;
        });
    });
}

// Full ABC-SMC run.  Generation 0: proposals are prior draws keyed
// RngStream(derive_seed(seed,{0}), p) (run_prior_predictive row layout), all
// non-failed rows accepted, equal weights.  Generation g>=1: epsilon_g = type-7
// quantile of the previous rho; kernel = chol(scale * weighted cov); proposals
// evaluated in rounds of round_size until at least N are accepted; the first N
// accepted by proposal index form the population; weights normalised by the
// canonical sum.
int vxo_abcsmc_run(const vxb_model* m, const vxb_abcsmc_cfg* cfg, const double* observed,
                   vxb_abcsmc_out* out, unsigned threads) {
    return guarded([&] {
        const Logistic lg(*m);
        const std::uint64_t n = cfg->particles;
        const std::size_t d = 3;
        require(n >= 2, "insufficient-data", "need at least two particles");
        require(cfg->generations >= 1, "invalid-argument", "need at least one generation");
        require(cfg->quantile > 0.0 && cfg->quantile <= 1.0, "invalid-argument",
                "quantile must lie in (0, 1]");
        const std::uint64_t round = cfg->round_size ? cfg->round_size : n;
        const std::uint64_t max_rounds = cfg->max_rounds ? cfg->max_rounds : 1000;
        std::vector<double> theta(n * d), w(n), rho(n), cum(n);
        std::vector<double> th_new(n * d), rho_new(n), w_new(n);
        std::vector<double> p_theta(round * d), p_rho(round);
        std::vector<std::uint8_t> p_flag(round);
        for (std::uint32_t g = 0; g < cfg->generations; ++g) {
            double eps = std::numeric_limits<double>::infinity();
            double chol[9] = {0};
            if (g >= 1) {
                eps = quantile(rho.data(), n, cfg->quantile);
                double mean[3], cov[9];
                vxo_weighted_moments_impl(theta.data(), w.data(), n, d, mean, cov);
                require(vxo_make_kernel(cov, d, cfg->kernel_scale, cfg->jitter, chol) == 0,
                        "degenerate-ensemble", "covariance is rank deficient beyond jitter");
                canon_cumsum(w.data(), n, cum.data());
            }
            std::uint64_t got = 0, evaluated = 0, accepted_total = 0;
            for (std::uint64_t t = 0; t < max_rounds && got < n; ++t) {
                if (g == 0) {
                    vxb_keying key{VXB_KEY_PARTICLE, 1, 1, 0, derive_seed1(cfg->seed, 0)};
                    std::vector<std::uint8_t> failed(round);
                    const std::uint64_t total = (t + 1) * round;
                    require(vxo_abc_prior_predictive(m, &key, total, t * round, round, observed,
                                                     p_theta.data(), nullptr, p_rho.data(),
                                                     failed.data(), nullptr, threads) == 0,
                            "internal", "prior predictive failed");
                    for (std::uint64_t r = 0; r < round; ++r) p_flag[r] = failed[r] ? 3 : 1;
                } else {
                    require(vxo_abcsmc_propose(m, cfg->seed, g, t * round, round, n, theta.data(),
                                               cum.data(), chol, observed, eps, p_theta.data(),
                                               p_rho.data(), p_flag.data(), threads) == 0,
                            "internal", "propose failed");
                }
                evaluated += round;
                for (std::uint64_t r = 0; r < round; ++r) {
                    if (p_flag[r] != 1) continue;
                    ++accepted_total;
                    if (got < n) {
                        std::copy_n(p_theta.data() + r * d, d, th_new.data() + got * d);
                        rho_new[got] = p_rho[r];
                        ++got;
                    }
                }
            }
            require(got == n, "empty-set", "generation did not fill within max_rounds");
            if (g == 0) {
                for (std::uint64_t i = 0; i < n; ++i) w_new[i] = 1.0 / static_cast<double>(n);
            } else {
                require(vxo_abcsmc_weights(d, n, th_new.data(), n, theta.data(), w.data(), chol,
                                           w_new.data(), threads) == 0,
                        "internal", "weights failed");
                const double total = canon_sum(n, [&](std::size_t i) { return w_new[i]; });
                require(std::isfinite(total) && total > 0.0, "degenerate-ensemble",
                        "weight sum is not finite");
                for (std::uint64_t i = 0; i < n; ++i) w_new[i] = w_new[i] / total;
            }
            theta.swap(th_new);
            rho.swap(rho_new);
            w.swap(w_new);
            double mean[3], cov[9];
            const double s2 = vxo_weighted_moments_impl(theta.data(), w.data(), n, d, mean, cov);
            if (out->epsilon) out->epsilon[g] = eps;
            if (out->ess) out->ess[g] = 1.0 / s2;
            if (out->accept_rate)
                out->accept_rate[g] =
                    static_cast<double>(accepted_total) / static_cast<double>(evaluated);
            if (out->proposals) out->proposals[g] = evaluated;
            if (out->mean) std::copy(mean, mean + d, out->mean + g * d);
            if (out->cov) std::copy(cov, cov + d * d, out->cov + g * d * d);
        }
        if (out->theta) std::copy(theta.begin(), theta.end(), out->theta);
        if (out->weight) std::copy(w.begin(), w.end(), out->weight);
        if (out->rho) std::copy(rho.begin(), rho.end(), out->rho);
    });
}

// ------------------------------------------------- tau-leap MLMC (C4)
// NOT IN THE REFERENCE (tau-leap is out of scope; no Poisson
// sampler in rng.cpp).  Defined here in the style of tb_model.cpp:39-116
// (propensities from the state, uniforms through next_unit, rate <= 0 guard
// :57-60):
//  * Poisson(lam) by CDF inversion from one uniform: p0 = exp(-lam) through
//    exp2_clamped, p_k = (p_{k-1} * lam) * (1/k), at most 1023 terms;
//  * propensities from max(X, 0): a1 = (k1*S)*E, a2 = k2*C, a3 = k3*C;
//  * level 0: plain tau-leap, step s uses positions 4s + r (r = reaction);
//  * level l >= 1: Anderson-Higham coupling of a fine path (tau_l) and a coarse
//    path (M tau_l): per fine step and reaction r, with the coarse propensity
//    frozen over the coarse step: m = min(af, ac), P1 ~ Poi(m tau),
//    P2 ~ Poi((af-m) tau), P3 ~ Poi((ac-m) tau); reaction r of fine step s owns
//    the Philox block 3s + r: position 6s + 2r drives P1, position 6s + 2r + 1 the
//    residual (at most one of P2, P3 has a positive rate, so they share it);
//    fine fires P1+P2, coarse fires P1+P3;
//  * path `i` of level l owns RngStream(derive_seed(seed,{l}), i).
static int poisson_inv(double lam, double u, std::int64_t* iters) {
    if (!(lam > 0.0)) return 0;
    double p = exp2_clamped((-lam) * kInvLn2);
    double cdf = p;
    int k = 0;
    while (u > cdf && k < 1023) {
        ++k;
        p = (p * lam) * (1.0 / static_cast<double>(k));
        cdf += p;
        ++*iters;
    }
    return k;
}

struct MM {
    std::int32_t s, e, c, p;
    void fire(int k1, int k2, int k3) {
        s += -k1 + k2;
        e += -k1 + k2 + k3;
        c += k1 - k2 - k3;
        p += k3;
    }
    void prop(const double* k, double* a) const {
        const double ds = static_cast<double>(s > 0 ? s : 0);
        const double de = static_cast<double>(e > 0 ? e : 0);
        const double dc = static_cast<double>(c > 0 ? c : 0);
        a[0] = (k[0] * ds) * de;
        a[1] = k[1] * dc;
        a[2] = k[2] * dc;
    }
};

int vxo_mlmc_level(const vxb_model* m, const vxb_mlmc_cfg* cfg, std::uint32_t level,
                   std::uint64_t first, std::uint64_t count, std::int64_t* sums,
                   std::int32_t* y_out, unsigned threads) {
    return guarded([&] {
        require(m->model == VXB_MODEL_MM_TAULEAP, "invalid-argument", "not the tau-leap model");
        require(cfg->refine >= 2 && level < cfg->levels, "invalid-argument", "bad level");
        require(cfg->tau0 > 0.0 && cfg->t_end > 0.0, "invalid-horizon", "need a positive horizon");
        const std::uint64_t steps0 = static_cast<std::uint64_t>(std::llround(cfg->t_end / cfg->tau0));
        require(steps0 >= 1, "invalid-horizon", "need at least one step");
        std::uint64_t nf = steps0;
        for (std::uint32_t l = 0; l < level; ++l) nf *= cfg->refine;
        const double tau = cfg->t_end / static_cast<double>(nf);
        const double kr[3] = {m->consts[4], m->consts[5], m->consts[6]};
        const MM init{static_cast<std::int32_t>(m->consts[0]), static_cast<std::int32_t>(m->consts[1]),
                      static_cast<std::int32_t>(m->consts[2]), static_cast<std::int32_t>(m->consts[3])};
        const std::uint64_t sl = derive_seed1(cfg->seed, level);
        const unsigned nt = std::max(1u, threads);
        std::vector<std::int64_t> acc(4 * nt, 0);
        auto body = [&](unsigned t) {
            std::int64_t sy = 0, sy2 = 0, sp = 0, it = 0;
            for (std::uint64_t r = t; r < count; r += nt) {
                Stream s(sl, first + r);
                MM f = init, c = init;
                double af[3], ac[3];
                if (level == 0) {
                    for (std::uint64_t st = 0; st < nf; ++st) {
                        f.prop(kr, af);
                        int k[3];
                        for (int q = 0; q < 3; ++q) {
                            s.pos = 4 * st + q;
                            k[q] = poisson_inv(af[q] * tau, s.next_unit(), &it);
                        }
                        f.fire(k[0], k[1], k[2]);
                    }
                } else {
                    for (std::uint64_t st = 0; st < nf; ++st) {
                        if (st % cfg->refine == 0) c.prop(kr, ac);
                        f.prop(kr, af);
                        int kf[3], kc[3];
                        for (int q = 0; q < 3; ++q) {
                            const double mn = af[q] < ac[q] ? af[q] : ac[q];
                            s.pos = 6 * st + 2 * q;
                            const double u1 = s.next_unit(), u2 = s.next_unit();
                            const int p1 = poisson_inv(mn * tau, u1, &it);
                            // at most one residual rate is positive: they share u2
                            const int p2 = poisson_inv((af[q] - mn) * tau, u2, &it);
                            const int p3 = poisson_inv((ac[q] - mn) * tau, u2, &it);
                            kf[q] = p1 + p2;
                            kc[q] = p1 + p3;
                        }
                        f.fire(kf[0], kf[1], kf[2]);
                        c.fire(kc[0], kc[1], kc[2]);
                    }
                }
                const std::int32_t y = level == 0 ? f.p : f.p - c.p;
                if (y_out) y_out[r] = y;
                sy += y;
                sy2 += static_cast<std::int64_t>(y) * y;
                sp += f.p;
            }
            acc[4 * t] = sy;
            acc[4 * t + 1] = sy2;
            acc[4 * t + 2] = sp;
            acc[4 * t + 3] = it;
        };
        if (nt == 1) {
            body(0);
        } else {
            std::vector<std::thread> pool;
            for (unsigned t = 0; t < nt; ++t) pool.emplace_back(body, t);
            for (auto& th : pool) th.join();
        }
        for (int q = 0; q < 4; ++q) {
            sums[q] = 0;
            for (unsigned t = 0; t < nt; ++t) sums[q] += acc[4 * t + q];
        }
    });
}

// Estimator: sum over levels of the sample mean of Y_l; variance of the
// estimator = sum var_l / paths (n-1 divisor, numeric.cpp:45-51).
int vxo_mlmc_tauleap(const vxb_model* m, const vxb_mlmc_cfg* cfg, vxb_mlmc_out* out,
                     unsigned threads) {
    return guarded([&] {
        require(cfg->paths >= 2, "insufficient-data", "variance needs at least two values");
        double est = 0.0, var = 0.0;
        std::uint64_t steps = static_cast<std::uint64_t>(std::llround(cfg->t_end / cfg->tau0));
        for (std::uint32_t l = 0; l < cfg->levels; ++l) {
            std::int64_t sums[4];
            require(vxo_mlmc_level(m, cfg, l, 0, cfg->paths, sums, nullptr, threads) == 0,
                    "internal", "level failed");
            const double n = static_cast<double>(cfg->paths);
            const double mean = static_cast<double>(sums[0]) / n;
            const double v =
                (static_cast<double>(sums[1]) - static_cast<double>(sums[0]) * mean) / (n - 1.0);
            if (out->level_mean) out->level_mean[l] = mean;
            if (out->level_var) out->level_var[l] = v;
            if (out->level_cost)
                out->level_cost[l] = static_cast<double>(l == 0 ? steps : steps + steps / cfg->refine);
            est += mean;
            var += v / n;
            steps *= cfg->refine;
        }
        out->estimate = est;
        out->std_error = std::sqrt(var);
    });
}

// Exact Gillespie (direct method) for the same network, restated from the
// event loop of tb_model.cpp:39-116 (total rate, exponential waiting time from
// one uniform through ln_pos, inverse-CDF reaction choice from a second).
// Anchor for the MLMC estimate only.  Path i owns RngStream(derive_seed(seed,{99}), i).
int vxo_mm_gillespie(const vxb_model* m, double t_end, std::uint64_t paths, std::uint64_t seed,
                     double* mean_p, double* var_p, unsigned threads) {
    return guarded([&] {
        const double kr[3] = {m->consts[4], m->consts[5], m->consts[6]};
        const MM init{static_cast<std::int32_t>(m->consts[0]), static_cast<std::int32_t>(m->consts[1]),
                      static_cast<std::int32_t>(m->consts[2]), static_cast<std::int32_t>(m->consts[3])};
        const std::uint64_t sg = derive_seed1(seed, 99);
        const unsigned nt = std::max(1u, threads);
        std::vector<std::int64_t> acc(2 * nt, 0);
        auto body = [&](unsigned t) {
            for (std::uint64_t r = t; r < paths; r += nt) {
                Stream s(sg, r);
                MM x = init;
                double now = 0.0;
                for (;;) {
                    double a[3];
                    x.prop(kr, a);
                    const double total = (a[0] + a[1]) + a[2];
                    if (!(total > 0.0)) break;
                    const double u = s.next_unit();
                    const double wait = -ln_pos(1.0 - u) / total;
                    now += wait;
                    if (now > t_end) break;
                    const double pick = s.next_unit() * total;
                    if (pick < a[0]) x.fire(1, 0, 0);
                    else if (pick < a[0] + a[1]) x.fire(0, 1, 0);
                    else x.fire(0, 0, 1);
                }
                acc[2 * t] += x.p;
                acc[2 * t + 1] += static_cast<std::int64_t>(x.p) * x.p;
            }
        };
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nt; ++t) pool.emplace_back(body, t);
        for (auto& th : pool) th.join();
        std::int64_t s1 = 0, s2 = 0;
        for (unsigned t = 0; t < nt; ++t) {
            s1 += acc[2 * t];
            s2 += acc[2 * t + 1];
        }
        const double n = static_cast<double>(paths);
        *mean_p = static_cast<double>(s1) / n;
        *var_p = (static_cast<double>(s2) - static_cast<double>(s1) * *mean_p) / (n - 1.0);
    });
}

// ------------------------- likelihood-annealed SMC on the bioassay model (8f-3)
// Restates, operation for operation, what the weak-informativity test runs for
// every (dataset, prior) pair: the model of weak_info.cpp:18-160 inside the
// adaptive sampler smc::run_smc (smc.cpp:352-488) with workers = 1, fixed scale
// (no ESJD).  Particles are independent given the iteration's temperature and
// kernel, and every variate has a fixed stream position (smc.cpp:66-76), so the
// loops below run over particles where the reference runs over lane blocks.
struct Bioassay {
    std::uint32_t groups;
    double dose[16], miss[16], hit[16], log_choose[16];
    double l1, l2, log_norm;
    // -log p = log(1 + e^b), weak_info.cpp:20-24
    static double softplus(double b) {
        const double pos = b > 0.0 ? b : 0.0;
        const double mag = b > 0.0 ? b : -b;
        return pos + ln_pos(1.0 + exp2_clamped(-mag * kInvLn2));
    }
    // ll_lane: weak_info.cpp:26-40
    double log_lik(double b0, double b1) const {
        double total = 0.0;
        for (std::uint32_t g = 0; g < groups; ++g) {
            const double b = b0 + b1 * dose[g];
            const double lse = softplus(b);
            total += log_choose[g];
            if (hit[g] > 0.0) total -= hit[g] * lse;
            if (miss[g] > 0.0) total += miss[g] * (b - lse);
        }
        return total;
    }
    // log_prior hook: weak_info.cpp:144-148
    double log_prior(double b0, double b1) const {
        const double a = b0 / l1;
        const double b = b1 / l2;
        return log_norm - 0.5 * (a * a + b * b);
    }
};

static Bioassay make_bioassay(const double* dose, const std::uint32_t* group_size,
                              const std::uint32_t* deaths, std::uint32_t groups, double l1,
                              double l2) {
    require(groups >= 1 && groups <= 16, "invalid-argument", "between 1 and 16 dose groups");
    require(l1 > 0.0 && l2 > 0.0, "invalid-argument", "prior scales must be positive");
    Bioassay m{};
    m.groups = groups;
    m.l1 = l1;
    m.l2 = l2;
    m.log_norm = -std::log(2.0 * 3.141592653589793238462643 * l1 * l2);  // weak_info.cpp:135
    for (std::uint32_t g = 0; g < groups; ++g) {
        require(deaths[g] <= group_size[g], "invalid-argument", "more deaths than animals in a group");
        m.dose[g] = dose[g];
        m.hit[g] = deaths[g];
        m.miss[g] = group_size[g] - deaths[g];
        // log_binomial: numeric.cpp:98-102
        m.log_choose[g] = std::lgamma(group_size[g] + 1.0) - std::lgamma(deaths[g] + 1.0) -
                          std::lgamma(static_cast<double>(group_size[g] - deaths[g]) + 1.0);
    }
    return m;
}

// sample_prior_predictive (weak_info.cpp:82-106) from RngStream(seed, 0)
static void bioassay_draw(double l1, double l2, const double* dose, const std::uint32_t* group_size,
                          std::uint32_t groups, std::uint64_t seed, double* theta,
                          std::uint32_t* deaths) {
    require(l1 >= 0.0 && l2 >= 0.0, "invalid-argument", "prior scales must be nonnegative");
    Stream s(seed, 0);
    s.align_even();
    const double z0 = s.next_gaussian(0.0, 1.0), z1 = s.next_gaussian(0.0, 1.0);
    theta[0] = l1 * z0;
    theta[1] = l2 * z1;
    for (std::uint32_t g = 0; g < groups; ++g) {
        const double b = theta[0] + theta[1] * dose[g];
        const double p = exp2_clamped(-Bioassay::softplus(b) * kInvLn2);
        std::uint32_t k = 0;
        for (std::uint32_t j = 0; j < group_size[g]; ++j) k += s.next_unit() < p ? 1 : 0;
        deaths[g] = k;
    }
}

struct AnnealTrace {
    std::vector<double> temperature, ess, accept, evidence, scale;
    std::vector<std::uint64_t> steps;
};

// stream ids of the sampler: (iteration << 16) | (worker << 2) | role, smc.cpp:21-28
enum { kPilotRole = 0, kMoveRole = 1, kTrialRole = 2, kCoordinatorRole = 3 };
static std::uint64_t anneal_stream(std::uint64_t iteration, std::uint64_t role) {
    return static_cast<std::uint32_t>((iteration << 16) | role);
}

struct Annealed {
    const Bioassay& model;
    std::uint64_t np, seed;
    std::vector<double> theta, lw, ll, lp;
    double temperature = 0.0, log_evidence = 0.0;

    // reweighted ESS at temperature increment dt: smc.cpp:226-239
    double ess_after(double dt) const {
        double top = -std::numeric_limits<double>::infinity();
        for (std::uint64_t i = 0; i < np; ++i) top = std::max(top, lw[i] + dt * ll[i]);
        if (top == -std::numeric_limits<double>::infinity()) return 0.0;
        double s1 = 0.0, s2 = 0.0;
        for (std::uint64_t i = 0; i < np; ++i) {
            const double e = std::exp(lw[i] + dt * ll[i] - top);
            s1 += e;
            s2 += e * e;
        }
        return s1 * s1 / s2;
    }
    // find_temperature: smc.cpp:221-253
    double next_temperature(double tol) const {
        const double target = static_cast<double>(np) / 2.0;
        const double room = 1.0 - temperature;
        if (ess_after(room) >= target) return 1.0;
        double lo = 0.0, hi = room;
        while (hi - lo > tol) {
            const double mid = 0.5 * (lo + hi);
            (ess_after(mid) >= target ? lo : hi) = mid;
        }
        return temperature + 0.5 * (lo + hi);
    }
    // one tempered random-walk sweep of `steps` steps: move_range, smc.cpp:77-150
    // `base`: stream position the sweep starts at (even); `scales`: per-particle
    // proposal scales, assigned cyclically (ESJD trial); `jumps`: h^2 |z|^2 of the
    // accepted proposals is added per particle (smc.cpp:138-144)
    std::uint64_t sweep(const double* chol, double h_all, std::uint64_t role, std::uint64_t iteration,
                        std::uint64_t steps, std::uint64_t base = 0, const double* scales = nullptr,
                        std::uint64_t n_scales = 0, double* jumps = nullptr) {
        const std::uint64_t gauss_total = np * steps * 2;
        std::uint64_t accepted = 0;
        Stream s(seed, anneal_stream(iteration, role));
        for (std::uint64_t q = 0; q < np; ++q)
            for (std::uint64_t r = 0; r < steps; ++r) {
                const double h = n_scales ? scales[q % n_scales] : h_all;
                s.pos = base + (q * steps + r) * 2;
                const double z0 = s.next_gaussian(0.0, 1.0), z1 = s.next_gaussian(0.0, 1.0);
                double inc0 = 0.0, inc1 = 0.0;
                inc0 += chol[0] * z0;
                inc1 += chol[2] * z0;
                inc1 += chol[3] * z1;
                const double p0 = theta[2 * q] + h * inc0, p1 = theta[2 * q + 1] + h * inc1;
                const double lp_new = model.log_prior(p0, p1);
                const double ll_new = model.log_lik(p0, p1);
                const double log_alpha = temperature * (ll_new - ll[q]) + lp_new - lp[q];
                s.pos = base + gauss_total + q * steps + r;
                const double u = s.next_unit();
                const double log_u = u > 0.0 ? ln_pos(u) : -std::numeric_limits<double>::infinity();
                if (!std::isnan(log_alpha) && log_alpha > -std::numeric_limits<double>::infinity() &&
                    log_u <= log_alpha) {
                    ++accepted;
                    theta[2 * q] = p0;
                    theta[2 * q + 1] = p1;
                    ll[q] = ll_new;
                    lp[q] = lp_new;
                    if (jumps) {
                        double zz = 0.0;
                        zz += z0 * z0;
                        zz += z1 * z1;
                        jumps[q] += h * h * zz;
                    }
                }
            }
        return accepted;
    }
};

// type-7 median of a sample (numeric.cpp:20-36,53)
static double median_of(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const std::size_t n = v.size();
    if (n == 1) return v[0];
    const double h = static_cast<double>(n - 1) * 0.5;
    const std::size_t lo = static_cast<std::size_t>(h);
    if (lo + 1 >= n) return v[n - 1];
    const double frac = h - static_cast<double>(lo);
    return v[lo] + frac * (v[lo + 1] - v[lo]);
}

static void anneal_run(const Bioassay& model, std::uint64_t np, std::uint64_t block_width, double c,
                       double scale, std::uint64_t seed, double* log_evidence,
                       std::uint64_t* iterations, AnnealTrace* trace, double* ensemble = nullptr,
                       const double* esjd_scales = nullptr, std::uint64_t n_scales = 0) {
    const double tol = 1e-10, jitter = 1e-10;            // SmcConfig defaults, smc.hpp:120-121
    const std::uint64_t max_iterations = 1000, step_cap = 100;
    require(supported_width(block_width), "invalid-shape", "unsupported block width");
    require(np >= 2 * block_width, "invalid-shape", "need at least two particle blocks");
    require(c > 0.0 && c < 1.0, "invalid-argument", "tuning constant must lie in (0, 1)");
    Annealed a{model, np, seed, std::vector<double>(2 * np), std::vector<double>(np),
               std::vector<double>(np), std::vector<double>(np)};
    {   // initial ensemble: prior draws in particle order, smc.cpp:386-393
        Stream s(seed, anneal_stream(0, kPilotRole));
        bool any = false;
        for (std::uint64_t i = 0; i < np; ++i) {
            s.align_even();
            const double z0 = s.next_gaussian(0.0, 1.0), z1 = s.next_gaussian(0.0, 1.0);
            a.theta[2 * i] = model.l1 * z0;
            a.theta[2 * i + 1] = model.l2 * z1;
            a.lw[i] = -std::log(static_cast<double>(np));
            a.ll[i] = model.log_lik(a.theta[2 * i], a.theta[2 * i + 1]);
            a.lp[i] = model.log_prior(a.theta[2 * i], a.theta[2 * i + 1]);
            require(!std::isnan(a.ll[i]) && a.ll[i] < std::numeric_limits<double>::infinity(),
                    "invalid-model", "log-likelihood is not finite at initialization");
            any = any || a.ll[i] > -std::numeric_limits<double>::infinity();
        }
        require(any, "invalid-model", "likelihood is zero for every initial particle");
    }
    const double h = scale > 0.0 ? scale : 2.38 / std::sqrt(2.0);
    std::uint64_t n = 0;
    while (a.temperature < 1.0) {
        ++n;
        require(n <= max_iterations, "non-convergence",
                "temperature failed to reach 1 within the iteration cap");
        const double t_next = a.next_temperature(tol);
        {   // reweight_and_update_evidence: smc.cpp:255-266
            const double before = logsumexp(a.lw.data(), np);
            const double dt = t_next - a.temperature;
            for (std::uint64_t i = 0; i < np; ++i) a.lw[i] += dt * a.ll[i];
            a.log_evidence += logsumexp(a.lw.data(), np) - before;
            a.temperature = t_next;
        }
        double ess_now = 0.0;
        require(vxo_ess(a.lw.data(), np, &ess_now) == 0, "degenerate-ensemble", "all weights are zero");
        {   // resample_multinomial: smc.cpp:268-300, coordinator stream
            std::vector<double> packed(4 * np), out(4 * np);
            for (std::uint64_t i = 0; i < np; ++i) {
                packed[4 * i] = a.theta[2 * i];
                packed[4 * i + 1] = a.theta[2 * i + 1];
                packed[4 * i + 2] = a.ll[i];
                packed[4 * i + 3] = a.lp[i];
            }
            require(vxo_resample_multinomial(np, 4, a.lw.data(), packed.data(), seed,
                                             anneal_stream(n, kCoordinatorRole), out.data(),
                                             nullptr) == 0,
                    "degenerate-ensemble", "weight sum is not finite");
            for (std::uint64_t i = 0; i < np; ++i) {
                a.theta[2 * i] = out[4 * i];
                a.theta[2 * i + 1] = out[4 * i + 1];
                a.ll[i] = out[4 * i + 2];
                a.lp[i] = out[4 * i + 3];
                a.lw[i] = -std::log(static_cast<double>(np));
            }
        }
        double chol[4];
        {   // make_kernel: smc.cpp:311-325
            double cov[4];
            sample_covariance(a.theta.data(), np, 2, cov);
            require(vxo_make_kernel(cov, 2, 1.0, jitter, chol) == 0, "degenerate-ensemble",
                    "covariance is rank deficient beyond jitter");
        }
        double p_acc, h_used;
        std::uint64_t steps;
        if (!n_scales) {
            const std::uint64_t pilot = a.sweep(chol, h, kPilotRole, n, 1);
            p_acc = static_cast<double>(pilot) / static_cast<double>(np);
            // steps_from_acceptance: smc.cpp:302-309
            const double p = std::min(std::max(p_acc, 0.01), 0.99);
            const double raw = std::ceil(std::log(c) / std::log(1.0 - p));
            steps = !(raw >= 1.0) ? 1 : std::min<std::uint64_t>(static_cast<std::uint64_t>(raw), step_cap);
            a.sweep(chol, h, kMoveRole, n, steps);
            h_used = h;
        } else {
            // esjd_core: smc.cpp:156-204 (streams: trial role for the trial step, move role,
            // continued from sweep to sweep, for the moves)
            std::vector<double> jumps(np, 0.0);
            const std::uint64_t trial = a.sweep(chol, 0.0, kTrialRole, n, 1, 0, esjd_scales, n_scales, jumps.data());
            p_acc = static_cast<double>(trial) / static_cast<double>(np);
            const double trial_median = median_of(jumps);
            double best = -1.0;
            bool any_jump = false;
            h_used = 0.0;
            for (std::uint64_t sidx = 0; sidx < n_scales; ++sidx) {
                std::vector<double> part;
                for (std::uint64_t i = sidx; i < np; i += n_scales) part.push_back(jumps[i]);
                if (part.empty()) continue;
                const double med = median_of(part);
                if (med > 0.0) any_jump = true;
                if (med > best) {
                    best = med;
                    h_used = esjd_scales[sidx];
                }
            }
            if (!any_jump)
                for (double j : jumps) any_jump = any_jump || j > 0.0;
            if (!any_jump) h_used = 2.38 / std::sqrt(2.0);
            steps = 0;
            std::uint64_t pos = 0;  // position of the move stream
            while (steps < step_cap) {
                std::uint64_t moved = 0;
                for (double cj : jumps) moved += cj > trial_median ? 1 : 0;
                if (2 * moved >= np) break;
                pos += pos & 1;  // align_even
                a.sweep(chol, h_used, kMoveRole, n, 1, pos, nullptr, 0, jumps.data());
                pos += 3 * np;
                ++steps;
            }
        }
        if (trace) {
            trace->temperature.push_back(a.temperature);
            trace->ess.push_back(ess_now);
            trace->accept.push_back(p_acc);
            trace->steps.push_back(steps);
            trace->evidence.push_back(a.log_evidence);
            trace->scale.push_back(h_used);
        }
    }
    *log_evidence = a.log_evidence;
    *iterations = n;
    for (std::uint64_t i = 0; ensemble && i < np; ++i) {  // SmcResult::ensemble, smc.cpp:478-487
        ensemble[i] = a.theta[2 * i];
        ensemble[np + i] = a.theta[2 * i + 1];
        ensemble[2 * np + i] = a.lw[i];
        ensemble[3 * np + i] = a.ll[i];
        ensemble[4 * np + i] = a.lp[i];
    }
}

int vxo_bioassay_ll(const double* beta, std::uint64_t lanes, const double* dose,
                    const std::uint32_t* group_size, const std::uint32_t* deaths,
                    std::uint32_t groups, double* out) {
    return guarded([&] {
        const Bioassay m = make_bioassay(dose, group_size, deaths, groups, 1.0, 1.0);
        for (std::uint64_t l = 0; l < lanes; ++l) out[l] = m.log_lik(beta[2 * l], beta[2 * l + 1]);
    });
}
int vxo_bioassay_sample(double lambda1, double lambda2, const double* dose,
                        const std::uint32_t* group_size, std::uint32_t groups, std::uint64_t seed,
                        double* theta, std::uint32_t* deaths) {
    return guarded([&] { bioassay_draw(lambda1, lambda2, dose, group_size, groups, seed, theta, deaths); });
}
// trace (optional): rows of (iteration, temperature, ess, log_evidence=nan, steps, p_acc, h)
// are not produced here; trace_out receives iterations x 4 doubles
// (temperature, ess, steps, p_acc), at most trace_cap rows.
// One run with its final ensemble (5 x particles: theta0, theta1, log weights, log
// likelihoods, log priors) and a 5-column trace (… , log evidence so far).
int vxo_smc_bioassay_ensemble(const double* dose, const std::uint32_t* group_size,
                              const std::uint32_t* deaths, std::uint32_t groups, double lambda1,
                              double lambda2, std::uint64_t particles, std::uint64_t block_width,
                              double c, double scale, std::uint64_t seed, double* log_evidence,
                              std::uint64_t* iterations, double* ensemble, double* trace_out,
                              std::uint64_t trace_cap, const double* esjd_scales,
                              std::uint64_t n_scales) {
    return guarded([&] {
        const Bioassay m = make_bioassay(dose, group_size, deaths, groups, lambda1, lambda2);
        AnnealTrace tr;
        anneal_run(m, particles, block_width, c, scale, seed, log_evidence, iterations, &tr, ensemble,
                   esjd_scales, n_scales);
        for (std::uint64_t i = 0; trace_out && i < tr.steps.size() && i < trace_cap; ++i) {
            trace_out[6 * i] = tr.temperature[i];
            trace_out[6 * i + 1] = tr.ess[i];
            trace_out[6 * i + 2] = static_cast<double>(tr.steps[i]);
            trace_out[6 * i + 3] = tr.accept[i];
            trace_out[6 * i + 4] = tr.evidence[i];
            trace_out[6 * i + 5] = tr.scale[i];
        }
    });
}

int vxo_smc_bioassay(const double* dose, const std::uint32_t* group_size,
                     const std::uint32_t* deaths, std::uint32_t groups, double lambda1,
                     double lambda2, std::uint64_t particles, std::uint64_t block_width, double c,
                     double scale, std::uint64_t seed, double* log_evidence,
                     std::uint64_t* iterations, double* trace_out, std::uint64_t trace_cap) {
    return guarded([&] {
        const Bioassay m = make_bioassay(dose, group_size, deaths, groups, lambda1, lambda2);
        AnnealTrace tr;
        anneal_run(m, particles, block_width, c, scale, seed, log_evidence, iterations,
                   trace_out ? &tr : nullptr);
        for (std::uint64_t i = 0; trace_out && i < tr.steps.size() && i < trace_cap; ++i) {
            trace_out[4 * i] = tr.temperature[i];
            trace_out[4 * i + 1] = tr.ess[i];
            trace_out[4 * i + 2] = static_cast<double>(tr.steps[i]);
            trace_out[4 * i + 3] = tr.accept[i];
        }
    });
}

// run_weak_info_test: weak_info.cpp:163-277 (default design, shared or redrawn
// base datasets); `threads` spreads the hyperparameter rows.
int vxo_weak_info_test(std::uint64_t hyper_count, std::uint64_t datasets, std::uint64_t particles,
                       double alpha, double c, double scale, std::uint64_t threads,
                       std::uint64_t block_width, std::uint64_t seed, int redraw_base,
                       double* lambda, double* gamma, std::uint8_t* weakly,
                       std::uint64_t* completed, const char* /*csv_path*/) {
    return guarded([&] {
        require(datasets >= 1, "invalid-argument", "need at least one dataset per prior");
        require(threads >= 1, "invalid-argument", "need at least one worker");
        const double dose[4] = {-0.86, -0.3, -0.05, -0.75};  // default_design, weak_info.cpp:62-64
        const std::uint32_t size[4] = {5, 5, 5, 5};
        const double base[2] = {10.0, 2.5};                  // kBasePrior, weak_info.hpp:21
        const std::uint64_t rows = hyper_count + 1;
        lambda[0] = base[0];
        lambda[1] = base[1];
        {
            const std::uint64_t path[1] = {1};
            Stream s(derive_seed(seed, path, 1), 0);
            for (std::uint64_t k = 1; k < rows; ++k) {
                lambda[2 * k] = s.next_uniform(0.1, 10.0);
                lambda[2 * k + 1] = s.next_uniform(0.1, 20.0);
            }
        }
        std::vector<std::uint32_t> shared(4 * datasets);
        if (!redraw_base)
            for (std::uint64_t i = 0; i < datasets; ++i) {
                const std::uint64_t path[2] = {2, i};
                double theta[2];
                bioassay_draw(base[0], base[1], dose, size, 4, derive_seed(seed, path, 2), theta,
                              &shared[4 * i]);
            }
        const auto evidence = [&](const std::uint32_t* deaths, const double* prior,
                                  std::uint64_t run_seed, double* out) {
            std::uint64_t it = 0;
            const int rc = guarded([&] {
                const Bioassay m = make_bioassay(dose, size, deaths, 4, prior[0], prior[1]);
                anneal_run(m, particles, block_width, c, scale, run_seed, out, &it, nullptr);
            });
            return rc == 0;
        };
        parallel_for(rows, static_cast<unsigned>(threads), [&](std::uint64_t k) {
            const double* prior = lambda + 2 * k;
            std::vector<double> ev_base, ev_hyper;
            std::uint64_t both = 0;
            for (std::uint64_t i = 0; i < datasets; ++i) {
                std::uint32_t base_y[4], hyper_y[4];
                double theta[2];
                if (redraw_base) {
                    const std::uint64_t path[3] = {5, k, i};
                    bioassay_draw(base[0], base[1], dose, size, 4, derive_seed(seed, path, 3), theta, base_y);
                } else {
                    std::copy_n(&shared[4 * i], 4, base_y);
                }
                const std::uint64_t hp[3] = {3, k, i};
                bioassay_draw(prior[0], prior[1], dose, size, 4, derive_seed(seed, hp, 3), theta, hyper_y);
                const std::uint64_t sb[4] = {4, k, 0, i}, sh[4] = {4, k, 1, i};
                double eb = 0.0, eh = 0.0;
                const bool ok_b = evidence(base_y, prior, derive_seed(seed, sb, 4), &eb);
                const bool ok_h = evidence(hyper_y, prior, derive_seed(seed, sh, 4), &eh);
                if (ok_b) ev_base.push_back(eb);
                if (ok_h) ev_hyper.push_back(eh);
                both += (ok_b && ok_h) ? 1 : 0;
            }
            completed[k] = both;
            gamma[k] = std::numeric_limits<double>::quiet_NaN();
            if (ev_base.empty() || ev_hyper.empty()) return;
            std::vector<double> pv(ev_base.size());
            vxo_estimate_pvalues(ev_base.data(), ev_base.size(), ev_hyper.data(), ev_hyper.size(),
                                 pv.data());
            vxo_compute_cutoff(pv.data(), pv.size(), alpha, &gamma[k]);
        });
        for (std::uint64_t k = 0; k < rows; ++k) weakly[k] = (k != 0 && gamma[k] > gamma[0]) ? 1 : 0;
    });
}

// ----------------------------------------- TB Gillespie ABC
// Restates tb::gillespie_simulate (tb_model.cpp:39-127), tb_summaries (:129-138),
// sample_prior (:151-156) and the row sequence of abc.cpp:51-60.  The state keeps
// the genotype counts in slot order; the lookup is "first slot whose running
// count exceeds the target" (upper_bound over the cumulative array,
// tb_model.cpp:31-34) -- the reference's cumulative array and its compaction
// (:108-118) are bookkeeping that never changes which slot that is.
struct TbPath {
    std::vector<std::uint32_t> slots;
    double time = 0.0, total = 0.0;
    std::uint64_t genotypes = 0;
};
static TbPath tb_path(const double* theta, std::uint64_t initial, double horizon, double target,
                      Stream& s) {
    require(initial >= 1, "invalid-shape", "need at least one initial case");
    require(theta[0] >= 0 && theta[1] >= 0 && theta[2] >= 0, "invalid-argument",
            "rates must be nonnegative");
    TbPath p;
    p.slots.assign(1, static_cast<std::uint32_t>(initial));
    p.total = static_cast<double>(initial);
    p.genotypes = 1;
    while (p.time < horizon && p.total < target && p.total > 0) {
        const double birth = theta[0] * p.total, death = theta[1] * p.total, mut = theta[2] * p.total;
        const double rate = birth + death + mut;
        if (rate <= 0.0) {
            p.time = horizon;
            break;
        }
        const double wait = -ln_pos(1.0 - s.next_unit()) / rate;
        if (p.time + wait > horizon) {
            p.time = horizon;
            break;
        }
        p.time += wait;
        const double kind = s.next_unit() * rate;
        const double pick = s.next_unit() * p.total;
        std::size_t idx = 0;
        double run = 0.0;
        for (; idx < p.slots.size(); ++idx) {
            run += p.slots[idx];
            if (run > pick) break;
        }
        require(idx < p.slots.size(), "internal", "genotype lookup ran past the population");
        const auto take_one = [&] {
            if (--p.slots[idx] == 0) --p.genotypes;
        };
        if (kind < birth) {
            ++p.slots[idx];
            p.total += 1.0;
        } else if (kind < birth + death) {
            take_one();
            p.total -= 1.0;
        } else {
            take_one();
            p.slots.push_back(1);
            ++p.genotypes;
        }
    }
    return p;
}
// (G, H) with H = 1 - sum (X_i / N)^2 evaluated as 1 - ss / (n n); false when extinct
static bool tb_summaries(const TbPath& p, double* out) {
    if (!(p.total >= 1.0)) return false;
    double ss = 0.0;
    for (std::uint32_t c : p.slots) ss += static_cast<double>(c) * static_cast<double>(c);
    out[0] = static_cast<double>(p.genotypes);
    out[1] = 1.0 - ss / (p.total * p.total);
    return true;
}

int vxo_tb_simulate(const double* theta, std::uint64_t initial, double horizon, double target,
                    std::uint64_t seed, std::uint64_t id, std::uint64_t pos,
                    std::uint64_t /*block_width*/, double* out, std::uint64_t* pos_after,
                    double* counts_out, std::uint64_t counts_cap, std::uint64_t* n_counts) {
    return guarded([&] {
        Stream s(seed, id);
        s.pos = pos;
        const TbPath p = tb_path(theta, initial, horizon, target, s);
        out[0] = p.time;
        out[1] = p.total;
        out[2] = static_cast<double>(p.genotypes);
        out[3] = out[4] = std::numeric_limits<double>::quiet_NaN();
        tb_summaries(p, out + 3);
        if (pos_after) *pos_after = s.pos;
        std::uint64_t k = 0;
        for (std::uint32_t c : p.slots)
            if (c) {
                if (counts_out && k < counts_cap) counts_out[k] = c;
                ++k;
            }
        if (n_counts) *n_counts = k;
    });
}

int vxo_tb_abc_particle(std::uint64_t initial, double horizon, double target, std::uint64_t first,
                        std::uint64_t count, std::uint64_t seed, const double* observed,
                        double* params, double* summaries, double* rho, std::uint8_t* failed,
                        unsigned threads) {
    return guarded([&] {
        require(initial >= 1, "invalid-shape", "need at least one initial case");
        parallel_for(count, threads, [&](std::uint64_t r) {
            Stream s(seed, first + r);
            double theta[3];  // sample_prior: tb_model.cpp:151-156
            theta[0] = s.next_uniform(0.0, 2.0);
            theta[1] = s.next_uniform(0.0, theta[0]);
            theta[2] = s.next_uniform(0.0, 1.0);
            s.align_even();
            const TbPath p = tb_path(theta, initial, horizon, target, s);
            double sm[2] = {0.0, 0.0};
            const bool ok = tb_summaries(p, sm);
            if (params) std::copy(theta, theta + 3, params + r * 3);
            if (summaries) std::copy(sm, sm + 2, summaries + r * 2);
            if (rho) rho[r] = ok ? discrepancy<double>(sm, observed, 2)
                                 : std::numeric_limits<double>::quiet_NaN();
            if (failed) failed[r] = ok ? 0 : 1;
        });
    });
}

// bench::tb_observed_summaries (bench.cpp:79-92): theta = (0.2, 0.1, 0.05), stream
// RngStream(derive_seed(seed,{91}), 0) consumed across up to 64 attempts
int vxo_tb_observed(std::uint64_t initial, double horizon, double target, std::uint64_t seed,
                    std::uint64_t /*block_width*/, double* out) {
    return guarded([&] {
        const double theta[3] = {0.2, 0.1, 0.05};
        Stream s(derive_seed1(seed, 91), 0);
        for (int attempt = 0; attempt < 64; ++attempt) {
            const TbPath p = tb_path(theta, initial, horizon, target, s);
            if (tb_summaries(p, out)) return;
        }
        require(false, "empty-set", "synthetic tb population kept going extinct");
    });
}

}  // extern "C"
