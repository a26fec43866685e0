// vexbayes/bench.hpp (B200 shim) -- the reference's benchmark harness interface
// (bench.hpp:11-103, bench.cpp) over the device-backed experiments.
//
// What stays: the record / summary types, the CSV layout byte for byte
// (records section, summary section, "%.6g" times; bench.cpp:22-31,215-230),
// parse_csv, amdahl_bound, the timing protocol (one discarded warm-up per cell,
// steady_clock around the body only, failures become NaN + flag;
// bench.cpp:140-172).  `threads` and `block_width` keep their meaning as the
// (P, V) of the reference keying, so a cell simulates the very samples the CPU
// run of that cell simulates.
// What changes: the body runs on the GPU; only the experiments with a device
// path can run (toggle-abc, weakinfo, tb) -- bege raises unsupported-model.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <istream>
#include <limits>
#include <map>
#include <ostream>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "abc.hpp"
#include "tb_model.hpp"
#include "toggle_switch.hpp"
#include "weak_info.hpp"

namespace vexbayes::bench {

enum class Experiment { toggle_abc, weakinfo, bege, tb };
enum class Mode { scalar, blocked };

namespace detail {
inline constexpr const char* kExperimentNames[] = {"toggle-abc", "weakinfo", "bege", "tb"};
inline constexpr const char* kModeNames[] = {"scalar", "blocked"};
inline constexpr const char* kRecordColumns =
    "experiment,mode,threads,block_width,replicate,runtime_seconds,failed";
inline constexpr const char* kSummaryColumns =
    "experiment,mode,threads,block_width,mean_runtime,speedup_vs_baseline";
inline std::string six_digits(double seconds) {
    char text[48];
    std::snprintf(text, sizeof(text), "%.6g", seconds);
    return text;
}
}  // namespace detail

inline std::string to_string(Experiment e) {
    const auto k = static_cast<std::size_t>(e);
    require(k < 4, "invalid-input", "unknown experiment enum value");
    return detail::kExperimentNames[k];
}
inline std::string to_string(Mode m) { return detail::kModeNames[m == Mode::scalar ? 0 : 1]; }
inline Experiment experiment_from_string(const std::string& name) {
    for (std::size_t k = 0; k < 4; ++k)
        if (name == detail::kExperimentNames[k]) return static_cast<Experiment>(k);
    raise("invalid-input", "unknown experiment: " + name);
}
inline Mode mode_from_string(const std::string& name) {
    if (name == detail::kModeNames[0]) return Mode::scalar;
    if (name == detail::kModeNames[1]) return Mode::blocked;
    raise("invalid-input", "unknown mode: " + name);
}

struct BenchmarkRecord {
    Experiment experiment;
    Mode mode;
    std::size_t threads;
    std::size_t block_width;
    std::size_t replicate;
    double runtime_seconds;
    bool failed;
};

struct ExperimentSizes {
    std::size_t samples = 64;  // prior predictive draws
    std::size_t cells = 256;   // toggle C
    std::size_t steps = 100;   // toggle T
    std::size_t particles = 200;  // SMC N_p
    std::size_t hypers = 2;       // weak-info K
    std::size_t datasets = 8;     // weak-info N
    std::size_t tb_initial = 10;
    double tb_horizon = 10.0;
    double tb_target = 10000.0;
};

struct BenchConfig {
    Experiment experiment = Experiment::toggle_abc;
    std::vector<std::size_t> threads = {1, 2, 4, 8, 16};
    std::vector<std::size_t> block_widths = {1, 4, 8};
    std::size_t replicates = 4;
    std::uint64_t seed = 1337;
    ExperimentSizes sizes;
    bool warmup = true;
};

struct SummaryRow {
    Experiment experiment;
    Mode mode;
    std::size_t threads;
    std::size_t block_width;
    double mean_runtime;
    double speedup_vs_baseline;
};

inline double amdahl_bound(double serial_seconds, double parallel_seconds, double units) {
    require(serial_seconds >= 0.0 && parallel_seconds >= 0.0, "invalid-input",
            "runtimes must be nonnegative");
    require(serial_seconds + parallel_seconds > 0.0, "invalid-input",
            "total runtime must be positive");
    require(units >= 1.0, "invalid-input", "need at least one processing unit");
    const double total = serial_seconds + parallel_seconds;
    return total / (serial_seconds + parallel_seconds / units);
}

// bench.cpp:69-77: one simulation at the prior midpoints from
// RngStream(derive_seed(seed,{90}), 0).  A single simulation from position 0 does
// not depend on the block width (cell c owns positions [c*2T, (c+1)*2T)).
inline std::vector<double> toggle_observed_summaries(std::size_t steps, std::size_t cells,
                                                     std::uint64_t seed, std::size_t) {
    const toggle::ToggleParams midpoint{325.0, 0.275, 0.2, 25.0, 25.0, 3.5, 3.5};
    const std::uint64_t path[1] = {90};
    return toggle::simulate_summaries(toggle::make_abc_model(steps, cells), midpoint,
                                      vxb_derive_seed(seed, path, 1), 0, 0);
}

// bench.cpp:79-92: theta = (0.2, 0.1, 0.05) from RngStream(derive_seed(seed,{91}), 0),
// retried (up to 64 paths off the same stream) while the population dies out.
inline std::vector<double> tb_observed_summaries(std::size_t initial_cases, tb::StopRule stop,
                                                 std::uint64_t seed, std::size_t) {
    const std::uint64_t path[1] = {91};
    const tb::TbSummaries s = tb::simulate_summaries({0.2, 0.1, 0.05}, initial_cases, stop,
                                                     vxb_derive_seed(seed, path, 1), 0, 0, 64);
    return {s.genotypes, s.diversity};
}

inline void run_experiment_once(Experiment experiment, const ExperimentSizes& sizes,
                                std::size_t threads, std::size_t block_width, std::uint64_t seed) {
    if (experiment == Experiment::weakinfo) {  // bench.cpp:113-123
        weakinfo::WeakInfoConfig config;
        config.hyper_count = sizes.hypers;
        config.datasets = sizes.datasets;
        config.particles = sizes.particles;
        config.workers = threads;
        config.block_width = block_width;
        config.seed = seed;
        weakinfo::run_weak_info_test(config);
        return;
    }
    if (experiment == Experiment::tb) {  // bench.cpp:104-111
        const tb::StopRule stop{sizes.tb_horizon, sizes.tb_target};
        const auto observed = tb_observed_summaries(sizes.tb_initial, stop, seed, block_width);
        abc::run_prior_predictive(tb::make_abc_model(sizes.tb_initial, stop), sizes.samples, threads,
                                  block_width, seed, observed);
        return;
    }
    require(experiment == Experiment::toggle_abc, "unsupported-model",
            "experiment " + to_string(experiment) + " has no device path");
    const auto observed = toggle_observed_summaries(sizes.steps, sizes.cells, seed, block_width);
    const auto model = toggle::make_abc_model(sizes.steps, sizes.cells);
    abc::run_prior_predictive(model, sizes.samples, threads, block_width, seed, observed);
}

inline std::vector<BenchmarkRecord> run_benchmark(const BenchConfig& config) {
    require(config.replicates >= 1, "invalid-input", "need at least one replicate");
    require(!config.threads.empty() && !config.block_widths.empty(), "invalid-input",
            "thread and block-width lists must not be empty");
    using clock = std::chrono::steady_clock;
    std::vector<BenchmarkRecord> records;
    for (const std::size_t width : config.block_widths)
        for (const std::size_t workers : config.threads) {
            const auto body = [&] {
                run_experiment_once(config.experiment, config.sizes, workers, width, config.seed);
            };
            if (config.warmup) {
                try {
                    body();
                } catch (const std::exception&) {
                }
            }
            for (std::size_t rep = 0; rep < config.replicates; ++rep) {
                BenchmarkRecord rec{config.experiment, width == 1 ? Mode::scalar : Mode::blocked,
                                    workers, width, rep,
                                    std::numeric_limits<double>::quiet_NaN(), true};
                try {
                    const auto t0 = clock::now();
                    body();
                    rec.runtime_seconds = std::chrono::duration<double>(clock::now() - t0).count();
                    rec.failed = false;
                } catch (const std::exception&) {
                }
                records.push_back(rec);
            }
        }
    return records;
}

// Per-cell means over the non-failed replicates, in order of first appearance,
// and the speed-up against the first (scalar, threads = 1) cell.
inline std::vector<SummaryRow> summarize(const std::vector<BenchmarkRecord>& records) {
    using Cell = std::tuple<int, int, std::size_t, std::size_t>;
    std::map<Cell, std::size_t> slot;
    std::vector<SummaryRow> rows;
    std::vector<std::size_t> good;
    for (const BenchmarkRecord& r : records) {
        const Cell cell{static_cast<int>(r.experiment), static_cast<int>(r.mode), r.threads,
                        r.block_width};
        auto [it, fresh] = slot.try_emplace(cell, rows.size());
        if (fresh) {
            rows.push_back({r.experiment, r.mode, r.threads, r.block_width, 0.0, 0.0});
            good.push_back(0);
        }
        if (!r.failed) {
            rows[it->second].mean_runtime += r.runtime_seconds;
            ++good[it->second];
        }
    }
    double baseline = std::numeric_limits<double>::quiet_NaN();
    for (std::size_t k = 0; k < rows.size(); ++k)
        rows[k].mean_runtime = good[k] ? rows[k].mean_runtime / static_cast<double>(good[k])
                                       : std::numeric_limits<double>::quiet_NaN();
    for (const SummaryRow& row : rows)
        if (row.mode == Mode::scalar && row.threads == 1) {
            baseline = row.mean_runtime;
            break;
        }
    for (SummaryRow& row : rows) row.speedup_vs_baseline = baseline / row.mean_runtime;
    return rows;
}

inline void write_csv(const std::vector<BenchmarkRecord>& records, std::ostream& out) {
    out << detail::kRecordColumns << '\n';
    for (const BenchmarkRecord& r : records)
        out << to_string(r.experiment) << ',' << to_string(r.mode) << ',' << r.threads << ','
            << r.block_width << ',' << r.replicate << ',' << detail::six_digits(r.runtime_seconds)
            << ',' << (r.failed ? 1 : 0) << '\n';
    out << detail::kSummaryColumns << '\n';
    for (const SummaryRow& s : summarize(records))
        out << to_string(s.experiment) << ',' << to_string(s.mode) << ',' << s.threads << ','
            << s.block_width << ',' << detail::six_digits(s.mean_runtime) << ','
            << detail::six_digits(s.speedup_vs_baseline) << '\n';
}
inline void write_csv(const std::vector<BenchmarkRecord>& records, const std::string& path) {
    std::ofstream out(path);
    require(out.good(), "io-error", "cannot open " + path + " for writing");
    write_csv(records, out);
    require(out.good(), "io-error", "write to " + path + " failed");
}

// The records section written by write_csv (stops at the summary header).
inline std::vector<BenchmarkRecord> parse_csv(std::istream& in) {
    const auto chomp = [](std::string& s) {
        if (!s.empty() && s.back() == '\r') s.pop_back();
    };
    std::string line;
    require(static_cast<bool>(std::getline(in, line)), "io-error", "empty benchmark file");
    chomp(line);
    require(line == detail::kRecordColumns, "io-error", "unexpected benchmark header: " + line);
    std::vector<BenchmarkRecord> records;
    while (std::getline(in, line)) {
        chomp(line);
        if (line.empty()) continue;
        if (line == detail::kSummaryColumns) break;
        std::vector<std::string> cells;
        std::istringstream row(line);
        for (std::string cell; std::getline(row, cell, ',');) cells.push_back(cell);
        require(cells.size() >= 7, "io-error", "malformed benchmark row: " + line);
        records.push_back({experiment_from_string(cells[0]), mode_from_string(cells[1]),
                           std::stoull(cells[2]), std::stoull(cells[3]), std::stoull(cells[4]),
                           std::stod(cells[5]), std::stoi(cells[6]) != 0});
    }
    return records;
}

}  // namespace vexbayes::bench
