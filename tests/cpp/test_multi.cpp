// Multi-GPU behind the C ABI and the C++ shim (include/vexbayes_cuda.h, section
// "multi-GPU"): the drivers shard rows over the devices in use and gather the
// accepted samples over the library's own NCCL communicator.
//
//  * every device count: abc::run_prior_predictive and the whole-job
//    reject_fixed_epsilon over all visible devices (dumped for the Python side to
//    compare with the oracle), a 1-rank NCCL communicator doing a real all-gather
//    and all-reduce, and the packed accepted-set round trip;
//  * two or more devices: the same calls restricted to device 0 must give the
//    identical bytes, and the SPMD form (one host thread per device, each with
//    its own vxb_ctx + vxb_comm created from a shared unique id) must agree too.
//    With one device this part prints "multi_gpu skipped".
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "vexbayes/abc.hpp"
#include "vexbayes/logistic.hpp"
#include "vexbayes/smc.hpp"

using namespace vexbayes;

static void dump(const char* name, const std::vector<double>& v) {
    std::printf("%s %zu", name, v.size());
    for (double x : v) {
        unsigned long long b;
        std::memcpy(&b, &x, 8);
        std::printf(" %016llx", b);
    }
    std::printf("\n");
}
static void dump_rows(const char* name, const std::vector<std::uint64_t>& v) {
    std::printf("%s %zu", name, v.size());
    for (auto x : v) std::printf(" %llu", static_cast<unsigned long long>(x));
    std::printf("\n");
}
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (!(cond)) {                                                         \
            std::printf("FAILED %s:%d %s\n", __FILE__, __LINE__, #cond);       \
            return 1;                                                          \
        }                                                                      \
    } while (0)

int main() {
    const int n_dev = cuda::device_count();
    std::printf("devices %d\n", n_dev);
    CHECK(n_dev >= 1);
    const ModelHooks model = logistic::make_abc_model();
    const auto observed = logistic::simulate_at(model, std::vector<double>{0.5, 100.0, 0.05},
                                                0x9b1d6f0c5a3e7c21ULL, 0, 0);
    dump("observed", observed);

    // ---- all visible devices through the shim
    std::printf("in_use %d\n", cuda::devices_in_use());
    const auto set = abc::run_prior_predictive(model, 1003, 3, 4, 1337, observed);
    dump("rho", set.discrepancies);
    dump("params", set.params);
    const auto sel = abc::select_epsilon(set, 0.05);
    const auto acc = abc::reject_fixed_epsilon(model, 30001, 1337, observed, sel.epsilon, 4000);
    std::printf("epsilon 1 %.17g\n", sel.epsilon);
    dump_rows("reject_rows", acc.rows);
    dump("reject_rho", acc.discrepancies);
    dump("reject_params", acc.params);
    std::printf("reject_total %llu\n", static_cast<unsigned long long>(acc.total_accepted));
    // a capped job reports the full count
    const auto capped = abc::reject_fixed_epsilon(model, 30001, 1337, observed, sel.epsilon, 5);
    CHECK(capped.total_accepted == acc.total_accepted && capped.rows.size() == 5);
    for (int k = 0; k < 5; ++k) CHECK(capped.rows[k] == acc.rows[k]);

    // ABC-SMC through the shim: every GPU in use, weight sum / particles over NCCL
    smc::AbcSmcConfig scfg;
    scfg.particles = 1500;
    scfg.generations = 3;
    scfg.round_size = 700;
    scfg.seed = 77;
    const auto pop = smc::run_abc_smc(model, scfg, observed);
    dump("smc_particles", pop.particles);
    dump("smc_weights", pop.weights);
    dump("smc_epsilon", pop.epsilon);

    // ---- the library's NCCL with one rank: a real communicator, real collectives
    {
        vxb_ctx* ctx = cuda::context();
        int version = 0;
        cuda::check(vxb_comm_version(&version));
        std::printf("nccl_version %d\n", version);
        unsigned char id[VXB_COMM_ID_BYTES];
        cuda::check(vxb_comm_unique_id(id));
        vxb_comm* comm = nullptr;
        cuda::check(vxb_comm_init_rank(ctx, id, 0, 1, &comm));
        CHECK(vxb_comm_rank(comm) == 0 && vxb_comm_size(comm) == 1);
        void *a = nullptr, *b = nullptr;
        cuda::check(vxb_device_alloc(ctx, 4096, &a));
        cuda::check(vxb_device_alloc(ctx, 4096, &b));
        std::vector<double> h(512), back(512);
        for (int i = 0; i < 512; ++i) h[i] = 0.5 * i;
        cuda::check(vxb_copy(ctx, a, h.data(), 4096));
        cuda::check(vxb_comm_allgather(comm, a, b, 4096));
        cuda::check(vxb_comm_allreduce(comm, b, 512, VXB_DT_F64, VXB_OP_SUM));
        cuda::check(vxb_copy(ctx, back.data(), b, 4096));
        CHECK(back == h);
        // packed accepted set through the SPMD entry point with that communicator
        vxb_accept_layout lay;
        cuda::check(vxb_accept_layout_of(VXB_F64, 3, 4000, &lay));
        void *local = nullptr, *all = nullptr;
        cuda::check(vxb_device_alloc(ctx, lay.stride, &local));
        cuda::check(vxb_device_alloc(ctx, lay.stride, &all));
        vxb_keying key{VXB_KEY_PARTICLE, 1, 1, 0, 1337};
        cuda::check(vxb_sharded_abc_reject(ctx, comm, model.device.get(), &key, 30001, observed.data(),
                                           sel.epsilon, &lay, local, all));
        std::vector<unsigned char> host(lay.stride);
        cuda::check(vxb_copy(ctx, host.data(), all, lay.stride));
        std::uint64_t n_acc = 0;
        std::vector<std::uint64_t> rows(4000);
        std::vector<double> rho(4000);
        int over = 1;
        cuda::check(vxb_accept_unpack(&lay, VXB_F64, 3, 1, host.data(), 4000, &n_acc, rows.data(),
                                      nullptr, rho.data(), &over, nullptr));
        CHECK(n_acc == acc.total_accepted && over == 0);
        for (std::uint64_t k = 0; k < n_acc; ++k)
            CHECK(rows[k] == acc.rows[k] && rho[k] == acc.discrepancies[k]);
        vxb_comm_destroy(comm);
        cuda::check(vxb_device_free(ctx, a));
        cuda::check(vxb_device_free(ctx, b));
        cuda::check(vxb_device_free(ctx, local));
        cuda::check(vxb_device_free(ctx, all));
        std::printf("nccl_one_rank ok\n");
    }

    // ---- three ranks on ONE device through the loopback group: the multi-rank code of
    // the C ABI (sharding, packed gather, rounds, weight gather, chunk-total reduction)
    // runs for real on a one-GPU box and must reproduce the results above
    {
        vxb_multi* loop = nullptr;
        cuda::check(vxb_multi_init_loopback(&loop, 0, 3));
        CHECK(vxb_multi_size(loop) == 3 && vxb_multi_comm(loop, 2) != nullptr);
        vxb_keying key{VXB_KEY_PARTICLE, 1, 1, 0, 1337};
        std::uint64_t n_acc = 0;
        std::vector<std::uint64_t> rows(4000);
        std::vector<double> rho(4000), params(3 * 4000);
        cuda::check(vxb_multi_abc_reject(loop, model.device.get(), &key, 30001, observed.data(), sel.epsilon,
                                         4000, &n_acc, rows.data(), params.data(), rho.data()));
        CHECK(n_acc == acc.total_accepted);
        rows.resize(n_acc);
        rho.resize(n_acc);
        params.resize(3 * n_acc);
        CHECK(rows == acc.rows && rho == acc.discrepancies && params == acc.params);
        std::vector<double> th(pop.particles.size()), w(pop.weights.size()), r(pop.weights.size());
        std::vector<double> eps(3), ess(3), rate(3), mean(9), cov(27);
        std::vector<std::uint64_t> props(3);
        vxb_abcsmc_cfg c{scfg.particles, 3, 0, scfg.quantile, scfg.kernel_scale, scfg.jitter,
                         scfg.round_size, scfg.max_rounds, scfg.seed};
        vxb_abcsmc_out o{th.data(), w.data(), r.data(), eps.data(), ess.data(), rate.data(), props.data(),
                         mean.data(), cov.data()};
        cuda::check(vxb_multi_abcsmc_run(loop, model.device.get(), &c, observed.data(), &o));
        CHECK(th == pop.particles && w == pop.weights && eps == pop.epsilon && props == pop.proposals);
        // select_epsilon over the sharded distances (all-reduced digit histograms)
        double eps3 = 0.0;
        std::vector<std::uint64_t> idx3(set.rows);
        cuda::check(vxb_multi_select_epsilon(loop, VXB_F64, set.discrepancies.data(), set.failed.data(), set.rows,
                                             0.05, &eps3, idx3.size(), &n_acc, idx3.data()));
        idx3.resize(n_acc);
        CHECK(eps3 == sel.epsilon && idx3.size() == sel.accepted.size());
        for (std::size_t i = 0; i < idx3.size(); ++i) CHECK(idx3[i] == sel.accepted[i]);
        vxb_multi_shutdown(loop);
        std::printf("loopback_three_ranks ok\n");
    }

    if (n_dev < 2) {
        std::printf("multi_gpu skipped (1 device)\n");
        return 0;
    }

    // ---- two or more devices: G devices == one device, bit for bit
    CHECK(cuda::devices_in_use() == n_dev);
    cuda::set_devices({0});
    CHECK(cuda::devices_in_use() == 1);
    const auto set1 = abc::run_prior_predictive(model, 1003, 3, 4, 1337, observed);
    const auto acc1 = abc::reject_fixed_epsilon(model, 30001, 1337, observed, sel.epsilon, 4000);
    CHECK(set1.discrepancies.size() == set.discrepancies.size());
    CHECK(std::memcmp(set1.discrepancies.data(), set.discrepancies.data(), 8 * set.discrepancies.size()) == 0);
    CHECK(std::memcmp(set1.params.data(), set.params.data(), 8 * set.params.size()) == 0);
    CHECK(std::memcmp(set1.summaries.data(), set.summaries.data(), 8 * set.summaries.size()) == 0);
    CHECK(set1.failed == set.failed);
    CHECK(acc1.total_accepted == acc.total_accepted && acc1.rows == acc.rows);
    CHECK(acc1.discrepancies == acc.discrepancies && acc1.params == acc.params);
    const auto pop1 = smc::run_abc_smc(model, scfg, observed);
    CHECK(pop1.particles == pop.particles && pop1.weights == pop.weights && pop1.epsilon == pop.epsilon);
    CHECK(pop1.proposals == pop.proposals && pop1.ess == pop.ess);

    // ---- SPMD: one host thread per device, own ctx + comm from a shared unique id
    unsigned char id[VXB_COMM_ID_BYTES];
    cuda::check(vxb_comm_unique_id(id));
    vxb_accept_layout lay;
    cuda::check(vxb_accept_layout_of(VXB_F64, 3, 4000, &lay));
    std::vector<std::vector<unsigned char>> gathered(n_dev, std::vector<unsigned char>(n_dev * lay.stride));
    std::vector<int> rc(n_dev, 0);
    std::vector<std::thread> pool;
    for (int r = 0; r < n_dev; ++r)
        pool.emplace_back([&, r] {
            vxb_ctx* ctx = nullptr;
            vxb_comm* comm = nullptr;
            void *local = nullptr, *all = nullptr;
            vxb_keying key{VXB_KEY_PARTICLE, 1, 1, 0, 1337};
            rc[r] = vxb_init(&ctx, r) || vxb_comm_init_rank(ctx, id, r, n_dev, &comm) ||
                    vxb_device_alloc(ctx, lay.stride, &local) ||
                    vxb_device_alloc(ctx, n_dev * lay.stride, &all) ||
                    vxb_sharded_abc_reject(ctx, comm, model.device.get(), &key, 30001, observed.data(),
                                           sel.epsilon, &lay, local, all) ||
                    vxb_copy(ctx, gathered[r].data(), all, n_dev * lay.stride);
            if (rc[r]) std::printf("rank %d: %s\n", r, vxb_last_error());
            vxb_comm_destroy(comm);
            if (ctx) {
                vxb_device_free(ctx, local);
                vxb_device_free(ctx, all);
            }
            vxb_shutdown(ctx);
        });
    for (auto& t : pool) t.join();
    for (int r = 0; r < n_dev; ++r) {
        CHECK(rc[r] == 0);
        CHECK(gathered[r] == gathered[0]);  // every rank holds the same gathered bytes
    }
    std::uint64_t n_acc = 0;
    std::vector<std::uint64_t> rows(4000);
    std::vector<double> rho(4000), params(3 * 4000);
    int over = 1;
    cuda::check(vxb_accept_unpack(&lay, VXB_F64, 3, n_dev, gathered[0].data(), 4000, &n_acc, rows.data(),
                                  params.data(), rho.data(), &over, nullptr));
    CHECK(n_acc == acc.total_accepted && over == 0);
    rows.resize(n_acc);
    rho.resize(n_acc);
    params.resize(3 * n_acc);
    CHECK(rows == acc.rows && rho == acc.discrepancies && params == acc.params);
    std::printf("multi_gpu ok %d devices\n", n_dev);
    return 0;
}
