// vxb_internal.cuh -- functions shared between the C-ABI translation units.
#pragma once

#include "vxb_common.cuh"
#include "vxb_logistic.cuh"

namespace vxb {

// vxb_logistic.cu
LogisticModel make_logistic(const vxb_model& m);

// vxb_toggle.cu
void toggle_launch(vxb_ctx* ctx, const vxb_model& m, const Keying& key, uint64_t first,
                   uint64_t count, uint64_t block_width, const double* observed_host,
                   const double* theta_dev, double* params, double* summaries, double* rho,
                   uint8_t* failed);

// vxb_tb.cu
void tb_launch(vxb_ctx* ctx, const vxb_model& m, uint64_t seed, uint64_t first, uint64_t count,
               const double* observed_host, double* params, double* summaries, double* rho,
               uint8_t* failed);
void tb_simulate_fixed(vxb_ctx* ctx, const vxb_model& m, const double* theta_dev, uint64_t key,
                       uint64_t pos, uint32_t attempts, double* summary_dev, uint8_t* failed_dev,
                       double* detail_dev);

// vxb_select.cu
void compact_accepted_device(vxb_ctx* ctx, int precision, const void* rho_dev,
                             const uint8_t* failed_dev, uint64_t n, double epsilon,
                             uint64_t index_base, uint64_t cap, uint64_t* n_accepted_host,
                             uint64_t* idx_dev);
void order_statistics_any(vxb_ctx* ctx, int precision, const void* rho_dev,
                          const uint8_t* failed_dev, uint64_t n, const uint64_t* ranks,
                          int n_ranks, double* values, vxb_comm* comm = nullptr);
uint64_t count_valid_any(vxb_ctx* ctx, int precision, const void* rho_dev,
                         const uint8_t* failed_dev, uint64_t n, uint64_t* only_flag = nullptr,
                         vxb_comm* comm = nullptr);
// type-7 quantile (numeric.cpp:20-36) of n device-resident values (all valid)
double quantile_device(vxb_ctx* ctx, const double* values_dev, uint64_t n, double level);

// vxb_comm.cu -- the communicator as the other translation units see it (comm may be
// null: one rank).  The collectives are queued on the communicator's context stream
// and raise vxb::Error on failure.
int comm_rank(const vxb_comm* comm);
int comm_size(const vxb_comm* comm);
void comm_allgather(vxb_comm* comm, const void* send, void* recv, size_t bytes);
void comm_allreduce_sum_f64(vxb_comm* comm, double* buf, size_t count);
void comm_allreduce_sum_i64(vxb_comm* comm, long long* buf, size_t count);
void comm_allreduce_sum_u32(vxb_comm* comm, unsigned int* buf, size_t count);
// partition(total, world, 1) (blocked.cpp:34-63): range of worker `rank`
void shard_of(uint64_t total, uint64_t world, uint64_t rank, uint64_t* begin, uint64_t* end);

}  // namespace vxb
