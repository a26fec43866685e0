// vxb_comm.cu -- multi-GPU behind the C ABI: the NCCL communicator (loaded at run
// time), the packed accepted-set exchange of config 1 and the one-process /
// several-GPUs drivers (vxb_multi_*).
//
// Replaces the reference's only parallelism, the std::thread fork-join over
// `workers` row ranges (abc.cpp:43-71; partition, blocked.cpp:34-63): a device
// takes the place of a worker thread.  Rows are keyed globally, so the data path
// needs no collective; NCCL over NVLink only moves results (the gather of accepted
// samples).  See include/vexbayes_cuda.h, section "multi-GPU".

#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nccl.h>

#include "vxb_internal.cuh"

namespace vxb {

// ------------------------------------------------------------- NCCL binding
// dlopen instead of a link-time dependency: libvexbayes_cuda.so loads (and runs on
// one GPU) on hosts without NCCL, and inside a Python process that already holds
// torch's bundled libnccl.so.2 the same soname resolves to that copy.
struct Nccl {
    void* handle = nullptr;
    decltype(&ncclGetVersion) GetVersion = nullptr;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    std::string error;
};

static Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = getenv("VXB_NCCL_LIBRARY");
        const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
        for (const char* name : names) {
            if (!name || !*name) continue;
            n.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.handle) break;
            n.error = dlerror();
        }
        if (!n.handle) return;
        auto sym = [&](const char* s) {
            void* p = dlsym(n.handle, s);
            if (!p) n.error = std::string("missing symbol ") + s;
            return p;
        };
        n.GetVersion = reinterpret_cast<decltype(n.GetVersion)>(sym("ncclGetVersion"));
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
        n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
        if (!n.GetVersion || !n.GetUniqueId || !n.CommInitRank || !n.CommDestroy ||
            !n.GetErrorString || !n.AllGather || !n.AllReduce || !n.GroupStart || !n.GroupEnd) {
            dlclose(n.handle);
            n.handle = nullptr;
        }
    });
    if (!n.handle)
        raise("device-error", "NCCL is not available (" + n.error +
                                  "); several GPUs need libnccl.so.2 (set VXB_NCCL_LIBRARY)");
    return n;
}

static void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess && r != ncclInProgress)
        raise("device-error", std::string(what) + ": " + nccl().GetErrorString(r));
}
#define VXB_NCCL(call) ::vxb::nccl_check((call), #call)

static uint64_t align16(uint64_t v) { return (v + 15) & ~uint64_t(15); }

// partition(total, workers, 1) (blocked.cpp:34-63): range of worker `rank`
void shard_of(uint64_t total, uint64_t world, uint64_t rank, uint64_t* begin, uint64_t* end) {
    const uint64_t base = total / world, extra = total % world;
    *begin = rank * base + std::min(rank, extra);
    *end = *begin + base + (rank < extra ? 1 : 0);
}

}  // namespace vxb

// Loopback group (diagnostics): the ranks are host threads of ONE process, each with
// its own vxb_ctx -- all of them may sit on the same GPU -- and a collective is a host
// rendezvous: every rank drains its stream, the ranks meet at a barrier, each copies the
// others' buffers device-to-device on its own stream, and they meet again.  No kernel
// ever waits for another rank (the profiling guide's rule for one-GPU emulation), so the
// multi-rank drivers (sharding offsets, packed gathers, chunk-total reduction, append
// order) run for real on a one-GPU box.  Same results as NCCL by construction: an
// all-gather is a copy, and the only all-reduce of the path adds vectors with one
// non-zero contributor per entry (added here in rank order).
static const char* const kPeerFailed = "another rank of the group failed before the collective";
struct vxb_loopback {
    int size = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long generation = 0;
    std::vector<const void*> slot;
    bool aborted = false;  // a rank failed: nobody may wait for it (fork_join)
    std::atomic<int> fail_rank{-1};  // one-shot fault injection for the tests (VXB_LOOPBACK_FAIL_RANK)
    void barrier() {
        std::unique_lock<std::mutex> lock(m);
        const unsigned long long gen = generation;
        if (!aborted && ++arrived == size) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return;
        }
        cv.wait(lock, [&] { return generation != gen || aborted; });
        if (generation == gen) vxb::raise("device-error", kPeerFailed);
    }
    void abort() {
        std::lock_guard<std::mutex> lock(m);
        aborted = true;
        cv.notify_all();
    }
    void reset() {  // every rank's thread has been joined
        std::lock_guard<std::mutex> lock(m);
        aborted = false;
        arrived = 0;
    }
};

struct vxb_comm {
    vxb_ctx* ctx = nullptr;
    ncclComm_t comm = nullptr;
    int rank = 0, size = 1;
    vxb_loopback* loop = nullptr;  // non-null: loopback group instead of NCCL
};

struct vxb_multi {
    std::vector<vxb_ctx*> ctx;
    std::vector<vxb_comm*> comm;  // empty with one device
    vxb_loopback* loop = nullptr;  // owned (vxb_multi_init_loopback)
};

namespace vxb {
template <class T>
__global__ void loopback_sum_kernel(const T* __restrict__ all, int ranks, size_t count,
                                    T* __restrict__ out) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    T s = 0;
    for (int r = 0; r < ranks; ++r) s = s + all[static_cast<size_t>(r) * count + i];  // rank order
    out[i] = s;
}
static void loopback_allgather(vxb_comm* c, const void* send, void* recv, size_t bytes) {
    vxb_loopback* g = c->loop;
    VXB_CUDA(cudaStreamSynchronize(c->ctx->stream));  // my block is complete
    g->slot[c->rank] = send;
    g->barrier();
    for (int r = 0; r < c->size; ++r)
        VXB_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + static_cast<size_t>(r) * bytes, g->slot[r], bytes,
                                 cudaMemcpyDefault, c->ctx->stream));
    VXB_CUDA(cudaStreamSynchronize(c->ctx->stream));
    g->barrier();  // nobody reuses its send buffer before everyone has copied it
}
template <class T>
static void loopback_allreduce_sum(vxb_comm* c, T* buf, size_t count) {
    Scratch all(c->ctx, static_cast<size_t>(c->size) * count * sizeof(T));
    loopback_allgather(c, buf, all.as<void>(), count * sizeof(T));
    loopback_sum_kernel<T><<<grid_for(count, 256), 256, 0, c->ctx->stream>>>(all.as<T>(), c->size, count, buf);
    check_launch("loopback_sum_kernel");
    VXB_CUDA(cudaStreamSynchronize(c->ctx->stream));
}
}  // namespace vxb

namespace vxb {
int comm_rank(const vxb_comm* comm) { return comm ? comm->rank : 0; }
int comm_size(const vxb_comm* comm) { return comm ? comm->size : 1; }
void comm_allgather(vxb_comm* comm, const void* send, void* recv, size_t bytes) {
    require(comm != nullptr, "invalid-argument", "null communicator");
    if (comm->loop) return loopback_allgather(comm, send, recv, bytes);
    VXB_NCCL(nccl().AllGather(send, recv, bytes, ncclUint8, comm->comm, comm->ctx->stream));
}
void comm_allreduce_sum_f64(vxb_comm* comm, double* buf, size_t count) {
    require(comm != nullptr, "invalid-argument", "null communicator");
    if (comm->loop) return loopback_allreduce_sum<double>(comm, buf, count);
    VXB_NCCL(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, comm->comm, comm->ctx->stream));
}
void comm_allreduce_sum_i64(vxb_comm* comm, long long* buf, size_t count) {
    require(comm != nullptr, "invalid-argument", "null communicator");
    if (comm->loop) return loopback_allreduce_sum<long long>(comm, buf, count);
    VXB_NCCL(nccl().AllReduce(buf, buf, count, ncclInt64, ncclSum, comm->comm, comm->ctx->stream));
}
void comm_allreduce_sum_u32(vxb_comm* comm, unsigned int* buf, size_t count) {
    require(comm != nullptr, "invalid-argument", "null communicator");
    if (comm->loop) return loopback_allreduce_sum<unsigned int>(comm, buf, count);
    VXB_NCCL(nccl().AllReduce(buf, buf, count, ncclUint32, ncclSum, comm->comm, comm->ctx->stream));
}
}  // namespace vxb

using namespace vxb;

// Runs body(rank) on one host thread per device and joins (the fork-join of
// abc.cpp:64-71); the first failure is re-raised on the calling thread.
template <class F>
static void fork_join(vxb_multi* m, F&& body) {
    const int g = static_cast<int>(m->ctx.size());
    std::vector<std::string> err(g);
    auto run = [&](int r) {
        try {
            int expect = r;
            if (m->loop && m->loop->fail_rank.compare_exchange_strong(expect, -1))
                raise("internal", "injected failure (VXB_LOOPBACK_FAIL_RANK)");
            body(r);
        } catch (const Error& e) {
            err[r] = e.code + ": " + e.message;
        } catch (const std::exception& e) {
            err[r] = std::string("internal: ") + e.what();
        }
        // a rank that failed will not arrive at the next collective: the loopback group
        // releases the ranks waiting for it (they fail with kPeerFailed) instead of
        // hanging.  With NCCL a rank-local failure in the middle of a call leaves the
        // peers waiting, as in any NCCL program; argument and shape errors are raised
        // identically on every rank before the first collective.
        if (!err[r].empty() && m->loop) m->loop->abort();
    };
    if (g == 1) {
        run(0);
    } else {
        std::vector<std::thread> pool;
        for (int r = 0; r < g; ++r) pool.emplace_back(run, r);
        for (auto& t : pool) t.join();
    }
    if (m->loop) m->loop->reset();
    for (int pass = 0; pass < 2; ++pass)  // the root cause before the ranks it released
    for (int r = 0; r < g; ++r)
        if (!err[r].empty() && (pass == 1 || err[r].find(kPeerFailed) == std::string::npos)) {
            const size_t c = err[r].find(": ");
            raise(err[r].substr(0, c).c_str(), err[r].substr(c == std::string::npos ? 0 : c + 2) +
                                                   " (device rank " + std::to_string(r) + ")");
        }
}
// an ABI call made on a worker thread: its thread-local error text becomes an Error
static void abi(int rc) {
    if (rc == 0) return;
    const std::string text = vxb_last_error();
    const size_t c = text.find(": ");
    if (c == std::string::npos) raise("internal", text);
    raise(text.substr(0, c).c_str(), text.substr(c + 2));
}

extern "C" int vxb_device_count(int* count) {
    return guarded([&] {
        require(count != nullptr, "invalid-argument", "null output");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *count = n;
    });
}

extern "C" int vxb_comm_version(int* version) {
    return guarded([&] {
        require(version != nullptr, "invalid-argument", "null output");
        VXB_NCCL(nccl().GetVersion(version));
    });
}

extern "C" int vxb_comm_unique_id(void* id) {
    return guarded([&] {
        require(id != nullptr, "invalid-argument", "null output");
        static_assert(sizeof(ncclUniqueId) == VXB_COMM_ID_BYTES, "unique id size");
        ncclUniqueId u;
        VXB_NCCL(nccl().GetUniqueId(&u));
        std::memcpy(id, &u, sizeof(u));
    });
}

extern "C" int vxb_comm_init_rank(vxb_ctx* ctx, const void* id, int rank, int n_ranks,
                                  vxb_comm** comm) {
    return guarded([&] {
        use(ctx);
        require(id && comm, "invalid-argument", "null argument");
        require(n_ranks >= 1 && rank >= 0 && rank < n_ranks, "invalid-argument", "bad rank");
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        auto* c = new vxb_comm();
        c->ctx = ctx;
        c->rank = rank;
        c->size = n_ranks;
        const ncclResult_t r = nccl().CommInitRank(&c->comm, n_ranks, u, rank);
        if (r != ncclSuccess) {
            delete c;
            nccl_check(r, "ncclCommInitRank");
        }
        *comm = c;
    });
}

extern "C" void vxb_comm_destroy(vxb_comm* comm) {
    if (!comm) return;
    if (comm->comm && !comm->loop) {
        cudaSetDevice(comm->ctx->device);
        cudaStreamSynchronize(comm->ctx->stream);
        nccl().CommDestroy(comm->comm);
    }
    delete comm;
}

extern "C" int vxb_comm_rank(const vxb_comm* comm) { return comm ? comm->rank : 0; }
extern "C" int vxb_comm_size(const vxb_comm* comm) { return comm ? comm->size : 1; }

extern "C" int vxb_comm_allgather(vxb_comm* comm, const void* send, void* recv, size_t bytes) {
    return guarded([&] {
        require(comm && send && recv, "invalid-argument", "null argument");
        use(comm->ctx);
        comm_allgather(comm, send, recv, bytes);
    });
}

extern "C" int vxb_comm_allreduce(vxb_comm* comm, void* buf, size_t count, int dtype, int op) {
    return guarded([&] {
        require(comm && buf, "invalid-argument", "null argument");
        use(comm->ctx);
        if (comm->loop) {
            require(op == VXB_OP_SUM && (dtype == VXB_DT_F64 || dtype == VXB_DT_I64 || dtype == VXB_DT_U64),
                    "invalid-argument", "the loopback group reduces 64-bit elements by SUM only");
            if (dtype == VXB_DT_F64) return comm_allreduce_sum_f64(comm, static_cast<double*>(buf), count);
            return comm_allreduce_sum_i64(comm, static_cast<long long*>(buf), count);
        }
        ncclDataType_t dt;
        switch (dtype) {
            case VXB_DT_U8: dt = ncclUint8; break;
            case VXB_DT_I64: dt = ncclInt64; break;
            case VXB_DT_U64: dt = ncclUint64; break;
            case VXB_DT_U32: dt = ncclUint32; break;
            case VXB_DT_F64: dt = ncclFloat64; break;
            default: raise("invalid-argument", "unknown element type");
        }
        require(op == VXB_OP_SUM || op == VXB_OP_MAX, "invalid-argument", "unknown reduction");
        VXB_NCCL(nccl().AllReduce(buf, buf, count, dt, op == VXB_OP_SUM ? ncclSum : ncclMax,
                                  comm->comm, comm->ctx->stream));
    });
}

// ----------------------------------------------- packed accepted sets (config 1)
extern "C" int vxb_accept_layout_of(int precision, uint32_t dim, uint64_t cap,
                                    vxb_accept_layout* out) {
    return guarded([&] {
        require(out != nullptr, "invalid-argument", "null output");
        require(precision == VXB_F64 || precision == VXB_F32, "invalid-argument", "bad precision");
        require(dim >= 1 && cap >= 1, "invalid-shape", "need dim >= 1 and cap >= 1");
        const uint64_t real = precision == VXB_F32 ? 4 : 8;
        out->cap = cap;
        out->off_count = 0;
        out->off_idx = 16;
        out->off_params = out->off_idx + align16(cap * 8);
        out->off_rho = out->off_params + align16(cap * dim * real);
        out->stride = out->off_rho + align16(cap * real);
    });
}

extern "C" int vxb_sharded_abc_reject(vxb_ctx* ctx, vxb_comm* comm, const vxb_model* model,
                                      const vxb_keying* key, uint64_t n_total,
                                      const double* observed, double epsilon,
                                      const vxb_accept_layout* layout, void* packed_local,
                                      void* packed_all) {
    return guarded([&] {
        use(ctx);
        require(model && key && layout && packed_local, "invalid-argument", "null argument");
        require(is_device_pointer(packed_local), "invalid-argument", "packed_local is a device buffer");
        require(!comm || comm->ctx == ctx, "invalid-argument", "communicator of another context");
        const int world = comm ? comm->size : 1, rank = comm ? comm->rank : 0;
        require(world == 1 || (packed_all && is_device_pointer(packed_all)), "invalid-argument",
                "packed_all is a device buffer of n_ranks blocks");
        uint64_t begin, end;
        shard_of(n_total, world, rank, &begin, &end);
        char* base = static_cast<char*>(packed_local);
        abi(vxb_abc_reject(ctx, model, key, n_total, begin, end - begin, observed, epsilon,
                           layout->cap, reinterpret_cast<uint64_t*>(base + layout->off_count),
                           reinterpret_cast<uint64_t*>(base + layout->off_idx),
                           base + layout->off_params, base + layout->off_rho));
        if (comm && packed_all)  // a one-rank communicator gathers too (the NCCL path on a one-GPU box)
            comm_allgather(comm, packed_local, packed_all, layout->stride);
        else if (packed_all && packed_all != packed_local)
            VXB_CUDA(cudaMemcpyAsync(packed_all, packed_local, layout->stride,
                                     cudaMemcpyDeviceToDevice, ctx->stream));
    });
}

extern "C" int vxb_accept_unpack(const vxb_accept_layout* layout, int precision, uint32_t dim,
                                 int n_ranks, const void* packed_all_host, uint64_t cap_out,
                                 uint64_t* n_accepted, uint64_t* idx, void* params, void* rho,
                                 int* overflowed, uint64_t* n_written) {
    return guarded([&] {
        require(layout && packed_all_host && n_accepted && n_ranks >= 1, "invalid-argument",
                "null argument");
        const uint64_t real = precision == VXB_F32 ? 4 : 8;
        uint64_t total = 0, kept = 0;
        bool over = false;
        for (int r = 0; r < n_ranks; ++r) {
            const char* base = static_cast<const char*>(packed_all_host) + r * layout->stride;
            uint64_t c;
            std::memcpy(&c, base + layout->off_count, 8);
            total += c;
            if (c > layout->cap) {
                over = true;
                c = layout->cap;
            }
            const uint64_t take = std::min(c, cap_out - std::min(cap_out, kept));
            if (take) {
                if (idx) std::memcpy(idx + kept, base + layout->off_idx, take * 8);
                if (params)
                    std::memcpy(static_cast<char*>(params) + kept * dim * real,
                                base + layout->off_params, take * dim * real);
                if (rho)
                    std::memcpy(static_cast<char*>(rho) + kept * real, base + layout->off_rho,
                                take * real);
            }
            kept += take;
        }
        *n_accepted = total;
        if (overflowed) *overflowed = over ? 1 : 0;
        if (n_written) *n_written = kept;
    });
}

// ---------------------------------------------- one process, several GPUs
extern "C" int vxb_multi_init(vxb_multi** multi, const int* device_ids, int n_dev) {
    return guarded([&] {
        require(multi != nullptr, "invalid-argument", "null output");
        int visible = 0;
        if (cudaGetDeviceCount(&visible) != cudaSuccess || visible == 0)
            raise("device-error", "no CUDA device available (there is no CPU fallback)");
        std::vector<int> ids;
        if (!device_ids || n_dev <= 0)
            for (int d = 0; d < visible; ++d) ids.push_back(d);
        else
            ids.assign(device_ids, device_ids + n_dev);
        for (size_t a = 0; a < ids.size(); ++a) {
            require(ids[a] >= 0 && ids[a] < visible, "invalid-argument", "device index out of range");
            for (size_t b = 0; b < a; ++b)
                require(ids[a] != ids[b], "invalid-argument", "a device is listed twice");
        }
        auto* m = new vxb_multi();
        try {
            for (int d : ids) {
                vxb_ctx* c = nullptr;
                abi(vxb_init(&c, d));
                m->ctx.push_back(c);
            }
            const int g = static_cast<int>(ids.size());
            if (g > 1) {
                ncclUniqueId u;
                VXB_NCCL(nccl().GetUniqueId(&u));
                m->comm.resize(g, nullptr);
                // all ranks of one process: group the blocking initialisations
                VXB_NCCL(nccl().GroupStart());
                for (int r = 0; r < g; ++r) {
                    auto* c = new vxb_comm();
                    c->ctx = m->ctx[r];
                    c->rank = r;
                    c->size = g;
                    m->comm[r] = c;
                    VXB_CUDA(cudaSetDevice(ids[r]));
                    VXB_NCCL(nccl().CommInitRank(&c->comm, g, u, r));
                }
                VXB_NCCL(nccl().GroupEnd());
            }
        } catch (...) {
            vxb_multi_shutdown(m);
            throw;
        }
        *multi = m;
    });
}

// Diagnostics: n_ranks contexts on ONE device joined by a loopback group, so that every
// vxb_multi_* driver runs its multi-rank logic on a one-GPU box.
extern "C" int vxb_multi_init_loopback(vxb_multi** multi, int device, int n_ranks) {
    return guarded([&] {
        require(multi != nullptr && n_ranks >= 1 && n_ranks <= 64, "invalid-argument", "bad rank count");
        auto* m = new vxb_multi();
        try {
            m->loop = new vxb_loopback();
            m->loop->size = n_ranks;
            m->loop->slot.assign(n_ranks, nullptr);
            if (const char* f = getenv("VXB_LOOPBACK_FAIL_RANK")) m->loop->fail_rank = atoi(f);
            for (int r = 0; r < n_ranks; ++r) {
                vxb_ctx* c = nullptr;
                abi(vxb_init(&c, device));
                m->ctx.push_back(c);
            }
            if (n_ranks > 1)
                for (int r = 0; r < n_ranks; ++r) {
                    auto* c = new vxb_comm();
                    c->ctx = m->ctx[r];
                    c->rank = r;
                    c->size = n_ranks;
                    c->loop = m->loop;
                    m->comm.push_back(c);
                }
        } catch (...) {
            vxb_multi_shutdown(m);
            throw;
        }
        *multi = m;
    });
}

extern "C" void vxb_multi_shutdown(vxb_multi* m) {
    if (!m) return;
    for (vxb_comm* c : m->comm) vxb_comm_destroy(c);
    for (vxb_ctx* c : m->ctx) vxb_shutdown(c);
    delete m->loop;
    delete m;
}

extern "C" int vxb_multi_size(const vxb_multi* m) { return m ? static_cast<int>(m->ctx.size()) : 0; }
extern "C" vxb_ctx* vxb_multi_ctx(vxb_multi* m, int rank) {
    return m && rank >= 0 && rank < static_cast<int>(m->ctx.size()) ? m->ctx[rank] : nullptr;
}
extern "C" vxb_comm* vxb_multi_comm(vxb_multi* m, int rank) {
    return m && rank >= 0 && rank < static_cast<int>(m->comm.size()) ? m->comm[rank] : nullptr;
}

extern "C" int vxb_multi_abc_prior_predictive(vxb_multi* m, const vxb_model* model,
                                              const vxb_keying* key, uint64_t n,
                                              const double* observed, void* params,
                                              void* summaries, void* rho, uint8_t* failed) {
    return guarded([&] {
        require(m && model && key && observed, "invalid-argument", "null argument");
        require(n >= 1, "invalid-shape", "need at least one prior predictive sample");
        const uint64_t real = model->precision == VXB_F32 ? 4 : 8;
        const uint64_t g = m->ctx.size();
        fork_join(m, [&](int r) {
            uint64_t b, e;
            shard_of(n, g, r, &b, &e);
            if (e == b) return;
            auto at = [&](void* p, uint64_t row_bytes) {
                return p ? static_cast<void*>(static_cast<char*>(p) + b * row_bytes) : nullptr;
            };
            abi(vxb_abc_prior_predictive(m->ctx[r], model, key, n, b, e - b, observed,
                                         at(params, model->dim * real),
                                         at(summaries, model->summary_dim * real), at(rho, real),
                                         failed ? failed + b : nullptr, nullptr));
        });
    });
}

extern "C" int vxb_multi_abc_reject(vxb_multi* m, const vxb_model* model, const vxb_keying* key,
                                    uint64_t n_total, const double* observed, double epsilon,
                                    uint64_t cap, uint64_t* n_accepted, uint64_t* idx, void* params,
                                    void* rho) {
    return guarded([&] {
        require(m && model && key && observed && n_accepted, "invalid-argument", "null argument");
        const int g = static_cast<int>(m->ctx.size());
        // per-rank capacity: the whole budget (a rank may hold every accepted row)
        vxb_accept_layout lay;
        abi(vxb_accept_layout_of(model->precision, model->dim, std::max<uint64_t>(cap, 1), &lay));
        std::vector<char> host(static_cast<size_t>(g) * lay.stride);
        fork_join(m, [&](int r) {
            vxb_ctx* ctx = m->ctx[r];
            VXB_CUDA(cudaSetDevice(ctx->device));
            Scratch local(ctx, lay.stride), all(ctx, g > 1 ? g * lay.stride : 0);
            abi(vxb_sharded_abc_reject(ctx, g > 1 ? m->comm[r] : nullptr, model, key, n_total,
                                       observed, epsilon, &lay, local.as<void>(), all.as<void>()));
            if (r == 0)  // every device holds the gathered set; device 0 hands it to the host
                VXB_CUDA(cudaMemcpyAsync(host.data(), g > 1 ? all.as<void>() : local.as<void>(),
                                         host.size(), cudaMemcpyDeviceToHost, ctx->stream));
            VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        });
        int over = 0;
        abi(vxb_accept_unpack(&lay, model->precision, model->dim, g, host.data(), cap, n_accepted, idx,
                              params, rho, &over, nullptr));
    });
}

// select_epsilon (abc.cpp:74-106) over a prior predictive set held in host arrays: every
// device takes the rows of its partition range, the digit histograms are all-reduced and
// the accepted indices come back in ascending order (rank order = row order).
extern "C" int vxb_multi_select_epsilon(vxb_multi* m, int precision, const void* rho,
                                        const uint8_t* failed, uint64_t n, double accept_fraction,
                                        double* epsilon, uint64_t cap, uint64_t* n_accepted,
                                        uint64_t* idx) {
    return guarded([&] {
        require(m && rho && epsilon && n_accepted, "invalid-argument", "null argument");
        require(n >= 1, "empty-set", "every prior predictive row failed");
        require(!is_device_pointer(rho), "invalid-argument", "vxb_multi_select_epsilon takes host arrays");
        const int g = static_cast<int>(m->ctx.size());
        const uint64_t real = precision == VXB_F32 ? 4 : 8;
        const size_t block = VXB_INDEX_BLOCK_BYTES(cap);
        std::vector<char> host(cap ? static_cast<size_t>(g) * block : 0);
        fork_join(m, [&](int r) {
            vxb_ctx* ctx = m->ctx[r];
            VXB_CUDA(cudaSetDevice(ctx->device));
            uint64_t b, e;
            shard_of(n, g, r, &b, &e);
            Scratch local(ctx, cap ? block : 0), all(ctx, cap && g > 1 ? g * block : 0);
            double eps = 0.0;
            uint64_t total = 0;
            abi(vxb_sharded_select_epsilon(ctx, g > 1 ? m->comm[r] : nullptr, precision,
                                           static_cast<const char*>(rho) + b * real,
                                           failed ? failed + b : nullptr, e - b, b, accept_fraction, &eps,
                                           &total, cap, local.as<void>(), all.as<void>()));
            if (r == 0) {
                *epsilon = eps;
                *n_accepted = total;
                if (cap)
                    VXB_CUDA(cudaMemcpyAsync(host.data(), g > 1 ? all.as<void>() : local.as<void>(),
                                             host.size(), cudaMemcpyDeviceToHost, ctx->stream));
            }
            VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        });
        uint64_t kept = 0;
        for (int r = 0; r < g && idx && cap; ++r) {
            uint64_t c;
            std::memcpy(&c, host.data() + r * block, 8);
            const uint64_t take = std::min(std::min(c, cap), cap - kept);
            std::memcpy(idx + kept, host.data() + r * block + 16, take * 8);
            kept += take;
        }
    });
}

extern "C" int vxb_multi_ppp_pvalues(vxb_multi* m, const vxb_model* model, const double* lambda,
                                     const double* log_norm, uint32_t n_lambda, uint64_t m_total,
                                     uint64_t seed, double ybar_obs, uint64_t* counts,
                                     double* pvalues) {
    return guarded([&] {
        require(m && model && lambda && log_norm && counts, "invalid-argument", "null argument");
        const int g = static_cast<int>(m->ctx.size());
        fork_join(m, [&](int r) {  // SPMD on one host thread per device; rank 0 reports
            std::vector<uint64_t> c(n_lambda);
            abi(vxb_sharded_ppp_pvalues(m->ctx[r], g > 1 ? m->comm[r] : nullptr, model, lambda, log_norm,
                                        n_lambda, m_total, seed, ybar_obs, r == 0 ? counts : c.data(),
                                        r == 0 ? pvalues : nullptr));
        });
    });
}

extern "C" int vxb_multi_mlmc_tauleap(vxb_multi* m, const vxb_model* model, const vxb_mlmc_cfg* cfg,
                                      vxb_mlmc_out* out) {
    return guarded([&] {
        require(m && model && cfg && out, "invalid-argument", "null argument");
        const int g = static_cast<int>(m->ctx.size());
        fork_join(m, [&](int r) {
            vxb_mlmc_out none{};
            abi(vxb_sharded_mlmc_tauleap(m->ctx[r], g > 1 ? m->comm[r] : nullptr, model, cfg,
                                         r == 0 ? out : &none));
        });
    });
}

// ABC-SMC over all devices: every device runs the SPMD driver on its own host thread;
// device 0's copy of the (replicated) result goes to the caller.
extern "C" int vxb_multi_abcsmc_run(vxb_multi* m, const vxb_model* model, const vxb_abcsmc_cfg* cfg,
                                    const double* observed, vxb_abcsmc_out* out) {
    return guarded([&] {
        require(m && model && cfg && observed && out, "invalid-argument", "null argument");
        const int g = static_cast<int>(m->ctx.size());
        fork_join(m, [&](int r) {
            vxb_abcsmc_out none{};  // the other ranks compute the same numbers and drop them
            abi(vxb_sharded_abcsmc_run(m->ctx[r], g > 1 ? m->comm[r] : nullptr, model, cfg, observed,
                                       r == 0 ? out : &none));
        });
    });
}

// run_weak_info_test (weak_info.cpp:163-277) with the hyperparameter rows split over
// the devices -- the reference's own task parallelism (weak_info.cpp:248-270: `workers`
// threads over rows); sampler seeds are keyed by (row, dataset), so the table does not
// depend on the device count.  No collective: every device writes its rows of the
// caller's host evidence table.
extern "C" int vxb_multi_weak_info_test(vxb_multi* m, const vxb_weakinfo_cfg* cfg, double* lambda,
                                        double* gamma, uint8_t* weakly, uint64_t* completed,
                                        double* evidence) {
    return guarded([&] {
        require(m && cfg && lambda && gamma && weakly && completed, "invalid-argument", "null argument");
        require(cfg->datasets >= 1, "invalid-argument", "need at least one dataset per prior");
        require(cfg->alpha > 0.0 && cfg->alpha < 1.0, "invalid-argument", "alpha must lie in (0, 1)");
        const uint64_t rows = cfg->hyper_count + 1, g = m->ctx.size();
        std::vector<double> own;
        if (!evidence) {
            own.resize(rows * cfg->datasets * 2);
            evidence = own.data();
        }
        abi(vxb_weak_info_lambdas(m->ctx[0], cfg, lambda));
        fork_join(m, [&](int r) {
            uint64_t b, e;
            shard_of(rows, g, r, &b, &e);
            if (e == b) return;
            abi(vxb_weak_info_evidence(m->ctx[r], cfg, lambda, b, e - b, evidence + b * cfg->datasets * 2));
        });
        abi(vxb_weak_info_cutoffs(cfg, evidence, gamma, weakly, completed));
    });
}

// ---- SPMD forms of configs 2 and 4 (every rank calls them; comm == NULL: one rank):
// disjoint dataset / path ranges per rank, ONE all-reduce(SUM) of the 64-bit integer
// counters (exact in any order), every rank receives the job's totals.
extern "C" int vxb_sharded_ppp_pvalues(vxb_ctx* ctx, vxb_comm* comm, const vxb_model* model,
                                       const double* lambda, const double* log_norm,
                                       uint32_t n_lambda, uint64_t m_total, uint64_t seed,
                                       double ybar_obs, uint64_t* counts, double* pvalues) {
    return guarded([&] {
        use(ctx);
        require(model && lambda && log_norm && counts && n_lambda >= 1, "invalid-argument", "null argument");
        require(!comm || comm->ctx == ctx, "invalid-argument", "communicator of another context");
        const uint64_t world = comm_size(comm), rank = comm_rank(comm);
        uint64_t b, e;
        shard_of(m_total, world, rank, &b, &e);
        std::vector<uint64_t> local(n_lambda, 0);
        if (e > b)
            abi(vxb_ppp_pvalues(ctx, model, lambda, log_norm, n_lambda, m_total, b, e - b, seed, ybar_obs,
                                local.data(), nullptr, nullptr));
        if (comm) {
            Scratch d(ctx, n_lambda * 8);
            VXB_CUDA(cudaMemcpyAsync(d.as<void>(), local.data(), n_lambda * 8, cudaMemcpyHostToDevice, ctx->stream));
            comm_allreduce_sum_i64(comm, d.as<long long>(), n_lambda);
            VXB_CUDA(cudaMemcpyAsync(local.data(), d.as<void>(), n_lambda * 8, cudaMemcpyDeviceToHost, ctx->stream));
            VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        for (uint32_t k = 0; k < n_lambda; ++k) {
            counts[k] = local[k];
            if (pvalues) pvalues[k] = static_cast<double>(local[k]) / static_cast<double>(m_total);
        }
    });
}

extern "C" int vxb_sharded_mlmc_tauleap(vxb_ctx* ctx, vxb_comm* comm, const vxb_model* model,
                                        const vxb_mlmc_cfg* cfg, vxb_mlmc_out* out) {
    return guarded([&] {
        use(ctx);
        require(model && cfg && out, "invalid-argument", "null argument");
        require(cfg->paths >= 2, "insufficient-data", "variance needs at least two values");
        require(cfg->tau0 > 0.0 && cfg->t_end > 0.0, "invalid-horizon", "need a positive horizon");
        require(!comm || comm->ctx == ctx, "invalid-argument", "communicator of another context");
        const uint64_t world = comm_size(comm), rank = comm_rank(comm);
        uint64_t b, e;
        shard_of(cfg->paths, world, rank, &b, &e);
        std::vector<long long> sums(cfg->levels * 4, 0);
        if (e > b)
            for (uint32_t l = 0; l < cfg->levels; ++l)
                abi(vxb_mlmc_level(ctx, model, cfg, l, b, e - b, reinterpret_cast<int64_t*>(sums.data() + 4 * l),
                                   nullptr));
        if (comm) {
            Scratch d(ctx, sums.size() * 8);
            VXB_CUDA(cudaMemcpyAsync(d.as<void>(), sums.data(), sums.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            comm_allreduce_sum_i64(comm, d.as<long long>(), sums.size());
            VXB_CUDA(cudaMemcpyAsync(sums.data(), d.as<void>(), sums.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
            VXB_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        double est = 0.0, var = 0.0;
        uint64_t steps = static_cast<uint64_t>(std::llround(cfg->t_end / cfg->tau0));
        const double n = static_cast<double>(cfg->paths);
        for (uint32_t l = 0; l < cfg->levels; ++l) {
            const double s0 = static_cast<double>(sums[4 * l]), s1 = static_cast<double>(sums[4 * l + 1]);
            const double mean = s0 / n;
            const double v = (s1 - s0 * mean) / (n - 1.0);
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
