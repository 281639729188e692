// Shard collectives (exchange.hpp): NCCL over NVLink / NVSwitch, or in-process device copies.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "device.hpp"
#include "exchange.hpp"

namespace qsr {

namespace {

// ---- local transport -----------------------------------------------------------------
constexpr int kMaxLocal = 64;
struct PtrList { uint8_t *p[kMaxLocal]; };

__global__ void k_max_u8(PtrList bufs, int nbuf, size_t bytes) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < bytes;
         i += size_t(gridDim.x) * blockDim.x) {
        uint8_t v = bufs.p[0][i];
        for (int b = 1; b < nbuf; ++b) v = max(v, bufs.p[b][i]);
        for (int b = 0; b < nbuf; ++b) bufs.p[b][i] = v;
    }
}

__global__ void k_max_u64(PtrList bufs, int nbuf, size_t words) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < words;
         i += size_t(gridDim.x) * blockDim.x) {
        uint64_t v = reinterpret_cast<const uint64_t *>(bufs.p[0])[i];
        for (int b = 1; b < nbuf; ++b) v = max(v, reinterpret_cast<const uint64_t *>(bufs.p[b])[i]);
        for (int b = 0; b < nbuf; ++b) reinterpret_cast<uint64_t *>(bufs.p[b])[i] = v;
    }
}

class LocalExchange final : public Exchange {
  public:
    LocalExchange(int w, const std::vector<cudaStream_t> &st) {
        if (w < 1 || w > kMaxLocal) fail(QSR_INVALID_ARGUMENT, "local exchange: 1..64 shards");
        if (int(st.size()) != w) fail(QSR_INTERNAL, "local exchange: one stream per shard");
        world = w;
        streams = st;
        for (int r = 0; r < w; ++r) ranks.push_back(r);
        events.resize(w);
        for (auto &e : events) QSR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    ~LocalExchange() override {
        for (auto e : events) cudaEventDestroy(e);
    }
    // Every stream waits for the work enqueued so far on every other stream.
    void barrier() {
        for (int i = 0; i < world; ++i) QSR_CUDA(cudaEventRecord(events[i], streams[i]));
        for (int i = 0; i < world; ++i)
            for (int j = 0; j < world; ++j)
                if (i != j) QSR_CUDA(cudaStreamWaitEvent(streams[i], events[j], 0));
    }
    void broadcast(const std::vector<void *> &buf, size_t bytes, int root) override {
        barrier();
        for (int i = 0; i < world; ++i)
            if (i != root)
                QSR_CUDA(cudaMemcpyAsync(buf[i], buf[root], bytes, cudaMemcpyDeviceToDevice,
                                         streams[i]));
        barrier();
    }
    void allgather(const std::vector<const void *> &send, const std::vector<void *> &recv,
                   size_t bytes) override {
        barrier();
        for (int i = 0; i < world; ++i)
            for (int j = 0; j < world; ++j)
                QSR_CUDA(cudaMemcpyAsync(static_cast<uint8_t *>(recv[i]) + size_t(j) * bytes,
                                         send[j], bytes, cudaMemcpyDeviceToDevice, streams[i]));
        barrier();
    }
    void allreduce_max_u8(const std::vector<void *> &buf, size_t bytes) override {
        if (bytes == 0) return;
        barrier();
        PtrList pl{};
        for (int i = 0; i < world; ++i) pl.p[i] = static_cast<uint8_t *>(buf[i]);
        const unsigned blocks = unsigned(std::min<size_t>((bytes + 255) / 256, 1024));
        k_max_u8<<<blocks, 256, 0, streams[0]>>>(pl, world, bytes);
        QSR_CUDA(cudaGetLastError());
        count_launch();
        barrier();
    }
    void allreduce_max_u64(const std::vector<void *> &buf, size_t words) override {
        if (words == 0) return;
        barrier();
        PtrList pl{};
        for (int i = 0; i < world; ++i) pl.p[i] = static_cast<uint8_t *>(buf[i]);
        const unsigned blocks = unsigned(std::min<size_t>((words + 255) / 256, 1024));
        k_max_u64<<<blocks, 256, 0, streams[0]>>>(pl, world, words);
        QSR_CUDA(cudaGetLastError());
        count_launch();
        barrier();
    }
    const char *kind() const override { return "local"; }

  private:
    std::vector<cudaEvent_t> events;
};

// ---- NCCL transport (libnccl.so.2 loaded at first use) ---------------------------------
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api = [] {
        NcclApi a;
        // Prefer the NCCL already mapped into the process (torch's), then $QSR_NCCL_LIB, then
        // the system library.
        a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!a.h)
            if (const char *p = getenv("QSR_NCCL_LIB")) a.h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
        if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!a.h) return a;
        auto sym = [&](auto &fn, const char *s) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(a.h, s)); };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.Broadcast, "ncclBroadcast");
        sym(a.AllGather, "ncclAllGather");
        sym(a.AllReduce, "ncclAllReduce");
        sym(a.GetErrorString, "ncclGetErrorString");
        return a;
    }();
    if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.Broadcast || !api.AllGather ||
        !api.AllReduce)
        fail(QSR_NCCL_ERROR, "NCCL (libnccl.so.2) is not available in this process");
    return api;
}

void nccl_check(ncclResult_t r, const char *what) {
    if (r == ncclSuccess) return;
    const char *m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    fail(QSR_NCCL_ERROR, std::string(what) + ": " + m);
}

// Communicators are cached per (unique id, world, rank, device): a ncclUniqueId's bootstrap
// root serves exactly one ncclCommInitRank round, so an engine rebuilt with the same id (bench.py
// recreates the sharded engine every e2e step) must reuse the communicator instead of
// re-initialising — a second init on a spent id would wait for the root forever. Engines sharing
// a communicator run one after another (calls are synchronous), never concurrently.
std::mutex g_comm_mu;
std::map<std::string, ncclComm_t> g_comms;

ncclComm_t comm_for(int w, int rank, const void *uid) {
    int dev = 0;
    QSR_CUDA(cudaGetDevice(&dev));
    std::string key(static_cast<const char *>(uid), sizeof(ncclUniqueId));
    key += ":" + std::to_string(w) + ":" + std::to_string(rank) + ":" + std::to_string(dev);
    std::lock_guard<std::mutex> g(g_comm_mu);
    auto it = g_comms.find(key);
    if (it != g_comms.end()) return it->second;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    ncclComm_t c = nullptr;
    nccl_check(nccl().CommInitRank(&c, w, id, rank), "ncclCommInitRank");
    g_comms.emplace(key, c);
    return c;
}

class NcclExchange final : public Exchange {
  public:
    NcclExchange(int w, int rank, cudaStream_t st, const void *uid) {
        if (w < 1 || rank < 0 || rank >= w) fail(QSR_INVALID_ARGUMENT, "nccl exchange: bad rank/world");
        world = w;
        ranks = {rank};
        streams = {st};
        comm = comm_for(w, rank, uid);
    }
    ~NcclExchange() override = default; // the communicator stays cached (see comm_for)
    void broadcast(const std::vector<void *> &buf, size_t bytes, int root) override {
        nccl_check(nccl().Broadcast(buf[0], buf[0], bytes, ncclUint8, root, comm, streams[0]),
                   "ncclBroadcast");
    }
    void allgather(const std::vector<const void *> &send, const std::vector<void *> &recv,
                   size_t bytes) override {
        nccl_check(nccl().AllGather(send[0], recv[0], bytes, ncclUint8, comm, streams[0]),
                   "ncclAllGather");
    }
    void allreduce_max_u8(const std::vector<void *> &buf, size_t bytes) override {
        if (bytes == 0) return;
        nccl_check(nccl().AllReduce(buf[0], buf[0], bytes, ncclUint8, ncclMax, comm, streams[0]),
                   "ncclAllReduce");
    }
    void allreduce_max_u64(const std::vector<void *> &buf, size_t words) override {
        if (words == 0) return;
        nccl_check(nccl().AllReduce(buf[0], buf[0], words, ncclUint64, ncclMax, comm, streams[0]),
                   "ncclAllReduce");
    }
    const char *kind() const override { return "nccl"; }

  private:
    ncclComm_t comm = nullptr;
};

} // namespace

std::unique_ptr<Exchange> make_local_exchange(int world, const std::vector<cudaStream_t> &streams) {
    return std::make_unique<LocalExchange>(world, streams);
}

std::unique_ptr<Exchange> make_nccl_exchange(int world, int rank, cudaStream_t stream,
                                             const void *unique_id) {
    return std::make_unique<NcclExchange>(world, rank, stream, unique_id);
}

void nccl_unique_id(void *out) {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

} // namespace qsr
