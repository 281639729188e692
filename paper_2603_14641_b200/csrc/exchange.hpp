// Collectives between the generator-word shards of one tableau.
//
// The sharded engine (shard.cpp) is written once against this interface; two transports
// implement it:
//   * NCCL  — one process per GPU (torch.distributed rendezvous hands over the ncclUniqueId);
//             broadcast / all-gather / max-all-reduce run over NVLink / NVSwitch on the
//             shard's own stream, ordered with its kernels, no host synchronisation.
//   * local — every shard of the tableau lives in this process (on one device): the same
//             collectives as device-to-device copies ordered by events. It runs the exact
//             sharded algorithm on a single GPU, so the multi-GPU measurement protocol is
//             parity-tested bit-for-bit on the one-GPU boxes available to the tests.
// Every call is collective over all `world` shards; buffers are device pointers, one per
// local shard, in the order of `ranks`.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

namespace qsr {

class Exchange {
  public:
    virtual ~Exchange() = default;
    int world = 1;
    std::vector<int> ranks;            // global rank of each local shard (ascending)
    std::vector<cudaStream_t> streams; // the local shards' streams

    // In place: every shard's buf receives root's bytes (root = global rank).
    virtual void broadcast(const std::vector<void *> &buf, size_t bytes, int root) = 0;
    // recv[i] receives world * bytes: shard r's `send` at offset r * bytes.
    virtual void allgather(const std::vector<const void *> &send, const std::vector<void *> &recv,
                           size_t bytes) = 0;
    // In place, element-wise max over uint8.
    virtual void allreduce_max_u8(const std::vector<void *> &buf, size_t bytes) = 0;
    // In place, element-wise max over uint64: a broadcast from a root the host does not know
    // when every other shard contributes zeros (the batch block, shard.cpp).
    virtual void allreduce_max_u64(const std::vector<void *> &buf, size_t words) = 0;
    virtual const char *kind() const = 0;
};

// All `world` shards in this process on one device, one stream each.
std::unique_ptr<Exchange> make_local_exchange(int world, const std::vector<cudaStream_t> &streams);
// This process drives shard `rank` of `world` on the current device (collective init).
std::unique_ptr<Exchange> make_nccl_exchange(int world, int rank, cudaStream_t stream,
                                             const void *unique_id /* 128 bytes */);
// ncclGetUniqueId through the dynamically loaded NCCL (throws QSR_NCCL_ERROR if unavailable).
void nccl_unique_id(void *out /* 128 bytes */);

} // namespace qsr
