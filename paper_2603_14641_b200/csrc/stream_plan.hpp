// Planner of the streaming single-shot driver (stream.cpp), host only: the one-pass round closed
// form of the window scheduler (host_circuit.cpp plan_windows; reference schedule.hpp:51-137)
// applied chunk by chunk, each gate appended to the bucket of its window key.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "host.hpp"

namespace qsr {

// Buckets of packed gates per window key, in pages that never move: the planner appends to keys
// at or above the published limit while the emitter reads (and recycles) keys below it.
class BucketDir {
  public:
    explicit BucketDir(uint64_t max_keys) : pages_((max_keys + kPage - 1) / kPage) {}
    std::vector<uint64_t> &operator[](uint64_t key) {
        auto &pg = pages_[key / kPage];
        if (!pg) pg = std::make_unique<Page>();
        return (*pg)[key % kPage];
    }
    std::vector<uint64_t> *find(uint64_t key) {
        auto &pg = pages_[key / kPage];
        return pg ? &(*pg)[key % kPage] : nullptr;
    }

  private:
    static constexpr uint64_t kPage = 1024;
    using Page = std::array<std::vector<uint64_t>, kPage>;
    std::vector<std::unique_ptr<Page>> pages_;
};

// Wire state = round << 1 | (the wire's last gate was a MEASURE). plan() raises the reference's
// scheduling errors (check_valid, circuit.hpp:108-115; a measurement chained behind another in one
// window, measure.hpp:394-395) at the offending gate.
template <typename FreshBucket>
class ChunkPlanner {
  public:
    ChunkPlanner(uint32_t n, BucketDir &b, FreshBucket fresh) : n_(n), wire_(n, 0), buckets_(b), fresh_(fresh) {}

    void plan(const qsr_gate *gates, uint64_t i0, uint64_t i1) {
        uint32_t *wire = wire_.data();
        const uint32_t n = n_;
        // Consecutive gates of a layer share a key: the bucket is looked up only when it changes
        // (a bucket never moves; the emitter only touches keys below the published limit, and no
        // gate planned later has such a key).
        uint64_t cur_key = ~uint64_t(0);
        std::vector<uint64_t> *cur = nullptr;
        for (uint64_t i = i0; i < i1; ++i) {
            const qsr_gate g = gates[i];
            const uint32_t kind = g.kind;
            if (kind > QSR_MEASURE) fail(QSR_INVALID_ARGUMENT, "unknown gate kind");
            const bool two = kind >= QSR_CX && kind <= QSR_ISWAP;
            const uint32_t q0 = g.q0, q1 = two ? g.q1 : g.q0;
            if (q0 >= n || q1 >= n) fail(QSR_OUT_OF_RANGE, "gate operand out of range");
            if (two && q0 == q1) fail(QSR_INVALID_ARGUMENT, "two-qubit gate with equal operands");
            const uint32_t w0 = wire[q0], w1 = wire[q1];
            const uint32_t r0 = w0 >> 1, r1 = w1 >> 1;
            const uint32_t meas = kind == QSR_MEASURE;
            const uint32_t r = meas ? (r0 > 1 ? r0 : 1) : 1 + (r0 > r1 ? r0 : r1);
            if (meas & w0 & 1u) fail(QSR_INVALID_ARGUMENT, "measure_window: qubit measured twice");
            wire[q0] = (r << 1) | meas;
            wire[q1] = (r << 1) | meas;
            const uint64_t key = 2 * uint64_t(r) + meas;
            if (key != cur_key) {
                cur_key = key;
                max_key_ = std::max(max_key_, key);
                cur = &buckets_[key];
                if (cur->capacity() == 0) fresh_(*cur);
            }
            cur->push_back(pack_gate(g));
        }
    }
    // Every window with key < 2 * min_round() + 1 is final (stream.cpp header).
    uint32_t min_round() const {
        uint32_t rmin = 0xFFFFFFFFu;
        for (uint32_t w : wire_) rmin = std::min(rmin, w >> 1);
        return rmin;
    }
    uint64_t max_key() const { return max_key_; }

  private:
    uint32_t n_;
    std::vector<uint32_t> wire_;
    BucketDir &buckets_;
    FreshBucket fresh_;
    uint64_t max_key_ = 0;
};

} // namespace qsr
