// Host-only timing of the streaming driver's two serial stages on a generated circuit: the chunk
// planner (stream_plan.hpp) and the gate fuser (fuse.hpp) over the same windows in key order.
//   g++ -O3 -std=c++17 -I include -I paper_2603_14641_b200/csrc tools/plan_bench.cpp \
//       paper_2603_14641_b200/csrc/host_circuit.cpp paper_2603_14641_b200/csrc/fuse.cpp -pthread -o /tmp/plan_bench
//   /tmp/plan_bench [n] [depth] [p] [reps]
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "fuse.hpp"
#include "stream_plan.hpp"

using namespace qsr;

int main(int argc, char **argv) {
    const uint32_t n = argc > 1 ? uint32_t(atoi(argv[1])) : 20000;
    const uint32_t depth = argc > 2 ? uint32_t(atoi(argv[2])) : 1000;
    const double p = argc > 3 ? atof(argv[3]) : 0.01;
    const int reps = argc > 4 ? atoi(argv[4]) : 3;
    Circuit c = generate_random(n, depth, 42, p);
    const uint64_t G = c.gates.size();
    using clk = std::chrono::steady_clock;
    for (int rep = 0; rep < reps; ++rep) {
        BucketDir buckets(2 * G + 4);
        auto fresh = [&](std::vector<uint64_t> &b) { b.reserve(size_t(n) * 3 / 4 + 16); };
        ChunkPlanner<decltype(fresh)> planner(n, buckets, fresh);
        auto t0 = clk::now();
        planner.plan(c.gates.data(), 0, G);
        const double plan_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
        Fuser fuser(n);
        WordVec dev;
        uint64_t out = 0;
        t0 = clk::now();
        for (uint64_t key = 2; key <= planner.max_key(); ++key) {
            std::vector<uint64_t> *b = buckets.find(key);
            if (!b || b->empty()) continue;
            dev.clear();
            if ((key & 1) == 0) fuser.unitary(b->data(), b->size(), dev);
            else fuser.flush(dev);
            out += dev.size();
        }
        const double fuse_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
        printf("n=%u depth=%u gates=%llu: plan %.1f ms (%.2f ns/gate), fuse %.1f ms (%.2f ns/gate), device gates %llu\n",
               n, depth, (unsigned long long)G, plan_ms, plan_ms * 1e6 / double(G), fuse_ms,
               fuse_ms * 1e6 / double(G), (unsigned long long)out);
    }
}
