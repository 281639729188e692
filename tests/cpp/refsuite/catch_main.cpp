// Runner of the Catch2 stand-in: every registered case (optionally those whose name contains
// argv[1]); prints failures and the totals; exit 1 on any failure.
#include <chrono>
#include <cstring>

#include "catch2/catch_amalgamated.hpp"

#include <cstdint>

// Present when the suites are linked against libqsr (route_gpu.hpp): device kernel launches.
extern "C" uint64_t qsr_launch_count(void) __attribute__((weak));

int main(int argc, char **argv) {
    const char *filter = argc > 1 ? argv[1] : nullptr;
    int passed = 0, failed = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (const auto &c : catch_standin::registry()) {
        if (filter && !std::strstr(c.name.c_str(), filter)) continue;
        try {
            c.fn();
            ++passed;
        } catch (const std::exception &e) {
            ++failed;
            std::cout << "FAILED: " << c.name << "\n  " << e.what() << "\n";
        }
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::cout << "cases: " << passed + failed << " passed: " << passed << " failed: " << failed
              << " assertions: " << catch_standin::assertions() << " seconds: " << s;
    if (qsr_launch_count) std::cout << " libqsr_kernel_launches: " << qsr_launch_count();
    std::cout << "\n";
    return failed ? 1 : 0;
}
