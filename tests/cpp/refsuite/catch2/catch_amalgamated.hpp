// A minimal stand-in for the parts of Catch2 v3 the reference's unit suites use (TEST_CASE,
// TEMPLATE_TEST_CASE, REQUIRE, REQUIRE_THROWS_AS, INFO, FAIL): Catch2 is not installed here and
// there is no network. Test infrastructure only; our own code.
#pragma once

#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <typeinfo>
#include <utility>
#include <vector>

namespace catch_standin {

struct Case {
    std::string name;
    std::function<void()> fn;
};
inline std::vector<Case> &registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(std::string n, std::function<void()> f) { registry().push_back({std::move(n), std::move(f)}); }
};
template <typename T>
struct TypeTag {
    using type = T;
};
template <typename... Ts>
struct TemplateReg {
    template <typename F>
    TemplateReg(const std::string &n, F f) {
        (registry().push_back({n + " - " + typeid(Ts).name(), [f] { f(TypeTag<Ts>{}); }}), ...);
    }
};
inline long long &assertions() {
    static long long a = 0;
    return a;
}
inline std::vector<std::string> &info() {
    static std::vector<std::string> s;
    return s;
}
struct InfoScope {
    explicit InfoScope(std::string s) { info().push_back(std::move(s)); }
    ~InfoScope() { info().pop_back(); }
};
struct Failure : std::exception {
    std::string msg;
    explicit Failure(std::string m) : msg(std::move(m)) {}
    const char *what() const noexcept override { return msg.c_str(); }
};
[[noreturn]] inline void fail(const std::string &what, const char *file, int line) {
    std::ostringstream os;
    os << file << ":" << line << ": " << what;
    for (const auto &i : info()) os << "\n    with: " << i;
    throw Failure(os.str());
}

} // namespace catch_standin

#define CATCH_STANDIN_CAT2(a, b) a##b
#define CATCH_STANDIN_CAT(a, b) CATCH_STANDIN_CAT2(a, b)
#define CATCH_STANDIN_ID(p) CATCH_STANDIN_CAT(p, __LINE__)

#define TEST_CASE(tc_name, ...)                                                                    \
    static void CATCH_STANDIN_ID(catch_standin_case_)();                                           \
    static ::catch_standin::Reg CATCH_STANDIN_ID(catch_standin_reg_)(tc_name,                      \
                                                                   &CATCH_STANDIN_ID(catch_standin_case_)); \
    static void CATCH_STANDIN_ID(catch_standin_case_)()

#define TEMPLATE_TEST_CASE(tc_name, tags, ...)                                                      \
    template <typename TestType>                                                                   \
    static void CATCH_STANDIN_ID(catch_standin_tcase_)();                                          \
    static ::catch_standin::TemplateReg<__VA_ARGS__> CATCH_STANDIN_ID(catch_standin_treg_)(          \
        tc_name, [](auto tag) { CATCH_STANDIN_ID(catch_standin_tcase_)<typename decltype(tag)::type>(); }); \
    template <typename TestType>                                                                   \
    static void CATCH_STANDIN_ID(catch_standin_tcase_)()

#define REQUIRE(...)                                                                               \
    do {                                                                                           \
        ++::catch_standin::assertions();                                                           \
        if (!(__VA_ARGS__)) ::catch_standin::fail("REQUIRE(" #__VA_ARGS__ ")", __FILE__, __LINE__); \
    } while (0)

#define REQUIRE_THROWS_AS(expr, exc_type)                                                          \
    do {                                                                                           \
        ++::catch_standin::assertions();                                                           \
        bool catch_standin_caught = false;                                                         \
        try {                                                                                      \
            (void)(expr);                                                                          \
        } catch (const exc_type &) {                                                               \
            catch_standin_caught = true;                                                           \
        } catch (...) {                                                                            \
        }                                                                                          \
        if (!catch_standin_caught)                                                                 \
            ::catch_standin::fail("REQUIRE_THROWS_AS(" #expr ", " #exc_type ")", __FILE__, __LINE__); \
    } while (0)

#define INFO(msg)                                                                                  \
    ::catch_standin::InfoScope CATCH_STANDIN_ID(catch_standin_info_)(                              \
        (std::ostringstream() << msg).str())

#define FAIL(msg) ::catch_standin::fail((std::ostringstream() << msg).str(), __FILE__, __LINE__)
