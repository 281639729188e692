// Error plumbing of the C ABI (shared by capi.cpp and shard.cpp): library errors are thrown as
// qsr::Error inside and converted to a qsr_status + thread-local message at the boundary.
#pragma once

#include <new>
#include <string>

#include "host.hpp"

namespace qsr {

extern thread_local std::string g_err;
extern thread_local int g_qasm_line, g_qasm_column; // position of the last QSR_PARSE_ERROR

template <typename F>
qsr_status guard(F &&f) {
    try {
        f();
        return QSR_OK;
    } catch (const Error &e) {
        g_err = e.what();
        return e.status;
    } catch (const QasmFailure &e) {
        g_err = e.what();
        g_qasm_line = e.line;
        g_qasm_column = e.column;
        return QSR_PARSE_ERROR;
    } catch (const std::bad_alloc &) {
        g_err = "host allocation failed";
        return QSR_OUT_OF_MEMORY;
    } catch (const std::exception &e) {
        g_err = e.what();
        return QSR_INTERNAL;
    }
}

#define REQUIRE_PTR(p)                                                                      \
    do {                                                                                    \
        if (!(p)) fail(QSR_INVALID_ARGUMENT, #p " must not be NULL");                       \
    } while (0)

} // namespace qsr

// Opaque C handles of include/qsr.h.
struct qsr_circuit : qsr::Circuit {};
struct qsr_schedule : qsr::Schedule {};
