// C ABI of libqsr (include/qsr.h): object lifetimes, host-side validation, layout conversion
// between the reference's host storage and the device layouts, and the single-shot /
// sampling drivers (reference simulator.hpp:46-76, frames.hpp:163-204).
#include <chrono>
#include <mutex>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <unordered_map>

#include "abi.hpp"
#include "engine.hpp"

using namespace qsr;


namespace qsr {

uint64_t g_launches = 0;
thread_local std::string g_err;
thread_local int g_qasm_line = 0, g_qasm_column = 0;

void cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return;
    cudaGetLastError();
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation) fail(QSR_OUT_OF_MEMORY, m);
    fail(QSR_CUDA_ERROR, m);
}

// Caching allocator for the four tableau planes (GBs each): released planes are kept per
// (device, bytes) and handed to the next tableau of the same shape, so repeated calls do not pay
// cudaMalloc / cudaFree of tens of GB. On an allocation failure the cache is flushed and the
// allocation retried; QSR_PLANE_CACHE=0 disables it; qsr_release_cached_memory() empties it.
namespace {
struct PlaneCache {
    std::mutex mu;
    // ready: recorded on the releasing owner's stream when a block is released mid-life, so the
    // next owner never races the kernels still queued on it; null = already idle.
    struct Entry { int device; uint64_t bytes; void *p; cudaEvent_t ready; };
    static void wait_ready(cudaEvent_t ev) {
        if (!ev) return;
        cudaEventSynchronize(ev);
        cudaEventDestroy(ev);
    }
    std::vector<Entry> free_list;
    static bool enabled() {
        static const bool on = [] {
            const char *e = getenv("QSR_PLANE_CACHE");
            return !(e && e[0] == '0');
        }();
        return on;
    }
    void *acquire(int device, uint64_t bytes) {
        {
            std::lock_guard<std::mutex> g(mu);
            for (size_t i = 0; i < free_list.size(); ++i)
                if (free_list[i].device == device && free_list[i].bytes == bytes) {
                    void *p = free_list[i].p;
                    const cudaEvent_t ev = free_list[i].ready;
                    free_list.erase(free_list.begin() + long(i));
                    wait_ready(ev);
                    return p;
                }
        }
        void *p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            flush(device);
            e = cudaMalloc(&p, bytes);
        }
        QSR_CUDA(e);
        return p;
    }
    void release(int device, uint64_t bytes, void *p, cudaStream_t after = nullptr) {
        if (!p) return;
        cudaEvent_t ev = nullptr;
        if (after) {
            QSR_CUDA(cudaSetDevice(device));
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            QSR_CUDA(cudaStreamIsCapturing(after, &cs));
            if (cs != cudaStreamCaptureStatusNone) // graphs are captured once every buffer is sized
                fail(QSR_INTERNAL, "scratch block released during stream capture");
            QSR_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            QSR_CUDA(cudaEventRecord(ev, after));
        }
        if (!enabled()) { wait_ready(ev); cudaFree(p); return; }
        std::lock_guard<std::mutex> g(mu);
        free_list.push_back({device, bytes, p, ev});
    }
    void flush(int device) {
        std::lock_guard<std::mutex> g(mu);
        for (auto it = free_list.begin(); it != free_list.end();) {
            if (device < 0 || it->device == device) {
                cudaSetDevice(it->device);
                wait_ready(it->ready);
                cudaFree(it->p);
                it = free_list.erase(it);
            } else {
                ++it;
            }
        }
    }
};
PlaneCache &plane_cache() {
    static PlaneCache *c = new PlaneCache(); // leaked on purpose: outlives static destructors
    return *c;
}

// Pinned 32-byte read-back slots (batch control words), recycled across tableaux.
std::mutex g_pinned_mu;
std::vector<uint32_t *> g_pinned_free;
uint32_t *pinned_slot() {
    {
        std::lock_guard<std::mutex> g(g_pinned_mu);
        if (!g_pinned_free.empty()) {
            uint32_t *p = g_pinned_free.back();
            g_pinned_free.pop_back();
            return p;
        }
    }
    uint32_t *p = nullptr;
    QSR_CUDA(cudaMallocHost(&p, 2 * 8 * 4));
    std::memset(p, 0, 2 * 8 * 4);
    return p;
}
void pinned_slot_release(uint32_t *p) {
    if (!p) return;
    std::lock_guard<std::mutex> g(g_pinned_mu);
    g_pinned_free.push_back(p);
}

// Two page-locked staging buffers for downloads into pageable memory (download_2d), shared by
// the process and allocated on first use.
constexpr size_t kStageBytes = size_t(16) << 20;
std::mutex g_stage_mu;
uint8_t *g_stage[2] = {nullptr, nullptr};
} // namespace

// Device -> host copy of `rows` rows of `width` bytes. Page-locked destinations take one DMA
// copy. Pageable ones go through the two pinned staging buffers in chunks of whole rows: chunk
// i + 1 is in flight while chunk i is copied out on the host. (A direct copy into pageable
// memory is staged by the driver at a fraction of PCIe bandwidth and has stalled for seconds
// on freshly allocated arrays.)
void download_2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t rows,
                 cudaStream_t st) {
    if (!rows || !width) return;
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, dst) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError(); // (a pageable pointer may leave an error on older runtimes)
    if (pinned || width > kStageBytes) {
        QSR_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToHost, st));
        QSR_CUDA(cudaStreamSynchronize(st));
        return;
    }
    std::lock_guard<std::mutex> g(g_stage_mu);
    for (auto &b : g_stage)
        if (!b) QSR_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&b), kStageBytes, cudaHostAllocPortable));
    const size_t per = std::max<size_t>(1, kStageBytes / width);
    const size_t nchunks = (rows + per - 1) / per;
    cudaEvent_t ev[2];
    for (auto &e : ev) QSR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    auto enqueue = [&](size_t c) {
        const size_t r0 = c * per, nr = std::min(per, rows - r0);
        QSR_CUDA(cudaMemcpy2DAsync(g_stage[c & 1], width, static_cast<const uint8_t *>(src) + r0 * spitch, spitch,
                                   width, nr, cudaMemcpyDeviceToHost, st));
        QSR_CUDA(cudaEventRecord(ev[c & 1], st));
    };
    enqueue(0);
    for (size_t c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) enqueue(c + 1); // its buffer was copied out in iteration c - 1
        QSR_CUDA(cudaEventSynchronize(ev[c & 1]));
        const size_t r0 = c * per, nr = std::min(per, rows - r0);
        uint8_t *d = static_cast<uint8_t *>(dst) + r0 * dpitch;
        if (dpitch == width) {
            std::memcpy(d, g_stage[c & 1], nr * width);
        } else {
            for (size_t r = 0; r < nr; ++r) std::memcpy(d + r * dpitch, g_stage[c & 1] + r * width, width);
        }
    }
    for (auto e : ev) cudaEventDestroy(e);
}

void *cache_acquire(int device, uint64_t bytes) { return plane_cache().acquire(device, bytes); }
void cache_release(int device, uint64_t bytes, void *p, cudaStream_t after) {
    plane_cache().release(device, bytes, p, after);
}

DeviceTableau::DeviceTableau(uint64_t n_, int dev, uint64_t j0, uint64_t kg_) : device(dev), n(n_) {
    if (n == 0) fail(QSR_INVALID_ARGUMENT, "Tableau: n must be >= 1");
    if (n > kMaxQubits) fail(QSR_INVALID_ARGUMENT, "Tableau: n exceeds the supported maximum");
    QSR_CUDA(cudaSetDevice(device));
    k = (n + 63) / 64;
    n_pad = 64 * k;
    kg = kg_ ? kg_ : k;
    if (j0 + kg > k) fail(QSR_INVALID_ARGUMENT, "Tableau: generator shard out of range");
    g0 = 64 * j0;
    ng = 64 * kg;
    n_gen = std::min<uint64_t>(ng, n > g0 ? n - g0 : 0);
    cm_pitch = round_up(2 * kg, 16);
    rm_pitch = round_up(k, 16);
    plane_words = std::max(n_pad * cm_pitch, 2 * ng * rm_pitch);
    QSR_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device));
    QSR_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    for (uint64_t **pp : {&x, &z, &x2, &z2}) {
        *pp = static_cast<uint64_t *>(plane_cache().acquire(device, plane_words * 8));
        QSR_CUDA(cudaMemsetAsync(*pp, 0, plane_words * 8, stream));
    }
    // The fixed-size scratch lives in ONE arena from the plane cache (one acquire / release per
    // tableau instead of ~20 cudaMalloc / cudaFree), zeroed once.
    const uint64_t vwords = uint64_t(kMaxBatch) * 2 * rm_pitch;
    const uint64_t info_words = (kVinfoWords + 4 + 1) / 2;
    ms.batch_block_bytes = (vwords + info_words) * 8;
    struct Piece { void **p; uint64_t bytes; };
    const Piece pieces[] = {
        {reinterpret_cast<void **>(&s), cm_pitch * 8},
        {reinterpret_cast<void **>(&tile_counters), (cm_pitch / 64 + 2) * 4},
        {reinterpret_cast<void **>(&ms.mask), (2 * kg + 2) * 8},
        {reinterpret_cast<void **>(&ms.rows), 2 * ng * 4},
        {reinterpret_cast<void **>(&ms.ctl), 64},
        {reinterpret_cast<void **>(&ms.partial_x), 128 * rm_pitch * 8},
        {reinterpret_cast<void **>(&ms.partial_z), 128 * rm_pitch * 8},
        {reinterpret_cast<void **>(&ms.partial_e), 128 * 8},
        {reinterpret_cast<void **>(&ms.coin_index), 8},
        {reinterpret_cast<void **>(&ms.err), 4},
        {reinterpret_cast<void **>(&ms.colbits), 2 * ng * 4},
        {reinterpret_cast<void **>(&ms.batch_block), ms.batch_block_bytes},
        {reinterpret_cast<void **>(&ms.nz), (ng / 32 + 1) * 4},
        {reinterpret_cast<void **>(&ms.pcount), 2 * kMaxBatch * sizeof(int)},
        {reinterpret_cast<void **>(&ms.vinfo_b), (kVinfoWords + 8) * 4},
        {reinterpret_cast<void **>(&ms.colbits_b), 2 * ng * 4},
        {reinterpret_cast<void **>(&ms.nz_b), (ng / 32 + 1) * 4},
        {reinterpret_cast<void **>(&ms.pcount_b), 2 * kMaxBatch * sizeof(int)},
        {reinterpret_cast<void **>(&ms.d_pos), 4},
    };
    arena_bytes = 0;
    for (const Piece &pc : pieces) arena_bytes += round_up(pc.bytes, 256);
    arena = static_cast<uint8_t *>(plane_cache().acquire(device, arena_bytes));
    QSR_CUDA(cudaMemsetAsync(arena, 0, arena_bytes, stream));
    uint64_t off = 0;
    for (const Piece &pc : pieces) {
        *pc.p = arena + off;
        off += round_up(pc.bytes, 256);
    }
    ms.Vx = ms.batch_block;
    ms.Vz = ms.batch_block + rm_pitch;
    ms.vstride = 2 * rm_pitch;
    ms.vinfo = reinterpret_cast<uint32_t *>(ms.batch_block + vwords);
    ms.bctl = ms.vinfo + kVinfoWords;
    ms.bctl_b = ms.vinfo_b + kVinfoWords;
    ms.h_bctl = pinned_slot();
    for (auto &e : ms.bev) QSR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    configure_measure_kernels(*this);
    QSR_CUDA(cudaStreamSynchronize(stream));
}

DeviceTableau::~DeviceTableau() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    pinned_slot_release(ms.h_bctl);
    for (auto e : ms.bev)
        if (e) cudaEventDestroy(e);
    for (uint64_t *p : {x, z, x2, z2}) plane_cache().release(device, plane_words * 8, p);
    if (gate_buf) plane_cache().release(device, gate_buf_cap * 8, gate_buf);
    gate_buf = nullptr;
    plane_cache().release(device, arena_bytes, arena);
    // Lazily sized scratch returns to the cache too (the next tableau of this shape reuses it).
    plane_cache().release(device, sign_partial_chunks * cm_pitch * 8, sign_partials);
    plane_cache().release(device, ms.partial_bytes, ms.partial);
    release_window_cap();
    if (stream) cudaStreamDestroy(stream);
}

void DeviceTableau::ensure_gate_buf(uint64_t ng) {
    if (ng <= gate_buf_cap) return;
    if (gate_buf) plane_cache().release(device, gate_buf_cap * 8, gate_buf, stream);
    gate_buf_cap = std::max<uint64_t>(ng, 1024);
    gate_buf = static_cast<uint64_t *>(plane_cache().acquire(device, gate_buf_cap * 8));
}

// Per-window measurement scratch: six arrays of window_cap entries in one cached block.
static uint64_t window_block_bytes(uint64_t cap) { return cap * (1 + 1 + sizeof(qsr_record_entry) + 4 + 4 + 4) + 256; }

void DeviceTableau::release_window_cap() {
    if (ms.window_cap) plane_cache().release(device, window_block_bytes(ms.window_cap), ms.coin_buf, stream);
    ms.coin_buf = ms.flags = nullptr;
    ms.out = nullptr;
    ms.mqubits = ms.fq = ms.fidx = nullptr;
    ms.window_cap = 0;
}

void DeviceTableau::ensure_window_cap(uint64_t m) {
    if (m <= ms.window_cap) return;
    release_window_cap();
    const uint64_t cap = std::max<uint64_t>(m, 64);
    uint8_t *b = static_cast<uint8_t *>(plane_cache().acquire(device, window_block_bytes(cap)));
    ms.window_cap = cap;
    // coin_buf first (the block's base pointer), 4-byte arrays 16-byte aligned.
    ms.coin_buf = b;
    ms.flags = b + cap;
    uint64_t off = round_up(2 * cap, 16);
    ms.out = reinterpret_cast<qsr_record_entry *>(b + off);
    off += round_up(cap * sizeof(qsr_record_entry), 16);
    ms.mqubits = reinterpret_cast<uint32_t *>(b + off);
    off += round_up(cap * 4, 16);
    ms.fq = reinterpret_cast<uint32_t *>(b + off);
    off += round_up(cap * 4, 16);
    ms.fidx = reinterpret_cast<uint32_t *>(b + off);
}

void DeviceTableau::sync() { QSR_CUDA(cudaStreamSynchronize(stream)); }

} // namespace qsr

struct qsr_tableau {
    std::unique_ptr<DeviceTableau> t;
};

namespace {

void check_cm(const DeviceTableau &t, const char *who) {
    if (t.layout != QSR_COLUMN_MAJOR)
        fail(QSR_INVALID_ARGUMENT, std::string(who) + ": tableau must be ColumnMajor");
}
void check_rm(const DeviceTableau &t, const char *who) {
    if (t.layout != QSR_ROW_MAJOR)
        fail(QSR_INVALID_ARGUMENT, std::string(who) + ": tableau must be RowMajor");
}

std::vector<uint64_t> pack(const qsr_gate *g, uint64_t n) {
    std::vector<uint64_t> v(n);
    for (uint64_t i = 0; i < n; ++i) v[i] = pack_gate(g[i]);
    return v;
}

// One RM word of the X plane (row r, qubit-word i).
uint64_t rm_word_x(DeviceTableau &t, uint64_t r, uint64_t i) {
    uint64_t v = 0;
    QSR_CUDA(cudaMemcpyAsync(&v, t.x + r * t.rm_pitch + i, 8, cudaMemcpyDeviceToHost, t.stream));
    t.sync();
    return v;
}

} // namespace

// ================================ C ABI ===============================================

extern "C" {

const char *qsr_last_error(void) { return g_err.c_str(); }
void qsr_release_cached_memory(void) { plane_cache().flush(-1); }
int qsr_abi_version(void) { return QSR_ABI_VERSION; }
uint64_t qsr_launch_count(void) { return g_launches; }

qsr_status qsr_host_alloc(uint64_t bytes, void **out) {
    return guard([&] {
        REQUIRE_PTR(out);
        QSR_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
    });
}
void qsr_host_free(void *p) {
    if (p) cudaFreeHost(p);
}

qsr_status qsr_device_count(int *count) {
    return guard([&] {
        REQUIRE_PTR(count);
        QSR_CUDA(cudaGetDeviceCount(count));
    });
}

void qsr_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    philox_block(ctr, key, out);
}
uint64_t qsr_philox_word(uint64_t seed, uint32_t stream, uint32_t ctx, uint64_t index) {
    return philox_word(seed, stream, ctx, index);
}

// ---- circuits ---------------------------------------------------------------------
qsr_status qsr_circuit_create(uint32_t num_qubits, const qsr_gate *gates, uint64_t ngates,
                              qsr_circuit **out) {
    return guard([&] {
        REQUIRE_PTR(out);
        if (ngates) REQUIRE_PTR(gates);
        auto c = std::make_unique<qsr_circuit>();
        c->num_qubits = num_qubits;
        c->gates.resize(ngates);
        const unsigned T = std::max(1u, std::min<unsigned>(host_threads(), unsigned(ngates >> 22) + 1));
        parallel_chunks(ngates, T, [&](unsigned, uint64_t b, uint64_t e) {
            if (e > b) std::memcpy(c->gates.data() + b, gates + b, (e - b) * sizeof(qsr_gate));
        });
        c->check_valid();
        *out = c.release();
    });
}

qsr_status qsr_generate_random(uint32_t n, uint32_t depth, uint64_t seed, double p,
                               qsr_circuit **out) {
    return guard([&] {
        REQUIRE_PTR(out);
        auto c = std::make_unique<qsr_circuit>();
        static_cast<Circuit &>(*c) = generate_random(n, depth, seed, p);
        *out = c.release();
    });
}

qsr_status qsr_circuit_info(const qsr_circuit *c, uint32_t *nq, uint64_t *ng, uint64_t *nm) {
    return guard([&] {
        REQUIRE_PTR(c);
        if (nq) *nq = c->num_qubits;
        if (ng) *ng = c->gates.size();
        if (nm) *nm = c->measure_count();
    });
}
const qsr_gate *qsr_circuit_gates(const qsr_circuit *c) { return c ? c->gates.data() : nullptr; }
void qsr_circuit_destroy(qsr_circuit *c) { delete c; }

qsr_status qsr_circuit_clbits(const qsr_circuit *c, uint32_t *num_clbits) {
    return guard([&] {
        REQUIRE_PTR(c); REQUIRE_PTR(num_clbits);
        *num_clbits = c->num_clbits;
    });
}
qsr_status qsr_circuit_set_clbits(qsr_circuit *c, uint32_t num_clbits) {
    return guard([&] {
        REQUIRE_PTR(c);
        c->num_clbits = num_clbits;
    });
}

void qsr_set_num_threads(unsigned threads) { set_host_threads(threads); }
unsigned qsr_get_num_threads(void) { return host_threads(); }

// ---- OpenQASM / schedule text -----------------------------------------------------
extern "C++" {
namespace {
// Size query (buf == NULL) or fill; *len = bytes (no terminator is written).
template <typename F>
void text_out(F &&emit, char *buf, uint64_t cap, uint64_t *len) {
    REQUIRE_PTR(len);
    const uint64_t need = emit(nullptr);
    *len = need;
    if (!buf) return;
    if (cap < need) fail(QSR_INVALID_ARGUMENT, "output buffer too small (" + std::to_string(need) + " bytes needed)");
    emit(buf);
}
} // namespace
}

qsr_status qsr_parse_qasm(const char *text, uint64_t len, qsr_circuit **out, qsr_qasm_error *err) {
    const qsr_status st = guard([&] {
        REQUIRE_PTR(out);
        if (len) REQUIRE_PTR(text);
        auto c = std::make_unique<qsr_circuit>();
        static_cast<Circuit &>(*c) = parse_qasm(text ? text : "", len);
        *out = c.release();
    });
    if (err) *err = st == QSR_PARSE_ERROR ? qsr_qasm_error{g_qasm_line, g_qasm_column} : qsr_qasm_error{0, 0};
    return st;
}

qsr_status qsr_emit_qasm(const qsr_circuit *c, char *buf, uint64_t cap, uint64_t *len) {
    return guard([&] {
        REQUIRE_PTR(c);
        text_out([&](char *o) { return emit_qasm(*c, o); }, buf, cap, len);
    });
}

qsr_status qsr_schedule_text(const qsr_schedule *s, char *buf, uint64_t cap, uint64_t *len) {
    return guard([&] {
        REQUIRE_PTR(s);
        text_out([&](char *o) { return schedule_text(*s, o); }, buf, cap, len);
    });
}

qsr_status qsr_validate_schedule(const qsr_circuit *c, const qsr_schedule *s, char *buf, uint64_t cap,
                                 uint64_t *len) {
    return guard([&] {
        REQUIRE_PTR(c); REQUIRE_PTR(s);
        const std::string v = validate_schedule(*c, *s);
        text_out([&](char *o) {
            if (o) std::memcpy(o, v.data(), v.size());
            return uint64_t(v.size());
        }, buf, cap, len);
    });
}

// ---- schedules --------------------------------------------------------------------
qsr_status qsr_schedule_windows(const qsr_circuit *c, int mode, qsr_schedule **out) {
    return guard([&] {
        REQUIRE_PTR(c);
        REQUIRE_PTR(out);
        auto s = std::make_unique<qsr_schedule>();
        static_cast<Schedule &>(*s) = schedule_windows(*c, mode);
        *out = s.release();
    });
}

qsr_status qsr_schedule_create(const qsr_gate *gates, const uint64_t *offsets,
                               const uint8_t *is_meas, uint64_t nwin, int mode,
                               qsr_schedule **out) {
    return guard([&] {
        REQUIRE_PTR(out);
        REQUIRE_PTR(offsets);
        if (nwin) REQUIRE_PTR(is_meas);
        auto s = std::make_unique<qsr_schedule>();
        s->mode = mode;
        s->offsets.assign(offsets, offsets + nwin + 1);
        if (s->offsets[0] != 0) fail(QSR_INVALID_ARGUMENT, "schedule offsets must start at 0");
        for (uint64_t w = 0; w < nwin; ++w)
            if (s->offsets[w + 1] < s->offsets[w])
                fail(QSR_INVALID_ARGUMENT, "schedule offsets must be non-decreasing");
        s->is_meas.assign(is_meas, is_meas + nwin);
        uint64_t G = s->offsets[nwin];
        if (G) REQUIRE_PTR(gates);
        s->gates.assign(gates, gates + G);
        *out = s.release();
    });
}

qsr_status qsr_schedule_info(const qsr_schedule *s, uint64_t *nwin, uint64_t *ng, int *mode) {
    return guard([&] {
        REQUIRE_PTR(s);
        if (nwin) *nwin = s->num_windows();
        if (ng) *ng = s->gates.size();
        if (mode) *mode = s->mode;
    });
}
const qsr_gate *qsr_schedule_gates(const qsr_schedule *s) { return s ? s->gates.data() : nullptr; }
const uint64_t *qsr_schedule_offsets(const qsr_schedule *s) { return s ? s->offsets.data() : nullptr; }
const uint8_t *qsr_schedule_is_measurement(const qsr_schedule *s) {
    return s ? s->is_meas.data() : nullptr;
}
void qsr_schedule_destroy(qsr_schedule *s) { delete s; }

// ---- tableau ----------------------------------------------------------------------
qsr_status qsr_tableau_create(uint64_t n, int device, qsr_tableau **out) {
    return guard([&] {
        REQUIRE_PTR(out);
        auto h = std::make_unique<qsr_tableau>();
        h->t = std::make_unique<DeviceTableau>(n, device);
        *out = h.release();
    });
}

qsr_status qsr_tableau_basis_state(qsr_tableau *h, const uint8_t *init) {
    return guard([&] {
        REQUIRE_PTR(h);
        DeviceTableau &t = *h->t;
        QSR_CUDA(cudaSetDevice(t.device));
        if (t.layout != QSR_COLUMN_MAJOR) { std::swap(t.x, t.x2); std::swap(t.z, t.z2); }
        uint8_t *d_init = nullptr;
        if (init) {
            QSR_CUDA(cudaMalloc(&d_init, t.n));
            QSR_CUDA(cudaMemcpyAsync(d_init, init, t.n, cudaMemcpyHostToDevice, t.stream));
        }
        launch_zero_state(t, d_init);
        t.trusted = true;
        t.sync();
        if (d_init) cudaFree(d_init);
    });
}

qsr_status qsr_tableau_info(const qsr_tableau *h, uint64_t *n, uint64_t *k, uint64_t *n_pad,
                            int *layout) {
    return guard([&] {
        REQUIRE_PTR(h);
        if (n) *n = h->t->n;
        if (k) *k = h->t->k;
        if (n_pad) *n_pad = h->t->n_pad;
        if (layout) *layout = h->t->layout;
    });
}

qsr_status qsr_tableau_upload(qsr_tableau *h, const uint64_t *x, const uint64_t *z,
                              const uint64_t *s, int layout) {
    return guard([&] {
        REQUIRE_PTR(h); REQUIRE_PTR(x); REQUIRE_PTR(z); REQUIRE_PTR(s);
        if (layout != QSR_COLUMN_MAJOR && layout != QSR_ROW_MAJOR)
            fail(QSR_INVALID_ARGUMENT, "unknown layout");
        DeviceTableau &t = *h->t;
        QSR_CUDA(cudaSetDevice(t.device));
        upload_planes(t, x, z, layout);
        t.trusted = false;
        QSR_CUDA(cudaMemcpyAsync(t.s, s, 2 * t.k * 8, cudaMemcpyHostToDevice, t.stream));
        t.sync();
    });
}

qsr_status qsr_tableau_download(const qsr_tableau *h, uint64_t *x, uint64_t *z, uint64_t *s) {
    return guard([&] {
        REQUIRE_PTR(h);
        DeviceTableau &t = *h->t;
        QSR_CUDA(cudaSetDevice(t.device));
        download_planes(t, x, z);
        if (s) {
            auto sv = download_signs(t);
            std::memcpy(s, sv.data(), sv.size() * 8);
        }
    });
}

qsr_status qsr_tableau_clone(const qsr_tableau *h, qsr_tableau **out) {
    return guard([&] {
        REQUIRE_PTR(h); REQUIRE_PTR(out);
        const DeviceTableau &t = *h->t;
        auto c = std::make_unique<qsr_tableau>();
        c->t = std::make_unique<DeviceTableau>(t.n, t.device);
        DeviceTableau &d = *c->t;
        QSR_CUDA(cudaMemcpyAsync(d.x, t.x, t.plane_words * 8, cudaMemcpyDeviceToDevice, d.stream));
        QSR_CUDA(cudaMemcpyAsync(d.z, t.z, t.plane_words * 8, cudaMemcpyDeviceToDevice, d.stream));
        QSR_CUDA(cudaMemcpyAsync(d.x2, t.x2, t.plane_words * 8, cudaMemcpyDeviceToDevice, d.stream));
        QSR_CUDA(cudaMemcpyAsync(d.z2, t.z2, t.plane_words * 8, cudaMemcpyDeviceToDevice, d.stream));
        QSR_CUDA(cudaMemcpyAsync(d.s, t.s, t.cm_pitch * 8, cudaMemcpyDeviceToDevice, d.stream));
        d.layout = t.layout;
        d.sync();
        *out = c.release();
    });
}

void qsr_tableau_destroy(qsr_tableau *h) {
    TraceScope tr("tableau destroy");
    delete h;
}

qsr_status qsr_tableau_check_validity(qsr_tableau *h, char *buf, uint64_t cap, uint64_t *len) {
    return guard([&] {
        REQUIRE_PTR(h);
        DeviceTableau &t = *h->t;
        QSR_CUDA(cudaSetDevice(t.device));
        const std::string v = check_group_validity(t);
        text_out([&](char *o) {
            if (o) std::memcpy(o, v.data(), v.size());
            return uint64_t(v.size());
        }, buf, cap, len);
    });
}

qsr_status qsr_transpose_in_place(qsr_tableau *h) {
    return guard([&] {
        REQUIRE_PTR(h);
        DeviceTableau &t = *h->t;
        QSR_CUDA(cudaSetDevice(t.device));
        if (t.layout == QSR_COLUMN_MAJOR) transpose_to_rm(t);
        else transpose_to_cm(t);
        t.sync();
    });
}

qsr_status qsr_apply_window(qsr_tableau *h, const qsr_gate *gates, uint64_t ng) {
    return guard([&] {
        REQUIRE_PTR(h);
        if (ng) REQUIRE_PTR(gates);
        DeviceTableau &t = *h->t;
        check_cm(t, "apply_window");
        std::vector<uint32_t> stamp;
        validate_window(t.n, gates, ng, false, stamp, 1);
        QSR_CUDA(cudaSetDevice(t.device));
        auto packed = pack(gates, ng);
        t.ensure_gate_buf(ng);
        QSR_CUDA(cudaMemcpyAsync(t.gate_buf, packed.data(), ng * 8, cudaMemcpyHostToDevice, t.stream));
        launch_gate_window(t, t.gate_buf, ng);
        t.sync();
    });
}

qsr_status qsr_find_probabilistic(qsr_tableau *h, const qsr_gate *gates, uint64_t ng, int64_t *out) {
    return guard([&] {
        REQUIRE_PTR(h);
        if (ng) { REQUIRE_PTR(gates); REQUIRE_PTR(out); }
        DeviceTableau &t = *h->t;
        check_rm(t, "find_probabilistic");
        std::vector<uint32_t> qs(ng);
        for (uint64_t i = 0; i < ng; ++i) {
            if (gates[i].q0 >= t.n) fail(QSR_OUT_OF_RANGE, "find_probabilistic: qubit out of range");
            qs[i] = gates[i].q0;
        }
        QSR_CUDA(cudaSetDevice(t.device));
        std::vector<int64_t> res;
        rm_find_probabilistic(t, qs, res);
        std::memcpy(out, res.data(), ng * 8);
    });
}

qsr_status qsr_find_and_compact_pivots(qsr_tableau *h, uint64_t q, int64_t *entries,
                                       uint64_t *count) {
    return guard([&] {
        REQUIRE_PTR(h); REQUIRE_PTR(entries); REQUIRE_PTR(count);
        DeviceTableau &t = *h->t;
        check_rm(t, "find_and_compact_pivots");
        if (q >= t.n) fail(QSR_OUT_OF_RANGE, "find_and_compact_pivots: qubit out of range");
        QSR_CUDA(cudaSetDevice(t.device));
        std::vector<int64_t> e;
        rm_find_pivots(t, q, e, *count);
        std::memcpy(entries, e.data(), t.n * 8);
    });
}

qsr_status qsr_parallel_ge(qsr_tableau *h, const int64_t *entries, uint64_t count,
                           uint64_t block_targets) {
    return guard([&] {
        REQUIRE_PTR(h);
        DeviceTableau &t = *h->t;
        check_rm(t, "parallel_ge");
        if (count == 0) fail(QSR_INVALID_ARGUMENT, "parallel_ge: empty pivot list");
        if (block_targets < 1) fail(QSR_INVALID_ARGUMENT, "parallel_ge: block size must be >= 1");
        REQUIRE_PTR(entries);
        std::vector<int64_t> piv(entries, entries + count);
        for (int64_t p : piv)
            if (p < 0 || uint64_t(p) >= t.n) fail(QSR_OUT_OF_RANGE, "parallel_ge: pivot out of range");
        QSR_CUDA(cudaSetDevice(t.device));
        // The result is independent of block_targets by construction (the reference's
        // three-pass scan reproduces the ordered sequential product for any block size).
        rm_parallel_ge(t, piv);
        t.sync();
    });
}

qsr_status qsr_swap_anti_commuting(qsr_tableau *h, uint64_t p, uint64_t q) {
    return guard([&] {
        REQUIRE_PTR(h);
        DeviceTableau &t = *h->t;
        check_rm(t, "swap_anti_commuting");
        if (p >= t.n || q >= t.n) fail(QSR_OUT_OF_RANGE, "swap_anti_commuting: index out of range");
        QSR_CUDA(cudaSetDevice(t.device));
        uint64_t w = rm_word_x(t, t.ng + p, q / 64);
        if (!((w >> (q % 64)) & 1))
            fail(QSR_INVALID_ARGUMENT, "swap_anti_commuting: stabilizer p commutes with Z_q");
        rm_swap_anti_commuting(t, p, q);
        if (read_error_flag(t))
            fail(QSR_LOGIC_ERROR, "product of anti-commuting rows (corrupted tableau)");
    });
}

qsr_status qsr_inject_x(qsr_tableau *h, uint64_t p) {
    return guard([&] {
        REQUIRE_PTR(h);
        DeviceTableau &t = *h->t;
        if (p >= t.n) fail(QSR_OUT_OF_RANGE, "inject_x: index out of range");
        QSR_CUDA(cudaSetDevice(t.device));
        flip_sign_bit(t, t.kg + p / 64, p % 64);
        t.sync();
    });
}

qsr_status qsr_deterministic_outcome(qsr_tableau *h, uint64_t q, uint8_t *outcome) {
    return guard([&] {
        REQUIRE_PTR(h); REQUIRE_PTR(outcome);
        DeviceTableau &t = *h->t;
        check_rm(t, "deterministic_outcome");
        if (q >= t.n) fail(QSR_OUT_OF_RANGE, "deterministic_outcome: qubit out of range");
        QSR_CUDA(cudaSetDevice(t.device));
        *outcome = rm_deterministic_outcome(t, q) ? 1 : 0;
    });
}

qsr_status qsr_measure_window(qsr_tableau *h, const qsr_gate *gates, uint64_t ng, uint64_t seed,
                              uint64_t *coin_index, qsr_record_entry *out,
                              qsr_phase_timers *timers) {
    return guard([&] {
        REQUIRE_PTR(h); REQUIRE_PTR(coin_index);
        if (ng) { REQUIRE_PTR(gates); REQUIRE_PTR(out); }
        DeviceTableau &t = *h->t;
        check_cm(t, "measure_window");
        std::vector<uint32_t> stamp;
        validate_window(t.n, gates, ng, true, stamp, 1);
        QSR_CUDA(cudaSetDevice(t.device));
        std::vector<uint32_t> qs(ng);
        for (uint64_t i = 0; i < ng; ++i) qs[i] = gates[i].q0;
        t.ensure_window_cap(ng);
        QSR_CUDA(cudaMemcpyAsync(t.ms.coin_index, coin_index, 8, cudaMemcpyHostToDevice, t.stream));
        if (ng)
            QSR_CUDA(cudaMemcpyAsync(t.ms.mqubits, qs.data(), ng * 4, cudaMemcpyHostToDevice, t.stream));
        std::vector<uint8_t> flags;
        double t_ms = 0, ge_ms = 0, cmp_ms = 0;
        measure_window_device(t, ng, seed, qs, flags, timers != nullptr, &t_ms, &ge_ms, &cmp_ms);
        if (ng)
            QSR_CUDA(cudaMemcpyAsync(out, t.ms.out, ng * sizeof(qsr_record_entry),
                                     cudaMemcpyDeviceToHost, t.stream));
        QSR_CUDA(cudaMemcpyAsync(coin_index, t.ms.coin_index, 8, cudaMemcpyDeviceToHost, t.stream));
        t.sync();
        if (read_error_flag(t))
            fail(QSR_LOGIC_ERROR, "product of anti-commuting rows (corrupted tableau)");
        if (timers) {
            timers->t_seconds += t_ms * 1e-3;
            timers->ge_seconds += ge_ms * 1e-3;
            timers->cmp_seconds += cmp_ms * 1e-3;
        }
    });
}

qsr_status qsr_measure_window_coins(qsr_tableau *h, const qsr_gate *gates, uint64_t ng,
                                    const uint8_t *coins, uint64_t ncoins, uint64_t *used,
                                    qsr_record_entry *out, qsr_phase_timers *timers) {
    return guard([&] {
        REQUIRE_PTR(h); REQUIRE_PTR(used);
        if (ng) { REQUIRE_PTR(gates); REQUIRE_PTR(out); }
        DeviceTableau &t = *h->t;
        check_cm(t, "measure_window");
        std::vector<uint32_t> stamp;
        validate_window(t.n, gates, ng, true, stamp, 1);
        // At most one coin per measurement of the window is ever drawn.
        if (ncoins < ng) fail(QSR_INVALID_ARGUMENT, "measure_window: fewer coins than measurements");
        if (ng) REQUIRE_PTR(coins);
        QSR_CUDA(cudaSetDevice(t.device));
        std::vector<uint32_t> qs(ng);
        for (uint64_t i = 0; i < ng; ++i) qs[i] = gates[i].q0;
        t.ensure_window_cap(ng);
        const uint64_t zero = 0;
        QSR_CUDA(cudaMemcpyAsync(t.ms.coin_index, &zero, 8, cudaMemcpyHostToDevice, t.stream));
        if (ng) {
            QSR_CUDA(cudaMemcpyAsync(t.ms.mqubits, qs.data(), ng * 4, cudaMemcpyHostToDevice, t.stream));
            QSR_CUDA(cudaMemcpyAsync(t.ms.coin_buf, coins, ng, cudaMemcpyHostToDevice, t.stream));
        }
        t.ms.coin_table = t.ms.coin_buf;
        std::vector<uint8_t> flags;
        double t_ms = 0, ge_ms = 0, cmp_ms = 0;
        try {
            measure_window_device(t, ng, 0, qs, flags, timers != nullptr, &t_ms, &ge_ms, &cmp_ms);
        } catch (...) {
            t.ms.coin_table = nullptr;
            throw;
        }
        t.ms.coin_table = nullptr;
        if (ng)
            QSR_CUDA(cudaMemcpyAsync(out, t.ms.out, ng * sizeof(qsr_record_entry),
                                     cudaMemcpyDeviceToHost, t.stream));
        QSR_CUDA(cudaMemcpyAsync(used, t.ms.coin_index, 8, cudaMemcpyDeviceToHost, t.stream));
        t.sync();
        if (read_error_flag(t))
            fail(QSR_LOGIC_ERROR, "product of anti-commuting rows (corrupted tableau)");
        if (timers) {
            timers->t_seconds += t_ms * 1e-3;
            timers->ge_seconds += ge_ms * 1e-3;
            timers->cmp_seconds += cmp_ms * 1e-3;
        }
    });
}

qsr_status qsr_run_single_shot(const qsr_circuit *c, const qsr_schedule *s, uint64_t seed,
                               int device, qsr_tableau **out_tableau, qsr_record_entry *record,
                               qsr_run_report *report) {
    return guard([&] {
        TraceScope tr_all("run_single_shot");
        auto wall0 = std::chrono::steady_clock::now();
        REQUIRE_PTR(c);
        const uint64_t nm = c->measure_count();
        if (nm) REQUIRE_PTR(record);
        auto h = std::make_unique<qsr_tableau>();
        {
            TraceScope tr("tableau alloc");
            h->t = std::make_unique<DeviceTableau>(c->num_qubits, device);
        }
        DeviceTableau &t = *h->t;
        // Circuit only: the scheduler runs overlapped with the device (stream.cpp); a caller's
        // Schedule is validated window by window and uploaded first (QSR_STREAM=0 forces that
        // path for circuits too).
        const bool streaming = !s && !(getenv("QSR_STREAM") && getenv("QSR_STREAM")[0] == '0');
        std::unique_ptr<DeviceSchedule> ds;
        if (!streaming) {
            ds = s ? upload_schedule(t.n, *s, device, t.stream, true) : upload_circuit(*c, device, t.stream, true);
            if (ds->measure_count != nm)
                fail(QSR_INVALID_ARGUMENT, "schedule does not match the circuit's measurement count");
        }
        qsr_record_entry *d_rec = nullptr;
        QSR_CUDA(cudaMalloc(&d_rec, std::max<uint64_t>(nm, 1) * sizeof(qsr_record_entry)));
        RunTimes rt;
        try {
            TraceScope tr("run_device");
            if (streaming) {
                StreamCounts sc;
                run_circuit_streaming(t, *c, seed, d_rec, rt, sc);
                ds = std::make_unique<DeviceSchedule>();
                ds->device = device;
                ds->unitary_count = sc.unitary;
                ds->measure_count = sc.measures;
                ds->is_meas.resize(sc.windows);
            } else {
                run_device(t, *ds, seed, d_rec, rt);
            }
        } catch (...) {
            cudaFree(d_rec);
            throw;
        }
        std::vector<qsr_record_entry> host_rec(nm);
        if (nm)
            QSR_CUDA(cudaMemcpyAsync(host_rec.data(), d_rec, nm * sizeof(qsr_record_entry),
                                     cudaMemcpyDeviceToHost, t.stream));
        t.sync();
        cudaFree(d_rec);
        if (nm) std::memcpy(record, host_rec.data(), nm * sizeof(qsr_record_entry));
        double wall =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
        fill_report(report, rt, *ds, host_rec, wall);
        if (out_tableau) *out_tableau = h.release();
    });
}

// ---- resident engine --------------------------------------------------------------
// QSR_GRAPHS=0 keeps the resident engine on per-window launches.
static bool graphs_enabled() {
    static const bool on = [] {
        const char *e = getenv("QSR_GRAPHS");
        return !(e && e[0] == '0');
    }();
    return on;
}

struct qsr_engine {
    std::unique_ptr<DeviceTableau> t;
    std::unique_ptr<DeviceSchedule> ds;
    qsr_record_entry *d_rec = nullptr;
    RunTimes last;
    double frames_ms = 0; // frames-window device time of the last qsr_engine_sample
    uint64_t launches = 0;
    ~qsr_engine() {
        if (d_rec) cudaFree(d_rec);
    }
};

qsr_status qsr_engine_create(const qsr_circuit *c, const qsr_schedule *s, int device,
                             qsr_engine **out) {
    return guard([&] {
        REQUIRE_PTR(c); REQUIRE_PTR(out);
        auto e = std::make_unique<qsr_engine>();
        e->t = std::make_unique<DeviceTableau>(c->num_qubits, device);
        e->ds = s ? upload_schedule(e->t->n, *s, device, e->t->stream, true)
                  : upload_circuit(*c, device, e->t->stream, true);
        e->ds->use_graphs = graphs_enabled();
        QSR_CUDA(cudaMalloc(&e->d_rec,
                            std::max<uint64_t>(e->ds->measure_count, 1) * sizeof(qsr_record_entry)));
        *out = e.release();
    });
}

qsr_status qsr_engine_run(qsr_engine *e, uint64_t seed, double *device_ms) {
    return guard([&] {
        REQUIRE_PTR(e);
        QSR_CUDA(cudaSetDevice(e->t->device));
        uint64_t l0 = g_launches;
        e->last = RunTimes{};
        run_device(*e->t, *e->ds, seed, e->d_rec, e->last);
        e->launches = g_launches - l0;
        if (device_ms) *device_ms = e->last.total_ms;
    });
}

qsr_status qsr_engine_stats(const qsr_engine *e, double *gate_ms, uint64_t *gate_launches,
                            double *transpose_ms, double *measure_ms, uint64_t *launches) {
    return guard([&] {
        REQUIRE_PTR(e);
        if (gate_ms) *gate_ms = e->last.to_ms;
        if (gate_launches) *gate_launches = e->last.gate_launches;
        if (transpose_ms) *transpose_ms = e->last.t_ms;
        if (measure_ms) *measure_ms = e->last.ge_ms + e->last.cmp_ms;
        if (launches) *launches = e->launches;
    });
}

qsr_status qsr_engine_gate_bytes(const qsr_engine *e, double *bytes) {
    return guard([&] {
        REQUIRE_PTR(e);
        REQUIRE_PTR(bytes);
        *bytes = e->last.gate_bytes;
    });
}

qsr_status qsr_engine_record(const qsr_engine *e, qsr_record_entry *record) {
    return guard([&] {
        REQUIRE_PTR(e);
        uint64_t nm = e->ds->measure_count;
        if (nm) {
            REQUIRE_PTR(record);
            QSR_CUDA(cudaMemcpyAsync(record, e->d_rec, nm * sizeof(qsr_record_entry),
                                     cudaMemcpyDeviceToHost, e->t->stream));
        }
        e->t->sync();
    });
}

qsr_status qsr_engine_tableau(const qsr_engine *e, uint64_t *x, uint64_t *z, uint64_t *s) {
    return guard([&] {
        REQUIRE_PTR(e);
        DeviceTableau &t = *e->t;
        download_planes(t, x, z);
        if (s) {
            auto sv = download_signs(t);
            std::memcpy(s, sv.data(), sv.size() * 8);
        }
    });
}

qsr_status qsr_engine_profile(qsr_engine *e, uint64_t seed, qsr_kernel_profile *out) {
    return guard([&] {
        REQUIRE_PTR(e);
        REQUIRE_PTR(out);
        DeviceTableau &t = *e->t;
        QSR_CUDA(cudaSetDevice(t.device));
        DeviceTableau::AbsorbProfile prof;
        QSR_CUDA(cudaMalloc(&prof.d_rows, sizeof(unsigned long long)));
        QSR_CUDA(cudaMemsetAsync(prof.d_rows, 0, sizeof(unsigned long long), t.stream));
        t.prof = &prof;
        RunTimes rt;
        try {
            run_device(t, *e->ds, seed, e->d_rec, rt);
        } catch (...) {
            t.prof = nullptr;
            for (auto &p : prof.ev) cudaEventDestroy(p.first), cudaEventDestroy(p.second);
            cudaFree(prof.d_rows);
            throw;
        }
        t.prof = nullptr;
        t.sync();
        *out = qsr_kernel_profile{};
        for (auto &p : prof.ev) {
            float ms = 0;
            QSR_CUDA(cudaEventElapsedTime(&ms, p.first, p.second));
            out->absorb_ms += ms;
            cudaEventDestroy(p.first);
            cudaEventDestroy(p.second);
        }
        unsigned long long rows = 0;
        QSR_CUDA(cudaMemcpy(&rows, prof.d_rows, sizeof(rows), cudaMemcpyDeviceToHost));
        cudaFree(prof.d_rows);
        out->absorb_launches = prof.ev.size();
        out->absorb_rows = rows;
        out->absorb_slices = (t.rm_pitch + 63) / 64;
        out->row_words = t.k;
        out->total_ms = rt.total_ms;
    });
}

void qsr_engine_destroy(qsr_engine *e) { delete e; }

// ---- frames -----------------------------------------------------------------------
struct qsr_frames {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    uint64_t n = 0, shots = 0, kf = 0, pitch = 0; // kf: shot-words held here
    uint64_t j0 = 0;                                // global index of the first one
    uint32_t wbits = 64; // reference word type whose Philox draws the Z frames follow
    uint64_t *xf = nullptr, *zf = nullptr;
    uint64_t *rec = nullptr;  // record rows [cap][pitch]
    uint64_t rec_cap = 0;
    std::vector<uint32_t> measured;
    std::vector<int64_t> row_of; // qubit -> record row
    uint64_t *gate_buf = nullptr;
    uint64_t gate_cap = 0;
    uint64_t *xs = nullptr, *zs = nullptr; // row un-permute targets (fused windows)
    uint32_t *d_idx = nullptr;   // qubits + rows staging
    uint64_t idx_cap = 0;
    uint64_t plane_bytes = 0; // xf / zf come from the plane cache (no cudaMalloc per sample())
    ~qsr_frames() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        for (uint64_t *p : {xf, zf, xs, zs}) plane_cache().release(device, plane_bytes, p);
        if (rec) plane_cache().release(device, rec_cap * pitch * 8, rec);
        for (void *p : {(void *)gate_buf, (void *)d_idx})
            if (p) cudaFree(p);
        if (stream) cudaStreamDestroy(stream);
    }
    void ensure_rows(uint64_t rows) {
        if (rows <= rec_cap) return;
        uint64_t cap = std::max<uint64_t>(rows, std::min<uint64_t>(n, std::max<uint64_t>(rec_cap * 2, 64)));
        uint64_t *nr = static_cast<uint64_t *>(plane_cache().acquire(device, cap * pitch * 8));
        QSR_CUDA(cudaMemsetAsync(nr, 0, cap * pitch * 8, stream));
        if (rec) {
            QSR_CUDA(cudaMemcpyAsync(nr, rec, rec_cap * pitch * 8, cudaMemcpyDeviceToDevice, stream));
            QSR_CUDA(cudaStreamSynchronize(stream));
            plane_cache().release(device, rec_cap * pitch * 8, rec);
        }
        rec = nr;
        rec_cap = cap;
    }
    void ensure_idx(uint64_t m) {
        if (m <= idx_cap) return;
        if (d_idx) QSR_CUDA(cudaFree(d_idx));
        idx_cap = std::max<uint64_t>(m, 64);
        QSR_CUDA(cudaMalloc(&d_idx, idx_cap * 2 * 4));
    }
};

namespace {

void check_word_bits(unsigned wbits) {
    if (wbits != 8 && wbits != 16 && wbits != 32 && wbits != 64)
        fail(QSR_INVALID_ARGUMENT, "word size must be one of 8, 16, 32, 64");
}

std::unique_ptr<qsr_frames> make_frames(uint64_t n, uint64_t shots, uint64_t seed, int device,
                                        uint64_t j0 = 0, uint64_t nw = 0, unsigned wbits = 64) {
    check_word_bits(wbits);
    if (shots < 1) fail(QSR_INVALID_ARGUMENT, "init_frames: shots must be >= 1");
    if (n > kMaxQubits) fail(QSR_INVALID_ARGUMENT, "init_frames: n exceeds the supported maximum");
    auto f = std::make_unique<qsr_frames>();
    f->device = device;
    QSR_CUDA(cudaSetDevice(device));
    QSR_CUDA(cudaDeviceGetAttribute(&f->num_sms, cudaDevAttrMultiProcessorCount, device));
    QSR_CUDA(cudaStreamCreateWithFlags(&f->stream, cudaStreamNonBlocking));
    f->n = n;
    f->shots = shots;
    f->kf = nw ? nw : (shots + 63) / 64;
    f->j0 = j0;
    if (f->j0 + f->kf > (shots + 63) / 64) fail(QSR_INVALID_ARGUMENT, "init_frames: shot slice out of range");
    f->pitch = round_up(f->kf, 16);
    uint64_t words = std::max<uint64_t>(n, 1) * f->pitch;
    f->plane_bytes = words * 8;
    f->xf = static_cast<uint64_t *>(plane_cache().acquire(device, words * 8));
    f->zf = static_cast<uint64_t *>(plane_cache().acquire(device, words * 8));
    QSR_CUDA(cudaMemsetAsync(f->xf, 0, words * 8, f->stream));
    QSR_CUDA(cudaMemsetAsync(f->zf, 0, words * 8, f->stream));
    f->row_of.assign(n, -1);
    f->wbits = wbits;
    if (n) launch_frames_init(f->zf, n, f->kf, f->j0, f->pitch, shots, seed, 0, wbits, f->stream);
    return f;
}

void frames_window(qsr_frames &f, const uint64_t *d_gates, uint64_t ng) {
    launch_frame_window(f.xf, f.zf, f.pitch, d_gates, ng, f.num_sms, f.stream);
}

extern "C++" template <typename QubitOf>
void frames_measure_q(qsr_frames &f, QubitOf qubit_of, uint64_t ng, uint64_t seed, uint32_t epoch,
                      cudaStream_t st = nullptr) {
    if (!st) st = f.stream;
    std::vector<uint32_t> idx(2 * ng);
    for (uint64_t i = 0; i < ng; ++i) {
        uint32_t q = qubit_of(i);
        if (f.row_of[q] < 0) {
            f.row_of[q] = int64_t(f.measured.size());
            f.measured.push_back(q);
        }
        idx[i] = q;
        idx[ng + i] = uint32_t(f.row_of[q]);
    }
    f.ensure_rows(f.measured.size());
    f.ensure_idx(ng);
    QSR_CUDA(cudaMemcpyAsync(f.d_idx, idx.data(), 2 * ng * 4, cudaMemcpyHostToDevice, st));
    launch_measure_sample(f.xf, f.zf, f.pitch, f.kf, f.j0, f.shots, f.rec, f.d_idx, f.d_idx + ng, ng,
                          seed, epoch, f.wbits, st);
    QSR_CUDA(cudaStreamSynchronize(st)); // idx staging reused next call
}

void frames_measure(qsr_frames &f, const qsr_gate *gates, uint64_t ng, uint64_t seed, uint32_t epoch) {
    frames_measure_q(f, [&](uint64_t i) { return gates[i].q0; }, ng, seed, epoch);
}

// sample()'s frames as the passenger of a reference-shot run (streamed or resident): the same
// device windows, row un-permutes and measurement windows, on the tableau's stream.
struct FramesRider final : FramesSink {
    qsr_frames &f;
    uint64_t seed;
    uint32_t epoch = 1;
    FramesRider(qsr_frames &ff, uint64_t s) : f(ff), seed(s) { row_words = ff.kf; }
    void unitary(const uint64_t *g, uint64_t cnt, cudaStream_t st) override {
        launch_frame_window(f.xf, f.zf, f.pitch, g, cnt, f.num_sms, st);
    }
    void unpermute(const uint32_t *perm, cudaStream_t st) override {
        if (!f.xs) {
            f.xs = static_cast<uint64_t *>(plane_cache().acquire(f.device, f.plane_bytes));
            f.zs = static_cast<uint64_t *>(plane_cache().acquire(f.device, f.plane_bytes));
        }
        launch_unpermute_frame_rows(f.xf, f.xs, f.pitch, f.n, perm, f.num_sms, st);
        launch_unpermute_frame_rows(f.zf, f.zs, f.pitch, f.n, perm, f.num_sms, st);
        std::swap(f.xf, f.xs);
        std::swap(f.zf, f.zs);
    }
    void measure(const uint32_t *qubits, uint64_t m, cudaStream_t st) override {
        frames_measure_q(f, [&](uint64_t i) { return qubits[i]; }, m, seed, epoch++, st);
    }
};

// Fold in the reference outcomes: per_qubit() = last outcome per qubit (measure.hpp:50-64,
// frames.hpp:183-202); rows whose reference bit is 1 are flipped on the device.
void fold_reference(qsr_frames &f, const std::vector<qsr_record_entry> &ref, uint64_t num_qubits,
                    cudaStream_t st) {
    std::vector<int8_t> last(num_qubits, -1);
    for (const auto &e : ref) last[e.qubit] = int8_t(e.outcome ? 1 : 0);
    std::vector<uint32_t> flip_rows;
    for (uint64_t r = 0; r < f.measured.size(); ++r)
        if (last[f.measured[r]] == 1) flip_rows.push_back(uint32_t(r));
    if (!flip_rows.empty()) {
        f.ensure_idx(flip_rows.size());
        QSR_CUDA(cudaMemcpyAsync(f.d_idx, flip_rows.data(), flip_rows.size() * 4, cudaMemcpyHostToDevice, st));
        launch_record_fold(f.rec, f.pitch, f.kf, f.j0, f.shots, f.d_idx, flip_rows.size(), st);
    }
    QSR_CUDA(cudaStreamSynchronize(st));
}

uint64_t circuit_distinct_measured(const Circuit &c) {
    std::vector<uint8_t> seen(c.num_qubits, 0);
    uint64_t distinct = 0;
    for (const qsr_gate &g : c.gates)
        if (g.kind == QSR_MEASURE && g.q0 < c.num_qubits && !seen[g.q0]) { seen[g.q0] = 1; ++distinct; }
    return distinct;
}

void validate_frames_window(const qsr_frames &f, const qsr_gate *gates, uint64_t ng, bool meas,
                            const char *who) {
    std::vector<uint32_t> stamp;
    if (meas) {
        stamp.assign(f.n, 0);
        for (uint64_t i = 0; i < ng; ++i) {
            if (gates[i].q0 >= f.n) fail(QSR_OUT_OF_RANGE, std::string(who) + ": qubit out of range");
            if (stamp[gates[i].q0])
                fail(QSR_INVALID_ARGUMENT, "measure_sample: qubit measured twice in window");
            stamp[gates[i].q0] = 1;
        }
        return;
    }
    validate_window(f.n, gates, ng, false, stamp, 1);
}

} // namespace

qsr_status qsr_init_frames(uint64_t n, uint64_t shots, uint64_t seed, int device, qsr_frames **out) {
    return qsr_init_frames_word(n, shots, seed, 64, device, out);
}

qsr_status qsr_init_frames_word(uint64_t n, uint64_t shots, uint64_t seed, unsigned word_bits, int device,
                                qsr_frames **out) {
    return guard([&] {
        REQUIRE_PTR(out);
        auto f = make_frames(n, shots, seed, device, 0, 0, word_bits);
        QSR_CUDA(cudaStreamSynchronize(f->stream));
        *out = f.release();
    });
}

qsr_status qsr_frames_info(const qsr_frames *f, uint64_t *n, uint64_t *shots, uint64_t *kf) {
    return guard([&] {
        REQUIRE_PTR(f);
        if (n) *n = f->n;
        if (shots) *shots = f->shots;
        if (kf) *kf = f->kf;
    });
}

qsr_status qsr_frames_shot_words(const qsr_frames *f, uint64_t *j0, uint64_t *nw) {
    return guard([&] {
        REQUIRE_PTR(f);
        if (j0) *j0 = f->j0;
        if (nw) *nw = f->kf;
    });
}

qsr_status qsr_frames_download(const qsr_frames *f, uint64_t *xf, uint64_t *zf) {
    return guard([&] {
        REQUIRE_PTR(f);
        QSR_CUDA(cudaSetDevice(f->device));
        if (f->n == 0) return;
        if (xf) download_2d(xf, f->kf * 8, f->xf, f->pitch * 8, f->kf * 8, f->n, f->stream);
        if (zf) download_2d(zf, f->kf * 8, f->zf, f->pitch * 8, f->kf * 8, f->n, f->stream);
    });
}

qsr_status qsr_frames_upload(qsr_frames *f, const uint64_t *xf, const uint64_t *zf) {
    return guard([&] {
        REQUIRE_PTR(f); REQUIRE_PTR(xf); REQUIRE_PTR(zf);
        QSR_CUDA(cudaSetDevice(f->device));
        if (f->n == 0) return;
        QSR_CUDA(cudaMemcpy2DAsync(f->xf, f->pitch * 8, xf, f->kf * 8, f->kf * 8, f->n,
                                   cudaMemcpyHostToDevice, f->stream));
        QSR_CUDA(cudaMemcpy2DAsync(f->zf, f->pitch * 8, zf, f->kf * 8, f->kf * 8, f->n,
                                   cudaMemcpyHostToDevice, f->stream));
        QSR_CUDA(cudaStreamSynchronize(f->stream));
    });
}

qsr_status qsr_apply_window_frames(qsr_frames *f, const qsr_gate *gates, uint64_t ng, int is_meas) {
    return guard([&] {
        REQUIRE_PTR(f);
        if (ng) REQUIRE_PTR(gates);
        if (is_meas) fail(QSR_INVALID_ARGUMENT, "apply_window_frames: measurement window");
        validate_frames_window(*f, gates, ng, false, "apply_window_frames");
        QSR_CUDA(cudaSetDevice(f->device));
        if (ng > f->gate_cap) {
            if (f->gate_buf) QSR_CUDA(cudaFree(f->gate_buf));
            f->gate_cap = std::max<uint64_t>(ng, 1024);
            QSR_CUDA(cudaMalloc(&f->gate_buf, f->gate_cap * 8));
        }
        auto packed = pack(gates, ng);
        QSR_CUDA(cudaMemcpyAsync(f->gate_buf, packed.data(), ng * 8, cudaMemcpyHostToDevice, f->stream));
        frames_window(*f, f->gate_buf, ng);
        QSR_CUDA(cudaStreamSynchronize(f->stream));
    });
}

qsr_status qsr_measure_sample(qsr_frames *f, const qsr_gate *gates, uint64_t ng, int is_meas,
                              uint64_t seed, uint32_t epoch) {
    return guard([&] {
        REQUIRE_PTR(f);
        if (ng) REQUIRE_PTR(gates);
        if (!is_meas) fail(QSR_INVALID_ARGUMENT, "measure_sample: not a measurement window");
        validate_frames_window(*f, gates, ng, true, "measure_sample");
        QSR_CUDA(cudaSetDevice(f->device));
        frames_measure(*f, gates, ng, seed, epoch);
    });
}

qsr_status qsr_frames_record(const qsr_frames *f, uint64_t *nrows, uint32_t *measured,
                             uint64_t *words) {
    return guard([&] {
        TraceScope tr(words ? "frames_record (download)" : "frames_record (size)");
        REQUIRE_PTR(f); REQUIRE_PTR(nrows);
        *nrows = f->measured.size();
        if (measured) std::memcpy(measured, f->measured.data(), f->measured.size() * 4);
        if (words && !f->measured.empty()) {
            QSR_CUDA(cudaSetDevice(f->device));
            const uint64_t rows = f->measured.size();
            download_2d(words, f->kf * 8, f->rec, f->pitch * 8, f->kf * 8, rows, f->stream);
        }
    });
}

void qsr_frames_destroy(qsr_frames *f) {
    TraceScope tr("frames_destroy");
    delete f;
}

static qsr_status sample_impl(const qsr_circuit *c, uint64_t shots, uint64_t seed, int device, int world,
                       int rank, qsr_frames **out, qsr_run_report *report, unsigned wbits = 64) {
    return guard([&] {
        check_word_bits(wbits);
        auto wall0 = std::chrono::steady_clock::now();
        REQUIRE_PTR(c); REQUIRE_PTR(out);
        if (shots < 1) fail(QSR_INVALID_ARGUMENT, "init_frames: shots must be >= 1");
        const uint64_t kf_all = (shots + 63) / 64;
        if (world < 1 || uint64_t(world) > kf_all || rank < 0 || rank >= world)
            fail(QSR_INVALID_ARGUMENT, "sample: world must be in [1, ceil(shots/64)], 0 <= rank < world");
        const uint64_t w0 = kf_all * uint64_t(rank) / uint64_t(world);
        const uint64_t nw = kf_all * uint64_t(rank + 1) / uint64_t(world) - w0;
        TraceScope tr_all("sample");
        // One record allocation: the distinct measured qubits of the circuit.
        auto distinct_measured = [&] { return circuit_distinct_measured(*c); };
        DeviceTableau t(c->num_qubits, device);
        const uint64_t nm = c->measure_count();
        qsr_record_entry *d_rec = nullptr;
        QSR_CUDA(cudaMalloc(&d_rec, std::max<uint64_t>(nm, 1) * sizeof(qsr_record_entry)));
        std::vector<qsr_record_entry> ref(nm);
        std::unique_ptr<qsr_frames> f;
        const bool streaming = !(getenv("QSR_STREAM") && getenv("QSR_STREAM")[0] == '0');
        try {
            if (streaming) {
                // The reference shot (frames.hpp:167) streamed as in run_single_shot (schedule
                // overlapped with the device, fused windows), and the frames (frames.hpp:171-181)
                // riding the same device windows, row un-permutes and measurement windows on the
                // tableau's stream: the Pauli frames follow the same Clifford conjugation, so
                // fusion is exact for them too.
                TraceScope tr("  reference shot + frames (streamed)");
                f = make_frames(c->num_qubits, shots, seed, device, w0, nw, wbits);
                if (const uint64_t d = distinct_measured()) f->ensure_rows(d);
                QSR_CUDA(cudaStreamSynchronize(f->stream));
                FramesRider sink(*f, seed);
                RunTimes rt;
                StreamCounts sc;
                run_circuit_streaming(t, *c, seed, d_rec, rt, sc, &sink);
                if (nm)
                    QSR_CUDA(cudaMemcpyAsync(ref.data(), d_rec, nm * sizeof(qsr_record_entry),
                                             cudaMemcpyDeviceToHost, t.stream));
                t.sync();
                if (report) {
                    DeviceSchedule cnt;
                    cnt.device = device;
                    cnt.unitary_count = sc.unitary;
                    cnt.measure_count = sc.measures;
                    cnt.is_meas.resize(sc.windows);
                    double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
                    fill_report(report, rt, cnt, ref, wall);
                }
            } else {
                // Reference shot on the O(G) plan scattered straight into packed device gates
                // (schedule_windows' windows; the sampling mode is only a tag, schedule.hpp:37-42);
                // the frames then replay the same device-resident windows.
                TraceScope tr_ref("  reference shot");
                auto ds = upload_circuit(*c, device, t.stream, /*fuse=*/false);
                RunTimes rt;
                run_device(t, *ds, seed, d_rec, rt);
                if (nm)
                    QSR_CUDA(cudaMemcpyAsync(ref.data(), d_rec, nm * sizeof(qsr_record_entry),
                                             cudaMemcpyDeviceToHost, t.stream));
                t.sync();
                if (report) {
                    double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
                    fill_report(report, rt, *ds, ref, wall);
                }
                f = make_frames(c->num_qubits, shots, seed, device, w0, nw, wbits);
                if (const uint64_t d = distinct_measured()) f->ensure_rows(d);
                QSR_CUDA(cudaStreamSynchronize(f->stream));
                TraceScope tr_frames("  frames windows");
                uint32_t epoch = 1;
                const uint64_t W = ds->is_meas.size();
                for (uint64_t w = 0; w < W;) {
                    const uint64_t b = ds->offsets[w], e = ds->offsets[w + 1];
                    if (ds->is_meas[w]) {
                        const auto &mq = ds->mqubits[w];
                        frames_measure_q(*f, [&](uint64_t i) { return mq[i]; }, e - b, seed, epoch++);
                        ++w;
                        continue;
                    }
                    uint64_t w1 = w;
                    while (w1 < W && !ds->is_meas[w1]) ++w1;
                    for (uint64_t v = w; v < w1; ++v)
                        frames_window(*f, ds->d_gates + ds->offsets[v], ds->offsets[v + 1] - ds->offsets[v]);
                    w = w1;
                }
            }
        } catch (...) {
            cudaFree(d_rec);
            throw;
        }
        cudaFree(d_rec);
        fold_reference(*f, ref, c->num_qubits, f->stream);
        *out = f.release();
    });
}

qsr_status qsr_sample(const qsr_circuit *c, uint64_t shots, uint64_t seed, int device,
                      qsr_frames **out, qsr_run_report *report) {
    return sample_impl(c, shots, seed, device, 1, 0, out, report);
}

qsr_status qsr_sample_word(const qsr_circuit *c, uint64_t shots, uint64_t seed, unsigned word_bits,
                           int device, qsr_frames **out, qsr_run_report *report) {
    return sample_impl(c, shots, seed, device, 1, 0, out, report, word_bits);
}

qsr_status qsr_frames_word_bits(const qsr_frames *f, unsigned *word_bits) {
    return guard([&] {
        REQUIRE_PTR(f); REQUIRE_PTR(word_bits);
        *word_bits = f->wbits;
    });
}

// sample(circuit, shots, seed) on a resident engine (frames.hpp:163-204): the reference shot is
// the engine's run, and the frames ride its windows on the same stream; *device_ms = CUDA-event
// time of the whole call on that stream (frames init, reference shot + frames, record fold).
qsr_status qsr_engine_sample(qsr_engine *e, uint64_t shots, uint64_t seed, int world, int rank,
                             qsr_frames **out, double *device_ms) {
    return guard([&] {
        REQUIRE_PTR(e); REQUIRE_PTR(out);
        if (shots < 1) fail(QSR_INVALID_ARGUMENT, "init_frames: shots must be >= 1");
        const uint64_t kf_all = (shots + 63) / 64;
        if (world < 1 || uint64_t(world) > kf_all || rank < 0 || rank >= world)
            fail(QSR_INVALID_ARGUMENT, "sample: world must be in [1, ceil(shots/64)], 0 <= rank < world");
        const uint64_t w0 = kf_all * uint64_t(rank) / uint64_t(world);
        const uint64_t nw = kf_all * uint64_t(rank + 1) / uint64_t(world) - w0;
        DeviceTableau &t = *e->t;
        QSR_CUDA(cudaSetDevice(t.device));
        std::vector<uint8_t> seen(t.n, 0);
        uint64_t distinct = 0;
        for (const auto &mq : e->ds->mqubits)
            for (uint32_t q : mq)
                if (!seen[q]) { seen[q] = 1; ++distinct; }
        cudaEvent_t a, b, fdone;
        QSR_CUDA(cudaEventCreate(&a));
        QSR_CUDA(cudaEventCreate(&b));
        QSR_CUDA(cudaEventCreateWithFlags(&fdone, cudaEventDisableTiming));
        QSR_CUDA(cudaEventRecord(a, t.stream));
        const uint64_t l0 = g_launches;
        // The frames never read the tableau: on their own stream their windows overlap the
        // reference shot's (small, L2-resident tableau windows and the collapse chain).
        auto f = make_frames(t.n, shots, seed, t.device, w0, nw, 64);
        QSR_CUDA(cudaStreamWaitEvent(f->stream, a, 0));
        if (distinct) f->ensure_rows(distinct);
        FramesRider rider(*f, seed);
        rider.own = f->stream;
        e->last = RunTimes{};
        run_device(t, *e->ds, seed, e->d_rec, e->last, &rider);
        QSR_CUDA(cudaEventRecord(fdone, f->stream));
        QSR_CUDA(cudaStreamWaitEvent(t.stream, fdone, 0));
        const uint64_t nm = e->ds->measure_count;
        std::vector<qsr_record_entry> ref(nm);
        if (nm)
            QSR_CUDA(cudaMemcpyAsync(ref.data(), e->d_rec, nm * sizeof(qsr_record_entry), cudaMemcpyDeviceToHost,
                                     t.stream));
        t.sync();
        fold_reference(*f, ref, t.n, t.stream);
        e->frames_ms = 0;
        for (auto &r : rider.runs) {
            float fm = 0;
            QSR_CUDA(cudaEventElapsedTime(&fm, r.first, r.second));
            e->frames_ms += fm;
            cudaEventDestroy(r.first);
            cudaEventDestroy(r.second);
        }
        cudaEventDestroy(fdone);
        QSR_CUDA(cudaEventRecord(b, t.stream));
        QSR_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        QSR_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        e->launches = g_launches - l0;
        if (device_ms) *device_ms = ms;
        *out = f.release();
    });
}

qsr_status qsr_engine_frames_bytes(const qsr_engine *e, double *bytes, double *ms) {
    return guard([&] {
        REQUIRE_PTR(e);
        REQUIRE_PTR(bytes);
        *bytes = e->last.frames_bytes;
        if (ms) *ms = e->frames_ms;
    });
}

qsr_status qsr_sample_shard(const qsr_circuit *c, uint64_t shots, uint64_t seed, int world, int rank,
                            int device, qsr_frames **out, qsr_run_report *report) {
    return sample_impl(c, shots, seed, device, world, rank, out, report);
}

} // extern "C"
