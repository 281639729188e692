// Window pairing (host side): two consecutive unitary windows as small independent components.
//
// A window's gates act on disjoint rows, so each window is a matching on the CM rows and the
// union of two consecutive windows A, B is a set of paths and cycles. After gate fusion about half
// of the rows carry a two-qubit gate per window, so a path continues through a row with
// probability ~1/2 and components are short (mean ~2 gates). A component is applied by one warp
// that loads its rows once, applies A's gates then B's gates in registers and stores once
// (k_gates.cu K1p): every row touched by both windows moves once instead of twice. Components of
// more than kPairRows rows or kPairGates gates keep the plain path (their A gates in one window,
// then their B gates in the next; rows are disjoint from every record, so the order against the
// records is free). Exact: the gates of every row run in the original order.
//
// Record (kPairRecWords = 16 words, 128 B):
//   w0: bits 0-3 rows, 4-7 gates, 8-23 per-row read planes (2 bits per row: x, z),
//       24-39 per-row written planes
//   w1..w4: rows (32 bits each, two per word); w5..w12: gates (packed device words whose q0 / q1
//   are local row indices; A's gates first); w13..w15: zero.
#pragma once

#include <cstdint>
#include <vector>

namespace qsr {

struct PairOut {
    std::vector<uint64_t> records;   // kPairRecWords words each
    std::vector<uint64_t> rest_a;    // gates of oversized components, window A
    std::vector<uint64_t> rest_b;    // ... window B
    uint64_t record_words = 0;       // words moved per generator-word by the records (bytes model)
};

class Pairer {
  public:
    explicit Pairer(uint32_t rows);
    void pair(const uint64_t *a, uint64_t na, const uint64_t *b, uint64_t nb, PairOut &out);

  private:
    std::vector<int32_t> ia_, ib_;    // row -> gate index in A / B (-1 = none)
    std::vector<uint32_t> stamp_;     // row -> component stamp
    uint32_t cur_ = 0;
    std::vector<uint8_t> seen_a_, seen_b_;
};

// Pairing pays where windows are big enough for the saved bytes to outweigh the extra launches
// of the remainder windows (c5: ~56 k gates per fused window; c2's ~14 k-gate windows do not).
constexpr uint64_t kPairMinGates = 16384;
// Opt-in: QSR_PAIR=1 pairs windows of every size (tests), QSR_PAIR=2 windows >= kPairMinGates.
bool pairing_enabled();
bool pair_windows_of(uint64_t na, uint64_t nb);

} // namespace qsr
