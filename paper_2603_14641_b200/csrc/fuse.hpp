// Exact gate fusion for whole-circuit runs (host side): fewer tableau bytes per gate, identical
// results.
//
//  * SWAP is a pure exchange of two qubit rows (gates.hpp:92-96, no sign), so it becomes a
//    relabelling: `pi` maps each logical qubit to the physical CM row holding it. ISWAP is the
//    swap followed by a residual that is symmetric in its operands (gates.hpp:97-110): relabel,
//    then a read-4 / write-2 K_ISWAP_R gate instead of read-4 / write-4.
//  * Runs of single-qubit gates compose into one of the 24 single-qubit Cliffords (GF(2) 2x2
//    matrix on (x, z) + sign flips of the images of X, Z, Y). A run is kept pending per logical
//    qubit and applied as a pre-operation of the next two-qubit gate on that qubit (whose words are
//    loaded anyway), so the run itself moves no bytes. Pending operations are flushed as K_C1
//    gates in a window of their own before every measurement window and at the end.
// Every rule acts on each generator bit independently, so composing the per-bit actions composes
// the gates exactly (conjugation is a group homomorphism, signs included). Gates of one window act
// on disjoint logical qubits, hence on disjoint physical rows; the emitted windows stay disjoint.
// Before every measurement window (and at the end) the device rows are un-permuted to logical
// order and the map reset, so measurements see logical qubits (their batch qubits stay adjacent
// in the tableau words, and the record needs no fix-up).
#pragma once

#include <cstdint>
#include <vector>

#include "host.hpp"

namespace qsr {

// Host copies of the 24-element group (same encoding as common.cuh kCliff1).
extern const uint8_t kCliff1Host[24];
// compose[e][k]: element after applying gate kind k (X Y Z H S SDG = 0..5) following e.
extern const uint8_t kCliff1Compose[24][6];

// Operand words (bit0 x0, bit1 z0, bit2 x1, bit3 z1) a packed gate reads / writes on the device,
// with signs (kind_reads / gate_writes of common.cuh). For the bytes-moved accounting.
uint32_t packed_reads(uint64_t w);
uint32_t packed_writes(uint64_t w);
// The same without signs (Pauli frames, frames.hpp:76-94: X / Y / Z read nothing).
uint32_t packed_reads_frames(uint64_t w);

class Fuser {
  public:
    explicit Fuser(uint32_t n);
    // One unitary window of packed logical gates -> packed physical device gates (appended).
    void unitary(const uint64_t *in, uint64_t cnt, WordVec &out);
    // All pending single-qubit operations as K_C1 gates (appended; one window's worth).
    void flush(WordVec &out);
    bool pending() const { return !pend_list_.empty(); }
    uint32_t phys(uint32_t q) const { return st_[q].pi; }
    std::vector<uint32_t> permutation() const; // logical -> physical
    bool identity_permutation() const;
    // After the device rows were un-permuted to logical order.
    void reset_permutation();

  private:
    // One 8-byte record per logical qubit: an operand costs one cache access.
    struct Q {
        uint32_t pi;     // physical row
        uint8_t pend;    // pending single-qubit Clifford, 0 = identity
        uint8_t listed;  // in pend_list_
        uint16_t pad;
    };
    std::vector<Q> st_;
    std::vector<uint32_t> pend_list_;
    void note(uint32_t q) {
        if (!st_[q].listed) { st_[q].listed = 1; pend_list_.push_back(q); }
    }
};

// QSR_FUSE=0 disables fusion (plain device gates).
bool fusion_enabled();

} // namespace qsr
