// K13-K16 — Pauli-frame sampling kernels (reference frames.hpp:46-204) and the basis-state
// initialiser of the tableau (tableau.hpp:120-131).
//
// Frames are qubit-major, shot-packed: word (q, j) at q*pitch + j holds shots j*64..j*64+63.
// Every (qubit, shot-word) is independent, so init / measure_sample / the reference fold are
// flat grid-stride kernels; Philox words are keyed by (seed, 1, epoch, (q<<24)|j), exactly
// the reference's key, so results do not depend on launch geometry or shot sharding.
#include "common.cuh"
#include "device.hpp"

namespace qsr {

namespace {

// Z-frame word (q, j) of the 64-bit device layout for the reference word type W = wbits
// (frames.hpp:55-66, 141-145): the reference keys one Philox word per W-bit word j_W and keeps its
// low W bits, so a 64-bit device word is 64 / W such draws (j_W = j * 64 / W + i), shot order kept.
__device__ __forceinline__ uint64_t frame_word(uint64_t seed, uint32_t epoch, uint64_t q, uint64_t jg,
                                               uint32_t wbits) {
    if (wbits == 64) return d_philox_word(seed, 1, epoch, (q << 24) | jg);
    const uint32_t per = 64 / wbits;
    const uint64_t m = (uint64_t(1) << wbits) - 1;
    uint64_t w = 0;
    for (uint32_t i = 0; i < per; ++i)
        w |= (d_philox_word(seed, 1, epoch, (q << 24) | (jg * per + i)) & m) << (i * wbits);
    return w;
}

// kf = shot-words held here, j0 = their global offset, jl = global index of the last word
// (the one the last-word mask applies to). Unsharded: j0 = 0, jl = kf - 1.
__global__ void k_frames_init(uint64_t *__restrict__ zf, uint64_t n, uint64_t kf, uint64_t j0,
                              uint64_t jl, uint64_t pitch, uint64_t last_mask, uint64_t seed,
                              uint32_t epoch, uint32_t wbits) {
    const uint64_t total = n * kf;
    for (uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t q = idx / kf, j = idx % kf, jg = j0 + j;
        uint64_t w = frame_word(seed, epoch, q, jg, wbits);
        if (jg == jl) w &= last_mask;
        zf[q * pitch + j] = w;
    }
}

__global__ void k_measure_sample(const uint64_t *__restrict__ xf, uint64_t *__restrict__ zf,
                                 uint64_t pitch, uint64_t kf, uint64_t j0, uint64_t jl,
                                 uint64_t last_mask,
                                 uint64_t *__restrict__ rec, const uint32_t *__restrict__ qubits,
                                 const uint32_t *__restrict__ rows, uint64_t m, uint64_t seed,
                                 uint32_t epoch, uint32_t wbits) {
    const uint64_t total = m * kf;
    for (uint64_t item = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; item < total;
         item += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t i = item / kf, j = item % kf, jg = j0 + j;
        uint64_t q = qubits[i];
        rec[uint64_t(rows[i]) * pitch + j] = xf[q * pitch + j];
        uint64_t w = frame_word(seed, epoch, q, jg, wbits);
        if (jg == jl) w &= last_mask;
        zf[q * pitch + j] = w;
    }
}

__global__ void k_record_fold(uint64_t *__restrict__ rec, uint64_t pitch, uint64_t kf,
                              uint64_t j0, uint64_t jl, uint64_t last_mask,
                              const uint32_t *__restrict__ flip_rows, uint64_t nflip) {
    const uint64_t total = nflip * kf;
    for (uint64_t item = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; item < total;
         item += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t i = item / kf, j = item % kf;
        uint64_t *p = rec + uint64_t(flip_rows[i]) * pitch + j;
        uint64_t mask = j0 + j == jl ? last_mask : ~0ull;
        *p = (*p ^ ~0ull) & mask;
    }
}

__global__ void k_basis_state(uint64_t *__restrict__ x, uint64_t *__restrict__ z,
                              uint64_t *__restrict__ s, uint64_t g0, uint64_t n_gen, uint64_t kg,
                              uint64_t pitch, const uint8_t *__restrict__ init) {
    // Destabilizer g = (-1)^b X_g, stabilizer g = (-1)^b Z_g (tableau.hpp:120-129), for the
    // generators g0 .. g0+n_gen-1 this tableau (shard) holds; local generator l = g - g0.
    for (uint64_t l = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; l < n_gen;
         l += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t q = g0 + l;
        x[q * pitch + l / 64] = 1ull << (l % 64);
        z[q * pitch + kg + l / 64] = 1ull << (l % 64);
    }
    if (init) {
        // Sign words: one thread per word (no write conflicts).
        for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < kg;
             w += uint64_t(gridDim.x) * blockDim.x) {
            uint64_t v = 0;
            for (uint64_t b = 0; b < 64 && w * 64 + b < n_gen; ++b)
                v |= uint64_t(init[g0 + w * 64 + b] & 1) << b;
            s[w] = v;
            s[kg + w] = v;
        }
    }
}

inline uint64_t last_mask_for(uint64_t shots) {
    uint64_t r = shots % 64;
    return r == 0 ? ~0ull : ((1ull << r) - 1);
}

inline unsigned grid_for(uint64_t total, unsigned threads) {
    uint64_t b = (total + threads - 1) / threads;
    if (b > 148u * 32u) b = 148u * 32u;
    if (b < 1) b = 1;
    return unsigned(b);
}

} // namespace

void launch_frames_init(uint64_t *zf, uint64_t n, uint64_t kf, uint64_t j0, uint64_t pitch,
                        uint64_t shots, uint64_t seed, uint32_t epoch, uint32_t wbits, cudaStream_t st) {
    k_frames_init<<<grid_for(n * kf, 256), 256, 0, st>>>(zf, n, kf, j0, (shots + 63) / 64 - 1, pitch,
                                                         last_mask_for(shots), seed, epoch, wbits);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void launch_measure_sample(uint64_t *xf, uint64_t *zf, uint64_t pitch, uint64_t kf, uint64_t j0,
                           uint64_t shots, uint64_t *rec, const uint32_t *qubits,
                           const uint32_t *rows, uint64_t m, uint64_t seed, uint32_t epoch,
                           uint32_t wbits, cudaStream_t st) {
    if (m == 0) return;
    k_measure_sample<<<grid_for(m * kf, 256), 256, 0, st>>>(xf, zf, pitch, kf, j0, (shots + 63) / 64 - 1,
                                                            last_mask_for(shots), rec, qubits, rows,
                                                            m, seed, epoch, wbits);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void launch_record_fold(uint64_t *rec, uint64_t pitch, uint64_t kf, uint64_t j0, uint64_t shots,
                        const uint32_t *flip_rows, uint64_t nflip, cudaStream_t st) {
    if (nflip == 0) return;
    k_record_fold<<<grid_for(nflip * kf, 256), 256, 0, st>>>(rec, pitch, kf, j0, (shots + 63) / 64 - 1,
                                                             last_mask_for(shots), flip_rows, nflip);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void launch_zero_state(DeviceTableau &t, const uint8_t *d_init) {
    QSR_CUDA(cudaMemsetAsync(t.x, 0, t.plane_words * 8, t.stream));
    QSR_CUDA(cudaMemsetAsync(t.z, 0, t.plane_words * 8, t.stream));
    QSR_CUDA(cudaMemsetAsync(t.s, 0, t.cm_pitch * 8, t.stream));
    k_basis_state<<<grid_for(std::max<uint64_t>(t.n_gen, t.kg), 256), 256, 0, t.stream>>>(
        t.x, t.z, t.s, t.g0, t.n_gen, t.kg, t.cm_pitch, d_init);
    QSR_CUDA(cudaGetLastError());
    count_launch();
    t.layout = QSR_COLUMN_MAJOR;
    t.trusted = true;
}

} // namespace qsr
