// Device MT19937-64 (std::mt19937_64, the engine behind the reference's Rng, rng.hpp:11-66)
// and derive_seed (SplitMix64, rng.hpp), shared by the frame generator (gen_kernels.cu) and
// the FPS-SFT slope / offset draws (sft_kernels.cu).  Integer-only: bit-identical to libstdc++.
#pragma once
#include <cstdint>

namespace ofdmr {
namespace mt64 {

constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMatA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;

__device__ __forceinline__ uint64_t splitmix(uint64_t base, uint64_t stream) {
    // rng.hpp derive_seed (SplitMix64 of base ^ golden * (stream + 1))
    uint64_t z = base + 0x9E3779B97F4A7C15ull * (stream + 1ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}
__device__ __forceinline__ uint64_t twist1(uint64_t a, uint64_t b, uint64_t m) {
    const uint64_t x = (a & kUpper) | (b & kLower);
    return m ^ (x >> 1) ^ ((x & 1ull) ? kMatA : 0ull);
}

// init_genrand64 (sequential; one thread)
__device__ inline void mt_seed(uint64_t* mt, uint64_t seed) {
    mt[0] = seed;
    for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
}

// Scalar generator (one thread walks the stream; the twist is done in place every 312 outputs).
struct MtScalar {
    uint64_t* mt;
    int idx;
    __device__ uint64_t next() {
        if (idx >= kMtN) {
            for (int i = 0; i < kMtN; ++i) mt[i] = twist1(mt[i], mt[(i + 1) % kMtN], mt[(i + kMtM) % kMtN]);
            idx = 0;
        }
        return temper(mt[idx++]);
    }
    __device__ double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
    __device__ double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    // Rng::uniform_int (rng.hpp): rejection with limit = UINT64_MAX - UINT64_MAX % n; rej is set
    // when a rejection happened (the generator regenerates such frames on the CPU)
    __device__ uint64_t uniform_int(uint64_t n, int& rej) {
        const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        uint64_t v;
        do {
            v = next();
            if (v >= limit) rej = 1;
        } while (v >= limit);
        return v % n;
    }
    __device__ uint64_t uniform_int(uint64_t n) {
        int rej = 0;
        return uniform_int(n, rej);
    }
};

// Warp-parallel twist + temper: appends 312 outputs to the ring out[(pos + i) & mask].
__device__ inline void mt_block(uint64_t* mt, uint64_t* out, uint32_t pos, uint32_t mask) {
    const int lane = threadIdx.x & 31;
    // first half: i < 156 reads only old words
    for (int b = 0; b < kMtM; b += 32) {
        const int i = b + lane;
        uint64_t v = 0;
        if (i < kMtM) v = twist1(mt[i], mt[i + 1], mt[i + kMtM]);
        __syncwarp();
        if (i < kMtM) mt[i] = v;
        __syncwarp();
    }
    // second half: 156 <= i < 311 reads old mt[i], mt[i+1] and new mt[i-156]
    for (int b = kMtM; b < kMtN - 1; b += 32) {
        const int i = b + lane;
        uint64_t v = 0;
        if (i < kMtN - 1) v = twist1(mt[i], mt[i + 1], mt[i - kMtM]);
        __syncwarp();
        if (i < kMtN - 1) mt[i] = v;
        __syncwarp();
    }
    if (lane == 0) mt[kMtN - 1] = twist1(mt[kMtN - 1], mt[0], mt[kMtM - 1]);
    __syncwarp();
    for (int i = lane; i < kMtN; i += 32) out[(pos + i) & mask] = temper(mt[i]);
    __syncwarp();
}

}  // namespace mt64
}  // namespace ofdmr
