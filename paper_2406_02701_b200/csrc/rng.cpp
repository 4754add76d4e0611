// The reference's portable generator (proj/core/src/rng.cpp:9-53): splitmix64
// seeding, xorshift64* stream, 53-bit uniforms, Box-Muller normals with the
// second value cached.  Host code: the synthetic inputs the reference's
// acceptance tests and CLI draw (Rng(1000 + n) uniforms, acceptance.cpp:30-36
// and :158-162; sample_gp's normals, workloads.cpp:41-49) are reproduced
// bit for bit before upload.
#include <cmath>
#include <cstdint>

#include "internal.hpp"

namespace {

struct Rng {
    uint64_t state;
    bool has_cached = false;
    double cached = 0.0;

    explicit Rng(uint64_t seed) {
        uint64_t x = seed + 0x9E3779B97F4A7C15ull;  // splitmix64 (rng.cpp:9-15)
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        state = z ^ (z >> 31);
        if (state == 0) state = 0x2545F4914F6CDD1Dull;
    }
    uint64_t next_bits() {  // xorshift64* (rng.cpp:25-32)
        uint64_t x = state;
        x ^= x >> 12;
        x ^= x << 25;
        x ^= x >> 27;
        state = x;
        return x * 0x2545F4914F6CDD1Dull;
    }
    double uniform() { return static_cast<double>(next_bits() >> 11) * 0x1p-53; }
    double normal() {  // Box-Muller, pairs cached (rng.cpp:38-50)
        if (has_cached) {
            has_cached = false;
            return cached;
        }
        double u1 = uniform();
        while (u1 == 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * M_PI * u2;
        cached = r * std::sin(theta);
        has_cached = true;
        return r * std::cos(theta);
    }
};

}  // namespace

extern "C" {

mp_status mp_rng_uniform(uint64_t seed, int64_t skip, int64_t n, double* out) {
    if ((n > 0 && !out) || n < 0 || skip < 0) return MP_INVALID_PARAM;
    Rng r(seed);
    for (int64_t i = 0; i < skip; ++i) r.next_bits();
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
    return MP_OK;
}

mp_status mp_rng_normal(uint64_t seed, int64_t n, double* out) {
    if ((n > 0 && !out) || n < 0) return MP_INVALID_PARAM;
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
    return MP_OK;
}

}  // extern "C"
