// Device-side numeric helpers: bit-exact storage conversions that reproduce
// the reference's set_linear / at_linear semantics (array.cpp:97-133,
// precision.cpp:49-109) and the x86-64 cast behaviour the reference compiles
// to (cvtsd2ss / cvtss2sd NaN payload rules).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mpcr {

// ---- storage <-> compute ---------------------------------------------------
// Half storage is carried as raw uint16_t bits everywhere.

// decode_f16 (precision.cpp:95-109) into float: exact; NaN -> 0x7FC00000 (the
// float image of the canonical double quiet NaN the reference decodes to).
__device__ __forceinline__ float h2f(uint16_t b) {
    if ((b & 0x7C00u) == 0x7C00u && (b & 0x3FFu)) return __int_as_float(0x7FC00000);
    float f;
    asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(b));
    return f;
}
// decode_f16 into double: exact; NaN -> 0x7FF8000000000000 (quiet_NaN()).
__device__ __forceinline__ double h2d(uint16_t b) {
    if ((b & 0x7C00u) == 0x7C00u && (b & 0x3FFu))
        return __longlong_as_double(0x7FF8000000000000ll);
    float f;
    asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(b));
    return static_cast<double>(f);
}
// encode_f16 (precision.cpp:49-93): RNE from float (exact as from double since
// float is a subset); NaN -> 0x7E00.
__device__ __forceinline__ uint16_t f2h(float f) {
    if (f != f) return 0x7E00u;
    uint16_t h;
    asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(f));
    return h;
}
// encode_f16 straight from double (single rounding, no double rounding).
__device__ __forceinline__ uint16_t d2h(double d) {
    if (d != d) return 0x7E00u;
    uint16_t h;
    asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(d));
    return h;
}
// static_cast<float>(double) as x86 cvtsd2ss: RNE; NaN keeps sign and the top
// 22 payload bits with the quiet bit forced.
__device__ __forceinline__ float d2f(double d) {
    if (d != d) {
        const uint64_t u = static_cast<uint64_t>(__double_as_longlong(d));
        const uint32_t s = static_cast<uint32_t>(u >> 63) << 31;
        const uint32_t pay = static_cast<uint32_t>((u >> 29) & 0x3FFFFFu);
        return __int_as_float(static_cast<int>(s | 0x7FC00000u | pay));
    }
    return __double2float_rn(d);
}
// static_cast<double>(float) as x86 cvtss2sd: exact; NaN payload shifted up
// with the quiet bit forced.
__device__ __forceinline__ double f2d(float f) {
    if (f != f) {
        const uint32_t u = static_cast<uint32_t>(__float_as_int(f));
        const uint64_t s = static_cast<uint64_t>(u >> 31) << 63;
        const uint64_t pay = static_cast<uint64_t>(u & 0x3FFFFFu) << 29;
        return __longlong_as_double(static_cast<long long>(s | 0x7FF8000000000000ull | pay));
    }
    return static_cast<double>(f);
}

// Storage type per precision.
template <int P> struct Storage;
template <> struct Storage<0> { using T = uint16_t; };
template <> struct Storage<1> { using T = float; };
template <> struct Storage<2> { using T = double; };

// Load a stored element widened to compute type C (float or double).
template <typename C> __device__ __forceinline__ C load_as(const uint16_t* p, int64_t i);
template <typename C> __device__ __forceinline__ C load_as(const float* p, int64_t i);
template <typename C> __device__ __forceinline__ C load_as(const double* p, int64_t i);
template <> __device__ __forceinline__ float load_as<float>(const uint16_t* p, int64_t i) { return h2f(p[i]); }
template <> __device__ __forceinline__ double load_as<double>(const uint16_t* p, int64_t i) { return h2d(p[i]); }
template <> __device__ __forceinline__ float load_as<float>(const float* p, int64_t i) { return p[i]; }
template <> __device__ __forceinline__ double load_as<double>(const float* p, int64_t i) { return f2d(p[i]); }
template <> __device__ __forceinline__ float load_as<float>(const double* p, int64_t i) { return d2f(p[i]); }
template <> __device__ __forceinline__ double load_as<double>(const double* p, int64_t i) { return p[i]; }

// Store a compute value with set_linear rounding.
__device__ __forceinline__ void store_from(uint16_t* p, int64_t i, float v) { p[i] = f2h(v); }
__device__ __forceinline__ void store_from(uint16_t* p, int64_t i, double v) { p[i] = d2h(v); }
__device__ __forceinline__ void store_from(float* p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void store_from(float* p, int64_t i, double v) { p[i] = d2f(v); }
__device__ __forceinline__ void store_from(double* p, int64_t i, float v) { p[i] = f2d(v); }
__device__ __forceinline__ void store_from(double* p, int64_t i, double v) { p[i] = v; }

// Non-contracted IEEE arithmetic (the reference never fuses).
__device__ __forceinline__ float op_rn(int op, float x, float y) {
    switch (op) {
        case 0: return __fadd_rn(x, y);
        case 1: return __fsub_rn(x, y);
        case 2: return __fmul_rn(x, y);
        default: return __fdiv_rn(x, y);
    }
}
__device__ __forceinline__ double op_rn(int op, double x, double y) {
    switch (op) {
        case 0: return __dadd_rn(x, y);
        case 1: return __dsub_rn(x, y);
        case 2: return __dmul_rn(x, y);
        default: return __ddiv_rn(x, y);
    }
}

inline int grid_for(int64_t n, int threads, int sm_count, int per_sm = 8) {
    int64_t b = (n + threads - 1) / threads;
    const int64_t cap = static_cast<int64_t>(sm_count) * per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return static_cast<int>(b);
}

}  // namespace mpcr
