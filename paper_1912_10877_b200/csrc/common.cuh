// common.cuh — shared device/host helpers for the qbg engine (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/qbg.h"

namespace qbg {

// ---- errors: qblock::Error hierarchy (errors.hpp:24-81) mapped onto QBG_ERR_* -----------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

#define QBG_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (call);                                                                \
        if (_e != cudaSuccess)                                                                  \
            ::qbg::raise(QBG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));   \
    } while (0)

// ---- complex arithmetic on CUDA vector types ---------------------------------------------
// c128 = double2, c64 = float2; accumulations of reductions are always done in double.
template <typename V>
struct real_of;
template <>
struct real_of<double2> {
    using type = double;
};
template <>
struct real_of<float2> {
    using type = float;
};

template <typename V>
__host__ __device__ __forceinline__ V mk(typename real_of<V>::type r, typename real_of<V>::type i) {
    V v;
    v.x = r;
    v.y = i;
    return v;
}
template <typename V>
__host__ __device__ __forceinline__ V cmul(V a, V b) {
    return mk<V>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a + b*c
template <typename V>
__host__ __device__ __forceinline__ V cfma(V a, V b, V c) {
    return mk<V>(a.x + b.x * c.x - b.y * c.y, a.y + b.x * c.y + b.y * c.x);
}
template <typename V>
__host__ __device__ __forceinline__ V cadd(V a, V b) {
    return mk<V>(a.x + b.x, a.y + b.y);
}
template <typename V>
__host__ __device__ __forceinline__ V cconj(V a) {
    return mk<V>(a.x, -a.y);
}
template <typename V>
__host__ __device__ __forceinline__ V cscale(V a, typename real_of<V>::type s) {
    return mk<V>(a.x * s, a.y * s);
}

// Complex constant stored in double precision in kernel parameters / device tables.
struct cdbl {
    double re, im;
};
template <typename V>
__host__ __device__ __forceinline__ V from_cd(cdbl c) {
    return mk<V>(static_cast<typename real_of<V>::type>(c.re), static_cast<typename real_of<V>::type>(c.im));
}

// Inserts a zero bit at every set position of `mask` (ascending) into x: maps a dense
// counter onto the base indices whose masked bits are all zero (the reference's subset
// walk, register.hpp:343-350, in closed form).
__host__ __device__ __forceinline__ uint64_t deposit_zeros(uint64_t x, const uint8_t* pos, int npos) {
    for (int k = 0; k < npos; ++k) {
        uint64_t low = x & ((uint64_t{1} << pos[k]) - 1);
        x = ((x >> pos[k]) << (pos[k] + 1)) | low;
    }
    return x;
}

// ---- launch accounting + optional per-kernel CUDA-event timing -------------------------------
void note_launch(const char* name, double bytes);  // host; counts and (if enabled) times
struct LaunchScope {
    const char* name;
    double bytes;
    LaunchScope(const char* n, double b, double flops = 0.0);
    ~LaunchScope();
};

cudaStream_t stream();
int num_sms();

}  // namespace qbg
