// krylov.cu — multi-vector kernels of the Lanczos time evolution (capi.cu qbg_time_evolve;
// SPEC.md:397-405).  Re-orthogonalising w against the whole basis one vector at a time costs
// 2k kernels, 2k host round trips and reads w 2k times; these read w once per chunk of 8 basis
// vectors and produce all k projections (or apply all k corrections) in one launch.
#include <algorithm>
#include <cstring>

#include "engine.h"

namespace qbg {

namespace {

constexpr int kChunk = 8;
constexpr int kMaxVec = 64;

struct VecPtrs {
    const void* v[kMaxVec];
};
struct Coefs {
    double c[2 * kMaxVec];  // complex coefficient per basis vector (single batch column)
};

// partial[blk][2i..2i+1] = Σ_{e in block} conj(v_i[e]) w[e], i in [i0, i0 + nv)
template <typename V>
__global__ void __launch_bounds__(256) k_multi_inner(const V* __restrict__ w, VecPtrs vp, int i0, int nv, uint64_t n,
                                                     double* __restrict__ partial, int ld) {
    double ar[kChunk], ai[kChunk];
#pragma unroll
    for (int i = 0; i < kChunk; ++i) ar[i] = ai[i] = 0.0;
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const V x = w[e];
#pragma unroll
        for (int i = 0; i < kChunk; ++i) {
            if (i >= nv) break;
            const V v = static_cast<const V*>(vp.v[i0 + i])[e];
            ar[i] += static_cast<double>(v.x) * x.x + static_cast<double>(v.y) * x.y;
            ai[i] += static_cast<double>(v.x) * x.y - static_cast<double>(v.y) * x.x;
        }
    }
    __shared__ double red[256];
    for (int i = 0; i < nv; ++i) {
        for (int part = 0; part < 2; ++part) {
            red[threadIdx.x] = part ? ai[i] : ar[i];
            __syncthreads();
            for (int h = blockDim.x / 2; h > 0; h >>= 1) {
                if (static_cast<int>(threadIdx.x) < h) red[threadIdx.x] += red[threadIdx.x + h];
                __syncthreads();
            }
            if (threadIdx.x == 0) partial[static_cast<size_t>(blockIdx.x) * ld + 2 * (i0 + i) + part] = red[0];
            __syncthreads();
        }
    }
}

// w[e] += Σ_i c_i v_i[e]
template <typename V>
__global__ void k_multi_axpy(V* __restrict__ w, VecPtrs vp, Coefs cf, int k, uint64_t n) {
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double xr = w[e].x, xi = w[e].y;
        for (int i = 0; i < k; ++i) {
            const V v = static_cast<const V*>(vp.v[i])[e];
            const double cr = cf.c[2 * i], ci = cf.c[2 * i + 1];
            xr += cr * v.x - ci * v.y;
            xi += cr * v.y + ci * v.x;
        }
        V o;
        o.x = static_cast<decltype(o.x)>(xr);
        o.y = static_cast<decltype(o.y)>(xi);
        w[e] = o;
    }
}

unsigned blocks_for(uint64_t n) {
    return static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(num_sms()) * 4));
}

}  // namespace

void multi_inner(const DevState& w, const std::vector<DevState>& vs, double* d_out) {
    const int k = static_cast<int>(vs.size());
    if (k > kMaxVec) raise(QBG_ERR_UNSUPPORTED, "krylov: too many basis vectors");
    if (w.B != 1) raise(QBG_ERR_UNSUPPORTED, "krylov: multi-vector kernels need one batch column");
    VecPtrs vp{};
    for (int i = 0; i < k; ++i) vp.v[i] = vs[i].ptr;
    const uint64_t n = w.count();
    const unsigned nb = blocks_for(n);
    // sized for the largest basis at once: a growing basis must not re-allocate (sync + free) per step
    double* part = static_cast<double*>(scratch(static_cast<size_t>(nb) * 2 * kMaxVec * sizeof(double), 19));
    for (int i0 = 0; i0 < k; i0 += kChunk) {
        const int nv = std::min(kChunk, k - i0);
        LaunchScope ls("krylov_inner", (1.0 + nv) * w.bytes());
        if (w.dtype == QBG_C128)
            k_multi_inner<double2><<<nb, 256, 0, stream()>>>(static_cast<const double2*>(w.ptr), vp, i0, nv, n, part,
                                                             2 * k);
        else
            k_multi_inner<float2><<<nb, 256, 0, stream()>>>(static_cast<const float2*>(w.ptr), vp, i0, nv, n, part,
                                                            2 * k);
        QBG_CUDA(cudaGetLastError());
    }
    sum_partials(part, nb, 2 * k, d_out);
}

void multi_axpy(const DevState& w, const std::vector<DevState>& vs, const std::vector<double>& coef) {
    const int k = static_cast<int>(vs.size());
    if (k > kMaxVec) raise(QBG_ERR_UNSUPPORTED, "krylov: too many basis vectors");
    VecPtrs vp{};
    Coefs cf{};
    for (int i = 0; i < k; ++i) {
        vp.v[i] = vs[i].ptr;
        cf.c[2 * i] = coef[2 * i];
        cf.c[2 * i + 1] = coef[2 * i + 1];
    }
    const uint64_t n = w.count();
    LaunchScope ls("krylov_axpy", (2.0 + k) * w.bytes());
    if (w.dtype == QBG_C128)
        k_multi_axpy<double2><<<blocks_for(n), 256, 0, stream()>>>(static_cast<double2*>(w.ptr), vp, cf, k, n);
    else
        k_multi_axpy<float2><<<blocks_for(n), 256, 0, stream()>>>(static_cast<float2*>(w.ptr), vp, cf, k, n);
    QBG_CUDA(cudaGetLastError());
}

}  // namespace qbg
