// sparse.cu — a full-register sparse operator on the device: the reference's Cached block
// (Listings 6-7) applies its matrix with matvec_cols over SparseColumns
// (matrix.hpp:680-724).  Here the matrix is kept in CSR (converted once from the reference's
// column-major CSC on the host) so every output amplitude is one gather over its row: no atomics,
// deterministic, and batch-innermost columns read coalesced.
#include <algorithm>

#include "engine.h"

namespace qbg {

namespace {

template <typename V>
__global__ void k_spmv(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                       const double2* __restrict__ val, const V* __restrict__ x, V* __restrict__ y, uint64_t rows,
                       int64_t B) {
    const uint64_t n = rows * static_cast<uint64_t>(B);
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = B == 1 ? e : e / static_cast<uint64_t>(B);
        const int64_t b = B == 1 ? 0 : static_cast<int64_t>(e - r * static_cast<uint64_t>(B));
        double sr = 0.0, si = 0.0;
        for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
            const double2 a = val[k];
            const V v = x[static_cast<int64_t>(col[k]) * B + b];
            sr = fma(a.x, static_cast<double>(v.x), fma(-a.y, static_cast<double>(v.y), sr));
            si = fma(a.x, static_cast<double>(v.y), fma(a.y, static_cast<double>(v.x), si));
        }
        V o;
        o.x = static_cast<decltype(o.x)>(sr);
        o.y = static_cast<decltype(o.y)>(si);
        y[e] = o;
    }
}

}  // namespace

void launch_spmv(const DevState& x, const DevState& y, const int64_t* d_rowptr, const int32_t* d_col,
                 const double* d_val, int64_t nnz) {
    LaunchScope ls("spmv", 2.0 * x.bytes() + static_cast<double>(nnz) * 20.0);
    const uint64_t n = x.count();
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(num_sms()) * 8));
    if (x.dtype == QBG_C128)
        k_spmv<double2><<<grid, 256, 0, stream()>>>(d_rowptr, d_col, reinterpret_cast<const double2*>(d_val),
                                                     static_cast<const double2*>(x.ptr), static_cast<double2*>(y.ptr),
                                                     x.rows(), x.B);
    else
        k_spmv<float2><<<grid, 256, 0, stream()>>>(d_rowptr, d_col, reinterpret_cast<const double2*>(d_val),
                                                    static_cast<const float2*>(x.ptr), static_cast<float2*>(y.ptr),
                                                    x.rows(), x.B);
    QBG_CUDA(cudaGetLastError());
}

}  // namespace qbg
