// kernels.cu — per-gate kernels, reductions and elementwise helpers.
//
// The per-gate kernel is the device form of the reference's instruct kernel
// (register.hpp:352-385): one thread per (base index, batch column), the base index obtained
// in closed form by inserting zero bits at the target/control positions (the reference's
// subset walk for_each_base, register.hpp:343-350), controls fixed through cval
// (make_plan, 299-339).  Batch is innermost, so a warp reads 32 consecutive batch columns
// (B >= 32) or 32 consecutive base indices (B == 1): every access is a full 128-B line for
// every target stride.  Used for single instruct calls and as the fallback of the fused
// engine (fused.cu) for gates it does not tile (t >= 3).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "engine.h"

namespace qbg {

namespace {

constexpr int kInline = 64;  // complex entries carried in the kernel parameter block

struct GateArgs {
    uint64_t nunits;  // number of (base, batch) units
    int64_t B;
    int bshift;  // log2(B) when B is a power of two, else -1
    int nfix;
    uint8_t fixpos[64];
    uint64_t cval;
    int64_t offB[32];   // element offset of sub-index k (= off[k]*B)
    int64_t poffB[32];  // element offset of sub-index perm[k]
    cdbl inl[kInline];
    const cdbl* ext;  // dense payload for dim > 8
};

GateArgs make_args(const DevState& s, const Gate& g) {
    GateArgs a;
    std::memset(&a, 0, sizeof(a));
    a.B = s.B;
    a.bshift = (s.B & (s.B - 1)) == 0 ? __builtin_ctzll(static_cast<uint64_t>(s.B)) : -1;
    uint64_t fix = g.tmask | g.cmask;
    a.nfix = 0;
    for (int p = 0; p < 64; ++p)
        if ((fix >> p) & 1) a.fixpos[a.nfix++] = static_cast<uint8_t>(p);
    a.nunits = (s.rows() >> a.nfix) * static_cast<uint64_t>(s.B);
    a.cval = g.cval;
    for (int k = 0; k < g.dim; ++k) {
        uint64_t o = 0;
        for (int q = 0; q < g.t; ++q)
            if ((k >> q) & 1) o |= uint64_t{1} << g.tbit[q];
        a.offB[k] = static_cast<int64_t>(o) * s.B;
    }
    if (g.kind == QBG_MAT_PERMUTATION)
        for (int k = 0; k < g.dim; ++k) a.poffB[k] = a.offB[g.perm[k]];
    if (static_cast<int>(g.m.size()) <= kInline) {
        std::copy(g.m.begin(), g.m.end(), a.inl);
        a.ext = nullptr;
    } else {
        void* d = scratch(g.m.size() * sizeof(cdbl), 7);
        QBG_CUDA(cudaMemcpyAsync(d, g.m.data(), g.m.size() * sizeof(cdbl), cudaMemcpyHostToDevice, stream()));
        a.ext = static_cast<const cdbl*>(d);
    }
    return a;
}

__device__ __forceinline__ void split_unit(const GateArgs& a, uint64_t u, uint64_t& r, uint64_t& b) {
    if (a.bshift >= 0) {
        r = u >> a.bshift;
        b = u & ((uint64_t{1} << a.bshift) - 1);
    } else {
        r = u / static_cast<uint64_t>(a.B);
        b = u - r * static_cast<uint64_t>(a.B);
    }
}

template <typename V, int T>
__device__ __forceinline__ V mat_at(const GateArgs& a, int idx) {
    if constexpr ((1 << T) * (1 << T) <= kInline) {
        return from_cd<V>(a.inl[idx]);
    } else {
        return from_cd<V>(a.ext[idx]);
    }
}

// y = U x on one gathered sub-vector (x, y may alias only for DIAG)
template <typename V, int T, int KIND>
__device__ __forceinline__ void apply_sub(const GateArgs& a, V* x, V* y) {
    constexpr int D = 1 << T;
    if constexpr (KIND == QBG_MAT_DIAGONAL) {
#pragma unroll
        for (int k = 0; k < D; ++k) y[k] = cmul(x[k], from_cd<V>(a.inl[k]));
    } else if constexpr (KIND == QBG_MAT_PERMUTATION) {
        // x was gathered in permuted order (poffB), so row k reads x[k]
#pragma unroll
        for (int k = 0; k < D; ++k) y[k] = cmul(from_cd<V>(a.inl[k]), x[k]);
    } else {
#pragma unroll
        for (int r = 0; r < D; ++r) {
            V acc = mk<V>(0, 0);
#pragma unroll
            for (int j = 0; j < D; ++j) {
                // the reference's dense path skips exactly-zero inputs (register.hpp:379): a
                // non-finite matrix column then contributes nothing where x == 0 (select, no branch)
                const V t = cfma(acc, mat_at<V, T>(a, j * D + r), x[j]);
                const bool zero = x[j].x == 0 && x[j].y == 0;
                acc.x = zero ? acc.x : t.x;
                acc.y = zero ? acc.y : t.y;
            }
            y[r] = acc;
        }
    }
}

template <typename V, int T, int KIND>
__global__ void __launch_bounds__(256) k_gate(V* __restrict__ st, const __grid_constant__ GateArgs a) {
    constexpr int D = 1 << T;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < a.nunits; u += stride) {
        uint64_t r, b;
        split_unit(a, u, r, b);
        uint64_t base = deposit_zeros(r, a.fixpos, a.nfix) | a.cval;
        V* p = st + base * static_cast<uint64_t>(a.B) + b;
        V x[D], y[D];
#pragma unroll
        for (int k = 0; k < D; ++k) x[k] = p[KIND == QBG_MAT_PERMUTATION ? a.poffB[k] : a.offB[k]];
        apply_sub<V, T, KIND>(a, x, y);
#pragma unroll
        for (int k = 0; k < D; ++k) p[a.offB[k]] = y[k];
    }
}

// ---- reverse step (fallback of fused.cu's backward tiles) ---------------------------------
struct KArgs {
    int kind;          // 0 none, DIAGONAL or DENSE
    const cdbl* ext;   // dense generators wider than 3 qubits (32 x 32 at t = 5) live in global memory
    cdbl m[64];
};

template <int T>
__device__ __forceinline__ cdbl k_at(const KArgs& k, int idx) {
    if constexpr ((1 << T) * (1 << T) <= 64) {
        return k.m[idx];
    } else {
        return k.ext[idx];
    }
}

template <typename V, int T>
__device__ __forceinline__ double grad_term(const KArgs& k, const V* ps, const V* ad) {
    constexpr int D = 1 << T;
    double s = 0.0;
    if (k.kind == QBG_MAT_DIAGONAL) {
#pragma unroll
        for (int r = 0; r < D; ++r) {
            V kp = cmul(from_cd<V>(k.m[r]), ps[r]);
            s += static_cast<double>(ad[r].x) * kp.y - static_cast<double>(ad[r].y) * kp.x;
        }
    } else if (k.kind == QBG_MAT_DENSE) {
#pragma unroll
        for (int r = 0; r < D; ++r) {
            V kp = mk<V>(0, 0);
#pragma unroll
            for (int j = 0; j < D; ++j) kp = cfma(kp, from_cd<V>(k_at<T>(k, j * D + r)), ps[j]);
            s += static_cast<double>(ad[r].x) * kp.y - static_cast<double>(ad[r].y) * kp.x;
        }
    }
    return s;
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (blockDim.x + 31) / 32; ++k) t += red[k];
    __syncthreads();
    return t;
}

template <typename V, int T, int KIND>
__global__ void __launch_bounds__(256)
    k_gate_back(V* __restrict__ psi, V* __restrict__ adj, const __grid_constant__ GateArgs a,
                const __grid_constant__ KArgs kk, double* __restrict__ partials) {
    constexpr int D = 1 << T;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    double g = 0.0;
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < a.nunits; u += stride) {
        uint64_t r, b;
        split_unit(a, u, r, b);
        uint64_t base = deposit_zeros(r, a.fixpos, a.nfix) | a.cval;
        uint64_t e0 = base * static_cast<uint64_t>(a.B) + b;
        V xp[D], xa[D], y[D];
        // gather once in the order apply_sub reads (permuted for PERMUTATION); the gradient term
        // needs the natural order, which for DENSE / DIAGONAL is the same registers
#pragma unroll
        for (int k = 0; k < D; ++k) {
            int64_t o = KIND == QBG_MAT_PERMUTATION ? a.poffB[k] : a.offB[k];
            xp[k] = psi[e0 + o];
            xa[k] = adj[e0 + o];
        }
        if (kk.kind) {
            if constexpr (KIND == QBG_MAT_PERMUTATION) {
                V ps[D], ad[D];
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    ps[k] = psi[e0 + a.offB[k]];
                    ad[k] = adj[e0 + a.offB[k]];
                }
                g += grad_term<V, T>(kk, ps, ad);
            } else {
                g += grad_term<V, T>(kk, xp, xa);
            }
        }
        apply_sub<V, T, KIND>(a, xp, y);
#pragma unroll
        for (int k = 0; k < D; ++k) psi[e0 + a.offB[k]] = y[k];
        apply_sub<V, T, KIND>(a, xa, y);
#pragma unroll
        for (int k = 0; k < D; ++k) adj[e0 + a.offB[k]] = y[k];
    }
    if (partials) {
        double t = block_sum(g);
        if (threadIdx.x == 0) partials[blockIdx.x] = t;
    }
}

int grid_for(uint64_t units, int block) {
    uint64_t want = (units + block - 1) / block;
    uint64_t cap = static_cast<uint64_t>(num_sms()) * 8;
    return static_cast<int>(std::max<uint64_t>(1, std::min(want, cap)));
}

template <typename V, int T>
void dispatch_kind(const DevState& s, const Gate& g, const GateArgs& a) {
    int grid = grid_for(a.nunits, 256);
    V* p = static_cast<V*>(s.ptr);
    LaunchScope ls("gate", 2.0 * s.bytes());
    switch (g.kind) {
        case QBG_MAT_DIAGONAL:
            k_gate<V, T, QBG_MAT_DIAGONAL><<<grid, 256, 0, stream()>>>(p, a);
            break;
        case QBG_MAT_PERMUTATION:
            k_gate<V, T, QBG_MAT_PERMUTATION><<<grid, 256, 0, stream()>>>(p, a);
            break;
        default:
            k_gate<V, T, QBG_MAT_DENSE><<<grid, 256, 0, stream()>>>(p, a);
    }
    QBG_CUDA(cudaGetLastError());
}

template <typename V>
void dispatch_t(const DevState& s, const Gate& g) {
    GateArgs a = make_args(s, g);
    switch (g.t) {
        case 1: dispatch_kind<V, 1>(s, g, a); break;
        case 2: dispatch_kind<V, 2>(s, g, a); break;
        case 3: dispatch_kind<V, 3>(s, g, a); break;
        case 4: dispatch_kind<V, 4>(s, g, a); break;
        case 5: dispatch_kind<V, 5>(s, g, a); break;
        default: raise(QBG_ERR_UNSUPPORTED, "instruct: more than 5 targets");
    }
}

template <typename V, int T>
void dispatch_back_kind(const DevState& psi, const DevState& adj, const Gate& g, const GateArgs& a, const KArgs& kk,
                        double* partials, int grid) {
    V* p = static_cast<V*>(psi.ptr);
    V* q = static_cast<V*>(adj.ptr);
    LaunchScope ls("gate_back", 4.0 * psi.bytes());
    switch (g.kind) {
        case QBG_MAT_DIAGONAL:
            k_gate_back<V, T, QBG_MAT_DIAGONAL><<<grid, 256, 0, stream()>>>(p, q, a, kk, partials);
            break;
        case QBG_MAT_PERMUTATION:
            k_gate_back<V, T, QBG_MAT_PERMUTATION><<<grid, 256, 0, stream()>>>(p, q, a, kk, partials);
            break;
        default:
            k_gate_back<V, T, QBG_MAT_DENSE><<<grid, 256, 0, stream()>>>(p, q, a, kk, partials);
    }
    QBG_CUDA(cudaGetLastError());
}

template <typename V>
void dispatch_back(const DevState& psi, const DevState& adj, const Gate& g, const Gate* K, double* partials,
                   int64_t cap, int* used) {
    GateArgs a = make_args(psi, g);
    KArgs kk;
    std::memset(&kk, 0, sizeof(kk));
    if (K) {
        if (K->kind == QBG_MAT_DIAGONAL || K->kind == QBG_MAT_IDENTITY) {
            kk.kind = QBG_MAT_DIAGONAL;
            for (int r = 0; r < K->dim; ++r) kk.m[r] = K->kind == QBG_MAT_IDENTITY ? cdbl{1, 0} : K->m[r];
        } else {
            kk.kind = QBG_MAT_DENSE;
            std::vector<cdbl> dn(static_cast<size_t>(K->dim) * K->dim, cdbl{0, 0});
            if (K->kind == QBG_MAT_DENSE) {
                dn = K->m;
            } else {  // permutation -> dense
                for (int r = 0; r < K->dim; ++r) dn[K->perm[r] * K->dim + r] = K->m[r];
            }
            if (dn.size() <= 64) {
                std::copy(dn.begin(), dn.end(), kk.m);
            } else {  // 4- and 5-qubit generators: stream-ordered copy to a library scratch slot
                void* d = scratch(dn.size() * sizeof(cdbl), 20);
                QBG_CUDA(cudaMemcpyAsync(d, dn.data(), dn.size() * sizeof(cdbl), cudaMemcpyHostToDevice, stream()));
                QBG_CUDA(cudaStreamSynchronize(stream()));  // dn is a host temporary
                kk.ext = static_cast<const cdbl*>(d);
            }
        }
    }
    int grid = static_cast<int>(std::min<int64_t>(grid_for(a.nunits, 256), cap));
    if (used) *used = grid;
    switch (g.t) {
        case 1: dispatch_back_kind<V, 1>(psi, adj, g, a, kk, partials, grid); break;
        case 2: dispatch_back_kind<V, 2>(psi, adj, g, a, kk, partials, grid); break;
        case 3: dispatch_back_kind<V, 3>(psi, adj, g, a, kk, partials, grid); break;
        case 4: dispatch_back_kind<V, 4>(psi, adj, g, a, kk, partials, grid); break;
        case 5: dispatch_back_kind<V, 5>(psi, adj, g, a, kk, partials, grid); break;
        default: raise(QBG_ERR_UNSUPPORTED, "backward: more than 5 targets");
    }
}

// ---- reductions -----------------------------------------------------------------------------
// Block (BX batch columns x BY rows).  partial[blockIdx.x][b] (2 doubles) for every batch
// column b; the row range of a block is fixed, so the tree is deterministic.
template <typename V, bool SELF>
__global__ void __launch_bounds__(256)
    k_reduce_inner(const V* __restrict__ a, const V* __restrict__ c, uint64_t rows, int64_t B,
                   uint64_t rows_per_block, double2* __restrict__ partial) {
    const int bx = blockDim.x, by = blockDim.y;
    const int64_t b = static_cast<int64_t>(blockIdx.y) * bx + threadIdx.x;
    uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * rows_per_block;
    uint64_t r1 = min(rows, r0 + rows_per_block);
    double sr = 0.0, si = 0.0;
    if (b < B) {
        for (uint64_t r = r0 + threadIdx.y; r < r1; r += by) {
            V x = a[r * B + b];
            if constexpr (SELF) {
                sr += static_cast<double>(x.x) * x.x + static_cast<double>(x.y) * x.y;
            } else {
                V y = c[r * B + b];
                sr += static_cast<double>(x.x) * y.x + static_cast<double>(x.y) * y.y;
                si += static_cast<double>(x.x) * y.y - static_cast<double>(x.y) * y.x;
            }
        }
    }
    __shared__ double2 red[256];
    int tid = threadIdx.y * bx + threadIdx.x;
    red[tid] = make_double2(sr, si);
    __syncthreads();
    for (int h = by / 2; h > 0; h >>= 1) {
        if (threadIdx.y < h) {
            double2 o = red[tid + h * bx];
            red[tid].x += o.x;
            red[tid].y += o.y;
        }
        __syncthreads();
    }
    if (threadIdx.y == 0 && b < B) partial[blockIdx.x * B + b] = red[threadIdx.x];
}

// out[c] = sum_r part[r][c] for (nrows x ncols) doubles, fixed order
__global__ void k_sum_partials(const double* __restrict__ part, int64_t nrows, int64_t ncols, double* __restrict__ out) {
    int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= ncols) return;
    double s = 0.0;
    for (int64_t r = 0; r < nrows; ++r) s += part[r * ncols + c];
    out[c] = s;
}

template <typename V>
__global__ void k_scale(V* st, uint64_t n, double re, double im) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        st[i] = cmul(st[i], mk<V>(re, im));
}

template <typename V>
__global__ void k_axpy(V* y, const V* x, uint64_t n, double re, double im) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        y[i] = cfma(y[i], mk<V>(re, im), x[i]);
}

// y[i, b] (+)= c_b x[i, b] with one complex coefficient per batch column (Krylov bases)
template <typename V>
__global__ void k_axpy_b(V* y, const V* x, uint64_t n, int64_t B, const double* __restrict__ coef, bool overwrite) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int64_t b = B == 1 ? 0 : static_cast<int64_t>(i % static_cast<uint64_t>(B));
        const V c = mk<V>(coef[2 * b], coef[2 * b + 1]);
        y[i] = overwrite ? cmul(c, x[i]) : cfma(y[i], c, x[i]);
    }
}

template <typename V>
__global__ void k_set_basis(V* st, uint64_t rows, int64_t B, const uint64_t* bits, int64_t nbits) {
    uint64_t total = rows * B;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t r = i / B, b = i - r * B;
        uint64_t want = bits[nbits == 1 ? 0 : b];
        st[i] = mk<V>(r == want ? 1 : 0, 0);
    }
}

// reference layout (batch slowest) <-> device layout (batch innermost), tiled transpose
template <typename V>
__global__ void k_transpose(const V* __restrict__ src, V* __restrict__ dst, uint64_t rows, int64_t B, bool to_dev) {
    __shared__ V tile[32][33];
    // source viewed as matrix [R][C]: to_dev: src is [B][rows] -> dst [rows][B]
    uint64_t R = to_dev ? static_cast<uint64_t>(B) : rows, C = to_dev ? rows : static_cast<uint64_t>(B);
    uint64_t c0 = static_cast<uint64_t>(blockIdx.x) * 32, r0 = static_cast<uint64_t>(blockIdx.y) * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        uint64_t r = r0 + k, c = c0 + threadIdx.x;
        if (r < R && c < C) tile[k][threadIdx.x] = src[r * C + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        uint64_t c = c0 + k, r = r0 + threadIdx.x;
        if (r < R && c < C) dst[c * R + r] = tile[threadIdx.x][k];
    }
}

// phi (+)= c * P psi,  (P psi)[i] = (-1)^{|(i^x)&z|} psi[i^x]   (i^{nY} folded into c)
template <typename V>
__global__ void k_pauli_axpy(const V* __restrict__ psi, V* __restrict__ phi, uint64_t rows, int64_t B, uint64_t xm,
                             uint64_t zm, double cre, double cim, bool overwrite) {
    uint64_t total = rows * B;
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t i = B == 1 ? e : e / B;
        uint64_t b = e - i * B;
        uint64_t j = i ^ xm;
        V v = psi[j * B + b];
        double s = (__popcll(j & zm) & 1) ? -1.0 : 1.0;
        V t = cmul(mk<V>(cre * s, cim * s), v);
        phi[e] = overwrite ? t : cadd(phi[e], t);
    }
}

struct PermArgs {
    int n;
    int8_t new_of_old[64];
};

template <typename V>
__global__ void k_permute(const V* __restrict__ src, V* __restrict__ dst, uint64_t rows, int64_t B,
                          const __grid_constant__ PermArgs pa) {
    uint64_t total = rows * B;
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t g = B == 1 ? e : e / B;
        uint64_t b = e - g * B;
        uint64_t ng = 0;
        for (int k = 0; k < pa.n; ++k) ng |= ((g >> k) & 1) << pa.new_of_old[k];
        dst[ng * B + b] = src[e];
    }
}

// p[i] = sum_env |psi(i + env*2^a, b)|^2 with unfused products (bit-exact with the
// reference's std::norm built with -ffp-contract=off, register.hpp:421)
template <typename V>
__global__ void k_probabilities(const V* __restrict__ st, uint64_t rows_active, uint64_t env, int64_t B, int64_t b,
                                double* __restrict__ p) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows_active;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (uint64_t e = 0; e < env; ++e) {
            V v = st[(e * rows_active + i) * B + b];
            double x = v.x, y = v.y;
            acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
        }
        p[i] = acc;
    }
}

template <typename V>
__global__ void k_collapse(V* st, uint64_t rows_active, uint64_t env, int64_t B, int64_t b, uint64_t hit, double inv) {
    uint64_t total = rows_active * env;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t i = k % rows_active;
        V& v = st[k * B + b];
        v = i == hit ? mk<V>(__dmul_rn(static_cast<double>(v.x), inv), __dmul_rn(static_cast<double>(v.y), inv)) : mk<V>(0, 0);
    }
}

int egrid(uint64_t n) { return grid_for(n, 256); }

}  // namespace

bool is_diagonal(const Gate& g) { return g.kind == QBG_MAT_DIAGONAL || g.kind == QBG_MAT_IDENTITY; }

Gate adjoint(const Gate& g) {
    Gate a = g;
    if (g.kind == QBG_MAT_DIAGONAL) {
        for (auto& e : a.m) e.im = -e.im;
    } else if (g.kind == QBG_MAT_PERMUTATION) {
        for (int i = 0; i < g.dim; ++i) {
            a.perm[g.perm[i]] = i;
            a.m[g.perm[i]] = cdbl{g.m[i].re, -g.m[i].im};
        }
    } else if (g.kind == QBG_MAT_DENSE) {
        for (int c = 0; c < g.dim; ++c)
            for (int r = 0; r < g.dim; ++r) a.m[r * g.dim + c] = cdbl{g.m[c * g.dim + r].re, -g.m[c * g.dim + r].im};
    }
    return a;
}

namespace {
std::atomic<int> g_dense_path{1};
}
int dense_path() { return g_dense_path.load(); }
void set_dense_path(int p) { g_dense_path.store(p); }

void launch_gate(const DevState& s, const Gate& g) {
    if (g.kind == QBG_MAT_IDENTITY) return;
    // dense 3..5-qubit gates (qbg_set_dense_path): 1 (default) the FP64 tensor cores (dense_mma.cu,
    // complex64 widened to FP64), 2 complex64 on tcgen05 (kind::tf32, 3-piece split, dense_tc.cu;
    // faster than the CUDA cores but the tensor cores' fp32 accumulation drifts the norm by ~6e-7
    // per block, profiles/r02/cfg4_30q_dense_ab_c64.jsonl), 0 the CUDA-core kernel below
    const int path = dense_path();
    if (path == 2 && g.t >= 3 && g.kind == QBG_MAT_DENSE && launch_dense_tc(s, g)) return;
    if (path >= 1 && g.t >= 3 && g.kind == QBG_MAT_DENSE && launch_dense_mma(s, g)) return;
    if (s.dtype == QBG_C128)
        dispatch_t<double2>(s, g);
    else
        dispatch_t<float2>(s, g);
}

void launch_gate_back(const DevState& psi, const DevState& adj, const Gate& gdag, const Gate* K, double* partials,
                      int64_t cap, int* used) {
    // a constant dense 3..5-qubit gate (no gradient term): the uncompute of ψ and of φ̄ are two
    // GEMMs on the tensor cores instead of the register-spilling per-gate reverse kernel
    if (!K && gdag.t >= 3 && gdag.kind == QBG_MAT_DENSE && dense_path() >= 1 && launch_dense_mma(psi, gdag)) {
        if (!launch_dense_mma(adj, gdag)) raise(QBG_ERR_INTERNAL, "dense reverse: adjoint state not accepted");
        if (used) *used = 0;
        return;
    }
    Gate g = gdag;
    if (g.kind == QBG_MAT_IDENTITY) {  // still need the gradient term: apply the identity as a diagonal
        g.kind = QBG_MAT_DIAGONAL;
        g.m.assign(g.dim, cdbl{1, 0});
    }
    if (psi.dtype == QBG_C128)
        dispatch_back<double2>(psi, adj, g, K, partials, cap, used);
    else
        dispatch_back<float2>(psi, adj, g, K, partials, cap, used);
}

void reduce_inner(const DevState& a, const DevState* c, double* d_out) {
    int bx = a.B == 1 ? 1 : 32;
    int by = 256 / bx;
    uint64_t rows = a.rows();
    int gy = static_cast<int>((a.B + bx - 1) / bx);
    uint64_t nblk = std::min<uint64_t>(std::max<uint64_t>(1, rows / 64), static_cast<uint64_t>(num_sms()) * 8 / gy + 1);
    uint64_t rpb = (rows + nblk - 1) / nblk;
    nblk = (rows + rpb - 1) / rpb;
    double* part = static_cast<double*>(scratch(nblk * a.B * sizeof(double2), 1));
    dim3 grid(static_cast<unsigned>(nblk), gy), block(bx, by);
    {
        LaunchScope ls("reduce_inner", (c ? 2.0 : 1.0) * a.bytes());
        if (a.dtype == QBG_C128) {
            if (c)
                k_reduce_inner<double2, false><<<grid, block, 0, stream()>>>(
                    static_cast<const double2*>(a.ptr), static_cast<const double2*>(c->ptr), rows, a.B, rpb,
                    reinterpret_cast<double2*>(part));
            else
                k_reduce_inner<double2, true><<<grid, block, 0, stream()>>>(static_cast<const double2*>(a.ptr), nullptr,
                                                                            rows, a.B, rpb,
                                                                            reinterpret_cast<double2*>(part));
        } else {
            if (c)
                k_reduce_inner<float2, false><<<grid, block, 0, stream()>>>(
                    static_cast<const float2*>(a.ptr), static_cast<const float2*>(c->ptr), rows, a.B, rpb,
                    reinterpret_cast<double2*>(part));
            else
                k_reduce_inner<float2, true><<<grid, block, 0, stream()>>>(static_cast<const float2*>(a.ptr), nullptr,
                                                                           rows, a.B, rpb,
                                                                           reinterpret_cast<double2*>(part));
        }
        QBG_CUDA(cudaGetLastError());
    }
    sum_partials(part, static_cast<int64_t>(nblk), 2 * a.B, d_out);
}

void sum_partials(const double* d_part, int64_t nrows, int64_t ncols, double* d_out) {
    LaunchScope ls("sum_partials", 8.0 * nrows * ncols);
    k_sum_partials<<<static_cast<unsigned>((ncols + 127) / 128), 128, 0, stream()>>>(d_part, nrows, ncols, d_out);
    QBG_CUDA(cudaGetLastError());
}

namespace {
__global__ void k_row_sums(const double* __restrict__ part, int64_t nrows, int64_t cap, double* __restrict__ out) {
    int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    double s = 0.0;
    for (int64_t b = 0; b < cap; ++b) s += part[r * cap + b];
    out[r] = s;
}
__global__ void k_scatter_slots(const double* __restrict__ sums, int64_t nslots, const int* __restrict__ map,
                                double* __restrict__ grads) {
    if (threadIdx.x == 0 && blockIdx.x == 0)
        for (int64_t s = 0; s < nslots; ++s) grads[map[s]] += sums[s];
}
}  // namespace

void accumulate_grads(const double* d_part, int64_t nslots, int64_t cap, const int* d_slot_param, double* d_grads) {
    double* sums = static_cast<double*>(scratch(nslots * sizeof(double), 12));
    {
        LaunchScope ls("grad_rows", 8.0 * nslots * cap);
        k_row_sums<<<static_cast<unsigned>((nslots + 127) / 128), 128, 0, stream()>>>(d_part, nslots, cap, sums);
        QBG_CUDA(cudaGetLastError());
    }
    LaunchScope ls("grad_scatter", 8.0 * nslots);
    k_scatter_slots<<<1, 32, 0, stream()>>>(sums, nslots, d_slot_param, d_grads);
    QBG_CUDA(cudaGetLastError());
}

void launch_scale(const DevState& s, double re, double im) {
    LaunchScope ls("scale", 2.0 * s.bytes());
    if (s.dtype == QBG_C128)
        k_scale<double2><<<egrid(s.count()), 256, 0, stream()>>>(static_cast<double2*>(s.ptr), s.count(), re, im);
    else
        k_scale<float2><<<egrid(s.count()), 256, 0, stream()>>>(static_cast<float2*>(s.ptr), s.count(), re, im);
    QBG_CUDA(cudaGetLastError());
}

void launch_axpy_batch(const DevState& y, const DevState& x, const double* d_coef, bool overwrite) {
    LaunchScope ls("axpy_batch", (overwrite ? 2.0 : 3.0) * y.bytes());
    if (y.dtype == QBG_C128)
        k_axpy_b<double2><<<egrid(y.count()), 256, 0, stream()>>>(static_cast<double2*>(y.ptr),
                                                                  static_cast<const double2*>(x.ptr), y.count(), y.B,
                                                                  d_coef, overwrite);
    else
        k_axpy_b<float2><<<egrid(y.count()), 256, 0, stream()>>>(static_cast<float2*>(y.ptr),
                                                                 static_cast<const float2*>(x.ptr), y.count(), y.B,
                                                                 d_coef, overwrite);
    QBG_CUDA(cudaGetLastError());
}

void launch_axpy(const DevState& y, const DevState& x, double re, double im) {
    LaunchScope ls("axpy", 3.0 * y.bytes());
    if (y.dtype == QBG_C128)
        k_axpy<double2><<<egrid(y.count()), 256, 0, stream()>>>(static_cast<double2*>(y.ptr),
                                                               static_cast<const double2*>(x.ptr), y.count(), re, im);
    else
        k_axpy<float2><<<egrid(y.count()), 256, 0, stream()>>>(static_cast<float2*>(y.ptr),
                                                              static_cast<const float2*>(x.ptr), y.count(), re, im);
    QBG_CUDA(cudaGetLastError());
}

void launch_set_basis(const DevState& s, const uint64_t* d_bits, int64_t nbits) {
    LaunchScope ls("set_basis", 1.0 * s.bytes());
    if (s.dtype == QBG_C128)
        k_set_basis<double2><<<egrid(s.count()), 256, 0, stream()>>>(static_cast<double2*>(s.ptr), s.rows(), s.B,
                                                                     d_bits, nbits);
    else
        k_set_basis<float2><<<egrid(s.count()), 256, 0, stream()>>>(static_cast<float2*>(s.ptr), s.rows(), s.B, d_bits,
                                                                    nbits);
    QBG_CUDA(cudaGetLastError());
}

void launch_transpose(const void* src, void* dst, uint64_t rows, int64_t B, int dtype, bool to_dev) {
    uint64_t R = to_dev ? static_cast<uint64_t>(B) : rows, C = to_dev ? rows : static_cast<uint64_t>(B);
    dim3 grid(static_cast<unsigned>((C + 31) / 32), static_cast<unsigned>((R + 31) / 32)), block(32, 8);
    LaunchScope ls("transpose", 2.0 * rows * B * (dtype == QBG_C128 ? 16 : 8));
    if (dtype == QBG_C128)
        k_transpose<double2><<<grid, block, 0, stream()>>>(static_cast<const double2*>(src), static_cast<double2*>(dst),
                                                           rows, B, to_dev);
    else
        k_transpose<float2><<<grid, block, 0, stream()>>>(static_cast<const float2*>(src), static_cast<float2*>(dst),
                                                          rows, B, to_dev);
    QBG_CUDA(cudaGetLastError());
}

void launch_pauli_axpy(const DevState& psi, const DevState& phi, uint64_t xmask, uint64_t zmask, double cre, double cim,
                       bool overwrite) {
    LaunchScope ls("pauli_axpy", (overwrite ? 2.0 : 3.0) * psi.bytes());
    if (psi.dtype == QBG_C128)
        k_pauli_axpy<double2><<<egrid(psi.count()), 256, 0, stream()>>>(
            static_cast<const double2*>(psi.ptr), static_cast<double2*>(phi.ptr), psi.rows(), psi.B, xmask, zmask, cre,
            cim, overwrite);
    else
        k_pauli_axpy<float2><<<egrid(psi.count()), 256, 0, stream()>>>(static_cast<const float2*>(psi.ptr),
                                                                       static_cast<float2*>(phi.ptr), psi.rows(), psi.B,
                                                                       xmask, zmask, cre, cim, overwrite);
    QBG_CUDA(cudaGetLastError());
}

void launch_permute_bits(const DevState& src, const DevState& dst, const int* new_of_old) {
    PermArgs pa;
    pa.n = src.n;
    for (int k = 0; k < src.n; ++k) pa.new_of_old[k] = static_cast<int8_t>(new_of_old[k]);
    LaunchScope ls("permute_bits", 2.0 * src.bytes());
    if (src.dtype == QBG_C128)
        k_permute<double2><<<egrid(src.count()), 256, 0, stream()>>>(static_cast<const double2*>(src.ptr),
                                                                     static_cast<double2*>(dst.ptr), src.rows(), src.B,
                                                                     pa);
    else
        k_permute<float2><<<egrid(src.count()), 256, 0, stream()>>>(static_cast<const float2*>(src.ptr),
                                                                    static_cast<float2*>(dst.ptr), src.rows(), src.B,
                                                                    pa);
    QBG_CUDA(cudaGetLastError());
}

void launch_probabilities(const DevState& s, int nactive, int64_t batch, double* d_p) {
    uint64_t ra = uint64_t{1} << nactive, env = uint64_t{1} << (s.n - nactive);
    LaunchScope ls("probabilities", static_cast<double>(s.rows()) * s.elem());
    if (s.dtype == QBG_C128)
        k_probabilities<double2><<<egrid(ra), 256, 0, stream()>>>(static_cast<const double2*>(s.ptr), ra, env, s.B,
                                                                  batch, d_p);
    else
        k_probabilities<float2><<<egrid(ra), 256, 0, stream()>>>(static_cast<const float2*>(s.ptr), ra, env, s.B,
                                                                 batch, d_p);
    QBG_CUDA(cudaGetLastError());
}

void launch_collapse(const DevState& s, int nactive, int64_t batch, uint64_t hit, double inv) {
    uint64_t ra = uint64_t{1} << nactive, env = uint64_t{1} << (s.n - nactive);
    LaunchScope ls("collapse", 2.0 * s.rows() * s.elem());
    if (s.dtype == QBG_C128)
        k_collapse<double2><<<egrid(ra * env), 256, 0, stream()>>>(static_cast<double2*>(s.ptr), ra, env, s.B, batch,
                                                                   hit, inv);
    else
        k_collapse<float2><<<egrid(ra * env), 256, 0, stream()>>>(static_cast<float2*>(s.ptr), ra, env, s.B, batch,
                                                                  hit, inv);
    QBG_CUDA(cudaGetLastError());
}

}  // namespace qbg
