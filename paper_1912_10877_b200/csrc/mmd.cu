// mmd.cu — the squared maximum mean discrepancy between the circuit's output distribution
// p = |ψ|² and a target q (SPEC.md:446-449 MMDLoss, 497-505 mmd_expect / mmd_grad; PAPER.md
// §3.2, Listing 12):
//
//     L = Σ_{x,y} K(x,y) (p−q)_x (p−q)_y,   K(x,y) = Σ_σ exp(−(x−y)² / (2σ²))
//
// K depends on |x−y| only (Toeplitz), so K·(p−q) is a 1-D convolution along the basis index
// with the taps w[k] = Σ_σ exp(−k²/(2σ²)).  Beyond k = 38.6·σ_max every tap is exactly 0.0
// in double precision, so the banded sum over |k| ≤ D equals the dense one (never 4^n work).
// The reverse-mode seed is φ̄ = ∂L/∂ψ* = (∂L/∂p) ψ = 2 (K(p−q))_x ψ_x.
//
// One kernel, three modes over a tile of TX basis rows × BC batch columns (batch innermost):
//   LOSS : part_b += d_x · (K d)_x                        (d = |ψ|² − q)
//   SEED : part_b += d_x · (K d)_x,  φ̄_x = 2 (K d)_x ψ_x
//   CROSS: part_b += |a_x|² · (K d)_x                    (a second register; the paper's
//          E_{x∼p_a, y∼p} K(x,y) − E_{x∼p_a, y∼q} K(x,y) of the shift-rule estimator)
// The tile's d values plus a halo of D rows on each side are staged in shared memory; the
// per-batch partial sums reduce in a fixed order (deterministic).
#include <algorithm>

#include "engine.h"

namespace qbg {

namespace {

template <typename V>
__device__ __forceinline__ double abs2(V v) {
    return static_cast<double>(v.x) * static_cast<double>(v.x) + static_cast<double>(v.y) * static_cast<double>(v.y);
}

constexpr int kThreads = 256;

template <typename V, int MODE>
__global__ void __launch_bounds__(kThreads) k_mmd(const V* __restrict__ psi, const V* __restrict__ other,
                                                  V* __restrict__ adj, const double* __restrict__ q,
                                                  const double* __restrict__ w, int D, uint64_t rows, int64_t B,
                                                  int TX, int BC, double* __restrict__ part) {
    extern __shared__ double sm[];
    double* sw = sm;            // D + 1 taps
    double* sd = sm + (D + 1);  // (TX + 2D) x BC values of d
    double* sred = sd + static_cast<size_t>(TX + 2 * D) * BC;  // kThreads partials
    const int tid = threadIdx.x;
    const int64_t nbc = (B + BC - 1) / BC;
    const uint64_t tile = blockIdx.x / nbc;
    const int64_t b0 = static_cast<int64_t>(blockIdx.x % nbc) * BC;
    const int64_t x0 = static_cast<int64_t>(tile) * TX;
    for (int k = tid; k <= D; k += kThreads) sw[k] = w[k];
    const int nload = (TX + 2 * D) * BC;
    for (int i = tid; i < nload; i += kThreads) {
        const int64_t x = x0 - D + i / BC;
        const int64_t b = b0 + i % BC;
        double d = 0.0;
        if (x >= 0 && x < static_cast<int64_t>(rows) && b < B) d = abs2(psi[x * B + b]) - q[x];
        sd[i] = d;
    }
    __syncthreads();
    const int bi = tid % BC;  // every thread keeps one batch column (kThreads % BC == 0)
    const int64_t b = b0 + bi;
    double acc = 0.0;
    for (int r = tid / BC; r < TX; r += kThreads / BC) {
        const int64_t x = x0 + r;
        if (x >= static_cast<int64_t>(rows) || b >= B) continue;
        const double* c = sd + static_cast<size_t>(r + D) * BC + bi;
        double g = sw[0] * c[0];
        for (int k = 1; k <= D; ++k) g = fma(sw[k], c[-static_cast<int64_t>(k) * BC] + c[static_cast<int64_t>(k) * BC], g);
        if (MODE == 2) {
            acc = fma(abs2(other[x * B + b]), g, acc);
        } else {
            acc = fma(c[0], g, acc);
            if (MODE == 1) {
                const V v = psi[x * B + b];
                V o;
                o.x = static_cast<decltype(o.x)>(2.0 * g * static_cast<double>(v.x));
                o.y = static_cast<decltype(o.y)>(2.0 * g * static_cast<double>(v.y));
                adj[x * B + b] = o;
            }
        }
    }
    sred[tid] = acc;
    __syncthreads();
    if (tid < BC && b0 + tid < B) {
        double s = 0.0;
        for (int t = tid; t < kThreads; t += BC) s += sred[t];
        part[static_cast<int64_t>(tile) * B + b0 + tid] = s;
    }
}

}  // namespace

bool mmd_geometry(uint64_t rows, int64_t B, int D, int* TX, int* BC, size_t* smem) {
    int bc = 1;
    while (bc < 32 && bc < B) bc <<= 1;
    for (; bc >= 1; bc >>= 1) {
        const int tx = std::max(8, 1024 / bc);
        const size_t s = (static_cast<size_t>(D) + 1 + static_cast<size_t>(tx + 2 * D) * bc + kThreads) * sizeof(double);
        if (s <= 200 * 1024) {
            *TX = static_cast<int>(std::min<uint64_t>(tx, rows));
            *BC = bc;
            *smem = (static_cast<size_t>(D) + 1 + static_cast<size_t>(*TX + 2 * D) * bc + kThreads) * sizeof(double);
            return true;
        }
    }
    return false;
}

void launch_mmd(int mode, const DevState& psi, const DevState* other, const DevState* adj, const double* d_q,
                const double* d_w, int D, double* d_loss) {
    int TX = 0, BC = 0;
    size_t smem = 0;
    if (!mmd_geometry(psi.rows(), psi.B, D, &TX, &BC, &smem))
        raise(QBG_ERR_UNSUPPORTED, "mmd: kernel bandwidth too wide for the banded convolution (shared memory)");
    const uint64_t ntiles = (psi.rows() + TX - 1) / TX;
    const int64_t nbc = (psi.B + BC - 1) / BC;
    const uint64_t grid = ntiles * static_cast<uint64_t>(nbc);
    double* part = static_cast<double*>(scratch(ntiles * psi.B * sizeof(double), 18));
    {
        const double reads = (mode == 2 ? 2.0 : 1.0) * psi.bytes() + (mode == 1 ? 1.0 : 0.0) * psi.bytes();
        LaunchScope ls(mode == 0 ? "mmd_loss" : mode == 1 ? "mmd_seed" : "mmd_cross", reads);
        auto go = [&](auto tag) {
            using V = decltype(tag);
            auto* kfn = mode == 0 ? k_mmd<V, 0> : mode == 1 ? k_mmd<V, 1> : k_mmd<V, 2>;
            if (smem > 48 * 1024)
                QBG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            kfn<<<static_cast<unsigned>(grid), kThreads, smem, stream()>>>(
                static_cast<const V*>(psi.ptr), other ? static_cast<const V*>(other->ptr) : nullptr,
                adj ? static_cast<V*>(adj->ptr) : nullptr, d_q, d_w, D, psi.rows(), psi.B, TX, BC, part);
        };
        if (psi.dtype == QBG_C128)
            go(double2{});
        else
            go(float2{});
        QBG_CUDA(cudaGetLastError());
    }
    sum_partials(part, static_cast<int64_t>(ntiles), psi.B, d_loss);
}

}  // namespace qbg
