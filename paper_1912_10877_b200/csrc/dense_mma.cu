// dense_mma.cu — dense k-qubit blocks (k = 3..5) on the FP64 tensor cores (DMMA), complex128.
//
// The reference's dense fallback (register.hpp:371-384) gathers the 2^k amplitudes of every base
// index and multiplies them by the column-major matrix.  Over all bases that is one GEMM,
//     Y (2^k x N) = U (2^k x 2^k) · X (2^k x N),   N = 2^(n-k) bases x B batch columns,
// so a 5-qubit block is 8 flop per byte of the state (complex128 read + write) — above the B200
// FP64 ridge (~5.6 flop/B): compute-bound, GEMM-shaped, the one place on this path the north star
// puts on FP64 tensor cores.  tcgen05 has no f64 kind; sm_100a keeps the warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), which is what this kernel issues.
//
// Complex as real: with K ordered (re, im) per amplitude, the real 2D x 2D matrix has 2x2 blocks
// [[a, -b], [b, a]] for U_rc = a + ib, and the state tile of a column is its 2^k complex amplitudes
// read as 2^(k+1) doubles — no repacking.  Each warp owns 16 columns (two n-tiles of 8): it loads
// them global -> shared (coalesced: the tile's bit set is the targets plus the 4 lowest free bits,
// in ascending order), runs all (M/8) x (K/4) x 2 DMMA with the accumulators in registers, writes
// the results back over its own columns (only __syncwarp — no CTA barrier) and stores them.  The
// real matrix sits in shared memory (row stride padded by 4 doubles: conflict-free fragments).
#include <algorithm>
#include <cmath>
#include <type_traits>
#include <vector>

#include "engine.h"

namespace qbg {
namespace {

constexpr int kWarps = 8;   // warps per CTA
constexpr int kCols = 16;   // columns (bases x batch) per warp: two 8-wide n-tiles

struct MmaArgs {
    uint64_t ntiles;         // warp tiles over the whole register
    int nq;                  // bits of the tile index deposited around the fixed bits
    uint8_t qpos[16];        // tile-local bit b -> element bit position (ascending)
    uint8_t qrole[16];       // tile-local bit b: target q (0..4) or column bit 8 + c
    int ntile_bits;          // t + 4
    uint8_t fixpos[64];      // element bits the tile index skips (tile bits + controls), ascending
    int nfix;
    uint64_t cval;           // control values (element bit mask)
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// V = double2 (complex128) or float2 (complex64: widened to FP64 in shared memory, one rounding
// on the store — more accurate than an FP32 GEMM and free on an FP64-bound kernel)
template <int T, typename V>
__global__ void __launch_bounds__(kWarps * 32) k_dense_mma(V* __restrict__ st, const double* __restrict__ areal,
                                                          const __grid_constant__ MmaArgs a) {
    constexpr int D = 1 << T, KR = 2 * D, MB = KR / 8, KS = KR / 4;
    constexpr int AS = KR + 4;  // padded row stride (doubles) of the real matrix and of a column
    extern __shared__ __align__(16) double smem[];
    double* sa = smem;                                   // [KR][AS]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* sc = smem + KR * AS + warp * kCols * AS;     // this warp's columns [kCols][AS]
    for (int i = threadIdx.x; i < KR * KR; i += blockDim.x) sa[(i / KR) * AS + (i % KR)] = areal[i];
    __syncthreads();
    constexpr int NE = D * kCols;  // complex elements per warp tile
    const uint64_t wstride = static_cast<uint64_t>(gridDim.x) * kWarps;
    for (uint64_t tile = static_cast<uint64_t>(blockIdx.x) * kWarps + warp; tile < a.ntiles; tile += wstride) {
        const uint64_t base = deposit_zeros(tile, a.fixpos, a.nfix) | a.cval;
        // element e of the tile: its tile-local bits placed at qpos; smem slot (column c, amplitude j)
        auto where = [&](int e, uint64_t& off, int& slot) {
            off = 0;
            int c = 0, j = 0;
#pragma unroll
            for (int b = 0; b < T + 4; ++b) {
                const int bit = (e >> b) & 1;
                off |= static_cast<uint64_t>(bit) << a.qpos[b];
                const int r = a.qrole[b];
                if (r >= 8) c |= bit << (r - 8); else j |= bit << r;
            }
            slot = c * AS + 2 * j;
        };
#pragma unroll 4
        for (int e = lane; e < NE; e += 32) {
            uint64_t off;
            int slot;
            where(e, off, slot);
            const V v = st[base + off];
            sc[slot] = static_cast<double>(v.x);
            sc[slot + 1] = static_cast<double>(v.y);
        }
        __syncwarp();
        double acc[2][MB][2];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) acc[nt][mb][0] = acc[nt][mb][1] = 0.0;
        const int fr = lane >> 2, fc = lane & 3;  // fragment row / column of this lane
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const double b0 = sc[(0 * 8 + fr) * AS + 4 * ks + fc];
            const double b1 = sc[(1 * 8 + fr) * AS + 4 * ks + fc];
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
                const double av = sa[(8 * mb + fr) * AS + 4 * ks + fc];
                dmma(acc[0][mb][0], acc[0][mb][1], av, b0);
                dmma(acc[1][mb][0], acc[1][mb][1], av, b1);
            }
        }
        __syncwarp();  // every lane's fragment reads of the columns are done: overwrite in place
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
                // D fragment: row 8 mb + fr (output real index), columns 8 nt + 2 fc + {0, 1}
                sc[(8 * nt + 2 * fc) * AS + 8 * mb + fr] = acc[nt][mb][0];
                sc[(8 * nt + 2 * fc + 1) * AS + 8 * mb + fr] = acc[nt][mb][1];
            }
        __syncwarp();
#pragma unroll 4
        for (int e = lane; e < NE; e += 32) {
            uint64_t off;
            int slot;
            where(e, off, slot);
            V r;
            r.x = static_cast<typename real_of<V>::type>(sc[slot]);
            r.y = static_cast<typename real_of<V>::type>(sc[slot + 1]);
            st[base + off] = r;
        }
        __syncwarp();
    }
}

}  // namespace

// true when the gate ran on the tensor-core kernel (dense-able 3..5-qubit gate, power-of-two batch,
// finite matrix, enough free bits for a 16-column warp tile); complex64 computes in FP64 too
bool launch_dense_mma(const DevState& s, const Gate& g) {
    if (g.t < 3 || g.t > 5 || g.kind == QBG_MAT_IDENTITY) return false;
    if (s.B & (s.B - 1)) return false;
    int bb = 0;
    while ((int64_t{1} << bb) < s.B) ++bb;
    const int nbits = s.n + bb;  // element index bits: batch lowest, then rows
    uint64_t fixed_rows = g.tmask | g.cmask;
    // column bits: the 4 lowest element bits that are neither targets nor controls
    std::vector<int> colpos;
    for (int p = 0; p < nbits && static_cast<int>(colpos.size()) < 4; ++p) {
        const bool is_row = p >= bb;
        if (is_row && ((fixed_rows >> (p - bb)) & 1)) continue;
        colpos.push_back(p);
    }
    if (colpos.size() < 4) return false;
    const int D = g.dim;
    std::vector<cdbl> u(static_cast<size_t>(D) * D, cdbl{0, 0});  // column-major u[c*D + r]
    if (g.kind == QBG_MAT_DENSE) {
        u = g.m;
    } else if (g.kind == QBG_MAT_DIAGONAL) {
        for (int r = 0; r < D; ++r) u[r * D + r] = g.m[r];
    } else {
        for (int r = 0; r < D; ++r) u[g.perm[r] * D + r] = g.m[r];
    }
    for (auto& v : u)
        if (!std::isfinite(v.re) || !std::isfinite(v.im)) return false;  // keep the reference's x == 0 skip
    const int KR = 2 * D;
    std::vector<double> ar(static_cast<size_t>(KR) * KR);
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c) {
            const cdbl x = u[static_cast<size_t>(c) * D + r];
            ar[(2 * r) * KR + 2 * c] = x.re;
            ar[(2 * r) * KR + 2 * c + 1] = -x.im;
            ar[(2 * r + 1) * KR + 2 * c] = x.im;
            ar[(2 * r + 1) * KR + 2 * c + 1] = x.re;
        }
    MmaArgs a{};
    // tile bits: targets (element position tbit[q] + bb, role q) and columns (role 8 + c), ascending
    std::vector<std::pair<int, int>> tb;
    for (int q = 0; q < g.t; ++q) tb.emplace_back(g.tbit[q] + bb, q);
    for (int c = 0; c < 4; ++c) tb.emplace_back(colpos[c], 8 + c);
    std::sort(tb.begin(), tb.end());
    a.ntile_bits = static_cast<int>(tb.size());
    uint64_t fixmask = 0;
    for (size_t b = 0; b < tb.size(); ++b) {
        a.qpos[b] = static_cast<uint8_t>(tb[b].first);
        a.qrole[b] = static_cast<uint8_t>(tb[b].second);
        fixmask |= uint64_t{1} << tb[b].first;
    }
    for (int p = 0; p < s.n; ++p)
        if ((g.cmask >> p) & 1) fixmask |= uint64_t{1} << (p + bb);
    a.nfix = 0;
    for (int p = 0; p < nbits; ++p)
        if ((fixmask >> p) & 1) a.fixpos[a.nfix++] = static_cast<uint8_t>(p);
    a.cval = g.cval << bb;
    a.ntiles = (uint64_t{1} << nbits) >> a.nfix;
    double* d_ar = static_cast<double*>(scratch(ar.size() * sizeof(double), 21));
    QBG_CUDA(cudaMemcpyAsync(d_ar, ar.data(), ar.size() * sizeof(double), cudaMemcpyHostToDevice, stream()));
    const int AS = KR + 4;
    const size_t smem = static_cast<size_t>(KR * AS + kWarps * kCols * AS) * sizeof(double);
    const uint64_t want = (a.ntiles + kWarps - 1) / kWarps;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(want, static_cast<uint64_t>(num_sms()) * 2));
    // algorithmic work of the processed columns: 2 x element bytes per amplitude, 8 D^2 flop per column
    const double cols = static_cast<double>(a.ntiles) * kCols;
    LaunchScope ls("dense_mma", 2.0 * s.elem() * D * cols, 8.0 * D * D * cols);
    auto go = [&](auto* p) {
        using V = std::remove_pointer_t<decltype(p)>;
        static bool attr_set[6] = {false, false, false, false, false, false};
        auto run = [&](auto kern) {
            if (!attr_set[g.t]) {
                QBG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(smem)));
                attr_set[g.t] = true;
            }
            kern<<<grid, kWarps * 32, smem, stream()>>>(p, d_ar, a);
        };
        if (g.t == 3) run(k_dense_mma<3, V>);
        else if (g.t == 4) run(k_dense_mma<4, V>);
        else run(k_dense_mma<5, V>);
    };
    if (s.dtype == QBG_C128)
        go(static_cast<double2*>(s.ptr));
    else
        go(static_cast<float2*>(s.ptr));
    QBG_CUDA(cudaGetLastError());
    return true;
}

}  // namespace qbg
