// dense_tc.cu — dense k-qubit blocks (k = 3..5) on the 5th-generation tensor cores (tcgen05,
// kind::tf32, accumulators in TMEM), complex64, with the 3xTF32 split for fp32 accuracy.
//
// The same GEMM as dense_mma.cu (the reference's dense fallback, register.hpp:371-384, over all
// bases at once), oriented for tcgen05: D[m][n] = Σ_k X[m][k] W[n][k] with
//   m = one of 128 state columns (bases x batch) of a CTA tile  -> the 128 TMEM lanes (M = 128),
//   k = the column's 2^k amplitudes as (re, im) floats           -> K = 2^(k+1), steps of 8,
//   n = output amplitude (re, im)                                -> N = 2^(k+1) TMEM columns,
// W = the real 2D x 2D form of U ([[a, -b], [b, a]] blocks).  Plain TF32 keeps 11 bits, far from
// the 1e-5 complex64 contract, so each operand is split into three TF32 pieces x = x0 + x1 + x2 and
// D = x0w0 + (x0w1 + x1w0) + (x0w2 + x1w1 + x2w0): six MMA chains into the same TMEM accumulator,
// every dropped product below 2^-33 — fp32-level (the 2-piece "3xTF32" leaves the truncation of
// the low piece at 2^-22, which drifts the norm by ~5e-5 over 80 blocks at 30 qubits).  FP32 CUDA
// cores would need 8 D flop per amplitude (256 at k = 5: compute-bound at ~75 TFLOP/s); the six
// TF32 tensor-core passes keep the block HBM-bound.
//
// Per 128-column tile (one persistent CTA per SM, 4 warps): the tile is in registers (D float2 per
// thread), split and stored in the canonical no-swizzle K-major layout ([k/4][m][4] floats: 8-row
// x 16-B core matrices, SBO = 128 B, LBO = 128 x 16 B), fenced to the async proxy; one thread
// issues the 6 x K/8 tcgen05.mma and commits to an mbarrier; meanwhile every thread issues the
// NEXT tile's global loads into registers; then each warp reads its 32 TMEM lanes (tcgen05.ld
// 32x32b), stages the rows in shared memory and the CTA scatters them back coalesced.  The W pieces
// are loaded once per CTA.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "engine.h"

namespace qbg {
namespace {

constexpr int kCols = 128;  // state columns per tile = tcgen05 M

struct TcArgs {
    uint64_t ntiles;
    uint8_t qpos[16];   // tile-local bit b -> element bit position (ascending)
    uint8_t qrole[16];  // target q (0..4) or column bit 8 + c
    uint8_t fixpos[64];
    int nfix;
    uint64_t cval;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// canonical K-major, no-swizzle UMMA shared-memory descriptor (Blackwell version 1)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3fff);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3fff) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3fff) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version
    return d;                              // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n}\n"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, float* v) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// accumulators per tile: the K dimension is split over NACC TMEM accumulators summed in registers
// (round to nearest) — each one accumulates fewer steps in the tensor cores' truncating fp32 adder
template <int T>
constexpr int tc_nacc() { return T == 5 ? 4 : 2; }

template <int T>
__global__ void __launch_bounds__(128, 2) k_dense_tc(float2* __restrict__ st, const float* __restrict__ w3,
                                                     const __grid_constant__ TcArgs a) {
    constexpr int D = 1 << T, KR = 2 * D, N = KR, KS = KR / 8;
    constexpr int NACC = tc_nacc<T>();
    constexpr int OS = KR + 4;         // staging row stride (floats)
    constexpr int XSZ = KR * kCols;    // floats of one X piece ([KR/4][128][4])
    constexpr int WSZ = KR * N;        // floats of one W piece ([KR/4][N][4])
    constexpr int PER = D;             // complex elements per thread per tile (D * 128 / 128)
    extern __shared__ __align__(128) unsigned char smraw[];
    float* xs = reinterpret_cast<float*>(smraw);   // X pieces 0..1
    float* ws = xs + 2 * XSZ;                      // W pieces 0..2
    float* out = xs;                               // staging [128][OS], reuses the X pieces after the MMAs
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5;
    constexpr uint32_t cols = NACC * N < 32 ? 32 : NACC * N;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" :: "r"(su32(&tmem_base_s)), "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(su32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int i = tid; i < 3 * WSZ; i += 128) ws[i] = w3[i];
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    // instruction descriptor: D f32, A / B tf32, both K-major, N, M = 128
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | ((128u >> 4) << 24);
    // element e = tid + 128 i of a tile: the low 7 tile bits come from tid, the high T from i, so
    // its offset / column / amplitude split into a per-thread part and a per-i part
    uint64_t off_t = 0;
    int m_t = 0, j_t = 0;
#pragma unroll
    for (int b = 0; b < 7; ++b) {
        const int bit = (tid >> b) & 1;
        off_t |= static_cast<uint64_t>(bit) << a.qpos[b];
        const int r = a.qrole[b];
        if (r >= 8) m_t |= bit << (r - 8); else j_t |= bit << r;
    }
    auto part_i = [&](int i, uint64_t& off, int& m, int& j) {
        off = off_t;
        m = m_t;
        j = j_t;
#pragma unroll
        for (int b = 0; b < T; ++b) {
            const int bit = (i >> b) & 1;
            off |= static_cast<uint64_t>(bit) << a.qpos[7 + b];
            const int r = a.qrole[7 + b];
            if (r >= 8) m |= bit << (r - 8); else j |= bit << r;
        }
    };
    float2 v[PER];
    auto load = [&](uint64_t tile) {
        const uint64_t base = deposit_zeros(tile, a.fixpos, a.nfix) | a.cval;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            uint64_t off;
            int m, j;
            part_i(i, off, m, j);
            v[i] = st[base + off];
        }
    };
    uint32_t phase = 0;
    uint64_t tile = blockIdx.x;
    if (tile < a.ntiles) load(tile);
    for (; tile < a.ntiles; tile += gridDim.x) {
        const uint64_t base = deposit_zeros(tile, a.fixpos, a.nfix) | a.cval;
        // split x = x0 + x1 (tf32 pieces; the second keeps the residual's leading 11 bits) and store
        // them K-major: (re, im) of amplitude j are k = 2j, 2j + 1 -> chunk j / 2, lanes 2 (j & 1) + {0, 1}
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            uint64_t off;
            int m, j;
            part_i(i, off, m, j);
            const float r0 = tf32_rna(v[i].x), i0 = tf32_rna(v[i].y);
            const int o = (((j >> 1) * kCols + m) << 2) + ((j & 1) << 1);
            *reinterpret_cast<float2*>(xs + o) = make_float2(r0, i0);
            *reinterpret_cast<float2*>(xs + XSZ + o) = make_float2(tf32_rna(v[i].x - r0), tf32_rna(v[i].y - i0));
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> tensor-core reads
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            constexpr uint32_t XL = kCols * 16, WL = N * 16;  // LBO: next 16-B K chunk
            const uint32_t x0 = su32(xs), w0 = su32(ws);
            // D = x0 w0 + x0 w1 + x1 w0 + x0 w2 + x1 w1, K split over the NACC accumulators
#pragma unroll
            for (int ac = 0; ac < NACC; ++ac)
#pragma unroll
                for (int pr = 0; pr < 5; ++pr) {
                    const int px = pr == 2 || pr == 4 ? 1 : 0;
                    const int pw = pr == 1 || pr == 4 ? 1 : pr == 3 ? 2 : 0;
#pragma unroll
                    for (int s3 = 0; s3 < KS / NACC; ++s3) {
                        const int s2 = ac * (KS / NACC) + s3;
                        const uint32_t xo = px * XSZ * 4 + s2 * 2 * XL, wo = pw * WSZ * 4 + s2 * 2 * WL;
                        mma_tf32(tmem + ac * N, umma_desc(x0 + xo, XL, 128), umma_desc(w0 + wo, WL, 128), idesc,
                                 pr > 0 || s3 > 0);
                    }
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                         :: "r"(su32(&mbar)) : "memory");
        }
        // the next tile's loads fly while the tensor cores work
        if (tile + gridDim.x < a.ntiles) load(tile + gridDim.x);
        {
            uint32_t done = 0;
            unsigned long long spins = 0;
            while (!done) {
                asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
                             : "=r"(done) : "r"(su32(&mbar)), "r"(phase), "r"(0x989680u) : "memory");
                if (++spins > 4096) __trap();  // ~40 s of suspended waits: a lost commit traps, never hangs
            }
            phase ^= 1u;
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        // TMEM lane tid (warp w reads lanes 32w..32w+31) = tile column tid
        const uint32_t lane_addr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += 16) {
            float r[16];
            tmem_ld16(lane_addr + c0, r);
#pragma unroll
            for (int ac = 1; ac < NACC; ++ac) {
                float r2[16];
                tmem_ld16(lane_addr + ac * N + c0, r2);
#pragma unroll
                for (int q = 0; q < 16; ++q) r[q] += r2[q];
            }
#pragma unroll
            for (int q = 0; q < 16; q += 4)
                *reinterpret_cast<float4*>(out + tid * OS + c0 + q) = make_float4(r[q], r[q + 1], r[q + 2], r[q + 3]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            uint64_t off;
            int m, j;
            part_i(i, off, m, j);
            st[base + off] = *reinterpret_cast<const float2*>(out + m * OS + 2 * j);
        }
        __syncthreads();
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tmem), "r"(cols));
}

float tf32_host(float x) {  // cvt.rna.tf32.f32 on the host: round to 10 mantissa bits, ties away
    uint32_t b;
    std::memcpy(&b, &x, 4);
    b = (b + 0x1000u) & ~0x1fffu;
    float r;
    std::memcpy(&r, &b, 4);
    return r;
}

}  // namespace

// true when the gate ran on tcgen05 (complex64, 3..5 qubits, power-of-two batch, >= 7 free bits)
bool launch_dense_tc(const DevState& s, const Gate& g) {
    if (s.dtype != QBG_C64 || g.t < 3 || g.t > 5 || g.kind != QBG_MAT_DENSE) return false;
    if (s.B & (s.B - 1)) return false;
    int bb = 0;
    while ((int64_t{1} << bb) < s.B) ++bb;
    const int nbits = s.n + bb;
    std::vector<int> colpos;
    for (int p = 0; p < nbits && static_cast<int>(colpos.size()) < 7; ++p) {
        if (p >= bb && (((g.tmask | g.cmask) >> (p - bb)) & 1)) continue;
        colpos.push_back(p);
    }
    if (colpos.size() < 7) return false;
    for (auto& v : g.m)
        if (!std::isfinite(v.re) || !std::isfinite(v.im)) return false;
    const int D = g.dim, KR = 2 * D, N = KR;
    // W[n][k] (real form of U, U_rc = m[c*D + r]) in the [k/4][n][4] layout, split hi / lo
    const size_t wsz = static_cast<size_t>(KR) * N;
    std::vector<float> w3(3 * wsz);  // w = w0 + w1 + w2, each tf32
    auto put = [&](int n, int k, double val) {
        const size_t o = (static_cast<size_t>(k >> 2) * N + n) * 4 + (k & 3);
        const float f = static_cast<float>(val), h = tf32_host(f), r = f - h, m = tf32_host(r);
        w3[o] = h;
        w3[wsz + o] = m;
        w3[2 * wsz + o] = tf32_host(r - m);
    };
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c) {
            const cdbl x = g.m[static_cast<size_t>(c) * D + r];
            put(2 * r, 2 * c, x.re);
            put(2 * r, 2 * c + 1, -x.im);
            put(2 * r + 1, 2 * c, x.im);
            put(2 * r + 1, 2 * c + 1, x.re);
        }
    TcArgs a{};
    std::vector<std::pair<int, int>> tb;
    for (int q = 0; q < g.t; ++q) tb.emplace_back(g.tbit[q] + bb, q);
    for (int c = 0; c < 7; ++c) tb.emplace_back(colpos[c], 8 + c);
    std::sort(tb.begin(), tb.end());
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
    float* dw = static_cast<float*>(scratch(w3.size() * sizeof(float), 22));
    QBG_CUDA(cudaMemcpyAsync(dw, w3.data(), w3.size() * sizeof(float), cudaMemcpyHostToDevice, stream()));
    QBG_CUDA(cudaStreamSynchronize(stream()));  // w3 is a host temporary
    const size_t smem = std::max<size_t>(static_cast<size_t>(2 * KR * kCols + 3 * KR * N) * sizeof(float),
                                         static_cast<size_t>(kCols * (KR + 4)) * sizeof(float));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(a.ntiles, static_cast<uint64_t>(num_sms()) * 2));
    const double cols = static_cast<double>(a.ntiles) * kCols;
    // algorithmic: 2 x 8 B per amplitude; 8 D^2 flop per column (the tensor cores run 6 TF32 products)
    LaunchScope ls("dense_tc", 2.0 * 8.0 * D * cols, 8.0 * D * D * cols);
    static bool attr_set[6] = {false, false, false, false, false, false};
    auto attr = [&](const void* k) {
        if (!attr_set[g.t]) {
            QBG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            attr_set[g.t] = true;
        }
    };
    auto* p = static_cast<float2*>(s.ptr);
    switch (g.t) {
        case 3:
            attr(reinterpret_cast<const void*>(k_dense_tc<3>));
            k_dense_tc<3><<<grid, 128, smem, stream()>>>(p, dw, a);
            break;
        case 4:
            attr(reinterpret_cast<const void*>(k_dense_tc<4>));
            k_dense_tc<4><<<grid, 128, smem, stream()>>>(p, dw, a);
            break;
        default:
            attr(reinterpret_cast<const void*>(k_dense_tc<5>));
            k_dense_tc<5><<<grid, 128, smem, stream()>>>(p, dw, a);
    }
    QBG_CUDA(cudaGetLastError());
    return true;
}

}  // namespace qbg
