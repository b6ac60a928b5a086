// fused.cu — the tiled multi-gate engine (forward, adjoint, reverse-AD and observable seed).
//
// Why this shape (B200, complex128): one gate is 8 flop/element against 32 B of HBM traffic,
// so a per-gate kernel is HBM-bound at ~0.16 ms per 25-qubit gate and the 2050-gate apply+grad
// costs ~0.5 s at the per-gate roofline.  Fusing every gate whose non-diagonal targets fall in
// the tile's qubit set into one pass trades HBM passes for FP64 work done in registers: the
// pass is bound by max(HBM time of its tiles, FP64 time of its gates, smem time of its
// transposes).  Diagonal gates and controls never force a qubit into the tile: they read the
// element's global index bits from wherever they live (register / thread / tile-outer bits).
//
// Reverse pass: consecutive uncontrolled 1-qubit gates on one qubit (the Rz·Rx·Rz rotor of the
// variational circuit) are uncomputed as ONE 2x2 and their gradients come from one 2x2 cross
// matrix C_ab = Σ conj(φ̄_a) ψ_b taken before the uncompute:  θ̄_k = Im Σ_ab (W_k K_k W_k†)_ab C_ab
// with W_k the product of the run's gates after k (derivation in DESIGN.md §AD).  Gradients
// are reduced per warp into shared cells, per CTA into a partials buffer, then in a fixed
// order: deterministic for a given grid.
// See fused.h for the tile/stage vocabulary and DESIGN.md for the roofline numbers.
#include <algorithm>
#include <array>
#include <cstring>
#include <map>
#include <memory>

#include "fused.h"
#include "program.h"

namespace qbg {

using namespace fz;

// =====================================================================================
// device side
// =====================================================================================
namespace {

constexpr int kMaxOps = 256;    // ops per pass (smem resident)
constexpr int kMaxMats = 512;   // complex matrix entries per pass (smem resident)
constexpr int kMaxComps = 256;  // gradient components per pass

template <typename V>
__device__ __forceinline__ V ld_mat(const cdbl* m, int i) {
    return from_cd<V>(m[i]);
}

template <typename V>
__device__ __forceinline__ double im_conj_mul(V a, V b) {  // Im(conj(a) * b)
    return static_cast<double>(a.x) * b.y - static_cast<double>(a.y) * b.x;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---- register-slot gate kernels ---------------------------------------------------------
// CHECK = false: no control on register slots (the common case: no per-pair predicate)
template <typename V, int RB, int K, bool CHECK>
__device__ __forceinline__ void dense1_k(V* x, V m00, V m10, V m01, V m11, int cm, int cv) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (j & (1 << K)) continue;
        if (CHECK && (j & cm) != cv) continue;
        V a = x[j], b = x[j | (1 << K)];
        x[j] = cfma(cmul(m00, a), m01, b);
        x[j | (1 << K)] = cfma(cmul(m10, a), m11, b);
    }
}

template <typename V, int RB, int K, bool CHECK>
__device__ __forceinline__ void swap1_k(V* x, int cm, int cv) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (j & (1 << K)) continue;
        if (CHECK && (j & cm) != cv) continue;
        V a = x[j];
        x[j] = x[j | (1 << K)];
        x[j | (1 << K)] = a;
    }
}

// swap on slot K controlled by slot C == CV (all compile time: pure register moves)
template <typename V, int RB, int K, int C, int CV>
__device__ __forceinline__ void cswap1_k(V* x) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (j & (1 << K)) continue;
        if (((j >> C) & 1) != CV) continue;
        V a = x[j];
        x[j] = x[j | (1 << K)];
        x[j | (1 << K)] = a;
    }
}

template <typename V, int RB, int K, bool CHECK>
__device__ __forceinline__ void diag1_k(V* x, V d0, V d1, int cm, int cv) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (CHECK && (j & cm) != cv) continue;
        x[j] = cmul(x[j], (j & (1 << K)) ? d1 : d0);
    }
}

template <typename V, int RB, int K0, int K1>
__device__ __forceinline__ void dense2_k(V* x, const cdbl* m, int cm, int cv) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (j & ((1 << K0) | (1 << K1))) continue;
        if ((j & cm) != cv) continue;
        const int i0 = j, i1 = j | (1 << K0), i2 = j | (1 << K1), i3 = j | (1 << K0) | (1 << K1);
        V a0 = x[i0], a1 = x[i1], a2 = x[i2], a3 = x[i3];
        V r[4];
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
            V acc = cmul(ld_mat<V>(m, rr), a0);
            acc = cfma(acc, ld_mat<V>(m, 4 + rr), a1);
            acc = cfma(acc, ld_mat<V>(m, 8 + rr), a2);
            r[rr] = cfma(acc, ld_mat<V>(m, 12 + rr), a3);
        }
        x[i0] = r[0];
        x[i1] = r[1];
        x[i2] = r[2];
        x[i3] = r[3];
    }
}

// gradient terms: Σ Im(conj(adj) * (K psi)) over the thread's elements
template <typename V, int RB, int K>
__device__ __forceinline__ double gdense1_k(const V* p, const V* a, V k00, V k10, V k01, V k11, int cm, int cv) {
    double g = 0.0;
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (j & (1 << K)) continue;
        if ((j & cm) != cv) continue;
        V p0 = p[j], p1 = p[j | (1 << K)];
        g += im_conj_mul(a[j], cfma(cmul(k00, p0), k01, p1));
        g += im_conj_mul(a[j | (1 << K)], cfma(cmul(k10, p0), k11, p1));
    }
    return g;
}

template <typename V, int RB, int K>
__device__ __forceinline__ double gdiag1_k(const V* p, const V* a, V d0, V d1, int cm, int cv) {
    double g = 0.0;
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if ((j & cm) != cv) continue;
        g += im_conj_mul(a[j], cmul((j & (1 << K)) ? d1 : d0, p[j]));
    }
    return g;
}

template <typename V, int RB, int K0, int K1>
__device__ __forceinline__ double gdense2_k(const V* p, const V* a, const cdbl* m, int cm, int cv) {
    double g = 0.0;
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (j & ((1 << K0) | (1 << K1))) continue;
        if ((j & cm) != cv) continue;
        const int idx[4] = {j, j | (1 << K0), j | (1 << K1), j | (1 << K0) | (1 << K1)};
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
            V acc = cmul(ld_mat<V>(m, rr), p[idx[0]]);
            acc = cfma(acc, ld_mat<V>(m, 4 + rr), p[idx[1]]);
            acc = cfma(acc, ld_mat<V>(m, 8 + rr), p[idx[2]]);
            acc = cfma(acc, ld_mat<V>(m, 12 + rr), p[idx[3]]);
            g += im_conj_mul(a[idx[rr]], acc);
        }
    }
    return g;
}

// C_ab = Σ conj(adj_a) psi_b over pairs on slot K: c[2*(2a+b)] = Re, c[2*(2a+b)+1] = Im
template <typename V, int RB, int K>
__device__ __forceinline__ void gcross1_k(const V* p, const V* a, double* c) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (j & (1 << K)) continue;
        const V av[2] = {a[j], a[j | (1 << K)]};
        const V pv[2] = {p[j], p[j | (1 << K)]};
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y) {
                c[2 * (2 * x + y)] += static_cast<double>(av[x].x) * pv[y].x + static_cast<double>(av[x].y) * pv[y].y;
                c[2 * (2 * x + y) + 1] += static_cast<double>(av[x].x) * pv[y].y - static_cast<double>(av[x].y) * pv[y].x;
            }
    }
}

// Reduce 8 per-lane values over the warp by halving exchanges (9 double shuffles instead of
// 40); returns the full sum of component (lane >> 2) in lanes with lane % 4 == 0.
__device__ __forceinline__ double warp_sum8(double* v, int lane) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const bool hi = lane & 16;
        double send = hi ? v[k] : v[k + 4];
        double keep = hi ? v[k + 4] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const bool hi = lane & 8;
        double send = hi ? v[k] : v[k + 2];
        double keep = hi ? v[k + 2] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
        const bool hi = lane & 4;
        double send = hi ? v[0] : v[1];
        double keep = hi ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    double s = v[0];
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    return s;
}

// runtime slot -> compile-time slot
#define QBG_SLOT_SWITCH(slot, RB, CALL)                         \
    switch (slot) {                                             \
        case 0: CALL(0); break;                                 \
        case 1: if constexpr (RB > 1) { CALL(1); } break;        \
        case 2: if constexpr (RB > 2) { CALL(2); } break;        \
        case 3: if constexpr (RB > 3) { CALL(3); } break;        \
        case 4: if constexpr (RB > 4) { CALL(4); } break;        \
        default: break;                                         \
    }

template <typename V, int RB>
__device__ __forceinline__ void dense2_dispatch(V* x, int a, int b, const cdbl* m, int cm, int cv) {
#define QBG_D2(A, B_)                                                                  \
    if constexpr (A < RB && B_ < RB && A != B_) {                                      \
        if (a == A && b == B_) { dense2_k<V, RB, A, B_>(x, m, cm, cv); return; }       \
    }
    QBG_D2(0, 1) QBG_D2(1, 0) QBG_D2(0, 2) QBG_D2(2, 0) QBG_D2(1, 2) QBG_D2(2, 1)
    QBG_D2(0, 3) QBG_D2(3, 0) QBG_D2(1, 3) QBG_D2(3, 1) QBG_D2(2, 3) QBG_D2(3, 2)
    QBG_D2(0, 4) QBG_D2(4, 0) QBG_D2(1, 4) QBG_D2(4, 1) QBG_D2(2, 4) QBG_D2(4, 2) QBG_D2(3, 4) QBG_D2(4, 3)
#undef QBG_D2
}

template <typename V, int RB>
__device__ __forceinline__ double gdense2_dispatch(const V* p, const V* q, int a, int b, const cdbl* m, int cm, int cv) {
#define QBG_G2(A, B_)                                                              \
    if constexpr (A < RB && B_ < RB && A != B_) {                                  \
        if (a == A && b == B_) return gdense2_k<V, RB, A, B_>(p, q, m, cm, cv);    \
    }
    QBG_G2(0, 1) QBG_G2(1, 0) QBG_G2(0, 2) QBG_G2(2, 0) QBG_G2(1, 2) QBG_G2(2, 1)
    QBG_G2(0, 3) QBG_G2(3, 0) QBG_G2(1, 3) QBG_G2(3, 1) QBG_G2(2, 3) QBG_G2(3, 2)
    QBG_G2(0, 4) QBG_G2(4, 0) QBG_G2(1, 4) QBG_G2(4, 1) QBG_G2(2, 4) QBG_G2(4, 2) QBG_G2(3, 4) QBG_G2(4, 3)
#undef QBG_G2
    return 0.0;
}

// controlled swap with one control on a register slot (CNOT with both ends in registers)
template <typename V, int RB>
__device__ __forceinline__ bool cswap_dispatch(V* x, int k, int c, int cv) {
#define QBG_CS(K, C)                                                                   \
    if constexpr (K < RB && C < RB && K != C) {                                        \
        if (k == K && c == C) {                                                        \
            if (cv) cswap1_k<V, RB, K, C, 1>(x); else cswap1_k<V, RB, K, C, 0>(x);     \
            return true;                                                               \
        }                                                                              \
    }
    QBG_CS(0, 1) QBG_CS(1, 0) QBG_CS(0, 2) QBG_CS(2, 0) QBG_CS(1, 2) QBG_CS(2, 1)
    QBG_CS(0, 3) QBG_CS(3, 0) QBG_CS(1, 3) QBG_CS(3, 1) QBG_CS(2, 3) QBG_CS(3, 2)
    QBG_CS(0, 4) QBG_CS(4, 0) QBG_CS(1, 4) QBG_CS(4, 1) QBG_CS(2, 4) QBG_CS(4, 2) QBG_CS(3, 4) QBG_CS(4, 3)
#undef QBG_CS
    return false;
}

// index of the DIAGK entry for register element j
__device__ __forceinline__ int diagk_index(const DOp& op, int j, int tid, uint64_t outer) {
    int idx = 0;
    for (int q = 0; q < op.t; ++q) {
        uint32_t loc = static_cast<uint32_t>((op.aux >> (8 * q)) & 0xff);
        uint32_t ty = loc >> 6, pos = loc & 63;
        int bit = ty == LOC_REG ? ((j >> pos) & 1) : ty == LOC_THR ? ((tid >> pos) & 1) : static_cast<int>((outer >> pos) & 1);
        idx |= bit << q;
    }
    return idx;
}

template <typename V, int RB, bool BACK>
__device__ __forceinline__ void run_ops(V* x, V* y, const DOp* ops, int b0, int b1, const cdbl* mats, int tid,
                                        uint64_t outer, double* sg, int nw) {
    constexpr int R = 1 << RB;
    const int warp = tid >> 5, lane = tid & 31;
    for (int i = b0; i < b1; ++i) {
        const DOp& op = ops[i];
        const bool ok = ((outer & op.ctile_mask) == op.ctile_val) && ((static_cast<uint32_t>(tid) & op.cthr_mask) == op.cthr_val);
        const int cm = op.creg_mask, cv = op.creg_val;
        const cdbl* m = mats + op.mat;
        switch (op.code) {
            case OP_DENSE1: {
                if (!ok) break;
                V m00 = ld_mat<V>(m, 0), m10 = ld_mat<V>(m, 1), m01 = ld_mat<V>(m, 2), m11 = ld_mat<V>(m, 3);
                if (cm == 0) {
#define QBG_C(K)                                                  \
    dense1_k<V, RB, K, false>(x, m00, m10, m01, m11, 0, 0);       \
    if constexpr (BACK) dense1_k<V, RB, K, false>(y, m00, m10, m01, m11, 0, 0);
                    QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                } else {
#define QBG_C(K)                                                  \
    dense1_k<V, RB, K, true>(x, m00, m10, m01, m11, cm, cv);      \
    if constexpr (BACK) dense1_k<V, RB, K, true>(y, m00, m10, m01, m11, cm, cv);
                    QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                }
                break;
            }
            case OP_X1: {
                if (!ok) break;
                if (cm == 0) {
#define QBG_C(K)                                  \
    swap1_k<V, RB, K, false>(x, 0, 0);            \
    if constexpr (BACK) swap1_k<V, RB, K, false>(y, 0, 0);
                    QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                } else if (__popc(cm) == 1) {
                    const int c = __ffs(cm) - 1;
                    cswap_dispatch<V, RB>(x, op.a, c, cv != 0);
                    if constexpr (BACK) cswap_dispatch<V, RB>(y, op.a, c, cv != 0);
                } else {
#define QBG_C(K)                                  \
    swap1_k<V, RB, K, true>(x, cm, cv);           \
    if constexpr (BACK) swap1_k<V, RB, K, true>(y, cm, cv);
                    QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                }
                break;
            }
            case OP_PERM1: {
                if (!ok) break;
                // y0 = v0 x[p0], y1 = v1 x[p1]: a swap (b = 1) followed by a diagonal
                if (op.b) {
#define QBG_C(K)                                  \
    swap1_k<V, RB, K, true>(x, cm, cv);           \
    if constexpr (BACK) swap1_k<V, RB, K, true>(y, cm, cv);
                    QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                }
                V d0 = ld_mat<V>(m, 0), d1 = ld_mat<V>(m, 1);
#define QBG_C(K)                                          \
    diag1_k<V, RB, K, true>(x, d0, d1, cm, cv);           \
    if constexpr (BACK) diag1_k<V, RB, K, true>(y, d0, d1, cm, cv);
                QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                break;
            }
            case OP_DIAG1R: {
                if (!ok) break;
                V d0 = ld_mat<V>(m, 0), d1 = ld_mat<V>(m, 1);
                if (cm == 0) {
#define QBG_C(K)                                          \
    diag1_k<V, RB, K, false>(x, d0, d1, 0, 0);            \
    if constexpr (BACK) diag1_k<V, RB, K, false>(y, d0, d1, 0, 0);
                    QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                } else {
#define QBG_C(K)                                          \
    diag1_k<V, RB, K, true>(x, d0, d1, cm, cv);           \
    if constexpr (BACK) diag1_k<V, RB, K, true>(y, d0, d1, cm, cv);
                    QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                }
                break;
            }
            case OP_DIAG1T:
            case OP_DIAG1G: {
                if (!ok) break;
                int bit = op.code == OP_DIAG1T ? ((tid >> op.a) & 1) : static_cast<int>((outer >> op.a) & 1);
                V d = ld_mat<V>(m, bit);
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    if ((j & cm) != cv) continue;
                    x[j] = cmul(x[j], d);
                    if constexpr (BACK) y[j] = cmul(y[j], d);
                }
                break;
            }
            case OP_DENSE2: {
                if (!ok) break;
                dense2_dispatch<V, RB>(x, op.a, op.b, m, cm, cv);
                if constexpr (BACK) dense2_dispatch<V, RB>(y, op.a, op.b, m, cm, cv);
                break;
            }
            case OP_DIAGK: {
                if (!ok) break;
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    if ((j & cm) != cv) continue;
                    V d = ld_mat<V>(m, diagk_index(op, j, tid, outer));
                    x[j] = cmul(x[j], d);
                    if constexpr (BACK) y[j] = cmul(y[j], d);
                }
                break;
            }
            case G_CROSS1: {
                if constexpr (BACK) {
                    double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    if (ok) {
#define QBG_C(K) gcross1_k<V, RB, K>(x, y, c);
                        QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                    }
                    double s = warp_sum8(c, lane);
                    if ((lane & 3) == 0) sg[(op.gslot + (lane >> 2)) * nw + warp] += s;
                }
                break;
            }
            default: {
                if constexpr (BACK) {
                    double g = 0.0;
                    if (ok) {
                        if (op.code == G_DENSE1) {
                            V k00 = ld_mat<V>(m, 0), k10 = ld_mat<V>(m, 1), k01 = ld_mat<V>(m, 2), k11 = ld_mat<V>(m, 3);
#define QBG_C(K) g = gdense1_k<V, RB, K>(x, y, k00, k10, k01, k11, cm, cv);
                            QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                        } else if (op.code == G_DIAG1R) {
                            V d0 = ld_mat<V>(m, 0), d1 = ld_mat<V>(m, 1);
#define QBG_C(K) g = gdiag1_k<V, RB, K>(x, y, d0, d1, cm, cv);
                            QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                        } else if (op.code == G_DIAG1U) {
                            int bit = op.b == 0 ? ((tid >> op.a) & 1) : static_cast<int>((outer >> op.a) & 1);
                            V d = ld_mat<V>(m, bit);
                            double sr = 0.0, si = 0.0;  // Σ conj(adj) psi
#pragma unroll
                            for (int j = 0; j < R; ++j) {
                                if ((j & cm) != cv) continue;
                                sr += static_cast<double>(y[j].x) * x[j].x + static_cast<double>(y[j].y) * x[j].y;
                                si += static_cast<double>(y[j].x) * x[j].y - static_cast<double>(y[j].y) * x[j].x;
                            }
                            g = static_cast<double>(d.x) * si + static_cast<double>(d.y) * sr;
                        } else if (op.code == G_DENSE2) {
                            g = gdense2_dispatch<V, RB>(x, y, op.a, op.b, m, cm, cv);
                        } else if (op.code == G_DIAGK) {
#pragma unroll
                            for (int j = 0; j < R; ++j) {
                                if ((j & cm) != cv) continue;
                                V d = ld_mat<V>(m, diagk_index(op, j, tid, outer));
                                g += im_conj_mul(y[j], cmul(d, x[j]));
                            }
                        }
                    }
                    g = warp_sum(g);
                    if (lane == 0) sg[op.gslot * nw + warp] += g;
                }
                break;
            }
        }
    }
}

template <int W>
__device__ __forceinline__ uint32_t sm_thr(const DStage& S, int tid) {
    uint32_t o = 0;
#pragma unroll
    for (int p = 0; p < W; ++p)
        if ((tid >> p) & 1) o ^= S.sthr[p];
    return o;
}
template <int RB>
__device__ __forceinline__ uint32_t sm_reg(const DStage& S, int j) {
    uint32_t o = 0;
#pragma unroll
    for (int k = 0; k < RB; ++k)
        if ((j >> k) & 1) o ^= S.sreg[k];
    return o;
}
template <int W>
__device__ __forceinline__ int64_t g_thr(const DStage& S, int tid) {
    int64_t o = 0;
#pragma unroll
    for (int p = 0; p < W; ++p)
        if ((tid >> p) & 1) o += S.gthr[p];
    return o;
}
template <int RB>
__device__ __forceinline__ int64_t g_reg(const DStage& S, int j) {
    int64_t o = 0;
#pragma unroll
    for (int k = 0; k < RB; ++k)
        if ((j >> k) & 1) o += S.greg[k];
    return o;
}

template <typename V, int M, bool BACK>
constexpr size_t fused_smem_bytes(int ncomps_cells) {
    return (BACK ? 2 : 1) * (sizeof(V) << M) + static_cast<size_t>(ncomps_cells) * 8 + kMaxOps * sizeof(DOp) +
           kMaxMats * sizeof(cdbl);
}

// One pass over the whole state: grid-stride over tiles.
template <typename V, int M, int RB, bool BACK>
__global__ void __launch_bounds__(1 << (M - RB), 2)
    k_fused(V* __restrict__ psi, V* __restrict__ adj, const __grid_constant__ DPass P, const DOp* __restrict__ gops,
            const cdbl* __restrict__ gmats, double* __restrict__ gpart, int64_t gcols) {
    constexpr int R = 1 << RB, W = M - RB, T = 1 << W, NW = T / 32;
    extern __shared__ __align__(16) unsigned char smraw[];
    V* sx = reinterpret_cast<V*>(smraw);
    V* sy = sx + (1 << M);
    unsigned char* p = smraw + (BACK ? 2 : 1) * (sizeof(V) << M);
    DOp* sops = reinterpret_cast<DOp*>(p);
    p += kMaxOps * sizeof(DOp);
    cdbl* smats = reinterpret_cast<cdbl*>(p);
    p += kMaxMats * sizeof(cdbl);
    double* sg = reinterpret_cast<double*>(p);
    const int tid = threadIdx.x;
    {
        const int4* src = reinterpret_cast<const int4*>(gops + P.op_base);
        int4* dst = reinterpret_cast<int4*>(sops);
        for (int i = tid; i < P.nops * 3; i += T) dst[i] = src[i];
        for (int i = tid; i < P.nmats; i += T) smats[i] = gmats[P.mat_base + i];
        if constexpr (BACK)
            for (int i = tid; i < P.ngrad * NW; i += T) sg[i] = 0.0;
        __syncthreads();
    }
    V x[R], y[BACK ? R : 1];
    const int64_t bc = int64_t{1} << P.nb;
    for (uint64_t tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
        const uint64_t o = tile / static_cast<uint64_t>(P.nchunks);
        const uint64_t c = tile - o * static_cast<uint64_t>(P.nchunks);
        const uint64_t outer = deposit_zeros(o, P.qpos, P.mq);
        const int64_t tbase = static_cast<int64_t>(outer) * P.B + static_cast<int64_t>(c) * bc;
        {
            const DStage& S = P.st[0];
            const int64_t gt = tbase + g_thr<W>(S, tid);
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int64_t e = gt + g_reg<RB>(S, j);
                x[j] = psi[e];
                if constexpr (BACK) y[j] = adj[e];
            }
        }
        for (int s = 0; s < P.nstages; ++s) {
            const DStage& S = P.st[s];
            if (s > 0) {
                const DStage& Sp = P.st[s - 1];
                const uint32_t tp = sm_thr<W>(Sp, tid);
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const uint32_t a = tp ^ sm_reg<RB>(Sp, j);
                    sx[a] = x[j];
                    if constexpr (BACK) sy[a] = y[j];
                }
                __syncthreads();
                const uint32_t tc = sm_thr<W>(S, tid);
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const uint32_t a = tc ^ sm_reg<RB>(S, j);
                    x[j] = sx[a];
                    if constexpr (BACK) y[j] = sy[a];
                }
                __syncthreads();
            }
            run_ops<V, RB, BACK>(x, BACK ? y : nullptr, sops, S.op_begin, S.op_end, smats, tid, outer, sg, NW);
        }
        {
            const DStage& S = P.st[P.nstages - 1];
            const int64_t gt = tbase + g_thr<W>(S, tid);
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int64_t e = gt + g_reg<RB>(S, j);
                psi[e] = x[j];
                if constexpr (BACK) adj[e] = y[j];
            }
        }
    }
    if constexpr (BACK) {
        __syncthreads();
        for (int sl = tid; sl < P.ngrad; sl += T) {
            double s = 0.0;
            for (int w = 0; w < NW; ++w) s += sg[sl * NW + w];
            gpart[static_cast<int64_t>(P.grad_base + sl) * gcols + blockIdx.x] = s;
        }
    }
}

// ---- gradient epilogue: partial rows -> parameter gradients (fixed order) ----------------------
struct GradEntry {
    int32_t type;  // 0 scalar component, 1 cross matrix (8 components)
    int32_t comp;
    int32_t param;
    int32_t pad;
    cdbl A[4];     // column-major 2x2, cross entries only
};

__global__ void k_grad_epilogue(const double* __restrict__ sums, const GradEntry* __restrict__ e, int64_t n,
                                double* __restrict__ grads) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int64_t k = 0; k < n; ++k) {
        const GradEntry& g = e[k];
        if (g.type == 0) {
            grads[g.param] += sums[g.comp];
        } else {
            // θ̄ = Im Σ_ab A_ab C_ab, C_ab at comp + 2(2a+b)
            double acc = 0.0;
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b) {
                    const cdbl A = g.A[b * 2 + a];
                    const double cr = sums[g.comp + 2 * (2 * a + b)], ci = sums[g.comp + 2 * (2 * a + b) + 1];
                    acc += A.re * ci + A.im * cr;
                }
            grads[g.param] += acc;
        }
    }
}

__global__ void k_rows(const double* __restrict__ part, int64_t nrows, int64_t cols, double* __restrict__ out) {
    int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    double s = 0.0;
    for (int64_t b = 0; b < cols; ++b) s += part[r * cols + b];
    out[r] = s;
}

// ---- observable seed: phi (+)= Σ_groups Σ_terms c (-1)^{|src & z|} psi[src], src = l ^ xloc ----
struct SPass {
    int32_t mq, nb;
    uint8_t qpos[64];
    int64_t B, nchunks;
    uint64_t ntiles;
    int32_t g0, g1;  // groups of this pass
    int32_t first, last;
};

template <typename V, int M>
__global__ void __launch_bounds__(256)
    k_seed(const V* __restrict__ psi, V* __restrict__ phi, const __grid_constant__ SPass P,
           const SGroup* __restrict__ groups, const STerm* __restrict__ terms, double* __restrict__ epart) {
    extern __shared__ __align__(16) unsigned char smraw[];
    V* sp = reinterpret_cast<V*>(smraw);
    constexpr int L = 1 << M;
    const int T = blockDim.x;
    const int64_t bc = int64_t{1} << P.nb;
    __shared__ double red[256];
    for (uint64_t tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
        const uint64_t o = tile / static_cast<uint64_t>(P.nchunks);
        const uint64_t c = tile - o * static_cast<uint64_t>(P.nchunks);
        const uint64_t outer = deposit_zeros(o, P.qpos, P.mq);
        const int64_t tbase = static_cast<int64_t>(outer) * P.B + static_cast<int64_t>(c) * bc;
        auto goff = [&](uint32_t l) -> int64_t {
            int64_t e = l & (bc - 1);
            uint32_t q = l >> P.nb;
            for (int k = 0; q; ++k, q >>= 1)
                if (q & 1) e += P.B << P.qpos[k];
            return e;
        };
        __syncthreads();
        for (uint32_t l = threadIdx.x; l < L; l += T) sp[l] = psi[tbase + goff(l)];
        __syncthreads();
        double eacc = 0.0;
        for (uint32_t l = threadIdx.x; l < L; l += T) {
            const int64_t e = tbase + goff(l);
            V acc = P.first ? mk<V>(0, 0) : phi[e];
            for (int gi = P.g0; gi < P.g1; ++gi) {
                const SGroup g = groups[gi];
                const uint32_t src = l ^ g.xloc;
                const V v = sp[src];
                double cr = 0.0, ci = 0.0;
                for (int ti = g.term_begin; ti < g.term_end; ++ti) {
                    const STerm t = terms[ti];
                    const int par = (__popc(src & t.zloc) + __popcll(outer & t.zout)) & 1;
                    cr += par ? -t.cre : t.cre;
                    ci += par ? -t.cim : t.cim;
                }
                acc = cfma(acc, mk<V>(cr, ci), v);
            }
            phi[e] = acc;
            if (P.last) {
                const V pv = sp[l];
                eacc += static_cast<double>(pv.x) * acc.x + static_cast<double>(pv.y) * acc.y;
            }
        }
        if (P.last) {
            red[threadIdx.x] = eacc;
            __syncthreads();
            if (threadIdx.x < bc) {
                double s = 0.0;
                for (int k = threadIdx.x; k < T; k += static_cast<int>(bc)) s += red[k];
                epart[tile * bc + threadIdx.x] = s;
            }
        }
    }
}

// E[b] = Σ_{tiles of chunk b/bc} epart[tile][b % bc]
__global__ void k_energy(const double* __restrict__ epart, uint64_t nouter, int64_t nchunks, int64_t bc, int64_t B,
                         double* __restrict__ e) {
    int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= B) return;
    int64_t c = b / bc, beta = b - c * bc;
    double s = 0.0;
    for (uint64_t o = 0; o < nouter; ++o) s += epart[(o * nchunks + c) * bc + beta];
    e[b] = s;
}

}  // namespace

// =====================================================================================
// host side: planner
// =====================================================================================
namespace {

constexpr int kFwdM = 12, kFwdRB = 4;  // 4096-element tiles, 256 threads x 16 registers
constexpr int kBwdM = 11, kBwdRB = 3;  // two states: 2048-element tiles, 256 threads x 2x8
constexpr int kSeedM = 12;

inline uint32_t swz(uint32_t l) { return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9) ^ (l >> 12) ^ (l >> 15)) & 7u); }

struct RunGrad {  // one gradient of a fused rotation run: θ̄ = Im Σ A_ab C_ab
    int param;
    cdbl A[4];
};

struct PG {  // a gate as the planner sees it
    const Gate* g = nullptr;
    Gate own;  // fused product
    const Gate* k = nullptr;   // scalar gradient generator
    int param = -1;
    std::vector<RunGrad> run;  // cross-matrix gradients of a fused run (backward)
    const Gate& gate() const { return g ? *g : own; }
    uint64_t nd() const { return is_diagonal(gate()) ? 0 : gate().tmask; }
    uint64_t all() const { return gate().tmask | gate().cmask; }
};

std::vector<cdbl> dense_of(const Gate& g) {
    std::vector<cdbl> d(static_cast<size_t>(g.dim) * g.dim, cdbl{0, 0});
    for (int r = 0; r < g.dim; ++r) {
        if (g.kind == QBG_MAT_IDENTITY) d[r * g.dim + r] = cdbl{1, 0};
        if (g.kind == QBG_MAT_DIAGONAL) d[r * g.dim + r] = g.m[r];
        if (g.kind == QBG_MAT_PERMUTATION) d[g.perm[r] * g.dim + r] = g.m[r];
    }
    if (g.kind == QBG_MAT_DENSE) d = g.m;
    return d;
}

cdbl cm(cdbl a, cdbl b) { return cdbl{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
cdbl ca(cdbl a, cdbl b) { return cdbl{a.re + b.re, a.im + b.im}; }
cdbl cc(cdbl a) { return cdbl{a.re, -a.im}; }

using M2 = std::array<cdbl, 4>;  // column-major 2x2
M2 m2_of(const Gate& g) {
    auto d = dense_of(g);
    return {d[0], d[1], d[2], d[3]};
}
M2 m2_mul(const M2& A, const M2& Bm) {
    M2 r{};
    for (int c = 0; c < 2; ++c)
        for (int rr = 0; rr < 2; ++rr)
            r[c * 2 + rr] = ca(cm(A[rr], Bm[c * 2]), cm(A[2 + rr], Bm[c * 2 + 1]));
    return r;
}
M2 m2_dag(const M2& A) { return {cc(A[0]), cc(A[2]), cc(A[1]), cc(A[3])}; }
M2 m2_id() { return {cdbl{1, 0}, cdbl{0, 0}, cdbl{0, 0}, cdbl{1, 0}}; }

// new ∘ old for two 1-qubit gates on the same qubit
Gate compose1(const Gate& nw, const Gate& old) {
    Gate r = old;
    if (is_diagonal(nw) && is_diagonal(old)) {
        r.kind = QBG_MAT_DIAGONAL;
        auto dn = dense_of(nw), dold = dense_of(old);
        r.m = {cm(dn[0], dold[0]), cm(dn[3], dold[3])};
        r.perm.clear();
        return r;
    }
    M2 p = m2_mul(m2_of(nw), m2_of(old));
    r.kind = QBG_MAT_DENSE;
    r.m.assign(p.begin(), p.end());
    r.perm.clear();
    return r;
}

// Fuses consecutive (in dependency order) uncontrolled 1-qubit gates on one qubit.  In the
// reverse pass (backward = true) each merged gate carries its cross-matrix gradient: with the
// run's previously merged uncompute M_prev = V_{k+1}†…V_L†, W_k = M_prev† and A_k = W_k K_k W_k†.
std::vector<PG> fuse_runs(std::vector<PG> in, bool backward) {
    std::vector<PG> out;
    out.reserve(in.size());
    int open[64];
    std::fill(open, open + 64, -1);
    for (auto& pg : in) {
        const Gate& g = pg.gate();
        if (g.kind == QBG_MAT_IDENTITY && g.cmask == 0 && !pg.k) continue;
        if (g.t == 1 && g.cmask == 0) {
            int q = g.tbit[0];
            if (open[q] < 0) {
                out.push_back(std::move(pg));
                PG& o = out.back();
                if (backward && o.k) {
                    // first gate of the run: W = I, A = K
                    RunGrad rg{o.param, {}};
                    M2 K = m2_of(*o.k);
                    std::copy(K.begin(), K.end(), rg.A);
                    o.run.push_back(rg);
                    o.k = nullptr;
                }
                if (backward && o.run.empty()) o.run.reserve(4);
                open[q] = static_cast<int>(out.size()) - 1;
                continue;
            }
            PG& o = out[open[q]];
            if (backward && pg.k) {
                M2 Mp = m2_of(o.gate());  // uncompute so far
                M2 W = m2_dag(Mp);
                M2 A = m2_mul(m2_mul(W, m2_of(*pg.k)), Mp);
                RunGrad rg{pg.param, {}};
                std::copy(A.begin(), A.end(), rg.A);
                o.run.push_back(rg);
            }
            o.own = compose1(g, o.gate());
            o.g = nullptr;
            continue;
        }
        uint64_t touch = g.tmask | g.cmask;
        for (int q = 0; q < 64; ++q)
            if ((touch >> q) & 1) open[q] = -1;
        out.push_back(std::move(pg));
    }
    return out;
}

struct Step {
    bool tile = false;
    DPass pass;
    int single = -1;
    int single_comp = -1;
};

}  // namespace

struct FusedPlan {
    uint64_t version = ~uint64_t{0};
    int64_t B = 0;
    int dtype = -1, n = 0, dir = -1;
    std::vector<PG> gates;
    std::vector<Step> steps;
    std::vector<DOp> ops;
    std::vector<cdbl> mats;
    std::vector<GradEntry> epi;
    int64_t ncomps = 0;
    DOp* d_ops = nullptr;
    cdbl* d_mats = nullptr;
    GradEntry* d_epi = nullptr;
    int64_t tile_passes = 0;
    // observable seed
    std::vector<SPass> spasses;
    std::vector<SGroup> groups;
    std::vector<STerm> terms;
    SGroup* d_groups = nullptr;
    STerm* d_terms = nullptr;
    ~FusedPlan() {
        cudaFree(d_ops);
        cudaFree(d_mats);
        cudaFree(d_epi);
        cudaFree(d_groups);
        cudaFree(d_terms);
    }
};

namespace {

template <class T>
T* upload(const std::vector<T>& v) {
    T* d = nullptr;
    if (v.empty()) return nullptr;
    QBG_CUDA(cudaMalloc(&d, v.size() * sizeof(T)));
    QBG_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

int popc(uint64_t x) { return __builtin_popcountll(x); }

struct TileGeom {
    int M, RB, nb, mq;
    uint64_t Q;
    int local[64];
    int64_t gw[32];
};

TileGeom geom(int M, int RB, int nb, uint64_t Q, int64_t B) {
    TileGeom t{};
    t.M = M;
    t.RB = RB;
    t.nb = nb;
    t.Q = Q;
    t.mq = popc(Q);
    std::fill(t.local, t.local + 64, -1);
    for (int b = 0; b < nb; ++b) t.gw[b] = int64_t{1} << b;
    int k = nb;
    for (int q = 0; q < 64; ++q)
        if ((Q >> q) & 1) {
            t.local[q] = k;
            t.gw[k] = B << q;
            ++k;
        }
    return t;
}

// resources one gate adds to a pass (ops, matrix entries, gradient components), conservative
void gate_cost(const PG& g, int& ops, int& mats, int& comps) {
    const Gate& u = g.gate();
    ops = 1 + (g.k ? 1 : 0) + (g.run.empty() ? 0 : 1);
    mats = u.dim * u.dim + (g.k ? g.k->dim * g.k->dim : 0);
    comps = (g.k ? 1 : 0) + (g.run.empty() ? 0 : 8);
}

// Greedy pass construction (see fused.h): a gate joins the pass when it does not conflict with
// any gate already passed over and its non-diagonal targets fit in the tile qubit set.
void plan_passes(FusedPlan& pl, int M, int RB, int nb, bool backward) {
    const int n = pl.n;
    const int mq = M - nb;
    const uint64_t full = n >= 64 ? ~uint64_t{0} : (uint64_t{1} << n) - 1;
    uint64_t Qc = 0;  // coalescing: local bits 0..2 must be contiguous in memory
    for (int b = 0; b < 3 - nb; ++b) Qc |= uint64_t{1} << b;
    std::vector<int> remaining(pl.gates.size());
    for (size_t i = 0; i < remaining.size(); ++i) remaining[i] = static_cast<int>(i);
    auto tileable = [&](const PG& g) { return g.gate().t <= 2 || is_diagonal(g.gate()); };
    while (!remaining.empty()) {
        // phase 1: grow Q greedily
        uint64_t Q = Qc;
        {
            uint64_t bnd = 0, ball = 0;
            for (int gi : remaining) {
                const PG& g = pl.gates[gi];
                bool conflict = (g.nd() & ball) | (g.all() & bnd);
                if (!tileable(g) || conflict) {
                    bnd |= g.nd();
                    ball |= g.all();
                    continue;
                }
                uint64_t need = g.nd();
                if ((need & ~Q) == 0) continue;
                if (popc(Q | need) <= mq) {
                    Q |= need;
                } else {
                    bnd |= g.nd();
                    ball |= g.all();
                }
            }
        }
        for (int q = n - 1; q >= 0 && popc(Q) < mq; --q) Q |= uint64_t{1} << q;
        Q &= full;
        // phase 2: select with Q fixed, within the pass's smem budgets
        std::vector<int> sel, rest;
        {
            uint64_t bnd = 0, ball = 0;
            int nops = 0, nmats = 0, ncomps = 0;
            for (int gi : remaining) {
                const PG& g = pl.gates[gi];
                bool conflict = (g.nd() & ball) | (g.all() & bnd);
                int co, cmx, cc2;
                gate_cost(g, co, cmx, cc2);
                bool fits = nops + co <= kMaxOps && nmats + cmx <= kMaxMats && ncomps + cc2 <= kMaxComps;
                if (tileable(g) && !conflict && (g.nd() & ~Q) == 0 && fits) {
                    sel.push_back(gi);
                    nops += co;
                    nmats += cmx;
                    ncomps += cc2;
                } else {
                    bnd |= g.nd();
                    ball |= g.all();
                    rest.push_back(gi);
                }
            }
        }
        if (sel.empty()) {
            Step st;
            st.single = remaining.front();
            pl.steps.push_back(st);
            remaining.erase(remaining.begin());
            continue;
        }
        remaining = rest;

        // ---- stages ----
        TileGeom tg = geom(M, RB, nb, Q, pl.B);
        const int R = RB, Wn = M - RB;
        struct StagePlan {
            uint32_t S = 0;  // local register bits
            std::vector<int> gates;
        };
        std::vector<StagePlan> stages;
        StagePlan cur;
        for (int gi : sel) {
            const Gate& g = pl.gates[gi].gate();
            uint32_t need = 0;
            if (!is_diagonal(g))
                for (int q = 0; q < g.t; ++q) need |= 1u << tg.local[g.tbit[q]];
            if ((need & ~cur.S) == 0) {
                cur.gates.push_back(gi);
            } else if (__builtin_popcount(cur.S | need) <= R) {
                cur.S |= need;
                cur.gates.push_back(gi);
            } else {
                stages.push_back(cur);
                cur = StagePlan{};
                cur.S = need;
                cur.gates.push_back(gi);
            }
        }
        stages.push_back(cur);
        if (static_cast<int>(stages.size()) > kMaxStages - 2) {
            std::vector<int> back;
            for (size_t s = kMaxStages - 2; s < stages.size(); ++s)
                back.insert(back.end(), stages[s].gates.begin(), stages[s].gates.end());
            stages.resize(kMaxStages - 2);
            std::vector<int> merged;
            std::sort(back.begin(), back.end());
            std::merge(back.begin(), back.end(), remaining.begin(), remaining.end(), std::back_inserter(merged));
            remaining = merged;
        }
        const uint32_t C = 7u;  // coalescing / bank lane bits
        const uint32_t qbits = ((1u << M) - 1) & ~((1u << nb) - 1);
        auto fill = [&](uint32_t S) {
            for (int b = M - 1; b >= 0 && __builtin_popcount(S) < R; --b)
                if (((qbits >> b) & 1) && !((S >> b) & 1) && !((C >> b) & 1)) S |= 1u << b;
            for (int b = M - 1; b >= 0 && __builtin_popcount(S) < R; --b)
                if (((qbits >> b) & 1) && !((S >> b) & 1)) S |= 1u << b;
            return S;
        };
        for (auto& s : stages) s.S = fill(s.S);
        if (stages.front().S & C) stages.insert(stages.begin(), StagePlan{fill(0), {}});
        if (stages.back().S & C) stages.push_back(StagePlan{fill(0), {}});

        Step step;
        step.tile = true;
        DPass& P = step.pass;
        std::memset(&P, 0, sizeof(P));
        P.nstages = static_cast<int>(stages.size());
        P.mq = mq;
        P.nb = nb;
        {
            int k = 0;
            for (int q = 0; q < 64; ++q)
                if ((Q >> q) & 1) P.qpos[k++] = static_cast<uint8_t>(q);
        }
        P.B = pl.B;
        P.nchunks = pl.B >> nb;
        P.ntiles = (uint64_t{1} << (n - mq)) * static_cast<uint64_t>(P.nchunks);
        P.op_base = static_cast<int>(pl.ops.size());
        P.mat_base = static_cast<int>(pl.mats.size());
        P.grad_base = static_cast<int>(pl.ncomps);
        int ncomp = 0;
        for (int s = 0; s < P.nstages; ++s) {
            const StagePlan& sp = stages[s];
            DStage& D = P.st[s];
            int regb[kMaxR], thrb[kMaxW];
            {
                int k = 0;
                for (int b = 0; b < M; ++b)
                    if ((sp.S >> b) & 1) regb[k++] = b;
            }
            {
                std::vector<int> avail;
                for (int b = 0; b < M; ++b)
                    if (!((sp.S >> b) & 1)) avail.push_back(b);
                std::vector<int> order;
                if ((sp.S & C) == 0) {
                    order = {0, 1, 2};
                } else {
                    bool used[3] = {false, false, false};
                    for (int b : avail)
                        if (!used[b % 3] && order.size() < 3) {
                            used[b % 3] = true;
                            order.push_back(b);
                        }
                }
                for (int b : avail)
                    if (std::find(order.begin(), order.end(), b) == order.end()) order.push_back(b);
                for (int p = 0; p < Wn; ++p) thrb[p] = order[p];
            }
            int slot_of[32], pos_of[32];
            std::fill(slot_of, slot_of + 32, -1);
            std::fill(pos_of, pos_of + 32, -1);
            for (int k = 0; k < R; ++k) {
                slot_of[regb[k]] = k;
                D.sreg[k] = swz(1u << regb[k]);
                D.greg[k] = tg.gw[regb[k]];
            }
            for (int p = 0; p < Wn; ++p) {
                pos_of[thrb[p]] = p;
                D.sthr[p] = swz(1u << thrb[p]);
                D.gthr[p] = tg.gw[thrb[p]];
            }
            D.op_begin = static_cast<int>(pl.ops.size()) - P.op_base;
            for (int gi : sp.gates) {
                const PG& pg = pl.gates[gi];
                const Gate& g = pg.gate();
                DOp base{};
                base.gslot = -1;
                for (int q = 0; q < 64; ++q) {
                    if (!((g.cmask >> q) & 1)) continue;
                    uint32_t v = (g.cval >> q) & 1;
                    int L = tg.local[q];
                    if (L < 0) {
                        base.ctile_mask |= uint64_t{1} << q;
                        base.ctile_val |= static_cast<uint64_t>(v) << q;
                    } else if (slot_of[L] >= 0) {
                        base.creg_mask |= 1u << slot_of[L];
                        base.creg_val |= v << slot_of[L];
                    } else {
                        base.cthr_mask |= 1u << pos_of[L];
                        base.cthr_val |= v << pos_of[L];
                    }
                }
                auto loc_code = [&](int q) -> uint8_t {
                    int L = tg.local[q];
                    if (L < 0) return static_cast<uint8_t>((LOC_TILE << 6) | q);
                    if (slot_of[L] >= 0) return static_cast<uint8_t>((LOC_REG << 6) | slot_of[L]);
                    return static_cast<uint8_t>((LOC_THR << 6) | pos_of[L]);
                };
                auto emit_mat = [&](const std::vector<cdbl>& m) {
                    int off = static_cast<int>(pl.mats.size()) - P.mat_base;
                    pl.mats.insert(pl.mats.end(), m.begin(), m.end());
                    return off;
                };
                // gradient ops first (reverse pass: before the uncompute)
                if (backward && !pg.run.empty()) {
                    DOp o = base;
                    o.code = G_CROSS1;
                    o.a = static_cast<uint8_t>(slot_of[tg.local[g.tbit[0]]]);
                    o.gslot = ncomp;
                    for (const RunGrad& rg : pg.run) {
                        GradEntry e{};
                        e.type = 1;
                        e.comp = static_cast<int>(P.grad_base) + ncomp;
                        e.param = rg.param;
                        std::copy(rg.A, rg.A + 4, e.A);
                        pl.epi.push_back(e);
                    }
                    ncomp += 8;
                    pl.ops.push_back(o);
                }
                if (backward && pg.k) {
                    const Gate& K = *pg.k;
                    DOp o = base;
                    o.gslot = ncomp;
                    GradEntry e{};
                    e.type = 0;
                    e.comp = static_cast<int>(P.grad_base) + ncomp;
                    e.param = pg.param;
                    pl.epi.push_back(e);
                    ncomp += 1;
                    if (is_diagonal(K)) {
                        std::vector<cdbl> d(K.dim);
                        for (int r = 0; r < K.dim; ++r) d[r] = K.kind == QBG_MAT_IDENTITY ? cdbl{1, 0} : K.m[r];
                        if (K.t == 1) {
                            uint8_t lc = loc_code(K.tbit[0]);
                            if ((lc >> 6) == LOC_REG) {
                                o.code = G_DIAG1R;
                                o.a = lc & 63;
                            } else {
                                o.code = G_DIAG1U;
                                o.a = lc & 63;
                                o.b = (lc >> 6) == LOC_TILE ? 1 : 0;
                            }
                        } else {
                            o.code = G_DIAGK;
                            o.t = static_cast<uint8_t>(K.t);
                            for (int q = 0; q < K.t; ++q) o.aux |= static_cast<uint64_t>(loc_code(K.tbit[q])) << (8 * q);
                        }
                        o.mat = emit_mat(d);
                    } else if (K.t == 1) {
                        o.code = G_DENSE1;
                        o.a = static_cast<uint8_t>(slot_of[tg.local[K.tbit[0]]]);
                        o.mat = emit_mat(dense_of(K));
                    } else {
                        o.code = G_DENSE2;
                        o.a = static_cast<uint8_t>(slot_of[tg.local[K.tbit[0]]]);
                        o.b = static_cast<uint8_t>(slot_of[tg.local[K.tbit[1]]]);
                        o.mat = emit_mat(dense_of(K));
                    }
                    pl.ops.push_back(o);
                }
                if (g.kind == QBG_MAT_IDENTITY) continue;
                DOp o = base;
                if (is_diagonal(g)) {
                    if (g.t == 1) {
                        uint8_t lc = loc_code(g.tbit[0]);
                        o.code = (lc >> 6) == LOC_REG ? OP_DIAG1R : (lc >> 6) == LOC_THR ? OP_DIAG1T : OP_DIAG1G;
                        o.a = lc & 63;
                    } else {
                        o.code = OP_DIAGK;
                        o.t = static_cast<uint8_t>(g.t);
                        for (int q = 0; q < g.t; ++q) o.aux |= static_cast<uint64_t>(loc_code(g.tbit[q])) << (8 * q);
                    }
                    o.mat = emit_mat(g.m);
                } else if (g.t == 1) {
                    o.a = static_cast<uint8_t>(slot_of[tg.local[g.tbit[0]]]);
                    if (g.kind == QBG_MAT_PERMUTATION) {
                        bool swapped = g.perm[0] == 1;
                        bool ones = g.m[0].re == 1 && g.m[0].im == 0 && g.m[1].re == 1 && g.m[1].im == 0;
                        if (swapped && ones) {
                            o.code = OP_X1;
                        } else {
                            o.code = OP_PERM1;
                            o.b = swapped ? 1 : 0;
                            o.mat = emit_mat(g.m);
                        }
                    } else {
                        o.code = OP_DENSE1;
                        o.mat = emit_mat(g.m);
                    }
                } else {
                    o.code = OP_DENSE2;
                    o.a = static_cast<uint8_t>(slot_of[tg.local[g.tbit[0]]]);
                    o.b = static_cast<uint8_t>(slot_of[tg.local[g.tbit[1]]]);
                    o.mat = emit_mat(dense_of(g));
                }
                pl.ops.push_back(o);
            }
            D.op_end = static_cast<int>(pl.ops.size()) - P.op_base;
        }
        P.nops = static_cast<int>(pl.ops.size()) - P.op_base;
        P.nmats = static_cast<int>(pl.mats.size()) - P.mat_base;
        P.ngrad = ncomp;
        if (P.nops > kMaxOps || P.nmats > kMaxMats || P.ngrad > kMaxComps)
            raise(QBG_ERR_INTERNAL, "fused plan: pass exceeds its shared-memory budget");
        pl.ncomps += ncomp;
        pl.steps.push_back(step);
        pl.tile_passes++;
    }
}

// ---- execution ---------------------------------------------------------------------------------
template <typename V, int M, int RB, bool BACK>
void launch_fused(V* psi, V* adj, const DPass& P, const FusedPlan& pl, double* gpart, int64_t gcols) {
    constexpr int T = 1 << (M - RB), NW = T / 32;
    constexpr size_t smem_max = fused_smem_bytes<V, M, BACK>(BACK ? kMaxComps * NW : 0);
    static int per_sm = 0;
    auto kern = k_fused<V, M, RB, BACK>;
    if (per_sm == 0) {
        QBG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_max)));
        QBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem_max));
        per_sm = std::max(1, per_sm);
    }
    size_t smem = fused_smem_bytes<V, M, BACK>(BACK ? P.ngrad * NW : 0);
    int64_t grid = std::min<int64_t>(static_cast<int64_t>(P.ntiles), static_cast<int64_t>(num_sms()) * per_sm);
    if (BACK) grid = std::min<int64_t>(grid, gcols);
    double bytes = static_cast<double>(P.ntiles) * (1 << M) * sizeof(V) * (BACK ? 4.0 : 2.0);
    LaunchScope ls(BACK ? "fused_bwd" : "fused_fwd", bytes);
    kern<<<static_cast<unsigned>(grid), T, smem, stream()>>>(psi, adj, P, pl.d_ops, pl.d_mats, gpart, gcols);
    QBG_CUDA(cudaGetLastError());
}

int batch_bits(int64_t B) {
    int nb = 0;
    while (nb < 5 && (B % (int64_t{2} << nb)) == 0) ++nb;
    return nb;
}

std::shared_ptr<FusedPlan> get_plan(std::vector<std::shared_ptr<FusedPlan>>& cache, const Program& p,
                                    const DevState& s, int dir) {
    for (auto& c : cache)
        if (c->dir == dir && c->B == s.B && c->dtype == s.dtype && c->n == s.n && c->version == p.version) return c;
    cache.erase(std::remove_if(cache.begin(), cache.end(),
                               [&](const std::shared_ptr<FusedPlan>& c) { return c->dir == dir && c->B == s.B; }),
                cache.end());
    auto pl = std::make_shared<FusedPlan>();
    pl->version = p.version;
    pl->B = s.B;
    pl->dtype = s.dtype;
    pl->n = s.n;
    pl->dir = dir;
    const size_t N = p.real.size();
    std::vector<PG> gs;
    gs.reserve(N);
    for (size_t q = 0; q < N; ++q) {
        PG g;
        if (dir == 0) {
            g.g = &p.real[q].u;
        } else {
            const RealOp& r = p.real[N - 1 - q];
            g.g = &r.udag;
            if (dir == 2 && r.param >= 0) {
                g.k = &r.k;
                g.param = r.param;
            }
        }
        gs.push_back(std::move(g));
    }
    pl->gates = fuse_runs(std::move(gs), dir == 2);
    const int nb = batch_bits(s.B);
    const int M = dir == 2 ? kBwdM : kFwdM, RB = dir == 2 ? kBwdRB : kFwdRB;
    plan_passes(*pl, M, RB, nb, dir == 2);
    // per-gate fallback steps with a scalar gradient get their own component rows
    for (auto& st : pl->steps)
        if (!st.tile && pl->gates[st.single].k) {
            st.single_comp = static_cast<int>(pl->ncomps++);
            GradEntry e{};
            e.type = 0;
            e.comp = st.single_comp;
            e.param = pl->gates[st.single].param;
            pl->epi.push_back(e);
        } else if (!st.tile && !pl->gates[st.single].run.empty()) {
            raise(QBG_ERR_INTERNAL, "fused plan: untiled rotation run");
        }
    pl->d_ops = upload(pl->ops);
    pl->d_mats = upload(pl->mats);
    pl->d_epi = upload(pl->epi);
    cache.push_back(pl);
    return pl;
}

bool fusable(const DevState& s, int M) {
    int nb = batch_bits(s.B);
    return s.n >= M - nb && s.n <= 62;
}

template <typename V>
void run_forward(const DevState& s, FusedPlan& pl) {
    V* psi = static_cast<V*>(s.ptr);
    for (auto& st : pl.steps) {
        if (st.tile)
            launch_fused<V, kFwdM, kFwdRB, false>(psi, nullptr, st.pass, pl, nullptr, 0);
        else
            launch_gate(s, pl.gates[st.single].gate());
    }
}

template <typename V>
void run_backward(const DevState& psi, const DevState& adj, FusedPlan& pl, double* d_grads) {
    const int64_t cols = static_cast<int64_t>(num_sms()) * 8;
    const int64_t total = pl.ncomps;
    double* part = static_cast<double*>(scratch(std::max<int64_t>(1, total) * cols * sizeof(double), 13));
    if (total) QBG_CUDA(cudaMemsetAsync(part, 0, total * cols * sizeof(double), stream()));
    for (auto& st : pl.steps) {
        if (st.tile) {
            launch_fused<V, kBwdM, kBwdRB, true>(static_cast<V*>(psi.ptr), static_cast<V*>(adj.ptr), st.pass, pl, part,
                                                  cols);
        } else {
            const PG& g = pl.gates[st.single];
            int used = 0;
            launch_gate_back(psi, adj, g.gate(), g.k, g.k ? part + st.single_comp * cols : nullptr, cols, &used);
        }
    }
    if (total) {
        double* sums = static_cast<double*>(scratch(total * sizeof(double), 12));
        {
            LaunchScope ls("grad_rows", 8.0 * total * cols);
            k_rows<<<static_cast<unsigned>((total + 127) / 128), 128, 0, stream()>>>(part, total, cols, sums);
            QBG_CUDA(cudaGetLastError());
        }
        LaunchScope ls("grad_epilogue", 8.0 * total);
        k_grad_epilogue<<<1, 32, 0, stream()>>>(sums, pl.d_epi, static_cast<int64_t>(pl.epi.size()), d_grads);
        QBG_CUDA(cudaGetLastError());
    }
}

}  // namespace

bool fused_forward(const DevState& s, Program& p, bool adjoint) {
    if (!fusable(s, kFwdM)) return false;
    auto pl = get_plan(p.plans, p, s, adjoint ? 1 : 0);
    if (s.dtype == QBG_C128)
        run_forward<double2>(s, *pl);
    else
        run_forward<float2>(s, *pl);
    return true;
}

bool fused_backward(const DevState& psi, const DevState& adj, Program& p, double* d_grads) {
    if (!fusable(psi, kBwdM)) return false;
    auto pl = get_plan(p.plans, p, psi, 2);
    if (psi.dtype == QBG_C128)
        run_backward<double2>(psi, adj, *pl, d_grads);
    else
        run_backward<float2>(psi, adj, *pl, d_grads);
    return true;
}

void fused_stats(const Program& p, int64_t* f, int64_t* b) {
    *f = 0;
    *b = 0;
    for (auto& c : p.plans) {
        int64_t steps = static_cast<int64_t>(c->steps.size());
        if (c->dir == 0) *f = steps;
        if (c->dir == 2) *b = steps;
    }
}

// ---- observable seed ------------------------------------------------------------------------------
namespace {

std::shared_ptr<FusedPlan> get_seed_plan(Observable& o, const DevState& s) {
    for (auto& c : o.plans)
        if (c->B == s.B && c->dtype == s.dtype && c->n == s.n) return c;
    auto pl = std::make_shared<FusedPlan>();
    pl->B = s.B;
    pl->dtype = s.dtype;
    pl->n = s.n;
    pl->dir = 3;
    const int nb = batch_bits(s.B);
    const int mq = kSeedM - nb;
    const int n = s.n;
    uint64_t Qc = 0;
    for (int b = 0; b < 3 - nb; ++b) Qc |= uint64_t{1} << b;
    std::map<uint64_t, std::vector<int>> byx;
    std::vector<uint64_t> order;
    for (size_t t = 0; t < o.terms.size(); ++t) {
        uint64_t x = o.terms[t].xmask;
        if (!byx.count(x)) order.push_back(x);
        byx[x].push_back(static_cast<int>(t));
    }
    std::vector<uint64_t> left = order;
    bool first = true;
    while (!left.empty()) {
        uint64_t Q = Qc;
        std::vector<uint64_t> take, rest;
        for (uint64_t x : left) {
            if (popc(x) > mq) raise(QBG_ERR_UNSUPPORTED, "observable term wider than a tile");
            if (popc(Q | x) <= mq) {
                Q |= x;
                take.push_back(x);
            } else {
                rest.push_back(x);
            }
        }
        for (int q = n - 1; q >= 0 && popc(Q) < mq; --q) Q |= uint64_t{1} << q;
        TileGeom tg = geom(kSeedM, 0, nb, Q, s.B);
        SPass sp{};
        sp.mq = mq;
        sp.nb = nb;
        int k = 0;
        for (int q = 0; q < 64; ++q)
            if ((Q >> q) & 1) sp.qpos[k++] = static_cast<uint8_t>(q);
        sp.B = s.B;
        sp.nchunks = s.B >> nb;
        sp.ntiles = (uint64_t{1} << (n - mq)) * static_cast<uint64_t>(sp.nchunks);
        sp.g0 = static_cast<int>(pl->groups.size());
        for (uint64_t x : take) {
            SGroup g{};
            for (int q = 0; q < 64; ++q)
                if ((x >> q) & 1) g.xloc |= 1u << tg.local[q];
            g.term_begin = static_cast<int>(pl->terms.size());
            for (int t : byx[x]) {
                const qbg_pauli_term& pt = o.terms[t];
                STerm st{};
                st.cre = pt.coef_re;
                st.cim = pt.coef_im;
                for (int q = 0; q < 64; ++q) {
                    if (!((pt.zmask >> q) & 1)) continue;
                    if (tg.local[q] >= 0)
                        st.zloc |= 1u << tg.local[q];
                    else
                        st.zout |= uint64_t{1} << q;
                }
                pl->terms.push_back(st);
            }
            g.term_end = static_cast<int>(pl->terms.size());
            pl->groups.push_back(g);
        }
        sp.g1 = static_cast<int>(pl->groups.size());
        sp.first = first ? 1 : 0;
        first = false;
        pl->spasses.push_back(sp);
        left = rest;
    }
    if (!pl->spasses.empty()) pl->spasses.back().last = 1;
    pl->d_groups = upload(pl->groups);
    pl->d_terms = upload(pl->terms);
    o.plans.push_back(pl);
    return pl;
}

template <typename V>
void run_seed(const DevState& psi, const DevState& phi, FusedPlan& pl, double* d_energy) {
    constexpr int T = 256;
    size_t smem = sizeof(V) << kSeedM;
    auto kern = k_seed<V, kSeedM>;
    static int per_sm = 0;
    if (per_sm == 0) {
        QBG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        QBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem));
        per_sm = std::max(1, per_sm);
    }
    const SPass& last = pl.spasses.back();
    const int64_t bc = int64_t{1} << last.nb;
    double* epart = static_cast<double*>(scratch(last.ntiles * bc * sizeof(double), 14));
    for (auto& sp : pl.spasses) {
        int64_t grid = std::min<int64_t>(static_cast<int64_t>(sp.ntiles), static_cast<int64_t>(num_sms()) * per_sm);
        LaunchScope ls("seed", (sp.first ? 2.0 : 3.0) * psi.bytes());
        kern<<<static_cast<unsigned>(grid), T, smem, stream()>>>(static_cast<const V*>(psi.ptr), static_cast<V*>(phi.ptr),
                                                              sp, pl.d_groups, pl.d_terms, epart);
        QBG_CUDA(cudaGetLastError());
    }
    if (d_energy) {
        LaunchScope ls("energy", 8.0 * last.ntiles * bc);
        uint64_t nouter = uint64_t{1} << (pl.n - last.mq);
        k_energy<<<static_cast<unsigned>((psi.B + 127) / 128), 128, 0, stream()>>>(epart, nouter, last.nchunks, bc, psi.B,
                                                                                 d_energy);
        QBG_CUDA(cudaGetLastError());
    }
}

}  // namespace

bool fused_obs_apply(const DevState& psi, const DevState& phi, Observable& o, double* d_energy) {
    const int nb = batch_bits(psi.B);
    if (psi.n < kSeedM - nb || o.terms.empty()) return false;
    auto pl = get_seed_plan(o, psi);
    if (psi.dtype == QBG_C128)
        run_seed<double2>(psi, phi, *pl, d_energy);
    else
        run_seed<float2>(psi, phi, *pl, d_energy);
    return true;
}

}  // namespace qbg
