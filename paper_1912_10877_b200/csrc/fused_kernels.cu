// fused_kernels.cu — device side of the tiled engine: the generic (interpreter) tile kernel,
// the observable seed kernel and the gradient / energy epilogues.  The planner and the
// specialised (JIT) kernels live in fused.cu / jit_prelude.h.
#include <algorithm>
#include <cstring>

#include "fused.h"
#include "fused_kernels.h"

namespace qbg {

using namespace fz;

namespace {


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
            case G_CROSSD: {  // diagonal run: Im C00, Im C11 by the run bit (register / thread / tile)
                if constexpr (BACK) {
                    double h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    if (ok) {
#pragma unroll
                        for (int j = 0; j < (1 << RB); ++j) {
                            const int bit = op.b == 0 ? ((j >> op.a) & 1)
                                          : op.b == 1 ? ((tid >> op.a) & 1)
                                                      : static_cast<int>((outer >> op.a) & 1ull);
                            const double v = static_cast<double>(y[j].x) * x[j].y - static_cast<double>(y[j].y) * x[j].x;
                            if (bit) h[1] += v; else h[0] += v;
                        }
                    }
                    double s = warp_sum8(h, lane);
                    if ((lane & 3) == 0 && (lane >> 2) < 4) sg[(op.gslot + (lane >> 2)) * nw + warp] += s;
                }
                break;
            }
            case G_CROSSH: {  // (planned for JIT kernels; folded from the 8 components here)
                if constexpr (BACK) {
                    double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    if (ok) {
#define QBG_C(K) gcross1_k<V, RB, K>(x, y, c);
                        QBG_SLOT_SWITCH(op.a, RB, QBG_C)
#undef QBG_C
                    }
                    double h[8] = {c[1], c[7], c[3] + c[5], c[2] - c[4], 0, 0, 0, 0};
                    double s = warp_sum8(h, lane);
                    if ((lane & 3) == 0 && (lane >> 2) < 4) sg[(op.gslot + (lane >> 2)) * nw + warp] += s;
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

// one thread per gradient entry: its contribution (scalar component or Im Σ_ab A_ab C_ab)
__global__ void k_grad_values(const double* __restrict__ sums, const GradEntry* __restrict__ e, int64_t n,
                              double* __restrict__ vals) {
    int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const GradEntry& g = e[k];
    if (g.type == 0) {
        vals[k] = sums[g.comp];
        return;
    }
    const cdbl* GA = reinterpret_cast<const cdbl*>(g.A);
    if (g.type == 2) {  // Hermitian M = A: M00 Im C00 + M11 Im C11 + Re M01 Im(C01+C10) + Im M01 Re(C01−C10)
        const double r = 0.5 * (GA[2].re + GA[1].re), s = 0.5 * (GA[2].im - GA[1].im);
        vals[k] = GA[0].re * sums[g.comp] + GA[3].re * sums[g.comp + 1] + r * sums[g.comp + 2] + s * sums[g.comp + 3];
        return;
    }
    double acc = 0.0;  // C_ab at comp + 2(2a+b)
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            const cdbl A = GA[b * 2 + a];
            const double cr = sums[g.comp + 2 * (2 * a + b)], ci = sums[g.comp + 2 * (2 * a + b) + 1];
            acc += A.re * ci + A.im * cr;
        }
    vals[k] = acc;
}

// one thread per parameter: its entries (CSR, in plan order) summed in a fixed order
__global__ void k_grad_csr(const double* __restrict__ vals, const int* __restrict__ ptr, const int* __restrict__ idx,
                           int64_t nparams, double* __restrict__ grads) {
    int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= nparams) return;
    double s = 0.0;
    for (int k = ptr[p]; k < ptr[p + 1]; ++k) s += vals[idx[k]];
    if (ptr[p + 1] > ptr[p]) grads[p] += s;
}

// One warp per row: lane l sums columns l, l+32, … in order (coalesced across the warp), then a
// fixed xor-butterfly — the same order on every run (deterministic gradients).
__global__ void k_rows(const double* __restrict__ part, int64_t nrows, int64_t cols, double* __restrict__ out) {
    const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= nrows) return;
    const double* row = part + r * cols;
    double s = 0.0;
    for (int64_t b = lane; b < cols; b += 32) s += row[b];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = s;
}

// ---- observable seed: phi (+)= Σ_groups Σ_terms c (-1)^{|src & z|} psi[src], src = l ^ xloc ----

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
// one block per batch column, fixed strided split + fixed tree: deterministic
__global__ void __launch_bounds__(256) k_energy(const double* __restrict__ epart, uint64_t nouter, int64_t nchunks,
                                                int64_t bc, int64_t B, double* __restrict__ e) {
    const int64_t b = blockIdx.x;
    const int64_t c = b / bc, beta = b - c * bc;
    double s = 0.0;
    for (uint64_t o = threadIdx.x; o < nouter; o += blockDim.x) s += epart[(o * nchunks + c) * bc + beta];
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) e[b] = red[0];
}

}  // namespace

namespace {
template <typename V, int M, int RB, bool BACK>
void launch_fused(V* psi, V* adj, const DPass& P, const DOp* d_ops, const cdbl* d_mats, double* gpart, int64_t gcols) {
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
    kern<<<static_cast<unsigned>(grid), T, smem, stream()>>>(psi, adj, P, d_ops, d_mats, gpart, gcols);
    QBG_CUDA(cudaGetLastError());
}


}  // namespace

void launch_interp(int dtype, bool back, void* psi, void* adj, const DPass& P, const DOp* d_ops, const cdbl* d_mats,
                   double* gpart, int64_t gcols) {
    if (dtype == QBG_C128) {
        if (back)
            launch_fused<double2, 11, 3, true>(static_cast<double2*>(psi), static_cast<double2*>(adj), P, d_ops, d_mats, gpart, gcols);
        else
            launch_fused<double2, 12, 4, false>(static_cast<double2*>(psi), nullptr, P, d_ops, d_mats, gpart, gcols);
    } else {
        if (back)
            launch_fused<float2, 11, 3, true>(static_cast<float2*>(psi), static_cast<float2*>(adj), P, d_ops, d_mats, gpart, gcols);
        else
            launch_fused<float2, 12, 4, false>(static_cast<float2*>(psi), nullptr, P, d_ops, d_mats, gpart, gcols);
    }
}

void launch_grad_rows(const double* part, int64_t nrows, int64_t cols, double* sums) {
    LaunchScope ls("grad_rows", 8.0 * nrows * cols);
    k_rows<<<static_cast<unsigned>((nrows + 7) / 8), 256, 0, stream()>>>(part, nrows, cols, sums);
    QBG_CUDA(cudaGetLastError());
}

void launch_grad_epilogue(const double* sums, const GradEntry* d_epi, int64_t n, const int* d_ptr, const int* d_idx,
                          int64_t nparams, double* grads) {
    double* vals = static_cast<double*>(scratch(std::max<int64_t>(1, n) * sizeof(double), 15));
    {
        LaunchScope ls("grad_values", 80.0 * n);
        k_grad_values<<<static_cast<unsigned>((n + 127) / 128), 128, 0, stream()>>>(sums, d_epi, n, vals);
        QBG_CUDA(cudaGetLastError());
    }
    LaunchScope ls("grad_csr", 16.0 * n);
    k_grad_csr<<<static_cast<unsigned>((nparams + 127) / 128), 128, 0, stream()>>>(vals, d_ptr, d_idx, nparams, grads);
    QBG_CUDA(cudaGetLastError());
}

void launch_seed(int dtype, const void* psi, void* phi, const SPass& sp, const SGroup* g, const STerm* t, double* epart,
                 double bytes) {
    constexpr int T = 256;
    constexpr int M = 12;
    static int per_sm[2] = {0, 0};
    const int di = dtype == QBG_C128 ? 0 : 1;
    size_t smem = (dtype == QBG_C128 ? 16 : 8) << M;
    if (per_sm[di] == 0) {
        if (di == 0) {
            QBG_CUDA(cudaFuncSetAttribute(k_seed<double2, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            QBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[di], k_seed<double2, M>, T, smem));
        } else {
            QBG_CUDA(cudaFuncSetAttribute(k_seed<float2, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            QBG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[di], k_seed<float2, M>, T, smem));
        }
        per_sm[di] = std::max(1, per_sm[di]);
    }
    int64_t grid = std::min<int64_t>(static_cast<int64_t>(sp.ntiles), static_cast<int64_t>(num_sms()) * per_sm[di]);
    LaunchScope ls("seed", bytes);
    if (di == 0)
        k_seed<double2, M><<<static_cast<unsigned>(grid), T, smem, stream()>>>(static_cast<const double2*>(psi),
                                                                           static_cast<double2*>(phi), sp, g, t, epart);
    else
        k_seed<float2, M><<<static_cast<unsigned>(grid), T, smem, stream()>>>(static_cast<const float2*>(psi),
                                                                          static_cast<float2*>(phi), sp, g, t, epart);
    QBG_CUDA(cudaGetLastError());
}

void launch_energy(const double* epart, uint64_t nouter, int64_t nchunks, int64_t bc, int64_t B, double* e) {
    LaunchScope ls("energy", 8.0 * nouter * nchunks * bc);
    k_energy<<<static_cast<unsigned>(B), 256, 0, stream()>>>(epart, nouter, nchunks, bc, B, e);
    QBG_CUDA(cudaGetLastError());
}

}  // namespace qbg
