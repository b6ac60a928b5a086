// fused.h — device descriptors of the tiled multi-gate engine (fused.cu, planner.cpp).
//
// A PASS streams the state through the SMs once.  Each CTA owns one TILE at a time: the 2^m
// elements whose "tile qubits" Q (plus nb low batch bits) vary and whose other bits are
// fixed.  The tile lives in registers: each of T = 2^(m-r) threads holds R = 2^r elements.
// A pass is a sequence of STAGES; in each stage r of the tile's local bits are register bits
// (gates on them are applied in registers), the rest are thread bits.  Between stages the
// tile is re-laid through shared memory (one transpose).  Diagonal gates and controls need
// no register bit: they read the element's global index bits wherever they live (register,
// thread or tile-outer bits).  The gradient ops of the reverse pass reduce
// Im<φ̄|K|ψ> over the tile into per-warp shared accumulators (deterministic).
#pragma once

#include <cstdint>

namespace qbg {
namespace fz {

enum : uint8_t {
    OP_DENSE1 = 1,  // 2x2 on register slot a
    OP_X1,          // swap on slot a
    OP_PERM1,       // generalised permutation on slot a: y0 = v0 x[p0], y1 = v1 x[p1] (b = 1: swapped)
    OP_DIAG1R,      // diag on slot a
    OP_DIAG1T,      // diag on thread-index bit a (uniform per thread)
    OP_DIAG1G,      // diag on tile-outer global bit a (uniform per tile)
    OP_DENSE2,      // 4x4 on slots (a = matrix qubit 0, b = matrix qubit 1)
    OP_DIAGK,       // diag over t targets at mixed locations (aux)
    OP_DENSE3,      // 8x8 on slots (a, b, aux & 0xff) = matrix qubits 0, 1, 2 (JIT kernels only)
    OP_DENSE4,      // 16x16 on slots (a, b, aux & 0xff, aux >> 8 & 0xff) (JIT kernels only)
    G_DENSE1 = 16,  // gradient Im<adj|K psi>, K 2x2 on slot a
    G_DIAG1R,       // K diag on slot a
    G_DIAG1U,       // K diag on a thread bit (b = 0) or a tile bit (b = 1) at position a
    G_DENSE2,       // K 4x4 on slots a, b
    G_DIAGK,        // K diag over t targets at mixed locations
    G_CROSS1,       // 2x2 cross matrix C_ab = Σ conj(adj_a) psi_b on slot a (8 components):
                    // the gradients of a whole same-qubit rotation run follow from C on the host
    G_CROSSH,       // the same for a run whose gradient matrices are Hermitian: 4 components
                    // Im C00, Im C11, Im(C01 + C10), Re(C01 − C10) (JIT kernels only)
    G_CROSSD        // a diagonal run (Rz / shift / phase only) on a register slot (b = 0), thread
                    // bit (b = 1) or tile bit (b = 2) at position a: Im C00, Im C11 (+ 2 zero
                    // components, the G_CROSSH layout; its A are diagonal)
};

// DIAGK target locations (aux, 8 bits per target: [7:6] type, [5:0] position)
enum : uint8_t { LOC_REG = 0, LOC_THR = 1, LOC_TILE = 2 };

struct DOp {
    uint8_t code, a, b, t;
    uint8_t creg_mask, creg_val, pad0, pad1;
    uint32_t cthr_mask, cthr_val;
    int32_t mat;    // offset (complex entries) into the plan's matrix table
    int32_t gslot;  // gradient slot within the pass (G_*), else -1
    uint64_t ctile_mask, ctile_val;
    uint64_t aux;
};
static_assert(sizeof(DOp) == 48, "DOp layout");

constexpr int kMaxR = 5;
constexpr int kMaxFoldM = 16;     // local index bits a fold map covers
constexpr int kMaxFoldOuter = 8;  // outer-controlled folded gates per pass (distinct controls)
constexpr int kMaxW = 10;
constexpr int kMaxStages = 12;

struct DStage {
    int32_t op_begin, op_end;
    uint32_t sreg[kMaxR];  // swizzled smem offset of register slot k's unit vector
    uint32_t sthr[kMaxW];  // swizzled smem offset of tid bit p's unit vector
    int64_t greg[kMaxR];   // global element-offset weight of register slot k
    int64_t gthr[kMaxW];   // global element-offset weight of tid bit p
    uint8_t lreg[kMaxR];   // local bit of register slot k
    uint8_t lthr[kMaxW];   // local bit of tid bit p
};

struct DPass {
    int32_t nstages;
    int32_t ngrad;     // gradient slots used by this pass
    int32_t mq;        // tile qubits
    int32_t nb;        // batch bits in the tile
    uint8_t qpos[64];  // sorted global positions of the tile qubits (deposit of the tile id)
    int64_t B;         // batch count (row stride)
    int64_t nchunks;   // B / 2^nb
    uint64_t ntiles;   // 2^(n-mq) * nchunks
    int32_t op_base;   // first op of the pass in the plan's op array
    int32_t nops;
    int32_t mat_base;  // first matrix entry of the pass in the plan's matrix table
    int32_t nmats;
    int32_t grad_base; // first gradient component of the pass (row of the partials buffer)
    DStage st[kMaxStages];
    // Folded permutation gates (specialised pipelined kernels only): the CNOT / X gates at the
    // start of a forward pass (at the end of a checkpointed reverse pass) are not register-stage
    // ops but an affine map F of the tile's local index, applied to the slot address of the
    // stage-0 read (forward) or of the write that feeds the tile's TMA store (reverse):
    //   F(l) = XOR_k l_k fcol[k]  ^  fd  ^  XOR_i outer_bit(foq[i]) fow[i]
    int32_t nfold;      // folded gates (0: none)
    int32_t nfo;        // outer-controlled terms
    uint32_t fcol[kMaxFoldM];
    uint32_t fd;
    uint8_t foq[kMaxFoldOuter];   // global qubit of an outer control
    uint32_t fow[kMaxFoldOuter];  // its local mask
};

// Observable seed pass: groups of Pauli terms sharing one local X mask.
struct SGroup {
    uint32_t xloc;          // X support in local bits
    int32_t term_begin, term_end;
};
struct STerm {
    double cre, cim;        // coefficient with i^{nY} folded in
    uint32_t zloc;          // Z support inside the tile (local bits)
    uint32_t pad;
    uint64_t zout;          // Z support outside the tile (global bits)
};

constexpr int kMaxOps = 256;    // ops per pass (smem resident)
constexpr int kMaxMats = 512;   // complex matrix entries per pass (smem resident, interpreter kernels)
constexpr int kMaxMatsJit = 512;  // ... specialised kernels (a __grid_constant__ parameter; 1024 measured slower: constant-cache misses)
constexpr int kMaxComps = 256;  // gradient components per pass

struct GradEntry {
    int32_t type;  // 0 scalar component, 1 cross matrix (8 components), 2 Hermitian cross (4)
    int32_t comp;
    int32_t param;
    int32_t pad;
    double A[8];  // cdbl A[4]     // column-major 2x2, cross entries only
};

struct SPass {
    int32_t mq, nb;
    uint8_t qpos[64];
    int64_t B, nchunks;
    uint64_t ntiles;
    int32_t g0, g1;  // groups of this pass
    int32_t first, last;
};

}  // namespace fz
}  // namespace qbg
