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
//
// Execution (gen_pass, default): one persistent CTA per SM, warp-specialised.  A producer
// warpgroup streams tiles into a ring of shared-memory slots — one TMA tensor box per tile
// (cp.async fallback for layouts beyond 5 dimensions) completing the slot's `full` mbarrier —
// and, in the forward pass, drains computed slots back with one TMA tensor store.  Two consumer
// groups take alternate tiles; a slot's previous use may belong to the other group, so a group
// waits for that release (`done`) before the fill's parity wait.
// See fused.h for the tile/stage vocabulary and DESIGN.md for the roofline numbers.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <array>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <set>
#include <unordered_map>
#include <memory>

#include <sstream>

#include "fused.h"
#include "jit.h"
#include "fused_kernels.h"
#include "program.h"

namespace qbg {

using namespace fz;
static_assert(kMaxComps <= 256, "statistic slots are packed 8 bits each (checkpointed statistics groups)");

// =====================================================================================
// device side
// =====================================================================================

// =====================================================================================
// host side: planner
// =====================================================================================
namespace {

constexpr int kFwdM = 12, kFwdRB = 4;  // 4096-element tiles, 256 threads x 16 registers
constexpr int kBwdM = 11, kBwdRB = 3;  // two states: 2048-element tiles, 256 threads x 2x8
constexpr int kSeedM = 12;

// Tile geometry of a direction: M local bits, RB register bits, `coal` low qubit bits every
// tile must hold so that loads/stores are contiguous (3 = 128-B runs at complex128).  The
// interpreter kernels exist for the defaults only; other geometries need the JIT path.
// Overridable for tuning: QBG_FWD_M / QBG_FWD_RB / QBG_BWD_M / QBG_BWD_RB / QBG_COALESCE.
struct Geo {
    int M, RB, coal;
};
int env_int(const char* k, int d) {
    const char* e = std::getenv(k);
    return (e && *e) ? std::atoi(e) : d;
}
Geo geo_for(int dir);
// Warp-specialised pipelined passes (QBG_PIPE=G, G = 1 or 2): a producer warpgroup streams
// tiles global -> shared with 16-B cp.async into a ring of slots tracked by mbarriers
// (cp.async.mbarrier.arrive.noinc); G consumer groups of TH threads take alternate tiles
// (ping-pong), so one group's loads / transposes / stores overlap the other's FP64 work.
// With G = 2 the producer gives registers back (setmaxnreg) to the consumers.
// Default on (2 groups) for the specialised kernels; QBG_PIPE=0 selects the plain tile loop.
bool pipeline_enabled() {
    static const bool on = jit::enabled() && env_int("QBG_PIPE", 2) > 0;
    return on;
}
int consumer_groups(bool back) {
    // (4 groups of 64 threads with 2^10 tiles measured slower per gate; 2 is the design point)
    // QBG_FWD_GROUPS / QBG_BWD_GROUPS (1..4) override per direction
    static const int g = std::min(2, std::max(1, env_int("QBG_PIPE", 2)));
    static const int f = std::min(4, std::max(1, env_int("QBG_FWD_GROUPS", g)));
    static const int b = std::min(4, std::max(1, env_int("QBG_BWD_GROUPS", g)));
    return back ? b : f;
}
constexpr int kProducerThreads = 128;  // one producer warpgroup per CTA
constexpr int kSeedMinB = 2;  // CTAs per SM the seed kernels are compiled for (measured: 0.343 vs 0.373 ms at 1)
bool jit_check_mode() {
    static const bool on = env_int("QBG_JIT_CHECK", 0) != 0;
    return on;
}
// Gradient-statistic stores: after the butterfly reduction every lane of a group holds the same
// sum; ONE lane per group read-modify-writes the shared cell, by a predicated store (sg_acc in
// jit_prelude.h) rather than an `if`, so a stage stays one basic block and ptxas can overlap a
// run's shuffle chain with the next run's FP64 work (measured: 0.643 -> 0.620 ms per reverse pass
// against the branch).
bool perm_ctrl_regs() {
    static const bool on = env_int("QBG_PERM_CTRL_REGS", 1) != 0;
    return on;
}
constexpr int kProducerRegsDefault = 40;
int producer_regs() {  // registers the producer warpgroup keeps after setmaxnreg.dec (QBG_PRODUCER_REGS)
    static const int r = std::min(64, std::max(24, env_int("QBG_PRODUCER_REGS", kProducerRegsDefault) / 8 * 8));
    return r;
}
// ring slots that fit next to the gradient cells and barriers (<= 220 KB, 2..6 slots)
int pipe_slots(bool back, int M, bool c128, int ngrad, int nwt) {
    const size_t tile = (static_cast<size_t>(back ? 2 : 1) << M) * (c128 ? 16 : 8);
    const size_t cells = back ? static_cast<size_t>(ngrad) * (nwt + 1) * 8 : 0;
    static const int cap_b = env_int("QBG_BWD_SLOTS", 6), cap_f = env_int("QBG_FWD_SLOTS", 6);
    int n = std::max(2, back ? cap_b : cap_f);
    while (n > 2 && n * tile + cells + 128 > 220 * 1024) --n;
    return n;
}
// Checkpointed reverse passes: the slot (ψ and φ̄ tiles) is needed only until the statistics and the
// read of φ̄ are done; φ̄'s transposes then use a private scratch tile of the consumer group, and the
// slot is released at once, so the next tile loads during the whole uncompute sweep.  One slot per
// consumer group (QBG_CK_SCRATCH=0: the shared ring, slot held to the end of the tile; A/B).
bool ck_scratch() {
    static const bool on = env_int("QBG_CK_SCRATCH", 1) != 0;
    return on;
}
// Specialised-kernel defaults (measured on B200, 25q apply+grad, tools/sweep.py logs in
// profiles/): forward 2^11-element tiles of 128 threads x 16 registers, 3 CTAs/SM; reverse
// 2^11 x 2 states of 128 threads x 2x16, 2 CTAs/SM.  The interpreter keeps (12,4) / (11,3).
constexpr int kJitFwdM = 11, kJitFwdRB = 4, kJitFwdMinB = 3;
constexpr int kJitBwdM = 11, kJitBwdRB = 4, kJitBwdMinB = 2;
int ctas_per_sm(bool back, int threads) {
    static const int f = env_int("QBG_FWD_MINB", 0), b = env_int("QBG_BWD_MINB", 0);
    const int o = back ? b : f;
    if (o > 0) return o;
    if (jit::enabled()) {
        const Geo g = geo_for(back ? 2 : 0);
        if (!back && g.M == kJitFwdM && g.RB == kJitFwdRB) return kJitFwdMinB;
        if (back && g.M == kJitBwdM && g.RB == kJitBwdRB) return kJitBwdMinB;
    }
    return threads >= 512 ? 1 : 2;
}
Geo geo_for(int dir) {
    const bool j = jit::enabled();
    static const Geo f{env_int("QBG_FWD_M", j ? kJitFwdM : kFwdM), env_int("QBG_FWD_RB", j ? kJitFwdRB : kFwdRB),
                       env_int("QBG_COALESCE", 3)};
    static const Geo b{env_int("QBG_BWD_M", j ? kJitBwdM : kBwdM), env_int("QBG_BWD_RB", j ? kJitBwdRB : kBwdRB),
                       env_int("QBG_COALESCE", 3)};
    return dir == 2 ? b : f;
}

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
    std::vector<int> src;      // program ops (indices into Program::real) fused into this gate
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
            o.src.insert(o.src.end(), pg.src.begin(), pg.src.end());
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

// Whether every cross matrix A_k of a run is Hermitian (4 statistics suffice, G_CROSSH).
bool run_hermitian(const PG& pg) {
    for (const RunGrad& rg : pg.run) {
        double sc = 0.0;
        for (int k = 0; k < 4; ++k) sc = std::max(sc, std::hypot(rg.A[k].re, rg.A[k].im));
        const double tol = 1e-12 * std::max(sc, 1e-300);
        if (std::fabs(rg.A[0].im) > tol || std::fabs(rg.A[3].im) > tol || std::fabs(rg.A[2].re - rg.A[1].re) > tol ||
            std::fabs(rg.A[2].im + rg.A[1].im) > tol)
            return false;
    }
    return true;
}

// Where a plan matrix came from (plan_passes' emit_mat), so a new θ can rewrite the values only.
enum { MS_G = 0, MS_GDENSE = 1, MS_KDIAG = 2, MS_KDENSE = 3 };
struct MatSrc {
    int gi;    // index into FusedPlan::gates
    int what;  // MS_*
};

// Everything plan_passes reads from a fused gate apart from its matrix values: kinds, qubits,
// controls, permutations, parameters, and the value-dependent predicates the emission branches
// on (identity, X, Hermitian cross matrices).  Equal signatures => identical passes and ops.
uint64_t pg_sig(const PG& pg) {
    uint64_t h = 1469598103934665603ULL;
    auto mix = [&](uint64_t v) {
        h ^= v;
        h *= 1099511628211ULL;
        h ^= h >> 29;
    };
    auto mixg = [&](const Gate& g) {
        mix(static_cast<uint64_t>(g.kind));
        mix(static_cast<uint64_t>(g.t));
        mix(static_cast<uint64_t>(g.dim));
        for (int q = 0; q < g.t; ++q) mix(g.tbit[q]);
        mix(g.tmask);
        mix(g.cmask);
        mix(g.cval);
        mix(g.m.size());
        mix(g.perm.size());
        for (int v : g.perm) mix(static_cast<uint64_t>(v));
    };
    const Gate& g = pg.gate();
    mixg(g);
    mix(static_cast<uint64_t>(pg.param + 1));
    mix(pg.k != nullptr);
    if (pg.k) mixg(*pg.k);
    mix(pg.run.size());
    for (const RunGrad& rg : pg.run) mix(static_cast<uint64_t>(rg.param + 1));
    mix(run_hermitian(pg));
    const bool x1 = g.kind == QBG_MAT_PERMUTATION && g.t == 1 && g.perm[0] == 1 && g.m[0].re == 1 &&
                    g.m[0].im == 0 && g.m[1].re == 1 && g.m[1].im == 0;
    mix(x1);
    return h;
}

struct Step {
    bool tile = false;
    DPass pass;
    std::vector<int> members;    // the plan gates of a tile pass (checkpointed reverse plans)
    int seg = -1;                // checkpoint segment of a mirror forward step (dir 4)
    int single = -1;
    int single_comp = -1;
    int jk = -1;                 // specialised kernel (index into the plan's kernel list)
    std::vector<char> blob;      // its matrix parameter (PM<T, 2*nmats>)
    size_t smem = 0;
    double flops = 0;            // algorithmic FP64 flops of one launch (pass_flops)
    int msrc_begin = 0, msrc_end = 0;  // its matrices' entries in FusedPlan::msrc (refresh_segment)
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
    // values-only refresh (new θ, same structure, refresh_values): where each matrix entry and
    // each cross-gradient entry came from, and the structural signature of the fused gate list
    std::vector<MatSrc> msrc;
    std::vector<std::pair<int, int>> esrc;  // (gate, run index), (-1, -1): no value
    std::vector<uint64_t> sig;
    // checkpointed expect' (dir 4 = forward mirror of the dir-5 reverse plan): per segment the
    // program ops it applies (forward order), and the serial of the reverse plan it mirrors
    std::vector<std::vector<int>> part;
    std::vector<uint64_t> part_q;      // tile qubits of a segment's passes (0: a single-gate step)
    std::vector<int> seg_steps;        // first step of each segment (+ end)
    std::vector<int> seg_gates;        // first fused gate of each segment (+ end)
    uint64_t serial = 0, mirror_of = 0;
    int64_t ncomps = 0;
    std::vector<jit::Kernel> jk;
    DOp* d_ops = nullptr;
    cdbl* d_mats = nullptr;
    GradEntry* d_epi = nullptr;
    std::vector<int> csr_ptr, csr_idx;  // gradient entries per parameter, in plan order
    int* d_ptr = nullptr;
    int* d_idx = nullptr;
    int64_t tile_passes = 0;
    int M = 0, RB = 0;         // tile geometry of this plan
    bool energy_only = false;  // seed plans: <O> without materialising φ = Oψ
    // observable seed
    std::vector<SPass> spasses;
    std::vector<SGroup> groups;
    std::vector<STerm> terms;
    std::vector<int> sjk;                  // specialised seed kernel per seed pass
    std::vector<std::vector<char>> sblob;  // its coefficient parameter
    SGroup* d_groups = nullptr;
    STerm* d_terms = nullptr;
    ~FusedPlan() {
        for (void* p : {static_cast<void*>(d_ops), static_cast<void*>(d_mats), static_cast<void*>(d_epi),
                        static_cast<void*>(d_ptr), static_cast<void*>(d_idx), static_cast<void*>(d_groups),
                        static_cast<void*>(d_terms)})
            if (p) cudaFreeAsync(p, stream());
    }
};

namespace {

// Plan tables are small and re-made for every new parameter vector: stream-ordered allocation,
// copy and free (cudaMalloc / cudaMemcpy / cudaFree would synchronise the device and serialise
// the host planning of the reverse pass behind the forward passes already queued).
template <class T>
T* upload(const std::vector<T>& v) {
    T* d = nullptr;
    if (v.empty()) return nullptr;
    QBG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), v.size() * sizeof(T), stream()));
    QBG_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, stream()));
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

bool pg_grad(const PG& g) { return !g.run.empty() || g.k != nullptr; }

std::vector<int> emit_pass(FusedPlan& pl, int M, int RB, int nb, bool backward, int coal, uint64_t Q,
                           const std::vector<int>& sel);
bool tma_box_ok(const DPass& P, int M);  // the tile is a <= 5-D TMA box (complex128)
bool tma_enabled();

// Greedy pass construction (see fused.h): a gate joins the pass when it does not conflict with
// any gate already passed over and its non-diagonal targets fit in the tile qubit set.
// ck (checkpointed reverse plans): the pass's gradient statistics are all taken at its start,
// against the checkpointed ψ, so a gate with a gradient joins only when no gate already in the
// pass touches its qubits (a run's cross matrix is invariant under gates on other qubits only).
void plan_passes(FusedPlan& pl, int M, int RB, int nb, bool backward, int coal = 3, bool ck = false) {
    const int n = pl.n;
    const int mq = M - nb;
    const uint64_t full = n >= 64 ? ~uint64_t{0} : (uint64_t{1} << n) - 1;
    uint64_t Qc = 0;  // coalescing: local bits 0..2 must be contiguous in memory
    for (int b = 0; b < coal - nb; ++b) Qc |= uint64_t{1} << b;
    std::vector<int> remaining(pl.gates.size());
    for (size_t i = 0; i < remaining.size(); ++i) remaining[i] = static_cast<int>(i);
    // 3- and 4-qubit non-diagonal gates (dense matblocks, permutations) are a stage op over three /
    // four register slots in the specialised kernels; with a gradient (a parameterised multi-qubit
    // generator) they keep their own pass
    static const bool dense3 = env_int("QBG_TILE_DENSE3", 1) != 0;  // (diagnostics: A/B of the stage op)
    const int max_mats = jit::enabled() ? kMaxMatsJit : kMaxMats;
    auto tileable = [&](const PG& g) {
        const Gate& u = g.gate();
        return u.t <= 2 || is_diagonal(u) ||
               (dense3 && (u.t == 3 || u.t == 4) && RB >= u.t && jit::enabled() && !g.k && g.run.empty());
    };
    // phase 1 grows Q greedily; phase 2 selects with Q fixed, within the pass's smem budgets.
    // reserve: the gates with a gradient may claim at most mq - reserve qubits of Q (checkpointed
    // plans try several: the CNOT ring after a rotation layer needs target qubits the rotations
    // would otherwise take, and the ck rule keeps later rotations out of a pass with those CNOTs)
    auto select = [&](int reserve, uint64_t& Q, std::vector<int>& sel, std::vector<int>& rest) {
        Q = Qc;
        sel.clear();
        rest.clear();
        {
            uint64_t bnd = 0, ball = 0, touched = 0;
            for (int gi : remaining) {
                const PG& g = pl.gates[gi];
                bool conflict = (g.nd() & ball) | (g.all() & bnd);
                if (ck && pg_grad(g) && (g.all() & touched)) conflict = true;
                if (!tileable(g) || conflict) {
                    bnd |= g.nd();
                    ball |= g.all();
                    continue;
                }
                uint64_t need = g.nd();
                if ((need & ~Q) == 0) {
                    touched |= g.all();
                    continue;
                }
                if (popc(Q | need) <= (pg_grad(g) ? mq - reserve : mq)) {
                    Q |= need;
                    touched |= g.all();
                } else {
                    bnd |= g.nd();
                    ball |= g.all();
                }
            }
        }
        for (int q = n - 1; q >= 0 && popc(Q) < mq; --q) Q |= uint64_t{1} << q;
        Q &= full;
        {
            uint64_t bnd = 0, ball = 0, touched = 0;
            int nops = 0, nmats = 0, ncomps = 0;
            for (int gi : remaining) {
                const PG& g = pl.gates[gi];
                bool conflict = (g.nd() & ball) | (g.all() & bnd);
                if (ck && pg_grad(g) && (g.all() & touched)) conflict = true;
                int co, cmx, cc2;
                gate_cost(g, co, cmx, cc2);
                bool fits = nops + co <= kMaxOps && nmats + cmx <= max_mats && ncomps + cc2 <= kMaxComps;
                if (tileable(g) && !conflict && (g.nd() & ~Q) == 0 && fits) {
                    sel.push_back(gi);
                    touched |= g.all();
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
    };
    while (!remaining.empty()) {
        uint64_t Q = 0;
        std::vector<int> sel, rest;
        select(0, Q, sel, rest);
        for (int reserve = 1; ck && reserve <= 4 && reserve < mq - coal; ++reserve) {
            uint64_t Q2 = 0;
            std::vector<int> sel2, rest2;
            select(reserve, Q2, sel2, rest2);
            if (sel2.size() > sel.size()) {
                Q = Q2;
                sel.swap(sel2);
                rest.swap(rest2);
            }
        }
        if (sel.empty()) {
            Step st;
            st.single = remaining.front();
            pl.steps.push_back(st);
            remaining.erase(remaining.begin());
            continue;
        }
        std::vector<int> back = emit_pass(pl, M, RB, nb, backward, coal, Q, sel);
        std::vector<int> merged;
        std::merge(back.begin(), back.end(), rest.begin(), rest.end(), std::back_inserter(merged));
        remaining = merged;
    }
}

// One tile pass over the gates `sel` (plan order) with tile qubits Q: stages, ops, matrices and
// gradient entries appended to the plan.  Returns the gates beyond the stage budget (sorted), which
// the caller plans into a later pass.
std::vector<int> emit_pass(FusedPlan& pl, int M, int RB, int nb, bool backward, int coal, uint64_t Q,
                           const std::vector<int>& sel) {
    const int n = pl.n;
    const int mq = M - nb;
    const int max_mats = jit::enabled() ? kMaxMatsJit : kMaxMats;
    std::vector<int> back;
    {
        TileGeom tg = geom(M, RB, nb, Q, pl.B);
        // ---- permutation folding (DPass::nfold) ----
        // Forward passes (plans 0, 4): the CNOT / X gates that can be hoisted to the pass start
        // (every gate before them that stays a stage op touches other qubits) become the affine
        // map of the stage-0 slot read.  Checkpointed reverse passes (plan 5): the ones that can
        // sink to the pass end become the map of the scratch write feeding the tile's TMA store.
        // They then need no register stage: a CNOT ring otherwise costs a register slot per stage
        // for its next target.
        DPass probe{};
        probe.mq = mq;
        probe.nb = nb;
        {
            int k = 0;
            for (int q = 0; q < 64; ++q)
                if ((Q >> q) & 1) probe.qpos[k++] = static_cast<uint8_t>(q);
        }
        probe.B = pl.B;
        probe.nchunks = pl.B >> nb;
        probe.ntiles = (uint64_t{1} << (n - mq)) * static_cast<uint64_t>(probe.nchunks);
        // the reverse pass stores through its scratch tile with one TMA tensor store
        const bool rstore_tma = backward && pl.dir == 5 && pipeline_enabled() && jit::enabled() && ck_scratch() &&
                                tma_enabled() && pl.dtype == QBG_C128 && tma_box_ok(probe, M);
        static const bool fold_env = env_int("QBG_FOLD", 1) != 0;  // (0: CNOTs stay stage ops; A/B)
        const bool fold_on = fold_env && jit::enabled() && pipeline_enabled() && M <= kMaxFoldM &&
                             (backward ? rstore_tma : (pl.dir == 0 || pl.dir == 4));
        std::vector<int> folded;  // application order
        std::vector<int> work = sel;
        if (fold_on) {
            auto foldable = [&](const PG& pg) {
                const Gate& g = pg.gate();
                if (pg.k || !pg.run.empty() || g.kind != QBG_MAT_PERMUTATION || g.t != 1 || popc(g.cmask) > 1) return false;
                const bool x1 = g.perm[0] == 1 && g.m[0].re == 1 && g.m[0].im == 0 && g.m[1].re == 1 && g.m[1].im == 0;
                return x1 && tg.local[g.tbit[0]] >= 0;
            };
            uint64_t blocked = 0;
            std::vector<int> keep;
            std::vector<uint64_t> outer_ctl;
            auto take = [&](int gi) {
                const PG& pg = pl.gates[gi];
                if (!foldable(pg) || (pg.all() & blocked)) return false;
                const uint64_t cm = pg.gate().cmask;
                if (cm && tg.local[__builtin_ctzll(cm)] < 0 &&
                    std::find(outer_ctl.begin(), outer_ctl.end(), cm) == outer_ctl.end()) {
                    if (static_cast<int>(outer_ctl.size()) >= kMaxFoldOuter) return false;
                    outer_ctl.push_back(cm);
                }
                return true;
            };
            if (!backward) {
                for (int gi : sel) {
                    if (take(gi)) folded.push_back(gi);
                    else {
                        blocked |= pl.gates[gi].all();
                        keep.push_back(gi);
                    }
                }
            } else {
                for (size_t i = sel.size(); i-- > 0;) {
                    const int gi = sel[i];
                    if (take(gi)) folded.push_back(gi);
                    else {
                        blocked |= pl.gates[gi].all();
                        keep.push_back(gi);
                    }
                }
                std::reverse(folded.begin(), folded.end());
                std::reverse(keep.begin(), keep.end());
            }
            work.swap(keep);
        }
        // ---- stages ----
        const int R = RB, Wn = M - RB;
        struct StagePlan {
            uint32_t S = 0;  // local register bits
            std::vector<int> gates;
        };
        // Stages with lookahead: a stage takes every pending gate whose non-diagonal targets fit
        // its register set and that commutes with the gates it passes over (same rule as the
        // pass selection), so a CNOT ring and its rotation runs share stages.
        // The register set of a stage is seeded: besides the plain scan (the set grows with the
        // gates in order), the targets of any one or two of the first pending gates seed it, and the
        // stage that takes the most gates wins — a CNOT chain's next target then gets its register
        // before the rotation runs fill the set (fewer stages, i.e. transposes, per pass).
        std::vector<StagePlan> stages;
        {
            auto need_of = [&](int gi) {
                const Gate& g = pl.gates[gi].gate();
                uint32_t need = 0;
                if (!is_diagonal(g))
                    for (int q = 0; q < g.t; ++q) need |= 1u << tg.local[g.tbit[q]];
                // a permutation (CNOT, Toffoli, controlled SWAP) whose controls are register bits is
                // a compile-time register rename; a control on a thread bit would make it a
                // runtime conditional swap of the whole register tile (128 moves for 2 x 16 c128)
                // (measured: forward passes gain ~2%; reverse passes lose more to the extra
                // stages than the moves cost next to the FP64 work, so forward only)
                if (g.kind == QBG_MAT_PERMUTATION && !backward && perm_ctrl_regs())
                    for (int q = 0; q < 64; ++q)
                        if (((g.cmask >> q) & 1) && tg.local[q] >= 0) need |= 1u << tg.local[q];
                return need;
            };
            auto scan = [&](uint32_t S0, const std::vector<int>& pending, StagePlan& cur, std::vector<int>& left) {
                cur = StagePlan{};
                cur.S = S0;
                left.clear();
                uint64_t bnd = 0, ball = 0;
                for (int gi : pending) {
                    const PG& pg = pl.gates[gi];
                    const uint32_t need = need_of(gi);
                    bool conflict = (pg.nd() & ball) | (pg.all() & bnd);
                    if (!conflict && __builtin_popcount(cur.S | need) <= R) {
                        cur.S |= need;
                        cur.gates.push_back(gi);
                    } else {
                        bnd |= pg.nd();
                        ball |= pg.all();
                        left.push_back(gi);
                    }
                }
            };
            static const int seeds = env_int("QBG_STAGE_SEEDS", 16);  // (0: the plain scan; A/B)
            std::vector<int> pending = work;
            while (!pending.empty()) {
                StagePlan best, c;
                std::vector<int> bleft, l;
                scan(0, pending, best, bleft);
                std::vector<uint32_t> cand;  // target sets of the first pending gates
                for (int gi : pending) {
                    if (static_cast<int>(cand.size()) >= seeds) break;
                    const uint32_t nd = need_of(gi);
                    if (nd && __builtin_popcount(nd) <= R && std::find(cand.begin(), cand.end(), nd) == cand.end())
                        cand.push_back(nd);
                }
                for (size_t i = 0; i < cand.size(); ++i)
                    for (size_t j = i; j < cand.size(); ++j) {
                        const uint32_t S0 = cand[i] | cand[j];
                        if (__builtin_popcount(S0) > R) continue;
                        scan(S0, pending, c, l);
                        if (c.gates.size() > best.gates.size()) {
                            best = c;
                            bleft = l;
                        }
                    }
                stages.push_back(best);
                pending = bleft;
            }
        }
        if (static_cast<int>(stages.size()) > kMaxStages - 2) {
            for (size_t s = kMaxStages - 2; s < stages.size(); ++s)
                back.insert(back.end(), stages[s].gates.begin(), stages[s].gates.end());
            stages.resize(kMaxStages - 2);
            // a sunk gate must not overtake a deferred one: the reverse pass keeps none
            if (backward) back.insert(back.end(), folded.begin(), folded.end()), folded.clear();
            std::sort(back.begin(), back.end());
        }
        // coalescing lane bits of the load / store layouts: the batch bits and the low qubits
        const uint32_t C = (1u << std::max(coal, nb)) - 1;
        const uint32_t qbits = ((1u << M) - 1) & ~((1u << nb) - 1);
        auto fill = [&](uint32_t S) {
            for (int b = M - 1; b >= 0 && __builtin_popcount(S) < R; --b)
                if (((qbits >> b) & 1) && !((S >> b) & 1) && !((C >> b) & 1)) S |= 1u << b;
            for (int b = M - 1; b >= 0 && __builtin_popcount(S) < R; --b)
                if (((qbits >> b) & 1) && !((S >> b) & 1)) S |= 1u << b;
            return S;
        };
        for (auto& s : stages) s.S = fill(s.S);
        // The first stage's layout reads the tile, the last one's writes it.  Without the pipeline
        // these are global accesses and must be coalesced (no low bit in registers).  Pipelined, the
        // producer moves the tile and the consumers read / write its linear image in shared
        // memory: one low bit in registers is a 2-way bank conflict on that access — cheaper than
        // an extra stage (a transpose).  The reverse pass's consumers store to global memory.
        // (A checkpointed reverse pass with a TMA tensor store writes its tile to the scratch in
        // the linear layout first, like the forward's drain.)
        auto needs_extra = [&](uint32_t S, bool store) {
            if (!pipeline_enabled() || (store && backward && !rstore_tma)) return (S & C) != 0;
            return __builtin_popcount(S & C) >= 2;
        };
        if (stages.empty()) stages.push_back(StagePlan{fill(0), {}});  // every gate folded
        // Before adding a layout-only stage, try to move the offending first / last stage inward
        // past stages whose gates all commute with its own (disjoint qubits): a pass of rotation
        // runs whose CNOTs are folded then needs no extra transpose for its low-qubit runs.
        auto commute = [&](const StagePlan& a, const StagePlan& b) {
            for (int ga : a.gates)
                for (int gb : b.gates)
                    if (pl.gates[ga].all() & pl.gates[gb].all()) return false;
            return true;
        };
        const int ns = static_cast<int>(stages.size());
        if (ns >= 3 && needs_extra(stages.front().S, false)) {
            int best = -1;
            for (int p = 1; p <= ns - 2 && commute(stages[0], stages[p]); ++p)
                if (!needs_extra(stages[1].S, false)) best = p;
            if (best > 0) std::rotate(stages.begin(), stages.begin() + 1, stages.begin() + best + 1);
        }
        if (ns >= 3 && needs_extra(stages.back().S, true)) {
            int best = -1;
            for (int p = ns - 2; p >= 1 && commute(stages[ns - 1], stages[p]); --p)
                if (!needs_extra(stages[ns - 2].S, true)) best = p;
            if (best > 0) std::rotate(stages.begin() + best, stages.end() - 1, stages.end());
        }
        if (needs_extra(stages.front().S, false)) stages.insert(stages.begin(), StagePlan{fill(0), {}});
        if (needs_extra(stages.back().S, true)) stages.push_back(StagePlan{fill(0), {}});

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
        step.msrc_begin = static_cast<int>(pl.msrc.size());
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
                // lanes 0..2 first: the coalescing bits when they are thread bits, completed to
                // three bits of distinct (bit mod 3) so the swizzled 16-B accesses of a quarter
                // warp hit 8 distinct bank groups
                bool used[3] = {false, false, false};
                for (int b = 0; b < 32 && order.size() < 3; ++b)
                    if (((C >> b) & 1) && !((sp.S >> b) & 1) && !used[b % 3]) {
                        order.push_back(b);
                        used[b % 3] = true;
                    }
                for (int b : avail)
                    if (!used[b % 3] && order.size() < 3 &&
                        std::find(order.begin(), order.end(), b) == order.end()) {
                        used[b % 3] = true;
                        order.push_back(b);
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
                D.lreg[k] = static_cast<uint8_t>(regb[k]);
            }
            for (int p = 0; p < Wn; ++p) {
                pos_of[thrb[p]] = p;
                D.sthr[p] = swz(1u << thrb[p]);
                D.gthr[p] = tg.gw[thrb[p]];
                D.lthr[p] = static_cast<uint8_t>(thrb[p]);
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
                auto emit_mat = [&](const std::vector<cdbl>& m, int what) {
                    int off = static_cast<int>(pl.mats.size()) - P.mat_base;
                    pl.mats.insert(pl.mats.end(), m.begin(), m.end());
                    pl.msrc.push_back({gi, what});
                    return off;
                };
                // gradient ops first (reverse pass: before the uncompute)
                if (backward && !pg.run.empty()) {
                    // Hermitian A (every rotation / shift / phase generator): 4 statistics suffice
                    const uint8_t rl = loc_code(g.tbit[0]);
                    const bool diag_run = is_diagonal(g);
                    if ((rl >> 6) != LOC_REG && !diag_run)
                        raise(QBG_ERR_INTERNAL, "fused plan: a non-diagonal run off the register slots");
                    bool herm = jit::enabled() && run_hermitian(pg);
                    // a diagonal run only needs Im C00 / Im C11, wherever its qubit lives (its
                    // A_k = K_k are diagonal); it may sit on a thread or tile bit
                    if (diag_run) herm = true;
                    DOp o = base;
                    o.code = diag_run ? G_CROSSD : herm ? G_CROSSH : G_CROSS1;
                    o.a = static_cast<uint8_t>(rl & 63);
                    o.b = static_cast<uint8_t>(rl >> 6);
                    o.gslot = ncomp;
                    for (size_t r = 0; r < pg.run.size(); ++r) {
                        const RunGrad& rg = pg.run[r];
                        GradEntry e{};
                        e.type = herm ? 2 : 1;
                        e.comp = static_cast<int>(P.grad_base) + ncomp;
                        e.param = rg.param;
                        std::memcpy(e.A, rg.A, sizeof(e.A));
                        pl.epi.push_back(e);
                        pl.esrc.push_back({gi, static_cast<int>(r)});
                    }
                    ncomp += herm ? 4 : 8;
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
                    pl.esrc.push_back({-1, -1});
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
                        o.mat = emit_mat(d, MS_KDIAG);
                    } else if (K.t == 1) {
                        o.code = G_DENSE1;
                        o.a = static_cast<uint8_t>(slot_of[tg.local[K.tbit[0]]]);
                        o.mat = emit_mat(dense_of(K), MS_KDENSE);
                    } else {
                        o.code = G_DENSE2;
                        o.a = static_cast<uint8_t>(slot_of[tg.local[K.tbit[0]]]);
                        o.b = static_cast<uint8_t>(slot_of[tg.local[K.tbit[1]]]);
                        o.mat = emit_mat(dense_of(K), MS_KDENSE);
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
                    o.mat = emit_mat(g.m, MS_G);
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
                            o.mat = emit_mat(g.m, MS_G);
                        }
                    } else {
                        o.code = OP_DENSE1;
                        o.mat = emit_mat(g.m, MS_G);
                    }
                } else if (g.t == 2) {
                    o.code = OP_DENSE2;
                    o.a = static_cast<uint8_t>(slot_of[tg.local[g.tbit[0]]]);
                    o.b = static_cast<uint8_t>(slot_of[tg.local[g.tbit[1]]]);
                    o.mat = emit_mat(dense_of(g), MS_GDENSE);
                } else {
                    o.code = g.t == 3 ? OP_DENSE3 : OP_DENSE4;
                    o.a = static_cast<uint8_t>(slot_of[tg.local[g.tbit[0]]]);
                    o.b = static_cast<uint8_t>(slot_of[tg.local[g.tbit[1]]]);
                    o.aux = static_cast<uint64_t>(slot_of[tg.local[g.tbit[2]]]);
                    if (g.t == 4) o.aux |= static_cast<uint64_t>(slot_of[tg.local[g.tbit[3]]]) << 8;
                    o.mat = emit_mat(dense_of(g), MS_GDENSE);
                }
                pl.ops.push_back(o);
            }
            D.op_end = static_cast<int>(pl.ops.size()) - P.op_base;
        }
        P.nops = static_cast<int>(pl.ops.size()) - P.op_base;
        P.nmats = static_cast<int>(pl.mats.size()) - P.mat_base;
        P.ngrad = ncomp;
        if (P.nops > kMaxOps || P.nmats > max_mats || P.ngrad > kMaxComps)
            raise(QBG_ERR_INTERNAL, "fused plan: pass exceeds its shared-memory budget");
        step.msrc_end = static_cast<int>(pl.msrc.size());
        for (const StagePlan& sp : stages) step.members.insert(step.members.end(), sp.gates.begin(), sp.gates.end());
        step.members.insert(step.members.end(), folded.begin(), folded.end());
        std::sort(step.members.begin(), step.members.end());
        // the fold map: forward F = C_1 ∘ … ∘ C_m (slot address of the element a register holds),
        // reverse F = D_m ∘ … ∘ D_1 (where the element lands); both built by right composition
        // F ← F ∘ G of an X / CNOT G: l ↦ l ⊕ [control = v] e_t (G is an involution)
        if (!folded.empty()) {
            P.nfold = static_cast<int>(folded.size());
            for (int k = 0; k < kMaxFoldM; ++k) P.fcol[k] = k < M ? 1u << k : 0u;
            auto rcompose = [&](const Gate& g) {
                const uint32_t ct = P.fcol[tg.local[g.tbit[0]]];
                if (g.cmask == 0) {
                    P.fd ^= ct;
                    return;
                }
                const int q = __builtin_ctzll(g.cmask);
                if (!((g.cval >> q) & 1)) P.fd ^= ct;  // control on 0: [l_c = 0] = l_c ⊕ 1
                const int c = tg.local[q];
                if (c >= 0) {
                    P.fcol[c] ^= ct;
                    return;
                }
                int i = 0;
                while (i < P.nfo && P.foq[i] != q) ++i;
                if (i == P.nfo) {
                    P.foq[i] = static_cast<uint8_t>(q);
                    P.fow[i] = 0;
                    ++P.nfo;
                }
                P.fow[i] ^= ct;
            };
            if (!backward)
                for (int gi : folded) rcompose(pl.gates[gi].gate());
            else
                for (size_t i = folded.size(); i-- > 0;) rcompose(pl.gates[folded[i]].gate());
        }
        pl.ncomps += ncomp;
        pl.steps.push_back(step);
        pl.tile_passes++;
    }
    return back;
}

// ---- code generation: one straight-line kernel per distinct pass structure -----------------------
std::string hex(uint64_t v) {
    char b[32];
    std::snprintf(b, sizeof(b), "0x%llxull", static_cast<unsigned long long>(v));
    return b;
}

// Σ over tid bits p of ((tid >> p) & 1) * w[p]  (as a C expression)
template <class W>
std::string tid_sum(const W* w, int nbits, bool xr) {
    std::ostringstream s;
    bool any = false;
    for (int p = 0; p < nbits; ++p) {
        if (w[p] == 0) continue;
        if (any) s << (xr ? " ^ " : " + ");
        if (xr)
            s << "(((tid >> " << p << ") & 1) ? " << static_cast<unsigned long long>(w[p]) << "u : 0u)";
        else
            s << "((i64)((tid >> " << p << ") & 1) * " << static_cast<long long>(w[p]) << "ll)";
        any = true;
    }
    if (!any) return xr ? "0u" : "0ll";
    return s.str();
}

// ---- TMA tile loads (default; QBG_TMA=0 disables): the tile as a <= 5-D box of the state -------
// (passes whose layout needs more than 5 dimensions keep the cp.async producer)
bool tma_store_enabled() {  // forward drain by one TMA tensor store per tile (QBG_TMA_STORE)
    static const bool on = env_int("QBG_TMA_STORE", 1) != 0;
    return on;
}
bool tma_enabled() {  // default on; QBG_TMA=0 selects the cp.async producer
    static const bool on = env_int("QBG_TMA", 1) != 0;
    return on;
}
struct TmaDim {
    uint64_t size;    // in FP64 units for dim 0, elements otherwise... (see tma_layout)
    uint64_t stride;  // bytes (ignored for dim 0)
    uint32_t box;
    int coord;        // 0: zero; 1: the batch chunk c; 2: (outer >> shift) & mask
    int shift;
    uint64_t mask;
};
// The element index splits into runs of bits that are all in the tile (box = run) or all outside
// (box 1, coordinate from the tile's outer index).  FP64 data type; the (re, im) pair folds into
// the innermost run when it is in the tile and contiguous, else it is its own dimension.
bool tma_layout(const DPass& P, int M, bool c128, std::vector<TmaDim>& dims) {
    dims.clear();
    if (!c128) return false;
    int n = P.mq;
    for (uint64_t t = P.ntiles / static_cast<uint64_t>(P.nchunks); t > 1; t >>= 1) ++n;
    uint64_t Q = 0;
    for (int k = 0; k < P.mq; ++k) Q |= uint64_t{1} << P.qpos[k];
    struct Run { uint64_t elems_w; int len; bool in; int coord; int shift; };
    std::vector<Run> runs;
    if (P.B > 1) {
        if (P.nb > 0) runs.push_back({1, P.nb, true, 0, 0});
        if (P.nchunks > 1) runs.push_back({uint64_t{1} << P.nb, -static_cast<int>(P.nchunks), false, 1, 0});
    }
    for (int q = 0; q < n;) {
        const bool in = (Q >> q) & 1;
        int e = q;
        while (e < n && (((Q >> e) & 1) != 0) == in) ++e;
        runs.push_back({static_cast<uint64_t>(P.B) << q, e - q, in, in ? 0 : 2, q});
        q = e;
    }
    for (size_t i = 0; i < runs.size(); ++i) {
        const Run& r = runs[i];
        const uint64_t size = r.len < 0 ? static_cast<uint64_t>(-r.len) : (uint64_t{1} << r.len);
        if (r.in) {  // split into pieces of <= 8 bits (box limit 256; 7 bits when it carries (re, im))
            int done = 0;
            while (done < r.len) {
                const bool first = dims.empty() && r.elems_w == 1 && done == 0;
                const int piece = std::min(r.len - done, first ? 7 : 8);
                TmaDim d{};
                d.size = (uint64_t{1} << piece) * (first ? 2 : 1);
                d.stride = (r.elems_w << done) * 16;
                d.box = static_cast<uint32_t>(d.size);
                d.coord = 0;
                dims.push_back(d);
                done += piece;
            }
        } else {
            if (dims.empty()) dims.push_back({2, 8, 2, 0, 0, 0});  // (re, im) on its own
            TmaDim d{};
            d.size = size;
            d.stride = r.elems_w * 16;
            d.box = 1;
            d.coord = r.coord;
            d.shift = r.shift;
            d.mask = size - 1;
            dims.push_back(d);
        }
    }
    return dims.size() <= 5;
}
bool tma_box_ok(const DPass& P, int M) {
    std::vector<TmaDim> dims;
    return tma_layout(P, M, true, dims);
}

std::string gen_pass(const DPass& P, const DOp* ops, int nmats, int M, int RB, bool back, bool c128, bool ck = false) {
    const int R = 1 << RB, W = M - RB, TH = 1 << W, NW = TH / 32;
    const size_t elem = c128 ? 16 : 8;
    // pipe mode (warp-specialised, see pipeline_enabled): NG consumer groups of TH threads take
    // alternate tiles from a ring of nbuf shared-memory slots filled by a cp.async producer warpgroup
    const bool pipe = pipeline_enabled();
    if (ck && (!back || !pipe)) raise(QBG_ERR_INTERNAL, "jit: a checkpointed pass is a pipelined reverse pass");
    const int NG = pipe ? consumer_groups(back) : 1;
    const int NWT = NG * NW;  // consumer warps
    const int CS = NWT + 1;   // gradient cell stride (odd: the lanes of a warp_sum hit distinct banks)
    const bool scr = ck && ck_scratch();  // φ̄ scratch per group, early slot release (see ck_scratch)
    const int nbuf = !pipe ? 1 : scr ? NG : pipe_slots(back, M, c128, P.ngrad, NWT);
    // who writes the results: with a deep ring the producer drains each computed slot to global
    // memory (consumers only compute); with a shallow one (reverse pass: 3 slots of 2 states) the
    // drain would delay the refill, so the consumers store from registers and release the slot
    const bool pstore = pipe && nbuf >= 2 * NG + 2;  // the drain needs NG + 2 spare slots
    const size_t tile_elems = static_cast<size_t>(back ? 2 : 1) << M;
    const size_t tile_bytes = tile_elems * elem;
    const std::string SYNC = pipe ? "group_bar<" + std::to_string(TH) + ">(1 + cg);\n" : "__syncthreads();\n";
    std::ostringstream s;
    const int NP = pipe ? kProducerThreads : 0;
    std::vector<TmaDim> td;
    const bool use_tma = pipe && tma_enabled() && tma_layout(P, M, c128, td);
    const bool tstore = use_tma && tma_store_enabled();  // (used where the producer drains: pstore)
    // checkpointed reverse pass: the consumers store φ̄ by a TMA tensor store from their scratch
    // (emit_pass plans the last stage for it: rstore_tma)
    const bool rstore = ck && scr && use_tma;
    if (P.nfold && (!pipe || (back && !rstore)))
        raise(QBG_ERR_INTERNAL, "jit: folded permutations need the pipelined load (forward) or the TMA store (reverse)");
    auto tma_coords = [&](const std::string& outer, const std::string& tile) {
        std::ostringstream co;
        for (size_t d = 0; d < td.size(); ++d) {
            if (td[d].coord == 0) co << "0";
            else if (td[d].coord == 1) co << "(int)c_of(" << tile << ")";
            else co << "(int)((" << outer << " >> " << td[d].shift << ") & " << td[d].mask << "ull)";
            if (d + 1 < td.size()) co << ", ";
        }
        return co.str();
    };
    s << "extern \"C\" __global__ void __launch_bounds__(" << NG * TH + NP << ", "
      << (pipe ? 1 : ctas_per_sm(back, TH)) << ") __NAME__(" << (c128 ? "c128" : "c64") << "* __restrict__ psi, "
      << (c128 ? "c128" : "c64")
      << "* __restrict__ adj, double* __restrict__ gpart, long long gcols, int gbase, const __grid_constant__ PM<"
      << (c128 ? "double" : "float") << ", " << std::max(2, 2 * nmats)
      << "> pm, const __grid_constant__ TMap tmp, const __grid_constant__ TMap tma) {\n";
    s << "typedef " << (c128 ? "c128" : "c64") << " V;\nconstexpr int R = " << R << ";\n";
    // forward: the tile is stored to adj when given (out-of-place pass: load psi, store adj; the
    // first pass of an out-of-place expect' reads the caller's register directly), else in place
    if (!back) s << "V* const outp = adj ? adj : psi;\nconst TMap* const outm = adj ? &tma : &tmp;\n";
    s << (pipe ? "const int tid_all = threadIdx.x;\n" : "const int tid = threadIdx.x;\n");
    s << "#define MV(i) mk<V>(pm.m[2 * (i)], pm.m[2 * (i) + 1])\n";
    // index checks (QBG_JIT_CHECK=1: every global / shared tile index is bounds-checked and traps;
    // the stand-in for memcheck where compute-sanitizer is unavailable)
    if (jit_check_mode()) {
        s << "#define GI(e) qchk((i64)(e), " << static_cast<int64_t>(P.ntiles) * (int64_t{1} << M) << "ll)\n";
        s << "#define SI(e) (unsigned)qchk((i64)(e), " << static_cast<int64_t>(tile_elems) << "ll)\n";
    } else {
        s << "#define GI(e) (e)\n#define SI(e) (e)\n";
    }
    s << "extern __shared__ __align__(128) unsigned char smraw[];\n";
    if (pstore && scr) raise(QBG_ERR_INTERNAL, "jit: a checkpointed pass drains no slot");
    const size_t scr_off = nbuf * tile_bytes;
    const size_t cells_off = scr_off + (scr ? static_cast<size_t>(NG) * (elem << M) : 0);
    const size_t bar_off = (cells_off + (back ? static_cast<size_t>(P.ngrad) * CS * 8 : 0) + 15) & ~size_t{15};
    if (pipe) {
        s << "V* ring = (V*)smraw;\n";
        s << "unsigned long long* full = (unsigned long long*)(smraw + " << bar_off << ");\nunsigned long long* done = full + "
          << nbuf << ";\n";
    } else {
        s << "V* sx = (V*)smraw;\nV* sy = sx + " << (1 << M) << ";\n";
    }
    if (back) s << "double* sg = (double*)(smraw + " << cells_off << ");\n";
    // tile id -> (outer index, element base)
    s << "auto tile_geo = [&](u64 tile, u64& outer, i64& tb) {\n";
    if (P.nchunks == 1)
        s << "const u64 o = tile; const u64 c = 0;\n";
    else
        s << "const u64 o = tile / " << P.nchunks << "ull; const u64 c = tile - o * " << P.nchunks << "ull;\n";
    s << "outer = o;\n";
    for (int k = 0; k < P.mq; ++k) {
        int p = P.qpos[k];
        s << "outer = ((outer >> " << p << ") << " << p + 1 << ") | (outer & " << hex((uint64_t{1} << p) - 1) << ");\n";
    }
    s << "tb = (i64)outer * " << P.B << "ll + (i64)c * " << (int64_t{1} << P.nb) << "ll;\n};\n";
    s << "auto c_of = [&](u64 tile) -> u64 { return " << (P.nchunks == 1 ? std::string("0ull") : "tile % " + std::to_string(P.nchunks) + "ull")
      << "; };\n";
    if (pipe) {
        int64_t gw[32];
        for (int b = 0; b < M; ++b) gw[b] = b < P.nb ? (int64_t{1} << b) : (P.B << P.qpos[b - P.nb]);
        s << "if (tid_all == 0) { for (int i = 0; i < " << nbuf << "; ++i) { mbar_init(full + i, " << (use_tma ? 1 : NP)
          << "); mbar_init(done + i, 1); } }\n";
        if (back) s << "for (int i = tid_all; i < " << P.ngrad * CS << "; i += " << NG * TH + NP << ") sg[i] = 0.0;\n";
        s << "__syncthreads();\npdl_wait();\n";  // the previous pass's writes are visible after this
        s << "if (tid_all >= " << NG * TH << ") {  // producer warpgroup\n";
        if (NG > 1 && 65536 / (NG * TH + NP) / 8 * 8 > producer_regs()) s << "reg_dealloc<" << producer_regs() << ">();\n";
        s << "const int lane = tid_all - " << NG * TH << ";\n";
        // with TMA only lane 0 issues copies: producer warps 1..3 retire here instead of spinning on the
        // slot barriers (24% of the reverse pass's executed instructions were such spins, taking issue
        // slots from the FP64 warps on their SMSPs; profiles/r02/ncu_baseline/bwd_instruction_mix.txt)
        if (use_tma && (!pstore || tstore)) s << "if (lane >= 32) return;\n";
        // iteration it: store the results of tile it - nbuf (slot computed), then load tile it
        s << "const u64 nt = (" << P.ntiles << "ull - blockIdx.x + gridDim.x - 1) / gridDim.x;\n";
        // element l = lane + NP*k (linear local index): thread part once, k part literal
        int64_t lp[8] = {0};
        int nlb = 0;
        while ((1 << nlb) < NP) ++nlb;
        for (int b = 0; b < nlb; ++b) lp[b] = gw[b];
        std::string gp = tid_sum(lp, nlb, false);
        for (size_t at = gp.find("tid"); at != std::string::npos; at = gp.find("tid", at)) gp.replace(at, 3, "lane");
        s << "const i64 gp = " << gp << ";\nconst unsigned sl = swz(lane);\n";
        s << "for (u64 it = 0; it < nt" << (pstore ? " + " + std::to_string(nbuf) : std::string()) << "; ++it) {\n";
        s << "const unsigned slot = (unsigned)(it % " << nbuf << "), use = (unsigned)(it / " << nbuf << ");\n";
        s << "V* buf = ring + (size_t)slot * " << tile_elems << "u;\n";
        s << "if (use > 0) {\nmbar_wait(done + slot, (use - 1u) & 1u);\n";
        if (pstore) s << "u64 outer; i64 tb; tile_geo(blockIdx.x + (it - " << nbuf << ") * gridDim.x, outer, tb);\n";
        auto kgo = [&](int k) {
            int64_t gk = 0;
            for (int b = nlb; b < M; ++b)
                if (((static_cast<int64_t>(k) * NP) >> b) & 1) gk += gw[b];
            return gk;
        };
        if (pstore && tstore && ck) raise(QBG_ERR_INTERNAL, "jit: checkpointed pass with a TMA drain");
        if (pstore && tstore) {
            // one elected thread: the computed tile (linear layout) back as one TMA tensor store, and
            // its shared-memory reads retired before the slot is refilled
            s << "if (lane == 0) {\nconst u64 ptile = blockIdx.x + (it - " << nbuf << ") * gridDim.x;\n";
            s << "tma_store" << td.size() << (back ? "(&tmp" : "(outm") << ", buf, " << tma_coords("outer", "ptile") << ");\n";
            if (back) s << "tma_store" << td.size() << "(&tma, buf + " << (1 << M) << ", " << tma_coords("outer", "ptile") << ");\n";
            s << "tma_commit();\ntma_wait_read0();\n}\n";
        } else if (pstore) {
            // element by element: shared-memory read, then its global store
            for (int k = 0; k < (1 << M) / NP; ++k) {
                const uint32_t sk = swz(static_cast<uint32_t>(k * NP));
                if (!ck)
                    s << "{ const V d = buf[SI(sl ^ " << sk << "u)]; " << (back ? "psi" : "outp") << "[GI(tb + gp + "
                      << kgo(k) << "ll)] = d;";
                else
                    s << "{";
                if (back)
                    s << " const V e = buf[SI(" << (1 << M) << " + (sl ^ " << sk << "u))]; adj[GI(tb + gp + " << kgo(k)
                      << "ll)] = e;";
                s << " }\n";
            }
            if (use_tma) s << "fence_proxy_async();\n";
            s << "group_bar<" << NP << ">(" << 2 + NG << ");\n";  // slot read out before it is refilled
        }
        s << "}\n";
        s << "if (it < nt) {\nu64 outer; i64 tb; tile_geo(blockIdx.x + it * gridDim.x, outer, tb);\n";
        if (use_tma) {
            // one thread: expect the tile's bytes, then one (two) bulk tensor copies
            s << "if (lane == 0) {\nmbar_arrive_tx(full + slot, " << tile_bytes << "u);\n";
            const std::string co = tma_coords("outer", "(blockIdx.x + it * gridDim.x)");
            s << "tma_load" << td.size() << "(buf, &tmp, full + slot, " << co << ");\n";
            if (back) s << "tma_load" << td.size() << "(buf + " << (1 << M) << ", &tma, full + slot, " << co << ");\n";
            s << "}\n}\n";
        }
        if (!use_tma) {
            for (int k = 0; k < (1 << M) / NP; ++k) {
                s << "cpa(buf + SI(lane + " << k * NP << "), psi + GI(tb + gp + " << kgo(k) << "ll));";
                if (back) s << " cpa(buf + SI(" << (1 << M) << " + lane + " << k * NP << "), adj + GI(tb + gp + " << kgo(k) << "ll));";
                s << "\n";
            }
            s << "cp_arrive_noinc(full + slot);\n}\n";
        }
        if (tstore) s << "}\nif (lane == 0) tma_wait0();\nreturn;\n}\n";
        else s << "}\nreturn;\n}\n";
        if (NG > 1) {
            // ptxas gives a setmaxnreg kernel the launch-bound register count L per thread; the
            // consumers may grow only into what the producer frees (else TRY_ALLOC never succeeds)
            const int L = 65536 / (NG * TH + NP) / 8 * 8;
            const int inc = ((NG * TH + NP) * L - NP * producer_regs()) / (NG * TH) / 8 * 8;
            if (inc > L) s << "reg_alloc<" << std::min(inc, 248) << ">();\n";
        }
        s << "const int cg = tid_all / " << TH << ", tid = tid_all & " << TH - 1 << ";\n";
        if (scr) s << "V* const scr = (V*)(smraw + " << scr_off << ") + (size_t)cg * " << (1 << M) << "u;\n";
        if (back) s << "const int warp = cg * " << NW << " + (tid >> 5), lane = tid & 31;\n";
    } else if (back) {
        s << "for (int i = tid; i < " << P.ngrad * CS << "; i += " << TH << ") sg[i] = 0.0;\n" << SYNC;
        s << "const int warp = tid >> 5, lane = tid & 31;\n";
    }
    // hoisted thread parts of every stage's offsets
    const DStage& S0 = P.st[0];
    const DStage& SL = P.st[P.nstages - 1];
    s << "const i64 g0 = " << tid_sum(S0.gthr, W, false) << ";\n";
    s << "const i64 gL = " << tid_sum(SL.gthr, W, false) << ";\n";
    for (int k = 0; k < P.nstages; ++k) s << "const unsigned st" << k << " = " << tid_sum(P.st[k].sthr, W, true) << ";\n";
    if (pipe) {
        uint32_t lw[kMaxW];
        for (int p = 0; p < W; ++p) lw[p] = 1u << S0.lthr[p];
        s << "const unsigned lin0 = " << tid_sum(lw, W, true) << ";\n";
        if (ck) {
            for (int p = 0; p < W; ++p) lw[p] = 1u << SL.lthr[p];
            s << "const unsigned linL = " << tid_sum(lw, W, true) << ";\n";
        }
    }
    s << "V x[R];\n" << (back ? "V y[R];\n" : "");
    auto goff = [&](const DStage& S, int j) {
        int64_t o = 0;
        for (int k = 0; k < RB; ++k)
            if ((j >> k) & 1) o += S.greg[k];
        return o;
    };
    auto loff = [&](const DStage& S, int j) {
        uint32_t o = 0;
        for (int k = 0; k < RB; ++k)
            if ((j >> k) & 1) o |= 1u << S.lreg[k];
        return o;
    };
    // the fold map (DPass::nfold) of a local offset, and the per-thread / per-tile parts of a
    // folded stage-0 read (forward) or scratch write (reverse)
    auto fmap = [&](uint32_t l) {
        uint32_t o = 0;
        for (int k = 0; k < M; ++k)
            if ((l >> k) & 1) o ^= P.nfold ? P.fcol[k] : 1u << k;
        return o;
    };
    auto fthr = [&](const DStage& S) {
        uint32_t w[kMaxW];
        for (int p = 0; p < W; ++p) w[p] = fmap(1u << S.lthr[p]);
        return tid_sum(w, W, true);
    };
    auto ftile = [&]() {
        std::ostringstream o;
        o << (P.nfold ? P.fd : 0u) << "u";
        for (int i = 0; i < P.nfo; ++i)
            o << " ^ (((outer >> " << int(P.foq[i]) << ") & 1ull) ? " << P.fow[i] << "u : 0u)";
        return o.str();
    };
    auto soff = [&](const DStage& S, int j) {
        uint32_t o = 0;
        for (int k = 0; k < RB; ++k)
            if ((j >> k) & 1) o ^= S.sreg[k];
        return o;
    };
    // diagnostics only (QBG_EXP): 1 = no global traffic (synthetic tile, stores never taken),
    // 2 = no gate ops (pure load / transpose / store) — splits a pass into compute and memory time;
    // checkpointed reverse passes: 4 = no transposes, 7 = no statistics, 8 = no uncompute ops,
    // 9 = at most two statistics groups, 10 = slot released before the statistics
    const int exp_mode = env_int("QBG_EXP", 0);
    if (!pipe) {
        s << "pdl_wait();\n";
        s << "for (u64 tile = blockIdx.x; tile < " << P.ntiles << "ull; tile += gridDim.x) {\n";
        s << "u64 outer; i64 tb; tile_geo(tile, outer, tb);\n";
        for (int j = 0; j < R; ++j) {
            if (exp_mode == 1) {
                s << "x[" << j << "] = mk<V>((double)(tid + " << j << ") * 1e-3, (double)tile * 1e-9);";
                if (back) s << " y[" << j << "] = mk<V>((double)(tid - " << j << ") * 1e-3, 1e-9);";
            } else {
                s << "x[" << j << "] = psi[GI(tb + g0 + " << goff(S0, j) << "ll)];";
                if (back) s << " y[" << j << "] = adj[GI(tb + g0 + " << goff(S0, j) << "ll)];";
            }
            s << "\n";
        }
    } else {
        s << "for (u64 it = cg;; it += " << NG << ") {\n";
        s << "const u64 tile = blockIdx.x + it * gridDim.x;\nif (tile >= " << P.ntiles << "ull) break;\n";
        s << "const unsigned slot = (unsigned)(it % " << nbuf << "), use = (unsigned)(it / " << nbuf << ");\n";
        // A slot alternates between the two consumer groups (nbuf odd): the previous use of this slot
        // belongs to the other group, whose fill may still be in flight when this group gets here.
        // A parity wait two phases ahead would pass at once, so first wait until that previous use
        // has been released (done[slot] phase use-1); then the full-phase parity is unambiguous.
        if (NG > 1 && nbuf % NG != 0) s << "if (use > 0) mbar_wait(done + slot, (use - 1u) & 1u);\n";
        s << "mbar_wait(full + slot, use & 1u);\n";
        s << "V* sx = ring + (size_t)slot * " << tile_elems << "u; V* sy = sx + " << (1 << M) << ";\n";
        s << "u64 outer; i64 tb; tile_geo(tile, outer, tb);\n";
        if (!ck) {
            for (int j = 0; j < R; ++j) {  // stage 0 from the linear (copied) layout
                if (exp_mode == 5 || exp_mode == 6) {  // (diagnostics: synthetic tile, no slot reads / global stores)
                    s << "x[" << j << "] = mk<V>((double)(tid + " << j << ") * 1e-3, (double)tile * 1e-9);";
                    if (back) s << " y[" << j << "] = mk<V>((double)(tid - " << j << ") * 1e-3, 1e-9);";
                } else if (P.nfold && !back) {  // folded permutations: the affine slot address
                    if (j == 0) s << "const unsigned lin0f = (" << fthr(S0) << ") ^ (" << ftile() << ");\n";
                    s << "x[" << j << "] = sx[SI(lin0f ^ " << fmap(loff(S0, j)) << "u)];";
                } else {
                    s << "x[" << j << "] = sx[SI(lin0 | " << loff(S0, j) << "u)];";
                    if (back) s << " y[" << j << "] = sy[SI(lin0 | " << loff(S0, j) << "u)];";
                }
                s << "\n";
            }
            if (P.nstages > 1) s << SYNC;  // the transposes overwrite the slot
        }
    }
    // register tile <-> shared memory: written with stage a's layout, read back with stage b's
    std::string ybuf = "sy";  // where φ̄'s transposes go (checkpointed, after the slot release: scr)
    auto transpose = [&](int a, int b, bool tx, bool ty) {
        const DStage& Sa = P.st[a];
        const DStage& Sb = P.st[b];
        for (int j = 0; j < R; ++j) {
            if (tx) s << "sx[SI(st" << a << " ^ " << soff(Sa, j) << "u)] = x[" << j << "];";
            if (ty) s << " " << ybuf << "[SI(st" << a << " ^ " << soff(Sa, j) << "u)] = y[" << j << "];";
            s << "\n";
        }
        s << SYNC;
        for (int j = 0; j < R; ++j) {
            if (tx) s << "x[" << j << "] = sx[SI(st" << b << " ^ " << soff(Sb, j) << "u)];";
            if (ty) s << " y[" << j << "] = " << ybuf << "[SI(st" << b << " ^ " << soff(Sb, j) << "u)];";
            s << "\n";
        }
        s << SYNC;
    };
    bool ex = true, ey = back;  // the states a gate op acts on (x = ψ, y = φ̄; checkpointed: φ̄ only)
    std::string cfix;           // statistics of a lane-flipped register slot: per-lane component fix-up
    auto emit_op = [&](const DOp& op) {
            const int o = op.mat;
            std::ostringstream ctl;
            bool has_ctl = false;
            if (op.cthr_mask) {
                ctl << "(((unsigned)tid & " << op.cthr_mask << "u) == " << op.cthr_val << "u)";
                has_ctl = true;
            }
            if (op.ctile_mask) {
                if (has_ctl) ctl << " && ";
                ctl << "((outer & " << hex(op.ctile_mask) << ") == " << hex(op.ctile_val) << ")";
                has_ctl = true;
            }
            const std::string cond = has_ctl ? ctl.str() : "true";
            const std::string t5 = std::to_string(op.creg_mask) + ", " + std::to_string(op.creg_val);
            // planner invariants the templates rely on (a violation is a planner bug: fail at plan
            // time, on the host, instead of generating undefined register indexing)
            {
                const bool reg_a = op.code == OP_DENSE1 || op.code == OP_X1 || op.code == OP_PERM1 ||
                                   op.code == OP_DIAG1R || op.code == OP_DENSE2 || op.code == OP_DENSE3 || op.code == OP_DENSE4 ||
                                   op.code == G_DENSE1 ||
                                   op.code == G_DIAG1R || op.code == G_DENSE2 || op.code == G_CROSS1 ||
                                   op.code == G_CROSSH || (op.code == G_CROSSD && op.b == LOC_REG);
                const bool reg_b = op.code == OP_DENSE2 || op.code == G_DENSE2 || op.code == OP_DENSE3 || op.code == OP_DENSE4;
                const bool reg_c = op.code == OP_DENSE3 || op.code == OP_DENSE4;
                const bool reg_d = op.code == OP_DENSE4;
                if ((reg_a && op.a >= RB) || (reg_b && op.b >= RB) || (reg_c && (op.aux & 0xff) >= static_cast<uint64_t>(RB)) ||
                    (reg_d && ((op.aux >> 8) & 0xff) >= static_cast<uint64_t>(RB)) ||
                    (op.creg_mask >> RB) != 0 ||
                    (op.cthr_mask >> W) != 0 || ((op.code == OP_DIAG1T || (op.code == G_CROSSD && op.b == LOC_THR)) && op.a >= W))
                    raise(QBG_ERR_INTERNAL, "fused plan: op " + std::to_string(op.code) + " refers to a register / thread slot "
                                            "outside the stage layout");
            }
            auto both = [&](const std::string& call_x, const std::string& call_y) {
                if (ex) s << call_x;
                if (ey) s << " " << call_y;
            };
            auto mvs = [&](int base, int n) {
                std::ostringstream t;
                for (int k = 0; k < n; ++k) t << (k ? ", " : "") << "MV(" << base + k << ")";
                return t.str();
            };
            switch (op.code) {
                case OP_DENSE1: {
                    s << "if (" << cond << ") { const V m00 = MV(" << o << "), m10 = MV(" << o + 1 << "), m01 = MV(" << o + 2
                      << "), m11 = MV(" << o + 3 << "); ";
                    std::string tp = "<V, R, " + std::to_string(op.a) + ", " + t5 + ">";
                    both("dense1" + tp + "(x, m00, m10, m01, m11);", "dense1" + tp + "(y, m00, m10, m01, m11);");
                    s << " }\n";
                    break;
                }
                case OP_X1: {
                    std::string tp = "<V, R, " + std::to_string(op.a) + ", " + t5 + ">";
                    s << "if (" << cond << ") { ";
                    both("swap1" + tp + "(x);", "swap1" + tp + "(y);");
                    s << " }\n";
                    break;
                }
                case OP_PERM1: {
                    std::string tp = "<V, R, " + std::to_string(op.a) + ", " + t5 + ">";
                    s << "if (" << cond << ") { ";
                    if (op.b) both("swap1" + tp + "(x);", "swap1" + tp + "(y);");
                    both("diag1" + tp + "(x, MV(" + std::to_string(o) + "), MV(" + std::to_string(o + 1) + "));",
                         "diag1" + tp + "(y, MV(" + std::to_string(o) + "), MV(" + std::to_string(o + 1) + "));");
                    s << " }\n";
                    break;
                }
                case OP_DIAG1R: {
                    std::string tp = "<V, R, " + std::to_string(op.a) + ", " + t5 + ">";
                    s << "if (" << cond << ") { ";
                    both("diag1" + tp + "(x, MV(" + std::to_string(o) + "), MV(" + std::to_string(o + 1) + "));",
                         "diag1" + tp + "(y, MV(" + std::to_string(o) + "), MV(" + std::to_string(o + 1) + "));");
                    s << " }\n";
                    break;
                }
                case OP_DIAG1T:
                case OP_DIAG1G: {
                    std::string bit = op.code == OP_DIAG1T ? "((tid >> " + std::to_string(op.a) + ") & 1)"
                                                           : "((outer >> " + std::to_string(op.a) + ") & 1ull)";
                    s << "if (" << cond << ") { const V d = " << bit << " ? MV(" << o + 1 << ") : MV(" << o << "); ";
                    both("scale<V, R, " + t5 + ">(x, d);", "scale<V, R, " + t5 + ">(y, d);");
                    s << " }\n";
                    break;
                }
                case OP_DENSE3:
                case OP_DENSE4: {
                    const bool four = op.code == OP_DENSE4;
                    std::string tp = "<V, R, " + std::to_string(op.a) + ", " + std::to_string(op.b) + ", " +
                                     std::to_string(op.aux & 0xff) +
                                     (four ? ", " + std::to_string((op.aux >> 8) & 0xff) : std::string()) + ", " + t5 + ">";
                    const std::string fn = four ? "dense4" : "dense3";
                    s << "if (" << cond << ") { const V m[" << (four ? 256 : 64) << "] = {" << mvs(o, four ? 256 : 64) << "}; ";
                    both(fn + tp + "(x, m);", fn + tp + "(y, m);");
                    s << " }\n";
                    break;
                }
                case OP_DENSE2: {
                    std::string tp = "<V, R, " + std::to_string(op.a) + ", " + std::to_string(op.b) + ", " + t5 + ">";
                    s << "if (" << cond << ") { const V m[16] = {" << mvs(o, 16) << "}; ";
                    both("dense2" + tp + "(x, m);", "dense2" + tp + "(y, m);");
                    s << " }\n";
                    break;
                }
                case OP_DIAGK:
                case G_DIAGK: {
                    // per element: index from register bits (literal) | thread / tile bits (runtime)
                    std::ostringstream rt;
                    int regpart_mask[8] = {0};
                    rt << "0";
                    for (int q = 0; q < op.t; ++q) {
                        uint32_t loc = static_cast<uint32_t>((op.aux >> (8 * q)) & 0xff);
                        uint32_t ty = loc >> 6, pos = loc & 63;
                        if (ty == LOC_THR) rt << " | (((tid >> " << pos << ") & 1) << " << q << ")";
                        if (ty == LOC_TILE) rt << " | ((int)((outer >> " << pos << ") & 1ull) << " << q << ")";
                        if (ty == LOC_REG) regpart_mask[q] = 1;
                    }
                    const bool grad = op.code == G_DIAGK;
                    s << "{ " << (grad ? "double g = 0.0; " : "") << "if (" << cond << ") { const int ib = " << rt.str() << "; ";
                    for (int j = 0; j < R; ++j) {
                        if ((j & op.creg_mask) != op.creg_val) continue;
                        int lit = 0;
                        for (int q = 0; q < op.t; ++q) {
                            uint32_t loc = static_cast<uint32_t>((op.aux >> (8 * q)) & 0xff);
                            if (regpart_mask[q] && ((j >> (loc & 63)) & 1)) lit |= 1 << q;
                        }
                        s << "{ const int ix = " << o << " + (ib | " << lit << "); const V d = mk<V>(pm.m[2 * ix], pm.m[2 * ix + 1]); ";
                        if (grad)
                            s << "g += imcm(y[" << j << "], cmul(d, x[" << j << "])); }";
                        else {
                            if (ex) s << "x[" << j << "] = cmul(x[" << j << "], d);";
                            if (ey) s << " y[" << j << "] = cmul(y[" << j << "], d);";
                            s << " }";
                        }
                    }
                    s << " }";
                    if (grad) s << " g = warp_sum(g); sg_acc(&sg[" << op.gslot * CS << " + warp], g, lane == 0);";
                    s << " }\n";
                    break;
                }
                case G_CROSS1: {
                    s << "{ double c[8] = {0, 0, 0, 0, 0, 0, 0, 0}; if (" << cond << ") gcross1<V, R, " << int(op.a)
                      << ">(x, y, c); " << cfix << "const double v = warp_sum8(c, lane); sg_acc(&sg[(" << op.gslot
                      << " + (lane >> 2)) * " << CS << " + warp], v, (lane & 3) == 0); }\n";
                    break;
                }
                case G_CROSSD: {
                    std::string call;
                    if (op.b == LOC_REG)
                        call = "gcrossd_r<V, R, " + std::to_string(op.a) + ">(x, y, c);";
                    else if (op.b == LOC_THR)
                        call = "gcrossd_u<V, R>(x, y, c, (tid >> " + std::to_string(op.a) + ") & 1);";
                    else
                        call = "gcrossd_u<V, R>(x, y, c, (int)((outer >> " + std::to_string(op.a) + ") & 1ull));";
                    s << "{ double c[4] = {0, 0, 0, 0}; if (" << cond << ") " << call << " " << cfix
                      << "const double v = warp_sum4(c, lane); sg_acc(&sg[(" << op.gslot
                      << " + (lane >> 3)) * " << CS << " + warp], v, (lane & 7) == 0); }\n";
                    break;
                }
                case G_CROSSH: {
                    if (exp_mode == 3) {  // (diagnostics: statistics without the warp reduction)
                        s << "{ double c[4] = {0, 0, 0, 0}; if (" << cond << ") gcrossh<V, R, " << int(op.a)
                          << ">(x, y, c); if (c[0] + c[1] + c[2] + c[3] == 1.2345) sg[" << op.gslot * CS << " + warp] += 1.0; }\n";
                        break;
                    }
                    s << "{ double c[4] = {0, 0, 0, 0}; if (" << cond << ") " << "gcrossh1"
                      << "<V, R, " << int(op.a)
                      << ">(x, y, c); " << cfix << "const double v = warp_sum4(c, lane); sg_acc(&sg[(" << op.gslot
                      << " + (lane >> 3)) * " << CS << " + warp], v, (lane & 7) == 0); }\n";
                    break;
                }
                case G_DENSE1:
                case G_DIAG1R:
                case G_DIAG1U:
                case G_DENSE2: {
                    s << "{ double g = 0.0; if (" << cond << ") { ";
                    if (op.code == G_DENSE1)
                        s << "g = gdense1<V, R, " << int(op.a) << ", " << t5 << ">(x, y, " << mvs(o, 4) << ");";
                    else if (op.code == G_DIAG1R)
                        s << "g = gdiag1<V, R, " << int(op.a) << ", " << t5 << ">(x, y, " << mvs(o, 2) << ");";
                    else if (op.code == G_DIAG1U)
                        s << "const V d = " << (op.b == 0 ? "((tid >> " + std::to_string(op.a) + ") & 1)"
                                                          : "((outer >> " + std::to_string(op.a) + ") & 1ull)")
                          << " ? MV(" << o + 1 << ") : MV(" << o << "); g = gscale<V, R, " << t5 << ">(x, y, d);";
                    else
                        s << "const V m[16] = {" << mvs(o, 16) << "}; g = gdense2<V, R, " << int(op.a) << ", " << int(op.b)
                          << ", " << t5 << ">(x, y, m);";
                    s << " } g = warp_sum(g); sg_acc(&sg[" << op.gslot * CS << " + warp], g, lane == 0); }\n";
                    break;
                }
                default:
                    raise(QBG_ERR_INTERNAL, "jit: unknown op");
            }
    };
    auto is_stat = [](const DOp& op) { return op.code >= G_DENSE1; };
    int cur = 0;  // checkpointed pass: the stage layout the registers hold at the store
    if (!ck) {
        for (int st = 0; st < P.nstages; ++st) {
            const DStage& S = P.st[st];
            if (st > 0 && exp_mode != 4 && exp_mode != 6) transpose(st - 1, st, true, back);  // (QBG_EXP=4/6: none)
            for (int i = S.op_begin; i < (exp_mode == 2 ? S.op_begin : S.op_end); ++i) emit_op(ops[i]);
        }
    } else {
        // Checkpointed reverse pass (plan_passes' ck rule): every gradient statistic of the pass is
        // taken first, against the checkpointed ψ (x) and the incoming φ̄ (y), visiting the stages
        // that hold statistics from the last to the first (the tile arrives in the last stage's
        // layout); then φ̄ alone is uncomputed through the stages in order.  ψ is neither
        // uncomputed nor stored: 28 instead of 44 FP64 instructions per element pair and rotation run.
        // The statistics need no stage layout of the uncompute: their qubits are grouped RB at a time,
        // and each group reads ψ and φ̄ from the tile's linear image in the slot (read-only, no
        // transposes) with its own register layout.  Bank conflicts: the local bits below nlow
        // select the 16-B bank group; those in thread bits take lanes 0.., those in register bits are
        // XOR-ed per lane with a lane bit whose own local bit is high ("flipped" slots), so the 8
        // lanes of every quarter warp hit 8 distinct groups.  A flipped slot swaps the roles of its
        // qubit's values 0 and 1 in that lane: fixed up on the statistic before the warp reduction.
        struct StatOp {
            DOp op;
            int lbit;  // the run qubit's local bit (-1: a tile-outer bit)
        };
        std::vector<StatOp> rops, dops;  // runs needing a register slot / diagonal runs
        bool generic = false;            // other gradient ops (controlled generators): stage layouts
        for (int st = 0; st < P.nstages; ++st)
            for (int i = P.st[st].op_begin; i < P.st[st].op_end; ++i) {
                const DOp& op = ops[i];
                if (!is_stat(op)) continue;
                const DStage& S = P.st[st];
                if (op.creg_mask || op.cthr_mask || op.ctile_mask) generic = true;
                if (op.code == G_CROSSH || op.code == G_CROSS1)
                    rops.push_back({op, S.lreg[op.a]});
                else if (op.code == G_CROSSD)
                    dops.push_back({op, op.b == LOC_REG ? S.lreg[op.a] : op.b == LOC_THR ? S.lthr[op.a] : -1});
                else
                    generic = true;
            }
        if (!generic) {
            const int nlow = c128 ? 3 : 4;
            int ngroups = rops.empty() ? (dops.empty() ? 0 : 1) : static_cast<int>((rops.size() + RB - 1) / RB);
            if (exp_mode == 7) ngroups = 0;  // (diagnostics: checkpointed pass without its statistics)
            if (exp_mode == 9) ngroups = std::min(ngroups, 2);  // (diagnostics: at most two groups)
            if (exp_mode == 10 && scr) {  // (diagnostics: slot released before the statistics; wrong results)
                if (use_tma) s << "fence_proxy_async();\n";
                s << "if (tid == 0) mbar_arrive(done + slot);\n";
            }
            for (int g = 0; g < ngroups; ++g) {
                std::vector<int> rb;  // register slot k -> local bit
                for (size_t r = static_cast<size_t>(g) * RB; r < rops.size() && rb.size() < static_cast<size_t>(RB); ++r)
                    rb.push_back(rops[r].lbit);
                auto in_rb = [&](int b) { return std::find(rb.begin(), rb.end(), b) != rb.end(); };
                for (int b = M - 1; b >= nlow && static_cast<int>(rb.size()) < RB; --b)
                    if (!in_rb(b)) rb.push_back(b);
                for (int b = 0; b < M && static_cast<int>(rb.size()) < RB; ++b)
                    if (!in_rb(b)) rb.push_back(b);
                std::vector<int> th;  // thread bit p -> local bit: the low ones first
                for (int b = 0; b < nlow; ++b)
                    if (!in_rb(b)) th.push_back(b);
                for (int b = nlow; b < M; ++b)
                    if (!in_rb(b)) th.push_back(b);
                if (static_cast<int>(th.size()) != W) raise(QBG_ERR_INTERNAL, "jit: statistics group layout");
                uint32_t w[kMaxW];
                for (int p = 0; p < W; ++p) w[p] = 1u << th[p];
                int flip_lane[kMaxR];  // lane bit XOR-ed into register slot k (-1: none)
                std::fill(flip_lane, flip_lane + kMaxR, -1);
                int nextp = 0;
                while (nextp < nlow && nextp < W && th[nextp] < nlow) ++nextp;
                for (int k = 0; k < RB; ++k)
                    if (rb[k] < nlow && nextp < nlow && nextp < W) {
                        flip_lane[k] = nextp;
                        w[nextp] ^= 1u << rb[k];
                        ++nextp;
                    }
                auto lo = [&](int j) {
                    uint32_t o = 0;
                    for (int k = 0; k < RB; ++k)
                        if ((j >> k) & 1) o |= 1u << rb[k];
                    return o;
                };
                s << "{ const unsigned lg = " << tid_sum(w, W, true) << ";\n";
                for (int j = 0; j < R; ++j)
                    s << "x[" << j << "] = sx[SI(lg ^ " << lo(j) << "u)]; y[" << j << "] = sy[SI(lg ^ " << lo(j) << "u)];\n";
                auto fix = [&](int k, int code) -> std::string {
                    if (flip_lane[k] < 0) return std::string();
                    const std::string f = "((tid >> " + std::to_string(flip_lane[k]) + ") & 1)";
                    if (code == G_CROSSH)
                        return "{ const bool f = " + f + "; const double t = c[0]; c[0] = f ? c[1] : t; c[1] = f ? t : c[1]; "
                               "c[3] = f ? -c[3] : c[3]; } ";
                    if (code == G_CROSSD) return "{ const bool f = " + f + "; const double t = c[0]; c[0] = f ? c[1] : t; c[1] = f ? t : c[1]; } ";
                    std::string r = "{ const bool f = " + f + ";";  // G_CROSS1: C_uv <-> C_(1-u)(1-v)
                    for (int pr : {0, 1, 2, 3}) {
                        const int a0 = pr < 2 ? pr : pr + 2, b0 = pr < 2 ? pr + 6 : pr + 2;
                        r += " { const double t = c[" + std::to_string(a0) + "]; c[" + std::to_string(a0) + "] = f ? c[" +
                             std::to_string(b0) + "] : t; c[" + std::to_string(b0) + "] = f ? t : c[" + std::to_string(b0) + "]; }";
                    }
                    return r + " } ";
                };
                const size_t r0 = static_cast<size_t>(g) * RB, r1 = std::min(rops.size(), r0 + RB);
                bool herm = r1 - r0 >= 2 && RB == 4;
                for (size_t r = r0; r < r1; ++r) herm = herm && rops[r].op.code == G_CROSSH;
                if (herm) {
                    // the group's Hermitian runs together: one pass over the pairs per slot, one
                    // 16-component warp reduction (lane l: run ((l >> 1) & 15) >> 2, component l/2 & 3)
                    const int nk = static_cast<int>(r1 - r0);
                    s << "{ double c[16]; gstat_group<V, R, " << nk << ">(x, y, c);\n";
                    for (int k = 0; k < nk; ++k) {
                        std::string fx = fix(k, G_CROSSH);
                        for (size_t at = fx.find("c["); at != std::string::npos; at = fx.find("c[", at + 2)) {
                            const size_t e = fx.find(']', at);
                            const int ci = std::stoi(fx.substr(at + 2, e - at - 2));
                            fx.replace(at, e - at + 1, "c[" + std::to_string(4 * k + ci) + "]");
                        }
                        s << fx;
                    }
                    // the runs' statistic slots (< kMaxComps = 256) packed in one immediate: a ternary
                    // chain here compiled to branches that split the statistics code (0.40 -> 0.38 ms)
                    uint32_t pack = 0;
                    for (int k = 0; k < nk; ++k) pack |= static_cast<uint32_t>(rops[r0 + k].op.gslot) << (8 * k);
                    s << "const double v = warp_sum16(c, lane); const int m = (lane >> 1) & 15, rr = m >> 2; const int gs = (int)(("
                      << pack << "u >> (8 * rr)) & 255u); sg_acc(&sg[(gs + (m & 3)) * " << CS << " + warp], v, (lane & 1) == 0 && rr < "
                      << nk << "); }\n";
                } else {
                    for (size_t r = r0; r < r1; ++r) {
                        DOp o2 = rops[r].op;
                        o2.a = static_cast<uint8_t>(r - r0);
                        cfix = fix(o2.a, o2.code);
                        emit_op(o2);
                    }
                }
                if (g == 0)
                    for (const StatOp& d : dops) {
                        DOp o2 = d.op;
                        cfix.clear();
                        if (d.lbit >= 0) {
                            const int k = static_cast<int>(std::find(rb.begin(), rb.end(), d.lbit) - rb.begin());
                            if (k < RB) {
                                o2.b = LOC_REG;
                                o2.a = static_cast<uint8_t>(k);
                                cfix = fix(k, G_CROSSD);
                            } else {
                                o2.b = LOC_THR;
                                o2.a = static_cast<uint8_t>(std::find(th.begin(), th.end(), d.lbit) - th.begin());
                            }
                        }
                        emit_op(o2);
                    }
                cfix.clear();
                s << "}\n";
            }
            for (int j = 0; j < R; ++j) s << "y[" << j << "] = sy[SI(lin0 | " << loff(S0, j) << "u)];\n";
            if (P.nstages > 1) s << SYNC;  // the transposes overwrite the slot
        } else {
            // generic: the stages that hold statistics, from the last (the tile arrives in the last
            // stage's linear layout) to the first, transposing ψ and φ̄ between them
            std::vector<int> vis;
            for (int st = P.nstages - 1; st >= 0; --st)
                for (int i = P.st[st].op_begin; i < P.st[st].op_end; ++i)
                    if (is_stat(ops[i])) {
                        vis.push_back(st);
                        break;
                    }
            if (!vis.empty()) {
                cur = P.nstages - 1;
                for (int j = 0; j < R; ++j)
                    s << "x[" << j << "] = sx[SI(linL | " << loff(SL, j) << "u)]; y[" << j << "] = sy[SI(linL | "
                      << loff(SL, j) << "u)];\n";
            } else {
                for (int j = 0; j < R; ++j) s << "y[" << j << "] = sy[SI(lin0 | " << loff(S0, j) << "u)];\n";
            }
            if (P.nstages > 1) s << SYNC;  // the transposes overwrite the slot
            for (int st : vis) {
                if (st != cur) {
                    transpose(cur, st, true, true);
                    cur = st;
                }
                for (int i = P.st[st].op_begin; i < P.st[st].op_end; ++i)
                    if (is_stat(ops[i])) emit_op(ops[i]);
            }
        }
        if (scr) {
            // every read of the slot is done: release it (the producer refills it during the sweep).
            // With the TMA store, the group's previous store must have read the scratch before the
            // sweep writes it again (it had the whole statistics phase to do so).
            if (use_tma) s << "fence_proxy_async();\nif (tid == 0) tma_wait_read0();\n";
            s << SYNC;
            if (exp_mode != 10 || generic) s << "if (tid == 0) mbar_arrive(done + slot);\n";
            ybuf = "scr";
        }
        ex = false;
        for (int st = 0; st < P.nstages; ++st) {
            bool any = false;
            for (int i = P.st[st].op_begin; i < P.st[st].op_end; ++i) any |= !is_stat(ops[i]);
            if (!any && st != P.nstages - 1) continue;
            if (st != cur) {
                if (exp_mode != 4) transpose(cur, st, false, true);  // (QBG_EXP=4: no transposes)
                cur = st;
            }
            for (int i = P.st[st].op_begin; i < P.st[st].op_end; ++i)
                if (!is_stat(ops[i]) && exp_mode != 8) emit_op(ops[i]);  // (QBG_EXP=8: no uncompute)
        }
    }
    if (pstore) {
        // results go back into the slot (swizzled: element l at swz(l)); the producer writes
        // them to global memory while this group computes its next tile
        const int ls = P.nstages - 1;
        if (P.nstages == 1) s << SYNC;  // other threads may still read stage 0 from the slot
        if (tstore) {  // linear layout (the TMA box order); the last stage's thread bits hold the low qubits
            uint32_t lwl[kMaxW];
            for (int p = 0; p < W; ++p) lwl[p] = 1u << SL.lthr[p];
            s << "{ const unsigned linL = " << tid_sum(lwl, W, true) << ";\n";
            for (int j = 0; j < R; ++j) {
                s << "sx[SI(linL | " << loff(SL, j) << "u)] = x[" << j << "];";
                if (back) s << " sy[SI(linL | " << loff(SL, j) << "u)] = y[" << j << "];";
                s << "\n";
            }
            s << "}\n";
        } else {
            for (int j = 0; j < R; ++j) {
                if (!ck) s << "sx[SI(st" << ls << " ^ " << soff(SL, j) << "u)] = x[" << j << "];";
                if (back) s << " sy[SI(st" << ls << " ^ " << soff(SL, j) << "u)] = y[" << j << "];";
                s << "\n";
            }
        }
        if (use_tma) s << "fence_proxy_async();\n";
        s << SYNC << "if (tid == 0) mbar_arrive(done + slot);\n";
    } else {
        if (exp_mode == 1 || exp_mode == 5 || exp_mode == 6) s << "if (outer == ~0ull) {\n";
        if (rstore) {
            // checkpointed reverse pass: φ̄ into the group's scratch in the tile's linear (TMA box)
            // layout — through the fold map when the pass ends with folded permutations — then one
            // TMA tensor store by one thread
            const DStage& SC = P.st[cur];
            s << "{ const unsigned linS = (" << fthr(SC) << ") ^ (" << ftile() << ");\n";
            for (int j = 0; j < R; ++j) s << "scr[SI(linS ^ " << fmap(loff(SC, j)) << "u)] = y[" << j << "];\n";
            s << "}\nfence_proxy_async();\n" << SYNC;
            s << "if (tid == 0) {\ntma_store" << td.size() << "(&tma, scr, " << tma_coords("outer", "tile") << ");\ntma_commit();\n}\n";
        } else {
            for (int j = 0; j < R; ++j) {
                if (!ck) s << (back ? "psi" : "outp") << "[GI(tb + gL + " << goff(SL, j) << "ll)] = x[" << j << "];";
                if (back) s << " adj[GI(tb + gL + " << goff(SL, j) << "ll)] = y[" << j << "];";
                s << "\n";
            }
        }
        if (exp_mode == 1 || exp_mode == 5 || exp_mode == 6) s << "}\n";
        if (pipe && !scr) {
            if (use_tma) s << "fence_proxy_async();\n";
            s << SYNC << "if (tid == 0) mbar_arrive(done + slot);\n";
        }
    }
    s << "}\n";  // tile loop
    if (rstore) s << "if (tid == 0) tma_wait0();\n";
    if (back) {
        if (pipe)
            s << "group_bar<" << NG * TH << ">(" << 1 + NG << ");\nconst int tc = tid_all;\n";
        else
            s << SYNC << "const int tc = tid;\n";
        s << "for (int sl = tc; sl < " << P.ngrad << "; sl += " << NG * TH
          << ") { double a = 0.0; for (int w = 0; w < " << NWT << "; ++w) a += sg[sl * " << CS
          << " + w]; gpart[(i64)(gbase + sl) * gcols + blockIdx.x] = a; }\n";
    }
    s << "#undef MV\n#undef GI\n#undef SI\n}\n";
    return s.str();
}

// Generates, compiles (cached) and attaches the specialised kernels of a plan.
// Algorithmic floating-point work of a pass (complex mul = 6, add = 2 flops; controls scale
// by the fraction of elements they select): forward ops on one state, reverse ops on two
// (uncompute of ψ and φ̄; one, φ̄, in a checkpointed pass: two = false) plus the gradient
// statistics once.  Reported beside the bytes.
double pass_flops(const DPass& P, const DOp* ops, int M, bool back) {
    double per_elem = 0;
    for (int i = 0; i < P.nops; ++i) {
        const DOp& o = ops[i];
        const double frac = std::ldexp(1.0, -(popc(o.creg_mask) + popc(o.cthr_mask) + popc(o.ctile_mask)));
        double f = 0;
        switch (o.code) {
            case OP_DENSE1: f = 14; break;
            case OP_PERM1: case OP_DIAG1R: case OP_DIAG1T: case OP_DIAG1G: case OP_DIAGK: f = 6; break;
            case OP_DENSE2: f = 30; break;
            case OP_DENSE3: f = 62; break;
            case OP_DENSE4: f = 126; break;
            case OP_X1: f = 0; break;
            default: f = 0;
        }
        if (o.code < G_DENSE1) {
            per_elem += frac * f * (back ? 2 : 1);
            continue;
        }
        switch (o.code) {
            case G_CROSSH: f = 12; break;
            case G_CROSS1: f = 16; break;
            case G_CROSSD: f = 4; break;
            case G_DENSE1: f = 17; break;
            case G_DENSE2: f = 33; break;
            default: f = 9;
        }
        per_elem += frac * f;
    }
    return per_elem * static_cast<double>(P.ntiles) * std::ldexp(1.0, M);
}

// Structure key of a pass: everything gen_pass reads (not the matrix values), so a new
// parameter vector finds its kernels without regenerating / hashing their source.
uint64_t pass_key(const DPass& P, const DOp* ops, int M, int RB, bool back, bool c128, bool ck) {
    uint64_t h = 1469598103934665603ULL;
    auto mix = [&](const void* p, size_t n) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) {
            h ^= c[i];
            h *= 1099511628211ULL;
        }
    };
    auto mixv = [&](int64_t v) { mix(&v, sizeof(v)); };
    const int W = M - RB;
    for (int64_t v : {int64_t{M}, int64_t{RB}, int64_t{back} + 2 * int64_t{ck}, int64_t{c128}, int64_t{P.nstages}, int64_t{P.ngrad},
                      int64_t{P.mq}, int64_t{P.nb}, P.B, P.nchunks, static_cast<int64_t>(P.ntiles), int64_t{P.nops},
                      int64_t{P.nmats}})
        mixv(v);
    mix(P.qpos, static_cast<size_t>(P.mq));
    for (int k = 0; k < P.nstages; ++k) {
        const DStage& S = P.st[k];
        mixv(S.op_begin);
        mixv(S.op_end);
        mix(S.sreg, sizeof(uint32_t) * RB);
        mix(S.sthr, sizeof(uint32_t) * W);
        mix(S.greg, sizeof(int64_t) * RB);
        mix(S.gthr, sizeof(int64_t) * W);
        mix(S.lreg, static_cast<size_t>(RB));
        mix(S.lthr, static_cast<size_t>(W));
    }
    mixv(P.nfold);
    if (P.nfold) {
        mix(P.fcol, sizeof(uint32_t) * M);
        mixv(P.fd);
        mixv(P.nfo);
        mix(P.foq, static_cast<size_t>(P.nfo));
        mix(P.fow, sizeof(uint32_t) * P.nfo);
    }
    mix(ops, sizeof(DOp) * static_cast<size_t>(P.nops));
    return h;
}

std::mutex g_pass_mu;
std::unordered_map<uint64_t, jit::Kernel> g_pass_kernels;  // pass_key -> loaded kernel

// The specialised kernel's matrix parameter (PM<T, 2*nmats>): the pass's matrices by value.
void fill_blob(Step& st, const std::vector<cdbl>& mats, bool c128) {
    const DPass& P = st.pass;
    const int nm2 = std::max(2, 2 * P.nmats);
    st.blob.assign(static_cast<size_t>(nm2) * (c128 ? 8 : 4), 0);
    for (int k = 0; k < P.nmats; ++k) {
        const cdbl& v = mats[P.mat_base + k];
        if (c128) {
            double* d = reinterpret_cast<double*>(st.blob.data());
            d[2 * k] = v.re;
            d[2 * k + 1] = v.im;
        } else {
            float* f = reinterpret_cast<float*>(st.blob.data());
            f[2 * k] = static_cast<float>(v.re);
            f[2 * k + 1] = static_cast<float>(v.im);
        }
    }
}

void jit_prepare(FusedPlan& pl, int M, int RB, bool back, bool c128, bool check_only = false) {
    const int NW = (1 << (M - RB)) / 32;
    const size_t elem = c128 ? 16 : 8;
    auto fill = [&](Step& st) {  // matrix parameter blob + shared memory of one step
        const DPass& P = st.pass;
        st.flops = pass_flops(P, pl.ops.data() + P.op_base, M, back && pl.dir != 5);
        fill_blob(st, pl.mats, c128);
        const size_t tile_bytes = (back ? 2 : 1) * (elem << M);
        const int nwt = (pipeline_enabled() ? consumer_groups(back) : 1) * NW;
        const size_t cells = back ? static_cast<size_t>(P.ngrad) * (nwt + 1) * 8 : 0;
        if (pipeline_enabled()) {
            const bool scr = pl.dir == 5 && ck_scratch();
            const int ng = consumer_groups(back);
            const int nbuf = scr ? ng : pipe_slots(back, M, c128, P.ngrad, nwt);
            const size_t scratch = scr ? static_cast<size_t>(ng) * (elem << M) : 0;
            st.smem = ((nbuf * tile_bytes + scratch + cells + 15) & ~size_t{15}) + 2 * nbuf * 8;
        } else {
            st.smem = (P.nstages > 1 || back ? tile_bytes : 0) + cells;
        }
    };
    std::vector<uint64_t> keys;
    if (!check_only) {
        bool all = true;
        {
            std::lock_guard<std::mutex> lk(g_pass_mu);
            for (auto& st : pl.steps) {
                if (!st.tile) continue;
                keys.push_back(pass_key(st.pass, pl.ops.data() + st.pass.op_base, M, RB, back, c128, pl.dir == 5));
                if (!g_pass_kernels.count(keys.back())) all = false;
            }
            if (all) {  // re-parameterised circuit: every kernel is known
                pl.jk.clear();
                size_t i = 0;
                for (auto& st : pl.steps) {
                    if (!st.tile) continue;
                    st.jk = static_cast<int>(pl.jk.size());
                    pl.jk.push_back(g_pass_kernels[keys[i++]]);
                    fill(st);
                }
                return;
            }
        }
    }
    std::map<uint64_t, int> uniq;  // body hash -> kernel index
    std::vector<std::string> names, bodies;
    for (auto& st : pl.steps) {
        if (!st.tile) continue;
        const DPass& P = st.pass;
        std::string body = gen_pass(P, pl.ops.data() + P.op_base, P.nmats, M, RB, back, c128, pl.dir == 5);
        uint64_t h = jit::fnv(body);
        auto it = uniq.find(h);
        if (it == uniq.end()) {
            char nm[40];
            std::snprintf(nm, sizeof(nm), "qbg_%016llx", static_cast<unsigned long long>(h));
            body.replace(body.find("__NAME__"), 8, nm);
            bodies.push_back(std::move(body));
            it = uniq.emplace(h, static_cast<int>(names.size())).first;
            names.push_back(nm);
        }
        st.jk = it->second;
        fill(st);
    }
    if (names.empty()) return;
    if (const char* d = std::getenv("QBG_JIT_SRC")) {  // diagnostics: keep the generated source
        std::ofstream f(std::string(d) + "/" + names[0] + ".cu");
        for (auto& b : bodies) f << b << "\n";
    }
    if (check_only) {
        jit::compile_only_parallel(bodies);
        return;
    }
    pl.jk = jit::compile_parallel(bodies, names);
    std::lock_guard<std::mutex> lk(g_pass_mu);
    size_t i = 0;
    for (auto& st : pl.steps)
        if (st.tile) g_pass_kernels[keys[i++]] = pl.jk[st.jk];
}

// ---- execution ---------------------------------------------------------------------------------
// Profiling label of a tile pass.  QBG_PROF_KERNELS=1 (diagnostics) splits the fused_fwd /
// fused_bwd totals of qbg_profile_report by pass structure: "<kind>:<stages>s<ops>o" plus the
// per-stage op counts, so one bench run times each pass type without a profiler.
const char* prof_name(const char* kind, const Step& st) {
    static const bool on = env_int("QBG_PROF_KERNELS", 0) != 0;
    if (!on) return kind;
    static std::mutex mu;
    static std::set<std::string> names;  // node-based: c_str() pointers stay valid
    std::string n = std::string(kind) + ":" + std::to_string(st.pass.nstages) + "s" + std::to_string(st.pass.nops) + "o[";
    for (int k = 0; k < st.pass.nstages; ++k)
        n += std::to_string(st.pass.st[k].op_end - st.pass.st[k].op_begin) + (k + 1 < st.pass.nstages ? " " : "]");
    std::lock_guard<std::mutex> lk(mu);
    return names.insert(n).first->c_str();
}
template <typename V, bool BACK>
void launch_jit(V* psi, V* adj, Step& st, FusedPlan& pl, double* gpart, int64_t gcols) {
    const int T = 1 << (pl.M - pl.RB);
    const DPass& P = st.pass;
    const bool pipe = pipeline_enabled();
    const int per_sm = pipe ? 1 : ctas_per_sm(BACK, T);
    int64_t grid = std::min<int64_t>(static_cast<int64_t>(P.ntiles), static_cast<int64_t>(num_sms()) * per_sm);
    if (BACK) grid = std::min<int64_t>(grid, gcols);
    // algorithmic bytes: ψ in/out (forward); ψ, φ̄ in/out (reverse); checkpointed reverse: ψ in, φ̄ in/out
    double bytes = static_cast<double>(P.ntiles) * (int64_t{1} << pl.M) * sizeof(V) * (BACK ? (pl.dir == 5 ? 3.0 : 4.0) : 2.0);
    int gbase = P.grad_base;
    alignas(64) unsigned char tmp[128] = {0}, tma[128] = {0};
    if (pipe && tma_enabled()) {
        std::vector<TmaDim> td;
        if (tma_layout(P, pl.M, sizeof(V) == 16, td)) {
            uint64_t sz[5], st[5];
            uint32_t bx[5];
            for (size_t d = 0; d < td.size(); ++d) {
                sz[d] = td[d].size;
                st[d] = td[d].stride;
                bx[d] = td[d].box;
            }
            jit::encode_tensor_map(tmp, psi, static_cast<int>(td.size()), sz, st, bx);
            if (adj) jit::encode_tensor_map(tma, adj, static_cast<int>(td.size()), sz, st, bx);
        }
    }
    void* args[] = {&psi, &adj, &gpart, &gcols, &gbase, st.blob.data(), tmp, tma};
    LaunchScope ls(prof_name(BACK ? "fused_bwd" : "fused_fwd", st), bytes, st.flops);
    jit::launch(pl.jk[st.jk], static_cast<unsigned>(grid), pipe ? consumer_groups(BACK) * T + kProducerThreads : T, st.smem,
                args);
    static const bool sync_each = env_int("QBG_SYNC_EACH", 0) != 0;  // diagnostics: localise a failing pass
    if (sync_each) {
        cudaError_t e = cudaStreamSynchronize(stream());
        if (e != cudaSuccess) {
            std::ostringstream m;
            m << "pass failed (" << (BACK ? "reverse" : "forward") << ", tile Q=";
            for (int k = 0; k < P.mq; ++k) m << (k ? "," : "") << int(P.qpos[k]);
            m << ", stages " << P.nstages << ", ops " << P.nops << ", ntiles " << P.ntiles << ", grid " << grid
              << ", smem " << st.smem << "): " << cudaGetErrorString(e);
            std::vector<TmaDim> td;
            if (tma_enabled() && tma_layout(P, pl.M, sizeof(V) == 16, td)) {
                m << "; tma rank " << td.size() << ":";
                for (auto& d : td) m << " [" << d.size << " x" << d.stride << "B box " << d.box << " c" << d.coord << "]";
            }
            raise(QBG_ERR_CUDA, m.str());
        }
    }
}

int batch_bits(int64_t B) {
    int nb = 0;
    while (nb < 5 && (B % (int64_t{2} << nb)) == 0) ++nb;
    return nb;
}

std::shared_ptr<FusedPlan> build_host_plan(const Program& p, const DevState& s, int dir);
std::shared_ptr<FusedPlan> build_mirror_plan(const Program& p, const FusedPlan& rev);
bool refresh_values(FusedPlan& pl, const Program& p);
void finalize_plan(FusedPlan& pl, const DevState& s, int dir);

std::shared_ptr<FusedPlan> get_plan(std::vector<std::shared_ptr<FusedPlan>>& cache, const Program& p,
                                    const DevState& s, int dir) {
    for (auto& c : cache)
        if (c->dir == dir && c->B == s.B && c->dtype == s.dtype && c->n == s.n && c->version == p.version) return c;
    static const bool refresh = env_int("QBG_PLAN_REFRESH", 1) != 0;  // 0: rebuild the plan on every new θ
    if (refresh)
        for (auto& c : cache)
            if (c->dir == dir && c->B == s.B && c->dtype == s.dtype && c->n == s.n && !c->msrc.empty() &&
                refresh_values(*c, p))
                return c;
    cache.erase(std::remove_if(cache.begin(), cache.end(),
                               [&](const std::shared_ptr<FusedPlan>& c) { return c->dir == dir && c->B == s.B; }),
                cache.end());
    auto pl = build_host_plan(p, s, dir);
    finalize_plan(*pl, s, dir);
    cache.push_back(pl);
    return pl;
}

// JIT kernels and device tables of a freshly planned plan.
void finalize_plan(FusedPlan& plr, const DevState& s, int dir) {
    FusedPlan* pl = &plr;
    const int M = pl->M, RB = pl->RB;
    const bool default_geo = M == (dir == 2 ? kBwdM : kFwdM) && RB == (dir == 2 ? kBwdRB : kFwdRB);
    if (!jit::enabled() && !default_geo) raise(QBG_ERR_UNSUPPORTED, "fused: non-default tile geometry needs the JIT");
    if (jit::enabled()) {
        try {
            jit_prepare(*pl, M, RB, dir == 2 || dir == 5, s.dtype == QBG_C128);
        } catch (const Error& e) {
            static bool warned = false;
            const char* strict = std::getenv("QBG_JIT_STRICT");
            if (strict && strict[0] == '1') throw;
            // the interpreter kernels know neither folded permutations nor the JIT-only stage ops:
            // such a plan must not fall back silently
            for (const auto& st : pl->steps) {
                if (!st.tile) continue;
                bool jit_only = st.pass.nfold != 0;
                for (int i = 0; i < st.pass.nops && !jit_only; ++i) {
                    const uint8_t c = pl->ops[st.pass.op_base + i].code;
                    jit_only = c == OP_DENSE3 || c == OP_DENSE4 || c == G_CROSSH;
                }
                if (jit_only) throw;
            }
            if (!warned) std::fprintf(stderr, "qbg: JIT specialisation failed, using the interpreter kernels: %s\n", e.what());
            warned = true;
            for (auto& st : pl->steps) st.jk = -1;
        }
    }
    pl->d_ops = upload(pl->ops);
    pl->d_mats = upload(pl->mats);
    pl->d_epi = upload(pl->epi);
    {
        int np = 0;
        for (auto& e : pl->epi) np = std::max(np, e.param + 1);
        pl->csr_ptr.assign(np + 1, 0);
        for (auto& e : pl->epi) pl->csr_ptr[e.param + 1]++;
        for (int k = 0; k < np; ++k) pl->csr_ptr[k + 1] += pl->csr_ptr[k];
        pl->csr_idx.assign(pl->epi.size(), 0);
        std::vector<int> cur(pl->csr_ptr.begin(), pl->csr_ptr.end() - 1);
        for (size_t k = 0; k < pl->epi.size(); ++k) pl->csr_idx[cur[pl->epi[k].param]++] = static_cast<int>(k);
        pl->d_ptr = upload(pl->csr_ptr);
        pl->d_idx = upload(pl->csr_idx);
    }
}

// The realised program as the planner's fused gate list (dir 0 forward, 1 adjoint, 2 reverse).
std::vector<PG> plan_gates(const Program& p, int dir) {
    const size_t N = p.real.size();
    std::vector<PG> gs;
    gs.reserve(N);
    for (size_t q = 0; q < N; ++q) {
        PG g;
        if (dir == 0) {
            g.g = &p.real[q].u;
            g.src.push_back(static_cast<int>(q));
        } else {
            const RealOp& r = p.real[N - 1 - q];
            g.g = &r.udag;
            g.src.push_back(static_cast<int>(N - 1 - q));
            if (dir == 2 && r.param >= 0) {
                g.k = &r.k;
                g.param = r.param;
            }
        }
        gs.push_back(std::move(g));
    }
    return fuse_runs(std::move(gs), dir == 2);
}

// The gate list of a checkpoint mirror plan: each segment's program ops in forward order, runs
// fused within the segment only.  seg_begin (optional) receives each segment's first gate.
std::vector<PG> mirror_gates(const Program& p, const std::vector<std::vector<int>>& part, std::vector<int>* seg_begin) {
    std::vector<PG> out;
    for (const auto& seg : part) {
        if (seg_begin) seg_begin->push_back(static_cast<int>(out.size()));
        std::vector<PG> gs;
        for (int i : seg) {
            PG g;
            g.g = &p.real[static_cast<size_t>(i)].u;
            g.src.push_back(i);
            gs.push_back(std::move(g));
        }
        for (PG& g : fuse_runs(std::move(gs), false)) out.push_back(std::move(g));
    }
    if (seg_begin) seg_begin->push_back(static_cast<int>(out.size()));
    return out;
}

// New θ on a program whose plan exists: when the fused gate list keeps its structure (pg_sig),
// the passes, ops and specialised kernels stay; only the matrix values, the cross-gradient
// matrices and the kernels' matrix parameters are rewritten (no plan_passes, no JIT lookup).
// Returns false when the structure changed (the caller rebuilds).
bool refresh_values(FusedPlan& pl, const Program& p) {
    std::vector<PG> gates = pl.dir == 4 ? mirror_gates(p, pl.part, nullptr) : plan_gates(p, pl.dir == 5 ? 2 : pl.dir);
    if (gates.size() != pl.sig.size()) return false;
    for (size_t i = 0; i < gates.size(); ++i)
        if (pg_sig(gates[i]) != pl.sig[i]) return false;
    std::vector<cdbl> mats;
    mats.reserve(pl.mats.size());
    for (const MatSrc& ms : pl.msrc) {
        const Gate& g = gates[ms.gi].gate();
        switch (ms.what) {
            case MS_G:
                mats.insert(mats.end(), g.m.begin(), g.m.end());
                break;
            case MS_GDENSE: {
                std::vector<cdbl> d = dense_of(g);
                mats.insert(mats.end(), d.begin(), d.end());
                break;
            }
            case MS_KDIAG: {
                const Gate& K = *gates[ms.gi].k;
                for (int r = 0; r < K.dim; ++r) mats.push_back(K.kind == QBG_MAT_IDENTITY ? cdbl{1, 0} : K.m[r]);
                break;
            }
            default: {
                std::vector<cdbl> d = dense_of(*gates[ms.gi].k);
                mats.insert(mats.end(), d.begin(), d.end());
            }
        }
    }
    if (mats.size() != pl.mats.size() || pl.esrc.size() != pl.epi.size())
        raise(QBG_ERR_INTERNAL, "fused plan: value refresh does not match the plan layout");
    for (size_t e = 0; e < pl.epi.size(); ++e)
        if (pl.esrc[e].first >= 0)
            std::memcpy(pl.epi[e].A, gates[pl.esrc[e].first].run[pl.esrc[e].second].A, sizeof(pl.epi[e].A));
    pl.mats.swap(mats);
    pl.gates = std::move(gates);
    const bool c128 = pl.dtype == QBG_C128;
    for (auto& st : pl.steps)
        if (st.tile) fill_blob(st, pl.mats, c128);
    // stream-ordered: passes of the previous θ still queued read the old values first
    if (!pl.mats.empty())
        QBG_CUDA(cudaMemcpyAsync(pl.d_mats, pl.mats.data(), pl.mats.size() * sizeof(cdbl), cudaMemcpyHostToDevice,
                                 stream()));
    if (!pl.epi.empty())
        QBG_CUDA(cudaMemcpyAsync(pl.d_epi, pl.epi.data(), pl.epi.size() * sizeof(GradEntry), cudaMemcpyHostToDevice,
                                 stream()));
    pl.version = p.version;
    return true;
}

// The values-only refresh of one segment of a mirror plan (dir 4): its fused gates, matrices and
// kernel parameters, so the checkpointed forward can launch segment k while the host refreshes
// segment k + 1.  False when the segment's structure changed (the caller rebuilds the plans).
bool refresh_segment(FusedPlan& pl, const Program& p, size_t k) {
    std::vector<PG> gs = mirror_gates(p, {pl.part[k]}, nullptr);
    const int g0 = pl.seg_gates[k], g1 = pl.seg_gates[k + 1];
    if (static_cast<int>(gs.size()) != g1 - g0) return false;
    for (size_t i = 0; i < gs.size(); ++i)
        if (pg_sig(gs[i]) != pl.sig[g0 + i]) return false;
    for (size_t i = 0; i < gs.size(); ++i) pl.gates[g0 + i] = std::move(gs[i]);
    const bool c128 = pl.dtype == QBG_C128;
    for (int si = pl.seg_steps[k]; si < pl.seg_steps[k + 1]; ++si) {
        Step& st = pl.steps[si];
        if (!st.tile) continue;
        size_t at = static_cast<size_t>(st.pass.mat_base);
        for (int m = st.msrc_begin; m < st.msrc_end; ++m) {
            const MatSrc& ms = pl.msrc[m];
            const Gate& g = pl.gates[ms.gi].gate();
            std::vector<cdbl> v = ms.what == MS_G ? g.m : dense_of(g);  // (mirror plans: no K matrices)
            if (at + v.size() > pl.mats.size()) raise(QBG_ERR_INTERNAL, "fused plan: segment refresh out of range");
            std::copy(v.begin(), v.end(), pl.mats.begin() + static_cast<std::ptrdiff_t>(at));
            at += v.size();
        }
        if (at != static_cast<size_t>(st.pass.mat_base + st.pass.nmats))
            raise(QBG_ERR_INTERNAL, "fused plan: segment refresh does not match the plan layout");
        fill_blob(st, pl.mats, c128);
        if (st.jk < 0 && st.pass.nmats)  // interpreter kernels read the device table
            QBG_CUDA(cudaMemcpyAsync(pl.d_mats + st.pass.mat_base, pl.mats.data() + st.pass.mat_base,
                                     st.pass.nmats * sizeof(cdbl), cudaMemcpyHostToDevice, stream()));
    }
    return true;
}

std::atomic<uint64_t> g_plan_serial{0};

// The forward mirror (dir 4) of a checkpointed reverse plan (dir 5): one segment per reverse step,
// in reverse order, applying the same program ops in forward order on the same tile qubits, so the
// state after segment k is exactly the ψ the matching reverse pass reads as its checkpoint.
std::shared_ptr<FusedPlan> build_mirror_plan(const Program& p, const FusedPlan& rev) {
    auto pl = std::make_shared<FusedPlan>();
    pl->version = p.version;
    pl->B = rev.B;
    pl->dtype = rev.dtype;
    pl->n = rev.n;
    pl->dir = 4;
    pl->serial = ++g_plan_serial;
    pl->mirror_of = rev.serial;
    for (size_t r = rev.steps.size(); r-- > 0;) {
        const Step& st = rev.steps[r];
        std::vector<int> src;
        uint64_t Q = 0;
        if (st.tile) {
            for (int gi : st.members) src.insert(src.end(), rev.gates[gi].src.begin(), rev.gates[gi].src.end());
            for (int k = 0; k < st.pass.mq; ++k) Q |= uint64_t{1} << st.pass.qpos[k];
        } else {
            src = rev.gates[st.single].src;
        }
        std::sort(src.begin(), src.end());
        pl->part.push_back(std::move(src));
        pl->part_q.push_back(Q);
    }
    std::vector<int> seg_begin;
    pl->gates = mirror_gates(p, pl->part, &seg_begin);
    pl->seg_gates = seg_begin;
    pl->sig.reserve(pl->gates.size());
    for (const PG& g : pl->gates) pl->sig.push_back(pg_sig(g));
    const int nb = batch_bits(rev.B);
    const Geo g = geo_for(0);
    pl->M = rev.M;
    pl->RB = g.RB;
    for (size_t k = 0; k < pl->part.size(); ++k) {
        pl->seg_steps.push_back(static_cast<int>(pl->steps.size()));
        std::vector<int> sel;
        for (int gi = seg_begin[k]; gi < seg_begin[k + 1]; ++gi) sel.push_back(gi);
        if (pl->part_q[k] == 0) {  // a single-gate reverse step: the same gate alone
            for (int gi : sel) {
                Step st;
                st.single = gi;
                st.seg = static_cast<int>(k);
                pl->steps.push_back(st);
            }
            continue;
        }
        while (!sel.empty()) {
            const size_t first = pl->steps.size();
            sel = emit_pass(*pl, pl->M, pl->RB, nb, false, g.coal, pl->part_q[k], sel);
            for (size_t i = first; i < pl->steps.size(); ++i) pl->steps[i].seg = static_cast<int>(k);
        }
    }
    pl->seg_steps.push_back(static_cast<int>(pl->steps.size()));
    return pl;
}

// The planner alone (no device, no JIT): used by get_plan and by the host-only preview.
std::shared_ptr<FusedPlan> build_host_plan(const Program& p, const DevState& s, int dir) {
    auto pl = std::make_shared<FusedPlan>();
    pl->version = p.version;
    pl->B = s.B;
    pl->dtype = s.dtype;
    pl->n = s.n;
    pl->dir = dir;
    pl->serial = ++g_plan_serial;
    pl->gates = plan_gates(p, dir == 5 ? 2 : dir);
    pl->sig.reserve(pl->gates.size());
    for (const PG& g : pl->gates) pl->sig.push_back(pg_sig(g));
    const int nb = batch_bits(s.B);
    const Geo g = geo_for(dir == 5 ? 2 : dir);
    pl->M = g.M;
    pl->RB = g.RB;
    plan_passes(*pl, g.M, g.RB, nb, dir >= 2, g.coal, dir == 5);
    // per-gate fallback steps with a scalar gradient get their own component rows
    for (auto& st : pl->steps)
        if (!st.tile && pl->gates[st.single].k) {
            st.single_comp = static_cast<int>(pl->ncomps++);
            GradEntry e{};
            e.type = 0;
            e.comp = st.single_comp;
            e.param = pl->gates[st.single].param;
            pl->epi.push_back(e);
            pl->esrc.push_back({-1, -1});
        } else if (!st.tile && !pl->gates[st.single].run.empty()) {
            raise(QBG_ERR_INTERNAL, "fused plan: untiled rotation run");
        }
    return pl;
}

bool fusable(const DevState& s, int M) {
    int nb = batch_bits(s.B);
    return s.n >= M - nb && s.n <= 62;
}

// src (optional): the input state when it is not s itself — the first pass then loads from src
// and stores to s (specialised tile kernels), else src is copied into s first.
template <typename V>
void run_forward(const DevState& s, FusedPlan& pl, const void* src) {
    V* psi = static_cast<V*>(s.ptr);
    static const bool oop = env_int("QBG_FWD_OOP", 1) != 0;  // 0: always copy, then in place
    if (src) {
        const Step* f = pl.steps.empty() ? nullptr : &pl.steps.front();
        if (oop && f && f->tile && f->jk >= 0) {
            launch_jit<V, false>(static_cast<V*>(const_cast<void*>(src)), psi, pl.steps.front(), pl, nullptr, 0);
        } else {
            QBG_CUDA(cudaMemcpyAsync(psi, src, s.bytes(), cudaMemcpyDeviceToDevice, stream()));
            src = nullptr;
        }
    }
    bool skip = src != nullptr;
    for (auto& st : pl.steps) {
        if (skip) {
            skip = false;
            continue;
        }
        if (st.tile)
            if (st.jk >= 0)
                launch_jit<V, false>(psi, nullptr, st, pl, nullptr, 0);
            else
                launch_interp(pl.dtype, false, psi, nullptr, st.pass, pl.d_ops, pl.d_mats, nullptr, 0);
        else
            launch_gate(s, pl.gates[st.single].gate());
    }
}

// arena (checkpointed plans, dir 5): reverse step r reads ψ from checkpoint r instead of psi
template <typename V>
void run_backward(const DevState& psi, const DevState& adj, FusedPlan& pl, double* d_grads, char* arena = nullptr) {
    const int64_t cols = static_cast<int64_t>(num_sms()) * 8;
    const int64_t total = pl.ncomps;
    double* part = static_cast<double*>(scratch(std::max<int64_t>(1, total) * cols * sizeof(double), 13));
    if (total) QBG_CUDA(cudaMemsetAsync(part, 0, total * cols * sizeof(double), stream()));
    for (size_t r = 0; r < pl.steps.size(); ++r) {
        Step& st = pl.steps[r];
        DevState ps = psi;
        if (arena) ps.ptr = arena + r * psi.bytes();
        if (st.tile) {
            if (st.jk >= 0)
                launch_jit<V, true>(static_cast<V*>(ps.ptr), static_cast<V*>(adj.ptr), st, pl, part, cols);
            else if (!arena)
                launch_interp(pl.dtype, true, ps.ptr, adj.ptr, st.pass, pl.d_ops, pl.d_mats, part, cols);
            else
                raise(QBG_ERR_INTERNAL, "fused: a checkpointed pass without its specialised kernel");
        } else {
            // (per-gate step; with checkpoints its uncompute of ψ only consumes checkpoint r)
            const PG& g = pl.gates[st.single];
            int used = 0;
            launch_gate_back(ps, adj, g.gate(), g.k, g.k ? part + st.single_comp * cols : nullptr, cols, &used);
        }
    }
    if (total) {
        double* sums = static_cast<double*>(scratch(total * sizeof(double), 12));
        launch_grad_rows(part, total, cols, sums);
        launch_grad_epilogue(sums, pl.d_epi, static_cast<int64_t>(pl.epi.size()), pl.d_ptr, pl.d_idx,
                             static_cast<int64_t>(pl.csr_ptr.size()) - 1, d_grads);
    }
}

}  // namespace

bool fused_forward(const DevState& s, Program& p, bool adjoint, const void* src) {
    if (!fusable(s, geo_for(0).M)) return false;
    auto pl = get_plan(p.plans, p, s, adjoint ? 1 : 0);
    if (s.dtype == QBG_C128)
        run_forward<double2>(s, *pl, src);
    else
        run_forward<float2>(s, *pl, src);
    return true;
}

bool fused_backward(const DevState& psi, const DevState& adj, Program& p, double* d_grads) {
    if (!fusable(psi, geo_for(2).M)) return false;
    auto pl = get_plan(p.plans, p, psi, 2);
    if (psi.dtype == QBG_C128)
        run_backward<double2>(psi, adj, *pl, d_grads);
    else
        run_backward<float2>(psi, adj, *pl, d_grads);
    return true;
}

// ---- checkpointed expect' (dir 4 forward mirror, dir 5 reverse) ---------------------------------
// The forward passes write the state after every reverse pass's segment (out of place, into an
// arena of checkpoints); each reverse pass then reads its ψ instead of uncomputing it.  Same HBM
// traffic per step as the uncompute design (3S + 3S per pass pair instead of 2S + 4S), 36% less
// FP64 in the reverse passes, and the caller's register is never modified.
namespace {
std::atomic<bool> g_ckpt_on{true};  // qbg_set_checkpointing
bool ckpt_enabled() {  // QBG_CKPT=0: the uncompute design (A/B)
    static const bool on = pipeline_enabled() && env_int("QBG_CKPT", 1) != 0;
    return on && g_ckpt_on.load();
}

std::shared_ptr<FusedPlan> get_mirror(Program& p, const DevState& s, const FusedPlan& rev) {
    for (auto& c : p.plans)
        if (c->dir == 4 && c->B == s.B && c->dtype == s.dtype && c->n == s.n && c->mirror_of == rev.serial &&
            (c->version == p.version || refresh_values(*c, p)))
            return c;
    p.plans.erase(std::remove_if(p.plans.begin(), p.plans.end(),
                                 [&](const std::shared_ptr<FusedPlan>& c) { return c->dir == 4 && c->B == s.B; }),
                  p.plans.end());
    auto pl = build_mirror_plan(p, rev);
    finalize_plan(*pl, s, 4);
    p.plans.push_back(pl);
    return pl;
}

template <typename V>
bool run_ckpt_forward(const DevState& in, FusedPlan& fw, char* arena, const Program* refresh = nullptr) {
    const size_t nseg = fw.part.size(), sb = in.bytes();
    const void* cur = in.ptr;
    for (size_t k = 0; k < nseg; ++k) {
        if (refresh && !refresh_segment(fw, *refresh, k)) return false;
        DevState d = in;
        d.ptr = arena + (nseg - 1 - k) * sb;  // checkpoint of reverse step nseg-1-k
        bool placed = false;
        for (int i = fw.seg_steps[k]; i < fw.seg_steps[k + 1]; ++i) {
            Step& st = fw.steps[i];
            if (!placed && st.tile && st.jk >= 0) {  // out of place: previous checkpoint -> this one
                launch_jit<V, false>(static_cast<V*>(const_cast<void*>(cur)), static_cast<V*>(d.ptr), st, fw, nullptr, 0);
                placed = true;
                continue;
            }
            if (!placed) {
                QBG_CUDA(cudaMemcpyAsync(d.ptr, cur, sb, cudaMemcpyDeviceToDevice, stream()));
                placed = true;
            }
            if (st.tile && st.jk >= 0)
                launch_jit<V, false>(static_cast<V*>(d.ptr), nullptr, st, fw, nullptr, 0);
            else if (st.tile)
                launch_interp(fw.dtype, false, d.ptr, nullptr, st.pass, fw.d_ops, fw.d_mats, nullptr, 0);
            else
                launch_gate(d, fw.gates[st.single].gate());
        }
        if (!placed) QBG_CUDA(cudaMemcpyAsync(d.ptr, cur, sb, cudaMemcpyDeviceToDevice, stream()));
        cur = d.ptr;
    }
    if (refresh) {
        if (!fw.mats.empty())  // the whole device table at once (only interpreter kernels read it)
            QBG_CUDA(cudaMemcpyAsync(fw.d_mats, fw.mats.data(), fw.mats.size() * sizeof(cdbl), cudaMemcpyHostToDevice,
                                     stream()));
        fw.version = refresh->version;
    }
    return true;
}
}  // namespace

void fused_set_checkpointing(bool on) { g_ckpt_on.store(on); }

// A new θ rewrites the values of both plans (refresh_values: the program's fused gates, their
// signatures, matrices and gradient matrices — host work of a few hundred µs per plan).  The
// reverse plan's refresh is deferred until the forward passes are queued (fused_ckpt_sync), so it
// overlaps them instead of delaying the step's first launch; the step count and the segments the
// forward needs are structure, which a value refresh never changes.
namespace {
std::shared_ptr<FusedPlan> peek_plan(Program& p, const DevState& s, int dir) {
    for (auto& c : p.plans)
        if (c->dir == dir && c->B == s.B && c->dtype == s.dtype && c->n == s.n) return c;
    return nullptr;
}
std::shared_ptr<FusedPlan> find_mirror(Program& p, const DevState& s, const FusedPlan& rev) {
    for (auto& c : p.plans)
        if (c->dir == 4 && c->B == s.B && c->dtype == s.dtype && c->n == s.n && c->mirror_of == rev.serial) return c;
    return nullptr;
}
}  // namespace

int64_t fused_ckpt_states(Program& p, const DevState& s) {
    if (!ckpt_enabled() || !fusable(s, geo_for(2).M)) return 0;
    auto rev = peek_plan(p, s, 5);
    if (!rev) rev = get_plan(p.plans, p, s, 5);
    for (auto& st : rev->steps)
        if (st.tile && st.jk < 0) return 0;  // (JIT unavailable: the interpreter has no checkpointed pass)
    return static_cast<int64_t>(rev->steps.size());
}

bool fused_ckpt_forward(const DevState& in, Program& p, void* arena, int64_t k) {
    auto rev = peek_plan(p, in, 5);
    if (!rev) rev = get_plan(p.plans, p, in, 5);
    auto fw = find_mirror(p, in, *rev);
    auto run = [&](FusedPlan& f, const Program* refresh) {
        return in.dtype == QBG_C128 ? run_ckpt_forward<double2>(in, f, static_cast<char*>(arena), refresh)
                                    : run_ckpt_forward<float2>(in, f, static_cast<char*>(arena), refresh);
    };
    // a new θ on a known structure: each segment is refreshed right before its passes are queued
    static const bool lazy = env_int("QBG_LAZY_REFRESH", 1) != 0;  // (0: the whole plan first; A/B)
    if (fw && fw->version != p.version && !fw->seg_gates.empty() && lazy && run(*fw, &p)) return true;
    if (!fw || !(fw->version == p.version || refresh_values(*fw, p))) {
        // first use, or the program's structure changed with θ: the reverse plan first
        rev = get_plan(p.plans, p, in, 5);
        if (static_cast<int64_t>(rev->steps.size()) != k) return false;
        fw = get_mirror(p, in, *rev);
    }
    return run(*fw, nullptr);
}

bool fused_ckpt_sync(Program& p, const DevState& s, int64_t k) {
    auto rev = get_plan(p.plans, p, s, 5);  // refresh (or rebuild: a new serial)
    auto fw = find_mirror(p, s, *rev);
    return fw && fw->version == p.version && static_cast<int64_t>(rev->steps.size()) == k;
}

void fused_ckpt_backward(const DevState& adj, Program& p, void* arena, double* d_grads) {
    auto rev = get_plan(p.plans, p, adj, 5);
    if (adj.dtype == QBG_C128)
        run_backward<double2>(adj, adj, *rev, d_grads, static_cast<char*>(arena));
    else
        run_backward<float2>(adj, adj, *rev, d_grads, static_cast<char*>(arena));
}

void fused_stats(const Program& p, int64_t* f, int64_t* b) {
    *f = 0;
    *b = 0;
    bool ck = false;
    for (auto& c : p.plans) ck |= c->dir == 5;
    for (auto& c : p.plans) {
        int64_t steps = static_cast<int64_t>(c->steps.size());
        if (c->dir == (ck ? 4 : 0)) *f = steps;
        if (c->dir == (ck ? 5 : 2)) *b = steps;
    }
}

namespace {
std::string plans_text(const std::vector<std::shared_ptr<FusedPlan>>& plans);
}

std::string fused_plan_info(const Program& p) { return plans_text(p.plans); }

std::string fused_plan_preview(const Program& p, int64_t B, int dtype) {
    DevState s;
    s.n = p.n;
    s.B = B;
    s.dtype = dtype;
    std::vector<std::shared_ptr<FusedPlan>> v;
    if (fusable(s, geo_for(0).M)) v.push_back(build_host_plan(p, s, 0));
    if (fusable(s, geo_for(2).M)) {
        v.push_back(build_host_plan(p, s, 2));
        if (env_int("QBG_CKPT", 1) != 0) {  // the checkpointed pair expect' runs when the checkpoints fit
            auto rev = build_host_plan(p, s, 5);
            v.push_back(build_mirror_plan(p, *rev));
            v.push_back(rev);
        }
    }
    return plans_text(v);
}

namespace {
std::string plans_text(const std::vector<std::shared_ptr<FusedPlan>>& plans) {
    std::ostringstream s;
    for (auto& c : plans) {
        s << "plan dir=" << c->dir << " B=" << c->B << " steps=" << c->steps.size() << " kernels=" << c->jk.size()
          << " comps=" << c->ncomps << "\n";
        for (auto& st : c->steps) {
            if (!st.tile) {
                s << "  single gate t=" << c->gates[st.single].gate().t << "\n";
                continue;
            }
            const DPass& P = st.pass;
            s << "  tile Q=";
            for (int k = 0; k < P.mq; ++k) s << int(P.qpos[k]) << (k + 1 < P.mq ? "," : "");
            s << " stages=" << P.nstages << " ops=" << P.nops << " [";
            for (int k = 0; k < P.nstages; ++k) s << P.st[k].op_end - P.st[k].op_begin << (k + 1 < P.nstages ? " " : "");
            s << "] comps=" << P.ngrad << " smem=" << st.smem;
            if (P.nfold) s << " fold=" << P.nfold;
            s << "\n";
            static const bool verbose = env_int("QBG_PREVIEW_OPS", 0) != 0;  // diagnostics: stage layouts, ops
            if (verbose)
                for (int k = 0; k < P.nstages; ++k) {
                    const DStage& S = P.st[k];
                    s << "    stage " << k << " reg=";
                    for (int r = 0; r < kMaxR && r < 4; ++r) s << int(S.lreg[r]) << (r < 3 ? "," : "");
                    s << " ops:";
                    for (int i = S.op_begin; i < S.op_end; ++i) {
                        const DOp& o = c->ops[P.op_base + i];
                        s << " " << int(o.code) << "(" << int(o.a) << "," << int(o.b) << ")";
                        if (o.creg_mask) s << "r" << o.creg_mask;
                        if (o.cthr_mask) s << "t" << o.cthr_mask;
                        if (o.ctile_mask) s << "g";
                    }
                    s << "\n";
                }
        }
    }
    return s.str();
}
}  // namespace

// ---- observable seed ------------------------------------------------------------------------------
namespace {

std::shared_ptr<FusedPlan> make_seed_plan(const Observable& o, const DevState& s, bool check_only, bool energy_only);
void seed_jit_prepare(FusedPlan& pl, bool c128, bool check_only);

std::shared_ptr<FusedPlan> get_seed_plan(Observable& o, const DevState& s, bool energy_only) {
    for (auto& c : o.plans)
        if (c->B == s.B && c->dtype == s.dtype && c->n == s.n && c->energy_only == energy_only) return c;
    auto pl = make_seed_plan(o, s, false, energy_only);
    o.plans.push_back(pl);
    return pl;
}

std::shared_ptr<FusedPlan> make_seed_plan(const Observable& o, const DevState& s, bool check_only, bool energy_only) {
    auto pl = std::make_shared<FusedPlan>();
    pl->B = s.B;
    pl->dtype = s.dtype;
    pl->n = s.n;
    pl->dir = 3;
    pl->energy_only = energy_only;
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
    if (check_only) {
        seed_jit_prepare(*pl, s.dtype == QBG_C128, true);
        return pl;
    }
    if (jit::enabled()) {
        try {
            seed_jit_prepare(*pl, s.dtype == QBG_C128, false);
        } catch (const Error& e) {
            const char* strict = std::getenv("QBG_JIT_STRICT");
            if (strict && strict[0] == '1') throw;
            std::fprintf(stderr, "qbg: JIT seed specialisation failed, using the generic kernel: %s\n", e.what());
            pl->sjk.clear();
        }
    }
    pl->d_groups = upload(pl->groups);
    pl->d_terms = upload(pl->terms);
    return pl;
}

// Specialised seed pass: the ψ tile is staged in shared memory (linear layout), each thread
// accumulates 2^M/256 elements l = tid + 256k of φ̄ in registers.  For a group with X support x
// and term Z supports z_t:  φ̄_l += Σ_t c_t (-1)^{|src & z_t|} ψ_src,  src = l ^ x.  The parity
// splits into a thread/tile part (per thread, once per tile) and a k part (compile time), and
// terms with equal k-part Z mask are pre-summed per thread.
// energy_only: every pass starts from zero and contributes Re Σ conj(ψ_l) (O_pass ψ)_l to the energy
// directly (the groups' contributions are independent), so φ is never written.
bool seed_tma(const SPass& sp, bool c128, std::vector<TmaDim>& td);
std::string gen_seed(const SPass& sp, const std::vector<SGroup>& groups, const std::vector<STerm>& terms, bool c128,
                     bool energy_only) {
    constexpr int M = kSeedM, TB = 8, T = 1 << TB, R = 1 << (M - TB);
    const int64_t bc = int64_t{1} << sp.nb;
    std::ostringstream s;
    int nterm = 0;
    for (int gi = sp.g0; gi < sp.g1; ++gi) nterm += groups[gi].term_end - groups[gi].term_begin;
    // Pipelined seed (complex128, tile a <= 5-D TMA box): one persistent CTA per SM, the ψ tile
    // double-buffered in shared memory and loaded by TMA one tile ahead, so the next tile's load
    // overlaps this tile's Pauli terms (the plain loop loads, synchronises, computes, stores).
    std::vector<TmaDim> td;
    const bool tpipe = seed_tma(sp, c128, td);
    const size_t tile_bytes = static_cast<size_t>(c128 ? 16 : 8) << M;
    s << "extern \"C\" __global__ void __launch_bounds__(" << T << ", " << (tpipe ? 1 : kSeedMinB) << ") __NAME__(const "
      << (c128 ? "c128" : "c64") << "* __restrict__ psi, " << (c128 ? "c128" : "c64")
      << "* __restrict__ phi, double* __restrict__ epart, const __grid_constant__ PM<" << (c128 ? "double" : "float")
      << ", " << std::max(2, 2 * nterm) << "> pm" << (tpipe ? ", const __grid_constant__ TMap tmp" : "") << ") {\n";
    s << "typedef " << (c128 ? "c128" : "c64") << " V;\nconst int tid = threadIdx.x;\n";
    s << "extern __shared__ __align__(128) unsigned char smraw[];\n__shared__ double red[" << T << "];\n";
    if (!tpipe) s << "V* sp = (V*)smraw;\n";
    // element offset of local index l: batch bits, then tile qubits
    auto goff = [&](uint32_t l) {
        int64_t e = l & (bc - 1);
        uint32_t q = l >> sp.nb;
        for (int k = 0; q; ++k, q >>= 1)
            if (q & 1) e += sp.B << sp.qpos[k];
        return e;
    };
    int64_t wt[TB];
    for (int p = 0; p < TB; ++p) wt[p] = goff(1u << p);
    s << "const i64 gt = " << tid_sum(wt, TB, false) << ";\n";
    s << "V acc[" << R << "];\n";
    // the tile's outer index (tile qubits deposited as zero bits) and batch chunk
    s << "auto geo = [&](u64 tile, u64& outer, u64& c) {\n";
    if (sp.nchunks == 1)
        s << "const u64 o = tile; c = 0;\n";
    else
        s << "const u64 o = tile / " << sp.nchunks << "ull; c = tile - o * " << sp.nchunks << "ull;\n";
    s << "outer = o;\n";
    for (int k = 0; k < sp.mq; ++k) {
        int p = sp.qpos[k];
        s << "outer = ((outer >> " << p << ") << " << p + 1 << ") | (outer & " << hex((uint64_t{1} << p) - 1) << ");\n";
    }
    s << "};\n";
    if (tpipe) {
        std::ostringstream co;  // TMA coordinates of a tile (outer, c), tma_layout's dimension order
        for (size_t d = 0; d < td.size(); ++d) {
            if (td[d].coord == 0) co << "0";
            else if (td[d].coord == 1) co << "(int)c2";
            else co << "(int)((o2 >> " << td[d].shift << ") & " << td[d].mask << "ull)";
            if (d + 1 < td.size()) co << ", ";
        }
        s << "V* const sb = (V*)smraw;\nunsigned long long* const fb = (unsigned long long*)(smraw + " << 2 * tile_bytes << ");\n";
        s << "if (tid == 0) { mbar_init(fb, 1); mbar_init(fb + 1, 1); }\n__syncthreads();\n";
        s << "pdl_wait();\n";
        s << "auto issue = [&](u64 t2, unsigned b2) { u64 o2, c2; geo(t2, o2, c2); mbar_arrive_tx(fb + b2, " << tile_bytes
          << "u); tma_load" << td.size() << "(sb + b2 * " << (1u << M) << "u, &tmp, fb + b2, " << co.str() << "); };\n";
        s << "if (tid == 0 && blockIdx.x < " << sp.ntiles << "ull) issue(blockIdx.x, 0u);\n";
        s << "u64 it = 0;\n";
        s << "for (u64 tile = blockIdx.x; tile < " << sp.ntiles << "ull; tile += gridDim.x, ++it) {\n";
        s << "const unsigned b = (unsigned)(it & 1);\n";
        // the other buffer was last read in the previous iteration (fenced and synchronised)
        s << "if (tid == 0 && tile + gridDim.x < " << sp.ntiles << "ull) issue(tile + gridDim.x, b ^ 1u);\n";
        s << "u64 outer, c; geo(tile, outer, c);\n";
        s << "const i64 tb = (i64)outer * " << sp.B << "ll + (i64)c * " << bc << "ll + gt;\n";
        for (int k = 0; k < R; ++k) {
            if (sp.first || energy_only)
                s << "acc[" << k << "] = mk<V>(0, 0);\n";
            else
                s << "acc[" << k << "] = phi[tb + " << goff(static_cast<uint32_t>(k) << TB) << "ll];\n";
        }
        s << "mbar_wait(fb + b, (unsigned)(it >> 1) & 1u);\nconst V* sp = sb + b * " << (1u << M) << "u;\n";
    } else {
        s << "pdl_wait();\n";  // launched with programmatic stream serialisation (jit::launch)
        s << "for (u64 tile = blockIdx.x; tile < " << sp.ntiles << "ull; tile += gridDim.x) {\n";
        s << "u64 outer, c; geo(tile, outer, c);\n";
        s << "const i64 tb = (i64)outer * " << sp.B << "ll + (i64)c * " << bc << "ll + gt;\n";
        s << "__syncthreads();\n";
        for (int k = 0; k < R; ++k) s << "sp[tid + " << k * T << "] = psi[tb + " << goff(static_cast<uint32_t>(k) << TB) << "ll];\n";
        for (int k = 0; k < R; ++k) {
            if (sp.first || energy_only)
                s << "acc[" << k << "] = mk<V>(0, 0);\n";
            else
                s << "acc[" << k << "] = phi[tb + " << goff(static_cast<uint32_t>(k) << TB) << "ll];\n";
        }
        s << "__syncthreads();\n";
    }
    // real coefficients (every Hermitian Pauli sum with i^{nY} folded in, e.g. heisenberg): the
    // per-element update is a real scale-accumulate, 2 FMA instead of a complex one's 4
    bool real = true;
    for (int gi = sp.g0; gi < sp.g1; ++gi)
        for (int t = groups[gi].term_begin; t < groups[gi].term_end; ++t) real = real && terms[t].cim == 0.0;
    const char* WT = real ? "RT<V>::T" : "V";
    int tix = 0;
    for (int gi = sp.g0; gi < sp.g1; ++gi) {
        const SGroup& g = groups[gi];
        const uint32_t xlow = g.xloc & (T - 1), xhigh = g.xloc >> TB;
        std::map<uint32_t, std::vector<int>> byh;
        for (int t = g.term_begin; t < g.term_end; ++t) byh[terms[t].zloc >> TB].push_back(t);
        s << "{\n";
        int hi = 0;
        std::vector<uint32_t> hs;
        for (auto& [h, ts] : byh) {
            s << WT << " W" << hi << " = " << (real ? "0" : "mk<V>(0, 0)") << ";\n";
            for (int t : ts) {
                const STerm& st = terms[t];
                const int pidx = tix + (t - g.term_begin);
                s << "{ const int par = (__popc((tid ^ " << xlow << "u) & " << (st.zloc & (T - 1)) << "u) + __popcll(outer & "
                  << hex(st.zout) << ")) & 1; ";
                if (real)
                    s << "const RT<V>::T c = pm.m[" << 2 * pidx << "]; W" << hi << " = par ? W" << hi << " - c : W" << hi
                      << " + c; }\n";
                else
                    s << "const V c = mk<V>(pm.m[" << 2 * pidx << "], pm.m[" << 2 * pidx + 1 << "]); W" << hi
                      << " = par ? mk<V>(W" << hi << ".x - c.x, W" << hi << ".y - c.y) : mk<V>(W" << hi << ".x + c.x, W" << hi
                      << ".y + c.y); }\n";
            }
            hs.push_back(h);
            ++hi;
        }
        for (int k = 0; k < R; ++k) {
            const uint32_t kk = static_cast<uint32_t>(k) ^ xhigh;
            s << "{ const V v = sp[(tid ^ " << xlow << "u) + " << (kk << TB) << "u]; ";
            if (real) {
                s << "RT<V>::T cf = 0;";
                for (size_t h = 0; h < hs.size(); ++h)
                    s << " cf " << ((__builtin_popcount(kk & hs[h]) & 1) ? "-" : "+") << "= W" << h << ";";
                s << " acc[" << k << "] = mk<V>(fma(cf, v.x, acc[" << k << "].x), fma(cf, v.y, acc[" << k << "].y)); }\n";
            } else {
                s << "V cf = mk<V>(0, 0);";
                for (size_t h = 0; h < hs.size(); ++h) {
                    const bool neg = __builtin_popcount(kk & hs[h]) & 1;
                    s << " cf = mk<V>(cf.x " << (neg ? "-" : "+") << " W" << h << ".x, cf.y " << (neg ? "-" : "+") << " W" << h
                      << ".y);";
                }
                s << " acc[" << k << "] = cfma(acc[" << k << "], cf, v); }\n";
            }
        }
        s << "}\n";
        tix += g.term_end - g.term_begin;
    }
    if (!energy_only)
        for (int k = 0; k < R; ++k) s << "phi[tb + " << goff(static_cast<uint32_t>(k) << TB) << "ll] = acc[" << k << "];\n";
    if (sp.last || energy_only) {
        s << "double e = 0.0;\n";
        for (int k = 0; k < R; ++k)
            s << "{ const V p = sp[tid + " << k * T << "]; e += (double)p.x * acc[" << k << "].x + (double)p.y * acc[" << k
              << "].y; }\n";
        s << "red[tid] = e;\n__syncthreads();\n";
        s << "if (tid < " << bc << ") { double t = 0.0; for (int m = tid; m < " << T << "; m += " << bc
          << ") t += red[m]; epart[tile * " << bc << "ull + tid] = t; }\n";
    }
    // (pipelined: every read of this buffer retired before the next TMA write into it)
    if (tpipe) s << "fence_proxy_async();\n__syncthreads();\n";
    s << "}\n}\n";
    return s.str();
}

// Whether a seed pass runs pipelined (TMA double buffer): complex128 tiles that are a TMA box.
bool seed_tma(const SPass& sp, bool c128, std::vector<TmaDim>& td) {
    static const bool on = env_int("QBG_SEED_TMA", 1) != 0;  // (0: the plain tile loop; A/B)
    if (!on || !c128 || !tma_enabled()) return false;
    DPass probe{};
    probe.mq = sp.mq;
    probe.nb = sp.nb;
    std::memcpy(probe.qpos, sp.qpos, sizeof(probe.qpos));
    probe.B = sp.B;
    probe.nchunks = sp.nchunks;
    probe.ntiles = sp.ntiles;
    return tma_layout(probe, kSeedM, true, td);
}

void seed_jit_prepare(FusedPlan& pl, bool c128, bool check_only) {
    std::map<uint64_t, int> uniq;
    std::vector<std::string> names;
    std::string src;
    std::vector<std::string> sbodies;
    pl.sjk.clear();
    pl.sblob.clear();
    for (auto& sp : pl.spasses) {
        std::string body = gen_seed(sp, pl.groups, pl.terms, c128, pl.energy_only);
        uint64_t h = jit::fnv(body);
        auto it = uniq.find(h);
        if (it == uniq.end()) {
            char nm[40];
            std::snprintf(nm, sizeof(nm), "qbs_%016llx", static_cast<unsigned long long>(h));
            std::string b = body;
            b.replace(b.find("__NAME__"), 8, nm);
            src += b;
            sbodies.push_back(std::move(b));
            it = uniq.emplace(h, static_cast<int>(names.size())).first;
            names.push_back(nm);
        }
        pl.sjk.push_back(it->second);
        std::vector<char> blob;
        int nterm = 0;
        for (int gi = sp.g0; gi < sp.g1; ++gi) nterm += pl.groups[gi].term_end - pl.groups[gi].term_begin;
        blob.assign(static_cast<size_t>(std::max(2, 2 * nterm)) * (c128 ? 8 : 4), 0);
        int tix = 0;
        for (int gi = sp.g0; gi < sp.g1; ++gi)
            for (int t = pl.groups[gi].term_begin; t < pl.groups[gi].term_end; ++t, ++tix) {
                if (c128) {
                    reinterpret_cast<double*>(blob.data())[2 * tix] = pl.terms[t].cre;
                    reinterpret_cast<double*>(blob.data())[2 * tix + 1] = pl.terms[t].cim;
                } else {
                    reinterpret_cast<float*>(blob.data())[2 * tix] = static_cast<float>(pl.terms[t].cre);
                    reinterpret_cast<float*>(blob.data())[2 * tix + 1] = static_cast<float>(pl.terms[t].cim);
                }
            }
        pl.sblob.push_back(std::move(blob));
    }
    if (check_only)
        jit::compile_only_parallel(sbodies);
    else
        pl.jk = jit::compile_parallel(sbodies, names);
}

void run_seed(const DevState& psi, const DevState& phi, FusedPlan& pl, double* d_energy) {
    const SPass& last = pl.spasses.back();
    const int64_t bc = int64_t{1} << last.nb;
    const int64_t per_pass = static_cast<int64_t>(last.ntiles) * bc;
    const int64_t npart = pl.energy_only ? static_cast<int64_t>(pl.spasses.size()) : 1;
    double* epart = static_cast<double*>(scratch(npart * per_pass * sizeof(double), 14));
    if (!pl.sjk.empty()) {
        for (size_t k = 0; k < pl.spasses.size(); ++k) {
            const SPass& sp = pl.spasses[k];
            const void* pp = psi.ptr;
            void* qq = phi.ptr;
            double* ep = epart + (pl.energy_only ? static_cast<int64_t>(k) * per_pass : 0);
            alignas(64) unsigned char tmp[128] = {0};
            std::vector<TmaDim> td;
            const bool tpipe = seed_tma(sp, psi.dtype == QBG_C128, td);
            if (tpipe) {
                uint64_t sz[5], stv[5];
                uint32_t bx[5];
                for (size_t d = 0; d < td.size(); ++d) {
                    sz[d] = td[d].size;
                    stv[d] = td[d].stride;
                    bx[d] = td[d].box;
                }
                jit::encode_tensor_map(tmp, const_cast<void*>(pp), static_cast<int>(td.size()), sz, stv, bx);
            }
            void* args[] = {&pp, &qq, &ep, pl.sblob[k].data(), tmp};
            int64_t grid = std::min<int64_t>(static_cast<int64_t>(sp.ntiles), static_cast<int64_t>(num_sms()) * (tpipe ? 1 : 2));
            static const bool by_pass = env_int("QBG_PROF_KERNELS", 0) != 0;  // (diagnostics: see prof_name)
            const char* nm = !by_pass ? "seed" : sp.first ? "seed:first" : sp.last ? "seed:last" : "seed:mid";
            LaunchScope ls(nm, (pl.energy_only ? 1.0 : sp.first ? 2.0 : 3.0) * psi.bytes());
            jit::launch(pl.jk[pl.sjk[k]], static_cast<unsigned>(grid), 256,
                        tpipe ? 2 * (psi.elem() << kSeedM) + 16 : psi.elem() << kSeedM, args);
        }
    } else {
        for (auto& sp : pl.spasses)
            launch_seed(psi.dtype, psi.ptr, phi.ptr, sp, pl.d_groups, pl.d_terms, epart,
                        (sp.first ? 2.0 : 3.0) * psi.bytes());
    }
    // energy-only passes each left their own partials: sum them as extra "outer" tiles
    if (d_energy)
        launch_energy(epart, (uint64_t{1} << (pl.n - last.mq)) * static_cast<uint64_t>(npart), last.nchunks, bc, psi.B,
                      d_energy);
}

}  // namespace

// Host-only: generate and NVRTC-compile (no device) every specialised kernel a program and an
// observable need on a 2^n x B register.  Returns the number of kernels source-compiled.
int64_t fused_jit_check(const Program& p, const Observable* o, int64_t B, int dtype) {
    DevState s;
    s.n = p.n;
    s.B = B;
    s.dtype = dtype;
    int64_t count = 0;
    if (fusable(s, geo_for(0).M)) {
        auto pl = build_host_plan(p, s, 0);
        jit_prepare(*pl, pl->M, pl->RB, false, dtype == QBG_C128, true);
        count += static_cast<int64_t>(pl->steps.size());
    }
    if (fusable(s, geo_for(2).M)) {
        auto pl = build_host_plan(p, s, 2);
        jit_prepare(*pl, pl->M, pl->RB, true, dtype == QBG_C128, true);
        count += static_cast<int64_t>(pl->steps.size());
        if (ckpt_enabled()) {  // the checkpointed pair (expect' when its checkpoints fit)
            auto rev = build_host_plan(p, s, 5);
            jit_prepare(*rev, rev->M, rev->RB, true, dtype == QBG_C128, true);
            auto fw = build_mirror_plan(p, *rev);
            jit_prepare(*fw, fw->M, fw->RB, false, dtype == QBG_C128, true);
            count += static_cast<int64_t>(rev->steps.size() + fw->steps.size());
        }
    }
    if (o && !o->terms.empty() && s.n >= kSeedM - batch_bits(B)) {
        for (bool energy_only : {false, true}) {  // expect' (φ̄ = Oψ) and expect (energies only)
            auto pl = make_seed_plan(*o, s, true, energy_only);
            count += static_cast<int64_t>(pl->spasses.size());
        }
    }
    return count;
}

bool fused_obs_apply(const DevState& psi, const DevState& phi, Observable& o, double* d_energy) {
    const int nb = batch_bits(psi.B);
    if (psi.n < kSeedM - nb || o.terms.empty()) return false;
    const bool energy_only = phi.ptr == nullptr;
    auto pl = get_seed_plan(o, psi, energy_only);
    if (energy_only && pl->sjk.empty()) return false;  // the generic seed kernel needs φ
    run_seed(psi, phi, *pl, d_energy);
    return true;
}

}  // namespace qbg
