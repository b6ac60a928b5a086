// qbg/blocks.hpp — the SPEC's block / autodiff / circuits API in C++  over the
// B200 engine.  Header-only, on top of qbg/qblock.hpp (the register shim) and the C-ABI.
//
//   Blocks: shared-ownership DAG nodes, `BlockPtr`.  Primitives X, Y, Z, H, I2,
//   S, Sdag, T, Tdag, SWAP, CNOT, CZ, Toffoli, P0, P1, Pu, Pd (gates.hpp:112-128), Rx/Ry/Rz/rot
//   (e^{-iΣθ/2}), shift, phase, matblock; composites chain, put, control, kron, repeat,
//   subroutine, add, scale, dagger (adjoint_block), cache.
//   Parameters: parameters / nparameters / dispatch(vec | op,vec | "random"),
//   depth-first, each distinct node once.
//   Evaluation: apply(reg, b), expect(obs, reg) / expect(obs, reg, circuit)
//   (452-460), expect_grad(obs, reg, circuit) -> GradResult{state_grad, param_grads} (479-487).
//   Circuits: variational_circuit(n, d), heisenberg(n, periodic), qft(n).
//
// apply does not issue one C call per primitive: the tree is lowered depth-first (Chain left to
// right; Put/Kron/Repeat/Subroutine remap locations; Control adds control masks) into ONE flat
// qbg_op program, compiled once by the engine (fusion plan + tile kernels) and cached on the block;
// dispatch only changes θ, which is re-synchronised on the next use.  The lowering is the same
// as the Python package's (blocks.py _lower), so both produce identical device programs.
#pragma once

#include <cmath>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "qblock.hpp"

namespace qbg {
namespace qblock {

struct Block;
using BlockPtr = std::shared_ptr<Block>;

enum class BlockKind {
    Constant, Rotation, Shift, Phase, Matrix,                              // primitives
    Chain, Put, Control, Kron, Repeat, Subroutine, Add, Scale, Daggered, Cached  // composites
};

namespace detail {
struct Compiled;     // a qbg_prog + the θ it was last realised at
struct CompiledObs;  // a qbg_obs (Pauli sum)
}  // namespace detail

struct Block {
    BlockKind kind = BlockKind::Constant;
    std::size_t nqubits = 0;
    std::string name;                    // Constant: registry name
    std::optional<MatrixRepr> mat;       // Constant / Matrix
    BlockPtr generator;                  // Rotation: Σ (hermitian, reflexive)
    double theta = 0.0;                  // Rotation / Shift / Phase
    std::vector<BlockPtr> children;      // Chain / Add / Kron: all; others: one
    std::vector<std::size_t> locs;       // Put / Control / Repeat / Subroutine
    std::vector<std::size_t> ctrl_locs;  // Control
    std::vector<int> ctrl_config;        // Control (1 = control, 0 = inverse control)
    std::vector<std::vector<std::size_t>> kron_locs;  // Kron: locations of children[k]
    cplx factor{1.0};                    // Scale
    // engine caches: structure is immutable after construction (only θ changes)
    mutable std::shared_ptr<detail::Compiled> compiled;
    mutable std::shared_ptr<detail::CompiledObs> observable;
    bool parameterised() const {
        return kind == BlockKind::Rotation || kind == BlockKind::Shift || kind == BlockKind::Phase;
    }
};

namespace detail {
inline void check_locs(std::size_t n, const std::vector<std::size_t>& locs, const char* what) {
    for (std::size_t i = 0; i < locs.size(); ++i) {
        if (locs[i] < 1 || locs[i] > n) throw RangeError(std::string(what) + ": location out of range");
        for (std::size_t j = 0; j < i; ++j)
            if (locs[j] == locs[i]) throw ValidationError(std::string(what) + ": duplicate location");
    }
}
inline std::size_t nq_of_dim(std::size_t d) {
    std::size_t q = 0;
    while ((std::size_t{1} << q) < d) ++q;
    if ((std::size_t{1} << q) != d) throw ValidationError("matrix dimension must be a power of 2");
    return q;
}
inline BlockPtr make(BlockKind k, std::size_t n) {
    auto b = std::make_shared<Block>();
    b->kind = k;
    b->nqubits = n;
    return b;
}
}  // namespace detail

// ---- primitives ---------------------------------------------------------------------------------------
// a constant gate node from the registry (a new node each call: define_const_gate may redefine a
// name, and constant nodes carry no parameters, so sharing them buys nothing)
inline BlockPtr constant(const std::string& name) {
    const ConstGateDef* def = find_gate(name);
    if (!def) throw DispatchError("unknown constant gate: " + name);
    auto b = detail::make(BlockKind::Constant, def->nqubits);
    b->name = name;
    b->mat = def->mat;
    return b;
}
inline BlockPtr X() { return constant("X"); }
inline BlockPtr Y() { return constant("Y"); }
inline BlockPtr Z() { return constant("Z"); }
inline BlockPtr H() { return constant("H"); }
inline BlockPtr I2() { return constant("I2"); }
inline BlockPtr S() { return constant("S"); }
inline BlockPtr Sdag() { return constant("Sdag"); }
inline BlockPtr T() { return constant("T"); }
inline BlockPtr Tdag() { return constant("Tdag"); }
inline BlockPtr SWAP() { return constant("SWAP"); }
inline BlockPtr CNOT() { return constant("CNOT"); }
inline BlockPtr CZ() { return constant("CZ"); }
inline BlockPtr Toffoli() { return constant("Toffoli"); }
inline BlockPtr P0() { return constant("P0"); }
inline BlockPtr P1() { return constant("P1"); }
inline BlockPtr Pu() { return constant("Pu"); }
inline BlockPtr Pd() { return constant("Pd"); }

inline BlockPtr rot(const BlockPtr& generator, double theta) {
    auto b = detail::make(BlockKind::Rotation, generator->nqubits);
    b->generator = generator;
    b->theta = theta;
    return b;
}
inline BlockPtr Rx(double theta) { return rot(X(), theta); }
inline BlockPtr Ry(double theta) { return rot(Y(), theta); }
inline BlockPtr Rz(double theta) { return rot(Z(), theta); }
inline BlockPtr shift(double theta) {
    auto b = detail::make(BlockKind::Shift, 1);
    b->theta = theta;
    return b;
}
inline BlockPtr phase(double theta) {
    auto b = detail::make(BlockKind::Phase, 1);
    b->theta = theta;
    return b;
}
inline BlockPtr matblock(const MatrixRepr& m) {
    auto b = detail::make(BlockKind::Matrix, detail::nq_of_dim(mat_dim(m)));
    b->mat = m;
    return b;
}

// ---- composites ----------------------------------------------------------------------------------------
inline BlockPtr chain(std::size_t n, std::vector<BlockPtr> blocks) {
    for (auto& c : blocks)
        if (c->nqubits != n) throw ShapeError("chain: child qubit count differs from the chain's");
    auto b = detail::make(BlockKind::Chain, n);
    b->children = std::move(blocks);
    return b;
}
inline BlockPtr chain(std::vector<BlockPtr> blocks) {
    if (blocks.empty()) throw ValidationError("chain: give the qubit count for an empty chain");
    const std::size_t n = blocks.front()->nqubits;
    return chain(n, std::move(blocks));
}
inline BlockPtr put(std::size_t n, std::vector<std::size_t> locs, const BlockPtr& blk) {
    detail::check_locs(n, locs, "put");
    if (locs.size() != blk->nqubits) throw ShapeError("put: location count differs from the block's qubit count");
    auto b = detail::make(BlockKind::Put, n);
    b->locs = std::move(locs);
    b->children = {blk};
    return b;
}
// control(n, ctrl_locs, locs => blk); a negative control location is an inverse control (Yao's -c)
inline BlockPtr control(std::size_t n, std::vector<long> ctrl, std::vector<std::size_t> locs, const BlockPtr& blk) {
    auto b = detail::make(BlockKind::Control, n);
    for (long c : ctrl) {
        b->ctrl_locs.push_back(static_cast<std::size_t>(c < 0 ? -c : c));
        b->ctrl_config.push_back(c < 0 ? 0 : 1);
    }
    std::vector<std::size_t> all = locs;
    all.insert(all.end(), b->ctrl_locs.begin(), b->ctrl_locs.end());
    detail::check_locs(n, all, "control");
    if (locs.size() != blk->nqubits) throw ShapeError("control: location count differs from the block's qubit count");
    b->locs = std::move(locs);
    b->children = {blk};
    return b;
}
inline BlockPtr control(std::size_t n, std::vector<std::size_t> ctrl_locs, std::vector<int> ctrl_config,
                        std::vector<std::size_t> locs, const BlockPtr& blk) {
    if (ctrl_locs.size() != ctrl_config.size())
        throw ValidationError("control: control locations and configuration differ in length");
    std::vector<long> c;
    for (std::size_t k = 0; k < ctrl_locs.size(); ++k) {
        if (ctrl_config[k] != 0 && ctrl_config[k] != 1) throw ValidationError("control: configuration must be 0 or 1");
        c.push_back(ctrl_config[k] ? static_cast<long>(ctrl_locs[k]) : -static_cast<long>(ctrl_locs[k]));
    }
    return control(n, std::move(c), std::move(locs), blk);
}
inline BlockPtr kron(std::size_t n, std::vector<std::pair<std::vector<std::size_t>, BlockPtr>> pairs) {
    auto b = detail::make(BlockKind::Kron, n);
    std::vector<std::size_t> all;
    for (auto& [l, c] : pairs) {
        if (l.size() != c->nqubits) throw ShapeError("kron: location count differs from the block's qubit count");
        all.insert(all.end(), l.begin(), l.end());
        b->kron_locs.push_back(l);
        b->children.push_back(c);
    }
    detail::check_locs(n, all, "kron");
    return b;
}
// kron(b1, b2, ...) on consecutive qubits (b1 on the lowest)
inline BlockPtr kron(std::vector<BlockPtr> blocks) {
    std::vector<std::pair<std::vector<std::size_t>, BlockPtr>> pairs;
    std::size_t q = 1;
    for (auto& c : blocks) {
        std::vector<std::size_t> l;
        for (std::size_t k = 0; k < c->nqubits; ++k) l.push_back(q++);
        pairs.emplace_back(std::move(l), c);
    }
    return kron(q - 1, std::move(pairs));
}
inline BlockPtr repeat(std::size_t n, const BlockPtr& blk, std::vector<std::size_t> locs = {}) {
    if (locs.empty())
        for (std::size_t q = 1; q <= n; ++q) locs.push_back(q);
    detail::check_locs(n, locs, "repeat");
    if (blk->nqubits != 1) throw ShapeError("repeat: the repeated block must act on one qubit");
    auto b = detail::make(BlockKind::Repeat, n);
    b->locs = std::move(locs);
    b->children = {blk};
    return b;
}
// Subroutine (Listing 16): focus(locs) -> apply child -> relax, i.e. the child on
// a local scope.  For a unitary child this is exactly put(n, locs => child), and it lowers so.
inline BlockPtr subroutine(std::size_t n, const BlockPtr& blk, std::vector<std::size_t> locs) {
    detail::check_locs(n, locs, "subroutine");
    if (locs.size() != blk->nqubits) throw ShapeError("subroutine: location count differs from the block's qubit count");
    auto b = detail::make(BlockKind::Subroutine, n);
    b->locs = std::move(locs);
    b->children = {blk};
    return b;
}
inline BlockPtr add(std::vector<BlockPtr> blocks) {
    auto b = detail::make(BlockKind::Add, 0);
    for (auto& c : blocks) {
        if (c->kind == BlockKind::Add)
            b->children.insert(b->children.end(), c->children.begin(), c->children.end());
        else
            b->children.push_back(c);
    }
    if (b->children.empty()) throw ValidationError("Add: needs at least one child");
    b->nqubits = b->children.front()->nqubits;
    for (auto& c : b->children)
        if (c->nqubits != b->nqubits) throw ShapeError("Add: children differ in qubit count");
    return b;
}
inline BlockPtr scale(cplx factor, const BlockPtr& blk) {
    auto b = detail::make(BlockKind::Scale, blk->nqubits);
    b->factor = factor;
    b->children = {blk};
    return b;
}
inline BlockPtr cache(const BlockPtr& blk) {
    auto b = detail::make(BlockKind::Cached, blk->nqubits);
    b->children = {blk};
    return b;
}
// operator product in matrix order: (A * B)|ψ> = A(B|ψ>)
inline BlockPtr operator*(const BlockPtr& a, const BlockPtr& b) { return chain(a->nqubits, {b, a}); }
inline BlockPtr operator*(cplx c, const BlockPtr& b) { return scale(c, b); }
inline BlockPtr operator+(const BlockPtr& a, const BlockPtr& b) { return add({a, b}); }

// adjoint_block
inline BlockPtr dagger(const BlockPtr& b) {
    using K = BlockKind;
    auto same = [&](K k) {
        auto o = detail::make(k, b->nqubits);
        *o = *b;
        o->compiled.reset();
        o->observable.reset();
        return o;
    };
    switch (b->kind) {
        case K::Constant: {
            static const std::map<std::string, std::string> pairs = {{"S", "Sdag"}, {"Sdag", "S"}, {"T", "Tdag"},
                                                                     {"Tdag", "T"}, {"Pu", "Pd"}, {"Pd", "Pu"}};
            static const char* herm[] = {"X", "Y", "Z", "H", "I2", "SWAP", "CNOT", "CZ", "Toffoli", "P0", "P1"};
            for (auto* h : herm)
                if (b->name == h) return b;
            if (auto it = pairs.find(b->name); it != pairs.end()) return constant(it->second);
            return matblock(adjoint_mat(*b->mat));
        }
        case K::Matrix: return matblock(adjoint_mat(*b->mat));
        case K::Rotation: return rot(b->generator, -b->theta);
        case K::Shift: return shift(-b->theta);
        case K::Phase: return phase(-b->theta);
        case K::Chain: {
            std::vector<BlockPtr> r;
            for (auto it = b->children.rbegin(); it != b->children.rend(); ++it) r.push_back(dagger(*it));
            return chain(b->nqubits, std::move(r));
        }
        case K::Add: {
            std::vector<BlockPtr> r;
            for (auto& c : b->children) r.push_back(dagger(c));
            return add(std::move(r));
        }
        case K::Kron: {
            auto o = same(K::Kron);
            for (auto& c : o->children) c = dagger(c);
            return o;
        }
        case K::Scale: {
            auto o = same(K::Scale);
            o->factor = std::conj(b->factor);
            o->children = {dagger(b->children[0])};
            return o;
        }
        case K::Daggered: return b->children[0];
        default: {  // Put / Control / Repeat / Subroutine / Cached: adjoint of the child in place
            auto o = same(b->kind);
            o->children = {dagger(b->children[0])};
            return o;
        }
    }
}

// ---- parameters ------------------------------------------------------------------------
namespace detail {
inline void param_nodes(const BlockPtr& b, std::vector<Block*>& out, std::unordered_set<const Block*>& seen) {
    if (b->parameterised()) {
        if (seen.insert(b.get()).second) out.push_back(b.get());  // a shared node contributes once
        return;
    }
    for (auto& c : b->children) param_nodes(c, out, seen);
}
}  // namespace detail
inline std::vector<Block*> parameter_nodes(const BlockPtr& b) {
    std::vector<Block*> out;
    std::unordered_set<const Block*> seen;
    detail::param_nodes(b, out, seen);
    return out;
}
inline std::vector<double> parameters(const BlockPtr& b) {
    std::vector<double> v;
    for (auto* p : parameter_nodes(b)) v.push_back(p->theta);
    return v;
}
inline std::size_t nparameters(const BlockPtr& b) { return parameter_nodes(b).size(); }
inline const BlockPtr& dispatch(const BlockPtr& b, std::span<const double> theta) {
    auto nodes = parameter_nodes(b);
    if (theta.size() != nodes.size()) throw ValidationError("dispatch: parameter count mismatch");
    for (std::size_t k = 0; k < nodes.size(); ++k) nodes[k]->theta = theta[k];
    return b;
}
// dispatch(b, op, vec): θ <- op(θ, v) (Listing 9's dispatch!(-, circuit, lr * grad))
inline const BlockPtr& dispatch(const BlockPtr& b, const std::function<double(double, double)>& op,
                                std::span<const double> v) {
    auto nodes = parameter_nodes(b);
    if (v.size() != nodes.size()) throw ValidationError("dispatch: parameter count mismatch");
    for (std::size_t k = 0; k < nodes.size(); ++k) nodes[k]->theta = op(nodes[k]->theta, v[k]);
    return b;
}
// dispatch(b, "random", rng): U(0, 2π) per parameter, depth-first
inline const BlockPtr& dispatch(const BlockPtr& b, const std::string& how, Rng& rng) {
    if (how != "random") throw ValidationError("dispatch: unknown mode " + how);
    for (auto* p : parameter_nodes(b)) p->theta = rng.uniform(0.0, 2 * std::numbers::pi);
    return b;
}
inline const BlockPtr& dispatch(const BlockPtr& b, const std::string& how) {
    Rng r(42);
    return dispatch(b, how, r);
}

// gatecount (SPEC.md; Listing 9): primitive occurrences, controlled ones keyed Control{name}
namespace detail {
inline std::string gate_name(const Block& b) {
    switch (b.kind) {
        case BlockKind::Constant: return b.name;
        case BlockKind::Rotation:
            if (b.generator->kind == BlockKind::Constant &&
                (b.generator->name == "X" || b.generator->name == "Y" || b.generator->name == "Z"))
                return std::string("R") + static_cast<char>(std::tolower(b.generator->name[0]));
            return "rot";
        case BlockKind::Shift: return "shift";
        case BlockKind::Phase: return "phase";
        default: return "matrix";
    }
}
inline void gatecount(const BlockPtr& b, std::map<std::string, std::size_t>& out, bool ctrl) {
    if (b->kind <= BlockKind::Matrix) {
        out[ctrl ? "Control{" + gate_name(*b) + "}" : gate_name(*b)] += 1;
        return;
    }
    if (b->kind == BlockKind::Control) return gatecount(b->children[0], out, true);
    if (b->kind == BlockKind::Repeat) {
        for (std::size_t k = 0; k < b->locs.size(); ++k) gatecount(b->children[0], out, ctrl);
        return;
    }
    for (auto& c : b->children) gatecount(c, out, ctrl);
}
}  // namespace detail
inline std::map<std::string, std::size_t> gatecount(const BlockPtr& b) {
    std::map<std::string, std::size_t> out;
    detail::gatecount(b, out, false);
    return out;
}

// ---- dense matrices of small blocks (host; generators of rot and tests) ------------------------------------
namespace detail {
using DMat = std::vector<cplx>;  // row-major d x d
inline DMat dmul(const DMat& a, const DMat& b, std::size_t d) {
    DMat o(d * d, 0.0);
    for (std::size_t i = 0; i < d; ++i)
        for (std::size_t k = 0; k < d; ++k)
            if (a[i * d + k] != cplx(0.0))
                for (std::size_t j = 0; j < d; ++j) o[i * d + j] += a[i * d + k] * b[k * d + j];
    return o;
}
// operator of m (on t qubits) placed on locs of an n-qubit space, with control projectors
inline DMat embed(std::size_t n, const std::vector<std::size_t>& locs, const DMat& m, const std::vector<std::size_t>& ctrls = {},
                  const std::vector<int>& cfg = {}) {
    const std::size_t d = std::size_t{1} << n, t = locs.size();
    DMat out(d * d, 0.0);
    for (std::size_t col = 0; col < d; ++col) {
        bool on = true;
        for (std::size_t k = 0; k < ctrls.size(); ++k)
            if (static_cast<int>((col >> (ctrls[k] - 1)) & 1) != cfg[k]) on = false;
        if (!on) {
            out[col * d + col] += 1.0;
            continue;
        }
        std::size_t sub = 0, base = col;
        for (std::size_t q = 0; q < t; ++q) {
            sub |= ((col >> (locs[q] - 1)) & 1) << q;
            base &= ~(std::size_t{1} << (locs[q] - 1));
        }
        for (std::size_t r = 0; r < (std::size_t{1} << t); ++r) {
            std::size_t row = base;
            for (std::size_t q = 0; q < t; ++q)
                if ((r >> q) & 1) row |= std::size_t{1} << (locs[q] - 1);
            out[row * d + col] += m[r * (std::size_t{1} << t) + sub];
        }
    }
    return out;
}
inline DMat eye(std::size_t d) {
    DMat o(d * d, 0.0);
    for (std::size_t i = 0; i < d; ++i) o[i * d + i] = 1.0;
    return o;
}
}  // namespace detail

// mat(b): dense operator (row-major); Chain multiplies in reverse order.  n <= 12.
inline detail::DMat mat(const BlockPtr& b) {
    using K = BlockKind;
    const std::size_t n = b->nqubits, d = std::size_t{1} << n;
    if (n > 12) throw UndecidableError("mat: block too large to densify");
    switch (b->kind) {
        case K::Constant:
        case K::Matrix: {
            Dense a = to_dense(*b->mat);
            detail::DMat o(d * d);
            for (std::size_t r = 0; r < d; ++r)
                for (std::size_t c = 0; c < d; ++c) o[r * d + c] = a.at(r, c);
            return o;
        }
        case K::Rotation: {
            auto g = mat(b->generator);
            const double c = std::cos(b->theta / 2), s = std::sin(b->theta / 2);
            for (auto& v : g) v *= cplx(0.0, -s);
            for (std::size_t i = 0; i < d; ++i) g[i * d + i] += c;
            return g;
        }
        case K::Shift: return {1.0, 0.0, 0.0, std::polar(1.0, b->theta)};
        case K::Phase: return {std::polar(1.0, b->theta), 0.0, 0.0, std::polar(1.0, b->theta)};
        case K::Chain: {
            auto o = detail::eye(d);
            for (auto& c : b->children) o = detail::dmul(mat(c), o, d);
            return o;
        }
        case K::Put:
        case K::Subroutine: return detail::embed(n, b->locs, mat(b->children[0]));
        case K::Control: return detail::embed(n, b->locs, mat(b->children[0]), b->ctrl_locs, b->ctrl_config);
        case K::Kron: {
            auto o = detail::eye(d);
            for (std::size_t k = 0; k < b->children.size(); ++k)
                o = detail::dmul(detail::embed(n, b->kron_locs[k], mat(b->children[k])), o, d);
            return o;
        }
        case K::Repeat: {
            auto o = detail::eye(d);
            auto m = mat(b->children[0]);
            for (auto l : b->locs) o = detail::dmul(detail::embed(n, {l}, m), o, d);
            return o;
        }
        case K::Add: {
            detail::DMat o(d * d, 0.0);
            for (auto& c : b->children) {
                auto m = mat(c);
                for (std::size_t i = 0; i < o.size(); ++i) o[i] += m[i];
            }
            return o;
        }
        case K::Scale: {
            auto o = mat(b->children[0]);
            for (auto& v : o) v *= b->factor;
            return o;
        }
        case K::Daggered: {
            auto m = mat(b->children[0]);
            detail::DMat o(d * d);
            for (std::size_t r = 0; r < d; ++r)
                for (std::size_t c = 0; c < d; ++c) o[r * d + c] = std::conj(m[c * d + r]);
            return o;
        }
        case K::Cached: return mat(b->children[0]);
    }
    throw UnsupportedError("mat: unsupported block");
}

// ---- lowering to a device program (the same walk as blocks.py _lower) ----------------------------------------
namespace detail {
struct Emitter {
    std::vector<qbg_op> ops;
    std::vector<cplx> vals;
    std::vector<int64_t> perms;
    std::vector<Block*> slots;  // parameter nodes, in parameter order
    std::unordered_map<const Block*, int> slot_index;
    void set_slots(std::vector<Block*> s) {
        slots = std::move(s);
        for (std::size_t k = 0; k < slots.size(); ++k) slot_index.emplace(slots[k], static_cast<int>(k));
    }
    int slot_of(const Block* b) const {
        auto it = slot_index.find(b);
        if (it == slot_index.end()) throw InternalLoweringError();
        return it->second;
    }
    struct InternalLoweringError : Error {
        InternalLoweringError() : Error("lowering: parameter node not found") {}
    };
    // payload in the C-ABI classes (identity / diagonal / permutation / dense column-major)
    void emit(const MatrixRepr* m, int gen, int param, const std::vector<std::size_t>& targets,
              const std::vector<std::size_t>& ctrls, const std::vector<int>& cfg, std::size_t dim) {
        if (targets.size() > QBG_MAX_TARGETS) throw UnsupportedError("apply: primitive wider than 5 qubits");
        if (ctrls.size() > QBG_MAX_CTRLS) throw UnsupportedError("apply: more than 16 controls");
        qbg_op op{};
        op.gen = gen;
        op.param = param;
        op.ntarget = static_cast<int32_t>(targets.size());
        op.nctrl = static_cast<int32_t>(ctrls.size());
        op.dim = static_cast<int32_t>(dim);
        for (std::size_t k = 0; k < targets.size(); ++k) op.targets[k] = static_cast<int32_t>(targets[k]);
        for (std::size_t k = 0; k < ctrls.size(); ++k) {
            op.ctrls[k] = static_cast<int32_t>(ctrls[k]);
            op.ctrl_cfg[k] = cfg[k];
        }
        op.data = static_cast<int64_t>(vals.size());
        op.perm = static_cast<int64_t>(perms.size());
        if (!m) {
            op.kind = QBG_MAT_DIAGONAL;
            op.data = 0;
            op.perm = 0;
        } else {
            switch (kind_of(*m)) {
                case MatKind::I: op.kind = QBG_MAT_IDENTITY; break;
                case MatKind::D: {
                    op.kind = QBG_MAT_DIAGONAL;
                    auto& dg = std::get<Diagonal>(*m).diag;
                    vals.insert(vals.end(), dg.begin(), dg.end());
                    break;
                }
                case MatKind::P: {
                    op.kind = QBG_MAT_PERMUTATION;
                    auto& p = std::get<Permutation>(*m);
                    vals.insert(vals.end(), p.vals.begin(), p.vals.end());
                    for (auto v : p.perm) perms.push_back(static_cast<int64_t>(v));
                    break;
                }
                default: {
                    op.kind = QBG_MAT_DENSE;
                    auto a = to_dense(*m).a;
                    vals.insert(vals.end(), a.begin(), a.end());
                }
            }
        }
        ops.push_back(op);
    }
};
// the generator's matrix in its most specific class (diagonal / permutation / dense)
inline MatrixRepr class_matrix(const BlockPtr& g) {
    if (g->kind == BlockKind::Constant || g->kind == BlockKind::Matrix) {
        const MatKind k = kind_of(*g->mat);
        if (k == MatKind::S || k == MatKind::Outer) return to_dense(*g->mat);
        return *g->mat;
    }
    const std::size_t d = std::size_t{1} << g->nqubits;
    auto m = mat(g);
    bool diag = true, perm = true;
    std::vector<std::size_t> pm(d);
    std::vector<cplx> pv(d), dv(d);
    std::vector<int> colhits(d, 0);
    for (std::size_t r = 0; r < d; ++r) {
        int hits = 0;
        for (std::size_t c = 0; c < d; ++c)
            if (m[r * d + c] != cplx(0.0)) {
                if (r != c) diag = false;
                ++hits;
                ++colhits[c];
                pm[r] = c;
                pv[r] = m[r * d + c];
            }
        if (hits != 1) perm = false;
        dv[r] = m[r * d + r];
    }
    for (int h : colhits)
        if (h != 1) perm = false;
    if (diag) return Diagonal(dv);
    if (perm) return Permutation(pm, pv);
    Dense out(d);
    for (std::size_t r = 0; r < d; ++r)
        for (std::size_t c = 0; c < d; ++c) out.at(r, c) = m[r * d + c];
    return out;
}
inline void lower(const BlockPtr& b, const std::vector<std::size_t>& qmap, const std::vector<std::size_t>& ctrls,
                  const std::vector<int>& cfg, Emitter& em, bool adj) {
    using K = BlockKind;
    auto sub = [&](const std::vector<std::size_t>& locs) {
        std::vector<std::size_t> q;
        for (auto l : locs) q.push_back(qmap[l - 1]);
        return q;
    };
    auto no_dagger = [&] {
        if (adj) throw UnsupportedError("Daggered parameterised block: use dagger(block)");
    };
    switch (b->kind) {
        case K::Constant:
        case K::Matrix: {
            MatrixRepr m = adj ? adjoint_mat(*b->mat) : *b->mat;
            em.emit(&m, QBG_GEN_NONE, -1, qmap, ctrls, cfg, mat_dim(m));
            return;
        }
        case K::Rotation: {
            no_dagger();
            MatrixRepr g = class_matrix(b->generator);
            em.emit(&g, QBG_GEN_ROTATION, em.slot_of(b.get()), qmap, ctrls, cfg, std::size_t{1} << b->nqubits);
            return;
        }
        case K::Shift:
            no_dagger();
            em.emit(nullptr, QBG_GEN_SHIFT, em.slot_of(b.get()), qmap, ctrls, cfg, 2);
            return;
        case K::Phase:
            no_dagger();
            em.emit(nullptr, QBG_GEN_PHASE, em.slot_of(b.get()), qmap, ctrls, cfg, std::size_t{1} << b->nqubits);
            return;
        case K::Chain:
            if (adj)
                for (auto it = b->children.rbegin(); it != b->children.rend(); ++it) lower(*it, qmap, ctrls, cfg, em, adj);
            else
                for (auto& c : b->children) lower(c, qmap, ctrls, cfg, em, adj);
            return;
        case K::Put:
        case K::Subroutine: lower(b->children[0], sub(b->locs), ctrls, cfg, em, adj); return;
        case K::Control: {
            auto c2 = ctrls;
            auto f2 = cfg;
            for (std::size_t k = 0; k < b->ctrl_locs.size(); ++k) {
                c2.push_back(qmap[b->ctrl_locs[k] - 1]);
                f2.push_back(b->ctrl_config[k]);
            }
            lower(b->children[0], sub(b->locs), c2, f2, em, adj);
            return;
        }
        case K::Kron: {
            const std::size_t nk = b->children.size();
            for (std::size_t i = 0; i < nk; ++i) {
                const std::size_t k = adj ? nk - 1 - i : i;
                lower(b->children[k], sub(b->kron_locs[k]), ctrls, cfg, em, adj);
            }
            return;
        }
        case K::Repeat: {
            const std::size_t nl = b->locs.size();
            for (std::size_t i = 0; i < nl; ++i) {
                const std::size_t l = b->locs[adj ? nl - 1 - i : i];
                lower(b->children[0], {qmap[l - 1]}, ctrls, cfg, em, adj);
            }
            return;
        }
        case K::Daggered: lower(b->children[0], qmap, ctrls, cfg, em, !adj); return;
        case K::Cached: lower(b->children[0], qmap, ctrls, cfg, em, adj); return;
        default: throw UnsupportedError("apply: Add / Scale are not circuit blocks (non-unitary)");
    }
}

struct Compiled {
    qbg_prog* h = nullptr;
    std::vector<Block*> nodes;
    std::vector<double> theta;
    bool realised = false;
    ~Compiled() {
        if (h) qbg_prog_destroy(h);
    }
    void sync() {
        std::vector<double> th(nodes.size());
        for (std::size_t k = 0; k < nodes.size(); ++k) th[k] = nodes[k]->theta;
        if (realised && th == theta) return;
        check(qbg_prog_set_params(h, th.data(), static_cast<int64_t>(th.size())));
        theta = std::move(th);
        realised = true;
    }
};
}  // namespace detail

// the compiled program of a circuit block (built once, cached on the block; θ re-synchronised)
inline detail::Compiled& compile_block(const BlockPtr& b) {
    if (!b->compiled) {
        detail::Emitter em;
        em.set_slots(parameter_nodes(b));
        std::vector<std::size_t> qmap;
        for (std::size_t q = 1; q <= b->nqubits; ++q) qmap.push_back(q);
        detail::lower(b, qmap, {}, {}, em, false);
        auto c = std::make_shared<detail::Compiled>();
        c->nodes = em.slots;
        const cplx zero(0.0);
        const int64_t zperm = 0;
        check(qbg_prog_create(static_cast<int32_t>(b->nqubits), em.ops.data(), static_cast<int64_t>(em.ops.size()),
                              reinterpret_cast<const double*>(em.vals.empty() ? &zero : em.vals.data()),
                              static_cast<int64_t>(em.vals.size()), em.perms.empty() ? &zperm : em.perms.data(),
                              static_cast<int64_t>(em.perms.size()), &c->h));
        b->compiled = c;
    }
    b->compiled->sync();
    return *b->compiled;
}

// ---- observables: Pauli sums (Add / Scale / Chain / Put / Kron / Repeat of X, Y, Z, I2) -----------------------
struct PauliTerm {
    cplx coef;
    std::uint64_t xmask, zmask;  // bit q-1: X = x, Z = z, Y = x & z
};
namespace detail {
// σ(x1,z1)·σ(x2,z2) = phase · σ(x1^x2, z1^z2) per qubit (σ: I, X, Y = (1,1), Z)
inline PauliTerm pmul(const PauliTerm& a, const PauliTerm& b) {
    cplx ph = 1.0;
    std::uint64_t q = a.xmask | a.zmask | b.xmask | b.zmask;
    while (q) {
        const std::uint64_t bit = q & (~q + 1);
        q ^= bit;
        const int s1 = ((a.xmask & bit) ? 1 : 0) | ((a.zmask & bit) ? 2 : 0);
        const int s2 = ((b.xmask & bit) ? 1 : 0) | ((b.zmask & bit) ? 2 : 0);
        // index: 0 I, 1 X, 3 Y, 2 Z; table of the phase of σ_s1 σ_s2
        static const cplx I{0.0, 1.0};
        cplx t = 1.0;
        if (s1 == 1 && s2 == 3) t = I;   // XY = iZ
        if (s1 == 1 && s2 == 2) t = -I;  // XZ = -iY
        if (s1 == 3 && s2 == 1) t = -I;  // YX = -iZ
        if (s1 == 3 && s2 == 2) t = I;   // YZ = iX
        if (s1 == 2 && s2 == 1) t = I;   // ZX = iY
        if (s1 == 2 && s2 == 3) t = -I;  // ZY = -iX
        ph *= t;
    }
    return PauliTerm{a.coef * b.coef * ph, a.xmask ^ b.xmask, a.zmask ^ b.zmask};
}
inline std::vector<PauliTerm> pauli_terms(const BlockPtr& b, const std::vector<std::size_t>& qmap) {
    using K = BlockKind;
    auto sub = [&](const std::vector<std::size_t>& locs) {
        std::vector<std::size_t> q;
        for (auto l : locs) q.push_back(qmap[l - 1]);
        return q;
    };
    auto product = [](std::vector<std::vector<PauliTerm>> parts) {
        std::vector<PauliTerm> acc{PauliTerm{1.0, 0, 0}};
        for (auto& p : parts) {
            std::vector<PauliTerm> nxt;
            for (auto& a : acc)
                for (auto& t : p) nxt.push_back(pmul(a, t));
            acc = std::move(nxt);
        }
        return acc;
    };
    switch (b->kind) {
        case K::Constant: {
            if (b->nqubits != 1 || (b->name != "X" && b->name != "Y" && b->name != "Z" && b->name != "I2"))
                throw UnsupportedError("observable: not a Pauli expression");
            const std::uint64_t bit = std::uint64_t{1} << (qmap[0] - 1);
            const bool x = b->name == "X" || b->name == "Y", z = b->name == "Z" || b->name == "Y";
            return {PauliTerm{1.0, x ? bit : 0, z ? bit : 0}};
        }
        case K::Add: {
            std::vector<PauliTerm> out;
            for (auto& c : b->children) {
                auto t = pauli_terms(c, qmap);
                out.insert(out.end(), t.begin(), t.end());
            }
            return out;
        }
        case K::Cached: return pauli_terms(b->children[0], qmap);
        case K::Scale: {
            auto t = pauli_terms(b->children[0], qmap);
            for (auto& x : t) x.coef *= b->factor;
            return t;
        }
        case K::Put: return pauli_terms(b->children[0], sub(b->locs));
        case K::Chain: {  // operator product: later blocks multiply from the left
            std::vector<std::vector<PauliTerm>> parts;
            for (auto it = b->children.rbegin(); it != b->children.rend(); ++it) parts.push_back(pauli_terms(*it, qmap));
            return product(std::move(parts));
        }
        case K::Kron: {
            std::vector<std::vector<PauliTerm>> parts;
            for (std::size_t k = 0; k < b->children.size(); ++k) parts.push_back(pauli_terms(b->children[k], sub(b->kron_locs[k])));
            return product(std::move(parts));
        }
        case K::Repeat: {
            std::vector<std::vector<PauliTerm>> parts;
            for (auto l : b->locs) parts.push_back(pauli_terms(b->children[0], {qmap[l - 1]}));
            return product(std::move(parts));
        }
        default: throw UnsupportedError("observable: not a Pauli expression");
    }
}
struct CompiledObs {
    qbg_obs* h = nullptr;
    ~CompiledObs() {
        if (h) qbg_obs_destroy(h);
    }
};
}  // namespace detail

inline std::vector<PauliTerm> pauli_terms(const BlockPtr& b) {
    std::vector<std::size_t> qmap;
    for (std::size_t q = 1; q <= b->nqubits; ++q) qmap.push_back(q);
    return detail::pauli_terms(b, qmap);
}
inline qbg_obs* compile_observable(const BlockPtr& b) {
    if (!b->observable) {
        auto terms = pauli_terms(b);
        std::vector<qbg_pauli_term> t(std::max<std::size_t>(1, terms.size()));
        for (std::size_t k = 0; k < terms.size(); ++k)
            t[k] = qbg_pauli_term{terms[k].coef.real(), terms[k].coef.imag(), terms[k].xmask, terms[k].zmask};
        auto o = std::make_shared<detail::CompiledObs>();
        check(qbg_obs_create(static_cast<int32_t>(b->nqubits), t.data(), static_cast<int64_t>(terms.size()), &o->h));
        b->observable = o;
    }
    return b->observable->h;
}

// ---- evaluation ------------------------------------------------------------------------------------------------
inline bool is_circuit(const BlockPtr& b) {
    if (b->kind == BlockKind::Add || b->kind == BlockKind::Scale) return false;
    for (auto& c : b->children)
        if (!is_circuit(c)) return false;
    return true;
}

// apply!(reg, b) in place.  Add / Scale (observables) act as linear maps on
// clones (<= 2 scratch states); a Subroutine around a non-circuit child runs as
// focus -> apply -> relax.
inline Register& apply(Register& reg, const BlockPtr& b) {
    if (b->nqubits != reg.nactive()) throw ShapeError("apply: block qubit count differs from active qubits");
    if (is_circuit(b)) {
        check(qbg_apply(reg.handle(), compile_block(b).h));
        return reg;
    }
    switch (b->kind) {
        case BlockKind::Scale:
            qblock::apply(reg, b->children[0]);
            reg.scale(b->factor);
            return reg;
        case BlockKind::Add: {
            const Register src = reg;
            bool first = true;
            for (auto& c : b->children) {
                Register tmp = src;
                qblock::apply(tmp, c);
                if (first) {
                    reg = tmp;
                    first = false;
                } else {
                    reg.add_scaled(tmp, 1.0);
                }
            }
            return reg;
        }
        case BlockKind::Subroutine: {
            const std::size_t na = reg.nactive();
            reg.focus(b->locs);
            qblock::apply(reg, b->children[0]);
            reg.relax(b->locs, na);
            return reg;
        }
        case BlockKind::Cached: return qblock::apply(reg, b->children[0]);
        default: throw UnsupportedError("apply: non-unitary block inside a circuit composite");
    }
}

// expect(O, reg): Re <ψ_b|O|ψ_b> per batch, for a Pauli-sum observable
inline std::vector<double> expect(const BlockPtr& obs, const Register& reg) {
    std::vector<double> out(reg.nbatch());
    check(qbg_expect(reg.handle(), compile_observable(obs), out.data()));
    return out;
}
// expect(O, reg => circuit): the circuit on a copy of reg
inline std::vector<double> expect(const BlockPtr& obs, const Register& reg, const BlockPtr& circuit) {
    Register psi = reg;
    qblock::apply(psi, circuit);
    return expect(obs, psi);
}

struct GradResult {
    std::optional<Register> state_grad;  // adjoint of the input state (∂L/∂ψ_in*)
    std::vector<double> param_grads;     // parameters() order, summed over the batch
    std::vector<double> energies;        // <O> per batch (the forward value, no extra pass)
};

// expect'(O, reg => circuit): forward on a work copy, φ̄ = Oψ, reverse pass
// (uncompute + gradient accumulation); reg is left unchanged.
inline GradResult expect_grad(const BlockPtr& obs, const Register& reg, const BlockPtr& circuit,
                              bool want_state_grad = true) {
    if (!is_circuit(circuit)) throw UnsupportedError("expect': the circuit must be unitary (no Add / Scale)");
    auto& prog = compile_block(circuit);
    GradResult r;
    r.energies.assign(reg.nbatch(), 0.0);
    r.param_grads.assign(prog.nodes.size(), 0.0);
    qbg_reg* sg = nullptr;
    if (want_state_grad) {
        r.state_grad.emplace(reg.nqubits(), reg.nbatch(), 42);
        sg = r.state_grad->handle();
    }
    check(qbg_expect_grad(reg.handle(), prog.h, compile_observable(obs), 0, r.energies.data(),
                          r.param_grads.empty() ? nullptr : r.param_grads.data(), sg));
    return r;
}

// parameter-shift gradient, exact mode: ½(<O>_{θ+π/2} − <O>_{θ−π/2}) per
// parameter, summed over the batch; every parameter must be a rotation with a reflexive generator
namespace detail {
// a rotation under a Control node has the generator P_ctrl ⊗ Σ, which is not reflexive
inline bool controlled_param(const BlockPtr& b, bool under) {
    if (b->parameterised()) return under;
    for (auto& c : b->children)
        if (controlled_param(c, under || b->kind == BlockKind::Control)) return true;
    return false;
}
}  // namespace detail
inline std::vector<double> faithful_grad(const BlockPtr& obs, const Register& reg, const BlockPtr& circuit) {
    auto nodes = parameter_nodes(circuit);
    for (auto* p : nodes)
        if (p->kind != BlockKind::Rotation) throw UnsupportedError("faithful_grad: shift/phase parameters have no shift rule");
    if (detail::controlled_param(circuit, false))
        throw UnsupportedError("faithful_grad: a controlled rotation's generator is not reflexive (no shift rule)");
    std::vector<double> g(nodes.size(), 0.0);
    for (std::size_t k = 0; k < nodes.size(); ++k) {
        const double th = nodes[k]->theta;
        nodes[k]->theta = th + std::numbers::pi / 2;
        auto ep = expect(obs, reg, circuit);
        nodes[k]->theta = th - std::numbers::pi / 2;
        auto em = expect(obs, reg, circuit);
        nodes[k]->theta = th;
        for (std::size_t b = 0; b < ep.size(); ++b) g[k] += 0.5 * (ep[b] - em[b]);
    }
    return g;
}

// ---- circuits --------------------------------------------------------------------------------
// initial Rx layer; then depth x [CNOT ring i -> i mod n + 1; Rz, Rx, Rz on each qubit]
inline BlockPtr variational_circuit(std::size_t n, std::size_t depth) {
    if (n < 2 || depth < 1) throw ValidationError("variational_circuit: need n >= 2 and depth >= 1");
    std::vector<BlockPtr> bl;
    for (std::size_t q = 1; q <= n; ++q) bl.push_back(put(n, {q}, Rx(0.0)));
    for (std::size_t d = 0; d < depth; ++d) {
        for (std::size_t i = 1; i <= n; ++i) bl.push_back(control(n, std::vector<long>{static_cast<long>(i)}, {i % n + 1}, X()));
        for (std::size_t q = 1; q <= n; ++q) bl.push_back(put(n, {q}, chain(1, {Rz(0.0), Rx(0.0), Rz(0.0)})));
    }
    return chain(n, std::move(bl));
}
// Σ_bonds (XX + YY + ZZ), open chain; periodic adds the (n, 1) bond (App G)
inline BlockPtr heisenberg(std::size_t n, bool periodic = false) {
    if (n < 2) throw ValidationError("heisenberg: need n >= 2");
    std::vector<BlockPtr> terms;
    auto bond = [&](std::size_t i, std::size_t j) {
        for (auto s : {X(), Y(), Z()}) terms.push_back(put(n, {i}, s) * put(n, {j}, s));
    };
    for (std::size_t i = 1; i < n; ++i) bond(i, i + 1);
    if (periodic) bond(n, 1);
    return add(std::move(terms));
}
// Listing 1: chain of hcphases; cphase(i, j) = control(i, j => shift(2π / 2^(i-j+1)))
inline BlockPtr qft(std::size_t n) {
    std::vector<BlockPtr> outer;
    for (std::size_t i = 1; i <= n; ++i) {
        std::vector<BlockPtr> inner{put(n, {i}, H())};
        for (std::size_t j = i + 1; j <= n; ++j)
            inner.push_back(control(n, std::vector<long>{static_cast<long>(j)}, {i},
                                    shift(2 * std::numbers::pi / static_cast<double>(std::size_t{1} << (j - i + 1)))));
        outer.push_back(chain(n, std::move(inner)));
    }
    return chain(n, std::move(outer));
}

}  // namespace qblock
}  // namespace qbg
