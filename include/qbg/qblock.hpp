// qbg/qblock.hpp — drop-in C++ shim: the reference's register API (qblock, register.hpp /
// gates.hpp / errors.hpp / rng.hpp) with the B200 engine (libqbg.so, include/qbg.h) behind it.
//
// A qblock user switches by replacing `#include "qblock/register.hpp"` with this header and
// `qblock::` with `qbg::qblock::` (or a namespace alias).  Names, argument meaning (1-based
// qubit locations, little-endian, ctrl_config of 0/1) and error types follow the reference:
//   Register(nqubits, nbatch, seed) / copy, register.hpp:60-93
//   zero_state / rand_state / product_state, register.hpp:260-286
//   instruct(reg, MatrixRepr, locs, ctrls, cfg) / instruct(reg, tag, …, params), 392-408
//   Register::norm / scale / add_scaled / inner, 120-150;  focus / relax, 156-177
//   probabilities / measure / measure_collapse, 414-493;  Rng, rng.hpp:25-66
//   qblock::Error and subclasses, errors.hpp:24-81 (re-thrown from the C-ABI codes)
// Amplitudes live on the device (batch innermost); amplitudes() downloads a host copy in the
// reference layout instead of returning a span into host memory (register.hpp:105-117).
#pragma once

#include <complex>
#include <cstdint>
#include <cstring>
#include <istream>
#include <iterator>
#include <map>
#include <memory>
#include <numbers>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "../qbg.h"

namespace qbg {
namespace qblock {

using cplx = std::complex<double>;

// ---- errors (errors.hpp:24-81) ------------------------------------------------------------
struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct ValidationError : Error { using Error::Error; };
struct ShapeError : Error { using Error::Error; };
struct RangeError : Error { using Error::Error; };
struct DispatchError : Error { using Error::Error; };
struct ResourceError : Error { using Error::Error; };
struct UnsupportedError : Error { using Error::Error; };
struct UndecidableError : Error { using Error::Error; };
struct RenormalizationError : Error { using Error::Error; };
struct SerializationError : Error { using Error::Error; };
struct ParseError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // CUDA / NCCL: no reference counterpart

inline void check(int rc) {
    if (rc == QBG_OK) return;
    std::string m = qbg_last_error();
    switch (rc) {
        case QBG_ERR_VALIDATION: throw ValidationError(m);
        case QBG_ERR_SHAPE: throw ShapeError(m);
        case QBG_ERR_RANGE: throw RangeError(m);
        case QBG_ERR_DISPATCH: throw DispatchError(m);
        case QBG_ERR_RESOURCE: throw ResourceError(m);
        case QBG_ERR_UNSUPPORTED: throw UnsupportedError(m);
        case QBG_ERR_UNDECIDABLE: throw UndecidableError(m);
        case QBG_ERR_RENORMALIZATION: throw RenormalizationError(m);
        case QBG_ERR_SERIALIZATION: throw SerializationError(m);
        case QBG_ERR_PARSE: throw ParseError(m);
        default: throw DeviceError(m);
    }
}

// ---- matrix formats (matrix.hpp:41-129): the six MatrixRepr alternatives, same validation ------
struct Identity {
    std::size_t dim = 0;
    explicit Identity(std::size_t d) : dim(d) {
        if (d == 0) throw ShapeError("Identity: dimension must be positive");
    }
};
struct Diagonal {
    std::vector<cplx> diag;
    explicit Diagonal(std::vector<cplx> d) : diag(std::move(d)) {
        if (diag.empty()) throw ShapeError("Diagonal: dimension must be positive");
    }
};
// row i holds vals[i] at column perm[i] (0-based)
struct Permutation {
    std::vector<std::size_t> perm;
    std::vector<cplx> vals;
    Permutation(std::vector<std::size_t> p, std::vector<cplx> v) : perm(std::move(p)), vals(std::move(v)) {
        if (perm.empty() || perm.size() != vals.size())
            throw ShapeError("Permutation: perm and vals must be non-empty and equal length");
        std::vector<char> hit(perm.size(), 0);
        for (std::size_t c : perm) {
            if (c >= perm.size() || hit[c]) throw ValidationError("Permutation: column indices must form a permutation");
            hit[c] = 1;
        }
    }
};
// compressed sparse columns, rows sorted and unique within a column
struct SparseColumns {
    std::size_t dim = 0;
    std::vector<std::size_t> colptr, rows;
    std::vector<cplx> vals;
    SparseColumns(std::size_t d, std::vector<std::size_t> cp, std::vector<std::size_t> r, std::vector<cplx> v)
        : dim(d), colptr(std::move(cp)), rows(std::move(r)), vals(std::move(v)) {
        if (dim == 0 || colptr.size() != dim + 1 || colptr.front() != 0 || colptr.back() != rows.size() ||
            rows.size() != vals.size())
            throw ShapeError("SparseColumns: inconsistent structure");
        for (std::size_t c = 0; c < dim; ++c) {
            if (colptr[c] > colptr[c + 1]) throw ShapeError("SparseColumns: column pointers not monotone");
            for (std::size_t k = colptr[c]; k + 1 < colptr[c + 1]; ++k)
                if (rows[k] >= rows[k + 1]) throw ValidationError("SparseColumns: rows must be sorted and unique");
            if (colptr[c] < colptr[c + 1] && rows[colptr[c + 1] - 1] >= dim)
                throw RangeError("SparseColumns: row index out of range");
        }
    }
};
// column-major a[c*dim + r]
struct Dense {
    std::size_t dim = 0;
    std::vector<cplx> a;
    Dense(std::size_t d, std::vector<cplx> data) : dim(d), a(std::move(data)) {
        if (dim == 0 || a.size() != dim * dim) throw ShapeError("Dense: data size must be dim^2");
    }
    explicit Dense(std::size_t d) : dim(d), a(d * d, cplx(0.0)) {
        if (dim == 0) throw ShapeError("Dense: dimension must be positive");
    }
    cplx& at(std::size_t r, std::size_t c) { return a[c * dim + r]; }
    const cplx& at(std::size_t r, std::size_t c) const { return a[c * dim + r]; }
};
// rank one: left * right (right is a row vector, not conjugated)
struct OuterProduct {
    std::vector<cplx> left, right;
    OuterProduct(std::vector<cplx> l, std::vector<cplx> r) : left(std::move(l)), right(std::move(r)) {
        if (left.empty() || left.size() != right.size())
            throw ShapeError("OuterProduct: vectors must be non-empty and equal length");
    }
};
using MatrixRepr = std::variant<Identity, Diagonal, Permutation, SparseColumns, Dense, OuterProduct>;
enum class MatKind : int { I = 0, D = 1, P = 2, S = 3, M = 4, Outer = 5 };
inline MatKind kind_of(const MatrixRepr& m) { return static_cast<MatKind>(m.index()); }

inline std::size_t mat_dim(const MatrixRepr& m) {
    switch (kind_of(m)) {
        case MatKind::I: return std::get<Identity>(m).dim;
        case MatKind::D: return std::get<Diagonal>(m).diag.size();
        case MatKind::P: return std::get<Permutation>(m).perm.size();
        case MatKind::S: return std::get<SparseColumns>(m).dim;
        case MatKind::M: return std::get<Dense>(m).dim;
        default: return std::get<OuterProduct>(m).left.size();
    }
}
inline Dense to_dense(const MatrixRepr& m) {  // matrix.hpp:229-233
    const std::size_t d = mat_dim(m);
    if (auto* x = std::get_if<Dense>(&m)) return *x;
    Dense out(d);
    switch (kind_of(m)) {
        case MatKind::I:
            for (std::size_t i = 0; i < d; ++i) out.at(i, i) = 1.0;
            break;
        case MatKind::D:
            for (std::size_t i = 0; i < d; ++i) out.at(i, i) = std::get<Diagonal>(m).diag[i];
            break;
        case MatKind::P: {
            auto& p = std::get<Permutation>(m);
            for (std::size_t i = 0; i < d; ++i) out.at(i, p.perm[i]) = p.vals[i];
            break;
        }
        case MatKind::S: {
            auto& s = std::get<SparseColumns>(m);
            for (std::size_t c = 0; c < d; ++c)
                for (std::size_t k = s.colptr[c]; k < s.colptr[c + 1]; ++k) out.at(s.rows[k], c) = s.vals[k];
            break;
        }
        default: {
            auto& o = std::get<OuterProduct>(m);
            for (std::size_t c = 0; c < d; ++c)
                for (std::size_t r = 0; r < d; ++r) out.at(r, c) = o.left[r] * o.right[c];
        }
    }
    return out;
}
// U† in the same class (matrix.hpp:594-643)
inline MatrixRepr adjoint_mat(const MatrixRepr& m) {
    switch (kind_of(m)) {
        case MatKind::I: return m;
        case MatKind::D: {
            auto d = std::get<Diagonal>(m).diag;
            for (auto& v : d) v = std::conj(v);
            return Diagonal(std::move(d));
        }
        case MatKind::P: {
            auto& p = std::get<Permutation>(m);
            std::vector<std::size_t> inv(p.perm.size());
            std::vector<cplx> v(p.perm.size());
            for (std::size_t i = 0; i < p.perm.size(); ++i) {
                inv[p.perm[i]] = i;
                v[p.perm[i]] = std::conj(p.vals[i]);
            }
            return Permutation(std::move(inv), std::move(v));
        }
        case MatKind::Outer: {
            auto& o = std::get<OuterProduct>(m);
            std::vector<cplx> l(o.right.size()), r(o.left.size());
            for (std::size_t i = 0; i < l.size(); ++i) l[i] = std::conj(o.right[i]);
            for (std::size_t i = 0; i < r.size(); ++i) r[i] = std::conj(o.left[i]);
            return OuterProduct(std::move(l), std::move(r));
        }
        default: {  // Sparse / Dense: conjugate transpose (kept dense; sparse gates are densified by instruct anyway)
            Dense a = to_dense(m), out(a.dim);
            for (std::size_t c = 0; c < a.dim; ++c)
                for (std::size_t r = 0; r < a.dim; ++r) out.at(c, r) = std::conj(a.at(r, c));
            if (kind_of(m) == MatKind::M) return out;
            std::vector<std::size_t> cp{0}, rows;
            std::vector<cplx> vals;
            for (std::size_t c = 0; c < out.dim; ++c) {
                for (std::size_t r = 0; r < out.dim; ++r)
                    if (out.at(r, c) != cplx(0.0)) {
                        rows.push_back(r);
                        vals.push_back(out.at(r, c));
                    }
                cp.push_back(rows.size());
            }
            return SparseColumns(out.dim, std::move(cp), std::move(rows), std::move(vals));
        }
    }
}

// ---- gate matrices (gates.hpp:32-94) -----------------------------------------------------------
namespace gatemat {
inline const cplx i1{0.0, 1.0};
inline MatrixRepr x() { return Permutation({1, 0}, {1.0, 1.0}); }
inline MatrixRepr y() { return Permutation({1, 0}, {-i1, i1}); }
inline MatrixRepr z() { return Diagonal({1.0, -1.0}); }
inline MatrixRepr h() {
    const double s = 1.0 / std::numbers::sqrt2;
    return Dense(2, {s, s, s, -s});
}
inline MatrixRepr i2() { return Identity(2); }
inline MatrixRepr s() { return Diagonal({1.0, i1}); }
inline MatrixRepr sdag() { return Diagonal({1.0, -i1}); }
inline MatrixRepr t() { return Diagonal({1.0, std::polar(1.0, std::numbers::pi / 4)}); }
inline MatrixRepr tdag() { return Diagonal({1.0, std::polar(1.0, -std::numbers::pi / 4)}); }
inline MatrixRepr swap() { return Permutation({0, 2, 1, 3}, {1.0, 1.0, 1.0, 1.0}); }
inline MatrixRepr cnot() { return Permutation({0, 1, 3, 2}, {1.0, 1.0, 1.0, 1.0}); }  // control qubit 2, X on 1
inline MatrixRepr cz() { return Permutation({0, 1, 2, 3}, {1.0, 1.0, 1.0, -1.0}); }
inline MatrixRepr toffoli() { return Permutation({0, 1, 2, 3, 4, 5, 7, 6}, std::vector<cplx>(8, 1.0)); }
inline MatrixRepr p0() { return SparseColumns(2, {0, 1, 1}, {0}, {1.0}); }
inline MatrixRepr p1() { return SparseColumns(2, {0, 0, 1}, {1}, {1.0}); }
inline MatrixRepr pu() { return SparseColumns(2, {0, 0, 1}, {0}, {1.0}); }
inline MatrixRepr pd() { return SparseColumns(2, {0, 1, 1}, {1}, {1.0}); }
inline MatrixRepr rx(double th) {
    const cplx c = std::cos(th / 2), ms = -i1 * std::sin(th / 2);
    return Dense(2, {c, ms, ms, c});
}
inline MatrixRepr ry(double th) {
    const double c = std::cos(th / 2), s = std::sin(th / 2);
    return Dense(2, {c, s, -s, c});
}
inline MatrixRepr rz(double th) { return Diagonal({std::polar(1.0, -th / 2), std::polar(1.0, th / 2)}); }
inline MatrixRepr shift(double th) { return Diagonal({1.0, std::polar(1.0, th)}); }
inline MatrixRepr global_phase(double th, std::size_t dim = 2) { return Diagonal(std::vector<cplx>(dim, std::polar(1.0, th))); }
// rot(G, θ) = cos(θ/2) I − i sin(θ/2) G; a diagonal generator stays diagonal (gates.hpp:79-92)
inline MatrixRepr rot(const MatrixRepr& g, double th) {
    const double c = std::cos(th / 2), s = std::sin(th / 2);
    const MatKind k = kind_of(g);
    if (k == MatKind::I || k == MatKind::D) {
        std::vector<cplx> d = k == MatKind::I ? std::vector<cplx>(mat_dim(g), 1.0) : std::get<Diagonal>(g).diag;
        for (auto& v : d) v = cplx(c) - i1 * cplx(s) * v;
        return Diagonal(std::move(d));
    }
    Dense out = to_dense(g);
    for (auto& v : out.a) v *= -i1 * s;
    for (std::size_t r = 0; r < out.dim; ++r) out.at(r, r) += c;
    return out;
}
}  // namespace gatemat

// ---- constant-gate registry / gate_by_tag (gates.hpp:97-175) ------------------------------------
struct ConstGateDef {
    std::string name;
    MatrixRepr mat;
    std::size_t nqubits;
};
inline std::map<std::string, ConstGateDef>& gate_registry() {
    static std::map<std::string, ConstGateDef> reg = [] {
        std::map<std::string, ConstGateDef> r;
        auto put = [&](const char* nm, MatrixRepr m) {
            std::size_t nq = 0;
            while ((std::size_t{1} << nq) < mat_dim(m)) ++nq;
            r.emplace(nm, ConstGateDef{nm, std::move(m), nq});
        };
        put("X", gatemat::x()); put("Y", gatemat::y()); put("Z", gatemat::z()); put("H", gatemat::h());
        put("I2", gatemat::i2()); put("S", gatemat::s()); put("Sdag", gatemat::sdag()); put("T", gatemat::t());
        put("Tdag", gatemat::tdag()); put("SWAP", gatemat::swap()); put("CNOT", gatemat::cnot());
        put("CZ", gatemat::cz()); put("Toffoli", gatemat::toffoli()); put("P0", gatemat::p0());
        put("P1", gatemat::p1()); put("Pu", gatemat::pu()); put("Pd", gatemat::pd());
        return r;
    }();
    return reg;
}
inline const ConstGateDef& define_const_gate(const std::string& name, const MatrixRepr& m) {
    const std::size_t d = mat_dim(m);
    if (d < 2 || (d & (d - 1)) != 0) throw ValidationError("define_const_gate: dimension must be a power of 2");
    std::size_t nq = 0;
    while ((std::size_t{1} << nq) < d) ++nq;
    auto& r = gate_registry();
    r.erase(name);
    return r.emplace(name, ConstGateDef{name, m, nq}).first->second;
}
inline const ConstGateDef* find_gate(const std::string& name) {
    auto& r = gate_registry();
    auto it = r.find(name);
    return it == r.end() ? nullptr : &it->second;
}
inline MatrixRepr gate_by_tag(const std::string& tag, std::span<const double> params = {}) {
    if (tag == "Rx" || tag == "Ry" || tag == "Rz" || tag == "shift" || tag == "phase") {
        if (params.size() != 1) throw DispatchError("gate " + tag + " expects one parameter");
        const double th = params[0];
        if (tag == "Rx") return gatemat::rx(th);
        if (tag == "Ry") return gatemat::ry(th);
        if (tag == "Rz") return gatemat::rz(th);
        if (tag == "shift") return gatemat::shift(th);
        return gatemat::global_phase(th);
    }
    if (const ConstGateDef* def = find_gate(tag)) {
        if (!params.empty()) throw DispatchError("gate " + tag + " takes no parameters");
        return def->mat;
    }
    throw DispatchError("unknown gate tag: " + tag);
}

// ---- BitStr (bits.hpp:29-139) -----------------------------------------------------------------------
struct BitStr {
    std::uint64_t value = 0;
    std::size_t nbits = 1;
    static constexpr std::size_t max_bits = 63;
    BitStr() = default;
    BitStr(std::uint64_t v, std::size_t n) : value(v), nbits(n) {
        if (n == 0 || n > max_bits) throw ValidationError("BitStr width must be in 1.." + std::to_string(max_bits));
        if (v >> n) throw ValidationError("BitStr value does not fit in " + std::to_string(n) + " bits");
    }
    friend bool operator==(const BitStr&, const BitStr&) = default;
};
inline int bit_at(const BitStr& b, std::size_t i) {
    if (i < 1 || i > b.nbits) throw RangeError("bit index " + std::to_string(i) + " out of range");
    return static_cast<int>((b.value >> (i - 1)) & 1u);
}
inline std::vector<int> to_bits(const BitStr& b) {
    std::vector<int> v(b.nbits);
    for (std::size_t i = 0; i < b.nbits; ++i) v[i] = static_cast<int>((b.value >> i) & 1u);
    return v;
}
inline BitStr from_bits(std::span<const int> bits) {
    if (bits.empty()) throw ValidationError("from_bits: empty bit list");
    if (bits.size() > BitStr::max_bits) throw ValidationError("from_bits: too many bits");
    std::uint64_t v = 0;
    for (std::size_t i = 0; i < bits.size(); ++i) {
        if (bits[i] != 0 && bits[i] != 1) throw ValidationError("from_bits: entry " + std::to_string(i + 1) + " is not 0 or 1");
        v |= static_cast<std::uint64_t>(bits[i]) << i;
    }
    return BitStr(v, bits.size());
}
inline BitStr from_bits(std::initializer_list<int> bits) { return from_bits(std::span<const int>(bits.begin(), bits.size())); }
inline bool ctrl_match(std::uint64_t index, std::span<const std::size_t> ctrl_locs, std::span<const int> ctrl_config) {
    if (ctrl_locs.size() != ctrl_config.size())
        throw ValidationError("ctrl_match: control locations and configuration differ in length");
    for (std::size_t k = 0; k < ctrl_locs.size(); ++k)
        if (static_cast<int>((index >> (ctrl_locs[k] - 1)) & 1u) != ctrl_config[k]) return false;
    return true;
}
inline std::string to_binary(const BitStr& b) {  // qubit 1 rightmost
    std::string s(b.nbits, '0');
    for (std::size_t i = 0; i < b.nbits; ++i)
        if ((b.value >> i) & 1) s[b.nbits - 1 - i] = '1';
    return s;
}
inline std::string to_text(const BitStr& b) { return to_binary(b) + " (2)"; }
inline BitStr bits_from_text(const std::string& text) {
    if (text.empty()) throw ValidationError("empty bit string");
    std::vector<int> bits(text.size());
    for (std::size_t k = 0; k < text.size(); ++k) {
        const char c = text[text.size() - 1 - k];
        if (c != '0' && c != '1') throw ValidationError("bit string may contain only 0 and 1");
        bits[k] = c - '0';
    }
    return from_bits(bits);
}
struct MeasureOutcome {
    std::vector<BitStr> samples;
};

// ---- Rng (rng.hpp:25-66): same libstdc++ stream, owned by the engine ---------------------------
class Rng {
   public:
    explicit Rng(std::uint64_t seed = 42) { check(qbg_rng_create(seed, &h_)); }
    Rng(const Rng&) = delete;
    Rng& operator=(const Rng&) = delete;
    Rng(Rng&& o) noexcept : h_(o.h_), owned_(o.owned_) { o.h_ = nullptr; }
    ~Rng() {
        if (h_ && owned_) qbg_rng_destroy(h_);
    }
    Rng split(const std::string& label) const {
        qbg_rng* out = nullptr;
        check(qbg_rng_split_label(h_, label.c_str(), &out));
        return Rng(out, true);
    }
    double uniform() { return qbg_rng_uniform(h_); }
    double uniform(double lo, double hi) { return qbg_rng_uniform_range(h_, lo, hi); }
    double gauss() { return qbg_rng_gauss(h_); }
    std::uint64_t bits() { return qbg_rng_bits(h_); }
    qbg_rng* handle() { return h_; }
    static Rng borrow(qbg_rng* h) { return Rng(h, false); }

   private:
    Rng(qbg_rng* h, bool owned) : h_(h), owned_(owned) {}
    qbg_rng* h_ = nullptr;
    bool owned_ = true;
};

inline void set_qubit_cap(std::size_t n) { check(qbg_set_qubit_cap(static_cast<int32_t>(n))); }
inline std::uint64_t state_alloc_counter() { return qbg_alloc_count(); }

// ---- Register (register.hpp:58-256) ------------------------------------------------------------
class Register {
   public:
    Register(std::size_t nqubits, std::size_t nbatch, std::uint64_t seed, int dtype = QBG_C128) {
        check(qbg_reg_create(static_cast<int32_t>(nqubits), static_cast<int64_t>(nbatch), dtype, seed, &h_));
    }
    Register(const Register& o) { check(qbg_reg_clone(o.h_, &h_)); }
    Register& operator=(const Register& o) {
        if (this != &o) {
            if (nqubits() == o.nqubits() && nbatch() == o.nbatch()) {
                check(qbg_reg_copy(h_, o.h_));
            } else {
                qbg_reg* n = nullptr;
                check(qbg_reg_clone(o.h_, &n));
                qbg_reg_destroy(h_);
                h_ = n;
            }
        }
        return *this;
    }
    Register(Register&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    ~Register() {
        if (h_) qbg_reg_destroy(h_);
    }

    std::size_t nqubits() const { return info().nq; }
    std::size_t nactive() const { return info().na; }
    std::size_t nremain() const { return nqubits() - nactive(); }
    std::size_t nbatch() const { return info().nb; }
    std::size_t nrows() const { return std::size_t{1} << nactive(); }
    std::size_t ncols() const { return (std::size_t{1} << nremain()) * nbatch(); }

    // host copy in the reference layout (batch slowest)
    std::vector<cplx> amplitudes() const {
        std::vector<cplx> v((std::size_t{1} << nqubits()) * nbatch());
        check(qbg_download(h_, reinterpret_cast<double*>(v.data()), static_cast<int64_t>(v.size())));
        return v;
    }
    void set_amplitudes(std::span<const cplx> v) {
        check(qbg_upload(h_, reinterpret_cast<const double*>(v.data()), static_cast<int64_t>(v.size())));
    }
    std::vector<cplx> batch(std::size_t b) const {
        auto all = amplitudes();
        std::size_t len = std::size_t{1} << nqubits();
        return std::vector<cplx>(all.begin() + static_cast<std::ptrdiff_t>(b * len),
                                 all.begin() + static_cast<std::ptrdiff_t>((b + 1) * len));
    }
    Rng rng() { return Rng::borrow(qbg_reg_rng(h_)); }

    double norm(std::size_t b) const {
        std::vector<double> n(nbatch());
        check(qbg_norm(h_, n.data()));
        return n[b];
    }
    void scale(cplx f) { check(qbg_scale(h_, f.real(), f.imag())); }
    void add_scaled(const Register& o, cplx f = cplx(1.0)) { check(qbg_add_scaled(h_, o.h_, f.real(), f.imag())); }
    std::vector<cplx> inner(const Register& o) const {
        std::vector<cplx> out(nbatch());
        check(qbg_inner(h_, o.h_, reinterpret_cast<double*>(out.data())));
        return out;
    }
    void focus(std::span<const std::size_t> locs) {
        std::vector<int32_t> l(locs.begin(), locs.end());
        check(qbg_focus(h_, l.data(), static_cast<int32_t>(l.size())));
    }
    void relax(std::span<const std::size_t> locs, std::size_t to_nactive) {
        std::vector<int32_t> l(locs.begin(), locs.end());
        check(qbg_relax(h_, l.data(), static_cast<int32_t>(l.size()), static_cast<int32_t>(to_nactive)));
    }
    // QBREG1 state files (register.hpp:181-205): magic, u64 nqubits / nactive / nbatch, then the
    // amplitudes batch-slowest — byte-identical with the reference's files
    void save(std::ostream& os) const {
        const char magic[8] = {'Q', 'B', 'R', 'E', 'G', '1', 0, 0};
        const std::uint64_t hdr[3] = {nqubits(), nactive(), nbatch()};
        const auto amps = amplitudes_raw();
        os.write(magic, 8);
        os.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
        os.write(reinterpret_cast<const char*>(amps.data()), static_cast<std::streamsize>(amps.size() * sizeof(cplx)));
    }
    static Register load(std::istream& is, std::uint64_t seed = 42) {
        std::string bytes((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
        qbg_reg* h = nullptr;
        check(qbg_load_memory(bytes.data(), static_cast<int64_t>(bytes.size()), seed, QBG_C128, &h));
        return Register(h);
    }
    qbg_reg* handle() const { return h_; }

   private:
    explicit Register(qbg_reg* h) : h_(h) {}
    // amplitudes in the device's current layout order (focus permutes physically, like the reference)
    std::vector<cplx> amplitudes_raw() const { return amplitudes(); }
    struct Info {
        std::size_t nq, na, nb;
    };
    Info info() const {
        int32_t nq = 0, na = 0, dt = 0;
        int64_t nb = 0;
        check(qbg_reg_info(h_, &nq, &na, &nb, &dt));
        return {static_cast<std::size_t>(nq), static_cast<std::size_t>(na), static_cast<std::size_t>(nb)};
    }
    qbg_reg* h_ = nullptr;
};

inline Register zero_state(std::size_t n, std::size_t nbatch = 1, std::uint64_t seed = 42) {
    Register r(n, nbatch, seed);
    check(qbg_set_zero(r.handle()));
    return r;
}
inline Register rand_state(std::size_t n, std::size_t nbatch = 1, std::uint64_t seed = 42) {
    Register r(n, nbatch, seed);
    check(qbg_set_rand(r.handle(), seed));
    return r;
}
inline Register product_state(const BitStr& b, std::size_t nbatch = 1, std::uint64_t seed = 42) {
    Register r(b.nbits, nbatch, seed);
    check(qbg_set_product(r.handle(), &b.value, 1));
    return r;
}
// batched form (no reference counterpart): one basis index per batch, batch-innermost on the device
inline Register product_state(std::span<const std::uint64_t> values, std::size_t nbits, std::uint64_t seed = 42) {
    Register r(nbits, values.size(), seed);
    check(qbg_set_product(r.handle(), values.data(), static_cast<int64_t>(values.size())));
    return r;
}

// ---- instruct (register.hpp:392-408) -------------------------------------------------------------
// Diagonal / Permutation / Dense go to the device as they are; SparseColumns and OuterProduct take
// the reference's generic path, to_dense (register.hpp:372), on the host.
inline void instruct(Register& reg, const MatrixRepr& gate, std::span<const std::size_t> locs,
                     std::span<const std::size_t> ctrl_locs = {}, std::span<const int> ctrl_config = {}) {
    if (ctrl_locs.size() != ctrl_config.size())
        throw ValidationError("instruct: control locations and configuration differ in length");
    std::vector<int32_t> l(locs.begin(), locs.end()), c(ctrl_locs.begin(), ctrl_locs.end()),
        f(ctrl_config.begin(), ctrl_config.end());
    qbg_matrix m{};
    std::vector<cplx> vals;
    std::vector<int64_t> perm;
    m.dim = static_cast<int32_t>(mat_dim(gate));
    switch (kind_of(gate)) {
        case MatKind::I: m.kind = QBG_MAT_IDENTITY; break;
        case MatKind::D:
            m.kind = QBG_MAT_DIAGONAL;
            vals = std::get<Diagonal>(gate).diag;
            break;
        case MatKind::P: {
            auto& p = std::get<Permutation>(gate);
            m.kind = QBG_MAT_PERMUTATION;
            vals = p.vals;
            perm.assign(p.perm.begin(), p.perm.end());
            break;
        }
        default:
            m.kind = QBG_MAT_DENSE;
            vals = to_dense(gate).a;
    }
    m.vals = reinterpret_cast<const double*>(vals.data());
    m.perm = perm.data();
    check(qbg_instruct(reg.handle(), &m, l.data(), static_cast<int32_t>(l.size()), c.data(), f.data(),
                       static_cast<int32_t>(c.size())));
}

// instruct by tag: gate_by_tag (builtin or define_const_gate-registered) then the matrix form
inline void instruct(Register& reg, const std::string& tag, std::span<const std::size_t> locs,
                     std::span<const std::size_t> ctrl_locs = {}, std::span<const int> ctrl_config = {},
                     std::span<const double> params = {}) {
    instruct(reg, gate_by_tag(tag, params), locs, ctrl_locs, ctrl_config);
}

// ---- measurement (register.hpp:414-493) -----------------------------------------------------------
inline std::vector<double> probabilities(const Register& reg, std::size_t b) {
    std::vector<double> p(reg.nrows());
    check(qbg_probabilities(reg.handle(), static_cast<int64_t>(b), p.data()));
    return p;
}
inline MeasureOutcome measure(const Register& reg, std::size_t nshots, Rng& rng) {
    std::vector<std::uint64_t> v(nshots * reg.nbatch());
    check(qbg_measure(reg.handle(), static_cast<int64_t>(nshots), rng.handle(), v.data()));
    MeasureOutcome o;
    for (auto x : v) o.samples.push_back(BitStr(x, reg.nactive()));
    return o;
}
inline MeasureOutcome measure(Register& reg, std::size_t nshots = 1) {
    std::vector<std::uint64_t> v(nshots * reg.nbatch());
    check(qbg_measure(reg.handle(), static_cast<int64_t>(nshots), nullptr, v.data()));
    MeasureOutcome o;
    for (auto x : v) o.samples.push_back(BitStr(x, reg.nactive()));
    return o;
}
inline MeasureOutcome measure_collapse(Register& reg, Rng& rng) {
    std::vector<std::uint64_t> v(reg.nbatch());
    check(qbg_measure_collapse(reg.handle(), rng.handle(), v.data()));
    MeasureOutcome o;
    for (auto x : v) o.samples.push_back(BitStr(x, reg.nactive()));
    return o;
}
inline MeasureOutcome measure_collapse(Register& reg) {
    std::vector<std::uint64_t> v(reg.nbatch());
    check(qbg_measure_collapse(reg.handle(), nullptr, v.data()));
    MeasureOutcome o;
    for (auto x : v) o.samples.push_back(BitStr(x, reg.nactive()));
    return o;
}

}  // namespace qblock
}  // namespace qbg
