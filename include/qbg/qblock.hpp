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
#include <memory>
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

// ---- matrix formats passed to instruct (matrix.hpp:41-129) -----------------------------------
struct Identity { std::size_t dim; };
struct Diagonal { std::vector<cplx> diag; };
struct Permutation { std::vector<std::size_t> perm; std::vector<cplx> vals; };
struct Dense { std::size_t dim; std::vector<cplx> a; };  // column-major a[c*dim + r]
using MatrixRepr = std::variant<Identity, Diagonal, Permutation, Dense>;

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
    qbg_reg* handle() const { return h_; }

   private:
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
inline Register product_state(std::uint64_t value, std::size_t nbits, std::size_t nbatch = 1, std::uint64_t seed = 42) {
    Register r(nbits, nbatch, seed);
    check(qbg_set_product(r.handle(), &value, 1));
    return r;
}

// ---- instruct (register.hpp:392-408) -------------------------------------------------------------
inline void instruct(Register& reg, const MatrixRepr& gate, std::span<const std::size_t> locs,
                     std::span<const std::size_t> ctrl_locs = {}, std::span<const int> ctrl_config = {}) {
    if (ctrl_locs.size() != ctrl_config.size())
        throw ValidationError("instruct: control locations and configuration differ in length");
    std::vector<int32_t> l(locs.begin(), locs.end()), c(ctrl_locs.begin(), ctrl_locs.end()),
        f(ctrl_config.begin(), ctrl_config.end());
    qbg_matrix m{};
    std::vector<cplx> vals;
    std::vector<int64_t> perm;
    if (auto* id = std::get_if<Identity>(&gate)) {
        m.kind = QBG_MAT_IDENTITY;
        m.dim = static_cast<int32_t>(id->dim);
    } else if (auto* d = std::get_if<Diagonal>(&gate)) {
        m.kind = QBG_MAT_DIAGONAL;
        m.dim = static_cast<int32_t>(d->diag.size());
        vals = d->diag;
    } else if (auto* p = std::get_if<Permutation>(&gate)) {
        m.kind = QBG_MAT_PERMUTATION;
        m.dim = static_cast<int32_t>(p->perm.size());
        vals = p->vals;
        perm.assign(p->perm.begin(), p->perm.end());
    } else {
        const Dense& dn = std::get<Dense>(gate);
        m.kind = QBG_MAT_DENSE;
        m.dim = static_cast<int32_t>(dn.dim);
        vals = dn.a;
    }
    m.vals = reinterpret_cast<const double*>(vals.data());
    m.perm = perm.data();
    check(qbg_instruct(reg.handle(), &m, l.data(), static_cast<int32_t>(l.size()), c.data(), f.data(),
                       static_cast<int32_t>(c.size())));
}

inline void instruct(Register& reg, const std::string& tag, std::span<const std::size_t> locs,
                     std::span<const std::size_t> ctrl_locs = {}, std::span<const int> ctrl_config = {},
                     std::span<const double> params = {}) {
    if (ctrl_locs.size() != ctrl_config.size())
        throw ValidationError("instruct: control locations and configuration differ in length");
    std::vector<int32_t> l(locs.begin(), locs.end()), c(ctrl_locs.begin(), ctrl_locs.end()),
        f(ctrl_config.begin(), ctrl_config.end());
    check(qbg_instruct_tag(reg.handle(), tag.c_str(), l.data(), static_cast<int32_t>(l.size()), c.data(), f.data(),
                           static_cast<int32_t>(c.size()), params.data(), static_cast<int32_t>(params.size())));
}

// ---- measurement (register.hpp:414-493) -----------------------------------------------------------
struct BitStr {
    std::uint64_t value = 0;
    std::size_t nbits = 1;
    friend bool operator==(const BitStr&, const BitStr&) = default;
};
struct MeasureOutcome {
    std::vector<BitStr> samples;
};

inline std::vector<double> probabilities(const Register& reg, std::size_t b) {
    std::vector<double> p(reg.nrows());
    check(qbg_probabilities(reg.handle(), static_cast<int64_t>(b), p.data()));
    return p;
}
inline MeasureOutcome measure(const Register& reg, std::size_t nshots, Rng& rng) {
    std::vector<std::uint64_t> v(nshots * reg.nbatch());
    check(qbg_measure(reg.handle(), static_cast<int64_t>(nshots), rng.handle(), v.data()));
    MeasureOutcome o;
    for (auto x : v) o.samples.push_back(BitStr{x, reg.nactive()});
    return o;
}
inline MeasureOutcome measure(Register& reg, std::size_t nshots = 1) {
    std::vector<std::uint64_t> v(nshots * reg.nbatch());
    check(qbg_measure(reg.handle(), static_cast<int64_t>(nshots), nullptr, v.data()));
    MeasureOutcome o;
    for (auto x : v) o.samples.push_back(BitStr{x, reg.nactive()});
    return o;
}
inline MeasureOutcome measure_collapse(Register& reg, Rng& rng) {
    std::vector<std::uint64_t> v(reg.nbatch());
    check(qbg_measure_collapse(reg.handle(), rng.handle(), v.data()));
    MeasureOutcome o;
    for (auto x : v) o.samples.push_back(BitStr{x, reg.nactive()});
    return o;
}
inline MeasureOutcome measure_collapse(Register& reg) {
    std::vector<std::uint64_t> v(reg.nbatch());
    check(qbg_measure_collapse(reg.handle(), nullptr, v.data()));
    MeasureOutcome o;
    for (auto x : v) o.samples.push_back(BitStr{x, reg.nactive()});
    return o;
}

inline std::string to_text(const BitStr& b) {  // bits.hpp:104-112
    std::string s(b.nbits, '0');
    for (std::size_t i = 0; i < b.nbits; ++i)
        if ((b.value >> i) & 1) s[b.nbits - 1 - i] = '1';
    return s + " (2)";
}

}  // namespace qblock
}  // namespace qbg
