// ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// Exposes the same C ABI as qbg_oracle.cpp (orc_*), but every operation runs through the
// UNMODIFIED reference headers (/root/reference/proj/include/qblock, included in place by
// oracle/Makefile via -I; nothing is copied into this repo):
//   qblock::Register, zero/rand_state, instruct (register.hpp:392-408), inner/norm,
//   probabilities/measure/measure_collapse (414-493), focus/relax (156-177),
//   gatemat::rot/shift/global_phase (gates.hpp:72-92), gate_by_tag (156-175),
//   adjoint_mat / scale_mat / add (matrix.hpp:525, 594-647), qblock::Rng (rng.hpp).
// The reference has no code for expect / expect_grad (SPEC.md:452-487 only), so those are
// the SPEC algorithm written on top of the reference's own instruct + adjoint_mat + gate
// table (P0/P1 projectors restrict mat_back to the controlled subspace).
// Built into oracle/_ref/libqbref.so (git-ignored; it travels to the GPU box with gpurun).
#include <chrono>
#include <complex>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "qblock/register.hpp"
#include "../include/qbg.h"

using qblock::cplx;
using qblock::MatrixRepr;

namespace {

thread_local std::string g_err;
double g_kernel_s = 0.0;  // compute time of the last timed call, excluding Register marshalling

struct Timer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void stop() { g_kernel_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return QBG_OK;
    } catch (const qblock::ValidationError& e) {
        g_err = e.what();
        return QBG_ERR_VALIDATION;
    } catch (const qblock::ShapeError& e) {
        g_err = e.what();
        return QBG_ERR_SHAPE;
    } catch (const qblock::RangeError& e) {
        g_err = e.what();
        return QBG_ERR_RANGE;
    } catch (const qblock::DispatchError& e) {
        g_err = e.what();
        return QBG_ERR_DISPATCH;
    } catch (const qblock::ResourceError& e) {
        g_err = e.what();
        return QBG_ERR_RESOURCE;
    } catch (const qblock::RenormalizationError& e) {
        g_err = e.what();
        return QBG_ERR_RENORMALIZATION;
    } catch (const qblock::Error& e) {
        g_err = e.what();
        return QBG_ERR_INTERNAL;
    }
}

MatrixRepr payload(const qbg_op& op, const double* vals, const std::int64_t* perms) {
    const cplx* v = reinterpret_cast<const cplx*>(vals) + (vals ? op.data : 0);
    std::size_t d = static_cast<std::size_t>(op.dim);
    switch (op.kind) {
        case QBG_MAT_IDENTITY:
            return qblock::Identity(d);
        case QBG_MAT_DIAGONAL:
            return qblock::Diagonal(std::vector<cplx>(v, v + d));
        case QBG_MAT_PERMUTATION:
            return qblock::Permutation(std::vector<std::size_t>(perms + op.perm, perms + op.perm + d),
                                       std::vector<cplx>(v, v + d));
        default:
            return qblock::Dense(d, std::vector<cplx>(v, v + d * d));
    }
}

MatrixRepr realise(const qbg_op& op, const double* vals, const std::int64_t* perms, const double* theta) {
    if (op.gen == QBG_GEN_NONE) return payload(op, vals, perms);
    double th = theta[op.param];
    if (op.gen == QBG_GEN_ROTATION) return qblock::gatemat::rot(payload(op, vals, perms), th);
    if (op.gen == QBG_GEN_SHIFT) return qblock::gatemat::shift(th);
    return qblock::gatemat::global_phase(th, static_cast<std::size_t>(op.dim));
}

MatrixRepr realise_deriv(const qbg_op& op, const double* vals, const std::int64_t* perms, const double* theta) {
    double th = theta[op.param];
    const cplx I(0.0, 1.0);
    std::size_t d = static_cast<std::size_t>(op.dim);
    if (op.gen == QBG_GEN_ROTATION) {
        double c = std::cos(th / 2), s = std::sin(th / 2);
        return qblock::add(qblock::scale_mat(cplx(-s / 2), qblock::Identity(d)),
                           qblock::scale_mat(-I * (c / 2), payload(op, vals, perms)));
    }
    if (op.gen == QBG_GEN_SHIFT) return qblock::Diagonal({cplx(0.0), I * std::polar(1.0, th)});
    return qblock::Diagonal(std::vector<cplx>(d, I * std::polar(1.0, th)));
}

struct Loc {
    std::vector<std::size_t> locs, ctrls;
    std::vector<int> cfg;
    explicit Loc(const qbg_op& op) {
        for (int k = 0; k < op.ntarget; ++k) locs.push_back(static_cast<std::size_t>(op.targets[k]));
        for (int k = 0; k < op.nctrl; ++k) {
            ctrls.push_back(static_cast<std::size_t>(op.ctrls[k]));
            cfg.push_back(op.ctrl_cfg[k]);
        }
    }
};

void to_reg(qblock::Register& r, const double* st) {
    auto a = r.amplitudes();
    std::memcpy(a.data(), st, a.size() * sizeof(cplx));
}
void from_reg(const qblock::Register& r, double* st) {
    auto a = r.amplitudes();
    std::memcpy(st, a.data(), a.size() * sizeof(cplx));
}

void pin_active(qblock::Register& r, int nactive) {
    if (static_cast<std::size_t>(nactive) == r.nqubits()) return;
    std::vector<std::size_t> locs;
    for (int q = 1; q <= nactive; ++q) locs.push_back(static_cast<std::size_t>(q));
    r.focus(locs);  // identity permutation, sets nactive
}

void obs_apply(const qblock::Register& psi, qblock::Register& phi, const qbg_pauli_term* terms, std::int64_t nterms) {
    phi.scale(cplx(0.0));
    for (std::int64_t t = 0; t < nterms; ++t) {
        qblock::Register tmp = psi;
        for (std::size_t q = 0; q < psi.nqubits(); ++q) {
            bool x = (terms[t].xmask >> q) & 1, z = (terms[t].zmask >> q) & 1;
            if (!x && !z) continue;
            std::size_t loc[1] = {q + 1};
            qblock::instruct(tmp, x && z ? "Y" : (x ? "X" : "Z"), loc);
        }
        phi.add_scaled(tmp, cplx(terms[t].coef_re, terms[t].coef_im));
    }
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
double orc_last_kernel_seconds(void) { return g_kernel_s; }

void* orc_rng_new(std::uint64_t seed) { return new qblock::Rng(seed); }
void orc_rng_free(void* r) { delete static_cast<qblock::Rng*>(r); }
void* orc_rng_split_label(void* r, const char* label) {
    return new qblock::Rng(static_cast<qblock::Rng*>(r)->split(label));
}
double orc_rng_uniform(void* r) { return static_cast<qblock::Rng*>(r)->uniform(); }
double orc_rng_uniform_range(void* r, double a, double b) { return static_cast<qblock::Rng*>(r)->uniform(a, b); }
double orc_rng_gauss(void* r) { return static_cast<qblock::Rng*>(r)->gauss(); }
std::uint64_t orc_rng_bits(void* r) { return static_cast<qblock::Rng*>(r)->bits(); }

void orc_dispatch_random(double* theta, std::int64_t n, std::uint64_t seed) {
    qblock::Rng r(seed);
    for (std::int64_t k = 0; k < n; ++k) theta[k] = r.uniform(0.0, 2 * M_PI);
}

int orc_rand_state(double* st, int n, std::int64_t B, std::uint64_t seed) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        auto r = qblock::rand_state(static_cast<std::size_t>(n), static_cast<std::size_t>(B), seed);
        from_reg(r, st);
    });
}

int orc_instruct(double* st, int n, int nactive, std::int64_t B, int kind, int dim, const double* vals,
                 const std::int64_t* perm, const std::int32_t* locs, int nloc, const std::int32_t* ctrls,
                 const std::int32_t* cfg, int nctrl) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register r(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42);
        to_reg(r, st);
        pin_active(r, nactive);
        qbg_op op{};
        op.kind = kind;
        op.dim = dim;
        MatrixRepr m = payload(op, vals, perm);
        std::vector<std::size_t> l(locs, locs + nloc), c(ctrls, ctrls + nctrl);
        std::vector<int> f(cfg, cfg + nctrl);
        qblock::instruct(r, m, l, c, f);
        from_reg(r, st);
    });
}

int orc_apply_program(double* st, int n, std::int64_t B, const qbg_op* ops, std::int64_t nops,
                      const double* vals, const std::int64_t* perms, const double* theta, int adjoint) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register r(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42);
        to_reg(r, st);
        Timer tm;
        for (std::int64_t q = 0; q < nops; ++q) {
            std::int64_t k = adjoint ? nops - 1 - q : q;
            MatrixRepr m = realise(ops[k], vals, perms, theta);
            if (adjoint) m = qblock::adjoint_mat(m);
            Loc L(ops[k]);
            qblock::instruct(r, m, L.locs, L.ctrls, L.cfg);
        }
        tm.stop();
        from_reg(r, st);
    });
}

int orc_inner(const double* a, const double* b, int n, std::int64_t B, double* out) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register x(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42), y = x;
        to_reg(x, a);
        to_reg(y, b);
        auto ip = x.inner(y);
        for (std::int64_t k = 0; k < B; ++k) {
            out[2 * k] = ip[k].real();
            out[2 * k + 1] = ip[k].imag();
        }
    });
}

int orc_norm(const double* a, int n, std::int64_t B, double* out) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register x(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42);
        to_reg(x, a);
        for (std::int64_t k = 0; k < B; ++k) out[k] = x.norm(static_cast<std::size_t>(k));
    });
}

int orc_obs_apply(const double* st, int n, std::int64_t B, const qbg_pauli_term* terms, std::int64_t nterms,
                  double* phi_out, double* energies) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register psi(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42);
        to_reg(psi, st);
        qblock::Register phi = psi;
        Timer tm;
        obs_apply(psi, phi, terms, nterms);
        if (energies) {
            auto ip = psi.inner(phi);
            for (std::int64_t k = 0; k < B; ++k) energies[k] = ip[k].real();
        }
        tm.stop();
        if (phi_out) from_reg(phi, phi_out);
    });
}

int orc_expect(const double* st, int n, std::int64_t B, const qbg_pauli_term* terms, std::int64_t nterms,
               double* energies) {
    return orc_obs_apply(st, n, B, terms, nterms, nullptr, energies);
}

int orc_expect_grad(const double* st_in, int n, std::int64_t B, const qbg_op* ops, std::int64_t nops,
                    const double* vals, const std::int64_t* perms, const double* theta, std::int64_t nparams,
                    const qbg_pauli_term* terms, std::int64_t nterms, double* energies, double* grads,
                    double* psi_out, double* state_grad) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register psi(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42);
        to_reg(psi, st_in);
        for (std::int64_t k = 0; k < nops; ++k) {
            Loc L(ops[k]);
            qblock::instruct(psi, realise(ops[k], vals, perms, theta), L.locs, L.ctrls, L.cfg);
        }
        qblock::Register phi = psi;
        obs_apply(psi, phi, terms, nterms);
        auto e = psi.inner(phi);
        for (std::int64_t b = 0; b < B; ++b) energies[b] = e[b].real();
        for (std::int64_t p = 0; p < nparams; ++p) grads[p] = 0.0;
        qblock::Register chi = psi;
        for (std::int64_t k = nops - 1; k >= 0; --k) {
            Loc L(ops[k]);
            MatrixRepr ud = qblock::adjoint_mat(realise(ops[k], vals, perms, theta));
            qblock::instruct(psi, ud, L.locs, L.ctrls, L.cfg);
            if (ops[k].gen != QBG_GEN_NONE) {
                chi = psi;
                for (std::size_t c = 0; c < L.ctrls.size(); ++c) {
                    std::size_t loc[1] = {L.ctrls[c]};
                    qblock::instruct(chi, L.cfg[c] ? "P1" : "P0", loc);
                }
                qblock::instruct(chi, realise_deriv(ops[k], vals, perms, theta), L.locs);
                auto ip = phi.inner(chi);
                double g = 0.0;
                for (std::int64_t b = 0; b < B; ++b) g += 2.0 * ip[b].real();
                grads[ops[k].param] += g;
            }
            qblock::instruct(phi, ud, L.locs, L.ctrls, L.cfg);
        }
        if (psi_out) from_reg(psi, psi_out);
        if (state_grad) from_reg(phi, state_grad);
    });
}

int orc_backward(double* st, double* ph, int n, std::int64_t B, const qbg_op* ops, std::int64_t nops,
                 const double* vals, const std::int64_t* perms, const double* theta, double* grads) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register psi(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42), phi = psi, chi = psi;
        to_reg(psi, st);
        to_reg(phi, ph);
        Timer tm;
        for (std::int64_t k = nops - 1; k >= 0; --k) {
            Loc L(ops[k]);
            MatrixRepr ud = qblock::adjoint_mat(realise(ops[k], vals, perms, theta));
            qblock::instruct(psi, ud, L.locs, L.ctrls, L.cfg);
            if (ops[k].gen != QBG_GEN_NONE) {
                chi = psi;
                for (std::size_t c = 0; c < L.ctrls.size(); ++c) {
                    std::size_t loc[1] = {L.ctrls[c]};
                    qblock::instruct(chi, L.cfg[c] ? "P1" : "P0", loc);
                }
                qblock::instruct(chi, realise_deriv(ops[k], vals, perms, theta), L.locs);
                auto ip = phi.inner(chi);
                for (std::int64_t b = 0; b < B; ++b) grads[ops[k].param] += 2.0 * ip[b].real();
            }
            qblock::instruct(phi, ud, L.locs, L.ctrls, L.cfg);
        }
        tm.stop();
        from_reg(psi, st);
        from_reg(phi, ph);
    });
}

// utils.hpp:28-33 thread_count: the reference parallelises over columns only
void orc_set_threads(int n) { qblock::set_thread_count(static_cast<unsigned>(n)); }

int orc_probabilities(const double* st, int n, int nactive, std::int64_t b, double* p) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register r(static_cast<std::size_t>(n), static_cast<std::size_t>(b + 1), 42);
        // only batch b matters: place it at slot b
        auto sl = r.batch(static_cast<std::size_t>(b));
        std::memcpy(sl.data(), st + 2 * b * (std::int64_t{1} << n), sl.size() * sizeof(cplx));
        pin_active(r, nactive);
        auto pr = qblock::probabilities(r, static_cast<std::size_t>(b));
        std::memcpy(p, pr.data(), pr.size() * sizeof(double));
    });
}

int orc_measure(const double* st, int n, int nactive, std::int64_t B, std::int64_t nshots, void* rng,
                std::uint64_t* out) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register r(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42);
        to_reg(r, st);
        pin_active(r, nactive);
        auto res = qblock::measure(r, static_cast<std::size_t>(nshots), *static_cast<qblock::Rng*>(rng));
        for (std::size_t k = 0; k < res.samples.size(); ++k) out[k] = res.samples[k].value;
    });
}

int orc_measure_collapse(double* st, int n, int nactive, std::int64_t B, void* rng, std::uint64_t* out) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register r(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42);
        to_reg(r, st);
        pin_active(r, nactive);
        auto res = qblock::measure_collapse(r, *static_cast<qblock::Rng*>(rng));
        for (std::size_t k = 0; k < res.samples.size(); ++k) out[k] = res.samples[k].value;
        from_reg(r, st);
    });
}

// Register::save / load (register.hpp:181-205), for file interchange tests
int orc_save(const double* st, int n, int nactive, std::int64_t B, const char* path) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register r(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42);
        to_reg(r, st);
        pin_active(r, nactive);
        std::ofstream f(path, std::ios::binary);
        r.save(f);
    });
}

int orc_load(const char* path, double* st, std::int64_t cap, int* n, int* nactive, std::int64_t* B) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        std::ifstream f(path, std::ios::binary);
        auto r = qblock::Register::load(f);
        *n = static_cast<int>(r.nqubits());
        *nactive = static_cast<int>(r.nactive());
        *B = static_cast<std::int64_t>(r.nbatch());
        auto a = r.amplitudes();
        if (static_cast<std::int64_t>(a.size()) > cap) throw qblock::ShapeError("orc_load: buffer too small");
        std::memcpy(st, a.data(), a.size() * sizeof(cplx));
    });
}

int orc_focus(double* st, int n, std::int64_t B, const std::int32_t* locs, int nloc) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register r(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42);
        to_reg(r, st);
        std::vector<std::size_t> l(locs, locs + nloc);
        r.focus(l);
        from_reg(r, st);
    });
}

int orc_relax(double* st, int n, std::int64_t B, const std::int32_t* locs, int nloc) {
    return guarded([&] {
        qblock::set_qubit_cap(63);
        qblock::Register r(static_cast<std::size_t>(n), static_cast<std::size_t>(B), 42);
        to_reg(r, st);
        // relax needs the matching focus on the same Register object; a buffer that is
        // already in the focused layout is relaxed by focusing on the inverse of the focus
        // order given as a full location list (a full list is taken verbatim, 209-223).
        std::vector<std::size_t> src(locs, locs + nloc);
        std::vector<bool> used(static_cast<std::size_t>(n) + 1, false);
        for (auto l : src) used[l] = true;
        for (std::size_t q = 1; q <= static_cast<std::size_t>(n); ++q)
            if (!used[q]) src.push_back(q);
        std::vector<std::size_t> inv(src.size());
        for (std::size_t k = 0; k < src.size(); ++k) inv[src[k] - 1] = k + 1;
        r.focus(inv);
        from_reg(r, st);
    });
}

}  // extern "C"
