// qbg_oracle.cpp — CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load this library, and only as the checker.  The product path (libqbg.so) never
// links or calls it.
//
// A plain, single-threaded restatement of the reference algorithm for the state-vector hot
// path, written against the reference *behaviour* (not its code):
//   gate application   register.hpp:292-385 (make_plan validation order, subset walk,
//                      diagonal / permutation / dense paths incl. the x==0 skip at 379)
//   parameterised gates gates.hpp:61-92 (rot(G,θ) = cos(θ/2)I − i sin(θ/2)G, shift, phase)
//   adjoint            matrix.hpp:594-643
//   inner / norm       register.hpp:120-150
//   probabilities, measure, measure_collapse   register.hpp:414-493
//   rand_state         register.hpp:266-280;   Rng rng.hpp:25-66
//   focus / relax      register.hpp:156-177, 209-248
//   expect / expect_grad  SPEC.md:452-487 (mat_back through the outer product, eq.
//                      outer-product PAPER.md:549-556: θ̄ = 2 Re <φ̄_{k+1}| ∂U/∂θ |ψ_k>)
// Host layout = the reference's: batch slowest, each batch a contiguous 2^n slice.
// Build: oracle/Makefile (g++ -O2 -std=c++20 -ffp-contract=off).  Parity against the
// compiled reference (oracle/_ref/libqbref.so, same C ABI) is checked in tests/.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../include/qbg.h"

using cd = std::complex<double>;

namespace {

thread_local std::string g_err;
double g_kernel_s = 0.0;  // compute time of the last timed call

struct Timer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void stop() { g_kernel_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
};

int fail(int code, const char* msg) {
    g_err = msg;
    return code;
}

// ---- Rng (rng.hpp:25-66) --------------------------------------------------------------
std::uint64_t sm64(std::uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

struct ORng {
    std::uint64_t key;
    std::mt19937_64 mt;
    explicit ORng(std::uint64_t seed) : key(sm64(seed)), mt(sm64(seed)) {}
    double unif() { return std::uniform_real_distribution<double>(0.0, 1.0)(mt); }
    double unif(double a, double b) { return std::uniform_real_distribution<double>(a, b)(mt); }
    double normal() { return std::normal_distribution<double>(0.0, 1.0)(mt); }
    ORng child(const char* label) const {
        std::uint64_t h = key;
        for (const char* p = label; *p; ++p) h = sm64(h ^ static_cast<unsigned char>(*p));
        return ORng(h);
    }
};

// ---- gate matrices --------------------------------------------------------------------
struct Mat {
    int kind = QBG_MAT_IDENTITY;
    int dim = 0;
    std::vector<cd> v;           // DIAGONAL/PERMUTATION: dim, DENSE: dim*dim col-major
    std::vector<std::int64_t> p; // PERMUTATION
};

Mat read_payload(const qbg_op& op, const double* vals, const std::int64_t* perms) {
    Mat m;
    m.kind = op.kind;
    m.dim = op.dim;
    const cd* src = reinterpret_cast<const cd*>(vals) + (vals ? op.data : 0);
    if (op.kind == QBG_MAT_DIAGONAL || op.kind == QBG_MAT_PERMUTATION) m.v.assign(src, src + op.dim);
    if (op.kind == QBG_MAT_DENSE) m.v.assign(src, src + static_cast<std::size_t>(op.dim) * op.dim);
    if (op.kind == QBG_MAT_PERMUTATION) m.p.assign(perms + op.perm, perms + op.perm + op.dim);
    return m;
}

Mat densify(const Mat& m) {
    Mat d;
    d.kind = QBG_MAT_DENSE;
    d.dim = m.dim;
    d.v.assign(static_cast<std::size_t>(m.dim) * m.dim, cd(0.0));
    for (int r = 0; r < m.dim; ++r) {
        if (m.kind == QBG_MAT_IDENTITY) d.v[r * m.dim + r] += cd(1.0);
        if (m.kind == QBG_MAT_DIAGONAL) d.v[r * m.dim + r] += m.v[r];
        if (m.kind == QBG_MAT_PERMUTATION) d.v[m.p[r] * m.dim + r] += m.v[r];
    }
    if (m.kind == QBG_MAT_DENSE) d.v = m.v;
    return d;
}

// rot(G, θ), gates.hpp:79-92 — same arithmetic sequence so the realised matrix is bitwise
// the reference's.
Mat rotation(const Mat& g, double theta) {
    const cd I(0.0, 1.0);
    double c = std::cos(theta / 2), s = std::sin(theta / 2);
    if (g.kind == QBG_MAT_IDENTITY || g.kind == QBG_MAT_DIAGONAL) {
        Mat r;
        r.kind = QBG_MAT_DIAGONAL;
        r.dim = g.dim;
        for (int k = 0; k < g.dim; ++k) {
            cd gk = g.kind == QBG_MAT_IDENTITY ? cd(1.0) : g.v[k];
            r.v.push_back(cd(c) - I * cd(s) * gk);
        }
        return r;
    }
    Mat r = densify(g);
    cd f = -I * s;
    for (auto& e : r.v) e *= f;
    for (int k = 0; k < r.dim; ++k) r.v[k * r.dim + k] += c;
    return r;
}

// d rot(G,θ)/dθ = −(s/2) I − i (c/2) G
Mat rotation_deriv(const Mat& g, double theta) {
    const cd I(0.0, 1.0);
    double c = std::cos(theta / 2), s = std::sin(theta / 2);
    Mat r = densify(g);
    for (auto& e : r.v) e *= -I * (c / 2);
    for (int k = 0; k < r.dim; ++k) r.v[k * r.dim + k] += -s / 2;
    return r;
}

Mat realise(const qbg_op& op, const double* vals, const std::int64_t* perms, const double* theta) {
    if (op.gen == QBG_GEN_NONE) return read_payload(op, vals, perms);
    double th = theta[op.param];
    if (op.gen == QBG_GEN_ROTATION) return rotation(read_payload(op, vals, perms), th);
    Mat m;
    m.kind = QBG_MAT_DIAGONAL;
    m.dim = op.dim;
    if (op.gen == QBG_GEN_SHIFT) {
        m.v = {cd(1.0), std::polar(1.0, th)};
    } else {
        m.v.assign(op.dim, std::polar(1.0, th));
    }
    return m;
}

Mat realise_deriv(const qbg_op& op, const double* vals, const std::int64_t* perms, const double* theta) {
    double th = theta[op.param];
    const cd I(0.0, 1.0);
    if (op.gen == QBG_GEN_ROTATION) return rotation_deriv(read_payload(op, vals, perms), th);
    Mat m;
    m.kind = QBG_MAT_DIAGONAL;
    m.dim = op.dim;
    if (op.gen == QBG_GEN_SHIFT) {
        m.v = {cd(0.0), I * std::polar(1.0, th)};
    } else {
        m.v.assign(op.dim, I * std::polar(1.0, th));
    }
    return m;
}

// adjoint_mat, matrix.hpp:594-643
Mat dagger(const Mat& m) {
    Mat a = m;
    if (m.kind == QBG_MAT_DIAGONAL) {
        for (auto& e : a.v) e = std::conj(e);
    } else if (m.kind == QBG_MAT_PERMUTATION) {
        for (int i = 0; i < m.dim; ++i) {
            a.p[m.p[i]] = i;
            a.v[m.p[i]] = std::conj(m.v[i]);
        }
    } else if (m.kind == QBG_MAT_DENSE) {
        for (int c = 0; c < m.dim; ++c)
            for (int r = 0; r < m.dim; ++r) a.v[r * m.dim + c] = std::conj(m.v[c * m.dim + r]);
    }
    return a;
}

// ---- instruct --------------------------------------------------------------------------
struct Placement {
    int t = 0;
    std::uint64_t tmask = 0, cmask = 0, cval = 0;
    std::vector<std::uint64_t> sub;  // basis offset of every sub-index (register.hpp:331-337)
};

// Validation in the order of make_plan, register.hpp:301-323.
int place(int nactive, const std::int32_t* locs, int nloc, const std::int32_t* ctrls, const std::int32_t* cfg,
          int nctrl, Placement& pl) {
    if (nloc < 1) return fail(QBG_ERR_VALIDATION, "instruct: need at least one target qubit");
    if (nctrl < 0) return fail(QBG_ERR_VALIDATION, "instruct: control locations and configuration differ in length");
    for (int k = 0; k < nloc; ++k) {
        if (locs[k] < 1 || locs[k] > nactive) return fail(QBG_ERR_RANGE, "instruct: target qubit out of range");
        std::uint64_t b = std::uint64_t{1} << (locs[k] - 1);
        if (pl.tmask & b) return fail(QBG_ERR_VALIDATION, "instruct: duplicate target qubit");
        pl.tmask |= b;
    }
    for (int k = 0; k < nctrl; ++k) {
        if (ctrls[k] < 1 || ctrls[k] > nactive) return fail(QBG_ERR_RANGE, "instruct: control qubit out of range");
        if (cfg[k] != 0 && cfg[k] != 1) return fail(QBG_ERR_VALIDATION, "instruct: control configuration must be 0 or 1");
        std::uint64_t b = std::uint64_t{1} << (ctrls[k] - 1);
        if ((pl.tmask | pl.cmask) & b) return fail(QBG_ERR_VALIDATION, "instruct: control qubit overlaps another location");
        pl.cmask |= b;
        if (cfg[k]) pl.cval |= b;
    }
    pl.t = nloc;
    pl.sub.resize(std::size_t{1} << nloc);
    for (std::size_t k = 0; k < pl.sub.size(); ++k) {
        std::uint64_t o = 0;
        for (int q = 0; q < nloc; ++q)
            if ((k >> q) & 1) o |= std::uint64_t{1} << (locs[q] - 1);
        pl.sub[k] = o;
    }
    return QBG_OK;
}

// Applies m on the placement to every column of length 2^nactive.  zero_outside: amplitudes
// whose controls do not match are zeroed instead of left alone (projector P_ctrl ⊗ m, used
// for mat_back restricted to the controlled subspace).
void apply_mat(cd* st, std::size_t rows, std::size_t ncols, const Mat& m, const Placement& pl,
               bool zero_outside = false) {
    std::size_t sub = pl.sub.size();
    Mat dn = (m.kind == QBG_MAT_DENSE || m.kind == QBG_MAT_IDENTITY || m.kind == QBG_MAT_DIAGONAL ||
              m.kind == QBG_MAT_PERMUTATION)
                 ? m
                 : densify(m);
    std::vector<cd> x(sub), y(sub);
    for (std::size_t c = 0; c < ncols; ++c) {
        cd* col = st + c * rows;
        for (std::size_t i = 0; i < rows; ++i) {
            if (i & pl.tmask) continue;  // visit each base (all target bits clear) once
            if ((i & pl.cmask) != pl.cval) {
                if (zero_outside)
                    for (std::size_t k = 0; k < sub; ++k) col[i + pl.sub[k]] = cd(0.0);
                continue;
            }
            if (m.kind == QBG_MAT_IDENTITY) continue;
            if (m.kind == QBG_MAT_DIAGONAL) {
                for (std::size_t k = 0; k < sub; ++k) col[i + pl.sub[k]] *= m.v[k];
                continue;
            }
            for (std::size_t k = 0; k < sub; ++k) x[k] = col[i + pl.sub[k]];
            if (m.kind == QBG_MAT_PERMUTATION) {
                for (std::size_t k = 0; k < sub; ++k) col[i + pl.sub[k]] = m.v[k] * x[m.p[k]];
                continue;
            }
            for (auto& e : y) e = cd(0.0);
            for (std::size_t j = 0; j < sub; ++j) {
                if (x[j] == cd(0.0)) continue;  // register.hpp:379
                for (std::size_t r = 0; r < sub; ++r) y[r] += dn.v[j * sub + r] * x[j];
            }
            for (std::size_t k = 0; k < sub; ++k) col[i + pl.sub[k]] = y[k];
        }
    }
}

struct View {
    cd* st;
    int n, nactive;
    std::int64_t B;
    std::size_t rows() const { return std::size_t{1} << nactive; }
    std::size_t cols() const { return (std::size_t{1} << (n - nactive)) * static_cast<std::size_t>(B); }
    std::size_t len() const { return std::size_t{1} << n; }
};

int apply_op(View v, const qbg_op& op, const Mat& m, bool zero_outside = false) {
    Placement pl;
    int rc = place(v.nactive, op.targets, op.ntarget, op.ctrls, op.ctrl_cfg, op.nctrl, pl);
    if (rc) return rc;
    if (m.dim != (1 << pl.t)) return fail(QBG_ERR_SHAPE, "instruct: gate dimension does not match target count");
    apply_mat(v.st, v.rows(), v.cols(), m, pl, zero_outside);
    return QBG_OK;
}

// P|j> for a Pauli string: Y = i X Z, so (P psi)[i] = i^{nY} (-1)^{|(i^x)&z|} psi[i^x]
void pauli_axpy(const cd* psi, cd* out, std::size_t len, const qbg_pauli_term& t) {
    int ny = __builtin_popcountll(t.xmask & t.zmask) & 3;
    const cd iy[4] = {cd(1, 0), cd(0, 1), cd(-1, 0), cd(0, -1)};
    cd c = cd(t.coef_re, t.coef_im) * iy[ny];
    for (std::size_t i = 0; i < len; ++i) {
        std::size_t j = i ^ t.xmask;
        double sgn = (__builtin_popcountll(j & t.zmask) & 1) ? -1.0 : 1.0;
        out[i] += c * (sgn * psi[j]);
    }
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
double orc_last_kernel_seconds(void) { return g_kernel_s; }

// ---- Rng ---------------------------------------------------------------------------------
void* orc_rng_new(std::uint64_t seed) { return new ORng(seed); }
void orc_rng_free(void* r) { delete static_cast<ORng*>(r); }
void* orc_rng_split_label(void* r, const char* label) { return new ORng(static_cast<ORng*>(r)->child(label)); }
double orc_rng_uniform(void* r) { return static_cast<ORng*>(r)->unif(); }
double orc_rng_uniform_range(void* r, double a, double b) { return static_cast<ORng*>(r)->unif(a, b); }
double orc_rng_gauss(void* r) { return static_cast<ORng*>(r)->normal(); }
std::uint64_t orc_rng_bits(void* r) { return static_cast<ORng*>(r)->mt(); }

// dispatch(b, "random"): U(0, 2π) per parameter in depth-first order
void orc_dispatch_random(double* theta, std::int64_t n, std::uint64_t seed) {
    ORng r(seed);
    for (std::int64_t k = 0; k < n; ++k) theta[k] = r.unif(0.0, 2 * M_PI);
}

// ---- states --------------------------------------------------------------------------------
int orc_rand_state(double* st, int n, std::int64_t B, std::uint64_t seed) {
    ORng g = ORng(seed).child("rand_state");
    std::size_t len = std::size_t{1} << n;
    cd* s = reinterpret_cast<cd*>(st);
    for (std::int64_t b = 0; b < B; ++b) {
        cd* sl = s + b * len;
        double acc = 0.0;
        for (std::size_t i = 0; i < len; ++i) {
            // g++ evaluates the two constructor arguments right to left (pinned against the
            // compiled reference in tests/test_oracle.py)
            double im = g.normal();
            double re = g.normal();
            sl[i] = cd(re, im);
            acc += std::norm(sl[i]);
        }
        double inv = 1.0 / std::sqrt(acc);
        for (std::size_t i = 0; i < len; ++i) sl[i] *= inv;
    }
    return QBG_OK;
}

// ---- instruct ----------------------------------------------------------------------------------
int orc_instruct(double* st, int n, int nactive, std::int64_t B, int kind, int dim, const double* vals,
                 const std::int64_t* perm, const std::int32_t* locs, int nloc, const std::int32_t* ctrls,
                 const std::int32_t* cfg, int nctrl) {
    qbg_op op{};
    op.kind = kind;
    op.dim = dim;
    op.ntarget = nloc;
    op.nctrl = nctrl;
    if (nloc > QBG_MAX_TARGETS || nctrl > QBG_MAX_CTRLS) return fail(QBG_ERR_VALIDATION, "too many locations");
    for (int k = 0; k < nloc; ++k) op.targets[k] = locs[k];
    for (int k = 0; k < nctrl; ++k) {
        op.ctrls[k] = ctrls[k];
        op.ctrl_cfg[k] = cfg[k];
    }
    Mat m = read_payload(op, vals, perm);
    return apply_op(View{reinterpret_cast<cd*>(st), n, nactive, B}, op, m);
}

int orc_apply_program(double* st, int n, std::int64_t B, const qbg_op* ops, std::int64_t nops,
                      const double* vals, const std::int64_t* perms, const double* theta, int adjoint) {
    View v{reinterpret_cast<cd*>(st), n, n, B};
    Timer tm;
    for (std::int64_t q = 0; q < nops; ++q) {
        std::int64_t k = adjoint ? nops - 1 - q : q;
        Mat m = realise(ops[k], vals, perms, theta);
        if (adjoint) m = dagger(m);
        int rc = apply_op(v, ops[k], m);
        if (rc) return rc;
    }
    tm.stop();
    return QBG_OK;
}

// ---- algebra -----------------------------------------------------------------------------------
int orc_inner(const double* a, const double* b, int n, std::int64_t B, double* out) {
    std::size_t len = std::size_t{1} << n;
    const cd* x = reinterpret_cast<const cd*>(a);
    const cd* y = reinterpret_cast<const cd*>(b);
    for (std::int64_t k = 0; k < B; ++k) {
        cd s(0.0);
        for (std::size_t i = 0; i < len; ++i) s += std::conj(x[k * len + i]) * y[k * len + i];
        out[2 * k] = s.real();
        out[2 * k + 1] = s.imag();
    }
    return QBG_OK;
}

int orc_norm(const double* a, int n, std::int64_t B, double* out) {
    std::size_t len = std::size_t{1} << n;
    const cd* x = reinterpret_cast<const cd*>(a);
    for (std::int64_t k = 0; k < B; ++k) {
        double s = 0.0;
        for (std::size_t i = 0; i < len; ++i) s += std::norm(x[k * len + i]);
        out[k] = std::sqrt(s);
    }
    return QBG_OK;
}

// φ = O ψ (Add of Pauli products), E_b = Re <ψ_b|φ_b>
int orc_obs_apply(const double* st, int n, std::int64_t B, const qbg_pauli_term* terms, std::int64_t nterms,
                  double* phi_out, double* energies) {
    std::size_t len = std::size_t{1} << n;
    const cd* psi = reinterpret_cast<const cd*>(st);
    Timer tm;
    std::vector<cd> phi(len * B, cd(0.0));
    for (std::int64_t b = 0; b < B; ++b)
        for (std::int64_t t = 0; t < nterms; ++t) pauli_axpy(psi + b * len, phi.data() + b * len, len, terms[t]);
    if (energies) {
        std::vector<double> ip(2 * B);
        orc_inner(st, reinterpret_cast<const double*>(phi.data()), n, B, ip.data());
        for (std::int64_t b = 0; b < B; ++b) energies[b] = ip[2 * b];
    }
    tm.stop();
    if (phi_out) std::memcpy(phi_out, phi.data(), len * B * sizeof(cd));
    return QBG_OK;
}

int orc_expect(const double* st, int n, std::int64_t B, const qbg_pauli_term* terms, std::int64_t nterms,
               double* energies) {
    return orc_obs_apply(st, n, B, terms, nterms, nullptr, energies);
}

// expect'(O, ψ0 ⇒ circuit).  grads are summed over the batch; psi_out
// (optional) receives the uncomputed input state, state_grad (optional) the input adjoint.
int orc_expect_grad(const double* st_in, int n, std::int64_t B, const qbg_op* ops, std::int64_t nops,
                    const double* vals, const std::int64_t* perms, const double* theta, std::int64_t nparams,
                    const qbg_pauli_term* terms, std::int64_t nterms, double* energies, double* grads,
                    double* psi_out, double* state_grad) {
    std::size_t len = std::size_t{1} << n;
    std::size_t total = len * B;
    std::vector<cd> psi(reinterpret_cast<const cd*>(st_in), reinterpret_cast<const cd*>(st_in) + total);
    std::vector<cd> phi(total), chi(total);
    int rc = orc_apply_program(reinterpret_cast<double*>(psi.data()), n, B, ops, nops, vals, perms, theta, 0);
    if (rc) return rc;
    orc_obs_apply(reinterpret_cast<double*>(psi.data()), n, B, terms, nterms, reinterpret_cast<double*>(phi.data()),
                  energies);
    for (std::int64_t p = 0; p < nparams; ++p) grads[p] = 0.0;
    View vp{psi.data(), n, n, B}, vf{phi.data(), n, n, B}, vc{chi.data(), n, n, B};
    for (std::int64_t k = nops - 1; k >= 0; --k) {
        const qbg_op& op = ops[k];
        Mat u = realise(op, vals, perms, theta);
        Mat ud = dagger(u);
        if ((rc = apply_op(vp, op, ud))) return rc;  // ψ_k = U_k† ψ_{k+1}
        if (op.gen != QBG_GEN_NONE) {
            // Ū = φ̄_{k+1} <ψ_k| ; θ̄ = 2 Re <∂U/∂θ, Ū> restricted to the control subspace
            chi = psi;
            Mat du = realise_deriv(op, vals, perms, theta);
            if ((rc = apply_op(vc, op, du, true))) return rc;
            std::vector<double> ip(2 * B);
            orc_inner(reinterpret_cast<double*>(phi.data()), reinterpret_cast<double*>(chi.data()), n, B, ip.data());
            double g = 0.0;
            for (std::int64_t b = 0; b < B; ++b) g += 2.0 * ip[2 * b];
            grads[op.param] += g;
        }
        if ((rc = apply_op(vf, op, ud))) return rc;  // φ̄_k = U_k† φ̄_{k+1}
    }
    if (psi_out) std::memcpy(psi_out, psi.data(), total * sizeof(cd));
    if (state_grad) std::memcpy(state_grad, phi.data(), total * sizeof(cd));
    return QBG_OK;
}

// The reverse loop of expect_grad alone (apply_back over a program): psi holds ψ_N, phi
// holds φ̄_N on entry; grads[nparams] accumulates.  Used to time the backward on a sample.
int orc_backward(double* st, double* ph, int n, std::int64_t B, const qbg_op* ops, std::int64_t nops,
                 const double* vals, const std::int64_t* perms, const double* theta, double* grads) {
    std::size_t total = (std::size_t{1} << n) * B;
    std::vector<cd> chi(total);
    View vp{reinterpret_cast<cd*>(st), n, n, B}, vf{reinterpret_cast<cd*>(ph), n, n, B}, vc{chi.data(), n, n, B};
    int rc;
    Timer tm;
    for (std::int64_t k = nops - 1; k >= 0; --k) {
        const qbg_op& op = ops[k];
        Mat ud = dagger(realise(op, vals, perms, theta));
        if ((rc = apply_op(vp, op, ud))) return rc;
        if (op.gen != QBG_GEN_NONE) {
            std::copy(reinterpret_cast<const cd*>(st), reinterpret_cast<const cd*>(st) + total, chi.begin());
            Mat du = realise_deriv(op, vals, perms, theta);
            if ((rc = apply_op(vc, op, du, true))) return rc;
            std::vector<double> ip(2 * B);
            orc_inner(ph, reinterpret_cast<double*>(chi.data()), n, B, ip.data());
            for (std::int64_t b = 0; b < B; ++b) grads[op.param] += 2.0 * ip[2 * b];
        }
        if ((rc = apply_op(vf, op, ud))) return rc;
    }
    tm.stop();
    return QBG_OK;
}

void orc_set_threads(int) {}  // the restatement is single-threaded

// ---- measurement (register.hpp:414-493) -------------------------------------------------------------
int orc_probabilities(const double* st, int n, int nactive, std::int64_t b, double* p) {
    std::size_t rows = std::size_t{1} << nactive, env = std::size_t{1} << (n - nactive);
    const cd* sl = reinterpret_cast<const cd*>(st) + b * (std::size_t{1} << n);
    for (std::size_t i = 0; i < rows; ++i) p[i] = 0.0;
    for (std::size_t e = 0; e < env; ++e)
        for (std::size_t i = 0; i < rows; ++i) p[i] += std::norm(sl[e * rows + i]);
    return QBG_OK;
}

static std::size_t draw(const std::vector<double>& cum, double u) {
    double target = u * cum.back();
    std::size_t lo = 0, hi = cum.size();  // first index with cum[idx] > target
    while (lo < hi) {
        std::size_t mid = lo + (hi - lo) / 2;
        if (cum[mid] > target) hi = mid;
        else lo = mid + 1;
    }
    return lo < cum.size() ? lo : cum.size() - 1;
}

int orc_measure(const double* st, int n, int nactive, std::int64_t B, std::int64_t nshots, void* rng,
                std::uint64_t* out) {
    if (nshots < 1) return fail(QBG_ERR_VALIDATION, "measure: nshots must be positive");
    ORng* r = static_cast<ORng*>(rng);
    std::size_t rows = std::size_t{1} << nactive;
    std::vector<double> p(rows), cum(rows);
    for (std::int64_t b = 0; b < B; ++b) {
        orc_probabilities(st, n, nactive, b, p.data());
        double run = 0.0;
        for (std::size_t i = 0; i < rows; ++i) cum[i] = (run += p[i]);
        for (std::int64_t s = 0; s < nshots; ++s) out[b * nshots + s] = draw(cum, r->unif());
    }
    return QBG_OK;
}

int orc_measure_collapse(double* st, int n, int nactive, std::int64_t B, void* rng, std::uint64_t* out) {
    ORng* r = static_cast<ORng*>(rng);
    std::size_t rows = std::size_t{1} << nactive, env = std::size_t{1} << (n - nactive);
    std::vector<double> p(rows), cum(rows);
    for (std::int64_t b = 0; b < B; ++b) {
        orc_probabilities(st, n, nactive, b, p.data());
        double run = 0.0;
        for (std::size_t i = 0; i < rows; ++i) cum[i] = (run += p[i]);
        std::size_t hit = draw(cum, r->unif());
        if (p[hit] <= 1e-300) return fail(QBG_ERR_RENORMALIZATION, "measure!: outcome has numerically zero probability");
        double inv = 1.0 / std::sqrt(p[hit]);
        cd* sl = reinterpret_cast<cd*>(st) + b * (std::size_t{1} << n);
        for (std::size_t e = 0; e < env; ++e)
            for (std::size_t i = 0; i < rows; ++i) sl[e * rows + i] = i == hit ? sl[e * rows + i] * inv : cd(0.0);
        out[b] = hit;
    }
    return QBG_OK;
}

// ---- state files (register.hpp:181-205): "QBREG1\0\0", 3 x u64, raw complex doubles ------------------
int orc_save(const double* st, int n, int nactive, std::int64_t B, const char* path) {
    FILE* f = std::fopen(path, "wb");
    if (!f) return fail(QBG_ERR_SERIALIZATION, "state file: cannot open");
    const char magic[8] = {'Q', 'B', 'R', 'E', 'G', '1', 0, 0};
    std::uint64_t hdr[3] = {static_cast<std::uint64_t>(n), static_cast<std::uint64_t>(nactive),
                            static_cast<std::uint64_t>(B)};
    std::size_t cnt = (std::size_t{1} << n) * static_cast<std::size_t>(B) * 2;
    bool ok = std::fwrite(magic, 1, 8, f) == 8 && std::fwrite(hdr, 8, 3, f) == 3 && std::fwrite(st, 8, cnt, f) == cnt;
    ok = std::fclose(f) == 0 && ok;
    return ok ? QBG_OK : fail(QBG_ERR_SERIALIZATION, "state file: write failed");
}

int orc_load(const char* path, double* st, std::int64_t cap, int* n, int* nactive, std::int64_t* B) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(QBG_ERR_SERIALIZATION, "state file: cannot open");
    char magic[8];
    std::uint64_t hdr[3];
    if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, "QBREG1\0\0", 8) != 0) {
        std::fclose(f);
        return fail(QBG_ERR_SERIALIZATION, "state file: bad magic");
    }
    if (std::fread(hdr, 8, 3, f) != 3 || hdr[0] < 1 || hdr[1] > hdr[0]) {
        std::fclose(f);
        return fail(QBG_ERR_SERIALIZATION, "state file: bad header");
    }
    std::size_t cnt = (std::size_t{1} << hdr[0]) * hdr[2];
    if (static_cast<std::int64_t>(cnt) > cap) {
        std::fclose(f);
        return fail(QBG_ERR_SHAPE, "orc_load: buffer too small");
    }
    bool ok = std::fread(st, 16, cnt, f) == cnt;
    std::fclose(f);
    if (!ok) return fail(QBG_ERR_SERIALIZATION, "state file: truncated amplitudes");
    *n = static_cast<int>(hdr[0]);
    *nactive = static_cast<int>(hdr[1]);
    *B = static_cast<std::int64_t>(hdr[2]);
    return QBG_OK;
}

// ---- focus / relax (register.hpp:156-177, 209-248) ---------------------------------------------------
static int order_of(int n, const std::int32_t* locs, int nloc, std::vector<int>& src) {
    if (nloc < 1) return fail(QBG_ERR_VALIDATION, "focus: need at least one location");
    std::vector<char> seen(n, 0);
    for (int k = 0; k < nloc; ++k) {
        if (locs[k] < 1 || locs[k] > n) return fail(QBG_ERR_RANGE, "focus: location out of range");
        if (seen[locs[k] - 1]) return fail(QBG_ERR_VALIDATION, "focus: duplicate location");
        seen[locs[k] - 1] = 1;
        src.push_back(locs[k] - 1);
    }
    for (int q = 0; q < n; ++q)
        if (!seen[q]) src.push_back(q);
    return QBG_OK;
}

static void permute_bits(cd* st, int n, std::int64_t B, const std::vector<int>& src) {
    std::size_t len = std::size_t{1} << n;
    std::vector<cd> tmp(len);
    for (std::int64_t b = 0; b < B; ++b) {
        cd* sl = st + b * len;
        for (std::size_t g = 0; g < len; ++g) {
            std::size_t dst = 0;
            for (int k = 0; k < n; ++k) dst |= ((g >> src[k]) & 1u) << k;
            tmp[dst] = sl[g];
        }
        std::copy(tmp.begin(), tmp.end(), sl);
    }
}

int orc_focus(double* st, int n, std::int64_t B, const std::int32_t* locs, int nloc) {
    std::vector<int> src;
    int rc = order_of(n, locs, nloc, src);
    if (rc) return rc;
    permute_bits(reinterpret_cast<cd*>(st), n, B, src);
    return QBG_OK;
}

int orc_relax(double* st, int n, std::int64_t B, const std::int32_t* locs, int nloc) {
    std::vector<int> src;
    int rc = order_of(n, locs, nloc, src);
    if (rc) return rc;
    std::vector<int> inv(n);
    for (int k = 0; k < n; ++k) inv[src[k]] = k;
    permute_bits(reinterpret_cast<cd*>(st), n, B, inv);
    return QBG_OK;
}

}  // extern "C"
