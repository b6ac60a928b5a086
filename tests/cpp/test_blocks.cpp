// C++ consumer of the block / autodiff API (include/qbg/blocks.hpp) on the B200 engine: the paper's
// and the SPEC's examples written against the C++ API alone (no Python on the path).
//   argv[1]: output file for variational_circuit(16,10) expect' (energy, 16*31 gradients as raw
//   doubles) that the pytest wrapper compares with the reference-generated golden;
//   argv[2]: a QBREG1 file written by the reference (loaded and re-saved byte-identically).
// Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <numbers>
#include <sstream>

#include "qbg/blocks.hpp"

namespace qb = qbg::qblock;
using qb::BlockPtr;

static int failures = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

static double maxdiff(const std::vector<qb::cplx>& a, const std::vector<qb::cplx>& b) {
    double d = 0;
    for (std::size_t i = 0; i < a.size(); ++i) d = std::max(d, std::abs(a[i] - b[i]));
    return d;
}

int main(int argc, char** argv) {
    // App G: E and the three gradients with a periodic heisenberg(3)
    {
        auto circ = qb::chain(3, {qb::put(3, {2}, qb::Rx(0.5)), qb::control(3, std::vector<long>{2}, {1}, qb::Ry(0.7)),
                                  qb::put(3, {1, 2}, qb::rot(qb::kron({qb::X(), qb::X()}), 0.8))});
        auto h = qb::heisenberg(3, true);
        auto r = qb::expect_grad(h, qb::zero_state(3), circ);
        CHECK(std::abs(r.energies[0] - 1.9542144196547988) <= 1e-12);
        const double want[3] = {-1.2280830050051128, -0.31110858256435187, -1.5656386306937393};
        CHECK(r.param_grads.size() == 3);
        for (int k = 0; k < 3; ++k) CHECK(std::abs(r.param_grads[k] - want[k]) <= 1e-12);
        // expect through the pair form agrees with the forward value of expect'
        CHECK(std::abs(qb::expect(h, qb::zero_state(3), circ)[0] - r.energies[0]) <= 1e-13);
        // the controlled Ry has no shift rule (generator P1 ⊗ Y is not reflexive): rejected
        bool threw = false;
        try {
            qb::faithful_grad(h, qb::zero_state(3), circ);
        } catch (const qb::UnsupportedError&) {
            threw = true;
        }
        CHECK(threw);
    }
    // shift rule (exact mode) = reverse mode on an all-rotation circuit (gradient triangle)
    {
        auto c = qb::variational_circuit(4, 2);
        qb::Rng rng(3);
        qb::dispatch(c, "random", rng);
        auto h = qb::heisenberg(4);
        auto r = qb::expect_grad(h, qb::rand_state(4, 2, 1), c);
        auto fg = qb::faithful_grad(h, qb::rand_state(4, 2, 1), c);
        for (std::size_t k = 0; k < fg.size(); ++k) CHECK(std::abs(fg[k] - r.param_grads[k]) <= 1e-12);
    }
    // SPEC.md:459 / 469: <Z> after Rx(0.4) = cos 0.4, θ̄ = −sin 0.4; heisenberg(2) on |00> = 1
    {
        auto c = qb::chain(1, {qb::Rx(0.4)});
        auto r = qb::expect_grad(qb::Z(), qb::zero_state(1), c);
        CHECK(std::abs(r.energies[0] - std::cos(0.4)) <= 1e-15);
        CHECK(std::abs(r.param_grads[0] + std::sin(0.4)) <= 1e-15);
        CHECK(std::abs(qb::expect(qb::heisenberg(2), qb::zero_state(2))[0] - 1.0) <= 1e-15);
    }
    // parameters / dispatch / gatecount (Listing 9)
    {
        auto c = qb::variational_circuit(10, 3);
        CHECK(qb::nparameters(c) == 100);
        auto gc = qb::gatecount(c);
        CHECK(gc["Rz"] == 60 && gc["Rx"] == 40 && gc["Control{X}"] == 30);
        qb::Rng rng(42);
        qb::dispatch(c, "random", rng);
        auto th = qb::parameters(c);
        std::vector<double> neg(th.size());
        for (std::size_t k = 0; k < th.size(); ++k) neg[k] = -th[k];
        qb::dispatch(c, neg);
        qb::dispatch(c, [](double a, double b) { return a + 2 * b; }, std::span<const double>(th));
        CHECK(qb::parameters(c) == th);
        // shared node: one parameter, gradients summed over its occurrences
        auto shared = qb::Rx(0.3);
        auto c2 = qb::chain(2, {qb::put(2, {1}, shared), qb::put(2, {2}, shared)});
        CHECK(qb::nparameters(c2) == 1);
    }
    // apply then dagger(apply) restores the state; dagger of qft(3)
    {
        auto c = qb::variational_circuit(12, 2);
        qb::Rng rng(7);
        qb::dispatch(c, "random", rng);
        auto reg = qb::rand_state(12, 2, 5);
        auto before = reg.amplitudes();
        qb::apply(reg, c);
        qb::apply(reg, qb::dagger(c));
        CHECK(maxdiff(reg.amplitudes(), before) <= 1e-13);
        auto q = qb::qft(3);
        auto r3 = qb::rand_state(3, 1, 9);
        auto b3 = r3.amplitudes();
        qb::apply(r3, q);
        qb::apply(r3, qb::dagger(q));
        CHECK(maxdiff(r3.amplitudes(), b3) <= 1e-14);
    }
    // Subroutine (Listing 16): qft(4)' on qubits 1..4 of a 5-qubit register equals
    // the explicit focus -> apply -> relax sequence (Listing 15)
    {
        auto sub = qb::subroutine(5, qb::dagger(qb::qft(4)), {1, 2, 3, 4});
        auto a = qb::rand_state(5, 1, 11), b = a;
        qb::apply(a, sub);
        std::size_t locs[] = {1, 2, 3, 4};
        b.focus(locs);
        qb::apply(b, qb::dagger(qb::qft(4)));
        b.relax(locs, 5);
        CHECK(maxdiff(a.amplitudes(), b.amplitudes()) <= 1e-14);
        // subroutine on permuted locations = put on them
        auto c = qb::put(5, {4, 2}, qb::CNOT());
        auto s = qb::subroutine(5, qb::chain(2, {qb::put(2, {1, 2}, qb::CNOT())}), {4, 2});
        auto x = qb::rand_state(5, 1, 12), y = x;
        qb::apply(x, c);
        qb::apply(y, s);
        CHECK(maxdiff(x.amplitudes(), y.amplitudes()) <= 1e-15);
    }
    // observables: Add/Scale apply as linear maps; <O> from Pauli terms equals <ψ|Oψ>
    {
        auto h = qb::heisenberg(6);
        auto reg = qb::rand_state(6, 1, 3);
        auto hpsi = reg;
        qb::apply(hpsi, h);
        const double e = reg.inner(hpsi)[0].real();
        CHECK(std::abs(qb::expect(h, reg)[0] - e) <= 1e-13);
        auto o = qb::scale(0.5, qb::put(6, {2}, qb::Z())) + qb::kron(6, {{{1}, qb::X()}, {{3}, qb::Y()}});
        CHECK(qb::pauli_terms(o).size() == 2);
    }
    // shim surface: product_state(BitStr), gatemat / gate_by_tag, SparseColumns instruct, QBREG1 streams
    {
        auto reg = qb::product_state(qb::bits_from_text("0110"));
        CHECK(reg.nqubits() == 4 && std::abs(reg.amplitudes()[6] - qb::cplx(1.0)) == 0.0);
        CHECK(qb::to_text(qb::from_bits({0, 1, 1, 0})) == "0110 (2)");
        std::size_t l[] = {2};
        qb::instruct(reg, qb::gatemat::p1(), l);  // SparseColumns -> densified (register.hpp:372)
        CHECK(std::abs(reg.amplitudes()[6] - qb::cplx(1.0)) == 0.0);
        double th[] = {0.9};
        auto a = qb::rand_state(6, 1, 4), b = a;
        qb::instruct(a, qb::gatemat::rot(qb::gatemat::x(), 0.9), l);
        qb::instruct(b, "Rx", l, {}, {}, th);
        CHECK(maxdiff(a.amplitudes(), b.amplitudes()) <= 1e-15);
        qb::define_const_gate("ISWAP", qb::Permutation({0, 2, 1, 3}, {1.0, qb::cplx(0, 1), qb::cplx(0, 1), 1.0}));
        std::size_t l2[] = {1, 3};
        qb::instruct(a, "ISWAP", l2);
        std::stringstream ss;
        a.save(ss);
        auto c = qb::Register::load(ss);
        CHECK(maxdiff(c.amplitudes(), a.amplitudes()) == 0.0 && c.nactive() == 6);
    }
    // a QBREG1 file written by the reference itself (tests/golden/state_qbreg1.bin, nactive 3 of 4)
    if (argc > 2) {
        std::ifstream f(argv[2], std::ios::binary);
        auto r = qb::Register::load(f, 7);
        CHECK(r.nqubits() == 4 && r.nactive() == 3 && r.nbatch() == 2);
        std::stringstream back;
        r.save(back);
        std::ifstream f2(argv[2], std::ios::binary);
        std::string orig((std::istreambuf_iterator<char>(f2)), std::istreambuf_iterator<char>());
        CHECK(back.str() == orig);  // byte-identical round trip
    }
    // variational_circuit(16, 10), θ = dispatch("random") from Rng(42): expect' through the C++ API
    {
        auto c = qb::variational_circuit(16, 10);
        qb::Rng rng(42);
        qb::dispatch(c, "random", rng);
        auto r = qb::expect_grad(qb::heisenberg(16), qb::zero_state(16), c, false);
        if (argc > 1) {
            std::ofstream f(argv[1], std::ios::binary);
            f.write(reinterpret_cast<const char*>(r.energies.data()), sizeof(double));
            f.write(reinterpret_cast<const char*>(r.param_grads.data()),
                    static_cast<std::streamsize>(r.param_grads.size() * sizeof(double)));
        }
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "blocks ok", failures);
    return failures ? 1 : 0;
}
