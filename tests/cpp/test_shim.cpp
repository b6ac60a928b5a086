// C++ consumer of the drop-in shim (include/qbg/qblock.hpp): the reference's own examples written
// against qbg::qblock exactly as they would be against qblock.  Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <numbers>

#include "qbg/qblock.hpp"

namespace qb = qbg::qblock;

static int failures = 0;
#define CHECK(c)                                                         \
    do {                                                                 \
        if (!(c)) {                                                      \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                  \
        }                                                                \
    } while (0)

int main() {
    // Listing 13 / SPEC.md:235: X on qubit 2 of zero_state(4), three shots -> 0010 (2)
    {
        auto reg = qb::zero_state(4);
        std::size_t l[] = {2};
        qb::instruct(reg, "X", l);
        auto out = qb::measure(reg, 3);
        CHECK(out.samples.size() == 3);
        for (auto& s : out.samples) CHECK(qb::to_text(s) == "0010 (2)");
    }
    // CNOT as instruct(X, (1,), (2,), (1,)) on |10> (qubit 2 set) -> |11>
    {
        auto reg = qb::product_state(qb::BitStr(0b10, 2));
        std::size_t t[] = {1}, c[] = {2};
        int cfg[] = {1};
        qb::instruct(reg, "X", t, c, cfg);
        auto a = reg.amplitudes();
        CHECK(std::abs(a[3] - qb::cplx(1.0)) < 1e-15);
    }
    // <Z> after Rx(0.4) = cos 0.4 (via probabilities)
    {
        auto reg = qb::zero_state(1);
        std::size_t l[] = {1};
        double th[] = {0.4};
        qb::instruct(reg, "Rx", l, {}, {}, th);
        auto p = qb::probabilities(reg, 0);
        CHECK(std::abs((p[0] - p[1]) - std::cos(0.4)) < 1e-14);
    }
    // Dense MatrixRepr path, norm preservation, inner
    {
        auto reg = qb::rand_state(10, 2, 7);
        double s = 1.0 / std::numbers::sqrt2;
        qb::MatrixRepr h = qb::Dense{2, {s, s, s, -s}};
        std::size_t l[] = {5};
        qb::instruct(reg, h, l);
        CHECK(std::abs(reg.norm(1) - 1.0) < 1e-13);
        qb::Register copy = reg;
        auto ip = reg.inner(copy);
        CHECK(std::abs(ip[0] - qb::cplx(1.0)) < 1e-13);
    }
    // Errors map to the reference's exception types
    {
        auto reg = qb::zero_state(3);
        bool ok = false;
        try {
            std::size_t l[] = {4};
            qb::instruct(reg, "X", l);
        } catch (const qb::RangeError&) {
            ok = true;
        }
        CHECK(ok);
        ok = false;
        try {
            std::size_t l[] = {1};
            qb::instruct(reg, "NoSuchGate", l);
        } catch (const qb::DispatchError&) {
            ok = true;
        }
        CHECK(ok);
    }
    // focus / relax round trip (register.hpp:156-177)
    {
        auto reg = qb::rand_state(6, 1, 3);
        auto before = reg.amplitudes();
        std::size_t l[] = {3, 6, 1, 2};
        reg.focus(l);
        CHECK(reg.nactive() == 4);
        reg.relax(l, 6);
        auto after = reg.amplitudes();
        double d = 0;
        for (std::size_t i = 0; i < after.size(); ++i) d = std::max(d, std::abs(after[i] - before[i]));
        CHECK(d == 0.0);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "shim ok", failures);
    return failures ? 1 : 0;
}
