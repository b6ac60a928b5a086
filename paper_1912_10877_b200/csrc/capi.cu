// capi.cu — the extern "C" boundary (include/qbg.h) over the device engine.
//
// Replaces the reference's register "instruction set" (register.hpp:58-493) and the SPEC's
// apply / expect / expect_grad.  All device work is issued on
// one stream per process (qbg_set_stream); calls that return host values synchronise it.
// There is no CPU fallback: without a CUDA device every call fails with QBG_ERR_CUDA.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <numbers>
#include <random>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "engine.h"
#include "program.h"
#include "jit.h"

// ---- opaque handles ---------------------------------------------------------------------------
struct qbg_rng {
    uint64_t state;
    std::mt19937_64 eng;
    explicit qbg_rng(uint64_t seed);
};

struct qbg_reg {
    qbg::DevState s;
    int nactive = 0;
    qbg_rng rng{42};
    std::vector<std::vector<int32_t>> focus_stack;
};

struct qbg_prog {
    qbg::Program p;
};
struct qbg_obs {
    qbg::Observable o;
};

namespace qbg {

// ---- library state ---------------------------------------------------------------------------
namespace {
thread_local std::string g_err;
std::atomic<int32_t> g_cap{30};
std::atomic<uint64_t> g_allocs{0};
std::atomic<uint64_t> g_launches{0};
cudaStream_t g_stream = nullptr;
int g_device = 0;
// Set once the library holds anything on g_device (registers, scratch, workspace, plan tables,
// loaded kernels): from then on qbg_set_device may not move the library to another device, since
// every cached pointer / CUfunction belongs to this device's context.
std::atomic<bool> g_bound{false};
int g_sms = 0;
bool g_fusion = true;
bool g_profile = false;

struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
    double bytes;
    double flops;
};
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t get_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    QBG_CUDA(cudaEventCreate(&e));
    return e;
}

struct Scratch {
    void* p = nullptr;
    size_t bytes = 0;
};
Scratch g_scratch[24];  // slots: see the scratch(…, k) call sites (one owner each while live)

uint64_t mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return QBG_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return QBG_ERR_RESOURCE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return QBG_ERR_INTERNAL;
    }
}

void ensure_device() {
    static bool init = false;
    if (init) return;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        raise(QBG_ERR_CUDA, std::string("no CUDA device available (") + cudaGetErrorString(e) +
                                "); the qbg engine has no CPU fallback");
    QBG_CUDA(cudaSetDevice(g_device));
    QBG_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, g_device));
    init = true;
}

void* dev_alloc(size_t bytes, bool state) {
    ensure_device();
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        raise(QBG_ERR_RESOURCE, "device allocation of " + std::to_string(bytes) + " bytes failed: " +
                                    cudaGetErrorString(e));
    }
    if (state) g_allocs.fetch_add(1);
    g_bound.store(true);
    return p;
}

// ---- library-owned full-state workspace (the expect' work copy and adjoint; Krylov bases) ----
// Replaces per-thread static buffers: owned here, counted by qbg_alloc_count, released by
// qbg_release_workspace and automatically once no live register is as large as a buffer.
std::mutex g_ws_mu;
std::vector<qbg_reg*> g_live;  // live registers (for the release rule)
DevState g_ws[2];              // [0] forward work state (out-of-place expect'), [1] adjoint buffer
// checkpoints of the checkpointed expect' (fused_ckpt_*): one allocation of k full states
struct CkptArena {
    void* ptr = nullptr;
    size_t bytes = 0, state_bytes = 0;
} g_ckpt;
std::atomic<int64_t> g_ckpt_limit{-1};  // qbg_set_checkpoint_limit (bytes; -1: free memory less a reserve)

void ws_free(DevState& d) {
    if (!d.ptr) return;
    QBG_CUDA(cudaStreamSynchronize(g_stream));
    QBG_CUDA(cudaFree(d.ptr));
    d = DevState{};
}
// a buffer shaped like s (reused when it is at least as large and of the same dtype)
DevState& ws_get(int k, const DevState& s) {
    DevState& d = g_ws[k];
    if (!(d.ptr && d.bytes() >= s.bytes() && d.dtype == s.dtype)) {
        ws_free(d);
        d = s;
        d.ptr = dev_alloc(s.bytes(), true);
    }
    return d;
}

void ckpt_free() {
    if (!g_ckpt.ptr) return;
    QBG_CUDA(cudaStreamSynchronize(g_stream));
    QBG_CUDA(cudaFree(g_ckpt.ptr));
    g_ckpt = CkptArena{};
}
// k checkpoints shaped like s, or nullptr when they would not leave a reserve of device memory free
// (max(4 GiB, 1/16 of the device)) — the caller then runs the uncompute design
void* ckpt_get(int64_t k, const DevState& s) {
    const size_t need = static_cast<size_t>(k) * s.bytes();
    const int64_t lim = g_ckpt_limit.load();
    if (lim >= 0 && need > static_cast<size_t>(lim)) return nullptr;
    if (g_ckpt.ptr && g_ckpt.bytes >= need) {
        g_ckpt.state_bytes = std::max(g_ckpt.state_bytes, s.bytes());
        return g_ckpt.ptr;
    }
    ensure_device();
    size_t fr = 0, tot = 0;
    QBG_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t reserve = std::max<size_t>(size_t{4} << 30, tot / 16);
    // (a request that cannot fit leaves the current arena alone)
    if (need + reserve > fr + g_ckpt.bytes) return nullptr;
    ckpt_free();
    QBG_CUDA(cudaMemGetInfo(&fr, &tot));
    if (need + reserve > fr) return nullptr;
    void* p = nullptr;
    if (cudaMalloc(&p, need) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    g_allocs.fetch_add(1);
    g_bound.store(true);
    g_ckpt.ptr = p;
    g_ckpt.bytes = need;
    g_ckpt.state_bytes = s.bytes();
    return p;
}

void stream_sync() { QBG_CUDA(cudaStreamSynchronize(g_stream)); }

qbg_reg* new_reg(int n, int64_t B, int dtype) {
    if (n < 1) raise(QBG_ERR_VALIDATION, "Register: need at least one qubit");
    if (n > g_cap.load())
        raise(QBG_ERR_RESOURCE, "Register: " + std::to_string(n) + " qubits exceeds the cap of " +
                                    std::to_string(g_cap.load()));
    if (B < 1) raise(QBG_ERR_VALIDATION, "Register: batch count must be positive");
    if (dtype != QBG_C128 && dtype != QBG_C64) raise(QBG_ERR_VALIDATION, "Register: unknown dtype");
    auto* r = new qbg_reg;
    r->s.n = n;
    r->s.B = B;
    r->s.dtype = dtype;
    r->nactive = n;
    try {
        r->s.ptr = dev_alloc(r->s.bytes(), true);
    } catch (...) {
        delete r;
        throw;
    }
    std::lock_guard<std::mutex> lk(g_ws_mu);
    g_live.push_back(r);
    return r;
}

void check_reg(const qbg_reg* r) {
    if (!r || !r->s.ptr) raise(QBG_ERR_VALIDATION, "null register");
}

void same_shape(const qbg_reg* a, const qbg_reg* b, const char* what) {
    check_reg(a);
    check_reg(b);
    if (a->s.n != b->s.n || a->s.B != b->s.B || a->s.dtype != b->s.dtype)
        raise(QBG_ERR_SHAPE, std::string(what) + ": shape mismatch");
}

// ---- gate table (gates.hpp:32-94) on the host -------------------------------------------
using cd = std::complex<double>;

struct HostGate {
    int kind;
    int dim;
    std::vector<cd> v;
    std::vector<int> perm;
};

HostGate H_diag(std::vector<cd> d) { return HostGate{QBG_MAT_DIAGONAL, static_cast<int>(d.size()), d, {}}; }
HostGate H_perm(std::vector<int> p, std::vector<cd> v) {
    return HostGate{QBG_MAT_PERMUTATION, static_cast<int>(p.size()), v, p};
}
HostGate H_dense(int dim, std::vector<cd> a) { return HostGate{QBG_MAT_DENSE, dim, a, {}}; }

HostGate gate_by_tag(const std::string& tag, const double* params, int nparams) {
    const cd i1(0.0, 1.0);
    if (tag == "Rx" || tag == "Ry" || tag == "Rz" || tag == "shift" || tag == "phase") {
        if (nparams != 1) raise(QBG_ERR_DISPATCH, "gate " + tag + " expects one parameter");
        double th = params[0];
        if (tag == "Rx") {
            cd c = std::cos(th / 2), ms = -i1 * std::sin(th / 2);
            return H_dense(2, {c, ms, ms, c});
        }
        if (tag == "Ry") {
            double c = std::cos(th / 2), s = std::sin(th / 2);
            return H_dense(2, {c, s, -s, c});
        }
        if (tag == "Rz") return H_diag({std::polar(1.0, -th / 2), std::polar(1.0, th / 2)});
        if (tag == "shift") return H_diag({1.0, std::polar(1.0, th)});
        return H_diag({std::polar(1.0, th), std::polar(1.0, th)});
    }
    if (nparams != 0) {
        static const char* known[] = {"X",  "Y",    "Z",  "H",  "I2", "S",  "Sdag", "T",  "Tdag",
                                      "SWAP", "CNOT", "CZ", "Toffoli", "P0", "P1", "Pu", "Pd"};
        for (auto* k : known)
            if (tag == k) raise(QBG_ERR_DISPATCH, "gate " + tag + " takes no parameters");
    }
    double s = 1.0 / std::numbers::sqrt2;
    if (tag == "X") return H_perm({1, 0}, {1.0, 1.0});
    if (tag == "Y") return H_perm({1, 0}, {-i1, i1});
    if (tag == "Z") return H_diag({1.0, -1.0});
    if (tag == "H") return H_dense(2, {s, s, s, -s});
    if (tag == "I2") return HostGate{QBG_MAT_IDENTITY, 2, {}, {}};
    if (tag == "S") return H_diag({1.0, i1});
    if (tag == "Sdag") return H_diag({1.0, -i1});
    if (tag == "T") return H_diag({1.0, std::polar(1.0, std::numbers::pi / 4)});
    if (tag == "Tdag") return H_diag({1.0, std::polar(1.0, -std::numbers::pi / 4)});
    if (tag == "SWAP") return H_perm({0, 2, 1, 3}, {1.0, 1.0, 1.0, 1.0});
    if (tag == "CNOT") return H_perm({0, 1, 3, 2}, {1.0, 1.0, 1.0, 1.0});
    if (tag == "CZ") return H_perm({0, 1, 2, 3}, {1.0, 1.0, 1.0, -1.0});
    if (tag == "Toffoli") return H_perm({0, 1, 2, 3, 4, 5, 7, 6}, std::vector<cd>(8, 1.0));
    // projectors (SparseColumns in the reference, densified by its generic path)
    if (tag == "P0") return H_dense(2, {1.0, 0.0, 0.0, 0.0});
    if (tag == "P1") return H_dense(2, {0.0, 0.0, 0.0, 1.0});
    if (tag == "Pu") return H_dense(2, {0.0, 0.0, 1.0, 0.0});
    if (tag == "Pd") return H_dense(2, {0.0, 1.0, 0.0, 0.0});
    raise(QBG_ERR_DISPATCH, "unknown gate tag: " + tag);
}

std::vector<cdbl> to_cdbl(const std::vector<cd>& v) {
    std::vector<cdbl> o(v.size());
    for (size_t k = 0; k < v.size(); ++k) o[k] = cdbl{v[k].real(), v[k].imag()};
    return o;
}

}  // namespace

// ---- shared helpers used by the other translation units -----------------------------------
cudaStream_t stream() { return g_stream; }
int num_sms() {
    ensure_device();
    return g_sms;
}

void release_krylov(size_t keep_bytes);  // capi.cu, below the Krylov driver
void release_scratch() {
    QBG_CUDA(cudaStreamSynchronize(g_stream));
    for (auto& s : g_scratch) {
        if (s.p) QBG_CUDA(cudaFree(s.p));
        s = Scratch{};
    }
}

void* scratch(size_t bytes, int slot) {
    Scratch& s = g_scratch[slot];
    if (s.bytes < bytes) {
        if (s.p) {
            QBG_CUDA(cudaStreamSynchronize(g_stream));
            QBG_CUDA(cudaFree(s.p));
        }
        s.p = dev_alloc(bytes, false);
        s.bytes = bytes;
    }
    return s.p;
}

LaunchScope::LaunchScope(const char* n, double b, double flops) : name(n), bytes(b) {
    g_launches.fetch_add(1);
    if (g_profile) {
        cudaEvent_t a = get_event();
        QBG_CUDA(cudaEventRecord(a, g_stream));
        g_prof.push_back(ProfRec{n, a, nullptr, b, flops});
    }
}
LaunchScope::~LaunchScope() {
    if (g_profile && !g_prof.empty() && g_prof.back().name == name && g_prof.back().b == nullptr) {
        cudaEvent_t e = get_event();
        cudaEventRecord(e, g_stream);
        g_prof.back().b = e;
    }
}

// make_plan's validation order (register.hpp:301-323)
void validate_op(int nactive, const qbg_op& op) {
    if (op.ntarget < 1) raise(QBG_ERR_VALIDATION, "instruct: need at least one target qubit");
    if (op.ntarget > QBG_MAX_TARGETS) raise(QBG_ERR_UNSUPPORTED, "instruct: more than 5 targets");
    if (op.nctrl < 0 || op.nctrl > QBG_MAX_CTRLS)
        raise(QBG_ERR_VALIDATION, "instruct: control locations and configuration differ in length");
    uint64_t lm = 0, cm = 0;
    for (int k = 0; k < op.ntarget; ++k) {
        int l = op.targets[k];
        if (l < 1 || l > nactive) raise(QBG_ERR_RANGE, "instruct: target qubit out of range");
        uint64_t b = uint64_t{1} << (l - 1);
        if (lm & b) raise(QBG_ERR_VALIDATION, "instruct: duplicate target qubit");
        lm |= b;
    }
    for (int k = 0; k < op.nctrl; ++k) {
        int l = op.ctrls[k];
        if (l < 1 || l > nactive) raise(QBG_ERR_RANGE, "instruct: control qubit out of range");
        if (op.ctrl_cfg[k] != 0 && op.ctrl_cfg[k] != 1)
            raise(QBG_ERR_VALIDATION, "instruct: control configuration must be 0 or 1");
        uint64_t b = uint64_t{1} << (l - 1);
        if ((lm | cm) & b) raise(QBG_ERR_VALIDATION, "instruct: control qubit overlaps another location");
        cm |= b;
    }
    if (op.dim != (1 << op.ntarget)) raise(QBG_ERR_SHAPE, "instruct: gate dimension does not match target count");
}

Gate place_gate(const qbg_op& op, int kind, int dim, const std::vector<cdbl>& m, const std::vector<int>& perm) {
    Gate g;
    g.kind = kind;
    g.t = op.ntarget;
    g.dim = dim;
    for (int q = 0; q < op.ntarget; ++q) {
        g.tbit[q] = static_cast<uint8_t>(op.targets[q] - 1);
        g.tmask |= uint64_t{1} << (op.targets[q] - 1);
    }
    for (int k = 0; k < op.nctrl; ++k) {
        uint64_t b = uint64_t{1} << (op.ctrls[k] - 1);
        g.cmask |= b;
        if (op.ctrl_cfg[k]) g.cval |= b;
    }
    g.m = m;
    g.perm = perm;
    return g;
}

// rot(G, θ) with the exact arithmetic sequence of gates.hpp:79-92
void realise(Program& p) {
    const cd I(0.0, 1.0);
    p.real.resize(p.ops.size());
    for (size_t k = 0; k < p.ops.size(); ++k) {
        const qbg_op& op = p.ops[k];
        int dim = op.dim;
        std::vector<cd> pay;
        std::vector<int> perm;
        const cdbl* src = p.vals.data() + op.data;
        if (op.kind == QBG_MAT_DIAGONAL || op.kind == QBG_MAT_PERMUTATION)
            for (int r = 0; r < dim; ++r) pay.emplace_back(src[r].re, src[r].im);
        if (op.kind == QBG_MAT_DENSE)
            for (int r = 0; r < dim * dim; ++r) pay.emplace_back(src[r].re, src[r].im);
        if (op.kind == QBG_MAT_PERMUTATION)
            for (int r = 0; r < dim; ++r) perm.push_back(static_cast<int>(p.perms[op.perm + r]));
        RealOp ro;
        ro.param = op.gen == QBG_GEN_NONE ? -1 : op.param;
        if (op.gen == QBG_GEN_NONE) {
            ro.u = place_gate(op, op.kind, dim, to_cdbl(pay), perm);
        } else if (op.gen == QBG_GEN_ROTATION) {
            double th = p.theta[op.param];
            double c = std::cos(th / 2), s = std::sin(th / 2);
            if (op.kind == QBG_MAT_IDENTITY || op.kind == QBG_MAT_DIAGONAL) {
                std::vector<cd> d(dim);
                for (int r = 0; r < dim; ++r) {
                    cd g = op.kind == QBG_MAT_IDENTITY ? cd(1.0) : pay[r];
                    d[r] = cd(c) - I * cd(s) * g;
                }
                ro.u = place_gate(op, QBG_MAT_DIAGONAL, dim, to_cdbl(d), {});
                std::vector<cd> kd(dim);
                for (int r = 0; r < dim; ++r) kd[r] = op.kind == QBG_MAT_IDENTITY ? cd(1.0) : pay[r];
                ro.k = place_gate(op, QBG_MAT_DIAGONAL, dim, to_cdbl(kd), {});
            } else {
                std::vector<cd> dn(static_cast<size_t>(dim) * dim, cd(0.0));
                if (op.kind == QBG_MAT_PERMUTATION)
                    for (int r = 0; r < dim; ++r) dn[perm[r] * dim + r] += pay[r];
                else
                    dn = pay;
                std::vector<cd> u = dn;
                cd f = -I * s;
                for (auto& e : u) e *= f;
                for (int r = 0; r < dim; ++r) u[r * dim + r] += c;
                ro.u = place_gate(op, QBG_MAT_DENSE, dim, to_cdbl(u), {});
                ro.k = op.kind == QBG_MAT_PERMUTATION ? place_gate(op, QBG_MAT_PERMUTATION, dim, to_cdbl(pay), perm)
                                                      : place_gate(op, QBG_MAT_DENSE, dim, to_cdbl(dn), {});
            }
        } else if (op.gen == QBG_GEN_SHIFT) {
            double th = p.theta[op.param];
            ro.u = place_gate(op, QBG_MAT_DIAGONAL, dim, to_cdbl({cd(1.0), std::polar(1.0, th)}), {});
            ro.k = place_gate(op, QBG_MAT_DIAGONAL, dim, to_cdbl({cd(0.0), cd(-2.0)}), {});
        } else {
            double th = p.theta[op.param];
            ro.u = place_gate(op, QBG_MAT_DIAGONAL, dim, to_cdbl(std::vector<cd>(dim, std::polar(1.0, th))), {});
            ro.k = place_gate(op, QBG_MAT_DIAGONAL, dim, to_cdbl(std::vector<cd>(dim, cd(-2.0))), {});
        }
        ro.udag = adjoint(ro.u);
        p.real[k] = std::move(ro);
    }
    p.realised = true;
}

// A new parameter vector on an already realised program: only the parameterised ops change, and
// only their matrix values (kind, placement and generator stay), so they are rewritten in place —
// the same arithmetic as realise(), without its per-op allocations (dispatch → apply is on the
// end-to-end path of every optimiser step).
void realise_params(Program& p) {
    const cd I(0.0, 1.0);
    for (size_t k = 0; k < p.ops.size(); ++k) {
        const qbg_op& op = p.ops[k];
        if (op.gen == QBG_GEN_NONE) continue;
        RealOp& ro = p.real[k];
        const int dim = op.dim;
        const cdbl* src = p.vals.data() + op.data;
        const double th = p.theta[op.param];
        std::vector<cdbl>& u = ro.u.m;
        if (op.gen == QBG_GEN_ROTATION) {
            const double c = std::cos(th / 2), s = std::sin(th / 2);
            if (op.kind == QBG_MAT_IDENTITY || op.kind == QBG_MAT_DIAGONAL) {
                for (int r = 0; r < dim; ++r) {
                    const cd g = op.kind == QBG_MAT_IDENTITY ? cd(1.0) : cd(src[r].re, src[r].im);
                    const cd d = cd(c) - I * cd(s) * g;
                    u[r] = cdbl{d.real(), d.imag()};
                }
            } else {
                const cd f = -I * s;
                for (auto& e : u) e = cdbl{0.0, 0.0};
                if (op.kind == QBG_MAT_PERMUTATION) {
                    for (int r = 0; r < dim; ++r) {
                        const size_t at = static_cast<size_t>(p.perms[op.perm + r]) * dim + r;
                        cd e(u[at].re, u[at].im);
                        e += cd(src[r].re, src[r].im);
                        u[at] = cdbl{e.real(), e.imag()};
                    }
                } else {
                    for (int r = 0; r < dim * dim; ++r) u[r] = src[r];
                }
                for (auto& e : u) {
                    cd v(e.re, e.im);
                    v *= f;
                    e = cdbl{v.real(), v.imag()};
                }
                for (int r = 0; r < dim; ++r) {
                    cd v(u[r * dim + r].re, u[r * dim + r].im);
                    v += c;  // as realise(): complex += double leaves the imaginary part alone
                    u[r * dim + r] = cdbl{v.real(), v.imag()};
                }
            }
        } else if (op.gen == QBG_GEN_SHIFT) {
            const cd e = std::polar(1.0, th);
            u[0] = cdbl{1.0, 0.0};
            u[1] = cdbl{e.real(), e.imag()};
        } else {
            const cd e = std::polar(1.0, th);
            for (auto& v : u) v = cdbl{e.real(), e.imag()};
        }
        // udag = adjoint(u) (kernels.cu), in place
        std::vector<cdbl>& a = ro.udag.m;
        if (ro.u.kind == QBG_MAT_DENSE) {
            for (int cc = 0; cc < dim; ++cc)
                for (int r = 0; r < dim; ++r) a[r * dim + cc] = cdbl{u[cc * dim + r].re, -u[cc * dim + r].im};
        } else {
            for (size_t r = 0; r < u.size(); ++r) a[r] = cdbl{u[r].re, -u[r].im};
        }
    }
}

namespace {

// NVTX ranges around the engine's phases (visible to ncu --nvtx / nsys; no cost without a tool)
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

// src (optional): the input when it is not s — s receives U·src (out-of-place apply).
void run_program(const DevState& s, Program& p, bool adjoint, const void* src = nullptr) {
    Nvtx r(adjoint ? "qbg.apply_adjoint" : "qbg.apply");
    if (!p.realised) realise(p);
    if (g_fusion && fused_forward(s, p, adjoint, src)) return;
    if (src) QBG_CUDA(cudaMemcpyAsync(s.ptr, src, s.bytes(), cudaMemcpyDeviceToDevice, g_stream));
    size_t N = p.real.size();
    for (size_t q = 0; q < N; ++q) {
        size_t k = adjoint ? N - 1 - q : q;
        launch_gate(s, adjoint ? p.real[k].udag : p.real[k].u);
    }
}

void run_obs(const DevState& psi, const DevState& phi, Observable& o, double* d_energy) {
    Nvtx r("qbg.observable");
    if (g_fusion && fused_obs_apply(psi, phi, o, d_energy)) return;
    if (o.terms.empty()) {
        QBG_CUDA(cudaMemsetAsync(phi.ptr, 0, phi.bytes(), g_stream));
    }
    for (size_t t = 0; t < o.terms.size(); ++t)
        launch_pauli_axpy(psi, phi, o.terms[t].xmask, o.terms[t].zmask, o.terms[t].coef_re, o.terms[t].coef_im,
                          t == 0);
    if (d_energy) {
        double* ip = static_cast<double*>(scratch(2 * psi.B * sizeof(double), 2));
        reduce_inner(psi, &phi, ip);
        // keep only the real parts: energies are read back by the caller from ip
        QBG_CUDA(cudaMemcpy2DAsync(d_energy, sizeof(double), ip, 2 * sizeof(double), sizeof(double), psi.B,
                                   cudaMemcpyDeviceToDevice, g_stream));
    }
}

// reverse pass; d_grads (device, nparams) receives the accumulated gradient
void run_backward(const DevState& psi, const DevState& adj, Program& p, double* d_grads) {
    Nvtx r("qbg.backward");
    if (!p.realised) realise(p);
    if (g_fusion && fused_backward(psi, adj, p, d_grads)) return;
    size_t N = p.real.size();
    int64_t cap = static_cast<int64_t>(num_sms()) * 8;
    int64_t nparam_ops = 0;
    for (auto& r : p.real) nparam_ops += r.param >= 0;
    double* part = static_cast<double*>(scratch(std::max<int64_t>(1, nparam_ops) * cap * sizeof(double), 3));
    QBG_CUDA(cudaMemsetAsync(part, 0, std::max<int64_t>(1, nparam_ops) * cap * sizeof(double), g_stream));
    std::vector<int> slot_param;
    for (size_t q = 0; q < N; ++q) {
        size_t k = N - 1 - q;
        const RealOp& r = p.real[k];
        int used = 0;
        if (r.param >= 0) {
            launch_gate_back(psi, adj, r.udag, &r.k, part + slot_param.size() * cap, cap, &used);
            slot_param.push_back(r.param);
        } else {
            launch_gate_back(psi, adj, r.udag, nullptr, nullptr, cap, &used);
        }
    }
    if (slot_param.empty()) return;
    int* dmap = static_cast<int*>(scratch(slot_param.size() * sizeof(int), 4));
    QBG_CUDA(cudaMemcpyAsync(dmap, slot_param.data(), slot_param.size() * sizeof(int), cudaMemcpyHostToDevice,
                             g_stream));
    accumulate_grads(part, static_cast<int64_t>(slot_param.size()), cap, dmap, d_grads);
    stream_sync();  // slot_param (host) must outlive the async copy
}

}  // namespace
}  // namespace qbg

using namespace qbg;

qbg_rng::qbg_rng(uint64_t seed) : state(qbg::mix(seed)), eng(qbg::mix(seed)) {}

extern "C" {

const char* qbg_last_error(void) { return g_err.c_str(); }
const char* qbg_version(void) { return "qbg 0.1 (sm_100a)"; }

int qbg_set_qubit_cap(int32_t cap) {
    return guarded([&] {
        if (cap < 1 || cap > 62) raise(QBG_ERR_VALIDATION, "qubit cap must be in 1..62");
        g_cap.store(cap);
    });
}
int32_t qbg_get_qubit_cap(void) { return g_cap.load(); }
uint64_t qbg_alloc_count(void) { return g_allocs.load(); }

int qbg_set_device(int32_t device) {
    return guarded([&] {
        if (device != g_device && g_bound.load())
            raise(QBG_ERR_VALIDATION, "qbg_set_device: the library already holds resources on device " +
                                          std::to_string(g_device) + " (registers, workspace, plans, kernels); "
                                          "select the device before the first allocation (one device per process)");
        g_device = device;
        QBG_CUDA(cudaSetDevice(device));
        QBG_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, device));
    });
}
int qbg_set_stream(void* s) {
    g_stream = static_cast<cudaStream_t>(s);
    return QBG_OK;
}
int qbg_synchronize(void) {
    return guarded([&] {
        ensure_device();
        stream_sync();
    });
}
int qbg_set_dense_path(int32_t path) {
    return guarded([&] {
        if (path < 0 || path > 2) raise(QBG_ERR_VALIDATION, "dense path must be 0 (CUDA cores), 1 (FP64 tensor cores) or 2 (tcgen05 TF32)");
        set_dense_path(path);
    });
}
int qbg_set_fusion(int32_t on) {
    g_fusion = on != 0;
    return QBG_OK;
}
int qbg_set_checkpointing(int32_t on) {
    fused_set_checkpointing(on != 0);
    return QBG_OK;
}
int qbg_set_checkpoint_limit(int64_t bytes) {
    g_ckpt_limit.store(bytes < 0 ? -1 : bytes);
    return QBG_OK;
}
int qbg_profile_enable(int32_t on) {
    g_profile = on != 0;
    return QBG_OK;
}
int qbg_profile_reset(void) {
    return guarded([&] {
        for (auto& r : g_prof) {
            g_event_pool.push_back(r.a);
            if (r.b) g_event_pool.push_back(r.b);
        }
        g_prof.clear();
    });
}
int qbg_profile_report(char* buf, int64_t cap) {
    return guarded([&] {
        stream_sync();
        struct Agg {
            int64_t n = 0;
            double ms = 0, bytes = 0, flops = 0;
        };
        std::map<std::string, Agg> agg;
        for (auto& r : g_prof) {
            if (!r.b) continue;
            float ms = 0;
            QBG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
            auto& a = agg[r.name];
            a.n++;
            a.ms += ms;
            a.bytes += r.bytes;
            a.flops += r.flops;
        }
        std::string out;
        char line[256];
        for (auto& [k, a] : agg) {
            std::snprintf(line, sizeof(line), "%s\t%lld\t%.6f\t%.6e\t%.6e\n", k.c_str(), static_cast<long long>(a.n),
                          a.ms, a.bytes, a.flops);
            out += line;
        }
        if (cap > 0) {
            std::strncpy(buf, out.c_str(), static_cast<size_t>(cap - 1));
            buf[cap - 1] = 0;
        }
    });
}
uint64_t qbg_launch_count(void) { return g_launches.load(); }
int qbg_launch_count_reset(void) {
    g_launches.store(0);
    return QBG_OK;
}

// ---- rng ---------------------------------------------------------------------------------------
int qbg_rng_create(uint64_t seed, qbg_rng** out) {
    return guarded([&] { *out = new qbg_rng(seed); });
}
int qbg_rng_destroy(qbg_rng* r) {
    delete r;
    return QBG_OK;
}
int qbg_rng_split_label(const qbg_rng* r, const char* label, qbg_rng** out) {
    return guarded([&] {
        uint64_t h = r->state;
        for (const char* c = label; *c; ++c) h = mix(h ^ static_cast<uint64_t>(static_cast<unsigned char>(*c)));
        *out = new qbg_rng(h);
    });
}
int qbg_rng_split_salt(const qbg_rng* r, uint64_t salt, qbg_rng** out) {
    return guarded([&] { *out = new qbg_rng(mix(r->state ^ salt)); });
}
double qbg_rng_uniform(qbg_rng* r) { return std::uniform_real_distribution<double>(0.0, 1.0)(r->eng); }
double qbg_rng_uniform_range(qbg_rng* r, double lo, double hi) {
    return std::uniform_real_distribution<double>(lo, hi)(r->eng);
}
double qbg_rng_gauss(qbg_rng* r) { return std::normal_distribution<double>(0.0, 1.0)(r->eng); }
uint64_t qbg_rng_bits(qbg_rng* r) { return r->eng(); }

// ---- registers ----------------------------------------------------------------------------------
int qbg_reg_create(int32_t nqubits, int64_t nbatch, int32_t dtype, uint64_t seed, qbg_reg** out) {
    return guarded([&] {
        qbg_reg* r = new_reg(nqubits, nbatch, dtype);
        r->rng = qbg_rng(seed);
        QBG_CUDA(cudaMemsetAsync(r->s.ptr, 0, r->s.bytes(), g_stream));
        *out = r;
    });
}
int qbg_reg_destroy(qbg_reg* r) {
    return guarded([&] {
        if (!r) return;
        if (r->s.ptr) {
            QBG_CUDA(cudaStreamSynchronize(g_stream));
            QBG_CUDA(cudaFree(r->s.ptr));
        }
        std::lock_guard<std::mutex> lk(g_ws_mu);
        g_live.erase(std::remove(g_live.begin(), g_live.end(), r), g_live.end());
        delete r;
        // release workspace no live register can use any more (an expect' of a large register
        // must not keep two of its states resident after the register is gone)
        size_t need = 0;
        for (auto* x : g_live) need = std::max(need, x->s.bytes());
        for (auto& w : g_ws)
            if (w.ptr && w.bytes() > need) ws_free(w);
        if (g_ckpt.ptr && g_ckpt.state_bytes > need) ckpt_free();
        release_krylov(need);
    });
}
int qbg_release_workspace(void) {
    return guarded([&] {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        for (auto& w : g_ws) ws_free(w);
        ckpt_free();
        release_krylov(0);
        release_scratch();
    });
}
int qbg_reg_clone(const qbg_reg* src, qbg_reg** out) {
    return guarded([&] {
        check_reg(src);
        qbg_reg* r = new_reg(src->s.n, src->s.B, src->s.dtype);
        r->nactive = src->nactive;
        r->rng = src->rng;
        r->focus_stack = src->focus_stack;
        QBG_CUDA(cudaMemcpyAsync(r->s.ptr, src->s.ptr, src->s.bytes(), cudaMemcpyDeviceToDevice, g_stream));
        *out = r;
    });
}
int qbg_reg_copy(qbg_reg* dst, const qbg_reg* src) {
    return guarded([&] {
        same_shape(dst, src, "Register::operator=");
        if (dst == src) return;
        dst->nactive = src->nactive;
        dst->rng = src->rng;
        dst->focus_stack = src->focus_stack;
        QBG_CUDA(cudaMemcpyAsync(dst->s.ptr, src->s.ptr, src->s.bytes(), cudaMemcpyDeviceToDevice, g_stream));
    });
}
int qbg_reg_info(const qbg_reg* r, int32_t* nq, int32_t* na, int64_t* nb, int32_t* dt) {
    return guarded([&] {
        check_reg(r);
        if (nq) *nq = r->s.n;
        if (na) *na = r->nactive;
        if (nb) *nb = r->s.B;
        if (dt) *dt = r->s.dtype;
    });
}
void* qbg_reg_device_ptr(qbg_reg* r) { return r ? r->s.ptr : nullptr; }
qbg_rng* qbg_reg_rng(qbg_reg* r) { return r ? &r->rng : nullptr; }

int qbg_set_zero(qbg_reg* r) {
    uint64_t z = 0;
    return qbg_set_product(r, &z, 1);
}
int qbg_set_product(qbg_reg* r, const uint64_t* bits, int64_t nbits) {
    return guarded([&] {
        check_reg(r);
        if (nbits != 1 && nbits != r->s.B) raise(QBG_ERR_SHAPE, "product_state: one basis index per batch");
        for (int64_t k = 0; k < nbits; ++k)
            if (bits[k] >> r->s.n) raise(QBG_ERR_VALIDATION, "BitStr value does not fit in the register");
        uint64_t* d = static_cast<uint64_t*>(scratch(nbits * sizeof(uint64_t), 5));
        QBG_CUDA(cudaMemcpyAsync(d, bits, nbits * sizeof(uint64_t), cudaMemcpyHostToDevice, g_stream));
        launch_set_basis(r->s, d, nbits);
    });
}
int qbg_set_rand(qbg_reg* r, uint64_t seed) {
    return guarded([&] {
        check_reg(r);
        // rand_state, register.hpp:266-280: host Gaussians from Rng(seed).split("rand_state")
        qbg_rng root(seed);
        uint64_t h = root.state;
        for (const char* c = "rand_state"; *c; ++c) h = mix(h ^ static_cast<uint64_t>(static_cast<unsigned char>(*c)));
        qbg_rng g(h);
        uint64_t len = r->s.rows();
        std::vector<std::complex<double>> host(len * r->s.B);
        for (int64_t b = 0; b < r->s.B; ++b) {
            auto* sl = host.data() + b * len;
            double nrm2 = 0.0;
            for (uint64_t i = 0; i < len; ++i) {
                double im = std::normal_distribution<double>(0.0, 1.0)(g.eng);  // g++ evaluates right to left
                double re = std::normal_distribution<double>(0.0, 1.0)(g.eng);
                sl[i] = std::complex<double>(re, im);
                nrm2 += std::norm(sl[i]);
            }
            double inv = 1.0 / std::sqrt(nrm2);
            for (uint64_t i = 0; i < len; ++i) sl[i] *= inv;
        }
        int rc = qbg_upload(r, reinterpret_cast<const double*>(host.data()), static_cast<int64_t>(host.size()));
        if (rc) raise(rc, g_err);
        stream_sync();
    });
}

int qbg_upload(qbg_reg* r, const double* host, int64_t n) {
    return guarded([&] {
        check_reg(r);
        if (static_cast<uint64_t>(n) != r->s.count()) raise(QBG_ERR_SHAPE, "upload: element count mismatch");
        if (r->s.dtype == QBG_C64) {
            std::vector<float> f(2 * n);
            for (int64_t k = 0; k < 2 * n; ++k) f[k] = static_cast<float>(host[k]);
            if (r->s.B == 1) {
                QBG_CUDA(cudaMemcpyAsync(r->s.ptr, f.data(), r->s.bytes(), cudaMemcpyHostToDevice, g_stream));
            } else {
                void* tmp = scratch(r->s.bytes(), 6);
                QBG_CUDA(cudaMemcpyAsync(tmp, f.data(), r->s.bytes(), cudaMemcpyHostToDevice, g_stream));
                launch_transpose(tmp, r->s.ptr, r->s.rows(), r->s.B, r->s.dtype, true);
            }
            stream_sync();
            return;
        }
        if (r->s.B == 1) {
            QBG_CUDA(cudaMemcpyAsync(r->s.ptr, host, r->s.bytes(), cudaMemcpyHostToDevice, g_stream));
        } else {
            void* tmp = scratch(r->s.bytes(), 6);
            QBG_CUDA(cudaMemcpyAsync(tmp, host, r->s.bytes(), cudaMemcpyHostToDevice, g_stream));
            launch_transpose(tmp, r->s.ptr, r->s.rows(), r->s.B, r->s.dtype, true);
        }
    });
}
int qbg_download(const qbg_reg* r, double* host, int64_t n) {
    return guarded([&] {
        check_reg(r);
        if (static_cast<uint64_t>(n) != r->s.count()) raise(QBG_ERR_SHAPE, "download: element count mismatch");
        const void* src = r->s.ptr;
        if (r->s.B != 1) {
            void* tmp = scratch(r->s.bytes(), 6);
            launch_transpose(r->s.ptr, tmp, r->s.rows(), r->s.B, r->s.dtype, false);
            src = tmp;
        }
        if (r->s.dtype == QBG_C64) {
            std::vector<float> f(2 * n);
            QBG_CUDA(cudaMemcpyAsync(f.data(), src, r->s.bytes(), cudaMemcpyDeviceToHost, g_stream));
            stream_sync();
            for (int64_t k = 0; k < 2 * n; ++k) host[k] = f[k];
            return;
        }
        QBG_CUDA(cudaMemcpyAsync(host, src, r->s.bytes(), cudaMemcpyDeviceToHost, g_stream));
        stream_sync();
    });
}
int qbg_upload_raw(qbg_reg* r, const void* host, int64_t nbytes) {
    return guarded([&] {
        check_reg(r);
        if (static_cast<size_t>(nbytes) != r->s.bytes()) raise(QBG_ERR_SHAPE, "upload_raw: byte count mismatch");
        QBG_CUDA(cudaMemcpyAsync(r->s.ptr, host, nbytes, cudaMemcpyHostToDevice, g_stream));
    });
}
int qbg_download_raw(const qbg_reg* r, void* host, int64_t nbytes) {
    return guarded([&] {
        check_reg(r);
        if (static_cast<size_t>(nbytes) != r->s.bytes()) raise(QBG_ERR_SHAPE, "download_raw: byte count mismatch");
        QBG_CUDA(cudaMemcpyAsync(host, r->s.ptr, nbytes, cudaMemcpyDeviceToHost, g_stream));
        stream_sync();
    });
}

// ---- instruct -------------------------------------------------------------------------------------
int qbg_instruct(qbg_reg* r, const qbg_matrix* gate, const int32_t* locs, int32_t nloc, const int32_t* ctrl_locs,
                 const int32_t* ctrl_cfg, int32_t nctrl) {
    return guarded([&] {
        check_reg(r);
        qbg_op op{};
        op.kind = gate->kind;
        op.ntarget = nloc;
        op.nctrl = nctrl;
        op.dim = gate->dim;
        if (nloc < 1) raise(QBG_ERR_VALIDATION, "instruct: need at least one target qubit");
        if (nloc > QBG_MAX_TARGETS) raise(QBG_ERR_UNSUPPORTED, "instruct: more than 5 targets");
        if (nctrl > QBG_MAX_CTRLS) raise(QBG_ERR_UNSUPPORTED, "instruct: too many controls");
        for (int k = 0; k < nloc; ++k) op.targets[k] = locs[k];
        for (int k = 0; k < nctrl; ++k) {
            op.ctrls[k] = ctrl_locs[k];
            op.ctrl_cfg[k] = ctrl_cfg[k];
        }
        validate_op(r->nactive, op);
        std::vector<cdbl> m;
        std::vector<int> perm;
        int d = gate->dim;
        const cdbl* v = reinterpret_cast<const cdbl*>(gate->vals);
        if (gate->kind == QBG_MAT_IDENTITY) return;
        if (gate->kind == QBG_MAT_DIAGONAL || gate->kind == QBG_MAT_PERMUTATION) m.assign(v, v + d);
        else if (gate->kind == QBG_MAT_DENSE) m.assign(v, v + static_cast<size_t>(d) * d);
        else raise(QBG_ERR_VALIDATION, "instruct: unknown matrix class");
        if (gate->kind == QBG_MAT_PERMUTATION) {
            std::vector<char> seen(d, 0);
            for (int k = 0; k < d; ++k) {
                if (gate->perm[k] < 0 || gate->perm[k] >= d || seen[gate->perm[k]])
                    raise(QBG_ERR_VALIDATION, "Permutation: column indices must form a permutation");
                seen[gate->perm[k]] = 1;
                perm.push_back(static_cast<int>(gate->perm[k]));
            }
        }
        launch_gate(r->s, place_gate(op, gate->kind, d, m, perm));
    });
}

int qbg_instruct_tag(qbg_reg* r, const char* tag, const int32_t* locs, int32_t nloc, const int32_t* ctrl_locs,
                     const int32_t* ctrl_cfg, int32_t nctrl, const double* params, int32_t nparams) {
    return guarded([&] {
        HostGate hg = gate_by_tag(tag, params, nparams);
        std::vector<int64_t> perm(hg.perm.begin(), hg.perm.end());
        qbg_matrix m{hg.kind, hg.dim, reinterpret_cast<const double*>(hg.v.data()), perm.data()};
        int rc = qbg_instruct(r, &m, locs, nloc, ctrl_locs, ctrl_cfg, nctrl);
        if (rc) raise(rc, g_err);
    });
}

// ---- algebra -------------------------------------------------------------------------------------
int qbg_norm(const qbg_reg* r, double* out) {
    return guarded([&] {
        check_reg(r);
        double* d = static_cast<double*>(scratch(2 * r->s.B * sizeof(double), 2));
        reduce_inner(r->s, nullptr, d);
        std::vector<double> h(2 * r->s.B);
        QBG_CUDA(cudaMemcpyAsync(h.data(), d, h.size() * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        stream_sync();
        for (int64_t b = 0; b < r->s.B; ++b) out[b] = std::sqrt(h[2 * b]);
    });
}
int qbg_inner(const qbg_reg* a, const qbg_reg* b, double* out) {
    return guarded([&] {
        same_shape(a, b, "Register::inner");
        double* d = static_cast<double*>(scratch(2 * a->s.B * sizeof(double), 2));
        reduce_inner(a->s, &b->s, d);
        QBG_CUDA(cudaMemcpyAsync(out, d, 2 * a->s.B * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        stream_sync();
    });
}
int qbg_scale(qbg_reg* r, double re, double im) {
    return guarded([&] {
        check_reg(r);
        launch_scale(r->s, re, im);
    });
}
int qbg_add_scaled(qbg_reg* r, const qbg_reg* o, double re, double im) {
    return guarded([&] {
        same_shape(r, o, "Register::add_scaled");
        launch_axpy(r->s, o->s, re, im);
    });
}

// ---- measurement (register.hpp:414-493) ----------------------------------------------------------
namespace {
std::vector<double> probs(const qbg_reg* r, int64_t b) {
    uint64_t ra = uint64_t{1} << r->nactive;
    double* d = static_cast<double*>(scratch(ra * sizeof(double), 8));
    launch_probabilities(r->s, r->nactive, b, d);
    std::vector<double> p(ra);
    QBG_CUDA(cudaMemcpyAsync(p.data(), d, ra * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
    stream_sync();
    return p;
}
// the reference's sequential prefix sum (register.hpp:444-449) and upper_bound (428-432)
uint64_t sample(const std::vector<double>& cum, double u) {
    auto it = std::upper_bound(cum.begin(), cum.end(), u * cum.back());
    uint64_t idx = static_cast<uint64_t>(it - cum.begin());
    return idx < cum.size() ? idx : cum.size() - 1;
}
}  // namespace

int qbg_probabilities(const qbg_reg* r, int64_t b, double* out) {
    return guarded([&] {
        check_reg(r);
        if (b < 0 || b >= r->s.B) raise(QBG_ERR_RANGE, "probabilities: batch out of range");
        auto p = probs(r, b);
        std::copy(p.begin(), p.end(), out);
    });
}
int qbg_measure(const qbg_reg* r, int64_t nshots, qbg_rng* rng, uint64_t* out) {
    return guarded([&] {
        check_reg(r);
        if (nshots < 1) raise(QBG_ERR_VALIDATION, "measure: nshots must be positive");
        qbg_rng* g = rng ? rng : const_cast<qbg_rng*>(&r->rng);
        for (int64_t b = 0; b < r->s.B; ++b) {
            auto p = probs(r, b);
            std::vector<double> cum(p.size());
            double acc = 0.0;
            for (size_t i = 0; i < p.size(); ++i) {
                acc += p[i];
                cum[i] = acc;
            }
            for (int64_t s = 0; s < nshots; ++s) out[b * nshots + s] = sample(cum, qbg_rng_uniform(g));
        }
    });
}
int qbg_measure_collapse(qbg_reg* r, qbg_rng* rng, uint64_t* out) {
    return guarded([&] {
        check_reg(r);
        qbg_rng* g = rng ? rng : &r->rng;
        for (int64_t b = 0; b < r->s.B; ++b) {
            auto p = probs(r, b);
            std::vector<double> cum(p.size());
            double acc = 0.0;
            for (size_t i = 0; i < p.size(); ++i) {
                acc += p[i];
                cum[i] = acc;
            }
            uint64_t hit = sample(cum, qbg_rng_uniform(g));
            double prob = p[hit];
            if (prob <= 1e-300)
                raise(QBG_ERR_RENORMALIZATION, "measure!: outcome has numerically zero probability");
            launch_collapse(r->s, r->nactive, b, hit, 1.0 / std::sqrt(prob));
            out[b] = hit;
        }
        stream_sync();
    });
}

// ---- focus / relax (register.hpp:156-177, 209-248) ----------------------------------------------------
namespace {
std::vector<int> focus_src(const qbg_reg* r, const int32_t* locs, int32_t nloc) {
    if (nloc < 1) raise(QBG_ERR_VALIDATION, "focus: need at least one location");
    std::vector<char> used(r->s.n, 0);
    std::vector<int> src;
    for (int k = 0; k < nloc; ++k) {
        if (locs[k] < 1 || locs[k] > r->s.n) raise(QBG_ERR_RANGE, "focus: location out of range");
        if (used[locs[k] - 1]) raise(QBG_ERR_VALIDATION, "focus: duplicate location");
        used[locs[k] - 1] = 1;
        src.push_back(locs[k] - 1);
    }
    for (int q = 0; q < r->s.n; ++q)
        if (!used[q]) src.push_back(q);
    return src;
}
// new bit k takes old bit src[k]; launch with new_of_old[src[k]] = k
void permute(qbg_reg* r, const std::vector<int>& src) {
    bool ident = true;
    for (size_t k = 0; k < src.size(); ++k) ident &= src[k] == static_cast<int>(k);
    if (ident) return;
    std::vector<int> new_of_old(src.size());
    for (size_t k = 0; k < src.size(); ++k) new_of_old[src[k]] = static_cast<int>(k);
    DevState tmp = r->s;
    tmp.ptr = scratch(r->s.bytes(), 6);
    launch_permute_bits(r->s, tmp, new_of_old.data());
    QBG_CUDA(cudaMemcpyAsync(r->s.ptr, tmp.ptr, r->s.bytes(), cudaMemcpyDeviceToDevice, g_stream));
}
}  // namespace

int qbg_focus(qbg_reg* r, const int32_t* locs, int32_t nloc) {
    return guarded([&] {
        check_reg(r);
        auto src = focus_src(r, locs, nloc);
        permute(r, src);
        r->focus_stack.emplace_back(locs, locs + nloc);
        r->nactive = nloc;
    });
}
int qbg_relax(qbg_reg* r, const int32_t* locs, int32_t nloc, int32_t to_nactive) {
    return guarded([&] {
        check_reg(r);
        if (r->focus_stack.empty()) raise(QBG_ERR_VALIDATION, "relax: no focus to undo");
        const auto& top = r->focus_stack.back();
        if (!std::equal(top.begin(), top.end(), locs, locs + nloc))
            raise(QBG_ERR_VALIDATION, "relax: locations do not match the previous focus");
        if (to_nactive > r->s.n) raise(QBG_ERR_VALIDATION, "relax: to_nactive exceeds qubit count");
        auto src = focus_src(r, locs, nloc);
        std::vector<int> inv(src.size());
        for (size_t k = 0; k < src.size(); ++k) inv[src[k]] = static_cast<int>(k);
        permute(r, inv);
        r->focus_stack.pop_back();
        r->nactive = to_nactive;
    });
}

// ---- sharded states: sub-block pack / unpack and staging buffers ---------------
int qbg_shard_pack(const qbg_reg* r, const int32_t* fix_locs, int32_t nfix, uint64_t fix_val, int64_t row0,
                   int64_t nrows, void* dst) {
    return guarded([&] {
        check_reg(r);
        if (nfix > 0 && !fix_locs) raise(QBG_ERR_VALIDATION, "shard pack: null locations");
        int pos[8];
        for (int i = 0; i < nfix && i < 8; ++i) pos[i] = fix_locs[i] - 1;
        if (row0 < 0 || nrows < 0) raise(QBG_ERR_RANGE, "shard pack: negative row range");
        launch_shard_copy(r->s, true, pos, nfix, fix_val, static_cast<uint64_t>(row0), static_cast<uint64_t>(nrows), dst);
    });
}
int qbg_shard_unpack(qbg_reg* r, const int32_t* fix_locs, int32_t nfix, uint64_t fix_val, int64_t row0, int64_t nrows,
                     const void* src) {
    return guarded([&] {
        check_reg(r);
        if (nfix > 0 && !fix_locs) raise(QBG_ERR_VALIDATION, "shard unpack: null locations");
        int pos[8];
        for (int i = 0; i < nfix && i < 8; ++i) pos[i] = fix_locs[i] - 1;
        if (row0 < 0 || nrows < 0) raise(QBG_ERR_RANGE, "shard unpack: negative row range");
        launch_shard_copy(r->s, false, pos, nfix, fix_val, static_cast<uint64_t>(row0), static_cast<uint64_t>(nrows),
                          const_cast<void*>(src));
    });
}
int qbg_buffer_alloc(int64_t bytes, void** out) {
    return guarded([&] {
        if (bytes <= 0 || !out) raise(QBG_ERR_VALIDATION, "buffer: size must be positive");
        *out = dev_alloc(static_cast<size_t>(bytes), false);
    });
}
int qbg_buffer_free(void* p) {
    return guarded([&] {
        if (!p) return;
        QBG_CUDA(cudaStreamSynchronize(g_stream));
        QBG_CUDA(cudaFree(p));
    });
}

// ---- state files (register.hpp:181-205) -------------------------------------------------------------
int qbg_save(const qbg_reg* r, const char* path) {
    return guarded([&] {
        check_reg(r);
        std::vector<double> host(2 * r->s.count());
        int rc = qbg_download(r, host.data(), static_cast<int64_t>(r->s.count()));
        if (rc) raise(rc, g_err);
        FILE* f = std::fopen(path, "wb");
        if (!f) raise(QBG_ERR_SERIALIZATION, std::string("state file: cannot open ") + path);
        const char magic[8] = {'Q', 'B', 'R', 'E', 'G', '1', 0, 0};
        uint64_t hdr[3] = {static_cast<uint64_t>(r->s.n), static_cast<uint64_t>(r->nactive),
                           static_cast<uint64_t>(r->s.B)};
        bool ok = std::fwrite(magic, 1, 8, f) == 8 && std::fwrite(hdr, 8, 3, f) == 3 &&
                  std::fwrite(host.data(), sizeof(double), host.size(), f) == host.size();
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) raise(QBG_ERR_SERIALIZATION, "state file: write failed");
    });
}

int qbg_load_memory(const void* data, int64_t nbytes, uint64_t seed, int32_t dtype, qbg_reg** out) {
    return guarded([&] {
        const char* p = static_cast<const char*>(data);
        if (!p || nbytes < 8 || std::memcmp(p, "QBREG1\0\0", 8) != 0) raise(QBG_ERR_SERIALIZATION, "state file: bad magic");
        uint64_t hdr[3];
        if (nbytes < 32) raise(QBG_ERR_SERIALIZATION, "state file: bad header");
        std::memcpy(hdr, p + 8, sizeof(hdr));
        if (hdr[0] < 1 || hdr[1] > hdr[0] || hdr[0] > 62 || hdr[2] < 1) raise(QBG_ERR_SERIALIZATION, "state file: bad header");
        const uint64_t count = (uint64_t{1} << hdr[0]) * hdr[2];
        if (static_cast<uint64_t>(nbytes) - 32 < 16 * count) raise(QBG_ERR_SERIALIZATION, "state file: truncated amplitudes");
        qbg_reg* r = nullptr;
        int rc = qbg_reg_create(static_cast<int32_t>(hdr[0]), static_cast<int64_t>(hdr[2]), dtype, seed, &r);
        if (rc) raise(rc, g_err);
        std::vector<double> host(2 * count);  // aligned copy of the amplitudes
        std::memcpy(host.data(), p + 32, 16 * count);
        rc = qbg_upload(r, host.data(), static_cast<int64_t>(count));
        if (rc) {
            qbg_reg_destroy(r);
            raise(rc, g_err);
        }
        r->nactive = static_cast<int>(hdr[1]);
        stream_sync();
        *out = r;
    });
}

int qbg_load(const char* path, uint64_t seed, int32_t dtype, qbg_reg** out) {
    std::vector<char> buf;
    int rc = guarded([&] {
        FILE* f = std::fopen(path, "rb");
        if (!f) raise(QBG_ERR_SERIALIZATION, std::string("state file: cannot open ") + path);
        char chunk[1 << 16];
        size_t got;
        while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) buf.insert(buf.end(), chunk, chunk + got);
        std::fclose(f);
    });
    if (rc) return rc;
    return qbg_load_memory(buf.data(), static_cast<int64_t>(buf.size()), seed, dtype, out);
}

// ---- programs -----------------------------------------------------------------------------------------
int qbg_prog_create(int32_t n, const qbg_op* ops, int64_t nops, const double* vals, int64_t nvals,
                    const int64_t* perms, int64_t nperms, qbg_prog** out) {
    return guarded([&] {
        if (n < 1 || n > 62) raise(QBG_ERR_VALIDATION, "program: qubit count out of range");
        auto* p = new qbg_prog;
        try {
            p->p.n = n;
            p->p.ops.assign(ops, ops + nops);
            const cdbl* v = reinterpret_cast<const cdbl*>(vals);
            p->p.vals.assign(v, v + nvals);
            p->p.perms.assign(perms, perms + nperms);
            int64_t np = 0;
            for (auto& op : p->p.ops) {
                validate_op(n, op);
                if (op.gen != QBG_GEN_NONE) {
                    if (op.param < 0) raise(QBG_ERR_VALIDATION, "program: parameterised op without a slot");
                    np = std::max<int64_t>(np, op.param + 1);
                    if (op.gen == QBG_GEN_SHIFT && op.dim != 2) raise(QBG_ERR_SHAPE, "shift acts on one qubit");
                }
                int64_t need = op.kind == QBG_MAT_DENSE ? int64_t{op.dim} * op.dim
                               : (op.kind == QBG_MAT_IDENTITY || op.gen == QBG_GEN_SHIFT || op.gen == QBG_GEN_PHASE)
                                   ? 0
                                   : op.dim;
                if (need && (op.data < 0 || op.data + need > nvals)) raise(QBG_ERR_SHAPE, "program: payload out of range");
                if (op.kind == QBG_MAT_PERMUTATION && op.gen != QBG_GEN_SHIFT && op.gen != QBG_GEN_PHASE) {
                    if (op.perm < 0 || op.perm + op.dim > nperms) raise(QBG_ERR_SHAPE, "program: permutation out of range");
                    std::vector<char> seen(op.dim, 0);
                    for (int k = 0; k < op.dim; ++k) {
                        int64_t c = perms[op.perm + k];
                        if (c < 0 || c >= op.dim || seen[c])
                            raise(QBG_ERR_VALIDATION, "Permutation: column indices must form a permutation");
                        seen[c] = 1;
                    }
                }
            }
            p->p.nparams = np;
            p->p.theta.assign(np, 0.0);
            realise(p->p);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}
int qbg_prog_destroy(qbg_prog* p) {
    delete p;
    return QBG_OK;
}
int64_t qbg_prog_nparams(const qbg_prog* p) { return p ? p->p.nparams : -1; }
int qbg_prog_set_params(qbg_prog* p, const double* theta, int64_t n) {
    return guarded([&] {
        if (n != p->p.nparams) raise(QBG_ERR_VALIDATION, "dispatch: parameter count mismatch");
        p->p.theta.assign(theta, theta + n);
        static const bool fast = [] {
            const char* e = std::getenv("QBG_REALISE_FULL");  // diagnostics: always rebuild every op
            return !(e && e[0] == '1');
        }();
        if (fast && p->p.realised && p->p.real.size() == p->p.ops.size())
            realise_params(p->p);
        else
            realise(p->p);
        p->p.version++;
    });
}
int qbg_prog_stats(const qbg_prog* prog, int64_t* fwd, int64_t* bwd, int64_t* gates) {
    return guarded([&] {
        int64_t f = 0, b = 0;
        fused_stats(prog->p, &f, &b);
        if (fwd) *fwd = f;
        if (bwd) *bwd = b;
        if (gates) *gates = static_cast<int64_t>(prog->p.ops.size());
    });
}
int qbg_prog_plan_info(const qbg_prog* prog, char* buf, int64_t cap) {
    return guarded([&] {
        std::string s = fused_plan_info(prog->p);
        if (cap > 0) {
            std::strncpy(buf, s.c_str(), static_cast<size_t>(cap - 1));
            buf[cap - 1] = 0;
        }
    });
}
int qbg_prog_plan_preview(const qbg_prog* prog, int64_t nbatch, int32_t dtype, char* buf, int64_t cap) {
    return guarded([&] {
        std::string s = fused_plan_preview(prog->p, nbatch, dtype);
        if (cap > 0) {
            std::strncpy(buf, s.c_str(), static_cast<size_t>(cap - 1));
            buf[cap - 1] = 0;
        }
    });
}
int qbg_jit_check(const qbg_prog* prog, const qbg_obs* obs, int64_t nbatch, int32_t dtype, int64_t* nkernels) {
    return guarded([&] {
        int64_t n = fused_jit_check(prog->p, obs ? &obs->o : nullptr, nbatch, dtype);
        if (nkernels) *nkernels = n;
    });
}
int qbg_jit_stats(int64_t* nvrtc_builds, int64_t* cache_hits) {
    return guarded([&] { jit::stats(nvrtc_builds, cache_hits); });
}
int qbg_apply(qbg_reg* r, const qbg_prog* prog) {
    return guarded([&] {
        check_reg(r);
        if (prog->p.n != r->nactive) raise(QBG_ERR_SHAPE, "apply: block qubit count differs from active qubits");
        run_program(r->s, const_cast<qbg_prog*>(prog)->p, false);
    });
}
int qbg_apply_adjoint(qbg_reg* r, const qbg_prog* prog) {
    return guarded([&] {
        check_reg(r);
        if (prog->p.n != r->nactive) raise(QBG_ERR_SHAPE, "apply: block qubit count differs from active qubits");
        run_program(r->s, const_cast<qbg_prog*>(prog)->p, true);
    });
}

// ---- observables / AD ---------------------------------------------------------------------------------
int qbg_obs_create(int32_t n, const qbg_pauli_term* terms, int64_t nterms, qbg_obs** out) {
    return guarded([&] {
        auto* o = new qbg_obs;
        o->o.n = n;
        uint64_t full = n >= 64 ? ~uint64_t{0} : (uint64_t{1} << n) - 1;
        for (int64_t t = 0; t < nterms; ++t) {
            qbg_pauli_term q = terms[t];
            if ((q.xmask | q.zmask) & ~full) {
                delete o;
                raise(QBG_ERR_RANGE, "observable: Pauli factor outside the register");
            }
            // fold i^{nY} (Y = i X Z) into the coefficient exactly
            int ny = __builtin_popcountll(q.xmask & q.zmask) & 3;
            double re = q.coef_re, im = q.coef_im;
            for (int k = 0; k < ny; ++k) {
                double t2 = re;
                re = -im;
                im = t2;
            }
            q.coef_re = re;
            q.coef_im = im;
            o->o.terms.push_back(q);
        }
        *out = o;
    });
}
int qbg_obs_destroy(qbg_obs* o) {
    delete o;
    return QBG_OK;
}
int qbg_obs_apply(const qbg_reg* r, const qbg_obs* o, qbg_reg* out) {
    return guarded([&] {
        same_shape(r, out, "obs_apply");
        if (o->o.n != r->nactive) raise(QBG_ERR_SHAPE, "observable qubit count differs from active qubits");
        run_obs(r->s, out->s, const_cast<qbg_obs*>(o)->o, nullptr);
    });
}
int qbg_expect(const qbg_reg* r, const qbg_obs* o, double* out) {
    return guarded([&] {
        check_reg(r);
        if (o->o.n != r->nactive) raise(QBG_ERR_SHAPE, "observable qubit count differs from active qubits");
        double* e = static_cast<double*>(scratch(r->s.B * sizeof(double), 10));
        // energy-only fused seed: no second full state (a 33-qubit register is 128 GiB)
        DevState none = r->s;
        none.ptr = nullptr;
        if (!(g_fusion && fused_obs_apply(r->s, none, const_cast<qbg_obs*>(o)->o, e))) {
            DevState phi = r->s;
            phi.ptr = scratch(r->s.bytes(), 9);
            run_obs(r->s, phi, const_cast<qbg_obs*>(o)->o, e);
        }
        QBG_CUDA(cudaMemcpyAsync(out, e, r->s.B * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        stream_sync();
    });
}
int qbg_backward(qbg_reg* psi, qbg_reg* adj, const qbg_prog* prog, double* grads) {
    return guarded([&] {
        same_shape(psi, adj, "backward");
        auto& p = const_cast<qbg_prog*>(prog)->p;
        if (p.n != psi->nactive) raise(QBG_ERR_SHAPE, "backward: block qubit count differs from active qubits");
        double* dg = static_cast<double*>(scratch(std::max<int64_t>(1, p.nparams) * sizeof(double), 11));
        QBG_CUDA(cudaMemcpyAsync(dg, grads, p.nparams * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        run_backward(psi->s, adj->s, p, dg);
        QBG_CUDA(cudaMemcpyAsync(grads, dg, p.nparams * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        stream_sync();
    });
}
}  // extern "C"

namespace qbg {
namespace {
// forward → seed → reverse pass with at most two extra live full states;
// seed(psi_out, adj, d_vals) writes the adjoint seed and the per-batch loss values.
template <class Seed>
void grad_driver(qbg_reg* r, Program& p, int32_t inplace, qbg_reg* state_grad, double* vals, double* grads,
                 Seed&& seed) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    DevState adj = r->s;
    adj.ptr = state_grad ? state_grad->s.ptr : ws_get(1, r->s).ptr;
    if (!p.realised) realise(p);
    // checkpointed design (default when the checkpoints fit): the forward passes leave the state
    // after every reverse segment in an arena, the reverse passes read ψ instead of uncomputing it;
    // the caller's register is not modified (in place or not, it ends as it started)
    if (g_fusion) {
        int64_t k = fused_ckpt_states(p, r->s);
        void* arena = k > 0 ? ckpt_get(k, r->s) : nullptr;
        if (arena && !(fused_ckpt_forward(r->s, p, arena, k) && fused_ckpt_sync(p, r->s, k))) {
            // the program's structure changed with θ: the plans are rebuilt, run the forward again
            k = fused_ckpt_states(p, r->s);
            arena = k > 0 ? ckpt_get(k, r->s) : nullptr;
            if (arena && !(fused_ckpt_forward(r->s, p, arena, k) && fused_ckpt_sync(p, r->s, k)))
                raise(QBG_ERR_INTERNAL, "expect': checkpointed plans inconsistent after a rebuild");
        }
        if (arena) {
            Nvtx nv("qbg.expect_grad.checkpointed");
            DevState psi = r->s;
            psi.ptr = arena;  // checkpoint 0: the output state
            double* e = static_cast<double*>(scratch(r->s.B * sizeof(double), 10));
            seed(psi, adj, e);
            double* dg = static_cast<double*>(scratch(std::max<int64_t>(1, p.nparams) * sizeof(double), 11));
            QBG_CUDA(cudaMemsetAsync(dg, 0, std::max<int64_t>(1, p.nparams) * sizeof(double), g_stream));
            fused_ckpt_backward(adj, p, arena, dg);
            QBG_CUDA(cudaMemcpyAsync(vals, e, r->s.B * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
            QBG_CUDA(cudaMemcpyAsync(grads, dg, p.nparams * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
            stream_sync();
            return;
        }
    }
    DevState psi = r->s;
    if (!inplace) psi.ptr = ws_get(0, r->s).ptr;
    // out-of-place: the first forward pass reads the caller's register (no separate copy)
    run_program(psi, p, false, inplace ? nullptr : r->s.ptr);
    double* e = static_cast<double*>(scratch(r->s.B * sizeof(double), 10));
    seed(psi, adj, e);
    double* dg = static_cast<double*>(scratch(std::max<int64_t>(1, p.nparams) * sizeof(double), 11));
    QBG_CUDA(cudaMemsetAsync(dg, 0, std::max<int64_t>(1, p.nparams) * sizeof(double), g_stream));
    run_backward(psi, adj, p, dg);
    QBG_CUDA(cudaMemcpyAsync(vals, e, r->s.B * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
    QBG_CUDA(cudaMemcpyAsync(grads, dg, p.nparams * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
    stream_sync();
}
}  // namespace
}  // namespace qbg

struct qbg_mmd {
    int n = 0;
    int D = 0;
    double* q = nullptr;  // device, 2^n
    double* w = nullptr;  // device, D + 1 taps
    std::vector<double> sigmas;
};

extern "C" {

int qbg_expect_grad(qbg_reg* r, const qbg_prog* prog, const qbg_obs* o, int32_t inplace, double* energies,
                    double* grads, qbg_reg* state_grad) {
    return guarded([&] {
        check_reg(r);
        auto& p = const_cast<qbg_prog*>(prog)->p;
        auto& ob = const_cast<qbg_obs*>(o)->o;
        if (p.n != r->nactive || ob.n != r->nactive)
            raise(QBG_ERR_SHAPE, "expect': block qubit count differs from active qubits");
        if (state_grad) same_shape(r, state_grad, "expect' state_grad");
        grad_driver(r, p, inplace, state_grad, energies, grads,
                    [&](const DevState& psi, const DevState& adj, double* e) { run_obs(psi, adj, ob, e); });
    });
}

int qbg_run_program(qbg_reg* reg, const qbg_op* ops, int64_t nops, const double* vals, int64_t nvals,
                    const int64_t* perms, int64_t nperms, const double* theta, int64_t nparams) {
    qbg_prog* p = nullptr;
    int rc = qbg_prog_create(reg ? reg->nactive : 0, ops, nops, vals, nvals, perms, nperms, &p);
    if (rc) return rc;
    if (nparams > 0) rc = qbg_prog_set_params(p, theta, nparams);
    if (!rc) rc = qbg_apply(reg, p);
    const std::string err = g_err;
    qbg_prog_destroy(p);
    if (rc) g_err = err;
    return rc;
}

int qbg_expect_pauli_sum(const qbg_reg* reg, const qbg_pauli_term* terms, int64_t nterms, double* out) {
    qbg_obs* o = nullptr;
    int rc = qbg_obs_create(reg ? reg->nactive : 0, terms, nterms, &o);
    if (rc) return rc;
    rc = qbg_expect(reg, o, out);
    const std::string err = g_err;
    qbg_obs_destroy(o);
    if (rc) g_err = err;
    return rc;
}

int qbg_axpy(qbg_reg* y, const qbg_reg* x, double re, double im) { return qbg_add_scaled(y, x, re, im); }

int qbg_collapse(qbg_reg* reg, qbg_rng* rng, uint64_t* out) { return qbg_measure_collapse(reg, rng, out); }

int qbg_mmd_create(int32_t n, const double* target_p, const double* sigmas, int32_t nsigma, qbg_mmd** out) {
    return guarded([&] {
        ensure_device();
        if (!out || !target_p || !sigmas) raise(QBG_ERR_VALIDATION, "mmd: null argument");
        if (n < 1 || n > g_cap.load()) raise(QBG_ERR_RANGE, "mmd: qubit count out of range");
        if (nsigma < 1) raise(QBG_ERR_VALIDATION, "mmd: the kernel needs at least one bandwidth");
        const uint64_t rows = uint64_t{1} << n;
        double sum = 0.0;
        for (uint64_t x = 0; x < rows; ++x) {
            if (!(target_p[x] >= 0.0) || !std::isfinite(target_p[x]))
                raise(QBG_ERR_VALIDATION, "mmd: target_p must be finite and non-negative");
            sum += target_p[x];
        }
        if (std::fabs(sum - 1.0) > 1e-12) raise(QBG_ERR_VALIDATION, "mmd: target_p must sum to 1 within 1e-12");
        double smax = 0.0;
        for (int i = 0; i < nsigma; ++i) {
            if (!(sigmas[i] > 0.0) || !std::isfinite(sigmas[i])) raise(QBG_ERR_VALIDATION, "mmd: sigma must be > 0");
            smax = std::max(smax, sigmas[i]);
        }
        // taps: w[k] = sum_s exp(-k^2 / (2 s^2)); the band ends where every tap underflows to 0
        std::vector<double> w;
        for (uint64_t k = 0; k < rows; ++k) {
            double t = 0.0;
            for (int i = 0; i < nsigma; ++i) t += std::exp(-static_cast<double>(k) * static_cast<double>(k) /
                                                           (2.0 * sigmas[i] * sigmas[i]));
            if (t == 0.0) break;
            w.push_back(t);
        }
        auto* m = new qbg_mmd;
        m->n = n;
        m->D = static_cast<int>(w.size()) - 1;
        m->sigmas.assign(sigmas, sigmas + nsigma);
        try {
            int TX, BC;
            size_t sm;
            if (!mmd_geometry(rows, 1, m->D, &TX, &BC, &sm))
                raise(QBG_ERR_UNSUPPORTED, "mmd: kernel bandwidth too wide for the banded convolution");
            m->q = static_cast<double*>(dev_alloc(rows * sizeof(double), false));
            m->w = static_cast<double*>(dev_alloc(w.size() * sizeof(double), false));
            QBG_CUDA(cudaMemcpyAsync(m->q, target_p, rows * sizeof(double), cudaMemcpyHostToDevice, g_stream));
            QBG_CUDA(cudaMemcpyAsync(m->w, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice, g_stream));
            stream_sync();
        } catch (...) {
            if (m->q) cudaFree(m->q);
            if (m->w) cudaFree(m->w);
            delete m;
            throw;
        }
        *out = m;
    });
}

int qbg_mmd_destroy(qbg_mmd* m) {
    return guarded([&] {
        if (!m) return;
        stream_sync();
        if (m->q) QBG_CUDA(cudaFree(m->q));
        if (m->w) QBG_CUDA(cudaFree(m->w));
        delete m;
    });
}

int qbg_mmd_band(const qbg_mmd* m, int32_t* band) {
    return guarded([&] {
        if (!m || !band) raise(QBG_ERR_VALIDATION, "mmd: null argument");
        *band = m->D;
    });
}

}  // extern "C"

namespace qbg {
namespace {
void mmd_check(const qbg_reg* r, const qbg_mmd* m) {
    check_reg(r);
    if (!m) raise(QBG_ERR_VALIDATION, "mmd: null loss handle");
    if (r->s.n != m->n || r->nactive != r->s.n)
        raise(QBG_ERR_SHAPE, "mmd: circuit output dimension differs from target_p (register must be relaxed)");
}
void mmd_to_host(double* out, const double* d, int64_t B) {
    QBG_CUDA(cudaMemcpyAsync(out, d, B * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
    stream_sync();
}
}  // namespace
}  // namespace qbg

extern "C" {

int qbg_mmd_loss(const qbg_reg* r, const qbg_mmd* m, double* loss) {
    return guarded([&] {
        mmd_check(r, m);
        double* e = static_cast<double*>(scratch(r->s.B * sizeof(double), 10));
        launch_mmd(0, r->s, nullptr, nullptr, m->q, m->w, m->D, e);
        mmd_to_host(loss, e, r->s.B);
    });
}

int qbg_mmd_seed(const qbg_reg* r, const qbg_mmd* m, qbg_reg* adj, double* loss) {
    return guarded([&] {
        mmd_check(r, m);
        same_shape(r, adj, "mmd seed");
        double* e = static_cast<double*>(scratch(r->s.B * sizeof(double), 10));
        launch_mmd(1, r->s, nullptr, &adj->s, m->q, m->w, m->D, e);
        mmd_to_host(loss, e, r->s.B);
    });
}

int qbg_mmd_cross(const qbg_reg* a, const qbg_reg* r, const qbg_mmd* m, double* out) {
    return guarded([&] {
        mmd_check(r, m);
        same_shape(r, a, "mmd cross");
        double* e = static_cast<double*>(scratch(r->s.B * sizeof(double), 10));
        launch_mmd(2, r->s, &a->s, nullptr, m->q, m->w, m->D, e);
        mmd_to_host(out, e, r->s.B);
    });
}

}  // extern "C"

// ---- time evolution: e^{-iHt}|psi> by Lanczos on the device (matrix.hpp:680-724) --
namespace qbg {
namespace {

// symmetric Jacobi eigen-decomposition of a small dense matrix (row-major, destroyed); Q columns
// are the eigenvectors
void jacobi_eig(int m, std::vector<double>& A, std::vector<double>& Q, std::vector<double>& lam) {
    Q.assign(static_cast<size_t>(m) * m, 0.0);
    for (int i = 0; i < m; ++i) Q[i * m + i] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < m; ++p)
            for (int q = p + 1; q < m; ++q) off += A[p * m + q] * A[p * m + q];
        if (off < 1e-34) break;
        for (int p = 0; p < m; ++p)
            for (int q = p + 1; q < m; ++q) {
                const double apq = A[p * m + q];
                if (std::fabs(apq) < 1e-300) continue;
                const double th = (A[q * m + q] - A[p * m + p]) / (2.0 * apq);
                const double tt = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
                const double c = 1.0 / std::sqrt(tt * tt + 1.0), sn = tt * c;
                for (int k = 0; k < m; ++k) {  // rotate columns p, q
                    const double akp = A[k * m + p], akq = A[k * m + q];
                    A[k * m + p] = c * akp - sn * akq;
                    A[k * m + q] = sn * akp + c * akq;
                }
                for (int k = 0; k < m; ++k) {  // rotate rows p, q
                    const double apk = A[p * m + k], aqk = A[q * m + k];
                    A[p * m + k] = c * apk - sn * aqk;
                    A[q * m + k] = sn * apk + c * aqk;
                }
                for (int k = 0; k < m; ++k) {
                    const double qkp = Q[k * m + p], qkq = Q[k * m + q];
                    Q[k * m + p] = c * qkp - sn * qkq;
                    Q[k * m + q] = sn * qkp + c * qkq;
                }
            }
    }
    lam.resize(m);
    for (int i = 0; i < m; ++i) lam[i] = A[i * m + i];
}

// y = exp(-i T t) e_1 for the symmetric tridiagonal T = tri(beta, alpha, beta)
std::vector<std::complex<double>> tri_expm_e1(int k, const double* alpha, const double* beta, double t) {
    std::vector<double> A(static_cast<size_t>(k) * k, 0.0), Q, lam;
    for (int i = 0; i < k; ++i) {
        A[i * k + i] = alpha[i];
        if (i + 1 < k) A[i * k + i + 1] = A[(i + 1) * k + i] = beta[i];
    }
    jacobi_eig(k, A, Q, lam);
    std::vector<std::complex<double>> y(k, 0.0);
    for (int j = 0; j < k; ++j) {
        const std::complex<double> ph = std::exp(std::complex<double>(0.0, -lam[j] * t)) * Q[0 * k + j];
        for (int i = 0; i < k; ++i) y[i] += Q[i * k + j] * ph;
    }
    return y;
}

// Krylov basis buffers, kept between calls (cudaMalloc / cudaFree of tens of state-sized buffers
// per evolve call would dominate); released when the state shape changes
struct KrylovBuf {
    std::vector<DevState> v;
    void fit(const DevState& s) {
        if (!v.empty() && (v[0].bytes() != s.bytes() || v[0].dtype != s.dtype)) {
            stream_sync();
            for (auto& d : v)
                if (d.ptr) cudaFree(d.ptr);
            v.clear();
        }
    }
    void release() {
        if (v.empty()) return;
        stream_sync();
        for (auto& d : v)
            if (d.ptr) cudaFree(d.ptr);
        v.clear();
    }
};
KrylovBuf g_krylov;  // library-owned (released with the workspace)

// Lanczos on every batch column: builds the Krylov basis of H at psi until the residual estimate
// of e^{-iH dt} drops below tol (or maxdim vectors); when the full basis does not reach tol for dt,
// the largest dt' <= dt it does reach is taken instead (no matvec is wasted).  psi advances by the
// returned time.
using MatVec = std::function<void(const DevState& in, const DevState& out)>;

double lanczos_step(const DevState& psi, const MatVec& matvec, double dt, double tol, int maxdim, KrylovBuf& kb,
                    int* used) {
    const int64_t B = psi.B;
    kb.v.reserve(static_cast<size_t>(maxdim) + 2);
    auto vec = [&](int i) -> DevState {  // by value: the buffer list grows while vectors are in use
        while (static_cast<int>(kb.v.size()) <= i) {
            DevState d = psi;
            d.ptr = dev_alloc(psi.bytes(), true);
            kb.v.push_back(d);
        }
        DevState d = kb.v[i];
        d.n = psi.n;  // same bytes / dtype; the view follows the caller's shape
        d.B = psi.B;
        return d;
    };
    const size_t nd = static_cast<size_t>(2 * std::max<int64_t>(B, maxdim + 2));
    double* d_ip = static_cast<double*>(scratch(nd * sizeof(double), 16));
    double* d_cf = static_cast<double*>(scratch(nd * sizeof(double), 17));
    std::vector<double> ip(nd), cf(nd);
    auto fetch = [&](size_t cnt) {
        QBG_CUDA(cudaMemcpyAsync(ip.data(), d_ip, cnt * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        stream_sync();
    };
    auto inner = [&](const DevState& a, const DevState* c) {
        reduce_inner(a, c, d_ip);
        fetch(2 * B);
        return ip;
    };
    auto axpy = [&](const DevState& y, const DevState& x, bool overwrite) {
        QBG_CUDA(cudaMemcpyAsync(d_cf, cf.data(), 2 * B * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        launch_axpy_batch(y, x, d_cf, overwrite);
    };
    // W is slot 0, the basis v_i is slot i + 1
    std::vector<double> beta0(B);
    {
        auto n2 = inner(psi, nullptr);
        for (int64_t b = 0; b < B; ++b) {
            beta0[b] = std::sqrt(std::max(0.0, n2[2 * b]));
            cf[2 * b] = beta0[b] > 0 ? 1.0 / beta0[b] : 0.0;
            cf[2 * b + 1] = 0.0;
        }
        axpy(vec(1), psi, true);
    }
    std::vector<std::vector<double>> alpha(B), beta(B);
    auto error_at = [&](int k, double t) {  // max over batch columns of beta_k |e_k^T exp(-iTt) e_1|
        double err = 0.0;
        for (int64_t b = 0; b < B; ++b) {
            auto y = tri_expm_e1(k, alpha[b].data(), beta[b].data(), t);
            err = std::max(err, beta[b][k - 1] * std::abs(y[k - 1]));
        }
        return err;
    };
    int k = 0;
    double adv = 0.0;
    for (int j = 0; j < maxdim; ++j) {
        const DevState W = vec(0);
        matvec(vec(j + 1), W);
        // full re-orthogonalisation, two classical Gram-Schmidt passes (keeps the basis orthonormal
        // to rounding, so the small-matrix exponential is the exact projection)
        if (B == 1) {
            // first pass also measures ||W||^2 (W against itself); the second pass runs only when
            // the projection removed more than half of it (DGKS criterion: cancellation)
            std::vector<DevState> basis;
            for (int i = 0; i <= j; ++i) basis.push_back(vec(i + 1));
            for (int pass = 0; pass < 2; ++pass) {
                std::vector<DevState> with_w = basis;
                if (pass == 0) with_w.push_back(W);
                multi_inner(W, with_w, d_ip);
                fetch(2 * with_w.size());
                if (pass == 0) alpha[0].push_back(ip[2 * j]);
                std::vector<double> c(2 * (j + 1));
                double proj = 0.0;
                for (int i = 0; i <= j; ++i) {
                    c[2 * i] = -ip[2 * i];
                    c[2 * i + 1] = -ip[2 * i + 1];
                    proj += ip[2 * i] * ip[2 * i] + ip[2 * i + 1] * ip[2 * i + 1];
                }
                multi_axpy(W, basis, c);
                if (pass == 0 && proj < 0.5 * ip[2 * (j + 1)]) break;
            }
        } else {
            for (int pass = 0; pass < 2; ++pass)
                for (int i = 0; i <= j; ++i) {
                    auto h = inner(vec(i + 1), &W);
                    for (int64_t b = 0; b < B; ++b) {
                        if (pass == 0 && i == j) alpha[b].push_back(h[2 * b]);
                        cf[2 * b] = -h[2 * b];
                        cf[2 * b + 1] = -h[2 * b + 1];
                    }
                    axpy(W, vec(i + 1), false);
                }
        }
        auto n2 = inner(W, nullptr);
        bool breakdown = true;
        for (int64_t b = 0; b < B; ++b) {
            const double bj = std::sqrt(std::max(0.0, n2[2 * b]));
            beta[b].push_back(bj);
            if (bj > 1e-14 * std::max(1.0, std::fabs(alpha[b].back()))) breakdown = false;
        }
        k = j + 1;
        if (breakdown || error_at(k, dt) < tol) {
            adv = dt;
            break;
        }
        if (j + 1 < maxdim) {
            for (int64_t b = 0; b < B; ++b) {
                cf[2 * b] = beta[b][j] > 0 ? 1.0 / beta[b][j] : 0.0;
                cf[2 * b + 1] = 0.0;
            }
            axpy(vec(j + 2), W, true);
        }
    }
    if (adv == 0.0) {  // the full basis: the largest step it resolves to tol (bisection on |t|)
        double lo = 0.0, hi = dt;
        for (int it = 0; it < 60; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (error_at(k, mid) < tol)
                lo = mid;
            else
                hi = mid;
        }
        adv = lo;
        if (adv == 0.0) return 0.0;
    }
    // psi = beta0 * V y(adv)
    std::vector<std::vector<std::complex<double>>> ys(B);
    for (int64_t b = 0; b < B; ++b) ys[b] = tri_expm_e1(k, alpha[b].data(), beta[b].data(), adv);
    if (B == 1) {
        std::vector<DevState> basis;
        std::vector<double> c(2 * k);
        for (int i = 0; i < k; ++i) {
            basis.push_back(vec(i + 1));
            c[2 * i] = beta0[0] * ys[0][i].real();
            c[2 * i + 1] = beta0[0] * ys[0][i].imag();
        }
        QBG_CUDA(cudaMemsetAsync(psi.ptr, 0, psi.bytes(), g_stream));
        multi_axpy(psi, basis, c);
    } else {
        for (int i = 0; i < k; ++i) {
            for (int64_t b = 0; b < B; ++b) {
                cf[2 * b] = beta0[b] * ys[b][i].real();
                cf[2 * b + 1] = beta0[b] * ys[b][i].imag();
            }
            axpy(psi, vec(i + 1), i == 0);
        }
    }
    *used = std::max(*used, k);
    return adv;
}

}  // namespace
}  // namespace qbg

extern "C" {

}  // extern "C"

namespace qbg {
namespace {
// e^{-iHt} on the register by Lanczos steps (the step advances as far as the basis resolves)
void evolve_driver(qbg_reg* r, const MatVec& matvec, double t, double tol, int32_t maxdim, int32_t* krylov_dim) {
    if (!std::isfinite(t)) raise(QBG_ERR_VALIDATION, "time_evolve: non-finite time");
    if (maxdim <= 0) maxdim = 30;
    maxdim = std::min(maxdim, 60);
    if (tol <= 0) tol = 1e-12;
    int used = 0;
    if (t != 0.0) {
        KrylovBuf& kb = g_krylov;
        kb.fit(r->s);
        double rem = t;
        int steps = 0;
        while (rem != 0.0) {
            const double adv = lanczos_step(r->s, matvec, rem, tol, maxdim, kb, &used);
            if (adv == 0.0 || ++steps > 100000) raise(QBG_ERR_INTERNAL, "time_evolve: Krylov iteration made no progress");
            rem -= adv;
            if (std::fabs(rem) <= 1e-14 * std::fabs(t)) rem = 0.0;
        }
    }
    if (krylov_dim) *krylov_dim = used;
    stream_sync();
}
}  // namespace
}  // namespace qbg

namespace qbg {
void release_krylov(size_t keep_bytes) {
    if (!g_krylov.v.empty() && g_krylov.v[0].bytes() > keep_bytes) g_krylov.release();
}
}  // namespace qbg

struct qbg_sparse {
    int n = 0;
    int64_t nnz = 0;
    int64_t* rowptr = nullptr;  // device CSR
    int32_t* col = nullptr;
    double* val = nullptr;  // complex, interleaved
    bool hermitian = false;
};

extern "C" {

int qbg_time_evolve(qbg_reg* r, const qbg_obs* h, double t, double tol, int32_t maxdim, int32_t* krylov_dim) {
    return guarded([&] {
        check_reg(r);
        if (!h) raise(QBG_ERR_VALIDATION, "time_evolve: null Hamiltonian");
        auto& H = const_cast<qbg_obs*>(h)->o;
        if (H.n != r->nactive) raise(QBG_ERR_SHAPE, "time_evolve: Hamiltonian qubit count differs from active qubits");
        for (const auto& term : H.terms) {  // Hermitian: real coefficients once i^{nY} is divided out
            const int ny = __builtin_popcountll(term.xmask & term.zmask);
            std::complex<double> c(term.coef_re, term.coef_im);
            for (int k = 0; k < ny; ++k) c *= std::complex<double>(0.0, -1.0);
            if (std::fabs(c.imag()) > 1e-12 * std::max(1.0, std::abs(c)))
                raise(QBG_ERR_VALIDATION, "time_evolve: the Hamiltonian is not hermitian");
        }
        if (H.terms.empty()) {
            if (krylov_dim) *krylov_dim = 0;
            return;
        }
        evolve_driver(r, [&](const DevState& in, const DevState& out) { run_obs(in, out, H, nullptr); }, t, tol,
                      maxdim, krylov_dim);
    });
}

int qbg_sparse_create(int32_t n, int64_t nnz, const int64_t* colptr, const int64_t* rows, const double* vals,
                      qbg_sparse** out) {
    return guarded([&] {
        ensure_device();
        if (!out || !colptr || (nnz > 0 && (!rows || !vals))) raise(QBG_ERR_VALIDATION, "sparse: null argument");
        if (n < 1 || n > g_cap.load()) raise(QBG_ERR_RANGE, "sparse: qubit count out of range");
        const int64_t d = int64_t{1} << n;
        if (colptr[0] != 0 || colptr[d] != nnz) raise(QBG_ERR_SHAPE, "sparse: colptr does not span nnz entries");
        // CSC (the reference's SparseColumns, matrix.hpp) -> CSR for the row-gather kernel
        std::vector<int64_t> rp(d + 1, 0);
        for (int64_t c = 0; c < d; ++c) {
            if (colptr[c + 1] < colptr[c]) raise(QBG_ERR_VALIDATION, "sparse: colptr not monotone");
            for (int64_t k = colptr[c]; k < colptr[c + 1]; ++k) {
                if (rows[k] < 0 || rows[k] >= d) raise(QBG_ERR_RANGE, "sparse: row index out of range");
                rp[rows[k] + 1]++;
            }
        }
        for (int64_t r = 0; r < d; ++r) rp[r + 1] += rp[r];
        std::vector<int32_t> ci(nnz);
        std::vector<double> cv(2 * nnz);
        std::vector<int64_t> cur(rp.begin(), rp.end() - 1);
        std::map<std::pair<int64_t, int64_t>, std::complex<double>> entries;
        for (int64_t c = 0; c < d; ++c)
            for (int64_t k = colptr[c]; k < colptr[c + 1]; ++k) {
                const int64_t at = cur[rows[k]]++;
                ci[at] = static_cast<int32_t>(c);
                cv[2 * at] = vals[2 * k];
                cv[2 * at + 1] = vals[2 * k + 1];
                entries[{rows[k], c}] += std::complex<double>(vals[2 * k], vals[2 * k + 1]);
            }
        bool herm = true;
        double scale = 0.0;
        for (auto& [rc, v] : entries) scale = std::max(scale, std::abs(v));
        for (auto& [rc, v] : entries) {
            auto it = entries.find({rc.second, rc.first});
            const std::complex<double> w = it == entries.end() ? 0.0 : it->second;
            if (std::abs(v - std::conj(w)) > 1e-12 * std::max(1.0, scale)) {
                herm = false;
                break;
            }
        }
        auto* m = new qbg_sparse;
        m->n = n;
        m->nnz = nnz;
        m->hermitian = herm;
        try {
            m->rowptr = static_cast<int64_t*>(dev_alloc((d + 1) * sizeof(int64_t), false));
            m->col = static_cast<int32_t*>(dev_alloc(std::max<int64_t>(1, nnz) * sizeof(int32_t), false));
            m->val = static_cast<double*>(dev_alloc(std::max<int64_t>(1, nnz) * 2 * sizeof(double), false));
            QBG_CUDA(cudaMemcpyAsync(m->rowptr, rp.data(), (d + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, g_stream));
            if (nnz) {
                QBG_CUDA(cudaMemcpyAsync(m->col, ci.data(), nnz * sizeof(int32_t), cudaMemcpyHostToDevice, g_stream));
                QBG_CUDA(cudaMemcpyAsync(m->val, cv.data(), 2 * nnz * sizeof(double), cudaMemcpyHostToDevice, g_stream));
            }
            stream_sync();
        } catch (...) {
            if (m->rowptr) cudaFree(m->rowptr);
            if (m->col) cudaFree(m->col);
            if (m->val) cudaFree(m->val);
            delete m;
            throw;
        }
        *out = m;
    });
}

int qbg_sparse_destroy(qbg_sparse* m) {
    return guarded([&] {
        if (!m) return;
        stream_sync();
        cudaFree(m->rowptr);
        cudaFree(m->col);
        cudaFree(m->val);
        delete m;
    });
}

int qbg_sparse_apply(const qbg_reg* in, const qbg_sparse* m, qbg_reg* out) {
    return guarded([&] {
        check_reg(in);
        if (!m) raise(QBG_ERR_VALIDATION, "sparse: null operator");
        same_shape(in, out, "sparse apply");
        if (in == out) raise(QBG_ERR_VALIDATION, "sparse apply: input and output must differ");
        if (m->n != in->s.n || in->nactive != in->s.n) raise(QBG_ERR_SHAPE, "sparse apply: dimension mismatch");
        launch_spmv(in->s, out->s, m->rowptr, m->col, m->val, m->nnz);
        stream_sync();
    });
}

int qbg_time_evolve_sparse(qbg_reg* r, const qbg_sparse* m, double t, double tol, int32_t maxdim,
                           int32_t* krylov_dim) {
    return guarded([&] {
        check_reg(r);
        if (!m) raise(QBG_ERR_VALIDATION, "time_evolve: null operator");
        if (m->n != r->s.n || r->nactive != r->s.n) raise(QBG_ERR_SHAPE, "time_evolve: dimension mismatch");
        if (!m->hermitian) raise(QBG_ERR_VALIDATION, "time_evolve: the Hamiltonian is not hermitian");
        evolve_driver(r, [&](const DevState& in, const DevState& out) {
            launch_spmv(in, out, m->rowptr, m->col, m->val, m->nnz);
        }, t, tol, maxdim, krylov_dim);
    });
}

int qbg_mmd_grad(qbg_reg* r, const qbg_prog* prog, const qbg_mmd* m, int32_t inplace, double* loss, double* grads,
                 qbg_reg* state_grad) {
    return guarded([&] {
        mmd_check(r, m);
        auto& p = const_cast<qbg_prog*>(prog)->p;
        if (p.n != r->nactive) raise(QBG_ERR_SHAPE, "expect'(mmd): block qubit count differs from active qubits");
        if (state_grad) same_shape(r, state_grad, "expect'(mmd) state_grad");
        grad_driver(r, p, inplace, state_grad, loss, grads, [&](const DevState& psi, const DevState& adj, double* e) {
            launch_mmd(1, psi, nullptr, &adj, m->q, m->w, m->D, e);
        });
    });
}

}  // extern "C"
