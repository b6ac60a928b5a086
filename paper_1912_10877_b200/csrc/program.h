// program.h — compiled gate programs and observables (host side).
#pragma once

#include <memory>
#include <vector>

#include "engine.h"

namespace qbg {

struct FusedPlan;  // fused.cu

// Realised instruction: U, U^† and the gradient generator K with θ̄ = Im <φ̄|K|ψ_{k+1}>
// on the control subspace (rotation: K = G; shift: K = −2 P1; phase: K = −2 I).
struct RealOp {
    Gate u, udag, k;
    int param = -1;
};

struct Program {
    int n = 0;
    std::vector<qbg_op> ops;
    std::vector<cdbl> vals;
    std::vector<int64_t> perms;
    int64_t nparams = 0;
    std::vector<double> theta;
    std::vector<RealOp> real;  // realised at theta
    bool realised = false;
    // fused plans cached per (B, dtype); rebuilt on structural change only
    std::vector<std::shared_ptr<FusedPlan>> plans;
    uint64_t version = 0;  // bumps on set_params
};

struct Observable {
    int n = 0;
    std::vector<qbg_pauli_term> terms;  // coefficient already multiplied by i^{nY}
    std::vector<std::shared_ptr<FusedPlan>> plans;
};

void validate_op(int nactive, const qbg_op& op);  // make_plan checks, register.hpp:299-339
Gate place_gate(const qbg_op& op, int kind, int dim, const std::vector<cdbl>& m, const std::vector<int>& perm);
void realise(Program& p);

// fused engine (fused.cu); return false when the plan does not apply (caller falls back)
// src: optional input state (not s): the first pass reads it and writes s (out-of-place start)
bool fused_forward(const DevState& s, Program& p, bool adjoint, const void* src = nullptr);
bool fused_backward(const DevState& psi, const DevState& adj, Program& p, double* d_grads /* nparams, += */);
bool fused_obs_apply(const DevState& psi, const DevState& phi, Observable& o, double* d_energy /* B or null */);
// passes of the most recently built forward / backward plans (0 when unfused)
void fused_stats(const Program& p, int64_t* fwd, int64_t* bwd);
// checkpointed expect' (fused.cu): the number of full-state checkpoints the program needs on s (0:
// unavailable, use fused_forward / fused_backward); the forward writes them into arena (checkpoint 0
// = the output state), the reverse pass reads them
int64_t fused_ckpt_states(Program& p, const DevState& s);
// false: the program's structure changed with θ (plans rebuilt); the caller sizes the arena again
bool fused_ckpt_forward(const DevState& in, Program& p, void* arena, int64_t k);
// after the forward is queued: brings the reverse plan up to date; false if the forward just run
// used segments of a stale structure (the caller runs the forward again)
bool fused_ckpt_sync(Program& p, const DevState& s, int64_t k);
void fused_ckpt_backward(const DevState& adj, Program& p, void* arena, double* d_grads /* nparams, += */);
void fused_set_checkpointing(bool on);  // qbg_set_checkpointing (default on unless QBG_CKPT=0)
std::string fused_plan_info(const Program& p);  // human-readable pass/stage layout
// Host-only planner run (no device): forward + reverse plans for a 2^n x B register.
std::string fused_plan_preview(const Program& p, int64_t B, int dtype);
// Host-only NVRTC compile of every specialised kernel (program + observable); no device.
int64_t fused_jit_check(const Program& p, const Observable* o, int64_t B, int dtype);

}  // namespace qbg
