/*
 * qbg.h — C-ABI of the B200 state-vector engine (the drop-in boundary).
 *
 * The reference (`/root/reference/proj/include/qblock`, header-only C++20) exposes the
 * register "instruction set" that Yao's GPU backend overloads:
 * Register construction, instruct, inner/norm/scale/add_scaled, probabilities/measure,
 * focus/relax.  SPEC.md adds apply/expect/expect_grad above it.
 * Every entry point below names the reference interface it replaces.
 *
 * Conventions (bits.hpp:27-28, register.hpp:54-57):
 *   - qubits are 1-based at this interface; qubit 1 is the least significant bit;
 *   - host buffers use the reference layout: batch slowest, each batch a contiguous
 *     slice of 2^n interleaved complex doubles (re, im);
 *   - on the device a register is stored batch-innermost ([2^n][B]); upload/download
 *     transpose.
 *   - every call returns an int error code (errors.hpp:24-81 mapped to QBG_ERR_*);
 *     qbg_last_error() returns the thread-local message of the last failure.
 * No torch types cross this boundary: plain pointers and sizes only.
 */
#ifndef QBG_H
#define QBG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes: qblock::Error subclasses, errors.hpp:24-81 ---------------------- */
enum {
    QBG_OK = 0,
    QBG_ERR_VALIDATION = 1,      /* ValidationError     errors.hpp:29-31 */
    QBG_ERR_SHAPE = 2,           /* ShapeError          errors.hpp:34-36 */
    QBG_ERR_RANGE = 3,           /* RangeError          errors.hpp:39-41 */
    QBG_ERR_DISPATCH = 4,        /* DispatchError       errors.hpp:44-46 */
    QBG_ERR_RESOURCE = 5,        /* ResourceError       errors.hpp:49-51 */
    QBG_ERR_UNSUPPORTED = 6,     /* UnsupportedError    errors.hpp:54-56 */
    QBG_ERR_UNDECIDABLE = 7,     /* UndecidableError    errors.hpp:59-61 */
    QBG_ERR_RENORMALIZATION = 8, /* RenormalizationError errors.hpp:64-66 */
    QBG_ERR_SERIALIZATION = 9,   /* SerializationError  errors.hpp:69-71 */
    QBG_ERR_PARSE = 10,          /* ParseError          errors.hpp:74-81 */
    QBG_ERR_CUDA = 100,          /* CUDA runtime failure (no reference counterpart) */
    QBG_ERR_NCCL = 101,          /* NCCL failure */
    QBG_ERR_INTERNAL = 102
};

/* ---- element types ----------------------------------------------------------------- */
enum { QBG_C128 = 0, QBG_C64 = 1 };

/* ---- matrix classes: the MatrixRepr alternatives, matrix.hpp:41-129 ---------------- */
enum {
    QBG_MAT_IDENTITY = 0,    /* Identity      matrix.hpp:42-47 */
    QBG_MAT_DIAGONAL = 1,    /* Diagonal      matrix.hpp:49-54  vals: dim complex */
    QBG_MAT_PERMUTATION = 2, /* Permutation   matrix.hpp:59-75  row i -> (perm[i], vals[i]) */
    QBG_MAT_DENSE = 4        /* Dense         matrix.hpp:104-115 column-major a[c*dim+r] */
    /* SparseColumns/OuterProduct are densified by the caller exactly like the reference's
       generic fallback (register.hpp:372, to_dense matrix.hpp:229-233). */
};

/* ---- parameterised primitives (SPEC.md:300-308 Rotation/Shift/Phase) ---------------- */
enum {
    QBG_GEN_NONE = 0,     /* constant gate: payload is the gate matrix itself */
    QBG_GEN_ROTATION = 1, /* rot(G, θ) = cos(θ/2) I − i sin(θ/2) G, gates.hpp:79-92; payload is G */
    QBG_GEN_SHIFT = 2,    /* diag(1, e^{iθ}), gates.hpp:72; no payload */
    QBG_GEN_PHASE = 3     /* e^{iθ}·I, gates.hpp:73-75; no payload */
};

#define QBG_MAX_TARGETS 5
#define QBG_MAX_CTRLS 16

/* One gate matrix passed to qbg_instruct (register.hpp:392 `const MatrixRepr& gate`). */
typedef struct qbg_matrix {
    int32_t kind;          /* QBG_MAT_* */
    int32_t dim;           /* 2^t */
    const double* vals;    /* interleaved complex; DIAGONAL/PERMUTATION: dim, DENSE: dim*dim */
    const int64_t* perm;   /* PERMUTATION only */
} qbg_matrix;

/* One instruction of a gate program: the flat lowering of a block tree (SPEC.md:315-323:
   Put/Control/Kron/Repeat each become one instruct).  Matrix payloads live in the program's
   value array (complex elements, offset `data`) and permutation array (offset `perm`). */
typedef struct qbg_op {
    int32_t kind;      /* QBG_MAT_* class of the payload (of G for QBG_GEN_ROTATION) */
    int32_t gen;       /* QBG_GEN_* */
    int32_t param;     /* parameter slot (>= 0) for gen != NONE, else -1 */
    int32_t ntarget;   /* 1..QBG_MAX_TARGETS */
    int32_t nctrl;     /* 0..QBG_MAX_CTRLS */
    int32_t dim;       /* 2^ntarget */
    int32_t targets[QBG_MAX_TARGETS]; /* 1-based; matrix qubit q acts on targets[q] */
    int32_t ctrls[QBG_MAX_CTRLS];     /* 1-based */
    int32_t ctrl_cfg[QBG_MAX_CTRLS];  /* 0 or 1 */
    int64_t data;      /* offset (complex elements) of the payload in the value array */
    int64_t perm;      /* offset of the permutation in the index array (PERMUTATION) */
} qbg_op;

/* One Pauli-string term c·P of an observable (heisenberg: SPEC.md:557-565, an Add of
   Put·Put products).  Bit (q-1) of xmask/zmask: X = x, Z = z, Y = x&z. */
typedef struct qbg_pauli_term {
    double coef_re, coef_im;
    uint64_t xmask, zmask;
} qbg_pauli_term;

typedef struct qbg_reg qbg_reg;   /* device register: replaces qblock::Register (register.hpp:58-256) */
typedef struct qbg_prog qbg_prog; /* compiled gate program (fusion plan + realised matrices) */
typedef struct qbg_obs qbg_obs;   /* compiled observable (sum of Pauli terms) */
typedef struct qbg_rng qbg_rng;   /* host RNG: replaces qblock::Rng (rng.hpp:25-66) */
typedef struct qbg_mmd qbg_mmd;   /* MMD loss: target distribution + RBF-mixture kernel */
typedef struct qbg_sparse qbg_sparse; /* full-register sparse operator: the Cached block's matrix */

/* ---- library ------------------------------------------------------------------------- */
const char* qbg_last_error(void);
const char* qbg_version(void);
/* qubit_cap / set_qubit_cap, register.hpp:36-41 (default 30; raise for large states) */
int qbg_set_qubit_cap(int32_t cap);
int32_t qbg_get_qubit_cap(void);
/* state_alloc_counter, register.hpp:45-48: counts full-state device allocations */
uint64_t qbg_alloc_count(void);
/* Select the CUDA device and the stream (a cudaStream_t, 0 = legacy default) new work is
   issued on.  One device per process: once the library holds anything on a device (registers,
   workspace, plans, loaded kernels) a different device is rejected with QBG_ERR_VALIDATION. */
int qbg_set_device(int32_t device);
/* Frees the library-owned device workspace: the expect' work/adjoint states, the Krylov basis and
   the scratch slots (counted by qbg_alloc_count while held).  Workspace larger than every live
   register is also released automatically when a register is destroyed. */
int qbg_release_workspace(void);
int qbg_set_stream(void* stream);
int qbg_synchronize(void);
/* Fusion switch: 1 (default) = tiled multi-gate passes, 0 = one kernel per gate. */
int qbg_set_fusion(int32_t enabled);
/* expect' design: 1 (default) = checkpointed (the forward passes keep the state after every
   reverse segment, the reverse passes read it instead of uncomputing it; used when those
   checkpoints fit in device memory, the register is left unmodified), 0 = uncompute (two extra
   full states at most, the register is uncomputed back to the input when in place). */
int qbg_set_checkpointing(int32_t enabled);
/* Upper bound on the device memory the checkpoints may take (bytes; -1, the default: whatever is
   free less a reserve of max(4 GiB, 1/16 of the device)).  Above it expect' uncomputes. */
int qbg_set_checkpoint_limit(int64_t bytes);
/* Kernel for dense 3..5-qubit gates (register.hpp:371-384 as one GEMM over all bases):
   1 (default) FP64 tensor cores, DMMA m8n8k4 (complex64 is widened to FP64 and rounded once);
   2 complex64 on tcgen05 kind::tf32 with a 3-piece operand split (faster; the tensor cores' fp32
   accumulation drifts the norm by ~6e-7 per block); 0 the CUDA-core per-gate kernel. */
int qbg_set_dense_path(int32_t path);
/* Per-kernel CUDA-event timing of the library's own launches (measurement hook). */
int qbg_profile_enable(int32_t enabled);
int qbg_profile_reset(void);
/* Writes up to `cap` records "name\tlaunches\ttotal_ms\tbytes\tflops" separated by '\n'
   (bytes / flops: the algorithmic traffic and floating-point work of those launches). */
int qbg_profile_report(char* buf, int64_t cap);
/* Number of kernels the library launched since the last reset. */
uint64_t qbg_launch_count(void);
int qbg_launch_count_reset(void);

/* ---- RNG: qblock::Rng, rng.hpp:25-66 (SplitMix64-mixed seed -> std::mt19937_64) -------- */
int qbg_rng_create(uint64_t seed, qbg_rng** out);
int qbg_rng_destroy(qbg_rng* rng);
int qbg_rng_split_label(const qbg_rng* rng, const char* label, qbg_rng** out); /* rng.hpp:30-36 */
int qbg_rng_split_salt(const qbg_rng* rng, uint64_t salt, qbg_rng** out);      /* rng.hpp:38 */
double qbg_rng_uniform(qbg_rng* rng);                                          /* rng.hpp:43 */
double qbg_rng_uniform_range(qbg_rng* rng, double lo, double hi);              /* rng.hpp:46-48 */
double qbg_rng_gauss(qbg_rng* rng);                                            /* rng.hpp:51 */
uint64_t qbg_rng_bits(qbg_rng* rng);                                           /* rng.hpp:53 */

/* ---- registers: Register ctor/copy, register.hpp:60-93 --------------------------------- */
int qbg_reg_create(int32_t nqubits, int64_t nbatch, int32_t dtype, uint64_t seed, qbg_reg** out);
int qbg_reg_destroy(qbg_reg* reg);
int qbg_reg_clone(const qbg_reg* reg, qbg_reg** out);            /* Register(const Register&) */
int qbg_reg_copy(qbg_reg* dst, const qbg_reg* src);               /* operator= (same shape)   */
int qbg_reg_info(const qbg_reg* reg, int32_t* nqubits, int32_t* nactive, int64_t* nbatch,
                 int32_t* dtype);
/* Raw device pointer of the batch-innermost buffer (for interop / collectives). */
void* qbg_reg_device_ptr(qbg_reg* reg);
qbg_rng* qbg_reg_rng(qbg_reg* reg);                               /* Register::rng(), 118 */
/* zero_state / product_state, register.hpp:260-264, 282-286.  `bits` holds one basis index
   per batch (nbits == nbatch) or a single index broadcast to all batches (nbits == 1). */
int qbg_set_zero(qbg_reg* reg);
int qbg_set_product(qbg_reg* reg, const uint64_t* bits, int64_t nbits);
/* rand_state, register.hpp:266-280: Gaussian amplitudes from Rng(seed).split("rand_state")
   drawn on the host (libstdc++ normal_distribution is implementation-defined) and uploaded. */
int qbg_set_rand(qbg_reg* reg, uint64_t seed);
/* Host <-> device with the batch transpose; n_complex = 2^n * B. */
int qbg_upload(qbg_reg* reg, const double* host, int64_t n_complex);
int qbg_download(const qbg_reg* reg, double* host, int64_t n_complex);
/* Same, device layout ([2^n][B]) host buffer — no transpose. */
int qbg_upload_raw(qbg_reg* reg, const void* host, int64_t nbytes);
int qbg_download_raw(const qbg_reg* reg, void* host, int64_t nbytes);

/* ---- instruction set: instruct, register.hpp:392-408 ----------------------------------- */
int qbg_instruct(qbg_reg* reg, const qbg_matrix* gate, const int32_t* locs, int32_t nloc,
                 const int32_t* ctrl_locs, const int32_t* ctrl_cfg, int32_t nctrl);
/* gate_by_tag, gates.hpp:156-175: "X","Y","Z","H","I2","S","Sdag","T","Tdag","SWAP","CNOT",
   "CZ","Toffoli","P0","P1","Pu","Pd","Rx","Ry","Rz","shift","phase". */
int qbg_instruct_tag(qbg_reg* reg, const char* tag, const int32_t* locs, int32_t nloc,
                     const int32_t* ctrl_locs, const int32_t* ctrl_cfg, int32_t nctrl,
                     const double* params, int32_t nparams);

/* ---- register algebra: register.hpp:120-150 -------------------------------------------- */
int qbg_norm(const qbg_reg* reg, double* out /* nbatch */);
int qbg_inner(const qbg_reg* a, const qbg_reg* b, double* out /* 2*nbatch, <a|b> */);
int qbg_scale(qbg_reg* reg, double re, double im);
int qbg_add_scaled(qbg_reg* reg, const qbg_reg* other, double re, double im);

/* ---- measurement: register.hpp:414-493 --------------------------------------------------- */
int qbg_probabilities(const qbg_reg* reg, int64_t batch, double* out /* 2^nactive */);
/* measure(const Register&, nshots, Rng&): out holds nshots*nbatch basis indices grouped by
   batch; rng == NULL uses the register's own stream (register.hpp:457-459). */
int qbg_measure(const qbg_reg* reg, int64_t nshots, qbg_rng* rng, uint64_t* out);
int qbg_measure_collapse(qbg_reg* reg, qbg_rng* rng, uint64_t* out /* nbatch */);

/* ---- focus / relax: register.hpp:156-177 --------------------------------------------------- */
int qbg_focus(qbg_reg* reg, const int32_t* locs, int32_t nloc);
int qbg_relax(qbg_reg* reg, const int32_t* locs, int32_t nloc, int32_t to_nactive);

/* ---- state files: Register::save / load, register.hpp:181-205 ------------------------------
   "QBREG1\0\0", u64 nqubits, u64 nactive, u64 nbatch, then the amplitudes in the reference
   layout (batch slowest) as little-endian complex doubles.  Files interchange with qblock. */
int qbg_save(const qbg_reg* reg, const char* path);
int qbg_load(const char* path, uint64_t seed, int32_t dtype, qbg_reg** out);
/* The same format from memory (Register::load(std::istream&) of the C++ shim). */
int qbg_load_memory(const void* data, int64_t nbytes, uint64_t seed, int32_t dtype, qbg_reg** out);

/* ---- sharded states (SPEC.md:290 makes distributed state a non-goal of the
   reference, so these have no reference counterpart) ---------------------------------------------
   A state of n qubits over 2^g ranks is one register of n-g local qubits per rank.  Moving global
   qubits k_1..k_j against local qubits l_1..l_j exchanges, with each partner, the sub-block of rows
   whose local qubits l_i are fixed to the partner's bits.  pack copies sub-block rows
   [row0, row0 + nrows) (rows in increasing order; each row carries its nbatch amplitudes) into the
   device buffer dst; unpack writes them back.  fix_locs are 1-based local qubits (<= 8), bit i of
   fix_val is the value of fix_locs[i].  Stream-ordered on the library stream. */
int qbg_shard_pack(const qbg_reg* reg, const int32_t* fix_locs, int32_t nfix, uint64_t fix_val, int64_t row0,
                   int64_t nrows, void* dst);
int qbg_shard_unpack(qbg_reg* reg, const int32_t* fix_locs, int32_t nfix, uint64_t fix_val, int64_t row0,
                     int64_t nrows, const void* src);
/* device staging buffers owned by the library (exchange chunks) */
int qbg_buffer_alloc(int64_t bytes, void** out);
int qbg_buffer_free(void* ptr);

/* ---- gate programs: apply(reg, block) lowered to instruct, SPEC.md:315-323 --------------- */
int qbg_prog_create(int32_t nqubits, const qbg_op* ops, int64_t nops, const double* vals,
                    int64_t nvals, const int64_t* perms, int64_t nperms, qbg_prog** out);
int qbg_prog_destroy(qbg_prog* prog);
int64_t qbg_prog_nparams(const qbg_prog* prog);
/* dispatch(b, vec): realise every parameterised matrix at θ. */
int qbg_prog_set_params(qbg_prog* prog, const double* theta, int64_t nparams);
/* Number of device passes the fusion planner emits for forward / backward. */
int qbg_prog_stats(const qbg_prog* prog, int64_t* fwd_passes, int64_t* bwd_passes,
                   int64_t* fwd_gates);
/* Text description of the fusion plans built so far (passes, tile qubits, stages, ops). */
int qbg_prog_plan_info(const qbg_prog* prog, char* buf, int64_t cap);
/* Runs the fusion planner on the host only (no device needed) for an nbatch register. */
int qbg_prog_plan_preview(const qbg_prog* prog, int64_t nbatch, int32_t dtype, char* buf, int64_t cap);
/* Generates and compiles (NVRTC -> sm_100a cubin, no device needed) every specialised kernel the
   program (and observable, may be NULL) would use; *nkernels receives the number of passes. */
int qbg_jit_check(const qbg_prog* prog, const qbg_obs* obs, int64_t nbatch, int32_t dtype, int64_t* nkernels);
/* Kernel-cache statistics since load: NVRTC compilations vs cubins found in the cache (the
   ahead-of-time cache built by build() lives in jit_cache/ next to libqbg.so). */
int qbg_jit_stats(int64_t* nvrtc_builds, int64_t* cache_hits);
int qbg_apply(qbg_reg* reg, const qbg_prog* prog);
/* Applies the adjoint program (Daggered chain). */
int qbg_apply_adjoint(qbg_reg* reg, const qbg_prog* prog);

/* ---- observables and AD: SPEC.md:433-527 ---------------------------------------------------- */
int qbg_obs_create(int32_t nqubits, const qbg_pauli_term* terms, int64_t nterms, qbg_obs** out);
int qbg_obs_destroy(qbg_obs* obs);
/* expect(O, reg): out[b] = Re <psi_b|O|psi_b>. */
int qbg_expect(const qbg_reg* reg, const qbg_obs* obs, double* out /* nbatch */);
/* out_reg := O |reg> (Add of Put·Put, "Add: Σ child|ψ>"). */
int qbg_obs_apply(const qbg_reg* reg, const qbg_obs* obs, qbg_reg* out_reg);
/* Reverse pass (apply_back + mat_back): given psi = U|psi_0> and
   adj = dL/d<psi|, uncomputes psi -> psi_0, back-propagates adj, and ADDS the parameter
   gradient (summed over the batch) into grads[nparams]. */
int qbg_backward(qbg_reg* psi, qbg_reg* adj, const qbg_prog* prog, double* grads);
/* expect'(O, reg => circuit).  Runs forward on a copy of `reg` (or on reg
   itself when inplace != 0; it is uncomputed back to the input), seeds adj = O psi,
   runs the reverse pass.  energies[nbatch] = <O>, grads[nparams] (summed over the batch),
   state_grad (optional, may be NULL) receives the adjoint of the input state. */
int qbg_expect_grad(qbg_reg* reg, const qbg_prog* prog, const qbg_obs* obs, int32_t inplace,
                    double* energies, double* grads, qbg_reg* state_grad);

/* e^{-iHt}|reg> in place for a hermitian Pauli-sum H (SPEC.md:397-405 time_evolve; matrix.hpp:680-724
   matvec_cols): Lanczos on the device with full re-orthogonalisation, subspace <= maxdim (<= 0:
   30), residual estimate < tol (<= 0: 1e-12), the step halved until it converges.  Every batch
   column evolves independently.  krylov_dim (may be NULL) receives the largest subspace used.
   Errors: non-hermitian H -> QBG_ERR_VALIDATION; qubit mismatch -> QBG_ERR_SHAPE. */
int qbg_time_evolve(qbg_reg* reg, const qbg_obs* h, double t, double tol, int32_t maxdim, int32_t* krylov_dim);

/* ---- sparse operators (SPEC.md:397 cache(b); matrix.hpp:680-724 matvec_cols over SparseColumns) ----
   A is given like the reference's SparseColumns (CSC): colptr[2^n + 1], rows[nnz], vals[2*nnz]
   (complex interleaved); kept on the device in CSR.  Errors: malformed CSC -> QBG_ERR_VALIDATION /
   QBG_ERR_RANGE / QBG_ERR_SHAPE. */
int qbg_sparse_create(int32_t nqubits, int64_t nnz, const int64_t* colptr, const int64_t* rows, const double* vals,
                      qbg_sparse** out);
int qbg_sparse_destroy(qbg_sparse* a);
/* out = A in, every batch column (the register must be relaxed; out != in) */
int qbg_sparse_apply(const qbg_reg* in, const qbg_sparse* a, qbg_reg* out);
/* e^{-iAt}|reg> for a hermitian sparse A (Lanczos as qbg_time_evolve); non-hermitian -> QBG_ERR_VALIDATION */
int qbg_time_evolve_sparse(qbg_reg* reg, const qbg_sparse* a, double t, double tol, int32_t maxdim,
                           int32_t* krylov_dim);

/* ---- one-call forms named in SURVEY §8(b) (thin wrappers over the handle API above) --------- */
/* apply a flat program once: create (theta: nparams values, may be NULL when none), apply,
   destroy.  Re-used circuits should keep a qbg_prog (plans and specialised kernels are cached on it). */
int qbg_run_program(qbg_reg* reg, const qbg_op* ops, int64_t nops, const double* vals, int64_t nvals,
                    const int64_t* perms, int64_t nperms, const double* theta, int64_t nparams);
/* <O>_b for a Pauli sum given as terms (one call: create, expect, destroy) */
int qbg_expect_pauli_sum(const qbg_reg* reg, const qbg_pauli_term* terms, int64_t nterms, double* out);
/* y += (re + i im) x   (= qbg_add_scaled, register.hpp:130-133) */
int qbg_axpy(qbg_reg* y, const qbg_reg* x, double re, double im);
/* = qbg_measure_collapse (register.hpp:470-493) */
int qbg_collapse(qbg_reg* reg, qbg_rng* rng, uint64_t* out);

/* ---- MMD loss (SPEC.md:446-449 MMDLoss, 497-505 mmd_expect / mmd_grad; §3.2,
   Listing 12 "expect'(mmd, zero_state(5)=>circuit)") -------------------------
   L_b = sum_{x,y} K(x,y) (p_b - q)_x (p_b - q)_y with p_b = |psi_b|^2 over the 2^n basis states
   and K(x,y) = sum_s exp(-(x-y)^2 / (2 sigma_s^2)) (the radial-basis mixture over the integer
   distance, brbf_kernel(sigma)).  Errors: target_p must be >= 0 and sum to 1 within 1e-12,
   sigmas > 0 (QBG_ERR_VALIDATION); the register must have nqubits == n and no focus
   (QBG_ERR_SHAPE). */
int qbg_mmd_create(int32_t nqubits, const double* target_p, const double* sigmas, int32_t nsigma, qbg_mmd** out);
int qbg_mmd_destroy(qbg_mmd* m);
/* taps kept by the banded convolution (every dropped tap is exactly 0.0 in double) */
int qbg_mmd_band(const qbg_mmd* m, int32_t* band);
/* loss[nbatch] */
int qbg_mmd_loss(const qbg_reg* reg, const qbg_mmd* m, double* loss);
/* loss[nbatch] and the reverse-mode seed adj = dL/dpsi* = 2 (K (p - q))_x psi_x */
int qbg_mmd_seed(const qbg_reg* psi, const qbg_mmd* m, qbg_reg* adj, double* loss);
/* out[b] = sum_{x,y} K(x,y) p^a_b(x) (p_b(y) - q(y)) with p^a = |a|^2, p = |reg|^2: the
   shift-rule building block  dL/dtheta = sum_b cross(psi(theta+pi/2), psi) - cross(psi(theta-pi/2), psi) */
int qbg_mmd_cross(const qbg_reg* a, const qbg_reg* reg, const qbg_mmd* m, double* out);
/* expect'(mmd, reg => prog): forward, seed, reverse pass (as qbg_expect_grad). */
int qbg_mmd_grad(qbg_reg* reg, const qbg_prog* prog, const qbg_mmd* m, int32_t inplace, double* loss,
                 double* grads, qbg_reg* state_grad);

#ifdef __cplusplus
}
#endif
#endif /* QBG_H */
