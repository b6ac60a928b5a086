// engine.h — host-side interfaces of the device engine (kernels live in *.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

namespace qbg {

// A device state vector: 2^n rows of B batch-innermost complex amplitudes.
struct DevState {
    void* ptr = nullptr;
    int n = 0;
    int64_t B = 1;
    int dtype = QBG_C128;
    size_t elem() const { return dtype == QBG_C128 ? 16 : 8; }
    uint64_t rows() const { return uint64_t{1} << n; }
    uint64_t count() const { return rows() * static_cast<uint64_t>(B); }
    size_t bytes() const { return static_cast<size_t>(count()) * elem(); }
};

// A realised gate placed on 0-based bit positions (register.hpp:292-339 KernelPlan).
struct Gate {
    int kind = QBG_MAT_IDENTITY;  // QBG_MAT_*
    int t = 0;                    // number of targets
    int dim = 0;                  // 2^t
    uint8_t tbit[QBG_MAX_TARGETS] = {0};  // matrix qubit q acts on bit tbit[q]
    uint64_t tmask = 0, cmask = 0, cval = 0;
    std::vector<cdbl> m;     // DIAGONAL/PERMUTATION: dim; DENSE: dim*dim column-major
    std::vector<int> perm;   // PERMUTATION: row k takes column perm[k]
};

Gate adjoint(const Gate& g);      // matrix.hpp:594-643
bool is_diagonal(const Gate& g);  // IDENTITY or DIAGONAL

// ---- generic per-gate kernels (register.hpp:352-385 on the device) --------------------
void launch_gate(const DevState& s, const Gate& g);
int dense_path();            // qbg_set_dense_path
void set_dense_path(int p);
// 3..5-qubit gate as a GEMM on the FP64 tensor cores (DMMA); false when not applicable (c64,
// non-power-of-two batch, non-finite matrix, too few free bits) — the caller falls back
bool launch_dense_mma(const DevState& s, const Gate& g);
// the same on tcgen05 (kind::tf32, 3xTF32 split, TMEM accumulators) for complex64 registers
bool launch_dense_tc(const DevState& s, const Gate& g);
// Reverse step of one gate on (psi, adj): grad_slot (if >= 0) receives, per block, the
// partial Im <adj| K |psi> (K restricted to the control subspace) BEFORE the uncompute;
// then psi <- U^† psi, adj <- U^† adj with U^† = gdag.
void launch_gate_back(const DevState& psi, const DevState& adj, const Gate& gdag, const Gate* K,
                      double* partials, int64_t nblocks_cap, int* nblocks_used);

// ---- reductions (register.hpp:120-150), deterministic two-level trees ------------------
// out[2*b], out[2*b+1] = <a_b|c_b> (c == nullptr: a := c, i.e. squared norm in .re)
void reduce_inner(const DevState& a, const DevState* c, double* d_out /* device, 2*B */);
void sum_partials(const double* d_part, int64_t nrows, int64_t ncols, double* d_out);
// part is [nslots][cap]; grads[slot_param[s]] += sum_b part[s][b], slots in order
void accumulate_grads(const double* d_part, int64_t nslots, int64_t cap, const int* d_slot_param, double* d_grads);

// ---- elementwise -------------------------------------------------------------------------
void launch_scale(const DevState& s, double re, double im);
void launch_axpy(const DevState& y, const DevState& x, double re, double im);
// y (+)= c_b x with c_b = (d_coef[2b], d_coef[2b+1]) per batch column (device array)
void launch_axpy_batch(const DevState& y, const DevState& x, const double* d_coef, bool overwrite);
void launch_set_basis(const DevState& s, const uint64_t* d_bits, int64_t nbits);
void launch_transpose(const void* src, void* dst, uint64_t rows, int64_t B, int dtype, bool to_device_layout);
void launch_pauli_axpy(const DevState& psi, const DevState& phi, uint64_t xmask, uint64_t zmask, double cre,
                       double cim, bool overwrite);
void launch_permute_bits(const DevState& src, const DevState& dst, const int* new_of_old);
void launch_probabilities(const DevState& s, int nactive, int64_t batch, double* d_p);
void launch_collapse(const DevState& s, int nactive, int64_t batch, uint64_t hit, double inv);

// ---- MMD loss (mmd.cu): mode 0 loss, 1 loss + seed adj = 2 (K d) psi, 2 cross with `other` ----
// d_loss[b] (device) receives the per-batch sum; taps d_w[0..D]; target d_q[2^n]
void launch_mmd(int mode, const DevState& psi, const DevState* other, const DevState* adj, const double* d_q,
                const double* d_w, int D, double* d_loss);
bool mmd_geometry(uint64_t rows, int64_t B, int D, int* TX, int* BC, size_t* smem);

// ---- Krylov multi-vector kernels (krylov.cu; one batch column) ----
// d_out[2i], d_out[2i+1] = <vs[i] | w>;  w += Σ_i coef_i vs[i]
void multi_inner(const DevState& w, const std::vector<DevState>& vs, double* d_out);
void multi_axpy(const DevState& w, const std::vector<DevState>& vs, const std::vector<double>& coef);

// ---- sparse operator (sparse.cu): y = A x, A in CSR (complex values interleaved) ----
void launch_spmv(const DevState& x, const DevState& y, const int64_t* d_rowptr, const int32_t* d_col,
                 const double* d_val, int64_t nnz);

// ---- sharded states (shard.cu): copy the rows of a sub-block (nfix fixed 0-based row bits with
// values fix_val bit i -> fix_pos[i]) in sub-row range [h0, h0 + count) to / from a flat buffer ----
void launch_shard_copy(const DevState& s, bool pack, const int* fix_pos, int nfix, uint64_t fix_val, uint64_t h0,
                       uint64_t count, void* buf);

// scratch device memory owned by the library (grows; stream-ordered reuse)
void* scratch(size_t bytes, int slot);

}  // namespace qbg
