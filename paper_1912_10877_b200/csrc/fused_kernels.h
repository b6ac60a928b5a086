// fused_kernels.h — launchers of the device kernels in fused_kernels.cu
#pragma once

#include "engine.h"
#include "fused.h"

namespace qbg {

void launch_interp(int dtype, bool back, void* psi, void* adj, const fz::DPass& P, const fz::DOp* d_ops,
                   const cdbl* d_mats, double* gpart, int64_t gcols);
void launch_grad_rows(const double* part, int64_t nrows, int64_t cols, double* sums);
// grads[p] += Σ_{entries k of p, plan order} value_k   (CSR ptr/idx over parameters)
void launch_grad_epilogue(const double* sums, const fz::GradEntry* d_epi, int64_t n, const int* d_ptr, const int* d_idx,
                          int64_t nparams, double* grads);
void launch_seed(int dtype, const void* psi, void* phi, const fz::SPass& sp, const fz::SGroup* g, const fz::STerm* t,
                 double* epart, double bytes);
void launch_energy(const double* epart, uint64_t nouter, int64_t nchunks, int64_t bc, int64_t B, double* e);

}  // namespace qbg
