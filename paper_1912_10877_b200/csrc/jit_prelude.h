// jit_prelude.h — device templates the generated tile-pass kernels are written in.
// Every slot index and register-control mask is a template argument: in the generated
// straight-line code a controlled swap is a compile-time register rename (no instruction), a
// register-controlled gate has no per-pair predicate, and matrix entries are constant-bank
// operands of the FMAs (the pass's matrices are a __grid_constant__ kernel parameter).
#pragma once

namespace qbg {
namespace jit {

static const char kPrelude[] = R"QBGJIT(
typedef unsigned long long u64;
typedef long long i64;
struct __align__(16) c128 { double x, y; };
struct __align__(8) c64 { float x, y; };
template <class V> struct RT;
template <> struct RT<c128> { typedef double T; };
template <> struct RT<c64> { typedef float T; };
template <class T, int N> struct PM { T m[N]; };

template <class V> __device__ __forceinline__ V mk(typename RT<V>::T a, typename RT<V>::T b) { V v; v.x = a; v.y = b; return v; }
template <class V> __device__ __forceinline__ V cmul(V a, V b) { return mk<V>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
template <class V> __device__ __forceinline__ V cfma(V a, V b, V c) { return mk<V>(a.x + b.x * c.x - b.y * c.y, a.y + b.x * c.y + b.y * c.x); }
template <class V> __device__ __forceinline__ double imcm(V a, V b) { return (double)a.x * b.y - (double)a.y * b.x; }

template <class V, int R, int K, int CM, int CV>
__device__ __forceinline__ void dense1(V* x, V m00, V m10, V m01, V m11) {
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (j & (1 << K)) continue;
    if ((j & CM) != CV) continue;
    V a = x[j], b = x[j | (1 << K)];
    x[j] = cfma(cmul(m00, a), m01, b);
    x[j | (1 << K)] = cfma(cmul(m10, a), m11, b);
  }
}
template <class V, int R, int K, int CM, int CV>
__device__ __forceinline__ void swap1(V* x) {
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (j & (1 << K)) continue;
    if ((j & CM) != CV) continue;
    V a = x[j]; x[j] = x[j | (1 << K)]; x[j | (1 << K)] = a;
  }
}
template <class V, int R, int K, int CM, int CV>
__device__ __forceinline__ void diag1(V* x, V d0, V d1) {
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if ((j & CM) != CV) continue;
    x[j] = cmul(x[j], (j & (1 << K)) ? d1 : d0);
  }
}
template <class V, int R, int CM, int CV>
__device__ __forceinline__ void scale(V* x, V d) {
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if ((j & CM) != CV) continue;
    x[j] = cmul(x[j], d);
  }
}
template <class V, int R, int K0, int K1, int CM, int CV>
__device__ __forceinline__ void dense2(V* x, const V* m) {
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (j & ((1 << K0) | (1 << K1))) continue;
    if ((j & CM) != CV) continue;
    const int i0 = j, i1 = j | (1 << K0), i2 = j | (1 << K1), i3 = j | (1 << K0) | (1 << K1);
    V a0 = x[i0], a1 = x[i1], a2 = x[i2], a3 = x[i3];
    V r[4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      V acc = cmul(m[rr], a0);
      acc = cfma(acc, m[4 + rr], a1);
      acc = cfma(acc, m[8 + rr], a2);
      r[rr] = cfma(acc, m[12 + rr], a3);
    }
    x[i0] = r[0]; x[i1] = r[1]; x[i2] = r[2]; x[i3] = r[3];
  }
}
// 8x8 (column-major m[c * 8 + r]) on the register slots K0, K1, K2 (matrix qubits 0, 1, 2)
template <class V, int R, int K0, int K1, int K2, int CM, int CV>
__device__ __forceinline__ void dense3(V* x, const V* m) {
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (j & ((1 << K0) | (1 << K1) | (1 << K2))) continue;
    if ((j & CM) != CV) continue;
    V a[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = x[j | ((c & 1) << K0) | (((c >> 1) & 1) << K1) | (((c >> 2) & 1) << K2)];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      V acc = cmul(m[r], a[0]);
#pragma unroll
      for (int c = 1; c < 8; ++c) acc = cfma(acc, m[8 * c + r], a[c]);
      x[j | ((r & 1) << K0) | (((r >> 1) & 1) << K1) | (((r >> 2) & 1) << K2)] = acc;
    }
  }
}
// 16x16 (column-major m[c * 16 + r]) on the register slots K0..K3 (matrix qubits 0..3)
template <class V, int R, int K0, int K1, int K2, int K3, int CM, int CV>
__device__ __forceinline__ void dense4(V* x, const V* m) {
  constexpr int MASK = (1 << K0) | (1 << K1) | (1 << K2) | (1 << K3);
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (j & MASK) continue;
    if ((j & CM) != CV) continue;
    V a[16];
#pragma unroll
    for (int c = 0; c < 16; ++c)
      a[c] = x[j | ((c & 1) << K0) | (((c >> 1) & 1) << K1) | (((c >> 2) & 1) << K2) | (((c >> 3) & 1) << K3)];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      V acc = cmul(m[r], a[0]);
#pragma unroll
      for (int c = 1; c < 16; ++c) acc = cfma(acc, m[16 * c + r], a[c]);
      x[j | ((r & 1) << K0) | (((r >> 1) & 1) << K1) | (((r >> 2) & 1) << K2) | (((r >> 3) & 1) << K3)] = acc;
    }
  }
}
// ---- gradient terms Σ Im(conj(adj) (K psi)) ----
template <class V, int R, int K, int CM, int CV>
__device__ __forceinline__ double gdense1(const V* p, const V* a, V k00, V k10, V k01, V k11) {
  double g = 0.0;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (j & (1 << K)) continue;
    if ((j & CM) != CV) continue;
    V p0 = p[j], p1 = p[j | (1 << K)];
    g += imcm(a[j], cfma(cmul(k00, p0), k01, p1));
    g += imcm(a[j | (1 << K)], cfma(cmul(k10, p0), k11, p1));
  }
  return g;
}
template <class V, int R, int K, int CM, int CV>
__device__ __forceinline__ double gdiag1(const V* p, const V* a, V d0, V d1) {
  double g = 0.0;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if ((j & CM) != CV) continue;
    g += imcm(a[j], cmul((j & (1 << K)) ? d1 : d0, p[j]));
  }
  return g;
}
template <class V, int R, int CM, int CV>
__device__ __forceinline__ double gscale(const V* p, const V* a, V d) {
  double sr = 0.0, si = 0.0;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if ((j & CM) != CV) continue;
    sr += (double)a[j].x * p[j].x + (double)a[j].y * p[j].y;
    si += (double)a[j].x * p[j].y - (double)a[j].y * p[j].x;
  }
  return (double)d.x * si + (double)d.y * sr;
}
template <class V, int R, int K0, int K1, int CM, int CV>
__device__ __forceinline__ double gdense2(const V* p, const V* a, const V* m) {
  double g = 0.0;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (j & ((1 << K0) | (1 << K1))) continue;
    if ((j & CM) != CV) continue;
    const int idx[4] = {j, j | (1 << K0), j | (1 << K1), j | (1 << K0) | (1 << K1)};
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      V acc = cmul(m[rr], p[idx[0]]);
      acc = cfma(acc, m[4 + rr], p[idx[1]]);
      acc = cfma(acc, m[8 + rr], p[idx[2]]);
      acc = cfma(acc, m[12 + rr], p[idx[3]]);
      g += imcm(a[idx[rr]], acc);
    }
  }
  return g;
}
// C_ab = Σ conj(adj_a) psi_b over the pairs on slot K: c[2(2a+b)] = Re, c[2(2a+b)+1] = Im
template <class V, int R, int K>
__device__ __forceinline__ void gcross1(const V* p, const V* a, double* c) {
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (j & (1 << K)) continue;
    const V av[2] = {a[j], a[j | (1 << K)]};
    const V pv[2] = {p[j], p[j | (1 << K)]};
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) {  // explicit FMA chains: 4 DFMA per complex product-accumulate
        c[2 * (2 * u + v)] = fma((double)av[u].y, (double)pv[v].y, fma((double)av[u].x, (double)pv[v].x, c[2 * (2 * u + v)]));
        c[2 * (2 * u + v) + 1] = fma(-(double)av[u].y, (double)pv[v].x, fma((double)av[u].x, (double)pv[v].y, c[2 * (2 * u + v) + 1]));
      }
  }
}
// Hermitian-run cross statistics (4 components instead of 8): for Hermitian M,
//   Im Σ_ab M_ab C_ab = M00 Im C00 + M11 Im C11 + Re M01 Im(C01 + C10) + Im M01 Re(C01 − C10)
// c[0] = Im C00, c[1] = Im C11, c[2] = Im(C01 + C10), c[3] = Re(C01 − C10): 12 DFMA per pair.
template <class V, int R, int K>
__device__ __forceinline__ void gcrossh1(const V* p, const V* a, double* c) {
  typedef typename RT<V>::T T;
  T c0 = 0, c1 = 0, i01 = 0, i10 = 0, r01 = 0, r10 = 0;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (j & (1 << K)) continue;
    const T a0x = a[j].x, a0y = a[j].y, a1x = a[j | (1 << K)].x, a1y = a[j | (1 << K)].y;
    const T p0x = p[j].x, p0y = p[j].y, p1x = p[j | (1 << K)].x, p1y = p[j | (1 << K)].y;
    c0 = fma(a0x, p0y, fma(-a0y, p0x, c0));
    c1 = fma(a1x, p1y, fma(-a1y, p1x, c1));
    i01 = fma(a0x, p1y, fma(-a0y, p1x, i01));
    i10 = fma(a1x, p0y, fma(-a1y, p0x, i10));
    r01 = fma(a0x, p1x, fma(a0y, p1y, r01));
    r10 = fma(a1x, p0x, fma(a1y, p0y, r10));
  }
  c[0] = (double)c0;  // assigned: every caller hands in a fresh c
  c[1] = (double)c1;
  c[2] = (double)i01 + (double)i10;
  c[3] = (double)r01 - (double)r10;
}
// diagonal run: c[b] += Σ Im(conj(a) p) over the elements whose run bit is b — register slot K
template <class V, int R, int K>
__device__ __forceinline__ void gcrossd_r(const V* p, const V* a, double* c) {
#pragma unroll
  for (int j = 0; j < R; ++j) c[(j >> K) & 1] = fma((double)a[j].x, (double)p[j].y, fma(-(double)a[j].y, (double)p[j].x, c[(j >> K) & 1]));
}
// ... or a bit uniform over the thread's elements (thread / tile bit)
template <class V, int R>
__device__ __forceinline__ void gcrossd_u(const V* p, const V* a, double* c, int bit) {
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < R; ++j) s = fma((double)a[j].x, (double)p[j].y, fma(-(double)a[j].y, (double)p[j].x, s));
  if (bit) c[1] += s; else c[0] += s;
}
// global -> shared async copy of one element (LDGSTS); completion via cp_commit / cp_wait
template <class V>
__device__ __forceinline__ void cpa(V* sdst, const V* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  if (sizeof(V) == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(s), "l"(gsrc) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" :: "r"(s), "l"(gsrc) : "memory");
}
// ---- warp-specialised pipeline: mbarriers, bulk async copies (TMA engine), named barriers ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(smem_u32(b)) : "memory");
}
// bounded wait: a schedule bug traps (kernel error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  // spin (no suspend-time hint: measured 0.611 -> 0.63 ms per reverse pass with the 10-ms hint —
  // the waiting consumer wakes late on the critical path)
  unsigned done = 0;
  unsigned long long spins = 0;
  while (true) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
    if (done) break;
    if (++spins > (1ull << 27)) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               :: "r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// arrive on the mbarrier when all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_arrive_noinc(unsigned long long* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" :: "r"(smem_u32(b)) : "memory");
}
template <int NT>
__device__ __forceinline__ void named_bar() { asm volatile("bar.sync 1, %0;\n" :: "n"(NT) : "memory"); }
// tensor-memory-access (TMA) tile loads: one elected thread copies the tile box into the slot and
// the transfer completes the slot's mbarrier (the map is a __grid_constant__ kernel parameter)
struct __align__(64) TMap { unsigned long long w[16]; };
__device__ __forceinline__ void tma_load1(void* dst, const TMap* m, unsigned long long* bar, int c0) {
  asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];\n"
               :: "r"(smem_u32(dst)), "l"(m), "r"(c0), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load2(void* dst, const TMap* m, unsigned long long* bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
               :: "r"(smem_u32(dst)), "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load3(void* dst, const TMap* m, unsigned long long* bar, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
               :: "r"(smem_u32(dst)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load4(void* dst, const TMap* m, unsigned long long* bar, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
               :: "r"(smem_u32(dst)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load5(void* dst, const TMap* m, unsigned long long* bar, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
               :: "r"(smem_u32(dst)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)) : "memory");
}
// TMA tensor stores of a computed tile (shared -> global, bulk-group completion)
__device__ __forceinline__ void tma_store1(const TMap* m, const void* src, int c0) {
  asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];\n"
               :: "l"(m), "r"(c0), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_store2(const TMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n"
               :: "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_store3(const TMap* m, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n"
               :: "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_store4(const TMap* m, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n"
               :: "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_store5(const TMap* m, const void* src, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n"
               :: "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void tma_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void tma_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// bounds check of a generated index (QBG_JIT_CHECK builds): trap instead of reading / writing out of range
__device__ __forceinline__ long long qchk(long long i, long long n) {
  if ((unsigned long long)i >= (unsigned long long)n) __trap();
  return i;
}
// shared-memory swizzle of a tile-local element index (same as the host planner's swz)
__device__ __forceinline__ unsigned swz(unsigned l) { return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9) ^ (l >> 12) ^ (l >> 15)) & 7u); }
// programmatic dependent launch: block until the preceding grid in the stream has completed and
// its memory is visible (every specialised kernel calls this before touching global memory)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// barrier over NT threads with a runtime id (one id per consumer group)
template <int NT>
__device__ __forceinline__ void group_bar(int id) { asm volatile("bar.sync %0, %1;\n" :: "r"(id), "n"(NT) : "memory"); }
// warpgroup register reallocation (producer gives registers to the consumers)
template <int N>
__device__ __forceinline__ void reg_alloc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" :: "n"(N)); }
template <int N>
__device__ __forceinline__ void reg_dealloc() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" :: "n"(N)); }
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" :: "n"(N) : "memory"); }
// one writer per reduction group: every lane reads the cell (harmless), the lane with w set stores
// cell + v by a predicated st.shared — no branch, so the stage stays one basic block
__device__ __forceinline__ void sg_acc(double* cell, double v, bool w) {
  const double nv = *cell + v;
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.shared.f64 [%0], %1;\n}\n"
               :: "r"(smem_u32(cell)), "d"(nv), "r"((unsigned)w) : "memory");
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Hermitian cross statistics of the runs on register slots 0..NK-1 together (the checkpointed
// reverse pass's statistics groups): c[4k .. 4k+3] = Im C00, Im C11, Im(C01 + C10), Re(C01 - C10)
// of slot k, zero for k >= NK.  The diagonal parts are sums of the per-element Im(conj(a) p), shared
// by the slots; the off-diagonal accumulators alternate between two halves (8-deep FMA chains).
template <class V, int R, int NK>
__device__ __forceinline__ void gstat_group(const V* p, const V* a, double* c) {
  typedef typename RT<V>::T T;
  T d[R];
#pragma unroll
  for (int j = 0; j < R; ++j) d[j] = fma((T)a[j].x, (T)p[j].y, -((T)a[j].y * (T)p[j].x));
  T t[R];
#pragma unroll
  for (int j = 0; j < R; ++j) t[j] = d[j];
#pragma unroll
  for (int w = R / 2; w >= 1; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; ++i) t[i] += t[i + w];
  const T tot = t[0];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k >= NK) {
      c[4 * k] = 0.0; c[4 * k + 1] = 0.0; c[4 * k + 2] = 0.0; c[4 * k + 3] = 0.0;
      continue;
    }
    T s0[2] = {0, 0}, i01[2] = {0, 0}, i10[2] = {0, 0}, r01[2] = {0, 0}, r10[2] = {0, 0};
    int h = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (j & (1 << k)) continue;
      const int j1 = j | (1 << k);
      const T a0x = a[j].x, a0y = a[j].y, a1x = a[j1].x, a1y = a[j1].y;
      const T p0x = p[j].x, p0y = p[j].y, p1x = p[j1].x, p1y = p[j1].y;
      s0[h] += d[j];
      i01[h] = fma(a0x, p1y, fma(-a0y, p1x, i01[h]));
      i10[h] = fma(a1x, p0y, fma(-a1y, p0x, i10[h]));
      r01[h] = fma(a0x, p1x, fma(a0y, p1y, r01[h]));
      r10[h] = fma(a1x, p0x, fma(a1y, p0y, r10[h]));
      h ^= 1;
    }
    const T sz = s0[0] + s0[1];
    c[4 * k] = (double)sz;
    c[4 * k + 1] = (double)(tot - sz);
    c[4 * k + 2] = (double)((i01[0] + i01[1]) + (i10[0] + i10[1]));
    c[4 * k + 3] = (double)((r01[0] + r01[1]) - (r10[0] + r10[1]));
  }
}
// 16 values per lane -> lane l holds the warp total of component (l >> 1) & 15 (16 shuffles)
__device__ __forceinline__ double warp_sum16(double* v, int lane) {
#pragma unroll
  for (int o = 16, n = 8; o >= 2; o >>= 1, n >>= 1) {
    const bool hi = lane & o;
#pragma unroll
    for (int k = 0; k < n; ++k) {
      const double send = hi ? v[k] : v[k + n], keep = hi ? v[k + n] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}
// 8 values over the warp by halving exchanges; lane 4c ends with the sum of component c
// 4 values per lane -> lane l holds the warp total of component (l >> 3) & 3
__device__ __forceinline__ double warp_sum4(double* v, int lane) {
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      double send = hi ? v[k] : v[k + 2], keep = hi ? v[k + 2] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  {
    const bool hi = lane & 8;
    double send = hi ? v[0] : v[1], keep = hi ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double s = v[0];
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}
__device__ __forceinline__ double warp_sum8(double* v, int lane) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool hi = lane & 16;
    double send = hi ? v[k] : v[k + 4], keep = hi ? v[k + 4] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool hi = lane & 8;
    double send = hi ? v[k] : v[k + 2], keep = hi ? v[k + 2] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const bool hi = lane & 4;
    double send = hi ? v[0] : v[1], keep = hi ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  double s = v[0];
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}
)QBGJIT";

}  // namespace jit
}  // namespace qbg
