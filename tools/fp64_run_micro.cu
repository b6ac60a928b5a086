// fp64_run_micro.cu — FP64 pipe efficiency of the reverse pass's per-run register work in
// isolation (no global / shared traffic): each thread holds x[16], y[16] (complex128), a "run"
// on register slot K is   [cross statistics (12 DFMA/pair)] + 2x2 on x + 2x2 on y  (16 + 16),
// optionally followed by the 4-value warp reduction into a per-warp shared cell.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_run_micro tools/fp64_run_micro.cu
//   /tmp/fp64_run_micro        (prints one line per variant / launch shape)
#include <cstdio>
#include <cuda_runtime.h>

struct __align__(16) c128 { double x, y; };
__device__ __forceinline__ c128 mk(double a, double b) { c128 v; v.x = a; v.y = b; return v; }
__device__ __forceinline__ c128 cmul(c128 a, c128 b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ c128 cfma(c128 a, c128 b, c128 c) { return mk(a.x + b.x * c.x - b.y * c.y, a.y + b.x * c.y + b.y * c.x); }

template <int K>
__device__ __forceinline__ void dense1(c128* x, c128 m00, c128 m10, c128 m01, c128 m11) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j & (1 << K)) continue;
    c128 a = x[j], b = x[j | (1 << K)];
    x[j] = cfma(cmul(m00, a), m01, b);
    x[j | (1 << K)] = cfma(cmul(m10, a), m11, b);
  }
}
template <int K>
__device__ __forceinline__ void crossh(const c128* p, const c128* a, double* c) {
  double i01 = 0, i10 = 0, r01 = 0, r10 = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j & (1 << K)) continue;
    const double a0x = a[j].x, a0y = a[j].y, a1x = a[j | (1 << K)].x, a1y = a[j | (1 << K)].y;
    const double p0x = p[j].x, p0y = p[j].y, p1x = p[j | (1 << K)].x, p1y = p[j | (1 << K)].y;
    c[0] = fma(a0x, p0y, fma(-a0y, p0x, c[0]));
    c[1] = fma(a1x, p1y, fma(-a1y, p1x, c[1]));
    i01 = fma(a0x, p1y, fma(-a0y, p1x, i01));
    i10 = fma(a1x, p0y, fma(-a1y, p0x, i10));
    r01 = fma(a0x, p1x, fma(a0y, p1y, r01));
    r10 = fma(a1x, p0x, fma(a1y, p0y, r10));
  }
  c[2] += i01 + i10;
  c[3] += r01 - r10;
}
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

struct PMx { double m[64]; };

// MODE 0: uncompute only; 1: + cross stats accumulated in registers; 2: + per-run warp reduction
template <int MODE, int TPB, int MINB>
__global__ void __launch_bounds__(TPB, MINB) k_runs(int iters, const __grid_constant__ PMx pm, double* out) {
  __shared__ double sg[64 * 33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  c128 x[16], y[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) { x[j] = mk(1e-3 * (tid + j), 1e-4 * j); y[j] = mk(1e-4 * (tid - j), 1e-3); }
  for (int i = tid; i < 64 * 33; i += TPB) sg[i] = 0;
  __syncthreads();
  double acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0;
#define M(i) mk(pm.m[2 * (i)], pm.m[2 * (i) + 1])
#define RUN(K, S)                                                                                          \
  {                                                                                                        \
    if (MODE >= 1) {                                                                                       \
      double c[4] = {0, 0, 0, 0};                                                                          \
      crossh<K>(x, y, c);                                                                                  \
      if (MODE == 2) {                                                                                     \
        const double v = warp_sum4(c, lane);                                                               \
        if ((lane & 7) == 0) sg[((S) * 4 + (lane >> 3)) * 33 + warp] += v;                                  \
      } else {                                                                                             \
        acc[(S) * 4 + 0] += c[0]; acc[(S) * 4 + 1] += c[1]; acc[(S) * 4 + 2] += c[2]; acc[(S) * 4 + 3] += c[3]; \
      }                                                                                                    \
    }                                                                                                      \
    dense1<K>(x, M(4 * (S)), M(4 * (S) + 1), M(4 * (S) + 2), M(4 * (S) + 3));                             \
    dense1<K>(y, M(4 * (S)), M(4 * (S) + 1), M(4 * (S) + 2), M(4 * (S) + 3));                             \
  }
  for (int it = 0; it < iters; ++it) {
    RUN(0, 0) RUN(1, 1) RUN(2, 2) RUN(3, 3)
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j].x + y[j].y;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  __syncthreads();
  if (s == 12345.678) out[blockIdx.x * TPB + tid] = s + sg[tid];
}

template <int MODE, int TPB, int MINB>
void run(const char* name, int sms, double clk_ghz) {
  PMx pm;
  for (int i = 0; i < 64; ++i) pm.m[i] = 0.3 + 0.01 * i;
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
  const int iters = 2000;
  const int blocks = sms * MINB;
  k_runs<MODE, TPB, MINB><<<blocks, TPB>>>(10, pm, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_runs<MODE, TPB, MINB><<<blocks, TPB>>>(iters, pm, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  // fp64 instructions per run per thread: 2 x 128 (uncompute) + 96 (cross) + 4 (DADD) [+ 3 reduction DADD]
  const double per_run = 256.0 + (MODE >= 1 ? 96.0 + 2.0 : 0.0) + (MODE == 2 ? 5.0 : 4.0 * (MODE == 1));
  const double inst = per_run * 4.0 * iters * TPB * (double)blocks;
  const double rate = inst / (ms * 1e-3);           // fp64 thread-instructions per second
  const double peak = 64.0 * sms * clk_ghz * 1e9;   // DFMA lanes per second
  std::printf("%-28s TPB=%4d blocks/SM=%d : %8.3f ms  fp64 pipe %.1f%% of peak\n", name, TPB, MINB, ms,
              100.0 * rate / peak);
  cudaFree(out);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double ghz = clk / 1e6;
  std::printf("SMs %d, clock %.3f GHz\n", sms, ghz);
  run<0, 128, 1>("uncompute only", sms, ghz);
  run<0, 128, 2>("uncompute only", sms, ghz);
  run<0, 256, 1>("uncompute only", sms, ghz);
  run<1, 128, 1>("+cross (reg acc)", sms, ghz);
  run<1, 128, 2>("+cross (reg acc)", sms, ghz);
  run<1, 256, 1>("+cross (reg acc)", sms, ghz);
  run<2, 128, 1>("+cross +warp_sum4", sms, ghz);
  run<2, 128, 2>("+cross +warp_sum4", sms, ghz);
  run<2, 256, 1>("+cross +warp_sum4", sms, ghz);
  return 0;
}
