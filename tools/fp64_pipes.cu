// fp64_pipes.cu — measures B200 FP64 throughput of DFMA (CUDA cores), DMMA (mma.sync m8n8k4 f64,
// legacy tensor path) and both interleaved, to decide whether FP64 tensor ops add throughput.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_pipes.cu -o build/fp64_pipes
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
    double x[16];
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    double s = 0;
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, double a, double b) {
    double c[16];
    for (int i = 0; i < 16; ++i) c[i] = 0;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 16; i += 2) dmma(c[i], c[i + 1], a, b);
    double s = 0;
    for (int i = 0; i < 16; ++i) s += c[i];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_both(double* out, double a, double b) {
    double c[8], x[8];
    for (int i = 0; i < 8; ++i) c[i] = 0, x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; i += 2) dmma(c[i], c[i + 1], a, b);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i] + x[i];
    if (s == 1.2345) out[0] = s;
}

template <class K>
float time_it(K k, int blocks, int threads, double* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<blocks, threads>>>(out, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int blocks = sms * 8, threads = 256;
    const double warps = blocks * threads / 32.0;
    float t1 = time_it(k_dfma, blocks, threads, out);
    double f1 = blocks * threads * 16.0 * ITERS * 2 / (t1 * 1e-3) / 1e12;
    float t2 = time_it(k_dmma, blocks, threads, out);
    double f2 = warps * 8.0 * ITERS * (8 * 8 * 4 * 2) / (t2 * 1e-3) / 1e12;
    float t3 = time_it(k_both, blocks, threads, out);
    double f3 = (warps * 4.0 * ITERS * (8 * 8 * 4 * 2) + blocks * threads * 8.0 * ITERS * 2) / (t3 * 1e-3) / 1e12;
    std::printf("{\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"both_tflops\": %.2f, \"ms\": [%.3f, %.3f, %.3f]}\n",
                f1, f2, f3, t1, t2, t3);
    return 0;
}
