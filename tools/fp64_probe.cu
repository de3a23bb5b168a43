// FP64 pipe probe on sm_100a: DFMA (register / constant-bank operand), DMMA
// (mma.sync.m8n8k4.f64) and the two interleaved in one warp.  Decides whether
// FP64 tensor-core contractions can add throughput next to the DFMA pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

struct Coef { double c[8]; };

__global__ void dfma_reg(double* out, int iters, double a) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  double b = a * 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void dfma_const(double* out, int iters, const __grid_constant__ Coef k) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], k.c[i], k.c[7 - i]);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2];
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void mixed(double* out, int iters, double a) {
  double acc[4][2];
  double x[8];
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0;
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  double av = threadIdx.x * 1e-3, bv = 1.0 - threadIdx.x * 1e-4, b = a * 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) dmma(acc[i][0], acc[i][1], av, bv);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, blocks = sms * 4, threads = 256;
  Coef k;
  for (int i = 0; i < 8; ++i) k.c[i] = 0.999 + i * 1e-6;
  auto run = [&](const char* name, auto launch, double flops_per_thread_iter) {
    launch();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = double(blocks) * threads * iters * flops_per_thread_iter;
    printf("%-12s %8.3f ms  %7.2f TFLOP/s\n", name, ms, fl / (ms * 1e-3) / 1e12);
  };
  run("dfma_reg", [&] { dfma_reg<<<blocks, threads>>>(out, iters, 0.999); }, 8 * 2.0);
  run("dfma_const", [&] { dfma_const<<<blocks, threads>>>(out, iters, k); }, 8 * 2.0);
  // one m8n8k4 = 256 FMA per warp = 8 FMA per thread = 16 flops per thread
  run("dmma", [&] { dmma_loop<<<blocks, threads>>>(out, iters); }, 8 * 16.0);
  run("mixed", [&] { mixed<<<blocks, threads>>>(out, iters, 0.999); }, 4 * 16.0 + 8 * 2.0);
  cudaError_t err = cudaGetLastError();
  printf("status: %s, SMs %d\n", cudaGetErrorString(err), sms);
  return 0;
}
