// Measured FP64 (DFMA) throughput and dependent-chain latency on this GPU:
// the compute roof the stage kernel runs against.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_chains(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void dfma_latency(double* out, int iters, double a, double b, long long* cycles) {
  double x = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  if (x == 12345.678) out[0] = x;
}

template <int ILP>
static double run(int blocks, int threads, int iters) {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_chains<ILP><<<blocks, threads>>>(d, 100, 0.999999, 1e-7);
  cudaEventRecord(e0);
  dfma_chains<ILP><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(d);
  return 2.0 * ILP * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d", p.name, sms);
  double best = 0;
  for (int w : {8, 16, 32}) {
    const double t4 = run<4>(sms * 4, w * 8, 20000), t8 = run<8>(sms * 4, w * 8, 10000);
    printf(", \"dfma_tflops_warps%d_ilp4\": %.2f, \"dfma_tflops_warps%d_ilp8\": %.2f", w, t4, w, t8);
    best = t4 > best ? t4 : best;
    best = t8 > best ? t8 : best;
  }
  double* d;
  long long* c;
  cudaMalloc(&d, 8);
  cudaMalloc(&c, 8);
  dfma_latency<<<1, 32>>>(d, 4096, 0.999999, 1e-7, c);
  long long h = 0;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf(", \"dfma_peak_tflops\": %.2f, \"dfma_dependent_latency_cycles\": %.2f}\n", best, h / 4096.0);
  return 0;
}
