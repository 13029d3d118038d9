// FP64 issue microbenchmark for the stage kernels' operating point
// (DESIGN.md section 5): FP64 instruction rate at a given number of warps per
// SM and independent chains per thread, with and without one interleaved
// 32-bit integer instruction per FP64 instruction.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_mix tools/fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, bool INT>
__global__ void mix(double* out, unsigned* iout, int iters, double a, double b) {
  double x[ILP];
  unsigned k[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) {
    x[j] = threadIdx.x * 1e-3 + j;
    k[j] = threadIdx.x * 7u + j;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
      x[j] = fma(x[j], a, b);
      if (INT) k[j] = k[j] * 1664525u + 1013904223u;  // one IMAD per DFMA
    }
  }
  double s = 0.0;
  unsigned t = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) {
    s += x[j];
    t ^= k[j];
  }
  if (s == 12345.678) out[0] = s;
  if (t == 0x12345678u) iout[0] = t;
}

template <int ILP, bool INT>
static double rate(int sms, int warps_per_sm, int iters) {
  double* d;
  unsigned* u;
  cudaMalloc(&d, 8);
  cudaMalloc(&u, 4);
  // one block of `warps_per_sm` warps per SM
  const int threads = 32 * warps_per_sm;
  mix<ILP, INT><<<sms, threads>>>(d, u, 100, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<ILP, INT><<<sms, threads>>>(d, u, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(d);
  cudaFree(u);
  return (double)ILP * iters * sms * threads / (ms * 1e-3) / 1e12;  // T FP64 thread-instr / s
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d, \"unit\": \"T DFMA thread-instructions/s\"", p.name, sms);
  for (int w : {8, 12, 16, 32}) {
    printf(", \"w%d_ilp1\": %.2f, \"w%d_ilp2\": %.2f, \"w%d_ilp4\": %.2f", w, rate<1, false>(sms, w, 40000), w,
           rate<2, false>(sms, w, 20000), w, rate<4, false>(sms, w, 10000));
    printf(", \"w%d_ilp2_int\": %.2f, \"w%d_ilp4_int\": %.2f", w, rate<2, true>(sms, w, 20000), w,
           rate<4, true>(sms, w, 10000));
  }
  printf("}\n");
  return 0;
}
