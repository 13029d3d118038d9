// Measures the relative error of the MUFU.RCP64H / RSQ64H seeds and of one /
// two Newton steps, to size the fast-mode reciprocal (run on a B200).
#include <cstdio>
#include <cmath>
#include <curand_kernel.h>
__global__ void k(double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  curandStatePhilox4_32_10_t st;
  curand_init(1234, i, 0, &st);
  double x = exp(curand_uniform_double(&st) * 40.0 - 20.0);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  double r1 = fma(r, e, r);
  double e2 = fma(-x, r1, 1.0);
  double r2 = fma(r1, e2, r1);
  double ex = 1.0 / x;
  double r3 = fma(r, fma(e, e, e), r);  // third-order step used by fvb_physics.cuh frcp
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double ey = 1.0 / sqrt(x);
  double hx = 0.5 * x;
  double y1 = y * fma(-hx * y, y, 1.5);
  double s1 = x * y1;
  double s1c = fma(fma(-s1, s1, x), 0.5 * y1, s1);
  double y2 = y1 * fma(-hx * y1, y1, 1.5);
  double s2 = x * y2;
  double s2c = fma(fma(-s2, s2, x), 0.5 * y2, s2);
  double sq = sqrt(x);
  // fvb_physics.cuh fsqrt (fast mode): one third-order step on s = x*y
  double s3 = x * y;
  double e3 = fma(-s3, y, 1.0);
  s3 = fma(s3 * e3, fma(e3, 0.375, 0.5), s3);
  out[i * 9 + 7] = fabs(s3 - sq) / sq;
  out[i * 9 + 8] = fabs(s3 - sq) / (nextafter(sq, 1e300) - sq);  // ulps
  out[i * 9 + 0] = fabs(r - ex) / ex;
  out[i * 9 + 1] = fabs(r1 - ex) / ex;
  out[i * 9 + 2] = fabs(r3 - ex) / ex;
  (void)r2;
  out[i * 9 + 3] = fabs(y - ey) / ey;
  out[i * 9 + 4] = fabs(s1c - sq) / sq;
  out[i * 9 + 5] = fabs(s2c - sq) / sq;
  out[i * 9 + 6] = (s1c == sq) ? 0.0 : 1.0;
}
int main() {
  const int n = 1 << 22;
  double* d;
  cudaMalloc(&d, sizeof(double) * 9 * n);
  k<<<n / 256, 256>>>(d, n);
  double* h = new double[9 * (size_t)n];
  cudaMemcpy(h, d, sizeof(double) * 9 * n, cudaMemcpyDeviceToHost);
  double mx[9] = {0};
  double cnt = 0;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < 9; ++j) if (j != 6) mx[j] = fmax(mx[j], h[i * 9 + j]);
    cnt += h[i * 9 + 6];
  }
  printf("rcp seed %.3e  1NR %.3e  cubic %.3e\n", mx[0], mx[1], mx[2]);
  printf("rsq seed %.3e  sqrt(1NR+corr) %.3e  sqrt(2NR+corr) %.3e  (1NR+corr != sqrt in %.4f%%)\n", mx[3], mx[4],
         mx[5], 100.0 * cnt / n);
  printf("sqrt(third-order step) max rel %.3e  max ulp %.2f\n", mx[7], mx[8]);
  return 0;
}
