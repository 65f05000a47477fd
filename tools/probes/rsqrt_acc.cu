#include <cstdio>
#include <cmath>
__global__ void k(const double* in, double* o1, double* o2, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double y1, y2;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y1) : "d"(in[i]));
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y2) : "d"(in[i]));
  o1[i] = y1; o2[i] = y2;
}
int main() {
  const int n = 1 << 20;
  double *in, *o1, *o2;
  cudaMallocManaged(&in, n * 8); cudaMallocManaged(&o1, n * 8); cudaMallocManaged(&o2, n * 8);
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; in[i] = std::ldexp(1.0 + (s >> 11) * 0x1p-53, (int)(s % 40) - 20); }
  k<<<n / 256, 256>>>(in, o1, o2, n);
  cudaDeviceSynchronize();
  double e1 = 0, e2 = 0;
  for (int i = 0; i < n; ++i) {
    long double t = 1.0L / sqrtl((long double)in[i]);
    e1 = fmax(e1, (double)fabsl((o1[i] - t) / t)); e2 = fmax(e2, (double)fabsl((o2[i] - t) / t));
  }
  printf("max rel err: rsqrt.approx.f64 %.3e (2^%.1f)  rsqrt.approx.ftz.f64 %.3e (2^%.1f)\n", e1, log2(e1), e2, log2(e2));
}
