// fp64_latency.cu -- dependent-chain latencies on this GPU (one warp, clock64): DFMA, DADD,
// rsqrt.approx.f64, SHFL.IDX, LDS->DFMA. Sizes the serial POTRF pivot chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_latency fp64_latency.cu
#include <cstdio>

__global__ void probe(double* out, long long* cyc, double seed, int iters) {
  __shared__ double sh[64];
  const int lane = threadIdx.x;
  sh[lane] = seed + lane;
  sh[lane + 32] = 0.5;
  __syncwarp();
  double x = seed + lane * 1e-3, y = 1.0000001;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = x + 1e-9;
  t1 = clock64();
  cyc[1] = t1 - t0;
  // rsqrt.approx.f64 chain
  double r = x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double z;
    asm volatile("rsqrt.approx.f64 %0, %1;" : "=d"(z) : "d"(r));
    r = z + 1.0;
  }
  t1 = clock64();
  cyc[2] = t1 - t0;
  // SHFL chain (double)
  double s = x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = __shfl_sync(0xffffffffu, s, (lane + 1) & 31) + 1e-9;
  t1 = clock64();
  cyc[3] = t1 - t0;
  // LDS -> DFMA -> STS chain (through shared memory, one lane's value)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double v = sh[(i + lane) & 31];
    sh[(i + lane + 1) & 31] = fma(v, y, 1e-9);
    __syncwarp();
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  // DMUL + DFMA (div_by-like: 3 dependent ops)
  double a = x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double q = a * 0.999;
    a = fma(fma(-q, 1.001, a), 0.999, q);
  }
  t1 = clock64();
  cyc[5] = t1 - t0;
  out[lane] = x + r + s + sh[lane] + a;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * sizeof(double));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  const int iters = 4096;
  probe<<<1, 32>>>(out, cyc, 1.0, iters);
  probe<<<1, 32>>>(out, cyc, 1.0, iters);
  cudaDeviceSynchronize();
  const char* names[6] = {"DFMA", "DADD", "rsqrt.approx.f64 (+DADD)", "SHFL.IDX f64 (+DADD)",
                          "LDS->DFMA->STS+syncwarp", "div_by (DMUL+2 DFMA)"};
  for (int k = 0; k < 6; ++k)
    std::printf("%-28s %7.1f cycles per dependent step\n", names[k], (double)cyc[k] / iters);
  return 0;
}
