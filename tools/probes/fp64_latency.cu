// fp64_latency.cu -- dependent-chain latencies on this GPU (one warp, clock64): DFMA, DADD,
// rsqrt.approx.f64, SHFL.IDX, LDS->DFMA, DMMA. Sizes the serial POTRF pivot chain.
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
  // DMMA m8n8k4 chain (accumulator dependency)
  double c0 = x, c1 = y, av = 1e-3 * lane, bv = 1e-3;
  t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1) : "d"(av), "d"(bv));
  t1 = clock64();
  cyc[6] = t1 - t0;
  // 4 independent DMMA chains (per-warp issue rate)
  double e0 = x, e1 = y, f0 = x, f1 = y, g0 = x, g1 = y, h0 = x, h1 = y;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(e0), "+d"(e1) : "d"(av), "d"(bv));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(f0), "+d"(f1) : "d"(av), "d"(bv));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(g0), "+d"(g1) : "d"(av), "d"(bv));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(h0), "+d"(h1) : "d"(av), "d"(bv));
  }
  t1 = clock64();
  cyc[7] = t1 - t0;
  out[lane] = x + r + s + sh[lane] + a + c0 + c1 + e0 + f1 + g0 + h1;
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
  const char* names[8] = {"DFMA", "DADD", "rsqrt.approx.f64 (+DADD)", "SHFL.IDX f64 (+DADD)",
                          "LDS->DFMA->STS+syncwarp", "div_by (DMUL+2 DFMA)", "DMMA m8n8k4 chain",
                          "DMMA, 4 independent chains"};
  for (int k = 0; k < 8; ++k)
    std::printf("%-28s %7.1f cycles per dependent step\n", names[k], (double)cyc[k] / iters);
  return 0;
}
