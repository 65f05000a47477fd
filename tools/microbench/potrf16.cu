// Cycle cost of the DIAG pivot block (kernels_chol.cu potrf_row16: 16x16 Cholesky, one lane per
// row, register-only) and of the panel substitution (solve_row16), one warp per CTA, with
// variants that remove one ingredient at a time to find the critical path:
//   0  as in the kernel
//   1  no update shuffles (each lane updates with its own quotient: wrong values, same chain)
//   2  quotient = a * r (no FMA residual correction)
//   3  pivot root: d = s * y, no Markstein step
//   4  update quotients broadcast through shared memory (one STS per lane, LDS.64 broadcasts)
//   5  as 4 with LDS.128 (two quotients per load)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o potrf16 potrf16.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double div_by(double a, double d, double r) {
  const double x0 = a * r;
  return fma(fma(-x0, d, a), r, x0);
}

template <int V>
__device__ __forceinline__ void pivot_root(double s, double& d, double& r) {
  double y;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(s));
  const double d0 = s * y;
  d = V == 3 ? d0 : fma(fma(-d0, d0, s), 0.5 * y, d0);
  r = y;
}

template <int V>
__device__ __forceinline__ bool potrf_row16(double (&xr)[16], double* rinv, int lane, double* qs) {
  double d, r;
  double s = __shfl_sync(0xffffffffu, xr[0], 0);
  bool ok = s > 0.0;
  if (!ok) s = 1.0;
  pivot_root<V>(s, d, r);
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const double q = V == 2 ? xr[c] * r : div_by(xr[c], d, r);
    if (lane == c) rinv[c] = r;
    xr[c] = lane > c ? q : (lane == c ? d : xr[c]);
    if (c < 15) {
      double sn = __shfl_sync(0xffffffffu, fma(-q, q, xr[c + 1]), c + 1);
      ok = ok && sn > 0.0;
      if (!ok) sn = 1.0;
      pivot_root<V>(sn, d, r);
    }
    if (V >= 4) {
      if (lane < 16) qs[16 * (c & 1) + lane] = q;  // double-buffered by column parity
      __syncwarp();
      const double* qc = qs + 16 * (c & 1);
      if (V == 4) {
#pragma unroll
        for (int c2 = c + 1; c2 < 16; ++c2) xr[c2] = fma(-q, qc[c2], xr[c2]);
      } else {
#pragma unroll
        for (int c2 = c + 1; c2 < 16; ++c2) {
          if (((c2 & 1) == 0) && c2 + 1 < 16) {
            const double2 v = *reinterpret_cast<const double2*>(qc + c2);
            xr[c2] = fma(-q, v.x, xr[c2]);
            xr[c2 + 1] = fma(-q, v.y, xr[c2 + 1]);
          } else if ((c2 & 1) == 1 && c2 == c + 1) {
            xr[c2] = fma(-q, qc[c2], xr[c2]);
          }
        }
      }
    } else {
#pragma unroll
      for (int c2 = c + 1; c2 < 16; ++c2)
        xr[c2] = fma(-q, V == 1 ? q : __shfl_sync(0xffffffffu, q, c2), xr[c2]);
    }
  }
  return ok;
}

template <int V>
__global__ void bench(const double* in, double* out, long long* cyc, int reps) {
  __shared__ double rinv[16];
  __shared__ __align__(16) double qs[32];
  const int lane = threadIdx.x;
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    double xr[16];
    // an SPD block: diagonally dominant, lane = row
#pragma unroll
    for (int c = 0; c < 16; ++c) xr[c] = in[(lane & 15) * 16 + c] + (c == (lane & 15) ? 16.0 + it * 1e-9 : 0.0);
    potrf_row16<V>(xr, rinv, lane, qs);
#pragma unroll
    for (int c = 0; c < 16; ++c) acc += xr[c];
  }
  long long t1 = clock64();
  out[blockIdx.x * 32 + lane] = acc;
  if (lane == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

int main() {
  double *in, *out;
  long long* cyc;
  cudaMalloc(&in, 256 * 8);
  cudaMalloc(&out, 148 * 32 * 8);
  cudaMalloc(&cyc, 148 * 8);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = 0.01 * ((i * 37) % 17) / 17.0;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  long long hc[1];
  const char* names[] = {"as in kernel", "no update shuffles", "quotient a*r", "no Markstein", "smem LDS.64",
                         "smem LDS.128"};
#define RUN(V)                                                            \
  bench<V><<<1, 32>>>(in, out, cyc, 200);                                 \
  bench<V><<<1, 32>>>(in, out, cyc, 2000);                                \
  cudaDeviceSynchronize();                                                \
  cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);                         \
  printf("variant %d (%s): %lld cycles per 16x16 pivot block\n", V, names[V], hc[0]);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5)
  // parity of the smem variants against the shuffle version (same operations, same order)
  {
    double a[148 * 32], b[148 * 32];
    bench<0><<<1, 32>>>(in, out, cyc, 7);
    cudaMemcpy(a, out, 32 * 8, cudaMemcpyDeviceToHost);
    bench<5><<<1, 32>>>(in, out, cyc, 7);
    cudaMemcpy(b, out, 32 * 8, cudaMemcpyDeviceToHost);
    int same = 1;
    for (int i = 0; i < 16; ++i) same &= a[i] == b[i];
    printf("variant 5 bitwise equal to variant 0: %d\n", same);
  }
  return 0;
}
