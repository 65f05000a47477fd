// Cycle cost of the DIAG pivot block as the kernel runs it (kernels_chol.cu potrf_row16, round 2:
// shared-memory quotient broadcast, no compare/select on the pivot chain) and variants aimed at
// the chain that is left between one column's quotient and the next one's:
//   0  as in the kernel
//   1  column c+1's update of every lane's xr[c+1] from a shuffle of lane c+1's quotient
//      (issued next to the pivot shuffle) instead of the shared-memory round trip
//   2  as 1, with the lane index pinned in a register (no S2R rematerialisation in the loop)
//   3  chain only: pivot shuffle -> root -> quotient -> next pivot (wrong values, lower bound)
// Every variant except 3 is checked bitwise against variant 0.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o potrf16b potrf16b.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double div_by(double a, double d, double r) {
  const double x0 = a * r;
  return fma(fma(-x0, d, a), r, x0);
}
__device__ __forceinline__ void pivot_root(double s, double& d, double& r) {
  double y;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(s));
  const double d0 = s * y;
  d = fma(fma(-d0, d0, s), 0.5 * y, d0);
  r = y;
}

template <int V>
__device__ __forceinline__ bool potrf_row16(double (&xr)[16], double* rinv, int lane, double* qs) {
  double d, r;
  const double s = __shfl_sync(0xffffffffu, xr[0], 0);
  bool ok = s > 0.0;
  pivot_root(s, d, r);
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const double q = div_by(xr[c], d, r);
    if (V != 3 && lane == c) rinv[c] = r;
    if (V != 3) xr[c] = lane > c ? q : (lane == c ? d : xr[c]);
    double qn = 0.0;
    if (c < 15) {
      const double sn = __shfl_sync(0xffffffffu, fma(-q, q, xr[c + 1]), c + 1);
      if (V == 1 || V == 2) qn = __shfl_sync(0xffffffffu, q, c + 1);
      ok = ok && sn > 0.0;
      pivot_root(sn, d, r);
    }
    if (V == 3) {
      if (c < 15) xr[c + 1] = fma(-q, q, xr[c + 1]);
      continue;
    }
    if (lane < 16) qs[16 * (c & 1) + lane] = q;
    __syncwarp();
    if ((V == 1 || V == 2) && c < 15) xr[c + 1] = fma(-q, qn, xr[c + 1]);
#pragma unroll
    for (int c2 = c + 1; c2 < 16; ++c2) {
      if ((V == 1 || V == 2) && c2 == c + 1) continue;
      xr[c2] = fma(-q, qs[16 * (c & 1) + c2], xr[c2]);
    }
  }
  return ok;
}

template <int V>
__global__ void bench(const double* in, double* out, long long* cyc, int reps) {
  __shared__ double rinv[16];
  __shared__ __align__(16) double qs[32];
  int lane = threadIdx.x;
  if (V == 2) asm volatile("mov.u32 %0, %0;" : "+r"(lane));
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    double xr[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) xr[c] = in[(lane & 15) * 16 + c] + (c == (lane & 15) ? 16.0 + it * 1e-9 : 0.0);
    potrf_row16<V>(xr, rinv, lane, qs);
#pragma unroll
    for (int c = 0; c < 16; ++c) acc += (c <= (lane & 15)) ? xr[c] : 0.0;
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
  const char* names[] = {"as in kernel", "xr[c+1] update by shuffle", "as 1, lane pinned", "chain only"};
  double ref[32], got[32];
#define RUN(V)                                                                               \
  bench<V><<<1, 32>>>(in, out, cyc, 200);                                                    \
  bench<V><<<1, 32>>>(in, out, cyc, 2000);                                                   \
  cudaDeviceSynchronize();                                                                   \
  cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);                                            \
  bench<V><<<1, 32>>>(in, out, cyc, 7);                                                      \
  cudaMemcpy(V == 0 ? ref : got, out, 32 * 8, cudaMemcpyDeviceToHost);                       \
  {                                                                                          \
    int same = 1;                                                                            \
    for (int i = 0; i < 16; ++i) same &= (V == 0 ? ref[i] : got[i]) == ref[i];               \
    printf("variant %d (%s): %lld cycles per 16x16 pivot block, bitwise %d\n", V, names[V], \
           hc[0], same);                                                                     \
  }
  RUN(0) RUN(1) RUN(2) RUN(3)
  return 0;
}
