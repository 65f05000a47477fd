// Cycle cost of the 16-column row substitution (kernels_chol.cu solve_row16p: X = B D^-T, one
// lane per row, D packed lower in shared memory, quotient = a*r + one FMA correction), one warp
// per CTA, lanes < 16 active as in the TRSM / panel solve:
//   0  as in the kernel (D read from shared memory at each use)
//   1  D preloaded into registers (the dependent chain alone)
//   2  the loads of column c+1 issued before column c's updates (explicit software pipelining)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o solve16 solve16.cu
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ double div_by(double a, double d, double r) {
  const double x0 = a * r;
  return fma(fma(-x0, d, a), r, x0);
}

template <int V>
__device__ __forceinline__ void solve(double (&xr)[16], const double* D, const double* ri) {
  if (V == 1) {
    double Dr[136];
#pragma unroll
    for (int i = 0; i < 136; ++i) Dr[i] = D[i];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      xr[c] = div_by(xr[c], Dr[c * (c + 1) / 2 + c], ri[c]);
#pragma unroll
      for (int c2 = c + 1; c2 < 16; ++c2) xr[c2] -= xr[c] * Dr[c2 * (c2 + 1) / 2 + c];
    }
  } else if (V == 2) {
    double col[16], nxt[16];
    double dd = D[0], rr = ri[0];
#pragma unroll
    for (int c2 = 1; c2 < 16; ++c2) col[c2] = D[c2 * (c2 + 1) / 2];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      double ddn = 0.0, rrn = 0.0;
      if (c < 15) {  // next column's operands first
        ddn = D[(c + 1) * (c + 2) / 2 + c + 1];
        rrn = ri[c + 1];
#pragma unroll
        for (int c2 = c + 2; c2 < 16; ++c2) nxt[c2] = D[c2 * (c2 + 1) / 2 + c + 1];
      }
      xr[c] = div_by(xr[c], dd, rr);
#pragma unroll
      for (int c2 = c + 1; c2 < 16; ++c2) xr[c2] -= xr[c] * col[c2];
      dd = ddn;
      rr = rrn;
#pragma unroll
      for (int c2 = c + 2; c2 < 16; ++c2) col[c2] = nxt[c2];
    }
  } else if (V == 3) {
    // the next column's division started right after its one dependent update; the remaining
    // updates of column c fill the division's latency (same operations, same order per element)
    double x0 = xr[0] * ri[0];
    double q = fma(fma(-x0, D[0], xr[0]), ri[0], x0);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      xr[c] = q;
      double e = 0.0, xn = 0.0;
      if (c < 15) {
        const int cn = c + 1;
        xr[cn] -= q * D[cn * (cn + 1) / 2 + c];
        xn = xr[cn] * ri[cn];
        e = fma(-xn, D[cn * (cn + 1) / 2 + cn], xr[cn]);
      }
#pragma unroll
      for (int c2 = c + 2; c2 < 16; ++c2) xr[c2] -= q * D[c2 * (c2 + 1) / 2 + c];
      if (c < 15) q = fma(e, ri[c + 1], xn);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      xr[c] = div_by(xr[c], D[c * (c + 1) / 2 + c], ri[c]);
#pragma unroll
      for (int c2 = c + 1; c2 < 16; ++c2) xr[c2] -= xr[c] * D[c2 * (c2 + 1) / 2 + c];
    }
  }
}

template <int V>
__global__ void bench(const double* in, double* out, long long* cyc, int reps) {
  __shared__ double D[136];
  __shared__ double ri[16];
  const int lane = threadIdx.x;
  for (int i = lane; i < 136; i += 32) D[i] = 1.0 + 0.01 * (i % 7);
  if (lane < 16) ri[lane] = 1.0 / D[lane * (lane + 1) / 2 + lane];
  __syncwarp();
  double acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = 0.0;
  double base[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) base[c] = in[(lane & 15) * 16 + c];
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    if (lane < 16) {
      double xr[16];
      const double jt = it * 1e-12;
#pragma unroll
      for (int c = 0; c < 16; ++c) xr[c] = base[c] + jt;
      solve<V>(xr, D, ri);
#pragma unroll
      for (int c = 0; c < 16; ++c) acc[c] += xr[c];
    }
    __syncwarp();
  }
  long long t1 = clock64();
  double sum = 0.0;
#pragma unroll
  for (int c = 0; c < 16; ++c) sum += acc[c];
  out[lane] = sum;
  if (lane == 0) cyc[0] = (t1 - t0) / reps;
}

// dependent DFMA chain latency (cycles per FMA)
__global__ void fma_chain(double* out, long long* cyc, int n) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x = fma(x, 1.0000001, 1e-9);
    x = fma(x, 0.9999999, -1e-9);
    x = fma(x, 1.0000001, 1e-9);
    x = fma(x, 0.9999999, -1e-9);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / (4 * n);
}

int main() {
  double *in, *out;
  long long* cyc;
  cudaMalloc(&in, 256 * 8);
  cudaMalloc(&out, 32 * 8);
  cudaMalloc(&cyc, 8);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = 0.3 * ((i * 37) % 17) / 17.0;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  long long hc;
  double a[32], b[32];
  const char* names[] = {"as in kernel", "D in registers", "software-pipelined loads", "next division first"};
#define RUN(V)                                                               \
  bench<V><<<1, 32>>>(in, out, cyc, 200);                                    \
  bench<V><<<1, 32>>>(in, out, cyc, 2000);                                   \
  cudaDeviceSynchronize();                                                   \
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);                           \
  cudaMemcpy(V == 0 ? a : b, out, 32 * 8, cudaMemcpyDeviceToHost);           \
  printf("variant %d (%s): %lld cycles per 16-column substitution%s\n", V, names[V], hc, \
         V == 0 ? "" : (memcmp(a, b, 16 * 8) == 0 ? " (bitwise equal)" : " (DIFFERS)"));
  RUN(0) RUN(1) RUN(2) RUN(3)
  fma_chain<<<1, 32>>>(out, cyc, 1000);
  fma_chain<<<1, 32>>>(out, cyc, 10000);
  cudaDeviceSynchronize();
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent DFMA: %lld cycles each\n", hc);
  return 0;
}
