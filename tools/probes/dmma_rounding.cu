// dmma_rounding.cu -- how DMMA.8x8x4 (mma.sync m8n8k4 f64) rounds its four products: compared
// bit for bit with sequential FMA chains in k order 0..3 and 3..0 on random operands with heavy
// cancellation. Decides whether a DMMA update can be restated as per-lane DFMAs bitwise.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_rounding dmma_rounding.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void probe(const double* A, const double* B, const double* C, int trials, int* counts) {
  const int lane = threadIdx.x;
  const int r = lane >> 2, q = lane & 3;
  int same_fwd = 0, same_rev = 0, n = 0;
  for (int t = 0; t < trials; ++t) {
    const double* At = A + t * 32;  // [8][4] row-major
    const double* Bt = B + t * 32;  // [4][8] row-major (k, n)
    const double* Ct = C + t * 64;  // [8][8]
    double c0 = Ct[r * 8 + 2 * q], c1 = Ct[r * 8 + 2 * q + 1];
    const double a = At[r * 4 + q], b = Bt[q * 8 + r];
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
    for (int e = 0; e < 2; ++e) {
      const int col = 2 * q + e;
      double f = Ct[r * 8 + col], g = Ct[r * 8 + col];
      for (int k = 0; k < 4; ++k) f = fma(At[r * 4 + k], Bt[k * 8 + col], f);
      for (int k = 3; k >= 0; --k) g = fma(At[r * 4 + k], Bt[k * 8 + col], g);
      const double dv = e ? c1 : c0;
      same_fwd += dv == f;
      same_rev += dv == g;
      ++n;
    }
  }
  atomicAdd(&counts[0], same_fwd);
  atomicAdd(&counts[1], same_rev);
  atomicAdd(&counts[2], n);
}

int main() {
  const int T = 20000;
  double *hA = (double*)malloc(T * 32 * 8), *hB = (double*)malloc(T * 32 * 8), *hC = (double*)malloc(T * 64 * 8);
  srand(7);
  auto rnd = []() { return (rand() / (double)RAND_MAX - 0.5) * (1 + (rand() % 1000) / 7.0); };
  for (int i = 0; i < T * 32; ++i) { hA[i] = rnd(); hB[i] = rnd(); }
  for (int i = 0; i < T * 64; ++i) hC[i] = rnd() * 3;
  double *A, *B, *C;
  int* cnt;
  cudaMalloc(&A, T * 32 * 8); cudaMalloc(&B, T * 32 * 8); cudaMalloc(&C, T * 64 * 8); cudaMalloc(&cnt, 12);
  cudaMemcpy(A, hA, T * 32 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, T * 32 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(C, hC, T * 64 * 8, cudaMemcpyHostToDevice);
  cudaMemset(cnt, 0, 12);
  probe<<<1, 32>>>(A, B, C, T, cnt);
  int h[3];
  cudaMemcpy(h, cnt, 12, cudaMemcpyDeviceToHost);
  printf("DMMA vs sequential FMA k=0..3: %d / %d equal; k=3..0: %d / %d equal\n", h[0], h[2], h[1], h[2]);
  return 0;
}
