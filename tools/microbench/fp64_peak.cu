// FP64 pipe micro-benchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64).
// Measures sustained FLOP/s of the two FP64 paths the Cholesky trailing
// update can use. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
  const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

template <int SHAPE>
__global__ void dmma_kernel(double* out, int iters) {
  // SHAPE 0: m8n8k4, 1: m16n8k4, 2: m16n8k8, 3: m16n8k16
  const int lane = threadIdx.x & 31;
  double acc[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (lane + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (lane - i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if constexpr (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[q][0]), "+d"(acc[q][1]) : "d"(a[q]), "d"(b[q]));
      } else if constexpr (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[q][0]), "+d"(acc[q][1]), "+d"(acc[q][2]), "+d"(acc[q][3]) : "d"(a[q]), "d"(a[q+4]), "d"(b[q]));
      } else if constexpr (SHAPE == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[q][0]), "+d"(acc[q][1]), "+d"(acc[q][2]), "+d"(acc[q][3])
                     : "d"(a[q]), "d"(a[q+1]), "d"(a[q+2]), "d"(a[q+3]), "d"(b[q]), "d"(b[(q+1)&3]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[q][0]), "+d"(acc[q][1]), "+d"(acc[q][2]), "+d"(acc[q][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j];
  if (s == 12345.0) out[0] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();  // warm-up
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s sms=%d\n", prop.name, sms);
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    int iters = 20000;
    float ms = time_it([&] { dfma_kernel<<<blocks, tpb>>>(out, iters); });
    double flops = 2.0 * 8 * iters * double(blocks) * tpb;
    printf("DFMA tpb=%d blocks=%d: %.3f ms  %.2f TFLOP/s\n", tpb, blocks, ms, flops / ms / 1e9);
  }
  const int shapes_k[4] = {4, 4, 8, 16};
  const int shapes_m[4] = {8, 16, 16, 16};
  for (int s = 0; s < 4; ++s) {
    for (int tpb : {128, 256, 512}) {
      int blocks = sms * 4;
      int iters = 20000;
      float ms;
      if (s == 0) ms = time_it([&] { dmma_kernel<0><<<blocks, tpb>>>(out, iters); });
      else if (s == 1) ms = time_it([&] { dmma_kernel<1><<<blocks, tpb>>>(out, iters); });
      else if (s == 2) ms = time_it([&] { dmma_kernel<2><<<blocks, tpb>>>(out, iters); });
      else ms = time_it([&] { dmma_kernel<3><<<blocks, tpb>>>(out, iters); });
      double flops = 2.0 * shapes_m[s] * 8 * shapes_k[s] * 4.0 * iters * double(blocks) * (tpb / 32);
      printf("DMMA m%dn8k%d tpb=%d: %.3f ms  %.2f TFLOP/s\n", shapes_m[s], shapes_k[s], tpb, ms, flops / ms / 1e9);
    }
  }
  return 0;
}
