// Do DMMA (tensor pipe) and DFMA (FP64 pipe) share throughput on B200? Warps 0..K-1 run
// DMMA chains, the others DFMA chains, concurrently on every SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mixed(double* out, int iters, int dmma_warps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s = 0;
  if (warp < dmma_warps) {
    double acc[8][2];
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0;
    double a = 1e-3 * lane, b = 2e-3 * lane;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[q][0]), "+d"(acc[q][1]) : "d"(a), "d"(b));
    }
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  } else {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    // 8 DMMA (2048 FMA/warp) per iteration on the tensor side; match with DFMA: 64 per thread
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
    }
    for (int i = 0; i < 8; ++i) s += x[i];
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000, warps = 8;
  for (int dw : {8, 0, 4, 6, 2}) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mixed<<<sms, warps * 32>>>(out, 100, dw);
    cudaEventRecord(e0);
    mixed<<<sms, warps * 32>>>(out, iters, dw);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per iteration per warp: 8 DMMA x 256 FMA = 2048 FMA; DFMA warp: 64 x 32 = 2048 FMA
    const double flops = 2.0 * 2048.0 * iters * warps * sms;
    printf("dmma warps %d / dfma warps %d: %.3f ms -> %.2f TFLOP/s combined\n", dw, warps - dw, ms,
           flops / ms / 1e9);
  }
  return 0;
}
