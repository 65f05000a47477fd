// kernels_predict.cu -- K4: batched kriging prediction (BLUP) and MSE on sm_100a.
//
// Reference: predictor.hpp:20-50 (relative to /root/reference/proj/include/gpemu/)
//   yhat_j = mu_hat + dot_accumulate(r(x_j), alpha),  r_i = corr_vector (correlation.hpp:67-91)
// The reference has no predictive variance; the MSE here is the
// constant-mean kriging variance s2 = sigma2 (1 - w'w + (1 - v'w)^2 / v'v),
// w = L^-1 r, v = L^-1 1, checked against oracle/ (parity unpinned).
//
// yhat: each CTA owns kPts test points; training points are staged through
// shared memory in chunks of 256 (x_i and alpha_i), every thread evaluates
// d exp/log pairs + one exp per (test, train) pair and keeps kPts partial dots;
// a fixed-order block reduction finishes each dot (deterministic).
#include <cuda_runtime.h>

#include "kernels.h"
#include "layout.cuh"

namespace gpemu_dev {

constexpr int kPts = 16;
constexpr int kTrainChunk = 256;

__device__ __forceinline__ double pow_abs_p(double delta, double p) {
  if (delta == 0.0) return 0.0;
  const double a = delta < 0.0 ? -delta : delta;
  return exp(__dmul_rn(p, log(a)));
}

__global__ void __launch_bounds__(256) predict_kernel(const double* __restrict__ Xt, int N,
                                                      const double* __restrict__ X, int n, int d,
                                                      const double* __restrict__ theta, double p,
                                                      double mu, const double* __restrict__ alpha,
                                                      double* __restrict__ yhat, int* bad) {
  extern __shared__ double dyn[];
  double* xs = dyn;                          // [kTrainChunk][d]
  double* as = xs + kTrainChunk * d;         // [kTrainChunk]
  double* ts = as + kTrainChunk;             // [kPts][d]
  double* th = ts + kPts * d;                // [d]
  __shared__ double red[kPts][256 / 32];
  const int j0 = blockIdx.x * kPts;
  const int np = min(kPts, N - j0);
  for (int q = threadIdx.x; q < kPts * d; q += blockDim.x) {
    const int pj = q / d, k = q - pj * d;
    ts[pj * d + k] = pj < np ? Xt[(size_t)(j0 + pj) * d + k] : 0.0;
  }
  for (int k = threadIdx.x; k < d; k += blockDim.x) th[k] = theta[k];
  double acc[kPts];
#pragma unroll
  for (int pj = 0; pj < kPts; ++pj) acc[pj] = 0.0;
  for (int c0 = 0; c0 < n; c0 += kTrainChunk) {
    const int cn = min(kTrainChunk, n - c0);
    __syncthreads();
    for (int q = threadIdx.x; q < cn * d; q += blockDim.x) {
      const int i = q / d, k = q - i * d;
      xs[i * d + k] = X[(size_t)(c0 + i) * d + k];
    }
    for (int q = threadIdx.x; q < cn; q += blockDim.x) as[q] = alpha[c0 + q];
    __syncthreads();
    const int i = threadIdx.x;
    if (i < cn) {
      const double ai = as[i];
#pragma unroll
      for (int pj = 0; pj < kPts; ++pj) {
        if (pj < np) {
          double s = 0.0;
          for (int k = 0; k < d; ++k) {
            const double term = pow_abs_p(ts[pj * d + k] - xs[i * d + k], p);
            s = __dadd_rn(s, __dmul_rn(th[k], term));
          }
          const double r = exp(-s);
          if (!isfinite(r)) *bad = 1;
          acc[pj] = fma(r, ai, acc[pj]);
        }
      }
    }
  }
  // deterministic block reduction: warp shuffle tree, then warps in order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int pj = 0; pj < kPts; ++pj) {
    double v = acc[pj];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0) red[pj][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < np) {
    double s = 0.0;
    for (int w = 0; w < 256 / 32; ++w) s += red[threadIdx.x][w];
    yhat[j0 + threadIdx.x] = mu + s;
  }
}

void launch_predict(const double* Xt, int N, const double* X, int n, int d, const double* theta,
                    double p, double mu, const double* alpha, double* yhat, int* bad,
                    cudaStream_t s) {
  if (N <= 0) return;
  const size_t smem = ((size_t)kTrainChunk * d + kTrainChunk + (size_t)kPts * d + d) * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  predict_kernel<<<(N + kPts - 1) / kPts, 256, smem, s>>>(Xt, N, X, n, d, theta, p, mu, alpha,
                                                          yhat, bad);
}

// MSE, one CTA per test point: r into shared memory, column-oriented forward
// substitution w = L^-1 r on the tiled factor, then w'w and v'w.
__global__ void __launch_bounds__(512) mse_point_kernel(const double* __restrict__ Xt,
                                                        const double* __restrict__ X, int n, int d,
                                                        const double* __restrict__ theta, double p,
                                                        double sigma2,
                                                        const double* __restrict__ tiles,
                                                        const double* __restrict__ v, double vtv,
                                                        double* __restrict__ mse, int* bad) {
  extern __shared__ double w[];
  __shared__ double red[2][16];
  const int j = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double term = pow_abs_p(Xt[(size_t)j * d + k] - X[(size_t)i * d + k], p);
      s = __dadd_rn(s, __dmul_rn(theta[k], term));
    }
    const double r = exp(-s);
    if (!isfinite(r)) *bad = 1;
    w[i] = r;
  }
  __syncthreads();
  auto Lat = [&](int i, int c) {
    return tiles[tile_index(i >> 7, c >> 7) * TILE_ELEMS + elem_off(i & 127, c & 127)];
  };
  for (int k = 0; k < n; ++k) {
    const double xk = w[k] / Lat(k, k);
    __syncthreads();
    for (int l = k + 1 + threadIdx.x; l < n; l += blockDim.x) w[l] -= Lat(l, k) * xk;
    if (threadIdx.x == 0) w[k] = xk;
    __syncthreads();
  }
  double wtw = 0.0, vtw = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    wtw = fma(w[i], w[i], wtw);
    vtw = fma(v[i], w[i], vtw);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = 16; off > 0; off >>= 1) {
    wtw += __shfl_down_sync(0xffffffffu, wtw, off);
    vtw += __shfl_down_sync(0xffffffffu, vtw, off);
  }
  if (lane == 0) {
    red[0][warp] = wtw;
    red[1][warp] = vtw;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      a += red[0][q];
      b += red[1][q];
    }
    const double one_minus = 1.0 - b;
    double s2 = sigma2 * (1.0 - a + one_minus * one_minus / vtv);
    mse[j] = s2 < 0.0 ? 0.0 : s2;
  }
}

void launch_predict_mse(const double* Xt, int N, const double* X, int n, int d,
                        const double* theta, double p, double sigma2, const double* tiles, int NT,
                        const double* v, double vtv, double* work, double* mse, int* bad,
                        cudaStream_t s) {
  (void)NT;
  (void)work;
  if (N <= 0) return;
  const size_t smem = (size_t)n * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(mse_point_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mse_point_kernel<<<N, 512, smem, s>>>(Xt, X, n, d, theta, p, sigma2, tiles, v, vtv, mse, bad);
}

}  // namespace gpemu_dev

namespace gpemu_dev {

// ---------------------------------------------------------------------------
// MSE at scale: test points become extra row tiles below the factor. The DAG engine in
// extension mode turns each row of cross-correlations r into w = L^-1 r with DMMA tiles
// (the same OFF-task path as the factorization), then one warp per point reduces its row.

// Cross-correlation tile (It, J): rows = test points It*128 + r, cols = design points
// J*128 + c; corr_vector arithmetic (correlation.hpp:84-87): sequential k, no FMA.
__global__ void __launch_bounds__(256) cross_tiles_kernel(const double* __restrict__ Xt, int N,
                                                          const double* __restrict__ X, int n,
                                                          int d, const double* __restrict__ theta,
                                                          double p, int NT,
                                                          double* __restrict__ ext, int* bad) {
  extern __shared__ double sm[];
  double* xt = sm;                 // [128][d]
  double* xs = xt + TILE * d;      // [128][d]
  double* th = xs + TILE * d;      // [d]
  const int tile = blockIdx.x;
  const int It = tile / NT, J = tile - It * NT;
  for (int q = threadIdx.x; q < TILE * d; q += blockDim.x) {
    const int r = q / d, k = q - r * d;
    const int pt = It * TILE + r, pi = J * TILE + r;
    xt[q] = pt < N ? Xt[(size_t)pt * d + k] : 0.0;
    xs[q] = pi < n ? X[(size_t)pi * d + k] : 0.0;
  }
  for (int k = threadIdx.x; k < d; k += blockDim.x) th[k] = theta[k];
  __syncthreads();
  double* out = ext + (size_t)tile * TILE_ELEMS;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < TILE_ELEMS; e += gridDim.y * blockDim.x) {
    int r, c;
    elem_rc(e, r, c);
    double v = 0.0;
    if (It * TILE + r < N && J * TILE + c < n) {
      double s = 0.0;
      for (int k = 0; k < d; ++k)
        s = __dadd_rn(s, __dmul_rn(th[k], pow_abs_p(xt[r * d + k] - xs[c * d + k], p)));
      v = exp(-s);
      if (!isfinite(v)) *bad = 1;
    }
    out[e] = v;
  }
}

void launch_cross_tiles(const double* Xt, int N, const double* X, int n, int d,
                        const double* theta, double p, int NT, int RT, double* ext, int* bad,
                        cudaStream_t s) {
  const size_t smem = (2 * (size_t)TILE * d + d) * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(cross_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cross_tiles_kernel<<<dim3(RT * NT, 4), 256, smem, s>>>(Xt, N, X, n, d, theta, p, NT, ext, bad);
}

// One warp per test point: fixed-order lane partials + shuffle tree (deterministic).
__global__ void __launch_bounds__(256) ext_reduce_kernel(const double* __restrict__ ext, int N,
                                                         int n, int NT,
                                                         const double* __restrict__ u,
                                                         const double* __restrict__ v, double mu,
                                                         double sigma2, double vtv,
                                                         double* __restrict__ yhat,
                                                         double* __restrict__ mse) {
  const int lane = threadIdx.x & 31;
  const int pt = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (pt >= N) return;
  const int It = pt >> 7, r = pt & 127;
  double ww = 0.0, vw = 0.0, yw = 0.0;
  for (int J = 0; J < NT; ++J) {
    const double* tl = ext + ((size_t)It * NT + J) * TILE_ELEMS;
#pragma unroll
    for (int sl = 0; sl < SLABS_PER_TILE; ++sl) {
      const int c = sl * SLAB + lane;
      const int col = J * TILE + c;
      if (col < n) {
        const double w = tl[elem_off(r, c)];
        ww = fma(w, w, ww);
        vw = fma(v[col], w, vw);
        yw = fma(u[col] - mu * v[col], w, yw);
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    ww += __shfl_xor_sync(0xffffffffu, ww, off);
    vw += __shfl_xor_sync(0xffffffffu, vw, off);
    yw += __shfl_xor_sync(0xffffffffu, yw, off);
  }
  if (lane == 0) {
    if (yhat) yhat[pt] = mu + yw;
    if (mse) {
      const double a = 1.0 - vw;
      const double s2 = sigma2 * (1.0 - ww + a * a / vtv);
      mse[pt] = s2 < 0.0 ? 0.0 : s2;
    }
  }
}

void launch_ext_reduce(const double* ext, int N, int n, int NT, const double* u, const double* v,
                       double mu, double sigma2, double vtv, double* yhat, double* mse,
                       cudaStream_t s) {
  ext_reduce_kernel<<<(N + 7) / 8, 256, 0, s>>>(ext, N, n, NT, u, v, mu, sigma2, vtv, yhat, mse);
}

}  // namespace gpemu_dev
