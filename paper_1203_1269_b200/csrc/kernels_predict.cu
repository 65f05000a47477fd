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

#include "fastmath.cuh"
#include "kernels.h"
#include "layout.cuh"

namespace gpemu_dev {

constexpr int kPredThreads = 128;
constexpr int kTrainBlock = 1024;  // training rows per partial dot (fixed: bits independent of N)
constexpr int kTrainStage = 128;   // rows staged in shared memory at a time

__device__ __forceinline__ double pow_abs_p(double delta, double p) { return pow_abs_fast(delta, p); }

// yhat_j = mu + sum_i r_i(x_j) alpha_i (predictor.hpp:36-44): one thread per test point,
// ascending i (dot_accumulate, matrix.hpp:64-69) inside each 128-row tile; tile partials are
// added in order inside fixed kTrainBlock blocks (blockIdx.y), each block's partial goes to
// part[blk][j] and predict_combine adds them in block order. The order is independent of N
// and identical to yhat_tiles_kernel's (the MSE path), so yhat is the same bits either way. Staged
// training rows are read by every thread at the same address (shared-memory broadcast);
// MAXD unrolls the d pow terms so they interleave (fastmath.cuh is branch-free).
template <int MAXD>
__global__ void __launch_bounds__(kPredThreads, 4) predict_kernel(
    const double* __restrict__ Xt, int N, const double* __restrict__ X, int n, int d,
    const double* __restrict__ theta, double p, const double* __restrict__ alpha,
    double* __restrict__ part, int* bad) {
  __shared__ double xs[kTrainStage][MAXD];
  __shared__ double as[kTrainStage];
  const int j = blockIdx.x * kPredThreads + threadIdx.x;
  const int jc = min(j, N - 1);
  double xt[MAXD], th[MAXD];
#pragma unroll
  for (int k = 0; k < MAXD; ++k) {
    xt[k] = k < d ? Xt[(size_t)jc * d + k] : 0.0;
    th[k] = k < d ? theta[k] : 0.0;  // zero terms leave the sequential sum unchanged
  }
  const int i0 = blockIdx.y * kTrainBlock, i1 = min(n, i0 + kTrainBlock);
  double acc = 0.0;
  bool nonfinite = false;
  for (int c0 = i0; c0 < i1; c0 += kTrainStage) {
    const int cn = min(kTrainStage, i1 - c0);
    __syncthreads();
    for (int q = threadIdx.x; q < kTrainStage * MAXD; q += kPredThreads) {
      const int r = q / MAXD, k = q - r * MAXD;
      xs[r][k] = (r < cn && k < d) ? X[(size_t)(c0 + r) * d + k] : 0.0;
    }
    for (int q = threadIdx.x; q < kTrainStage; q += kPredThreads) as[q] = q < cn ? alpha[c0 + q] : 0.0;
    __syncthreads();
    double tacc = 0.0;  // this 128-row tile's partial (yhat_tiles_kernel uses the same order)
    for (int r = 0; r < cn; ++r) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < MAXD; ++k) s = __dadd_rn(s, __dmul_rn(th[k], pow_abs_p(xt[k] - xs[r][k], p)));
      const double v = exp_neg(s);
      nonfinite |= !isfinite(v) || isnan(s);
      tacc = fma(v, as[r], tacc);
    }
    acc = __dadd_rn(acc, tacc);
  }
  if (j < N) {
    part[(size_t)blockIdx.y * N + j] = acc;
    if (nonfinite) *bad = 1;
  }
}

// Any d (the d > 32 path): predict_kernel's arithmetic and summation order, coordinates and
// theta read from global memory (the training row is the same address across the block).
__global__ void __launch_bounds__(kPredThreads) predict_generic_kernel(
    const double* __restrict__ Xt, int N, const double* __restrict__ X, int n, int d,
    const double* __restrict__ theta, double p, const double* __restrict__ alpha,
    double* __restrict__ part, int* bad) {
  const int j = blockIdx.x * kPredThreads + threadIdx.x;
  const int jc = min(j, N - 1);
  const double* xt = Xt + (size_t)jc * d;
  const int i0 = blockIdx.y * kTrainBlock, i1 = min(n, i0 + kTrainBlock);
  double acc = 0.0;
  bool nonfinite = false;
  for (int c0 = i0; c0 < i1; c0 += kTrainStage) {
    const int cn = min(kTrainStage, i1 - c0);
    double tacc = 0.0;
    for (int r = 0; r < cn; ++r) {
      const double* xr = X + (size_t)(c0 + r) * d;
      double s = 0.0;
      for (int k = 0; k < d; ++k) s = __dadd_rn(s, __dmul_rn(__ldg(theta + k), pow_abs_p(xt[k] - __ldg(xr + k), p)));
      const double v = exp_neg(s);
      nonfinite |= !isfinite(v) || isnan(s);
      tacc = fma(v, __ldg(alpha + c0 + r), tacc);
    }
    acc = __dadd_rn(acc, tacc);
  }
  if (j < N) {
    part[(size_t)blockIdx.y * N + j] = acc;
    if (nonfinite) *bad = 1;
  }
}

__global__ void predict_combine_kernel(const double* __restrict__ part, int N, int nblk, double mu,
                                       double* __restrict__ yhat) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  double s = part[j];
  for (int b = 1; b < nblk; ++b) s += part[(size_t)b * N + j];
  yhat[j] = mu + s;
}

int predict_blocks(int n) { return (n + kTrainBlock - 1) / kTrainBlock; }

template <int MAXD>
static void launch_pred(dim3 grid, cudaStream_t s, const double* Xt, int N, const double* X, int n,
                        int d, const double* theta, double p, const double* alpha, double* part,
                        int* bad) {
  predict_kernel<MAXD><<<grid, kPredThreads, 0, s>>>(Xt, N, X, n, d, theta, p, alpha, part, bad);
}

// part: predict_blocks(n) * N doubles of scratch.
void launch_predict(const double* Xt, int N, const double* X, int n, int d, const double* theta,
                    double p, double mu, const double* alpha, double* part, double* yhat, int* bad,
                    cudaStream_t s) {
  if (N <= 0) return;
  const int nblk = predict_blocks(n);
  const dim3 grid((N + kPredThreads - 1) / kPredThreads, nblk);
#define GPEMU_PRED(D) launch_pred<D>(grid, s, Xt, N, X, n, d, theta, p, alpha, part, bad)
  if (d <= 1) GPEMU_PRED(1);
  else if (d <= 2) GPEMU_PRED(2);
  else if (d <= 3) GPEMU_PRED(3);
  else if (d <= 4) GPEMU_PRED(4);
  else if (d <= 6) GPEMU_PRED(6);
  else if (d <= 8) GPEMU_PRED(8);
  else if (d <= 10) GPEMU_PRED(10);
  else if (d <= 12) GPEMU_PRED(12);
  else if (d <= 16) GPEMU_PRED(16);
  else if (d <= 20) GPEMU_PRED(20);
  else if (d <= 24) GPEMU_PRED(24);
  else if (d <= 32) GPEMU_PRED(32);
  else predict_generic_kernel<<<grid, kPredThreads, 0, s>>>(Xt, N, X, n, d, theta, p, alpha, part, bad);
#undef GPEMU_PRED
  predict_combine_kernel<<<(N + 255) / 256, 256, 0, s>>>(part, N, nblk, mu, yhat);
}

}  // namespace gpemu_dev

namespace gpemu_dev {

// ---------------------------------------------------------------------------
// MSE at scale: test points become extra row tiles below the factor. The DAG engine in
// extension mode turns each row of cross-correlations r into w = L^-1 r with DMMA tiles
// (the same OFF-task path as the factorization), then one warp per point reduces its row.

// Cross-correlation tile (It, J): rows = test points It*128 + r, cols = design points
// J*128 + c; corr_vector arithmetic (correlation.hpp:84-87): sequential k, no FMA. Design
// coordinates are staged [k][c] (consecutive c across a warp: conflict-free), test
// coordinates [r][k] (one r per warp row: broadcast); padding rows/cols are computed on
// clamped coordinates and written as 0, so the MAXD-unrolled body has no branches.
template <int MAXD>
__global__ void __launch_bounds__(256) cross_tiles_kernel(const double* __restrict__ Xt, int N,
                                                          const double* __restrict__ X, int n,
                                                          int d, const double* __restrict__ theta,
                                                          double p, int NT,
                                                          double* __restrict__ ext, int* bad) {
  extern __shared__ double cross_sm[];  // xt[TILE][MAXD], xs[MAXD][TILE], th[MAXD]
  double(*xt)[MAXD] = reinterpret_cast<double(*)[MAXD]>(cross_sm);
  double(*xs)[TILE] = reinterpret_cast<double(*)[TILE]>(cross_sm + TILE * MAXD);
  double* th = cross_sm + 2 * TILE * MAXD;
  const int tile = blockIdx.x;
  const int It = tile / NT, J = tile - It * NT;
  for (int q = threadIdx.x; q < TILE * MAXD; q += blockDim.x) {
    const int r = q / MAXD, k = q - r * MAXD;
    const int pt = min(It * TILE + r, N - 1), pi = min(J * TILE + r, n - 1);
    xt[r][k] = k < d ? Xt[(size_t)pt * d + k] : 0.0;
    xs[k][r] = k < d ? X[(size_t)pi * d + k] : 0.0;
  }
  for (int k = threadIdx.x; k < MAXD; k += blockDim.x) th[k] = k < d ? theta[k] : 0.0;
  __syncthreads();
  double* out = ext + (size_t)tile * TILE_ELEMS;
  bool nonfinite = false;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < TILE_ELEMS; e += gridDim.y * blockDim.x) {
    int r, c;
    elem_rc(e, r, c);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < MAXD; ++k) s = __dadd_rn(s, __dmul_rn(th[k], pow_abs_p(xt[r][k] - xs[k][c], p)));
    const double v = exp_neg(s);
    const bool live = It * TILE + r < N && J * TILE + c < n;
    nonfinite |= live && (!isfinite(v) || isnan(s));
    out[e] = live ? v : 0.0;
  }
  if (nonfinite) *bad = 1;
}

// Any d (the d > 32 path): cross_tiles_kernel's arithmetic from global-memory coordinates.
__global__ void __launch_bounds__(256) cross_tiles_generic_kernel(const double* __restrict__ Xt, int N,
                                                                  const double* __restrict__ X, int n,
                                                                  int d, const double* __restrict__ theta,
                                                                  double p, int NT,
                                                                  double* __restrict__ ext, int* bad) {
  const int tile = blockIdx.x;
  const int It = tile / NT, J = tile - It * NT;
  double* out = ext + (size_t)tile * TILE_ELEMS;
  bool nonfinite = false;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < TILE_ELEMS; e += gridDim.y * blockDim.x) {
    int r, c;
    elem_rc(e, r, c);
    const int pt = min(It * TILE + r, N - 1), pi = min(J * TILE + c, n - 1);
    double s = 0.0;
    for (int k = 0; k < d; ++k)
      s = __dadd_rn(s, __dmul_rn(__ldg(theta + k), pow_abs_p(__ldg(Xt + (size_t)pt * d + k) - __ldg(X + (size_t)pi * d + k), p)));
    const double v = exp_neg(s);
    const bool live = It * TILE + r < N && J * TILE + c < n;
    nonfinite |= live && (!isfinite(v) || isnan(s));
    out[e] = live ? v : 0.0;
  }
  if (nonfinite) *bad = 1;
}

template <int MAXD>
static void launch_cross(dim3 grid, cudaStream_t s, const double* Xt, int N, const double* X, int n,
                         int d, const double* theta, double p, int NT, double* ext, int* bad) {
  const int smem = (2 * TILE * MAXD + MAXD) * (int)sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(cross_tiles_kernel<MAXD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cross_tiles_kernel<MAXD><<<grid, 256, smem, s>>>(Xt, N, X, n, d, theta, p, NT, ext, bad);
}

void launch_cross_tiles(const double* Xt, int N, const double* X, int n, int d,
                        const double* theta, double p, int NT, int RT, double* ext, int* bad,
                        cudaStream_t s) {
  const dim3 grid(RT * NT, 4);
#define GPEMU_CROSS(D) launch_cross<D>(grid, s, Xt, N, X, n, d, theta, p, NT, ext, bad)
  if (d <= 1) GPEMU_CROSS(1);
  else if (d <= 2) GPEMU_CROSS(2);
  else if (d <= 3) GPEMU_CROSS(3);
  else if (d <= 4) GPEMU_CROSS(4);
  else if (d <= 6) GPEMU_CROSS(6);
  else if (d <= 8) GPEMU_CROSS(8);
  else if (d <= 10) GPEMU_CROSS(10);
  else if (d <= 12) GPEMU_CROSS(12);
  else if (d <= 16) GPEMU_CROSS(16);
  else if (d <= 20) GPEMU_CROSS(20);
  else if (d <= 24) GPEMU_CROSS(24);
  else if (d <= 32) GPEMU_CROSS(32);
  else cross_tiles_generic_kernel<<<grid, 256, 0, s>>>(Xt, N, X, n, d, theta, p, NT, ext, bad);
#undef GPEMU_CROSS
}

// yhat from the cross-correlation tiles of one chunk (before the extension DAG overwrites
// them with W = L^-1 r): CTA (It, blk) owns 128 test points and the kTrainBlock/128 tiles
// of training block blk; each slab (128 x 32, contiguous) is staged through shared memory and
// thread r walks its row in ascending column order -- predict_kernel's summation order.
__global__ void __launch_bounds__(128) yhat_tiles_kernel(const double* __restrict__ ext, int Nc,
                                                         int n, int NT,
                                                         const double* __restrict__ alpha,
                                                         double* __restrict__ part, size_t N,
                                                         size_t p0) {
  __shared__ double slab[SLAB_ELEMS];
  __shared__ double al[SLAB];
  const int It = blockIdx.x, blk = blockIdx.y;
  const int r = threadIdx.x;
  const int J0 = blk * (kTrainBlock / TILE), J1 = min(NT, J0 + kTrainBlock / TILE);
  double acc = 0.0;
  for (int J = J0; J < J1; ++J) {
    const double* tl = ext + ((size_t)It * NT + J) * TILE_ELEMS;
    double tacc = 0.0;
    for (int sl = 0; sl < SLABS_PER_TILE; ++sl) {
      const int cbase = J * TILE + sl * SLAB;
      if (cbase >= n) break;  // all-padding slab: r = 0 there (same as predict_kernel's rows)
      __syncthreads();
      const double2* src = reinterpret_cast<const double2*>(tl + sl * SLAB_ELEMS);
      double2* dst = reinterpret_cast<double2*>(slab);
      for (int q = threadIdx.x; q < SLAB_ELEMS / 2; q += blockDim.x) dst[q] = src[q];
      if (threadIdx.x < SLAB) al[threadIdx.x] = cbase + (int)threadIdx.x < n ? alpha[cbase + threadIdx.x] : 0.0;
      __syncthreads();
      const int cn = min(SLAB, n - cbase);
      for (int cc = 0; cc < cn; ++cc) tacc = fma(slab[slab_off(r, cc)], al[cc], tacc);
    }
    acc = __dadd_rn(acc, tacc);
  }
  const int pt = It * TILE + r;
  if (pt < Nc) part[(size_t)blk * N + p0 + pt] = acc;
}

void launch_yhat_tiles(const double* ext, int Nc, int n, int NT, const double* alpha, double* part,
                       size_t N, size_t p0, cudaStream_t s) {
  const dim3 grid((Nc + TILE - 1) / TILE, predict_blocks(n));
  yhat_tiles_kernel<<<grid, TILE, 0, s>>>(ext, Nc, n, NT, alpha, part, N, p0);
}

void launch_predict_combine(const double* part, int N, int n, double mu, double* yhat,
                            cudaStream_t s) {
  predict_combine_kernel<<<(N + 255) / 256, 256, 0, s>>>(part, N, predict_blocks(n), mu, yhat);
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
