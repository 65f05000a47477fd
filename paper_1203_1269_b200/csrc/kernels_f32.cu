// kernels_f32.cu -- single-precision (Precision::kSingle) companions of K1/K3/K4.
//
// The float instantiation of the reference (core.hpp:86-96; ProfileEvaluator<float>,
// likelihood.hpp:74-158) casts the design, y, theta, p and the nugget to float and runs the
// correlation build, factor and solves in float, while log|R| (backend.hpp:111-113) and the
// three dots (dot_accumulate, matrix.hpp:64-69) accumulate in double. These kernels follow
// that split. Float tiles are 128 x 128 column-major (element (r, c) at c * 128 + r), the
// layout kernels_chol_f32.cu streams by TMA.
//   pow_abs<float>       correlation.hpp:29-34   expf(p logf|d|), d == 0 -> 0, in float
//   theta_weighted_sum   correlation.hpp:42-47   float sum over k
//   build_into<float>    correlation.hpp:187-223 R_ij = expf(-s), R_ii = 1 + nugget
//   factorize_into       backend.hpp:102-120     + jitter on the diagonal (float)
#include <cuda_runtime.h>

#include <cfloat>

#include "fastmath.cuh"
#include "kernels.h"
#include "layout.cuh"

namespace gpemu_dev {

__device__ __forceinline__ float pow_abs_f(float delta, float p) {
  if (delta == 0.0f) return 0.0f;
  return expf(p * logf(fabsf(delta)));
}

// |x_ik - x_jk|^p for every element of every lower tile, in DOUBLE from the double design
// (fastmath.cuh pow, <= 1 ulp from glibc), column-major per tile: [tile][k][c * 128 + r].
// A float table would carry a 6e-8 relative error into s = sum theta_k T_k, i.e. a
// 6e-8 * s relative error into R (s reaches ~30): larger than float rounding of R itself;
// keeping T in double makes each float R_ij the rounding of the double value.
__global__ void pow_table_cm_kernel(const double* __restrict__ X, int n, int d, double p, int NT,
                                    double* __restrict__ table) {
  const int tile = blockIdx.x;
  int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
  while ((I + 1) * (I + 2) / 2 <= tile) ++I;
  while (I * (I + 1) / 2 > tile) --I;
  const int J = tile - I * (I + 1) / 2;
  double* tb = table + (size_t)tile * d * TILE_ELEMS;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < TILE_ELEMS; e += gridDim.y * blockDim.x) {
    const int c = e >> 7, r = e & 127;
    const int i = I * TILE + r, j = J * TILE + c;
    const bool live = i < n && j < n && i != j;
    for (int k = 0; k < d; ++k) {
      double v = 0.0;
      if (live) v = pow_abs_fast(X[(size_t)i * d + k] - X[(size_t)j * d + k], p);
      tb[(size_t)k * TILE_ELEMS + e] = v;
    }
  }
}

void launch_pow_table_f32(const double* X, int n, int d, double p, int NT, double* table,
                          cudaStream_t s) {
  pow_table_cm_kernel<<<dim3(num_tiles(NT), 8), 256, 0, s>>>(X, n, d, p, NT, table);
}

constexpr int kAsmChunkF = 64;
constexpr int kSlotILPF = 8;

// R for every candidate of the batch (the FP64 assemble's structure: one element per thread,
// table values in registers, 8 candidates in flight, padded slot groups so the loop has no
// per-slot guard): s and exp(-s) in double, R_ij rounded once to float.
template <int MAXD>
__global__ void __launch_bounds__(256) assemble_f32_kernel(
    const double* __restrict__ table, const double* __restrict__ theta, int n, int d, double nugget,
    int NT, const int* __restrict__ slots, int nslots, const double* __restrict__ jitter,
    float* __restrict__ factors, size_t slot_stride, int* __restrict__ status) {
  __shared__ double th[kAsmChunkF * MAXD];
  __shared__ int sl[kAsmChunkF];
  __shared__ long long soff[kAsmChunkF];
  const int tile = blockIdx.x;
  int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
  while ((I + 1) * (I + 2) / 2 <= tile) ++I;
  while (I * (I + 1) / 2 > tile) --I;
  const int J = tile - I * (I + 1) / 2;
  const double* tb = table + (size_t)tile * d * TILE_ELEMS;
  const float diag_base = 1.0f + (float)nugget;  // correlation.hpp:193, Scalar(1) + nugget
  float* const fbase = factors + (size_t)tile * TILE_ELEMS;
  for (int c0 = 0; c0 < nslots; c0 += kAsmChunkF) {
    const int cn = min(kAsmChunkF, nslots - c0);
    __syncthreads();
    for (int q = threadIdx.x; q < kAsmChunkF * MAXD; q += blockDim.x) {
      const int si = q / MAXD, k = q - si * MAXD;
      th[q] = k < d ? theta[(size_t)slots[c0 + min(si, cn - 1)] * d + k] : 0.0;
    }
    for (int q = threadIdx.x; q < kAsmChunkF; q += blockDim.x) {
      const int slot = slots[c0 + min(q, cn - 1)];
      sl[q] = slot;
      soff[q] = (long long)slot * (long long)slot_stride;
    }
    __syncthreads();
    const int cn_pad = (cn + kSlotILPF - 1) / kSlotILPF * kSlotILPF;
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < TILE_ELEMS; e += gridDim.y * blockDim.x) {
      const int c = e >> 7, r = e & 127;
      const int i = I * TILE + r, j = J * TILE + c;
      const bool pad = i >= n || j >= n;
      float* dst = fbase + e;
      if (pad || i == j) {
        for (int si = 0; si < cn; ++si) {
          const int slot = sl[si];
          // factorize_into: lower(i,i) += (float)jitter (backend.hpp:107-109)
          dst[soff[si]] = pad ? (i == j ? 1.0f : 0.0f) : diag_base + (float)jitter[slot];
        }
        continue;
      }
      double t[MAXD];
#pragma unroll
      for (int k = 0; k < MAXD; ++k) t[k] = k < d ? __ldg(tb + (size_t)k * TILE_ELEMS + e) : 0.0;
      for (int s0 = 0; s0 < cn_pad; s0 += kSlotILPF) {
        double s[kSlotILPF], v[kSlotILPF];
#pragma unroll
        for (int q = 0; q < kSlotILPF; ++q) s[q] = 0.0;
#pragma unroll
        for (int k = 0; k < MAXD; ++k)
#pragma unroll
          for (int q = 0; q < kSlotILPF; ++q) s[q] = fma(th[(s0 + q) * MAXD + k], t[k], s[q]);
#pragma unroll
        for (int q = 0; q < kSlotILPF; ++q) v[q] = exp_neg(s[q]);
#pragma unroll
        for (int q = 0; q < kSlotILPF; ++q) {
          dst[soff[s0 + q]] = (float)v[q];
          if (!isfinite(v[q]) || isnan(s[q])) status[sl[s0 + q]] = 2;  // GPEMU_SLOT_NONFINITE
        }
      }
    }
  }
}

// Any d (the d > 32 path): assemble_f32_kernel's arithmetic with the table and theta read from
// global memory.
__global__ void __launch_bounds__(256) assemble_f32_generic_kernel(
    const double* __restrict__ table, const double* __restrict__ theta, int n, int d, double nugget,
    int NT, const int* __restrict__ slots, int nslots, const double* __restrict__ jitter,
    float* __restrict__ factors, size_t slot_stride, int* __restrict__ status) {
  const int tile = blockIdx.x;
  int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
  while ((I + 1) * (I + 2) / 2 <= tile) ++I;
  while (I * (I + 1) / 2 > tile) --I;
  const int J = tile - I * (I + 1) / 2;
  const double* tb = table + (size_t)tile * d * TILE_ELEMS;
  const float diag_base = 1.0f + (float)nugget;
  float* const fbase = factors + (size_t)tile * TILE_ELEMS;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < TILE_ELEMS; e += gridDim.y * blockDim.x) {
    const int c = e >> 7, r = e & 127;
    const int i = I * TILE + r, j = J * TILE + c;
    const bool pad = i >= n || j >= n;
    float* dst = fbase + e;
    for (int si = 0; si < nslots; ++si) {
      const int slot = slots[si];
      float v;
      if (pad || i == j) {
        v = pad ? (i == j ? 1.0f : 0.0f) : diag_base + (float)jitter[slot];
      } else {
        double sacc = 0.0;
        for (int k = 0; k < d; ++k)
          sacc = fma(__ldg(theta + (size_t)slot * d + k), __ldg(tb + (size_t)k * TILE_ELEMS + e), sacc);
        const double ev = exp_neg(sacc);
        v = (float)ev;
        if (!isfinite(ev) || isnan(sacc)) status[slot] = 2;
      }
      dst[(size_t)slot * slot_stride] = v;
    }
  }
}

template <int MAXD>
static void launch_asm_f(dim3 grid, cudaStream_t s, const double* table, const double* theta, int n,
                         int d, double nugget, int NT, const int* slots, int nslots,
                         const double* jitter, float* factors, size_t slot_stride, int* status) {
  assemble_f32_kernel<MAXD><<<grid, 256, 0, s>>>(table, theta, n, d, nugget, NT, slots, nslots,
                                                 jitter, factors, slot_stride, status);
}

__global__ void border_init_f32_kernel(const double* __restrict__ y, int n, int Npad,
                                       const int* __restrict__ slots, float* __restrict__ borders,
                                       int* __restrict__ status) {
  const int slot = slots[blockIdx.y];
  float* u = borders + (size_t)slot * 2 * Npad;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Npad; i += gridDim.x * blockDim.x) {
    u[i] = i < n ? (float)y[i] : 0.0f;
    u[Npad + i] = i < n ? 1.0f : 0.0f;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) status[slot] = 0;
}

void launch_assemble_f32(const double* table, const double* theta, const double* y, int n, int d,
                         double nugget, int NT, const int* slots, int nslots, const double* jitter,
                         float* factors, size_t slot_stride, float* borders, int* status,
                         cudaStream_t s) {
  const int Npad = NT * TILE;
  border_init_f32_kernel<<<dim3((Npad + 255) / 256 < 32 ? (Npad + 255) / 256 : 32, nslots), 256, 0, s>>>(
      y, n, Npad, slots, borders, status);
  const dim3 grid(num_tiles(NT), 8);
#define GPEMU_ASMF(D) \
  launch_asm_f<D>(grid, s, table, theta, n, d, nugget, NT, slots, nslots, jitter, factors, slot_stride, status)
  if (d <= 1) GPEMU_ASMF(1);
  else if (d <= 2) GPEMU_ASMF(2);
  else if (d <= 3) GPEMU_ASMF(3);
  else if (d <= 4) GPEMU_ASMF(4);
  else if (d <= 6) GPEMU_ASMF(6);
  else if (d <= 8) GPEMU_ASMF(8);
  else if (d <= 10) GPEMU_ASMF(10);
  else if (d <= 12) GPEMU_ASMF(12);
  else if (d <= 16) GPEMU_ASMF(16);
  else if (d <= 20) GPEMU_ASMF(20);
  else if (d <= 24) GPEMU_ASMF(24);
  else if (d <= 32) GPEMU_ASMF(32);
  else
    assemble_f32_generic_kernel<<<grid, 256, 0, s>>>(table, theta, n, d, nugget, NT, slots, nslots,
                                                     jitter, factors, slot_stride, status);
#undef GPEMU_ASMF
}

// Deviance tail (likelihood.hpp:124-140) for float factors: log|R| = 2 sum log(double(L_ii))
// in sequence (backend.hpp:111-113), the three dots in double (matrix.hpp:64-69), the rest
// in double exactly as finalize_kernel.
constexpr int kLogChunkF = 2048;
__global__ void __launch_bounds__(256) finalize_f32_kernel(
    const float* __restrict__ factors, size_t slot_stride, const float* __restrict__ borders,
    const int* __restrict__ status, const double* __restrict__ jitter, int n, int NT,
    const int* __restrict__ slots, double* __restrict__ out, int spec_off) {
  __shared__ double logs[kLogChunkF];
  __shared__ double dots[3];
  const int slot = slots[blockIdx.x];
  const int Npad = NT * TILE;
  const float* fac = factors + (size_t)slot * slot_stride;
  const float* u = borders + (size_t)slot * 2 * Npad;
  const float* v = u + Npad;
  const int st = status[slot];
  const int dst = spec_record_dst(status, slot, st, spec_off);
  if (dst < 0) return;  // uniform
  double logsum = 0.0;
  if (st == 0) {
    for (int c0 = 0; c0 < n; c0 += kLogChunkF) {
      const int cn = min(kLogChunkF, n - c0);
      for (int q = threadIdx.x; q < cn; q += blockDim.x) {
        const int i = c0 + q;
        logs[q] = log((double)fac[tile_index(i >> 7, i >> 7) * TILE_ELEMS + (i & 127) * TILE + (i & 127)]);
      }
      __syncthreads();
      if (threadIdx.x == 0)
        for (int q = 0; q < cn; ++q) logsum = __dadd_rn(logsum, logs[q]);
      __syncthreads();
    }
    if (threadIdx.x < 3) {
      const float* a = threadIdx.x == 2 ? v : u;
      const float* b = threadIdx.x == 0 ? u : v;
      double s = 0.0;
      for (int i = 0; i < n; ++i) s = __dadd_rn(s, __dmul_rn((double)a[i], (double)b[i]));
      dots[threadIdx.x] = s;
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  double* o = out + (size_t)dst * REC_SIZE;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  o[REC_NEG2] = inf;
  o[REC_MU] = 0.0;
  o[REC_SIGMA2] = 0.0;
  o[REC_JITTER] = 0.0;
  o[REC_LOGDET] = 0.0;
  o[REC_UTU] = 0.0;
  o[REC_VTV] = 0.0;
  if (st != 0) {
    o[REC_STATUS] = (double)st;
    return;
  }
  const double log_det = __dmul_rn(2.0, logsum);
  const double utu = dots[0], vtu = dots[1], vtv = dots[2];
  o[REC_LOGDET] = log_det;
  o[REC_UTU] = utu;
  o[REC_VTV] = vtv;
  if (!(vtv > 0.0)) {
    o[REC_STATUS] = 3.0;
    return;
  }
  const double mu = vtu / vtv;
  const double t1 = __dmul_rn(__dmul_rn(2.0, mu), vtu);
  const double t2 = __dmul_rn(__dmul_rn(mu, mu), vtv);
  double s2 = __dadd_rn(__dsub_rn(utu, t1), t2) / (double)n;
  if (s2 < 0.0) s2 = 0.0;
  const double qf = __dmul_rn((double)n, s2);
  const double qf_floored = qf > DBL_MIN ? qf : DBL_MIN;
  o[REC_NEG2] = __dadd_rn(log_det, __dmul_rn((double)n, log(qf_floored)));
  o[REC_MU] = mu;
  o[REC_SIGMA2] = s2;
  o[REC_JITTER] = jitter[slot];
  o[REC_STATUS] = 0.0;
}

void launch_finalize_f32(const float* factors, size_t slot_stride, const float* borders,
                         const int* status, const double* jitter, int n, int NT, const int* slots,
                         int nslots, double* out, int spec_off, cudaStream_t s) {
  finalize_f32_kernel<<<nslots, 256, 0, s>>>(factors, slot_stride, borders, status, jitter, n, NT,
                                             slots, out, spec_off);
}

// alpha = solve_full(factor, y - mu) in float (likelihood.hpp:228-229, backend.hpp:129-169):
// column-oriented substitution, one CTA; per entry the same subtraction order as the
// reference's row loops (ascending k forward, descending backward).
__global__ void __launch_bounds__(1024) alpha_f32_kernel(const float* __restrict__ tiles, int n,
                                                        const double* __restrict__ y, double mu,
                                                        double* __restrict__ alpha) {
  extern __shared__ float w[];
  const float muf = (float)mu;
  for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] = (float)y[i] - muf;
  __syncthreads();
  auto Lat = [&](int i, int j) {  // lower element (i >= j), column-major tiles
    return tiles[tile_index(i >> 7, j >> 7) * TILE_ELEMS + (j & 127) * TILE + (i & 127)];
  };
  for (int k = 0; k < n; ++k) {  // L u = b
    const float xk = __fdiv_rn(w[k], Lat(k, k));
    __syncthreads();
    for (int l = k + 1 + threadIdx.x; l < n; l += blockDim.x) w[l] = __fsub_rn(w[l], __fmul_rn(Lat(l, k), xk));
    if (threadIdx.x == 0) w[k] = xk;
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {  // L^T x = u
    const float xk = __fdiv_rn(w[k], Lat(k, k));
    __syncthreads();
    for (int l = threadIdx.x; l < k; l += blockDim.x) w[l] = __fsub_rn(w[l], __fmul_rn(Lat(k, l), xk));
    if (threadIdx.x == 0) w[k] = xk;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) alpha[i] = (double)w[i];
}

void launch_alpha_f32(const float* tiles, int n, const double* y, double mu, double* alpha,
                      cudaStream_t s) {
  const size_t smem = (size_t)n * sizeof(float);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(alpha_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  alpha_f32_kernel<<<1, 1024, smem, s>>>(tiles, n, y, mu, alpha);
}

// Float column-major tiles -> the FP64 engine's swizzled double tiles (exact widening), so a
// float model can reuse the FP64 extension-mode DAG for the kriging MSE.
__global__ void tiles_f32_to_f64_kernel(const float* __restrict__ src, double* __restrict__ dst) {
  const size_t tile = blockIdx.x;
  const float* s = src + tile * TILE_ELEMS;
  double* o = dst + tile * TILE_ELEMS;
  for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x) {
    const int c = e >> 7, r = e & 127;
    o[elem_off(r, c)] = (double)s[e];
  }
}

void launch_tiles_f32_to_f64(const float* src, int NT, double* dst, cudaStream_t s) {
  tiles_f32_to_f64_kernel<<<num_tiles(NT), 256, 0, s>>>(src, dst);
}

// Row-major lower factor from float tiles (last_factor / try_cholesky readback), as double.
__global__ void tiles_f32_to_rowmajor_kernel(const float* __restrict__ tiles, int n, double* __restrict__ L) {
  const int i = blockIdx.y;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    L[(size_t)i * n + j] = j <= i ? (double)tiles[tile_index(i >> 7, j >> 7) * TILE_ELEMS + (j & 127) * TILE + (i & 127)] : 0.0;
}

void launch_tiles_f32_to_rowmajor(const float* tiles, int n, int NT, double* L, cudaStream_t s) {
  (void)NT;
  tiles_f32_to_rowmajor_kernel<<<dim3((n + 255) / 256, n), 256, 0, s>>>(tiles, n, L);
}

// predict (predictor.hpp:36-44) for a float model: x cast to float, corr_vector<float>
// (float terms, float weighted sum, expf), yhat = mu + dot_accumulate<float>(r, alpha): the
// products and the ascending sum in double, one thread per test point.
__global__ void __launch_bounds__(128) predict_f32_kernel(const double* __restrict__ Xt, int N,
                                                         const double* __restrict__ X, int n, int d,
                                                         const double* __restrict__ theta, double p,
                                                         double mu, const double* __restrict__ alpha,
                                                         double* __restrict__ yhat, int* bad) {
  __shared__ float xs[128][33];
  __shared__ double as[128];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int jc = min(j, N - 1);
  float xt[32], th[32];
  for (int k = 0; k < 32; ++k) {
    xt[k] = k < d ? (float)Xt[(size_t)jc * d + k] : 0.0f;
    th[k] = k < d ? (float)theta[k] : 0.0f;
  }
  const float pf = (float)p;
  double acc = 0.0;
  bool nonfinite = false;
  for (int c0 = 0; c0 < n; c0 += 128) {
    const int cn = min(128, n - c0);
    __syncthreads();
    for (int q = threadIdx.x; q < 128 * d; q += blockDim.x) {
      const int r = q / d, k = q - r * d;
      xs[r][k] = r < cn ? (float)X[(size_t)(c0 + r) * d + k] : 0.0f;
    }
    for (int q = threadIdx.x; q < 128; q += blockDim.x) as[q] = q < cn ? alpha[c0 + q] : 0.0;
    __syncthreads();
    for (int r = 0; r < cn; ++r) {
      float s = 0.0f;
      for (int k = 0; k < d; ++k) s = fmaf(th[k], pow_abs_f(xt[k] - xs[r][k], pf), s);
      const float v = expf(-s);
      nonfinite |= !isfinite(v);
      acc = __dadd_rn(acc, __dmul_rn((double)v, as[r]));
    }
  }
  if (j < N) {
    yhat[j] = mu + acc;
    if (nonfinite) *bad = 1;
  }
}

// Any d (the d > 32 path): predict_f32_kernel's float arithmetic from global-memory coordinates.
__global__ void __launch_bounds__(128) predict_f32_generic_kernel(const double* __restrict__ Xt, int N,
                                                                 const double* __restrict__ X, int n, int d,
                                                                 const double* __restrict__ theta, double p,
                                                                 double mu, const double* __restrict__ alpha,
                                                                 double* __restrict__ yhat, int* bad) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int jc = min(j, N - 1);
  const float pf = (float)p;
  double acc = 0.0;
  bool nonfinite = false;
  for (int r = 0; r < n; ++r) {
    float s = 0.0f;
    for (int k = 0; k < d; ++k)
      s = fmaf((float)__ldg(theta + k),
               pow_abs_f((float)__ldg(Xt + (size_t)jc * d + k) - (float)__ldg(X + (size_t)r * d + k), pf), s);
    const float v = expf(-s);
    nonfinite |= !isfinite(v);
    acc = __dadd_rn(acc, __dmul_rn((double)v, __ldg(alpha + r)));
  }
  if (j < N) {
    yhat[j] = mu + acc;
    if (nonfinite) *bad = 1;
  }
}

void launch_predict_f32(const double* Xt, int N, const double* X, int n, int d, const double* theta,
                        double p, double mu, const double* alpha, double* yhat, int* bad, cudaStream_t s) {
  if (N <= 0) return;
  if (d > 32)
    predict_f32_generic_kernel<<<(N + 127) / 128, 128, 0, s>>>(Xt, N, X, n, d, theta, p, mu, alpha, yhat, bad);
  else
    predict_f32_kernel<<<(N + 127) / 128, 128, 0, s>>>(Xt, N, X, n, d, theta, p, mu, alpha, yhat, bad);
}

}  // namespace gpemu_dev
