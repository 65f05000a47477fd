// kernels_misc.cu -- K3 deviance finalisation, layout conversion.
//
// Reference (relative to /root/reference/proj/include/gpemu/):
//   factorize_into log-det    backend.hpp:111-113   2 * sum_i log L_ii, sequential, double
//   dot_accumulate            matrix.hpp:64-69      sequential double dot
//   eval tail                 likelihood.hpp:124-140
//   sigma2_hat_from_parts     likelihood.hpp:63-66
// The scalar tail keeps the reference's sequential summation order (one thread
// per sum, the four sums concurrent, operands staged in shared memory) and rounds
// every product/sum separately.
#include <cuda_runtime.h>

#include <cfloat>

#include "kernels.h"
#include "layout.cuh"

namespace gpemu_dev {

constexpr int kLogChunk = 960;

// One block per candidate. Per chunk of kLogChunk rows the block stages log L_ii, u_i and v_i
// into shared memory, and the four sequential sums run concurrently from shared memory: the
// log-sum in warp 1, utu / vtu / vtv in lanes 0-2 of warp 0. Each sum keeps the reference's
// element order and separate roundings (backend.hpp:111-113, matrix.hpp:64-69). The chunks are
// double-buffered: while the four sums consume chunk c, warps 2..7 stage chunk c+1, so the
// staging (the logs) overlaps the dependent add chains -- what a single-candidate evaluation
// waits for: 51 -> 41 us at n = 4096.
__global__ void __launch_bounds__(256) finalize_kernel(
    const double* __restrict__ factors, size_t slot_stride, const double* __restrict__ borders,
    const int* __restrict__ status, const double* __restrict__ jitter, int n, int NT,
    const int* __restrict__ slots, double* __restrict__ out, int spec_off) {
  __shared__ double logs[2][kLogChunk], su[2][kLogChunk], sv[2][kLogChunk];
  __shared__ double sums[4];
  const int slot = slots[blockIdx.x];
  const int Npad = NT * TILE;
  const double* fac = factors + (size_t)slot * slot_stride;
  const double* u = borders + (size_t)slot * 2 * Npad;
  const double* v = u + Npad;
  const int st = status[slot];
  const int dst = spec_record_dst(status, slot, st, spec_off);
  if (dst < 0) return;  // uniform
  if (st == 0) {
    double acc = 0.0;  // warp 1 lane 0: logsum; warp 0 lanes 0..2: utu, vtu (v.u), vtv
    const int t = threadIdx.x;
    const bool summer = t < 3 || t == 32;
    // stagers: warps 2..7 (whole warps, so that no warp splits between a sum and the staging;
    // leaving the sums' sub-partitions to them alone made the staging the bound: 41 -> 53 us)
    const int sidx = t - 64;
    const int nstage = blockDim.x - 64;
    const bool stager = t >= 64;
    auto stage = [&](int c0, int buf) {
      const int cn = min(kLogChunk, n - c0);
      for (int q = sidx; q < cn; q += nstage) {
        const int i = c0 + q;
        logs[buf][q] = log(fac[tile_index(i >> 7, i >> 7) * TILE_ELEMS + elem_off(i & 127, i & 127)]);
        su[buf][q] = u[i];
        sv[buf][q] = v[i];
      }
    };
    if (stager) stage(0, 0);
    __syncthreads();
    for (int c0 = 0, buf = 0; c0 < n; c0 += kLogChunk, buf ^= 1) {
      const int cn = min(kLogChunk, n - c0);
      if (summer) {
        const double* a = t == 2 ? sv[buf] : su[buf];
        const double* b = t == 0 ? su[buf] : sv[buf];
        if (t == 32) {
#pragma unroll 8
          for (int q = 0; q < cn; ++q) acc = __dadd_rn(acc, logs[buf][q]);
        } else {
#pragma unroll 8
          for (int q = 0; q < cn; ++q) acc = __dadd_rn(acc, __dmul_rn(a[q], b[q]));
        }
      } else if (stager && c0 + kLogChunk < n) {
        stage(c0 + kLogChunk, buf ^ 1);
      }
      __syncthreads();
    }
    if (t < 3) sums[t] = acc;
    if (t == 32) sums[3] = acc;
    __syncthreads();
  }
  const double logsum = st == 0 ? sums[3] : 0.0;
  const double dots[3] = {st == 0 ? sums[0] : 0.0, st == 0 ? sums[1] : 0.0, st == 0 ? sums[2] : 0.0};
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
  if (!(vtv > 0.0)) {  // likelihood.hpp:127
    o[REC_STATUS] = 3.0;
    return;
  }
  const double mu = vtu / vtv;
  const double t1 = __dmul_rn(__dmul_rn(2.0, mu), vtu);
  const double t2 = __dmul_rn(__dmul_rn(mu, mu), vtv);
  double s2 = __dadd_rn(__dsub_rn(utu, t1), t2) / (double)n;
  if (s2 < 0.0) s2 = 0.0;
  const double qf = __dmul_rn((double)n, s2);
  const double qf_floored = qf > DBL_MIN ? qf : DBL_MIN;  // likelihood.hpp:134
  o[REC_NEG2] = __dadd_rn(log_det, __dmul_rn((double)n, log(qf_floored)));
  o[REC_MU] = mu;
  o[REC_SIGMA2] = s2;
  o[REC_JITTER] = jitter[slot];
  o[REC_STATUS] = 0.0;
}

void launch_finalize(const double* factors, size_t slot_stride, const double* borders,
                     const int* status, const double* jitter, int n, int NT, const int* slots,
                     int nslots, double* out, int spec_off, cudaStream_t s) {
  finalize_kernel<<<nslots, 256, 0, s>>>(factors, slot_stride, borders, status, jitter, n, NT,
                                         slots, out, spec_off);
}

// ---------------------------------------------------------------------------
__global__ void rowmajor_to_tiles_kernel(const double* __restrict__ A, int n, double jitter,
                                         double* __restrict__ tiles) {
  const int tile = blockIdx.x;
  int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
  while ((I + 1) * (I + 2) / 2 <= tile) ++I;
  while (I * (I + 1) / 2 > tile) --I;
  const int J = tile - I * (I + 1) / 2;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < TILE_ELEMS; e += gridDim.y * blockDim.x) {
    int r, c;
    elem_rc(e, r, c);
    const int i = I * TILE + r, j = J * TILE + c;
    double v;
    if (i >= n || j >= n) {
      v = (i == j) ? 1.0 : 0.0;
    } else if (i == j) {
      v = __dadd_rn(A[(size_t)i * n + i], jitter);
    } else {
      v = i > j ? A[(size_t)i * n + j] : A[(size_t)j * n + i];  // lower triangle only
    }
    tiles[(size_t)tile * TILE_ELEMS + e] = v;
  }
}

void launch_rowmajor_to_tiles(const double* A, int n, int NT, double jitter, double* tiles,
                              cudaStream_t s) {
  rowmajor_to_tiles_kernel<<<dim3(num_tiles(NT), 8), 256, 0, s>>>(A, n, jitter, tiles);
}

__global__ void tiles_to_rowmajor_kernel(const double* __restrict__ tiles, int n,
                                         double* __restrict__ L) {
  const int i = blockIdx.y;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    L[(size_t)i * n + j] =
        j <= i ? tiles[tile_index(i >> 7, j >> 7) * TILE_ELEMS + elem_off(i & 127, j & 127)] : 0.0;
  }
}

void launch_tiles_to_rowmajor(const double* tiles, int n, int NT, double* L, cudaStream_t s) {
  tiles_to_rowmajor_kernel<<<dim3((n + 255) / 256, n), 256, 0, s>>>(tiles, n, L);
}

// dot_accumulate (matrix.hpp:64-69): sequential double dot in the reference's element order.
__global__ void dot_seq_kernel(const double* __restrict__ a, const double* __restrict__ b, int n,
                               double* __restrict__ out) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, __dmul_rn(a[i], b[i]));
  *out = s;
}

void launch_dot_seq(const double* a, const double* b, int n, double* out, cudaStream_t s) {
  dot_seq_kernel<<<1, 1, 0, s>>>(a, b, n, out);
}

}  // namespace gpemu_dev
