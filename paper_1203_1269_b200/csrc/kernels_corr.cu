// kernels_corr.cu -- K1: power-exponential correlation assembly on sm_100a.
//
// Reference: correlation.hpp (paths relative to /root/reference/proj/include/gpemu/).
//   pow_abs            :31-35   |dx|^p = exp(p log|dx|), dx == 0 -> 0
//   theta_weighted_sum :42-47   sum_k theta_k * term_k, sequential in k,
//                               products and sums rounded separately
//   CorrelationPlan    :156-180 per-design |dx|^p table
//   build_into         :187-223 R_ij = exp(-s), R_ii = 1 + nugget
// build_corr_matrix / corr_vector reproduce the sequential, separately rounded sum
// with __dmul_rn / __dadd_rn. The batched hot-path assembly keeps the sequential
// k order but fuses each term (fma), as the reference's own -march=native build
// does for part of the sum: half the FP64 issue, <= 1 ulp in s.
// exp/log are CUDA libdevice (<= 1 ulp from glibc): R matches to ~1e-16, not bitwise.
#include <cuda_runtime.h>

#include <algorithm>

#include "fastmath.cuh"
#include "kernels.h"
#include "layout.cuh"

namespace gpemu_dev {


__device__ __forceinline__ double pow_abs(double delta, double p) { return pow_abs_fast(delta, p); }

// Table: [tile][k][elem], tile-major over the packed lower tiles.
__global__ void pow_table_kernel(const double* __restrict__ X, int n, int d, double p, int NT,
                                 double* __restrict__ table) {
  const int tile = blockIdx.x;
  // tile -> (I, J)
  int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
  while ((I + 1) * (I + 2) / 2 <= tile) ++I;
  while (I * (I + 1) / 2 > tile) --I;
  const int J = tile - I * (I + 1) / 2;
  double* out = table + (size_t)tile * d * TILE_ELEMS;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < TILE_ELEMS; e += gridDim.y * blockDim.x) {
    int r, c;
    elem_rc(e, r, c);
    const int i = I * TILE + r, j = J * TILE + c;
    const bool live = i < n && j < n && i != j;
    for (int k = 0; k < d; ++k) {
      double v = 0.0;
      if (live) v = pow_abs(X[(size_t)i * d + k] - X[(size_t)j * d + k], p);
      out[(size_t)k * TILE_ELEMS + e] = v;
    }
  }
}

void launch_pow_table(const double* X, int n, int d, double p, int NT, double* table,
                      cudaStream_t s) {
  dim3 grid(num_tiles(NT), 16);
  pow_table_kernel<<<grid, 256, 0, s>>>(X, n, d, p, NT, table);
}

// Border rows [y; 1] (the bordered-matrix form of the two forward solves,
// likelihood.hpp:122-123) and the slot status reset.
__global__ void border_init_kernel(const double* __restrict__ y, int n, int Npad,
                                   const int* __restrict__ slots, double* __restrict__ borders,
                                   int* __restrict__ status) {
  const int slot = slots[blockIdx.y];
  double* u = borders + (size_t)slot * 2 * Npad;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Npad; i += gridDim.x * blockDim.x) {
    u[i] = i < n ? y[i] : 0.0;
    u[Npad + i] = i < n ? 1.0 : 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) status[slot] = 0;
}

constexpr int kAsmSlotChunk = 64;
constexpr int kSlotILP = 4;  // candidates per thread at a time (8: +1.5% at C3; 16 slower still)

// One element per thread: its d table values stay in registers and are reused by every
// candidate of the batch; kSlotILP candidates are processed together, branch-free (exp_neg,
// stores predicated), so their k-sums and exps interleave. MAXD is a compile-time bound on d
// (dispatch below), so the k loop is fully unrolled with no dead iterations.
template <int MAXD, bool kSplit, int ILP = kSlotILP>
__global__ void __launch_bounds__(256) assemble_kernel(
    const double* __restrict__ table, const double* __restrict__ theta, int n, int d,
    double nugget, int NT, const int* __restrict__ slots, int nslots,
    const double* __restrict__ jitter, double* __restrict__ factors, size_t slot_stride,
    int* __restrict__ status, int chunk) {
  __shared__ __align__(16) double th[kAsmSlotChunk * MAXD];  // [k][slot]: slot pairs load as double2
  __shared__ int sl[kAsmSlotChunk];
  __shared__ long long soff[kAsmSlotChunk];
  const int tile = blockIdx.x;
  int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
  while ((I + 1) * (I + 2) / 2 <= tile) ++I;
  while (I * (I + 1) / 2 > tile) --I;
  const int J = tile - I * (I + 1) / 2;
  const double* tb = table + (size_t)tile * d * TILE_ELEMS;
  const double diag_base = __dadd_rn(1.0, nugget);  // correlation.hpp:193
  double* const fbase = factors + (size_t)tile * TILE_ELEMS;

  // candidate chunks of `chunk` (<= kAsmSlotChunk) slots, spread over blockIdx.z on small designs
  // (kSplit: a separate instantiation, so the large-design code keeps its register allocation)
  const int cstep = kSplit ? chunk : kAsmSlotChunk;
  for (int c0 = kSplit ? blockIdx.z * chunk : 0; c0 < nslots; c0 += kSplit ? gridDim.z * chunk : kAsmSlotChunk) {
    const int cn = min(cstep, nslots - c0);
    __syncthreads();
    // Entries past cn replicate the last live slot (same theta -> the same value rewritten
    // to the same address), so the kSlotILP groups below need no per-slot guard.
    for (int q = threadIdx.x; q < kAsmSlotChunk * MAXD; q += blockDim.x) {
      const int si = q / MAXD, k = q - si * MAXD;
      th[k * kAsmSlotChunk + si] = k < d ? theta[(size_t)slots[c0 + min(si, cn - 1)] * d + k] : 0.0;
    }
    for (int q = threadIdx.x; q < kAsmSlotChunk; q += blockDim.x) {
      const int slot = slots[c0 + min(q, cn - 1)];
      sl[q] = slot;
      soff[q] = (long long)slot * (long long)slot_stride;
    }
    __syncthreads();
    const int cn_pad = (cn + ILP - 1) / ILP * ILP;
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < TILE_ELEMS;
         e += gridDim.y * blockDim.x) {
      int r, c;
      elem_rc(e, r, c);
      const int i = I * TILE + r, j = J * TILE + c;
      const bool pad = i >= n || j >= n;
      double* dst = fbase + e;
      if (pad || i == j) {
        for (int si = 0; si < cn; ++si) {
          const int slot = sl[si];
          dst[soff[si]] = pad ? (i == j ? 1.0 : 0.0) : __dadd_rn(diag_base, jitter[slot]);  // backend.hpp:107-109
        }
        continue;
      }
      double t[MAXD];
#pragma unroll
      for (int k = 0; k < MAXD; ++k) t[k] = (k < d) ? __ldg(tb + (size_t)k * TILE_ELEMS + e) : 0.0;
      for (int s0 = 0; s0 < cn_pad; s0 += ILP) {
        double s[ILP], v[ILP];
#pragma unroll
        for (int q = 0; q < ILP; ++q) s[q] = 0.0;
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
          if constexpr (ILP == 1) {
            s[0] = fma(th[k * kAsmSlotChunk + s0], t[k], s[0]);
          } else {
#pragma unroll
            for (int q = 0; q < ILP; q += 2) {
              const double2 tq = *reinterpret_cast<const double2*>(th + k * kAsmSlotChunk + s0 + q);
              s[q] = fma(tq.x, t[k], s[q]);
              s[q + 1] = fma(tq.y, t[k], s[q + 1]);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < ILP; ++q) v[q] = exp_neg(s[q]);
#pragma unroll
        for (int q = 0; q < ILP; ++q) {
          dst[soff[s0 + q]] = v[q];
          // GPEMU_SLOT_NONFINITE (correlation.hpp:58-61): s >= 0 for validated inputs, so exp(-s)
          // is non-finite exactly when s is NaN (exp_neg maps NaN to 0)
          if (s[q] != s[q]) status[sl[s0 + q]] = 2;
        }
      }
    }
  }
}

// Any d (the d > 32 path): the same arithmetic as assemble_kernel -- s = fma(theta_k, T_k, s)
// in ascending k, R = exp_neg(s), the same diagonal -- with the table and theta read from
// global memory (L1-cached) instead of registers / shared memory.
__global__ void __launch_bounds__(256) assemble_generic_kernel(
    const double* __restrict__ table, const double* __restrict__ theta, int n, int d,
    double nugget, int NT, const int* __restrict__ slots, int nslots,
    const double* __restrict__ jitter, double* __restrict__ factors, size_t slot_stride,
    int* __restrict__ status) {
  const int tile = blockIdx.x;
  int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
  while ((I + 1) * (I + 2) / 2 <= tile) ++I;
  while (I * (I + 1) / 2 > tile) --I;
  const int J = tile - I * (I + 1) / 2;
  const double* tb = table + (size_t)tile * d * TILE_ELEMS;
  const double diag_base = __dadd_rn(1.0, nugget);
  double* const fbase = factors + (size_t)tile * TILE_ELEMS;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < TILE_ELEMS; e += gridDim.y * blockDim.x) {
    int r, c;
    elem_rc(e, r, c);
    const int i = I * TILE + r, j = J * TILE + c;
    const bool pad = i >= n || j >= n;
    double* dst = fbase + e;
    if (pad || i == j) {
      for (int si = 0; si < nslots; ++si) {
        const int slot = slots[si];
        dst[(size_t)slot * slot_stride] = pad ? (i == j ? 1.0 : 0.0) : __dadd_rn(diag_base, jitter[slot]);
      }
      continue;
    }
    for (int s0 = 0; s0 < nslots; s0 += kSlotILP) {
      int sl[kSlotILP];
      double sacc[kSlotILP];
#pragma unroll
      for (int q = 0; q < kSlotILP; ++q) {
        sl[q] = slots[min(s0 + q, nslots - 1)];
        sacc[q] = 0.0;
      }
      for (int k = 0; k < d; ++k) {
        const double t = __ldg(tb + (size_t)k * TILE_ELEMS + e);
#pragma unroll
        for (int q = 0; q < kSlotILP; ++q) sacc[q] = fma(__ldg(theta + (size_t)sl[q] * d + k), t, sacc[q]);
      }
#pragma unroll
      for (int q = 0; q < kSlotILP; ++q) {
        if (s0 + q >= nslots) break;
        const double v = exp_neg(sacc[q]);
        dst[(size_t)sl[q] * slot_stride] = v;
        if (!isfinite(v) || isnan(sacc[q])) status[sl[q]] = 2;
      }
    }
  }
}

template <int MAXD>
static void launch_asm(dim3 grid, cudaStream_t s, const double* table, const double* theta, int n,
                       int d, double nugget, int NT, const int* slots, int nslots,
                       const double* jitter, double* factors, size_t slot_stride, int* status, int chunk) {
  if (grid.z > 1)
    assemble_kernel<MAXD, true><<<grid, 256, 0, s>>>(table, theta, n, d, nugget, NT, slots, nslots, jitter,
                                                     factors, slot_stride, status, chunk);
  else if (nslots == 1)  // one candidate (model building, B=1): no padded ILP groups of copies
    assemble_kernel<MAXD, false, 1><<<grid, 256, 0, s>>>(table, theta, n, d, nugget, NT, slots, nslots, jitter,
                                                         factors, slot_stride, status, chunk);
  else
    assemble_kernel<MAXD, false><<<grid, 256, 0, s>>>(table, theta, n, d, nugget, NT, slots, nslots, jitter,
                                                      factors, slot_stride, status, chunk);
}

void launch_assemble(const double* table, const double* theta, const double* y, int n, int d,
                     double nugget, int NT, const int* slots, int nslots, const double* jitter,
                     double* factors, size_t slot_stride, double* borders, int* status,
                     int num_sms, cudaStream_t s) {
  const int Npad = NT * TILE;
  border_init_kernel<<<dim3((Npad + 255) / 256 < 32 ? (Npad + 255) / 256 : 32, nslots), 256, 0, s>>>(
      y, n, Npad, slots, borders, status);
  // at least ~8 blocks per SM on small designs (n=200 has 3 tiles: 24 blocks with a fixed 8),
  // at most one element per thread per slot chunk (TILE_ELEMS / 256 = 64)
  const int tiles = num_tiles(NT);
  const int gy = std::min(64, std::max(8, (8 * num_sms + tiles - 1) / tiles));
  // Small designs (n=200: 3 tiles, 192 blocks) are too few blocks to keep the R stores in flight:
  // split the candidates over blockIdx.z as well (each block then reloads its elements' table
  // values, which large designs avoid). C1: 33 -> ~10 us per batch.
  int chunk = kAsmSlotChunk, gz = 1;
  if (tiles * gy < 4 * num_sms && nslots > 8) {
    gz = std::min((nslots + 7) / 8, (4 * num_sms + tiles * gy - 1) / (tiles * gy));
    chunk = std::min(kAsmSlotChunk, ((nslots + gz - 1) / gz + 7) / 8 * 8);
    gz = (nslots + chunk - 1) / chunk;
  }
  const dim3 grid(tiles, gy, gz);
  // theta entries beyond d are zero in shared memory, so a looser bound is only slower
#define GPEMU_ASM(D) \
  launch_asm<D>(grid, s, table, theta, n, d, nugget, NT, slots, nslots, jitter, factors, slot_stride, status, chunk)
  if (d <= 1) GPEMU_ASM(1);
  else if (d <= 2) GPEMU_ASM(2);
  else if (d <= 3) GPEMU_ASM(3);
  else if (d <= 4) GPEMU_ASM(4);
  else if (d <= 6) GPEMU_ASM(6);
  else if (d <= 8) GPEMU_ASM(8);
  else if (d <= 10) GPEMU_ASM(10);
  else if (d <= 12) GPEMU_ASM(12);
  else if (d <= 16) GPEMU_ASM(16);
  else if (d <= 20) GPEMU_ASM(20);
  else if (d <= 24) GPEMU_ASM(24);
  else if (d <= 32) GPEMU_ASM(32);
  else
    assemble_generic_kernel<<<dim3(grid.x, grid.y), 256, 0, s>>>(table, theta, n, d, nugget, NT, slots, nslots, jitter,
                                                 factors, slot_stride, status);
#undef GPEMU_ASM
}

// build_corr_matrix (correlation.hpp:99-146): row-major, strict lower computed
// once and mirrored.
__global__ void build_corr_rowmajor_kernel(const double* __restrict__ X, int n, int d,
                                           const double* __restrict__ theta, double p,
                                           double nugget, double* __restrict__ R, int* bad) {
  const int i = blockIdx.y;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= i; j += gridDim.x * blockDim.x) {
    if (j == i) {
      R[(size_t)i * n + i] = __dadd_rn(1.0, nugget);
      continue;
    }
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double term = pow_abs(X[(size_t)i * d + k] - X[(size_t)j * d + k], p);
      s = __dadd_rn(s, __dmul_rn(theta[k], term));
    }
    const double v = exp_neg(s);
    if (!isfinite(v) || isnan(s)) *bad = 1;
    R[(size_t)i * n + j] = v;
    R[(size_t)j * n + i] = v;
  }
}

void launch_build_corr_rowmajor(const double* X, int n, int d, const double* theta, double p,
                                double nugget, double* R, int* bad, cudaStream_t s) {
  dim3 grid((n + 255) / 256, n);
  build_corr_rowmajor_kernel<<<grid, 256, 0, s>>>(X, n, d, theta, p, nugget, R, bad);
}

// corr_vector (correlation.hpp:67-91) for N test points: r[j*n + i].
__global__ void corr_vectors_kernel(const double* __restrict__ Xt, int N,
                                    const double* __restrict__ X, int n, int d,
                                    const double* __restrict__ theta, double p,
                                    double* __restrict__ r, int* bad) {
  const int j = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double term = pow_abs(Xt[(size_t)j * d + k] - X[(size_t)i * d + k], p);
      s = __dadd_rn(s, __dmul_rn(theta[k], term));
    }
    const double v = exp_neg(s);
    if (!isfinite(v) || isnan(s)) *bad = 1;
    r[(size_t)j * n + i] = v;
  }
}

void launch_corr_vectors(const double* Xt, int N, const double* X, int n, int d,
                         const double* theta, double p, double* r, int* bad, cudaStream_t s) {
  dim3 grid((n + 255) / 256, N);
  corr_vectors_kernel<<<grid, 256, 0, s>>>(Xt, N, X, n, d, theta, p, r, bad);
}

}  // namespace gpemu_dev
