// kernels_trsv.cu -- blocked triangular solve on the packed tile factor (one right-hand side).
//
// Reference (relative to /root/reference/proj/include/gpemu/):
//   solve_lower_into   backend.hpp:129-140   L x = b, forward substitution
//   solve_upper_into   backend.hpp:143-153   L^T x = b, backward substitution
//   solve_full         backend.hpp:163-169   alpha = (R + jI)^-1 (y - mu 1), likelihood.hpp:226-230
//
// The reference substitutes one unknown at a time over a dense row-major L. Here the factor
// stays in the engine's packed lower 128 x 128 tiles and the solve is blocked by tile:
//   forward  x_I = L_II^-1  (b_I - sum_{J<I} L_IJ   x_J)
//   backward x_J = L_JJ^-T  (b_J - sum_{I>J} L_IJ^T x_I)
// A persistent kernel takes blocks in dependency order from a ticket counter (a block only waits
// on lower tickets, so it is deadlock-free without co-residency). Per block:
//   * the diagonal tile goes to shared memory by TMA (cp.async.bulk) when the block starts;
//   * the off-diagonal tiles stream from HBM with coalesced 256 B rows, each tile's loads
//     issued BEFORE waiting for the x block it multiplies, so only the last tile's FMAs and
//     one reduction sit on the dependency chain;
//   * one warp substitutes the 128 unknowns from shared memory (lane owns rows l + 32m; the
//     quotient is s * (1/L_ii) with one FMA correction, i.e. the division's rounding without
//     the DDIV sequence), then publishes the block with a release flag (epoch-valued, nothing
//     is cleared between launches).
// The solve is chain-bound: NT dependent block solves of 128 serial substitution steps. The L
// read (n^2/2 doubles) overlaps the chain. For alpha the right-hand side is formed in the
// kernel from the factor's border rows: L^-1 (y - mu 1) = u - mu v, so only the backward solve
// runs (the reference runs a forward solve first).
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.h"
#include "layout.cuh"
#include "ptx.cuh"

namespace gpemu_dev {

namespace {

constexpr int kThreads = 256;
constexpr long long kTrsvSpinLimit = 20000000000LL;  // ~10 s at 1.9 GHz: deadlock guard

struct TrsvSmem {
  double diag[TILE_ELEMS];   // L_BB (swizzled slab layout, as in HBM)
  double red[8][TILE];       // per-warp partial sums
  double xs[TILE];           // the x block being multiplied
  double rb[TILE];           // right-hand side of the block (b_B - partial)
  uint64_t bar;              // diag tile TMA barrier
  int ticket;
};

__device__ __forceinline__ bool wait_epoch(const int* flag, int epoch, int* error) {
  if (ld_acquire_gpu(flag) == epoch) return true;
  const long long t0 = clock64();
  while (ld_acquire_gpu(flag) != epoch) {
    __nanosleep(32);
    if (clock64() - t0 > kTrsvSpinLimit) {
      atomicExch(error, 1);
      return false;
    }
  }
  return true;
}

// q = s / d with d_inv = 1 / d: one corrected product (the quotient's rounding without DDIV).
__device__ __forceinline__ double quot(double s, double d, double d_inv) {
  const double q = s * d_inv;
  return fma(fma(-q, d, s), d_inv, q);
}

template <bool upper>
__global__ void __launch_bounds__(kThreads, 1) tile_trsv_kernel(
    const double* __restrict__ tiles, int NT, const double* __restrict__ b,
    const double* __restrict__ b2, double mu, int nb, double* __restrict__ x,
    int* __restrict__ flags, int* __restrict__ counter, int epoch, int* __restrict__ error) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TrsvSmem& S = *reinterpret_cast<TrsvSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    fence_mbar_init();
  }
  uint32_t phase = 0;
  for (;;) {
    __syncthreads();  // previous block's shared memory reads are done
    if (tid == 0) S.ticket = atomicAdd(counter, 1);
    __syncthreads();
    const int t = S.ticket;
    if (t >= NT) break;
    const int B = upper ? NT - 1 - t : t;
    if (tid == 0) {
      fence_proxy_async_shared();
      mbar_arrive_expect_tx(&S.bar, TILE_ELEMS * sizeof(double));
      const double* src = tiles + tile_index(B, B) * TILE_ELEMS;
#pragma unroll
      for (int s = 0; s < SLABS_PER_TILE; ++s)
        bulk_g2s(S.diag + s * SLAB_ELEMS, src + s * SLAB_ELEMS, SLAB_ELEMS * sizeof(double), &S.bar);
    }
    if (tid < TILE) {
      const int i = B * TILE + tid;
      double r = 0.0;
      if (i < nb) r = b2 ? fma(-mu, b2[i], b[i]) : b[i];
      S.rb[tid] = r;
    }
    // ---- off-diagonal tiles: partial = sum_dep L-tile (x)_dep ----
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    const int ndep = upper ? NT - 1 - B : B;
    for (int k = 0; k < ndep; ++k) {
      // dependency in readiness order: forward J = 0, 1, ...; backward I = NT-1, NT-2, ...
      const int D = upper ? NT - 1 - k : k;
      const double* tl = tiles + (upper ? tile_index(D, B) : tile_index(B, D)) * TILE_ELEMS;
      double v[64];
      if constexpr (upper) {
        // lane = column c of each slab, warp = rows 16w..16w+15: one 256 B row per load
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int rr = 0; rr < 16; ++rr) {
            const int r = warp * 16 + rr;
            v[s * 16 + rr] = __ldcs(tl + s * SLAB_ELEMS + slab_off(r, lane));
          }
      } else {
        // warp = rows 16w..16w+15 (512 contiguous doubles per slab), lane = a double2 of
        // row 16w + 2i + (lane >> 4)
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const double2 p =
                __ldcs(reinterpret_cast<const double2*>(tl + s * SLAB_ELEMS + warp * 512 + i * 64) + lane);
            v[s * 16 + 2 * i] = p.x;
            v[s * 16 + 2 * i + 1] = p.y;
          }
      }
      if (tid == 0) wait_epoch(flags + D, epoch, error);
      __syncthreads();
      if (tid < TILE) S.xs[tid] = __ldcg(x + (size_t)D * TILE + tid);
      __syncthreads();
      if constexpr (upper) {
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int rr = 0; rr < 16; ++rr) acc[s] = fma(v[s * 16 + rr], S.xs[warp * 16 + rr], acc[s]);
      } else {
        const int w2 = (2 * lane) & 31;
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = warp * 16 + 2 * i + (lane >> 4);
            const int c = s * 32 + ((((w2 >> 2) ^ (r & 7))) << 2) + (w2 & 3);
            acc[i] = fma(v[s * 16 + 2 * i], S.xs[c], acc[i]);
            acc[i] = fma(v[s * 16 + 2 * i + 1], S.xs[c + 1], acc[i]);
          }
      }
    }
    // ---- reduce the partials into rb ----
    if (ndep > 0) {
      if constexpr (upper) {
#pragma unroll
        for (int s = 0; s < 4; ++s) S.red[warp][s * 32 + lane] = acc[s];
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          double a = acc[i];
          a += __shfl_xor_sync(0xffffffffu, a, 1);
          a += __shfl_xor_sync(0xffffffffu, a, 2);
          a += __shfl_xor_sync(0xffffffffu, a, 4);
          a += __shfl_xor_sync(0xffffffffu, a, 8);
          acc[i] = a;
        }
        // lanes 0 / 16 hold rows 16w + 2i / 16w + 2i + 1
        if ((lane & 15) == 0)
#pragma unroll
          for (int i = 0; i < 8; ++i) S.red[0][warp * 16 + 2 * i + (lane >> 4)] = acc[i];
      }
      __syncthreads();
      if (tid < TILE) {
        double p;
        if constexpr (upper) {
          p = S.red[0][tid];
#pragma unroll
          for (int w = 1; w < 8; ++w) p += S.red[w][tid];
        } else {
          p = S.red[0][tid];
        }
        S.rb[tid] -= p;
      }
    }
    __syncthreads();
    // ---- diagonal block: one warp substitutes ----
    if (warp == 0) {
      mbar_wait(&S.bar, phase);
      double r[4], dg[4], di[4], xr[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int i = lane + 32 * m;
        r[m] = S.rb[i];
        dg[m] = S.diag[elem_off(i, i)];
        di[m] = 1.0 / dg[m];
        xr[m] = 0.0;
      }
      if constexpr (!upper) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
#pragma unroll
          for (int o = 0; o < 32; ++o) {
            const int c = 32 * m + o;
            double xc = 0.0;
            if (lane == o) {
              xc = quot(r[m], dg[m], di[m]);
              xr[m] = xc;
            }
            xc = __shfl_sync(0xffffffffu, xc, o);
#pragma unroll
            for (int m2 = m; m2 < 4; ++m2) {
              const double l = S.diag[elem_off(lane + 32 * m2, c)];
              if (m2 > m || lane > o) r[m2] = fma(-l, xc, r[m2]);
            }
          }
        }
      } else {
#pragma unroll
        for (int m = 3; m >= 0; --m) {
#pragma unroll
          for (int o = 31; o >= 0; --o) {
            const int j = 32 * m + o;
            double xj = 0.0;
            if (lane == o) {
              xj = quot(r[m], dg[m], di[m]);
              xr[m] = xj;
            }
            xj = __shfl_sync(0xffffffffu, xj, o);
#pragma unroll
            for (int m2 = 0; m2 <= m; ++m2) {
              const double l = S.diag[elem_off(j, lane + 32 * m2)];
              if (m2 < m || lane < o) r[m2] = fma(-l, xj, r[m2]);
            }
          }
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) x[(size_t)B * TILE + lane + 32 * m] = xr[m];
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        st_release_gpu(flags + B, epoch);
      }
    }
    phase ^= 1u;
  }
}

}  // namespace

size_t tile_trsv_smem_bytes() { return sizeof(TrsvSmem); }

void launch_tile_trsv(const double* tiles, int NT, const double* b, const double* b2, double mu,
                      int nb, double* x, int upper, int* flags, int* counter, int epoch,
                      int* error, int num_sms, cudaStream_t s) {
  const int smem = (int)sizeof(TrsvSmem);
  cudaMemsetAsync(counter, 0, sizeof(int), s);
  int grid = NT < num_sms ? NT : num_sms;
  // test hook: fewer CTAs than blocks exercises the persistent ticket loop at small n
  if (const char* e = std::getenv("GPEMU_TRSV_MAX_GRID")) {
    const int g = std::atoi(e);
    if (g > 0 && g < grid) grid = g;
  }
  if (upper) {
    cudaFuncSetAttribute(tile_trsv_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tile_trsv_kernel<true><<<grid, kThreads, smem, s>>>(tiles, NT, b, b2, mu, nb, x, flags, counter,
                                                         epoch, error);
  } else {
    cudaFuncSetAttribute(tile_trsv_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tile_trsv_kernel<false><<<grid, kThreads, smem, s>>>(tiles, NT, b, b2, mu, nb, x, flags, counter,
                                                          epoch, error);
  }
}

}  // namespace gpemu_dev
