// kernels_chol.cu -- K2: batched FP64 Cholesky of R + jitter*I on sm_100a.
//
// Reference: backend.hpp (relative to /root/reference/proj/include/gpemu/)
//   factorize_into     :102-120  jitter ladder, pivot test !(s > 0), log-det
//   ReferenceBackend   :189-206  unblocked dot-product Cholesky
//   ParallelBackend    :226-311  right-looking 64-blocked Cholesky
//   solve_lower_into   :129-140  u = L^-1 y, v = L^-1 1 (likelihood.hpp:122-123)
//
// Two engines over the same tiled HBM layout (layout.cuh):
//
// * chol_dag_kernel -- the product engine. A persistent kernel (one CTA per SM)
//   pulls tasks from a global ticket counter. The task order is a topological
//   order of the left-looking tile Cholesky of every candidate in the batch,
//   with a one-column lookahead (the diagonal task of column j+1 is issued within
//   the column-j group, after the task that produces its last input), so waits
//   only ever target lower tickets (deadlock free) and the serial panel chain of
//   one candidate is hidden behind the other candidates' work.
//     DIAG(b, j):  C = R(j,j) - sum_{K<j} L(j,K) L(j,K)^T     (DMMA)
//                  L(j,j) = chol(C)      blocked 16-wide in shared memory
//                  border rows: [u_j; v_j] = ([y_j; 1_j] - sum_K [u_K; v_K] L(j,K)^T) L(j,j)^-T
//   (every update is applied as a running residual: accumulators start at R)
//     OFF(b, j, I): C = R(I,j) - sum_{K<j} L(I,K) L(j,K)^T    (DMMA)
//                  L(I,j) = C L(j,j)^-T  blocked 16-wide (substitution + DMMA updates)
//   The two forward solves of the reference are the bordered rows [y 1]^T of
//   the factorization, so u and v fall out of the same tile pass and the solves
//   never re-read L. Operand k-slabs (128 x 32 doubles, 32 KB) are streamed by a
//   producer warp with cp.async.bulk (TMA) into a 3-stage mbarrier ring; eight
//   consumer warps run m8n8k4 DMMA on a 128x128 accumulator tile (64x32 per warp).
//   Two instantiations (launch_chol_dag picks by tickets per CTA):
//   * chol_dag_kernel<false> (throughput-bound batches such as a GA generation): a CTA takes
//     its next ticket at mainloop end and bulk-prefetches that task's R tile into L2;
//   * chol_dag_kernel<true> (B=1 models, refine batches: bound by each candidate's serial
//     chain): the sub-diagonal tile L(j+1,j) is released slab by slab so DIAG(j+1)'s last
//     k-step overlaps its TRSM.
//   Both produce bitwise the same factor.
//
// * chol_simple_kernel -- validation engine: one CTA per candidate, unblocked
//   right-looking, products and differences rounded separately, so on identical
//   R it reproduces the reference's arithmetic order bit for bit.
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels.h"
#include "layout.cuh"
#include "ptx.cuh"

namespace gpemu_dev {

// ============================================================================
// Simple engine
// ============================================================================

__device__ __forceinline__ double* tile_elem(double* base, int i, int j) {
  return base + tile_index(i >> 7, j >> 7) * TILE_ELEMS + elem_off(i & 127, j & 127);
}

__global__ void __launch_bounds__(1024) chol_simple_kernel(DagLaunch a) {
  const int slot = a.slots[blockIdx.x];
  double* base = a.factors + (size_t)slot * a.slot_stride;
  const int Npad = a.NT * TILE;
  double* u = a.borders + (size_t)slot * 2 * Npad;
  double* v = u + Npad;
  __shared__ double dsh;
  __shared__ int fail;
  if (threadIdx.x == 0) fail = (a.status[slot] != 0);
  __syncthreads();
  if (fail) return;
  for (int k = 0; k < Npad; ++k) {
    if (threadIdx.x == 0) {
      const double s = *tile_elem(base, k, k);
      if (!(s > 0.0)) {
        fail = 1;
      } else {
        const double dd = sqrt(s);
        *tile_elem(base, k, k) = dd;
        dsh = dd;
      }
    }
    __syncthreads();
    if (fail) break;
    const double dd = dsh;
    for (int i = k + 1 + threadIdx.x; i < Npad; i += blockDim.x) {
      double* p = tile_elem(base, i, k);
      *p = *p / dd;
    }
    if (threadIdx.x == 0) {
      u[k] = u[k] / dd;
      v[k] = v[k] / dd;
    }
    __syncthreads();
    const int m = Npad - k - 1;
    const long long npairs = (long long)m * (m + 1) / 2;
    for (long long q = threadIdx.x; q < npairs; q += blockDim.x) {
      int ii = (int)((sqrt(8.0 * (double)q + 1.0) - 1.0) * 0.5);
      while ((long long)(ii + 1) * (ii + 2) / 2 <= q) ++ii;
      while ((long long)ii * (ii + 1) / 2 > q) --ii;
      const int ll = (int)(q - (long long)ii * (ii + 1) / 2);
      const int i = k + 1 + ii, l = k + 1 + ll;
      double* p = tile_elem(base, i, l);
      *p = __dsub_rn(*p, __dmul_rn(*tile_elem(base, i, k), *tile_elem(base, l, k)));
    }
    for (int l = k + 1 + threadIdx.x; l < Npad; l += blockDim.x) {
      const double lk = *tile_elem(base, l, k);
      u[l] = __dsub_rn(u[l], __dmul_rn(u[k], lk));
      v[l] = __dsub_rn(v[l], __dmul_rn(v[k], lk));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && fail) a.status[slot] = 1;  // GPEMU_SLOT_NOT_PD
}

void launch_chol_simple(const DagLaunch& a, cudaStream_t s) {
  chol_simple_kernel<<<a.nslots, 1024, 0, s>>>(a);
}

// ============================================================================
// DAG engine
// ============================================================================

namespace {
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;  // 256
constexpr int kThreads = kConsumers;             // thread 0 also issues the TMA loads
constexpr int kStages = 3;
constexpr int kSlabBytes = SLAB_ELEMS * 8;              // 32 KB
constexpr int kStageBytes = 2 * kSlabBytes;             // A + B slab
constexpr int kOffStages = 0;                           // [0, 192K)
constexpr int kOffC = 0;                                // epilogue tile [0, 128K)
constexpr int kOffBar = kStages * kStageBytes;          // 192K: mbarriers
constexpr int kOffW = kOffBar + 256;                    // border w: 2 x 128 doubles
constexpr int kOffRinvD = kOffW + 2 * TILE * 8;        // 1 / L_cc of the DIAG tile
constexpr int kOffMisc = kOffRinvD + TILE * 8;          // task scalars
constexpr long long kSpinLimitCycles = 20000000000LL;  // ~10 s: declare deadlock
constexpr int kStageLd = 18;  // row stride (doubles) of the per-warp TRSM staging block
// The OFF-task TRSM keeps its staging blocks and the packed diagonal blocks of L(j,j) above
// the ring (L(j,j) itself occupies stages 0-1), so stage 2 stays free during the TRSM and
// takes the next task's first slab.
constexpr int kOffTrsmSt = kOffMisc + 160;                                  // [8 warps][16][kStageLd]
constexpr int kTriElems = 136;                                              // packed 16x16 lower
constexpr int kOffTrsmD = kOffTrsmSt + kConsumerWarps * 16 * kStageLd * 8;  // [8][kTriElems]
constexpr int kSmemBytes = kOffTrsmD + 8 * kTriElems * 8;
static_assert(kSmemBytes <= 227 * 1024, "shared memory");

struct Misc {  // per-task scalars in shared memory (kept out of the mainloop's registers)
  int ticket;
  int skip;
  int fail;
  int bpos;
  int I, j;
  unsigned ljj_phase;  // uses of ljj_bar (the OFF-task L(j,j) load)
  int next;           // ticket taken ahead (prefetch of its seed tile), -1: none
  long long t_begin;   // PR_TOTAL start (profiling)
  unsigned ready[16];  // K-tiles 1..255 whose operand flags were published at task start
  int pre_next;        // the previous task issued slab 0 of ticket `next` into stage 2
  int pre;             // this task's slab 0 is in stage 2 already
  int run;             // OFF task: the candidate was still unfailed at the TRSM start
  int pcnt[4];         // DIAG: warp blocks of each L(j,j) slab stored (progressive publication)
  int ljj_issued;      // OFF (chain-bound launches): L(j,j) slabs whose loads are issued
  int freed[3];        // DIAG (chain-bound): slab + 1 whose ring stage's refill was decided
  int pend[3];         // ... and was deferred (its progress flags were not yet published)
};
static_assert(sizeof(Misc) <= 160, "Misc overlaps the TRSM staging area");

__device__ __forceinline__ void consumer_sync() { named_bar_sync(1, kConsumers); }

// Spin until *flag == epoch (acquire). On timeout record an error and proceed.
__device__ __forceinline__ void wait_flag(const int* flag, int epoch, int* error) {
  if (ld_acquire_gpu(flag) == epoch) return;
  const long long t0 = clock64();
  while (ld_acquire_gpu(flag) != epoch) {  // tight spin: each poll is an L2 round trip anyway
    if (clock64() - t0 > kSpinLimitCycles) {
      atomicExch(error, 1);
      return;
    }
  }
}

// Spin until *flag >= target (acquire): the slab-progress word of a sub-diagonal tile.
__device__ __forceinline__ void wait_flag_geq(const int* flag, int target, int* error) {
  if (ld_acquire_gpu(flag) >= target) return;
  const long long t0 = clock64();
  while (ld_acquire_gpu(flag) < target) {  // (a 64 ns back-off cost 0.4% on a B=1 evaluation)
    if (clock64() - t0 > kSpinLimitCycles) {
      atomicExch(error, 1);
      return;
    }
  }
}

__device__ __forceinline__ void publish_flag(int* flag, int epoch) {
  __threadfence();
  fence_proxy_async_global();
  st_release_gpu(flag, epoch);
}

// Optional per-CTA phase cycle counters (DagLaunch::prof, null in production).
enum {
  PR_TICKET = 0, PR_GEMM, PR_ACC_STORE, PR_POTRF, PR_DIAG_STORE, PR_BORDER, PR_OFF_WAIT, PR_TRSM,
  PR_OFF_STORE, PR_TASK_END, PR_PROD_FLAGS, PR_PROD_EMPTY, PR_N_DIAG, PR_N_OFF, PR_SLABS, PR_TOTAL,
  PR_FULL_WAIT, PR_DIAG_FULL_WAIT, PR_DIAG_GEMM, PR_P_PIV, PR_P_BDW, PR_P_PANEL, PR_P_BPW, PR_P_UPD,
  PR_COUNT_USED
};
constexpr int PR_COUNT = 24;
struct Prof {
  unsigned long long* p;
  long long last;
  __device__ __forceinline__ void start() {
    if (p) last = clock64();
  }
  __device__ __forceinline__ void lap(int k) {
    if (p) {
      const long long now = clock64();
      p[k] += (unsigned long long)(now - last);
      last = now;
    }
  }
  __device__ __forceinline__ void add(int k, unsigned long long v) {
    if (p) p[k] += v;
  }
};

// Task decode (see header comment): ticket -> (bpos, j, I).
__device__ __forceinline__ void decode_task(int t, int B, int NT, int& bpos, int& j, int& I) {
  if (t < B) {
    bpos = t;
    j = 0;
    I = 0;
    return;
  }
  t -= B;
  int jj = 0;
  while (true) {
    const int g = B * (NT - jj);
    if (t < g) break;
    t -= g;
    ++jj;
  }
  // candidate bpos, column group jj: OFF(jj+1, jj) first (DIAG(jj+1)'s last input), the other
  // OFF(I, jj), then DIAG(jj+1) last -- by the time a CTA takes it, OFF(jj+1, jj) is usually
  // done, so the CTA does not idle on the flag (-0.3% at C3 vs DIAG right after it)
  const int per = NT - jj;
  bpos = t / per;
  const int pos = t - bpos * per;
  if (pos == 0) {
    j = jj;
    I = jj + 1;
  } else if (pos == per - 1) {
    j = jj + 1;
    I = jj + 1;
  } else {
    j = jj;
    I = jj + pos + 1;
  }
}

// ticket -> task through the launch's order table when it has one
__device__ __forceinline__ void task_of(const int* order, int t, int B, int NT, int& bpos, int& j, int& I) {
  if (order) {
    const int v = __ldg(order + t);
    bpos = v >> 16;
    I = (v >> 8) & 255;
    j = v & 255;
  } else {
    decode_task(t, B, NT, bpos, j, I);
  }
}

// Offset (tile layout) of the double pair (row r, cols 8 ni + 2 lc + {0,1}) held by a
// DMMA accumulator fragment.
__device__ __forceinline__ int acc_off(int r, int ni, int lc) {
  return ((ni >> 2) << 12) + r * 32 + (((2 * (ni & 3) + (lc >> 1)) ^ (r & 7)) << 2) + 2 * (lc & 1);
}


// a / d given r = 1/d: the rounding of a true division (a*r + one FMA residual
// correction) without the DDIV call sequence.
__device__ __forceinline__ double div_by(double a, double d, double r) {
  const double x0 = a * r;
  return fma(fma(-x0, d, a), r, x0);
}

// ---- register-layout helpers: warp w owns rows [16w, 16w+16) as acc[2][16][2] ----------
// (acc[mi][ni] = rows 8mi + lr, cols 8ni + 2lc + {0,1}; the "window" block is ni = 0..1)

// window block (16 x 16) <-> per-warp staging St[16][kStageLd] (row r at St + r*kStageLd)
__device__ __forceinline__ void stage_out(const double (&acc)[2][16][2], double* St, int lr, int lc) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nsub = 0; nsub < 2; ++nsub)
      *reinterpret_cast<double2*>(St + (8 * mi + lr) * kStageLd + 8 * nsub + 2 * lc) =
          make_double2(acc[mi][nsub][0], acc[mi][nsub][1]);
}
__device__ __forceinline__ void stage_in(double (&acc)[2][16][2], const double* St, int lr, int lc) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nsub = 0; nsub < 2; ++nsub) {
      const double2 v = *reinterpret_cast<const double2*>(St + (8 * mi + lr) * kStageLd + 8 * nsub + 2 * lc);
      acc[mi][nsub][0] = v.x;
      acc[mi][nsub][1] = v.y;
    }
}

// solve_row16 with D packed lower (row r at r(r+1)/2): the same operations in the same order.
__device__ __forceinline__ void solve_row16p(double (&xr)[16], const double* D, const double* ri) {
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    xr[c] = div_by(xr[c], D[c * (c + 1) / 2 + c], ri[c]);
#pragma unroll
    for (int c2 = c + 1; c2 < 16; ++c2) xr[c2] -= xr[c] * D[c2 * (c2 + 1) / 2 + c];
  }
}

// One lane owns one row (16 values) of a block: X = B D^-T with D dense lower [16][16]
// (warp-uniform broadcast loads) and ri[c] = 1 / D[c][c].
__device__ __forceinline__ void solve_row16(double (&xr)[16], const double* D, const double* ri) {
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    xr[c] = div_by(xr[c], D[c * 16 + c], ri[c]);
#pragma unroll
    for (int c2 = c + 1; c2 < 16; ++c2) xr[c2] -= xr[c] * D[c2 * 16 + c];
  }
}

__device__ __forceinline__ void load_row16(double (&xr)[16], const double* row) {
#pragma unroll
  for (int c = 0; c < 16; c += 2) {
    const double2 v = *reinterpret_cast<const double2*>(row + c);
    xr[c] = v.x;
    xr[c + 1] = v.y;
  }
}
__device__ __forceinline__ void store_row16(const double (&xr)[16], double* row) {
#pragma unroll
  for (int c = 0; c < 16; c += 2) *reinterpret_cast<double2*>(row + c) = make_double2(xr[c], xr[c + 1]);
}

// Negated A fragments (m8n8k4, k = window columns) of the window block, from the
// accumulator layout by quad shuffles.
__device__ __forceinline__ void window_afrags(const double (&acc)[2][16][2], double (&av)[2][4], int lane) {
  const int lc = lane & 3, qbase = lane & ~3;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int src = qbase | (2 * (ks & 1) + (lc >> 1));
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const double v0 = __shfl_sync(0xffffffffu, acc[mi][ks >> 1][0], src);
      const double v1 = __shfl_sync(0xffffffffu, acc[mi][ks >> 1][1], src);
      av[mi][ks] = -((lc & 1) ? v1 : v0);
    }
  }
}

// The same three helpers for a window at absolute n-tile w (fully unrolled callers: no
// register rotation needed).
__device__ __forceinline__ void stage_out_at(const double (&acc)[2][16][2], int w, double* St, int lr, int lc) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nsub = 0; nsub < 2; ++nsub)
      *reinterpret_cast<double2*>(St + (8 * mi + lr) * kStageLd + 8 * nsub + 2 * lc) =
          make_double2(acc[mi][w + nsub][0], acc[mi][w + nsub][1]);
}
__device__ __forceinline__ void stage_in_at(double (&acc)[2][16][2], int w, const double* St, int lr, int lc) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int nsub = 0; nsub < 2; ++nsub) {
      const double2 v = *reinterpret_cast<const double2*>(St + (8 * mi + lr) * kStageLd + 8 * nsub + 2 * lc);
      acc[mi][w + nsub][0] = v.x;
      acc[mi][w + nsub][1] = v.y;
    }
}
__device__ __forceinline__ void window_afrags_at(const double (&acc)[2][16][2], int w, double (&av)[2][4], int lane) {
  const int lc = lane & 3, qbase = lane & ~3;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int src = qbase | (2 * (ks & 1) + (lc >> 1));
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const double v0 = __shfl_sync(0xffffffffu, acc[mi][w + (ks >> 1)][0], src);
      const double v1 = __shfl_sync(0xffffffffu, acc[mi][w + (ks >> 1)][1], src);
      av[mi][ks] = -((lc & 1) ? v1 : v0);
    }
  }
}

__device__ __forceinline__ void rotate_window(double (&acc)[2][16][2]) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 14; ++ni) {
      acc[mi][ni][0] = acc[mi][ni + 2][0];
      acc[mi][ni][1] = acc[mi][ni + 2][1];
    }
}

// Dense panel buffer [128][16] with the 4-double chunks of row r XOR-swizzled by (r & 3).
__device__ __forceinline__ int p_off(int r, int c) {
  return r * 16 + ((((c >> 2) ^ (r & 3)) << 2) | (c & 3));
}

// Pivot root and reciprocal without the sqrt / DDIV call sequences: y ~ 1/sqrt(s) from
// rsqrt.approx.f64, which sm_100a implements as MUFU.RSQ64H plus one refinement (max relative
// error 2^-53 measured, tools/probes/rsqrt_acc.cu), d = s*y corrected once (Markstein: the
// correctly rounded sqrt except in rare ties), r = y as the approximate reciprocal that
// div_by corrects with one FMA residual. Evaluated redundantly by every lane from the
// broadcast pivot.
__device__ __forceinline__ void pivot_root(double s, double& d, double& r) {
  double y;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(s));
  const double d0 = s * y;
  d = fma(fma(-d0, d0, s), 0.5 * y, d0);
  r = y;
}

// In-register Cholesky of a 16x16 diagonal block, lane r (< 16) holding row r in xr.
// Right-looking, branch-free and register-only: the quotients of column c are broadcast by
// shuffles, and the next pivot (lane c+1's diagonal minus its own quotient squared) is
// formed and rooted before column c's updates are applied, so the serial pivot chain is
// shfl -> root -> div -> fma with the updates filling its latency. Every lower-triangle
// element gets the same operations in the same order as a column-by-column right-looking
// loop; the upper triangle of xr is left undefined (never read). Pivot reciprocals ->
// rinv[0..15]. Returns false (uniform) on a failed pivot (backend.hpp:238).
__device__ __forceinline__ bool potrf_row16(double (&xr)[16], double* rinv, int lane, double* qs) {
  double d, r;
  const double s = __shfl_sync(0xffffffffu, xr[0], 0);
  bool ok = s > 0.0;  // uniform: every lane sees the same pivots
  // (after a failed pivot the arithmetic runs on with NaN / inf: the block is discarded, and
  // keeping the compare and select off the pivot chain saves their latency every column)
  pivot_root(s, d, r);
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const double q = div_by(xr[c], d, r);
    if (lane == c) rinv[c] = r;
    xr[c] = lane > c ? q : (lane == c ? d : xr[c]);
    if (c < 15) {  // the next pivot first: it depends only on lane c+1's own quotient
      const double sn = __shfl_sync(0xffffffffu, fma(-q, q, xr[c + 1]), c + 1);
      ok = ok && sn > 0.0;
      pivot_root(sn, d, r);
    }
    // column c's quotients to every lane through shared memory (one STS per lane, broadcast
    // LDS): 15 - c double shuffles per column made the block 1.65x slower
    // (tools/microbench/potrf16.cu: 7.6k -> 4.6k cycles); double-buffered by column parity
    if (lane < 16) qs[16 * (c & 1) + lane] = q;
    __syncwarp();
#pragma unroll
    for (int c2 = c + 1; c2 < 16; ++c2) xr[c2] = fma(-q, qs[16 * (c & 1) + c2], xr[c2]);
  }
  return ok;
}

// C tile accessors in shared memory (tile layout).
__device__ __forceinline__ double& Cs(double* C, int r, int c) { return C[elem_off(r, c)]; }

// Unblocked 16x16 Cholesky of the diagonal block at offset o (warp 0, lanes < 16).
// Returns false (uniform across the warp) on a failed pivot.


// DIAG-task POTRF of the 128x128 tile C (tile layout in shared memory, = R - sum L L^T):
// blocked right-looking in the register layout, warp w owning rows 16w..16w+15, with a one-
// block look-ahead. Step kb: warp kb factors its 16x16 diagonal block in registers (one lane
// per row) and releases it (named barrier BD); each warp w > kb solves its panel block against
// it and publishes it to a dense panel buffer; warp kb+1 then updates only its own diagonal
// block with its own panel and goes on to factor step kb+1 at once, while warps > kb+1 wait
// for all step-kb panels (named barrier BP) and update their trailing columns with DMMA. The
// serial chain per step is factor -> one panel solve -> one 16x16 update (the trailing
// updates of the other warps run under the next factorization). Every element gets the same
// operations in the same order as without the look-ahead. Each warp moves its block of the
// step into the row layout before it waits for the pivot, and the look-ahead warp leaves the
// step loop into its own pivot step carrying only its diagonal block, so the accumulators are
// dead on the chain (C3 -0.3%, B=1 -1.6%). BD is split: the look-ahead warp waits only for
// the pivot (named barrier 8/9), the warps below it on their own barrier. Pivot blocks and
// panels are double-
// buffered by step parity (the barriers keep any warp within one step of its readers).
// Finished blocks are written back into C. Reciprocal pivots -> rinvD[0..127]. Returns false
// on a failed pivot (uniform): the factorization stops at that step with the barriers balanced,
// and the tile is discarded.
__device__ __noinline__ bool diag_potrf(unsigned char* smem, double* C, double* rinvD, double* W, Misc* misc,
                                        int warp, int lane, unsigned long long* pp, double* gt, int* prog,
                                        int pbase, double* bg, int npad, int* bprog) {
  const int lr = lane >> 2, lc = lane & 3;
  // Row block of this warp: blocks 2i and 2i+1 on warps i and i+4, i.e. on the same SM
  // sub-partition (warp w issues from SMSP w % 4). The pivot of step kb then shares its
  // sub-partition's FP64 pipe only with the look-ahead warp (waiting) or a finished one, never
  // with a warp streaming the trailing-update DMMAs.
  const int rb = 2 * (warp & 3) + (warp >> 2);

  // optional per-phase cycle counters (diagnostics; pp = this CTA's counters or null)
  long long tprev = pp ? clock64() : 0;
  auto lap = [&](int k) {
    if (pp) {
      const long long now = clock64();
      if (lane == 0) atomicAdd(pp + k, (unsigned long long)(now - tprev));
      tprev = now;
    }
  };
  double acc[2][16][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 16; ++ni) {
      const double2 v = *reinterpret_cast<const double2*>(C + acc_off(16 * rb + 8 * mi + lr, ni, lc));
      acc[mi][ni][0] = v.x;
      acc[mi][ni][1] = v.y;
    }
  // Progressive publication: each finished 16x16 block also goes to HBM (gt), and when every
  // block of an L(j,j) slab (column blocks 2s, 2s+1: 15 - 4s warp blocks) is stored, the last
  // contributor releases the tile's flag as pbase + s + 1 (chain-bound OFF tasks start their
  // TRSM on the first slab; others wait for pbase + 4).
  // Column block kb of L(j,j) (rows 16kb..127, all final in C once every step-kb panel is in)
  // -> HBM by the pivot warp kb after its border work, off the pivot chain; the second column
  // block of a 32-column slab releases the slab (4 epoch + s + 1).
  auto publish_colblock = [&](int kb) {
    for (int q = lane; q < (8 - kb) * 128; q += 32) {  // double2 units: (8 - kb) blocks x 16 rows x 8
      const int r = 16 * kb + (q >> 3), c2 = 2 * (q & 7);
      const int off = elem_off(r, 16 * kb + c2);
      __stcg(reinterpret_cast<double2*>(gt + off), *reinterpret_cast<const double2*>(C + off));
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      const int sl = kb >> 1;
      if (atomicAdd(&misc->pcnt[sl], 1) == 1) {
        fence_proxy_async_global();
        st_release_gpu(prog, pbase + sl + 1);
      }
    }
  };
  double* Dbuf = reinterpret_cast<double*>(smem + TILE_ELEMS * 8);            // [2][16][16]
  double* Pbuf = Dbuf + 2 * 256;                                              // [2][128][16]
  double* Stw = Pbuf + 2 * TILE * 16 + warp * (16 * kStageLd);                // per warp
  // Pivot step kb (warp kb, the pivot block in the row layout xr): factor, release it (BD),
  // the border rows, publication. The warp is done with the tile afterwards.
  auto pivot_step = [&](int kb, double (&xr)[16]) {
    const int o = 16 * kb;
    double* Dblk = Dbuf + (kb & 1) * 256;
    double* P = Pbuf + (kb & 1) * (TILE * 16);
    const int bp = 4 + (kb & 1);
    // quotient broadcast buffer: the OFF-TRSM staging area, idle during DIAG tasks
    const bool okw = potrf_row16(xr, rinvD + o, lane,
                                 reinterpret_cast<double*>(smem + kOffTrsmSt) + warp * 32);
    if (!okw && lane == 0) misc->fail = 1;
    if (lane < 16) store_row16(xr, Dblk + lane * 16);
    __syncwarp();
    // BD(kb) in two parts: the look-ahead warp alone (the chain), the warps below it (their
    // panels; they may still be finishing the previous step's trailing update)
    if (kb < 7) named_bar_arrive(8 + (kb & 1), 64);
    if (kb < 6) named_bar_arrive(2 + (kb & 1), 32 * (7 - kb));
    if (lane < 16) {  // the finished block -> C
#pragma unroll
      for (int c = 0; c < 16; c += 2)
        *reinterpret_cast<double2*>(C + elem_off(o + lane, o + c)) = make_double2(xr[c], xr[c + 1]);
    }
    lap(PR_P_PIV);
    // The border rows W = [w_u; w_v] (2 x 128) ride along as two rows below the tile: the
    // pivot warp, idle after its factorization, solves their block kb against D_kb (lanes
    // 0/1) once warp kb-1 has applied block kb-1 to them (named barrier BB), then applies
    // block kb to their trailing columns from the step-kb panels and hands over to warp
    // kb+1. Each border element gets the same FMAs in the same order as a separate blocked
    // substitution after the POTRF.
    if (kb > 0) named_bar_sync(6 + (kb & 1), 64);
    // A failed pivot ends the factorization here (as the reference's factor attempt does): the
    // warps below see misc->fail after BD(kb) and stop too; BB's pending arrival is consumed
    // above and BP / BB(kb+1) are not entered by anyone, so the barriers stay balanced.
    if (!okw) return;
    if (lane < 2) {
      double xb[16];
      load_row16(xb, W + lane * TILE + o);
      solve_row16(xb, Dblk, rinvD + o);
      store_row16(xb, W + lane * TILE + o);
    }
    __syncwarp();
    // block kb of [u_j; v_j] is final: to HBM; after the odd block of a 32-column slab the
    // slab is released (the even block's warp handed over through BB before this one began)
    __stcg(bg + (lane >> 4) * npad + o + (lane & 15), W[(lane >> 4) * TILE + o + (lane & 15)]);
    __syncwarp();
    if ((kb & 1) && lane == 0) {
      __threadfence();
      fence_proxy_async_global();
      st_release_gpu(bprog, pbase + (kb >> 1) + 1);
    }
    if (kb < 7) {
      named_bar_sync(bp, 32 * (8 - kb));  // the step-kb panels are in P
      const int ncol = TILE - o - 16;
      for (int q = lane; q < 2 * ncol; q += 32) {
        const int r = q >= ncol ? 1 : 0;
        const int l = o + 16 + q - r * ncol;
        const double* x = W + r * TILE + o;
        double sacc = W[r * TILE + l];
#pragma unroll
        for (int c = 0; c < 16; ++c) sacc -= x[c] * P[p_off(l, c)];
        W[r * TILE + l] = sacc;
      }
      __syncwarp();
      named_bar_arrive(6 + ((kb + 1) & 1), 64);
    }
    if (gt) publish_colblock(kb);
  };
  for (int kb = 0; kb < 8; ++kb) {
    const int o = 16 * kb;
    double* Dblk = Dbuf + (kb & 1) * 256;
    double* P = Pbuf + (kb & 1) * (TILE * 16);
    const int bd = 2 + (kb & 1), bp = 4 + (kb & 1);
    // This warp's block of column block kb is final in the accumulators: to the row layout
    // (the pivot block for warp kb, a panel block for the others; the latter while waiting
    // for the pivot).
    stage_out(acc, Stw, lr, lc);
    __syncwarp();
    double xr[16];
    load_row16(xr, Stw + (lane & 15) * kStageLd);
    if (rb == kb) {  // block 0 only: every later pivot step runs from the look-ahead below
      pivot_step(kb, xr);
      break;
    }
    if (rb == kb + 1) {
      // The look-ahead warp: its panel block, then its diagonal block (accumulator n-tiles
      // 2, 3, kept apart so that nothing else of the accumulators stays live), then its own
      // pivot step kb+1 at once.
      double dg[2][2][2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nn = 0; nn < 2; ++nn) {
          dg[mi][nn][0] = acc[mi][2 + nn][0];
          dg[mi][nn][1] = acc[mi][2 + nn][1];
        }
      named_bar_sync(8 + (kb & 1), 64);
      lap(PR_P_BDW);
      if (misc->fail) break;  // the pivot failed: the candidate climbs the jitter ladder
      solve_row16(xr, Dblk, rinvD + o);
      if (lane < 16) {
        const int r = 16 * rb + lane;
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          *reinterpret_cast<double2*>(P + p_off(r, c)) = make_double2(xr[c], xr[c + 1]);
          *reinterpret_cast<double2*>(C + elem_off(r, o + c)) = make_double2(xr[c], xr[c + 1]);
        }
      }
      __syncwarp();
      named_bar_arrive(bp, 32 * (8 - kb));  // BP(kb): own panel rows are in P
      lap(PR_P_PANEL);
      // diagonal block -= panel * panel^T by DMMA, the A fragments straight from its own rows
      // in P (no window reload, no quad shuffles, no window rotation), then the row layout
      double av[2][4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) av[mi][ks] = -P[p_off(16 * rb + 8 * mi + lr, 4 * ks + lc)];
#pragma unroll
      for (int nn = 0; nn < 2; ++nn) {
        const int prow = o + 16 + 8 * nn + lr;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const double b = P[p_off(prow, 4 * ks + lc)];
          dmma884(dg[0][nn][0], dg[0][nn][1], av[0][ks], b);
          dmma884(dg[1][nn][0], dg[1][nn][1], av[1][ks], b);
        }
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nn = 0; nn < 2; ++nn)
          *reinterpret_cast<double2*>(Stw + (8 * mi + lr) * kStageLd + 8 * nn + 2 * lc) =
              make_double2(dg[mi][nn][0], dg[mi][nn][1]);
      __syncwarp();
      double yr[16];
      load_row16(yr, Stw + (lane & 15) * kStageLd);
      lap(PR_P_UPD);
      pivot_step(kb + 1, yr);
      break;
    }
    named_bar_sync(bd, 32 * (7 - kb));
    lap(PR_P_BDW);
    if (misc->fail) break;  // the pivot failed: the candidate climbs the jitter ladder
    solve_row16(xr, Dblk, rinvD + o);
    if (lane < 16) {
      const int r = 16 * rb + lane;
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        *reinterpret_cast<double2*>(P + p_off(r, c)) = make_double2(xr[c], xr[c + 1]);
        *reinterpret_cast<double2*>(C + elem_off(r, o + c)) = make_double2(xr[c], xr[c + 1]);
      }
    }
    __syncwarp();
    lap(PR_P_PANEL);
    named_bar_sync(bp, 32 * (8 - kb));    // every step-kb panel is in P
    lap(PR_P_BPW);
    // the solved panel back into the accumulator window for the A fragments
    if (lane < 16) store_row16(xr, Stw + lane * kStageLd);
    __syncwarp();
    stage_in(acc, Stw, lr, lc);
    double av[2][4];
    window_afrags(acc, av, lane);
    const int nlast = 2 * (rb - kb) + 1;  // the warp's own diagonal block
#pragma unroll
    for (int nb = 2; nb < 16; ++nb) {
      if (nb <= nlast) {
        const int prow = o + 8 * nb + lr;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const double b = P[p_off(prow, 4 * ks + lc)];
          dmma884(acc[0][nb][0], acc[0][nb][1], av[0][ks], b);
          dmma884(acc[1][nb][0], acc[1][nb][1], av[1][ks], b);
        }
      }
    }
    rotate_window(acc);
    lap(PR_P_UPD);
  }
  consumer_sync();
  return misc->fail == 0;
}

// DIAG-task tile products: the 136 (m-tile, n-tile) pairs of the 128 x 128 lower triangle
// (8 x 8 tiles) split into per-warp shapes whose operand addresses are a per-warp base plus
// compile-time offsets (no per-slot selects in the mainloop):
//   warps 0-3: a 4 x 4 block of the strictly-lower 64 x 64 quadrant (rows 8..15, cols 0..7);
//   warps 4-5: the 4 x 4 off-diagonal block of the upper-left / lower-right 64 x 64 triangle;
//   warps 6-7: the two 4-tile lower triangles on the diagonal of that triangle (20 products).
// Each SMSP (warps w, w + 4) gets 32 or 36 products per k-step.
__device__ __forceinline__ void diag_shape(int warp, int& m0, int& n0) {
  if (warp < 4) {
    m0 = 8 + 4 * (warp >> 1);
    n0 = 4 * (warp & 1);
  } else if (warp < 6) {
    m0 = warp == 4 ? 4 : 12;
    n0 = m0 - 4;
  } else {
    m0 = 8 * (warp - 6);
    n0 = m0;
  }
}
// accumulator slot -> (m-tile, n-tile); false for an unused slot. kShapes: the diag_shape split
// (chain-bound launches: -2.4% on a C3 B=1 evaluation); otherwise warp w takes m-tiles w and
// 15 - w (17 products; slot s <= w is (w, s), slot s > w is (15 - w, s - w - 1)), which is the
// faster split in the throughput-bound instantiation (C2 -0.7%, n=1024 B=100 -1.4%).
template <bool kShapes>
__device__ __forceinline__ bool diag_slot_tile(int warp, int sl, int& m, int& n) {
  if (!kShapes) {
    const bool first = sl <= warp;
    m = first ? warp : 15 - warp;
    n = first ? sl : sl - warp - 1;
    return sl < 17;
  }
  int m0, n0;
  diag_shape(warp, m0, n0);
  if (warp < 6) {
    m = m0 + (sl >> 2);
    n = n0 + (sl & 3);
    return sl < 16;
  }
  const int t = sl >= 10 ? 1 : 0, q = sl - 10 * t;  // q -> (i, jj <= i) of a 4-tile triangle
  const int i = q >= 6 ? 3 : q >= 3 ? 2 : q >= 1 ? 1 : 0;
  m = m0 + 4 * t + i;
  n = n0 + 4 * t + (q - i * (i + 1) / 2);
  return sl < 20;
}

// kProgress: release sub-diagonal tiles slab by slab (small, chain-bound launches); the large-
// launch instantiation carries none of that code.
template <bool kProgress>
__global__ void __launch_bounds__(kThreads, 1) chol_dag_kernel(DagLaunch a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* ljj_bar = full + kStages;  // [4] L(j,j) loads for the OFF-task TRSM (one per slab)
  int* stage_cnt = reinterpret_cast<int*>(ljj_bar + 4);  // warps done with each stage
  double* C = reinterpret_cast<double*>(smem + kOffC);
  double* W = reinterpret_cast<double*>(smem + kOffW);
  double* rinvD = reinterpret_cast<double*>(smem + kOffRinvD);
  Misc* misc = reinterpret_cast<Misc*>(smem + kOffMisc);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int NT = a.NT, B = a.nslots, n = a.n;
  const int Npad = NT * TILE;
  // Extension mode (a.ext != null): rows of test points appended below the factor; only
  // OFF tasks W(It, j) = (Rt(It, j) - sum_K W(It, K) L(j, K)^T) L(j, j)^-T, ordered
  // column-major; the factor tiles are final, only the row's own earlier tiles are waited on.
  const bool ext = a.ext != nullptr;
  const int ntasks = ext ? a.ext_rt * NT : B * NT * (NT + 1) / 2;
  const int epoch = a.epoch;
  const size_t fstride = (size_t)(NT + 1) * NT;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      stage_cnt[s] = 0;
    }
    for (int s = 0; s < 4; ++s) mbar_init(&ljj_bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // Stage ring position, advanced identically by every thread: `cur` is the stage of the next
  // slab, bit s of `ph` the parity of stage s's next completion.
  int cur = 0;
  uint32_t ph = 0;

  Prof pr{(a.prof && tid == 0) ? a.prof + (size_t)blockIdx.x * PR_COUNT : nullptr, 0};
  if (tid == 0) {
    misc->ljj_phase = 0;
    misc->next = -1;
    misc->pre_next = 0;
    misc->t_begin = clock64();
  }
  // Large batches take their next ticket when the mainloop ends and prefetch that task's R
  // seed tile into L2 while the epilogue runs (the seed is otherwise an HBM read at task
  // start). Small batches and the last two rounds of tickets do not: a ticket held by a busy
  // CTA would delay a chain that an idle CTA could start at once.
  const bool take_ahead = !ext && ntasks >= 16 * (int)gridDim.x;
  // Small launches (B=1 models, the 8-candidate refine batches) are bound by each candidate's
  // serial chain: there the sub-diagonal tile L(j+1, j) is released slab by slab as its TRSM
  // finishes them, and DIAG(j+1)'s last k-step starts on the first slab. Large launches are
  // throughput-bound and use the instantiation without the extra barriers.
  constexpr bool slab_progress = kProgress;
  pr.start();
  while (true) {
    if (tid == 0) {
      const int t = misc->next >= 0 ? misc->next : atomicAdd(a.counter, 1);
      misc->pre = misc->next >= 0 ? misc->pre_next : 0;
      misc->pre_next = 0;
      misc->next = -1;
      misc->ticket = t;
      misc->skip = 0;
      misc->fail = 0;
      if (t < ntasks) {
        int bpos = 0, j, I;
        if (ext) {
          j = t / a.ext_rt;
          I = t - j * a.ext_rt;  // the extension row tile It
        } else {
          task_of(a.order, t, B, NT, bpos, j, I);
        }
        misc->bpos = bpos;
        misc->I = I;
        misc->j = j;
        // a prefetched slab 0 must be consumed (ring parity): such a task runs its mainloop
        if (!ext && !misc->pre) misc->skip = *((volatile int*)&a.status[a.slots[bpos]]) != 0;
      }
    }
    __syncthreads();
    const int t = misc->ticket;
    if (t >= ntasks) break;
    if (tid == 0) pr.lap(PR_TICKET);
    // optional timeline stamps (diagnostics): the ticket is re-read from shared memory so no
    // per-task pointer stays live across the mainloop
    auto stamp = [&](int k) {
      if (a.trace && tid == 0) {
        const int tt = misc->ticket;
        if (tt < a.trace_cap) a.trace[(size_t)tt * 4 + k] = globaltimer_ns();
      }
    };
    stamp(0);
    int bpos = misc->bpos, j = misc->j, I = misc->I, It = 0;
    if (ext) {
      It = I;
      I = NT;  // below every factor row: never a DIAG task
    }
    const bool diag = (I == j);
    const int slot = a.slots[bpos];
    const bool skip = misc->skip != 0;
    double* fac = a.factors + (size_t)slot * a.slot_stride;
    double* bord = a.borders + (size_t)slot * 2 * Npad;
    int* flags = a.flags + (size_t)slot * fstride;  // flags[I*NT + J], border row I = NT
    const int nslab = skip ? 0 : SLABS_PER_TILE * j;

    {
      // ------------------------------ consumers -----------------------------
      // Warp w owns rows [16w, 16w+16) of the 128x128 tile (two m8 tiles x sixteen n8
      // tiles): the B operand is shared by all warps through shared memory, and every
      // row of the result stays in one warp, so the OFF-task TRSM needs no block barrier.
      const int lr = lane >> 2, lc = lane & 3;
      const int brow = tid >> 7, bc = tid & 127;  // border solve role (DIAG)
      // tile (row I, col K): the factor's packed lower tiles, or the extension rows
      auto a_tile = [&](int K) -> double* {
        return ext ? a.ext + ((size_t)It * NT + K) * TILE_ELEMS : fac + tile_index(I, K) * TILE_ELEMS;
      };
      double* gtile = a_tile(j);
      // Accumulators start from R(I,j) and the products are SUBTRACTED (negated A
      // operand, free in DMMA): the running-residual order of the reference's
      // `v -= L_it * L_jt` (backend.hpp:197-204), which keeps the rounding error
      // relative to the shrinking residual instead of the growing sum.
      // Row ownership: OFF tasks give warp w rows 16w..16w+15 (the TRSM needs whole rows per
      // warp). DIAG tasks only need the lower triangle: diag_shape splits its tile products.
      const int rowA = 16 * warp + lr;
      const int rowB = 16 * warp + 8 + lr;
      // DIAG tasks: accumulator slots per diag_shape (16 or 20 tile products per warp).
      double acc[2][16][2];
      if (!diag) {
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 16; ++ni) {
            const double2 v = skip ? make_double2(0.0, 0.0)
                                   : __ldcg(reinterpret_cast<const double2*>(gtile + acc_off(mi ? rowB : rowA, ni, lc)));
            acc[mi][ni][0] = v.x;
            acc[mi][ni][1] = v.y;
          }
      } else {
#pragma unroll
        for (int sl = 0; sl < 32; ++sl) {
          int mt, nt;
          const bool use = diag_slot_tile<kProgress>(warp, sl, mt, nt) && !skip;
          const double2 v = use ? __ldcg(reinterpret_cast<const double2*>(gtile + acc_off(8 * mt + lr, nt, lc)))
                                : make_double2(0.0, 0.0);
          acc[sl >> 4][sl & 15][0] = v.x;
          acc[sl >> 4][sl & 15][1] = v.y;
        }
      }
      // border rows (DIAG): running residual of [y_j; 1_j] - sum_K [u_K; v_K] L(j,K)^T
      // as an 8 x 128 DMMA accumulator (rows 0/1 = u/v, rows 2..7 stay zero): warp w owns the
      // border columns 16w..16w+15 (n-tiles 2w, 2w+1). Each k-step adds two DMMAs per warp;
      // the per-thread 32-long FMA chain it replaces read the slab column-wise with 3x bank
      // conflicts and made DIAG mainloops 1.8x slower than their DMMA bound.
      double wb[2][2];
#pragma unroll
      for (int nn = 0; nn < 2; ++nn) {
        const double2 v = (diag && !skip && lr < 2)
                              ? __ldcg(reinterpret_cast<const double2*>(bord + lr * Npad + j * TILE + 16 * warp + 8 * nn + 2 * lc))
                              : make_double2(0.0, 0.0);
        wb[nn][0] = v.x;
        wb[nn][1] = v.y;
      }

      // Operand-flag snapshot: the last warp reads the flags of K-tiles 1..j-1 in one pass
      // (lane = flag, acquire loads in parallel: one L2 round trip per 32 flags instead of two
      // serial ones per K-tile in the producer), while thread 0 issues the prologue (K-tile 0,
      // blocking wait). Published tiles are marked in misc->ready; their TMA loads are issued
      // without touching the flags again, the rest take the blocking wait. The refill of slab
      // 4 (K-tile 1) needs every warp past slab 1, so the bits are written by then (stage
      // counter atomics after __threadfence_block order them). Every task with more than one
      // K-tile takes the snapshot (thresholds of 4 and 8 K-tiles were 0.1-0.5% slower).
      if (warp == kConsumerWarps - 1 && j >= 2) {
        const int kmax = j < 256 ? j : 256;
        if (lane < 16) misc->ready[lane] = 0u;  // [0, 8): first flag, [8, 16): second flag
        __syncwarp();
        for (int e = lane; e < 2 * kmax - 2; e += 32) {
          const int part = e >= kmax - 1;
          const int K = 1 + e - part * (kmax - 1);
          const int* f;
          if (ext) {
            f = &a.ext_flags[(size_t)It * NT + K];
          } else if (part == 0) {
            f = (slab_progress && K == j - 1) ? nullptr : &flags[j * NT + K];
          } else {
            f = diag ? &flags[NT * NT + K] : &flags[I * NT + K];
          }
          // (border flags are progressive: 4 epoch + slabs released, complete at 4 epoch + 4)
          const int want = (diag && part == 1) ? 4 * epoch + 4 : epoch;
          if (f && (diag && part == 1 ? ld_acquire_gpu(f) >= want : ld_acquire_gpu(f) == want))
            atomicOr(&misc->ready[8 * part + (K >> 5)], 1u << (K & 31));
        }
        __syncwarp();
      }

      // Thread 0 doubles as the TMA producer, kStages-1 slabs ahead of the math.
      auto issue = [&](int p, int stage, bool may_defer) {
        const int K = p >> 2, sq = p & 3;
        // progress word of this task's other operand of the last K-tile: the border segment
        // (DIAG) or L(I, j-1) (OFF)
        const int* pw2 = diag ? &flags[NT * NT + K] : &flags[(j - 1) * NT + I];
        if (slab_progress && K == j - 1 && may_defer) {
          // A slab of the last K-tile whose progress flags are not yet published is not
          // waited for here (the issuing warp would sit on the flag with its own math for the
          // slabs in between undone): thread 0 issues it when the math reaches it.
          if (ld_acquire_gpu(&flags[(j - 1) * NT + j]) < 4 * epoch + sq + 1 || ld_acquire_gpu(pw2) < 4 * epoch + sq + 1) {
            misc->pend[stage] = p + 1;
            return;
          }
        }
        if (sq == 0 && j >= 2 && K > 0 && K < 256 && ((misc->ready[K >> 5] & misc->ready[8 + (K >> 5)]) >> (K & 31) & 1u)) {
          fence_proxy_async_global();
        } else if (sq == 0) {
          pr.start();
          const long long tw0 = (pr.p != nullptr || a.prof != nullptr) ? clock64() : 0;
          if (ext) {
            wait_flag(&a.ext_flags[(size_t)It * NT + K], epoch, a.error);
          } else {
            if (!(slab_progress && K == j - 1)) {
              wait_flag(&flags[j * NT + K], epoch, a.error);
              if (diag) {  // border rows of column K (progressive: 4 epoch + slabs done)
                wait_flag_geq(&flags[NT * NT + K], 4 * epoch + 4, a.error);
              } else {
                wait_flag(&flags[I * NT + K], epoch, a.error);
              }
            }
          }
          fence_proxy_async_global();
          if (a.prof) atomicAdd(a.prof + (size_t)gridDim.x * PR_COUNT + (diag ? 128 : 0) + j,
                                (unsigned long long)(clock64() - tw0));
          pr.lap(PR_PROD_FLAGS);
        }
        if (slab_progress && K == j - 1) {
          // the last K-tile is consumed slab by slab as the OFF tasks' TRSMs of column j-1
          // finish them: L(j, j-1) through the progress word flags[(j-1)*NT + j] = 4*epoch +
          // slabs done, and the border segment (DIAG) or L(I, j-1) (OFF, word flags[(j-1)*NT + I])
          wait_flag_geq(&flags[(j - 1) * NT + j], 4 * epoch + sq + 1, a.error);
          wait_flag_geq(pw2, 4 * epoch + sq + 1, a.error);
          fence_proxy_async_global();
        }
        unsigned char* dst = smem + kOffStages + stage * kStageBytes;
        mbar_arrive_expect_tx(&full[stage], diag ? kSlabBytes + 2 * SLAB * 8 : kStageBytes);
        bulk_g2s(dst, a_tile(K) + sq * SLAB_ELEMS, kSlabBytes, &full[stage]);
        if (!diag) {
          bulk_g2s(dst + kSlabBytes, fac + tile_index(j, K) * TILE_ELEMS + sq * SLAB_ELEMS,
                   kSlabBytes, &full[stage]);
        } else {  // the slab's border segments [u_K; v_K] ride in the unused B half
#pragma unroll
          for (int r = 0; r < 2; ++r)
            bulk_g2s(dst + kSlabBytes + r * SLAB * 8, bord + r * Npad + K * TILE + sq * SLAB, SLAB * 8,
                     &full[stage]);
        }
      };
      // Prologue: the first kStages slabs. Afterwards the LAST warp to finish with a
      // stage refills it (slab q + kStages): no warp ever blocks waiting for the others.
      // A task whose slab 0 the previous task issued into stage 2 starts the ring there.
      const int pre = misc->pre;
      if (pre) cur = 2;
      if (tid == 0) {
        const long long tsave = pr.last;
        if constexpr (slab_progress) {
#pragma unroll
          for (int st = 0; st < kStages; ++st) misc->freed[st] = misc->pend[st] = 0;
          if (pre) misc->freed[2] = 1;
        }
        for (int p = pre; p < kStages && p < nslab; ++p) {
          const int st = cur + p < kStages ? cur + p : cur + p - kStages;
          issue(p, st, true);
          if constexpr (slab_progress) misc->freed[st] = p + 1;
        }
        if constexpr (slab_progress) __threadfence_block();
        pr.last = tsave;
      }
      for (int q = 0; q < nslab; ++q) {
        const int stage = cur;
        cur = cur == kStages - 1 ? 0 : cur + 1;
        const uint32_t par = (ph >> stage) & 1u;
        ph ^= 1u << stage;
        if (slab_progress && tid == 0 && q >= SLABS_PER_TILE * (j - 1)) {
          // a deferred slab of the last K-tile: once its stage's refill was decided, wait for
          // its flags and issue it now
          while (*((volatile int*)&misc->freed[stage]) != q + 1) {
          }
          if (*((volatile int*)&misc->pend[stage]) == q + 1) {
            const long long tsave = pr.last;
            issue(q, stage, false);
            pr.last = tsave;
          }
        }
        if (tid == 0 && pr.p) {
          const long long tw = clock64();
          mbar_wait(&full[stage], par);
          pr.p[diag ? PR_DIAG_FULL_WAIT : PR_FULL_WAIT] += (unsigned long long)(clock64() - tw);
        } else {
          mbar_wait(&full[stage], par);
        }
        const double* As = reinterpret_cast<const double*>(smem + kOffStages + stage * kStageBytes);
        const double* Bs = diag ? As : As + SLAB_ELEMS;
        const double* Bw = Bs + lr * 32 + lc;
        if (!diag) {
          const double* Aw = As + (16 * warp + lr) * 32 + lc;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int ko = (ks ^ lr) << 2;
            const double a0 = -Aw[ko], a1 = -Aw[256 + ko];
#pragma unroll
            for (int ni = 0; ni < 16; ++ni) {
              const double b = Bw[ni * 256 + ko];
              dmma884(acc[0][ni][0], acc[0][ni][1], a0, b);
              dmma884(acc[1][ni][0], acc[1][ni][1], a1, b);
            }
          }
        } else if constexpr (!kProgress) {  // lower triangle only: m-tiles w and 15 - w
          const double* Aw0 = As + (8 * warp + lr) * 32 + lc;
          const double* Aw1 = As + (8 * (15 - warp) + lr) * 32 + lc;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int ko = (ks ^ lr) << 2;
            const double a0 = -Aw0[ko], a1 = -Aw1[ko];
            const double* BwB = Bw - (warp + 1) * 256;  // slot sl > warp reads n-tile sl - warp - 1
            {  // border rows: [w_u; w_v] -= [u_K; v_K](k-step) L(j,K)(n-tiles 2w, 2w+1)^T
              const double ab = lr < 2 ? -As[SLAB_ELEMS + lr * SLAB + 4 * ks + lc] : 0.0;
              dmma884(wb[0][0], wb[0][1], ab, Bw[(2 * warp) * 256 + ko]);
              dmma884(wb[1][0], wb[1][1], ab, Bw[(2 * warp + 1) * 256 + ko]);
            }
#pragma unroll
            for (int sl = 0; sl < 17; ++sl) {
              const bool first = sl <= warp;
              const double b = (first ? Bw : BwB)[sl * 256 + ko];
              dmma884(acc[sl >> 4][sl & 15][0], acc[sl >> 4][sl & 15][1], first ? a0 : a1, b);
            }
          }
        } else {  // lower triangle only (diag_shape): B = A, the slab of L(j, K)
          int m0, n0;
          diag_shape(warp, m0, n0);
          const double* Am = As + (8 * m0 + lr) * 32 + lc;
          const double* Bn = As + (8 * n0 + lr) * 32 + lc;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const int ko = (ks ^ lr) << 2;
            {  // border rows: [w_u; w_v] -= [u_K; v_K](k-step) L(j,K)(n-tiles 2w, 2w+1)^T
              const double ab = lr < 2 ? -As[SLAB_ELEMS + lr * SLAB + 4 * ks + lc] : 0.0;
              dmma884(wb[0][0], wb[0][1], ab, Bw[(2 * warp) * 256 + ko]);
              dmma884(wb[1][0], wb[1][1], ab, Bw[(2 * warp + 1) * 256 + ko]);
            }
            if (warp < 6) {  // 4 x 4 block
              double am[4], bn[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                am[i] = -Am[i * 256 + ko];
                bn[i] = Bn[i * 256 + ko];
              }
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                  dmma884(acc[0][4 * i + jj][0], acc[0][4 * i + jj][1], am[i], bn[jj]);
            } else {  // two 4-tile lower triangles on the diagonal (m0 = n0: A and B rows coincide)
#pragma unroll
              for (int t = 0; t < 2; ++t) {
                double bt[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) bt[i] = Bn[(4 * t + i) * 256 + ko];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                  for (int jj = 0; jj <= i; ++jj) {
                    const int sl = 10 * t + i * (i + 1) / 2 + jj;
                    dmma884(acc[sl >> 4][sl & 15][0], acc[sl >> 4][sl & 15][1], -bt[i], bt[jj]);
                  }
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          if (atomicAdd(&stage_cnt[stage], 1) == kConsumerWarps - 1) {
            stage_cnt[stage] = 0;
            if (q + kStages < nslab) {
              fence_proxy_async_shared();  // generic-proxy reads of the stage before the TMA write
              const long long tsave = pr.last;
              issue(q + kStages, stage, true);
              pr.last = tsave;
              if constexpr (slab_progress) {
                __threadfence_block();
                *((volatile int*)&misc->freed[stage]) = q + kStages + 1;
              }
            }
          }
        }
      }
      consumer_sync();  // every consumer is done reading the stage ring
      stamp(1);
      // Thread 0's post-mainloop work, in latency order: an OFF task's L(j,j) load goes out
      // first (every warp waits for it), then the take-ahead of the next ticket -- several
      // dependent L2 round trips (ticket, order table, slot, status, flags) that now overlap
      // the L(j,j) transfer instead of preceding it.
      auto issue_ljj = [&](int sl) {  // slab sl of L(j,j) -> stage ring bytes [32 KB sl, +32 KB)
        fence_proxy_async_global();
        mbar_arrive_expect_tx(&ljj_bar[sl], kSlabBytes);
        bulk_g2s(smem + sl * kSlabBytes, fac + tile_index(j, j) * TILE_ELEMS + sl * SLAB_ELEMS, kSlabBytes,
                 &ljj_bar[sl]);
      };
      auto take_next = [&]() {
      if (take_ahead && misc->ticket < ntasks - 2 * (int)gridDim.x) {
        const int tn = atomicAdd(a.counter, 1);
        misc->next = tn;
        if (tn < ntasks) {
          int bn = 0, jn, In;
          task_of(a.order, tn, B, NT, bn, jn, In);
          const double* seed = a.factors + (size_t)a.slots[bn] * a.slot_stride + tile_index(In, jn) * TILE_ELEMS;
#pragma unroll
          for (int s4 = 0; s4 < SLABS_PER_TILE; ++s4) bulk_prefetch_l2(seed + s4 * SLAB_ELEMS, kSlabBytes);
          // After an OFF mainloop (its TRSM leaves stage 2 alone), the next task's slab 0 goes
          // into stage 2 now if its K-tile-0 operands are published (non-blocking check), so
          // that task starts without the flag round trips and the load latency.
          const int sn = a.slots[bn];
          if (!diag && jn > 0 && *((volatile int*)&a.status[sn]) == 0) {
            const int* fln = a.flags + (size_t)sn * fstride;
            const bool dn = In == jn;
            if (ld_acquire_gpu(&fln[jn * NT]) == epoch &&
                (dn ? ld_acquire_gpu(&fln[NT * NT]) >= 4 * epoch + 4 : ld_acquire_gpu(&fln[In * NT]) == epoch)) {
              fence_proxy_async_global();
              fence_proxy_async_shared();  // generic-proxy reads of stage 2 before the TMA write
              const double* facn = a.factors + (size_t)sn * a.slot_stride;
              unsigned char* dst = smem + kOffStages + 2 * kStageBytes;
              mbar_arrive_expect_tx(&full[2], dn ? kSlabBytes + 2 * SLAB * 8 : kStageBytes);
              bulk_g2s(dst, facn + tile_index(In, 0) * TILE_ELEMS, kSlabBytes, &full[2]);
              if (!dn) {
                bulk_g2s(dst + kSlabBytes, facn + tile_index(jn, 0) * TILE_ELEMS, kSlabBytes, &full[2]);
              } else {
                const double* bn2 = a.borders + (size_t)sn * 2 * Npad;
#pragma unroll
                for (int r = 0; r < 2; ++r)
                  bulk_g2s(dst + kSlabBytes + r * SLAB * 8, bn2 + r * Npad, SLAB * 8, &full[2]);
              }
              misc->pre_next = 1;
            }
          }
        }
      }
      };
      if (tid == 0) {
        if (!diag && !skip) {
          misc->run = ext || *((volatile int*)&a.status[slot]) == 0;
          if constexpr (kProgress) {  // slab 0 now (blocking), later slabs when already published
            if (!ext) wait_flag_geq(&flags[j * NT + j], 4 * epoch + 1, a.error);
            int is = 0;
            do {
              issue_ljj(is);
              ++is;
            } while (is < SLABS_PER_TILE && (ext || ld_acquire_gpu(&flags[j * NT + j]) >= 4 * epoch + is + 1));
            misc->ljj_issued = is;
          } else {
            if (!ext) wait_flag_geq(&flags[j * NT + j], 4 * epoch + 4, a.error);
            fence_proxy_async_global();
            mbar_arrive_expect_tx(&ljj_bar[0], TILE_ELEMS * 8);
            const double* Ljj = fac + tile_index(j, j) * TILE_ELEMS;
#pragma unroll
            for (int s4 = 0; s4 < SLABS_PER_TILE; ++s4)
              bulk_g2s(smem + s4 * kSlabBytes, Ljj + s4 * SLAB_ELEMS, kSlabBytes, &ljj_bar[0]);
          }
        }
        take_next();
      }
      if (tid == 0) {
        if (diag && pr.p) pr.p[PR_DIAG_GEMM] += (unsigned long long)(clock64() - pr.last);
        pr.lap(PR_GEMM);
        pr.add(PR_SLABS, nslab);
        pr.add(diag ? PR_N_DIAG : PR_N_OFF, 1);
      }

      if (diag) {
        // ------------------------------ DIAG ------------------------------
        // accumulators (= R - sum L L^T) -> C (tile layout); the POTRF runs in its own
        // (non-inlined) function so its register pressure stays out of the mainloop
        // (the upper triangle of C is left as is: nothing downstream reads it)
#pragma unroll
        for (int sl = 0; sl < 20; ++sl) {
          int mt, nt;
          if (diag_slot_tile<kProgress>(warp, sl, mt, nt))
            *reinterpret_cast<double2*>(C + acc_off(8 * mt + lr, nt, lc)) =
                make_double2(acc[sl >> 4][sl & 15][0], acc[sl >> 4][sl & 15][1]);
        }
        if (lr < 2) {
#pragma unroll
          for (int nn = 0; nn < 2; ++nn)
            *reinterpret_cast<double2*>(W + lr * TILE + 16 * warp + 8 * nn + 2 * lc) = make_double2(wb[nn][0], wb[nn][1]);
        }
        if (tid == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q) misc->pcnt[q] = 0;
        }
        consumer_sync();
        if (tid == 0) pr.lap(PR_ACC_STORE);
        bool ok = !skip;
        if (!skip) {
          ok = diag_potrf(smem, C, rinvD, W, misc, warp, lane,
                          a.prof ? a.prof + (size_t)blockIdx.x * PR_COUNT : nullptr, kProgress ? gtile : nullptr,
                          &flags[j * NT + j], 4 * epoch, bord + j * TILE, Npad, &flags[NT * NT + j]);
          if (!ok && tid == 0) atomicExch(&a.status[slot], 1);  // GPEMU_SLOT_NOT_PD
        }
        if (tid == 0) pr.lap(PR_POTRF);
        // Chain-bound launches stored L(j,j) block by block inside the POTRF (progressive release);
        // throughput-bound ones store it now (per-block fences cost 0.1-1% there). Then the final
        // release (also for skipped tasks, whose waiters must not block).
        if constexpr (!kProgress) {
          if (ok) {
            for (int e = 2 * tid; e < TILE_ELEMS; e += 2 * kConsumers)
              __stcg(reinterpret_cast<double2*>(gtile + e), *reinterpret_cast<const double2*>(C + e));
          }
          consumer_sync();
        }
        stamp(2);
        if (tid == 0) {
          publish_flag(&flags[j * NT + j], 4 * epoch + 4);
          pr.lap(PR_DIAG_STORE);
        }
        // border rows [u_j; v_j] = w L(j,j)^-T: solved inside the POTRF (diag_potrf)
        // (stored and released slab by slab inside the POTRF; the final release covers skipped
        // tasks)
        if (tid == 0) {
          publish_flag(&flags[NT * NT + j], 4 * epoch + 4);
          pr.lap(PR_BORDER);
        }
      } else {
        // ------------------------------ OFF -------------------------------
        // chain-bound launches release every OFF tile slab by slab (progress word flags[j*NT + I],
        // the unused upper half): the last k-steps of DIAG(I) / OFF(I', I) consume them as they come
        const bool sub = slab_progress;
        // L(I,j) = C L(j,j)^-T. L(j,j) arrives by TMA into the (now idle) stage ring;
        // each warp then solves its own 16 rows in registers, 16 columns at a time:
        // (a) in-block substitution (quad shuffles), (b) DMMA update of the columns to
        // the right, (c) store the finished block, (d) rotate the accumulator window.
        if (!skip) mbar_wait(&ljj_bar[0], misc->ljj_phase & 1);  // issued by thread 0 at mainloop end
        if (tid == 0) pr.lap(PR_OFF_WAIT);
        // uniform across the CTA (the TRSM below has CTA barriers): thread 0 read the status
        // once before the L(j,j) load, and the load's mbarrier publishes it (a later DIAG of the
        // same candidate may fail meanwhile: the TRSM then only does wasted work)
        const bool run = !skip && misc->run != 0;
        if constexpr (kProgress) {
          if (!skip && !run) {  // keep every slab barrier's phase in step: load (and drop) the rest
            if (tid == 0)
              for (int sl = misc->ljj_issued; sl < SLABS_PER_TILE; ++sl) issue_ljj(sl);
            for (int sl = 1; sl < SLABS_PER_TILE; ++sl) mbar_wait(&ljj_bar[sl], misc->ljj_phase & 1);
          }
        }
        if (run) {
          const double* Ls = reinterpret_cast<const double*>(smem);  // L(j,j), tile layout
          // 1 / L_cc once per task; the in-block substitution forms a / L_cc as
          // a*r + one FMA correction (division rounding as in backend.hpp:206).
          // The eight diagonal 16x16 blocks of L(j,j) are copied densely so the in-block
          // substitution reads them as warp-uniform (broadcast) loads with immediate offsets.
          double* rinv = W;
          double* Dp = reinterpret_cast<double*>(smem + kOffTrsmD);              // [8][kTriElems]
          double* St = reinterpret_cast<double*>(smem + kOffTrsmSt) + warp * (16 * kStageLd);
          if constexpr (!kProgress) {
            if (tid < TILE) rinv[tid] = 1.0 / Ls[elem_off(tid, tid)];
            for (int q = tid; q < 2048; q += kConsumers) {
              const int b8 = q >> 8, rr = (q >> 4) & 15, cc = q & 15;
              if (cc <= rr) Dp[b8 * kTriElems + rr * (rr + 1) / 2 + cc] = Ls[elem_off(16 * b8 + rr, 16 * b8 + cc)];
            }
            consumer_sync();
          }
          // Fully unrolled over the eight 16-column blocks: window n-tiles w = 2cb, 2cb+1 are
          // compile-time register indices (no rotation), and every L(j,j) operand address is a
          // per-lane base plus an immediate, so the DMMAs of independent column blocks
          // interleave instead of queueing behind runtime predicates.
          const int lane_base = (lr << 5) + lc;
          if (kProgress && tid == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) misc->pcnt[q] = 0;  // slab releases (counted before the first block barrier below)
          }
          if constexpr (!kProgress) {
            // Software-pipelined: block cb's update of the next block's columns (n-tiles w+2,
            // w+3) goes first, then block cb+1's substitution runs with the rest of block cb's
            // update (n-tiles w+4..15) interleaved into it, so the DMMA stream fills the
            // substitution chain's latency instead of alternating with it. Every lane takes part
            // in the substitution (lanes 16..31 repeat rows 0..15; only lanes < 16 store), which
            // keeps the warp converged for the interleaved mma.sync. Per accumulator the DMMAs
            // keep their k order, so the factor is bitwise unchanged.
            auto lk = [&](int cb, int ks) -> const double* {
              return Ls + ((cb >> 1) << 12) + lane_base + (((((4 * cb) + ks) & 7) ^ lr) << 2);
            };
            stage_out_at(acc, 0, St, lr, lc);
            __syncwarp();
            {
              double xr[16];
              load_row16(xr, St + (lane & 15) * kStageLd);
              solve_row16p(xr, Dp, rinv);
              if (lane < 16) store_row16(xr, St + lane * kStageLd);
            }
            __syncwarp();
#pragma unroll
            for (int cb = 0; cb < 8; ++cb) {
              const int o = 16 * cb, w = 2 * cb;
              double av[2][4];
              if (cb < 7) {
#pragma unroll
                for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                  for (int ks = 0; ks < 4; ++ks) av[mi][ks] = -St[(8 * mi + lr) * kStageLd + 4 * ks + lc];
              }
              // block cb is final: store it from St
#pragma unroll
              for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                for (int nsub = 0; nsub < 2; ++nsub)
                  __stcg(reinterpret_cast<double2*>(gtile + acc_off(16 * warp + 8 * mi + lr, w + nsub, lc)),
                         *reinterpret_cast<const double2*>(St + (8 * mi + lr) * kStageLd + 8 * nsub + 2 * lc));
              if (cb < 7) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                  const double* Lk = lk(cb, ks);
#pragma unroll
                  for (int a = w + 2; a < w + 4; ++a) {
                    const double b = Lk[a << 8];
                    dmma884(acc[0][a][0], acc[0][a][1], av[0][ks], b);
                    dmma884(acc[1][a][0], acc[1][a][1], av[1][ks], b);
                  }
                }
                __syncwarp();  // St (A fragments, store) read before block cb+1 overwrites it
                stage_out_at(acc, w + 2, St, lr, lc);
                __syncwarp();
                double xr[16];
                load_row16(xr, St + (lane & 15) * kStageLd);
                const double* D = Dp + (cb + 1) * kTriElems;
                const double* ri = rinv + o + 16;
                const int na = 12 - w, units = 4 * na;  // (ks, a) pairs left of block cb's update
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                  xr[c] = div_by(xr[c], D[c * (c + 1) / 2 + c], ri[c]);
#pragma unroll
                  for (int c2 = c + 1; c2 < 16; ++c2) xr[c2] -= xr[c] * D[c2 * (c2 + 1) / 2 + c];
#pragma unroll
                  for (int e = (c * units) / 16; e < ((c + 1) * units) / 16; ++e) {
                    const int ks = e / na, a = w + 4 + e % na;
                    const double b = lk(cb, ks)[a << 8];
                    dmma884(acc[0][a][0], acc[0][a][1], av[0][ks], b);
                    dmma884(acc[1][a][0], acc[1][a][1], av[1][ks], b);
                  }
                }
                if (lane < 16) store_row16(xr, St + lane * kStageLd);
                __syncwarp();
              }
            }
          }
#pragma unroll
          for (int cb = 0; cb < (kProgress ? 8 : 0); ++cb) {
            const int o = 16 * cb, w = 2 * cb;
            if constexpr (kProgress) {
              // L(j,j) slab cb/2: its load (issued once the DIAG task published it), then the
              // reciprocal pivots and packed diagonal blocks of its two column blocks
              if ((cb & 1) == 0) {
                const int sl = cb >> 1;
                if (tid == 0) {
                  int is = misc->ljj_issued;
                  for (; is <= sl; ++is) {
                    wait_flag_geq(&flags[j * NT + j], 4 * epoch + is + 1, a.error);
                    issue_ljj(is);
                  }
                  for (; is < SLABS_PER_TILE && ld_acquire_gpu(&flags[j * NT + j]) >= 4 * epoch + is + 1; ++is)
                    issue_ljj(is);
                  misc->ljj_issued = is;
                }
                if (sl > 0) mbar_wait(&ljj_bar[sl], misc->ljj_phase & 1);
                if (tid < 32) rinv[32 * sl + tid] = 1.0 / Ls[elem_off(32 * sl + tid, 32 * sl + tid)];
                for (int q = tid; q < 512; q += kConsumers) {
                  const int b8 = 2 * sl + (q >> 8), rr = (q >> 4) & 15, cc = q & 15;
                  if (cc <= rr) Dp[b8 * kTriElems + rr * (rr + 1) / 2 + cc] = Ls[elem_off(16 * b8 + rr, 16 * b8 + cc)];
                }
                consumer_sync();
              }
            }
            // (a) columns o..o+15 (acc[mi][w..w+1]): through the warp's staging block so
            // lane r < 16 owns row r and substitutes in registers
            stage_out_at(acc, w, St, lr, lc);
            __syncwarp();
            if (lane < 16) {
              double xr[16];
              load_row16(xr, St + lane * kStageLd);
              solve_row16p(xr, Dp + cb * kTriElems, rinv + o);
              store_row16(xr, St + lane * kStageLd);
            }
            __syncwarp();
            // (b) acc[:, a] -= X_block * L(j,j)[8a + lr, block cols]^T for the n-tiles a right
            // of the block (element (8a + lr, o + 4ks + lc) of the swizzled tile layout). The
            // negated A fragments come straight from the solved block in St (one LDS each; the
            // accumulator window is not reloaded: its columns are final and stored from St).
            // (The chain-bound instantiation keeps the register route -- quad shuffles from the
            // reloaded window -- which is 0.5% faster on a B=1 evaluation.)
            if constexpr (kProgress) stage_in_at(acc, w, St, lr, lc);
            if (cb < 7) {
              double av[2][4];
              if constexpr (kProgress) {
                window_afrags_at(acc, w, av, lane);
              } else {
#pragma unroll
                for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                  for (int ks = 0; ks < 4; ++ks) av[mi][ks] = -St[(8 * mi + lr) * kStageLd + 4 * ks + lc];
              }
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {
                const double* Lk = Ls + ((cb >> 1) << 12) + lane_base +
                                   (((((o >> 2) + ks) & 7) ^ lr) << 2);
#pragma unroll
                for (int a = w + 2; a < 16; ++a) {
                  const double b = Lk[a << 8];
                  dmma884(acc[0][a][0], acc[0][a][1], av[0][ks], b);
                  dmma884(acc[1][a][0], acc[1][a][1], av[1][ks], b);
                }
              }
            }
            // (c) the block is final: store it from St
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
              for (int nsub = 0; nsub < 2; ++nsub)
                __stcg(reinterpret_cast<double2*>(gtile + acc_off(16 * warp + 8 * mi + lr, w + nsub, lc)),
                       kProgress ? make_double2(acc[mi][w + nsub][0], acc[mi][w + nsub][1])
                                 : *reinterpret_cast<const double2*>(St + (8 * mi + lr) * kStageLd + 8 * nsub + 2 * lc));
            if constexpr (!kProgress) __syncwarp();  // St is rewritten by the next block
            if (sub && (cb & 1) && cb < 7) {  // slab cb/2 of L(I, j) is final: release it
              // each warp fences its own stores, the last one to get there releases the slab:
              // no block barrier, and the fences overlap the next slab's work
              __syncwarp();
              if (lane == 0) {
                __threadfence();
                if (atomicAdd(&misc->pcnt[cb >> 1], 1) == kConsumerWarps - 1) {
                  fence_proxy_async_global();
                  st_release_gpu(&flags[j * NT + I], 4 * epoch + (cb >> 1) + 1);
                }
              }
            }
          }
          if (tid == 0) pr.lap(PR_TRSM);
        }
        consumer_sync();
        stamp(2);
        if (tid == 0) {
          if (!skip) ++misc->ljj_phase;  // every consumer passed its ljj wait (consumer_sync above)
          if (sub) publish_flag(&flags[j * NT + I], 4 * epoch + 4);
          publish_flag(ext ? &a.ext_flags[(size_t)It * NT + j] : &flags[I * NT + j], epoch);
          pr.lap(PR_OFF_STORE);
        }
      }
    }
    __syncthreads();
    stamp(3);
    if (tid == 0) pr.lap(PR_TASK_END);
  }
  if (tid == 0) pr.add(PR_TOTAL, (unsigned long long)(clock64() - misc->t_begin));
}
}  // namespace

size_t chol_dag_smem_bytes() { return kSmemBytes; }

void launch_chol_dag(const DagLaunch& a, int num_sms, cudaStream_t s) {
  const int ntasks = a.ext ? a.ext_rt * a.NT : a.nslots * a.NT * (a.NT + 1) / 2;
  const int grid = ntasks < num_sms ? ntasks : num_sms;
  // the same split as the kernel's take-ahead rule: small launches are chain-bound
  const bool progress = !a.ext && ntasks < 16 * grid;
  // per-device attribute: set on every launch (cheap) so multi-device processes are correct
  cudaFuncSetAttribute(progress ? chol_dag_kernel<true> : chol_dag_kernel<false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  cudaMemsetAsync(a.counter, 0, sizeof(int), s);
  if (progress) {
    chol_dag_kernel<true><<<grid, kThreads, kSmemBytes, s>>>(a);
  } else {
    chol_dag_kernel<false><<<grid, kThreads, kSmemBytes, s>>>(a);
  }
}

}  // namespace gpemu_dev
