// kernels_chol_f32.cu -- single-precision tile-DAG Cholesky (Precision::kSingle) on sm_100a.
//
// Reference: the float instantiation of Backend<float>::factorize_into / try_cholesky /
// solve_lower_into (backend.hpp:102-153, 226-311) as ProfileEvaluator<float> runs it
// (likelihood.hpp:108-141; precision = single, core.hpp:86-96, bench.hpp:489-490).
//
// FP32 has no tensor-core path with FP32 accuracy short of split-TF32, so this engine runs on
// the FP32 FFMA pipes (~74 TF/s on B200, about twice the FP64 DMMA rate). It keeps the FP64
// engine's scheduling (persistent CTAs, ticket counter, left-looking tile DAG with one-column
// lookahead, epoch flags, bordered [y; 1] rows, running-residual accumulation) and changes
// the data path:
//   * float tiles, 128 x 128, COLUMN-major (element (r, c) at c * 128 + r, 64 KB); a k-slab
//     is 32 consecutive columns (16 KB), one cp.async.bulk copy, in a 3-stage mbarrier ring;
//   * warp w owns rows 16w..16w+15; lane (rg = lane / 16, cg = lane % 16) holds the 8 x 8
//     register block rows 16w + 8rg.., cols 8cg..: per k it reads 8 A and 8 B floats (four
//     LDS.128, A broadcast across the half-warp) for 64 FFMAs;
//   * <= 128 registers so two CTAs share an SM;
//   * DIAG: blocked (16-column) POTRF of the tile in shared memory (pivot test !(s > 0),
//     backend.hpp:238; IEEE sqrt and division), border rows solved by two warps;
//   * OFF: X = C L(j,j)^-T in 8-column blocks: the two lanes holding a block substitute their
//     rows (IEEE division), publish the block through a per-warp buffer, lanes to the right
//     apply it with FFMAs.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "layout.cuh"
#include "ptx.cuh"

namespace gpemu_dev {
namespace {

constexpr int kThreadsF = 256;
constexpr int kWarpsF = 8;
constexpr int kStagesF = 3;
constexpr int kSlabF = TILE * SLAB;                 // 4096 floats
constexpr int kSlabBytesF = kSlabF * 4;             // 16 KB
constexpr int kStageBytesF = 2 * kSlabBytesF;       // A + B slab
constexpr int kTileBytesF = TILE_ELEMS * 4;         // 64 KB
constexpr int kOffRingF = 0;                        // [0, 96K): ring; C / L(j,j) alias [0, 64K)
constexpr int kOffXwF = kStagesF * kStageBytesF;    // 96K: per-warp 16 x 8 X block
constexpr int kOffWF = kOffXwF + kWarpsF * 16 * 8 * 4;  // border w: 2 x 128 floats
constexpr int kOffBarF = kOffWF + 2 * TILE * 4;     // mbarriers
constexpr int kOffMiscF = kOffBarF + 128;
constexpr int kSmemBytesF = kOffMiscF + 64;
constexpr long long kSpinLimitF = 20000000000LL;    // ~10 s: declare deadlock

struct MiscF {
  int ticket, skip, fail, bpos, I, j;
  unsigned ljj_phase;
  int pad;
};

__device__ __forceinline__ void csync() { named_bar_sync(1, kThreadsF); }

__device__ __forceinline__ void wait_flag_f(const int* flag, int epoch, int* error) {
  if (ld_acquire_gpu(flag) == epoch) return;
  const long long t0 = clock64();
  while (ld_acquire_gpu(flag) != epoch) {
    __nanosleep(64);
    if (clock64() - t0 > kSpinLimitF) {
      atomicExch(error, 1);
      return;
    }
  }
}

__device__ __forceinline__ void publish_f(int* flag, int epoch) {
  __threadfence();
  fence_proxy_async_global();
  st_release_gpu(flag, epoch);
}

// Ticket -> (bpos, j, I): the FP64 engine's one-column-lookahead topological order.
__device__ __forceinline__ void decode_task_f(int t, int B, int NT, int& bpos, int& j, int& I) {
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
  const int per = NT - jj;
  bpos = t / per;
  const int pos = t - bpos * per;
  if (pos == 0) {
    j = jj;
    I = jj + 1;
  } else if (pos == 1) {
    j = jj + 1;
    I = jj + 1;
  } else {
    j = jj;
    I = jj + pos;
  }
}

__device__ __forceinline__ void ld8(float (&v)[8], const float* p) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// a / d given r ~ 1/d (IEEE reciprocal): one FMA residual correction gives the rounding of
// the true quotient (the reference divides, backend.hpp:206 / :138).
__device__ __forceinline__ float div_by_f(float a, float d, float r) {
  const float q0 = a * r;
  return fmaf(fmaf(-q0, d, a), r, q0);
}

// DIAG POTRF of the column-major tile C in shared memory (lower triangle), blocked in
// 16-column steps with three CTA barriers per step: (i) warp 0 factors the 16 x 16 diagonal
// block in registers (lane r holds row r, columns broadcast by shuffles); (ii) one thread per
// row solves the panel below against it; (iii) the trailing lower triangle is updated with
// the 16-wide panel, each thread owning 4 rows (strided, conflict-free) of one column at a
// time (the column's panel values are read once for the 4 rows). Pivot test !(s > 0) as backend.hpp:238. Returns
// false (uniform) on a failed pivot.
__device__ __noinline__ bool potrf_tile_f32(float* C, int* fail) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int kb = 0; kb < 8; ++kb) {
    const int o = 16 * kb;
    if (warp == 0) {
      float xr[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) xr[c] = lane < 16 ? C[(o + c) * TILE + o + lane] : 1.0f;
      bool ok = true;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        float s = __shfl_sync(0xffffffffu, xr[c], c);
        ok = ok && s > 0.0f;
        if (!ok) s = 1.0f;
        const float d = __fsqrt_rn(s);
        if (lane == c) xr[c] = d;
        if (lane > c) xr[c] = __fdiv_rn(xr[c], d);
#pragma unroll
        for (int c2 = c + 1; c2 < 16; ++c2) {
          const float l = __shfl_sync(0xffffffffu, xr[c], c2);  // L[c2][c]
          if (lane >= c2) xr[c2] = fmaf(-xr[c], l, xr[c2]);
        }
      }
      if (lane < 16) {
#pragma unroll
        for (int c = 0; c < 16; ++c) C[(o + c) * TILE + o + lane] = xr[c];
      }
      if (!ok && lane == 0) *fail = 1;
    }
    csync();
    if (*fail) return false;
    const int r0 = o + 16, m = TILE - r0;  // rows below the diagonal block
    if (tid < m) {  // (ii) panel: row r, X = A L_bb^-T
      const int r = r0 + tid;
      float xr[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) xr[c] = C[(o + c) * TILE + r];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        xr[c] = __fdiv_rn(xr[c], C[(o + c) * TILE + o + c]);
#pragma unroll
        for (int c2 = c + 1; c2 < 16; ++c2) xr[c2] = fmaf(-xr[c], C[(o + c) * TILE + o + c2], xr[c2]);
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) C[(o + c) * TILE + r] = xr[c];
    }
    csync();
    if (m > 0) {  // (iii) trailing: C[r][c] -= sum_k L[r][o+k] L[c][o+k], r0 <= c <= r
      const int groups = (m + 3) / 4;  // a thread owns rows r0 + g + q * groups, q < 4
      for (int w = tid; w < groups * m; w += kThreadsF) {
        const int g = w % groups, cc = w / groups;
        const int c = r0 + cc;
        if (r0 + g + 3 * groups < c) continue;  // all four rows are above the diagonal
        float lc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) lc[k] = C[(o + k) * TILE + c];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = r0 + g + q * groups;
          if (r < c || r >= TILE) continue;
          float s = C[c * TILE + r];
#pragma unroll
          for (int k = 0; k < 16; ++k) s = fmaf(-C[(o + k) * TILE + r], lc[k], s);
          C[c * TILE + r] = s;
        }
      }
    }
    csync();
  }
  return true;
}

__global__ void __launch_bounds__(kThreadsF, 2) chol_dag_f32_kernel(DagLaunch a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOffBarF);
  uint64_t* ljj_bar = full + kStagesF;
  int* stage_cnt = reinterpret_cast<int*>(ljj_bar + 1);
  float* C = reinterpret_cast<float*>(smem + kOffRingF);
  float* W = reinterpret_cast<float*>(smem + kOffWF);
  MiscF* misc = reinterpret_cast<MiscF*>(smem + kOffMiscF);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rg = lane >> 4, cg = lane & 15;
  const int R0 = 16 * warp + 8 * rg, C0 = 8 * cg;  // this lane's 8 x 8 block
  const int NT = a.NT, B = a.nslots;
  const int Npad = NT * TILE;
  const int ntasks = B * NT * (NT + 1) / 2;
  const int epoch = a.epoch;
  const size_t fstride = (size_t)(NT + 1) * NT;
  float* Xw = reinterpret_cast<float*>(smem + kOffXwF) + warp * 128;  // [16 rows][8 cols]

  if (tid == 0) {
    for (int s = 0; s < kStagesF; ++s) {
      mbar_init(&full[s], 1);
      stage_cnt[s] = 0;
    }
    mbar_init(ljj_bar, 1);
    fence_mbar_init();
    misc->ljj_phase = 0;
  }
  __syncthreads();

  uint32_t it = 0;
  while (true) {
    if (tid == 0) {
      const int t = atomicAdd(a.counter, 1);
      misc->ticket = t;
      misc->skip = 0;
      misc->fail = 0;
      if (t < ntasks) {
        int bpos, j, I;
        decode_task_f(t, B, NT, bpos, j, I);
        misc->bpos = bpos;
        misc->I = I;
        misc->j = j;
        misc->skip = *((volatile int*)&a.status[a.slots[bpos]]) != 0;
      }
    }
    __syncthreads();
    const int t = misc->ticket;
    if (t >= ntasks) break;
    const int bpos = misc->bpos, j = misc->j, I = misc->I;
    const bool diag = (I == j);
    const int slot = a.slots[bpos];
    const bool skip = misc->skip != 0;
    float* fac = reinterpret_cast<float*>(a.factors) + (size_t)slot * a.slot_stride;
    float* bord = reinterpret_cast<float*>(a.borders) + (size_t)slot * 2 * Npad;
    int* flags = a.flags + (size_t)slot * fstride;
    const int nslab = skip ? 0 : SLABS_PER_TILE * j;
    float* gtile = fac + tile_index(I, j) * TILE_ELEMS;

    // running residual: accumulators start from R(I, j)
    float acc[8][8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (skip) {
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[r][c] = 0.f;
      } else {
        const float4 x = __ldcg(reinterpret_cast<const float4*>(gtile + (C0 + c) * TILE + R0));
        const float4 y = __ldcg(reinterpret_cast<const float4*>(gtile + (C0 + c) * TILE + R0 + 4));
        acc[0][c] = x.x; acc[1][c] = x.y; acc[2][c] = x.z; acc[3][c] = x.w;
        acc[4][c] = y.x; acc[5][c] = y.y; acc[6][c] = y.z; acc[7][c] = y.w;
      }
    }
    const int brow = tid >> 7, bc = tid & 127;  // border role (DIAG)
    float wacc = (diag && !skip) ? __ldcg(bord + brow * Npad + j * TILE + bc) : 0.f;

    auto issue = [&](int p, uint32_t itp) {
      const int K = p >> 2, sq = p & 3;
      if (sq == 0) {
        wait_flag_f(&flags[j * NT + K], epoch, a.error);
        wait_flag_f(diag ? &flags[NT * NT + K] : &flags[I * NT + K], epoch, a.error);
        fence_proxy_async_global();
      }
      const int stage = itp % kStagesF;
      unsigned char* dst = smem + kOffRingF + stage * kStageBytesF;
      mbar_arrive_expect_tx(&full[stage], diag ? kSlabBytesF : kStageBytesF);
      bulk_g2s(dst, fac + tile_index(I, K) * TILE_ELEMS + sq * kSlabF, kSlabBytesF, &full[stage]);
      if (!diag)
        bulk_g2s(dst + kSlabBytesF, fac + tile_index(j, K) * TILE_ELEMS + sq * kSlabF, kSlabBytesF,
                 &full[stage]);
    };
    if (tid == 0)
      for (int p = 0; p < kStagesF && p < nslab; ++p) issue(p, it + p);
    for (int q = 0; q < nslab; ++q, ++it) {
      const int stage = it % kStagesF;
      mbar_wait(&full[stage], (it / kStagesF) & 1);
      const float* As = reinterpret_cast<const float*>(smem + kOffRingF + stage * kStageBytesF);
      const float* Bs = diag ? As : As + kSlabF;
#pragma unroll 4
      for (int kk = 0; kk < SLAB; ++kk) {
        float av[8], bv[8];
        ld8(av, As + kk * TILE + R0);
        ld8(bv, Bs + kk * TILE + C0);
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(-av[r], bv[c], acc[r][c]);
      }
      if (diag) {  // border rows: wacc -= sum_kk u_K[32 sq + kk] * L(j,K)[bc][32 sq + kk]
        const int K = q >> 2, sq = q & 3;
        const float* ub = bord + brow * Npad + K * TILE + sq * SLAB;
#pragma unroll 8
        for (int kk = 0; kk < SLAB; ++kk) wacc = fmaf(-__ldcg(ub + kk), Bs[kk * TILE + bc], wacc);
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&stage_cnt[stage], 1) == kWarpsF - 1) {
          stage_cnt[stage] = 0;
          if (q + kStagesF < nslab) {
            fence_proxy_async_shared();
            issue(q + kStagesF, it + kStagesF);
          }
        }
      }
    }
    csync();  // the ring is idle

    if (diag) {
      // ------------------------------ DIAG ------------------------------
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int r = 0; r < 8; ++r) C[(C0 + c) * TILE + R0 + r] = acc[r][c];
      if (!skip) W[brow * TILE + bc] = wacc;
      csync();
      bool ok = !skip;
      if (!skip) {
        ok = potrf_tile_f32(C, &misc->fail);
        if (!ok && tid == 0) atomicExch(&a.status[slot], 1);  // GPEMU_SLOT_NOT_PD
        csync();
      }
      if (ok)
        for (int e = 4 * tid; e < TILE_ELEMS; e += 4 * kThreadsF)
          __stcg(reinterpret_cast<float4*>(gtile + e), *reinterpret_cast<const float4*>(C + e));
      csync();
      if (tid == 0) publish_f(&flags[j * NT + j], epoch);
      // border solve: [u_j; v_j] = w L(j,j)^-T (column-oriented substitution)
      if (ok && warp < 2) {
        float* w = W + warp * TILE;
        for (int c = 0; c < TILE; ++c) {
          const float x = __fdiv_rn(w[c], C[c * TILE + c]);
          __syncwarp();
          for (int l = c + 1 + lane; l < TILE; l += 32) w[l] = fmaf(-x, C[c * TILE + l], w[l]);
          if (lane == 0) w[c] = x;
          __syncwarp();
        }
        for (int l = lane; l < TILE; l += 32) __stcg(bord + warp * Npad + j * TILE + l, w[l]);
      }
      csync();
      if (tid == 0) publish_f(&flags[NT * NT + j], epoch);
    } else {
      // ------------------------------ OFF -------------------------------
      if (!skip) {
        if (tid == 0) {
          wait_flag_f(&flags[j * NT + j], epoch, a.error);
          fence_proxy_async_global();
          mbar_arrive_expect_tx(ljj_bar, kTileBytesF);
          const float* Ljj = fac + tile_index(j, j) * TILE_ELEMS;
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4)
            bulk_g2s(smem + kOffRingF + s4 * kSlabBytesF, Ljj + s4 * kSlabF, kSlabBytesF, ljj_bar);
        }
        mbar_wait(ljj_bar, misc->ljj_phase & 1);
      }
      const bool run = !skip && *((volatile int*)&a.status[slot]) == 0;
      float* rinv = W;  // 1 / L_cc (IEEE), read by the substituting lanes
      if (run && tid < TILE) rinv[tid] = __frcp_rn(C[tid * TILE + tid]);
      csync();
      if (run) {
        const float* L = C;  // L(j,j), column-major
        for (int cb = 0; cb < 16; ++cb) {
          // (a) the two lanes holding column block cb substitute their 8 rows
          if (cg == cb) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float dcc = L[(C0 + c) * TILE + C0 + c], rcc = rinv[C0 + c];
#pragma unroll
              for (int r = 0; r < 8; ++r) acc[r][c] = div_by_f(acc[r][c], dcc, rcc);
#pragma unroll
              for (int c2 = c + 1; c2 < 8; ++c2) {
                const float l = L[(C0 + c) * TILE + C0 + c2];
#pragma unroll
                for (int r = 0; r < 8; ++r) acc[r][c2] = fmaf(-acc[r][c], l, acc[r][c2]);
              }
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              *reinterpret_cast<float4*>(Xw + (8 * rg + r) * 8) = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
              *reinterpret_cast<float4*>(Xw + (8 * rg + r) * 8 + 4) = make_float4(acc[r][4], acc[r][5], acc[r][6], acc[r][7]);
            }
          }
          __syncwarp();
          // (b) lanes to the right: acc[:, c'] -= X_block * L(j,j)[C0 + c', 8cb + c]^T
          if (cg > cb) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              float lv[8];
              ld8(lv, L + (8 * cb + c) * TILE + C0);
#pragma unroll
              for (int r = 0; r < 8; ++r) {
                const float x = Xw[(8 * rg + r) * 8 + c];
#pragma unroll
                for (int c2 = 0; c2 < 8; ++c2) acc[r][c2] = fmaf(-x, lv[c2], acc[r][c2]);
              }
            }
          }
          __syncwarp();
        }
        // L(I, j) -> HBM
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          __stcg(reinterpret_cast<float4*>(gtile + (C0 + c) * TILE + R0),
                 make_float4(acc[0][c], acc[1][c], acc[2][c], acc[3][c]));
          __stcg(reinterpret_cast<float4*>(gtile + (C0 + c) * TILE + R0 + 4),
                 make_float4(acc[4][c], acc[5][c], acc[6][c], acc[7][c]));
        }
      }
      csync();
      if (tid == 0) {
        if (!skip) ++misc->ljj_phase;
        publish_f(&flags[I * NT + j], epoch);
      }
    }
    __syncthreads();
  }
}

}  // namespace

size_t chol_dag_f32_smem_bytes() { return kSmemBytesF; }

void launch_chol_dag_f32(const DagLaunch& a, int num_sms, cudaStream_t s) {
  cudaFuncSetAttribute(chol_dag_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytesF);
  const int ntasks = a.nslots * a.NT * (a.NT + 1) / 2;
  const int slots = 2 * num_sms;  // two CTAs per SM
  const int grid = ntasks < slots ? ntasks : slots;
  cudaMemsetAsync(a.counter, 0, sizeof(int), s);
  chol_dag_f32_kernel<<<grid, kThreadsF, kSmemBytesF, s>>>(a);
}

}  // namespace gpemu_dev
