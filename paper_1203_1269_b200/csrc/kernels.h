// kernels.h -- host-side launchers for the sm_100a kernels (no torch types).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace gpemu_dev {

// ---- K1: correlation (kernels_corr.cu) -------------------------------------
// CorrelationPlan ctor (correlation.hpp:156-180): |x_ik - x_jk|^p for every
// lower-tile element, tile-major [tile][k][elem].
void launch_pow_table(const double* X, int n, int d, double p, int NT, double* table,
                      cudaStream_t s);
// CorrelationPlan::build_into (:187-223) + the ladder's diagonal jitter
// (backend.hpp:106-109) + border rows [y; 1] for every listed slot.
// slots[q] (q < nslots) indexes the slot; jitter[slot] is added to the diagonal.
void launch_assemble(const double* table, const double* theta /*[slot][d]*/, const double* y,
                     int n, int d, double nugget, int NT, const int* slots, int nslots,
                     const double* jitter, double* factors, size_t slot_stride, double* borders,
                     int* status, int num_sms, cudaStream_t s);
// Row-major n x n R for one theta (build_corr_matrix, correlation.hpp:99-146).
void launch_build_corr_rowmajor(const double* X, int n, int d, const double* theta, double p,
                                double nugget, double* R, int* bad, cudaStream_t s);
// Cross-correlation matrix r[j][i] for test points (corr_vector, :67-91).
void launch_corr_vectors(const double* Xt, int N, const double* X, int n, int d,
                         const double* theta, double p, double* r, int* bad, cudaStream_t s);

// ---- K2: Cholesky (kernels_chol.cu) ----------------------------------------
struct DagLaunch {
  double* factors;
  double* borders;
  size_t slot_stride;
  int n, NT;
  const int* slots;
  int nslots;
  int* counter;
  int* flags;      // [slot][NT+1][NT]
  int epoch;
  int* status;     // [slot]
  int* error;      // deadlock / timeout word
  unsigned long long* prof = nullptr;  // optional [grid][16] phase cycle counters
  // extension mode (prediction MSE): ext_rt row tiles of test points, [It][NT] tiles
  double* ext = nullptr;
  int ext_rt = 0;
  int* ext_flags = nullptr;  // [It][NT]
  // optional per-task timeline (diagnostics): trace[ticket][4] = globaltimer ns at task start,
  // after the GEMM phase, before the publish, and at the end; tickets >= trace_cap skipped
  unsigned long long* trace = nullptr;
  int trace_cap = 0;
  // optional ticket order (large launches): order[ticket] = bpos << 16 | I << 8 | j, a
  // topological order from a critical-path list schedule; null = the built-in column order
  const int* order = nullptr;
};

void launch_chol_dag(const DagLaunch& a, int num_sms, cudaStream_t s);
void launch_chol_simple(const DagLaunch& a, cudaStream_t s);
size_t chol_dag_smem_bytes();

// ---- K3: deviance (kernels_misc.cu) ----------------------------------------
// ProfileEvaluator::eval tail (likelihood.hpp:124-140).
// spec_off > 0: slots >= spec_off are speculation slots (layout.cuh spec_record_dst).
void launch_finalize(const double* factors, size_t slot_stride, const double* borders,
                     const int* status, const double* jitter, int n, int NT, const int* slots,
                     int nslots, double* out /*[slot][REC_SIZE]*/, int spec_off, cudaStream_t s);

// ---- layout conversions / solves (kernels_misc.cu) -------------------------
// Row-major n x n (lower used) + jitter on diagonal -> tiled slot storage.
void launch_rowmajor_to_tiles(const double* A, int n, int NT, double jitter, double* tiles,
                              cudaStream_t s);
// dot_accumulate (matrix.hpp:64-69) on the device: one thread, the reference's order.
void launch_dot_seq(const double* a, const double* b, int n, double* out, cudaStream_t s);
// Tiled -> row-major lower with strict upper zeroed.
void launch_tiles_to_rowmajor(const double* tiles, int n, int NT, double* L, cudaStream_t s);
// Blocked triangular solve on a tiled factor (kernels_trsv.cu, backend.hpp:129-153): forward
// (upper=0: L x = b) or backward (upper=1: L^T x = b). Right-hand side b[i] - mu * b2[i]
// (b2 nullable) for i < nb, zero past it; x: NT * 128 doubles (also the inter-block exchange).
// flags: NT ints never equal to a fresh `epoch` (epoch-valued, not cleared); counter: 1 int
// (reset by the launcher); error: deadlock-guard word.
void launch_tile_trsv(const double* tiles, int NT, const double* b, const double* b2, double mu,
                      int nb, double* x, int upper, int* flags, int* counter, int epoch,
                      int* error, int num_sms, cudaStream_t s);
size_t tile_trsv_smem_bytes();

// ---- K4: prediction (kernels_predict.cu) -----------------------------------
// yhat_j = mu + r_j' alpha for N test points (predictor.hpp:20-50), in a fixed summation
// order (128-row tiles inside 1024-row blocks) shared by the yhat-only and the MSE paths.
int predict_blocks(int n);
// yhat partials from a chunk's cross tiles (before the extension DAG), same order as predict
void launch_yhat_tiles(const double* ext, int Nc, int n, int NT, const double* alpha, double* part,
                       size_t N, size_t p0, cudaStream_t s);
void launch_predict_combine(const double* part, int N, int n, double mu, double* yhat,
                            cudaStream_t s);
// part: predict_blocks(n) * N doubles of scratch
void launch_predict(const double* Xt, int N, const double* X, int n, int d, const double* theta,
                    double p, double mu, const double* alpha, double* part, double* yhat, int* bad,
                    cudaStream_t s);
// Cross-correlation tiles of RT*128 test points against the design, [It][J] tile layout
// (rows past N and columns past n are zero).
void launch_cross_tiles(const double* Xt, int N, const double* X, int n, int d,
                        const double* theta, double p, int NT, int RT, double* ext, int* bad,
                        cudaStream_t s);
// Per test point from W = L^-1 r (ext tiles): yhat = mu + w.(u - mu v), mse =
// sigma2 (1 - w'w + (1 - v'w)^2 / v'v).
void launch_ext_reduce(const double* ext, int N, int n, int NT, const double* u, const double* v,
                       double mu, double sigma2, double vtv, double* yhat, double* mse,
                       cudaStream_t s);

// ---- single precision (kernels_f32.cu, kernels_chol_f32.cu) ------------------
// Float tiles are column-major 128 x 128 (element (r, c) at c * 128 + r); same packed-lower
// tile_index, slots, borders [y; 1] and record layout as the FP64 path.
// the single-precision plan keeps its |dx|^p table in double (column-major tiles)
void launch_pow_table_f32(const double* X, int n, int d, double p, int NT, double* table, cudaStream_t s);
void launch_assemble_f32(const double* table, const double* theta, const double* y, int n, int d,
                         double nugget, int NT, const int* slots, int nslots, const double* jitter,
                         float* factors, size_t slot_stride, float* borders, int* status, cudaStream_t s);
// DagLaunch with factors / borders pointing at float storage; no extension mode.
void launch_chol_dag_f32(const DagLaunch& a, int num_sms, cudaStream_t s);
size_t chol_dag_f32_smem_bytes();
void launch_finalize_f32(const float* factors, size_t slot_stride, const float* borders,
                         const int* status, const double* jitter, int n, int NT, const int* slots,
                         int nslots, double* out, int spec_off, cudaStream_t s);
void launch_alpha_f32(const float* tiles, int n, const double* y, double mu, double* alpha, cudaStream_t s);
void launch_tiles_f32_to_f64(const float* src, int NT, double* dst, cudaStream_t s);
void launch_tiles_f32_to_rowmajor(const float* tiles, int n, int NT, double* L, cudaStream_t s);
void launch_predict_f32(const double* Xt, int N, const double* X, int n, int d, const double* theta,
                        double p, double mu, const double* alpha, double* yhat, int* bad, cudaStream_t s);

// ---- design generation (kernels_design.cu) --------------------------------------
// maximin_lhd's tracker set-up and exchange loop (experiment.hpp:62-172) on a row-major n x d
// design already on the device. draws: 3 ints (k, a, b) per swap from the reference's RNG.
struct MaximinLaunch {
  double* x;
  int n, d, budget;
  const int* draws;
  unsigned long long* rmin0;  // per-row minimum distances (double bits), two buffers
  unsigned long long* rmin1;
  double* dra;                // new distances to the swapped rows
  double* drb;
  int* flist;                 // rows recomputed in full (<= n)
  unsigned long long* red;    // 8 words, host-initialised {inf, inf, inf, 0} x 2
  unsigned long long* init_min;  // global minimum of the start design, host-initialised to inf
  double* result;             // [final minimum distance, accepted swaps]
};
cudaError_t launch_maximin(const MaximinLaunch& a, int num_sms, cudaStream_t s);

}  // namespace gpemu_dev
