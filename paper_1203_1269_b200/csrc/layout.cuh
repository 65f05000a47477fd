// layout.cuh -- HBM layout of correlation / factor tiles for the B200 engine.
//
// The reference keeps R and its factor as dense row-major n x n matrices
// (matrix.hpp:14-59, backend.hpp:54-70). On the device each candidate's matrix
// lives as PACKED LOWER 128x128 TILES (only the lower triangle of tiles is
// stored: NT(NT+1)/2 tiles, NT = ceil(n/128), padded with an identity block).
// A tile is four contiguous 32-column "slabs" (128 rows x 32 cols, 32 KB) so a
// whole GEMM k-slab is one cp.async.bulk (TMA) copy; inside a slab rows are
// 32 doubles and the 4-double (32 B) chunks of row r are XOR-swizzled by
// (r & 7) so DMMA m8n8k4 fragment loads (8 rows x 4 k) hit distinct banks.
// The same element map is used in HBM and in shared memory.
#pragma once
#include <cstddef>
#include <cstdint>

namespace gpemu_dev {

constexpr int TILE = 128;
constexpr int SLAB = 32;
constexpr int TILE_ELEMS = TILE * TILE;  // 16384 doubles = 128 KB
constexpr int SLAB_ELEMS = TILE * SLAB;  // 4096 doubles = 32 KB
constexpr int SLABS_PER_TILE = TILE / SLAB;

// (row, col) inside a slab -> offset in doubles.
__host__ __device__ __forceinline__ int slab_off(int r, int cc) {
  return (r << 5) + ((((cc >> 2) ^ (r & 7))) << 2) + (cc & 3);
}

// (row, col) inside a tile -> offset in doubles.
__host__ __device__ __forceinline__ int elem_off(int r, int c) {
  return ((c >> 5) << 12) + slab_off(r, c & 31);
}

// Inverse of elem_off.
__host__ __device__ __forceinline__ void elem_rc(int off, int& r, int& c) {
  const int s = off >> 12;
  const int rem = off & 4095;
  r = rem >> 5;
  const int w = rem & 31;
  const int chunk = (w >> 2) ^ (r & 7);
  c = (s << 5) + (chunk << 2) + (w & 3);
}

__host__ __device__ __forceinline__ size_t tile_index(int I, int J) {
  return (size_t)I * (I + 1) / 2 + (size_t)J;
}

__host__ __device__ __forceinline__ int num_tiles(int NT) { return NT * (NT + 1) / 2; }

// Record destination of a finalize block (the speculative first ladder rung, capi.cu run_batch):
// with spec_off > 0, slot s >= spec_off evaluates candidate s - spec_off at jitter 1e-8 and
// writes that candidate's record when its jitter-0 attempt failed (status 1) and this one held;
// the base slot then writes nothing. -1: no record from this block.
__host__ __device__ __forceinline__ int spec_record_dst(const int* status, int slot, int st, int spec_off) {
  if (spec_off <= 0) return slot;
  if (slot >= spec_off) return (status[slot - spec_off] == 1 && st == 0) ? slot - spec_off : -1;
  return (st == 1 && status[slot + spec_off] == 0) ? -1 : slot;
}

// Per-slot result record (gpemu_eval_batch_device d_out layout).
enum { REC_NEG2 = 0, REC_MU, REC_SIGMA2, REC_JITTER, REC_LOGDET, REC_STATUS, REC_UTU, REC_VTV,
       REC_SIZE };

}  // namespace gpemu_dev
