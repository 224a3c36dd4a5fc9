// The reference's grouped apply, as written, on the device — a design
// comparison for DESIGN.md ("No grouping on the device"), not a product route.
//
// _native.pyx:15-49 walks the CSC group tables: per (column j, distinct
// |mantissa| g) one multiplication t = coeff_g * x_j, then `out[row] += +-t` for
// every entry of the group. Here one warp takes a column, its lanes take the
// column's groups, and the scatter is an fp64 atomic add (the order of the adds
// into a row is therefore not the reference's: not bitwise). The kernel streams
// what the reference streams — 16 B per group (coefficient + group pointer) and
// 5 B per entry (row + sign) — plus 8 B of atomic traffic per entry.
#include "common.cuh"
#include <algorithm>

namespace invop {

__global__ void k_grouped_csc(int64_t n, const int64_t* __restrict__ col_ptr,
                              const double* __restrict__ coeff, const int64_t* __restrict__ gptr,
                              const int32_t* __restrict__ rows, const int8_t* __restrict__ signs,
                              const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += warps) {
    const int64_t g0 = col_ptr[j], g1 = col_ptr[j + 1];
    const double xj = x[j];
    for (int64_t g = g0 + lane; g < g1; g += 32) {
      const double t = __dmul_rn(coeff[g], xj);                 // one multiply per group
      for (int64_t e = gptr[g]; e < gptr[g + 1]; ++e)
        atomicAdd(&y[rows[e]], signs[e] > 0 ? t : -t);          // one add per entry
    }
  }
}

}  // namespace invop

using namespace invop;

extern "C" int invop_apply_grouped_csc(int64_t n, const int64_t* col_ptr, const double* group_coeff,
                                       const int64_t* group_ptr, const int32_t* entry_rows,
                                       const int8_t* entry_signs, const double* x, double* y,
                                       void* stream) {
  if (n < 0 || (n > 0 && (!col_ptr || !group_ptr || !x || !y)))
    return fail(INVOP_E_VALUE, "NULL argument");
  if (n == 0) return INVOP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  INVOP_CUDA(cudaMemsetAsync(y, 0, (size_t)n * sizeof(double), s));
  const int grid = (int)std::min<int64_t>(num_sms() * 8, cdiv(n, 8));
  k_grouped_csc<<<grid, 256, 0, s>>>(n, col_ptr, group_coeff, group_ptr, entry_rows, entry_signs, x, y);
  INVOP_CHECK_LAUNCH("k_grouped_csc");
  return INVOP_OK;
}
