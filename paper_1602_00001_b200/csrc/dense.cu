// Dense fp64 helpers beside the apply path (setup / the unrounded route):
//  * invop_dense_invert — Gauss-Jordan with partial pivoting for an arbitrary
//    dense matrix (reference dense.invert, dense.py:36-62, same singularity
//    rule: a pivot below PIVOT_RTOL*max|a| with PIVOT_RTOL = 1e-13). Grid
//    operators take the block-tridiagonal constructor instead (construct.cu).
//  * invop_dense_matvec — the reference's conventional dense multiply
//    (_native.pyx:75-92 / dense.apply_dense, dense.py:74-82): acc = m[r,0]*x[0],
//    then acc += m[r,j]*x[j] in ascending j, fp64, no FMA — bitwise equal.
#include "common.cuh"
#include <algorithm>
#include <cmath>

namespace invop {

// argmax_{i >= k} |M[i][k]|, first index on ties (BLAS idamax rule)
__global__ void k_gj_pivot(const double* __restrict__ M, int64_t n, int64_t ld, int64_t k,
                           int64_t* piv_row, double tol, int* status) {
  __shared__ double sv[1024];
  __shared__ int64_t si[1024];
  double best = -1.0;
  int64_t bi = k;
  for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) {
    double v = fabs(M[i * ld + k]);
    if (v > best) { best = v; bi = i; }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      double a = sv[threadIdx.x], b = sv[threadIdx.x + s];
      int64_t ia = si[threadIdx.x], ib = si[threadIdx.x + s];
      if (b > a || (b == a && ib < ia)) { sv[threadIdx.x] = b; si[threadIdx.x] = ib; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *piv_row = si[0];
    if (!(sv[0] >= tol)) *status = 1;
  }
}

// swap rows k <-> p over all 2n columns, compute the elimination factors of
// column k and scale the pivot row
__global__ void k_gj_swap(double* __restrict__ M, int64_t n, int64_t ld, int64_t k,
                          const int64_t* piv_row, double* __restrict__ f, const int* status) {
  if (*status) return;
  const int64_t p = *piv_row;
  const int64_t w = 2 * n;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < w;
       j += (int64_t)gridDim.x * blockDim.x) {
    if (p != k) {
      double t = M[k * ld + j];
      M[k * ld + j] = M[p * ld + j];
      M[p * ld + j] = t;
    }
  }
}

__global__ void k_gj_factors(double* __restrict__ M, int64_t n, int64_t ld, int64_t k,
                             double* __restrict__ f, const int* status) {
  if (*status) return;
  const double piv = M[k * ld + k];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    f[i] = (i == k) ? 0.0 : M[i * ld + k] / piv;
}

__global__ void k_gj_update(double* __restrict__ M, int64_t n, int64_t ld, int64_t k,
                            const double* __restrict__ f, const int* status) {
  if (*status) return;
  const int64_t w = 2 * n;
  // rows other than k: M[i][j] -= f[i] * M[k][j]   (column k ends at zero)
  int64_t total = n * w;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx / w, j = idx - i * w;
    if (i == k) continue;
    if (j == k) M[i * ld + j] = 0.0;
    else if (f[i] != 0.0) M[i * ld + j] -= f[i] * M[k * ld + j];
  }
}

__global__ void k_gj_scale(double* __restrict__ M, int64_t n, int64_t ld, int64_t k,
                           const int* status) {
  if (*status) return;
  const double piv = M[k * ld + k];
  const int64_t w = 2 * n;
  // column k of the pivot row is read by every thread: leave it for last
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < w;
       j += (int64_t)gridDim.x * blockDim.x)
    if (j != k) M[k * ld + j] = M[k * ld + j] / piv;
}

__global__ void k_gj_setup(const double* __restrict__ a, int64_t n, double* __restrict__ M,
                           int64_t ld) {
  int64_t total = n * 2 * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx / (2 * n), j = idx - i * 2 * n;
    M[i * ld + j] = j < n ? a[i * n + j] : (j - n == i ? 1.0 : 0.0);
  }
}

__global__ void k_gj_extract(const double* __restrict__ M, int64_t n, int64_t ld,
                             double* __restrict__ out) {
  int64_t total = n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx / n, j = idx - i * n;
    out[idx] = M[i * ld + n + j];
  }
}

// ordered dense matvec: warp per 32 rows, 32x32 tiles transposed through smem
__global__ void __launch_bounds__(128) k_dense_matvec(const double* __restrict__ m, int64_t rows,
                                                      int64_t cols, int64_t ld,
                                                      const double* __restrict__ x,
                                                      double* __restrict__ y) {
  __shared__ double tile[4][32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = ((int64_t)blockIdx.x * 4 + warp) * 32;
  if (row0 >= rows) return;
  double acc = 0.0;
  for (int64_t c0 = 0; c0 < cols; c0 += 32) {
    for (int r = 0; r < 32; ++r) {
      int64_t gr = row0 + r, gc = c0 + lane;
      tile[warp][r][lane] = (gr < rows && gc < cols) ? m[gr * ld + gc] : 0.0;
    }
    __syncwarp();
    int cend = (int)min((int64_t)32, cols - c0);
    for (int c = 0; c < cend; ++c) {
      double prod = __dmul_rn(tile[warp][lane][c], x[c0 + c]);
      acc = (c0 + c == 0) ? prod : __dadd_rn(acc, prod);
    }
    __syncwarp();
  }
  if (row0 + lane < rows) y[row0 + lane] = acc;
}

}  // namespace invop

using namespace invop;

extern "C" int invop_dense_invert(const double* a, int64_t n, double* out, double tol,
                                  void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0) return fail(INVOP_E_VALUE, "n < 0");
  if (n == 0) return INVOP_OK;
  int64_t ld = 2 * n;
  double* M = nullptr;
  double* f = nullptr;
  int64_t* piv = nullptr;
  int* status = nullptr;
  INVOP_CUDA(cudaMalloc(&M, (size_t)n * ld * sizeof(double)));
  INVOP_CUDA(cudaMalloc(&f, (size_t)n * sizeof(double)));
  INVOP_CUDA(cudaMalloc(&piv, sizeof(int64_t)));
  INVOP_CUDA(cudaMalloc(&status, sizeof(int)));
  INVOP_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
  int blocks = (int)std::min<int64_t>(cdiv(n * ld, 256), (int64_t)num_sms() * 8);
  int rb = (int)std::min<int64_t>(cdiv(ld, 256), (int64_t)num_sms() * 4);
  k_gj_setup<<<blocks, 256, 0, s>>>(a, n, M, ld);
  for (int64_t k = 0; k < n; ++k) {
    k_gj_pivot<<<1, 1024, 0, s>>>(M, n, ld, k, piv, tol, status);
    k_gj_swap<<<rb, 256, 0, s>>>(M, n, ld, k, piv, f, status);
    k_gj_factors<<<(int)std::min<int64_t>(cdiv(n, 256), 1024), 256, 0, s>>>(M, n, ld, k, f,
                                                                           status);
    k_gj_update<<<blocks, 256, 0, s>>>(M, n, ld, k, f, status);
    k_gj_scale<<<rb, 256, 0, s>>>(M, n, ld, k, status);
  }
  k_gj_extract<<<blocks, 256, 0, s>>>(M, n, ld, out);
  int h = 0;
  cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(M); cudaFree(f); cudaFree(piv); cudaFree(status);
  if (e != cudaSuccess) return cuda_fail(e, "dense_invert");
  if (h) return fail(INVOP_E_SINGULAR, "pivot below threshold; matrix is singular to working precision");
  return INVOP_OK;
}

extern "C" int invop_dense_matvec(const double* m, int64_t rows, int64_t cols, int64_t ld,
                                  const double* x, double* y, void* stream) {
  if (rows < 0 || cols < 0 || ld < cols) return fail(INVOP_E_VALUE, "bad geometry");
  if (rows == 0) return INVOP_OK;
  if (cols == 0) {
    INVOP_CUDA(cudaMemsetAsync(y, 0, rows * sizeof(double), (cudaStream_t)stream));
    return INVOP_OK;
  }
  int64_t warps = cdiv(rows, 32);
  k_dense_matvec<<<(unsigned)cdiv(warps, 4), 128, 0, (cudaStream_t)stream>>>(m, rows, cols, ld,
                                                                             x, y);
  INVOP_CHECK_LAUNCH("dense_matvec");
  return INVOP_OK;
}
