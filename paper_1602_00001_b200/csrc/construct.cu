// K4 — device construction of rows of L^-1 (setup, fp64), fused with K1 encode.
//
// Reference: the operator is assembled densely (grid.py:157-186) and inverted
// with LAPACK getrf/getrs on the identity (dense.py:36-62): O(N^3) flops and
// N^2 fp64 of host memory, capped at N <= 8192 (grid.py:21).
//
// Here the 5-point operator A on an nx x ny interior grid is kept as its five
// stencil diagonals. A is block tridiagonal (one nx x nx block per grid line),
// so rows R of A^-1 are obtained by solving M Z = E_R with M = A^T (columns of
// A^-T are rows of A^-1) by block LU without pivoting (A is a nonsingular
// M-matrix):
//   factor  : D_0 = B_0^T,  D_k = B_k^T - diag(lo_k) D_{k-1}^-1 diag(up_{k-1})
//   forward : G_k = D_k^-1 (F_k - diag(lo_k) G_{k-1})
//   backward: Z_k = G_k - (D_k^-1 diag(up_k)) Z_{k+1}
// The factorisation is sequential over grid lines (one CTA, Gauss-Jordan
// per block); the solves are independent per right-hand side, so each CTA
// owns a tile of T rows of L^-1 and sweeps the grid lines with dense fp64
// GEMMs against the cached D_k^-1 (L2-resident). Each finished tile is
// quantized (round half away from zero, quant.py:56-57) and written straight
// into the byte-plane code layout: the fp64 L^-1 is never stored.
// Work: ~4 nx^3 ny flops per right-hand side, i.e. 4 n^5 for the whole inverse
// of an n x n grid, versus (2/3+2) N^3 = (8/3) n^6 for dense LU + solve.
#include "common.cuh"
#include <cooperative_groups.h>
#include <algorithm>
#include <vector>
#include <cmath>
#include <cstring>

namespace invop {

namespace cg = cooperative_groups;

constexpr int K4_T = 32;        // right-hand sides (rows of L^-1) per tile
constexpr int K4_THREADS = 256;
constexpr int K4_KC = 16;       // K chunk of the D^-1 tile staged in smem
constexpr int K4_BLD = K4_T + 1; // padded row of the right-hand-side panel

static inline int64_t nx_pad(int64_t nx) { return round_up(nx, 32); }

// --------------------------------------------------------------- factor
// One CTA. D (nxp x nxp) lives in `work` (shared memory when it fits, else
// global). Writes Dinv_k and Q_k = Dinv_k diag(up_k) (zero padded).
__global__ void __launch_bounds__(1024) k4_factor(const double* __restrict__ diag,
                                                  const double* __restrict__ ww,
                                                  const double* __restrict__ we,
                                                  const double* __restrict__ ws,
                                                  const double* __restrict__ wn, int nx, int ny,
                                                  int nxp, double tol, double* __restrict__ dinv,
                                                  double* __restrict__ qmat,
                                                  double* __restrict__ gwork, int use_smem,
                                                  int* status) {
  extern __shared__ double sh[];
  double* D = use_smem ? sh : gwork;
  double* col = use_smem ? sh + (size_t)nxp * nxp : gwork + (size_t)nxp * nxp;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = nx;
  for (int k = 0; k < ny; ++k) {
    // build D_k (only the n x n leading part is meaningful)
    const double* prev = k > 0 ? dinv + (size_t)(k - 1) * nxp * nxp : nullptr;
    for (int idx = tid; idx < n * n; idx += nt) {
      int i = idx / n, j = idx - i * n;
      int64_t p = (int64_t)k * nx + i;
      double v = 0.0;
      if (i == j) v = diag[p];
      else if (j == i - 1) v = -we[p - 1];   // B^T[i][i-1] = B[i-1][i] = -w_east[p-1]
      else if (j == i + 1) v = -ww[p + 1];   // B^T[i][i+1] = B[i+1][i] = -w_west[p+1]
      if (k > 0) {
        double lo = -wn[(int64_t)(k - 1) * nx + i];   // M[(k,i),(k-1,i)] = A[(k-1,i),(k,i)]
        double up = -ws[(int64_t)k * nx + j];         // M[(k-1,j),(k,j)] = A[(k,j),(k-1,j)]
        v = __dsub_rn(v, __dmul_rn(__dmul_rn(lo, prev[(size_t)i * nxp + j]), up));
      }
      D[(size_t)i * nxp + j] = v;
    }
    __syncthreads();
    // in-place Gauss-Jordan (no pivoting: D_k is a diagonally dominant M-matrix)
    for (int piv = 0; piv < n; ++piv) {
      double pv = D[(size_t)piv * nxp + piv];
      if (!(fabs(pv) >= tol)) {
        if (tid == 0) *status = 1;
        return;  // uniform across the CTA
      }
      double inv_p = 1.0 / pv;
      for (int i = tid; i < n; i += nt) col[i] = D[(size_t)i * nxp + piv];
      __syncthreads();
      for (int j = tid; j < n; j += nt)
        D[(size_t)piv * nxp + j] = (j == piv) ? inv_p : D[(size_t)piv * nxp + j] * inv_p;
      __syncthreads();
      for (int idx = tid; idx < n * n; idx += nt) {
        int i = idx / n, j = idx - i * n;
        if (i == piv) continue;
        double f = col[i];
        if (j == piv) D[(size_t)i * nxp + j] = -f * inv_p;
        else D[(size_t)i * nxp + j] -= f * D[(size_t)piv * nxp + j];
      }
      __syncthreads();
    }
    // store Dinv_k and Q_k (zero padded to nxp)
    double* dk = dinv + (size_t)k * nxp * nxp;
    double* qk = qmat + (size_t)k * nxp * nxp;
    for (int idx = tid; idx < nxp * nxp; idx += nt) {
      int i = idx / nxp, j = idx - i * nxp;
      double v = (i < n && j < n) ? D[(size_t)i * nxp + j] : 0.0;
      dk[idx] = v;
      double up = (k + 1 < ny && j < n) ? -ws[(int64_t)(k + 1) * nx + j] : 0.0;
      qk[idx] = v * up;
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------- factor on a cluster
// The same block LU and the same per-element arithmetic as k4_factor (so the
// same bits), with the nx x nx Schur block distributed over a cluster of CL
// CTAs, K4C_R rows each, held in shared memory for the whole factorisation
// (one CTA kept it in global memory for nx > 160 and ran 1.4 s at config 5).
// Per pivot p: one cluster barrier (every CTA finished pivot p-1, so row p is
// final), every CTA copies row p from its owner through DSMEM into a
// double-buffered pivot row, scales it by 1/D[p][p] locally and eliminates its
// own rows; the owner writes the scaled row p back lazily at pivot p+1 (after
// the next barrier, when no CTA reads it any more). D_{k+1} is built from the
// CTA's own rows of D_k^-1 (elementwise), so block steps need no exchange.
constexpr int K4C_R = 16;        // rows per CTA
constexpr int K4C_THREADS = 256;

__global__ void __launch_bounds__(K4C_THREADS) k4_factor_cl(
    const double* __restrict__ diag, const double* __restrict__ ww, const double* __restrict__ we,
    const double* __restrict__ ws, const double* __restrict__ wn, int nx, int ny, int nxp,
    double tol, double* __restrict__ dinv, double* __restrict__ qmat, int* status) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double shc[];
  double* D = shc;                                  // [K4C_R][nxp] own rows
  double* prow = shc + (size_t)K4C_R * nxp;         // [2][nxp] pivot row copies
  const int c = (int)cl.block_rank();
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = nx;
  const int r0 = c * K4C_R;                         // first global row of this CTA
  for (int k = 0; k < ny; ++k) {
    // D_k rows r0 .. r0+R (own), from the CTA's own rows of D_{k-1}^-1
    for (int idx = tid; idx < K4C_R * n; idx += nt) {
      const int li = idx / n, j = idx - li * n, i = r0 + li;
      if (i >= n) continue;
      const int64_t p = (int64_t)k * nx + i;
      double v = 0.0;
      if (i == j) v = diag[p];
      else if (j == i - 1) v = -we[p - 1];
      else if (j == i + 1) v = -ww[p + 1];
      if (k > 0) {
        const double lo = -wn[(int64_t)(k - 1) * nx + i];
        const double up = -ws[(int64_t)k * nx + j];
        v = __dsub_rn(v, __dmul_rn(__dmul_rn(lo, D[(size_t)li * nxp + j]), up));
      }
      D[(size_t)li * nxp + j] = v;
    }
    // Gauss-Jordan, pivots in order (diagonally dominant M-matrix: no pivoting)
    for (int piv = 0; piv < n; ++piv) {
      cl.sync();                                    // pivot piv-1 done everywhere
      const int owner = piv / K4C_R, lrow = piv - owner * K4C_R;
      double* pr = prow + (size_t)(piv & 1) * nxp;
      // lazy write-back of the previous scaled pivot row (its owner only)
      if (piv > 0 && (piv - 1) / K4C_R == c) {
        const double* pp = prow + (size_t)((piv - 1) & 1) * nxp;
        const int lq = (piv - 1) - c * K4C_R;
        const double inv_q = 1.0 / pp[piv - 1];
        for (int j = tid; j < n; j += nt)
          D[(size_t)lq * nxp + j] = (j == piv - 1) ? inv_q : pp[j] * inv_q;
      }
      const double* src = cl.map_shared_rank(D + (size_t)lrow * nxp, owner);
      for (int j = tid; j < n; j += nt) pr[j] = src[j];
      __syncthreads();
      const double pv = pr[piv];
      if (!(fabs(pv) >= tol)) {
        if (tid == 0 && c == 0) *status = 1;
        cl.sync();                                  // uniform: every CTA saw the same pivot
        return;
      }
      const double inv_p = 1.0 / pv;
      for (int idx = tid; idx < K4C_R * n; idx += nt) {
        const int li = idx / n, j = idx - li * n, i = r0 + li;
        if (i >= n || i == piv) continue;
        const double f = D[(size_t)li * nxp + piv];
        // same arithmetic as k4_factor: the pivot row is scaled first
        if (j != piv) D[(size_t)li * nxp + j] -= f * (pr[j] * inv_p);
      }
      __syncthreads();
      for (int li = tid; li < K4C_R; li += nt) {
        const int i = r0 + li;
        if (i < n && i != piv) D[(size_t)li * nxp + piv] = -D[(size_t)li * nxp + piv] * inv_p;
      }
    }
    cl.sync();
    if ((n - 1) / K4C_R == c) {                     // the last pivot row's write-back
      const double* pp = prow + (size_t)((n - 1) & 1) * nxp;
      const int lq = (n - 1) - c * K4C_R;
      const double inv_q = 1.0 / pp[n - 1];
      for (int j = tid; j < n; j += nt) D[(size_t)lq * nxp + j] = (j == n - 1) ? inv_q : pp[j] * inv_q;
    }
    __syncthreads();
    // store own rows of Dinv_k and Q_k (zero padded to nxp)
    double* dk = dinv + (size_t)k * nxp * nxp;
    double* qk = qmat + (size_t)k * nxp * nxp;
    for (int idx = tid; idx < K4C_R * nxp; idx += nt) {
      const int li = idx / nxp, j = idx - li * nxp, i = r0 + li;
      if (i >= nxp) continue;
      const double v = (i < n && j < n) ? D[(size_t)li * nxp + j] : 0.0;
      dk[(size_t)i * nxp + j] = v;
      const double up = (k + 1 < ny && j < n) ? -ws[(int64_t)(k + 1) * nx + j] : 0.0;
      qk[(size_t)i * nxp + j] = v * up;
    }
  }
  cl.sync();                                        // peers may read our D until here
}

// --------------------------------------------------------------- sweeps
struct SweepArgs {
  const double* dinv;
  const double* qmat;
  const double* wn;
  int nx, ny, nxp;
  int64_t N;
  int64_t row0, rows;     // rows of L^-1 to produce
  double* zbuf;           // [grid][T][N] scratch
  // outputs (one of the two)
  double* out_f64; int64_t ld_out;
  uint8_t* planes[4]; int64_t ld_planes; int P_alloc;
  double p10;
  long long* stats;              // min, max, nnz
  unsigned long long* maxabs_bits;
};

// C[nxp x T] = A[nxp x nxp] * Bs[nxp x T] (Bs in smem, row-major [kk][t]).
// Thread (ti, tj): rows ti + 32*m, columns 4*tj .. 4*tj+3.
template <int MR>
__device__ __forceinline__ void gemm_tile(const double* __restrict__ A, const double* Bs,
                                          double* As, int nxp, double (&acc)[MR][4]) {
  const int tid = threadIdx.x;
  const int ti = tid & 31, tj = tid >> 5;  // tj in 0..7
  for (int m = 0; m < MR; ++m)
    for (int c = 0; c < 4; ++c) acc[m][c] = 0.0;
  for (int k0 = 0; k0 < nxp; k0 += K4_KC) {
    // stage A[:, k0:k0+KC] as As[i][kk]
    for (int idx = tid; idx < nxp * K4_KC; idx += K4_THREADS) {
      int i = idx / K4_KC, kk = idx - i * K4_KC;
      As[i * (K4_KC + 1) + kk] = A[(size_t)i * nxp + k0 + kk];
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < K4_KC; ++kk) {
      double b[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[(k0 + kk) * K4_BLD + tj * 4 + c];
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        int i = ti + 32 * m;
        if (i < nxp) {
          double av = As[i * (K4_KC + 1) + kk];
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[m][c] = fma(av, b[c], acc[m][c]);
        }
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double round_half_away_k4(double e, double p10) {
  double scaled = __dmul_rn(e, p10);
  double m = floor(__dadd_rn(fabs(scaled), 0.5));
  return copysign(m, scaled);
}

template <int MR>
__global__ void __launch_bounds__(K4_THREADS) k4_sweep(SweepArgs a) {
  extern __shared__ double sm4[];
  double* Bs = sm4;                                   // [nxp][T+1]
  double* As = sm4 + (size_t)a.nxp * K4_BLD;          // [nxp][KC+1]
  const int tid = threadIdx.x;
  const int ti = tid & 31, tj = tid >> 5;
  const int nx = a.nx, nxp = a.nxp, ny = a.ny;
  const int64_t N = a.N;
  double* Z = a.zbuf + (size_t)blockIdx.x * K4_T * N;  // [T][N]
  const int64_t ntiles = cdiv(a.rows, K4_T);

  int64_t mn = INT64_MAX, mx = INT64_MIN, nz = 0;
  unsigned long long mab = 0;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t rbase = a.row0 + tile * K4_T;
    const int k_start = (int)(rbase / nx);
    // ---------------- forward sweep
    for (int k = k_start; k < ny; ++k) {
      // Bs = F_k - diag(lo_k) G_{k-1}
      for (int idx = tid; idx < nxp * K4_T; idx += K4_THREADS) {
        int t = idx / nxp, i = idx - t * nxp;
        double v = 0.0;
        if (i < nx) {
          int64_t p = (int64_t)k * nx + i;
          int64_t r = rbase + t;
          if (r == p && r < a.row0 + a.rows) v = 1.0;
          if (k > k_start) {
            double lo = -a.wn[(int64_t)(k - 1) * nx + i];
            v = __dsub_rn(v, __dmul_rn(lo, Z[(size_t)t * N + (int64_t)(k - 1) * nx + i]));
          }
        }
        Bs[i * K4_BLD + t] = v;
      }
      __syncthreads();
      double acc[MR][4];
      gemm_tile<MR>(a.dinv + (size_t)k * nxp * nxp, Bs, As, nxp, acc);
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        int i = ti + 32 * m;
        if (i < nx)
#pragma unroll
          for (int c = 0; c < 4; ++c) Z[(size_t)(tj * 4 + c) * N + (int64_t)k * nx + i] = acc[m][c];
      }
      __syncthreads();
    }
    // ---------------- backward sweep: Z_k = G_k - Q_k Z_{k+1}
    for (int k = ny - 2; k >= 0; --k) {
      for (int idx = tid; idx < nxp * K4_T; idx += K4_THREADS) {
        int t = idx / nxp, i = idx - t * nxp;
        Bs[i * K4_BLD + t] = i < nx ? Z[(size_t)t * N + (int64_t)(k + 1) * nx + i] : 0.0;
      }
      __syncthreads();
      double acc[MR][4];
      gemm_tile<MR>(a.qmat + (size_t)k * nxp * nxp, Bs, As, nxp, acc);
#pragma unroll
      for (int m = 0; m < MR; ++m) {
        int i = ti + 32 * m;
        if (i < nx)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            size_t zi = (size_t)(tj * 4 + c) * N + (int64_t)k * nx + i;
            double g = k >= k_start ? Z[zi] : 0.0;
            Z[zi] = __dsub_rn(g, acc[m][c]);
          }
      }
      __syncthreads();
    }
    // ---------------- emit rows rbase .. rbase+T-1 of L^-1
    for (int t = 0; t < K4_T; ++t) {
      int64_t r = rbase + t;
      if (r >= a.row0 + a.rows) break;
      const double* zr = Z + (size_t)t * N;
      int64_t lr = r - a.row0;
      if (a.out_f64) {
        for (int64_t j = tid; j < N; j += K4_THREADS) a.out_f64[lr * a.ld_out + j] = zr[j];
      } else {
        for (int64_t j = tid; j < a.ld_planes; j += K4_THREADS) {
          uint64_t u = 0;
          if (j < N) {
            double mf = round_half_away_k4(zr[j], a.p10);
            unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(mf));
            mab = bits > mab ? bits : mab;
            int64_t v = (int64_t)mf;
            mn = min(mn, v); mx = max(mx, v); nz += (v != 0);
            u = (uint64_t)v;
          }
          for (int b = 0; b < a.P_alloc; ++b)
            a.planes[b][lr * a.ld_planes + j] = (uint8_t)(u >> (8 * b));
        }
      }
    }
    __syncthreads();
  }
  if (!a.out_f64) {
    // block-level commit of the encode statistics
    __shared__ long long s_mn[K4_THREADS / 32], s_mx[K4_THREADS / 32], s_nz[K4_THREADS / 32];
    __shared__ unsigned long long s_ma[K4_THREADS / 32];
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, (int64_t)__shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, mx, o));
      nz += __shfl_xor_sync(0xffffffffu, nz, o);
      unsigned long long t2 = __shfl_xor_sync(0xffffffffu, mab, o);
      mab = t2 > mab ? t2 : mab;
    }
    int w = tid >> 5;
    if ((tid & 31) == 0) { s_mn[w] = mn; s_mx[w] = mx; s_nz[w] = nz; s_ma[w] = mab; }
    __syncthreads();
    if (tid == 0) {
      nz = 0;
      for (int i = 0; i < K4_THREADS / 32; ++i) {
        mn = min(mn, (int64_t)s_mn[i]); mx = max(mx, (int64_t)s_mx[i]); nz += s_nz[i];
        mab = s_ma[i] > mab ? s_ma[i] : mab;
      }
      atomicMin(&a.stats[0], (long long)mn);
      atomicMax(&a.stats[1], (long long)mx);
      atomicAdd((unsigned long long*)&a.stats[2], (unsigned long long)nz);
      atomicMax(a.maxabs_bits, mab);
    }
  }
}

template <int MR>
static int launch_sweep(const SweepArgs& a, int grid, cudaStream_t s) {
  size_t smem = ((size_t)a.nxp * K4_BLD + (size_t)a.nxp * (K4_KC + 1)) * sizeof(double);
  cudaFuncSetAttribute(k4_sweep<MR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)std::max<size_t>(smem, 48 * 1024));
  k4_sweep<MR><<<grid, K4_THREADS, smem, s>>>(a);
  INVOP_CHECK_LAUNCH("k4_sweep");
  return INVOP_OK;
}

static int run_sweep(SweepArgs a, cudaStream_t s) {
  int64_t ntiles = cdiv(a.rows, K4_T);
  // scratch: one [T][N] fp64 panel per resident CTA, capped at ~4 GB
  int64_t per = (int64_t)K4_T * a.N * 8;
  int64_t cap = std::max<int64_t>(1, ((int64_t)4 << 30) / per);
  int grid = (int)std::min<int64_t>({ntiles, (int64_t)num_sms() * 2, cap});
  double* z = nullptr;
  INVOP_CUDA(cudaMalloc(&z, (size_t)grid * per));
  a.zbuf = z;
  int mr = a.nxp / 32;
  int rc;
  switch (mr) {
    case 1: rc = launch_sweep<1>(a, grid, s); break;
    case 2: rc = launch_sweep<2>(a, grid, s); break;
    case 3: rc = launch_sweep<3>(a, grid, s); break;
    case 4: rc = launch_sweep<4>(a, grid, s); break;
    case 5: rc = launch_sweep<5>(a, grid, s); break;
    case 6: rc = launch_sweep<6>(a, grid, s); break;
    case 7: rc = launch_sweep<7>(a, grid, s); break;
    case 8: rc = launch_sweep<8>(a, grid, s); break;
    default: rc = fail(INVOP_E_UNSUPPORTED, "grid lines longer than 256 points");
  }
  cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(z);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "k4_sweep");
  return INVOP_OK;
}

}  // namespace invop

using namespace invop;

extern "C" int invop_operator_create(int64_t nx, int64_t ny, const double* diag,
                                     const double* w_west, const double* w_east,
                                     const double* w_south, const double* w_north, void* stream,
                                     invop_operator** out) {
  if (!out) return fail(INVOP_E_VALUE, "out is NULL");
  *out = nullptr;
  if (nx < 1 || ny < 1) return fail(INVOP_E_VALUE, "grid needs at least one interior point");
  if (nx > 256) return fail(INVOP_E_UNSUPPORTED, "grid lines longer than 256 points");
  cudaStream_t s = (cudaStream_t)stream;
  invop_operator* op = new invop_operator();
  op->nx = nx; op->ny = ny; op->N = nx * ny;
  size_t b = (size_t)op->N * sizeof(double);
  const double* src[5] = {diag, w_west, w_east, w_south, w_north};
  double** dst[5] = {&op->diag, &op->ww, &op->we, &op->ws, &op->wn};
  double mx = 0.0;
  for (int i = 0; i < 5; ++i) {
    if (cudaMalloc(dst[i], b) != cudaSuccess) {
      invop_operator_destroy(op);
      return fail(INVOP_E_CUDA, "cudaMalloc operator");
    }
    cudaMemcpyAsync(*dst[i], src[i], b, cudaMemcpyHostToDevice, s);
    for (int64_t p = 0; p < op->N; ++p) mx = std::max(mx, std::fabs(src[i][p]));
  }
  // couplings across the boundary must be zero (Dirichlet neighbours dropped)
  for (int64_t r = 0; r < ny; ++r)
    for (int64_t c = 0; c < nx; ++c) {
      int64_t p = r * nx + c;
      if ((c == 0 && w_west[p] != 0.0) || (c == nx - 1 && w_east[p] != 0.0) ||
          (r == 0 && w_south[p] != 0.0) || (r == ny - 1 && w_north[p] != 0.0)) {
        invop_operator_destroy(op);
        return fail(INVOP_E_VALUE, "stencil couples to a point outside the interior grid");
      }
    }
  op->max_entry = mx;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { invop_operator_destroy(op); return cuda_fail(e, "operator upload"); }
  *out = op;
  return INVOP_OK;
}

extern "C" int invop_operator_destroy(invop_operator* op) {
  if (!op) return INVOP_OK;
  double* ptrs[7] = {op->diag, op->ww, op->we, op->ws, op->wn, op->dinv, op->qmat};
  for (double* p : ptrs)
    if (p) cudaFree(p);
  delete op;
  return INVOP_OK;
}

extern "C" int invop_operator_factor(invop_operator* op, void* stream) {
  if (!op) return fail(INVOP_E_VALUE, "operator is NULL");
  if (op->factored) return INVOP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t nxp = nx_pad(op->nx);
  size_t blk = (size_t)nxp * nxp * sizeof(double);
  INVOP_CUDA(cudaMalloc(&op->dinv, blk * op->ny));
  INVOP_CUDA(cudaMalloc(&op->qmat, blk * op->ny));
  double tol_c = 1e-13 * op->max_entry;  // PIVOT_RTOL of dense.py:16
  const char* kc = getenv("INVOP_K4_CLUSTER");
  if (nxp <= 16 * K4C_R && !(kc && *kc == '0')) {
    // Schur block distributed over a cluster (one cluster barrier per pivot)
    const int clsz = (int)(nxp / K4C_R);
    int* status = nullptr;
    INVOP_CUDA(cudaMalloc(&status, sizeof(int)));
    INVOP_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
    const size_t csm = ((size_t)K4C_R + 2) * nxp * sizeof(double);
    if (clsz > 8) INVOP_CUDA(cudaFuncSetAttribute(k4_factor_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    INVOP_CUDA(cudaFuncSetAttribute(k4_factor_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(csm, 48 * 1024)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clsz);
    cfg.blockDim = dim3(K4C_THREADS);
    cfg.dynamicSmemBytes = csm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = clsz;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e1 = cudaLaunchKernelEx(&cfg, k4_factor_cl, (const double*)op->diag, (const double*)op->ww,
                                        (const double*)op->we, (const double*)op->ws,
                                        (const double*)op->wn, (int)op->nx, (int)op->ny, (int)nxp, tol_c,
                                        op->dinv, op->qmat, status);
    int h = 0;
    cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    cudaFree(status);
    if (e1 != cudaSuccess) return cuda_fail(e1, "k4_factor_cl launch");
    if (e != cudaSuccess) return cuda_fail(e, "k4_factor_cl");
    if (h) return fail(INVOP_E_SINGULAR, "block pivot below 1e-13*max|entry|; operator is singular");
    op->factored = 1;
    return INVOP_OK;
  }
  size_t smem = blk + nxp * sizeof(double);
  int use_smem = smem <= 200 * 1024;
  double* gwork = nullptr;
  if (!use_smem) INVOP_CUDA(cudaMalloc(&gwork, blk + nxp * sizeof(double)));
  int* status = nullptr;
  INVOP_CUDA(cudaMalloc(&status, sizeof(int)));
  INVOP_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
  size_t dyn = use_smem ? smem : 0;
  cudaFuncSetAttribute(k4_factor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)std::max<size_t>(dyn, 48 * 1024));
  double tol = 1e-13 * op->max_entry;  // PIVOT_RTOL of dense.py:16
  k4_factor<<<1, 1024, dyn, s>>>(op->diag, op->ww, op->we, op->ws, op->wn, (int)op->nx,
                                 (int)op->ny, (int)nxp, tol, op->dinv, op->qmat, gwork,
                                 use_smem, status);
  int h = 0;
  cudaError_t e1 = cudaGetLastError();
  cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(status);
  if (gwork) cudaFree(gwork);
  if (e1 != cudaSuccess) return cuda_fail(e1, "k4_factor launch");
  if (e != cudaSuccess) return cuda_fail(e, "k4_factor");
  if (h) return fail(INVOP_E_SINGULAR, "block pivot below 1e-13*max|entry|; operator is singular");
  op->factored = 1;
  return INVOP_OK;
}

static int construct_common(invop_operator* op, int64_t row0, int64_t rows) {
  if (!op) return fail(INVOP_E_VALUE, "operator is NULL");
  if (row0 < 0 || rows < 0 || row0 + rows > op->N) return fail(INVOP_E_VALUE, "bad row range");
  return INVOP_OK;
}

extern "C" int invop_construct_rows_f64(invop_operator* op, int64_t row0, int64_t rows,
                                        double* out, int64_t ld, void* stream) {
  int rc = construct_common(op, row0, rows);
  if (rc) return rc;
  if (ld < op->N) return fail(INVOP_E_VALUE, "ld < N");
  rc = invop_operator_factor(op, stream);
  if (rc) return rc;
  if (rows == 0) return INVOP_OK;
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.dinv = op->dinv; a.qmat = op->qmat; a.wn = op->wn;
  a.nx = (int)op->nx; a.ny = (int)op->ny; a.nxp = (int)nx_pad(op->nx); a.N = op->N;
  a.row0 = row0; a.rows = rows;
  a.out_f64 = out; a.ld_out = ld;
  return run_sweep(a, (cudaStream_t)stream);
}

extern "C" int invop_construct_rows(invop_operator* op, int64_t row0, int64_t rows, int digits,
                                    void* stream, invop_plan** out) {
  if (!out) return fail(INVOP_E_VALUE, "out is NULL");
  *out = nullptr;
  int rc = construct_common(op, row0, rows);
  if (rc) return rc;
  if (digits < 0 || digits > 12) return fail(INVOP_E_VALUE, "digits must be in 0..12");
  cudaStream_t s = (cudaStream_t)stream;
  rc = invop_operator_factor(op, stream);
  if (rc) return rc;
  invop_plan* p = new invop_plan();
  p->n = op->N; p->rows = rows; p->row0 = row0; p->digits = digits;
  p->ld = round_up(op->N, 512);
  p->scale = 1.0 / invop_pow10_exact(digits);
  cudaGetDevice(&p->device);
  const int P_alloc = 4;
  rc = plan_alloc_planes(p, P_alloc);
  if (rc) { invop_plan_destroy(p); return rc; }
  long long* stats = nullptr;
  if (cudaMalloc(&stats, 4 * sizeof(long long)) != cudaSuccess) {
    invop_plan_destroy(p);
    return fail(INVOP_E_CUDA, "cudaMalloc stats");
  }
  long long init[4] = {INT64_MAX, INT64_MIN, 0, 0};
  cudaMemcpyAsync(stats, init, sizeof(init), cudaMemcpyHostToDevice, s);
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.dinv = op->dinv; a.qmat = op->qmat; a.wn = op->wn;
  a.nx = (int)op->nx; a.ny = (int)op->ny; a.nxp = (int)nx_pad(op->nx); a.N = op->N;
  a.row0 = row0; a.rows = rows;
  for (int b = 0; b < 4; ++b) a.planes[b] = p->planes[b];
  a.ld_planes = p->ld; a.P_alloc = P_alloc;
  a.p10 = invop_pow10_exact(digits);
  a.stats = stats;
  a.maxabs_bits = (unsigned long long*)(stats + 3);
  rc = rows > 0 ? run_sweep(a, s) : INVOP_OK;
  long long h[4] = {0, 0, 0, 0};
  cudaMemcpy(h, stats, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(stats);
  if (rc) { invop_plan_destroy(p); return rc; }
  double worst;
  memcpy(&worst, &h[3], sizeof(double));
  if (rows > 0 && worst > 9007199254740992.0) {
    invop_plan_destroy(p);
    return fail(INVOP_E_OVERFLOW, "mantissa beyond 2^53");
  }
  if (rows > 0 && (h[0] < -(1ll << 31) || h[1] > (1ll << 31) - 1)) {
    invop_plan_destroy(p);
    return fail(INVOP_E_UNSUPPORTED, "constructed mantissas need more than 4 bytes");
  }
  plan_finalize_width(p, rows > 0 ? h[0] : 0, rows > 0 ? h[1] : 0, h[2]);
  // narrowest width; the low planes already hold the right bytes
  int sgn = 1;
  int P = 4;
  for (int q = 1; q <= 4; ++q) {
    int64_t lo = -(1ll << (8 * q - 1)), hi = (1ll << (8 * q - 1)) - 1;
    if (p->min_val >= lo && p->max_val <= hi) { P = q; sgn = 1; break; }
    if (p->min_val >= 0 && (uint64_t)p->max_val < (1ull << (8 * q))) { P = q; sgn = 0; break; }
  }
  for (int b = P; b < 4; ++b) { cudaFree(p->planes[b]); p->planes[b] = nullptr; }
  p->P = P;
  p->is_signed = sgn;
  *out = p;
  return INVOP_OK;
}
