// Row-difference layout (DL) and its single right-hand-side apply k2_dl.
//
// Rows of the quantized inverse of a smooth operator are smooth functions of
// the row index: row r and rows r-1, r-2 are Green's functions of neighbouring
// grid points. DL stores, per row, the second-order residual
//
//     e_r = v_r - 2 v_{r-1} + v_{r-2}        (order 2)
//
// (order 1, e_r = v_r - v_{r-1}, for the second row of a CTA's row range and
// order 0, e_r = v_r, for its first), with a byte width chosen per 512-column
// chunk: 1.57 B/entry at config 4 and 1.06 B/entry at config 5, against 3 and 2
// for the byte planes (tools/delta_stats.py).
//
// The apply stays exact. The matvec is linear, so with D_r = sum_j e_rj X_j
// (exact int64, X the 23-bit fixed-point x piece of a warp) each consumer warp
// rebuilds its piece's row sum Y_r = D_r + 2 Y_{r-1} - Y_{r-2} in registers as
// it walks its CTA's rows in order. Y_r is the same integer k2_stream sums
// from the plain codes, so k2_dl returns the same bits as k2_stream.
//
// One unit = (row, 16384-column slab), stored contiguously in processing order
// (CTA, slab, row):
//   [48 B header: u8 start[33], start of chunk c in 512-byte blocks after the
//    header; chunk c has w = start[c+1] - start[c] byte planes]
//   [chunk 0: w_0 planes of 512 B][chunk 1] ...
// A residual is stored as balanced base-256 digits, e = sum_b 256^b s_b with
// every s_b in [-128, 127] (plane b holds s_b); a chunk keeps as many planes
// as its largest residual needs. Codes of at most 3 bytes (|e| < 2^25).
//
// A consumer warp whose x piece holds inf/nan cannot use residuals (the
// reference skips zero mantissas): it reads that row piece's codes from the
// byte planes instead (rare path).
#include "common.cuh"
#include "ptx.cuh"
#include <algorithm>
#include <vector>

namespace invop {

constexpr int DL_SLAB = 16384;       // columns per unit: 32 chunks, one mask word
constexpr int DL_HDR = 48;

// CTA of row r: row ranges [rowlo[b], rowlo[b+1]) chosen at build time so that
// every CTA streams about the same number of bytes
__host__ __device__ inline int dl_cta_of(int64_t r, const int64_t* rowlo, int grid) {
  int lo = 0, hi = grid - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (rowlo[mid] <= r) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// A CTA's rows [lo, lo + n) are split into G segments of consecutive rows
// (the first n % G one row longer), one per consumer group. Residual orders
// restart at every segment start; the units of a slab are interleaved across
// segments: row i of segment g is unit i*G + g of the slab.
struct DlPos {
  int64_t lo, n;       // CTA row range
  int g;               // segment
  int64_t i;           // row index within the segment
};
__host__ __device__ inline DlPos dl_pos(int64_t r, const int64_t* rowlo, int grid, int G) {
  DlPos p;
  const int b = dl_cta_of(r, rowlo, grid);
  p.lo = rowlo[b];
  p.n = rowlo[b + 1] - p.lo;
  const int64_t l = r - p.lo, base = p.n / G, rem = p.n % G;
  if (l < rem * (base + 1)) {
    p.g = (int)(l / (base + 1));
    p.i = l - p.g * (base + 1);
  } else {
    p.g = (int)(rem + (l - rem * (base + 1)) / base);
    p.i = l - rem * (base + 1) - (p.g - rem) * base;
  }
  return p;
}

// code j of a lane's 16 (bytes from up to 3 planes) -> int32
__device__ __forceinline__ void dl_load16(const uint8_t* const* planes, int P, int sgn,
                                          int64_t off, int32_t* v) {
  uint4 w[3];
  for (int b = 0; b < 3; ++b)
    w[b] = b < P ? *reinterpret_cast<const uint4*>(planes[b] + off) : make_uint4(0, 0, 0, 0);
  const int sh = 32 - 8 * P;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    uint32_t u = 0;
#pragma unroll
    for (int b = 0; b < 3; ++b) u |= ((u4get(w[b], q >> 2) >> (8 * (q & 3))) & 0xffu) << (8 * b);
    v[q] = sgn ? ((int32_t)(u << sh) >> sh) : (int32_t)u;
  }
}

// balanced base-256 digit b of e
__host__ __device__ inline int32_t dl_digit(int32_t e, int b) {
  for (int i = 0; i < b; ++i) {
    const int32_t d = ((e + 128) & 255) - 128;
    e = (e - d) >> 8;
  }
  return ((e + 128) & 255) - 128;
}

// number of balanced digits of e (>= 1)
__device__ __forceinline__ uint32_t dl_width(int32_t e) {
  uint32_t w = 1;
  for (;;) {
    const int32_t d = ((e + 128) & 255) - 128;
    e = (e - d) >> 8;
    if (e == 0) return w;
    ++w;
  }
}

struct DlBuild {
  const uint8_t* planes[3];
  int P, sgn;
  int64_t rows, n, ld;
  int nch, nslabs, grid, groups;
  const int64_t* rowlo;       // [grid + 1] CTA row ranges
  int cd;                     // store column differences of the residuals within each chunk
};

// Column difference inside a 512-column chunk (one warp, 16 columns per lane):
// f_j = e_j - e_{j-1}, f = e at the chunk's first column. The apply multiplies
// f by the suffix sums of X within the chunk (sum_j e_j X_j = sum_i f_i S_i,
// S_i = sum_{j >= i} X_j), so the change costs nothing per row; the residuals
// of neighbouring columns are close, so f needs fewer bytes (config 4: 1.56 ->
// 1.32 B/entry, tools/predictor_study.py).
__device__ __forceinline__ void dl_coldiff16(int32_t* e, int lane) {
  int32_t prev = __shfl_up_sync(0xffffffffu, e[15], 1);
  if (lane == 0) prev = 0;
#pragma unroll
  for (int q = 15; q > 0; --q) e[q] -= e[q - 1];
  e[0] -= prev;
}

__device__ __forceinline__ void dl_residual16(const DlBuild& a, int64_t r, int c, int lane,
                                              int32_t* e) {
  const DlPos ps = dl_pos(r, a.rowlo, a.grid, a.groups);
  const int order = (int)(ps.i < 2 ? ps.i : 2);
  const int64_t off = r * a.ld + (int64_t)c * 512 + lane * 16;
  dl_load16(a.planes, a.P, a.sgn, off, e);
  if (order >= 1) {
    int32_t v1[16];
    dl_load16(a.planes, a.P, a.sgn, off - a.ld, v1);
    if (order == 2) {
      int32_t v2[16];
      dl_load16(a.planes, a.P, a.sgn, off - 2 * a.ld, v2);
#pragma unroll
      for (int q = 0; q < 16; ++q) e[q] = e[q] - 2 * v1[q] + v2[q];
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) e[q] -= v1[q];
    }
  }
}

// one warp per (row, chunk): residual byte width of the chunk
__global__ void k_dl_width(DlBuild a, uint8_t* __restrict__ width) {
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= a.rows * a.nch) return;
  const int64_t r = gw / a.nch;
  const int c = (int)(gw - r * a.nch);
  int32_t e[16];
  dl_residual16(a, r, c, lane, e);
  if (a.cd) dl_coldiff16(e, lane);
  uint32_t w = 1;
#pragma unroll
  for (int q = 0; q < 16; ++q) w = max(w, dl_width(e[q]));
  w = __reduce_max_sync(0xffffffffu, w);
  if (lane == 0) width[gw] = (uint8_t)w;
}

// unit index of (row r, slab s) in processing order (CTA, slab, segment row,
// segment)
__host__ __device__ inline int64_t dl_unit(int64_t r, int s, const int64_t* rowlo, int nslabs,
                                           int grid, int G) {
  const DlPos p = dl_pos(r, rowlo, grid, G);
  return p.lo * nslabs + (int64_t)s * p.n + p.i * G + p.g;
}

// one thread per (row, slab): header (chunk starts) and byte size of the unit
__global__ void k_dl_units(DlBuild a, const uint8_t* __restrict__ width, uint4* __restrict__ hdrs,
                           int64_t* __restrict__ size, unsigned long long* __restrict__ maxsize) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= a.rows * a.nslabs) return;
  const int64_t r = t / a.nslabs;
  const int s = (int)(t - r * a.nslabs);
  const int c0 = s * 32, cn = min(32, a.nch - c0);
  uint32_t h[12] = {0};
  uint32_t start = 0;
  for (int c = 0; c <= 32; ++c) {
    h[c >> 2] |= start << (8 * (c & 3));
    if (c < cn) start += width[r * a.nch + c0 + c];
  }
  const int64_t u = dl_unit(r, s, a.rowlo, a.nslabs, a.grid, a.groups);
  for (int k = 0; k < 3; ++k) hdrs[3 * u + k] = make_uint4(h[4 * k], h[4 * k + 1], h[4 * k + 2], h[4 * k + 3]);
  const int64_t bytes = DL_HDR + 512 * (int64_t)start;
  size[u] = bytes;
  atomicMax(maxsize, (unsigned long long)bytes);
}

__global__ void k_dl_scan(int64_t units, const int64_t* __restrict__ size,
                          int64_t* __restrict__ off) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int64_t per = (units + T - 1) / T;
  const int64_t a0 = t * per, a1 = min(units, a0 + per);
  int64_t s = 0;
  for (int64_t u = a0; u < a1; ++u) s += size[u];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int i = 0; i < T; ++i) { const int64_t v = part[i]; part[i] = acc; acc += v; }
    off[units] = acc;
  }
  __syncthreads();
  int64_t acc = part[t];
  for (int64_t u = a0; u < a1; ++u) { off[u] = acc; acc += size[u]; }
}

__device__ __forceinline__ uint4 dl_bytes16(const int32_t* e, int b) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) x |= ((uint32_t)dl_digit(e[4 * k + i], b) & 0xffu) << (8 * i);
    w[k] = x;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// one warp per (row, chunk): write the residual bytes (and the unit header)
__global__ void k_dl_write(DlBuild a, const uint4* __restrict__ hdrs,
                           const int64_t* __restrict__ off, uint8_t* __restrict__ data) {
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= a.rows * a.nch) return;
  const int64_t r = gw / a.nch;
  const int c = (int)(gw - r * a.nch);
  const int s = c / 32, cl = c % 32;
  const int64_t u = dl_unit(r, s, a.rowlo, a.nslabs, a.grid, a.groups);
  uint8_t* unit = data + off[u];
  const uint8_t* h = reinterpret_cast<const uint8_t*>(hdrs + 3 * u);
  if (cl == 0 && lane < 3) reinterpret_cast<uint4*>(unit)[lane] = hdrs[3 * u + lane];
  int32_t e[16];
  dl_residual16(a, r, c, lane, e);
  if (a.cd) dl_coldiff16(e, lane);
  const int s0 = h[cl], w = h[cl + 1] - s0;
  for (int b = 0; b < w; ++b)
    *reinterpret_cast<uint4*>(unit + DL_HDR + (int64_t)(s0 + b) * 512 + lane * 16) = dl_bytes16(e, b);
}

struct DlArgs {
  const uint8_t* data;
  const int64_t* uoff;          // [units + 1]
  const uint8_t* planes[3];     // plain codes, for warps whose x piece is not finite
  const int64_t* rowlo;         // [grid + 1] CTA row ranges
  int P, sgn;
  int64_t rows, n, ld;
  int nslabs;
  double scale;
  const void* x;                // fp32, or fp64 when F64IO (rounded to fp32 on load)
  void* y;                      // fp32, or fp64 when F64IO (the fp32 result widened)
  int ring_bytes;               // variable-size unit ring (FIFO) in shared memory
};

#ifndef DL_NS_OVERRIDE
constexpr int DL_NS = 16;        // units in flight at most (barrier pairs)
#else
constexpr int DL_NS = DL_NS_OVERRIDE;
#endif

__device__ __forceinline__ uint4 dl_lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t dl_lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// plane b of a lane's 16 residual digits times the ND digit words of X: the
// (b, d) partial lands in S[b + d] (weight 256^(b+d)). Exact in int32: one
// DP4A adds at most 4 * 128 * 128 = 2^16.
template <int B, int ND>
__device__ __forceinline__ void dl_plane(const uint4& cw, const uint32_t (*xd)[4], int32_t* S) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int d = 0; d < ND; ++d) S[B + d] = dp4a_ss(u4get(cw, k), xd[d][k], S[B + d]);
}

// planes 1.. of one chunk (width w >= 2), warp-uniform branches
template <int ND>
__device__ __forceinline__ void dl_upper(uint32_t pa, uint32_t w, const uint32_t (*xd)[4], int32_t* S) {
  if (w >= 2) {
    dl_plane<1, ND>(dl_lds128(pa + 512), xd, S);
    if (w >= 3) {
      dl_plane<2, ND>(dl_lds128(pa + 1024), xd, S);
      if (w >= 4) dl_plane<3, ND>(dl_lds128(pa + 1536), xd, S);
    }
  }
}

// exact warp sum of the weight classes. ND = 3: |e| < 2^25, |X| <= 2^22, 16
// codes per lane -> |acc| < 2^54, two 27-bit halves. ND = 4 (column
// differences against suffix sums): |f| < 2^26, |S| < 2^30 ->
// |acc| < 2^60, three parts of 26 + 26 + the rest
template <int ND>
__device__ __forceinline__ long long dl_warp_sum(const int32_t* S) {
  long long acc = (long long)S[0] + ((long long)S[1] << 8) + ((long long)S[2] << 16) +
                  ((long long)S[3] << 24) + ((long long)S[4] << 32) + ((long long)S[5] << 40);
  if (ND == 3) {
    const uint32_t lo = __reduce_add_sync(0xffffffffu, (uint32_t)acc & 0x7FFFFFFu);
    const int32_t hi = __reduce_add_sync(0xffffffffu, (int32_t)(acc >> 27));
    return ((long long)hi << 27) + (long long)lo;
  }
  acc += (long long)S[6] << 48;
  const uint32_t lo = __reduce_add_sync(0xffffffffu, (uint32_t)acc & 0x3FFFFFFu);
  const uint32_t mid = __reduce_add_sync(0xffffffffu, (uint32_t)(acc >> 26) & 0x3FFFFFFu);
  const int32_t hi = __reduce_add_sync(0xffffffffu, (int32_t)(acc >> 52));
  return ((long long)hi << 52) + ((long long)mid << 26) + (long long)lo;
}

__device__ __forceinline__ void dl_slot(double* sp, bool first, long long Y, double inv2e, int lane) {
  const double v = (double)Y * inv2e;
  if (lane == 0) *sp = first ? v : (*sp + v);
}

template <bool F64IO>
__device__ __forceinline__ float dl_x(const DlArgs& a, int64_t j) {
  return F64IO ? (float)static_cast<const double*>(a.x)[j] : static_cast<const float*>(a.x)[j];
}

// the rows of one consumer iteration: headers of all (row, chunk), then the
// plane-0 words, then the DP4As of all rows (independent chains); upper planes
// last (warp-uniform branches on the chunk widths)
template <int SW, int ROWS, int WPG, int ND>
__device__ __forceinline__ void dl_rows_phased(const uint32_t* sb, int q, uint32_t stepv,
                                               const uint32_t (*xd)[ND][4], int lane,
                                               int32_t (*Sa)[7]) {
  uint32_t h[ROWS][SW], w[ROWS][SW];
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int t = 0; t < SW; ++t) {
      const int c = q + t * WPG;
      h[r][t] = dl_lds_u8(sb[r] + c);
      w[r][t] = dl_lds_u8(sb[r] + c + 1) - h[r][t];
    }
  uint4 cw[ROWS][SW];
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int t = 0; t < SW; ++t) {
      h[r][t] = sb[r] + DL_HDR + h[r][t] * 512 + lane * 16;      // chunk address
      cw[r][t] = ((stepv >> t) & 1u) ? dl_lds128(h[r][t]) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int k = 0; k < 7; ++k) Sa[r][k] = 0;
#pragma unroll
  for (int t = 0; t < SW; ++t)
#pragma unroll
    for (int r = 0; r < ROWS; ++r) dl_plane<0, ND>(cw[r][t], xd[t], Sa[r]);
#pragma unroll
  for (int t = 0; t < SW; ++t) {
    if (!((stepv >> t) & 1u)) continue;                      // warp-uniform
#pragma unroll
    for (int r = 0; r < ROWS; ++r) dl_upper<ND>(h[r][t], w[r][t], xd[t], Sa[r]);
  }
}

// chunk by chunk (fewer live registers for many chunks per warp)
template <int SW, int ROWS, int WPG, int ND>
__device__ __forceinline__ void dl_rows_lazy(const uint32_t* sb, int q, uint32_t stepv,
                                             const uint32_t (*xd)[ND][4], int lane,
                                             int32_t (*Sa)[7]) {
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int k = 0; k < 7; ++k) Sa[r][k] = 0;
#pragma unroll
  for (int t = 0; t < SW; ++t) {
    if (!((stepv >> t) & 1u)) continue;                      // warp-uniform
    const int c = q + t * WPG;
    uint32_t pa[ROWS], wd[ROWS];
    uint4 cw[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const uint32_t h = dl_lds_u8(sb[r] + c);
      wd[r] = dl_lds_u8(sb[r] + c + 1) - h;
      pa[r] = sb[r] + DL_HDR + h * 512 + lane * 16;
      cw[r] = dl_lds128(pa[r]);
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) dl_plane<0, ND>(cw[r], xd[t], Sa[r]);
#pragma unroll
    for (int r = 0; r < ROWS; ++r) dl_upper<ND>(pa[r], wd[r], xd[t], Sa[r]);
  }
}

// 16 consecutive x values from column c0 (zero past n): 128-bit loads when the
// run is inside x and aligned
template <bool F64IO>
__device__ __forceinline__ void dl_x16(const DlArgs& a, int64_t c0, bool inside, float* v) {
  if (inside && c0 + 16 <= a.n &&
      ((reinterpret_cast<uintptr_t>(a.x) + (uintptr_t)c0 * (F64IO ? 8 : 4)) & 15) == 0) {
    if (F64IO) {
      const double2* p = reinterpret_cast<const double2*>(static_cast<const double*>(a.x) + c0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double2 d = __ldg(p + k);
        v[2 * k] = (float)d.x;
        v[2 * k + 1] = (float)d.y;
      }
    } else {
      const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(a.x) + c0);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 f = __ldg(p + k);
        v[4 * k] = f.x; v[4 * k + 1] = f.y; v[4 * k + 2] = f.z; v[4 * k + 3] = f.w;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = (inside && c0 + k < a.n) ? dl_x<F64IO>(a, c0 + k) : 0.0f;
  }
}

// CONS consumer warps in G groups. Group g walks segment g of the CTA's rows
// (ROWS rows per iteration); warp q of a group owns chunks q + t*(CONS/G) of
// every slab, its x piece held in registers as balanced digits.
template <int CONS, int G, int ROWS, bool F64IO, bool CD = false>
__global__ void __launch_bounds__((CONS + 1) * 32, 1) k2_dl(DlArgs a) {
  constexpr int ND = CD ? 4 : 3;        // digit planes of the x-side operand
  constexpr int WPG = CONS / G;
  constexpr int SW = DL_SLAB / (WPG * 512);
  extern __shared__ __align__(128) unsigned char smem[];
  // [ring][full[NS], empty[NS]][unit pos[NS], alloc[NS]][slot: nrows x WPG doubles][unit offsets]
  constexpr int S = DL_NS;
  const uint32_t R = (uint32_t)a.ring_bytes;
  unsigned char* ring = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + R);
  uint32_t* s_pos = reinterpret_cast<uint32_t*>(bars + 2 * S);
  double* slot = reinterpret_cast<double*>(s_pos + 2 * S);
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
  // the next apply in the stream (launched as a programmatic dependent) may
  // take SMs as soon as this grid's CTAs retire: its producers start
  // streaming the operator while this grid's slowest CTAs finish; its
  // consumers wait for this grid before reading x (which may be this grid's
  // y) and before writing y
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row_lo = a.rowlo[blockIdx.x];
  const int64_t row_hi = a.rowlo[blockIdx.x + 1];
  const int64_t nrows = row_hi - row_lo;
  const int64_t units = nrows * a.nslabs;
  const int64_t ubase = row_lo * a.nslabs;
  int64_t* s_off = reinterpret_cast<int64_t*>(slot + nrows * WPG);
  for (int64_t i = threadIdx.x; i <= units; i += blockDim.x) s_off[i] = a.uoff[ubase + i];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(bar_s + 8 * i, 1);
      mbar_init(bar_s + 8 * (S + i), WPG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CONS) {
    if (lane == 0) {
      // FIFO of variable-size units: a unit goes at the ring head (or at 0 when
      // it would run past the end); the oldest units are retired (all warps of
      // their group arrived on the empty barrier) until it fits and a slot is free
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      uint32_t* s_alloc = s_pos + S;
      uint32_t head = 0, used = 0;
      int oldest = 0;
      for (int u = 0; u < (int)units; ++u) {
        const uint32_t bytes = (uint32_t)(s_off[u + 1] - s_off[u]);
        uint32_t pos, gap;
        for (;;) {
          pos = head;
          gap = 0;
          if (head + bytes > R) { gap = R - head; pos = 0; }
          if (used + gap + bytes <= R && u - oldest < S) break;
          const int so = oldest % S;
          mbar_wait(bar_s + 8 * (S + so), (uint32_t)(oldest / S) & 1u);
          used -= s_alloc[so];
          ++oldest;
          if (used == 0) head = 0;
        }
        const int sl = u % S;
        s_pos[sl] = pos;
        s_alloc[sl] = gap + bytes;
        used += gap + bytes;
        head = pos + bytes;
        mbar_expect_tx(bar_s + 8 * sl, bytes);
        bulk_g2s(ring_s + pos, a.data + s_off[u], bytes, bar_s + 8 * sl, policy);
      }
    }
  } else {
    const int g = warp / WPG, q = warp - g * WPG;
    const int64_t sbase = nrows / G, srem = nrows % G;
    const int segn = (int)(sbase + (g < srem ? 1 : 0));
    const int seglo = (int)(g * sbase + (g < srem ? g : srem));
    // balanced base-256 digits of the fixed-point x piece (CD: of its suffix
    // sums within each chunk)
    uint32_t xd[SW][ND][4];
    uint32_t stepv = 0;             // bit t: chunk t of this warp lies inside the operator
    for (int slab = 0; slab < a.nslabs; ++slab) {
      stepv = 0;
      // x may come from the preceding grid (programmatic dependent launch of
      // the host entry: that grid pulls x over PCIe while the producer
      // already streams the operator); a no-op for ordinary launches
      // x may be the preceding grid's output (chained applies): wait for
      // that grid before reading it (the producer has been streaming)
      if (slab == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
      // x piece of this warp -> 23-bit fixed point (warp-wide exponent):
      // one pass for max|x| and finiteness, one for the digits (SW > 2; the
      // values stay in registers for SW <= 2)
      bool masked;
      double inv2e;
      {
        constexpr int KEEP = SW <= 2 ? SW : 1;
        float xk[KEEP][16];
        bool finite = true;
        float mx = 0.0f;
#pragma unroll
        for (int t = 0; t < SW; ++t) {
          const int64_t col = (int64_t)slab * DL_SLAB + (int64_t)(q + t * WPG) * 512;
          if (col < a.n) stepv |= 1u << t;
          float* v = xk[SW <= 2 ? t : 0];
          dl_x16<F64IO>(a, col + lane * 16, col < a.n, v);
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            finite = finite && isfinite(v[k]);
            mx = fmaxf(mx, fabsf(v[k]));
          }
        }
        masked = __any_sync(0xffffffffu, !finite);
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        int e = 0;
        if (mx > 0.0f && !masked) {
          int ex;
          frexpf(mx, &ex);
          // |X| <= 2^22; CD: |X| <= 2^21 so that the 512 suffix sums stay
          // below 2^30 (four balanced digits)
          e = (CD ? 21 : 22) - ex;
        }
        inv2e = ldexp(1.0, -e);
#pragma unroll
        for (int t = 0; t < SW; ++t) {
          const int64_t c0 = (int64_t)slab * DL_SLAB + (int64_t)(q + t * WPG) * 512 + lane * 16;
          float* v = xk[SW <= 2 ? t : 0];
          if (SW > 2) dl_x16<F64IO>(a, c0, (stepv >> t) & 1u, v);
          if (CD) {
            // S_i = sum of X over columns >= i of the chunk: lane-local suffix,
            // then the totals of the lanes to the right
            int32_t sfx[16];
#pragma unroll
            for (int k = 15; k >= 0; --k) {
              const int32_t X = masked ? 0 : __float2int_rn(ldexpf(v[k], e));
              sfx[k] = k == 15 ? X : X + sfx[k + 1];
            }
            int32_t inc = sfx[0];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int32_t u = __shfl_down_sync(0xffffffffu, inc, o);
              if (lane + o < 32) inc += u;
            }
            const int32_t right = inc - sfx[0];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              int32_t X[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) X[i] = sfx[4 * k + i] + right;
              uint32_t dw[4];
              x_digits4w(X, dw);
#pragma unroll
              for (int d = 0; d < ND; ++d) xd[t][d][k] = dw[d];
            }
          } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            int32_t X[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) X[i] = masked ? 0 : __float2int_rn(ldexpf(v[4 * k + i], e));
            uint32_t dw[3];
            x_digits4(X, dw);
            xd[t][0][k] = dw[0]; xd[t][1][k] = dw[1]; xd[t][2][k] = dw[2];
          }
          }
        }
      }
      long long Y1 = 0, Y2 = 0;
      const uint32_t ub = slab * (uint32_t)nrows + g;
      for (int i = 0; i < segn;) {
        // ROWS rows per iteration (their loads, DP4As and warp sums interleave)
        const int nr = masked ? 1 : min(ROWS, segn - i);
        uint32_t st[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          const uint32_t u = ub + (i + r) * G;
          st[r] = u % S;
          if (r < nr) mbar_wait(bar_s + 8 * st[r], (u / S) & 1u);
        }
        const uint32_t stA = st[0];
        const int lr = seglo + i;
        if (!masked) {
          uint32_t sb[ROWS];
#pragma unroll
          for (int r = 0; r < ROWS; ++r) sb[r] = ring_s + s_pos[r < nr ? st[r] : st[0]];
          int32_t Sa[ROWS][7];
          if (G == 1) dl_rows_phased<SW, ROWS, WPG, ND>(sb, q, stepv, xd, lane, Sa);
          else dl_rows_lazy<SW, ROWS, WPG, ND>(sb, q, stepv, xd, lane, Sa);
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int r = 0; r < ROWS; ++r)
              if (r < nr) mbar_arrive(bar_s + 8 * (S + st[r]));
          }
#pragma unroll
          for (int r = 0; r < ROWS; ++r) {
            if (r < nr) {
              const int ir = i + r;
              const long long Y = dl_warp_sum<ND>(Sa[r]) + (ir >= 2 ? 2 * Y1 - Y2 : (ir == 1 ? Y1 : 0));
              Y2 = Y1;
              Y1 = Y;
              dl_slot(&slot[(lr + r) * WPG + q], slab == 0, Y, inv2e, lane);
            }
          }
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_s + 8 * (S + stA));
          // inf/nan in this warp's x: plain codes from the byte planes, the
          // reference's zero skip, fp32 accumulation (as k2_stream)
          float acc = 0.0f;
          const int64_t r = row_lo + lr;
          for (int t = 0; t < SW; ++t) {
            if (!((stepv >> t) & 1u)) continue;
            const int64_t c0 = (int64_t)slab * DL_SLAB + (int64_t)(q + t * WPG) * 512 + lane * 16;
            int32_t v[16];
            dl_load16(a.planes, a.P, a.sgn, r * a.ld + c0, v);
            for (int k = 0; k < 16; ++k) {
              if (v[k] == 0 || c0 + k >= a.n) continue;
              acc = fmaf((float)v[k], dl_x<F64IO>(a, c0 + k), acc);
            }
          }
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (lane == 0) {
            double* sp = &slot[lr * WPG + q];
            *sp = (slab == 0) ? (double)acc : (*sp + (double)acc);
          }
        }
        i += nr;
      }
    }
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");   // the preceding grid's y is done
  for (int64_t r = threadIdx.x; r < nrows; r += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < WPG; ++c) s += slot[r * WPG + c];
    const float yv = (float)(s * a.scale);
    if (F64IO) static_cast<double*>(a.y)[row_lo + r] = (double)yv;
    else static_cast<float*>(a.y)[row_lo + r] = yv;
  }
}

static bool layout_flag_dl(const char* env, bool dflt) {
  const char* v = getenv(env);
  if (!v || !*v) return dflt;
  return *v != '0';
}

// every apply is launched as a programmatic dependent of the preceding grid
// (overlaps the previous apply's tail); INVOP_DL_PDL=0 disables
static bool dl_pdl_env() {
  const char* v = getenv("INVOP_DL_PDL");
  return !(v && *v == '0');
}

static int dl_consumers() {
  const char* v = getenv("INVOP_DL_CONS");
  return v && atoi(v) == 8 ? 8 : 16;
}

// consumer groups: one for short CTA row ranges (config 4: 111 rows, where the
// per-CTA start-up dominates), two for long ones (config 5: 443 rows, 4 slabs)
static int dl_groups_for(int64_t rows_per_cta) {
  if (const char* v = getenv("INVOP_DL_GROUPS")) return atoi(v) == 2 ? 2 : 1;
  return rows_per_cta >= 256 ? 2 : 1;
}

// shared memory besides the ring: slot + unit offsets of the largest CTA
static size_t dl_side_bytes(const invop_plan* p, int cons) {
  const int64_t rpc = p->dl_maxrows;
  return (size_t)rpc * (cons / p->dl_groups) * 8 + (size_t)(rpc * p->dl_nslabs + 1) * 8 + 64 +
         DL_NS * 24;
}

// units that must fit in the ring at once (see the producer): G == 1: the two
// units of a consumer iteration plus a wrap gap; G groups: 2G
static int dl_ring_units(int G) { return G == 1 ? 3 : 2 * G; }

int dl_build(invop_plan* p, cudaStream_t s) {
  if (p->dl_ready) return p->dl_ready > 0 ? INVOP_OK : INVOP_E_UNSUPPORTED;
  if (p->P > 3 || p->rows == 0 || p->ld % 512) {
    p->dl_ready = -1;
    return INVOP_E_UNSUPPORTED;
  }
  DlBuild a;
  for (int b = 0; b < 3; ++b) a.planes[b] = p->planes[b < p->P ? b : 0];
  a.P = p->P;
  a.sgn = p->is_signed;
  a.rows = p->rows; a.n = p->n; a.ld = p->ld;
  a.nch = (int)(p->ld / 512);
  a.nslabs = (int)cdiv(a.nch, 32);
  a.grid = (int)std::min<int64_t>(num_sms(), p->rows);
  a.groups = dl_groups_for(cdiv(p->rows, a.grid));
  if (dl_consumers() % a.groups) a.groups = 1;
  p->dl_grid = a.grid;
  p->dl_groups = a.groups;
  p->dl_nslabs = a.nslabs;
  const int64_t units = p->rows * a.nslabs;
  uint8_t* width = nullptr;
  uint4* hdrs = nullptr;
  int64_t* size = nullptr;
  unsigned long long* dmax = nullptr;
  INVOP_CUDA(cudaMalloc(&width, (size_t)p->rows * a.nch));
  INVOP_CUDA(cudaMalloc(&hdrs, (size_t)units * 48));
  INVOP_CUDA(cudaMalloc(&size, (size_t)units * 8 + 8));
  dmax = reinterpret_cast<unsigned long long*>(size + units);
  INVOP_CUDA(cudaMalloc(&p->dl_uoff, (size_t)(units + 1) * 8));
  INVOP_CUDA(cudaMemsetAsync(dmax, 0, 8, s));
  const int64_t warps = p->rows * a.nch;
  // CTA row ranges: equal row counts. INVOP_DL_BALANCE=1 re-cuts them so that
  // every CTA gets the same sum over its rows of max(streaming bytes, per-row
  // consumer time in bytes) (rows near the domain boundary have smaller
  // residuals: +8 % bytes max/mean at config 4). Measured at config 4: pure
  // byte balance 10 % slower, the max() model 0.8 % faster; off by default.
  // The widths are recomputed because residual orders restart at every range
  // start.
  std::vector<int64_t> lo(a.grid + 1);
  for (int b = 0; b <= a.grid; ++b) lo[b] = (int64_t)b * p->rows / a.grid;
  if (!p->dl_rowlo) INVOP_CUDA(cudaMalloc(&p->dl_rowlo, (size_t)(a.grid + 1) * 8));
  INVOP_CUDA(cudaMemcpyAsync(p->dl_rowlo, lo.data(), lo.size() * 8, cudaMemcpyHostToDevice, s));
  a.rowlo = p->dl_rowlo;
  a.cd = 0;
  k_dl_width<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(a, width);
  {
    // INVOP_DL_CD=1: column differences inside the chunks (the kernel then
    // multiplies by suffix sums of x). Measured at config 4: 423.9 -> 357.3 MB
    // per apply but 0.0665 -> 0.0697 ms: the x-side operand grows from 3 to 4
    // digit planes (+13 % DP4A) and the kernel turns issue-bound, so it is
    // opt-in. One consumer group only (x digits per chunk live in registers).
    const char* ce = getenv("INVOP_DL_CD");
    const bool cd_ok = a.groups == 1 && dl_consumers() == 16 && !getenv("INVOP_DL_ROWS");
    if (cd_ok && ce && *ce == '1') {
      a.cd = 1;
      k_dl_width<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(a, width);
    }
    p->dl_cd = a.cd;
  }
  if (a.grid > 1 && layout_flag_dl("INVOP_DL_BALANCE", false)) {
    std::vector<uint8_t> w((size_t)p->rows * a.nch);
    INVOP_CUDA(cudaMemcpyAsync(w.data(), width, w.size(), cudaMemcpyDeviceToHost, s));
    INVOP_CUDA(cudaStreamSynchronize(s));
    std::vector<double> pre(p->rows + 1, 0.0);
    // per-row consumer time in bytes streamed meanwhile (~0.63 us per row at
    // ~44 GB/s per SM: ~27 KB per 16384-column slab)
    double rowcost = 27648.0;
    if (const char* v = getenv("INVOP_DL_ROWCOST")) rowcost = atof(v);
    for (int64_t r = 0; r < p->rows; ++r) {
      int64_t planes = 0;
      for (int c = 0; c < a.nch; ++c) planes += w[(size_t)r * a.nch + c];
      // a row costs its streaming time or its consumer time, whichever is
      // longer (the pipeline overlaps the two)
      pre[r + 1] = pre[r] + std::max(rowcost * a.nslabs, 48.0 * a.nslabs + 512.0 * (double)planes);
    }
    for (int b = 1; b < a.grid; ++b) {
      const double target = pre[p->rows] * b / a.grid;
      int64_t r = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
      r = std::max<int64_t>(r, lo[b - 1] + 2);
      r = std::min<int64_t>(r, p->rows - 2 * (a.grid - b));
      lo[b] = r;
    }
    INVOP_CUDA(cudaMemcpyAsync(p->dl_rowlo, lo.data(), lo.size() * 8, cudaMemcpyHostToDevice, s));
    k_dl_width<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(a, width);
  }
  p->dl_maxrows = 0;
  for (int b = 0; b < a.grid; ++b) p->dl_maxrows = std::max<int64_t>(p->dl_maxrows, lo[b + 1] - lo[b]);
  k_dl_units<<<(unsigned)cdiv(units, 256), 256, 0, s>>>(a, width, hdrs, size, dmax);
  k_dl_scan<<<1, 1024, 0, s>>>(units, size, p->dl_uoff);
  int64_t total = 0;
  unsigned long long mx = 0;
  INVOP_CUDA(cudaMemcpyAsync(&total, p->dl_uoff + units, 8, cudaMemcpyDeviceToHost, s));
  INVOP_CUDA(cudaMemcpyAsync(&mx, dmax, 8, cudaMemcpyDeviceToHost, s));
  INVOP_CUDA(cudaStreamSynchronize(s));
  p->dl_bytes = total;
  p->dl_maxunit = (int64_t)mx;
  int rc = INVOP_OK;
  const size_t need = (size_t)dl_ring_units(a.groups) * mx + dl_side_bytes(p, dl_consumers()) + 128;
  if (total >= (int64_t)p->P * p->rows * p->ld || need > 225 * 1024) {
    rc = INVOP_E_UNSUPPORTED;          // no gain over the byte planes / does not fit
  } else {
    INVOP_CUDA(cudaMalloc(&p->dl_data, total));
    k_dl_write<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(a, hdrs, p->dl_uoff, p->dl_data);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_fail(e, "dl build");
  }
  cudaFree(width);
  cudaFree(hdrs);
  cudaFree(size);
  if (rc != INVOP_OK) {
    cudaFree(p->dl_uoff);
    p->dl_uoff = nullptr;
    p->dl_ready = -1;
    return rc;
  }
  p->dl_ready = 1;
  return INVOP_OK;
}

template <int CONS, int G, int ROWS, bool F64IO, bool CD = false>
static cudaError_t dl_launch(const DlArgs& a, int grid, size_t smem, bool pdl, cudaStream_t s) {
  static size_t smem_set = 0;            // opt-in once per instantiation and size
  auto kern = k2_dl<CONS, G, ROWS, F64IO, CD>;
  if (smem_set < smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3((CONS + 1) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

int apply_dl_launch(invop_plan* p, const void* x, void* y, bool f64io, cudaStream_t s) {
  DlArgs a;
  a.data = p->dl_data;
  a.uoff = p->dl_uoff;
  a.rowlo = p->dl_rowlo;
  for (int b = 0; b < 3; ++b) a.planes[b] = p->planes[b < p->P ? b : 0];
  a.P = p->P;
  a.sgn = p->is_signed;
  a.rows = p->rows; a.n = p->n; a.ld = p->ld;
  a.nslabs = p->dl_nslabs;
  a.scale = p->scale;
  a.x = x; a.y = y;
  int cons = dl_consumers();
  if (cons % p->dl_groups) cons = 16;
  const size_t side = dl_side_bytes(p, cons);
  int64_t ring = (225 * 1024 - (int64_t)side) / 128 * 128;
  if (const char* v = getenv("INVOP_DL_RING_KB")) ring = std::min<int64_t>(ring, atoi(v) * 1024);
  if (ring < dl_ring_units(p->dl_groups) * p->dl_maxunit)
    return fail(INVOP_E_UNSUPPORTED, "k2_dl: not enough shared memory");
  a.ring_bytes = (int)ring;
  const size_t smem = (size_t)ring + side;
  int rows = 2;
  if (const char* v = getenv("INVOP_DL_ROWS")) rows = atoi(v) == 1 ? 1 : 2;
  const int key = p->dl_cd * 100000 + cons * 1000 + p->dl_groups * 100 + rows * 10 + (f64io ? 1 : 0);
  cudaError_t e = cudaSuccess;
  switch (key) {
    case 116120: e = dl_launch<16, 1, 2, false, true>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 116121: e = dl_launch<16, 1, 2, true, true>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 16120: e = dl_launch<16, 1, 2, false>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 16121: e = dl_launch<16, 1, 2, true>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 16110: e = dl_launch<16, 1, 1, false>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 16111: e = dl_launch<16, 1, 1, true>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 16210: e = dl_launch<16, 2, 1, false>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 16211: e = dl_launch<16, 2, 1, true>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 16220: e = dl_launch<16, 2, 2, false>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 16221: e = dl_launch<16, 2, 2, true>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 8120: e = dl_launch<8, 1, 2, false>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 8121: e = dl_launch<8, 1, 2, true>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 8110: e = dl_launch<8, 1, 1, false>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 8111: e = dl_launch<8, 1, 1, true>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 8210: e = dl_launch<8, 2, 1, false>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 8211: e = dl_launch<8, 2, 1, true>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 8220: e = dl_launch<8, 2, 2, false>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    case 8221: e = dl_launch<8, 2, 2, true>(a, p->dl_grid, smem, dl_pdl_env(), s); break;
    default: return fail(INVOP_E_VALUE, "k2_dl: unsupported consumer layout");
  }
  if (e != cudaSuccess) return cuda_fail(e, "k2_dl launch");
  INVOP_LAUNCHED(1);
  INVOP_CHECK_LAUNCH("k2_dl");
  return INVOP_OK;
}

}  // namespace invop
