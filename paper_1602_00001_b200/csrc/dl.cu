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

namespace invop {

constexpr int DL_SLAB = 16384;       // columns per unit: 32 chunks, one mask word
constexpr int DL_HDR = 48;

__host__ __device__ inline int dl_cta_of(int64_t r, int64_t rows, int grid) {
  int b = (int)(r * grid / rows);
  while (b + 1 < grid && (int64_t)(b + 1) * rows / grid <= r) ++b;
  while (b > 0 && (int64_t)b * rows / grid > r) --b;
  return b;
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
  int nch, nslabs, grid;
};

__device__ __forceinline__ void dl_residual16(const DlBuild& a, int64_t r, int c, int lane,
                                              int32_t* e) {
  const int b = dl_cta_of(r, a.rows, a.grid);
  const int64_t lo = (int64_t)b * a.rows / a.grid;
  const int order = (int)(r - lo < 2 ? r - lo : 2);
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
  uint32_t w = 1;
#pragma unroll
  for (int q = 0; q < 16; ++q) w = max(w, dl_width(e[q]));
  w = __reduce_max_sync(0xffffffffu, w);
  if (lane == 0) width[gw] = (uint8_t)w;
}

// unit index of (row r, slab s) in processing order (CTA, slab, row)
__host__ __device__ inline int64_t dl_unit(int64_t r, int s, int64_t rows, int nslabs, int grid) {
  const int b = dl_cta_of(r, rows, grid);
  const int64_t lo = (int64_t)b * rows / grid, hi = (int64_t)(b + 1) * rows / grid;
  return lo * nslabs + (int64_t)s * (hi - lo) + (r - lo);
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
  const int64_t u = dl_unit(r, s, a.rows, a.nslabs, a.grid);
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
  const int64_t u = dl_unit(r, s, a.rows, a.nslabs, a.grid);
  uint8_t* unit = data + off[u];
  const uint8_t* h = reinterpret_cast<const uint8_t*>(hdrs + 3 * u);
  if (cl == 0 && lane < 3) reinterpret_cast<uint4*>(unit)[lane] = hdrs[3 * u + lane];
  int32_t e[16];
  dl_residual16(a, r, c, lane, e);
  const int s0 = h[cl], w = h[cl + 1] - s0;
  for (int b = 0; b < w; ++b)
    *reinterpret_cast<uint4*>(unit + DL_HDR + (int64_t)(s0 + b) * 512 + lane * 16) = dl_bytes16(e, b);
}

struct DlArgs {
  const uint8_t* data;
  const int64_t* uoff;          // [units + 1]
  const uint8_t* planes[3];     // plain codes, for warps whose x piece is not finite
  int P, sgn;
  int64_t rows, n, ld;
  int nslabs;
  double scale;
  const void* x;                // fp32, or fp64 when F64IO (rounded to fp32 on load)
  void* y;                      // fp32, or fp64 when F64IO (the fp32 result widened)
  int ring_bytes;               // variable-size unit ring (FIFO) in shared memory
};

constexpr int DL_NS = 8;         // units in flight at most (barrier pairs)

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

// plane b of a lane's 16 residual digits times the 3 digit words of X: the
// (b, d) partial lands in S[b + d] (weight 256^(b+d)). Exact in int32: one
// DP4A adds at most 4 * 128 * 128 = 2^16.
template <int B>
__device__ __forceinline__ void dl_plane(const uint4& cw, const uint32_t (*xd)[4], int32_t* S) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int d = 0; d < 3; ++d) S[B + d] = dp4a_ss(u4get(cw, k), xd[d][k], S[B + d]);
}

template <bool F64IO>
__device__ __forceinline__ float dl_x(const DlArgs& a, int64_t j) {
  return F64IO ? (float)static_cast<const double*>(a.x)[j] : static_cast<const float*>(a.x)[j];
}

template <int CONS, bool F64IO>
__global__ void __launch_bounds__((CONS + 1) * 32, 1) k2_dl(DlArgs a) {
  constexpr int SW = DL_SLAB / (CONS * 512);
  extern __shared__ __align__(128) unsigned char smem[];
  // [ring][full[NS], empty[NS]][unit pos[NS]][slot: nrows x CONS doubles][unit offsets]
  constexpr int S = DL_NS;
  const uint32_t R = (uint32_t)a.ring_bytes;
  unsigned char* ring = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + R);
  uint32_t* s_pos = reinterpret_cast<uint32_t*>(bars + 2 * S);
  double* slot = reinterpret_cast<double*>(s_pos + 2 * S);
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row_lo = (int64_t)blockIdx.x * a.rows / gridDim.x;
  const int64_t row_hi = (int64_t)(blockIdx.x + 1) * a.rows / gridDim.x;
  const int64_t nrows = row_hi - row_lo;
  const int64_t units = nrows * a.nslabs;
  const int64_t ubase = row_lo * a.nslabs;
  int64_t* s_off = reinterpret_cast<int64_t*>(slot + nrows * CONS);
  for (int64_t i = threadIdx.x; i <= units; i += blockDim.x) s_off[i] = a.uoff[ubase + i];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(bar_s + 8 * i, 1);
      mbar_init(bar_s + 8 * (S + i), CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CONS) {
    if (lane == 0) {
      // FIFO of variable-size units: a unit goes at the ring head (or at 0 when
      // it would run past the end); the oldest units are retired (all consumer
      // warps arrived on their empty barrier) until it fits and a slot is free
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
    const int wc = warp;
    uint32_t xd[SW][3][4];          // balanced base-256 digits of the fixed-point x piece
    bool stepv[SW];
    bool masked = false;
    double inv2e = 1.0;
    long long Y1 = 0, Y2 = 0;
    int st = 0, slab = 0;
    uint32_t ph = 0;
    int lr = 0;
    for (int u = 0; u < (int)units;) {
      if (lr == 0) {
        // new slab: x piece of this warp -> 23-bit fixed point (as k2_stream);
        // x is read once (it may live in mapped host memory)
        float xv[SW][16];
        bool finite = true;
        float mx = 0.0f;
#pragma unroll
        for (int t = 0; t < SW; ++t) {
          const int64_t col = (int64_t)slab * DL_SLAB + (int64_t)(wc + t * CONS) * 512;
          stepv[t] = col < a.n;
          const int64_t c0 = col + lane * 16;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            xv[t][q] = (stepv[t] && c0 + q < a.n) ? dl_x<F64IO>(a, c0 + q) : 0.0f;
            finite = finite && isfinite(xv[t][q]);
            mx = fmaxf(mx, fabsf(xv[t][q]));
          }
        }
        masked = __any_sync(0xffffffffu, !finite);
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        int e = 0;
        if (mx > 0.0f && !masked) {
          int ex;
          frexpf(mx, &ex);
          e = 22 - ex;
        }
        inv2e = ldexp(1.0, -e);
#pragma unroll
        for (int t = 0; t < SW; ++t) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            int32_t X[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) X[i] = masked ? 0 : __float2int_rn(ldexpf(xv[t][4 * k + i], e));
            uint32_t dw[3];
            x_digits4(X, dw);
            xd[t][0][k] = dw[0]; xd[t][1][k] = dw[1]; xd[t][2][k] = dw[2];
          }
        }
        Y1 = 0;
        Y2 = 0;
      }
      // two rows per iteration when both are in this slab: their loads, DP4As
      // and warp sums interleave (the per-row chain is latency bound)
      const bool two = !masked && lr + 1 < (int)nrows;
      const int stB = st + 1 == S ? 0 : st + 1;
      const uint32_t phB = st + 1 == S ? ph ^ 1u : ph;
      mbar_wait(bar_s + 8 * st, ph);
      if (two) mbar_wait(bar_s + 8 * stB, phB);
      if (!masked) {
        const uint32_t sbA = ring_s + s_pos[st];
        const uint32_t sbB = ring_s + s_pos[two ? stB : st];
        uint32_t csA[SW], wA[SW], csB[SW], wB[SW];
#pragma unroll
        for (int t = 0; t < SW; ++t) {
          const int c = wc + t * CONS;
          csA[t] = dl_lds_u8(sbA + c);
          wA[t] = dl_lds_u8(sbA + c + 1) - csA[t];
          csB[t] = dl_lds_u8(sbB + c);
          wB[t] = dl_lds_u8(sbB + c + 1) - csB[t];
        }
        uint4 pA[SW], pB[SW];
#pragma unroll
        for (int t = 0; t < SW; ++t) {
          pA[t] = stepv[t] ? dl_lds128(sbA + DL_HDR + csA[t] * 512 + lane * 16) : make_uint4(0, 0, 0, 0);
          pB[t] = stepv[t] ? dl_lds128(sbB + DL_HDR + csB[t] * 512 + lane * 16) : make_uint4(0, 0, 0, 0);
        }
        int32_t SA[6] = {0, 0, 0, 0, 0, 0}, SB[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int t = 0; t < SW; ++t) {
          dl_plane<0>(pA[t], xd[t], SA);
          dl_plane<0>(pB[t], xd[t], SB);
        }
#pragma unroll
        for (int t = 0; t < SW; ++t) {
          if (!stepv[t]) continue;                      // warp-uniform
          const uint32_t pa = sbA + DL_HDR + csA[t] * 512 + lane * 16;
          if (wA[t] >= 2) {
            dl_plane<1>(dl_lds128(pa + 512), xd[t], SA);
            if (wA[t] >= 3) {
              dl_plane<2>(dl_lds128(pa + 1024), xd[t], SA);
              if (wA[t] >= 4) dl_plane<3>(dl_lds128(pa + 1536), xd[t], SA);
            }
          }
          const uint32_t pbb = sbB + DL_HDR + csB[t] * 512 + lane * 16;
          if (wB[t] >= 2) {
            dl_plane<1>(dl_lds128(pbb + 512), xd[t], SB);
            if (wB[t] >= 3) {
              dl_plane<2>(dl_lds128(pbb + 1024), xd[t], SB);
              if (wB[t] >= 4) dl_plane<3>(dl_lds128(pbb + 1536), xd[t], SB);
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(bar_s + 8 * (S + st));
          if (two) mbar_arrive(bar_s + 8 * (S + stB));
        }
        const long long accA = (long long)SA[0] + ((long long)SA[1] << 8) + ((long long)SA[2] << 16) +
                               ((long long)SA[3] << 24) + ((long long)SA[4] << 32) + ((long long)SA[5] << 40);
        const long long accB = (long long)SB[0] + ((long long)SB[1] << 8) + ((long long)SB[2] << 16) +
                               ((long long)SB[3] << 24) + ((long long)SB[4] << 32) + ((long long)SB[5] << 40);
        // exact warp sums: |e| < 2^25, |X| <= 2^22, 32 codes per lane -> |acc| < 2^52
        const uint32_t loA = __reduce_add_sync(0xffffffffu, (uint32_t)accA & 0x7FFFFFFu);
        const int32_t hiA = __reduce_add_sync(0xffffffffu, (int32_t)(accA >> 27));
        const uint32_t loB = __reduce_add_sync(0xffffffffu, (uint32_t)accB & 0x7FFFFFFu);
        const int32_t hiB = __reduce_add_sync(0xffffffffu, (int32_t)(accB >> 27));
        const long long DA = ((long long)hiA << 27) + (long long)loA;
        const long long DB = ((long long)hiB << 27) + (long long)loB;
        const long long YA = DA + (lr >= 2 ? 2 * Y1 - Y2 : (lr == 1 ? Y1 : 0));
        Y2 = Y1;
        Y1 = YA;
        if (lane == 0) {
          double* sp = &slot[lr * CONS + wc];
          *sp = (slab == 0) ? (double)YA * inv2e : (*sp + (double)YA * inv2e);
        }
        if (two) {
          const long long YB = DB + (lr + 1 >= 2 ? 2 * Y1 - Y2 : Y1);
          Y2 = Y1;
          Y1 = YB;
          if (lane == 0) {
            double* sp = &slot[(lr + 1) * CONS + wc];
            *sp = (slab == 0) ? (double)YB * inv2e : (*sp + (double)YB * inv2e);
          }
        }
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_s + 8 * (S + st));
        // inf/nan in this warp's x: plain codes from the byte planes, the
        // reference's zero skip, fp32 accumulation (as k2_stream)
        float acc = 0.0f;
        const int64_t r = row_lo + lr;
        for (int t = 0; t < SW; ++t) {
          if (!stepv[t]) continue;
          const int64_t c0 = (int64_t)slab * DL_SLAB + (int64_t)(wc + t * CONS) * 512 + lane * 16;
          int32_t v[16];
          dl_load16(a.planes, a.P, a.sgn, r * a.ld + c0, v);
          for (int q = 0; q < 16; ++q) {
            if (v[q] == 0 || c0 + q >= a.n) continue;
            acc = fmaf((float)v[q], dl_x<F64IO>(a, c0 + q), acc);
          }
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
          double* sp = &slot[lr * CONS + wc];
          *sp = (slab == 0) ? (double)acc : (*sp + (double)acc);
        }
      }
      if (two) {
        st = stB == S - 1 ? 0 : stB + 1;
        ph = stB == S - 1 ? phB ^ 1u : phB;
        u += 2;
        lr += 2;
      } else {
        if (++st == S) { st = 0; ph ^= 1; }
        u += 1;
        lr += 1;
      }
      if (lr == (int)nrows) { lr = 0; ++slab; }
    }
  }
  __syncthreads();
  for (int64_t r = threadIdx.x; r < nrows; r += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CONS; ++c) s += slot[r * CONS + c];
    const float yv = (float)(s * a.scale);
    if (F64IO) static_cast<double*>(a.y)[row_lo + r] = (double)yv;
    else static_cast<float*>(a.y)[row_lo + r] = yv;
  }
}

static int dl_consumers() {
  const char* v = getenv("INVOP_DL_CONS");
  return v && atoi(v) == 8 ? 8 : 16;
}

static size_t dl_side_bytes(const invop_plan* p, int cons) {
  const int64_t rpc = cdiv(p->rows, p->dl_grid);
  return (size_t)rpc * cons * 8 + (size_t)(rpc * p->dl_nslabs + 1) * 8 + 64;
}

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
  p->dl_grid = a.grid;
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
  k_dl_width<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(a, width);
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
  const size_t need = 3 * (size_t)mx + dl_side_bytes(p, dl_consumers()) + DL_NS * 24 + 128;
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

int apply_dl_launch(invop_plan* p, const void* x, void* y, bool f64io, cudaStream_t s) {
  DlArgs a;
  a.data = p->dl_data;
  a.uoff = p->dl_uoff;
  for (int b = 0; b < 3; ++b) a.planes[b] = p->planes[b < p->P ? b : 0];
  a.P = p->P;
  a.sgn = p->is_signed;
  a.rows = p->rows; a.n = p->n; a.ld = p->ld;
  a.nslabs = p->dl_nslabs;
  a.scale = p->scale;
  a.x = x; a.y = y;
  const int cons = dl_consumers();
  const size_t side = dl_side_bytes(p, cons) + DL_NS * 24;
  int64_t ring = (225 * 1024 - (int64_t)side) / 128 * 128;
  if (const char* v = getenv("INVOP_DL_RING_KB")) ring = std::min<int64_t>(ring, atoi(v) * 1024);
  // consumers take two consecutive units at once: with a ring of >= 3 max
  // units, any two consecutive units fit side by side after a wrap
  if (ring < 3 * p->dl_maxunit) return fail(INVOP_E_UNSUPPORTED, "k2_dl: not enough shared memory");
  a.ring_bytes = (int)ring;
  const size_t smem = (size_t)ring + side;
  auto kern = cons == 8 ? (f64io ? k2_dl<8, true> : k2_dl<8, false>)
                        : (f64io ? k2_dl<16, true> : k2_dl<16, false>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<p->dl_grid, (cons + 1) * 32, smem, s>>>(a);
  INVOP_LAUNCHED(1);
  INVOP_CHECK_LAUNCH("k2_dl");
  return INVOP_OK;
}

}  // namespace invop
