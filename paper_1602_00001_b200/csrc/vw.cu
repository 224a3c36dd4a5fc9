// Variable-width chunk layout ("VW") and its single-RHS streaming apply.
//
// The byte planes store every code in the plan-wide width P (3 bytes at
// config 4, whose largest mantissa is ~2^19.5). Most of a row does not need
// it: the inverse decays away from the diagonal, so a 512-column chunk of a
// row usually spans a much smaller range. VW stores each (row, chunk) as
//     base = min over the chunk (int32)   and   u = v - base  in w bytes,
// w = bytes(max - min) in {0..4}, w byte planes of 512 bytes each, chunks of
// a row packed back to back (measured 2.32 B/entry at config 4 vs 3).
//
// Apply: sum_j v_j x_j = base * sum_j x_j + sum_j u_j x_j per chunk, so the
// decode is the same PRMT + IMAD.WIDE integer path as k2_stream with one
// extra IMAD per chunk and lane (base times the lane's x sum). A stage is one
// row x 16K-column slab: the slab's chunk metadata (256 B) plus its packed
// payload (variable size), fetched by two bulk copies.
#include "common.cuh"
#include "ptx.cuh"
#include <algorithm>
#include <vector>

namespace invop {

constexpr int VW_CH = 512;                       // columns per chunk
constexpr int VW_CONS = 16;                      // consumer warps
constexpr int VW_SW = 2;                         // chunks per consumer per slab
constexpr int VW_SLABCH = VW_CONS * VW_SW;       // 32 chunks per slab
constexpr int VW_SLAB = VW_SLABCH * VW_CH;       // 16384 columns
constexpr int VW_META = VW_SLABCH * 8;           // 256 B of metadata per stage

struct VwPlanes {
  const uint8_t* p[INVOP_MAX_PLANES];
};

__device__ __forceinline__ int64_t vw_load_code(const VwPlanes& pl, int P, int is_signed,
                                                int64_t off) {
  uint64_t u = 0;
  for (int b = 0; b < P; ++b) u |= (uint64_t)pl.p[b][off] << (8 * b);
  if (is_signed && P < 8) {
    const int sh = 64 - 8 * P;
    return (int64_t)(u << sh) >> sh;
  }
  return (int64_t)u;
}

// one warp per (row, chunk): base = min, width of max - min
__global__ void k_vw_stats(VwPlanes pl, int P, int is_signed, int64_t rows, int64_t ld,
                           int nch, int nchp, int2* __restrict__ meta) {
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= rows * nch) return;
  const int64_t r = gw / nch;
  const int c = (int)(gw - r * nch);
  int64_t mn = INT64_MAX, mx = INT64_MIN;
  const int64_t base_off = r * ld + (int64_t)c * VW_CH + lane * 16;
  for (int q = 0; q < 16; ++q) {
    const int64_t v = vw_load_code(pl, P, is_signed, base_off + q);
    mn = min(mn, v);
    mx = max(mx, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, (int64_t)__shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    const uint64_t range = (uint64_t)(mx - mn);
    const int w = range == 0 ? 0 : range < 256 ? 1 : range < 65536 ? 2 : range < (1ull << 24) ? 3 : 4;
    meta[r * nchp + c] = make_int2((int)mn, w);
  }
}

// per row: chunk offsets (in 512 B units) and the row's payload size
__global__ void k_vw_rowscan(int64_t rows, int nch, int nchp, int2* __restrict__ meta,
                             int64_t* __restrict__ rowsize, uint32_t* __restrict__ slaboff,
                             int nslabs) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  uint32_t off = 0;
  for (int c = 0; c < nch; ++c) {
    if (c % VW_SLABCH == 0) slaboff[r * (nslabs + 1) + c / VW_SLABCH] = off;
    int2 m = meta[r * nchp + c];
    const int w = m.y & 7;
    m.y = (int)((off << 3) | w);
    meta[r * nchp + c] = m;
    off += w;
  }
  for (int c = nch; c < nchp; ++c) meta[r * nchp + c] = make_int2(0, (int)(off << 3));
  slaboff[r * (nslabs + 1) + nslabs] = off;
  rowsize[r] = off;
}

// exclusive scan of row sizes (single block): rowptr[r] in 512 B units
__global__ void k_vw_rowptr(int64_t rows, const int64_t* __restrict__ rowsize,
                            int64_t* __restrict__ rowptr) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int64_t per = (rows + T - 1) / T;
  const int64_t r0 = t * per, r1 = min(rows, r0 + per);
  int64_t s = 0;
  for (int64_t r = r0; r < r1; ++r) s += rowsize[r];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int i = 0; i < T; ++i) { int64_t v = part[i]; part[i] = acc; acc += v; }
    rowptr[rows] = acc;
  }
  __syncthreads();
  int64_t acc = part[t];
  for (int64_t r = r0; r < r1; ++r) { rowptr[r] = acc; acc += rowsize[r]; }
}

// one warp per (row, chunk): u = v - base into w planes of 512 B
__global__ void k_vw_write(VwPlanes pl, int P, int is_signed, int64_t rows, int64_t ld, int nch,
                           int nchp, const int2* __restrict__ meta,
                           const int64_t* __restrict__ rowptr, uint8_t* __restrict__ data) {
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= rows * nch) return;
  const int64_t r = gw / nch;
  const int c = (int)(gw - r * nch);
  const int2 m = meta[r * nchp + c];
  const int w = m.y & 7;
  if (w == 0) return;
  const int64_t dst = (rowptr[r] + ((uint32_t)m.y >> 3)) * VW_CH + lane * 16;
  const int64_t src = r * ld + (int64_t)c * VW_CH + lane * 16;
  uint8_t buf[4][16];
  for (int q = 0; q < 16; ++q) {
    const uint32_t u = (uint32_t)(vw_load_code(pl, P, is_signed, src + q) - (int64_t)m.x);
    for (int b = 0; b < 4; ++b) buf[b][q] = (uint8_t)(u >> (8 * b));
  }
  for (int b = 0; b < w; ++b)
    *reinterpret_cast<uint4*>(data + dst + b * VW_CH) = *reinterpret_cast<const uint4*>(buf[b]);
}

// ------------------------------------------------------------------ apply
struct VwArgs {
  const uint8_t* data;
  const int2* meta;
  const int64_t* rowptr;     // [rows+1], 512 B units
  const uint32_t* slaboff;   // [rows][nslabs+1] chunk-payload offsets of each slab
  int64_t rows, n;
  int nch, nchp;
  double scale;
  const float* x;
  float* y;
  int nslabs;
  int stages;
  int stage_bytes;           // VW_META + wmax * VW_SLAB
  int xbits;                 // fixed-point bits of x (overflow-safe int64 sums)
};

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(addr));
  return r;
}

template <int W>
__device__ __forceinline__ long long vw_chunk_dot(uint32_t cp, const int32_t* X) {
  long long acc = 0, acc2 = 0;
  uint4 cw[W > 0 ? W : 1];
#pragma unroll
  for (int b = 0; b < W; ++b) cw[b] = lds128(cp + b * VW_CH);
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t wds[4];
#pragma unroll
    for (int b = 0; b < W; ++b) wds[b] = u4get(cw[b], w);
    if (W == 4) {
      // unsigned 32-bit offsets: 64-bit products
      const uint32_t t01 = prmt(wds[0], wds[1], 0x5140), t23 = prmt(wds[0], wds[1], 0x7362);
      const uint32_t h01 = prmt(wds[2], wds[3], 0x5140), h23 = prmt(wds[2], wds[3], 0x7362);
      const uint32_t u0 = prmt(t01, h01, 0x5410), u1 = prmt(t01, h01, 0x7632);
      const uint32_t u2 = prmt(t23, h23, 0x5410), u3 = prmt(t23, h23, 0x7632);
      acc += (long long)u0 * X[4 * w + 0];
      acc2 += (long long)u1 * X[4 * w + 1];
      acc += (long long)u2 * X[4 * w + 2];
      acc2 += (long long)u3 * X[4 * w + 3];
    } else {
      int32_t uv[4];
      dec_int4<W, false>(wds, uv);
      acc = madw(uv[0], X[4 * w + 0], acc);
      acc2 = madw(uv[1], X[4 * w + 1], acc2);
      acc = madw(uv[2], X[4 * w + 2], acc);
      acc2 = madw(uv[3], X[4 * w + 3], acc2);
    }
  }
  return acc + acc2;
}

__global__ void __launch_bounds__((VW_CONS + 1) * 32, 1) k2_vw(VwArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = a.stages;
  unsigned char* ring = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * a.stage_bytes);
  double* slot = reinterpret_cast<double*>(bars + 2 * S);   // [rows of CTA][VW_CONS]
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int64_t row_lo = (int64_t)blockIdx.x * a.rows / gridDim.x;
  const int64_t row_hi = (int64_t)(blockIdx.x + 1) * a.rows / gridDim.x;
  const int64_t nrows = row_hi - row_lo;
  const int64_t units = nrows * a.nslabs;

  // producer lookups (row start, slab offsets) staged once: no dependent
  // global loads on the per-stage issue path
  int64_t* s_rowptr = reinterpret_cast<int64_t*>(slot + nrows * VW_CONS);
  uint32_t* s_slab = reinterpret_cast<uint32_t*>(s_rowptr + nrows);
  for (int64_t i = threadIdx.x; i < nrows; i += blockDim.x) s_rowptr[i] = a.rowptr[row_lo + i];
  for (int64_t i = threadIdx.x; i < nrows * (a.nslabs + 1); i += blockDim.x)
    s_slab[i] = a.slaboff[row_lo * (a.nslabs + 1) + i];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(bar_s + 8 * i, 1);
      mbar_init(bar_s + 8 * (S + i), VW_CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == VW_CONS) {
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      int st = 0, slab = 0;
      uint32_t ph = 0;
      int64_t lr = 0;
      for (int64_t u = 0; u < units; ++u) {
        if (u >= S) mbar_wait(bar_s + 8 * (S + st), ph ^ 1);
        const int64_t r = row_lo + lr;
        const int c0 = slab * VW_SLABCH;
        const int c1 = min(a.nch, c0 + VW_SLABCH);
        const int2* mrow = a.meta + r * a.nchp;
        const uint32_t o0 = s_slab[lr * (a.nslabs + 1) + slab];
        const uint32_t o1 = s_slab[lr * (a.nslabs + 1) + slab + 1];
        const uint32_t pay = (o1 - o0) * VW_CH;
        const uint32_t mbytes = (uint32_t)(((c1 - c0) + 1) & ~1) * 8;
        const uint32_t sb = ring_s + st * a.stage_bytes;
        mbar_expect_tx(bar_s + 8 * st, mbytes + pay);
        bulk_g2s(sb, mrow + c0, mbytes, bar_s + 8 * st, policy);
        if (pay)
          bulk_g2s(sb + VW_META, a.data + (s_rowptr[lr] + o0) * VW_CH, pay, bar_s + 8 * st, policy);
        if (++st == S) { st = 0; ph ^= 1; }
        if (++lr == nrows) { lr = 0; ++slab; }
      }
    }
  } else {
    const int wc = warp;
    int32_t X[VW_SW][16];
    int32_t Xs[VW_SW];
    bool stepv[VW_SW];
    bool masked = false;
    double inv2e = 1.0;
    int cur_slab = -1;
    int st = 0, slab = 0;
    uint32_t ph = 0;
    int64_t lr = 0;
    for (int64_t u = 0; u < units; ++u) {
      if (slab != cur_slab) {
        cur_slab = slab;
        bool finite = true;
        float mx = 0.0f;
#pragma unroll
        for (int t = 0; t < VW_SW; ++t) {
          const int64_t col = (int64_t)slab * VW_SLAB + (int64_t)(wc + t * VW_CONS) * VW_CH;
          stepv[t] = col < a.n;
          const int64_t c0 = col + lane * 16;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float v = (stepv[t] && c0 + q < a.n) ? a.x[c0 + q] : 0.0f;
            finite = finite && isfinite(v);
            mx = fmaxf(mx, fabsf(v));
          }
        }
        masked = __any_sync(0xffffffffu, !finite);
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        int e = 0;
        if (mx > 0.0f && !masked) {
          int ex;
          frexpf(mx, &ex);
          e = a.xbits - ex;
        }
        inv2e = ldexp(1.0, -e);
#pragma unroll
        for (int t = 0; t < VW_SW; ++t) {
          const int64_t c0 = (int64_t)slab * VW_SLAB + (int64_t)(wc + t * VW_CONS) * VW_CH + lane * 16;
          int32_t s = 0;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float v = (stepv[t] && c0 + q < a.n) ? a.x[c0 + q] : 0.0f;
            X[t][q] = masked ? 0 : __float2int_rn(ldexpf(v, e));
            s += X[t][q];
          }
          Xs[t] = s;
        }
      }
      mbar_wait(bar_s + 8 * st, ph);
      const unsigned char* sb = ring + (size_t)st * a.stage_bytes;
      const uint32_t sb_s = ring_s + st * a.stage_bytes;
      const int2* sm = reinterpret_cast<const int2*>(sb);
      const uint32_t o0 = (uint32_t)sm[0].y >> 3;
      double part = 0.0;
      if (!masked) {
        long long acc = 0;
#pragma unroll
        for (int t = 0; t < VW_SW; ++t) {
          if (!stepv[t]) continue;                 // warp-uniform
          const int2 m = sm[wc + t * VW_CONS];
          const int w = m.y & 7;
          const uint32_t cp = sb_s + VW_META + (((uint32_t)m.y >> 3) - o0) * VW_CH + lane * 16;
          acc += (long long)m.x * Xs[t];
          switch (w) {                             // warp-uniform
            case 1: acc += vw_chunk_dot<1>(cp, X[t]); break;
            case 2: acc += vw_chunk_dot<2>(cp, X[t]); break;
            case 3: acc += vw_chunk_dot<3>(cp, X[t]); break;
            case 4: acc += vw_chunk_dot<4>(cp, X[t]); break;
            default: break;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_s + 8 * (S + st));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        part = (double)acc * inv2e;
      } else {
        // inf/nan in this warp's x: fp32 with the reference's zero skip
        float acc = 0.0f;
#pragma unroll
        for (int t = 0; t < VW_SW; ++t) {
          if (!stepv[t]) continue;
          const int2 m = sm[wc + t * VW_CONS];
          const int w = m.y & 7;
          const unsigned char* cp = sb + VW_META + (((uint32_t)m.y >> 3) - o0) * VW_CH;
          const int64_t gc = (int64_t)slab * VW_SLAB + (int64_t)(wc + t * VW_CONS) * VW_CH + lane * 16;
          for (int q = 0; q < 16; ++q) {
            uint32_t u = 0;
            for (int b = 0; b < w; ++b) u |= (uint32_t)cp[b * VW_CH + lane * 16 + q] << (8 * b);
            const long long v = (long long)m.x + (long long)u;
            if (v == 0) continue;
            const float xv = gc + q < a.n ? a.x[gc + q] : 0.0f;
            acc = fmaf((float)v, xv, acc);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_s + 8 * (S + st));
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        part = (double)acc;
      }
      if (lane == 0) {
        double* sp = &slot[lr * VW_CONS + wc];
        *sp = (slab == 0) ? part : (*sp + part);
      }
      if (++st == S) { st = 0; ph ^= 1; }
      if (++lr == nrows) { lr = 0; ++slab; }
    }
  }
  __syncthreads();
  for (int64_t r = threadIdx.x; r < nrows; r += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < VW_CONS; ++c) s += slot[r * VW_CONS + c];
    a.y[row_lo + r] = (float)(s * a.scale);
  }
}

// ------------------------------------------------------------------ host
int vw_build(invop_plan* p, cudaStream_t s) {
  if (p->vw_ready) return p->vw_ready > 0 ? INVOP_OK : INVOP_E_UNSUPPORTED;
  if (p->min_val < INT32_MIN || p->max_val > INT32_MAX || p->rows == 0) {
    p->vw_ready = -1;
    return INVOP_E_UNSUPPORTED;
  }
  const int nch = (int)(p->ld / VW_CH);
  const int nchp = (nch + 1) & ~1;
  VwPlanes pl;
  for (int b = 0; b < INVOP_MAX_PLANES; ++b) pl.p[b] = p->planes[b];
  INVOP_CUDA(cudaMalloc(&p->vw_meta, (size_t)p->rows * nchp * sizeof(int2)));
  INVOP_CUDA(cudaMalloc(&p->vw_rowptr, (size_t)(p->rows + 1) * sizeof(int64_t)));
  int64_t* rowsize = nullptr;
  INVOP_CUDA(cudaMalloc(&rowsize, (size_t)p->rows * sizeof(int64_t)));
  const int nslabs = (nch + VW_SLABCH - 1) / VW_SLABCH;
  INVOP_CUDA(cudaMalloc(&p->vw_slaboff, (size_t)p->rows * (nslabs + 1) * sizeof(uint32_t)));
  const int64_t warps = p->rows * nch;
  k_vw_stats<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(pl, p->P, p->is_signed, p->rows,
                                                             p->ld, nch, nchp, (int2*)p->vw_meta);
  k_vw_rowscan<<<(unsigned)cdiv(p->rows, 256), 256, 0, s>>>(p->rows, nch, nchp,
                                                            (int2*)p->vw_meta, rowsize,
                                                            p->vw_slaboff, nslabs);
  k_vw_rowptr<<<1, 1024, 0, s>>>(p->rows, rowsize, p->vw_rowptr);
  int64_t total = 0;
  INVOP_CUDA(cudaMemcpyAsync(&total, p->vw_rowptr + p->rows, sizeof(int64_t),
                             cudaMemcpyDeviceToHost, s));
  INVOP_CUDA(cudaStreamSynchronize(s));
  cudaFree(rowsize);
  p->vw_bytes = total * VW_CH;
  INVOP_CUDA(cudaMalloc(&p->vw_data, p->vw_bytes > 0 ? p->vw_bytes : 16));
  k_vw_write<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(pl, p->P, p->is_signed, p->rows,
                                                             p->ld, nch, nchp,
                                                             (const int2*)p->vw_meta,
                                                             p->vw_rowptr, p->vw_data);
  INVOP_CHECK_LAUNCH("vw build");
  // the widest chunk (bounds the stage size): bytes of the plan's value range
  const uint64_t range = (uint64_t)(p->max_val - p->min_val);
  p->vw_wmax = range == 0 ? 1 : range < 256 ? 1 : range < 65536 ? 2 : range < (1ull << 24) ? 3 : 4;
  p->vw_ready = 1;
  return INVOP_OK;
}

int apply_vw_launch(invop_plan* p, const float* x, float* y, cudaStream_t s) {
  VwArgs a;
  a.data = p->vw_data;
  a.meta = (const int2*)p->vw_meta;
  a.rowptr = p->vw_rowptr;
  a.slaboff = p->vw_slaboff;
  a.rows = p->rows; a.n = p->n;
  a.nch = (int)(p->ld / VW_CH);
  a.nchp = (a.nch + 1) & ~1;
  a.scale = p->scale;
  a.x = x; a.y = y;
  a.nslabs = (int)cdiv(a.nch, VW_SLABCH);
  a.stage_bytes = VW_META + p->vw_wmax * VW_SLAB;
  // x bits so that |sum_j v_j X_j| stays below 2^61 in int64
  int vb = 1;
  while (vb < 62 && ((int64_t)1 << vb) <= p->max_abs) ++vb;
  int nb = 1;
  while (nb < 40 && ((int64_t)1 << nb) < p->n) ++nb;
  a.xbits = std::max(8, std::min(22, 61 - vb - nb));
  int grid = (int)std::min<int64_t>(num_sms(), p->rows);
  const int64_t rows_per_cta = cdiv(p->rows, grid);
  const size_t slot_bytes = (size_t)rows_per_cta * VW_CONS * sizeof(double) +
                            (size_t)rows_per_cta * 8 + (size_t)rows_per_cta * (a.nslabs + 1) * 4 + 16;
  const size_t budget = 225 * 1024;
  int stages = (int)((budget - slot_bytes - 256) / (a.stage_bytes + 16));
  stages = std::min(stages, 8);
  if (stages < 2) return fail(INVOP_E_UNSUPPORTED, "k2_vw: not enough shared memory");
  a.stages = stages;
  const size_t smem = (size_t)stages * a.stage_bytes + 2 * stages * 8 + slot_bytes;
  cudaFuncSetAttribute(k2_vw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k2_vw<<<grid, (VW_CONS + 1) * 32, smem, s>>>(a);
  INVOP_LAUNCHED(1);
  INVOP_CHECK_LAUNCH("k2_vw");
  return INVOP_OK;
}

}  // namespace invop
