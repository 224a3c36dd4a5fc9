// "Sparse high plane" layout (HL) for 3-byte codes and its apply k2_hl.
//
// With P = 3 (config 4: mantissas up to ~2^19.5) the top byte plane is needed
// only where a value leaves the 16-bit range; at config 4 that is 29 % of the
// 512-column chunks of a row. HL keeps the two low planes of every row and the
// top plane only for those chunks:
//
//   row = [u32 chunk mask, 12 B pad][plane 0: ld B][plane 1: ld B][top plane of
//          each masked chunk: 512 B each, in chunk order]
//
// (2.29 B/entry at config 4 instead of 3). A chunk without its top plane
// decodes as a 16-bit code (two's complement when the plan is signed); with it,
// as the 24-bit code. The apply is k2_stream's structure unchanged — one row per
// stage, one bulk copy per row (the row is contiguous), 8 consumer warps with
// 23-bit fixed-point x in registers and exact int64 row sums — so the decode
// stays two PRMTs per code and the work per warp is nearly uniform.
// Rows up to 16384 columns (one x slab).
#include "common.cuh"
#include "ptx.cuh"
#include <algorithm>

namespace invop {

constexpr int HL_MAXCOLS = 32 * 512;   // 16384: 32 chunks (one mask word)
constexpr int HL_HDR = 16;

// one warp per (row, chunk): does the chunk need its top byte?
__global__ void k_hl_mask(const uint8_t* __restrict__ p0, const uint8_t* __restrict__ p1,
                          const uint8_t* __restrict__ p2, int is_signed, int64_t rows,
                          int64_t ld, int nch, uint32_t* __restrict__ mask) {
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= rows * nch) return;
  const int64_t r = gw / nch;
  const int c = (int)(gw - r * nch);
  const int64_t off = r * ld + (int64_t)c * 512 + lane * 16;
  const uint4 hi = *reinterpret_cast<const uint4*>(p2 + off);
  bool need;
  if (is_signed) {
    // top byte must equal the sign extension of bit 15 (byte 1's msb)
    const uint4 b1 = *reinterpret_cast<const uint4*>(p1 + off);
    const uint32_t h[4] = {hi.x, hi.y, hi.z, hi.w}, m[4] = {b1.x, b1.y, b1.z, b1.w};
    need = false;
    for (int w = 0; w < 4; ++w) need |= h[w] != prmt(m[w], 0, 0xBA98);
  } else {
    need = (hi.x | hi.y | hi.z | hi.w) != 0;
  }
  (void)p0;
  if (__any_sync(0xffffffffu, need) && lane == 0) atomicOr(&mask[r], 1u << c);
}

__global__ void k_hl_rowsize(int64_t rows, int64_t ld, const uint32_t* __restrict__ mask,
                             int64_t* __restrict__ size) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < rows) size[r] = HL_HDR + 2 * ld + (int64_t)__popc(mask[r]) * 512;
}

__global__ void k_hl_scan(int64_t rows, const int64_t* __restrict__ size,
                          int64_t* __restrict__ rowptr) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int64_t per = (rows + T - 1) / T;
  const int64_t a0 = t * per, a1 = min(rows, a0 + per);
  int64_t s = 0;
  for (int64_t r = a0; r < a1; ++r) s += size[r];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int i = 0; i < T; ++i) { const int64_t v = part[i]; part[i] = acc; acc += v; }
    rowptr[rows] = acc;
  }
  __syncthreads();
  int64_t acc = part[t];
  for (int64_t r = a0; r < a1; ++r) { rowptr[r] = acc; acc += size[r]; }
}

// one warp per (row, chunk): copy the low planes, the top plane if masked, the header
__global__ void k_hl_write(const uint8_t* __restrict__ p0, const uint8_t* __restrict__ p1,
                           const uint8_t* __restrict__ p2, int64_t rows, int64_t ld, int nch,
                           const uint32_t* __restrict__ mask, const int64_t* __restrict__ rowptr,
                           uint8_t* __restrict__ data) {
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= rows * nch) return;
  const int64_t r = gw / nch;
  const int c = (int)(gw - r * nch);
  const int64_t src = r * ld + (int64_t)c * 512 + lane * 16;
  uint8_t* row = data + rowptr[r];
  const uint32_t m = mask[r];
  if (c == 0 && lane == 0) *reinterpret_cast<uint4*>(row) = make_uint4(m, 0, 0, 0);
  *reinterpret_cast<uint4*>(row + HL_HDR + (int64_t)c * 512 + lane * 16) =
      *reinterpret_cast<const uint4*>(p0 + src);
  *reinterpret_cast<uint4*>(row + HL_HDR + ld + (int64_t)c * 512 + lane * 16) =
      *reinterpret_cast<const uint4*>(p1 + src);
  if ((m >> c) & 1u) {
    const int pos = __popc(m & ((1u << c) - 1u));
    *reinterpret_cast<uint4*>(row + HL_HDR + 2 * ld + (int64_t)pos * 512 + lane * 16) =
        *reinterpret_cast<const uint4*>(p2 + src);
  }
}

struct HlArgs {
  const uint8_t* data;
  const int64_t* rowptr;
  int64_t rows, n, ld;
  double scale;
  const float* x;
  float* y;
  int stages;
  int stage_bytes;
  uint32_t piece;     // bulk-copy piece size
};

// CONS consumer warps, each holding SW = 32 / CONS chunks of x in registers
template <bool SIGNED, int CONS>
__global__ void __launch_bounds__((CONS + 1) * 32, 1) k2_hl(HlArgs a) {
  constexpr int HL_CONS = CONS, HL_SW = 32 / CONS;
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = a.stages;
  unsigned char* ring = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * a.stage_bytes);
  double* slot = reinterpret_cast<double*>(bars + 2 * S);
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row_lo = (int64_t)blockIdx.x * a.rows / gridDim.x;
  const int64_t row_hi = (int64_t)(blockIdx.x + 1) * a.rows / gridDim.x;
  const int64_t nrows = row_hi - row_lo;
  int64_t* s_rowptr = reinterpret_cast<int64_t*>(slot + nrows * HL_CONS);
  for (int64_t i = threadIdx.x; i <= nrows; i += blockDim.x) s_rowptr[i] = a.rowptr[row_lo + i];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(bar_s + 8 * i, 1);
      mbar_init(bar_s + 8 * (S + i), HL_CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == HL_CONS) {
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      int st = 0;
      uint32_t ph = 0;
      for (int64_t lr = 0; lr < nrows; ++lr) {
        if (lr >= S) mbar_wait(bar_s + 8 * (S + st), ph ^ 1);
        const uint32_t bytes = (uint32_t)(s_rowptr[lr + 1] - s_rowptr[lr]);
        mbar_expect_tx(bar_s + 8 * st, bytes);
        for (uint32_t o = 0; o < bytes; o += a.piece)
          bulk_g2s(ring_s + st * a.stage_bytes + o, a.data + s_rowptr[lr] + o,
                   min(a.piece, bytes - o), bar_s + 8 * st, policy);
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
  } else {
    const int wc = warp;
    int32_t X[HL_SW][16];
    bool stepv[HL_SW];
    bool finite = true;
    float mx = 0.0f;
#pragma unroll
    for (int t = 0; t < HL_SW; ++t) {
      const int64_t col = (int64_t)(wc + t * HL_CONS) * 512;
      stepv[t] = col < a.n;
      const int64_t c0 = col + lane * 16;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float v = (stepv[t] && c0 + q < a.n) ? a.x[c0 + q] : 0.0f;
        finite = finite && isfinite(v);
        mx = fmaxf(mx, fabsf(v));
      }
    }
    const bool masked = __any_sync(0xffffffffu, !finite);
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int e = 0;
    if (mx > 0.0f && !masked) {
      int ex;
      frexpf(mx, &ex);
      e = 22 - ex;
    }
    const double inv2e = ldexp(1.0, -e);
#pragma unroll
    for (int t = 0; t < HL_SW; ++t) {
      const int64_t c0 = (int64_t)(wc + t * HL_CONS) * 512 + lane * 16;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float v = (stepv[t] && c0 + q < a.n) ? a.x[c0 + q] : 0.0f;
        X[t][q] = masked ? 0 : __float2int_rn(ldexpf(v, e));
      }
    }
    const uint32_t ld = (uint32_t)a.ld;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t lr = 0; lr < nrows; ++lr) {
      mbar_wait(bar_s + 8 * st, ph);
      const unsigned char* sb = ring + (size_t)st * a.stage_bytes;
      const uint32_t mask = *reinterpret_cast<const uint32_t*>(sb);
      double part;
      if (!masked) {
        long long acc = 0, acc2 = 0;
#pragma unroll
        for (int t = 0; t < HL_SW; ++t) {
          if (!stepv[t]) continue;
          const int c = wc + t * HL_CONS;
          const unsigned char* lo = sb + HL_HDR + c * 512 + lane * 16;
          const uint4 w0 = *reinterpret_cast<const uint4*>(lo);
          const uint4 w1 = *reinterpret_cast<const uint4*>(lo + ld);
          if ((mask >> c) & 1u) {                       // warp-uniform
            const uint4 w2 = *reinterpret_cast<const uint4*>(
                sb + HL_HDR + 2 * ld + __popc(mask & ((1u << c) - 1u)) * 512 + lane * 16);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              const uint32_t wds[3] = {u4get(w0, w), u4get(w1, w), u4get(w2, w)};
              int32_t uv[4];
              dec_int4<3, SIGNED>(wds, uv);
              acc = madw(uv[0], X[t][4 * w + 0], acc);
              acc2 = madw(uv[1], X[t][4 * w + 1], acc2);
              acc = madw(uv[2], X[t][4 * w + 2], acc);
              acc2 = madw(uv[3], X[t][4 * w + 3], acc2);
            }
          } else {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              const uint32_t wds[2] = {u4get(w0, w), u4get(w1, w)};
              int32_t uv[4];
              dec_int4<2, SIGNED>(wds, uv);
              acc = madw(uv[0], X[t][4 * w + 0], acc);
              acc2 = madw(uv[1], X[t][4 * w + 1], acc2);
              acc = madw(uv[2], X[t][4 * w + 2], acc);
              acc2 = madw(uv[3], X[t][4 * w + 3], acc2);
            }
          }
        }
        acc += acc2;
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_s + 8 * (S + st));
        // exact warp sum with two REDUX: |acc| < 64 * 2^24 * 2^22 = 2^52, so the
        // 27-bit low parts sum below 2^32 and the high parts below 2^30
        const uint32_t slo = __reduce_add_sync(0xffffffffu, (uint32_t)acc & 0x7FFFFFFu);
        const int32_t shi = __reduce_add_sync(0xffffffffu, (int32_t)(acc >> 27));
        part = (double)(((long long)shi << 27) + (long long)slo) * inv2e;
      } else {
        // inf/nan in this warp's x: reference zero skip, one double per code
        double acc = 0.0;
        for (int t = 0; t < HL_SW; ++t) {
          if (!stepv[t]) continue;
          const int c = wc + t * HL_CONS;
          const unsigned char* lo = sb + HL_HDR + c * 512 + lane * 16;
          const bool hi = (mask >> c) & 1u;
          const unsigned char* hp = sb + HL_HDR + 2 * ld + __popc(mask & ((1u << c) - 1u)) * 512 + lane * 16;
          for (int q = 0; q < 16; ++q) {
            int32_t v = (int32_t)lo[q] | ((int32_t)lo[ld + q] << 8);
            if (hi) {
              v |= (int32_t)hp[q] << 16;
              if (SIGNED) v = (v << 8) >> 8;
            } else if (SIGNED) {
              v = (int32_t)(int16_t)v;
            }
            if (v == 0) continue;
            const int64_t col = (int64_t)c * 512 + lane * 16 + q;
            if (col < a.n) acc += (double)v * (double)a.x[col];
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_s + 8 * (S + st));
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        part = acc;
      }
      if (lane == 0) slot[lr * HL_CONS + wc] = part;
      if (++st == S) { st = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  for (int64_t r = threadIdx.x; r < nrows; r += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < HL_CONS; ++c) s += slot[r * HL_CONS + c];
    a.y[row_lo + r] = (float)(s * a.scale);
  }
}

int hl_build(invop_plan* p, cudaStream_t s) {
  if (p->hl_ready) return p->hl_ready > 0 ? INVOP_OK : INVOP_E_UNSUPPORTED;
  if (p->P != 3 || p->ld > HL_MAXCOLS || p->rows == 0) {
    p->hl_ready = -1;
    return INVOP_E_UNSUPPORTED;
  }
  const int nch = (int)(p->ld / 512);
  uint32_t* mask = nullptr;
  int64_t* size = nullptr;
  INVOP_CUDA(cudaMalloc(&mask, (size_t)p->rows * 4));
  INVOP_CUDA(cudaMalloc(&size, (size_t)p->rows * 8));
  INVOP_CUDA(cudaMalloc(&p->hl_rowptr, (size_t)(p->rows + 1) * 8));
  INVOP_CUDA(cudaMemsetAsync(mask, 0, (size_t)p->rows * 4, s));
  const int64_t warps = p->rows * nch;
  k_hl_mask<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(p->planes[0], p->planes[1], p->planes[2],
                                                            p->is_signed, p->rows, p->ld, nch, mask);
  k_hl_rowsize<<<(unsigned)cdiv(p->rows, 256), 256, 0, s>>>(p->rows, p->ld, mask, size);
  k_hl_scan<<<1, 1024, 0, s>>>(p->rows, size, p->hl_rowptr);
  int64_t total = 0;
  INVOP_CUDA(cudaMemcpyAsync(&total, p->hl_rowptr + p->rows, 8, cudaMemcpyDeviceToHost, s));
  INVOP_CUDA(cudaStreamSynchronize(s));
  p->hl_bytes = total;
  INVOP_CUDA(cudaMalloc(&p->hl_data, total));
  k_hl_write<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(p->planes[0], p->planes[1], p->planes[2],
                                                             p->rows, p->ld, nch, mask, p->hl_rowptr,
                                                             p->hl_data);
  cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(mask);
  cudaFree(size);
  if (e != cudaSuccess) return cuda_fail(e, "hl build");
  p->hl_ready = 1;
  return INVOP_OK;
}

int apply_hl_launch(invop_plan* p, const float* x, float* y, cudaStream_t s) {
  HlArgs a;
  a.data = p->hl_data;
  a.rowptr = p->hl_rowptr;
  a.rows = p->rows; a.n = p->n; a.ld = p->ld;
  a.scale = p->scale;
  a.x = x; a.y = y;
  a.stage_bytes = (int)(HL_HDR + 3 * p->ld);
  a.piece = 16384;
  if (const char* v = getenv("INVOP_HL_PIECE")) a.piece = (uint32_t)std::max(512, atoi(v)) & ~15u;
  const int grid = (int)std::min<int64_t>(num_sms(), p->rows);
  const int64_t rows_per_cta = cdiv(p->rows, grid);
  int cons = 16;                  // 16 consumers x 2 chunks: 0.106 ms vs 0.117 ms with 8 x 4
  if (const char* v = getenv("INVOP_HL_CONS")) cons = atoi(v) == 8 ? 8 : 16;
  const size_t side = (size_t)rows_per_cta * cons * 8 + (size_t)(rows_per_cta + 1) * 8 + 64;
  const int fit = (int)((225 * 1024 - (int64_t)side) / (a.stage_bytes + 16));
  int stages = 3;                 // measured best at config 4 (3: 0.106 ms, 4: 0.108 ms)
  if (const char* v = getenv("INVOP_HL_STAGES")) stages = std::max(2, atoi(v));
  stages = std::min(stages, fit);
  if (stages < 2) return fail(INVOP_E_UNSUPPORTED, "k2_hl: not enough shared memory");
  a.stages = stages;
  const size_t smem = (size_t)stages * a.stage_bytes + 2 * stages * 8 + side;
  auto kern = cons == 16 ? (p->is_signed ? k2_hl<true, 16> : k2_hl<false, 16>)
                         : (p->is_signed ? k2_hl<true, 8> : k2_hl<false, 8>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, (cons + 1) * 32, smem, s>>>(a);
  INVOP_LAUNCHED(1);
  INVOP_CHECK_LAUNCH("k2_hl");
  return INVOP_OK;
}

}  // namespace invop
