// Tiled variable-width layout ("TVW") and its single-RHS apply k2_tvw.
//
// Layout. Rows are grouped 32 at a time (a row group = one warp, lane = row);
// a row group's columns are cut into 64-column tiles. Each tile (32 x 64
// mantissas) stores base = min over the tile (int32) and u = v - base in
// w = bytes(max - min) bytes per entry (w in 0..4), as w byte planes of 2 KB;
// inside a plane row r's 64 bytes sit at r*64 with 16-byte chunk c stored at
// chunk position c ^ ((r >> 1) & 3), which makes the per-lane 128-bit shared
// loads conflict-free. Tiles of a row group are packed back to back, row
// groups back to back; per tile an int2 {base, (offset_2KB << 3) | w}.
// Config 4: 2.17 B/entry (vs 3 for the byte planes): the inverse is smooth
// over a 32 x 64 block away from the diagonal.
//
// Apply (fp32 I/O, exact per-tile integer sums). A pre-pass turns x into one
// record per 64-column tile: X_j = rint(x_j * 2^e_tile) (23 bits), sum_j X_j,
// e_tile. A work unit is (row group, K part). One producer thread bulk-copies
// stages of 8 consecutive tiles (payload + metadata + x records) into a ring;
// consumer warp k takes tile k of every stage, each lane owns one row:
//   acc = base * sum_j X_j + sum_j u_rj X_j        (int64, exact)
//   part_r += acc * 2^-e_tile                        (fp64)
// so there is no cross-lane reduction on the streaming path at all. At the end
// of a unit the 8 warps' partials are added in fixed order; K parts of a row
// group are combined by the last CTA to finish (deterministic).
#include "common.cuh"
#include "ptx.cuh"
#include <algorithm>

namespace invop {

constexpr int TV_RG = 32;                  // rows per group (lanes)
constexpr int TV_TC = 64;                  // columns per tile
constexpr int TV_PLANE = TV_RG * TV_TC;    // 2 KB per plane of a tile
constexpr int TV_CONS = 8;                 // consumer warps = tiles per stage
constexpr int TV_XREC = 272;               // X[64] int32 + int64 sum + int32 e + pad

struct TvPlanes {
  const uint8_t* p[INVOP_MAX_PLANES];
};

__device__ __forceinline__ int64_t tv_load_code(const TvPlanes& pl, int P, int is_signed,
                                                int64_t off) {
  uint64_t u = 0;
  for (int b = 0; b < P; ++b) u |= (uint64_t)pl.p[b][off] << (8 * b);
  if (is_signed && P < 8) {
    const int sh = 64 - 8 * P;
    return (int64_t)(u << sh) >> sh;
  }
  return (int64_t)u;
}

__device__ __forceinline__ int tv_width(uint64_t range) {
  return range == 0 ? 0 : range < 256 ? 1 : range < 65536 ? 2 : range < (1ull << 24) ? 3 : 4;
}

// one warp per (row group, tile): base and width
__global__ void k_tv_stats(TvPlanes pl, int P, int is_signed, int64_t rows, int64_t ld,
                           int64_t groups, int nt, int2* __restrict__ meta) {
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= groups * nt) return;
  const int64_t g = gw / nt;
  const int t = (int)(gw - g * nt);
  const int64_t row = g * TV_RG + lane;
  int64_t mn = INT64_MAX, mx = INT64_MIN;
  if (row < rows) {
    const int64_t off = row * ld + (int64_t)t * TV_TC;
    for (int j = 0; j < TV_TC; ++j) {
      const int64_t v = tv_load_code(pl, P, is_signed, off + j);
      mn = min(mn, v);
      mx = max(mx, v);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, (int64_t)__shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) meta[g * nt + t] = make_int2((int)mn, tv_width((uint64_t)(mx - mn)));
}

// per row group: tile offsets (2 KB units, relative to the group) and size
__global__ void k_tv_groupscan(int64_t groups, int nt, int2* __restrict__ meta,
                               int64_t* __restrict__ gsize) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= groups) return;
  uint32_t off = 0;
  for (int t = 0; t < nt; ++t) {
    int2 m = meta[g * nt + t];
    const int w = m.y & 7;
    m.y = (int)((off << 3) | w);
    meta[g * nt + t] = m;
    off += w;
  }
  gsize[g] = off;
}

__global__ void k_tv_scan(int64_t groups, const int64_t* __restrict__ gsize,
                          int64_t* __restrict__ gptr) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int64_t per = (groups + T - 1) / T;
  const int64_t a0 = t * per, a1 = min(groups, a0 + per);
  int64_t s = 0;
  for (int64_t g = a0; g < a1; ++g) s += gsize[g];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int i = 0; i < T; ++i) { const int64_t v = part[i]; part[i] = acc; acc += v; }
    gptr[groups] = acc;
  }
  __syncthreads();
  int64_t acc = part[t];
  for (int64_t g = a0; g < a1; ++g) { gptr[g] = acc; acc += gsize[g]; }
}

// stage boundary table: absolute payload offset (2 KB units) at tiles 0, 8, 16, ...
__global__ void k_tv_soff(int64_t groups, int nt, const int2* __restrict__ meta,
                          const int64_t* __restrict__ gptr, int64_t* __restrict__ soff) {
  const int nst = (nt + TV_CONS - 1) / TV_CONS;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= groups * (nst + 1)) return;
  const int64_t g = k / (nst + 1);
  const int s = (int)(k - g * (nst + 1));
  const int t = s * TV_CONS;
  soff[k] = t < nt ? gptr[g] + ((uint32_t)meta[g * nt + t].y >> 3) : gptr[g + 1];
}

// one warp per (row group, tile): lane r writes row r's 64 offsets, swizzled
__global__ void k_tv_write(TvPlanes pl, int P, int is_signed, int64_t rows, int64_t ld,
                           int64_t groups, int nt, const int2* __restrict__ meta,
                           const int64_t* __restrict__ gptr, uint8_t* __restrict__ data) {
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= groups * nt) return;
  const int64_t g = gw / nt;
  const int t = (int)(gw - g * nt);
  const int2 m = meta[g * nt + t];
  const int w = m.y & 7;
  if (w == 0) return;
  const int64_t row = g * TV_RG + lane;
  uint8_t* tile = data + (gptr[g] + ((uint32_t)m.y >> 3)) * (int64_t)TV_PLANE;
  for (int c = 0; c < 4; ++c) {
    uint8_t buf[4][16];
    for (int q = 0; q < 16; ++q) {
      uint32_t u = 0;
      if (row < rows)
        u = (uint32_t)(tv_load_code(pl, P, is_signed, row * ld + (int64_t)t * TV_TC + c * 16 + q) -
                       (int64_t)m.x);
      for (int b = 0; b < 4; ++b) buf[b][q] = (uint8_t)(u >> (8 * b));
    }
    const int pos = lane * TV_TC + ((c ^ ((lane >> 1) & 3)) << 4);
    for (int b = 0; b < w; ++b)
      *reinterpret_cast<uint4*>(tile + b * TV_PLANE + pos) = *reinterpret_cast<const uint4*>(buf[b]);
  }
}

// x -> one record per 64-column tile: X[64] (int32), sum X (int64), e (int32)
constexpr int TV_MASKED = -100000;          // e sentinel: tile of x holds inf/nan

__global__ void k_tv_xprep(const float* __restrict__ x, int64_t n, int nt, int xbits,
                           unsigned char* __restrict__ rec) {
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nt) return;
  const int64_t c0 = t * TV_TC + lane * 2;
  const float v0 = c0 < n ? x[c0] : 0.0f, v1 = c0 + 1 < n ? x[c0 + 1] : 0.0f;
  float m = fmaxf(fabsf(v0), fabsf(v1));
  const bool bad = !(isfinite(v0) && isfinite(v1));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  int e = 0;
  if (m > 0.0f && isfinite(m)) {
    int ex;
    frexpf(m, &ex);
    e = xbits - ex;
  }
  const int X0 = bad ? 0 : __float2int_rn(ldexpf(v0, e));
  const int X1 = bad ? 0 : __float2int_rn(ldexpf(v1, e));
  long long s = (long long)X0 + X1;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  unsigned char* r = rec + t * TV_XREC;
  reinterpret_cast<int2*>(r)[lane] = make_int2(X0, X1);
  const bool any_bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    *reinterpret_cast<long long*>(r + 256) = s;
    *reinterpret_cast<int*>(r + 264) = any_bad ? TV_MASKED : e;
  }
}

struct TvArgs {
  const float* x;
  int64_t n;
  const uint8_t* data;
  const int2* meta;          // [groups][nt]
  const int64_t* gptr;       // [groups+1], 2 KB units
  const int64_t* soff;       // [groups][nst+1] absolute offsets at every 8-tile stage boundary
  const unsigned char* xrec; // [nt] x records
  int64_t rows;
  int64_t groups;
  int nt;                    // tiles per row group
  int parts;                 // K parts per row group
  int tiles_per_part;
  int stages;
  int stage_bytes;
  int payload_off;           // start of the payload inside a stage
  double scale;
  float* y;
  double* partial;           // [groups*32][parts]
  int* counters;             // [groups]
};

__device__ __forceinline__ uint4 tv_lds128(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(addr));
  return r;
}

// row lane's 64 codes of a tile (w planes) against the tile's X record
template <int W>
__device__ __forceinline__ long long tv_tile_dot(uint32_t tile_s, uint32_t xrec_s, int lane) {
  long long acc = 0, acc2 = 0;
  const uint32_t rowb = tile_s + lane * TV_TC;
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t pos = rowb + ((c ^ sw) << 4);
    uint4 cw[W];
#pragma unroll
    for (int b = 0; b < W; ++b) cw[b] = tv_lds128(pos + b * TV_PLANE);
    const uint4 x0 = tv_lds128(xrec_s + c * 64), x1 = tv_lds128(xrec_s + c * 64 + 16);
    const uint4 x2 = tv_lds128(xrec_s + c * 64 + 32), x3 = tv_lds128(xrec_s + c * 64 + 48);
    const int32_t Xc[16] = {(int)x0.x, (int)x0.y, (int)x0.z, (int)x0.w, (int)x1.x, (int)x1.y,
                            (int)x1.z, (int)x1.w, (int)x2.x, (int)x2.y, (int)x2.z, (int)x2.w,
                            (int)x3.x, (int)x3.y, (int)x3.z, (int)x3.w};
#pragma unroll
    for (int wd = 0; wd < 4; ++wd) {
      uint32_t wds[4];
#pragma unroll
      for (int b = 0; b < W; ++b) wds[b] = u4get(cw[b], wd);
      if (W == 4) {
        const uint32_t t01 = prmt(wds[0], wds[1], 0x5140), t23 = prmt(wds[0], wds[1], 0x7362);
        const uint32_t h01 = prmt(wds[2], wds[3], 0x5140), h23 = prmt(wds[2], wds[3], 0x7362);
        acc += (long long)prmt(t01, h01, 0x5410) * Xc[4 * wd + 0];
        acc2 += (long long)prmt(t01, h01, 0x7632) * Xc[4 * wd + 1];
        acc += (long long)prmt(t23, h23, 0x5410) * Xc[4 * wd + 2];
        acc2 += (long long)prmt(t23, h23, 0x7632) * Xc[4 * wd + 3];
      } else {
        int32_t uv[4];
        dec_int4<W, false>(wds, uv);
        acc = madw(uv[0], Xc[4 * wd + 0], acc);
        acc2 = madw(uv[1], Xc[4 * wd + 1], acc2);
        acc = madw(uv[2], Xc[4 * wd + 2], acc);
        acc2 = madw(uv[3], Xc[4 * wd + 3], acc2);
      }
    }
  }
  return acc + acc2;
}

__global__ void __launch_bounds__((TV_CONS + 1) * 32, 1) k2_tvw(TvArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = a.stages;
  unsigned char* ring = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * a.stage_bytes);
  double* red = reinterpret_cast<double*>(bars + 2 * S);   // [TV_CONS][32]
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bars);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t units = a.groups * a.parts;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(bar_s + 8 * i, 1);
      mbar_init(bar_s + 8 * (S + i), TV_CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == TV_CONS) {
    // ------------------------------------------------------------ producer
    // The whole warp walks the units; per unit its lanes fetch the stage
    // boundary offsets in one parallel load (no dependent global load per
    // stage), lane 0 issues the copies.
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    int st = 0;
    uint32_t ph = 0;
    int64_t it = 0;
    const int nst = (a.nt + TV_CONS - 1) / TV_CONS;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int64_t g = u / a.parts;
      const int part = (int)(u - g * a.parts);
      const int t0 = part * a.tiles_per_part;
      const int t1 = min(a.nt, t0 + a.tiles_per_part);
      const int2* mg = a.meta + g * a.nt;
      const int k0 = t0 / TV_CONS, k1 = (t1 + TV_CONS - 1) / TV_CONS;   // stage range
      for (int kc = k0; kc < k1; kc += 31) {
        const int kn = min(31, k1 - kc);
        // lane i holds the offset at stage boundary kc + i (i <= kn)
        int64_t off = 0;
        if (lane <= kn) off = a.soff[g * (nst + 1) + kc + lane];
        for (int i = 0; i < kn; ++i, ++it) {
          const int64_t o0 = __shfl_sync(0xffffffffu, off, i);
          const int64_t o1 = __shfl_sync(0xffffffffu, off, i + 1);
          if (lane == 0) {
            const int ts = (kc + i) * TV_CONS;
            const int te = min(t1, ts + TV_CONS);
            if (it >= S) mbar_wait(bar_s + 8 * (S + st), ph ^ 1);
            const uint32_t pay = (uint32_t)(o1 - o0) * TV_PLANE;
            const uint32_t mbytes = (uint32_t)(((te - ts) + 1) & ~1) * 8;
            const uint32_t xbytes = (uint32_t)(te - ts) * TV_XREC;
            const uint32_t sb = ring_s + st * a.stage_bytes;
            mbar_expect_tx(bar_s + 8 * st, mbytes + xbytes + pay);
            bulk_g2s(sb, mg + ts, mbytes, bar_s + 8 * st, policy);
            bulk_g2s(sb + 64, a.xrec + (int64_t)ts * TV_XREC, xbytes, bar_s + 8 * st, policy);
            if (pay)
              bulk_g2s(sb + a.payload_off, a.data + o0 * (int64_t)TV_PLANE, pay, bar_s + 8 * st,
                       policy);
          }
          if (++st == S) { st = 0; ph ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    int st = 0;
    uint32_t ph = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      const int64_t g = u / a.parts;
      const int part = (int)(u - g * a.parts);
      const int t0 = part * a.tiles_per_part;
      const int t1 = min(a.nt, t0 + a.tiles_per_part);
      double row_part = 0.0;
      for (int ts = t0; ts < t1; ts += TV_CONS) {
        mbar_wait(bar_s + 8 * st, ph);
        const uint32_t sb = ring_s + st * a.stage_bytes;
        const int t = ts + warp;
        if (t < t1) {
          const int2* sm = reinterpret_cast<const int2*>(ring + (size_t)st * a.stage_bytes);
          const uint32_t o0 = (uint32_t)sm[0].y >> 3;
          const int2 m = sm[warp];
          const int w = m.y & 7;
          const uint32_t tile_s = sb + a.payload_off + (((uint32_t)m.y >> 3) - o0) * TV_PLANE;
          const uint32_t xrec_s = sb + 64 + warp * TV_XREC;
          const unsigned char* xr = ring + (size_t)st * a.stage_bytes + 64 + warp * TV_XREC;
          const int e = *reinterpret_cast<const int*>(xr + 264);
          if (e == TV_MASKED) {
            // inf/nan in this tile of x: fp64 with the reference's zero skip
            const unsigned char* tp = ring + (size_t)st * a.stage_bytes + a.payload_off +
                                      (((uint32_t)m.y >> 3) - o0) * TV_PLANE;
            const int sw = (lane >> 1) & 3;
            for (int j = 0; j < TV_TC; ++j) {
              const int pos = lane * TV_TC + (((j >> 4) ^ sw) << 4) + (j & 15);
              uint32_t uu = 0;
              for (int b = 0; b < w; ++b) uu |= (uint32_t)tp[b * TV_PLANE + pos] << (8 * b);
              const long long v = (long long)m.x + (long long)uu;
              const int64_t col = (int64_t)t * TV_TC + j;
              if (v != 0 && col < a.n) row_part += (double)v * (double)a.x[col];
            }
          } else {
            long long acc = (long long)m.x * *reinterpret_cast<const long long*>(xr + 256);
            switch (w) {                                 // warp-uniform
              case 1: acc += tv_tile_dot<1>(tile_s, xrec_s, lane); break;
              case 2: acc += tv_tile_dot<2>(tile_s, xrec_s, lane); break;
              case 3: acc += tv_tile_dot<3>(tile_s, xrec_s, lane); break;
              case 4: acc += tv_tile_dot<4>(tile_s, xrec_s, lane); break;
              default: break;
            }
            row_part = fma((double)acc, ldexp(1.0, -e), row_part);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_s + 8 * (S + st));
        if (++st == S) { st = 0; ph ^= 1; }
      }
      // fixed-order combination of the 8 warps' partials of this unit
      red[warp * 32 + lane] = row_part;
      asm volatile("bar.sync 1, %0;" ::"r"(TV_CONS * 32));
      if (warp == 0) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < TV_CONS; ++k) s += red[k * 32 + lane];
        const int64_t row = g * TV_RG + lane;
        if (a.parts == 1) {
          if (row < a.rows) a.y[row] = (float)(s * a.scale);
        } else {
          a.partial[(g * TV_RG + lane) * a.parts + part] = s;
          __threadfence();
          __syncwarp();
          int last = 0;
          if (lane == 0) last = atomicAdd(&a.counters[g], 1) == a.parts - 1;
          last = __shfl_sync(0xffffffffu, last, 0);
          if (last) {
            __threadfence();
            double tot = 0.0;
            for (int k = 0; k < a.parts; ++k)
              tot += __ldcg(&a.partial[(g * TV_RG + lane) * a.parts + k]);
            if (row < a.rows) a.y[row] = (float)(tot * a.scale);
            if (lane == 0) a.counters[g] = 0;
          }
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(TV_CONS * 32));
    }
  }
}

// ------------------------------------------------------------------ host
int tvw_build(invop_plan* p, cudaStream_t s) {
  if (p->tv_ready) return p->tv_ready > 0 ? INVOP_OK : INVOP_E_UNSUPPORTED;
  if (p->min_val < INT32_MIN || p->max_val > INT32_MAX || p->rows == 0 || p->ld % TV_TC) {
    p->tv_ready = -1;
    return INVOP_E_UNSUPPORTED;
  }
  const int64_t groups = cdiv(p->rows, TV_RG);
  const int nt = (int)(p->ld / TV_TC);
  TvPlanes pl;
  for (int b = 0; b < INVOP_MAX_PLANES; ++b) pl.p[b] = p->planes[b];
  INVOP_CUDA(cudaMalloc(&p->tv_meta, (size_t)(groups * nt + 2) * sizeof(int2)));
  INVOP_CUDA(cudaMalloc(&p->tv_gptr, (size_t)(groups + 1) * sizeof(int64_t)));
  int64_t* gsize = nullptr;
  INVOP_CUDA(cudaMalloc(&gsize, (size_t)groups * sizeof(int64_t)));
  const int64_t warps = groups * nt;
  k_tv_stats<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(pl, p->P, p->is_signed, p->rows,
                                                             p->ld, groups, nt, (int2*)p->tv_meta);
  k_tv_groupscan<<<(unsigned)cdiv(groups, 256), 256, 0, s>>>(groups, nt, (int2*)p->tv_meta, gsize);
  k_tv_scan<<<1, 1024, 0, s>>>(groups, gsize, p->tv_gptr);
  int64_t total = 0;
  INVOP_CUDA(cudaMemcpyAsync(&total, p->tv_gptr + groups, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  INVOP_CUDA(cudaStreamSynchronize(s));
  cudaFree(gsize);
  p->tv_bytes = total * TV_PLANE;
  const int nst = (nt + TV_CONS - 1) / TV_CONS;
  INVOP_CUDA(cudaMalloc(&p->tv_soff, (size_t)groups * (nst + 1) * sizeof(int64_t)));
  k_tv_soff<<<(unsigned)cdiv(groups * (nst + 1), 256), 256, 0, s>>>(groups, nt,
                                                                    (const int2*)p->tv_meta,
                                                                    p->tv_gptr, p->tv_soff);
  INVOP_CUDA(cudaMalloc(&p->tv_data, p->tv_bytes > 0 ? p->tv_bytes : 16));
  k_tv_write<<<(unsigned)cdiv(warps * 32, 256), 256, 0, s>>>(pl, p->P, p->is_signed, p->rows,
                                                             p->ld, groups, nt,
                                                             (const int2*)p->tv_meta, p->tv_gptr,
                                                             p->tv_data);
  INVOP_CHECK_LAUNCH("tvw build");
  const uint64_t range = (uint64_t)(p->max_val - p->min_val);
  p->tv_wmax = range < 256 ? 1 : range < 65536 ? 2 : range < (1ull << 24) ? 3 : 4;
  p->tv_ready = 1;
  return INVOP_OK;
}

int64_t tvw_stream_bytes(const invop_plan* p) {
  const int64_t groups = cdiv(p->rows, TV_RG), nt = p->ld / TV_TC;
  return p->tv_bytes + groups * nt * 8 + (groups + 1) * 8;
}

int apply_tvw_launch(invop_plan* p, const float* x, float* y, cudaStream_t s) {
  const int64_t groups = cdiv(p->rows, TV_RG);
  const int nt = (int)(p->ld / TV_TC);
  const int sms = num_sms();
  // K parts: fill the SMs in whole waves
  int parts = 1;
  double best = -1.0;
  for (int pc = 1; pc <= 8; ++pc) {
    const int64_t units = groups * pc;
    double eff = (double)units / ((double)cdiv(units, sms) * sms) - 0.01 * pc;
    if (eff > best + 1e-9) { best = eff; parts = pc; }
  }
  int tpp = (int)cdiv(nt, parts);
  tpp = (int)round_up(tpp, TV_CONS);
  parts = (int)cdiv(nt, tpp);
  // workspace: x records | partials | counters
  const size_t xrec_bytes = (size_t)nt * TV_XREC;
  const size_t part_off = round_up(xrec_bytes, 256);
  const size_t part_bytes = parts > 1 ? (size_t)groups * TV_RG * parts * 8 : 0;
  const size_t cnt_off = round_up(part_off + part_bytes, 256);
  const size_t cnt_bytes = (size_t)groups * 4;
  void* before = p->tv_ws;
  int rc = ensure_scratch(&p->tv_ws, &p->tv_ws_bytes, cnt_off + cnt_bytes);
  if (rc) return rc;
  if (p->tv_ws != before || p->tv_ws_cnt_off != (int64_t)cnt_off) {
    // completion counters start at zero; the last CTA of a row group resets its own
    INVOP_CUDA(cudaMemsetAsync((char*)p->tv_ws + cnt_off, 0, cnt_bytes, s));
    p->tv_ws_cnt_off = (int64_t)cnt_off;
  }
  unsigned char* xrec = (unsigned char*)p->tv_ws;
  int vb = 1;
  while (vb < 62 && ((int64_t)1 << vb) <= p->max_abs) ++vb;
  const int xbits = std::max(8, std::min(22, 61 - vb - 7));   // 64 terms per tile
  k_tv_xprep<<<(unsigned)cdiv((int64_t)nt * 32, 256), 256, 0, s>>>(x, p->n, nt, xbits, xrec);
  TvArgs a;
  a.x = x;
  a.n = p->n;
  a.data = p->tv_data;
  a.meta = (const int2*)p->tv_meta;
  a.gptr = p->tv_gptr;
  a.soff = p->tv_soff;
  a.xrec = xrec;
  a.rows = p->rows;
  a.groups = groups;
  a.nt = nt;
  a.parts = parts;
  a.tiles_per_part = tpp;
  a.scale = p->scale;
  a.y = y;
  a.partial = (double*)((char*)p->tv_ws + part_off);
  a.counters = (int*)((char*)p->tv_ws + cnt_off);
  a.payload_off = (int)round_up(64 + TV_CONS * TV_XREC, 128);
  a.stage_bytes = a.payload_off + p->tv_wmax * TV_CONS * TV_PLANE;
  const size_t red_bytes = TV_CONS * 32 * sizeof(double);
  int stages = (int)((225 * 1024 - red_bytes - 256) / (a.stage_bytes + 16));
  stages = std::min(stages, 12);
  if (stages < 2) return fail(INVOP_E_UNSUPPORTED, "k2_tvw: not enough shared memory");
  a.stages = stages;
  const size_t smem = (size_t)stages * a.stage_bytes + 2 * stages * 8 + red_bytes;
  cudaFuncSetAttribute(k2_tvw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = (int)std::min<int64_t>(sms, groups * parts);
  k2_tvw<<<grid, (TV_CONS + 1) * 32, smem, s>>>(a);
  INVOP_LAUNCHED(2);   // + k_tv_xprep
  INVOP_CHECK_LAUNCH("k2_tvw");
  return INVOP_OK;
}

}  // namespace invop
