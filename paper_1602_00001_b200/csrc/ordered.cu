// k2_ordered — the bitwise fp64 apply (INVOP_MODE_ORDERED) on sm_100a.
//
// Reference contract: invop.apply -> _kernels.plan_apply
//   /root/reference/pkg/src/invop/applyplan.py:4-8,175-191
//   /root/reference/pkg/src/invop/_kernels/_native.pyx:15-49
// Every output row accumulates t = (|v| * 10^-m) * x_j in ascending j, in fp64,
// product and sum rounded separately (no FMA across them), zero mantissas
// skipped. The chain of a row is sequential by contract, so one thread owns
// one row and a warp owns 32 rows; what the design can choose is how the warp
// is fed and how few instructions it spends per element beside the three
// fp64 operations (coefficient, product, ordered add):
//
//  * a block is one producer warp plus four consumer warps, one consumer per
//    SM scheduler (a lone chain is latency-bound: 8 cycles per DADD link, so
//    what matters is that no two chains share a scheduler while another
//    idles). Per 128-column tile the producer issues ONE 2-D tensor copy per
//    byte plane (box 128 B x 128 rows, 128-byte swizzle: a thread's row walk is
//    conflict-free LDS.128) and one bulk copy of the x tile into a stage ring
//    shared by the consumers (full / empty mbarriers), and leaves a flag when
//    the tile's x holds inf/nan (read one tile ahead, off the critical path);
//  * consumers walk their rows as a software pipeline carried through
//    registers: the 16 products of chunk c are added while chunk c+1 is decoded
//    and multiplied — two independent value sets, so ptxas interleaves them
//    (it schedules a product right before its add otherwise);
//  * codes are assembled with PRMT (sign-replicate mode supplies the fourth
//    byte of 3-byte codes whose top bit is clear, so no mask);
//  * the coefficient is one fp64 operation: fma(2^52 + |v|, s, -2^52 s);
//  * more row blocks than SMs: shallower rings, two blocks per SM; more than
//    two per SM: 224-row blocks of seven consumers reading x from global
//    memory (all row warps of config 5 in one round).
// INVOP_ORD_PROBE (measurement only): 1 copies without arithmetic, 2 arithmetic
// without copies, 4 arithmetic without barriers.
#include "common.cuh"
#include "ptx.cuh"
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace invop {

constexpr int ORD_TILE = 128;   // columns per stage

struct OrdArgs {
  int64_t rows, n;
  double scale;
  double neg_scale52;   // -(2^52 * scale), exact
  const double* x;
  int64_t ldx;
  double* y;
  int64_t ldy;
  // accumulate mode (the reference seam's `out +=` contract, _native.pyx:43-46):
  // each row's chain starts at y[row] instead of +0, and zero codes are
  // skipped outright (the reference never adds them; -0 + +0 would be +0)
  int accumulate;
  // x tiles by bulk copy (x and its leading dimension 16-byte aligned);
  // otherwise the lanes copy them
  int xbulk;
  // measurement probes (INVOP_ORD_PROBE): 1 = consumers skip the arithmetic
  // (copy pipeline alone), 2 = the producer skips the copies (arithmetic alone)
  int probe;
};

template <int P>
struct alignas(64) OrdMaps {
  unsigned char m[P][128];
};

template <int P, bool SIGNED>
__device__ __forceinline__ double code_to_double(const uint8_t* bytes) {
  uint64_t u = 0;
#pragma unroll
  for (int b = 0; b < P; ++b) u |= (uint64_t)bytes[b] << (8 * b);
  int64_t v;
  if (SIGNED && P < 8) {
    const int sh = 64 - 8 * P;
    v = (int64_t)(u << sh) >> sh;
  } else {
    v = (int64_t)u;
  }
  return (double)v;  // exact for |v| <= 2^53 (quantize guarantees it)
}

// P planes, SIGNED coefficient path (negative codes present), SX: decode with
// the sign-extending PRMT although the codes are non-negative (top stored bit
// clear), KR right-hand sides per pass
__device__ __forceinline__ uint4 lds_u4(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
  return r;
}
__device__ __forceinline__ double2 lds_d2(uint32_t addr) {
  double2 r;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(addr));
  return r;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(addr));
  return r;
}

// Block = NC consumer warps (32 rows each) + one producer warp. All consumers
// share the stage ring: a stage holds, per byte plane, one tensor-copy box of
// NC*32 rows x 128 columns and the x tile(s); per stage a full barrier (the
// producer's arrive + the copies' bytes), an empty barrier (one arrive per
// active consumer warp) and a flag word (tile needs the zero-skip path).
// NC = 4 puts one consumer on each of the SM's four schedulers.
// XG: the stages hold the code tiles only and the consumers read x from global
// memory (L1/L2-resident) — what lets two blocks of seven consumers share an SM.
template <int P, bool SIGNED, bool SX, int KR, int NC, int S, bool XG = false>
__global__ void __launch_bounds__((NC + 1) * 32, XG ? 2 : 1)
    k2_ordered(const __grid_constant__ OrdMaps<P> maps, OrdArgs a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nc = NC;
  constexpr int ORD_STAGES = S;
  constexpr int PLANE_BYTES = NC * 32 * ORD_TILE;           // per plane per stage
  constexpr int CODE_BYTES = PLANE_BYTES;
  constexpr int X_BYTES = ORD_TILE * 8 * KR;                // per stage
  constexpr int STAGE_BYTES = PLANE_BYTES * P + (XG ? 0 : X_BYTES);
  const uint32_t sm_s = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t ctl_s = sm_s + (uint32_t)S * STAGE_BYTES;  // control words after the stages
  // per stage: full @ +0, empty @ +8, flag @ +16 (padded to 32 bytes)
  auto full_bar = [&](int st) { return ctl_s + (uint32_t)st * 32; };
  auto empty_bar = [&](int st) { return ctl_s + (uint32_t)st * 32 + 8; };
  auto flag_addr = [&](int st) { return ctl_s + (uint32_t)st * 32 + 16; };
  const int64_t ntiles = (a.n + ORD_TILE - 1) / ORD_TILE;
  const int64_t brow0 = (int64_t)blockIdx.x * (NC * 32);
  const int active = (int)min((int64_t)NC, (a.rows - brow0 + 31) / 32);   // consumer warps with rows

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full_bar(i), 1);
      mbar_init(empty_bar(i), (uint32_t)active);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == nc) {
    // ------------------------------------------------------------ producer
    if (a.probe & 4) return;
    uint64_t pol_stream, pol_keep;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    // x of a tile, 4 columns per lane and right-hand side (lane + 32 i):
    // loaded one tile ahead so its latency hides behind the previous tile's
    // issue; used for the inf/nan flag and for the lane-copied tiles
    double xv[KR][4], xn[KR][4];
    auto load_x = [&](int64_t t, double (&v)[KR][4]) {
#pragma unroll
      for (int k = 0; k < KR; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t col = t * ORD_TILE + lane + 32 * i;
          v[k][i] = col < a.n ? a.x[k * a.ldx + col] : 0.0;
        }
    };
    load_x(0, xv);
    for (int64_t t = 0; t < ntiles; ++t) {
      const int st = (int)(t % ORD_STAGES);
      const uint32_t ph = (uint32_t)((t / ORD_STAGES) & 1);
      const int64_t col0 = t * ORD_TILE;
      const bool xb = !XG && a.xbulk && col0 + ORD_TILE <= a.n;
      bool fin = true;
#pragma unroll
      for (int k = 0; k < KR; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) fin = fin && isfinite(xv[k][i]);
      const uint32_t flag = (a.accumulate || __any_sync(0xffffffffu, !fin)) ? 1u : 0u;
      if (t + 1 < ntiles) load_x(t + 1, xn);
      mbar_wait(empty_bar(st), ph ^ 1);      // every consumer released this stage
      const uint32_t sb = sm_s + (uint32_t)st * STAGE_BYTES;
      if (!xb && !XG) {
        // tail tile or unaligned x: the lanes copy it (zero past n)
#pragma unroll
        for (int k = 0; k < KR; ++k)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(sb + P * CODE_BYTES +
                                                         (k * ORD_TILE + lane + 32 * i) * 8),
                         "d"(xv[k][i]) : "memory");
        __syncwarp();
      }
      if (lane == 0 && (a.probe & 2)) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(flag_addr(st)), "r"(flag) : "memory");
        mbar_arrive(full_bar(st));
      } else if (lane == 0) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(flag_addr(st)), "r"(flag) : "memory");
        const uint32_t bar = full_bar(st);
        mbar_expect_tx(bar, (uint32_t)(P * CODE_BYTES + (xb ? X_BYTES : 0)));
#pragma unroll
        for (int b = 0; b < P; ++b)
          tma_load_2d(sb + b * CODE_BYTES, maps.m[b], (int)col0, (int)brow0, bar, pol_stream);
        if (xb) {
#pragma unroll
          for (int k = 0; k < KR; ++k)
            bulk_g2s(sb + P * CODE_BYTES + k * ORD_TILE * 8, a.x + k * a.ldx + col0,
                     ORD_TILE * 8, bar, pol_keep);
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < KR; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) xv[k][i] = xn[k][i];
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int64_t row0 = brow0 + warp * 32;
  if (row0 >= a.rows) return;  // whole warp idle (warp-uniform; not counted in `active`)
  const int64_t myrow = row0 + lane;
  // my row's 128-byte line inside a code tile; 16-byte chunk c sits at c ^ (row & 7)
  const uint32_t row_off = (uint32_t)(warp * 32 + lane) * 128;
  const uint32_t swz = (uint32_t)(lane & 7);

  double acc[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k)
    acc[k] = (a.accumulate && myrow < a.rows) ? a.y[k * a.ldy + myrow] : 0.0;

  auto stage_of = [&](int64_t t) -> uint32_t {
    return sm_s + (uint32_t)(t % ORD_STAGES) * STAGE_BYTES;
  };
  // waits for tile t; returns its zero-skip flag.
  // For finite x, adding (0*10^-m)*x_j = +-0 leaves the accumulator bitwise
  // unchanged (it starts at +0 and x+(-x) rounds to +0), so the reference's
  // zero skip only matters when the tile holds inf/nan (or in accumulate
  // mode): then the chain does not advance on a zero code.
  auto wait_tile = [&](int64_t t) -> bool {
    const int st = (int)(t % ORD_STAGES);
    if (a.probe & 4) return false;
    mbar_wait(full_bar(st), (uint32_t)((t / ORD_STAGES) & 1));
    return lds_u32(flag_addr(st)) != 0;
  };
  auto release_tile = [&](int64_t t) {
    if (a.probe & 4) return;
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar((int)(t % ORD_STAGES)));
  };
  // coefficients of the 16 codes of chunk c of a staged tile.
  // fl(|v| * 10^-m) in ONE fp64 operation: V = 2^52 + |v| is built from bits,
  // and fma(V, s, -2^52 s) = round((2^52 + |v|) s - 2^52 s) = round(|v| s)
  // exactly, because 2^52 s is exact (a power-of-two multiple of the double s).
  // The sign is applied to the rounded coefficient (rounding to nearest is
  // sign-symmetric), as the reference applies it to its products
  // (_native.pyx:43-46).
  auto chunk_coeffs = [&](uint32_t sb, int c, double (&d)[16]) {
    uint4 w[P];
    const uint32_t ca = sb + row_off + (((uint32_t)c ^ swz) << 4);
#pragma unroll
    for (int b = 0; b < P; ++b) w[b] = lds_u4(ca + b * CODE_BYTES);
    if constexpr (P <= 4) {
#pragma unroll
      for (int wd = 0; wd < 4; ++wd) {
        uint32_t wds[4];
#pragma unroll
        for (int b = 0; b < P; ++b) wds[b] = u4get(w[b], wd);
        int32_t uv[4];
        dec_int4<P, SIGNED || SX>(wds, uv);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (SIGNED) {
            const int32_t sv = uv[i];
            const int32_t sgn = sv >> 31;
            const uint32_t av = (uint32_t)((sv ^ sgn) - sgn);
            const double cf = __fma_rn(__hiloint2double(0x43300000, (int)av), a.scale, a.neg_scale52);
            d[4 * wd + i] = __hiloint2double(__double2hiint(cf) ^ (int)((uint32_t)sgn & 0x80000000u),
                                             __double2loint(cf));
          } else {
            d[4 * wd + i] = __fma_rn(__hiloint2double(0x43300000, uv[i]), a.scale, a.neg_scale52);
          }
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        uint8_t bytes[P];
#pragma unroll
        for (int b = 0; b < P; ++b) bytes[b] = (uint8_t)(u4get(w[b], q >> 2) >> (8 * (q & 3)));
        d[q] = __dmul_rn(code_to_double<P, SIGNED>(bytes), a.scale);
      }
    }
  };
  // products of chunk c against right-hand side k
  auto chunk_products = [&](uint32_t sb, int64_t t, int c, int k, const double (&d)[16],
                            double (&t2)[16]) {
    const uint32_t xa = sb + P * CODE_BYTES + (uint32_t)(k * ORD_TILE + c * 16) * 8;
    // XG: the launcher guarantees 16-byte aligned x rows and n % 128 == 0
    const double2* xg =
        reinterpret_cast<const double2*>(a.x + k * a.ldx + t * ORD_TILE + c * 16);
#pragma unroll
    for (int q2 = 0; q2 < 8; ++q2) {
      const double2 xv = XG ? __ldg(xg + q2) : lds_d2(xa + q2 * 16);
      t2[2 * q2] = __dmul_rn(d[2 * q2], xv.x);
      t2[2 * q2 + 1] = __dmul_rn(d[2 * q2 + 1], xv.y);
    }
  };
  // one tile, straight-line (8 chunks of 16 codes, no guards: rows and columns
  // past the operator are zero-filled by the tensor copy, x past n is zero)
  auto tile_pass = [&](uint32_t sb, int64_t t, auto masked_tag) {
    constexpr bool MASKED = decltype(masked_tag)::value;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double d[16];
      chunk_coeffs(sb, c, d);
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        double t2[16];
        chunk_products(sb, t, c, k, d, t2);
        if (MASKED) {
          // the reference's zero skip (_native.pyx:32-46 never sees a zero
          // mantissa): the chain does not advance on a zero code
#pragma unroll
          for (int q = 0; q < 16; ++q) acc[k] = d[q] != 0.0 ? __dadd_rn(acc[k], t2[q]) : acc[k];
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) acc[k] = __dadd_rn(acc[k], t2[q]);
        }
      }
    }
  };

  if constexpr (KR == 1 && P <= 4) {
    // Single right-hand side: a software pipeline carried through registers.
    // One loop iteration adds the 16 products of chunk c (formed in the
    // previous iteration) while it decodes chunk c+1 and forms its products;
    // the two halves share no value, so the ordered DADD chain (8 cycles per
    // link, sequential by contract) is the only dependency in the block and
    // everything else fills its issue gaps. Two product sets alternate (even /
    // odd chunks in separate blocks), so no register copies rotate them.
    double ttA[16], ttB[16];
    double a0 = acc[0];
    auto chain = [&](const double (&t2)[16]) {
#pragma unroll
      for (int q = 0; q < 16; ++q) a0 = __dadd_rn(a0, t2[q]);
    };
    auto products = [&](uint32_t sb, int64_t t, int c, double (&t2)[16]) {
      double d[16];
      chunk_coeffs(sb, c, d);
      chunk_products(sb, t, c, 0, d, t2);
    };
    bool have = false;         // ttA holds chunk 0 of tile t
    bool waited = false, masked = false;
    for (int64_t t = 0; t < ntiles; ++t) {
      const uint32_t sb = stage_of(t);
      if (a.probe & 1) {
        wait_tile(t);
        release_tile(t);
        continue;
      }
      if (!waited) masked = wait_tile(t);
      waited = false;
      if (masked) {
        acc[0] = a0;
        tile_pass(sb, t, std::true_type{});
        a0 = acc[0];
        have = false;
        release_tile(t);
        continue;
      }
      if (!have) products(sb, t, 0, ttA);
#pragma unroll
      for (int c = 0; c < 7; ++c) {
        if ((c & 1) == 0) {
          chain(ttA);
          products(sb, t, c + 1, ttB);
        } else {
          chain(ttB);
          products(sb, t, c + 1, ttA);
        }
      }
      release_tile(t);
      // chunk 7 is added while chunk 0 of the next tile is prepared
      have = false;
      if (t + 1 < ntiles) {
        masked = wait_tile(t + 1);
        waited = true;
        if (!masked) {
          chain(ttB);
          products(stage_of(t + 1), t + 1, 0, ttA);
          have = true;
        }
      }
      if (!have) chain(ttB);
    }
    acc[0] = a0;
  } else {
    for (int64_t t = 0; t < ntiles; ++t) {
      const uint32_t sb = stage_of(t);
      if (wait_tile(t)) tile_pass(sb, t, std::true_type{});
      else tile_pass(sb, t, std::false_type{});
      release_tile(t);
    }
  }
  if (myrow < a.rows) {
#pragma unroll
    for (int k = 0; k < KR; ++k) a.y[k * a.ldy + myrow] = acc[k];
  }
}

// consumer warps per block and stages for a code width: four consumers (one
// per scheduler) whenever two stages of 128-row boxes fit in shared memory
constexpr int ord_nc(int P) { return P <= 6 ? 4 : 2; }
constexpr int ord_stage_bytes(int P, int KR) { return ord_nc(P) * 32 * ORD_TILE * P + ORD_TILE * 8 * KR; }
constexpr int ord_stages(int P, int KR) {
  return (220 * 1024) / ord_stage_bytes(P, KR) < 4 ? (220 * 1024) / ord_stage_bytes(P, KR) : 4;
}

// the plan's per-plane tensor maps (built once per geometry)
static int ord_get_maps(const invop_plan* cp, int box_rows, const unsigned char (**out)[128]) {
  invop_plan* p = const_cast<invop_plan*>(cp);
  const int64_t geom[4] = {p->rows, p->n, p->ld, p->P * 1000 + box_rows};
  if (p->ord_maps_key != p->planes[0] || memcmp(geom, p->ord_maps_geom, sizeof(geom)) != 0) {
    p->ord_maps_key = nullptr;
    for (int b = 0; b < p->P; ++b) {
      // columns past n and rows past the shard read as zero codes
      int rc = make_tensor_map_u8(p->ord_maps[b], p->planes[b], (uint64_t)p->n, (uint64_t)p->rows,
                                  (uint64_t)p->ld, ORD_TILE, (uint32_t)box_rows, 128);
      if (rc) return rc;
    }
    memcpy(p->ord_maps_geom, geom, sizeof(geom));
    p->ord_maps_key = p->planes[0];
  }
  *out = p->ord_maps;
  return INVOP_OK;
}

// stages such that two blocks share an SM (two consumers per scheduler)
constexpr int ord_stages2(int P, int KR) {
  return (112 * 1024) / ord_stage_bytes(P, KR) < 4 ? (112 * 1024) / ord_stage_bytes(P, KR) : 4;
}

template <int P, bool SIGNED, bool SX, int KR, int NC, int S, bool XG>
static int launch_ord_s(const invop_plan* p, OrdArgs a, cudaStream_t s) {
  const unsigned char (*maps)[128] = nullptr;
  const int rc = ord_get_maps(p, NC * 32, &maps);
  if (rc) return rc;
  const size_t smem = (size_t)(NC * 32 * ORD_TILE * P + (XG ? 0 : ORD_TILE * 8 * KR)) * S + 32 * S;
  auto kern = k2_ordered<P, SIGNED, SX, KR, NC, S, XG>;
  INVOP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  OrdMaps<P> m;
  memcpy(m.m, maps, sizeof(m.m));
  const int64_t grid = cdiv(a.rows, NC * 32);
  kern<<<(unsigned)grid, (NC + 1) * 32, smem, s>>>(m, a);
  INVOP_LAUNCHED(1);
  INVOP_CHECK_LAUNCH("k2_ordered");
  return INVOP_OK;
}

template <int P, bool SIGNED, bool SX, int KR>
static int launch_ord_t(const invop_plan* p, OrdArgs a, cudaStream_t s) {
  constexpr int NC = ord_nc(P);
  constexpr int S = ord_stages(P, KR), S2 = ord_stages2(P, KR);
  static_assert(S >= 2, "ordered kernel needs two stages");
  // More row blocks than SMs: shallower rings so that two blocks are resident
  // per SM (the second consumer on each scheduler fills the issue slots the
  // first leaves open; a single consumer is latency-bound on its DADD chain).
  if constexpr (S2 >= 2 && S2 < S) {
    // INVOP_ORD_DEEP: 1 one block per SM, 0 two blocks, 2 seven-consumer blocks
    const char* fe = std::getenv("INVOP_ORD_DEEP");
    const int force = fe && *fe ? atoi(fe) : -1;
    const int64_t blocks = cdiv(a.rows, NC * 32);
    if constexpr (P <= 2 && KR == 1) {
      // Still more than two blocks per SM: blocks of seven consumers (224
      // rows; two-stage rings of code tiles only, x read from global memory)
      // when that saves whole rounds of blocks — config 5: 512 blocks in two
      // rounds become 293 blocks in one.
      const int64_t slots = 2 * (int64_t)num_sms();
      const bool wide = a.xbulk && a.n % ORD_TILE == 0 && !a.accumulate &&
                        cdiv(cdiv(a.rows, 7 * 32), slots) < cdiv(blocks, slots);
      if (force == 2 || (force < 0 && wide)) {
        if (a.xbulk && a.n % ORD_TILE == 0)
          return launch_ord_s<P, SIGNED, SX, KR, 7, 2, true>(p, a, s);
      }
    }
    const bool two = force >= 0 ? force == 0 : blocks > num_sms();
    if (two) return launch_ord_s<P, SIGNED, SX, KR, NC, S2, false>(p, a, s);
  }
  return launch_ord_s<P, SIGNED, SX, KR, NC, S, false>(p, a, s);
}

template <int P, bool SIGNED, bool SX>
static int launch_ord_p(const invop_plan* p, OrdArgs a, int KR, cudaStream_t s) {
  if (KR >= 4 && P <= 4) return launch_ord_t<P, SIGNED, SX, 4>(p, a, s);
  if (KR >= 2) return launch_ord_t<P, SIGNED, SX, 2>(p, a, s);
  return launch_ord_t<P, SIGNED, SX, 1>(p, a, s);
}

int apply_ordered_launch(const invop_plan* p, const double* x, int64_t ldx, double* y,
                         int64_t ldy, int64_t nrhs, cudaStream_t s, bool accumulate) {
  if (p->rows == 0 || nrhs == 0) return INVOP_OK;
  int rc = INVOP_OK;
  // non-negative codes in signed planes decode identically as unsigned (the
  // cheaper coefficient path)
  const int sgn = p->is_signed && p->min_val < 0 ? 1 : 0;
  // 3-byte non-negative codes below 2^23: the sign-extending PRMT yields the
  // zero top byte without a mask
  const bool sx3 = !sgn && p->P == 3 && p->min_val >= 0 && p->max_val < (1 << 23);
  for (int64_t k0 = 0; k0 < nrhs;) {
    int KR = nrhs - k0 >= 4 && p->P <= 4 ? 4 : (nrhs - k0 >= 2 ? 2 : 1);
    OrdArgs a;
    a.rows = p->rows; a.n = p->n; a.scale = p->scale;
    a.neg_scale52 = -ldexp(p->scale, 52);
    a.x = x + k0 * ldx; a.ldx = ldx;
    a.y = y + k0 * ldy; a.ldy = ldy;
    a.accumulate = accumulate ? 1 : 0;
    a.xbulk = ((uintptr_t)a.x % 16 == 0) && (KR == 1 || ldx % 2 == 0) ? 1 : 0;
    static const int probe = std::getenv("INVOP_ORD_PROBE") ? atoi(std::getenv("INVOP_ORD_PROBE")) : 0;
    a.probe = probe;
    switch (p->P * 2 + sgn) {
      case 2: rc = launch_ord_p<1, false, false>(p, a, KR, s); break;
      case 3: rc = launch_ord_p<1, true, false>(p, a, KR, s); break;
      case 4: rc = launch_ord_p<2, false, false>(p, a, KR, s); break;
      case 5: rc = launch_ord_p<2, true, false>(p, a, KR, s); break;
      case 6: rc = sx3 ? launch_ord_p<3, false, true>(p, a, KR, s)
                       : launch_ord_p<3, false, false>(p, a, KR, s); break;
      case 7: rc = launch_ord_p<3, true, false>(p, a, KR, s); break;
      case 8: rc = launch_ord_p<4, false, false>(p, a, KR, s); break;
      case 9: rc = launch_ord_p<4, true, false>(p, a, KR, s); break;
      case 10: rc = launch_ord_p<5, false, false>(p, a, KR, s); break;
      case 11: rc = launch_ord_p<5, true, false>(p, a, KR, s); break;
      case 12: rc = launch_ord_p<6, false, false>(p, a, KR, s); break;
      case 13: rc = launch_ord_p<6, true, false>(p, a, KR, s); break;
      case 14: rc = launch_ord_p<7, false, false>(p, a, KR, s); break;
      case 15: rc = launch_ord_p<7, true, false>(p, a, KR, s); break;
      case 16: rc = launch_ord_p<8, false, false>(p, a, KR, s); break;
      default: rc = launch_ord_p<8, true, false>(p, a, KR, s); break;
    }
    if (rc) return rc;
    k0 += KR;
  }
  return INVOP_OK;
}

}  // namespace invop
