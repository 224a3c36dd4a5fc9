// K3 — batched multi-RHS apply on the 5th-generation tensor cores (sm_100a).
//
// Y[t, i] = 10^-m * sum_j v_ij x_tj for up to 64 right-hand sides t at once
// (the reference applies one vector at a time, applyplan.py:175-191; the
// multi-RHS contraction is new).
//
// Exact integer formulation on kind::i8 MMAs:
//   * each right-hand side t is converted to 23-bit fixed point
//     X_tj = rint(x_tj * 2^e_t), |X| < 2^22, and split into balanced base-256
//     digits X = d0 + 256 d1 + 65536 d2 with d_l in [-128, 127] (signed 8-bit);
//   * the codes are already byte planes: v = q0 + 256 q1 (q0 unsigned byte,
//     q1 signed or unsigned byte);
//   * v * X = sum_{p,l} q_p d_l 256^(p+l): every (plane, digit) pair is one
//     8-bit MMA, pairs of equal weight p+l share an int32 TMEM accumulator
//     (4 accumulators for 2-byte codes), and the epilogue combines
//     acc_0 + 256 acc_1 + 65536 acc_2 + 2^24 acc_3 exactly in int64.
//   The only rounding is x -> X (relative 2^-23 of max|x_t|) and the final
//   fp32 store; int32 accumulators cannot overflow because a work unit spans
//   at most 32768 columns (2 products of |q d| <= 32640 per column).
//
// Pipeline (one CTA per SM, warp-specialised, persistent over work units =
// pairs of 128-row tiles x K splits): warp 0 issues TMA loads of the A tiles
// (2 row tiles x P planes x 128 rows x 64 K-bytes, SWIZZLE_64B) and the B
// tile (3 digits x 64 RHS x 64 K-bytes) into a 4-stage mbarrier ring; warp 1
// (one elected thread) issues tcgen05.mma.cta_group::1.kind::i8 (M=128, N=64,
// K=32) into TMEM and commits each stage back to the producer; warps 2-5 drain
// TMEM with tcgen05.ld, combine the digit products and store Y (or add the
// exact int64 partial of a K split atomically). Both row tiles of a unit share
// every B tile in shared memory, halving the L2 re-reads of the digits.
#include "common.cuh"
#include <cuda.h>
#include <cooperative_groups.h>
#include <algorithm>
#include <cstring>
#include <cstdio>
#include <cstdlib>

namespace invop {

namespace cg = cooperative_groups;

static bool layout_flag(const char* env, bool dflt) {
  const char* v = getenv(env);
  if (!v || !*v) return dflt;
  return *v != '0';
}

// INVOP_K3_BULK=0: operand tiles stored row-major and swizzled by tensor
// copies (the round-1 form); default: stored pre-swizzled, 1-D bulk copies
static int k3_bulk_env() {
  static const int v = []() {
    const char* e = getenv("INVOP_K3_BULK");
    return e && *e == '0' ? 0 : 1;
  }();
  return v;
}

// INVOP_K3_BTILE=0: x digits row-major [192][ldb]; default: pre-swizzled tiles
static int k3_btile_env() {
  static const int v = []() {
    const char* e = getenv("INVOP_K3_BTILE");
    return e && *e == '0' ? 0 : 1;
  }();
  return v;
}

constexpr int K3_BM = 128;            // rows per MMA tile
constexpr int K3_TILES = 2;           // row tiles per work unit (share B)
constexpr int K3_BK = 64;             // K bytes per stage (SWIZZLE_64B row)
constexpr int K3_NR = 64;             // right-hand sides per MMA (N)
constexpr int K3_ND = 3;              // x digits
constexpr int K3_STAGES = 4;
#ifndef K3_DL_STAGES_OVERRIDE
constexpr int K3_DL_STAGES = 5;       // DL: 44 KB stages + a 4 KB zero B tile fit 5
#else
constexpr int K3_DL_STAGES = K3_DL_STAGES_OVERRIDE;
#endif
constexpr int K3_THREADS = 192;       // warp0 TMA, warp1 MMA+TMEM, warps 2-5 epilogue
constexpr int K3_KMAX = 32768;        // max columns per work unit (int32 safety)

constexpr int K3_A_TILE = K3_BM * K3_BK;              // 8 KB per plane per row tile
constexpr int K3_B_TILE = K3_NR * K3_BK;              // 4 KB per digit

struct K3Args {
  int64_t rows, n;
  int P, hi_signed;
  int kblocks_total;       // ceil(n / K3_BK)
  int kb_stride;           // tiles per row tile in the tiled planes (ld / K3_BK)
  int kblocks_per_unit;
  int splits;
  int64_t pairs;           // ceil(rows / (K3_TILES*K3_BM))
  int nrhs;
  long long* yacc;         // [64][rows] exact int64 row sums (DL: of the residuals)
  const int* idx1;         // DL: compact index of a tile's digit-1 plane, -1 if absent
  int ysh;                 // DL: tensor rows are 64 << ysh bytes wide (2: pre-swizzled tiles)
  int btile;               // x digits stored as pre-swizzled [K block][192][64] tiles
  // pre-swizzled tiles are contiguous images: plain bulk copies (no tensor map)
  const uint8_t* t0; const uint8_t* t1; const uint8_t* t2; const int8_t* B; int bulk;
};

__host__ __device__ inline int64_t k3d_tile0(int64_t rt, int64_t kb, int64_t kbs);

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void k3_mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void k3_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void k3_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void k3_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "K3W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra K3W_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                       uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void k3_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                        uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
// K-major operand tile, rows of 64 bytes, SWIZZLE_64B (8-row atoms of 512 B)
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);   // start address
  d |= (uint64_t)1 << 16;                    // leading byte offset (unused, swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;           // stride byte offset: 8 rows x 64 B
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;                    // layout: SWIZZLE_64B
  return d;
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(
          tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate), "r"(0), "r"(0), "r"(0), "r"(0));
}
// warp-wide issue: every lane executes (operands stay warp-uniform, so they
// live in uniform registers) and elect.sync picks the one issuing thread
__device__ __forceinline__ void mma_i8_elect(uint32_t tmem_d, uint64_t da, uint64_t db,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(
          tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate), "r"(0), "r"(0), "r"(0), "r"(0));
}
__device__ __forceinline__ void mma_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          bar)
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// kind::i8 instruction descriptor: D=s32, A u8/s8, B s8, both K-major
__host__ __device__ constexpr uint32_t idesc_i8(int a_signed, int n = K3_NR) {
  return (2u << 4) | ((uint32_t)a_signed << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(K3_BM >> 4) << 24);
}

// ------------------------------------------------------------ main kernel
// DL = true: A holds the balanced base-256 digits of second-order row
// residuals (both planes signed; the digit-1 plane of a tile is present only
// where a residual needs it, idx1 >= 0), and the epilogue writes the exact
// int64 D = E X for the double prefix sum along rows (k3d_scan).
template <int P, int TILES, int STAGES, bool DL>
__global__ void __launch_bounds__(K3_THREADS, 1)
    k3_batched(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapA1,
               const __grid_constant__ CUtensorMap mapA2, const __grid_constant__ CUtensorMap mapB,
               K3Args a) {
  constexpr int NACC = P + K3_ND - 1;                      // weights 0 .. P+1
  constexpr int A_BYTES = TILES * P * K3_A_TILE;
  constexpr int STAGE = A_BYTES + K3_ND * K3_B_TILE;
  extern __shared__ __align__(1024) unsigned char k3s[];
  unsigned char* base = (unsigned char*)(((uintptr_t)k3s + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull, tempty;
  __shared__ uint32_t tmem_slot;
  __shared__ uint32_t s_mask[STAGES];                       // DL: tiles whose digit-1 plane is loaded
  // DL: an all-zero operand tile after the stages (initialises the
  // accumulator that only digit-1 planes feed when the unit's first K block
  // has none): a B tile (4 KB) for the straight-line issue, an A tile otherwise
  constexpr int ZERO_BYTES = (P >= 2 && K3_ND == 3) ? K3_B_TILE : K3_A_TILE;
  unsigned char* zero_tile = base + (size_t)STAGES * STAGE;
  if (DL || P >= 2) {
    for (int i = threadIdx.x; i < ZERO_BYTES / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(zero_tile)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      k3_mbar_init(smem_u32(&full[i]), 1);
      k3_mbar_init(smem_u32(&empty[i]), 1);
    }
    k3_mbar_init(smem_u32(&tfull), 1);
    k3_mbar_init(smem_u32(&tempty), 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  asm volatile("griddepcontrol.wait;" ::: "memory");       // programmatic dependent of k3_digits
  const uint32_t tmem = tmem_slot;
  const int64_t units = a.pairs * a.splits;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      // the operator streams through L2 once (evict first); the x digits are
      // re-read by every row-tile pair and must stay L2-resident (evict last)
      uint64_t pol_a, pol_b;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_a));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_b));
      int st = 0;
      uint32_t ph = 0;
      int64_t it = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t pair = u / a.splits;
        const int split = (int)(u - pair * a.splits);
        const int kb0 = split * a.kblocks_per_unit;
        const int kb1 = min(a.kblocks_total, kb0 + a.kblocks_per_unit);
        const int row0 = (int)(pair * TILES * K3_BM);
        // rotated K order: concurrent CTAs read different x-digit tiles (a hot
        // L2 line shared by every SM serialises in one slice)
        const int nkb = kb1 - kb0, rot = (int)(blockIdx.x % nkb);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int kb = kb0 + (i + rot) % nkb;
          if (it >= STAGES) k3_wait(smem_u32(&empty[st]), ph ^ 1);
          const uint32_t sb = smem_u32(base + (size_t)st * STAGE);
          const uint32_t fb = smem_u32(&full[st]);
          if (DL) {
            int i1[TILES];
#ifdef K3_PROBE_NOB
            uint32_t mask = 0, bytes = TILES * K3_A_TILE;
#else
            uint32_t mask = 0, bytes = TILES * K3_A_TILE + K3_ND * K3_B_TILE;
#endif
#pragma unroll
            for (int ti = 0; ti < TILES; ++ti) {
              i1[ti] = a.idx1[(int64_t)(row0 / K3_BM + ti) * a.kb_stride + kb];
              if (i1[ti] >= 0) { mask |= 1u << ti; bytes += K3_A_TILE; }
            }
            s_mask[st] = mask;
#ifdef K3_PROBE_NOTMA
            k3_arrive(fb);
            if (++st == STAGES) { st = 0; ph ^= 1; }
            continue;
#endif
            k3_expect_tx(fb, bytes);
            if (P == 2 && TILES == 2) {
              // stage: [digit-0 tile 0][digit-0 tile 1][digit-1 tile 0][digit-1 tile 1]
              const int trow = (int)(k3d_tile0(row0 / K3_BM, kb, a.kb_stride) * K3_BM);
              if (a.bulk) {
                k3_bulk(sb, a.t0 + (int64_t)trow * K3_BK, 2 * K3_A_TILE, fb, pol_a);
#pragma unroll
                for (int ti = 0; ti < TILES; ++ti)
                  if (i1[ti] >= 0)
                    k3_bulk(sb + (TILES + ti) * K3_A_TILE, a.t1 + (int64_t)i1[ti] * K3_A_TILE,
                            K3_A_TILE, fb, pol_a);
              } else {
              tma_2d(sb, &mapA0, 0, trow >> a.ysh, fb, pol_a);         // both digit-0 tiles
#pragma unroll
              for (int ti = 0; ti < TILES; ++ti)
                if (i1[ti] >= 0)
                  tma_2d(sb + (TILES + ti) * K3_A_TILE, &mapA1, 0, (i1[ti] * K3_BM) >> a.ysh, fb, pol_a);
              }
            } else {
#pragma unroll
              for (int ti = 0; ti < TILES; ++ti) {
                const int trow = (int)(k3d_tile0(row0 / K3_BM + ti, kb, a.kb_stride) * K3_BM);
                tma_2d(sb + (ti * P + 0) * K3_A_TILE, &mapA0, 0, trow >> a.ysh, fb, pol_a);
                if (i1[ti] >= 0)
                  tma_2d(sb + (ti * P + 1) * K3_A_TILE, &mapA1, 0, (i1[ti] * K3_BM) >> a.ysh, fb, pol_a);
              }
            }
          } else {
            k3_expect_tx(fb, STAGE);
#pragma unroll
            for (int ti = 0; ti < TILES; ++ti) {
              // tiled planes: tile (rt, kb) starts at tensor row (rt*kblocks + kb)*128
              const int64_t tix = (int64_t)(row0 / K3_BM + ti) * a.kb_stride + kb;
              const int trow = (int)(tix * K3_BM);
              if (a.bulk) {
                k3_bulk(sb + (ti * P + 0) * K3_A_TILE, a.t0 + tix * K3_A_TILE, K3_A_TILE, fb, pol_a);
                if (P > 1) k3_bulk(sb + (ti * P + 1) * K3_A_TILE, a.t1 + tix * K3_A_TILE, K3_A_TILE, fb, pol_a);
                if (P > 2) k3_bulk(sb + (ti * P + 2) * K3_A_TILE, a.t2 + tix * K3_A_TILE, K3_A_TILE, fb, pol_a);
                continue;
              }
              tma_2d(sb + (ti * P + 0) * K3_A_TILE, &mapA0, 0, trow, fb, pol_a);
              if (P > 1) tma_2d(sb + (ti * P + 1) * K3_A_TILE, &mapA1, 0, trow, fb, pol_a);
              if (P > 2) tma_2d(sb + (ti * P + 2) * K3_A_TILE, &mapA2, 0, trow, fb, pol_a);
            }
          }
          // the three digit tiles are consecutive rows of B: one 192-row box
#ifndef K3_PROBE_NOB
          if (a.bulk)
            k3_bulk(sb + A_BYTES, a.B + (int64_t)kb * (K3_ND * K3_B_TILE), K3_ND * K3_B_TILE, fb, pol_b);
          else
            tma_2d(sb + A_BYTES, &mapB, a.btile ? 0 : kb * K3_BK,
                   a.btile ? kb * (K3_ND * K3_NR / 4) : 0, fb, pol_b);
#endif
          if (++st == STAGES) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    int st = 0;
    uint32_t ph = 0;
    int64_t ucount = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++ucount) {
      const int64_t pair = u / a.splits;
      const int split = (int)(u - pair * a.splits);
      const int kb0 = split * a.kblocks_per_unit;
      const int kb1 = min(a.kblocks_total, kb0 + a.kblocks_per_unit);
      if (ucount > 0) k3_wait(smem_u32(&tempty), (uint32_t)((ucount - 1) & 1));
      tc_fence_after();
      const int nkb = kb1 - kb0;
      for (int i = 0; i < nkb; ++i) {
        k3_wait(smem_u32(&full[st]), ph);
        tc_fence_after();
        {
          // descriptors: one base per stage plus compile-time offsets (>> 4)
          const uint32_t sb = smem_u32(base + (size_t)st * STAGE);
          const uint64_t dbase = desc_sw64(sb);
          const uint64_t dzero = desc_sw64(smem_u32(zero_tile));
          const uint32_t id_lo = idesc_i8(DL ? 1 : 0), id_hi = idesc_i8(DL ? 1 : a.hi_signed);
          const uint32_t mask = DL ? s_mask[st] : 0xffffffffu;
#ifdef K3_PROBE_NOMMA
          if (true) {
            (void)dbase; (void)id_lo; (void)id_hi; (void)mask;
          } else
#endif
          if constexpr (DL && P == 2 && K3_ND == 3) {
            // straight-line issue with N = 192: the three digit tiles of B
            // are contiguous in shared memory and the weight classes of a
            // tile are contiguous in TMEM (class w = plane + digit at column
            // 64 w), so plane 0 x all digits is ONE MMA into classes 0-2 and
            // plane 1 x all digits one MMA into classes 1-3 (a third of the
            // MMAs of the N = 64 form; the tensor core re-reads A per MMA).
            // Class 3 is started by a zero tile at the unit's first K block.
            const uint32_t id0 = idesc_i8(1, K3_ND * K3_NR);
#ifdef K3_MMA_ELECT_EACH
#pragma unroll
            for (int kk = 0; kk < K3_BK / 32; ++kk) {
              const uint32_t cont = (i > 0 || kk > 0) ? 1u : 0u;
              const uint64_t db = dbase + (uint64_t)((A_BYTES + kk * 32) >> 4);
#pragma unroll
              for (int ti = 0; ti < TILES; ++ti) {
                const uint32_t t0 = tmem + (uint32_t)(ti * NACC * K3_NR);
                const uint64_t a0 = dbase + (uint64_t)((ti * K3_A_TILE + kk * 32) >> 4);
                if (!cont)                                    // class 3 = A x 0
                  mma_i8_elect(t0 + 3 * K3_NR, a0, dzero + (uint64_t)((kk * 32) >> 4), id_hi, 0u);
                mma_i8_elect(t0, a0, db, id0, cont);
                if ((mask >> ti) & 1u) {                     // warp-uniform
                  const uint64_t a1 = dbase + (uint64_t)(((TILES + ti) * K3_A_TILE + kk * 32) >> 4);
                  mma_i8_elect(t0 + 1 * K3_NR, a1, db, id0, 1u);
                }
              }
            }
#else
            // one elected thread issues the whole stage (no per-MMA election)
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < K3_BK / 32; ++kk) {
                const uint32_t cont = (i > 0 || kk > 0) ? 1u : 0u;
                const uint64_t db = dbase + (uint64_t)((A_BYTES + kk * 32) >> 4);
#pragma unroll
                for (int ti = 0; ti < TILES; ++ti) {
                  const uint32_t t0 = tmem + (uint32_t)(ti * NACC * K3_NR);
                  const uint64_t a0 = dbase + (uint64_t)((ti * K3_A_TILE + kk * 32) >> 4);
                  if (!cont)                                  // class 3 = A x 0
                    mma_i8(t0 + 3 * K3_NR, a0, dzero + (uint64_t)((kk * 32) >> 4), id_hi, 0u);
                  mma_i8(t0, a0, db, id0, cont);
                  if ((mask >> ti) & 1u) {
                    const uint64_t a1 = dbase + (uint64_t)(((TILES + ti) * K3_A_TILE + kk * 32) >> 4);
                    mma_i8(t0 + 1 * K3_NR, a1, db, id0, 1u);
                  }
                }
              }
              mma_commit(smem_u32(&empty[st]));          // stage free once these MMAs complete
            }
            __syncwarp();
            if (++st == STAGES) { st = 0; ph ^= 1; }
            continue;
#endif
          } else if constexpr (!DL && P >= 2 && K3_ND == 3) {
            // byte planes, straight-line issue with N = 192: plane p x all
            // three digits is ONE MMA into the contiguous classes p .. p+2; at
            // a unit's first K step plane 0 starts classes 0-2 and a zero B
            // tile starts the class each further plane opens (p + 2).
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < K3_BK / 32; ++kk) {
                const uint32_t cont = (i > 0 || kk > 0) ? 1u : 0u;
                const uint64_t db = dbase + (uint64_t)((A_BYTES + kk * 32) >> 4);
#pragma unroll
                for (int ti = 0; ti < TILES; ++ti) {
                  const uint32_t t0 = tmem + (uint32_t)(ti * NACC * K3_NR);
#pragma unroll
                  for (int p = 0; p < P; ++p) {
                    const int sg = (p == P - 1) ? a.hi_signed : 0;
                    const uint64_t ap = dbase + (uint64_t)(((ti * P + p) * K3_A_TILE + kk * 32) >> 4);
                    if (!cont && p >= 1)
                      mma_i8(t0 + (uint32_t)((p + 2) * K3_NR), ap, dzero + (uint64_t)((kk * 32) >> 4),
                             idesc_i8(sg), 0u);
                    mma_i8(t0 + (uint32_t)(p * K3_NR), ap, db, idesc_i8(sg, K3_ND * K3_NR),
                           p == 0 ? cont : 1u);
                  }
                }
              }
              mma_commit(smem_u32(&empty[st]));          // stage free once these MMAs complete
            }
            __syncwarp();
            if (++st == STAGES) { st = 0; ph ^= 1; }
            continue;
          } else
#pragma unroll
          for (int kk = 0; kk < K3_BK / 32; ++kk) {
#pragma unroll
            for (int ti = 0; ti < TILES; ++ti) {
              const bool have1 = (mask >> ti) & 1u;          // warp-uniform
#pragma unroll
              for (int w = 0; w < NACC; ++w) {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                  const int l = w - p;
                  if (l < 0 || l >= K3_ND) continue;
                  // first product of weight w at the unit's first K step starts the accumulator
                  const bool first_pair = (p == (w < K3_ND ? 0 : w - K3_ND + 1));
                  const uint32_t acc = (i > 0 || kk > 0 || !first_pair) ? 1u : 0u;
                  uint64_t da = dbase + (uint64_t)(((ti * P + p) * K3_A_TILE + kk * 32) >> 4);
                  if (DL && p == 1 && !have1) {
                    // plane absent: only the accumulator start it owns is needed
                    if (acc) continue;
                    da = dzero + (uint64_t)((kk * 32) >> 4);
                  }
                  const uint64_t db = dbase + (uint64_t)((A_BYTES + l * K3_B_TILE + kk * 32) >> 4);
                  mma_i8_elect(tmem + (uint32_t)((ti * NACC + w) * K3_NR), da, db,
                               (p == P - 1) ? id_hi : id_lo, acc);
                }
              }
            }
          }
#ifdef K3_PROBE_NOMMA
          if (lane == 0) k3_arrive(smem_u32(&empty[st]));
#else
          mma_commit_elect(smem_u32(&empty[st]));   // stage free once these MMAs complete
#endif
        }
        __syncwarp();
        if (++st == STAGES) { st = 0; ph ^= 1; }
      }
#ifdef K3_PROBE_NOMMA
      if (lane == 0) k3_arrive(smem_u32(&tfull));
#else
      mma_commit_elect(smem_u32(&tfull));
#endif
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                  // TMEM lane quarter of this warp
    int64_t ucount = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++ucount) {
      const int64_t pair = u / a.splits;
      k3_wait(smem_u32(&tfull), (uint32_t)(ucount & 1));
      tc_fence_after();
#ifdef K3_PROBE_NOEPI
      if (true) {} else
#endif
#pragma unroll 1
      for (int ti = 0; ti < TILES; ++ti) {
        const int64_t row = pair * TILES * K3_BM + ti * K3_BM + q * 32 + lane;
#pragma unroll 1
        for (int c0 = 0; c0 < K3_NR; c0 += 16) {
          int32_t r[NACC][16];
#pragma unroll
          for (int w = 0; w < NACC; ++w)
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((ti * NACC + w) * K3_NR + c0),
                      r[w]);
          tmem_wait_ld();
          if (row < a.rows) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int t = c0 + j;
              if (t >= a.nrhs) break;
              long long v = 0;
#pragma unroll
              for (int w = 0; w < NACC; ++w) v += (long long)r[w][j] * (1LL << (8 * w));
              if (a.splits == 1) {
                a.yacc[(int64_t)t * a.rows + row] = v;
              } else {
                atomicAdd((unsigned long long*)&a.yacc[(int64_t)t * a.rows + row],
                          (unsigned long long)v);
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) k3_arrive(smem_u32(&tempty));
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ------------------------------------------------------------ tiled planes
// K3 streams 128-row x 64-column tiles. In the row-major planes a tile is 128
// separate 64-byte pieces (one per row, ld bytes apart): every TMA box then
// touches 128 DRAM pages. The tensor-core path therefore reads a tiled copy of
// the planes, built once per plan: tile (rt, kb) = rows [128 rt, 128 rt+128) x
// columns [64 kb, 64 kb+64) stored as one contiguous 8 KB block, tiles of a row
// tile consecutive along K, so a row tile's whole K range is one contiguous run.
// presw: 16-byte chunks stored where the 64-byte shared-memory swizzle puts
// them (the tile is then moved by one 1-D bulk copy).
__global__ void k3_tile_planes(const uint8_t* __restrict__ in, int64_t rows, int64_t ld,
                               uint8_t* __restrict__ out, int64_t rtiles, int presw) {
  const int64_t kbt = ld / K3_BK;
  const int64_t total16 = rtiles * kbt * (K3_A_TILE / 16);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total16;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = k / (K3_A_TILE / 16);
    const int within = (int)(k - tile * (K3_A_TILE / 16));
    const int r = within >> 2, c16 = within & 3;
    const int64_t rt = tile / kbt, kb = tile - rt * kbt;
    const int64_t row = rt * K3_BM + r;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < rows) v = *reinterpret_cast<const uint4*>(in + row * ld + kb * K3_BK + c16 * 16);
    const int cs = presw ? (c16 ^ ((r >> 1) & 3)) : c16;
    *reinterpret_cast<uint4*>(out + tile * K3_A_TILE + r * K3_BK + cs * 16) = v;
  }
}

// ------------------------------------------------------------ x preparation
// Two single-phase kernels (no cluster barriers; a programmatic dependent
// launch chain hides the boundary), grid (column chunks, 64 right-hand sides):
//  k3_xmax: max |x_tj| over the finite entries -> atomicMax on the float bits
//    (maxbits[t], non-negative floats order like their bits); columns whose x
//    is inf/nan are listed instead (nf_cols[t][.]): the reference skips zero
//    mantissas (_native.pyx:32-46), so those columns are applied exactly by
//    k3_post and enter the digits as 0;
//  k3_digits: e_t (max|x_t| 2^e_t < 2^22) and the balanced base-256 digits of
//    X = rint(x 2^e_t) into B[l][t][j] (int8), 16 columns per thread, three
//    16-byte stores; right-hand sides t >= nrhs get zeros. DL: plan rows 0
//    and 1 are stored as zero residuals; their exact sums Y_0, Y_1 come from
//    the byte-plane codes and the same X (16-byte plane loads beside the
//    digits), added atomically into y01[t] (k3_post folds them into D_0, D_1).
// maxbits, nf_count and y01 are zero on entry: k3_post resets them.
constexpr int K3X_COLS = 8192;        // columns per k3_xmax CTA
constexpr int K3X_TPB = 256;
constexpr int K3G_TPB = 256;          // k3_digits: 16 columns per thread
constexpr int K3G_COLS = K3G_TPB * 16;

struct K3Prep {
  const float* x;
  int64_t n, ldx;
  int nrhs;
  int8_t* B;
  int64_t ldb;
  int* e;
  unsigned int* maxbits;      // [64]
  int* nf_count;
  int* nf_cols;
  const uint8_t* planes[2];   // rows 0/1 codes (DL)
  int64_t ld, rows;
  int P, sgn, rows01;
  unsigned long long* y01;    // [64][2] exact sums of plan rows 0, 1 (DL)
  // B as [K block][192 rows][64 bytes] tiles, each row's 16-byte chunks where
  // the 64-byte shared-memory swizzle puts them (a contiguous image of the
  // operand tile: copied as 256-byte rows); 0: row-major [192][ldb]
  int btile;
};

__device__ __forceinline__ int k3_exponent(float m) {
  int ex = 0;
  if (m > 0.0f && isfinite(m)) frexpf(m, &ex);
  return (m > 0.0f && isfinite(m)) ? 22 - ex : 0;   // max|x_t| * 2^e_t < 2^22
}

__device__ __forceinline__ int32_t k3_code16(uint32_t lo, uint32_t hi, int bb, int P, int sgn) {
  uint32_t u = (lo >> bb) & 255u;
  if (P > 1) u |= ((hi >> bb) & 255u) << 8;
  const int sh = 32 - 8 * P;
  return sgn ? ((int32_t)(u << sh) >> sh) : (int32_t)u;
}

__global__ void __launch_bounds__(K3X_TPB) k3_xmax(K3Prep a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");       // x may be the previous apply's y
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ float s_warp[K3X_TPB / 32];
  const int t = blockIdx.y;
  if (t >= a.nrhs) return;
  const float* xt = a.x + (int64_t)t * a.ldx;
  const int64_t j0 = (int64_t)blockIdx.x * K3X_COLS, j1 = min(a.n, j0 + K3X_COLS);
  float m = 0.0f;
  const bool vec = ((((uintptr_t)xt) | (uintptr_t)(a.ldx * 4)) & 15) == 0;
  if (vec) {
    // all of the thread's loads first (coalesced 16-byte loads, 8 in flight),
    // then the scan: an atomic in the load loop would serialise the loads
    constexpr int U = K3X_COLS / (4 * K3X_TPB);
    float4 f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + 4 * ((int64_t)threadIdx.x + (int64_t)u * K3X_TPB);
      if (j + 4 <= j1) {
        f[u] = *reinterpret_cast<const float4*>(xt + j);
      } else {
        f[u].x = j < j1 ? xt[j] : 0.0f;
        f[u].y = j + 1 < j1 ? xt[j + 1] : 0.0f;
        f[u].z = j + 2 < j1 ? xt[j + 2] : 0.0f;
        f[u].w = j + 3 < j1 ? xt[j + 3] : 0.0f;
      }
    }
    bool bad = false;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float v[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        bad |= !isfinite(v[i]);
        m = fmaxf(m, isfinite(v[i]) ? fabsf(v[i]) : 0.0f);
      }
    }
    if (bad) {                       // rare: list the non-finite columns
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float v[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
        const int64_t j = j0 + 4 * ((int64_t)threadIdx.x + (int64_t)u * K3X_TPB);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (!isfinite(v[i]) && j + i < j1) {
            const int k = atomicAdd(&a.nf_count[t], 1);
            a.nf_cols[(int64_t)t * a.n + k] = (int)(j + i);
          }
      }
    }
  } else {
    for (int64_t j = j0 + threadIdx.x; j < j1; j += K3X_TPB) {
      const float v = xt[j];
      if (isfinite(v)) {
        m = fmaxf(m, fabsf(v));
      } else {
        const int k = atomicAdd(&a.nf_count[t], 1);
        a.nf_cols[(int64_t)t * a.n + k] = (int)j;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = 0.0f;
#pragma unroll
    for (int w = 0; w < K3X_TPB / 32; ++w) v = fmaxf(v, s_warp[w]);
    atomicMax(&a.maxbits[t], __float_as_uint(v));
  }
}

__global__ void __launch_bounds__(K3G_TPB, 6) k3_digits(K3Prep a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");       // k3_xmax complete
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ long long s_w01[K3G_TPB / 32][2];
  const int t = blockIdx.y;
  const bool live = t < a.nrhs;
  const float* xt = a.x + (int64_t)t * a.ldx;
  const int et = live ? k3_exponent(__uint_as_float(a.maxbits[t])) : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.e[t] = et;
  // 2^e_t as two float factors (e_t may exceed 127 for tiny x): x * 2^e_t is
  // exact for the in-range products, the same value ldexpf returns
  const int e1 = et > 126 ? 126 : (et < -126 ? -126 : et), e2 = et - e1;
  const float f1 = __int_as_float((127 + e1) << 23), f2 = __int_as_float((127 + e2) << 23);
  const int64_t jb = (int64_t)blockIdx.x * K3G_COLS + (int64_t)threadIdx.x * 16;
  long long s0 = 0, s1 = 0;
  if (jb < a.ldb) {
    float xv[16];
    if (live && jb + 16 <= a.n && (((uintptr_t)(xt + jb)) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 16; i += 4) {
        const float4 f = *reinterpret_cast<const float4*>(xt + jb + i);
        xv[i] = f.x; xv[i + 1] = f.y; xv[i + 2] = f.z; xv[i + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) xv[i] = (live && jb + i < a.n) ? xt[jb + i] : 0.0f;
    }
    int X[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) X[i] = isfinite(xv[i]) ? __float2int_rn((xv[i] * f1) * f2) : 0;
    uint32_t w[3][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t b0 = 0, b1 = 0, b2 = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int Xv = X[4 * q + i];
        const int d0 = ((Xv + 128) & 255) - 128;
        const int X1 = (Xv - d0) >> 8;
        const int d1 = ((X1 + 128) & 255) - 128;
        const int d2 = (X1 - d1) >> 8;
        b0 |= ((uint32_t)d0 & 255u) << (8 * i);
        b1 |= ((uint32_t)d1 & 255u) << (8 * i);
        b2 |= ((uint32_t)d2 & 255u) << (8 * i);
      }
      w[0][q] = b0; w[1][q] = b1; w[2][q] = b2;
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const int row = l * K3_NR + t;
      int8_t* dst = a.btile ? a.B + (jb / K3_BK) * (int64_t)(K3_ND * K3_NR * K3_BK) + row * K3_BK +
                                  (((int)((jb % K3_BK) >> 4) ^ ((row >> 1) & 3)) << 4)
                            : a.B + (int64_t)row * a.ldb + jb;
      *reinterpret_cast<uint4*>(dst) = make_uint4(w[l][0], w[l][1], w[l][2], w[l][3]);
    }
    if (a.rows01 && live) {
      // plane rows are ld >= ldb bytes with zero padding: 16-byte loads
      const uint4 p00 = *reinterpret_cast<const uint4*>(a.planes[0] + jb);
      const uint4 p01 = *reinterpret_cast<const uint4*>(a.planes[1] + jb);
      const bool two = a.rows > 1;
      const uint4 p10 = two ? *reinterpret_cast<const uint4*>(a.planes[0] + a.ld + jb) : make_uint4(0, 0, 0, 0);
      const uint4 p11 = two ? *reinterpret_cast<const uint4*>(a.planes[1] + a.ld + jb) : make_uint4(0, 0, 0, 0);
      const uint32_t A0[4] = {p00.x, p00.y, p00.z, p00.w}, A1[4] = {p01.x, p01.y, p01.z, p01.w};
      const uint32_t B0[4] = {p10.x, p10.y, p10.z, p10.w}, B1[4] = {p11.x, p11.y, p11.z, p11.w};
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int q = i >> 2, bb = 8 * (i & 3);
        s0 += (long long)k3_code16(A0[q], A1[q], bb, a.P, a.sgn) * X[i];
        s1 += (long long)k3_code16(B0[q], B1[q], bb, a.P, a.sgn) * X[i];
      }
    }
  }
  if (a.rows01 && live) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if ((threadIdx.x & 31) == 0) { s_w01[threadIdx.x >> 5][0] = s0; s_w01[threadIdx.x >> 5][1] = s1; }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long v0 = 0, v1 = 0;
#pragma unroll
      for (int w = 0; w < K3G_TPB / 32; ++w) { v0 += s_w01[w][0]; v1 += s_w01[w][1]; }
      atomicAdd(&a.y01[2 * t], (unsigned long long)v0);
      atomicAdd(&a.y01[2 * t + 1], (unsigned long long)v1);
    }
  }
}

// cluster barrier halves: arrive without a release fence (only register or
// shared-memory state the peers already consumed is involved) / wait
__device__ __forceinline__ void k3_cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void k3_cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// ------------------------------------------------------------ K3 on row residuals
// Residual of plan row r (plan-local): e_r = v_r - 2 v_{r-1} + v_{r-2} for
// r >= 2; rows 0 and 1 are stored as zero and their sums computed exactly from
// the codes (k3d_rows01), so D_0 = Y_0, D_1 = Y_1 - 2 Y_0 and Y is the double
// prefix sum of D along rows (k3d_scan). Digits are balanced base-256.
__device__ __forceinline__ int32_t k3d_code(const uint8_t* const* planes, int P, int sgn,
                                            int64_t off) {
  uint32_t u = 0;
  for (int b = 0; b < P; ++b) u |= (uint32_t)planes[b][off] << (8 * b);
  const int sh = 32 - 8 * P;
  return sgn ? ((int32_t)(u << sh) >> sh) : (int32_t)u;
}

struct K3DBuild {
  const uint8_t* planes[2];
  int P, sgn;
  int64_t rows, ld;
  int64_t kbs, rtiles;
};

// digit-0 tiles: the two row tiles of a pair at the same K block are adjacent,
// so one 256-row TMA box loads both
__host__ __device__ inline int64_t k3d_tile0(int64_t rt, int64_t kb, int64_t kbs) {
  return ((rt >> 1) * kbs + kb) * 2 + (rt & 1);
}

__device__ __forceinline__ int32_t k3d_resid(const K3DBuild& a, int64_t r, int64_t j) {
  if (r < 2 || r >= a.rows) return 0;
  const int64_t off = r * a.ld + j;
  return k3d_code(a.planes, a.P, a.sgn, off) - 2 * k3d_code(a.planes, a.P, a.sgn, off - a.ld) +
         k3d_code(a.planes, a.P, a.sgn, off - 2 * a.ld);
}

// one thread per (row, K block): digit count of its 64 residuals -> tile max
__global__ void k3d_width(K3DBuild a, int* __restrict__ tilew, int* __restrict__ wmax) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= a.rows * a.kbs) return;
  const int64_t r = t / a.kbs, kb = t - r * a.kbs;
  int w = 1;
  for (int q = 0; q < K3_BK; ++q) {
    int32_t e = k3d_resid(a, r, kb * K3_BK + q);
    int n = 1;
    for (;;) {
      const int32_t d = ((e + 128) & 255) - 128;
      e = (e - d) >> 8;
      if (e == 0) break;
      ++n;
    }
    w = max(w, n);
  }
  atomicMax(&tilew[(r / K3_BM) * a.kbs + kb], w);
  atomicMax(wmax, w);
}

// compact index of the tiles that need a digit-1 plane (one block)
__global__ void k3d_index(int64_t tiles, const int* __restrict__ tilew, int* __restrict__ idx1,
                          int64_t* __restrict__ n1) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int64_t per = (tiles + T - 1) / T;
  const int64_t a0 = t * per, a1 = min(tiles, a0 + per);
  int64_t c = 0;
  for (int64_t i = a0; i < a1; ++i) c += tilew[i] >= 2;
  part[t] = c;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int i = 0; i < T; ++i) { const int64_t v = part[i]; part[i] = acc; acc += v; }
    *n1 = acc;
  }
  __syncthreads();
  int64_t acc = part[t];
  for (int64_t i = a0; i < a1; ++i) idx1[i] = tilew[i] >= 2 ? (int)acc++ : -1;
}

// one thread per (row, K block): write the residual digits into the tiles
// presw: the 16-byte chunks of a tile row are stored where the 64-byte
// shared-memory swizzle puts them (chunk c of row r at c ^ ((r >> 1) & 3)), so
// a tile is a contiguous image of its shared-memory form and the copy engine
// moves it as wide unswizzled rows
__global__ void k3d_write(K3DBuild a, const int* __restrict__ idx1, uint8_t* __restrict__ t0,
                          uint8_t* __restrict__ t1, int presw) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= a.rows * a.kbs) return;
  const int64_t r = t / a.kbs, kb = t - r * a.kbs;
  const int64_t tile = (r / K3_BM) * a.kbs + kb;
  const int i1 = idx1[tile];
  uint8_t* d0 = t0 + k3d_tile0(r / K3_BM, kb, a.kbs) * K3_A_TILE + (r % K3_BM) * K3_BK;
  uint8_t* d1 = i1 >= 0 ? t1 + (int64_t)i1 * K3_A_TILE + (r % K3_BM) * K3_BK : nullptr;
  for (int q0 = 0; q0 < K3_BK; q0 += 16) {
    uint32_t w0[4] = {0, 0, 0, 0}, w1[4] = {0, 0, 0, 0};
    for (int q = 0; q < 16; ++q) {
      const int32_t e = k3d_resid(a, r, kb * K3_BK + q0 + q);
      const int32_t g0 = ((e + 128) & 255) - 128;
      const int32_t g1 = (e - g0) >> 8;
      w0[q >> 2] |= ((uint32_t)g0 & 255u) << (8 * (q & 3));
      w1[q >> 2] |= ((uint32_t)g1 & 255u) << (8 * (q & 3));
    }
    const int qs = presw ? (((q0 >> 4) ^ (int)(((r % K3_BM) >> 1) & 3)) << 4) : q0;
    *reinterpret_cast<uint4*>(d0 + qs) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
    if (d1) *reinterpret_cast<uint4*>(d1 + qs) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
  }
}

// ------------------------------------------------------------ k3_post
// From the exact int64 row sums the tensor-core pass accumulated in yacc to
// fp32 y; one cluster of K3Q_CL CTAs per right-hand side (grid (K3Q_CL, nrhs)),
// each CTA a contiguous block of rows in tiles of K3Q_TILE. Global memory is
// touched only by coalesced row-strided accesses; a padded shared-memory
// transpose gives every thread K3Q_RPT consecutive rows for the scans.
//  * DL: yacc holds D = E X for the second-order row residuals (+ k3_digits's
//    rows 0/1 corrections). Y is the double prefix sum of D along rows: per
//    tile two block scans (thread sums of d, then of the thread-local second
//    prefix), each CTA publishes (sum D, sum z, length) in shared memory and
//    folds its predecessors' triples (DSMEM) into its carry-in
//    (composition of consecutive blocks A, B: sumZ = sumZ_A + sumZ_B +
//    len_B sumD_A);
//  * byte planes: yacc holds Y itself;
//  * y = fl32(Y 10^-m 2^-e_t); columns whose x is inf/nan (k3_xmax's list)
//    are applied as the reference loop would (zero mantissas skipped): nan if
//    any non-zero v_ij meets a nan or both infinite signs occur, else +-inf;
//  * yacc is reset to zero behind the read, ready for the next apply's
//    atomic K-split partials (no memset launch).
constexpr int K3Q_CL = 16;             // non-portable cluster size (opt-in at launch)
constexpr int K3Q_TPB = 256;
constexpr int K3Q_RPT = 16;
constexpr int K3Q_TILE = K3Q_TPB * K3Q_RPT;
constexpr int K3Q_SMEM = K3Q_TILE + K3Q_TILE / 16;   // 8-byte words, one pad per 16

__device__ __forceinline__ int k3q_pad(int k) { return k + (k >> 4); }

struct K3Post {
  long long* yacc;
  int64_t rows, n, ld;
  const uint8_t* planes[3];
  int P, sgn;
  const int* e;
  double scale;
  int* nf_count;
  const int* nf_cols;
  long long* y01;                 // k3_digits's exact sums of plan rows 0, 1 (reset here)
  unsigned int* maxbits;          // k3_xmax's max|x_t| bits (reset here)
  const float* x;
  int64_t ldx;
  float* y;
  int64_t ldy;
};

__device__ __forceinline__ long long k3q_block_excl(long long v, long long* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    long long s = lane < K3Q_TPB / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += u;
    }
    sh[lane] = s;
  }
  __syncthreads();
  const long long r = inc - v + (w > 0 ? sh[w - 1] : 0);
  __syncthreads();
  return r;
}

// tile s (L valid rows) -> d[]: coalesced row-strided loads into padded
// shared memory, then this thread's K3Q_RPT consecutive rows
__device__ __forceinline__ void k3q_load(const K3Post& a, int t, int64_t s, int64_t L,
                                         long long add0, long long add1, long long* d,
                                         long long* sd) {
  const long long* src = a.yacc + (int64_t)t * a.rows + s;
#pragma unroll
  for (int i = 0; i < K3Q_RPT; ++i) {
    const int k = i * K3Q_TPB + threadIdx.x;
    long long v = k < L ? src[k] : 0;
    if (s + k == 0) v += add0;          // plan rows 0 and 1 (DL corrections; 0 otherwise)
    if (s + k == 1) v += add1;
    sd[k3q_pad(k)] = v;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < K3Q_RPT; ++i) d[i] = sd[k3q_pad(threadIdx.x * K3Q_RPT + i)];
  __syncthreads();
}

// d[] -> the thread's exclusive block prefixes: ze (first prefix) and we
// (second prefix, relative to the tile start); tile sums via the thread
// holding the tile's last valid row
__device__ __forceinline__ void k3q_scan(const long long* d, int64_t L, long long* sh,
                                         long long* s_tile, long long& ze, long long& we,
                                         long long& sD, long long& sZ) {
  long long S = 0, C = 0;
#pragma unroll
  for (int i = 0; i < K3Q_RPT; ++i) { S += d[i]; C += S; }
  ze = k3q_block_excl(S, sh);
  const long long W = (long long)K3Q_RPT * ze + C;   // sum of the thread's second prefix
  we = k3q_block_excl(W, sh);
  const int64_t last = L - 1;
  if ((int64_t)threadIdx.x == last / K3Q_RPT) {
    const int il = (int)(last % K3Q_RPT);
    long long cs = 0, cc = 0;
#pragma unroll
    for (int i = 0; i < K3Q_RPT; ++i) {
      cs += d[i];
      cc += ze + cs;
      if (i == il) { s_tile[0] = ze + cs; s_tile[1] = we + cc; }
    }
  }
  __syncthreads();
  sD = s_tile[0];
  sZ = s_tile[1];
  __syncthreads();
}

// Y of the thread's rows (running prefixes from base_z / base_y) -> fp32 in
// shared memory -> coalesced stores of y and zeros into yacc
template <bool DL>
__device__ __forceinline__ void k3q_store(const K3Post& a, int t, int64_t s, int64_t L,
                                          const long long* d, long long base_z, long long base_y,
                                          double sc, float* sy) {
  long long z = base_z, yv = base_y;
#pragma unroll
  for (int i = 0; i < K3Q_RPT; ++i) {
    long long Y;
    if (DL) { z += d[i]; yv += z; Y = yv; } else { Y = d[i]; }
    sy[k3q_pad(threadIdx.x * K3Q_RPT + i)] = (float)((double)Y * sc);
  }
  __syncthreads();
  float* dst = a.y + (int64_t)t * a.ldy + s;
  long long* acc = a.yacc + (int64_t)t * a.rows + s;
#pragma unroll
  for (int i = 0; i < K3Q_RPT; ++i) {
    const int k = i * K3Q_TPB + threadIdx.x;
    if (k < L) {
      dst[k] = sy[k3q_pad(k)];
      acc[k] = 0;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float k3q_nonfinite(const K3Post& a, int t, int64_t r, float v, int nf) {
  bool isn = false, pos = false, neg = false;
  for (int k = 0; k < nf; ++k) {
    const int64_t j = a.nf_cols[(int64_t)t * a.n + k];
    const int64_t off = r * a.ld + j;
    uint32_t u = a.planes[0][off];
    if (a.P > 1) u |= (uint32_t)a.planes[1][off] << 8;
    if (a.P > 2) u |= (uint32_t)a.planes[2][off] << 16;
    const int sh = 32 - 8 * a.P;
    const int32_t q = a.sgn ? ((int32_t)(u << sh) >> sh) : (int32_t)u;
    if (q == 0) continue;
    const float xv = a.x[(int64_t)t * a.ldx + j];
    if (isnan(xv)) isn = true;
    else if ((q < 0) != (xv < 0.0f)) neg = true;
    else pos = true;
  }
  if (isn || (pos && neg)) return __int_as_float(0x7fc00000);
  if (pos) return __int_as_float(0x7f800000);
  if (neg) return __int_as_float(0xff800000);
  return v;
}

// columns with inf/nan x (rare): after the CTA's rows are stored
__device__ __forceinline__ void k3q_fix_nonfinite(const K3Post& a, int t, int64_t r0, int64_t r1,
                                                  int nf) {
  __syncthreads();
  for (int64_t r = r0 + threadIdx.x; r < r1; r += K3Q_TPB) {
    float* dst = a.y + (int64_t)t * a.ldy + r;
    *dst = k3q_nonfinite(a, t, r, *dst, nf);
  }
}

template <bool DL>
__global__ void __launch_bounds__(K3Q_TPB, 4) k3_post(K3Post a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");       // the tensor-core pass is complete
  asm volatile("griddepcontrol.launch_dependents;");
  cg::cluster_group cl = cg::this_cluster();
  __shared__ long long sd[K3Q_SMEM];
  __shared__ long long sh[32];
  __shared__ long long s_tile[2];
  __shared__ long long s_tot[3];
  __shared__ long long s_carry[2];
  float* sy = reinterpret_cast<float*>(sd);
  const int t = blockIdx.y;
  const int c = (int)cl.block_rank();
  const int64_t per = cdiv(a.rows, K3Q_CL);
  const int64_t r0 = min(a.rows, (int64_t)c * per), r1 = min(a.rows, r0 + per);
  const long long add0 = DL ? a.y01[2 * t] : 0;
  const long long add1 = DL ? a.y01[2 * t + 1] - 2 * a.y01[2 * t] : 0;   // D_1 += Y_1 - 2 Y_0
  if (c == 0 && threadIdx.x == 0) a.maxbits[t] = 0;     // read by k3_digits only (complete)
  const double sc = ldexp(a.scale, -a.e[t]);
  const int nf = a.nf_count[t];
  long long d[K3Q_RPT];
  if (!DL) {
    for (int64_t s = r0; s < r1; s += K3Q_TILE) {
      const int64_t L = min((int64_t)K3Q_TILE, r1 - s);
      k3q_load(a, t, s, L, 0, 0, d, sd);
      k3q_store<false>(a, t, s, L, d, 0, 0, sc, sy);
    }
    if (nf > 0) {
      k3q_fix_nonfinite(a, t, r0, r1, nf);
      cl.sync();                     // every CTA has read nf_count[t]
      if (c == 0 && threadIdx.x == 0) a.nf_count[t] = 0;
    }
    return;
  }
  const bool one = r1 - r0 <= K3Q_TILE;          // the rows stay in registers
  long long ze = 0, we = 0, sD = 0, sZ = 0;
  long long SD = 0, SZ = 0;
  for (int64_t s = r0; s < r1; s += K3Q_TILE) {
    const int64_t L = min((int64_t)K3Q_TILE, r1 - s);
    k3q_load(a, t, s, L, add0, add1, d, sd);
    k3q_scan(d, L, sh, s_tile, ze, we, sD, sZ);
    SZ += sZ + L * SD;
    SD += sD;
  }
  if (threadIdx.x == 0) { s_tot[0] = SD; s_tot[1] = SZ; s_tot[2] = r1 - r0; }
  cl.sync();
  // lane r of warp 0 reads the triple of peer r < c (parallel DSMEM loads);
  // lane 0 folds them in rank order
  if (threadIdx.x < 32) {
    long long pd = 0, pz = 0, pl = 0;
    if ((int)threadIdx.x < c) {
      const long long* p = cl.map_shared_rank(s_tot, (int)threadIdx.x);
      pd = p[0];
      pz = p[1];
      pl = p[2];
    }
    long long zi = 0, yi = 0;
    for (int r = 0; r < c; ++r) {
      const long long d_ = __shfl_sync(0xffffffffu, pd, r);
      const long long z_ = __shfl_sync(0xffffffffu, pz, r);
      const long long l_ = __shfl_sync(0xffffffffu, pl, r);
      yi += l_ * zi + z_;
      zi += d_;
    }
    if (threadIdx.x == 0) { s_carry[0] = zi; s_carry[1] = yi; }
  }
  k3_cluster_arrive_relaxed();     // this CTA is done reading its peers
  __syncthreads();
  long long Zin = s_carry[0], Yin = s_carry[1];
  for (int64_t s = r0; s < r1; s += K3Q_TILE) {
    const int64_t L = min((int64_t)K3Q_TILE, r1 - s);
    if (!one) {
      k3q_load(a, t, s, L, add0, add1, d, sd);
      k3q_scan(d, L, sh, s_tile, ze, we, sD, sZ);
    }
    // row s + off + i: Z = Zin + ze + cs_i, Y = Yin + (off + i + 1) Zin + we + sum_{i'<=i} (ze + cs_i')
    const int64_t off = (int64_t)threadIdx.x * K3Q_RPT;
    k3q_store<true>(a, t, s, L, d, Zin + ze, Yin + off * Zin + we, sc, sy);
    Yin += L * Zin + sZ;
    Zin += sD;
  }
  if (nf > 0) k3q_fix_nonfinite(a, t, r0, r1, nf);
  k3_cluster_wait();               // peers read s_tot through DSMEM until here
  if (c == 0 && threadIdx.x == 0) {  // every CTA read these above
    if (nf > 0) a.nf_count[t] = 0;
    a.y01[2 * t] = 0;
    a.y01[2 * t + 1] = 0;
  }
}

// ------------------------------------------------------------ DL kernel on SM pairs
// k3_dl2: the residual-tile apply with tcgen05.mma.cta_group::2 (config 5's
// route). Probes of the one-SM kernel (k3_batched<2,2,5,true>) put it at
// 0.92 ms while the TMA pipeline alone streams in 0.77 ms and the MMAs alone
// (real operand addresses) take 0.66 ms: the two share the SM's shared
// memory, and every N = 192 MMA re-reads the 6 KB x-digit operand for each
// 128-row tile. On an SM pair one MMA covers M = 256 rows (128 per SM) and
// each SM holds and reads only half of B (96 of the 192 digit rows), so the
// B bytes an SM stages and the tensor core reads per row are halved, and the
// leader issues one MMA where two were issued before.
//   cluster (2,1,1); CTA r of cluster c owns row tiles 4q+2r, 4q+2r+1 of quad q
//   per stage and CTA: [digit-0 pair 16 KB][digit-1 slot 0][digit-1 slot 1][B half 6 KB]
//   A digit-1 slot is loaded when either SM's tile needs it (the SM without a
//   digit-1 tile loads the all-zero tile stored after the compact ones), so
//   one MMA serves both SMs.
//   full[s] (leader): both producers arrive with their own transaction bytes;
//   empty[s], tfull (each CTA): the leader's commit multicasts to both;
//   tempty (leader): the epilogue warps of both CTAs arrive.
constexpr int K3Q2_STAGES = 5;
constexpr int K3Q2_BH = (K3_ND * K3_NR / 2) * K3_BK;          // 6 KB: half the digit rows
constexpr int K3Q2_STAGE = 2 * K3_A_TILE + 2 * K3_A_TILE + K3Q2_BH;
constexpr size_t K3Q2_SMEM = 1024 + (size_t)K3Q2_STAGES * K3Q2_STAGE + K3_B_TILE;

__device__ __forceinline__ uint32_t k3_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t k3_mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void k3_cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void k3_expect_tx_cluster(uint32_t bar_cl, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar_cl),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void k3_arrive_cluster_relaxed(uint32_t bar_cl) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cl) : "memory");
}
__device__ __forceinline__ void k3_arrive_cluster(uint32_t bar_cl) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cl) : "memory");
}
__device__ __forceinline__ void tma_2d_pair(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint32_t bar_cl, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_cl), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          bar),
      "h"((uint16_t)0x3)
      : "memory");
}
// kind::i8 instruction descriptor for the SM-pair MMA (M = 256)
__host__ __device__ constexpr uint32_t idesc_i8_pair(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

struct K3PairArgs {
  int64_t rows;
  int kblocks_total, kb_stride, kblocks_per_unit, splits;
  int64_t quads;            // ceil(rows / 512)
  int nrhs;
  long long* yacc;
  const int* idx1;          // [rtiles][kbs] compact digit-1 index, -1 if absent
  int zero1;                // index of the all-zero digit-1 tile
  int ysh;                  // tensor rows are 64 << ysh bytes wide (2: pre-swizzled tiles)
  int btile;                // x digits stored as pre-swizzled [K block][192][64] tiles
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(K3_THREADS, 1)
    k3_dl2(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapA1,
           const __grid_constant__ CUtensorMap mapBh, K3PairArgs a) {
  constexpr int NACC = 4;
  extern __shared__ __align__(1024) unsigned char k3s[];
  unsigned char* base = (unsigned char*)(((uintptr_t)k3s + 1023) & ~(uintptr_t)1023);
  unsigned char* zero_tile = base + (size_t)K3Q2_STAGES * K3Q2_STAGE;
  __shared__ __align__(8) uint64_t full[K3Q2_STAGES], empty[K3Q2_STAGES], tfull, tempty;
  __shared__ uint32_t tmem_slot;
  __shared__ uint32_t s_mask[K3Q2_STAGES];
  for (int i = threadIdx.x; i < K3_B_TILE / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(zero_tile)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t rank = k3_cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < K3Q2_STAGES; ++i) {
      k3_mbar_init(smem_u32(&full[i]), 1);        // the leader's producer arrives for both CTAs
      k3_mbar_init(smem_u32(&empty[i]), 1);
    }
    k3_mbar_init(smem_u32(&tfull), 1);
    k3_mbar_init(smem_u32(&tempty), 8);           // 4 epilogue warps per CTA (leader's copy is used)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  k3_cluster_sync_all();
  tc_fence_after();
  // launched as a programmatic dependent of k3_digits: the prologue above
  // overlaps its tail; B (the x digits) and yacc are read after this
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const int64_t units = a.quads * a.splits;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      uint64_t pol_a, pol_b;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_a));
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_b));
      int st = 0;
      uint32_t ph = 0;
      int64_t it = 0;
      for (int64_t u = cid; u < units; u += ncl) {
        const int64_t quad = u / a.splits;
        const int split = (int)(u - quad * a.splits);
        const int kb0 = split * a.kblocks_per_unit;
        const int kb1 = min(a.kblocks_total, kb0 + a.kblocks_per_unit);
        const int64_t rt_own = quad * 4 + rank * 2, rt_peer = quad * 4 + (rank ^ 1) * 2;
        const int nkb = kb1 - kb0, rot = cid % nkb;
        for (int i = 0; i < nkb; ++i, ++it) {
          const int kb = kb0 + (i + rot) % nkb;
          if (it >= K3Q2_STAGES) k3_wait(smem_u32(&empty[st]), ph ^ 1);
          const uint32_t sb = smem_u32(base + (size_t)st * K3Q2_STAGE);
          const uint32_t fb = k3_mapa(smem_u32(&full[st]), 0);      // the leader's barrier
          int own1[2];
          uint32_t mask = 0;
#pragma unroll
          for (int ti = 0; ti < 2; ++ti) {
            own1[ti] = a.idx1[(rt_own + ti) * a.kb_stride + kb];
            const int peer1 = a.idx1[(rt_peer + ti) * a.kb_stride + kb];
            if (own1[ti] >= 0 || peer1 >= 0) mask |= 1u << ti;
          }
          if (rank == 0) s_mask[st] = mask;
#ifdef K3P2_NOTMA
          if (rank == 0) k3_arrive(smem_u32(&full[st]));
          if (++st == K3Q2_STAGES) { st = 0; ph ^= 1; }
          continue;
#endif
          // the leader expects both CTAs' bytes (the peer's loads may land
          // first: the transaction count may go negative until then)
          if (rank == 0) k3_expect_tx(smem_u32(&full[st]), 2 * (2 * K3_A_TILE + K3Q2_BH + __popc(mask) * K3_A_TILE));
          tma_2d_pair(sb, &mapA0, 0, (int)(k3d_tile0(rt_own, kb, a.kb_stride) * K3_BM) >> a.ysh, fb, pol_a);
#pragma unroll
          for (int ti = 0; ti < 2; ++ti)
            if ((mask >> ti) & 1u)
              tma_2d_pair(sb + (2 + ti) * K3_A_TILE, &mapA1, 0,
                          ((own1[ti] >= 0 ? own1[ti] : a.zero1) * K3_BM) >> a.ysh, fb, pol_a);
          tma_2d_pair(sb + 4 * K3_A_TILE, &mapBh, a.btile ? 0 : kb * K3_BK,
                      a.btile ? kb * (K3_ND * K3_NR / 4) + (int)rank * (K3_ND * K3_NR / 8)
                              : (int)rank * (K3_ND * K3_NR / 2), fb, pol_b);
          if (++st == K3Q2_STAGES) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (rank == 0) {
      const uint64_t dzero = desc_sw64(smem_u32(zero_tile));
      const uint32_t id64 = idesc_i8_pair(K3_NR), id192 = idesc_i8_pair(K3_ND * K3_NR);
      int st = 0;
      uint32_t ph = 0;
      int64_t ucount = 0;
      for (int64_t u = cid; u < units; u += ncl, ++ucount) {
        const int64_t quad = u / a.splits;
        const int split = (int)(u - quad * a.splits);
        const int kb0 = split * a.kblocks_per_unit;
        const int kb1 = min(a.kblocks_total, kb0 + a.kblocks_per_unit);
        if (ucount > 0) k3_wait(smem_u32(&tempty), (uint32_t)((ucount - 1) & 1));
        tc_fence_after();
        const int nkb = kb1 - kb0;
        for (int i = 0; i < nkb; ++i) {
          k3_wait(smem_u32(&full[st]), ph);
          tc_fence_after();
          const uint32_t mask = s_mask[st];
          const uint64_t dbase = desc_sw64(smem_u32(base + (size_t)st * K3Q2_STAGE));
#ifdef K3P2_NOMMA
          if (lane == 0) { k3_arrive(smem_u32(&empty[st])); k3_arrive_cluster_relaxed(k3_mapa(smem_u32(&empty[st]), 1)); }
          (void)mask; (void)dbase; (void)dzero; (void)id64; (void)id192;
          __syncwarp();
          if (++st == K3Q2_STAGES) { st = 0; ph ^= 1; }
          continue;
#endif
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < K3_BK / 32; ++kk) {
              const uint32_t cont = (i > 0 || kk > 0) ? 1u : 0u;
              const uint64_t db = dbase + (uint64_t)((4 * K3_A_TILE + kk * 32) >> 4);
#pragma unroll
              for (int ti = 0; ti < 2; ++ti) {
                const uint32_t t0 = tmem + (uint32_t)(ti * NACC * K3_NR);
                const uint64_t a0 = dbase + (uint64_t)((ti * K3_A_TILE + kk * 32) >> 4);
                if (!cont) mma_i8_pair(t0 + 3 * K3_NR, a0, dzero + (uint64_t)((kk * 32) >> 4), id64, 0u);
                mma_i8_pair(t0, a0, db, id192, cont);
                if ((mask >> ti) & 1u) {
                  const uint64_t a1 = dbase + (uint64_t)(((2 + ti) * K3_A_TILE + kk * 32) >> 4);
                  mma_i8_pair(t0 + 1 * K3_NR, a1, db, id192, 1u);
                }
              }
            }
            mma_commit_pair(smem_u32(&empty[st]));   // both CTAs' stage st is free
          }
          __syncwarp();
          if (++st == K3Q2_STAGES) { st = 0; ph ^= 1; }
        }
#ifdef K3P2_NOMMA
        if (lane == 0) { k3_arrive(smem_u32(&tfull)); k3_arrive_cluster(k3_mapa(smem_u32(&tfull), 1)); }
#else
        if (elect_one()) mma_commit_pair(smem_u32(&tfull));
#endif
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    const uint32_t tempty_leader = k3_mapa(smem_u32(&tempty), 0);
    int64_t ucount = 0;
    for (int64_t u = cid; u < units; u += ncl, ++ucount) {
      const int64_t quad = u / a.splits;
      k3_wait(smem_u32(&tfull), (uint32_t)(ucount & 1));
      tc_fence_after();
#pragma unroll 1
      for (int ti = 0; ti < 2; ++ti) {
        const int64_t row = (quad * 4 + rank * 2 + ti) * K3_BM + q * 32 + lane;
#pragma unroll 1
        for (int c0 = 0; c0 < K3_NR; c0 += 16) {
          int32_t r[NACC][16];
#pragma unroll
          for (int w = 0; w < NACC; ++w)
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((ti * NACC + w) * K3_NR + c0), r[w]);
          tmem_wait_ld();
          if (row < a.rows) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int t = c0 + j;
              if (t >= a.nrhs) break;
              long long v = 0;
#pragma unroll
              for (int w = 0; w < NACC; ++w) v += (long long)r[w][j] * (1LL << (8 * w));
              if (a.splits == 1)
                a.yacc[(int64_t)t * a.rows + row] = v;
              else
                atomicAdd((unsigned long long*)&a.yacc[(int64_t)t * a.rows + row], (unsigned long long)v);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) k3_arrive_cluster(tempty_leader);
    }
  }
  tc_fence_before();
  __syncthreads();
  k3_cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

int make_tensor_map_u8(void* map128, const void* ptr, uint64_t inner, uint64_t outer,
                       uint64_t pitch, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return fail(INVOP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc((CUtensorMap*)map128, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr),
                   dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(INVOP_E_CUDA, "cuTensorMapEncodeTiled failed");
  return INVOP_OK;
}

static int make_map_u8(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                       uint64_t pitch, uint32_t box_inner, uint32_t box_outer) {
  return make_tensor_map_u8(m, ptr, inner, outer, pitch, box_inner, box_outer, 64);
}

// a plain grid launched as a programmatic dependent of the preceding kernel
template <typename Kern, typename Arg>
static int launch_pdl(Kern kern, const Arg& arg, dim3 grid, int threads, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  INVOP_CUDA(cudaLaunchKernelEx(&cfg, kern, arg));
  return INVOP_OK;
}

// k3_post runs as one cluster of CL CTAs per right-hand side
// (CL = 16 is a non-portable size, opted in here)
template <typename Kern, typename Arg>
static int launch_cluster(Kern kern, const Arg& arg, int nr, int threads, int cl, cudaStream_t s) {
  if (cl > 8) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return cuda_fail(e, "cluster attribute");
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cl, (unsigned)nr);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  INVOP_CUDA(cudaLaunchKernelEx(&cfg, kern, arg));
  return INVOP_OK;
}

bool batched_supported(const invop_plan* p, int64_t nrhs) {
  // Two or more right-hand sides: one pass of the tensor-core kernel over the
  // operator (HBM-bound) beats per-RHS / 4-RHS passes of the CUDA-core kernels
  // (config 4: 7 RHS 0.716 -> 0.125 ms; config 5: 8.04 -> 0.763 ms).
  // INVOP_K3_MIN_RHS restores a higher threshold (round 1: 8).
  static const int min_rhs = []() {
    const char* e = getenv("INVOP_K3_MIN_RHS");
    return e && *e ? std::max(2, atoi(e)) : 2;
  }();
  // small batches on tiny operators stay on the single-launch kernel (config 1:
  // 7-10 us against ~19 us for the four-kernel chain)
  if (nrhs < 8 && p->rows * p->n < ((int64_t)1 << 20)) return false;
  return p->P <= 3 && nrhs >= min_rhs && p->n >= K3_BK && p->rows >= 1 && encode_fn() != nullptr;
}

template <int P, int TILES, int STAGES, bool DL = false>
static int launch_k3(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& a2,
                     const CUtensorMap& b, const K3Args& args, int grid, cudaStream_t s) {
  constexpr int STAGE = TILES * P * K3_A_TILE + K3_ND * K3_B_TILE;
  size_t smem = (size_t)STAGES * STAGE + 1024 + (P >= 2 ? K3_B_TILE : (DL ? K3_A_TILE : 0));
  auto kern = k3_batched<P, TILES, STAGES, DL>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, K3_THREADS, smem, s>>>(a0, a1, a2, b, args);
  INVOP_CHECK_LAUNCH("k3_batched");
  return INVOP_OK;
}

// SM pairs that can be resident at once (a persistent grid must not exceed
// it: TPC/GPC fragmentation leaves fewer than sms / 2 pairs)
static int k3_pair_slots() {
  static int slots = 0;
  if (!slots) {
    int n = num_sms() / 2;
    if (cudaFuncSetAttribute(k3_dl2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3Q2_SMEM) !=
        cudaSuccess)
      return num_sms() / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(num_sms());
    cfg.blockDim = dim3(K3_THREADS);
    cfg.dynamicSmemBytes = K3Q2_SMEM;
    int m = 0;
    if (cudaOccupancyMaxActiveClusters(&m, k3_dl2, &cfg) == cudaSuccess && m > 0) n = std::min(n, m);
    slots = n;
  }
  return slots;
}

// launched as a programmatic dependent of k3_digits
static int launch_k3_dl2(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& bh,
                         const K3PairArgs& args, int clusters, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k3_dl2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3Q2_SMEM);
  if (e != cudaSuccess) return cuda_fail(e, "k3_dl2 smem attribute");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(K3_THREADS);
  cfg.dynamicSmemBytes = K3Q2_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  INVOP_CUDA(cudaLaunchKernelEx(&cfg, k3_dl2, a0, a1, bh, args));
  return INVOP_OK;
}

// residual tiles for the K3 DL path; declined (k3d_ready = -1) when some
// residual needs a third digit or the layout would not be smaller
// row tiles of the residual layout: a multiple of 4 (SM pairs take quads)
static int64_t k3d_rtiles(const invop_plan* p) { return round_up(cdiv(p->rows, K3_BM), 4); }

// one thread per (row-tile pair slot of a quad, K block): 1 if either SM's tile has digit 1
__global__ void k3d_union(const int* __restrict__ idx1, int64_t rtiles, int64_t kbs,
                          int64_t* __restrict__ n1u) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int c = 0;
  if (t < rtiles / 2 * kbs) {
    const int64_t slot = t / kbs, kb = t - slot * kbs;     // slot = quad * 2 + ti
    const int64_t quad = slot >> 1, ti = slot & 1;
    c = (idx1[(quad * 4 + ti) * kbs + kb] >= 0 || idx1[(quad * 4 + 2 + ti) * kbs + kb] >= 0) ? 1 : 0;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long*)n1u, (unsigned long long)c);
}

static int k3d_build(invop_plan* p, cudaStream_t s) {
  if (p->k3d_ready) return p->k3d_ready > 0 ? INVOP_OK : INVOP_E_UNSUPPORTED;
  p->k3d_ready = -1;
  if (p->P > 2 || p->rows < 4 || !layout_flag("INVOP_K3_DL", true)) return INVOP_E_UNSUPPORTED;
  K3DBuild a;
  a.planes[0] = p->planes[0];
  a.planes[1] = p->planes[p->P > 1 ? 1 : 0];
  a.P = p->P;
  a.sgn = p->is_signed;
  a.rows = p->rows;
  a.ld = p->ld;
  a.kbs = p->ld / K3_BK;
  a.rtiles = k3d_rtiles(p);
  const int64_t tiles = a.rtiles * a.kbs;
  int* tilew = nullptr;
  int64_t* n1d = nullptr;
  INVOP_CUDA(cudaMalloc(&tilew, (size_t)tiles * 4 + 16));
  INVOP_CUDA(cudaMalloc(&n1d, 16));
  int* wmaxd = tilew + tiles;
  INVOP_CUDA(cudaMemsetAsync(tilew, 0, (size_t)tiles * 4 + 16, s));
  const int64_t thr = p->rows * a.kbs;
  k3d_width<<<(unsigned)cdiv(thr, 256), 256, 0, s>>>(a, tilew, wmaxd);
  int wmax = 0;
  INVOP_CUDA(cudaMemcpyAsync(&wmax, wmaxd, 4, cudaMemcpyDeviceToHost, s));
  INVOP_CUDA(cudaStreamSynchronize(s));
  int rc = INVOP_E_UNSUPPORTED;
  if (wmax <= 2) {
    INVOP_CUDA(cudaMalloc(&p->k3d_idx1, (size_t)tiles * 4));
    k3d_index<<<1, 1024, 0, s>>>(tiles, tilew, p->k3d_idx1, n1d);
    INVOP_CUDA(cudaMemcpyAsync(&p->k3d_n1, n1d, 8, cudaMemcpyDeviceToHost, s));
    INVOP_CUDA(cudaStreamSynchronize(s));
    if (tiles + p->k3d_n1 < (int64_t)p->P * tiles) {
      INVOP_CUDA(cudaMalloc(&p->k3d_tiles[0], (size_t)tiles * K3_A_TILE));
      // compact digit-1 tiles + one all-zero tile (the SM-pair kernel loads it
      // for an SM whose tile has no digit-1 plane while its peer's has)
      INVOP_CUDA(cudaMalloc(&p->k3d_tiles[1], (size_t)(p->k3d_n1 + 1) * K3_A_TILE));
      INVOP_CUDA(cudaMemsetAsync(p->k3d_tiles[0], 0, (size_t)tiles * K3_A_TILE, s));
      INVOP_CUDA(cudaMemsetAsync(p->k3d_tiles[1] + (size_t)p->k3d_n1 * K3_A_TILE, 0, K3_A_TILE, s));
      // INVOP_K3_PRESW=0: tiles stored row-major, swizzled by the tensor copy
      // (64-byte rows); default: stored pre-swizzled and copied as 256-byte rows
      const char* pe = std::getenv("INVOP_K3_PRESW");
      const int presw = pe && *pe == '0' ? 0 : 1;
      p->k3d_ysh = presw ? 2 : 0;
      k3d_write<<<(unsigned)cdiv(thr, 256), 256, 0, s>>>(a, p->k3d_idx1, p->k3d_tiles[0],
                                                         p->k3d_tiles[1], presw);
      const uint64_t wide = (uint64_t)K3_BK << p->k3d_ysh;
      const uint32_t brows = (uint32_t)((p->P == 2 ? 2 * K3_BM : K3_BM) >> p->k3d_ysh);
      rc = make_tensor_map_u8(p->k3d_mapA[0], p->k3d_tiles[0], wide,
                              ((uint64_t)tiles * K3_BM) >> p->k3d_ysh, wide, (uint32_t)wide, brows,
                              presw ? 0 : 64);
      if (!rc)
        rc = make_tensor_map_u8(p->k3d_mapA[1], p->k3d_tiles[1], wide,
                                ((uint64_t)(p->k3d_n1 + 1) * K3_BM) >> p->k3d_ysh, wide,
                                (uint32_t)wide, (uint32_t)(K3_BM >> p->k3d_ysh), presw ? 0 : 64);
      // digit-1 MMAs the SM-pair kernel issues: (quad, K block, slot) where
      // either SM's tile has a digit-1 plane
      if (!rc) {
        INVOP_CUDA(cudaMemsetAsync(n1d, 0, 8, s));
        k3d_union<<<(unsigned)cdiv(a.rtiles / 2 * a.kbs, 256), 256, 0, s>>>(p->k3d_idx1, a.rtiles, a.kbs, n1d);
        INVOP_CUDA(cudaMemcpyAsync(&p->k3d_n1u, n1d, 8, cudaMemcpyDeviceToHost, s));
      }
      cudaError_t ce = cudaStreamSynchronize(s);
      if (!rc && ce != cudaSuccess) rc = cuda_fail(ce, "k3d build");
      if (!rc) p->k3d_ready = 1;
    }
  }
  cudaFree(tilew);
  cudaFree(n1d);
  if (p->k3d_ready < 0) {
    for (int b = 0; b < 2; ++b) {
      if (p->k3d_tiles[b]) cudaFree(p->k3d_tiles[b]);
      p->k3d_tiles[b] = nullptr;
    }
    if (p->k3d_idx1) cudaFree(p->k3d_idx1);
    p->k3d_idx1 = nullptr;
    return rc ? rc : INVOP_E_UNSUPPORTED;
  }
  return INVOP_OK;
}

// The residual tiles go to the SM-pair kernel (k3_dl2) or the one-SM kernel
// (k3_batched<..., DL>): INVOP_K3_PAIR=1/0 forces one; otherwise the plan's
// choice, timed once on the device when the layout is built (k3_autotune) —
// which of the two is faster depends on how many SM pairs of this particular
// GPU can be co-resident (floor-swept parts differ: 0.87-0.94 ms for the pair
// kernel against 0.89-0.90 ms for the one-SM kernel at config 5 across boxes).
static bool k3_pair_enabled(const invop_plan* p) {
  const char* v = getenv("INVOP_K3_PAIR");
  if (v && *v) return *v != '0';
  return p->k3_pair != 0;
}

// the DL kernel serves a batched apply when its residual tiles were built and
// no INVOP_K3_CFG variant selects a byte-plane configuration
bool k3_uses_dl(const invop_plan* p) {
  if (p->k3d_ready <= 0) return false;
  int tiles = K3_TILES, stages = K3_STAGES;
  if (const char* v = getenv("INVOP_K3_CFG")) sscanf(v, "%d,%d", &tiles, &stages);
  return tiles == K3_TILES && stages == K3_STAGES;
}

// the residual-tile apply runs on SM pairs (k3_dl2)
bool k3_uses_pair(const invop_plan* p) { return k3_uses_dl(p) && k3_pair_enabled(p); }

static int batched_launch(invop_plan* p, const float* x, int64_t ldx, float* y, int64_t ldy,
                          int64_t nrhs, cudaStream_t s, int pair_sel);

// hashed noise in (-1, 1): the tensor-core kernels run power-capped, and their
// time depends on how much the operands toggle (zeros time ~8 % faster)
__global__ void k3_fill_noise(float* __restrict__ x, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t h = (uint32_t)i * 2654435761u + (uint32_t)(i >> 32) * 40503u + 12345u;
  h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16;
  x[i] = (float)(int32_t)h * (1.0f / 2147483648.0f);
}

// One-time choice between the SM-pair and the one-SM kernel for this plan on
// this GPU: both run a 64-RHS apply of noise, 2 warm-up + 3 timed launches each.
static int k3_autotune(invop_plan* p, cudaStream_t s) {
  if (p->k3_pair >= 0 || !k3_uses_dl(p)) return INVOP_OK;
  const char* v = getenv("INVOP_K3_PAIR");
  if (v && *v) return INVOP_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return INVOP_OK;          // decided by a later call outside the capture
  }
  float *x = nullptr, *y = nullptr;
  const size_t xb = (size_t)K3_NR * p->n * 4, yb = (size_t)K3_NR * p->rows * 4;
  if (cudaMalloc(&x, xb) != cudaSuccess || cudaMalloc(&y, yb) != cudaSuccess) {
    cudaGetLastError();
    if (x) cudaFree(x);
    p->k3_pair = 1;           // no room to measure: keep the default
    return INVOP_OK;
  }
  k3_fill_noise<<<(unsigned)cdiv((int64_t)K3_NR * p->n, 256), 256, 0, s>>>(x, (int64_t)K3_NR * p->n);
  cudaEvent_t e0, e1;
  INVOP_CUDA(cudaEventCreate(&e0));
  INVOP_CUDA(cudaEventCreate(&e1));
  float best_ms = 0.f;
  int best = 1, rc = INVOP_OK;
  for (int sel = 1; sel >= 0 && !rc; --sel) {
    for (int i = 0; i < 2 && !rc; ++i) rc = batched_launch(p, x, p->n, y, p->rows, K3_NR, s, sel);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 3 && !rc; ++i) rc = batched_launch(p, x, p->n, y, p->rows, K3_NR, s, sel);
    cudaEventRecord(e1, s);
    if (cudaEventSynchronize(e1) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "k3 autotune");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (getenv("INVOP_K3_DEBUG")) fprintf(stderr, "k3 autotune: %s %.4f ms\n", sel ? "pair" : "single", ms / 3);
    if (sel == 1 || ms < best_ms) { best_ms = ms; best = sel; }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(x);
  cudaFree(y);
  if (!rc) p->k3_pair = best;
  return rc;
}

// lazily built layouts of the batched apply (DL residual tiles) and the
// kernel choice
int k3_prepare(invop_plan* p, cudaStream_t s) {
  const int rc = k3d_build(p, s);
  if (rc != INVOP_OK) return rc == INVOP_E_UNSUPPORTED ? INVOP_OK : rc;
  return k3_autotune(p, s);
}

// int8 tensor operations (2*M*N*K per MMA) one batched apply of nrhs
// right-hand sides issues: per 64-RHS batch, per (row tile, K block) the
// MMAs of the operand tiles present (DL: plane 0 always and plane 1 where
// stored, N = 192; byte planes: P x 3 plane-digit products, N = 64)
int64_t k3_tensor_ops(const invop_plan* p, int64_t nrhs) {
  const int64_t batches = cdiv(nrhs, K3_NR);
  const int64_t kbs = p->ld / K3_BK;
  const int64_t rtiles = round_up(cdiv(p->rows, K3_BM), 2);
  const int64_t per_tile_kb = 2LL * K3_BM * (K3_ND * K3_NR) * K3_BK;   // one plane x all digits
  if (k3_uses_dl(p)) {
    const int64_t rt = k3d_rtiles(p);
    // SM pairs: digit-1 MMAs wherever either SM's tile needs one (k3d_union)
    if (k3_pair_enabled(p)) return batches * per_tile_kb * (rt * kbs + 2 * p->k3d_n1u);
    return batches * per_tile_kb * (rt * kbs + p->k3d_n1);
  }
  return batches * per_tile_kb * p->P * rtiles * kbs;
}

int64_t k3d_bytes(const invop_plan* p) {
  if (!k3_uses_dl(p)) return -1;   // DL kernel not used
  const int64_t tiles = k3d_rtiles(p) * (p->ld / K3_BK);
  return (tiles + p->k3d_n1) * K3_A_TILE + tiles * 4;
}

int apply_batched_launch(invop_plan* p, const float* x, int64_t ldx, float* y, int64_t ldy,
                         int64_t nrhs, cudaStream_t s) {
  const int rc = k3_prepare(p, s);
  if (rc) return rc;
  return batched_launch(p, x, ldx, y, ldy, nrhs, s, -1);
}

// pair_sel: 1 / 0 force the SM-pair / one-SM kernel (autotune), -1 the plan's choice
static int batched_launch(invop_plan* p, const float* x, int64_t ldx, float* y, int64_t ldy,
                          int64_t nrhs, cudaStream_t s, int pair_sel) {
  const int64_t ldb = round_up(p->n, K3_BK);
  const int kblocks = (int)(ldb / K3_BK);
  // variant: row tiles per unit (share B) and pipeline depth
  int tiles = K3_TILES, stages = K3_STAGES;
  if (const char* v = getenv("INVOP_K3_CFG")) sscanf(v, "%d,%d", &tiles, &stages);
  if (p->P == 3) { tiles = 1; stages = 5; }     // the one 3-plane configuration
  const int sms = num_sms();
  int krc = k3d_build(p, s);
  if (krc != INVOP_OK && krc != INVOP_E_UNSUPPORTED) return krc;
  const bool dl = k3_uses_dl(p);
  const bool pair = dl && (pair_sel >= 0 ? pair_sel != 0 : k3_pair_enabled(p));
  // work items: row-tile pairs on one SM, quads of row tiles on an SM pair
  const int64_t pairs = pair ? cdiv(p->rows, 4 * K3_BM) : cdiv(p->rows, tiles * K3_BM);
  const int slots = pair ? k3_pair_slots() : sms;
  // K splits: each unit spans <= 32768 columns; then pick the split count that
  // best fills the SMs (SM pairs) in whole waves
  // int32 class sums: up to min(P, 3) products of at most 255 * 128 per column
  const int kmax = p->P >= 3 ? K3_KMAX / 2 : K3_KMAX;
  int min_split = (int)cdiv(kblocks, kmax / K3_BK);
  int best = min_split;
  double best_eff = -1.0;
  for (int sp = min_split; sp <= std::max(min_split, 16); ++sp) {
    int64_t units = pairs * sp;
    double eff = (double)units / ((double)cdiv(units, slots) * slots);
    eff -= 0.005 * sp;   // atomics and partial tiles cost a little
    if (eff > best_eff + 1e-9) { best_eff = eff; best = sp; }
  }
  if (const char* v = getenv("INVOP_K3_SPLITS")) best = std::max(min_split, atoi(v));
  const int kpu = (int)cdiv(kblocks, best);
  const int splits = (int)cdiv(kblocks, kpu);   // no empty K ranges
  if (getenv("INVOP_K3_DEBUG"))
    fprintf(stderr, "k3: %s slots %d work %lld splits %d units %lld\n", pair ? "pair" : "single", slots,
            (long long)pairs, splits, (long long)(pairs * splits));
  // workspace: digits | exponents | non-finite counts | int64 row sums |
  // non-finite column lists. The row sums are zero between applies (k3_post
  // resets them behind its read), so K-split partials add atomically.
  const size_t b_bytes = (size_t)K3_ND * K3_NR * ldb;
  const size_t e_off = round_up(b_bytes, 256);
  const size_t nfc_off = e_off + 256;
  const size_t y01_off = nfc_off + 256;                   // [64][2] int64
  const size_t maxb_off = y01_off + 1024;                 // [64] max|x_t| bits
  const size_t acc_off = maxb_off + 256;
  const size_t acc_bytes = (size_t)K3_NR * p->rows * 8;
  const size_t nfl_off = round_up(acc_off + acc_bytes, 256);
  const size_t ws_bytes = nfl_off + (size_t)K3_NR * p->n * 4;
  if (p->k3_ws_bytes < ws_bytes || !p->k3_ws) {
    int rc = ensure_scratch(&p->k3_ws, &p->k3_ws_bytes, ws_bytes);
    if (rc) return rc;
    INVOP_CUDA(cudaMemsetAsync(p->k3_ws, 0, ws_bytes, s));
  }
  int8_t* B = (int8_t*)p->k3_ws;
  int* e = (int*)((char*)p->k3_ws + e_off);
  int* nfc = (int*)((char*)p->k3_ws + nfc_off);
  long long* y01 = (long long*)((char*)p->k3_ws + y01_off);
  unsigned int* maxb = (unsigned int*)((char*)p->k3_ws + maxb_off);
  long long* yacc = (long long*)((char*)p->k3_ws + acc_off);
  int* nfl = (int*)((char*)p->k3_ws + nfl_off);
  int rc = INVOP_OK;
  if (!dl && !p->k3_maps_ready) {
    const int64_t rtiles = round_up(cdiv(p->rows, K3_BM), 2);   // row tiles (even)
    const int64_t tile_bytes = rtiles * (p->ld / K3_BK) * K3_A_TILE;
    for (int b = 0; b < p->P; ++b) {
      if (!p->k3_tiles[b]) INVOP_CUDA(cudaMalloc(&p->k3_tiles[b], tile_bytes));
      k3_tile_planes<<<(unsigned)std::min<int64_t>(cdiv(tile_bytes / 16, 256), sms * 16), 256, 0, s>>>(
          p->planes[b], p->rows, p->ld, p->k3_tiles[b], rtiles, k3_bulk_env() && k3_btile_env());
      INVOP_LAUNCHED(1);
      INVOP_CHECK_LAUNCH("k3_tile_planes");
    }
    const uint64_t trows = (uint64_t)rtiles * (p->ld / K3_BK) * K3_BM;
    rc = make_map_u8((CUtensorMap*)p->k3_mapA[0], p->k3_tiles[0], K3_BK, trows, K3_BK, K3_BK, K3_BM);
    if (!rc && p->P > 1)
      rc = make_map_u8((CUtensorMap*)p->k3_mapA[1], p->k3_tiles[1], K3_BK, trows, K3_BK, K3_BK, K3_BM);
    if (!rc && p->P > 2)
      rc = make_map_u8((CUtensorMap*)p->k3_mapA[2], p->k3_tiles[2], K3_BK, trows, K3_BK, K3_BK, K3_BM);
    if (rc) return rc;
    if (p->P == 1) memcpy(p->k3_mapA[1], p->k3_mapA[0], sizeof(CUtensorMap));
    p->k3_maps_ready = 1;
    p->k3_presw = k3_bulk_env() && k3_btile_env();
  }
  CUtensorMap mapB;
  const int btile = k3_btile_env();
  if (btile)      // [kblocks * 48 rows][256 bytes], one K block's operand = 48 (pair: 24) rows
    rc = make_tensor_map_u8(&mapB, B, 4 * K3_BK, (uint64_t)kblocks * (K3_ND * K3_NR / 4), 4 * K3_BK,
                            4 * K3_BK, pair ? K3_ND * K3_NR / 8 : K3_ND * K3_NR / 4, 0);
  else
    rc = pair ? make_map_u8(&mapB, B, ldb, (uint64_t)K3_ND * K3_NR, ldb, K3_BK, K3_ND * K3_NR / 2)
              : make_map_u8(&mapB, B, ldb, (uint64_t)K3_ND * K3_NR, ldb, K3_BK, K3_ND * K3_NR);
  if (rc) return rc;
  for (int64_t t0 = 0; t0 < nrhs; t0 += K3_NR) {
    const int nr = (int)std::min<int64_t>(K3_NR, nrhs - t0);
    // 1. max|x_t| per right-hand side, exponents, digits, non-finite columns
    K3Prep pr;
    pr.x = x + t0 * ldx; pr.n = p->n; pr.ldx = ldx; pr.nrhs = nr;
    pr.B = B; pr.ldb = ldb; pr.e = e; pr.maxbits = maxb; pr.nf_count = nfc; pr.nf_cols = nfl;
    pr.planes[0] = p->planes[0];
    pr.planes[1] = p->planes[p->P > 1 ? 1 : 0];
    pr.ld = p->ld; pr.rows = p->rows; pr.P = p->P; pr.sgn = p->is_signed;
    pr.rows01 = dl ? 1 : 0; pr.y01 = (unsigned long long*)y01;
    pr.btile = btile;
    // 3. (arguments) rows 0/1 + double prefix (DL), scaling, non-finite
    // columns, y
    K3Post q;
    q.yacc = yacc; q.rows = p->rows; q.n = p->n; q.ld = p->ld;
    q.planes[0] = p->planes[0];
    q.planes[1] = p->planes[p->P > 1 ? 1 : 0];
    q.planes[2] = p->planes[p->P > 2 ? 2 : 0];
    q.P = p->P; q.sgn = p->is_signed;
    q.e = e; q.scale = p->scale;
    q.nf_count = nfc; q.nf_cols = nfl; q.y01 = y01; q.maxbits = maxb;
    q.x = x + t0 * ldx; q.ldx = ldx;
    q.y = y + t0 * ldy; q.ldy = ldy;
    int grid = (int)std::min<int64_t>(slots, pairs * splits);
#if !defined(K3_PROBE_NOSIDE) && !defined(K3_PROBE_NOPREP)
    rc = launch_pdl(k3_xmax, pr, dim3((unsigned)cdiv(p->n, K3X_COLS), K3_NR), K3X_TPB, s);
    if (!rc) rc = launch_pdl(k3_digits, pr, dim3((unsigned)cdiv(ldb, K3G_COLS), K3_NR), K3G_TPB, s);
    if (rc) return rc;
#endif
    // 2. the tensor-core pass: exact int64 row sums into yacc
    K3Args a;
    a.idx1 = p->k3d_idx1;
    a.ysh = p->k3d_ysh;
    a.btile = btile;
    a.B = B;
    if (dl) {
      a.t0 = p->k3d_tiles[0]; a.t1 = p->k3d_tiles[1]; a.t2 = nullptr;
      a.bulk = k3_bulk_env() && p->k3d_ysh == 2 && btile ? 1 : 0;
    } else {
      a.t0 = p->k3_tiles[0]; a.t1 = p->k3_tiles[1]; a.t2 = p->k3_tiles[2];
      a.bulk = p->k3_presw && btile ? 1 : 0;
    }
    a.rows = p->rows; a.n = p->n; a.P = p->P; a.hi_signed = p->is_signed;
    a.kblocks_total = kblocks; a.kblocks_per_unit = kpu; a.splits = splits;
    a.kb_stride = (int)(p->ld / K3_BK);
    a.pairs = pairs; a.nrhs = nr; a.yacc = yacc;
    const CUtensorMap* A0 = (const CUtensorMap*)(dl ? p->k3d_mapA[0] : p->k3_mapA[0]);
    const CUtensorMap* A1 = (const CUtensorMap*)(dl ? p->k3d_mapA[1] : p->k3_mapA[1]);
    const int key = dl ? 999 : p->P * 100 + tiles * 10 + stages;
    switch (key) {
      case 999:
        if (pair) {
          K3PairArgs pa;
          pa.rows = p->rows; pa.kblocks_total = kblocks; pa.kb_stride = (int)(p->ld / K3_BK);
          pa.kblocks_per_unit = kpu; pa.splits = splits; pa.quads = pairs; pa.nrhs = nr;
          pa.yacc = yacc; pa.idx1 = p->k3d_idx1; pa.zero1 = (int)p->k3d_n1;
          pa.ysh = p->k3d_ysh; pa.btile = btile;
          rc = launch_k3_dl2(*A0, *A1, mapB, pa, grid, s);
        } else {
          rc = launch_k3<2, 2, K3_DL_STAGES, true>(*A0, *A1, *A1, mapB, a, grid, s);
        }
        break;
      case 124: rc = launch_k3<1, 2, 4>(*A0, *A1, *A1, mapB, a, grid, s); break;
      case 116: rc = launch_k3<1, 1, 6>(*A0, *A1, *A1, mapB, a, grid, s); break;
      case 224: rc = launch_k3<2, 2, 4>(*A0, *A1, *A1, mapB, a, grid, s); break;
      case 216: rc = launch_k3<2, 1, 6>(*A0, *A1, *A1, mapB, a, grid, s); break;
      case 214: rc = launch_k3<2, 1, 4>(*A0, *A1, *A1, mapB, a, grid, s); break;
      case 223: rc = launch_k3<2, 2, 3>(*A0, *A1, *A1, mapB, a, grid, s); break;
      // 3-byte codes: one row tile per unit (5 weight classes x 64 TMEM columns)
      case 315: rc = launch_k3<3, 1, 5>(*A0, *A1, *(const CUtensorMap*)p->k3_mapA[2], mapB, a, grid, s); break;
      default: return fail(INVOP_E_VALUE, "unsupported INVOP_K3_CFG");
    }
    if (rc) return rc;
#if !defined(K3_PROBE_NOSIDE) && !defined(K3_PROBE_NOPOST)
    rc = dl ? launch_cluster(k3_post<true>, q, nr, K3Q_TPB, K3Q_CL, s)
            : launch_cluster(k3_post<false>, q, nr, K3Q_TPB, K3Q_CL, s);
#endif
    if (rc) return rc;
    INVOP_LAUNCHED(4);   // k3_xmax + k3_digits + k3_batched / k3_dl2 + k3_post
  }
  return INVOP_OK;
}

}  // namespace invop
