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
#include <algorithm>
#include <cstring>
#include <cstdio>
#include <cstdlib>

namespace invop {

static bool layout_flag(const char* env, bool dflt) {
  const char* v = getenv(env);
  if (!v || !*v) return dflt;
  return *v != '0';
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
  const int* e;            // [64] fixed-point exponents
  double scale;
  float* y;
  int64_t ldy;
  long long* yacc;         // [64][rows] when splits > 1 (DL: always; holds D)
  const int* idx1;         // DL: compact index of a tile's digit-1 plane, -1 if absent
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
               const __grid_constant__ CUtensorMap mapB, K3Args a) {
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
  constexpr int ZERO_BYTES = (P == 2 && K3_ND == 3) ? K3_B_TILE : K3_A_TILE;
  unsigned char* zero_tile = base + (size_t)STAGES * STAGE;
  if (DL) {
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
            uint32_t mask = 0, bytes = TILES * K3_A_TILE + K3_ND * K3_B_TILE;
#pragma unroll
            for (int ti = 0; ti < TILES; ++ti) {
              i1[ti] = a.idx1[(int64_t)(row0 / K3_BM + ti) * a.kb_stride + kb];
              if (i1[ti] >= 0) { mask |= 1u << ti; bytes += K3_A_TILE; }
            }
            s_mask[st] = mask;
            k3_expect_tx(fb, bytes);
            if (P == 2 && TILES == 2) {
              // stage: [digit-0 tile 0][digit-0 tile 1][digit-1 tile 0][digit-1 tile 1]
              const int trow = (int)(k3d_tile0(row0 / K3_BM, kb, a.kb_stride) * K3_BM);
              tma_2d(sb, &mapA0, 0, trow, fb, pol_a);         // both digit-0 tiles
#pragma unroll
              for (int ti = 0; ti < TILES; ++ti)
                if (i1[ti] >= 0)
                  tma_2d(sb + (TILES + ti) * K3_A_TILE, &mapA1, 0, i1[ti] * K3_BM, fb, pol_a);
            } else {
#pragma unroll
              for (int ti = 0; ti < TILES; ++ti) {
                const int trow = (int)(k3d_tile0(row0 / K3_BM + ti, kb, a.kb_stride) * K3_BM);
                tma_2d(sb + (ti * P + 0) * K3_A_TILE, &mapA0, 0, trow, fb, pol_a);
                if (i1[ti] >= 0) tma_2d(sb + (ti * P + 1) * K3_A_TILE, &mapA1, 0, i1[ti] * K3_BM, fb, pol_a);
              }
            }
          } else {
            k3_expect_tx(fb, STAGE);
#pragma unroll
            for (int ti = 0; ti < TILES; ++ti) {
              // tiled planes: tile (rt, kb) starts at tensor row (rt*kblocks + kb)*128
              const int trow = (int)(((int64_t)(row0 / K3_BM + ti) * a.kb_stride + kb) * K3_BM);
              tma_2d(sb + (ti * P + 0) * K3_A_TILE, &mapA0, 0, trow, fb, pol_a);
              if (P > 1) tma_2d(sb + (ti * P + 1) * K3_A_TILE, &mapA1, 0, trow, fb, pol_a);
            }
          }
          // the three digit tiles are consecutive rows of B: one 192-row box
          tma_2d(sb + A_BYTES, &mapB, kb * K3_BK, 0, fb, pol_b);
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
          if constexpr (DL && P == 2 && K3_ND == 3) {
            // straight-line issue with N = 192: the three digit tiles of B
            // are contiguous in shared memory and the weight classes of a
            // tile are contiguous in TMEM (class w = plane + digit at column
            // 64 w), so plane 0 x all digits is ONE MMA into classes 0-2 and
            // plane 1 x all digits one MMA into classes 1-3 (a third of the
            // MMAs of the N = 64 form; the tensor core re-reads A per MMA).
            // Class 3 is started by a zero tile at the unit's first K block.
            const uint32_t id0 = idesc_i8(1, K3_ND * K3_NR);
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
          mma_commit_elect(smem_u32(&empty[st]));   // stage free once these MMAs complete
        }
        __syncwarp();
        if (++st == STAGES) { st = 0; ph ^= 1; }
      }
      mma_commit_elect(smem_u32(&tfull));
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
              if (DL && a.splits == 1) {
                a.yacc[(int64_t)t * a.rows + row] = v;
              } else if (a.splits == 1) {
                a.y[(int64_t)t * a.ldy + row] = (float)((double)v * ldexp(a.scale, -a.e[t]));
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
__global__ void k3_tile_planes(const uint8_t* __restrict__ in, int64_t rows, int64_t ld,
                               uint8_t* __restrict__ out, int64_t rtiles) {
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
    *reinterpret_cast<uint4*>(out + tile * K3_A_TILE + r * K3_BK + c16 * 16) = v;
  }
}

// ------------------------------------------------------------ x preparation
// max |x_t| for every right-hand side (as the bits of a non-negative float,
// combined with atomicMax) plus an inf/nan flag; grid = (column chunks, RHS)
__global__ void k3_xmax(const float* __restrict__ x, int64_t n, int64_t ldx,
                        unsigned int* __restrict__ maxbits, int* __restrict__ nonfinite) {
  const int t = blockIdx.y;
  float m = 0.0f;
  bool bad = false;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[t * ldx + j];
    bad |= !isfinite(v);
    m = fmaxf(m, fabsf(v));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
  // one atomic per block (per-warp atomics on one address serialise in L2)
  __shared__ float wm[32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0.0f;
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) atomicMax(&maxbits[t], __float_as_uint(v));
  }
}

__device__ __forceinline__ int k3_exponent(unsigned int bits) {
  const float m = __uint_as_float(bits);
  int ex = 0;
  if (m > 0.0f && isfinite(m)) frexpf(m, &ex);
  return (m > 0.0f && isfinite(m)) ? 22 - ex : 0;   // max|x_t| * 2^e_t < 2^22
}

// balanced base-256 digits of X = rint(x * 2^e), into B[l][t][j] (int8);
// one thread per 16 consecutive columns of one right-hand side (ldb is a
// multiple of 64): three 16-byte stores
__global__ void k3_digits(const float* __restrict__ x, int64_t n, int64_t ldx, int nrhs,
                          const unsigned int* __restrict__ maxbits, int* __restrict__ e,
                          int8_t* __restrict__ B, int64_t ldb) {
  const int64_t per = ldb / 16;
  const int64_t total = (int64_t)K3_NR * per;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(k / per);
    const int64_t j0 = (k - (int64_t)t * per) * 16;
    const int et = t < nrhs ? k3_exponent(maxbits[t]) : 0;
    if (j0 == 0) e[t] = et;
    uint32_t w[3][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t b0 = 0, b1 = 0, b2 = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t j = j0 + 4 * q + i;
        int X = 0;
        if (t < nrhs && j < n) X = __float2int_rn(ldexpf(x[t * ldx + j], et));
        const int d0 = ((X + 128) & 255) - 128;
        const int X1 = (X - d0) >> 8;
        const int d1 = ((X1 + 128) & 255) - 128;
        const int d2 = (X1 - d1) >> 8;
        b0 |= ((uint32_t)d0 & 255u) << (8 * i);
        b1 |= ((uint32_t)d1 & 255u) << (8 * i);
        b2 |= ((uint32_t)d2 & 255u) << (8 * i);
      }
      w[0][q] = b0; w[1][q] = b1; w[2][q] = b2;
    }
#pragma unroll
    for (int l = 0; l < 3; ++l)
      *reinterpret_cast<uint4*>(B + (int64_t)(l * K3_NR + t) * ldb + j0) =
          make_uint4(w[l][0], w[l][1], w[l][2], w[l][3]);
  }
}

__global__ void k3_finalize(const long long* __restrict__ yacc, int64_t rows, int nrhs,
                            const int* __restrict__ e, double scale, float* __restrict__ y,
                            int64_t ldy) {
  const int64_t total = (int64_t)nrhs * rows;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(k / rows);
    const int64_t i = k - (int64_t)t * rows;
    y[t * ldy + i] = (float)((double)yacc[t * rows + i] * ldexp(scale, -e[t]));
  }
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
__global__ void k3d_write(K3DBuild a, const int* __restrict__ idx1, uint8_t* __restrict__ t0,
                          uint8_t* __restrict__ t1) {
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
    *reinterpret_cast<uint4*>(d0 + q0) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
    if (d1) *reinterpret_cast<uint4*>(d1 + q0) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
  }
}

// exact Y_0, Y_1 from the plain codes and the same x digits, added as
// D_0 += Y_0, D_1 += Y_1 - 2 Y_0 (linear, so column pieces add atomically;
// the tensor-core pass left 0 in both rows). grid = (column pieces, RHS),
// 16 columns per thread
__global__ void k3d_rows01(const uint8_t* p0, const uint8_t* p1, int P, int sgn, int64_t n,
                           int64_t ld, int64_t rows, const int8_t* __restrict__ B, int64_t ldb,
                           long long* __restrict__ yacc) {
  const int t = blockIdx.y;
  const int64_t j0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 16;
  long long s0 = 0, s1 = 0;
  if (j0 < n) {
    const uint4 g0 = *reinterpret_cast<const uint4*>(B + (0 * K3_NR + t) * ldb + j0);
    const uint4 g1 = *reinterpret_cast<const uint4*>(B + (1 * K3_NR + t) * ldb + j0);
    const uint4 g2 = *reinterpret_cast<const uint4*>(B + (2 * K3_NR + t) * ldb + j0);
    const uint4 a0 = *reinterpret_cast<const uint4*>(p0 + j0);
    const uint4 a1 = P > 1 ? *reinterpret_cast<const uint4*>(p1 + j0) : make_uint4(0, 0, 0, 0);
    const uint4 b0 = rows > 1 ? *reinterpret_cast<const uint4*>(p0 + ld + j0) : make_uint4(0, 0, 0, 0);
    const uint4 b1 = (rows > 1 && P > 1) ? *reinterpret_cast<const uint4*>(p1 + ld + j0)
                                         : make_uint4(0, 0, 0, 0);
    const uint32_t G0[4] = {g0.x, g0.y, g0.z, g0.w}, G1[4] = {g1.x, g1.y, g1.z, g1.w},
                   G2[4] = {g2.x, g2.y, g2.z, g2.w}, A0[4] = {a0.x, a0.y, a0.z, a0.w},
                   A1[4] = {a1.x, a1.y, a1.z, a1.w}, B0[4] = {b0.x, b0.y, b0.z, b0.w},
                   B1[4] = {b1.x, b1.y, b1.z, b1.w};
    const int sh = 32 - 8 * P;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int w = q >> 2, bb = 8 * (q & 3);
      const long long X = (long long)(int8_t)(G0[w] >> bb) + 256LL * (int8_t)(G1[w] >> bb) +
                          65536LL * (int8_t)(G2[w] >> bb);
      uint32_t u0 = ((A0[w] >> bb) & 255u) | (((A1[w] >> bb) & 255u) << 8);
      uint32_t u1 = ((B0[w] >> bb) & 255u) | (((B1[w] >> bb) & 255u) << 8);
      const int32_t v0 = sgn ? ((int32_t)(u0 << sh) >> sh) : (int32_t)u0;
      const int32_t v1 = sgn ? ((int32_t)(u1 << sh) >> sh) : (int32_t)u1;
      s0 += (long long)v0 * X;
      s1 += (long long)v1 * X;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd((unsigned long long*)&yacc[(int64_t)t * rows], (unsigned long long)s0);
    if (rows > 1)
      atomicAdd((unsigned long long*)&yacc[(int64_t)t * rows + 1], (unsigned long long)(s1 - 2 * s0));
  }
}

// Y = double prefix sum of D along rows, exact in int64, in segments of
// K3D_SEG rows: pass 1 gives per segment (sum D, sum z_local) with z_local the
// segment-local first prefix; the carries (Z_in, Y_in) follow sequentially per
// RHS; pass 2 rebuilds y_r = y_local + (r - r0 + 1) Z_in + Y_in and scales.
constexpr int K3D_SEG = 1024;

__device__ __forceinline__ long long k3d_block_incl(long long v, long long* sh) {
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
    long long s = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += u;
    }
    sh[lane] = s;
  }
  __syncthreads();
  const long long r = inc + (w > 0 ? sh[w - 1] : 0);
  __syncthreads();
  return r;
}

// grid = (segments, RHS), K3D_TPB threads x K3D_RPT consecutive rows each:
// thread-local prefixes, then one block scan per prefix level
constexpr int K3D_RPT = 4;
constexpr int K3D_TPB = K3D_SEG / K3D_RPT;

// d[] -> z[] (inclusive prefix over the segment) and yl[] (prefix of z)
__device__ __forceinline__ void k3d_seg_prefix(const long long* d, long long* z, long long* yl,
                                               long long* sh) {
  long long c[K3D_RPT];
  c[0] = d[0];
#pragma unroll
  for (int i = 1; i < K3D_RPT; ++i) c[i] = c[i - 1] + d[i];
  const long long ze = k3d_block_incl(c[K3D_RPT - 1], sh) - c[K3D_RPT - 1];
#pragma unroll
  for (int i = 0; i < K3D_RPT; ++i) z[i] = ze + c[i];
  long long w[K3D_RPT];
  w[0] = z[0];
#pragma unroll
  for (int i = 1; i < K3D_RPT; ++i) w[i] = w[i - 1] + z[i];
  const long long we = k3d_block_incl(w[K3D_RPT - 1], sh) - w[K3D_RPT - 1];
#pragma unroll
  for (int i = 0; i < K3D_RPT; ++i) yl[i] = we + w[i];
}

__global__ void __launch_bounds__(K3D_TPB) k3d_seg_sums(const long long* __restrict__ yacc,
                                                        int64_t rows, long long* __restrict__ seg) {
  __shared__ long long sh[32];
  const int t = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * K3D_SEG + threadIdx.x * K3D_RPT;
  long long d[K3D_RPT], z[K3D_RPT], yl[K3D_RPT];
#pragma unroll
  for (int i = 0; i < K3D_RPT; ++i) d[i] = r0 + i < rows ? yacc[(int64_t)t * rows + r0 + i] : 0;
  k3d_seg_prefix(d, z, yl, sh);
  if (threadIdx.x == K3D_TPB - 1) {
    seg[((int64_t)t * gridDim.x + blockIdx.x) * 2 + 0] = z[K3D_RPT - 1];    // sum of D
    seg[((int64_t)t * gridDim.x + blockIdx.x) * 2 + 1] = yl[K3D_RPT - 1];   // sum of z_local
  }
}

// segment carries in place, (sum D, sum z) -> (Z_in, Y_in): one block per RHS,
// one thread per segment (nseg <= K3D_SEG), two block scans:
//   Z_in(k) = sum_{j<k} sumD_j,  Y_in(k) = sum_{j<k} (K3D_SEG Z_in(j) + sumz_j)
__global__ void __launch_bounds__(K3D_SEG) k3d_seg_carry(long long* __restrict__ seg, int nseg) {
  __shared__ long long sh[32];
  const int t = blockIdx.x, k = threadIdx.x;
  long long* p = seg + ((int64_t)t * nseg + k) * 2;
  const long long sd = k < nseg ? p[0] : 0, sz = k < nseg ? p[1] : 0;
  const long long zin = k3d_block_incl(sd, sh) - sd;
  const long long term = (long long)K3D_SEG * zin + sz;
  const long long yin = k3d_block_incl(term, sh) - term;
  if (k < nseg) {
    p[0] = zin;
    p[1] = yin;
  }
}

__global__ void __launch_bounds__(K3D_TPB) k3d_seg_apply(const long long* __restrict__ yacc,
                                                         int64_t rows, const long long* __restrict__ seg,
                                                         const int* __restrict__ e, double scale,
                                                         float* __restrict__ y, int64_t ldy) {
  __shared__ long long sh[32];
  const int t = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * K3D_SEG + threadIdx.x * K3D_RPT;
  long long d[K3D_RPT], z[K3D_RPT], yl[K3D_RPT];
#pragma unroll
  for (int i = 0; i < K3D_RPT; ++i) d[i] = r0 + i < rows ? yacc[(int64_t)t * rows + r0 + i] : 0;
  k3d_seg_prefix(d, z, yl, sh);
  const long long* c = seg + ((int64_t)t * gridDim.x + blockIdx.x) * 2;
  const long long zin = c[0], yin = c[1];
  const double sc = ldexp(scale, -e[t]);
#pragma unroll
  for (int i = 0; i < K3D_RPT; ++i) {
    const long long Y = yl[i] + (long long)(threadIdx.x * K3D_RPT + i + 1) * zin + yin;
    if (r0 + i < rows) y[(int64_t)t * ldy + r0 + i] = (float)((double)Y * sc);
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

static int make_map_u8(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                       uint64_t pitch, uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return fail(INVOP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(INVOP_E_CUDA, "cuTensorMapEncodeTiled failed");
  return INVOP_OK;
}

bool batched_supported(const invop_plan* p, int64_t nrhs) {
  return p->P <= 2 && nrhs >= 8 && p->n >= K3_BK && p->rows >= 1 && encode_fn() != nullptr;
}

template <int P, int TILES, int STAGES, bool DL = false>
static int launch_k3(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b,
                     const K3Args& args, int grid, cudaStream_t s) {
  constexpr int STAGE = TILES * P * K3_A_TILE + K3_ND * K3_B_TILE;
  size_t smem = (size_t)STAGES * STAGE + 1024 + (DL ? (P == 2 ? K3_B_TILE : K3_A_TILE) : 0);
  auto kern = k3_batched<P, TILES, STAGES, DL>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, K3_THREADS, smem, s>>>(a0, a1, b, args);
  INVOP_CHECK_LAUNCH("k3_batched");
  return INVOP_OK;
}

// residual tiles for the K3 DL path; declined (k3d_ready = -1) when some
// residual needs a third digit or the layout would not be smaller
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
  a.rtiles = round_up(cdiv(p->rows, K3_BM), 2);
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
      INVOP_CUDA(cudaMalloc(&p->k3d_tiles[1], (size_t)std::max<int64_t>(p->k3d_n1, 1) * K3_A_TILE));
      INVOP_CUDA(cudaMemsetAsync(p->k3d_tiles[0], 0, (size_t)tiles * K3_A_TILE, s));
      k3d_write<<<(unsigned)cdiv(thr, 256), 256, 0, s>>>(a, p->k3d_idx1, p->k3d_tiles[0],
                                                         p->k3d_tiles[1]);
      rc = make_map_u8((CUtensorMap*)p->k3d_mapA[0], p->k3d_tiles[0], K3_BK,
                       (uint64_t)tiles * K3_BM, K3_BK, K3_BK, p->P == 2 ? 2 * K3_BM : K3_BM);
      if (!rc)
        rc = make_map_u8((CUtensorMap*)p->k3d_mapA[1], p->k3d_tiles[1], K3_BK,
                         (uint64_t)std::max<int64_t>(p->k3d_n1, 1) * K3_BM, K3_BK, K3_BK, K3_BM);
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

// the DL kernel serves a batched apply when its residual tiles were built,
// the row prefix sum covers the rows (<= 1024 segments) and no INVOP_K3_CFG
// variant selects a byte-plane configuration
bool k3_uses_dl(const invop_plan* p) {
  if (p->k3d_ready <= 0 || cdiv(p->rows, K3D_SEG) > K3D_SEG) return false;
  int tiles = K3_TILES, stages = K3_STAGES;
  if (const char* v = getenv("INVOP_K3_CFG")) sscanf(v, "%d,%d", &tiles, &stages);
  return tiles == K3_TILES && stages == K3_STAGES;
}

// lazily built layouts of the batched apply (DL residual tiles)
int k3_prepare(invop_plan* p, cudaStream_t s) {
  const int rc = k3d_build(p, s);
  return rc == INVOP_E_UNSUPPORTED ? INVOP_OK : rc;
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
  if (k3_uses_dl(p)) return batches * per_tile_kb * (rtiles * kbs + p->k3d_n1);
  return batches * per_tile_kb * p->P * rtiles * kbs;
}

int64_t k3d_bytes(const invop_plan* p) {
  if (!k3_uses_dl(p)) return -1;   // DL kernel not used
  const int64_t tiles = round_up(cdiv(p->rows, K3_BM), 2) * (p->ld / K3_BK);
  return (tiles + p->k3d_n1) * K3_A_TILE + tiles * 4;
}

int apply_batched_launch(invop_plan* p, const float* x, int64_t ldx, float* y, int64_t ldy,
                         int64_t nrhs, cudaStream_t s) {
  const int64_t ldb = round_up(p->n, K3_BK);
  const int kblocks = (int)(ldb / K3_BK);
  // variant: row tiles per unit (share B) and pipeline depth
  int tiles = K3_TILES, stages = K3_STAGES;
  if (const char* v = getenv("INVOP_K3_CFG")) sscanf(v, "%d,%d", &tiles, &stages);
  const int64_t pairs = cdiv(p->rows, tiles * K3_BM);
  const int sms = num_sms();
  // K splits: each unit spans <= 32768 columns; then pick the split count that
  // best fills the SMs in whole waves
  int min_split = (int)cdiv(kblocks, K3_KMAX / K3_BK);
  int best = min_split;
  double best_eff = -1.0;
  for (int sp = min_split; sp <= std::max(min_split, 16); ++sp) {
    int64_t units = pairs * sp;
    double eff = (double)units / ((double)cdiv(units, sms) * sms);
    eff -= 0.005 * sp;   // atomics and partial tiles cost a little
    if (eff > best_eff + 1e-9) { best_eff = eff; best = sp; }
  }
  if (const char* v = getenv("INVOP_K3_SPLITS")) best = std::max(min_split, atoi(v));
  const int kpu = (int)cdiv(kblocks, best);
  const int splits = (int)cdiv(kblocks, kpu);   // no empty K ranges
  // workspace: digits | exponents | int64 partial sums
  size_t b_bytes = (size_t)K3_ND * K3_NR * ldb;
  size_t e_off = round_up(b_bytes, 256);
  size_t flag_off = e_off + 256;                          // e[64] ints | flag
  size_t max_off = flag_off + 256;                        // max|x_t| bits [nrhs]
  size_t acc_off = round_up(max_off + (size_t)nrhs * 4, 256);
  int krc = k3d_build(p, s);
  if (krc != INVOP_OK && krc != INVOP_E_UNSUPPORTED) return krc;
  const bool dl = k3_uses_dl(p);
  size_t acc_bytes = splits > 1 ? (size_t)K3_NR * p->rows * 8 : 0;
  if (dl)   // + segment carries of the row prefix sums
    acc_bytes = (size_t)K3_NR * p->rows * 8 + (size_t)K3_NR * cdiv(p->rows, K3D_SEG) * 16;
  int rc = ensure_scratch(&p->k3_ws, &p->k3_ws_bytes, acc_off + acc_bytes);
  if (rc) return rc;
  unsigned int* maxbits = (unsigned int*)((char*)p->k3_ws + max_off);
  int* flag = (int*)((char*)p->k3_ws + flag_off);
  // max|x_t| of every right-hand side in one launch. inf/nan in x needs the
  // reference's zero-mantissa skip (fp32 masked kernels): the flag travels to
  // page-locked host memory behind an event while the tensor-core apply is
  // enqueued speculatively; the host reads it once the event fires (the GPU
  // is busy with the apply meanwhile) and, if set, enqueues the masked apply,
  // which overwrites y in stream order.
  if (!p->k3_flag_host) {
    INVOP_CUDA(cudaHostAlloc((void**)&p->k3_flag_host, 64, cudaHostAllocDefault));
    INVOP_CUDA(cudaEventCreateWithFlags(&p->k3_flag_event, cudaEventDisableTiming));
  }
  {
    INVOP_CUDA(cudaMemsetAsync((char*)p->k3_ws + flag_off, 0, max_off - flag_off + (size_t)nrhs * 4, s));
    dim3 g((unsigned)std::min<int64_t>(cdiv(p->n, 256), 64), (unsigned)nrhs);
    k3_xmax<<<g, 256, 0, s>>>(x, p->n, ldx, maxbits, flag);
    INVOP_LAUNCHED(1);
    INVOP_CUDA(cudaMemcpyAsync(p->k3_flag_host, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    INVOP_CUDA(cudaEventRecord(p->k3_flag_event, s));
  }
  if (rc) return rc;
  int8_t* B = (int8_t*)p->k3_ws;
  int* e = (int*)((char*)p->k3_ws + e_off);
  long long* yacc = (long long*)((char*)p->k3_ws + acc_off);
  if (!dl && !p->k3_maps_ready) {
    const int64_t rtiles = round_up(cdiv(p->rows, K3_BM), 2);   // row tiles (even)
    const int64_t tile_bytes = rtiles * (p->ld / K3_BK) * K3_A_TILE;
    for (int b = 0; b < p->P; ++b) {
      if (!p->k3_tiles[b]) INVOP_CUDA(cudaMalloc(&p->k3_tiles[b], tile_bytes));
      k3_tile_planes<<<(unsigned)std::min<int64_t>(cdiv(tile_bytes / 16, 256), sms * 16), 256, 0, s>>>(
          p->planes[b], p->rows, p->ld, p->k3_tiles[b], rtiles);
      INVOP_LAUNCHED(1);
      INVOP_CHECK_LAUNCH("k3_tile_planes");
    }
    const uint64_t trows = (uint64_t)rtiles * (p->ld / K3_BK) * K3_BM;
    rc = make_map_u8((CUtensorMap*)p->k3_mapA[0], p->k3_tiles[0], K3_BK, trows, K3_BK, K3_BK, K3_BM);
    if (!rc && p->P > 1)
      rc = make_map_u8((CUtensorMap*)p->k3_mapA[1], p->k3_tiles[1], K3_BK, trows, K3_BK, K3_BK, K3_BM);
    if (rc) return rc;
    if (p->P == 1) memcpy(p->k3_mapA[1], p->k3_mapA[0], sizeof(CUtensorMap));
    p->k3_maps_ready = 1;
  }
  CUtensorMap mapB;
  rc = make_map_u8(&mapB, B, ldb, (uint64_t)K3_ND * K3_NR, ldb, K3_BK, K3_ND * K3_NR);
  if (rc) return rc;
  for (int64_t t0 = 0; t0 < nrhs; t0 += K3_NR) {
    const int nr = (int)std::min<int64_t>(K3_NR, nrhs - t0);
    k3_digits<<<(unsigned)std::min<int64_t>(cdiv((int64_t)K3_NR * ldb / 16, 256), sms * 16), 256, 0, s>>>(
        x + t0 * ldx, p->n, ldx, nr, maxbits + t0, e, B, ldb);
    INVOP_LAUNCHED(2);   // k3_digits + k3_batched
    if (splits > 1) INVOP_CUDA(cudaMemsetAsync(yacc, 0, acc_bytes, s));
    K3Args a;
    a.idx1 = p->k3d_idx1;
    a.rows = p->rows; a.n = p->n; a.P = p->P; a.hi_signed = p->is_signed;
    a.kblocks_total = kblocks; a.kblocks_per_unit = kpu; a.splits = splits;
    a.kb_stride = (int)(p->ld / K3_BK);
    a.pairs = pairs; a.nrhs = nr; a.e = e; a.scale = p->scale;
    a.y = y + t0 * ldy; a.ldy = ldy; a.yacc = yacc;
    int grid = (int)std::min<int64_t>(sms, pairs * splits);
    const CUtensorMap* A0 = (const CUtensorMap*)(dl ? p->k3d_mapA[0] : p->k3_mapA[0]);
    const CUtensorMap* A1 = (const CUtensorMap*)(dl ? p->k3d_mapA[1] : p->k3_mapA[1]);
    const int key = dl ? 999 : p->P * 100 + tiles * 10 + stages;
    switch (key) {
      case 999: rc = launch_k3<2, 2, K3_DL_STAGES, true>(*A0, *A1, mapB, a, grid, s); break;
      case 124: rc = launch_k3<1, 2, 4>(*A0, *A1, mapB, a, grid, s); break;
      case 116: rc = launch_k3<1, 1, 6>(*A0, *A1, mapB, a, grid, s); break;
      case 224: rc = launch_k3<2, 2, 4>(*A0, *A1, mapB, a, grid, s); break;
      case 216: rc = launch_k3<2, 1, 6>(*A0, *A1, mapB, a, grid, s); break;
      case 214: rc = launch_k3<2, 1, 4>(*A0, *A1, mapB, a, grid, s); break;
      case 223: rc = launch_k3<2, 2, 3>(*A0, *A1, mapB, a, grid, s); break;
      default: return fail(INVOP_E_VALUE, "unsupported INVOP_K3_CFG");
    }
    if (rc) return rc;
    if (dl) {
      // rows 0/1 from the codes, then the double prefix sum along rows
      dim3 g01((unsigned)cdiv(cdiv(p->n, 16), 256), (unsigned)nr);
      k3d_rows01<<<g01, 256, 0, s>>>(p->planes[0], p->planes[p->P > 1 ? 1 : 0], p->P, p->is_signed,
                                     p->n, p->ld, p->rows, B, ldb, yacc);
      const int nseg = (int)cdiv(p->rows, K3D_SEG);
      long long* seg = yacc + (size_t)K3_NR * p->rows;
      dim3 gs((unsigned)nseg, (unsigned)nr);
      k3d_seg_sums<<<gs, K3D_TPB, 0, s>>>(yacc, p->rows, seg);
      k3d_seg_carry<<<nr, (unsigned)round_up(nseg, 32), 0, s>>>(seg, nseg);
      k3d_seg_apply<<<gs, K3D_TPB, 0, s>>>(yacc, p->rows, seg, e, p->scale, y + t0 * ldy, ldy);
      INVOP_LAUNCHED(4);
    } else if (splits > 1) {
      int64_t tot = (int64_t)nr * p->rows;
      k3_finalize<<<(unsigned)std::min<int64_t>(cdiv(tot, 256), sms * 8), 256, 0, s>>>(
          yacc, p->rows, nr, e, p->scale, y + t0 * ldy, ldy);
      INVOP_LAUNCHED(1);
    }
  }
  INVOP_CHECK_LAUNCH("k3 epilogue");
  INVOP_CUDA(cudaEventSynchronize(p->k3_flag_event));
  if (*(volatile int*)p->k3_flag_host) return apply_fast_launch(p, x, ldx, y, ldy, nrhs, s);
  return INVOP_OK;
}

}  // namespace invop
