// Shared inline-PTX helpers (sm_100a): mbarriers, bulk copies, PRMT decode.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace invop {

__device__ __forceinline__ uint32_t u4get(const uint4& v, int w) {
  return w == 0 ? v.x : (w == 1 ? v.y : (w == 2 ? v.z : v.w));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

// 2-D tiled TMA load (tensor map in kernel parameter space), completing on an
// mbarrier of this CTA
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* map, int x, int y,
                                            uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "l"(policy)
      : "memory");
}

// acc + (int64)a * b as one IMAD.WIDE (keeps the compiler from hoisting a
// sign-extended 64-bit copy of a loop-invariant operand and multiplying 64x64)
__device__ __forceinline__ long long madw(int32_t a, int32_t b, long long c) {
  long long r;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
  return r;
}

// 4-way byte dot products with int32 accumulate: signed x signed and
// unsigned (a) x signed (b)
__device__ __forceinline__ int32_t dp4a_ss(uint32_t a, uint32_t b, int32_t c) {
  int32_t r;
  asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ int32_t dp4a_us(uint32_t a, uint32_t b, int32_t c) {
  int32_t r;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

// balanced base-256 digits of |X| <= 2^22: X = d0 + 256 d1 + 65536 d2, each
// digit in [-128, 127]; 4 consecutive values' digit d packed into word d
__device__ __forceinline__ void x_digits4(const int32_t* X, uint32_t* w) {
  uint32_t p0 = 0, p1 = 0, p2 = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int32_t x = X[i];
    const int32_t d0 = ((x + 128) & 255) - 128;
    const int32_t x1 = (x - d0) >> 8;
    const int32_t d1 = ((x1 + 128) & 255) - 128;
    const int32_t d2 = (x1 - d1) >> 8;
    p0 |= (uint32_t)(d0 & 255) << (8 * i);
    p1 |= (uint32_t)(d1 & 255) << (8 * i);
    p2 |= (uint32_t)(d2 & 255) << (8 * i);
  }
  w[0] = p0; w[1] = p1; w[2] = p2;
}

// balanced base-256 digits of |X| < 2^31 - 2^23: four digits, packed like x_digits4
__device__ __forceinline__ void x_digits4w(const int32_t* X, uint32_t* w) {
  uint32_t p0 = 0, p1 = 0, p2 = 0, p3 = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int32_t x = X[i];
    const int32_t d0 = ((x + 128) & 255) - 128;
    const int32_t x1 = (x - d0) >> 8;
    const int32_t d1 = ((x1 + 128) & 255) - 128;
    const int32_t x2 = (x1 - d1) >> 8;
    const int32_t d2 = ((x2 + 128) & 255) - 128;
    const int32_t d3 = (x2 - d2) >> 8;
    p0 |= (uint32_t)(d0 & 255) << (8 * i);
    p1 |= (uint32_t)(d1 & 255) << (8 * i);
    p2 |= (uint32_t)(d2 & 255) << (8 * i);
    p3 |= (uint32_t)(d3 & 255) << (8 * i);
  }
  w[0] = p0; w[1] = p1; w[2] = p2; w[3] = p3;
}

// PRMT with the full selector nibble (bit 3 = replicate the sign of the
// selected byte); __byte_perm only honours the low 3 bits of each nibble.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// 4 integer mantissas from the P plane words (byte q of word b = byte b of
// code q). SIGNED: two's complement, sign-extended with PRMT's replicate mode.
template <int P, bool SIGNED>
__device__ __forceinline__ void dec_int4(const uint32_t* wds, int32_t* u) {
  if (P == 1) {
    const uint32_t a = wds[0];
    if (SIGNED) {
      u[0] = (int32_t)prmt(a, 0, 0x8880); u[1] = (int32_t)prmt(a, 0, 0x9991);
      u[2] = (int32_t)prmt(a, 0, 0xAAA2); u[3] = (int32_t)prmt(a, 0, 0xBBB3);
    } else {
      u[0] = (int32_t)prmt(a, 0, 0x4440); u[1] = (int32_t)prmt(a, 0, 0x4441);
      u[2] = (int32_t)prmt(a, 0, 0x4442); u[3] = (int32_t)prmt(a, 0, 0x4443);
    }
  } else if (P == 2) {
    const uint32_t t01 = prmt(wds[0], wds[1], 0x5140);   // [a0 b0 a1 b1]
    const uint32_t t23 = prmt(wds[0], wds[1], 0x7362);   // [a2 b2 a3 b3]
    if (SIGNED) {
      u[0] = (int32_t)prmt(t01, 0, 0x9910); u[1] = (int32_t)prmt(t01, 0, 0xBB32);
      u[2] = (int32_t)prmt(t23, 0, 0x9910); u[3] = (int32_t)prmt(t23, 0, 0xBB32);
    } else {
      u[0] = (int32_t)(t01 & 0xffffu); u[1] = (int32_t)(t01 >> 16);
      u[2] = (int32_t)(t23 & 0xffffu); u[3] = (int32_t)(t23 >> 16);
    }
  } else {
    const uint32_t t01 = prmt(wds[0], wds[1], 0x5140);
    const uint32_t t23 = prmt(wds[0], wds[1], 0x7362);
    const uint32_t c = wds[2];
    if (P == 3) {
      if (SIGNED) {
        u[0] = (int32_t)prmt(t01, c, 0xC410); u[1] = (int32_t)prmt(t01, c, 0xD532);
        u[2] = (int32_t)prmt(t23, c, 0xE610); u[3] = (int32_t)prmt(t23, c, 0xF732);
      } else {
        u[0] = (int32_t)(prmt(t01, c, 0x0410) & 0xffffffu);
        u[1] = (int32_t)(prmt(t01, c, 0x0532) & 0xffffffu);
        u[2] = (int32_t)(prmt(t23, c, 0x0610) & 0xffffffu);
        u[3] = (int32_t)(prmt(t23, c, 0x0732) & 0xffffffu);
      }
    } else {
      const uint32_t h01 = prmt(wds[2], wds[3], 0x5140);
      const uint32_t h23 = prmt(wds[2], wds[3], 0x7362);
      u[0] = (int32_t)prmt(t01, h01, 0x5410); u[1] = (int32_t)prmt(t01, h01, 0x7632);
      u[2] = (int32_t)prmt(t23, h23, 0x5410); u[3] = (int32_t)prmt(t23, h23, 0x7632);
    }
  }
}

}  // namespace invop
