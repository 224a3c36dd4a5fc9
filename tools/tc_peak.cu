// int8 tensor-core (tcgen05.mma kind::i8) throughput probe for the K3 roofline:
// one CTA per SM issues back-to-back M=128 x N x K=32 MMAs from shared
// memory into TMEM (the K3 operand layout: 64-byte K-major rows, SWIZZLE_64B),
// for N = 64, 192 and 256. Prints TOPS (2*M*N*K per MMA) from CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_peak tools/tc_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, int* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (8192 + N * 64) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warp == 1) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(base);
    const uint64_t da = desc_sw64(sa), db = desc_sw64(sa + 8192);
    constexpr uint32_t id = idesc_i8(N);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da + (kk * 32 >> 4)), "l"(db + (kk * 32 >> 4)), "r"(id), "r"((i | kk) ? 1 : 0));
      }
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra W_%=;\n}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar))
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (threadIdx.x == 0) sink[blockIdx.x] = (int)r;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

template <int N>
static double run(int sms, int iters) {
  int* sink;
  cudaMalloc(&sink, sms * 4);
  size_t smem = 1024 + 8192 + N * 64;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<N><<<sms, 128, smem>>>(100, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<N><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int h = 0;
  cudaMemcpy(&h, sink, 4, cudaMemcpyDeviceToHost);
  const double ops = 2.0 * 128 * N * 32 * 2.0 * iters * sms;
  printf("N=%d: %.3f ms, %.1f TOPS (acc[0]=%d, expect %d)\n", N, ms, ops / (ms * 1e-3) / 1e12, h,
         64 * iters);
  cudaFree(sink);
  return ops / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 200000;
  double t64 = run<64>(sms, iters);
  double t192 = run<192>(sms, iters);
  double t256 = run<256>(sms, iters);
  cudaError_t e = cudaGetLastError();
  printf("{\"tops\": %.1f, \"tops_n192\": %.1f, \"tops_n64\": %.1f, \"sms\": %d, \"how\": \"tcgen05.mma.cta_group::1.kind::i8 M=128 K=32 back to back from SMEM, one CTA per SM, CUDA events\", \"err\": \"%s\"}\n",
         t256, t192, t64, sms, cudaGetErrorString(e));
  return 0;
}
