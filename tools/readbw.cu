// Read-bandwidth ceiling probe: how fast can a B200 stream N bytes with
// (a) plain LDG.128 (many in flight) and (b) bulk copies into shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void rd_ldg(const uint4* __restrict__ p, size_t n16, unsigned* out) {
  unsigned acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(p + i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p + i + stride));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(p + i + 2 * stride));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(d.x), "=r"(d.y), "=r"(d.z), "=r"(d.w) : "l"(p + i + 3 * stride));
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n16; i += stride) acc ^= p[i].x;
  if (acc == 0x12345678u) out[0] = acc;
}
__global__ void rd_bulk(const uint8_t* __restrict__ p, size_t bytes, size_t chunk, unsigned* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[8];
  const int S = 4;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t bb = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bb + 8 * i));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  size_t nchunks = bytes / chunk;
  size_t c0 = (size_t)blockIdx.x * nchunks / gridDim.x, c1 = (size_t)(blockIdx.x + 1) * nchunks / gridDim.x;
  unsigned acc = 0;
  if (threadIdx.x == 0) {
    for (size_t c = c0; c < c1 && c < c0 + S; ++c) {
      int st = (c - c0) % S;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bb + 8 * st), "r"((unsigned)chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sb + st * (unsigned)chunk), "l"(p + c * chunk), "r"((unsigned)chunk), "r"(bb + 8 * st) : "memory");
    }
  }
  for (size_t c = c0; c < c1; ++c) {
    int st = (c - c0) % S; unsigned ph = ((c - c0) / S) & 1;
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}" :: "r"(bb + 8 * st), "r"(ph) : "memory");
    acc ^= ((unsigned*)(sm + st * chunk))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && c + S < c1) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bb + 8 * st), "r"((unsigned)chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sb + st * (unsigned)chunk), "l"(p + (c + S) * chunk), "r"((unsigned)chunk), "r"(bb + 8 * st) : "memory");
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}
int main() {
  size_t bytes = 805306368;
  uint8_t* p; unsigned* o;
  cudaMalloc(&p, bytes); cudaMalloc(&o, 4); cudaMemset(p, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocksPerSM : {2, 4, 8}) for (int th : {256, 512, 1024}) {
    if (blocksPerSM * th > 2048) continue;
    int grid = sms * blocksPerSM;
    for (int w = 0; w < 3; ++w) rd_ldg<<<grid, th>>>((const uint4*)p, bytes / 16, o);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) rd_ldg<<<grid, th>>>((const uint4*)p, bytes / 16, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("ldg  grid=%d x %d : %.1f GB/s (%.1f us)\n", grid, th, bytes * 20 / (ms * 1e-3) / 1e9, ms * 1e3 / 20);
  }
  for (size_t chunk : {16384, 32768, 49152}) for (int bps : {1, 2}) {
    size_t smem = 4 * chunk;
    if (smem * bps > 220 * 1024) continue;
    cudaFuncSetAttribute(rd_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int grid = sms * bps;
    for (int w = 0; w < 3; ++w) rd_bulk<<<grid, 256, smem>>>(p, bytes, chunk, o);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) rd_bulk<<<grid, 256, smem>>>(p, bytes, chunk, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("bulk chunk=%zu grid=%d : %.1f GB/s (%.1f us) %s\n", chunk, grid, bytes * 20 / (ms * 1e-3) / 1e9, ms * 1e3 / 20, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
