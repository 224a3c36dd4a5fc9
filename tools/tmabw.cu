// Copy-engine probe: how fast can one CTA per SM stream a buffer into shared
// memory with (a) 1-D bulk copies of CHUNK bytes and (b) 2-D tensor copies of
// INNER x ROWS byte boxes (pitch = PITCH)? Answers whether small boxes / short
// rows cap the stream below the HBM rate.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tmabw tools/tmabw.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}" ::"r"(bar), "r"(ph) : "memory");
}

// nreq requests of `chunk` bytes fill one stage; S stages
__global__ void rd_bulk(const uint8_t* __restrict__ p, size_t bytes, unsigned chunk, unsigned nreq, int S, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const unsigned stage = chunk * nreq;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t bb = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb + 8 * i));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  size_t n = bytes / stage;
  size_t c0 = (size_t)blockIdx.x * n / gridDim.x, c1 = (size_t)(blockIdx.x + 1) * n / gridDim.x;
  unsigned acc = 0;
  auto issue = [&](size_t c) {
    int st = (c - c0) % S;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb + 8 * st), "r"(stage));
    for (unsigned r = 0; r < nreq; ++r)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sb + st * stage + r * chunk), "l"(p + c * stage + (size_t)r * chunk), "r"(chunk), "r"(bb + 8 * st) : "memory");
  };
  if (threadIdx.x == 0)
    for (size_t c = c0; c < c1 && c < c0 + S; ++c) issue(c);
  for (size_t c = c0; c < c1; ++c) {
    int st = (c - c0) % S; unsigned ph = ((c - c0) / S) & 1;
    wait(bb + 8 * st, ph);
    acc ^= ((unsigned*)(sm + st * stage))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && c + S < c1) issue(c + S);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// boxes of inner x rows bytes; nbox boxes per stage (stacked along rows)
__global__ void rd_tma(const __grid_constant__ CUtensorMap map, size_t total_rows, unsigned inner, unsigned rows, unsigned nbox, int S, unsigned ncolblk, unsigned* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const unsigned box = inner * rows, stage = box * nbox;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t bb = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb + 8 * i));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // work item = (row block of rows*nbox, column block)
  size_t n = total_rows / (rows * nbox) * ncolblk;
  size_t c0 = (size_t)blockIdx.x * n / gridDim.x, c1 = (size_t)(blockIdx.x + 1) * n / gridDim.x;
  unsigned acc = 0;
  auto issue = [&](size_t c) {
    int st = (c - c0) % S;
    size_t rb = c / ncolblk; unsigned cb = c % ncolblk;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb + 8 * st), "r"(stage));
    for (unsigned r = 0; r < nbox; ++r)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(sb + st * stage + r * box), "l"(&map), "r"((int)(cb * inner)), "r"((int)(rb * rows * nbox + r * rows)), "r"(bb + 8 * st) : "memory");
  };
  if (threadIdx.x == 0)
    for (size_t c = c0; c < c1 && c < c0 + S; ++c) issue(c);
  for (size_t c = c0; c < c1; ++c) {
    int st = (c - c0) % S; unsigned ph = ((c - c0) / S) & 1;
    wait(bb + 8 * st, ph);
    acc ^= ((unsigned*)(sm + st * stage))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && c + S < c1) issue(c + S);
  }
  if (acc == 0x12345678u) out[0] = acc;
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  size_t bytes = 805306368;
  uint8_t* p; unsigned* o;
  cudaMalloc(&p, bytes); cudaMalloc(&o, 4); cudaMemset(p, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fp, 12000, cudaEnableDefault, &q);
  PFN enc = (PFN)fp;
  const int S = 4;
  // (a) bulk copies: stage 32 KB made of nreq requests
  for (unsigned chunk : {128u, 256u, 512u, 1024u, 4096u, 16384u, 32768u}) {
    unsigned nreq = 32768 / chunk;
    size_t smem = (size_t)S * 32768;
    cudaFuncSetAttribute(rd_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int w = 0; w < 2; ++w) rd_bulk<<<sms, 128, smem>>>(p, bytes, chunk, nreq, S, o);
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) rd_bulk<<<sms, 128, smem>>>(p, bytes, chunk, nreq, S, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("bulk chunk=%6u x %4u per 32 KB stage: %.1f GB/s (%.1f us) %s\n", chunk, nreq, bytes * 10 / (ms * 1e-3) / 1e9, ms * 1e3 / 10, cudaGetErrorString(cudaGetLastError()));
  }
  // (b) 2-D boxes. pitch 16384 (row-major planes) or pitch = inner (pre-tiled, contiguous boxes)
  struct Cfg { unsigned inner, rows, nbox; size_t pitch; CUtensorMapSwizzle sw; const char* name; };
  Cfg cfgs[] = {
      {128, 32, 8, 16384, CU_TENSOR_MAP_SWIZZLE_128B, "planes 128Bx32 sw128 x8"},
      {128, 64, 4, 16384, CU_TENSOR_MAP_SWIZZLE_128B, "planes 128Bx64 sw128 x4"},
      {128, 128, 2, 16384, CU_TENSOR_MAP_SWIZZLE_128B, "planes 128Bx128 sw128 x2"},
      {128, 256, 1, 16384, CU_TENSOR_MAP_SWIZZLE_128B, "planes 128Bx256 sw128 x1"},
      {256, 32, 4, 16384, CU_TENSOR_MAP_SWIZZLE_NONE, "planes 256Bx32 none x4"},
      {256, 128, 1, 16384, CU_TENSOR_MAP_SWIZZLE_NONE, "planes 256Bx128 none x1"},
      {64, 256, 2, 64, CU_TENSOR_MAP_SWIZZLE_64B, "tiled 64Bx256 sw64 x2 (K3)"},
      {64, 256, 2, 64, CU_TENSOR_MAP_SWIZZLE_NONE, "tiled 64Bx256 none x2"},
      {128, 256, 1, 128, CU_TENSOR_MAP_SWIZZLE_128B, "tiled 128Bx256 sw128 x1"},
      {128, 32, 8, 128, CU_TENSOR_MAP_SWIZZLE_128B, "tiled 128Bx32 sw128 x8"},
  };
  for (auto& c : cfgs) {
    size_t total_rows = bytes / c.pitch;
    unsigned ncolblk = (unsigned)(c.pitch / c.inner);
    CUtensorMap m;
    cuuint64_t dims[2] = {c.pitch, total_rows};
    cuuint64_t strides[1] = {c.pitch};
    cuuint32_t box[2] = {c.inner, c.rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", c.name, (int)r); continue; }
    size_t smem = (size_t)S * c.inner * c.rows * c.nbox;
    cudaFuncSetAttribute(rd_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int w = 0; w < 2; ++w) rd_tma<<<sms, 128, smem>>>(m, total_rows, c.inner, c.rows, c.nbox, S, ncolblk, o);
    cudaEventRecord(a);
    for (int rr = 0; rr < 10; ++rr) rd_tma<<<sms, 128, smem>>>(m, total_rows, c.inner, c.rows, c.nbox, S, ncolblk, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("tma  %-28s stage %u KB: %.1f GB/s (%.1f us) %s\n", c.name, c.inner * c.rows * c.nbox / 1024, bytes * 10 / (ms * 1e-3) / 1e9, ms * 1e3 / 10, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
