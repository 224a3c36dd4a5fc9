// Launch/sync cost of cluster kernels on B200 (probe for the K3 side kernels).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_probe tools/cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_plain(float* out) {
  if (threadIdx.x == 0 && out) out[blockIdx.y * gridDim.x + blockIdx.x] = 1.0f;
}
__global__ void k_cluster(float* out, int syncs) {
  cg::cluster_group cl = cg::this_cluster();
  for (int i = 0; i < syncs; ++i) cl.sync();
  if (threadIdx.x == 0 && out) out[blockIdx.y * gridDim.x + blockIdx.x] = 1.0f;
}
__global__ void k_copy(const float4* __restrict__ in, float4* __restrict__ o, long n4) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  for (; i < n4; i += (long)gridDim.x * blockDim.x) o[i] = in[i];
}

static float time_it(void (*f)(cudaStream_t), int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) f(0);
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) f(0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.0f / iters;
}
static float* g_out;
static int g_cl = 16, g_syncs = 0, g_thr = 256;
static void run_cluster(cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16, 64); cfg.blockDim = dim3(g_thr); cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = g_cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_cluster, g_out, g_syncs);
}
static void run_plain(cudaStream_t s) { k_plain<<<dim3(16, 64), g_thr, 0, s>>>(g_out); }
static float4 *g_in4, *g_o4;
static long g_n4;
static void run_copy(cudaStream_t s) { k_copy<<<148 * 8, 256, 0, s>>>(g_in4, g_o4, g_n4); }

int main() {
  cudaMalloc(&g_out, 1 << 20);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("plain grid(16,64)x256: %.2f us\n", time_it(run_plain, 200));
  for (int cl : {1, 2, 4, 8, 16}) {
    for (int sy : {0, 1, 3}) {
      g_cl = cl; g_syncs = sy;
      printf("cluster %2d syncs %d: %.2f us (%s)\n", cl, sy, time_it(run_cluster, 200),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  g_n4 = (16L << 20) / 16;   // 16 MB
  cudaMalloc(&g_in4, g_n4 * 16); cudaMalloc(&g_o4, g_n4 * 16);
  printf("copy 16 MB: %.2f us\n", time_it(run_copy, 200));
  g_n4 = (64L << 20) / 16;
  cudaFree(g_in4); cudaFree(g_o4);
  cudaMalloc(&g_in4, g_n4 * 16); cudaMalloc(&g_o4, g_n4 * 16);
  printf("copy 64 MB: %.2f us\n", time_it(run_copy, 200));
  return 0;
}
