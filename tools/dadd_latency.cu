// fp64 dependent-chain latency probe (DADD and DMUL) on one warp
#include <cstdio>
__global__ void chain(double* out, double a, double b, int iters, long long* cyc) {
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __dadd_rn(x, y); x = __dadd_rn(x, -y); }
  long long t1 = clock64();
  double z = a;
  for (int i = 0; i < iters; ++i) { z = __dmul_rn(z, b); z = __dmul_rn(z, 1.0 / b); }
  long long t2 = clock64();
  out[threadIdx.x] = x + z;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMalloc(&c, 16);
  const int it = 100000;
  chain<<<1, 32>>>(o, 1.0, 1e-3, it, c);
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles; DMUL: %.2f cycles\n", h[0] / (2.0 * it), h[1] / (2.0 * it));
  return 0;
}
