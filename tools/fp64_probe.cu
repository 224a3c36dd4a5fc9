// fp64 latency / issue probe on one warp (B200): dependent chains of DADD,
// DMUL, DFMA, mixed chains, and a DADD chain with independent fp64 / integer
// work between consecutive links. Prints cycles per chain link.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cstdint>
#define IT 20000
template <int MODE>
__global__ void k(double* out, double a, double b, unsigned u, long long* cyc) {
  double x = a, y = b, z = a * 0.5, w0 = b * 3, w1 = b * 5, w2 = b * 7, w3 = b * 11;
  unsigned i0 = u, i1 = u * 3, i2 = u * 5, i3 = u * 7;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) x = __dadd_rn(x, y);
      if (MODE == 1) x = __dmul_rn(x, y);
      if (MODE == 2) x = __fma_rn(x, y, z);
      if (MODE == 3) { double t = __dmul_rn(x, y); x = __dadd_rn(t, z); }              // 2 links
      if (MODE == 4) { double c = __fma_rn(x, y, z); double t = __dmul_rn(c, y); x = __dadd_rn(x, t); }  // FMA->MUL->ADD, chain through x
      if (MODE == 5) { x = __dadd_rn(x, y); w0 = __dmul_rn(w0, y); }                   // +1 independent DMUL
      if (MODE == 6) { x = __dadd_rn(x, y); w0 = __dmul_rn(w0, y); w1 = __fma_rn(w1, y, z); }   // +2 independent
      if (MODE == 7) { x = __dadd_rn(x, y); w0 = __dmul_rn(w0, y); w1 = __fma_rn(w1, y, z); w2 = __dmul_rn(w2, y); }  // +3
      if (MODE == 8) { x = __dadd_rn(x, y); i0 = __byte_perm(i0, i1, 0x5140); i1 = i1 * 3 + i0; i2 = __byte_perm(i2, i3, 0x7362); i3 ^= i2; }  // +4 int
      if (MODE == 9) { x = __dadd_rn(x, y); w0 = __dmul_rn(w0, y); w1 = __fma_rn(w1, y, z);
                       i0 = __byte_perm(i0, i1, 0x5140); i1 = i1 * 3 + i0; i2 = __byte_perm(i2, i3, 0x7362); i3 ^= i2; }  // realistic mix: 3 fp64 + 4 int
      if (MODE == 10) { // independent products feeding the chain with distance: t computed from w (independent), added to x
        double t = __dmul_rn(w0, y); w0 = __fma_rn(w0, y, z); x = __dadd_rn(x, t); }
    }
  }
  long long t1 = clock64();
  out[threadIdx.x & 31] = x + w0 + w1 + w2 + w3 + (double)(i0 ^ i1 ^ i2 ^ i3);
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int MODE>
void run(const char* name, double* o, long long* c, int links) {
  printf("%-58s", name);
  for (int threads : {32, 64, 128, 256}) {       // warps per SM: 1, 2, 4 (one per scheduler), 8
    k<MODE><<<148, threads>>>(o, 1.0, 1.0000001, 12345u, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf(" %6.2f", h / (double)(IT * 8));
  }
  printf("  cycles per step at 1/2/4/8 warps per SM\n");
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMalloc(&c, 16);
  run<0>("DADD chain", o, c, 1);
  run<1>("DMUL chain", o, c, 1);
  run<2>("DFMA chain", o, c, 1);
  run<3>("DMUL->DADD chain (2 links per step)", o, c, 2);
  run<4>("DFMA->DMUL->DADD, all dependent (3 links per step)", o, c, 3);
  run<5>("DADD chain + 1 independent DMUL per link", o, c, 1);
  run<6>("DADD chain + 2 independent fp64 per link", o, c, 1);
  run<7>("DADD chain + 3 independent fp64 per link", o, c, 1);
  run<8>("DADD chain + 4 integer ops per link", o, c, 1);
  run<9>("DADD chain + 2 fp64 + 4 integer per link", o, c, 1);
  run<10>("DADD chain fed by DMUL of an independent DFMA chain", o, c, 1);
  return 0;
}
