// Shared definitions for libinvop_b200 (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include "../../include/invop_b200.h"

#define INVOP_MAX_PLANES 8

// Compressed device layout of a quantized operator shard.
//
// A mantissa v (int64) of row i, column j is stored as P little-endian bytes,
// byte b in plane b: planes[b][i*ld + j] = (v >> 8b) & 0xff. P is the smallest
// width that holds every mantissa (two's complement when any mantissa < 0).
// ld (bytes per plane row) is n rounded up to 128 so every row of every plane
// starts 128-byte aligned; padding bytes are 0. Keeping bytes in separate
// planes lets (a) the fp32 apply assemble 16-bit halves with PRMT and
// (b) the tensor-core batched apply feed each plane straight to an 8-bit MMA.
struct invop_plan {
  int64_t n = 0, rows = 0, row0 = 0, ld = 0;
  int digits = 0;
  double scale = 1.0;  // 10.0 ** -digits, bit-identical to Python's value
  int P = 1;
  int is_signed = 0;
  uint8_t* planes[INVOP_MAX_PLANES] = {nullptr};
  int64_t min_val = 0, max_val = 0, max_abs = 0;
  int64_t nnz = 0;     // planned additions (E)
  int64_t mults = -1;  // planned multiplications (G), lazily computed
  int device = 0;
  // scratch owned by the plan (grown on demand)
  float* partial = nullptr; size_t partial_bytes = 0;
  int* counters = nullptr; size_t counters_n = 0;
  void* dev_x = nullptr; size_t dev_x_bytes = 0;

  void* dev_y = nullptr; size_t dev_y_bytes = 0;
  double* host_pinned = nullptr; size_t host_pinned_bytes = 0;
  void* shard_stage = nullptr; size_t shard_stage_bytes = 0;   // sharded.cu all-gather staging
  // K3 (tensor-core batched apply): workspace and cached TMA descriptors
  void* k3_ws = nullptr; size_t k3_ws_bytes = 0;
  uint8_t* k3_tiles[3] = {nullptr, nullptr, nullptr};   // tiled copy of planes 0..2
  // HL layout (hl.cu): two low byte planes + top plane only where a chunk needs it
  uint8_t* hl_data = nullptr;
  int64_t* hl_rowptr = nullptr;     // [rows+1] byte offsets
  int64_t hl_bytes = 0;
  int hl_ready = 0;
  // DL layout (dl.cu): second-order row residuals, per-chunk byte width
  uint8_t* dl_data = nullptr;
  int64_t* dl_uoff = nullptr;       // [units+1] byte offsets, units in (CTA, slab, row) order
  int64_t dl_bytes = 0, dl_maxunit = 0;
  int dl_ready = 0, dl_grid = 0, dl_nslabs = 0, dl_groups = 1;
  int64_t* dl_rowlo = nullptr;      // [grid + 1] CTA row ranges (byte-balanced)
  int64_t dl_maxrows = 0;
  int dl_cd = 0;                    // residuals stored as column differences inside each chunk
  alignas(64) unsigned char k3_mapA[3][128];
  int k3_maps_ready = 0;
  int k3_presw = 0;                  // tiled planes stored pre-swizzled (bulk copies)
  // K3 on row residuals (batched.cu): digit-0 tiles for every (row tile, K
  // block), digit-1 tiles only where needed (compact, indexed by k3d_idx1)
  alignas(64) unsigned char k3d_mapA[2][128];
  uint8_t* k3d_tiles[2] = {nullptr, nullptr};
  int* k3d_idx1 = nullptr;
  int64_t k3d_n1 = 0;
  int64_t k3d_n1u = 0;               // (quad, K block, slot) with a digit-1 tile on either SM
  int k3d_ready = 0;
  int k3_pair = -1;                  // 1: SM-pair kernel, 0: one-SM kernel, -1: not timed yet
  int k3d_ysh = 0;                   // tensor rows of the residual tiles are 64 << k3d_ysh bytes
  // ordered kernel (ordered.cu): one 128-byte-swizzled TMA descriptor per byte
  // plane, cached with the geometry it was built for
  alignas(64) unsigned char ord_maps[INVOP_MAX_PLANES][128];
  const void* ord_maps_key = nullptr; int64_t ord_maps_geom[4] = {0, 0, 0, 0};
};

struct invop_operator {
  int64_t nx = 0, ny = 0, N = 0;
  double* diag = nullptr;  // device [N]
  double* ww = nullptr;    // device [N] west weights
  double* we = nullptr;
  double* ws = nullptr;
  double* wn = nullptr;
  double* dinv = nullptr;  // device [ny][nx][nx]: inverses of Schur blocks
  double* qmat = nullptr;  // device [ny][nx][nx]: Dinv_k * diag(up_k)
  double max_entry = 0.0;
  int factored = 0;
};

namespace invop {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define INVOP_CUDA(call)                                   \
  do {                                                     \
    cudaError_t _e = (call);                               \
    if (_e != cudaSuccess) return ::invop::cuda_fail(_e, #call); \
  } while (0)

#define INVOP_CHECK_LAUNCH(what) INVOP_CUDA(cudaGetLastError())

// kernels launched by the apply entry points (invop_apply / invop_apply_host),
// cumulative; read through invop_launch_count() by the benchmark
void count_launches(int n);
#define INVOP_LAUNCHED(n) ::invop::count_launches(n)

__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

int num_sms();
int ensure_scratch(void** ptr, size_t* have, size_t need);

// encode.cu
int encode_int64(invop_plan* p, const int64_t* mant, int64_t ldm, cudaStream_t s);
int plan_alloc_planes(invop_plan* p, int P);
int plan_finalize_width(invop_plan* p, int64_t mn, int64_t mx, int64_t nnz);
// apply kernels
int apply_fast_launch(const invop_plan* p, const float* x, int64_t ldx, float* y,
                      int64_t ldy, int64_t nrhs, cudaStream_t s);
bool batched_supported(const invop_plan* p, int64_t nrhs);
bool stream_selected(const invop_plan* p, int64_t nrhs);
int apply_batched_launch(invop_plan* p, const float* x, int64_t ldx, float* y, int64_t ldy,
                         int64_t nrhs, cudaStream_t s);
// 2-D uint8 tensor map (inner = bytes along a row); swizzle_bytes 0, 64 or 128
int make_tensor_map_u8(void* map128, const void* ptr, uint64_t inner, uint64_t outer,
                       uint64_t pitch, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes);
int64_t k3d_bytes(const invop_plan* p);
bool k3_uses_dl(const invop_plan* p);
bool k3_uses_pair(const invop_plan* p);
int64_t k3_tensor_ops(const invop_plan* p, int64_t nrhs);
int k3_prepare(invop_plan* p, cudaStream_t s);
int hl_build(invop_plan* p, cudaStream_t s);
int dl_build(invop_plan* p, cudaStream_t s);
int apply_dl_launch(invop_plan* p, const void* x, void* y, bool f64io, cudaStream_t s);
int apply_hl_launch(invop_plan* p, const float* x, float* y, cudaStream_t s);
int apply_ordered_launch(const invop_plan* p, const double* x, int64_t ldx, double* y,
                         int64_t ldy, int64_t nrhs, cudaStream_t s, bool accumulate = false);

}  // namespace invop

// exact powers of ten used by quantize (10.0 ** d for d in 0..22 is exact)
__host__ __device__ inline double invop_pow10_exact(int d) {
  double r = 1.0;
  for (int i = 0; i < d; ++i) r *= 10.0;
  return r;
}
