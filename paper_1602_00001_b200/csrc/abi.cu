// C ABI plumbing of libinvop_b200: errors, plan lifetime, apply entry points.
#include "common.cuh"
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

namespace invop {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static std::atomic<long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return INVOP_E_CUDA;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 1;
  }
  return cached[dev];
}

int ensure_scratch(void** ptr, size_t* have, size_t need) {
  if (*have >= need && *ptr) return INVOP_OK;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *have = 0;
  INVOP_CUDA(cudaMalloc(ptr, need > 0 ? need : 16));
  *have = need;
  return INVOP_OK;
}

}  // namespace invop

using namespace invop;

extern "C" const char* invop_last_error(void) { return g_last_error.c_str(); }

extern "C" int invop_abi_version(void) { return 1; }

extern "C" int64_t invop_launch_count(void) { return invop::g_launches.load(); }

extern "C" int invop_plan_destroy(invop_plan* p) {
  if (!p) return INVOP_OK;
  for (int b = 0; b < INVOP_MAX_PLANES; ++b)
    if (p->planes[b]) cudaFree(p->planes[b]);
  if (p->partial) cudaFree(p->partial);
  if (p->counters) cudaFree(p->counters);
  if (p->dev_x) cudaFree(p->dev_x);
  if (p->k3_flag_host) cudaFreeHost(p->k3_flag_host);
  if (p->k3_flag_event) cudaEventDestroy(p->k3_flag_event);
  if (p->dev_y) cudaFree(p->dev_y);
  if (p->k3_ws) cudaFree(p->k3_ws);
  for (int b = 0; b < 2; ++b)
    if (p->k3_tiles[b]) cudaFree(p->k3_tiles[b]);
  if (p->vw_data) cudaFree(p->vw_data);
  if (p->vw_meta) cudaFree(p->vw_meta);
  if (p->vw_rowptr) cudaFree(p->vw_rowptr);
  if (p->vw_slaboff) cudaFree(p->vw_slaboff);
  if (p->tv_data) cudaFree(p->tv_data);
  if (p->tv_meta) cudaFree(p->tv_meta);
  if (p->tv_gptr) cudaFree(p->tv_gptr);
  if (p->tv_soff) cudaFree(p->tv_soff);
  if (p->tv_ws) cudaFree(p->tv_ws);
  if (p->hl_data) cudaFree(p->hl_data);
  if (p->hl_rowptr) cudaFree(p->hl_rowptr);
  for (int b = 0; b < 2; ++b)
    if (p->k3d_tiles[b]) cudaFree(p->k3d_tiles[b]);
  if (p->k3d_idx1) cudaFree(p->k3d_idx1);
  if (p->dl_data) cudaFree(p->dl_data);
  if (p->dl_uoff) cudaFree(p->dl_uoff);
  if (p->dl_rowlo) cudaFree(p->dl_rowlo);
  if (p->host_pinned) cudaFreeHost(p->host_pinned);
  delete p;
  return INVOP_OK;
}

extern "C" int invop_plan_info(const invop_plan* p, int64_t* n, int64_t* rows, int64_t* row0,
                               int* scale_digits, int* code_bytes, int* is_signed,
                               int64_t* device_bytes, int64_t* max_abs) {
  if (!p) return fail(INVOP_E_VALUE, "plan is NULL");
  if (n) *n = p->n;
  if (rows) *rows = p->rows;
  if (row0) *row0 = p->row0;
  if (scale_digits) *scale_digits = p->digits;
  if (code_bytes) *code_bytes = p->P;
  if (is_signed) *is_signed = p->is_signed;
  if (device_bytes) *device_bytes = (int64_t)p->P * p->rows * p->ld;
  if (max_abs) *max_abs = p->max_abs;
  return INVOP_OK;
}

static bool aligned16(const void* ptr) { return ((uintptr_t)ptr & 15u) == 0; }

static bool layout_enabled(const char* env, bool dflt) {
  const char* v = getenv(env);
  if (!v || !*v) return dflt;
  return *v != '0';
}

// Which kernel serves a fast-mode apply. Single right-hand side over long
// rows: 3-byte codes take the HL layout (default; INVOP_HL=0 disables), TVW
// and VW are opt-in (INVOP_TVW=1 / INVOP_VW=1); everything else streams the
// byte planes (k2_stream / k2_fast). Many right-hand sides of <= 2-byte codes
// go to the tensor-core kernel (K3; INVOP_NO_TC=1 disables).
enum { ROUTE_PLANES = 0, ROUTE_K3, ROUTE_DL, ROUTE_HL, ROUTE_TVW, ROUTE_VW };

static int fast_route(const invop_plan* p, int64_t nrhs) {
  if (!layout_enabled("INVOP_NO_TC", false) && batched_supported(p, nrhs)) return ROUTE_K3;
  if (nrhs != 1 || p->ld / 512 < 16) return ROUTE_PLANES;
  if (p->P <= 3 && p->dl_ready >= 0 && layout_enabled("INVOP_DL", true)) return ROUTE_DL;
  if (p->P == 3 && p->ld <= 16384 && p->hl_ready >= 0 && layout_enabled("INVOP_HL", true))
    return ROUTE_HL;
  if (p->tv_ready >= 0 && layout_enabled("INVOP_TVW", false)) return ROUTE_TVW;
  if (p->vw_ready >= 0 && layout_enabled("INVOP_VW", false)) return ROUTE_VW;
  return ROUTE_PLANES;
}

extern "C" const char* invop_apply_kernel(const invop_plan* p, int64_t nrhs, int mode) {
  if (!p) return "";
  if (mode == INVOP_MODE_ORDERED) return "k2_ordered";
  switch (fast_route(p, nrhs)) {
    case ROUTE_K3: return k3d_bytes(p) > 0 ? "k3_batched_dl" : "k3_batched";
    case ROUTE_DL: return "k2_dl";
    case ROUTE_HL: return "k2_hl";
    case ROUTE_TVW: return "k2_tvw";
    case ROUTE_VW: return "k2_vw";
    default: return stream_selected(p, nrhs) ? "k2_stream" : "k2_fast";
  }
}

extern "C" int invop_apply(const invop_plan* p, const void* x, int64_t ldx, void* y,
                           int64_t ldy, int64_t nrhs, int dtype, int mode, void* stream) {
  if (!p) return fail(INVOP_E_VALUE, "plan is NULL");
  if (nrhs < 0) return fail(INVOP_E_VALUE, "nrhs < 0");
  if (nrhs > 1 && (ldx < p->n || ldy < p->rows))
    return fail(INVOP_E_VALUE, "leading dimensions too small");
  if (nrhs == 0 || p->rows == 0) return INVOP_OK;
  if ((!x && p->n > 0) || !y) return fail(INVOP_E_VALUE, "NULL vector");
  cudaStream_t s = (cudaStream_t)stream;
  if (p->n == 0) {
    // empty operator: rows == 0 handled above
    return INVOP_OK;
  }
  if (mode == INVOP_MODE_ORDERED) {
    if (dtype != INVOP_F64)
      return fail(INVOP_E_VALUE, "ordered (bitwise) mode computes in fp64: dtype must be F64");
    if (!aligned16(x) || (nrhs > 1 && (ldx & 1)))
      return fail(INVOP_E_VALUE, "x must be 16-byte aligned with an even leading dimension");
    return apply_ordered_launch(p, (const double*)x, nrhs > 1 ? ldx : p->n, (double*)y,
                                nrhs > 1 ? ldy : p->rows, nrhs, s);
  }
  if (mode == INVOP_MODE_FAST) {
    if (dtype != INVOP_F32) return fail(INVOP_E_VALUE, "fast mode computes in fp32: dtype F32");
    invop_plan* mp = const_cast<invop_plan*>(p);
    const int route = fast_route(p, nrhs);
    if (route == ROUTE_K3)
      return apply_batched_launch(mp, (const float*)x, nrhs > 1 ? ldx : p->n, (float*)y,
                                  nrhs > 1 ? ldy : p->rows, nrhs, s);
    if (route != ROUTE_PLANES) {
      int rc = route == ROUTE_DL ? dl_build(mp, s) : route == ROUTE_HL ? hl_build(mp, s)
             : route == ROUTE_TVW ? tvw_build(mp, s) : vw_build(mp, s);
      if (rc == INVOP_OK) {
        rc = route == ROUTE_DL ? apply_dl_launch(mp, x, y, false, s)
           : route == ROUTE_HL ? apply_hl_launch(mp, (const float*)x, (float*)y, s)
           : route == ROUTE_TVW ? apply_tvw_launch(mp, (const float*)x, (float*)y, s)
                                : apply_vw_launch(mp, (const float*)x, (float*)y, s);
      }
      if (rc != INVOP_E_UNSUPPORTED) return rc;
      if (route == ROUTE_HL) mp->hl_ready = -1;
      if (route == ROUTE_DL) mp->dl_ready = -1;
      if (route == ROUTE_DL || route == ROUTE_HL)
        return invop_apply(p, x, ldx, y, ldy, nrhs, dtype, mode, stream);   // next route
      // layout not applicable to this plan: plain byte planes below
    }
    return apply_fast_launch(p, (const float*)x, nrhs > 1 ? ldx : p->n, (float*)y,
                             nrhs > 1 ? ldy : p->rows, nrhs, s);
  }
  return fail(INVOP_E_VALUE, "unknown mode");
}

extern "C" int invop_plan_apply_bytes(invop_plan* p, int64_t nrhs, int mode, int64_t* bytes,
                                      void* stream) {
  // bytes of operator data one fast/ordered apply streams from HBM (the
  // roofline numerator), building the lazily created layouts first
  if (!p || !bytes) return fail(INVOP_E_VALUE, "NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == INVOP_MODE_FAST) {
    const int route = fast_route(p, nrhs);
    if (route == ROUTE_K3 && k3d_bytes(p) > 0) {
      *bytes = k3d_bytes(p);
      return INVOP_OK;
    }
    int rc = route == ROUTE_DL ? dl_build(p, s) : route == ROUTE_HL ? hl_build(p, s)
           : route == ROUTE_TVW ? tvw_build(p, s) : route == ROUTE_VW ? vw_build(p, s)
           : INVOP_E_UNSUPPORTED;
    if (rc == INVOP_E_UNSUPPORTED && (route == ROUTE_DL || route == ROUTE_HL))
      return invop_plan_apply_bytes(p, nrhs, mode, bytes, stream);   // next route
    if (rc == INVOP_OK) {
      if (route == ROUTE_DL) {
        *bytes = p->dl_bytes + (p->rows * p->dl_nslabs + 1) * 8;
      } else if (route == ROUTE_HL) {
        *bytes = p->hl_bytes + (p->rows + 1) * 8;
      } else if (route == ROUTE_TVW) {
        *bytes = tvw_stream_bytes(p);
      } else {
        const int64_t nch = p->ld / 512, nchp = (nch + 1) & ~1;
        *bytes = p->vw_bytes + p->rows * nchp * 8 + (p->rows + 1) * 8;
      }
      return INVOP_OK;
    }
    if (rc != INVOP_E_UNSUPPORTED) return rc;
  }
  *bytes = (int64_t)p->P * p->rows * p->ld;
  return INVOP_OK;
}

__global__ void k_f64_to_f32(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}
__global__ void k_f32_to_f64(const float* __restrict__ a, double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (double)a[i];
}

// x from page-locked host memory (mapped) into device memory; the dependent
// apply grid may launch immediately
__global__ void k_pull_x(const double* __restrict__ xh, double* __restrict__ xd, int64_t n) {
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t n2 = n / 2;
  const double2* h2 = reinterpret_cast<const double2*>(xh);
  double2* d2 = reinterpret_cast<double2*>(xd);
  const bool vec = ((reinterpret_cast<uintptr_t>(xh) | reinterpret_cast<uintptr_t>(xd)) & 15) == 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (vec ? n2 : 0);
       i += (int64_t)gridDim.x * blockDim.x)
    d2[i] = h2[i];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + (vec ? 2 * n2 : 0); i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    xd[i] = xh[i];
}

// device alias of page-locked (mapped) host memory; false for pageable memory
static bool host_alias(const void* ptr, void** alias) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess || at.type != cudaMemoryTypeHost ||
      !at.devicePointer) {
    cudaGetLastError();
    return false;
  }
  *alias = at.devicePointer;
  return true;
}

extern "C" int invop_apply_host(invop_plan* p, const double* x, double* y, int64_t nrhs,
                                int mode, void* stream) {
  if (!p) return fail(INVOP_E_VALUE, "plan is NULL");
  if (nrhs <= 0 || p->rows == 0) return INVOP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  size_t xb = (size_t)nrhs * p->n * sizeof(double);
  size_t yb = (size_t)nrhs * p->rows * sizeof(double);
  void* ydev = nullptr;
  if (mode == INVOP_MODE_FAST && nrhs == 1 && fast_route(p, 1) == ROUTE_DL &&
      dl_build(p, s) == INVOP_OK && host_alias(y, &ydev)) {
    // page-locked y: the DL kernel writes its fp64 rows straight into host
    // memory (each row once; zero copy). x is read by every CTA, so it is
    // staged in device memory: page-locked x is pulled over PCIe by a small
    // grid that lets the apply grid start at once (programmatic dependent
    // launch: the producer streams the operator while x arrives; the
    // consumers wait for it); otherwise one H2D copy. (Polling a mapped
    // completion word published by the grid's last CTA instead of
    // synchronising the stream was measured slower: the system-scope fences
    // at the grid's tail cost more than the synchronisation.)
    int rc = ensure_scratch(&p->dev_x, &p->dev_x_bytes, xb + 64);
    if (rc) return rc;
    void* xdev = nullptr;
    const bool pdl = host_alias(x, &xdev);
    if (pdl) {
      k_pull_x<<<(unsigned)std::min<int64_t>(cdiv(p->n, 512), 64), 256, 0, s>>>(
          (const double*)xdev, (double*)p->dev_x, p->n);
      INVOP_LAUNCHED(1);
    } else {
      INVOP_CUDA(cudaMemcpyAsync(p->dev_x, x, xb, cudaMemcpyHostToDevice, s));
    }
    rc = apply_dl_launch(p, p->dev_x, ydev, true, s, pdl);
    if (rc == INVOP_OK) {
      INVOP_CUDA(cudaStreamSynchronize(s));
      return INVOP_OK;
    }
    cudaGetLastError();
  }
  // fp64 staging + fp32 copies for the fast path
  int rc = ensure_scratch(&p->dev_x, &p->dev_x_bytes, xb + xb / 2 + 64);
  if (rc) return rc;
  rc = ensure_scratch(&p->dev_y, &p->dev_y_bytes, yb + yb / 2 + 64);
  if (rc) return rc;
  double* dx = (double*)p->dev_x;
  double* dy = (double*)p->dev_y;
  INVOP_CUDA(cudaMemcpyAsync(dx, x, xb, cudaMemcpyHostToDevice, s));
  if (mode == INVOP_MODE_ORDERED) {
    rc = invop_apply(p, dx, p->n, dy, p->rows, nrhs, INVOP_F64, mode, stream);
    if (rc) return rc;
  } else if (nrhs == 1 && fast_route(p, 1) == ROUTE_DL && dl_build(p, s) == INVOP_OK &&
             apply_dl_launch(p, dx, dy, true, s) == INVOP_OK) {
    // DL kernel reads the fp64 x and writes the fp64 y itself (same values as
    // the fp32 path: x rounded to fp32 on load, y widened from fp32)
  } else {
    float* fx = (float*)((char*)p->dev_x + ((xb + 15) & ~(size_t)15));
    float* fy = (float*)((char*)p->dev_y + ((yb + 15) & ~(size_t)15));
    int64_t nx = nrhs * p->n, ny = nrhs * p->rows;
    k_f64_to_f32<<<(unsigned)std::min<int64_t>(cdiv(nx, 256), 4096), 256, 0, s>>>(dx, fx, nx);
    INVOP_LAUNCHED(2);   // + k_f32_to_f64 below
    rc = invop_apply(p, fx, p->n, fy, p->rows, nrhs, INVOP_F32, mode, stream);
    if (rc) return rc;
    k_f32_to_f64<<<(unsigned)std::min<int64_t>(cdiv(ny, 256), 4096), 256, 0, s>>>(fy, dy, ny);
  }
  INVOP_CUDA(cudaMemcpyAsync(y, dy, yb, cudaMemcpyDeviceToHost, s));
  INVOP_CUDA(cudaStreamSynchronize(s));
  return INVOP_OK;
}

extern "C" int invop_apply_naive(const invop_plan* p, const double* x, double* y, int64_t nrhs,
                                 void* stream) {
  // apply_naive_quantized (applyplan.py:194-209) accumulates mant*scale*x_j per
  // nonzero in ascending column order: the arithmetic of ORDERED mode.
  if (!p) return fail(INVOP_E_VALUE, "plan is NULL");
  return invop_apply(p, x, p->n, y, p->rows, nrhs, INVOP_F64, INVOP_MODE_ORDERED, stream);
}
