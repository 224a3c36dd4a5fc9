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
  if (p->dev_y) cudaFree(p->dev_y);
  if (p->k3_ws) cudaFree(p->k3_ws);
  for (int b = 0; b < 3; ++b)
    if (p->k3_tiles[b]) cudaFree(p->k3_tiles[b]);
  if (p->hl_data) cudaFree(p->hl_data);
  if (p->hl_rowptr) cudaFree(p->hl_rowptr);
  for (int b = 0; b < 2; ++b)
    if (p->k3d_tiles[b]) cudaFree(p->k3d_tiles[b]);
  if (p->k3d_idx1) cudaFree(p->k3d_idx1);
  if (p->dl_data) cudaFree(p->dl_data);
  if (p->dl_uoff) cudaFree(p->dl_uoff);
  if (p->dl_rowlo) cudaFree(p->dl_rowlo);
  if (p->host_pinned) cudaFreeHost(p->host_pinned);
  if (p->shard_stage) cudaFree(p->shard_stage);
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

static bool layout_enabled(const char* env, bool dflt) {
  const char* v = getenv(env);
  if (!v || !*v) return dflt;
  return *v != '0';
}

// Which kernel serves a fast-mode apply. Single right-hand side over long
// rows: codes of <= 3 bytes take the DL layout (second-order row residuals,
// default; INVOP_DL=0 disables), 3-byte codes the HL layout when DL is
// declined (INVOP_HL=0 disables); everything else streams the byte planes
// (k2_stream / k2_fast). Two or more right-hand sides of <= 3-byte codes go
// to the tensor-core kernels (K3; INVOP_NO_TC=1 disables; tiny operators with
// fewer than eight right-hand sides stay on k2_fast).
enum { ROUTE_PLANES = 0, ROUTE_K3, ROUTE_DL, ROUTE_HL };

static int fast_route(const invop_plan* p, int64_t nrhs) {
  if (!layout_enabled("INVOP_NO_TC", false) && batched_supported(p, nrhs)) return ROUTE_K3;
  if (nrhs != 1 || p->ld / 512 < 16) return ROUTE_PLANES;
  if (p->P <= 3 && p->dl_ready >= 0 && layout_enabled("INVOP_DL", true)) return ROUTE_DL;
  if (p->P == 3 && p->ld <= 16384 && p->hl_ready >= 0 && layout_enabled("INVOP_HL", true))
    return ROUTE_HL;
  return ROUTE_PLANES;
}

extern "C" const char* invop_apply_kernel(const invop_plan* p, int64_t nrhs, int mode) {
  if (!p) return "";
  if (mode == INVOP_MODE_ORDERED) return "k2_ordered";
  switch (fast_route(p, nrhs)) {
    case ROUTE_K3: return k3_uses_pair(p) ? "k3_dl2" : (k3_uses_dl(p) ? "k3_batched_dl" : "k3_batched");
    case ROUTE_DL: return "k2_dl";
    case ROUTE_HL: return "k2_hl";
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
    // any 8-byte aligned x / leading dimension: x tiles that cannot be bulk
    // copied are copied by the producer warp's lanes (ordered.cu)
    if ((uintptr_t)x % 8 != 0) return fail(INVOP_E_VALUE, "x must be 8-byte aligned (fp64)");
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
    if (route == ROUTE_DL || route == ROUTE_HL) {
      int rc = route == ROUTE_DL ? dl_build(mp, s) : hl_build(mp, s);
      if (rc == INVOP_OK)
        rc = route == ROUTE_DL ? apply_dl_launch(mp, x, y, false, s)
                               : apply_hl_launch(mp, (const float*)x, (float*)y, s);
      if (rc != INVOP_E_UNSUPPORTED) return rc;
      // layout not applicable to this plan: the next route
      if (route == ROUTE_HL) mp->hl_ready = -1;
      if (route == ROUTE_DL) mp->dl_ready = -1;
      return invop_apply(p, x, ldx, y, ldy, nrhs, dtype, mode, stream);
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
    if (route == ROUTE_K3) {
      const int rc = k3_prepare(p, s);
      if (rc) return rc;
      *bytes = k3_uses_dl(p) ? k3d_bytes(p) : (int64_t)p->P * p->rows * p->ld;
      return INVOP_OK;
    }
    if (route == ROUTE_DL || route == ROUTE_HL) {
      const int rc = route == ROUTE_DL ? dl_build(p, s) : hl_build(p, s);
      if (rc == INVOP_E_UNSUPPORTED) {
        if (route == ROUTE_HL) p->hl_ready = -1;
        if (route == ROUTE_DL) p->dl_ready = -1;
        return invop_plan_apply_bytes(p, nrhs, mode, bytes, stream);   // next route
      }
      if (rc) return rc;
      *bytes = route == ROUTE_DL ? p->dl_bytes + (p->rows * p->dl_nslabs + 1) * 8
                                 : p->hl_bytes + (p->rows + 1) * 8;
      return INVOP_OK;
    }
  }
  *bytes = (int64_t)p->P * p->rows * p->ld;
  return INVOP_OK;
}

extern "C" int invop_plan_tensor_ops(invop_plan* p, int64_t nrhs, int mode, int64_t* ops,
                                     void* stream) {
  if (!p || !ops) return fail(INVOP_E_VALUE, "NULL argument");
  *ops = 0;
  if (mode != INVOP_MODE_FAST || fast_route(p, nrhs) != ROUTE_K3) return INVOP_OK;
  const int rc = k3_prepare(p, (cudaStream_t)stream);
  if (rc) return rc;
  *ops = k3_tensor_ops(p, nrhs);
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
  {
    // pageable host buffers (numpy arrays of a reference-style caller): stage
    // them through plan-owned page-locked memory so that the zero-copy paths
    // below apply (x copied in, y written by the kernel and copied out);
    // INVOP_HOST_STAGING=0 keeps the driver's pageable copies
    static const bool staging = !(getenv("INVOP_HOST_STAGING") && *getenv("INVOP_HOST_STAGING") == '0');
    void* tmp = nullptr;
    if (staging && x && y && xb + yb <= ((size_t)64 << 20) && !host_alias(y, &tmp) &&
        !host_alias(x, &tmp)) {
      const size_t need = ((xb + 255) & ~(size_t)255) + yb;
      if (p->host_pinned_bytes < need) {
        if (p->host_pinned) cudaFreeHost(p->host_pinned);
        p->host_pinned = nullptr;
        p->host_pinned_bytes = 0;
        if (cudaHostAlloc((void**)&p->host_pinned, need, cudaHostAllocDefault) == cudaSuccess)
          p->host_pinned_bytes = need;
        else
          cudaGetLastError();
      }
      if (p->host_pinned_bytes >= need) {
        double* px = p->host_pinned;
        double* py = (double*)((char*)p->host_pinned + ((xb + 255) & ~(size_t)255));
        memcpy(px, x, xb);
        const int rc = invop_apply_host(p, px, py, nrhs, mode, stream);
        if (rc == INVOP_OK) memcpy(y, py, yb);
        return rc;
      }
    }
  }
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
    // x pulled by a kernel (the apply below is launched as its programmatic
    // dependent, like every k2_dl launch) or copied by the copy engine
    if (host_alias(x, &xdev)) {
      k_pull_x<<<(unsigned)std::min<int64_t>(cdiv(p->n, 512), 64), 256, 0, s>>>(
          (const double*)xdev, (double*)p->dev_x, p->n);
      INVOP_LAUNCHED(1);
    } else {
      INVOP_CUDA(cudaMemcpyAsync(p->dev_x, x, xb, cudaMemcpyHostToDevice, s));
    }
    rc = apply_dl_launch(p, p->dev_x, ydev, true, s);
    if (rc == INVOP_OK) {
      INVOP_CUDA(cudaStreamSynchronize(s));
      return INVOP_OK;
    }
    cudaGetLastError();
  }
  if (mode == INVOP_MODE_ORDERED && p->n > 0 && host_alias(y, &ydev)) {
    // page-locked y: the ordered kernel stores each row's fp64 sum straight
    // into host memory (one 8-byte store per row; no device-to-host copy). x
    // is staged in device memory (every block reads all of it).
    int rc = ensure_scratch(&p->dev_x, &p->dev_x_bytes, xb + 64);
    if (rc) return rc;
    INVOP_CUDA(cudaMemcpyAsync(p->dev_x, x, xb, cudaMemcpyHostToDevice, s));
    rc = apply_ordered_launch(p, (const double*)p->dev_x, p->n, (double*)ydev, p->rows, nrhs, s);
    if (rc) return rc;
    INVOP_CUDA(cudaStreamSynchronize(s));
    return INVOP_OK;
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

// reference-seam entry (_kernels.plan_apply accumulates into the caller's
// `out`, _native.pyx:43-46): ordered fp64, each row's chain starts at y[row]
extern "C" int invop_apply_host_acc(invop_plan* p, const double* x, double* y, int64_t nrhs,
                                    void* stream) {
  if (!p) return fail(INVOP_E_VALUE, "plan is NULL");
  if (nrhs <= 0 || p->rows == 0) return INVOP_OK;
  if (!x || !y) return fail(INVOP_E_VALUE, "NULL vector");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t xb = (size_t)nrhs * p->n * sizeof(double);
  const size_t yb = (size_t)nrhs * p->rows * sizeof(double);
  int rc = ensure_scratch(&p->dev_x, &p->dev_x_bytes, xb + 64);
  if (rc) return rc;
  rc = ensure_scratch(&p->dev_y, &p->dev_y_bytes, yb + 64);
  if (rc) return rc;
  double* dx = (double*)p->dev_x;
  double* dy = (double*)p->dev_y;
  INVOP_CUDA(cudaMemcpyAsync(dx, x, xb, cudaMemcpyHostToDevice, s));
  INVOP_CUDA(cudaMemcpyAsync(dy, y, yb, cudaMemcpyHostToDevice, s));
  if (p->n > 0) {
    rc = apply_ordered_launch(p, dx, p->n, dy, p->rows, nrhs, s, /*accumulate=*/true);
    if (rc) return rc;
  }
  INVOP_CUDA(cudaMemcpyAsync(y, dy, yb, cudaMemcpyDeviceToHost, s));
  INVOP_CUDA(cudaStreamSynchronize(s));
  return INVOP_OK;
}

// host-table variant of invop_plan_from_csc (the reference-side binding
// holds numpy arrays, applyplan.py:42-98): upload, build, free
extern "C" int invop_plan_from_csc_host(int64_t n, int scale_digits, const int64_t* col_ptr,
                                        const int64_t* group_abs_mantissa, const int64_t* group_ptr,
                                        const int32_t* entry_rows, const int8_t* entry_signs,
                                        int64_t groups, int64_t entries, void* stream,
                                        invop_plan** out) {
  if (!out) return fail(INVOP_E_VALUE, "out is NULL");
  *out = nullptr;
  if (n < 0 || groups < 0 || entries < 0) return fail(INVOP_E_VALUE, "bad table sizes");
  if (!col_ptr || !group_ptr || (groups > 0 && !group_abs_mantissa) ||
      (entries > 0 && (!entry_rows || !entry_signs)))
    return fail(INVOP_E_VALUE, "NULL table");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t b_col = (size_t)(n + 1) * 8, b_gabs = (size_t)groups * 8,
               b_gptr = (size_t)(groups + 1) * 8, b_rows = (size_t)entries * 4,
               b_sign = (size_t)entries;
  const size_t o_gabs = round_up(b_col, 256), o_gptr = o_gabs + round_up(b_gabs, 256),
               o_rows = o_gptr + round_up(b_gptr, 256), o_sign = o_rows + round_up(b_rows, 256),
               total = o_sign + round_up(b_sign, 256) + 256;
  char* d = nullptr;
  INVOP_CUDA(cudaMalloc(&d, total));
  int rc = INVOP_OK;
  cudaError_t e = cudaMemcpyAsync(d, col_ptr, b_col, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && b_gabs) e = cudaMemcpyAsync(d + o_gabs, group_abs_mantissa, b_gabs, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d + o_gptr, group_ptr, b_gptr, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && b_rows) e = cudaMemcpyAsync(d + o_rows, entry_rows, b_rows, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && b_sign) e = cudaMemcpyAsync(d + o_sign, entry_signs, b_sign, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) rc = cuda_fail(e, "plan_from_csc_host upload");
  if (!rc)
    rc = invop_plan_from_csc(n, scale_digits, (const int64_t*)d, (const int64_t*)(d + o_gabs),
                             (const int64_t*)(d + o_gptr), (const int32_t*)(d + o_rows),
                             (const int8_t*)(d + o_sign), groups, entries, stream, out);
  cudaStreamSynchronize(s);
  cudaFree(d);
  return rc;
}

// host-buffer variant of invop_dense_matvec (the reference seam's
// dense_matvec(mat, x, out), _native.pyx:75-92): synchronous
extern "C" int invop_dense_matvec_host(const double* m, int64_t rows, int64_t cols, int64_t ld,
                                       const double* x, double* y, void* stream) {
  if (rows < 0 || cols < 0 || ld < cols) return fail(INVOP_E_VALUE, "bad geometry");
  if (rows == 0) return INVOP_OK;
  if (!m || !x || !y) return fail(INVOP_E_VALUE, "NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bm = (size_t)rows * ld * 8, bx = (size_t)cols * 8, by = (size_t)rows * 8;
  char* d = nullptr;
  INVOP_CUDA(cudaMalloc(&d, round_up(bm, 256) + round_up(bx, 256) + by + 256));
  double* dm = (double*)d;
  double* dx = (double*)(d + round_up(bm, 256));
  double* dy = (double*)(d + round_up(bm, 256) + round_up(bx, 256));
  int rc = INVOP_OK;
  cudaError_t e = cudaMemcpyAsync(dm, m, bm, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && bx) e = cudaMemcpyAsync(dx, x, bx, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) rc = cuda_fail(e, "dense_matvec_host upload");
  if (!rc) rc = invop_dense_matvec(dm, rows, cols, ld, dx, dy, stream);
  if (!rc) {
    e = cudaMemcpyAsync(y, dy, by, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) rc = cuda_fail(e, "dense_matvec_host download");
  }
  cudaStreamSynchronize(s);
  cudaFree(d);
  return rc;
}

extern "C" int invop_apply_naive(const invop_plan* p, const double* x, double* y, int64_t nrhs,
                                 void* stream) {
  // apply_naive_quantized (applyplan.py:194-209) accumulates mant*scale*x_j per
  // nonzero in ascending column order: the arithmetic of ORDERED mode.
  if (!p) return fail(INVOP_E_VALUE, "plan is NULL");
  return invop_apply(p, x, p->n, y, p->rows, nrhs, INVOP_F64, INVOP_MODE_ORDERED, stream);
}
