/*
 * invop_b200.h — C ABI of libinvop_b200.so, the B200 (sm_100a) implementation
 * of the quantized inverse-operator apply of arXiv 1602.00001 (reference
 * package `invop`).
 *
 * The reference binds its hot path through one Python-level seam,
 *   invop._kernels.plan_apply(col_ptr, group_coeff, group_ptr, entry_rows,
 *                             entry_signs, x, out) -> (mults, adds)
 *   (/root/reference/pkg/src/invop/_kernels/_native.pyx:15-49, selected in
 *    /root/reference/pkg/src/invop/_kernels/__init__.py:14-39)
 * which takes HOST CSC group tables. That is the wrong granularity for a device
 * layout (5 B/entry + 16 B/group of pointer-chasing), so this ABI moves the seam
 * up to the plan level: a plan owns the quantized operator in a compressed
 * device layout (narrow integer codes stored as byte planes), and every entry
 * point below replaces one reference function, cited per declaration.
 *
 * Conventions
 *  - Plain C types only: pointers, int64_t sizes, int status codes.
 *  - Every function returns INVOP_OK (0) or a negative-free status code; the
 *    message of the last failure on the calling thread is invop_last_error().
 *  - "device" pointers are CUDA device memory of the current device; "host"
 *    pointers are ordinary (preferably pinned) host memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All device work is stream-ordered and asynchronous unless stated.
 *  - Matrices are row-major; a plan holds rows [row0, row0+rows) of an n x n
 *    operator (a row shard; row0 = 0 and rows = n for the whole operator).
 *  - Vectors for multi-RHS calls are stored RHS-major: X[t*ldx + j] is entry j
 *    of right-hand side t; Y[t*ldy + i] is output row (row0+i) of RHS t.
 */
#ifndef INVOP_B200_H
#define INVOP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct invop_plan invop_plan;
typedef struct invop_operator invop_operator;

/* status codes (mirror the reference error hierarchy,
   /root/reference/pkg/src/invop/errors.py:4-25) */
enum {
  INVOP_OK = 0,
  INVOP_E_VALUE = 1,       /* ValueError: bad shape / argument            */
  INVOP_E_OVERFLOW = 2,    /* MantissaOverflowError (quant.py:58-64)      */
  INVOP_E_CAPACITY = 3,    /* CapacityError (grid.py:149-154)             */
  INVOP_E_SINGULAR = 4,    /* SingularMatrixError (dense.py:54-60)        */
  INVOP_E_CUDA = 5,        /* CUDA runtime failure                         */
  INVOP_E_UNSUPPORTED = 6  /* valid request this build cannot serve      */
};

/* arithmetic of an apply */
enum { INVOP_F32 = 0, INVOP_F64 = 1 };
/* INVOP_MODE_ORDERED: fp64, each output row accumulates (mant*10^-m)*x_j in
   ascending column order, zero mantissas skipped — bitwise equal to the
   reference apply (applyplan.py:4-8, _native.pyx:32-46).
   INVOP_MODE_FAST: fp32 I/O; x is split into 512-column pieces, each turned
   into 23-bit fixed point, sum_j mant_ij*X_j accumulated exactly in integers
   and scaled by 10^-m * 2^-e once per row (fp32 relative error <= 1e-5). */
enum { INVOP_MODE_FAST = 0, INVOP_MODE_ORDERED = 1 };

const char* invop_last_error(void);
int invop_abi_version(void);
/* Kernels launched so far by the apply entry points (invop_apply,
   invop_apply_host) in this process — the benchmark's gpu_launches. */
int64_t invop_launch_count(void);

/* A1 — quantize (reference: invop.quantize, quant.py:48-65).
   entries: device fp64 [rows x cols] (leading dim ld). mant: device int64
   [rows x cols] (leading dim ldm). Rounds half away from zero exactly like
   numpy: copysign(floor(|e*10^d|+0.5), e*10^d). If any |mantissa| > 2^53 the
   call returns INVOP_E_OVERFLOW and *bad_index = i*cols + j of the first
   maximal offender (synchronous on failure check). */
int invop_quantize(const double* entries, int64_t rows, int64_t cols, int64_t ld,
                   int digits, int64_t* mant, int64_t ldm, int64_t* bad_index,
                   void* stream);

/* A4/A5 — build a plan (reference: invop.build_plan, applyplan.py:116-172)
   from device int64 mantissas of rows [row0,row0+rows) of an n x n matrix.
   Chooses the narrowest byte-plane code width that holds every mantissa. */
int invop_plan_create(const int64_t* mant, int64_t rows, int64_t n, int64_t ldm,
                      int64_t row0, int scale_digits, void* stream, invop_plan** out);

/* Fused A1+A4: quantize device fp64 rows and encode them into a plan without
   materialising int64 mantissas. Same overflow contract as invop_quantize. */
int invop_plan_from_f64(const double* entries, int64_t rows, int64_t n, int64_t ld,
                        int64_t row0, int digits, int64_t* bad_index, void* stream,
                        invop_plan** out);

/* Build a plan from the reference's CSC group tables (device arrays; the
   layout of ApplyPlan, applyplan.py:42-98). Used for the drop-in of the
   _kernels.plan_apply seam. */
int invop_plan_from_csc(int64_t n, int scale_digits, const int64_t* col_ptr,
                        const int64_t* group_abs_mantissa, const int64_t* group_ptr,
                        const int32_t* entry_rows, const int8_t* entry_signs,
                        int64_t groups, int64_t entries, void* stream, invop_plan** out);

/* Same, from HOST arrays (what a reference-side binding holds: the numpy
   tables of ApplyPlan); synchronous. */
int invop_plan_from_csc_host(int64_t n, int scale_digits, const int64_t* col_ptr,
                             const int64_t* group_abs_mantissa, const int64_t* group_ptr,
                             const int32_t* entry_rows, const int8_t* entry_signs,
                             int64_t groups, int64_t entries, void* stream, invop_plan** out);

int invop_plan_destroy(invop_plan* plan);

/* plan geometry and storage */
int invop_plan_info(const invop_plan* plan, int64_t* n, int64_t* rows, int64_t* row0,
                    int* scale_digits, int* code_bytes, int* is_signed,
                    int64_t* device_bytes, int64_t* max_abs);

/* A5/A9 — planned counters (reference: ApplyPlan.planned_multiplications /
   planned_additions, applyplan.py:92-98; quant.sparsity_stats :73-82).
   adds = number of nonzero mantissas; mults = sum over columns of the number
   of distinct nonzero |mantissa| in that column (over the plan's rows).
   Computed on device on first request and cached (synchronous). */
int invop_plan_counts(invop_plan* plan, int64_t* mults, int64_t* adds, void* stream);
/* per-column distinct counts (device int64[n]) and nonzeros (device int64[n]) */
int invop_plan_column_stats(invop_plan* plan, int64_t* distinct, int64_t* nonzero,
                            void* stream);

/* f1 — compressed on-disk format (reference IVOP files store int64
   mantissas, cache.py:67-115): copy the byte planes out to host memory
   (P planes of rows*n bytes, plane-major, row-major; synchronous) and build a
   plan back from them. */
int invop_plan_get_planes(const invop_plan* plan, uint8_t* host, void* stream);
int invop_plan_from_planes(const uint8_t* host, int code_bytes, int is_signed, int64_t rows,
                           int64_t n, int64_t row0, int scale_digits, void* stream,
                           invop_plan** out);

/* A2/A3 — expand codes back to int64 mantissas (device [rows x n], ldm). */
int invop_plan_decode(const invop_plan* plan, int64_t* mant, int64_t ldm, void* stream);
/* Selected rows only: rows is a device int64 list of plan-local row indices
   (each in [0, rows)); mant is device [nrows x n] (ldm). */
int invop_plan_decode_rows(const invop_plan* plan, const int64_t* rows, int64_t nrows,
                           int64_t* mant, int64_t ldm, void* stream);

/* A4 — the reference's CSC group tables, built on device from the codes.
   Pass NULL outputs to query sizes: *groups and *entries are returned
   (synchronous). Outputs are device arrays sized n+1, G, G, G+1, E, E. */
int invop_plan_csc(invop_plan* plan, int64_t* col_ptr, int64_t* group_abs_mantissa,
                   double* group_coeff, int64_t* group_ptr, int32_t* entry_rows,
                   int8_t* entry_signs, int64_t* groups, int64_t* entries, void* stream);

/* A6/A7 — apply (reference: invop.apply -> _kernels.plan_apply,
   applyplan.py:175-191, _native.pyx:15-49).
   x: device [nrhs x n] (ldx), y: device [nrhs x rows] (ldy), both of `dtype`.
   mode INVOP_MODE_ORDERED requires dtype INVOP_F64.
   y is overwritten (the reference zero-fills then accumulates, :181).
   The first call on a plan builds its lazily created layouts (row residuals,
   tensor-core tiles) and synchronises; every later call is stream-ordered,
   asynchronous and capturable in a CUDA graph — including the tensor-core
   route with inf/nan in x (the zero-mantissa skip is applied on the device). */
int invop_apply(const invop_plan* plan, const void* x, int64_t ldx, void* y, int64_t ldy,
                int64_t nrhs, int dtype, int mode, void* stream);

/* Same contract with HOST fp64 buffers x [nrhs x n], y [nrhs x rows]
   (contiguous); the host<->device copies are part of the call (synchronous).
   This is the end-to-end entry a reference-side binding calls. */
int invop_apply_host(invop_plan* plan, const double* x, double* y, int64_t nrhs,
                     int mode, void* stream);

/* Reference-seam variant (_kernels.plan_apply accumulates into the caller's
   zero-filled `out`, _native.pyx:43-46): ordered fp64 with HOST buffers, y
   read as each row's initial accumulator and overwritten with the result;
   zero mantissas are skipped exactly as the reference skips them
   (synchronous). */
int invop_apply_host_acc(invop_plan* plan, const double* x, double* y, int64_t nrhs,
                         void* stream);

/* Bytes of operator data one apply of `nrhs` right-hand sides in `mode`
   streams from HBM (codes + per-chunk metadata), i.e. the algorithmic bytes
   of the roofline; builds the lazily created layouts first (synchronous). */
int invop_plan_apply_bytes(invop_plan* plan, int64_t nrhs, int mode, int64_t* bytes,
                           void* stream);

/* int8 tensor-core operations (2*M*N*K summed over the tcgen05 MMAs) one
   apply of `nrhs` right-hand sides in `mode` issues; 0 for applies that do not
   run on the tensor cores. Builds the lazily created layouts first
   (synchronous). */
int invop_plan_tensor_ops(invop_plan* plan, int64_t nrhs, int mode, int64_t* ops, void* stream);

/* Name of the kernel an apply of `nrhs` right-hand sides in `mode` launches
   ("k2_dl", "k2_hl", "k2_stream", "k2_fast", "k3_dl2", "k3_batched_dl",
   "k3_batched", "k2_ordered"), for
   benchmark labels; static string, "" for a NULL plan. */
const char* invop_apply_kernel(const invop_plan* plan, int64_t nrhs, int mode);

/* The reference's grouped apply as written (_native.pyx:15-49) on device CSC
   tables (invop_plan_csc): one multiplication per (column, distinct value),
   an fp64 atomic add per entry into y (zeroed first; add order differs from
   the reference, so NOT bitwise). A design comparison, not an apply route:
   it streams 16 B per group + 5 B per entry. All pointers are device memory. */
int invop_apply_grouped_csc(int64_t n, const int64_t* col_ptr, const double* group_coeff,
                            const int64_t* group_ptr, const int32_t* entry_rows,
                            const int8_t* entry_signs, const double* x, double* y, void* stream);

/* Row-sharded multi-GPU apply (new — the reference is one
   process). Each rank holds the plan of its rows [row_offsets[rank],
   row_offsets[rank+1]) of the operator; x: device [nrhs x n] (ldx), the full
   right-hand sides on every rank; y: device [nrhs x n] (ldy >= n) receives
   every rank's rows. The local rows are applied into this rank's slice of a
   staging buffer [nranks][nrhs][pad] (pad = largest shard, owned by the
   plan), ONE ncclAllGather over `nccl_comm` (an ncclComm_t of the ranks, in
   rank order) fills every slice, and one kernel (invop_unshard) scatters them
   into y. row_offsets: host int64 [nranks + 1], nranks <= 64. Stream-ordered
   on `stream`; NCCL is resolved from the process at run time
   (INVOP_E_UNSUPPORTED when it is not loaded). */
int invop_apply_sharded(invop_plan* shard, void* nccl_comm, const int64_t* row_offsets,
                        const void* x, int64_t ldx, void* y, int64_t ldy, int64_t nrhs,
                        int dtype, int mode, void* stream);

/* The reassembly step of the sharded apply on its own, for callers that run
   the all-gather themselves (torch.distributed): stage is device
   [world][nrhs][pad] (slice r holds rows row_offsets[r].. of every RHS, ld
   pad), y is device [nrhs x n] (ldy >= n = row_offsets[world]); one launch. */
int invop_unshard(const void* stage, int world, const int64_t* row_offsets, int64_t nrhs,
                  int64_t pad, void* y, int64_t ldy, int dtype, void* stream);

/* A8 — naive quantized apply of the reference (applyplan.py:194-209):
   identical arithmetic to ORDERED mode; provided under its own name. */
int invop_apply_naive(const invop_plan* plan, const double* x, double* y, int64_t nrhs,
                      void* stream);

/* A10/A11 — device construction of rows of L^-1 (setup; reference builds the
   operator with grid.build_uniform/build_variable, grid.py:157-186, and
   inverts it densely with dense.invert, dense.py:36-62).
   The operator is a 5-point stencil on an nx x ny interior grid, unknown
   p = r*nx + c (r slow): row p has diag[p] on the diagonal and -w_west[p],
   -w_east[p], -w_south[p], -w_north[p] towards (r,c-1),(r,c+1),(r-1,c),(r+1,c);
   couplings to outside the grid must be 0. Arrays are host fp64 [nx*ny]. */
int invop_operator_create(int64_t nx, int64_t ny, const double* diag, const double* w_west,
                          const double* w_east, const double* w_south,
                          const double* w_north, void* stream, invop_operator** out);
/* block-LU factorisation (sequential over grid lines, fp64, on device).
   Returns INVOP_E_SINGULAR if a pivot falls below 1e-13*max|entry|. */
int invop_operator_factor(invop_operator* op, void* stream);
int invop_operator_destroy(invop_operator* op);
/* rows [row0,row0+rows) of L^-1 by batched multi-RHS block solves, quantized
   to `digits` and encoded straight into a plan (fp64 L^-1 never stored). */
int invop_construct_rows(invop_operator* op, int64_t row0, int64_t rows, int digits,
                         void* stream, invop_plan** out);
/* rows [row0,row0+rows) of L^-1 in fp64 into device memory out[rows x N] (ld). */
int invop_construct_rows_f64(invop_operator* op, int64_t row0, int64_t rows, double* out,
                             int64_t ld, void* stream);

/* A10 (generic) — inverse of an arbitrary dense fp64 matrix (device a[n x n]
   -> device out[n x n]) by Gauss-Jordan with partial pivoting; returns
   INVOP_E_SINGULAR if a pivot falls below `tol` (reference: dense.invert,
   dense.py:36-62, tol = 1e-13*max|a|). Synchronous. */
int invop_dense_invert(const double* a, int64_t n, double* out, double tol, void* stream);

/* next (f2) — conventional dense multiply of the reference (_native.pyx:75-92,
   dense.apply_dense dense.py:74-82): y_r = m[r,0]*x[0] + m[r,1]*x[1] + ...
   accumulated left to right in fp64 without FMA (bitwise equal). Device
   pointers, m is [rows x cols] with leading dimension ld. */
int invop_dense_matvec(const double* m, int64_t rows, int64_t cols, int64_t ld,
                       const double* x, double* y, void* stream);
/* Same with HOST buffers (the reference seam's dense_matvec(mat, x, out));
   synchronous. */
int invop_dense_matvec_host(const double* m, int64_t rows, int64_t cols, int64_t ld,
                            const double* x, double* y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* INVOP_B200_H */
