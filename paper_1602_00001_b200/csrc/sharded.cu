// Row-sharded multi-GPU apply: each rank owns rows
// [row0, row0 + rows) of the operator (its own plan, built from its own K4
// construction), applies them to the full x, and the row slices are exchanged
// so that every rank ends with the whole y. The reference has no
// multi-process path; this is the data path `sharded.py` drives
// through torch.distributed and `invop_apply_sharded` drives through a
// caller-owned NCCL communicator.
//
// Exchange: every rank's slice is padded to pad = max shard rows and laid out
// [rank][rhs][pad] in a staging buffer, so ONE all-gather moves every slice
// of every right-hand side (uneven N included); k_unshard then scatters the
// staging buffer into y[rhs][n] (one launch).
//
// NCCL is resolved at run time from the process (torch loads its own copy;
// linking a second one would mix two NCCL builds in one process).
#include "common.cuh"
#include <dlfcn.h>
#include <algorithm>

namespace invop {

typedef int (*PFN_ncclAllGather)(const void*, void*, size_t, int /*ncclDataType_t*/, void* comm,
                                 cudaStream_t);
typedef int (*PFN_ncclCommCount)(void* comm, int* count);
typedef int (*PFN_ncclCommUserRank)(void* comm, int* rank);

struct NcclFns {
  PFN_ncclAllGather allgather = nullptr;
  PFN_ncclCommCount count = nullptr;
  PFN_ncclCommUserRank rank = nullptr;
};

static const NcclFns* nccl() {
  static NcclFns f;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // 1. the instance loaded under the NCCL soname (torch's), 2. a global
    // definition already in the process (NCCL linked statically into the
    // caller: RTLD_DEFAULT is a null handle on glibc, so resolve through it
    // explicitly), 3. load one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    bool global = false;
    if (!h && dlsym(RTLD_DEFAULT, "ncclAllGather")) global = true;
    if (!h && !global) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h && !global) return nullptr;
    void* src = global ? RTLD_DEFAULT : h;
    f.allgather = (PFN_ncclAllGather)dlsym(src, "ncclAllGather");
    f.count = (PFN_ncclCommCount)dlsym(src, "ncclCommCount");
    f.rank = (PFN_ncclCommUserRank)dlsym(src, "ncclCommUserRank");
  }
  return (f.allgather && f.count && f.rank) ? &f : nullptr;
}

// staging [world][nrhs][pad] -> y[t * ldy + row_offsets[r] + i]; row_offsets
// in constant-size device-side argument (<= 64 ranks)
constexpr int UNSHARD_MAX_RANKS = 64;
struct UnshardArgs {
  int64_t off[UNSHARD_MAX_RANKS + 1];
  int world;
  int64_t nrhs, pad, ldy;
};

template <typename T>
__global__ void k_unshard(const T* __restrict__ stage, T* __restrict__ y, UnshardArgs a) {
  const int64_t n = a.off[a.world];
  const int64_t total = a.nrhs * n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = k / n, row = k - t * n;
    int r = 0;
    while (row >= a.off[r + 1]) ++r;     // <= 64 ranks: a short scan
    y[t * a.ldy + row] = stage[((int64_t)r * a.nrhs + t) * a.pad + (row - a.off[r])];
  }
}

static int unshard_launch(const void* stage, int world, const int64_t* row_offsets, int64_t nrhs,
                          int64_t pad, void* y, int64_t ldy, int dtype, cudaStream_t s) {
  if (world < 1 || world > UNSHARD_MAX_RANKS) return fail(INVOP_E_VALUE, "1 <= world <= 64");
  UnshardArgs a;
  for (int r = 0; r <= world; ++r) a.off[r] = row_offsets[r];
  for (int r = 0; r < world; ++r)
    if (a.off[r + 1] < a.off[r] || a.off[r + 1] - a.off[r] > pad)
      return fail(INVOP_E_VALUE, "row_offsets must ascend with shards of at most pad rows");
  a.world = world;
  a.nrhs = nrhs;
  a.pad = pad;
  a.ldy = ldy;
  if (ldy < a.off[world]) return fail(INVOP_E_VALUE, "ldy < n");
  const int64_t total = nrhs * a.off[world];
  if (total == 0) return INVOP_OK;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), (int64_t)num_sms() * 8);
  if (dtype == INVOP_F64)
    k_unshard<double><<<grid, 256, 0, s>>>((const double*)stage, (double*)y, a);
  else
    k_unshard<float><<<grid, 256, 0, s>>>((const float*)stage, (float*)y, a);
  INVOP_LAUNCHED(1);
  INVOP_CHECK_LAUNCH("k_unshard");
  return INVOP_OK;
}

}  // namespace invop

using namespace invop;

extern "C" int invop_unshard(const void* stage, int world, const int64_t* row_offsets,
                             int64_t nrhs, int64_t pad, void* y, int64_t ldy, int dtype,
                             void* stream) {
  if (!stage || !row_offsets || !y) return fail(INVOP_E_VALUE, "NULL argument");
  if (nrhs <= 0) return INVOP_OK;
  return unshard_launch(stage, world, row_offsets, nrhs, pad, y, ldy, dtype, (cudaStream_t)stream);
}

extern "C" int invop_apply_sharded(invop_plan* shard, void* nccl_comm, const int64_t* row_offsets,
                                   const void* x, int64_t ldx, void* y, int64_t ldy, int64_t nrhs,
                                   int dtype, int mode, void* stream) {
  if (!shard || !nccl_comm || !row_offsets) return fail(INVOP_E_VALUE, "NULL argument");
  if (nrhs <= 0) return INVOP_OK;
  const NcclFns* f = nccl();
  if (!f) return fail(INVOP_E_UNSUPPORTED, "NCCL is not loaded in this process");
  int nranks = 0, me = 0;
  if (f->count(nccl_comm, &nranks) != 0 || f->rank(nccl_comm, &me) != 0)
    return fail(INVOP_E_VALUE, "invalid NCCL communicator");
  if (nranks > UNSHARD_MAX_RANKS) return fail(INVOP_E_VALUE, "at most 64 ranks");
  if (row_offsets[me] != shard->row0 || row_offsets[me + 1] - row_offsets[me] != shard->rows ||
      row_offsets[0] != 0 || row_offsets[nranks] != shard->n)
    return fail(INVOP_E_VALUE, "row_offsets do not match this rank's shard");
  if (ldy < shard->n) return fail(INVOP_E_VALUE, "ldy < n: y must hold every row");
  int64_t pad = 0;
  for (int r = 0; r < nranks; ++r) pad = std::max<int64_t>(pad, row_offsets[r + 1] - row_offsets[r]);
  const size_t es = dtype == INVOP_F64 ? 8 : 4;
  cudaStream_t s = (cudaStream_t)stream;
  // staging [nranks][nrhs][pad], owned by the plan
  const size_t slice = (size_t)nrhs * pad * es;
  int rc = ensure_scratch(&shard->shard_stage, &shard->shard_stage_bytes, slice * nranks);
  if (rc) return rc;
  char* stage = static_cast<char*>(shard->shard_stage);
  // this rank's rows straight into its slice of the staging buffer (ldy = pad)
  rc = invop_apply(shard, x, ldx, stage + slice * me, pad, nrhs, dtype, mode, stream);
  if (rc) return rc;
  // one in-place all-gather of every slice (ncclFloat32 = 7, ncclFloat64 = 8)
  if (f->allgather(stage + slice * me, stage, slice / es, dtype == INVOP_F64 ? 8 : 7, nccl_comm, s) != 0)
    return fail(INVOP_E_CUDA, "ncclAllGather failed");
  return unshard_launch(stage, nranks, row_offsets, nrhs, pad, y, ldy, dtype, s);
}
