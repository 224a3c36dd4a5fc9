// invop_apply_sharded — the row-sharded multi-GPU apply:
// each rank owns rows [row0, row0 + rows) of the operator (its own plan,
// built from its own K4 construction), applies them to the full x, and the
// slices are exchanged so that every rank ends with the whole y. The exchange
// is one NCCL group of in-place broadcasts, one per (rank, right-hand side):
// it handles uneven shards and writes straight into y (no staging, no
// transpose). The reference has no multi-process path; this is
// the data path `sharded.py` drives through torch.distributed.
//
// NCCL is resolved at run time from the process (torch loads its own copy;
// linking a second one would mix two NCCL builds in one process).
#include "common.cuh"
#include <dlfcn.h>

namespace invop {

typedef int (*PFN_ncclBroadcast)(const void*, void*, size_t, int /*ncclDataType_t*/, int root,
                                 void* comm, cudaStream_t);
typedef int (*PFN_ncclGroup)();
typedef int (*PFN_ncclCommCount)(void* comm, int* count);
typedef int (*PFN_ncclCommUserRank)(void* comm, int* rank);

struct NcclFns {
  PFN_ncclBroadcast bcast = nullptr;
  PFN_ncclGroup start = nullptr, end = nullptr;
  PFN_ncclCommCount count = nullptr;
  PFN_ncclCommUserRank rank = nullptr;
};

static const NcclFns* nccl() {
  static NcclFns f;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // the instance already loaded under the NCCL soname (torch's), else any
    // global definition, else load one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && dlsym(RTLD_DEFAULT, "ncclBroadcast")) h = RTLD_DEFAULT;
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return nullptr;
    f.bcast = (PFN_ncclBroadcast)dlsym(h, "ncclBroadcast");
    f.start = (PFN_ncclGroup)dlsym(h, "ncclGroupStart");
    f.end = (PFN_ncclGroup)dlsym(h, "ncclGroupEnd");
    f.count = (PFN_ncclCommCount)dlsym(h, "ncclCommCount");
    f.rank = (PFN_ncclCommUserRank)dlsym(h, "ncclCommUserRank");
  }
  return (f.bcast && f.start && f.end && f.count && f.rank) ? &f : nullptr;
}

}  // namespace invop

using namespace invop;

extern "C" int invop_apply_sharded(const invop_plan* shard, void* nccl_comm, const int64_t* row_offsets,
                                   const void* x, int64_t ldx, void* y, int64_t ldy, int64_t nrhs,
                                   int dtype, int mode, void* stream) {
  if (!shard || !nccl_comm || !row_offsets) return fail(INVOP_E_VALUE, "NULL argument");
  if (nrhs <= 0) return INVOP_OK;
  const NcclFns* f = nccl();
  if (!f) return fail(INVOP_E_UNSUPPORTED, "NCCL is not loaded in this process");
  int nranks = 0, me = 0;
  if (f->count(nccl_comm, &nranks) != 0 || f->rank(nccl_comm, &me) != 0)
    return fail(INVOP_E_VALUE, "invalid NCCL communicator");
  if (row_offsets[me] != shard->row0 || row_offsets[me + 1] - row_offsets[me] != shard->rows ||
      row_offsets[0] != 0 || row_offsets[nranks] != shard->n)
    return fail(INVOP_E_VALUE, "row_offsets do not match this rank's shard");
  if (ldy < shard->n) return fail(INVOP_E_VALUE, "ldy < n: y must hold every row");
  const size_t es = dtype == INVOP_F64 ? 8 : 4;
  char* yb = static_cast<char*>(y);
  // this rank's rows, in place in the full y
  int rc = invop_apply(shard, x, ldx, yb + (size_t)shard->row0 * es, ldy, nrhs, dtype, mode, stream);
  if (rc) return rc;
  // every rank's slice to every rank (in-place broadcasts; ncclFloat32 = 7,
  // ncclFloat64 = 8)
  const int dt = dtype == INVOP_F64 ? 8 : 7;
  cudaStream_t s = (cudaStream_t)stream;
  if (f->start() != 0) return fail(INVOP_E_CUDA, "ncclGroupStart failed");
  int nrc = 0;
  for (int r = 0; r < nranks && !nrc; ++r) {
    const int64_t off = row_offsets[r], cnt = row_offsets[r + 1] - off;
    if (cnt <= 0) continue;
    for (int64_t t = 0; t < nrhs && !nrc; ++t) {
      char* p = yb + ((size_t)t * ldy + off) * es;
      nrc = f->bcast(p, p, (size_t)cnt, dt, r, nccl_comm, s);
    }
  }
  const int erc = f->end();
  if (nrc != 0 || erc != 0) return fail(INVOP_E_CUDA, "NCCL broadcast failed");
  return INVOP_OK;
}
