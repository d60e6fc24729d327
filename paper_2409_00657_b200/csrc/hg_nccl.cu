// NCCL collectives of the micrograph step, issued from C on the caller's
// stream (no Python in the per-iteration path):
//   * hg_allreduce_sgd: gradient all-reduce (model.py:299-324 sync_and_update:
//     g = sum(acc)/batch_total; theta -= lr * g) fused with the SGD kernel;
//   * hg_shift: the model hop ring shift of (params, accumulator) by delta
//     servers (engine.py:610-618), one grouped send/recv.
// The communicator is created from a unique id the host broadcasts once.
#include <cstring>

#include "hg_common.cuh"

#ifdef HG_HAVE_NCCL
#include <nccl.h>

#define HG_NCCL_TRY(expr)                                                        \
  do {                                                                           \
    ncclResult_t _r = (expr);                                                    \
    if (_r != ncclSuccess) return hg_fail(HG_ENCCL, "NCCL %s: %s", #expr, ncclGetErrorString(_r)); \
  } while (0)

extern "C" int hg_sgd_update(float* params, float* grads, void* shadow_bf16, int64_t n, float lr,
                             float inv_batch, void* stream);

extern "C" int hg_nccl_unique_id(void* out /* 128 bytes */) {
  ncclUniqueId id;
  HG_NCCL_TRY(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return HG_OK;
}

extern "C" int hg_nccl_init(const void* id_bytes, int nranks, int rank, void** comm_out) {
  ncclUniqueId id;
  memcpy(&id, id_bytes, sizeof(id));
  ncclComm_t comm;
  HG_NCCL_TRY(ncclCommInitRank(&comm, nranks, id, rank));
  *comm_out = comm;
  return HG_OK;
}

extern "C" int hg_nccl_destroy(void* comm) {
  if (comm) HG_NCCL_TRY(ncclCommDestroy((ncclComm_t)comm));
  return HG_OK;
}

extern "C" int hg_allreduce_sgd(void* comm, float* params, float* grads, int64_t n, float lr,
                                float inv_batch, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (comm) HG_NCCL_TRY(ncclAllReduce(grads, grads, (size_t)n, ncclFloat32, ncclSum,
                                      (ncclComm_t)comm, s));
  return hg_sgd_update(params, grads, nullptr, n, lr, inv_batch, stream);
}

extern "C" int hg_sgd_refresh(const hg_step_desc* d, float* params, float* grads, int64_t n,
                              float lr, float inv_batch, int32_t update, void* stream);

extern "C" int hg_allreduce_sgd_refresh(void* comm, const hg_step_desc* d, float* params,
                                        float* grads, int64_t n, float lr, float inv_batch,
                                        void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (comm) HG_NCCL_TRY(ncclAllReduce(grads, grads, (size_t)n, ncclFloat32, ncclSum,
                                      (ncclComm_t)comm, s));
  return hg_sgd_refresh(d, params, grads, n, lr, inv_batch, 1, stream);
}

extern "C" int hg_shift(void* comm, int rank, int nranks, int delta, const float* send0,
                        const float* send1, float* recv0, float* recv1, int64_t n, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int to = (rank + delta) % nranks, from = ((rank - delta) % nranks + nranks) % nranks;
  HG_NCCL_TRY(ncclGroupStart());
  HG_NCCL_TRY(ncclSend(send0, (size_t)n, ncclFloat32, to, (ncclComm_t)comm, s));
  HG_NCCL_TRY(ncclSend(send1, (size_t)n, ncclFloat32, to, (ncclComm_t)comm, s));
  HG_NCCL_TRY(ncclRecv(recv0, (size_t)n, ncclFloat32, from, (ncclComm_t)comm, s));
  HG_NCCL_TRY(ncclRecv(recv1, (size_t)n, ncclFloat32, from, (ncclComm_t)comm, s));
  HG_NCCL_TRY(ncclGroupEnd());
  return HG_OK;
}

#else  // built without NCCL headers: the entry points exist and fail loudly

extern "C" int hg_nccl_unique_id(void*) { return hg_fail(HG_ENCCL, "built without NCCL"); }
extern "C" int hg_nccl_init(const void*, int, int, void**) { return hg_fail(HG_ENCCL, "built without NCCL"); }
extern "C" int hg_nccl_destroy(void*) { return HG_OK; }
extern "C" int hg_allreduce_sgd(void*, float*, float*, int64_t, float, float, void*) {
  return hg_fail(HG_ENCCL, "built without NCCL");
}
extern "C" int hg_allreduce_sgd_refresh(void*, const hg_step_desc*, float*, float*, int64_t, float,
                                        float, void*) {
  return hg_fail(HG_ENCCL, "built without NCCL");
}
extern "C" int hg_shift(void*, int, int, int, const float*, const float*, float*, float*, int64_t,
                        void*) {
  return hg_fail(HG_ENCCL, "built without NCCL");
}
#endif
