// NCCL communicators of the plan executor, owned by the C side and driven on
// the caller's CUDA stream (so they can sit inside CUDA-graph captures and carry
// no per-call Python overhead).  Replaces the modeled `collective_time` /
// `transfer_time` of the reference (costs.py:63-92) for:
//   all_reduce   k-split matmul partial sums (sharding.py:284-291), split-softmax
//                row statistics, gradient reduction (intra.py:404-424)
//   all_gather   local all-gather of a cross-mesh replica group (reshard.py:155)
//                and dim-0 relayouts
//   send / recv  cross-mesh Transfers (reshard.py:32-37) and box relayouts
#include <cuda_runtime.h>
#include <nccl.h>
#include <string>
#include "common.cuh"
#include "../../include/mp_exec.h"

namespace mp {

static ncclDataType_t nccl_dtype(int d) {
  switch (d) {
    case 0: return ncclBfloat16;
    case 1: return ncclFloat32;
    default: return ncclUint8;
  }
}

#define MP_NCCL(call)                                                                  \
  do {                                                                                 \
    ncclResult_t r__ = (call);                                                         \
    if (r__ != ncclSuccess) {                                                          \
      ::mp::set_error(std::string(__func__) + ": " + ncclGetErrorString(r__) + " (" +  \
                      ncclGetLastError(nullptr) + ")");                                \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

}  // namespace mp

using namespace mp;

extern "C" {

int mp_nccl_version(void) {
  int v = 0;
  ncclGetVersion(&v);
  return v;
}

int mp_nccl_unique_id(void* out128) {
  clear_error();
  MP_CHECK_ARG(out128, "null output");
  ncclUniqueId id;
  MP_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
  memcpy(out128, &id, sizeof(id));
  return 0;
}

int mp_comm_init(const void* uid128, int nranks, int rank, void** comm_out) {
  clear_error();
  MP_CHECK_ARG(uid128 && comm_out && nranks >= 1 && rank >= 0 && rank < nranks, "bad args");
  ncclUniqueId id;
  memcpy(&id, uid128, sizeof(id));
  ncclComm_t c;
  MP_NCCL(ncclCommInitRank(&c, nranks, id, rank));
  *comm_out = c;
  return 0;
}

int mp_comm_destroy(void* comm) {
  clear_error();
  if (!comm) return 0;
  MP_NCCL(ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm)));
  return 0;
}

// Watchdog support (the deadlock half of SimError, sim.py:172-178): a hung
// collective is released by aborting its communicator; asynchronous NCCL
// failures (a peer died, a network error) are polled without blocking.
int mp_comm_abort(void* comm) {
  clear_error();
  if (!comm) return 0;
  MP_NCCL(ncclCommAbort(reinterpret_cast<ncclComm_t>(comm)));
  return 0;
}

int mp_comm_async_error(void* comm, int* nccl_result) {
  clear_error();
  MP_CHECK_ARG(comm && nccl_result, "bad args");
  ncclResult_t r = ncclSuccess;
  MP_NCCL(ncclCommGetAsyncError(reinterpret_cast<ncclComm_t>(comm), &r));
  *nccl_result = (int)r;
  if (r != ncclSuccess && r != ncclInProgress) set_error(ncclGetErrorString(r));
  return 0;
}

int mp_allreduce(void* comm, void* buf, int64_t count, int dtype, int op, void* stream) {
  clear_error();
  MP_CHECK_ARG(comm && buf && count >= 0 && (op == 0 || op == 1), "bad args");
  if (count == 0) return 0;
  MP_NCCL(ncclAllReduce(buf, buf, (size_t)count, nccl_dtype(dtype), op ? ncclMax : ncclSum,
                        reinterpret_cast<ncclComm_t>(comm), reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}

int mp_allgather(void* comm, const void* send, void* recv, int64_t sendcount, int dtype,
                 void* stream) {
  clear_error();
  MP_CHECK_ARG(comm && send && recv && sendcount >= 0, "bad args");
  if (sendcount == 0) return 0;
  MP_NCCL(ncclAllGather(send, recv, (size_t)sendcount, nccl_dtype(dtype),
                        reinterpret_cast<ncclComm_t>(comm), reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}

int mp_reduce_scatter(void* comm, const void* send, void* recv, int64_t recvcount, int dtype,
                      int op, void* stream) {
  clear_error();
  MP_CHECK_ARG(comm && send && recv && recvcount >= 0, "bad args");
  if (recvcount == 0) return 0;
  MP_NCCL(ncclReduceScatter(send, recv, (size_t)recvcount, nccl_dtype(dtype),
                            op == 1 ? ncclMax : ncclSum, reinterpret_cast<ncclComm_t>(comm),
                            reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}

// All-to-all of equal chunks (the resharding_cost all_to_all, sharding.py:346): chunk i
// of `send` goes to rank i, chunk i of `recv` comes from rank i, `count` elements per
// chunk; one NCCL group of sends / recvs to every rank (NCCL has no all-to-all
// primitive; grouped point-to-point is its documented form).
int mp_alltoall(void* comm, const void* send, void* recv, int64_t count, int dtype, void* stream) {
  clear_error();
  MP_CHECK_ARG(comm && send && recv && count >= 0, "bad args");
  if (count == 0) return 0;
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
  int n = 0;
  MP_NCCL(ncclCommCount(c, &n));
  const size_t eb = dtype == 0 ? 2 : (dtype == 1 ? 4 : 1);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  MP_NCCL(ncclGroupStart());
  for (int r = 0; r < n; ++r) {
    const ncclResult_t a = ncclSend(static_cast<const char*>(send) + (size_t)r * count * eb,
                                    (size_t)count, nccl_dtype(dtype), r, c, st);
    const ncclResult_t b = ncclRecv(static_cast<char*>(recv) + (size_t)r * count * eb,
                                    (size_t)count, nccl_dtype(dtype), r, c, st);
    if (a != ncclSuccess || b != ncclSuccess) {
      ncclGroupEnd();
      set_error(std::string("mp_alltoall: ") + ncclGetErrorString(a != ncclSuccess ? a : b));
      return 1;
    }
  }
  MP_NCCL(ncclGroupEnd());
  return 0;
}

int mp_group_start(void) {
  clear_error();
  MP_NCCL(ncclGroupStart());
  return 0;
}

int mp_group_end(void) {
  clear_error();
  MP_NCCL(ncclGroupEnd());
  return 0;
}

int mp_send(void* comm, const void* buf, int64_t count, int dtype, int peer, void* stream) {
  clear_error();
  MP_CHECK_ARG(comm && buf && count >= 0 && peer >= 0, "bad args");
  if (count == 0) return 0;
  MP_NCCL(ncclSend(buf, (size_t)count, nccl_dtype(dtype), peer,
                   reinterpret_cast<ncclComm_t>(comm), reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}

int mp_recv(void* comm, void* buf, int64_t count, int dtype, int peer, void* stream) {
  clear_error();
  MP_CHECK_ARG(comm && buf && count >= 0 && peer >= 0, "bad args");
  if (count == 0) return 0;
  MP_NCCL(ncclRecv(buf, (size_t)count, nccl_dtype(dtype), peer,
                   reinterpret_cast<ncclComm_t>(comm), reinterpret_cast<cudaStream_t>(stream)));
  return 0;
}

}  // extern "C"
