// libucp_b200_comm.so -- NCCL transport for the rank-homed load exchange
// (ucp_comm_init / ucp_alltoallv / ucp_comm_destroy; §8(e)).
//
// One process per GPU: rank 0 creates a ucp_comm_id, the caller distributes
// it (e.g. torch.distributed broadcast), every rank calls ucp_comm_init.
// ucp_alltoallv is one grouped ncclSend/ncclRecv over NVLink / NVSwitch.
// The default transport of the product is the fused kernel writing straight
// into peer memory (ucp_ipc_*, include/ucp_b200.h); this library is the
// collective alternative and the C entry point for non-Python callers.

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include "ucp_b200_comm.h"

static_assert(sizeof(ncclUniqueId) == sizeof(ucp_comm_id), "ncclUniqueId size");

extern "C" {

int ucp_comm_version(void) { return UCP_COMM_ABI_VERSION; }

#ifndef UCP_BUILD_ID
#define UCP_BUILD_ID "unknown"
#endif
const char* ucp_comm_build_id(void) { return "UCP_BUILD_ID:" UCP_BUILD_ID; }

int ucp_comm_unique_id(ucp_comm_id* out) {
  if (!out) return UCP_COMM_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return UCP_COMM_ENCCL;
  memcpy(out->bytes, &id, sizeof(id));
  return 0;
}

int ucp_comm_init(int nranks, int rank, const ucp_comm_id* id, void** comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return UCP_COMM_EINVAL;
  ncclUniqueId uid;
  memcpy(&uid, id->bytes, sizeof(uid));
  ncclComm_t c = nullptr;
  if (ncclCommInitRank(&c, nranks, uid, rank) != ncclSuccess) return UCP_COMM_ENCCL;
  *comm = c;
  return 0;
}

int ucp_alltoallv(void* comm, const void* send, const uint64_t* send_counts, void* recv,
                  const uint64_t* recv_counts, void* stream) {
  if (!comm || !send_counts || !recv_counts) return UCP_COMM_EINVAL;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int n = 0;
  if (ncclCommCount(c, &n) != ncclSuccess) return UCP_COMM_ENCCL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const char* sb = static_cast<const char*>(send);
  char* rb = static_cast<char*>(recv);
  uint64_t so = 0, ro = 0;
  if (ncclGroupStart() != ncclSuccess) return UCP_COMM_ENCCL;
  for (int p = 0; p < n; ++p) {
    if (send_counts[p] &&
        ncclSend(sb + so, send_counts[p], ncclUint8, p, c, s) != ncclSuccess) {
      ncclGroupEnd();
      return UCP_COMM_ENCCL;
    }
    if (recv_counts[p] &&
        ncclRecv(rb + ro, recv_counts[p], ncclUint8, p, c, s) != ncclSuccess) {
      ncclGroupEnd();
      return UCP_COMM_ENCCL;
    }
    so += send_counts[p];
    ro += recv_counts[p];
  }
  return ncclGroupEnd() == ncclSuccess ? 0 : UCP_COMM_ENCCL;
}

int ucp_comm_destroy(void* comm) {
  if (!comm) return 0;
  return ncclCommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? 0 : UCP_COMM_ENCCL;
}

}  // extern "C"
