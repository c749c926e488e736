/*
 * ucp_b200_comm.h -- C ABI of libucp_b200_comm.so: the NCCL all-to-all-v
 * of the rank-homed load exchange (SURVEY §8(b) ucp_comm_init /
 * ucp_alltoallv / ucp_comm_destroy, §8(e)). The reference has no collective
 * at all: its load "simulates" the all-gather in one process
 * (ucp/load.py:185-206; the paper's system all-gathers over NVLink,
 * PAPER.md:531).
 *
 * One process per GPU. Counts are bytes, in HOST arrays of nranks entries;
 * send/recv are device buffers holding the per-peer chunks back to back in
 * rank order. Calls are stream-ordered. Returns 0 or a negative code.
 */
#ifndef UCP_B200_COMM_H
#define UCP_B200_COMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UCP_COMM_ABI_VERSION 1
#define UCP_COMM_EINVAL (-10)
#define UCP_COMM_ENCCL (-12)

typedef struct ucp_comm_id {
  char bytes[128]; /* ncclUniqueId */
} ucp_comm_id;

int ucp_comm_version(void);
/* "UCP_BUILD_ID:" + sha256(csrc/ucp_comm.cpp || this header)[:32 hex] */
const char* ucp_comm_build_id(void);
int ucp_comm_unique_id(ucp_comm_id* out);
int ucp_comm_init(int nranks, int rank, const ucp_comm_id* id, void** comm);
int ucp_alltoallv(void* comm, const void* send, const uint64_t* send_counts, void* recv,
                  const uint64_t* recv_counts, void* stream);
int ucp_comm_destroy(void* comm);

#ifdef __cplusplus
}
#endif

#endif /* UCP_B200_COMM_H */
