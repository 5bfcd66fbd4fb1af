// Inter-rank transport of the strip partition: neighbour halo
// exchange and all-gather, stream-ordered on the caller's stream.
//   * NcclComm: NCCL point-to-point / all-gather over NVLink (libnccl.so.2 opened
//     at run time; one process per GPU, unique id from rank 0 via torch.distributed).
//   * LoopComm: ranks as host threads of one process sharing a hub (tests on one
//     GPU): each rank's kernels run on its own stream, the hand-over of finished
//     buffers is a host barrier plus device-to-device copies -- no kernel waits on
//     another rank's kernel.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <string>

namespace wrmg {

struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() {}
  // Send nL doubles to rank-1 and nR to rank+1; receive nL from rank-1 into recvL
  // and nR from rank+1 into recvR (counts are symmetric by construction).
  virtual void exchange(const double *sendL, double *recvL, size_t nL, const double *sendR, double *recvR, size_t nR,
                        cudaStream_t s) = 0;
  // recv[q n .. (q+1) n) = send of rank q.
  virtual void allgather(const double *send, double *recv, size_t n, cudaStream_t s) = 0;
};

// Returns nullptr and sets err on failure.
Comm *make_nccl_comm(const void *unique_id, int rank, int nranks, std::string &err);
Comm *make_loop_comm(void *hub, int rank, int nranks, std::string &err);
void *loop_hub_create(int nranks);
void loop_hub_destroy(void *hub);
bool nccl_get_unique_id(void *out128, std::string &err);

}  // namespace wrmg
