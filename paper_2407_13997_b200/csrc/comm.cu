// Transports of the strip partition (comm.h).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "comm.h"

namespace wrmg {
namespace {

// ------------------------------------------------------------------- NCCL
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl(std::string &err) {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // prefer an already loaded libnccl (torch's), else the system one
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
#define SYM(f) api.f = (decltype(api.f))dlsym(h, "nccl" #f)
      SYM(GetUniqueId);
      SYM(CommInitRank);
      SYM(CommDestroy);
      SYM(Send);
      SYM(Recv);
      SYM(GroupStart);
      SYM(GroupEnd);
      SYM(AllGather);
      SYM(GetErrorString);
#undef SYM
      api.ok = api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.GroupStart && api.GroupEnd &&
               api.AllGather && api.CommDestroy;
    }
  }
  if (!api.ok) err = "libnccl.so.2 not found or incomplete";
  return api;
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclApi *api = nullptr;
  void check(ncclResult_t r) {
    if (r != ncclSuccess) throw std::string("NCCL: ") + (api->GetErrorString ? api->GetErrorString(r) : "error");
  }
  ~NcclComm() override {
    if (comm) api->CommDestroy(comm);
  }
  void exchange(const double *sendL, double *recvL, size_t nL, const double *sendR, double *recvR, size_t nR,
                cudaStream_t s) override {
    check(api->GroupStart());
    if (rank > 0 && nL) {
      check(api->Send(sendL, nL, ncclFloat64, rank - 1, comm, s));
      check(api->Recv(recvL, nL, ncclFloat64, rank - 1, comm, s));
    }
    if (rank < nranks - 1 && nR) {
      check(api->Send(sendR, nR, ncclFloat64, rank + 1, comm, s));
      check(api->Recv(recvR, nR, ncclFloat64, rank + 1, comm, s));
    }
    check(api->GroupEnd());
  }
  void allgather(const double *send, double *recv, size_t n, cudaStream_t s) override {
    check(api->AllGather(send, recv, n, ncclFloat64, comm, s));
  }
};

// --------------------------------------------------------------- loopback
struct Hub {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int count = 0;
  long gen = 0;
  std::vector<const double *> pl, pr, pg;
  explicit Hub(int n_) : n(n_), pl(n_), pr(n_), pg(n_) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long g = gen;
    if (++count == n) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LoopComm : Comm {
  Hub *hub = nullptr;
  void ck(cudaError_t e) {
    if (e != cudaSuccess) throw std::string("loopback: ") + cudaGetErrorString(e);
  }
  void exchange(const double *sendL, double *recvL, size_t nL, const double *sendR, double *recvR, size_t nR,
                cudaStream_t s) override {
    ck(cudaStreamSynchronize(s));  // this rank's send buffers are packed
    hub->pl[rank] = sendL;
    hub->pr[rank] = sendR;
    hub->barrier();
    if (rank > 0 && nL) ck(cudaMemcpyAsync(recvL, hub->pr[rank - 1], nL * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (rank < nranks - 1 && nR)
      ck(cudaMemcpyAsync(recvR, hub->pl[rank + 1], nR * sizeof(double), cudaMemcpyDeviceToDevice, s));
    ck(cudaStreamSynchronize(s));
    hub->barrier();  // the neighbours' send buffers may be reused after this
  }
  void allgather(const double *send, double *recv, size_t n, cudaStream_t s) override {
    ck(cudaStreamSynchronize(s));
    hub->pg[rank] = send;
    hub->barrier();
    for (int q = 0; q < nranks; ++q)
      ck(cudaMemcpyAsync(recv + (size_t)q * n, hub->pg[q], n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    ck(cudaStreamSynchronize(s));
    hub->barrier();
  }
};

}  // namespace

bool nccl_get_unique_id(void *out128, std::string &err) {
  NcclApi &api = nccl(err);
  if (!api.ok) return false;
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) {
    err = "ncclGetUniqueId failed";
    return false;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out128, &id, 128);
  return true;
}

Comm *make_nccl_comm(const void *unique_id, int rank, int nranks, std::string &err) {
  NcclApi &api = nccl(err);
  if (!api.ok) return nullptr;
  if (!unique_id) {
    err = "nccl_unique_id is NULL";
    return nullptr;
  }
  ncclUniqueId id;
  memcpy(&id, unique_id, 128);
  auto *c = new NcclComm();
  c->api = &api;
  c->rank = rank;
  c->nranks = nranks;
  ncclResult_t r = api.CommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + (api.GetErrorString ? api.GetErrorString(r) : "error");
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

void *loop_hub_create(int nranks) { return new Hub(nranks); }
void loop_hub_destroy(void *hub) { delete static_cast<Hub *>(hub); }

Comm *make_loop_comm(void *hub, int rank, int nranks, std::string &err) {
  Hub *h = static_cast<Hub *>(hub);
  if (!h || h->n != nranks) {
    err = "loopback hub missing or sized for another rank count";
    return nullptr;
  }
  auto *c = new LoopComm();
  c->hub = h;
  c->rank = rank;
  c->nranks = nranks;
  return c;
}

}  // namespace wrmg
