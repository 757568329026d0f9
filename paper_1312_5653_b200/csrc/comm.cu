// comm.cu — see comm.hpp.
#include <nccl.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "comm.hpp"
#include "host_core.hpp"

namespace fetigpu {

#define CUC(call)                                                                                \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) throw RuntimeError(std::string("CUDA error: ") + cudaGetErrorString(e_)); \
  } while (0)
#define NCC(call)                                                                                \
  do {                                                                                           \
    ncclResult_t r_ = (call);                                                                    \
    if (r_ != ncclSuccess) throw RuntimeError(std::string("NCCL error: ") + ncclGetErrorString(r_)); \
  } while (0)

// ------------------------------------------------------------------ thread emulation
void ThreadComm::reduce(double* buf, size_t count, cudaStream_t s, bool max) {
  host_a_.resize(count);
  host_b_.resize(count);
  CUC(cudaMemcpyAsync(host_a_.data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUC(cudaStreamSynchronize(s));
  g_->posted[rank_] = host_a_.data();
  g_->barrier();
  // every rank sums the posted host copies in rank order: identical results everywhere
  for (size_t i = 0; i < count; ++i) {
    double acc = g_->posted[0][i];
    for (int q = 1; q < g_->world; ++q) acc = max ? std::max(acc, g_->posted[q][i]) : acc + g_->posted[q][i];
    host_b_[i] = acc;
  }
  g_->barrier();
  CUC(cudaMemcpyAsync(buf, host_b_.data(), count * sizeof(double), cudaMemcpyHostToDevice, s));
  CUC(cudaStreamSynchronize(s));
}

void ThreadComm::exchange(const double* send_up, size_t n_send_up, double* recv_up, size_t n_recv_up,
                          const double* send_down, size_t n_send_down, double* recv_down, size_t n_recv_down,
                          cudaStream_t s) {
  (void)n_send_up;
  (void)n_send_down;
  CUC(cudaStreamSynchronize(s));
  g_->posted[rank_] = send_up;
  g_->posted2[rank_] = send_down;
  g_->barrier();
  if (rank_ + 1 < g_->world && n_recv_up)
    CUC(cudaMemcpyAsync(recv_up, g_->posted2[rank_ + 1], n_recv_up * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (rank_ > 0 && n_recv_down)
    CUC(cudaMemcpyAsync(recv_down, g_->posted[rank_ - 1], n_recv_down * sizeof(double), cudaMemcpyDeviceToDevice, s));
  CUC(cudaStreamSynchronize(s));
  g_->barrier();
}

void ThreadComm::allgatherv(double* buf, const std::vector<size_t>& first, const std::vector<size_t>& count,
                            cudaStream_t s) {
  CUC(cudaStreamSynchronize(s));
  g_->posted[rank_] = buf;
  g_->barrier();
  for (int q = 0; q < g_->world; ++q)
    if (q != rank_ && count[q])
      CUC(cudaMemcpyAsync(buf + first[q], g_->posted[q] + first[q], count[q] * sizeof(double),
                          cudaMemcpyDeviceToDevice, s));
  CUC(cudaStreamSynchronize(s));
  g_->barrier();
}

// ------------------------------------------------------------------ NCCL
class NcclComm : public Comm {
 public:
  NcclComm(const unsigned char* id, int rank, int world, int device) : rank_(rank), world_(world) {
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == 128, "unexpected ncclUniqueId size");
    std::memcpy(uid.internal, id, 128);
    CUC(cudaSetDevice(device));
    NCC(ncclCommInitRank(&comm_, world, uid, rank));
  }
  ~NcclComm() override {
    if (comm_) ncclCommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  void allreduce_sum(double* buf, size_t count, cudaStream_t s) override {
    NCC(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, comm_, s));
  }
  void allreduce_max(double* buf, size_t count, cudaStream_t s) override {
    NCC(ncclAllReduce(buf, buf, count, ncclDouble, ncclMax, comm_, s));
  }
  void exchange(const double* send_up, size_t n_send_up, double* recv_up, size_t n_recv_up, const double* send_down,
                size_t n_send_down, double* recv_down, size_t n_recv_down, cudaStream_t s) override {
    NCC(ncclGroupStart());
    if (rank_ + 1 < world_) {
      if (n_send_up) NCC(ncclSend(send_up, n_send_up, ncclDouble, rank_ + 1, comm_, s));
      if (n_recv_up) NCC(ncclRecv(recv_up, n_recv_up, ncclDouble, rank_ + 1, comm_, s));
    }
    if (rank_ > 0) {
      if (n_send_down) NCC(ncclSend(send_down, n_send_down, ncclDouble, rank_ - 1, comm_, s));
      if (n_recv_down) NCC(ncclRecv(recv_down, n_recv_down, ncclDouble, rank_ - 1, comm_, s));
    }
    NCC(ncclGroupEnd());
  }
  void allgatherv(double* buf, const std::vector<size_t>& first, const std::vector<size_t>& count,
                  cudaStream_t s) override {
    NCC(ncclGroupStart());
    for (int q = 0; q < world_; ++q)
      if (count[q]) NCC(ncclBroadcast(buf + first[q], buf + first[q], count[q], ncclDouble, q, comm_, s));
    NCC(ncclGroupEnd());
  }

 private:
  ncclComm_t comm_ = nullptr;
  int rank_, world_;
};

std::unique_ptr<Comm> make_nccl_comm(const unsigned char* unique_id, int rank, int world, int device) {
  return std::make_unique<NcclComm>(unique_id, rank, world, device);
}

int nccl_unique_id(unsigned char* out128) {
  ncclUniqueId uid;
  NCC(ncclGetUniqueId(&uid));
  std::memcpy(out128, uid.internal, 128);
  return 0;
}

}  // namespace fetigpu
