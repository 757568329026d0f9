// comm.hpp — inter-rank communication of the sharded FETI-DP path.
//
//   NcclComm   one process per GPU, NCCL over NVLink/NVSwitch: ncclAllReduce for the coarse
//              rhs and the Krylov dot vectors, grouped ncclSend/ncclRecv for the cut-line
//              halo (~16 KB per neighbour per exchange), grouped ncclBroadcast to assemble
//              the primal solution.
//   ThreadComm W ranks emulated by W host threads of one process on ONE device: at every
//              collective each rank synchronises its own stream, meets the others at a host
//              barrier and copies device-to-device.  Kernels never wait on other ranks'
//              kernels; only host threads wait.  Used to test the sharded logic on one GPU.
// All counts are in doubles (a complex value is 2 doubles).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <vector>

namespace fetigpu {

struct Comm {
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  virtual void allreduce_sum(double* buf, size_t count, cudaStream_t s) = 0;
  virtual void allreduce_max(double* buf, size_t count, cudaStream_t s) = 0;
  // neighbour exchange: send_up -> rank+1 (which receives it as its recv_down) and
  // send_down -> rank-1 (received as its recv_up).  Missing neighbours are skipped.
  virtual void exchange(const double* send_up, size_t n_send_up, double* recv_up, size_t n_recv_up,
                        const double* send_down, size_t n_send_down, double* recv_down, size_t n_recv_down,
                        cudaStream_t s) = 0;
  // in place: rank q's segment [first[q], first[q] + count[q]) is replicated on every rank
  virtual void allgatherv(double* buf, const std::vector<size_t>& first, const std::vector<size_t>& count,
                          cudaStream_t s) = 0;
};

// ------------------------------------------------------------------ thread emulation
struct ThreadGroup {
  explicit ThreadGroup(int w) : world(w), posted(w, nullptr), posted2(w, nullptr), tmp(w, nullptr) {}
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<const double*> posted, posted2;
  std::vector<double*> tmp;
  bool aborted = false;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (aborted) throw std::runtime_error("rank group aborted");
    const long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen || aborted; });
      if (aborted && generation == gen) throw std::runtime_error("rank group aborted");
    }
  }
  // a failing rank releases the others (they throw instead of waiting forever)
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

class ThreadComm : public Comm {
 public:
  ThreadComm(std::shared_ptr<ThreadGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
  int rank() const override { return rank_; }
  int world() const override { return g_->world; }
  void allreduce_sum(double* buf, size_t count, cudaStream_t s) override { reduce(buf, count, s, false); }
  void allreduce_max(double* buf, size_t count, cudaStream_t s) override { reduce(buf, count, s, true); }
  void exchange(const double* send_up, size_t n_send_up, double* recv_up, size_t n_recv_up, const double* send_down,
                size_t n_send_down, double* recv_down, size_t n_recv_down, cudaStream_t s) override;
  void allgatherv(double* buf, const std::vector<size_t>& first, const std::vector<size_t>& count,
                  cudaStream_t s) override;

 private:
  void reduce(double* buf, size_t count, cudaStream_t s, bool max);
  std::shared_ptr<ThreadGroup> g_;
  int rank_;
  std::vector<double> host_a_, host_b_;
};

// ------------------------------------------------------------------ NCCL
std::unique_ptr<Comm> make_nccl_comm(const unsigned char* unique_id, int rank, int world, int device);
int nccl_unique_id(unsigned char* out128);

}  // namespace fetigpu
