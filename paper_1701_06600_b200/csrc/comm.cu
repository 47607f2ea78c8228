// Backends of the sharded path's communication plane (comm.hpp).
#include "comm.hpp"

#include <nccl.h>

#include <cstring>
#include <string>

#include "devutil.cuh"

namespace cpb {

namespace {

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + ncclGetErrorString(r));
}

class NcclComm final : public Comm {
 public:
  NcclComm(const unsigned char id[128], int r, int p, int dev) {
    rank = r;
    nranks = p;
    device = dev;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    CPB_CUDA(cudaSetDevice(dev));
    nccl_ok(ncclCommInitRank(&comm_, p, uid, r), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) ncclCommDestroy(comm_);
  }
  void allreduce_sum(double* buf, i64 n, cudaStream_t st) override {
    if (n == 0) return;
    nccl_ok(ncclAllReduce(buf, buf, static_cast<size_t>(n), ncclDouble, ncclSum, comm_, st), "ncclAllReduce");
  }
  void allgather(double* buf, i64 per_rank, cudaStream_t st) override {
    if (per_rank == 0) return;
    nccl_ok(ncclAllGather(buf + static_cast<i64>(rank) * per_rank, buf, static_cast<size_t>(per_rank), ncclDouble,
                          comm_, st),
            "ncclAllGather");
  }
  void exchange(const std::vector<const double*>& send, const std::vector<i64>& sc, const std::vector<double*>& recv,
                const std::vector<i64>& rc, cudaStream_t st) override {
    nccl_ok(ncclGroupStart(), "ncclGroupStart");
    for (int q = 0; q < nranks; ++q)
      if (sc[static_cast<size_t>(q)] > 0)
        nccl_ok(ncclSend(send[static_cast<size_t>(q)], static_cast<size_t>(sc[static_cast<size_t>(q)]), ncclDouble, q,
                         comm_, st),
                "ncclSend");
    for (int q = 0; q < nranks; ++q)
      if (rc[static_cast<size_t>(q)] > 0)
        nccl_ok(ncclRecv(recv[static_cast<size_t>(q)], static_cast<size_t>(rc[static_cast<size_t>(q)]), ncclDouble, q,
                         comm_, st),
                "ncclRecv");
    nccl_ok(ncclGroupEnd(), "ncclGroupEnd");
  }
  const char* kind() const override { return "nccl"; }

 private:
  ncclComm_t comm_ = nullptr;
};

constexpr int kMaxLoopRanks = 16;
struct PtrSet {
  const double* p[kMaxLoopRanks];
};

// out[e] = sum_q in.p[q][e], q = 0, 1, ... (rank order)
__global__ void rank_order_sum_kernel(PtrSet in, int nranks, i64 n, double* __restrict__ out) {
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nranks; ++q) s += in.p[q][e];
    out[e] = s;
  }
}

class LoopbackComm final : public Comm {
 public:
  LoopbackComm(std::shared_ptr<LoopbackGroup> g, int r, int dev) : g_(std::move(g)) {
    rank = r;
    nranks = g_->nranks;
    device = dev;
  }
  ~LoopbackComm() override {
    if (tmp_) cudaFree(tmp_);
  }
  void allreduce_sum(double* buf, i64 n, cudaStream_t st) override {
    CPB_CUDA(cudaStreamSynchronize(st));  // this rank's partial is complete
    g_->slot[static_cast<size_t>(rank)] = buf;
    g_->bar.arrive_and_wait();  // every partial is published
    if (n > 0) {
      if (n > tmp_n_) {
        if (tmp_) CPB_CUDA(cudaFree(tmp_));
        CPB_CUDA(cudaMalloc(&tmp_, static_cast<size_t>(n) * sizeof(double)));
        tmp_n_ = n;
      }
      PtrSet ps{};
      for (int q = 0; q < nranks; ++q) ps.p[q] = g_->slot[static_cast<size_t>(q)];
      const int grid = static_cast<int>(std::min<i64>((n + 255) / 256, 1024));
      rank_order_sum_kernel<<<grid, 256, 0, st>>>(ps, nranks, n, tmp_);
      CPB_LAUNCH_CHECK();
      CPB_CUDA(cudaStreamSynchronize(st));
    }
    g_->bar.arrive_and_wait();  // every rank has read every partial
    if (n > 0) CPB_CUDA(cudaMemcpyAsync(buf, tmp_, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  void allgather(double* buf, i64 per_rank, cudaStream_t st) override {
    CPB_CUDA(cudaStreamSynchronize(st));
    g_->slot[static_cast<size_t>(rank)] = buf;
    g_->bar.arrive_and_wait();
    if (per_rank > 0) {
      for (int q = 0; q < nranks; ++q)
        if (q != rank)
          CPB_CUDA(cudaMemcpyAsync(buf + static_cast<i64>(q) * per_rank,
                                   g_->slot[static_cast<size_t>(q)] + static_cast<i64>(q) * per_rank,
                                   static_cast<size_t>(per_rank) * sizeof(double), cudaMemcpyDeviceToDevice, st));
      CPB_CUDA(cudaStreamSynchronize(st));
    }
    g_->bar.arrive_and_wait();  // nobody rewrites its block before every rank copied it
  }
  void exchange(const std::vector<const double*>& send, const std::vector<i64>& sc, const std::vector<double*>& recv,
                const std::vector<i64>& rc, cudaStream_t st) override {
    CPB_CUDA(cudaStreamSynchronize(st));
    g_->sends[static_cast<size_t>(rank)] = send;
    g_->counts[static_cast<size_t>(rank)] = sc;
    g_->bar.arrive_and_wait();
    for (int q = 0; q < nranks; ++q) {
      const i64 want = rc[static_cast<size_t>(q)];
      const i64 have = g_->counts[static_cast<size_t>(q)][static_cast<size_t>(rank)];
      if (want != have) throw InvalidArgument("loopback exchange: send / receive counts disagree");
      if (want > 0)
        CPB_CUDA(cudaMemcpyAsync(recv[static_cast<size_t>(q)], g_->sends[static_cast<size_t>(q)][static_cast<size_t>(rank)],
                                 static_cast<size_t>(want) * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    CPB_CUDA(cudaStreamSynchronize(st));
    g_->bar.arrive_and_wait();
  }
  const char* kind() const override { return "loopback"; }

 private:
  std::shared_ptr<LoopbackGroup> g_;
  double* tmp_ = nullptr;
  i64 tmp_n_ = 0;
};

}  // namespace

LoopbackGroup::LoopbackGroup(int p)
    : nranks(p), bar(p), slot(static_cast<size_t>(p), nullptr),
      sends(static_cast<size_t>(p)), counts(static_cast<size_t>(p)) {
  if (p < 1 || p > kMaxLoopRanks) throw InvalidArgument("loopback group: 1..16 ranks");
}

std::unique_ptr<Comm> make_nccl_comm(const unsigned char id[128], int rank, int nranks, int device) {
  return std::make_unique<NcclComm>(id, rank, nranks, device);
}

void nccl_unique_id(unsigned char out[128]) {
  ncclUniqueId id;
  nccl_ok(ncclGetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
}

std::unique_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank, int device) {
  if (rank < 0 || rank >= g->nranks) throw InvalidArgument("bad rank");
  return std::make_unique<LoopbackComm>(std::move(g), rank, device);
}

}  // namespace cpb
