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

  // CUDA IPC: peers' allocations mapped into this process (NVLink P2P).
  // share_pointers returns an empty vector (on every rank) when some rank
  // could not map a peer's memory; the session then runs the chain.
  int peer_mode() const override { return 1; }
  std::vector<void*> share_pointers(void* mine) override {
    cudaIpcMemHandle_t h;
    CPB_CUDA(cudaIpcGetMemHandle(&h, mine));
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    char* d = nullptr;
    CPB_CUDA(cudaMalloc(&d, hb * static_cast<size_t>(nranks)));
    CPB_CUDA(cudaMemcpy(d + hb * static_cast<size_t>(rank), &h, hb, cudaMemcpyHostToDevice));
    nccl_ok(ncclAllGather(d + hb * static_cast<size_t>(rank), d, hb, ncclChar, comm_, nullptr), "ncclAllGather");
    CPB_CUDA(cudaStreamSynchronize(nullptr));
    std::vector<char> all(hb * static_cast<size_t>(nranks));
    CPB_CUDA(cudaMemcpy(all.data(), d, all.size(), cudaMemcpyDeviceToHost));
    CPB_CUDA(cudaFree(d));
    std::vector<void*> out(static_cast<size_t>(nranks), nullptr);
    double ok = 1.0;
    for (int q = 0; q < nranks; ++q) {
      if (q == rank) {
        out[static_cast<size_t>(q)] = mine;
        continue;
      }
      cudaIpcMemHandle_t hq;
      std::memcpy(&hq, all.data() + hb * static_cast<size_t>(q), hb);
      if (cudaIpcOpenMemHandle(&out[static_cast<size_t>(q)], hq, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        out[static_cast<size_t>(q)] = nullptr;
        ok = 0.0;
      }
    }
    double* dk = nullptr;  // every rank must have mapped every peer
    CPB_CUDA(cudaMalloc(&dk, sizeof(double)));
    CPB_CUDA(cudaMemcpy(dk, &ok, sizeof(double), cudaMemcpyHostToDevice));
    nccl_ok(ncclAllReduce(dk, dk, 1, ncclDouble, ncclMin, comm_, nullptr), "ncclAllReduce");
    CPB_CUDA(cudaStreamSynchronize(nullptr));
    CPB_CUDA(cudaMemcpy(&ok, dk, sizeof(double), cudaMemcpyDeviceToHost));
    CPB_CUDA(cudaFree(dk));
    if (ok < 0.5) {
      release_pointers(out);
      return {};
    }
    return out;
  }
  void release_pointers(std::vector<void*>& ptrs) override {
    for (int q = 0; q < static_cast<int>(ptrs.size()); ++q)
      if (q != rank && ptrs[static_cast<size_t>(q)]) cudaIpcCloseMemHandle(ptrs[static_cast<size_t>(q)]);
    ptrs.clear();
  }

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

  int peer_mode() const override { return 2; }
  std::vector<void*> share_pointers(void* mine) override {
    g_->ptrs[static_cast<size_t>(rank)] = mine;
    g_->bar.arrive_and_wait();
    std::vector<void*> out = g_->ptrs;
    g_->bar.arrive_and_wait();
    return out;
  }
  void launch_group(const void* my_args, cudaStream_t st,
                    const std::function<void(const std::vector<const void*>&, cudaStream_t)>& launch) override {
    // every rank's stream position, then one launch on rank 0's stream that
    // all ranks' streams wait for (no rank's kernel waits on another launch)
    CPB_CUDA(cudaEventRecord(g_->ev[static_cast<size_t>(rank)], st));
    g_->ptrs[static_cast<size_t>(rank)] = const_cast<void*>(my_args);
    g_->bar.arrive_and_wait();
    if (rank == 0) {
      for (int q = 1; q < nranks; ++q) CPB_CUDA(cudaStreamWaitEvent(st, g_->ev[static_cast<size_t>(q)], 0));
      std::vector<const void*> args(g_->ptrs.begin(), g_->ptrs.end());
      launch(args, st);
      CPB_CUDA(cudaEventRecord(g_->ev_launch, st));
    }
    g_->bar.arrive_and_wait();
    if (rank != 0) CPB_CUDA(cudaStreamWaitEvent(st, g_->ev_launch, 0));
  }

 private:
  std::shared_ptr<LoopbackGroup> g_;
  double* tmp_ = nullptr;
  i64 tmp_n_ = 0;
};

}  // namespace

LoopbackGroup::LoopbackGroup(int p)
    : nranks(p), bar(p), slot(static_cast<size_t>(p), nullptr),
      sends(static_cast<size_t>(p)), counts(static_cast<size_t>(p)), ptrs(static_cast<size_t>(p), nullptr),
      ev(static_cast<size_t>(p), nullptr) {
  if (p < 1 || p > kMaxLoopRanks) throw InvalidArgument("loopback group: 1..16 ranks");
  for (auto& e : ev) CPB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CPB_CUDA(cudaEventCreateWithFlags(&ev_launch, cudaEventDisableTiming));
}

LoopbackGroup::~LoopbackGroup() {
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  if (ev_launch) cudaEventDestroy(ev_launch);
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
