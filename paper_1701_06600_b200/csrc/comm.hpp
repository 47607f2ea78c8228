// Communication plane of the slab-sharded path: the three
// exchanges the sharded CPRAND / CPRAND-MIX loop needs, behind one interface.
//
//   allreduce_sum  RHS partials (R x I_n), column sums of squares, fit values
//   allgather      the last mode's factor slabs / RHS slabs (in place)
//   exchange       grouped point-to-point blocks (the distributed mixing
//                  pass's all-to-all)
//
// Backends:
//   NcclComm      production: one process per GPU, NCCL over NVLink/NVSwitch
//   LoopbackComm  P ranks of one process on one device (one host thread per
//                 rank), exchanging through each other's device buffers in
//                 rank order behind host barriers. It runs the product's
//                 sharded session code at P > 1 where only one GPU exists
//                 (tests); no rank's kernel ever waits on another rank's
//                 kernel: every rendezvous is a host barrier after a stream
//                 synchronize.
#pragma once

#include <cuda_runtime.h>

#include <barrier>
#include <functional>
#include <memory>
#include <vector>

#include "common.cuh"

namespace cpb {

class Comm {
 public:
  virtual ~Comm() = default;
  int rank = 0, nranks = 1, device = 0;
  // buf[0, n) <- sum over ranks (every rank gets the same values)
  virtual void allreduce_sum(double* buf, i64 n, cudaStream_t st) = 0;
  // buf[q * per_rank, (q + 1) * per_rank) <- rank q's block of its own buf
  virtual void allgather(double* buf, i64 per_rank, cudaStream_t st) = 0;
  // send[q] (send_count[q] doubles) goes to rank q, recv[q] (recv_count[q])
  // comes from rank q; zero counts are skipped
  virtual void exchange(const std::vector<const double*>& send, const std::vector<i64>& send_count,
                        const std::vector<double*>& recv, const std::vector<i64>& recv_count, cudaStream_t st) = 0;
  virtual const char* kind() const = 0;

  // ---- peer path (the slab-sharded CPRAND kernel exchanging through peer
  // memory inside the kernel)
  // 0: no peer access; 1: one kernel per rank, peers' buffers mapped into
  // this process (CUDA IPC over NVLink); 2: the ranks share one device and
  // one launch runs every rank's group (launch_group)
  virtual int peer_mode() const { return 0; }
  // every rank's device allocation `mine` (a cudaMalloc base) as this rank
  // addresses it; [rank] = mine. Collective.
  virtual std::vector<void*> share_pointers(void* mine) { return {mine}; }
  // undo share_pointers' mappings
  virtual void release_pointers(std::vector<void*>& ptrs) { ptrs.clear(); }
  // peer_mode 2: collective; rank 0 launches `launch(args of every rank, its
  // stream)` once every rank's stream reached this point, and every rank's
  // stream then waits for that launch
  virtual void launch_group(const void* my_args, cudaStream_t st,
                            const std::function<void(const std::vector<const void*>&, cudaStream_t)>& launch) {
    launch({my_args}, st);
  }
};

std::unique_ptr<Comm> make_nccl_comm(const unsigned char id[128], int rank, int nranks, int device);
void nccl_unique_id(unsigned char out[128]);

// Shared state of the P ranks of one loopback group.
struct LoopbackGroup {
  explicit LoopbackGroup(int p);
  ~LoopbackGroup();
  int nranks;
  std::barrier<> bar;
  std::vector<const double*> slot;                // [rank] published buffer
  std::vector<std::vector<const double*>> sends;  // [rank][peer]
  std::vector<std::vector<i64>> counts;           // [rank][peer]
  std::vector<void*> ptrs;                        // [rank] share_pointers / launch_group slots
  std::vector<cudaEvent_t> ev;                    // [rank] stream positions before a group launch
  cudaEvent_t ev_launch = nullptr;                // the group launch (rank 0's stream)
};
std::unique_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank, int device);

}  // namespace cpb
