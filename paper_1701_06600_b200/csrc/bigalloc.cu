// Device blocks of tensor size (the tensor a one-shot cprand_solve uploads,
// the private mixed copy, the mode-major replicas) are kept after release
// and handed out again for a request of the same size on the same device:
// repeated solves on same-shaped tensors (the e2e path, a serving loop) do
// not pay cudaMalloc / cudaFree of tens of GB each call. A failed cudaMalloc
// flushes the cache and retries; replica planning counts cached bytes as
// free (big_cached_bytes).
#include <mutex>
#include <vector>

#include "devutil.cuh"

namespace cpb {

namespace {
struct Block {
  int device;
  size_t bytes;
  void* p;
};
constexpr size_t kBigMin = size_t{256} << 20;  // cache blocks of >= 256 MB
constexpr int kMaxCached = 8;
std::mutex g_mu;
std::vector<Block> g_cache;  // oldest first

void flush_device(int dev) {
  for (auto it = g_cache.begin(); it != g_cache.end();) {
    if (it->device == dev) {
      cudaFree(it->p);
      it = g_cache.erase(it);
    } else {
      ++it;
    }
  }
}
}  // namespace

void* big_alloc(size_t bytes) {
  if (bytes == 0) bytes = 1;
  int dev = 0;
  CPB_CUDA(cudaGetDevice(&dev));
  if (bytes >= kBigMin) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
      if (it->device == dev && it->bytes == bytes) {
        void* p = it->p;
        g_cache.erase(it);
        return p;
      }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    {
      std::lock_guard<std::mutex> lk(g_mu);
      flush_device(dev);
    }
    e = cudaMalloc(&p, bytes);
  }
  CPB_CUDA(e);
  return p;
}

void big_free(void* p, size_t bytes) {
  if (!p) return;
  int dev = 0;
  if (bytes >= kBigMin && cudaGetDevice(&dev) == cudaSuccess) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_cache.push_back({dev, bytes, p});
    while (static_cast<int>(g_cache.size()) > kMaxCached) {
      cudaFree(g_cache.front().p);
      g_cache.erase(g_cache.begin());
    }
    return;
  }
  cudaFree(p);
}

size_t big_cached_bytes() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  std::lock_guard<std::mutex> lk(g_mu);
  size_t s = 0;
  for (const auto& b : g_cache)
    if (b.device == dev) s += b.bytes;
  return s;
}

void big_release_all() {
  std::lock_guard<std::mutex> lk(g_mu);
  for (const auto& b : g_cache) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(b.device);
    cudaFree(b.p);
    cudaSetDevice(cur);
  }
  g_cache.clear();
}

// Small pinned, device-mapped host blocks (a session's per-iteration stop
// marks): cudaHostAlloc costs milliseconds, so released blocks are kept for
// the next session (a time-to-fit measurement creates a session per run).
namespace {
struct HostBlock {
  size_t bytes;
  void* p;
};
std::vector<HostBlock> g_host;
constexpr int kMaxHostCached = 32;
}  // namespace

// Requests are rounded to a power of two (>= 4 KB) on both sides, so a
// released block serves any later request of its size class: sessions of
// different shapes in one process (the bench, a serving loop) then reuse
// each other's blocks instead of evicting them (cudaHostAlloc / cudaFreeHost
// of a few MB cost milliseconds and wait for the device).
static size_t host_class(size_t bytes) {
  size_t c = 4096;
  while (c < bytes) c <<= 1;
  return c;
}

void* pinned_mapped_alloc(size_t bytes) {
  const size_t cls = host_class(bytes);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_host.begin(); it != g_host.end(); ++it)
      if (it->bytes == cls) {
        void* p = it->p;
        g_host.erase(it);
        return p;
      }
  }
  void* p = nullptr;
  CPB_CUDA(cudaHostAlloc(&p, cls, cudaHostAllocMapped | cudaHostAllocPortable));
  return p;
}

void pinned_mapped_free(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_mu);
  g_host.push_back({host_class(bytes), p});
  if (static_cast<int>(g_host.size()) > kMaxHostCached) {
    cudaFreeHost(g_host.front().p);
    g_host.erase(g_host.begin());
  }
}

}  // namespace cpb
