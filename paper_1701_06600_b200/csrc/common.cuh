// Shared definitions for the B200 CPRAND kernels (sm_100a) and host runtime.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace cpb {

using i64 = std::int64_t;
using u64 = std::uint64_t;

constexpr int kMaxOrder = 8;  // tensor order supported by the device path
constexpr int kMaxRank = 128;      // R of the multi-kernel chain (RT buckets 16/32/64/128)
constexpr int kMaxFusedRank = 64;  // R of the persistent kernels and the sharded / mixing paths

// Error taxonomy of the C ABI (include/cprand_b200.h).
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
struct InvalidArgument : Error {
  explicit InvalidArgument(const std::string& m) : Error(2, m) {}
};
struct NumericalError : Error {
  explicit NumericalError(const std::string& m) : Error(3, m) {}
};
struct CudaError : Error {
  explicit CudaError(const std::string& m) : Error(4, m) {}
};
struct Unsupported : Error {
  explicit Unsupported(const std::string& m) : Error(5, m) {}
};

#define CPB_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::cpb::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_) + " (" + \
                             __FILE__ + ":" + std::to_string(__LINE__) + ")");          \
  } while (0)

#define CPB_LAUNCH_CHECK() CPB_CUDA(cudaGetLastError())

// Per-mode view handed to the fused gather/SKR/Gram/RHS kernel. Factor
// matrices live on the device ROW-major (I_m x R, ld = R) so one sampled
// factor row is R contiguous doubles.
struct ModeView {
  const double* x;           // tensor, generalized column-major
  i64 in;                    // I_n
  i64 stride;                // stride_n = prod_{m<n} I_m (elements)
  int s;                     // samples S
  int r;                     // rank R
  int kept;                  // N-1
  const int* rows[kMaxOrder];      // per kept mode c: S row indices (ascending mode order)
  const double* fac[kMaxOrder];    // per kept mode c: factor (row-major, ld R) used for Z
  const double* nrm[kMaxOrder];    // per kept mode c: column norms the factor is divided by (or null)
  const i64* base;                 // S base offsets sum_{k!=n} i_k stride_k
  // bounds for the device-check build (CPB_DEVICE_CHECKS; 0 = unknown)
  i64 xsize;                       // elements behind x (the tensor or a replica)
  i64 kdim[kMaxOrder];             // per kept mode c: rows of fac[c]
};

inline int ceil_div(i64 a, i64 b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace cpb
