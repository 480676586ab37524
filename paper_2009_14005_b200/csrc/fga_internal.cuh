// fga_internal.cuh -- shared device/host definitions for libfga (sm_100a).
//
// Data layout in HBM:
//   * template state (the swarm) is SoA fp64: pos[3][m], vel[3][m], mass[m],
//     permuted once into Morton order so a warp's 32 queries are spatial
//     neighbours (rigid motion preserves that locality for the whole run);
//   * the reference tree is stored twice: ascending preorder (the reference's
//     own numbering, bhtree.py:77, used for export/parity) and *mirrored*
//     preorder (children in descending slot order), which is exactly the
//     order the reference's stack traversal visits nodes (_kernels.py:44-48
//     pushes slots 0..7, so 7 pops first).  Traversal records:
//       NodeA32 {com.xyz, mass} float4  + NodeB32 {length^2 | -inf, skip}
//       NodeA64 {com.xyz, mass} double4 + NodeB64 {length^2 | -inf, skip}
//     skip = index just past the node's subtree, so a stackless traversal
//     that only ever moves forward reproduces the reference visit set.
#pragma once
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace fga {

constexpr int kMaxLevels = 21;  // 3 bits per level in a 64-bit key
constexpr int kMaxLevelsDeep = 42;  // ... in a 128-bit key (max_depth > 21 builds)
constexpr int kPartialStride = 18;  // doubles per warp partial (see PartialSlot)

// Slots of a per-warp (and, after reduction, per-iteration) partial record.
enum PartialSlot : int {
  kSumU = 0,      // sum (y - s)            [3]
  kSumW = 3,      // sum (y + d - s)        [3]
  kSumWU = 6,     // sum (y+d-s)_i (y-s)_j  [9], row-major i,j
  kAccepted = 15, // accepted node interactions (exact integer in a double)
  kVisits = 16,   // node visits
  kGpe = 17,      // sum_i m_y,i * sum_j m_x,j / (|y_i - x_j| + eps)
};

struct NodeB32 {
  float l2;  // length^2 as float, -inf for a leaf (always accepted)
  int skip;  // first node after this subtree (mirrored preorder)
};
struct NodeB64 {
  double l2;  // length*length exactly as the reference computes it; -inf leaf
  long long skip;
};

// Device-resident per-session iteration state (written by the update kernel).
struct IterState {
  double Rp[9], tp[3];      // pending step transform, applied at the start of the next pass
  double Racc[9], tacc[3];  // accumulated transform (registration.py:137-138)
  double shift[3];          // Kabsch shift s (= mean of the current positions)
  long long iter;           // completed iterations
  int done, converged;
  int gpe_pending;          // 1: the next reduced kGpe slot belongs to gpe_trace[iter-1]
  int pad;
};

struct SimParams {
  double G, eps, eps2, eta, dt, theta, theta2, conv_tol;
  long long max_iters;
  long long m_total;  // template size across all shards (Kabsch mean divisor)
  int trace_gpe;
  int dim;            // 2 or 3 (2-D clouds are carried as z = const)
  int count_visits;   // FP32 force pass counts node visits (fga_options.count_visits)
};

// ---------------------------------------------------------------- checks
// Device-side invariant checks (bounds of shared/global indices, the tree
// build's arrival counters), compiled in only for the FGA_CHECKS=1 test
// build (tools/build_variant.sh checks "-DFGA_CHECKS=1"): a failure traps, so
// the launch fails loudly (FGA_CHECKS=2 also prints the site).  compute-sanitizer is not
// available on this GPU pool; this build + tests/test_gpu_determinism.py are
// the race / out-of-bounds evidence (profiles/r02/README.md).
#ifndef FGA_CHECKS
#define FGA_CHECKS 0
#endif
#define FGA_CHECK(cond)                                                              \
  do {                                                                               \
    if (FGA_CHECKS && !(cond)) {                                                     \
      if (FGA_CHECKS > 1)                                                            \
        printf("FGA_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,  \
               __LINE__, (int)blockIdx.x, (int)threadIdx.x);                         \
      __trap();                                                                      \
    }                                                                                \
  } while (0)

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
const char* last_error();

#define FGA_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      ::fga::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_) + " at " + \
                       __FILE__ + ":" + std::to_string(__LINE__));                  \
      return FGA_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

// Grow-only device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n ? n : 16);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block reduction (kOp 0 sum, 1 min, 2 max); the result is valid
// on every thread.  Deterministic for a given blockDim.
template <int kOp>
__device__ __forceinline__ double op3(double a, double b) {
  return kOp == 0 ? a + b : (kOp == 1 ? fmin(a, b) : fmax(a, b));
}
template <int kOp>
__device__ double block_reduce(double v) {
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op3<kOp>(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();  // sh may still be read by a previous call
  if (lane == 0) sh[w] = v;
  __syncthreads();
  v = sh[0];
  for (int j = 1; j < nw; j++) v = op3<kOp>(v, sh[j]);
  return v;
}

}  // namespace fga
