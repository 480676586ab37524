// tree.cu -- GPU build of the reference's Barnes-Hut 2^D tree (bhtree.py:56-122).
//
// The reference recursively splits a per-axis tight bounding box at its fp64
// midpoint (`center = bmin + (bmax - bmin) / 2.0`, bhtree.py:90; `>=` goes to
// the upper child, :93; slot bits with x as MSB, :94-96), numbering nodes in
// preorder (:77, :104).  Because every split only depends on the point's own
// coordinate along that axis, replaying the recursion per axis in fp64 gives
// each point an exact 3-bit-per-level key; quantized Morton codes do NOT
// reproduce the reference's splits.  From the sorted keys the
// whole topology has a closed form:
//   c_i   = levels shared by keys i-1 and i (c_0 = c_N = -1)
//   s_i   = c_i + 1          first level at which point i opens a segment
//   e_i   = min(L, c_{i+1}+1) deepest node that starts at point i
//   count = s_i > L ? 0 : max(1, e_i - s_i + 1)
//   preorder(i, l) = excl_scan(count)_i + (l - s_i)
// which is exactly the reference's preorder: (start, level) lexicographic.
// Node aggregates are reduced bottom-up (last-arriving child computes the
// parent, children in slot order: deterministic), then the traversal records
// are written in *mirrored* preorder (see fga_internal.cuh).
//
// Kernels (all HBM/L2-bound integer + fp64 work; no tensor cores):
//   k_bbox_*        root bbox = per-axis min/max (bhtree.py:107-108)
//   k_keys          exact per-axis fp64 split replay -> 3L-bit key
//   (cub radix sort, stable: keeps the reference's within-leaf index order)
//   k_levels        c_i and per-point node counts
//   (cub exclusive scan) -> node offsets, node count
//   k_emit          per node: level, start, occupancy, skip, parent, slot,
//                   children[parent][slot], bbox replay -> length (:83)
//   k_summarize     mass, m*com bottom-up (:78-82)
//   k_records       mirrored traversal records (fp32 and fp64)
#include <cub/cub.cuh>

#include "fga_internal.cuh"
#include "fga_tree.cuh"
#include "fga_device.cuh"
#include "../../include/fga.h"

namespace fga {

namespace {

constexpr int kThreads = 256;

inline int blocks_for(int64_t n, int t = kThreads) {
  int64_t b = (n + t - 1) / t;
  return (int)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------- bbox
__global__ void k_bbox_partial(const double* __restrict__ pts, int64_t n, double* __restrict__ part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; k++) {
      double v = pts[i * 3 + k];
      lo[k] = fmin(lo[k], v);
      hi[k] = fmax(hi[k], v);
    }
  }
  __shared__ double s[6][kThreads / 32];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  }
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
    for (int k = 0; k < 3; k++) {
      s[k][w] = lo[k];
      s[3 + k][w] = hi[k];
    }
  __syncthreads();
  if (threadIdx.x < 6) {
    double r = s[threadIdx.x][0];
    for (int j = 1; j < (int)(blockDim.x >> 5); j++)
      r = threadIdx.x < 3 ? fmin(r, s[threadIdx.x][j]) : fmax(r, s[threadIdx.x][j]);
    part[blockIdx.x * 6 + threadIdx.x] = r;
  }
}

__global__ void k_bbox_final(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  int k = threadIdx.x;
  if (k >= 6) return;
  double r = part[k];
  for (int j = 1; j < nparts; j++) r = k < 3 ? fmin(r, part[j * 6 + k]) : fmax(r, part[j * 6 + k]);
  out[k] = r;
}

// ---------------------------------------------------------------- keys
// Exact replay of the per-axis fp64 midpoint recursion.  __dadd_rn/__dmul_rn
// keep nvcc from contracting anything: (hi - lo) / 2.0 == (hi - lo) * 0.5
// exactly in binary floating point.
__global__ void k_keys(const double* __restrict__ pts, int64_t n, const double* __restrict__ box,
                       int L, unsigned long long* __restrict__ keys, int* __restrict__ idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3], lo[3], hi[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    p[k] = pts[i * 3 + k];
    lo[k] = box[k];
    hi[k] = box[3 + k];
  }
  unsigned long long key = 0;
  for (int l = 0; l < L; l++) {
    unsigned digit = 0;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      double c = __dadd_rn(lo[k], __dmul_rn(__dsub_rn(hi[k], lo[k]), 0.5));
      bool up = p[k] >= c;
      digit = (digit << 1) | (up ? 1u : 0u);
      if (up) lo[k] = c; else hi[k] = c;
    }
    key = (key << 3) | digit;
  }
  keys[i] = key;
  idx[i] = (int)i;
}

// c_i for i in [0, N] and the number of nodes each point starts.
__global__ void k_levels(const unsigned long long* __restrict__ keys, int64_t n, int L,
                         signed char* __restrict__ clev, int* __restrict__ count) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  int c = (i == 0 || i == n) ? -1 : common_levels(keys[i - 1], keys[i], L);
  clev[i] = (signed char)c;
  if (i == n) {
    count[i] = 0;
    return;
  }
  int cn = (i + 1 == n) ? -1 : common_levels(keys[i], keys[i + 1], L);
  int s = c + 1;
  int cnt = 0;
  if (s <= L) {
    int e = min(L, cn + 1);
    cnt = max(1, e - s + 1);
  }
  count[i] = cnt;
}

// first j in [lo, hi) with keys[j] > bound (keys sorted)
__device__ __forceinline__ int64_t upper_bound_key(const unsigned long long* keys, int64_t lo,
                                                   int64_t hi, unsigned long long bound) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] > bound) hi = mid; else lo = mid + 1;
  }
  return lo;
}
// first j in [lo, hi) with keys[j] >= bound
__device__ __forceinline__ int64_t lower_bound_key(const unsigned long long* keys, int64_t lo,
                                                   int64_t hi, unsigned long long bound) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] >= bound) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__global__ void k_emit(const unsigned long long* __restrict__ keys, int64_t n, int L,
                       const signed char* __restrict__ clev, const int* __restrict__ offset,
                       const double* __restrict__ box, TreeNodesView t) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int ci = clev[i], cn = clev[i + 1];
  const int s = ci + 1;
  if (s > L) return;  // exact duplicate of the previous key: no new node
  const int e = max(s, min(L, cn + 1));
  const int base = offset[i];
  const unsigned long long k = keys[i];
  for (int l = s; l <= e; l++) {
    const int node = base + (l - s);
    int64_t end;
    if (l == 0) end = n;
    else if (l > cn) end = i + 1;
    else end = upper_bound_key(keys, i + 1, n, k | low_mask(3 * (L - l)));
    const int occ = (int)(end - i);
    t.level[node] = (signed char)l;
    t.start[node] = (int)i;
    t.occ[node] = occ;
    t.skip[node] = offset[end];
    int parent = -1;
    if (l > s) {
      parent = node - 1;
    } else if (l > 0) {
      const unsigned long long pre = k & ~low_mask(3 * (L - l + 1));
      const int64_t p = lower_bound_key(keys, 0, i, pre);
      parent = offset[p] + (l - 1 - ((int)clev[p] + 1));
    }
    t.parent[node] = parent;
    if (parent >= 0) {
      const unsigned slot = (unsigned)(k >> (3 * (L - l))) & 7u;
      t.children[(int64_t)parent * 8 + slot] = node;
      atomicOr(&t.childmask[parent], 1u << slot);
    }
    double lo[3], hi[3];
    node_bbox(k, l, L, box, lo, hi);
    double sq = 0.0;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      double ex = __dsub_rn(hi[a], lo[a]);
      sq = __dadd_rn(sq, __dmul_rn(ex, ex));
    }
    t.length[node] = __dsqrt_rn(sq);
  }
}

// numpy's pairwise 1-D sum for n <= 128 (loops_utils.h.src); leaves hold one
// point except at the depth cap, where this makes the leaf mass bit-exact.
__device__ double pairwise_mass(const int* __restrict__ idx, int64_t lo, int64_t cnt,
                                const double* __restrict__ m) {
  if (cnt < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < cnt; i++) r = __dadd_rn(r, m[idx[lo + i]]);
    return r;
  } else if (cnt <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; j++) r[j] = m[idx[lo + j]];
    for (i = 8; i < cnt - (cnt % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], m[idx[lo + i + j]]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < cnt; i++) res = __dadd_rn(res, m[idx[lo + i]]);
    return res;
  }
  int64_t n2 = cnt / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_mass(idx, lo, n2, m), pairwise_mass(idx, lo + n2, cnt - n2, m));
}

// Leaves sum their points in the reference's order (bhtree.py:78-82); every
// internal node is reduced by the last of its children to finish (children in
// slot order), so the result does not depend on scheduling.
__global__ void k_summarize(TreeNodesView t, int64_t n_nodes, int L, const int* __restrict__ idx,
                            const double* __restrict__ pts, const double* __restrict__ masses) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n_nodes) return;
  const int occ = t.occ[x];
  if (!(occ == 1 || t.level[x] == L)) return;
  const int start = t.start[x];
  double ms = pairwise_mass(idx, start, occ, masses);
  double mc[3] = {0.0, 0.0, 0.0};
  for (int j = 0; j < occ; j++) {
    const int p = idx[start + j];
    const double w = masses[p];
#pragma unroll
    for (int k = 0; k < 3; k++) mc[k] = __dadd_rn(mc[k], __dmul_rn(pts[(int64_t)p * 3 + k], w));
  }
  t.mass[x] = ms;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    t.mc[x * 3 + k] = mc[k];
    t.com[x * 3 + k] = __ddiv_rn(mc[k], ms);
  }
  int node = (int)x;
  while (true) {
    const int par = t.parent[node];
    if (par < 0) break;
    __threadfence();
    const int nk = __popc(t.childmask[par]);
    if (atomicAdd(&t.arrive[par], 1) != nk - 1) break;
    __threadfence();
    double s = 0.0, c[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int slot = 0; slot < 8; slot++) {
      const int ch = __ldcg(&t.children[(int64_t)par * 8 + slot]);
      if (ch < 0) continue;
      s = __dadd_rn(s, __ldcg(&t.mass[ch]));
#pragma unroll
      for (int k = 0; k < 3; k++) c[k] = __dadd_rn(c[k], __ldcg(&t.mc[(int64_t)ch * 3 + k]));
    }
    t.mass[par] = s;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      t.mc[(int64_t)par * 3 + k] = c[k];
      t.com[(int64_t)par * 3 + k] = __ddiv_rn(c[k], s);
    }
    node = par;
  }
}

// Ascending preorder X -> mirrored preorder: mirror(X) = level + n - skip(X)
// (ancestors, then every larger-slot sibling subtree of X and its ancestors).
__global__ void k_records(TreeNodesView t, int64_t n_nodes, int L, TreeRecords r) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n_nodes) return;
  const int lev = t.level[x];
  const int skip = t.skip[x];
  const int mir = lev + (int)n_nodes - skip;
  const int size = skip - (int)x;
  const bool leaf = t.occ[x] == 1 || lev == L;
  const double cx = t.com[x * 3], cy = t.com[x * 3 + 1], cz = t.com[x * 3 + 2];
  const double ms = t.mass[x];
  const double len = t.length[x];
  const double l2 = __dmul_rn(len, len);
  r.a64[mir] = make_double4(cx, cy, cz, ms);
  r.b64[mir] = NodeB64{leaf ? -INFINITY : l2, (long long)(mir + size)};
  r.a32[mir] = make_float4((float)cx, (float)cy, (float)cz, (float)ms);
  r.b32[mir] = NodeB32{leaf ? -INFINITY : (float)l2, mir + size};
}

__global__ void k_export(TreeNodesView t, int64_t n_nodes, int L, const double* __restrict__ box,
                         const unsigned long long* __restrict__ keys, long long* children,
                         double* com, double* mass, double* length, long long* occupancy,
                         long long* depth, double* bmin, double* bmax) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n_nodes) return;
  if (children)
    for (int s = 0; s < 8; s++) children[x * 8 + s] = t.children[x * 8 + s];
  if (com)
    for (int k = 0; k < 3; k++) com[x * 3 + k] = t.com[x * 3 + k];
  if (mass) mass[x] = t.mass[x];
  if (length) length[x] = t.length[x];
  if (occupancy) occupancy[x] = t.occ[x];
  if (depth) depth[x] = t.level[x];
  if (bmin || bmax) {
    double lo[3], hi[3];
    node_bbox(keys[t.start[x]], t.level[x], L, box, lo, hi);
    for (int k = 0; k < 3; k++) {
      if (bmin) bmin[x * 3 + k] = lo[k];
      if (bmax) bmax[x * 3 + k] = hi[k];
    }
  }
}

}  // namespace

// ------------------------------------------------------------------ host side
int tree_build_dev(TreeDev& T, const double* pts_dev, const double* masses_dev, int64_t n, int L,
                   cudaStream_t st) {
  if (n <= 0) {
    set_error("tree build: empty cloud");
    return FGA_ERR_EMPTY;
  }
  if (n >= (1ll << 31) - 2) {
    set_error("tree build: more than 2^31 points");
    return FGA_ERR_UNSUPPORTED;
  }
  if (L < 1 || L > kMaxLevels) {
    set_error("tree build: max_depth must be in [1, 21] on the GPU path");
    return FGA_ERR_UNSUPPORTED;
  }
  T.n_points = n;
  T.L = L;
  T.pts = pts_dev;
  T.masses = masses_dev;
  const int nb = (int)std::min<int64_t>(blocks_for(n), 4 * 148);
  FGA_CUDA_TRY(T.scratch.reserve(sizeof(double) * 6 * (nb + 1)));
  FGA_CUDA_TRY(T.box.reserve(sizeof(double) * 6));
  k_bbox_partial<<<nb, kThreads, 0, st>>>(pts_dev, n, T.scratch.as<double>());
  k_bbox_final<<<1, 32, 0, st>>>(T.scratch.as<double>(), nb, T.box.as<double>());

  FGA_CUDA_TRY(T.keys_in.reserve(sizeof(unsigned long long) * n));
  FGA_CUDA_TRY(T.keys.reserve(sizeof(unsigned long long) * n));
  FGA_CUDA_TRY(T.idx_in.reserve(sizeof(int) * n));
  FGA_CUDA_TRY(T.idx.reserve(sizeof(int) * n));
  k_keys<<<blocks_for(n), kThreads, 0, st>>>(pts_dev, n, T.box.as<double>(), L,
                                             T.keys_in.as<unsigned long long>(), T.idx_in.as<int>());
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, T.keys_in.as<unsigned long long>(),
                                  T.keys.as<unsigned long long>(), T.idx_in.as<int>(),
                                  T.idx.as<int>(), (int)n, 0, 3 * L, st);
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int*)nullptr, (int*)nullptr, (int)(n + 1), st);
  FGA_CUDA_TRY(T.cub_tmp.reserve(std::max(tmp_bytes, scan_bytes)));
  FGA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(
      T.cub_tmp.p, tmp_bytes, T.keys_in.as<unsigned long long>(), T.keys.as<unsigned long long>(),
      T.idx_in.as<int>(), T.idx.as<int>(), (int)n, 0, 3 * L, st));

  FGA_CUDA_TRY(T.clev.reserve(n + 1));
  FGA_CUDA_TRY(T.count.reserve(sizeof(int) * (n + 1)));
  FGA_CUDA_TRY(T.offset.reserve(sizeof(int) * (n + 1)));
  k_levels<<<blocks_for(n + 1), kThreads, 0, st>>>(T.keys.as<unsigned long long>(), n, L,
                                                   T.clev.as<signed char>(), T.count.as<int>());
  scan_bytes = T.cub_tmp.bytes;
  FGA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(T.cub_tmp.p, scan_bytes, T.count.as<int>(),
                                             T.offset.as<int>(), (int)(n + 1), st));
  // node count and root box to the host (one sync per build)
  int nn = 0;
  double box[6];
  FGA_CUDA_TRY(cudaMemcpyAsync(&nn, T.offset.as<int>() + n, sizeof(int), cudaMemcpyDeviceToHost, st));
  FGA_CUDA_TRY(cudaMemcpyAsync(box, T.box.p, sizeof(box), cudaMemcpyDeviceToHost, st));
  FGA_CUDA_TRY(cudaStreamSynchronize(st));
  T.n_nodes = nn;
  T.cmag = 0.0;
  for (int k = 0; k < 6; k++) T.cmag = std::max(T.cmag, std::fabs(box[k]));
  for (int k = 0; k < 6; k++) T.box_host[k] = box[k];

  const int64_t nn64 = nn;
  FGA_CUDA_TRY(T.level.reserve(nn64));
  FGA_CUDA_TRY(T.start.reserve(sizeof(int) * nn64));
  FGA_CUDA_TRY(T.occ.reserve(sizeof(int) * nn64));
  FGA_CUDA_TRY(T.skip.reserve(sizeof(int) * nn64));
  FGA_CUDA_TRY(T.parent.reserve(sizeof(int) * nn64));
  FGA_CUDA_TRY(T.childmask.reserve(sizeof(unsigned) * nn64));
  FGA_CUDA_TRY(T.arrive.reserve(sizeof(int) * nn64));
  FGA_CUDA_TRY(T.children.reserve(sizeof(int) * 8 * nn64));
  FGA_CUDA_TRY(T.mass.reserve(sizeof(double) * nn64));
  FGA_CUDA_TRY(T.mc.reserve(sizeof(double) * 3 * nn64));
  FGA_CUDA_TRY(T.com.reserve(sizeof(double) * 3 * nn64));
  FGA_CUDA_TRY(T.length.reserve(sizeof(double) * nn64));
  FGA_CUDA_TRY(T.a32.reserve(sizeof(float4) * nn64));
  FGA_CUDA_TRY(T.b32.reserve(sizeof(NodeB32) * nn64));
  FGA_CUDA_TRY(T.a64.reserve(sizeof(double4) * nn64));
  FGA_CUDA_TRY(T.b64.reserve(sizeof(NodeB64) * nn64));
  FGA_CUDA_TRY(cudaMemsetAsync(T.children.p, 0xff, sizeof(int) * 8 * nn64, st));
  FGA_CUDA_TRY(cudaMemsetAsync(T.childmask.p, 0, sizeof(unsigned) * nn64, st));
  FGA_CUDA_TRY(cudaMemsetAsync(T.arrive.p, 0, sizeof(int) * nn64, st));

  TreeNodesView v = T.view();
  k_emit<<<blocks_for(n), kThreads, 0, st>>>(T.keys.as<unsigned long long>(), n, L,
                                             T.clev.as<signed char>(), T.offset.as<int>(),
                                             T.box.as<double>(), v);
  k_summarize<<<blocks_for(nn64), kThreads, 0, st>>>(v, nn64, L, T.idx.as<int>(), pts_dev,
                                                     masses_dev);
  k_records<<<blocks_for(nn64), kThreads, 0, st>>>(v, nn64, L, T.records());
  FGA_CUDA_TRY(cudaGetLastError());
  T.exportable = true;
  return FGA_OK;
}

int tree_export_host(TreeDev& T, cudaStream_t st, int64_t* children, double* com, double* mass,
                     double* length, int64_t* occupancy, int64_t* depth, double* bmin,
                     double* bmax) {
  if (!T.exportable || T.n_nodes <= 0) {
    set_error("tree export: no GPU-built tree in this context");
    return FGA_ERR_STATE;
  }
  const int64_t nn = T.n_nodes;
  DevBuf& b = T.export_buf;
  const size_t bytes = sizeof(double) * nn * (8 + 3 + 1 + 1 + 1 + 1 + 3 + 3);
  FGA_CUDA_TRY(b.reserve(bytes));
  char* p = b.as<char>();
  long long* d_children = (long long*)p; p += sizeof(long long) * 8 * nn;
  double* d_com = (double*)p; p += sizeof(double) * 3 * nn;
  double* d_mass = (double*)p; p += sizeof(double) * nn;
  double* d_len = (double*)p; p += sizeof(double) * nn;
  long long* d_occ = (long long*)p; p += sizeof(long long) * nn;
  long long* d_depth = (long long*)p; p += sizeof(long long) * nn;
  double* d_bmin = (double*)p; p += sizeof(double) * 3 * nn;
  double* d_bmax = (double*)p;
  k_export<<<blocks_for(nn), kThreads, 0, st>>>(T.view(), nn, T.L, T.box.as<double>(),
                                                T.keys.as<unsigned long long>(), d_children, d_com,
                                                d_mass, d_len, d_occ, d_depth, d_bmin, d_bmax);
  FGA_CUDA_TRY(cudaGetLastError());
#define CP(dst, src, cnt)                                                                 \
  if (dst) FGA_CUDA_TRY(cudaMemcpyAsync(dst, src, sizeof(double) * (cnt), cudaMemcpyDeviceToHost, st));
  CP(children, d_children, 8 * nn);
  CP(com, d_com, 3 * nn);
  CP(mass, d_mass, nn);
  CP(length, d_len, nn);
  CP(occupancy, d_occ, nn);
  CP(depth, d_depth, nn);
  CP(bmin, d_bmin, 3 * nn);
  CP(bmax, d_bmax, 3 * nn);
#undef CP
  FGA_CUDA_TRY(cudaStreamSynchronize(st));
  return FGA_OK;
}

// Load a reference-built BHTree (preorder arrays, bhtree.py:14-45).  The
// mirrored layout is derived on the host in O(n): skip pointers from the last
// present child, depth from the parents.
int tree_upload_host(TreeDev& T, const int64_t* children, const double* com, const double* mass,
                     const double* length, int64_t nn, int n_child, cudaStream_t st) {
  if (nn <= 0 || n_child != 8) {
    set_error("tree upload: need a non-empty 3-D tree (8 child slots)");
    return nn <= 0 ? FGA_ERR_EMPTY : FGA_ERR_UNSUPPORTED;
  }
  std::vector<int64_t> skip(nn), depth(nn, 0);
  for (int64_t x = 0; x < nn; x++)
    for (int c = 0; c < 8; c++) {
      int64_t ch = children[x * 8 + c];
      if (ch >= 0) {
        if (ch <= x || ch >= nn) {
          set_error("tree upload: nodes are not in preorder");
          return FGA_ERR_INVALID;
        }
        depth[ch] = depth[x] + 1;
      }
    }
  for (int64_t x = nn - 1; x >= 0; x--) {
    int64_t last = -1;
    for (int c = 0; c < 8; c++)
      if (children[x * 8 + c] >= 0) last = children[x * 8 + c];
    skip[x] = last < 0 ? x + 1 : skip[last];
  }
  std::vector<double4> a64(nn);
  std::vector<NodeB64> b64(nn);
  std::vector<float4> a32(nn);
  std::vector<NodeB32> b32(nn);
  double cmag = 0.0;
  for (int64_t x = 0; x < nn; x++) {
    bool leaf = true;
    for (int c = 0; c < 8; c++)
      if (children[x * 8 + c] >= 0) leaf = false;
    const int64_t mir = depth[x] + nn - skip[x];
    const int64_t size = skip[x] - x;
    const double l2 = length[x] * length[x];
    a64[mir] = make_double4(com[x * 3], com[x * 3 + 1], com[x * 3 + 2], mass[x]);
    b64[mir] = NodeB64{leaf ? -INFINITY : l2, (long long)(mir + size)};
    a32[mir] = make_float4((float)com[x * 3], (float)com[x * 3 + 1], (float)com[x * 3 + 2],
                           (float)mass[x]);
    b32[mir] = NodeB32{leaf ? -INFINITY : (float)l2, (int)(mir + size)};
    for (int k = 0; k < 3; k++) cmag = std::max(cmag, std::fabs(com[x * 3 + k]));
  }
  FGA_CUDA_TRY(T.a32.reserve(sizeof(float4) * nn));
  FGA_CUDA_TRY(T.b32.reserve(sizeof(NodeB32) * nn));
  FGA_CUDA_TRY(T.a64.reserve(sizeof(double4) * nn));
  FGA_CUDA_TRY(T.b64.reserve(sizeof(NodeB64) * nn));
  FGA_CUDA_TRY(cudaMemcpyAsync(T.a32.p, a32.data(), sizeof(float4) * nn, cudaMemcpyHostToDevice, st));
  FGA_CUDA_TRY(cudaMemcpyAsync(T.b32.p, b32.data(), sizeof(NodeB32) * nn, cudaMemcpyHostToDevice, st));
  FGA_CUDA_TRY(cudaMemcpyAsync(T.a64.p, a64.data(), sizeof(double4) * nn, cudaMemcpyHostToDevice, st));
  FGA_CUDA_TRY(cudaMemcpyAsync(T.b64.p, b64.data(), sizeof(NodeB64) * nn, cudaMemcpyHostToDevice, st));
  FGA_CUDA_TRY(cudaStreamSynchronize(st));
  T.n_nodes = nn;
  T.cmag = cmag;
  T.exportable = false;
  return FGA_OK;
}

}  // namespace fga
