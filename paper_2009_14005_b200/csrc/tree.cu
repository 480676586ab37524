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
// Children of a node in ascending preorder are x+1, skip[x+1], ... < skip[x]
// in slot order, so no child table is kept.  Node aggregates are reduced
// level by level from the depth cap up (children in slot order:
// deterministic), and each node's traversal records are written in the same
// pass, in *mirrored* preorder (see fga_internal.cuh).
//
// Kernels (all HBM/L2-bound integer + fp64 work; no tensor cores):
//   k_bbox_*        root bbox = per-axis min/max (bhtree.py:107-108)
//   k_keys          per-axis fp64 split recursion -> 3L-bit key (dyadic fast
//                   path with an exact-replay fallback near split planes)
//   (cub radix sort, stable: keeps the reference's within-leaf index order)
//   k_levels        c_i, per-point node counts, per-block per-level counts
//   (cub exclusive scan) -> preorder node offsets, node count
//   k_level_scan    per level: block offsets -> level-major (BFS) positions
//   k_emit          per node, in BFS order: start, occupancy, first child,
//                   mirrored index, bbox replay -> length (:83)
//   k_sum_level x (L+1)  mass, m*com bottom-up (:78-82) + mirrored records
#include <cub/cub.cuh>

#include "fga_internal.cuh"
#include "fga_tree.cuh"
#include "fga_device.cuh"
#include "../../include/fga.h"

#define TRY_RC(x)                 \
  do {                            \
    const int rc_ = (x);          \
    if (rc_ != FGA_OK) return rc_; \
  } while (0)

namespace fga {

namespace {

constexpr int kThreads = 256;
// points per block of k_levels / k_emit / k_export (they share the block
// mapping of the per-level block offsets; large blocks keep the scan short)
constexpr int kLT = 256;  // (1024 measured 5-11% slower: emit latency-bound)

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

// box[0..5] = lo, hi; box[6..8] = 2^L / (hi - lo) per axis; box[9] = the
// fast-key guard (see k_keys)
__global__ void k_bbox_final(const double* __restrict__ part, int nparts, int L,
                             double* __restrict__ out) {
  for (int k = 0; k < 6; k++) {
    double v = k < 3 ? INFINITY : -INFINITY;
    for (int j = threadIdx.x; j < nparts; j += blockDim.x)
      v = k < 3 ? fmin(v, part[j * 6 + k]) : fmax(v, part[j * 6 + k]);
    v = k < 3 ? block_reduce<1>(v) : block_reduce<2>(v);
    if (threadIdx.x == 0) out[k] = v;
  }
  if (threadIdx.x == 0) {
    double R = 0.0;
    for (int k = 0; k < 3; k++) {
      const double w = out[3 + k] - out[k];
      out[6 + k] = w > 0.0 ? ldexp(1.0, L) / w : 0.0;
      R = fmax(R, fmax(fabs(out[k]), fabs(out[3 + k])));
    }
    out[9] = 256.0 * 1.1102230246251565e-16 * R;  // 256 u R
  }
}

// ---------------------------------------------------------------- keys
// Keys = the per-axis fp64 midpoint recursion of the reference
// (bhtree.py:89-104): c = lo + (hi - lo)/2, bit = x >= c, 3 bits per level,
// x most significant.
//
// Fast path: every split plane the recursion produces is the exact dyadic
// plane lo0 + j (hi0 - lo0)/2^(l+1) up to accumulated rounding (<= ~4u R per
// level, R = max |box|), and the planes a point is tested against include
// the two finest-grid lines around it, the nearest planes of all.  So when
// f = (x - lo0) 2^L/(hi0 - lo0) is farther than a guard (256 u R, x units)
// from an integer, the recursion's bits are exactly floor(f).  Otherwise (a
// few points in 1e7, the top corner, flat axes) the recursion is replayed
// with __dadd_rn/__dmul_rn, so the result always equals the reference's.
__device__ __forceinline__ unsigned long long spread3(unsigned long long v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

__device__ __forceinline__ bool fast_axis(double x, double lo0, double scale, double gf, int L,
                                          unsigned long long& q) {
  if (!(scale > 0.0)) {  // flat axis (hi == lo, e.g. a 2-D cloud's z): every split is lo,
    if (x != lo0) return false;  // x >= lo at every level -> all ones
    q = (1ull << L) - 1ull;
    return true;
  }
  const double f = (x - lo0) * scale;
  const double fl = floor(f);
  const double fr = f - fl;
  if (!(fmin(fr, 1.0 - fr) > gf) || fl < 0.0 || fl >= ldexp(1.0, L)) return false;
  q = (unsigned long long)fl;
  return true;
}

__device__ __forceinline__ unsigned long long point_key(const double p[3],
                                                        const double* __restrict__ box, int L) {
  const double guard = box[9];
  unsigned long long q[3];
  bool fast = true;
#pragma unroll
  for (int k = 0; k < 3; k++)
    fast = fast_axis(p[k], box[k], box[6 + k], guard * box[6 + k], L, q[k]) && fast;
  if (fast) return (spread3(q[0]) << 2) | (spread3(q[1]) << 1) | spread3(q[2]);
  double lo[3], hi[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    lo[k] = box[k];
    hi[k] = box[3 + k];
  }
  unsigned long long key = 0;
  for (int l = 0; l < L; l++) {
    unsigned digit = 0;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const double c = __dadd_rn(lo[k], __dmul_rn(__dsub_rn(hi[k], lo[k]), 0.5));
      const bool up = p[k] >= c;
      digit = (digit << 1) | (up ? 1u : 0u);
      if (up) lo[k] = c; else hi[k] = c;
    }
    key = (key << 3) | digit;
  }
  return key;
}

// Key of every point in input order, the sort's index payload and the packed
// (x, y, z, m) record.  The sort runs on the top 32 key bits (keys32, 4 radix
// passes instead of 8); keys64 (the full key) is written only for the
// fallback full sort.
__global__ void k_keys(const double* __restrict__ pts, const double* __restrict__ masses, int64_t n,
                       const double* __restrict__ box, int L, int shift,
                       unsigned* __restrict__ keys32, unsigned long long* __restrict__ keys64,
                       int* __restrict__ idx, double4* __restrict__ packed) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3];
#pragma unroll
  for (int k = 0; k < 3; k++) p[k] = pts[i * 3 + k];
  packed[i] = make_double4(p[0], p[1], p[2], masses[i]);  // one 32 B record per point
  const unsigned long long key = point_key(p, box, L);
  if (keys64) keys64[i] = key;
  else keys32[i] = (unsigned)(key >> shift);
  idx[i] = (int)i;
}

// Sorted copy of the points (one random gather of the packed records) and,
// when the sort ran on the top key bits only, the full key recomputed from
// the point (no second gather).
__global__ void k_gather_sorted(const double4* __restrict__ packed, const int* __restrict__ idx,
                                int64_t n, const double* __restrict__ box, int L,
                                double4* __restrict__ sp, unsigned long long* __restrict__ keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 v = packed[idx[i]];
  sp[i] = v;
  if (keys) {
    const double p[3] = {v.x, v.y, v.z};
    keys[i] = point_key(p, box, L);
  }
}

// After the (stable) sort on the top 32 bits: every run of equal top bits is
// put in full-key order by one thread (stable insertion sort, so equal keys
// keep index order as the reference's partition does).  Runs longer than
// kRun set *overflow and the build falls back to the full 64-bit sort.
constexpr int kRun = 64;
__global__ void k_fixup_runs(const unsigned* __restrict__ hi, int64_t n,
                             unsigned long long* __restrict__ key, int* __restrict__ idx,
                             double4* __restrict__ sp, int* __restrict__ overflow) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned h = hi[i];
  if ((i > 0 && hi[i - 1] == h) || i + 1 >= n || hi[i + 1] != h) return;  // not a run head
  int len = 2;
  while (i + len < n && hi[i + len] == h)
    if (++len > kRun) {
      atomicOr(overflow, 1);
      return;
    }
  for (int a = 1; a < len; a++) {
    const unsigned long long kk = key[i + a];
    int b = a - 1;
    if (key[i + b] <= kk) continue;
    const int id = idx[i + a];
    const double4 v = sp[i + a];
    for (; b >= 0 && key[i + b] > kk; b--) {
      key[i + b + 1] = key[i + b];
      idx[i + b + 1] = idx[i + b];
      sp[i + b + 1] = sp[i + b];
    }
    key[i + b + 1] = kk;
    idx[i + b + 1] = id;
    sp[i + b + 1] = v;
  }
}

// Point i's chain of nodes: (i, l) for s <= l <= e, where s = c_i + 1 and
// e = max(s, min(L, c_{i+1} + 1)); none when s > L (a duplicate key).  The
// nodes below e are internal (they also hold point i+1, which shares c_{i+1}
// >= l levels) and (i, e) is always a leaf: it holds point i alone, or sits at
// the depth cap.
struct Chain {
  int s, e, cn;
};
__device__ __forceinline__ Chain chain_of(const signed char* __restrict__ clev, int64_t i,
                                          int64_t n, int L) {
  Chain c{L + 1, -1, -1};
  if (i < n) {
    c.cn = clev[i + 1];
    c.s = clev[i] + 1;
    if (c.s <= L) c.e = max(c.s, min(L, c.cn + 1));
  }
  return c;
}

// c_i for i in [0, N], the number of nodes each point starts, and per block
// of kLT points the number of nodes it starts at each level:
// bcount[l * nb + block] (all nodes) and bcount[(L + 1 + l) * nb + block]
// (internal nodes).
__global__ void __launch_bounds__(kLT) k_levels(const unsigned long long* __restrict__ keys,
                                                     int64_t n, int L,
                                                     signed char* __restrict__ clev,
                                                     int* __restrict__ count,
                                                     int* __restrict__ bcount) {
  __shared__ int hist[2 * (kMaxLevels + 1)];
  if (threadIdx.x < 2 * (kMaxLevels + 1)) hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i <= n) {
    const int c = (i == 0 || i == n) ? -1 : common_levels(keys[i - 1], keys[i], L);
    clev[i] = (signed char)c;
    int cnt = 0;
    if (i < n) {
      const int cn = (i + 1 == n) ? -1 : common_levels(keys[i], keys[i + 1], L);
      const int s = c + 1;
      if (s <= L) {
        const int e = max(s, min(L, cn + 1));
        cnt = e - s + 1;
        for (int l = s; l <= e; l++) atomicAdd(&hist[l], 1);
        for (int l = s; l < e; l++) atomicAdd(&hist[L + 1 + l], 1);
      }
    }
    count[i] = cnt;
  }
  __syncthreads();
  if (threadIdx.x < 2 * (L + 1))
    bcount[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = hist[threadIdx.x];
}

// Per row (one block each): exclusive scan of the block counts in place, the
// row total into row_total[row].
__global__ void __launch_bounds__(1024) k_level_scan(int* __restrict__ bcount, int nb,
                                                     int* __restrict__ row_total) {
  const int row = blockIdx.x;
  int* v = bcount + (int64_t)row * nb;
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int b0 = min(nb, (int)threadIdx.x * per), b1 = min(nb, b0 + per);
  int sum = 0;
  for (int b = b0; b < b1; b++) sum += v[b];
  __shared__ int sh[1024];
  sh[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // inclusive Hillis-Steele
    const int t = threadIdx.x >= (unsigned)o ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += t;
    __syncthreads();
  }
  int acc = sh[threadIdx.x] - sum;
  for (int b = b0; b < b1; b++) {
    const int t = v[b];
    v[b] = acc;
    acc += t;
  }
  if (threadIdx.x == blockDim.x - 1) row_total[row] = sh[threadIdx.x];
}

// lvl_off[l]: first BFS position of level l (lvl_off[L+1] = lvl_off[L+2] =
// node count); ilvl_off[l]: first slot of level l in the internal-node list.
__global__ void k_level_offsets(const int* __restrict__ row_total, int L, int* __restrict__ lvl_off,
                                int* __restrict__ ilvl_off) {
  if (threadIdx.x != 0) return;
  int a = 0, b = 0;
  for (int l = 0; l <= L; l++) {
    lvl_off[l] = a;
    ilvl_off[l] = b;
    a += row_total[l];
    b += row_total[L + 1 + l];
  }
  lvl_off[L + 1] = lvl_off[L + 2] = a;
  ilvl_off[L + 1] = b;
}

// first j in [from, n) with keys[j] > bound (keys sorted): galloping search
// from `from` (subtree ends are near the start for all but the top levels)
__device__ __forceinline__ int64_t upper_bound_gallop(const unsigned long long* keys, int64_t from,
                                                      int64_t n, unsigned long long bound) {
  int64_t lo = from, hi = n, step = 1;
  while (true) {
    const int64_t j = lo + step - 1;
    if (j >= n) break;
    if (keys[j] > bound) {
      hi = j;
      break;
    }
    lo = j + 1;
    step <<= 1;
  }
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] > bound) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// One bbox split step of the reference's recursion (bhtree.py:90-103) along
// the key digit of level `lev`.
__device__ __forceinline__ void bbox_step(unsigned long long key, int lev, int L, double lo[3],
                                          double hi[3]) {
  const unsigned digit = (unsigned)(key >> (3 * (L - lev))) & 7u;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const double c = __dadd_rn(lo[k], __dmul_rn(__dsub_rn(hi[k], lo[k]), 0.5));
    if ((digit >> (2 - k)) & 1u) lo[k] = c; else hi[k] = c;
  }
}

// numpy's pairwise 1-D sum (loops_utils.h.src) of the masses of sorted
// points [lo, lo + cnt); leaves hold one point except at the depth cap,
// where this makes the leaf mass bit-exact.
__device__ double pairwise_mass(const double4* __restrict__ sp, int64_t lo, int64_t cnt) {
  if (cnt < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < cnt; i++) r = __dadd_rn(r, sp[lo + i].w);
    return r;
  } else if (cnt <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; j++) r[j] = sp[lo + j].w;
    for (i = 8; i < cnt - (cnt % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], sp[lo + i + j].w);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < cnt; i++) res = __dadd_rn(res, sp[lo + i].w);
    return res;
  }
  int64_t n2 = cnt / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_mass(sp, lo, n2), pairwise_mass(sp, lo + n2, cnt - n2));
}

// Leaf aggregate (bhtree.py:78-82): pairwise mass, sequential sum of m*p.
__device__ __forceinline__ void leaf_sums(const double4* __restrict__ sp, int start, int occ,
                                          double& ms, double mc[3]) {
  ms = occ == 1 ? sp[start].w : pairwise_mass(sp, start, occ);
  mc[0] = mc[1] = mc[2] = 0.0;
  for (int q = 0; q < occ; q++) {
    const double4 v = sp[start + q];
    mc[0] = __dadd_rn(mc[0], __dmul_rn(v.x, v.w));
    mc[1] = __dadd_rn(mc[1], __dmul_rn(v.y, v.w));
    mc[2] = __dadd_rn(mc[2], __dmul_rn(v.z, v.w));
  }
}

// The node's traversal records at its mirrored-preorder index.
__device__ __forceinline__ void write_records(const TreeRecords& r, int mir, int rskip, bool leaf,
                                              double len, double ms, const double mc[3]) {
  const double cx = __ddiv_rn(mc[0], ms), cy = __ddiv_rn(mc[1], ms), cz = __ddiv_rn(mc[2], ms);
  const double l2 = __dmul_rn(len, len);
  r.a64[mir] = make_double4(cx, cy, cz, ms);
  r.b64[mir] = NodeB64{leaf ? -INFINITY : l2, (long long)rskip};
  r.a32[mir] = make_float4((float)cx, (float)cy, (float)cz, (float)ms);
  r.b32[mir] = NodeB32{leaf ? -INFINITY : (float)l2, rskip};
}


// Within-block ranks of the threads whose chains hold a node at level l
// (all nodes, and internal nodes only): warp ballots + warp prefix in shared
// memory.  Must be called by the whole block.
struct BlockRanks {
  unsigned bal[2][kMaxLevels + 1][kLT / 32];
  int pre[2][kMaxLevels + 1][kLT / 32];
};
__device__ __forceinline__ void block_ranks(BlockRanks& R, const Chain& c, int L) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int l = 0; l <= L; l++) {
    const unsigned ba = __ballot_sync(0xffffffffu, c.s <= l && l <= c.e);
    const unsigned bi = __ballot_sync(0xffffffffu, c.s <= l && l < c.e);
    if (lane == 0) {
      R.bal[0][l][w] = ba;
      R.pre[0][l][w] = __popc(ba);
      R.bal[1][l][w] = bi;
      R.pre[1][l][w] = __popc(bi);
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * (L + 1)) {
    const int k = threadIdx.x > L, l = threadIdx.x - k * (L + 1);
    int acc = 0;
    for (int q = 0; q < kLT / 32; q++) {
      const int v = R.pre[k][l][q];
      R.pre[k][l][q] = acc;
      acc += v;
    }
  }
  __syncthreads();
}
// slot of this thread's node at level l among all (k=0) / internal (k=1)
// level-l nodes: global offsets + block offset + warp prefix + lane rank
__device__ __forceinline__ int level_slot(const BlockRanks& R, int k, int l, int L,
                                          const int* __restrict__ off,
                                          const int* __restrict__ boff) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  return off[l] + boff[(int64_t)(k * (L + 1) + l) * gridDim.x + blockIdx.x] + R.pre[k][l][w] +
         __popc(R.bal[k][l][w] & ((1u << lane) - 1u));
}

// Internal node of the level lists (one 32-byte record).
struct InNode {
  int pos;    // BFS position (sums[] / sizep[] index)
  int fc;     // BFS position of the first child = the chain's next node
  int x;      // preorder index (bhtree.py:77)
  int pad;
  double len; // bbox diagonal (bhtree.py:83)
  double pad2;
};

// Per point i, the nodes (i, s_i..e_i), one level per loop turn for the
// whole block so that each level's writes are contiguous.  Node (i, l) has
// BFS position lvl_off[l] + (level-l nodes started before i): each level is
// contiguous and sorted by start, and the children of consecutive internal
// nodes are consecutive one level down.  Internal nodes go to the per-level
// list `in` (their subtree sizes are found bottom-up);
// the chain's leaf (i, e) is summarized here (bhtree.py:78-82) and writes its
// traversal records.  Preorder numbering from offset[]: x = offset[i] + l -
// s_i, skip = x + subtree size.  The bbox (for the length, :83) is replayed
// incrementally along the chain.  Same point->block mapping as k_levels.
__global__ void __launch_bounds__(kLT) k_emit(const unsigned long long* __restrict__ keys,
                                                   int64_t n, int L,
                                                   const signed char* __restrict__ clev,
                                                   const int* __restrict__ offset,
                                                   const int* __restrict__ boff,
                                                   const int* __restrict__ lvl_off,
                                                   const int* __restrict__ ilvl_off,
                                                   const double* __restrict__ box, int n_nodes,
                                                   const double4* __restrict__ sp,
                                                   InNode* __restrict__ in,
                                                   double4* __restrict__ sums,
                                                   int* __restrict__ sizep, TreeRecords r) {
  __shared__ BlockRanks R;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const Chain c = chain_of(clev, i, n, L);
  block_ranks(R, c, L);
  if (c.s > c.e) return;
  const unsigned long long k = keys[i];
  const int base = offset[i];
  double lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    lo[a] = box[a];
    hi[a] = box[3 + a];
  }
  double len = 0.0;
  int pos = 0;
  for (int l = 0; l <= c.e; l++) {
    if (l > 0) bbox_step(k, l, L, lo, hi);
    if (l < c.s) continue;
    double sq = 0.0;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const double ex = __dsub_rn(hi[a], lo[a]);
      sq = __dadd_rn(sq, __dmul_rn(ex, ex));
    }
    len = __dsqrt_rn(sq);
    pos = level_slot(R, 0, l, L, lvl_off, boff);
    if (l < c.e)
      in[level_slot(R, 1, l, L, ilvl_off, boff)] =
          InNode{pos, level_slot(R, 0, l + 1, L, lvl_off, boff), base + (l - c.s), 0, len, 0.0};
  }
  // the chain's leaf (i, e): point i alone, or a depth-cap cell of duplicates
  int64_t end;
  if (c.e > c.cn) end = i + 1;
  else if (c.e == 0) end = n;
  else end = upper_bound_gallop(keys, i + 1, n, k | low_mask(3 * (L - c.e)));
  double ms, mc[3];
  leaf_sums(sp, (int)i, (int)(end - i), ms, mc);
  sums[pos] = make_double4(ms, mc[0], mc[1], mc[2]);
  sizep[pos] = 1;
  const int x = base + (c.e - c.s);
  const int mir = c.e + n_nodes - (x + 1);  // skip = x + 1
  write_records(r, mir, mir + 1, true, len, ms, mc);
}

// Level l of the bottom-up summary (bhtree.py:77-83), levels L-1..0 in
// order, over the level's internal nodes: the children of internal node k are
// the BFS range [fc_k, fc_{k+1}) one level down (the last one's ends with the
// level), summed in slot order -- a fixed order, independent of scheduling.
// The node's traversal records are written here too, at its mirrored index.
// subtree size = 1 + the children's (preorder skip = x + size)
__device__ __forceinline__ void sum_internal(int l, int k, int e, int lend, int n_nodes,
                                             const InNode* __restrict__ in,
                                             double4* __restrict__ sums, int* __restrict__ sizep,
                                             const TreeRecords& r) {
  const InNode nd = in[k];
  const int cend = k + 1 < e ? in[k + 1].fc : lend;
  double ms = 0.0, mc[3] = {0.0, 0.0, 0.0};
  int size = 1;
  for (int ch = nd.fc; ch < cend; ch++) {
    const double4 v = sums[ch];
    ms = __dadd_rn(ms, v.x);
    mc[0] = __dadd_rn(mc[0], v.y);
    mc[1] = __dadd_rn(mc[1], v.z);
    mc[2] = __dadd_rn(mc[2], v.w);
    size += sizep[ch];
  }
  sums[nd.pos] = make_double4(ms, mc[0], mc[1], mc[2]);
  sizep[nd.pos] = size;
  const int mir = l + n_nodes - (nd.x + size);
  write_records(r, mir, mir + size, false, nd.len, ms, mc);
}

// one large level over the whole grid
__global__ void __launch_bounds__(256) k_sum_level(int l, const int* __restrict__ lvl_off,
                                                   const int* __restrict__ ilvl_off, int n_nodes,
                                                   const InNode* __restrict__ in,
                                                   double4* __restrict__ sums,
                                                   int* __restrict__ sizep, TreeRecords r) {
  const int b = ilvl_off[l], e = ilvl_off[l + 1], lend = lvl_off[l + 2];
  for (int k = b + blockIdx.x * blockDim.x + threadIdx.x; k < e; k += gridDim.x * blockDim.x)
    sum_internal(l, k, e, lend, n_nodes, in, sums, sizep, r);
}

// consecutive small levels l_hi..l_lo (descending) in one block
__global__ void __launch_bounds__(1024) k_sum_levels_small(int l_hi, int l_lo,
                                                           const int* __restrict__ lvl_off,
                                                           const int* __restrict__ ilvl_off,
                                                           int n_nodes,
                                                           const InNode* __restrict__ in,
                                                           double4* __restrict__ sums,
                                                           int* __restrict__ sizep,
                                                           TreeRecords r) {
  for (int l = l_hi; l >= l_lo; l--) {
    const int b = ilvl_off[l], e = ilvl_off[l + 1], lend = lvl_off[l + 2];
    for (int k = b + threadIdx.x; k < e; k += blockDim.x)
      sum_internal(l, k, e, lend, n_nodes, in, sums, sizep, r);
    __syncthreads();  // level l complete before its parents
  }
}

// first p in [0, to) with keys[p] >= bound, galloping backwards from `to`
__device__ __forceinline__ int64_t lower_bound_gallop(const unsigned long long* keys, int64_t to,
                                                      unsigned long long bound) {
  int64_t lo = 0, hi = to, step = 1;
  while (true) {
    const int64_t j = hi - step;
    if (j < 0) break;
    if (keys[j] < bound) {
      lo = j + 1;
      break;
    }
    hi = j;
    step <<= 1;
  }
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] >= bound) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// The reference's preorder arrays (bhtree.py:14-45), re-derived per chain
// node exactly as k_emit does; each node registers itself in its parent's
// child slot (parent: the chain's previous node, or found by a backwards
// search for the start of the parent's key prefix).  children must be -1
// filled.  Export only, not on the registration path.
__global__ void __launch_bounds__(kLT) k_export(const unsigned long long* __restrict__ keys,
                                                     int64_t n, int L,
                                                     const signed char* __restrict__ clev,
                                                     const int* __restrict__ offset,
                                                     const int* __restrict__ boff,
                                                     const int* __restrict__ lvl_off,
                                                     const double* __restrict__ box,
                                                     const double4* __restrict__ sums,
                                                     long long* children, double* com,
                                                     double* mass, double* length,
                                                     long long* occupancy, long long* depth,
                                                     double* bmin, double* bmax) {
  __shared__ BlockRanks R;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const Chain c = chain_of(clev, i, n, L);
  block_ranks(R, c, L);
  if (c.s > c.e) return;
  const unsigned long long k = keys[i];
  const int base = offset[i];
  double lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    lo[a] = box[a];
    hi[a] = box[3 + a];
  }
  for (int l = 0; l <= c.e; l++) {
    if (l > 0) bbox_step(k, l, L, lo, hi);
    if (l < c.s) continue;
    int64_t end;
    if (l == 0) end = n;
    else if (l > c.cn) end = i + 1;
    else end = upper_bound_gallop(keys, i + 1, n, k | low_mask(3 * (L - l)));
    const int64_t x = base + (l - c.s);
    const double4 v = sums[level_slot(R, 0, l, L, lvl_off, boff)];
    if (mass) mass[x] = v.x;
    if (com) {
      com[x * 3] = __ddiv_rn(v.y, v.x);
      com[x * 3 + 1] = __ddiv_rn(v.z, v.x);
      com[x * 3 + 2] = __ddiv_rn(v.w, v.x);
    }
    if (occupancy) occupancy[x] = end - i;
    if (depth) depth[x] = l;
    if (length) {
      double sq = 0.0;
      for (int a = 0; a < 3; a++) {
        const double ex = __dsub_rn(hi[a], lo[a]);
        sq = __dadd_rn(sq, __dmul_rn(ex, ex));
      }
      length[x] = __dsqrt_rn(sq);
    }
    for (int a = 0; a < 3; a++) {
      if (bmin) bmin[x * 3 + a] = lo[a];
      if (bmax) bmax[x * 3 + a] = hi[a];
    }
    if (children && l > 0) {
      int64_t parent;
      if (l > c.s) {
        parent = x - 1;
      } else {
        const int64_t p = lower_bound_gallop(keys, i, k & ~low_mask(3 * (L - l + 1)));
        parent = offset[p] + (l - 1 - ((int)clev[p] + 1));
      }
      const unsigned slot = (unsigned)(k >> (3 * (L - l))) & 7u;
      children[parent * 8 + slot] = x;
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
  FGA_CUDA_TRY(T.box.reserve(sizeof(double) * 10));
  k_bbox_partial<<<nb, kThreads, 0, st>>>(pts_dev, n, T.scratch.as<double>());
  k_bbox_final<<<1, 256, 0, st>>>(T.scratch.as<double>(), nb, L, T.box.as<double>());

  const int shift = std::max(0, 3 * L - 32);
  const int sort_bits = std::min(32, 3 * L);
  FGA_CUDA_TRY(T.keys.reserve(sizeof(unsigned long long) * n));
  FGA_CUDA_TRY(T.keys32_in.reserve(sizeof(unsigned) * n));
  FGA_CUDA_TRY(T.keys32.reserve(sizeof(unsigned) * n));
  FGA_CUDA_TRY(T.idx_in.reserve(sizeof(int) * n));
  FGA_CUDA_TRY(T.idx.reserve(sizeof(int) * n));
  FGA_CUDA_TRY(T.packed.reserve(sizeof(double4) * n));
  FGA_CUDA_TRY(T.sp.reserve(sizeof(double4) * n));
  FGA_CUDA_TRY(T.clev.reserve(n + 1));
  FGA_CUDA_TRY(T.count.reserve(sizeof(int) * (n + 1)));
  FGA_CUDA_TRY(T.offset.reserve(sizeof(int) * (n + 1)));
  const int nbl = blocks_for(n + 1, kLT);
  FGA_CUDA_TRY(T.bcount.reserve(sizeof(int) * (int64_t)2 * (L + 1) * nbl));
  FGA_CUDA_TRY(T.lvl.reserve(sizeof(int) * (kLvlInts + 1)));
  int* row_total = T.lvl.as<int>();
  int* lvl_off = row_total + 2 * (kMaxLevels + 1);
  int* ilvl_off = lvl_off + (kMaxLevels + 3);
  int* overflow = T.lvl.as<int>() + kLvlInts;
  {
    size_t b32 = 0, b64 = 0, bscan = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b32, T.keys32_in.as<unsigned>(), T.keys32.as<unsigned>(),
                                    T.idx_in.as<int>(), T.idx.as<int>(), (int)n, 0, sort_bits, st);
    cub::DeviceRadixSort::SortPairs(nullptr, b64, (const unsigned long long*)nullptr,
                                    (unsigned long long*)nullptr, T.idx_in.as<int>(),
                                    T.idx.as<int>(), (int)n, 0, 3 * L, st);
    cub::DeviceScan::ExclusiveSum(nullptr, bscan, (int*)nullptr, (int*)nullptr, (int)(n + 1), st);
    FGA_CUDA_TRY(T.cub_tmp.reserve(std::max(std::max(b32, b64), bscan)));
  }
  FGA_CUDA_TRY(cudaMemsetAsync(overflow, 0, sizeof(int), st));
  k_keys<<<blocks_for(n), kThreads, 0, st>>>(pts_dev, masses_dev, n, T.box.as<double>(), L, shift,
                                             T.keys32_in.as<unsigned>(), nullptr, T.idx_in.as<int>(),
                                             T.packed.as<double4>());
  size_t tmp_bytes = T.cub_tmp.bytes;
  FGA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(T.cub_tmp.p, tmp_bytes, T.keys32_in.as<unsigned>(),
                                               T.keys32.as<unsigned>(), T.idx_in.as<int>(),
                                               T.idx.as<int>(), (int)n, 0, sort_bits, st));
  k_gather_sorted<<<blocks_for(n), kThreads, 0, st>>>(T.packed.as<double4>(), T.idx.as<int>(), n,
                                                      T.box.as<double>(), L, T.sp.as<double4>(),
                                                      T.keys.as<unsigned long long>());
  if (shift > 0)
    k_fixup_runs<<<blocks_for(n), kThreads, 0, st>>>(T.keys32.as<unsigned>(), n,
                                                     T.keys.as<unsigned long long>(),
                                                     T.idx.as<int>(), T.sp.as<double4>(), overflow);
  // levels, per-level block counts, preorder offsets (rerun after a fallback)
  auto levels = [&]() -> int {
    k_levels<<<nbl, kLT, 0, st>>>(T.keys.as<unsigned long long>(), n, L,
                                       T.clev.as<signed char>(), T.count.as<int>(),
                                       T.bcount.as<int>());
    k_level_scan<<<2 * (L + 1), 1024, 0, st>>>(T.bcount.as<int>(), nbl, row_total);
    k_level_offsets<<<1, 32, 0, st>>>(row_total, L, lvl_off, ilvl_off);
    size_t sb = T.cub_tmp.bytes;
    FGA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(T.cub_tmp.p, sb, T.count.as<int>(),
                                               T.offset.as<int>(), (int)(n + 1), st));
    return FGA_OK;
  };
  TRY_RC(levels());
  // node count, per-level counts, run overflow and root box to the host
  // (one sync per build)
  int nn = 0;
  double box[6];
  int lvl_host[kLvlInts + 1];
  auto fetch = [&]() -> int {
    FGA_CUDA_TRY(cudaMemcpyAsync(&nn, T.offset.as<int>() + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    FGA_CUDA_TRY(cudaMemcpyAsync(box, T.box.p, sizeof(box), cudaMemcpyDeviceToHost, st));
    FGA_CUDA_TRY(cudaMemcpyAsync(lvl_host, T.lvl.p, sizeof(lvl_host), cudaMemcpyDeviceToHost, st));
    FGA_CUDA_TRY(cudaStreamSynchronize(st));
    return FGA_OK;
  };
  TRY_RC(fetch());
  if (lvl_host[kLvlInts]) {  // a long run of equal top bits: full 64-bit sort
    FGA_CUDA_TRY(T.keys_in.reserve(sizeof(unsigned long long) * n));
    k_keys<<<blocks_for(n), kThreads, 0, st>>>(pts_dev, masses_dev, n, T.box.as<double>(), L, 0,
                                               nullptr, T.keys_in.as<unsigned long long>(),
                                               T.idx_in.as<int>(), T.packed.as<double4>());
    tmp_bytes = T.cub_tmp.bytes;
    FGA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(
        T.cub_tmp.p, tmp_bytes, T.keys_in.as<unsigned long long>(), T.keys.as<unsigned long long>(),
        T.idx_in.as<int>(), T.idx.as<int>(), (int)n, 0, 3 * L, st));
    k_gather_sorted<<<blocks_for(n), kThreads, 0, st>>>(T.packed.as<double4>(), T.idx.as<int>(), n,
                                                        T.box.as<double>(), L, T.sp.as<double4>(),
                                                        nullptr);
    TRY_RC(levels());
    TRY_RC(fetch());
  }
  T.n_nodes = nn;
  T.cmag = 0.0;
  for (int k = 0; k < 6; k++) T.cmag = std::max(T.cmag, std::fabs(box[k]));
  for (int k = 0; k < 6; k++) T.box_host[k] = box[k];

  const int64_t nn64 = nn;
  FGA_CUDA_TRY(T.inodes.reserve(sizeof(InNode) * nn64));
  FGA_CUDA_TRY(T.sums.reserve(sizeof(double4) * nn64));
  FGA_CUDA_TRY(T.sizep.reserve(sizeof(int) * nn64));
  FGA_CUDA_TRY(T.a32.reserve(sizeof(float4) * nn64));
  FGA_CUDA_TRY(T.b32.reserve(sizeof(NodeB32) * nn64));
  FGA_CUDA_TRY(T.a64.reserve(sizeof(double4) * nn64));
  FGA_CUDA_TRY(T.b64.reserve(sizeof(NodeB64) * nn64));

  k_emit<<<nbl, kLT, 0, st>>>(T.keys.as<unsigned long long>(), n, L, T.clev.as<signed char>(),
                                   T.offset.as<int>(), T.bcount.as<int>(), lvl_off, ilvl_off,
                                   T.box.as<double>(), nn, T.sp.as<double4>(),
                                   T.inodes.as<InNode>(), T.sums.as<double4>(), T.sizep.as<int>(),
                                   T.records());
  // levels L-1..0 bottom-up (level L holds leaves only): a level with many
  // internal nodes gets its own grid; runs of small levels share one block
  const int* internal = lvl_host + (L + 1);  // row totals, internal nodes per level
  constexpr int kSmall = 2048;
  for (int l = L - 1; l >= 0;) {
    if (internal[l] > kSmall) {
      const int grid = (int)std::min<int64_t>(blocks_for(internal[l]), 148 * 8);
      k_sum_level<<<grid, 256, 0, st>>>(l, lvl_off, ilvl_off, nn, T.inodes.as<InNode>(),
                                        T.sums.as<double4>(), T.sizep.as<int>(), T.records());
      l--;
      continue;
    }
    int lo = l;
    while (lo - 1 >= 0 && internal[lo - 1] <= kSmall) lo--;
    k_sum_levels_small<<<1, 1024, 0, st>>>(l, lo, lvl_off, ilvl_off, nn, T.inodes.as<InNode>(),
                                           T.sums.as<double4>(), T.sizep.as<int>(), T.records());
    l = lo - 1;
  }
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
  if (children) FGA_CUDA_TRY(cudaMemsetAsync(d_children, 0xff, sizeof(long long) * 8 * nn, st));
  const int* lvl_off = T.lvl.as<int>() + 2 * (kMaxLevels + 1);
  k_export<<<blocks_for(T.n_points + 1, kLT), kLT, 0, st>>>(
      T.keys.as<unsigned long long>(), T.n_points, T.L, T.clev.as<signed char>(),
      T.offset.as<int>(), T.bcount.as<int>(), lvl_off, T.box.as<double>(), T.sums.as<double4>(),
      children ? d_children : nullptr, com ? d_com : nullptr, mass ? d_mass : nullptr,
      length ? d_len : nullptr, occupancy ? d_occ : nullptr, depth ? d_depth : nullptr,
      bmin ? d_bmin : nullptr, bmax ? d_bmax : nullptr);
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
