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
//   k_gather_sorted sorted points + full keys; k_fixup_runs low key bits
//   k_count         c_i and per-point node counts
//   (cub exclusive scan) -> preorder offsets, node count
//   k_subtrees      per block of 512 sorted points: the chains top-down
//                   (bbox replay -> length, skip = offset[end]) and the
//                   aggregates bottom-up in shared memory; mirrored records
//   k_crossing      nodes that cross block boundaries: partials combined
#include <cub/cub.cuh>

#include <cstring>

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
__device__ __forceinline__ int chain_end(int s, int cn, int L) { return max(s, min(L, cn + 1)); }

// c_i for i in [0, N] (c_0 = c_N = -1) and the number of nodes each point
// starts (count[N] = 0, so the exclusive scan's last entry is the node count).
__global__ void k_count(const unsigned long long* __restrict__ keys, int64_t n, int L,
                        signed char* __restrict__ clev, int* __restrict__ count) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  const int c = (i == 0 || i == n) ? -1 : common_levels(keys[i - 1], keys[i], L);
  clev[i] = (signed char)c;
  int cnt = 0;
  if (i < n) {
    const int cn = (i + 1 == n) ? -1 : common_levels(keys[i], keys[i + 1], L);
    const int s = c + 1;
    if (s <= L) cnt = chain_end(s, cn, L) - s + 1;
  }
  count[i] = cnt;
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

__device__ __forceinline__ double diag_len(const double lo[3], const double hi[3]) {
  double sq = 0.0;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const double ex = __dsub_rn(hi[a], lo[a]);
    sq = __dadd_rn(sq, __dmul_rn(ex, ex));
  }
  return __dsqrt_rn(sq);  // np.linalg.norm (bhtree.py:83)
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

// Leaf aggregate (bhtree.py:78-82): pairwise mass, sequential sum of m*p, as
// {m, m x, m y, m z}.
__device__ __forceinline__ double4 leaf_sums(const double4* __restrict__ sp, int64_t start,
                                             int64_t occ) {
  double4 r;
  r.x = occ == 1 ? sp[start].w : pairwise_mass(sp, start, occ);
  r.y = r.z = r.w = 0.0;
  for (int64_t q = 0; q < occ; q++) {
    const double4 v = sp[start + q];
    r.y = __dadd_rn(r.y, __dmul_rn(v.x, v.w));
    r.z = __dadd_rn(r.z, __dmul_rn(v.y, v.w));
    r.w = __dadd_rn(r.w, __dmul_rn(v.z, v.w));
  }
  return r;
}

__device__ __forceinline__ void add4(double4& a, const double4& b) {
  a.x = __dadd_rn(a.x, b.x);
  a.y = __dadd_rn(a.y, b.y);
  a.z = __dadd_rn(a.z, b.z);
  a.w = __dadd_rn(a.w, b.w);
}

// The node's traversal records at its mirrored-preorder index, in two halves:
// the structural one ({l^2, skip}, known top-down) and the aggregate one
// ({com, mass}, known bottom-up).
__device__ __forceinline__ void write_records_b(const TreeRecords& r, int mir, int rskip, bool leaf,
                                                double len) {
  const double l2 = __dmul_rn(len, len);
  r.b64[mir] = NodeB64{leaf ? -INFINITY : l2, (long long)rskip};
  const float l2f = leaf ? -INFINITY : (float)l2;
  r.c32[2 * mir + 1] = make_float4(l2f, __int_as_float(rskip), 0.f, l2f);
}
__device__ __forceinline__ void write_records_a(const TreeRecords& r, int mir, const double4& v) {
  const double cx = __ddiv_rn(v.y, v.x), cy = __ddiv_rn(v.z, v.x), cz = __ddiv_rn(v.w, v.x);
  r.a64[mir] = make_double4(cx, cy, cz, v.x);
  r.c32[2 * mir] = make_float4((float)cx, (float)cy, (float)cz, (float)v.x);
}

// ---------------------------------------------------------------- hierarchy
// Node (i, l) holds the sorted points [i, end), end = first j > i with
// c_j < l, and its preorder subtree is the chain rest of i plus every chain
// of the points in (i, end); so its preorder skip is offset[end] and its
// mirrored index is l + n_nodes - offset[end] -- no bottom-up size pass.
//
// The aggregates (mass, m*p) are reduced bottom-up inside blocks of kST
// consecutive sorted points (k_subtrees): a node is summed over its children
// in slot order, starting from 0.0.  A node that crosses block boundaries gets
// one partial per block it touches (the same fold over its children inside
// that block, a crossing child contributing its own partial); k_crossing adds
// them in a fixed dyadic shape.  Every result is a fixed function of the input
// (kST is a constant), whatever the scheduling.
#ifndef FGA_KST
#define FGA_KST 128
#endif
constexpr int kST = FGA_KST;
constexpr int kSW = kST / 32;
#ifndef FGA_STB
#define FGA_STB (1536 / kST)
#endif
constexpr int kSTBlocks = FGA_STB;  // resident blocks per SM (40 registers at 128 threads; 12 measured 2% faster than 10 and 8% than 8)

// Per (level, block) boundary partials, SoA by level (index l * nb + b):
//   pr/prx/prlen: the node owned by block b (starting in it) that runs past
//                 its end, if any (prx = preorder index, -1 = none)
//   pl/plend:     the node that starts before block b and covers its first
//                 point, and where it ends inside b (-1 = past the block)
//   mn[b]:        min c_j over the block's points 1..kST (the next block's
//                 first point included): a level-l node covering the block's
//                 first point ends inside it iff mn[b] < l
// plus the dyadic sums / minima over aligned runs of 2^k blocks (k >= 1):
//   hs[l * hn + ho[k] + j] = hs_{k-1}[2j] + hs_{k-1}[2j+1] (hs_0 = pl),
//   hm[ho[k] + j] = min of the same runs of mn.
constexpr int kMaxHier = 32;
struct Cross {
  double4* pr;
  double4* pl;
  double* prlen;
  int* prx;
  int* plend;
  int* mn;
  double4* hs;
  int* hm;
  int hn;  // entries per level in hs (sum of the dyadic level sizes)
  int K;   // dyadic levels: 2^K >= nb
  int ho[kMaxHier + 1];
};

// first set bit at a position > j of a kST-bit mask (nz: its non-zero words);
// kST when none
__device__ __forceinline__ int next_bit(const unsigned* __restrict__ m, unsigned nz, int j) {
  const int wd = (j + 1) >> 5;
  if (wd >= kSW) return kST;
  const unsigned v = m[wd] & (~0u << ((j + 1) & 31));
  if (v) return (wd << 5) + __ffs(v) - 1;
  const unsigned z = nz & (~0u << (wd + 1));
  if (!z) return kST;
  const int w2 = __ffs(z) - 1;
  return (w2 << 5) + __ffs(m[w2]) - 1;
}

// last set bit at a position <= j of a kST-bit mask (nz: its non-zero words);
// the caller guarantees one exists
__device__ __forceinline__ int prev_bit_incl(const unsigned* __restrict__ m, unsigned nz, int j) {
  const int wd = j >> 5;
  const unsigned v = m[wd] & (0xffffffffu >> (31 - (j & 31)));
  if (v) return (wd << 5) + 31 - __clz(v);
  const int w2 = 31 - __clz(nz & ((1u << wd) - 1u));
  return (w2 << 5) + 31 - __clz(m[w2]);
}

// number of set bits at positions [a, b) of a kST-bit mask
__device__ __forceinline__ int count_bits(const unsigned* __restrict__ m, int a, int b) {
  if (a >= b) return 0;
  const int wa = a >> 5, wb = (b - 1) >> 5;
  const unsigned lo = ~0u << (a & 31), hi = 0xffffffffu >> (31 - ((b - 1) & 31));
  if (wa == wb) return __popc(m[wa] & lo & hi);
  int c = __popc(m[wa] & lo) + __popc(m[wb] & hi);
  for (int q = wa + 1; q < wb; q++) c += __popc(m[q]);
  return c;
}

// One block = kST sorted points, one thread each.  Per level l, bit masks
// over the block's points: B_l (c_j < l: a node at level <= l starts at j, so
// it ends every level-l range) and H_l (a level-l node starts at j, or j = 0
// and the level-l node covering it started earlier -- the "pseudo head").
// All the block's points share the levels <= lca (the common levels of its
// first and last key), so above lca only position 0 has nodes, one child each.
//   leaves: every thread sums its chain's leaf (bhtree.py:78-82);
//   top-down, one node per thread: bbox replay from the shared level-lca box
//     (bhtree.py:90-103) -> length, skip = offset[end] -> structural record;
//   bottom-up, no barriers: each thread climbs from its leaf; a node's
//     children report to a per-(level, head) counter and the last one to
//     arrive folds them in slot order (starting from 0.0) and climbs on.
__global__ void __launch_bounds__(kST, kSTBlocks) k_subtrees(const unsigned long long* __restrict__ keys,
                                                     int64_t n, int L,
                                                     const signed char* __restrict__ clev,
                                                     const int* __restrict__ offset,
                                                     const double* __restrict__ box,
                                                     const double4* __restrict__ sp,
                                                     TreeRecords r, Cross cr, int nb) {
  __shared__ unsigned mB[kMaxLevels + 2][kSW], mH[kMaxLevels + 2][kSW];
  __shared__ unsigned nzB[kMaxLevels + 2], nzH[kMaxLevels + 2];
  __shared__ unsigned arrived[kMaxLevels + 1][kST / 4];
  __shared__ int offs[kST + 1];
  __shared__ signed char cs[kST + 1];
  __shared__ unsigned long long skey[kST];
  __shared__ double4 V[kST];
  __shared__ double pbox[6];
  __shared__ int s_maxe, s_mn, s_q;
  constexpr int kMap = 4 * kST;  // node -> point map of the top-down pass
  __shared__ short nmap[kMap];
  __shared__ double4 qv[kST];  // queued aggregate records of the climb
  __shared__ int qmir[kST];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5, b = blockIdx.x;
  const int64_t B0 = (int64_t)b * kST, i = B0 + t;
  const int64_t last = min(B0 + kST, n) - 1;
  const int nn = offset[n];
  cs[t] = i <= n ? clev[i] : (signed char)-1;
  offs[t] = i <= n ? offset[i] : nn;
  skey[t] = i < n ? keys[i] : 0ull;
  if (t == 0) {
    const int64_t j = B0 + kST;
    cs[kST] = j <= n ? clev[j] : (signed char)-1;
    offs[kST] = j <= n ? offset[j] : nn;
    s_maxe = -1;
    s_mn = kMaxLevels + 1;
    s_q = 0;
  }
  if (t <= L) cr.prx[t * nb + b] = -1;
  __syncthreads();
  const unsigned long long k0 = skey[0];
  const int lca = last > B0 ? common_levels(k0, skey[last - B0], L) : L;
  const int c = cs[t], c0 = cs[0], cend = cs[kST];
  const bool has = i < n && c + 1 <= L;
  const int s = c + 1, e = has ? chain_end(s, cs[t + 1], L) : -1;
  if (has) atomicMax(&s_maxe, e);
  if (t > 0) atomicMin(&s_mn, c);
  if (t == kST - 1) {
    atomicMin(&s_mn, cend);
    // the box of the level-lca node holding every point of the block
    double lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      lo[a] = box[a];
      hi[a] = box[3 + a];
    }
    for (int l = 1; l <= lca; l++) bbox_step(k0, l, L, lo, hi);
#pragma unroll
    for (int a = 0; a < 3; a++) {
      pbox[a] = lo[a];
      pbox[3 + a] = hi[a];
    }
  }
  // leaf sums (bhtree.py:78-82) and the leaf's aggregate record
  double4 leafv = make_double4(0.0, 0.0, 0.0, 0.0);
  if (has) {
    int64_t end;  // point i alone, or a depth-cap cell of duplicates
    if (e > cs[t + 1]) end = i + 1;
    else if (e == 0) end = n;
    else end = upper_bound_gallop(keys, i + 1, n, skey[t] | low_mask(3 * (L - e)));
    leafv = leaf_sums(sp, i, end - i);
    write_records_a(r, e + nn - (offs[t] + (e - s) + 1), leafv);
    const int x0 = offs[t] - offs[0];
    if (x0 + (e - s) < kMap)
      for (int q = 0; q <= e - s; q++) nmap[x0 + q] = (short)t;
  }
  V[t] = leafv;
  __syncthreads();
  const int top = s_maxe;
  const int mtop = max(top, min(c0, L));  // deepest level with a head
  for (int l = lca; l <= mtop; l++) {
    const bool ph = t == 0 && l <= c0;
    const unsigned bb = __ballot_sync(0xffffffffu, c < l);
    const unsigned bh = __ballot_sync(0xffffffffu, (has && s <= l && l <= e) || ph);
    if (lane == 0) {
      mB[l][w] = bb;
      mH[l][w] = bh;
    }
  }
  if (t < kST / 4)
    for (int l = lca; l < mtop; l++) arrived[l][t] = 0u;
  __syncthreads();
  if (t >= lca && t <= mtop) {  // per level: non-zero word summaries
    unsigned zb = 0, zh = 0;
    for (int q = 0; q < kSW; q++) {
      zb |= (mB[t][q] != 0u ? 1u : 0u) << q;
      zh |= (mH[t][q] != 0u ? 1u : 0u) << q;
    }
    nzB[t] = zb;
    nzH[t] = zh;
  }
  __syncthreads();
  if (t == 0) cr.mn[b] = s_mn;

  // top-down, one node per thread (the block's nodes are the preorder range
  // [offs[0], offs[kST])); a node that runs past the block leaves its length
  // and preorder index to k_crossing
  {
    const int offs0 = offs[0], nbn = offs[kST] - offs0;
    for (int kk = t; kk < nbn; kk += kST) {
      const int x = offs0 + kk;
      int j;  // the point whose chain holds node x
      if (nbn <= kMap) {
        j = nmap[kk];
      } else {
        int lo_ = 0, hi_ = kST;
        while (hi_ - lo_ > 1) {
          const int mid = (lo_ + hi_) >> 1;
          if (offs[mid] <= x) lo_ = mid; else hi_ = mid;
        }
        j = lo_;
      }
      const int sj = cs[j] + 1, ej = chain_end(sj, cs[j + 1], L);
      const int l = sj + (x - offs[j]);
      const unsigned long long key = skey[j];
      double bl[3], bh[3];
      int lv;
      if (l <= lca) {  // (position 0 only: the other points start below lca)
        lv = 0;
#pragma unroll
        for (int a = 0; a < 3; a++) {
          bl[a] = box[a];
          bh[a] = box[3 + a];
        }
      } else {
        lv = lca;
#pragma unroll
        for (int a = 0; a < 3; a++) {
          bl[a] = pbox[a];
          bh[a] = pbox[3 + a];
        }
      }
      while (lv < l) bbox_step(key, ++lv, L, bl, bh);
      const double len = diag_len(bl, bh);
      FGA_CHECK(j >= 0 && j < kST && l >= sj && l <= ej && x >= offs[j] && x < offs[j + 1]);
      if (l == ej) {
        const int mir = l + nn - (x + 1);
        FGA_CHECK(mir >= 0 && mir < nn);
        write_records_b(r, mir, mir + 1, true, len);
      } else {
        const int p = l <= lca ? kST : next_bit(mB[l], nzB[l], j);
        if (p < kST || cend < l) {
          const int skipp = offs[p];
          const int mir = l + nn - skipp;
          write_records_b(r, mir, mir + (skipp - x), false, len);
        } else {
          cr.prx[l * nb + b] = x;
          cr.prlen[l * nb + b] = len;
        }
      }
    }
  }

  // bottom-up.  A climb starts at every leaf: the thread's own, and at
  // position 0 the depth-cap duplicate run owned by an earlier block (its
  // value here is 0).
  int pos = t, lev = has ? e : (t == 0 && c0 == L ? L : -1);
  double4 v = leafv;
  bool up = lev >= 0;
  while (up && lev > lca) {
    const int pl = lev - 1;
    const int hp = prev_bit_incl(mH[pl], nzH[pl], pos);  // the parent's head
    const int pend = next_bit(mB[pl], nzB[pl], hp);       // ... and range end
    const int nch = count_bits(mH[lev], hp, pend);
    __threadfence_block();  // this child's V before the arrival
    const unsigned sh = 8u * (hp & 3);  // byte counters, four per word
    FGA_CHECK(hp >= 0 && hp < kST && pend > hp && pend <= kST && nch >= 1 && nch <= 8);
    const unsigned old_ = atomicAdd(&arrived[pl][hp >> 2], 1u << sh);
    FGA_CHECK((int)((old_ >> sh) & 0xffu) < nch);  // never more arrivals than children
    if ((int)((old_ >> sh) & 0xffu) != nch - 1) {
      up = false;
      break;
    }
    __threadfence_block();  // every child's V after it
    v = make_double4(0.0, 0.0, 0.0, 0.0);
    {  // children: the H_lev bits in [hp, pend), in slot order
      const unsigned* mh = mH[lev];
      int wd = hp >> 5;
      unsigned m = mh[wd] & (~0u << (hp & 31));
      while (true) {
        while (m) {
          const int q = (wd << 5) + __ffs(m) - 1;
          if (q >= pend) break;
          add4(v, V[q]);
          m &= m - 1u;
        }
        if (++wd >= kSW || (wd << 5) >= pend) break;
        m = mh[wd];
      }
    }
    V[hp] = v;
    const bool local = pend < kST || cend < pl;
    if (hp == 0 && pl <= c0) {
      cr.pl[pl * nb + b] = v;
      cr.plend[pl * nb + b] = local ? pend : -1;
    } else if (local) {  // queued: the divisions run compacted after the climb
      const int slot = atomicAdd(&s_q, 1);
      FGA_CHECK(pl + nn - offs[pend] >= 0 && pl + nn - offs[pend] < nn);
      if (slot < kST) {
        qv[slot] = v;
        qmir[slot] = pl + nn - offs[pend];
      } else {
        write_records_a(r, pl + nn - offs[pend], v);
      }
    } else {
      cr.pr[pl * nb + b] = v;
    }
    pos = hp;
    lev = pl;
  }
  if (up) {  // this thread holds position 0's node at level lev <= lca; each
             // level above has one node there (pseudo up to c0, then the
             // chain of point 0), with one child
    for (int l = lev - 1; l >= 0; l--) {
      v = make_double4(__dadd_rn(0.0, v.x), __dadd_rn(0.0, v.y), __dadd_rn(0.0, v.z),
                       __dadd_rn(0.0, v.w));  // the one-child fold
      const bool local = cend < l;
      if (l <= c0) {
        cr.pl[l * nb + b] = v;
        cr.plend[l * nb + b] = local ? (int)(n - B0 < kST ? n - B0 : (int64_t)kST) : -1;  // (the last block ends at n)
      } else if (local) {
        write_records_a(r, l + nn - offs[kST], v);
      } else {
        cr.pr[l * nb + b] = v;
      }
    }
  }
  __syncthreads();
  const int nq = min(s_q, kST);
  for (int k = t; k < nq; k += kST) write_records_a(r, qmir[k], qv[k]);
}

// Dyadic sums (per level) and minima over aligned runs of 2^k blocks, fixed
// shape: hs_k[j] = hs_{k-1}[2j] + hs_{k-1}[2j+1].  One launch builds levels
// k0+1..k0+5 from level k0: each warp takes 32 consecutive level-k0 entries
// and pairs them up through shuffles (blockIdx.y = tree level, L + 1 = the
// minima).
__global__ void __launch_bounds__(256) k_hier(int L, int nb, int k0, Cross cr) {
  const int l = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int sz0 = (nb + (1 << k0) - 1) >> k0;
  if (j - lane >= sz0) return;  // (whole warps only)
  if (l <= L) {
    const double4* src = k0 == 0 ? cr.pl + (int64_t)l * nb : cr.hs + (int64_t)l * cr.hn + cr.ho[k0];
    double4 v = j < sz0 ? src[j] : make_double4(0.0, 0.0, 0.0, 0.0);
    for (int d = 1; d <= 5 && k0 + d <= cr.K; d++) {
      double4 y;
      y.x = __shfl_down_sync(0xffffffffu, v.x, 1 << (d - 1));
      y.y = __shfl_down_sync(0xffffffffu, v.y, 1 << (d - 1));
      y.z = __shfl_down_sync(0xffffffffu, v.z, 1 << (d - 1));
      y.w = __shfl_down_sync(0xffffffffu, v.w, 1 << (d - 1));
      const int szd = (nb + (1 << (k0 + d)) - 1) >> (k0 + d);
      const int jd = j >> d;
      if ((lane & ((1 << d) - 1)) == 0) {
        if (((j >> (d - 1)) + 1) < ((nb + (1 << (k0 + d - 1)) - 1) >> (k0 + d - 1))) add4(v, y);
        if (jd < szd) cr.hs[(int64_t)l * cr.hn + cr.ho[k0 + d] + jd] = v;
      }
    }
  } else {
    const int* src = k0 == 0 ? cr.mn : cr.hm + cr.ho[k0];
    int v = j < sz0 ? src[j] : -1;
    for (int d = 1; d <= 5 && k0 + d <= cr.K; d++) {
      const int y = __shfl_down_sync(0xffffffffu, v, 1 << (d - 1));
      const int szd = (nb + (1 << (k0 + d)) - 1) >> (k0 + d);
      const int jd = j >> d;
      if ((lane & ((1 << d) - 1)) == 0) {
        if (((j >> (d - 1)) + 1) < ((nb + (1 << (k0 + d - 1)) - 1) >> (k0 + d - 1))) v = min(v, y);
        if (jd < szd) cr.hm[cr.ho[k0 + d] + jd] = v;
      }
    }
  }
}

__device__ __forceinline__ int hier_min(const Cross& cr, int k, int j) {
  return k == 0 ? cr.mn[j] : cr.hm[cr.ho[k] + j];
}

// One thread per (level, block) with an owned crossing node: the block where
// it ends (first later block with mn < l, by the dyadic minima), its partials
// over the blocks after its own (the canonical dyadic cover, left to right),
// and its records.
__global__ void __launch_bounds__(256) k_crossing(int L, int nb, int64_t n,
                                                  const int* __restrict__ offset, Cross cr,
                                                  TreeRecords r) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= (int64_t)(L + 1) * nb) return;
  const int l = (int)(g / nb), b = (int)(g % nb);
  const int x = cr.prx[l * nb + b];
  if (x < 0) return;
  // end block: first bb > b with mn[bb] < l
  int p = b + 1, k = 0;
  while (true) {
    while (k < cr.K && (p & ((2 << k) - 1)) == 0 && hier_min(cr, k + 1, p >> (k + 1)) >= l) k++;
    if (hier_min(cr, k, p >> k) >= l) {
      p += 1 << k;
      continue;
    }
    break;
  }
  while (k > 0) {
    k--;
    if (hier_min(cr, k, p >> k) >= l) p += 1 << k;
  }
  const int bend = p;
  double4 v = cr.pr[l * nb + b];
  for (int q = b + 1; q <= bend;) {
    int kk = min(__ffs(q) - 1, cr.K);
    while (q + (1 << kk) - 1 > bend) kk--;
    add4(v, kk == 0 ? cr.pl[l * nb + q] : cr.hs[(int64_t)l * cr.hn + cr.ho[kk] + (q >> kk)]);
    q += 1 << kk;
  }
  const int64_t end = (int64_t)bend * kST + cr.plend[l * nb + bend];
  const int nn = offset[n];
  const int skipp = offset[end];
  const int mir = l + nn - skipp;
  write_records_b(r, mir, mir + (skipp - x), false, cr.prlen[l * nb + b]);
  write_records_a(r, mir, v);
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
// node as k_subtrees does; mass and com are read back from the node's fp64
// record (mirrored index l + n_nodes - offset[end]).  Each node registers
// itself in its parent's child slot (parent: the chain's previous node, or
// found by a backwards search for the start of the parent's key prefix).
// children must be -1 filled.  Export only, not on the registration path.
__global__ void __launch_bounds__(256) k_export(const unsigned long long* __restrict__ keys,
                                                int64_t n, int L,
                                                const signed char* __restrict__ clev,
                                                const int* __restrict__ offset,
                                                const double* __restrict__ box,
                                                const double4* __restrict__ a64,
                                                long long* children, double* com,
                                                double* mass, double* length,
                                                long long* occupancy, long long* depth,
                                                double* bmin, double* bmax) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = clev[i] + 1, cn = clev[i + 1];
  if (s > L) return;
  const int e = chain_end(s, cn, L);
  const int nn = offset[n];
  const unsigned long long k = keys[i];
  const int base = offset[i];
  double lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    lo[a] = box[a];
    hi[a] = box[3 + a];
  }
  for (int l = 0; l <= e; l++) {
    if (l > 0) bbox_step(k, l, L, lo, hi);
    if (l < s) continue;
    int64_t end;
    if (l == 0) end = n;
    else if (l > cn) end = i + 1;
    else end = upper_bound_gallop(keys, i + 1, n, k | low_mask(3 * (L - l)));
    const int64_t x = base + (l - s);
    const double4 v = a64[l + nn - offset[end]];
    if (mass) mass[x] = v.w;
    if (com) {
      com[x * 3] = v.x;
      com[x * 3 + 1] = v.y;
      com[x * 3 + 2] = v.z;
    }
    if (occupancy) occupancy[x] = end - i;
    if (depth) depth[x] = l;
    if (length) length[x] = diag_len(lo, hi);
    for (int a = 0; a < 3; a++) {
      if (bmin) bmin[x * 3 + a] = lo[a];
      if (bmax) bmax[x * 3 + a] = hi[a];
    }
    if (children && l > 0) {
      int64_t parent;
      if (l > s) {
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

// cells at the level cap holding >= 2 points (bit 0) and whether two of
// them are distinct (bit 1): clev[i] == L means point i shares all L levels
// with point i - 1
__global__ void k_cap_runs(const double4* __restrict__ sp, const signed char* __restrict__ clev,
                           int64_t n, int L, int* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1;
  if (i >= n || clev[i] < L) return;
  const double4 a = sp[i - 1], b = sp[i];
  atomicOr(flag, (a.x != b.x || a.y != b.y || a.z != b.z) ? 3 : 1);
}

// ------------------------------------------------------------------ host side
int tree_build_dev(TreeDev& T, const double* pts_dev, const double* masses_dev, int64_t n, int L,
                   cudaStream_t st) {
  T.generation++;  // any (re)build, even a failed one, invalidates cached host views
  if (n <= 0) {
    set_error("tree build: empty cloud");
    return FGA_ERR_EMPTY;
  }
  if (n >= (1ll << 31) - 2) {
    set_error("tree build: more than 2^31 points");
    return FGA_ERR_UNSUPPORTED;
  }
  if (L < 1) {
    set_error("tree build: max_depth must be >= 1");
    return FGA_ERR_INVALID;
  }
  T.L_requested = L;
  T.cap_runs = T.cap_distinct = false;
  if (L > kMaxLevels) L = kMaxLevels;  // see TreeDev::L_requested
  T.n_points = n;
  T.L = L;
  T.pts = pts_dev;
  T.masses = masses_dev;
  const int nb = (int)std::min<int64_t>(blocks_for(n), 4 * 148);
  FGA_CUDA_TRY(T.scratch.reserve(sizeof(double) * 6 * (nb + 1)));
  FGA_CUDA_TRY(T.box.reserve(sizeof(double) * 10));
  k_bbox_partial<<<nb, kThreads, 0, st>>>(pts_dev, n, T.scratch.as<double>());
  k_bbox_final<<<1, 256, 0, st>>>(T.scratch.as<double>(), nb, L, T.box.as<double>());

  // The sort runs on the top key bits only (3 radix passes for 24 bits, 4 for
  // 32) and k_fixup_runs orders each run of equal top bits by the full key;
  // a run longer than kRun retries with 32 bits, then with the full key.
  // 24 bits first only for small clouds (dense clusters of a large cloud
  // overflow the runs).
  int top_bits = n <= (1 << 22) ? 24 : 32;
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
  FGA_CUDA_TRY(T.flags.reserve(sizeof(int) * 2));
  int* overflow = T.flags.as<int>();  // a run of > kRun equal top key bits
  {
    size_t b32 = 0, b64 = 0, bscan = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b32, T.keys32_in.as<unsigned>(), T.keys32.as<unsigned>(),
                                    T.idx_in.as<int>(), T.idx.as<int>(), (int)n, 0, 32, st);
    cub::DeviceRadixSort::SortPairs(nullptr, b64, (const unsigned long long*)nullptr,
                                    (unsigned long long*)nullptr, T.idx_in.as<int>(),
                                    T.idx.as<int>(), (int)n, 0, 3 * L, st);
    cub::DeviceScan::ExclusiveSum(nullptr, bscan, (int*)nullptr, (int*)nullptr, (int)(n + 1), st);
    FGA_CUDA_TRY(T.cub_tmp.reserve(std::max(std::max(b32, b64), bscan)));
  }
  size_t tmp_bytes = T.cub_tmp.bytes;
  auto sort_top = [&](int bits) -> int {
    const int shift = std::max(0, 3 * L - bits);
    FGA_CUDA_TRY(cudaMemsetAsync(overflow, 0, sizeof(int), st));
    k_keys<<<blocks_for(n), kThreads, 0, st>>>(pts_dev, masses_dev, n, T.box.as<double>(), L, shift,
                                               T.keys32_in.as<unsigned>(), nullptr,
                                               T.idx_in.as<int>(), T.packed.as<double4>());
    tmp_bytes = T.cub_tmp.bytes;
    FGA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(T.cub_tmp.p, tmp_bytes, T.keys32_in.as<unsigned>(),
                                                 T.keys32.as<unsigned>(), T.idx_in.as<int>(),
                                                 T.idx.as<int>(), (int)n, 0, std::min(bits, 3 * L),
                                                 st));
    k_gather_sorted<<<blocks_for(n), kThreads, 0, st>>>(T.packed.as<double4>(), T.idx.as<int>(), n,
                                                        T.box.as<double>(), L, T.sp.as<double4>(),
                                                        T.keys.as<unsigned long long>());
    if (shift > 0)
      k_fixup_runs<<<blocks_for(n), kThreads, 0, st>>>(T.keys32.as<unsigned>(), n,
                                                       T.keys.as<unsigned long long>(),
                                                       T.idx.as<int>(), T.sp.as<double4>(), overflow);
    return FGA_OK;
  };
  TRY_RC(sort_top(top_bits));
  // c_i, node counts, preorder offsets (rerun after a fallback)
  auto levels = [&]() -> int {
    k_count<<<blocks_for(n + 1), kThreads, 0, st>>>(T.keys.as<unsigned long long>(), n, L,
                                                    T.clev.as<signed char>(), T.count.as<int>());
    size_t sb = T.cub_tmp.bytes;
    FGA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(T.cub_tmp.p, sb, T.count.as<int>(),
                                               T.offset.as<int>(), (int)(n + 1), st));
    return FGA_OK;
  };
  TRY_RC(levels());
  // node count, run overflow and root box to the host (one sync per build)
  int nn = 0, ovf = 0;
  double box[6];
  auto fetch = [&]() -> int {
    FGA_CUDA_TRY(cudaMemcpyAsync(&nn, T.offset.as<int>() + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    FGA_CUDA_TRY(cudaMemcpyAsync(box, T.box.p, sizeof(box), cudaMemcpyDeviceToHost, st));
    FGA_CUDA_TRY(cudaMemcpyAsync(&ovf, overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
    FGA_CUDA_TRY(cudaStreamSynchronize(st));
    return FGA_OK;
  };
  TRY_RC(fetch());
  if (ovf && top_bits < 32) {  // a long run of equal top 24 bits: 32 bits
    top_bits = 32;
    TRY_RC(sort_top(top_bits));
    TRY_RC(levels());
    TRY_RC(fetch());
  }
  if (ovf) {  // a long run of equal top bits: full 64-bit sort
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
  FGA_CUDA_TRY(T.c32.reserve(2 * sizeof(float4) * nn64));
  FGA_CUDA_TRY(T.band_scratch.reserve(64));
  FGA_CUDA_TRY(T.a64.reserve(sizeof(double4) * nn64));
  FGA_CUDA_TRY(T.b64.reserve(sizeof(NodeB64) * nn64));
  const int nbs = (int)((n + kST - 1) / kST);
  const int64_t ncr = (int64_t)(L + 1) * nbs;
  Cross cr{};
  cr.K = 0;
  while ((1ll << cr.K) < nbs) cr.K++;
  cr.hn = 0;
  for (int k = 1; k <= cr.K; k++) {
    cr.ho[k] = cr.hn;
    cr.hn += (nbs + (1 << k) - 1) >> k;
  }
  FGA_CUDA_TRY(T.cross.reserve(ncr * (2 * sizeof(double4) + sizeof(double) + 2 * sizeof(int)) +
                               sizeof(int) * nbs + sizeof(double4) * (L + 1) * (int64_t)cr.hn +
                               sizeof(int) * cr.hn + 64));
  {
    char* q = T.cross.as<char>();
    cr.pr = (double4*)q; q += sizeof(double4) * ncr;
    cr.pl = (double4*)q; q += sizeof(double4) * ncr;
    cr.hs = (double4*)q; q += sizeof(double4) * (L + 1) * (int64_t)cr.hn;
    cr.prlen = (double*)q; q += sizeof(double) * ncr;
    cr.prx = (int*)q; q += sizeof(int) * ncr;
    cr.plend = (int*)q; q += sizeof(int) * ncr;
    cr.mn = (int*)q; q += sizeof(int) * nbs;
    cr.hm = (int*)q;
  }
  k_subtrees<<<nbs, kST, 0, st>>>(T.keys.as<unsigned long long>(), n, L, T.clev.as<signed char>(),
                                  T.offset.as<int>(), T.box.as<double>(), T.sp.as<double4>(),
                                  T.records(), cr, nbs);
  if (nbs > 1) {
    for (int k0 = 0; k0 < cr.K; k0 += 5) {
      const int sz0 = (nbs + (1 << k0) - 1) >> k0;
      k_hier<<<dim3((sz0 + 255) / 256, L + 2), 256, 0, st>>>(L, nbs, k0, cr);
    }
    k_crossing<<<(int)((ncr + 255) / 256), 256, 0, st>>>(L, nbs, n, T.offset.as<int>(), cr,
                                                         T.records());
  }
  FGA_CUDA_TRY(cudaGetLastError());
  T.exportable = true;
  if (T.L_requested > kMaxLevels) {  // cells at the 21-level cap: one sync, rare path
    FGA_CUDA_TRY(cudaMemsetAsync(T.flags.as<int>() + 1, 0, sizeof(int), st));
    k_cap_runs<<<blocks_for(n), kThreads, 0, st>>>(T.sp.as<double4>(), T.clev.as<signed char>(), n,
                                                   L, T.flags.as<int>() + 1);
    int f = 0;
    FGA_CUDA_TRY(cudaMemcpyAsync(&f, T.flags.as<int>() + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    FGA_CUDA_TRY(cudaStreamSynchronize(st));
    T.cap_runs = (f & 1) != 0;
    T.cap_distinct = (f & 2) != 0;
  }
  return FGA_OK;
}

namespace {
// a depth-cap leaf holding two distinct points (equal full keys, different
// coordinates): the only way a leaf aggregates more than one position
__global__ void k_shared_leaf(const double4* __restrict__ sp, const signed char* __restrict__ clev,
                              int64_t n, int L, int* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1;
  if (i >= n || clev[i] < L) return;
  const double4 a = sp[i - 1], b = sp[i];
  if (a.x != b.x || a.y != b.y || a.z != b.z) atomicOr(flag, 1);
}
}  // namespace

int tree_any_shared_leaf(TreeDev& T, cudaStream_t st, int* host_flag) {
  *host_flag = 0;
  if (!T.exportable || T.n_points < 2) return FGA_OK;
  int* f = T.flags.as<int>() + 1;
  FGA_CUDA_TRY(cudaMemsetAsync(f, 0, sizeof(int), st));
  k_shared_leaf<<<blocks_for(T.n_points - 1), kThreads, 0, st>>>(
      T.sp.as<double4>(), T.clev.as<signed char>(), T.n_points, T.L, f);
  FGA_CUDA_TRY(cudaMemcpyAsync(host_flag, f, sizeof(int), cudaMemcpyDeviceToHost, st));
  FGA_CUDA_TRY(cudaStreamSynchronize(st));
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
  k_export<<<blocks_for(T.n_points), 256, 0, st>>>(
      T.keys.as<unsigned long long>(), T.n_points, T.L, T.clev.as<signed char>(),
      T.offset.as<int>(), T.box.as<double>(), T.a64.as<double4>(),
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
  T.generation++;
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
  std::vector<float4> c32(2 * nn);
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
    c32[2 * mir] = make_float4((float)com[x * 3], (float)com[x * 3 + 1], (float)com[x * 3 + 2],
                               (float)mass[x]);
    const float l2f = leaf ? -INFINITY : (float)l2;
    float skipf;
    const int skipi = (int)(mir + size);
    std::memcpy(&skipf, &skipi, sizeof(float));
    c32[2 * mir + 1] = make_float4(l2f, skipf, 0.f, l2f);
    for (int k = 0; k < 3; k++) cmag = std::max(cmag, std::fabs(com[x * 3 + k]));
  }
  FGA_CUDA_TRY(T.a64.reserve(sizeof(double4) * nn));
  FGA_CUDA_TRY(T.b64.reserve(sizeof(NodeB64) * nn));
  FGA_CUDA_TRY(T.c32.reserve(2 * sizeof(float4) * nn));
  FGA_CUDA_TRY(T.band_scratch.reserve(64));
  FGA_CUDA_TRY(cudaMemcpyAsync(T.c32.p, c32.data(), 2 * sizeof(float4) * nn, cudaMemcpyHostToDevice,
                               st));
  FGA_CUDA_TRY(cudaMemcpyAsync(T.a64.p, a64.data(), sizeof(double4) * nn, cudaMemcpyHostToDevice, st));
  FGA_CUDA_TRY(cudaMemcpyAsync(T.b64.p, b64.data(), sizeof(NodeB64) * nn, cudaMemcpyHostToDevice, st));
  FGA_CUDA_TRY(cudaStreamSynchronize(st));
  T.n_nodes = nn;
  T.cmag = cmag;
  T.exportable = false;
  return FGA_OK;
}

}  // namespace fga
