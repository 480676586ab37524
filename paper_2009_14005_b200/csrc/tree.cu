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
// in slot order, so no child table is kept.  Node aggregates are exact
// fixed-point sums over each node's point range (differences of prefix sums,
// see "aggregates" below), so they are independent of how the work is split;
// each node's traversal records are written in *mirrored* preorder (see
// fga_internal.cuh).
//
// Kernels (all HBM/L2-bound integer + fp64 work; no tensor cores):
//   k_bbox_*        root bbox = per-axis min/max (bhtree.py:107-108), max |m|
//   k_keys          per-axis fp64 split recursion -> 3L-bit key (dyadic fast
//                   path with an exact-replay fallback near split planes)
//   (cub radix sort, stable: keeps the reference's within-leaf index order)
//   k_gather_sorted sorted points + full keys; k_fixup_runs low key bits
//   k_count         c_i and per-point node counts
//   (cub exclusive scan) -> preorder offsets, node count
//   k_subtrees      per block of kST sorted points: exact prefix sums, then
//                   one node per thread (bbox replay -> length, end -> skip
//                   and sums) -> records
//   k_tscan1/2      prefix sums of the block totals
//   k_crossing      nodes that run past their block: sums from the prefixes
#include <cub/cub.cuh>

#include <cstdlib>
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
__global__ void k_bbox_partial(const double* __restrict__ pts, const double* __restrict__ masses,
                               int64_t n, double* __restrict__ part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  double mm = 0.0;  // max |mass| (the fixed-point scale of the node sums)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; k++) {
      double v = pts[i * 3 + k];
      lo[k] = fmin(lo[k], v);
      hi[k] = fmax(hi[k], v);
    }
    mm = fmax(mm, fabs(masses[i]));
  }
  __shared__ double s[7][kThreads / 32];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  }
  for (int o = 16; o > 0; o >>= 1) mm = fmax(mm, __shfl_xor_sync(0xffffffffu, mm, o));
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    for (int k = 0; k < 3; k++) {
      s[k][w] = lo[k];
      s[3 + k][w] = hi[k];
    }
    s[6][w] = mm;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    double r = s[threadIdx.x][0];
    for (int j = 1; j < (int)(blockDim.x >> 5); j++)
      r = threadIdx.x < 3 ? fmin(r, s[threadIdx.x][j]) : fmax(r, s[threadIdx.x][j]);
    part[blockIdx.x * 7 + threadIdx.x] = r;
  }
}

__device__ __forceinline__ void fixed_scale(const double* box, int64_t n, double* out);

// box[0..5] = lo, hi; box[6..8] = 2^L / (hi - lo) per axis; box[9] = the
// fast-key guard (see k_keys); box[10] = max |mass|, box[11..13] the
// fixed-point scale of the node sums (see fixed_scale)
__global__ void k_bbox_final(const double* __restrict__ part, int nparts, int L, int64_t n,
                             double* __restrict__ out) {
  for (int k = 0; k < 7; k++) {
    double v = k < 3 ? INFINITY : (k < 6 ? -INFINITY : 0.0);
    for (int j = threadIdx.x; j < nparts; j += blockDim.x)
      v = k < 3 ? fmin(v, part[j * 7 + k]) : fmax(v, part[j * 7 + k]);
    v = k < 3 ? block_reduce<1>(v) : block_reduce<2>(v);
    if (threadIdx.x == 0) out[k < 6 ? k : 10] = v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double R = 0.0;
    for (int k = 0; k < 3; k++) {
      const double w = out[3 + k] - out[k];
      out[6 + k] = w > 0.0 ? ldexp(1.0, L) / w : 0.0;
      R = fmax(R, fmax(fabs(out[k]), fabs(out[3 + k])));
    }
    out[9] = 256.0 * 1.1102230246251565e-16 * R;  // 256 u R
    fixed_scale(out, n, out);
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

// Keys: 3 bits per level, level 1 most significant, in a 64-bit word for
// L <= 21 (kMaxLevels) or a 128-bit one for L <= 42 (kMaxLevelsDeep: the
// reference's max_depth beyond 21, bhtree.py:89).
typedef unsigned long long K64;
typedef unsigned __int128 K128;
__device__ __forceinline__ int kclz(K64 x) { return __clzll((long long)x); }
__device__ __forceinline__ int kclz(K128 x) {
  const K64 hi = (K64)(x >> 64);
  return hi ? __clzll((long long)hi) : 64 + __clzll((long long)(K64)x);
}
template <class K>
__device__ __forceinline__ int klevels(K a, K b, int L) {  // common levels of two keys
  const K x = a ^ b;
  if (x == (K)0) return L;
  return (kclz(x) - (8 * (int)sizeof(K) - 3 * L)) / 3;
}
template <class K>
__device__ __forceinline__ K klow(int bits) {
  return bits >= 8 * (int)sizeof(K) ? ~(K)0 : (((K)1 << bits) - (K)1);
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

template <class K>
__device__ __forceinline__ K point_key(const double p[3], const double* __restrict__ box, int L) {
  const double guard = box[9];
  unsigned long long q[3];
  bool fast = true;
#pragma unroll
  for (int k = 0; k < 3; k++)
    fast = fast_axis(p[k], box[k], box[6 + k], guard * box[6 + k], L, q[k]) && fast;
  if (fast) {
    if constexpr (sizeof(K) == 8) return (spread3(q[0]) << 2) | (spread3(q[1]) << 1) | spread3(q[2]);
    // 42 bits per axis: the top 21 levels' interleave above the low 63 bits
    const K hi = (spread3(q[0] >> 21) << 2) | (spread3(q[1] >> 21) << 1) | spread3(q[2] >> 21);
    const K lo = (spread3(q[0]) << 2) | (spread3(q[1]) << 1) | spread3(q[2]);
    return (hi << 63) | lo;
  }
  double lo[3], hi[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    lo[k] = box[k];
    hi[k] = box[3 + k];
  }
  K key = 0;
  for (int l = 0; l < L; l++) {
    unsigned digit = 0;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const double c = __dadd_rn(lo[k], __dmul_rn(__dsub_rn(hi[k], lo[k]), 0.5));
      const bool up = p[k] >= c;
      digit = (digit << 1) | (up ? 1u : 0u);
      if (up) lo[k] = c; else hi[k] = c;
    }
    key = (key << 3) | (K)digit;
  }
  return key;
}

// Key of every point in input order, the sort's index payload and the packed
// (x, y, z, m) record.  The sort runs on the top 32 key bits (keys32, 4 radix
// passes instead of 8); keys64 (the full key) is written only for the
// fallback full sort.
template <class K>
__global__ void k_keys(const double* __restrict__ pts, const double* __restrict__ masses, int64_t n,
                       const double* __restrict__ box, int L, int shift,
                       unsigned* __restrict__ keys32, K* __restrict__ keys64,
                       int* __restrict__ idx, double4* __restrict__ packed) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3];
#pragma unroll
  for (int k = 0; k < 3; k++) p[k] = pts[i * 3 + k];
  packed[i] = make_double4(p[0], p[1], p[2], masses[i]);  // one 32 B record per point
  const K key = point_key<K>(p, box, L);
  if (keys64) keys64[i] = key;
  else keys32[i] = (unsigned)(key >> shift);
  idx[i] = (int)i;
}

// Sorted copy of the points (one random gather of the packed records) and,
// when the sort ran on the top key bits only, the full key recomputed from
// the point (no second gather).
template <class K>
__global__ void k_gather_sorted(const double4* __restrict__ packed, const int* __restrict__ idx,
                                int64_t n, const double* __restrict__ box, int L,
                                double4* __restrict__ sp, K* __restrict__ keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 v = packed[idx[i]];
  sp[i] = v;
  if (keys) {
    const double p[3] = {v.x, v.y, v.z};
    keys[i] = point_key<K>(p, box, L);
  }
}

// After the (stable) sort on the top 32 bits: every run of equal top bits is
// put in full-key order by one thread (stable insertion sort, so equal keys
// keep index order as the reference's partition does).  Runs longer than
// kRun set *overflow and the build falls back to the full 64-bit sort.
constexpr int kRun = 64;
template <class K>
__global__ void k_fixup_runs(const unsigned* __restrict__ hi, int64_t n,
                             K* __restrict__ key, int* __restrict__ idx,
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
    const K kk = key[i + a];
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
template <class K>
__global__ void k_count(const K* __restrict__ keys, int64_t n, int L,
                        signed char* __restrict__ clev, int* __restrict__ count) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  const int c = (i == 0 || i == n) ? -1 : klevels(keys[i - 1], keys[i], L);
  clev[i] = (signed char)c;
  int cnt = 0;
  if (i < n) {
    const int cn = (i + 1 == n) ? -1 : klevels(keys[i], keys[i + 1], L);
    const int s = c + 1;
    if (s <= L) cnt = chain_end(s, cn, L) - s + 1;
  }
  count[i] = cnt;
}

// first j in [from, n) with keys[j] > bound (keys sorted): galloping search
// from `from` (subtree ends are near the start for all but the top levels)
template <class K>
__device__ __forceinline__ int64_t upper_bound_gallop(const K* keys, int64_t from, int64_t n,
                                                      K bound) {
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
template <class K>
__device__ __forceinline__ void bbox_step(K key, int lev, int L, double lo[3],
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

// ---------------------------------------------------------------- aggregates
// A node's mass and m*p sums (bhtree.py:78-82) are sums over its points; the
// reference adds them in its own order (numpy's pairwise sum for the mass,
// row by row for m*p), so no fp64 grouping a parallel build can use gives its
// last bits.  Here every point's terms (m, m x, m y, m z) -- the products
// rounded to fp64 as the reference rounds them -- become 128-bit fixed-point
// integers under one scale 2^S for the whole build, S chosen from the largest
// possible |term| and n so that no partial sum can overflow and every term
// above 2^-S is exact.  A node's sums are then differences of prefix sums:
// exact integers, independent of how the work is split over blocks, threads
// or crossing partials, and converted to fp64 once (com = one division of the
// two rounded sums, as the reference's `sum / total`).  The tests hold the
// aggregates to 1e-12 of the reference's (the topology, lengths and skips
// are bit-exact).
typedef unsigned __int128 u128;
struct __align__(16) Q4 {
  u128 v[4];
};

// The scale (k_bbox_final): sums of up to n terms each below max|m| *
// max(1, max|coord|) stay below 2^122; S <= 1074 (every double is then a
// multiple of 2^-S: all terms exact), S >= -1000.  box[11] = S, box[12] =
// 2^(S-64), box[13] = 2^-S.
__device__ __forceinline__ void fixed_scale(const double* box, int64_t n, double* out) {
  double R = 1.0;
#pragma unroll
  for (int k = 0; k < 6; k++) R = fmax(R, fabs(box[k]));
  const double bound = box[10] * R * (double)n;
  int S = 0;
  if (bound > 0.0 && bound < 1e300) {
    int e;
    frexp(bound, &e);  // bound < 2^e
    S = min(122 - e, 1074);
  } else if (bound > 0.0) {
    S = -1000;
  }
  out[11] = (double)S;
  out[12] = ldexp(1.0, S - 64);
  out[13] = ldexp(1.0, -S);
}

// round(v * 2^S) as a two's-complement 128-bit integer (s64 = 2^(S-64)):
// |v| 2^(S-64) = h + r, h = floor (< 2^58), r in [0, 1) exact, low word =
// r 2^64 rounded to nearest
__device__ __forceinline__ u128 to_fixed(double v, double s64) {
  const double a = fabs(v) * s64;
  const double h = floor(a);
  const unsigned long long lo = __double2ull_rn((a - h) * 18446744073709551616.0);
  const u128 q = ((u128)__double2ull_rn(h) << 64) | lo;
  return v < 0.0 ? (u128)0 - q : q;
}

// the two's-complement integer as fp64 (hi * 2^64 + lo, one fused rounding
// after the exact conversion of hi: within one unit of the last place, and a
// fixed function of the integer)
__device__ __forceinline__ double fixed_to_double(u128 u) {
  const long long hi = (long long)(unsigned long long)(u >> 64);
  return __fma_rn(__ll2double_rn(hi), 18446744073709551616.0,
                  __ull2double_rn((unsigned long long)u));
}

__device__ __forceinline__ void point_terms(const double4& p, double s64, u128 q[4]) {
  q[0] = to_fixed(p.w, s64);
  q[1] = to_fixed(__dmul_rn(p.x, p.w), s64);
  q[2] = to_fixed(__dmul_rn(p.y, p.w), s64);
  q[3] = to_fixed(__dmul_rn(p.z, p.w), s64);
}

__device__ __forceinline__ u128 shfl_up128(u128 v, int d) {
  const unsigned long long lo = __shfl_up_sync(0xffffffffu, (unsigned long long)v, d);
  const unsigned long long hi = __shfl_up_sync(0xffffffffu, (unsigned long long)(v >> 64), d);
  return ((u128)hi << 64) | lo;
}

// inclusive block scan of q over the block's threads (wt: one Q4 per warp,
// shared; one barrier inside)
__device__ __forceinline__ void block_scan_q4(u128 q[4], Q4* wt) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int c = 0; c < 4; c++) {
      const u128 y = shfl_up128(q[c], d);
      if (lane >= d) q[c] += y;
    }
  }
  if (lane == 31)
#pragma unroll
    for (int c = 0; c < 4; c++) wt[w].v[c] = q[c];
  __syncthreads();
  for (int ww = 0; ww < w; ww++)
#pragma unroll
    for (int c = 0; c < 4; c++) q[c] += wt[ww].v[c];
}

// The node's traversal records at its mirrored-preorder index: fp64 {com,
// mass} and {l^2 | -inf, skip}, and the packed FP32 record (NodeC32).
__device__ __forceinline__ void write_node(const TreeRecords& r, int mir, int rskip, bool leaf,
                                           double len, double cx, double cy, double cz,
                                           double m) {
  const double l2 = __dmul_rn(len, len);
  r.a64[mir] = make_double4(cx, cy, cz, m);
  r.b64[mir] = NodeB64{leaf ? -INFINITY : l2, (long long)rskip};
  const float l2f = leaf ? -INFINITY : (float)l2;
  r.c32[2 * mir] = make_float4((float)cx, (float)cy, (float)cz, (float)m);
  r.c32[2 * mir + 1] = make_float4(l2f, __int_as_float(rskip), 0.f, l2f);
}

// records of a node whose exact sums are a[0..3] (scaled by 2^S)
__device__ __forceinline__ void write_node_sums(const TreeRecords& r, int mir, int rskip,
                                                double len, const u128 a[4], double sinv) {
  const double am = fixed_to_double(a[0]);
  write_node(r, mir, rskip, false, len, __ddiv_rn(fixed_to_double(a[1]), am),
             __ddiv_rn(fixed_to_double(a[2]), am), __ddiv_rn(fixed_to_double(a[3]), am),
             am * sinv);
}

// ---------------------------------------------------------------- hierarchy
// Node (i, l) holds the sorted points [i, end), end = first j > i with
// c_j < l, and its preorder subtree is the chain rest of i plus every chain
// of the points in (i, end); so its preorder skip is offset[end] and its
// mirrored index is l + n_nodes - offset[end] -- no bottom-up pass at all:
// with the exact prefix sums a node's aggregate is E[end] - E[i].
//
// Blocks of kST consecutive sorted points (k_subtrees) hold their own
// exclusive prefix sums E_b; a node that runs past its block's end (at most
// one per level per block) is finished by k_crossing from
//   G(b) = sum of the totals of blocks < b   (k_tscan1/2)
//   pst  = E_b(i) of its start                (k_subtrees, owner block)
//   plE  = E_b'(end) inside the end block b'  (k_subtrees of b': the level-l
//          node covering b's first point ends there)
// as G(b') + plE - G(b) - pst.
#ifndef FGA_KST
#define FGA_KST 128
#endif
constexpr int kST = FGA_KST;
constexpr int kSW = kST / 32;
#ifndef FGA_STB
#define FGA_STB (1536 / kST)
#endif
constexpr int kSTBlocks = FGA_STB;  // resident blocks per SM
constexpr int kTScan = 256;         // blocks per chunk of the block-total scan

struct Cross {
  int* prx;      // [(L+1) nb] preorder index of the owned crossing node, -1 none
  int* prs;      // its start point
  double* prlen; // its length
  Q4* pst;       // E_b at its start
  Q4* plE;       // E_b at the end of the level-l node covering b's first point
  Q4* T;         // [nb] block totals
  Q4* Gi;        // [nb] inclusive scan of T within chunks of kTScan blocks
  Q4* CS;        // [nc] chunk totals
  Q4* CX;        // [nc + 1] exclusive scan of CS (CX[nc] = grand total)
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

__device__ __forceinline__ u128 e_limb(const unsigned long long (*E)[kST + 1], int c, int p) {
  return ((u128)E[2 * c + 1][p] << 64) | E[2 * c][p];
}
__device__ __forceinline__ Q4 e_at(const unsigned long long (*E)[kST + 1], int p) {
  Q4 r;
#pragma unroll
  for (int c = 0; c < 4; c++) r.v[c] = e_limb(E, c, p);
  return r;
}

// One block = kST sorted points, one thread each.  Per level l a bit mask
// over the block's points: B_l (c_j < l: a node at level <= l starts at j, so
// it ends every level-l range).  All the block's points share the levels <=
// lca (the common levels of its first and last key), so above lca only
// position 0 has nodes.  One node per thread: bbox replay from the shared
// level-lca box (bhtree.py:90-103) -> length; end = the next B_l bit ->
// skip = offset[end] and the sums E[end] - E[j]; records.
template <class K>
__global__ void __launch_bounds__(kST, kSTBlocks) k_subtrees(const K* __restrict__ keys,
                                                     int64_t n, int L,
                                                     const signed char* __restrict__ clev,
                                                     const int* __restrict__ offset,
                                                     const double* __restrict__ box,
                                                     const double4* __restrict__ sp,
                                                     TreeRecords r, Cross cr, int nb) {
  constexpr int kLv = sizeof(K) == 8 ? kMaxLevels : kMaxLevelsDeep;
  __shared__ unsigned mB[kLv + 2][kSW];
  __shared__ unsigned nzB[kLv + 2];
  __shared__ int offs[kST + 1];
  __shared__ signed char cs[kST + 1];
  __shared__ K skey[kST];
  // SoA in shared memory (64-bit words per thread: no bank conflicts)
  __shared__ double P[4][kST];                     // the block's points x, y, z, m
  __shared__ unsigned long long E[8][kST + 1];     // prefix sums: limb 2c = low, 2c+1 = high
  __shared__ Q4 wt[kSW];
  __shared__ double pbox[6];
  __shared__ int s_maxe;
  constexpr int kMap = 4 * kST;  // node -> point map of the node pass
  __shared__ short nmap[kMap];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5, b = blockIdx.x;
  const int64_t B0 = (int64_t)b * kST, i = B0 + t;
  const int64_t last = min(B0 + kST, n) - 1;
  const int nn = offset[n];
  const double s64 = box[12], sinv = box[13];
  cs[t] = i <= n ? clev[i] : (signed char)-1;
  offs[t] = i <= n ? offset[i] : nn;
  skey[t] = i < n ? keys[i] : (K)0;
  const double4 pv = i < n ? sp[i] : make_double4(0.0, 0.0, 0.0, 0.0);
  P[0][t] = pv.x;
  P[1][t] = pv.y;
  P[2][t] = pv.z;
  P[3][t] = pv.w;
  if (t == 0) {
    const int64_t j = B0 + kST;
    cs[kST] = j <= n ? clev[j] : (signed char)-1;
    offs[kST] = j <= n ? offset[j] : nn;
    s_maxe = -1;
  }
  if (t <= L) cr.prx[t * nb + b] = -1;
  {  // the block's exclusive prefix sums E[0..kST]: per component a warp
     // scan into E, then (after the next barrier) the earlier warps' totals
#pragma unroll 1
    for (int c = 0; c < 4; c++) {
      const double tv = c == 0 ? pv.w : __dmul_rn(c == 1 ? pv.x : (c == 2 ? pv.y : pv.z), pv.w);
      u128 q = to_fixed(tv, s64);
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u128 y = shfl_up128(q, d);
        if (lane >= d) q += y;
      }
      E[2 * c][t + 1] = (unsigned long long)q;
      E[2 * c + 1][t + 1] = (unsigned long long)(q >> 64);
      if (lane == 31) wt[w].v[c] = q;
    }
    if (t == 0)
      for (int c = 0; c < 8; c++) E[c][0] = 0ull;
  }
  __syncthreads();  // cs, offs, skey, s_maxe
  const K k0 = skey[0];
  const int lca = last > B0 ? klevels(k0, skey[last - B0], L) : L;
  const int c = cs[t], c0 = cs[0], cend = cs[kST];
  const bool has = i < n && c + 1 <= L;
  const int s = c + 1, e = has ? chain_end(s, cs[t + 1], L) : -1;
  if (has) {
    atomicMax(&s_maxe, e);
    const int x0 = offs[t] - offs[0];
    if (x0 + (e - s) < kMap)
      for (int q = 0; q <= e - s; q++) nmap[x0 + q] = (short)t;
  }
  if (t == kST - 1) {  // the box of the level-lca node holding every point of the block
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
  __syncthreads();
  if (w > 0)  // the earlier warps' totals into this thread's prefix sums
#pragma unroll 1
    for (int cc = 0; cc < 4; cc++) {
      u128 add = wt[0].v[cc];
      for (int ww = 1; ww < w; ww++) add += wt[ww].v[cc];
      const u128 v = e_limb(E, cc, t + 1) + add;
      E[2 * cc][t + 1] = (unsigned long long)v;
      E[2 * cc + 1][t + 1] = (unsigned long long)(v >> 64);
    }
  const int top = s_maxe;
  const int mtop = max(top, min(c0, L));  // deepest level with a node here
  for (int l = lca; l <= mtop; l++) {
    const unsigned bb = __ballot_sync(0xffffffffu, c < l);
    if (lane == 0) mB[l][w] = bb;
  }
  __syncthreads();
  if (t >= lca && t <= mtop) {  // per level: non-zero word summary
    unsigned zb = 0;
    for (int q = 0; q < kSW; q++) zb |= (mB[t][q] != 0u ? 1u : 0u) << q;
    nzB[t] = zb;
  }
  __syncthreads();
  if (t == 0) cr.T[b] = e_at(E, kST);
  if (t <= min(c0, L)) {  // level-t node covering position 0 (owned earlier): its end here
    const int l = t;
    const int p = l <= lca ? kST : next_bit(mB[l], nzB[l], 0);
    if (p < kST || cend < l) cr.plE[l * nb + b] = e_at(E, p);
  }

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
    const K key = skey[j];
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
    if (l == ej) {  // leaf: point j alone, or a depth-cap cell of duplicates
      const int mir = l + nn - (x + 1);
      FGA_CHECK(mir >= 0 && mir < nn);
      const int64_t gi = B0 + j;
      if (ej > cs[j + 1]) {  // one point: (x m) / m, as the reference's sums of one row
        const double4 v = make_double4(P[0][j], P[1][j], P[2][j], P[3][j]);
        write_node(r, mir, mir + 1, true, len, __ddiv_rn(__dadd_rn(0.0, __dmul_rn(v.x, v.w)), v.w),
                   __ddiv_rn(__dadd_rn(0.0, __dmul_rn(v.y, v.w)), v.w),
                   __ddiv_rn(__dadd_rn(0.0, __dmul_rn(v.z, v.w)), v.w), v.w);
      } else {
        const int64_t end = ej == 0 ? n : upper_bound_gallop(keys, gi + 1, n, key | klow<K>(3 * (L - ej)));
        u128 a[4] = {0, 0, 0, 0};
        for (int64_t q = gi; q < end; q++) {
          u128 tq[4];
          point_terms(sp[q], s64, tq);
#pragma unroll
          for (int cc = 0; cc < 4; cc++) a[cc] += tq[cc];
        }
        const double am = fixed_to_double(a[0]);
        write_node(r, mir, mir + 1, true, len, __ddiv_rn(fixed_to_double(a[1]), am),
                   __ddiv_rn(fixed_to_double(a[2]), am), __ddiv_rn(fixed_to_double(a[3]), am),
                   am * sinv);
      }
    } else {
      const int p = l <= lca ? kST : next_bit(mB[l], nzB[l], j);
      if (p < kST || cend < l) {
        const int skipp = offs[p];
        const int mir = l + nn - skipp;
        FGA_CHECK(mir >= 0 && mir < nn);
        u128 a[4];
#pragma unroll
        for (int cc = 0; cc < 4; cc++) a[cc] = e_limb(E, cc, p) - e_limb(E, cc, j);
        write_node_sums(r, mir, mir + (skipp - x), len, a, sinv);
      } else {  // runs past the block: k_crossing
        cr.prx[l * nb + b] = x;
        cr.prs[l * nb + b] = (int)(B0 + j);
        cr.prlen[l * nb + b] = len;
        cr.pst[l * nb + b] = e_at(E, j);
      }
    }
  }
}

// Scan of the block totals: inclusive within chunks of kTScan blocks, and the
// chunk totals.
__global__ void __launch_bounds__(kTScan) k_tscan1(int nb, Cross cr) {
  __shared__ Q4 wt[kTScan / 32];
  const int b = blockIdx.x * kTScan + threadIdx.x;
  u128 q[4] = {0, 0, 0, 0};
  if (b < nb)
#pragma unroll
    for (int c = 0; c < 4; c++) q[c] = cr.T[b].v[c];
  block_scan_q4(q, wt);
  if (b < nb)
#pragma unroll
    for (int c = 0; c < 4; c++) cr.Gi[b].v[c] = q[c];
  if (threadIdx.x == kTScan - 1)
#pragma unroll
    for (int c = 0; c < 4; c++) cr.CS[blockIdx.x].v[c] = q[c];
}

// Exclusive scan of the chunk totals (one block; CX[nc] = grand total).
__global__ void __launch_bounds__(kTScan) k_tscan2(int nc, Cross cr) {
  __shared__ Q4 wt[kTScan / 32];
  __shared__ Q4 carry;
  if (threadIdx.x == 0)
    for (int c = 0; c < 4; c++) carry.v[c] = 0;
  __syncthreads();
  for (int base = 0; base < nc; base += kTScan) {
    const int k = base + threadIdx.x;
    u128 q[4] = {0, 0, 0, 0}, own[4] = {0, 0, 0, 0};
    if (k < nc)
#pragma unroll
      for (int c = 0; c < 4; c++) own[c] = q[c] = cr.CS[k].v[c];
    block_scan_q4(q, wt);
    if (k < nc)
#pragma unroll
      for (int c = 0; c < 4; c++) cr.CX[k].v[c] = carry.v[c] + q[c] - own[c];
    __syncthreads();
    if (threadIdx.x == kTScan - 1)
#pragma unroll
      for (int c = 0; c < 4; c++) carry.v[c] += q[c];
    __syncthreads();
  }
  if (threadIdx.x == 0) cr.CX[nc] = carry;
}

// sum of the totals of blocks < b
__device__ __forceinline__ void block_prefix(const Cross& cr, int nb, int b, u128 g[4]) {
  if (b >= nb) {
    const int nc = (nb + kTScan - 1) / kTScan;
#pragma unroll
    for (int c = 0; c < 4; c++) g[c] = cr.CX[nc].v[c];
    return;
  }
#pragma unroll
  for (int c = 0; c < 4; c++) g[c] = cr.Gi[b].v[c] - cr.T[b].v[c] + cr.CX[b / kTScan].v[c];
}

// One thread per (level, block) with an owned crossing node: its end (the
// first later key outside its prefix), its exact sums from the block prefix
// sums, and its records.
template <class K>
__global__ void __launch_bounds__(256) k_crossing(int L, int nb, int64_t n,
                                                  const K* __restrict__ keys,
                                                  const int* __restrict__ offset,
                                                  const double* __restrict__ box, Cross cr,
                                                  TreeRecords r) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= (int64_t)(L + 1) * nb) return;
  const int l = (int)(g / nb), b = (int)(g % nb);
  const int x = cr.prx[l * nb + b];
  if (x < 0) return;
  const int64_t i = cr.prs[l * nb + b];
  const int64_t end = l == 0 ? n : upper_bound_gallop(keys, i + 1, n, keys[i] | klow<K>(3 * (L - l)));
  const int bend = (int)(end / kST), pe = (int)(end - (int64_t)bend * kST);
  u128 ge[4], gb[4], a[4];
  block_prefix(cr, nb, bend, ge);
  block_prefix(cr, nb, b, gb);
#pragma unroll
  for (int c = 0; c < 4; c++) {
    a[c] = ge[c] - gb[c] - cr.pst[l * nb + b].v[c];
    if (pe > 0) a[c] += cr.plE[l * nb + bend].v[c];
  }
  const int nn = offset[n];
  const int skipp = offset[end];
  const int mir = l + nn - skipp;
  FGA_CHECK(mir >= 0 && mir < nn && bend > b);
  write_node_sums(r, mir, mir + (skipp - x), cr.prlen[l * nb + b], a, box[13]);
}

// first p in [0, to) with keys[p] >= bound, galloping backwards from `to`
template <class K>
__device__ __forceinline__ int64_t lower_bound_gallop(const K* keys, int64_t to, K bound) {
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
template <class K>
__global__ void __launch_bounds__(256) k_export(const K* __restrict__ keys,
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
  const K k = keys[i];
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
    else end = upper_bound_gallop(keys, i + 1, n, k | klow<K>(3 * (L - l)));
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
        const int64_t p = lower_bound_gallop(keys, i, k & ~klow<K>(3 * (L - l + 1)));
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
template <class K>
static int tree_build_k(TreeDev& T, const double* pts_dev, const double* masses_dev, int64_t n,
                        int L, cudaStream_t st);

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
  if (L > kMaxLevelsDeep) L = kMaxLevelsDeep;  // see TreeDev::L_requested
  T.wide_keys = L > kMaxLevels;  // 128-bit keys beyond 21 levels
  return T.wide_keys ? tree_build_k<K128>(T, pts_dev, masses_dev, n, L, st)
                     : tree_build_k<K64>(T, pts_dev, masses_dev, n, L, st);
}

template <class K>
static int tree_build_k(TreeDev& T, const double* pts_dev, const double* masses_dev, int64_t n,
                        int L, cudaStream_t st) {
  T.n_points = n;
  T.L = L;
  T.pts = pts_dev;
  T.masses = masses_dev;
  const int nb = (int)std::min<int64_t>(blocks_for(n), 4 * 148);
  FGA_CUDA_TRY(T.scratch.reserve(sizeof(double) * 7 * (nb + 1)));
  FGA_CUDA_TRY(T.box.reserve(sizeof(double) * 16));
  k_bbox_partial<<<nb, kThreads, 0, st>>>(pts_dev, masses_dev, n, T.scratch.as<double>());
  k_bbox_final<<<1, 256, 0, st>>>(T.scratch.as<double>(), nb, L, n, T.box.as<double>());

  // The sort runs on the top key bits only (3 radix passes for 24 bits, 4 for
  // 32) and k_fixup_runs orders each run of equal top bits by the full key;
  // a run longer than kRun retries with 32 bits, then with the full key.
  // 24 bits first only for small clouds (dense clusters of a large cloud
  // overflow the runs).
  int top_bits = n <= (1 << 22) ? 24 : 32;
  FGA_CUDA_TRY(T.keys.reserve(sizeof(K) * n));
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
    cub::DeviceRadixSort::SortPairs(nullptr, b64, (const K*)nullptr, (K*)nullptr,
                                    T.idx_in.as<int>(),
                                    T.idx.as<int>(), (int)n, 0, 3 * L, st);
    cub::DeviceScan::ExclusiveSum(nullptr, bscan, (int*)nullptr, (int*)nullptr, (int)(n + 1), st);
    FGA_CUDA_TRY(T.cub_tmp.reserve(std::max(std::max(b32, b64), bscan)));
  }
  size_t tmp_bytes = T.cub_tmp.bytes;
  auto sort_top = [&](int bits) -> int {
    const int shift = std::max(0, 3 * L - bits);
    FGA_CUDA_TRY(cudaMemsetAsync(overflow, 0, sizeof(int), st));
    k_keys<K><<<blocks_for(n), kThreads, 0, st>>>(pts_dev, masses_dev, n, T.box.as<double>(), L, shift,
                                               T.keys32_in.as<unsigned>(), nullptr,
                                               T.idx_in.as<int>(), T.packed.as<double4>());
    tmp_bytes = T.cub_tmp.bytes;
    FGA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(T.cub_tmp.p, tmp_bytes, T.keys32_in.as<unsigned>(),
                                                 T.keys32.as<unsigned>(), T.idx_in.as<int>(),
                                                 T.idx.as<int>(), (int)n, 0, std::min(bits, 3 * L),
                                                 st));
    k_gather_sorted<K><<<blocks_for(n), kThreads, 0, st>>>(T.packed.as<double4>(), T.idx.as<int>(), n,
                                                        T.box.as<double>(), L, T.sp.as<double4>(),
                                                        T.keys.as<K>());
    if (shift > 0)
      k_fixup_runs<<<blocks_for(n), kThreads, 0, st>>>(T.keys32.as<unsigned>(), n,
                                                       T.keys.as<K>(),
                                                       T.idx.as<int>(), T.sp.as<double4>(), overflow);
    return FGA_OK;
  };
  TRY_RC(sort_top(top_bits));
  // c_i, node counts, preorder offsets (rerun after a fallback)
  auto levels = [&]() -> int {
    k_count<<<blocks_for(n + 1), kThreads, 0, st>>>(T.keys.as<K>(), n, L,
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
    FGA_CUDA_TRY(T.keys_in.reserve(sizeof(K) * n));
    k_keys<K><<<blocks_for(n), kThreads, 0, st>>>(pts_dev, masses_dev, n, T.box.as<double>(), L, 0,
                                               nullptr, T.keys_in.as<K>(),
                                               T.idx_in.as<int>(), T.packed.as<double4>());
    tmp_bytes = T.cub_tmp.bytes;
    FGA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(
        T.cub_tmp.p, tmp_bytes, T.keys_in.as<K>(), T.keys.as<K>(),
        T.idx_in.as<int>(), T.idx.as<int>(), (int)n, 0, 3 * L, st));
    k_gather_sorted<K><<<blocks_for(n), kThreads, 0, st>>>(T.packed.as<double4>(), T.idx.as<int>(), n,
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
  const int nc = (nbs + kTScan - 1) / kTScan;
  const int64_t ncr = (int64_t)(L + 1) * nbs;
  Cross cr{};
  FGA_CUDA_TRY(T.cross.reserve(sizeof(Q4) * (2 * ncr + 2 * (int64_t)nbs + 2 * (int64_t)nc + 1) +
                               ncr * (2 * sizeof(int) + sizeof(double)) + 256));
  {
    char* q = T.cross.as<char>();  // (Q4 arrays first: 16 B alignment)
    cr.pst = (Q4*)q; q += sizeof(Q4) * ncr;
    cr.plE = (Q4*)q; q += sizeof(Q4) * ncr;
    cr.T = (Q4*)q; q += sizeof(Q4) * nbs;
    cr.Gi = (Q4*)q; q += sizeof(Q4) * nbs;
    cr.CS = (Q4*)q; q += sizeof(Q4) * nc;
    cr.CX = (Q4*)q; q += sizeof(Q4) * (nc + 1);
    cr.prlen = (double*)q; q += sizeof(double) * ncr;
    cr.prx = (int*)q; q += sizeof(int) * ncr;
    cr.prs = (int*)q;
  }
  k_subtrees<<<nbs, kST, 0, st>>>(T.keys.as<K>(), n, L, T.clev.as<signed char>(),
                                  T.offset.as<int>(), T.box.as<double>(), T.sp.as<double4>(),
                                  T.records(), cr, nbs);
  if (nbs > 1) {
    k_tscan1<<<nc, kTScan, 0, st>>>(nbs, cr);
    k_tscan2<<<1, kTScan, 0, st>>>(nc, cr);
    k_crossing<<<(int)((ncr + 255) / 256), 256, 0, st>>>(L, nbs, n, T.keys.as<K>(),
                                                         T.offset.as<int>(), T.box.as<double>(), cr,
                                                         T.records());
  }
  FGA_CUDA_TRY(cudaGetLastError());
  T.exportable = true;
  if (T.L_requested > L) {  // cells at the 42-level cap: one sync, rare path
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
  auto exp = [&](auto* keys) {
    k_export<<<blocks_for(T.n_points), 256, 0, st>>>(
        keys, T.n_points, T.L, T.clev.as<signed char>(), T.offset.as<int>(), T.box.as<double>(),
        T.a64.as<double4>(), children ? d_children : nullptr, com ? d_com : nullptr,
        mass ? d_mass : nullptr, length ? d_len : nullptr, occupancy ? d_occ : nullptr,
        depth ? d_depth : nullptr, bmin ? d_bmin : nullptr, bmax ? d_bmax : nullptr);
  };
  if (T.wide_keys) exp(T.keys.as<K128>());
  else exp(T.keys.as<K64>());
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
