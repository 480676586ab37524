// fga_device.cuh -- device building blocks shared by the kernel files
// (forces.cu: single-pair force passes; batched.cu: the persistent
// many-pair registration kernel).  Everything here is header-local
// (anonymous namespace per translation unit).
#pragma once
#include <climits>

#include "fga_session.cuh"

namespace fga {
namespace {

constexpr int kWin = 32;
constexpr int kNumSMs = 148;
constexpr int kWarps = kForceThreads / 32;
constexpr int kTile = 1024;

struct Win32 {
  float4 a[kWin];
  NodeB32 b[kWin];
};

// exact fp64 MAC of the reference (_kernels.py:26-29, :37)
__device__ __noinline__ bool mac_exact(const double4* __restrict__ A64,
                                       const NodeB64* __restrict__ B64, int node, double qx,
                                       double qy, double qz, double theta2) {
  const double4 a = A64[node];
  const double dx = __dsub_rn(qx, a.x), dy = __dsub_rn(qy, a.y), dz = __dsub_rn(qz, a.z);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return B64[node].l2 < __dmul_rn(theta2, d2);
}

__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// band of a node (see the guard note below); -inf for a leaf (l2 = -inf),
// so a leaf is never re-checked.  gA = 1.25*2 sqrt3 delta theta, gB = the
// delta^2 term.
__device__ __forceinline__ float node_band(float l2, float gA, float gB) {
  const float len = l2 > 0.f ? l2 * rsqrt_approx(l2) : 0.f;
  return fmaf(gA, len, fmaf(13.0f * 5.97e-8f, l2, gB));
}

// numpy's float64 sum of a contiguous 1-D array (pairwise_sum_DOUBLE,
// numpy umath loops_utils.h.src), bit for bit: n < 8 sequential from 0;
// n <= 128 eight interleaved accumulators combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the n%8 tail; larger n split at
// n/2 - (n/2)%8.
__device__ __noinline__ double np_pairwise_sum(const double* __restrict__ a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; i++) r = __dadd_rn(r, a[i]);
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sum(a, n2), np_pairwise_sum(a + n2, n - n2));
}

// The recursion node (lo, len) reached from the root by the d path bits of t
// (most significant = first split).
__device__ __forceinline__ void np_pairwise_node(int64_t n, int d, int64_t t, int64_t& lo,
                                                 int64_t& len) {
  lo = 0;
  len = n;
  for (int l = d - 1; l >= 0; l--) {
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    if ((t >> l) & 1) {
      lo += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
}

// depth (<= dmax) down to which every node of the recursion is internal
__device__ __forceinline__ int np_pairwise_depth(int64_t n, int dmax) {
  int64_t sz[8] = {n};
  int cnt = 1, d = 0;
  while (d < dmax) {
    int64_t mn = sz[0];
    for (int k = 1; k < cnt; k++) mn = mn < sz[k] ? mn : sz[k];
    if (mn <= 128) break;
    int64_t nx[8];
    int nc = 0;
    for (int k = 0; k < cnt; k++) {
      int64_t n2 = sz[k] / 2;
      n2 -= n2 % 8;
      const int64_t c2[2] = {n2, sz[k] - n2};
      for (int q = 0; q < 2; q++) {
        bool seen = false;
        for (int u = 0; u < nc; u++) seen |= nx[u] == c2[q];
        if (!seen && nc < 8) nx[nc++] = c2[q];
      }
    }
    for (int k = 0; k < nc; k++) sz[k] = nx[k];
    cnt = nc;
    d++;
  }
  return d;
}

// Blocked summation of the FP32 force: the per-lane fp32 partial is folded
// into an fp64 sum whenever the warp's node index passes the next multiple of
// FGA_FOLD, so no fp32 sum runs over more than one chunk's terms.
// tools/fp32_error.py (configs[2], 16k queries): one fp32 running sum over the
// ~5.5k terms of a query limits the per-query error to 5.5e-5 relative;
// folding every 4096 node indices into fp64 gives 2.0e-6 (fp32 terms summed
// exactly: 0.9e-6).  The test rides on the loop's exit check, so it costs
// nothing per step.
#ifndef FGA_FOLD
#define FGA_FOLD 4096
#endif
static_assert(FGA_FOLD >= 0, "FGA_FOLD: node-index chunk of the blocked force sum (0 = off)");
__device__ __forceinline__ int fold_limit(int n, int n_nodes) {
  if (FGA_FOLD <= 0) return n_nodes;
  const int next = (n / FGA_FOLD + 1) * FGA_FOLD;
  return next < n_nodes ? next : n_nodes;
}

struct NodeC32 {
  float4 a, b;
};

struct Trav32Out {
  double ax, ay, az;  // sum of m * (com - q) / r^3, fp32 terms, blocked sum
  int visits, accepted;
};

// FP32 warp-coherent traversal.  All 32 lanes must call it (inactive lanes
// pass active=false).  Branch-free step: every lane evaluates the node at the
// warp-minimum cursor and the results are committed only on the lanes whose
// cursor is that node (SIMT issues the instructions once per warp either way,
// so predication is cheaper than divergent branches + reconvergence).
//
// Exact-MAC guard: with q and com rounded to fp32 (each coordinate off by at
// most delta = (|q|max + |com|max) * 2^-24) the fp32 d^2 differs from the
// fp64 one by at most err(d) = 2*delta*(|dx|+|dy|+|dz|) + 3*delta^2 + 4u*d^2.
// The fp32 decision can only be wrong when |theta^2 d^2 - l^2| <= err(d)
// (the exact difference has the other sign), which pins D = theta*|d| to
// within ~2 sqrt3 delta theta of len.  There err(d) <= 2 sqrt3 delta theta len
// + 21 delta^2 theta^2 + 13u l^2, so one band per node,
//   band = 1.25*(2 sqrt3 delta theta) len + 13u l^2 + 1.25*27 delta^2 theta^2,
// computed when the node enters the window, covers every wrong decision:
// inside it the decision is re-made exactly in fp64 from the fp64 records,
// so the accepted set always equals the reference's (_kernels.py:37).
// delta is the warp maximum, so the band is warp-uniform per node.
struct WinRec32 {
  float4 a;  // com.xyz, mass
  float4 b;  // l2 | -inf, skip (int bits), band, unused
};
struct WinBuf32 {
  WinRec32 r[kWin];
};

// kW: nodes per window refill (<= 32); 0 = no window, every step reads the
// node with one warp-uniform (broadcast) load through L1.
template <bool kGuardZero, int kW = kWin>
__device__ __forceinline__ Trav32Out traverse32(const float4* __restrict__ A,
                                                const NodeB32* __restrict__ B,
                                                const double4* __restrict__ A64,
                                                const NodeB64* __restrict__ B64, int n_nodes,
                                                float qx, float qy, float qz, bool active,
                                                float theta2, double theta2_64, float eps2,
                                                float gA, float gB, const double* qpx,
                                                const double* qpy, const double* qpz, int64_t qi,
                                                WinBuf32* win, int lane) {
  float ax = 0.f, ay = 0.f, az = 0.f;     // the current chunk's partial force
  double hx = 0.0, hy = 0.0, hz = 0.0;  // folded chunks
  int visits = 0, accepted = 0;
  int cursor = active ? 0 : n_nodes;
  int wbase = INT_MIN / 2;
  const int64_t qs = active ? qi : 0;  // inactive lanes join the exact re-check
  // one band per warp: the largest lane delta (inactive lanes pass 0)
  gA = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(gA)));
  gB = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(gB)));
  int lim = fold_limit(0, n_nodes);
  while (true) {
    const int n = __reduce_min_sync(0xffffffffu, cursor);
    if (n >= lim) {  // exit, or fold the chunk's partial into the running sum
      if (n >= n_nodes) break;
      hx += (double)ax;
      hy += (double)ay;
      hz += (double)az;
      ax = ay = az = 0.f;
      lim = fold_limit(n, n_nodes);
    }
    float4 a, b;
    if constexpr (kW == 0) {
      a = __ldg(&A[n]);
      const float2 nb = __ldg(reinterpret_cast<const float2*>(B) + n);
      b = make_float4(nb.x, nb.y, node_band(nb.x, gA, gB), 0.f);
    } else {
      if ((unsigned)(n - wbase) >= (unsigned)kW) {
        wbase = n;
        __syncwarp();
        const int j = n + lane;
        if (lane < kW && j < n_nodes) {
          const float4 ga = __ldg(&A[j]);
          const NodeB32 gb = B[j];
          win->r[lane].a = ga;
          win->r[lane].b = make_float4(gb.l2, __int_as_float(gb.skip), node_band(gb.l2, gA, gB), 0.f);
        }
        __syncwarp();
      }
      const WinRec32& rec = win->r[n - wbase];
      a = rec.a;
      b = rec.b;
    }
    const bool mine = cursor == n;
    const float dx = a.x - qx, dy = a.y - qy, dz = a.z - qz;
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float t2d2 = theta2 * d2;
    bool acc = b.x < t2d2;
    const bool near = mine && fabsf(t2d2 - b.x) <= b.z;
    if (__any_sync(0xffffffffu, near)) {  // warp-uniform branch, rarely taken
      // every lane makes the (cheap, L2-resident) exact check so the call is
      // not divergent; only the near lanes use it
      const bool e = mac_exact(A64, B64, n, qpx[qs], qpy[qs], qpz[qs], theta2_64);
      acc = near ? e : acc;
    }
    const bool take = mine && acc;
    const float r2 = d2 + eps2;
    const float inv = rsqrt_approx(r2);
    float w = a.w * (inv * inv * inv);
    if (!take) w = 0.f;
    if (kGuardZero && !(r2 > 0.f)) w = 0.f;  // reference skips d2+eps2 == 0 (:39)
    ax = fmaf(w, dx, ax);
    ay = fmaf(w, dy, ay);
    az = fmaf(w, dz, az);
    asm("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %2, 0;\n\tsetp.ne.b32 q, %3, 0;\n\t"
        "@p add.s32 %0, %0, 1;\n\t@q add.s32 %1, %1, 1;\n\t}"
        : "+r"(visits), "+r"(accepted) : "r"((int)mine), "r"((int)take));
    const int next = acc ? __float_as_int(b.y) : n + 1;
    cursor = mine ? next : cursor;
  }
  return Trav32Out{hx + (double)ax, hy + (double)ay, hz + (double)az, visits, accepted};
}

// Direct FP32 traversal (the single-pair force passes, forces.cu): every step
// reads node n's packed 32 B record (TreeRecords::c32) with two warp-uniform
// (broadcast) loads through L1 -- consecutive nodes share cache lines and the
// warps of an SM walk neighbouring regions -- instead of staging a 32-node
// window through shared memory (a per-lane LDG + 2 STS refill on ~37% of the
// steps: 15.85 -> 14.1 ms per 1M iteration).  The record carries this
// launch's guard band and l^2 + theta^2 eps^2 (launch_node_bands), so the MAC
// is one FFMA on d^2 + eps^2 (which the force needs anyway):
//   diff = theta^2 (d^2 + eps^2) - (l^2 + theta^2 eps^2),
// accept iff diff > 0, and re-decide in fp64 iff |diff| <= band (14.1 ->
// 13.5 ms).  Visits are counted only when asked (kCountVisits; 2.5% of the
// step).
// kStatic (the wide batched kernels, batched.cu): the records are static,
// {l^2 | -inf, skip, length, 0}, and the band is formed per step from the
// warp's coefficients gA / gB (guard_coeffs) -- no per-launch band pass;
// qidx >= 0 gives the re-check's query index explicitly.
// kSmem: C points to the records copied into shared memory (small trees,
// k_bh_iterate_small); plain loads instead of the read-only global path
// kRange: only the nodes in [lo, hi) contribute (a part of a split warp,
// k_bh_split): the walk to lo jumps every subtree that ends at or before lo
// and re-decides the chain spanning lo by the same MAC without counting it.
// kTrace: records the warp's node index every 256 steps (trace[0..63]) and
// its step count (trace[64]) -- the split points of later passes.
// kSteps: only the step count (trace[64]).
template <bool kGuardZero, bool kCountVisits, bool kStatic = false, bool kSmem = false,
          bool kRange = false, bool kTrace = false, bool kSteps = false>
__device__ __forceinline__ Trav32Out traverse32d(const float4* __restrict__ C,
                                                 const double4* __restrict__ A64,
                                                 const NodeB64* __restrict__ B64, int n_nodes,
                                                 float qx, float qy, float qz, bool active,
                                                 float theta2, double theta2_64, float eps2,
                                                 const double* qpx, const double* qpy,
                                                 const double* qpz, int64_t m_queries,
                                                 double* hs = nullptr, float gA = 0.f,
                                                 float gB = 0.f, int64_t qidx = -1,
                                                 unsigned* hc = nullptr,
                                                 const double* qsh = nullptr, int lo = 0,
                                                 int hi = -1, int* trace = nullptr,
                                                 const int* border = nullptr) {
  // border (optional): the block -> chunk order of the launch (the query of
  // the exact re-check is chunk * blockDim + thread)
  // qsh (optional): the lanes' fp64 queries in shared memory (3 per thread)
  // for the exact re-check, instead of pointers + index held across the loop
  // hs (optional): the block's fp64 fold sums in shared memory, 3 per thread
  // (hs[3 threadIdx.x ..]), so they hold no registers across the loop (folds
  // are rare; the address is re-derived at each fold)
  float ax = 0.f, ay = 0.f, az = 0.f;     // the current chunk's partial force
  double hx = 0.0, hy = 0.0, hz = 0.0;  // folded chunks
  if (hs) {
    double* h = hs + 3 * threadIdx.x;
    h[0] = h[1] = h[2] = 0.0;
  }
  int visits = 0, accepted = 0;
  // kPacked (counting visits with hc given): one register holds (visits <<
  // 16) | accepted of the current fold chunk -- at most FGA_FOLD node indices,
  // each visited at most once -- and the folds add it to the per-thread
  // totals in shared memory (hc[2 threadIdx.x ..])
  // a split part counts visits in plain registers (the operator's split
  // passes, forces.cu k_bh_op_split): nodes before lo are not its visits
  constexpr bool kPackable = kCountVisits && !kRange && FGA_FOLD > 0 && FGA_FOLD <= 65535;
  const bool packed = kPackable && hc != nullptr;
  unsigned cnt = 0;
  if (packed) hc[2 * threadIdx.x] = hc[2 * threadIdx.x + 1] = 0u;
  int cursor = active ? 0 : n_nodes;
  if constexpr (kStatic) {  // one band per warp: the largest lane delta
    gA = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(gA)));
    gB = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(gB)));
  }
  const int end = (kRange && hi >= 0) ? hi : n_nodes;
  int lim = fold_limit(0, end);
  int steps = 0;  // (kTrace)
  // kSmem (one latency-bound wave, records in shared memory): the next n is
  // one vote after the MAC, the other lanes' minimum computed off the chain
  // (1M, issue-bound: 11.6 -> 13.0 ms, so the REDUX-at-top form stays there;
  // configs[0]: loop 1.61 -> 1.50 ms)
  constexpr bool kVote = kSmem;
  int n = __reduce_min_sync(0xffffffffu, cursor);
  while (true) {
    if (!kVote) n = __reduce_min_sync(0xffffffffu, cursor);
    if constexpr (kTrace) {
      if ((steps & 255) == 0 && (threadIdx.x & 31) == 0 && (steps >> 8) < 64) trace[steps >> 8] = n;
    }
    if constexpr (kTrace || kSteps) steps++;
    if (n >= lim) {  // exit, or fold the chunk's partial into the fp64 sum
      if (n >= end) break;
      if (hs) {
        double* h = hs + 3 * threadIdx.x;
        h[0] += (double)ax;
        h[1] += (double)ay;
        h[2] += (double)az;
      } else {
        hx += (double)ax;
        hy += (double)ay;
        hz += (double)az;
      }
      ax = ay = az = 0.f;
      if (kPackable && packed) {
        unsigned* hcc = hc + 2 * threadIdx.x;
        hcc[0] += cnt >> 16;
        hcc[1] += cnt & 0xffffu;
        cnt = 0;
      }
      lim = fold_limit(n, end);
    }
    FGA_CHECK(n >= 0 && n < n_nodes);
    const NodeC32* rec = reinterpret_cast<const NodeC32*>(C) + n;
    const float4 a = kSmem ? rec->a : __ldg(&rec->a);
    const float4 b = kSmem ? rec->b : __ldg(&rec->b);
    const bool mine = cursor == n;
    bool pre = false;  // (kRange) a node before lo: decides the walk, adds nothing
    if constexpr (kRange) {
      if (n < lo) {
        const int skp = __float_as_int(b.y);
        if (skp <= lo) {  // its whole subtree lies before lo (warp-uniform)
          if (mine) cursor = skp;
          continue;
        }
        pre = true;
      }
    }
    // (kVote) the other lanes' cursors do not move this step
    const int m_other = kVote ? __reduce_min_sync(0xffffffffu, mine ? INT_MAX : cursor) : 0;
    const float dx = a.x - qx, dy = a.y - qy, dz = a.z - qz;
    float r2, diff, band;
    if constexpr (kStatic) {
      const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      diff = fmaf(theta2, d2, -b.x);
      band = fmaf(gA, b.z, fmaf(13.0f * 5.97e-8f, b.x, gB));
      r2 = d2 + eps2;
    } else {
      r2 = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, eps2)));  // d^2 + eps^2
      diff = fmaf(theta2, r2, -b.x);
      band = b.z;
    }
    bool acc = diff > 0.f;
    const bool near = mine && fabsf(diff) <= band;
    if (__any_sync(0xffffffffu, near)) {  // warp-uniform branch, rarely taken
      // this lane's query, re-derived here (query i = global thread index;
      // inactive lanes read the last query and ignore the result) so no
      // register holds it across the loop
      bool e;
      if (qsh) {
        const double* q = qsh + 3 * threadIdx.x;
        e = mac_exact(A64, B64, n, q[0], q[1], q[2], theta2_64);
      } else {
        const int64_t blk = border ? border[blockIdx.x] : blockIdx.x;
        int64_t qs = qidx >= 0 ? qidx : blk * (int64_t)blockDim.x + threadIdx.x;
        qs = qs < m_queries ? qs : m_queries - 1;
        e = mac_exact(A64, B64, n, qpx[qs], qpy[qs], qpz[qs], theta2_64);
      }
      acc = near ? e : acc;
    }
    const bool take = mine && acc && !pre;
    const float inv = rsqrt_approx(r2);
    float w = a.w * (inv * inv * inv);
    if (!take) w = 0.f;
    if (kGuardZero && !(r2 > 0.f)) w = 0.f;  // reference skips d2+eps2 == 0 (:39)
    ax = fmaf(w, dx, ax);
    ay = fmaf(w, dy, ay);
    az = fmaf(w, dz, az);
    if (kPackable && packed) {
      asm("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %1, 0;\n\tsetp.ne.b32 q, %2, 0;\n\t"
          "@p add.u32 %0, %0, 65536;\n\t@q add.u32 %0, %0, 1;\n\t}"
          : "+r"(cnt) : "r"((int)mine), "r"((int)take));
    } else if constexpr (kCountVisits) {
      asm("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %2, 0;\n\tsetp.ne.b32 q, %3, 0;\n\t"
          "@p add.s32 %0, %0, 1;\n\t@q add.s32 %1, %1, 1;\n\t}"
          : "+r"(visits), "+r"(accepted) : "r"((int)(mine && !pre)), "r"((int)take));
    } else {
      asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t@q add.s32 %0, %0, 1;\n\t}"
          : "+r"(accepted) : "r"((int)take));
    }
    const int next = acc ? __float_as_int(b.y) : n + 1;
    cursor = mine ? next : cursor;
    if (kVote)
      n = __any_sync(0xffffffffu, mine && !acc) ? n + 1 : min(__float_as_int(b.y), m_other);
  }
  if constexpr (kTrace || kSteps) {
    if ((threadIdx.x & 31) == 0) trace[64] = steps;
  }
  if (kPackable && packed) {
    const unsigned* hcc = hc + 2 * threadIdx.x;
    visits = (int)(hcc[0] + (cnt >> 16));
    accepted = (int)(hcc[1] + (cnt & 0xffffu));
  }
  if (hs) {
    const double* h = hs + 3 * threadIdx.x;
    hx = h[0];
    hy = h[1];
    hz = h[2];
  }
  return Trav32Out{hx + (double)ax, hy + (double)ay, hz + (double)az, visits, accepted};
}

struct Trav64Out {
  double fx, fy, fz;
  int visits, accepted;
};

// FP64 traversal: the reference's arithmetic and order exactly (gq = G*m_q),
// each node's records read straight from global memory (warp-uniform
// addresses: one L1 request per record per step; round 1 staged them through
// a per-warp shared window that every skip past its end refilled: 30.3 ->
// 28.6 ms at 1M).
// trace (optional): the warp's step count -> trace[64] (the launch order of
// later passes, forces.cu k_block_work)
__device__ __forceinline__ Trav64Out traverse64d(const double4* __restrict__ A,
                                                 const NodeB64* __restrict__ B, int n_nodes,
                                                 double qx, double qy, double qz, double gq,
                                                 bool active, double theta2, double eps2,
                                                 int* trace = nullptr) {
  Trav64Out o{0.0, 0.0, 0.0, 0, 0};
  int cursor = active ? 0 : n_nodes;
  int steps = 0;
  while (true) {
    const int n = __reduce_min_sync(0xffffffffu, cursor);
    if (n >= n_nodes) break;
    steps++;
    const double2 a01 = __ldg(reinterpret_cast<const double2*>(A + n));
    const double2 a23 = __ldg(reinterpret_cast<const double2*>(A + n) + 1);
    const double4 a = make_double4(a01.x, a01.y, a23.x, a23.y);
    const double2 bb = __ldg(reinterpret_cast<const double2*>(B) + n);
    if (cursor == n) {
      const double dx = __dsub_rn(qx, a.x), dy = __dsub_rn(qy, a.y), dz = __dsub_rn(qz, a.z);
      const double d2 =
          __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      o.visits++;
      if (bb.x < __dmul_rn(theta2, d2)) {
        o.accepted++;
        const double denom = __dadd_rn(d2, eps2);
        if (denom > 0.0) {
          const double w = __ddiv_rn(__dmul_rn(gq, a.w), __dmul_rn(denom, __dsqrt_rn(denom)));
          o.fx = __dsub_rn(o.fx, __dmul_rn(w, dx));
          o.fy = __dsub_rn(o.fy, __dmul_rn(w, dy));
          o.fz = __dsub_rn(o.fz, __dmul_rn(w, dz));
        }
        cursor = (int)__double_as_longlong(bb.y);
      } else {
        cursor = n + 1;
      }
    }
  }
  if (trace && (threadIdx.x & 31) == 0) trace[64] = steps;
  return o;
}

// Per-lane guard coefficients (see traverse32): band(node) = gA*len + kRel*l2 + gB.
__device__ __forceinline__ void guard_coeffs(float qmag, float cmag, float theta2, float& gA,
                                             float& gB) {
  const float delta = (qmag + cmag) * 5.97e-8f;
  gA = 4.34f * delta * sqrtf(theta2);         // 1.25 * 2 sqrt3 delta theta
  gB = 34.f * delta * delta * theta2 + 1e-37f;  // 1.25 * 27 delta^2 theta^2
}

// ---------------------------------------------------------------- iterate epilogue
struct Partial {
  double v[17];
};

__device__ __forceinline__ void partial_zero(Partial& p) {
#pragma unroll
  for (int k = 0; k < 17; k++) p.v[k] = 0.0;
}

// Applies R,t of the previous step to (y, v') in place (registration.py:135-136).
__device__ __forceinline__ void apply_pending(const IterState* st, double y[3], double v[3]) {
  double ny[3], nv[3];
#pragma unroll
  for (int r = 0; r < 3; r++) {
    ny[r] = st->Rp[3 * r] * y[0] + st->Rp[3 * r + 1] * y[1] + st->Rp[3 * r + 2] * y[2] + st->tp[r];
    nv[r] = st->Rp[3 * r] * v[0] + st->Rp[3 * r + 1] * v[1] + st->Rp[3 * r + 2] * v[2];
  }
#pragma unroll
  for (int r = 0; r < 3; r++) {
    y[r] = ny[r];
    v[r] = nv[r];
  }
}

// total_force + step (dynamics.py:40, :45-46) in the reference's operation
// order, then this query's contribution to the Kabsch sums.
__device__ __forceinline__ void step_and_accumulate(const double F[3], const double y[3],
                                                    const double v[3], double mq,
                                                    const SimParams& sp, const double s[3],
                                                    double vp[3], Partial& p) {
  double w[3], u[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const double f = __dsub_rn(F[k], __dmul_rn(sp.eta, v[k]));
    vp[k] = __dadd_rn(v[k], __ddiv_rn(__dmul_rn(sp.dt, f), mq));
    const double d = __dmul_rn(sp.dt, vp[k]);
    u[k] = y[k] - s[k];
    w[k] = (y[k] + d) - s[k];
  }
#pragma unroll
  for (int k = 0; k < 3; k++) {
    p.v[kSumU + k] += u[k];
    p.v[kSumW + k] += w[k];
  }
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) p.v[kSumWU + 3 * i + j] = fma(w[i], u[j], p.v[kSumWU + 3 * i + j]);
}

__device__ __forceinline__ void warp_store_partial(Partial& p, int lane, double* out) {
#pragma unroll
  for (int k = 0; k < 17; k++) p.v[k] = warp_sum(p.v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 17; k++) out[k] = p.v[k];
    out[17] = 0.0;
  }
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fma2s(float s, float2 b, float2 c) {  // s*b + c
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%2};\n\tmov.b64 rb, {%3,%4};\n\t"
      "mov.b64 rc, {%5,%6};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(s), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// K11 energy.  Per pair: |y - x| (MUFU.SQRT) and 1/(|y - x| + eps).  The two
// MUFU ops per pair make the scalar kernel MUFU-bound (16/clk/SM), so half of
// the pairs (pack 1) compute the reciprocal on the FMA pipe instead: a
// bit-trick seed and three Newton steps on w = -1/x (w' = w (2 + x w), error
// 0.125^8 ~ 6e-8), in packed FP32x2 arithmetic.  FP32 within a tile, fp64
// across tiles and across queries (<= 1e-6 relative, tested).
// ---- packed FP32x2 arithmetic (sm_100 FFMA2/FADD2/FMUL2): two queries per
// instruction, which halves the issue slots of the FP32 inner loops (they are
// issue-bound with scalar FP32: ncu showed 84% issue-slot utilisation at 56%
// of FP32 peak).  A scalar operand {s, s} becomes the .F32 broadcast form.
__device__ __forceinline__ float2 sub2s(float s, float2 q) {  // s - q
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%2};\n\tmov.b64 rb, {%3,%4};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(s), "f"(q.x), "f"(q.y));
  return d;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mov.b64 rc, {%6,%7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 mul2s(float s, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%2};\n\tmov.b64 rb, {%3,%4};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(s), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 add2s(float2 a, float s) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%4};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(s));
  return d;
}

// FP32 tile loop: P packs of 2 queries against jmax staged sources
// {x, y, z, m}.  Per source and pack: 3 FADD2, 3 FFMA2 (r^2 + eps^2),
// 2 MUFU.RSQ, 3 FMUL2 (m r^-3), 3 FFMA2 (accumulate) = 20 FLOP per pair in
// 7 issue slots per pair.  kGuard handles eps == 0 (coincident points).
template <int P, bool kGuard>
__device__ __forceinline__ void direct_tile32(const float4* __restrict__ sm, int jmax,
                                              const float2 (&qx)[P], const float2 (&qy)[P],
                                              const float2 (&qz)[P], float eps2,
                                              float2 (&ax)[P], float2 (&ay)[P],
                                              float2 (&az)[P]) {
  const float2 e2 = make_float2(eps2, eps2);
#pragma unroll 4
  for (int j = 0; j < jmax; j++) {
    const float4 s = sm[j];
#pragma unroll
    for (int k = 0; k < P; k++) {
      const float2 dx = sub2s(s.x, qx[k]), dy = sub2s(s.y, qy[k]), dz = sub2s(s.z, qz[k]);
      const float2 r2 = fma2(dx, dx, fma2(dy, dy, fma2(dz, dz, e2)));
      float2 inv;
      inv.x = rsqrt_approx(r2.x);
      inv.y = rsqrt_approx(r2.y);
      float2 w = mul2(mul2s(s.w, inv), mul2(inv, inv));
      if (kGuard) {
        if (!(r2.x > 0.f)) w.x = 0.f;
        if (!(r2.y > 0.f)) w.y = 0.f;
      }
      ax[k] = fma2(w, dx, ax[k]);
      ay[k] = fma2(w, dy, ay[k]);
      az[k] = fma2(w, dz, az[k]);
    }
  }
}

// fp64 brute force term (bhtree.py:158-164): w = m / d2^1.5, sum w*delta.
__device__ __forceinline__ void direct_tile64(const double4* __restrict__ sm, int jmax, double qx,
                                              double qy, double qz, double eps2, double& sx,
                                              double& sy, double& sz) {
  for (int j = 0; j < jmax; j++) {
    const double4 s = sm[j];
    const double dx = __dsub_rn(qx, s.x), dy = __dsub_rn(qy, s.y), dz = __dsub_rn(qz, s.z);
    const double d2 = __dadd_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)), eps2);
    const double w = d2 > 0.0 ? __ddiv_rn(s.w, __dmul_rn(d2, __dsqrt_rn(d2))) : 0.0;
    sx = __dadd_rn(sx, __dmul_rn(w, dx));
    sy = __dadd_rn(sy, __dmul_rn(w, dy));
    sz = __dadd_rn(sz, __dmul_rn(w, dz));
  }
}

// K11 energy inner loop: 2*NP queries (NP packs of 2) against jmax staged
// sources.  Even packs use MUFU sqrt+rcp; odd packs take the reciprocal on
// the FMA pipe (bit-trick seed + 3 Newton steps on w = -1/x, accumulating
// -m/x), which balances the MUFU and FMA pipes.  acc[k] += +-sum m/(d+eps).
template <bool kNewton, int NP>
__device__ __forceinline__ void gpe_tile32(const float4* __restrict__ sm, int jmax,
                                           const float2 (&qx)[NP], const float2 (&qy)[NP],
                                           const float2 (&qz)[NP], float eps,
                                           float2 (&acc)[NP]) {
  const float2 e2 = make_float2(eps, eps);
  const float2 two = make_float2(2.f, 2.f);
#pragma unroll 2
  for (int j = 0; j < jmax; j++) {
    const float4 s = sm[j];
#pragma unroll
    for (int k = 0; k < NP; k++) {
      const float2 dx = sub2s(s.x, qx[k]), dy = sub2s(s.y, qy[k]), dz = sub2s(s.z, qz[k]);
      const float2 d2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
      float2 den;
      den.x = sqrt_approx(d2.x);
      den.y = sqrt_approx(d2.y);
      den = add2(den, e2);
      float2 w;
      if (kNewton && (k & 1)) {
        w.x = __int_as_float(0xFEF311C3u - __float_as_uint(den.x));
        w.y = __int_as_float(0xFEF311C3u - __float_as_uint(den.y));
#pragma unroll
        for (int it = 0; it < 3; it++) w = mul2(w, fma2(den, w, two));
      } else {
        w.x = rcp_approx(den.x);
        w.y = rcp_approx(den.y);
      }
      acc[k] = fma2s(s.w, w, acc[k]);
    }
  }
}

// ---------------------------------------------------------------- rigid
// ------------------------------------------------------------------ 3x3 SVD
// One-sided Jacobi on the columns of A (3x3, row-major): A V = U S.
__device__ void svd3(const double C[9], double U[9], double S[3], double V[9]) {
  double A[9];
  for (int k = 0; k < 9; k++) A[k] = C[k];
  for (int k = 0; k < 9; k++) V[k] = (k % 4 == 0) ? 1.0 : 0.0;
  const int P[3] = {0, 0, 1}, Q[3] = {1, 2, 2};
  for (int sweep = 0; sweep < 30; sweep++) {
    double off = 0.0;
    for (int r = 0; r < 3; r++) {
      const int p = P[r], q = Q[r];
      double alpha = 0.0, beta = 0.0, gamma = 0.0;
      for (int k = 0; k < 3; k++) {
        alpha += A[3 * k + p] * A[3 * k + p];
        beta += A[3 * k + q] * A[3 * k + q];
        gamma += A[3 * k + p] * A[3 * k + q];
      }
      if (gamma == 0.0) continue;
      const double rel = fabs(gamma) / sqrt(alpha * beta);
      off = fmax(off, rel);
      if (!(rel > 1e-17)) continue;
      const double zeta = (beta - alpha) / (2.0 * gamma);
      const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
      const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
      for (int k = 0; k < 3; k++) {
        const double ap = A[3 * k + p], aq = A[3 * k + q];
        A[3 * k + p] = c * ap - s * aq;
        A[3 * k + q] = s * ap + c * aq;
        const double vp = V[3 * k + p], vq = V[3 * k + q];
        V[3 * k + p] = c * vp - s * vq;
        V[3 * k + q] = s * vp + c * vq;
      }
    }
    if (off < 1e-16) break;
  }
  // singular values = column norms, sorted descending (LAPACK order)
  int ord[3] = {0, 1, 2};
  double nrm[3];
  for (int j = 0; j < 3; j++)
    nrm[j] = sqrt(A[j] * A[j] + A[3 + j] * A[3 + j] + A[6 + j] * A[6 + j]);
  for (int a = 0; a < 2; a++)
    for (int b = 0; b < 2 - a; b++)
      if (nrm[ord[b]] < nrm[ord[b + 1]]) {
        int tmp = ord[b];
        ord[b] = ord[b + 1];
        ord[b + 1] = tmp;
      }
  double Vs[9];
  for (int j = 0; j < 3; j++) {
    S[j] = nrm[ord[j]];
    for (int k = 0; k < 3; k++) {
      Vs[3 * k + j] = V[3 * k + ord[j]];
      U[3 * k + j] = S[j] > 0.0 ? A[3 * k + ord[j]] / S[j] : 0.0;
    }
  }
  for (int k = 0; k < 9; k++) V[k] = Vs[k];
  // Orthonormal completion: u1 normalized, u2 Gram-Schmidt, u3 = u1 x u2.
  double u1[3] = {U[0], U[3], U[6]}, u2[3] = {U[1], U[4], U[7]};
  double n1 = sqrt(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]);
  if (!(n1 > 0.0)) {
    u1[0] = 1.0;
    u1[1] = u1[2] = 0.0;
    n1 = 1.0;
  }
  for (int k = 0; k < 3; k++) u1[k] /= n1;
  double d12 = u1[0] * u2[0] + u1[1] * u2[1] + u1[2] * u2[2];
  for (int k = 0; k < 3; k++) u2[k] -= d12 * u1[k];
  double n2 = sqrt(u2[0] * u2[0] + u2[1] * u2[1] + u2[2] * u2[2]);
  if (!(n2 > 1e-300)) {  // rank <= 1: any unit vector orthogonal to u1
    const int a = fabs(u1[0]) < 0.9 ? 0 : 1;
    double e[3] = {0, 0, 0};
    e[a] = 1.0;
    d12 = u1[a];
    for (int k = 0; k < 3; k++) u2[k] = e[k] - d12 * u1[k];
    n2 = sqrt(u2[0] * u2[0] + u2[1] * u2[1] + u2[2] * u2[2]);
  }
  for (int k = 0; k < 3; k++) u2[k] /= n2;
  const double u3[3] = {u1[1] * u2[2] - u1[2] * u2[1], u1[2] * u2[0] - u1[0] * u2[2],
                        u1[0] * u2[1] - u1[1] * u2[0]};
  for (int k = 0; k < 3; k++) {
    U[3 * k] = u1[k];
    U[3 * k + 1] = u2[k];
    U[3 * k + 2] = u3[k];
  }
}

__device__ __forceinline__ double det3(const double M[9]) {
  return M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
         M[2] * (M[3] * M[7] - M[4] * M[6]);
}

// procrustes.solve_rotation (procrustes.py:12-35) from the cross-covariance.
__device__ void kabsch_rotation(const double C[9], double R[9], int* degenerate) {
  double U[9], S[3], V[9];
  svd3(C, U, S, V);
  // sign(det(U Vt)) (:28-30); det(U) = +1 by construction
  double sgn = det3(V) < 0.0 ? -1.0 : 1.0;
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++)
      R[3 * i + j] = U[3 * i] * V[3 * j] + U[3 * i + 1] * V[3 * j + 1] + sgn * U[3 * i + 2] * V[3 * j + 2];
  if (degenerate) {
    const double tol = 1e-12 * fmax(S[0], 1e-300);  // _DEGENERATE_REL_TOL (:8)
    int rank = (S[0] > tol) + (S[1] > tol) + (S[2] > tol);
    *degenerate = rank < 2;
  }
}


// procrustes.solve_rotation for D = 2 (procrustes.py:12-35): the SVD
// solution U diag(1, sign det(U V^T)) V^T is the maximiser of tr(R^T C) over
// SO(2), i.e. the rotation by atan2(C10 - C01, C00 + C11).  C is the 3x3
// buffer of the z-padded problem; the result is embedded as diag(R2, 1).
__device__ void kabsch_rotation_2d(const double C[9], double R[9], int* degenerate) {
  const double c = C[0] + C[4], s = C[3] - C[1];
  const double h = sqrt(c * c + s * s);
  double cs = 1.0, sn = 0.0;
  if (h > 0.0) {
    cs = c / h;
    sn = s / h;
  }
  R[0] = cs;
  R[1] = -sn;
  R[2] = 0.0;
  R[3] = sn;
  R[4] = cs;
  R[5] = 0.0;
  R[6] = 0.0;
  R[7] = 0.0;
  R[8] = 1.0;
  if (degenerate) {  // singular values of the 2x2 block
    const double a = C[0], b = C[1], cc = C[3], d = C[4];
    const double s1 = sqrt((a + d) * (a + d) + (cc - b) * (cc - b));
    const double s2 = sqrt((a - d) * (a - d) + (cc + b) * (cc + b));
    const double smax = 0.5 * (s1 + s2), smin = 0.5 * fabs(s1 - s2);
    const double tol = 1e-12 * fmax(smax, 1e-300);
    *degenerate = ((smax > tol) + (smin > tol)) < 1;
  }
}

// ---------------------------------------------------------------- tree keys
__device__ __forceinline__ int common_levels(unsigned long long a, unsigned long long b, int L) {
  unsigned long long x = a ^ b;
  if (x == 0ull) return L;
  int lz = __clzll((long long)x) - (64 - 3 * L);
  return lz / 3;
}

__device__ __forceinline__ unsigned long long low_mask(int bits) {
  return bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
}

// Replays the bbox of the node at level `l` on the path of `key`.
__device__ __forceinline__ void node_bbox(unsigned long long key, int l, int L,
                                          const double* __restrict__ box, double lo[3],
                                          double hi[3]) {
#pragma unroll
  for (int k = 0; k < 3; k++) {
    lo[k] = box[k];
    hi[k] = box[3 + k];
  }
  for (int lev = 1; lev <= l; lev++) {
    unsigned digit = (unsigned)(key >> (3 * (L - lev))) & 7u;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      double c = __dadd_rn(lo[k], __dmul_rn(__dsub_rn(hi[k], lo[k]), 0.5));
      if ((digit >> (2 - k)) & 1u) lo[k] = c; else hi[k] = c;
    }
  }
}


// ---------------------------------------------------------------- NIV
// idx = clip(floor((p - a) / edge), 0, rho-1) with numpy's float->int64 cast
// (out-of-range values become INT64_MIN, then clip to 0).
__device__ __forceinline__ long long niv_axis(double p, double a, double edge, int rho) {
  const double f = floor(__ddiv_rn(__dsub_rn(p, a), edge));
  long long v;
  if (!(f >= -9.223372036854775808e18 && f < 9.223372036854775808e18)) v = LLONG_MIN;
  else v = (long long)f;
  return v < 0 ? 0 : (v > rho - 1 ? rho - 1 : v);
}


}  // namespace
}  // namespace fga
