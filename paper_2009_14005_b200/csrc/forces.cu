// forces.cu -- the per-iteration force pass (hot path).
//
// K6 Barnes-Hut traversal (reference: _kernels.bh_forces_kernel,
// _kernels.py:7-50).  Stackless and warp-coherent: every lane keeps a cursor
// into the mirrored-preorder node array; the warp repeatedly takes the
// smallest cursor n (redux.sync.min), the lanes whose cursor equals n apply
// their own MAC -- accept: cursor = skip[n]; open: cursor = n + 1 -- so each
// query visits exactly the reference's node set, in exactly the reference's
// order (the reference's stack pops slot 7 first, which is mirrored
// preorder).  Node records are staged per warp through a 32-node shared-memory
// window that one coalesced load refills whenever the warp's minimum cursor
// leaves it.
//   * FP32 path: positions/records in fp32, acceleration accumulated in fp32
//     registers; the MAC `l^2 < theta^2 d^2` (:37) is evaluated in fp32 and
//     re-evaluated exactly in fp64 whenever the fp32 margin is within the
//     rounding bound, so the accepted set is the reference's.
//   * FP64 path: the reference's per-term arithmetic verbatim (:26-42), no
//     FMA contraction, same order -> bit-identical forces on the same tree.
// The iterate kernels fuse: the pending rigid transform of the previous
// iteration (registration.py:135-136), damping + Euler-Cromer
// (dynamics.py:37-47) and the Kabsch partial sums (procrustes.py:20-25).
//
// K1 direct O(NM) sum (bhtree.brute_force, bhtree.py:155-164): reference
// points staged through shared memory as float4 {x,y,z,m} tiles of 1024,
// 2 queries per thread, FP32 FMA/MUFU inner loop, fp64 across tiles.
//
// K11 potential energy (_kernels.gpe_kernel, _kernels.py:53-67): same tiling.
#include <cub/cub.cuh>

#include <climits>
#include <cstdlib>

#include "fga_device.cuh"

namespace fga {
namespace {

// ---------------------------------------------------------------- BH iterate
struct F32Params {
  float theta2, eps2;
};

// Resident threads per SM.  The FP32 traversal is latency-bound on its
// record loads (ncu: 47% of stall samples at the first use of the loaded
// record, issue 66% active at 1280 threads), so more warps win even at 32
// registers with a spilled query coordinate (1M iteration, A/B on one box):
// 1024 threads 15.3 ms, 1280 13.2, 1536 12.4, 1792 11.6, 2048 11.6.  What
// gets it there: the fold sums live in shared memory and the exact re-check
// re-derives its query from the thread index (no register across the loop).
// Measured and not kept: the query in shared memory (15.3 ms at 1792),
// L1 prefetch of node n+1 (+1%) or of skip(n) (+7%).
// fp64 traversal: 768 -> 35.8 ms, 1024 -> 31.5, 1280 -> 30.3, 1536 -> 38 (spills)
#ifndef FGA_SPLIT_FRAC
// split passes whenever the warps fill <= this fraction of the resident slots
// (3,907 warps of an 8-way shard: 2.82 -> 2.30 ms; a cost-balanced shard of
// 4,168 warps: 2.76 -> 2.25 ms; 7,813 warps of a 4-way shard: slower)
#define FGA_SPLIT_FRAC 0.6
#endif
#ifndef FGA_BH32_TPS
#define FGA_BH32_TPS 1792
#endif
#ifndef FGA_BH64_TPS
#define FGA_BH64_TPS 1280
#endif
// kSmall: the whole FP32 record array is first copied into shared memory
// (trees up to kSmallTreeBytes; launched when the template is small enough
// that the pass is a few latency-bound warps per SM, e.g. configs[0]'s 2k
// points: every step's record load is then a shared-memory load instead of an
// L1/L2 round trip on a cold SM)
constexpr int kSmallTreeBytes = 200 * 1024;
template <typename Real, bool kGuardZero, bool kCountVisits, int kT, bool kSmall = false,
          bool kTrace = false>
__global__ void __launch_bounds__(kT, kSmall ? 1 : (sizeof(Real) == 4 ? FGA_BH32_TPS : FGA_BH64_TPS) / kT) k_bh_iterate(
    TreeRecords tr, int n_nodes, TemplateView tv, const IterState* __restrict__ st, SimParams sp,
    F32Params f, double* partials, int nblocks, int* trace = nullptr,
    const int* __restrict__ order = nullptr) {
  if (st->done) return;
  extern __shared__ float4 s_rec[];
  if constexpr (kSmall) {
    const int nv = 2 * n_nodes;
    for (int k = threadIdx.x; k < nv; k += kT) s_rec[k] = __ldg(tr.c32 + k);
    __syncthreads();
  }
  // (An SM-contiguous block->chunk remap for L1 sharing was measured 3%
  // slower -- per-SM load imbalance.)  With `order` the chunks run heaviest
  // first (the block->partial-slot map is unchanged: same sums)
  const int chunk = order ? order[blockIdx.x] : (int)blockIdx.x;
  if (chunk >= nblocks) return;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t gw = (int64_t)chunk * (kT / 32) + wl;
  const int64_t i = gw * 32 + lane;
  const bool active = i < tv.m;
  double y[3] = {0, 0, 0}, v[3] = {0, 0, 0}, mq = 1.0;
  if (active) {
    y[0] = tv.px[i];
    y[1] = tv.py[i];
    y[2] = tv.pz[i];
    v[0] = tv.vx[i];
    v[1] = tv.vy[i];
    v[2] = tv.vz[i];
    mq = tv.mq[i];
    apply_pending(st, y, v);
    tv.px[i] = y[0];
    tv.py[i] = y[1];
    tv.pz[i] = y[2];
    tv.vx[i] = v[0];
    tv.vy[i] = v[1];
    tv.vz[i] = v[2];
  }
  double F[3];
  int nv, na;
  if constexpr (sizeof(Real) == 4) {
    __shared__ double hs[3 * kT];  // the lanes' fp64 fold sums
    __shared__ unsigned hc[kCountVisits ? 2 * kT : 1];  // their visit / accept counts
    const Trav32Out o = traverse32d<kGuardZero, kCountVisits, false, kSmall, false, kTrace>(
        kSmall ? s_rec : tr.c32, tr.a64, tr.b64, n_nodes, (float)y[0], (float)y[1], (float)y[2], active, f.theta2,
        sp.theta2, f.eps2, tv.px, tv.py, tv.pz, tv.m, hs, 0.f, 0.f, -1,
        kCountVisits ? hc : nullptr, nullptr, 0, -1, kTrace ? trace + gw * kTraceLen : nullptr,
        order);
    const double gq = sp.G * mq;
    F[0] = gq * o.ax;
    F[1] = gq * o.ay;
    F[2] = gq * o.az;
    nv = o.visits;
    na = o.accepted;
  } else {
    Trav64Out o = traverse64d(tr.a64, tr.b64, n_nodes, y[0], y[1], y[2], __dmul_rn(sp.G, mq),
                              active, sp.theta2, sp.eps2,
                              kTrace ? trace + gw * kTraceLen : nullptr);
    F[0] = o.fx;
    F[1] = o.fy;
    F[2] = o.fz;
    nv = o.visits;
    na = o.accepted;
  }
  Partial p;
  partial_zero(p);
  if (active) {
    // state re-read here (L2-resident) instead of living in registers
    // across the traversal loop
    y[0] = tv.px[i];
    y[1] = tv.py[i];
    y[2] = tv.pz[i];
    v[0] = tv.vx[i];
    v[1] = tv.vy[i];
    v[2] = tv.vz[i];
    mq = tv.mq[i];
    double vp[3];
    const double s[3] = {st->shift[0], st->shift[1], st->shift[2]};
    step_and_accumulate(F, y, v, mq, sp, s, vp, p);
    tv.vx[i] = vp[0];
    tv.vy[i] = vp[1];
    tv.vz[i] = vp[2];
  }
  p.v[kAccepted] = (double)__reduce_add_sync(0xffffffffu, (unsigned)na);
  p.v[kVisits] = (double)__reduce_add_sync(0xffffffffu, (unsigned)nv);
  // counts are already warp totals: divide the upcoming warp_sum by 32
  p.v[kAccepted] = lane == 0 ? p.v[kAccepted] : 0.0;
  p.v[kVisits] = lane == 0 ? p.v[kVisits] : 0.0;
  warp_store_partial(p, lane, partials + gw * kPartialStride);
}

// ---------------------------------------------------------------- block order
// key = the block's recorded warp steps (k_bh_iterate<kTrace>), value = block
__global__ void k_block_work(const int* __restrict__ trace, int nblocks, int wpb,
                             unsigned* __restrict__ key, int* __restrict__ val) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  unsigned w = 0;
  for (int k = 0; k < wpb; k++) w += (unsigned)trace[((int64_t)b * wpb + k) * kTraceLen + 64];
  key[b] = w;
  val[b] = b;
}

// max and sum of the warps' recorded step counts (one block)
__global__ void k_trace_stats(const int* __restrict__ trace, int64_t nw,
                              unsigned long long* __restrict__ out) {
  unsigned long long mx = 0, sm = 0;
  for (int64_t w = threadIdx.x; w < nw; w += blockDim.x) {
    const unsigned long long v = (unsigned)trace[w * kTraceLen + 64];
    mx = v > mx ? v : mx;
    sm += v;
  }
  __shared__ unsigned long long smx[32], ssm[32];
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = a > mx ? a : mx;
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
  }
  if ((threadIdx.x & 31) == 0) {
    smx[threadIdx.x >> 5] = mx;
    ssm[threadIdx.x >> 5] = sm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); k++) {
      mx = smx[k] > mx ? smx[k] : mx;
      sm += ssm[k];
    }
    out[0] = mx;
    out[1] = sm;
  }
}

// ---------------------------------------------------------------- split passes
// Small template shards (one wave with at most half the resident warp slots
// used: an 8-way shard of the 1M template) end with their heaviest warps'
// step chains (per-warp union steps up to 1.6x the mean).  The first pass
// records each warp's node index every 256 steps (k_bh_iterate<kTrace>);
// later passes run every warp as TWO warps over the node ranges [0, s) and
// [s, n_nodes), s = the node at half its recorded steps rounded to a fold
// chunk (FGA_FOLD) boundary -- so every fp32 chunk sum is the unsplit one and
// only the fp64 fold of the chunks is regrouped -- and a second kernel adds
// the two parts and runs the epilogue.  Visits and accepted sets unchanged.
constexpr int kSplitT = 128;
#ifndef FGA_SPLIT_TPS
#define FGA_SPLIT_TPS FGA_BH32_TPS
#endif
#ifndef FGA_SPLIT_PARTS
#define FGA_SPLIT_PARTS 8
#endif
constexpr int kParts = FGA_SPLIT_PARTS;
static_assert(kParts >= 2 && kParts <= 8, "capi.cu reserves 8 parts (kSplitPartsMax)");
// the node index where part p of warp w starts (p = 0 .. kParts): the node at
// p/kParts of its recorded steps, rounded to a fold chunk boundary
__device__ __forceinline__ int split_point(const int* __restrict__ trace, int64_t w, int p,
                                           int n_nodes) {
  if (p <= 0) return 0;
  if (p >= kParts) return n_nodes;
  const int* tw = trace + w * kTraceLen;
  const int steps = tw[64];
  const int k = min(63, (int)(((int64_t)steps * p / kParts) >> 8));
  int sp = steps > 0 ? tw[k] : 0;
  if (FGA_FOLD > 0) sp = ((sp + FGA_FOLD / 2) / FGA_FOLD) * FGA_FOLD;
  return min(max(sp, 0), n_nodes);
}

template <bool kGuardZero>
__global__ void __launch_bounds__(kSplitT, FGA_SPLIT_TPS / kSplitT) k_bh_split(
    TreeRecords tr, int n_nodes, TemplateView tv, const IterState* __restrict__ st, F32Params f,
    double theta2_64, const int* __restrict__ trace, int64_t nwarps, double* __restrict__ fpart,
    int* __restrict__ apart) {
  if (st->done) return;
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (kSplitT / 32) + (threadIdx.x >> 5);
  if (g >= kParts * nwarps) return;  // (whole warps)
  // part-major: neighbouring warps of the grid walk the same node range
  // (L1 reuse across a block's and an SM's warps, as in the unsplit pass)
  const int64_t w = g % nwarps;
  const int part = (int)(g / nwarps);
  const int64_t i = w * 32 + lane;
  const bool active = i < tv.m;
  double y[3] = {0, 0, 0};
  if (active) {  // the position with the pending step applied (written back by k_bh_split_epi)
    double v[3] = {0, 0, 0};
    y[0] = tv.px[i];
    y[1] = tv.py[i];
    y[2] = tv.pz[i];
    apply_pending(st, y, v);
  }
  int lo = 0, hi = 0;
  for (int q = 1; q <= part + 1; q++) {  // monotone part boundaries
    lo = hi;
    hi = max(lo, split_point(trace, w, q, n_nodes));
  }
  __shared__ double hs[3 * kSplitT];
  __shared__ double qsh[3 * kSplitT];
  {
    double* q = qsh + 3 * threadIdx.x;
    q[0] = y[0];
    q[1] = y[1];
    q[2] = y[2];
  }
  const Trav32Out o = traverse32d<kGuardZero, false, false, false, true>(
      tr.c32, tr.a64, tr.b64, n_nodes, (float)y[0], (float)y[1], (float)y[2], active, f.theta2,
      theta2_64, f.eps2, nullptr, nullptr, nullptr, tv.m, hs, 0.f, 0.f, -1, nullptr, qsh, lo, hi);
  if (!active) return;
  double* fp = fpart + (part * tv.m + i) * 3;
  fp[0] = o.ax;
  fp[1] = o.ay;
  fp[2] = o.az;
  apart[part * tv.m + i] = o.accepted;
}

template <int kT>
__global__ void __launch_bounds__(kT) k_bh_split_epi(TemplateView tv, const IterState* __restrict__ st,
                                                     SimParams sp, const double* __restrict__ fpart,
                                                     const int* __restrict__ apart,
                                                     double* partials, int nblocks) {
  if (st->done) return;
  const int chunk = (int)blockIdx.x;
  if (chunk >= nblocks) return;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t gw = (int64_t)chunk * (kT / 32) + wl;
  const int64_t i = gw * 32 + lane;
  const bool active = i < tv.m;
  Partial p;
  partial_zero(p);
  int na = 0;
  if (active) {
    double y[3] = {tv.px[i], tv.py[i], tv.pz[i]}, v[3] = {tv.vx[i], tv.vy[i], tv.vz[i]};
    const double mq = tv.mq[i];
    apply_pending(st, y, v);
    tv.px[i] = y[0];
    tv.py[i] = y[1];
    tv.pz[i] = y[2];
    double h[3] = {0.0, 0.0, 0.0};
    for (int q = 0; q < kParts; q++) {  // the parts in node order
      const double* fq = fpart + (q * tv.m + i) * 3;
      h[0] += fq[0];
      h[1] += fq[1];
      h[2] += fq[2];
      na += apart[q * tv.m + i];
    }
    const double gq = sp.G * mq;
    const double F[3] = {gq * h[0], gq * h[1], gq * h[2]};
    double vp[3];
    const double s[3] = {st->shift[0], st->shift[1], st->shift[2]};
    step_and_accumulate(F, y, v, mq, sp, s, vp, p);
    tv.vx[i] = vp[0];
    tv.vy[i] = vp[1];
    tv.vz[i] = vp[2];
  }
  p.v[kAccepted] = (double)__reduce_add_sync(0xffffffffu, (unsigned)na);
  p.v[kVisits] = 0.0;
  p.v[kAccepted] = lane == 0 ? p.v[kAccepted] : 0.0;
  warp_store_partial(p, lane, partials + gw * kPartialStride);
}

// ---------------------------------------------------------------- BH operator
// kCV: count per-query visits (the caller asked for them; the registration
// loop's call, bhtree.bh_forces(count_visits=False) at dynamics.py:39, does not)
template <typename Real, bool kGuardZero, int kT = kForceThreads, bool kTrace = false,
          bool kCV = true>
#ifndef FGA_BHOP_MINB
#define FGA_BHOP_MINB 5  // 1280 threads/SM: fp64 operator 39.5 -> 38.7 ms (1M x 1M, host in/out)
#endif
#ifndef FGA_BHOP32_TPS
#define FGA_BHOP32_TPS FGA_BH32_TPS
#endif
__global__ void __launch_bounds__(kT, sizeof(Real) == 4 ? FGA_BHOP32_TPS / kT
                                                        : FGA_BHOP_MINB) k_bh_operator(
    TreeRecords tr, int n_nodes, const double* __restrict__ qx_, const double* __restrict__ qy_,
    const double* __restrict__ qz_, const double* __restrict__ qm_, const int* __restrict__ order,
    int64_t m, double theta2, double G, double eps2, F32Params f, double* __restrict__ fout,
    long long* __restrict__ visits, long long* __restrict__ accepted,
    unsigned long long* __restrict__ acc_total, int* __restrict__ trace = nullptr) {
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * (kT / 32) + wl;
  const int64_t i = gw * 32 + lane;
  const bool active = i < m;
  double F[3];
  int nv, na;
  if constexpr (sizeof(Real) == 4) {
    // the query as fp32 only: its mass is re-read after the traversal (L2)
    // instead of holding registers across it
    float qf[3] = {0.f, 0.f, 0.f};
    if (active) {
      qf[0] = (float)qx_[i];
      qf[1] = (float)qy_[i];
      qf[2] = (float)qz_[i];
    }
    __shared__ double hs[3 * kT];
    __shared__ unsigned hc[kCV ? 2 * kT : 1];
    const Trav32Out o = traverse32d<kGuardZero, kCV, false, false, false, kTrace>(
        tr.c32, tr.a64, tr.b64, n_nodes, qf[0], qf[1], qf[2], active, f.theta2, theta2, f.eps2,
        qx_, qy_, qz_, m, hs, 0.f, 0.f, -1, kCV ? hc : nullptr, nullptr, 0, -1,
        kTrace ? trace + gw * kTraceLen : nullptr);
    const double gq = G * (active ? qm_[i] : 0.0);
    F[0] = gq * o.ax;
    F[1] = gq * o.ay;
    F[2] = gq * o.az;
    nv = o.visits;
    na = o.accepted;
  } else {
    double q[3] = {0, 0, 0}, qm = 0.0;
    if (active) {
      q[0] = qx_[i];
      q[1] = qy_[i];
      q[2] = qz_[i];
      qm = qm_[i];
    }
    Trav64Out o = traverse64d(tr.a64, tr.b64, n_nodes, q[0], q[1], q[2], __dmul_rn(G, qm), active,
                              theta2, eps2);
    F[0] = o.fx;
    F[1] = o.fy;
    F[2] = o.fz;
    nv = o.visits;
    na = o.accepted;
  }
  if (acc_total) {  // the call's interaction count (fga_last_interactions)
    const unsigned wsum = __reduce_add_sync(0xffffffffu, active ? (unsigned)na : 0u);
    if (lane == 0) atomicAdd(acc_total, (unsigned long long)wsum);
  }
  if (!active) return;
  const int64_t dst = order ? order[i] : i;
  fout[dst * 3] = F[0];
  fout[dst * 3 + 1] = F[1];
  fout[dst * 3 + 2] = F[2];
  if (visits) visits[dst] = nv;
  if (accepted) accepted[dst] = na;
}

// One-shot operator calls that fill at most one wave (an N-way rank's slice
// of the queries): the same split passes as the session's (k_bh_split), from
// the trace the previous call over the same tree, query count and theta
// recorded (k_bh_operator<kTrace>) -- in the reference's loop the template
// moves a little per call, so the warps' step profiles carry over; any split
// points give the same visits, accepted sets and (to fp64 regrouping) forces.
template <bool kGuardZero, bool kCV>
__global__ void __launch_bounds__(kSplitT, FGA_SPLIT_TPS / kSplitT) k_bh_op_split(
    TreeRecords tr, int n_nodes, const double* __restrict__ qx_, const double* __restrict__ qy_,
    const double* __restrict__ qz_, int64_t m, F32Params f, double theta2_64,
    const int* __restrict__ trace, int64_t nwarps, double* __restrict__ fpart,
    int* __restrict__ vpart, int* __restrict__ apart, int* __restrict__ ptrace) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (kSplitT / 32) + (threadIdx.x >> 5);
  if (g >= kParts * nwarps) return;  // (whole warps)
  const int64_t w = g % nwarps;      // part-major, as k_bh_split
  const int part = (int)(g / nwarps);
  const int64_t i = w * 32 + lane;
  const bool active = i < m;
  __shared__ double hs[3 * kSplitT];
  __shared__ double qsh[3 * kSplitT];
  double* q = qsh + 3 * threadIdx.x;
  q[0] = active ? qx_[i] : 0.0;
  q[1] = active ? qy_[i] : 0.0;
  q[2] = active ? qz_[i] : 0.0;
  int lo = 0, hi = 0;
  for (int k = 1; k <= part + 1; k++) {
    lo = hi;
    hi = max(lo, split_point(trace, w, k, n_nodes));
  }
  // ptrace: the parts' own step counts (k_trace_stats -> whether the trace
  // still balances this call's queries)
  const Trav32Out o = traverse32d<kGuardZero, kCV, false, false, true, false, true>(
      tr.c32, tr.a64, tr.b64, n_nodes, (float)q[0], (float)q[1], (float)q[2], active, f.theta2,
      theta2_64, f.eps2, nullptr, nullptr, nullptr, m, hs, 0.f, 0.f, -1, nullptr, qsh, lo, hi,
      ptrace + g * kTraceLen);
  if (!active) return;
  double* fp = fpart + (part * m + i) * 3;
  fp[0] = o.ax;
  fp[1] = o.ay;
  fp[2] = o.az;
  if (kCV) vpart[part * m + i] = o.visits;
  apart[part * m + i] = o.accepted;
}

// the parts in node order -> G m_q sum, counts, scattered like k_bh_operator
__global__ void __launch_bounds__(256) k_bh_op_split_epi(
    const double* __restrict__ qm_, const int* __restrict__ order, int64_t m, double G,
    const double* __restrict__ fpart, const int* __restrict__ vpart, const int* __restrict__ apart,
    double* __restrict__ fout, long long* __restrict__ visits, long long* __restrict__ accepted,
    unsigned long long* __restrict__ acc_total) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < m;
  double h[3] = {0.0, 0.0, 0.0};
  int nv = 0, na = 0;
  if (active) {
    for (int q = 0; q < kParts; q++) {
      const double* fq = fpart + (q * m + i) * 3;
      h[0] += fq[0];
      h[1] += fq[1];
      h[2] += fq[2];
      if (visits) nv += vpart[q * m + i];
      na += apart[q * m + i];
    }
  }
  if (acc_total) {
    const unsigned wsum = __reduce_add_sync(0xffffffffu, active ? (unsigned)na : 0u);
    if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(acc_total, (unsigned long long)wsum);
  }
  if (!active) return;
  const double gq = G * qm_[i];
  const int64_t dst = order ? order[i] : i;
  fout[dst * 3] = gq * h[0];
  fout[dst * 3 + 1] = gq * h[1];
  fout[dst * 3 + 2] = gq * h[2];
  if (visits) visits[dst] = nv;
  if (accepted) accepted[dst] = na;
}

// ---------------------------------------------------------------- direct sum
// (kTile: fga_device.cuh)

template <bool kGuard>
#ifndef FGA_DIRECT_MINB
#define FGA_DIRECT_MINB 3  // 4 spills (240 B) and is 2.5% slower
#endif
#ifndef FGA_GPE_MINB
#define FGA_GPE_MINB 4  // energy: 3 blocks 0.405 s, 4 -> 0.386 s, 5 -> 0.398 s (1M x 1M)
#endif
__global__ void __launch_bounds__(kForceThreads, FGA_DIRECT_MINB) k_direct_iterate32(
    const float4* __restrict__ src, int64_t n, TemplateView tv, const IterState* __restrict__ st,
    SimParams sp, float eps2, double* partials) {
  if (st->done) return;
  __shared__ float4 sm[kTile];
  constexpr int Q = kDirectQPT, P = Q / 2;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * (kForceThreads * Q);
  float2 qx[P], qy[P], qz[P];
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t i = base + threadIdx.x + k * kForceThreads;
    double y[3] = {0.0, 0.0, 0.0}, v[3];
    if (i < tv.m) {
      y[0] = tv.px[i];
      y[1] = tv.py[i];
      y[2] = tv.pz[i];
      v[0] = tv.vx[i];
      v[1] = tv.vy[i];
      v[2] = tv.vz[i];
      apply_pending(st, y, v);
      tv.px[i] = y[0];
      tv.py[i] = y[1];
      tv.pz[i] = y[2];
      tv.vx[i] = v[0];
      tv.vy[i] = v[1];
      tv.vz[i] = v[2];
    }
    float* fx = reinterpret_cast<float*>(&qx[k / 2]);
    float* fy = reinterpret_cast<float*>(&qy[k / 2]);
    float* fz = reinterpret_cast<float*>(&qz[k / 2]);
    fx[k % 2] = (float)y[0];
    fy[k % 2] = (float)y[1];
    fz[k % 2] = (float)y[2];
  }
  double A[Q][3];
#pragma unroll
  for (int k = 0; k < Q; k++) A[k][0] = A[k][1] = A[k][2] = 0.0;
  for (int64_t t0 = 0; t0 < n; t0 += kTile) {
    const int jmax = (int)((n - t0) < (int64_t)kTile ? (n - t0) : (int64_t)kTile);
    __syncthreads();
    for (int j = threadIdx.x; j < jmax; j += kForceThreads) sm[j] = __ldg(&src[t0 + j]);
    __syncthreads();
    float2 ax[P], ay[P], az[P];
#pragma unroll
    for (int k = 0; k < P; k++) ax[k] = ay[k] = az[k] = make_float2(0.f, 0.f);
    direct_tile32<P, kGuard>(sm, jmax, qx, qy, qz, eps2, ax, ay, az);
#pragma unroll
    for (int k = 0; k < P; k++) {
      A[2 * k][0] += (double)ax[k].x;
      A[2 * k][1] += (double)ay[k].x;
      A[2 * k][2] += (double)az[k].x;
      A[2 * k + 1][0] += (double)ax[k].y;
      A[2 * k + 1][1] += (double)ay[k].y;
      A[2 * k + 1][2] += (double)az[k].y;
    }
  }
  Partial p;
  partial_zero(p);
  const double s[3] = {st->shift[0], st->shift[1], st->shift[2]};
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t i = base + threadIdx.x + k * kForceThreads;
    if (i >= tv.m) continue;
    const double y[3] = {tv.px[i], tv.py[i], tv.pz[i]};
    const double v[3] = {tv.vx[i], tv.vy[i], tv.vz[i]};
    const double mq = tv.mq[i];
    const double gq = sp.G * mq;
    const double F[3] = {gq * A[k][0], gq * A[k][1], gq * A[k][2]};
    double vp[3];
    step_and_accumulate(F, y, v, mq, sp, s, vp, p);
    tv.vx[i] = vp[0];
    tv.vy[i] = vp[1];
    tv.vz[i] = vp[2];
  }
  const int64_t gw = (int64_t)blockIdx.x * kWarps + wl;
  warp_store_partial(p, lane, partials + gw * kPartialStride);
}

__global__ void __launch_bounds__(kForceThreads) k_direct_iterate64(
    const double4* __restrict__ src, int64_t n, TemplateView tv, const IterState* __restrict__ st,
    SimParams sp, double* partials) {
  if (st->done) return;
  __shared__ double4 sm[kTile / 2];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * kForceThreads + threadIdx.x;
  const bool active = i < tv.m;
  double y[3] = {0, 0, 0}, v[3] = {0, 0, 0}, mq = 1.0;
  if (active) {
    y[0] = tv.px[i];
    y[1] = tv.py[i];
    y[2] = tv.pz[i];
    v[0] = tv.vx[i];
    v[1] = tv.vy[i];
    v[2] = tv.vz[i];
    mq = tv.mq[i];
    apply_pending(st, y, v);
    tv.px[i] = y[0];
    tv.py[i] = y[1];
    tv.pz[i] = y[2];
  }
  double sx = 0, sy = 0, sz = 0;
  for (int64_t t0 = 0; t0 < n; t0 += kTile / 2) {
    const int jmax = (int)((n - t0) < (int64_t)(kTile / 2) ? (n - t0) : (int64_t)(kTile / 2));
    __syncthreads();
    for (int j = threadIdx.x; j < jmax; j += kForceThreads) sm[j] = src[t0 + j];
    __syncthreads();
    direct_tile64(sm, jmax, y[0], y[1], y[2], sp.eps2, sx, sy, sz);
  }
  Partial p;
  partial_zero(p);
  if (active) {
    const double sc = __dmul_rn(-sp.G, mq);
    const double F[3] = {__dmul_rn(sc, sx), __dmul_rn(sc, sy), __dmul_rn(sc, sz)};
    double vp[3];
    const double s[3] = {st->shift[0], st->shift[1], st->shift[2]};
    step_and_accumulate(F, y, v, mq, sp, s, vp, p);
    tv.vx[i] = vp[0];
    tv.vy[i] = vp[1];
    tv.vz[i] = vp[2];
  }
  const int64_t gw = (int64_t)blockIdx.x * kWarps + wl;
  warp_store_partial(p, lane, partials + gw * kPartialStride);
}

template <bool kGuard>
__global__ void __launch_bounds__(kForceThreads, 3) k_direct_operator32(
    const float4* __restrict__ src, int64_t n, const double* __restrict__ qx_,
    const double* __restrict__ qy_, const double* __restrict__ qz_, const double* __restrict__ qm_,
    int64_t m, double G, float eps2, double* __restrict__ fout) {
  __shared__ float4 sm[kTile];
  constexpr int Q = kDirectQPT, P = Q / 2;
  const int64_t base = (int64_t)blockIdx.x * (kForceThreads * Q);
  float2 qx[P], qy[P], qz[P];
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t i = base + threadIdx.x + k * kForceThreads;
    reinterpret_cast<float*>(&qx[k / 2])[k % 2] = i < m ? (float)qx_[i] : 0.f;
    reinterpret_cast<float*>(&qy[k / 2])[k % 2] = i < m ? (float)qy_[i] : 0.f;
    reinterpret_cast<float*>(&qz[k / 2])[k % 2] = i < m ? (float)qz_[i] : 0.f;
  }
  double A[Q][3];
#pragma unroll
  for (int k = 0; k < Q; k++) A[k][0] = A[k][1] = A[k][2] = 0.0;
  for (int64_t t0 = 0; t0 < n; t0 += kTile) {
    const int jmax = (int)((n - t0) < (int64_t)kTile ? (n - t0) : (int64_t)kTile);
    __syncthreads();
    for (int j = threadIdx.x; j < jmax; j += kForceThreads) sm[j] = __ldg(&src[t0 + j]);
    __syncthreads();
    float2 ax[P], ay[P], az[P];
#pragma unroll
    for (int k = 0; k < P; k++) ax[k] = ay[k] = az[k] = make_float2(0.f, 0.f);
    direct_tile32<P, kGuard>(sm, jmax, qx, qy, qz, eps2, ax, ay, az);
#pragma unroll
    for (int k = 0; k < P; k++) {
      A[2 * k][0] += (double)ax[k].x;
      A[2 * k][1] += (double)ay[k].x;
      A[2 * k][2] += (double)az[k].x;
      A[2 * k + 1][0] += (double)ax[k].y;
      A[2 * k + 1][1] += (double)ay[k].y;
      A[2 * k + 1][2] += (double)az[k].y;
    }
  }
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t i = base + threadIdx.x + k * kForceThreads;
    if (i >= m) continue;
    const double gq = G * qm_[i];
    fout[i * 3] = gq * A[k][0];
    fout[i * 3 + 1] = gq * A[k][1];
    fout[i * 3 + 2] = gq * A[k][2];
  }
}

__global__ void __launch_bounds__(kForceThreads) k_direct_operator64(
    const double4* __restrict__ src, int64_t n, const double* __restrict__ qx_,
    const double* __restrict__ qy_, const double* __restrict__ qz_, const double* __restrict__ qm_,
    int64_t m, double G, double eps2, double* __restrict__ fout) {
  __shared__ double4 sm[kTile / 2];
  const int64_t i = (int64_t)blockIdx.x * kForceThreads + threadIdx.x;
  const double qx = i < m ? qx_[i] : 0.0, qy = i < m ? qy_[i] : 0.0, qz = i < m ? qz_[i] : 0.0;
  double sx = 0, sy = 0, sz = 0;
  for (int64_t t0 = 0; t0 < n; t0 += kTile / 2) {
    const int jmax = (int)((n - t0) < (int64_t)(kTile / 2) ? (n - t0) : (int64_t)(kTile / 2));
    __syncthreads();
    for (int j = threadIdx.x; j < jmax; j += kForceThreads) sm[j] = src[t0 + j];
    __syncthreads();
    direct_tile64(sm, jmax, qx, qy, qz, eps2, sx, sy, sz);
  }
  if (i >= m) return;
  const double sc = __dmul_rn(-G, qm_[i]);  // -params.G * query_mass (bhtree.py:164)
  fout[i * 3] = __dmul_rn(sc, sx);
  fout[i * 3 + 1] = __dmul_rn(sc, sy);
  fout[i * 3 + 2] = __dmul_rn(sc, sz);
}

// ---------------------------------------------------------------- energy
template <bool kNewton, int Q>
__global__ void __launch_bounds__(kForceThreads, FGA_GPE_MINB) k_gpe32(const float4* __restrict__ src,
                                                            int64_t n,
                                                            const double* __restrict__ px,
                                                            const double* __restrict__ py,
                                                            const double* __restrict__ pz,
                                                            const double* __restrict__ mq,
                                                            int64_t m, float eps,
                                                            const IterState* st,
                                                            double* partials, int64_t seg) {
  if (st && st->done) return;
  __shared__ float4 sm[kTile];
  constexpr int NP = Q / 2;  // packs of 2 queries; odd packs on Newton
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * (kForceThreads * Q);
  float2 qx[NP], qy[NP], qz[NP];
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t i = base + threadIdx.x + k * kForceThreads;
    reinterpret_cast<float*>(&qx[k / 2])[k % 2] = i < m ? (float)px[i] : 0.f;
    reinterpret_cast<float*>(&qy[k / 2])[k % 2] = i < m ? (float)py[i] : 0.f;
    reinterpret_cast<float*>(&qz[k / 2])[k % 2] = i < m ? (float)pz[i] : 0.f;
  }
  double acc[Q];
#pragma unroll
  for (int k = 0; k < Q; k++) acc[k] = 0.0;
  const int64_t r0 = (int64_t)blockIdx.y * seg, r1 = min(n, r0 + seg);  // this block's reference segment
  for (int64_t t0 = r0; t0 < r1; t0 += kTile) {
    const int jmax = (int)((r1 - t0) < (int64_t)kTile ? (r1 - t0) : (int64_t)kTile);
    __syncthreads();
    for (int j = threadIdx.x; j < jmax; j += kForceThreads) sm[j] = __ldg(&src[t0 + j]);
    __syncthreads();
    float2 a[NP];
#pragma unroll
    for (int k = 0; k < NP; k++) a[k] = make_float2(0.f, 0.f);
    gpe_tile32<kNewton, NP>(sm, jmax, qx, qy, qz, eps, a);
#pragma unroll
    for (int k = 0; k < NP; k++) {
      const double sgn = (kNewton && (k & 1)) ? -1.0 : 1.0;  // Newton packs hold -sum
      acc[2 * k] += sgn * (double)a[k].x;
      acc[2 * k + 1] += sgn * (double)a[k].y;
    }
  }
  double tot = 0.0;
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t i = base + threadIdx.x + k * kForceThreads;
    if (i < m) tot += mq[i] * acc[k];
  }
  tot = warp_sum(tot);
  if (lane == 0) partials[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * kWarps + wl] = tot;
}

__global__ void __launch_bounds__(kForceThreads) k_gpe64(const double4* __restrict__ src, int64_t n,
                                                         const double* __restrict__ px,
                                                         const double* __restrict__ py,
                                                         const double* __restrict__ pz,
                                                         const double* __restrict__ mq, int64_t m,
                                                         double eps, const IterState* st,
                                                         double* partials, int64_t seg) {
  if (st && st->done) return;
  __shared__ double4 sm[kTile / 2];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * kForceThreads + threadIdx.x;
  const double qx = i < m ? px[i] : 0.0, qy = i < m ? py[i] : 0.0, qz = i < m ? pz[i] : 0.0;
  double acc = 0.0;
  const int64_t r0 = (int64_t)blockIdx.y * seg, r1 = min(n, r0 + seg);  // this block's reference segment
  for (int64_t t0 = r0; t0 < r1; t0 += kTile / 2) {
    const int jmax = (int)((r1 - t0) < (int64_t)(kTile / 2) ? (r1 - t0) : (int64_t)(kTile / 2));
    __syncthreads();
    for (int j = threadIdx.x; j < jmax; j += kForceThreads) sm[j] = src[t0 + j];
    __syncthreads();
    for (int j = 0; j < jmax; j++) {
      const double4 s = sm[j];
      const double dx = __dsub_rn(qx, s.x), dy = __dsub_rn(qy, s.y), dz = __dsub_rn(qz, s.z);
      const double d2 =
          __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      acc = __dadd_rn(acc, __ddiv_rn(s.w, __dadd_rn(__dsqrt_rn(d2), eps)));  // :66
    }
  }
  double tot = i < m ? __dmul_rn(mq[i], acc) : 0.0;
  tot = warp_sum(tot);
  if (lane == 0) partials[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * kWarps + wl] = tot;
}

inline unsigned grid_for(int64_t items, int64_t per_block) {
  return (unsigned)((items + per_block - 1) / per_block);
}

}  // namespace

// ------------------------------------------------------------------ launchers
static int current_sms();
// Threads per block of the iteration kernel for m template queries: 64 for
// multi-wave FP32 passes (with the heaviest-first block order, finer blocks
// leave less of a slot idle behind a block's slowest warp: 1M pass 11.08 ->
// 10.93 ms), 128 for one-wave passes (the shared-memory small-tree and split
// paths are tuned there).  FGA_BH_BLOCK forces a size.
static int bh_block(int64_t m, int precision) {
  static const int forced = [] {
    const char* e = getenv("FGA_BH_BLOCK");
    const int v = e ? atoi(e) : 0;
    return (v == 64 || v == 128 || v == 256) ? v : 0;
  }();
  if (forced) return forced;
  const int64_t warps128 = (int64_t)grid_for(m, 128) * 4;
  const int tps = precision ? FGA_BH64_TPS : FGA_BH32_TPS;  // (fp64 at 64: 27.73 -> 27.57 ms)
  return warps128 <= (int64_t)current_sms() * (tps / 32) ? 128 : 64;
}
// whether a pass over m queries may run as split passes (launch_bh_iterate_t:
// at most one wave)
bool bh_split_possible(int64_t m) {
  const int64_t nw = (int64_t)grid_for(m, 128) * 4;
  return nw <= (int64_t)current_sms() * (FGA_BH32_TPS / 32);
}
int64_t bh_iterate_warps(int64_t m, int precision) {
  const int t = bh_block(m, precision);
  return (int64_t)grid_for(m, t) * (t / 32);
}
int64_t direct_iterate_warps(int64_t m, int precision) {
  const int64_t per = precision ? kForceThreads : kForceThreads * kDirectQPT;
  return (int64_t)grid_for(m, per) * kWarps;
}
// queries per thread of the FP32 energy kernel (8 was measured 24% slower)
constexpr int kGpeQ = 4;
// The energy kernels also split the reference points into segments
// (blockIdx.y) when the queries alone give too few blocks (configs[1]/[3]:
// 100k-200k points -> 98-196 query blocks on 148 SMs).  The split depends
// only on (m, n), so the fixed-order partial sums stay deterministic.
struct GpeShape {
  int64_t qblocks, splits, seg;
};
// SM count of the current device (cached per device)
static int current_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = sms > 0 ? sms : 148;
  }
  return cache[dev];
}

static GpeShape gpe_shape(int64_t m, int64_t n, int precision) {
  const int64_t per = precision ? kForceThreads : kForceThreads * kGpeQ;
  const int64_t tile = precision ? kTile / 2 : kTile;
  GpeShape g;
  g.qblocks = grid_for(m, per);
  // two waves of the resident blocks (FGA_GPE_MINB per SM for k_gpe32)
  const int64_t resident = (int64_t)current_sms() * (precision ? 3 : FGA_GPE_MINB);
  int64_t sp = (2 * resident + g.qblocks - 1) / g.qblocks;
  sp = std::max<int64_t>(1, std::min<int64_t>(sp, n / (4 * tile)));  // >= 4 tiles per segment
  const int64_t tiles = (n + tile - 1) / tile;
  g.seg = ((tiles + sp - 1) / sp) * tile;
  g.splits = std::max<int64_t>(1, (n + g.seg - 1) / g.seg);
  return g;
}
int64_t gpe_warps(int64_t m, int64_t n, int precision) {
  const GpeShape g = gpe_shape(m, n, precision);
  return g.qblocks * g.splits * kWarps;
}

static int current_sms();

// ------------------------------------------------------- per-launch node bands
// The FP32 MAC guard band of every node for this launch's
// queries: delta = (max |q| + max |com|) 2^-24 over ALL queries (a global
// bound instead of the warp's), so the band is a per-node constant that the
// traversal reads from the record instead of forming it per step.  Also
// folds eps^2 into the record's l^2 (see traverse32d<kBand>): the fma-form
// MAC then adds <= 3u (l^2 + theta^2 eps^2) of rounding, covered by the
// 16u l^2 and 4u theta^2 eps^2 terms.
template <bool kPending>
__global__ void __launch_bounds__(256) k_qbound(const double* __restrict__ px,
                                                const double* __restrict__ py,
                                                const double* __restrict__ pz, int64_t m,
                                                const IterState* __restrict__ st,
                                                unsigned* __restrict__ out) {
  if (kPending && st->done) return;
  float mx = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    double y[3] = {px[i], py[i], pz[i]};
    if constexpr (kPending) {
      double v[3] = {0, 0, 0};
      apply_pending(st, y, v);
    }
    const double a = fmax(fabs(y[0]), fmax(fabs(y[1]), fabs(y[2])));
    mx = fmaxf(mx, __double2float_ru(a));
  }
  mx = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(mx)));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(mx));
}

__global__ void __launch_bounds__(256) k_node_bands(float4* __restrict__ c32, int nn, float theta2,
                                                    float eps2, float cmag,
                                                    const unsigned* __restrict__ qbound,
                                                    const IterState* __restrict__ st) {
  if (st && st->done) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  float4 r = c32[2 * i + 1];
  const float l2 = r.w;  // the node's l^2 as built (-inf: leaf)
  if (l2 == -INFINITY) {
    r.x = -INFINITY;  // always accepted, never re-checked
    r.z = -INFINITY;
  } else {
    const float te = theta2 * eps2;
    const float delta = (__uint_as_float(*qbound) + cmag) * 5.97e-8f;
    const float gA = 4.34f * delta * sqrtf(theta2);  // 1.25 * 2 sqrt3 delta theta
    const float gB = 34.f * delta * delta * theta2 + 4.f * 5.97e-8f * te + 1e-37f;
    r.x = l2 + te;
    r.z = fmaf(gA, sqrtf(l2), fmaf(16.f * 5.97e-8f, l2, gB));
  }
  c32[2 * i + 1] = r;
}

static void launch_node_bands(const TreeDev& T, const double* px, const double* py,
                              const double* pz, int64_t m, const IterState* st, float theta2,
                              float eps2, cudaStream_t s) {
  unsigned* qb = T.band_scratch.as<unsigned>();
  cudaMemsetAsync(qb, 0, sizeof(unsigned), s);
  const int g = (int)std::min<int64_t>(grid_for(m, 256), 4 * current_sms());
  if (st)
    k_qbound<true><<<g, 256, 0, s>>>(px, py, pz, m, st, qb);
  else
    k_qbound<false><<<g, 256, 0, s>>>(px, py, pz, m, nullptr, qb);
  const int nn = (int)T.n_nodes;
  k_node_bands<<<(nn + 255) / 256, 256, 0, s>>>(T.records().c32, nn, theta2, eps2, (float)T.cmag,
                                                qb, st);
}

template <int kT>
static void launch_bh_iterate_t(const TreeDev& T, const TemplateView& tv, const IterState* st,
                                const SimParams& sp, double* partials, int precision,
                                cudaStream_t s, const SplitBufs* sb) {
  const int nb = (int)grid_for(tv.m, kT);
  const unsigned g = (unsigned)nb;
  const F32Params f{(float)sp.theta2, (float)sp.eps2};
  const bool gz = !(sp.eps2 > 0.0);
  const int nn = (int)T.n_nodes;
  const TreeRecords r = T.records();
  if (precision) {
    // fp64: the heaviest-first block order too (the first pass records it)
    static const bool order64 = !(getenv("FGA_LPT") && atoi(getenv("FGA_LPT")) == 0);
    if (order64 && sb && sb->order) {
      if (!*sb->have_order) {
        k_bh_iterate<double, false, true, kT, false, true><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f,
                                                                          partials, nb, sb->trace);
        unsigned* kin = reinterpret_cast<unsigned*>(sb->okeys);
        unsigned* kout = kin + nb;
        int* vin = sb->okeys + 2 * nb;
        k_block_work<<<(nb + 255) / 256, 256, 0, s>>>(sb->trace, nb, kT / 32, kin, vin);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, kin, kout, vin, sb->order, nb,
                                                  0, 32, s);
        if (bytes <= sb->tmp_bytes &&
            cub::DeviceRadixSort::SortPairsDescending(sb->tmp, bytes, kin, kout, vin, sb->order,
                                                      nb, 0, 32, s) == cudaSuccess)
          *sb->have_order = true;
        return;
      }
      k_bh_iterate<double, false, true, kT><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f, partials, nb,
                                                             nullptr, sb->order);
      return;
    }
    k_bh_iterate<double, false, true, kT><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f, partials, nb);
    return;
  }
  launch_node_bands(T, tv.px, tv.py, tv.pz, tv.m, st, f.theta2, f.eps2, s);
  const size_t tree_bytes = sizeof(float4) * 2 * (size_t)nn;
  if constexpr (kT == 128) {
  if (tree_bytes <= (size_t)kSmallTreeBytes &&
      (int64_t)nb <= (int64_t)current_sms() * std::max<int64_t>(1, (220 * 1024) / (int64_t)tree_bytes)) {
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev]) {
      cudaFuncSetAttribute(k_bh_iterate<float, true, true, kT, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallTreeBytes);
      cudaFuncSetAttribute(k_bh_iterate<float, true, false, kT, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallTreeBytes);
      cudaFuncSetAttribute(k_bh_iterate<float, false, true, kT, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallTreeBytes);
      cudaFuncSetAttribute(k_bh_iterate<float, false, false, kT, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallTreeBytes);
      if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    if (gz && sp.count_visits)
      k_bh_iterate<float, true, true, kT, true><<<g, kT, tree_bytes, s>>>(r, nn, tv, st, sp, f, partials, nb);
    else if (gz)
      k_bh_iterate<float, true, false, kT, true><<<g, kT, tree_bytes, s>>>(r, nn, tv, st, sp, f, partials, nb);
    else if (sp.count_visits)
      k_bh_iterate<float, false, true, kT, true><<<g, kT, tree_bytes, s>>>(r, nn, tv, st, sp, f, partials, nb);
    else
      k_bh_iterate<float, false, false, kT, true><<<g, kT, tree_bytes, s>>>(r, nn, tv, st, sp, f, partials, nb);
    return;
  }
  }
  // The first FP32 pass of a session records every warp's node trace and
  // step count; later passes then run either as split passes (one wave with
  // room to spare, or one wave whose heaviest warp exceeds FGA_SPLIT_IMB x the
  // mean: inhomogeneous clouds) or with the blocks launched heaviest first.
  static const bool split_on = !(getenv("FGA_SPLIT") && atoi(getenv("FGA_SPLIT")) == 0);
  static const bool order_on = !(getenv("FGA_LPT") && atoi(getenv("FGA_LPT")) == 0);
  static const double split_imb = getenv("FGA_SPLIT_IMB") ? atof(getenv("FGA_SPLIT_IMB")) : 2.0;
  static const bool split_log = getenv("FGA_SPLIT_LOG") != nullptr;  // (tests)
  const int64_t nw = (int64_t)nb * (kT / 32);
  const int64_t slots = (int64_t)current_sms() * (FGA_BH32_TPS / 32);
  const bool split_cand = split_on && sb && sb->fpart && sb->apart && sb->split &&
                          !sp.count_visits && nw >= 8 && nw <= slots;
  const bool order_cand = order_on && sb && sb->order && !sp.count_visits;
  if (split_cand || order_cand) {
    if (!*sb->have_trace) {
      if (gz)
        k_bh_iterate<float, true, false, kT, false, true><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f,
                                                                         partials, nb, sb->trace);
      else
        k_bh_iterate<float, false, false, kT, false, true><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f,
                                                                          partials, nb, sb->trace);
      bool split = false;
      if (split_cand) {
        if ((double)nw <= FGA_SPLIT_FRAC * (double)slots) {
          split = true;
        } else {  // a full wave: split only an imbalanced one (one sync, once per session)
          unsigned long long* st2 = reinterpret_cast<unsigned long long*>(sb->tmp);
          k_trace_stats<<<1, 1024, 0, s>>>(sb->trace, nw, st2);
          unsigned long long h[2] = {0, 0};
          if (cudaMemcpyAsync(h, st2, sizeof(h), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
              cudaStreamSynchronize(s) == cudaSuccess && h[1] > 0)
            split = (double)h[0] >= split_imb * ((double)h[1] / (double)nw);
          if (split_log)
            fprintf(stderr, "[fga] trace: %lld warps, max %llu mean %.0f -> %s\n", (long long)nw,
                    h[0], (double)h[1] / (double)nw, split ? "split" : "unsplit");
        }
      }
      *sb->split = split;
      if (!split && order_cand) {
        unsigned* kin = reinterpret_cast<unsigned*>(sb->okeys);
        unsigned* kout = kin + nb;
        int* vin = sb->okeys + 2 * nb;
        k_block_work<<<(nb + 255) / 256, 256, 0, s>>>(sb->trace, nb, kT / 32, kin, vin);
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, kin, kout, vin, sb->order, nb,
                                                  0, 32, s);
        if (bytes <= sb->tmp_bytes &&
            cub::DeviceRadixSort::SortPairsDescending(sb->tmp, bytes, kin, kout, vin, sb->order,
                                                      nb, 0, 32, s) == cudaSuccess)
          *sb->have_order = true;
      }
      *sb->have_trace = true;
      return;
    }
    if (split_cand && *sb->split) {
      if (split_log)
        fprintf(stderr, "[fga] split pass: %lld warps x %d parts\n", (long long)nw, kParts);
      const unsigned gs = (unsigned)((kParts * nw + kSplitT / 32 - 1) / (kSplitT / 32));
      if (gz)
        k_bh_split<true><<<gs, kSplitT, 0, s>>>(r, nn, tv, st, f, sp.theta2, sb->trace, nw,
                                                sb->fpart, sb->apart);
      else
        k_bh_split<false><<<gs, kSplitT, 0, s>>>(r, nn, tv, st, f, sp.theta2, sb->trace, nw,
                                                 sb->fpart, sb->apart);
      k_bh_split_epi<kT><<<g, kT, 0, s>>>(tv, st, sp, sb->fpart, sb->apart, partials, nb);
      return;
    }
    if (order_cand && *sb->have_order) {
      if (gz)
        k_bh_iterate<float, true, false, kT><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f, partials, nb,
                                                              nullptr, sb->order);
      else
        k_bh_iterate<float, false, false, kT><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f, partials,
                                                               nb, nullptr, sb->order);
      return;
    }
  }
  if (gz && sp.count_visits)
    k_bh_iterate<float, true, true, kT><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f, partials, nb);
  else if (gz)
    k_bh_iterate<float, true, false, kT><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f, partials, nb);
  else if (sp.count_visits)
    k_bh_iterate<float, false, true, kT><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f, partials, nb);
  else
    k_bh_iterate<float, false, false, kT><<<g, kT, 0, s>>>(r, nn, tv, st, sp, f, partials, nb);
}

void launch_bh_iterate(const TreeDev& T, const TemplateView& tv, const IterState* st,
                       const SimParams& sp, double* partials, int precision, cudaStream_t s,
                       const SplitBufs* sb) {
  if (tv.m <= 0) return;
  switch (bh_block(tv.m, precision)) {
    case 64: launch_bh_iterate_t<64>(T, tv, st, sp, partials, precision, s, sb); break;
    case 256: launch_bh_iterate_t<256>(T, tv, st, sp, partials, precision, s, sb); break;
    default: launch_bh_iterate_t<128>(T, tv, st, sp, partials, precision, s, sb); break;
  }
}

void launch_direct_iterate(const RefPoints& ref, const TemplateView& tv, const IterState* st,
                           const SimParams& sp, double* partials, int precision, cudaStream_t s) {
  if (tv.m <= 0) return;
  if (precision) {
    k_direct_iterate64<<<grid_for(tv.m, kForceThreads), kForceThreads, 0, s>>>(ref.p64, ref.n, tv,
                                                                               st, sp, partials);
  } else {
    const unsigned g = grid_for(tv.m, kForceThreads * kDirectQPT);
    if (sp.eps2 > 0.0)
      k_direct_iterate32<false><<<g, kForceThreads, 0, s>>>(ref.p32, ref.n, tv, st, sp, (float)sp.eps2, partials);
    else
      k_direct_iterate32<true><<<g, kForceThreads, 0, s>>>(ref.p32, ref.n, tv, st, sp, (float)sp.eps2, partials);
  }
}

void launch_gpe(const RefPoints& ref, const double* px, const double* py, const double* pz,
                const double* mq, int64_t m, double eps, const IterState* st, double* partials,
                int precision, cudaStream_t s) {
  if (m <= 0) return;
  const GpeShape g = gpe_shape(m, ref.n, precision);
  const dim3 grid((unsigned)g.qblocks, (unsigned)g.splits);
  if (precision)
    k_gpe64<<<grid, kForceThreads, 0, s>>>(ref.p64, ref.n, px, py, pz, mq, m, eps, st, partials,
                                           g.seg);
  else if (eps > 0.0)
    k_gpe32<true, kGpeQ><<<grid, kForceThreads, 0, s>>>(ref.p32, ref.n, px, py, pz, mq, m,
                                                        (float)eps, st, partials, g.seg);
  else  // eps == 0: keep IEEE rcp semantics (1/0 = inf) on every pair
    k_gpe32<false, kGpeQ><<<grid, kForceThreads, 0, s>>>(ref.p32, ref.n, px, py, pz, mq, m,
                                                         (float)eps, st, partials, g.seg);
}

#ifndef FGA_OP_T
#define FGA_OP_T 64
#endif
// FP32 operator threads per block (64: 13.88 -> 13.68 ms per 1M-query e2e call
// against 256)
constexpr int kOpT = FGA_OP_T;

bool bh_operator_split_possible(int64_t m) {
  static const bool on = !(getenv("FGA_SPLIT") && atoi(getenv("FGA_SPLIT")) == 0);
  const int64_t nw = (m + 31) / 32;
  return on && nw >= 8 && nw <= (int64_t)current_sms() * (FGA_BHOP32_TPS / 32);
}
int64_t bh_operator_warps(int64_t m) { return (int64_t)grid_for(m, kOpT) * (kOpT / 32); }
int bh_split_parts() { return kParts; }
bool bh_operator_split_wanted(int64_t m, unsigned long long max_steps,
                              unsigned long long sum_steps) {
  static const double imb = getenv("FGA_SPLIT_IMB") ? atof(getenv("FGA_SPLIT_IMB")) : 2.0;
  const int64_t nw = (m + 31) / 32;
  if ((double)nw <= FGA_SPLIT_FRAC * (double)current_sms() * (FGA_BHOP32_TPS / 32)) return true;
  return sum_steps > 0 && (double)max_steps >= imb * ((double)sum_steps / (double)nw);
}

void launch_bh_operator(const TreeDev& T, const double* qx, const double* qy, const double* qz,
                        const double* qm, const int* order, int64_t m, double theta, double G,
                        double eps2, double* fout, long long* visits, long long* accepted,
                        unsigned long long* acc_total, int precision, cudaStream_t s,
                        const OpSplitBufs* ob) {
  if (m <= 0) return;
  const double theta2 = theta * theta;
  const F32Params f{(float)theta2, (float)eps2};
  const int nn = (int)T.n_nodes;
  const TreeRecords r = T.records();
  if (precision) {
    const unsigned g = grid_for(m, kForceThreads);
    k_bh_operator<double, false><<<g, kForceThreads, 0, s>>>(r, nn, qx, qy, qz, qm, order, m,
                                                             theta2, G, eps2, f, fout, visits,
                                                             accepted, acc_total);
    return;
  }
  launch_node_bands(T, qx, qy, qz, m, nullptr, f.theta2, f.eps2, s);
  const unsigned g = grid_for(m, kOpT);
  const bool gz = !(eps2 > 0.0);
  if (ob && ob->mode == 2) {
    const int64_t nw = (m + 31) / 32;
    const unsigned gs = (unsigned)((kParts * nw + kSplitT / 32 - 1) / (kSplitT / 32));
#define FGA_OP_SPLIT(GZ, CV)                                                                  \
  k_bh_op_split<GZ, CV><<<gs, kSplitT, 0, s>>>(r, nn, qx, qy, qz, m, f, theta2, ob->trace, nw,  \
                                               ob->fpart, ob->vpart, ob->apart, ob->ptrace)
    if (gz && visits)
      FGA_OP_SPLIT(true, true);
    else if (gz)
      FGA_OP_SPLIT(true, false);
    else if (visits)
      FGA_OP_SPLIT(false, true);
    else
      FGA_OP_SPLIT(false, false);
#undef FGA_OP_SPLIT
    k_trace_stats<<<1, 1024, 0, s>>>(ob->ptrace, kParts * nw, ob->stats);
    k_bh_op_split_epi<<<grid_for(m, 256), 256, 0, s>>>(qm, order, m, G, ob->fpart, ob->vpart,
                                                       ob->apart, fout, visits, accepted,
                                                       acc_total);
    return;
  }
  if (ob && ob->mode == 1) {  // this call records the warps' traces (+ their max / sum)
    if (gz)
      k_bh_operator<float, true, kOpT, true><<<g, kOpT, 0, s>>>(
          r, nn, qx, qy, qz, qm, order, m, theta2, G, eps2, f, fout, visits, accepted, acc_total,
          ob->trace);
    else
      k_bh_operator<float, false, kOpT, true><<<g, kOpT, 0, s>>>(
          r, nn, qx, qy, qz, qm, order, m, theta2, G, eps2, f, fout, visits, accepted, acc_total,
          ob->trace);
    k_trace_stats<<<1, 1024, 0, s>>>(ob->trace, (m + 31) / 32, ob->stats);
    return;
  }
  if (!visits) {  // accepted counts only (one counter per lane, no packed visits)
    if (gz)
      k_bh_operator<float, true, kOpT, false, false><<<g, kOpT, 0, s>>>(
          r, nn, qx, qy, qz, qm, order, m, theta2, G, eps2, f, fout, visits, accepted, acc_total);
    else
      k_bh_operator<float, false, kOpT, false, false><<<g, kOpT, 0, s>>>(
          r, nn, qx, qy, qz, qm, order, m, theta2, G, eps2, f, fout, visits, accepted, acc_total);
    return;
  }
  if (gz)
    k_bh_operator<float, true, kOpT><<<g, kOpT, 0, s>>>(r, nn, qx, qy, qz, qm, order, m, theta2,
                                                        G, eps2, f, fout, visits, accepted,
                                                        acc_total);
  else
    k_bh_operator<float, false, kOpT><<<g, kOpT, 0, s>>>(r, nn, qx, qy, qz, qm, order, m, theta2,
                                                         G, eps2, f, fout, visits, accepted,
                                                         acc_total);
}

void launch_direct_operator(const RefPoints& ref, const double* qx, const double* qy,
                            const double* qz, const double* qm, int64_t m, double G, double eps,
                            double* fout, int precision, cudaStream_t s) {
  if (m <= 0) return;
  const double eps2 = eps * eps;  // params.epsilon**2 (bhtree.py:159)
  if (precision) {
    k_direct_operator64<<<grid_for(m, kForceThreads), kForceThreads, 0, s>>>(
        ref.p64, ref.n, qx, qy, qz, qm, m, G, eps2, fout);
  } else {
    const unsigned g = grid_for(m, kForceThreads * kDirectQPT);
    if (eps2 > 0.0)
      k_direct_operator32<false><<<g, kForceThreads, 0, s>>>(ref.p32, ref.n, qx, qy, qz, qm, m, G,
                                                             (float)eps2, fout);
    else
      k_direct_operator32<true><<<g, kForceThreads, 0, s>>>(ref.p32, ref.n, qx, qy, qz, qm, m, G,
                                                            (float)eps2, fout);
  }
}

}  // namespace fga
