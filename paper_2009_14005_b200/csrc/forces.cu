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
#include <climits>
#include <cstdlib>

#include "fga_session.cuh"

namespace fga {
namespace {

constexpr int kWin = 32;
constexpr int kNumSMs = 148;
constexpr int kWarps = kForceThreads / 32;

struct Win32 {
  float4 a[kWin];
  NodeB32 b[kWin];
};
struct Win64 {
  double4 a[kWin];
  NodeB64 b[kWin];
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

struct Trav32Out {
  float ax, ay, az;
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
// fp64 one by at most 2*delta*(|dx|+|dy|+|dz|) + 3*delta^2 + 4u*d^2.  When
// |theta^2 d^2 - l^2| is inside that bound (plus the rounding of l^2 and of
// theta^2 d^2) the decision is re-made exactly in fp64 from the fp64 records,
// so the accepted set always equals the reference's (_kernels.py:37).
// gA = 2*delta*theta^2*1.25, gB = 3*delta^2*theta^2*1.25 (per lane).
struct WinRec32 {
  float4 a;  // com.xyz, mass
  float4 b;  // l2 | -inf, skip (int bits), unused, unused
};
struct WinBuf32 {
  WinRec32 r[kWin];
};

template <bool kGuardZero>
__device__ __forceinline__ Trav32Out traverse32(const float4* __restrict__ A,
                                                const NodeB32* __restrict__ B,
                                                const double4* __restrict__ A64,
                                                const NodeB64* __restrict__ B64, int n_nodes,
                                                float qx, float qy, float qz, bool active,
                                                float theta2, double theta2_64, float eps2,
                                                float gA, float gB, const double* qpx,
                                                const double* qpy, const double* qpz, int64_t qi,
                                                WinBuf32* win, int lane) {
  float ax = 0.f, ay = 0.f, az = 0.f;
  int visits = 0, accepted = 0;
  int cursor = active ? 0 : n_nodes;
  int wbase = INT_MIN / 2;
  constexpr float kRel = 12.0f * 5.97e-8f;  // unit roundoffs of d^2, theta^2 d^2 and l^2 (~ t2d2 at a tie)
  constexpr float kSqrt3 = 1.7320508f;
  const float theta = sqrtf(theta2), itheta = theta > 0.f ? 1.0f / theta : 0.f;
  while (true) {
    const int n = __reduce_min_sync(0xffffffffu, cursor);
    if (n >= n_nodes) break;
    if ((unsigned)(n - wbase) >= (unsigned)kWin) {
      wbase = n;
      __syncwarp();
      const int j = n + lane;
      if (j < n_nodes) {
        const float4 a = __ldg(&A[j]);
        const NodeB32 b = B[j];
        win->r[lane].a = a;
        // p = sqrt3*theta/len, q = sqrt3*len/theta: 2|d|delta <= delta*(d2*p + q) with
        // the AM-GM pivot at |d| = len/theta, where MAC ties happen
        const float il = b.l2 > 0.f ? rsqrt_approx(b.l2) : 0.f;
        win->r[lane].b = make_float4(b.l2, __int_as_float(b.skip), kSqrt3 * theta * il,
                                     kSqrt3 * b.l2 * il * itheta);
      }
      __syncwarp();
    }
    const WinRec32& rec = win->r[n - wbase];
    const float4 a = rec.a;
    const float4 b = rec.b;
    const bool mine = cursor == n;
    const float dx = a.x - qx, dy = a.y - qy, dz = a.z - qz;
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float t2d2 = theta2 * d2;
    bool acc = b.x < t2d2;
    const float band = fmaf(gA, fmaf(d2, b.z, b.w), fmaf(kRel, t2d2, gB));
    const bool near = mine && fabsf(t2d2 - b.x) <= band;
    if (__any_sync(0xffffffffu, near)) {  // warp-uniform branch, rarely taken
      if (near) acc = mac_exact(A64, B64, n, qpx[qi], qpy[qi], qpz[qi], theta2_64);
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
  return Trav32Out{ax, ay, az, visits, accepted};
}

struct Trav64Out {
  double fx, fy, fz;
  int visits, accepted;
};

// FP64 traversal: the reference's arithmetic and order exactly.  gq = G*m_q.
__device__ __forceinline__ Trav64Out traverse64(const double4* __restrict__ A,
                                                const NodeB64* __restrict__ B, int n_nodes,
                                                double qx, double qy, double qz, double gq,
                                                bool active, double theta2, double eps2,
                                                Win64* win, int lane) {
  Trav64Out o{0.0, 0.0, 0.0, 0, 0};
  int cursor = active ? 0 : n_nodes;
  int wbase = INT_MIN / 2;
  while (true) {
    const int n = __reduce_min_sync(0xffffffffu, cursor);
    if (n >= n_nodes) break;
    if ((unsigned)(n - wbase) >= (unsigned)kWin) {
      wbase = n;
      __syncwarp();
      const int j = n + lane;
      if (j < n_nodes) {
        win->a[lane] = A[j];
        win->b[lane] = B[j];
      }
      __syncwarp();
    }
    if (cursor == n) {
      const double4 a = win->a[n - wbase];
      const NodeB64 b = win->b[n - wbase];
      const double dx = __dsub_rn(qx, a.x), dy = __dsub_rn(qy, a.y), dz = __dsub_rn(qz, a.z);
      const double d2 =
          __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      o.visits++;
      if (b.l2 < __dmul_rn(theta2, d2)) {
        o.accepted++;
        const double denom = __dadd_rn(d2, eps2);
        if (denom > 0.0) {
          const double w = __ddiv_rn(__dmul_rn(gq, a.w), __dmul_rn(denom, __dsqrt_rn(denom)));
          o.fx = __dsub_rn(o.fx, __dmul_rn(w, dx));
          o.fy = __dsub_rn(o.fy, __dmul_rn(w, dy));
          o.fz = __dsub_rn(o.fz, __dmul_rn(w, dz));
        }
        cursor = (int)b.skip;
      } else {
        cursor = n + 1;
      }
    }
  }
  return o;
}

// Per-lane guard coefficients (see traverse32).
__device__ __forceinline__ void guard_coeffs(float qmag, float cmag, float theta2, float& gA,
                                             float& gB) {
  const float delta = (qmag + cmag) * 5.97e-8f;
  gA = 1.25f * delta * theta2;                    // times (d2*p + q) >= 2*sqrt3*|d|
  gB = 3.75f * delta * delta * theta2 + 1e-37f;
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

// ---------------------------------------------------------------- BH iterate
template <typename Real>
struct WinOf;
template <>
struct WinOf<float> {
  using T = WinBuf32;
};
template <>
struct WinOf<double> {
  using T = Win64;
};

struct F32Params {
  float theta2, eps2;
};

template <typename Real, bool kGuardZero, int kT>
__global__ void __launch_bounds__(kT, (sizeof(Real) == 4 ? 1280 : 768) / kT) k_bh_iterate(
    TreeRecords tr, int n_nodes, TemplateView tv, const IterState* __restrict__ st, SimParams sp,
    F32Params f, double* partials, float cmag, int nblocks, int per_sm) {
  if (st->done) return;
  // (An SM-contiguous block->chunk remap for L1 sharing was measured 3%
  // slower -- per-SM load imbalance -- so blocks map to chunks in order.)
  (void)per_sm;
  const int chunk = (int)blockIdx.x;
  if (chunk >= nblocks) return;
  __shared__ typename WinOf<Real>::T wins[kT / 32];
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
    const float qx = (float)y[0], qy = (float)y[1], qz = (float)y[2];
    float gA, gB;
    guard_coeffs(fmaxf(fabsf(qx), fmaxf(fabsf(qy), fabsf(qz))), cmag, f.theta2, gA, gB);
    Trav32Out o = traverse32<kGuardZero>(tr.a32, tr.b32, tr.a64, tr.b64, n_nodes, qx, qy, qz,
                                         active, f.theta2, sp.theta2, f.eps2, gA, gB, tv.px,
                                         tv.py, tv.pz, i, &wins[wl], lane);
    const double gq = sp.G * mq;
    F[0] = gq * (double)o.ax;
    F[1] = gq * (double)o.ay;
    F[2] = gq * (double)o.az;
    nv = o.visits;
    na = o.accepted;
  } else {
    Trav64Out o = traverse64(tr.a64, tr.b64, n_nodes, y[0], y[1], y[2], __dmul_rn(sp.G, mq),
                             active, sp.theta2, sp.eps2, &wins[wl], lane);
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

// ---------------------------------------------------------------- BH operator
template <typename Real, bool kGuardZero>
__global__ void __launch_bounds__(kForceThreads) k_bh_operator(
    TreeRecords tr, int n_nodes, const double* __restrict__ qx_, const double* __restrict__ qy_,
    const double* __restrict__ qz_, const double* __restrict__ qm_, const int* __restrict__ order,
    int64_t m, double theta2, double G, double eps2, F32Params f, double* __restrict__ fout,
    long long* __restrict__ visits, long long* __restrict__ accepted, float cmag) {
  __shared__ typename WinOf<Real>::T wins[kWarps];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t i = ((int64_t)blockIdx.x * kWarps + wl) * 32 + lane;
  const bool active = i < m;
  double q[3] = {0, 0, 0}, qm = 0.0;
  if (active) {
    q[0] = qx_[i];
    q[1] = qy_[i];
    q[2] = qz_[i];
    qm = qm_[i];
  }
  double F[3];
  int nv, na;
  if constexpr (sizeof(Real) == 4) {
    const float fx = (float)q[0], fy = (float)q[1], fz = (float)q[2];
    float gA, gB;
    guard_coeffs(fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz))), cmag, f.theta2, gA, gB);
    Trav32Out o = traverse32<kGuardZero>(tr.a32, tr.b32, tr.a64, tr.b64, n_nodes, fx, fy, fz,
                                         active, f.theta2, theta2, f.eps2, gA, gB, qx_, qy_, qz_,
                                         i, &wins[wl], lane);
    const double gq = G * qm;
    F[0] = gq * (double)o.ax;
    F[1] = gq * (double)o.ay;
    F[2] = gq * (double)o.az;
    nv = o.visits;
    na = o.accepted;
  } else {
    Trav64Out o = traverse64(tr.a64, tr.b64, n_nodes, q[0], q[1], q[2], __dmul_rn(G, qm), active,
                             theta2, eps2, &wins[wl], lane);
    F[0] = o.fx;
    F[1] = o.fy;
    F[2] = o.fz;
    nv = o.visits;
    na = o.accepted;
  }
  if (!active) return;
  const int64_t dst = order ? order[i] : i;
  fout[dst * 3] = F[0];
  fout[dst * 3 + 1] = F[1];
  fout[dst * 3 + 2] = F[2];
  if (visits) visits[dst] = nv;
  if (accepted) accepted[dst] = na;
}

// ---------------------------------------------------------------- direct sum
constexpr int kTile = 1024;

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

template <bool kGuard>
__global__ void __launch_bounds__(kForceThreads, 3) k_direct_iterate32(
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
template <bool kNewton>
__global__ void __launch_bounds__(kForceThreads, 3) k_gpe32(const float4* __restrict__ src,
                                                            int64_t n,
                                                            const double* __restrict__ px,
                                                            const double* __restrict__ py,
                                                            const double* __restrict__ pz,
                                                            const double* __restrict__ mq,
                                                            int64_t m, float eps,
                                                            const IterState* st,
                                                            double* partials) {
  if (st && st->done) return;
  __shared__ float4 sm[kTile];
  constexpr int Q = kDirectQPT;  // 4 queries = pack 0 (MUFU) + pack 1 (Newton)
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * (kForceThreads * Q);
  float2 qx[2], qy[2], qz[2];
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
  const float2 e2 = make_float2(eps, eps);
  const float2 two = make_float2(2.f, 2.f);
  for (int64_t t0 = 0; t0 < n; t0 += kTile) {
    const int jmax = (int)((n - t0) < (int64_t)kTile ? (n - t0) : (int64_t)kTile);
    __syncthreads();
    for (int j = threadIdx.x; j < jmax; j += kForceThreads) sm[j] = __ldg(&src[t0 + j]);
    __syncthreads();
    float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int j = 0; j < jmax; j++) {
      const float4 s = sm[j];
      {  // pack 0: MUFU reciprocal
        const float2 dx = sub2s(s.x, qx[0]), dy = sub2s(s.y, qy[0]), dz = sub2s(s.z, qz[0]);
        const float2 d2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
        float2 den;
        den.x = sqrt_approx(d2.x);
        den.y = sqrt_approx(d2.y);
        den = add2(den, e2);
        float2 r;
        r.x = rcp_approx(den.x);
        r.y = rcp_approx(den.y);
        a0 = fma2s(s.w, r, a0);
      }
      {  // pack 1: Newton reciprocal (accumulates -m/x)
        const float2 dx = sub2s(s.x, qx[1]), dy = sub2s(s.y, qy[1]), dz = sub2s(s.z, qz[1]);
        const float2 d2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
        float2 den;
        den.x = sqrt_approx(d2.x);
        den.y = sqrt_approx(d2.y);
        den = add2(den, e2);
        float2 w;
        if (kNewton) {
          w.x = __int_as_float(0xFEF311C3u - __float_as_uint(den.x));
          w.y = __int_as_float(0xFEF311C3u - __float_as_uint(den.y));
#pragma unroll
          for (int it = 0; it < 3; it++) w = mul2(w, fma2(den, w, two));
        } else {
          w.x = -rcp_approx(den.x);
          w.y = -rcp_approx(den.y);
        }
        a1 = fma2s(s.w, w, a1);
      }
    }
    acc[0] += (double)a0.x;
    acc[1] += (double)a0.y;
    acc[2] -= (double)a1.x;
    acc[3] -= (double)a1.y;
  }
  double tot = 0.0;
#pragma unroll
  for (int k = 0; k < Q; k++) {
    const int64_t i = base + threadIdx.x + k * kForceThreads;
    if (i < m) tot += mq[i] * acc[k];
  }
  tot = warp_sum(tot);
  if (lane == 0) partials[(int64_t)blockIdx.x * kWarps + wl] = tot;
}

__global__ void __launch_bounds__(kForceThreads) k_gpe64(const double4* __restrict__ src, int64_t n,
                                                         const double* __restrict__ px,
                                                         const double* __restrict__ py,
                                                         const double* __restrict__ pz,
                                                         const double* __restrict__ mq, int64_t m,
                                                         double eps, const IterState* st,
                                                         double* partials) {
  if (st && st->done) return;
  __shared__ double4 sm[kTile / 2];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * kForceThreads + threadIdx.x;
  const double qx = i < m ? px[i] : 0.0, qy = i < m ? py[i] : 0.0, qz = i < m ? pz[i] : 0.0;
  double acc = 0.0;
  for (int64_t t0 = 0; t0 < n; t0 += kTile / 2) {
    const int jmax = (int)((n - t0) < (int64_t)(kTile / 2) ? (n - t0) : (int64_t)(kTile / 2));
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
  if (lane == 0) partials[(int64_t)blockIdx.x * kWarps + wl] = tot;
}

inline unsigned grid_for(int64_t items, int64_t per_block) {
  return (unsigned)((items + per_block - 1) / per_block);
}

}  // namespace

// ------------------------------------------------------------------ launchers
static int bh_block() {
  static int b = [] {
    const char* e = getenv("FGA_BH_BLOCK");
    int v = e ? atoi(e) : 128;
    return (v == 64 || v == 128 || v == 256) ? v : 128;
  }();
  return b;
}
int64_t bh_iterate_warps(int64_t m) {
  const int t = bh_block();
  return (int64_t)grid_for(m, t) * (t / 32);
}
int64_t direct_iterate_warps(int64_t m, int precision) {
  const int64_t per = precision ? kForceThreads : kForceThreads * kDirectQPT;
  return (int64_t)grid_for(m, per) * kWarps;
}
int64_t gpe_warps(int64_t m, int precision) { return direct_iterate_warps(m, precision); }

template <int kT>
static void launch_bh_iterate_t(const TreeDev& T, const TemplateView& tv, const IterState* st,
                                const SimParams& sp, double* partials, int precision,
                                cudaStream_t s) {
  const int nb = (int)grid_for(tv.m, kT);
  const int per = 0;
  const unsigned g = (unsigned)nb;
  const F32Params f{(float)sp.theta2, (float)sp.eps2};
  const bool gz = !(sp.eps2 > 0.0);
  const int nn = (int)T.n_nodes;
  const float cm = (float)T.cmag;
  if (precision)
    k_bh_iterate<double, false, kT><<<g, kT, 0, s>>>(T.records(), nn, tv, st, sp, f, partials, cm,
                                                     nb, per);
  else if (gz)
    k_bh_iterate<float, true, kT><<<g, kT, 0, s>>>(T.records(), nn, tv, st, sp, f, partials, cm,
                                                   nb, per);
  else
    k_bh_iterate<float, false, kT><<<g, kT, 0, s>>>(T.records(), nn, tv, st, sp, f, partials, cm,
                                                    nb, per);
}

void launch_bh_iterate(const TreeDev& T, const TemplateView& tv, const IterState* st,
                       const SimParams& sp, double* partials, int precision, cudaStream_t s) {
  if (tv.m <= 0) return;
  switch (bh_block()) {
    case 64: launch_bh_iterate_t<64>(T, tv, st, sp, partials, precision, s); break;
    case 256: launch_bh_iterate_t<256>(T, tv, st, sp, partials, precision, s); break;
    default: launch_bh_iterate_t<128>(T, tv, st, sp, partials, precision, s); break;
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
  if (precision)
    k_gpe64<<<grid_for(m, kForceThreads), kForceThreads, 0, s>>>(ref.p64, ref.n, px, py, pz, mq, m,
                                                                 eps, st, partials);
  else if (eps > 0.0)
    k_gpe32<true><<<grid_for(m, kForceThreads * kDirectQPT), kForceThreads, 0, s>>>(
        ref.p32, ref.n, px, py, pz, mq, m, (float)eps, st, partials);
  else  // eps == 0: keep IEEE rcp semantics (1/0 = inf) on every pair
    k_gpe32<false><<<grid_for(m, kForceThreads * kDirectQPT), kForceThreads, 0, s>>>(
        ref.p32, ref.n, px, py, pz, mq, m, (float)eps, st, partials);
}

void launch_bh_operator(const TreeDev& T, const double* qx, const double* qy, const double* qz,
                        const double* qm, const int* order, int64_t m, double theta, double G,
                        double eps2, double* fout, long long* visits, long long* accepted,
                        int precision, cudaStream_t s) {
  if (m <= 0) return;
  const unsigned g = grid_for(m, kForceThreads);
  const double theta2 = theta * theta;
  const F32Params f{(float)theta2, (float)eps2};
  const int nn = (int)T.n_nodes;
  const float cm = (float)T.cmag;
  if (precision)
    k_bh_operator<double, false><<<g, kForceThreads, 0, s>>>(T.records(), nn, qx, qy, qz, qm,
                                                             order, m, theta2, G, eps2, f, fout,
                                                             visits, accepted, cm);
  else if (!(eps2 > 0.0))
    k_bh_operator<float, true><<<g, kForceThreads, 0, s>>>(T.records(), nn, qx, qy, qz, qm,
                                                           order, m, theta2, G, eps2, f, fout,
                                                           visits, accepted, cm);
  else
    k_bh_operator<float, false><<<g, kForceThreads, 0, s>>>(T.records(), nn, qx, qy, qz, qm,
                                                            order, m, theta2, G, eps2, f, fout,
                                                            visits, accepted, cm);
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
