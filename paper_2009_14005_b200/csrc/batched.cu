// batched.cu -- K13: persistent many-pair registration (BASELINE configs[4]:
// thousands of independent 3DMatch-fragment-sized pairs).
//
// One CTA (32 warps) runs the WHOLE reference register() for one pair at a
// time (registration.py:91-166) and then takes the next pair from a global
// counter, so there is no host round-trip and no launch per iteration:
//   normalize (numpy-order column means)  -> NIV lattice masses + rescale
//   -> tree build in shared memory (exact fp64 split keys, (key, index)
//      bitonic sort == the reference's stable partition order, closed-form
//      preorder emission, level-synchronous mass/COM reduction, mirrored
//      traversal records) -> template Morton order -> energy
//   -> iterations: warp-coherent exact-MAC traversal over the pair's tree
//      (records L1/L2-resident), fused Euler-Cromer step + Kabsch moments,
//      fp64 SVD update by one thread, transform applied at once
//   -> energy -> denormalized transform.
// Everything a pair needs lives in this CTA's shared memory plus a private
// global scratch slot, so pairs are independent and the result of a pair does
// not depend on which CTA ran it (deterministic).
#include "../../include/fga.h"
#include "fga_batched.cuh"
#include "fga_device.cuh"

namespace fga {
namespace {

#ifndef FGA_KBT
#define FGA_KBT 1024
#endif
constexpr int kBT = FGA_KBT;  // threads per CTA
constexpr int kBW = kBT / 32;
static_assert(kBT % 32 == 0 && kBT >= 64, "whole warps, at least two");

// ---------------------------------------------------------------- block helpers
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int j = 0; j < kBW; j++) t += red[j];  // fixed order, every thread
  return t;
}
// numpy's sum of a[0..n) (bit-exact, see np_pairwise_sum), whole block;
// red holds >= 64 doubles.  The recursion is complete down to depth d0 <= 6,
// one thread per node there, then the top levels pairwise in order.
__device__ double block_np_sum(const double* a, int n, double* red) {
  const int d0 = np_pairwise_depth(n, 6);
  __syncthreads();
  if (threadIdx.x < (1u << d0)) {
    int64_t lo, len;
    np_pairwise_node(n, d0, threadIdx.x, lo, len);
    red[threadIdx.x] = np_pairwise_sum(a + lo, len);
  }
  __syncthreads();
  for (int l = d0; l > 0; l--) {
    const int cnt = 1 << (l - 1);
    double v = 0.0;
    if (threadIdx.x < (unsigned)cnt) v = __dadd_rn(red[2 * threadIdx.x], red[2 * threadIdx.x + 1]);
    __syncthreads();
    if (threadIdx.x < (unsigned)cnt) red[threadIdx.x] = v;
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}
__device__ __forceinline__ double block_min(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = red[0];
  for (int j = 1; j < kBW; j++) t = fmin(t, red[j]);
  return t;
}
__device__ __forceinline__ double block_max(double v, double* red) {
  return -block_min(-v, red);
}

// (key, index) bitonic sort of P = 2^k entries in shared memory; ties on key
// are ordered by index, i.e. a stable sort of the unpadded prefix.
__device__ void bitonic_sort(unsigned long long* key, int* idx, int P) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += kBT) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const unsigned long long ka = key[i], kb = key[l];
          const int ia = idx[i], ib = idx[l];
          const bool gt = ka > kb || (ka == kb && ia > ib);
          if (gt == up) {
            key[i] = kb;
            key[l] = ka;
            idx[i] = ib;
            idx[l] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
}

// exclusive scan of n ints in smem (in place), returns the total
__device__ int block_exclusive_scan(int* a, int n, int* red) {
  const int per = (n + kBT - 1) / kBT;
  const int b0 = threadIdx.x * per, b1 = min(n, b0 + per);
  int s = 0;
  for (int i = b0; i < b1; i++) s += a[i];
  // warp inclusive scan of s
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) red[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int j = 0; j < kBW; j++) {
      const int t = red[j];
      red[j] = acc;
      acc += t;
    }
    red[kBW] = acc;
  }
  __syncthreads();
  int run = red[w] + x - s;
  for (int i = b0; i < b1; i++) {
    const int t = a[i];
    a[i] = run;
    run += t;
  }
  const int total = red[kBW];
  __syncthreads();
  return total;
}

__device__ __forceinline__ int64_t ub_key(const unsigned long long* keys, int64_t lo, int64_t hi,
                                          unsigned long long bound) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] > bound) hi = mid; else lo = mid + 1;
  }
  return lo;
}
__device__ __forceinline__ int64_t lb_key(const unsigned long long* keys, int64_t lo, int64_t hi,
                                          unsigned long long bound) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] >= bound) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// numpy pairwise sum (n <= 128 path + recursion) of m[idx[lo..lo+cnt)]
__device__ double pairwise_gather(const int* idx, int lo, int cnt, const double* m) {
  if (cnt < 8) {
    double r = 0.0;
    for (int i = 0; i < cnt; i++) r = __dadd_rn(r, m[idx[lo + i]]);
    return r;
  }
  if (cnt <= 128) {
    double r[8];
    int i;
    for (int j = 0; j < 8; j++) r[j] = m[idx[lo + j]];
    for (i = 8; i < cnt - (cnt % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], m[idx[lo + i + j]]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < cnt; i++) res = __dadd_rn(res, m[idx[lo + i]]);
    return res;
  }
  int n2 = cnt / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_gather(idx, lo, n2, m), pairwise_gather(idx, lo + n2, cnt - n2, m));
}

// numpy-order column mean (registration.py -> normalize.py:47-48): warp w<6
// streams column (w%3) of cloud (w<3 ? x : y) through a double buffer; lane 0
// adds sequentially.
__device__ void colmeans(const double* x, int n, const double* y, int m, double* buf,
                         double* out6) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w < 6) {
    const double* p = w < 3 ? x : y;
    const int cnt = w < 3 ? n : m;
    const int k = w % 3;
    double* b = buf + w * 512;
    double s = 0.0;
    for (int c0 = 0; c0 < cnt; c0 += 256) {
      const int len = min(256, cnt - c0);
      for (int j = lane; j < len; j += 32) b[j] = p[(int64_t)(c0 + j) * 3 + k];
      __syncwarp();
      if (lane == 0)
        for (int j = 0; j < len; j++) s = __dadd_rn(s, b[j]);
      __syncwarp();
    }
    if (lane == 0) out6[w] = __ddiv_rn(s, (double)cnt);
  }
  __syncthreads();
}

struct BatchSmem {
  unsigned long long* keys;  // P
  int* idx;                  // P
  int* offs;                 // nmax + 1
  signed char* clev;         // nmax + 1
  int* counts;               // rho^3
  WinBuf32* wins;            // kBW
  double* red;               // 64
  double* part;              // kBW * kPartialStride
  PairState* st;
};

}  // namespace

// The persistent kernel.  Scratch slot = blockIdx.x.
// kGuardZero: epsilon = 0, so a template point on a reference leaf's COM has
// d2 + eps2 = 0 and the reference skips that term (_kernels.py:38-42)
template <bool kGuardZero>
__global__ void __launch_bounds__(kBT, 1) k_register_batch(BatchArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BatchSmem S;
  {
    unsigned char* p = smem_raw;
    S.wins = reinterpret_cast<WinBuf32*>(p);
    p += sizeof(WinBuf32) * kBW;
    S.keys = reinterpret_cast<unsigned long long*>(p);
    p += sizeof(unsigned long long) * a.P;
    S.part = reinterpret_cast<double*>(p);
    p += sizeof(double) * kBW * kPartialStride;
    S.red = reinterpret_cast<double*>(p);
    p += sizeof(double) * 64;
    S.st = reinterpret_cast<PairState*>(p);
    p += (sizeof(PairState) + 15) / 16 * 16;
    S.idx = reinterpret_cast<int*>(p);
    p += sizeof(int) * a.P;
    S.offs = reinterpret_cast<int*>(p);
    p += sizeof(int) * (a.nmax + 1);
    S.counts = reinterpret_cast<int*>(p);
    p += sizeof(int) * a.ncell;
    S.clev = reinterpret_cast<signed char*>(p);
  }
  __shared__ int next_pair;
  __shared__ int next_chunk;
  PairState& st = *S.st;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int L = a.p.max_depth;
  // per-slot global scratch
  const size_t slot = blockIdx.x;
  double* xn = a.scratch.xn + slot * a.nmax * 3;
  double* yn = a.scratch.yn + slot * a.mmax * 3;
  double* mx = a.scratch.mx + slot * a.nmax;
  double* my = a.scratch.my + slot * a.mmax;
  int* flat = a.scratch.flat + slot * (size_t)max(a.nmax, a.mmax);
  float4* const ref32_slot = a.scratch.ref32 + slot * a.nmax;
  const size_t cap = a.node_cap;
  signed char* nlev = a.scratch.nlev + slot * cap;
  int* nstart = a.scratch.nstart + slot * cap;
  int* nocc = a.scratch.nocc + slot * cap;
  int* nskip = a.scratch.nskip + slot * cap;
  int* nchild = a.scratch.nchild + slot * cap * 8;
  double* nmass = a.scratch.nmass + slot * cap;
  double* nmc = a.scratch.nmc + slot * cap * 3;
  double* nlen = a.scratch.nlen + slot * cap;
  float4* const ra32 = a.scratch.ra32 + slot * cap;
  NodeB32* rb32 = a.scratch.rb32 + slot * cap;
  double4* const ra64_slot = a.scratch.ra64 + slot * cap;
  NodeB64* const rb64_slot = a.scratch.rb64 + slot * cap;
  double* const tp_slot = a.scratch.tpl + slot * a.mmax * 7;
  const double dt = a.p.dt, eta = a.p.eta, G = a.p.G, eps = a.p.epsilon;
  const double theta2 = a.theta2;

  while (true) {
    if (tid == 0) next_pair = atomicAdd(a.counter, 1);
    __syncthreads();
    const int pi = next_pair;
    __syncthreads();
    if (pi >= a.n_pairs) break;
    const int64_t x0 = a.xoff[pi], y0 = a.yoff[pi];
    const int n = (int)(a.xoff[pi + 1] - x0), m = (int)(a.yoff[pi + 1] - y0);
    const double* X = a.x + x0 * 3;
    const double* Y = a.y + y0 * 3;
    // wide modes keep the pair's records / template / reference copy in
    // per-pair storage (they outlive this CTA's turn on the pair)
    const bool wide = a.mode != 0;
    float4* const ref32 = wide ? a.wide.ref32 + (size_t)pi * a.nmax : ref32_slot;
    double* const tp = wide ? a.wide.tpl + (size_t)pi * a.mmax * 7 : tp_slot;
    double4* const ra64 = wide ? a.wide.a64 + (size_t)pi * cap : ra64_slot;
    NodeB64* const rb64 = wide ? a.wide.b64 + (size_t)pi * cap : rb64_slot;
    float4* const c32 = wide ? a.wide.c32 + (size_t)pi * cap * 2 : nullptr;
    if (a.mode == 2) {  // wide finish: the state the iterations left
      if (tid == 0) st = a.wide.st[pi];
    } else if (tid == 0) {
      st.status = 0;
      st.n = n;
      st.m = m;
      st.done = 0;
      st.converged = 0;
      st.iter = 0;
      st.interactions = 0;
      st.n_nodes = 0;
      st.gpe_initial = st.gpe_final = 0.0;
      if (n <= 0 || m <= 0) st.status = FGA_ERR_EMPTY;
      else if (n > a.nmax || m > a.mmax) st.status = FGA_ERR_UNSUPPORTED;
    }
    __syncthreads();
    if (st.status) goto finish;
    if (a.mode != 2) {  // setup (modes 0, 1); the wide finish starts from the saved state

    // ---------------------------------------------------- normalize
    if (a.opt.normalize) {
      double* mean6 = S.red + 32;
      colmeans(X, n, Y, m, reinterpret_cast<double*>(S.wins), mean6);
      double lo = INFINITY, hi = -INFINITY;
      for (int e = tid; e < 3 * (n + m); e += kBT) {
        const bool isx = e < 3 * n;
        const int f = isx ? e : e - 3 * n;
        const double v = __dsub_rn(isx ? X[f] : Y[f], mean6[(isx ? 0 : 3) + f % 3]);
        lo = fmin(lo, v);
        hi = fmax(hi, v);
      }
      const double l = block_min(lo, S.red);
      const double r = block_max(hi, S.red);
      if (tid == 0) {
        for (int k = 0; k < 6; k++) st.ctx[k] = mean6[k];
        st.ctx[6] = l;
        st.ctx[7] = r;
        st.ctx[8] = a.p.norm_a;
        st.ctx[9] = a.p.norm_b;
        if (!(r > l)) st.status = FGA_ERR_DEGENERATE;
      }
      __syncthreads();
      if (st.status) goto finish;
      const double s = __ddiv_rn(__dsub_rn(a.p.norm_b, a.p.norm_a), __dsub_rn(r, l));
      for (int e = tid; e < 3 * (n + m); e += kBT) {
        const bool isx = e < 3 * n;
        const int f = isx ? e : e - 3 * n;
        const double c = __dsub_rn(isx ? X[f] : Y[f], st.ctx[(isx ? 0 : 3) + f % 3]);
        const double v = __dadd_rn(__dmul_rn(__dsub_rn(c, l), s), a.p.norm_a);
        if (isx) xn[f] = v; else yn[f] = v;
      }
    } else {
      for (int e = tid; e < 3 * n; e += kBT) xn[e] = X[e];
      for (int e = tid; e < 3 * m; e += kBT) yn[e] = Y[e];
      if (tid == 0) {
        for (int k = 0; k < 6; k++) st.ctx[k] = 0.0;
        st.ctx[6] = st.ctx[8] = a.p.norm_a;
        st.ctx[7] = st.ctx[9] = a.p.norm_b;
      }
    }
    __syncthreads();

    // ---------------------------------------------------- masses (registration.py:64-88)
    for (int cloud = 0; cloud < 2; cloud++) {
      const double* P = cloud ? yn : xn;
      double* out = cloud ? my : mx;
      const int cnt = cloud ? m : n;
      const double* wext = cloud ? a.y_weights : a.x_weights;
      if (wext) {
        const double* wp = wext + (cloud ? y0 : x0);
        for (int i = tid; i < cnt; i += kBT) out[i] = fmax(wp[i], 1e-6);
        continue;
      }
      const int rho = a.p.rho;
      for (int c = tid; c < a.ncell; c += kBT) S.counts[c] = 0;
      __syncthreads();
      const double ca = st.ctx[8];
      for (int i = tid; i < cnt; i += kBT) {
        const long long ix = niv_axis(P[i * 3], ca, a.cell_edge, rho);
        const long long iy = niv_axis(P[i * 3 + 1], ca, a.cell_edge, rho);
        const long long iz = niv_axis(P[i * 3 + 2], ca, a.cell_edge, rho);
        const int f = (int)((ix * rho + iy) * rho + iz);
        flat[i] = f;
        atomicAdd(&S.counts[f], 1);
      }
      __syncthreads();
      double nz = 0.0;
      for (int c = tid; c < a.ncell; c += kBT) nz += S.counts[c] > 0 ? 1.0 : 0.0;
      const double nnz = block_sum(nz, S.red);
      const double total_vol = __dmul_rn(nnz, a.cell_vol);
      for (int i = tid; i < cnt; i += kBT) {
        const int c = S.counts[flat[i]];
        const double uni = fmin(__dmul_rn((double)c, a.ball_vol), a.cell_vol);
        const double v = __ddiv_rn(__dmul_rn(total_vol, a.cell_vol), uni > 0.0 ? uni : 1.0);
        out[i] = fmax(v, 1e-6);
      }
      __syncthreads();
    }
    __syncthreads();
    {
      double myx = -INFINITY;
      for (int i = tid; i < m; i += kBT) myx = fmax(myx, my[i]);
      const double sumx = block_np_sum(mx, n, S.red);  // sx.sum() (registration.py:85)
      const double maxy = block_max(myx, S.red);
      const double budget = 16.0 * sqrt((double)n / 2000.0);
      const double floor_ = fmax(1e-6, dt * eta);
      for (int i = tid; i < n; i += kBT) mx[i] = fmin(__ddiv_rn(__dmul_rn(budget, mx[i]), sumx), 0.022);
      for (int i = tid; i < m; i += kBT) my[i] = fmax(__ddiv_rn(__dmul_rn(0.1, my[i]), maxy), floor_);
    }
    __syncthreads();

    // ---------------------------------------------------- tree (bhtree.py:56-122)
    {
      double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int i = tid; i < n; i += kBT)
        for (int k = 0; k < 3; k++) {
          lo[k] = fmin(lo[k], xn[i * 3 + k]);
          hi[k] = fmax(hi[k], xn[i * 3 + k]);
        }
      for (int k = 0; k < 3; k++) {
        const double vlo = block_min(lo[k], S.red);
        const double vhi = block_max(hi[k], S.red);
        if (tid == 0) {
          st.box[k] = vlo;
          st.box[3 + k] = vhi;
        }
      }
      __syncthreads();
      for (int i = tid; i < a.P; i += kBT) {
        unsigned long long key = ~0ull;
        if (i < n) {
          double p[3], bl[3], bh[3];
          for (int k = 0; k < 3; k++) {
            p[k] = xn[i * 3 + k];
            bl[k] = st.box[k];
            bh[k] = st.box[3 + k];
          }
          key = 0;
          for (int l = 0; l < L; l++) {
            unsigned dg = 0;
            for (int k = 0; k < 3; k++) {
              const double c = __dadd_rn(bl[k], __dmul_rn(__dsub_rn(bh[k], bl[k]), 0.5));
              const bool up = p[k] >= c;
              dg = (dg << 1) | (up ? 1u : 0u);
              if (up) bl[k] = c; else bh[k] = c;
            }
            key = (key << 3) | dg;
          }
        }
        S.keys[i] = key;
        S.idx[i] = i;
      }
#if FGA_CHECKS
      {  // (status-based: trap-based checks perturbed this kernel, profiles/r02/README.md)
        __syncthreads();
        bitonic_sort(S.keys, S.idx, a.P);
        int bad = 0;
        for (int i = tid + 1; i < a.P; i += kBT) bad |= S.keys[i - 1] > S.keys[i];
        bad = __syncthreads_or(bad);
        if (bad && tid == 0) st.status = FGA_ERR_STATE;
        __syncthreads();
        if (st.status) goto finish;
      }
#endif
      __syncthreads();
      bitonic_sort(S.keys, S.idx, a.P);
      for (int i = tid; i <= n; i += kBT) {
        const int c = (i == 0 || i == n) ? -1 : common_levels(S.keys[i - 1], S.keys[i], L);
        S.clev[i] = (signed char)c;
      }
      __syncthreads();
      for (int i = tid; i <= n; i += kBT) {
        int cnt = 0;
        if (i < n) {
          const int s = S.clev[i] + 1;
          if (s <= L) cnt = max(1, min(L, S.clev[i + 1] + 1) - s + 1);
        }
        S.offs[i] = cnt;
      }
      __syncthreads();
      const int nn = block_exclusive_scan(S.offs, n + 1, reinterpret_cast<int*>(S.red));
      if (tid == 0) {
        st.n_nodes = nn;
        if ((size_t)nn > cap) st.status = FGA_ERR_UNSUPPORTED;
      }
      __syncthreads();
      if (st.status) goto finish;
      for (int e = tid; e < nn * 8; e += kBT) nchild[e] = -1;
      __syncthreads();
      for (int i = tid; i < n; i += kBT) {
        const int ci = S.clev[i], cn = S.clev[i + 1];
        const int s = ci + 1;
        if (s > L) continue;
        const int e = max(s, min(L, cn + 1));
        const int base = S.offs[i];
        const unsigned long long k = S.keys[i];
        for (int l = s; l <= e; l++) {
          const int node = base + (l - s);
          int end;
          if (l == 0) end = n;
          else if (l > cn) end = i + 1;
          else end = (int)ub_key(S.keys, i + 1, n, k | low_mask(3 * (L - l)));
          nlev[node] = (signed char)l;
          nstart[node] = i;
          nocc[node] = end - i;
          nskip[node] = S.offs[end];
          int parent = -1;
          if (l > s) parent = node - 1;
          else if (l > 0) {
            const int p = (int)lb_key(S.keys, 0, i, k & ~low_mask(3 * (L - l + 1)));
            parent = S.offs[p] + (l - 1 - ((int)S.clev[p] + 1));
          }
          if (parent >= 0) nchild[parent * 8 + ((k >> (3 * (L - l))) & 7u)] = node;
          double blo[3], bhi[3];
          node_bbox(k, l, L, st.box, blo, bhi);
          double sq = 0.0;
          for (int q = 0; q < 3; q++) {
            const double ex = __dsub_rn(bhi[q], blo[q]);
            sq = __dadd_rn(sq, __dmul_rn(ex, ex));
          }
          nlen[node] = __dsqrt_rn(sq);
        }
      }
      __syncthreads();
      // level-synchronous bottom-up aggregates (children in slot order)
      for (int lev = L; lev >= 0; lev--) {
        for (int x = tid; x < nn; x += kBT) {
          if (nlev[x] != lev) continue;
          const int occ = nocc[x];
          double ms, mc[3] = {0.0, 0.0, 0.0};
          if (occ == 1 || lev == L) {
            const int st0 = nstart[x];
            ms = pairwise_gather(S.idx, st0, occ, mx);
            for (int j = 0; j < occ; j++) {
              const int p = S.idx[st0 + j];
              for (int q = 0; q < 3; q++)
                mc[q] = __dadd_rn(mc[q], __dmul_rn(xn[p * 3 + q], mx[p]));
            }
          } else {
            ms = 0.0;
            for (int sl = 0; sl < 8; sl++) {
              const int ch = nchild[x * 8 + sl];
              if (ch < 0) continue;
              ms = __dadd_rn(ms, nmass[ch]);
              for (int q = 0; q < 3; q++) mc[q] = __dadd_rn(mc[q], nmc[ch * 3 + q]);
            }
          }
          nmass[x] = ms;
          for (int q = 0; q < 3; q++) nmc[x * 3 + q] = mc[q];
        }
        __syncthreads();
      }
      // mirrored traversal records
      for (int x = tid; x < nn; x += kBT) {
        const int lev = nlev[x], skip = nskip[x];
        const int mir = lev + nn - skip;
        const int size = skip - x;
        const bool leaf = nocc[x] == 1 || lev == L;
        const double ms = nmass[x];
        const double cx = __ddiv_rn(nmc[x * 3], ms), cy = __ddiv_rn(nmc[x * 3 + 1], ms),
                     cz = __ddiv_rn(nmc[x * 3 + 2], ms);
        const double l2 = __dmul_rn(nlen[x], nlen[x]);
        ra64[mir] = make_double4(cx, cy, cz, ms);
        rb64[mir] = NodeB64{leaf ? -INFINITY : l2, (long long)(mir + size)};
        ra32[mir] = make_float4((float)cx, (float)cy, (float)cz, (float)ms);
        rb32[mir] = NodeB32{leaf ? -INFINITY : (float)l2, mir + size};
        if (wide) {
          c32[2 * mir] = ra32[mir];
          c32[2 * mir + 1] = make_float4(leaf ? -INFINITY : (float)l2, __int_as_float(mir + size),
                                         leaf ? 0.f : (float)nlen[x], 0.f);
        }
      }
      for (int i = tid; i < n; i += kBT)
        ref32[i] = make_float4((float)xn[i * 3], (float)xn[i * 3 + 1], (float)xn[i * 3 + 2],
                               (float)mx[i]);
      if (tid == 0) {
        double cm = 0.0;
        for (int k = 0; k < 6; k++) cm = fmax(cm, fabs(st.box[k]));
        st.cmag = (float)cm;
      }
      __syncthreads();
    }

    // ---------------------------------------------------- template (Hilbert order)
    {
      double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int i = tid; i < m; i += kBT)
        for (int k = 0; k < 3; k++) {
          lo[k] = fmin(lo[k], yn[i * 3 + k]);
          hi[k] = fmax(hi[k], yn[i * 3 + k]);
        }
      double bl[3], bh[3];
      for (int k = 0; k < 3; k++) {
        bl[k] = block_min(lo[k], S.red);
        bh[k] = block_max(hi[k], S.red);
      }
      for (int i = tid; i < a.P; i += kBT) {
        unsigned long long key = ~0ull;
        if (i < m) {
          unsigned long long q[3];
          for (int k = 0; k < 3; k++) {
            const double ext = bh[k] - bl[k];
            double f = ext > 0.0 ? (yn[i * 3 + k] - bl[k]) / ext : 0.0;
            f = fmin(fmax(f, 0.0), 1.0);
            q[k] = (unsigned long long)(f * 1023.0);
          }
          // 10-bit 3-D Hilbert index (Skilling's transpose; see setup.cu
          // hilbert3): more compact 32-query warps than Morton order
          unsigned X[3] = {(unsigned)q[0], (unsigned)q[1], (unsigned)q[2]};
          for (unsigned Q = 1u << 9; Q > 1; Q >>= 1) {
            const unsigned P = Q - 1;
            for (int d = 0; d < 3; d++) {
              if (X[d] & Q) {
                X[0] ^= P;
              } else {
                const unsigned t = (X[0] ^ X[d]) & P;
                X[0] ^= t;
                X[d] ^= t;
              }
            }
          }
          X[1] ^= X[0];
          X[2] ^= X[1];
          unsigned tg = 0;
          for (unsigned Q = 1u << 9; Q > 1; Q >>= 1)
            if (X[2] & Q) tg ^= Q - 1;
          key = 0;
          for (int b = 9; b >= 0; b--)
            key = (key << 3) | ((((X[0] ^ tg) >> b) & 1) << 2) | ((((X[1] ^ tg) >> b) & 1) << 1) |
                  (((X[2] ^ tg) >> b) & 1);
        }
        S.keys[i] = key;
        S.idx[i] = i;
      }
      __syncthreads();
      bitonic_sort(S.keys, S.idx, a.P);
      double sy[3] = {0, 0, 0};
      for (int i = tid; i < m; i += kBT) {
        const int src = S.idx[i];
        tp[i] = yn[src * 3];
        tp[a.mmax + i] = yn[src * 3 + 1];
        tp[2 * a.mmax + i] = yn[src * 3 + 2];
        tp[3 * a.mmax + i] = 0.0;
        tp[4 * a.mmax + i] = 0.0;
        tp[5 * a.mmax + i] = 0.0;
        tp[6 * a.mmax + i] = my[src];
      }
      for (int i = tid; i < m; i += kBT)
        for (int k = 0; k < 3; k++) sy[k] += yn[i * 3 + k];
      for (int k = 0; k < 3; k++) {
        const double v = block_sum(sy[k], S.red);
        if (tid == 0) st.shift[k] = v / (double)m;
      }
      if (tid == 0) {
        for (int k = 0; k < 9; k++) st.Racc[k] = (k % 4 == 0) ? 1.0 : 0.0;
        for (int k = 0; k < 3; k++) st.tacc[k] = 0.0;
      }
      __syncthreads();
    }

    }  // setup

    {
      // energy of the current positions (_kernels.py:53-67), reused below
      auto energy = [&]() -> double {
        const double* px = tp;
        const double* py = tp + a.mmax;
        const double* pz = tp + 2 * a.mmax;
        const double* pm = tp + 6 * a.mmax;
        float4* tile = reinterpret_cast<float4*>(S.keys);  // P*8 bytes >= 1024*16? see host
        const int tileN = min(1024, a.P / 2);
        double tot = 0.0;
        for (int q0 = 0; q0 < m; q0 += 4 * kBT) {
          float2 qx[2], qy[2], qz[2];
          int qi[4];
          for (int k = 0; k < 4; k++) {
            qi[k] = q0 + tid + k * kBT;
            const bool ok = qi[k] < m;
            reinterpret_cast<float*>(&qx[k / 2])[k % 2] = ok ? (float)px[qi[k]] : 0.f;
            reinterpret_cast<float*>(&qy[k / 2])[k % 2] = ok ? (float)py[qi[k]] : 0.f;
            reinterpret_cast<float*>(&qz[k / 2])[k % 2] = ok ? (float)pz[qi[k]] : 0.f;
          }
          double acc[4] = {0, 0, 0, 0};
          for (int t0 = 0; t0 < n; t0 += tileN) {
            const int jmax = min(tileN, n - t0);
            __syncthreads();
            for (int j = tid; j < jmax; j += kBT) tile[j] = ref32[t0 + j];
            __syncthreads();
            float2 a2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            gpe_tile32<true, 2>(tile, jmax, qx, qy, qz, (float)eps, a2);
            acc[0] += (double)a2[0].x;
            acc[1] += (double)a2[0].y;
            acc[2] -= (double)a2[1].x;
            acc[3] -= (double)a2[1].y;
          }
          for (int k = 0; k < 4; k++)
            if (qi[k] < m) tot += pm[qi[k]] * acc[k];
        }
        __syncthreads();
        return -G * block_sum(tot, S.red);
      };

      if (a.mode != 2 && a.opt.compute_gpe) {
        const double e = energy();
        if (tid == 0) st.gpe_initial = e;
      }
      __syncthreads();
      if (a.mode == 2) {  // wide finish: apply the last step transform (pending)
        for (int i = tid; i < m; i += kBT) {
          double* px = tp;
          double* py = tp + a.mmax;
          double* pz = tp + 2 * a.mmax;
          const double y[3] = {px[i], py[i], pz[i]};
          for (int r = 0; r < 3; r++) {
            const double ny = st.R[3 * r] * y[0] + st.R[3 * r + 1] * y[1] + st.R[3 * r + 2] * y[2] + st.t[r];
            (r == 0 ? px : r == 1 ? py : pz)[i] = ny;
          }
        }
        __syncthreads();
      }
      if (a.mode == 1 && tid == 0) {  // the iterations run as wide launches: pending = identity
        for (int k = 0; k < 9; k++) st.R[k] = (k % 4 == 0) ? 1.0 : 0.0;
        for (int k = 0; k < 3; k++) st.t[k] = 0.0;
      }

      // ---------------------------------------------------- iterations
      if (a.mode == 0) {
      const float theta2f = a.theta2f, eps2f = a.eps2f;
      const int nchunks = (m + 31) / 32;
      double* px = tp;
      double* py = tp + a.mmax;
      double* pz = tp + 2 * a.mmax;
      double* vx = tp + 3 * a.mmax;
      double* vy = tp + 4 * a.mmax;
      double* vz = tp + 5 * a.mmax;
      const double* pm = tp + 6 * a.mmax;
      const int nn = (int)st.n_nodes;
      SimParams sp{};
      sp.G = G;
      sp.eta = eta;
      sp.dt = dt;
      double* cpart = a.scratch.cpart + slot * (size_t)kPartialStride * ((a.mmax + 31) / 32);
      for (int it = 0; it < a.p.max_iters; it++) {
        // 32-query chunks are claimed dynamically (the traversal cost varies
        // per chunk); each chunk's moment sums go to its own record and are
        // added in chunk order below, so the result is deterministic
        if (tid == 0) next_chunk = 0;
        __syncthreads();
        const double shift[3] = {st.shift[0], st.shift[1], st.shift[2]};
        while (true) {
          int c = 0;
          if (lane == 0) c = atomicAdd(&next_chunk, 1);
          c = __shfl_sync(0xffffffffu, c, 0);
          if (c >= nchunks) break;
          const int i = c * 32 + lane;
          const bool active = i < m;
          const float qxf = active ? (float)px[i] : 0.f, qyf = active ? (float)py[i] : 0.f,
                      qzf = active ? (float)pz[i] : 0.f;
          float gA, gB;
          guard_coeffs(fmaxf(fabsf(qxf), fmaxf(fabsf(qyf), fabsf(qzf))), st.cmag, theta2f, gA, gB);
          const Trav32Out o = traverse32<kGuardZero>(ra32, rb32, ra64, rb64, nn, qxf, qyf, qzf, active,
                                                theta2f, theta2, eps2f, gA, gB, px, py, pz, i,
                                                &S.wins[w], lane);
          Partial p;
          partial_zero(p);
          if (active) {
            const double y[3] = {px[i], py[i], pz[i]};
            const double v[3] = {vx[i], vy[i], vz[i]};
            const double mq = pm[i];
            const double gq = G * mq;
            const double F[3] = {gq * (double)o.ax, gq * (double)o.ay, gq * (double)o.az};
            double vp[3];
            step_and_accumulate(F, y, v, mq, sp, shift, vp, p);
            vx[i] = vp[0];
            vy[i] = vp[1];
            vz[i] = vp[2];
          }
          const unsigned acc_w = __reduce_add_sync(0xffffffffu, (unsigned)o.accepted);
          p.v[kAccepted] = lane == 0 ? (double)acc_w : 0.0;
#pragma unroll
          for (int k = 0; k < 16; k++) {
            const double v = warp_sum(p.v[k]);
            if (lane == k) cpart[(size_t)c * kPartialStride + k] = v;
          }
        }
        __syncthreads();
        {  // chunk sums in a fixed order, all threads: 16 moments x kBT/16 contiguous chunk ranges,
           // ranges paired in the warp, then the 32 warp results in warp order
          constexpr int kRanges = kBT / 16;
          const int k = tid & 15, part = tid >> 4;
          const int c0 = (int)((int64_t)nchunks * part / kRanges);
          const int c1 = (int)((int64_t)nchunks * (part + 1) / kRanges);
          double v = 0.0;
          for (int c = c0; c < c1; c++) v += __ldcg(&cpart[(size_t)c * kPartialStride + k]);
          v += __shfl_down_sync(0xffffffffu, v, 16);  // part 2w + part 2w+1
          if (lane < 16) S.part[w * 16 + k] = v;
          __syncthreads();
          if (tid < 16) {
            double t = 0.0;
            for (int q = 0; q < kBW; q++) t += S.part[q * 16 + tid];
            S.part[kBW * 16 + tid] = t;
          }
        }
        __syncthreads();
        if (tid == 0) {
          double sums[16];
          for (int k = 0; k < 16; k++) sums[k] = S.part[kBW * 16 + k];
          const double M = (double)m;
          double mu_u[3], mu_w[3], C[9], R[9], t[3];
          for (int k = 0; k < 3; k++) {
            mu_u[k] = sums[kSumU + k] / M;
            mu_w[k] = sums[kSumW + k] / M;
          }
          for (int r = 0; r < 3; r++)
            for (int cc = 0; cc < 3; cc++)
              C[3 * r + cc] = sums[kSumWU + 3 * r + cc] - M * mu_w[r] * mu_u[cc];
          kabsch_rotation(C, R, nullptr);
          double mu_y[3], mu_d[3];
          for (int k = 0; k < 3; k++) {
            mu_y[k] = mu_u[k] + st.shift[k];
            mu_d[k] = mu_w[k] + st.shift[k];
          }
          for (int k = 0; k < 3; k++)
            t[k] = mu_d[k] - (R[3 * k] * mu_y[0] + R[3 * k + 1] * mu_y[1] + R[3 * k + 2] * mu_y[2]);
          double Ra[9], ta[3], delta = 0.0;
          for (int r = 0; r < 3; r++) {
            for (int cc = 0; cc < 3; cc++)
              Ra[3 * r + cc] = R[3 * r] * st.Racc[cc] + R[3 * r + 1] * st.Racc[3 + cc] +
                               R[3 * r + 2] * st.Racc[6 + cc];
            ta[r] = t[r] + (R[3 * r] * st.tacc[0] + R[3 * r + 1] * st.tacc[1] + R[3 * r + 2] * st.tacc[2]);
          }
          for (int r = 0; r < 3; r++) {
            for (int cc = 0; cc < 3; cc++) {
              const double e = Ra[3 * r + cc] - st.Racc[3 * r + cc];
              delta += e * e;
            }
            const double e = ta[r] - st.tacc[r];
            delta += e * e;
          }
          for (int k = 0; k < 9; k++) {
            st.R[k] = R[k];
            st.Racc[k] = Ra[k];
          }
          for (int k = 0; k < 3; k++) {
            st.t[k] = t[k];
            st.tacc[k] = ta[k];
            st.shift[k] = mu_d[k];
          }
          st.interactions += (long long)sums[kAccepted];
          if (a.deltas) a.deltas[(size_t)pi * a.p.max_iters + it] = delta;
          st.iter = it + 1;
          if (delta < a.p.conv_tol) {
            st.converged = 1;
            st.done = 1;
          } else if (it + 1 >= a.p.max_iters) {
            st.done = 1;
          }
        }
        __syncthreads();
        // apply the step transform now (registration.py:135-136)
        for (int i = tid; i < m; i += kBT) {
          const double y[3] = {px[i], py[i], pz[i]};
          const double v[3] = {vx[i], vy[i], vz[i]};
          for (int r = 0; r < 3; r++) {
            const double ny = st.R[3 * r] * y[0] + st.R[3 * r + 1] * y[1] + st.R[3 * r + 2] * y[2] + st.t[r];
            const double nv = st.R[3 * r] * v[0] + st.R[3 * r + 1] * v[1] + st.R[3 * r + 2] * v[2];
            (r == 0 ? px : r == 1 ? py : pz)[i] = ny;
            (r == 0 ? vx : r == 1 ? vy : vz)[i] = nv;
          }
        }
        __syncthreads();
        if (st.done) break;
      }
      }
      if (a.mode != 1 && a.opt.compute_gpe) {
        const double e = energy();
        if (tid == 0) st.gpe_final = e;
      }
      __syncthreads();
    }

  finish:
    __syncthreads();
    if (tid == 0 && a.mode == 1) {  // wide setup: the state the iterations start from
      a.wide.st[pi] = st;
      if (st.status == 0) a.wide.list[0][atomicAdd(&a.wide.counts[0], 1)] = pi;
    }
    if (tid == 0) {
      fga_pair_result r{};
      r.status = st.status;
      r.iterations = st.iter;
      r.converged = st.converged;
      r.gpe_initial = st.gpe_initial;
      r.gpe_final = st.gpe_final;
      r.interactions = st.interactions;
      r.n_nodes = st.n_nodes;
      if (st.status == 0) {
        // denormalize_translation (normalize.py:73-84)
        const double* c = st.ctx;
        const double l = c[6], rr = c[7], aa = c[8], bb = c[9];
        const double inv = (rr - l) / (bb - aa);
        for (int k = 0; k < 9; k++) r.R[k] = st.Racc[k];
        for (int i = 0; i < 3; i++) {
          double v1 = 0.0, v2 = 0.0;
          for (int k = 0; k < 3; k++) {
            v1 += -st.Racc[3 * i + k] * (c[3 + k] + l);
            v2 += st.Racc[3 * i + k] * aa;
          }
          r.t[i] = ((v1 + inv * ((v2 + st.tacc[i]) - aa)) + c[i]) + l;
        }
      }
      a.out[pi] = r;  // (wide setup: provisional, the finish rewrites it)
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ wide iterations
// One iteration of every active pair: a persistent grid of warps claims
// (pair, 32-query chunk) items; each applies the pair's pending step
// transform to its queries (registration.py:135-136), traverses the pair's
// tree (traverse32d<kStatic>: static records, per-warp guard band), takes
// the fused step and writes its chunk's moment sums.  k_wide_update then adds
// each pair's chunk sums in chunk order (deterministic) and runs the rigid
// update.  Pairs are independent, so results do not depend on the schedule.
constexpr int kWT = 128;
#ifndef FGA_WIDE_TPS
#define FGA_WIDE_TPS 1792  // 1280: 505 ms, 1792: 470 ms for the iterations of the 4,096-pair batch
#endif

template <bool kGuardZero>
__global__ void __launch_bounds__(kWT, FGA_WIDE_TPS / kWT) k_wide_forces(BatchArgs a, int cur) {
  __shared__ double hs[3 * kWT];  // the lanes' fp64 fold sums
  __shared__ double qsh[3 * kWT];  // ... and fp64 queries (the exact re-check)
  const int lane = threadIdx.x & 31;
  const int n_active = a.wide.counts[cur];
  const int chunks = a.wide.chunks;
  const int items = n_active * chunks;
  const int* list = a.wide.list[cur];
  SimParams sp{};
  sp.G = a.p.G;
  sp.eta = a.p.eta;
  sp.dt = a.p.dt;
  while (true) {
    int item = 0;
    if (lane == 0) item = atomicAdd(&a.wide.counts[2], 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= items) break;
    const int pi = list[item / chunks];
    const int c = item % chunks;
    const PairState* st = a.wide.st + pi;
    const int m = st->m;
    if (c * 32 >= m) continue;
    const int i = c * 32 + lane;
    const bool active = i < m;
    double* px = a.wide.tpl + (size_t)pi * a.mmax * 7;
    double* py = px + a.mmax;
    double* pz = px + 2 * a.mmax;
    double* vx = px + 3 * a.mmax;
    double* vy = px + 4 * a.mmax;
    double* vz = px + 5 * a.mmax;
    const double* pm = px + 6 * a.mmax;
    float qxf = 0.f, qyf = 0.f, qzf = 0.f;
    if (active) {
      const double y0[3] = {px[i], py[i], pz[i]}, v0[3] = {vx[i], vy[i], vz[i]};
      double y[3], v[3];
      for (int r = 0; r < 3; r++) {  // the pending step transform
        y[r] = st->R[3 * r] * y0[0] + st->R[3 * r + 1] * y0[1] + st->R[3 * r + 2] * y0[2] + st->t[r];
        v[r] = st->R[3 * r] * v0[0] + st->R[3 * r + 1] * v0[1] + st->R[3 * r + 2] * v0[2];
      }
      px[i] = y[0];
      py[i] = y[1];
      pz[i] = y[2];
      vx[i] = v[0];
      vy[i] = v[1];
      vz[i] = v[2];
      qxf = (float)y[0];
      qyf = (float)y[1];
      qzf = (float)y[2];
    }
    // the fp32 query lives in registers across the traversal (the fp64 state
    // is re-read afterwards, L1/L2-resident): otherwise the compiler keeps
    // the doubles and re-converts them (F2F) inside the loop
    asm volatile("" : "+f"(qxf), "+f"(qyf), "+f"(qzf));
    {
      double* q = qsh + 3 * threadIdx.x;
      q[0] = active ? px[i] : 0.0;
      q[1] = active ? py[i] : 0.0;
      q[2] = active ? pz[i] : 0.0;
    }
    float gA, gB;
    guard_coeffs(fmaxf(fabsf(qxf), fmaxf(fabsf(qyf), fabsf(qzf))), st->cmag, a.theta2f, gA, gB);
    const size_t cap = a.node_cap;
    // the pair's record base, formed once: left to itself the compiler
    // re-derives pi * cap * 32 + base on the uniform datapath at every
    // traversal step (8 issue slots per step)
    const float4* c32 = a.wide.c32 + (size_t)pi * cap * 2;
    asm volatile("" : "+l"(c32));
    const Trav32Out o = traverse32d<kGuardZero, false, true>(
        c32, a.wide.a64 + (size_t)pi * cap, a.wide.b64 + (size_t)pi * cap, (int)st->n_nodes, qxf,
        qyf, qzf, active, a.theta2f, a.theta2, a.eps2f, nullptr, nullptr, nullptr, m, hs, gA, gB,
        -1, nullptr, qsh);
    Partial p;
    partial_zero(p);
    if (active) {
      const double y[3] = {px[i], py[i], pz[i]}, v[3] = {vx[i], vy[i], vz[i]};
      const double mq = pm[i];
      const double gq = sp.G * mq;
      const double F[3] = {gq * o.ax, gq * o.ay, gq * o.az};
      double vp[3];
      const double shift[3] = {st->shift[0], st->shift[1], st->shift[2]};
      step_and_accumulate(F, y, v, mq, sp, shift, vp, p);
      vx[i] = vp[0];
      vy[i] = vp[1];
      vz[i] = vp[2];
    }
    const unsigned acc_w = __reduce_add_sync(0xffffffffu, (unsigned)o.accepted);
    p.v[kAccepted] = lane == 0 ? (double)acc_w : 0.0;
    double* cp = a.wide.cpart + ((size_t)pi * chunks + c) * kPartialStride;
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const double sv = warp_sum(p.v[k]);
      if (lane == k) cp[k] = sv;
    }
  }
}

// The rigid update of every active pair (one warp per pair): chunk sums in
// chunk order, then the update of registration.py:131-154 by lane 0.
__global__ void __launch_bounds__(kWT) k_wide_update(BatchArgs a, int cur, int it) {
  const int lane = threadIdx.x & 31;
  const int wa = (int)((blockIdx.x * (int64_t)kWT + threadIdx.x) >> 5);
  if (wa >= a.wide.counts[cur]) return;
  const int pi = a.wide.list[cur][wa];
  PairState& st = a.wide.st[pi];
  const int m = st.m, nchunks = (m + 31) / 32;
  const double* cp = a.wide.cpart + (size_t)pi * a.wide.chunks * kPartialStride;
  double v = 0.0;
  if (lane < 16)
    for (int c = 0; c < nchunks; c++) v += cp[(size_t)c * kPartialStride + lane];
  double sums[16];
#pragma unroll
  for (int k = 0; k < 16; k++) sums[k] = __shfl_sync(0xffffffffu, v, k);
  if (lane != 0) return;
  const double M = (double)m;
  double mu_u[3], mu_w[3], C[9], R[9], t[3];
  for (int k = 0; k < 3; k++) {
    mu_u[k] = sums[kSumU + k] / M;
    mu_w[k] = sums[kSumW + k] / M;
  }
  for (int r = 0; r < 3; r++)
    for (int cc = 0; cc < 3; cc++) C[3 * r + cc] = sums[kSumWU + 3 * r + cc] - M * mu_w[r] * mu_u[cc];
  kabsch_rotation(C, R, nullptr);
  double mu_y[3], mu_d[3];
  for (int k = 0; k < 3; k++) {
    mu_y[k] = mu_u[k] + st.shift[k];
    mu_d[k] = mu_w[k] + st.shift[k];
  }
  for (int k = 0; k < 3; k++)
    t[k] = mu_d[k] - (R[3 * k] * mu_y[0] + R[3 * k + 1] * mu_y[1] + R[3 * k + 2] * mu_y[2]);
  double Ra[9], ta[3], delta = 0.0;
  for (int r = 0; r < 3; r++) {
    for (int cc = 0; cc < 3; cc++)
      Ra[3 * r + cc] = R[3 * r] * st.Racc[cc] + R[3 * r + 1] * st.Racc[3 + cc] +
                       R[3 * r + 2] * st.Racc[6 + cc];
    ta[r] = t[r] + (R[3 * r] * st.tacc[0] + R[3 * r + 1] * st.tacc[1] + R[3 * r + 2] * st.tacc[2]);
  }
  for (int r = 0; r < 3; r++) {
    for (int cc = 0; cc < 3; cc++) {
      const double e = Ra[3 * r + cc] - st.Racc[3 * r + cc];
      delta += e * e;
    }
    const double e = ta[r] - st.tacc[r];
    delta += e * e;
  }
  for (int k = 0; k < 9; k++) {
    st.R[k] = R[k];
    st.Racc[k] = Ra[k];
  }
  for (int k = 0; k < 3; k++) {
    st.t[k] = t[k];
    st.tacc[k] = ta[k];
    st.shift[k] = mu_d[k];
  }
  st.interactions += (long long)sums[kAccepted];
  if (a.deltas) a.deltas[(size_t)pi * a.p.max_iters + it] = delta;
  st.iter = it + 1;
  if (delta < a.p.conv_tol) {
    st.converged = 1;
    st.done = 1;
  } else if (it + 1 >= a.p.max_iters) {
    st.done = 1;
  }
  if (!st.done) a.wide.list[1 - cur][atomicAdd(&a.wide.counts[1 - cur], 1)] = pi;
}

int launch_wide_iteration(const BatchArgs& a, int cur, int it, cudaStream_t s) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // next list empty, chunk counter zero
  FGA_CUDA_TRY(cudaMemsetAsync(a.wide.counts + (1 - cur), 0, sizeof(int), s));
  FGA_CUDA_TRY(cudaMemsetAsync(a.wide.counts + 2, 0, sizeof(int), s));
  const int grid = sms * (FGA_WIDE_TPS / kWT);
  if (a.eps2f > 0.f)
    k_wide_forces<false><<<grid, kWT, 0, s>>>(a, cur);
  else
    k_wide_forces<true><<<grid, kWT, 0, s>>>(a, cur);
  k_wide_update<<<(a.n_pairs + kWT / 32 - 1) / (kWT / 32), kWT, 0, s>>>(a, cur, it);
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

size_t batch_smem_bytes(int P, int nmax, int ncell) {
  size_t b = sizeof(WinBuf32) * kBW + sizeof(unsigned long long) * P +
             sizeof(double) * kBW * kPartialStride + sizeof(double) * 64 +
             (sizeof(PairState) + 15) / 16 * 16 + sizeof(int) * P + sizeof(int) * (nmax + 1) +
             sizeof(int) * ncell + (nmax + 1) + 16;
  return b;
}

int launch_register_batch(const BatchArgs& a, int grid, size_t smem, cudaStream_t s) {
  auto kern = a.eps2f > 0.f ? k_register_batch<false> : k_register_batch<true>;
  FGA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, kBT, smem, s>>>(a);
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

}  // namespace fga
