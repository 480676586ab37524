// setup.cu -- once-per-registration O(N) work on the device: joint
// normalization (normalize.py:36-60), NIV lattice masses (masses.py:85-116),
// the mass rescale (registration.py:85-87), reference-point packing for the
// direct sum / energy kernels, and the Morton ordering of the template.
//
// Every element-wise fp64 expression uses explicit round-to-nearest
// intrinsics in the reference's operation order so the results are
// bit-identical to numpy's (tests/test_gpu_setup.py).  The cloud means use a
// sequential column sum because that IS numpy's order for an axis-0
// reduction of an (n,3) C-contiguous array.
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/fga.h"
#include "fga_device.cuh"

namespace fga {
namespace {

constexpr int kT = 256;
inline unsigned nblk(int64_t n, int t = kT) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// numpy mean(axis=0): sequential accumulation over rows, then / n.  One warp
// per column (x0, x1, x2, y0, y1, y2): the warp streams 256-row chunks of its
// column into shared memory with cp.async (double-buffered) while lane 0 adds
// the previous chunk in row order, so the serial fp64 add chain -- which IS
// numpy's rounding order -- runs at DADD latency instead of load latency.
constexpr int kColChunk = 256;
__global__ void __launch_bounds__(192) k_colmean_seq(const double* __restrict__ x, int64_t n,
                                                     const double* __restrict__ y, int64_t m,
                                                     double* __restrict__ out6) {
  __shared__ double buf[6][2][kColChunk];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* p = w < 3 ? x : y;
  const int64_t cnt = w < 3 ? n : m;
  const int k = w % 3;
  const int64_t nch = (cnt + kColChunk - 1) / kColChunk;
  auto issue = [&](int64_t c) {
    const int64_t r0 = c * kColChunk;
    double* dst = buf[w][c & 1];
    for (int j = lane; j < kColChunk; j += 32) {
      const int64_t r = r0 + j;
      if (r < cnt) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + j);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(p + r * 3 + k));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double s = 0.0;
  if (nch > 0) issue(0);
  for (int64_t c = 0; c < nch; c++) {
    if (c + 1 < nch) {
      issue(c + 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncwarp();
    if (lane == 0) {
      const double* b = buf[w][c & 1];
      const int64_t rem = cnt - c * kColChunk;
      const int len = rem < kColChunk ? (int)rem : kColChunk;
      for (int j = 0; j < len; j++) s = __dadd_rn(s, b[j]);
    }
    __syncwarp();
  }
  if (lane == 0) out6[w] = __ddiv_rn(s, (double)cnt);
}

// min/max over all centred coordinates of both clouds (scalar l, r).
__global__ void k_centred_minmax(const double* __restrict__ x, int64_t n,
                                 const double* __restrict__ y, int64_t m,
                                 const double* __restrict__ mean6, double* __restrict__ part) {
  double lo = INFINITY, hi = -INFINITY;
  const int64_t tot = (n + m) * 3;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const bool isx = e < n * 3;
    const int64_t f = isx ? e : e - n * 3;
    const double v = __dsub_rn(isx ? x[f] : y[f], mean6[(isx ? 0 : 3) + (int)(f % 3)]);
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ double s[2][kT / 32];
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = lo;
    s[1][threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < kT / 32; j++) {
      lo = fmin(lo, s[0][j]);
      hi = fmax(hi, s[1][j]);
    }
    part[blockIdx.x * 2] = fmin(s[0][0], lo);
    part[blockIdx.x * 2 + 1] = fmax(s[1][0], hi);
  }
}

__global__ void k_norm_ctx(const double* __restrict__ part, int nparts, const double* mean6,
                           double a, double b, double* ctx10) {
  if (threadIdx.x != 0) return;
  double lo = part[0], hi = part[1];
  for (int j = 1; j < nparts; j++) {
    lo = fmin(lo, part[2 * j]);
    hi = fmax(hi, part[2 * j + 1]);
  }
  for (int k = 0; k < 6; k++) ctx10[k] = mean6[k];
  ctx10[6] = lo;
  ctx10[7] = hi;
  ctx10[8] = a;
  ctx10[9] = b;
}

// p' = (p - mu - l) * s + a, s = (b - a) / (r - l)   (normalize.py:55-58)
__global__ void k_norm_apply(const double* __restrict__ x, int64_t n, const double* __restrict__ y,
                             int64_t m, const double* __restrict__ ctx10, double* __restrict__ xn,
                             double* __restrict__ yn) {
  const int64_t tot = (n + m) * 3;
  const double l = ctx10[6], r = ctx10[7], a = ctx10[8], b = ctx10[9];
  const double s = __ddiv_rn(__dsub_rn(b, a), __dsub_rn(r, l));
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const bool isx = e < n * 3;
    const int64_t f = isx ? e : e - n * 3;
    const double c = __dsub_rn(isx ? x[f] : y[f], ctx10[(isx ? 0 : 3) + (int)(f % 3)]);
    const double v = __dadd_rn(__dmul_rn(__dsub_rn(c, l), s), a);
    if (isx) xn[f] = v; else yn[f] = v;
  }
}

// ---------------------------------------------------------------- NIV
__global__ void k_niv_hist(const double* __restrict__ pts, int64_t n, int dim, int rho, double a,
                           double edge, int* __restrict__ flat,
                           unsigned long long* __restrict__ counts) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long ix = niv_axis(pts[i * 3], a, edge, rho);
  const long long iy = niv_axis(pts[i * 3 + 1], a, edge, rho);
  long long f = ix * rho + iy;  // masses.py:106-108
  if (dim == 3) f = f * rho + niv_axis(pts[i * 3 + 2], a, edge, rho);
  flat[i] = (int)f;
  atomicAdd(&counts[f], 1ull);
}

__global__ void k_niv_nnz(const unsigned long long* __restrict__ counts, int cells,
                          unsigned long long* __restrict__ nnz) {
  unsigned long long c = 0;
  for (int j = threadIdx.x; j < cells; j += blockDim.x) c += counts[j] > 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ unsigned long long s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int j = 0; j < (int)(blockDim.x >> 5); j++) t += s[j];
    *nnz = t;
  }
}

// cell_value = total_vol * cell_vol / min(count * ball_vol, cell_vol)  (:111-114)
__global__ void k_niv_cells(const unsigned long long* __restrict__ counts, int cells,
                            const unsigned long long* __restrict__ nnz, double cell_vol,
                            double ball_vol, double* __restrict__ value) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cells) return;
  const unsigned long long c = counts[j];
  if (c == 0) {
    value[j] = 0.0;
    return;
  }
  const double total_vol = __dmul_rn((double)*nnz, cell_vol);
  const double uni = fmin(__dmul_rn((double)c, ball_vol), cell_vol);
  value[j] = __ddiv_rn(__dmul_rn(total_vol, cell_vol), uni > 0.0 ? uni : 1.0);
}

__global__ void k_niv_gather(const int* __restrict__ flat, int64_t n,
                             const double* __restrict__ value, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = fmax(value[flat[i]], 1e-6);  // MASS_FLOOR (masses.py:16, :116)
}

__global__ void k_external(const double* __restrict__ w, int64_t n, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = fmax(w[i], 1e-6);  // masses.py:135
}

// ---------------------------------------------------------------- rescale
// ---- numpy's float64 sum of a contiguous 1-D array, bit for bit:
// pairwise_sum_DOUBLE (numpy umath loops_utils.h.src) splits n at
// n2 = n/2 - (n/2)%8 until n <= 128, sums such a block with 8 interleaved
// accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the
// n%8 tail, and n < 8 sequentially from 0.  The recursion tree depends on n
// only: one thread per node at a depth d0 where every shallower node is
// internal (the tree is complete down to d0), then the complete top d0 levels
// are combined pairwise, left + right, in one block.
__global__ void k_pw_nodes(const double* __restrict__ a, int64_t n, int d0, double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (1ll << d0)) return;
  int64_t lo, len;
  np_pairwise_node(n, d0, t, lo, len);
  out[t] = np_pairwise_sum(a + lo, len);
}

// buf holds 2^d0 node sums; ping-pongs with buf + 2^d0; result -> *out
__global__ void k_pw_combine(double* __restrict__ buf, int d0, double* __restrict__ out) {
  double* src = buf;
  double* dst = buf + (1ll << d0);
  for (int l = d0; l > 0; l--) {
    const int cnt = 1 << (l - 1);
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) dst[k] = __dadd_rn(src[2 * k], src[2 * k + 1]);
    __syncthreads();
    double* t = src;
    src = dst;
    dst = t;
  }
  if (threadIdx.x == 0) *out = src[0];
}

// max(sy): per-block partials, then one block (order-free)
__global__ void k_max_partial(const double* __restrict__ sy, int64_t m, double* __restrict__ part) {
  double mx = -INFINITY;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += stride)
    mx = fmax(mx, sy[i]);
  mx = block_reduce<2>(mx);
  if (threadIdx.x == 0) part[blockIdx.x] = mx;
}
__global__ void k_max_final(const double* __restrict__ part, int nparts, double* out) {
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < nparts; j += blockDim.x) mx = fmax(mx, part[j]);
  mx = block_reduce<2>(mx);
  if (threadIdx.x == 0) *out = mx;
}

__global__ void k_rescale(double* sx, int64_t n, double* sy, int64_t m, const double* sm2,
                          double budget, double floor_) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) sx[i] = fmin(__ddiv_rn(__dmul_rn(budget, sx[i]), sm2[0]), 0.022);
  if (i < m) sy[i] = fmax(__ddiv_rn(__dmul_rn(0.1, sy[i]), sm2[1]), floor_);
}

__global__ void k_pack_ref(const double* __restrict__ xn, const double* __restrict__ mx, int64_t n,
                           float4* __restrict__ p32, double4* __restrict__ p64) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = xn[i * 3], y = xn[i * 3 + 1], z = xn[i * 3 + 2], w = mx[i];
  if (p32) p32[i] = make_float4((float)x, (float)y, (float)z, (float)w);
  if (p64) p64[i] = make_double4(x, y, z, w);
}

// deterministic column means (two-level fixed-order tree)
__global__ void k_mean_partial(const double* __restrict__ p, int64_t n, double* __restrict__ part) {
  double s[3] = {0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < 3; k++) s[k] += p[i * 3 + k];
  __shared__ double sm[3][kT / 32];
  for (int k = 0; k < 3; k++) {
    const double v = warp_sum(s[k]);
    if ((threadIdx.x & 31) == 0) sm[k][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int j = 0; j < kT / 32; j++) v += sm[threadIdx.x][j];
    part[blockIdx.x * 3 + threadIdx.x] = v;
  }
}
__global__ void k_mean_final(const double* __restrict__ part, int nparts, int64_t n, double* out3) {
  for (int k = 0; k < 3; k++) {
    double v = 0.0;
    for (int j = threadIdx.x; j < nparts; j += blockDim.x) v += part[j * 3 + k];
    v = block_reduce<0>(v);
    if (threadIdx.x == 0) out3[k] = v / (double)n;
  }
}

__global__ void k_bbox6_partial(const double* __restrict__ p, int64_t n, double* __restrict__ part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < 3; k++) {
      lo[k] = fmin(lo[k], p[i * 3 + k]);
      hi[k] = fmax(hi[k], p[i * 3 + k]);
    }
  for (int k = 0; k < 3; k++)
    for (int o = 16; o > 0; o >>= 1) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  __shared__ double sm[6][kT / 32];
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 3; k++) {
      sm[k][threadIdx.x >> 5] = lo[k];
      sm[3 + k][threadIdx.x >> 5] = hi[k];
    }
  __syncthreads();
  if (threadIdx.x < 6) {
    double v = sm[threadIdx.x][0];
    for (int j = 1; j < kT / 32; j++)
      v = threadIdx.x < 3 ? fmin(v, sm[threadIdx.x][j]) : fmax(v, sm[threadIdx.x][j]);
    part[blockIdx.x * 6 + threadIdx.x] = v;
  }
}
__global__ void k_bbox6_final(const double* __restrict__ part, int nparts, double* out6) {
  for (int k = 0; k < 6; k++) {
    double v = k < 3 ? INFINITY : -INFINITY;
    for (int j = threadIdx.x; j < nparts; j += blockDim.x)
      v = k < 3 ? fmin(v, part[j * 6 + k]) : fmax(v, part[j * 6 + k]);
    v = k < 3 ? block_reduce<1>(v) : block_reduce<2>(v);
    if (threadIdx.x == 0) out6[k] = v;
  }
}

// 21-bit-per-axis Morton key over the cloud's own bbox (locality only).
__device__ __forceinline__ unsigned long long spread21(unsigned long long v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
// 3-D Hilbert index of 21-bit coordinates (Skilling's transpose, then the
// bits interleaved like a Morton key).  Consecutive Hilbert cells are always
// face neighbours, so a 32-query warp of the template is more compact than
// with Morton order: the warp's union traversal visits fewer nodes per query
// (CPU model tools/sim_traversal.py: 1.35 vs 1.40 warp steps per query visit).
__device__ __forceinline__ unsigned long long hilbert3(unsigned x0, unsigned x1, unsigned x2) {
  constexpr int kBits = 21;
  unsigned X[3] = {x0, x1, x2};
  for (unsigned Q = 1u << (kBits - 1); Q > 1; Q >>= 1) {
    const unsigned P = Q - 1;
#pragma unroll
    for (int i = 0; i < 3; i++) {
      if (X[i] & Q) {
        X[0] ^= P;
      } else {
        const unsigned t = (X[0] ^ X[i]) & P;
        X[0] ^= t;
        X[i] ^= t;
      }
    }
  }
  X[1] ^= X[0];
  X[2] ^= X[1];
  unsigned t = 0;
  for (unsigned Q = 1u << (kBits - 1); Q > 1; Q >>= 1)
    if (X[2] & Q) t ^= Q - 1;
  X[0] ^= t;
  X[1] ^= t;
  X[2] ^= t;
  return (spread21(X[0]) << 2) | (spread21(X[1]) << 1) | spread21(X[2]);
}

__global__ void k_morton(const double* __restrict__ p, int64_t n, const double* __restrict__ box,
                         unsigned long long* __restrict__ keys, int* __restrict__ idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned q[3];
  for (int k = 0; k < 3; k++) {
    const double ext = box[3 + k] - box[k];
    double f = ext > 0.0 ? (p[i * 3 + k] - box[k]) / ext : 0.0;
    f = fmin(fmax(f, 0.0), 1.0);
    q[k] = (unsigned)(f * 2097151.0);
  }
#ifdef FGA_MORTON
  keys[i] = (spread21(q[0]) << 2) | (spread21(q[1]) << 1) | spread21(q[2]);
#else
  keys[i] = hilbert3(q[0], q[1], q[2]);
#endif
  idx[i] = (int)i;
}

__global__ void k_gather_tpl(const double* __restrict__ pts, const double* __restrict__ mass,
                             const int* __restrict__ order, int64_t begin, TemplateView tv) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= tv.m) return;
  const int64_t src = order[begin + i];
  tv.px[i] = pts[src * 3];
  tv.py[i] = pts[src * 3 + 1];
  tv.pz[i] = pts[src * 3 + 2];
  tv.vx[i] = 0.0;
  tv.vy[i] = 0.0;
  tv.vz[i] = 0.0;
  const_cast<double*>(tv.mq)[i] = mass[src];
}

__global__ void k_gather_q(const double* __restrict__ q, const double* __restrict__ qm,
                           const int* __restrict__ order, int64_t m, double* qx, double* qy,
                           double* qz, double* qms) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t src = order ? order[i] : i;
  qx[i] = q[src * 3];
  qy[i] = q[src * 3 + 1];
  qz[i] = q[src * 3 + 2];
  qms[i] = qm[src];
}

}  // namespace

size_t scratch_doubles_for(int64_t n) { (void)n; return 6 * 1024 + 64; }

int normalize_pair_dev(const double* x, int64_t n, const double* y, int64_t m, double a, double b,
                       double* xn, double* yn, double* ctx10_dev, double* scratch,
                       size_t scratch_bytes, double* ctx10_host, cudaStream_t s) {
  (void)scratch_bytes;
  double* mean6 = scratch;
  double* part = scratch + 8;
  const int nb = (int)std::min<int64_t>(nblk((n + m) * 3), 592);
  k_colmean_seq<<<1, 192, 0, s>>>(x, n, y, m, mean6);
  k_centred_minmax<<<nb, kT, 0, s>>>(x, n, y, m, mean6, part);
  k_norm_ctx<<<1, 32, 0, s>>>(part, nb, mean6, a, b, ctx10_dev);
  FGA_CUDA_TRY(cudaMemcpyAsync(ctx10_host, ctx10_dev, sizeof(double) * 10, cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  if (!(ctx10_host[7] > ctx10_host[6])) {  // normalize.py:53-54
    set_error("all centered coordinates coincide");
    return FGA_ERR_DEGENERATE;
  }
  k_norm_apply<<<(unsigned)std::min<int64_t>(nblk((n + m) * 3), 4 * 592), kT, 0, s>>>(x, n, y, m, ctx10_dev, xn, yn);
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

int niv_masses_dev(const double* pts, int64_t n, int dim, int rho, double a, double b,
                   int max_depth, double* out, int* flat, long long* counts, double* cell_value,
                   cudaStream_t s) {
  if (rho < 2) {
    set_error("invalid parameter rho");
    return FGA_ERR_INVALID;
  }
  const int64_t ncell64 = (int64_t)rho * rho * (dim == 3 ? rho : 1);
  if (ncell64 > (1ll << 26)) {
    set_error("niv: rho^3 too large for the device lattice");
    return FGA_ERR_UNSUPPORTED;
  }
  const int ncell = (int)ncell64;
  // Python-float scalars exactly as masses.py:97-102 computes them
  const double extent = b - a;
  const double cell_edge = extent / rho;
  const double cell_vol = std::pow(cell_edge, dim);  // masses.py:98
  const double r_ball = extent / (2.0 * max_depth * rho);
  const double ball_vol = dim == 2 ? M_PI * std::pow(r_ball, 2)  // :102
                                   : (4.0 / 3.0) * M_PI * std::pow(r_ball, 3);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(counts);
  FGA_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (ncell + 1), s));
  k_niv_hist<<<nblk(n), kT, 0, s>>>(pts, n, dim, rho, a, cell_edge, flat, cnt);
  k_niv_nnz<<<1, 1024, 0, s>>>(cnt, ncell, cnt + ncell);
  k_niv_cells<<<nblk(ncell), kT, 0, s>>>(cnt, ncell, cnt + ncell, cell_vol, ball_vol, cell_value);
  k_niv_gather<<<nblk(n), kT, 0, s>>>(flat, n, cell_value, out);
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

void launch_external_masses(const double* w, int64_t n, double* out, cudaStream_t s) {
  k_external<<<nblk(n), kT, 0, s>>>(w, n, out);
}

// registration.py:85-87 (FIELD_MASS=16, FIELD_MASS_POINTS=2000,
// REFERENCE_POINT_CAP=0.022, TEMPLATE_PEAK_MASS=0.1, floor max(1e-6, dt*eta))
// depth d0 <= 16 of the pairwise recursion down to which every node is
// internal (sizes at one depth take only a few distinct values)
static int pw_depth(int64_t n) {
  std::vector<int64_t> sizes{n};
  int d = 0;
  while (d < 16) {
    int64_t mn = sizes[0];
    for (int64_t v : sizes) mn = std::min(mn, v);
    if (mn <= 128) break;
    std::vector<int64_t> next;
    for (int64_t v : sizes) {
      int64_t n2 = v / 2;
      n2 -= n2 % 8;
      for (int64_t c : {n2, v - n2})
        if (std::find(next.begin(), next.end(), c) == next.end()) next.push_back(c);
    }
    sizes.swap(next);
    d++;
  }
  return d;
}

size_t pairwise_sum_scratch_doubles(int64_t n) { return 2 * ((size_t)1 << pw_depth(n)); }

// numpy float64 sum(a) of a contiguous device array -> *out (device)
void launch_np_sum(const double* a, int64_t n, double* out, double* scratch, cudaStream_t s) {
  const int d0 = pw_depth(n);
  const int64_t nodes = 1ll << d0;
  k_pw_nodes<<<(unsigned)((nodes + 127) / 128), 128, 0, s>>>(a, n, d0, scratch);
  k_pw_combine<<<1, 1024, 0, s>>>(scratch, d0, out);
}

// registration.py:85-87 (FIELD_MASS=16, FIELD_MASS_POINTS=2000,
// REFERENCE_POINT_CAP=0.022, TEMPLATE_PEAK_MASS=0.1, floor max(1e-6, dt*eta));
// sx.sum() is numpy's pairwise sum, reproduced exactly.  scratch: 8 +
// pairwise_sum_scratch_doubles(n) + 600 doubles.
void launch_rescale(double* sx, int64_t n, double* sy, int64_t m, double dt, double eta,
                    double* scratch, cudaStream_t s) {
  const double budget = 16.0 * std::sqrt((double)n / 2000.0);
  const double floor_ = std::max(1e-6, dt * eta);
  double* pw = scratch + 8;
  double* part = pw + pairwise_sum_scratch_doubles(n);
  launch_np_sum(sx, n, scratch, pw, s);
  const int nb = (int)std::min<int64_t>(nblk(m), 592);
  k_max_partial<<<nb, kT, 0, s>>>(sy, m, part);
  k_max_final<<<1, 256, 0, s>>>(part, nb, scratch + 1);
  k_rescale<<<nblk(std::max(n, m)), kT, 0, s>>>(sx, n, sy, m, scratch, budget, floor_);
}

void launch_pack_ref(const double* xn, const double* mx, int64_t n, float4* p32, double4* p64,
                     cudaStream_t s) {
  k_pack_ref<<<nblk(n), kT, 0, s>>>(xn, mx, n, p32, p64);
}

void launch_mean3(const double* pts, int64_t n, double* scratch, double* out3, cudaStream_t s) {
  const int nb = (int)std::min<int64_t>(nblk(n), 592);
  k_mean_partial<<<nb, kT, 0, s>>>(pts, n, scratch);
  k_mean_final<<<1, 256, 0, s>>>(scratch, nb, n, out3);
}

void launch_bbox(const double* pts, int64_t n, double* scratch, double* out6, cudaStream_t s) {
  const int nb = (int)std::min<int64_t>(nblk(n), 592);
  k_bbox6_partial<<<nb, kT, 0, s>>>(pts, n, scratch);
  k_bbox6_final<<<1, 256, 0, s>>>(scratch, nb, out6);
}

void launch_morton_keys(const double* pts, int64_t n, const double* box6,
                        unsigned long long* keys, int* idx, cudaStream_t s) {
  k_morton<<<nblk(n), kT, 0, s>>>(pts, n, box6, keys, idx);
}

void launch_gather_template(const double* pts, const double* mass, const int* order,
                            int64_t begin, int64_t count, TemplateView tv, cudaStream_t s) {
  tv.m = count;
  if (count <= 0) return;
  k_gather_tpl<<<nblk(count), kT, 0, s>>>(pts, mass, order, begin, tv);
}

void launch_gather_queries(const double* q, const double* qm, const int* order, int64_t m,
                           double* qx, double* qy, double* qz, double* qms, cudaStream_t s) {
  if (m <= 0) return;
  k_gather_q<<<nblk(m), kT, 0, s>>>(q, qm, order, m, qx, qy, qz, qms);
}

}  // namespace fga
