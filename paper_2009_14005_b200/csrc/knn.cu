// knn.cu -- grid-bucketed exact k-nearest-neighbour search and the kNN
// smooth-particle mass field (BASELINE configs[3], north_star item 1).
//
// The reference's default SPM field is the NIV lattice (masses.py:85-116);
// kNN masses are an OPT-IN extension that plugs into the same place as the
// reference's external-weights hook (registration.py:72-83): mass_i =
// (4/3) pi r_k(i)^3 / k, the volume per point of the ball holding the k
// nearest other points -- denser regions get smaller masses, like NIV.
//
// Algorithm: uniform grid with cell edge h = 0.5 (V k / n)^(1/3) over the
// cloud's bbox (measured best of 0.35 / 0.5 / 0.7 / 1.0 on a clustered blob
// and the configs[3] partial-overlap cloud); points counting-sorted by cell
// (cub radix sort on the cell id) and gathered into cell order (fp64 and fp32
// copies), with per-cell offsets over ALL cells so a run of consecutive cells
// is one contiguous range.  One thread per query (queries in cell order for
// warp coherence) scans Chebyshev shells s = 0, 1, 2, ... row by row (a face
// row of the shell is one range; an interior row contributes its two end
// cells), keeping the k best (d^2, index) pairs in registers, and stops once
// it holds k candidates and the k-th d^2 <= (s h + gap)^2 where gap is the
// query's distance to its cell boundary -- every point closer than that lies
// in the scanned cube, so the set is exact.  Candidates are prefiltered in
// fp32 against the current k-th fp64 distance plus the fp32 rounding bound
// (never rejects a true neighbour); distances are fp64; ties by index.
#include <cub/cub.cuh>

#include "../../include/fga.h"
#include "fga_device.cuh"

namespace fga {
namespace {

constexpr int kKnnMax = 32;
constexpr int kKT = 128;

struct Grid {
  double lo[3];
  double h, inv_h;
  int dim[3];
};

__global__ void k_cell_ids(const double* __restrict__ p, int64_t n, Grid g,
                           unsigned* __restrict__ cell, int* __restrict__ idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c[3];
  for (int k = 0; k < 3; k++) {
    int v = (int)floor((p[i * 3 + k] - g.lo[k]) * g.inv_h);
    c[k] = min(max(v, 0), g.dim[k] - 1);
  }
  cell[i] = ((unsigned)c[0] * g.dim[1] + c[1]) * g.dim[2] + c[2];
  idx[i] = (int)i;
}

// count[c] = end[c] - start[c] (0 for an empty cell), in place over `start`
__global__ void k_cell_count(int* __restrict__ start, const int* __restrict__ end, int64_t ncell) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > ncell) return;
  start[c] = c < ncell ? end[c] - start[c] : 0;
}

__global__ void k_cell_bounds(const unsigned* __restrict__ cell_sorted, int64_t n,
                              int* __restrict__ start, int* __restrict__ end) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned c = cell_sorted[i];
  if (i == 0 || cell_sorted[i - 1] != c) start[c] = (int)i;
  if (i == n - 1 || cell_sorted[i + 1] != c) end[c] = (int)i + 1;
}

template <int K>
__device__ __forceinline__ void insert(double (&bd)[K], int (&bi)[K], double d2, int j) {
  // keep ascending (d2, j); bd[K-1] is the current k-th
  if (d2 > bd[K - 1] || (d2 == bd[K - 1] && j >= bi[K - 1])) return;
  int pos = K - 1;
#pragma unroll
  for (int q = K - 1; q > 0; q--) {
    const bool shift = d2 < bd[q - 1] || (d2 == bd[q - 1] && j < bi[q - 1]);
    if (shift && pos == q) {
      bd[q] = bd[q - 1];
      bi[q] = bi[q - 1];
      pos = q - 1;
    }
  }
  bd[pos] = d2;
  bi[pos] = j;
}

// points in cell order as contiguous (x, y, z, pad) records
__global__ void k_gather_cells(const double* __restrict__ p, int64_t n,
                               const int* __restrict__ order, double4* __restrict__ ps,
                               float4* __restrict__ ps32) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t j = order[u];
  const double x = p[j * 3], y = p[j * 3 + 1], z = p[j * 3 + 2];
  ps[u] = make_double4(x, y, z, 0.0);
  ps32[u] = make_float4((float)x, (float)y, (float)z, 0.f);
}

// fp32 prefilter threshold: a candidate whose fp32 d^2 exceeds this cannot
// beat the current k-th fp64 d^2 T.  Coordinates rounded to fp32 are off by
// <= delta each, so |d2_32 - d2| <= 2 sqrt3 delta |d| + 3 delta^2 + 4u d2;
// with |d| <= sqrt(T) at the boundary (plus a 2x / 1.25x margin).
__device__ __forceinline__ float prefilter_threshold(double T, double delta) {
  if (!(T < INFINITY)) return INFINITY;
  const double err = 1.25 * (2.0 * 1.7320508075688772 * delta * sqrt(T) * 1.01 +
                             4.0 * delta * delta + 8.0 * 5.97e-8 * T) + 1e-37;
  return __double2float_ru(T + err);
}

// keep the K smallest d2 ascending (values only: the k-th distance does not
// depend on which of several equidistant points is kept)
template <int K>
__device__ __forceinline__ void insert_d(double (&bd)[K], double d2) {
  if (!(d2 < bd[K - 1])) return;
  int pos = K - 1;
#pragma unroll
  for (int q = K - 1; q > 0; q--) {
    const bool shift = d2 < bd[q - 1];
    if (shift && pos == q) {
      bd[q] = bd[q - 1];
      pos = q - 1;
    }
  }
  bd[pos] = d2;
}

// Same search over the cell-ordered coordinates (contiguous reads per cell;
// the original index is loaded only for an inserted candidate, and not at
// all when only the masses are wanted).
template <int K, bool kIdx>
__global__ void __launch_bounds__(kKT) k_knn_sorted(const double4* __restrict__ ps,
                                                    const float4* __restrict__ ps32, int64_t n,
                                                    const int* __restrict__ order,
                                                    const unsigned* __restrict__ cell_sorted,
                                                    Grid g, double cmax,
                                                    const int* __restrict__ coff, int k,
                                                    long long* __restrict__ out_idx,
                                                    double* __restrict__ out_d2,
                                                    double* __restrict__ out_mass, int dim) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double4 qv = ps[t];
  const double q[3] = {qv.x, qv.y, qv.z};
  const float qf[3] = {(float)qv.x, (float)qv.y, (float)qv.z};
  const double delta =
      (fmax(fabs(q[0]), fmax(fabs(q[1]), fabs(q[2]))) + cmax) * 5.97e-8;  // 2^-24 (|q| + |x|)
  const unsigned cid = cell_sorted[t];
  const int c2 = (int)(cid % g.dim[2]);
  const int c1 = (int)((cid / g.dim[2]) % g.dim[1]);
  const int c0 = (int)(cid / ((unsigned)g.dim[2] * g.dim[1]));
  const int cc[3] = {c0, c1, c2};
  double gap = INFINITY;
  for (int a = 0; a < 3; a++) {
    const double lo = g.lo[a] + cc[a] * g.h;
    gap = fmin(gap, fmin(q[a] - lo, lo + g.h - q[a]));
  }
  gap = fmax(gap, 0.0);
  double bd[K];
  int bi[kIdx ? K : 1];
#pragma unroll
  for (int j = 0; j < K; j++) bd[j] = INFINITY;
  if constexpr (kIdx) {
#pragma unroll
    for (int j = 0; j < K; j++) bi[j] = INT_MAX;
  }
  float thr = INFINITY;
  int found = 0;
  // scan sorted points [b, e) (one or more consecutive cells)
  auto scan = [&](int b, int e) {
    found += e - b;
    for (int u = b; u < e; u++) {
      const float4 f = ps32[u];
      const float fx = f.x - qf[0], fy = f.y - qf[1], fz = f.z - qf[2];
      if (fmaf(fx, fx, fmaf(fy, fy, fz * fz)) > thr || u == t) continue;
      const double4 v = ps[u];
      const double ex = __dsub_rn(v.x, q[0]);
      const double ey = __dsub_rn(v.y, q[1]);
      const double ez = __dsub_rn(v.z, q[2]);
      const double d2 =
          __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
      if constexpr (kIdx) insert<K>(bd, bi, d2, order[u]);
      else insert_d<K>(bd, d2);
      thr = prefilter_threshold(bd[K - 1], delta);
    }
  };
  const int smax = max(g.dim[0], max(g.dim[1], g.dim[2]));
  for (int s = 0; s <= smax; s++) {
    for (int dx = -s; dx <= s; dx++) {
      const int x = cc[0] + dx;
      if (x < 0 || x >= g.dim[0]) continue;
      for (int dy = -s; dy <= s; dy++) {
        const int y = cc[1] + dy;
        if (y < 0 || y >= g.dim[1]) continue;
        const int row = (x * g.dim[1] + y) * g.dim[2];
        if (abs(dx) == s || abs(dy) == s) {  // a face row: z in [cz-s, cz+s], contiguous
          const int z0 = max(cc[2] - s, 0), z1 = min(cc[2] + s, g.dim[2] - 1);
          scan(coff[row + z0], coff[row + z1 + 1]);
        } else {  // interior row of the shell: only its two end cells
          if (cc[2] - s >= 0) scan(coff[row + cc[2] - s], coff[row + cc[2] - s + 1]);
          if (cc[2] + s < g.dim[2]) scan(coff[row + cc[2] + s], coff[row + cc[2] + s + 1]);
        }
      }
    }
    const double cover = (s * g.h + gap) * (1.0 - 1e-12);
    if (found > k && bd[k - 1] <= cover * cover) break;  // found counts the query itself
  }
  const int i = order[t];
  if constexpr (kIdx) {
    if (out_idx)
      for (int j = 0; j < k; j++) out_idx[(int64_t)i * k + j] = bi[j] == INT_MAX ? -1 : bi[j];
  }
  if (out_d2)
    for (int j = 0; j < k; j++) out_d2[(int64_t)i * k + j] = bd[j];
  if (out_mass) {
    const double r = sqrt(bd[k - 1]);
    const double vol = !isfinite(r) ? 0.0
                       : dim == 2   ? M_PI * r * r / k
                                    : (4.0 / 3.0) * M_PI * r * r * r / k;
    out_mass[i] = fmax(vol, 1e-6);
  }
}

}  // namespace

int knn_dev(const double* pts, int64_t n, int dim, int k, long long* out_idx, double* out_d2,
            double* out_mass, DevBuf& scratch, DevBuf& cub_tmp, cudaStream_t s) {
  if (n <= 0) return FGA_OK;
  if (k < 1 || k > kKnnMax || k >= n) {
    set_error("knn: need 1 <= k < n and k <= 32");
    return FGA_ERR_INVALID;
  }
  // bbox on the host (one sync; kNN runs once per registration)
  double box[6];
  {
    FGA_CUDA_TRY(scratch.reserve(sizeof(double) * (6 * 600 + 16)));
    double* b = scratch.as<double>() + 6 * 600;
    launch_bbox(pts, n, scratch.as<double>(), b, s);
    FGA_CUDA_TRY(cudaMemcpyAsync(box, b, sizeof(box), cudaMemcpyDeviceToHost, s));
    FGA_CUDA_TRY(cudaStreamSynchronize(s));
  }
  Grid g;
  double vol = 1.0;
  double ext[3];
  for (int a = 0; a < 3; a++) {
    g.lo[a] = box[a];
    ext[a] = std::max(box[3 + a] - box[a], 1e-12);
    if (a < dim) vol *= ext[a];
  }
  // cell edge: a fraction of the mean k-NN ball (smaller cells scan less
  // volume around the k-NN radius; FGA_KNN_CELL scales it for experiments)
  static const double cell_scale = [] {
    const char* e = getenv("FGA_KNN_CELL");
    const double v = e ? atof(e) : 0.5;
    return v > 0.05 && v < 4.0 ? v : 0.5;
  }();
  double h = cell_scale * (dim == 2 ? std::sqrt(vol * std::max(k, 2) / (double)n)
                                    : std::cbrt(vol * std::max(k, 2) / (double)n));
  for (int a = 0; a < 3; a++) h = std::max(h, ext[a] / 512.0);  // <= 512 cells per axis
  g.h = h;
  g.inv_h = 1.0 / h;
  int64_t ncell = 1;
  for (int a = 0; a < 3; a++) {
    g.dim[a] = std::max(1, (int)std::ceil(ext[a] / h));
    ncell *= g.dim[a];
  }
  const size_t need = sizeof(unsigned) * 2 * n + sizeof(int) * 2 * n +
                      sizeof(int) * 2 * (ncell + 1) + sizeof(double4) * n + sizeof(float4) * n +
                      1024;
  DevBuf& buf = scratch;  // reuse: bbox scratch no longer needed
  FGA_CUDA_TRY(buf.reserve(need));
  char* q = buf.as<char>();
  unsigned* cell = (unsigned*)q;
  q += sizeof(unsigned) * n;
  unsigned* cell_s = (unsigned*)q;
  q += sizeof(unsigned) * n;
  int* idx = (int*)q;
  q += sizeof(int) * n;
  int* order = (int*)q;
  q += sizeof(int) * n;
  int* cstart = (int*)q;
  q += sizeof(int) * (ncell + 1);
  int* cend = (int*)q;
  q += sizeof(int) * (ncell + 1);
  q = (char*)(((uintptr_t)q + 31) & ~(uintptr_t)31);
  double4* ps = (double4*)q;
  float4* ps32 = (float4*)(ps + n);
  double cmax = 0.0;  // max |coordinate|, for the fp32 prefilter bound
  for (int a = 0; a < 6; a++) cmax = std::max(cmax, std::fabs(box[a]));
  const unsigned nb = (unsigned)((n + 255) / 256);
  k_cell_ids<<<nb, 256, 0, s>>>(pts, n, g, cell, idx);
  int bits = 1;
  while ((1ll << bits) < ncell) bits++;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, cell, cell_s, idx, order, (int)n, 0, bits, s);
  FGA_CUDA_TRY(cub_tmp.reserve(tb));
  FGA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp.p, tb, cell, cell_s, idx, order, (int)n, 0,
                                               bits, s));
  // cell offsets: coff[c] = points in cells < c (empty cells included), so a
  // run of consecutive cells is one range of the sorted points
  FGA_CUDA_TRY(cudaMemsetAsync(cstart, 0, sizeof(int) * (ncell + 1), s));
  FGA_CUDA_TRY(cudaMemsetAsync(cend, 0, sizeof(int) * (ncell + 1), s));
  k_cell_bounds<<<nb, 256, 0, s>>>(cell_s, n, cstart, cend);
  k_cell_count<<<(unsigned)((ncell + 256) / 256), 256, 0, s>>>(cstart, cend, ncell);
  int* ccount = cstart;  // ncell + 1 counts, scanned into coff (reuses cend)
  int* coff = cend;
  {
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, ccount, coff, (int)(ncell + 1), s);
    FGA_CUDA_TRY(cub_tmp.reserve(std::max(sb, cub_tmp.bytes)));
    sb = cub_tmp.bytes;
    FGA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(cub_tmp.p, sb, ccount, coff, (int)(ncell + 1), s));
  }
  k_gather_cells<<<nb, 256, 0, s>>>(pts, n, order, ps, ps32);
  const unsigned kb = (unsigned)((n + kKT - 1) / kKT);
  if (out_idx) {
    if (k <= 16)
      k_knn_sorted<16, true><<<kb, kKT, 0, s>>>(ps, ps32, n, order, cell_s, g, cmax, coff, k, out_idx,
                                                out_d2, out_mass, dim);
    else
      k_knn_sorted<32, true><<<kb, kKT, 0, s>>>(ps, ps32, n, order, cell_s, g, cmax, coff, k, out_idx,
                                                out_d2, out_mass, dim);
  } else {
    if (k <= 16)
      k_knn_sorted<16, false><<<kb, kKT, 0, s>>>(ps, ps32, n, order, cell_s, g, cmax, coff, k, nullptr,
                                                 out_d2, out_mass, dim);
    else
      k_knn_sorted<32, false><<<kb, kKT, 0, s>>>(ps, ps32, n, order, cell_s, g, cmax, coff, k, nullptr,
                                                 out_d2, out_mass, dim);
  }
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

}  // namespace fga
