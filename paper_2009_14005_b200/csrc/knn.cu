// knn.cu -- grid-bucketed exact k-nearest-neighbour search and the kNN
// smooth-particle mass field (BASELINE configs[3], north_star item 1).
//
// The reference's default SPM field is the NIV lattice (masses.py:85-116);
// kNN masses are an OPT-IN extension that plugs into the same place as the
// reference's external-weights hook (registration.py:72-83): mass_i =
// (4/3) pi r_k(i)^3 / k, the volume per point of the ball holding the k
// nearest other points -- denser regions get smaller masses, like NIV.
//
// Algorithm: uniform grid with cell edge h ~ (V k / n)^(1/3) over the cloud's
// bbox; points counting-sorted by cell (cub radix sort on the cell id); one
// thread per query (queries visited in cell order for warp coherence) scans
// Chebyshev shells s = 0, 1, 2, ... of cells around its own cell keeping the k
// best (d^2, index) pairs in registers (insertion into a sorted list), and
// stops once it holds k candidates and the k-th d^2 <= (s h + gap)^2 where gap
// is the query's distance to its cell boundary -- every point closer than that
// lies in the scanned cube, so the set is exact.  Distances in fp64; ties are
// broken by point index.
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

template <int K>
__global__ void __launch_bounds__(kKT) k_knn(const double* __restrict__ p, int64_t n,
                                             const int* __restrict__ order,  // points by cell
                                             const unsigned* __restrict__ cell_sorted, Grid g,
                                             const int* __restrict__ cstart,
                                             const int* __restrict__ cend, int k,
                                             long long* __restrict__ out_idx,
                                             double* __restrict__ out_d2,
                                             double* __restrict__ out_mass, int dim) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int i = order[t];
  const double q[3] = {p[(int64_t)i * 3], p[(int64_t)i * 3 + 1], p[(int64_t)i * 3 + 2]};
  const unsigned cid = cell_sorted[t];
  const int c2 = (int)(cid % g.dim[2]);
  const int c1 = (int)((cid / g.dim[2]) % g.dim[1]);
  const int c0 = (int)(cid / ((unsigned)g.dim[2] * g.dim[1]));
  const int cc[3] = {c0, c1, c2};
  // distance from q to the boundary of its own cell (>= 0)
  double gap = INFINITY;
  for (int a = 0; a < 3; a++) {
    const double lo = g.lo[a] + cc[a] * g.h;
    gap = fmin(gap, fmin(q[a] - lo, lo + g.h - q[a]));
  }
  gap = fmax(gap, 0.0);
  double bd[K];
  int bi[K];
#pragma unroll
  for (int j = 0; j < K; j++) {
    bd[j] = INFINITY;
    bi[j] = INT_MAX;
  }
  const int smax = max(g.dim[0], max(g.dim[1], g.dim[2]));
  for (int s = 0; s <= smax; s++) {
    for (int dx = -s; dx <= s; dx++) {
      const int x = cc[0] + dx;
      if (x < 0 || x >= g.dim[0]) continue;
      for (int dy = -s; dy <= s; dy++) {
        const int y = cc[1] + dy;
        if (y < 0 || y >= g.dim[1]) continue;
        const bool face = abs(dx) == s || abs(dy) == s;
        for (int dz = -s; dz <= s; dz += (face ? 1 : 2 * s)) {
          const int z = cc[2] + dz;
          if (z >= 0 && z < g.dim[2]) {
            const unsigned c = ((unsigned)x * g.dim[1] + y) * g.dim[2] + z;
            const int b = cstart[c], e = cend[c];
            for (int u = b; u < e; u++) {
              const int j = order[u];
              if (j == i) continue;
              const double ex = __dsub_rn(p[(int64_t)j * 3], q[0]);
              const double ey = __dsub_rn(p[(int64_t)j * 3 + 1], q[1]);
              const double ez = __dsub_rn(p[(int64_t)j * 3 + 2], q[2]);
              const double d2 =
                  __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
              insert<K>(bd, bi, d2, j);
            }
          }
          if (s == 0) break;
        }
      }
    }
    // every point closer than `cover` lies in the scanned cube (shrunk by a
    // relative 1e-12 against cell-assignment rounding)
    const double cover = (s * g.h + gap) * (1.0 - 1e-12);
    if (bi[k - 1] != INT_MAX && bd[k - 1] <= cover * cover) break;
  }
  if (out_idx)
    for (int j = 0; j < k; j++) out_idx[(int64_t)i * k + j] = bi[j] == INT_MAX ? -1 : bi[j];
  if (out_d2)
    for (int j = 0; j < k; j++) out_d2[(int64_t)i * k + j] = bd[j];
  if (out_mass) {
    const double r = sqrt(bd[k - 1]);
    // volume (area for D = 2) per point of the k-NN ball
    const double v = !isfinite(r) ? 0.0
                     : dim == 2   ? M_PI * r * r / k
                                  : (4.0 / 3.0) * M_PI * r * r * r / k;
    out_mass[i] = fmax(v, 1e-6);
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
  double h = dim == 2 ? std::sqrt(vol * std::max(k, 2) / (double)n)
                      : std::cbrt(vol * std::max(k, 2) / (double)n);
  for (int a = 0; a < 3; a++) h = std::max(h, ext[a] / 512.0);  // <= 512 cells per axis
  g.h = h;
  g.inv_h = 1.0 / h;
  int64_t ncell = 1;
  for (int a = 0; a < 3; a++) {
    g.dim[a] = std::max(1, (int)std::ceil(ext[a] / h));
    ncell *= g.dim[a];
  }
  const size_t need = sizeof(unsigned) * 2 * n + sizeof(int) * 2 * n + sizeof(int) * 2 * ncell + 1024;
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
  q += sizeof(int) * ncell;
  int* cend = (int*)q;
  const unsigned nb = (unsigned)((n + 255) / 256);
  k_cell_ids<<<nb, 256, 0, s>>>(pts, n, g, cell, idx);
  int bits = 1;
  while ((1ll << bits) < ncell) bits++;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, cell, cell_s, idx, order, (int)n, 0, bits, s);
  FGA_CUDA_TRY(cub_tmp.reserve(tb));
  FGA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp.p, tb, cell, cell_s, idx, order, (int)n, 0,
                                               bits, s));
  FGA_CUDA_TRY(cudaMemsetAsync(cstart, 0, sizeof(int) * ncell, s));
  FGA_CUDA_TRY(cudaMemsetAsync(cend, 0, sizeof(int) * ncell, s));
  k_cell_bounds<<<nb, 256, 0, s>>>(cell_s, n, cstart, cend);
  const unsigned kb = (unsigned)((n + kKT - 1) / kKT);
  if (k <= 16)
    k_knn<16><<<kb, kKT, 0, s>>>(pts, n, order, cell_s, g, cstart, cend, k, out_idx, out_d2,
                                 out_mass, dim);
  else
    k_knn<32><<<kb, kKT, 0, s>>>(pts, n, order, cell_s, g, cstart, cend, k, out_idx, out_d2,
                                 out_mass, dim);
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

}  // namespace fga
