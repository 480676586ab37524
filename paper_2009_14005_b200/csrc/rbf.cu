// rbf.cu -- landmark RBF mass field (masses.py:55-82) and the SPM product
// (masses.py:119-125), the "landmarks" branch of registration._mass_fields
// (registration.py:74-83).
//
// Collocation: K_ij = exp(-|c_i - c_j|^2 / sigma^2) over the m anchor points,
// rejected as SingularCollocation when cond_2(K) is not finite or > 1e12
// (:72-75); lambda = K^-1 1 (:78); value(p) = sum_j exp(-|p - c_j|^2/sigma^2)
// lambda_j, floored at 1e-6 (:80-82).  K is symmetric positive semi-definite,
// so one thread diagonalises it with cyclic Jacobi in shared memory (m is a
// handful of landmarks; capped at 64): cond_2 = max|ev| / min|ev| and
// lambda = V diag(1/ev) V^T 1.  The O(N m) evaluation is one thread per point.
#include "../../include/fga.h"
#include "fga_device.cuh"

namespace fga {
namespace {

constexpr int kRbfMax = 64;

__global__ void k_gather_anchors(const double* __restrict__ pts, const long long* __restrict__ idx,
                                 int m, double* __restrict__ centers) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  for (int k = 0; k < 3; k++) centers[j * 3 + k] = pts[idx[j] * 3 + k];
}

// _gauss_kernel (masses.py:50-51): exp(-(dist * dist) / (sigma * sigma))
__device__ __forceinline__ double gauss(double d2, double s2) { return exp(-d2 / s2); }

// distance as numpy's norm of the difference, squared again (masses.py:67-68, :50-51)
__device__ __forceinline__ double dist_sq(const double* a, const double* b) {
  double s = 0.0;
  for (int k = 0; k < 3; k++) {
    const double e = a[k] - b[k];
    s += e * e;
  }
  const double d = sqrt(s);
  return d * d;
}

__global__ void k_rbf_solve(const double* __restrict__ centers, int m, double sigma,
                            double* __restrict__ lam, int* __restrict__ status) {
  extern __shared__ double sh[];
  if (threadIdx.x != 0) return;
  double* K = sh;               // m*m, becomes the eigenvalues on the diagonal
  double* V = sh + m * m;       // m*m eigenvectors
  const double s2 = sigma * sigma;
  for (int i = 0; i < m; i++)
    for (int j = 0; j < m; j++) {
      K[i * m + j] = gauss(dist_sq(centers + 3 * i, centers + 3 * j), s2);
      V[i * m + j] = i == j ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 60; sweep++) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < m; i++) {
      diag += K[i * m + i] * K[i * m + i];
      for (int j = i + 1; j < m; j++) off += K[i * m + j] * K[i * m + j];
    }
    if (off <= 1e-32 * diag) break;
    for (int p = 0; p < m; p++)
      for (int q = p + 1; q < m; q++) {
        const double apq = K[p * m + q];
        if (apq == 0.0) continue;
        const double theta = (K[q * m + q] - K[p * m + p]) / (2.0 * apq);
        const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < m; k++) {  // rotate rows/cols p, q
          const double kp = K[k * m + p], kq = K[k * m + q];
          K[k * m + p] = c * kp - s * kq;
          K[k * m + q] = s * kp + c * kq;
        }
        for (int k = 0; k < m; k++) {
          const double pk = K[p * m + k], qk = K[q * m + k];
          K[p * m + k] = c * pk - s * qk;
          K[q * m + k] = s * pk + c * qk;
        }
        for (int k = 0; k < m; k++) {
          const double vp = V[k * m + p], vq = V[k * m + q];
          V[k * m + p] = c * vp - s * vq;
          V[k * m + q] = s * vp + c * vq;
        }
      }
  }
  double emax = 0.0, emin = INFINITY;
  for (int i = 0; i < m; i++) {
    const double e = fabs(K[i * m + i]);
    emax = fmax(emax, e);
    emin = fmin(emin, e);
  }
  const double cond = emax / emin;
  if (!isfinite(cond) || cond > 1e12) {
    *status = FGA_ERR_SINGULAR;
    return;
  }
  for (int i = 0; i < m; i++) {  // lambda = V diag(1/ev) V^T 1
    double acc = 0.0;
    for (int j = 0; j < m; j++) {
      double vt1 = 0.0;
      for (int k = 0; k < m; k++) vt1 += V[k * m + j];
      acc += V[i * m + j] * vt1 / K[j * m + j];
    }
    lam[i] = acc;
  }
  *status = 0;
}

// mode 0: out = rbf values (floored); mode 1: out *= rbf (SPM product)
__global__ void k_rbf_eval(const double* __restrict__ pts, int64_t n,
                           const double* __restrict__ centers, const double* __restrict__ lam,
                           int m, double sigma, const int* __restrict__ status, int mode,
                           double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || *status) return;
  const double s2 = sigma * sigma;
  double v = 0.0;
  for (int j = 0; j < m; j++) v += gauss(dist_sq(pts + 3 * i, centers + 3 * j), s2) * lam[j];
  v = fmax(v, 1e-6);
  out[i] = mode ? out[i] * v : v;
}

}  // namespace

// Multiplies (mode 1) or overwrites (mode 0) out with the RBF field of `pts`
// anchored at pts[anchor_idx].  Synchronises once to report singularity.
int rbf_apply_dev(const double* pts, int64_t n, const long long* anchor_idx_dev, int m,
                  double sigma, int mode, double* out, DevBuf& scratch, cudaStream_t s) {
  if (sigma <= 0.0) {
    set_error("invalid parameter sigma=" + std::to_string(sigma));
    return FGA_ERR_INVALID;
  }
  if (m <= 0) {
    if (mode == 0) {
      std::vector<double> ones(n, 1.0);  // no anchors: uniform 1.0 (masses.py:63-64)
      FGA_CUDA_TRY(cudaMemcpyAsync(out, ones.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
      FGA_CUDA_TRY(cudaStreamSynchronize(s));
    }
    return FGA_OK;
  }
  if (m > kRbfMax) {
    set_error("rbf: at most 64 landmarks on the device path");
    return FGA_ERR_UNSUPPORTED;
  }
  FGA_CUDA_TRY(scratch.reserve(sizeof(double) * (4 * m + 8)));
  double* centers = scratch.as<double>();
  double* lam = centers + 3 * m;
  int* status = reinterpret_cast<int*>(lam + m);
  k_gather_anchors<<<1, 64, 0, s>>>(pts, anchor_idx_dev, m, centers);
  k_rbf_solve<<<1, 32, sizeof(double) * 2 * m * m, s>>>(centers, m, sigma, lam, status);
  k_rbf_eval<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pts, n, centers, lam, m, sigma, status,
                                                          mode, out);
  FGA_CUDA_TRY(cudaGetLastError());
  int st = 0;
  FGA_CUDA_TRY(cudaMemcpyAsync(&st, status, sizeof(int), cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  if (st) {
    set_error("kernel matrix condition > 1e12");
    return FGA_ERR_SINGULAR;
  }
  return FGA_OK;
}

}  // namespace fga
