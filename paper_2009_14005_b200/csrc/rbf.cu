// rbf.cu -- landmark RBF mass field (masses.py:55-82) and the SPM product
// (masses.py:119-125), the "landmarks" branch of registration._mass_fields
// (registration.py:74-83).
//
// Collocation: K_ij = exp(-|c_i - c_j|^2 / sigma^2) over the m anchor points,
// rejected as SingularCollocation when cond_2(K) is not finite or > 1e12
// (:72-75); lambda = K^-1 1 (:78); value(p) = sum_j exp(-|p - c_j|^2/sigma^2)
// lambda_j, floored at 1e-6 (:80-82).  K is symmetric positive semi-definite,
// so it is diagonalised with Jacobi rotations: cond_2 = max|ev| / min|ev| and
// lambda = V diag(1/ev) V^T 1.  Up to 64 landmarks (the reference uses 3-4)
// one thread runs cyclic Jacobi in shared memory; above that one 1024-thread
// CTA runs parallel (round-robin) Jacobi on K and V in global memory, all
// M/2 disjoint rotations of a round applied at once (K <- J^T K J), up to
// kRbfMaxLarge landmarks.  The O(N m) evaluation is one thread per point.
#include "../../include/fga.h"
#include "fga_device.cuh"

namespace fga {
namespace {

constexpr int kRbfMax = 64;          // shared-memory single-thread solve
constexpr int kRbfMaxLarge = 2048;   // global-memory parallel solve
constexpr int kRbfThreads = 1024;

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

// Parallel Jacobi for m > kRbfMax.  M = m rounded up to even; an odd m gets
// a dummy index M-1 with K = 1 on its diagonal and 0 off it (never rotated,
// excluded from cond and lambda).  W: 2 M^2 + M doubles (K, V, g).
__global__ void __launch_bounds__(kRbfThreads) k_rbf_solve_large(const double* __restrict__ centers,
                                                                int m, double sigma, double* W,
                                                                double* __restrict__ lam,
                                                                int* __restrict__ status) {
  const int M = (m + 1) & ~1;
  double* K = W;
  double* V = W + (size_t)M * M;
  __shared__ double cs[kRbfMaxLarge / 2], sn[kRbfMaxLarge / 2];
  __shared__ int pp[kRbfMaxLarge / 2], qq[kRbfMaxLarge / 2];
  __shared__ double red[2 * 32];
  const double s2 = sigma * sigma;
  const int tid = threadIdx.x;
  for (int e = tid; e < M * M; e += kRbfThreads) {
    const int i = e / M, j = e % M;
    double kv;
    if (i < m && j < m) kv = gauss(dist_sq(centers + 3 * i, centers + 3 * j), s2);
    else kv = i == j ? 1.0 : 0.0;
    K[e] = kv;
    V[e] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  const int half = M / 2;
  for (int sweep = 0; sweep < 60; sweep++) {
    double off = 0.0, diag = 0.0;  // convergence: off-diagonal vs diagonal mass
    for (int e = tid; e < M * M; e += kRbfThreads) {
      const int i = e / M, j = e % M;
      const double v = K[e] * K[e];
      if (i == j) diag += v;
      else if (j > i) off += v;
    }
    for (int o = 16; o > 0; o >>= 1) {
      off += __shfl_xor_sync(0xffffffffu, off, o);
      diag += __shfl_xor_sync(0xffffffffu, diag, o);
    }
    if ((tid & 31) == 0) {
      red[tid >> 5] = off;
      red[32 + (tid >> 5)] = diag;
    }
    __syncthreads();
    double offt = 0.0, diagt = 0.0;
    for (int w = 0; w < kRbfThreads / 32; w++) {
      offt += red[w];
      diagt += red[32 + w];
    }
    __syncthreads();
    if (offt <= 1e-32 * diagt) break;
    for (int r = 0; r < M - 1; r++) {
      for (int k = tid; k < half; k += kRbfThreads) {  // round-robin pairs of round r
        int p, q;
        if (k == 0) {
          p = r;
          q = M - 1;
        } else {
          p = (r + k) % (M - 1);
          q = (r - k + (M - 1)) % (M - 1);
        }
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        const double apq = K[(size_t)p * M + q];
        double c = 1.0, sv = 0.0;
        if (apq != 0.0) {
          const double th = (K[(size_t)q * M + q] - K[(size_t)p * M + p]) / (2.0 * apq);
          const double t = copysign(1.0, th) / (fabs(th) + sqrt(th * th + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          sv = t * c;
        }
        pp[k] = p;
        qq[k] = q;
        cs[k] = c;
        sn[k] = sv;
      }
      __syncthreads();
      for (int e = tid; e < M * half; e += kRbfThreads) {  // K <- K J, V <- V J (columns)
        const int row = e / half, k = e % half;
        const int p = pp[k], q = qq[k];
        const double c = cs[k], sv = sn[k];
        const double kp = K[(size_t)row * M + p], kq = K[(size_t)row * M + q];
        K[(size_t)row * M + p] = c * kp - sv * kq;
        K[(size_t)row * M + q] = sv * kp + c * kq;
        const double vp = V[(size_t)row * M + p], vq = V[(size_t)row * M + q];
        V[(size_t)row * M + p] = c * vp - sv * vq;
        V[(size_t)row * M + q] = sv * vp + c * vq;
      }
      __syncthreads();
      for (int e = tid; e < M * half; e += kRbfThreads) {  // K <- J^T K (rows)
        const int col = e / half, k = e % half;
        const int p = pp[k], q = qq[k];
        const double c = cs[k], sv = sn[k];
        const double pk = K[(size_t)p * M + col], qk = K[(size_t)q * M + col];
        K[(size_t)p * M + col] = c * pk - sv * qk;
        K[(size_t)q * M + col] = sv * pk + c * qk;
      }
      __syncthreads();
    }
  }
  // cond and lambda over the m real indices (the dummy's eigenpair is exact:
  // its row / column were never rotated)
  __shared__ double s_emax, s_emin;
  if (tid == 0) {
    double emax = 0.0, emin = INFINITY;
    for (int i = 0; i < m; i++) {
      const double e = fabs(K[(size_t)i * M + i]);
      emax = fmax(emax, e);
      emin = fmin(emin, e);
    }
    s_emax = emax;
    s_emin = emin;
    *status = (!isfinite(emax / emin) || emax / emin > 1e12) ? FGA_ERR_SINGULAR : 0;
  }
  __syncthreads();
  if (!(isfinite(s_emax / s_emin) && s_emax / s_emin <= 1e12)) return;
  // lambda = V diag(1/ev) V^T 1: g_j = (sum_k V_kj) / ev_j, then lambda_i = sum_j V_ij g_j
  double* g = W + 2 * (size_t)M * M;
  for (int j = tid; j < m; j += kRbfThreads) {
    double a = 0.0;
    for (int k = 0; k < m; k++) a += V[(size_t)k * M + j];
    g[j] = a / K[(size_t)j * M + j];
  }
  __syncthreads();
  for (int i = tid; i < m; i += kRbfThreads) {
    double acc = 0.0;
    for (int j = 0; j < m; j++) acc += V[(size_t)i * M + j] * g[j];
    lam[i] = acc;
  }
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
  if (m > kRbfMaxLarge) {
    set_error("rbf: at most 2048 landmarks on the device path");
    return FGA_ERR_UNSUPPORTED;
  }
  const int M = (m + 1) & ~1;
  const size_t work = m > kRbfMax ? 2 * (size_t)M * M + M : 0;
  FGA_CUDA_TRY(scratch.reserve(sizeof(double) * (4 * m + 8 + work)));
  double* centers = scratch.as<double>();
  double* lam = centers + 3 * m;
  int* status = reinterpret_cast<int*>(lam + m);
  double* W = lam + m + 8;
  k_gather_anchors<<<(m + 63) / 64, 64, 0, s>>>(pts, anchor_idx_dev, m, centers);
  if (m <= kRbfMax)
    k_rbf_solve<<<1, 32, sizeof(double) * 2 * m * m, s>>>(centers, m, sigma, lam, status);
  else
    k_rbf_solve_large<<<1, kRbfThreads, 0, s>>>(centers, m, sigma, W, lam, status);
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
