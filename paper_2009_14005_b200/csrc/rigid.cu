// rigid.cu -- K7/K8: deterministic reduction of the Kabsch partials and the
// fp64 rigid update (procrustes.py:12-49, registration.py:133-154).
//
// The cross-covariance is assembled from shifted moments
//     C = sum w u^T - M * mean(w) mean(u)^T,  u = y - s, w = y + d - s
// with s = the current template mean (carried from the previous update), so
// there is no cancellation; C equals the reference's yd_c.T @ yc
// (procrustes.py:23-25) up to rounding.  The 3x3 SVD is a one-sided Jacobi in
// fp64 (no LAPACK on the device); the reflection guard and the rotation are
// the reference's (:27-33): R = U diag(1, 1, sign det(U V^T)) V^T.
#include "fga_device.cuh"

namespace fga {
namespace {

constexpr int kReduceThreads = 1024;

// Sums of the per-warp partial records in a fixed order: kRedBlocks blocks
// each reduce a contiguous range of warps (thread-strided, then a fixed block
// tree), one warp adds the block results in block order.
constexpr int kRedBlocks = 148;
constexpr int kRedThreads = 256;
constexpr int64_t kFuseWarps = 2048;

// Fixed-order block sum of the kPartialStride accumulators of every thread:
// a shuffle tree per warp, then thread k adds the warps' results in warp
// order (two barriers in all, where one block_reduce per slot took 2 x 18).
// out: shared, kPartialStride doubles, valid after the call.
template <int kThreads>
__device__ __forceinline__ void block_sum_slots(double (&acc)[kPartialStride], double* out) {
  __shared__ double ws[kThreads / 32][kPartialStride];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kPartialStride; k++) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) ws[w][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < kPartialStride) {
    double v = 0.0;
    for (int q = 0; q < kThreads / 32; q++) v += ws[q][threadIdx.x];
    out[threadIdx.x] = v;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kRedThreads) k_reduce_stage(const double* __restrict__ partials,
                                                             int64_t nwarps,
                                                             const double* __restrict__ gpe_part,
                                                             int64_t ngwarps,
                                                             double* __restrict__ stage) {
  const int64_t b = blockIdx.x, nb = gridDim.x;
  const int64_t w0 = nwarps * b / nb, w1 = nwarps * (b + 1) / nb;
  const int64_t g0 = ngwarps * b / nb, g1 = ngwarps * (b + 1) / nb;
  double acc[kPartialStride];
#pragma unroll
  for (int k = 0; k < kPartialStride; k++) acc[k] = 0.0;
  for (int64_t w = w0 + threadIdx.x; w < w1; w += kRedThreads) {
#pragma unroll
    for (int k = 0; k < 17; k++) acc[k] += partials[w * kPartialStride + k];
  }
  for (int64_t w = g0 + threadIdx.x; w < g1; w += kRedThreads) acc[kGpe] += gpe_part[w];
  __shared__ double out[kPartialStride];
  block_sum_slots<kRedThreads>(acc, out);
  if (threadIdx.x < kPartialStride) stage[b * kPartialStride + threadIdx.x] = out[threadIdx.x];
}

__global__ void k_reduce_final(const double* __restrict__ stage, int nb, double direct_pairs,
                               double* __restrict__ sums) {
  const int k = threadIdx.x;
  if (k >= kPartialStride) return;
  double v = 0.0;
  for (int b = 0; b < nb; b++) v += stage[b * kPartialStride + k];
  if (direct_pairs >= 0.0 && (k == kAccepted || k == kVisits)) v = direct_pairs;
  sums[k] = v;
}

__device__ void update_body(const double* sums, IterState* st, const SimParams& sp,
                            double* rec_delta, double* rec_traj, double* rec_gpe,
                            long long* rec_inter, long long* rec_visits, int has_gpe) {
  if (st->done) return;
  const double M = (double)sp.m_total;
  double mu_u[3], mu_w[3], C[9];
  for (int k = 0; k < 3; k++) {
    mu_u[k] = sums[kSumU + k] / M;
    mu_w[k] = sums[kSumW + k] / M;
  }
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) C[3 * i + j] = sums[kSumWU + 3 * i + j] - M * mu_w[i] * mu_u[j];
  double R[9];
  if (sp.dim == 2) kabsch_rotation_2d(C, R, nullptr);
  else kabsch_rotation(C, R, nullptr);
  double mu_y[3], mu_d[3], t[3];
  for (int k = 0; k < 3; k++) {
    mu_y[k] = mu_u[k] + st->shift[k];
    mu_d[k] = mu_w[k] + st->shift[k];
  }
  for (int k = 0; k < 3; k++)
    t[k] = mu_d[k] - (R[3 * k] * mu_y[0] + R[3 * k + 1] * mu_y[1] + R[3 * k + 2] * mu_y[2]);  // :42
  const long long it = st->iter;
  if (has_gpe && it > 0 && rec_gpe) rec_gpe[it - 1] = -sp.G * sums[kGpe];
  // R_acc <- R R_acc ; t_acc <- t + R t_acc  (registration.py:137-138)
  double Ra[9], ta[3], delta = 0.0;
  for (int i = 0; i < 3; i++) {
    for (int j = 0; j < 3; j++)
      Ra[3 * i + j] = R[3 * i] * st->Racc[j] + R[3 * i + 1] * st->Racc[3 + j] + R[3 * i + 2] * st->Racc[6 + j];
    ta[i] = t[i] + (R[3 * i] * st->tacc[0] + R[3 * i + 1] * st->tacc[1] + R[3 * i + 2] * st->tacc[2]);
  }
  // delta = ||[R_acc|t_acc] - prev||_F^2 (:140-142)
  for (int i = 0; i < 3; i++) {
    for (int j = 0; j < 3; j++) {
      const double e = Ra[3 * i + j] - st->Racc[3 * i + j];
      delta += e * e;
    }
    const double e = ta[i] - st->tacc[i];
    delta += e * e;
  }
  for (int k = 0; k < 9; k++) {
    st->Rp[k] = R[k];
    st->Racc[k] = Ra[k];
  }
  for (int k = 0; k < 3; k++) {
    st->tp[k] = t[k];
    st->tacc[k] = ta[k];
    st->shift[k] = mu_d[k];  // mean of R y + t
  }
  if (rec_delta) rec_delta[it] = delta;
  if (rec_traj)
    for (int i = 0; i < 3; i++) {
      for (int j = 0; j < 3; j++) rec_traj[it * 12 + 4 * i + j] = Ra[3 * i + j];
      rec_traj[it * 12 + 4 * i + 3] = ta[i];
    }
  if (rec_inter) rec_inter[it] = (long long)sums[kAccepted];
  if (rec_visits) rec_visits[it] = (long long)sums[kVisits];
  st->iter = it + 1;
  if (delta < sp.conv_tol) {  // :152-154
    st->converged = 1;
    st->done = 1;
  } else if (it + 1 >= sp.max_iters) {
    st->done = 1;
  }
}

__global__ void k_update(const double* __restrict__ sums, IterState* st, SimParams sp,
                         double* rec_delta, double* rec_traj, double* rec_gpe,
                         long long* rec_inter, long long* rec_visits, int has_gpe) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  update_body(sums, st, sp, rec_delta, rec_traj, rec_gpe, rec_inter, rec_visits, has_gpe);
}

// Small passes (<= kFuseWarps warp partials): the fixed-order reduction in
// ONE block and the rigid update in the same kernel (one launch per
// iteration instead of three; configs[0]-sized registrations are bound by
// these per-iteration latencies).
constexpr int kFuseThreads = 256;
__global__ void __launch_bounds__(kFuseThreads) k_reduce_update(
    const double* __restrict__ partials, int64_t nwarps, const double* __restrict__ gpe_part,
    int64_t ngwarps, double direct_pairs, double* __restrict__ sums, IterState* st, SimParams sp,
    double* rec_delta, double* rec_traj, double* rec_gpe, long long* rec_inter,
    long long* rec_visits, int has_gpe) {
  double acc[kPartialStride];
#pragma unroll
  for (int k = 0; k < kPartialStride; k++) acc[k] = 0.0;
  for (int64_t w = threadIdx.x; w < nwarps; w += kFuseThreads) {
#pragma unroll
    for (int k = 0; k < 17; k++) acc[k] += partials[w * kPartialStride + k];
  }
  for (int64_t w = threadIdx.x; w < ngwarps; w += kFuseThreads) acc[kGpe] += gpe_part[w];
  __shared__ double out[kPartialStride];
  block_sum_slots<kFuseThreads>(acc, out);
  if (threadIdx.x < kPartialStride) {
    const int k = threadIdx.x;
    double v = out[k];
    if (direct_pairs >= 0.0 && (k == kAccepted || k == kVisits)) v = direct_pairs;
    out[k] = v;
    sums[k] = v;
  }
  __syncthreads();
  if (st && threadIdx.x == 0)  // (st == nullptr: the reduction alone, launch_reduce)
    update_body(out, st, sp, rec_delta, rec_traj, rec_gpe, rec_inter, rec_visits, has_gpe);
}

__global__ void k_apply_pending(TemplateView tv, const IterState* __restrict__ st) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tv.m) return;
  const double y[3] = {tv.px[i], tv.py[i], tv.pz[i]};
  double ny[3];
  for (int r = 0; r < 3; r++)
    ny[r] = st->Rp[3 * r] * y[0] + st->Rp[3 * r + 1] * y[1] + st->Rp[3 * r + 2] * y[2] + st->tp[r];
  tv.px[i] = ny[0];
  tv.py[i] = ny[1];
  tv.pz[i] = ny[2];
}

// Session state in input order (checkpoint / teacher forcing): positions and
// velocities with the pending step transform applied (the state entering the
// next iteration), without changing the session.
__global__ void k_state_get(TemplateView tv, const IterState* __restrict__ st,
                            const int* __restrict__ order, int64_t begin, double* __restrict__ pos,
                            double* __restrict__ vel) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tv.m) return;
  double y[3] = {tv.px[i], tv.py[i], tv.pz[i]}, v[3] = {tv.vx[i], tv.vy[i], tv.vz[i]};
  apply_pending(st, y, v);
  const int64_t src = order[begin + i];
  for (int k = 0; k < 3; k++) {
    pos[src * 3 + k] = y[k];
    vel[src * 3 + k] = v[k];
  }
}
__global__ void k_state_set(TemplateView tv, const int* __restrict__ order, int64_t begin,
                            const double* __restrict__ pos, const double* __restrict__ vel) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= tv.m) return;
  const int64_t src = order[begin + i];
  tv.px[i] = pos[src * 3];
  tv.py[i] = pos[src * 3 + 1];
  tv.pz[i] = pos[src * 3 + 2];
  tv.vx[i] = vel[src * 3];
  tv.vy[i] = vel[src * 3 + 1];
  tv.vz[i] = vel[src * 3 + 2];
}

__global__ void k_state_init(IterState* st, const double* __restrict__ mean3) {
  if (threadIdx.x != 0) return;
  for (int k = 0; k < 9; k++) {
    st->Rp[k] = (k % 4 == 0) ? 1.0 : 0.0;
    st->Racc[k] = st->Rp[k];
  }
  for (int k = 0; k < 3; k++) {
    st->tp[k] = 0.0;
    st->tacc[k] = 0.0;
    st->shift[k] = mean3[k];
  }
  st->iter = 0;
  st->done = 0;
  st->converged = 0;
  st->gpe_pending = 0;
  st->pad = 0;
}

// solve_rigid operator: two deterministic passes (means, then centred
// cross-covariance) in one block, then the Kabsch rotation.
__global__ void __launch_bounds__(kReduceThreads) k_solve_rigid(const double* __restrict__ y,
                                                                const double* __restrict__ yd,
                                                                int64_t m, int dim,
                                                                double* out13) {
  __shared__ double sm[kReduceThreads / 32][9];
  __shared__ double mean[6];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  double a[9];
  for (int k = 0; k < 6; k++) a[k] = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += kReduceThreads)
    for (int k = 0; k < 3; k++) {
      a[k] += y[i * 3 + k];
      a[3 + k] += yd[i * 3 + k];
    }
  for (int k = 0; k < 6; k++) {
    const double v = warp_sum(a[k]);
    if (lane == 0) sm[wl][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double v = 0.0;
    for (int j = 0; j < kReduceThreads / 32; j++) v += sm[j][threadIdx.x];
    mean[threadIdx.x] = v / (double)m;
  }
  __syncthreads();
  for (int k = 0; k < 9; k++) a[k] = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += kReduceThreads) {
    double yc[3], dc[3];
    for (int k = 0; k < 3; k++) {
      yc[k] = y[i * 3 + k] - mean[k];
      dc[k] = yd[i * 3 + k] - mean[3 + k];
    }
    for (int r = 0; r < 3; r++)
      for (int c = 0; c < 3; c++) a[3 * r + c] = fma(dc[r], yc[c], a[3 * r + c]);
  }
  __syncthreads();
  for (int k = 0; k < 9; k++) {
    const double v = warp_sum(a[k]);
    if (lane == 0) sm[wl][k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double C[9], R[9];
    for (int k = 0; k < 9; k++) {
      double v = 0.0;
      for (int j = 0; j < kReduceThreads / 32; j++) v += sm[j][k];
      C[k] = v;
    }
    int degenerate = 0;
    if (dim == 2) kabsch_rotation_2d(C, R, &degenerate);
    else kabsch_rotation(C, R, &degenerate);
    for (int k = 0; k < 9; k++) out13[k] = R[k];
    for (int k = 0; k < 3; k++)  // t = mean(y_d) - R mean(y) (:42)
      out13[9 + k] = mean[3 + k] - (R[3 * k] * mean[0] + R[3 * k + 1] * mean[1] + R[3 * k + 2] * mean[2]);
    out13[12] = degenerate;
  }
}

}  // namespace

size_t reduce_stage_doubles() { return (size_t)kRedBlocks * kPartialStride; }

void launch_reduce(const double* partials, int64_t nwarps, const double* gpe_partials,
                   int64_t ngwarps, double direct_pairs, double* sums, double* stage,
                   cudaStream_t s) {
  if (nwarps <= kFuseWarps && ngwarps <= kFuseWarps) {  // the fused kernel's order, no update
    k_reduce_update<<<1, kFuseThreads, 0, s>>>(partials, nwarps, gpe_partials, ngwarps,
                                               direct_pairs, sums, nullptr, SimParams{}, nullptr,
                                               nullptr, nullptr, nullptr, nullptr, 0);
    return;
  }
  k_reduce_stage<<<kRedBlocks, kRedThreads, 0, s>>>(partials, nwarps, gpe_partials, ngwarps, stage);
  k_reduce_final<<<1, 32, 0, s>>>(stage, kRedBlocks, direct_pairs, sums);
}

bool reduce_update_fusable(int64_t nwarps, int64_t ngwarps) {
  return nwarps <= kFuseWarps && ngwarps <= kFuseWarps;
}

void launch_reduce_update(const double* partials, int64_t nwarps, const double* gpe_partials,
                          int64_t ngwarps, double direct_pairs, double* sums, IterState* st,
                          const SimParams& sp, double* rec_delta, double* rec_traj,
                          double* rec_gpe, long long* rec_inter, long long* rec_visits,
                          int has_gpe, cudaStream_t s) {
  k_reduce_update<<<1, kFuseThreads, 0, s>>>(partials, nwarps, gpe_partials, ngwarps,
                                             direct_pairs, sums, st, sp, rec_delta, rec_traj,
                                             rec_gpe, rec_inter, rec_visits, has_gpe);
}

void launch_update(const double* sums, IterState* st, const SimParams& sp, double* rec_delta,
                   double* rec_traj, double* rec_gpe, long long* rec_inter, long long* rec_visits,
                   int has_gpe, cudaStream_t s) {
  k_update<<<1, 32, 0, s>>>(sums, st, sp, rec_delta, rec_traj, rec_gpe, rec_inter, rec_visits,
                            has_gpe);
}

void launch_apply_pending(const TemplateView& tv, const IterState* st, cudaStream_t s) {
  if (tv.m <= 0) return;
  k_apply_pending<<<(unsigned)((tv.m + 255) / 256), 256, 0, s>>>(tv, st);
}

void launch_state_get(const TemplateView& tv, const IterState* st, const int* order, int64_t begin,
                      double* pos, double* vel, cudaStream_t s) {
  if (tv.m <= 0) return;
  k_state_get<<<(unsigned)((tv.m + 255) / 256), 256, 0, s>>>(tv, st, order, begin, pos, vel);
}
void launch_state_set(const TemplateView& tv, const int* order, int64_t begin, const double* pos,
                      const double* vel, cudaStream_t s) {
  if (tv.m <= 0) return;
  k_state_set<<<(unsigned)((tv.m + 255) / 256), 256, 0, s>>>(tv, order, begin, pos, vel);
}

void launch_state_init(IterState* st, const double* mean3, cudaStream_t s) {
  k_state_init<<<1, 32, 0, s>>>(st, mean3);
}

void launch_solve_rigid(const double* y, const double* yd, int64_t m, int dim, double* out13,
                        cudaStream_t s) {
  k_solve_rigid<<<1, kReduceThreads, 0, s>>>(y, yd, m, dim, out13);
}

}  // namespace fga
