// fga_session.cuh -- launch interfaces between capi.cu and the kernel files.
#pragma once
#include "fga_internal.cuh"
#include "fga_tree.cuh"

namespace fga {

// Template swarm state for one shard, SoA fp64 in Morton order.
struct TemplateView {
  double *px, *py, *pz;  // positions (pending transform not yet applied)
  double *vx, *vy, *vz;  // velocities v' of the last step (pre-rotation)
  const double* mq;      // masses
  int64_t m;
};

// Reference points for the direct sum / energy: {x, y, z, m}.
struct RefPoints {
  const float4* p32;
  const double4* p64;
  int64_t n;
};

constexpr int kForceThreads = 256;
constexpr int kDirectQPT = 4;  // queries per thread in the FP32 direct sum (2 FFMA2 packs)

int64_t bh_iterate_warps(int64_t m, int precision);
bool bh_split_possible(int64_t m);
int64_t direct_iterate_warps(int64_t m, int precision);
int64_t gpe_warps(int64_t m, int64_t n, int precision);

constexpr int kTraceLen = 65;  // per-warp split trace: 64 node indices + the step count

// One force pass of the iteration: applies the pending transform, evaluates
// forces, fused Euler-Cromer step, per-warp Kabsch partials.
// split passes of small template shards (forces.cu k_bh_split): the warps'
// recorded traces (65 ints per warp), the two parts' fp64 force sums (2 m x 3)
// and accepted counts (2 m), and whether the trace has been recorded
struct SplitBufs {
  int* trace;
  double* fpart;
  int* apart;
  bool* have_trace;
  // multi-wave passes: blocks launched heaviest first (LPT order from the
  // first pass's trace): order/okeys (4 x blocks ints), CUB scratch
  int* order = nullptr;
  int* okeys = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  bool* have_order = nullptr;
  bool* split = nullptr;  // this session's later passes run split
};
void launch_bh_iterate(const TreeDev& T, const TemplateView& tv, const IterState* st,
                       const SimParams& sp, double* partials, int precision, cudaStream_t s,
                       const SplitBufs* sb = nullptr);
void launch_direct_iterate(const RefPoints& ref, const TemplateView& tv, const IterState* st,
                           const SimParams& sp, double* partials, int precision, cudaStream_t s);
// Energy of the current (already transformed) positions: per-warp partials of
// sum_i m_i * sum_j m_j / (|y_i - x_j| + eps).  Skipped when st->done.
void launch_gpe(const RefPoints& ref, const double* px, const double* py, const double* pz,
                const double* mq, int64_t m, double eps, const IterState* st, double* partials,
                int precision, cudaStream_t s);

// Operator-level (no state): queries SoA fp64 (already in traversal order),
// outputs scattered back through `order` (may be null = identity).
// FP32 calls that fill at most one wave (bh_operator_split_possible) may run
// as split passes: mode 1 records the warps' traces (ceil(m/32) x 65 ints)
// and their max / sum of steps (stats[2]); mode 2 runs split passes from
// them (fpart: 8 m x 3 doubles, vpart / apart: 8 m ints) and records the
// parts' steps (ptrace: 8 x ceil(m/32) x 65 ints; their max / sum -> stats);
// mode 0 plain.
struct OpSplitBufs {
  int mode;
  int* trace;
  unsigned long long* stats;
  double* fpart;
  int *vpart, *apart, *ptrace;
};
int bh_split_parts();
bool bh_operator_split_possible(int64_t m);
int64_t bh_operator_warps(int64_t m);
bool bh_operator_split_wanted(int64_t m, unsigned long long max_steps,
                              unsigned long long sum_steps);
void launch_bh_operator(const TreeDev& T, const double* qx, const double* qy, const double* qz,
                        const double* qm, const int* order, int64_t m, double theta, double G,
                        double eps2, double* fout, long long* visits, long long* accepted,
                        unsigned long long* acc_total, int precision, cudaStream_t s,
                        const OpSplitBufs* ob = nullptr);
void launch_direct_operator(const RefPoints& ref, const double* qx, const double* qy,
                            const double* qz, const double* qm, int64_t m, double G, double eps,
                            double* fout, int precision, cudaStream_t s);

// Rigid side (rigid.cu)
size_t reduce_stage_doubles();
void launch_reduce(const double* partials, int64_t nwarps, const double* gpe_partials,
                   int64_t ngwarps, double direct_pairs, double* sums, double* stage,
                   cudaStream_t s);
bool reduce_update_fusable(int64_t nwarps, int64_t ngwarps);
void launch_reduce_update(const double* partials, int64_t nwarps, const double* gpe_partials,
                          int64_t ngwarps, double direct_pairs, double* sums, IterState* st,
                          const SimParams& sp, double* rec_delta, double* rec_traj,
                          double* rec_gpe, long long* rec_inter, long long* rec_visits,
                          int has_gpe, cudaStream_t s);
void launch_update(const double* sums, IterState* st, const SimParams& sp, double* rec_delta,
                   double* rec_traj, double* rec_gpe, long long* rec_inter, long long* rec_visits,
                   int has_gpe, cudaStream_t s);
void launch_apply_pending(const TemplateView& tv, const IterState* st, cudaStream_t s);
void launch_state_get(const TemplateView& tv, const IterState* st, const int* order, int64_t begin,
                      double* pos, double* vel, cudaStream_t s);
void launch_state_set(const TemplateView& tv, const int* order, int64_t begin, const double* pos,
                      const double* vel, cudaStream_t s);
void launch_state_init(IterState* st, const double* mean3, cudaStream_t s);
void launch_solve_rigid(const double* y, const double* yd, int64_t m, int dim, double* out13,
                        cudaStream_t s);

// Setup (setup.cu)
int normalize_pair_dev(const double* x, int64_t n, const double* y, int64_t m, double a, double b,
                       double* xn, double* yn, double* ctx10_dev, double* scratch,
                       size_t scratch_bytes, double* ctx10_host, cudaStream_t s);
int niv_masses_dev(const double* pts, int64_t n, int dim, int rho, double a, double b, int max_depth,
                   double* out, int* flat_scratch, long long* counts_scratch, double* cells_scratch,
                   cudaStream_t s);
void launch_external_masses(const double* w, int64_t n, double* out, cudaStream_t s);
size_t pairwise_sum_scratch_doubles(int64_t n);
void launch_np_sum(const double* a, int64_t n, double* out, double* scratch, cudaStream_t s);
void launch_rescale(double* sx, int64_t n, double* sy, int64_t m, double dt, double eta,
                    double* scratch, cudaStream_t s);
void launch_pack_ref(const double* xn, const double* mx, int64_t n, float4* p32, double4* p64,
                     cudaStream_t s);
size_t scratch_doubles_for(int64_t n);
void launch_mean3(const double* pts_aos, int64_t n, double* scratch, double* out3, cudaStream_t s);
void launch_bbox(const double* pts_aos, int64_t n, double* scratch, double* out6, cudaStream_t s);
void launch_morton_keys(const double* pts_aos, int64_t n, const double* box6,
                        unsigned long long* keys, int* idx, cudaStream_t s);
void launch_gather_template(const double* pts_aos, const double* mass, const int* order,
                            int64_t begin, int64_t count, TemplateView tv, cudaStream_t s);
void launch_gather_queries(const double* q_aos, const double* qm, const int* order, int64_t m,
                           double* qx, double* qy, double* qz, double* qms, cudaStream_t s);

int knn_dev(const double* pts, int64_t n, int dim, int k, long long* out_idx, double* out_d2,
            double* out_mass, DevBuf& scratch, DevBuf& cub_tmp, cudaStream_t s);

int rbf_apply_dev(const double* pts, int64_t n, const long long* anchor_idx_dev, int m,
                  double sigma, int mode, double* out, DevBuf& scratch, cudaStream_t s);

}  // namespace fga
