// capi.cu -- the C ABI (include/fga.h): context, operator entry points and the
// registration driver (registration.py:91-166) as a device-resident loop.
//
// The whole registration state lives in HBM inside the context.  One
// iteration is three stream-ordered launches -- force pass (traversal or
// direct sum, fused step + Kabsch partials), partial reduction, rigid update
// -- and the host only polls the device convergence flag every
// `poll_every` iterations; kernels enqueued after convergence exit at once
// (they read the same flag), so the result is exactly the reference's
// stop-at-first-delta<tol semantics (registration.py:152-154).
#include <cub/cub.cuh>

#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fga.h"
#include "fga_session.cuh"
#include "fga_batched.cuh"

namespace fga {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }
}  // namespace fga

using namespace fga;

namespace {

struct Session {
  bool active = false;
  fga_params P{};
  fga_options O{};
  SimParams sp{};
  int precision = 0;
  bool direct = false;  // theta == 0: exact O(NM) direct sum instead of the tree
  int64_t n = 0, m = 0, m_begin = 0, m_local = 0;
  int shard_rank = 0, shard_count = 1;
  double ctx10[10] = {0};
  double gpe_initial = NAN, gpe_final = NAN;
  bool have_gpe_initial = false, have_gpe_final = false;
  bool applied = false;
  int64_t passes = 0;      // force passes enqueued
  bool last_pass_gpe = false;
  bool fused_update = false;  // the last session_forces also ran the update
  bool split_traced = false;  // small shards: the warps' split trace is recorded
  bool order_ready = false;   // multi-wave passes: the heaviest-first block order is set
  bool split_mode = false;    // the later passes run as split passes
  DevBuf split_trace, split_f, split_a, order_buf;
  DevBuf x_raw, y_raw, xn, yn, ctx_dev, mx, my, flat, counts, cells, ref32, ref64;
  DevBuf tkeys_in, tkeys, tidx_in, tidx, cub_tmp, tpl;
  DevBuf partials, gpe_part, sums, state, scratch, lm_idx, rbf_scratch, red_stage;
  DevBuf gpe_snap, gpe_part2, gpe_sums2;  // initial energy on the aux stream
  DevBuf ckpt;                            // device-side checkpoint (fga_session_checkpoint)
  bool have_ckpt = false;
  DevBuf rec_delta, rec_traj, rec_gpe, rec_inter, rec_visits;
  // the session's own reference tree: operator-level builds / uploads into
  // the context (fga_tree_*) never disturb a live registration, and a
  // registration never replaces the operator tree
  TreeDev tree;
  float setup_ms = 0.f, loop_ms = 0.f, gpe_ms = 0.f;

  TemplateView view() const {
    double* b = tpl.as<double>();
    const int64_t ml = m_local;
    return TemplateView{b, b + ml, b + 2 * ml, b + 3 * ml, b + 4 * ml, b + 5 * ml, b + 6 * ml, ml};
  }
  double* sums_ext = nullptr;  // caller-owned sums buffer (fga_session_bind_sums)
  double* sums_ptr() const { return sums_ext ? sums_ext : sums.as<double>(); }
  RefPoints ref() const { return RefPoints{ref32.as<float4>(), ref64.as<double4>(), n}; }
  IterState* st() const { return state.as<IterState>(); }
};

}  // namespace

struct fga_ctx {
  int device = 0;
  DevBuf batch_in[6], batch_scratch, batch_out, batch_deltas, batch_counter, batch_wide;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  TreeDev tree;
  DevBuf tree_pts, tree_masses;
  DevBuf op[8];
  DevBuf op_total;               // device counter: accepted nodes of the last operator call
  // one-wave FP32 operator calls (an N-way rank's slice): the split trace
  // the last call over the same tree, query count and theta recorded
  DevBuf op_trace, op_fpart, op_cnt;
  struct OpSplitKey {
    uint64_t generation = 0;
    int64_t m = -1;
    double theta = 0.0, eps2 = 0.0;
    unsigned long long max_steps = 0;  // the heaviest warp's steps when traced
    unsigned long long part_max = 0;   // the heaviest part's steps, first split call after
    bool traced = false, split = false;
  } op_split;
  // pinned staging ring of fga_register_batch_list (kStageSlots chunks)
  char* stage[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t stage_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t last_interactions = -1;
  Session S;
  int* pinned = nullptr;  // poll buffer: done, pad, iter(lo,hi)
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  // second stream for the initial energy, which runs alongside the iterations
  cudaStream_t aux = nullptr;
  cudaEvent_t aev[3] = {nullptr, nullptr, nullptr};
  // fga_bh_forces_kernel upload cache: the reference calls the kernel once per
  // force evaluation with the same (immutable) BHTree arrays, so the tree is
  // re-uploaded only when the arrays' addresses, size or sampled contents
  // change, or another build/upload replaced the context's tree since.
  struct ShimKey {
    const void* p[4] = {nullptr, nullptr, nullptr, nullptr};
    int64_t n_nodes = -1;
    int n_child = 0, dim = 0;
    uint64_t hash = 0, generation = 0;
    bool valid = false;
  } shim;
};

namespace {

int check_ctx(fga_ctx* c) {
  if (!c) {
    set_error("null context");
    return FGA_ERR_INVALID;
  }
  if (cudaSetDevice(c->device) != cudaSuccess) {
    set_error("cudaSetDevice failed");
    return FGA_ERR_CUDA;
  }
  return FGA_OK;
}

#define CTX_TRY(c)                 \
  do {                             \
    int r_ = check_ctx(c);         \
    if (r_) return r_;             \
  } while (0)
#define TRY(expr)                  \
  do {                             \
    int r_ = (expr);               \
    if (r_) return r_;             \
  } while (0)

// D = 2 clouds ride the 3-D machinery as z = 0 (the tree then only ever
// takes the upper z child, so topology, preorder, lengths and forces are the
// quadtree's).  Host-side pad / unpad of (n, dim) arrays.
struct Pad3 {
  std::vector<double> buf;
  const double* ptr = nullptr;
};
Pad3 pad3(const double* p, int64_t n, int dim) {
  Pad3 r;
  if (dim == 3 || !p) {
    r.ptr = p;
    return r;
  }
  r.buf.assign((size_t)n * 3, 0.0);
  for (int64_t i = 0; i < n; i++)
    for (int k = 0; k < dim; k++) r.buf[i * 3 + k] = p[i * dim + k];
  r.ptr = r.buf.data();
  return r;
}
void unpad3(const double* p3, int64_t n, int dim, double* out) {
  for (int64_t i = 0; i < n; i++)
    for (int k = 0; k < dim; k++) out[i * dim + k] = p3[i * 3 + k];
}
int check_dim(int dim) {
  if (dim != 2 && dim != 3) {
    set_error("invalid parameter points=dimension " + std::to_string(dim));
    return FGA_ERR_INVALID;
  }
  return FGA_OK;
}

int invalid(const char* name, double v) {
  set_error(std::string("invalid parameter ") + name + "=" + std::to_string(v));
  return FGA_ERR_INVALID;
}

// Python repr() of a float: the shortest round-tripping digits, with ".0"
// on integral values and repr's exponent form (1e+16, 1e-05)
std::string py_repr(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  char buf[64];
  for (int p = 1; p <= 17; p++) {
    snprintf(buf, sizeof(buf), "%.*g", p, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string r(buf);
  const size_t e = r.find('e');
  if (e != std::string::npos) {
    const double ax = std::fabs(v);
    if (ax >= 1e-4 && ax < 1e16) {  // repr switches to exponent form outside this range
      snprintf(buf, sizeof(buf), "%.17f", v);
      r = buf;
      while (!r.empty() && r.back() == '0') r.pop_back();
      for (int p = 1; p <= 17; p++) {  // shortest fixed-form digits
        snprintf(buf, sizeof(buf), "%.*f", p, v);
        if (std::strtod(buf, nullptr) == v) {
          r = buf;
          break;
        }
      }
    } else {
      std::string mant = r.substr(0, e), ex = r.substr(e + 1);
      const char sign = ex[0] == '-' ? '-' : '+';
      if (ex[0] == '-' || ex[0] == '+') ex = ex.substr(1);
      while (ex.size() > 2 && ex[0] == '0') ex = ex.substr(1);
      return mant + "e" + sign + ex;
    }
  }
  if (r.find('.') == std::string::npos && r.find('e') == std::string::npos) r += ".0";
  return r;
}

// core.validate (core.py:127-151): first failing field.
int validate(const fga_params* p) {
  if (!p) {
    set_error("null params");
    return FGA_ERR_INVALID;
  }
  if (!(p->G > 0)) return invalid("G", p->G);
  if (!(p->epsilon >= 0)) return invalid("epsilon", p->epsilon);
  if (!(p->eta >= 0 && p->eta < 1)) return invalid("eta", p->eta);
  if (!(p->dt > 0)) return invalid("dt", p->dt);
  if (!(p->theta >= 0 && p->theta <= 1)) return invalid("theta", p->theta);
  if (!(p->sigma > 0)) return invalid("sigma", p->sigma);
  if (!(p->rho >= 2)) return invalid("rho", p->rho);
  if (!(p->max_depth >= 1)) return invalid("max_depth", p->max_depth);
  if (!(p->norm_a < p->norm_b)) {  // InvalidParam("norm_range", params.norm_range)
    set_error("invalid parameter norm_range=(" + py_repr(p->norm_a) + ", " + py_repr(p->norm_b) +
              ")");
    return FGA_ERR_INVALID;
  }
  if (!(p->conv_tol > 0)) return invalid("conv_tol", p->conv_tol);
  if (!(p->max_iters >= 1)) return invalid("max_iters", p->max_iters);
  return FGA_OK;
}

template <typename T>
int h2d(DevBuf& b, const T* src, int64_t count, cudaStream_t s) {
  FGA_CUDA_TRY(b.reserve(sizeof(T) * std::max<int64_t>(count, 1)));
  if (count > 0) FGA_CUDA_TRY(cudaMemcpyAsync(b.p, src, sizeof(T) * count, cudaMemcpyHostToDevice, s));
  return FGA_OK;
}

int sort_keys(DevBuf& tmp, DevBuf& kin, DevBuf& kout, DevBuf& iin, DevBuf& iout, int64_t n,
              int begin_bit, int end_bit, cudaStream_t s) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin.as<unsigned long long>(),
                                  kout.as<unsigned long long>(), iin.as<int>(), iout.as<int>(),
                                  (int)n, begin_bit, end_bit, s);
  FGA_CUDA_TRY(tmp.reserve(bytes));
  FGA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, kin.as<unsigned long long>(),
                                               kout.as<unsigned long long>(), iin.as<int>(),
                                               iout.as<int>(), (int)n, begin_bit, end_bit, s));
  return FGA_OK;
}

// Space-filling-curve (Hilbert, setup.cu k_morton) order of an AoS (n,3)
// device cloud -> iout (int, n)
int morton_order(const double* pts, int64_t n, DevBuf& kin, DevBuf& kout, DevBuf& iin,
                 DevBuf& iout, DevBuf& tmp, DevBuf& scratch, cudaStream_t s) {
  FGA_CUDA_TRY(kin.reserve(sizeof(unsigned long long) * n));
  FGA_CUDA_TRY(kout.reserve(sizeof(unsigned long long) * n));
  FGA_CUDA_TRY(iin.reserve(sizeof(int) * n));
  FGA_CUDA_TRY(iout.reserve(sizeof(int) * n));
  FGA_CUDA_TRY(scratch.reserve(sizeof(double) * (6 * 600 + 16)));
  double* box = scratch.as<double>() + 6 * 600;
  launch_bbox(pts, n, scratch.as<double>(), box, s);
  launch_morton_keys(pts, n, box, kin.as<unsigned long long>(), iin.as<int>(), s);
  // locality only: the top 30 bits (10 per axis, 4 radix passes instead of 8)
  // order the cloud; equal prefixes keep their input order (stable sort)
  return sort_keys(tmp, kin, kout, iin, iout, n, 33, 63, s);
}

// -------------------------------------------------------------------- session

// every stride-th entry of a permutation (balanced_cut's query sample)
__global__ void k_capi_strided_order(const int* __restrict__ order, int64_t ms, int64_t stride,
                                     int* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ms) out[i] = order[i * stride];
}

// Template shards of equal COST instead of equal count (shard_count > 1, BH):
// the per-query visit counts of every stride-th template point in Morton
// order (one FP32 operator pass over <= 65,536 sampled queries, identical on
// every rank: same inputs, integer counts), their running sum, and rank r's
// chunk between the sample positions where it crosses r/N and (r+1)/N of the
// total.  Equal-count shards of the 1M pair differed by up to 1.2x in cost
// (tools/smallm_timing.py).  FGA_SHARD_BALANCE=0: equal counts.
int balanced_cut(Session& S, int64_t m, cudaStream_t s) {
  static const bool on = !(getenv("FGA_SHARD_BALANCE") && atoi(getenv("FGA_SHARD_BALANCE")) == 0);
  if (!on || m < 2 * (int64_t)S.shard_count) return FGA_OK;
  const int64_t stride = std::max<int64_t>(1, (m + 65535) / 65536);
  const int64_t ms = (m + stride - 1) / stride;
  DevBuf ord, q, out;
  FGA_CUDA_TRY(ord.reserve(sizeof(int) * ms));
  FGA_CUDA_TRY(q.reserve(sizeof(double) * 4 * ms));
  FGA_CUDA_TRY(out.reserve(sizeof(double) * 3 * ms + sizeof(long long) * ms));
  k_capi_strided_order<<<(unsigned)((ms + 255) / 256), 256, 0, s>>>(
      S.tidx.as<int>(), ms, stride, ord.as<int>());
  double* b = q.as<double>();
  launch_gather_queries(S.yn.as<double>(), S.my.as<double>(), ord.as<int>(), ms, b, b + ms,
                        b + 2 * ms, b + 3 * ms, s);
  long long* vis = reinterpret_cast<long long*>(out.as<double>() + 3 * ms);
  launch_bh_operator(S.tree, b, b + ms, b + 2 * ms, b + 3 * ms, nullptr, ms, S.P.theta, S.sp.G,
                     S.sp.eps2, out.as<double>(), vis, nullptr, nullptr, FGA_PREC_FP32, s);
  std::vector<long long> v(ms);
  FGA_CUDA_TRY(cudaMemcpyAsync(v.data(), vis, sizeof(long long) * ms, cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  double total = 0.0;
  for (long long x : v) total += (double)x;
  if (!(total > 0.0)) return FGA_OK;
  // the first sample index whose running sum reaches frac * total, as a
  // template position (ranks 0 and N get 0 and m)
  auto cut = [&](int r) -> int64_t {
    if (r <= 0) return 0;
    if (r >= S.shard_count) return m;
    const double target = total * (double)r / (double)S.shard_count;
    double c = 0.0;
    for (int64_t j = 0; j < ms; j++) {
      c += (double)v[j];
      if (c >= target) return std::min<int64_t>(m, (j + 1) * stride);
    }
    return m;
  };
  const int64_t b0 = cut(S.shard_rank), b1 = cut(S.shard_rank + 1);
  S.m_begin = b0;
  S.m_local = std::max<int64_t>(0, b1 - b0);
  return FGA_OK;
}

int session_setup(fga_ctx* c, const double* x_dev, const double* y_dev) {
  Session& S = c->S;
  cudaStream_t s = c->stream;
  const int64_t n = S.n, m = S.m;
  const double a = S.P.norm_a, b = S.P.norm_b;
  FGA_CUDA_TRY(cudaEventRecord(c->ev[0], s));
  FGA_CUDA_TRY(S.xn.reserve(sizeof(double) * 3 * n));
  FGA_CUDA_TRY(S.yn.reserve(sizeof(double) * 3 * m));
  FGA_CUDA_TRY(S.ctx_dev.reserve(sizeof(double) * 16));
  FGA_CUDA_TRY(S.scratch.reserve(sizeof(double) * 8192));
  if (S.O.normalize) {
    TRY(normalize_pair_dev(x_dev, n, y_dev, m, a, b, S.xn.as<double>(), S.yn.as<double>(),
                           S.ctx_dev.as<double>(), S.scratch.as<double>(), S.scratch.bytes,
                           S.ctx10, s));
  } else {
    // registration.py:108-114: identity context spanning [a, b]
    FGA_CUDA_TRY(cudaMemcpyAsync(S.xn.p, x_dev, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
    FGA_CUDA_TRY(cudaMemcpyAsync(S.yn.p, y_dev, sizeof(double) * 3 * m, cudaMemcpyDeviceToDevice, s));
    const double z[10] = {0, 0, 0, 0, 0, 0, a, b, a, b};
    std::memcpy(S.ctx10, z, sizeof(z));
  }
  // mass fields (registration.py:64-88)
  FGA_CUDA_TRY(S.mx.reserve(sizeof(double) * n));
  FGA_CUDA_TRY(S.my.reserve(sizeof(double) * m));
  const int64_t ncell = (int64_t)S.P.rho * S.P.rho * (S.sp.dim == 3 ? S.P.rho : 1);
  FGA_CUDA_TRY(S.flat.reserve(sizeof(int) * std::max(n, m)));
  FGA_CUDA_TRY(S.counts.reserve(sizeof(long long) * (ncell + 1)));
  FGA_CUDA_TRY(S.cells.reserve(sizeof(double) * ncell));
  const double ca = S.ctx10[8], cb = S.ctx10[9];
  if (S.O.x_weights) {
    TRY(h2d(S.scratch, S.O.x_weights, n, s));
    launch_external_masses(S.scratch.as<double>(), n, S.mx.as<double>(), s);
    FGA_CUDA_TRY(cudaStreamSynchronize(s));
  } else if (S.O.mass_field == 1) {
    TRY(knn_dev(S.xn.as<double>(), n, S.sp.dim, S.O.knn_k, nullptr, nullptr, S.mx.as<double>(),
                S.scratch, S.cub_tmp, s));
  } else {
    TRY(niv_masses_dev(S.xn.as<double>(), n, S.sp.dim, S.P.rho, ca, cb, S.P.max_depth, S.mx.as<double>(),
                       S.flat.as<int>(), S.counts.as<long long>(), S.cells.as<double>(), s));
  }
  if (S.O.y_weights) {
    TRY(h2d(S.scratch, S.O.y_weights, m, s));
    launch_external_masses(S.scratch.as<double>(), m, S.my.as<double>(), s);
    FGA_CUDA_TRY(cudaStreamSynchronize(s));
  } else if (S.O.mass_field == 1) {
    TRY(knn_dev(S.yn.as<double>(), m, S.sp.dim, S.O.knn_k, nullptr, nullptr, S.my.as<double>(),
                S.scratch, S.cub_tmp, s));
  } else {
    TRY(niv_masses_dev(S.yn.as<double>(), m, S.sp.dim, S.P.rho, ca, cb, S.P.max_depth, S.my.as<double>(),
                       S.flat.as<int>(), S.counts.as<long long>(), S.cells.as<double>(), s));
  }
  // landmark SPM: field * RBF (registration.py:74-83; only for NIV fields)
  if (S.O.n_landmarks > 0) {
    const int L = S.O.n_landmarks;
    if (!S.O.x_weights) {
      TRY(h2d(S.lm_idx, reinterpret_cast<const long long*>(S.O.x_landmarks), L, s));
      TRY(rbf_apply_dev(S.xn.as<double>(), n, S.lm_idx.as<long long>(), L, S.P.sigma, 1,
                        S.mx.as<double>(), S.rbf_scratch, s));
    }
    if (!S.O.y_weights) {
      TRY(h2d(S.lm_idx, reinterpret_cast<const long long*>(S.O.y_landmarks), L, s));
      TRY(rbf_apply_dev(S.yn.as<double>(), m, S.lm_idx.as<long long>(), L, S.P.sigma, 1,
                        S.my.as<double>(), S.rbf_scratch, s));
    }
  }
  FGA_CUDA_TRY(S.scratch.reserve(sizeof(double) * (8 + pairwise_sum_scratch_doubles(n) + 600)));
  launch_rescale(S.mx.as<double>(), n, S.my.as<double>(), m, S.P.dt, S.P.eta,
                 S.scratch.as<double>(), s);
  // reference side: tree (BH) and packed points (direct sum, energy)
  if (!S.direct || S.P.theta == 0.0) {
    TRY(tree_build_dev(S.tree, S.xn.as<double>(), S.mx.as<double>(), n, S.P.max_depth, s));
    S.tree.dim = S.sp.dim;
    if (S.tree.cap_distinct) {
      set_error("max_depth > 42 with distinct reference points closer than 2^-42 of the box "
                "(the GPU tree has at most 42 levels)");
      return FGA_ERR_UNSUPPORTED;
    }
  }
  if (S.P.theta == 0.0) {
    // theta = 0 opens every cell, so the reference sums over the leaves
    // (_kernels.py:30-42): the exact O(NM) sum equals that only when no leaf
    // aggregates two distinct points; otherwise traverse the tree at theta=0
    int shared = 0;
    TRY(tree_any_shared_leaf(S.tree, s, &shared));
    S.direct = !shared;
  }
  FGA_CUDA_TRY(S.ref32.reserve(sizeof(float4) * n));
  if (S.precision) FGA_CUDA_TRY(S.ref64.reserve(sizeof(double4) * n));
  launch_pack_ref(S.xn.as<double>(), S.mx.as<double>(), n, S.ref32.as<float4>(),
                  S.precision ? S.ref64.as<double4>() : nullptr, s);
  // template: Morton order, this shard's contiguous chunk
  TRY(morton_order(S.yn.as<double>(), m, S.tkeys_in, S.tkeys, S.tidx_in, S.tidx, S.cub_tmp,
                   S.scratch, s));
  S.m_begin = m * S.shard_rank / S.shard_count;
  S.m_local = m * (S.shard_rank + 1) / S.shard_count - S.m_begin;
  if (S.shard_count > 1 && !S.direct) TRY(balanced_cut(S, m, s));
  FGA_CUDA_TRY(S.tpl.reserve(sizeof(double) * 7 * std::max<int64_t>(S.m_local, 1)));
  launch_gather_template(S.yn.as<double>(), S.my.as<double>(), S.tidx.as<int>(), S.m_begin,
                         S.m_local, S.view(), s);
  // iteration state
  FGA_CUDA_TRY(S.state.reserve(sizeof(IterState)));
  FGA_CUDA_TRY(S.sums.reserve(sizeof(double) * kPartialStride));
  launch_mean3(S.yn.as<double>(), m, S.scratch.as<double>(), S.scratch.as<double>() + 4096, s);
  launch_state_init(S.st(), S.scratch.as<double>() + 4096, s);
  const int64_t nw = S.direct ? direct_iterate_warps(S.m_local, S.precision)
                              : bh_iterate_warps(S.m_local, S.precision);
  FGA_CUDA_TRY(S.partials.reserve(sizeof(double) * kPartialStride * std::max<int64_t>(nw, 1)));
  FGA_CUDA_TRY(S.gpe_part.reserve(sizeof(double) * std::max<int64_t>(gpe_warps(S.m_local, n, S.precision), 1)));
  FGA_CUDA_TRY(S.red_stage.reserve(sizeof(double) * reduce_stage_doubles()));
  const int64_t mi = S.P.max_iters;
  FGA_CUDA_TRY(S.rec_delta.reserve(sizeof(double) * mi));
  FGA_CUDA_TRY(S.rec_traj.reserve(sizeof(double) * 12 * mi));
  FGA_CUDA_TRY(S.rec_gpe.reserve(sizeof(double) * mi));
  FGA_CUDA_TRY(S.rec_inter.reserve(sizeof(long long) * mi));
  FGA_CUDA_TRY(S.rec_visits.reserve(sizeof(long long) * mi));
  FGA_CUDA_TRY(cudaMemsetAsync(S.rec_gpe.p, 0xff, sizeof(double) * mi, s));  // NaN
  FGA_CUDA_TRY(cudaEventRecord(c->ev[1], s));
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

int session_begin_common(fga_ctx* c, int64_t n, int64_t m, int dim, const fga_params* params,
                         const fga_options* options, int shard_rank, int shard_count) {
  TRY(validate(params));
  if (n <= 0 || m <= 0) {
    set_error("registration requires a non-empty cloud");
    return FGA_ERR_EMPTY;
  }
  TRY(check_dim(dim));
  if (shard_count < 1 || shard_rank < 0 || shard_rank >= shard_count) {
    set_error("invalid shard_rank/shard_count");
    return FGA_ERR_INVALID;
  }
  Session& S = c->S;
  S.active = false;
  S.P = *params;
  fga_options def{};
  def.normalize = 1;
  def.compute_gpe = 1;
  S.O = options ? *options : def;
  if (S.O.poll_every <= 0) S.O.poll_every = 8;
  if (S.O.knn_k <= 0) S.O.knn_k = 16;
  if (S.O.n_landmarks > 0) {  // LandmarkSet.check_bounds (masses.py:44-48)
    for (int j = 0; j < S.O.n_landmarks; j++) {
      if (S.O.y_landmarks[j] < 0 || S.O.y_landmarks[j] >= m) {
        set_error("invalid parameter pairs=template index out of range");
        return FGA_ERR_INVALID;
      }
      if (S.O.x_landmarks[j] < 0 || S.O.x_landmarks[j] >= n) {
        set_error("invalid parameter pairs=reference index out of range");
        return FGA_ERR_INVALID;
      }
    }
  }
  if (S.O.mass_field == 1 && (S.O.knn_k >= n || S.O.knn_k >= m || S.O.knn_k > 32)) {
    set_error("invalid parameter knn_k=" + std::to_string(S.O.knn_k));
    return FGA_ERR_INVALID;
  }
  S.precision = S.O.precision ? 1 : 0;
  S.direct = params->theta == 0.0;
  S.n = n;
  S.m = m;
  S.shard_rank = shard_rank;
  S.shard_count = shard_count;
  S.sp.G = params->G;
  S.sp.eps = params->epsilon;
  S.sp.eps2 = params->epsilon * params->epsilon;  // float(params.epsilon) ** 2 (bhtree.py:142)
  S.sp.eta = params->eta;
  S.sp.dt = params->dt;
  S.sp.theta = params->theta;
  S.sp.theta2 = params->theta * params->theta;  // _kernels.py:14
  S.sp.conv_tol = params->conv_tol;
  S.sp.max_iters = params->max_iters;
  S.sp.m_total = m;
  S.sp.trace_gpe = S.O.trace_gpe;
  S.sp.count_visits = S.O.count_visits ? 1 : 0;
  S.sp.dim = dim;
  S.gpe_initial = S.gpe_final = NAN;
  S.have_gpe_initial = S.have_gpe_final = false;
  S.applied = false;
  S.passes = 0;
  S.last_pass_gpe = false;
  S.split_traced = false;
  S.order_ready = false;
  S.split_mode = false;
  S.sums_ext = nullptr;
  return FGA_OK;
}

int session_gpe(fga_ctx* c, const IterState* gate) {
  Session& S = c->S;
  TemplateView tv = S.view();
  const int64_t ngw = gpe_warps(S.m_local, S.ref().n, S.precision);
  launch_gpe(S.ref(), tv.px, tv.py, tv.pz, tv.mq, S.m_local, S.sp.eps, gate, S.gpe_part.as<double>(),
             S.precision, c->stream);
  launch_reduce(S.partials.as<double>(), 0, S.gpe_part.as<double>(), S.m_local > 0 ? ngw : 0, -1.0,
                S.sums_ptr(), S.red_stage.as<double>(), c->stream);
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

// fuse: the caller runs the update right after (fga_session_iterate): small
// passes then reduce and update in one kernel (launch_reduce_update)
constexpr int64_t kSplitPartsMax = 8;  // >= forces.cu FGA_SPLIT_PARTS
int session_forces(fga_ctx* c, bool fuse = false) {
  Session& S = c->S;
  cudaStream_t s = c->stream;
  TemplateView tv = S.view();
  int64_t nw;
  if (S.direct) {
    launch_direct_iterate(S.ref(), tv, S.st(), S.sp, S.partials.as<double>(), S.precision, s);
    nw = direct_iterate_warps(S.m_local, S.precision);
  } else {
    SplitBufs sb{nullptr, nullptr, nullptr, &S.split_traced};
    if (S.m_local > 0) {
      const int64_t nwq = (S.m_local + 31) / 32;
      FGA_CUDA_TRY(S.split_trace.reserve(sizeof(int) * kTraceLen * (nwq + 8)));
      sb.trace = S.split_trace.as<int>();
      // the split parts' buffers only where split passes can run (a pass of
      // at most one wave: forces.cu bh_split_possible)
      if (!S.precision && bh_split_possible(S.m_local)) {
        FGA_CUDA_TRY(S.split_f.reserve(sizeof(double) * 3 * kSplitPartsMax * S.m_local));
        FGA_CUDA_TRY(S.split_a.reserve(sizeof(int) * kSplitPartsMax * S.m_local));
        sb.fpart = S.split_f.as<double>();
        sb.apart = S.split_a.as<int>();
      }
      const int64_t nblk = nwq / 2 + 8;  // >= blocks of any block size >= 64 threads
      FGA_CUDA_TRY(S.order_buf.reserve(sizeof(int) * 4 * nblk + (4 << 20)));
      sb.order = S.order_buf.as<int>();
      sb.okeys = sb.order + nblk;
      const uintptr_t t0 = reinterpret_cast<uintptr_t>(sb.okeys + 3 * nblk);
      sb.tmp = reinterpret_cast<void*>((t0 + 255) & ~uintptr_t(255));
      sb.tmp_bytes = (4 << 20) - 256;
      sb.have_order = &S.order_ready;
      sb.split = &S.split_mode;
    }
    launch_bh_iterate(c->S.tree, tv, S.st(), S.sp, S.partials.as<double>(), S.precision, s,
                      sb.trace ? &sb : nullptr);
    nw = bh_iterate_warps(S.m_local, S.precision);
  }
  if (S.m_local <= 0) nw = 0;
  const bool with_gpe = S.O.trace_gpe && S.passes > 0;
  int64_t ngw = 0;
  if (with_gpe && S.m_local > 0) {
    launch_gpe(S.ref(), tv.px, tv.py, tv.pz, tv.mq, S.m_local, S.sp.eps, S.st(),
               S.gpe_part.as<double>(), S.precision, s);
    ngw = gpe_warps(S.m_local, S.ref().n, S.precision);
  }
  const double pairs = S.direct ? (double)S.n * (double)S.m_local : -1.0;
  S.last_pass_gpe = with_gpe;
  S.passes++;
  if (fuse && reduce_update_fusable(nw, ngw)) {
    launch_reduce_update(S.partials.as<double>(), nw, S.gpe_part.as<double>(), ngw, pairs,
                         S.sums_ptr(), S.st(), S.sp, S.rec_delta.as<double>(),
                         S.rec_traj.as<double>(), S.rec_gpe.as<double>(),
                         S.rec_inter.as<long long>(), S.rec_visits.as<long long>(),
                         with_gpe ? 1 : 0, s);
    S.fused_update = true;
  } else {
    launch_reduce(S.partials.as<double>(), nw, S.gpe_part.as<double>(), ngw, pairs,
                  S.sums_ptr(), S.red_stage.as<double>(), s);
    S.fused_update = false;
  }
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

int session_update(fga_ctx* c) {
  Session& S = c->S;
  launch_update(S.sums_ptr(), S.st(), S.sp, S.rec_delta.as<double>(),
                S.rec_traj.as<double>(), S.rec_gpe.as<double>(), S.rec_inter.as<long long>(),
                S.rec_visits.as<long long>(), S.last_pass_gpe ? 1 : 0, c->stream);
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

int session_poll(fga_ctx* c, int* done, int64_t* iters) {
  Session& S = c->S;
  const char* st = reinterpret_cast<const char*>(S.st());
  FGA_CUDA_TRY(cudaMemcpyAsync(c->pinned, st + offsetof(IterState, iter), sizeof(long long) + 2 * sizeof(int),
                               cudaMemcpyDeviceToHost, c->stream));
  FGA_CUDA_TRY(cudaStreamSynchronize(c->stream));
  long long it;
  std::memcpy(&it, c->pinned, sizeof(long long));
  int dn;
  std::memcpy(&dn, reinterpret_cast<char*>(c->pinned) + sizeof(long long), sizeof(int));
  if (done) *done = dn;
  if (iters) *iters = it;
  return FGA_OK;
}

int session_apply(fga_ctx* c) {
  Session& S = c->S;
  if (!S.applied) {
    launch_apply_pending(S.view(), S.st(), c->stream);
    S.applied = true;
  }
  FGA_CUDA_TRY(cudaGetLastError());
  return FGA_OK;
}

int take_gpe(fga_ctx* c, double* value) {
  Session& S = c->S;
  double v = 0.0;
  FGA_CUDA_TRY(cudaMemcpyAsync(&v, S.sums_ptr() + kGpe, sizeof(double), cudaMemcpyDeviceToHost,
                               c->stream));
  FGA_CUDA_TRY(cudaStreamSynchronize(c->stream));
  *value = -S.P.G * v;  // _kernels.py:67
  return FGA_OK;
}

// denormalize_translation (normalize.py:73-84)
void denormalize(const double R[9], const double t[3], const double* ctx, double tout[3]) {
  const double l = ctx[6], r = ctx[7], a = ctx[8], b = ctx[9];
  const double inv_scale = (r - l) / (b - a);
  for (int i = 0; i < 3; i++) {
    double v1 = 0.0, v2 = 0.0;
    for (int k = 0; k < 3; k++) {
      v1 += -R[3 * i + k] * (ctx[3 + k] + l);
      v2 += R[3 * i + k] * a;
    }
    tout[i] = ((v1 + inv_scale * ((v2 + t[i]) - a)) + ctx[i]) + l;
  }
}

}  // namespace

// ======================================================================== C ABI
extern "C" {

int fga_version(void) { return 100; }
const char* fga_last_error(void) { return fga::last_error(); }

int fga_device_count(int* count) {
  if (!count) return FGA_ERR_INVALID;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    set_error(std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    return FGA_ERR_CUDA;
  }
  *count = n;
  return FGA_OK;
}

int fga_create(fga_ctx** out, int device) {
  if (!out) return FGA_ERR_INVALID;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
    set_error("no CUDA device visible: libfga has no CPU fallback");
    return FGA_ERR_CUDA;
  }
  if (device < 0 || device >= n) {
    set_error("device index out of range");
    return FGA_ERR_INVALID;
  }
  FGA_CUDA_TRY(cudaSetDevice(device));
  fga_ctx* c = new fga_ctx();
  c->device = device;
  FGA_CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->own_stream = true;
  FGA_CUDA_TRY(cudaMallocHost(&c->pinned, 64));
  for (auto& e : c->ev) FGA_CUDA_TRY(cudaEventCreate(&e));
  *out = c;
  return FGA_OK;
}

int fga_destroy(fga_ctx* c) {
  if (!c) return FGA_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  c->tree.release();
  c->S.tree.release();
  c->tree_pts.release();
  c->tree_masses.release();
  for (auto& b : c->op) b.release();
  for (auto& b : c->batch_in) b.release();
  c->batch_scratch.release();
  c->batch_out.release();
  c->batch_deltas.release();
  c->batch_counter.release();
  c->batch_wide.release();
  c->op_total.release();
  c->op_trace.release();
  c->op_fpart.release();
  c->op_cnt.release();
  for (int k = 0; k < 4; k++) {
    if (c->stage[k]) cudaFreeHost(c->stage[k]);
    if (c->stage_ev[k]) cudaEventDestroy(c->stage_ev[k]);
    c->stage[k] = nullptr;
    c->stage_ev[k] = nullptr;
  }
  Session& S = c->S;
  S.lm_idx.release();
  S.rbf_scratch.release();
  S.ckpt.release();
  S.split_trace.release();
  S.split_f.release();
  S.split_a.release();
  S.order_buf.release();
  DevBuf* all[] = {&S.x_raw,   &S.y_raw,  &S.xn,        &S.yn,       &S.ctx_dev,   &S.mx,
                   &S.my,      &S.flat,   &S.counts,    &S.cells,    &S.ref32,     &S.ref64,
                   &S.tkeys_in, &S.tkeys, &S.tidx_in,   &S.tidx,     &S.cub_tmp,   &S.tpl,
                   &S.partials, &S.gpe_part, &S.sums,   &S.state,    &S.scratch,   &S.rec_delta,
                   &S.rec_traj, &S.rec_gpe, &S.rec_inter, &S.rec_visits};
  for (DevBuf* b : all) b->release();
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->aev)
    if (e) cudaEventDestroy(e);
  if (c->aux) {
    cudaStreamSynchronize(c->aux);
    cudaStreamDestroy(c->aux);
  }
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return FGA_OK;
}

int fga_set_stream(fga_ctx* c, void* stream) {
  CTX_TRY(c);
  if (c->own_stream && c->stream) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
  }
  c->stream = (cudaStream_t)stream;  // NULL = the legacy default stream (torch's default)
  c->own_stream = false;
  return FGA_OK;
}

int fga_synchronize(fga_ctx* c) {
  CTX_TRY(c);
  FGA_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FGA_OK;
}

// ------------------------------------------------------------------ session
int fga_session_begin_dev(fga_ctx* c, const double* x_dev, int64_t n, const double* y_dev,
                          int64_t m, int dim, const fga_params* params,
                          const fga_options* options, int shard_rank, int shard_count) {
  CTX_TRY(c);
  if (dim != 3) {
    set_error("fga_session_begin_dev: device inputs must be (n, 3)");
    return FGA_ERR_UNSUPPORTED;
  }
  TRY(session_begin_common(c, n, m, dim, params, options, shard_rank, shard_count));
  TRY(session_setup(c, x_dev, y_dev));
  c->S.active = true;
  return FGA_OK;
}

int fga_session_begin(fga_ctx* c, const double* x, int64_t n, const double* y, int64_t m, int dim,
                      const fga_params* params, const fga_options* options, int shard_rank,
                      int shard_count) {
  CTX_TRY(c);
  TRY(session_begin_common(c, n, m, dim, params, options, shard_rank, shard_count));
  Session& S = c->S;
  const Pad3 px = pad3(x, n, dim), py = pad3(y, m, dim);
  TRY(h2d(S.x_raw, px.ptr, 3 * n, c->stream));
  TRY(h2d(S.y_raw, py.ptr, 3 * m, c->stream));
  FGA_CUDA_TRY(cudaStreamSynchronize(c->stream));  // pad buffers die here
  TRY(session_setup(c, S.x_raw.as<double>(), S.y_raw.as<double>()));
  S.active = true;
  return FGA_OK;
}

#define SESSION_TRY(c)                                   \
  do {                                                   \
    CTX_TRY(c);                                          \
    if (!c->S.active) {                                  \
      set_error("no active registration session");      \
      return FGA_ERR_STATE;                              \
    }                                                    \
  } while (0)

int fga_session_forces(fga_ctx* c) {
  SESSION_TRY(c);
  return session_forces(c);
}
int fga_session_sums(fga_ctx* c, void** dev_ptr) {
  SESSION_TRY(c);
  if (!dev_ptr) return FGA_ERR_INVALID;
  *dev_ptr = c->S.sums_ptr();
  return FGA_OK;
}
int fga_session_bind_sums(fga_ctx* c, void* dev_ptr) {
  SESSION_TRY(c);
  c->S.sums_ext = static_cast<double*>(dev_ptr);
  return FGA_OK;
}
int fga_session_update(fga_ctx* c) {
  SESSION_TRY(c);
  return session_update(c);
}
int fga_session_iterate(fga_ctx* c, int k) {
  SESSION_TRY(c);
  if (c->S.shard_count != 1) {
    set_error("fga_session_iterate: sharded sessions need the host collective between passes");
    return FGA_ERR_STATE;
  }
  for (int i = 0; i < k; i++) {
    TRY(session_forces(c, true));
    if (!c->S.fused_update) TRY(session_update(c));
  }
  return FGA_OK;
}
int fga_session_gpe(fga_ctx* c) {
  SESSION_TRY(c);
  return session_gpe(c, nullptr);
}
int fga_session_take_gpe(fga_ctx* c, double* value) {
  SESSION_TRY(c);
  if (!value) return FGA_ERR_INVALID;
  return take_gpe(c, value);
}
int fga_session_set_gpe(fga_ctx* c, int which, double value) {
  SESSION_TRY(c);
  if (which == 0) {
    c->S.gpe_initial = value;
    c->S.have_gpe_initial = true;
  } else {
    c->S.gpe_final = value;
    c->S.have_gpe_final = true;
  }
  return FGA_OK;
}
int fga_session_poll(fga_ctx* c, int* done, int64_t* iterations) {
  SESSION_TRY(c);
  return session_poll(c, done, iterations);
}
int fga_session_apply_pending(fga_ctx* c) {
  SESSION_TRY(c);
  return session_apply(c);
}
int fga_session_info(fga_ctx* c, int64_t* m_local, int64_t* n_nodes) {
  SESSION_TRY(c);
  if (m_local) *m_local = c->S.m_local;
  if (n_nodes) *n_nodes = c->S.direct ? 0 : c->S.tree.n_nodes;
  return FGA_OK;
}

int fga_session_get_state(fga_ctx* c, double* pos, double* vel, double* racc9, double* tacc3,
                          int64_t* iter) {
  SESSION_TRY(c);
  Session& S = c->S;
  cudaStream_t s = c->stream;
  if (pos || vel) {
    FGA_CUDA_TRY(S.scratch.reserve(sizeof(double) * 6 * std::max<int64_t>(S.m, 1)));
    double* dp = S.scratch.as<double>();
    double* dv = dp + 3 * S.m;
    if (pos) FGA_CUDA_TRY(cudaMemcpyAsync(dp, pos, sizeof(double) * 3 * S.m, cudaMemcpyHostToDevice, s));
    if (vel) FGA_CUDA_TRY(cudaMemcpyAsync(dv, vel, sizeof(double) * 3 * S.m, cudaMemcpyHostToDevice, s));
    launch_state_get(S.view(), S.st(), S.tidx.as<int>(), S.m_begin, dp, dv, s);
    FGA_CUDA_TRY(cudaGetLastError());
    if (pos) FGA_CUDA_TRY(cudaMemcpyAsync(pos, dp, sizeof(double) * 3 * S.m, cudaMemcpyDeviceToHost, s));
    if (vel) FGA_CUDA_TRY(cudaMemcpyAsync(vel, dv, sizeof(double) * 3 * S.m, cudaMemcpyDeviceToHost, s));
  }
  IterState st;
  FGA_CUDA_TRY(cudaMemcpyAsync(&st, S.st(), sizeof(st), cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  if (racc9)
    for (int k = 0; k < 9; k++) racc9[k] = st.Racc[k];
  if (tacc3)
    for (int k = 0; k < 3; k++) tacc3[k] = st.tacc[k];
  if (iter) *iter = st.iter;
  return FGA_OK;
}

int fga_session_set_state(fga_ctx* c, const double* pos, const double* vel, const double* racc9,
                          const double* tacc3, int64_t iter) {
  SESSION_TRY(c);
  Session& S = c->S;
  cudaStream_t s = c->stream;
  if (!pos || !vel || !racc9 || !tacc3) {
    set_error("set_state: positions, velocities, R_acc and t_acc are required");
    return FGA_ERR_INVALID;
  }
  if (iter < 0 || iter >= S.sp.max_iters) {
    set_error("set_state: iteration outside [0, max_iters)");
    return FGA_ERR_INVALID;
  }
  FGA_CUDA_TRY(S.scratch.reserve(sizeof(double) * 6 * std::max<int64_t>(S.m, 1)));
  double* dp = S.scratch.as<double>();
  double* dv = dp + 3 * S.m;
  FGA_CUDA_TRY(cudaMemcpyAsync(dp, pos, sizeof(double) * 3 * S.m, cudaMemcpyHostToDevice, s));
  FGA_CUDA_TRY(cudaMemcpyAsync(dv, vel, sizeof(double) * 3 * S.m, cudaMemcpyHostToDevice, s));
  launch_state_set(S.view(), S.tidx.as<int>(), S.m_begin, dp, dv, s);
  FGA_CUDA_TRY(cudaGetLastError());
  IterState st;
  FGA_CUDA_TRY(cudaMemcpyAsync(&st, S.st(), sizeof(st), cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  double mean[3] = {0.0, 0.0, 0.0};
  for (int64_t i = 0; i < S.m; i++)
    for (int k = 0; k < 3; k++) mean[k] += pos[i * 3 + k];
  for (int k = 0; k < 9; k++) {
    st.Rp[k] = (k % 4 == 0) ? 1.0 : 0.0;
    st.Racc[k] = racc9[k];
  }
  for (int k = 0; k < 3; k++) {
    st.tp[k] = 0.0;
    st.tacc[k] = tacc3[k];
    st.shift[k] = S.m > 0 ? mean[k] / (double)S.m : 0.0;
  }
  st.iter = iter;
  st.done = 0;
  st.converged = 0;
  st.gpe_pending = 0;
  FGA_CUDA_TRY(cudaMemcpyAsync(S.st(), &st, sizeof(st), cudaMemcpyHostToDevice, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  S.applied = false;
  S.have_gpe_final = false;
  return FGA_OK;
}

int fga_session_checkpoint(fga_ctx* c, int restore) {
  SESSION_TRY(c);
  Session& S = c->S;
  cudaStream_t s = c->stream;
  const size_t tpl = sizeof(double) * 7 * std::max<int64_t>(S.m_local, 1);
  if (!restore) {
    FGA_CUDA_TRY(S.ckpt.reserve(tpl + sizeof(IterState)));
    FGA_CUDA_TRY(cudaMemcpyAsync(S.ckpt.p, S.tpl.p, tpl, cudaMemcpyDeviceToDevice, s));
    FGA_CUDA_TRY(cudaMemcpyAsync(S.ckpt.as<char>() + tpl, S.state.p, sizeof(IterState),
                                 cudaMemcpyDeviceToDevice, s));
    S.have_ckpt = true;
    return FGA_OK;
  }
  if (!S.have_ckpt) {
    set_error("checkpoint: nothing saved in this session");
    return FGA_ERR_STATE;
  }
  FGA_CUDA_TRY(cudaMemcpyAsync(S.tpl.p, S.ckpt.p, tpl, cudaMemcpyDeviceToDevice, s));
  FGA_CUDA_TRY(cudaMemcpyAsync(S.state.p, S.ckpt.as<char>() + tpl, sizeof(IterState),
                               cudaMemcpyDeviceToDevice, s));
  S.applied = false;
  S.have_gpe_final = false;
  return FGA_OK;
}

int fga_session_masses(fga_ctx* c, double* mx, double* my) {
  SESSION_TRY(c);
  Session& S = c->S;
  if (mx)
    FGA_CUDA_TRY(cudaMemcpyAsync(mx, S.mx.p, sizeof(double) * S.n, cudaMemcpyDeviceToHost, c->stream));
  if (my)
    FGA_CUDA_TRY(cudaMemcpyAsync(my, S.my.p, sizeof(double) * S.m, cudaMemcpyDeviceToHost, c->stream));
  FGA_CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FGA_OK;
}

int fga_session_finish(fga_ctx* c, fga_result* out, double* deltas, double* traj,
                       double* gpe_trace, int64_t* inter, int64_t* visits) {
  SESSION_TRY(c);
  Session& S = c->S;
  cudaStream_t s = c->stream;
  TRY(session_apply(c));
  if (S.O.compute_gpe && !S.have_gpe_final && S.shard_count == 1) {
    FGA_CUDA_TRY(cudaEventRecord(c->ev[4], s));
    TRY(session_gpe(c, nullptr));
    double v;
    TRY(take_gpe(c, &v));
    FGA_CUDA_TRY(cudaEventRecord(c->ev[5], s));
    S.gpe_final = v;
    S.have_gpe_final = true;
  }
  IterState st;
  FGA_CUDA_TRY(cudaMemcpyAsync(&st, S.st(), sizeof(IterState), cudaMemcpyDeviceToHost, s));
  const int64_t it = 0;
  (void)it;
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t iters = st.iter;
  std::vector<long long> iv(std::max<int64_t>(iters, 1)), vv(std::max<int64_t>(iters, 1));
  if (iters > 0) {
    if (deltas) FGA_CUDA_TRY(cudaMemcpyAsync(deltas, S.rec_delta.p, sizeof(double) * iters, cudaMemcpyDeviceToHost, s));
    if (traj) FGA_CUDA_TRY(cudaMemcpyAsync(traj, S.rec_traj.p, sizeof(double) * 12 * iters, cudaMemcpyDeviceToHost, s));
    if (gpe_trace) FGA_CUDA_TRY(cudaMemcpyAsync(gpe_trace, S.rec_gpe.p, sizeof(double) * iters, cudaMemcpyDeviceToHost, s));
    FGA_CUDA_TRY(cudaMemcpyAsync(iv.data(), S.rec_inter.p, sizeof(long long) * iters, cudaMemcpyDeviceToHost, s));
    FGA_CUDA_TRY(cudaMemcpyAsync(vv.data(), S.rec_visits.p, sizeof(long long) * iters, cudaMemcpyDeviceToHost, s));
  }
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  // the last trace entry is the energy of the final positions (registration.py:146-148)
  if (gpe_trace && S.O.trace_gpe && iters > 0) gpe_trace[iters - 1] = S.gpe_final;
  if (inter)
    for (int64_t k = 0; k < iters; k++) inter[k] = iv[k];
  if (visits)
    for (int64_t k = 0; k < iters; k++) visits[k] = vv[k];
  if (out) {
    std::memset(out, 0, sizeof(*out));
    std::memcpy(out->R, st.Racc, sizeof(st.Racc));
    std::memcpy(out->R_norm, st.Racc, sizeof(st.Racc));
    std::memcpy(out->t_norm, st.tacc, sizeof(st.tacc));
    denormalize(st.Racc, st.tacc, S.ctx10, out->t);
    out->iterations = iters;
    out->converged = st.converged;
    out->gpe_initial = S.gpe_initial;
    out->gpe_final = S.gpe_final;
    std::memcpy(out->norm_ctx, S.ctx10, sizeof(S.ctx10));
    for (int64_t k = 0; k < iters; k++) {
      out->interactions += iv[k];
      out->visits += vv[k];
    }
    out->n_nodes = S.direct ? 0 : S.tree.n_nodes;
    cudaEventElapsedTime(&S.setup_ms, c->ev[0], c->ev[1]);
    out->setup_ms = S.setup_ms;
    out->loop_ms = S.loop_ms;
    out->gpe_ms = S.gpe_ms;
  }
  S.active = false;
  return FGA_OK;
}

// ------------------------------------------------------------------ driver
int fga_register(fga_ctx* c, const double* x, int64_t n, const double* y, int64_t m, int dim,
                 const fga_params* params, const fga_options* options, fga_result* out,
                 double* deltas, double* traj, double* gpe_trace, int64_t* inter) {
  CTX_TRY(c);
  TRY(fga_session_begin(c, x, n, y, m, dim, params, options, 0, 1));
  Session& S = c->S;
  cudaStream_t s = c->stream;
  float gpe_ms = 0.f;
  // The initial energy (registration.py:124) only reads the initial template
  // state: it runs on a second stream from a snapshot of that state, next to
  // the iterations (a MUFU-bound pass beside an issue-bound one).
  static const bool async_gpe = [] {
    const char* e = getenv("FGA_ASYNC_GPE");
    return !(e && atoi(e) == 0);
  }();
  const bool gpe_async = S.O.compute_gpe && async_gpe && !S.O.trace_gpe && S.m_local > 0;
  if (gpe_async) {
    if (!c->aux) {
      FGA_CUDA_TRY(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
      for (auto& e : c->aev) FGA_CUDA_TRY(cudaEventCreate(&e));
    }
    const int64_t ml = S.m_local;
    const TemplateView tv = S.view();
    FGA_CUDA_TRY(S.gpe_snap.reserve(sizeof(double) * 4 * ml));
    double* snap = S.gpe_snap.as<double>();
    FGA_CUDA_TRY(cudaMemcpyAsync(snap, tv.px, sizeof(double) * 3 * ml, cudaMemcpyDeviceToDevice, s));
    FGA_CUDA_TRY(cudaMemcpyAsync(snap + 3 * ml, tv.mq, sizeof(double) * ml, cudaMemcpyDeviceToDevice, s));
    const int64_t ngw = gpe_warps(ml, S.ref().n, S.precision);
    FGA_CUDA_TRY(S.gpe_part2.reserve(sizeof(double) * std::max<int64_t>(ngw, 1)));
    FGA_CUDA_TRY(S.gpe_sums2.reserve(sizeof(double) * (kPartialStride + reduce_stage_doubles())));
    FGA_CUDA_TRY(cudaEventRecord(c->aev[0], s));
    FGA_CUDA_TRY(cudaStreamWaitEvent(c->aux, c->aev[0], 0));
    FGA_CUDA_TRY(cudaEventRecord(c->aev[1], c->aux));
    launch_gpe(S.ref(), snap, snap + ml, snap + 2 * ml, snap + 3 * ml, ml, S.sp.eps, nullptr,
               S.gpe_part2.as<double>(), S.precision, c->aux);
    launch_reduce(nullptr, 0, S.gpe_part2.as<double>(), ngw, -1.0, S.gpe_sums2.as<double>(),
                  S.gpe_sums2.as<double>() + kPartialStride, c->aux);
    FGA_CUDA_TRY(cudaGetLastError());
    FGA_CUDA_TRY(cudaEventRecord(c->aev[2], c->aux));
  } else if (S.O.compute_gpe) {
    FGA_CUDA_TRY(cudaEventRecord(c->ev[4], s));
    TRY(session_gpe(c, nullptr));
    FGA_CUDA_TRY(cudaEventRecord(c->ev[5], s));
    TRY(take_gpe(c, &S.gpe_initial));
    S.have_gpe_initial = true;
    cudaEventElapsedTime(&gpe_ms, c->ev[4], c->ev[5]);
  }
  FGA_CUDA_TRY(cudaEventRecord(c->ev[2], s));
  int done = 0;
  int64_t iters = 0;
  while (!done) {
    const int64_t left = S.P.max_iters - S.passes;
    const int k = (int)std::min<int64_t>(S.O.poll_every, std::max<int64_t>(left, 1));
    TRY(fga_session_iterate(c, k));
    TRY(session_poll(c, &done, &iters));
    if (S.passes >= S.P.max_iters) done = 1;
  }
  FGA_CUDA_TRY(cudaEventRecord(c->ev[3], s));
  FGA_CUDA_TRY(cudaEventSynchronize(c->ev[3]));
  cudaEventElapsedTime(&S.loop_ms, c->ev[2], c->ev[3]);
  if (gpe_async) {
    FGA_CUDA_TRY(cudaEventSynchronize(c->aev[2]));
    double v = 0.0;
    FGA_CUDA_TRY(cudaMemcpy(&v, S.gpe_sums2.as<double>() + kGpe, sizeof(double),
                            cudaMemcpyDeviceToHost));
    S.gpe_initial = -S.P.G * v;  // _kernels.py:67
    S.have_gpe_initial = true;
    cudaEventElapsedTime(&gpe_ms, c->aev[1], c->aev[2]);
  }
  TRY(session_apply(c));
  if (S.O.compute_gpe) {
    FGA_CUDA_TRY(cudaEventRecord(c->ev[4], s));
    TRY(session_gpe(c, nullptr));
    FGA_CUDA_TRY(cudaEventRecord(c->ev[5], s));
    TRY(take_gpe(c, &S.gpe_final));
    S.have_gpe_final = true;
    float ms2 = 0.f;
    cudaEventElapsedTime(&ms2, c->ev[4], c->ev[5]);
    gpe_ms += ms2;
  }
  S.gpe_ms = gpe_ms;
  return fga_session_finish(c, out, deltas, traj, gpe_trace, inter, nullptr);
}

// ------------------------------------------------------------------ batched
int fga_register_batch_dev(fga_ctx* c, const double* x_all, const int64_t* x_offsets,
                           const double* y_all, const int64_t* y_offsets, int64_t n_pairs,
                           int nmax, int mmax, int dim, const fga_params* params,
                           const fga_options* options, fga_pair_result* out_dev,
                           double* deltas_dev) {
  CTX_TRY(c);
  TRY(validate(params));
  if (dim != 3) {
    set_error("the B200 path implements D=3 (D=2 is not built yet)");
    return FGA_ERR_UNSUPPORTED;
  }
  if (n_pairs <= 0) return FGA_OK;
  fga_options def{};
  def.normalize = 1;
  def.compute_gpe = 1;
  const fga_options O = options ? *options : def;
  if (O.precision != FGA_PREC_FP32) {
    set_error("fga_register_batch: FP32 force precision only");
    return FGA_ERR_UNSUPPORTED;
  }
  if (params->max_depth > kMaxLevels) {
    set_error("max_depth must be <= 21 on the GPU path");
    return FGA_ERR_UNSUPPORTED;
  }
  nmax = std::max(nmax, 1);
  mmax = std::max(mmax, 1);
  if (nmax > 8192 || mmax > 8192) {
    set_error("fga_register_batch: pairs are limited to 8192 points per cloud");
    return FGA_ERR_UNSUPPORTED;
  }
  const int64_t ncell64 = (int64_t)params->rho * params->rho * params->rho;
  if (ncell64 > 16384) {
    set_error("fga_register_batch: rho^3 must be <= 16384");
    return FGA_ERR_UNSUPPORTED;
  }
  int P = 2048;
  while (P < std::max(nmax, mmax)) P <<= 1;
  const int ncell = (int)ncell64;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const int grid = (int)std::min<int64_t>(n_pairs, sms);
  const size_t cap = (size_t)4 * nmax + 64 * (size_t)params->max_depth;
  const size_t smem = batch_smem_bytes(P, nmax, ncell);
  // per-slot scratch
  const size_t per_slot = sizeof(double) * ((size_t)nmax * 3 + (size_t)mmax * 3 + nmax + mmax) +
                          sizeof(int) * std::max(nmax, mmax) + sizeof(float4) * nmax +
                          cap * (1 + 4 * 3 + 4 * 8 + 8 + 24 + 8 + 16 + 8 + 32 + 16) +
                          sizeof(double) * (size_t)mmax * 7 +
                          sizeof(double) * kPartialStride * (((size_t)mmax + 31) / 32) + 1024;
  FGA_CUDA_TRY(c->batch_scratch.reserve(per_slot * grid + 8192));
  BatchArgs a{};
  char* q = c->batch_scratch.as<char>();
  auto take = [&](size_t bytes) {
    char* r = q;
    q += (bytes + 255) / 256 * 256;
    return r;
  };
  const size_t g = grid;
  a.scratch.xn = (double*)take(sizeof(double) * nmax * 3 * g);
  a.scratch.yn = (double*)take(sizeof(double) * mmax * 3 * g);
  a.scratch.mx = (double*)take(sizeof(double) * nmax * g);
  a.scratch.my = (double*)take(sizeof(double) * mmax * g);
  a.scratch.flat = (int*)take(sizeof(int) * std::max(nmax, mmax) * g);
  a.scratch.ref32 = (float4*)take(sizeof(float4) * nmax * g);
  a.scratch.nlev = (signed char*)take(cap * g);
  a.scratch.nstart = (int*)take(sizeof(int) * cap * g);
  a.scratch.nocc = (int*)take(sizeof(int) * cap * g);
  a.scratch.nskip = (int*)take(sizeof(int) * cap * g);
  a.scratch.nchild = (int*)take(sizeof(int) * 8 * cap * g);
  a.scratch.nmass = (double*)take(sizeof(double) * cap * g);
  a.scratch.nmc = (double*)take(sizeof(double) * 3 * cap * g);
  a.scratch.nlen = (double*)take(sizeof(double) * cap * g);
  a.scratch.ra32 = (float4*)take(sizeof(float4) * cap * g);
  a.scratch.rb32 = (NodeB32*)take(sizeof(NodeB32) * cap * g);
  a.scratch.ra64 = (double4*)take(sizeof(double4) * cap * g);
  a.scratch.rb64 = (NodeB64*)take(sizeof(NodeB64) * cap * g);
  a.scratch.tpl = (double*)take(sizeof(double) * mmax * 7 * g);
  a.scratch.cpart = (double*)take(sizeof(double) * kPartialStride * ((mmax + 31) / 32) * g);
  if ((size_t)(q - c->batch_scratch.as<char>()) > c->batch_scratch.bytes) {
    set_error("internal: batched scratch sizing");
    return FGA_ERR_NOMEM;
  }
  FGA_CUDA_TRY(c->batch_counter.reserve(sizeof(int)));
  FGA_CUDA_TRY(cudaMemsetAsync(c->batch_counter.p, 0, sizeof(int), c->stream));
  a.x = x_all;
  a.y = y_all;
  a.xoff = reinterpret_cast<const long long*>(x_offsets);
  a.yoff = reinterpret_cast<const long long*>(y_offsets);
  a.x_weights = O.x_weights;
  a.y_weights = O.y_weights;
  a.n_pairs = (int)n_pairs;
  a.nmax = nmax;
  a.mmax = mmax;
  a.P = P;
  a.ncell = ncell;
  a.node_cap = cap;
  const double extent = params->norm_b - params->norm_a;
  a.cell_edge = extent / params->rho;
  a.cell_vol = std::pow(a.cell_edge, 3);
  a.theta2 = params->theta * params->theta;
  a.eps2 = params->epsilon * params->epsilon;
  a.theta2f = (float)a.theta2;
  a.eps2f = (float)a.eps2;
  const double r_ball = extent / (2.0 * params->max_depth * params->rho);
  a.ball_vol = (4.0 / 3.0) * M_PI * std::pow(r_ball, 3);
  a.p = *params;
  a.opt = O;
  a.counter = c->batch_counter.as<int>();
  a.out = out_dev;
  a.deltas = deltas_dev;
  a.mode = 0;
  cudaStream_t s = c->stream;
  // Wide mode (enough pairs to fill the GPU): setup per pair in the
  // persistent kernel, then one wide launch per iteration over all active
  // pairs' query chunks, then the finish (fga_batched.cuh BatchWide).
  static const int wide_env = [] {
    const char* e = getenv("FGA_BATCH_WIDE");
    return e ? atoi(e) : -1;
  }();
  const bool use_wide = wide_env >= 0 ? wide_env != 0 : n_pairs >= sms;
  if (!use_wide) return launch_register_batch(a, grid, smem, s);
  (void)0;
  const int chunks = (mmax + 31) / 32;
  const size_t P64 = (size_t)n_pairs;
  const size_t wide_bytes =
      P64 * (cap * (2 * sizeof(float4) + sizeof(double4) + sizeof(NodeB64)) +
             sizeof(double) * (size_t)mmax * 7 + sizeof(float4) * (size_t)nmax +
             sizeof(PairState) + sizeof(double) * kPartialStride * chunks + 2 * sizeof(int)) +
      16 * 256 + 64;
  FGA_CUDA_TRY(c->batch_wide.reserve(wide_bytes));
  q = c->batch_wide.as<char>();
  a.wide.c32 = (float4*)take(2 * sizeof(float4) * cap * P64);
  a.wide.a64 = (double4*)take(sizeof(double4) * cap * P64);
  a.wide.b64 = (NodeB64*)take(sizeof(NodeB64) * cap * P64);
  a.wide.tpl = (double*)take(sizeof(double) * (size_t)mmax * 7 * P64);
  a.wide.ref32 = (float4*)take(sizeof(float4) * (size_t)nmax * P64);
  a.wide.st = (PairState*)take(sizeof(PairState) * P64);
  a.wide.cpart = (double*)take(sizeof(double) * kPartialStride * chunks * P64);
  a.wide.list[0] = (int*)take(sizeof(int) * P64);
  a.wide.list[1] = (int*)take(sizeof(int) * P64);
  a.wide.counts = (int*)take(sizeof(int) * 4);
  a.wide.chunks = chunks;
  if ((size_t)(q - c->batch_wide.as<char>()) > c->batch_wide.bytes) {
    set_error("internal: batched wide sizing");
    return FGA_ERR_NOMEM;
  }
  FGA_CUDA_TRY(cudaMemsetAsync(a.wide.counts, 0, sizeof(int) * 4, s));
  static const bool phase_times = getenv("FGA_BATCH_PHASES") != nullptr;
  cudaEvent_t pe[4];
  if (phase_times)
    for (auto& e : pe) cudaEventCreate(&e);
  if (phase_times) cudaEventRecord(pe[0], s);
  a.mode = 1;
  TRY(launch_register_batch(a, grid, smem, s));
  if (phase_times) cudaEventRecord(pe[1], s);
  int cur = 0;
  static const bool iter_times = phase_times && atoi(getenv("FGA_BATCH_PHASES")) == 2;
  for (int it = 0; it < params->max_iters; it++) {
    cudaEvent_t ie[2];
    if (iter_times) {
      for (auto& e : ie) cudaEventCreate(&e);
      cudaEventRecord(ie[0], s);
    }
    TRY(launch_wide_iteration(a, cur, it, s));
    cur = 1 - cur;
    if (iter_times) {  // (design tool: per-iteration time and active pairs)
      cudaEventRecord(ie[1], s);
      int act = 0;
      cudaMemcpyAsync(&act, a.wide.counts + cur, sizeof(int), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      float ms = 0;
      cudaEventElapsedTime(&ms, ie[0], ie[1]);
      fprintf(stderr, "it %d %.3f ms active-after %d\n", it, ms, act);
      for (auto& e : ie) cudaEventDestroy(e);
    }
    if ((it & 3) == 3 || it + 1 == params->max_iters) {  // stop once every pair is done
      int active = 0;
      FGA_CUDA_TRY(cudaMemcpyAsync(&active, a.wide.counts + cur, sizeof(int),
                                   cudaMemcpyDeviceToHost, s));
      FGA_CUDA_TRY(cudaStreamSynchronize(s));
      if (active == 0) break;
    }
  }
  FGA_CUDA_TRY(cudaMemsetAsync(c->batch_counter.p, 0, sizeof(int), s));
  if (phase_times) cudaEventRecord(pe[2], s);
  a.mode = 2;
  TRY(launch_register_batch(a, grid, smem, s));
  if (phase_times) {  // (design tool: FGA_BATCH_PHASES=1)
    cudaEventRecord(pe[3], s);
    cudaEventSynchronize(pe[3]);
    float t1 = 0, t2 = 0, t3 = 0;
    cudaEventElapsedTime(&t1, pe[0], pe[1]);
    cudaEventElapsedTime(&t2, pe[1], pe[2]);
    cudaEventElapsedTime(&t3, pe[2], pe[3]);
    fprintf(stderr, "batch wide phases: setup %.2f ms, iterations %.2f ms, finish %.2f ms\n", t1,
            t2, t3);
    for (auto& e : pe) cudaEventDestroy(e);
  }
  return FGA_OK;
}

int fga_register_batch(fga_ctx* c, const double* x_all, const int64_t* x_offsets,
                       const double* y_all, const int64_t* y_offsets, int64_t n_pairs, int dim,
                       const fga_params* params, const fga_options* options,
                       fga_pair_result* out, double* deltas) {
  CTX_TRY(c);
  if (n_pairs <= 0) return FGA_OK;
  if (!x_offsets || !y_offsets || !out) return FGA_ERR_INVALID;
  int nmax = 0, mmax = 0;
  for (int64_t p = 0; p < n_pairs; p++) {
    nmax = (int)std::max<int64_t>(nmax, x_offsets[p + 1] - x_offsets[p]);
    mmax = (int)std::max<int64_t>(mmax, y_offsets[p + 1] - y_offsets[p]);
  }
  const int64_t nx = x_offsets[n_pairs], ny = y_offsets[n_pairs];
  cudaStream_t s = c->stream;
  TRY(h2d(c->batch_in[0], x_all, 3 * nx, s));
  TRY(h2d(c->batch_in[1], y_all, 3 * ny, s));
  TRY(h2d(c->batch_in[2], x_offsets, n_pairs + 1, s));
  TRY(h2d(c->batch_in[3], y_offsets, n_pairs + 1, s));
  fga_options O;
  if (options) {
    O = *options;
  } else {
    O = fga_options{};
    O.normalize = 1;
    O.compute_gpe = 1;
  }
  if (O.x_weights) {
    TRY(h2d(c->batch_in[4], O.x_weights, nx, s));
    O.x_weights = c->batch_in[4].as<double>();
  }
  if (O.y_weights) {
    TRY(h2d(c->batch_in[5], O.y_weights, ny, s));
    O.y_weights = c->batch_in[5].as<double>();
  }
  FGA_CUDA_TRY(c->batch_out.reserve(sizeof(fga_pair_result) * n_pairs));
  if (deltas) FGA_CUDA_TRY(c->batch_deltas.reserve(sizeof(double) * n_pairs * params->max_iters));
  TRY(fga_register_batch_dev(c, c->batch_in[0].as<double>(), c->batch_in[2].as<int64_t>(),
                             c->batch_in[1].as<double>(), c->batch_in[3].as<int64_t>(), n_pairs,
                             nmax, mmax, dim, params, &O, c->batch_out.as<fga_pair_result>(),
                             deltas ? c->batch_deltas.as<double>() : nullptr));
  FGA_CUDA_TRY(cudaMemcpyAsync(out, c->batch_out.p, sizeof(fga_pair_result) * n_pairs,
                               cudaMemcpyDeviceToHost, s));
  if (deltas)
    FGA_CUDA_TRY(cudaMemcpyAsync(deltas, c->batch_deltas.p,
                                 sizeof(double) * n_pairs * params->max_iters,
                                 cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  return FGA_OK;
}

}  // extern "C" (C++ helpers of fga_register_batch_list)
namespace fga {
void host_gather_segments(const char* const* src, const int64_t* prefix, int64_t nseg,
                          int64_t lo, int64_t hi, char* dst);
}

namespace {
constexpr int kStageSlots = 4;
constexpr int64_t kStageBytes = 32ll << 20;

// host segments -> one contiguous device buffer through the pinned ring: the
// host threads fill chunk k+1 while the copy engine moves chunk k
int stage_segments_h2d(fga_ctx* c, const char* const* src, const int64_t* prefix, int64_t nseg,
                       char* dst_dev, cudaStream_t s) {
  for (int k = 0; k < kStageSlots; k++) {
    if (!c->stage[k]) {
      FGA_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&c->stage[k]), kStageBytes,
                                 cudaHostAllocDefault));
      FGA_CUDA_TRY(cudaEventCreateWithFlags(&c->stage_ev[k], cudaEventDisableTiming));
      FGA_CUDA_TRY(cudaEventRecord(c->stage_ev[k], s));
    }
  }
  const int64_t total = prefix[nseg];
  int slot = 0;
  for (int64_t lo = 0; lo < total; lo += kStageBytes, slot = (slot + 1) % kStageSlots) {
    const int64_t hi = std::min(total, lo + kStageBytes);
    FGA_CUDA_TRY(cudaEventSynchronize(c->stage_ev[slot]));  // its previous copy is done
    fga::host_gather_segments(src, prefix, nseg, lo, hi, c->stage[slot]);
    FGA_CUDA_TRY(cudaMemcpyAsync(dst_dev + lo, c->stage[slot], (size_t)(hi - lo),
                                 cudaMemcpyHostToDevice, s));
    FGA_CUDA_TRY(cudaEventRecord(c->stage_ev[slot], s));
  }
  return FGA_OK;
}
}  // namespace
extern "C" {

int fga_register_batch_list(fga_ctx* c, const double* const* xs, const int64_t* xn,
                            const double* const* ys, const int64_t* yn, int64_t n_pairs, int dim,
                            const fga_params* params, const fga_options* options,
                            fga_pair_result* out, double* deltas) {
  CTX_TRY(c);
  if (n_pairs <= 0) return FGA_OK;
  if (!xs || !xn || !ys || !yn || !out) return FGA_ERR_INVALID;
  if (options && (options->x_weights || options->y_weights)) {
    set_error("fga_register_batch_list: external weights need fga_register_batch");
    return FGA_ERR_INVALID;
  }
  std::vector<int64_t> xo(n_pairs + 1, 0), yo(n_pairs + 1, 0);
  int nmax = 0, mmax = 0;
  for (int64_t p = 0; p < n_pairs; p++) {
    if (xn[p] < 0 || yn[p] < 0) return FGA_ERR_INVALID;
    xo[p + 1] = xo[p] + xn[p];
    yo[p + 1] = yo[p] + yn[p];
    nmax = (int)std::max<int64_t>(nmax, xn[p]);
    mmax = (int)std::max<int64_t>(mmax, yn[p]);
  }
  // one virtual concatenation: the x clouds, then the y clouds (bytes)
  std::vector<const char*> src(2 * n_pairs);
  std::vector<int64_t> pre(2 * n_pairs + 1, 0);
  for (int64_t p = 0; p < n_pairs; p++) {
    src[p] = reinterpret_cast<const char*>(xs[p]);
    src[n_pairs + p] = reinterpret_cast<const char*>(ys[p]);
  }
  for (int64_t k = 0; k < 2 * n_pairs; k++)
    pre[k + 1] = pre[k] + 3 * (int64_t)sizeof(double) * (k < n_pairs ? xn[k] : yn[k - n_pairs]);
  const int64_t nx = xo[n_pairs], ny = yo[n_pairs];
  cudaStream_t s = c->stream;
  FGA_CUDA_TRY(c->batch_in[0].reserve(sizeof(double) * 3 * (nx + ny)));
  TRY(stage_segments_h2d(c, src.data(), pre.data(), 2 * n_pairs, c->batch_in[0].as<char>(), s));
  TRY(h2d(c->batch_in[2], xo.data(), n_pairs + 1, s));
  TRY(h2d(c->batch_in[3], yo.data(), n_pairs + 1, s));
  fga_options O;
  if (options) {
    O = *options;
  } else {
    O = fga_options{};
    O.normalize = 1;
    O.compute_gpe = 1;
  }
  FGA_CUDA_TRY(c->batch_out.reserve(sizeof(fga_pair_result) * n_pairs));
  if (deltas) FGA_CUDA_TRY(c->batch_deltas.reserve(sizeof(double) * n_pairs * params->max_iters));
  const double* X = c->batch_in[0].as<double>();
  TRY(fga_register_batch_dev(c, X, c->batch_in[2].as<int64_t>(), X + 3 * nx,
                             c->batch_in[3].as<int64_t>(), n_pairs, nmax, mmax, dim, params, &O,
                             c->batch_out.as<fga_pair_result>(),
                             deltas ? c->batch_deltas.as<double>() : nullptr));
  FGA_CUDA_TRY(cudaMemcpyAsync(out, c->batch_out.p, sizeof(fga_pair_result) * n_pairs,
                               cudaMemcpyDeviceToHost, s));
  if (deltas)
    FGA_CUDA_TRY(cudaMemcpyAsync(deltas, c->batch_deltas.p,
                                 sizeof(double) * n_pairs * params->max_iters,
                                 cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  return FGA_OK;
}

// ------------------------------------------------------------------ tree ops
int fga_tree_build(fga_ctx* c, const double* pts, const double* masses, int64_t n, int dim,
                   int max_depth, int64_t* n_nodes) {
  CTX_TRY(c);
  TRY(check_dim(dim));
  if (n <= 0) {
    set_error("registration requires a non-empty cloud");
    return FGA_ERR_EMPTY;
  }
  const Pad3 pp = pad3(pts, n, dim);
  TRY(h2d(c->tree_pts, pp.ptr, 3 * n, c->stream));
  TRY(h2d(c->tree_masses, masses, n, c->stream));
  TRY(tree_build_dev(c->tree, c->tree_pts.as<double>(), c->tree_masses.as<double>(), n, max_depth,
                     c->stream));
  FGA_CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (c->tree.cap_runs) {  // the exported arrays would lack the chains below level 21
    set_error("max_depth > 42 with two reference points in one cell of level 42 (the GPU "
              "tree has at most 42 levels)");
    return FGA_ERR_UNSUPPORTED;
  }
  c->tree.dim = dim;
  if (n_nodes) *n_nodes = c->tree.n_nodes;
  return FGA_OK;
}

int fga_tree_build_dev(fga_ctx* c, const double* pts_dev, const double* masses_dev, int64_t n,
                       int max_depth, int64_t* n_nodes) {
  CTX_TRY(c);
  if (n <= 0) {
    set_error("registration requires a non-empty cloud");
    return FGA_ERR_EMPTY;
  }
  TRY(tree_build_dev(c->tree, pts_dev, masses_dev, n, max_depth, c->stream));
  c->tree.dim = 3;
  if (c->tree.cap_runs) {
    set_error("max_depth > 42 with two reference points in one cell of level 42 (the GPU "
              "tree has at most 42 levels)");
    return FGA_ERR_UNSUPPORTED;
  }
  if (n_nodes) *n_nodes = c->tree.n_nodes;
  return FGA_OK;
}

int fga_tree_export(fga_ctx* c, int64_t* children, double* com, double* mass, double* length,
                    int64_t* occupancy, int64_t* depth, double* bbox_min, double* bbox_max) {
  CTX_TRY(c);
  TreeDev& T = c->tree;
  if (T.dim == 3)
    return tree_export_host(T, c->stream, children, com, mass, length, occupancy, depth, bbox_min,
                            bbox_max);
  // D = 2: the z bit of every child slot is 1 (z = 0 >= centre 0), so the
  // quadtree slot is slot3 >> 1; drop the z column of com / bbox.
  const int64_t nn = T.n_nodes;
  std::vector<int64_t> ch(children ? nn * 8 : 0);
  std::vector<double> cm(com ? nn * 3 : 0), bl(bbox_min ? nn * 3 : 0), bh(bbox_max ? nn * 3 : 0);
  TRY(tree_export_host(T, c->stream, children ? ch.data() : nullptr, com ? cm.data() : nullptr,
                       mass, length, occupancy, depth, bbox_min ? bl.data() : nullptr,
                       bbox_max ? bh.data() : nullptr));
  if (children)
    for (int64_t x = 0; x < nn; x++)
      for (int q = 0; q < 4; q++) children[x * 4 + q] = ch[x * 8 + 2 * q + 1];
  if (com) unpad3(cm.data(), nn, 2, com);
  if (bbox_min) unpad3(bl.data(), nn, 2, bbox_min);
  if (bbox_max) unpad3(bh.data(), nn, 2, bbox_max);
  return FGA_OK;
}

int fga_tree_upload(fga_ctx* c, const int64_t* children, const double* com, const double* mass,
                    const double* length, int64_t n_nodes, int n_child, int dim) {
  CTX_TRY(c);
  TRY(check_dim(dim));
  if (n_child != (1 << dim)) {
    set_error("tree upload: children must have 2^dim slots");
    return FGA_ERR_INVALID;
  }
  if (dim == 3) {
    c->tree.dim = 3;
    return tree_upload_host(c->tree, children, com, mass, length, n_nodes, 8, c->stream);
  }
  std::vector<int64_t> ch((size_t)std::max<int64_t>(n_nodes, 0) * 8, -1);
  for (int64_t x = 0; x < n_nodes; x++)
    for (int q = 0; q < 4; q++) ch[x * 8 + 2 * q + 1] = children[x * 4 + q];
  const Pad3 pc = pad3(com, n_nodes, 2);
  TRY(tree_upload_host(c->tree, ch.data(), pc.ptr, mass, length, n_nodes, 8, c->stream));
  c->tree.dim = 2;
  return FGA_OK;
}

int fga_tree_forces(fga_ctx* c, const double* queries, const double* qm, int64_t m, double theta,
                    double G, double eps2, int precision, double* forces, int64_t* visits,
                    int64_t* accepted) {
  CTX_TRY(c);
  if (c->tree.n_nodes <= 0) {
    set_error("no tree in this context (fga_tree_build / fga_tree_upload first)");
    return FGA_ERR_STATE;
  }
  if (m <= 0) return FGA_OK;
  const int dim = c->tree.dim;
  cudaStream_t s = c->stream;
  DevBuf &q = c->op[0], &qmd = c->op[1], &soa = c->op[2], &out = c->op[3];
  DevBuf &kin = c->op[4], &kout = c->op[5], &iin = c->op[6], &iout = c->op[7];
  const Pad3 pq = pad3(queries, m, dim);
  TRY(h2d(q, pq.ptr, 3 * m, s));
  TRY(h2d(qmd, qm, m, s));
  DevBuf& tmp = c->S.cub_tmp;
  DevBuf& scratch = c->S.scratch;
  TRY(morton_order(q.as<double>(), m, kin, kout, iin, iout, tmp, scratch, s));
  FGA_CUDA_TRY(soa.reserve(sizeof(double) * 4 * m));
  double* b = soa.as<double>();
  launch_gather_queries(q.as<double>(), qmd.as<double>(), iout.as<int>(), m, b, b + m, b + 2 * m,
                        b + 3 * m, s);
  FGA_CUDA_TRY(out.reserve(sizeof(double) * 5 * m));
  double* f = out.as<double>();
  long long* vis = reinterpret_cast<long long*>(f + 3 * m);
  long long* acc = vis + m;
  FGA_CUDA_TRY(c->op_total.reserve(sizeof(unsigned long long)));
  FGA_CUDA_TRY(cudaMemsetAsync(c->op_total.p, 0, sizeof(unsigned long long), s));
  // one-wave FP32 calls: split passes from the previous call's trace (the
  // first call over a tree / query count / theta records it, and its max and
  // mean warp steps decide whether later calls split, as the session does)
  OpSplitBufs ob{0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  fga_ctx::OpSplitKey& ok = c->op_split;
  unsigned long long* stats = nullptr;
  if (precision == FGA_PREC_FP32 && bh_operator_split_possible(m)) {
    const bool same = ok.traced && ok.generation == c->tree.generation && ok.m == m &&
                      ok.theta == theta && ok.eps2 == eps2;
    const int64_t nw = bh_operator_warps(m);
    if (!same) {
      ok.traced = false;
      FGA_CUDA_TRY(c->op_trace.reserve(sizeof(int) * kTraceLen * nw +
                                       2 * sizeof(unsigned long long) + 8));
      ob.mode = 1;
    } else if (ok.split) {
      const int64_t P = bh_split_parts();
      FGA_CUDA_TRY(c->op_fpart.reserve(sizeof(double) * 3 * P * m));
      FGA_CUDA_TRY(
          c->op_cnt.reserve(sizeof(int) * (2 * P * m + kTraceLen * P * ((m + 31) / 32))));
      ob.mode = 2;
      ob.fpart = c->op_fpart.as<double>();
      ob.vpart = c->op_cnt.as<int>();
      ob.apart = ob.vpart + P * m;
      ob.ptrace = ob.apart + P * m;
    }
    if (ob.mode) {
      ob.trace = c->op_trace.as<int>();
      // (8-byte aligned: kTraceLen nw ints rounded up)
      const size_t off = (sizeof(int) * kTraceLen * nw + 7) & ~size_t(7);
      stats = reinterpret_cast<unsigned long long*>(c->op_trace.as<char>() + off);
      ob.stats = stats;
    }
  }
  // Pinned (device-mapped) host outputs: the kernel stores each query's
  // results straight into them, so the device->host transfer overlaps the
  // traversal instead of following it
  // (measured on the 1M drop-in: 14.00 -> 13.83 ms; FGA_ZERO_COPY=0 turns it off).
  // Not for split passes: their epilogue would scatter every query's results
  // over PCIe at the end of the call (125k queries: ~1.1 ms against a 4 MB copy)
  static const bool zc_on = !(getenv("FGA_ZERO_COPY") && atoi(getenv("FGA_ZERO_COPY")) == 0);
  double* fz = nullptr;
  long long* vz = nullptr;
  if (zc_on && dim == 3 && ob.mode != 2) {
    auto mapped = [](void* h) -> void* {
      cudaPointerAttributes a{};
      if (!h || cudaPointerGetAttributes(&a, h) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
    };
    fz = static_cast<double*>(mapped(forces));
    vz = visits ? static_cast<long long*>(mapped(visits)) : nullptr;
    if (!fz || (visits && !vz)) fz = nullptr, vz = nullptr;
  }
  launch_bh_operator(c->tree, b, b + m, b + 2 * m, b + 3 * m, iout.as<int>(), m, theta, G, eps2,
                     fz ? fz : f, fz ? vz : (visits ? vis : nullptr), accepted ? acc : nullptr,
                     c->op_total.as<unsigned long long>(), precision, s, ob.mode ? &ob : nullptr);
  FGA_CUDA_TRY(cudaGetLastError());
  std::vector<double> f3(dim == 3 ? 0 : 3 * m);
  if (!fz) {
    FGA_CUDA_TRY(cudaMemcpyAsync(dim == 3 ? forces : f3.data(), f, sizeof(double) * 3 * m,
                                 cudaMemcpyDeviceToHost, s));
    if (visits)
      FGA_CUDA_TRY(cudaMemcpyAsync(visits, vis, sizeof(long long) * m, cudaMemcpyDeviceToHost, s));
  }
  if (accepted) FGA_CUDA_TRY(cudaMemcpyAsync(accepted, acc, sizeof(long long) * m, cudaMemcpyDeviceToHost, s));
  unsigned long long total = 0, st2[2] = {0, 0};
  FGA_CUDA_TRY(cudaMemcpyAsync(&total, c->op_total.p, sizeof(total), cudaMemcpyDeviceToHost, s));
  if (ob.mode)
    FGA_CUDA_TRY(cudaMemcpyAsync(st2, stats, sizeof(st2), cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  c->last_interactions = (int64_t)total;
  static const bool split_log = getenv("FGA_SPLIT_LOG") != nullptr;  // (tests)
  if (ob.mode == 1) {
    ok.generation = c->tree.generation;
    ok.m = m;
    ok.theta = theta;
    ok.eps2 = eps2;
    ok.max_steps = st2[0];
    ok.part_max = 0;
    ok.split = bh_operator_split_wanted(m, st2[0], st2[1]);
    ok.traced = true;
    if (split_log)
      fprintf(stderr, "[fga] operator trace: %lld queries, max %llu sum %llu -> %s\n",
              (long long)m, st2[0], st2[1], ok.split ? "split" : "unsplit");
  } else if (ob.mode == 2) {
    // the trace no longer balances these queries (another query set of the
    // same size, or the template moved far): the heaviest part's steps grew
    // past FGA_SPLIT_STALE x those of the first split call after the trace
    // (a stale trace measured 3.6-4x) -> record a new one next call
    static const double stale = getenv("FGA_SPLIT_STALE") ? atof(getenv("FGA_SPLIT_STALE")) : 2.0;
    if (!ok.part_max)
      ok.part_max = std::max<unsigned long long>(1, st2[0]);
    else if ((double)st2[0] > stale * (double)ok.part_max)
      ok.traced = false;
    if (split_log)
      fprintf(stderr, "[fga] operator split: %lld queries, part max %llu (trace max %llu)%s\n",
              (long long)m, st2[0], ok.max_steps, ok.traced ? "" : " -> retrace");
  }
  if (dim != 3) unpad3(f3.data(), m, dim, forces);
  return FGA_OK;
}

namespace {
// FNV-1a over ~4k evenly spaced 8-byte words of each array plus its last word
// (~0.1 ms for a 1M-point tree): detects a different tree at a recycled
// address; in-place edits of an uploaded tree are not supported (the
// reference's BHTree is immutable, bhtree.py:14-45).
uint64_t sampled_hash(uint64_t h, const void* base, int64_t words) {
  const uint64_t* w = static_cast<const uint64_t*>(base);
  if (!w || words <= 0) return h;
  const int64_t step = std::max<int64_t>(1, words / 4096);
  auto mix = [&](uint64_t v) {
    for (int b = 0; b < 8; b++) {
      h ^= (v >> (8 * b)) & 0xff;
      h *= 1099511628211ull;
    }
  };
  for (int64_t i = 0; i < words; i += step) mix(w[i]);
  mix(w[words - 1]);
  return h;
}
}  // namespace

int fga_last_interactions(fga_ctx* c, int64_t* accepted_total) {
  CTX_TRY(c);
  if (accepted_total) *accepted_total = c->last_interactions;
  return FGA_OK;
}

int fga_tree_generation(fga_ctx* c, int64_t* generation) {
  CTX_TRY(c);
  if (generation) *generation = (int64_t)c->tree.generation;
  return FGA_OK;
}

int fga_bh_forces_kernel(fga_ctx* c, const int64_t* children, const double* com,
                         const double* mass, const double* length, int64_t n_nodes, int n_child,
                         const double* queries, const double* qm, int64_t m, int dim,
                         double theta, double G, double eps2, int64_t stack_cap, double* forces,
                         int64_t* visits) {
  (void)stack_cap;  // the stackless traversal needs no stack
  CTX_TRY(c);
  uint64_t h = 1469598103934665603ull;
  h = sampled_hash(h, children, n_nodes * n_child);
  h = sampled_hash(h, com, n_nodes * dim);
  h = sampled_hash(h, mass, n_nodes);
  h = sampled_hash(h, length, n_nodes);
  fga_ctx::ShimKey& k = c->shim;
  const bool hit = k.valid && k.generation == c->tree.generation && k.p[0] == children &&
                   k.p[1] == com && k.p[2] == mass && k.p[3] == length && k.n_nodes == n_nodes &&
                   k.n_child == n_child && k.dim == dim && k.hash == h;
  if (!hit) {
    k.valid = false;
    TRY(fga_tree_upload(c, children, com, mass, length, n_nodes, n_child, dim));
    k.p[0] = children;
    k.p[1] = com;
    k.p[2] = mass;
    k.p[3] = length;
    k.n_nodes = n_nodes;
    k.n_child = n_child;
    k.dim = dim;
    k.hash = h;
    k.generation = c->tree.generation;
    k.valid = true;
  }
  return fga_tree_forces(c, queries, qm, m, theta, G, eps2, FGA_PREC_FP64, forces, visits, nullptr);
}

int fga_direct_forces(fga_ctx* c, const double* ref, const double* rm, int64_t n,
                      const double* queries, const double* qm, int64_t m, int dim, double G,
                      double eps, int precision, double* forces) {
  CTX_TRY(c);
  TRY(check_dim(dim));
  if (n <= 0) {
    set_error("registration requires a non-empty cloud");
    return FGA_ERR_EMPTY;
  }
  if (m <= 0) return FGA_OK;
  cudaStream_t s = c->stream;
  DevBuf &r = c->op[0], &rmd = c->op[1], &pk = c->op[2], &q = c->op[3], &qmd = c->op[4],
         &soa = c->op[5], &out = c->op[6];
  const Pad3 pr = pad3(ref, n, dim), pq = pad3(queries, m, dim);
  TRY(h2d(r, pr.ptr, 3 * n, s));
  TRY(h2d(rmd, rm, n, s));
  FGA_CUDA_TRY(pk.reserve(precision ? sizeof(double4) * n : sizeof(float4) * n));
  launch_pack_ref(r.as<double>(), rmd.as<double>(), n, precision ? nullptr : pk.as<float4>(),
                  precision ? pk.as<double4>() : nullptr, s);
  TRY(h2d(q, pq.ptr, 3 * m, s));
  TRY(h2d(qmd, qm, m, s));
  FGA_CUDA_TRY(soa.reserve(sizeof(double) * 4 * m));
  double* b = soa.as<double>();
  launch_gather_queries(q.as<double>(), qmd.as<double>(), nullptr, m, b, b + m, b + 2 * m, b + 3 * m, s);
  FGA_CUDA_TRY(out.reserve(sizeof(double) * 3 * m));
  RefPoints rp{precision ? nullptr : pk.as<float4>(), precision ? pk.as<double4>() : nullptr, n};
  launch_direct_operator(rp, b, b + m, b + 2 * m, b + 3 * m, m, G, eps, out.as<double>(), precision, s);
  FGA_CUDA_TRY(cudaGetLastError());
  std::vector<double> f3(dim == 3 ? 0 : 3 * m);
  FGA_CUDA_TRY(cudaMemcpyAsync(dim == 3 ? forces : f3.data(), out.p, sizeof(double) * 3 * m,
                               cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  if (dim != 3) unpad3(f3.data(), m, dim, forces);
  return FGA_OK;
}

int fga_gpe_kernel(fga_ctx* c, const double* pos_y, const double* mass_y, int64_t m,
                   const double* pos_x, const double* mass_x, int64_t n, int dim, double G,
                   double eps, int precision, double* value) {
  CTX_TRY(c);
  TRY(check_dim(dim));
  if (!value) return FGA_ERR_INVALID;
  cudaStream_t s = c->stream;
  if (m <= 0 || n <= 0) {
    *value = -G * 0.0;
    return FGA_OK;
  }
  DevBuf &r = c->op[0], &rmd = c->op[1], &pk = c->op[2], &q = c->op[3], &qmd = c->op[4],
         &soa = c->op[5], &part = c->op[6], &sums = c->op[7];
  const Pad3 pr = pad3(pos_x, n, dim), pq = pad3(pos_y, m, dim);
  TRY(h2d(r, pr.ptr, 3 * n, s));
  TRY(h2d(rmd, mass_x, n, s));
  FGA_CUDA_TRY(pk.reserve(precision ? sizeof(double4) * n : sizeof(float4) * n));
  launch_pack_ref(r.as<double>(), rmd.as<double>(), n, precision ? nullptr : pk.as<float4>(),
                  precision ? pk.as<double4>() : nullptr, s);
  TRY(h2d(q, pq.ptr, 3 * m, s));
  TRY(h2d(qmd, mass_y, m, s));
  FGA_CUDA_TRY(soa.reserve(sizeof(double) * 4 * m));
  double* b = soa.as<double>();
  launch_gather_queries(q.as<double>(), qmd.as<double>(), nullptr, m, b, b + m, b + 2 * m, b + 3 * m, s);
  const int64_t ngw = gpe_warps(m, n, precision);
  FGA_CUDA_TRY(part.reserve(sizeof(double) * ngw));
  FGA_CUDA_TRY(sums.reserve(sizeof(double) * (kPartialStride + reduce_stage_doubles())));
  RefPoints rp{precision ? nullptr : pk.as<float4>(), precision ? pk.as<double4>() : nullptr, n};
  launch_gpe(rp, b, b + m, b + 2 * m, b + 3 * m, m, eps, nullptr, part.as<double>(), precision, s);
  launch_reduce(nullptr, 0, part.as<double>(), ngw, -1.0, sums.as<double>(),
                sums.as<double>() + kPartialStride, s);
  FGA_CUDA_TRY(cudaGetLastError());
  double v = 0.0;
  FGA_CUDA_TRY(cudaMemcpyAsync(&v, sums.as<double>() + kGpe, sizeof(double), cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  *value = -G * v;
  return FGA_OK;
}

int fga_knn(fga_ctx* c, const double* pts, int64_t n, int dim, int k, int64_t* idx, double* d2) {
  CTX_TRY(c);
  TRY(check_dim(dim));
  if (n <= 0) return FGA_OK;
  cudaStream_t s = c->stream;
  DevBuf &p = c->op[0], &oi = c->op[1], &od = c->op[2], &sc = c->op[3], &tmp = c->op[4];
  const Pad3 pp = pad3(pts, n, dim);
  TRY(h2d(p, pp.ptr, 3 * n, s));
  FGA_CUDA_TRY(oi.reserve(sizeof(long long) * n * std::max(k, 1)));
  FGA_CUDA_TRY(od.reserve(sizeof(double) * n * std::max(k, 1)));
  TRY(knn_dev(p.as<double>(), n, dim, k, idx ? oi.as<long long>() : nullptr,
              d2 ? od.as<double>() : nullptr, nullptr, sc, tmp, s));
  if (idx) FGA_CUDA_TRY(cudaMemcpyAsync(idx, oi.p, sizeof(long long) * n * k, cudaMemcpyDeviceToHost, s));
  if (d2) FGA_CUDA_TRY(cudaMemcpyAsync(d2, od.p, sizeof(double) * n * k, cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  return FGA_OK;
}

int fga_knn_masses(fga_ctx* c, const double* pts, int64_t n, int dim, int k, double* out) {
  CTX_TRY(c);
  TRY(check_dim(dim));
  if (n <= 0) return FGA_OK;
  cudaStream_t s = c->stream;
  DevBuf &p = c->op[0], &o = c->op[1], &sc = c->op[3], &tmp = c->op[4];
  const Pad3 pp = pad3(pts, n, dim);
  TRY(h2d(p, pp.ptr, 3 * n, s));
  FGA_CUDA_TRY(o.reserve(sizeof(double) * n));
  TRY(knn_dev(p.as<double>(), n, dim, k, nullptr, nullptr, o.as<double>(), sc, tmp, s));
  FGA_CUDA_TRY(cudaMemcpyAsync(out, o.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  return FGA_OK;
}

int fga_rbf_masses(fga_ctx* c, const double* pts, int64_t n, int dim, const int64_t* anchors,
                   int m, double sigma, double* out) {
  CTX_TRY(c);
  TRY(check_dim(dim));
  if (!(sigma > 0)) return invalid("sigma", sigma);
  if (n <= 0) return FGA_OK;
  for (int j = 0; j < m; j++)
    if (anchors[j] < 0 || anchors[j] >= n) {
      set_error("invalid parameter anchors=index out of range");
      return FGA_ERR_INVALID;
    }
  cudaStream_t s = c->stream;
  DevBuf &p = c->op[0], &o = c->op[1], &ix = c->op[2], &sc = c->op[3];
  const Pad3 pp = pad3(pts, n, dim);
  TRY(h2d(p, pp.ptr, 3 * n, s));
  if (m > 0) TRY(h2d(ix, reinterpret_cast<const long long*>(anchors), m, s));
  else FGA_CUDA_TRY(ix.reserve(sizeof(long long)));
  FGA_CUDA_TRY(o.reserve(sizeof(double) * n));
  TRY(rbf_apply_dev(p.as<double>(), n, ix.as<long long>(), m, sigma, 0, o.as<double>(), sc, s));
  FGA_CUDA_TRY(cudaMemcpyAsync(out, o.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  return FGA_OK;
}

int fga_niv_masses(fga_ctx* c, const double* pts, int64_t n, int dim, int rho, double a, double b,
                   int max_depth, double* out) {
  CTX_TRY(c);
  TRY(check_dim(dim));
  if (rho < 2) return invalid("rho", rho);
  if (n <= 0) return FGA_OK;
  cudaStream_t s = c->stream;
  DevBuf &p = c->op[0], &o = c->op[1], &flat = c->op[2], &cnt = c->op[3], &cells = c->op[4];
  const Pad3 pp = pad3(pts, n, dim);
  TRY(h2d(p, pp.ptr, 3 * n, s));
  const int64_t ncell = (int64_t)rho * rho * (dim == 3 ? rho : 1);
  FGA_CUDA_TRY(o.reserve(sizeof(double) * n));
  FGA_CUDA_TRY(flat.reserve(sizeof(int) * n));
  FGA_CUDA_TRY(cnt.reserve(sizeof(long long) * (ncell + 1)));
  FGA_CUDA_TRY(cells.reserve(sizeof(double) * ncell));
  TRY(niv_masses_dev(p.as<double>(), n, dim, rho, a, b, max_depth, o.as<double>(),
                     flat.as<int>(), cnt.as<long long>(), cells.as<double>(), s));
  FGA_CUDA_TRY(cudaMemcpyAsync(out, o.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  return FGA_OK;
}

int fga_normalize_pair(fga_ctx* c, const double* x, int64_t n, const double* y, int64_t m, int dim,
                       double a, double b, double* xn, double* yn, double* ctx10) {
  CTX_TRY(c);
  TRY(check_dim(dim));
  if (n <= 0 || m <= 0) {
    set_error("registration requires a non-empty cloud");
    return FGA_ERR_EMPTY;
  }
  cudaStream_t s = c->stream;
  DevBuf &dx = c->op[0], &dy = c->op[1], &ox = c->op[2], &oy = c->op[3], &cd = c->op[4],
         &sc = c->op[5];
  const Pad3 px = pad3(x, n, dim), py = pad3(y, m, dim);
  TRY(h2d(dx, px.ptr, 3 * n, s));
  TRY(h2d(dy, py.ptr, 3 * m, s));
  FGA_CUDA_TRY(ox.reserve(sizeof(double) * 3 * n));
  FGA_CUDA_TRY(oy.reserve(sizeof(double) * 3 * m));
  FGA_CUDA_TRY(cd.reserve(sizeof(double) * 16));
  FGA_CUDA_TRY(sc.reserve(sizeof(double) * 8192));
  double host_ctx[10];
  TRY(normalize_pair_dev(dx.as<double>(), n, dy.as<double>(), m, a, b, ox.as<double>(),
                         oy.as<double>(), cd.as<double>(), sc.as<double>(), sc.bytes, host_ctx, s));
  std::vector<double> hx(3 * n), hy(3 * m);
  FGA_CUDA_TRY(cudaMemcpyAsync(hx.data(), ox.p, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaMemcpyAsync(hy.data(), oy.p, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  unpad3(hx.data(), n, dim, xn);
  unpad3(hy.data(), m, dim, yn);
  if (ctx10) std::memcpy(ctx10, host_ctx, sizeof(host_ctx));
  return FGA_OK;
}

int fga_solve_rigid(fga_ctx* c, const double* y, const double* yd, int64_t m, int dim, double* R,
                    double* t, int32_t* degenerate) {
  CTX_TRY(c);
  TRY(check_dim(dim));
  if (m <= 0) {
    set_error("registration requires a non-empty cloud");
    return FGA_ERR_EMPTY;
  }
  cudaStream_t s = c->stream;
  DevBuf &dy = c->op[0], &dd = c->op[1], &o = c->op[2];
  const Pad3 py = pad3(y, m, dim), pd = pad3(yd, m, dim);
  TRY(h2d(dy, py.ptr, 3 * m, s));
  TRY(h2d(dd, pd.ptr, 3 * m, s));
  FGA_CUDA_TRY(o.reserve(sizeof(double) * 16));
  launch_solve_rigid(dy.as<double>(), dd.as<double>(), m, dim, o.as<double>(), s);
  FGA_CUDA_TRY(cudaGetLastError());
  double h[13];
  FGA_CUDA_TRY(cudaMemcpyAsync(h, o.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  FGA_CUDA_TRY(cudaStreamSynchronize(s));
  if (R)
    for (int i = 0; i < dim; i++)
      for (int j = 0; j < dim; j++) R[i * dim + j] = h[i * 3 + j];
  if (t)
    for (int i = 0; i < dim; i++) t[i] = h[9 + i];
  if (degenerate) *degenerate = (int32_t)h[12];
  return FGA_OK;
}

}  // extern "C"
