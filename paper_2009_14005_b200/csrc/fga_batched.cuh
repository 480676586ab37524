// fga_batched.cuh -- arguments of the persistent many-pair kernel (batched.cu)
#pragma once
#include "../../include/fga.h"
#include "fga_internal.cuh"

namespace fga {

// Per-CTA-slot global scratch (slot stride = the *max sizes below).
struct BatchScratch {
  double *xn, *yn, *mx, *my;
  int* flat;
  float4* ref32;
  signed char* nlev;
  int *nstart, *nocc, *nskip, *nchild;
  double *nmass, *nmc, *nlen;
  float4* ra32;
  NodeB32* rb32;
  double4* ra64;
  NodeB64* rb64;
  double* tpl;
  double* cpart;  // per 32-query chunk: kPartialStride moment sums
};

// Per-pair state of one registration in the batch (device).
struct PairState {
  double R[9], t[3], Racc[9], tacc[3], shift[3];
  double ctx[10];
  double gpe_initial, gpe_final;
  long long iter, interactions, n_nodes;
  int done, converged, status;
  int n, m, pad;
  double box[6];
  double sum_mx, max_my;
  float cmag;
};

// "Wide" batch mode (many pairs): the setup (normalize, masses, tree,
// template order, initial energy) and the finish (final energy, results) run
// in the persistent kernel, one CTA per pair at a time, while the iterations
// run as one wide launch per iteration over the 32-query chunks of ALL
// active pairs (k_wide_forces) plus a per-pair update (k_wide_update), so a
// pair's iterations are spread over the whole GPU instead of one SM.  The
// per-pair records, template state and PairState persist between launches.
struct BatchWide {
  float4* c32;      // n_pairs * node_cap * 2: {com, mass}, {l2 | -inf, skip, len, 0}
  double4* a64;     // n_pairs * node_cap
  NodeB64* b64;     // n_pairs * node_cap
  double* tpl;      // n_pairs * mmax * 7 (px py pz vx vy vz m, Hilbert order)
  float4* ref32;    // n_pairs * nmax (energy)
  PairState* st;    // n_pairs
  double* cpart;    // n_pairs * chunks * kPartialStride
  int* list[2];     // active pair lists (ping-pong)
  int* counts;      // [0], [1]: list sizes; [2]: chunk work counter
  int chunks;       // 32-query chunks per pair = ceil(mmax / 32)
};

struct BatchArgs {
  const double* x;            // concatenated reference clouds (sum n, 3)
  const double* y;            // concatenated template clouds
  const long long* xoff;      // P+1
  const long long* yoff;      // P+1
  const double* x_weights;    // optional, concatenated like x
  const double* y_weights;
  int n_pairs;
  int nmax, mmax;             // max cloud sizes in the batch
  int P;                      // sort length: next pow2 >= max(nmax, mmax)
  int ncell;                  // rho^3
  size_t node_cap;            // node capacity per slot
  double cell_edge, cell_vol, ball_vol;
  // theta^2 and eps^2, precomputed: the traversal loop re-reads them from the
  // constant bank every step (register-bound at 1024 threads)
  double theta2, eps2;
  float theta2f, eps2f;
  fga_params p;
  fga_options opt;
  BatchScratch scratch;
  int* counter;               // pair work counter (zeroed before launch)
  fga_pair_result* out;       // device, n_pairs
  double* deltas;             // device, n_pairs * max_iters (optional)
  int mode;                   // 0: whole registration per pair; 1: wide setup; 2: wide finish
  BatchWide wide;
};

size_t batch_smem_bytes(int P, int nmax, int ncell);
int launch_register_batch(const BatchArgs& a, int grid, size_t smem, cudaStream_t s);
// one wide iteration over the active pairs (list `cur`, next list `1 - cur`)
int launch_wide_iteration(const BatchArgs& a, int cur, int it, cudaStream_t s);

}  // namespace fga
