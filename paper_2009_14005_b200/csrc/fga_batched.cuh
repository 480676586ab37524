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
};

size_t batch_smem_bytes(int P, int nmax, int ncell);
int launch_register_batch(const BatchArgs& a, int grid, size_t smem, cudaStream_t s);

}  // namespace fga
