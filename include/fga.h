/*
 * fga.h -- C ABI of libfga, the B200 (sm_100a) implementation of the Fast
 * Gravitational Approach (FGA, arXiv 2009.14005) per-iteration hot path.
 *
 * Plain pointers and sizes only; no torch or CUDA types in any signature
 * (streams are passed as void*).  All functions return FGA_OK (0) or a negative
 * FGA_ERR_* code; fga_last_error() gives a thread-local message.  A context
 * (fga_ctx) owns device memory and is bound to one CUDA device and one stream;
 * it is not re-entrant (one context per thread/device).
 *
 * Each entry point names the reference interface it replaces (paths are
 * under the reference package gravreg 0.1.0, pkg/src/gravreg/).
 *
 * Pointer conventions: functions without a `_dev` suffix take HOST arrays in
 * the reference's numpy layouts (C-contiguous float64 (n,3) points, int64
 * indices with -1 = absent) and copy in/out themselves.  `_dev` functions take
 * device pointers and are stream-ordered on the context's stream.
 */
#ifndef FGA_H_
#define FGA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FGA_OK 0
#define FGA_ERR_INVALID (-1)     /* invalid argument (maps to InvalidParam)      */
#define FGA_ERR_CUDA (-2)        /* CUDA runtime failure                         */
#define FGA_ERR_NOMEM (-3)       /* allocation failure                           */
#define FGA_ERR_UNSUPPORTED (-4) /* valid for the reference, not built here yet  */
#define FGA_ERR_EMPTY (-5)       /* EmptyCloud                                   */
#define FGA_ERR_DEGENERATE (-6)  /* DegenerateExtent                             */
#define FGA_ERR_NONFINITE (-7)   /* NonFiniteWeight                              */
#define FGA_ERR_LENGTH (-8)      /* LengthMismatch                               */
#define FGA_ERR_STATE (-9)       /* call order (e.g. no tree built yet)          */
#define FGA_ERR_SINGULAR (-10)   /* SingularCollocation (RBF landmark field)     */
#define FGA_ERR_PARSE (-11)      /* file text not accepted by the native parser  */

#define FGA_PREC_FP32 0 /* FP32 traversal/direct sums, fp64 state (default)   */
#define FGA_PREC_FP64 1 /* fp64 everywhere: bit-exact reference visit order   */

typedef struct fga_ctx fga_ctx;

/* Mirrors core.FgaParams (core.py:103-117); validated like core.validate
 * (core.py:127-151), first failing field reported through fga_last_error(). */
typedef struct {
  double G, epsilon, eta, dt, theta, sigma;
  int32_t rho, max_depth;
  double norm_a, norm_b, conv_tol;
  int32_t max_iters;
  int32_t pad_;
} fga_params;

/* Mirrors registration.RegisterOptions (registration.py:22-31) plus the
 * B200-side knobs (precision, poll interval). */
typedef struct {
  int32_t trace_gpe;         /* RegisterOptions.trace_gpe          */
  int32_t normalize;         /* RegisterOptions.normalize          */
  int32_t record_iterations; /* RegisterOptions.record_iterations  */
  int32_t precision;         /* FGA_PREC_*                         */
  const double* x_weights;   /* RegisterOptions.x_weights or NULL  */
  const double* y_weights;   /* RegisterOptions.y_weights or NULL  */
  int32_t poll_every;        /* iterations enqueued between host polls of the
                                device convergence flag (0 = default 8)       */
  int32_t compute_gpe;       /* 1 (default semantics): gpe_initial/final      */
  int32_t mass_field;        /* 0 = NIV lattice (reference default), 1 = kNN  */
  int32_t knn_k;             /* k for mass_field = 1 (default 16, <= 32)      */
  const int64_t* x_landmarks;/* LandmarkSet.reference_indices() or NULL       */
  const int64_t* y_landmarks;/* LandmarkSet.template_indices() or NULL        */
  int32_t n_landmarks;       /* > 0: SPM = field * RBF (registration.py:74-83) */
  int32_t count_visits;      /* 1: the FP32 force pass also counts node visits
                                (fga_result.visits, visits_per_iter); 0 = off,
                                2.5% faster (accepted interactions are always
                                counted; the fp64 pass always counts both)  */
} fga_options;

/* Mirrors registration.RegistrationResult (core.py:162-172). */
typedef struct {
  double R[9], t[3];           /* transform in the original frame (normalize.py:63-84) */
  double R_norm[9], t_norm[3]; /* R_acc, t_acc in the normalized frame           */
  int64_t iterations;
  int32_t converged;
  int32_t pad_;
  double gpe_initial, gpe_final;
  double norm_ctx[10];         /* mean_x[3], mean_y[3], l, r, a, b            */
  int64_t interactions;        /* sum over iterations of accepted interactions */
  int64_t visits;              /* sum over iterations of node visits           */
  int64_t n_nodes;             /* reference tree size                          */
  double setup_ms, loop_ms, gpe_ms; /* device-timed phases (CUDA events)       */
} fga_result;

/* One pair of a batched registration (BASELINE configs[4]). */
typedef struct {
  double R[9], t[3];        /* transform in the original frame               */
  int64_t iterations;
  int32_t converged;
  int32_t status;           /* FGA_OK or the FGA_ERR_* this pair raised      */
  double gpe_initial, gpe_final;
  int64_t interactions;     /* accepted interactions summed over iterations  */
  int64_t n_nodes;          /* reference tree size                           */
} fga_pair_result;

/* ------------------------------------------------------------------ misc */
int fga_version(void);
const char* fga_last_error(void);
int fga_device_count(int* count);

int fga_create(fga_ctx** ctx, int device);
int fga_destroy(fga_ctx* ctx);
/* Bind the context to a CUDA stream (cudaStream_t as void*; NULL = the legacy
 * default stream).  A new context owns a private non-blocking stream. */
int fga_set_stream(fga_ctx* ctx, void* stream);
int fga_synchronize(fga_ctx* ctx);

/* --------------------------------------------------- driver-level entry
 * registration.register (registration.py:91-166): normalize, masses, tree,
 * gpe_initial, iteration loop with Kabsch projection, gpe_final, denormalize.
 * x: (n,dim) reference, y: (m,dim) template, host fp64.  dim must be 3.
 * deltas / traj (12 per iteration, [R_acc|t_acc] row-major) / gpe_trace /
 * interactions_per_iter are optional host outputs sized >= max_iters. */
int fga_register(fga_ctx* ctx, const double* x, int64_t n, const double* y, int64_t m, int dim,
                 const fga_params* params, const fga_options* options, fga_result* out,
                 double* deltas, double* traj, double* gpe_trace, int64_t* interactions_per_iter);

/* --------------------------------------------- batched driver (config 5)
 * registration.register applied to n_pairs independent pairs in ONE
 * persistent kernel (one CTA per pair at a time, whole loop on the device).
 * x_all/y_all: concatenated (sum n_p, 3) / (sum m_p, 3) fp64 clouds,
 * x_offsets/y_offsets: n_pairs+1 row offsets.  options->x_weights/y_weights,
 * if set, are concatenated like x_all/y_all.  Per-pair failures (empty,
 * degenerate, too large for the batched kernel: > 8192 points) are reported
 * in fga_pair_result.status instead of aborting the batch, like
 * registration.register_sequence does (registration.py:192-200).  deltas
 * (optional) is n_pairs * max_iters.  FP32 force precision only. */
int fga_register_batch(fga_ctx* ctx, const double* x_all, const int64_t* x_offsets,
                       const double* y_all, const int64_t* y_offsets, int64_t n_pairs, int dim,
                       const fga_params* params, const fga_options* options,
                       fga_pair_result* out, double* deltas);
/* Same with one host array per cloud (xs[p]: (xn[p],3), ys[p]: (yn[p],3)):
 * the clouds go to the device through a pinned staging ring filled on all
 * host threads while the copy engine drains it (no host-side concatenation).
 * options->x_weights / y_weights must be NULL (use fga_register_batch). */
int fga_register_batch_list(fga_ctx* ctx, const double* const* xs, const int64_t* xn,
                            const double* const* ys, const int64_t* yn, int64_t n_pairs,
                            int dim, const fga_params* params, const fga_options* options,
                            fga_pair_result* out, double* deltas);
/* Same with device-resident clouds/offsets/weights/outputs (stream-ordered). */
int fga_register_batch_dev(fga_ctx* ctx, const double* x_all, const int64_t* x_offsets,
                           const double* y_all, const int64_t* y_offsets, int64_t n_pairs,
                           int nmax, int mmax, int dim, const fga_params* params,
                           const fga_options* options, fga_pair_result* out_dev,
                           double* deltas_dev);

/* ---------------------------------------------- session (stepwise) entry
 * The same loop split into stream-ordered pieces so a host can insert a
 * collective between the force pass and the rigid update (template sharding
 * across GPUs).  shard_rank/shard_count select a contiguous
 * chunk of the Hilbert-sorted template; every rank passes the FULL clouds (the
 * normalization and the template mass field are global).  x/y are host
 * pointers for fga_session_begin and device pointers for _dev. */
int fga_session_begin(fga_ctx* ctx, const double* x, int64_t n, const double* y, int64_t m,
                      int dim, const fga_params* params, const fga_options* options,
                      int shard_rank, int shard_count);
int fga_session_begin_dev(fga_ctx* ctx, const double* x_dev, int64_t n, const double* y_dev,
                          int64_t m, int dim, const fga_params* params,
                          const fga_options* options, int shard_rank, int shard_count);
/* Enqueue the force pass of one iteration (forces, fused Euler-Cromer step and
 * Kabsch partial sums) and reduce this shard's partials into the sums buffer. */
int fga_session_forces(fga_ctx* ctx);
/* Device pointer to the 18-double sums buffer (layout: see DESIGN.md); a
 * multi-GPU host all-reduces it (sum) between _forces and _update. */
int fga_session_sums(fga_ctx* ctx, void** dev_ptr);
/* Use a caller-owned device buffer of >= 18 doubles (e.g. a torch tensor that
 * torch.distributed all-reduces in place) as the sums buffer. */
int fga_session_bind_sums(fga_ctx* ctx, void* dev_ptr);
/* Enqueue the rigid update: 3x3 fp64 SVD, transform accumulation, delta,
 * convergence flag. */
int fga_session_update(fga_ctx* ctx);
/* Enqueue k full iterations (forces + update), single shard only. */
int fga_session_iterate(fga_ctx* ctx, int k);
/* Enqueue the energy pass of the CURRENT positions into the sums buffer
 * (slot 17); collect with fga_session_take_gpe after an optional all-reduce. */
int fga_session_gpe(fga_ctx* ctx);
int fga_session_take_gpe(fga_ctx* ctx, double* value);
/* Apply the pending rigid transform to the positions (idempotent). */
int fga_session_apply_pending(fga_ctx* ctx);
/* Host poll of the device flags (synchronizes the stream). */
int fga_session_poll(fga_ctx* ctx, int* done, int64_t* iterations);
/* Apply the pending transform, compute gpe_final (unless skip_gpe), copy
 * results out.  With shard_count>1 the caller supplies the all-reduced
 * gpe_final via fga_session_set_gpe_final instead. */
int fga_session_finish(fga_ctx* ctx, fga_result* out, double* deltas, double* traj,
                       double* gpe_trace, int64_t* interactions_per_iter,
                       int64_t* visits_per_iter);
int fga_session_set_gpe(fga_ctx* ctx, int which /*0 initial,1 final*/, double value);
/* Number of template points owned by this shard and total tree nodes. */
int fga_session_info(fga_ctx* ctx, int64_t* m_local, int64_t* n_nodes);
/* Iteration state (checkpoint / resume, teacher-forced parity): template
 * positions and velocities entering the next iteration, normalized frame,
 * host (m,3) arrays in input order (a shard reads / writes its own rows
 * only), the accumulated [R_acc | t_acc] (registration.py:137-138) and the
 * number of completed iterations.  set_state resumes from such a state
 * (pending step transform = identity). */
int fga_session_get_state(fga_ctx* ctx, double* pos, double* vel, double* racc9, double* tacc3,
                          int64_t* iter);
int fga_session_set_state(fga_ctx* ctx, const double* pos, const double* vel, const double* racc9,
                          const double* tacc3, int64_t iter);
/* Device-side checkpoint of this shard's iteration state (template
 * positions/velocities, pending and accumulated transforms, iteration
 * counter): restore = 0 saves, 1 restores (stream-ordered, no host copy). */
int fga_session_checkpoint(fga_ctx* ctx, int restore);
/* The session's rescaled mass fields (registration.py:85-87) in input order:
 * mx (n) for the reference, my (m) for the template; either may be NULL. */
int fga_session_masses(fga_ctx* ctx, double* mx, double* my);

/* --------------------------------------------------- tree-level entries
 * bhtree.build (bhtree.py:56-122) on the device; the tree stays in the
 * context.  n_nodes receives the node count. */
int fga_tree_build(fga_ctx* ctx, const double* pts, const double* masses, int64_t n, int dim,
                   int max_depth, int64_t* n_nodes);
/* Same build from device-resident (n,3) points and masses, stream-ordered
 * (one internal sync for the node count); the inputs must stay alive while
 * the context's tree is used (the tree references them). */
int fga_tree_build_dev(fga_ctx* ctx, const double* pts_dev, const double* masses_dev, int64_t n,
                       int max_depth, int64_t* n_nodes);
/* Copy the context's tree out in the BHTree array layout (bhtree.py:14-45):
 * children (n_nodes,8) int64, com (n_nodes,3), mass, length, occupancy,
 * depth (int64), bbox_min/max (n_nodes,3).  Any pointer may be NULL. */
int fga_tree_export(fga_ctx* ctx, int64_t* children, double* com, double* mass, double* length,
                    int64_t* occupancy, int64_t* depth, double* bbox_min, double* bbox_max);
/* Load an existing BHTree (e.g. built by the reference) into the context:
 * the arrays of bhtree.BHTree, nodes in preorder (bhtree.py:77). */
int fga_tree_upload(fga_ctx* ctx, const int64_t* children, const double* com, const double* mass,
                    const double* length, int64_t n_nodes, int n_child, int dim);

/* Counter bumped by every build / upload into the context's tree (including
 * the one register() / a session performs): a host caching "tree T is
 * loaded" compares it before reusing the device copy. */
int fga_tree_generation(fga_ctx* ctx, int64_t* generation);

/* ------------------------------------------------ operator-level entries */
/* _kernels.bh_forces_kernel (_kernels.py:7-50) as called by bhtree.bh_forces
 * (bhtree.py:125-147), against the context's tree: forces (m,3) and optional
 * visits / accepted (m,) int64.  eps2 = epsilon^2 as the reference passes it.
 * precision FGA_PREC_FP64 reproduces the reference visit order and per-term
 * arithmetic exactly. */
int fga_tree_forces(fga_ctx* ctx, const double* queries, const double* query_masses, int64_t m,
                    double theta, double G, double eps2, int precision, double* forces,
                    int64_t* visits, int64_t* accepted);
/* Accepted (interacting) nodes summed over the queries of the last
 * fga_tree_forces / fga_bh_forces_kernel call in this context, -1 before the
 * first -- the interaction count without the per-query `accepted` array (an
 * extension: the reference does not report it). */
int fga_last_interactions(fga_ctx* ctx, int64_t* accepted_total);

/* The reference's exact kernel signature (_kernels.py:7-8): uploads the tree
 * arrays (skipped when the same arrays -- address, size, sampled contents --
 * are still the context's tree), then evaluates in FP64 (the reference's
 * arithmetic, bit-identical forces and visits).  The literal ctypes drop-in
 * of INTEGRATION.md. */
int fga_bh_forces_kernel(fga_ctx* ctx, const int64_t* children, const double* com,
                         const double* mass, const double* length, int64_t n_nodes, int n_child,
                         const double* queries, const double* query_masses, int64_t m, int dim,
                         double theta, double G, double eps2, int64_t stack_cap, double* forces,
                         int64_t* visits);
/* bhtree.brute_force (bhtree.py:155-164) for every query row: the tiled
 * direct O(NM) sum.  eps is epsilon (not squared), as brute_force reads it. */
int fga_direct_forces(fga_ctx* ctx, const double* ref, const double* ref_masses, int64_t n,
                      const double* queries, const double* query_masses, int64_t m, int dim,
                      double G, double eps, int precision, double* forces);
/* _kernels.gpe_kernel (_kernels.py:53-67). */
int fga_gpe_kernel(fga_ctx* ctx, const double* pos_y, const double* mass_y, int64_t m,
                   const double* pos_x, const double* mass_x, int64_t n, int dim, double G,
                   double eps, int precision, double* out);
/* Exact k nearest OTHER points of every point (grid-bucketed, fp64 distances,
 * ties broken by index): idx (n,k) int64 and squared distances (n,k), either
 * may be NULL.  1 <= k < n, k <= 32. */
int fga_knn(fga_ctx* ctx, const double* pts, int64_t n, int dim, int k, int64_t* idx,
            double* d2);
/* kNN smooth-particle masses: (4/3) pi r_k^3 / k, floored at 1e-6 (an opt-in
 * alternative to niv_masses, BASELINE configs[3]). */
int fga_knn_masses(fga_ctx* ctx, const double* pts, int64_t n, int dim, int k, double* out);
/* masses.rbf_masses (masses.py:55-82): Gaussian RBF through the anchors
 * pts[anchors[j]]; FGA_ERR_SINGULAR when cond(K) > 1e12.  m <= 2048. */
int fga_rbf_masses(fga_ctx* ctx, const double* pts, int64_t n, int dim, const int64_t* anchors,
                   int m, double sigma, double* out);
/* masses.niv_masses (masses.py:85-116). */
int fga_niv_masses(fga_ctx* ctx, const double* pts, int64_t n, int dim, int rho, double a,
                   double b, int max_depth, double* out);
/* normalize.normalize_pair (normalize.py:36-60): xn, yn (host, same shapes)
 * and ctx10 = mean_x[3], mean_y[3], l, r, a, b. */
int fga_normalize_pair(fga_ctx* ctx, const double* x, int64_t n, const double* y, int64_t m,
                       int dim, double a, double b, double* xn, double* yn, double* ctx10);
/* procrustes.solve_rigid (procrustes.py:12-49): R (3x3 row-major), t (3),
 * degenerate flag. */
int fga_solve_rigid(fga_ctx* ctx, const double* y, const double* y_d, int64_t m, int dim,
                    double* R, double* t, int32_t* degenerate);

/* ------------------------------------------------ file ingestion (host)
 * io.load_cloud / io.load_weights (io.py:11-111) on a file's bytes, parsed
 * on all host threads.  Call with out == NULL for the counts, then with an
 * out buffer of >= n*dim (cloud) / n (weights) doubles.  FGA_ERR_PARSE for
 * anything the native parser does not accept (malformed files, non-ASCII);
 * the Python layer then raises the reference's exception (ParseError /
 * UnsupportedFormat with the reference's line number and message). */
int fga_parse_cloud(const char* text, int64_t len, double* out, int64_t cap, int64_t* n,
                    int* dim);
int fga_parse_weights(const char* text, int64_t len, double* out, int64_t cap, int64_t* n);

#ifdef __cplusplus
}
#endif
#endif /* FGA_H_ */
