// fga_tree.cuh -- device tree containers shared by tree.cu / forces.cu / capi.cu
#pragma once
#include <algorithm>
#include <cmath>
#include <vector>

#include "fga_internal.cuh"

namespace fga {

// Mirrored-preorder traversal records.
struct TreeRecords {
  double4* a64;
  NodeB64* b64;
  // packed FP32 traversal record, 32 B per node (NodeC32):
  //   c32[2x]   = {com.xyz, mass}
  //   c32[2x+1] = {l^2 + theta^2 eps^2 | -inf, skip (int bits), band, l^2 | -inf}
  // .x and .z are (re)written per launch by launch_node_bands (forces.cu)
  // from the raw l^2 in .w; the build writes .x = .w = l^2, .z = 0.
  float4* c32;
};

struct TreeDev {
  int64_t n_points = 0, n_nodes = 0;
  int L = 0;
  int dim = 3;  // 2: quadtree carried as z = 0 (see capi.cu pad3)
  double cmag = 0.0;  // max |coordinate| over node centres (fp32 MAC guard)
  double box_host[6] = {0, 0, 0, 0, 0, 0};
  bool exportable = false;
  // bumped by every build / upload into this container: host-side caches of
  // "which tree is loaded" (the Python BHTree token, the bh_forces_kernel
  // shim's upload key) compare against it (fga_tree_generation)
  uint64_t generation = 0;
  // max_depth 22..42 builds with 128-bit keys (wide_keys), exactly the
  // reference's tree.  max_depth > 42 (kMaxLevelsDeep): built with 42
  // levels; valid when no level-42 cell holds two points (the trees are then
  // equal), and for a registration also when such cells hold only exact
  // duplicates (the reference's extra single-child chain below them changes
  // visit counts, never an accepted term: same com, same mass).  Set by
  // tree_build_dev.
  int L_requested = 0;
  bool wide_keys = false;     // L > 21: 128-bit keys (tree.cu K128)
  bool cap_runs = false;      // some cell at the level cap holds >= 2 points
  bool cap_distinct = false;  // ... of which two are distinct
  const double* pts = nullptr;     // (n,3) device, not owned
  const double* masses = nullptr;  // (n,) device, not owned
  DevBuf box, scratch, keys_in, keys, idx_in, idx, clev, count, offset, cub_tmp;
  // build intermediates: packed (x,y,z,m) in input order, sorted copy, the
  // run-overflow flag, per-(level, block) boundary partials (tree.cu Cross)
  DevBuf keys32_in, keys32, packed, sp, flags, cross;
  DevBuf a64, b64, c32;
  DevBuf band_scratch;  // per-launch query bound of the node bands (forces.cu)
  DevBuf export_buf;

  TreeRecords records() const {
    return TreeRecords{a64.as<double4>(), b64.as<NodeB64>(), c32.as<float4>()};
  }
  void release() {
    DevBuf* all[] = {&box,    &scratch, &keys_in, &keys,   &idx_in, &idx, &clev,
                     &count,  &offset,  &cub_tmp, &keys32_in, &keys32, &packed, &sp,     &flags,
                     &cross,  &a64,    &b64,    &c32, &band_scratch, &export_buf};
    for (DevBuf* b : all) b->release();
    n_nodes = 0;
    exportable = false;
  }
};

int tree_build_dev(TreeDev& T, const double* pts_dev, const double* masses_dev, int64_t n, int L,
                   cudaStream_t st);
// 1 when some leaf of the built tree aggregates two distinct points (a
// depth-cap leaf): then the theta = 0 tree sum differs from the exact O(NM)
// sum (synchronizes the stream)
int tree_any_shared_leaf(TreeDev& T, cudaStream_t st, int* host_flag);
int tree_export_host(TreeDev& T, cudaStream_t st, int64_t* children, double* com, double* mass,
                     double* length, int64_t* occupancy, int64_t* depth, double* bmin,
                     double* bmax);
int tree_upload_host(TreeDev& T, const int64_t* children, const double* com, const double* mass,
                     const double* length, int64_t nn, int n_child, cudaStream_t st);

}  // namespace fga
