/*
 * fga_oracle.c -- CPU ORACLE FOR PARITY TESTS.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is a plain-C restatement of the reference (gravreg 0.1.0) hot-path
 * arithmetic.  It exists so that tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py have a checker and a CPU
 * baseline that travels to the GPU box (the Python reference does not).
 * Nothing in paper_2009_14005_b200/ may import, link or call it.
 *
 * Pinning: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py
 * imports /root/reference/pkg/src/gravreg in the build container).
 *
 * Build: see oracle/Makefile.  MUST be compiled with -ffp-contract=off and
 * without -ffast-math so that every multiply/add rounds exactly like numba's
 * (non-fastmath) LLVM code and numpy's element-wise loops.
 *
 * Functions and the reference lines they restate:
 *   orc_pairwise_sum   numpy's 1-D add.reduce (used by masses.sum() in
 *                      bhtree.py:79 and registration.py:85)
 *   orc_tree_build     bhtree.build, bhtree.py:56-122
 *   orc_bh_forces      _kernels.bh_forces_kernel, _kernels.py:7-50
 *                      (+ an `accepted` counter: leaf+cell interactions)
 *   orc_brute_forces   bhtree.brute_force, bhtree.py:155-164 (batched)
 *   orc_gpe            _kernels.gpe_kernel, _kernels.py:53-67
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
 * DOUBLE_pairwise_sum): blocks of <=128 with 8 partial sums. */
static double pairwise(const double* a, int64_t n, int64_t stride) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r += a[i * stride];
        return r;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j * stride];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[(i + j) * stride];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i * stride];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise(a, n2, stride) + pairwise(a + n2 * stride, n - n2, stride);
    }
}

double orc_pairwise_sum(const double* a, int64_t n) { return pairwise(a, n, 1); }

/* ------------------------------------------------------------------------ */
/* Tree build: bhtree.py:56-122                                              */
/* ------------------------------------------------------------------------ */
typedef struct {
    int d, n_child, max_depth;
    int64_t n, cap, count;
    int64_t* children; /* (cap, n_child) */
    double* com;       /* (cap, d) */
    double* mass;
    double* length;
    int64_t* occupancy;
    int64_t* depth;
    double* bmin;      /* (cap, d) */
    double* bmax;
    const double* pts;
    const double* masses;
    double* scratch_m; /* gathered masses for the pairwise sum */
} orc_tree;

static int grow(orc_tree* t) {
    int64_t cap = t->cap ? t->cap * 2 : 1024;
#define GROW(ptr, type, width)                                              \
    do {                                                                    \
        void* p_ = realloc(t->ptr, (size_t)cap * (width) * sizeof(type));   \
        if (!p_) return -1;                                                 \
        t->ptr = (type*)p_;                                                 \
    } while (0)
    GROW(children, int64_t, t->n_child);
    GROW(com, double, t->d);
    GROW(mass, double, 1);
    GROW(length, double, 1);
    GROW(occupancy, int64_t, 1);
    GROW(depth, int64_t, 1);
    GROW(bmin, double, t->d);
    GROW(bmax, double, t->d);
#undef GROW
    t->cap = cap;
    return 0;
}

/* new_node (bhtree.py:76-105).  idx is the node's point list in the
 * reference's order (ascending original index: stable partitions of arange). */
static int64_t new_node(orc_tree* t, int64_t* idx, int64_t cnt, const double* bmin,
                        const double* bmax, int depth, int64_t* work) {
    const int d = t->d;
    if (t->count == t->cap && grow(t)) return -2;
    const int64_t node = t->count++;
    /* total = m.sum() : 1-D pairwise (bhtree.py:78-79) */
    for (int64_t i = 0; i < cnt; i++) t->scratch_m[i] = t->masses[idx[i]];
    const double total = pairwise(t->scratch_m, cnt, 1);
    for (int c = 0; c < t->n_child; c++) t->children[node * t->n_child + c] = -1;
    /* com = (pts[idx] * m[:, None]).sum(axis=0) / total : row-sequential (:80) */
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t i = 0; i < cnt; i++)
        for (int k = 0; k < d; k++) acc[k] += t->pts[idx[i] * d + k] * t->masses[idx[i]];
    for (int k = 0; k < d; k++) t->com[node * d + k] = acc[k] / total;
    t->mass[node] = total;
    /* length = ||bmax - bmin||_2 (:83); sequential dot, no FMA */
    double sq = 0.0;
    for (int k = 0; k < d; k++) {
        double e = bmax[k] - bmin[k];
        sq += e * e;
    }
    t->length[node] = sqrt(sq);
    t->occupancy[node] = cnt;
    t->depth[node] = depth;
    for (int k = 0; k < d; k++) {
        t->bmin[node * d + k] = bmin[k];
        t->bmax[node * d + k] = bmax[k];
    }
    if (cnt > 1 && depth < t->max_depth) {
        double center[3];
        for (int k = 0; k < d; k++) center[k] = bmin[k] + (bmax[k] - bmin[k]) / 2.0; /* :90 */
        /* slot = sum_k (p_k >= center_k) << (d-1-k)  (:93-96) */
        int64_t counts[8] = {0};
        int8_t* slot = (int8_t*)(work);
        for (int64_t i = 0; i < cnt; i++) {
            int s = 0;
            for (int k = 0; k < d; k++) s = s * 2 + (t->pts[idx[i] * d + k] >= center[k]);
            slot[i] = (int8_t)s;
            counts[s]++;
        }
        /* stable partition of idx by slot (:97-98) into a temp buffer */
        int64_t* part = (int64_t*)malloc((size_t)cnt * sizeof(int64_t));
        if (!part) return -2;
        int64_t off[8];
        int64_t o = 0;
        for (int c = 0; c < t->n_child; c++) { off[c] = o; o += counts[c]; }
        for (int64_t i = 0; i < cnt; i++) part[off[(int)slot[i]]++] = idx[i];
        memcpy(idx, part, (size_t)cnt * sizeof(int64_t));
        free(part);
        o = 0;
        for (int c = 0; c < t->n_child; c++) {
            if (counts[c] == 0) continue;
            double cmin[3], cmax[3];
            for (int k = 0; k < d; k++) {
                int bit = (c >> (d - 1 - k)) & 1; /* :100-103 */
                cmin[k] = bit ? center[k] : bmin[k];
                cmax[k] = bit ? bmax[k] : center[k];
            }
            int64_t child = new_node(t, idx + o, counts[c], cmin, cmax, depth + 1, work);
            if (child < 0) return child;
            t->children[node * t->n_child + c] = child;
            o += counts[c];
        }
    }
    return node;
}

/* Returns node count (>0) or a negative error.  *out receives the tree. */
int64_t orc_tree_build(const double* pts, const double* masses, int64_t n, int d, int max_depth,
                       orc_tree** out) {
    if (n <= 0 || (d != 2 && d != 3)) return -1;
    orc_tree* t = (orc_tree*)calloc(1, sizeof(orc_tree));
    if (!t) return -2;
    t->d = d;
    t->n_child = 1 << d;
    t->max_depth = max_depth;
    t->n = n;
    t->pts = pts;
    t->masses = masses;
    t->scratch_m = (double*)malloc((size_t)n * sizeof(double));
    int64_t* idx = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    int64_t* work = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    if (!t->scratch_m || !idx || !work) return -2;
    for (int64_t i = 0; i < n; i++) idx[i] = i;
    double bmin[3], bmax[3]; /* root bbox = per-axis min/max (:107-108) */
    for (int k = 0; k < d; k++) {
        bmin[k] = pts[k];
        bmax[k] = pts[k];
    }
    for (int64_t i = 1; i < n; i++)
        for (int k = 0; k < d; k++) {
            double v = pts[i * d + k];
            if (v < bmin[k]) bmin[k] = v;
            if (v > bmax[k]) bmax[k] = v;
        }
    int64_t r = new_node(t, idx, n, bmin, bmax, 0, work);
    free(idx);
    free(work);
    free(t->scratch_m);
    t->scratch_m = NULL;
    t->pts = NULL;
    t->masses = NULL;
    if (r < 0) return r;
    *out = t;
    return t->count;
}

void orc_tree_copy(const orc_tree* t, int64_t* children, double* com, double* mass, double* length,
                   int64_t* occupancy, int64_t* depth, double* bbox_min, double* bbox_max) {
    const int64_t n = t->count;
    memcpy(children, t->children, (size_t)n * t->n_child * sizeof(int64_t));
    memcpy(com, t->com, (size_t)n * t->d * sizeof(double));
    memcpy(mass, t->mass, (size_t)n * sizeof(double));
    memcpy(length, t->length, (size_t)n * sizeof(double));
    memcpy(occupancy, t->occupancy, (size_t)n * sizeof(int64_t));
    memcpy(depth, t->depth, (size_t)n * sizeof(int64_t));
    memcpy(bbox_min, t->bmin, (size_t)n * t->d * sizeof(double));
    memcpy(bbox_max, t->bmax, (size_t)n * t->d * sizeof(double));
}

void orc_tree_free(orc_tree* t) {
    if (!t) return;
    free(t->children);
    free(t->com);
    free(t->mass);
    free(t->length);
    free(t->occupancy);
    free(t->depth);
    free(t->bmin);
    free(t->bmax);
    free(t);
}

/* ------------------------------------------------------------------------ */
/* Tree traversal forces: _kernels.py:7-50                                   */
/* ------------------------------------------------------------------------ */
int orc_bh_forces(const int64_t* children, const double* com, const double* mass,
                  const double* length, int64_t n_nodes, int n_child, const double* queries,
                  const double* qmasses, int64_t m, int d, double theta, double G, double eps2,
                  int64_t stack_cap, double* forces, int64_t* visits, int64_t* accepted,
                  int nthreads) {
    (void)n_nodes;
    const double theta2 = theta * theta;
    int err = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        int64_t* stack = (int64_t*)malloc((size_t)stack_cap * sizeof(int64_t));
        if (!stack) err = -2;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
        for (int64_t q = 0; q < m; q++) {
            if (!stack) continue;
            double f[3] = {0.0, 0.0, 0.0};
            int64_t sp = 0, nv = 0, na = 0;
            stack[sp++] = 0;
            while (sp > 0) {
                int64_t node = stack[--sp];
                nv++;
                double d2 = 0.0;
                for (int k = 0; k < d; k++) {
                    double dk = queries[q * d + k] - com[node * d + k];
                    d2 += dk * dk;
                }
                int leaf = 1;
                for (int c = 0; c < n_child; c++)
                    if (children[node * n_child + c] >= 0) { leaf = 0; break; }
                if (leaf || length[node] * length[node] < theta2 * d2) {
                    na++;
                    double denom = d2 + eps2;
                    if (denom > 0.0) {
                        double w = G * qmasses[q] * mass[node] / (denom * sqrt(denom));
                        for (int k = 0; k < d; k++) f[k] -= w * (queries[q * d + k] - com[node * d + k]);
                    }
                } else {
                    for (int c = 0; c < n_child; c++) {
                        int64_t ch = children[node * n_child + c];
                        if (ch >= 0) {
                            if (sp >= stack_cap) { err = -3; sp = 0; break; }
                            stack[sp++] = ch;
                        }
                    }
                }
            }
            for (int k = 0; k < d; k++) forces[q * d + k] = f[k];
            if (visits) visits[q] = nv;
            if (accepted) accepted[q] = na;
        }
        free(stack);
    }
    return err;
}

/* ------------------------------------------------------------------------ */
/* Exact O(NM) sum: bhtree.brute_force (bhtree.py:155-164), per query        */
/* ------------------------------------------------------------------------ */
void orc_brute_forces_out(const double* ref, const double* rmass, int64_t n,
                          const double* queries, const double* qmass, int64_t m, int d, double G,
                          double eps, double* out, int nthreads) {
    const double eps2 = eps * eps; /* params.epsilon**2 */
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 16)
#endif
    for (int64_t q = 0; q < m; q++) {
        double s[3] = {0.0, 0.0, 0.0};
        for (int64_t j = 0; j < n; j++) {
            double delta[3], dd = 0.0;
            for (int k = 0; k < d; k++) {
                delta[k] = queries[q * d + k] - ref[j * d + k];
                dd += delta[k] * delta[k];
            }
            double d2 = dd + eps2;
            double w = d2 > 0 ? rmass[j] / pow(d2, 1.5) : 0.0;
            for (int k = 0; k < d; k++) s[k] += w * delta[k];
        }
        double scale = -G * qmass[q];
        for (int k = 0; k < d; k++) out[q * d + k] = scale * s[k];
    }
}

/* ------------------------------------------------------------------------ */
/* Potential energy: _kernels.gpe_kernel (_kernels.py:53-67)                 */
/* Per-row sums are computed in parallel, the outer sum stays sequential in  */
/* row order, so the result is bit-identical to the serial reference.        */
/* ------------------------------------------------------------------------ */
double orc_gpe(const double* pos_y, const double* mass_y, int64_t m, const double* pos_x,
               const double* mass_x, int64_t n, int d, double G, double eps, int nthreads) {
    double* rows = (double*)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    if (!rows) return NAN;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 16)
#endif
    for (int64_t i = 0; i < m; i++) {
        double acc = 0.0;
        for (int64_t j = 0; j < n; j++) {
            double d2 = 0.0;
            for (int k = 0; k < d; k++) {
                double dk = pos_y[i * d + k] - pos_x[j * d + k];
                d2 += dk * dk;
            }
            acc += mass_x[j] / (sqrt(d2) + eps);
        }
        rows[i] = acc;
    }
    double total = 0.0;
    for (int64_t i = 0; i < m; i++) total += mass_y[i] * rows[i];
    free(rows);
    return -G * total;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
