/*
 * CPU oracle for the octfuse hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's native kernel module
 * (/root/reference/pkg/src/octfuse/_kernels.pyx, mirrored in _pykernels.py),
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as
 * the checker.  Nothing in the product path (paper_1608_07411_b200/) links
 * or calls this library.
 *
 * Pools follow the reference layout exactly: node 0 is the root, children of
 * a node are 8 contiguous slots, child[n] is the first child or -1, and
 * state = {slots used, free-list head, live nodes}.  Arithmetic keeps the
 * reference's evaluation order (no FMA contraction: built with
 * -ffp-contract=off) so results are bit-identical to the compiled reference.
 */
#ifndef OCTFUSE_ORACLE_H
#define OCTFUSE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes */
#define ORC_OK 0
#define ORC_EDEPTH 1   /* d_max > 60             (ValueError)   */
#define ORC_ENOMEM 2   /* scratch allocation     (MemoryError)  */
#define ORC_EPOOL 3    /* pool capacity exhausted (RuntimeError) */

/* _kernels.pyx:21-77 -- spread-rule build from flattened pyramids.
 * value_is_f32 selects the value pool type (float32 for view trees). */
int orc_build_tree(const double *meanf, const double *minf, const double *maxf,
                   const int64_t *offs, int has_w, const uint8_t *wminf,
                   const uint8_t *wmaxf, const double *wmeanf, double tau,
                   void *value, int value_is_f32, float *weight,
                   int32_t *child, int64_t *state, int d_max);

/* _kernels.pyx:80-113 -- inner value = sequential sum of children / 8 */
int orc_propagate_f64(double *value, const int32_t *child, int64_t cap);
int orc_propagate_f32(float *value, const int32_t *child, int64_t cap);

/* _kernels.pyx:116-158 -- scatter leaves into a dense (2^d)^3 grid */
int orc_densify_f64(const double *value, const int32_t *child, int d_max,
                    double *out);
int orc_densify_f32(const float *value, const int32_t *child, int d_max,
                    double *out);

/* _kernels.pyx:384-461 -- one Jacobi descent pass with in-pass split and
 * join cascades, then the sweep that frees joined subtrees.  Returns an
 * error code; counters are written to out3 = {splits, joins, log rows}. */
int orc_iterate_pass(double *uval, double *usnap, int32_t *uchild,
                     uint8_t *ujoined, int64_t *ustate, int64_t cap,
                     int nviews, const float *const *vval,
                     const float *const *vw, const int32_t *const *vchild,
                     int d_max, double lam, double eps, double gamma,
                     double xi, double tau_s, double tau_j, int clamp,
                     int reverse, double *jlog, int64_t jcap, int64_t *out3);

/* _kernels.pyx:466-578 -- leaf-summed energy, Morton order, f64 */
int orc_tree_energy(const double *uval, const int32_t *uchild, int nviews,
                    const float *const *vval, const float *const *vw,
                    const int32_t *const *vchild, int d_max, double lam,
                    double eps, double gamma, double *out);

/* pd_oracle.c -- the north_star's TV-L1 primal-dual pass (PARITY UNPINNED:
 * no reference implementation exists; see the definition in that file). */
int orc_pd_pass(const double *u, const double *ub, const double *px,
                const double *py, const double *pz, double *u_o, double *ub_o,
                double *px_o, double *py_o, double *pz_o,
                const int32_t *child, int64_t used, int nviews,
                const float *const *vval, const float *const *vw,
                const int32_t *const *vchild, int d_max, double lam, double tau,
                double sigma, double gamma, int clamp, double *energy);

/* pd-mode split/join after a pass (definition in pd_oracle.c); out2 =
 * {splits, joins} */
int orc_pd_restructure(double *u, double *ub, double *px, double *py,
                       double *pz, int32_t *child, int64_t *state, int64_t cap,
                       int d_max, double tau_s, double tau_j, int64_t *out2);

#ifdef __cplusplus
}
#endif
#endif
