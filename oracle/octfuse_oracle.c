/*
 * CPU oracle for the octfuse hot path -- TEST INFRASTRUCTURE ONLY.
 * See octfuse_oracle.h.  Each routine cites the reference lines it restates
 * (paths relative to /root/reference/pkg/src/octfuse/).
 *
 * Floating-point rule: every expression is written with the reference's
 * operand order and compiled with -ffp-contract=off, so the doubles produced
 * here equal the compiled reference's bit for bit.
 */
#include "octfuse_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* child index of a cell inside its parent: x is the high bit
 * (_kernels.pyx:71-73, :269) */
static inline int octant(int x, int y, int z) {
    return ((x & 1) << 2) | ((y & 1) << 1) | (z & 1);
}

typedef struct {
    int64_t node;
    int x, y, z, lvl;
} cell_t;

/* ---------------------------------------------------------------- build --
 * _kernels.pyx:21-77.  Depth-first with an explicit LIFO: children are
 * pushed 0..7 so child 7 is expanded (and allocates) first, which fixes the
 * pool layout the reference produces. */
int orc_build_tree(const double *meanf, const double *minf, const double *maxf,
                   const int64_t *offs, int has_w, const uint8_t *wminf,
                   const uint8_t *wmaxf, const double *wmeanf, double tau,
                   void *value, int value_is_f32, float *weight,
                   int32_t *child, int64_t *state, int d_max) {
    if (d_max > 60) return ORC_EDEPTH;
    cell_t stk[512];
    int top = 0;
    state[0] = 1;
    state[1] = -1;
    state[2] = 1;
    stk[top++] = (cell_t){0, 0, 0, 0, 0};
    while (top > 0) {
        cell_t c = stk[--top];
        int64_t n1 = (int64_t)1 << c.lvl;
        int64_t k = offs[c.lvl] + ((int64_t)c.x * n1 + c.y) * n1 + c.z;
        if (value_is_f32)
            ((float *)value)[c.node] = (float)meanf[k];
        else
            ((double *)value)[c.node] = meanf[k];
        if (has_w) weight[c.node] = (float)wmeanf[k];
        int split = 0;
        if (c.lvl < d_max) {
            if (maxf[k] - minf[k] > tau)
                split = 1;
            else if (has_w && wminf[k] != wmaxf[k])
                split = 1;
        }
        if (!split) {
            child[c.node] = -1;
            continue;
        }
        int64_t b = state[0];
        state[0] = b + 8;
        state[2] += 8;
        child[c.node] = (int32_t)b;
        for (int q = 0; q < 8; ++q)
            stk[top++] = (cell_t){b + q, 2 * c.x + ((q >> 2) & 1),
                                  2 * c.y + ((q >> 1) & 1), 2 * c.z + (q & 1),
                                  c.lvl + 1};
    }
    return ORC_OK;
}

/* ------------------------------------------------------------ propagate --
 * _kernels.pyx:80-113: list inner nodes parent-before-child, then average
 * children in reverse list order (children first), sequential f64 sum. */
#define DEFINE_PROPAGATE(NAME, T)                                            \
    int NAME(T *value, const int32_t *child, int64_t cap) {                  \
        int64_t *inner = (int64_t *)malloc((size_t)cap * sizeof(int64_t));  \
        int64_t *todo = (int64_t *)malloc((size_t)cap * sizeof(int64_t));    \
        if (!inner || !todo) {                                               \
            free(inner);                                                     \
            free(todo);                                                      \
            return ORC_ENOMEM;                                               \
        }                                                                    \
        int64_t ni = 0, nt = 0;                                              \
        todo[nt++] = 0;                                                      \
        while (nt > 0) {                                                     \
            int64_t n = todo[--nt];                                          \
            int64_t b = child[n];                                            \
            if (b < 0) continue;                                             \
            inner[ni++] = n;                                                 \
            for (int q = 0; q < 8; ++q) todo[nt++] = b + q;                  \
        }                                                                    \
        while (ni > 0) {                                                     \
            int64_t n = inner[--ni];                                         \
            int64_t b = child[n];                                            \
            double acc = 0.0;                                                \
            for (int q = 0; q < 8; ++q) acc += (double)value[b + q];         \
            value[n] = (T)(acc / 8.0);                                       \
        }                                                                    \
        free(inner);                                                         \
        free(todo);                                                          \
        return ORC_OK;                                                       \
    }
DEFINE_PROPAGATE(orc_propagate_f64, double)
DEFINE_PROPAGATE(orc_propagate_f32, float)

/* -------------------------------------------------------------- densify --
 * _kernels.pyx:116-158 */
#define DEFINE_DENSIFY(NAME, T)                                              \
    int NAME(const T *value, const int32_t *child, int d_max, double *out) { \
        if (d_max > 60) return ORC_EDEPTH;                                   \
        int64_t n = (int64_t)1 << d_max;                                     \
        cell_t stk[512];                                                     \
        int top = 0;                                                         \
        stk[top++] = (cell_t){0, 0, 0, 0, 0};                                \
        while (top > 0) {                                                    \
            cell_t c = stk[--top];                                           \
            int64_t b = child[c.node];                                       \
            if (b >= 0) {                                                    \
                for (int q = 0; q < 8; ++q)                                  \
                    stk[top++] = (cell_t){b + q, 2 * c.x + ((q >> 2) & 1),   \
                                          2 * c.y + ((q >> 1) & 1),          \
                                          2 * c.z + (q & 1), c.lvl + 1};     \
                continue;                                                    \
            }                                                                \
            int s = d_max - c.lvl;                                           \
            int64_t w = (int64_t)1 << s;                                     \
            double v = (double)value[c.node];                                \
            int64_t x0 = (int64_t)c.x << s, y0 = (int64_t)c.y << s,          \
                    z0 = (int64_t)c.z << s;                                  \
            for (int64_t i = x0; i < x0 + w; ++i)                            \
                for (int64_t j = y0; j < y0 + w; ++j)                        \
                    for (int64_t k = z0; k < z0 + w; ++k)                    \
                        out[(i * n + j) * n + k] = v;                        \
        }                                                                    \
        return ORC_OK;                                                       \
    }
DEFINE_DENSIFY(orc_densify_f64, double)
DEFINE_DENSIFY(orc_densify_f32, float)

/* --------------------------------------------------------- descent pass --
 * State shared by the recursive walk (_kernels.pyx:163-190). */
typedef struct {
    double *u, *snap;
    int32_t *child;
    uint8_t *joined;
    int64_t *state;
    int64_t cap;
    int nv;
    const float *const *vval;
    const float *const *vw;
    const int32_t *const *vchild;
    int64_t *vcur; /* nv rows of (d_max+1) per-level view nodes */
    int d_max;
    double lam, eps2, gamma, xi, tau_s, tau_j;
    int clamp, reverse;
    double *jlog;
    int64_t jcap, splits, joins, jrows;
    int failed;
} pass_t;

/* deepest node at level <= lvl on the root path of (x,y,z)@lvl, read from
 * the snapshot (_kernels.pyx:193-202; octree.py:148-166) */
static double snap_at(const pass_t *P, const double *arr, int x, int y, int z,
                      int lvl) {
    int64_t n = 0;
    for (int l = 0; l < lvl && P->child[n] >= 0; ++l) {
        int s = lvl - l - 1;
        n = P->child[n] + octant(x >> s, y >> s, z >> s);
    }
    return arr[n];
}

/* forward-difference flux g / sqrt(|g|^2 + eps^2) at a cell
 * (_kernels.pyx:205-220) */
static void cell_flux(const pass_t *P, int x, int y, int z, int lvl,
                      double out[3]) {
    int m = 1 << lvl;
    double h = (double)(1 << (P->d_max - lvl));
    double c = snap_at(P, P->snap, x, y, z, lvl);
    double gx = 0.0, gy = 0.0, gz = 0.0;
    if (x + 1 < m) gx = (snap_at(P, P->snap, x + 1, y, z, lvl) - c) / h;
    if (y + 1 < m) gy = (snap_at(P, P->snap, x, y + 1, z, lvl) - c) / h;
    if (z + 1 < m) gz = (snap_at(P, P->snap, x, y, z + 1, lvl) - c) / h;
    double gn = sqrt(gx * gx + gy * gy + gz * gz + P->eps2);
    out[0] = gx / gn;
    out[1] = gy / gn;
    out[2] = gz / gn;
}

/* update direction lam*div(p) - data'(u) (_kernels.pyx:223-253) */
static double descent_dir(const pass_t *P, int64_t node, int x, int y, int z,
                          int lvl) {
    double h = (double)(1 << (P->d_max - lvl));
    double c = P->snap[node];
    double p[3], q[3];
    double bx = 0.0, by = 0.0, bz = 0.0;
    cell_flux(P, x, y, z, lvl, p);
    if (x > 0) {
        cell_flux(P, x - 1, y, z, lvl, q);
        bx = q[0];
    }
    if (y > 0) {
        cell_flux(P, x, y - 1, z, lvl, q);
        by = q[1];
    }
    if (z > 0) {
        cell_flux(P, x, y, z - 1, lvl, q);
        bz = q[2];
    }
    double div = ((p[0] - bx) + (p[1] - by) + (p[2] - bz)) / h;
    double num = 0.0, den = P->gamma;
    for (int v = 0; v < P->nv; ++v) {
        int64_t vn = P->vcur[(int64_t)v * (P->d_max + 1) + lvl];
        double wv = (double)P->vw[v][vn];
        if (wv != 0.0) {
            double d = c - (double)P->vval[v][vn];
            num += wv * d / sqrt(d * d + P->eps2);
            den += wv;
        }
    }
    return P->lam * div - num / den;
}

/* step the per-view cursors from the parent level to this cell
 * (_kernels.pyx:265-273) */
static void views_descend(pass_t *P, int x, int y, int z, int lvl) {
    int stride = P->d_max + 1;
    if (lvl == 0) {
        for (int v = 0; v < P->nv; ++v) P->vcur[(int64_t)v * stride] = 0;
        return;
    }
    int sel = octant(x, y, z);
    for (int v = 0; v < P->nv; ++v) {
        int64_t *row = P->vcur + (int64_t)v * stride;
        int64_t par = row[lvl - 1];
        int64_t b = P->vchild[v][par];
        row[lvl] = b >= 0 ? b + sel : par;
    }
}

static void walk(pass_t *P, int64_t node, int x, int y, int z, int lvl);

static void walk_children(pass_t *P, int64_t b, int x, int y, int z, int lvl) {
    for (int i = 0; i < 8; ++i) {
        int q = P->reverse ? 7 - i : i;
        walk(P, b + q, 2 * x + ((q >> 2) & 1), 2 * y + ((q >> 1) & 1),
             2 * z + (q & 1), lvl + 1);
    }
}

/* claim eight slots: free list first, then the bump pointer
 * (_kernels.pyx:279-289; octree.py:126-138) */
static int64_t claim_block(pass_t *P) {
    int64_t head = P->state[1];
    int64_t b;
    if (head >= 0) {
        b = head;
        P->state[1] = P->child[b];
    } else {
        b = P->state[0];
        if (b + 8 > P->cap) return -1;
        P->state[0] = b + 8;
    }
    P->state[2] += 8;
    return b;
}

/* the recursive visit (_kernels.pyx:256-354) */
static void walk(pass_t *P, int64_t node, int x, int y, int z, int lvl) {
    if (P->failed) return;
    views_descend(P, x, y, z, lvl);
    double dn = P->snap[node] + P->xi * descent_dir(P, node, x, y, z, lvl);
    int64_t b = P->child[node];
    if (b < 0) {
        if (lvl < P->d_max && fabs(dn) < P->tau_s) {
            int64_t nb = claim_block(P);
            if (nb < 0) {
                P->failed = 1;
                return;
            }
            double pu = P->u[node], ps = P->snap[node];
            for (int q = 0; q < 8; ++q) {
                P->u[nb + q] = pu;
                P->snap[nb + q] = ps;
                P->child[nb + q] = -1;
                P->joined[nb + q] = 0;
            }
            P->child[node] = (int32_t)nb;
            P->splits++;
            walk_children(P, nb, x, y, z, lvl);
            return;
        }
        if (P->clamp) dn = dn > 1.0 ? 1.0 : (dn < -1.0 ? -1.0 : dn);
        P->u[node] = dn;
        return;
    }
    walk_children(P, b, x, y, z, lvl);
    if (P->failed || !(fabs(dn) > P->tau_j)) return;
    /* join test on the children's post-update values */
    int pos = 0, neg = 0;
    double acc = 0.0;
    for (int q = 0; q < 8; ++q) {
        int64_t cn = b + q;
        if (P->child[cn] >= 0 && !P->joined[cn]) return;
        double val = P->u[cn];
        if (!(val > P->tau_j || val < -P->tau_j)) return;
        if (val > 0.0)
            pos = 1;
        else
            neg = 1;
        acc += val;
    }
    if (pos && neg) return;
    P->joined[node] = 1;
    P->u[node] = acc / 8.0;
    P->joins++;
    if (P->jrows < P->jcap) {
        double *row = P->jlog + P->jrows * 12;
        row[0] = lvl;
        row[1] = x;
        row[2] = y;
        row[3] = z;
        for (int q = 0; q < 8; ++q) row[4 + q] = P->u[b + q];
        P->jrows++;
    }
}

/* free a joined node's whole subtree, deepest blocks first
 * (_kernels.pyx:357-368) */
static void release_subtree(pass_t *P, int64_t node) {
    int64_t b = P->child[node];
    if (b < 0) return;
    for (int q = 0; q < 8; ++q) {
        release_subtree(P, b + q);
        P->joined[b + q] = 0;
    }
    P->child[node] = -1;
    P->child[b] = (int32_t)P->state[1];
    P->state[1] = b;
    P->state[2] -= 8;
}

/* _kernels.pyx:371-381 */
static void sweep_joined(pass_t *P, int64_t node) {
    int64_t b = P->child[node];
    if (b < 0) return;
    if (P->joined[node]) {
        release_subtree(P, node);
        P->joined[node] = 0;
        return;
    }
    for (int q = 0; q < 8; ++q) sweep_joined(P, b + q);
}

int orc_iterate_pass(double *uval, double *usnap, int32_t *uchild,
                     uint8_t *ujoined, int64_t *ustate, int64_t cap,
                     int nviews, const float *const *vval,
                     const float *const *vw, const int32_t *const *vchild,
                     int d_max, double lam, double eps, double gamma,
                     double xi, double tau_s, double tau_j, int clamp,
                     int reverse, double *jlog, int64_t jcap, int64_t *out3) {
    if (d_max > 60) return ORC_EDEPTH;
    memcpy(usnap, uval, (size_t)ustate[0] * sizeof(double));
    pass_t P;
    memset(&P, 0, sizeof P);
    P.u = uval;
    P.snap = usnap;
    P.child = uchild;
    P.joined = ujoined;
    P.state = ustate;
    P.cap = cap;
    P.nv = nviews;
    P.vval = vval;
    P.vw = vw;
    P.vchild = vchild;
    P.d_max = d_max;
    P.lam = lam;
    P.eps2 = eps * eps;
    P.gamma = gamma;
    P.xi = xi;
    P.tau_s = tau_s;
    P.tau_j = tau_j;
    P.clamp = clamp;
    P.reverse = reverse;
    P.jlog = jcap > 0 ? jlog : NULL;
    P.jcap = jcap > 0 ? jcap : 0;
    P.vcur = (int64_t *)malloc((size_t)(nviews > 0 ? nviews : 1) *
                               (size_t)(d_max + 1) * sizeof(int64_t));
    if (!P.vcur) return ORC_ENOMEM;
    walk(&P, 0, 0, 0, 0, 0);
    if (!P.failed) sweep_joined(&P, 0);
    free(P.vcur);
    if (P.failed) return ORC_EPOOL;
    out3[0] = P.splits;
    out3[1] = P.joins;
    out3[2] = P.jrows;
    return ORC_OK;
}

/* --------------------------------------------------------------- energy --
 * _kernels.pyx:466-578: leaves in depth-first order (children 0..7),
 * per leaf [data/(gamma+sum w) + lam*sqrt(|grad u|^2+eps^2)] * h^3 */
typedef struct {
    const double *u;
    const int32_t *child;
    int nv;
    const float *const *vval;
    const float *const *vw;
    const int32_t *const *vchild;
    int64_t *vcur;
    int d_max;
    double lam, eps2, gamma, total;
} energy_t;

static double value_at(const energy_t *E, int x, int y, int z, int lvl) {
    int64_t n = 0;
    for (int l = 0; l < lvl && E->child[n] >= 0; ++l) {
        int s = lvl - l - 1;
        n = E->child[n] + octant(x >> s, y >> s, z >> s);
    }
    return E->u[n];
}

static void energy_walk(energy_t *E, int64_t node, int x, int y, int z,
                        int lvl) {
    int stride = E->d_max + 1;
    if (lvl == 0) {
        for (int v = 0; v < E->nv; ++v) E->vcur[(int64_t)v * stride] = 0;
    } else {
        int sel = octant(x, y, z);
        for (int v = 0; v < E->nv; ++v) {
            int64_t *row = E->vcur + (int64_t)v * stride;
            int64_t par = row[lvl - 1];
            int64_t b = E->vchild[v][par];
            row[lvl] = b >= 0 ? b + sel : par;
        }
    }
    int64_t b = E->child[node];
    if (b >= 0) {
        for (int q = 0; q < 8; ++q)
            energy_walk(E, b + q, 2 * x + ((q >> 2) & 1),
                        2 * y + ((q >> 1) & 1), 2 * z + (q & 1), lvl + 1);
        return;
    }
    int m = 1 << lvl;
    double h = (double)(1 << (E->d_max - lvl));
    double c = E->u[node];
    double gx = x + 1 < m ? (value_at(E, x + 1, y, z, lvl) - c) / h : 0.0;
    double gy = y + 1 < m ? (value_at(E, x, y + 1, z, lvl) - c) / h : 0.0;
    double gz = z + 1 < m ? (value_at(E, x, y, z + 1, lvl) - c) / h : 0.0;
    double smooth = E->lam * sqrt(gx * gx + gy * gy + gz * gz + E->eps2);
    double num = 0.0, den = E->gamma;
    for (int v = 0; v < E->nv; ++v) {
        int64_t vn = E->vcur[(int64_t)v * stride + lvl];
        double wv = (double)E->vw[v][vn];
        if (wv != 0.0) {
            double d = c - (double)E->vval[v][vn];
            num += wv * sqrt(d * d + E->eps2);
            den += wv;
        }
    }
    E->total += (num / den + smooth) * (h * h * h);
}

int orc_tree_energy(const double *uval, const int32_t *uchild, int nviews,
                    const float *const *vval, const float *const *vw,
                    const int32_t *const *vchild, int d_max, double lam,
                    double eps, double gamma, double *out) {
    if (d_max > 60) return ORC_EDEPTH;
    energy_t E;
    memset(&E, 0, sizeof E);
    E.u = uval;
    E.child = uchild;
    E.nv = nviews;
    E.vval = vval;
    E.vw = vw;
    E.vchild = vchild;
    E.d_max = d_max;
    E.lam = lam;
    E.eps2 = eps * eps;
    E.gamma = gamma;
    E.vcur = (int64_t *)malloc((size_t)(nviews > 0 ? nviews : 1) *
                               (size_t)(d_max + 1) * sizeof(int64_t));
    if (!E.vcur) return ORC_ENOMEM;
    energy_walk(&E, 0, 0, 0, 0, 0);
    free(E.vcur);
    *out = E.total;
    return ORC_OK;
}
