/*
 * CPU restatement of the TV-L1 primal-dual pass -- TEST INFRASTRUCTURE ONLY.
 *
 * PARITY UNPINNED: the reference has no primal-dual solver (
 * PAPER.md:315 names it as future work).  This file is the written-down
 * definition the GPU's solver="pd" mode is checked against; it is not a
 * restatement of reference code.  Definition (per pass, Jacobi on a frozen
 * tree, every leaf at its own level L with spacing h = 2^(d_max-L) in
 * finest-cell units, lookups as in the reference's descent,
 * _kernels.pyx:193-202):
 *
 *   energy   E(u) = sum_leaves h^3 [ lam |grad u| + sum_i w_i|u-f_i| / (W+gamma) ]
 *   dual     p'(q) = P( p(q) + sigma*lam * grad ubar(q) ),  P = projection
 *            onto the unit ball, grad = forward differences (0 at the border)
 *   primal   v = u + tau*lam * div p',  div = backward differences of p' at
 *            level L (p' of a backward neighbour evaluated at level L)
 *            u' = prox_{tau D}(v) = argmin_x (x-v)^2/2 + c sum_i w_i|x-f_i|,
 *            c = tau/(W+gamma): generalised weighted median, samples sorted
 *            by (f, view index); a -0 sample is taken as +0 (so the sorted
 *            values do not depend on how a sort orders equal keys).  Every
 *            per-leaf sum (W, the energy's data term) runs over the samples
 *            in this sorted order: the GPU sorts each leaf's samples once
 *            when they are gathered and keeps them sorted.
 *   extrapolation  ubar' = 2u' - u;  u' clamped to [-1,1] when clamp.
 * Inner nodes of u, ubar, p are child means (propagate) after every pass.
 * Built with -ffp-contract=off; the GPU's f64 mode keeps this exact order.
 *
 * What ties it to the reference (tests/test_pd_energy_pin.py): E(u) equals
 * the reference's energy (octfuse_oracle.c orc_tree_energy, pinned to the
 * reference's fixtures) at eps = 1e-9 on the states a run visits, and the
 * prox is checked as the minimiser of its objective.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "octfuse_oracle.h"

static inline int octant3(int x, int y, int z) {
    return ((x & 1) << 2) | ((y & 1) << 1) | (z & 1);
}

static int64_t node_at(const int32_t *child, int L, int x, int y, int z) {
    int64_t n = 0;
    for (int l = 0; l < L && child[n] >= 0; ++l) {
        int s = L - l - 1;
        n = child[n] + octant3(x >> s, y >> s, z >> s);
    }
    return n;
}

typedef struct {
    const double *u, *ub, *px, *py, *pz;
    const int32_t *child;
    int d_max;
    double lam, tau, sigma, gamma;
} pd_in;

/* dual at cell q of level L (evaluated at that level) */
static void dual_at(const pd_in *I, int L, int x, int y, int z, double out[3]) {
    int m = 1 << L;
    double h = (double)(1 << (I->d_max - L));
    int64_t q = node_at(I->child, L, x, y, z);
    double c = I->ub[q];
    double gx = 0.0, gy = 0.0, gz = 0.0;
    if (x + 1 < m) gx = (I->ub[node_at(I->child, L, x + 1, y, z)] - c) / h;
    if (y + 1 < m) gy = (I->ub[node_at(I->child, L, x, y + 1, z)] - c) / h;
    if (z + 1 < m) gz = (I->ub[node_at(I->child, L, x, y, z + 1)] - c) / h;
    double sl = I->sigma * I->lam;
    double ax = I->px[q] + sl * gx;
    double ay = I->py[q] + sl * gy;
    double az = I->pz[q] + sl * gz;
    double nrm = sqrt(ax * ax + ay * ay + az * az);
    double s = nrm > 1.0 ? nrm : 1.0;
    out[0] = ax / s;
    out[1] = ay / s;
    out[2] = az / s;
}

/* prox of c*sum w_i|x-f_i| at v over n samples sorted ascending */
static double wmedian_prox(const double *f, const double *w, int n, double W,
                           double v, double c) {
    double S = 0.0;
    for (int k = 0; k <= n; ++k) {
        double cand = v - c * (2.0 * S - W);
        if (k > 0 && cand < f[k - 1]) return f[k - 1];
        if (k == n || cand <= f[k]) return cand;
        S += w[k];
    }
    return v; /* unreachable */
}

static void walk_leaves(const int32_t *child, int64_t node, int L, int x, int y,
                        int z, int64_t *nodes, int *lv, int *cx, int *cy,
                        int *cz, int64_t *count) {
    int64_t b = child[node];
    if (b < 0) {
        nodes[*count] = node;
        lv[*count] = L;
        cx[*count] = x;
        cy[*count] = y;
        cz[*count] = z;
        (*count)++;
        return;
    }
    for (int q = 0; q < 8; ++q)
        walk_leaves(child, b + q, L + 1, 2 * x + ((q >> 2) & 1),
                    2 * y + ((q >> 1) & 1), 2 * z + (q & 1), nodes, lv, cx, cy,
                    cz, count);
}

/* one pass; *_o outputs hold the new leaf values (inner nodes untouched).
 * Returns the energy of the incoming state u in *energy. */
int orc_pd_pass(const double *u, const double *ub, const double *px,
                const double *py, const double *pz, double *u_o, double *ub_o,
                double *px_o, double *py_o, double *pz_o,
                const int32_t *child, int64_t used, int nviews,
                const float *const *vval, const float *const *vw,
                const int32_t *const *vchild, int d_max, double lam, double tau,
                double sigma, double gamma, int clamp, double *energy) {
    if (d_max > 60) return ORC_EDEPTH;
    int64_t *nodes = (int64_t *)malloc((size_t)used * sizeof(int64_t));
    int *lv = (int *)malloc((size_t)used * sizeof(int));
    int *cx = (int *)malloc((size_t)used * sizeof(int));
    int *cy = (int *)malloc((size_t)used * sizeof(int));
    int *cz = (int *)malloc((size_t)used * sizeof(int));
    double *fs = (double *)malloc((size_t)(nviews + 1) * sizeof(double));
    double *ws = (double *)malloc((size_t)(nviews + 1) * sizeof(double));
    int *ix = (int *)malloc((size_t)(nviews + 1) * sizeof(int));
    if (!nodes || !lv || !cx || !cy || !cz || !fs || !ws || !ix) {
        free(nodes); free(lv); free(cx); free(cy); free(cz);
        free(fs); free(ws); free(ix);
        return ORC_ENOMEM;
    }
    int64_t nl = 0;
    walk_leaves(child, 0, 0, 0, 0, 0, nodes, lv, cx, cy, cz, &nl);
    pd_in I = {u, ub, px, py, pz, child, d_max, lam, tau, sigma, gamma};
    double total = 0.0;
    for (int64_t j = 0; j < nl; ++j) {
        int64_t n = nodes[j];
        int L = lv[j], x = cx[j], y = cy[j], z = cz[j];
        int m = 1 << L;
        double h = (double)(1 << (d_max - L));
        /* samples at the leaf's level (view order), then sorted */
        int ns = 0;
        for (int v = 0; v < nviews; ++v) {
            int64_t vn = node_at(vchild[v], L, x, y, z);
            double w = (double)vw[v][vn];
            if (w != 0.0) {
                fs[ns] = (double)vval[v][vn] + 0.0; /* -0 -> +0 */
                ws[ns] = w;
                ix[ns] = v;
                ns++;
            }
        }
        /* insertion sort by (f, view index) */
        for (int a = 1; a < ns; ++a) {
            double ff = fs[a], ww = ws[a];
            int ii = ix[a], b = a - 1;
            while (b >= 0 && (fs[b] > ff || (fs[b] == ff && ix[b] > ii))) {
                fs[b + 1] = fs[b];
                ws[b + 1] = ws[b];
                ix[b + 1] = ix[b];
                b--;
            }
            fs[b + 1] = ff;
            ws[b + 1] = ww;
            ix[b + 1] = ii;
        }
        /* weight sum in sorted order (the GPU keeps each leaf's samples
         * sorted once, so every per-leaf sum below runs in that order) */
        double W = 0.0;
        for (int k = 0; k < ns; ++k) W += ws[k];
        double den = W + gamma;
        /* energy of the incoming u */
        {
            double c0 = u[n];
            double gx = x + 1 < m ? (u[node_at(child, L, x + 1, y, z)] - c0) / h : 0.0;
            double gy = y + 1 < m ? (u[node_at(child, L, x, y + 1, z)] - c0) / h : 0.0;
            double gz = z + 1 < m ? (u[node_at(child, L, x, y, z + 1)] - c0) / h : 0.0;
            double tv = lam * sqrt(gx * gx + gy * gy + gz * gz);
            double num = 0.0; /* sorted order */
            for (int k = 0; k < ns; ++k) num += ws[k] * fabs(c0 - fs[k]);
            total += (num / den + tv) * (h * h * h);
        }
        double P[3], B[3];
        dual_at(&I, L, x, y, z, P);
        double bx = 0.0, by = 0.0, bz = 0.0;
        if (x > 0) { dual_at(&I, L, x - 1, y, z, B); bx = B[0]; }
        if (y > 0) { dual_at(&I, L, x, y - 1, z, B); by = B[1]; }
        if (z > 0) { dual_at(&I, L, x, y, z - 1, B); bz = B[2]; }
        double div = ((P[0] - bx) + (P[1] - by) + (P[2] - bz)) / h;
        double v0 = u[n] + (tau * lam) * div;
        double xn = wmedian_prox(fs, ws, ns, W, v0, tau / den);
        if (clamp) xn = xn > 1.0 ? 1.0 : (xn < -1.0 ? -1.0 : xn);
        u_o[n] = xn;
        ub_o[n] = 2.0 * xn - u[n];
        px_o[n] = P[0];
        py_o[n] = P[1];
        pz_o[n] = P[2];
    }
    *energy = total;
    free(nodes); free(lv); free(cx); free(cy); free(cz);
    free(fs); free(ws); free(ix);
    return ORC_OK;
}

/* ------------------------------------------------------- restructuring --
 * solver="pd" with split/join (north_star item (d): "split/join
 * restructuring after each step, which flags leaves by their |u| band").
 * Definition (PARITY UNPINNED -- the reference has no primal-dual mode), run
 * after a pass and the propagate of u, ubar, p:
 *   split  a leaf at level L < d_max with |u| < tau_s gets eight children
 *          carrying its u, ubar, p (no cascade within a pass);
 *   join   an inner node whose eight children are leaves, each with
 *          |u| > tau_j and all of one sign, becomes a leaf; its u, ubar, p
 *          are the children's means (sequential f64 sum / 8, i.e. the
 *          propagated values) and its child block is freed.
 * With 0 <= tau_s < tau_j (FusionParams validation) no node both splits and
 * joins.  Visit order and slot allocation are the descent's
 * (_kernels.pyx:256-381, orc_iterate_pass above): depth-first children
 * 0..7, a split claims the free-list head else the bump pointer, joined
 * blocks are pushed in visit order after the walk. */
typedef struct {
    double *f[5];
    int32_t *child;
    uint8_t *joined;
    int64_t *state;
    int64_t cap;
    int d_max;
    double tau_s, tau_j;
    int64_t splits, joins;
    int failed;
} pdr_t;

static int64_t pdr_claim(pdr_t *R) {
    int64_t head = R->state[1], b;
    if (head >= 0) {
        b = head;
        R->state[1] = R->child[b];
    } else {
        b = R->state[0];
        if (b + 8 > R->cap) return -1;
        R->state[0] = b + 8;
    }
    R->state[2] += 8;
    return b;
}

static void pdr_walk(pdr_t *R, int64_t node, int lvl) {
    if (R->failed) return;
    int64_t b = R->child[node];
    if (b < 0) {
        if (lvl < R->d_max && fabs(R->f[0][node]) < R->tau_s) {
            int64_t nb = pdr_claim(R);
            if (nb < 0) {
                R->failed = 1;
                return;
            }
            for (int q = 0; q < 8; ++q) {
                for (int k = 0; k < 5; ++k) R->f[k][nb + q] = R->f[k][node];
                R->child[nb + q] = -1;
            }
            R->child[node] = (int32_t)nb;
            R->splits++;
        }
        return;
    }
    for (int q = 0; q < 8; ++q) pdr_walk(R, b + q, lvl + 1);
    if (R->failed) return;
    int pos = 0, neg = 0;
    for (int q = 0; q < 8; ++q) {
        if (R->child[b + q] >= 0) return;
        double v = R->f[0][b + q];
        if (!(v > R->tau_j || v < -R->tau_j)) return;
        if (v > 0.0)
            pos = 1;
        else
            neg = 1;
    }
    if (pos && neg) return;
    for (int k = 0; k < 5; ++k) {
        double acc = 0.0;
        for (int q = 0; q < 8; ++q) acc += R->f[k][b + q];
        R->f[k][node] = acc / 8.0;
    }
    R->joined[node] = 1;
    R->joins++;
}

static void pdr_sweep(pdr_t *R, int64_t node) {
    int64_t b = R->child[node];
    if (b < 0) return;
    if (R->joined[node]) {
        R->joined[node] = 0;
        R->child[node] = -1;
        R->child[b] = (int32_t)R->state[1];
        R->state[1] = b;
        R->state[2] -= 8;
        return;
    }
    for (int q = 0; q < 8; ++q) pdr_sweep(R, b + q);
}

int orc_pd_restructure(double *u, double *ub, double *px, double *py,
                       double *pz, int32_t *child, int64_t *state, int64_t cap,
                       int d_max, double tau_s, double tau_j, int64_t *out2) {
    if (d_max > 60) return ORC_EDEPTH;
    pdr_t R = {{u, ub, px, py, pz}, child, NULL, state, cap, d_max,
               tau_s, tau_j, 0, 0, 0};
    R.joined = (uint8_t *)calloc((size_t)cap, 1);
    if (!R.joined) return ORC_ENOMEM;
    pdr_walk(&R, 0, 0);
    if (!R.failed) pdr_sweep(&R, 0);
    free(R.joined);
    if (R.failed) return ORC_EPOOL;
    out2[0] = R.splits;
    out2[1] = R.joins;
    return ORC_OK;
}
