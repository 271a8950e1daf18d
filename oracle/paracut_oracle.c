/*
 * paracut_oracle.c -- CPU restatement of the reference AAR chain-prox path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the
 * "port" CPU baseline; the product (paracut_b200/) never links or calls it.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so.
 *
 * What it restates (all citations into /root/reference/pkg/src/paracut/):
 *   orc_taut_string  -- _kernels.py:11-142  weighted 1D-TV prox (taut string
 *                       with convex-hull tube walk, restart at each touch)
 *   orc_prox_chains  -- _kernels.py:145-180 batched CSR gather/prox/scatter
 *   orc_aar_run      -- solvers.py:272-307 + projections.py:89-122, the AAR
 *                       loop z <- z + Pi_L(2 Pi_K z - z) - Pi_K z in the exact
 *                       operation order of the numpy reference (2.0*p - z,
 *                       class-ordered sum, (w - total)/d, (v + corr) - p,
 *                       z += dz), so results are bitwise equal to it.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).  FP
 * contraction must stay off: numba compiles the reference without fastmath
 * (_kernels.py:3-5), so every multiply and add is rounded separately.
 *
 * Parity pin: tests/test_oracle_golden.py checks this restatement bitwise
 * against fixtures produced by running the reference itself
 * (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;

/* Hull scratch for one chain: ceiling (cx, cy) and floor (fx, fy) stacks. */
typedef struct {
    i64 *cx, *fx;
    double *cy, *fy;
} hull_t;

/*
 * One chain: argmin_x 0.5||x - s||^2 + sum_i a_i |x_{i+1} - x_i|.
 * Running sums S_k of s define the tube S_k +- a_k; the cumulative string
 * is walked from an anchor gate, keeping the ceiling hull convex and the
 * floor hull concave.  When one hull crosses the other's cone the string
 * touches the tube at the first point of that hull; the segment from the
 * anchor to it is fixed and the walk restarts there (_kernels.py:33-142).
 */
void orc_taut_string(const double *s, const double *a, i64 m, double *x,
                     i64 *cx, double *cy, i64 *fx, double *fy)
{
    if (m == 1) { x[0] = s[0]; return; }
    i64 anc = 0;          /* anchor gate */
    double anc_y = 0.0;   /* string value at the anchor */
    int anc_side = 0;     /* -1 floor, +1 ceiling, 0 free */
    double anc_sum = 0.0; /* running sum at the anchor gate */
    while (anc < m) {
        i64 nc = 0, nf = 0, k = anc, hit_k = -1;
        double run = anc_sum, hit_y = 0.0;
        int hit_side = 0;
        while (k < m) {
            ++k;
            run += s[k - 1];
            double rad = (k < m) ? a[k - 1] : 0.0;
            /* ceiling point (k, run + rad) */
            double top = run + rad;
            while (nc >= 1) {
                i64 bx; double by;
                if (nc >= 2) { bx = cx[nc - 2]; by = cy[nc - 2]; }
                else { bx = anc; by = anc_y; }
                i64 tx = cx[nc - 1]; double ty = cy[nc - 1];
                if ((ty - by) * (double)(k - tx) >= (top - ty) * (double)(tx - bx)) --nc;
                else break;
            }
            cx[nc] = k; cy[nc] = top; ++nc;
            if (nf >= 1 && (cy[0] - anc_y) * (double)(fx[0] - anc)
                               < (fy[0] - anc_y) * (double)(cx[0] - anc)) {
                hit_k = fx[0]; hit_y = fy[0]; hit_side = -1;
                break;
            }
            /* floor point (k, run - rad) */
            double bot = run - rad;
            while (nf >= 1) {
                i64 bx; double by;
                if (nf >= 2) { bx = fx[nf - 2]; by = fy[nf - 2]; }
                else { bx = anc; by = anc_y; }
                i64 tx = fx[nf - 1]; double ty = fy[nf - 1];
                if ((ty - by) * (double)(k - tx) <= (bot - ty) * (double)(tx - bx)) --nf;
                else break;
            }
            fx[nf] = k; fy[nf] = bot; ++nf;
            if ((fy[0] - anc_y) * (double)(cx[0] - anc) > (cy[0] - anc_y) * (double)(fx[0] - anc)) {
                hit_k = cx[0]; hit_y = cy[0]; hit_side = 1;
                break;
            }
        }
        if (hit_k < 0) {
            /* end of chain: the end point S_m is mandatory (_kernels.py:97-114) */
            if (cx[0] != m && (cy[0] - anc_y) * (double)(m - anc) < (run - anc_y) * (double)(cx[0] - anc)) {
                hit_k = cx[0]; hit_y = cy[0]; hit_side = 1;
            } else if (fx[0] != m && (fy[0] - anc_y) * (double)(m - anc) > (run - anc_y) * (double)(fx[0] - anc)) {
                hit_k = fx[0]; hit_y = fy[0]; hit_side = -1;
            } else {
                hit_k = m; hit_y = run; hit_side = 0;
            }
        }
        /* constant segment [anc, hit_k): fresh sum plus tube offsets */
        double first = s[anc], tot = 0.0;
        int flat = 1;
        for (i64 j = anc; j < hit_k; ++j) {
            tot += s[j];
            if (s[j] != first) flat = 0;
        }
        double off = 0.0;
        if (hit_side != 0) off += (double)hit_side * a[hit_k - 1];
        if (anc_side != 0) off -= (double)anc_side * a[anc - 1];
        double val = (flat && off == 0.0) ? first : (tot + off) / (double)(hit_k - anc);
        for (i64 j = anc; j < hit_k; ++j) x[j] = val;
        anc = hit_k;
        anc_y = hit_y;
        anc_side = hit_side;
        anc_sum = (hit_side == 0) ? hit_y : hit_y - (double)hit_side * a[hit_k - 1];
    }
}

static int alloc_hull(hull_t *h, i64 m)
{
    h->cx = (i64 *)malloc(sizeof(i64) * (size_t)(m + 1));
    h->fx = (i64 *)malloc(sizeof(i64) * (size_t)(m + 1));
    h->cy = (double *)malloc(sizeof(double) * (size_t)(m + 1));
    h->fy = (double *)malloc(sizeof(double) * (size_t)(m + 1));
    return h->cx && h->fx && h->cy && h->fy;
}

static void free_hull(hull_t *h)
{
    free(h->cx); free(h->fx); free(h->cy); free(h->fy);
}

/* Chains [c_lo, c_hi) of one class; scratch is per call (_kernels.py:145-180). */
static void prox_range(const i64 *node_idx, const i64 *chain_ptr, const double *edge_w,
                       i64 c_lo, i64 c_hi, const double *v, double *out, int as_projection)
{
    i64 maxm = 0;
    for (i64 c = c_lo; c < c_hi; ++c) {
        i64 mm = chain_ptr[c + 1] - chain_ptr[c];
        if (mm > maxm) maxm = mm;
    }
    if (maxm == 0) return;
    double *sig = (double *)malloc(sizeof(double) * (size_t)maxm);
    double *px = (double *)malloc(sizeof(double) * (size_t)maxm);
    hull_t h;
    alloc_hull(&h, maxm);
    for (i64 c = c_lo; c < c_hi; ++c) {
        i64 b = chain_ptr[c], mm = chain_ptr[c + 1] - b;
        const i64 *ids = node_idx + b;
        for (i64 i = 0; i < mm; ++i) sig[i] = v[ids[i]];
        orc_taut_string(sig, edge_w + (b - c), mm, px, h.cx, h.cy, h.fx, h.fy);
        if (as_projection)
            for (i64 i = 0; i < mm; ++i) out[ids[i]] = sig[i] - px[i];
        else
            for (i64 i = 0; i < mm; ++i) out[ids[i]] = px[i];
    }
    free(sig); free(px); free_hull(&h);
}

void orc_prox_chains(const i64 *node_idx, const i64 *chain_ptr, const double *edge_w,
                     i64 c_lo, i64 c_hi, const double *v, double *out, int as_projection)
{
    prox_range(node_idx, chain_ptr, edge_w, c_lo, c_hi, v, out, as_projection);
}

/* Thread-parallel variant: contiguous blocks of chains, like ChainPool. */
void orc_prox_chains_mt(const i64 *node_idx, const i64 *chain_ptr, const double *edge_w,
                        i64 nchains, const double *v, double *out, int as_projection,
                        int threads)
{
    if (threads < 1) threads = 1;
    if (threads > nchains) threads = (int)(nchains > 0 ? nchains : 1);
#ifdef _OPENMP
#pragma omp parallel for num_threads(threads) schedule(static, 1)
#endif
    for (int b = 0; b < threads; ++b) {
        i64 lo = nchains * b / threads, hi = nchains * (b + 1) / threads;
        prox_range(node_idx, chain_ptr, edge_w, lo, hi, v, out, as_projection);
    }
}

/* Batched tv1d over a CSR of independent signals (tv1d.py:42-69). */
void orc_tv1d_batch(const double *s, const double *a, const i64 *ptr, i64 nchains, double *x)
{
    for (i64 c = 0; c < nchains; ++c) {
        i64 b = ptr[c], m = ptr[c + 1] - b;
        if (m <= 0) continue;
        hull_t h;
        alloc_hull(&h, m);
        orc_taut_string(s + b, a + (b - c), m, x + b, h.cx, h.cy, h.fx, h.fy);
        free_hull(&h);
    }
}

/*
 * Decomposition handed over from Python as r CSR classes, concatenated:
 * class j owns node_idx[node_off[j] .. node_off[j+1]), chain_ptr rows
 * [cp_off[j] .. cp_off[j+1]] (values relative to its own node_idx block),
 * edge_w[ew_off[j] ..).
 */
typedef struct {
    int r;
    i64 n;
    const i64 *node_idx, *node_off;
    const i64 *chain_ptr, *cp_off;
    const double *edge_w;
    const i64 *ew_off;
} orc_dec_t;

static void project_K(const orc_dec_t *d, const double *v, double *out, int threads)
{
    memset(out, 0, sizeof(double) * (size_t)d->r * (size_t)d->n);
    for (int j = 0; j < d->r; ++j) {
        i64 nch = d->cp_off[j + 1] - d->cp_off[j] - 1;
        if (nch <= 0) continue;
        orc_prox_chains_mt(d->node_idx + d->node_off[j], d->chain_ptr + d->cp_off[j],
                           d->edge_w + d->ew_off[j], nch, v + (size_t)j * d->n,
                           out + (size_t)j * d->n, 1, threads);
    }
}

/*
 * AAR in fixed-iteration form.  On entry z holds the AAR point z^0; on exit
 * z = z^iters and, if final_shadow, p = Pi_K(z^iters) (the shadow the
 * reference reports as DualState.y).  step_norm[k] = ||z^{k+1} - z^k|| (monitor aar_step_norm).
 * degree is r on every grid decomposition (test_projections.py:60).
 */
void orc_aar_run(int r, i64 n, const i64 *node_idx, const i64 *node_off,
                 const i64 *chain_ptr, const i64 *cp_off, const double *edge_w,
                 const i64 *ew_off, const double *w, double *z, double *p,
                 i64 iters, double *step_norm, int threads, int final_shadow)
{
    orc_dec_t d = {r, n, node_idx, node_off, chain_ptr, cp_off, edge_w, ew_off};
    const double deg = (double)r;
    for (i64 k = 0; k < iters; ++k) {
        project_K(&d, z, p, threads);
        double nrm2 = 0.0;
#ifdef _OPENMP
#pragma omp parallel for num_threads(threads) reduction(+ : nrm2) schedule(static)
#endif
        for (i64 i = 0; i < n; ++i) {
            double v[8];
            double total = 0.0;
            for (int j = 0; j < r; ++j) {
                v[j] = 2.0 * p[(size_t)j * n + i] - z[(size_t)j * n + i];
                total = (j == 0) ? v[0] : total + v[j];
            }
            double corr = (w[i] - total) / deg;
            for (int j = 0; j < r; ++j) {
                double dz = (v[j] + corr) - p[(size_t)j * n + i];
                z[(size_t)j * n + i] += dz;
                nrm2 += dz * dz;
            }
        }
        if (step_norm) step_norm[k] = sqrt(nrm2);
    }
    if (final_shadow) project_K(&d, z, p, threads);
}

int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
