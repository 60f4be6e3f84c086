/*
 * dr_oracle.c — plain, slow, obviously-correct fp64 CPU reference for the
 * DR-CircuitGNN hot path (arXiv 2508.16769).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this. It shares no
 * code, header, table or helper with the CUDA library under
 * paper_2508_16769_b200/ and must never be reached from the product path.
 *
 * Every function is the paper's definition written out as loops, in fp64.
 * Inputs arrive as fp64 arrays (the generator's / GPU's fp32 values promoted
 * exactly). Citations: P:<n> = /root/reference/PAPER.md line n.
 *
 * OpenMP is used only over disjoint output rows, so results do not depend on
 * the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------ normalisers
 * Degree normalisers of the two module kinds (SURVEY §8.0 'Degrees', reading
 * Q12 in DESIGN.md): degrees are unweighted edge counts clamped to >= 1.
 *   module 0 = SageConv mean  : c_i = 1/deg_in(i),        s_j = 1
 *   module 1 = GraphConv both : c_i = deg_in(i)^(-1/2),   s_j = deg_out(j)^(-1/2)
 * rows of the CSR are destinations (Eq. 4 convention). */
void or_normalisers(int64_t n_dst, int64_t n_src, const int64_t *ptr, const int32_t *col,
                    int module, double *c, double *s) {
    int64_t *dout = (int64_t *)calloc((size_t)(n_src > 0 ? n_src : 1), sizeof(int64_t));
    for (int64_t i = 0; i < n_dst; ++i)
        for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) dout[col[e]] += 1;
    for (int64_t i = 0; i < n_dst; ++i) {
        int64_t din = ptr[i + 1] - ptr[i];
        double d = (double)(din < 1 ? 1 : din);
        c[i] = module == 0 ? 1.0 / d : 1.0 / sqrt(d);
    }
    for (int64_t j = 0; j < n_src; ++j) {
        double d = (double)(dout[j] < 1 ? 1 : dout[j]);
        s[j] = module == 0 ? 1.0 : 1.0 / sqrt(d);
    }
    free(dout);
}

/* ------------------------------------------------------------------ D-ReLU
 * Eq. 2-3: th_i = min(topk(X_i,:, k)); keep X_id >= th_i.
 * Exactly k survivors per row (CBSR): ties at the threshold are broken
 * towards the lowest column index (north_star; reading Q5). Kept
 * values are copied verbatim, negatives included (reading Q6).
 * Method: order the columns by the key (-x_d, d) with a plain insertion sort,
 * keep the first k, emit them in ascending column order. -0.0 == +0.0 under
 * C's double comparison, so they tie and fall to column order. */
static int drelu_before(const double *row, int a, int b) {
    if (row[a] > row[b]) return 1;
    if (row[a] < row[b]) return 0;
    return a < b;
}

void or_drelu(const double *x, int64_t n, int d, int64_t ldx, int k, int32_t *idx, double *val) {
#pragma omp parallel
    {
        int *ord = (int *)malloc(sizeof(int) * (size_t)d);
        int *keep = (int *)malloc(sizeof(int) * (size_t)k);
#pragma omp for schedule(static)
        for (int64_t r = 0; r < n; ++r) {
            const double *row = x + r * ldx;
            for (int t = 0; t < d; ++t) ord[t] = t;
            for (int a = 1; a < d; ++a) {          /* insertion sort by (-x, col) */
                int v = ord[a], b = a - 1;
                while (b >= 0 && drelu_before(row, v, ord[b])) { ord[b + 1] = ord[b]; --b; }
                ord[b + 1] = v;
            }
            for (int t = 0; t < k; ++t) keep[t] = ord[t];
            for (int a = 1; a < k; ++a) {          /* ascending column order */
                int v = keep[a], b = a - 1;
                while (b >= 0 && keep[b] > v) { keep[b + 1] = keep[b]; --b; }
                keep[b + 1] = v;
            }
            for (int t = 0; t < k; ++t) {
                idx[r * k + t] = keep[t];
                val[r * k + t] = row[keep[t]];
            }
        }
        free(ord);
        free(keep);
    }
}

/* ------------------------------------------------------------------ DR-SpMM forward
 * Eq. 5-7, Alg. 1 stage 3 with W applied outside
 * (reading Q9): Z_i = c_i * sum_{e in row i} a_e * s_j * densify(H_j),
 * where densify puts H's k kept values at their CBSR indices.
 * a == NULL means unit edge weights (A_ij in R+). */
void or_spmm_fwd(int64_t n_dst, const int64_t *ptr, const int32_t *col, const double *a,
                 const double *c, const double *s, int k, int d,
                 const int32_t *hidx, const double *hval, double *z) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n_dst; ++i) {
        double *zi = z + i * d;
        for (int t = 0; t < d; ++t) zi[t] = 0.0;
        for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
            int64_t j = col[e];
            double w = (a ? a[e] : 1.0) * s[j];
            for (int t = 0; t < k; ++t) zi[hidx[j * k + t]] += w * hval[j * k + t];
        }
        for (int t = 0; t < d; ++t) zi[t] *= c[i];
    }
}

/* ------------------------------------------------------------------ DR-SpMM backward (SSpMM)
 * Eq. 10-11, Alg. 2: dL/dX_j = sum_{i: (i,j) in E}
 * A_ij dL/dY_i, here for the normalised adjacency c_i a_ij s_j and evaluated
 * only at source j's forward-kept CBSR indices (Alg. 2 stage 1, "Reuse
 * preserved ... CBSR indices"):
 *     g[j,t] = sum_{i: (i,j) in E} c_i * a_ij * s_j * dz[i, hidx[j,t]].
 * The transposed edge list (CSC, Alg. 2 stage 1 "Transpose A to CSC") is built
 * here by a plain counting pass so the sum runs over source rows; per-row
 * ownership replaces the paper's atomic add (reading Q23). */
void or_spmm_bwd(int64_t n_dst, int64_t n_src, const int64_t *ptr, const int32_t *col,
                 const double *a, const double *c, const double *s, int k, int d,
                 const int32_t *hidx, const double *dz, double *g) {
    int64_t nnz = ptr[n_dst];
    int64_t *cptr = (int64_t *)calloc((size_t)n_src + 1, sizeof(int64_t));
    int64_t *crow = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    int64_t *cedge = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    int64_t *fill = (int64_t *)calloc((size_t)n_src + 1, sizeof(int64_t));
    for (int64_t e = 0; e < nnz; ++e) cptr[col[e] + 1] += 1;
    for (int64_t j = 0; j < n_src; ++j) cptr[j + 1] += cptr[j];
    for (int64_t i = 0; i < n_dst; ++i)
        for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
            int64_t j = col[e];
            int64_t p = cptr[j] + fill[j]++;
            crow[p] = i;
            cedge[p] = e;
        }
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t j = 0; j < n_src; ++j) {
        for (int t = 0; t < k; ++t) {
            double acc = 0.0;
            int col_t = hidx[j * k + t];
            for (int64_t p = cptr[j]; p < cptr[j + 1]; ++p) {
                int64_t i = crow[p];
                double w = c[i] * (a ? a[cedge[p]] : 1.0) * s[j];
                acc += w * dz[i * d + col_t];
            }
            g[j * k + t] = acc;
        }
    }
    free(cptr); free(crow); free(cedge); free(fill);
}
