/* CPU ORACLE -- TEST INFRASTRUCTURE ONLY.  Never linked into the product.
 *
 * Businger-Golub pivoted Householder QR, Alg. 2 step 3 of arXiv 2011.07632
 * ("pivoted QR decomposition Psi P = QR"), with the rules of
 * reading R4: residual column norms RECOMPUTED at every step (no downdating),
 * ties to the lowest column index, stop at t = max_rank or at the first t with
 * |R_tt| <= rel_tol |R_00| (|R_tt| is the largest residual norm at step t),
 * Householder vectors chosen so that R_tt >= 0 (Golub & Van Loan Alg. 5.1.1).
 *
 * Plain loops; OpenMP only across independent columns of one step.
 * A: m x n column-major (lda = m), overwritten by R (upper part, pivoted
 * column order) and the Householder vectors below the diagonal (v_0 = 1
 * implicit).  piv[n] receives the column permutation, beta[min(m,n)] the
 * reflector coefficients.  Returns the rank r.
 */
#include <math.h>
#include <string.h>
#include <stdlib.h>

static void house(int len, double *x, double *beta)
{
    /* on exit x[0] = ||x|| (>= 0), x[1..] = v[1..] with v[0] = 1 */
    double sigma = 0.0;
    for (int i = 1; i < len; ++i) sigma += x[i] * x[i];
    double x0 = x[0];
    if (sigma == 0.0) {
        *beta = (x0 >= 0.0) ? 0.0 : 2.0;
        x[0] = fabs(x0);
        return;
    }
    double mu = sqrt(x0 * x0 + sigma);
    double v0 = (x0 <= 0.0) ? x0 - mu : -sigma / (x0 + mu);
    *beta = 2.0 * v0 * v0 / (sigma + v0 * v0);
    for (int i = 1; i < len; ++i) x[i] /= v0;
    x[0] = mu;
}

/* Follow mode (certified-tie protocol, reading R19): when follow != NULL the pivot
 * of step t < nfollow is the column whose ORIGINAL index is follow[t] (the pivots of
 * another implementation) instead of the argmax, and the factorization stops after
 * nfollow steps.  In both modes numax[t] (t <= rank, nullable) receives the largest
 * residual column norm at step t, nuf[t] (nullable) the norm of the column taken, and
 * nu2[t] / idx2[t] (nullable) the runner-up norm and its original column index;
 * the arithmetic of a step is the same.  Returns -1 if follow[t] is not a remaining
 * column. */
int oracle_qrcp_follow(int m, int n, double *A, int max_rank, double rel_tol,
                       int *piv, double *beta, const int *follow, int nfollow,
                       double *numax, double *nuf, double *nu2, int *idx2)
{
    int kmax = m < n ? m : n;
    if (max_rank < kmax) kmax = max_rank;
    double *norms = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
    double *v = (double *)malloc(sizeof(double) * (m > 0 ? m : 1));
    for (int j = 0; j < n; ++j) piv[j] = j;
    double nu0 = 0.0;
    int r = 0;
    for (int t = 0; t < kmax; ++t) {
        #pragma omp parallel for schedule(static)
        for (int j = t; j < n; ++j) {
            const double *c = A + (size_t)j * m;
            double s = 0.0;
            for (int i = t; i < m; ++i) s += c[i] * c[i];
            norms[j] = sqrt(s);
        }
        int p = t;
        for (int j = t + 1; j < n; ++j)
            if (norms[j] > norms[p]) p = j;          /* strict: lowest index wins ties */
        double nu = norms[p];
        if (t == 0) nu0 = nu;
        if (numax) numax[t] = nu;
        if (nu2) {                                   /* runner-up (lowest index on ties) */
            int q2 = -1;
            for (int j = t; j < n; ++j)
                if (j != p && (q2 < 0 || norms[j] > norms[q2])) q2 = j;
            nu2[t] = q2 < 0 ? -1.0 : norms[q2];
            if (idx2) idx2[t] = q2 < 0 ? -1 : piv[q2];
        }
        if (follow) {
            if (t >= nfollow) break;
            int q = -1;
            for (int j = t; j < n; ++j)
                if (piv[j] == follow[t]) { q = j; break; }
            if (q < 0) { r = -1; break; }
            p = q;
            if (nuf) nuf[t] = norms[p];
        } else {
            if (nuf) nuf[t] = nu;
            if (nu == 0.0 || nu <= rel_tol * nu0) break;
        }
        if (p != t) {
            double *a = A + (size_t)t * m, *b = A + (size_t)p * m;
            for (int i = 0; i < m; ++i) { double tmp = a[i]; a[i] = b[i]; b[i] = tmp; }
            int tp = piv[t]; piv[t] = piv[p]; piv[p] = tp;
        }
        double *ct = A + (size_t)t * m;
        double bt;
        house(m - t, ct + t, &bt);
        beta[t] = bt;
        v[t] = 1.0;
        for (int i = t + 1; i < m; ++i) v[i] = ct[i];
        #pragma omp parallel for schedule(static)
        for (int j = t + 1; j < n; ++j) {
            double *c = A + (size_t)j * m;
            double w = 0.0;
            for (int i = t; i < m; ++i) w += v[i] * c[i];
            w *= bt;
            for (int i = t; i < m; ++i) c[i] -= w * v[i];
        }
        r = t + 1;
    }
    free(norms);
    free(v);
    return r;
}

int oracle_qrcp(int m, int n, double *A, int max_rank, double rel_tol,
                int *piv, double *beta)
{
    return oracle_qrcp_follow(m, n, A, max_rank, rel_tol, piv, beta, NULL, 0, NULL, NULL, NULL, NULL);
}
