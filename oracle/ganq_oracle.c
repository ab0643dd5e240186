/*
 * ganq_oracle.c -- plain, slow, fp64 CPU oracle for GANQ (arxiv 2501.12956).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2501_12956_b200/csrc).  The product never calls it.
 *
 * Every function follows a passage of the paper (P:n = /root/reference/PAPER.md
 * line n) step by step, in the paper's order and notation.  Readings where the
 * paper is silent or garbled are the ones listed in DESIGN.md ("Readings") and
 * are tagged [R-x] below.  Arithmetic is fp64 except where a reading fixes fp32
 * (the initial codebook T^0, [R-6]).  Compile with -ffp-contract=off so that no
 * fused multiply-add changes a rounding the reading fixes.
 *
 * Parallelism: OpenMP over independent rows only (Eq. 2 decomposes the
 * problem into m independent sub-problems), so results do not depend on
 * the thread count.
 *
 * Pins (tests/test_oracle_pins.py): every function here is checked against
 * something other than itself -- numpy library routines, closed forms,
 * brute-force enumeration, the reverse-order GPTQ/OBS formulation of the
 * S-step, 1-D Lloyd for H = I.  See DESIGN.md "Oracle pins".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

#define OR_MAXLEV 256

/* ------------------------------------------------------------------------- */
/* bf16 -> double, exact (a bf16 is the top 16 bits of an IEEE binary32).     */
static double bf16_to_double(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

/*
 * H = X X^T  (Algorithm 1 line "Compute H = XX^T"; X in R^{n x p}).
 * Our X is stored token-major, p x n (row t is the activation x_t), so
 * H_jk = sum_t X[t][j] * X[t][k].  Symmetrised (H + H^T)/2 (it is symmetric
 * by construction; the loop below computes j >= k and mirrors it).
 */
int or_hessian_bf16(const uint16_t *X, int64_t p, int64_t n, double *H) {
    if (p < 1 || n < 1) return 1;
    double *Xd = (double *)malloc(sizeof(double) * (size_t)(p * n));
    if (!Xd) return 3;
    for (int64_t i = 0; i < p * n; ++i) Xd[i] = bf16_to_double(X[i]);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t k = 0; k <= j; ++k) {
            double s = 0.0;
            for (int64_t t = 0; t < p; ++t) s += Xd[t * n + j] * Xd[t * n + k];
            H[j * n + k] = s;
            H[k * n + j] = s;
        }
    }
    free(Xd);
    return 0;
}

/*
 * Preconditioning before Cholesky.
 *   policy 0 = ADAPTIVE (App. A, Eqs. 23-24):
 *       delta_i = max( sum_j |Sigma_ij| - 2 Sigma_ii , 1e-8 )       (Eq. 23)
 *     plus the jitter tau * mean(diag Sigma) on every delta_i       [R-3]
 *     (the literal delta only reaches *weak* dominance, which can be singular);
 *     H' = Sigma + Diag(delta)                                        (Eq. 24)
 *   policy 1 = FIXED_LAMBDA (Remark 1): H' = H + lambda I, lambda > 0
 *   policy 2 = NONE (Algorithm 1 literally): H' = H
 * delta (nullable) receives the diagonal offset actually added.
 */
int or_precondition(const double *H, int64_t n, int policy, double lambda, double tau,
                    double *Hp, double *delta) {
    if (n < 1) return 1;
    if (policy == 1 && !(lambda > 0.0)) return 1;
    if (policy < 0 || policy > 2) return 1;
    memcpy(Hp, H, sizeof(double) * (size_t)(n * n));
    double jitter = 0.0;
    if (policy == 0) {
        double md = 0.0;
        for (int64_t i = 0; i < n; ++i) md += H[i * n + i];
        md /= (double)n;
        jitter = tau * md;
    }
    for (int64_t i = 0; i < n; ++i) {
        double d = 0.0;
        if (policy == 0) {
            double rs = 0.0;
            for (int64_t j = 0; j < n; ++j) rs += fabs(H[i * n + j]);
            d = rs - 2.0 * H[i * n + i];
            if (d < 1e-8) d = 1e-8;
            d += jitter;
        } else if (policy == 1) {
            d = lambda;
        }
        Hp[i * n + i] += d;
        if (delta) delta[i] = d;
    }
    return 0;
}

/*
 * Cholesky  H' = L L^T  (Eq. 9), textbook unblocked column form,
 * reading only the lower triangle.  Returns -1 on success, otherwise the index
 * of the first non-positive pivot (the matrix is not positive definite).
 */
int64_t or_cholesky(const double *A, int64_t n, double *L) {
    memset(L, 0, sizeof(double) * (size_t)(n * n));
    for (int64_t j = 0; j < n; ++j) {
        double s = A[j * n + j];
        for (int64_t k = 0; k < j; ++k) s -= L[j * n + k] * L[j * n + k];
        if (!(s > 0.0)) return j;
        double ljj = sqrt(s);
        L[j * n + j] = ljj;
#pragma omp parallel for schedule(static)
        for (int64_t i = j + 1; i < n; ++i) {
            double t = A[i * n + j];
            for (int64_t k = 0; k < j; ++k) t -= L[i * n + k] * L[j * n + k];
            L[i * n + j] = t / ljj;
        }
    }
    return -1;
}

/*
 * Initial codebook T^0 (Algorithm 1 input; construction unspecified).
 * [R-6]: per-row uniform min-max grid computed in fp32:
 *     step = (max_i - min_i) / (2^N - 1);  t_s = min_i + s * step
 * (each operation rounded to fp32, no fused multiply-add).  A constant row
 * gives all levels equal to that constant.
 */
void or_init_codebook(const float *W, int64_t m, int64_t n, int nlev, float *T0) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        float mn = W[i * n], mx = W[i * n];
        for (int64_t j = 1; j < n; ++j) {
            float w = W[i * n + j];
            if (w < mn) mn = w;
            if (w > mx) mx = w;
        }
        float range = mx - mn;
        float step = range / (float)(nlev - 1);
        for (int s = 0; s < nlev; ++s) {
            float prod = (float)s * step;
            T0[i * nlev + s] = mn + prod;
        }
    }
}

/* argmin_s |z - t_s|, first (smallest) index on ties: strict '<' scan [R-7]. */
static int argmin_level(double z, const double *t, int nlev) {
    int best = 0;
    double bd = fabs(z - t[0]);
    for (int s = 1; s < nlev; ++s) {
        double d = fabs(z - t[s]);
        if (d < bd) { bd = d; best = s; }
    }
    return best;
}

/*
 * S-step: back-substitution (Eqs. 15-22; Algorithm 1 inner loop,
 * P:224-230), every row independently.  For j = n-1 down to 0:
 *     idx = argmin_s | W_ij + (1/L_jj) sum_{u=j+1}^{n-1} r_u L_uj - T_is |   (Eq. 22)
 *     Q_ij = idx,   r_j = W_ij - T_{i,idx}
 * The suffix sum is the literal dot product of Eq. 22 in ascending u; the
 * value Algorithm 1 computes "at j = 0" for column -1 is never formed [R-2].
 * L is given row-major; LT (n x n, scratch) holds its transpose so that the
 * column L_{:,j} is contiguous (a layout choice, not an arithmetic one).
 * Rerr (nullable, m x n) receives r_ij.
 */
void or_sstep(const double *W, const double *L, const double *T, int64_t m, int64_t n,
              int nlev, uint8_t *Q, double *Rerr) {
    double *LT = (double *)malloc(sizeof(double) * (size_t)(n * n));
    for (int64_t u = 0; u < n; ++u)
        for (int64_t j = 0; j < n; ++j) LT[j * n + u] = L[u * n + j];
#pragma omp parallel
    {
        double *r = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < m; ++i) {
            const double *Wi = W + i * n;
            const double *Ti = T + i * nlev;
            for (int64_t j = n - 1; j >= 0; --j) {
                const double *Lcol = LT + j * n; /* Lcol[u] = L_uj */
                double s = 0.0;
                for (int64_t u = j + 1; u < n; ++u) s += r[u] * Lcol[u];
                double z = Wi[j] + s / Lcol[j];
                int q = argmin_level(z, Ti, nlev);
                Q[i * n + j] = (uint8_t)q;
                r[j] = Wi[j] - Ti[q];
                if (Rerr) Rerr[i * n + j] = r[j];
            }
        }
        free(r);
    }
    free(LT);
}

/*
 * Teacher-forced S-step audit (parity rule P-3).  For every (i, j)
 * the oracle recomputes z_ij from the *given* codes Qg of the columns u > j
 * (not its own), the given codebook T and factor L, exactly as or_sstep does,
 * and reports its argmin s*_ij and the margin
 *     |z - t_{Qg_ij}| - |z - t_{s*}|   (>= 0; 0 when Qg agrees).
 */
void or_sstep_audit(const double *W, const double *L, const double *T, const uint8_t *Qg,
                    int64_t m, int64_t n, int nlev, uint8_t *Sstar, double *margin) {
    double *LT = (double *)malloc(sizeof(double) * (size_t)(n * n));
    for (int64_t u = 0; u < n; ++u)
        for (int64_t j = 0; j < n; ++j) LT[j * n + u] = L[u * n + j];
#pragma omp parallel
    {
        double *r = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < m; ++i) {
            const double *Wi = W + i * n;
            const double *Ti = T + i * nlev;
            for (int64_t j = n - 1; j >= 0; --j) {
                const double *Lcol = LT + j * n;
                double s = 0.0;
                for (int64_t u = j + 1; u < n; ++u) s += r[u] * Lcol[u];
                double z = Wi[j] + s / Lcol[j];
                int q = argmin_level(z, Ti, nlev);
                int qg = Qg[i * n + j];
                Sstar[i * n + j] = (uint8_t)q;
                margin[i * n + j] = fabs(z - Ti[qg]) - fabs(z - Ti[q]);
                r[j] = Wi[j] - Ti[qg]; /* teacher forcing: continue with the given code */
            }
        }
        free(r);
    }
    free(LT);
}

/*
 * Symmetric eigen-decomposition by cyclic Jacobi rotations (textbook), used
 * for the Moore-Penrose inverse of the 2^N x 2^N normal matrix.  A (d x d)
 * is destroyed; on return its diagonal holds the eigenvalues and V the
 * eigenvectors (columns).
 */
static void jacobi_eig(double *A, double *V, int d) {
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) V[i * d + j] = (i == j) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j) {
                tot += A[i * d + j] * A[i * d + j];
                if (i != j) off += A[i * d + j] * A[i * d + j];
            }
        if (off <= 1e-30 * tot || off == 0.0) break;
        for (int p = 0; p < d - 1; ++p)
            for (int q = p + 1; q < d; ++q) {
                double apq = A[p * d + q];
                if (apq == 0.0) continue;
                double app = A[p * d + p], aqq = A[q * d + q];
                double theta = (aqq - app) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < d; ++k) { /* A <- A J (columns p, q) */
                    double akp = A[k * d + p], akq = A[k * d + q];
                    A[k * d + p] = c * akp - s * akq;
                    A[k * d + q] = s * akp + c * akq;
                }
                for (int k = 0; k < d; ++k) { /* A <- J^T A (rows p, q) */
                    double apk = A[p * d + k], aqk = A[q * d + k];
                    A[p * d + k] = c * apk - s * aqk;
                    A[q * d + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < d; ++k) {
                    double vkp = V[k * d + p], vkq = V[k * d + q];
                    V[k * d + p] = c * vkp - s * vkq;
                    V[k * d + q] = s * vkp + c * vkq;
                }
            }
    }
}

/*
 * x = b M^dagger for a symmetric PSD d x d matrix M (Moore-Penrose):
 * M^dagger = V diag(1/lambda_k if lambda_k > cut else 0) V^T with
 * cut = d * eps64 * max_k |lambda_k|  [R-9].
 */
static void pinv_solve(const double *M, const double *b, double *x, int d) {
    double *Aw = (double *)malloc(sizeof(double) * (size_t)(d * d));
    double *V = (double *)malloc(sizeof(double) * (size_t)(d * d));
    memcpy(Aw, M, sizeof(double) * (size_t)(d * d));
    jacobi_eig(Aw, V, d);
    double lmax = 0.0;
    for (int k = 0; k < d; ++k) if (fabs(Aw[k * d + k]) > lmax) lmax = fabs(Aw[k * d + k]);
    double cut = (double)d * DBL_EPSILON * lmax;
    for (int a = 0; a < d; ++a) x[a] = 0.0;
    for (int k = 0; k < d; ++k) {
        double lam = Aw[k * d + k];
        if (!(lam > cut)) continue;
        double proj = 0.0; /* (b . v_k) / lambda_k */
        for (int a = 0; a < d; ++a) proj += b[a] * V[a * d + k];
        proj /= lam;
        for (int a = 0; a < d; ++a) x[a] += proj * V[a * d + k];
    }
    free(Aw);
    free(V);
}

/*
 * T-step: closed form (Eq. 6; Algorithm 1 "batch update"):
 *     T_i = W_i H S_i^T (S_i H S_i^T)^dagger
 * with raw H (the T-step of Algorithm 1 uses H, [R-4]).  Written out:
 *     G_i[a][b] = sum_{j,k} [Q_ij = a][Q_ik = b] H_jk     (S_i H S_i^T)
 *     b_i[a]    = sum_j [Q_ij = a] (W_i H)_j              (W_i H S_i^T)
 *     T_i       = b_i G_i^dagger                           (Moore-Penrose)
 * Levels no column uses have zero rows/columns in G_i and receive 0 from the
 * pseudo-inverse (empty_rule 0, paper-literal [R-9]); empty_rule 1 keeps the
 * previous value Tprev for them instead.
 * Gout / bout (nullable; m x nlev x nlev and m x nlev) receive G_i and b_i.
 */
int or_tstep(const double *W, const uint8_t *Q, const double *H, int64_t m, int64_t n, int nlev,
             int empty_rule, const double *Tprev, double *T, double *Gout, double *bout) {
    if (nlev < 1 || nlev > OR_MAXLEV) return 1;
#pragma omp parallel
    {
        double *WH = (double *)malloc(sizeof(double) * (size_t)n);
        double *G = (double *)malloc(sizeof(double) * (size_t)(nlev * nlev));
        double *b = (double *)malloc(sizeof(double) * (size_t)nlev);
        double *x = (double *)malloc(sizeof(double) * (size_t)nlev);
        int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)nlev);
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < m; ++i) {
            const double *Wi = W + i * n;
            const uint8_t *Qi = Q + i * n;
            for (int64_t j = 0; j < n; ++j) { /* (W_i H)_j */
                double s = 0.0;
                for (int64_t k = 0; k < n; ++k) s += Wi[k] * H[k * n + j];
                WH[j] = s;
            }
            memset(G, 0, sizeof(double) * (size_t)(nlev * nlev));
            memset(b, 0, sizeof(double) * (size_t)nlev);
            memset(cnt, 0, sizeof(int64_t) * (size_t)nlev);
            for (int64_t j = 0; j < n; ++j) {
                int a = Qi[j];
                cnt[a]++;
                b[a] += WH[j];
                for (int64_t k = 0; k < n; ++k) G[a * nlev + Qi[k]] += H[j * n + k];
            }
            pinv_solve(G, b, x, nlev);
            for (int a = 0; a < nlev; ++a) {
                if (cnt[a] == 0 && empty_rule == 1 && Tprev) x[a] = Tprev[i * nlev + a];
                T[i * nlev + a] = x[a];
            }
            if (Gout) memcpy(Gout + i * nlev * nlev, G, sizeof(double) * (size_t)(nlev * nlev));
            if (bout) memcpy(bout + i * nlev, b, sizeof(double) * (size_t)nlev);
        }
        free(WH); free(G); free(b); free(x); free(cnt);
    }
    return 0;
}

/*
 * Layer objective, Eq. (1) in its H form, Eq. (8):
 *     f = sum_i (W_i - T_i S_i) H (W_i - T_i S_i)^T ,  W~_ij = T_{i, Q_ij}
 * per_row (nullable, m) receives each row's term.
 */
double or_objective(const double *W, const uint8_t *Q, const double *T, const double *H,
                    int64_t m, int64_t n, int nlev, double *per_row) {
    double total = 0.0;
#pragma omp parallel
    {
        double *e = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 1) reduction(+ : total)
        for (int64_t i = 0; i < m; ++i) {
            for (int64_t j = 0; j < n; ++j) e[j] = W[i * n + j] - T[i * nlev + Q[i * n + j]];
            double f = 0.0;
            for (int64_t j = 0; j < n; ++j) {
                double s = 0.0;
                for (int64_t k = 0; k < n; ++k) s += H[j * n + k] * e[k];
                f += e[j] * s;
            }
            if (per_row) per_row[i] = f;
            total += f;
        }
        free(e);
    }
    return total;
}

/*
 * Algorithm 1 (GANQ) given H:
 *     H' = precondition(H)                   [R-3]   (App. A / Remark 1)
 *     L  = Cholesky(H')
 *     T^0 = T0 or the min-max grid           [R-6]
 *     for k = 0 .. K-1:
 *         Q^{k+1} = S-step(W, L, T^k)
 *         T^{k+1} = T-step(W, Q^{k+1}, H)  [R-4 raw H]
 *     return T^K, Q^K
 * obj_trace (nullable, K) receives Eq. (1) after each T-step.
 * T0 (nullable) is an fp32 m x nlev codebook.  Returns -1 on success,
 * -2 on an argument error, or the Cholesky failure index (>= 0).
 */
int64_t or_quantize(const double *W, int64_t m, int64_t n, const double *H, int nbits, int iters,
                    int policy, double lambda, double tau, const float *T0, int empty_rule,
                    uint8_t *Q, double *T, double *obj_trace) {
    if (m < 1 || n < 1 || nbits < 1 || nbits > 8 || iters < 1) return -2;
    int nlev = 1 << nbits;
    double *Hp = (double *)malloc(sizeof(double) * (size_t)(n * n));
    double *L = (double *)malloc(sizeof(double) * (size_t)(n * n));
    if (or_precondition(H, n, policy, lambda, tau, Hp, NULL) != 0) { free(Hp); free(L); return -2; }
    int64_t bad = or_cholesky(Hp, n, L);
    free(Hp);
    if (bad >= 0) { free(L); return bad; }
    double *Tk = (double *)malloc(sizeof(double) * (size_t)(m * nlev));
    double *Tn = (double *)malloc(sizeof(double) * (size_t)(m * nlev));
    if (T0) {
        for (int64_t i = 0; i < m * nlev; ++i) Tk[i] = (double)T0[i];
    } else {
        float *Wf = (float *)malloc(sizeof(float) * (size_t)(m * n));
        float *Tf = (float *)malloc(sizeof(float) * (size_t)(m * nlev));
        for (int64_t i = 0; i < m * n; ++i) Wf[i] = (float)W[i];
        or_init_codebook(Wf, m, n, nlev, Tf);
        for (int64_t i = 0; i < m * nlev; ++i) Tk[i] = (double)Tf[i];
        free(Wf); free(Tf);
    }
    for (int k = 0; k < iters; ++k) {
        or_sstep(W, L, Tk, m, n, nlev, Q, NULL);
        or_tstep(W, Q, H, m, n, nlev, empty_rule, Tk, Tn, NULL, NULL);
        memcpy(Tk, Tn, sizeof(double) * (size_t)(m * nlev));
        if (obj_trace) obj_trace[k] = or_objective(W, Q, Tk, H, m, n, nlev, NULL);
    }
    memcpy(T, Tk, sizeof(double) * (size_t)(m * nlev));
    free(Tk); free(Tn); free(L);
    return -1;
}

/* ========================================================================= */
/* NEXT-1: the inference side of Fig. 1a.                */
/* ========================================================================= */

/* Packing of Q ("a low-bit query matrix Q in {0..2^N-1}^{m x n}"), in the layout of
 * the storage accounting of Table 1: row i is a little-endian bitstream in which
 * code k occupies bits [k N, (k+1) N); each row is padded to a whole byte, so a row takes
 * ceil(n N / 8) bytes.  Returns -1, or the flat index of the first code >= 2^N (argument
 * error; nothing is written past it). */
int64_t or_pack(const uint8_t *Q, int64_t m, int64_t n, int N, uint8_t *P) {
    const int64_t rb = (n * N + 7) / 8;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t k = 0; k < n; ++k)
            if (Q[i * n + k] >= (1u << N)) return i * n + k;
    memset(P, 0, (size_t)(m * rb));
    for (int64_t i = 0; i < m; ++i)
        for (int64_t k = 0; k < n; ++k)
            for (int b = 0; b < N; ++b) {
                const int64_t bit = k * N + b;
                if ((Q[i * n + k] >> b) & 1u) P[i * rb + bit / 8] |= (uint8_t)(1u << (bit % 8));
            }
    return -1;
}

void or_unpack(const uint8_t *P, int64_t m, int64_t n, int N, uint8_t *Q) {
    const int64_t rb = (n * N + 7) / 8;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t k = 0; k < n; ++k) {
            unsigned v = 0;
            for (int b = 0; b < N; ++b) {
                const int64_t bit = k * N + b;
                v |= (unsigned)((P[i * rb + bit / 8] >> (bit % 8)) & 1u) << b;
            }
            Q[i * n + k] = (uint8_t)v;
        }
}

/* IEEE binary16 -> double, exact (Table 1 stores the codebook in fp16). */
static double half_to_double(uint16_t h) {
    const int s = (h >> 15) & 1, e = (h >> 10) & 31, f = h & 1023;
    double v;
    if (e == 0) v = ldexp((double)f, -24);                   /* subnormal */
    else if (e == 31) v = f ? NAN : INFINITY;
    else v = ldexp((double)(f | 1024), e - 25);
    return s ? -v : v;
}

/* LUT-based mpGEMM (Fig. 1a right; W~_ij = t_{i, Q_ij}):
 *   Y[t][i] = sum_j W~_ij X[t][j] = sum_j T16[i][Q_ij] X[t][j]
 * T16: m x 2^N fp16 codebook, X: p x n fp16 activations (token-major), Y: p x m, fp64,
 * the codes read from the packed rows one by one (no dense W~ is formed). */
void or_lut_gemm(const uint8_t *P, const uint16_t *T16, const uint16_t *X, int64_t m, int64_t n,
                 int64_t p, int N, double *Y) {
    const int64_t rb = (n * N + 7) / 8, nl = (int64_t)1 << N;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t t = 0; t < p; ++t) {
            double acc = 0.0;
            for (int64_t j = 0; j < n; ++j) {
                unsigned q = 0;
                for (int b = 0; b < N; ++b) {
                    const int64_t bit = j * N + b;
                    q |= (unsigned)((P[i * rb + bit / 8] >> (bit % 8)) & 1u) << b;
                }
                acc += half_to_double(T16[i * nl + q]) * half_to_double(X[t * n + j]);
            }
            Y[t * m + i] = acc;
        }
}

/* Storage of an m x n weight matrix, Table 1: fp16 2mn; per-channel uniform N-bit
 * mn N / 8 + 4m (fp16 scale and zero point); LUT mn N / 8 + 2 * 2^N m (fp16 codebook). */
double or_storage_bytes(int64_t m, int64_t n, int N, int scheme) {
    const double q = (double)m * (double)n * N / 8.0;
    if (scheme == 0) return 2.0 * (double)m * (double)n;
    if (scheme == 1) return q + 4.0 * (double)m;
    return q + 2.0 * (double)(1 << N) * (double)m;
}

/* ========================================================================= */
/* NEXT-2: GANQ* outlier extraction, Algorithm 2 (Appendix B).    */
/* ========================================================================= */

/* Cutoff indices of Algorithm 2 into the ascending-sorted row (0-based, reading R-21):
 *   p = 1 - 0.5 r;  upper = floor(n p);  lower = ceil(n (1 - p)). */
void or_outlier_indices(int64_t n, double r, int64_t *upper, int64_t *lower) {
    const double p = 1.0 - 0.5 * r;
    *upper = (int64_t)floor((double)n * p);
    *lower = (int64_t)ceil((double)n * (1.0 - p));
}

static int cmp_float(const void *a, const void *b) {
    const float x = *(const float *)a, y = *(const float *)b;
    return (x < y) ? -1 : (x > y) ? 1 : 0;
}

/* Algorithm 2, row by row: sort, c_upper = sorted[upper], c_lower = sorted[lower],
 * O = (W >= c_upper) | (W <= c_lower), W_sparse = W o M, W_dense = W - W_sparse.
 * Outputs: mask M (m x n bytes), W_dense (m x n), the two cutoffs per row. */
void or_outlier_split(const float *W, int64_t m, int64_t n, double r, uint8_t *M, float *Wd,
                      float *c_lo, float *c_hi) {
    int64_t up, lo;
    or_outlier_indices(n, r, &up, &lo);
#pragma omp parallel
    {
        float *srt = (float *)malloc(sizeof(float) * (size_t)n);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            memcpy(srt, W + i * n, sizeof(float) * (size_t)n);
            qsort(srt, (size_t)n, sizeof(float), cmp_float);
            const float cu = srt[up], cl = srt[lo];
            c_hi[i] = cu;
            c_lo[i] = cl;
            for (int64_t j = 0; j < n; ++j) {
                const float w = W[i * n + j];
                const int o = (w >= cu) || (w <= cl);
                M[i * n + j] = (uint8_t)o;
                const float ws = o ? w : 0.0f;          /* W o M */
                Wd[i * n + j] = w - ws;                  /* W - W_sparse (exact) */
            }
        }
        free(srt);
    }
}

/* Y (p x m) = X W_sparse^T, fp64, from a CSR (row offsets, column indices, values). */
void or_sparse_matmul(const int64_t *off, const int32_t *col, const float *val, int64_t m, int64_t n,
                      const double *X, int64_t p, double *Y) {
    (void)n;
    for (int64_t t = 0; t < p; ++t)
        for (int64_t i = 0; i < m; ++i) {
            double acc = 0.0;
            for (int64_t k = off[i]; k < off[i + 1]; ++k) acc += (double)val[k] * X[t * n + col[k]];
            Y[t * m + i] = acc;
        }
}

/* ========================================================================= */
/* NEXT-4: k-means initial codebook (per-row 1-D Lloyd), reading R-24.        */
/* ========================================================================= */
/* T0 = iters Lloyd iterations per row from the min-max grid of or_init_codebook [R-6]:
 * assign w_j to argmin_s |w_j - t_s| (fp64 distance of fp32 values, exact; first index on
 * ties [R-7]); t_s <- mean of its weights (fp64), empty levels keep their value; t_s rounded to
 * fp32 after each iteration (T0 is an fp32 input of Algorithm 1). */
void or_kmeans_codebook(const float *W, int64_t m, int64_t n, int nlev, int iters, float *T0) {
    or_init_codebook(W, m, n, nlev, T0);
#pragma omp parallel
    {
        double *sum = (double *)malloc(sizeof(double) * (size_t)nlev);
        int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)nlev);
        double *t = (double *)malloc(sizeof(double) * (size_t)nlev);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            for (int it = 0; it < iters; ++it) {
                for (int s = 0; s < nlev; ++s) { sum[s] = 0.0; cnt[s] = 0; t[s] = (double)T0[i * nlev + s]; }
                for (int64_t j = 0; j < n; ++j) {
                    const double w = (double)W[i * n + j];
                    const int q = argmin_level(w, t, nlev);
                    sum[q] += w;
                    cnt[q] += 1;
                }
                for (int s = 0; s < nlev; ++s)
                    if (cnt[s] > 0) T0[i * nlev + s] = (float)(sum[s] / (double)cnt[s]);
            }
        }
        free(sum); free(cnt); free(t);
    }
}
