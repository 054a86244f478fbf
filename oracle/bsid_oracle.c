/*
 * bsid_oracle.c -- plain, slow, FP64 CPU oracle for the BSID MAP decoder of
 * arXiv 1802.08483 ("P:n" = line n of PAPER.md; equations cited by label).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_1802_08483_b200/csrc) and neither side includes the other.
 *
 * Every function follows the paper's definition written out, in the paper's
 * order and notation, with full 2-D arrays and no blocking, fusion or
 * reordering:
 *   - Q-dot               : P:207-215  (transmission metric)
 *   - lattice F_{r,j}     : eqn:F P:197-204, initial conditions P:216-225,
 *                           eqn:F_lastrow P:228-235, R = F_{n,mu} P:236-237,
 *                           corridor of width M_n P:250-254
 *   - gamma_i(m',m,D)     : eqn:gamma P:156-161 (prior x receiver metric)
 *   - alpha / beta        : eqn:alpha P:147-148, eqn:beta P:149-151,
 *                           normalisation eqn:alpha_norm/eqn:alpha_prenorm
 *                           P:257-271 ("similar argument" for beta)
 *   - L_i(D)              : eqn:L P:128-130 with lambda (eqn:lambda) and
 *                           sigma (eqn:sigma), divided LITERALLY by
 *                           lambda_N(rho-tau) -- not row-renormalised, so
 *                           sum_D L_i(D) = 1 is a real check.
 *
 * Readings where the paper is silent: R1 boundary
 * priors alpha_0 = delta(0), beta_N = delta(rho-tau); R3 1-based x_r, y_j;
 * R4 corridor m_n^- <= j-r <= m_n^+ relative to the window start; R5 edge
 * windows (gamma = 0 when s<0, s>rho, or the window end passes rho, or
 * m outside [m_tau^-, m_tau^+]); R9 inserted bits uniform (1/2 Pi);
 * R15 bit t of a codeword word is the t-th transmitted bit (LSB first).
 *
 * Parity pins (tests/test_oracle_pins.py): SPEC worked values, brute-force
 * enumeration of channel event sequences (lattice), exhaustive Bayes over
 * messages x event sequences (full decoder), closed forms (noiseless,
 * substitution-only), invariants (sum_D L = 1 with the literal lambda_N,
 * lambda-constancy), bit-complement symmetry.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_DRIFT_OUT_OF_RANGE 1
#define ORACLE_UNDERFLOW 2
#define ORACLE_EINVAL (-1)

/*
 * Host threads used INSIDE one frame (default 1).  Only loops whose iterations
 * are independent and each keep the serial summation order are split across
 * threads -- the m' loop of gamma (one lattice per (m', D)), the D
 * loop of L_i(D) and the m' loop of beta_i(m') -- so the result is
 * bit-identical to the single-threaded oracle for every thread count
 * (tests/test_oracle_pins.py::test_threaded_oracle_bit_identical).  The
 * alpha scatter (eqn:alpha) stays serial.  This is a speed knob for decoding a
 * full-length frame (C5: N = 10^4), not a change of the arithmetic.
 */
static int oracle_threads = 1;

int oracle_set_threads(int t)
{
    oracle_threads = t < 1 ? 1 : t;
    return oracle_threads;
}

/* Q(y|x) = Pt*Ps if y != x, Pt*(1-Ps) if y == x, Pt = 1-Pi-Pd. */
double oracle_qdot(int y, int x, double Pi, double Pd, double Ps)
{
    double Pt = 1.0 - Pi - Pd;
    if (y != x)
        return Pt * Ps;
    return Pt * (1.0 - Ps);
}

/*
 * Receiver-metric lattice.  x[0..n-1] are the codeword bits
 * x_1..x_n, y[0..mu-1] the received bits y_1..y_mu.  F is an (n+1) x (mu+1)
 * row-major array that receives every lattice node.  If use_corridor, only
 * nodes with mn_lo <= j-r <= mn_hi are computed; the others stay 0.
 */
int oracle_lattice(int n, const uint8_t *x, int mu, const uint8_t *y,
                   double Pi, double Pd, double Ps,
                   int use_corridor, int mn_lo, int mn_hi, double *F)
{
    int r, j;
    if (n < 1 || mu < 0 || F == NULL)
        return ORACLE_EINVAL;
    memset(F, 0, sizeof(double) * (size_t)(n + 1) * (size_t)(mu + 1));
    /* Initial conditions: F_{0,0} = 1; F_{i,j} = 0 for i<0 or j<0. */
    F[0] = 1.0;
    for (r = 0; r <= n; r++) {
        for (j = 0; j <= mu; j++) {
            double v = 0.0;
            if (r == 0 && j == 0)
                continue;
            if (use_corridor && (j - r < mn_lo || j - r > mn_hi))
                continue;
            /* eqn:F (rows r < n): insertion term 1/2 Pi F_{r,j-1} ... */
            if (r < n && j >= 1)
                v += 0.5 * Pi * F[(size_t)r * (mu + 1) + (j - 1)];
            /* ... deletion term Pd F_{r-1,j} (also in eqn:F_lastrow) ... */
            if (r >= 1)
                v += Pd * F[(size_t)(r - 1) * (mu + 1) + j];
            /* ... transmission term Q(y_j|x_r) F_{r-1,j-1} (also in eqn:F_lastrow). */
            if (r >= 1 && j >= 1)
                v += oracle_qdot(y[j - 1], x[r - 1], Pi, Pd, Ps) *
                     F[(size_t)(r - 1) * (mu + 1) + (j - 1)];
            F[(size_t)r * (mu + 1) + j] = v;
        }
    }
    return ORACLE_OK;
}

/* R(y|x) = F_{n,mu}. */
double oracle_receiver(int n, const uint8_t *x, int mu, const uint8_t *y,
                       double Pi, double Pd, double Ps,
                       int use_corridor, int mn_lo, int mn_hi)
{
    double *F = (double *)malloc(sizeof(double) * (size_t)(n + 1) * (size_t)(mu + 1));
    double R;
    if (F == NULL)
        return -1.0;
    if (oracle_lattice(n, x, mu, y, Pi, Pd, Ps, use_corridor, mn_lo, mn_hi, F) != ORACLE_OK) {
        free(F);
        return -1.0;
    }
    R = F[(size_t)n * (mu + 1) + mu];
    free(F);
    return R;
}

typedef struct {
    int q, n, N;
    const uint32_t *C; /* [N][q], bit t (LSB = 0) = x_{t+1} of C_i(D) */
    double Pi, Pd, Ps;
    int mn_lo, mn_hi, mt_lo, mt_hi;
    const uint8_t *y; /* y[0..rho-1], one bit per byte */
    int rho;
    const double *priors; /* [N][q] or NULL = uniform 1/q */
} oracle_problem;

static int check_problem(const oracle_problem *p)
{
    if (p->q < 2 || p->n < 1 || p->n > 32 || p->N < 1 || p->C == NULL)
        return 0;
    if (p->n < 32 && (uint64_t)p->q > ((uint64_t)1 << p->n))
        return 0;
    if (!(p->Pi >= 0 && p->Pd >= 0 && p->Ps >= 0 && p->Ps <= 1 && p->Pi + p->Pd < 1))
        return 0;
    if (!(p->mn_lo <= 0 && 0 <= p->mn_hi && p->mt_lo <= p->mn_lo && p->mt_hi >= p->mn_hi))
        return 0;
    if (p->rho < 0 || (p->rho > 0 && p->y == NULL))
        return 0;
    return 1;
}

/*
 * gamma_i(m', m, D) for one symbol index i (eqn:gamma), written to
 * g[(m'-mt_lo)][(m-m'-mn_lo)][D]; size M_tau x M_n x q.  One corridor lattice
 * per (m', D) run for the largest drift change; all m are read from its last
 * row.
 */
int oracle_gamma(const oracle_problem *p, int i, double *g)
{
    const int Mt = p->mt_hi - p->mt_lo + 1, Mn = p->mn_hi - p->mn_lo + 1, n = p->n;
    int mp, failed = 0;
    memset(g, 0, sizeof(double) * (size_t)Mt * Mn * p->q);
#pragma omp parallel num_threads(oracle_threads) reduction(| : failed)
    {
        int D, k, r;
        uint8_t x[32];
        double *F = (double *)malloc(sizeof(double) * (size_t)(n + 1) * (size_t)(n + p->mn_hi + 1));
        if (F == NULL)
            failed = 1;
#pragma omp for schedule(dynamic, 4)
        for (mp = p->mt_lo; mp <= p->mt_hi; mp++) {
            const int s = n * i + mp; /* Y[n i + m' ...] (eqn:gamma) */
            int W;
            if (F == NULL || s < 0 || s > p->rho)
                continue; /* R5: window outside the received sequence */
            W = n + p->mn_hi;
            if (p->rho - s < W)
                W = p->rho - s;
            for (D = 0; D < p->q; D++) {
                const uint32_t word = p->C[(size_t)i * p->q + D];
                const double prior = p->priors ? p->priors[(size_t)i * p->q + D] : 1.0 / p->q;
                for (r = 0; r < n; r++)
                    x[r] = (uint8_t)((word >> r) & 1u);
                oracle_lattice(n, x, W, p->y + s, p->Pi, p->Pd, p->Ps, 1, p->mn_lo, p->mn_hi, F);
                for (k = p->mn_lo; k <= p->mn_hi; k++) {
                    const int m = mp + k, j = n + k;
                    if (j < 0 || j > W || m < p->mt_lo || m > p->mt_hi)
                        continue;
                    /* gamma = P(D_i = D) R(Y[ni+m' .. n(i+1)+m) | C_i(D)) = prior * F_{n, n+k} */
                    g[((size_t)(mp - p->mt_lo) * Mn + (k - p->mn_lo)) * p->q + D] =
                        prior * F[(size_t)n * (W + 1) + j];
                }
            }
        }
        free(F);
    }
    return failed ? ORACLE_EINVAL : ORACLE_OK;
}

/*
 * Full forward-backward decode of one frame, all FP64.
 *   L[N][q]           : eqn:L, divided literally by lambda_N(rho - tau)
 *   log_lambda        : ln lambda_N(rho - tau) in the unnormalised metrics
 *   alpha_hat, beta_hat ((N+1) x M_tau, optional) and logA, logB ((N+1),
 *   optional): normalised rows and the log of the accumulated normalisers,
 *   so that alpha_i(m) = alpha_hat_i(m) exp(logA_i) (eqn:alpha_norm).
 *   alpha0, betaN (M_tau each, optional): the "prior probabilities of the frame
 *   boundaries" alpha_0(m), beta_N(m); NULL = point masses delta(0),
 *   delta(rho - tau) (reading R1).  With betaN given, rho - tau need not be a state.
 *   lambda_N = sum_m alpha_N(m) beta_N(m) (eqn:lambda at i = N).
 * Returns ORACLE_OK, ORACLE_DRIFT_OUT_OF_RANGE (rho - tau outside
 * [m_tau^-, m_tau^+] with the point-mass beta_N) or ORACLE_UNDERFLOW
 * (an all-zero alpha or beta row: Y impossible under the limits).
 */
int oracle_decode(int q, int n, int N, const uint32_t *C,
                  double Pi, double Pd, double Ps,
                  int mn_lo, int mn_hi, int mt_lo, int mt_hi,
                  const uint8_t *y, int rho, const double *priors,
                  const double *alpha0, const double *betaN,
                  double *L, double *log_lambda,
                  double *alpha_hat, double *beta_hat, double *logA, double *logB)
{
    oracle_problem p;
    int Mt, Mn, i, mp, k, D, m, status = ORACLE_OK;
    const int tau = n * N;
    double *A, *B, *lA, *lB, *g, lnlam;

    p.q = q; p.n = n; p.N = N; p.C = C; p.Pi = Pi; p.Pd = Pd; p.Ps = Ps;
    p.mn_lo = mn_lo; p.mn_hi = mn_hi; p.mt_lo = mt_lo; p.mt_hi = mt_hi;
    p.y = y; p.rho = rho; p.priors = priors;
    if (!check_problem(&p) || L == NULL)
        return ORACLE_EINVAL;
    Mt = mt_hi - mt_lo + 1;
    Mn = mn_hi - mn_lo + 1;
    memset(L, 0, sizeof(double) * (size_t)N * q);
    if (log_lambda)
        *log_lambda = -INFINITY;
    if (betaN == NULL && (rho - tau < mt_lo || rho - tau > mt_hi))
        return ORACLE_DRIFT_OUT_OF_RANGE;

    A = (double *)calloc((size_t)(N + 1) * Mt, sizeof(double));
    B = (double *)calloc((size_t)(N + 1) * Mt, sizeof(double));
    lA = (double *)calloc((size_t)(N + 1), sizeof(double));
    lB = (double *)calloc((size_t)(N + 1), sizeof(double));
    g = (double *)malloc(sizeof(double) * (size_t)Mt * Mn * q);
    if (!A || !B || !lA || !lB || !g) {
        free(A); free(B); free(lA); free(lB); free(g);
        return ORACLE_EINVAL;
    }

    /* Boundary priors (R1): alpha_0 = delta(0) or the given alpha0,
       normalised, its sum kept in the log scale. */
    if (alpha0) {
        double c = 0.0;
        for (m = 0; m < Mt; m++)
            c += alpha0[m];
        if (!(c > 0.0)) {
            free(A); free(B); free(lA); free(lB); free(g);
            return ORACLE_EINVAL;
        }
        for (m = 0; m < Mt; m++)
            A[m] = alpha0[m] / c;
        lA[0] = log(c);
    } else {
        A[0 - mt_lo] = 1.0;
        lA[0] = 0.0;
    }
    /* Forward pass, eqn:alpha_prenorm then eqn:alpha_norm, gamma_{i-1} on the fly. */
    for (i = 1; i <= N && status == ORACLE_OK; i++) {
        double c = 0.0;
        double *An = A + (size_t)i * Mt, *Ap = A + (size_t)(i - 1) * Mt;
        if (oracle_gamma(&p, i - 1, g) != ORACLE_OK) {
            status = ORACLE_EINVAL;
            break;
        }
        for (mp = 0; mp < Mt; mp++)
            for (k = 0; k < Mn; k++)
                for (D = 0; D < q; D++) {
                    m = mp + k + mn_lo; /* index of m = m' + (m - m') */
                    if (m < 0 || m >= Mt)
                        continue;
                    An[m] += Ap[mp] * g[((size_t)mp * Mn + k) * q + D];
                }
        for (m = 0; m < Mt; m++)
            c += An[m];
        if (!(c > 0.0)) {
            status = ORACLE_UNDERFLOW;
            break;
        }
        for (m = 0; m < Mt; m++)
            An[m] /= c;
        lA[i] = lA[i - 1] + log(c);
    }
    /* beta_N = delta(rho - tau) or the given betaN, normalised (log scale kept). */
    if (status == ORACLE_OK) {
        double *BN = B + (size_t)N * Mt;
        if (betaN) {
            double c = 0.0;
            for (m = 0; m < Mt; m++)
                c += betaN[m];
            if (!(c > 0.0)) {
                free(A); free(B); free(lA); free(lB); free(g);
                return ORACLE_EINVAL;
            }
            for (m = 0; m < Mt; m++)
                BN[m] = betaN[m] / c;
            lB[N] = log(c);
        } else {
            BN[rho - tau - mt_lo] = 1.0;
            lB[N] = 0.0;
        }
    }
    if (status == ORACLE_OK) {
        /* ln lambda_N = ln sum_m alpha_N(m) beta_N(m) (eqn:lambda at i = N) */
        double lam = 0.0;
        for (m = 0; m < Mt; m++)
            lam += A[(size_t)N * Mt + m] * B[(size_t)N * Mt + m];
        if (!(lam > 0.0))
            status = ORACLE_UNDERFLOW;
        else
            lnlam = lA[N] + lB[N] + log(lam);
    }
    /* Backward pass (eqn:beta, normalised like alpha) with L_i in the same
       pass (eqn:L/eqn:lambda/eqn:sigma): gamma_i recomputed once more. */
    if (status == ORACLE_OK) {
        for (i = N - 1; i >= 0; i--) {
            double c = 0.0;
            double *Bi = B + (size_t)i * Mt, *Bn = B + (size_t)(i + 1) * Mt, *Ai = A + (size_t)i * Mt;
            if (oracle_gamma(&p, i, g) != ORACLE_OK) {
                status = ORACLE_EINVAL;
                break;
            }
            /* L_i(D) = (1/lambda_N) sum_{m',m} alpha_i(m') gamma_i(m',m,D) beta_{i+1}(m) */
#pragma omp parallel for num_threads(oracle_threads) private(mp, k, m) schedule(static)
            for (D = 0; D < q; D++) {
                double s = 0.0;
                for (mp = 0; mp < Mt; mp++)
                    for (k = 0; k < Mn; k++) {
                        m = mp + k + mn_lo;
                        if (m < 0 || m >= Mt)
                            continue;
                        s += Ai[mp] * g[((size_t)mp * Mn + k) * q + D] * Bn[m];
                    }
                L[(size_t)i * q + D] = s * exp(lA[i] + lB[i + 1] - lnlam);
            }
            /* beta_i(m') = sum_{m,D} beta_{i+1}(m) gamma_i(m',m,D) (eqn:beta) */
#pragma omp parallel for num_threads(oracle_threads) private(k, D, m) schedule(static)
            for (mp = 0; mp < Mt; mp++)
                for (k = 0; k < Mn; k++)
                    for (D = 0; D < q; D++) {
                        m = mp + k + mn_lo;
                        if (m < 0 || m >= Mt)
                            continue;
                        Bi[mp] += Bn[m] * g[((size_t)mp * Mn + k) * q + D];
                    }
            for (mp = 0; mp < Mt; mp++)
                c += Bi[mp];
            if (!(c > 0.0)) {
                status = ORACLE_UNDERFLOW;
                break;
            }
            for (mp = 0; mp < Mt; mp++)
                Bi[mp] /= c;
            lB[i] = lB[i + 1] + log(c);
        }
    }
    if (status != ORACLE_OK)
        memset(L, 0, sizeof(double) * (size_t)N * q);
    else if (log_lambda)
        *log_lambda = lnlam;
    if (alpha_hat)
        memcpy(alpha_hat, A, sizeof(double) * (size_t)(N + 1) * Mt);
    if (beta_hat)
        memcpy(beta_hat, B, sizeof(double) * (size_t)(N + 1) * Mt);
    if (logA)
        memcpy(logA, lA, sizeof(double) * (size_t)(N + 1));
    if (logB)
        memcpy(logB, lB, sizeof(double) * (size_t)(N + 1));
    free(A); free(B); free(lA); free(lB); free(g);
    return status;
}

/* gamma for one index i of one frame, exported for element-wise parity. */
int oracle_gamma_at(int q, int n, int N, const uint32_t *C,
                    double Pi, double Pd, double Ps,
                    int mn_lo, int mn_hi, int mt_lo, int mt_hi,
                    const uint8_t *y, int rho, const double *priors, int i, double *g)
{
    oracle_problem p;
    p.q = q; p.n = n; p.N = N; p.C = C; p.Pi = Pi; p.Pd = Pd; p.Ps = Ps;
    p.mn_lo = mn_lo; p.mn_hi = mn_hi; p.mt_lo = mt_lo; p.mt_hi = mt_hi;
    p.y = y; p.rho = rho; p.priors = priors;
    if (!check_problem(&p) || i < 0 || i >= N || g == NULL)
        return ORACLE_EINVAL;
    return oracle_gamma(&p, i, g);
}

/*
 * Extrinsic output for iterative decoding:
 * E_i(D) = L_i(D) / P(D_i = D), normalised over D -- the APP with the symbol's own
 * prior removed.  E_i(D) = 0 where P(D_i = D) = 0; priors NULL = uniform (E = L).
 */
int oracle_extrinsic(int N, int q, const double *L, const double *priors, double *E)
{
    int i, D;
    if (N < 1 || q < 1 || L == NULL || E == NULL)
        return ORACLE_EINVAL;
    for (i = 0; i < N; i++) {
        double s = 0.0;
        for (D = 0; D < q; D++) {
            const double P = priors ? priors[(size_t)i * q + D] : 1.0 / q;
            E[(size_t)i * q + D] = P > 0.0 ? L[(size_t)i * q + D] / P : 0.0;
            s += E[(size_t)i * q + D];
        }
        for (D = 0; D < q; D++)
            E[(size_t)i * q + D] = s > 0.0 ? E[(size_t)i * q + D] / s : 0.0;
    }
    return ORACLE_OK;
}
