/*
 * latsum_oracle.c -- CPU ORACLE for the Epstein-zeta hot path.
 *
 *   TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 *   cpu_baseline / --impl reference legs of bench.py may load this library,
 *   and only as the checker or as the timed CPU baseline -- never as part of
 *   the product path (paper_2504_11989_b200 never imports it).
 *
 * A plain-C restatement, in long double (64-bit mantissa), of the reference
 * algorithm of /root/reference/pkg/src/latsum (L/ below):
 *   upper_gamma dispatch           L/incgamma.py:97-114 (+ helpers 27-94)
 *   exp1_plus_log                  L/incgamma.py:117-143
 *   classify_exponent              L/epstein.py:58-70
 *   shells / half lattice          L/epstein.py:73-90
 *   context constants              L/epstein.py:99-122
 *   _enumerate_direct/_reciprocal  L/epstein.py:126-198
 *   singular, _t0_reg, reg_zeta    L/epstein.py:202-289
 *   zeta (reduce, pole, shat/V)    L/epstein.py:291-320, L/lattice.py:107-112
 *   Duffy node layout              L/quadrature.py:136-177
 *   product of zetas               L/quadrature.py:393-397
 * The reference takes Gamma(s,x) from scipy (gammaincc, exp1; un-vendored,
 * scipy 1.18.1 here); this oracle restates those with the classic series /
 * Legendre continued fraction in long double.  It is PINNED against golden
 * vectors produced by running the reference itself (tests/golden/, generated
 * by tests/golden/make_golden.py) -- see tests/test_oracle.py.
 *
 * The Hessian (polynomial-weighted zeta) has no reference counterpart at
 * k != 0; the oracle evaluates the same Crandall split differentiated term by
 * term (rho-derivatives of |y|^{nu-d} Gamma(s, pi |y|^2/t) are
 * -|y|^{nu-d-2} Gamma(s+1, .) and |y|^{nu-d-4} Gamma(s+2, .)), pinned by the
 * exact identity tr M_nu(k) = Z_{nu-2}(k) against reference zeta values and
 * by finite differences of the reference Z_5.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

typedef long double R;
#define PI_L 3.141592653589793238462643383279502884L
#define EULER_L 0.577215664901532860606512090082402431L
#define MAXD 4

/* ---------------------------------------------------------------- threads */
typedef void (*body_fn)(long i, void* arg);
typedef struct { body_fn fn; void* arg; long n; atomic_long next; } ParJob;

static int nthreads_env(void) {
    const char* e = getenv("LATSUM_ORACLE_THREADS");
    long n = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
    return n < 1 ? 1 : (n > 256 ? 256 : (int)n);
}

static void* par_worker(void* p) {
    ParJob* j = (ParJob*)p;
    for (;;) {
        long i0 = atomic_fetch_add(&j->next, 8);
        if (i0 >= j->n) break;
        long i1 = i0 + 8 < j->n ? i0 + 8 : j->n;
        for (long i = i0; i < i1; ++i) j->fn(i, j->arg);
    }
    return NULL;
}

/* dynamic parallel loop over [0, n); results are written per index, so the
 * caller's fixed-order reductions stay deterministic */
static void par_for(long n, body_fn fn, void* arg) {
    ParJob job;
    job.fn = fn; job.arg = arg; job.n = n;
    atomic_init(&job.next, 0);
    int nt = nthreads_env();
    if (nt > n) nt = (int)(n > 0 ? n : 1);
    pthread_t th[256];
    for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, par_worker, &job);
    par_worker(&job);
    for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
}

/* ---------------------------------------------------------------- special functions */
static R lgamma_series_gamma_lower(R a, R x) { /* gamma(a,x) by series, a > 0 */
    R sum = 1.0L / a, del = sum, ap = a;
    for (int n = 0; n < 100000; ++n) {
        ap += 1.0L;
        del *= x / ap;
        sum += del;
        if (fabsl(del) < fabsl(sum) * 1e-21L) break;
    }
    return sum * expl(-x + a * logl(x));
}

static R gamma_upper_cf(R a, R x) { /* Legendre CF (modified Lentz), any real a, x > 0 */
    const R tiny = 1e-4000L;
    R b = x + 1.0L - a, c = 1.0L / tiny, d = 1.0L / b, h = d;
    for (int i = 1; i < 200000; ++i) {
        R an = -i * (i - a);
        b += 2.0L;
        d = an * d + b;
        if (fabsl(d) < tiny) d = tiny;
        c = b + an / c;
        if (fabsl(c) < tiny) c = tiny;
        d = 1.0L / d;
        R del = d * c;
        h *= del;
        if (fabsl(del - 1.0L) < 1e-21L) break;
    }
    return expl(-x + a * logl(x)) * h;
}

static R e1_l(R x) { /* exponential integral E_1 */
    if (x < 1.0L) {
        R term = 1.0L, acc = 0.0L;
        for (int n = 1; n < 200; ++n) {
            term *= -x / n;
            acc += -term / n;
            if (fabsl(term / n) < 1e-22L * fabsl(acc)) break;
        }
        return -EULER_L - logl(x) + acc;
    }
    return gamma_upper_cf(0.0L, x);
}

/* Gamma(s, x), dispatched like L/incgamma.py:97-114 */
R orc_upper_gamma_l(R s, R x) {
    if (s > 0.0L) {
        if (x < s + 1.0L) return tgammal(s) - lgamma_series_gamma_lower(s, x);
        return gamma_upper_cf(s, x);
    }
    R sr = roundl(s);
    if (fabsl(s - sr) < 1e-12L) { /* Gamma(-m, x) via E_1 and a finite sum (L/incgamma.py:58-75) */
        int m = (int)(-sr);
        R acc = 0.0L, inv = 1.0L / x, term = inv, sign = 1.0L, fact = 1.0L;
        for (int j = 0; j < m; ++j) {
            acc += sign * term;
            term *= (j + 1.0L) * inv;
            sign = -sign;
        }
        for (int j = 2; j <= m; ++j) fact *= j;
        return (e1_l(x) - expl(-x) * acc) * ((m % 2) ? -1.0L : 1.0L) / fact;
    }
    if (fabsl(s - sr) < 1e-3L) return gamma_upper_cf(s, x); /* near-integer: Lentz */
    /* downward recurrence from the anchor in (0, 1] (L/incgamma.py:78-94) */
    int m = (int)ceill(-s);
    R sigma = s + m;
    if (sigma <= 0.0L) { m += 1; sigma = s + m; }
    R g = (x < sigma + 1.0L) ? tgammal(sigma) - lgamma_series_gamma_lower(sigma, x) : gamma_upper_cf(sigma, x);
    R emx = expl(-x), lx = logl(x);
    for (int i = 0; i < m; ++i) {
        sigma -= 1.0L;
        g = (g - expl(sigma * lx) * emx) / sigma;
    }
    return g;
}

double orc_upper_gamma(double s, double x) { return (double)orc_upper_gamma_l(s, x); }

static R exp1_plus_log_l(R x) { /* L/incgamma.py:117-143 */
    if (x < 1.0L) {
        R acc = -EULER_L, term = 1.0L;
        for (int n = 1; n < 200; ++n) {
            term *= -x / n;
            R c = -term / n;
            acc += c;
            if (fabsl(c) < 1e-22L * (1.0L + fabsl(acc))) break;
        }
        return acc;
    }
    return e1_l(x) + logl(x);
}

/* ---------------------------------------------------------------- context */
typedef struct {
    int d, branch, log_m, pole; /* branch 0 generic, 1 log, 2 trivial */
    R A[MAXD * MAXD], B[MAXD * MAXD];
    R vol, t, nu, s, pref, rfac, bconst, kmax, scoef, cval;
    int ndir, nrec;
    R *dn, *dz, *dw; /* half-lattice: integer coords, z = A n, weights */
    R *rq;           /* reciprocal q = B n */
    int hdir, hrec;  /* widened sets for the Hessian (poly_order 2, gamma order s+2) */
    R *hdz, *hdw, *hrq;
} OCtx;

static void octx_free(OCtx* c) {
    free(c->dn); free(c->dz); free(c->dw); free(c->rq);
    free(c->hdz); free(c->hdw); free(c->hrq);
}

static int shell(int d, int r, int* out) { /* max-norm exactly r, lexicographic */
    int w = 2 * r + 1, cnt = 0;
    long total = 1;
    for (int i = 0; i < d; ++i) total *= w;
    for (long idx = 0; idx < total; ++idx) {
        long rem = idx;
        int n[MAXD], mx = 0;
        for (int i = d - 1; i >= 0; --i) {
            n[i] = (int)(rem % w) - r;
            rem /= w;
            if (abs(n[i]) > mx) mx = abs(n[i]);
        }
        if (mx == r) { memcpy(out + cnt * d, n, sizeof(int) * d); ++cnt; }
    }
    return cnt;
}

static int* shell_alloc(int* old, int d, int r) {
    long total = 1;
    for (int i = 0; i < d; ++i) total *= 2 * r + 1;
    return (int*)realloc(old, sizeof(int) * d * total);
}

static int lexpos(const int* n, int d) {
    for (int i = 0; i < d; ++i) { if (n[i] > 0) return 1; if (n[i] < 0) return 0; }
    return 0;
}

/* append-only dynamic array helper */
static void push(R** a, int* cap, int cnt, const R* v, int k) {
    if ((cnt + 1) * k > *cap) {
        *cap = (*cap ? *cap * 2 : 256);
        while (*cap < (cnt + 1) * k) *cap *= 2;
        *a = (R*)realloc(*a, sizeof(R) * (*cap));
    }
    memcpy(*a + cnt * k, v, sizeof(R) * k);
}

static int enum_direct(OCtx* c, int poly_order, R tol, R** pz, R** pw, R** pn) {
    int d = c->d, cnt = 0, capz = 0, capw = 0, capn = 0, below = 0;
    R total = 1.0L;
    int* sh = NULL;
    *pz = *pw = NULL;
    if (pn) *pn = NULL;
    for (int r = 1; r <= 80; ++r) {
        sh = shell_alloc(sh, d, r);
        int m = shell(d, r, sh), start = cnt;
        R mag = 0.0L, wsum = 0.0L;
        for (int i = 0; i < m; ++i) {
            int* n = sh + i * d;
            if (!lexpos(n, d)) continue;
            R z[MAXD], r2 = 0.0L, nn[MAXD];
            for (int a = 0; a < d; ++a) {
                z[a] = 0.0L;
                for (int b = 0; b < d; ++b) z[a] += c->A[a * d + b] * n[b];
                r2 += z[a] * z[a];
                nn[a] = n[a];
            }
            R w = orc_upper_gamma_l(c->nu / 2.0L, PI_L * c->t * r2) * powl(r2, -c->nu / 2.0L);
            R mg = fabsl(w) * powl(r2, poly_order / 2.0L);
            if (mg > mag) mag = mg;
            wsum += fabsl(w);
            push(pz, &capz, cnt, z, d);
            push(pw, &capw, cnt, &w, 1);
            if (pn) push(pn, &capn, cnt, nn, d);
            ++cnt;
        }
        if (mag > tol * total) { total += wsum; below = 0; }
        else { cnt = start; if (++below >= 2) { free(sh); return cnt; } }
    }
    free(sh);
    return -1;
}

static int enum_recip(OCtx* c, R gamma_order, R tol, R** pq) {
    int d = c->d, cnt = 0, cap = 0, below = 0;
    R total = 1.0L;
    int* sh = NULL;
    *pq = NULL;
    for (int r = 1; r <= 80; ++r) {
        sh = shell_alloc(sh, d, r);
        int m = shell(d, r, sh), start = cnt, inf = 0;
        R mag = 0.0L;
        R* rq = (R*)malloc(sizeof(R) * m);
        for (int i = 0; i < m; ++i) {
            R q[MAXD], r2 = 0.0L;
            for (int a = 0; a < d; ++a) {
                q[a] = 0.0L;
                for (int b = 0; b < d; ++b) q[a] += c->B[a * d + b] * sh[i * d + b];
                r2 += q[a] * q[a];
            }
            rq[i] = sqrtl(r2);
            if (rq[i] - c->kmax <= 0.05L) inf = 1;
            push(pq, &cap, cnt, q, d);
            ++cnt;
        }
        if (!inf)
            for (int i = 0; i < m; ++i) {
                R rl = rq[i] - c->kmax, xl = PI_L * rl * rl / c->t;
                R rp = (c->nu >= d) ? rq[i] + c->kmax : rl;
                R bd = fabsl(orc_upper_gamma_l(gamma_order, xl)) * powl(rp, c->nu - d);
                if (bd > mag) mag = bd;
            }
        free(rq);
        if (inf || mag > tol * total) { if (!inf) total += mag; below = 0; }
        else { cnt = start; if (++below >= 2) { free(sh); return cnt; } }
    }
    free(sh);
    return -1;
}

/* returns 0 ok, 1 bad exponent, 6 shell budget, 7 bad lattice */
static int octx_init(OCtx* c, int d, const double* a, double nu, int with_hess) {
    memset(c, 0, sizeof(*c));
    if (!isfinite(nu) || fabs(nu) > 100.0) return 1;
    c->d = d;
    for (int i = 0; i < d * d; ++i) c->A[i] = a[i];
    /* inverse by Gauss-Jordan */
    R m[MAXD][2 * MAXD], det = 1.0L;
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < 2 * d; ++j) m[i][j] = j < d ? c->A[i * d + j] : (j - d == i);
    for (int col = 0; col < d; ++col) {
        int p = col;
        for (int r = col + 1; r < d; ++r) if (fabsl(m[r][col]) > fabsl(m[p][col])) p = r;
        if (m[p][col] == 0.0L) return 7;
        if (p != col) { for (int j = 0; j < 2 * d; ++j) { R t = m[p][j]; m[p][j] = m[col][j]; m[col][j] = t; } det = -det; }
        det *= m[col][col];
        R pv = m[col][col];
        for (int j = 0; j < 2 * d; ++j) m[col][j] /= pv;
        for (int r = 0; r < d; ++r) if (r != col) { R f = m[r][col]; for (int j = 0; j < 2 * d; ++j) m[r][j] -= f * m[col][j]; }
    }
    for (int i = 0; i < d; ++i) for (int j = 0; j < d; ++j) c->B[i * d + j] = m[j][d + i]; /* A^{-T} */
    c->vol = fabsl(det);
    c->t = powl(c->vol, -2.0L / d);
    /* classify (Python round = half-even; ties never pass the 1e-12 test anyway) */
    R mm = nearbyintl((nu - d) / 2.0L);
    if (mm >= 0 && fabsl(nu - (d + 2 * mm)) < 1e-12L) { c->branch = 1; c->log_m = (int)mm; c->nu = d + 2 * mm; }
    else {
        R j = nearbyintl(-nu / 2.0L);
        if (j >= 0 && fabsl(nu + 2 * j) < 1e-12L) { c->branch = 2; c->nu = -2 * j; c->cval = (c->nu == 0.0L) ? -1.0L : 0.0L; return 0; }
        c->branch = 0; c->nu = nu;
    }
    c->pole = fabsl(c->nu - d) < 1e-10L;
    for (int corner = 0; corner < (1 << d); ++corner) {
        R r2 = 0.0L;
        for (int i = 0; i < d; ++i) {
            R v = 0.0L;
            for (int j = 0; j < d; ++j) v += c->B[i * d + j] * (((corner >> j) & 1) ? 0.5L : -0.5L);
            r2 += v * v;
        }
        if (sqrtl(r2) > c->kmax) c->kmax = sqrtl(r2);
    }
    c->s = (d - c->nu) / 2.0L;
    c->pref = 1.0L / tgammal(c->nu / 2.0L);
    c->rfac = powl(PI_L, c->nu - d / 2.0L) / c->vol;
    c->bconst = -2.0L * powl(PI_L * c->t, c->nu / 2.0L) / c->nu;
    if (c->branch == 1) {
        R f = 1.0L;
        for (int i = 2; i <= c->log_m; ++i) f *= i;
        c->scoef = powl(PI_L, 2 * c->log_m + d / 2.0L) / tgammal(c->log_m + d / 2.0L) * ((c->log_m % 2) ? 1.0L : -1.0L) / f;
    } else {
        c->scoef = powl(PI_L, c->nu - d / 2.0L) * tgammal((d - c->nu) / 2.0L) * c->pref;
    }
    c->ndir = enum_direct(c, 0, 1e-18L, &c->dz, &c->dw, &c->dn);
    c->nrec = enum_recip(c, c->s, 1e-18L, &c->rq);
    if (c->ndir < 0 || c->nrec < 0) return 6;
    if (with_hess) {
        c->hdir = enum_direct(c, 2, 1e-18L, &c->hdz, &c->hdw, NULL);
        c->hrec = enum_recip(c, c->s + 2.0L, 1e-18L, &c->hrq);
        if (c->hdir < 0 || c->hrec < 0) return 6;
    }
    return 0;
}

static R t0_reg(const OCtx* c, R rho) { /* L/epstein.py:235-259 */
    R x = PI_L * rho / c->t;
    if (c->branch == 1) {
        int m = c->log_m;
        R head = powl(rho, m) * (exp1_plus_log_l(x) + logl(c->t)), tail = 0.0L, sign = 1.0L, fac = 1.0L, mf = 1.0L;
        for (int j = 0; j < m; ++j) {
            tail += sign * fac * powl(c->t / PI_L, j + 1) * powl(rho, m - 1 - j);
            fac *= j + 1.0L;
            sign = -sign;
        }
        for (int i = 2; i <= m; ++i) mf *= i;
        return ((m % 2) ? -1.0L : 1.0L) / mf * (head - expl(-x) * tail);
    }
    R acc = 1.0L / c->s, term = 1.0L;
    for (int n = 1; n < 400; ++n) {
        term *= -x / n;
        R ct = term / (c->s + n);
        acc += ct;
        if (fabsl(ct) <= 1e-22L * fmaxl(fabsl(acc), 1.0L)) break;
    }
    return -powl(PI_L / c->t, c->s) * acc;
}

static R singular(const OCtx* c, R rho) {
    if (c->branch == 2) return 0.0L;
    if (c->branch == 1) return c->scoef * powl(rho, c->log_m) * logl(PI_L * rho);
    return c->scoef * powl(rho, (c->nu - c->d) / 2.0L);
}

/* flags: 1 no reduce, 2 reg only. returns status bit 1 on pole */
static int zeta_one(const OCtx* c, const double* kin, int flags, R* out) {
    int d = c->d;
    if (c->branch == 2) { *out = c->cval; return 0; }
    R k[MAXD], kap[MAXD];
    for (int a = 0; a < d; ++a) k[a] = kin[a];
    if (!(flags & 1)) {
        for (int a = 0; a < d; ++a) { kap[a] = 0.0L; for (int b = 0; b < d; ++b) kap[a] += c->A[b * d + a] * k[b]; }
        for (int a = 0; a < d; ++a) kap[a] -= floorl(kap[a] + 0.5L);
        for (int a = 0; a < d; ++a) { k[a] = 0.0L; for (int b = 0; b < d; ++b) k[a] += c->B[a * d + b] * kap[b]; }
    }
    R rho = 0.0L;
    for (int a = 0; a < d; ++a) rho += k[a] * k[a];
    if (!(flags & 1) && rho < 1e-28L && c->pole) return 1;
    R acc = c->bconst, dsum = 0.0L, rsum = 0.0L;
    for (int i = 0; i < c->ndir; ++i) {
        R ph = 0.0L;
        for (int a = 0; a < d; ++a) ph += k[a] * c->dz[i * d + a];
        dsum += c->dw[i] * cosl(2.0L * PI_L * ph);
    }
    acc += 2.0L * dsum;
    for (int i = 0; i < c->nrec; ++i) {
        R r2 = 0.0L;
        for (int a = 0; a < d; ++a) { R y = k[a] + c->rq[i * d + a]; r2 += y * y; }
        rsum += orc_upper_gamma_l(c->s, PI_L * r2 / c->t) * powl(r2, (c->nu - d) / 2.0L);
    }
    acc += c->rfac * (t0_reg(c, rho) + rsum);
    acc *= c->pref;
    if (!(flags & 2) && rho >= 1e-28L) acc += singular(c, rho) / c->vol;
    *out = acc;
    return 0;
}

/* full Hessian d_a d_b Z_nu(k) (unreduced k), d*d values */
static void hess_one(const OCtx* c, const double* kin, R* H) {
    int d = c->d;
    R k[MAXD];
    for (int a = 0; a < d; ++a) k[a] = kin[a];
    for (int i = 0; i < d * d; ++i) H[i] = 0.0L;
    if (c->branch == 2) return;
    R Dd[MAXD * MAXD] = {0}, Y[MAXD * MAXD] = {0}, G = 0.0L;
    for (int i = 0; i < c->hdir; ++i) {
        R ph = 0.0L;
        for (int a = 0; a < d; ++a) ph += k[a] * c->hdz[i * d + a];
        R cs = c->hdw[i] * cosl(2.0L * PI_L * ph);
        for (int a = 0; a < d; ++a) for (int b = 0; b < d; ++b) Dd[a * d + b] += cs * c->hdz[i * d + a] * c->hdz[i * d + b];
    }
    /* all q including q = 0: F(rho) = rho^{-s} Gamma(s, pi rho / t) */
    for (int i = -1; i < c->hrec; ++i) {
        R y[MAXD], r2 = 0.0L;
        for (int a = 0; a < d; ++a) { y[a] = k[a] + (i >= 0 ? c->hrq[i * d + a] : 0.0L); r2 += y[a] * y[a]; }
        R x = PI_L * r2 / c->t;
        R f1 = -powl(r2, -(c->s + 1.0L)) * orc_upper_gamma_l(c->s + 1.0L, x);
        R f2 = powl(r2, -(c->s + 2.0L)) * orc_upper_gamma_l(c->s + 2.0L, x);
        G += f1;
        for (int a = 0; a < d; ++a) for (int b = 0; b < d; ++b) Y[a * d + b] += y[a] * y[b] * f2;
    }
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b)
            H[a * d + b] = c->pref * (-8.0L * PI_L * PI_L * Dd[a * d + b] + c->rfac * (4.0L * Y[a * d + b] + (a == b ? 2.0L * G : 0.0L)));
}

/* ---------------------------------------------------------------- public API */
int orc_nthreads(void) { return nthreads_env(); }

int orc_context_counts(int d, const double* a, double nu, long* out4) {
    OCtx c;
    int rc = octx_init(&c, d, a, nu, 1);
    if (rc == 0) { out4[0] = c.ndir; out4[1] = c.nrec; out4[2] = c.hdir; out4[3] = c.hrec; }
    octx_free(&c);
    return rc;
}

typedef struct { const OCtx* c; const double* k; double* out; int flags; volatile int pole; } ZArgs;
static void zeta_body(long i, void* p) {
    ZArgs* a = (ZArgs*)p;
    R v = 0.0L;
    if (zeta_one(a->c, a->k + i * a->c->d, a->flags, &v)) a->pole = 1;
    a->out[i] = (double)v;
}

typedef struct { const OCtx* c; const double* k; double* out; } HArgs;
static void hess_body(long i, void* p) {
    HArgs* a = (HArgs*)p;
    int d = a->c->d;
    R H[MAXD * MAXD];
    hess_one(a->c, a->k + i * d, H);
    for (int j = 0; j < d * d; ++j) a->out[i * d * d + j] = (double)H[j];
}

/* Z (flags 0), Z_reg without reduction (flags 3) ... returns 2 on a pole */
int orc_zeta(int d, const double* a, double nu, const double* k, long n, double* out, int flags) {
    OCtx c;
    int rc = octx_init(&c, d, a, nu, 0);
    if (rc) { octx_free(&c); return rc; }
    ZArgs za = {&c, k, out, flags, 0};
    par_for(n, zeta_body, &za);
    octx_free(&c);
    return za.pole ? 2 : 0;
}

int orc_hessian(int d, const double* a, double nu, const double* k, long n, double* out) {
    OCtx c;
    int rc = octx_init(&c, d, a, nu, 1);
    if (rc) { octx_free(&c); return rc; }
    HArgs ha = {&c, k, out};
    par_for(n, hess_body, &ha);
    octx_free(&c);
    return 0;
}

/* ---------------------------------------------------------------- order-m derivatives at k
 * d^alpha Z(k), |alpha| = m >= 1, from the split differentiated term by term (the k != 0
 * generalisation of L/epstein.py:376-414: direct sum weighted by z^alpha, reciprocal Hermite
 * expansion with F^(p)(rho) = (-1)^p rho^{-s-p} Gamma(s+p, pi rho / t), q = 0 unsplit).
 * Multi-indices in the order of L/epstein.py:426-433 (head ascending). */
static int multi_rec(int d, int total, int* cur, int pos, int* out, int cnt) {
    if (pos == d - 1) {
        cur[pos] = total;
        for (int a = 0; a < d; ++a) out[cnt * d + a] = cur[a];
        return cnt + 1;
    }
    for (int h = 0; h <= total; ++h) {
        cur[pos] = h;
        cnt = multi_rec(d, total - h, cur, pos + 1, out, cnt);
    }
    return cnt;
}

int orc_multi_indices(int d, int order, int* out) {
    int cur[MAXD];
    return multi_rec(d, order, cur, 0, out, 0);
}

typedef struct {
    const OCtx* c;
    int order, na, nd, nr;
    const int* alphas;
    const R *dz, *dw, *rq;
    const double* k;
    double* out;
    double* out_abs;  /* optional: sum of |terms| (the cancellation scale of each value) */
} DArgs;

static R fact_l(int n) { R f = 1.0L; for (int i = 2; i <= n; ++i) f *= i; return f; }

static void deriv_body(long i, void* p) {
    DArgs* A = (DArgs*)p;
    const OCtx* c = A->c;
    int d = c->d, m = A->order;
    R k[MAXD];
    for (int a = 0; a < d; ++a) k[a] = A->k[i * d + a];
    R twopim = powl(2.0L * PI_L, (R)m);
    /* per direct point: w cos(2 pi k.z + m pi / 2); per q (q = 0 first, unsplit): y and
     * F^(pp)(|y|^2) = (-1)^pp |y|^{-2(s+pp)} Gamma(s + pp, pi |y|^2 / t), pp = 0..m -- evaluated
     * once and shared by every multi-index */
    R* dtr = (R*)malloc(sizeof(R) * (size_t)(A->nd > 0 ? A->nd : 1));
    R* ys = (R*)malloc(sizeof(R) * (size_t)(A->nr + 1) * d);
    R* fps = (R*)malloc(sizeof(R) * (size_t)(A->nr + 1) * (m + 1));
    for (int t = 0; t < A->nd; ++t) {
        R ph = 0.0L;
        for (int a = 0; a < d; ++a) ph += k[a] * A->dz[t * d + a];
        dtr[t] = A->dw[t] * cosl(2.0L * PI_L * ph + m * PI_L / 2.0L);
    }
    for (int t = -1; t < A->nr; ++t) {
        R r2 = 0.0L;
        R* y = ys + (size_t)(t + 1) * d;
        for (int a = 0; a < d; ++a) { y[a] = k[a] + (t >= 0 ? A->rq[t * d + a] : 0.0L); r2 += y[a] * y[a]; }
        R x = PI_L * r2 / c->t;
        for (int pp = (m + 1) / 2; pp <= m; ++pp)
            fps[(size_t)(t + 1) * (m + 1) + pp] =
                ((pp & 1) ? -1.0L : 1.0L) * powl(r2, -(c->s + pp)) * orc_upper_gamma_l(c->s + pp, x);
    }
    for (int j = 0; j < A->na; ++j) {
        const int* al = A->alphas + j * d;
        R dsum = 0.0L, rsum = 0.0L, dabs = 0.0L, rabs = 0.0L;
        for (int t = 0; t < A->nd; ++t) {
            R za = 1.0L;
            for (int a = 0; a < d; ++a)
                for (int e = 0; e < al[a]; ++e) za *= A->dz[t * d + a];
            dsum += dtr[t] * za;
            dabs += fabsl(dtr[t] * za);
        }
        /* Hermite terms: j_a <= alpha_a / 2 */
        int jm[MAXD], cnt = 1;
        for (int a = 0; a < d; ++a) { jm[a] = al[a] / 2; cnt *= jm[a] + 1; }
        for (int q = 0; q < cnt; ++q) {
            int rem = q, js = 0, jj[MAXD];
            R cf = 1.0L;
            for (int a = 0; a < d; ++a) {
                jj[a] = rem % (jm[a] + 1); rem /= jm[a] + 1; js += jj[a];
                cf *= fact_l(al[a]) / (fact_l(jj[a]) * fact_l(al[a] - 2 * jj[a]));
            }
            int pp = m - js;
            R part = 0.0L;
            for (int t = 0; t <= A->nr; ++t) {
                const R* y = ys + (size_t)t * d;
                R v = fps[(size_t)t * (m + 1) + pp];
                for (int a = 0; a < d; ++a)
                    for (int e = 0; e < al[a] - 2 * jj[a]; ++e) v *= 2.0L * y[a];
                part += v;
                rabs += fabsl(cf * v);
            }
            rsum += cf * part;
        }
        A->out[i * A->na + j] = (double)(c->pref * (2.0L * twopim * dsum + c->rfac * rsum));
        if (A->out_abs)
            A->out_abs[i * A->na + j] = (double)(fabsl(c->pref) * (2.0L * twopim * dabs + fabsl(c->rfac) * rabs));
    }
    free(dtr); free(ys); free(fps);
}

int orc_derivatives_abs(int d, const double* a, double nu, int order, const double* k, long n, double* out,
                        double* out_abs) {
    OCtx c;
    int rc = octx_init(&c, d, a, nu, 0);
    if (rc) { octx_free(&c); return rc; }
    if (order < 1 || order > 12 || c.branch == 2) { octx_free(&c); return 1; }
    R *dz = NULL, *dw = NULL, *rq = NULL;
    int nd = enum_direct(&c, order, 1e-20L, &dz, &dw, NULL);
    int nr = enum_recip(&c, c.s + order, 1e-20L, &rq);
    if (nd < 0 || nr < 0) { free(dz); free(dw); free(rq); octx_free(&c); return 6; }
    int* alph = (int*)malloc(sizeof(int) * 512 * MAXD);
    int na = orc_multi_indices(d, order, alph);
    DArgs A = {&c, order, na, nd, nr, alph, dz, dw, rq, k, out, out_abs};
    par_for(n, deriv_body, &A);
    free(alph); free(dz); free(dw); free(rq);
    octx_free(&c);
    return 0;
}

int orc_derivatives(int d, const double* a, double nu, int order, const double* k, long n, double* out) {
    return orc_derivatives_abs(d, a, nu, order, k, n, out, NULL);
}

/* Gauss-Legendre on [-1,1] (Newton, long double), ascending */
static void gl(int n, R* x, R* w) {
    for (int i = 0; i < n; ++i) {
        R z = cosl(PI_L * (i + 0.75L) / (n + 0.5L)), dp = 1.0L;
        for (int it = 0; it < 100; ++it) {
            R p0 = 1.0L, p1 = z;
            for (int k = 2; k <= n; ++k) { R p2 = ((2.0L * k - 1.0L) * z * p1 - (k - 1.0L) * p0) / k; p0 = p1; p1 = p2; }
            if (n == 1) { p0 = 1.0L; p1 = z; }
            dp = n * (z * p1 - p0) / (z * z - 1.0L);
            R dz = p1 / dp;
            z -= dz;
            if (fabsl(dz) < 1e-22L) break;
        }
        x[n - 1 - i] = z;
        w[n - 1 - i] = 2.0L / ((1.0L - z * z) * dp * dp);
    }
}

/* Duffy node `idx` of the grid (cell-major, then v (d-1 dims), u fastest): returns
 * k (Cartesian) and the weight wu * u^{d-1} * prod wv.  L/quadrature.py:136-177 */
typedef struct { int d, n_u, n_v, ncell; R *u, *wu, *v, *wv; long total; } OGrid;

static void ogrid_init(OGrid* g, int d, int n_u, int n_v, int q) {
    g->d = d; g->n_u = n_u; g->n_v = d > 1 ? n_v : 1; g->ncell = (1 << (d - 1)) * d;
    g->u = malloc(sizeof(R) * n_u); g->wu = malloc(sizeof(R) * n_u);
    g->v = malloc(sizeof(R) * g->n_v); g->wv = malloc(sizeof(R) * g->n_v);
    R* x = malloc(sizeof(R) * (n_u > n_v ? n_u : n_v) + 64);
    R* w = malloc(sizeof(R) * (n_u > n_v ? n_u : n_v) + 64);
    gl(n_u, x, w);
    for (int i = 0; i < n_u; ++i) {
        R t = (x[i] + 1.0L) / 2.0L, wt = w[i] / 2.0L;
        g->u[i] = 0.5L * powl(t, q);
        g->wu[i] = wt * 0.5L * q * powl(t, q - 1) * powl(g->u[i], d - 1);
    }
    if (d > 1) { gl(g->n_v, x, w); for (int i = 0; i < g->n_v; ++i) { g->v[i] = (x[i] + 1.0L) / 4.0L; g->wv[i] = w[i] / 4.0L; } }
    else { g->v[0] = 0.0L; g->wv[0] = 1.0L; }
    free(x); free(w);
    long nv = 1;
    for (int i = 0; i < d - 1; ++i) nv *= g->n_v;
    g->total = (long)g->ncell * nv * n_u;
}

static void ogrid_free(OGrid* g) { free(g->u); free(g->wu); free(g->v); free(g->wv); }

static void ogrid_node(const OGrid* g, const R* B, long idx, double* k, R* weight) {
    int d = g->d;
    int iu = (int)(idx % g->n_u);
    idx /= g->n_u;
    int iv[MAXD] = {0};
    for (int i = d - 2; i >= 0; --i) { iv[i] = (int)(idx % g->n_v); idx /= g->n_v; }
    int cell = (int)idx, pyr = cell % d, sidx = cell / d;
    R t[MAXD], w = g->wu[iu];
    for (int i = 0; i < d - 1; ++i) {
        R sg = ((sidx >> (d - 2 - i)) & 1) ? -1.0L : 1.0L;
        t[i] = 2.0L * sg * g->v[iv[i]];
        w *= g->wv[iv[i]];
    }
    t[d - 1] = 1.0L;
    R tr[MAXD];
    for (int i = 0; i < d; ++i) tr[i] = t[(i - pyr + d) % d];
    for (int a = 0; a < d; ++a) { R s = 0.0L; for (int b = 0; b < d; ++b) s += B[a * d + b] * tr[b]; k[a] = (double)(g->u[iu] * s); }
    *weight = w;
}

typedef struct { OCtx* cs; int nnu; const OGrid* g; long lo; R* vals; } PArgs;
static void prod_body(long i, void* p) {
    PArgs* a = (PArgs*)p;
    double k[MAXD];
    R w, pr = 1.0L, z;
    ogrid_node(a->g, a->cs[0].B, a->lo + i, k, &w);
    for (int j = 0; j < a->nnu; ++j) { zeta_one(&a->cs[j], k, 0, &z); pr *= z; }
    a->vals[i] = w * pr;
}

typedef struct { const OCtx *c3, *c5; const OGrid* g; long lo; R *v0, *v1; } AArgs;
static void atm_body(long i, void* p) {
    AArgs* a = (AArgs*)p;
    int d = a->c3->d;
    double k[MAXD];
    R w, z, H[MAXD * MAXD], M[MAXD * MAXD], tr = 0.0L;
    ogrid_node(a->g, a->c3->B, a->lo + i, k, &w);
    zeta_one(a->c3, k, 0, &z);
    hess_one(a->c5, k, H);
    for (int j = 0; j < d * d; ++j) M[j] = -H[j] / (4.0L * PI_L * PI_L);
    for (int x = 0; x < d; ++x) for (int y = 0; y < d; ++y) for (int e = 0; e < d; ++e) tr += M[x * d + y] * M[y * d + e] * M[e * d + x];
    a->v0[i] = w * z * z * z;
    a->v1[i] = w * tr;
}

/* sum over nodes [lo, hi) of weight * prod_j Z_{nu_j}(k); out[0] = sum (before 2^d). */
int orc_product_grid(int d, const double* a, const double* nus, int nnu, int n_u, int n_v, int q,
                     long lo, long hi, double* out) {
    OCtx* cs = calloc(nnu, sizeof(OCtx));
    for (int j = 0; j < nnu; ++j) {
        int rc = octx_init(&cs[j], d, a, nus[j], 0);
        if (rc) { for (int i = 0; i <= j; ++i) octx_free(&cs[i]); free(cs); return rc; }
    }
    OGrid g;
    ogrid_init(&g, d, n_u, n_v, q);
    if (hi <= 0 || hi > g.total) hi = g.total;
    long n = hi - lo;
    R* vals = malloc(sizeof(R) * (n > 0 ? n : 1));
    PArgs pa = {cs, nnu, &g, lo, vals};
    par_for(n, prod_body, &pa);
    R s = 0.0L;
    for (long i = 0; i < n; ++i) s += vals[i];
    out[0] = (double)s;
    free(vals);
    ogrid_free(&g);
    for (int j = 0; j < nnu; ++j) octx_free(&cs[j]);
    free(cs);
    return 0;
}

/* ATM integrand sums over nodes [lo, hi): out[0] = sum w Z3^3, out[1] = sum w tr(M5^3). */
int orc_atm_grid(int d, const double* a, int n_u, int n_v, int q, long lo, long hi, double* out) {
    OCtx c3, c5;
    int rc = octx_init(&c3, d, a, 3.0, 0);
    if (!rc) rc = octx_init(&c5, d, a, 5.0, 1);
    if (rc) { octx_free(&c3); return rc; }
    OGrid g;
    ogrid_init(&g, d, n_u, n_v, q);
    if (hi <= 0 || hi > g.total) hi = g.total;
    long n = hi - lo;
    R* v0 = malloc(sizeof(R) * (n > 0 ? n : 1));
    R* v1 = malloc(sizeof(R) * (n > 0 ? n : 1));
    AArgs aa = {&c3, &c5, &g, lo, v0, v1};
    par_for(n, atm_body, &aa);
    R s0 = 0.0L, s1 = 0.0L;
    for (long i = 0; i < n; ++i) { s0 += v0[i]; s1 += v1[i]; }
    out[0] = (double)s0;
    out[1] = (double)s1;
    free(v0); free(v1);
    ogrid_free(&g);
    octx_free(&c3);
    octx_free(&c5);
    return 0;
}

long orc_grid_nodes(int d, int n_u, int n_v) {
    long nv = 1;
    for (int i = 0; i < d - 1; ++i) nv *= n_v;
    return (long)((1 << (d - 1)) * d) * nv * n_u;
}
