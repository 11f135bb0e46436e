/*
 * lbo.c — CPU ORACLE (test infrastructure only; see lbo.h). A plain-C
 * restatement of the reference path; every function cites the reference
 * file:line it follows (paths relative to /root/reference/proj).
 *
 * Build: oracle/Makefile -> oracle/liblbo.so, compiled with -O2
 * -ffp-contract=off so no FMA contraction changes the reference's rounding.
 */
#include "lbo.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

#define AT(m, cols, i, j) ((m)[(i) * (cols) + (j)])

static cplx* as_c(double* p) { return (cplx*)p; }
static const cplx* as_cc(const double* p) { return (const cplx*)p; }

/* kron: src/complex_matrix.cpp:18-28 — out[(i*br+k),(j*bc+l)] = a[i,j]*b[k,l] */
void lbo_kron(const double* a_, size_t ar, size_t ac, const double* b_, size_t br, size_t bc,
              double* out_) {
    const cplx* a = as_cc(a_);
    const cplx* b = as_cc(b_);
    cplx* out = as_c(out_);
    const size_t oc = ac * bc;
    for (size_t i = 0; i < ar; ++i)
        for (size_t j = 0; j < ac; ++j) {
            const cplx aij = AT(a, ac, i, j);
            for (size_t k = 0; k < br; ++k)
                for (size_t l = 0; l < bc; ++l)
                    AT(out, oc, i * br + k, j * bc + l) = aij * AT(b, bc, k, l);
        }
}

/* matmul: src/complex_matrix.cpp:30-56 — i-k-j order, complex arithmetic
 * spelled out in doubles, accumulation from zero in ascending k. */
void lbo_matmul(const double* a, size_t ar, size_t ac, const double* b, size_t bc,
                double* out) {
    memset(out, 0, sizeof(double) * 2 * ar * bc);
    const size_t n = bc;
    for (size_t i = 0; i < ar; ++i) {
        double* crow = out + 2 * i * n;
        for (size_t k = 0; k < ac; ++k) {
            const double xr = a[2 * (i * ac + k)], xi = a[2 * (i * ac + k) + 1];
            const double* brow = b + 2 * k * n;
            for (size_t j = 0; j < n; ++j) {
                const double yr = brow[2 * j], yi = brow[2 * j + 1];
                crow[2 * j] += xr * yr - xi * yi;
                crow[2 * j + 1] += xr * yi + xi * yr;
            }
        }
    }
}

/* dagger: src/complex_matrix.cpp:58-63 */
void lbo_dagger(const double* a_, size_t r, size_t c, double* out_) {
    const cplx* a = as_cc(a_);
    cplx* out = as_c(out_);
    for (size_t i = 0; i < r; ++i)
        for (size_t j = 0; j < c; ++j) AT(out, r, j, i) = conj(AT(a, c, i, j));
}

/* one_norm: src/complex_matrix.cpp:78-86 — max column sum of moduli */
double lbo_one_norm(const double* a_, size_t r, size_t c) {
    const cplx* a = as_cc(a_);
    double best = 0.0;
    for (size_t j = 0; j < c; ++j) {
        double sum = 0.0;
        for (size_t i = 0; i < r; ++i) sum += cabs(AT(a, c, i, j));
        if (sum > best) best = sum;
    }
    return best;
}

static double max_abs(const cplx* a, size_t n) {
    double best = 0.0;
    for (size_t i = 0; i < n; ++i)
        if (cabs(a[i]) > best) best = cabs(a[i]);
    return best;
}

/* is_hermitian: src/lindblad.cpp:13-20 (relative tolerance on max |h| ) */
static int is_hermitian(const cplx* h, size_t d, double rel_tol) {
    double worst = 0.0;
    for (size_t i = 0; i < d; ++i)
        for (size_t j = 0; j < d; ++j) {
            const double e = cabs(AT(h, d, i, j) - conj(AT(h, d, j, i)));
            if (e > worst) worst = e;
        }
    const double scale = max_abs(h, d * d);
    return scale == 0.0 ? worst == 0.0 : worst <= rel_tol * scale;
}

/* build_lindbladian: src/lindblad.cpp:37-59
 *   L = -i (H (x) I - I (x) H^T)
 *     + sum_k [ L_k (x) conj(L_k) - 1/2 (L_k^dag L_k (x) I) - 1/2 (I (x) (L_k^dag L_k)^T) ] */
int lbo_build_lindbladian(size_t d, const double* h_, size_t n_ops, const double* ops,
                          double* out_) {
    const cplx* h = as_cc(h_);
    if (d == 0) return LBO_EINVAL;
    if (!is_hermitian(h, d, 1e-12)) return LBO_EINVAL;
    const size_t n = d * d, nn = n * n;
    cplx* eye = calloc(d * d, sizeof(cplx));
    cplx* ht = malloc(d * d * sizeof(cplx));
    cplx* k1 = malloc(nn * sizeof(cplx));
    cplx* k2 = malloc(nn * sizeof(cplx));
    cplx* tmp = malloc(d * d * sizeof(cplx));
    cplx* ldl = malloc(d * d * sizeof(cplx));
    cplx* lc = malloc(d * d * sizeof(cplx));
    cplx* out = as_c(out_);
    for (size_t i = 0; i < d; ++i) AT(eye, d, i, i) = 1.0;
    for (size_t i = 0; i < d; ++i)
        for (size_t j = 0; j < d; ++j) AT(ht, d, j, i) = AT(h, d, i, j);

    /* coherent part: mi * (kron(H, I) - kron(I, H^T)), lindblad.cpp:46-47 */
    lbo_kron(h_, d, d, (double*)eye, d, d, (double*)k1);
    lbo_kron((double*)eye, d, d, (double*)ht, d, d, (double*)k2);
    const cplx mi = CMPLX(0.0, -1.0);
    for (size_t e = 0; e < nn; ++e) out[e] = mi * (k1[e] - k2[e]);

    /* dissipators, lindblad.cpp:49-57: add_scaled = acc += alpha * x */
    for (size_t k = 0; k < n_ops; ++k) {
        const double* lk = ops + 2 * k * d * d;
        lbo_dagger(lk, d, d, (double*)tmp);
        lbo_matmul((double*)tmp, d, d, lk, d, (double*)ldl);
        for (size_t e = 0; e < d * d; ++e) lc[e] = conj(as_cc(lk)[e]);
        lbo_kron(lk, d, d, (double*)lc, d, d, (double*)k1);
        for (size_t e = 0; e < nn; ++e) out[e] += CMPLX(1.0, 0.0) * k1[e];
        lbo_kron((double*)ldl, d, d, (double*)eye, d, d, (double*)k1);
        for (size_t e = 0; e < nn; ++e) out[e] += CMPLX(-0.5, 0.0) * k1[e];
        for (size_t i = 0; i < d; ++i)
            for (size_t j = 0; j < d; ++j) AT(tmp, d, j, i) = AT(ldl, d, i, j);
        lbo_kron((double*)eye, d, d, (double*)tmp, d, d, (double*)k1);
        for (size_t e = 0; e < nn; ++e) out[e] += CMPLX(-0.5, 0.0) * k1[e];
    }
    free(eye); free(ht); free(k1); free(k2); free(tmp); free(ldl); free(lc);
    return LBO_OK;
}

/* lowering_operator: src/lindblad.cpp:76-80 — a|n> = sqrt(n)|n-1> */
void lbo_lowering_operator(size_t d, double* out) {
    memset(out, 0, sizeof(double) * 2 * d * d);
    for (size_t n = 1; n < d; ++n) out[2 * ((n - 1) * d + n)] = sqrt((double)n);
}

/* ---- expm: src/expm.cpp ---- */
static const double kPade13[14] = {
    64764752532480000.0, 32382376266240000.0, 7771770303897600.0, 1187353796428800.0,
    129060195264000.0,   10559470521600.0,    670442572800.0,     33522128640.0,
    1323241920.0,        40840800.0,          960960.0,           16380.0,
    182.0,               1.0};                      /* expm.cpp:12-16 */
static const double kTheta13 = 5.371920351148152;  /* expm.hpp:19 */

/* solve_in_place: expm.cpp:28-63 — partial-pivot Gaussian elimination,
 * b overwritten with a^-1 b. */
static int solve_in_place(cplx* a, cplx* b, size_t n, size_t bcols) {
    for (size_t col = 0; col < n; ++col) {
        size_t pivot = col;
        double best = cabs(AT(a, n, col, col));
        for (size_t r = col + 1; r < n; ++r) {
            const double mag = cabs(AT(a, n, r, col));
            if (mag > best) { best = mag; pivot = r; }
        }
        if (best == 0.0) return LBO_ERUNTIME;
        if (pivot != col) {
            for (size_t j = 0; j < n; ++j) {
                cplx t = AT(a, n, col, j); AT(a, n, col, j) = AT(a, n, pivot, j); AT(a, n, pivot, j) = t;
            }
            for (size_t j = 0; j < bcols; ++j) {
                cplx t = AT(b, bcols, col, j); AT(b, bcols, col, j) = AT(b, bcols, pivot, j); AT(b, bcols, pivot, j) = t;
            }
        }
        const cplx inv = 1.0 / AT(a, n, col, col);
        for (size_t r = col + 1; r < n; ++r) {
            const cplx factor = AT(a, n, r, col) * inv;
            if (factor == 0.0) continue;
            for (size_t j = col + 1; j < n; ++j) AT(a, n, r, j) -= factor * AT(a, n, col, j);
            for (size_t j = 0; j < bcols; ++j) AT(b, bcols, r, j) -= factor * AT(b, bcols, col, j);
        }
    }
    for (size_t col = n; col-- > 0;) {
        const cplx inv = 1.0 / AT(a, n, col, col);
        for (size_t j = 0; j < bcols; ++j) AT(b, bcols, col, j) *= inv;
        for (size_t r = 0; r < col; ++r) {
            const cplx factor = AT(a, n, r, col);
            if (factor == 0.0) continue;
            for (size_t j = 0; j < bcols; ++j) AT(b, bcols, r, j) -= factor * AT(b, bcols, col, j);
        }
    }
    return LBO_OK;
}

static void axpy(cplx* acc, double alpha, const cplx* x, size_t n) {
    for (size_t i = 0; i < n; ++i) acc[i] += CMPLX(alpha, 0.0) * x[i];
}

/* pade13_eval: expm.cpp:72-107 — even/odd split, 6 matmuls + one solve */
static int pade13_eval(const cplx* m, size_t n, cplx* result) {
    const size_t nn = n * n;
    const double* b = kPade13;
    cplx* m2 = malloc(nn * sizeof(cplx));
    cplx* m4 = malloc(nn * sizeof(cplx));
    cplx* m6 = malloc(nn * sizeof(cplx));
    cplx* inner = malloc(nn * sizeof(cplx));
    cplx* u = malloc(nn * sizeof(cplx));
    cplx* u2 = malloc(nn * sizeof(cplx));
    cplx* v = malloc(nn * sizeof(cplx));
    cplx* denom = malloc(nn * sizeof(cplx));
    lbo_matmul((const double*)m, n, n, (const double*)m, n, (double*)m2);
    lbo_matmul((double*)m2, n, n, (double*)m2, n, (double*)m4);
    lbo_matmul((double*)m2, n, n, (double*)m4, n, (double*)m6);

    for (size_t e = 0; e < nn; ++e) inner[e] = CMPLX(b[13], 0) * m6[e];
    axpy(inner, b[11], m4, nn);
    axpy(inner, b[9], m2, nn);
    lbo_matmul((double*)m6, n, n, (double*)inner, n, (double*)u);
    axpy(u, b[7], m6, nn);
    axpy(u, b[5], m4, nn);
    axpy(u, b[3], m2, nn);
    for (size_t i = 0; i < n; ++i) u[i * n + i] += CMPLX(b[1], 0) * 1.0;
    lbo_matmul((const double*)m, n, n, (double*)u, n, (double*)u2);

    for (size_t e = 0; e < nn; ++e) inner[e] = CMPLX(b[12], 0) * m6[e];
    axpy(inner, b[10], m4, nn);
    axpy(inner, b[8], m2, nn);
    lbo_matmul((double*)m6, n, n, (double*)inner, n, (double*)v);
    axpy(v, b[6], m6, nn);
    axpy(v, b[4], m4, nn);
    axpy(v, b[2], m2, nn);
    for (size_t i = 0; i < n; ++i) v[i * n + i] += CMPLX(b[0], 0) * 1.0;

    for (size_t e = 0; e < nn; ++e) {
        denom[e] = v[e] - u2[e];
        result[e] = v[e] + u2[e];
    }
    int rc = solve_in_place(denom, result, n, n);
    free(m2); free(m4); free(m6); free(inner); free(u); free(u2); free(v); free(denom);
    return rc;
}

/* expm: expm.cpp:109-134 — scaling and squaring around Pade-13 */
int lbo_expm(const double* a_, size_t n, double dt, double* out_) {
    const cplx* a = as_cc(a_);
    const size_t nn = n * n;
    if (!isfinite(dt)) return LBO_EINVAL;
    for (size_t e = 0; e < nn; ++e)
        if (!isfinite(creal(a[e])) || !isfinite(cimag(a[e]))) return LBO_EINVAL;
    cplx* m = malloc(nn * sizeof(cplx));
    for (size_t e = 0; e < nn; ++e) m[e] = CMPLX(dt, 0) * a[e];
    const double nrm = lbo_one_norm((double*)m, n, n);
    int s = 0;
    if (nrm > kTheta13) {
        s = (int)ceil(log2(nrm / kTheta13));
        if (s > 64) { free(m); return LBO_ERUNTIME; }
        for (size_t e = 0; e < nn; ++e) m[e] = CMPLX(ldexp(1.0, -s), 0) * m[e];
    }
    cplx* r = as_c(out_);
    int rc = pade13_eval(m, n, r);
    if (rc == LBO_OK && s > 0) {
        cplx* t = malloc(nn * sizeof(cplx));
        for (int i = 0; i < s; ++i) {
            lbo_matmul((double*)r, n, n, (double*)r, n, (double*)t);
            memcpy(r, t, nn * sizeof(cplx));
        }
        free(t);
    }
    free(m);
    return rc;
}

/* step_soa_kernel: src/kernels_variants.cpp:26-41 — ascending-j sums */
void lbo_step_soa(const double* p_re, const double* p_im, const double* v_re,
                  const double* v_im, double* out_re, double* out_im, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        const double* row_re = p_re + i * n;
        const double* row_im = p_im + i * n;
        double acc_re = 0.0, acc_im = 0.0;
        for (size_t j = 0; j < n; ++j) {
            acc_re += row_re[j] * v_re[j] - row_im[j] * v_im[j];
            acc_im += row_re[j] * v_im[j] + row_im[j] * v_re[j];
        }
        out_re[i] = acc_re;
        out_im[i] = acc_im;
    }
}

/* step_aos_kernel: src/kernels_variants.cpp:16-24 */
void lbo_step_aos(const double* p, const double* v, double* out, size_t n) {
    const cplx* pc = as_cc(p);
    const cplx* vc = as_cc(v);
    for (size_t i = 0; i < n; ++i) {
        cplx acc = 0.0;
        for (size_t j = 0; j < n; ++j) acc += pc[i * n + j] * vc[j];
        as_c(out)[i] = acc;
    }
}

/* check_state: src/validate.cpp:10-30 */
lbo_report lbo_check_state(const double* rho_, size_t d, double tol) {
    const cplx* rho = as_cc(rho_);
    lbo_report r;
    cplx trace = 0.0;
    double min_diag = d ? creal(rho[0]) : 0.0;
    double herm = 0.0;
    for (size_t i = 0; i < d; ++i) {
        trace += AT(rho, d, i, i);
        if (creal(AT(rho, d, i, i)) < min_diag) min_diag = creal(AT(rho, d, i, i));
        for (size_t j = 0; j < d; ++j) {
            const double e = cabs(AT(rho, d, i, j) - conj(AT(rho, d, j, i)));
            if (e > herm) herm = e;
        }
    }
    r.trace_error = cabs(trace - 1.0);
    r.hermiticity_error = herm;
    r.min_diagonal = min_diag;
    r.passed = r.trace_error <= tol && r.hermiticity_error <= tol && r.min_diagonal >= -tol;
    return r;
}

/* evolve (SoA layout): src/propagate.cpp:75-94 — check rho0, ping-pong steps */
int lbo_evolve(const double* p, size_t d, const double* rho0, size_t n_steps, double* out) {
    const size_t n = d * d;
    if (!lbo_check_state(rho0, d, 1e-8).passed) return LBO_EINVAL;
    if (n_steps == 0) {
        memcpy(out, rho0, sizeof(double) * 2 * n);
        return LBO_OK;
    }
    double* pr = malloc(sizeof(double) * n * n);
    double* pi = malloc(sizeof(double) * n * n);
    double* buf = malloc(sizeof(double) * 4 * n);
    for (size_t e = 0; e < n * n; ++e) { pr[e] = p[2 * e]; pi[e] = p[2 * e + 1]; }
    double *cr = buf, *ci = buf + n, *nr = buf + 2 * n, *ni = buf + 3 * n;
    for (size_t e = 0; e < n; ++e) { cr[e] = rho0[2 * e]; ci[e] = rho0[2 * e + 1]; }
    for (size_t s = 0; s < n_steps; ++s) {
        lbo_step_soa(pr, pi, cr, ci, nr, ni, n);
        double* t = cr; cr = nr; nr = t;
        t = ci; ci = ni; ni = t;
    }
    for (size_t e = 0; e < n; ++e) { out[2 * e] = cr[e]; out[2 * e + 1] = ci[e]; }
    free(pr); free(pi); free(buf);
    return LBO_OK;
}

/* ======================================================================
 * Configs (BASELINE.json "configs"). Not in the reference:
 * the reference has no multi-transmon models. The construction order below is
 * the spec DESIGN.md states; the product restates it independently and
 * tests/test_oracle.py checks the two agree.
 * ====================================================================== */
static const double kTwoPi = 6.283185307179586;
static const double kGamma1 = 2e-5, kGammaPhi = 7e-6, kDt = 0.1;

size_t lbo_config_dim(int cfg) {
    switch (cfg) {
        case 0: case 1: return 3;
        case 2: case 4: return 9;
        case 3: return 27;
    }
    return 0;
}
size_t lbo_config_nops(int cfg) { return cfg == 3 ? 6 : (cfg == 2 || cfg == 4) ? 4 : 2; }
double lbo_config_dt(void) { return kDt; }

/* a_q = I (x) .. (x) a (x) .. (x) I with the q-th factor (q = 0 leftmost) */
static void embed(const double* op3, size_t nq, size_t q, double* out) {
    double eye[18] = {0};
    for (int i = 0; i < 3; ++i) eye[2 * (i * 3 + i)] = 1.0;
    size_t dim = 3;
    double* cur = malloc(sizeof(double) * 2 * 27 * 27);
    double* nxt = malloc(sizeof(double) * 2 * 27 * 27);
    memcpy(cur, q == 0 ? op3 : eye, sizeof(double) * 18);
    for (size_t f = 1; f < nq; ++f) {
        lbo_kron(cur, dim, dim, f == q ? op3 : eye, 3, 3, nxt);
        dim *= 3;
        double* t = cur; cur = nxt; nxt = t;
    }
    memcpy(out, cur, sizeof(double) * 2 * dim * dim);
    free(cur); free(nxt);
}

static void add_real_scaled(double* acc, double c, const double* x, size_t n) {
    for (size_t e = 0; e < n; ++e) { acc[2 * e] += c * x[2 * e]; acc[2 * e + 1] += c * x[2 * e + 1]; }
}

void lbo_config_model(int cfg, double delta, double s, double* h, double* ops) {
    const size_t d = lbo_config_dim(cfg);
    const size_t nq = d == 3 ? 1 : d == 9 ? 2 : 3;
    const size_t dd = d * d;
    double alpha[3];
    if (nq == 1) alpha[0] = -kTwoPi * 0.3;
    else { alpha[0] = -kTwoPi * 0.30; alpha[1] = -kTwoPi * 0.28; alpha[2] = -kTwoPi * 0.32; }
    const double omega = kTwoPi * 0.02, g = kTwoPi * 0.005, detuning = kTwoPi * 0.1;

    double a3[18];
    lbo_lowering_operator(3, a3);
    double *a[3], *ad[3], *num[3];
    double* t1 = malloc(sizeof(double) * 2 * dd);
    double* t2 = malloc(sizeof(double) * 2 * dd);
    double* t3 = malloc(sizeof(double) * 2 * dd);
    for (size_t q = 0; q < nq; ++q) {
        a[q] = malloc(sizeof(double) * 2 * dd);
        ad[q] = malloc(sizeof(double) * 2 * dd);
        num[q] = malloc(sizeof(double) * 2 * dd);
        embed(a3, nq, q, a[q]);
        lbo_dagger(a[q], d, d, ad[q]);
        lbo_matmul(ad[q], d, d, a[q], d, num[q]);
    }
    memset(h, 0, sizeof(double) * 2 * dd);
    /* anharmonicity (alpha_q/2) a^dag a^dag a a, as in lindblad.cpp:90 */
    for (size_t q = 0; q < nq; ++q) {
        lbo_matmul(ad[q], d, d, ad[q], d, t1);
        lbo_matmul(a[q], d, d, a[q], d, t2);
        lbo_matmul(t1, d, d, t2, d, t3);
        add_real_scaled(h, alpha[q] / 2.0, t3, dd);
    }
    if (cfg == 2 || cfg == 4) add_real_scaled(h, detuning, num[1], dd);
    if (cfg == 4) {
        add_real_scaled(h, delta, num[0], dd);
        add_real_scaled(h, delta, num[1], dd);
    }
    for (size_t q = 0; q + 1 < nq; ++q) { /* exchange g(a_q^dag a_q+1 + a_q a_q+1^dag) */
        lbo_matmul(ad[q], d, d, a[q + 1], d, t1);
        lbo_matmul(a[q], d, d, ad[q + 1], d, t2);
        add_real_scaled(h, g, t1, dd);
        add_real_scaled(h, g, t2, dd);
    }
    const double drive = (s * omega) / 2.0; /* (s Omega / 2)(a_1 + a_1^dag) */
    add_real_scaled(h, drive, a[0], dd);
    add_real_scaled(h, drive, ad[0], dd);

    /* collapse ops per transmon: sqrt(g1) a_q, sqrt(2 gphi) a_q^dag a_q */
    const double c1 = sqrt(kGamma1), c2 = sqrt(2.0 * kGammaPhi);
    for (size_t q = 0; q < nq; ++q) {
        double* l1 = ops + 2 * (2 * q) * dd;
        double* l2 = ops + 2 * (2 * q + 1) * dd;
        for (size_t e = 0; e < 2 * dd; ++e) { l1[e] = c1 * a[q][e]; l2[e] = c2 * num[q][e]; }
    }
    for (size_t q = 0; q < nq; ++q) { free(a[q]); free(ad[q]); free(num[q]); }
    free(t1); free(t2); free(t3);
}

/* counter-based stream: splitmix64 finaliser over (seed, cfg, traj, k) */
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
double lbo_uniform(uint64_t seed, uint32_t cfg, uint64_t traj, uint64_t k) {
    const uint64_t key =
        mix64(mix64(mix64(seed + 0x9E3779B97F4A7C15ull) ^ ((uint64_t)cfg + 0x632BE59BD9B4E019ull)) ^
              (traj + 0xD6E8FEB86659FD93ull));
    const uint64_t w = mix64(key + (k + 1) * 0x9E3779B97F4A7C15ull);
    return ((double)(w >> 11) + 0.5) * 0x1.0p-53;
}

/* Ginibre G (N(0,1) re/im by explicit Box-Muller), rho = G G^dag / tr,
 * G G^dag formed like random.hpp:31-37 (matmul(g, dagger(g))) */
void lbo_ginibre_rho(uint64_t seed, uint32_t cfg, uint64_t traj, size_t d, double* out) {
    const size_t dd = d * d;
    double* g = malloc(sizeof(double) * 2 * dd);
    double* gd = malloc(sizeof(double) * 2 * dd);
    for (size_t p = 0; p < dd; ++p) {
        const double u1 = lbo_uniform(seed, cfg, traj, 2 * p);
        const double u2 = lbo_uniform(seed, cfg, traj, 2 * p + 1);
        const double r = sqrt(-2.0 * log(u1));
        const double th = kTwoPi * u2;
        g[2 * p] = r * cos(th);
        g[2 * p + 1] = r * sin(th);
    }
    lbo_dagger(g, d, d, gd);
    lbo_matmul(g, d, d, gd, d, out);
    double tr = 0.0;
    for (size_t i = 0; i < d; ++i) tr += out[2 * (i * d + i)];
    for (size_t e = 0; e < 2 * dd; ++e) out[e] = out[e] / tr;
    free(g); free(gd);
}

/* trajectories [first, first + count) of lbo_ginibre_rho, out: count x d x d */
void lbo_ginibre_batch(uint64_t seed, uint32_t cfg, uint64_t first, uint64_t count, size_t d, double* out) {
  for (uint64_t b = 0; b < count; ++b) lbo_ginibre_rho(seed, cfg, first + b, d, out + b * 2 * d * d);
}

void lbo_sweep_params(uint64_t seed, uint64_t traj, double* delta, double* s) {
    const double u = lbo_uniform(seed, 4, traj, 0);
    const double v = lbo_uniform(seed, 4, traj, 1);
    *delta = (kTwoPi * 0.005) * (2.0 * u - 1.0);
    *s = 0.9 + 0.2 * v;
}
