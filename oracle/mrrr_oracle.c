/*
 * mrrr_oracle.c -- TEST INFRASTRUCTURE ONLY (see mrrr_oracle.h).
 *
 * A plain, slow, sequential fp64 MRRR tridiagonal eigensolver, written in the
 * order of PAPER.md "The MRRR algorithm" (L1048-1122) with the gaps filled by
 * SURVEY.md §8(c) O1-O12 (readings 1-25 listed in DESIGN.md).  No blocking,
 * no fusion, no reordering: every step is a loop a reader can check by eye.
 *
 * Citations: P:Lx-y = /root/reference/PAPER.md lines x-y;
 *            S:Lx-y = /root/reference/SPEC.md lines x-y;  O# = SURVEY.md §8(c).
 */
#include "mrrr_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define EPS DBL_EPSILON /* 2^-52, O "Definitions" */
#ifndef ORACLE_INTERIOR_PROBES
#define ORACLE_INTERIOR_PROBES 4 /* reading 30: end members and the two next to the shift */
#endif
#ifndef ORACLE_INTERIOR_WG
#define ORACLE_INTERIOR_WG 4.0 /* reading 30: the interior child's weighted-growth bound (x spdiam) */
#endif

void oracle_default_opts(oracle_opts_t *o) {
  o->tol_relgap = 1e-3;                /* P:L1069-1072 footnote */
  o->rtol_class = ldexp(1.0, -20);     /* reading 4 */
  o->max_depth = 128;                  /* reading 21 */
  o->perturb_root = 1;                 /* reading 3 */
  o->seed = 0x1205210700000000ULL;     /* SURVEY §8(b) default seed */
  o->rtol_vec = 0.0;                   /* reading 10 */
  o->rqc_max = 10;                     /* reading 10 */
  o->shift_strategy = 1;               /* reading 30 (0: end shifts only) */
}

/* ------------------------------------------------------------------------ */
/* splitmix64 counter generator (reading 3).  The CUDA side implements the    */
/* same published generator independently.                                    */
static uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
double oracle_perturb_u(uint64_t seed, int64_t grow, int tag) {
  uint64_t x = sm64(seed ^ sm64((uint64_t)(2 * grow + tag)));
  return (double)(int64_t)(x >> 11) * ldexp(1.0, -52) - 1.0; /* [-1, 1) */
}

/* ------------------------------------------------------------------------ */
/* O2 -- norms.  ||T||_1 = max_i |e_{i-1}| + |d_i| + |e_i|; Gershgorin bounds. */
void oracle_norms(int64_t n, const double *d, const double *e, double *tnrm,
                  double *gl, double *gu) {
  double t = 0, lo = INFINITY, hi = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    double r = 0;
    if (i > 0) r += fabs(e[i - 1]);
    if (i < n - 1) r += fabs(e[i]);
    if (r + fabs(d[i]) > t) t = r + fabs(d[i]);
    if (d[i] - r < lo) lo = d[i] - r;
    if (d[i] + r > hi) hi = d[i] + r;
  }
  *tnrm = t; *gl = lo; *gu = hi;
}

/* O3 -- split where |e_i| <= eps*||T||_1 (P:L1052-1055 footnote; readings 1, 16). */
int64_t oracle_split(int64_t n, const double *d, const double *e, double tnrm,
                     int64_t *bstart) {
  (void)d;
  int64_t nb = 0;
  bstart[nb++] = 0;
  for (int64_t i = 0; i < n - 1; ++i)
    if (fabs(e[i]) <= EPS * tnrm) bstart[nb++] = i + 1;
  bstart[nb] = n;
  return nb;
}

/* Sturm count on T (classic LDL^T of T - xI, zero pivot -> -pivmin). */
int64_t oracle_sturm_T(int64_t n, const double *d, const double *e, double x) {
  double emax = 0;
  for (int64_t i = 0; i < n - 1; ++i) if (fabs(e[i]) > emax) emax = fabs(e[i]);
  double pivmin = DBL_MIN * fmax(1.0, emax * emax);
  int64_t c = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0) c++;
  for (int64_t i = 1; i < n; ++i) {
    q = (d[i] - x) - (e[i - 1] * e[i - 1]) / q;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0) c++;
  }
  return c;
}

/* count on a split matrix: sum over blocks, split e_i treated as 0 */
static int64_t sturm_split(int64_t n, const double *d, const double *e,
                           const int64_t *bs, int64_t nbk, double x) {
  int64_t c = 0;
  (void)n;
  for (int64_t b = 0; b < nbk; ++b)
    c += oracle_sturm_T(bs[b + 1] - bs[b], d + bs[b], e + bs[b], x);
  return c;
}

/* ------------------------------------------------------------------------ */
/* O5 -- root representation L0 D0 L0^T = T - sigma0 I, definite
 * (S:L235-243). */
int oracle_root_rrr(int64_t nb, const double *d, const double *e, double tnrm,
                    int side, int perturb, uint64_t seed, int64_t gbase,
                    double *D, double *L, double *sigma, int64_t *retries) {
  double tn, gl, gu;
  oracle_norms(nb, d, e, &tn, &gl, &gu);
  double delta = 4.0 * EPS * tnrm;
  for (int attempt = 0; attempt <= 6; ++attempt) {
    double s = (side > 0) ? gl - delta : gu + delta;
    int ok = 1;
    D[0] = d[0] - s;
    for (int64_t i = 0; i < nb - 1; ++i) {
      L[i] = e[i] / D[i];
      D[i + 1] = (d[i + 1] - s) - L[i] * e[i];
    }
    for (int64_t i = 0; i < nb; ++i)
      if (!isfinite(D[i]) || (side > 0 ? !(D[i] > 0) : !(D[i] < 0))) ok = 0;
    for (int64_t i = 0; i < nb - 1 && ok; ++i)
      if (!isfinite(L[i])) ok = 0;
    if (ok) {
      if (perturb) {
        for (int64_t i = 0; i < nb; ++i)
          D[i] = D[i] * (1.0 + 4.0 * EPS * oracle_perturb_u(seed, gbase + i, 0));
        for (int64_t i = 0; i < nb - 1; ++i)
          L[i] = L[i] * (1.0 + 4.0 * EPS * oracle_perturb_u(seed, gbase + i, 1));
      }
      *sigma = s;
      return 0;
    }
    delta *= 2.0;
    if (retries) (*retries)++;
  }
  return 1;
}

/* ------------------------------------------------------------------------ */
/* O6 -- negcount by the differential stationary qd transform.
 * NaN-safe re-sweep (reading 5, amended in DESIGN.md): the ratio S/D+ is
 * replaced by its limit 1 whenever it is NaN (inf/inf after a zero pivot), a
 * zero pivot counts as non-negative and the next pivot is then +-inf.  The
 * survey's "-pivmin" substitution overflows S/D+ (Clement, exact zero minors). */
int64_t oracle_negcount(int64_t nb, const double *D, const double *LLD,
                        double mu, double pivmin, int *resweep) {
  (void)pivmin;
  double S = -mu, Dp = 0;
  int64_t c = 0;
  for (int64_t i = 0; i < nb - 1; ++i) {
    Dp = D[i] + S;
    if (Dp < 0) c++;
    S = (S / Dp) * LLD[i] - mu;
  }
  Dp = D[nb - 1] + S;
  if (Dp < 0) c++;
  if (!isnan(Dp)) return c;
  if (resweep) *resweep = 1;
  S = -mu; c = 0;
  for (int64_t i = 0; i < nb - 1; ++i) {
    Dp = D[i] + S;
    if (Dp < 0) c++;
    double q = S / Dp;
    if (isnan(q)) q = 1.0;
    S = q * LLD[i] - mu;
  }
  Dp = D[nb - 1] + S;
  if (Dp < 0) c++;
  return c;
}

/* ------------------------------------------------------------------------ */
/* O8 -- classification by relative gap (readings 6, 7). */
void oracle_classify(int64_t k, const double *lo, const double *hi, double tol,
                     int *out) {
  for (int64_t j = 0; j + 1 < k; ++j) {
    double g = lo[j + 1] - hi[j];
    double m0 = 0.5 * (lo[j] + hi[j]), m1 = 0.5 * (lo[j + 1] + hi[j + 1]);
    out[j] = g > tol * fmax(fabs(m0), fabs(m1));
  }
}

/* ------------------------------------------------------------------------ */
/* O9.2 -- child representation by the stationary transform
 * L+ D+ L+^T = L D L^T - sigma I. */
int oracle_child_rrr(int64_t nb, const double *D, const double *L,
                     const double *LD, double sigma, double *Dp, double *Lp,
                     double *growth) {
  double S = -sigma, g = 0;
  int ok = 1;
  for (int64_t i = 0; i < nb - 1; ++i) {
    Dp[i] = D[i] + S;
    Lp[i] = LD[i] / Dp[i];
    S = Lp[i] * L[i] * S - sigma;
    if (!isfinite(Dp[i]) || !isfinite(Lp[i])) ok = 0;
    if (fabs(Dp[i]) > g) g = fabs(Dp[i]);
  }
  Dp[nb - 1] = D[nb - 1] + S;
  if (!isfinite(Dp[nb - 1])) ok = 0;
  if (fabs(Dp[nb - 1]) > g) g = fabs(Dp[nb - 1]);
  *growth = ok ? g : INFINITY;
  return ok ? 0 : 1;
}

/* ------------------------------------------------------------------------ */
/* O10 steps 1-4 -- twisted factorization N_r Delta_r N_r^T = LDL^T - lambda I
 * and solve N_r Delta_r N_r^T z = gamma_r e_r, z_r = 1. */
static int stationary(int64_t nb, const double *D, const double *L,
                      const double *LD, double lambda, double *Dp, double *Lp,
                      double *S) {
  double s = -lambda;
  int fin = 1;
  for (int64_t i = 0; i < nb - 1; ++i) {
    S[i] = s;
    double dp = D[i] + s;
    Dp[i] = dp;
    Lp[i] = LD[i] / dp;
    s = Lp[i] * L[i] * s - lambda;
    if (!isfinite(dp) || !isfinite(s) || !isfinite(Lp[i])) fin = 0;
  }
  S[nb - 1] = s;
  double dp = D[nb - 1] + s;
  Dp[nb - 1] = dp;
  if (!isfinite(dp)) fin = 0;
  return fin;
}
static int progressive(int64_t nb, const double *D, const double *L,
                       const double *LLD, double lambda, double *Dm, double *Um,
                       double *P) {
  double p = D[nb - 1] - lambda;
  int fin = isfinite(p);
  P[nb - 1] = p;
  for (int64_t i = nb - 2; i >= 0; --i) {
    double dm = LLD[i] + p;
    Dm[i + 1] = dm;
    double t = D[i] / dm;
    Um[i] = L[i] * t;
    p = p * t - lambda;
    P[i] = p;
    if (!isfinite(dm) || !isfinite(p) || !isfinite(t) || !isfinite(Um[i])) fin = 0;
  }
  return fin;
}

typedef struct {
  double *Dp, *Lp, *S, *Dm, *Um, *P;
} twscratch_t;

/* *lambda is in/out: if a sweep is not finite (lambda is an eigenvalue of a
 * leading or trailing submatrix, a zero pivot), lambda is nudged by
 * 2eps|lambda| (doubling) and the factorization redone -- reading 25 amended,
 * SPEC S:L302. */
static int twisted_ws(int64_t nb, const double *D, const double *L,
                      const double *LD, const double *LLD, double *lambda,
                      double pivmin, twscratch_t *ws, double *z, int64_t *r_out,
                      double *gamma_out, int64_t *negc_out, int *resweeps) {
  (void)pivmin;
  double lam = *lambda;
  if (nb == 1) {
    z[0] = 1.0; *r_out = 0; *gamma_out = D[0] - lam;
    *negc_out = (*gamma_out < 0); return 0;
  }
  double nudge = 2.0 * EPS * fabs(lam) + DBL_MIN;
  for (int tries = 0;; ++tries) {
    /* 1. stationary (top-down), 2. progressive (bottom-up) */
    int ok = stationary(nb, D, L, LD, lam, ws->Dp, ws->Lp, ws->S);
    ok = ok && progressive(nb, D, L, LLD, lam, ws->Dm, ws->Um, ws->P);
    if (ok || tries >= 60) break;
    (*resweeps)++;
    lam = *lambda + nudge;
    nudge *= 2.0;
  }
  *lambda = lam;
  double lambda_ = lam;
  /* 3. twist: gamma_r = S_r + P_r + lambda; r = argmin |gamma_r| (reading 11) */
  int64_t r = 0;
  double gmin = INFINITY, gr = 0;
  for (int64_t i = 0; i < nb; ++i) {
    double g = ws->S[i] + ws->P[i] + lambda_;
    if (fabs(g) < gmin) { gmin = fabs(g); gr = g; r = i; }
  }
  int64_t negc = (gr < 0);
  for (int64_t i = 0; i < r; ++i) negc += (ws->Dp[i] < 0);
  for (int64_t i = r + 1; i < nb; ++i) negc += (ws->Dm[i] < 0);
  /* 4. solve, z_r = 1 */
  z[r] = 1.0;
  for (int64_t i = r - 1; i >= 0; --i) {
    if (z[i + 1] != 0.0) z[i] = -ws->Lp[i] * z[i + 1];
    else z[i] = -(LD[i + 1] / LD[i]) * z[i + 2];
    if (fabs(z[i]) < DBL_MIN) z[i] = 0.0; /* reading 17 */
  }
  for (int64_t i = r; i < nb - 1; ++i) {
    if (z[i] != 0.0) z[i + 1] = -ws->Um[i] * z[i];
    else z[i + 1] = -(LD[i - 1] / LD[i]) * z[i - 1];
    if (fabs(z[i + 1]) < DBL_MIN) z[i + 1] = 0.0;
  }
  *r_out = r; *gamma_out = gr; *negc_out = negc;
  return 0;
}

static int alloc_ws(twscratch_t *ws, int64_t nb) {
  double *p = (double *)malloc(sizeof(double) * 6 * (size_t)(nb + 1));
  if (!p) return 6;
  ws->Dp = p; ws->Lp = p + (nb + 1); ws->S = p + 2 * (nb + 1);
  ws->Dm = p + 3 * (nb + 1); ws->Um = p + 4 * (nb + 1); ws->P = p + 5 * (nb + 1);
  return 0;
}

int oracle_twisted(int64_t nb, const double *D, const double *L,
                   const double *LD, const double *LLD, double lambda,
                   double pivmin, double *z, int64_t *r, double *gamma,
                   int64_t *negc) {
  twscratch_t ws;
  if (alloc_ws(&ws, nb)) return 6;
  int rs = 0;
  twisted_ws(nb, D, L, LD, LLD, &lambda, pivmin, &ws, z, r, gamma, negc, &rs);
  free(ws.Dp);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Solver context */
typedef struct {
  int64_t nb;
  double *D, *L, *LD, *LLD;
  double tau_hi, tau_lo; /* cumulative shift, T-coordinates = tau + local */
  double pivmin;
} rrr_t;

typedef struct {
  const oracle_opts_t *o;
  oracle_stats_t *st;
  double spdiam;     /* of the current block */
  int64_t nb;
  double *lo, *hi;   /* [nb+1], 1-based local eigen index, node coordinates */
  int *wanted;       /* [nb+1] */
  int64_t *pos;      /* [nb+1] output column, or -1 */
  double *w;         /* output */
  double *Z; int64_t ldz; int64_t gbase;
  twscratch_t ws;
  double *z;         /* [nb] */
  int err;
} ctx_t;

static int rrr_alloc(rrr_t *R, int64_t nb) {
  double *p = (double *)malloc(sizeof(double) * 4 * (size_t)(nb + 1));
  if (!p) return 6;
  R->nb = nb; R->D = p; R->L = p + (nb + 1); R->LD = p + 2 * (nb + 1);
  R->LLD = p + 3 * (nb + 1);
  return 0;
}
static void rrr_derive(rrr_t *R) {
  double m = 0;
  for (int64_t i = 0; i < R->nb - 1; ++i) {
    R->LD[i] = R->L[i] * R->D[i];
    R->LLD[i] = R->L[i] * R->LD[i];
    if (fabs(R->LLD[i]) > m) m = fabs(R->LLD[i]);
  }
  R->pivmin = DBL_MIN * fmax(1.0, m);
}

static int64_t negc(ctx_t *c, const rrr_t *R, double mu) {
  int rs = 0;
  int64_t v = oracle_negcount(R->nb, R->D, R->LLD, mu, R->pivmin, &rs);
  c->st->negcount_sweeps++;
  c->st->negcount_resweeps += rs;
  return v;
}

/* O7 bisection of eigen index j (1-based) on [lo,hi] with N(lo) < j <= N(hi)
 * until hi-lo <= rtol*max(|lo|,|hi|) or lo, hi adjacent doubles. */
static void bisect(ctx_t *c, const rrr_t *R, int64_t j, double rtol, double *plo,
                   double *phi) {
  double lo = *plo, hi = *phi;
  for (;;) {
    if (hi - lo <= rtol * fmax(fabs(lo), fabs(hi))) break;
    double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (negc(c, R, mid) >= j) hi = mid; else lo = mid;
  }
  *plo = lo; *phi = hi;
}

static void two_sum(double a, double b, double *s, double *err) {
  double x = a + b, bb = x - a;
  *err = (a - (x - bb)) + (b - bb);
  *s = x;
}

/* O10 -- singleton vector by Rayleigh-quotient correction on twisted
 * factorizations (readings 10, 24, 25).
 * Reading 10 (amended): at most opts.rqc_max factorizations (3), then the
 * bisection fallback; optionally (opts.rtol_vec > 0) the bracket is first
 * refined by bisection to that relative width. */
static void singleton(ctx_t *c, const rrr_t *R, int64_t j) {
  int64_t nb = R->nb;
  double lo = c->lo[j], hi = c->hi[j];
  if (c->o->rtol_vec > 0) bisect(c, R, j, c->o->rtol_vec, &lo, &hi);
  double lam = 0.5 * (lo + hi), lam_fin = lam;
  int64_t r, nc, nfact = 0;
  double gamma, nrm2 = 1;
  int converged = 0, rs = 0;
  double *z = c->z, delta_prev = INFINITY;
  for (int it = 0; it < (c->o->rqc_max > 0 ? c->o->rqc_max : 1); ++it) {
    twisted_ws(nb, R->D, R->L, R->LD, R->LLD, &lam, R->pivmin, &c->ws, z, &r,
               &gamma, &nc, &rs);
    nfact++;
    if (nc >= j) { if (lam < hi) hi = lam; } else { if (lam > lo) lo = lam; }
    nrm2 = 0;
    for (int64_t i = 0; i < nb; ++i) nrm2 += z[i] * z[i];
    double delta = gamma / nrm2;
    /* stop (reading 10): |delta| <= 4 eps |lambda|, fl(lambda + delta) ==
     * lambda, or stagnation -- the correction no longer halves (the
     * Rayleigh-quotient iteration converges cubically; a correction that
     * stops shrinking sits at the rounding floor of the twisted
     * factorization) */
    if (fabs(delta) <= 4.0 * EPS * fabs(lam) || lam + delta == lam ||
        (it > 0 && fabs(delta) >= 0.5 * fabs(delta_prev))) {
      lam_fin = lam + delta;
      converged = 1;
      break;
    }
    delta_prev = delta;
    /* safeguard (reading 24, amended twice): a step leaving [lo,hi] by at
     * most 4 eps |lambda + delta| is a rounding-level overshoot of an
     * eigenvalue at that end -- the end itself; otherwise a step leaving
     * [lo,hi] from the interior is clamped to the violated end and one from
     * an end bisects, and after such a safeguard step the stagnation test
     * (reading 10) starts afresh: it compares RQ corrections, and a
     * bisection halves the next one by construction.  A bracket of adjacent
     * doubles is converged. */
    double nw = lam + delta;
    if (nw <= lo || nw >= hi) {
      double slack = 4.0 * EPS * fabs(nw);
      if (nw <= lo && lo - nw <= slack) {
        nw = lo;
      } else if (nw >= hi && nw - hi <= slack) {
        nw = hi;
      } else if (lam == lo || lam == hi) {
        nw = 0.5 * (lo + hi);
        delta_prev = INFINITY;
        if (nw <= lo || nw >= hi) { lam_fin = lam; converged = 1; break; }
      } else {
        nw = (nw <= lo) ? lo : hi;
        delta_prev = INFINITY;
      }
    }
    lam = nw;
  }
  if (!converged) {
    c->st->rqc_fallbacks++;
    bisect(c, R, j, 4.0 * EPS, &lo, &hi);
    lam = 0.5 * (lo + hi);
    twisted_ws(nb, R->D, R->L, R->LD, R->LLD, &lam, R->pivmin, &c->ws, z, &r,
               &gamma, &nc, &rs);
    nfact++;
    nrm2 = 0;
    for (int64_t i = 0; i < nb; ++i) nrm2 += z[i] * z[i];
    lam_fin = lam;
  }
  c->st->twisted += nfact;
  c->st->twisted_resweeps += rs;
  c->st->rqc_hist[nfact > 10 ? 11 : nfact]++;
  c->st->singletons++;
  /* 6. output: column pos = z/||z||, w = tau + lambda (compensated tau) */
  int64_t p = c->pos[j];
  double nrm = sqrt(nrm2);
  c->w[p] = R->tau_hi + (R->tau_lo + lam_fin);
  if (c->Z) {
    double *col = c->Z + p * c->ldz;
    for (int64_t i = 0; i < nb; ++i) col[c->gbase + i] = z[i] / nrm;
  }
}

static void process_node(ctx_t *c, const rrr_t *R, int64_t c0, int64_t c1, int depth);

/* weighted growth (tier ii) of a candidate child Dp against one unit-free
 * vector z: sum_i |D+_i| z_i^2 / sum_i z_i^2. */
static double weighted_growth(int64_t nb, const double *z, const double *Dp) {
  double num = 0, den = 0;
  for (int64_t i = 0; i < nb; ++i) {
    num += fabs(Dp[i]) * z[i] * z[i];
    den += z[i] * z[i];
  }
  return num / den;
}

/* O9 -- cluster step: shift, child RRR, refine, recurse.
 * Shift choice, reading 9 (amended): six candidates at offsets
 * m = 1, 2, 4 beyond each end of the cluster (order L1 R1 L2 R2 L4 R4), all
 * evaluated; raw growth g = max_i |D+_i| (inf if a pivot is not finite or
 * zero), weighted growth wg = max over the parent's two end-eigenvalue
 * vectors z_L, z_R of sum |D+_i| z_i^2 / ||z||^2.
 *   (i)   some g <= 8 spdiam: the least g among those;
 *   (ii)  else, the least g among the candidates with wg <= 64 spdiam;
 *   (iii) else the least g if <= 1e8 spdiam; else error 2.
 * Ties go to the earlier candidate.  Evidence (oracle, glued Wilkinson
 * n=21000): the SURVEY rule (lower wg at the first passing offset) gave
 * orthogonality 2.7x the 10 n eps tolerance, this rule 0.46x; on Clement
 * n=20000 the SURVEY rule accepted a child with g = 3.5e5 spdiam (RQC
 * corrections 1e3 eps |lambda| for the far eigenvalues). */
static void cluster(ctx_t *c, const rrr_t *R, int64_t s, int64_t t, int depth) {
  int64_t nb = R->nb;
  double spd = c->spdiam;
  rrr_t C;
  if (rrr_alloc(&C, nb)) { c->err = 6; return; }
  double *DpA = (double *)malloc(sizeof(double) * 4 * (size_t)(nb + 1));
  if (!DpA) { free(C.D); c->err = 6; return; }
  double *LpA = DpA + (nb + 1), *zL = DpA + 2 * (nb + 1), *zR = DpA + 3 * (nb + 1);
  static const double mult[3] = {1.0, 2.0, 4.0};
  double cs[7], cg[7];
  /* offset unit (reading 8, amended): twice the end bracket's width, but at
   * least 2 rtol_c |lambda| -- the width classification guarantees -- so the
   * shift does not depend on how far below rtol_c a bracket happens to be */
  double rt2 = 2.0 * c->o->rtol_class;
  double dl = fmax(fmax(2.0 * (c->hi[s] - c->lo[s]), rt2 * fabs(c->lo[s])), 4.0 * EPS * fabs(c->lo[s]));
  double dr = fmax(fmax(2.0 * (c->hi[t] - c->lo[t]), rt2 * fabs(c->hi[t])), 4.0 * EPS * fabs(c->hi[t]));
  int best = -1;
  for (int mi = 0; mi < 3; ++mi) {
    cs[2 * mi] = c->lo[s] - mult[mi] * dl;
    cs[2 * mi + 1] = c->hi[t] + mult[mi] * dr;
  }
  /* reading 30 (shift_strategy 1): an interior candidate at the midpoint of
   * the widest conservative gap between consecutive members in the middle
   * half of the cluster ("close to one of the eigenvalues in the cluster",
   * P:L1102-1103), taken when that gap is resolvable (> 1e-10 relative: not
   * a degenerate group) and its child passes the growth tests (raw growth
   * <= 8 spdiam, or weighted growth <= 64 spdiam with the end probes and the
   * probes of the two members next to the shift) -- the cluster then splits
   * on both sides of the shift, and the tree's depth grows like log(m)
   * instead of m / (members peeled per level) */
  int64_t m = t - s + 1;
  if (c->o->shift_strategy == 1 && m >= 2000 && c->hi[t] - c->lo[s] > 1e-6 * spd) {
    int64_t a = s + m / 4, b = t - m / 4, jb = -1;
    double gb = -INFINITY;
    for (int64_t j = a; j < b; ++j) {
      double g = c->lo[j + 1] - c->hi[j];
      if (g > gb) { gb = g; jb = j; }
    }
    if (jb >= 0) {
      double la = 0.5 * (c->lo[jb] + c->hi[jb]), lb = 0.5 * (c->lo[jb + 1] + c->hi[jb + 1]);
      if (gb > 1e-10 * fmax(fabs(la), fabs(lb))) {
        double sg = 0.5 * (c->hi[jb] + c->lo[jb + 1]), g6;
        oracle_child_rrr(nb, R->D, R->L, R->LD, sg, DpA, LpA, &g6);
        c->st->child_sweeps++;
        int take = isfinite(g6) && g6 <= 8.0 * spd;
        if (!take && isfinite(g6) && g6 <= 1e8 * spd) {
          int64_t r, nc;
          double gg, lam;
          int rs = 0;
          double wg = 0;
          double lams[4] = {0.5 * (c->lo[s] + c->hi[s]), 0.5 * (c->lo[t] + c->hi[t]), la, lb};
          for (int q = 0; q < ORACLE_INTERIOR_PROBES; ++q) {
            lam = lams[q];
            twisted_ws(nb, R->D, R->L, R->LD, R->LLD, &lam, R->pivmin, &c->ws, zL, &r, &gg, &nc, &rs);
            wg = fmax(wg, weighted_growth(nb, zL, DpA));
          }
          take = wg <= ORACLE_INTERIOR_WG * spd;
        }
        if (take) {
          best = 6;
          cs[6] = sg; cg[6] = g6;
          c->st->interior++;
        }
      }
    }
  }
  for (int k = 0; k < 6 && best != 6; ++k) {
    oracle_child_rrr(nb, R->D, R->L, R->LD, cs[k], DpA, LpA, &cg[k]);
    c->st->child_sweeps++;
    if (cg[k] <= 8.0 * spd && (best < 0 || cg[k] < cg[best])) best = k;
  }
  if (best == 6) {
    /* interior shift taken */
  } else if (best >= 0) c->st->tier[0]++;
  else {
    int64_t r, nc;
    double g;
    int rs = 0;
    double lamL = 0.5 * (c->lo[s] + c->hi[s]), lamR = 0.5 * (c->lo[t] + c->hi[t]);
    twisted_ws(nb, R->D, R->L, R->LD, R->LLD, &lamL, R->pivmin, &c->ws, zL, &r, &g, &nc, &rs);
    twisted_ws(nb, R->D, R->L, R->LD, R->LLD, &lamR, R->pivmin, &c->ws, zR, &r, &g, &nc, &rs);
    for (int k = 0; k < 6; ++k) {
      if (!isfinite(cg[k])) continue;
      oracle_child_rrr(nb, R->D, R->L, R->LD, cs[k], DpA, LpA, &g);
      double wg = fmax(weighted_growth(nb, zL, DpA), weighted_growth(nb, zR, DpA));
      if (wg <= 64.0 * spd && (best < 0 || cg[k] < cg[best])) best = k;
    }
    if (best >= 0) c->st->tier[1]++;
  }
  if (best < 0) {  /* tier (iii) */
    for (int k = 0; k < 6; ++k)
      if (best < 0 || cg[k] < cg[best]) best = k;
    if (!(cg[best] <= 1e8 * spd)) { free(DpA); free(C.D); c->err = 2; return; }
    c->st->tier[2]++;
  }
  double sigma;
  sigma = cs[best];
  free(DpA);
  /* the accepted child */
  double g;
  oracle_child_rrr(nb, R->D, R->L, R->LD, sigma, C.D, C.L, &g);
  c->st->child_sweeps++;
  rrr_derive(&C);
  double sh, se;
  two_sum(R->tau_hi, sigma, &sh, &se);
  double lo2 = R->tau_lo + se;
  C.tau_hi = sh + lo2;
  C.tau_lo = lo2 - (C.tau_hi - sh);
  c->st->nodes++;
  if (depth + 1 > c->st->max_depth) c->st->max_depth = depth + 1;
  /* O9.4 refine members in child coordinates: widen, verify, bisect */
  for (int64_t j = s; j <= t; ++j) {
    double lam = 0.5 * (c->lo[j] + c->hi[j]);
    double wd = 2.0 * (c->hi[j] - c->lo[j]) + 4.0 * EPS * (fabs(sigma) + fabs(lam));
    double wl = wd, wu = wd;
    double a = c->lo[j] - sigma - wl, b = c->hi[j] - sigma + wu;
    int tries = 0;
    while (negc(c, &C, a) > j - 1) {
      wl *= 2.0; a = c->lo[j] - sigma - wl;
      if (++tries > 200) { c->err = 4; free(C.D); return; }
    }
    tries = 0;
    while (negc(c, &C, b) < j) {
      wu *= 2.0; b = c->hi[j] - sigma + wu;
      if (++tries > 200) { c->err = 4; free(C.D); return; }
    }
    bisect(c, &C, j, c->o->rtol_class, &a, &b);
    c->lo[j] = a; c->hi[j] = b;
  }
  process_node(c, &C, s, t, depth + 1);
  free(C.D);
}

static void process_node(ctx_t *c, const rrr_t *R, int64_t c0, int64_t c1, int depth) {
  if (c->err) return;
  if (depth > c->o->max_depth) { c->err = 3; return; }
  int64_t k = c1 - c0 + 1;
  int *bd = (int *)malloc(sizeof(int) * (size_t)(k + 1));
  if (!bd) { c->err = 6; return; }
  oracle_classify(k, c->lo + c0, c->hi + c0, c->o->tol_relgap, bd);
  int64_t s = c0;
  for (int64_t j = c0; j <= c1 && !c->err; ++j) {
    if (j == c1 || bd[j - c0]) {
      if (s == j) {
        if (c->wanted[j]) singleton(c, R, j);
      } else {
        int any = 0;
        for (int64_t q = s; q <= j; ++q) any |= c->wanted[q];
        if (any) cluster(c, R, s, j, depth);
      }
      s = j + 1;
    }
  }
  free(bd);
}

/* ------------------------------------------------------------------------ */
/* one block: root RRR (O5), root bisection (O7), tree (O8-O10) */
typedef struct {
  int64_t b0, nb;      /* rows */
  int64_t wa, wb;      /* wanted local indices (1-based), wa > wb => none */
} blockjob_t;

/* root interval verification: N(lo0) == 0, N(hi0) == nb */
static void root_interval(ctx_t *c, const rrr_t *R, int side, double gl,
                          double gu, double sigma, double *lo0, double *hi0) {
  double wid = 2.0 * EPS * c->spdiam + DBL_MIN;
  if (side > 0) {
    *lo0 = 0.0;
    for (;;) { *hi0 = (gu - sigma) + wid; if (negc(c, R, *hi0) >= R->nb) break; wid *= 2.0; }
  } else {
    *hi0 = 0.0;
    for (;;) { *lo0 = (gl - sigma) - wid; if (negc(c, R, *lo0) <= 0) break; wid *= 2.0; }
  }
}

static int setup_root(ctx_t *c, const double *d, const double *e, double tnrm,
                      const blockjob_t *bj, int side, rrr_t *R, double *lo0,
                      double *hi0) {
  double tn, gl, gu, sigma;
  oracle_norms(bj->nb, d + bj->b0, e + bj->b0, &tn, &gl, &gu);
  c->spdiam = gu - gl;
  if (rrr_alloc(R, bj->nb)) return 6;
  if (oracle_root_rrr(bj->nb, d + bj->b0, e + bj->b0, tnrm, side,
                      c->o->perturb_root, c->o->seed, bj->b0, R->D, R->L, &sigma,
                      &c->st->root_retries)) {
    free(R->D); return 1;
  }
  rrr_derive(R);
  R->tau_hi = sigma; R->tau_lo = 0.0;
  root_interval(c, R, side, gl, gu, sigma, lo0, hi0);
  return 0;
}

int oracle_stemr(int64_t n, const double *d, const double *e, int range,
                 double vl, double vu, int64_t il, int64_t iu,
                 const oracle_opts_t *opts, int64_t *m, double *w, double *Z,
                 int64_t ldz, oracle_stats_t *stats) {
  /* O1 -- validate (argument numbers follow include/mrrr.h) */
  if (n < 1) return -1;
  if (!d) return -2;
  for (int64_t i = 0; i < n; ++i) if (!isfinite(d[i])) return -2;
  if (n > 1 && !e) return -3;
  for (int64_t i = 0; i < n - 1; ++i) if (!isfinite(e[i])) return -3;
  if (range < 0 || range > 2) return -4;
  if (range == ORACLE_RANGE_VALUE) {
    if (!isfinite(vl)) return -5;
    if (!isfinite(vu) || !(vl < vu)) return -6;
  }
  if (range == ORACLE_RANGE_INDEX) {
    if (il < 1 || il > n) return -7;
    if (iu < il || iu > n) return -8;
  }
  if (!m) return -9;
  if (!w) return -10;
  if (Z && ldz < n) return -12;
  oracle_opts_t dflt;
  if (!opts) { oracle_default_opts(&dflt); opts = &dflt; }
  oracle_stats_t stl;
  if (!stats) stats = &stl;
  memset(stats, 0, sizeof(*stats));
  *m = 0;

  /* O2, O3 */
  double tnrm, gl, gu;
  oracle_norms(n, d, e, &tnrm, &gl, &gu);
  int64_t *bs = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  if (!bs) return 6;
  int64_t nbk = oracle_split(n, d, e, tnrm, bs);

  /* O4 -- wanted local index range per block */
  blockjob_t *jobs = (blockjob_t *)calloc((size_t)nbk, sizeof(blockjob_t));
  if (!jobs) { free(bs); return 6; }
  double xa = 0, xb = 0;
  int64_t base_rank = 0;
  if (range == ORACLE_RANGE_INDEX && nbk > 1) {
    /* brackets of the il-th and iu-th eigenvalue of the split matrix */
    double wid = 4.0 * EPS * tnrm;
    double a = gl - 2 * wid - DBL_MIN, b = gu + 2 * wid + DBL_MIN;
    double lo = a, hi = b;
    while (hi - lo > wid && 0.5 * (lo + hi) > lo && 0.5 * (lo + hi) < hi) {
      double mid = 0.5 * (lo + hi);
      if (sturm_split(n, d, e, bs, nbk, mid) >= il) hi = mid; else lo = mid;
    }
    xa = lo;
    lo = a; hi = b;
    while (hi - lo > wid && 0.5 * (lo + hi) > lo && 0.5 * (lo + hi) < hi) {
      double mid = 0.5 * (lo + hi);
      if (sturm_split(n, d, e, bs, nbk, mid) >= iu) hi = mid; else lo = mid;
    }
    xb = hi;
  }
  for (int64_t b = 0; b < nbk; ++b) {
    blockjob_t *bj = &jobs[b];
    bj->b0 = bs[b]; bj->nb = bs[b + 1] - bs[b];
    const double *db = d + bj->b0, *eb = e ? e + bj->b0 : NULL;
    if (range == ORACLE_RANGE_ALL) { bj->wa = 1; bj->wb = bj->nb; }
    else if (range == ORACLE_RANGE_VALUE) {
      bj->wa = oracle_sturm_T(bj->nb, db, eb, vl) + 1;
      bj->wb = oracle_sturm_T(bj->nb, db, eb, vu);
    } else if (nbk == 1) { bj->wa = il; bj->wb = iu; }
    else {
      int64_t ca = oracle_sturm_T(bj->nb, db, eb, xa);
      bj->wa = ca + 1;
      bj->wb = oracle_sturm_T(bj->nb, db, eb, xb);
      base_rank += ca;
    }
  }

  ctx_t c;
  memset(&c, 0, sizeof(c));
  c.o = opts; c.st = stats; c.Z = Z; c.ldz = ldz; c.w = w;
  int vectors = (Z != NULL);
  int rc = 0;

  /* candidate values for ordering when there are several blocks */
  int64_t ncand = 0;
  for (int64_t b = 0; b < nbk; ++b) if (jobs[b].wb >= jobs[b].wa) ncand += jobs[b].wb - jobs[b].wa + 1;
  double *cval = NULL; int64_t *cblk = NULL, *cidx = NULL, *order = NULL;
  int64_t **posb = (int64_t **)calloc((size_t)nbk, sizeof(int64_t *));
  if (!posb) { rc = 6; goto done; }
  if (nbk == 1) {
    blockjob_t *bj = &jobs[0];
    posb[0] = (int64_t *)malloc(sizeof(int64_t) * (size_t)(bj->nb + 2));
    if (!posb[0]) { rc = 6; goto done; }
    for (int64_t j = 0; j <= bj->nb + 1; ++j) posb[0][j] = -1;
    for (int64_t j = bj->wa; j <= bj->wb; ++j) posb[0][j] = j - bj->wa;
    *m = bj->wb >= bj->wa ? bj->wb - bj->wa + 1 : 0;
  } else {
    /* O4/O11 -- values of every candidate (root bisection to 4 eps), merged by
     * (value, block, local index); INDEX keeps global ranks il..iu. */
    cval = (double *)malloc(sizeof(double) * (size_t)(ncand + 1));
    cblk = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncand + 1));
    cidx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncand + 1));
    order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncand + 1));
    if (!cval || !cblk || !cidx || !order) { rc = 6; goto done; }
    int64_t q = 0;
    for (int64_t b = 0; b < nbk; ++b) {
      blockjob_t *bj = &jobs[b];
      posb[b] = (int64_t *)malloc(sizeof(int64_t) * (size_t)(bj->nb + 2));
      if (!posb[b]) { rc = 6; goto done; }
      for (int64_t j = 0; j <= bj->nb + 1; ++j) posb[b][j] = -1;
      if (bj->wb < bj->wa) continue;
      if (bj->nb == 1) { cval[q] = d[bj->b0]; cblk[q] = b; cidx[q] = 1; q++; continue; }
      int side = (bj->wa + bj->wb <= bj->nb + 1) ? 1 : -1;
      rrr_t R; double lo0, hi0;
      rc = setup_root(&c, d, e, tnrm, bj, side, &R, &lo0, &hi0);
      if (rc) goto done;
      double prev = -INFINITY;
      for (int64_t j = bj->wa; j <= bj->wb; ++j) {
        double lo = lo0, hi = hi0;
        bisect(&c, &R, j, 4.0 * EPS, &lo, &hi);
        double v = R.tau_hi + 0.5 * (lo + hi);
        if (v < prev) v = prev;
        prev = v;
        cval[q] = v; cblk[q] = b; cidx[q] = j; q++;
      }
      free(R.D);
    }
    for (int64_t i = 0; i < ncand; ++i) order[i] = i;
    /* insertion sort by (value, block, index) -- plain and obviously correct */
    for (int64_t i = 1; i < ncand; ++i) {
      int64_t x = order[i], k = i - 1;
      while (k >= 0 && (cval[order[k]] > cval[x] ||
                        (cval[order[k]] == cval[x] && (cblk[order[k]] > cblk[x] ||
                         (cblk[order[k]] == cblk[x] && cidx[order[k]] > cidx[x]))))) {
        order[k + 1] = order[k]; k--;
      }
      order[k + 1] = x;
    }
    int64_t cnt = 0;
    for (int64_t b = 0; b < nbk; ++b) { jobs[b].wa = jobs[b].nb + 1; jobs[b].wb = 0; }
    for (int64_t i = 0; i < ncand; ++i) {
      int64_t qq = order[i];
      int64_t rank = base_rank + i + 1;
      if (range == ORACLE_RANGE_INDEX && (rank < il || rank > iu)) continue;
      int64_t b = cblk[qq], j = cidx[qq];
      posb[b][j] = cnt++;
      if (j < jobs[b].wa) jobs[b].wa = j;
      if (j > jobs[b].wb) jobs[b].wb = j;
    }
    *m = cnt;
  }

  /* main pass per block */
  for (int64_t b = 0; b < nbk && !rc; ++b) {
    blockjob_t *bj = &jobs[b];
    if (bj->wb < bj->wa) continue;
    if (bj->nb == 1) {
      int64_t p = posb[b][1];
      w[p] = d[bj->b0];
      if (Z) { for (int64_t i = 0; i < n; ++i) Z[p * ldz + i] = 0.0; Z[p * ldz + bj->b0] = 1.0; }
      continue;
    }
    int side = (bj->wa + bj->wb <= bj->nb + 1) ? 1 : -1;
    rrr_t R; double lo0, hi0;
    rc = setup_root(&c, d, e, tnrm, bj, side, &R, &lo0, &hi0);
    if (rc) break;
    int64_t nbk1 = bj->nb + 2;
    c.nb = bj->nb; c.gbase = bj->b0; c.pos = posb[b];
    c.lo = (double *)malloc(sizeof(double) * (size_t)nbk1);
    c.hi = (double *)malloc(sizeof(double) * (size_t)nbk1);
    c.wanted = (int *)calloc((size_t)nbk1, sizeof(int));
    c.z = (double *)malloc(sizeof(double) * (size_t)nbk1);
    if (!c.lo || !c.hi || !c.wanted || !c.z || alloc_ws(&c.ws, bj->nb)) { rc = 6; break; }
    for (int64_t j = bj->wa; j <= bj->wb; ++j) c.wanted[j] = 1;
    int64_t ma = bj->wa > 1 ? bj->wa - 1 : 1;            /* gap neighbours (reading 7) */
    int64_t mb = bj->wb < bj->nb ? bj->wb + 1 : bj->nb;
    double rtol = (vectors && nbk == 1) ? opts->rtol_class : 4.0 * EPS;
    for (int64_t j = ma; j <= mb; ++j) {
      c.lo[j] = lo0; c.hi[j] = hi0;
      bisect(&c, &R, j, rtol, &c.lo[j], &c.hi[j]);
    }
    if (!vectors) {
      for (int64_t j = bj->wa; j <= bj->wb; ++j)
        w[c.pos[j]] = R.tau_hi + 0.5 * (c.lo[j] + c.hi[j]);
    } else {
      for (int64_t j = bj->wa; j <= bj->wb; ++j) {
        double *col = Z + c.pos[j] * ldz;
        for (int64_t i = 0; i < n; ++i) col[i] = 0.0;
      }
      process_node(&c, &R, ma, mb, 0);
      if (c.err) rc = c.err;
    }
    free(R.D); free(c.lo); free(c.hi); free(c.wanted); free(c.z); free(c.ws.Dp);
    c.lo = c.hi = c.z = NULL; c.wanted = NULL; c.ws.Dp = NULL;
  }
  /* O11 -- monotone fix of w across nodes/blocks */
  if (!rc) for (int64_t j = 1; j < *m; ++j) if (w[j] < w[j - 1]) w[j] = w[j - 1];
done:
  if (posb) { for (int64_t b = 0; b < nbk; ++b) free(posb[b]); free(posb); }
  free(cval); free(cblk); free(cidx); free(order);
  free(jobs); free(bs);
  free(c.lo); free(c.hi); free(c.wanted); free(c.z); free(c.ws.Dp);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Brute-force cyclic Jacobi for dense symmetric A, n <= 512.   */
int oracle_jacobi(int64_t n, const double *A, double *w, double *V) {
  if (n < 1 || n > 512) return -1;
  double *a = (double *)malloc(sizeof(double) * (size_t)(n * n));
  double *v = (double *)malloc(sizeof(double) * (size_t)(n * n));
  if (!a || !v) { free(a); free(v); return 6; }
  memcpy(a, A, sizeof(double) * (size_t)(n * n));
  for (int64_t i = 0; i < n * n; ++i) v[i] = 0.0;
  for (int64_t i = 0; i < n; ++i) v[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0, tot = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        tot += a[i * n + j] * a[i * n + j];
        if (i != j) off += a[i * n + j] * a[i * n + j];
      }
    if (off <= 1e-34 * tot || off == 0.0) break;
    for (int64_t p = 0; p < n - 1; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        double apq = a[p * n + q];
        if (apq == 0.0) continue;
        /* rotation annihilating a_pq (textbook symmetric Schur decomposition) */
        double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        for (int64_t k = 0; k < n; ++k) { /* A <- A J (columns p, q) */
          double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = cs * akp - sn * akq;
          a[k * n + q] = sn * akp + cs * akq;
        }
        for (int64_t k = 0; k < n; ++k) { /* A <- J^T A (rows p, q) */
          double apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = cs * apk - sn * aqk;
          a[q * n + k] = sn * apk + cs * aqk;
        }
        for (int64_t k = 0; k < n; ++k) { /* V <- V J */
          double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = cs * vkp - sn * vkq;
          v[k * n + q] = sn * vkp + cs * vkq;
        }
      }
  }
  /* sort ascending (selection sort), permuting columns of V */
  int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  if (!idx) { free(a); free(v); return 6; }
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  for (int64_t i = 0; i < n; ++i) {
    int64_t b = i;
    for (int64_t j = i + 1; j < n; ++j) if (a[idx[j] * n + idx[j]] < a[idx[b] * n + idx[b]]) b = j;
    int64_t tmp = idx[i]; idx[i] = idx[b]; idx[b] = tmp;
  }
  for (int64_t j = 0; j < n; ++j) {
    w[j] = a[idx[j] * n + idx[j]];
    for (int64_t i = 0; i < n; ++i) V[i * n + j] = v[i * n + idx[j]];
  }
  free(idx); free(a); free(v);
  return 0;
}
