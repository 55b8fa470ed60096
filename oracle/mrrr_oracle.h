/*
 * mrrr_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, sequential, fp64 CPU implementation of the MRRR symmetric tridiagonal
 * eigensolver ("The MRRR algorithm"), written step by step
 * from the paper plus the readings of SURVEY.md §8(c) O1-O12 (listed in
 * DESIGN.md "Readings").  It is the parity oracle for the CUDA path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library.  It shares no code, header, table or constant generator with
 * paper_1205_2107_b200/ (the product); neither includes the other.
 *
 * Compiled with: gcc -O2 -fno-fast-math -ffp-contract=off (no FMA contraction,
 * IEEE division).
 */
#ifndef MRRR_ORACLE_H
#define MRRR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_RANGE_ALL = 0, ORACLE_RANGE_INDEX = 1, ORACLE_RANGE_VALUE = 2 };

typedef struct {
  double tol_relgap;  /* singleton threshold, 1e-3 (PAPER.md L1069-1072 footnote) */
  double rtol_class;  /* relative bracket width before classification / RQC, 2^-20 */
  int max_depth;      /* representation-tree depth cap, 128 (error 3 beyond) */
  int perturb_root;   /* 1: seeded (1+4eps*u) perturbation of root D, L (reading 3) */
  uint64_t seed;      /* perturbation seed */
  double rtol_vec;    /* singleton bracket refinement before the RQC; 0 = none (reading 10) */
  int rqc_max;        /* RQC factorizations before the bisection fallback; 10 (reading 10) */
  int shift_strategy; /* 1 (default): an interior candidate first for large clusters (reading 30);
                         0: shifts at the cluster ends only (readings 8, 9) */
} oracle_opts_t;

typedef struct {
  int64_t negcount_sweeps;     /* O6 sweeps (bisection + refinement + bracket checks) */
  int64_t negcount_resweeps;   /* O6 NaN-safe re-sweeps */
  int64_t child_sweeps;        /* O9 stationary transforms (candidates) */
  int64_t twisted;             /* O10 twisted factorizations */
  int64_t twisted_resweeps;    /* NaN-safe re-sweeps inside O10 */
  int64_t rqc_fallbacks;       /* O10 bisection fallbacks */
  int64_t nodes;               /* cluster nodes created (child RRRs accepted) */
  int64_t max_depth;           /* deepest node */
  int64_t singletons;          /* vectors computed */
  int64_t root_retries;        /* O5 delta doublings */
  int64_t tier[4];             /* O9 acceptance tier counts (i)..(iv) */
  int64_t rqc_hist[12];        /* factorizations per vector (index = count, 11 = >10) */
  int64_t interior;            /* clusters whose child took the interior shift (reading 30) */
} oracle_stats_t;

void oracle_default_opts(oracle_opts_t *o);

/* Full solver.  Same contract as include/mrrr.h mrrr_stemr but on HOST memory:
 * d[n], e[n-1] read-only; w[m] ascending; Z (ldz x m, column major) or NULL for
 * values only.  il/iu 1-based inclusive (INDEX); (vl,vu] (VALUE).
 * Returns 0, -i for invalid argument i, 1 root RRR failure, 2 child RRR not
 * acceptable, 3 depth cap, 4 non-convergence, 6 out of memory. */
int oracle_stemr(int64_t n, const double *d, const double *e, int range,
                 double vl, double vu, int64_t il, int64_t iu,
                 const oracle_opts_t *opts, int64_t *m, double *w, double *Z,
                 int64_t ldz, oracle_stats_t *stats);

/* ---- step functions, exported for unit pins (tests/test_oracle_*.py) ---- */

/* O2: ||T||_1, Gershgorin bounds. */
void oracle_norms(int64_t n, const double *d, const double *e, double *tnrm,
                  double *gl, double *gu);
/* O3: irreducible blocks; bstart[0..nb] (bstart[nb] = n). Returns nb. */
int64_t oracle_split(int64_t n, const double *d, const double *e, double tnrm,
                     int64_t *bstart);
/* O5: root RRR of one block (rows gbase..gbase+nb-1).  side=+1 left (D>0),
 * -1 right (D<0).  Outputs D[nb], L[nb-1], sigma.  Returns 0 or 1. */
int oracle_root_rrr(int64_t nb, const double *d, const double *e, double tnrm,
                    int side, int perturb, uint64_t seed, int64_t gbase,
                    double *D, double *L, double *sigma, int64_t *retries);
/* O6: number of eigenvalues of L D L^T below mu (zero pivot counted negative). */
int64_t oracle_negcount(int64_t nb, const double *D, const double *LLD,
                        double mu, double pivmin, int *resweep);
/* Classic Sturm count on T itself (T - xI = L D L^T), used for VALUE/INDEX
 * range selection over split blocks. */
int64_t oracle_sturm_T(int64_t n, const double *d, const double *e, double x);
/* O8: boundaries; out[j] = 1 iff a boundary lies between j and j+1
 * (0-based, j = 0..k-2). */
void oracle_classify(int64_t k, const double *lo, const double *hi, double tol,
                     int *out);
/* O9.2: child RRR by the stationary transform L+D+L+^T = LDL^T - sigma I.
 * Returns 0 if all D+ finite, else 1.  growth = max |D+_i|. */
int oracle_child_rrr(int64_t nb, const double *D, const double *L,
                     const double *LD, double sigma, double *Dp, double *Lp,
                     double *growth);
/* O10 steps 1-4 (one twisted factorization + solve) at lambda.
 * Outputs z[nb] (z_r = 1, unnormalised), r (0-based), gamma_r, negcount. */
int oracle_twisted(int64_t nb, const double *D, const double *L,
                   const double *LD, const double *LLD, double lambda,
                   double pivmin, double *z, int64_t *r, double *gamma,
                   int64_t *negc);
/* Dense cyclic Jacobi for symmetric A (n x n, row major, n <= 512);
 * w ascending, V columns (row-major V[i*n+j] = component i of vector j). */
int oracle_jacobi(int64_t n, const double *A, double *w, double *V);
/* splitmix64-based counter generator for the root perturbation (reading 3):
 * u in [-1,1) for (seed, global row, tag 0=D / 1=L). */
double oracle_perturb_u(uint64_t seed, int64_t grow, int tag);

#ifdef __cplusplus
}
#endif
#endif
