/*
 * mrrr.h -- C ABI of the B200-native fp64 MRRR symmetric tridiagonal
 * eigensolver (the hot path of arxiv 1205.2107, "PMRRR").
 *
 * Operation ("STEP"): for the real
 * symmetric tridiagonal T = tridiag(e, d, e) compute all, an index range
 * il..iu, or a value range (vl, vu] of its eigenpairs T z_j = lambda_j z_j by
 * the MRRR algorithm: root representation
 * L0 D0 L0^T = T - sigma0 I, bisection, classification by relative gap
 * (tol 1e-3, L1069-1075), a representation tree of shifted child
 * representations for clusters (L1092-1111) and, for every singleton, a
 * Rayleigh-quotient-corrected twisted factorization giving z_j (L1013-1043).
 *
 * Accuracy contract (BASELINE.json, PAPER.md Eq. (Tresnorm), (Torthogo)):
 * |lambda_j - lambda_j(T)| <= 4 n eps ||T||_1,
 * ||T z_j - lambda_j z_j||_2 <= 10 n eps ||T||_1, |Z^T Z - I| <= 10 n eps.
 *
 * Every pointer argument of mrrr_stemr is DEVICE memory (cudaMalloc'd or
 * managed) unless stated otherwise; all work is enqueued on `stream` and the
 * call synchronises `stream` before returning, so *m and the return code are
 * valid on return.  The library takes its device workspace from chunks it
 * owns per host thread and device and KEEPS between calls (a repeated solve
 * allocates nothing; mrrr_trim_workspace releases them, thread exit frees
 * them; sizes: mrrr_workspace_bytes, mrrr_stats_t.workspace_bytes).  The
 * caller owns d, e, w,
 * Z; d and e are NOT modified.  Re-entrant on distinct streams.  Results are
 * bitwise deterministic for identical inputs, options and device type.
 *
 * Return codes (LAPACK INFO style): 0 ok; -i: argument i invalid (numbering
 * below); 1 root RRR not found; 2 child RRR not acceptable; 3 tree depth cap
 * exceeded; 4 bisection/RQC non-convergence; 5 CUDA error; 6 out of device
 * memory; 7 collective (multi-GPU) error.  On error, outputs are unspecified.
 *
 * Process environment: a solve runs on up to 11 CUDA streams of its own (the
 * tree, the vector pieces, the Z download), and streams that share one of the
 * context's hardware work queues wait for one another.  When the library is
 * LOADED it therefore sets CUDA_DEVICE_MAX_CONNECTIONS=32 in the process
 * environment if (and only if) the variable is not set; the driver reads it
 * when the CUDA context is created, so a process that created its context
 * before loading the library, or set the variable itself, keeps its setting
 * (the results are the same; with the default 8 queues the headline solve is
 * ~5 % slower).  Nothing else in the environment is written; the MRRR_*
 * variables the library reads are diagnostics.
 */
#ifndef MRRR_H
#define MRRR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MRRR_RANGE_ALL = 0,   /* all n eigenpairs */
  MRRR_RANGE_INDEX = 1, /* il..iu, 1-based inclusive, ascending order */
  MRRR_RANGE_VALUE = 2  /* eigenvalues in (vl, vu] (Sturm-count semantics) */
} mrrr_range_t;

enum {
  MRRR_OK = 0,
  MRRR_ERR_ROOT = 1,
  MRRR_ERR_CHILD = 2,
  MRRR_ERR_DEPTH = 3,
  MRRR_ERR_CONVERGE = 4,
  MRRR_ERR_CUDA = 5,
  MRRR_ERR_NOMEM = 6,
  MRRR_ERR_COMM = 7
};

/* Options; pass NULL for the defaults from mrrr_default_opts(). */
typedef struct {
  double tol_relgap;   /* singleton threshold on the relative gap; 1e-3
                          (PAPER.md L1069-1072 footnote) */
  double rtol_class;   /* relative bracket width before classification and RQC;
                          2^-20 (reading 4) */
  int max_depth;       /* representation-tree depth cap (error 3 beyond); 128 */
  int perturb_root;    /* 1: seeded (1 + 4 eps u) relative perturbation of the
                          root D, L (reading 3); 0: off */
  uint64_t seed;       /* perturbation seed; default 0x1205210700000000 */
  int multisection;    /* shifts evaluated per eigenvalue per bisection round
                          (1 = plain bisection); default 4 */
  int grid_factor;     /* root grid points per wanted eigenvalue; default 4;
                          0 disables the grid stage */
  double rtol_vec;     /* singleton brackets refined to this relative width
                          before the RQC; 0 = none (default; reading 10) */
  int rqc_max;         /* twisted factorizations of the RQC before the
                          bisection fallback; default 10 (reading 10) */
  int shift_strategy;  /* 1 (default): an interior shift first for clusters of
                          >= 2000 members -- shallower trees (DESIGN.md
                          reading 30); 0: child shifts at the cluster ends
                          only (readings 8, 9) */
  double scratch_gb;   /* cap (GB) of each of the two large scratch areas: the
                          vector checkpoints (4 n B per eigenvector in flight)
                          and the cluster-step scratch (144 n B per cluster of
                          a level); default 16.  Smaller caps bound the device
                          workspace at the price of smaller vector pieces and
                          grouped cluster steps (random n=1e5, B200: 16 -> Z +
                          37 GB, 1.20 s; 4 -> Z + 12.9 GB, 1.38 s; 3 -> Z +
                          10.9 GB, 1.56 s; 2 -> Z + 8.8 GB, 1.90 s; DESIGN.md
                          section 4.6) */
} mrrr_opts_t;

void mrrr_default_opts(mrrr_opts_t *opts);

/*
 * mrrr_stemr -- eigenpairs of T on one GPU.
 *  (1) n       order of T, n >= 1.
 *  (2) d       device, d[n], diagonal; finite.
 *  (3) e       device, e[n-1], off-diagonal; finite (may be NULL if n == 1).
 *  (4) range   MRRR_RANGE_*.
 *  (5) vl      VALUE: lower bound (exclusive).
 *  (6) vu      VALUE: upper bound (inclusive), vl < vu.
 *  (7) il      INDEX: first index, 1 <= il <= n.
 *  (8) iu      INDEX: last index, il <= iu <= n.
 *  (9) m       HOST out: number of eigenpairs returned.
 * (10) w       device out: w[m] ascending eigenvalues.  Capacity n for ALL and
 *              VALUE, iu-il+1 for INDEX.
 * (11) Z       device out: column-major ldz x m; column j is the unit
 *              eigenvector of w[j] (zero outside its irreducible block).  NULL
 *              => eigenvalues only.  Same capacity as w in columns.
 * (12) ldz     leading dimension of Z, ldz >= n when Z != NULL.
 * (13) stream  cudaStream_t (as void*), NULL = legacy default stream.
 * (14) opts    NULL or options.
 */
int mrrr_stemr(int64_t n, const double *d, const double *e, int range,
               double vl, double vu, int64_t il, int64_t iu, int64_t *m,
               double *w, double *Z, int64_t ldz, void *stream,
               const mrrr_opts_t *opts);

/*
 * mrrr_stemr_dist -- the same solve sharded over P ranks (one GPU each) by
 * eigen-index range ("PMRRR's parallelism").  Every rank
 * passes the same T, range and opts.  Protocol, the paper's
 * static division and task types adapted to GPUs:
 *   - the root representation is computed on every rank;
 *   - the root grid and the root bisection work are split into P shares and
 *     gathered (two all-gathers; "gather");
 *   - the m wanted columns are divided statically (epp = ceil(m/P)) and, with
 *     one irreducible block and vectors, each cut moves to the nearest root
 *     cluster boundary within epp/40 (a share holds at most epp + epp/20
 *     columns);
 *   - every tree level: a rank computes the child representations of the
 *     clusters holding one of its columns and refines only the members it
 *     owns (a cluster shared by several ranks is the paper's type-3 task,
 *     P:L1176-1182); one all-gather of the brackets (+ a status word) per
 *     level gives every rank the same classification;
 *   - vectors only for the rank's columns, into Z_local (Z never moves);
 *   - a final all-gather of w (+ status).
 * Every rank calls the same sequence of collectives whatever happens; an
 * error on one rank is carried by the status word and every rank returns
 * the worst code at the same exchange.
 * The collective is `allgather`, a caller-provided all-gather over the ranks
 * (NCCL over NVLink in the Python binding):
 *   allgather(ctx, send, recv, bytes, stream): recv[r*bytes .. ] <- rank r's
 *   send (bytes each), device buffers, enqueued on `stream` (the library's
 *   solve stream); returns 0 on success.
 * Arguments 1-8 and 14 as in mrrr_stemr; further:
 *  (9)  rank, (10) nranks (1 <= nranks, 0 <= rank < nranks),
 *  (11) allgather, (12) allgather_ctx,
 *  (13) m (HOST out, global count), (15) col_begin, (16) m_local (HOST out:
 *       this rank's columns [col_begin, col_begin + m_local)),
 *  (17) w_all (device out, all m eigenvalues on every rank; capacity as w),
 *  (18) Z_local (device out, ldz x m_local; NULL = values only; capacity
 *       ceil(k/P) + ceil(k/P)/20 columns with k the capacity of w),
 *  (19) ldz, (20) stream.
 */
typedef int (*mrrr_allgather_fn)(void *ctx, const void *send, void *recv,
                                 size_t bytes, void *stream);
int mrrr_stemr_dist(int64_t n, const double *d, const double *e, int range,
                    double vl, double vu, int64_t il, int64_t iu, int rank,
                    int nranks, mrrr_allgather_fn allgather,
                    void *allgather_ctx, int64_t *m, const mrrr_opts_t *opts,
                    int64_t *col_begin, int64_t *m_local, double *w_all,
                    double *Z_local, int64_t ldz, void *stream);

/*
 * mrrr_stemr_nccl -- mrrr_stemr_dist on an NCCL communicator (the sharded
 * solve of PAPER.md L1125-1182 with the paper's gathers as ncclAllGather
 * over NVLink).  `nccl_comm` is an ncclComm_t (passed as
 * void* so that this header needs no nccl.h) of P ranks, one GPU each, whose
 * device is the calling thread's current device; rank and P are read from
 * it, and every all-gather of the protocol is enqueued on `stream` as
 * ncclAllGather(send, recv, bytes, ncclInt8, comm, stream).  NCCL is
 * resolved at run time (the libnccl.so.2 the process has loaded, else the
 * one on the loader path): the library does not link against it, and the
 * communicator stays the caller's (created and destroyed by the caller; no
 * other NCCL call of the caller may be in flight on it during the solve).
 * Arguments 1-8 as in mrrr_stemr; (9) nccl_comm; (10) m (HOST out, global
 * count); (11) opts; (12) col_begin, (13) m_local (HOST out); (14) w_all;
 * (15) Z_local; (16) ldz; (17) stream -- meaning, capacities and layout as
 * in mrrr_stemr_dist.  Returns as mrrr_stemr_dist (-i counts THIS entry's
 * arguments; -9: NULL communicator or one of another device), 7
 * (MRRR_ERR_COMM) if NCCL cannot be loaded or a collective fails.
 */
int mrrr_stemr_nccl(int64_t n, const double *d, const double *e, int range,
                    double vl, double vu, int64_t il, int64_t iu,
                    void *nccl_comm, int64_t *m, const mrrr_opts_t *opts,
                    int64_t *col_begin, int64_t *m_local, double *w_all,
                    double *Z_local, int64_t ldz, void *stream);

/*
 * mrrr_stemr_host -- the same solve with HOST buffers (end-to-end entry):
 * d[n], e[n-1], w[k] and Z (ldz x k, column major, or NULL) are host memory
 * (pinned or pageable; pinned is faster).  The call allocates device buffers
 * stream-ordered, copies d, e in, runs mrrr_stemr on `stream` and copies w
 * and the m columns of Z back before returning.  Arguments and return codes
 * as in mrrr_stemr.
 */
int mrrr_stemr_host(int64_t n, const double *d, const double *e, int range,
                    double vl, double vu, int64_t il, int64_t iu, int64_t *m,
                    double *w, double *Z, int64_t ldz, void *stream,
                    const mrrr_opts_t *opts);

/* The shard planner of mrrr_stemr_dist (host only, for tests): cuts[0..nranks]
 * start as the static division r * ceil(m/nranks); every inner cut moves to
 * the nearest column j with free_cut[j] != 0 (free_cut[m+1]: a cluster
 * boundary between columns j-1 and j) within ceil(m/nranks)/40, ties to the
 * left.  Returns 0 or -i for an invalid argument i. */
int mrrr_plan_columns(int64_t m, int nranks, const unsigned char *free_cut, int64_t *cuts);

/* Upper bound (bytes) of the device workspace mrrr_stemr holds for an
 * order-n problem with k wanted eigenpairs, EXCEPT the child representations
 * of the tree's cluster nodes: 16 n bytes per slot, and slots are recycled
 * once a node's child steps and vector pieces are done, so the pool holds
 * about the clusters of the levels whose vectors are in flight, not the whole
 * tree (random n=20000: 2448 slots for 2638 nodes; n=1e5: 3280 for 13241;
 * mrrr_stats_t.pool_bytes reports it).  The bound covers the O(n) arrays,
 * the per-eigenvalue slot arrays, the vector checkpoints (capped at 16 GB)
 * and the cluster-step scratch (capped at 16 GB; MRRR_SCRATCH_GB lowers both
 * caps). */
size_t mrrr_workspace_bytes(int64_t n, int64_t k);

/* Workspace is taken from library-owned device chunks per host thread and
 * device, kept between calls (repeated solves allocate nothing); the buffers
 * of mrrr_stemr_host come from a library-owned stream-ordered pool.  Releases
 * the calling thread's chunks (cudaFree: synchronises the device) and the
 * pool's cached memory; the next call re-grows them.  Must not run while a
 * call of this thread is in flight (calls are synchronous, so it cannot).
 * Returns 0 or MRRR_ERR_CUDA. */
int mrrr_trim_workspace(void);

/*
 * mrrr_negcount -- diagnostic entry: the Sturm count the bisection kernels
 * compute, N(mu) = #eigenvalues of L D L^T less than mu (PAPER.md L1061-1067
 * "bisection"), for a caller-given representation, one count
 * per shift.  Used by the -m gpu tests to compare the GPU counts with the
 * oracle's bit for bit.
 *  (1) nb     order of the representation, 1 <= nb <= 2^30.
 *  (2) D      device, D[nb] (pivots).
 *  (3) LLD    device, LLD[nb-1] = L_i^2 D_i (may be NULL if nb == 1).
 *  (4) k      number of shifts, k >= 0.
 *  (5) mu     device, mu[k].
 *  (6) count  device out, count[k] (int64).
 *  (7) mode   0: the kernels' division-free projective sweep
 *             with its qd fallback when the sweep over/underflows; 1: the qd
 *             fallback alone (differential stationary qd, a zero pivot's NaN
 *             ratio replaced by its limit 1, reading 5); 2: the
 *             refinement kernels' twisted count (reading 32):
 *             stationary over rows 0 .. r-1, progressive over rows nb-2 .. r,
 *             plus the sign of gamma_r, r = 16 * floor((nb - 1) / 32).
 *  (8) stream cudaStream_t (as void*); the call synchronises it.
 * Returns 0, -i for an invalid argument i, 5 (CUDA) or 6 (out of memory).
 * Allocates nb * 16 bytes of stream-ordered scratch, freed before return.
 */
int mrrr_negcount(int64_t nb, const double *D, const double *LLD, int64_t k,
                  const double *mu, int64_t *count, int mode, void *stream);

/* Metrics: how many twisted factorizations the Rayleigh-quotient correction
 * of each eigenpair took in the calling thread's last mrrr_stemr* call
 * (the paper's step is one inverse iteration on a
 * twisted factorization; reading 10 iterates it).  hist16[k], k =
 * 1 .. 14: eigenpairs (of this rank) that needed k factorizations; [15]: 15
 * or more; [0]: unused.  sum_k hist16[k] = eigenvectors computed by the
 * tree's vector kernels (1 x 1 blocks are not counted), sum_k k hist16[k] =
 * mrrr_stats_t.rqc_iters without the fallback passes.  HOST out, 16 entries.
 * Returns 0 or -1 (NULL). */
int mrrr_get_rqc_histogram(int64_t *hist16);

/* Static description of a return code. */
const char *mrrr_strerror(int code);

/* Instrumentation of the last call on this host thread (DESIGN.md
 * "Instrumentation"): counts and per-phase device times. */
typedef struct {
  int64_t nodes;            /* cluster nodes (child RRRs) created */
  int64_t levels;           /* tree levels processed */
  int64_t singletons;       /* eigenvectors computed */
  int64_t root_sweeps;      /* Sturm sweeps in root grid + bisection */
  int64_t refine_sweeps;    /* Sturm sweeps in child refinement */
  int64_t child_sweeps;     /* stationary transforms (candidates + accepted) */
  int64_t rqc_iters;        /* twisted factorizations in the vector phase */
  int64_t rqc_fallbacks;    /* vectors that needed the bisection fallback */
  int64_t safe_resweeps;    /* projective sweeps redone by the qd safe path */
  int64_t kernel_launches;  /* kernels launched by this call */
  double ms_root;           /* device time: prep + root RRR + root bisection */
  double ms_tree;           /* device time: classification, children, refine (the vector
                               pieces run beside it on side streams) */
  double ms_vectors;        /* device time after the tree: the vector tail + output */
  double ms_total;          /* device time of the whole call */
  /* per-kernel device time (CUDA events on the call's stream) and the units
   * they processed, for the roofline of bench.py */
  double ms_k_root_bisect;  /* root grid + multisection kernels */
  double ms_k_vectors;      /* singleton RQC + twisted + Z kernels: sum of the pieces'
                               event times (pieces overlap each other and the tree) */
  int64_t vec_tasks;        /* eigenvectors computed by that kernel */
  int64_t vec_elems;        /* sum over those tasks of their block order */
  double ms_k_final_refine; /* RQC fallback: bracket refinement to 4 eps (0 without fallback) */
  int64_t vec_nudges;       /* vector factorizations redone at a nudged shift (reading 25) */
  int64_t vec_items;        /* warp work items of the vector kernels (lanes: vec_tasks) */
  int64_t pool_bytes;       /* child-representation slots allocated (16 n B each; recycled) */
  int64_t workspace_bytes;  /* device workspace held by this thread after the call (all of it) */
  int64_t z_copies;         /* device-to-host copies of Z column runs (mrrr_stemr_host) */
} mrrr_stats_t;
int mrrr_get_stats(mrrr_stats_t *out);

/* Library version string. */
const char *mrrr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MRRR_H */
