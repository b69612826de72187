/*
 * dmk.h -- C ABI of the B200-native DMK library (libdmk.so, built for sm_100a).
 *
 * The library evaluates the discrete sum of arXiv 2308.00292 (Jiang & Greengard,
 * "A dual-space multilevel kernel-splitting framework"),
 *
 *     u_i = sum_{j : x_j != x_i} K(x_i - x_j) rho_j ,   i = 1..N      (Eq. 1.1)
 *
 * with sources = targets, by the discrete DMK algorithm of Sec. 3.5
 * with the PSWF kernel split of Sec. 3.6 (Eq. 3.66) and the
 * parameters of Table 1.  Coincident pairs (x_j == x_i, including
 * j == i) are omitted, as the paper's self-interaction rule prescribes (PAPER.md:524-541,
 * 1192-1195).
 *
 * Supported (dim, kernel) pairs -- anything else returns DMK_ERR_UNSUPPORTED:
 *   dim = 3, DMK_KERNEL_LAPLACE  K(r) = 1/r                (Eq. 3.1)
 *   dim = 3, DMK_KERNEL_YUKAWA   K(r) = exp(-lambda r)/r   (Sec. 4.6, Eqs. 4.17-4.18,
 *                                PAPER.md:2395-2440); needs opt->lambda > 0 and
 *                                lambda * side < 2 c (side = the root cube's side, c of
 *                                Table 1), else DMK_ERR_ARG / DMK_ERR_UNSUPPORTED
 *   dim = 2, DMK_KERNEL_LOG      K(r) = -log r             (Sec. 4.6 at lambda = 0 in 2D,
 *                                PAPER.md:2441-2447)
 *
 * Conventions for every entry point
 *   - Return value: DMK_OK (0) on success, a negative DMK_ERR_* code otherwise.  The
 *     message of the last failure on the calling thread is returned by dmk_last_error().
 *     On failure no output buffer is partially meaningful.
 *   - Memory: `mem` says where a caller pointer lives: DMK_MEM_DEVICE (CUDA device
 *     memory on the plan's device) or DMK_MEM_HOST (pageable or pinned host memory).
 *     The library never takes ownership of caller buffers.  A plan owns its device
 *     memory until dmk_destroy().
 *   - Streams: all device work of a plan is ordered on the stream given at plan time
 *     (0 = legacy default stream).  Everything is stream-ordered: dmk_plan() waits for
 *     one read-back of the tree sizes in the middle of the build, then enqueues the rest
 *     and returns WITHOUT a final synchronisation, so DMK_MEM_DEVICE points must stay
 *     valid until the plan's stream reaches that work (the Python binding keeps them
 *     alive until close()).  dmk_eval() / dmk_upward() / dmk_downward() with
 *     DMK_MEM_DEVICE buffers are asynchronous with respect to the host; with DMK_MEM_HOST
 *     buffers they return after the result is in host memory.  An error raised by
 *     asynchronous device work surfaces on a later call.  Internally a plan forks onto
 *     pooled side streams (near field at low priority, far field at high priority) and
 *     joins back into the plan stream before any result is visible there.
 *   - Precision (reading R16 of DESIGN.md; the north star's "FP64 or FP32 chosen per
 *     precision tier").  eps = 1e-9 (p = 28) and every 2D plan: all arithmetic and
 *     storage in IEEE fp64.  3D with eps in {1e-3, 1e-6} (p <= 18): the tree, the
 *     moments after anterpolation, c2p/p2c, prox2pw and the local expansions are fp64;
 *     the outgoing plane waves are STORED in fp32; anterpolation, the colleague
 *     translation, the back transforms, the leaf evaluation and the P2P pairs compute
 *     in fp32 (double-single point coordinates for P2P) with fp64 accumulation across
 *     blocks.  Contract: the potentials match the fp64 direct sum to relative l2 error
 *     <= 2 eps on every tier (tests/test_gpu_*.py).
 *   - Step-1 tables (Sec. 3.5 Step 1) are computed on the host on first use and cached
 *     per (device, kernel, Table 1 row, lambda * side); the Yukawa entries, which depend
 *     on the data's extent, are bounded (least recently used evicted; live plans keep
 *     theirs).
 *   - There is no CPU fallback: without a usable CUDA device every call fails with
 *     DMK_ERR_CUDA.
 */
#ifndef DMK_H
#define DMK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DMK_OK 0
#define DMK_ERR_ARG (-1)          /* invalid argument (null pointer, bad size, bad enum) */
#define DMK_ERR_UNSUPPORTED (-2)  /* valid but not implemented (dim, kernel, precision) */
#define DMK_ERR_CUDA (-3)         /* CUDA runtime / launch failure, or no device */
#define DMK_ERR_STATE (-4)        /* call out of order (e.g. stage query before eval) */

#define DMK_MEM_DEVICE 0
#define DMK_MEM_HOST 1

/* Kernels (see the (dim, kernel) table above). */
#define DMK_KERNEL_LAPLACE 0
#define DMK_KERNEL_YUKAWA 1
#define DMK_KERNEL_LOG 2

typedef struct dmk_plan_s* dmk_plan_t;

/* Optional plan parameters; pass NULL for defaults. */
typedef struct dmk_options {
  int32_t leaf_capacity;   /* n_s: a box holding more than n_s points is refined
                              (PAPER.md:804-806); default 200 */
  int32_t min_level;       /* 0 (default), or L >= 1: every box of levels < L exists and is
                              refined (empty or not) -- the shared coarse tree of a
                              distributed evaluation (see dmk_level_moments) */
  double lambda;           /* Yukawa parameter lambda > 0 (DMK_KERNEL_YUKAWA only) */
  void* stream;            /* cudaStream_t for all device work; NULL = default stream */
  const double* root;      /* NULL (default: root box from the points, reading R5), or a
                              HOST array {lo_0, .., lo_{dim-1}, side}: the root box
                              [lo, lo + side]^dim to use (all points must lie inside) */
  int64_t n_targets;       /* 0 (default: every point is a target), or t in [1, n]: only
                              the first t points (caller order) are targets; the others
                              are sources only and get no meaningful potential (the halo
                              of a distributed evaluation) */
} dmk_options;

/* dmk_plan: build the plan for N points in `dim` dimensions.
 *   dim      3 (DMK_KERNEL_LAPLACE, DMK_KERNEL_YUKAWA) or 2 (DMK_KERNEL_LOG).
 *   kernel   DMK_KERNEL_*; other (dim, kernel) pairs: DMK_ERR_UNSUPPORTED.
 *   eps      requested precision; snapped to the next tighter Table 1 row among
 *            {1e-3, 1e-6, 1e-9}.  eps < 1e-9: DMK_ERR_UNSUPPORTED.
 *   n        number of points, 1 <= n < 2^31.
 *   points   n x dim row-major fp64 (point i at points[dim*i .. dim*i+dim-1]), in `mem`;
 *            must be finite (DMK_ERR_ARG otherwise).
 *   opt      see dmk_options (may be NULL).
 *   out      receives the plan handle (NULL on failure).
 * Work done (Sec. 3.5 Step 0 and Step 1): bounding cube, Morton keys, stable sort,
 * adaptive 2:1-balanced 2^dim-tree, colleague / plane-wave / direct interaction lists --
 * all in CUDA kernels on the device -- plus the Step-1 tables (host, cached, see the
 * conventions above).  */
int dmk_plan(int dim, int kernel, double eps, int64_t n, const double* points, int mem,
             const dmk_options* opt, dmk_plan_t* out);

/* dmk_eval: potentials for one charge vector (Sec. 3.5 Steps 2-5).
 *   charges     n fp64 (caller's point order), in `mem`.
 *   potentials  n fp64 output (caller's point order), in `mem`; may not alias charges. */
int dmk_eval(dmk_plan_t plan, const double* charges, double* potentials, int mem);

/* dmk_eval in two halves, for a distributed evaluation (paper_2308_00292_b200/parallel.py):
 *   dmk_upward    Step 2: charges (caller order, n fp64 in `mem`) ->
 *                 Chebyshev moments of every F_out box, kept in the plan.
 *   dmk_downward  Steps 3-5 from the plan's moments -> potentials
 *                 (caller order, n fp64 in `mem`).  DMK_ERR_STATE before dmk_upward.
 * dmk_upward + dmk_downward == dmk_eval.  2D plans: dmk_upward only gathers; the whole
 * evaluation runs in dmk_downward. */
int dmk_upward(dmk_plan_t plan, const double* charges, int mem);
int dmk_downward(dmk_plan_t plan, double* potentials, int mem);

/* dmk_level_moments: read (set = 0) or overwrite (set = 1) the Chebyshev moments of
 * every box of `level` (< the plan's min_level, 3D only) as a dense array
 * [8^level][p][p][p] indexed by the box's Morton code at that level (fp64 in `mem`,
 * count = 8^level p^3; absent boxes read as 0).  set = 1 also rebuilds the levels above
 * from it by T_c2p (Lemma 2.2) -- the coarse-level exchange of a distributed
 * evaluation: each rank reads the moments its own charges give, the ranks sum them
 * (all-reduce), and each rank sets the sum before dmk_downward.  Call after
 * dmk_upward. */
int dmk_level_moments(dmk_plan_t plan, int level, double* dense, int64_t count, int mem, int set);

/* dmk_box_moments: read (set = 0) or overwrite (set = 1) the Chebyshev moments of the
 * listed boxes of `level` (< the plan's min_level, 3D only): codes[nbox] (int64 in `mem`)
 * are the boxes' Morton codes at that level (host codes outside [0, 8^level) fail with
 * DMK_ERR_ARG, device codes outside it are skipped), values[nbox][p][p][p] (fp64 in
 * `mem`).  With DMK_MEM_DEVICE the call is stream-ordered and does not synchronise.  A box
 * without an outgoing expansion reads nothing and ignores its values.  set = 1 does NOT
 * rebuild other levels (unlike dmk_level_moments): the sparse exchange of a locally
 * essential tree (paper_2308_00292_b200/parallel.py) -- every rank completes the moments
 * of the boundary boxes it needs at the levels between the dense all-reduce level and
 * min_level, then sets the dense level (which rebuilds the levels above it).  Call after
 * dmk_upward. */
int dmk_box_moments(dmk_plan_t plan, int level, const int64_t* codes, int64_t nbox, double* values, int mem, int set);

/* dmk_destroy: free the plan (NULL is a no-op). */
int dmk_destroy(dmk_plan_t plan);

/* Last error message of the calling thread ("" if none). */
const char* dmk_last_error(void);

/* Library version string. */
const char* dmk_version(void);

/* ---------------------------------------------------------------------------
 * Introspection (used by the stage-by-stage parity tests).  All outputs are host
 * buffers the caller sized from dmk_plan_info().
 * ------------------------------------------------------------------------- */
typedef struct dmk_plan_info {
  int64_t n;          /* points */
  int64_t nbox;       /* boxes kept: all non-leaf boxes + non-empty leaves */
  int32_t nlevels;    /* levels 0..nlevels-1 */
  int32_t p;          /* Chebyshev order (Table 1) */
  int32_t nf;         /* difference-kernel Fourier half-width, N_1 = 2 nf + 1 */
  int32_t nf0;        /* root-window Fourier half-width */
  int64_t nfout;      /* boxes with an outgoing expansion (F_out) */
  int64_t nexp;       /* boxes with a local expansion */
  int64_t ndlist;     /* total entries of the direct lists */
  double lo[3];       /* root cube corner */
  double side;        /* root cube side */
  double c;           /* PSWF parameter (Table 1) */
  int32_t respoly_degree; /* degree of the residual-kernel polynomial */
  int32_t dim;            /* 2 or 3 */
} dmk_plan_info;

int dmk_plan_info_get(dmk_plan_t plan, dmk_plan_info* info);

/* Tree arrays, copied to host.  `which` selects the array; element types/sizes:
 *   DMK_TREE_PERM        int64[n]        sorted position -> caller index
 *   DMK_TREE_BOX_LEVEL   int64[nbox]
 *   DMK_TREE_BOX_CODE    int64[nbox]     Morton code of the box at its level
 *   DMK_TREE_BOX_START   int64[nbox]     first sorted point of the box
 *   DMK_TREE_BOX_END     int64[nbox]     one past the last
 *   DMK_TREE_BOX_LEAF    int64[nbox]     1 = leaf
 *   DMK_TREE_BOX_PARENT  int64[nbox]     -1 for the root
 *   DMK_TREE_COLLEAGUES  int64[27*nbox]  slot (dx+1)*9+(dy+1)*3+(dz+1), -1 if absent
 *   DMK_TREE_DLIST_OFF   int64[nbox+1]   CSR offsets of the direct lists (empty for
 *                                         boxes that are not non-empty leaves)
 *   DMK_TREE_DLIST       int64[ndlist]   source leaves of each target leaf (any order)
 *   DMK_TREE_FOUT        int64[nbox]     rank among F_out boxes, -1 if not F_out
 *   DMK_TREE_EXP         int64[nbox]     rank among local-expansion boxes, -1 if none */
#define DMK_TREE_PERM 0
#define DMK_TREE_BOX_LEVEL 1
#define DMK_TREE_BOX_CODE 2
#define DMK_TREE_BOX_START 3
#define DMK_TREE_BOX_END 4
#define DMK_TREE_BOX_LEAF 5
#define DMK_TREE_BOX_PARENT 6
#define DMK_TREE_COLLEAGUES 7
#define DMK_TREE_DLIST_OFF 8
#define DMK_TREE_DLIST 9
#define DMK_TREE_FOUT 10
#define DMK_TREE_EXP 11
int dmk_tree_copy(dmk_plan_t plan, int which, int64_t* host_out);

/* Intermediate results of the last dmk_eval, copied to host (fp64):
 *   DMK_STAGE_MOMENTS  [nfout][p][p][p]     Chebyshev moments mu_n = sum_j rho_j T_n(xi_j)
 *                                            of each F_out box (proxy charges = V^{-T} mu,
 *                                            Def. 2.1)
 *   DMK_STAGE_OUTGOING outgoing plane waves Phi_l(B) (Eq. 3.42) of the F_out boxes in
 *                                            rank order, in the real parity-split form: the
 *                                            root (rank 0) first with [nf0+1][8][nf0+1][nf0+1]
 *                                            values, then every other box with
 *                                            [nf+1][8][nf+1][nf+1]: F[a][pi][b][c], a,b,c =
 *                                            |m1|,|m2|,|m3|, pi = 4 pi1 + 2 pi2 + pi3, and
 *                                            Phi(m) = sum_pi i^(pi1+pi2+pi3) sgn(m1)^pi1
 *                                            sgn(m2)^pi2 sgn(m3)^pi3 F[|m1|][pi][|m2|][|m3|]
 *   DMK_STAGE_LOCAL    [nexp][p][p][p]      Chebyshev coefficients of the local expansion
 *                                            Lambda (Eq. 3.43) incl. parent contributions
 *   DMK_STAGE_UFAR     [n]                  far-field potential, sorted order, unit cube
 *   DMK_STAGE_UNEAR    [n]                  residual + self terms, sorted order, unit cube */
#define DMK_STAGE_MOMENTS 0
#define DMK_STAGE_OUTGOING 1
#define DMK_STAGE_LOCAL 2
#define DMK_STAGE_UFAR 3
#define DMK_STAGE_UNEAR 4
int dmk_stage_copy(dmk_plan_t plan, int which, double* host_out, int64_t count);

/* Number of fp64 values dmk_stage_copy(plan, which, ...) expects (>= 0), or < 0 on error. */
int64_t dmk_stage_size(dmk_plan_t plan, int which);

/* Per-kernel timing of the last dmk_eval (milliseconds, CUDA events on the plan
 * stream); fills up to `cap` entries, returns the number of timed phases or < 0.
 * Names: "gather","anterp","c2p","prox2pw","pwlocal","p2c","eval","p2p".
 * Enabled only when the plan was created with env DMK_PROFILE=1. */
int dmk_eval_timings(dmk_plan_t plan, double* ms, const char** names, int cap);

/* Cumulative count of kernel launches issued by libdmk since the library was
 * loaded: its own kernels (return value) and CUB device-algorithm calls
 * (sort / scan / select, each one or more CUB kernels) in *cub_calls (may be NULL). */
int64_t dmk_kernel_launches(int64_t* cub_calls);

#ifdef __cplusplus
}
#endif
#endif /* DMK_H */
