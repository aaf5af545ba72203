/*
 * domdec.h — C-ABI of the B200 (sm_100a) hot path of arXiv 2405.09400,
 * "Flow updates for domain decomposition of entropic optimal transport".
 *
 * The library (libdomdec.so) runs single-scale entropic domain decomposition
 * on N1 x N2 pixel grids with squared-Euclidean cost:
 *   domdec_sweep  = DomDecIter on partition A or B (Alg. 1, PAPER.md:261-285,
 *                   realised as Alg. 4): BasicToComposite,
 *                   batched log-domain separable Sinkhorn, CompositeToBasic,
 *                   Balance, Truncate — one fused CUDA kernel;
 *   flow_update   = the flow update (Def. flow-update, steps
 *                   of §5.1) with product gluing candidates
 *                   (PAPER.md:552): edge costs, exact min-cost flow on the GPU,
 *                   apply flow — CUDA kernels;
 *   marginal_error / primal_dual_gap = diagnostics of App. A.2.2
 *                   (PAPER.md:1357-1359, 1395-1419).
 * The state is dual potentials plus basic-cell Y-marginals in bounding-box
 * form.  See DESIGN.md for the readings (R#) of the
 * points where the paper is silent.
 *
 * Conventions
 *  - Pixel (r, c) has physical centre (-1 + (r+1/2) h, -1 + (c+1/2) h);
 *    cost c(x, y) = |x - y|^2 (physical), i.e. h^2 |k - l|^2 in pixels.
 *  - Basic cell i = i1 * n2 + i2 covers rows [i1 s, i1 s + s) and columns
 *    [i2 s, i2 s + s); n1 = N1/s, n2 = N2/s, I = n1 n2.
 *  - Arc order of the 5-point neighbourhood: 0 self, 1 up
 *    (i1-1), 2 down (i1+1), 3 left (i2-1), 4 right (i2+1).  Per-arc arrays
 *    are [I][5] row-major, indexed by the SOURCE cell.
 *  - Boxes: off = (row, col) of the lower corner, ext = (rows, cols); the
 *    data of a box is row-major with row stride ext[1].
 *  - All work is ordered on the ctx's CUDA stream.  Calls that return host
 *    values synchronise that stream; domdec_sweep / flow_update with a NULL
 *    stats pointer are fully asynchronous (no host round trip).  Errors raised
 *    inside asynchronous kernels are sticky and are reported by the next
 *    synchronising call.  A ctx is not thread-safe.
 *  - Every function returns dd_status and never aborts; dd_last_error()
 *    gives a message.  The library owns all device memory it allocates.
 *  - There is no CPU fallback: without a usable CUDA device domdec_init
 *    returns DD_ERR_CUDA.
 */
#ifndef DOMDEC_H
#define DOMDEC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dd_ctx dd_ctx;

typedef enum {
  DD_OK = 0,
  DD_ERR_ARG = 1,      /* bad argument (NULL, eps <= 0, s not dividing N, ...) */
  DD_ERR_PRECOND = 2,  /* violated precondition of the method (zero-mass basic
                          cell PAPER.md:233, initial boxes not reproducing nu,
                          ||nu_i|| != m_i, ...)                                 */
  DD_ERR_NUMERIC = 3,  /* box capacity exceeded, NaN/Inf, min-cost flow failure */
  DD_ERR_CUDA = 4,     /* CUDA runtime error / no device                        */
  DD_ERR_OOM = 6       /* device allocation failed                              */
} dd_status;

typedef enum { DD_PART_A = 0, DD_PART_B = 1 } dd_partition;

/* Problem data, host memory, copied by domdec_init (caller keeps ownership). */
typedef struct {
  int32_t N1, N2;          /* pixels per axis                                   */
  double h;                /* grid spacing (2/N on [-1,1]^2)      */
  double eps;              /* entropic regularisation in physical units (> 0)   */
  int32_t cell_size;       /* s, basic cells are s x s pixels; must divide N1,N2*/
  const double *mu;        /* [N1*N2] >= 0, row-major; every basic cell > 0     */
  const double *nu;        /* [N1*N2] >= 0, sum nu = sum mu                     */
  /* initial coupling as basic-cell Y-marginals nu_i^0 in bounding-box form    */
  const int32_t *init_off; /* [I][2]                                            */
  const int32_t *init_ext; /* [I][2]                                            */
  const int64_t *init_pos; /* [I] start of box i in init_data                   */
  const double *init_data; /* concatenated row-major boxes, values >= 0         */
  int32_t mass_exponent;   /* E: min-cost-flow supplies q_i = rint(m_i 2^E)     */
                           /* (exact for the dyadic synthetic inputs)           */
} dd_problem;

typedef struct {
  double err;          /* Sinkhorn stopping tolerance Err; 1e-4 */
  int32_t max_iter;    /* per-cell iteration cap per sweep (paper silent); 2000 */
  int32_t fixed_iter;  /* > 0: parity mode, exactly this many passes per cell   */
  double trunc;        /* truncation threshold tau; 1e-15       */
  int32_t slot_cap;    /* capacity (elements) of one basic-cell box slot;      */
                       /* 0 = automatic from eps                                */
  int32_t comp_cap;    /* composite box side of the fast size class of the     */
                       /* sweep kernel (larger hulls go to a second, large-    */
                       /* shared-memory class on the device); 0 = automatic    */
  int32_t device;      /* CUDA device ordinal                                   */
  void *stream;        /* cudaStream_t to order all work on (NULL = the legacy */
                       /* default stream)                                       */
  int32_t track_primal; /* 1: every sweep also records the primal score of its */
                       /* plans (needed by primal_dual_gap; ~5% sweep time)    */
  int32_t row_begin;   /* stripe mode: this context owns basic-  */
  int32_t row_end;     /* cell rows [row_begin, row_end) (even, or row_end =   */
                       /* n1) and solves only the A-cells of those rows and the */
                       /* B-cells with 2 b1 in [row_begin, row_end) (+ the last */
                       /* B row when row_end = n1).  0, 0 = the whole grid.     */
                       /* The caller exchanges halo rows (domdec_halo_pack /    */
                       /* _unpack) and runs the flow update through the hooks  */
                       /* (flow_edge_costs, dd_mincost_flow, flow_apply).       */
} dd_options;

/* Filled by domdec_sweep when a non-NULL pointer is passed (synchronises). */
typedef struct {
  int64_t cells;          /* composite cells solved                            */
  int64_t nonconverged;   /* cells that hit max_iter (counted, not an error)   */
  int64_t iters_total;    /* sum of Sinkhorn passes                            */
  int32_t iters_max;
  int32_t overflow;       /* cells left unchanged because a box exceeded caps  */
  double l1x_entry;       /* sum_J e_J after the first pass (reading R14)      */
  double l1x_final;       /* sum_J e_J of the returned plans = L1 X-error      */
  double dropped_mass;    /* mass removed by truncation in this sweep          */
  double mufu_ops;        /* algorithmic ex2 + lg2 count of this sweep         */
  double bytes;           /* algorithmic HBM bytes of this sweep               */
} dd_sweep_stats;

/* Filled by flow_update when a non-NULL pointer is passed (synchronises). */
typedef struct {
  int32_t stationary;     /* 1: the stationary flow is optimal, nothing moved */
  int32_t certificate;    /* 1: stationarity proven by the negative-cycle test */
  int32_t refines;        /* cost-scaling refine phases run by the solver      */
  int32_t rounds;         /* push/relabel rounds run by the solver             */
  int32_t label_rounds;   /* Bellman-Ford rounds (certificate, global price    */
                          /* updates, price refinement); each is one grid-wide */
                          /* barrier like a push/relabel round                 */
  int64_t objective;      /* optimal sum_ij w_ij C_ij (integer costs, R11)     */
  int64_t changed_cells;  /* basic cells whose marginal was rewritten          */
  double solver_ms;       /* device time of the min-cost-flow kernel (its own  */
                          /* %globaltimer; 0 when the certificate held)        */
} dd_flow_stats;

/* Create a context: validate (DD_ERR_ARG / DD_ERR_PRECOND), copy the problem to
 * the device, build the A and B composite partitions (2x2 groups, B staggered
 * by one basic cell with ragged border groups, reading R4).  *out receives the
 * context; on error *out is NULL. */
dd_status domdec_init(const dd_problem *problem, const dd_options *options, dd_ctx **out);

/* One DomDecIter on partition A or B (Alg. 1 / Alg. 4).  Warm start: the X
 * potential of the previous sweep on the same partition (zero on the first,
 * reading R7).  Per-cell stopping rule (readings R6/R6'):
 * sum_x mu |r - 2^(A - A')| <= err mu(X_J) after the Y-update, with
 * r = ||nu_J|| / mu(X_J) (1 unless truncation removed mass).  Cells that hit
 * max_iter are counted in stats->nonconverged, not an error.  A cell whose
 * truncation would annihilate a member keeps its previous marginals (counted
 * in stats->overflow; a stats call returns DD_ERR_NUMERIC).  If the marginal
 * pool is exhausted the state is invalid: the sweep's stats call and every
 * later synchronising call (marginal_error, domdec_counters) return
 * DD_ERR_NUMERIC.  Cells are processed in size classes by hull side (one
 * fused kernel per class); the result of a cell
 * depends only on its inputs and its class.  stats may be NULL
 * (asynchronous). */
dd_status domdec_sweep(dd_ctx *ctx, dd_partition part, dd_sweep_stats *stats);

/* One flow update (Def. flow-update) using the plan costs of
 * the most recent sweep: edge costs (product candidates), integer instance
 * (C_ij = rint(c_bar_ij[px^2] * 1024), q_i = rint(m_i 2^E)), negative-cycle
 * certificate, exact min-cost flow (GPU cost scaling) if needed, apply flow
 * iff the optimal objective is < 0.  Requires a previous sweep
 * (DD_ERR_PRECOND otherwise).  The context keeps the last optimal flow and
 * its prices on the device and starts the next solve from them (the supplies
 * q are static, so that flow stays feasible); the result is still an exactly
 * optimal flow, possibly a different one of several optima.
 * stats may be NULL (asynchronous). */
dd_status flow_update(dd_ctx *ctx, dd_flow_stats *stats);

/* Change the regularisation of a context to eps (physical units, 0 < eps <=
 * the eps it was built with: the pools are sized for that one), keeping the
 * physical dual potentials: the stored potentials (units of eps, base 2) are
 * multiplied by eps_old / eps_new (eps-scaling, App. A.2.1 PAPER.md:1285-1287,
 * reading R24').  The coupling is unchanged; the next sweeps solve the cell
 * problems at the new eps.  Asynchronous.  DD_ERR_ARG for an eps out of range. */
dd_status domdec_set_eps(dd_ctx *ctx, double eps);

/* The hybrid iteration (Alg. 3) run to convergence on the
 * device: cycles of sweep(A), sweep(B) and, every flow_every-th cycle, a
 * flow update (flow_every = 0: plain DomDec, Alg. 2).
 * Stops at the first cycle whose sweep-entry errors of both partitions,
 * divided by ||mu||, are <= conv (reading R14), or after max_cycles.
 * The cycles are launched as CUDA-graph units of G = 2 (flow_every = 0) or
 * 2 flow_every cycles (an even number of pool flips, so one captured graph
 * replays; the first unit runs eagerly and allocates), with one 32 G-byte
 * device-to-host read of the per-cycle errors per unit; the state is
 * therefore advanced to the end of the unit, up to G - 1 cycles past the
 * converged one, and up to G - 1 past max_cycles.  Falls back to eager
 * launches of the same unit when capture is unavailable.
 * Outputs (each may be NULL): cycles = cycles executed; entry_error = the
 * error of the first converged cycle, else of the last one; moved_flows =
 * flow updates that changed the coupling (non-stationary).  Same results as
 * the equivalent sequence of domdec_sweep / flow_update calls.  Not in
 * stripe mode (DD_ERR_ARG).  Synchronises once per unit. */
dd_status domdec_run_cycles(dd_ctx *ctx, int32_t max_cycles, int32_t flow_every, double conv, int32_t *cycles,
                            double *entry_error, int32_t *moved_flows);

/* L1 marginal errors (Table rows), fp64:
 * l1_x = sum_x |P_X pi(x) - mu(x)| of the last sweep's plans,
 * l1_y = sum_y |sum_i nu_i(y) - nu(y)| of the stored basic-cell marginals.
 * Synchronises. */
dd_status marginal_error(dd_ctx *ctx, double *l1_x, double *l1_y);

/* Primal score E(pi) = <c,pi> + eps KL(pi|mu (x) nu) of the last sweep's plans,
 * dual score D(alpha†, beta†) of the stitched potentials (reading R15) and the
 * relative gap (E - D)/D; transport_cost = <c, pi>, all
 * in physical units (c = h^2 |k - l|^2).  alpha† = the last A-sweep potential
 * shifted per A-cell along the comb tree; beta† = its exact global Y-response
 * (dense separable fp64 LSE, 2 N1 N2 (N1 + N2) terms).  Needs at least one A
 * and one B sweep and a last sweep run with options.track_primal = 1
 * (DD_ERR_PRECOND otherwise).  Any output pointer may be NULL.  Synchronises. */
dd_status primal_dual_gap(dd_ctx *ctx, double *primal, double *dual, double *rel_gap,
                          double *transport_cost);

/* Copy the basic-cell marginals to host buffers (boxes concatenated in cell
 * order).  Pass data == NULL to query the required length in *data_len.
 * off/ext are [I][2], pos is [I].  Synchronises. */
dd_status domdec_export_cells(dd_ctx *ctx, int32_t *off, int32_t *ext, int64_t *pos,
                              double *data, int64_t data_cap, int64_t *data_len);

/* Copy the X potential a = alpha/eps (dimensionless, global pixel gauge) of the
 * last sweep on a partition to host [N1*N2]; each composite cell is shifted so
 * that its mu-weighted mean is 0 (potentials are unique only up to constants,
 * PAPER.md:216).  DD_ERR_PRECOND if the partition was never swept. */
dd_status domdec_export_alpha(dd_ctx *ctx, dd_partition part, double *alpha);

/* Checkpoint / resume: set the warm-start potential of a partition (reading
 * R7) from host [N1*N2] in the format of domdec_export_alpha (a = alpha/eps,
 * any constant per composite cell).  With a context built by domdec_init from
 * the boxes of domdec_export_cells, this resumes a solve: the next sweeps
 * start from the exported potentials instead of alpha = 0.  Synchronises.
 * DD_ERR_ARG for a non-finite value on a pixel of a composite cell. */
dd_status domdec_import_alpha(dd_ctx *ctx, dd_partition part, const double *alpha);

/* Per basic cell plan cost of the last sweep, Q_i m_i = <c, pi_i> in pixel^2
 * units (reading R13), host [I].  Synchronises. */
dd_status domdec_export_plan_cost(dd_ctx *ctx, double *Qm);

/* Per composite cell statistics of the last sweep on a partition, in the
 * partition's cell order (row-major over the composite-cell grid; stripe
 * mode: the cells this context solves): Sinkhorn passes iters [ncells], the
 * X-error after the first pass e0 and of the returned plan e (reading R14),
 * host arrays, any may be NULL.  *ncells receives the count (ncells may be
 * NULL).  DD_ERR_PRECOND if the partition was never swept.  Synchronises. */
dd_status domdec_export_cell_stats(dd_ctx *ctx, dd_partition part, int32_t *iters, double *e0, double *e,
                                   int32_t *ncells);

/* Step 1 of the flow update alone: edge costs of the current state.
 * cbar [I][5] fp64 pixel^2 units (NaN on arcs leaving the grid, 0 on self),
 * C [I][5] int64 integer costs, q [I] supplies.  Any pointer may be NULL. */
dd_status flow_edge_costs(dd_ctx *ctx, double *cbar, int64_t *C, int64_t *q);

/* Step 3 of the flow update alone: apply a host flow w [I][5] (int64, must
 * satisfy both divergence constraints with the ctx supplies q, else
 * DD_ERR_PRECOND): nu_hat_j = sum_i (w_ij / q_i) nu_i,
 * then truncate + minimal box. */
dd_status flow_apply(dd_ctx *ctx, const int64_t *w);

/* Edge candidates of the flow update (Def. edge-candidates PAPER.md:409-412,
 * Remark eps-gamma PAPER.md:543-559).  candidate 0: the
 * product candidate mu_j/m_j (x) nu_i/m_i (default, reading R12); 1: the
 * gluing candidate (Def. glued-plan) with gamma_ij the
 * entropic OT plan between mu_i/m_i and mu_j/m_j for |x - x'|^2 with
 * regularisation eps_gamma_p (pixel^2 units; the paper's (dx/2)^2 is 0.25;
 * small values approach the optimal plan).  Selecting 1 computes the static
 * gamma tables (fp64 Sinkhorn with eps-scaling, one warp per arc;
 * DD_ERR_NUMERIC if an arc misses the 1e-12 marginal tolerance; cell_size
 * <= 8) and makes every later sweep also record per pixel the plan's
 * X-marginal and conditional mean displacement, from which flow_update's
 * edge costs follow (reading R26).  The next flow update needs a
 * sweep run after this call.  Synchronises. */
dd_status flow_set_candidate(dd_ctx *ctx, int32_t candidate, double eps_gamma_p);

/* Device-pointer variants of the flow-update hooks, fully asynchronous on
 * the ctx stream (stripe mode: the instance is all-gathered
 * over NCCL as a device tensor and solved by every rank):
 *  flow_edge_costs_device: cbar / C of the current state into device
 *    buffers [I][5] (either may be NULL); only the rows whose plan moments
 *    this ctx holds are meaningful in stripe mode;
 *  flow_solve: exact min-cost flow of the global instance d_C [I][5] (device,
 *    integer costs, column 0 ignored) with the ctx's supplies, warm-started
 *    from the ctx's previous optimal flow and prices like flow_update; the
 *    optimal flow goes to d_w (device [I][5], may be NULL) and stays in the
 *    ctx for flow_apply_device.  stats != NULL synchronises;
 *  flow_apply_device: apply a device flow d_w [I][5] (no divergence check:
 *    use flow_apply for untrusted host flows). */
dd_status flow_edge_costs_device(dd_ctx *ctx, double *d_cbar, int64_t *d_C);
dd_status flow_solve(dd_ctx *ctx, const int64_t *d_C, int64_t *d_w, dd_flow_stats *stats);
dd_status flow_apply_device(dd_ctx *ctx, const int64_t *d_w);

/* Standalone exact min-cost flow on the n1 x n2 grid graph (Eq. MinCostFlow
 * PAPER.md:378-381 with the divergence constraints PAPER.md:350-354) on the
 * GPU: q [I] > 0 supplies, C [I][5] integer arc costs (column 0 ignored, arcs
 * leaving the grid ignored), |C| < 2^40.  Writes an optimal flow w [I][5] and
 * the optimal objective.  Host buffers; stream may be NULL.  stats may be NULL. */
dd_status dd_mincost_flow(int32_t n1, int32_t n2, const int64_t *q, const int64_t *C,
                          int64_t *w, int64_t *objective, dd_flow_stats *stats,
                          int32_t device, void *stream);

/* Global separable log-domain Sinkhorn on the whole N1 x N2 grid, no domain
 * decomposition: the SinkhornGPU comparator of the paper's benchmark
 * (Table).
 * Potentials in units of eps: a = alpha/eps on X, b = beta/eps on Y; cost in
 * pixel units, eps_p = eps/h^2 (eps' of SURVEY 8).  Iterates the Y-update
 * b(l) = -LSE_k[a(k) + log mu(k) - |k-l|^2/eps_p] and the X-update
 * a(k) = -LSE_l[b(l) + log nu(l) - |k-l|^2/eps_p] (Eq. entropic-transport
 * PAPER.md:196-202, separable stages PAPER.md:1145) until the L1 X-marginal
 * error after the Y-update, sum_k mu(k)|1 - exp(a(k) - a'(k))|, is
 * <= err * ||mu||, checked every check_every iterations, or
 * max_iter iterations ran (err = 0 with check_every = max_iter: exactly
 * max_iter iterations, parity mode).  Then one final Y-update.
 * mu, nu: host [N1*N2] row-major, >= 0, equal total mass (else
 * DD_ERR_PRECOND).  alpha: host [N1*N2], in = initial a (zeros for a cold
 * start), out = final a on supp(mu) (0 elsewhere); beta: host [N1*N2] out,
 * final b on supp(nu) (0 elsewhere).  iters, l1_x (last checked error),
 * solve_ms (CUDA-event time of the device iterations, host copies excluded)
 * may be NULL.  stream may be NULL.  Errors: DD_ERR_ARG (bad sizes/values),
 * DD_ERR_OOM, DD_ERR_CUDA, DD_ERR_NUMERIC (non-finite error); message via
 * dd_last_error(NULL).  fp64 potentials and terms, fp32 exp2 of shifted terms. */
dd_status dd_sinkhorn_global(int32_t N1, int32_t N2, const double *mu, const double *nu, double eps_p,
                             double err, int32_t max_iter, int32_t check_every, int32_t device,
                             void *stream, double *alpha, double *beta, int32_t *iters, double *l1_x,
                             double *solve_ms);

/* Cumulative work counters since domdec_init / domdec_reset_counters (for
 * roofline accounting without per-call synchronisation).  Synchronises. */
typedef struct {
  int64_t sweeps;         /* domdec_sweep calls                                */
  int64_t flow_updates;   /* flow_update calls                                 */
  int64_t cells;          /* composite-cell solves                             */
  int64_t iters;          /* Sinkhorn passes                                   */
  double mufu_ops;        /* algorithmic ex2 + lg2 of the sweeps   */
  double bytes;           /* algorithmic HBM bytes of the sweeps               */
} dd_counters;
dd_status domdec_counters(dd_ctx *ctx, dd_counters *out);
dd_status domdec_reset_counters(dd_ctx *ctx);

/* Measured ex2.approx.f32 throughput of the device (ops/s): a grid-wide
 * kernel of independent MUFU chains — the denominator of the sweep roofline
 * (DESIGN.md "Roofline"). */
dd_status dd_mufu_peak(int32_t device, double *ops_per_s);

/* Stripe halo exchange: serialise the basic-cell marginals of
 * basic-cell row `row` (n2 cells) into the DEVICE buffer buf of capacity cap
 * bytes (layout: int64 total bytes, int32 off[n2][2], int32 ext[n2][2], then
 * the fp64 boxes in cell order, row-major).  buf = NULL: *bytes receives the
 * exact size (synchronises).  Otherwise fully asynchronous on the ctx stream
 * (no host round trip; *bytes, if given, receives cap); a row larger than cap
 * is not written and makes the next synchronising call return
 * DD_ERR_NUMERIC.  domdec_halo_capacity gives a cap that holds any row whose
 * boxes fit the shared-memory size classes.  Valid for any row whose
 * marginals are current in this context. */
dd_status domdec_halo_pack(dd_ctx *ctx, int32_t row, void *buf, int64_t cap, int64_t *bytes);
dd_status domdec_halo_capacity(dd_ctx *ctx, int64_t *bytes);

/* Replace the marginals of basic-cell row `row` by the content of the DEVICE
 * buffer buf (as written by domdec_halo_pack of another context of the same
 * problem; bytes = its capacity).  Fully asynchronous: the boxes are appended
 * to the current pool by a device-side allocation; a full pool or a header
 * inconsistent with bytes makes the next synchronising call return
 * DD_ERR_NUMERIC. */
dd_status domdec_halo_unpack(dd_ctx *ctx, int32_t row, const void *buf, int64_t bytes);

/* ---- Multiscale domain decomposition ----------------
 * App. A.2.1 "Multi-scale and eps-scaling" runs every
 * solver coarse to fine (the strategy of [BoSch2020, Sec. 6.4]);
 * the paper gives no procedure, so the library follows DESIGN.md readings
 * R23-R25: layers N_l = N / 2^(L-1-l) with the same cell size, mu_l and nu_l
 * 2x2 block sums of the next finer layer; eps = eps' h_l^2 on every layer;
 * refinement nu_i'(y') = (nu_i(y) (m_i'/m_i)) (nu(y') / nu_l(y)) for a fine
 * cell i' in coarse cell i and a fine pixel y' in coarse pixel y, then
 * truncation + minimal box; the coarsest layer starts from the product
 * coupling nu_i = m_i nu. */

/* A context whose initial coupling is the product coupling mu (x) nu
 * (nu_i = m_i nu on the box of supp(nu), truncated at options->trunc), built
 * on the device.  problem->init_* are ignored.  Errors as domdec_init. */
dd_status domdec_init_product(const dd_problem *problem, const dd_options *options, dd_ctx **out);

/* A context for the next finer layer (R25): fine->N1 = 2 coarse N1 (same for
 * N2), same cell size; fine->mu / nu (host) must coarsen (2x2 sums) to the
 * coarse problem's mu / nu (DD_ERR_PRECOND otherwise).  The initial coupling
 * is the refinement of the coarse context's current basic-cell marginals,
 * computed on the device; fine->init_* are ignored.  The coarse context is
 * not modified (its stream is used and synchronised). */
dd_status domdec_refine(dd_ctx *coarse, const dd_problem *fine, const dd_options *options, dd_ctx **out);

typedef struct {
  int32_t levels;       /* layers L (1..16); the coarsest grid is N / 2^(L-1), with >= 2 basic cells per axis */
  int32_t max_cycles;   /* cap of hybrid cycles per layer                                   */
  int32_t flow_every;   /* flow update after every k-th cycle; 0 = pure domdec */
  double conv;          /* layer done when both sweep-entry errors / ||mu|| <= conv (R14)   */
  double eps_scale;     /* F >= 1: eps-scaling inside every layer (reading R24'):
                           stages eps' F, eps' F / 2, ..., eps', each until conv; F = 4 spans the
                           paper's factor 4 per layer, so a layer starts at the eps the coarser
                           one ended with.  <= 1: eps' fixed on every layer (R24).            */
  int32_t eps_stage_cycles; /* cycles of every stage but the last (0: each stage until conv);
                           the last stage always runs until conv (or max_cycles)             */
} dd_ms_options;

typedef struct {
  int32_t levels;
  int32_t N[16];        /* grid side of each layer (N1)                                      */
  int32_t cycles[16];   /* hybrid cycles run per layer                                       */
  int32_t flows[16];    /* non-stationary flow updates per layer                             */
  int32_t converged[16];
  double entry_error[16];   /* max of the A and B sweep-entry errors / ||mu|| of the last cycle */
  double seconds[16];   /* wall time per layer (initial coupling / refinement included)      */
  double init_seconds[16];  /* of which: building the layer's context (product / refinement) */
  double flow_seconds[16];  /* of which: flow updates                                        */
  double total_seconds; /* wall time of the whole call                                       */
} dd_ms_stats;

/* Coarse-to-fine hybrid solve of the problem (init_* ignored; eps' =
 * eps / h^2 is the final eps' of every layer, R24; with eps_scale > 1 every
 * layer first runs the larger eps' stages of R24').  cycles[l] sums the
 * stages; converged[l] is the last stage's.  On success *out is the finest
 * layer's context in its final state (query it with marginal_error,
 * primal_dual_gap, exports, or keep iterating).  stats may be NULL.
 * Synchronises once per cycle (convergence test). */
dd_status dd_multiscale_solve(const dd_problem *problem, const dd_options *options, const dd_ms_options *ms,
                              dd_ctx **out, dd_ms_stats *stats);

/* Release all device memory of ctx.  NULL is a no-op. */
dd_status domdec_destroy(dd_ctx *ctx);

/* Message of the last error on ctx (or of the last failed domdec_init /
 * dd_mincost_flow when ctx is NULL).  Never NULL. */
const char *dd_last_error(const dd_ctx *ctx);

/* Library build string (arch, version). */
const char *dd_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DOMDEC_H */
