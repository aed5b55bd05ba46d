/*
 * fdl.h -- C ABI of libfdl.so, the B200 (sm_100a) hot path of Wang & Wang's
 * SOR force-directed (stress-majorization) layout, arXiv 1711.01228.
 *
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of
 * SPEC.md, "DESIGN Rk" = reading k in DESIGN.md §3.
 *
 * The method (§2 and §4):
 *   stress      f(X) = sum_{i<j} w_ij (||x_i - x_j|| - d_ij)^2           Eq. 1
 *   ideal dist  d_ij = k * hop(i,j) (graph distance, DESIGN R1)
 *   weights     w_ij = d_ij^-2; d_ij^alpha for weight_exp = alpha (NEXT-3)
 *   one step    solve L^W X^{k+1} = L^{X^k} X^k with x_0 = 0              Eq. 2-5, Prop. 2.3
 *   relaxation  Xt = (1+omega) X^{k+1} - omega X^k                       Eq. 10
 *   guard       if f(Xt) <= f(X^{k+1}) then X^{k+1} <- Xt                 Algorithm 2 l.6-8
 *   stop        (f_old - f_new)/f_old < tol, or f_new = 0, or it = max_iter (DESIGN R4)
 * Vocabulary of BASELINE north_star: "repulsion" R = L^X X (the right-hand
 * side), "attraction" A = L^W X, "force" F = R - A = -1/2 grad f.
 *
 * Conventions (all functions):
 *   - Every function returns fdl_status; 0 = OK, < 0 = error.  No C++
 *     exception crosses the ABI.
 *   - Vertex ids are 0-based; id 0 is the paper's vertex 1, pinned at the
 *     origin.  Positions are n*dim doubles, row-major (x_i contiguous).
 *   - All pointer arguments are HOST pointers unless the name says otherwise.
 *     Inputs are copied; the caller keeps ownership of its buffers.  Output
 *     buffers are caller-allocated with the exact element count stated.
 *   - A context owns all device memory it uses; it is not thread-safe;
 *     distinct contexts are independent.  Calls that return host data
 *     synchronise the context stream.
 *   - After a CUDA error inside a context every later call on it returns
 *     FDL_E_STATE; fdl_last_error() explains.
 */
#ifndef FDL_H_
#define FDL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDL_ABI_VERSION 3  /* 2: fdl_strategy ENUM = 1, PROB = 2; fdl_ctx_info setup breakdown;
                              3: p1_split = 2 (predicted two-set steps), fdl_stats.p1_predicted* */

typedef struct fdl_ctx fdl_ctx; /* opaque; owned by the library */

typedef enum {
    FDL_OK = 0,
    FDL_E_INVALID_ARG = -1,    /* null pointer, bad size, bad parameter value             */
    FDL_E_SELF_LOOP = -2,      /* CSR has an edge (v, v)                           */
    FDL_E_DUPLICATE_EDGE = -3, /* CSR row lists a neighbour twice                 */
    FDL_E_ASYMMETRIC = -4,     /* (u,v) present but (v,u) missing: graph must be undirected */
    FDL_E_DISCONNECTED = -5,   /* graph not connected: d_ij undefined        */
    FDL_E_BAD_LENGTH = -6,     /* an edge length is not positive and finite       */
    FDL_E_DIAMETER = -7,       /* hop count exceeds 65535                                 */
    FDL_E_OOM = -8,            /* device allocation failed                                */
    FDL_E_CUDA = -9,           /* CUDA runtime error                                      */
    FDL_E_NCCL = -10,          /* NCCL error / NCCL library not loadable                  */
    FDL_E_SOLVER = -11,        /* CG hit cg_max_iter before cg_rtol (S:223 NoConvergence) */
    FDL_E_NONFINITE = -12,     /* stress became NaN/Inf                           */
    FDL_E_UNSUPPORTED = -13,   /* parameter combination not implemented                   */
    FDL_E_STATE = -14          /* context unusable after an earlier CUDA/NCCL error       */
} fdl_status;

typedef enum {
    FDL_STRAT_FIXED = 0, /* omega constant; omega = 0 is Algorithm 1           */
    FDL_STRAT_ENUM = 1,  /* omega* = argmin_c f((1+w_c) X^{k+1} - w_c X^k) over w_c = c * enum_step,
                            c = 0..enum_count-1 ({0, 0.5, ..., 9}); ties to the smaller
                            omega. Single GPU; no step cap                                  */
    FDL_STRAT_PROB = 2   /* roulette over {0.5,1,1.5,2} w.p. {.3,.3,.2,.2} each iteration */
} fdl_strategy;

typedef enum {
    FDL_STOP_NONE = 0,
    FDL_STOP_REL_TOL = 1,     /* (f_old - f_new)/f_old < tol */
    FDL_STOP_ZERO_STRESS = 2, /* f_new == 0                  */
    FDL_STOP_MAX_ITER = 3     /* it == max_iter              */
} fdl_stop_reason;

typedef struct {
    uint32_t struct_size; /* sizeof(fdl_params); set by fdl_params_default               */
    int32_t dim;          /* embedding dimension d >= 1; kernels built for 2 and 3 */
    double k;             /* ideal edge length, d_ij = k*hop_ij; k <= 0 -> n^(-1/dim) (DESIGN R2) */
    double omega;         /* relax factor omega >= 0 (Eq. 10)                                      */
    double step;          /* cap on ||xt_i - x^{k+1}_i|| per vertex; +INF = paper-exact (DESIGN R14) */
    double tol;           /* "rel err" of Table 1 > 0                                       */
    int32_t max_iter;     /* >= 1                                                                   */
    double weight_exp;    /* alpha in w = d^alpha, finite; -2 in the paper. alpha != -2 or
                             edge lengths use fp32 path-length tiles (NEXT-3)           */
    double cg_rtol;       /* PCG relative residual; <= 0 -> min(1e-2*tol, 1e-9): X^{k+1} solved to the
                             precision at which the trajectory is the exact solve's (DESIGN R8);
                             1e-2*tol is faster and reproduces it on C1-C3/C5 only    */
    int32_t cg_max_iter;  /* PCG cap per outer iteration; <= 0 -> min(10n, 10000)           */
    int32_t strategy;     /* fdl_strategy                                                           */
    uint64_t seed;        /* roulette stream seed (FDL_STRAT_PROB)                                  */
    int32_t device;       /* CUDA device ordinal                                                    */
    int32_t a_refresh;    /* L^W X^k for the PCG warm start is carried forward from the previous
                             solve (L linear: A' = b - r_cg, A(Xt) = (1+w)A' - wA^k) and recomputed
                             by a full L^W pass every a_refresh steps; 1 = every step; <= 0 -> 10 */
    int32_t hop_bits;     /* minimum stored hop width: 0 = auto (narrowest that holds the diameter:
                             4 bits if diam <= 15, 8 if <= 255, else 16), or 4, 8, 16. The decoded
                             hop, hence every result, is the same for every width   */
    int32_t cg_extrap;    /* PCG start.  2 (default): X^k + V y, the Galerkin (A-norm optimal)
                             correction over the last cg_history step differences V, L^W V from the
                             carried products (DESIGN R27); 1: X^k + rho (X^k - X^{k-1}) with
                             rho the previous step's least-squares ratio of successive
                             corrections (R23); 0: X^k.  The solve runs to cg_rtol
                             from any of them: same minimiser, different PCG counts */
    int32_t enum_count;   /* FDL_STRAT_ENUM candidates, 1..32 (default 19)                     */
    double enum_step;     /* FDL_STRAT_ENUM candidate spacing > 0 (default 0.5)                */
    int32_t p1_split;     /* line 6 pass over {X^{k+1}, Xt}: 1 = stresses of both + R(Xt) only, with a
                             1-set pass for R(X^{k+1}) when the guard rejects Xt (one host sync per
                             step); 0 = stresses and R of both in one pass; 2 = 1, but a step whose
                             guard is predicted to reject (the first step of a run, or the last
                             step accepted Xt with f(X^{k+1}) - f(Xt) < 0.6 (f(X^k) - f(X^{k+1})))
                             runs the two-set pass of 0 instead (DESIGN R30); -1 (default) = 2
                             when n^2 >= 2^30, else 0. Same results either way (bitwise)           */
    int32_t use_graphs;   /* 1: each step is one CUDA-graph launch (the PCG loop a device-side WHILE
                             node), one host sync per step; 0: kernels launched eagerly with a host
                             sync per PCG iteration; -1 (default): 1 on one GPU when the split
                             line-6 pass is off (n^2 < 2^30). Same results either way (bitwise).
                             With graphs the stats time whole steps only (p1_ms = p2_ms = 0)     */
    int32_t cg_history;   /* cg_extrap = 2: step differences kept for the start, 1..8 (0 = default 8;
                             fewer vectors take more PCG steps, DESIGN R27)                      */
} fdl_params;

typedef struct {
    int32_t it;            /* 1-based iteration number just completed                    */
    int32_t accepted;      /* 1 if the relaxed point Xt replaced X^{k+1} (Alg. 2 line 7) */
    int32_t cg_iters;      /* PCG iterations (= L^W matvec passes) in this step           */
    int32_t stop;          /* fdl_stop_reason after this step (0 = keep going)            */
    double omega;          /* relax factor used                                          */
    double f_before;       /* f(X^k)                                                     */
    double f_next;         /* f(X^{k+1}) before relaxation                               */
    double f_relaxed;      /* f(Xt); NaN when omega == 0 (not evaluated); ENUM: f(Xt(w*))  */
    double f_after;        /* f of the accepted point                                    */
    double rel_decrease;   /* (f_before - f_after)/f_before                              */
    double cg_relres;      /* max over columns of ||r||/||b|| at PCG exit                */
    double maxdisp;        /* max_i ||x^{k+1}_i - x^k_i|| (diagnostic, original units)   */
} fdl_iter_info;

typedef struct {
    int32_t iterations;    /* iterations run by this call                 */
    int32_t accepted;      /* how many relaxations were accepted          */
    int32_t stop;          /* fdl_stop_reason                             */
    int32_t cg_iters;      /* total PCG iterations                        */
    double f_initial;      /* f before the first iteration of this call  */
    double f_final;        /* f after the last iteration                  */
} fdl_run_info;

typedef struct {
    int32_t n, dim;
    int32_t diameter;      /* max hop count found by the BFS                     */
    int32_t hop_bits;      /* 4, 8 or 16 bits per stored hop                     */
    int32_t rank, world;
    int64_t tile0, tile1;  /* hop tiles stored by this context [tile0, tile1)   */
    int32_t iterations;    /* iterations run so far on this context              */
    double k;              /* resolved ideal edge length                        */
    double f;              /* current stress                                    */
    uint64_t hop_matrix_bytes; /* device bytes of the hop tiles (this rank)     */
    uint64_t local_pairs;      /* unordered vertex pairs in this rank's tiles   */
    uint64_t device_bytes;     /* all device memory held by the context         */
    double setup_ms;       /* MS-BFS + rowsum + first stress pass at create     */
    double setup_dist_ms;  /* ... of which the ideal distances (MS-BFS with its
                              device-side level loop, or Bellman-Ford)          */
    uint64_t bfs_bytes;    /* MS-BFS level-kernel gather bytes (neighbour frontier
                              words, visited and new-frontier words; 128 B each per
                              vertex searched per level), all batches and widths */
} fdl_ctx_info;

/* Kernel accounting of the hot path, accumulated since fdl_reset_stats. */
typedef struct {
    uint64_t launches;        /* kernels launched by the library                     */
    uint64_t p1_launches;     /* all-pairs repulsion + stress kernel launches (P1)   */
    uint64_t p2_launches;     /* all-pairs L^W matvec kernel launches (P2)           */
    uint64_t p1_pairs;        /* unordered pair x position-set evaluations by P1     */
    uint64_t p2_pairs;        /* unordered pairs evaluated by P2                     */
    uint64_t p1_pairs_x2;     /* ... of which in launches over two position sets     */
    double p1_ms, p2_ms;      /* CUDA-event time of P1 / P2 launches (needs timing on) */
    double other_ms;          /* CUDA-event time of everything else in fdl_step       */
    uint64_t steps;           /* fdl_step calls                                      */
    uint64_t cg_iters;        /* PCG iterations                                      */
    uint64_t p1_pairs_nor;    /* P1 pair x set evaluations of stress only (no R)     */
    uint64_t p1_rejected;     /* split P1 steps whose guard rejected Xt (extra 1-set pass) */
    uint64_t p1s_launches;    /* ... of the P1 launches: split line-6 passes (P1S)         */
    double p1s_ms;            /* ... and their CUDA-event time (included in p1_ms)       */
    uint64_t p1_predicted;    /* p1_split = 2: two-set line-6 passes run on a predicted rejection */
    uint64_t p1_predicted_rejected; /* ... of which the guard did reject Xt                */
} fdl_stats;

/* Fill *p with defaults: dim 2, k auto, omega 1.5, step +INF, tol 1e-4,
 * max_iter 500, weight_exp -2, cg_rtol auto, cg_max_iter auto, FIXED, seed 1,
 * device 0. */
void fdl_params_default(fdl_params* p);

/* Build a layout context on one GPU.
 *   n        number of vertices (>= 1)
 *   row_ptr  int64[n+1], CSR offsets; col_idx int32[row_ptr[n]] neighbour ids.
 *            The graph must be undirected (both directions stored), without
 *            self-loops or duplicate neighbours, and connected.
 *   edge_len NULL (unit lengths: d_ij = k * hop) or double[row_ptr[n]], one
 *            positive finite length per stored direction, equal for both
 *            directions (not checked: row v's entry is used for v<-u): d_ij = k * shortest path length (Kamada-Kawai,
 *            P:32; weighted networks P:250).  Non-positive or non-finite
 *            -> FDL_E_BAD_LENGTH.
 *   p        parameters (NULL -> defaults).
 *   init_pos n*dim doubles (row-major) or NULL for the seeded uniform unit-cube
 *            placement.  Translated so x_0 = 0.
 * Computes the ideal distances on the device (multi-source BFS for unit
 * lengths and alpha = -2; fp64 multi-source Bellman-Ford otherwise), the Jacobi
 * diagonal, and f(X^0), L^{X^0} X^0.  On error *out = NULL. */
fdl_status fdl_create(int32_t n, const int64_t* row_ptr, const int32_t* col_idx,
                      const double* edge_len, const fdl_params* p,
                      const double* init_pos, fdl_ctx** out);

/* Same, for rank `rank` of `world` GPUs of one node.  `nccl_unique_id` is the
 * 128-byte ncclUniqueId created by rank 0 and broadcast by the caller (e.g.
 * over torch.distributed).  Rank g stores and evaluates the hop tiles
 * [t0, t1) given by fdl_shard_tiles(n, world, g) (upper-triangle tiles of
 * 128 x 128 vertex pairs, row-major); every rank keeps the O(n) state
 * (positions, forces, PCG vectors) replicated.  After each pair pass the
 * per-rank partial sums are all-gathered over NCCL and summed in rank order,
 * so all ranks hold identical state.  Every rank must pass identical graph,
 * parameters and init_pos.  world = 1 with a non-NULL id runs the same
 * distributed path through a one-rank communicator (results identical to
 * fdl_create's; steps are launched eagerly, not as CUDA graphs).  The
 * enumerating strategy is single-GPU only (FDL_E_UNSUPPORTED here). */
fdl_status fdl_create_sharded(int32_t n, const int64_t* row_ptr, const int32_t* col_idx,
                              const double* edge_len, const fdl_params* p,
                              const double* init_pos, const uint8_t* nccl_unique_id,
                              int32_t rank, int32_t world, fdl_ctx** out);

/* In-process loopback group (test hook of the multi-GPU path): `world` contexts
 * created with fdl_create_loopback in one process, each driven from its own host
 * thread, exchange their partial sums through a host buffer and a host barrier
 * instead of NCCL (every all-gather of fdl_create_sharded becomes a stream sync,
 * a device->host copy of the rank's slice, a barrier and a host->device copy).
 * No kernel waits for another rank, so the ranks may share one GPU; the results
 * are those of the NCCL path (same data movement).  The group outlives its
 * contexts; fdl_group_destroy frees it. */
typedef struct fdl_group fdl_group;
fdl_status fdl_group_create(int32_t world, fdl_group** out);
void fdl_group_destroy(fdl_group* group);
fdl_status fdl_create_loopback(int32_t n, const int64_t* row_ptr, const int32_t* col_idx,
                               const double* edge_len, const fdl_params* p, const double* init_pos,
                               fdl_group* group, int32_t rank, fdl_ctx** out);

/* Test hook of the sharded path on one GPU.  fdl_create_sharded with
 * nccl_unique_id == NULL and world > 1 builds an EMULATED rank: it stores and
 * evaluates only its own tiles and has no communicator, so it accepts only
 * fdl_eval_partial, fdl_get_info and fdl_destroy (others: FDL_E_UNSUPPORTED).
 * fdl_eval_partial evaluates, at placement X (n*dim doubles, original units),
 * one symmetric pass over this context's tiles and returns this rank's dense
 * partial sums: mode 0 -> out = partial L^X X (n*dim), *stress = partial f;
 * mode 1 -> out = partial L^W X (n*dim).  Summing the partials of ranks
 * 0..world-1 gives the full quantities (what the NCCL path all-gathers). */
fdl_status fdl_eval_partial(fdl_ctx* ctx, int32_t mode, const double* X, double* out, double* stress);

/* Tile range [t0, t1) of `rank` of `world`: equal shares of the
 * nb(nb+1)/2 upper-triangle tiles (nb = ceil(n / FDL_TILE)) in row-major
 * triangle order. */
#define FDL_TILE 128
fdl_status fdl_shard_tiles(int32_t n, int32_t world, int32_t rank, int64_t* t0, int64_t* t1);

/* Create a 128-byte NCCL unique id (rank 0 calls this). */
fdl_status fdl_nccl_unique_id(uint8_t* out128);

/* Enqueue all subsequent work on `cuda_stream` (a cudaStream_t, e.g. a torch
 * stream).  NULL = the context's own stream. */
fdl_status fdl_set_stream(fdl_ctx* ctx, void* cuda_stream);

/* One Algorithm-2 iteration on the device; info may be NULL.
 * Errors: FDL_E_STATE once the run has stopped (info->stop of the last step says
 * why; fdl_set_positions restarts) or after an earlier CUDA error;
 * FDL_E_SOLVER if PCG reaches cg_max_iter before cg_rtol: the step is
 * not applied (placement, stress and iteration count stay those of X^k, in
 * eager and CUDA-graph launches alike; the graph's lines 5-8 sit in an IF node
 * on the solve's convergence flag), so the caller may raise cg_max_iter /
 * cg_rtol through a new context or stop;
 * FDL_E_NONFINITE if the stress becomes NaN/Inf. */
fdl_status fdl_step(fdl_ctx* ctx, fdl_iter_info* info);

/* Iterate until a stop rule fires (DESIGN R4: rel decrease < tol, f = 0, or
 * max_iter).  info may be NULL.  Errors as fdl_step. */
fdl_status fdl_run_until_converged(fdl_ctx* ctx, fdl_run_info* info);

/* Current placement into the caller's buffer (count must be n*dim, else
 * FDL_E_INVALID_ARG), original units, x_0 = 0.  Synchronises the stream; a
 * page-locked buffer is filled by one DMA. */
fdl_status fdl_get_positions(const fdl_ctx* ctx, double* out, size_t count);

/* Replace the placement (count n*dim, all finite, else FDL_E_INVALID_ARG);
 * re-pins x_0 = 0, recomputes f, L^X X and L^W X at it (one fused pass)
 * and clears the stop flag (checkpoint resume / interactive layouts / parity).
 * The recycled PCG basis (DESIGN R27) belongs to L^W and is kept.  A placement
 * bitwise equal to the current one as fdl_get_positions returns it (a caller
 * that round-trips its layout through the host) keeps the context's state as it
 * is (f, forces, PCG history; no evaluation pass) and only clears the stop flag. */
fdl_status fdl_set_positions(fdl_ctx* ctx, const double* in, size_t count);

/* Per-vertex relax factors omega_i >= 0 (§6 (1), line 410:
 * x~_i = x_i^{k+1} + omega_i (x_i^{k+1} - x_i^k)), count = n, replacing the
 * scalar omega of Eq. 10 in every later step until cleared with omega = NULL.
 * The guard (lines 6-8) still compares f(X~) with f(X^{k+1}).  Requires the
 * fixed strategy (FDL_E_UNSUPPORTED otherwise); X~ is then not a scalar
 * combination of X^{k+1} and X^k, so L^W X^k is recomputed by a full pass
 * each step instead of being carried.  The array is copied. */
fdl_status fdl_set_omega_vertex(fdl_ctx* ctx, const double* omega, size_t count);

/* Forces at the current placement, original units (each n*dim, may be NULL):
 * R = L^X X ("repulsion"), A = L^W X ("attraction"); *stress = f(X). */
fdl_status fdl_eval_forces(fdl_ctx* ctx, double* R, double* A, double* stress);

/* Hop counts of rows [r0, r0+nrows): out[r*n + j] = hop(r0 + r, j), gathered from
 * the stored upper triangle (FDL_E_INVALID_ARG if an entry lives on another rank). */
fdl_status fdl_get_hop_rows(fdl_ctx* ctx, int32_t r0, int32_t nrows, uint16_t* out);

/* Ideal distances d_ij = k x (shortest path length) of rows [r0, r0+nrows),
 * original units, out[r*n + j] (n*nrows doubles), any stored width (hop tiles or
 * the fp32 path lengths of weighted graphs / general alpha). */
fdl_status fdl_get_dist_rows(fdl_ctx* ctx, int32_t r0, int32_t nrows, double* out);

/* Jacobi diagonal sum_{j != i} w_ij of all n rows, original units (count = n). */
fdl_status fdl_get_diag(fdl_ctx* ctx, double* out, size_t count);

/* Geometry, sizes and current state of the context (never fails on a valid ctx). */
fdl_status fdl_get_info(fdl_ctx* ctx, fdl_ctx_info* info);

/* Kernel statistics.  With timing on, every P1/P2 launch and the rest of each
 * step are bracketed by CUDA events on the context stream. */
fdl_status fdl_set_timing(fdl_ctx* ctx, int32_t enable);
fdl_status fdl_get_stats(fdl_ctx* ctx, fdl_stats* out);
fdl_status fdl_reset_stats(fdl_ctx* ctx);

/* FFMA-chain microbenchmark on `device`: achieved FP32 FLOP/s of a kernel that
 * issues only FFMA (the measured FP32 roofline denominator). */
fdl_status fdl_bench_ffma(int32_t device, double* tflops, double* ms);

/* Ceiling of the line-6 pass (P1S) on `device`: the same per-tile function the
 * pass runs (hop decode, pair arithmetic, j-side stores; 2-D, 4-bit hops 1..8)
 * repeated on one tile resident in shared memory, at the pass's occupancy, with
 * no HBM traffic, TMA pipeline or reductions.  *tflops counts the pass's 29
 * algorithmic flops per unordered pair. */
fdl_status fdl_bench_p1s_mix(int32_t device, double* tflops, double* ms);
/* Same for the PCG matvec pass (P2, product form): *hop_gbs = the pass's
 * algorithmic hop bytes (0.5 B per unordered pair at 4 bits) per second. */
fdl_status fdl_bench_p2_mix(int32_t device, double* hop_gbs, double* ms);

const char* fdl_status_str(fdl_status s);
const char* fdl_last_error(const fdl_ctx* ctx); /* valid until the next call on ctx */
void fdl_destroy(fdl_ctx* ctx);                 /* NULL-safe */
int32_t fdl_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FDL_H_ */
