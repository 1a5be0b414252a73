/*
 * tga.h -- C ABI of the B200-native full-neighbourhood VRP move evaluator.
 *
 * The hot path of arXiv 2506.17357 ("Speeding up Local Optimization in
 * Vehicle Routing with Tensor-based GPU Acceleration", TGA): for every
 * candidate of the 2-opt, 2-opt*, relocate, swap, or-opt and cross-exchange
 * operators, compute the delta cost and the capacity / time-window
 * feasibility from per-position attribute records, reduce to the best move,
 * and apply it with an incremental attribute rebuild.
 *
 * Citations: P:n = PAPER.md line n (with its section / equation).
 *   Problem statement and inputs .......... §2, P:49-58 (Eq. 1)
 *   Concatenation algebra ................. §4.3, Eq. 2,
 *                                           Eq. 3e-f, Eq. 4
 *   Workflow (init / evaluate / update) ... §5.1; Alg. A2
 *   Operators ............................. §4.1, Fig. `operators` P:107-149
 *   Evaluation + argmin ................... §5.3.4, Eq. 16
 *   Tensor update ......................... §5.3.5
 *
 * Conventions (all calls):
 *   - Every function returns an int32 status: TGA_OK (0), a positive
 *     informational code, or a negative error.  Nothing aborts and no C++
 *     exception crosses the boundary.  tga_last_error() returns a
 *     thread-local message for the last failing call on this thread.
 *   - Host pointers passed in are only read during the call (the library
 *     copies what it keeps); the caller keeps ownership.  Opaque objects are
 *     owned by the library and freed by their *_destroy.  A solution must not
 *     outlive its instance.
 *   - One host thread at a time per solution object.
 *   - Node 0 is the depot; customers are 1..n_nodes-1.
 *   - Travel time equals travel distance (T = C), as in the GH/Solomon
 *     convention; the inter-route kernels require a symmetric matrix.
 */
#ifndef TGA_H
#define TGA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
#define TGA_OK                    0
#define TGA_NO_IMPROVING_MOVE     1   /* best score >= 0, or every candidate infeasible */
#define TGA_ERR_INVALID_ARGUMENT (-1) /* sizes, e > l, d < 0, non-zero diagonal, capacity <= 0, NULL */
#define TGA_ERR_STRUCTURE        (-2) /* routes do not cover every customer exactly once / id out of range */
#define TGA_ERR_STALE            (-3) /* move from an older solution generation */
#define TGA_ERR_UNSUPPORTED      (-4) /* 2-opt on a time-windowed instance; asymmetric C; T != C */
#define TGA_ERR_CUDA             (-5)
#define TGA_ERR_NCCL             (-6)
#define TGA_ERR_OOM              (-7)

/* ------------------------------------------------------------ data types */
#define TGA_I32 0   /* integer distances (CVRP nint; VRPTW integer tenths) -> exact */
#define TGA_F32 1   /* real distances/times held in fp32 on the device            */

/* ------------------------------------------------------------ move variants
 * A variant is an operator with fixed segment lengths.  Its id is its rank in
 * the deterministic tie-break "lowest (score, variant, flat index)"
 * (reading 5 in DESIGN.md).  Candidate spaces (canonical slots):
 *   2OPT        intra, reverse customers u..v of one route (CVRP only)
 *   2OPT_STAR   inter, cut after slot u of route a and v of route b, route(u)<route(v)
 *   RELOCATE1   inter, move customer u after slot v of another route
 *   OROPT2/3    inter, move the segment u..u+N-1 (N=2,3) after slot v of another route
 *   SWAP11      inter, exchange customers u and v, route(u)<route(v)
 *   CROSSn1n2   inter, exchange segment u..u+N1-1 with v..v+N2-1 (N1<=N2; N1==N2 => route(u)<route(v))
 *   IRELOCATEn  intra, move segment u..u+N-1 after the node originally at slot v
 *   ISWAPn1n2   intra, exchange segments at u (length N1) and v (length N2), u+N1<=v
 * Reversed-segment variants ("Relocate and Swap can incorporate reversed subsequences by
 * exchanging the first and last node index tensors, as in 2-opt"):
 *   OROPTnR     inter, OROPTn with the segment inserted reversed (n = 2, 3)
 *   CROSSnnR    inter, CROSSnn with both segments inserted reversed (n = 2, 3), route(u)<route(v)
 * They rank after the 23 standard variants in the tie-break; TGA_OP_STANDARD is the
 * standard set (the benchmarked neighbourhood), TGA_OP_ALL includes the reversed ones.
 */
enum {
    TGA_V_2OPT = 0,
    TGA_V_2OPT_STAR = 1,
    TGA_V_RELOCATE1 = 2, TGA_V_OROPT2 = 3, TGA_V_OROPT3 = 4,
    TGA_V_SWAP11 = 5,
    TGA_V_CROSS12 = 6, TGA_V_CROSS13 = 7, TGA_V_CROSS22 = 8, TGA_V_CROSS23 = 9, TGA_V_CROSS33 = 10,
    TGA_V_IRELOCATE1 = 11, TGA_V_IRELOCATE2 = 12, TGA_V_IRELOCATE3 = 13,
    TGA_V_ISWAP11 = 14, TGA_V_ISWAP12 = 15, TGA_V_ISWAP13 = 16,
    TGA_V_ISWAP21 = 17, TGA_V_ISWAP22 = 18, TGA_V_ISWAP23 = 19,
    TGA_V_ISWAP31 = 20, TGA_V_ISWAP32 = 21, TGA_V_ISWAP33 = 22,
    TGA_V_OROPT2R = 23, TGA_V_OROPT3R = 24, TGA_V_CROSS22R = 25, TGA_V_CROSS33R = 26,
    TGA_N_VARIANTS = 27
};

/* operator masks (bit i = variant i); OR them for a fused sweep */
#define TGA_OP_2OPT           (1u << TGA_V_2OPT)
#define TGA_OP_2OPT_STAR      (1u << TGA_V_2OPT_STAR)
#define TGA_OP_RELOCATE       (1u << TGA_V_RELOCATE1)
#define TGA_OP_OR_OPT         ((1u << TGA_V_OROPT2) | (1u << TGA_V_OROPT3))
#define TGA_OP_SWAP           (1u << TGA_V_SWAP11)
#define TGA_OP_CROSS          (0x1Fu << TGA_V_CROSS12)
#define TGA_OP_INTRA_RELOCATE (0x7u << TGA_V_IRELOCATE1)
#define TGA_OP_INTRA_SWAP     (0x1FFu << TGA_V_ISWAP11)
#define TGA_OP_INTER          (0x7FEu)
#define TGA_OP_INTRA          (TGA_OP_2OPT | TGA_OP_INTRA_RELOCATE | TGA_OP_INTRA_SWAP)
#define TGA_OP_REVERSED       (0xFu << TGA_V_OROPT2R)
#define TGA_OP_STANDARD       ((1u << TGA_V_OROPT2R) - 1u)
#define TGA_OP_ALL            ((1u << TGA_N_VARIANTS) - 1u)
/* the north-star fused sweep: 2-opt* + relocate + swap */
#define TGA_OP_FUSED_NS       (TGA_OP_2OPT_STAR | TGA_OP_RELOCATE | TGA_OP_SWAP)
/* flag for tga_eval: keep the keys of the previous tga_eval of this generation and
 * MIN-combine into them (evaluate a neighbourhood in several launches) */
#define TGA_EVAL_ACCUMULATE   (1u << 31)

/* score modes (Eq. 16a: F = F(dD, dT_V, dL_V), never given by the paper; reading 4) */
#define TGA_SCORE_FEASIBLE  0   /* score = dD if both new routes are feasible, else +inf */
#define TGA_SCORE_PENALISED 1   /* score = dD + w_load * dL_V + w_tw * dT_V */

typedef struct tga_instance tga_instance;
typedef struct tga_solution tga_solution;

typedef struct {
    int32_t score_mode;  /* TGA_SCORE_*; default TGA_SCORE_FEASIBLE */
    int32_t w_load;      /* integer penalty weight on load excess (default 10) */
    int32_t w_tw;        /* integer penalty weight on time warp (default 10) */
    int32_t device;      /* CUDA device ordinal; -1 = current device */
    int32_t slack;       /* spare physical slots per route (0 = default 2, -1 = none): a move that
                            keeps both changed routes within their slots refreshes only them */
    int32_t granular_theta; /* 0 = full neighbourhood (NTGA).  > 0: edge-based neighbourhood (ETGA,
                            P:390-401) with granularity threshold theta: inter-route
                            candidates only where the edge mask keeps the node pair at (u, v) --
                            v among the theta nearest customers of u or u among those of v, or
                            either is the depot (reading 21); intra-route candidates stay
                            full.  Integer feasible-only fast path only (else
                            TGA_ERR_UNSUPPORTED at tga_eval). */
    int32_t reserved[10];
} tga_options;

typedef struct {
    int32_t variant;             /* TGA_V_* */
    int32_t n1, n2;              /* segment lengths (0 where not applicable) */
    int32_t route_a, pos_a;      /* route / position of slot u (position 0 = start depot) */
    int32_t route_b, pos_b;      /* route / position of slot v; route_a == route_b => intra */
    int32_t u, v;                /* canonical slot ids */
    int32_t feasible;            /* 1 if both changed routes are feasible */
    int64_t delta_i;             /* score in integer mode (TGA_I32); == dD in feasible-only mode */
    double  delta_f;             /* score as a double (both modes) */
    uint64_t key;                /* packed (order-preserving score << 32 | flat index) */
    uint64_t generation;         /* solution generation this move belongs to */
} tga_move;

/* ------------------------------------------------------------ instance
 * tga_instance_create: upload one instance (§2).
 *   n_nodes   number of nodes incl. the depot (>= 2)
 *   dist      n_nodes*n_nodes row-major distances c_ij (= travel times t_ij),
 *             int32 (dist_dtype TGA_I32) or float (TGA_F32); zero diagonal,
 *             non-negative, symmetric
 *   time      must be NULL (T = C); non-NULL => TGA_ERR_UNSUPPORTED
 *   demand    n_nodes int32 delivery demands d_i >= 0, d_0 = 0
 *   tw        NULL for CVRP, else n_nodes*3 floats {e_i, l_i, s_i} in the
 *             distance unit, e_i <= l_i, s_0 = 0
 *   capacity  vehicle capacity Q > 0
 *   opt       NULL = defaults
 *   out       receives the instance
 * Errors: TGA_ERR_INVALID_ARGUMENT, TGA_ERR_UNSUPPORTED, TGA_ERR_CUDA, TGA_ERR_OOM. */
int32_t tga_instance_create(int32_t n_nodes, const void *dist, int32_t dist_dtype,
                            const void *time, const int32_t *demand, const float *tw,
                            int32_t capacity, const tga_options *opt, tga_instance **out);
/* VRPSPDTW pickup demands ("the vehicle must deliver d_i units of goods
 * from the depot v_0 to v_i and pick up p_i units from v_i back to the depot"; load
 * attributes L_I, L_O, L_M of Eq. 3a-d).
 *   pickup: host int32[n_nodes], p_0 == 0, p_i >= 0; copied (caller keeps ownership).
 * With pickups the capacity constraint (and the load excess of the penalised score) is
 * on the largest load a route carries; evaluation takes the generic kernels (the fast
 * paths assume delivery sums) and 2-opt is unsupported (the paper applies it to the CVRP
 * only).  Must be called before any solution of the instance is loaded.
 * Errors: TGA_ERR_INVALID_ARGUMENT (NULL, p_0 != 0, p_i < 0, sum >= 2^30, solutions
 * already loaded), TGA_ERR_CUDA. */
int32_t tga_instance_set_pickup(tga_instance *inst, const int32_t *pickup);
int32_t tga_instance_destroy(tga_instance *inst);
/* n_nodes, granular_theta and the number of unordered customer pairs the edge
 * mask keeps (0 without a granular neighbourhood).  Any pointer may be NULL. */
int32_t tga_instance_info(const tga_instance *inst, int32_t *n_nodes, int32_t *theta, int64_t *n_edge_pairs);

/* ------------------------------------------------------------ solution
 * tga_solution_load: "a solution tensor T_s is first initialized on the GPU
 * using the attribute matrices derived from S".  Builds the slot
 * layout, the position-ordered distance matrix and the forward/backward
 * attribute records (attribute-rebuild scan).
 *   n_routes   number of routes R >= 1 (empty routes allowed; never renumbered)
 *   route_ptr  R+1 int32 CSR offsets into customers
 *   customers  route_ptr[R] int32 customer ids; every customer exactly once
 * Errors: TGA_ERR_STRUCTURE, TGA_ERR_INVALID_ARGUMENT, TGA_ERR_CUDA, TGA_ERR_OOM. */
int32_t tga_solution_load(tga_instance *inst, int32_t n_routes, const int32_t *route_ptr,
                          const int32_t *customers, tga_solution **out);
int32_t tga_solution_destroy(tga_solution *sol);

/* tga_eval: enqueue the evaluation of every variant in op_mask on
 * cuda_stream (a cudaStream_t; NULL = the solution's own stream) and return
 * without synchronising (Extraction/Concatenation/Differencing/Evaluation,
 * P:241 steps 1-4, fused into one kernel per candidate space).  With a
 * communicator (tga_comm_init) only this rank's shard of the candidate rows
 * is evaluated and the packed keys are MIN-allreduced over NCCL on the same
 * stream.  Errors: TGA_ERR_UNSUPPORTED (2-opt with time windows), TGA_ERR_CUDA. */
int32_t tga_eval(tga_solution *sol, uint32_t op_mask, void *cuda_stream);

/* tga_best_move: synchronise the stream, read the per-variant keys (8 B each)
 * and decode the best over op_mask ("transferred to the CPU").
 * Returns TGA_OK if the best score is < 0, TGA_NO_IMPROVING_MOVE otherwise
 * (out is still filled when any candidate was valid; out->key = ~0 if none). */
int32_t tga_best_move(tga_solution *sol, uint32_t op_mask, tga_move *out);

/* tga_apply_move: apply a move returned by tga_best_move for this generation
 * ("update the solution S, and synchronize the updated solution tensor",
 * P:241 step 5; §5.3.5): splice the 1-2 route lists, re-upload only the
 * changed slot span, refresh its rows/columns of the distance tile matrix and
 * re-scan the affected routes.  Errors: TGA_ERR_STALE, TGA_ERR_INVALID_ARGUMENT. */
int32_t tga_apply_move(tga_solution *sol, const tga_move *move);

/* Make the solution use cuda_stream (a cudaStream_t; NULL = its own stream)
 * for every later call (eval, best_move, apply, queries).  The stream must
 * belong to the solution's device and outlive the solution or the next call. */
int32_t tga_solution_set_stream(tga_solution *sol, void *cuda_stream);

/* tga_step: one best-improvement iteration of the feasible-and-infeasible
 * search (Alg. A2 lines 5-8): tga_eval(op_mask) + tga_best_move +
 * tga_apply_move when the best score is < 0.  out (may be NULL) receives the
 * move.  Returns TGA_OK if a move was applied, TGA_NO_IMPROVING_MOVE if not. */
int32_t tga_step(tga_solution *sol, uint32_t op_mask, tga_move *out);

/* tga_step_async: the same iteration entirely on the device, without a host
 * round trip: the evaluation kernels, then one kernel
 * that picks the best key, and -- if improving -- splices the changed routes
 * in the slot arrays, then the update kernel (bounds read on the device).
 * Enqueue-only; steps can be issued back to back (or captured in a CUDA
 * graph).  Host-side queries resynchronise the host route lists lazily.
 * A CUDA graph captured from these calls records decisions taken from the
 * solution's state at capture time (no key reset after a step, no rebuild of the
 * ETGA node -> slot map): replay it only while nothing but replays of that
 * graph modifies the solution.
 * The step consumes the keys (resets them to ~0 on the device), so the next
 * tga_eval enqueues no reset of its own; tga_solution_keys after a step
 * returns ~0 for every variant until the next tga_eval.
 * tga_solution_device_stats returns and clears the candidate counts per
 * variant accumulated by device steps (counts[TGA_N_VARIANTS]) and the number
 * of moves they applied (synchronises). */
int32_t tga_step_async(tga_solution *sol, uint32_t op_mask);
/* tga_descent: n_steps device-resident steps enqueued from C (a best-improvement
 * descent, Alg. A2).  Optional instrumentation: when step_ms is not
 * NULL, CUDA events bracket every step on the solution's stream and the
 * per-step device times are written there (synchronises); when l2_flush is not
 * NULL, flush_bytes of it are overwritten before every step, outside the
 * bracketed interval (cold-L2 timing). */
int32_t tga_descent(tga_solution *sol, uint32_t op_mask, int32_t n_steps, void *l2_flush, uint64_t flush_bytes,
                    float *step_ms);
int32_t tga_solution_device_stats(tga_solution *sol, uint64_t *counts, uint64_t *applied);

/* tga_solution_reload: load another solution of the same instance into an
 * existing solution object (same route count and customer count => same
 * device layout; no allocation): host arrays are copied, the slot layout is
 * re-uploaded, the distance tile matrix rebuilt and every route re-scanned,
 * asynchronously on the solution's stream.  Errors: TGA_ERR_STRUCTURE,
 * TGA_ERR_INVALID_ARGUMENT (different R), TGA_ERR_CUDA. */
int32_t tga_solution_reload(tga_solution *sol, int32_t n_routes, const int32_t *route_ptr,
                            const int32_t *customers);

/* Live kernel timing: when enabled, tga_eval records CUDA events around the
 * inter-route kernel launch on its stream; tga_solution_timings returns (and
 * clears) up to max_n recorded durations in milliseconds (synchronises).
 * Returns the number written in *n_out. */
int32_t tga_solution_enable_timing(tga_solution *sol, int32_t enable);
int32_t tga_solution_timings(tga_solution *sol, float *ms, int32_t max_n, int32_t *n_out);

/* Per-variant raw keys of the last tga_eval (synchronises). keys[TGA_N_VARIANTS];
 * ~0 = no valid candidate. */
int32_t tga_solution_keys(tga_solution *sol, uint64_t *keys);

/* Exact candidate counts per variant for the current solution (closed forms of
 * the full neighbourhood; host only). counts[TGA_N_VARIANTS].  With
 * granular_theta > 0 the inter-route candidates actually evaluated are counted
 * on the device instead (tga_solution_device_stats). */
int32_t tga_solution_counts(const tga_solution *sol, uint64_t *counts);

/* Totals from the device attribute records: distance D(S) (Eq. 1, mu1=0,
 * mu2=1), sum of load excess max(L-Q,0), sum of time warp. */
int32_t tga_solution_cost(tga_solution *sol, int64_t *dist_i, double *dist_f,
                          int64_t *load_excess, double *tw_excess);

/* Export the routes (CSR). route_ptr[R+1], customers[N]. */
int32_t tga_solution_routes(const tga_solution *sol, int32_t *route_ptr, int32_t *customers);
/* R, N, canonical slot count Q = N + R, generation */
int32_t tga_solution_info(const tga_solution *sol, int32_t *n_routes, int32_t *n_customers,
                          int32_t *n_slots, uint64_t *generation);

/* Attribute records per canonical slot (Q entries each), for parity with a
 * from-scratch rebuild: prefix [0..p] and suffix [p..L+1] loads and
 * distances; prefix/suffix time warp T_V; service start time at p derived
 * from the prefix record (start = T_E + T_D - T_V - s).  Any pointer may be NULL. */
int32_t tga_solution_attributes(tga_solution *sol, int64_t *pre_L, int64_t *suf_L,
                                double *pre_D, double *suf_D, double *pre_TV,
                                double *suf_TV, double *start);
/* VRPSPDTW load records for parity (Eq. 3a-d), per CANONICAL slot c (Q = N + R):
 * pre[3c .. 3c+2] = (L_I, L_O, L_M) of the prefix [0..p] of its route, suf[...] = those of
 * the suffix [p..L+1].  Caller-owned int32[3 Q] each.  TGA_ERR_UNSUPPORTED without pickups. */
int32_t tga_solution_load_records(tga_solution *sol, int32_t *pre, int32_t *suf);

/* ------------------------------------------------------------ multi-GPU
 * Row sharding: a solution with a shard plan (n_shards > 1) evaluates only
 * shard `shard` of the inter-route tile rows and intra-route slot rows.
 * tga_comm_init attaches an NCCL communicator (nccl_unique_id = 128-byte
 * ncclUniqueId shared by all ranks) and makes tga_eval MIN-allreduce the
 * packed keys (exact: keys are (score, canonical index)). */
int32_t tga_solution_set_shard(tga_solution *sol, int32_t shard, int32_t n_shards);
/* The row-shard plan (host only): items [lo, hi) of n_items for shard `shard` of
 * `n_shards` (contiguous, balanced to +-1, disjoint, covering). */
int32_t tga_shard_range(int64_t n_items, int32_t shard, int32_t n_shards, int64_t *lo, int64_t *hi);
int32_t tga_nccl_unique_id(void *out_128_bytes);
int32_t tga_comm_init(tga_solution *sol, int32_t rank, int32_t world, const void *nccl_unique_id);

/* ------------------------------------------------------------ population batch
 * A batch of solutions of one instance evaluated by single launches over
 * (solution, tile) work items (BASELINE config 5; "Population-based
 * metaheuristics can leverage parallel evaluation").
 * tga_batch_load: n_sol solutions; n_routes[k] routes each; route_ptr holds the
 * n_sol CSR offset arrays back to back (n_routes[k]+1 entries each, each
 * starting at 0); customers holds n_sol blocks of n_nodes-1 ids.
 * tga_batch_best_moves: out[n_sol] moves, status[n_sol] (TGA_OK = improving,
 * TGA_NO_IMPROVING_MOVE) -- may be NULL.  tga_batch_apply_moves applies
 * moves[k] where apply[k] != 0 (apply may be NULL = all with a valid variant).
 * tga_batch_solution returns a borrowed handle (owned by the batch). */
typedef struct tga_batch tga_batch;
int32_t tga_batch_load(tga_instance *inst, int32_t n_sol, const int32_t *n_routes,
                       const int32_t *route_ptr, const int32_t *customers, tga_batch **out);
int32_t tga_batch_destroy(tga_batch *batch);
int32_t tga_batch_size(const tga_batch *batch, int32_t *n_sol);
int32_t tga_batch_solution(tga_batch *batch, int32_t i, tga_solution **out);
int32_t tga_batch_eval(tga_batch *batch, uint32_t op_mask, void *cuda_stream);
int32_t tga_batch_keys(tga_batch *batch, uint64_t *keys);
int32_t tga_batch_best_moves(tga_batch *batch, uint32_t op_mask, tga_move *out, int32_t *status);
int32_t tga_batch_apply_moves(tga_batch *batch, const tga_move *moves, const int32_t *apply);
/* use cuda_stream for every later batch call (NULL = the batch's own stream) */
int32_t tga_batch_set_stream(tga_batch *batch, void *cuda_stream);
/* device-resident steps of every solution of the batch (see tga_step_async) */
int32_t tga_batch_step_async(tga_batch *batch, uint32_t op_mask);
int32_t tga_batch_device_stats(tga_batch *batch, uint64_t *counts, uint64_t *applied);

/* Diagnostics: phase probe of the device-resident step.  enable != 0 makes the
 * next pick/update launches record the SM cycle counter (clock64 of block 0)
 * at 8 phase points; out[16 + 1024] (may be NULL) receives the last record
 * and, from out[16], the globaltimer (ns) at the start / end of each block b < 512
 * of the last single-solution pick/update launch at out[16 + 2b], out[17 + 2b]
 * (synchronises).  Not used on any timed path. */
int32_t tga_solution_debug_probe(tga_solution *sol, int32_t enable, uint64_t *out);

/* Test-only: tga_debug_eval_dump evaluates op_mask once with the DUMP
 * instantiations of the SAME kernels and launch decisions as tga_eval (tile
 * body / cell formulas, intra kernels; no shards, no edge mask) which also
 * store the packed key of every candidate they evaluate.  out[TGA_N_VARIANTS
 * * Q * Q] (Q = canonical slots) receives, at [variant][u * Q + v] (canonical
 * u, v): 0 = the candidate was not evaluated, ~0 = evaluated and infeasible
 * (feasible-only mode) or structurally invalid, else its key with the
 * canonical flat index.  flags: 1 = force the warp-scan VRPTW intra kernel,
 * 2 = force the per-thread walk.  The keys of the call are left as by
 * tga_eval.  For parity tests of the per-candidate score and feasibility
 * mask (Eq. 16a-b); never on a timed path. */
int32_t tga_debug_eval_dump(tga_solution *sol, uint32_t op_mask, int32_t flags, uint64_t *out, int64_t out_len);

/* ------------------------------------------------------------ misc */
const char *tga_last_error(void);
const char *tga_version(void);
/* number of CUDA kernels this library launched so far (for the bench's gpu_launches) */
uint64_t tga_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TGA_H */
