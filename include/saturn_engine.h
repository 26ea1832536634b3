/*
 * saturn_engine.h -- C ABI of the B200 plan-search engine (libsaturn_b200.so).
 *
 * The engine replaces the Solver's plan search of the reference
 * (arXiv 2311.02840 "Saturn"; reference package /root/reference/pkg/src/jointsched):
 *
 *   sat_search_tree / sat_search_index
 *       replace branch_and_bound + solve_lp_relaxation (milp/__init__.py:6,
 *       SPEC.md:201-214) and brute_force_schedule (milp/__init__.py:3,
 *       SPEC.md:219-227): exhaustive search of (option per job) x (submission
 *       order), each candidate list-scheduled to its makespan (the SPEC.md:213
 *       "list-schedule earliest-fit"), best = lowest (makespan, index).
 *   sat_search_sampled
 *       replaces plan_random's draws (rng.py:20-56): candidate
 *       i is decoded from SplitMix64 substream(seed, i) or SplitMix64(seed + i).
 *   sat_schedule
 *       replaces decode_plan (milp/__init__.py:4) and the
 *       evaluation of fixed plans (plan_optimus / plan_current_practice,
 *       SPEC.md:285-320): per-job option, node and start of given candidates.
 *
 * Conventions
 *   - Problem tables (sat_problem_t) are HOST pointers, read during the call
 *     and packed into the launch; nothing is retained after return.
 *   - Outputs and workspaces are DEVICE pointers owned by the caller.
 *   - Every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and reentrant: no globals, one call per stream.
 *   - Returns SAT_OK or an error code; sat_error_string() explains it.
 *   - Results accumulate: *d_best is min-combined with what it already holds,
 *     so shards of one search can be issued back to back; sat_best_reset()
 *     initialises it.  Grid mode: d_best->hi = (makespan << idx_bits) | index.
 *     Float mode: d_best->hi = bit pattern of the fp64 makespan (positive
 *     doubles order like unsigned integers), d_best->lo = index.
 */
#ifndef SATURN_ENGINE_H
#define SATURN_ENGINE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAT_ABI_VERSION 8

/* status codes (mapped to reference errors.py classes by the host layer) */
#define SAT_OK              0
#define SAT_ERR_INVALID     1  /* bad shapes / arguments        -> InvariantViolation (errors.py:8) */
#define SAT_ERR_NO_OPTIONS  2  /* a job with zero options       -> NoFeasibleConfig   (errors.py:23) */
#define SAT_ERR_TOO_LARGE   3  /* index / key / table overflow  -> TooLarge           (errors.py:84) */
#define SAT_ERR_UNSUPPORTED 4  /* shape outside this kernel     -> TooLarge                       */
#define SAT_ERR_CUDA        5  /* CUDA launch / runtime failure -> PlanFailure / ReplanFailure     */

/* time modes */
#define SAT_TIME_GRID_I32 0    /* int32 interval durations d = ceil(T / delta) */
#define SAT_TIME_F64      1    /* float64 seconds, adds and max only: bit-exact vs CPU      */

/* candidate sources */
#define SAT_SRC_INDEX     0    /* index = c * J! + p             */
#define SAT_SRC_SUBSTREAM 1    /* candidate i <- SplitMix64 substream(seed, i) (rng.py:51) */
#define SAT_SRC_SEED      2    /* candidate i <- SplitMix64(seed + i): plan_random(seed+i) */
#define SAT_SRC_EXPLICIT  3    /* candidate i <- caller arrays options[i][J], order[i][J]  */
#define SAT_SRC_GREEDY    4    /* sat_local_search (ABI v6): walker i starts at the greedy  */
                               /* candidate -- every job at its least-area option, jobs in */
                               /* descending order of duration x (2^17 + u), u = the top 16 */
                               /* bits of draw j of substream(seed, i)                     */

#define SAT_MAX_JOBS   64
#define SAT_MAX_LANES  32      /* N nodes x G padded GPUs per node must fit one warp */

typedef struct sat_problem {
    int32_t J;              /* jobs (job axis = jobs sorted by id)                         */
    int32_t N;              /* nodes                                                       */
    int32_t G;              /* padded GPU slots per node: power of two >= max gpu_count   */
    int32_t Cmax;           /* row stride of the option tables                             */
    int32_t time_mode;      /* SAT_TIME_*                                                   */
    int32_t idx_bits;       /* grid mode: bits of the key holding the candidate index      */
    const int32_t  *radix;        /* [J]            options per job (>= 1)                 */
    const int32_t  *gpus;         /* [J*Cmax]       gang size g of option (j, o)           */
    const uint32_t *node_mask;    /* [J*Cmax]       bit n: option runnable on node n       */
    const int32_t  *dur_i32;      /* [J*Cmax*N]     grid durations (grid mode)             */
    const double   *dur_f64;      /* [J*Cmax*N]     seconds (float mode)                   */
    const int32_t  *node_gpus;    /* [N]            GPUs per node (<= G)                   */
    const int32_t  *release_i32;  /* [J] or NULL    earliest start per job                 */
    const double   *release_f64;  /* [J] or NULL                                           */
    const int32_t  *init_free_i32;/* [N*G] or NULL  ascending per-node GPU free times      */
    const double   *init_free_f64;/* [N*G] or NULL                                         */
} sat_problem_t;

typedef struct sat_best {
    uint64_t hi;
    uint64_t lo;
} sat_best_t;

typedef struct sat_tree_info {
    int32_t  prefix_len;    /* P: jobs fixed per lane; the other J-P are enumerated per warp */
    int32_t  n_sets;        /* C(J, P) prefix job sets                                       */
    uint64_t n_tasks;       /* warp tasks (32 prefixes of one set each)                      */
    uint64_t n_candidates;  /* = prod(radix) * J!                                            */
    uint64_t n_job_steps;   /* list-scheduling placements the prefix-shared walk performs    */
    int32_t  pair_packed;   /* 1: the last-two-jobs pass runs on 16-bit pairs (ABI v3)       */
    int32_t  reserved;
} sat_tree_info_t;

int         sat_abi_version(void);
const char *sat_error_string(int status);

/* device facts (sm count, compute capability) for launch sizing and reporting */
int sat_device_info(int device, int32_t *sm_count, int32_t *cc_major, int32_t *cc_minor);

/* *d_best <- "empty" (all ones) */
int sat_best_reset(sat_best_t *d_best, void *stream);

/* Workspace bytes needed by sat_search_index / sat_search_sampled / sat_schedule. */
int sat_workspace_bytes(const sat_problem_t *p, size_t *bytes);

/* Exhaustive search, per-candidate decode, candidates [lo, hi) of the index space. */
int sat_search_index(const sat_problem_t *p, uint64_t lo, uint64_t hi,
                     sat_best_t *d_best, void *d_ws, size_t ws_bytes, void *stream);

/* Sampled search: candidates [lo, hi) of source SAT_SRC_SUBSTREAM / SAT_SRC_SEED. */
int sat_search_sampled(const sat_problem_t *p, int32_t source, uint64_t seed,
                       uint64_t lo, uint64_t hi,
                       sat_best_t *d_best, void *d_ws, size_t ws_bytes, void *stream);

/* Prefix-shared exhaustive search (single node, grid mode, no release times).
 * sat_tree_plan fills *info for a prefix length (0 = engine's choice);
 * sat_search_tree walks warp tasks [task_lo, task_hi) of that layout; warps take
 * tasks from a cursor kept in the workspace (>= SAT_TREE_WS_BYTES, device memory;
 * the same workspace as the other searches is fine). */
#define SAT_TREE_WS_BYTES 256
int sat_tree_plan(const sat_problem_t *p, int32_t prefix_len, sat_tree_info_t *info);
int sat_search_tree(const sat_problem_t *p, int32_t prefix_len,
                    uint64_t task_lo, uint64_t task_hi,
                    sat_best_t *d_best, void *d_ws, size_t ws_bytes, void *stream);

/* Rank `rank` of `world`'s share of the layout's warp tasks: a contiguous range whose
 * full-scan work (placements) is 1/world of the total, so ranks finish together (task costs
 * differ by set; an even split of the task count leaves up to ~25 % imbalance at 8 ranks). */
int sat_tree_shard(const sat_problem_t *p, int32_t prefix_len, int32_t world, int32_t rank,
                   uint64_t *task_lo, uint64_t *task_hi);

/* Bound-and-prune over the same layout (replaces branch_and_bound):
 * subtrees whose makespan lower bound exceeds the best makespan found so far are
 * skipped; every candidate that could tie or beat the best is still scheduled, so the
 * key equals sat_search_tree's.  *d_best may be seeded with an upper bound key
 * (makespan << idx_bits | (2^idx_bits - 1)) from any known candidate.  Counters are
 * left in the workspace as uint64 words after the task cursor (index 1 + SAT_BNB_STAT_*). */
#define SAT_BNB_STAT_PRUNED_TASKS 0   /* warp tasks cut at the prefix          */
#define SAT_BNB_STAT_PAIR_NODES   1   /* two-job subtrees scheduled (per warp)  */
int sat_search_bnb(const sat_problem_t *p, int32_t prefix_len,
                   uint64_t task_lo, uint64_t task_hi,
                   sat_best_t *d_best, void *d_ws, size_t ws_bytes, void *stream);

/* Local search from sampled starting points (grid time): walker w starts at candidate w of
 * `source` (SAT_SRC_SUBSTREAM / SAT_SRC_SEED) and descends over swap / option / insertion
 * moves on (makespan, total GPU load) until no move improves or max_rounds rounds of 32
 * moves were scanned.  Result (ABI v5): the lowest
 * (makespan, rounds scanned, walker) as (makespan << (idx_bits + SAT_LS_ROUND_BITS)) |
 * (rounds << idx_bits) | walker -- among walkers ending at the same makespan, the one that got
 * there in the fewest rounds, then the lowest id (max_rounds < 2^SAT_LS_ROUND_BITS).
 * d_state_out (device, (hi - lo) x 2J bytes, or null) receives the final candidate of every
 * walker w (options then order, at (w - lo) * 2J) -- the winner's plan without a replay;
 * entries of abandoned walkers (below) are left untouched.  The number of rounds
 * scanned (each = up to 32 candidates scheduled) is left in the workspace as the uint64 word
 * after the walker cursor, which follows the problem blob at offset
 * sat_ls_counter_offset(p).  stop_ms >= 0 (the problem's lower bound): a walker ends as
 * soon as its makespan is <= stop_ms (its final state is the candidate at that point), and a
 * still-running walker that has scanned at least as many rounds as a key already in *d_best
 * with makespan <= stop_ms is abandoned; neither changes the result.  stop_ms < 0: walks run
 * to their local optimum. */
#define SAT_LS_ROUND_BITS 13
int sat_ls_counter_offset(const sat_problem_t *p, size_t *offset);
int sat_local_search(const sat_problem_t *p, int32_t source, uint64_t seed, uint64_t lo, uint64_t hi,
                     int32_t max_rounds, int32_t stop_ms, sat_best_t *d_best, uint8_t *d_state_out,
                     void *d_ws, size_t ws_bytes, void *stream);

/* Schedule n candidates and record the plan of each.
 *   source SAT_SRC_INDEX/SUBSTREAM/SEED: d_ids[n] candidate ids (seed used by streams)
 *   source SAT_SRC_EXPLICIT: d_explicit[n][2*J] = option digit per job, then order
 * Outputs (device, [n*J] each, any may be NULL): option, node, start (i32 or f64);
 * d_makespan_i64 / d_makespan_f64 [n]. */
int sat_schedule(const sat_problem_t *p, int32_t source, uint64_t seed,
                 const uint64_t *d_ids, const uint8_t *d_explicit, int32_t n,
                 int32_t *d_option, int32_t *d_node,
                 int32_t *d_start_i32, double *d_start_f64,
                 int64_t *d_makespan_i64, double *d_makespan_f64,
                 void *d_ws, size_t ws_bytes, void *stream);

/* Bytes of the launch-parameter block the tree / bnb searches pass by value (their
 * host-to-device traffic per launch, besides the 24-byte cursor reset). */
size_t sat_tree_param_bytes(void);

/* State-space search (one node, grid time; ABI v4): is there a candidate -- options + order,
 * list-scheduled exactly as by the other searches -- with makespan <= target?  Level k holds
 * the distinct states (jobs still to place, sorted GPU free times) after k placements; children
 * whose makespan lower bound exceeds `target` are cut; distinct states are kept in an exact
 * hash set in d_ws.  INFEASIBLE proves that no candidate of the whole space reaches `target`
 * (with a candidate at target + 1 in hand, that candidate is optimal -- the proof SPEC.md:210-214's
 * branch-and-bound returns as status Optimal).  FEASIBLE: h_candidate (host, 2J bytes: option
 * digit per job, then the order) receives one candidate with makespan <= target, chosen
 * deterministically (smallest final state key, then smallest parent keys, lowest options).
 * BUDGET: more than max_states states over all levels; nothing decided.  Synchronous: returns
 * after the search (one small read-back per level).  One node with 2^J x C(target + G, G) < 2^63:
 * exact states, 63-bit keys, candidate rebuilt.  Otherwise (several nodes, up to 8 and 32 GPUs
 * in all, or wider keys: 2^J x prod_n C(target + G_n, G_n) < 2^126) a PROVER on 128-bit keys:
 * interchangeable nodes are canonicalised and ties between nodes expanded both ways, so an
 * INFEASIBLE answer is still a proof, but FEASIBLE carries no candidate (info->makespan = -1);
 * shapes beyond that: SAT_ERR_UNSUPPORTED. */
#define SAT_DP_INFEASIBLE 0
#define SAT_DP_FEASIBLE   1
#define SAT_DP_BUDGET     2
typedef struct sat_dp_info {
    int32_t  status;        /* SAT_DP_*                                                     */
    int32_t  levels;        /* levels expanded                                              */
    uint64_t states;        /* distinct states over all levels                              */
    uint64_t widest_level;  /* states of the largest level                                   */
    int32_t  makespan;      /* FEASIBLE: makespan of the returned candidate                  */
    int32_t  reserved;
} sat_dp_info_t;
int sat_dp_workspace_bytes(const sat_problem_t *p, int32_t target, uint64_t max_states, size_t *bytes);
int sat_search_dp(const sat_problem_t *p, int32_t target, uint64_t max_states, uint8_t *h_candidate,
                  sat_dp_info_t *info, void *d_ws, size_t ws_bytes, void *stream);
/* ABI v8: the same with flags.  SAT_DP_EXACT on several nodes: labelled states (no canonical
 * node order) expanded by the list scheduler's own node choice (earliest end over every eligible
 * node, lowest label on ties; a child is cut when that node cannot reach the target), so the
 * levels hold exactly the candidates' states: INFEASIBLE is a proof as before, and FEASIBLE now
 * returns a candidate (rebuilt backwards like the one-node search: smallest labelled key, lowest
 * options).  More states than the prover where nodes are interchangeable.  One node: flags
 * change nothing (the one-node search is exact already). */
#define SAT_DP_EXACT 1
int sat_dp_workspace_bytes_ex(const sat_problem_t *p, int32_t target, uint64_t max_states, int32_t flags,
                              size_t *bytes);
int sat_search_dp_ex(const sat_problem_t *p, int32_t target, uint64_t max_states, int32_t flags,
                     uint8_t *h_candidate, sat_dp_info_t *info, void *d_ws, size_t ws_bytes, void *stream);

/* Cross-rank shared incumbent (ABI v4).  With several ranks (one process per GPU), every rank's
 * search kernels can atomicMin into -- and prune against -- ONE sat_best_t cell in the owner
 * rank's HBM, reached over NVLink peer memory: the MIN combine of SURVEY.md 8(e) happens inside
 * the searches tile by tile, so bound-and-prune and the local search's abandonment see the best
 * key of ALL ranks while they run.  The owner allocates the cell (two sat_best_t, all ones) and
 * exports a CUDA IPC handle (SAT_IPC_HANDLE_BYTES); the others open it (peer access enabled
 * lazily).  sat_peer_atomics reports whether two devices support native peer atomics (NVLink;
 * same device: yes).  sat_best_set writes a key (seeding), sat_best_copy reads one cell into
 * another (e.g. into a rank-local buffer after the searches). */
#define SAT_IPC_HANDLE_BYTES 64
int sat_best_set(sat_best_t *d_best, uint64_t hi, uint64_t lo, void *stream);
int sat_best_copy(sat_best_t *d_dst, const sat_best_t *d_src, void *stream);
int sat_shared_best_alloc(sat_best_t **d_cell, uint8_t *handle_out);
int sat_shared_best_open(const uint8_t *handle, sat_best_t **d_cell);
int sat_shared_best_close(sat_best_t *d_cell, int32_t owner);
int sat_peer_atomics(int32_t dev_a, int32_t dev_b, int32_t *supported);

/* Search key hand-off (ABI v7), one launch on `stream`: d_out[0..n_words) = the words of
 * *d_best with "empty" (all ones) mapped to INT64_MAX (the MIN identity of the cross-rank
 * all-reduce), d_out[n_words + e] = d_extra[e] for e < n_extra (e.g. bound-and-prune's counters,
 * so key and counters come back in one read); if d_ids != NULL, d_ids[0] = the candidate id
 * the winner replay decodes: the low idx_bits of the grid key, or 0 when the key is empty or
 * (check_range) >= n_idx.  d_best == NULL: only d_ids, from d_out[0] (after the all-reduce). */
int sat_key_finish(const sat_best_t *d_best, int32_t n_words, const uint64_t *d_extra, int32_t n_extra,
                   int64_t *d_out, uint64_t *d_ids, int32_t idx_bits, uint64_t n_idx, int32_t check_range,
                   void *stream);

/* INT32 min/max issue-rate probe for the roofline denominator: runs `iters`
 * dependent-chain IMNMX iterations on every SM; *d_ops_out = lane-ops done. */
int sat_alu_probe(int32_t blocks, int32_t threads, int32_t iters,
                  uint64_t *d_ops_out, int32_t *d_sink, void *stream);

/* The same probe on two 16-bit lanes per register (min/max .u16x2, VIMNMX.U16x2): the
 * denominator for k_tree launches whose pair pass is packed; counts 2 ops per lane-op. */
int sat_alu_probe16(int32_t blocks, int32_t threads, int32_t iters,
                    uint64_t *d_ops_out, int32_t *d_sink, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SATURN_ENGINE_H */
