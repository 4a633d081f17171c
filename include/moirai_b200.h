/*
 * moirai_b200.h — C ABI of the B200-native Moirai hot path (libmoirai_b200.so).
 *
 * Two data-parallel paths of the reference package `opplace` are replaced:
 *   1. batched makespan evaluation of candidate placements
 *      (reference: pkg/src/opplace/solver.py:80-148 `_schedule`, driven by
 *       `schedule_for_assignment` solver.py:151-165 and the `brute_force`
 *       keep-best loop solver.py:257-282), and
 *   2. GCOF fusion-rule coarsening (reference: pkg/src/opplace/fusion.py:271-304).
 *
 * Conventions
 *  - Every entry point returns int32 status: MP_OK (0) or a negative MP_ERR_*;
 *    an optional mp_error* receives the code plus two integer details and a
 *    message.  The Python host (paper_2312_04025_b200/_native.py) maps codes onto
 *    the reference exception tree (pkg/src/opplace/errors.py).
 *  - No C++ or torch types cross the boundary: plain pointers, sizes, and an
 *    opaque cudaStream_t passed as void* (NULL = the library's own stream, which is
 *    ordered with the legacy default stream like any blocking stream: work a caller
 *    enqueued on stream 0 before the call completes before the call's kernels read it).
 *  - Buffers are caller-owned.  Unless MP_DEVICE_PTRS is set in `flags`, array
 *    arguments are HOST pointers and the library stages them through its own
 *    pinned/device buffers (host<->device copies happen inside the call).
 *  - Op indices are 0..n_ops-1 = ascending reference op id
 *    (`AugGraph.op_ids`, graph.py:179).  Flow indices 0..n_flows-1 follow the
 *    graph's edge-list order (flow id = max op id + 1 + flow index,
 *    graph.py:185-196); node index of flow f is n_ops + f.
 *  - Device indices 0..n_dev-1 = ascending reference device id.
 *    A placement row is uint8[n_ops]: row[i] = device index of op i.
 *  - An mp_instance is immutable after creation; concurrent read-only use from
 *    several host threads on different streams is allowed.
 */
#ifndef MOIRAI_B200_H
#define MOIRAI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MP_ABI_VERSION 1

/* ---- status codes -------------------------------------------------------- */
#define MP_OK                    0
#define MP_ERR_INVALID          -1  /* bad argument (ValueError / KeyError side)            */
#define MP_ERR_EMPTY_GRAPH      -2  /* ValueError("cannot place an empty graph") solver.py:47 */
#define MP_ERR_CYCLE            -3  /* CycleError  graph.py:321 (witness built by the host)  */
#define MP_ERR_MISSING_COST     -4  /* MissingCostError(op, device) solver.py:52-55; a=op, b=dev */
#define MP_ERR_TOO_LARGE        -5  /* TooLargeError(ops, devices) solver.py:266-267          */
#define MP_ERR_UNSUPPORTED      -6  /* outside the GPU path's limits (a, b say which)         */
#define MP_ERR_CUDA             -7  /* CUDA runtime failure; a = cudaError_t                  */
#define MP_ERR_MEMORY_EXCEEDED  -8  /* MemoryExceededError(device, overflow) solver.py:85-87  */
#define MP_ERR_BAD_DEVICE       -9  /* KeyError: placement names an unknown device solver.py:163 */
#define MP_ERR_NO_GPU          -10  /* no CUDA device visible                                 */
#define MP_ERR_INFEASIBLE_MEMORY -11 /* InfeasibleMemoryError(needed=a, available=b) baselines.py:75-77 */

/* per-row status written by the batched calls */
#define MP_ROW_OK          0
#define MP_ROW_MEMORY      1  /* first device (ascending) over capacity; see mem_dev/overflow */
#define MP_ROW_BAD_DEVICE  2  /* row holds a device index >= n_dev */

/* flags */
#define MP_DEVICE_PTRS     1u  /* array arguments are device pointers (stream-ordered)      */

typedef struct mp_error {
    int32_t code;
    int64_t a;
    int64_t b;
    char msg[200];
} mp_error;

/* Flattened placement problem = the reference `_Instance` tables (solver.py:42-77). */
typedef struct mp_problem {
    int32_t n_ops;              /* alpha                                           */
    int32_t n_flows;            /* beta                                            */
    int32_t n_dev;              /* K (1..16 on the GPU path)                       */
    const double  *cost;        /* [n_ops*n_dev] p[i][k]; NaN = no entry (MissingCostError) */
    const int64_t *mem;         /* [n_ops] mem_bytes                                */
    const int32_t *flow_src;    /* [n_flows] op index of the edge source            */
    const int32_t *flow_dst;    /* [n_flows] op index of the edge destination       */
    const int64_t *payload;     /* [n_flows] payload_bytes                          */
    const int64_t *cap;         /* [n_dev] device mem_bytes                          */
    const double  *bw;          /* [n_dev*n_dev] effective bandwidth, row = source  */
} mp_problem;

typedef struct mp_instance mp_instance;

typedef struct mp_instance_info {
    int32_t n_ops, n_flows, n_dev;
    int32_t n_levels;           /* op-graph height levels used by the rank pass      */
    int32_t n_sources;
    int32_t ready_cap;          /* on-chip ready-set capacity per placement          */
    int32_t group_lanes;        /* lanes cooperating on one placement (G)            */
    int32_t lanes_used;         /* lanes per warp owning a placement (U)             */
    int32_t groups_per_cta;
    int32_t ctas;               /* persistent grid size                              */
    int32_t smem_bytes;         /* dynamic shared memory per CTA                     */
    int32_t onchip;             /* 1: tables + state in shared memory, 0: global     */
    int32_t device;
    int32_t n_multi;            /* ops with >= 2 in-flows (est/npred state kept)     */
    int32_t ready_bound;        /* path-cover bound on any ready set                 */
    int32_t colo;               /* 1: co-located flows are not dispatched (exact: all durations > 0) */
    int32_t colo_ok;            /* 1: the instance qualifies for colo                */
    int32_t peak_probe;         /* largest ready set on the creation-time calibration probe */
    int32_t prefilter;          /* 1: a memory-feasibility pass compacts rows before scheduling */
    int32_t mode;               /* 2: tables+state in smem, 1: state in smem, 0: all global */
    int32_t fastdiv;            /* 1: payload/bw by verified reciprocal + Markstein step */
    int64_t table_bytes;        /* instance tables staged per CTA                    */
    int64_t state_bytes;        /* per-placement dynamic state                       */
    int32_t tpp_ready_cap;      /* >0: thread-per-placement kernel in use, register ready capacity */
    int32_t tpp_threads;        /* placements per CTA of the thread-per-placement kernel */
    int32_t tpp_kind;           /* 1: ready set in registers, 2: in shared memory            */
    int32_t ls_ready_cap;       /* local search: proposals whose ready set exceeds it are rejected */
    int32_t dur_classes;        /* >0: crossing-flow durations come from a table of this many
                                   distinct payloads x K x K IEEE quotients (0: divided at run time) */
} mp_instance_info;

/* ---- library ------------------------------------------------------------ */
int32_t mp_abi_version(void);
int32_t mp_device_count(void);
/* Number of kernel launches this process has issued through the library. */
int64_t mp_launch_count(void);

/* ---- instances (replaces `_Instance.__init__`, solver.py:45-72) ---------- */
int32_t mp_instance_create(const mp_problem *prob, int32_t device,
                           mp_instance **out, mp_error *err);
void    mp_instance_destroy(mp_instance *inst);
int32_t mp_instance_info_get(const mp_instance *inst, mp_instance_info *info);
/* Override the launch shape: lanes per placement G in {1,2,4,8,16,32} (0 = auto),
 * lanes per warp that own a placement U (multiple of G, <= 32; 0 = auto), CTAs
 * per SM cap (0 = auto), on-chip ready capacity (0 = auto); flags bit 0
 * (MP_TUNE_NO_COLO) dispatches co-located flows as ordinary steps.  Results
 * never depend on these knobs. */
#define MP_TUNE_NO_COLO 1
#define MP_TUNE_TPP_REG 4   /* thread-per-placement with the ready set in registers (when the
                               calibrated peak fits a 4/8/16 template) instead of shared memory */
#define MP_TUNE_OFFCHIP 8   /* group kernel with per-placement state in global memory */
#define MP_TUNE_TPP_ROUND1 16 /* thread-per-placement: the round-1 shared-memory-ready-set evaluator (A/B only) */
#define MP_TUNE_NO_DURTAB 32 /* thread-per-placement: divide payload / bw at run time instead of
                               reading the flow-duration table (A/B and parity tests) */
#define MP_TUNE_COST_GLOBAL 64  /* thread-per-placement (duration table): op costs read through L1
                                  (default: only when that fits 1.5x the lanes, e.g. C3) */
#define MP_TUNE_COST_SMEM 128   /* ... op costs always staged in shared memory (A/B) */
#define MP_TUNE_ROW3 256       /* thread-per-placement: 3-bit row tile whenever K <= 8 (default: only
                                  where it fits more lanes than nibbles) */
#define MP_TUNE_NO_TPP  2   /* do not use the thread-per-placement kernels (used only with
                               automatic G/U) */
int32_t mp_instance_tune(mp_instance *inst, int32_t group_lanes, int32_t lanes_used, int32_t ctas_per_sm,
                         int32_t ready_cap, uint32_t flags);

/* ---- batched evaluation (K3; replaces one `_schedule` call per row) ------ */
/* makespan[p] = +inf unless status[p] == MP_ROW_OK.  mem_dev/overflow may be NULL. */
int32_t mp_evaluate_batch(mp_instance *inst, const uint8_t *placements, int64_t n_rows,
                          double *makespan, int8_t *status, int32_t *mem_dev,
                          int64_t *overflow, uint32_t flags, void *stream, mp_error *err);

/* Keep-best over supplied rows (K4): first (lowest-index) strict minimum among
 * feasible rows, as the `brute_force` loop (solver.py:271-279).  *best_row = -1
 * when no row is feasible.  makespan/status may be NULL (argmin only).
 * best_row / best_ms are always HOST pointers. */
int32_t mp_evaluate_argmin(mp_instance *inst, const uint8_t *placements, int64_t n_rows,
                           double *makespan, int8_t *status,
                           int64_t *best_row, double *best_ms,
                           uint32_t flags, void *stream, mp_error *err);

/* Enumerate rows first..first+count-1 of itertools.product(devices, repeat=n)
 * zipped onto op_order (solver.py:268-272; most significant digit = op_order[0])
 * and keep the best (K4 with on-chip placement generation).  op_order is a HOST
 * array of n_ops op indices.  Guard: n_ops*log2(n_dev) <= 24 else MP_ERR_TOO_LARGE. */
int32_t mp_enumerate_argmin(mp_instance *inst, const int32_t *op_order,
                            uint64_t first, uint64_t count,
                            int64_t *best_index, double *best_ms,
                            void *stream, mp_error *err);

/* Exact single schedule (schedule_for_assignment, solver.py:151-165): starts/ends
 * of all n_ops+n_flows nodes in node-index order.  HOST pointers.  Returns
 * MP_ERR_MEMORY_EXCEEDED with a=device index, b=overflow, or MP_ERR_BAD_DEVICE. */
int32_t mp_schedule_one(mp_instance *inst, const uint8_t *placement,
                        double *starts, double *ends, double *makespan, mp_error *err);

/* ---- GPU local search (K5; no reference analogue) ----------- */
/* n_chains independent chains start from `seed_rows` (n_seed rows, chain c uses
 * row c % n_seed), each runs `rounds` x `moves` single-op re-assignments with a
 * counter-based RNG keyed by (rng_seed, global chain id), accepting a move iff
 * the makespan does not increase.  The best row over all chains (lowest chain id
 * on ties) is written to best_row[n_ops] with its makespan; every chain's final
 * makespan to chain_ms[n_chains] when non-NULL.  chain_base offsets the global
 * chain id (for sharding chains across GPUs).  Host pointers. */
int32_t mp_local_search(mp_instance *inst, const uint8_t *seed_rows, int32_t n_seed,
                        int64_t n_chains, int64_t chain_base, int32_t moves,
                        uint64_t rng_seed, uint8_t *best_row, double *best_ms,
                        int64_t *best_chain, double *chain_ms, void *stream, mp_error *err);

/* ---- Branch and bound (replaces solve_exact, solver.py:172-254) ----------
 * Ops are branched in `op_order` (n_ops op indices = topo_order(gc),
 * solver.py:72), devices ascending; memory-prefix check (:233-234), the
 * reference's node bound (:197-215), strict incumbent rule (:225-230).  A round
 * bounds up to 65536 children on the GPU at once; leaves are scheduled exactly.
 * gap == 0: the optimum and, among optimal rows, the lexicographically smallest
 * in op_order (= brute_force's first strict minimum) whatever the seeds.
 * gap > 0: prune when bound >= best*(1-gap) (:239).  node_limit < 0 / time_limit_s
 * < 0 mean unlimited; limits are checked between rounds.  `seed_rows` (may be
 * NULL) are evaluated first as incumbent candidates.  solve_status receives
 * MP_SOLVE_* (Status.OPTIMAL / FEASIBLE / INFEASIBLE / BUDGET, placement.py:12-16);
 * best_row/best_ms are valid for OPTIMAL and FEASIBLE. */
#define MP_SOLVE_OPTIMAL    0
#define MP_SOLVE_FEASIBLE   1
#define MP_SOLVE_INFEASIBLE 2
#define MP_SOLVE_BUDGET     3
int32_t mp_branch_and_bound(mp_instance *inst, const int32_t *op_order, double gap,
                            int64_t node_limit, double time_limit_s,
                            const uint8_t *seed_rows, int32_t n_seed,
                            uint8_t *best_row, double *best_ms, int32_t *solve_status,
                            int64_t *visited, mp_error *err);

/* ---- greedy baselines (replaces greedy_place, baselines.py:27-86) ---------
 * One warp, lane k scores device k; ops in `op_order` (topo_order(gc)).  kind 0
 * = EARLIEST_FINISH, 1 = EARLIEST_START.  `row` receives the device index of each
 * op; the caller schedules it (mp_schedule_one) exactly as the reference's final
 * `_schedule` call.  MP_ERR_INFEASIBLE_MEMORY when no device can hold an op. */
int32_t mp_greedy_place(mp_instance *inst, const int32_t *op_order, int32_t kind,
                        uint8_t *row, mp_error *err);

/* ---- schedule audit (replaces check_feasibility, simulator.py:179-264) ----
 * starts/ends: [n_ops + n_flows] node times (index = node index).  Violations are
 * returned in the reference's report order; *n_out = their number (only the first
 * out_cap are written).  kind / x / y:
 *   0 memory-over          x = device index, y = load
 *   1 duration-mismatch    x = node index
 *   2 negative start       x = node index      (reported as duration-mismatch)
 *   3 precedence-break     x = link index (2f: src->flow f, 2f+1: flow f->dst)
 *   4 device-overlap       x, y = op indices (x < y)
 *   5 source-channel       x, y = flow indices (x < y)
 *   6 dest-channel         x, y = flow indices (x < y)                        */
typedef struct mp_violation {
    int32_t kind;
    int32_t pad;
    int64_t x, y;
} mp_violation;
int32_t mp_audit_schedule(mp_instance *inst, const uint8_t *row, const double *starts,
                          const double *ends, double tol, mp_violation *out, int64_t out_cap,
                          int64_t *n_out, mp_error *err);

/* ---- graph ingestion (replaces the parse of fileio.load_graph, fileio.py:58-70) ----
 * Streams a schema-1 graph document into flat arrays and applies the OpNode /
 * FlowEdge / CompGraph validations (graph.py:31-109).  MP_ERR_INVALID (message in
 * err) for anything off the fast path; the arrays live until mp_graph_doc_free.
 * Strings (op types, type sequences) are interned: string k is
 * str[str_beg[k] .. str_beg[k+1]) (UTF-8). */
typedef struct mp_graph_doc mp_graph_doc;
typedef struct mp_graph_view {
    int64_t n_nodes, n_edges, n_strings;
    const int64_t *id, *mem;            /* [n_nodes] in file order                       */
    const int8_t *tag;                  /* [n_nodes] 0 plain, 1 fused, 2 bound           */
    const int32_t *op_type;             /* [n_nodes] string index                        */
    const int32_t *seq_beg, *seq;       /* type_seq: seq[seq_beg[i] .. seq_beg[i+1])    */
    const int32_t *mem_beg;             /* members: members[mem_beg[i] .. mem_beg[i+1]) */
    const int64_t *members;
    const int32_t *ct_beg;              /* compute_time entries of node i, file order    */
    const int64_t *ct_dev;
    const double *ct_val;
    const int64_t *esrc, *edst, *epay;  /* [n_edges] in file order                      */
    const int64_t *str_beg;             /* [n_strings + 1]                               */
    const char *str;
} mp_graph_view;
int32_t mp_graph_load_json(const char *path, mp_graph_doc **doc, mp_graph_view *view, mp_error *err);
void    mp_graph_doc_free(mp_graph_doc *doc);

/* ---- GCOF coarsening (K1/K2; replaces gcof, fusion.py:271-304) ----------- */
typedef struct mp_coarsen_input {
    int32_t n_nodes;            /* V: input op nodes in ascending id order          */
    int32_t n_edges;            /* E: edges in the graph's edge-list order          */
    int32_t n_dev;              /* devices with costs; cost rows are [n_nodes*n_dev] */
    const int64_t *node_id;     /* [V] ascending                                    */
    const int32_t *seq_beg;     /* [V+1] CSR into seq_types: the node's type_seq     */
    const int32_t *seq_types;   /* interned type ids                                 */
    const int32_t *tag;         /* [V] 0 plain, 1 fused, 2 bound                     */
    const int64_t *mem;         /* [V]                                              */
    const double  *cost;        /* [V*n_dev]; NaN = device absent from compute_time */
    const int32_t *esrc;        /* [E] node index                                   */
    const int32_t *edst;        /* [E]                                              */
    const int64_t *payload;     /* [E]                                              */
    int32_t n_rules;
    const int32_t *rule_id;     /* [R]                                              */
    const int32_t *rule_beg;    /* [R+1] CSR into rule_types                        */
    const int32_t *rule_types;
    int32_t n_overrides;        /* fused-kernel cost overrides (profiles.py:140-160) */
    const int32_t *ov_beg;      /* [O+1] CSR into ov_types: the override's type_seq  */
    const int32_t *ov_types;
    const int32_t *ov_dev;      /* [O] device index                                 */
    const double  *ov_time;     /* [O]                                              */
    int32_t sum_mode;           /* fused-cost member sums: 1 = CPython >= 3.12 sum()
                                   (Neumaier-compensated, bltinmodule.c builtin_sum_impl),
                                   0 = plain left fold (CPython <= 3.11)              */
} mp_coarsen_input;

/* Output arrays are allocated by the library (free with mp_coarsen_free). */
typedef struct mp_coarsen_output {
    int32_t n_groups;           /* output nodes, ascending id (= min member id)     */
    int32_t n_edges;            /* quotient edges, sorted by (u, v)                  */
    int32_t *grp_node;          /* [n_groups] representative input node index        */
    int32_t *grp_tag;           /* [n_groups] 0 plain, 1 fused                       */
    int32_t *mem_beg;           /* [n_groups+1] CSR into members (input node indices, chain order) */
    int32_t *members;
    int64_t *grp_mem;           /* [n_groups] summed mem_bytes                        */
    double  *grp_cost;          /* [n_groups*n_dev] member-order sums / overrides; NaN = absent */
    int32_t *out_src;           /* [n_edges] group index                             */
    int32_t *out_dst;
    int64_t *out_payload;
    int32_t ordered_replay;     /* 1: order hazards present, the DFS was replayed in order;
                                   0: candidate chains resolved in parallel */
} mp_coarsen_output;

int32_t mp_coarsen(const mp_coarsen_input *in, int32_t device,
                   mp_coarsen_output *out, mp_error *err);
void    mp_coarsen_free(mp_coarsen_output *out);

#ifdef __cplusplus
}
#endif
#endif /* MOIRAI_B200_H */
