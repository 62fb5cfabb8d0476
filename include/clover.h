/*
 * clover.h -- C-ABI of libclover_b200.so, the B200 (sm_100a) configuration-search
 * hot path of Clover (arXiv 2304.09781).
 *
 * Plain C: pointers, sizes and PODs only; no torch types.  Every entry point
 * returns a clv_status; non-zero codes map 1:1 onto the reference exception
 * hierarchy (reference pkg/src/carbon_sched/errors.py:4-37) and
 * clv_last_error() returns the message.  Device pointers (suffix _dev) are
 * owned by the caller (cudaMalloc / torch.Tensor.data_ptr()); the context owns
 * the tables and scratch.  One context per device; calls are stream-ordered on
 * the cudaStream_t passed as `stream` (NULL = legacy default stream); calls
 * that fill a host-side clv_best synchronise that stream.
 *
 * A context is NOT re-entrant across streams: its scratch (selection partials,
 * the chain move log, the re-plan staging buffers, the DES workload cache) is
 * shared by every call, so all calls on one context must be issued from ONE
 * stream at a time (or be ordered by the caller with events).  Use one context
 * per concurrent stream.  ("not re-entrant, stream-ordered".)
 *
 * Reference interface each entry point replaces (SPEC = reference SPEC.md,
 * mig.py / core.py = reference pkg/src/carbon_sched/):
 *   clv_set_topology        MigTopology.__init__ / load_topology      mig.py:94-123, 201-217
 *   clv_set_profile         ProfileTable / memory_feasible
 *   clv_build_feasibility   MigTopology._partition_search (bulk)      mig.py:144-170
 *   clv_feasible            is_feasible_fleet                         mig.py:179-181, 234
 *   clv_realize             partition_fleet + realize                 mig.py:172-177
 *   clv_score_graphs        evaluate() over ConfigGraphs, Eqs 1-3,6
 *   clv_score_x             FleetConfig decode + evaluate             mig.py:237-299
 *   clv_oracle_search       oracle_search
 *   clv_anneal              anneal + sample_neighbor
 *   clv_sweep               blover_search draws (x-space sweep)
 *   clv_select_chains /
 *   clv_reduce_records      best tracking / fixed-order winner
 *   clv_derive_seed         derive_seed                               core.py:107-118
 *   clv_set_sim_profile /
 *   clv_simulate            simulate / p95 / overall_accuracy (batched serving DES,
 *                           one independent simulation per candidate)
 */
#ifndef CLOVER_B200_H
#define CLOVER_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CLV_ABI_VERSION 3
#define CLV_MAX_VARIANTS 8
#define CLV_MAX_EDGES 40
#define CLV_MAX_CONFIGS 32
#define CLV_MAX_FAMILIES 8
#define CLV_MAX_PODS 8

typedef enum clv_status {
    CLV_OK = 0,
    CLV_ERR_CARBON_SCHED = 1,          /* CarbonSchedError            errors.py:4  */
    CLV_ERR_INVALID_CONFIG = 2,        /* InvalidConfigError          errors.py:8  */
    CLV_ERR_INFEASIBLE_ASSIGNMENT = 3, /* InfeasibleAssignmentError   errors.py:12 */
    CLV_ERR_INCOMPATIBLE_GRAPHS = 4,   /* IncompatibleGraphsError     errors.py:16 */
    CLV_ERR_INFEASIBLE_GRAPH = 5,      /* InfeasibleGraphError        errors.py:20 */
    CLV_ERR_NO_NEIGHBOR = 6,           /* NoNeighborError             errors.py:24 */
    CLV_ERR_PROFILE = 7,               /* ProfileError                errors.py:28 */
    CLV_ERR_TRACE = 8,                 /* TraceError                  errors.py:32 */
    CLV_ERR_SIMULATION = 9,            /* SimulationError             errors.py:36 */
    CLV_ERR_CUDA = 100,
    CLV_ERR_OUT_OF_MEMORY = 101,
    CLV_ERR_NOT_READY = 102            /* tables / topology / feasibility not loaded */
} clv_status;

typedef struct clv_ctx clv_ctx;

/* Evaluation parameters of one scoring call (ObjectiveParams core.py:63-101 + workload). */
typedef struct clv_eval_params {
    double arrival_rps;      /* R: Poisson request rate                */
    double ci;               /* carbon intensity, gCO2/kWh           */
    double carbon_weight;    /* lambda of Eq. 3, clamped to [0,1]                 */
    double base_accuracy;    /* A_base of Eq. 1 (fraction)                       */
    double base_carbon_g;    /* C_base of Eq. 2 (gCO2/request)                   */
    double latency_slo_ms;   /* L_tail of Eq. 5                                  */
    double rho_sat;          /* queueing-factor saturation (0.999)               */
    int32_t strict_eq6;      /* 1 = verbatim Eq. 6 (CARBON_SCHED_STRICT_EQ6)     */
    int32_t n_gpus;          /* fleet size n                                     */
    double max_accuracy_loss_pct; /* accuracy_threshold_mode: candidates with
                                     dA < -max_loss count as SLA-violating; +inf = off */
} clv_eval_params;

/* Selected candidate of a scoring / search call. */
typedef struct clv_best {
    int64_t index;           /* candidate index (global), -1 if none            */
    double f, h, p95_ms, accuracy, energy_wh;
    int32_t sla_met;
    int32_t found;           /* 1 if at least one valid candidate was scored     */
    int64_t valid_count;     /* candidates that were feasible and scored         */
    int64_t sla_count;       /* of those, SLA-meeting                            */
} clv_best;

/* Selection rules (SPEC:464/482-483 vs SPEC:539/548). */
#define CLV_SELECT_BEST_H 0  /* (SLA desc, h asc, index asc)                                 */
#define CLV_SELECT_ORACLE 1  /* (SLA desc, f desc, index asc), none SLA: (p95 asc, index asc) */

/* Annealing schedule. */
typedef struct clv_anneal_params {
    double t_init, cooling_step, t_floor;
    int32_t stall_limit;
    int32_t max_steps;
    int32_t proposal;        /* 0 = best-h neighbour, 1 = uniform (min-hash) neighbour */
    int32_t evaluate;        /* 0 = score whole neighbourhood, 1 = score proposal only */
    int32_t flags;           /* CLV_ANNEAL_MULT_COOLING | CLV_ANNEAL_PAPER_MOVES (0 = SPEC defaults) */
} clv_anneal_params;

/* clv_anneal_params.flags */
#define CLV_ANNEAL_MULT_COOLING 1  /* T_k = max(t_floor, t_init (1 - cooling_step)^k), SPEC:492 option */
#define CLV_ANNEAL_PAPER_MOVES  2  /* + one-instance add / remove moves (GED 1):
                                      indices E*E + NP*NP + a (add on edge a), + E + r (remove from r) */

/* Per-chain result written by clv_anneal (device memory). */
typedef struct clv_chain_result {
    double f, h, p95_ms, accuracy, energy_wh;   /* best candidate */
    int32_t sla_met;
    int32_t status;          /* 0 max_steps, 1 stalled, 2 no neighbour, -1 invalid start */
    int32_t steps;
    int32_t best_step;       /* -1 = the start graph */
    int64_t best_index;      /* canonical neighbour index at best_step, -1 = start */
    int64_t evals;           /* candidates scored by this chain (start included) */
    int64_t edge_evals;      /* sum over steps of (non-zero edges of the centre x candidates scored):
                                the E_nz factor of the per-candidate work */
} clv_chain_result;

/* One row of the optional per-step log (SPEC:487 schema). */
typedef struct clv_log_row {
    double temp, f, h, p95_ms;
    int32_t iter, ged_from_center, sla_met, accepted, new_best, n_neighbours;
} clv_log_row;

/* 32-byte winner record exchanged between ranks (one per GPU per round). */
typedef struct clv_record {
    uint64_t k1;             /* 0 = SLA met, 1 = not (lexicographic primary)      */
    uint64_t k2;             /* order-preserving key of h                          */
    int64_t index;           /* global chain / candidate index                    */
    double h;
} clv_record;

/* One pod of a mixed-family sweep. */
typedef struct clv_pod {
    int32_t family;
    int32_t n_gpus;
    double weight;
    clv_eval_params params;
} clv_pod;

/* Serving workload of the discrete-event simulator. */
typedef struct clv_workload {
    double arrival_rps;      /* Poisson rate (or 1 / period in periodic mode)     */
    double duration_s;       /* arrivals in [0, duration)                          */
    uint64_t seed;           /* counter-RNG key of arrivals and service draws      */
    int32_t periodic;        /* 1 = the SPEC's degenerate periodic-arrival mode    */
    int32_t warmup;          /* completions excluded from latency stats; -1 = max(100, N/20) */
} clv_workload;

/* One simulation's SimReport. */
typedef struct clv_sim_report {
    double p95_ms, mean_latency_ms, throughput_rps;
    double energy_wh_total, energy_wh_per_request;   /* per request = active energy / completed */
    double accuracy;                                 /* overall_accuracy */
    int64_t completed;       /* requests served (all arrivals)                     */
    int64_t counted;         /* requests in the latency statistics (after warm-up) */
    int32_t sla_met;         /* p95_ms <= l_tail_ms                                */
    int32_t status;          /* 0 ok, else a clv_status of this simulation          */
} clv_sim_report;

int clv_abi_version(void);
int clv_create(int device, clv_ctx **out);
void clv_destroy(clv_ctx *ctx);
const char *clv_last_error(const clv_ctx *ctx);
uint64_t clv_derive_seed(const uint64_t *parts, int n_parts);

int clv_set_topology(clv_ctx *ctx, int n_configs, const int32_t *config_ids,
                     const int32_t *counts5, const double *memory_gb5);
/* Scoring rows of one profile family, edge e = (v-1)*5 + slice index:
 * fixed-point thr/acc/en rows, per-slice idle row, lat95 = p95 service time (ms, the value
 * a p95 estimate reports) and svc = mean service time (ms, the request shares of the
 * instance-pull p95 walk); both > 0, and lat95 must order the edges like svc
 * (one distribution family per catalog). */
int clv_set_profile(clv_ctx *ctx, int family, int n_variants,
                    const int64_t *thr_q, const int64_t *acc_q, const int64_t *en_q,
                    const int64_t *idle_q5, const double *lat95, const double *svc_ms,
                    const uint8_t *mem_ok, int kt, int ke, int ki);
int clv_build_feasibility(clv_ctx *ctx, int n_max, void *stream);
int64_t clv_feasibility_bytes(const clv_ctx *ctx);

int clv_feasible(clv_ctx *ctx, int n, const int32_t *vec5_dev, int64_t count,
                 uint8_t *out_dev, void *stream);
int clv_realize(clv_ctx *ctx, int n, const int32_t *vec5_host, int32_t *partitions_host,
                void *stream);

int clv_score_graphs(clv_ctx *ctx, int family, const uint16_t *w_dev, int64_t count,
                     int64_t index_base, const clv_eval_params *params, int select_mode,
                     double *f_dev, double *h_dev, uint8_t *sla_dev, uint8_t *feasible_dev,
                     double *p95_dev, clv_best *best, void *stream);
/* clv_score_x: rows of n partition ids (xp, uint8[count][n]) and CSR variant bytes
 * (xv, row c = xv[xv_offsets[c] .. xv_offsets[c+1])).  Row validation follows
 * FleetConfig.__init__ (mig.py:248-263), then evaluation: an unknown partition id ->
 * CLV_ERR_INVALID_CONFIG; else a length mismatch or a variant < 1 ->
 * CLV_ERR_CARBON_SCHED; else a variant > V or one that does not fit its slice ->
 * CLV_ERR_INFEASIBLE_ASSIGNMENT.  The error reported is that of the LOWEST failing
 * row (its index in the message), as a sequential loop would raise it. */
int clv_score_x(clv_ctx *ctx, int family, int n, const uint8_t *xp_dev,
                const uint8_t *xv_dev, const int64_t *xv_offsets_dev, int64_t count,
                int64_t index_base, const clv_eval_params *params, int select_mode,
                double *f_dev, double *h_dev, uint8_t *sla_dev, clv_best *best, void *stream);
int clv_oracle_search(clv_ctx *ctx, int family, int n, int64_t begin, int64_t end,
                      const clv_eval_params *params, clv_best *best, int64_t *total,
                      void *stream);
int clv_oracle_size(clv_ctx *ctx, int family, int64_t *total);
int clv_oracle_decode(clv_ctx *ctx, int family, int64_t index, int32_t *config_id,
                      int32_t *assignment7, int32_t *n_slices);
int clv_anneal(clv_ctx *ctx, int family, int n, int n_chains, int64_t chain_base,
               const uint16_t *start_w_dev, const clv_eval_params *params, int n_params,
               const clv_anneal_params *ap, uint64_t seed, int cluster_size,
               clv_chain_result *results_dev, uint16_t *best_w_dev, uint16_t *final_w_dev,
               clv_log_row *log_dev, void *stream);
int clv_select_chains(clv_ctx *ctx, const clv_chain_result *results_dev, int n_chains,
                      int64_t chain_base, clv_record *record_dev, void *stream);
/* clv_replan: one complete re-plan from HOST buffers in one call -- start graphs copied
 * H2D, clv_anneal, clv_select_chains, every output copied D2H, stream synchronised.
 * Device staging is context-owned; host buffers should be pinned for async copies.
 * Replaces the reference-side loop over independent anneal() runs
 * plus its best tracking for one GPU; multi-rank callers exchange the
 * returned record (clv_reduce_records). */
int clv_replan(clv_ctx *ctx, int family, int n, int n_chains, int64_t chain_base,
               const uint16_t *start_w_host, const clv_eval_params *params, int n_params,
               const clv_anneal_params *ap, uint64_t seed, int cluster_size,
               clv_chain_result *results_host, uint16_t *best_w_host, uint16_t *final_w_host,
               clv_record *record_host, void *stream);
int clv_reduce_records(clv_ctx *ctx, const clv_record *records_dev, int count,
                       clv_record *out_dev, void *stream);
int clv_sweep(clv_ctx *ctx, int n_pods, const clv_pod *pods, int64_t begin, int64_t end,
              uint64_t seed, double *f_dev, double *h_dev, uint8_t *sla_dev,
              clv_best *best, void *stream);
int clv_sweep_decode(clv_ctx *ctx, int n_pods, const clv_pod *pods, uint64_t seed,
                     int64_t index, int32_t *partitions_host, int32_t *assignments_host,
                     int32_t *n_assignments);

/* Simulator rows of a profile family: per edge e = (v-1)*5 + slice index the mean
 * service time, distribution (0 deterministic, 1 exponential, 2 lognormal), sigma
 * and active energy per request; idle power per slice kind; accuracy per variant. */
int clv_set_sim_profile(clv_ctx *ctx, int family, int n_variants, const double *mean_service_ms,
                        const int32_t *dist, const double *sigma, const double *energy_wh,
                        const double *idle_w5, const double *accuracy, const uint8_t *mem_ok);
/* Simulate `count` fleets.  Fleet c's instances are inst_edge_dev[inst_off_dev[c] ..
 * inst_off_dev[c+1]) (edge ids in FleetConfig.instances() order, at most
 * max_instances).  reports_dev[count]; optional variant_counts_dev[count][8] and
 * instance_counts_dev[inst_off[count]].  *n_requests (host, optional) receives the
 * workload's request count.  Synchronises the stream once (request-count readback). */
int clv_simulate(clv_ctx *ctx, int family, const clv_workload *workload, int64_t count,
                 const uint8_t *inst_edge_dev, const int64_t *inst_off_dev, int max_instances,
                 double l_tail_ms, clv_sim_report *reports_dev, int64_t *variant_counts_dev,
                 int64_t *instance_counts_dev, int64_t *n_requests, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CLOVER_B200_H */
