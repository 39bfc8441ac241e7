/*
 * saturn.h -- C ABI of the B200-native SPASE plan evaluator and searcher.
 *
 * SPASE (§4.1) asks, for every training job, for a parallelism (UPP), a
 * GPU count, a node and a start time that together minimise the makespan, given the
 * profiled runtime table (Table 1).  This library evaluates and searches
 * candidate plans in bulk on one B200 per process:
 *
 *   a plan = a GENOME: cfg[t] in [0, S_t) picks job t's configuration (one config per job,
 *   Eq. 3) and perm[0..T) is a priority permutation of the job ids.  A genome
 *   is turned into a schedule by the list-scheduling DECODER (reading A6): in
 *   priority order each job with config (g, R) starts at the g-th smallest free time of the
 *   node where that start is earliest (ties -> lowest node id), takes the g GPUs of that
 *   node free by then with the latest free times (ties -> lower GPU id), and holds them for
 *   [s, s+R).  The makespan is max_t (s_t + R_t) (Eq. 2).  Every decoded plan
 *   satisfies Eqs. 3-11: one node, exactly g GPUs, one gang start, no overlap on a GPU.
 *
 * Conventions
 *   - Every function is extern "C", returns saturn_status, never throws, never aborts.
 *     On failure saturn_last_error(p) describes the cause (owned by the handle, valid until
 *     the next call on it).
 *   - Host pointers are caller-owned; the library copies what it needs during the call.
 *     Pointers documented "device" are caller-owned CUDA device memory on the handle's
 *     device (e.g. torch tensor storage); the library never frees them.
 *   - Streams are caller-owned cudaStream_t passed as void* (NULL = legacy default stream).
 *     Device-output calls are stream-ordered and asynchronous; calls with host outputs
 *     synchronise the stream before returning.
 *   - Integers: runtimes are int32 seconds (reading A4/A5: integer time loses nothing).
 *   - A handle is not thread safe; distinct handles are independent.
 *   - Limits: 1 <= n_nodes, sum_n GPU_n <= 32; 1 <= T <= 255 jobs (u8 genes); R < 2^24 s;
 *     sum_t max_s R < 2^26 s (packed (makespan, index) keys); <= 255 configs per job;
 *     the packed table (4 B per (job, config) + 2 B per job) <= 48 KB.
 */
#ifndef SATURN_H
#define SATURN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct saturn_plan saturn_plan; /* opaque; owns the device table and workspaces */

typedef enum {
  SATURN_OK = 0,
  SATURN_EINVAL = 1,          /* bad argument or table value (message names it)            */
  SATURN_EUNSCHEDULABLE = 2,  /* a job has no feasible config fitting any node */
  SATURN_ELIMIT = 3,          /* a size limit (enumeration space, shared memory) exceeded   */
  SATURN_ECUDA = 4,           /* CUDA runtime error (message = cudaGetErrorString)          */
  SATURN_ENCCL = 5,           /* NCCL error or NCCL library not loadable                    */
  SATURN_ESTATE = 6           /* call out of order (e.g. evaluate before a table is loaded) */
} saturn_status;

/* saturn_result.flags */
enum { SATURN_PROVEN_OPTIMAL = 1, SATURN_INCUMBENT = 2, SATURN_PREFIX_SHARED = 4, SATURN_SYMMETRY_REDUCED = 8 };

/* saturn_set_decoder kinds (row a5: two device designs, chosen by measurement; NODE_SMEM =
 * the thread design with every node's sorted free-time vector in shared memory and a runtime
 * node count -- the default for clusters without a compiled register shape) */
enum { SATURN_DECODER_AUTO = 0, SATURN_DECODER_THREAD = 1, SATURN_DECODER_WARP = 2, SATURN_DECODER_NODE_SMEM = 3 };

/* One job of a decoded plan = the paper's per-task outputs (Table 1 B, O, P,
 * I): node n (O), UPP index and GPU count of the chosen config, the config index s into the
 * job's compacted list (B), the gang start I and end I + R, and bit g of gpu_mask set iff
 * the job holds GPU g of its node (P).  32 bytes. */
typedef struct {
  int32_t node;
  int32_t upp;
  int32_t gpus;
  int32_t cfg;
  int32_t start_s;
  int32_t end_s;
  uint64_t gpu_mask;
} saturn_placement;

typedef struct {
  int64_t makespan;       /* best makespan found (seconds)                              */
  uint64_t genome_index;  /* enumerate: index of the best genome (smallest on ties)     */
  uint64_t evaluated;     /* full decodes performed by this call, all ranks             */
  double seconds;         /* wall time of the call                                      */
  int32_t flags;          /* SATURN_PROVEN_OPTIMAL (enumerate) | SATURN_INCUMBENT (search) */
  int32_t generations;    /* search: generations run                                    */
  uint64_t leaves;        /* enumerate: leaves visited (prefix-shared DFS: after the
                             branch-and-bound cut; these are not full decodes)          */
} saturn_result;

/* Genetic search parameters (row a7, oracle/ga.py GA v5).
 * Probabilities are given as q32 thresholds (floor(p * 2^32)); every gate compares a 16-bit
 * Philox field h with threshold >> 16 and fires iff h < threshold >> 16, so the resolution is
 * 2^-16 and p = 1.0 (0xFFFFFFFF) fires with probability 65535/65536. */
typedef struct {
  uint64_t seed;
  int64_t population;            /* genomes per GPU, >= 64 and >= 2 * elites            */
  int64_t max_generations;       /* generations after the initial population (>= 0)     */
  double time_budget_s;          /* stop at the first epoch boundary past this; 0 = none */
  int32_t elites;                /* 1..32 genomes carried unchanged to the next generation */
  int32_t generations_per_epoch; /* island migration period (multi-GPU), >= 1           */
  uint32_t p_xover_q32;          /* per-pair crossover probability (both children)       */
  uint32_t p_cfg_mut_q32;        /* per-child probability that ONE job (drawn uniformly) gets
                                    a new config drawn uniformly from its S_t             */
  uint32_t p_perm_mut_q32;       /* per-child permutation mutation probability (swap or
                                    insertion, 50/50)                                    */
  const uint8_t *seed_cfg;       /* host [n_seed][T] genomes placed first, or NULL        */
  const uint8_t *seed_perm;      /* host [n_seed][T]                                      */
  int64_t n_seed;
  int32_t local_search_iters;    /* >0: memetic step -- at every epoch boundary the E elites
                                    get this many best-improvement local-search iterations
                                    (saturn_improve) before the exchange; 0 = off        */
} saturn_search_params;

/* Create a handle for a cluster of n_nodes nodes with node_gpus[n] GPUs each (Table 1: N,
 * GPU_n) on CUDA device `cuda_device`.  cuda_device = -1 creates a
 * HOST-ONLY handle: table loading/compaction, baselines and the other host calls work, every
 * device call returns ESTATE.  EINVAL: n_nodes < 1, n_nodes > 32, any GPU_n < 1,
 * sum GPU_n > 32 (reading A15: the trace decoder gives every GPU of the cluster one
 * lane of a warp; SURVEY.md §8b's u64 masks would allow 64).  ECUDA: device not usable. */
saturn_status saturn_plan_create(const int32_t *node_gpus, int32_t n_nodes, int32_t cuda_device,
                                 saturn_plan **out);

/* Device workspace (north star: "PyTorch used only for device memory").
 * saturn_workspace_bytes: bytes a freshly bound workspace needs for one saturn_search with
 * `sp` (NULL: evaluate / enumerate / best_plan only) on the loaded table, including the table
 * itself, the two populations (2 x population x record bytes), their makespans, the candidate
 * list, the elite records and the trace scratch.  Host-buffer calls (saturn_evaluate_host,
 * saturn_improve) need min(n, 2^24) x (2T + 4) bytes more.  ESTATE before a table is loaded or
 * on a host-only handle; EINVAL for out-of-range population / elites.
 * saturn_bind_workspace: bind a caller-owned device buffer (e.g. a torch.empty(bytes,
 * dtype=torch.uint8) tensor on the handle's device, 256-byte aligned) -- from then on every
 * device buffer the handle needs is carved from it instead of cudaMalloc (the peer-link
 * exchange buffers excepted: CUDA IPC needs their own allocations).  The caller keeps it
 * alive until it unbinds (d_workspace = NULL) or destroys the handle.  Binding synchronises
 * the device, drops the handle's previous buffers (the last search population becomes
 * unavailable) and moves a loaded table into the workspace.  A call that runs out of the bound
 * workspace returns ELIMIT naming the allocation.  EINVAL: not device memory of the
 * handle's device, or misaligned. */
saturn_status saturn_workspace_bytes(const saturn_plan *p, const saturn_search_params *sp, uint64_t *bytes);
saturn_status saturn_bind_workspace(saturn_plan *p, void *d_workspace, uint64_t bytes);

/* Load the profiled runtime table (row a1; Table 1 G_t, R_t; the Trial Runner grid over
 * "all supported parallelisms and GPU apportionment levels").
 * runtime_s: host int32 [n_jobs][n_upps][max_gpus], entry [t][u][g-1] = runtime of job t
 * under UPP u on g GPUs; <= 0 marks an infeasible (null) profile.
 * The table is compacted (row a2): job t's configs are its feasible entries with
 * g <= max_n GPU_n (single-node jobs) in UPP-major, ascending-g order
 * (SPEC.md:52); config index s in genomes and placements refers to this order.
 * EINVAL: n_jobs not in [1,255], n_upps not in [1,255], max_gpus < 1, R >= 2^24, sum_t max_s R >= 2^26,
 * > 255 configs for a job; EUNSCHEDULABLE: a job with no feasible config (message names it);
 * ELIMIT: packed table > 48 KB.  Replaces any previous table and search state. */
saturn_status saturn_load_runtime_table(saturn_plan *p, const int32_t *runtime_s, int32_t n_jobs,
                                        int32_t n_upps, int32_t max_gpus);

/* Shape of the compacted table: n_jobs and S_t (configs per job, host int32 [n_jobs], may
 * be NULL).  ESTATE before a table is loaded. */
saturn_status saturn_num_configs(const saturn_plan *p, int32_t *n_jobs, int32_t *configs_per_job);

/* Compacted config s of job t: UPP index, GPU count and runtime.  EINVAL if out of range. */
saturn_status saturn_config(const saturn_plan *p, int32_t job, int32_t cfg, int32_t *upp, int32_t *gpus,
                            int32_t *runtime_s);

/* Select the device decoder design (AUTO = thread design when compiled for the cluster shape,
 * else warp).  WARP applies to evaluate; NODE_SMEM applies to evaluate, search, local search
 * and enumeration (index order instead of the register-state DFS).  EINVAL for an unknown
 * kind. */
saturn_status saturn_set_decoder(saturn_plan *p, int32_t kind);

/* Decode n genomes (row a5).  d_cfg, d_perm: device uint8 [n][T] (genome-major rows);
 * d_makespan: device int32 [n].  An invalid genome (perm not a permutation of 0..T-1, or
 * cfg[t] >= S_t) yields makespan -1.  Asynchronous on `stream`.  ESTATE without a table. */
saturn_status saturn_evaluate(saturn_plan *p, const uint8_t *d_cfg, const uint8_t *d_perm, int64_t n,
                              int32_t *d_makespan, void *stream);

/* Node-gene variant (row f4): d_node device uint8 [n][T] gives each job's node (0xFF = the
 * decoder's greedy choice for that job).  With node genes the decoder space provably
 * contains the SPASE optimum.  A node gene naming a missing node or a
 * node with fewer than g GPUs makes the genome invalid (-1).  EINVAL for cluster shapes
 * without a compiled register decoder. */
saturn_status saturn_evaluate_nodes(saturn_plan *p, const uint8_t *d_cfg, const uint8_t *d_perm,
                                    const uint8_t *d_node, int64_t n, int32_t *d_makespan, void *stream);

/* Same with HOST buffers: copies genomes host->device and makespans device->host inside the
 * call (staged through the handle's device workspace); synchronous. */
saturn_status saturn_evaluate_host(saturn_plan *p, const uint8_t *h_cfg, const uint8_t *h_perm, int64_t n,
                                   int32_t *h_makespan, void *stream);

/* Trace-decode n genomes (row a8) into device placements [n][T] (saturn_placement, job-id
 * order) and device makespans [n].  Invalid genomes: makespan -1, placements unwritten. */
saturn_status saturn_trace(saturn_plan *p, const uint8_t *d_cfg, const uint8_t *d_perm, int64_t n,
                           saturn_placement *d_placements, int32_t *d_makespan, void *stream);

/* Size of the genome space, T! * prod_t S_t, if it is < 2^64 (else ELIMIT). */
saturn_status saturn_space_size(const saturn_plan *p, uint64_t *size);

/* Exhaustive enumeration (row a4-ii + a5 + a6): the minimum makespan over every genome and
 * the smallest genome index attaining it (reading A7).  Genome index G -> genome:
 * r_cfg = G mod prod S, r_perm = G div prod S, cfg[t] = (r_cfg div prod_{t'<t} S_t') mod S_t,
 * perm = lexicographic unrank of r_perm.  With an attached communicator the space is split
 * into `world` contiguous slices and the (makespan << 38 | index) keys are min-all-reduced
 * over NCCL; the result is identical for every world size.  ELIMIT if the space exceeds
 * max_genomes or 2^38, or T > 20.  flags = SATURN_PROVEN_OPTIMAL.  Synchronous. */
saturn_status saturn_enumerate(saturn_plan *p, uint64_t max_genomes, void *stream, saturn_result *out);

/* saturn_enumerate runs a depth-first enumeration with prefix sharing and a strict
 * branch-and-bound cut (incumbent = the best paper-baseline genome) when T >= 3 and the
 * cluster has a register decoder shape (flags |= SATURN_PREFIX_SHARED; `evaluated` = 0: it
 * performs no full T-step decode (SURVEY.md §8d counting rule: prefix-shared leaves are
 * reported separately, pruned plans never); `leaves` = leaves actually visited, each a
 * makespan completed from a shared prefix state; the space covered is saturn_space_size);
 * the result is identical to the index-order brute force (saturn_enumerate_range(0, space)
 * does the full decodes in index order).
 *
 * Symmetry reduction (row f4; reading A14): with
 * SATURN_ENUM_SYMMETRY set, jobs whose compacted config lists are the same (g, R) sequence
 * ("twins", e.g. the same model trained at several learning rates) are
 * placed in increasing job id order only: a genome that places a job before its previous
 * twin is skipped.  Relabelling twins maps every genome onto such a canonical genome with
 * the same makespan, so the minimum is unchanged; the returned index is the smallest
 * CANONICAL genome index attaining it, and the space shrinks by prod_c (k_c!) over twin
 * classes of size k_c.  Applies to the depth-first path only (flags |= SATURN_SYMMETRY_REDUCED
 * when a twin class exists); the odometer and range paths ignore it. */
enum { SATURN_ENUM_SYMMETRY = 1 };
saturn_status saturn_set_enumeration_options(saturn_plan *p, uint32_t options);

/*
 * Enumerate only genome indices [begin, end) on this device (no collective; full decodes). */
saturn_status saturn_enumerate_range(saturn_plan *p, uint64_t begin, uint64_t end, void *stream,
                                     saturn_result *out);

/* Genetic search (rows a4-iii, a5, a6, a7, oracle/ga.py GA v4):
 * an initial population, then max_generations generations of Philox tournament selection,
 * uniform (configs) / LOX (priority permutation) crossover and mutation, every child decoded
 * on the device, the elites carried over.  With an attached communicator or peer link each
 * GPU runs an island and every generations_per_epoch generations the elites of all islands
 * are exchanged and every island continues from the global best E.  Deterministic for fixed
 * (params, world size).  flags = SATURN_INCUMBENT.  Synchronous.  EINVAL for bad params;
 * ESTATE without a table. */
saturn_status saturn_search(saturn_plan *p, const saturn_search_params *sp, void *stream, saturn_result *out);

/* Several islands in one process (row e without NCCL): plans[0..k) -- handles with the same
 * cluster and table, on one or several devices, no communicator -- run saturn_search in
 * lock-step as islands 0..k-1 (the Philox rank id of island r is r) and exchange their
 * elite records every epoch by device-to-device copies (cudaMemcpyPeer), then every island
 * continues from the global best E -- exactly the NCCL island protocol of saturn_search with
 * world = k.  streams: k caller streams or NULL.  out: k results (evaluated = all islands).
 * Synchronous.  EINVAL for mismatched handles, ESTATE for host-only or attached handles. */
saturn_status saturn_search_group(saturn_plan **plans, int32_t k, const saturn_search_params *sp, void **streams,
                                  saturn_result *out);

/* Best-so-far curve of the last search: up to n_max (seconds, makespan) pairs, one per
 * epoch; *n_out = number written.  Seconds are device time since the search's first
 * operation on its stream (events; the epochs are recorded without host round trips). */
saturn_status saturn_search_history(const saturn_plan *p, int64_t n_max, double *t_s, int64_t *makespan,
                                    int64_t *n_out);

/* Best-improvement local search (row f4): each of n genomes
 * (host cfg/perm [n][T], updated in place) repeatedly moves to its best neighbour --
 * insertion moves of the permutation, then single-job config changes, smallest (makespan,
 * move index) -- while that strictly improves its makespan, at most `iters` times; one CTA
 * per genome, every neighbour decoded on the device.  h_makespan [n] receives the results.
 * Invalid genomes: EINVAL.  Synchronous. */
saturn_status saturn_improve(saturn_plan *p, uint8_t *h_cfg, uint8_t *h_perm, int64_t n, int32_t iters,
                             int32_t *h_makespan, void *stream);

/* Final population of the last search on this device: host uint8 cfg [P][T], perm [P][T],
 * int32 makespan [P] (each may be NULL), P = that search's population, returned in *n_out.
 * With every buffer NULL it only reports P.  (Used for operator-replay parity.)
 * EINVAL: capacity < P (the buffers are never written past `capacity` genomes);
 * ESTATE before a search (or after a workspace bind dropped the population). */
saturn_status saturn_search_population(const saturn_plan *p, int64_t capacity, uint8_t *h_cfg, uint8_t *h_perm,
                                       int32_t *h_makespan, int64_t *n_out);

/* Search-state checkpoint / resume (SURVEY.md §5 "Checkpoint / resume": a search is
 * deterministic and restartable from (seed, generation, population); the paper checkpoints
 * jobs at plan switches).  The state of the last search (or resume) on
 * this handle is a flat host byte buffer: a header (magic "SATSRCH1", T, record stride,
 * population P, elites E, island rank / world, seed, generation reached, an FNV-1a hash of
 * the cluster and runtime table, an FNV-1a hash of the payload), then the population
 * records [P][stride], their makespans int32 [P], the elite makespans int32 [E] and the
 * elite records [E][stride].
 *
 * saturn_search_save: with h_state NULL only *bytes_out is set; otherwise the state is
 * written to h_state (caller-owned host memory of `capacity` bytes; EINVAL if too small).
 * ESTATE before a search.  Synchronous.
 *
 * saturn_search_resume: continue a saved search on a handle with the same cluster and
 * runtime table (any handle on any device; EINVAL otherwise): sp->seed, population and
 * elites must equal the saved ones, the state's island / world must equal this handle's
 * rank / world, and every saved genome must be valid (EINVAL otherwise; also for a bad
 * magic, size or checksum; the saved makespans are trusted, not re-decoded).
 * sp->max_generations MORE generations are run, numbered from
 * the saved generation + 1 (their Philox streams and epoch boundaries are those the saved
 * search would have used next); sp->seed_cfg / n_seed are ignored.  For one island without
 * the memetic step, search(G1) + save + resume(G2) returns exactly what search(G1 + G2)
 * returns (final population, elites, best plan).  (With several islands or a memetic step
 * the saved state is taken after the search's final exchange, which the continuous search
 * does not run at generation G1.)  out->generations = generations run by this call.
 * Synchronous. */
saturn_status saturn_search_save(const saturn_plan *p, void *h_state, uint64_t capacity, uint64_t *bytes_out);
saturn_status saturn_search_resume(saturn_plan *p, const void *h_state, uint64_t bytes,
                                   const saturn_search_params *sp, void *stream, saturn_result *out);

/* The best plan of the last enumerate/search (row a8): placements host [T] (job-id order),
 * genome_out host [2T] (cfg then perm) or NULL, makespan.  ESTATE before any search. */
saturn_status saturn_best_plan(saturn_plan *p, saturn_placement *out, uint8_t *genome_out, int64_t *makespan);

/* The paper's baseline heuristics (row f2; Alg. 1 at 949-962) as genomes
 * for the decoder, and as GA seeds: MAX = every job on a full node, MIN = one GPU each plus
 * the surplus dealt round-robin, OPTIMUS = Optimus*-Greedy (Alg. 1, per node), RANDOM = a
 * uniform random genome.  Configs: best runtime at the chosen width (ties to the lower UPP
 * index); order: LPT.  Multi-node job groups are drawn with probability GPU_n / sum GPU
 * (PAPER.md:1002).  Exact rules: DESIGN.md "Baselines" / oracle/baselines.py.  On multi-node
 * clusters the genome alone fixes each job's WIDTH; decoded without node genes the decoder
 * re-picks every node greedily.  The per-node plan the paper's heuristics run is the genome
 * decoded with saturn_baseline_nodes' node genes (saturn_evaluate_nodes; reading A16).
 * cfg, perm: host uint8 [T].  Host-only (works on host-only handles).  ESTATE without a table. */
enum { SATURN_BASELINE_MAX = 1, SATURN_BASELINE_MIN = 2, SATURN_BASELINE_OPTIMUS = 3, SATURN_BASELINE_RANDOM = 4 };
saturn_status saturn_baseline_genome(const saturn_plan *p, int32_t kind, uint64_t seed, uint8_t *cfg, uint8_t *perm);

/* Node genes of a baseline's per-node plan (row f2; "one node at a time", PAPER.md:962,
 * 1002): node host uint8 [T] (job-id order) -- job t's distributed node when the config
 * saturn_baseline_genome(kind, seed) chose for it fits that node, else 0xFF (greedy; only
 * when even its narrowest width exceeds the node); RANDOM: all 0xFF.  Pass with that genome
 * to saturn_evaluate_nodes.  Host-only.  EINVAL for a bad kind, ESTATE without a table. */
saturn_status saturn_baseline_nodes(const saturn_plan *p, int32_t kind, uint64_t seed, uint8_t *node);

/* Round introspection (row f1; PAPER.md:241-262 App. algorithm, §4.4) on
 * the loaded workload W:  S = solve(W), M = makespan(S), time = 0; while M > I: W = W after I
 * seconds of S (residual runtimes, reading A10: a job that ran a s of its config with runtime
 * R0 keeps every config with R' = ceil(R (R0 - a) / R0); finished jobs leave), S = S[I:],
 * M -= I, time += I, apply the round's events, P = solve(W), adopt P iff makespan(P) <= M - T
 * (or unconditionally when a job arrived).  E2E makespan = time + M at the end.
 * solve = saturn_search (SATURN_SOLVER_SEARCH, with `search`) or saturn_enumerate
 * (SATURN_SOLVER_ENUMERATE, exact; tiny workloads).  The loaded table is restored afterwards.
 * Events, applied at round boundaries after the advance:
 * STOP removes job `job` (original id; arrivals are numbered T, T+1, ... in event order) from
 * W and from the current plan (M = the plan's latest end); ARRIVE adds a job with runtime row
 * runtime_s [n_upps][max_gpus] (the table's layout).  Events due after the workload is
 * exhausted never fire; a STOP naming a finished or unknown job is EINVAL.
 * Overlap mode: round k+1's proposal is solved on the SIMULATED
 * next-interval state advance(W, S, I) while round k runs, so the solver latency hides behind
 * the interval (interval_wall_s seconds of real time; 0 = interval_s); an event at that
 * boundary makes it stale and a fresh solve replaces it -- the E2E schedule is identical to
 * the sequential loop's.  round_log (host, may be NULL): per round {time, M after the shift,
 * makespan(P), adopted} as 4 int64.  Synchronous. */
enum { SATURN_SOLVER_SEARCH = 0, SATURN_SOLVER_ENUMERATE = 1 };
enum { SATURN_EVENT_STOP = 1, SATURN_EVENT_ARRIVE = 2 };
typedef struct {
  int32_t at_round;                   /* >= 1: applied at time at_round * I         */
  int32_t kind;                       /* SATURN_EVENT_STOP | SATURN_EVENT_ARRIVE     */
  int32_t job;                        /* STOP: original job id                      */
  int32_t pad;
  const int32_t *runtime_s;           /* ARRIVE: host [n_upps][max_gpus]            */
} saturn_introspect_event;
typedef struct {
  int64_t interval_s;                 /* I (the paper uses 1000 s)   */
  int64_t threshold_s;                /* T (500 s)             */
  int32_t solver;
  int32_t max_rounds;
  const saturn_search_params *search; /* SEARCH: parameters of every round's solve  */
  int32_t overlap;                    /* 1: overlap mode                            */
  int32_t n_events;
  const saturn_introspect_event *events;
  double interval_wall_s;             /* overlap latency accounting; 0 = interval_s */
} saturn_introspect_params;
typedef struct {
  int64_t one_shot_makespan;  /* makespan of the round-0 plan                       */
  int64_t e2e_makespan;       /* time until the workload is exhausted              */
  int32_t rounds;
  int32_t adopted;
  uint64_t evaluated;         /* decodes of all solves                              */
  int32_t stale;              /* overlap mode: proposals discarded because an event fired */
  int32_t solves;             /* solver calls (incl. stale ones)                   */
  double solve_s;             /* wall seconds of the re-solves (rounds >= 1)       */
  double exposed_solve_s;     /* of which on the critical path: sequential = all of it;
                                 overlap = sum max(0, t - interval_wall_s) + fresh
                                 re-solves after events                            */
} saturn_introspect_result;
saturn_status saturn_introspect(saturn_plan *p, const saturn_introspect_params *ip, void *stream,
                                saturn_introspect_result *out, int64_t *round_log);

/* Multi-GPU (row e): rank 0 creates an NCCL unique id (128 bytes), the caller broadcasts it
 * (e.g. torch.distributed), then every rank attaches.  ENCCL if NCCL cannot be loaded. */
saturn_status saturn_get_unique_id(uint8_t *id128);
saturn_status saturn_plan_attach_comm(saturn_plan *p, const uint8_t *id128, int32_t rank, int32_t world);

/* Multi-GPU without NCCL (row e; SURVEY.md §8e "B200-native alternative"): the `world`
 * ranks of one node (one process per GPU) pass the same fresh POSIX shared-memory name
 * ("/saturn_<nonce>", created by rank 0, removed once every rank is attached).  Each rank
 * exports a device exchange buffer with CUDA IPC and maps every peer's; the elite exchange
 * of saturn_search then PUSHES this island's E records into block `rank` of every rank's
 * buffer (device-to-device over NVLink, or within one device), passes a shared-memory
 * barrier and merges its own buffer -- the blocks an NCCL all-gather would produce, so the
 * island protocol and its results are those of saturn_plan_attach_comm / search_group.
 * saturn_enumerate reduces (MIN key, SUM leaves) the same way.  Collective and blocking.
 * Liveness: every rank heartbeats in the shared segment while it waits for its own GPU work
 * and at the barrier; a rank silent for SATURN_PEER_TIMEOUT_S (default 120 s: its process
 * died or hangs outside the library) fails the others with ECUDA instead of hanging -- a
 * rank that is only slow (long enumeration slice) keeps heartbeating and is waited for.
 * A failed barrier poisons the link: every later exchange on it fails fast (ECUDA) on every
 * rank until the handles re-attach.  Host-only handles attach the barrier alone (tests).
 * world <= 8.  ESTATE if the handle already has an NCCL communicator (and vice versa). */
saturn_status saturn_plan_attach_peers(saturn_plan *p, const char *name, int32_t rank, int32_t world);
/* Barrier over the ranks of the peer link (ESTATE without one). */
saturn_status saturn_plan_barrier(saturn_plan *p);

/* Contiguous slice [begin, end) of [0, total) owned by `rank` of `world` (pure host). */
saturn_status saturn_partition(uint64_t total, int32_t rank, int32_t world, uint64_t *begin, uint64_t *end);

/* Integer-ALU throughput probe on the handle's device: independent IMNMX/IADD3/ISETP/SEL
 * chains; *int_ops_per_s = measured integer operations per second (roofline check). */
saturn_status saturn_probe_int_peak(saturn_plan *p, double *int_ops_per_s);

/* Counters since the last reset (measurement support, row d): kernel launches issued by
 * the library, host<->device bytes it copied, and -- when profiling is on -- the summed
 * device time of the GA generation kernels, measured with CUDA events on the launching
 * stream. */
typedef struct {
  int64_t kernel_launches;
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int64_t ga_launches;      /* GA generation kernels timed (profiling on)            */
  double ga_kernel_ms;      /* their summed device time                             */
  int64_t ga_decodes;       /* children decoded by those launches                   */
} saturn_stats;
/* on = 0: off; on = n >= 1: time every n-th GA generation kernel of saturn_search with CUDA
 * events on the launching stream (1 = all; an event record between two kernels costs a few
 * microseconds, so bench.py samples every 4th). */
saturn_status saturn_set_profiling(saturn_plan *p, int32_t on);
saturn_status saturn_get_stats(const saturn_plan *p, saturn_stats *out);
saturn_status saturn_reset_stats(saturn_plan *p);

const char *saturn_last_error(const saturn_plan *p);
void saturn_plan_destroy(saturn_plan *p);

#ifdef __cplusplus
}
#endif
#endif /* SATURN_H */
