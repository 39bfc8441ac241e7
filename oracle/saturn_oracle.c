/*
 * oracle/saturn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the SPASE plan decoder and the
 * brute-force optimum.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2309_01226_b200/), and it never
 * reads anything the CUDA path wrote.
 *
 * What it computes:
 *
 *   O1 or_decode      -- genome (cfg[T], perm[T]) -> schedule and integer makespan.
 *                        The paper has no decoder (its optimizer is a black-box MILP,
 *                        PAPER.md:750, 923); O1 is reading A6: append-only list
 *                        scheduling of jobs in priority order, each job starting at the
 *                        g-th smallest free time of the node with the earliest such start
 *                        (ties -> lowest node id), taking the g latest-free GPUs among those
 *                        free by then (ties -> lower GPU id).  Each job is placed on one
 *                        node with exactly g GPUs and one start time: the MILP's
 *                        Eqs. 3-9; per-GPU free times enforce the task
 *                        isolation of Eqs. 10-11; the makespan is
 *                        Eq. 2, the latest start plus runtime.
 *   O2 or_brute_force -- min over genome indices [begin,end) of O1, first index kept
 *                        (reading A7: the reported plan is the smallest genome index).
 *                        Index G -> genome is the mixed-radix / factoradic unranking of
 *                        SURVEY.md §8a-a4(ii).
 *
 * Integers only (reading A4/A5): runtimes are int32 seconds, half-open intervals.
 * No blocking, no fusion, no clever data structures -- a reader should be able to check
 * every line against the algorithm above.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAX_GPUS 64
#define OR_MAX_JOBS 255

typedef struct {
    int32_t node;      /* O_{t,n}: the node the job runs on                  */
    int32_t upp;       /* filled by the Python side (the oracle keeps no UPP ids) */
    int32_t gpus;      /* G_{t,s}: number of GPUs                            */
    int32_t cfg;       /* index s into the job's compacted config list (B_t) */
    int32_t start_s;   /* I_{t,n,g}: common start time (gang)                */
    int32_t end_s;     /* start + R_{t,s}                                    */
    uint64_t gpu_mask; /* P_{t,n,g}: bit g set <=> job uses GPU g of its node */
} or_placement;

/*
 * O1.  Inputs:
 *   n_nodes, gpu_n[n]         the cluster (Table 1: N, GPU_n)
 *   n_jobs, stride            compacted table: job t, config s has
 *   cg[t*stride+s], cr[...]     G_{t,s} GPUs and runtime R_{t,s}; n_cfg[t] = S_t
 *   cfg[t], perm[p]           the genome
 *   node_gene[t]              NULL -> greedy node choice (O1); else job t must run on
 *                             node node_gene[t], or choose greedily if it is 0xFF
 *                             (node-gene variant: the completeness checks of SURVEY.md
 *                             §8c O2 and row f4)
 *   out[t]                    optional per-job placement record (job-id order)
 * Returns the makespan, or -1 if the genome is invalid (cfg out of range, perm not a
 * permutation, node gene out of range or too small for the config).
 */
int32_t or_decode(int32_t n_nodes, const int32_t *gpu_n, int32_t n_jobs, int32_t stride,
                  const int32_t *cg, const int32_t *cr, const int32_t *n_cfg,
                  const uint8_t *cfg, const uint8_t *perm, const uint8_t *node_gene,
                  or_placement *out)
{
    int32_t free_t[OR_MAX_GPUS];   /* free time of every GPU, node-major */
    int32_t first[OR_MAX_GPUS + 1]; /* first[n] = index of node n's GPU 0 in free_t */
    int seen[OR_MAX_JOBS];
    int32_t makespan = 0;

    if (n_nodes < 1 || n_jobs < 1 || n_jobs > OR_MAX_JOBS) return -1;
    first[0] = 0;
    for (int n = 0; n < n_nodes; ++n) first[n + 1] = first[n] + gpu_n[n];
    if (first[n_nodes] > OR_MAX_GPUS) return -1;
    for (int i = 0; i < first[n_nodes]; ++i) free_t[i] = 0;

    /* genome validity: perm is a permutation, every cfg gene in range */
    for (int t = 0; t < n_jobs; ++t) seen[t] = 0;
    for (int p = 0; p < n_jobs; ++p) {
        if (perm[p] >= n_jobs || seen[perm[p]]) return -1;
        seen[perm[p]] = 1;
    }
    for (int t = 0; t < n_jobs; ++t)
        if (cfg[t] >= n_cfg[t]) return -1;

    for (int p = 0; p < n_jobs; ++p) {
        int t = perm[p];
        int32_t g = cg[t * stride + cfg[t]];
        int32_t r = cr[t * stride + cfg[t]];

        /* start_n = g-th smallest free time on node n, for every node that fits g */
        int best_n = -1;
        int32_t best_s = 0;
        for (int n = 0; n < n_nodes; ++n) {
            if (gpu_n[n] < g) continue;
            if (node_gene && node_gene[t] != 0xFF && node_gene[t] != n) continue;
            int32_t sorted_free[OR_MAX_GPUS];
            int k = gpu_n[n];
            for (int i = 0; i < k; ++i) sorted_free[i] = free_t[first[n] + i];
            /* insertion sort, ascending */
            for (int i = 1; i < k; ++i) {
                int32_t x = sorted_free[i];
                int j = i - 1;
                while (j >= 0 && sorted_free[j] > x) { sorted_free[j + 1] = sorted_free[j]; --j; }
                sorted_free[j + 1] = x;
            }
            int32_t start_n = sorted_free[g - 1];
            /* earliest start; strict '<' keeps the lowest node id on ties */
            if (best_n < 0 || start_n < best_s) { best_n = n; best_s = start_n; }
        }
        if (best_n < 0) return -1;   /* no node can host g GPUs (or bad node gene) */

        /* choose g GPUs among those free by s: latest free time first, then lower id */
        int32_t s = best_s;
        int chosen[OR_MAX_GPUS];
        uint64_t mask = 0;
        for (int i = 0; i < gpu_n[best_n]; ++i) chosen[i] = 0;
        for (int k = 0; k < g; ++k) {
            int pick = -1;
            for (int i = 0; i < gpu_n[best_n]; ++i) {
                int32_t f = free_t[first[best_n] + i];
                if (chosen[i] || f > s) continue;
                if (pick < 0 || f > free_t[first[best_n] + pick]) pick = i;  /* '>' keeps lower id on ties */
            }
            if (pick < 0) return -1;  /* cannot happen: at least g GPUs are free by s */
            chosen[pick] = 1;
            mask |= (uint64_t)1 << pick;
        }
        for (int i = 0; i < gpu_n[best_n]; ++i)
            if (chosen[i]) free_t[first[best_n] + i] = s + r;

        if (s + r > makespan) makespan = s + r;
        if (out) {
            out[t].node = best_n;
            out[t].upp = -1;
            out[t].gpus = g;
            out[t].cfg = cfg[t];
            out[t].start_s = s;
            out[t].end_s = s + r;
            out[t].gpu_mask = mask;
        }
    }
    return makespan;
}

/* O1 over n genomes stored row by row: cfg[i*n_jobs + t], perm[i*n_jobs + p]. */
void or_decode_batch(int32_t n_nodes, const int32_t *gpu_n, int32_t n_jobs, int32_t stride,
                     const int32_t *cg, const int32_t *cr, const int32_t *n_cfg,
                     int64_t n, const uint8_t *cfg, const uint8_t *perm, int32_t *makespan)
{
    for (int64_t i = 0; i < n; ++i)
        makespan[i] = or_decode(n_nodes, gpu_n, n_jobs, stride, cg, cr, n_cfg,
                                cfg + i * n_jobs, perm + i * n_jobs, NULL, NULL);
}

/* O1 with node genes over n genomes: node[i*n_jobs + t] (0xFF = greedy for that job). */
void or_decode_batch_nodes(int32_t n_nodes, const int32_t *gpu_n, int32_t n_jobs, int32_t stride,
                           const int32_t *cg, const int32_t *cr, const int32_t *n_cfg,
                           int64_t n, const uint8_t *cfg, const uint8_t *perm, const uint8_t *node,
                           int32_t *makespan)
{
    for (int64_t i = 0; i < n; ++i)
        makespan[i] = or_decode(n_nodes, gpu_n, n_jobs, stride, cg, cr, n_cfg,
                                cfg + i * n_jobs, perm + i * n_jobs, node + i * n_jobs, NULL);
}

/*
 * Genome index -> genome:
 *   r_cfg = G mod prod_t S_t,  r_perm = G div prod_t S_t
 *   cfg[t] = (r_cfg div prod_{t'<t} S_t') mod S_t       (job 0 least significant)
 *   perm  = lexicographic unrank of r_perm               (perm[0] most significant)
 * Returns 0 on success, -1 if G is outside [0, T! * prod S).
 */
int or_unrank(int32_t n_jobs, const int32_t *n_cfg, uint64_t index, uint8_t *cfg, uint8_t *perm)
{
    unsigned __int128 cfg_space = 1, fact = 1;
    for (int t = 0; t < n_jobs; ++t) cfg_space *= (unsigned)n_cfg[t];
    for (int k = 2; k <= n_jobs; ++k) fact *= (unsigned)k;
    if ((unsigned __int128)index >= cfg_space * fact) return -1;

    uint64_t r_cfg = (uint64_t)((unsigned __int128)index % cfg_space);
    uint64_t r_perm = (uint64_t)((unsigned __int128)index / cfg_space);
    for (int t = 0; t < n_jobs; ++t) {
        cfg[t] = (uint8_t)(r_cfg % (uint64_t)n_cfg[t]);
        r_cfg /= (uint64_t)n_cfg[t];
    }
    int avail[OR_MAX_JOBS];
    int n_avail = n_jobs;
    for (int t = 0; t < n_jobs; ++t) avail[t] = t;
    for (int p = 0; p < n_jobs; ++p) {
        uint64_t f = 1;                     /* (T-1-p)! */
        for (int k = 2; k <= n_jobs - 1 - p; ++k) f *= (uint64_t)k;
        uint64_t idx = r_perm / f;
        r_perm %= f;
        perm[p] = (uint8_t)avail[idx];
        for (int j = (int)idx; j < n_avail - 1; ++j) avail[j] = avail[j + 1];
        --n_avail;
    }
    return 0;
}

/*
 * O2: the minimum of O1 over genome indices [begin, end), in index order, keeping the
 * first index that attains it.  Returns the minimum makespan (or -1 on an empty range /
 * invalid genome) and writes its index to *best_index.
 */
int32_t or_brute_force(int32_t n_nodes, const int32_t *gpu_n, int32_t n_jobs, int32_t stride,
                       const int32_t *cg, const int32_t *cr, const int32_t *n_cfg,
                       uint64_t begin, uint64_t end, uint64_t *best_index)
{
    uint8_t cfg[OR_MAX_JOBS], perm[OR_MAX_JOBS];
    int32_t best = -1;
    for (uint64_t G = begin; G < end; ++G) {
        if (or_unrank(n_jobs, n_cfg, G, cfg, perm) != 0) return -1;
        int32_t ms = or_decode(n_nodes, gpu_n, n_jobs, stride, cg, cr, n_cfg, cfg, perm, NULL, NULL);
        if (ms < 0) return -1;
        if (best < 0 || ms < best) { best = ms; *best_index = G; }
    }
    return best;
}
