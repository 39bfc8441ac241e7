/*
 * examples/saturn_demo.c -- using libsaturn through its C ABI only (no Python, no torch).
 *
 *   gcc -O2 -I include examples/saturn_demo.c -L paper_2309_01226_b200 -lsaturn \
 *       -Wl,-rpath,$PWD/paper_2309_01226_b200 -o examples/saturn_demo
 *   examples/saturn_demo [device]
 *
 * Builds a small two-node workload (6 jobs x {DDP, FSDP} x 1..4 GPUs on 2 x 4 GPUs), prints
 * the paper's Max-Heuristic plan, the exhaustive optimum
 * (saturn_enumerate) and the GA's best plan (saturn_search) with its schedule.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "saturn.h"

#define CHECK(call)                                                                        \
  do {                                                                                     \
    saturn_status s_ = (call);                                                             \
    if (s_ != SATURN_OK) {                                                                 \
      fprintf(stderr, "%s -> %d: %s\n", #call, (int)s_, saturn_last_error(plan));           \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)

enum { T = 6, U = 2, G = 4 };

static void print_plan(const saturn_placement *pl, int64_t makespan) {
  static const char *upp[] = {"DDP", "FSDP"};
  printf("  makespan %lld s\n", (long long)makespan);
  for (int t = 0; t < T; ++t)
    printf("  job %d: node %d GPUs 0x%llx (%d x %s) [%d, %d)\n", t, pl[t].node, (unsigned long long)pl[t].gpu_mask,
           pl[t].gpus, upp[pl[t].upp], pl[t].start_s, pl[t].end_s);
}

int main(int argc, char **argv) {
  const int device = argc > 1 ? atoi(argv[1]) : 0;
  const int32_t nodes[2] = {4, 4};
  saturn_plan *plan = NULL;
  saturn_status st = saturn_plan_create(nodes, 2, device, &plan);
  if (st != SATURN_OK) {
    fprintf(stderr, "saturn_plan_create -> %d (no usable CUDA device?)\n", (int)st);
    return 2;
  }
  /* runtime[t][u][g-1] = W_t (sigma_u + (1 - sigma_u) / g) + c_u (g - 1); 0 = infeasible */
  int32_t runtime[T][U][G];
  const int work[T] = {400, 900, 300, 650, 500, 800};
  for (int t = 0; t < T; ++t)
    for (int u = 0; u < U; ++u)
      for (int g = 1; g <= G; ++g) {
        const double sigma = u == 0 ? 0.03 : 0.06, comm = u == 0 ? 25.0 : 12.0;
        runtime[t][u][g - 1] = (int32_t)(work[t] * (sigma + (1.0 - sigma) / g) + comm * (g - 1) + 0.999);
        if (u == 0 && t % 3 == 1 && g == 1) runtime[t][u][g - 1] = 0; /* an OOM profile */
      }
  CHECK(saturn_load_runtime_table(plan, &runtime[0][0][0], T, U, G));

  saturn_placement pl[T];
  uint8_t cfg[T], perm[T];
  int32_t ms_max = 0;
  CHECK(saturn_baseline_genome(plan, SATURN_BASELINE_MAX, 0, cfg, perm));
  CHECK(saturn_evaluate_host(plan, cfg, perm, 1, &ms_max, NULL));
  printf("Max-Heuristic genome decodes to %d s\n", ms_max);

  saturn_result r;
  CHECK(saturn_enumerate(plan, (uint64_t)1 << 34, NULL, &r));
  int64_t ms = 0;
  uint64_t space = 0;
  CHECK(saturn_best_plan(plan, pl, NULL, &ms));
  CHECK(saturn_space_size(plan, &space));
  printf("exhaustive optimum over %llu genomes (%llu leaves visited, %.3f s):\n", (unsigned long long)space,
         (unsigned long long)r.leaves, r.seconds);
  print_plan(pl, ms);

  saturn_search_params sp = {0};
  sp.seed = 1;
  sp.population = 1 << 16;
  sp.max_generations = 50;
  sp.elites = 8;
  sp.generations_per_epoch = 10;
  sp.p_xover_q32 = 3865470566u;   /* 0.9 */
  sp.p_cfg_mut_q32 = 2147483648u; /* 0.5 */
  sp.p_perm_mut_q32 = 2147483648u;
  CHECK(saturn_search(plan, &sp, NULL, &r));
  CHECK(saturn_best_plan(plan, pl, NULL, &ms));
  printf("GA search: %llu plans in %.3f s (%.2e plans/s):\n", (unsigned long long)r.evaluated, r.seconds,
         r.evaluated / r.seconds);
  print_plan(pl, ms);
  saturn_plan_destroy(plan);
  return 0;
}
