// Host-side launchers for the saturn device kernels (internal to libsaturn; not the C ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace sat {

// Thread-decoder shapes (NN padded nodes x GP padded GPUs per node) compiled into the
// library.  Anything else runs on the warp decoder.
bool have_sorted_shape(int NN, int GP);

// Shared-memory bytes of the evaluate kernel for a given problem and shape.
size_t eval_smem_bytes(const Problem& pb, int NN, int GP);

// saturn_evaluate: one makespan per genome (rows of T bytes).  kind: 1 = thread, 2 = warp.
cudaError_t launch_evaluate(const Problem& pb, int NN, int GP, int kind, const uint8_t* cfg,
                            const uint8_t* perm, int64_t n, int32_t* out, int sms, cudaStream_t st);

// Node-gene decode (row f4): node[n][T], 0xFF = greedy for that job.  Register shapes only.
cudaError_t launch_evaluate_nodes(const Problem& pb, int NN, int GP, const uint8_t* cfg, const uint8_t* perm,
                                  const uint8_t* node, int64_t n, int32_t* out, int sms, cudaStream_t st);

// Trace decode (W design): placements[n][T] (32 B records, job-id order) and makespans.
cudaError_t launch_trace(const Problem& pb, const uint8_t* cfg, const uint8_t* perm, int64_t n,
                         void* placements, int32_t* out, int sms, cudaStream_t st);

// Mixed-radix / factoradic constants of the genome index space.
constexpr int ENUM_MAX_T = 20;
struct EnumSpace {
  uint64_t cfg_space;              // prod_t S_t
  uint64_t radix[ENUM_MAX_T];      // prod_{t' < t} S_t'
  uint64_t fact[ENUM_MAX_T + 1];   // k!
};
// Exhaustive enumeration of genome indices [begin, end): atomicMin of (ms << 38 | index).
cudaError_t launch_enumerate(const Problem& pb, int NN, int GP, const EnumSpace& es, uint64_t begin,
                             uint64_t end, unsigned long long* best_key, int sms, cudaStream_t st);

// Depth-first enumeration with prefix sharing and strict branch-and-bound (a4-ii): roots
// fix the (job, config) choices of the first D priority positions (a mixed-radix index over
// sum_t S_t pairs per level; roots repeating a job are skipped); below a root every prefix
// state is computed once and the last position is evaluated in closed form (g-th smallest
// start + R), so a leaf costs a few instructions instead of a T-step decode.  Leaf indices
// are exact, and only subtrees whose partial makespan exceeds the incumbent are cut, so the
// result is the same (makespan, smallest index) as the index-order brute force.
struct DfsSpace {
  EnumSpace es;
  int pre[ENUM_MAX_T + 1];   // prefix sums of S_t: pair index -> (job, config)
  int sumS;
  int D;                     // root depth
  uint64_t n_roots;          // sumS^D
  uint32_t twin_prev[ENUM_MAX_T];  // bit of job t's previous twin (symmetry reduction), or 0
};
cudaError_t launch_enumerate_dfs(const Problem& pb, int NN, int GP, const DfsSpace& ds, uint64_t root_begin,
                                 uint64_t root_end, unsigned long long* best_key, unsigned long long* leaves,
                                 int sms, cudaStream_t st);

struct GaParams {
  uint64_t seed;
  uint32_t rank;
  uint32_t gen;       // generation being produced (0 = initial population)
  int64_t P;          // population per rank
  int E;              // elites
  int GS;             // genome record stride in bytes (multiple of 16)
  uint32_t px, pc, pm;
};

// Generation 0: seed genomes then Philox-initialised genomes, all decoded.  Each CTA appends
// its top-E keys (ms << 32 | slot) that can still enter the elite set to cand[] and bumps the
// device counter *d_n_cand (zero on entry; k_select resets it).
cudaError_t launch_ga_init(const Problem& pb, int NN, int GP, const GaParams& gp, const uint8_t* seeds,
                           int64_t n_seed, uint8_t* pop, int32_t* ms, unsigned long long* cand, int* d_n_cand,
                           int sms, cudaStream_t st);
// Generation gen >= 1 from the previous population and the elite records.
cudaError_t launch_ga_generation(const Problem& pb, int NN, int GP, const GaParams& gp, const uint8_t* prev_pop,
                                 const int32_t* prev_ms, const int32_t* rec_ms, const uint8_t* rec_gen,
                                 uint8_t* pop, int32_t* ms, unsigned long long* cand, int* d_n_cand, int sms,
                                 cudaStream_t st);
// True when a generation is two kernels (breed, then decode); `mid` is recorded between them.
// Upper bound of the candidates one GA launch can append (grid x E).
int ga_max_candidates(const Problem& pb, int NN, int GP, int E, int GS, int64_t P, int sms);
// Top-E of the *d_n_cand candidate keys -> elite records (ms, genome) copied from `pop`.
cudaError_t launch_select(const unsigned long long* cand, int* d_n_cand, int E, int GS, const uint8_t* pop,
                          int32_t* rec_ms, uint8_t* rec_gen, cudaStream_t st, bool few = false);
// Island migration: the E best of W ranks' gathered records by (ms, rank, position).
cudaError_t launch_merge_elites(const int32_t* all_ms, const uint8_t* all_gen, int W, int E, int GS,
                                int32_t* rec_ms, uint8_t* rec_gen, cudaStream_t st);

// Best-improvement local search (row f4) on n genome records (GS bytes each) in place; ms[]
// holds their makespans on entry and the improved ones on exit.
cudaError_t launch_local_search(const Problem& pb, int NN, int GP, uint8_t* gen, int32_t* ms, int n, int GS, int iters,
                                cudaStream_t st);

// Integer-ALU throughput probe (independent IMNMX/ISETP/IADD3/SEL chains).  Returns the
// number of integer operations one launch performs.
double launch_int_probe(int sms, int* sink, cudaStream_t st);

}  // namespace sat
