// saturn device kernels for sm_100a: evaluate (K1), trace (K6), enumerate (K2),
// GA init/generation (K3 fused with K1), top-E select and elite merge (K4), and the
// integer-ALU probe used as the roofline denominator check.
//
// Every kernel stages the problem blob (packed config table + S_t + UPP ids, <= 48 KB)
// into shared memory once per persistent CTA with a 1-D TMA bulk copy (row a3).
#include <algorithm>
#include <climits>
#include <mutex>
#include <utility>
#include <vector>
#include <cstdlib>
#include <cstdio>

#include "decode.cuh"
#include "kernels.h"

namespace sat {

#ifndef SAT_EVAL_B
#define SAT_EVAL_B 128
#endif
constexpr int EVAL_B = SAT_EVAL_B;  // threads of the evaluate kernel
constexpr int EVAL_TILE = EVAL_B;  // genomes per tile (one per thread; 2 per thread measured no gain, r1)
constexpr int ENUM_B = 128;
constexpr int GA_B = 128;
constexpr int WARP_B = 128;

// ------------------------------------------------------------------ shapes
// (NN, GP): NN nodes (NN == 0: a run-time node count) of GP GPUs (padded to a power of two).
// One node keeps its sorted vector in registers (decode_sorted); several nodes keep theirs in
// shared memory (decode_col).
#define SAT_SHAPES(X) \
  X(1, 2) X(1, 4) X(1, 8) X(1, 16) X(1, 32) X(2, 2) X(2, 4) X(2, 8) X(4, 2) X(4, 4) X(4, 8) \
  X(0, 4) X(0, 8) X(0, 16) X(0, 32)

// Node-state design per kernel (measured r2 on one B200):
//  * registers (decode_sorted: sorted vectors in registers, barrel shift by select stages,
//    multi-node gather/scatter selects), or
//  * columns (decode_col: states in shared memory, one row per slot, shifted reads).
// Evaluate-type kernels (evaluate, index-order enumeration, local search) decode with the
// column states on every shape: TXT +10 %, MIX 2x8 +33 %, SWEEP 4x8 +34 % plans/s over the
// best register / row-layout shared-memory design -- except small single nodes (TINY 1x4,
// T = 3: registers 1.44e11 vs columns 1.30e11; the column init costs more than 1-2 steps
// save).  The GA kernel also holds a child row,
// Philox state and the tournament prefetch: there columns win on 16-slot states (MIX k_ga
// -4 %) but lose on one node (TXT +5.5 %) and on 32-slot states (SWEEP +37 %: 30 KB more
// shared memory per CTA, 3 instead of 4 CTAs per SM).  NN == 0 (run-time node count) is
// columns only.
// Modes: 0 registers, 1 columns with shifted reads, 2 columns with the shift in registers.
enum { ST_REG = 0, ST_COL = 1, ST_COLR = 2 };
__host__ __device__ __forceinline__ constexpr int eval_mode(int NN, int GP) {
  return NN == 1 ? (GP >= 8 ? ST_COL : ST_REG) : ST_COLR;
}
#ifndef SAT_GA_COL_MAX
#define SAT_GA_COL_MAX 16   // largest NN * GP the GA kernel decodes with column states
#endif
__host__ __device__ __forceinline__ constexpr bool ga_col(int NN, int GP) {
  return NN == 0 || (NN >= 2 && NN * GP <= SAT_GA_COL_MAX);
}
// Shared-memory bytes of the column node states for a block of B threads (0: registers).
__host__ __device__ __forceinline__ constexpr int ga_mode(int NN, int GP) { return ga_col(NN, GP) ? ST_COL : ST_REG; }
__host__ __device__ __forceinline__ size_t ns_bytes(const Problem& pb, int mode, int NN, int GP, int B) {
  return mode != ST_REG ? col_state_bytes(NN ? NN : pb.N, GP, B, mode == ST_COLR) : 0;
}

// Decode one genome with the (NN, GP) design; `ns` = this thread's node-state slice (NN == 0).
// STATE_MS: allow reading the makespan off the final state for one full node (decode_sorted);
// only the evaluate kernel uses it -- in k_ga the extra loop copy measured 3 % slower.
// COL: column states, `ns` = &state[threadIdx.x] of a block of B threads; else registers.
template <int NN, int GP, int B, int MODE, int CHECK, bool STATE_MS = false, class G>
__device__ __forceinline__ int decode_T(const uint32_t* tab, const uint8_t* S, int stride, const G& gen, int T,
                                        const Problem& pb, int* ns, uint32_t* mask = nullptr, int mstride = 0) {
  static_assert(MODE != ST_REG || NN >= 1, "a run-time node count needs the column states");
  if constexpr (MODE != ST_REG) return decode_col<NN, GP, B, MODE == ST_COLR, CHECK>(tab, S, stride, gen, T, pb, ns, mask, mstride);
  else if constexpr (STATE_MS) return decode_sorted<NN, GP, CHECK>(tab, S, stride, gen, T, pb, mask, mstride);
  else return decode_sorted_impl<NN, GP, CHECK, true>(tab, S, stride, gen, T, pb, mask, mstride);
}

bool have_sorted_shape(int NN, int GP) {
#define SAT_HAVE(a, b) if (NN == a && GP == b) return true;
  SAT_SHAPES(SAT_HAVE)
#undef SAT_HAVE
  return false;
}


// ------------------------------------------------------------------ warp-level top-E list
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_up_u64(uint64_t v, int d) {
  uint32_t lo = __shfl_up_sync(0xffffffffu, (uint32_t)v, d);
  uint32_t hi = __shfl_up_sync(0xffffffffu, (uint32_t)(v >> 32), d);
  return ((uint64_t)hi << 32) | lo;
}
// `lst` is a warp-distributed ascending list (lane k = k-th smallest key seen); insert
// each lane's `key` if it beats the E-th entry.  Keys are unique.
__device__ __forceinline__ void topE_insert(uint64_t& lst, uint64_t key, int E, uint64_t cap = ~0ull) {
  const int lane = threadIdx.x & 31;
  uint64_t thr = shfl_u64(lst, E - 1);
  uint32_t cm = __ballot_sync(0xffffffffu, key < thr && key <= cap);
  while (cm) {
    const int src = __ffs(cm) - 1;
    cm &= cm - 1;
    const uint64_t k = shfl_u64(key, src);
    thr = shfl_u64(lst, E - 1);
    if (k < thr) {
      const int pos = __popc(__ballot_sync(0xffffffffu, lst < k));
      const uint64_t up = shfl_up_u64(lst, 1);
      if (lane > pos) lst = up;
      else if (lane == pos) lst = k;
    }
  }
}

// ------------------------------------------------------------------ K1: evaluate (T design)
// Genome tiles are double-buffered (TMA of tile i+1 behind the decode of tile i) while two
// buffers stay small; long genomes (SWEEP, T = 100: 51 KB) use one buffer, so that more CTAs
// fit per SM (the decode needs warps more than it needs the copy overlap).
#ifndef SAT_EVAL_DB_LIMIT
#define SAT_EVAL_DB_LIMIT 16384
#endif
__host__ __device__ __forceinline__ int eval_nbuf(int T) { return 4 * EVAL_TILE * T <= SAT_EVAL_DB_LIMIT ? 2 : 1; }
size_t eval_smem_bytes(const Problem& pb, int NN, int GP) {
  return (size_t)pb.blob_bytes + ns_bytes(pb, eval_mode(NN, GP), NN, GP, EVAL_B) + 2u * eval_nbuf(pb.T) * EVAL_TILE * pb.T +
         4u * EVAL_B * ((pb.T + 31) / 32) + 3 * 8;
}

template <int NN, int GP>
__global__ void __launch_bounds__(EVAL_B) k_evaluate(Problem pb, const uint8_t* __restrict__ gcfg,
                                                     const uint8_t* __restrict__ gperm, int64_t n,
                                                     int32_t* __restrict__ out, int use_bulk) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int T = pb.T;
  const int tileB = EVAL_TILE * T;  // bytes per array per tile (multiple of 16)
  uint8_t* s_blob = sm;
  int* s_ns = reinterpret_cast<int*>(sm + pb.blob_bytes);
  const int nbuf = eval_nbuf(T);
  uint8_t* s_g = sm + pb.blob_bytes + ns_bytes(pb, eval_mode(NN, GP), NN, GP, EVAL_B);   // [nbuf buffers][cfg | perm]
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(s_g + 2 * nbuf * tileB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_mask + EVAL_B * ((T + 31) / 32));
  const int64_t ntiles = (n + EVAL_TILE - 1) / EVAL_TILE;
  const int tid = threadIdx.x;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    fence_mbar_init();
    mbar_expect_tx(&bars[2], pb.blob_bytes);
    bulk_g2s(s_blob, pb.blob, pb.blob_bytes, &bars[2]);
    const int64_t tile = blockIdx.x;
    if (use_bulk && tile < ntiles && (tile + 1) * EVAL_TILE <= n) {
      mbar_expect_tx(&bars[0], 2 * tileB);
      bulk_g2s(s_g, gcfg + tile * tileB, tileB, &bars[0]);
      bulk_g2s(s_g + tileB, gperm + tile * tileB, tileB, &bars[0]);
    }
  }
  __syncthreads();
  mbar_wait(&bars[2], 0);
  const uint32_t* tab = tab_of(s_blob);
  const uint8_t* S = S_of(s_blob, pb);

  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int buf = (nbuf == 2) ? (it & 1) : 0;
    uint8_t* bc = s_g + buf * 2 * tileB;
    uint8_t* bp = bc + tileB;
    const int64_t first = tile * EVAL_TILE;
    const bool full = use_bulk && first + EVAL_TILE <= n;
    if (full) {
      mbar_wait(&bars[buf], (nbuf == 2 ? (it >> 1) : it) & 1);
    } else {  // ragged last tile (or unaligned caller buffers): plain cooperative loads
      const int cnt = (int)min((int64_t)EVAL_TILE, n - first) * T;
      for (int k = tid; k < cnt; k += EVAL_B) {
        bc[k] = gcfg[first * T + k];
        bp[k] = gperm[first * T + k];
      }
      __syncthreads();
    }
    if (nbuf == 2 && tid == 0) {  // prefetch the next tile into the other buffer
      const int64_t nt = tile + gridDim.x;
      if (use_bulk && nt < ntiles && (nt + 1) * EVAL_TILE <= n) {
        uint8_t* nc = s_g + (buf ^ 1) * 2 * tileB;
        fence_proxy_async();
        mbar_expect_tx(&bars[buf ^ 1], 2 * tileB);
        bulk_g2s(nc, gcfg + nt * tileB, tileB, &bars[buf ^ 1]);
        bulk_g2s(nc + tileB, gperm + nt * tileB, tileB, &bars[buf ^ 1]);
      }
    }
    if (first + tid < n) {
      RowGenome gen{bc + tid * T, bp + tid * T};
      int* ns = s_ns + tid;
      out[first + tid] = (T <= 32) ? decode_T<NN, GP, EVAL_B, eval_mode(NN, GP), 1, true>(tab, S, pb.stride, gen, T, pb, ns)
                                   : decode_T<NN, GP, EVAL_B, eval_mode(NN, GP), 2, true>(tab, S, pb.stride, gen, T, pb, ns, s_mask + tid, EVAL_B);
    }
    __syncthreads();
    if (nbuf == 1 && tid == 0) {  // one buffer: the next tile's copy starts once it is free
      const int64_t nt = tile + gridDim.x;
      if (use_bulk && nt < ntiles && (nt + 1) * EVAL_TILE <= n) {
        fence_proxy_async();
        mbar_expect_tx(&bars[0], 2 * tileB);
        bulk_g2s(s_g, gcfg + nt * tileB, tileB, &bars[0]);
        bulk_g2s(s_g + tileB, gperm + nt * tileB, tileB, &bars[0]);
      }
    }
  }
}

// ------------------------------------------------------------------ K1-W / K6: warp decoder
static size_t warp_smem_bytes(const Problem& pb) {
  return (size_t)pb.blob_bytes + 4 * MAX_NODES + 4 * (WARP_B / 32) * 32 * 8 + 8;
}

template <bool TRACE>
__global__ void __launch_bounds__(WARP_B) k_eval_warp(Problem pb, const uint8_t* __restrict__ gcfg,
                                                      const uint8_t* __restrict__ gperm, int64_t n,
                                                      int32_t* __restrict__ out, Placement* __restrict__ rec) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint8_t* s_blob = sm;
  int* s_first = reinterpret_cast<int*>(sm + pb.blob_bytes);
  uint32_t* s_bits = reinterpret_cast<uint32_t*>(s_first + MAX_NODES);
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_bits + (WARP_B / 32) * 32 * 8);
  stage_problem(s_blob, pb, bar);
  const uint32_t* tab = tab_of(s_blob);
  const uint8_t* S = S_of(s_blob, pb);
  const uint8_t* G = G_of(S, pb);
  const uint8_t* upp = G + pb.N;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < pb.N; ++k) { s_first[k] = acc; acc += G[k]; }
  }
  __syncthreads();
  const int T = pb.T;
  const WarpLane L = warp_lane(pb, G);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gpw = 32 / L.seg;
  const int64_t wg = (int64_t)blockIdx.x * (WARP_B / 32) + warp;
  const int64_t wtot = (int64_t)gridDim.x * (WARP_B / 32);
  uint32_t* bits = s_bits + warp * 32 * 8 + (L.base / L.seg) * 8;

  for (int64_t base = wg * gpw; base < n; base += wtot * gpw) {
    const int64_t gi = base + lane / L.seg;
    const bool live = gi < n;
    const uint8_t* c = gcfg + (live ? gi : 0) * T;
    const uint8_t* p = gperm + (live ? gi : 0) * T;
    // genome validity, lanes of the segment cooperate
    for (int w = L.q; w < 8; w += L.seg) bits[w] = 0u;
    __syncwarp();
    bool bad = false;
    if (live) {
      for (int i = L.q; i < T; i += L.seg) {
        const int t = p[i];
        if (t >= T) { bad = true; continue; }
        const uint32_t bit = 1u << (t & 31);
        if (atomicOr(&bits[t >> 5], bit) & bit) bad = true;
        if (c[t] >= S[t]) bad = true;
      }
    }
    const bool segbad = (__ballot_sync(0xffffffffu, bad) & L.smask) != 0u;
    __syncwarp();
    const int ms = decode_warp(tab, pb.stride, c, p, T, L, live && !segbad, s_first, upp,
                               TRACE ? rec + (live ? gi : 0) * T : nullptr);
    if (live && L.q == 0) out[gi] = segbad ? -1 : ms;
  }
}

// ------------------------------------------------------------------ launch helpers
// Persistent grid = SMs x resident CTAs for (kernel, block, dynamic smem).  The attribute
// call and occupancy query cost ~10 us of host time, so results are cached per
// (kernel, threads, smem, device) -- a search launches two kernels per generation.
struct GridKey {
  const void* fn;
  int threads;
  size_t smem;
  int device;
  bool operator==(const GridKey& o) const {
    return fn == o.fn && threads == o.threads && smem == o.smem && device == o.device;
  }
};
static std::mutex g_grid_mu;
static std::vector<std::pair<GridKey, int>> g_grid_cache;

template <class K>
static int grid_for(K kernel, int threads, size_t smem, int sms, int64_t work_blocks) {
  int dev = 0;
  cudaGetDevice(&dev);
  const GridKey key{reinterpret_cast<const void*>(kernel), threads, smem, dev};
  int occ = -1;
  {
    std::lock_guard<std::mutex> lk(g_grid_mu);
    for (const auto& e : g_grid_cache)
      if (e.first == key) { occ = e.second; break; }
  }
  if (occ < 0) {
    // The attribute is per function: always allow the opt-in maximum (227 KB on B200), so a
    // later launch of the same kernel with a larger table never trips over a smaller value
    // set for an earlier one.  Occupancy is still computed for this launch's smem.
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kernel);
    const int max_dyn = optin - (int)fa.sharedSizeBytes;   // dynamic + static <= opt-in maximum
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             max_dyn > (int)smem ? max_dyn : (int)smem) != cudaSuccess)
      cudaGetLastError();  // leave no sticky error behind; the launch reports real problems
    occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    if (occ < 1) occ = 1;
    std::lock_guard<std::mutex> lk(g_grid_mu);
    g_grid_cache.push_back({key, occ});
  }
  int64_t g = (int64_t)sms * occ;
  if (work_blocks < g) g = work_blocks;
  return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_evaluate(const Problem& pb, int NN, int GP, int kind, const uint8_t* cfg, const uint8_t* perm,
                            int64_t n, int32_t* out, int sms, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (kind == 1) {
    const size_t smem = eval_smem_bytes(pb, NN, GP);
    const int use_bulk = ((((uintptr_t)cfg) | ((uintptr_t)perm)) & 15u) == 0;
    const int64_t ntiles = (n + EVAL_TILE - 1) / EVAL_TILE;
#define SAT_EVAL(a, b)                                                                   \
  if (NN == a && GP == b) {                                                              \
    const int g = grid_for(k_evaluate<a, b>, EVAL_B, smem, sms, ntiles);                 \
    k_evaluate<a, b><<<g, EVAL_B, smem, st>>>(pb, cfg, perm, n, out, use_bulk);          \
    return cudaGetLastError();                                                           \
  }
    SAT_SHAPES(SAT_EVAL)
#undef SAT_EVAL
    return cudaErrorInvalidConfiguration;
  }
  Problem pw = pb;               // the warp decoder stages the UPP ids too
  pw.blob_bytes = pb.full_bytes;
  const size_t smem = warp_smem_bytes(pw);
  int seg = 1;
  while (seg < pb.sumG) seg <<= 1;
  const int64_t per_block = (int64_t)(WARP_B / 32) * (32 / seg);
  const int g = grid_for(k_eval_warp<false>, WARP_B, smem, sms, (n + per_block - 1) / per_block);
  k_eval_warp<false><<<g, WARP_B, smem, st>>>(pw, cfg, perm, n, out, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_trace(const Problem& pb, const uint8_t* cfg, const uint8_t* perm, int64_t n, void* placements,
                         int32_t* out, int sms, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  Problem pw = pb;               // the trace reads the UPP ids
  pw.blob_bytes = pb.full_bytes;
  const size_t smem = warp_smem_bytes(pw);
  int seg = 1;
  while (seg < pb.sumG) seg <<= 1;
  const int64_t per_block = (int64_t)(WARP_B / 32) * (32 / seg);
  const int g = grid_for(k_eval_warp<true>, WARP_B, smem, sms, (n + per_block - 1) / per_block);
  k_eval_warp<true><<<g, WARP_B, smem, st>>>(pw, cfg, perm, n, out, static_cast<Placement*>(placements));
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K1 with node genes (f4)
constexpr int EVN_B = 128;
template <int NN, int GP>
__global__ void __launch_bounds__(EVN_B) k_evaluate_nodes(Problem pb, const uint8_t* __restrict__ gcfg,
                                                          const uint8_t* __restrict__ gperm,
                                                          const uint8_t* __restrict__ gnode, int64_t n,
                                                          int32_t* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint8_t* s_blob = sm;
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(sm + pb.blob_bytes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_mask + EVN_B * 8);
  stage_problem(s_blob, pb, bar);
  const uint32_t* tab = tab_of(s_blob);
  const int T = pb.T;
  for (int64_t i = (int64_t)blockIdx.x * EVN_B + threadIdx.x; i < n; i += (int64_t)gridDim.x * EVN_B)
    out[i] = decode_sorted_nodes<NN, GP>(tab, G_of(S_of(s_blob, pb), pb), pb.stride, gcfg + i * T, gperm + i * T, gnode + i * T, T, pb,
                                         s_mask + threadIdx.x, EVN_B);
}

cudaError_t launch_evaluate_nodes(const Problem& pb, int NN, int GP, const uint8_t* cfg, const uint8_t* perm,
                                  const uint8_t* node, int64_t n, int32_t* out, int sms, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = (size_t)pb.blob_bytes + 4 * 8 * EVN_B + 8;
  const int64_t blocks = (n + EVN_B - 1) / EVN_B;
#define SAT_EVN(a, b)                                                                 \
  if (NN == a && GP == b && a >= 1) {                                                 \
    const int g = grid_for(k_evaluate_nodes<(a >= 1 ? a : 1), b>, EVN_B, smem, sms, blocks); \
    k_evaluate_nodes<(a >= 1 ? a : 1), b><<<g, EVN_B, smem, st>>>(pb, cfg, perm, node, n, out); \
    return cudaGetLastError();                                                        \
  }
  SAT_SHAPES(SAT_EVN)
#undef SAT_EVN
  return cudaErrorInvalidConfiguration;
}

// ------------------------------------------------------------------ K2: enumerate
// Genome index G -> (cfg, perm): r_cfg = G mod prod S, r_perm = G div prod S,
// cfg[t] = (r_cfg div radix[t]) mod S_t, perm = lexicographic unrank of r_perm.
// Consecutive indices advance cfg like an odometer (job 0 fastest), then perm by
// next_permutation, so only the first index of a chunk is unranked.
static size_t enum_smem_bytes(const Problem& pb, int NN, int GP) {
  return (size_t)pb.blob_bytes + ns_bytes(pb, eval_mode(NN, GP), NN, GP, ENUM_B) + (size_t)ENUM_B * odd_row_stride(perm_offset(pb.T) + pb.T) +
         32 * 8 + 8;
}

template <int NN, int GP>
__global__ void __launch_bounds__(ENUM_B) k_enumerate(Problem pb, EnumSpace es, uint64_t begin, uint64_t end,
                                                      uint64_t chunk, unsigned long long* best_key) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint8_t* s_blob = sm;
  int* s_ns = reinterpret_cast<int*>(sm + pb.blob_bytes);
  uint8_t* s_gen = sm + pb.blob_bytes + ns_bytes(pb, eval_mode(NN, GP), NN, GP, ENUM_B);
  const int T = pb.T;
  const int RS = odd_row_stride(perm_offset(T) + T);
  uint64_t* s_red = reinterpret_cast<uint64_t*>(s_gen + ((ENUM_B * RS + 7) & ~7));
  uint64_t* bar = s_red + 32;
  stage_problem(s_blob, pb, bar);
  const uint32_t* tab = tab_of(s_blob);
  const uint8_t* S = S_of(s_blob, pb);
  RowG gen{s_gen + RS * threadIdx.x, perm_offset(T)};

  uint64_t best = ~0ull;
  const uint64_t total = end - begin;
  const uint64_t nchunks = (total + chunk - 1) / chunk;
  const uint64_t gt = (uint64_t)blockIdx.x * ENUM_B + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * ENUM_B;
  for (uint64_t ch = gt; ch < nchunks; ch += nthr) {
    const uint64_t i0 = begin + ch * chunk;
    const uint64_t i1 = min(i0 + chunk, end);
    // unrank i0
    uint64_t r_cfg = i0 % es.cfg_space;
    uint64_t r_perm = i0 / es.cfg_space;
    for (int t = 0; t < T; ++t) gen.c(t) = (uint8_t)((r_cfg / es.radix[t]) % (uint64_t)S[t]);
    uint32_t avail = (T == 32) ? 0xffffffffu : ((1u << T) - 1u);
    for (int p = 0; p < T; ++p) {
      const uint64_t f = es.fact[T - 1 - p];
      int d = (int)(r_perm / f);
      r_perm %= f;
      uint32_t m = avail;
      for (int k = 0; k < d; ++k) m &= m - 1;
      const int x = __ffs(m) - 1;
      avail &= ~(1u << x);
      gen.q(p) = (uint8_t)x;
    }
    for (uint64_t idx = i0; idx < i1; ++idx) {
      const int ms = decode_T<NN, GP, ENUM_B, eval_mode(NN, GP), 0>(tab, S, pb.stride, gen, T, pb,
                                         s_ns + threadIdx.x);
      const uint64_t key = ((uint64_t)ms << 38) | idx;
      best = key < best ? key : best;
      // odometer over cfg (job 0 least significant), carry into perm
      int t = 0;
      for (; t < T; ++t) {
        const int c = gen.c(t) + 1;
        if (c < S[t]) { gen.c(t) = (uint8_t)c; break; }
        gen.c(t) = 0;
      }
      if (t == T) {  // next lexicographic permutation of perm
        int k = T - 2;
        while (k >= 0 && gen.q(k) >= gen.q(k + 1)) --k;
        if (k >= 0) {
          int l = T - 1;
          while (gen.q(l) <= gen.q(k)) --l;
          uint8_t tmp = gen.q(k); gen.q(k) = gen.q(l); gen.q(l) = tmp;
          for (int a = k + 1, b = T - 1; a < b; ++a, --b) {
            tmp = gen.q(a); gen.q(a) = gen.q(b); gen.q(b) = tmp;
          }
        }
      }
    }
  }
  best = warp_min_u64(best);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) s_red[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t b = s_red[0];
    for (int w = 1; w < ENUM_B / 32; ++w) b = s_red[w] < b ? s_red[w] : b;
    if (b != ~0ull) atomicMin(best_key, (unsigned long long)b);
  }
}

cudaError_t launch_enumerate(const Problem& pb, int NN, int GP, const EnumSpace& es, uint64_t begin, uint64_t end,
                             unsigned long long* best_key, int sms, cudaStream_t st) {
  if (end <= begin) return cudaSuccess;
  const size_t smem = enum_smem_bytes(pb, NN, GP);
  const uint64_t total = end - begin;
#define SAT_ENUM(a, b)                                                                           \
  if (NN == a && GP == b) {                                                                      \
    const int g0 = grid_for(k_enumerate<a, b>, ENUM_B, smem, sms, 1 << 30);                      \
    const uint64_t thr = (uint64_t)g0 * ENUM_B;                                                  \
    uint64_t chunk = (total + thr - 1) / thr;                                                    \
    if (chunk > 4096) chunk = 4096;                                                              \
    if (chunk < 1) chunk = 1;                                                                    \
    const uint64_t nch = (total + chunk - 1) / chunk;                                            \
    int64_t blocks = (int64_t)((nch + ENUM_B - 1) / ENUM_B);                                     \
    const int g = (int)(blocks < g0 ? blocks : g0);                                              \
    k_enumerate<a, b><<<g, ENUM_B, smem, st>>>(pb, es, begin, end, chunk, best_key);             \
    return cudaGetLastError();                                                                   \
  }
  SAT_SHAPES(SAT_ENUM)
#undef SAT_ENUM
  return cudaErrorInvalidConfiguration;
}

// ------------------------------------------------------------------ K2b: DFS enumeration
constexpr int DFS_B = 64;
// per-level thread-private words: state (NN*GP), ms, rperm lo/hi, rcfg lo/hi, used, t, c
template <int NN, int GP>
struct DfsLayout {
  static constexpr int W = NN * GP + 8;
};

static size_t dfs_smem_bytes(const Problem& pb, int NN, int GP) {
  return (size_t)pb.blob_bytes + (size_t)4 * pb.T * (NN * GP + 8) * DFS_B + 32 * 8 + 8;
}

template <int NN, int GP>
__device__ __forceinline__ int start_of(const int (&a)[NN][GP], int g) {
  int best = mux<GP>(a[0], g - 1);
#pragma unroll
  for (int n = 1; n < NN; ++n) best = min(best, mux<GP>(a[n], g - 1));
  return best;
}

// place (g, R) on the cluster state a (greedy node, lowest id on ties); returns s + R
template <int NN, int GP>
__device__ __forceinline__ int place_T(int (&a)[NN][GP], int g, int R, int one) {
  if constexpr (NN == 1) {
    return place_sorted<GP>(a[0], g, R, one);
  } else {
    int best = mux<GP>(a[0], g - 1);
    int bn = 0;
#pragma unroll
    for (int n = 1; n < NN; ++n) {
      const int st = mux<GP>(a[n], g - 1);
      const bool lt = st < best;
      best = lt ? st : best;
      bn = lt ? n : bn;
    }
    int x[GP];
    gather_node<NN, GP>(x, a, bn, one);
    const int v = place_sorted<GP>(x, g, R, one);
    scatter_node<NN, GP>(a, x, bn, one);
    return v;
  }
}

template <int NN, int GP>
__global__ void __launch_bounds__(DFS_B) k_enumerate_dfs(Problem pb, DfsSpace ds, uint64_t root_begin,
                                                         uint64_t root_end, unsigned long long* best_key,
                                                         unsigned long long* leaves_out) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint8_t* s_blob = sm;
  int* s_lv = reinterpret_cast<int*>(sm + pb.blob_bytes);
  const int T = pb.T;
  constexpr int W = DfsLayout<NN, GP>::W;
  uint64_t* s_red = reinterpret_cast<uint64_t*>(s_lv + (size_t)T * W * DFS_B);
  uint64_t* bar = s_red + 32;
  stage_problem(s_blob, pb, bar);
  const uint32_t* tab = tab_of(s_blob);
  const uint8_t* S = S_of(s_blob, pb);
  const int tid = threadIdx.x;
  auto LV = [&](int level, int w) -> int& { return s_lv[((size_t)level * W + w) * DFS_B + tid]; };
  const uint32_t full = (T == 32) ? 0xffffffffu : ((1u << T) - 1u);
  const uint64_t C = ds.es.cfg_space;

  uint64_t best = ~0ull, leaves = 0;
  // Roots by the static grid stride (dynamic batches measured slower, r1: see api.cu).
  const uint64_t nthr = (uint64_t)gridDim.x * DFS_B;
  const uint64_t gtid = (uint64_t)blockIdx.x * DFS_B + tid;
  for (uint64_t root = root_begin + gtid;; root += nthr) {
    if (root >= root_end) break;
    const int inc = (int)(*reinterpret_cast<volatile unsigned long long*>(best_key) >> 38);
    const int inc_ms = min(inc, (int)(best >> 38));
    int a[NN][GP];
#pragma unroll
    for (int n = 0; n < NN; ++n)
#pragma unroll
      for (int i = 0; i < GP; ++i) a[n][i] = (n < pb.N && i < pb.gpu_n[n]) ? 0 : INF;
    int ms = 0;
    uint32_t used = 0;
    uint64_t rperm = 0, rcfg = 0;
    uint64_t rr = root;
    bool ok = true;
    for (int i = 0; i < ds.D && ok; ++i) {  // decode and place the root's prefix
      const int pi = (int)(rr % (uint64_t)ds.sumS);
      rr /= (uint64_t)ds.sumS;
      int t = 0;
      while (ds.pre[t + 1] <= pi) ++t;
      const int c = pi - ds.pre[t];
      if ((used & (1u << t)) || (used & ds.twin_prev[t]) != ds.twin_prev[t]) { ok = false; break; }
      const uint32_t w = tab[t * pb.stride + c];
      ms = max(ms, place_T<NN, GP>(a, (int)(w >> 24), (int)(w & R_MASK), pb.one));
      rperm += (uint64_t)__popc(~used & full & ((1u << t) - 1u)) * ds.es.fact[T - 1 - i];
      rcfg += (uint64_t)c * ds.es.radix[t];
      used |= 1u << t;
      if (ms > inc_ms) ok = false;
    }
    if (!ok) continue;
    // DFS over levels D .. T-1; level L's saved state = the cluster after L placements
    int level = ds.D;
    int tc = -1, cc = 0;  // iterator at the current level
    while (true) {
      if (level == T - 1) {  // last position: closed form for every config of the last job
        const int t = __ffs(~used & full) - 1;
        const uint64_t base = rperm * C + rcfg;
        for (int c = 0; c < S[t]; ++c) {
          const uint32_t w = tab[t * pb.stride + c];
          const int leaf = max(ms, start_of<NN, GP>(a, (int)(w >> 24)) + (int)(w & R_MASK));
          const uint64_t key = ((uint64_t)leaf << 38) | (base + (uint64_t)c * ds.es.radix[t]);
          best = key < best ? key : best;
        }
        leaves += (uint64_t)S[t];
        if (level == ds.D) break;
        // backtrack to the parent level
        --level;
        goto restore;
      }
      // next (job, config) candidate at this level among the unplaced jobs
      if (tc >= 0 && cc + 1 < S[tc]) {
        ++cc;
      } else {
        const uint32_t rem = ~used & full & (tc >= 0 ? ~((2u << tc) - 1u) : full);
        if (rem == 0) {  // level exhausted
          if (level == ds.D) break;
          --level;
          goto restore;
        }
        tc = __ffs(rem) - 1;
        cc = 0;
        if ((used & ds.twin_prev[tc]) != ds.twin_prev[tc]) {  // a twin before its predecessor
          cc = S[tc] - 1;
          continue;
        }
      }
      {
        const uint32_t w = tab[tc * pb.stride + cc];
        int b[NN][GP];
#pragma unroll
        for (int n = 0; n < NN; ++n)
#pragma unroll
          for (int i = 0; i < GP; ++i) b[n][i] = a[n][i];
        const int ms2 = max(ms, place_T<NN, GP>(b, (int)(w >> 24), (int)(w & R_MASK), pb.one));
        if (ms2 > inc_ms) continue;  // strict cut: no leaf below can reach the incumbent
        // save this level and descend
#pragma unroll
        for (int n = 0; n < NN; ++n)
#pragma unroll
          for (int i = 0; i < GP; ++i) LV(level, n * GP + i) = a[n][i];
        LV(level, NN * GP + 0) = ms;
        LV(level, NN * GP + 1) = (int)(uint32_t)rperm;
        LV(level, NN * GP + 2) = (int)(uint32_t)(rperm >> 32);
        LV(level, NN * GP + 3) = (int)(uint32_t)rcfg;
        LV(level, NN * GP + 4) = (int)(uint32_t)(rcfg >> 32);
        LV(level, NN * GP + 5) = (int)used;
        LV(level, NN * GP + 6) = tc;
        LV(level, NN * GP + 7) = cc;
        rperm += (uint64_t)__popc(~used & full & ((1u << tc) - 1u)) * ds.es.fact[T - 1 - level];
        rcfg += (uint64_t)cc * ds.es.radix[tc];
        used |= 1u << tc;
        ms = ms2;
#pragma unroll
        for (int n = 0; n < NN; ++n)
#pragma unroll
          for (int i = 0; i < GP; ++i) a[n][i] = b[n][i];
        ++level;
        tc = -1;
        cc = 0;
        continue;
      }
    restore:
#pragma unroll
      for (int n = 0; n < NN; ++n)
#pragma unroll
        for (int i = 0; i < GP; ++i) a[n][i] = LV(level, n * GP + i);
      ms = LV(level, NN * GP + 0);
      rperm = (uint64_t)(uint32_t)LV(level, NN * GP + 1) | ((uint64_t)(uint32_t)LV(level, NN * GP + 2) << 32);
      rcfg = (uint64_t)(uint32_t)LV(level, NN * GP + 3) | ((uint64_t)(uint32_t)LV(level, NN * GP + 4) << 32);
      used = (uint32_t)LV(level, NN * GP + 5);
      tc = LV(level, NN * GP + 6);
      cc = LV(level, NN * GP + 7);
    }
    // Share an improved incumbent as soon as this root's subtree is done, so other threads
    // (and, over peer memory, other ranks) prune against it from their next root on.  Only
    // improvements are published: a real leaf's (makespan, index) key, so the final
    // atomicMin result is unchanged.
    if ((int)(best >> 38) < inc) atomicMin(best_key, (unsigned long long)best);
  }
  best = warp_min_u64(best);
  const int lane = tid & 31, warp = tid >> 5;
  if (lane == 0) s_red[warp] = best;
  for (int m = 16; m >= 1; m >>= 1) leaves += __shfl_xor_sync(0xffffffffu, leaves, m);
  __syncthreads();
  if (tid == 0) {
    uint64_t b2 = s_red[0];
    for (int w = 1; w < DFS_B / 32; ++w) b2 = s_red[w] < b2 ? s_red[w] : b2;
    if (b2 != ~0ull) atomicMin(best_key, (unsigned long long)b2);
  }
  if (lane == 0 && leaves) atomicAdd(leaves_out, (unsigned long long)leaves);
}

cudaError_t launch_enumerate_dfs(const Problem& pb, int NN, int GP, const DfsSpace& ds, uint64_t root_begin,
                                 uint64_t root_end, unsigned long long* best_key, unsigned long long* leaves,
                                 int sms, cudaStream_t st) {
  if (root_end <= root_begin) return cudaSuccess;
  const size_t smem = dfs_smem_bytes(pb, NN, GP);
  const uint64_t total = root_end - root_begin;
#define SAT_DFS(a, b)                                                                              \
  if (NN == a && GP == b && a >= 1) {                                                              \
    constexpr int A_ = (a >= 1 ? a : 1);                                                           \
    const int g0 = grid_for(k_enumerate_dfs<A_, b>, DFS_B, smem, sms, 1 << 30);                    \
    const uint64_t need = (total + DFS_B - 1) / DFS_B;                                             \
    const int g = (int)(need < (uint64_t)g0 ? need : (uint64_t)g0);                                \
    k_enumerate_dfs<A_, b><<<g, DFS_B, smem, st>>>(pb, ds, root_begin, root_end, best_key, leaves);       \
    return cudaGetLastError();                                                                     \
  }
  SAT_SHAPES(SAT_DFS)
#undef SAT_DFS
  return cudaErrorInvalidConfiguration;
}

// ------------------------------------------------------------------ K3 (+K1): GA
// GA v5 (oracle/ga.py is the normative text): the generation kernel makes the two children
// of a PAIR of parents per thread iteration (complementary uniform crossover of the configs,
// LOX of the permutations with shared cuts, per-child mutations), so the tournaments, the
// parent reads, the cuts and the crossover bits are shared by two children.
// Thread-private genome rows in shared memory (RowG, odd-word stride RS >= GS): for short
// genomes (T <= 32) the child C, parent A and parent B; long genomes keep only C and read
// the parents from the population in global memory (L1/L2), plus the LOX slice bit set
// (ceil(T/32) words per thread, interleaved).  The init kernel keeps one row.
__host__ __device__ __forceinline__ int ga_rows(int T, bool init) { return (init || T > 32) ? 1 : 3; }
__host__ __device__ __forceinline__ size_t lox_bits_bytes(const Problem& pb, bool init) {
  return (init || pb.T <= 32) ? 0 : (size_t)4 * ((pb.T + 31) / 32) * GA_B;
}
// Long genomes on column states stage each child's parents in shared memory (cp.async, one
// round trip): X into the child row, Y into the idle node-state region, GS / 4 rows.
__host__ __device__ __forceinline__ size_t ga_ns_bytes(const Problem& pb, int NN, int GP, int GS) {
  const size_t col = ns_bytes(pb, ga_mode(NN, GP), NN, GP, GA_B);
  return (ga_col(NN, GP) && pb.T > 32 && (size_t)GS * GA_B > col) ? (size_t)GS * GA_B : col;
}
static size_t ga_smem_bytes(const Problem& pb, int NN, int GP, int GS, bool init) {
  return (size_t)pb.blob_bytes + ga_ns_bytes(pb, NN, GP, GS) +
         (size_t)ga_rows(pb.T, init) * GA_B * odd_row_stride(GS) + lox_bits_bytes(pb, init) + 8 * GA_B + 8;
}

// 4-byte asynchronous global -> shared copies (LDGSTS), completed by cp_async_wait_all.
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

#ifndef SAT_GA_CACHE_HINTS
#define SAT_GA_CACHE_HINTS 1   // r2: TXT k_ga -1.8 %, MIX -1.9 %, DRAM reads -14 % per launch
#endif
// Copy a GS-byte global record into a smem row (4-byte stores) and back.  STREAM: the
// record is read / written with the evict-first hint (ld/st .cs), so the population records
// (2 x P x GS bytes per generation, > L2) do not push the makespan array out of L2.
template <bool STREAM = false>
__device__ __forceinline__ void load_row(uint8_t* row, const uint8_t* __restrict__ g, int GS) {
  const uint4* src = reinterpret_cast<const uint4*>(g);
  uint32_t* d = reinterpret_cast<uint32_t*>(row);
  for (int k = 0; k < GS / 16; ++k) {
    const uint4 v = STREAM ? __ldcs(src + k) : src[k];
    d[4 * k] = v.x;
    d[4 * k + 1] = v.y;
    d[4 * k + 2] = v.z;
    d[4 * k + 3] = v.w;
  }
}
template <bool STREAM = false>
__device__ __forceinline__ void store_row(uint8_t* __restrict__ g, const uint8_t* row, int GS) {
  uint4* dst = reinterpret_cast<uint4*>(g);
  const uint32_t* s = reinterpret_cast<const uint32_t*>(row);
  for (int k = 0; k < GS / 16; ++k) {
    const uint4 v = make_uint4(s[4 * k], s[4 * k + 1], s[4 * k + 2], s[4 * k + 3]);
    if (STREAM) __stcs(dst + k, v);
    else dst[k] = v;
  }
}

#ifndef SAT_GA_L2PF
#define SAT_GA_L2PF 1   // long genomes: L2 prefetch of the next pair's parent records
#endif
#ifndef SAT_GA_VEC
#define SAT_GA_VEC 1   // long genomes on register states: parents read by 16-byte loads
#endif

template <int NN, int GP>
struct GaMinBlocks {
  static constexpr int STATE = (NN == 0 ? 1 : NN) * GP;
  // measured r1 (dynamic chunks): 7 CTAs/SM (72 registers) for one 8-GPU node and for
  // 16-slot states, 4 for 32-slot states (SWEEP's shared memory caps it at 3-5 anyway);
  // small states too since GA v5 (8 CTAs = 64 registers spill)
  static constexpr int value = NN == 0 ? (GP <= 8 ? 6 : (GP <= 16 ? 4 : 2))
                                       : (STATE <= 16 ? 7 : (STATE <= 32 ? 4 : 2));
};

// Dynamic work distribution: a warp's first chunk of 32 units comes from the static grid
// stride, later ones are claimed from a counter (n_cand[1], zeroed by the previous elite
// selection) one iteration before they are needed, so warps that finish early take more
// (the static stride left SMs idle in the tail -- measured r1: MIX k_ga -11 %, SWEEP -10 %).
// Only lane 0's `pending` is meaningful (read by the shuffle); the atomic's result is first
// consumed by the next advance(), not by a select right after it.
struct WarpChunks {
  unsigned int* work;
  int64_t nthr, next;
  unsigned int pending = 0u;
  int lane;
  __device__ __forceinline__ void claim() {
    if (lane == 0) pending = atomicAdd(work, 32u);
  }
  __device__ __forceinline__ WarpChunks(int* n_cand, int64_t nthr_, int lane_)
      : work(reinterpret_cast<unsigned int*>(n_cand + 1)), nthr(nthr_), lane(lane_) {
    claim();
    next = nthr + (int64_t)__shfl_sync(0xffffffffu, pending, 0);
    claim();
  }
  // the next chunk's base; the one after it is claimed now
  __device__ __forceinline__ int64_t advance() {
    const int64_t b = next;
    next = nthr + (int64_t)__shfl_sync(0xffffffffu, pending, 0);
    claim();
    return b;
  }
};

// Block-level merge of the warps' top-E lists -> this block's real keys appended to cand[].
__device__ __forceinline__ void emit_topE(uint64_t lst, uint64_t* s_lists, int E, unsigned long long* cand,
                                          int* n_cand) {
  const int tid = threadIdx.x, lane = tid & 31;
  s_lists[tid] = lst;
  __syncthreads();
  if (tid < 32) {
    uint64_t m = ~0ull;
    for (int w = 0; w < GA_B / 32; ++w) topE_insert(m, s_lists[w * 32 + lane], E);
    // append only the real keys (after the first generation most blocks have none)
    const bool real = lane < E && m != ~0ull;
    const uint32_t mask = __ballot_sync(0xffffffffu, real);
    int off = 0;
    if (lane == 0 && mask) off = atomicAdd(n_cand, __popc(mask));
    off = __shfl_sync(0xffffffffu, off, 0);
    if (real) cand[off + __popc(mask & ((1u << lane) - 1u))] = m;
  }
}

// Generation 0: seed genomes, then cfg[t] = U(S_t) and a Fisher-Yates shuffle from the
// slot's own Philox stream; every genome decoded.
template <int NN, int GP>
__global__ void __launch_bounds__(GA_B, GaMinBlocks<NN, GP>::value)
    k_ga_init(Problem pb, GaParams gp, const uint8_t* __restrict__ seeds, int64_t n_seed, uint8_t* __restrict__ pop,
              int32_t* __restrict__ ms_out, unsigned long long* __restrict__ cand, int* __restrict__ n_cand) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int T = pb.T, GS = gp.GS, RS = odd_row_stride(GS), Tp = perm_offset(T);
  uint8_t* s_blob = sm;
  int* s_ns = reinterpret_cast<int*>(sm + pb.blob_bytes);
  uint8_t* s_rows = sm + pb.blob_bytes + ga_ns_bytes(pb, NN, GP, GS);
  uint64_t* s_lists = reinterpret_cast<uint64_t*>(s_rows + GA_B * RS);
  uint64_t* bar = s_lists + GA_B;
  stage_problem(s_blob, pb, bar);
  const uint32_t* tab = tab_of(s_blob);
  const uint8_t* S = S_of(s_blob, pb);
  const int tid = threadIdx.x, lane = tid & 31;
  const RowG ch{s_rows + RS * tid, Tp};
  int* ns = s_ns + tid;
  uint64_t lst = ~0ull;
  WarpChunks wc(n_cand, (int64_t)gridDim.x * GA_B, lane);
  for (int64_t base = (int64_t)blockIdx.x * GA_B + (tid & ~31); base < gp.P; base = wc.advance()) {
    const int64_t slot = base + lane;
    const bool live = slot < gp.P;
    int msv = INT_MAX;
    if (live) {
      if (slot < n_seed) {
        load_row(ch.base, seeds + slot * GS, GS);
      } else {
        Philox rng(gp.seed, (uint32_t)slot, 0u, (gp.rank << 16) | 1u);
        for (int t = 0; t < GS; ++t) ch.base[t] = 0;
        for (int t = 0; t < T; ++t) ch.c(t) = (uint8_t)rng.below(S[t]);
        for (int t = 0; t < T; ++t) ch.q(t) = (uint8_t)t;
        for (int i = T - 1; i > 0; --i) {
          const int j = (int)rng.below(i + 1);
          const uint8_t a = ch.q(i);
          ch.q(i) = ch.q(j);
          ch.q(j) = a;
        }
      }
      msv = decode_T<NN, GP, GA_B, ga_mode(NN, GP), 0>(tab, S, pb.stride, ch, T, pb, ns);
      store_row(pop + slot * GS, ch.base, GS);
      ms_out[slot] = msv;
    }
    topE_insert(lst, live ? (((uint64_t)(uint32_t)msv << 32) | (uint64_t)slot) : ~0ull, gp.E);
  }
  emit_topE(lst, s_lists, gp.E, cand, n_cand);
}

// Generation gen >= 1 (pairs).  LONGT: T > 32 (parents from global memory, the LOX slice
// as a shared-memory bit set); otherwise parents staged in rows and the slice in a register.
template <int NN, int GP, bool LONGT>
__global__ void __launch_bounds__(GA_B, GaMinBlocks<NN, GP>::value)
    k_ga(Problem pb, GaParams gp, const uint8_t* __restrict__ prev_pop, const int32_t* __restrict__ prev_ms,
         const int32_t* __restrict__ rec_ms, const uint8_t* __restrict__ rec_gen, uint8_t* __restrict__ pop,
         int32_t* __restrict__ ms_out, unsigned long long* __restrict__ cand, int* __restrict__ n_cand) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int T = pb.T, GS = gp.GS, RS = odd_row_stride(GS), Tp = perm_offset(T);
  constexpr int ROWS = LONGT ? 1 : 3;
  uint8_t* s_blob = sm;
  int* s_ns = reinterpret_cast<int*>(sm + pb.blob_bytes);
  uint8_t* s_rows = sm + pb.blob_bytes + ga_ns_bytes(pb, NN, GP, GS);
  uint32_t* s_bits = reinterpret_cast<uint32_t*>(s_rows + ROWS * GA_B * RS);
  uint64_t* s_lists = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(s_bits) + lox_bits_bytes(pb, false));
  uint64_t* bar = s_lists + GA_B;
  stage_problem(s_blob, pb, bar);
  const uint32_t* tab = tab_of(s_blob);
  const uint8_t* S = S_of(s_blob, pb);
  const int tid = threadIdx.x, lane = tid & 31;
  const RowG ch{s_rows + RS * tid, Tp};
  uint8_t* const rowA = s_rows + GA_B * RS + RS * tid;   // (short genomes only)
  uint8_t* const rowB = rowA + GA_B * RS;
  uint32_t* inA = s_bits + tid;   // LOX slice set for T > 32: word w at inA[w * GA_B]
  const uint32_t P = (uint32_t)gp.P;
  const uint32_t NP = (P + 1) >> 1;
  const int nb = (T + 31) / 32;
  const int nw = (T + 3) >> 2;
  int* ns = s_ns + tid;
  const uint32_t px16 = gp.px >> 16, pc16 = gp.pc >> 16, pm16 = gp.pm >> 16;
  const uint32_t k0 = (uint32_t)gp.seed, k1 = (uint32_t)(gp.seed >> 32), c2 = gp.rank << 16;

  uint64_t lst = ~0ull;
  // The next top-E can only contain keys <= the last elite's key (the elites are carried):
  // only those are offered to the list.
  const uint64_t cap = ((uint64_t)(uint32_t)rec_ms[gp.E - 1] << 32) | (uint64_t)(gp.E - 1);
  // Tournament prefetch: the candidates' makespans of this thread's NEXT pair are loaded one
  // iteration ahead, so their latency hides behind the current pair's decodes.
  uint32_t t_i1 = 0, t_j1 = 0, t_i2 = 0, t_j2 = 0, t_m1 = 0, t_n1 = 0, t_m2 = 0, t_n2 = 0;
  auto prefetch = [&](int64_t q) {
    if (q < NP && 2 * q + 1 >= (int64_t)gp.E) {
      const uint4 w0 = philox_block(k0, k1, (uint32_t)q, gp.gen, c2, 0u);
      t_i1 = ubelow(w0.x, P); t_j1 = ubelow(w0.y, P); t_i2 = ubelow(w0.z, P); t_j2 = ubelow(w0.w, P);
      t_m1 = (uint32_t)prev_ms[t_i1]; t_n1 = (uint32_t)prev_ms[t_j1];
      t_m2 = (uint32_t)prev_ms[t_i2]; t_n2 = (uint32_t)prev_ms[t_j2];
    }
  };
  WarpChunks chunks(n_cand, (int64_t)gridDim.x * GA_B, lane);
  prefetch((int64_t)blockIdx.x * GA_B + (tid & ~31) + lane);
  for (int64_t base = (int64_t)blockIdx.x * GA_B + (tid & ~31); base < NP;) {
    const uint32_t q = (uint32_t)base + lane;   // P < 2^32 (validated at the boundary)
    const bool live = q < NP;
    const uint32_t s0 = 2 * q;
    const bool kid0 = live && s0 >= (uint32_t)gp.E;
    const bool kid1 = live && s0 + 1 < P && s0 + 1 >= (uint32_t)gp.E;
    const bool any = kid0 || kid1;
    uint32_t A = 0, B = 0;
    if (any) {  // 1. tournaments (words 0..3, makespans prefetched)
      A = ((((uint64_t)t_m1 << 32) | t_i1) < (((uint64_t)t_n1 << 32) | t_j1)) ? t_i1 : t_j1;
      B = ((((uint64_t)t_m2 << 32) | t_i2) < (((uint64_t)t_n2 << 32) | t_j2)) ? t_i2 : t_j2;
    }
    prefetch(chunks.next + lane);
    const uint4 w1 = philox_block(k0, k1, (uint32_t)q, gp.gen, c2, 1u);   // shared fields
    const uint8_t* gA = prev_pop + (uint64_t)A * GS;
    const uint8_t* gB = prev_pop + (uint64_t)B * GS;
    if (!LONGT && any) {
      load_row<SAT_GA_CACHE_HINTS>(rowA, gA, GS);
      load_row<SAT_GA_CACHE_HINTS>(rowB, gB, GS);
    }
    const bool xo = any && (w1.x & 0xffffu) < px16;
    uint32_t a = v16(w1.x >> 16, T), b = v16(w1.y & 0xffffu, T);
    if (a > b) { const uint32_t x = a; a = b; b = x; }
#pragma unroll 1
    for (int r = 0; r < 2; ++r) {
      const uint32_t slot = s0 + r;
      const bool in = live && slot < P;
      const bool elite = in && slot < (uint32_t)gp.E;
      const bool child = r ? kid1 : kid0;
      // 2. child r = X (A for r = 0, B for r = 1) crossed with Y (the other parent)
      const uint8_t* X = LONGT ? (r ? gB : gA) : (r ? rowB : rowA);
      const uint8_t* Y = LONGT ? (r ? gA : gB) : (r ? rowA : rowB);
      const uint4 wk = philox_block(k0, k1, (uint32_t)q, gp.gen, c2, 2u + (uint32_t)r);   // child r's fields
      int msv = INT_MAX;
      if (elite) {
        load_row(ch.base, rec_gen + (size_t)slot * GS, GS);
        msv = rec_ms[slot];
      }
      // Long genomes on column states: X's record is copied into the child row and Y's into
      // the idle node-state region (word w at ns[w * GA_B]) with cp.async, one round trip,
      // instead of the loops below waiting on global loads (12 warps per SM leave too few to
      // hide them).  The child then starts as X: crossover and LOX work in place.
      constexpr bool STAGE = LONGT && ga_col(NN, GP);
      if (STAGE && child) {
        const uint32_t* gx = reinterpret_cast<const uint32_t*>(X);
        const uint32_t* gy = reinterpret_cast<const uint32_t*>(Y);
        uint32_t* cw = reinterpret_cast<uint32_t*>(ch.base);
        for (int w = 0; w < GS / 4; ++w) {
          cp_async4(cw + w, gx + w);
          cp_async4(ns + w * GA_B, gy + w);
        }
        cp_async_wait_all();
        uint32_t* cwv = cw;
        const auto ys = [&](int w) -> uint32_t { return (uint32_t)ns[w * GA_B]; };
        const auto mixs = [&](int t, uint32_t bits) {
          const uint32_t nib = xo ? (~(bits >> (t & 31)) & 0xfu) : 0u;
          const uint32_t m = ((nib * 0x00204081u) & 0x01010101u) * 0xffu;
          cwv[t >> 2] = (cwv[t >> 2] & ~m) | (ys(t >> 2) & m);
        };
        for (int t0 = 0; t0 < T; t0 += 32) {
          const int k = t0 >> 5;
          const uint32_t bits =
              k == 0 ? w1.z : (k == 1 ? w1.w : philox_word(k0, k1, (uint32_t)q, gp.gen, c2, 16u + (k - 2)));
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (t0 + 4 * j < T) mixs(t0 + 4 * j, bits);
        }
      }
      if (!STAGE && child) {
        // 3. uniform crossover of the config genes, 4 genes per step (bit 1 -> X's gene);
        //    the permutation starts as a copy of X's
        const uint32_t* cx = reinterpret_cast<const uint32_t*>(X);
        const uint32_t* cy = reinterpret_cast<const uint32_t*>(Y);
        uint32_t* cw = reinterpret_cast<uint32_t*>(ch.base);
        const auto mix = [&](int t, uint32_t bits) {
          const uint32_t nib = xo ? (~(bits >> (t & 31)) & 0xfu) : 0u;     // 1 -> take Y's gene
          const uint32_t m = ((nib * 0x00204081u) & 0x01010101u) * 0xffu;  // nibble -> byte mask
          cw[t >> 2] = (cx[t >> 2] & ~m) | (cy[t >> 2] & m);               // pad bytes: 0 in both
        };
        if (!LONGT) {
          for (int t = 0; t < T; t += 4) mix(t, w1.z);
        } else {   // 32 genes per crossover word; the parents' 8 words of a block as two
                   // 16-byte loads each (records are 16-byte aligned; ceil(T/32)*32 <= GS)
          for (int t0 = 0; t0 < T; t0 += 32) {
            const int k = t0 >> 5;
            const uint32_t bits =
                k == 0 ? w1.z : (k == 1 ? w1.w : philox_word(k0, k1, (uint32_t)q, gp.gen, c2, 16u + (k - 2)));
#if SAT_GA_VEC
            const uint4* x4 = reinterpret_cast<const uint4*>(X) + 2 * k;
            const uint4* y4 = reinterpret_cast<const uint4*>(Y) + 2 * k;
            const uint4 xa = x4[0], xb = x4[1], ya = y4[0], yb = y4[1];
            const uint32_t xw[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
            const uint32_t yw[8] = {ya.x, ya.y, ya.z, ya.w, yb.x, yb.y, yb.z, yb.w};
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (t0 + 4 * j < T) {
                const uint32_t nib = xo ? (~(bits >> (4 * j)) & 0xfu) : 0u;
                const uint32_t m = ((nib * 0x00204081u) & 0x01010101u) * 0xffu;
                cw[(t0 >> 2) + j] = (xw[j] & ~m) | (yw[j] & m);
              }
#else
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (t0 + 4 * j < T) mix(t0 + 4 * j, bits);
#endif
          }
        }
        if (!LONGT || !SAT_GA_VEC) {
#pragma unroll 4
          for (int w = 0; w < nw; ++w) cw[(Tp >> 2) + w] = cx[(Tp >> 2) + w];
        } else {   // X's permutation words by 16-byte loads from the aligned word below Tp
          const uint4* x4 = reinterpret_cast<const uint4*>(X);
          const int w0 = Tp >> 2, w1e = w0 + nw;
          for (int u = w0 >> 2; 4 * u < w1e; ++u) {
            const uint4 v = x4[u];
            const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (4 * u + e >= w0 && 4 * u + e < w1e) cw[4 * u + e] = vw[e];
          }
        }
      }
      // 4. LOX: keep X.perm[a..b] in place; fill positions 0..a-1, then b+1..T-1, with Y's
      //    genes in Y's order from position 0, skipping the slice's genes.
      {
        uint8_t* const p0 = &ch.q(0);
        uint8_t* const pa = p0 + a;
        const uint32_t gap = b - a + 1;
        uint8_t* wp = (a == 0) ? p0 + gap : p0;
        const uint8_t* Yq = Y + Tp;
        if (!LONGT) {
          // Genes < 32: the slice is a bit set.  Four genes per shared-memory word, gene
          // bits by wrapping funnel shifts (x & 31 for free), positions a..b as a bit mask.
          const uint32_t* xq = reinterpret_cast<const uint32_t*>(p0);
          const uint32_t* yq = reinterpret_cast<const uint32_t*>(Yq);
          const uint32_t M = (0xffffffffu >> (31u - b)) & (0xffffffffu << a);   // b <= 31
          uint32_t kept = 0;
          for (int w = 0; w < nw; ++w) {   // pad genes lie outside a..b
            const uint32_t W = xq[w], Mw = M >> (4 * w);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (Mw & (1u << e)) kept |= __funnelshift_l(0u, 1u, W >> (8 * e));
          }
          if (!(xo && child)) kept = 0xffffffffu;   // nothing is taken
          // branch-free fill: predicated byte store (of the low byte), pointer arithmetic
          // on the complemented set: one funnel rotate + one AND-to-predicate per gene (r2:
          // TXT k_ga -1.0 %, MIX -0.5 to -1.5 % against ~(kept >> x) & 1 and a select)
          const uint32_t nk = ~kept;   // bit x set <=> gene x is taken
          const auto fill = [&](uint32_t x) {
            const uint32_t take = __funnelshift_r(nk, nk, x) & 1u;   // rotate: bit 0 = bit (x & 31)
            if (take) *wp = (uint8_t)x;
            wp += take;
            if (wp == pa) wp += gap;
          };
          const int nf = T >> 2;
          for (int w = 0; w < nf; ++w) {
            const uint32_t W = yq[w];
#pragma unroll
            for (int e = 0; e < 4; ++e) fill(W >> (8 * e));
          }
          if (T & 3) {   // the last, partial word (its pad bytes are not genes)
            const uint32_t W = yq[nf];
#pragma unroll
            for (int e = 0; e < 3; ++e)
              if (e < (T & 3)) fill(W >> (8 * e));
          }
        } else {
          // Rows of lanes without a child hold stale bytes: the word index is clamped so
          // those lanes stay inside this thread's ceil(T/32) words.
          // the complemented set (bit x set <=> gene x is taken), all clear when nothing
          // is taken: the fill's test is one rotate + one AND-to-predicate
          const uint32_t init = (xo && child) ? 0xffffffffu : 0u;
          for (int w = 0; w < nb; ++w) inA[w * GA_B] = init;
          for (int k = (int)a; k <= (int)b; ++k) {
            const int x = ch.q(k);
            inA[min(x >> 5, nb - 1) * GA_B] &= ~(1u << (x & 31));
          }
          const auto fill = [&](int x) {
            const uint32_t w = inA[min(x >> 5, nb - 1) * GA_B];
            const uint32_t take = __funnelshift_r(w, w, x) & 1u;
            if (take) *wp = (uint8_t)x;
            wp += take;
            if (wp == pa) wp += gap;
          };
          if constexpr (STAGE) {   // Y's permutation from the staged words
            for (int k = 0; k < T; k += 4) {
              const uint32_t y4 = child ? (uint32_t)ns[((Tp + k) >> 2) * GA_B] : 0u;
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if (k + e < T) fill((int)((y4 >> (8 * e)) & 0xffu));
            }
          } else if (SAT_GA_VEC) {   // Y's permutation 16 genes per load (aligned below Tp)
            const uint4* y4 = reinterpret_cast<const uint4*>(Y);
            const int g0 = Tp & ~15;
            for (int u = g0 >> 4; 16 * u < Tp + T; ++u) {
              const uint4 v = child ? y4[u] : make_uint4(0u, 0u, 0u, 0u);
              const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const int k = 16 * u + e - Tp;
                if (k >= 0 && k < T) fill((int)((vw[e >> 2] >> (8 * (e & 3))) & 0xffu));
              }
            }
          } else {
            for (int k = 0; k < T; ++k) fill(child ? Yq[k] : 0);
          }
        }
      }
      // 5. config mutation of one job
      if (child && (wk.z & 0xffffu) < pc16) {
        const int t = (int)v16(wk.z >> 16, T);
        ch.c(t) = (uint8_t)v16(wk.w & 0xffffu, S[t]);
      }
      // 6. permutation mutation.  Swap (kind 0): two byte moves.  Insertion (kind 1, remove
      //    the gene at i, reinsert it at j): positions between i and j shift by one toward i,
      //    a word (4 genes) at a time with funnel shifts and byte masks, then x -> j.
      if (child && (wk.x & 0xffffu) < pm16) {
        const int kind = (int)((wk.y >> 16) & 1u);
        const int mi = (int)v16(wk.x >> 16, T), mj = (int)v16(wk.y & 0xffffu, T);
        const uint8_t xi = ch.q(mi), xj = ch.q(mj);
        if (kind == 0) {
          ch.q(mi) = xj;
          ch.q(mj) = xi;
        } else if (mi != mj) {
          const int lo = min(mi, mj), hi = max(mi, mj);
          uint32_t* pw = reinterpret_cast<uint32_t*>(ch.base + Tp);
          int w = lo >> 2;
          uint32_t prev = (w > 0) ? pw[w - 1] : 0u, cur = pw[w];
          for (; w <= (hi >> 2); ++w) {
            const uint32_t next = (w + 1 < nw) ? pw[w + 1] : 0u;
            const uint32_t sh = (mi < mj) ? __funnelshift_r(cur, next, 8) : __funnelshift_l(prev, cur, 8);
            const int bl = max(lo - 4 * w, 0), bh = min(hi - 4 * w + 1, 4);
            const uint32_t m = (bh >= 4 ? 0xffffffffu : ((1u << (8 * bh)) - 1u)) & ~((1u << (8 * bl)) - 1u);
            pw[w] = (sh & m) | (cur & ~m);
            prev = cur;
            cur = next;
          }
          ch.q(mj) = xi;
        }
      }
      if (child) msv = decode_T<NN, GP, GA_B, ga_mode(NN, GP), 0>(tab, S, pb.stride, ch, T, pb, ns);
      if (in) {
        store_row<SAT_GA_CACHE_HINTS>(pop + (size_t)slot * GS, ch.base, GS);
        ms_out[slot] = msv;
      }
      topE_insert(lst, in ? (((uint64_t)(uint32_t)msv << 32) | (uint64_t)slot) : ~0ull, gp.E, cap);
    }
    if constexpr (LONGT && SAT_GA_L2PF) {   // (short genomes: measured +2.5 % TXT k_ga, r2)
      // The next pair's tournaments are decided now (their makespans arrived during this
      // pair's decodes) and both winners' records are pulled into L2: long genomes read
      // their parents straight from the population (an HBM-sized array), and the
      // crossover / LOX loops would otherwise wait for DRAM.
      if (chunks.next + lane < NP) {
        const uint32_t An = ((((uint64_t)t_m1 << 32) | t_i1) < (((uint64_t)t_n1 << 32) | t_j1)) ? t_i1 : t_j1;
        const uint32_t Bn = ((((uint64_t)t_m2 << 32) | t_i2) < (((uint64_t)t_n2 << 32) | t_j2)) ? t_i2 : t_j2;
        const uint8_t* ra = prev_pop + (uint64_t)An * GS;
        const uint8_t* rb = prev_pop + (uint64_t)Bn * GS;
        for (int o = 0; o < GS + 127; o += 128) {
          const int oo = min(o, GS - 1);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(ra + oo));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rb + oo));
        }
      }
    }
    base = chunks.advance();
  }
  emit_topE(lst, s_lists, gp.E, cand, n_cand);
}

template <int A, int B>
static cudaError_t ga_shape(const Problem& pb, const GaParams& gp, const uint8_t* seeds, int64_t n_seed,
                            const uint8_t* prev_pop, const int32_t* prev_ms, const int32_t* rec_ms,
                            const uint8_t* rec_gen, uint8_t* pop, int32_t* ms, unsigned long long* cand, int* d_n_cand,
                            int sms, cudaStream_t st) {
  const bool init = gp.gen == 0;
  const size_t smem = ga_smem_bytes(pb, A, B, gp.GS, init);
  if (init) {
    const int g = grid_for(k_ga_init<A, B>, GA_B, smem, sms, (gp.P + GA_B - 1) / GA_B);
    k_ga_init<A, B><<<g, GA_B, smem, st>>>(pb, gp, seeds, n_seed, pop, ms, cand, d_n_cand);
    return cudaGetLastError();
  }
  const int64_t blocks = ((gp.P + 1) / 2 + GA_B - 1) / GA_B;
  if (pb.T > 32) {
    const int g = grid_for(k_ga<A, B, true>, GA_B, smem, sms, blocks);
    k_ga<A, B, true><<<g, GA_B, smem, st>>>(pb, gp, prev_pop, prev_ms, rec_ms, rec_gen, pop, ms, cand, d_n_cand);
  } else {
    const int g = grid_for(k_ga<A, B, false>, GA_B, smem, sms, blocks);
    k_ga<A, B, false><<<g, GA_B, smem, st>>>(pb, gp, prev_pop, prev_ms, rec_ms, rec_gen, pop, ms, cand, d_n_cand);
  }
  return cudaGetLastError();
}
// grid size the largest variant of a shape can take (candidate buffer sizing)
template <int A, int B>
static int ga_grid_max(const Problem& pb, int GS, int sms, int64_t P) {
  const size_t s0 = ga_smem_bytes(pb, A, B, GS, true), s1 = ga_smem_bytes(pb, A, B, GS, false);
  const int64_t b0 = (P + GA_B - 1) / GA_B, b1 = ((P + 1) / 2 + GA_B - 1) / GA_B;
  return std::max(grid_for(k_ga_init<A, B>, GA_B, s0, sms, b0),
                  std::max(grid_for(k_ga<A, B, false>, GA_B, s1, sms, b1), grid_for(k_ga<A, B, true>, GA_B, s1, sms, b1)));
}

static cudaError_t launch_ga(const Problem& pb, int NN, int GP, const GaParams& gp, const uint8_t* seeds,
                             int64_t n_seed, const uint8_t* prev_pop, const int32_t* prev_ms, const int32_t* rec_ms,
                             const uint8_t* rec_gen, uint8_t* pop, int32_t* ms, unsigned long long* cand,
                             int* d_n_cand, int sms, cudaStream_t st) {
#define SAT_GA(a, b)                                                                                               \
  if (NN == a && GP == b)                                                                                          \
    return ga_shape<a, b>(pb, gp, seeds, n_seed, prev_pop, prev_ms, rec_ms, rec_gen, pop, ms, cand, d_n_cand, sms, \
                          st);
  SAT_SHAPES(SAT_GA)
#undef SAT_GA
  return cudaErrorInvalidConfiguration;
}

int ga_max_candidates(const Problem& pb, int NN, int GP, int E, int GS, int64_t P, int sms) {
  int g = 0;
#define SAT_GAC(a, b) \
  if (NN == a && GP == b) g = ga_grid_max<a, b>(pb, GS, sms, P);
  SAT_SHAPES(SAT_GAC)
#undef SAT_GAC
  return g * E;
}

cudaError_t launch_ga_init(const Problem& pb, int NN, int GP, const GaParams& gp, const uint8_t* seeds,
                           int64_t n_seed, uint8_t* pop, int32_t* ms, unsigned long long* cand, int* d_n_cand, int sms,
                           cudaStream_t st) {
  return launch_ga(pb, NN, GP, gp, seeds, n_seed, nullptr, nullptr, nullptr, nullptr, pop, ms, cand, d_n_cand, sms, st);
}
cudaError_t launch_ga_generation(const Problem& pb, int NN, int GP, const GaParams& gp, const uint8_t* prev_pop,
                                 const int32_t* prev_ms, const int32_t* rec_ms, const uint8_t* rec_gen, uint8_t* pop,
                                 int32_t* ms, unsigned long long* cand, int* d_n_cand, int sms, cudaStream_t st) {
  return launch_ga(pb, NN, GP, gp, nullptr, 0, prev_pop, prev_ms, rec_ms, rec_gen, pop, ms, cand, d_n_cand, sms, st);
}

// ------------------------------------------------------------------ f4: local search
// One CTA per genome: every thread decodes neighbours (insertion moves, then config moves;
// numbering as in oracle/local_search.py), the CTA moves to the best (ms, move) if it is a
// strict improvement, up to `iters` times.  Records are updated in place.
constexpr int LS_B = 128;
static size_t ls_smem_bytes(const Problem& pb, int NN, int GP, int GS) {
  return (size_t)pb.blob_bytes + ns_bytes(pb, eval_mode(NN, GP), NN, GP, LS_B) + (size_t)(LS_B + 1) * odd_row_stride(GS) +
         (size_t)4 * (pb.T + 1) + 8 * (LS_B / 32) + 16 + 8;
}

template <int NN, int GP>
__global__ void __launch_bounds__(LS_B) k_local_search(Problem pb, uint8_t* __restrict__ gen, int32_t* __restrict__ ms_io,
                                                       int GS, int iters) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int T = pb.T, Tp = perm_offset(T), RS = odd_row_stride(GS);
  uint8_t* s_blob = sm;
  int* s_ns = reinterpret_cast<int*>(sm + pb.blob_bytes);
  uint8_t* s_base = sm + pb.blob_bytes + ns_bytes(pb, eval_mode(NN, GP), NN, GP, LS_B);
  uint8_t* s_rows = s_base + RS;
  int* s_pre = reinterpret_cast<int*>(s_rows + LS_B * RS);       // prefix of (S_t - 1), T + 1 entries
  uint64_t* s_red = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(s_pre + T + 1) + 7) & ~uintptr_t(7));
  uint64_t* bar = s_red + LS_B / 32 + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* rec = gen + (size_t)blockIdx.x * GS;
  for (int k = tid; k < GS / 4; k += LS_B)
    reinterpret_cast<uint32_t*>(s_base)[k] = reinterpret_cast<const uint32_t*>(rec)[k];
  stage_problem(s_blob, pb, bar);   // its __syncthreads also publishes s_base
  const uint32_t* tab = tab_of(s_blob);
  const uint8_t* S = S_of(s_blob, pb);
  if (tid == 0) {
    int acc = 0;
    for (int t = 0; t < T; ++t) { s_pre[t] = acc; acc += S[t] - 1; }
    s_pre[T] = acc;
  }
  __syncthreads();
  const int n_ins = T * (T - 1), n_mov = n_ins + s_pre[T];
  int* ns = s_ns + tid;
  const RowG row{s_rows + RS * tid, Tp};
  const RowG base{s_base, Tp};
  int cur = ms_io[blockIdx.x];
  for (int it = 0; it < iters; ++it) {
    uint64_t best = ~0ull;
    for (int m = tid; m < n_mov; m += LS_B) {
      for (int k = 0; k < Tp / 4; ++k)
        reinterpret_cast<uint32_t*>(row.base)[k] = reinterpret_cast<const uint32_t*>(base.base)[k];
      if (m < n_ins) {
        const int i = m / (T - 1), jj = m - i * (T - 1), j = jj < i ? jj : jj + 1;
        const int lo = min(i, j), hi = max(i, j), d = (i < j) ? 1 : -1;
        for (int k = 0; k < T; ++k) {
          int src = (k >= lo && k <= hi) ? k + d : k;
          src = (k == j) ? i : src;
          row.q(k) = base.q(src);
        }
      } else {
        const int k2 = m - n_ins;
        int t = 0;
        while (s_pre[t + 1] <= k2) ++t;
        const int r = k2 - s_pre[t];
        row.c(t) = (uint8_t)(r < base.c(t) ? r : r + 1);
        for (int k = 0; k < T; ++k) row.q(k) = base.q(k);
      }
      const int msn = decode_T<NN, GP, LS_B, eval_mode(NN, GP), 0>(tab, S, pb.stride, row, T, pb, ns);
      const uint64_t key = ((uint64_t)(uint32_t)msn << 32) | (uint32_t)m;
      best = key < best ? key : best;
    }
    best = warp_min_u64(best);
    if (lane == 0) s_red[warp] = best;
    __syncthreads();
    if (tid == 0) {
      uint64_t b = s_red[0];
      for (int w = 1; w < LS_B / 32; ++w) b = s_red[w] < b ? s_red[w] : b;
      s_red[LS_B / 32] = b;
    }
    __syncthreads();
    const uint64_t b = s_red[LS_B / 32];
    const int bms = (int)(b >> 32);
    if (b == ~0ull || bms >= cur) break;  // local optimum (uniform across the CTA)
    if (tid == 0) {  // apply move b to the base genome
      const int m = (int)(b & 0xffffffffu);
      if (m < n_ins) {
        const int i = m / (T - 1), jj = m - i * (T - 1), j = jj < i ? jj : jj + 1;
        const int lo = min(i, j), hi = max(i, j), d = (i < j) ? 1 : -1;
        for (int k = 0; k < T; ++k) row.q(k) = base.q(k);
        for (int k = 0; k < T; ++k) {
          int src = (k >= lo && k <= hi) ? k + d : k;
          src = (k == j) ? i : src;
          base.q(k) = row.q(src);
        }
      } else {
        const int k2 = m - n_ins;
        int t = 0;
        while (s_pre[t + 1] <= k2) ++t;
        const int r = k2 - s_pre[t];
        base.c(t) = (uint8_t)(r < base.c(t) ? r : r + 1);
      }
    }
    cur = bms;
    __syncthreads();
  }
  for (int k = tid; k < GS / 4; k += LS_B)
    reinterpret_cast<uint32_t*>(rec)[k] = reinterpret_cast<const uint32_t*>(s_base)[k];
  if (tid == 0) ms_io[blockIdx.x] = cur;
}

cudaError_t launch_local_search(const Problem& pb, int NN, int GP, uint8_t* gen, int32_t* ms, int n, int GS, int iters,
                                cudaStream_t st) {
  if (n <= 0 || iters <= 0) return cudaSuccess;
  const size_t smem = ls_smem_bytes(pb, NN, GP, GS);
#define SAT_LS(a, b)                                                                        \
  if (NN == a && GP == b) {                                                                 \
    (void)grid_for(k_local_search<a, b>, LS_B, smem, 1, 1);                                 \
    k_local_search<a, b><<<n, LS_B, smem, st>>>(pb, gen, ms, GS, iters);                    \
    return cudaGetLastError();                                                              \
  }
  SAT_SHAPES(SAT_LS)
#undef SAT_LS
  return cudaErrorInvalidConfiguration;
}

// ------------------------------------------------------------------ K4: select / merge
__global__ void __launch_bounds__(1024) k_select(const unsigned long long* __restrict__ cand, int* __restrict__ n_cand,
                                                 int E, int GS, const uint8_t* __restrict__ pop,
                                                 int32_t* __restrict__ rec_ms, uint8_t* __restrict__ rec_gen) {
  __shared__ uint64_t s_l[32][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = *n_cand;
  uint64_t lst = ~0ull;
  constexpr int U = 8;  // independent loads in flight per thread
  for (int base = warp * 32; base < n; base += 1024 * U) {
    uint64_t k[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = base + j * 1024 + lane;
      k[j] = (i < n) ? cand[i] : ~0ull;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) topE_insert(lst, k[j], E);
  }
  s_l[warp][lane] = lst;
  __syncthreads();
  if (warp == 0) {
    lst = ~0ull;
    for (int w = 0; w < 32; ++w) topE_insert(lst, s_l[w][lane], E);
    if (lane < E) {
      const uint32_t slot = (uint32_t)(lst & 0xffffffffu);
      rec_ms[lane] = (int32_t)(lst >> 32);
      const uint4* src = reinterpret_cast<const uint4*>(pop + (uint64_t)slot * GS);
      uint4* dst = reinterpret_cast<uint4*>(rec_gen + (uint64_t)lane * GS);
      for (int k2 = 0; k2 < GS / 16; ++k2) dst[k2] = src[k2];
    }
    if (lane == 0) { n_cand[0] = 0; n_cand[1] = 0; }  // candidates and the GA work counter, next generation
  }
}

// One warp: after generation 0 only the children that beat the current E-th elite are
// appended (typically tens), so a single warp walks them without the block-wide merge.
__global__ void __launch_bounds__(32) k_select_warp(const unsigned long long* __restrict__ cand,
                                                    int* __restrict__ n_cand, int E, int GS,
                                                    const uint8_t* __restrict__ pop, int32_t* __restrict__ rec_ms,
                                                    uint8_t* __restrict__ rec_gen) {
  const int lane = threadIdx.x;
  const int n = *n_cand;
  uint64_t lst = ~0ull;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    topE_insert(lst, (i < n) ? cand[i] : ~0ull, E);
  }
  if (lane < E) {
    const uint32_t slot = (uint32_t)(lst & 0xffffffffu);
    rec_ms[lane] = (int32_t)(lst >> 32);
    const uint4* src = reinterpret_cast<const uint4*>(pop + (uint64_t)slot * GS);
    uint4* dst = reinterpret_cast<uint4*>(rec_gen + (uint64_t)lane * GS);
    for (int k2 = 0; k2 < GS / 16; ++k2) dst[k2] = src[k2];
  }
  if (lane == 0) { n_cand[0] = 0; n_cand[1] = 0; }
}

cudaError_t launch_select(const unsigned long long* cand, int* n_cand, int E, int GS, const uint8_t* pop,
                          int32_t* rec_ms, uint8_t* rec_gen, cudaStream_t st, bool few) {
  if (few)
    k_select_warp<<<1, 32, 0, st>>>(cand, n_cand, E, GS, pop, rec_ms, rec_gen);
  else
    k_select<<<1, 1024, 0, st>>>(cand, n_cand, E, GS, pop, rec_ms, rec_gen);
  return cudaGetLastError();
}

__global__ void k_merge(const int32_t* __restrict__ all_ms, const uint8_t* __restrict__ all_gen, int W, int E, int GS,
                        int32_t* __restrict__ rec_ms, uint8_t* __restrict__ rec_gen) {
  const int lane = threadIdx.x & 31;
  uint64_t lst = ~0ull;
  const int n = W * E;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const uint64_t key = (i < n) ? (((uint64_t)(uint32_t)all_ms[i] << 32) | (uint32_t)i) : ~0ull;
    topE_insert(lst, key, E);
  }
  if (lane < E) {
    const uint32_t i = (uint32_t)(lst & 0xffffffffu);
    rec_ms[lane] = (int32_t)(lst >> 32);
    const uint4* src = reinterpret_cast<const uint4*>(all_gen + (uint64_t)i * GS);
    uint4* dst = reinterpret_cast<uint4*>(rec_gen + (uint64_t)lane * GS);
    for (int k = 0; k < GS / 16; ++k) dst[k] = src[k];
  }
}

cudaError_t launch_merge_elites(const int32_t* all_ms, const uint8_t* all_gen, int W, int E, int GS, int32_t* rec_ms,
                                uint8_t* rec_gen, cudaStream_t st) {
  k_merge<<<1, 32, 0, st>>>(all_ms, all_gen, W, E, GS, rec_ms, rec_gen);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ integer-ALU probe
// 8 independent chains of IMNMX / IADD3 / ISETP+SEL per thread; 6 int ops per chain step.
constexpr int PROBE_ITERS = 4096;
__global__ void __launch_bounds__(256) k_int_probe(int* sink, int seed) {
  int x[8], y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { x[k] = seed + threadIdx.x + k; y[k] = seed ^ (k * 7919); }
  for (int i = 0; i < PROBE_ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int a = max(x[k], y[k]);       // IMNMX
      const int b = min(a + i, x[k] + 3);  // IADD3, IADD3, IMNMX
      y[k] = (b < y[k]) ? b : a;           // ISETP + SEL
      x[k] = b;
    }
  }
  int acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc ^= x[k] ^ y[k];
  if (acc == 0x12345678) sink[blockIdx.x] = acc;
}

double launch_int_probe(int sms, int* sink, cudaStream_t st) {
  const int blocks = sms * 8;
  k_int_probe<<<blocks, 256, 0, st>>>(sink, 1);
  return (double)blocks * 256 * PROBE_ITERS * 8 * 6;
}

}  // namespace sat
