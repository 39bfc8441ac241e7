// libsaturn host runtime: the C ABI of include/saturn.h (row b), table validation and
// compaction (rows a1/a2), workspace management, the search epoch loop and the island
// exchange (row e) over NCCL or over peer memory (peers.h).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: ranges cost nothing without a profiler
#include <memory>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/saturn.h"
#include "kernels.h"
#include "decode.cuh"
#include "peers.h"

using sat::Problem;

namespace {

// ------------------------------------------------------------------ NCCL (dlopen'ed)
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (tried) return n;
  tried = true;
  // Prefer the NCCL already loaded in the process (torch's), else the system one.
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    n.why = std::string("cannot load libnccl.so.2: ") + dlerror();
    return n;
  }
#define SAT_SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name));
  SAT_SYM(getUniqueId, "ncclGetUniqueId")
  SAT_SYM(commInitRank, "ncclCommInitRank")
  SAT_SYM(allReduce, "ncclAllReduce")
  SAT_SYM(allGather, "ncclAllGather")
  SAT_SYM(commDestroy, "ncclCommDestroy")
  SAT_SYM(getErrorString, "ncclGetErrorString")
#undef SAT_SYM
  n.ok = n.getUniqueId && n.commInitRank && n.allReduce && n.allGather && n.commDestroy && n.getErrorString;
  if (!n.ok) n.why = "libnccl is missing required symbols";
  return n;
}

// Caller-provided device workspace (saturn_bind_workspace): a bump arena every DevBuf of the
// handle carves from while it is bound, instead of cudaMalloc.  Nothing is freed inside it;
// saturn_workspace_bytes sizes it for one search (+ best_plan) from a fresh bind.
struct Arena {
  uint8_t* base = nullptr;
  size_t size = 0, off = 0;
  bool bound() const { return base != nullptr; }
};
constexpr size_t ARENA_ALIGN = 256;
inline size_t arena_round(size_t b) { return (b + ARENA_ALIGN - 1) & ~(ARENA_ALIGN - 1); }

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  bool owned = false;   // cudaMalloc'ed by the handle (else carved from the arena)
  Arena* arena = nullptr;
  cudaError_t ensure(size_t count) {
    if (count <= n && p) return cudaSuccess;
    release();
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (arena && arena->bound()) {
      const size_t b = arena_round(bytes);
      if (arena->off + b > arena->size) return cudaErrorMemoryAllocation;
      p = reinterpret_cast<T*>(arena->base + arena->off);
      arena->off += b;
      n = count;
      return cudaSuccess;
    }
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) {
      n = count;
      owned = true;
    } else {
      p = nullptr;
    }
    return e;
  }
  void release() {
    if (p && owned) cudaFree(p);
    p = nullptr;
    n = 0;
    owned = false;
  }
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// NVTX range for profilers (nsys / ncu --nvtx): search, epochs, exchanges, enumeration,
// introspection rounds.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

}  // namespace

struct saturn_plan {
  int device = 0;
  int sms = 148;
  std::vector<int> gpu_n;
  int sumG = 0, maxG = 0;
  // compacted table
  bool loaded = false;
  int T = 0, stride = 0;
  std::vector<int> S, cfg_g, cfg_r, cfg_u;   // [T], [T*stride] x3
  std::vector<int32_t> dense;                // the loaded runtime table [T][U][Gmax]
  int U = 0, Gmax = 0;
  int NN = 0, GP = 0;
  bool sorted_ok = false;
  int decoder = SATURN_DECODER_AUTO;
  uint32_t enum_options = 0;
  Arena arena;                // bound caller workspace (saturn_bind_workspace), or none
  DevBuf<uint8_t> blob;
  int blob_bytes = 0;
  void* pinned = nullptr;     // pinned host staging for the table upload
  size_t pinned_bytes = 0;
  Problem pb{};
  // workspaces
  DevBuf<uint8_t> ws_cfg, ws_perm;
  DevBuf<int32_t> ws_ms;
  DevBuf<unsigned long long> ws_key;
  DevBuf<saturn_placement> ws_place;
  DevBuf<uint8_t> pop[2];
  DevBuf<int32_t> pms[2];
  DevBuf<unsigned long long> cand;
  DevBuf<int> n_cand;
  DevBuf<int> flag;
  DevBuf<uint8_t> ls_gen;
  DevBuf<int32_t> ls_ms;
  DevBuf<int32_t> rec_ms, all_ms;
  DevBuf<uint8_t> rec_gen, all_gen, seeds;
  DevBuf<int> sink;
  // results
  bool have_best = false;
  std::vector<uint8_t> best_cfg, best_perm;
  int64_t best_ms = -1;
  bool have_pop = false;
  int last_pop = 0;
  int64_t pop_P = 0;
  int pop_GS = 0;
  // the last search's position (saturn_search_save / saturn_search_resume)
  int64_t last_gen = 0;
  uint64_t last_seed = 0;
  int last_E = 0, last_world = 1;
  uint32_t last_island = 0;
  std::vector<double> hist_t;
  std::vector<int64_t> hist_ms;
  // best-so-far records in flight: async D2H copies into pinned slots + an event each, read
  // back at the end of the search (no host round trip per epoch)
  static constexpr int HIST_SLOTS = 256;
  int32_t* hist_pin = nullptr;
  std::vector<cudaEvent_t> hist_ev;   // [0] = start of the search, [1 + k] = record k
  int hist_n = 0;
  // communicator: NCCL, or the peer-memory link (one of the two)
  ncclComm_t comm = nullptr;
  std::unique_ptr<sat::PeerLink> peers;
  int rank = 0, world = 1;
  // measurement
  int profiling = 0;          // 0: off; n >= 1: time every n-th GA generation with CUDA events
  saturn_stats stats{};
  std::vector<cudaEvent_t> ev_pool;
  std::string err;
};

namespace {

// Every device buffer the handle owns (table blob and workspaces; the peer-link exchange
// buffers live in PeerLink: CUDA IPC needs their own allocations).
template <class F>
void for_each_buf(saturn_plan* p, F f) {
  f(p->blob);
  f(p->ws_cfg);
  f(p->ws_perm);
  f(p->ws_ms);
  f(p->ws_key);
  f(p->ws_place);
  for (int b = 0; b < 2; ++b) {
    f(p->pop[b]);
    f(p->pms[b]);
  }
  f(p->cand);
  f(p->n_cand);
  f(p->flag);
  f(p->ls_gen);
  f(p->ls_ms);
  f(p->rec_ms);
  f(p->all_ms);
  f(p->rec_gen);
  f(p->all_gen);
  f(p->seeds);
  f(p->sink);
}

}  // namespace

namespace {

saturn_status fail(saturn_plan* p, saturn_status s, const char* fmt, ...) {
  if (p) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    p->err = buf;
  }
  return s;
}

#define CU(p, call)                                                                                   \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ == cudaErrorMemoryAllocation && (p)->arena.bound())                                        \
      return fail(p, SATURN_ELIMIT, "bound workspace exhausted (%zu of %zu B in use) at %s; size it "   \
                  "with saturn_workspace_bytes", (p)->arena.off, (p)->arena.size, #call);             \
    if (e_ != cudaSuccess) return fail(p, SATURN_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));     \
  } while (0)

#define NC(p, call)                                                                                   \
  do {                                                                                                \
    ncclResult_t r_ = (call);                                                                         \
    if (r_ != ncclSuccess) return fail(p, SATURN_ENCCL, "%s: %s", #call, nccl().getErrorString(r_)); \
  } while (0)

int pow2_at_least(int x) {
  int v = 1;
  while (v < x) v <<= 1;
  return v;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int gs_of(int T) { return sat::record_bytes(T); }  // cfg | pad | perm | pad

// Decoder shape of the search-side kernels (GA, local search, index-order enumeration):
// the load-time shape, or node vectors in shared memory (NN = 0) when the caller selected
// SATURN_DECODER_NODE_SMEM.
void run_shape(const saturn_plan* p, int* nn, int* gp) {
  if (p->decoder == SATURN_DECODER_NODE_SMEM) {
    *nn = 0;
    *gp = std::max(4, p->GP);
  } else {
    *nn = p->NN;
    *gp = p->GP;
  }
}

// Decoder shape for the evaluate kernel: the search-side shape (multi-node states are in
// shared memory in every kernel since r2, so evaluate needs no shape of its own).
void eval_shape(const saturn_plan* p, int* nn, int* gp) { run_shape(p, nn, gp); }

bool host_only(saturn_plan* p) {
  if (p->device < 0) {
    fail(p, SATURN_ESTATE, "host-only handle (created with cuda_device = -1)");
    return true;
  }
  return false;
}

saturn_status use_decoder_kind(saturn_plan* p, int* kind) {
  if (host_only(p)) return SATURN_ESTATE;
  int k = p->decoder;
  if (k == SATURN_DECODER_NODE_SMEM) k = SATURN_DECODER_THREAD;   // (shape from eval_shape)
  if (k == SATURN_DECODER_AUTO) k = p->sorted_ok ? SATURN_DECODER_THREAD : SATURN_DECODER_WARP;
  if (k == SATURN_DECODER_THREAD && !p->sorted_ok)
    return fail(p, SATURN_EINVAL, "thread decoder not compiled for %d nodes x %d GPUs (padded)", p->NN, p->GP);
  *kind = k;
  return SATURN_OK;
}

}  // namespace

extern "C" {

saturn_status saturn_plan_create(const int32_t* node_gpus, int32_t n_nodes, int32_t cuda_device, saturn_plan** out) {
  if (!out) return SATURN_EINVAL;
  *out = nullptr;
  if (!node_gpus || n_nodes < 1 || n_nodes > sat::MAX_NODES) return SATURN_EINVAL;
  int sum = 0, mx = 0;
  for (int n = 0; n < n_nodes; ++n) {
    if (node_gpus[n] < 1) return SATURN_EINVAL;
    sum += node_gpus[n];
    mx = std::max(mx, (int)node_gpus[n]);
  }
  if (sum > sat::MAX_GPUS) return SATURN_EINVAL;
  if (cuda_device == -1) {  // host-only handle
    saturn_plan* p = new saturn_plan();
    p->device = -1;
    p->gpu_n.assign(node_gpus, node_gpus + n_nodes);
    p->sumG = sum;
    p->maxG = mx;
    *out = p;
    return SATURN_OK;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) {
    cudaGetLastError();
    return SATURN_ECUDA;
  }
  saturn_plan* p = new saturn_plan();
  p->device = cuda_device;
  for_each_buf(p, [p](auto& b) { b.arena = &p->arena; });
  p->gpu_n.assign(node_gpus, node_gpus + n_nodes);
  p->sumG = sum;
  p->maxG = mx;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cuda_device) != cudaSuccess) {
    delete p;
    return SATURN_ECUDA;
  }
  p->sms = prop.multiProcessorCount;
  *out = p;
  return SATURN_OK;
}

// Device bytes one search with `sp` (NULL: evaluate / enumerate / best_plan only) needs from
// a freshly bound workspace: the table blob, the trace and enumeration scratch, and -- for a
// search -- two populations, their makespans, the candidate list, the elite records and the
// seed genomes.  Every buffer is rounded up to ARENA_ALIGN bytes as the arena carves it.
saturn_status saturn_workspace_bytes(const saturn_plan* pc, const saturn_search_params* sp, uint64_t* bytes) {
  saturn_plan* p = const_cast<saturn_plan*>(pc);
  if (!p || !bytes) return SATURN_EINVAL;
  if (host_only(p)) return fail(p, SATURN_ESTATE, "host-only handle has no device workspace");
  if (!p->loaded) return fail(p, SATURN_ESTATE, "workspace_bytes before load_runtime_table");
  const int T = p->T;
  size_t b = arena_round(p->blob_bytes);
  b += 2 * arena_round(T) + arena_round(4) + arena_round((size_t)T * sizeof(saturn_placement));   // trace
  b += arena_round(3 * 8) + arena_round(4);                                                     // keys, flag
  if (sp) {
    const int64_t P = sp->population;
    const int E = sp->elites;
    if (P < 64 || P < 2 * E || P > (int64_t(1) << 31) - 1 || E < 1 || E > 32)
      return fail(p, SATURN_EINVAL, "population=%lld / elites=%d out of range", (long long)P, E);
    const int GS = gs_of(T);
    const int world = std::max(p->world, 1);
    DeviceGuard dg(p->device);
    int rnn, rgp;
    run_shape(p, &rnn, &rgp);
    const size_t cand = (size_t)sat::ga_max_candidates(p->pb, rnn, rgp, E, GS, P, p->sms) + 64;
    b += 2 * arena_round((size_t)P * GS) + 2 * arena_round((size_t)P * 4) + arena_round(cand * 8) + arena_round(8);
    b += arena_round((size_t)E * 4) + arena_round((size_t)E * GS) + arena_round((size_t)E * world * 4) +
         arena_round((size_t)E * GS * world);
    if (sp->n_seed > 0) b += arena_round((size_t)std::min<int64_t>(sp->n_seed, P) * GS);
  }
  *bytes = b;
  return SATURN_OK;
}

// Bind (d_workspace != NULL) or unbind (NULL) a caller-owned device workspace.  Binding drops
// every workspace buffer the handle holds (populations and search results become invalid:
// search again) and re-homes the loaded table into the workspace.
saturn_status saturn_bind_workspace(saturn_plan* p, void* d_workspace, uint64_t bytes) {
  if (!p) return SATURN_EINVAL;
  if (host_only(p)) return fail(p, SATURN_ESTATE, "host-only handle has no device workspace");
  DeviceGuard dg(p->device);
  if (d_workspace) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, d_workspace) != cudaSuccess || a.type != cudaMemoryTypeDevice ||
        a.device != p->device) {
      cudaGetLastError();
      return fail(p, SATURN_EINVAL, "workspace is not device memory of device %d", p->device);
    }
    if (reinterpret_cast<uintptr_t>(d_workspace) % ARENA_ALIGN)
      return fail(p, SATURN_EINVAL, "workspace must be %zu-byte aligned", ARENA_ALIGN);
  }
  CU(p, cudaDeviceSynchronize());   // nothing in flight may still use the old buffers
  std::vector<uint8_t> blob;
  if (p->loaded && p->blob.p) {
    blob.resize(p->blob_bytes);
    CU(p, cudaMemcpy(blob.data(), p->blob.p, p->blob_bytes, cudaMemcpyDeviceToHost));
  }
  for_each_buf(p, [](auto& b) { b.release(); });
  p->arena = Arena{};
  if (d_workspace) {
    p->arena.base = static_cast<uint8_t*>(d_workspace);
    p->arena.size = bytes;
  }
  p->have_pop = false;
  if (!blob.empty()) {
    CU(p, p->blob.ensure(blob.size()));
    CU(p, cudaMemcpy(p->blob.p, blob.data(), blob.size(), cudaMemcpyHostToDevice));
    p->pb.blob = p->blob.p;
  }
  return SATURN_OK;
}

saturn_status saturn_load_runtime_table(saturn_plan* p, const int32_t* runtime_s, int32_t n_jobs, int32_t n_upps,
                                        int32_t max_gpus) {
  if (!p) return SATURN_EINVAL;
  if (!runtime_s) return fail(p, SATURN_EINVAL, "runtime_s is NULL");
  if (n_jobs < 1 || n_jobs > sat::MAX_JOBS) return fail(p, SATURN_EINVAL, "n_jobs=%d not in [1,255]", n_jobs);
  if (n_upps < 1 || n_upps > 255) return fail(p, SATURN_EINVAL, "n_upps=%d not in [1,255]", n_upps);
  if (max_gpus < 1) return fail(p, SATURN_EINVAL, "max_gpus=%d < 1", max_gpus);
  p->loaded = false;
  p->have_best = false;
  p->have_pop = false;
  const int T = n_jobs;
  std::vector<std::vector<int>> gs(T), rs(T), us(T);
  int64_t sum_max = 0;
  for (int t = 0; t < T; ++t) {
    int rmax = 0;
    for (int u = 0; u < n_upps; ++u)
      for (int g = 1; g <= max_gpus; ++g) {
        const int32_t r = runtime_s[((int64_t)t * n_upps + u) * max_gpus + (g - 1)];
        if (r <= 0 || g > p->maxG) continue;
        if (r >= (1 << 24))
          return fail(p, SATURN_EINVAL, "runtime[%d][%d][%d]=%d >= 2^24 s", t, u, g - 1, r);
        gs[t].push_back(g);
        rs[t].push_back(r);
        us[t].push_back(u);
        rmax = std::max(rmax, (int)r);
      }
    if (gs[t].empty())
      return fail(p, SATURN_EUNSCHEDULABLE, "job %d has no feasible configuration fitting a node", t);
    if (gs[t].size() > 255) return fail(p, SATURN_EINVAL, "job %d has %zu > 255 configurations", t, gs[t].size());
    sum_max += rmax;
  }
  if (sum_max >= (int64_t(1) << 26))
    return fail(p, SATURN_EINVAL, "sum of per-job max runtimes %lld >= 2^26 s", (long long)sum_max);
  int stride = 0;  // max_t S_t plus one zero sentinel column (invalid genes decode to it)
  for (int t = 0; t < T; ++t) stride = std::max(stride, (int)gs[t].size() + 1);
  const int NG = (int)p->gpu_n.size();
  const int raw = 4 * T * stride + T + NG + T * stride;   // tab | S | GPU_n | upp
  const int bytes = (raw + 15) & ~15;
  if (bytes > 48 * 1024) return fail(p, SATURN_ELIMIT, "packed table %d B > 48 KB", bytes);
  std::unique_ptr<DeviceGuard> dg;
  if (p->device >= 0) dg.reset(new DeviceGuard(p->device));

  std::vector<uint8_t> blob(bytes, 0);
  uint32_t* tab = reinterpret_cast<uint32_t*>(blob.data());
  uint8_t* Sb = blob.data() + 4 * T * stride;
  uint8_t* Gb = Sb + T;     // GPU_n per node (decoders index it with a runtime node id)
  uint8_t* upp = Gb + NG;
  for (int n = 0; n < NG; ++n) Gb[n] = (uint8_t)p->gpu_n[n];
  p->S.assign(T, 0);
  p->cfg_g.assign(T * stride, 0);
  p->cfg_r.assign(T * stride, 0);
  p->cfg_u.assign(T * stride, -1);
  for (int t = 0; t < T; ++t) {
    p->S[t] = (int)gs[t].size();
    Sb[t] = (uint8_t)gs[t].size();
    for (size_t s = 0; s < gs[t].size(); ++s) {
      tab[t * stride + s] = ((uint32_t)gs[t][s] << 24) | (uint32_t)rs[t][s];
      upp[t * stride + s] = (uint8_t)us[t][s];
      p->cfg_g[t * stride + s] = gs[t][s];
      p->cfg_r[t * stride + s] = rs[t][s];
      p->cfg_u[t * stride + s] = us[t][s];
    }
  }
  if (p->device >= 0) {
    // upload through a pinned staging buffer owned by the handle (true DMA, no bounce)
    CU(p, p->blob.ensure(bytes));
    if (p->pinned_bytes < (size_t)bytes) {
      if (p->pinned) cudaFreeHost(p->pinned);
      p->pinned = nullptr;
      p->pinned_bytes = 0;
      CU(p, cudaHostAlloc(&p->pinned, bytes, cudaHostAllocDefault));
      p->pinned_bytes = bytes;
    }
    memcpy(p->pinned, blob.data(), bytes);
    CU(p, cudaMemcpy(p->blob.p, p->pinned, bytes, cudaMemcpyHostToDevice));
    p->stats.h2d_bytes += bytes;
  }
  p->T = T;
  p->stride = stride;
  p->blob_bytes = bytes;
  p->dense.assign(runtime_s, runtime_s + (size_t)T * n_upps * max_gpus);
  p->U = n_upps;
  p->Gmax = max_gpus;
  Problem pb{};
  pb.blob = p->blob.p;
  pb.blob_bytes = std::min(bytes, (4 * T * stride + T + NG + 15) & ~15);   // tab + S + GPU_n (staged by the decoders)
  pb.full_bytes = bytes;
  pb.T = T;
  pb.stride = stride;
  pb.N = (int)p->gpu_n.size();
  pb.sumG = p->sumG;
  for (int n = 0; n < pb.N; ++n) pb.gpu_n[n] = (int8_t)p->gpu_n[n];
  p->pb = pb;
  // Decoder shape: node vectors in registers when that shape is compiled (faster: measured
  // r1 on MIX 2x8 and SWEEP 4x8, profiles/r1/README.md), else node vectors in shared
  // memory with a runtime node count (NN = 0; SATURN_DECODER_NODE_SMEM selects it for any
  // cluster).
  p->GP = std::max(2, pow2_at_least(p->maxG));
  p->NN = 1;
  if (p->gpu_n.size() > 1) {
    const int nn = pow2_at_least((int)p->gpu_n.size());
    if (sat::have_sorted_shape(nn, p->GP)) {
      p->NN = nn;
    } else {
      p->NN = 0;
      p->GP = std::max(4, p->GP);
    }
  }
  p->sorted_ok = sat::have_sorted_shape(p->NN, p->GP);
  // makespan read off the final state (decode_sorted) for one full node: measured r1 TXT
  // evaluate +2.7 %, k_ga -0.8 %; on 2x8 (MIX) the second loop copy cost k_ga 1 %, so
  // multi-node shapes keep the running max
  p->pb.one = 1;
  p->pb.full_nodes = (p->NN == 1 && p->gpu_n.size() == 1 && p->gpu_n[0] == p->GP) ? 1 : 0;
  if (sat::eval_smem_bytes(pb, p->NN, p->GP) > 227 * 1024)
    return fail(p, SATURN_ELIMIT, "evaluate tile exceeds shared memory");
  p->loaded = true;
  return SATURN_OK;
}

saturn_status saturn_num_configs(const saturn_plan* p, int32_t* n_jobs, int32_t* configs_per_job) {
  if (!p) return SATURN_EINVAL;
  if (!p->loaded) return SATURN_ESTATE;
  if (n_jobs) *n_jobs = p->T;
  if (configs_per_job)
    for (int t = 0; t < p->T; ++t) configs_per_job[t] = p->S[t];
  return SATURN_OK;
}

saturn_status saturn_config(const saturn_plan* p, int32_t job, int32_t cfg, int32_t* upp, int32_t* gpus,
                            int32_t* runtime_s) {
  if (!p) return SATURN_EINVAL;
  if (!p->loaded) return SATURN_ESTATE;
  if (job < 0 || job >= p->T || cfg < 0 || cfg >= p->S[job]) return SATURN_EINVAL;
  const int k = job * p->stride + cfg;
  if (upp) *upp = p->cfg_u[k];
  if (gpus) *gpus = p->cfg_g[k];
  if (runtime_s) *runtime_s = p->cfg_r[k];
  return SATURN_OK;
}

saturn_status saturn_set_decoder(saturn_plan* p, int32_t kind) {
  if (!p) return SATURN_EINVAL;
  if (kind < SATURN_DECODER_AUTO || kind > SATURN_DECODER_NODE_SMEM) return fail(p, SATURN_EINVAL, "decoder %d", kind);
  p->decoder = kind;
  return SATURN_OK;
}

saturn_status saturn_evaluate(saturn_plan* p, const uint8_t* d_cfg, const uint8_t* d_perm, int64_t n,
                              int32_t* d_makespan, void* stream) {
  if (!p) return SATURN_EINVAL;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "evaluate before load_runtime_table");
  if (n < 0) return fail(p, SATURN_EINVAL, "n < 0");
  if (n == 0) return SATURN_OK;
  if (!d_cfg || !d_perm || !d_makespan) return fail(p, SATURN_EINVAL, "NULL buffer");
  int kind;
  saturn_status s = use_decoder_kind(p, &kind);
  if (s != SATURN_OK) return s;
  DeviceGuard dg(p->device);
  int enn, egp;
  eval_shape(p, &enn, &egp);
  CU(p, sat::launch_evaluate(p->pb, enn, egp, kind, d_cfg, d_perm, n, d_makespan, p->sms,
                             static_cast<cudaStream_t>(stream)));
  p->stats.kernel_launches += 1;
  return SATURN_OK;
}

saturn_status saturn_evaluate_nodes(saturn_plan* p, const uint8_t* d_cfg, const uint8_t* d_perm,
                                    const uint8_t* d_node, int64_t n, int32_t* d_makespan, void* stream) {
  if (!p) return SATURN_EINVAL;
  if (host_only(p)) return SATURN_ESTATE;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "evaluate before load_runtime_table");
  if (n < 0) return fail(p, SATURN_EINVAL, "n < 0");
  if (n == 0) return SATURN_OK;
  if (!d_cfg || !d_perm || !d_node || !d_makespan) return fail(p, SATURN_EINVAL, "NULL buffer");
  // node genes need a register decoder shape; pick the one for the real node count
  const int nn = pow2_at_least((int)p->gpu_n.size());
  const int gp = std::max(2, pow2_at_least(p->maxG));
  if (!sat::have_sorted_shape(nn, gp))
    return fail(p, SATURN_EINVAL, "node genes need a compiled register shape (%d x %d)", nn, gp);
  DeviceGuard dg(p->device);
  CU(p, sat::launch_evaluate_nodes(p->pb, nn, gp, d_cfg, d_perm, d_node, n, d_makespan, p->sms,
                                   static_cast<cudaStream_t>(stream)));
  p->stats.kernel_launches += 1;
  return SATURN_OK;
}

saturn_status saturn_evaluate_host(saturn_plan* p, const uint8_t* h_cfg, const uint8_t* h_perm, int64_t n,
                                   int32_t* h_makespan, void* stream) {
  if (!p) return SATURN_EINVAL;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "evaluate before load_runtime_table");
  if (n < 0) return fail(p, SATURN_EINVAL, "n < 0");
  if (n == 0) return SATURN_OK;
  if (!h_cfg || !h_perm || !h_makespan) return fail(p, SATURN_EINVAL, "NULL buffer");
  int kind;
  saturn_status s = use_decoder_kind(p, &kind);
  if (s != SATURN_OK) return s;
  DeviceGuard dg(p->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t chunk = std::min<int64_t>(n, int64_t(1) << 24);
  CU(p, p->ws_cfg.ensure(chunk * p->T));
  CU(p, p->ws_perm.ensure(chunk * p->T));
  CU(p, p->ws_ms.ensure(chunk));
  for (int64_t off = 0; off < n; off += chunk) {
    const int64_t m = std::min(chunk, n - off);
    CU(p, cudaMemcpyAsync(p->ws_cfg.p, h_cfg + off * p->T, m * p->T, cudaMemcpyHostToDevice, st));
    CU(p, cudaMemcpyAsync(p->ws_perm.p, h_perm + off * p->T, m * p->T, cudaMemcpyHostToDevice, st));
    int enn, egp;
    eval_shape(p, &enn, &egp);
    CU(p, sat::launch_evaluate(p->pb, enn, egp, kind, p->ws_cfg.p, p->ws_perm.p, m, p->ws_ms.p, p->sms, st));
    CU(p, cudaMemcpyAsync(h_makespan + off, p->ws_ms.p, m * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    p->stats.kernel_launches += 1;
    p->stats.h2d_bytes += 2 * m * p->T;
    p->stats.d2h_bytes += m * (int64_t)sizeof(int32_t);
  }
  CU(p, cudaStreamSynchronize(st));
  return SATURN_OK;
}

saturn_status saturn_trace(saturn_plan* p, const uint8_t* d_cfg, const uint8_t* d_perm, int64_t n,
                           saturn_placement* d_placements, int32_t* d_makespan, void* stream) {
  if (p && host_only(p)) return SATURN_ESTATE;
  if (!p) return SATURN_EINVAL;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "trace before load_runtime_table");
  if (n < 0) return fail(p, SATURN_EINVAL, "n < 0");
  if (n == 0) return SATURN_OK;
  if (!d_cfg || !d_perm || !d_placements || !d_makespan) return fail(p, SATURN_EINVAL, "NULL buffer");
  DeviceGuard dg(p->device);
  CU(p, sat::launch_trace(p->pb, d_cfg, d_perm, n, d_placements, d_makespan, p->sms,
                          static_cast<cudaStream_t>(stream)));
  p->stats.kernel_launches += 1;
  return SATURN_OK;
}

saturn_status saturn_space_size(const saturn_plan* p, uint64_t* size) {
  if (!p || !size) return SATURN_EINVAL;
  if (!p->loaded) return SATURN_ESTATE;
  unsigned __int128 v = 1;
  for (int k = 2; k <= p->T; ++k) {
    v *= (unsigned)k;
    if (v >> 64) return SATURN_ELIMIT;
  }
  for (int t = 0; t < p->T; ++t) {
    v *= (unsigned)p->S[t];
    if (v >> 64) return SATURN_ELIMIT;
  }
  *size = (uint64_t)v;
  return SATURN_OK;
}

namespace {

// Host unrank of a genome index (same definition as the device kernel; used only to
// materialise the winner for best_plan).
void unrank_host(const saturn_plan* p, uint64_t G, std::vector<uint8_t>& cfg, std::vector<uint8_t>& perm) {
  const int T = p->T;
  uint64_t cs = 1;
  for (int t = 0; t < T; ++t) cs *= (uint64_t)p->S[t];
  uint64_t rc = G % cs, rp = G / cs;
  cfg.assign(T, 0);
  perm.assign(T, 0);
  for (int t = 0; t < T; ++t) {
    cfg[t] = (uint8_t)(rc % (uint64_t)p->S[t]);
    rc /= (uint64_t)p->S[t];
  }
  std::vector<int> avail(T);
  for (int t = 0; t < T; ++t) avail[t] = t;
  for (int i = 0; i < T; ++i) {
    uint64_t f = 1;
    for (int k = 2; k <= T - 1 - i; ++k) f *= (uint64_t)k;
    const uint64_t d = rp / f;
    rp %= f;
    perm[i] = (uint8_t)avail[d];
    avail.erase(avail.begin() + (long)d);
  }
}

// ---- peer-memory exchange helpers (row e without NCCL; peers.h)
bool distributed(const saturn_plan* p) { return p->world > 1 && (p->comm || p->peers); }

// MIN of key[0] and SUM of key[1] over the ranks: push this rank's pair into slot `rank` of
// every rank's exchange buffer, barrier, reduce the own buffer's slots on the host, barrier
// (so the next call's pushes cannot overtake a slow reader).  `key` is device memory [2].
saturn_status peer_reduce_keys(saturn_plan* p, unsigned long long* key, cudaStream_t st,
                               unsigned long long out[2]) {
  sat::PeerLink& L = *p->peers;
  for (int q = 0; q < L.world; ++q)
    CU(p, cudaMemcpyAsync(L.peer[q] + sat::PeerLayout::keys + 16 * L.rank, key, 16, cudaMemcpyDeviceToDevice, st));
  CU(p, L.wait_stream(st));
  if (!L.barrier()) return fail(p, SATURN_ECUDA, "%s", L.err.c_str());
  unsigned long long all[2 * sat::PEER_MAX];
  CU(p, cudaMemcpy(all, L.local + sat::PeerLayout::keys, 16 * L.world, cudaMemcpyDeviceToHost));
  out[0] = ~0ull;
  out[1] = 0;
  for (int q = 0; q < L.world; ++q) {
    out[0] = std::min(out[0], all[2 * q]);
    out[1] += all[2 * q + 1];
  }
  if (!L.barrier()) return fail(p, SATURN_ECUDA, "%s", L.err.c_str());
  return SATURN_OK;
}

// Fused enumeration collective over peer memory: the enumeration kernel of every rank folds
// its best (makespan << 38 | index) key with atomicMin -- and its leaf count with atomicAdd
// -- straight into ONE slot pair in rank 0's exchange buffer (a remote atomic over NVLink
// for the other GPUs), and the DFS reads that slot as its live branch-and-bound incumbent,
// so every rank prunes with every rank's best.  begin: rank 0 initialises the pair, barrier;
// end: barrier after all kernels, read the pair, barrier (before the next call re-inits).
// DFS roots by the static grid stride (measured r1: batches of roots claimed from a counter
// were slower -- 7 jobs on 1x4: 4.7 vs 3.7 ms -- consecutive roots find the good leaves later,
// the shared incumbent tightens later and 30 % more leaves are visited).
unsigned long long* peer_shared_slot(saturn_plan* p) {
  return reinterpret_cast<unsigned long long*>(p->peers->peer[0] + sat::PeerLayout::shared);
}
saturn_status peer_shared_begin(saturn_plan* p, const unsigned long long init[2], cudaStream_t st) {
  sat::PeerLink& L = *p->peers;
  if (L.rank == 0) {
    CU(p, cudaMemcpyAsync(peer_shared_slot(p), init, 16, cudaMemcpyHostToDevice, st));
    CU(p, L.wait_stream(st));
  }
  if (!L.barrier()) return fail(p, SATURN_ECUDA, "%s", L.err.c_str());
  return SATURN_OK;
}
saturn_status peer_shared_end(saturn_plan* p, cudaStream_t st, unsigned long long out[2]) {
  sat::PeerLink& L = *p->peers;
  CU(p, L.wait_stream(st));
  if (!L.barrier()) return fail(p, SATURN_ECUDA, "%s", L.err.c_str());
  CU(p, cudaMemcpy(out, peer_shared_slot(p), 16, cudaMemcpyDeviceToHost));
  if (!L.barrier()) return fail(p, SATURN_ECUDA, "%s", L.err.c_str());
  return SATURN_OK;
}

saturn_status enumerate_impl(saturn_plan* p, uint64_t begin, uint64_t end, uint64_t total, bool collective,
                             cudaStream_t st, saturn_result* out) {
  const double t0 = now_s();
  sat::EnumSpace es{};
  es.cfg_space = 1;
  for (int t = 0; t < p->T; ++t) {
    es.radix[t] = es.cfg_space;
    es.cfg_space *= (uint64_t)p->S[t];
  }
  es.fact[0] = 1;
  for (int k = 1; k <= p->T; ++k) es.fact[k] = es.fact[k - 1] * (uint64_t)k;
  int kind;
  saturn_status s = use_decoder_kind(p, &kind);
  if (s != SATURN_OK) return s;
  if (kind != SATURN_DECODER_THREAD)
    return fail(p, SATURN_EINVAL, "enumerate needs the thread decoder for this cluster shape");
  unsigned long long key = 0;
  p->stats.d2h_bytes += 8;
  if (collective && p->peers && p->world > 1) {   // fused: the kernel reduces into rank 0's slot
    const unsigned long long init[2] = {~0ull, 0ull};
    saturn_status sr = peer_shared_begin(p, init, st);
    if (sr != SATURN_OK) return sr;
    int enn, egp;
    run_shape(p, &enn, &egp);
    CU(p, sat::launch_enumerate(p->pb, enn, egp, es, begin, end, peer_shared_slot(p), p->sms, st));
    p->stats.kernel_launches += 1;
    unsigned long long r[2];
    sr = peer_shared_end(p, st, r);
    if (sr != SATURN_OK) return sr;
    key = r[0];
  } else {
    CU(p, p->ws_key.ensure(1));
    CU(p, cudaMemsetAsync(p->ws_key.p, 0xff, sizeof(unsigned long long), st));
    int enn, egp;
    run_shape(p, &enn, &egp);
    CU(p, sat::launch_enumerate(p->pb, enn, egp, es, begin, end, p->ws_key.p, p->sms, st));
    p->stats.kernel_launches += 1;
    if (collective && p->comm) {
      NC(p, nccl().allReduce(p->ws_key.p, p->ws_key.p, 1, ncclUint64, ncclMin, p->comm, st));
    }
    CU(p, cudaMemcpyAsync(&key, p->ws_key.p, sizeof key, cudaMemcpyDeviceToHost, st));
    CU(p, cudaStreamSynchronize(st));
  }
  if (out) {
    memset(out, 0, sizeof *out);
    out->evaluated = collective ? total : (end - begin);
    out->leaves = out->evaluated;
    out->seconds = now_s() - t0;
    out->flags = SATURN_PROVEN_OPTIMAL;
  }
  if (key == ~0ull) {  // empty range
    if (out) out->makespan = -1;
    return SATURN_OK;
  }
  const uint64_t idx = key & ((uint64_t(1) << 38) - 1);
  const int64_t ms = (int64_t)(key >> 38);
  unrank_host(p, idx, p->best_cfg, p->best_perm);
  p->best_ms = ms;
  p->have_best = true;
  if (out) {
    out->makespan = ms;
    out->genome_index = idx;
  }
  return SATURN_OK;
}

}  // namespace

// Full-space enumeration with the DFS kernel: roots partitioned over ranks, incumbent seeded
// with the best paper-baseline genome (any valid genome's makespan >= OPT, so the strict cut
// keeps every optimal leaf and the smallest-index tie-break stays exact).
static saturn_status enumerate_dfs_impl(saturn_plan* p, uint64_t total, cudaStream_t st, saturn_result* out) {
  const double t0 = now_s();
  const int T = p->T;
  sat::DfsSpace ds{};
  ds.es.cfg_space = 1;
  for (int t = 0; t < T; ++t) {
    ds.es.radix[t] = ds.es.cfg_space;
    ds.es.cfg_space *= (uint64_t)p->S[t];
  }
  ds.es.fact[0] = 1;
  for (int k = 1; k <= T; ++k) ds.es.fact[k] = ds.es.fact[k - 1] * (uint64_t)k;
  ds.pre[0] = 0;
  for (int t = 0; t < T; ++t) ds.pre[t + 1] = ds.pre[t] + p->S[t];
  ds.sumS = ds.pre[T];
  // symmetry reduction: twin = same (g, R) list; each job waits for its previous twin
  bool reduced = false;
  for (int t = 0; t < T; ++t) {
    ds.twin_prev[t] = 0;
    if (!(p->enum_options & SATURN_ENUM_SYMMETRY)) continue;
    for (int u = t - 1; u >= 0 && !ds.twin_prev[t]; --u) {
      bool same = p->S[u] == p->S[t];
      for (int c = 0; same && c < p->S[t]; ++c)
        same = p->cfg_g[u * p->stride + c] == p->cfg_g[t * p->stride + c] &&
               p->cfg_r[u * p->stride + c] == p->cfg_r[t * p->stride + c];
      if (same) ds.twin_prev[t] = 1u << u;
    }
    reduced |= ds.twin_prev[t] != 0;
  }
  // root depth: enough roots to fill the GPU (~32 per SM-thread slot), at most T - 1 levels
  ds.D = 1;
  ds.n_roots = (uint64_t)ds.sumS;
  const uint64_t want = (uint64_t)p->sms * 64 * 16;
  while (ds.D < T - 1 && ds.n_roots < want && ds.n_roots * (uint64_t)ds.sumS < (uint64_t(1) << 40)) {
    ds.n_roots *= (uint64_t)ds.sumS;
    ++ds.D;
  }
  // incumbent from the paper's baselines (row f2)
  int32_t inc = (int32_t)((1 << 26) - 1);
  {
    std::vector<uint8_t> c(4 * T), q(4 * T);
    for (int k = 0; k < 4; ++k) {
      saturn_status sb = saturn_baseline_genome(p, k + 1, 0, &c[k * T], &q[k * T]);
      if (sb != SATURN_OK) return sb;
    }
    int32_t ms[4];
    saturn_status se = saturn_evaluate_host(p, c.data(), q.data(), 4, ms, st);
    if (se != SATURN_OK) return se;
    for (int k = 0; k < 4; ++k)
      if (ms[k] > 0) inc = std::min(inc, ms[k]);
  }
  const unsigned long long init = ((unsigned long long)inc << 38) | ((1ull << 38) - 1ull);
  uint64_t rb = 0, re = ds.n_roots;
  saturn_partition(ds.n_roots, p->rank, p->world, &rb, &re);
  unsigned long long kl[2] = {0, 0};
  if (p->peers && p->world > 1) {   // fused: live shared incumbent + reduction in rank 0's slot
    const unsigned long long iv[2] = {init, 0ull};
    saturn_status sr = peer_shared_begin(p, iv, st);
    if (sr != SATURN_OK) return sr;
    unsigned long long* g = peer_shared_slot(p);
    CU(p, p->ws_key.ensure(3));
    CU(p, cudaMemsetAsync(p->ws_key.p + 2, 0, sizeof(unsigned long long), st));   // this rank's root counter
    CU(p, sat::launch_enumerate_dfs(p->pb, p->NN, p->GP, ds, rb, re, g, g + 1, p->sms, st));
    p->stats.kernel_launches += 1;
    sr = peer_shared_end(p, st, kl);
    if (sr != SATURN_OK) return sr;
  } else {
    CU(p, p->ws_key.ensure(3));
    CU(p, cudaMemcpyAsync(p->ws_key.p, &init, sizeof init, cudaMemcpyHostToDevice, st));
    CU(p, cudaMemsetAsync(p->ws_key.p + 1, 0, 2 * sizeof(unsigned long long), st));   // leaves, root counter
    CU(p, sat::launch_enumerate_dfs(p->pb, p->NN, p->GP, ds, rb, re, p->ws_key.p, p->ws_key.p + 1, p->sms, st));
    p->stats.kernel_launches += 1;
    if (p->comm && p->world > 1) {
      NC(p, nccl().allReduce(p->ws_key.p, p->ws_key.p, 1, ncclUint64, ncclMin, p->comm, st));
      NC(p, nccl().allReduce(p->ws_key.p + 1, p->ws_key.p + 1, 1, ncclUint64, ncclSum, p->comm, st));
    }
    CU(p, cudaMemcpyAsync(kl, p->ws_key.p, sizeof kl, cudaMemcpyDeviceToHost, st));
    CU(p, cudaStreamSynchronize(st));
  }
  p->stats.d2h_bytes += sizeof kl;
  const uint64_t idx = kl[0] & ((uint64_t(1) << 38) - 1);
  if (idx == (uint64_t(1) << 38) - 1) return fail(p, SATURN_ECUDA, "enumeration found no leaf");
  const int64_t ms = (int64_t)(kl[0] >> 38);
  unrank_host(p, idx, p->best_cfg, p->best_perm);
  p->best_ms = ms;
  p->have_best = true;
  if (out) {
    memset(out, 0, sizeof *out);
    out->makespan = ms;
    out->genome_index = idx;
    out->evaluated = 0;   // no full T-step decode: leaves are prefix-shared, pruned plans not counted (§8d)
    out->leaves = kl[1];
    out->seconds = now_s() - t0;
    out->flags = SATURN_PROVEN_OPTIMAL | SATURN_PREFIX_SHARED | (reduced ? SATURN_SYMMETRY_REDUCED : 0);
  }
  return SATURN_OK;
}

saturn_status saturn_enumerate(saturn_plan* p, uint64_t max_genomes, void* stream, saturn_result* out) {
  Nvtx r("saturn_enumerate");
  if (!p) return SATURN_EINVAL;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "enumerate before load_runtime_table");
  if (p->T > sat::ENUM_MAX_T) return fail(p, SATURN_ELIMIT, "T=%d > %d jobs for enumeration", p->T, sat::ENUM_MAX_T);
  uint64_t size = 0;
  if (saturn_space_size(p, &size) != SATURN_OK || size >= (uint64_t(1) << 38))
    return fail(p, SATURN_ELIMIT, "genome space too large for enumeration (>= 2^38)");
  if (size > max_genomes)
    return fail(p, SATURN_ELIMIT, "genome space %llu exceeds max_genomes %llu", (unsigned long long)size,
                (unsigned long long)max_genomes);
  DeviceGuard dg(p->device);
  int kind;
  saturn_status s0 = use_decoder_kind(p, &kind);
  if (s0 != SATURN_OK) return s0;
  if (p->T >= 3 && p->NN >= 1 && p->decoder != SATURN_DECODER_NODE_SMEM)
    return enumerate_dfs_impl(p, size, static_cast<cudaStream_t>(stream), out);
  uint64_t b = 0, e = size;
  saturn_partition(size, p->rank, p->world, &b, &e);
  return enumerate_impl(p, b, e, size, true, static_cast<cudaStream_t>(stream), out);
}

saturn_status saturn_set_enumeration_options(saturn_plan* p, uint32_t options) {
  if (!p) return SATURN_EINVAL;
  if (options & ~(uint32_t)SATURN_ENUM_SYMMETRY) return fail(p, SATURN_EINVAL, "unknown option bits 0x%x", options);
  p->enum_options = options;
  return SATURN_OK;
}

saturn_status saturn_enumerate_range(saturn_plan* p, uint64_t begin, uint64_t end, void* stream, saturn_result* out) {
  if (!p) return SATURN_EINVAL;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "enumerate before load_runtime_table");
  if (p->T > sat::ENUM_MAX_T) return fail(p, SATURN_ELIMIT, "T=%d > %d jobs for enumeration", p->T, sat::ENUM_MAX_T);
  uint64_t size = 0;
  if (saturn_space_size(p, &size) != SATURN_OK || size >= (uint64_t(1) << 38))
    return fail(p, SATURN_ELIMIT, "genome space too large for enumeration (>= 2^38)");
  if (begin > end || end > size) return fail(p, SATURN_EINVAL, "range [%llu,%llu) outside [0,%llu)",
                                             (unsigned long long)begin, (unsigned long long)end,
                                             (unsigned long long)size);
  DeviceGuard dg(p->device);
  return enumerate_impl(p, begin, end, size, false, static_cast<cudaStream_t>(stream), out);
}

namespace {

// One GA island's search state (row a7 + e).  saturn_search drives one island per process
// (exchanging elites over NCCL when a communicator is attached); saturn_search_group drives
// several islands in lock-step in one process and exchanges by device copies -- the same
// algorithm, so the island protocol is testable on one GPU.
struct Island {
  saturn_plan* p = nullptr;
  const saturn_search_params* sp = nullptr;
  cudaStream_t st = nullptr;
  uint32_t island = 0;      // Philox rank id of this island
  int world = 1;            // number of islands in the exchange
  int64_t P = 0;
  int E = 0, GS = 0, T = 0;
  int NN = 0, GP = 0;   // decoder shape of this search (run_shape)
  sat::GaParams gp{};
  uint64_t evaluated = 0;
  int cur = 0;
  int64_t n_prof = 0, n_timed = 0;
  double t0 = 0;
  const uint8_t* resume = nullptr;   // saved state payload (saturn_search_resume), or none
  int64_t gen0 = 0;                  // generation the state was saved at

  saturn_status validate() {
    if (!p->loaded) return fail(p, SATURN_ESTATE, "search before load_runtime_table");
    if (!sp) return fail(p, SATURN_EINVAL, "params is NULL");
    P = sp->population;
    E = sp->elites;
    if (E < 1 || E > 32) return fail(p, SATURN_EINVAL, "elites=%d not in [1,32]", E);
    if (P < 64 || P < 2 * E || P > (int64_t(1) << 31) - 1)
      return fail(p, SATURN_EINVAL, "population=%lld must be in [max(64, 2*elites), 2^31)", (long long)P);
    if (sp->max_generations < 0) return fail(p, SATURN_EINVAL, "max_generations < 0");
    if (sp->generations_per_epoch < 1) return fail(p, SATURN_EINVAL, "generations_per_epoch < 1");
    if (sp->n_seed < 0 || (sp->n_seed > 0 && (!sp->seed_cfg || !sp->seed_perm)))
      return fail(p, SATURN_EINVAL, "bad seed genomes");
    if (!p->sorted_ok) return fail(p, SATURN_EINVAL, "search needs the thread decoder for this cluster shape");
    T = p->T;
    GS = gs_of(T);
    for (int64_t i = 0; i < sp->n_seed; ++i) {  // seed genomes must be valid
      std::vector<int> seen(T, 0);
      for (int k = 0; k < T; ++k) {
        const int t = sp->seed_perm[i * T + k];
        if (t >= T || seen[t]++)
          return fail(p, SATURN_EINVAL, "seed genome %lld: perm is not a permutation", (long long)i);
        if (sp->seed_cfg[i * T + t] >= p->S[t])
          return fail(p, SATURN_EINVAL, "seed genome %lld: cfg out of range", (long long)i);
      }
    }
    return SATURN_OK;
  }

  // buffers + generation 0 (seed genomes, then Philox genomes) + the first elite selection
  saturn_status begin() {
    DeviceGuard dg(p->device);
    t0 = now_s();
    if (!p->hist_pin) CU(p, cudaHostAlloc(reinterpret_cast<void**>(&p->hist_pin), sizeof(int32_t) * p->HIST_SLOTS,
                                          cudaHostAllocDefault));
    while ((int)p->hist_ev.size() < 1 + p->HIST_SLOTS) {
      cudaEvent_t e;
      CU(p, cudaEventCreate(&e));
      p->hist_ev.push_back(e);
    }
    p->hist_n = 0;
    CU(p, cudaEventRecord(p->hist_ev[0], st));
    for (int b = 0; b < 2; ++b) {
      CU(p, p->pop[b].ensure((size_t)P * GS));
      CU(p, p->pms[b].ensure((size_t)P));
    }
    run_shape(p, &NN, &GP);
    CU(p, p->cand.ensure((size_t)sat::ga_max_candidates(p->pb, NN, GP, E, GS, P, p->sms) + 64));
    CU(p, p->n_cand.ensure(2));   // [0] appended candidates, [1] the GA kernels' work counter
    CU(p, cudaMemsetAsync(p->n_cand.p, 0, 2 * sizeof(int), st));
    CU(p, p->rec_ms.ensure(E));
    CU(p, p->rec_gen.ensure((size_t)E * GS));
    CU(p, p->all_ms.ensure((size_t)E * world));
    CU(p, p->all_gen.ensure((size_t)E * GS * world));
    const int64_t n_seed = resume ? 0 : std::min<int64_t>(sp->n_seed, P);
    if (n_seed > 0) {
      std::vector<uint8_t> packed((size_t)n_seed * GS, 0);
      for (int64_t i = 0; i < n_seed; ++i) {
        memcpy(&packed[i * GS], sp->seed_cfg + i * T, T);
        memcpy(&packed[i * GS + sat::perm_offset(T)], sp->seed_perm + i * T, T);
      }
      CU(p, p->seeds.ensure(packed.size()));
      CU(p, cudaMemcpyAsync(p->seeds.p, packed.data(), packed.size(), cudaMemcpyHostToDevice, st));
      p->stats.h2d_bytes += (int64_t)packed.size();
    }
    gp = sat::GaParams{};
    gp.seed = sp->seed;
    gp.rank = island;
    gp.gen = 0;
    gp.P = P;
    gp.E = E;
    gp.GS = GS;
    gp.px = sp->p_xover_q32;
    gp.pc = sp->p_cfg_mut_q32;
    gp.pm = sp->p_perm_mut_q32;
    cur = 0;
    if (resume) {   // population, makespans and elite records as saved (payload order)
      gp.gen = (uint32_t)gen0;
      evaluated = 0;
      const uint8_t* q = resume;
      CU(p, cudaMemcpyAsync(p->pop[0].p, q, (size_t)P * GS, cudaMemcpyHostToDevice, st));
      q += (size_t)P * GS;
      CU(p, cudaMemcpyAsync(p->pms[0].p, q, (size_t)P * 4, cudaMemcpyHostToDevice, st));
      q += (size_t)P * 4;
      CU(p, cudaMemcpyAsync(p->rec_ms.p, q, (size_t)E * 4, cudaMemcpyHostToDevice, st));
      q += (size_t)E * 4;
      CU(p, cudaMemcpyAsync(p->rec_gen.p, q, (size_t)E * GS, cudaMemcpyHostToDevice, st));
      p->stats.h2d_bytes += (int64_t)((size_t)P * (GS + 4) + (size_t)E * (GS + 4));
    } else {
      evaluated = (uint64_t)P;
      CU(p, sat::launch_ga_init(p->pb, NN, GP, gp, n_seed ? p->seeds.p : nullptr, n_seed, p->pop[0].p,
                                p->pms[0].p, p->cand.p, p->n_cand.p, p->sms, st));
      CU(p, sat::launch_select(p->cand.p, p->n_cand.p, E, GS, p->pop[0].p, p->rec_ms.p, p->rec_gen.p, st));
      p->stats.kernel_launches += 2;
    }
    // profiling: event triples around every `profiling`-th GA generation kernel (at most 512
    // per search).  An event record between kernels costs a few microseconds of drain, so
    // sampling keeps the instrumented step within ~1 % of the uninstrumented one.
    n_prof = p->profiling ? std::min<int64_t>(sp->max_generations / p->profiling + 1, 512) : 0;
    n_timed = 0;
    while ((int64_t)p->ev_pool.size() < 3 * n_prof) {
      cudaEvent_t e;
      CU(p, cudaEventCreate(&e));
      p->ev_pool.push_back(e);
    }
    p->hist_t.clear();
    p->hist_ms.clear();
    return SATURN_OK;
  }

  saturn_status generation(int64_t gen) {
    DeviceGuard dg(p->device);
    gp.gen = (uint32_t)gen;
    const int nxt = cur ^ 1;
    const int per = p->profiling;
    const bool timed = per > 0 && n_timed < n_prof && (gen % per) == (per / 2) % per;
    const int64_t ti = n_timed;
    if (timed) CU(p, cudaEventRecord(p->ev_pool[3 * ti], st));
    CU(p, sat::launch_ga_generation(p->pb, NN, GP, gp, p->pop[cur].p, p->pms[cur].p, p->rec_ms.p,
                                    p->rec_gen.p, p->pop[nxt].p, p->pms[nxt].p, p->cand.p, p->n_cand.p, p->sms, st));
    if (timed) {
      CU(p, cudaEventRecord(p->ev_pool[3 * ti + 1], st));
      ++n_timed;
    }
    CU(p, sat::launch_select(p->cand.p, p->n_cand.p, E, GS, p->pop[nxt].p, p->rec_ms.p, p->rec_gen.p, st,
                             /*few=*/true));   // generations >= 1 append only keys beating the E-th elite
    p->stats.kernel_launches += 2;
    evaluated += (uint64_t)(P - E);
    cur = nxt;
    return SATURN_OK;
  }

  // memetic step (row f4): improve the E elites, then re-sort them by (ms, position)
  saturn_status memetic() {
    if (sp->local_search_iters <= 0) return SATURN_OK;
    DeviceGuard dg(p->device);
    CU(p, cudaMemcpyAsync(p->all_ms.p, p->rec_ms.p, E * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    CU(p, cudaMemcpyAsync(p->all_gen.p, p->rec_gen.p, (size_t)E * GS, cudaMemcpyDeviceToDevice, st));
    CU(p, sat::launch_local_search(p->pb, NN, GP, p->all_gen.p, p->all_ms.p, E, GS, sp->local_search_iters,
                                   st));
    CU(p, sat::launch_merge_elites(p->all_ms.p, p->all_gen.p, 1, E, GS, p->rec_ms.p, p->rec_gen.p, st));
    p->stats.kernel_launches += 2;
    return SATURN_OK;
  }

  // after all islands' records sit in all_ms / all_gen (W blocks of E): the global best E
  saturn_status merge() {
    DeviceGuard dg(p->device);
    CU(p, sat::launch_merge_elites(p->all_ms.p, p->all_gen.p, world, E, GS, p->rec_ms.p, p->rec_gen.p, st));
    p->stats.kernel_launches += 1;
    return SATURN_OK;
  }

  // Best-so-far after an epoch (the anytime curve, saturn_search_history): an async copy
  // into a pinned slot plus an event; only a time-budgeted search waits for it (its stop
  // decision needs the host clock to match the device).
  saturn_status record() {
    DeviceGuard dg(p->device);
    if (p->hist_n == p->HIST_SLOTS) {
      saturn_status s = flush_history();
      if (s != SATURN_OK) return s;
    }
    const int k = p->hist_n++;
    CU(p, cudaMemcpyAsync(p->hist_pin + k, p->rec_ms.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CU(p, cudaEventRecord(p->hist_ev[1 + k], st));
    p->stats.d2h_bytes += sizeof(int32_t);
    if (sp->time_budget_s > 0) return flush_history();
    return SATURN_OK;
  }

  // Drain the in-flight records: seconds since the search started (device clock, from the
  // event recorded before its first kernel) and the best makespan at that point.
  saturn_status flush_history() {
    CU(p, cudaStreamSynchronize(st));
    for (int k = 0; k < p->hist_n; ++k) {
      float ms = 0.f;
      CU(p, cudaEventElapsedTime(&ms, p->hist_ev[0], p->hist_ev[1 + k]));
      p->hist_t.push_back(1e-3 * ms);
      p->hist_ms.push_back(p->hist_pin[k]);
    }
    p->hist_n = 0;
    return SATURN_OK;
  }

  saturn_status finish(int64_t gens_run, uint64_t world_evaluated, saturn_result* out) {
    DeviceGuard dg(p->device);
    std::vector<uint8_t> g0(GS);
    int32_t best = 0;
    CU(p, cudaMemcpyAsync(g0.data(), p->rec_gen.p, GS, cudaMemcpyDeviceToHost, st));
    CU(p, cudaMemcpyAsync(&best, p->rec_ms.p, sizeof best, cudaMemcpyDeviceToHost, st));
    saturn_status hs = flush_history();   // synchronises the stream
    if (hs != SATURN_OK) return hs;
    p->stats.d2h_bytes += GS + sizeof best;
    for (int64_t g = 1; g <= n_timed; ++g) {
      float ms = 0.f;
      CU(p, cudaEventElapsedTime(&ms, p->ev_pool[3 * (g - 1)], p->ev_pool[3 * (g - 1) + 1]));
      p->stats.ga_kernel_ms += ms;
      p->stats.ga_launches += 1;
      p->stats.ga_decodes += P - E;
    }
    p->best_cfg.assign(g0.begin(), g0.begin() + T);
    p->best_perm.assign(g0.begin() + sat::perm_offset(T), g0.begin() + sat::perm_offset(T) + T);
    p->best_ms = best;
    p->have_best = true;
    p->have_pop = true;
    p->last_pop = cur;
    p->pop_P = P;
    p->pop_GS = GS;
    p->last_gen = gen0 + gens_run;
    p->last_seed = sp->seed;
    p->last_E = E;
    p->last_island = island;
    p->last_world = world;
    if (out) {
      memset(out, 0, sizeof *out);
      out->makespan = best;
      out->evaluated = world_evaluated;
      out->seconds = now_s() - t0;
      out->flags = SATURN_INCUMBENT;
      out->generations = (int32_t)gens_run;
    }
    return SATURN_OK;
  }
};

}  // namespace

namespace {

// The search loop of saturn_search; with `resume` the island starts from a saved state at
// generation gen0 (population, makespans, elites) instead of generation 0, and runs
// generations gen0+1 .. gen0+max_generations -- the Philox streams, epoch boundaries and
// exchanges of those generations are the ones the saved search would have run next.
saturn_status search_run(saturn_plan* p, const saturn_search_params* sp, void* stream, saturn_result* out,
                         const uint8_t* resume, int64_t gen0) {
  Island is;
  is.p = p;
  is.sp = sp;
  is.st = static_cast<cudaStream_t>(stream);
  is.island = (uint32_t)p->rank;
  is.world = distributed(p) ? p->world : 1;
  is.resume = resume;
  is.gen0 = gen0;
  saturn_status s;
  if ((s = is.validate()) != SATURN_OK) return s;
  if ((s = is.begin()) != SATURN_OK) return s;
  cudaStream_t st = is.st;
  const int E = is.E, GS = is.GS;
  // epoch exchange: memetic step, then (multi-GPU) all-gather of every island's elites over
  // NCCL and the device merge -- every island continues from the global best E
  auto exchange = [&]() -> saturn_status {
    saturn_status e;
    if ((e = is.memetic()) != SATURN_OK) return e;
    if (is.world < 2) return SATURN_OK;
    DeviceGuard dg(p->device);
    if (p->peers) {
      // push this island's E records into block `rank` of every rank's exchange buffer
      // (epoch-parity half), barrier, merge the own buffer: the same blocks the NCCL
      // all-gather would have produced
      sat::PeerLink& L = *p->peers;
      if (E > sat::PEER_EMAX || GS > sat::PEER_GSMAX) return fail(p, SATURN_EINVAL, "peer exchange: E or genome too large");
      const int par = (int)(L.exchanges++ & 1);
      const size_t ms_off = sat::PeerLayout::ms0 + par * sat::PeerLayout::ms_bytes;
      const size_t gen_off = sat::PeerLayout::gen0 + par * sat::PeerLayout::gen_bytes;
      for (int q = 0; q < L.world; ++q) {
        CU(p, cudaMemcpyAsync(L.peer[q] + ms_off + (size_t)4 * E * L.rank, p->rec_ms.p, (size_t)4 * E,
                              cudaMemcpyDeviceToDevice, st));
        CU(p, cudaMemcpyAsync(L.peer[q] + gen_off + (size_t)E * GS * L.rank, p->rec_gen.p, (size_t)E * GS,
                              cudaMemcpyDeviceToDevice, st));
      }
      CU(p, L.wait_stream(st));
      if (!L.barrier()) return fail(p, SATURN_ECUDA, "%s", L.err.c_str());
      CU(p, sat::launch_merge_elites(reinterpret_cast<const int32_t*>(L.local + ms_off), L.local + gen_off, L.world,
                                     E, GS, p->rec_ms.p, p->rec_gen.p, st));
      p->stats.kernel_launches += 1;
      return SATURN_OK;
    }
    NC(p, nccl().allGather(p->rec_ms.p, p->all_ms.p, (size_t)E, ncclInt32, p->comm, st));
    NC(p, nccl().allGather(p->rec_gen.p, p->all_gen.p, (size_t)E * GS, ncclUint8, p->comm, st));
    return is.merge();
  };
  {
    Nvtx r("saturn_search: initial population + exchange");
    if (!resume && (s = exchange()) != SATURN_OK) return s;   // a saved state is post-exchange
    if ((s = is.record()) != SATURN_OK) return s;
  }
  int64_t gen = gen0 + 1;
  std::unique_ptr<Nvtx> epoch;
  for (; gen <= gen0 + sp->max_generations; ++gen) {
    if (!epoch) epoch.reset(new Nvtx("saturn_search: epoch"));
    if ((s = is.generation(gen)) != SATURN_OK) return s;
    if (gen % sp->generations_per_epoch == 0) {
      {
        Nvtx r("exchange");
        if ((s = exchange()) != SATURN_OK) return s;
      }
      if ((s = is.record()) != SATURN_OK) return s;
      epoch.reset();
      if (sp->time_budget_s > 0) {
        // The stop decision must be collective: every island runs the same number of
        // epochs, or the elite all-gathers would mismatch.  MAX-all-reduce of the flag.
        int stop = (now_s() - is.t0 >= sp->time_budget_s) ? 1 : 0;
        if (is.world > 1 && p->peers) {   // any rank's flag: SUM of the flags > 0
          DeviceGuard dg(p->device);
          CU(p, p->ws_key.ensure(2));
          const unsigned long long kf[2] = {~0ull, (unsigned long long)stop};
          CU(p, cudaMemcpyAsync(p->ws_key.p, kf, sizeof kf, cudaMemcpyHostToDevice, st));
          unsigned long long r[2];
          saturn_status sr = peer_reduce_keys(p, p->ws_key.p, st, r);
          if (sr != SATURN_OK) return sr;
          stop = r[1] > 0 ? 1 : 0;
        } else if (is.world > 1) {
          DeviceGuard dg(p->device);
          CU(p, p->flag.ensure(1));
          CU(p, cudaMemcpyAsync(p->flag.p, &stop, sizeof stop, cudaMemcpyHostToDevice, st));
          NC(p, nccl().allReduce(p->flag.p, p->flag.p, 1, ncclInt32, ncclMax, p->comm, st));
          CU(p, cudaMemcpyAsync(&stop, p->flag.p, sizeof stop, cudaMemcpyDeviceToHost, st));
          CU(p, cudaStreamSynchronize(st));
        }
        if (stop) {
          ++gen;
          break;
        }
      }
    }
  }
  epoch.reset();
  const int64_t gens_run = gen - 1 - gen0;
  Nvtx r("saturn_search: final exchange");
  if ((s = exchange()) != SATURN_OK) return s;
  if ((s = is.record()) != SATURN_OK) return s;
  return is.finish(gens_run, is.evaluated * (uint64_t)is.world, out);
}

// Saved search state: this header, then the payload -- population [P][GS] (genome records),
// makespans int32 [P], elite makespans int32 [E], elite records [E][GS].
struct SearchStateHeader {
  char magic[8];          // "SATSRCH1"
  int32_t T, GS;
  int64_t P;
  int32_t E, world;
  uint32_t island, reserved;
  uint64_t seed;
  int64_t generation;
  uint64_t table_hash;    // FNV-1a of the cluster and the loaded runtime table
  uint64_t payload_hash;  // FNV-1a of the payload
  uint64_t payload_bytes;
};
static_assert(sizeof(SearchStateHeader) == 80, "state header layout is part of the ABI");
constexpr char kStateMagic[8] = {'S', 'A', 'T', 'S', 'R', 'C', 'H', '1'};

uint64_t fnv1a(const void* d, size_t n, uint64_t h = 1469598103934665603ull) {
  const uint8_t* b = static_cast<const uint8_t*>(d);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}
uint64_t table_hash(const saturn_plan* p) {
  const int32_t dims[4] = {p->T, p->U, p->Gmax, (int32_t)p->gpu_n.size()};
  uint64_t h = fnv1a(dims, sizeof dims);
  h = fnv1a(p->gpu_n.data(), p->gpu_n.size() * sizeof(int), h);
  return fnv1a(p->dense.data(), p->dense.size() * sizeof(int32_t), h);
}
uint64_t state_payload_bytes(int64_t P, int E, int GS) {
  return (uint64_t)P * (uint64_t)(GS + 4) + (uint64_t)E * (uint64_t)(GS + 4);
}

}  // namespace

saturn_status saturn_search(saturn_plan* p, const saturn_search_params* sp, void* stream, saturn_result* out) {
  if (p && host_only(p)) return SATURN_ESTATE;
  if (!p) return SATURN_EINVAL;
  return search_run(p, sp, stream, out, nullptr, 0);
}

saturn_status saturn_search_save(const saturn_plan* pc, void* h_state, uint64_t capacity, uint64_t* bytes_out) {
  saturn_plan* p = const_cast<saturn_plan*>(pc);
  if (!p) return SATURN_EINVAL;
  if (!p->have_pop) return fail(p, SATURN_ESTATE, "no search state on this handle");
  const int64_t P = p->pop_P;
  const int E = p->last_E, GS = p->pop_GS;
  const uint64_t payload = state_payload_bytes(P, E, GS), total = sizeof(SearchStateHeader) + payload;
  if (bytes_out) *bytes_out = total;
  if (!h_state) return SATURN_OK;
  if (capacity < total)
    return fail(p, SATURN_EINVAL, "capacity %llu < state size %llu", (unsigned long long)capacity,
                (unsigned long long)total);
  DeviceGuard dg(p->device);
  SearchStateHeader h{};
  memcpy(h.magic, kStateMagic, 8);
  h.T = p->T;
  h.GS = GS;
  h.P = P;
  h.E = E;
  h.world = p->last_world;
  h.island = p->last_island;
  h.seed = p->last_seed;
  h.generation = p->last_gen;
  h.table_hash = table_hash(p);
  h.payload_bytes = payload;
  uint8_t* q = static_cast<uint8_t*>(h_state) + sizeof h;
  const int b = p->last_pop;
  CU(p, cudaMemcpy(q, p->pop[b].p, (size_t)P * GS, cudaMemcpyDeviceToHost));
  CU(p, cudaMemcpy(q + (size_t)P * GS, p->pms[b].p, (size_t)P * 4, cudaMemcpyDeviceToHost));
  CU(p, cudaMemcpy(q + (size_t)P * (GS + 4), p->rec_ms.p, (size_t)E * 4, cudaMemcpyDeviceToHost));
  CU(p, cudaMemcpy(q + (size_t)P * (GS + 4) + (size_t)E * 4, p->rec_gen.p, (size_t)E * GS, cudaMemcpyDeviceToHost));
  p->stats.d2h_bytes += (int64_t)payload;
  h.payload_hash = fnv1a(q, payload);
  memcpy(h_state, &h, sizeof h);
  return SATURN_OK;
}

saturn_status saturn_search_resume(saturn_plan* p, const void* h_state, uint64_t bytes,
                                   const saturn_search_params* sp, void* stream, saturn_result* out) {
  if (p && host_only(p)) return SATURN_ESTATE;
  if (!p || !sp) return SATURN_EINVAL;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "resume before load_runtime_table");
  if (!h_state || bytes < sizeof(SearchStateHeader)) return fail(p, SATURN_EINVAL, "state buffer too small");
  SearchStateHeader h;
  memcpy(&h, h_state, sizeof h);
  if (memcmp(h.magic, kStateMagic, 8) != 0) return fail(p, SATURN_EINVAL, "not a saturn search state");
  const int T = p->T, GS = gs_of(T);
  if (h.T != T || h.GS != GS) return fail(p, SATURN_EINVAL, "state has T=%d, the table has T=%d", h.T, T);
  if (h.table_hash != table_hash(p)) return fail(p, SATURN_EINVAL, "state was saved with another cluster or table");
  if (h.P < 1 || h.E < 1 || h.payload_bytes != state_payload_bytes(h.P, h.E, GS) ||
      bytes != sizeof h + h.payload_bytes)
    return fail(p, SATURN_EINVAL, "state size mismatch");
  const uint8_t* q = static_cast<const uint8_t*>(h_state) + sizeof h;
  if (fnv1a(q, h.payload_bytes) != h.payload_hash) return fail(p, SATURN_EINVAL, "state payload checksum mismatch");
  if (sp->population != h.P || sp->elites != h.E || sp->seed != h.seed)
    return fail(p, SATURN_EINVAL, "params (seed, population, elites) differ from the saved search's");
  const int world = distributed(p) ? p->world : 1;
  if (h.world != world || h.island != (uint32_t)p->rank)
    return fail(p, SATURN_EINVAL, "state is island %u of %d; this handle is rank %d of %d", h.island, h.world,
                p->rank, world);
  if (h.generation < 0 || h.generation + sp->max_generations >= (int64_t(1) << 32))
    return fail(p, SATURN_EINVAL, "generation counter out of range");
  // every genome of the population and of the elite records must be valid (the decoder
  // indexes the staged table with them)
  const int Tp = sat::perm_offset(T);
  auto valid = [&](const uint8_t* g) {
    uint32_t seen[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < T; ++k) {
      const int t = g[Tp + k];
      if (t >= T || (seen[t >> 5] >> (t & 31)) & 1u) return false;
      seen[t >> 5] |= 1u << (t & 31);
      if (g[t] >= p->S[t]) return false;
    }
    return true;
  };
  for (int64_t i = 0; i < h.P; ++i)
    if (!valid(q + (size_t)i * GS)) return fail(p, SATURN_EINVAL, "state genome %lld is invalid", (long long)i);
  const uint8_t* rec = q + (size_t)h.P * (GS + 4) + (size_t)h.E * 4;
  for (int i = 0; i < h.E; ++i)
    if (!valid(rec + (size_t)i * GS)) return fail(p, SATURN_EINVAL, "state elite %d is invalid", i);
  return search_run(p, sp, stream, out, q, h.generation);
}

saturn_status saturn_search_group(saturn_plan** plans, int32_t k, const saturn_search_params* sp, void** streams,
                                   saturn_result* out) {
  if (!plans || k < 1 || !sp) return SATURN_EINVAL;
  std::vector<Island> isl(k);
  for (int r = 0; r < k; ++r) {
    saturn_plan* p = plans[r];
    if (!p) return SATURN_EINVAL;
    if (host_only(p)) return SATURN_ESTATE;
    if (p->comm || p->peers)
      return fail(p, SATURN_ESTATE, "search_group islands must not have an NCCL communicator or a peer link");
    for (int q = 0; q < r; ++q)
      if (plans[q] == p) return fail(p, SATURN_EINVAL, "the same handle twice in a group");
    isl[r].p = p;
    isl[r].sp = sp;
    isl[r].st = streams ? static_cast<cudaStream_t>(streams[r]) : nullptr;
    isl[r].island = (uint32_t)r;
    isl[r].world = k;
    saturn_status s = isl[r].validate();
    if (s != SATURN_OK) return s;
    if (isl[r].T != isl[0].T || plans[r]->S != plans[0]->S || plans[r]->cfg_r != plans[0]->cfg_r ||
        plans[r]->gpu_n != plans[0]->gpu_n)
      return fail(p, SATURN_EINVAL, "islands of a group must load the same cluster and table");
  }
  saturn_status s;
  for (auto& is : isl)
    if ((s = is.begin()) != SATURN_OK) return s;
  const int E = isl[0].E, GS = isl[0].GS;
  // exchange by copies: island r's records land in block r of every island's all_* buffers
  auto exchange = [&]() -> saturn_status {
    saturn_status e;
    for (auto& is : isl)
      if ((e = is.memetic()) != SATURN_OK) return e;
    if (k < 2) return SATURN_OK;
    for (auto& is : isl) {  // the sources must be complete before anyone copies them
      DeviceGuard dg(is.p->device);
      CU(is.p, cudaStreamSynchronize(is.st));
    }
    for (auto& dst : isl) {
      DeviceGuard dg(dst.p->device);
      for (int r = 0; r < k; ++r) {
        saturn_plan* src = isl[r].p;
        CU(dst.p, cudaMemcpyPeerAsync(dst.p->all_ms.p + (size_t)r * E, dst.p->device, src->rec_ms.p, src->device,
                                      E * sizeof(int32_t), dst.st));
        CU(dst.p, cudaMemcpyPeerAsync(dst.p->all_gen.p + (size_t)r * E * GS, dst.p->device, src->rec_gen.p,
                                      src->device, (size_t)E * GS, dst.st));
      }
    }
    for (auto& dst : isl)  // all copies must read the old records before anyone merges
      CU(dst.p, cudaStreamSynchronize(dst.st));
    for (auto& is : isl)
      if ((e = is.merge()) != SATURN_OK) return e;
    return SATURN_OK;
  };
  auto record_all = [&]() -> saturn_status {
    saturn_status e;
    for (auto& is : isl)
      if ((e = is.record()) != SATURN_OK) return e;
    return SATURN_OK;
  };
  if ((s = exchange()) != SATURN_OK) return s;
  if ((s = record_all()) != SATURN_OK) return s;
  int64_t gen = 1;
  for (; gen <= sp->max_generations; ++gen) {
    for (auto& is : isl)
      if ((s = is.generation(gen)) != SATURN_OK) return s;
    if (gen % sp->generations_per_epoch == 0) {
      if ((s = exchange()) != SATURN_OK) return s;
      if ((s = record_all()) != SATURN_OK) return s;
      if (sp->time_budget_s > 0 && now_s() - isl[0].t0 >= sp->time_budget_s) {
        ++gen;
        break;
      }
    }
  }
  const int64_t gens_run = gen - 1;
  if ((s = exchange()) != SATURN_OK) return s;
  if ((s = record_all()) != SATURN_OK) return s;
  uint64_t total = 0;
  for (auto& is : isl) total += is.evaluated;
  for (int r = 0; r < k; ++r)
    if ((s = isl[r].finish(gens_run, total, out ? &out[r] : nullptr)) != SATURN_OK) return s;
  return SATURN_OK;
}

saturn_status saturn_improve(saturn_plan* p, uint8_t* h_cfg, uint8_t* h_perm, int64_t n, int32_t iters,
                             int32_t* h_makespan, void* stream) {
  if (!p) return SATURN_EINVAL;
  if (host_only(p)) return SATURN_ESTATE;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "improve before load_runtime_table");
  if (n < 0 || iters < 0 || (n > 0 && (!h_cfg || !h_perm || !h_makespan)))
    return fail(p, SATURN_EINVAL, "bad arguments");
  if (n == 0) return SATURN_OK;
  if (!p->sorted_ok) return fail(p, SATURN_EINVAL, "local search needs the thread decoder for this cluster shape");
  const int T = p->T, GS = gs_of(T), Tp = sat::perm_offset(T);
  std::vector<uint8_t> packed((size_t)n * GS, 0);
  for (int64_t i = 0; i < n; ++i) {
    std::vector<int> seen(T, 0);
    for (int k = 0; k < T; ++k) {
      const int t = h_perm[i * T + k];
      if (t >= T || seen[t]++) return fail(p, SATURN_EINVAL, "genome %lld: perm is not a permutation", (long long)i);
      if (h_cfg[i * T + t] >= p->S[t]) return fail(p, SATURN_EINVAL, "genome %lld: cfg out of range", (long long)i);
    }
    memcpy(&packed[i * GS], h_cfg + i * T, T);
    memcpy(&packed[i * GS + Tp], h_perm + i * T, T);
  }
  DeviceGuard dg(p->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CU(p, p->ls_gen.ensure(packed.size()));
  CU(p, p->ls_ms.ensure((size_t)n));
  CU(p, p->ws_cfg.ensure((size_t)n * T));
  CU(p, p->ws_perm.ensure((size_t)n * T));
  CU(p, cudaMemcpyAsync(p->ws_cfg.p, h_cfg, (size_t)n * T, cudaMemcpyHostToDevice, st));
  CU(p, cudaMemcpyAsync(p->ws_perm.p, h_perm, (size_t)n * T, cudaMemcpyHostToDevice, st));
  int inn, igp;
  run_shape(p, &inn, &igp);
  CU(p, sat::launch_evaluate(p->pb, inn, igp, SATURN_DECODER_THREAD, p->ws_cfg.p, p->ws_perm.p, n, p->ls_ms.p,
                             p->sms, st));
  CU(p, cudaMemcpyAsync(p->ls_gen.p, packed.data(), packed.size(), cudaMemcpyHostToDevice, st));
  CU(p, sat::launch_local_search(p->pb, inn, igp, p->ls_gen.p, p->ls_ms.p, (int)n, GS, iters, st));
  CU(p, cudaMemcpyAsync(packed.data(), p->ls_gen.p, packed.size(), cudaMemcpyDeviceToHost, st));
  CU(p, cudaMemcpyAsync(h_makespan, p->ls_ms.p, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CU(p, cudaStreamSynchronize(st));
  p->stats.kernel_launches += 2;
  p->stats.h2d_bytes += (int64_t)packed.size() + 2 * n * T;
  p->stats.d2h_bytes += (int64_t)packed.size() + n * 4;
  for (int64_t i = 0; i < n; ++i) {
    memcpy(h_cfg + i * T, &packed[i * GS], T);
    memcpy(h_perm + i * T, &packed[i * GS + Tp], T);
  }
  return SATURN_OK;
}

saturn_status saturn_search_history(const saturn_plan* p, int64_t n_max, double* t_s, int64_t* makespan,
                                    int64_t* n_out) {
  if (!p || !n_out) return SATURN_EINVAL;
  const int64_t n = std::min<int64_t>(n_max, (int64_t)p->hist_t.size());
  for (int64_t i = 0; i < n; ++i) {
    if (t_s) t_s[i] = p->hist_t[i];
    if (makespan) makespan[i] = p->hist_ms[i];
  }
  *n_out = n;
  return SATURN_OK;
}

saturn_status saturn_search_population(const saturn_plan* pc, int64_t capacity, uint8_t* h_cfg, uint8_t* h_perm,
                                       int32_t* h_makespan, int64_t* n_out) {
  saturn_plan* p = const_cast<saturn_plan*>(pc);
  if (!p) return SATURN_EINVAL;
  if (!p->have_pop) return fail(p, SATURN_ESTATE, "no search population on this handle");
  const int64_t P = p->pop_P;
  if (n_out) *n_out = P;
  if (!h_cfg && !h_perm && !h_makespan) return SATURN_OK;
  if (capacity < P)
    return fail(p, SATURN_EINVAL, "capacity %lld < population %lld", (long long)capacity, (long long)P);
  DeviceGuard dg(p->device);
  const int GS = p->pop_GS, T = p->T;
  if (h_cfg || h_perm) {
    std::vector<uint8_t> buf((size_t)P * GS);
    CU(p, cudaMemcpy(buf.data(), p->pop[p->last_pop].p, buf.size(), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < P; ++i) {
      if (h_cfg) memcpy(h_cfg + i * T, &buf[i * GS], T);
      if (h_perm) memcpy(h_perm + i * T, &buf[i * GS + sat::perm_offset(T)], T);
    }
  }
  if (h_makespan) CU(p, cudaMemcpy(h_makespan, p->pms[p->last_pop].p, P * sizeof(int32_t), cudaMemcpyDeviceToHost));
  return SATURN_OK;
}

saturn_status saturn_best_plan(saturn_plan* p, saturn_placement* out, uint8_t* genome_out, int64_t* makespan) {
  if (p && host_only(p)) return SATURN_ESTATE;
  if (!p) return SATURN_EINVAL;
  if (!p->have_best) return fail(p, SATURN_ESTATE, "best_plan before enumerate/search");
  DeviceGuard dg(p->device);
  const int T = p->T;
  if (out) {
    CU(p, p->ws_cfg.ensure(T));
    CU(p, p->ws_perm.ensure(T));
    CU(p, p->ws_ms.ensure(1));
    CU(p, p->ws_place.ensure(T));
    CU(p, cudaMemcpy(p->ws_cfg.p, p->best_cfg.data(), T, cudaMemcpyHostToDevice));
    CU(p, cudaMemcpy(p->ws_perm.p, p->best_perm.data(), T, cudaMemcpyHostToDevice));
    CU(p, sat::launch_trace(p->pb, p->ws_cfg.p, p->ws_perm.p, 1, p->ws_place.p, p->ws_ms.p, p->sms, 0));
    CU(p, cudaMemcpy(out, p->ws_place.p, T * sizeof(saturn_placement), cudaMemcpyDeviceToHost));
    int32_t ms = 0;
    CU(p, cudaMemcpy(&ms, p->ws_ms.p, sizeof ms, cudaMemcpyDeviceToHost));
    p->stats.kernel_launches += 1;
    p->stats.h2d_bytes += 2 * T;
    p->stats.d2h_bytes += T * (int64_t)sizeof(saturn_placement) + (int64_t)sizeof ms;
    if (ms != p->best_ms)
      return fail(p, SATURN_ECUDA, "trace makespan %d != recorded best %lld", ms, (long long)p->best_ms);
  }
  if (genome_out) {
    memcpy(genome_out, p->best_cfg.data(), T);
    memcpy(genome_out + T, p->best_perm.data(), T);
  }
  if (makespan) *makespan = p->best_ms;
  return SATURN_OK;
}

namespace {

// ------------------------------------------------------------------ f2: baseline genomes (host)
void philox_host(uint32_t k0, uint32_t k1, const uint32_t c[4], uint32_t out[4]) {
  uint32_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3];
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint64_t p0 = (uint64_t)0xD2511F53u * x0, p1 = (uint64_t)0xCD9E8D57u * x2;
    const uint32_t y0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0, y2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
    x0 = y0; x1 = (uint32_t)p1; x2 = y2; x3 = (uint32_t)p0;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}
// word k of the stream (c0, c1, c2) under key seed
uint32_t stream_word(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t k) {
  const uint32_t c[4] = {c0, c1, c2, k >> 2};
  uint32_t o[4];
  philox_host((uint32_t)seed, (uint32_t)(seed >> 32), c, o);
  return o[k & 3];
}
uint32_t ubelow_host(uint32_t u, uint32_t n) { return (uint32_t)(((uint64_t)u * n) >> 32); }

// best config of job t at g GPUs: least runtime, ties to the lower UPP (= lower index); -1 if none
int best_cfg(const saturn_plan* p, int t, int g) {
  int best = -1;
  for (int s = 0; s < p->S[t]; ++s) {
    const int k = t * p->stride + s;
    if (p->cfg_g[k] != g) continue;
    if (best < 0) { best = s; continue; }
    const int kb = t * p->stride + best;
    if (p->cfg_r[k] < p->cfg_r[kb] || (p->cfg_r[k] == p->cfg_r[kb] && p->cfg_u[k] < p->cfg_u[kb])) best = s;
  }
  return best;
}
// widest width <= limit that has a config (else the narrowest width of the job)
int widest_upto(const saturn_plan* p, int t, int limit) {
  int w = -1, narrow = 1 << 30;
  for (int s = 0; s < p->S[t]; ++s) {
    const int g = p->cfg_g[t * p->stride + s];
    if (g <= limit && g > w) w = g;
    narrow = std::min(narrow, g);
  }
  return w > 0 ? w : narrow;
}
std::vector<int> distribute_jobs(const saturn_plan* p, uint64_t seed) {
  const int N = (int)p->gpu_n.size();
  std::vector<int> node(p->T, 0);
  if (N == 1) return node;
  for (int t = 0; t < p->T; ++t) {
    const uint32_t u = ubelow_host(stream_word(seed, (uint32_t)t, 0u, 3u << 16, 0), (uint32_t)p->sumG);
    int acc = 0;
    for (int n = 0; n < N; ++n) {
      acc += p->gpu_n[n];
      if ((int)u < acc) { node[t] = n; break; }
    }
  }
  return node;
}
void lpt_genome(const saturn_plan* p, const std::vector<int>& cfg, uint8_t* out_cfg, uint8_t* out_perm) {
  std::vector<int> order(p->T);
  for (int t = 0; t < p->T; ++t) { order[t] = t; out_cfg[t] = (uint8_t)cfg[t]; }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return p->cfg_r[a * p->stride + cfg[a]] > p->cfg_r[b * p->stride + cfg[b]];
  });
  for (int i = 0; i < p->T; ++i) out_perm[i] = (uint8_t)order[i];
}

}  // namespace

saturn_status saturn_baseline_genome(const saturn_plan* cp, int32_t kind, uint64_t seed, uint8_t* cfg, uint8_t* perm) {
  saturn_plan* p = const_cast<saturn_plan*>(cp);
  if (!p || !cfg || !perm) return SATURN_EINVAL;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "baseline before load_runtime_table");
  const int T = p->T, N = (int)p->gpu_n.size();
  std::vector<int> chosen(T, 0);
  if (kind == SATURN_BASELINE_RANDOM) {  // = the GA's initial genome of slot 0
    uint32_t k = 0;
    for (int t = 0; t < T; ++t) cfg[t] = (uint8_t)ubelow_host(stream_word(seed, 0, 0, 1, k++), (uint32_t)p->S[t]);
    for (int t = 0; t < T; ++t) perm[t] = (uint8_t)t;
    for (int i = T - 1; i > 0; --i) {
      const int j = (int)ubelow_host(stream_word(seed, 0, 0, 1, k++), (uint32_t)(i + 1));
      std::swap(perm[i], perm[j]);
    }
    return SATURN_OK;
  }
  const std::vector<int> node = distribute_jobs(p, seed);
  if (kind == SATURN_BASELINE_MAX) {
    for (int t = 0; t < T; ++t) chosen[t] = best_cfg(p, t, widest_upto(p, t, p->gpu_n[node[t]]));
  } else if (kind == SATURN_BASELINE_MIN) {
    std::vector<int> share(T, 1);
    for (int n = 0; n < N; ++n) {
      std::vector<int> jobs;
      for (int t = 0; t < T; ++t)
        if (node[t] == n) jobs.push_back(t);
      if (jobs.empty()) continue;
      std::vector<int> cap;
      for (int t : jobs) {
        int c = 0;
        for (int s = 0; s < p->S[t]; ++s) {
          const int g = p->cfg_g[t * p->stride + s];
          if (g <= p->gpu_n[n]) c = std::max(c, g);
        }
        cap.push_back(c > 0 ? c : 1);
      }
      int surplus = p->gpu_n[n] - (int)jobs.size();
      while (surplus > 0) {
        bool progressed = false;
        for (size_t i = 0; i < jobs.size(); ++i)
          if (surplus > 0 && share[jobs[i]] < cap[i]) { ++share[jobs[i]]; --surplus; progressed = true; }
        if (!progressed) break;
      }
    }
    for (int t = 0; t < T; ++t) chosen[t] = best_cfg(p, t, widest_upto(p, t, share[t]));
  } else if (kind == SATURN_BASELINE_OPTIMUS) {  // Alg. 1, one node at a time
    std::vector<int> alloc(T, 1);
    for (int n = 0; n < N; ++n) {
      std::vector<int> jobs;
      for (int t = 0; t < T; ++t)
        if (node[t] == n) jobs.push_back(t);
      if (jobs.empty()) continue;
      auto Rbest = [&](int t, int g) -> int64_t {  // -1: no config at g GPUs on this node
        if (g > p->gpu_n[n]) return -1;
        const int s = best_cfg(p, t, g);
        return s < 0 ? -1 : p->cfg_r[t * p->stride + s];
      };
      std::vector<int> L(jobs.size(), 1);
      int sum = (int)jobs.size();
      while (sum < p->gpu_n[n]) {
        int arg = -1;
        int64_t best = 0;
        for (size_t i = 0; i < jobs.size(); ++i) {
          const int64_t cur = Rbest(jobs[i], L[i]), nxt = Rbest(jobs[i], L[i] + 1);
          if (cur < 0 || nxt < 0) continue;  // gain -inf
          const int64_t gain = cur - nxt;
          if (arg < 0 || gain > best) { arg = (int)i; best = gain; }
        }
        if (arg < 0) break;
        ++L[arg];
        ++sum;
      }
      for (size_t i = 0; i < jobs.size(); ++i) alloc[jobs[i]] = L[i];
    }
    for (int t = 0; t < T; ++t) {
      int s = best_cfg(p, t, alloc[t]);
      if (s < 0) s = best_cfg(p, t, widest_upto(p, t, alloc[t]));
      chosen[t] = s;
    }
  } else {
    return fail(p, SATURN_EINVAL, "unknown baseline kind %d", kind);
  }
  lpt_genome(p, chosen, cfg, perm);
  return SATURN_OK;
}

saturn_status saturn_baseline_nodes(const saturn_plan* cp, int32_t kind, uint64_t seed, uint8_t* node) {
  saturn_plan* p = const_cast<saturn_plan*>(cp);
  if (!p || !node) return SATURN_EINVAL;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "baseline before load_runtime_table");
  const int T = p->T;
  if (kind == SATURN_BASELINE_RANDOM) {
    memset(node, 0xFF, T);
    return SATURN_OK;
  }
  std::vector<uint8_t> cfg(T), perm(T);
  saturn_status s = saturn_baseline_genome(p, kind, seed, cfg.data(), perm.data());
  if (s != SATURN_OK) return s;
  const std::vector<int> nd = distribute_jobs(p, seed);
  for (int t = 0; t < T; ++t)
    node[t] = p->cfg_g[t * p->stride + cfg[t]] <= p->gpu_n[nd[t]] ? (uint8_t)nd[t] : (uint8_t)0xFF;
  return SATURN_OK;
}

saturn_status saturn_introspect(saturn_plan* p, const saturn_introspect_params* ip, void* stream,
                                saturn_introspect_result* out, int64_t* round_log) {
  if (!p) return SATURN_EINVAL;
  if (host_only(p)) return SATURN_ESTATE;
  if (!p->loaded) return fail(p, SATURN_ESTATE, "introspect before load_runtime_table");
  if (!ip || ip->interval_s < 1 || ip->threshold_s < 0 || ip->max_rounds < 0 || ip->n_events < 0 ||
      (ip->n_events > 0 && !ip->events))
    return fail(p, SATURN_EINVAL, "bad introspection parameters");
  if (ip->solver == SATURN_SOLVER_SEARCH && !ip->search) return fail(p, SATURN_EINVAL, "search params missing");
  const std::vector<int32_t> orig = p->dense;
  const int U = p->U, G = p->Gmax;
  const int64_t I = ip->interval_s, Tthr = ip->threshold_s;
  const double wall_I = ip->interval_wall_s > 0 ? ip->interval_wall_s : (double)I;
  for (int e = 0; e < ip->n_events; ++e) {
    const saturn_introspect_event& ev = ip->events[e];
    if (ev.at_round < 1 || (ev.kind != SATURN_EVENT_STOP && ev.kind != SATURN_EVENT_ARRIVE) ||
        (ev.kind == SATURN_EVENT_ARRIVE && !ev.runtime_s))
      return fail(p, SATURN_EINVAL, "bad introspection event %d", e);
  }
  std::vector<int32_t> W = orig;
  int Tn = p->T;
  std::vector<int> ids(Tn);   // original job id of every row of W
  for (int t = 0; t < Tn; ++t) ids[t] = t;
  int next_id = Tn;
  uint64_t evaluated = 0;
  int solves = 0;
  double solve_s = 0, exposed_s = 0;
  std::vector<saturn_placement> S;
  // solve the currently loaded workload -> S (placements, job-id order) and its makespan
  auto solve = [&](std::vector<saturn_placement>& plan, int64_t& ms, double* secs) -> saturn_status {
    const double t0 = now_s();
    saturn_status st;
    saturn_result r;
    if (ip->solver == SATURN_SOLVER_ENUMERATE) st = saturn_enumerate(p, uint64_t(1) << 38, stream, &r);
    else st = saturn_search(p, ip->search, stream, &r);
    if (st != SATURN_OK) return st;
    evaluated += r.evaluated;
    ++solves;
    plan.resize(p->T);
    st = saturn_best_plan(p, plan.data(), nullptr, &ms);
    if (secs) *secs = now_s() - t0;
    return st;
  };
  auto restore = [&](saturn_status st) {
    const std::string keep = p->err;
    saturn_load_runtime_table(p, orig.data(), (int32_t)(orig.size() / ((size_t)U * G)), U, G);
    if (st != SATURN_OK) p->err = keep;
    return st;
  };
  // W after I seconds of S (residual runtimes, reading A10) and S[I:]; `keep` = surviving rows
  auto advance = [&](const std::vector<int32_t>& Win, const std::vector<saturn_placement>& Sin,
                     std::vector<int32_t>& Wout, std::vector<saturn_placement>& Sout, std::vector<int>* keep) {
    Wout.clear();
    Sout.clear();
    if (keep) keep->clear();
    for (size_t t = 0; t < Sin.size(); ++t) {
      const saturn_placement& pl = Sin[t];
      if (pl.end_s <= I) continue;
      const int32_t* row = &Win[t * U * G];
      if (pl.start_s < I) {
        const int64_t R0 = pl.end_s - pl.start_s, a = I - pl.start_s;
        for (int k = 0; k < U * G; ++k)
          Wout.push_back(row[k] > 0 ? (int32_t)(((int64_t)row[k] * (R0 - a) + R0 - 1) / R0) : 0);
      } else {
        Wout.insert(Wout.end(), row, row + U * G);
      }
      saturn_placement q = pl;
      q.start_s = (int32_t)std::max<int64_t>(pl.start_s - I, 0);
      q.end_s = (int32_t)(pl.end_s - I);
      Sout.push_back(q);
      if (keep) keep->push_back((int)t);
    }
  };
  int64_t M = 0;
  saturn_status st = solve(S, M, nullptr);
  if (st != SATURN_OK) return restore(st);
  const int64_t one_shot = M;
  int64_t time = 0;
  int rounds = 0, adopted = 0, stale = 0;
  while (M > I && rounds < ip->max_rounds) {
    Nvtx nr("saturn_introspect: round");
    // overlap mode: round k+1's proposal from the simulated next-interval state, solved
    // while round k runs (its latency hides behind the interval)
    bool have_look = false;
    std::vector<saturn_placement> Plook;
    int64_t Mlook = 0;
    double t_look = 0;
    if (ip->overlap) {
      std::vector<int32_t> Wn;
      std::vector<saturn_placement> Sn;
      advance(W, S, Wn, Sn, nullptr);
      if (!Sn.empty()) {
        st = saturn_load_runtime_table(p, Wn.data(), (int32_t)Sn.size(), U, G);
        if (st != SATURN_OK) return restore(st);
        st = solve(Plook, Mlook, &t_look);
        if (st != SATURN_OK) return restore(st);
        have_look = true;
        solve_s += t_look;
        exposed_s += std::max(0.0, t_look - wall_I);
      }
    }
    std::vector<int32_t> W2;
    std::vector<saturn_placement> S2;
    std::vector<int> keep;
    advance(W, S, W2, S2, &keep);
    W.swap(W2);
    S.swap(S2);
    {
      std::vector<int> ids2;
      for (int k : keep) ids2.push_back(ids[k]);
      ids.swap(ids2);
    }
    M -= I;
    time += I;
    ++rounds;
    // events due at this boundary
    bool fired = false, arrived = false;
    for (int e = 0; e < ip->n_events; ++e) {
      const saturn_introspect_event& ev = ip->events[e];
      if (ev.at_round != rounds) continue;
      fired = true;
      if (ev.kind == SATURN_EVENT_STOP) {
        const auto it = std::find(ids.begin(), ids.end(), ev.job);
        if (it == ids.end()) {
          restore(SATURN_OK);
          return fail(p, SATURN_EINVAL, "stop event at round %d names job %d, finished or unknown", rounds, ev.job);
        }
        const size_t k = (size_t)(it - ids.begin());
        W.erase(W.begin() + k * U * G, W.begin() + (k + 1) * U * G);
        S.erase(S.begin() + k);
        ids.erase(it);
      } else {
        W.insert(W.end(), ev.runtime_s, ev.runtime_s + (size_t)U * G);
        ids.push_back(next_id++);
        arrived = true;
      }
    }
    if (fired) {
      stale += have_look ? 1 : 0;
      have_look = false;
      M = 0;
      for (const auto& q : S) M = std::max<int64_t>(M, q.end_s);
    }
    Tn = (int)ids.size();
    if (Tn == 0) {   // every job stopped: the workload is exhausted
      M = 0;
      if (round_log)
        for (int k = 0; k < 4; ++k) round_log[4 * (rounds - 1) + k] = k == 0 ? time : 0;
      break;
    }
    std::vector<saturn_placement> P;
    int64_t Mp = 0;
    if (have_look) {
      P.swap(Plook);
      Mp = Mlook;
    } else {
      st = saturn_load_runtime_table(p, W.data(), Tn, U, G);
      if (st != SATURN_OK) return restore(st);
      double t_fresh = 0;
      st = solve(P, Mp, &t_fresh);
      if (st != SATURN_OK) return restore(st);
      solve_s += t_fresh;
      exposed_s += t_fresh;   // solved at the boundary: on the critical path
    }
    const bool take = arrived || Mp <= M - Tthr;
    if (round_log) {
      round_log[4 * (rounds - 1) + 0] = time;
      round_log[4 * (rounds - 1) + 1] = M;
      round_log[4 * (rounds - 1) + 2] = Mp;
      round_log[4 * (rounds - 1) + 3] = take ? 1 : 0;
    }
    if (take) {
      S.swap(P);
      M = Mp;
      ++adopted;
    }
  }
  st = restore(SATURN_OK);
  if (st != SATURN_OK) return st;
  if (out) {
    memset(out, 0, sizeof *out);
    out->one_shot_makespan = one_shot;
    out->e2e_makespan = time + M;
    out->rounds = rounds;
    out->adopted = adopted;
    out->evaluated = evaluated;
    out->stale = stale;
    out->solves = solves;
    out->solve_s = solve_s;
    out->exposed_solve_s = exposed_s;
  }
  return SATURN_OK;
}

saturn_status saturn_get_unique_id(uint8_t* id128) {
  if (!id128) return SATURN_EINVAL;
  if (!nccl().ok) return SATURN_ENCCL;
  ncclUniqueId id;
  if (nccl().getUniqueId(&id) != ncclSuccess) return SATURN_ENCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id128, &id, 128);
  return SATURN_OK;
}

saturn_status saturn_plan_attach_comm(saturn_plan* p, const uint8_t* id128, int32_t rank, int32_t world) {
  if (p && host_only(p)) return SATURN_ESTATE;
  if (!p) return SATURN_EINVAL;
  if (!id128 || world < 1 || rank < 0 || rank >= world) return fail(p, SATURN_EINVAL, "bad rank/world");
  if (!nccl().ok) return fail(p, SATURN_ENCCL, "%s", nccl().why.c_str());
  if (p->peers) return fail(p, SATURN_ESTATE, "attach_comm: the handle already has a peer link");
  DeviceGuard dg(p->device);
  if (p->comm) {
    nccl().commDestroy(p->comm);
    p->comm = nullptr;
  }
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  NC(p, nccl().commInitRank(&p->comm, world, id, rank));
  p->rank = rank;
  p->world = world;
  return SATURN_OK;
}

saturn_status saturn_plan_attach_peers(saturn_plan* p, const char* name, int32_t rank, int32_t world) {
  if (!p) return SATURN_EINVAL;
  if (!name || name[0] != '/' || world < 1 || world > sat::PEER_MAX || rank < 0 || rank >= world)
    return fail(p, SATURN_EINVAL, "attach_peers: need a '/name', 1 <= world <= 8 and 0 <= rank < world");
  if (p->comm) return fail(p, SATURN_ESTATE, "attach_peers: the handle already has an NCCL communicator");
  std::unique_ptr<sat::PeerLink> L(new sat::PeerLink());
  const char* to = getenv("SATURN_PEER_TIMEOUT_S");
  const double timeout = to ? atof(to) : 120.0;
  if (host_only(p)) {
    if (!L->attach(name, rank, world, -1, timeout)) return fail(p, SATURN_ECUDA, "%s", L->err.c_str());
  } else {
    DeviceGuard dg(p->device);
    if (!L->attach(name, rank, world, p->device, timeout)) return fail(p, SATURN_ECUDA, "%s", L->err.c_str());
  }
  p->peers = std::move(L);
  p->rank = rank;
  p->world = world;
  return SATURN_OK;
}

saturn_status saturn_plan_barrier(saturn_plan* p) {
  if (!p) return SATURN_EINVAL;
  if (!p->peers) return fail(p, SATURN_ESTATE, "barrier: no peer link (saturn_plan_attach_peers)");
  if (!p->peers->barrier()) return fail(p, SATURN_ECUDA, "%s", p->peers->err.c_str());
  return SATURN_OK;
}

saturn_status saturn_partition(uint64_t total, int32_t rank, int32_t world, uint64_t* begin, uint64_t* end) {
  if (!begin || !end || world < 1 || rank < 0 || rank >= world) return SATURN_EINVAL;
  const unsigned __int128 tt = total;
  *begin = (uint64_t)(tt * (unsigned)rank / (unsigned)world);
  *end = (uint64_t)(tt * (unsigned)(rank + 1) / (unsigned)world);
  return SATURN_OK;
}

saturn_status saturn_probe_int_peak(saturn_plan* p, double* int_ops_per_s) {
  if (p && host_only(p)) return SATURN_ESTATE;
  if (!p || !int_ops_per_s) return SATURN_EINVAL;
  DeviceGuard dg(p->device);
  CU(p, p->sink.ensure(p->sms * 8));
  cudaEvent_t a, b;
  CU(p, cudaEventCreate(&a));
  CU(p, cudaEventCreate(&b));
  double ops = 0;
  for (int w = 0; w < 3; ++w) sat::launch_int_probe(p->sms, p->sink.p, 0);
  float best_ms = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CU(p, cudaEventRecord(a, 0));
    ops = sat::launch_int_probe(p->sms, p->sink.p, 0);
    CU(p, cudaEventRecord(b, 0));
    CU(p, cudaEventSynchronize(b));
    float ms = 0;
    CU(p, cudaEventElapsedTime(&ms, a, b));
    best_ms = std::min(best_ms, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  CU(p, cudaGetLastError());
  *int_ops_per_s = ops / (best_ms * 1e-3);
  return SATURN_OK;
}

saturn_status saturn_set_profiling(saturn_plan* p, int32_t on) {
  if (!p) return SATURN_EINVAL;
  p->profiling = on < 0 ? 0 : on;
  return SATURN_OK;
}

saturn_status saturn_get_stats(const saturn_plan* p, saturn_stats* out) {
  if (!p || !out) return SATURN_EINVAL;
  *out = p->stats;
  return SATURN_OK;
}

saturn_status saturn_reset_stats(saturn_plan* p) {
  if (!p) return SATURN_EINVAL;
  p->stats = saturn_stats{};
  return SATURN_OK;
}

const char* saturn_last_error(const saturn_plan* p) { return p ? p->err.c_str() : "NULL handle"; }

void saturn_plan_destroy(saturn_plan* p) {
  if (!p) return;
  if (p->device < 0) {
    delete p;
    return;
  }
  {
    DeviceGuard dg(p->device);
    if (p->comm && nccl().ok) nccl().commDestroy(p->comm);
    p->peers.reset();
    if (p->pinned) cudaFreeHost(p->pinned);
    for_each_buf(p, [](auto& b) { b.release(); });
    for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : p->hist_ev) cudaEventDestroy(e);
    if (p->hist_pin) cudaFreeHost(p->hist_pin);
  }
  delete p;
}

}  // extern "C"
