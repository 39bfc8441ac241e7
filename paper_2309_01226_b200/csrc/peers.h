// Peer-memory transport for the multi-GPU exchange steps (row e of SURVEY.md §8; §8e
// "B200-native alternative to measure"): the ranks of one node map each other's exchange
// buffers with CUDA IPC and synchronise through a barrier in a POSIX shared-memory segment,
// so the island elite exchange and the enumeration MIN need no NCCL.  Every rank PUSHES its
// contribution into block `rank` of every rank's buffer (device-to-device copies over
// NVLink, or within one device), passes the barrier, and reads its own buffer.
//
// Host code only; nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

namespace sat {

constexpr int PEER_MAX = 8;        // ranks per node
constexpr int PEER_EMAX = 32;      // elites per rank (saturn_search_params.elites <= 32)
constexpr int PEER_GSMAX = 528;    // genome record bytes for T <= 255

// Layout of every rank's exchange buffer (device memory).  The elite region is double
// buffered by epoch parity, so a rank one epoch ahead never overwrites a block a slower
// rank is still merging (one barrier per epoch suffices).
struct PeerLayout {
  static constexpr size_t keys = 0;                                   // u64 [PEER_MAX][2]
  static constexpr size_t flags = keys + 16 * PEER_MAX;               // i32 [PEER_MAX]
  static constexpr size_t shared = 192;                               // u64 [2]: the fused enumeration's
                                                                      // (key, leaves), used in rank 0's buffer
  static constexpr size_t ms0 = 256;                                  // i32 [2][PEER_MAX * E]
  static constexpr size_t ms_bytes = 4 * PEER_MAX * PEER_EMAX;
  static constexpr size_t gen0 = ms0 + 2 * ms_bytes;                  // u8 [2][PEER_MAX * E * GS]
  static constexpr size_t gen_bytes = (size_t)PEER_MAX * PEER_EMAX * PEER_GSMAX;
  static constexpr size_t bytes = gen0 + 2 * gen_bytes;
};

class PeerLink {
 public:
  ~PeerLink() { detach(); }
  // Collective over the `world` ranks that pass the same `name` (a fresh POSIX shm name,
  // e.g. "/saturn_<nonce>", created by rank 0).  device < 0: host-only (barrier only).
  // `timeout_s` is a LIVENESS timeout: a rank that stops heartbeating for that long (its
  // process died or hangs outside the library) fails every other rank's barrier.  A rank
  // that is merely slow (its GPU still busy) keeps heartbeating from wait_stream, so a long
  // or badly balanced enumeration never times out spuriously.
  bool attach(const char* name, int rank, int world, int device, double timeout_s);
  bool barrier();
  // cudaStreamSynchronize that heartbeats while the GPU works (use before a barrier).
  cudaError_t wait_stream(cudaStream_t st);
  bool broken() const;   // a barrier failed on some rank: every later barrier fails fast
  void detach();

  int rank = 0, world = 1;
  uint8_t* local = nullptr;              // this rank's exchange buffer (device)
  uint8_t* peer[PEER_MAX] = {};          // every rank's buffer in this process (peer[rank] == local)
  double timeout_s = 120.0;
  uint64_t exchanges = 0;                // elite exchanges so far (selects the parity half)
  std::string err;

 private:
  struct Shm;
  Shm* shm_ = nullptr;
  size_t shm_bytes_ = 0;
  bool broken_ = false;
  void heartbeat();
  int device_ = -1;
  std::string name_;
};

}  // namespace sat
