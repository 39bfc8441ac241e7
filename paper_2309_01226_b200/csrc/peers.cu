// Peer-memory transport (see peers.h): POSIX shared-memory rendezvous + barrier, CUDA IPC
// mapping of every rank's exchange buffer.
#include "peers.h"

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <new>

namespace sat {

namespace {
constexpr uint32_t MAGIC = 0x53415455u;  // "SATU"
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void pause_briefly(int spins) {
  if (spins < 64) {
    sched_yield();
  } else {
    timespec ts{0, 20000};  // 20 us
    nanosleep(&ts, nullptr);
  }
}
}  // namespace

static uint64_t mono_ms() {   // CLOCK_MONOTONIC: one clock for every process of the host
  timespec ts{};
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000u + (uint64_t)(ts.tv_nsec / 1000000);
}

struct PeerLink::Shm {
  std::atomic<uint32_t> magic;
  int32_t world;
  std::atomic<uint32_t> count;       // arrivals at the current barrier
  std::atomic<uint32_t> generation;  // bumped by the last arrival
  std::atomic<uint32_t> broken;      // set by a rank whose barrier failed: the link is poisoned
  std::atomic<uint64_t> beat[PEER_MAX];   // last heartbeat of every rank (mono_ms)
  std::atomic<uint32_t> published[PEER_MAX];
  int32_t device[PEER_MAX];
  int32_t has_buffer[PEER_MAX];
  cudaIpcMemHandle_t handle[PEER_MAX];
};

void PeerLink::heartbeat() {
  if (shm_) shm_->beat[rank].store(mono_ms(), std::memory_order_relaxed);
}

bool PeerLink::broken() const {
  return broken_ || (shm_ && shm_->broken.load(std::memory_order_acquire) != 0);
}

cudaError_t PeerLink::wait_stream(cudaStream_t st) {
  for (int spins = 0;; ++spins) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e != cudaErrorNotReady) return e;
    if ((spins & 63) == 0) heartbeat();
    timespec ts{0, 50000};  // 50 us
    nanosleep(&ts, nullptr);
  }
}

bool PeerLink::barrier() {
  if (!shm_) {
    err = "peer link not attached";
    return false;
  }
  if (broken()) {
    broken_ = true;
    err = "peer link broken by an earlier failed barrier (re-attach to continue)";
    return false;
  }
  heartbeat();
  const uint32_t g = shm_->generation.load(std::memory_order_acquire);
  if (shm_->count.fetch_add(1, std::memory_order_acq_rel) + 1 == (uint32_t)world) {
    shm_->count.store(0, std::memory_order_relaxed);
    shm_->generation.fetch_add(1, std::memory_order_release);
    return true;
  }
  const uint64_t limit = (uint64_t)(timeout_s * 1000.0);
  for (int spins = 0; shm_->generation.load(std::memory_order_acquire) == g; ++spins) {
    if ((spins & 255) == 0) {
      heartbeat();
      if (shm_->broken.load(std::memory_order_acquire)) {
        broken_ = true;
        err = "peer barrier: another rank's barrier failed (link broken)";
        return false;
      }
      const uint64_t now = mono_ms();
      for (int q = 0; q < world; ++q) {
        const uint64_t b = shm_->beat[q].load(std::memory_order_relaxed);
        if (now > b && now - b > limit) {   // q stopped heartbeating: dead or hung outside the library
          broken_ = true;
          shm_->broken.store(1, std::memory_order_release);
          char m[200];
          snprintf(m, sizeof m, "peer barrier: rank %d silent for %.0f s (rank %d waiting; link now broken)", q,
                   (now - b) / 1000.0, rank);
          err = m;
          return false;
        }
      }
    }
    pause_briefly(spins);
  }
  return true;
}

bool PeerLink::attach(const char* name, int rank_, int world_, int device, double timeout) {
  detach();
  err.clear();
  if (!name || name[0] != '/' || world_ < 1 || world_ > PEER_MAX || rank_ < 0 || rank_ >= world_) {
    err = "attach_peers: need a '/name', 1 <= world <= 8 and 0 <= rank < world";
    return false;
  }
  rank = rank_;
  world = world_;
  timeout_s = timeout;
  device_ = device;
  name_ = name;
  shm_bytes_ = sizeof(Shm);
  const double t0 = now_s();
  int fd = -1;
  if (rank == 0) {
    fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) {
      err = std::string("attach_peers: shm_open(create ") + name + ") failed: " + strerror(errno);
      return false;
    }
    if (ftruncate(fd, (off_t)shm_bytes_) != 0) {
      err = std::string("attach_peers: ftruncate failed: ") + strerror(errno);
      close(fd);
      shm_unlink(name);
      return false;
    }
  } else {
    for (int spins = 0;; ++spins) {  // wait for rank 0 to create and size the segment
      fd = shm_open(name, O_RDWR, 0600);
      if (fd >= 0) {
        struct stat st{};
        if (fstat(fd, &st) == 0 && (size_t)st.st_size >= shm_bytes_) break;
        close(fd);
        fd = -1;
      }
      if (now_s() - t0 > timeout_s) {
        err = std::string("attach_peers: segment ") + name + " did not appear (is rank 0 running?)";
        return false;
      }
      pause_briefly(spins);
    }
  }
  void* m = mmap(nullptr, shm_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (m == MAP_FAILED) {
    err = std::string("attach_peers: mmap failed: ") + strerror(errno);
    if (rank == 0) shm_unlink(name);
    return false;
  }
  shm_ = static_cast<Shm*>(m);
  if (rank == 0) {
    memset(m, 0, shm_bytes_);
    new (&shm_->count) std::atomic<uint32_t>(0);
    new (&shm_->generation) std::atomic<uint32_t>(0);
    new (&shm_->broken) std::atomic<uint32_t>(0);
    for (int r = 0; r < PEER_MAX; ++r) new (&shm_->beat[r]) std::atomic<uint64_t>(mono_ms());
    for (int r = 0; r < PEER_MAX; ++r) new (&shm_->published[r]) std::atomic<uint32_t>(0);
    shm_->world = world;
    shm_->magic.store(MAGIC, std::memory_order_release);
  } else {
    for (int spins = 0; shm_->magic.load(std::memory_order_acquire) != MAGIC; ++spins) {
      if (now_s() - t0 > timeout_s) {
        err = "attach_peers: segment never initialised by rank 0";
        detach();
        return false;
      }
      pause_briefly(spins);
    }
    if (shm_->world != world) {
      err = "attach_peers: ranks disagree on world size";
      detach();
      return false;
    }
  }
  // this rank's exchange buffer, exported
  if (device_ >= 0) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&local), PeerLayout::bytes);
    if (e == cudaSuccess) e = cudaMemset(local, 0, PeerLayout::bytes);
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&shm_->handle[rank], local);
    if (e != cudaSuccess) {
      err = std::string("attach_peers: exchange buffer: ") + cudaGetErrorString(e);
      detach();
      return false;
    }
    shm_->device[rank] = device_;
    shm_->has_buffer[rank] = 1;
  }
  shm_->published[rank].store(1, std::memory_order_release);
  if (!barrier()) return false;
  // map every peer's buffer
  for (int q = 0; q < world; ++q) {
    if (q == rank) {
      peer[q] = local;
      continue;
    }
    if (device_ < 0) continue;
    if (!shm_->has_buffer[q]) {
      err = "attach_peers: a peer attached without a device (host-only and device ranks mixed)";
      detach();
      return false;
    }
    void* ptr = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&ptr, shm_->handle[q], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      err = std::string("attach_peers: cudaIpcOpenMemHandle(rank ") + std::to_string(q) +
            "): " + cudaGetErrorString(e);
      detach();
      return false;
    }
    peer[q] = static_cast<uint8_t*>(ptr);
  }
  if (!barrier()) return false;
  if (rank == 0) shm_unlink(name);  // every rank holds its mapping; the name is no longer needed
  return true;
}

void PeerLink::detach() {
  broken_ = false;
  for (int q = 0; q < PEER_MAX; ++q) {
    if (peer[q] && peer[q] != local) cudaIpcCloseMemHandle(peer[q]);
    peer[q] = nullptr;
  }
  if (local) cudaFree(local);
  local = nullptr;
  if (shm_) munmap(shm_, shm_bytes_);
  shm_ = nullptr;
}

}  // namespace sat
