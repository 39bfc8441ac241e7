// Device-side building blocks shared by the saturn kernels (sm_100a only).
//
// Nothing here is shared with oracle/ (the CPU reference); see DESIGN.md "Boundary".
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "saturn kernels are written for sm_100a (B200) only"
#endif

namespace sat {

constexpr int INF = 0x7fffffff;          // "never free" / padded GPU slot
constexpr int MAX_JOBS = 255;            // u8 genes
constexpr int MAX_GPUS = 32;             // sum_n GPU_n (one warp of lanes in the W decoder)
constexpr int MAX_NODES = 32;
constexpr uint32_t R_MASK = 0x00ffffffu; // config word = (g << 24) | R, R < 2^24 s

// Problem description passed by value to every kernel.  The packed config table
// (u32 words, job-major, `stride` words per job) is followed in the same allocation by
// S[t] (u8, configs per job) and the UPP id of every config; `blob_bytes` (multiple of 16)
// covers the table and S so one bulk copy stages what the decoders read into shared memory
// (the UPP ids only matter to the trace decoder, which stages `full_bytes`).
struct Problem {
  const uint8_t* blob;     // device: tab[T*stride] u32, S[T] u8, GPU_n[N] u8, upp[T*stride] u8, zero padded
  int blob_bytes;          // staged prefix: tab + S + GPU_n, rounded up to 16 (all the decoders read)
  int full_bytes;          // the whole blob incl. the UPP ids (the trace decoder only)
  int T;                   // jobs
  int stride;              // words per job row = max_t S_t
  int N;                   // nodes
  int sumG;                // sum_n GPU_n
  int8_t gpu_n[MAX_NODES]; // GPU_n
  int full_nodes;          // 1: one node with exactly GP GPUs (decode reads the makespan off the state)
  int one;                 // 1, opaque to ptxas (predicated FMA-pipe moves, decode.cuh pmov_fma)
};

__device__ __forceinline__ const uint32_t* tab_of(const uint8_t* blob) {
  return reinterpret_cast<const uint32_t*>(blob);
}
__device__ __forceinline__ const uint8_t* S_of(const uint8_t* blob, const Problem& pb) {
  return blob + 4 * pb.T * pb.stride;
}
// GPU_n of every node, right after S in the staged blob: indexing the kernel parameter
// pb.gpu_n with a runtime node id would copy the whole Problem to local memory.
__device__ __forceinline__ const uint8_t* G_of(const uint8_t* S, const Problem& pb) { return S + pb.T; }

// ------------------------------------------------------------------ TMA bulk staging
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// 1-D TMA: cp.async.bulk global -> shared, completion counted on an mbarrier (SASS UBLKCP).
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Stage the problem blob into shared memory (one elected thread issues, all wait).
// Must be called by every thread of the block; `bar` is a fresh shared mbarrier.
__device__ __forceinline__ void stage_problem(uint8_t* s_blob, const Problem& pb, uint64_t* bar) {
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_expect_tx(bar, pb.blob_bytes);
    bulk_g2s(s_blob, pb.blob, pb.blob_bytes, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
}

// ------------------------------------------------------------------ Philox4x32-10
// Salmon et al. SC'11; counters (c0, c1, c2, c3) and key (k0, k1); 10 rounds.
__device__ __forceinline__ uint4 philox_block(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2,
                                              uint32_t c3) {
  uint32_t x0 = c0, x1 = c1, x2 = c2, x3 = c3, a = k0, b = k1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { a += 0x9E3779B9u; b += 0xBB67AE85u; }
    const uint32_t hi0 = __umulhi(0xD2511F53u, x0), lo0 = 0xD2511F53u * x0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, x2), lo1 = 0xCD9E8D57u * x2;
    const uint32_t y0 = hi1 ^ x1 ^ a, y2 = hi0 ^ x3 ^ b;
    x0 = y0; x1 = lo1; x2 = y2; x3 = lo0;
  }
  return make_uint4(x0, x1, x2, x3);
}

// Word k of the stream (c0, c1, c2): word k % 4 of block k / 4.
__device__ __forceinline__ uint32_t philox_word(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2,
                                                uint32_t k) {
  const uint4 v = philox_block(k0, k1, c0, c1, c2, k >> 2);
  const uint32_t j = k & 3u;
  return j == 0 ? v.x : (j == 1 ? v.y : (j == 2 ? v.z : v.w));
}

// U(n) = (u32 * n) >> 32, an integer in [0, n)
__device__ __forceinline__ uint32_t ubelow(uint32_t u, uint32_t n) { return (uint32_t)(((uint64_t)u * n) >> 32); }
// V(n) on a 16-bit field h: (h * n) >> 16, an integer in [0, n) for n <= 65536
__device__ __forceinline__ uint32_t v16(uint32_t h, uint32_t n) { return (h * n) >> 16; }

// Sequential stream: word k = word k % 4 of block k / 4 (used where every lane draws the
// same number of words at the same program points, so refills never diverge).
struct Philox {
  uint32_t k0, k1, c0, c1, c2, block;
  uint32_t b0, b1, b2, b3;  // unread words of the current block, consumed front first
  int left;
  __device__ __forceinline__ Philox(uint64_t seed, uint32_t a, uint32_t b, uint32_t c)
      : k0((uint32_t)seed), k1((uint32_t)(seed >> 32)), c0(a), c1(b), c2(c), block(0), left(0) {}
  __device__ __forceinline__ uint32_t u32() {
    if (left == 0) {
      const uint4 v = philox_block(k0, k1, c0, c1, c2, block);
      b0 = v.x; b1 = v.y; b2 = v.z; b3 = v.w;
      ++block;
      left = 4;
    }
    const uint32_t v = b0;
    b0 = b1; b1 = b2; b2 = b3;
    --left;
    return v;
  }
  __device__ __forceinline__ uint32_t below(uint32_t n) { return ubelow(u32(), n); }
};

// Fixed-position words: word(k) for any k, recomputing block k / 4 only when it changes.
// Callers request words at warp-uniform program points with warp-uniform k.
struct PhiloxWords {
  uint32_t k0, k1, c0, c1, c2;
  uint32_t blk;
  uint4 cur;
  __device__ __forceinline__ PhiloxWords(uint64_t seed, uint32_t a, uint32_t b, uint32_t c)
      : k0((uint32_t)seed), k1((uint32_t)(seed >> 32)), c0(a), c1(b), c2(c), blk(0xffffffffu) {}
  __device__ __forceinline__ uint4 block(uint32_t b) const { return philox_block(k0, k1, c0, c1, c2, b); }
  __device__ __forceinline__ uint32_t word(uint32_t k) {
    if ((k >> 2) != blk) { blk = k >> 2; cur = block(blk); }
    const uint32_t j = k & 3u;
    return j == 0 ? cur.x : (j == 1 ? cur.y : (j == 2 ? cur.z : cur.w));
  }
};

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  lo = __shfl_xor_sync(0xffffffffu, lo, m);
  hi = __shfl_xor_sync(0xffffffffu, hi, m);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    uint64_t o = shfl_xor_u64(v, m);
    v = o < v ? o : v;
  }
  return v;
}

}  // namespace sat
