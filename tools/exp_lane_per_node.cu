// Experiment (not product code): the "lane-per-node" T-design variant of SURVEY.md §8a-a5
// (SURVEY.md:483-489) for multi-node clusters, measured against the library's decoders
// (VERDICT r1 "Next round" item 4).  NN lanes decode one genome: lane `node` keeps that
// node's sorted free-time vector (GP registers), its start for a g-GPU job is its own
// a[g-1], the group's earliest start (ties to the lowest node) comes from a shuffle-xor
// min over (start << 2 | node), and only the winning lane updates its vector with the
// closed-form sorted update (same semantics as decode.cuh, reading A6).
//
// Built and driven by tools/exp_lane_per_node.py:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
//        -o tools/libexp_lanes.so tools/exp_lane_per_node.cu
#include <cstdint>
#include <cuda_runtime.h>

namespace {
constexpr int INF = 0x7fffffff;
constexpr int B = 128;   // threads per block

template <int GP>
__device__ __forceinline__ int mux(const int (&a)[GP], int k) {
  if constexpr (GP == 1) {
    return a[0];
  } else {
    int v[GP / 2];
#pragma unroll
    for (int i = 0; i < GP / 2; ++i) v[i] = (k & 1) ? a[2 * i + 1] : a[2 * i];
    return mux<GP / 2>(v, k >> 1);
  }
}

// the sorted update of decode.cuh (selects written plainly: this is an experiment)
template <int GP>
__device__ __forceinline__ void place(int (&x)[GP], int g, int R) {
  const int k = g - 1;
  int b[GP];
#pragma unroll
  for (int i = 0; i < GP; ++i) b[i] = x[i];
#pragma unroll
  for (int sh = 1; sh < GP; sh <<= 1) {
    const bool on = (k & sh) != 0;
#pragma unroll
    for (int i = 0; i < GP; ++i) b[i] = on ? ((i + sh < GP) ? b[i + sh] : INF) : b[i];
  }
  const int s = b[0], v = s + R;
#pragma unroll
  for (int i = 0; i < GP; ++i) {
    const int bn = (i + 1 < GP) ? b[i + 1] : INF;
    x[i] = (bn <= s) ? x[i] : min(bn, max(x[i], v));
  }
}

// One block = B / NN genomes per tile; genomes staged into shared memory (coalesced).
template <int NN, int GP>
__global__ void __launch_bounds__(B) k_lanes(const uint32_t* __restrict__ tab_g, int stride, int T,
                                             const uint8_t* __restrict__ gpu_n, const uint8_t* __restrict__ cfg,
                                             const uint8_t* __restrict__ perm, int64_t n, int32_t* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int GPB = B / NN;   // genomes per tile
  uint32_t* tab = reinterpret_cast<uint32_t*>(sm);
  uint8_t* sc = sm + 4 * ((T * stride + 3) & ~3);
  uint8_t* sp = sc + GPB * T;
  for (int i = threadIdx.x; i < T * stride; i += B) tab[i] = tab_g[i];
  const int lane = threadIdx.x & 31, node = lane % NN, sub = threadIdx.x / NN;
  const int my_g = gpu_n[node];
  const int64_t ntiles = (n + GPB - 1) / GPB;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t first = tile * GPB;
    const int cnt = (int)min((int64_t)GPB, n - first) * T;
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += B) {
      sc[k] = cfg[first * T + k];
      sp[k] = perm[first * T + k];
    }
    __syncthreads();
    const bool live = first + sub < n;
    const uint8_t* c = sc + sub * T;
    const uint8_t* p = sp + sub * T;
    int a[GP];
#pragma unroll
    for (int i = 0; i < GP; ++i) a[i] = (i < my_g) ? 0 : INF;
    int ms = 0;
    for (int q = 0; q < T; ++q) {
      const int t = live ? p[q] : 0;
      const int cc = live ? c[t] : 0;
      const uint32_t w = tab[t * stride + cc];
      const int g = (int)(w >> 24), R = (int)(w & 0xffffffu);
      const int st = mux<GP>(a, g - 1);
      uint32_t key = (st == INF) ? 0xffffffffu : (((uint32_t)st << 2) | (uint32_t)node);
#pragma unroll
      for (int m = 1; m < NN; m <<= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, m));
      if ((int)(key & 3u) == node) place<GP>(a, g, R);
      ms = max(ms, (int)(key >> 2) + R);
    }
    if (node == 0 && live) out[first + sub] = ms;
  }
}
}  // namespace

extern "C" int exp_lanes_evaluate(const uint32_t* d_tab, int stride, int T, int N, const uint8_t* d_gpu_n,
                                  const uint8_t* d_cfg, const uint8_t* d_perm, int64_t n, int32_t* d_out,
                                  cudaStream_t st) {
  const size_t smem = 4 * ((T * stride + 3) & ~3) + 2 * (B / N) * T;
  int sms = 0, dev = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (N == 4) {
    cudaFuncSetAttribute(k_lanes<4, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lanes<4, 8>, B, smem);
    k_lanes<4, 8><<<sms * occ, B, smem, st>>>(d_tab, stride, T, d_gpu_n, d_cfg, d_perm, n, d_out);
  } else if (N == 2) {
    cudaFuncSetAttribute(k_lanes<2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lanes<2, 8>, B, smem);
    k_lanes<2, 8><<<sms * occ, B, smem, st>>>(d_tab, stride, T, d_gpu_n, d_cfg, d_perm, n, d_out);
  } else {
    return -1;
  }
  return (int)cudaGetLastError();
}
