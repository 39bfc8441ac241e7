// The SPASE plan decoders (row a5 of SURVEY.md §8): genome -> integer makespan.
//
// Semantics (reading A6): jobs are placed in priority order
// perm[0..T); job t with config (g, R) = table[t][cfg[t]] starts at the g-th smallest free
// time of the node where that start is earliest (ties -> lowest node id); it takes the g
// GPUs of that node that are free by then with the LATEST free times (ties -> lower GPU
// id) and holds them for [s, s + R).  makespan = max_t (s_t + R_t)   (Eq. 2).
// One config per job and one node per job (Eq. 3), exactly g GPUs (Eqs. 4-5),
// one start for all of them (gang, Eqs. 8-9), no overlap on a GPU (Eqs. 10-11).
//
// Two device designs:
//   T  decode_sorted<NN, GP>  one thread per genome; each node's free times are kept as a
//      SORTED multiset in registers (GP slots, +inf padded).  Starts and makespans depend
//      only on those multisets, and the latest-free-first pick becomes a closed-form update
//        b = a shifted left by g-1 (so b[0] = a[g-1] = s),  v = s + R,
//        a'[i] = (b[i+1] <= s) ? a[i] : min(b[i+1], max(a[i], v))
//      (b[i+1] = a[i+g] <= s  <=>  i < m-g with m = #{a <= s}: the kept prefix; the rest is
//      the merge of a[m..] with g copies of v).  No GPU ids: used for throughput.
//   W  decode_warp            lanes = GPUs (node-major inside a pow2 segment, 32/seg genomes
//      per warp).  Each lane ranks its free time inside its node with warp shuffles, the
//      start of every node comes from a ballot, the earliest node from a shuffle-xor min,
//      and the chosen GPUs from a ballot count -- the north-star design.  It yields the GPU
//      ids, so it also produces the trace (row a8).
#pragma once
#include "common.cuh"

namespace sat {

#ifndef SAT_NODE_KEYS
#define SAT_NODE_KEYS 1   // multi-node register states hold (t << 2 | node) keys
#endif

// a[k] for a runtime k in [0, GP): binary mux tree on the bits of k (GP-1 selects).
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

// Select on the FMA pipe: p in {0, 1} -> p ? b : a, as a + p * (b - a) with two IMADs.
// The decode is ALU-pipe bound (SEL / VIMNMX / ISETP all issue there at half rate); moving
// part of the barrel shift onto the otherwise idle FMA pipe lets both pipes issue.
__device__ __forceinline__ int sel_fma(int p, int a, int b) {
  int d, r;
  asm("mad.lo.s32 %0, %1, -1, %2;" : "=r"(d) : "r"(a), "r"(b));
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(p), "r"(d), "r"(a));
  return r;
}

// Predicated move on the FMA pipe: if (p) d = s, as `@p IMAD d, s, one, RZ` with `one` a
// run-time 1 (Problem::one) that ptxas cannot fold -- a predicated MOV would become an ALU
// SEL.  One FMA-pipe instruction per element of an in-place barrel-shift stage.
// `bit` is tested for != 0 (pass k & sh, not a 0/1 value: one LOP3 makes the predicate).
__device__ __forceinline__ void pmov_fma(int& d, int s, int bit, int one) {
  asm("{.reg .pred q; setp.ne.b32 q, %2, 0; @q mad.lo.s32 %0, %1, %3, 0;}" : "+r"(d) : "r"(s), "r"(bit), "r"(one));
}
// if (bit) d = +inf, in place: d * zero + inf with a run-time zero (a loop-invariant
// `one * inf` would be hoisted and the predicated move turned back into an ALU SEL).
__device__ __forceinline__ void pinf_fma(int& d, int bit, int zero) {
  asm("{.reg .pred q; setp.ne.b32 q, %1, 0; @q mad.lo.s32 %0, %0, %2, 2147483647;}" : "+r"(d) : "r"(bit), "r"(zero));
}

// if (sel == N) d = s, in place on the FMA pipe (the multi-node gather / scatter of the
// chosen node's vector; ptxas shares the compare across the lanes).  Written as
// d = d * zero + s so the product depends on d: with s * one, ptxas computes it once for
// all nodes and turns every predicated move back into an ALU SEL.
template <int N>
__device__ __forceinline__ void pmov_eq(int& d, int s, int sel, int zero) {
  asm("{.reg .pred q; setp.eq.s32 q, %2, %4; @q mad.lo.s32 %0, %0, %3, %1;}" : "+r"(d) : "r"(s), "r"(sel), "r"(zero), "n"(N));
}

// Chosen node's vector out of / back into the register states a[NN][GP] (multi-node T
// design).  The first two gather steps are selects (ALU), the rest predicated moves (FMA
// pipe): the 4-node decode was ALU-bound on these selects (r2: 103 ALU + 59 FMA per job
// step; now 79 + 75).
template <int NN, int GP, int N = 1>
__device__ __forceinline__ void gather_node(int (&x)[GP], const int (&a)[NN][GP], int bn, int one) {
  if constexpr (N < NN) {
#pragma unroll
    for (int i = 0; i < GP; ++i) {
      if constexpr (N == 1) x[i] = (bn == 1) ? a[1][i] : a[0][i];
      else if constexpr (N == 2) x[i] = (bn == 2) ? a[2][i] : x[i];   // (pipe balance, 4 nodes)
      else pmov_eq<N>(x[i], a[N][i], bn, one - 1);
    }
    gather_node<NN, GP, N + 1>(x, a, bn, one);
  } else if constexpr (NN == 1) {
#pragma unroll
    for (int i = 0; i < GP; ++i) x[i] = a[0][i];
  }
}
template <int NN, int GP, int N = 0>
__device__ __forceinline__ void scatter_node(int (&a)[NN][GP], const int (&x)[GP], int bn, int one) {
  if constexpr (N < NN) {
#pragma unroll
    for (int i = 0; i < GP; ++i) pmov_eq<N>(a[N][i], x[i], bn, one - 1);
    scatter_node<NN, GP, N + 1>(a, x, bn, one);
  }
}

// In-place update of one node's sorted free-time vector after placing (g, R) at its
// g-th smallest free time.  Returns s + R.  `one` = Problem::one.
// The barrel shift is all on the FMA pipe (the decode's binding pipe is the ALU: VIMNMX /
// ISETP / SEL): b[i] <- b[i + sh] in place (ascending i reads lanes this stage has not
// written), lanes past the end shift in +inf; the first stage's lanes still read x, so they
// are two-source selects (the IMAD pair).  r1 ran every lane as an IMAD pair and the +inf
// lanes as ALU selects: 84 instead of 72 SASS per one-node step.
template <int GP>
__device__ __forceinline__ int place_sorted(int (&x)[GP], int g, int R, int one) {
  const int k = g - 1;
  int b[GP];
#pragma unroll
  for (int i = 0; i < GP; ++i) b[i] = x[i];
  int stage = 0;
#pragma unroll
  for (int sh = 1; sh < GP; sh <<= 1, ++stage) {
    const int p = (k >> stage) & 1;
#pragma unroll
    for (int i = 0; i < GP; ++i) {
      if (stage == 0)
        b[i] = sel_fma(p, b[i], (i + sh >= GP) ? INF : b[i + sh]);
      else if (i + sh >= GP)
        pinf_fma(b[i], k & sh, one - 1);
      else
        pmov_fma(b[i], b[i + sh], k & sh, one);
    }
  }
  const int s = b[0];
  const int v = s + R;
#pragma unroll
  for (int i = 0; i < GP; ++i) {
    const int bn = (i + 1 < GP) ? b[i + 1] : INF;
    const int merged = min(bn, max(x[i], v));
    x[i] = (bn <= s) ? x[i] : merged;
  }
  return v;
}

// Genome accessors.  RowGenome reads a genome stored as two T-byte rows (the caller's
// [n][T] layout, staged tile by tile).  RowG reads a thread-private genome row in shared
// memory: cfg at bytes [0, T), perm at [Tp, Tp + T) with Tp = roundup4(T) (the GA record
// layout); rows are an odd number of words apart, so same-index accesses of a warp are
// bank-conflict free and every byte address is one add.
struct RowGenome {
  const uint8_t* c;
  const uint8_t* p;
  __device__ __forceinline__ int cfg(int t) const { return c[t]; }
  __device__ __forceinline__ int perm(int i) const { return p[i]; }
};
struct RowG {
  uint8_t* base;
  int Tp;
  __device__ __forceinline__ uint8_t& c(int t) const { return base[t]; }
  __device__ __forceinline__ uint8_t& q(int i) const { return base[Tp + i]; }
  __device__ __forceinline__ int cfg(int t) const { return base[t]; }
  __device__ __forceinline__ int perm(int i) const { return base[Tp + i]; }
};
__host__ __device__ __forceinline__ int perm_offset(int T) { return (T + 3) & ~3; }
// record bytes of a genome (cfg | pad | perm | pad), multiple of 16
__host__ __device__ __forceinline__ int record_bytes(int T) { return (perm_offset(T) + T + 15) & ~15; }
// smem row stride >= bytes, an odd number of 4-byte words
__host__ __device__ __forceinline__ int odd_row_stride(int bytes) {
  int w = (bytes + 3) / 4;
  if ((w & 1) == 0) ++w;
  return 4 * w;
}

// T design.  `tab` = packed (g << 24 | R) words [T][stride] in shared memory (column
// stride-1 of every row is a zero sentinel), `S` the configs per job; `gen` a genome accessor.
// CHECK = 0: genome trusted.  CHECK = 1 (T <= 32) / 2 (any T): invalid genomes (perm not a
// permutation of 0..T-1, cfg[t] >= S_t) return -1; mode 1 keeps the seen-set in a register,
// mode 2 in `mask` (this thread's ceil(T/32) scratch words, `mstride` words apart).
// TRACK_MS = false (every node has exactly GP GPUs): the makespan is read off the final
// state instead of a running max -- a GPU's free time is the end of its last job, every job
// holds >= 1 GPU and a later job on a GPU ends later, so max_t (s_t + R_t) = max over the
// GPUs of their final free time = max over nodes of the sorted vector's last slot.
template <int NN, int GP, int CHECK, bool TRACK_MS, class G>
__device__ __forceinline__ int decode_sorted_impl(const uint32_t* __restrict__ tab, const uint8_t* __restrict__ S,
                                                  int stride, const G& gen, int T, const Problem& pb,
                                                  uint32_t* mask, int mstride);

template <int NN, int GP, int CHECK, class G>
__device__ __forceinline__ int decode_sorted(const uint32_t* __restrict__ tab, const uint8_t* __restrict__ S,
                                             int stride, const G& gen, int T, const Problem& pb,
                                             uint32_t* mask = nullptr, int mstride = 0) {
  if constexpr (NN == 1 && GP >= 8) {   // (the only shapes the host flags; smaller ones keep one loop copy)
    if (pb.full_nodes) return decode_sorted_impl<NN, GP, CHECK, false>(tab, S, stride, gen, T, pb, mask, mstride);
  }
  return decode_sorted_impl<NN, GP, CHECK, true>(tab, S, stride, gen, T, pb, mask, mstride);
}

template <int NN, int GP, int CHECK, bool TRACK_MS, class G>
__device__ __forceinline__ int decode_sorted_impl(const uint32_t* __restrict__ tab, const uint8_t* __restrict__ S,
                                                  int stride, const G& gen, int T, const Problem& pb,
                                                  uint32_t* mask, int mstride) {
  bool bad = false;
  int maxt = 0;
  uint32_t seen = 0u, minw = 0xffffffffu;
  if constexpr (CHECK == 2) {
    for (int w = 0; w < (T + 31) / 32; ++w) mask[w * mstride] = 0u;
  }
  // config word (g << 24 | R) of the job at priority position p (+ the validity bookkeeping)
  const auto fetch = [&](int p) -> uint32_t {
    int t = gen.perm(p);
    int c;
    if constexpr (CHECK != 0) {
      maxt = max(maxt, t);
      t = min(t, T - 1);
      if constexpr (CHECK == 1) {
        seen |= 1u << t;
      } else {
        uint32_t* mw = mask + (t >> 5) * mstride;
        const uint32_t bit = 1u << (t & 31);
        const uint32_t m = *mw;
        bad |= (m & bit) != 0;
        *mw = m | bit;
      }
      c = min(gen.cfg(t), stride - 1);   // out-of-range genes land on the zero sentinel
    } else {
      c = gen.cfg(t);
    }
    const uint32_t w = tab[t * stride + c];
    if constexpr (CHECK != 0) minw = min(minw, w);
    return w;
  };
  // Position 0 in closed form: every GPU is free at 0, so the first job starts at 0 on the
  // lowest node with >= g GPUs and (latest-free-first = all equal, lower ids first ... in the
  // multiset view: the g top slots of that node's GPU_n free ones) ends at R.
  // Several nodes: every free time is held as a node KEY (t << 2 | n).  Keys of one node
  // order like their times, so the sorted update runs on keys unchanged (with R << 2), and
  // the earliest start over the nodes with ties to the lowest node id is a plain min of the
  // nodes' g-th keys -- its low bits are the node (no compare / select chain).
  constexpr int KS = (NN >= 2 && SAT_NODE_KEYS) ? 2 : 0;
  int a[NN][GP];
  int ms;
  {
    const uint32_t w = fetch(0);
    const int g = (int)(w >> 24);
    const int R = (int)(w & R_MASK);
    if (NN == 1 && pb.full_nodes) {   // one node of exactly GP GPUs: R in the top g slots
#pragma unroll
      for (int i = 0; i < GP; ++i) a[0][i] = (i >= GP - g) ? R : 0;
    } else {
      int bn = NN;
#pragma unroll
      for (int n = NN - 1; n >= 0; --n) bn = (n < pb.N && g <= pb.gpu_n[n]) ? n : bn;
#pragma unroll
      for (int n = 0; n < NN; ++n) {
        const int gn = n < pb.N ? pb.gpu_n[n] : 0;
#pragma unroll
        for (int i = 0; i < GP; ++i)
          a[n][i] = (i < gn) ? ((((n == bn && i >= gn - g) ? R : 0) << KS) | (KS ? n : 0)) : INF;
      }
    }
    ms = R << KS;
  }
  // Positions 1 .. T-2: the full update.  The next position's config word is fetched one
  // step ahead (its three dependent shared-memory loads -- perm byte, cfg byte, table word
  // -- overlap this step's arithmetic instead of stalling the next one).
  // (4-node states: +1.6 % SWEEP k_ga in r1 at 128 registers; -0.6 % since the node keys and
  // the min-then-mux node choice freed registers, r2.)
  constexpr bool AHEAD = NN <= 4;
  uint32_t w = (AHEAD && T > 1) ? fetch(1) : 0u;
  // Unrolled by two (the loop counter and its compare once per two steps): SWEEP k_ga -2.8 %,
  // TXT / MIX equal (r2).  First-stage shift lanes as ALU selects instead of IMAD pairs:
  // TXT -0.3 %, SWEEP +2 % -- not adopted.
#pragma unroll 2
  for (int p = 1; p < T - 1; ++p) {
    if (!AHEAD) w = fetch(p);
    const uint32_t wn = AHEAD ? fetch(p + 1) : 0u;
    const int g = (int)(w >> 24);
    const int R = (int)(w & R_MASK);
    int v;
    if constexpr (NN == 1) {
      v = place_sorted<GP>(a[0], g, R, pb.one);
    } else {
      // start of every node: its g-th smallest free time (+inf if it has fewer GPUs)
      int best;
      int bn = 0;
      if constexpr (KS) {
        // min over the nodes slot by slot (3-input VIMNMX3), then one mux: the g-th key of
        // the min vector is the min over the nodes of their g-th keys
        int m[GP];
#pragma unroll
        for (int i = 0; i < GP; ++i) {
          m[i] = a[0][i];
#pragma unroll
          for (int n = 1; n < NN; ++n) m[i] = min(m[i], a[n][i]);
        }
        best = mux<GP>(m, g - 1);
        bn = best & 3;
      } else {
        best = mux<GP>(a[0], g - 1);
#pragma unroll
        for (int n = 1; n < NN; ++n) {
          const int st = mux<GP>(a[n], g - 1);
          const bool lt = st < best;   // strict: ties keep the lowest node id
          best = lt ? st : best;
          bn = lt ? n : bn;
        }
      }
      int x[GP];
      gather_node<NN, GP>(x, a, bn, pb.one);
      v = place_sorted<GP>(x, g, R << KS, pb.one);
      scatter_node<NN, GP>(a, x, bn, pb.one);
    }
    if constexpr (TRACK_MS) ms = max(ms, v);
    if (AHEAD) w = wn;
  }
  if (!AHEAD && T > 1) w = fetch(T - 1);
  if constexpr (!TRACK_MS) {
    ms = 0;
#pragma unroll
    for (int n = 0; n < NN; ++n) ms = max(ms, a[n][GP - 1]);
  }
  ms >>= KS;
  // Position T-1 (its word is in w): only its end matters (no later job reads the state):
  // earliest start + R.
  if (T > 1) {
    const int g = (int)(w >> 24);
    const int R = (int)(w & R_MASK);
    int best = mux<GP>(a[0], g - 1);
#pragma unroll
    for (int n = 1; n < NN; ++n) best = min(best, mux<GP>(a[n], g - 1));
    ms = max(ms, (best >> KS) + R);
  }
  if constexpr (CHECK == 1) bad = __popc(seen) != T;
  if constexpr (CHECK != 0) {
    bad |= maxt >= T || minw == 0u;
    return bad ? -1 : ms;
  }
  return ms;
}

// Node-gene variant (row f4; SURVEY.md §8c O2 -- with the node in the genome the decoder
// space provably contains the SPASE optimum): job t runs on node nd[t], or picks greedily
// if nd[t] == 0xFF.  Always validity-checked: a node gene naming a missing node or one with
// fewer than g GPUs makes the genome invalid (-1), like a bad cfg / perm.
template <int NN, int GP>
__device__ __forceinline__ int decode_sorted_nodes(const uint32_t* __restrict__ tab, const uint8_t* G, int stride,
                                                   const uint8_t* cfg, const uint8_t* perm, const uint8_t* nd,
                                                   int T, const Problem& pb, uint32_t* mask, int mstride) {
  int a[NN][GP];
#pragma unroll
  for (int n = 0; n < NN; ++n)
#pragma unroll
    for (int i = 0; i < GP; ++i) a[n][i] = (n < pb.N && i < pb.gpu_n[n]) ? 0 : INF;
  bool bad = false;
  int maxt = 0;
  uint32_t minw = 0xffffffffu;
  for (int w = 0; w < (T + 31) / 32; ++w) mask[w * mstride] = 0u;
  int ms = 0;
  for (int p = 0; p < T; ++p) {
    int t = perm[p];
    maxt = max(maxt, t);
    t = min(t, T - 1);
    uint32_t* mw = mask + (t >> 5) * mstride;
    const uint32_t bit = 1u << (t & 31);
    const uint32_t m = *mw;
    bad |= (m & bit) != 0;
    *mw = m | bit;
    const int c = min((int)cfg[t], stride - 1);
    const uint32_t w = tab[t * stride + c];
    minw = min(minw, w);
    const int g = (int)(w >> 24);
    const int R = (int)(w & R_MASK);
    const int want = nd[t];
    int best = INF, bn = 0;
#pragma unroll
    for (int n = 0; n < NN; ++n) {
      const int st = mux<GP>(a[n], max(g - 1, 0));
      const bool allowed = (want == 0xFF) || (want == n);
      const bool lt = allowed && st < best;
      best = lt ? st : best;
      bn = lt ? n : bn;
    }
    bad |= (want != 0xFF) && (want >= pb.N || g > G[min(want, pb.N - 1)]);
    bad |= best == INF;
    int x[GP];
#pragma unroll
    for (int i = 0; i < GP; ++i) {
      int y = a[0][i];
#pragma unroll
      for (int n = 1; n < NN; ++n) y = (bn == n) ? a[n][i] : y;
      x[i] = y;
    }
    int v = place_sorted<GP>(x, max(g, 1), R, pb.one);
    if (best == INF) v = 0;
#pragma unroll
    for (int n = 0; n < NN; ++n)
#pragma unroll
      for (int i = 0; i < GP; ++i) a[n][i] = (bn == n && best != INF) ? x[i] : a[n][i];
    ms = max(ms, v);
  }
  bad |= maxt >= T || minw == 0u;
  return bad ? -1 : ms;
}

// Column node states (decode_col): node n's sorted slot j of thread `tid` is the word
// ns[(n * col_rows(GP, rshift) + j) * B + tid] of a block of B threads -- every thread's same slot in
// one row, so any per-thread slot index is bank-conflict free.  Rows GP .. 2GP-2 of every
// node are +inf padding: slot j + g (g <= GP, j <= GP-2) reads +inf past the node's GPUs.
// RSHIFT variant: no padding rows (the chosen node's vector is shifted in registers).
__host__ __device__ __forceinline__ constexpr int col_rows(int GP, bool rshift) { return rshift ? GP : 2 * GP - 1; }
__host__ __device__ __forceinline__ size_t col_state_bytes(int N, int GP, int B, bool rshift) {
  return (size_t)4 * N * col_rows(GP, rshift) * B;
}

// T design for multi-node clusters with the node states in shared memory, column layout
// (above).  NN = node count at compile time (0: pb.N at run time).  `ns` = &state[tid].
// Per job step: one load per node for the starts (slot g-1), a strict-< argmin, then the
// chosen node's slots are read twice -- x[i] = slot i and the shifted b[i+1] = slot i+g
// (the barrel shift of place_sorted done by the LSU's addressing instead of select stages)
// -- and the update x'[i] = (b[i+1] <= s) ? x[i] : min(b[i+1], max(x[i], s+R)) is stored
// back.  No gather/scatter selects, no shift stages, 8-slot register footprint.
// RSHIFT: the chosen node's vector is read (GP loads), shifted and updated in registers
// (place_sorted: predicated FMA-pipe moves) and stored back -- 7 fewer shared-memory loads
// per step than the shifted reads and no padding rows: the multi-node evaluate is bound by
// shared-memory wavefronts, and there this measured SWEEP 1.83e9 -> 2.23e9, MIX 1.08e10 ->
// 1.20e10 plans/s (r2); a single node (TXT -4 %) and the MIX GA (+11 % time, the GA's own
// shared traffic no longer dominates) keep the shifted reads.
template <int NN, int GP, int B, bool RSHIFT, int CHECK, class G>
__device__ __forceinline__ int decode_col(const uint32_t* __restrict__ tab, const uint8_t* __restrict__ S,
                                          int stride, const G& gen, int T, const Problem& pb, int* ns,
                                          uint32_t* mask = nullptr, int mstride = 0) {
  constexpr int RW = col_rows(GP, RSHIFT);
  // node keys (t << KS | n) as in decode_sorted: the argmin over the nodes is a min
  // (a run-time node count needs 5 bits: times < 2^26 keep keys below 2^31 - 32 < INF).
  // Measured r2: SWEEP 4x8 evaluate +1.7 %; two nodes -2.8 % (MIX) -- they keep times.
  constexpr int KS = (NN == 1 || NN == 2 || !SAT_NODE_KEYS) ? 0 : (NN == 0 ? 5 : (NN <= 4 ? 2 : 3));
  const int N = NN ? NN : pb.N;
  bool bad = false;
  int maxt = 0;
  uint32_t seen = 0u, minw = 0xffffffffu;
  if constexpr (CHECK == 2) {
    for (int w = 0; w < (T + 31) / 32; ++w) mask[w * mstride] = 0u;
  }
  const auto fetch = [&](int p) -> uint32_t {
    int t = gen.perm(p);
    int c;
    if constexpr (CHECK != 0) {
      maxt = max(maxt, t);
      t = min(t, T - 1);
      if constexpr (CHECK == 1) {
        seen |= 1u << t;
      } else {
        uint32_t* mw = mask + (t >> 5) * mstride;
        const uint32_t bit = 1u << (t & 31);
        const uint32_t m = *mw;
        bad |= (m & bit) != 0;
        *mw = m | bit;
      }
      c = min(gen.cfg(t), stride - 1);
    } else {
      c = gen.cfg(t);
    }
    const uint32_t w = tab[t * stride + c];
    if constexpr (CHECK != 0) minw = min(minw, w);
    return w;
  };
  // the smallest start over the nodes for a g-GPU job (slot g-1 of every node), its node
  const auto start_min = [&](int g, int& bn) -> int {
    const int* cg = ns + (g - 1) * B;
    int best = cg[0];
    bn = 0;
    if constexpr (KS > 0) {
      if constexpr (NN > 0) {
#pragma unroll
        for (int n = 1; n < NN; ++n) best = min(best, cg[n * RW * B]);
      } else {
        for (int n = 1; n < N; ++n) best = min(best, cg[n * RW * B]);
      }
      bn = best & ((1 << KS) - 1);
    } else if constexpr (NN > 0) {
#pragma unroll
      for (int n = 1; n < NN; ++n) {
        const int st = cg[n * RW * B];
        const bool lt = st < best;   // strict: ties keep the lowest node id
        best = lt ? st : best;
        bn = lt ? n : bn;
      }
    } else {
      for (int n = 1; n < N; ++n) {
        const int st = cg[n * RW * B];
        const bool lt = st < best;
        best = lt ? st : best;
        bn = lt ? n : bn;
      }
    }
    return best;
  };
  // Position 0 in closed form (every GPU free at 0): the lowest node with >= g GPUs gets
  // R in its top g free slots; padding rows +inf.
  int ms;
  {
    const uint32_t w = fetch(0);
    const int g = (int)(w >> 24);
    const int R = (int)(w & R_MASK);
    const uint8_t* Gn = G_of(S, pb);
    int bn = N;
    for (int n = N - 1; n >= 0; --n) bn = (g <= Gn[n]) ? n : bn;
#pragma unroll(NN > 0 ? NN : 1)
    for (int n = 0; n < N; ++n) {
      const int gn = Gn[n];
      const int lo = (n == bn) ? gn - g : gn;
      int* row = ns + n * RW * B;
#pragma unroll
      for (int j = 0; j < RW; ++j) row[j * B] = (j < gn) ? ((((j >= lo) ? R : 0) << KS) | (KS ? n : 0)) : INF;
    }
    ms = R << KS;
  }
  uint32_t w = T > 1 ? fetch(1) : 0u;
  for (int p = 1; p < T - 1; ++p) {
    const uint32_t wn = fetch(p + 1);   // next position's word one step ahead
    const int g = (int)(w >> 24);
    const int R = (int)(w & R_MASK);
    int bn;
    const int s = start_min(g, bn);
    const int v = s + (R << KS);
    int* row = ns + bn * RW * B;
    if constexpr (RSHIFT) {   // the shift in registers (predicated FMA-pipe moves)
      int x[GP];
#pragma unroll
      for (int i = 0; i < GP; ++i) x[i] = row[i * B];
      place_sorted<GP>(x, g, R << KS, pb.one);
#pragma unroll
      for (int i = 0; i < GP; ++i) row[i * B] = x[i];
    } else {
    const int* sh = row + g * B;   // sh[i * B] = slot i + g = b[i + 1]
    int x[GP], y[GP];
#pragma unroll
    for (int i = 0; i < GP; ++i) x[i] = row[i * B];
#pragma unroll
    for (int i = 0; i + 1 < GP; ++i) y[i] = sh[i * B];
#pragma unroll
    for (int i = 0; i < GP; ++i) {
      if (i + 1 < GP) {
        const int merged = min(y[i], max(x[i], v));
        row[i * B] = (y[i] <= s) ? x[i] : merged;
      } else {
        row[i * B] = max(x[i], v);
      }
    }
    }
    ms = max(ms, v);
    w = wn;
  }
  // Position T-1 (its word is in w): earliest start + R, no state update.
  ms >>= KS;
  if (T > 1) {
    int bn;
    ms = max(ms, (start_min((int)(w >> 24), bn) >> KS) + (int)(w & R_MASK));
  }
  if constexpr (CHECK == 1) bad = __popc(seen) != T;
  if constexpr (CHECK != 0) {
    bad |= maxt >= T || minw == 0u;
    return bad ? -1 : ms;
  }
  return ms;
}

// Per-lane constants of the W design for a cluster with sumG <= 32 GPUs.
struct WarpLane {
  int seg;        // segment width (pow2 >= sumG)
  int q;          // GPU slot within the segment (node-major)
  int base;       // first lane of the segment
  int node;       // node of this GPU (-1: padding lane)
  int first;      // lane (within segment) of GPU 0 of this node
  int local;      // GPU id within the node
  int size;       // GPU_n of this node
  uint32_t nmask; // lanes (absolute) of this node
  uint32_t smask; // lanes (absolute) of this segment
  int maxg;       // max_n GPU_n
};

__device__ __forceinline__ WarpLane warp_lane(const Problem& pb, const uint8_t* G) {
  WarpLane L;
  int seg = 1;
  while (seg < pb.sumG) seg <<= 1;
  const int lane = threadIdx.x & 31;
  L.seg = seg;
  L.q = lane & (seg - 1);
  L.base = lane & ~(seg - 1);
  L.node = -1;
  L.first = 0;
  L.local = 0;
  L.size = 0;
  L.maxg = 0;
  int acc = 0;
  for (int n = 0; n < pb.N; ++n) {
    const int gn = G[n];
    if (L.q >= acc && L.q < acc + gn) { L.node = n; L.first = acc; L.local = L.q - acc; L.size = gn; }
    acc += gn;
    L.maxg = max(L.maxg, (int)gn);
  }
  L.smask = (seg == 32) ? 0xffffffffu : (((1u << seg) - 1u) << L.base);
  L.nmask = (L.node < 0) ? 0u : ((L.size == 32 ? 0xffffffffu : ((1u << L.size) - 1u)) << (L.base + L.first));
  return L;
}

// Per-job record written by the trace decoder; layout == saturn_placement (32 bytes).
struct Placement {
  int32_t node, upp, gpus, cfg, start_s, end_s;
  uint64_t gpu_mask;
};

// W design.  All 32 lanes must call it (shuffles use the full mask); `live` lanes belong to
// a real genome.  cfg/perm point at this segment's genome.  If `rec` is non-null, lane q==0
// of each live segment writes the T placement records (job-id order).  Lanes return the
// genome's makespan.
__device__ __forceinline__ int decode_warp(const uint32_t* __restrict__ tab, int stride, const uint8_t* cfg,
                                           const uint8_t* perm, int T, const WarpLane& L, bool live,
                                           const int* node_first, const uint8_t* upp, Placement* rec) {
  const int lane = threadIdx.x & 31;
  int f = (L.node >= 0) ? 0 : INF;
  int ms = 0;
  for (int p = 0; p < T; ++p) {
    const int t = live ? perm[p] : 0;
    const int c = live ? cfg[t] : 0;
    const uint32_t w = tab[t * stride + c];
    const int g = (int)(w >> 24);
    const int R = (int)(w & R_MASK);
    // rank of (f, local id) among the GPUs of my node
    int less = 0, eq = 0, eqpos = 0;
    for (int j = 0; j < L.maxg; ++j) {
      const int src = L.base + L.first + min(j, max(L.size - 1, 0));
      const int fj = __shfl_sync(0xffffffffu, f, src);
      const bool ok = j < L.size;
      less += (ok && fj < f);
      eq += (ok && fj == f);
      eqpos += (ok && fj == f && j < L.local);
    }
    const int rank = less + eqpos;
    // start of my node = free time of the lane whose rank is g-1
    const uint32_t hit = __ballot_sync(0xffffffffu, L.node >= 0 && rank == g - 1) & L.nmask;
    const int src = hit ? (__ffs(hit) - 1) : lane;
    const int fs = __shfl_sync(0xffffffffu, f, src);
    uint32_t key = hit ? (((uint32_t)fs << 5) | (uint32_t)L.node) : 0xffffffffu;
    for (int m = L.seg >> 1; m >= 1; m >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, m));
    const int nstar = (int)(key & 31u);
    const int s = (int)(key >> 5);
    const int v = s + R;
    const bool le = (L.node == nstar) && f <= s;
    const int m = __popc(__ballot_sync(0xffffffffu, le) & L.smask);
    const int rank2 = m - less - eq + eqpos;   // order: free time descending, then id ascending
    const bool chosen = le && rank2 < g;
    const uint32_t cb = __ballot_sync(0xffffffffu, chosen) & L.smask;
    f = chosen ? v : f;
    ms = max(ms, v);
    if (rec && live && L.q == 0) {
      Placement r;
      r.node = nstar;
      r.upp = upp[t * stride + c];
      r.gpus = g;
      r.cfg = c;
      r.start_s = s;
      r.end_s = v;
      r.gpu_mask = (uint64_t)(cb >> (L.base + node_first[nstar]));
      rec[t] = r;
    }
  }
  return ms;
}

}  // namespace sat
