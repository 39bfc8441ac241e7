/*
 * tools/cpu_ga.c -- the CPU search bar of SURVEY.md §8d ("5-minute CPU search bar", option
 * ii): the same genetic algorithm as the GPU search (GA v3, oracle/ga.py), run on all host
 * cores for a wall-clock budget, each thread an independent island, every child decoded by
 * the plain C oracle decoder (oracle/saturn_oracle.c, linked in).  Baseline tooling: it
 * shares no code with the CUDA path.
 *
 *   cc -O2 -pthread tools/cpu_ga.c oracle/saturn_oracle.c -o tools/cpu_ga
 *   tools/cpu_ga <table.bin> <seconds> <threads> <population> <seed>
 * table.bin: int32 N, GPU[N], T, stride, S[T], G[T*stride], R[T*stride] (written by
 * tools/quality_bar.py from the oracle's compaction).  Prints JSON lines of the anytime
 * curve and the final best.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef struct { int32_t node, upp, gpus, cfg, start_s, end_s; uint64_t gpu_mask; } or_placement;
int32_t or_decode(int32_t, const int32_t *, int32_t, int32_t, const int32_t *, const int32_t *, const int32_t *,
                  const uint8_t *, const uint8_t *, const uint8_t *, or_placement *);

static int N, T, stride, *gpu, *S, *G, *R;
static double budget, t0;
static int P_per, E = 16;
static uint64_t seed;
static uint32_t px = 3865470566u, pc, pm = 2147483648u;

static double now(void) { struct timespec ts; clock_gettime(CLOCK_MONOTONIC, &ts); return ts.tv_sec + 1e-9 * ts.tv_nsec; }

static void philox(uint32_t k0, uint32_t k1, uint32_t c[4], uint32_t out[4]) {
  uint32_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3];
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * x0, p1 = (uint64_t)0xCD9E8D57u * x2;
    uint32_t y0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0, y2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
    x0 = y0; x1 = (uint32_t)p1; x2 = y2; x3 = (uint32_t)p0;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}
static uint32_t word(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t k) {
  uint32_t c[4] = {c0, c1, c2, k >> 2}, o[4];
  philox((uint32_t)seed, (uint32_t)(seed >> 32), c, o);
  return o[k & 3];
}
static uint32_t U(uint32_t n, uint32_t w) { return (uint32_t)(((uint64_t)w * n) >> 32); }
static uint32_t V(uint32_t n, uint32_t h) { return (h * n) >> 16; }

typedef struct { int rank; int best; uint8_t *bc, *bp; long long evals; } island;
static pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;

static int cmp_key(int32_t *ms, int a, int b) { return ms[a] < ms[b] || (ms[a] == ms[b] && a < b); }

static void *run(void *arg) {
  island *is = (island *)arg;
  int P = P_per;
  uint8_t *cfg = malloc((size_t)P * T), *perm = malloc((size_t)P * T), *ncfg = malloc((size_t)P * T),
          *nperm = malloc((size_t)P * T);
  int32_t *ms = malloc(sizeof(int32_t) * P), *nms = malloc(sizeof(int32_t) * P);
  int *el = malloc(sizeof(int) * E);
  uint32_t rk = (uint32_t)is->rank << 16;
  for (int k = 0; k < P; ++k) {   /* initial genome: cfg[t] = U(S_t), Fisher-Yates */
    uint32_t n = 0;
    for (int t = 0; t < T; ++t) cfg[k * T + t] = (uint8_t)U(S[t], word(k, 0, rk | 1, n++));
    for (int t = 0; t < T; ++t) perm[k * T + t] = (uint8_t)t;
    for (int i = T - 1; i > 0; --i) {
      int j = (int)U(i + 1, word(k, 0, rk | 1, n++));
      uint8_t x = perm[k * T + i]; perm[k * T + i] = perm[k * T + j]; perm[k * T + j] = x;
    }
    ms[k] = or_decode(N, gpu, T, stride, G, R, S, cfg + k * T, perm + k * T, NULL, NULL);
  }
  is->evals += P;
  int nb = (T + 31) / 32;
  for (uint32_t gen = 1;; ++gen) {
    for (int e = 0; e < E; ++e) {  /* elites = E smallest (ms, slot) */
      int best = -1;
      for (int k = 0; k < P; ++k) {
        int taken = 0;
        for (int f = 0; f < e; ++f) taken |= el[f] == k;
        if (!taken && (best < 0 || cmp_key(ms, k, best))) best = k;
      }
      el[e] = best;
    }
    pthread_mutex_lock(&mu);
    if (ms[el[0]] < is->best || is->best < 0) {
      is->best = ms[el[0]];
      memcpy(is->bc, cfg + el[0] * T, T);
      memcpy(is->bp, perm + el[0] * T, T);
    }
    pthread_mutex_unlock(&mu);
    if (now() - t0 > budget) break;
    for (int e = 0; e < E; ++e) {
      memcpy(ncfg + e * T, cfg + el[e] * T, T); memcpy(nperm + e * T, perm + el[e] * T, T); nms[e] = ms[el[e]];
    }
    for (int k = E; k < P; ++k) {
      uint32_t w[16];
      for (int i = 0; i < 9 + nb; ++i) w[i] = word(k, gen, rk, i);
      uint32_t i1 = U(P, w[0]), j1 = U(P, w[1]), i2 = U(P, w[2]), j2 = U(P, w[3]);
      int A = cmp_key(ms, i1, j1) ? i1 : j1, B = cmp_key(ms, i2, j2) ? i2 : j2;
      uint8_t *c = ncfg + k * T, *q = nperm + k * T;
      memcpy(c, cfg + A * T, T); memcpy(q, perm + A * T, T);
      if ((w[4] & 0xFFFF) < (px >> 16)) {
        for (int t = 0; t < T; ++t) if (!((w[9 + t / 32] >> (t % 32)) & 1)) c[t] = cfg[B * T + t];
        int a = V(T, w[4] >> 16), b = V(T, w[5] & 0xFFFF);
        if (a > b) { int x = a; a = b; b = x; }
        uint8_t kept[256] = {0};
        for (int i = a; i <= b; ++i) kept[q[i]] = 1;
        int pos = (b + 1) % T;
        for (int i = 0; i < T; ++i) {
          uint8_t x = perm[B * T + (b + 1 + i) % T];
          if (!kept[x]) { q[pos] = x; pos = (pos + 1) % T; }
        }
      }
      if ((w[7] >> 16) < (pc >> 16)) { int t = V(T, w[8] & 0xFFFF); c[t] = (uint8_t)V(S[t], w[8] >> 16); }
      if ((w[5] >> 16) < (pm >> 16)) {
        int kind = w[6] & 1, i = V(T, w[6] >> 16), j = V(T, w[7] & 0xFFFF);
        if (kind == 0) { uint8_t x = q[i]; q[i] = q[j]; q[j] = x; }
        else {
          uint8_t x = q[i];
          if (i < j) for (int m = i; m < j; ++m) q[m] = q[m + 1];
          else for (int m = i; m > j; --m) q[m] = q[m - 1];
          q[j] = x;
        }
      }
      nms[k] = or_decode(N, gpu, T, stride, G, R, S, c, q, NULL, NULL);
    }
    is->evals += P - E;
    uint8_t *x; int32_t *y;
    x = cfg; cfg = ncfg; ncfg = x; x = perm; perm = nperm; nperm = x; y = ms; ms = nms; nms = y;
  }
  return NULL;
}

int main(int argc, char **argv) {
  if (argc < 6) { fprintf(stderr, "usage: cpu_ga table.bin seconds threads population seed\n"); return 2; }
  FILE *f = fopen(argv[1], "rb");
  if (!f) return 2;
  if (fread(&N, 4, 1, f) != 1) return 2;
  gpu = malloc(4 * N); if (fread(gpu, 4, N, f) != (size_t)N) return 2;
  if (fread(&T, 4, 1, f) != 1 || fread(&stride, 4, 1, f) != 1) return 2;
  S = malloc(4 * T); G = malloc(4 * T * stride); R = malloc(4 * T * stride);
  if (fread(S, 4, T, f) != (size_t)T || fread(G, 4, T * stride, f) != (size_t)(T * stride) ||
      fread(R, 4, T * stride, f) != (size_t)(T * stride)) return 2;
  fclose(f);
  budget = atof(argv[2]);
  int nt = atoi(argv[3]);
  P_per = atoi(argv[4]) / nt;
  seed = strtoull(argv[5], NULL, 10);
  pc = (uint32_t)(0.5 * 4294967296.0);
  t0 = now();
  pthread_t th[256];
  island is[256];
  for (int r = 0; r < nt; ++r) {
    is[r].rank = r; is[r].best = -1; is[r].evals = 0;
    is[r].bc = malloc(T); is[r].bp = malloc(T);
    pthread_create(&th[r], NULL, run, &is[r]);
  }
  double last = 0;
  while (now() - t0 < budget) {
    struct timespec ts = {0, 200000000};
    nanosleep(&ts, NULL);
    double t = now() - t0;
    if (t - last >= 5.0) {
      int b = -1; long long ev = 0;
      pthread_mutex_lock(&mu);
      for (int r = 0; r < nt; ++r) { if (is[r].best >= 0 && (b < 0 || is[r].best < b)) b = is[r].best; ev += is[r].evals; }
      pthread_mutex_unlock(&mu);
      printf("{\"t\": %.1f, \"best\": %d, \"evals\": %lld}\n", t, b, ev);
      fflush(stdout);
      last = t;
    }
  }
  for (int r = 0; r < nt; ++r) pthread_join(th[r], NULL);
  int br = 0; long long ev = 0;
  for (int r = 0; r < nt; ++r) { if (is[r].best < is[br].best) br = r; ev += is[r].evals; }
  printf("{\"final\": true, \"t\": %.1f, \"best\": %d, \"evals\": %lld, \"threads\": %d, \"cfg\": [", now() - t0, is[br].best, ev, nt);
  for (int t = 0; t < T; ++t) printf("%s%d", t ? ", " : "", is[br].bc[t]);
  printf("], \"perm\": [");
  for (int t = 0; t < T; ++t) printf("%s%d", t ? ", " : "", is[br].bp[t]);
  printf("]}\n");
  return 0;
}
