// Host-side probe: how fast can T threads widen 32-bit keys to 64-bit words (the narrow-download
// idea: ship 4-byte keys over PCIe, widen on the host)?   gcc -O3 -march=native -pthread
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
typedef struct { const uint32_t* src; uint64_t* dst; size_t lo, hi; } job_t;
static void* work(void* p) {
  job_t* j = (job_t*)p;
  for (size_t i = j->lo; i < j->hi; ++i) j->dst[i] = j->src[i];
  return 0;
}
static double now(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }
int main(int argc, char** argv) {
  size_t n = 125000000;
  uint32_t* src = malloc(n * 4);
  uint64_t* dst = malloc(n * 8);
  memset(src, 1, n * 4);
  memset(dst, 0, n * 8);                       // fault the pages in, like a reused pinned block
  for (int T = 1; T <= 32; T *= 2) {
    double best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      pthread_t th[32]; job_t jobs[32];
      double t0 = now();
      for (int t = 0; t < T; ++t) { jobs[t] = (job_t){src, dst, n * t / T, n * (t + 1) / T}; pthread_create(&th[t], 0, work, &jobs[t]); }
      for (int t = 0; t < T; ++t) pthread_join(th[t], 0);
      double dt = now() - t0; if (dt < best) best = dt;
    }
    printf("threads %2d: %.1f ms (%.1f GB/s of traffic)\n", T, 1e3 * best, 12.0 * n / best / 1e9);
  }
  return dst[12345] == 0;
}
