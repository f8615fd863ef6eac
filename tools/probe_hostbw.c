// Host write bandwidth probe: T threads writing a repeating pattern into a
// 128 MiB buffer (models the run-length expansion of the payload).
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
static unsigned char* buf; static size_t n = 128u << 20; static int T;
static void* work(void* a) {
  long t = (long)a; size_t per = n / T; unsigned char* p = buf + per * t;
  unsigned char pat[64]; for (int i = 0; i < 64; ++i) pat[i] = "hello\n"[i % 6];
  for (size_t o = 0; o + 64 <= per; o += 64) memcpy(p + o, pat, 64);
  return 0;
}
static double now() { struct timespec ts; clock_gettime(CLOCK_MONOTONIC, &ts); return ts.tv_sec + ts.tv_nsec * 1e-9; }
int main() {
  buf = aligned_alloc(4096, n); memset(buf, 1, n);
  for (T = 1; T <= 16; T *= 2) {
    double best = 1e9;
    for (int r = 0; r < 5; ++r) {
      pthread_t th[16]; double t0 = now();
      for (long i = 0; i < T; ++i) pthread_create(&th[i], 0, work, (void*)i);
      for (int i = 0; i < T; ++i) pthread_join(th[i], 0);
      double dt = now() - t0; if (dt < best) best = dt;
    }
    printf("threads=%2d  %.1f GB/s\n", T, n / best / 1e9);
  }
  return 0;
}
