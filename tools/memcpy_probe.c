// Host copy bandwidth on the GPU box: glibc memcpy vs AVX2 non-temporal
// stores, 1..16 threads, 128 MiB (the staging copy of hx_apply_host_staged).
//   gcc -O3 -mavx2 -pthread tools/memcpy_probe.c -o build/memcpy_probe
#include <immintrin.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define BYTES (128ul << 20)
static char *src, *dst;
static int nthreads, mode;

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + 1e-9 * t.tv_nsec;
}

static void nt_copy(char* d, const char* s, size_t n) {
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    __m256d a = _mm256_loadu_pd((const double*)(s + i));
    __m256d b = _mm256_loadu_pd((const double*)(s + i + 32));
    __m256d c = _mm256_loadu_pd((const double*)(s + i + 64));
    __m256d e = _mm256_loadu_pd((const double*)(s + i + 96));
    _mm256_stream_pd((double*)(d + i), a);
    _mm256_stream_pd((double*)(d + i + 32), b);
    _mm256_stream_pd((double*)(d + i + 64), c);
    _mm256_stream_pd((double*)(d + i + 96), e);
  }
  memcpy(d + i, s + i, n - i);
  _mm_sfence();
}

static void nt_copy_sse2(char* d, const char* s, size_t n) {
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    __m128d a = _mm_loadu_pd((const double*)(s + i));
    __m128d b = _mm_loadu_pd((const double*)(s + i + 16));
    __m128d c = _mm_loadu_pd((const double*)(s + i + 32));
    __m128d e = _mm_loadu_pd((const double*)(s + i + 48));
    _mm_stream_pd((double*)(d + i), a);
    _mm_stream_pd((double*)(d + i + 16), b);
    _mm_stream_pd((double*)(d + i + 32), c);
    _mm_stream_pd((double*)(d + i + 48), e);
  }
  memcpy(d + i, s + i, n - i);
  _mm_sfence();
}

static void* worker(void* arg) {
  long id = (long)arg;
  size_t piece = BYTES / nthreads;
  char* d = dst + id * piece;
  const char* s = src + id * piece;
  if (mode == 0)
    memcpy(d, s, piece);
  else if (mode == 1)
    nt_copy(d, s, piece);
  else
    nt_copy_sse2(d, s, piece);
  return NULL;
}

int main(void) {
  src = aligned_alloc(4096, BYTES);
  dst = aligned_alloc(4096, BYTES);
  memset(src, 1, BYTES);
  memset(dst, 2, BYTES);
  for (mode = 0; mode < 3; ++mode) {
    for (nthreads = 1; nthreads <= 16; nthreads *= 2) {
      double best = 1e9;
      for (int r = 0; r < 5; ++r) {
        pthread_t th[16];
        double t0 = now();
        for (long i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, worker, (void*)i);
        for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
        double t = now() - t0;
        if (t < best) best = t;
      }
      printf("%s threads %2d: %6.2f ms  %6.1f GB/s (copy rate)\n", mode == 0 ? "memcpy" : mode == 1 ? "nt256 " : "nt128 ",
             nthreads, best * 1e3, BYTES / best / 1e9);
    }
  }
  return 0;
}
