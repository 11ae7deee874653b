/*
 * model_oracle.c -- CPU helpers of the oracle forward (TEST INFRASTRUCTURE
 * ONLY, see oracle/__init__.py): bit-identical regeneration of the device's
 * random-init weights (paper_2603_18016_b200/csrc/layers.cu,
 * fill_uniform_kernel) as float32 holding bf16 values.
 */
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>
#include <unistd.h>

static inline uint64_t splitmix_at(uint64_t seed, uint64_t i) {
  uint64_t x = (i + seed * 0x100000000ull) * 0x9E3779B97F4A7C15ull + 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* round-to-nearest-even to bf16, returned widened to float (finite inputs) */
static inline float to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
  memcpy(&f, &u, 4);
  return f;
}

typedef struct {
  float* out;
  size_t lo, hi;
  uint64_t seed;
  float span;
  int op; /* 0 fill, 1 round */
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  for (size_t i = j->lo; i < j->hi; ++i) {
    if (j->op == 0) {
      const float u = (float)(splitmix_at(j->seed, i) >> 40) * (1.0f / 16777216.0f);
      j->out[i] = to_bf16((u - 0.5f) * j->span);
    } else {
      j->out[i] = to_bf16(j->out[i]);
    }
  }
  return NULL;
}

static void parallel(float* out, size_t n, uint64_t seed, float span, int op) {
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  if (n < (1u << 20)) nt = 1;
  pthread_t th[64];
  job_t jobs[64];
  for (long t = 0; t < nt; ++t) {
    jobs[t].out = out;
    jobs[t].lo = n * t / nt;
    jobs[t].hi = n * (t + 1) / nt;
    jobs[t].seed = seed;
    jobs[t].span = span;
    jobs[t].op = op;
    if (nt > 1) pthread_create(&th[t], NULL, run_job, &jobs[t]);
  }
  if (nt == 1) run_job(&jobs[0]);
  else
    for (long t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

/* element i of the tensor = bf16((u_i - 1/2) * span), u_i = splitmix64(seed, i) >> 40 / 2^24 */
void oracle_fill_uniform(float* out, size_t n, uint64_t seed, float span) {
  parallel(out, n, seed, span, 0);
}

/* in-place bf16 rounding of a float32 buffer (storage points of the GPU) */
void oracle_round_bf16(float* x, size_t n) { parallel(x, n, 0, 0.0f, 1); }
