/*
 * gett_oracle.c — CPU restatement of the reference xGETT hot loop.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the CPU baseline leg of bench.py; only tests/, __graft_entry__.smoke()
 * and bench.py (cpu_baseline / --impl reference) may load it.  The product path
 * (paper_2410_06770_b200) never links or calls it.
 *
 * Parity: pinned.  tests/test_oracle_golden.py checks it bitwise against the
 * golden vectors in tests/golden/ that tests/golden/make_golden.py produced by
 * running the reference gett.kernel.dgett/sgett itself.
 *
 * What it restates (reference = /root/reference/pkg/src/gett):
 *   - plan.py:258-289  _plan_tables: free table ordered by output dimension
 *     (A's free dims ascending then B's, placed at perm[i]), cont table per pair.
 *   - kernel.py:48-78  _contract_loop: for every output coordinate (dim 0
 *     fastest) resolve idx_c / free_a / free_b, then for every contracted
 *     coordinate (pair 0 fastest) do  c[idx_c] = c[idx_c] + a[idx_a]*b[idx_b]
 *     as an UNFUSED multiply then add in the element type (compile with
 *     -ffp-contract=off), starting from C's prior value.
 *   - kernel.py:34-45  _advance: the mixed-radix odometer.
 *   - kernel.py:93-94  empty iteration space writes nothing.
 *
 * Inputs are assumed already validated (plan.py:162-234); the oracle does not
 * re-validate.  Outputs [free_lo, free_hi) of the free iteration space are
 * computed (linear index in reference order); nthreads > 1 splits that range
 * across pthreads.  Each output element's K loop is sequential and in
 * reference order, so the threaded result is bitwise identical to the serial
 * one whenever distinct output coordinates address distinct C elements.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXR 64

typedef struct {
  int num_free, num_cont;
  int64_t out_inc[MAXR], src_inc[MAXR], ext_free[MAXR];
  int from_a[MAXR];
  int64_t inc_ca[MAXR], inc_cb[MAXR], ext_cont[MAXR];
  int64_t size_free, size_cont;
  int64_t base_a, base_b, base_c;
} oplan_t;

/* plan.py:258-289 */
static int build(oplan_t* p, int rank_a, const int64_t* ext_a, const int64_t* inc_a, int64_t off_a,
                 int rank_b, const int64_t* ext_b, const int64_t* inc_b, int64_t off_b,
                 int conts, const int64_t* cont_a, const int64_t* cont_b, const int64_t* perm,
                 const int64_t* inc_c, int64_t off_c) {
  int rank_c = rank_a + rank_b - 2 * conts;
  if (rank_c > MAXR || conts > MAXR || rank_c < 0) return -1;
  memset(p, 0, sizeof(*p));
  p->num_free = rank_c;
  p->num_cont = conts;
  int i = 0;
  for (int d = 0; d < rank_a; ++d) {
    int contracted = 0;
    for (int k = 0; k < conts; ++k) contracted |= (cont_a[k] == d);
    if (contracted) continue;
    int64_t q = perm[i++];
    p->ext_free[q] = ext_a[d];
    p->src_inc[q] = inc_a[d];
    p->out_inc[q] = inc_c[q];
    p->from_a[q] = 1;
  }
  for (int d = 0; d < rank_b; ++d) {
    int contracted = 0;
    for (int k = 0; k < conts; ++k) contracted |= (cont_b[k] == d);
    if (contracted) continue;
    int64_t q = perm[i++];
    p->ext_free[q] = ext_b[d];
    p->src_inc[q] = inc_b[d];
    p->out_inc[q] = inc_c[q];
    p->from_a[q] = 0;
  }
  p->size_free = 1;
  for (int q = 0; q < rank_c; ++q) p->size_free *= p->ext_free[q];
  p->size_cont = 1;
  for (int k = 0; k < conts; ++k) {
    p->ext_cont[k] = ext_a[cont_a[k]];
    p->inc_ca[k] = inc_a[cont_a[k]];
    p->inc_cb[k] = inc_b[cont_b[k]];
    p->size_cont *= p->ext_cont[k];
  }
  p->base_a = off_a;
  p->base_b = off_b;
  p->base_c = off_c;
  return 0;
}

/* kernel.py:34-45 */
static inline void advance(int64_t* coords, const int64_t* exts, int n) {
  if (n <= 0) return;
  int i = 0;
  for (;;) {
    coords[i] = (coords[i] + 1) % exts[i];
    i += 1;
    if (coords[i - 1] != 0 || i >= n) break;
  }
}

#define DEFINE_LOOP(NAME, T)                                                                  \
  static void NAME(const oplan_t* p, T* c, const T* a, const T* b, int64_t lo, int64_t hi) { \
    int64_t coord_free[MAXR];                                                                 \
    int64_t coord_cont[MAXR];                                                                 \
    int64_t rem = lo;                                                                         \
    for (int j = 0; j < p->num_free; ++j) {                                                   \
      coord_free[j] = rem % p->ext_free[j];                                                   \
      rem /= p->ext_free[j];                                                                  \
    }                                                                                         \
    for (int64_t f = lo; f < hi; ++f) {                                                       \
      int64_t idx_c = p->base_c, free_a = p->base_a, free_b = p->base_b;                      \
      for (int j = 0; j < p->num_free; ++j) {                                                 \
        idx_c += p->out_inc[j] * coord_free[j];                                               \
        if (p->from_a[j]) free_a += p->src_inc[j] * coord_free[j];                            \
        else free_b += p->src_inc[j] * coord_free[j];                                         \
      }                                                                                       \
      for (int k = 0; k < p->num_cont; ++k) coord_cont[k] = 0;                                \
      for (int64_t q = 0; q < p->size_cont; ++q) {                                            \
        int64_t idx_a = free_a, idx_b = free_b;                                               \
        for (int k = 0; k < p->num_cont; ++k) {                                               \
          idx_a += p->inc_ca[k] * coord_cont[k];                                              \
          idx_b += p->inc_cb[k] * coord_cont[k];                                              \
        }                                                                                     \
        T prod = a[idx_a] * b[idx_b];                                                         \
        c[idx_c] = c[idx_c] + prod;                                                           \
        advance(coord_cont, p->ext_cont, p->num_cont);                                        \
      }                                                                                       \
      advance(coord_free, p->ext_free, p->num_free);                                          \
    }                                                                                         \
  }

DEFINE_LOOP(loop_d, double)
DEFINE_LOOP(loop_s, float)

/* Complex (cgett/zgett, kernel.py:187-200): buffers are interleaved (re, im)
 * pairs.  The product is numba's complex multiply, unfused:
 *   re = a.re*b.re - a.im*b.im,  im = a.re*b.im + a.im*b.re,
 * then c = c + prod componentwise, in the element's real type. */
#define DEFINE_LOOP_C(NAME, T)                                                                \
  static void NAME(const oplan_t* p, T* c, const T* a, const T* b, int64_t lo, int64_t hi) { \
    int64_t coord_free[MAXR];                                                                 \
    int64_t coord_cont[MAXR];                                                                 \
    int64_t rem = lo;                                                                         \
    for (int j = 0; j < p->num_free; ++j) {                                                   \
      coord_free[j] = rem % p->ext_free[j];                                                   \
      rem /= p->ext_free[j];                                                                  \
    }                                                                                         \
    for (int64_t f = lo; f < hi; ++f) {                                                       \
      int64_t idx_c = p->base_c, free_a = p->base_a, free_b = p->base_b;                      \
      for (int j = 0; j < p->num_free; ++j) {                                                 \
        idx_c += p->out_inc[j] * coord_free[j];                                               \
        if (p->from_a[j]) free_a += p->src_inc[j] * coord_free[j];                            \
        else free_b += p->src_inc[j] * coord_free[j];                                         \
      }                                                                                       \
      for (int k = 0; k < p->num_cont; ++k) coord_cont[k] = 0;                                \
      for (int64_t q = 0; q < p->size_cont; ++q) {                                            \
        int64_t idx_a = free_a, idx_b = free_b;                                               \
        for (int k = 0; k < p->num_cont; ++k) {                                               \
          idx_a += p->inc_ca[k] * coord_cont[k];                                              \
          idx_b += p->inc_cb[k] * coord_cont[k];                                              \
        }                                                                                     \
        T ar = a[2 * idx_a], ai = a[2 * idx_a + 1], br = b[2 * idx_b], bi = b[2 * idx_b + 1];  \
        T ac = ar * br, bd = ai * bi, ad = ar * bi, bc = ai * br;                             \
        T pr = ac - bd, pi = ad + bc;                                                         \
        c[2 * idx_c] = c[2 * idx_c] + pr;                                                     \
        c[2 * idx_c + 1] = c[2 * idx_c + 1] + pi;                                             \
        advance(coord_cont, p->ext_cont, p->num_cont);                                        \
      }                                                                                       \
      advance(coord_free, p->ext_free, p->num_free);                                          \
    }                                                                                         \
  }

DEFINE_LOOP_C(loop_z, double)
DEFINE_LOOP_C(loop_c, float)

typedef struct {
  const oplan_t* p;
  void *c;
  const void *a, *b;
  int64_t lo, hi;
  int is_double;
} job_t;

/* is_double doubles as the element kind: 0 = s, 1 = d, 2 = c, 3 = z */
static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  switch (j->is_double) {
    case 1: loop_d(j->p, (double*)j->c, (const double*)j->a, (const double*)j->b, j->lo, j->hi); break;
    case 0: loop_s(j->p, (float*)j->c, (const float*)j->a, (const float*)j->b, j->lo, j->hi); break;
    case 3: loop_z(j->p, (double*)j->c, (const double*)j->a, (const double*)j->b, j->lo, j->hi); break;
    default: loop_c(j->p, (float*)j->c, (const float*)j->a, (const float*)j->b, j->lo, j->hi); break;
  }
  return NULL;
}

static int run(int is_double, int rank_a, const int64_t* ext_a, const int64_t* inc_a, const void* a,
               int64_t off_a, int rank_b, const int64_t* ext_b, const int64_t* inc_b, const void* b,
               int64_t off_b, int conts, const int64_t* cont_a, const int64_t* cont_b,
               const int64_t* perm, const int64_t* inc_c, void* c, int64_t off_c, int64_t free_lo,
               int64_t free_hi, int nthreads) {
  oplan_t p;
  if (build(&p, rank_a, ext_a, inc_a, off_a, rank_b, ext_b, inc_b, off_b, conts, cont_a, cont_b,
            perm, inc_c, off_c) != 0)
    return -1;
  /* kernel.py:93-94: an empty iteration space writes nothing */
  if (p.size_free == 0 || p.size_cont == 0) return 0;
  if (free_hi < 0 || free_hi > p.size_free) free_hi = p.size_free;
  if (free_lo < 0) free_lo = 0;
  if (free_lo >= free_hi) return 0;
  if (nthreads < 1) nthreads = 1;
  int64_t n = free_hi - free_lo;
  if (nthreads > n) nthreads = (int)n;
  if (nthreads == 1) {
    job_t j = {&p, c, a, b, free_lo, free_hi, is_double};
    run_job(&j);
    return 0;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * nthreads);
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (job_t){&p, c, a, b, free_lo + n * t / nthreads, free_lo + n * (t + 1) / nthreads,
                      is_double};
    pthread_create(&th[t], NULL, run_job, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}

int oracle_dgett(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const double* a,
                 int64_t off_a, int rank_b, const int64_t* ext_b, const int64_t* inc_b,
                 const double* b, int64_t off_b, int conts, const int64_t* cont_a,
                 const int64_t* cont_b, const int64_t* perm, const int64_t* inc_c, double* c,
                 int64_t off_c, int64_t free_lo, int64_t free_hi, int nthreads) {
  return run(1, rank_a, ext_a, inc_a, a, off_a, rank_b, ext_b, inc_b, b, off_b, conts, cont_a,
             cont_b, perm, inc_c, c, off_c, free_lo, free_hi, nthreads);
}

int oracle_sgett(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const float* a,
                 int64_t off_a, int rank_b, const int64_t* ext_b, const int64_t* inc_b,
                 const float* b, int64_t off_b, int conts, const int64_t* cont_a,
                 const int64_t* cont_b, const int64_t* perm, const int64_t* inc_c, float* c,
                 int64_t off_c, int64_t free_lo, int64_t free_hi, int nthreads) {
  return run(0, rank_a, ext_a, inc_a, a, off_a, rank_b, ext_b, inc_b, b, off_b, conts, cont_a,
             cont_b, perm, inc_c, c, off_c, free_lo, free_hi, nthreads);
}

/* interleaved (re, im) buffers; offsets, lengths and increments in complex elements */
int oracle_zgett(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const double* a,
                 int64_t off_a, int rank_b, const int64_t* ext_b, const int64_t* inc_b,
                 const double* b, int64_t off_b, int conts, const int64_t* cont_a,
                 const int64_t* cont_b, const int64_t* perm, const int64_t* inc_c, double* c,
                 int64_t off_c, int64_t free_lo, int64_t free_hi, int nthreads) {
  return run(3, rank_a, ext_a, inc_a, a, off_a, rank_b, ext_b, inc_b, b, off_b, conts, cont_a,
             cont_b, perm, inc_c, c, off_c, free_lo, free_hi, nthreads);
}

int oracle_cgett(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const float* a,
                 int64_t off_a, int rank_b, const int64_t* ext_b, const int64_t* inc_b,
                 const float* b, int64_t off_b, int conts, const int64_t* cont_a,
                 const int64_t* cont_b, const int64_t* perm, const int64_t* inc_c, float* c,
                 int64_t off_c, int64_t free_lo, int64_t free_hi, int nthreads) {
  return run(2, rank_a, ext_a, inc_a, a, off_a, rank_b, ext_b, inc_b, b, off_b, conts, cont_a,
             cont_b, perm, inc_c, c, off_c, free_lo, free_hi, nthreads);
}
