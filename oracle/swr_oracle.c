/*
 * oracle/swr_oracle.c -- plain, slow, fp64 CPU oracle for the Sliding Window
 * Recurrence (SWR) of arXiv 2512.13921, block length ell = 16.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2512_13921_b200/), and neither side includes the other.
 *
 * What it computes (citations are /root/reference/PAPER.md line numbers):
 *
 *   Eq. 2.1:  x_i = a_i x_{i-1} + u_i, initial state folded into
 *                          the first input.
 *   Jagged window (Eq. truncated_factorization, Eq. block_bidiagonal
 *   P:1304-1312, Eq. block_two_pass_map): the state of a token in
 *   block t depends only on the inputs of block t and of block t-1;
 *   inside that window the dynamics are untruncated.  Written out: the output
 *   for token n of block t is the recurrence (Eq. 2.1) restarted from a zero
 *   state at the first token of block t-1 (from the caller's initial state
 *   carry_in, or zero, at token 0 when t = 0; v_0 = 0 of Alg. 4).
 *
 * This is the plain definition of the operator L~u, NOT the Block Two-Pass
 * algorithm: there is no w_t / g_t / v_t split, no blocking beyond the window
 * definition, no fusion.  The backward is the literal reverse-mode of the same
 * loop (the paper gives no backward; reading R12).
 *
 * Layout: every d-tensor is a contiguous fp64 [B, L, H, D] array (D fastest),
 * decays a are [B, L, H], carries are [B, H, D].  Work is split over (b, h)
 * pairs on `nthreads` POSIX threads; each pair is computed by one thread with
 * the same sequential code, so results do not depend on the thread count.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ELL 16 /* block length ell = 16 */

typedef struct {
  int64_t B, L, H, D;
} swr_dims;

/* element offsets */
static inline int64_t off_a(const swr_dims* s, int64_t b, int64_t n, int64_t h) {
  return (b * s->L + n) * s->H + h;
}
static inline int64_t off_x(const swr_dims* s, int64_t b, int64_t n, int64_t h) {
  return off_a(s, b, n, h) * s->D;
}
static inline int64_t off_c(const swr_dims* s, int64_t b, int64_t h) {
  return (b * s->H + h) * s->D;
}
static inline int64_t min64(int64_t x, int64_t y) { return x < y ? x : y; }

/* ------------------------------------------------------------------------ */
/* forward, one (b, h) slice                                                 */
/* ------------------------------------------------------------------------ */
static void fwd_one(const swr_dims* s, int64_t b, int64_t h, const double* u, const double* a,
                    double* x, const double* carry_in, double* carry_out, double* st) {
  const int64_t L = s->L, D = s->D;
  const int64_t nb = (L + ELL - 1) / ELL;
  for (int64_t t = 0; t < nb; ++t) {
    /* window of block t: from the start of block t-1 (or token 0) to its end */
    const int64_t lo = (t == 0) ? 0 : ELL * (t - 1);
    const int64_t hi = min64(ELL * (t + 1), L);
    for (int64_t c = 0; c < D; ++c)
      st[c] = (t == 0 && carry_in) ? carry_in[off_c(s, b, h) + c] : 0.0; /* x_0 fold */
    for (int64_t n = lo; n < hi; ++n) {
      const double an = a[off_a(s, b, n, h)];
      const double* un = u + off_x(s, b, n, h);
      for (int64_t c = 0; c < D; ++c) st[c] = an * st[c] + un[c]; /* Eq. 2.1 */
      if (n >= ELL * t) {
        double* xn = x + off_x(s, b, n, h);
        for (int64_t c = 0; c < D; ++c) xn[c] = st[c];
      }
    }
  }
  if (carry_out && nb == 0) /* L == 0: no block, nothing carried */
    for (int64_t c = 0; c < D; ++c) carry_out[off_c(s, b, h) + c] = 0.0;
  if (carry_out && nb > 0) {
    /* Local end state of the last block: Eq. 2.1 restarted from zero at the
     * first token of the last block, run to token L-1.  This is v_b of
     * Alg. 4, the "carrier vector" handed to the next segment
     * (P:1526). */
    const int64_t lo = ELL * (nb - 1);
    for (int64_t c = 0; c < D; ++c) st[c] = 0.0;
    for (int64_t n = lo; n < L; ++n) {
      const double an = a[off_a(s, b, n, h)];
      const double* un = u + off_x(s, b, n, h);
      for (int64_t c = 0; c < D; ++c) st[c] = an * st[c] + un[c];
    }
    for (int64_t c = 0; c < D; ++c) carry_out[off_c(s, b, h) + c] = st[c];
  }
}

/* ------------------------------------------------------------------------ */
/* backward, one (b, h) slice: literal reverse mode of fwd_one               */
/*   inputs : u, a, G = dLoss/dx, carry_in (nullable), mu_in = dLoss/dcarry_out */
/*   outputs: du, da, mu_out = dLoss/dcarry_in                                */
/* z holds the chain states z[k] = state before token lo+k (k = 0 .. 2*ELL). */
/* ------------------------------------------------------------------------ */
static void chain_states(const swr_dims* s, int64_t b, int64_t h, const double* u, const double* a,
                         int64_t lo, int64_t hi, const double* s0, double* z) {
  const int64_t D = s->D;
  for (int64_t c = 0; c < D; ++c) z[c] = s0 ? s0[c] : 0.0;
  for (int64_t n = lo; n < hi; ++n) {
    const double an = a[off_a(s, b, n, h)];
    const double* un = u + off_x(s, b, n, h);
    const double* zp = z + (n - lo) * D;
    double* zn = z + (n - lo + 1) * D;
    for (int64_t c = 0; c < D; ++c) zn[c] = an * zp[c] + un[c];
  }
}

static void bwd_one(const swr_dims* s, int64_t b, int64_t h, const double* u, const double* a,
                    const double* G, double* du, double* da, const double* carry_in,
                    const double* mu_in, double* mu_out, double* z, double* lam) {
  const int64_t L = s->L, D = s->D;
  const int64_t nb = (L + ELL - 1) / ELL;
  if (mu_out) /* L == 0: the initial state reaches nothing */
    for (int64_t c = 0; c < D; ++c) mu_out[off_c(s, b, h) + c] = 0.0;
  for (int64_t n = 0; n < L; ++n) {
    da[off_a(s, b, n, h)] = 0.0;
    for (int64_t c = 0; c < D; ++c) du[off_x(s, b, n, h) + c] = 0.0;
  }
  for (int64_t t = 0; t < nb; ++t) {
    const int64_t lo = (t == 0) ? 0 : ELL * (t - 1);
    const int64_t hi = min64(ELL * (t + 1), L);
    const double* s0 = (t == 0 && carry_in) ? carry_in + off_c(s, b, h) : NULL;
    chain_states(s, b, h, u, a, lo, hi, s0, z);
    for (int64_t c = 0; c < D; ++c) lam[c] = 0.0;
    for (int64_t n = hi - 1; n >= lo; --n) {
      if (n >= ELL * t) { /* token n is an output of this chain */
        const double* gn = G + off_x(s, b, n, h);
        for (int64_t c = 0; c < D; ++c) lam[c] += gn[c];
      }
      /* adjoint of  s_n = a_n * s_{n-1} + u_n */
      const double* zp = z + (n - lo) * D; /* s_{n-1} */
      double* dun = du + off_x(s, b, n, h);
      double dot = 0.0;
      for (int64_t c = 0; c < D; ++c) {
        dun[c] += lam[c];
        dot += lam[c] * zp[c];
      }
      da[off_a(s, b, n, h)] += dot;
      const double an = a[off_a(s, b, n, h)];
      for (int64_t c = 0; c < D; ++c) lam[c] *= an;
    }
    if (t == 0 && mu_out) /* lam is now the adjoint of the initial state */
      for (int64_t c = 0; c < D; ++c) mu_out[off_c(s, b, h) + c] = lam[c];
  }
  if (mu_in && nb > 0) {
    /* reverse mode of the carry_out chain (last block, restarted from zero) */
    const int64_t lo = ELL * (nb - 1);
    chain_states(s, b, h, u, a, lo, L, NULL, z);
    for (int64_t c = 0; c < D; ++c) lam[c] = mu_in[off_c(s, b, h) + c];
    for (int64_t n = L - 1; n >= lo; --n) {
      const double* zp = z + (n - lo) * D;
      double* dun = du + off_x(s, b, n, h);
      double dot = 0.0;
      for (int64_t c = 0; c < D; ++c) {
        dun[c] += lam[c];
        dot += lam[c] * zp[c];
      }
      da[off_a(s, b, n, h)] += dot;
      const double an = a[off_a(s, b, n, h)];
      for (int64_t c = 0; c < D; ++c) lam[c] *= an;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* thread pool over (b, h) pairs                                             */
/* ------------------------------------------------------------------------ */
typedef struct {
  const swr_dims* s;
  int is_bwd;
  const double *u, *a, *G, *carry_in, *mu_in;
  double *x, *carry_out, *du, *da, *mu_out;
  int64_t first, last; /* [first, last) over b*H + h */
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  const int64_t D = j->s->D;
  double* st = (double*)malloc(sizeof(double) * D * (2 * ELL + 2));
  double* lam = (double*)malloc(sizeof(double) * D);
  for (int64_t p = j->first; p < j->last; ++p) {
    const int64_t b = p / j->s->H, h = p % j->s->H;
    if (!j->is_bwd)
      fwd_one(j->s, b, h, j->u, j->a, j->x, j->carry_in, j->carry_out, st);
    else
      bwd_one(j->s, b, h, j->u, j->a, j->G, j->du, j->da, j->carry_in, j->mu_in, j->mu_out, st, lam);
  }
  free(st);
  free(lam);
  return NULL;
}

static int run_pool(job_t proto, int nthreads) {
  const int64_t pairs = proto.s->B * proto.s->H;
  if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > pairs) nthreads = (int)pairs;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * nthreads);
  for (int i = 0; i < nthreads; ++i) {
    jobs[i] = proto;
    jobs[i].first = pairs * i / nthreads;
    jobs[i].last = pairs * (i + 1) / nthreads;
    if (nthreads == 1)
      run_job(&jobs[i]);
    else
      pthread_create(&th[i], NULL, run_job, &jobs[i]);
  }
  if (nthreads > 1)
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
  free(jobs);
  return nthreads;
}

/* ------------------------------------------------------------------------ */
/* exported entry points (called from oracle/oracle.py through ctypes)       */
/* Return value: number of threads actually used.                           */
/* ------------------------------------------------------------------------ */
int swr_oracle_fwd(const double* u, const double* a, double* x, const double* carry_in,
                   double* carry_out, int64_t B, int64_t L, int64_t H, int64_t D, int nthreads) {
  swr_dims s = {B, L, H, D};
  job_t j;
  memset(&j, 0, sizeof(j));
  j.s = &s;
  j.u = u;
  j.a = a;
  j.x = x;
  j.carry_in = carry_in;
  j.carry_out = carry_out;
  return run_pool(j, nthreads);
}

int swr_oracle_bwd(const double* u, const double* a, const double* G, double* du, double* da,
                   const double* carry_in, const double* mu_in, double* mu_out, int64_t B,
                   int64_t L, int64_t H, int64_t D, int nthreads) {
  swr_dims s = {B, L, H, D};
  job_t j;
  memset(&j, 0, sizeof(j));
  j.s = &s;
  j.is_bwd = 1;
  j.u = u;
  j.a = a;
  j.G = G;
  j.du = du;
  j.da = da;
  j.carry_in = carry_in;
  j.mu_in = mu_in;
  j.mu_out = mu_out;
  return run_pool(j, nthreads);
}
