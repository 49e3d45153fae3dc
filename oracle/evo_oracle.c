/* evo_oracle.c — CPU restatement of the reference tiled Evoformer attention.
 *
 * TEST INFRASTRUCTURE ONLY (see evo_oracle.h): the checker for the CUDA path,
 * never the product. Each block cites the reference lines it restates:
 *   /root/reference/proj/core/src/attention_tiled.cpp   forward :57-180, backward :182-340
 *   /root/reference/proj/core/include/evomem/numeric_format.hpp:60-71 (rounding)
 *   /root/reference/proj/core/src/numeric_format.cpp:42-78 (emulated RNE)
 * Pinned against the reference itself (oracle/_ref, built from the reference
 * sources by oracle/Makefile) in tests/test_oracle.py, bit for bit.
 */
#include "evo_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* numeric_format.hpp:60-71 — F32 re-rounds through float, F64 is exact. */
static inline double rnd(int fmt, double x) {
  return fmt == EVO_ORACLE_F32 ? (double)(float)x : x;
}

/* Row-range worker state: processes canonical rows [r0, r1) of the full
 * problem, so the threaded driver can shard rows without copying. */
typedef struct {
  const evo_oracle_problem* p;
  int64_t r0, r1;
  const double *q, *k, *v, *bias1, *bias2, *o, *lse_in, *dout;
  double *out, *lse, *dq, *dk, *dv, *dbias1, *dbias2;
  int status;
} rows_job;

static int validate(const evo_oracle_problem* p) {
  if (!p || p->B < 1 || p->L < 1 || p->H < 1 || p->D < 1 || p->Bo < 1 || p->B % p->Bo) return 1;
  if (p->tile_q < 1 || p->tile_k < 1 || p->tile_b < 1) return 1; /* TileConfig::validate :12-17 */
  if (p->fmt != EVO_ORACLE_F32 && p->fmt != EVO_ORACLE_F64) return 1;
  if (!isfinite(p->scale)) return 2; /* attention.cpp:83-85 */
  return 0;
}

static int has_nan(const double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (isnan(x[i])) return 1;
  return 0;
}

/* Scaled, biased logit for (h, b, i, j): attention_tiled.cpp:117-124 with the
 * mask term inserted before the pair bias. */
static inline double logit(const rows_job* J, int64_t h, int64_t b, int64_t i, int64_t j) {
  const evo_oracle_problem* p = J->p;
  const int fmt = p->fmt;
  const int64_t H = p->H, D = p->D, L = p->L;
  const double* qr = J->q + ((b * L + i) * H + h) * D;
  const double* kr = J->k + ((b * L + j) * H + h) * D;
  double dot = 0.0;
  for (int64_t d = 0; d < D; ++d) dot = rnd(fmt, dot + rnd(fmt, qr[d] * kr[d]));
  double s = rnd(fmt, p->scale * dot);
  if (J->bias1) s = rnd(fmt, s + J->bias1[b * L + j]);
  if (J->bias2) {
    const int64_t ob = b / (p->B / p->Bo);
    s = rnd(fmt, s + J->bias2[((ob * H + h) * L + i) * L + j]);
  }
  return s;
}

/* attn_forward_tiled, attention_tiled.cpp:83-177, restricted to rows [r0, r1). */
static void forward_rows(rows_job* J) {
  const evo_oracle_problem* p = J->p;
  const int fmt = p->fmt;
  const int64_t B = p->B, L = p->L, H = p->H, D = p->D;
  const int64_t tq = p->tile_q, tk = p->tile_k, tb = p->tile_b;
  double* acc = (double*)malloc(sizeof(double) * (size_t)(tq * D));
  double* mrow = (double*)malloc(sizeof(double) * (size_t)tq);
  double* lrow = (double*)malloc(sizeof(double) * (size_t)tq);
  double* tile = (double*)malloc(sizeof(double) * (size_t)(tq * (tk < L ? tk : L)));
  const int64_t tkm = tk < L ? tk : L;
  J->status = 0;
  for (int64_t h = 0; h < H; ++h) {
    for (int64_t b0 = J->r0; b0 < J->r1; b0 += tb) {
      const int64_t b1 = b0 + tb < J->r1 ? b0 + tb : J->r1;
      for (int64_t i0 = 0; i0 < L; i0 += tq) {
        const int64_t rows = tq < L - i0 ? tq : L - i0;
        for (int64_t b = b0; b < b1; ++b) {
          for (int64_t x = 0; x < rows * D; ++x) acc[x] = 0.0;
          for (int64_t r = 0; r < rows; ++r) { mrow[r] = -INFINITY; lrow[r] = 0.0; }
          for (int64_t j0 = 0; j0 < L; j0 += tk) {
            const int64_t cols = tk < L - j0 ? tk : L - j0;
            for (int64_t r = 0; r < rows; ++r)
              for (int64_t c = 0; c < cols; ++c) {
                const double s = logit(J, h, b, i0 + r, j0 + c);
                if (!isfinite(s)) { J->status = 2; goto done; } /* :125-127 */
                tile[r * tkm + c] = s;
              }
            /* online softmax update, :134-158 */
            for (int64_t r = 0; r < rows; ++r) {
              double mn = mrow[r];
              for (int64_t c = 0; c < cols; ++c) mn = tile[r * tkm + c] > mn ? tile[r * tkm + c] : mn;
              const double alpha = rnd(fmt, exp(rnd(fmt, mrow[r] - mn)));
              for (int64_t d = 0; d < D; ++d) acc[r * D + d] = rnd(fmt, acc[r * D + d] * alpha);
              double tsum = 0.0;
              for (int64_t c = 0; c < cols; ++c) {
                const double e = rnd(fmt, exp(rnd(fmt, tile[r * tkm + c] - mn)));
                tsum = rnd(fmt, tsum + e);
                const double* vr = J->v + ((b * L + j0 + c) * H + h) * D;
                for (int64_t d = 0; d < D; ++d)
                  acc[r * D + d] = rnd(fmt, acc[r * D + d] + rnd(fmt, e * vr[d]));
              }
              lrow[r] = rnd(fmt, rnd(fmt, lrow[r] * alpha) + tsum);
              mrow[r] = mn;
            }
          }
          /* finalize, :162-172; the statistic is stored widened_to_f32 */
          for (int64_t r = 0; r < rows; ++r) {
            double* orow = J->out + ((b * L + i0 + r) * H + h) * D;
            for (int64_t d = 0; d < D; ++d) orow[d] = rnd(fmt, acc[r * D + d] / lrow[r]);
            J->lse[(h * B + b) * L + i0 + r] = rnd(fmt, mrow[r] + log(lrow[r]));
          }
        }
      }
    }
  }
done:
  free(acc); free(mrow); free(lrow); free(tile);
}

/* attn_backward_tiled, attention_tiled.cpp:227-337, rows [r0, r1).
 * dq/dk/dv are fully owned by the row range; dbias1 rows likewise; dbias2 is
 * the caller's accumulator for this range (F32 per-add rounding, :318-323). */
static void backward_rows(rows_job* J) {
  const evo_oracle_problem* p = J->p;
  const int fmt = p->fmt;
  const int64_t B = p->B, L = p->L, H = p->H, D = p->D;
  const int64_t tq = p->tile_q, tk = p->tile_k, tb = p->tile_b;
  const int64_t nrows = J->r1 - J->r0;
  const int64_t tkm = tk < L ? tk : L;
  double* delta = (double*)malloc(sizeof(double) * (size_t)(nrows * L * H));
  double* tile = (double*)malloc(sizeof(double) * (size_t)(tq * tkm));
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)nrows);
  J->status = 0;
  /* delta[b,i,h] = sum_d dO*O, stored widened (:227-241) */
  for (int64_t b = J->r0; b < J->r1; ++b)
    for (int64_t i = 0; i < L; ++i)
      for (int64_t h = 0; h < H; ++h) {
        const int64_t base = ((b * L + i) * H + h) * D;
        double a = 0.0;
        for (int64_t d = 0; d < D; ++d) a = rnd(fmt, a + rnd(fmt, J->dout[base + d] * J->o[base + d]));
        delta[((b - J->r0) * L + i) * H + h] = rnd(fmt, a);
      }
  /* batch order, :249-252 */
  for (int64_t x = 0; x < nrows; ++x) order[x] = p->deterministic ? J->r0 + x : J->r1 - 1 - x;

  for (int64_t h = 0; h < H; ++h) {
    for (int64_t bo = 0; bo < nrows; bo += tb) {
      const int64_t bo1 = bo + tb < nrows ? bo + tb : nrows;
      for (int64_t i0 = 0; i0 < L; i0 += tq) {
        const int64_t rows = tq < L - i0 ? tq : L - i0;
        for (int64_t bi = bo; bi < bo1; ++bi) {
          const int64_t b = order[bi];
          const int64_t ob = b / (B / p->Bo);
          for (int64_t j0 = 0; j0 < L; j0 += tk) {
            const int64_t cols = tk < L - j0 ? tk : L - j0;
            /* recompute P = exp(S - lse), :268-288 */
            for (int64_t r = 0; r < rows; ++r) {
              const double rl = J->lse_in[(h * B + b) * L + i0 + r];
              for (int64_t c = 0; c < cols; ++c)
                tile[r * tkm + c] = rnd(fmt, exp(rnd(fmt, logit(J, h, b, i0 + r, j0 + c) - rl)));
            }
            /* gradient accumulation, :289-325 */
            for (int64_t r = 0; r < rows; ++r) {
              const int64_t i = i0 + r;
              const int64_t io_i = ((b * L + i) * H + h) * D;
              const double rd = delta[((b - J->r0) * L + i) * H + h];
              for (int64_t c = 0; c < cols; ++c) {
                const int64_t j = j0 + c;
                const int64_t io_j = ((b * L + j) * H + h) * D;
                const double pr = tile[r * tkm + c];
                for (int64_t d = 0; d < D; ++d)
                  J->dv[io_j + d] = rnd(fmt, J->dv[io_j + d] + rnd(fmt, pr * J->dout[io_i + d]));
                double dp = 0.0;
                for (int64_t d = 0; d < D; ++d)
                  dp = rnd(fmt, dp + rnd(fmt, J->dout[io_i + d] * J->v[io_j + d]));
                const double ds = rnd(fmt, pr * rnd(fmt, dp - rd));
                for (int64_t d = 0; d < D; ++d) {
                  J->dq[io_i + d] = rnd(fmt, J->dq[io_i + d] + rnd(fmt, ds * J->k[io_j + d]));
                  J->dk[io_j + d] = rnd(fmt, J->dk[io_j + d] + rnd(fmt, ds * J->q[io_i + d]));
                }
                if (J->dbias2) {
                  double* t = &J->dbias2[((ob * H + h) * L + i) * L + j];
                  *t = rnd(fmt, *t + ds); /* UpcastF32: F32-or-wider accumulator */
                }
                if (J->dbias1) {
                  double* t = &J->dbias1[b * L + j];
                  *t = rnd(fmt, *t + ds);
                }
              }
            }
          }
        }
      }
    }
  }
  /* deferred scale, :334-337 */
  for (int64_t b = J->r0; b < J->r1; ++b)
    for (int64_t x = 0; x < L * H * D; ++x) {
      const int64_t at = b * L * H * D + x;
      J->dq[at] = rnd(fmt, p->scale * J->dq[at]);
      J->dk[at] = rnd(fmt, p->scale * J->dk[at]);
    }
  free(delta); free(tile); free(order);
}

int evo_oracle_forward(const evo_oracle_problem* p, const double* q, const double* k,
                       const double* v, const double* bias1, const double* bias2,
                       double* o, double* lse) {
  int st = validate(p);
  if (st) return st;
  const int64_t n = p->B * p->L * p->H * p->D;
  if (has_nan(q, n) || has_nan(k, n) || has_nan(v, n)) return 2; /* :61-64 */
  if (bias1 && has_nan(bias1, p->B * p->L)) return 2;
  if (bias2 && has_nan(bias2, p->Bo * p->H * p->L * p->L)) return 2;
  rows_job J;
  memset(&J, 0, sizeof J);
  J.p = p; J.r0 = 0; J.r1 = p->B;
  J.q = q; J.k = k; J.v = v; J.bias1 = bias1; J.bias2 = bias2; J.out = o; J.lse = lse;
  forward_rows(&J);
  return J.status;
}

int evo_oracle_backward(const evo_oracle_problem* p, const double* q, const double* k,
                        const double* v, const double* bias1, const double* bias2,
                        const double* o, const double* lse, const double* dout,
                        double* dq, double* dk, double* dv, double* dbias1, double* dbias2) {
  int st = validate(p);
  if (st) return st;
  const int64_t n = p->B * p->L * p->H * p->D;
  if (has_nan(dout, n)) return 2; /* :208 */
  memset(dq, 0, sizeof(double) * (size_t)n);
  memset(dk, 0, sizeof(double) * (size_t)n);
  memset(dv, 0, sizeof(double) * (size_t)n);
  if (dbias1) memset(dbias1, 0, sizeof(double) * (size_t)(p->B * p->L));
  if (dbias2) memset(dbias2, 0, sizeof(double) * (size_t)(p->Bo * p->H * p->L * p->L));
  rows_job J;
  memset(&J, 0, sizeof J);
  J.p = p; J.r0 = 0; J.r1 = p->B;
  J.q = q; J.k = k; J.v = v; J.bias1 = bias1; J.bias2 = bias2; J.o = o; J.lse_in = lse;
  J.dout = dout; J.dq = dq; J.dk = dk; J.dv = dv; J.dbias1 = dbias1; J.dbias2 = dbias2;
  backward_rows(&J);
  return J.status;
}

/* numeric_format.cpp:42-78: RNE onto a (mantissa, exponent) grid with
 * subnormals, saturating to +-inf past the largest finite value. */
void evo_oracle_round(double* x, int64_t n, int mb, int eb) {
  const int bias = (1 << (eb - 1)) - 1;
  const int min_exp = 1 - bias;
  const double maxf = (2.0 - ldexp(1.0, -mb)) * ldexp(1.0, bias);
  for (int64_t t = 0; t < n; ++t) {
    const double v = x[t];
    if (v == 0.0 || !isfinite(v)) continue;
    int e2;
    frexp(v, &e2);
    const int ue = e2 - 1;
    const int lsb = (ue > min_exp ? ue : min_exp) - mb;
    const double sc = ldexp(v, -lsb);
    const double lo = floor(sc);
    const double fr = sc - lo;
    double ri = fr > 0.5 ? lo + 1.0 : (fr < 0.5 ? lo : (fmod(lo, 2.0) == 0.0 ? lo : lo + 1.0));
    double r = ldexp(ri, lsb);
    if (fabs(r) > maxf) r = v > 0 ? INFINITY : -INFINITY;
    x[t] = r;
  }
}

static void* fwd_bwd_thread(void* arg) {
  rows_job* J = (rows_job*)arg;
  forward_rows(J);
  if (J->status) return NULL;
  J->o = J->out;
  J->lse_in = J->lse;
  backward_rows(J);
  return NULL;
}

int evo_oracle_fwd_bwd_threaded(const evo_oracle_problem* p, int threads, const double* q,
                                const double* k, const double* v, const double* bias1,
                                const double* bias2, const double* dout, double* o,
                                double* lse, double* dq, double* dk, double* dv,
                                double* dbias2) {
  int st = validate(p);
  if (st) return st;
  if (threads < 1) threads = 1;
  if (threads > p->B) threads = (int)p->B;
  const int64_t n = p->B * p->L * p->H * p->D;
  const int64_t nb2 = p->Bo * p->H * p->L * p->L;
  memset(dq, 0, sizeof(double) * (size_t)n);
  memset(dk, 0, sizeof(double) * (size_t)n);
  memset(dv, 0, sizeof(double) * (size_t)n);
  rows_job* jobs = (rows_job*)calloc((size_t)threads, sizeof(rows_job));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  double* partial = dbias2 ? (double*)calloc((size_t)(threads * nb2), sizeof(double)) : NULL;
  for (int t = 0; t < threads; ++t) {
    rows_job* J = &jobs[t];
    J->p = p;
    J->r0 = p->B * t / threads;
    J->r1 = p->B * (t + 1) / threads;
    J->q = q; J->k = k; J->v = v; J->bias1 = bias1; J->bias2 = bias2; J->dout = dout;
    J->out = o; J->lse = lse; J->dq = dq; J->dk = dk; J->dv = dv;
    J->dbias2 = partial ? partial + (int64_t)t * nb2 : NULL;
    pthread_create(&tid[t], NULL, fwd_bwd_thread, J);
  }
  int status = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    if (jobs[t].status) status = jobs[t].status;
  }
  if (dbias2) {
    for (int64_t x = 0; x < nb2; ++x) {
      double a = 0.0;
      for (int t = 0; t < threads; ++t) a = rnd(p->fmt, a + partial[(int64_t)t * nb2 + x]);
      dbias2[x] = a;
    }
  }
  free(partial); free(jobs); free(tid);
  return status;
}
