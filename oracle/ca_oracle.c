/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the CA kernels. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline/reference legs load
 * it (through ctypes, as oracle/_ref/libca_oracle.so); the product path never
 * links, calls or falls back to it.
 *
 * PARITY UNPINNED (numerics): the reference is an analytical simulator with
 * no numerical attention (P/README.md:15-18), so no golden
 * vectors exist upstream. This file restates the operation the reference
 * models and the paper specifies:
 *   - O = softmax(QK^T)V with masking, no materialised P, small per-row
 *     softmax statistics recomputed in backward;
 *   - a CA-task is a query shard plus its full causal KV prefix
 *     (P/include/cadsim/types.hpp:101-111);
 *   - the query at absolute position p attends keys 0..p, i.e. a
 *     bottom-right-aligned causal mask inside [0, kv_extent)
 *     (P/src/oracle.cpp:50-54: pairs = sum_{p=kv-n_q}^{kv-1} (p+1));
 *   - softmax scale 1/sqrt(d) (conventional; the reference does not state
 *     one) and LSE in natural log.
 * It is pinned instead by self-consistency checks in tests/ (split-plan
 * outputs equal whole-document outputs, finite differences of the loss in
 * fp64, and an independent torch fp64 computation for golden fixtures).
 *
 * fp32 inputs/outputs, fp64 accumulation. Layouts match include/cad.h:
 * Q/O/dO [q_rows][h_q][d], K/V [kv_rows][h_kv][d], LSE [h_q][q_rows].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int64_t q_off, n_q, kv_off, kv_len;
} oracle_task;

static double dot(const float* a, const float* b, int d) {
  double s = 0.0;
  for (int i = 0; i < d; ++i) s += (double)a[i] * (double)b[i];
  return s;
}

/* Forward over every (task, head, query row). */
void oracle_ca_fwd(const oracle_task* tasks, int64_t n_tasks, int h_q, int h_kv, int d,
                   double scale, const float* q, const float* k, const float* v, float* o,
                   float* lse, int64_t q_rows, int threads) {
  const int group = h_q / h_kv;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  for (int64_t t = 0; t < n_tasks; ++t) {
    const oracle_task tk = tasks[t];
    const int64_t shift = tk.kv_len - tk.n_q;
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
    for (int h = 0; h < h_q; ++h) {
      for (int64_t i = 0; i < tk.n_q; ++i) {
        const int hk = h / group;
        const int64_t row = tk.q_off + i;
        const float* qi = q + (row * h_q + h) * d;
        const int64_t last = shift + i; /* keys 0..last */
        double* s = (double*)malloc(sizeof(double) * (size_t)(last + 1));
        double* acc = (double*)calloc((size_t)d, sizeof(double));
        double m = -INFINITY;
        for (int64_t j = 0; j <= last; ++j) {
          const float* kj = k + ((tk.kv_off + j) * h_kv + hk) * d;
          s[j] = scale * dot(qi, kj, d);
          if (s[j] > m) m = s[j];
        }
        double l = 0.0;
        for (int64_t j = 0; j <= last; ++j) {
          const double p = exp(s[j] - m);
          l += p;
          const float* vj = v + ((tk.kv_off + j) * h_kv + hk) * d;
          for (int c = 0; c < d; ++c) acc[c] += p * (double)vj[c];
        }
        float* oi = o + (row * h_q + h) * d;
        for (int c = 0; c < d; ++c) oi[c] = (float)(acc[c] / l);
        lse[(int64_t)h * q_rows + row] = (float)(m + log(l));
        free(s);
        free(acc);
      }
    }
  }
}

/* Backward. dq is overwritten for the rows the tasks cover; dk/dv are
 * accumulated (+=) in fp64 and added to the caller's arrays, so tasks sharing
 * a document's KV prefix sum their contributions. Three passes, each
 * parallel over independent outputs (no shared accumulators):
 *   1. per (head, query row): lse = log sum_j exp(s_ij), D = dO_i . O_i
 *   2. per (head, query row): dQ_i = scale sum_j dS_ij K_j
 *   3. per (KV head, key row): dK_j = scale sum_{h,i} dS_ij Q_i,
 *      dV_j = sum_{h,i} P_ij dO_i over every task whose KV range holds j
 * with P_ij = exp(s_ij - lse_i), dS_ij = P_ij (dO_i . V_j - D_i). */
static double score(const float* q, const float* k, const oracle_task* tk, int64_t i, int64_t j, int h, int hk,
                    int h_q, int h_kv, int d, double scale) {
  return scale * dot(q + ((tk->q_off + i) * h_q + h) * d, k + ((tk->kv_off + j) * h_kv + hk) * d, d);
}

void oracle_ca_bwd(const oracle_task* tasks, int64_t n_tasks, int h_q, int h_kv, int d,
                   double scale, const float* q, const float* k, const float* v, const float* o,
                   const float* dout, float* dq, float* dk, float* dv, int64_t q_rows,
                   int64_t kv_rows, int threads) {
  const int group = h_q / h_kv;
  if (d > 512) abort(); /* per-row fp64 scratch below holds 512 */
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  double* lse = (double*)malloc(sizeof(double) * (size_t)h_q * (size_t)q_rows);
  double* dsum = (double*)malloc(sizeof(double) * (size_t)h_q * (size_t)q_rows);
  for (int64_t t = 0; t < n_tasks; ++t) {
    const oracle_task tk = tasks[t];
    const int64_t shift = tk.kv_len - tk.n_q;
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
    for (int h = 0; h < h_q; ++h) {
      for (int64_t i = 0; i < tk.n_q; ++i) {
        const int hk = h / group;
        const int64_t row = tk.q_off + i, last = shift + i;
        double m = -INFINITY, l = 0.0;
        for (int64_t j = 0; j <= last; ++j) {
          const double sj = score(q, k, &tk, i, j, h, hk, h_q, h_kv, d, scale);
          if (sj > m) {
            l = l * exp(m - sj) + 1.0;
            m = sj;
          } else {
            l += exp(sj - m);
          }
        }
        lse[(int64_t)h * q_rows + row] = m + log(l);
        dsum[(int64_t)h * q_rows + row] = dot(dout + (row * h_q + h) * d, o + (row * h_q + h) * d, d);
      }
    }
    /* pass 2: dQ */
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
    for (int h = 0; h < h_q; ++h) {
      for (int64_t i = 0; i < tk.n_q; ++i) {
        const int hk = h / group;
        const int64_t row = tk.q_off + i, last = shift + i;
        const float* gi = dout + (row * h_q + h) * d;
        const double li = lse[(int64_t)h * q_rows + row], Di = dsum[(int64_t)h * q_rows + row];
        double gq[512];
        memset(gq, 0, sizeof(double) * (size_t)d);
        for (int64_t j = 0; j <= last; ++j) {
          const float* kj = k + ((tk.kv_off + j) * h_kv + hk) * d;
          const float* vj = v + ((tk.kv_off + j) * h_kv + hk) * d;
          const double p = exp(score(q, k, &tk, i, j, h, hk, h_q, h_kv, d, scale) - li);
          const double ds = p * (dot(gi, vj, d) - Di);
          for (int c = 0; c < d; ++c) gq[c] += ds * (double)kj[c];
        }
        float* dqi = dq + (row * h_q + h) * d;
        for (int c = 0; c < d; ++c) dqi[c] = (float)(scale * gq[c]);
      }
    }
  }
  /* pass 3: dK, dV per (KV head, key row) */
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
  for (int hk = 0; hk < h_kv; ++hk) {
    for (int64_t r = 0; r < kv_rows; ++r) {
      double gk[512], gv[512];
      memset(gk, 0, sizeof(double) * (size_t)d);
      memset(gv, 0, sizeof(double) * (size_t)d);
      int hit = 0;
      const float* kr = k + (r * h_kv + hk) * d;
      const float* vr = v + (r * h_kv + hk) * d;
      for (int64_t t = 0; t < n_tasks; ++t) {
        const oracle_task tk = tasks[t];
        const int64_t j = r - tk.kv_off;
        if (j < 0 || j >= tk.kv_len) continue;
        const int64_t shift = tk.kv_len - tk.n_q;
        const int64_t i0 = j - shift > 0 ? j - shift : 0; /* first query that sees key j */
        for (int h = hk * group; h < (hk + 1) * group; ++h) {
          for (int64_t i = i0; i < tk.n_q; ++i) {
            const int64_t row = tk.q_off + i;
            const float* qi = q + (row * h_q + h) * d;
            const float* gi = dout + (row * h_q + h) * d;
            const double p = exp(scale * dot(qi, kr, d) - lse[(int64_t)h * q_rows + row]);
            const double ds = p * (dot(gi, vr, d) - dsum[(int64_t)h * q_rows + row]);
            for (int c = 0; c < d; ++c) {
              gk[c] += ds * (double)qi[c];
              gv[c] += p * (double)gi[c];
            }
            hit = 1;
          }
        }
      }
      if (!hit) continue;
      float* dkr = dk + (r * h_kv + hk) * d;
      float* dvr = dv + (r * h_kv + hk) * d;
      for (int c = 0; c < d; ++c) {
        dkr[c] += (float)(scale * gk[c]);
        dvr[c] += (float)gv[c];
      }
    }
  }
  free(lse);
  free(dsum);
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
