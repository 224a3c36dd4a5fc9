/*
 * TEST INFRASTRUCTURE — CPU restatement of the reference apply, used only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker. Never linked into or called by the product path.
 *
 * oracle_plan_apply restates /root/reference/pkg/src/invop/_kernels/_native.pyx:15-49
 *   (column loop; t = group_coeff[g]*x[j] once per group; out[row] += t or -= t).
 * oracle_ordered_apply restates the same sum row by row: for each output row,
 *   acc = +0.0; for j ascending with mant != 0: acc (+|-)= (|mant|*10^-m)*x_j.
 *   Contributions reach a row in ascending j in both forms
 *   (/root/reference/pkg/src/invop/applyplan.py:4-8), so the two are bitwise
 *   equal; the row form parallelises over rows and needs no plan tables.
 * oracle_dense_matvec restates _native.pyx:75-92.
 * Build with -ffp-contract=off like the reference (pkg/setup.py:11-13).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

int64_t oracle_plan_apply(const int64_t* col_ptr, const double* group_coeff,
                          const int64_t* group_ptr, const int32_t* entry_rows,
                          const int8_t* entry_signs, const double* x, double* out, int64_t n,
                          int64_t* adds_out) {
  int64_t mults = 0, adds = 0;
  for (int64_t j = 0; j < n; ++j) {
    int64_t g0 = col_ptr[j], g1 = col_ptr[j + 1];
    if (g0 == g1) continue;
    double xj = x[j];
    for (int64_t g = g0; g < g1; ++g) {
      double t = group_coeff[g] * xj;
      int64_t e0 = group_ptr[g], e1 = group_ptr[g + 1];
      for (int64_t e = e0; e < e1; ++e) {
        if (entry_signs[e] > 0) out[entry_rows[e]] += t;
        else out[entry_rows[e]] -= t;
      }
      adds += e1 - e0;
    }
    mults += g1 - g0;
  }
  if (adds_out) *adds_out = adds;
  return mults;
}

typedef struct {
  const int64_t* mant;
  int64_t rows, n, ldm;
  double scale;
  const double* x;
  int64_t nrhs, ldx;
  double* y;
  int64_t ldy;
  int64_t r0, r1;
} ord_task;

static void* ord_worker(void* arg) {
  ord_task* t = (ord_task*)arg;
  for (int64_t k = 0; k < t->nrhs; ++k) {
    const double* x = t->x + k * t->ldx;
    for (int64_t i = t->r0; i < t->r1; ++i) {
      const int64_t* row = t->mant + i * t->ldm;
      double acc = 0.0;
      for (int64_t j = 0; j < t->n; ++j) {
        int64_t v = row[j];
        if (v == 0) continue;
        double c = (double)(v < 0 ? -v : v) * t->scale;  /* group_coeff */
        double p = c * x[j];
        if (v > 0) acc += p;
        else acc -= p;
      }
      t->y[k * t->ldy + i] = acc;
    }
  }
  return NULL;
}

void oracle_ordered_apply(const int64_t* mant, int64_t rows, int64_t n, int64_t ldm,
                          double scale, const double* x, int64_t nrhs, int64_t ldx, double* y,
                          int64_t ldy, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads > rows) threads = rows > 0 ? (int)rows : 1;
  pthread_t th[256];
  ord_task tasks[256];
  for (int t = 0; t < threads; ++t) {
    ord_task tk = {mant, rows, n, ldm, scale, x, nrhs, ldx, y, ldy,
                   rows * t / threads, rows * (t + 1) / threads};
    tasks[t] = tk;
    pthread_create(&th[t], NULL, ord_worker, &tasks[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

void oracle_dense_matvec(const double* m, int64_t rows, int64_t cols, const double* x,
                         double* out) {
  for (int64_t r = 0; r < rows; ++r) {
    double acc = m[r * cols] * x[0];
    for (int64_t j = 1; j < cols; ++j) acc += m[r * cols + j] * x[j];
    out[r] = acc;
  }
}
