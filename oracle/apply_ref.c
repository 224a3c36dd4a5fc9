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
 * oracle_plan_counts / oracle_plan_tables restate applyplan.py:116-172
 *   (build_plan) with a per-column radix sort (large matrices; see below).
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

/*
 * oracle_build_plan restates /root/reference/pkg/src/invop/applyplan.py:116-172
 * (build_plan) for large matrices: per column, the nonzero mantissas sorted by
 * (|v| ascending, row ascending) — the order of the reference's stable
 * lexsort((absvals, cols)) over a column-major nonzero scan — then one group
 * per run of equal |v|. Threads own contiguous column blocks; pass 1 counts
 * groups and entries per column, pass 2 writes the tables at the prefix-sum
 * offsets, so the output is independent of the thread count. group_coeff is
 * left to the caller (group_abs * scale, applyplan.py:168).
 */
typedef struct {
  const int64_t* mant;
  int64_t rows, cols, ldm;
  int64_t c0, c1;
  int64_t* gcount;   /* [cols] */
  int64_t* ecount;   /* [cols] */
  const int64_t* gstart; /* [cols] group offset of each column (pass 2) */
  const int64_t* estart; /* [cols] entry offset */
  int64_t* group_abs;
  int64_t* group_ptr;
  int32_t* entry_rows;
  int8_t* entry_signs;
  int pass;
} bp_task;

static void bp_radix(uint64_t* a, uint64_t* tmp, int64_t n, int bits) {
  /* LSD radix sort on the low `bits` bits, 11 bits per pass */
  for (int sh = 0; sh < bits; sh += 11) {
    int64_t cnt[2049];
    for (int i = 0; i <= 2048; ++i) cnt[i] = 0;
    for (int64_t i = 0; i < n; ++i) cnt[((a[i] >> sh) & 2047) + 1]++;
    for (int i = 0; i < 2048; ++i) cnt[i + 1] += cnt[i];
    for (int64_t i = 0; i < n; ++i) tmp[cnt[(a[i] >> sh) & 2047]++] = a[i];
    for (int64_t i = 0; i < n; ++i) a[i] = tmp[i];
  }
}

static void* bp_worker(void* arg) {
  bp_task* t = (bp_task*)arg;
  const int64_t B = 32;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(t->rows > 0 ? t->rows : 1) * B);
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(t->rows > 0 ? t->rows : 1));
  int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * B);
  int rbits = 1;
  while (((int64_t)1 << rbits) < t->rows) ++rbits;
  for (int64_t j0 = t->c0; j0 < t->c1; j0 += B) {
    const int64_t nb = (t->c1 - j0) < B ? (t->c1 - j0) : B;
    int64_t maxabs = 0;
    for (int64_t b = 0; b < nb; ++b) cnt[b] = 0;
    /* row-major scan of the column block: rows ascending per column */
    for (int64_t i = 0; i < t->rows; ++i) {
      const int64_t* r = t->mant + i * t->ldm + j0;
      for (int64_t b = 0; b < nb; ++b) {
        int64_t v = r[b];
        if (v == 0) continue;
        uint64_t a = (uint64_t)(v < 0 ? -v : v);
        if ((int64_t)a > maxabs) maxabs = (int64_t)a;
        /* key: |v|, then the row, then the sign bit (rows are unique
           within a column, so the order is (|v|, row) as in the reference) */
        keys[b * t->rows + cnt[b]++] = (a << (rbits + 1)) | ((uint64_t)i << 1) | (uint64_t)(v < 0);
      }
    }
    int vbits = 1;
    while (((int64_t)1 << vbits) <= maxabs) ++vbits;
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t j = j0 + b, n = cnt[b];
      uint64_t* k = keys + b * t->rows;
      bp_radix(k, tmp, n, rbits + vbits + 1);
      if (t->pass == 1) {
        int64_t g = 0;
        for (int64_t e = 0; e < n; ++e)
          if (e == 0 || (k[e] >> (rbits + 1)) != (k[e - 1] >> (rbits + 1))) ++g;
        t->gcount[j] = g;
        t->ecount[j] = n;
      } else {
        int64_t g = t->gstart[j] - 1, e0 = t->estart[j];
        const uint64_t rmask = ((uint64_t)1 << rbits) - 1;
        for (int64_t e = 0; e < n; ++e) {
          const uint64_t a = k[e] >> (rbits + 1);
          const int64_t row = (int64_t)((k[e] >> 1) & rmask);
          if (e == 0 || a != (k[e - 1] >> (rbits + 1))) {
            ++g;
            t->group_abs[g] = (int64_t)a;
            t->group_ptr[g] = e0 + e;
          }
          t->entry_rows[e0 + e] = (int32_t)row;
          t->entry_signs[e0 + e] = (k[e] & 1) ? -1 : 1;
        }
      }
    }
  }
  free(keys);
  free(tmp);
  free(cnt);
  return NULL;
}

static void bp_run(bp_task* proto, int threads) {
  pthread_t th[256];
  bp_task tasks[256];
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  for (int t = 0; t < threads; ++t) {
    tasks[t] = *proto;
    tasks[t].c0 = proto->cols * t / threads;
    tasks[t].c1 = proto->cols * (t + 1) / threads;
    pthread_create(&th[t], NULL, bp_worker, &tasks[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* pass 1: per-column group and entry counts (gcount, ecount: int64[cols]) */
void oracle_plan_counts(const int64_t* mant, int64_t rows, int64_t cols, int64_t ldm,
                        int64_t* gcount, int64_t* ecount, int threads) {
  bp_task p = {mant, rows, cols, ldm, 0, cols, gcount, ecount, NULL, NULL,
               NULL, NULL, NULL, NULL, 1};
  bp_run(&p, threads);
}

/* pass 2: tables at the offsets given by the exclusive prefix sums of the
   counts (gstart, estart); group_ptr[G] is set by the caller */
void oracle_plan_tables(const int64_t* mant, int64_t rows, int64_t cols, int64_t ldm,
                        const int64_t* gstart, const int64_t* estart, int64_t* group_abs,
                        int64_t* group_ptr, int32_t* entry_rows, int8_t* entry_signs,
                        int threads) {
  bp_task p = {mant, rows, cols, ldm, 0, cols, NULL, NULL, gstart, estart, group_abs,
               group_ptr, entry_rows, entry_signs, 2};
  bp_run(&p, threads);
}
