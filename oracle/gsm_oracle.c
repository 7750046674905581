/*
 * gsm_oracle.c — TEST INFRASTRUCTURE ONLY (parity checker / CPU baseline).
 *
 * A plain-C, single-threaded restatement of the reference's plan evaluator
 * (/root/reference/pkg/src/gsmat/executor.py) over the on-disk pair arrays
 * (storage.py:56-97).  It reproduces the reference's ROW ORDER, not just the
 * bag: regroup() is a stable first-occurrence group-by and candidates follow
 * the right table's scan order, exactly as executor.py does.  It is checked
 * row-for-row against the reference itself and against the reference's
 * golden vectors (tests/test_oracle.py); the CUDA product is then checked
 * against it as a multiset (tests/test_gpu_parity.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use
 * this file.  The product (paper_1807_07691_b200) never links or calls it.
 *
 * Semantics restated (file:line in /root/reference/pkg/src/gsmat/):
 *   scan            executor.py:94-127   shapes R1..R6
 *   regroup         executor.py:130-137  stable, first-occurrence key order
 *   _join_layout    executor.py:140-152  J = shared vars in left-schema order
 *   cross_product   executor.py:155-165  budget on |L|*|R|
 *   sm_join         executor.py:168-194  budget on emitted rows (sequential)
 *   preallocate     executor.py:197-215  E = sum over left rows of right
 *                                        rows sharing the first join key
 *   parallel budget executor.py:237-241  budget on E (pre-filter total)
 *   execute         executor.py:296-368  projection + first-occurrence DISTINCT
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t nnz;          /* pairs per orientation; 0 with NULL arrays = no matrix */
  const uint64_t* so;   /* 2*nnz: (s,o) sorted by (s,o)   storage.py:74-78 */
  const uint64_t* os;   /* 2*nnz: (o,s) sorted by (o,s) */
} orc_pred;

typedef struct {
  int32_t s_var;   /* variable index >= 0, or -1 when the subject is a constant */
  int32_t o_var;
  int64_t s_const; /* node id when s_var == -1 */
  int64_t o_const;
  int32_t pid;     /* predicate id; matrices missing for pid -> scan yields nothing */
  int32_t empty;   /* EncodedPattern.empty (qparser.py:303-323) */
} orc_pattern;

enum { ORC_OK = 0, ORC_ERR_VALUE = 1, ORC_ERR_RESOURCE = 4, ORC_ERR_NOMEM = 6 };

typedef struct {
  int32_t arity;
  int32_t schema[64];
  int64_t n;
  int64_t* rows; /* row-major n x arity */
} Table;

static char g_msg[512];

const char* orc_last_error(void) { return g_msg; }

static void* xalloc(size_t n) { return malloc(n ? n : 1); }

static void table_free(Table* t) {
  free(t->rows);
  t->rows = NULL;
  t->n = 0;
}

/* ---- integer hash map int64 -> int64 (open addressing) ---- */
typedef struct {
  int64_t* keys;
  int64_t* vals;
  uint8_t* used;
  uint64_t mask;
} Map;

static uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
  return x ^ (x >> 33);
}
static int map_init(Map* m, int64_t n) {
  uint64_t cap = 16;
  while (cap < (uint64_t)n * 2 + 2) cap <<= 1;
  m->keys = xalloc(cap * 8);
  m->vals = xalloc(cap * 8);
  m->used = calloc(cap, 1);
  m->mask = cap - 1;
  return m->keys && m->vals && m->used;
}
static void map_free(Map* m) { free(m->keys); free(m->vals); free(m->used); }
/* returns pointer to value; *fresh = 1 when the key was inserted now */
static int64_t* map_slot(Map* m, int64_t key, int* fresh) {
  uint64_t h = mix64((uint64_t)key) & m->mask;
  while (m->used[h]) {
    if (m->keys[h] == key) { *fresh = 0; return &m->vals[h]; }
    h = (h + 1) & m->mask;
  }
  m->used[h] = 1;
  m->keys[h] = key;
  *fresh = 1;
  return &m->vals[h];
}
static const int64_t* map_get(const Map* m, int64_t key) {
  uint64_t h = mix64((uint64_t)key) & m->mask;
  while (m->used[h]) {
    if (m->keys[h] == key) return &m->vals[h];
    h = (h + 1) & m->mask;
  }
  return NULL;
}

/* first index i in [lo,hi) of pairs (2*i) with pairs[2i] >= key */
static int64_t lower_key(const uint64_t* pairs, int64_t lo, int64_t hi, uint64_t key) {
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (pairs[2 * mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* executor.py:94-127 */
static int scan(const orc_pattern* p, const orc_pred* m, Table* t) {
  int sv = p->s_var >= 0, ov = p->o_var >= 0;
  t->rows = NULL;
  t->n = 0;
  if (sv && ov) {
    if (p->s_var == p->o_var) { t->arity = 1; t->schema[0] = p->s_var; }
    else { t->arity = 2; t->schema[0] = p->s_var; t->schema[1] = p->o_var; }
  } else if (sv) { t->arity = 1; t->schema[0] = p->s_var; }
  else if (ov) { t->arity = 1; t->schema[0] = p->o_var; }
  else t->arity = 0;
  if (p->empty || m == NULL || m->so == NULL) return ORC_OK;
  int64_t nnz = m->nnz;
  if (sv && ov) {
    t->rows = xalloc(sizeof(int64_t) * (size_t)nnz * t->arity);
    if (!t->rows) return ORC_ERR_NOMEM;
    if (p->s_var == p->o_var) {
      for (int64_t i = 0; i < nnz; i++)
        if (m->so[2 * i] == m->so[2 * i + 1]) t->rows[t->n++] = (int64_t)m->so[2 * i];
    } else {
      for (int64_t i = 0; i < nnz; i++) {
        t->rows[2 * i] = (int64_t)m->so[2 * i];
        t->rows[2 * i + 1] = (int64_t)m->so[2 * i + 1];
      }
      t->n = nnz;
    }
  } else if (sv || ov) {
    /* pairs_for_object(o) -> (a,) from os;  pairs_for_subject(s) -> (b,) from so */
    const uint64_t* pr = sv ? m->os : m->so;
    uint64_t key = (uint64_t)(sv ? p->o_const : p->s_const);
    int64_t lo = lower_key(pr, 0, nnz, key), hi = lower_key(pr, lo, nnz, key + 1);
    t->rows = xalloc(sizeof(int64_t) * (size_t)(hi - lo));
    if (!t->rows) return ORC_ERR_NOMEM;
    for (int64_t i = lo; i < hi; i++) t->rows[t->n++] = (int64_t)pr[2 * i + 1];
  } else {
    /* contains(s, o): any pair of the s-run with second == o */
    uint64_t s = (uint64_t)p->s_const, o = (uint64_t)p->o_const;
    int64_t lo = lower_key(m->so, 0, nnz, s), hi = lower_key(m->so, lo, nnz, s + 1);
    int hit = 0;
    for (int64_t i = lo; i < hi && !hit; i++) hit = m->so[2 * i + 1] == o;
    t->rows = xalloc(8);
    t->n = hit ? 1 : 0;
  }
  return ORC_OK;
}

static int schema_index(const Table* t, int32_t v) {
  for (int i = 0; i < t->arity; i++)
    if (t->schema[i] == v) return i;
  return -1;
}

/* executor.py:130-137: stable group-by on column idx, first-occurrence key order */
static int regroup(Table* t, int idx) {
  if (t->n == 0) return ORC_OK;
  Map m;
  if (!map_init(&m, t->n)) return ORC_ERR_NOMEM;
  int64_t ngroups = 0;
  int64_t* gid = xalloc(sizeof(int64_t) * (size_t)t->n);
  int64_t* cnt = xalloc(sizeof(int64_t) * (size_t)(t->n + 1));
  if (!gid || !cnt) return ORC_ERR_NOMEM;
  for (int64_t i = 0; i < t->n; i++) {
    int fresh;
    int64_t* v = map_slot(&m, t->rows[i * t->arity + idx], &fresh);
    if (fresh) { *v = ngroups; cnt[ngroups++] = 0; }
    gid[i] = *v;
    cnt[*v]++;
  }
  int64_t acc = 0;
  for (int64_t g = 0; g < ngroups; g++) { int64_t c = cnt[g]; cnt[g] = acc; acc += c; }
  int64_t* out = xalloc(sizeof(int64_t) * (size_t)t->n * (t->arity ? t->arity : 1));
  if (!out) return ORC_ERR_NOMEM;
  for (int64_t i = 0; i < t->n; i++) {
    int64_t dst = cnt[gid[i]]++;
    memcpy(out + dst * t->arity, t->rows + i * t->arity, sizeof(int64_t) * t->arity);
  }
  free(t->rows);
  t->rows = out;
  free(gid); free(cnt); map_free(&m);
  return ORC_OK;
}

/* executor.py:155-165 */
static int cross_product(Table* L, const Table* R, int64_t budget, Table* out) {
  int64_t total;
  if (__builtin_mul_overflow(L->n, R->n, &total) || total > budget) {
    snprintf(g_msg, sizeof g_msg, "cross product of %lld x %lld rows exceeds budget %lld",
             (long long)L->n, (long long)R->n, (long long)budget);
    return ORC_ERR_RESOURCE;
  }
  out->arity = L->arity + R->arity;
  if (out->arity > 64) { snprintf(g_msg, sizeof g_msg, "too many variables"); return ORC_ERR_VALUE; }
  memcpy(out->schema, L->schema, sizeof(int32_t) * L->arity);
  memcpy(out->schema + L->arity, R->schema, sizeof(int32_t) * R->arity);
  out->n = total;
  out->rows = xalloc(sizeof(int64_t) * (size_t)total * (out->arity ? out->arity : 1));
  if (!out->rows) return ORC_ERR_NOMEM;
  int64_t k = 0;
  for (int64_t i = 0; i < L->n; i++)
    for (int64_t j = 0; j < R->n; j++) {
      memcpy(out->rows + k, L->rows + i * L->arity, sizeof(int64_t) * L->arity);
      k += L->arity;
      memcpy(out->rows + k, R->rows + j * R->arity, sizeof(int64_t) * R->arity);
      k += R->arity;
    }
  return ORC_OK;
}

/* executor.py:140-152 + 168-194 (+ 197-215 for E, 237-241 for the parallel budget).
 * Row order equals sm_join's; parallel_sm_join's compacted order is the same
 * when the left table is regrouped on the first join variable (test_executor.py:127-135). */
static int join(Table* L, const Table* R, const int32_t* jv, int njv, int64_t budget,
                int budget_mode, int64_t* prealloc_total, Table* out) {
  int li = schema_index(L, jv[0]), ri = schema_index(R, jv[0]);
  int sec_l[64], sec_r[64], nsec = 0;
  for (int k = 1; k < njv; k++) {
    sec_l[nsec] = schema_index(L, jv[k]);
    sec_r[nsec] = schema_index(R, jv[k]);
    nsec++;
  }
  int rcols[64], nrc = 0;
  for (int i = 0; i < R->arity; i++)
    if (schema_index(L, R->schema[i]) < 0) rcols[nrc++] = i;
  out->arity = L->arity + nrc;
  if (out->arity > 64) { snprintf(g_msg, sizeof g_msg, "too many variables"); return ORC_ERR_VALUE; }
  memcpy(out->schema, L->schema, sizeof(int32_t) * L->arity);
  for (int i = 0; i < nrc; i++) out->schema[L->arity + i] = R->schema[rcols[i]];

  /* groups: key -> right rows in scan order (counting layout) */
  Map m;
  if (!map_init(&m, R->n)) return ORC_ERR_NOMEM;
  int64_t ng = 0;
  int64_t* gcnt = xalloc(sizeof(int64_t) * (size_t)(R->n + 1));
  int64_t* rg = xalloc(sizeof(int64_t) * (size_t)(R->n + 1));
  if (!gcnt || !rg) return ORC_ERR_NOMEM;
  for (int64_t j = 0; j < R->n; j++) {
    int fresh;
    int64_t* v = map_slot(&m, R->rows[j * R->arity + ri], &fresh);
    if (fresh) { *v = ng; gcnt[ng++] = 0; }
    rg[j] = *v;
    gcnt[*v]++;
  }
  int64_t* gstart = xalloc(sizeof(int64_t) * (size_t)(ng + 1));
  int64_t* order = xalloc(sizeof(int64_t) * (size_t)(R->n + 1));
  if (!gstart || !order) return ORC_ERR_NOMEM;
  int64_t acc = 0;
  for (int64_t g = 0; g < ng; g++) { gstart[g] = acc; acc += gcnt[g]; }
  gstart[ng] = acc;
  int64_t* fillp = xalloc(sizeof(int64_t) * (size_t)(ng + 1));
  memcpy(fillp, gstart, sizeof(int64_t) * (size_t)(ng + 1));
  for (int64_t j = 0; j < R->n; j++) order[fillp[rg[j]]++] = j;
  free(fillp);

  /* preallocate(): E = sum over left rows of the matching right-group size */
  int64_t E = 0;
  for (int64_t i = 0; i < L->n; i++) {
    const int64_t* g = map_get(&m, L->rows[i * L->arity + li]);
    if (g) E += gcnt[*g];
  }
  *prealloc_total = E;
  if (budget_mode == 1 && E > budget) {
    snprintf(g_msg, sizeof g_msg, "pre-allocated join region of %lld rows exceeds budget %lld",
             (long long)E, (long long)budget);
    free(gcnt); free(rg); free(gstart); free(order); map_free(&m);
    return ORC_ERR_RESOURCE;
  }

  int64_t cap = E > 0 ? E : 1;
  out->rows = xalloc(sizeof(int64_t) * (size_t)cap * (out->arity ? out->arity : 1));
  if (!out->rows) return ORC_ERR_NOMEM;
  out->n = 0;
  int rc = ORC_OK;
  for (int64_t i = 0; i < L->n && rc == ORC_OK; i++) {
    const int64_t* lrow = L->rows + i * L->arity;
    const int64_t* g = map_get(&m, lrow[li]);
    if (g) {
      for (int64_t q = gstart[*g]; q < gstart[*g + 1]; q++) {
        const int64_t* rrow = R->rows + order[q] * R->arity;
        int ok = 1;
        for (int k = 0; k < nsec && ok; k++) ok = lrow[sec_l[k]] == rrow[sec_r[k]];
        if (!ok) continue;
        int64_t* dst = out->rows + out->n * out->arity;
        memcpy(dst, lrow, sizeof(int64_t) * L->arity);
        for (int c = 0; c < nrc; c++) dst[L->arity + c] = rrow[rcols[c]];
        out->n++;
      }
    }
    if (budget_mode == 0 && out->n > budget) {
      snprintf(g_msg, sizeof g_msg, "join output exceeds row budget %lld", (long long)budget);
      rc = ORC_ERR_RESOURCE;
    }
  }
  free(gcnt); free(rg); free(gstart); free(order); map_free(&m);
  return rc;
}

/* ---- DISTINCT on projected rows: first occurrence kept (executor.py:360-367) ---- */
static uint64_t row_hash(const int64_t* r, int k) {
  uint64_t h = 0x9E3779B97F4A7C15ULL;
  for (int i = 0; i < k; i++) h = mix64(h ^ (uint64_t)r[i]) + (uint64_t)i;
  return h;
}

static int64_t distinct_rows(int64_t* rows, int64_t n, int k) {
  if (n == 0) return 0;
  uint64_t cap = 16;
  while (cap < (uint64_t)n * 2 + 2) cap <<= 1;
  int64_t* slot = xalloc(sizeof(int64_t) * cap);
  for (uint64_t i = 0; i < cap; i++) slot[i] = -1;
  int64_t m = 0;
  for (int64_t i = 0; i < n; i++) {
    const int64_t* r = rows + i * k;
    uint64_t h = row_hash(r, k) & (cap - 1);
    int dup = 0;
    while (slot[h] >= 0) {
      if (memcmp(rows + slot[h] * k, r, sizeof(int64_t) * k) == 0) { dup = 1; break; }
      h = (h + 1) & (cap - 1);
    }
    if (dup) continue;
    if (m != i) memmove(rows + m * k, r, sizeof(int64_t) * k);
    slot[h] = m;
    m++;
  }
  free(slot);
  return m;
}

/* executor.py:296-368.  budget_mode: 0 = sequential, 1 = parallel semantics.
 * step_rows/step_prealloc: per plan step (StepReport.rows / prealloc_total). */
int orc_execute_part(const orc_pred* preds, int32_t max_pid, const orc_pattern* pats, int32_t n,
                     const int32_t* proj, int32_t nproj, int32_t distinct, int64_t budget,
                     int32_t budget_mode, int64_t part, int64_t parts, int64_t* step_rows,
                     int64_t* step_prealloc, int64_t** out_rows, int64_t* out_n);

int orc_execute(const orc_pred* preds, int32_t max_pid, const orc_pattern* pats, int32_t n,
                const int32_t* proj, int32_t nproj, int32_t distinct, int64_t budget,
                int32_t budget_mode, int64_t* step_rows, int64_t* step_prealloc,
                int64_t** out_rows, int64_t* out_n) {
  return orc_execute_part(preds, max_pid, pats, n, proj, nproj, distinct, budget, budget_mode, 0, 1,
                          step_rows, step_prealloc, out_rows, out_n);
}

/* Row partitioning (the multi-GPU split of gsm_execute): only rows
 * [n*part/parts, n*(part+1)/parts) of the first table enter the chain. */
int orc_execute_part(const orc_pred* preds, int32_t max_pid, const orc_pattern* pats, int32_t n,
                     const int32_t* proj, int32_t nproj, int32_t distinct, int64_t budget,
                     int32_t budget_mode, int64_t part, int64_t parts, int64_t* step_rows,
                     int64_t* step_prealloc, int64_t** out_rows, int64_t* out_n) {
  g_msg[0] = 0;
  *out_rows = NULL;
  *out_n = 0;
  if (n <= 0) { snprintf(g_msg, sizeof g_msg, "cannot execute an empty plan"); return ORC_ERR_VALUE; }
#define MAT(p) (((p)->pid >= 1 && (p)->pid <= max_pid && preds[(p)->pid].so) ? &preds[(p)->pid] : NULL)
  Table cur;
  int rc = scan(&pats[0], MAT(&pats[0]), &cur);
  if (rc) return rc;
  if (parts > 1) {
    int64_t lo = (int64_t)((__int128)cur.n * part / parts);
    int64_t hi = (int64_t)((__int128)cur.n * (part + 1) / parts);
    if (lo > 0 && cur.arity > 0)
      memmove(cur.rows, cur.rows + lo * cur.arity, sizeof(int64_t) * (size_t)(hi - lo) * cur.arity);
    cur.n = hi - lo;
  }
  if (step_rows) step_rows[0] = cur.n;
  if (step_prealloc) step_prealloc[0] = 0;
  for (int32_t s = 1; s < n; s++) {
    Table right, next;
    memset(&next, 0, sizeof next);
    rc = scan(&pats[s], MAT(&pats[s]), &right);
    if (rc) { table_free(&cur); return rc; }
    int32_t jv[64];
    int njv = 0;
    for (int i = 0; i < cur.arity; i++)
      if (schema_index(&right, cur.schema[i]) >= 0) jv[njv++] = cur.schema[i];
    int64_t E = 0;
    if (njv == 0) {
      rc = cross_product(&cur, &right, budget, &next);
    } else {
      rc = regroup(&cur, schema_index(&cur, jv[0]));
      if (!rc) rc = join(&cur, &right, jv, njv, budget, budget_mode, &E, &next);
    }
    table_free(&right);
    table_free(&cur);
    if (rc) { table_free(&next); return rc; }
    cur = next;
    if (step_rows) step_rows[s] = cur.n;
    if (step_prealloc) step_prealloc[s] = E;
  }
#undef MAT
  int pidx[64];
  for (int j = 0; j < nproj; j++) {
    pidx[j] = schema_index(&cur, proj[j]);
    if (pidx[j] < 0) {
      snprintf(g_msg, sizeof g_msg, "projected variable %d not in result schema", proj[j]);
      table_free(&cur);
      return ORC_ERR_VALUE;
    }
  }
  int64_t* res = xalloc(sizeof(int64_t) * (size_t)cur.n * (nproj ? nproj : 1));
  if (!res) { table_free(&cur); return ORC_ERR_NOMEM; }
  for (int64_t i = 0; i < cur.n; i++)
    for (int j = 0; j < nproj; j++) res[i * nproj + j] = cur.rows[i * cur.arity + pidx[j]];
  int64_t m = cur.n;
  if (distinct) m = distinct_rows(res, cur.n, nproj);
  table_free(&cur);
  *out_rows = res;
  *out_n = m;
  return ORC_OK;
}

void orc_free(void* p) { free(p); }
