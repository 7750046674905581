/*
 * gsmgen — seeded synthetic RDF generators that write the gSMat store
 * directory layout directly (test/bench input tooling, not the product).
 *
 * The store layout is the reference's persist() format
 * (/root/reference/pkg/src/gsmat/storage.py:203-219):
 *   meta        "GSMAT1\n<triples>\n<predicates>\n<nodes>\n"
 *   nodes.dict  one escaped term per line, id = 1-based line number
 *   preds.dict  same for predicates
 *   p<ID>.so    u64 LE (s,o) pairs sorted by (s,o)
 *   p<ID>.os    u64 LE (o,s) pairs sorted by (o,s)
 *   stats.tsv   pid \t cardinality \t distinct_subjects \t distinct_objects
 *
 * Ids are assigned exactly as `gsmat build` assigns them
 * (cli.py:64-82 -> dictionary.py:57-72): for every triple in stream order
 * encode_node(s), encode_predicate(p), encode_node(o), first occurrence wins.
 * Duplicate triples are dropped per predicate (storage.py:165-177).  So
 * `gsmgen ... --nt X` followed by `gsmat build --input X` yields a
 * byte-identical store directory (checked in tests/test_datagen.py).
 *
 * Generators
 *   lubm      LUBM/UBA-style university data (universities -> departments ->
 *             faculty/students/courses/publications/research groups).
 *   watdiv    WatDiv-style e-commerce/social data (users, products, reviews,
 *             offers, retailers, websites, purchases), Zipf-skewed links.
 *   powerlaw  bit-exact restatement of generate.py (generate.py:17-64):
 *             CPython's MT19937 + random.choices(cum_weights=...) over a Zipf
 *             predicate distribution and i^-NODE_SKEW endpoint weights.
 */
#define _GNU_SOURCE
#include <errno.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>

static void die(const char* msg) {
  fprintf(stderr, "gsmgen: %s\n", msg);
  exit(1);
}

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) die("out of memory");
  return p;
}
static void* xrealloc(void* p, size_t n) {
  p = realloc(p, n ? n : 1);
  if (!p) die("out of memory");
  return p;
}

/* ------------------------------------------------------------------ */
/* Term dictionary: first-occurrence dense 1-based ids.               */
/* ------------------------------------------------------------------ */
typedef struct {
  char* bytes;       /* terms back to back */
  size_t nbytes, capbytes;
  uint64_t* start;   /* start[id-1] = offset of term id; start[count] = end */
  uint32_t count, capterms;
  uint32_t* slots;   /* hash slots holding ids, 0 = empty */
  uint64_t mask;
} Dict;

static uint64_t hash_bytes(const char* s, size_t n) {
  uint64_t h = 1469598103934665603ULL;
  for (size_t i = 0; i < n; i++) {
    h ^= (unsigned char)s[i];
    h *= 1099511628211ULL;
  }
  h ^= h >> 29;
  h *= 0xBF58476D1CE4E5B9ULL;
  h ^= h >> 32;
  return h;
}

static void dict_init(Dict* d, uint64_t slots_pow2) {
  memset(d, 0, sizeof(*d));
  d->capbytes = 1 << 20;
  d->bytes = xmalloc(d->capbytes);
  d->capterms = 1 << 16;
  d->start = xmalloc(sizeof(uint64_t) * (d->capterms + 1));
  d->start[0] = 0;
  d->mask = slots_pow2 - 1;
  d->slots = calloc(slots_pow2, sizeof(uint32_t));
  if (!d->slots) die("out of memory");
}

static int dict_eq(const Dict* d, uint32_t id, const char* s, size_t n) {
  uint64_t a = d->start[id - 1], b = d->start[id];
  return (b - a) == n && memcmp(d->bytes + a, s, n) == 0;
}

static void dict_grow_slots(Dict* d) {
  uint64_t ncap = (d->mask + 1) * 2;
  uint32_t* ns = calloc(ncap, sizeof(uint32_t));
  if (!ns) die("out of memory");
  for (uint32_t id = 1; id <= d->count; id++) {
    uint64_t a = d->start[id - 1], b = d->start[id];
    uint64_t h = hash_bytes(d->bytes + a, b - a) & (ncap - 1);
    while (ns[h]) h = (h + 1) & (ncap - 1);
    ns[h] = id;
  }
  free(d->slots);
  d->slots = ns;
  d->mask = ncap - 1;
}

static uint32_t dict_encode(Dict* d, const char* s, size_t n) {
  uint64_t h = hash_bytes(s, n) & d->mask;
  for (;;) {
    uint32_t id = d->slots[h];
    if (!id) break;
    if (dict_eq(d, id, s, n)) return id;
    h = (h + 1) & d->mask;
  }
  if (d->count == UINT32_MAX - 1) die("too many terms for 32-bit ids");
  if (d->nbytes + n > d->capbytes) {
    while (d->nbytes + n > d->capbytes) d->capbytes *= 2;
    d->bytes = xrealloc(d->bytes, d->capbytes);
  }
  memcpy(d->bytes + d->nbytes, s, n);
  d->nbytes += n;
  if (d->count + 1 > d->capterms) {
    d->capterms *= 2;
    d->start = xrealloc(d->start, sizeof(uint64_t) * (d->capterms + 1));
  }
  d->count++;
  d->start[d->count] = d->nbytes;
  d->slots[h] = d->count;
  if ((uint64_t)d->count * 2 > d->mask + 1) dict_grow_slots(d);
  return d->count;
}

/* ------------------------------------------------------------------ */
/* Triple stream                                                      */
/* ------------------------------------------------------------------ */
typedef struct {
  uint32_t *s, *p, *o;
  uint64_t n, cap;
} Triples;

static Dict g_nodes, g_preds;
static Triples g_tr;
static FILE* g_nt = NULL;

static void tr_push(uint32_t s, uint32_t p, uint32_t o) {
  if (g_tr.n == g_tr.cap) {
    g_tr.cap = g_tr.cap ? g_tr.cap * 2 : (1 << 20);
    g_tr.s = xrealloc(g_tr.s, g_tr.cap * 4);
    g_tr.p = xrealloc(g_tr.p, g_tr.cap * 4);
    g_tr.o = xrealloc(g_tr.o, g_tr.cap * 4);
  }
  g_tr.s[g_tr.n] = s;
  g_tr.p[g_tr.n] = p;
  g_tr.o[g_tr.n] = o;
  g_tr.n++;
}

static void nt_term(const char* t) {
  if (t[0] == '"') fputs(t, g_nt);  /* canonical literal keeps its quotes */
  else { fputc('<', g_nt); fputs(t, g_nt); fputc('>', g_nt); }
}

/* Emit one triple of canonical terms (IRIs bare, literals quoted). */
static void T(const char* s, const char* p, const char* o) {
  uint32_t si = dict_encode(&g_nodes, s, strlen(s));
  uint32_t pi = dict_encode(&g_preds, p, strlen(p));
  uint32_t oi = dict_encode(&g_nodes, o, strlen(o));
  tr_push(si, pi, oi);
  if (g_nt) {
    nt_term(s); fputc(' ', g_nt); nt_term(p); fputc(' ', g_nt); nt_term(o);
    fputs(" .\n", g_nt);
  }
}

/* ------------------------------------------------------------------ */
/* Store writer                                                       */
/* ------------------------------------------------------------------ */
static void radix_sort_u64(uint64_t* a, uint64_t n, uint64_t* tmp) {
  if (n < 2) return;
  uint64_t all_or = 0, all_and = ~0ULL;
  for (uint64_t i = 0; i < n; i++) { all_or |= a[i]; all_and &= a[i]; }
  static uint64_t cnt[1 << 16];
  uint64_t *src = a, *dst = tmp;
  for (int shift = 0; shift < 64; shift += 16) {
    uint64_t m = 0xFFFFULL << shift;
    if (((all_or ^ all_and) & m) == 0) continue; /* digit constant: skip */
    memset(cnt, 0, sizeof(cnt));
    for (uint64_t i = 0; i < n; i++) cnt[(src[i] >> shift) & 0xFFFF]++;
    uint64_t acc = 0;
    for (int d = 0; d < (1 << 16); d++) { uint64_t c = cnt[d]; cnt[d] = acc; acc += c; }
    for (uint64_t i = 0; i < n; i++) dst[cnt[(src[i] >> shift) & 0xFFFF]++] = src[i];
    uint64_t* t = src; src = dst; dst = t;
  }
  if (src != a) memcpy(a, src, n * sizeof(uint64_t));
}

static void write_escaped_dict(const char* path, const Dict* d) {
  FILE* f = fopen(path, "wb");
  if (!f) die("cannot open dictionary file for writing");
  setvbuf(f, NULL, _IOFBF, 1 << 22);
  for (uint32_t id = 1; id <= d->count; id++) {
    const char* s = d->bytes + d->start[id - 1];
    uint64_t n = d->start[id] - d->start[id - 1];
    for (uint64_t i = 0; i < n; i++) {  /* dictionary.escape_term */
      char c = s[i];
      if (c == '\\') fputs("\\\\", f);
      else if (c == '\n') fputs("\\n", f);
      else if (c == '\r') fputs("\\r", f);
      else if (c == '\t') fputs("\\t", f);
      else fputc(c, f);
    }
    fputc('\n', f);
  }
  fclose(f);
}

static void write_pairs(const char* path, const uint64_t* keys, uint64_t n) {
  FILE* f = fopen(path, "wb");
  if (!f) die("cannot open pair file for writing");
  setvbuf(f, NULL, _IOFBF, 1 << 22);
  uint64_t buf[2 * 4096];
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; i++) {
    buf[k++] = keys[i] >> 32;
    buf[k++] = keys[i] & 0xFFFFFFFFULL;
    if (k == 2 * 4096) { fwrite(buf, 8, k, f); k = 0; }
  }
  if (k) fwrite(buf, 8, k, f);
  fclose(f);
}

static uint64_t count_runs(const uint64_t* keys, uint64_t n) {
  uint64_t runs = 0;
  for (uint64_t i = 0; i < n; i++)
    if (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) runs++;
  return runs;
}

static void write_store(const char* dir) {
  if (mkdir(dir, 0755) != 0 && errno != EEXIST) die("cannot create store directory");
  char path[4096];
  uint32_t np = g_preds.count;
  /* bucket triples by predicate */
  uint64_t* cnt = calloc((size_t)np + 2, sizeof(uint64_t));
  for (uint64_t i = 0; i < g_tr.n; i++) cnt[g_tr.p[i] + 1]++;
  for (uint32_t p = 1; p <= np + 1; p++) cnt[p] += cnt[p - 1];
  uint64_t* keys = xmalloc(sizeof(uint64_t) * (g_tr.n + 1));
  uint64_t* fill = xmalloc(sizeof(uint64_t) * ((size_t)np + 2));
  memcpy(fill, cnt, sizeof(uint64_t) * ((size_t)np + 2));
  for (uint64_t i = 0; i < g_tr.n; i++)
    keys[fill[g_tr.p[i]]++] = ((uint64_t)g_tr.s[i] << 32) | g_tr.o[i];
  free(fill);
  uint64_t maxn = 0;
  for (uint32_t p = 1; p <= np; p++)
    if (cnt[p + 1] - cnt[p] > maxn) maxn = cnt[p + 1] - cnt[p];
  uint64_t* tmp = xmalloc(sizeof(uint64_t) * (maxn + 1));
  uint64_t* os = xmalloc(sizeof(uint64_t) * (maxn + 1));
  uint64_t total = 0;
  snprintf(path, sizeof path, "%s/stats.tsv", dir);
  FILE* st = fopen(path, "wb");
  if (!st) die("cannot write stats.tsv");
  for (uint32_t p = 1; p <= np; p++) {
    uint64_t* a = keys + cnt[p];
    uint64_t n = cnt[p + 1] - cnt[p];
    radix_sort_u64(a, n, tmp);
    uint64_t m = 0;  /* set semantics: drop duplicate triples */
    for (uint64_t i = 0; i < n; i++)
      if (m == 0 || a[i] != a[m - 1]) a[m++] = a[i];
    for (uint64_t i = 0; i < m; i++) os[i] = (a[i] << 32) | (a[i] >> 32);
    radix_sort_u64(os, m, tmp);
    snprintf(path, sizeof path, "%s/p%u.so", dir, p);
    write_pairs(path, a, m);
    snprintf(path, sizeof path, "%s/p%u.os", dir, p);
    write_pairs(path, os, m);
    fprintf(st, "%u\t%llu\t%llu\t%llu\n", p, (unsigned long long)m,
            (unsigned long long)count_runs(a, m), (unsigned long long)count_runs(os, m));
    total += m;
  }
  fclose(st);
  snprintf(path, sizeof path, "%s/nodes.dict", dir);
  write_escaped_dict(path, &g_nodes);
  snprintf(path, sizeof path, "%s/preds.dict", dir);
  write_escaped_dict(path, &g_preds);
  snprintf(path, sizeof path, "%s/meta", dir);
  FILE* mf = fopen(path, "wb");
  if (!mf) die("cannot write meta");
  fprintf(mf, "GSMAT1\n%llu\n%u\n%u\n", (unsigned long long)total, np, g_nodes.count);
  fclose(mf);
  fprintf(stdout, "%llu triples, %u predicates, %u nodes\n", (unsigned long long)total, np,
          g_nodes.count);
  free(cnt); free(keys); free(tmp); free(os);
}

/* ------------------------------------------------------------------ */
/* LUBM / UBA-style generator                                         */
/* ------------------------------------------------------------------ */
static uint64_t g_rng;
static uint64_t rnext(void) { /* splitmix64 */
  uint64_t z = (g_rng += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static int rrange(int lo, int hi) { return lo + (int)(rnext() % (uint64_t)(hi - lo + 1)); }

#define UB "http://swat.cse.lehigh.edu/onto/univ-bench.owl#"
#define RDF_TYPE "http://www.w3.org/1999/02/22-rdf-syntax-ns#type"

enum { FP = 0, AP = 1, ASP = 2, LEC = 3, NKIND = 4 };
static const char* KIND[NKIND] = {"FullProfessor", "AssociateProfessor", "AssistantProfessor",
                                  "Lecturer"};
static const int KMIN[NKIND] = {7, 10, 8, 5}, KMAX[NKIND] = {10, 14, 11, 7};
static const int PMIN[NKIND] = {15, 10, 5, 0}, PMAX[NKIND] = {20, 18, 10, 5};

static void gen_lubm(int univs, int pool) {
  char univ[128], dept[160], e[256], lit[512], x[512];
  int* npub = xmalloc(sizeof(int) * 64);
  int cap_npub = 64;
  for (int u = 0; u < univs; u++) {
    snprintf(univ, sizeof univ, "http://www.University%d.edu", u);
    T(univ, RDF_TYPE, UB "University");
    snprintf(lit, sizeof lit, "\"University%d\"", u);
    T(univ, UB "name", lit);
    int ndept = rrange(15, 25);
    for (int d = 0; d < ndept; d++) {
      snprintf(dept, sizeof dept, "http://www.Department%d.University%d.edu", d, u);
      T(dept, RDF_TYPE, UB "Department");
      snprintf(lit, sizeof lit, "\"Department%d\"", d);
      T(dept, UB "name", lit);
      T(dept, UB "subOrganizationOf", univ);
      int nk[NKIND], nfac = 0, nprof = 0;
      for (int k = 0; k < NKIND; k++) { nk[k] = rrange(KMIN[k], KMAX[k]); nfac += nk[k]; }
      nprof = nk[FP] + nk[AP] + nk[ASP];
      if (nfac > cap_npub) { cap_npub = nfac; npub = xrealloc(npub, sizeof(int) * cap_npub); }
      int ncourse = 0, ngcourse = 0, fi = 0;
      for (int k = 0; k < NKIND; k++) {
        for (int i = 0; i < nk[k]; i++, fi++) {
          snprintf(e, sizeof e, "%s/%s%d", dept, KIND[k], i);
          T(e, RDF_TYPE, k == FP ? UB "FullProfessor" : k == AP ? UB "AssociateProfessor"
                        : k == ASP ? UB "AssistantProfessor" : UB "Lecturer");
          snprintf(lit, sizeof lit, "\"%s%d\"", KIND[k], i);
          T(e, UB "name", lit);
          int nc = rrange(1, 2);
          for (int c = 0; c < nc; c++, ncourse++) {
            snprintf(x, sizeof x, "%s/Course%d", dept, ncourse);
            T(e, UB "teacherOf", x);
            T(x, RDF_TYPE, UB "Course");
            snprintf(lit, sizeof lit, "\"Course%d\"", ncourse);
            T(x, UB "name", lit);
          }
          if (k != LEC) {
            int ng = rrange(1, 2);
            for (int c = 0; c < ng; c++, ngcourse++) {
              snprintf(x, sizeof x, "%s/GraduateCourse%d", dept, ngcourse);
              T(e, UB "teacherOf", x);
              T(x, RDF_TYPE, UB "GraduateCourse");
              snprintf(lit, sizeof lit, "\"GraduateCourse%d\"", ngcourse);
              T(x, UB "name", lit);
            }
          }
          snprintf(x, sizeof x, "http://www.University%d.edu", rrange(0, pool - 1));
          T(e, UB "undergraduateDegreeFrom", x);
          snprintf(x, sizeof x, "http://www.University%d.edu", rrange(0, pool - 1));
          T(e, UB "mastersDegreeFrom", x);
          snprintf(x, sizeof x, "http://www.University%d.edu", rrange(0, pool - 1));
          T(e, UB "doctoralDegreeFrom", x);
          T(e, UB "worksFor", dept);
          if (k == FP && i == 0) T(e, UB "headOf", dept);
          snprintf(lit, sizeof lit, "\"%s%d@Department%d.University%d.edu\"", KIND[k], i, d, u);
          T(e, UB "emailAddress", lit);
          T(e, UB "telephone", "\"xxx-xxx-xxxx\"");
          snprintf(lit, sizeof lit, "\"Research%d\"", rrange(0, 29));
          T(e, UB "researchInterest", lit);
          npub[fi] = rrange(PMIN[k], PMAX[k]);
          for (int j = 0; j < npub[fi]; j++) {
            snprintf(x, sizeof x, "%s/Publication%d", e, j);
            T(x, RDF_TYPE, UB "Publication");
            snprintf(lit, sizeof lit, "\"Publication%d\"", j);
            T(x, UB "name", lit);
            T(x, UB "publicationAuthor", e);
          }
        }
      }
      /* professor index -> (kind, i) for advisor/co-author picks */
#define PROF_NAME(buf, idx)                                                   \
  do {                                                                        \
    int _q = (idx), _k = 0;                                                   \
    while (_q >= nk[_k]) { _q -= nk[_k]; _k++; }                              \
    snprintf(buf, sizeof buf, "%s/%s%d", dept, KIND[_k], _q);                 \
  } while (0)
      int nug = nfac * rrange(8, 14);
      for (int i = 0; i < nug; i++) {
        snprintf(e, sizeof e, "%s/UndergraduateStudent%d", dept, i);
        T(e, RDF_TYPE, UB "UndergraduateStudent");
        snprintf(lit, sizeof lit, "\"UndergraduateStudent%d\"", i);
        T(e, UB "name", lit);
        T(e, UB "memberOf", dept);
        snprintf(lit, sizeof lit, "\"UndergraduateStudent%d@Department%d.University%d.edu\"", i, d, u);
        T(e, UB "emailAddress", lit);
        T(e, UB "telephone", "\"xxx-xxx-xxxx\"");
        int nt = rrange(2, 4), taken[4];
        for (int c = 0; c < nt && c < ncourse; c++) {
          int pick, dup;
          do {
            pick = rrange(0, ncourse - 1);
            dup = 0;
            for (int q = 0; q < c; q++) dup |= taken[q] == pick;
          } while (dup);
          taken[c] = pick;
          snprintf(x, sizeof x, "%s/Course%d", dept, pick);
          T(e, UB "takesCourse", x);
        }
        if (rnext() % 5 == 0) {
          PROF_NAME(x, rrange(0, nprof - 1));
          T(e, UB "advisor", x);
        }
      }
      int ngr = nfac * rrange(3, 4);
      for (int i = 0; i < ngr; i++) {
        snprintf(e, sizeof e, "%s/GraduateStudent%d", dept, i);
        T(e, RDF_TYPE, UB "GraduateStudent");
        snprintf(lit, sizeof lit, "\"GraduateStudent%d\"", i);
        T(e, UB "name", lit);
        T(e, UB "memberOf", dept);
        snprintf(lit, sizeof lit, "\"GraduateStudent%d@Department%d.University%d.edu\"", i, d, u);
        T(e, UB "emailAddress", lit);
        T(e, UB "telephone", "\"xxx-xxx-xxxx\"");
        snprintf(x, sizeof x, "http://www.University%d.edu", rrange(0, pool - 1));
        T(e, UB "undergraduateDegreeFrom", x);
        int nt = rrange(1, 3), taken[3];
        for (int c = 0; c < nt && c < ngcourse; c++) {
          int pick, dup;
          do {
            pick = rrange(0, ngcourse - 1);
            dup = 0;
            for (int q = 0; q < c; q++) dup |= taken[q] == pick;
          } while (dup);
          taken[c] = pick;
          snprintf(x, sizeof x, "%s/GraduateCourse%d", dept, pick);
          T(e, UB "takesCourse", x);
        }
        PROF_NAME(x, rrange(0, nprof - 1));
        T(e, UB "advisor", x);
        if (rnext() % 4 == 0 && ncourse > 0) {
          snprintf(x, sizeof x, "%s/Course%d", dept, rrange(0, ncourse - 1));
          T(e, UB "teachingAssistantOf", x);
        }
        if (rnext() % 4 == 0) { /* co-author one publication of a faculty member */
          int f = rrange(0, nfac - 1);
          if (npub[f] > 0) {
            int q = f, k = 0;
            while (q >= nk[k]) { q -= nk[k]; k++; }
            snprintf(x, sizeof x, "%s/%s%d/Publication%d", dept, KIND[k], q, rrange(0, npub[f] - 1));
            T(x, UB "publicationAuthor", e);
          }
        }
      }
      int nrg = rrange(10, 20);
      for (int i = 0; i < nrg; i++) {
        snprintf(e, sizeof e, "%s/ResearchGroup%d", dept, i);
        T(e, RDF_TYPE, UB "ResearchGroup");
        T(e, UB "subOrganizationOf", dept);
      }
#undef PROF_NAME
    }
  }
  free(npub);
}

/* ------------------------------------------------------------------ */
/* WatDiv-style generator (configs[3]).  Entity model after the WatDiv  */
/* benchmark's schema: users, products, reviews, offers, retailers,    */
/* websites, purchases, cities/countries, genres, topics, ...  Entity  */
/* counts scale with --scale (scale 1000 ~ 100M triples); link         */
/* targets are Zipf-skewed so popular products/users become hubs.      */
/* ------------------------------------------------------------------ */
#define WSDBM "http://db.uwaterloo.ca/~galuc/wsdbm/"
#define SORG "http://schema.org/"
#define GR "http://purl.org/goodrelations/"
#define REV "http://purl.org/stuff/rev#"
#define OG "http://ogp.me/ns#"
#define FOAF "http://xmlns.com/foaf/"
#define DC "http://purl.org/dc/terms/"
#define GN "http://www.geonames.org/ontology#"
#define MO "http://purl.org/ontology/mo/"

/* Zipf(s) sample in [0, n) by inverse CDF on a precomputed table. */
typedef struct { double* cum; uint32_t n; } Zipf;
static Zipf zipf_make(uint32_t n, double s) {
  Zipf z;
  z.n = n;
  z.cum = xmalloc(sizeof(double) * n);
  double acc = 0;
  for (uint32_t i = 0; i < n; i++) { acc += pow((double)(i + 1), -s); z.cum[i] = acc; }
  return z;
}
static uint32_t zipf_draw(const Zipf* z) {
  double x = (double)(rnext() >> 11) * (1.0 / 9007199254740992.0) * z->cum[z->n - 1];
  uint32_t lo = 0, hi = z->n - 1;
  while (lo < hi) {
    uint32_t mid = (lo + hi) / 2;
    if (x < z->cum[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}
static int rchance(double p) { return (double)(rnext() >> 11) * (1.0 / 9007199254740992.0) < p; }

static void gen_watdiv(int scale) {
  const uint32_t nU = 3000u * scale, nP = 750u * scale, nR = 4500u * scale, nO = 2700u * scale;
  const uint32_t nRet = 36u * scale, nW = 150u * scale, nPur = 4500u * scale;
  const uint32_t nCity = 240, nCountry = 25, nGenre = 21, nSub = 145, nCat = 15, nTopic = 250;
  const uint32_t nLang = 25, nRole = 3, nAge = 9;
  Zipf zU = zipf_make(nU, 0.8), zP = zipf_make(nP, 0.8), zW = zipf_make(nW, 0.7);
  Zipf zTopic = zipf_make(nTopic, 1.0), zSub = zipf_make(nSub, 0.9), zCity = zipf_make(nCity, 1.0);
  char e[256], x[256], lit[256];
#define ENT(buf, kind, i) snprintf(buf, sizeof buf, WSDBM "%s%u", kind, (unsigned)(i))
  for (uint32_t i = 0; i < nCity; i++) {
    ENT(e, "City", i);
    ENT(x, "Country", i % nCountry);
    T(e, GN "parentCountry", x);
  }
  for (uint32_t i = 0; i < nSub; i++) {
    ENT(e, "SubGenre", i);
    ENT(x, "Genre", i % nGenre);
    T(e, OG "tag", x);
    T(e, RDF_TYPE, WSDBM "SubGenre");
  }
  for (uint32_t i = 0; i < nW; i++) {
    ENT(e, "Website", i);
    snprintf(lit, sizeof lit, "\"http://www.website%u.com/\"", i);
    T(e, SORG "url", lit);
    snprintf(lit, sizeof lit, "\"%u\"", (unsigned)rrange(1, 100000));
    T(e, WSDBM "hits", lit);
    ENT(x, "Language", rrange(0, nLang - 1));
    T(e, SORG "language", x);
  }
  for (uint32_t i = 0; i < nP; i++) {
    ENT(e, "Product", i);
    ENT(x, "ProductCategory", rrange(0, nCat - 1));
    T(e, RDF_TYPE, x);
    snprintf(lit, sizeof lit, "\"caption %u\"", i);
    if (rchance(0.5)) T(e, SORG "caption", lit);
    snprintf(lit, sizeof lit, "\"text %u\"", i);
    if (rchance(0.3)) T(e, SORG "text", lit);
    snprintf(lit, sizeof lit, "\"description %u\"", i);
    if (rchance(0.7)) T(e, SORG "description", lit);
    snprintf(lit, sizeof lit, "\"keywords %u\"", i % 1000);
    if (rchance(0.3)) T(e, SORG "keywords", lit);
    snprintf(lit, sizeof lit, "\"title %u\"", i);
    T(e, OG "title", lit);
    int ng = rrange(1, 3);
    for (int g = 0; g < ng; g++) { ENT(x, "SubGenre", zipf_draw(&zSub)); T(e, WSDBM "hasGenre", x); }
    int nt = rrange(0, 4);
    for (int g = 0; g < nt; g++) { ENT(x, "Topic", zipf_draw(&zTopic)); T(e, OG "tag", x); }
    if (rchance(0.4)) { ENT(x, "Website", zipf_draw(&zW)); T(e, FOAF "homepage", x); }
    snprintf(lit, sizeof lit, "\"%d\"", rrange(1, 5));
    if (rchance(0.3)) T(e, SORG "contentRating", lit);
    snprintf(lit, sizeof lit, "\"%dMB\"", rrange(1, 500));
    if (rchance(0.3)) T(e, SORG "contentSize", lit);
    if (rchance(0.2)) { ENT(x, "Language", rrange(0, nLang - 1)); T(e, SORG "language", x); }
    if (rchance(0.1)) { ENT(x, "Retailer", rrange(0, nRet - 1)); T(e, SORG "publisher", x); }
    if (rchance(0.1)) { snprintf(lit, sizeof lit, "\"trailer %u\"", i); T(e, SORG "trailer", lit); }
    if (rchance(0.1)) { ENT(x, "User", zipf_draw(&zU)); T(e, SORG "director", x); }
    if (rchance(0.2)) { ENT(x, "User", zipf_draw(&zU)); T(e, SORG "actor", x); }
    if (rchance(0.1)) { ENT(x, "User", zipf_draw(&zU)); T(x, MO "artist", e); }
    if (rchance(0.05)) { ENT(x, "User", zipf_draw(&zU)); T(e, MO "conductor", x); }
  }
  for (uint32_t i = 0; i < nR; i++) {
    ENT(e, "Review", i);
    ENT(x, "Product", zipf_draw(&zP));
    T(x, REV "hasReview", e);
    ENT(x, "User", zipf_draw(&zU));
    T(e, REV "reviewer", x);
    snprintf(lit, sizeof lit, "\"%d\"", rrange(1, 10));
    T(e, REV "rating", lit);
    snprintf(lit, sizeof lit, "\"review title %u\"", i % 5000);
    if (rchance(0.5)) T(e, REV "title", lit);
    snprintf(lit, sizeof lit, "\"review text %u\"", i);
    if (rchance(0.5)) T(e, REV "text", lit);
    snprintf(lit, sizeof lit, "\"%d\"", rrange(0, 100));
    if (rchance(0.3)) T(e, REV "totalVotes", lit);
  }
  for (uint32_t i = 0; i < nRet; i++) {
    ENT(e, "Retailer", i);
    snprintf(lit, sizeof lit, "\"Retailer %u Inc.\"", i);
    T(e, SORG "legalName", lit);
    ENT(x, "User", zipf_draw(&zU));
    T(e, SORG "employee", x);
  }
  for (uint32_t i = 0; i < nO; i++) {
    ENT(e, "Offer", i);
    ENT(x, "Retailer", rrange(0, nRet - 1));
    T(x, GR "offers", e);
    ENT(x, "Product", zipf_draw(&zP));
    T(e, GR "includes", x);
    snprintf(lit, sizeof lit, "\"%d.%02d\"", rrange(1, 500), rrange(0, 99));
    T(e, GR "price", lit);
    snprintf(lit, sizeof lit, "\"SN%u\"", i);
    T(e, GR "serialNumber", lit);
    snprintf(lit, sizeof lit, "\"2019-%02d-%02d\"", rrange(1, 12), rrange(1, 28));
    T(e, GR "validFrom", lit);
    snprintf(lit, sizeof lit, "\"2020-%02d-%02d\"", rrange(1, 12), rrange(1, 28));
    T(e, GR "validThrough", lit);
    snprintf(lit, sizeof lit, "\"%d\"", rrange(1, 50));
    T(e, SORG "eligibleQuantity", lit);
    ENT(x, "Country", rrange(0, nCountry - 1));
    T(e, SORG "eligibleRegion", x);
    snprintf(lit, sizeof lit, "\"2020-%02d-%02d\"", rrange(1, 12), rrange(1, 28));
    T(e, SORG "priceValidUntil", lit);
  }
  for (uint32_t i = 0; i < nU; i++) {
    ENT(e, "User", i);
    snprintf(lit, sizeof lit, "\"user%u@example.org\"", i);
    T(e, SORG "email", lit);
    ENT(x, "Role", rrange(0, nRole - 1));
    T(e, RDF_TYPE, x);
    ENT(x, "Gender", rrange(0, 1));
    if (rchance(0.6)) T(e, WSDBM "gender", x);
    ENT(x, "AgeGroup", rrange(0, nAge - 1));
    if (rchance(0.5)) T(e, FOAF "age", x);
    snprintf(lit, sizeof lit, "\"family%u\"", i % 2000);
    if (rchance(0.7)) T(e, FOAF "familyName", lit);
    snprintf(lit, sizeof lit, "\"given%u\"", i % 1000);
    if (rchance(0.7)) T(e, FOAF "givenName", lit);
    ENT(x, "Country", zipf_draw(&zCity) % nCountry);
    if (rchance(0.5)) T(e, SORG "nationality", x);
    ENT(x, "City", zipf_draw(&zCity));
    if (rchance(0.4)) T(e, DC "Location", x);
    snprintf(lit, sizeof lit, "\"job %d\"", rrange(0, 200));
    if (rchance(0.05)) T(e, SORG "jobTitle", lit);
    if (rchance(0.1)) { ENT(x, "Website", zipf_draw(&zW)); T(e, FOAF "homepage", x); }
    int nf = rchance(0.4) ? rrange(1, 20) : 0;
    for (int k = 0; k < nf; k++) { ENT(x, "User", zipf_draw(&zU)); T(e, WSDBM "follows", x); }
    int nfr = rchance(0.4) ? rrange(1, 10) : 0;
    for (int k = 0; k < nfr; k++) { ENT(x, "User", zipf_draw(&zU)); T(e, WSDBM "friendOf", x); }
    int nl = rchance(0.25) ? rrange(1, 5) : 0;
    for (int k = 0; k < nl; k++) { ENT(x, "Product", zipf_draw(&zP)); T(e, WSDBM "likes", x); }
    int ns = rchance(0.1) ? rrange(1, 3) : 0;
    for (int k = 0; k < ns; k++) { ENT(x, "Website", zipf_draw(&zW)); T(e, WSDBM "subscribes", x); }
  }
  for (uint32_t i = 0; i < nPur; i++) {
    ENT(e, "Purchase", i);
    ENT(x, "User", zipf_draw(&zU));
    T(x, WSDBM "makesPurchase", e);
    ENT(x, "Product", zipf_draw(&zP));
    T(e, WSDBM "purchaseFor", x);
    snprintf(lit, sizeof lit, "\"2019-%02d-%02d\"", rrange(1, 12), rrange(1, 28));
    T(e, WSDBM "purchaseDate", lit);
  }
#undef ENT
  free(zU.cum); free(zP.cum); free(zW.cum); free(zTopic.cum); free(zSub.cum); free(zCity.cum);
}

/* ------------------------------------------------------------------ */
/* generate.py restatement (power-law)                                */
/* CPython MT19937 + random.choices(cum_weights=...), bit-exact.      */
/* ------------------------------------------------------------------ */
static uint32_t mt[624];
static int mti = 625;
static void mt_init(uint32_t s) {
  mt[0] = s;
  for (mti = 1; mti < 624; mti++)
    mt[mti] = 1812433253U * (mt[mti - 1] ^ (mt[mti - 1] >> 30)) + (uint32_t)mti;
}
static void mt_init_by_array(const uint32_t* key, int klen) {
  mt_init(19650218U);
  int i = 1, j = 0;
  for (int k = (624 > klen ? 624 : klen); k; k--) {
    mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525U)) + key[j] + (uint32_t)j;
    i++; j++;
    if (i >= 624) { mt[0] = mt[623]; i = 1; }
    if (j >= klen) j = 0;
  }
  for (int k = 623; k; k--) {
    mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941U)) - (uint32_t)i;
    i++;
    if (i >= 624) { mt[0] = mt[623]; i = 1; }
  }
  mt[0] = 0x80000000U;
}
static uint32_t mt_next(void) {
  static const uint32_t mag01[2] = {0x0U, 0x9908b0dfU};
  uint32_t y;
  if (mti >= 624) {
    int kk;
    for (kk = 0; kk < 624 - 397; kk++) {
      y = (mt[kk] & 0x80000000U) | (mt[kk + 1] & 0x7fffffffU);
      mt[kk] = mt[kk + 397] ^ (y >> 1) ^ mag01[y & 1U];
    }
    for (; kk < 623; kk++) {
      y = (mt[kk] & 0x80000000U) | (mt[kk + 1] & 0x7fffffffU);
      mt[kk] = mt[kk + (397 - 624)] ^ (y >> 1) ^ mag01[y & 1U];
    }
    y = (mt[623] & 0x80000000U) | (mt[0] & 0x7fffffffU);
    mt[623] = mt[396] ^ (y >> 1) ^ mag01[y & 1U];
    mti = 0;
  }
  y = mt[mti++];
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680U;
  y ^= (y << 15) & 0xefc60000U;
  y ^= (y >> 18);
  return y;
}
static double py_random(void) { /* random_random in _randommodule.c */
  uint32_t a = mt_next() >> 5, b = mt_next() >> 6;
  return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
}
/* bisect_right(cum, x, 0, hi) */
static uint32_t bisect_right(const double* cum, double x, uint32_t hi) {
  uint32_t lo = 0;
  while (lo < hi) {
    uint32_t mid = (lo + hi) / 2;
    if (x < cum[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}
/* bisect_right(cum, x, 0, n-1) through a guide table: guide[b] =
   bisect_right(cum, b*total/G), so the answer for x in bucket b lies in
   [guide[b], guide[b+1]]; one bucket of slack on each side absorbs the
   rounding of x*G/total, and the final bisection compares against cum
   itself, so the result is exactly the full bisection's. */
typedef struct {
  const double* cum;
  uint32_t n, G;
  double scale; /* G / total */
  uint32_t* guide;  /* G + 1 entries */
} Guide;
static Guide guide_build(const double* cum, uint32_t n, uint32_t G) {
  Guide g = {cum, n, G, (double)G / cum[n - 1], xmalloc(sizeof(uint32_t) * ((size_t)G + 1))};
  const double total = cum[n - 1];
  uint32_t j = 0;
  for (uint32_t b = 0; b <= G; b++) {
    const double edge = total * ((double)b / (double)G);
    while (j < n - 1 && !(edge < cum[j])) j++;
    g.guide[b] = j;
  }
  return g;
}
static uint32_t guide_find(const Guide* g, double x) {
  double fb = x * g->scale;
  uint32_t b = fb <= 0.0 ? 0 : (fb >= (double)g->G ? g->G : (uint32_t)fb);
  uint32_t lo = g->guide[b > 0 ? b - 1 : 0];
  uint32_t hi = g->guide[b + 2 <= g->G ? b + 2 : g->G];
  if (hi > g->n - 1) hi = g->n - 1;
  while (lo < hi) {
    uint32_t mid = (lo + hi) / 2;
    if (x < g->cum[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}
static double* cumulative_weights(uint32_t n, double exponent) { /* generate.py:35-41 */
  double* cum = xmalloc(sizeof(double) * n);
  double acc = 0.0;
  for (uint32_t i = 1; i <= n; i++) { acc += pow((double)i, -exponent); cum[i - 1] = acc; }
  return cum;
}

static void gen_powerlaw(uint64_t triples, uint32_t predicates, double zipf, uint64_t seed,
                         uint64_t nodes_opt, double node_skew) {
  uint64_t nodes = nodes_opt ? nodes_opt : (triples / 4 > 4 ? triples / 4 : 4);
  if (nodes >= UINT32_MAX) die("too many nodes for 32-bit ids");
  uint32_t key[2];
  int klen;
  key[0] = (uint32_t)seed;
  key[1] = (uint32_t)(seed >> 32);
  klen = key[1] ? 2 : 1; /* CPython random_seed: abs(n) as little-endian u32 words */
  mt_init_by_array(key, klen);
  double* pcum = cumulative_weights(predicates, zipf);
  double* ncum = cumulative_weights((uint32_t)nodes, node_skew);
  double ptotal = pcum[predicates - 1] + 0.0, ntotal = ncum[nodes - 1] + 0.0;
  Guide ng = guide_build(ncum, (uint32_t)nodes, nodes > (1u << 24) ? (1u << 24) : (uint32_t)nodes);
  /* node/pred ids in first-occurrence order without string hashing: the terms
     are "n<k>" / "p<k>", so a direct k -> id table is an exact dictionary. */
  uint32_t* nid = calloc(nodes + 1, sizeof(uint32_t));
  uint32_t* pid = calloc((size_t)predicates + 1, sizeof(uint32_t));
  uint32_t* norder = xmalloc(sizeof(uint32_t) * (nodes + 1));
  uint32_t* porder = xmalloc(sizeof(uint32_t) * ((size_t)predicates + 1));
  uint32_t nn = 0, pn = 0;
  uint32_t *bp = xmalloc(4 * 10000), *bs = xmalloc(4 * 10000), *bo = xmalloc(4 * 10000);
  uint64_t remaining = triples;
  while (remaining > 0) {
    uint32_t k = remaining < 10000 ? (uint32_t)remaining : 10000;
    for (uint32_t i = 0; i < k; i++) bp[i] = 1 + bisect_right(pcum, py_random() * ptotal, predicates - 1);
    for (uint32_t i = 0; i < k; i++) bs[i] = 1 + guide_find(&ng, py_random() * ntotal);
    for (uint32_t i = 0; i < k; i++) bo[i] = 1 + guide_find(&ng, py_random() * ntotal);
    for (uint32_t i = 0; i < k; i++) {
      uint32_t s = bs[i], p = bp[i], o = bo[i];
      if (!nid[s]) { nid[s] = ++nn; norder[nn] = s; }
      if (!pid[p]) { pid[p] = ++pn; porder[pn] = p; }
      if (!nid[o]) { nid[o] = ++nn; norder[nn] = o; }
      tr_push(nid[s], pid[p], nid[o]);
      if (g_nt) fprintf(g_nt, "<n%u> <p%u> <n%u> .\n", s, p, o);
    }
    remaining -= k;
  }
  /* materialise the dictionaries in id order */
  char buf[32];
  for (uint32_t i = 1; i <= nn; i++) {
    int l = snprintf(buf, sizeof buf, "n%u", norder[i]);
    dict_encode(&g_nodes, buf, (size_t)l);
  }
  for (uint32_t i = 1; i <= pn; i++) {
    int l = snprintf(buf, sizeof buf, "p%u", porder[i]);
    dict_encode(&g_preds, buf, (size_t)l);
  }
  free(ng.guide);
  free(pcum); free(ncum); free(nid); free(pid); free(norder); free(porder);
  free(bp); free(bs); free(bo);
}

/* ------------------------------------------------------------------ */
static void usage(void) {
  fprintf(stderr,
          "usage:\n"
          "  gsmgen lubm --univ U [--seed S] [--pool P] --out DIR [--nt FILE]\n"
          "  gsmgen watdiv --scale F [--seed S] --out DIR [--nt FILE]\n"
          "  gsmgen powerlaw --triples T --predicates P [--zipf Z] [--seed S]\n"
          "                  [--nodes N] [--node-skew X] --out DIR [--nt FILE]\n");
  exit(1);
}

int main(int argc, char** argv) {
  if (argc < 2) usage();
  const char* mode = argv[1];
  const char *out = NULL, *nt = NULL;
  long long univ = 1, seed = 0, pool = 0, triples = 0, predicates = 0, nodes = 0, scale = 1;
  double zipf = 1.0, node_skew = 0.5;
  for (int i = 2; i < argc; i++) {
    const char* a = argv[i];
    if (i + 1 >= argc) usage();
    const char* v = argv[++i];
    if (!strcmp(a, "--out")) out = v;
    else if (!strcmp(a, "--nt")) nt = v;
    else if (!strcmp(a, "--univ")) univ = atoll(v);
    else if (!strcmp(a, "--scale")) scale = atoll(v);
    else if (!strcmp(a, "--seed")) seed = atoll(v);
    else if (!strcmp(a, "--pool")) pool = atoll(v);
    else if (!strcmp(a, "--triples")) triples = atoll(v);
    else if (!strcmp(a, "--predicates")) predicates = atoll(v);
    else if (!strcmp(a, "--nodes")) nodes = atoll(v);
    else if (!strcmp(a, "--zipf")) zipf = atof(v);
    else if (!strcmp(a, "--node-skew")) node_skew = atof(v);
    else usage();
  }
  if (!out) usage();
  if (nt) {
    g_nt = fopen(nt, "wb");
    if (!g_nt) die("cannot open --nt output");
    setvbuf(g_nt, NULL, _IOFBF, 1 << 22);
  }
  dict_init(&g_nodes, 1 << 20);
  dict_init(&g_preds, 1 << 10);
  if (!strcmp(mode, "lubm")) {
    if (univ < 1) die("--univ must be >= 1");
    g_rng = (uint64_t)seed * 0x2545F4914F6CDD1DULL + 0x1234567ULL;
    if (pool <= 0) pool = univ > 1000 ? univ : 1000;
    gen_lubm((int)univ, (int)pool);
  } else if (!strcmp(mode, "watdiv")) {
    if (scale < 1) die("--scale must be >= 1");
    g_rng = (uint64_t)seed * 0x9E3779B97F4A7C15ULL + 0xABCDEFULL;
    gen_watdiv((int)scale);
  } else if (!strcmp(mode, "powerlaw")) {
    if (triples < 1 || predicates < 1) die("--triples and --predicates must be >= 1");
    if (seed < 0) seed = -seed;
    gen_powerlaw((uint64_t)triples, (uint32_t)predicates, zipf, (uint64_t)seed, (uint64_t)nodes,
                 node_skew);
  } else {
    usage();
  }
  if (g_nt) fclose(g_nt);
  write_store(out);
  return 0;
}
