/*
 * gsmat_b200.h — C ABI of the B200-native gSMat join executor.
 *
 * The reference (arXiv 1807.07691's `gsmat` package, /root/reference/pkg) is
 * pure Python and has no FFI; its seam for this path is the Python function
 *
 *     executor.execute(query, plan, store, mode="sequential", worker_count=1,
 *                      row_budget=10**8, report=None) -> BindingTable
 *     (/root/reference/pkg/src/gsmat/executor.py:296-304)
 *
 * over a loaded store (storage.load, storage.py:222-271).  The entry points
 * below are exactly what a binding of that seam needs (the ctypes binding the
 * package ships is paper_1807_07691_b200/_lib.py; a cgo/N-API stub is shown in
 * INTEGRATION.md).  Plain pointers and sizes only; no torch or CUDA types.
 *
 * Conventions
 *   - Every function returns a gsm_status; 0 is success.  On failure
 *     gsm_last_error() returns a thread-local message.  Status codes map to
 *     the reference's exception classes (errors.py:4-53): see gsm_status.
 *   - Node ids are the reference dictionary's dense 1-based ids
 *     (dictionary.py:57-72); 0 is the "unknown constant" sentinel
 *     (qparser.py:340,348).  Ids must be < 2^32.
 *   - The library owns all device memory.  A store is immutable after
 *     gsm_store_finalize and may be shared by any number of contexts; a
 *     context (stream + arena) must be used by one host thread at a time.
 */
#ifndef GSMAT_B200_H
#define GSMAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GSM_OK = 0,
  GSM_ERR_VALUE = 1,           /* ValueError: bad mode / empty plan / bad argument      */
  GSM_ERR_STORE_FORMAT = 2,    /* StoreFormatError (storage.py:193-271 checks)          */
  GSM_ERR_UNKNOWN_PREDICATE = 3, /* UnknownPredicateError (storage.py:118-122)          */
  GSM_ERR_RESOURCE = 4,        /* ResourceLimitError: row budget (executor.py:158-163,
                                  192-193, 237-241) or device memory exhausted           */
  GSM_ERR_CUDA = 5,            /* driver/runtime failure                                */
  GSM_ERR_UNSORTED = 6,        /* ValueError "pair list not sorted" (storage.py:44-45)  */
  GSM_ERR_UNKNOWN_ID = 7,      /* UnknownIdError: decode of an absent id (dictionary.py:84-87) */
  GSM_ERR_PARSE = 8,           /* ParseError "line N: ..." (qparser.py:80-92)            */
  GSM_ERR_DEVICE_MEMORY = 9    /* ResourceLimitError subclass: an intermediate table does
                                  not fit device memory even after growing the arena; the
                                  host re-runs the plan in left-row chunks (part/parts)   */
} gsm_status;

typedef struct gsm_store gsm_store;
typedef struct gsm_context gsm_context;
typedef struct gsm_result gsm_result;
typedef struct gsm_text gsm_text;

/* One triple pattern of the plan, in plan order (planner.py:73-83 PlanStep.pattern;
 * fields of qparser.EncodedPattern, qparser.py:303-323).  Variables are small
 * integers assigned by the caller (same name -> same index). */
typedef struct {
  int32_t s_var;    /* variable index >= 0, or -1 if the subject is a constant */
  int32_t o_var;    /* variable index >= 0, or -1 if the object is a constant  */
  uint32_t s_const; /* node id when s_var == -1                                */
  uint32_t o_const; /* node id when o_var == -1                                */
  int32_t pid;      /* predicate id; no matrix for pid -> the scan is empty     */
  int32_t empty;    /* EncodedPattern.empty: unknown constant -> no rows        */
} gsm_pattern;

/* Budget semantics of the reference's two modes. */
enum { GSM_BUDGET_SEQUENTIAL = 0, /* emitted rows of a join   (executor.py:192-193) */
       GSM_BUDGET_PARALLEL = 1 }; /* pre-allocated E of a join (executor.py:237-241) */

/* Per-step report (executor.py:67-91 StepReport/ExecutionReport).  Arrays of
 * length n_steps, owned by the caller; any pointer may be NULL.  The scalar
 * fields are outputs filled on success. */
typedef struct {
  int64_t* rows;           /* StepReport.rows: rows of the table after the step     */
  int64_t* prealloc_total; /* StepReport.prealloc_total: E of the join, 0 for scans
                              and cross products                                     */
  float* device_ms;        /* device time of the step (CUDA events); NULL = skip    */
  int32_t* kind;           /* GSM_STEP_* of each step                               */
  int32_t* arity;          /* columns of the table after the step                   */
  float total_device_ms;   /* out: device time of the whole query (first H2D copy
                              to the last kernel), when device_ms != NULL           */
  int64_t h2d_bytes;       /* out: host->device bytes copied for this query          */
  int64_t d2h_bytes;       /* out: device->host bytes of the query incl. result rows */
  int64_t kernels;         /* out: kernels launched for this query                   */
  int32_t* fused;          /* 1 = the step ran inside the previous step's kernel
                              (k_group): its input table was never materialised    */
} gsm_report;

/* Step kinds reported in gsm_report.kind (SURVEY.md §8 join taxonomy). */
enum {
  GSM_STEP_SCAN = 0,   /* first pattern: R1-R6 table scan                      */
  GSM_STEP_EMPTY = 1,  /* right side has no matrix / unknown constant (R6)     */
  GSM_STEP_EXPAND = 2, /* J1: one shared variable, neighbour expand            */
  GSM_STEP_FILTER = 3, /* J2/J3: all right variables bound, membership filter  */
  GSM_STEP_CROSS = 4,  /* J0: no shared variable, cross product                */
  GSM_STEP_GATE = 5    /* J0 against a zero-arity (constant-constant) pattern  */
};

/* ---- device / store -------------------------------------------------- */

/* Number of visible CUDA devices. */
gsm_status gsm_device_count(int32_t* count);

/* Replaces storage.load()'s in-memory Store (storage.py:106-112,222-271):
 * creates an empty device store on `device` for node ids 1..node_count and
 * predicate ids 1..max_pid. */
gsm_status gsm_store_create(int32_t device, int64_t node_count, int32_t max_pid,
                            gsm_store** out);

/* Replaces PredicateMatrix(pid, so, os) (storage.py:56-72, fed by
 * _pairs_from_bytes storage.py:193-200): uploads one predicate's pair arrays
 * exactly as they sit in p<ID>.so / p<ID>.os (interleaved u64 LE pairs,
 * `so` sorted by (s,o), `os` sorted by (o,s)), nnz pairs each.  The caller
 * keeps ownership of the host buffers; they may be freed on return. */
gsm_status gsm_store_put_predicate(gsm_store* store, int32_t pid, const uint64_t* so_pairs,
                                   const uint64_t* os_pairs, int64_t nnz);

/* Sharded stores (SURVEY.md §8(e) sharded mode): one shard's part of a
 * predicate — the CSR rows it owns (so pairs whose subject is in its id
 * range) and the CSC rows it owns (os pairs whose object is in its range),
 * so the two orientations hold different pair counts. */
gsm_status gsm_store_put_predicate_shard(gsm_store* store, int32_t pid, const uint64_t* so_pairs,
                                         int64_t nnz_so, const uint64_t* os_pairs, int64_t nnz_os);

/* Loader fast path for storage.load (storage.py:193-200, 222-271): streams
 * the n predicates' pair files (p<ID>.so / p<ID>.os, nnz[i] u64 LE pairs
 * each, sizes already validated by the caller) straight to the device —
 * pinned double-buffered reads overlapped with the H2D copies and the
 * narrowing kernels — with the same sortedness / id-range errors as
 * gsm_store_put_predicate.  Equivalent to n gsm_store_put_predicate calls. */
gsm_status gsm_store_load_files(gsm_store* store, int32_t n, const int32_t* pids,
                                const char* const* so_paths, const char* const* os_paths,
                                const int64_t* nnz);

/* Replaces PredicateMatrix.__post_init__ / build_aux (storage.py:38-53,66-72):
 * builds the device row indexes (aux arrays, key -> segment lookup, diagonal
 * lists) for every uploaded predicate and validates sortedness. */
gsm_status gsm_store_finalize(gsm_store* store);

/* Bytes of device memory held by the store. */
gsm_status gsm_store_device_bytes(const gsm_store* store, int64_t* bytes);

gsm_status gsm_store_free(gsm_store* store);

/* ---- execution context ------------------------------------------------ */

/* A stream plus an HBM arena for intermediate binding tables.  arena_bytes = 0
 * picks a default (grown on demand up to the free device memory). */
gsm_status gsm_context_create(gsm_store* store, int64_t arena_bytes, gsm_context** out);
gsm_status gsm_context_free(gsm_context* ctx);

/* The context's CUDA stream (cudaStream_t as an integer): every launch of
 * the context is stream-ordered on it, so a caller can enqueue its own work
 * (e.g. NCCL collectives in the sharded mode) on the same stream and skip
 * host synchronisation between the library's launches and its own. */
gsm_status gsm_context_stream(gsm_context* ctx, uint64_t* stream);

/* Largest arena (bytes) the context can grow to: 90% of the free device
 * memory plus its current arena, capped by GSM_ARENA_MAX.  An intermediate
 * table of R rows x k columns needs 8*R*k bytes of it (two halves); larger
 * plans fail with GSM_ERR_DEVICE_MEMORY and are run in left-row chunks. */
gsm_status gsm_context_capacity(gsm_context* ctx, int64_t* bytes);

/* Replaces executor.execute (executor.py:296-368) for mode="gpu":
 * evaluates `n_steps` patterns in plan order as a left-deep chain of SM-based
 * joins on the device, then projects onto `proj` (variable indices, n_proj of
 * them) and applies DISTINCT when `distinct` != 0.  Join variables, cross
 * products and output schemas follow executor.py:340-356.  A budget violation
 * returns GSM_ERR_RESOURCE with the reference's message.
 *
 * part_index/part_count partition the FIRST step's rows into part_count
 * contiguous ranges and evaluate only range part_index (multi-GPU row
 * partitioning; 0/1 = whole query).  The union over all parts of the results
 * is the bag of the whole query (before DISTINCT). */
gsm_status gsm_execute(gsm_context* ctx, const gsm_pattern* steps, int32_t n_steps,
                       const int32_t* proj, int32_t n_proj, int32_t distinct,
                       int64_t row_budget, int32_t budget_mode, int64_t part_index,
                       int64_t part_count, gsm_report* report, gsm_result** out);

/* gsm_execute that also hands the rows over: when the result (n_rows x
 * n_cols ids, always set on success) fits dst_cap ids it is copied into dst
 * and *out is NULL; otherwise *out holds it as in gsm_execute.  One call for
 * what `execute` returns (executor.py:296-368: the projected rows). */
gsm_status gsm_execute_into(gsm_context* ctx, const gsm_pattern* steps, int32_t n_steps,
                            const int32_t* proj, int32_t n_proj, int32_t distinct,
                            int64_t row_budget, int32_t budget_mode, int64_t part_index,
                            int64_t part_count, gsm_report* report, uint32_t* dst,
                            int64_t dst_cap, int64_t* n_rows, int32_t* n_cols, gsm_result** out);

/* Sharded mode, one step at a time: like gsm_execute, but
 * step 0 is the caller's binding table instead of a scan — `seed_rows` is a
 * DEVICE pointer to n_seed x seed_k row-major uint32 ids whose columns bind
 * variables seed_vars[0..seed_k) — and `steps` (n_steps patterns, possibly
 * none) are joined onto it with the same rules as executor.py:340-356.  The
 * report arrays hold n_steps + 1 entries (entry 0 = the seed).  Never cached
 * as a CUDA graph (the seed buffer changes per call). */
gsm_status gsm_execute_seeded(gsm_context* ctx, const uint32_t* seed_rows, int64_t n_seed,
                              const int32_t* seed_vars, int32_t seed_k, const gsm_pattern* steps,
                              int32_t n_steps, const int32_t* proj, int32_t n_proj,
                              int32_t distinct, int64_t row_budget, int32_t budget_mode,
                              gsm_report* report, gsm_result** out);

/* Sharded-mode exchange (the partition side of an all-to-all): groups the
 * DEVICE rows `rows` (n x k row-major uint32) by destination shard and writes
 * them to the DEVICE buffer out_rows (destination 0 first), with the number
 * of rows per destination in counts[parts] (host).  Destination = the shard
 * owning the id in column key_col (owner(id) = (id-1)*parts/node_count, the
 * subject/object id ranges a sharded store is split by), or, with key_col < 0,
 * a hash of the whole row (distributed DISTINCT).  Synchronous. */
gsm_status gsm_partition_rows(gsm_context* ctx, const uint32_t* rows, int64_t n, int32_t k,
                              int32_t key_col, int64_t node_count, int32_t parts,
                              uint32_t* out_rows, int64_t* counts);

/* Sharded-mode cross product (executor.py:155-165) on DEVICE row-major
 * tables: out[g] = left[g / n_right] ++ right[g % n_right], out holding
 * n_left * n_right rows of a + b ids (caller-allocated).  Synchronous; the
 * budget rule is the caller's (it needs the global |L|). */
gsm_status gsm_cross_rows(gsm_context* ctx, const uint32_t* left, int64_t n_left, int32_t a,
                          const uint32_t* right, int64_t n_right, int32_t b, uint32_t* out);

/* One query of a batch: the arguments of gsm_execute. */
typedef struct {
  const gsm_pattern* steps;
  int32_t n_steps;
  const int32_t* proj;
  int32_t n_proj;
  int32_t distinct;
  int64_t row_budget;
  int32_t budget_mode;
  int64_t part_index;
  int64_t part_count;
  gsm_report* report; /* may be NULL */
} gsm_query;

/* Evaluates n_queries independent queries concurrently: query i runs on
 * ctxs[i] (distinct contexts = distinct streams and arenas of the same
 * store), all launch sequences are enqueued before any is awaited, so their
 * latency-bound join kernels overlap on the GPU (the serving counterpart of
 * calling execute() in a loop).  statuses[i] (may be NULL) and outs[i]
 * receive each query's outcome; the return value is the first failure in
 * query order (GSM_OK if none), with its message in gsm_last_error().
 * device_ms (may be NULL) receives the device time from the first launch to
 * the end of the last query's launch sequence (CUDA events). */
gsm_status gsm_execute_batch(gsm_context* const* ctxs, int32_t n_queries, const gsm_query* queries,
                             gsm_status* statuses, gsm_result** outs, float* device_ms);

/* gsm_execute_batch that also hands the rows over: query i's result rows
 * (n_rows[i] x n_cols[i], always set when statuses[i] == GSM_OK) are copied
 * into dst[i] when they fit dst_cap[i] ids, as soon as query i finishes
 * (while the rest of the batch still runs), and outs[i] is then NULL;
 * otherwise outs[i] holds the result as in gsm_execute_batch.  dst / dst_cap
 * may be NULL (nothing copied).  The reference's callers get a list of
 * BindingTables; this is the one-call form of execute + rows copy. */
gsm_status gsm_execute_batch_into(gsm_context* const* ctxs, int32_t n_queries,
                                  const gsm_query* queries, gsm_status* statuses,
                                  uint32_t* const* dst, const int64_t* dst_cap, int64_t* n_rows,
                                  int32_t* n_cols, gsm_result** outs, float* device_ms);

/* Replaces executor.sm_join / parallel_sm_join / cross_product
 * (executor.py:155-280) on arbitrary binding tables (not store-backed):
 * `left` is n_left x a and `right` n_right x b row-major uint32 host arrays.
 * join_left[i] / join_right[i] are the columns of the i-th shared variable
 * in each table, in LEFT-schema order (executor.py:343); the first drives the
 * match, the others are equality checks (executor.py:140-152, 186-191);
 * n_join = 0 is the cross product.  Result rows: left row ++ the right
 * columns not in join_right, in right order (executor.py:146-148), in the
 * reference's sm_join order (left rows in order, candidates in right-table
 * order).  prealloc_total (may be NULL) receives E, the first-variable match
 * total (executor.py:197-215); row_counts (may be NULL, n_left entries)
 * receives each left row's first-variable match count N.  Budget rules and
 * messages as gsm_execute (cross product: |L|*|R|).  out = NULL is the
 * counts-only mode of preallocate() (executor.py:197-215): E and the row
 * counts are returned without materialising any candidate (device memory
 * O(|L| + |R|)).  Under the sequential rule a join whose E exceeds the
 * budget counts its emitted rows before allocating E-sized buffers, so an
 * over-budget join raises the budget error, not an allocation failure. */
gsm_status gsm_table_join(gsm_context* ctx, const uint32_t* left, int64_t n_left, int32_t a,
                          const uint32_t* right, int64_t n_right, int32_t b,
                          const int32_t* join_left, const int32_t* join_right, int32_t n_join,
                          int64_t row_budget, int32_t budget_mode, int64_t* prealloc_total,
                          int64_t* row_counts, gsm_result** out);

/* ---- results ---------------------------------------------------------- */

/* Shape of the projected result: n_rows x n_cols (BindingTable.rows). */
gsm_status gsm_result_shape(const gsm_result* res, int64_t* n_rows, int32_t* n_cols);

/* Copies the result rows, row-major uint32 ids, into host memory
 * (n_rows * n_cols * 4 bytes).  Results up to the context's staging size are
 * already in pinned host memory when gsm_execute returns (copied inside the
 * query's launch sequence); such a result must be copied before the next
 * gsm_execute on the same context (else GSM_ERR_VALUE). */
gsm_status gsm_result_copy(const gsm_result* res, uint32_t* host_rows);

/* Device pointer of the row-major result (valid until gsm_result_free, or
 * until the next gsm_execute on the context for results left in its arena
 * because no separate buffer could be allocated). */
gsm_status gsm_result_device_ptr(const gsm_result* res, uint64_t* device_ptr);

/* Order-independent multiset fingerprint of the result rows, computed on the
 * device without copying the rows to the host: out[0] = rows, out[1] = sum,
 * out[2] = xor of the per-row splitmix64 chain over the row's ids (the
 * summary a left-row-chunked evaluation reports when the whole result would
 * not fit host memory; executor.execute_summary). */
gsm_status gsm_result_fingerprint(const gsm_result* res, uint64_t* out);

gsm_status gsm_result_free(gsm_result* res);

/* Batch helpers: shapes of n results (n_rows[i], n_cols[i]), and copy of
 * result i into host_rows[i] (skipped when NULL) followed by
 * gsm_result_free of every result when free_after != 0. */
gsm_status gsm_results_shape(gsm_result* const* res, int32_t n, int64_t* n_rows, int32_t* n_cols);
gsm_status gsm_results_copy(gsm_result* const* res, int32_t n, uint32_t* const* host_rows,
                            int32_t free_after);

/* ---- diagnostics ------------------------------------------------------ */

/* Thread-local message of the last failing call (empty string if none). */
const char* gsm_last_error(void);

/* Number of kernels this library launched since load (all threads). */
int64_t gsm_kernel_launches(void);

/* ---- result decoding ------------------------- */

/* Replaces the node half of TermDictionary.load (dictionary.py:107-125) for
 * decoding: the raw nodes.dict bytes and the [start, end) byte range of every
 * line (term id i+1 = line i).  Each term is rendered on the device into its
 * N-Triples surface form (unescape_term, dictionary.py:28-43, then
 * qparser.format_term, qparser.py:71-78) and kept resident. */
gsm_status gsm_store_put_dictionary(gsm_store* store, const char* nodes_dict, int64_t nbytes,
                                    const int64_t* line_starts, const int64_t* line_ends,
                                    int64_t n_terms);

/* Replaces the CLI's row loop (cli.py:102-105: "\t".join(format_term(
 * decode_node(v)) for v in row) + newline, per row): rows is a row-major
 * n_rows x k u32 table of node ids (host or device memory).  The TSV body is
 * built on the device and returned as a host text object.  An id outside the
 * dictionary -> GSM_ERR_UNKNOWN_ID ("no node term with id V"). */
gsm_status gsm_decode_rows(gsm_store* store, const uint32_t* rows, int64_t n_rows, int32_t k,
                           gsm_text** out);
gsm_status gsm_text_data(const gsm_text* text, const char** data, int64_t* nbytes);
gsm_status gsm_text_free(gsm_text* text);

/* ---- store build from N-Triples --------------- */

/* Replaces qparser.read_ntriples (qparser.py:80-111): parses an N-Triples
 * buffer with `threads` host threads and returns the canonical (subject,
 * predicate, object) terms of every statement, in input order, as
 * [u32 length][bytes] x 3 per triple.  A malformed statement ->
 * GSM_ERR_PARSE "line N: malformed N-Triples statement: '...'" (or "bad
 * literal escape \x"), the first one in input order. */
gsm_status gsm_ntriples_parse(const char* buf, int64_t nbytes, int32_t threads, gsm_text** out);

/* Replaces `gsmat build` (cli.py:64-82: read_ntriples -> TermDictionary
 * first-occurrence ids -> build_store -> persist, storage.py:165-177,
 * 203-219): parses nt_path on the host threads, encodes the terms and sorts /
 * deduplicates the per-predicate pair lists on `device`, and writes a store
 * directory byte-identical to the reference's into out_dir (which must
 * exist).  counts (optional) = {triples, predicates, nodes}. */
gsm_status gsm_build_store(const char* nt_path, const char* out_dir, int32_t device, int32_t threads,
                           int64_t* counts);

/* Replaces storage.build_store's partition / set / sort (storage.py:165-177)
 * for encoded triples (s[i], p[i], o[i]), p[i] <= max_pid: duplicates are
 * dropped and both orders sorted on the device.  so_pairs / os_pairs get the
 * pair-file images (u64 LE pairs) of every predicate in pid order; counts
 * (3 x (max_pid + 1) entries) = per pid (pairs, distinct subjects, distinct
 * objects). */
gsm_status gsm_sort_triples(int32_t device, const uint32_t* s, const uint32_t* p, const uint32_t* o,
                            int64_t n, int32_t max_pid, gsm_text** so_pairs, gsm_text** os_pairs,
                            int64_t* counts);

#ifdef __cplusplus
}
#endif

#endif /* GSMAT_B200_H */
