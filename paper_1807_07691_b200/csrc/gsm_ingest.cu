// gsm_ingest.cu — store build from N-Triples.
//
// Replaces `gsmat build` (cli._cmd_build, /root/reference/pkg/src/gsmat/
// cli.py:64-82): read_ntriples (qparser.py:80-111) -> TermDictionary
// first-occurrence encoding (dictionary.py:57-72) -> build_store (per
// predicate set of (s, o), sorted so/os, stats; storage.py:165-177) ->
// persist (storage.py:203-219).  The output directory is byte-identical to the
// reference's.
//
//   host   parse: the input split at line boundaries, one parser thread per
//          range (gsm_ntparse.cpp), canonical term bytes per occurrence
//   device encode (nodes, then predicates): 64-bit hash of every occurrence,
//          stable radix sort of (hash, occurrence), equal-neighbour byte check
//          (a collision re-runs with another hash seed), group heads -> the
//          first occurrence of each distinct term -> radix sort of the groups
//          by first occurrence = dense first-occurrence ids
//   device build: (p, s, o) radix-sorted (two stable passes), adjacent
//          duplicates dropped, per-predicate runs; again as (p, o, s); run
//          heads give distinct subjects / objects
//   host   persist: nodes.dict / preds.dict (escape_term, in slices on the
//          parse threads), meta, stats.tsv, p<ID>.so / p<ID>.os (u64 LE
//          pairs); every file written by its own thread
#include <cub/cub.cuh>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "gsm_internal.cuh"
#include "gsm_ntparse.h"

namespace gsm {
namespace {

__device__ __forceinline__ u64 mix64(u64 x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

// Hash of every occurrence's bytes (8-byte words, seeded).
__global__ void k_term_hash(const unsigned char* __restrict__ bytes, const u64* __restrict__ off,
                            const u32* __restrict__ len, u64 n, u64 seed, u64* __restrict__ h,
                            u32* __restrict__ idx) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned char* p = bytes + off[i];
    const u32 l = len[i];
    u64 x = seed ^ (0x9e3779b97f4a7c15ull * (u64)(l + 1));
    u32 k = 0;
    for (; k + 8 <= l; k += 8) {
      u64 w = 0;
      for (int b = 0; b < 8; b++) w |= (u64)p[k + b] << (8 * b);
      x = mix64(x ^ w) + 0x632be59bd9b4e019ull;
    }
    u64 w = 0;
    for (int b = 0; k + b < l; b++) w |= (u64)p[k + b] << (8 * b);
    h[i] = mix64(x ^ w ^ 0x94d049bb133111ebull);
    idx[i] = (u32)i;
  }
}

// Group heads of the sorted hashes; neighbours with equal hash must hold
// equal bytes (else: collision flag).
__global__ void k_term_heads(const u64* __restrict__ h, const u32* __restrict__ idx,
                             const unsigned char* __restrict__ bytes, const u64* __restrict__ off,
                             const u32* __restrict__ len, u64 n, u32* __restrict__ head,
                             u32* __restrict__ collision) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool hd = i == 0 || h[i] != h[i - 1];
    head[i] = hd;
    if (!hd) {
      const u32 a = idx[i - 1], b = idx[i];
      bool eq = len[a] == len[b];
      for (u32 k = 0; eq && k < len[a]; k++) eq = bytes[off[a] + k] == bytes[off[b] + k];
      if (!eq) atomicExch(collision, 1u);
    }
  }
}

// For each group: its first occurrence (stable sort: the group's first element).
__global__ void k_group_first(const u32* __restrict__ head, const u32* __restrict__ gid_incl,
                              const u32* __restrict__ idx, u64 n, u32* __restrict__ first,
                              u32* __restrict__ gkey) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    if (head[i]) {
      const u32 g = gid_incl[i] - 1;
      first[g] = idx[i];
      gkey[g] = g;
    }
}

__global__ void k_rank(const u32* __restrict__ gsorted, u64 G, u32* __restrict__ rank) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < G; r += stride) rank[gsorted[r]] = (u32)r + 1;
}

__global__ void k_assign_ids(const u32* __restrict__ idx, const u32* __restrict__ gid_incl,
                             const u32* __restrict__ rank, u64 n, u32* __restrict__ ids) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    ids[idx[i]] = rank[gid_incl[i] - 1];
}

// keep[i] = (p, key) differs from its predecessor (adjacent duplicates go)
__global__ void k_dedup_flags(const u32* __restrict__ p, const u64* __restrict__ k, u64 n,
                              unsigned char* __restrict__ keep) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    keep[i] = i == 0 || p[i] != p[i - 1] || k[i] != k[i - 1];
}

// Pair file images (u64 LE (key, value) per pair) and per-predicate counters:
// rows[p] += 1, heads[p] += first pair of its key run.  Sorted by p, a warp
// mostly holds one predicate: one aggregated atomic per (warp, predicate).
__global__ void k_pairs_out(const u32* __restrict__ p, const u64* __restrict__ k, u64 n,
                            u64* __restrict__ pairs, unsigned long long* __restrict__ rows,
                            unsigned long long* __restrict__ heads) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (u64 base = (u64)blockIdx.x * blockDim.x; base < n; base += stride) {
    const u64 i = base + threadIdx.x;
    const bool live = i < n;
    u32 pid = 0xFFFFFFFFu;
    bool head = false;
    if (live) {
      const u64 key = k[i] >> 32, val = k[i] & 0xffffffffull;
      pairs[2 * i] = key;
      pairs[2 * i + 1] = val;
      pid = p[i];
      head = i == 0 || p[i - 1] != pid || (k[i - 1] >> 32) != key;
    }
    const u32 same = __match_any_sync(0xffffffffu, pid);
    const u32 hm = __ballot_sync(0xffffffffu, head) & same;
    if (live && lane == __ffs(same) - 1) {
      atomicAdd(rows + pid, (unsigned long long)__popc(same));
      if (hm) atomicAdd(heads + pid, (unsigned long long)__popc(hm));
    }
  }
}

int gridn(u64 n) { return (int)std::max<u64>(1, std::min<u64>((n + 255) / 256, 148 * 32)); }

int bits_for(u64 maxv) {
  int b = 1;
  while (b < 64 && (maxv >> b)) b++;
  return b;
}

// Stream-ordered temporaries from the device's default memory pool, which
// keeps freed blocks (release threshold raised once): a build allocates and
// frees ~40 multi-MB buffers, which plain cudaMalloc / cudaFree (a device
// synchronisation each) made a visible part of the encode and sort phases.
void keep_pool(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done[device] = true;
}
struct DevBuf {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit DevBuf(cudaStream_t s) : st(s) {}
  ~DevBuf() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <class T>
  cudaError_t alloc(T** p, size_t count) {
    cudaError_t e = cudaMallocAsync((void**)p, std::max<size_t>(count * sizeof(T), 16), st);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
};

#define IG_CUDA(x)                                          \
  do {                                                      \
    cudaError_t e_ = (x);                                   \
    if (e_ != cudaSuccess) return cuda_error(e_, #x);       \
  } while (0)

// First-occurrence dense ids (1-based) of n occurrences whose canonical bytes
// are bytes[off[i], off[i] + len[i]).  first_occ[id - 1] = the occurrence
// that introduced the term.
// Host vectors the device overwrites whole: not zero-filled first.
template <class T>
using hvec = std::vector<T, uninit_alloc<T>>;

// d_ids_out != nullptr: the ids are copied there (device) instead of to `ids`.
template <class VOff, class VLen, class VIds>
gsm_status encode_terms(const unsigned char* d_bytes, const VOff& off, const VLen& len, cudaStream_t st,
                        VIds& ids, VIds& first_occ, u32* d_ids_out = nullptr) {
  const u64 n = off.size();
  ids.resize(d_ids_out ? 0 : n);
  first_occ.clear();
  if (n == 0) return GSM_OK;
  if (n >= 0xFFFFFFFFull) return set_error(GSM_ERR_VALUE, "more than 2^32 term occurrences");
  DevBuf b(st);
  u64 *d_off, *d_h, *d_h2;
  u32 *d_len, *d_idx, *d_idx2, *d_head, *d_gid, *d_coll, *d_first, *d_gkey, *d_first2, *d_gkey2, *d_rank, *d_ids;
  IG_CUDA(b.alloc(&d_off, n));
  IG_CUDA(b.alloc(&d_len, n));
  IG_CUDA(b.alloc(&d_h, n));
  IG_CUDA(b.alloc(&d_h2, n));
  IG_CUDA(b.alloc(&d_idx, n));
  IG_CUDA(b.alloc(&d_idx2, n));
  IG_CUDA(b.alloc(&d_head, n));
  IG_CUDA(b.alloc(&d_gid, n));
  IG_CUDA(b.alloc(&d_coll, 1));
  IG_CUDA(b.alloc(&d_ids, n));
  IG_CUDA(cudaMemcpyAsync(d_off, off.data(), 8 * n, cudaMemcpyHostToDevice, st));
  IG_CUDA(cudaMemcpyAsync(d_len, len.data(), 4 * n, cudaMemcpyHostToDevice, st));
  size_t tb = 0, tb2 = 0, tb3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, d_h, d_h2, d_idx, d_idx2, (int64_t)n, 0, 64, st);
  cub::DeviceScan::InclusiveSum(nullptr, tb2, d_head, d_gid, (int64_t)n, st);
  void* tmp;
  IG_CUDA(b.alloc((char**)&tmp, std::max(tb, tb2)));
  u64 G = 0;
  for (int attempt = 0;; attempt++) {
    if (attempt == 4) return set_error(GSM_ERR_VALUE, "term hash collisions persisted over 4 seeds");
    const u64 seed = 0x243f6a8885a308d3ull * (u64)(attempt + 1);
    k_term_hash<<<gridn(n), 256, 0, st>>>(d_bytes, d_off, d_len, n, seed, d_h, d_idx);
    cub::DeviceRadixSort::SortPairs(tmp, tb, d_h, d_h2, d_idx, d_idx2, (int64_t)n, 0, 64, st);
    IG_CUDA(cudaMemsetAsync(d_coll, 0, 4, st));
    k_term_heads<<<gridn(n), 256, 0, st>>>(d_h2, d_idx2, d_bytes, d_off, d_len, n, d_head, d_coll);
    cub::DeviceScan::InclusiveSum(tmp, tb2, d_head, d_gid, (int64_t)n, st);
    count_launch(4);
    u32 coll = 0, g32 = 0;
    IG_CUDA(cudaMemcpyAsync(&coll, d_coll, 4, cudaMemcpyDeviceToHost, st));
    IG_CUDA(cudaMemcpyAsync(&g32, d_gid + n - 1, 4, cudaMemcpyDeviceToHost, st));
    IG_CUDA(cudaStreamSynchronize(st));
    if (!coll) {
      G = g32;
      break;
    }
  }
  IG_CUDA(b.alloc(&d_first, G));
  IG_CUDA(b.alloc(&d_gkey, G));
  IG_CUDA(b.alloc(&d_first2, G));
  IG_CUDA(b.alloc(&d_gkey2, G));
  IG_CUDA(b.alloc(&d_rank, G));
  k_group_first<<<gridn(n), 256, 0, st>>>(d_head, d_gid, d_idx2, n, d_first, d_gkey);
  cub::DeviceRadixSort::SortPairs(nullptr, tb3, d_first, d_first2, d_gkey, d_gkey2, (int64_t)G, 0,
                                  bits_for(n), st);
  void* tmp3;
  IG_CUDA(b.alloc((char**)&tmp3, tb3));
  cub::DeviceRadixSort::SortPairs(tmp3, tb3, d_first, d_first2, d_gkey, d_gkey2, (int64_t)G, 0,
                                  bits_for(n), st);
  k_rank<<<gridn(G), 256, 0, st>>>(d_gkey2, G, d_rank);
  k_assign_ids<<<gridn(n), 256, 0, st>>>(d_idx2, d_gid, d_rank, n, d_ids);
  count_launch(4);
  first_occ.resize(G);
  IG_CUDA(cudaMemcpyAsync(first_occ.data(), d_first2, 4 * G, cudaMemcpyDeviceToHost, st));
  if (d_ids_out) IG_CUDA(cudaMemcpyAsync(d_ids_out, d_ids, 4 * n, cudaMemcpyDeviceToDevice, st));
  else IG_CUDA(cudaMemcpyAsync(ids.data(), d_ids, 4 * n, cudaMemcpyDeviceToHost, st));
  IG_CUDA(cudaStreamSynchronize(st));
  return GSM_OK;
}

// Sort keys of both orientations from the interleaved (s, o) node ids.
__global__ void k_pair_keys(const u32* __restrict__ ids, u64 T, u64* __restrict__ kso, u64* __restrict__ kos) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += stride) {
    const u64 sv = ids[2 * t], ov = ids[2 * t + 1];
    kso[t] = (sv << 32) | ov;
    kos[t] = (ov << 32) | sv;
  }
}

// One orientation: sort (p, key<<32|val) with two stable radix passes, drop
// adjacent duplicates, write the pair images and per-predicate counters.
// d_key_src / d_pid_src != nullptr: T keys / pids already on the device
// (key / pid are then not read).
template <class VKey, class VPid, class VPairs>
gsm_status build_orientation(const VKey& key, const VPid& pid, u32 max_pid, cudaStream_t st, VPairs& pairs,
                             std::vector<u64>& rows, std::vector<u64>& heads,
                             const u64* d_key_src = nullptr, const u32* d_pid_src = nullptr, u64 T_dev = 0) {
  const u64 T = d_key_src ? T_dev : key.size();
  rows.assign((size_t)max_pid + 1, 0);
  heads.assign((size_t)max_pid + 1, 0);
  pairs.clear();
  if (T == 0) return GSM_OK;
  DevBuf b(st);
  u64 *d_k, *d_k2, *d_k3, *d_pairs;
  u32 *d_p, *d_p2, *d_p3;
  unsigned char* d_keep;
  unsigned long long *d_rows, *d_heads;
  int* d_nsel;
  IG_CUDA(b.alloc(&d_k, T));
  IG_CUDA(b.alloc(&d_k2, T));
  IG_CUDA(b.alloc(&d_p, T));
  IG_CUDA(b.alloc(&d_p2, T));
  IG_CUDA(b.alloc(&d_keep, T));
  IG_CUDA(b.alloc(&d_nsel, 1));
  if (d_key_src) {
    IG_CUDA(cudaMemcpyAsync(d_k, d_key_src, 8 * T, cudaMemcpyDeviceToDevice, st));
    IG_CUDA(cudaMemcpyAsync(d_p, d_pid_src, 4 * T, cudaMemcpyDeviceToDevice, st));
  } else {
    IG_CUDA(cudaMemcpyAsync(d_k, key.data(), 8 * T, cudaMemcpyHostToDevice, st));
    IG_CUDA(cudaMemcpyAsync(d_p, pid.data(), 4 * T, cudaMemcpyHostToDevice, st));
  }
  // (key) then stable by p  ->  sorted by (p, key)
  size_t t1 = 0, t2 = 0, t3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, d_k, d_k2, d_p, d_p2, (int64_t)T, 0, 64, st);
  cub::DeviceRadixSort::SortPairs(nullptr, t2, d_p2, d_p, d_k2, d_k, (int64_t)T, 0, bits_for(max_pid), st);
  void* tmp;
  IG_CUDA(b.alloc((char**)&tmp, std::max(t1, t2)));
  cub::DeviceRadixSort::SortPairs(tmp, t1, d_k, d_k2, d_p, d_p2, (int64_t)T, 0, 64, st);
  cub::DeviceRadixSort::SortPairs(tmp, t2, d_p2, d_p, d_k2, d_k, (int64_t)T, 0, bits_for(max_pid), st);
  k_dedup_flags<<<gridn(T), 256, 0, st>>>(d_p, d_k, T, d_keep);
  IG_CUDA(b.alloc(&d_k3, T));
  IG_CUDA(b.alloc(&d_p3, T));
  cub::DeviceSelect::Flagged(nullptr, t3, d_k, d_keep, d_k3, d_nsel, (int64_t)T, st);
  void* tmp3;
  IG_CUDA(b.alloc((char**)&tmp3, t3));
  cub::DeviceSelect::Flagged(tmp3, t3, d_k, d_keep, d_k3, d_nsel, (int64_t)T, st);
  cub::DeviceSelect::Flagged(tmp3, t3, d_p, d_keep, d_p3, d_nsel, (int64_t)T, st);
  count_launch(5);
  int U = 0;
  IG_CUDA(cudaMemcpyAsync(&U, d_nsel, 4, cudaMemcpyDeviceToHost, st));
  IG_CUDA(cudaStreamSynchronize(st));
  IG_CUDA(b.alloc(&d_pairs, 2 * (size_t)U));
  IG_CUDA(b.alloc(&d_rows, (size_t)max_pid + 1));
  IG_CUDA(b.alloc(&d_heads, (size_t)max_pid + 1));
  IG_CUDA(cudaMemsetAsync(d_rows, 0, 8 * ((size_t)max_pid + 1), st));
  IG_CUDA(cudaMemsetAsync(d_heads, 0, 8 * ((size_t)max_pid + 1), st));
  k_pairs_out<<<gridn(U), 256, 0, st>>>(d_p3, d_k3, (u64)U, d_pairs, d_rows, d_heads);
  count_launch();
  pairs.resize(2 * (size_t)U);
  IG_CUDA(cudaMemcpyAsync(pairs.data(), d_pairs, 16 * (size_t)U, cudaMemcpyDeviceToHost, st));
  IG_CUDA(cudaMemcpyAsync(rows.data(), d_rows, 8 * ((size_t)max_pid + 1), cudaMemcpyDeviceToHost, st));
  IG_CUDA(cudaMemcpyAsync(heads.data(), d_heads, 8 * ((size_t)max_pid + 1), cudaMemcpyDeviceToHost, st));
  IG_CUDA(cudaStreamSynchronize(st));
  return GSM_OK;
}

// dictionary.escape_term (dictionary.py:18-25)
void escape_term(std::string& out, const char* p, u32 n) {
  u32 plain = 0;  // leading run without '\\', '\n', '\r', '\t': appended at once
  while (plain < n && p[plain] != '\\' && p[plain] != '\n' && p[plain] != '\r' && p[plain] != '\t') plain++;
  out.append(p, plain);
  for (u32 i = plain; i < n; i++) {
    const char c = p[i];
    if (c == '\\') out += "\\\\";
    else if (c == '\n') out += "\\n";
    else if (c == '\r') out += "\\r";
    else if (c == '\t') out += "\\t";
    else out += c;
  }
}

// Parse the whole input with `threads` host threads.
gsm_status parse_all(const char* buf, size_t n, int threads, std::vector<nt::Chunk>& chunks) {
  std::vector<size_t> bounds;
  std::vector<int64_t> first;
  nt::split_lines(buf, n, std::max(1, threads), bounds, first);
  chunks.assign(bounds.size() - 1, nt::Chunk());
  std::vector<std::thread> th;
  for (size_t r = 0; r + 1 < bounds.size(); r++)
    th.emplace_back([&, r] { nt::parse_range(buf, bounds[r], bounds[r + 1], first[r], chunks[r]); });
  for (auto& t : th) t.join();
  for (auto& c : chunks)
    if (c.err_line >= 0) {  // chunks are in input order: the first error is the reference's
      if (c.err_msg.rfind("invalid UTF-8", 0) == 0)
        return set_error(GSM_ERR_VALUE, "line " + std::to_string(c.err_line) + ": " + c.err_msg);
      return set_error(GSM_ERR_PARSE, "line " + std::to_string(c.err_line) + ": " + c.err_msg);
    }
  return GSM_OK;
}

}  // namespace
}  // namespace gsm

using namespace gsm;

extern "C" {

gsm_status gsm_ntriples_parse(const char* buf, int64_t nbytes, int32_t threads, gsm_text** out) {
  *out = nullptr;
  if (nbytes < 0 || (nbytes > 0 && !buf)) return set_error(GSM_ERR_VALUE, "bad arguments");
  std::vector<nt::Chunk> chunks;
  gsm_status st = parse_all(buf, (size_t)nbytes, threads, chunks);
  if (st != GSM_OK) return st;
  gsm_text* t = new gsm_text();
  for (auto& c : chunks)
    for (size_t i = 0; i < c.s.size(); i++)
      for (const nt::Term* term : {&c.s[i], &c.p[i], &c.o[i]}) {
        const u32 l = term->len;
        t->bytes.insert(t->bytes.end(), reinterpret_cast<const char*>(&l), reinterpret_cast<const char*>(&l) + 4);
        t->bytes.insert(t->bytes.end(), c.bytes.data() + term->off, c.bytes.data() + term->off + l);
      }
  *out = t;
  return GSM_OK;
}

// storage.build_store's partition / deduplicate / sort (storage.py:165-177)
// for already encoded triples: the (p, s, o) and (p, o, s) orders on the
// device.  so_pairs / os_pairs receive the pair-file images (u64 LE (key,
// value) pairs) of all predicates in pid order; counts[3 * pid + {0, 1, 2}]
// = (pairs, distinct subjects, distinct objects) for pid in [0, max_pid].
gsm_status gsm_sort_triples(int32_t device, const uint32_t* s, const uint32_t* p, const uint32_t* o,
                            int64_t n, int32_t max_pid, gsm_text** so_pairs, gsm_text** os_pairs,
                            int64_t* counts) {
  *so_pairs = *os_pairs = nullptr;
  if (n < 0 || max_pid < 0 || (n > 0 && (!s || !p || !o)) || !counts)
    return set_error(GSM_ERR_VALUE, "bad arguments");
  for (int64_t i = 0; i < n; i++)
    if ((int64_t)p[i] > max_pid) return set_error(GSM_ERR_VALUE, "predicate id above max_pid");
  GSM_CUDA(cudaSetDevice(device));
  cudaStream_t cs;
  GSM_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{cs};
  std::vector<u64> kso((size_t)n), kos((size_t)n);
  std::vector<u32> pid(p, p + n);
  for (int64_t i = 0; i < n; i++) {
    kso[(size_t)i] = ((u64)s[i] << 32) | o[i];
    kos[(size_t)i] = ((u64)o[i] << 32) | s[i];
  }
  std::vector<u64> sp, op, so_rows, so_heads, os_rows, os_heads;
  gsm_status st = build_orientation(kso, pid, (u32)max_pid, cs, sp, so_rows, so_heads);
  if (st != GSM_OK) return st;
  if ((st = build_orientation(kos, pid, (u32)max_pid, cs, op, os_rows, os_heads)) != GSM_OK) return st;
  gsm_text* a = new gsm_text();
  gsm_text* b = new gsm_text();
  a->bytes.assign(reinterpret_cast<const char*>(sp.data()), reinterpret_cast<const char*>(sp.data() + sp.size()));
  b->bytes.assign(reinterpret_cast<const char*>(op.data()), reinterpret_cast<const char*>(op.data() + op.size()));
  for (int32_t q = 0; q <= max_pid; q++) {
    counts[3 * q] = q < (int32_t)so_rows.size() ? (int64_t)so_rows[q] : 0;
    counts[3 * q + 1] = q < (int32_t)so_heads.size() ? (int64_t)so_heads[q] : 0;
    counts[3 * q + 2] = q < (int32_t)os_heads.size() ? (int64_t)os_heads[q] : 0;
  }
  *so_pairs = a;
  *os_pairs = b;
  return GSM_OK;
}

gsm_status gsm_build_store(const char* nt_path, const char* out_dir, int32_t device, int32_t threads,
                           int64_t* counts) {
  if (!nt_path || !out_dir) return set_error(GSM_ERR_VALUE, "null path");
  int fd = open(nt_path, O_RDONLY);
  if (fd < 0) return set_error(GSM_ERR_VALUE, std::string("cannot open ") + nt_path);
  struct stat sb;
  fstat(fd, &sb);
  const size_t n = (size_t)sb.st_size;
  const char* buf = nullptr;
  if (n > 0) {
    void* m = mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
    if (m == MAP_FAILED) {
      close(fd);
      return set_error(GSM_ERR_VALUE, std::string("cannot map ") + nt_path);
    }
    buf = static_cast<const char*>(m);
  }
  close(fd);
  struct Unmap {
    const char* b;
    size_t n;
    ~Unmap() {
      if (b) munmap(const_cast<char*>(b), n);
    }
  } unmap{buf, n};
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  // GSM_INGEST_TIMING=1: phase times on stderr
  const bool timing = getenv("GSM_INGEST_TIMING") && getenv("GSM_INGEST_TIMING")[0] == '1';
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t_last = now();
  std::string phases;
  auto phase = [&](const char* name) {
    if (!timing) return;
    const auto t = now();
    char b[64];
    snprintf(b, sizeof b, " %s %.1f ms", name, 1e3 * std::chrono::duration<double>(t - t_last).count());
    phases += b;
    t_last = t;
  };
  struct Report {
    const bool& on;
    std::string& ph;
    ~Report() {
      if (on) fprintf(stderr, "gsm ingest phases:%s\n", ph.c_str());
    }
  } report{timing, phases};
  std::vector<nt::Chunk> chunks;
  gsm_status st = parse_all(buf, n, threads, chunks);
  phase("parse");
  if (st != GSM_OK) return st;

  // occurrences in input order: nodes s0, o0, s1, o1, ...; predicates p0, p1, ...
  u64 T = 0, nb = 0;
  for (auto& c : chunks) {
    T += c.s.size();
    nb += c.bytes.size();
  }
  // the chunks' term bytes and offsets gathered into one array, each chunk
  // by its own thread (bases from a prefix over the chunks)
  GSM_CUDA(cudaSetDevice(device));
  cudaStream_t cs;
  GSM_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{cs};
  unsigned char* d_bytes = nullptr;
  keep_pool(device);
  GSM_CUDA(cudaMallocAsync(&d_bytes, std::max<size_t>(nb, 16), cs));
  struct FreeGuard {
    void* p;
    cudaStream_t s;
    ~FreeGuard() { cudaFreeAsync(p, s); }
  } fg{d_bytes, cs};
  GSM_CUDA(cudaStreamSynchronize(cs));  // d_bytes is written from the gather threads' streams
  std::vector<char, uninit_alloc<char>> bytes(nb);
  std::vector<cudaError_t> h2d_err(chunks.size(), cudaSuccess);
  std::vector<u64, uninit_alloc<u64>> noff(2 * T), poff(T);
  std::vector<u32, uninit_alloc<u32>> nlen(2 * T), plen(T);
  {
    std::vector<u64> bbase(chunks.size() + 1, 0), tbase(chunks.size() + 1, 0);
    for (size_t k = 0; k < chunks.size(); k++) {
      bbase[k + 1] = bbase[k] + chunks[k].bytes.size();
      tbase[k + 1] = tbase[k] + chunks[k].s.size();
    }
    std::vector<std::thread> th;
    for (size_t k = 0; k < chunks.size(); k++)
      th.emplace_back([&, k] {
        nt::Chunk& c = chunks[k];
        const u64 base = bbase[k];
        if (!c.bytes.empty()) {
          // this chunk's term bytes to the device from its own thread (the
          // pageable copies' staging runs on all gather threads at once)
          cudaStream_t ts = nullptr;
          cudaError_t e = cudaSetDevice(device);
          if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking);
          if (e == cudaSuccess)
            e = cudaMemcpyAsync(d_bytes + base, c.bytes.data(), c.bytes.size(), cudaMemcpyHostToDevice, ts);
          memcpy(bytes.data() + base, c.bytes.data(), c.bytes.size());
          if (e == cudaSuccess) e = cudaStreamSynchronize(ts);
          if (ts) cudaStreamDestroy(ts);
          h2d_err[k] = e;
        }
        u64 t = tbase[k];
        for (size_t i = 0; i < c.s.size(); i++, t++) {
          noff[2 * t] = base + c.s[i].off;
          nlen[2 * t] = c.s[i].len;
          noff[2 * t + 1] = base + c.o[i].off;
          nlen[2 * t + 1] = c.o[i].len;
          poff[t] = base + c.p[i].off;
          plen[t] = c.p[i].len;
        }
        std::vector<char>().swap(c.bytes);
      });
    for (auto& x : th) x.join();
  }
  phase("gather");
  for (cudaError_t e : h2d_err) GSM_CUDA(e);
  hvec<u32> node_ids, node_first, pred_ids, pred_first;
  // node / predicate ids stay on the device: the sort keys are built there
  DevBuf keys(cs);
  u32 *d_nids, *d_pids;
  u64 *d_kso, *d_kos;
  GSM_CUDA(keys.alloc(&d_nids, 2 * T));
  GSM_CUDA(keys.alloc(&d_pids, T));
  GSM_CUDA(keys.alloc(&d_kso, T));
  GSM_CUDA(keys.alloc(&d_kos, T));
  if ((st = encode_terms(d_bytes, noff, nlen, cs, node_ids, node_first, d_nids)) != GSM_OK) return st;
  phase("encode_nodes");
  if ((st = encode_terms(d_bytes, poff, plen, cs, pred_ids, pred_first, d_pids)) != GSM_OK) return st;
  phase("encode_preds");
  const u32 n_nodes = (u32)node_first.size(), n_preds = (u32)pred_first.size();

  // triples -> sorted, deduplicated so / os pair images
  if (T > 0) {
    k_pair_keys<<<gridn(T), 256, 0, cs>>>(d_nids, T, d_kso, d_kos);
    GSM_CUDA(cudaGetLastError());
    count_launch();
  }
  const hvec<u64> no_keys;
  hvec<u64> so_pairs, os_pairs;
  std::vector<u64> so_rows, so_heads, os_rows, os_heads;
  if ((st = build_orientation(no_keys, pred_ids, n_preds, cs, so_pairs, so_rows, so_heads, d_kso, d_pids, T)) !=
      GSM_OK)
    return st;
  if ((st = build_orientation(no_keys, pred_ids, n_preds, cs, os_pairs, os_rows, os_heads, d_kos, d_pids, T)) !=
      GSM_OK)
    return st;
  phase("sort");

  // persist (storage.py:203-219): the dictionaries rendered in slices and
  // every file written on its own thread (the pair files are most of the bytes)
  const std::string dir(out_dir);
  mkdir(dir.c_str(), 0777);
  u64 triples = 0;
  for (u32 p = 1; p <= n_preds; p++) triples += so_rows[p];
  const int nslice = std::max(1, std::min(threads, 64));
  std::vector<std::string> node_txt(nslice);
  {
    std::vector<std::thread> th;
    for (int k = 0; k < nslice; k++)
      th.emplace_back([&, k] {
        const u32 r0 = (u32)((u64)n_nodes * k / nslice), r1 = (u32)((u64)n_nodes * (k + 1) / nslice);
        std::string& s = node_txt[k];
        for (u32 r = r0; r < r1; r++) {
          const u64 occ = node_first[r];
          escape_term(s, bytes.data() + noff[occ], nlen[occ]);
          s += '\n';
        }
      });
    for (auto& x : th) x.join();
  }
  std::string pred_txt;
  for (u32 r = 0; r < n_preds; r++) {
    const u64 occ = pred_first[r];
    escape_term(pred_txt, bytes.data() + poff[occ], plen[occ]);
    pred_txt += '\n';
  }
  std::string meta = "GSMAT1\n" + std::to_string(triples) + "\n" + std::to_string(n_preds) + "\n" +
                     std::to_string(n_nodes) + "\n";
  std::string stats;
  for (u32 p = 1; p <= n_preds; p++)
    stats += std::to_string(p) + "\t" + std::to_string(so_rows[p]) + "\t" + std::to_string(so_heads[p]) + "\t" +
             std::to_string(os_heads[p]) + "\n";
  // jobs: (path, pieces); a file's pieces are written in order
  struct Job {
    std::string path;
    std::vector<std::pair<const void*, size_t>> pieces;
  };
  std::vector<Job> jobs;
  {
    Job nd{dir + "/nodes.dict", {}};
    for (auto& t : node_txt) nd.pieces.emplace_back(t.data(), t.size());
    jobs.push_back(std::move(nd));
    jobs.push_back(Job{dir + "/preds.dict", {{pred_txt.data(), pred_txt.size()}}});
    jobs.push_back(Job{dir + "/meta", {{meta.data(), meta.size()}}});
    jobs.push_back(Job{dir + "/stats.tsv", {{stats.data(), stats.size()}}});
    u64 at_so = 0, at_os = 0;
    for (u32 p = 1; p <= n_preds; p++) {
      const std::string base = dir + "/p" + std::to_string(p);
      jobs.push_back(Job{base + ".so", {{so_pairs.data() + 2 * at_so, 16 * so_rows[p]}}});
      jobs.push_back(Job{base + ".os", {{os_pairs.data() + 2 * at_os, 16 * os_rows[p]}}});
      at_so += so_rows[p];
      at_os += os_rows[p];
    }
  }
  std::atomic<size_t> next{0};
  std::atomic<int> failed{-1};
  {
    std::vector<std::thread> th;
    for (int k = 0; k < std::max(1, std::min(threads, (int)jobs.size())); k++)
      th.emplace_back([&] {
        for (size_t j; (j = next.fetch_add(1)) < jobs.size();) {
          FILE* f = fopen(jobs[j].path.c_str(), "wb");
          bool ok = f != nullptr;
          for (auto& pc : jobs[j].pieces)
            ok = ok && (pc.second == 0 || fwrite(pc.first, 1, pc.second, f) == pc.second);
          if (f) ok = fclose(f) == 0 && ok;
          if (!ok) {
            int expect = -1;
            failed.compare_exchange_strong(expect, (int)j);
          }
        }
      });
    for (auto& x : th) x.join();
  }
  if (failed.load() >= 0) {
    const std::string& path = jobs[(size_t)failed.load()].path;
    const std::string nm = path.substr(path.rfind('/') + 1);
    if (nm == "nodes.dict" || nm == "preds.dict" || nm == "meta" || nm == "stats.tsv")
      return set_error(GSM_ERR_VALUE, "cannot write " + nm);
    return set_error(GSM_ERR_VALUE, "cannot write pair files");
  }
  phase("persist");
  if (counts) {
    counts[0] = (int64_t)triples;
    counts[1] = n_preds;
    counts[2] = n_nodes;
  }
  return GSM_OK;
}

}  // extern "C"
