// gsm_common.cuh — shared types and device helpers of the B200 gSMat executor.
//
// HBM data layout (one predicate, one orientation):
//   src[nnz]  u32  row key of every pair   (so: s, os: o)
//   dst[nnz]  u32  other endpoint          (so: o, os: s), ascending within a row
//   key -> segment index, one of
//     dense   doff[node_count + 2] u32: segment of key k is [doff[k], doff[k+1])
//     hash    hs[cap] uint4 {key, begin, len, 0}, linear probing, key 0 = empty
// This is the reference's sorted pair list + aux array + per-key dict
// (storage.py:38-53, 66-72, 84-94) turned into flat HBM arrays.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "gsmat_b200.h"

typedef uint32_t u32;
typedef uint64_t u64;
typedef long long i64;

#define GSM_MAX_VARS 32
#define GSM_MAX_STEPS 64

namespace gsm {

struct Orient {
  const u32* src = nullptr;
  const u32* dst = nullptr;
  const u32* doff = nullptr;  // dense index or nullptr
  const uint4* hs = nullptr;  // hash index or nullptr
  u32 hmask = 0;
  u32 nnz = 0;
  u32 nrows = 0;
  u32 maxkey = 0;  // dense index covers keys 0..maxkey
  u32 kbias = 0;   // hash keys are stored as key + kbias (1 for table joins, where 0 is a legal id)
};

struct PredDev {
  Orient so, os;
  const u32* diag = nullptr;  // sorted x with (x,x) in M   (executor.py:117-118)
  u32 ndiag = 0;
  int present = 0;
};

// Device-side binding table descriptor.  Columns are separate u32 arrays
// (struct-of-arrays): n is written by the producing kernel, so downstream
// kernels never need the host to know a row count.
struct DTable {
  i64 n;
  u32* col[GSM_MAX_VARS];
};

struct StepStat {
  i64 e;         // prealloc_total (E)
  i64 rows;      // rows produced (uncapped)
  i64 overflow;  // 1 if rows exceeded the output capacity
  i64 pad;
};

__device__ __forceinline__ u32 hash32(u32 x) {
  x ^= x >> 16;
  x *= 0x85ebca6bu;
  x ^= x >> 13;
  x *= 0xc2b2ae35u;
  x ^= x >> 16;
  return x;
}

// key -> (begin, len) in R.dst.  Replaces PredicateMatrix._so_runs/_os_runs
// lookups (storage.py:71-72, 84-94).
__device__ __forceinline__ uint2 seg_lookup(const Orient& R, u32 key) {
  if (R.doff) {
    if (key > R.maxkey) return make_uint2(0, 0);
    u32 b = __ldg(R.doff + key), e = __ldg(R.doff + key + 1);
    return make_uint2(b, e - b);
  }
  if (R.hs) {
    key += R.kbias;
    u32 h = hash32(key) & R.hmask;
    for (;;) {
      uint4 s = __ldg(R.hs + h);
      if (s.x == key) return make_uint2(s.y, s.z);
      if (s.x == 0) return make_uint2(0, 0);
      h = (h + 1) & R.hmask;
    }
  }
  return make_uint2(0, 0);
}

// Membership of `v` in the ascending run a[0..len).  Latency, not bytes,
// decides here (one probe per left row or candidate, each a chain of
// dependent loads), so the search is 9-ary: each round loads 8 pivots at
// once and keeps the slice between the two that bracket v, until at most 8
// entries remain, which are compared with independent loads.  A run of 20
// costs 2 memory round trips (binary search: 5), a run of 1000 costs 4 (10).
__device__ __forceinline__ bool sorted_contains(const u32* a, u32 len, u32 v) {
  u32 lo = 0, hi = len;
  while (hi - lo > 8) {
    const u32 n = hi - lo;
    u32 pv[8];
#pragma unroll
    for (u32 i = 0; i < 8; i++) pv[i] = __ldg(a + lo + (u32)(((u64)(i + 1) * n) / 9));
    u32 c = 0;
    bool hit = false;
#pragma unroll
    for (u32 i = 0; i < 8; i++) {
      c += pv[i] < v;
      hit |= pv[i] == v;
    }
    if (hit) return true;
    const u32 nlo = c == 0 ? lo : lo + (u32)(((u64)c * n) / 9) + 1;
    const u32 nhi = c == 8 ? hi : lo + (u32)(((u64)(c + 1) * n) / 9);
    lo = nlo;
    hi = nhi;
  }
  bool hit = false;
#pragma unroll
  for (u32 i = 0; i < 8; i++)
    if (lo + i < hi) hit |= __ldg(a + lo + i) == v;
  return hit;
}

// Programmatic dependent launch (PDL): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; it must wait before touching the predecessor's output.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// Phase trace (diagnostic builds only, `make trace`): thread 0 of each block
// stamps %globaltimer and clock64 at phase boundaries of its first tiles.
constexpr int TRACE_SLOTS = 32;  // per block: 4 tiles x 8 phases
#ifdef GSM_TRACE
static __device__ unsigned long long g_trace[8192 * TRACE_SLOTS * 2];
__device__ __forceinline__ void trace_at(int tile_iter, int phase) {
  if (threadIdx.x == 0 && tile_iter < 4 && blockIdx.x < 8192) {
    unsigned long long g, c;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    const size_t i = ((size_t)blockIdx.x * TRACE_SLOTS + tile_iter * 8 + phase) * 2;
    g_trace[i] = g;
    g_trace[i + 1] = c;
  }
}
#else
__device__ __forceinline__ void trace_at(int, int) {}
#endif

}  // namespace gsm

// ---- host-side error plumbing (gsm_api.cu) ----
namespace gsm {
gsm_status set_error(gsm_status st, const std::string& msg);
gsm_status cuda_error(cudaError_t e, const char* what);
void count_launch(int n = 1);
}  // namespace gsm

#define GSM_CUDA(call)                                        \
  do {                                                        \
    cudaError_t _e = (call);                                  \
    if (_e != cudaSuccess) return ::gsm::cuda_error(_e, #call); \
  } while (0)
