// gsm_internal.cuh — host-side objects behind the C ABI handles.
#pragma once
#include <memory>
#include <utility>
#include <vector>

#include "gsm_common.cuh"

// Host copy of one orientation's aux array (storage.py:38-53): distinct keys
// and their run offsets.  Lets the host resolve constant-endpoint scans
// (R2/R3) without a device round trip.
struct HostAux {
  std::vector<u32> key;  // ascending distinct keys
  std::vector<u32> off;  // off[i]..off[i+1] = run of key[i]; size key.size()+1
  u32 max_run = 0;       // longest run (max degree in this orientation)
  bool find(u32 k, u32& begin, u32& len) const;
};

struct gsm_store {
  int device = 0;
  i64 node_count = 0;
  int max_pid = 0;
  std::vector<gsm::PredDev> preds;  // indexed by pid (0 unused)
  std::vector<HostAux> aux_so, aux_os;  // indexed by pid
  std::vector<void*> allocations;
  i64 bytes = 0;
  u32 max_nnz = 0;
  bool finalized = false;
  // rendered node terms for result decoding (gsm_store_put_dictionary):
  // term v = term_bytes[term_off[v-1], term_off[v])
  unsigned char* term_bytes = nullptr;
  u64* term_off = nullptr;
  i64 n_terms = 0, term_total = 0;
  u32* d_flag = nullptr;  // validation scratch: [0] min unsorted-key pos, [1] min unsorted-value pos, [2] id overflow
};

struct gsm_context;

// Allocator whose resize() leaves new elements uninitialised: a decoded
// result of 10^9 bytes is overwritten by its device copy right away, so
// zero-filling it first would cost a full extra pass over host memory.
template <class T>
struct uninit_alloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = uninit_alloc<U>;
  };
  uninit_alloc() = default;
  template <class U>
  uninit_alloc(const uninit_alloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};

// Host byte blob returned through the C ABI (decoded text, parsed triples).
struct gsm_text {
  std::vector<char, uninit_alloc<char>> bytes;
};

struct gsm_result {
  int device = 0;
  i64 n = 0;
  int k = 0;
  u32* rows = nullptr;         // device, row-major n x k (owned), or nullptr
  const u32* staged = nullptr; // rows in the context's pinned staging buffer
  const gsm_context* ctx = nullptr;
  u64 gen = 0;                 // staging generation the rows belong to
  bool zc = false;             // staged rows were written to host memory only (no device copy)
  const u32* dev_view = nullptr;  // rows left in the context's arena (not owned; valid while gen matches)
};

namespace gsm {
u64 context_generation(const gsm_context* c);
const u32* context_device_rows(const gsm_context* c);
}

namespace gsm {
cudaError_t store_alloc(gsm_store* s, void** p, size_t bytes);
}
