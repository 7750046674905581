// gsm_store.cu — HBM-resident predicate matrices and their row indexes.
//
// Replaces storage.PredicateMatrix / build_aux / Store.matrices
// (/root/reference/pkg/src/gsmat/storage.py:38-122).  The pair files are
// uploaded as-is (u64 LE pairs, storage.py:183-200) and narrowed to u32
// columns on the device; all index structures are built by device kernels.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gsm_internal.cuh"

bool HostAux::find(u32 k, u32& begin, u32& len) const {
  auto it = std::lower_bound(key.begin(), key.end(), k);
  if (it == key.end() || *it != k) {
    begin = 0;
    len = 0;
    return false;
  }
  size_t i = (size_t)(it - key.begin());
  begin = off[i];
  len = off[i + 1] - off[i];
  return true;
}

namespace gsm {

cudaError_t store_alloc(gsm_store* s, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes ? bytes : 4);
  if (e == cudaSuccess) {
    s->allocations.push_back(*p);
    s->bytes += (i64)bytes;
  }
  return e;
}

// Split interleaved u64 pairs into u32 key/value columns and validate order.
// flag[0]: min position with key < previous key (build_aux's ValueError,
// storage.py:44-45); flag[1]: min position whose value breaks ascending order
// inside a key run; flag[2]: an id >= 2^32.
__global__ void k_narrow_pairs(const u64* __restrict__ pairs, u32* __restrict__ src,
                               u32* __restrict__ dst, i64 chunk_begin, i64 n,
                               u32* __restrict__ flag) {
  i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    ulonglong2 pr = reinterpret_cast<const ulonglong2*>(pairs)[i];
    if ((pr.x >> 32) | (pr.y >> 32)) atomicExch(flag + 2, 1u);
    src[chunk_begin + i] = (u32)pr.x;
    dst[chunk_begin + i] = (u32)pr.y;
  }
}

__global__ void k_check_sorted(const u32* __restrict__ src, const u32* __restrict__ dst, i64 n,
                               u32* __restrict__ flag) {
  i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = 1 + (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u32 a = src[i - 1], b = src[i];
    if (b < a) atomicMin(flag + 0, (u32)i);
    else if (b == a && dst[i] < dst[i - 1]) atomicMin(flag + 1, (u32)i);
  }
}

__device__ __forceinline__ u32 lower_bound_u32(const u32* a, u32 n, u32 v) {
  u32 lo = 0, hi = n;
  while (lo < hi) {
    u32 mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Dense key index: doff[v] = first position with src >= v, v in [0, maxkey+1].
__global__ void k_dense_index(const u32* __restrict__ src, u32 nnz, u32* __restrict__ doff,
                              u32 nkeys) {
  u32 stride = gridDim.x * blockDim.x;
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < nkeys; v += stride)
    doff[v] = lower_bound_u32(src, nnz, v);
}

__global__ void k_count_heads(const u32* __restrict__ src, u32 nnz, u32* __restrict__ out) {
  u32 stride = gridDim.x * blockDim.x, c = 0;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride)
    c += (i == 0 || src[i] != src[i - 1]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Hash key index: one {key, begin, len} slot per aux-array entry.
__global__ void k_hash_index(const u32* __restrict__ src, u32 nnz, u32* __restrict__ slots,
                             u32 mask) {
  u32 stride = gridDim.x * blockDim.x;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride) {
    u32 key = src[i];
    if (i != 0 && src[i - 1] == key) continue;
    u32 end = i + lower_bound_u32(src + i, nnz - i, key + 1);
    u32 h = hash32(key) & mask;
    for (;;) {
      u32 prev = atomicCAS(slots + 4 * h, 0u, key);
      if (prev == 0u) {
        slots[4 * h + 1] = i;
        slots[4 * h + 2] = end - i;
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

struct DiagFlag {
  const u32* src;
  const u32* dst;
  __device__ bool operator()(const u32& i) const { return src[i] == dst[i]; }
};

__global__ void k_gather_u32(const u32* __restrict__ idx, const u32* __restrict__ n_dev,
                             const u32* __restrict__ vals, u32* __restrict__ out) {
  u32 n = *n_dev;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = vals[idx[i]];
}

static int grid_for(i64 n, int threads = 256) {
  i64 b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

static gsm_status build_orient(gsm_store* s, Orient& o) {
  if (o.nnz == 0) return GSM_OK;
  // distinct keys (len of the aux array, storage.py:38-53)
  u32* d_cnt;
  GSM_CUDA(cudaMalloc(&d_cnt, 4));
  GSM_CUDA(cudaMemset(d_cnt, 0, 4));
  k_count_heads<<<grid_for(o.nnz), 256>>>(o.src, o.nnz, d_cnt);
  count_launch();
  GSM_CUDA(cudaMemcpy(&o.nrows, d_cnt, 4, cudaMemcpyDeviceToHost));
  cudaFree(d_cnt);
  size_t cap = 16;
  while (cap < 2 * (size_t)o.nrows) cap <<= 1;
  size_t hash_bytes = cap * 16, dense_bytes = 4 * ((size_t)s->node_count + 2);
  if (dense_bytes <= 2 * hash_bytes) {
    u32* doff;
    GSM_CUDA(store_alloc(s, (void**)&doff, dense_bytes));
    u32 nkeys = (u32)(s->node_count + 2);
    k_dense_index<<<grid_for(nkeys), 256>>>(o.src, o.nnz, doff, nkeys);
    count_launch();
    o.doff = doff;
    o.maxkey = (u32)(s->node_count);
  } else {
    u32* slots;
    GSM_CUDA(store_alloc(s, (void**)&slots, hash_bytes));
    GSM_CUDA(cudaMemset(slots, 0, hash_bytes));
    k_hash_index<<<grid_for(o.nnz), 256>>>(o.src, o.nnz, slots, (u32)(cap - 1));
    count_launch();
    o.hs = reinterpret_cast<const uint4*>(slots);
    o.hmask = (u32)(cap - 1);
  }
  GSM_CUDA(cudaGetLastError());
  return GSM_OK;
}

// Host copy of an orientation's aux array (storage.py:38-53): run heads
// selected on the device (cub), then one copy of keys and offsets.
struct HeadFlag {
  const u32* src;
  __device__ bool operator()(const u32& i) const { return i == 0 || src[i] != src[i - 1]; }
};

static gsm_status build_host_aux(const Orient& o, HostAux& a) {
  a.key.clear();
  a.off.clear();
  a.max_run = 0;
  if (o.nnz == 0) {
    a.off.push_back(0);
    return GSM_OK;
  }
  u32 *d_pos, *d_n, *d_key;
  GSM_CUDA(cudaMalloc(&d_pos, 4 * (size_t)o.nrows + 4));
  GSM_CUDA(cudaMalloc(&d_key, 4 * (size_t)o.nrows + 4));
  GSM_CUDA(cudaMalloc(&d_n, 4));
  thrust::counting_iterator<u32> it(0);
  size_t tmp_bytes = 0;
  HeadFlag f{o.src};
  cub::DeviceSelect::If(nullptr, tmp_bytes, it, d_pos, d_n, (int64_t)o.nnz, f);
  void* tmp;
  GSM_CUDA(cudaMalloc(&tmp, tmp_bytes ? tmp_bytes : 4));
  cub::DeviceSelect::If(tmp, tmp_bytes, it, d_pos, d_n, (int64_t)o.nnz, f);
  k_gather_u32<<<grid_for(o.nrows), 256>>>(d_pos, d_n, o.src, d_key);
  count_launch(3);
  a.key.resize(o.nrows);
  a.off.resize((size_t)o.nrows + 1);
  GSM_CUDA(cudaMemcpy(a.key.data(), d_key, 4 * (size_t)o.nrows, cudaMemcpyDeviceToHost));
  GSM_CUDA(cudaMemcpy(a.off.data(), d_pos, 4 * (size_t)o.nrows, cudaMemcpyDeviceToHost));
  a.off[o.nrows] = o.nnz;
  for (u32 i = 0; i < o.nrows; i++) a.max_run = std::max(a.max_run, a.off[i + 1] - a.off[i]);
  cudaFree(tmp);
  cudaFree(d_pos);
  cudaFree(d_key);
  cudaFree(d_n);
  GSM_CUDA(cudaGetLastError());
  return GSM_OK;
}

static gsm_status build_diag(gsm_store* s, PredDev& p) {
  const Orient& o = p.so;
  if (o.nnz == 0) return GSM_OK;
  u32 *d_idx, *d_n;
  GSM_CUDA(cudaMalloc(&d_idx, 4 * (size_t)o.nnz));
  GSM_CUDA(cudaMalloc(&d_n, 4));
  thrust::counting_iterator<u32> it(0);
  size_t tmp_bytes = 0;
  DiagFlag f{o.src, o.dst};
  cub::DeviceSelect::If(nullptr, tmp_bytes, it, d_idx, d_n, (int64_t)o.nnz, f);
  void* tmp;
  GSM_CUDA(cudaMalloc(&tmp, tmp_bytes ? tmp_bytes : 4));
  cub::DeviceSelect::If(tmp, tmp_bytes, it, d_idx, d_n, (int64_t)o.nnz, f);
  count_launch(2);
  u32 nd = 0;
  GSM_CUDA(cudaMemcpy(&nd, d_n, 4, cudaMemcpyDeviceToHost));
  u32* diag;
  GSM_CUDA(store_alloc(s, (void**)&diag, 4 * (size_t)nd));
  if (nd) {
    k_gather_u32<<<grid_for(nd), 256>>>(d_idx, d_n, o.src, diag);
    count_launch();
  }
  p.diag = diag;
  p.ndiag = nd;
  cudaFree(tmp);
  cudaFree(d_idx);
  cudaFree(d_n);
  GSM_CUDA(cudaGetLastError());
  return GSM_OK;
}

}  // namespace gsm

using namespace gsm;

extern "C" {

gsm_status gsm_store_create(int32_t device, int64_t node_count, int32_t max_pid, gsm_store** out) {
  *out = nullptr;
  if (node_count < 0 || node_count > 0xFFFFFFF0LL)
    return set_error(GSM_ERR_VALUE, "node_count must be in [0, 2^32-16)");
  if (max_pid < 0) return set_error(GSM_ERR_VALUE, "max_pid must be >= 0");
  int ndev = 0;
  GSM_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return set_error(GSM_ERR_VALUE, "device index out of range");
  GSM_CUDA(cudaSetDevice(device));
  gsm_store* s = new gsm_store();
  s->device = device;
  s->node_count = node_count;
  s->max_pid = max_pid;
  s->preds.resize((size_t)max_pid + 1);
  s->aux_so.resize((size_t)max_pid + 1);
  s->aux_os.resize((size_t)max_pid + 1);
  cudaError_t e = cudaMalloc(&s->d_flag, 16);
  if (e != cudaSuccess) {
    delete s;
    return cuda_error(e, "cudaMalloc(flags)");
  }
  *out = s;
  return GSM_OK;
}

gsm_status gsm_store_put_predicate(gsm_store* s, int32_t pid, const uint64_t* so_pairs,
                                   const uint64_t* os_pairs, int64_t nnz) {
  return gsm_store_put_predicate_shard(s, pid, so_pairs, nnz, os_pairs, nnz);
}

gsm_status gsm_store_put_predicate_shard(gsm_store* s, int32_t pid, const uint64_t* so_pairs,
                                         int64_t nnz_so, const uint64_t* os_pairs, int64_t nnz_os) {
  if (!s) return set_error(GSM_ERR_VALUE, "null store");
  if (s->finalized) return set_error(GSM_ERR_VALUE, "store already finalized");
  if (pid < 1 || pid > s->max_pid) return set_error(GSM_ERR_UNKNOWN_PREDICATE, "no matrix for predicate id " + std::to_string(pid));
  if (nnz_so < 0 || nnz_so >= 0xFFFFFFF0LL || nnz_os < 0 || nnz_os >= 0xFFFFFFF0LL)
    return set_error(GSM_ERR_VALUE, "predicate pair count must be < 2^32");
  if ((nnz_so > 0 && !so_pairs) || (nnz_os > 0 && !os_pairs)) return set_error(GSM_ERR_VALUE, "null pair array");
  GSM_CUDA(cudaSetDevice(s->device));
  PredDev& p = s->preds[pid];
  if (p.present) return set_error(GSM_ERR_VALUE, "predicate uploaded twice");
  p.present = 1;
  const i64 CHUNK = 1 << 24;  // 16M pairs = 256 MiB staging
  const i64 nmax = std::max(nnz_so, nnz_os);
  u64* stage = nullptr;
  if (nmax > 0) GSM_CUDA(cudaMalloc(&stage, 16 * (size_t)std::min<i64>(nmax, CHUNK)));
  const uint64_t* hosts[2] = {so_pairs, os_pairs};
  const i64 counts[2] = {nnz_so, nnz_os};
  Orient* ors[2] = {&p.so, &p.os};
  for (int w = 0; w < 2; w++) {
    Orient& o = *ors[w];
    const i64 nnz = counts[w];
    u32 *src, *dst;
    GSM_CUDA(store_alloc(s, (void**)&src, 4 * (size_t)nnz));
    GSM_CUDA(store_alloc(s, (void**)&dst, 4 * (size_t)nnz));
    o.src = src;
    o.dst = dst;
    o.nnz = (u32)nnz;
    u32 init[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u};
    GSM_CUDA(cudaMemcpy(s->d_flag, init, 16, cudaMemcpyHostToDevice));
    for (i64 b = 0; b < nnz; b += CHUNK) {
      i64 m = std::min<i64>(CHUNK, nnz - b);
      GSM_CUDA(cudaMemcpy(stage, hosts[w] + 2 * b, 16 * (size_t)m, cudaMemcpyHostToDevice));
      k_narrow_pairs<<<grid_for(m), 256>>>(stage, src, dst, b, m, s->d_flag);
      count_launch();
    }
    if (nnz > 1) {
      k_check_sorted<<<grid_for(nnz), 256>>>(src, dst, nnz, s->d_flag);
      count_launch();
    }
    u32 flags[4];
    GSM_CUDA(cudaMemcpy(flags, s->d_flag, 16, cudaMemcpyDeviceToHost));
    const char* file = w == 0 ? "so" : "os";
    if (flags[2]) {
      cudaFree(stage);
      return set_error(GSM_ERR_STORE_FORMAT, "p" + std::to_string(pid) + "." + file +
                                                 ": node id >= 2^32 is not supported");
    }
    if (flags[0] != 0xFFFFFFFFu) {
      cudaFree(stage);
      return set_error(GSM_ERR_UNSORTED, "pair list not sorted at position " + std::to_string(flags[0]));
    }
    if (flags[1] != 0xFFFFFFFFu) {
      cudaFree(stage);
      return set_error(GSM_ERR_STORE_FORMAT,
                       "p" + std::to_string(pid) + "." + file +
                           ": pairs not sorted by (key, value) at position " +
                           std::to_string(flags[1]));
    }
  }
  if (stage) cudaFree(stage);
  s->max_nnz = std::max<u32>(s->max_nnz, (u32)nmax);
  GSM_CUDA(cudaGetLastError());
  return GSM_OK;
}

// Store loader fast path (storage.load's pair reads, storage.py:193-200,
// 222-271): every predicate's p<ID>.so / p<ID>.os file is streamed to the
// device in 32 MiB chunks.  Reader threads pread chunks into a ring of pinned
// buffers while the calling thread issues, per chunk, the H2D copy and the
// narrowing kernel on one stream, so disk / page-cache reads, PCIe transfers
// and the device work overlap.  Sortedness and id-range checks accumulate in
// per-file device flags, read back once at the end and reported in upload
// order with put_predicate's messages.
gsm_status gsm_store_load_files(gsm_store* s, int32_t n, const int32_t* pids,
                                const char* const* so_paths, const char* const* os_paths,
                                const int64_t* nnz) {
  if (!s) return set_error(GSM_ERR_VALUE, "null store");
  if (s->finalized) return set_error(GSM_ERR_VALUE, "store already finalized");
  if (n < 0 || (n > 0 && (!pids || !so_paths || !os_paths || !nnz)))
    return set_error(GSM_ERR_VALUE, "bad arguments");
  for (int i = 0; i < n; i++) {
    if (pids[i] < 1 || pids[i] > s->max_pid)
      return set_error(GSM_ERR_UNKNOWN_PREDICATE, "no matrix for predicate id " + std::to_string(pids[i]));
    if (nnz[i] < 0 || nnz[i] >= 0xFFFFFFF0LL) return set_error(GSM_ERR_VALUE, "predicate pair count must be < 2^32");
    if (s->preds[pids[i]].present) return set_error(GSM_ERR_VALUE, "predicate uploaded twice");
    for (int j = 0; j < i; j++)
      if (pids[j] == pids[i]) return set_error(GSM_ERR_VALUE, "predicate uploaded twice");
  }
  GSM_CUDA(cudaSetDevice(s->device));
  // files: 2 per predicate (so, os)
  const int nf = 2 * n;
  std::vector<int> fds((size_t)nf, -1);
  auto close_all = [&]() {
    for (int fd : fds)
      if (fd >= 0) close(fd);
  };
  for (int f = 0; f < nf; f++) {
    const char* path = (f & 1) ? os_paths[f / 2] : so_paths[f / 2];
    fds[f] = open(path, O_RDONLY);
    if (fds[f] < 0) {
      close_all();
      return set_error(GSM_ERR_STORE_FORMAT, std::string("cannot open ") + path + ": " + strerror(errno));
    }
  }
  // device columns
  for (int i = 0; i < n; i++) {
    PredDev& p = s->preds[pids[i]];
    for (Orient* o : {&p.so, &p.os}) {
      u32 *src, *dst;
      cudaError_t e = store_alloc(s, (void**)&src, 4 * (size_t)nnz[i]);
      if (e == cudaSuccess) e = store_alloc(s, (void**)&dst, 4 * (size_t)nnz[i]);
      if (e != cudaSuccess) {
        close_all();
        return cuda_error(e, "cudaMalloc(pair columns)");
      }
      o->src = src;
      o->dst = dst;
      o->nnz = (u32)nnz[i];
    }
  }
  // chunk list in upload order
  struct Chunk {
    int f;
    i64 off, m;
  };
  const i64 CH = (i64)1 << 21;  // pairs per chunk (32 MiB)
  std::vector<Chunk> chunks;
  i64 max_m = 0;
  for (int f = 0; f < nf; f++)
    for (i64 b = 0; b < nnz[f / 2]; b += CH) {
      const i64 m = std::min(CH, nnz[f / 2] - b);
      chunks.push_back({f, b, m});
      max_m = std::max(max_m, m);
    }
  const int NS = (int)std::min<size_t>(8, std::max<size_t>(1, chunks.size()));
  std::vector<u64*> hbuf((size_t)NS, nullptr), dbuf((size_t)NS, nullptr);
  std::vector<cudaEvent_t> ev((size_t)NS, nullptr);
  cudaStream_t st = nullptr;
  u32* d_flags = nullptr;
  auto release = [&]() {
    for (int k = 0; k < NS; k++) {
      if (hbuf[k]) cudaFreeHost(hbuf[k]);
      if (dbuf[k]) cudaFree(dbuf[k]);
      if (ev[k]) cudaEventDestroy(ev[k]);
    }
    if (st) cudaStreamDestroy(st);
    if (d_flags) cudaFree(d_flags);
    close_all();
  };
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&d_flags, 16 * (size_t)std::max(nf, 1));
  for (int k = 0; k < NS && e == cudaSuccess && max_m > 0; k++) {
    e = cudaMallocHost(&hbuf[k], 16 * (size_t)max_m);
    if (e == cudaSuccess) e = cudaMalloc(&dbuf[k], 16 * (size_t)max_m);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    release();
    return cuda_error(e, "loader buffers");
  }
  {
    std::vector<u32> init((size_t)4 * std::max(nf, 1));
    for (int f = 0; f < nf; f++) {
      init[4 * f] = init[4 * f + 1] = 0xFFFFFFFFu;
      init[4 * f + 2] = init[4 * f + 3] = 0u;
    }
    e = cudaMemcpy(d_flags, init.data(), 16 * (size_t)std::max(nf, 1), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      release();
      return cuda_error(e, "cudaMemcpy(flags)");
    }
  }
  // pipeline: chunk c uses slot c % NS; readers fill, this thread issues
  const int nc = (int)chunks.size();
  std::mutex mu;
  std::condition_variable cv;
  std::vector<char> ready((size_t)nc, 0);
  int issued = 0;  // chunks whose copy + kernel are enqueued (events recorded)
  bool failed = false;
  std::string read_err;
  std::atomic<int> next{0};
  auto reader = [&]() {
    for (;;) {
      const int c = next.fetch_add(1);
      if (c >= nc) return;
      const int k = c % NS;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return failed || issued > c - NS; });
        if (failed) return;
      }
      if (c >= NS) cudaEventSynchronize(ev[k]);  // the slot's previous copy is done
      const Chunk& ch = chunks[c];
      char* dst = reinterpret_cast<char*>(hbuf[k]);
      size_t want = 16 * (size_t)ch.m, got = 0;
      off_t off = (off_t)(16 * ch.off);
      while (got < want) {
        ssize_t r = pread(fds[ch.f], dst + got, want - got, off + (off_t)got);
        if (r <= 0) {
          std::lock_guard<std::mutex> lk(mu);
          if (!failed) {
            failed = true;
            const int pid = pids[ch.f / 2];
            read_err = "p" + std::to_string(pid) + ((ch.f & 1) ? ".os" : ".so") +
                       (r == 0 ? ": unexpected end of file" : std::string(": read error: ") + strerror(errno));
          }
          cv.notify_all();
          return;
        }
        got += (size_t)r;
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        ready[c] = 1;
      }
      cv.notify_all();
    }
  };
  const int nthreads = std::min(4, std::max(1, nc));
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; t++) th.emplace_back(reader);
  cudaError_t ce = cudaSuccess;
  for (int c = 0; c < nc && ce == cudaSuccess; c++) {
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [&] { return failed || ready[c]; });
      if (failed) break;
    }
    const int k = c % NS;
    const Chunk& ch = chunks[c];
    const PredDev& p = s->preds[pids[ch.f / 2]];
    const Orient& o = (ch.f & 1) ? p.os : p.so;
    ce = cudaMemcpyAsync(dbuf[k], hbuf[k], 16 * (size_t)ch.m, cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess) {
      k_narrow_pairs<<<grid_for(ch.m), 256, 0, st>>>(dbuf[k], const_cast<u32*>(o.src), const_cast<u32*>(o.dst), ch.off, ch.m, d_flags + 4 * ch.f);
      count_launch();
      ce = cudaEventRecord(ev[k], st);
    }
    {
      std::lock_guard<std::mutex> lk(mu);
      issued = c + 1;
      if (ce != cudaSuccess) failed = true;
    }
    cv.notify_all();
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    if (ce != cudaSuccess) failed = true;
    issued = nc + NS;  // release any waiting reader
  }
  cv.notify_all();
  for (auto& t : th) t.join();
  if (ce != cudaSuccess) {
    release();
    return cuda_error(ce, "loader copy");
  }
  if (failed) {
    release();
    return set_error(GSM_ERR_STORE_FORMAT, read_err);
  }
  for (int f = 0; f < nf; f++) {
    const PredDev& p = s->preds[pids[f / 2]];
    const Orient& o = (f & 1) ? p.os : p.so;
    if (o.nnz > 1) {
      k_check_sorted<<<grid_for(o.nnz), 256, 0, st>>>(o.src, o.dst, o.nnz, d_flags + 4 * f);
      count_launch();
    }
  }
  std::vector<u32> flags((size_t)4 * std::max(nf, 1));
  ce = cudaMemcpyAsync(flags.data(), d_flags, 16 * (size_t)std::max(nf, 1), cudaMemcpyDeviceToHost, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  release();
  if (ce != cudaSuccess) return cuda_error(ce, "loader flags");
  for (int f = 0; f < nf; f++) {
    const int pid = pids[f / 2];
    const char* file = (f & 1) ? "os" : "so";
    const u32* fl = &flags[4 * (size_t)f];
    if (fl[2])
      return set_error(GSM_ERR_STORE_FORMAT, "p" + std::to_string(pid) + "." + file +
                                                 ": node id >= 2^32 is not supported");
    if (fl[0] != 0xFFFFFFFFu)
      return set_error(GSM_ERR_UNSORTED, "pair list not sorted at position " + std::to_string(fl[0]));
    if (fl[1] != 0xFFFFFFFFu)
      return set_error(GSM_ERR_STORE_FORMAT, "p" + std::to_string(pid) + "." + file +
                                                 ": pairs not sorted by (key, value) at position " +
                                                 std::to_string(fl[1]));
  }
  for (int i = 0; i < n; i++) {
    s->preds[pids[i]].present = 1;
    s->max_nnz = std::max<u32>(s->max_nnz, (u32)nnz[i]);
  }
  return GSM_OK;
}

gsm_status gsm_store_finalize(gsm_store* s) {
  if (!s) return set_error(GSM_ERR_VALUE, "null store");
  if (s->finalized) return GSM_OK;
  GSM_CUDA(cudaSetDevice(s->device));
  for (int pid = 1; pid <= s->max_pid; pid++) {
    PredDev& p = s->preds[pid];
    if (!p.present) continue;
    gsm_status st;
    if ((st = build_orient(s, p.so)) != GSM_OK) return st;
    if ((st = build_orient(s, p.os)) != GSM_OK) return st;
    if ((st = build_host_aux(p.so, s->aux_so[pid])) != GSM_OK) return st;
    if ((st = build_host_aux(p.os, s->aux_os[pid])) != GSM_OK) return st;
    if ((st = build_diag(s, p)) != GSM_OK) return st;
  }
  GSM_CUDA(cudaDeviceSynchronize());
  s->finalized = true;
  return GSM_OK;
}

gsm_status gsm_store_device_bytes(const gsm_store* s, int64_t* bytes) {
  if (!s) return set_error(GSM_ERR_VALUE, "null store");
  *bytes = s->bytes;
  return GSM_OK;
}

gsm_status gsm_store_free(gsm_store* s) {
  if (!s) return GSM_OK;
  cudaSetDevice(s->device);
  for (void* p : s->allocations) cudaFree(p);
  if (s->d_flag) cudaFree(s->d_flag);
  if (s->term_bytes) cudaFree(s->term_bytes);
  if (s->term_off) cudaFree(s->term_off);
  delete s;
  return GSM_OK;
}

}  // extern "C"
