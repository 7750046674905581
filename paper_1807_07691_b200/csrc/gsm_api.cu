// gsm_api.cu — error plumbing, device queries, result handles.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>

#include "gsm_internal.cuh"

namespace gsm {

static thread_local std::string t_last_error;
static std::atomic<long long> g_launches{0};

gsm_status set_error(gsm_status st, const std::string& msg) {
  t_last_error = msg;
  return st;
}

gsm_status cuda_error(cudaError_t e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e),
           what);
  if (e == cudaErrorMemoryAllocation) return set_error(GSM_ERR_RESOURCE, buf);
  return set_error(GSM_ERR_CUDA, buf);
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace gsm

namespace {

// Multiset fingerprint of n row-major k-column rows: per row the splitmix64
// chain h = mix(h ^ id) from h0 = golden ratio, then sum and xor over rows
// (wrapping).  Rows are read with warp-contiguous loads: a warp walks 32
// consecutive rows, so its k strided loads cover one contiguous 128*k-byte
// span.  Reads host-mapped (staged) rows through UVA as well.
__device__ __forceinline__ u64 fp_mix(u64 h, u32 v) {
  u64 z = (h ^ (u64)v) + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) k_fingerprint(const u32* __restrict__ rows, i64 n, int k,
                                                     unsigned long long* __restrict__ out) {
  u64 s = 0, x = 0;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const u32* row = rows + r * k;
    u64 h = 0x9E3779B97F4A7C15ull;
    for (int c = 0; c < k; c++) h = fp_mix(h, __ldg(row + c));
    s += h;
    x ^= h;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    x ^= __shfl_xor_sync(0xffffffffu, x, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out + 1, (unsigned long long)s);
    atomicXor(out + 2, (unsigned long long)x);
  }
}

}  // namespace

extern "C" {

const char* gsm_last_error(void) { return gsm::t_last_error.c_str(); }

int64_t gsm_kernel_launches(void) { return gsm::g_launches.load(); }

gsm_status gsm_device_count(int32_t* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return gsm::cuda_error(e, "cudaGetDeviceCount");
  }
  *count = n;
  return GSM_OK;
}

gsm_status gsm_result_shape(const gsm_result* res, int64_t* n_rows, int32_t* n_cols) {
  if (!res) return gsm::set_error(GSM_ERR_VALUE, "null result");
  *n_rows = res->n;
  *n_cols = res->k;
  return GSM_OK;
}

gsm_status gsm_result_copy(const gsm_result* res, uint32_t* host_rows) {
  if (!res) return gsm::set_error(GSM_ERR_VALUE, "null result");
  size_t bytes = (size_t)res->n * (size_t)res->k * sizeof(u32);
  if (bytes == 0) return GSM_OK;
  if (res->staged) {
    if (gsm::context_generation(res->ctx) != res->gen)
      return gsm::set_error(GSM_ERR_VALUE, "result invalidated by a later gsm_execute on its context");
    memcpy(host_rows, res->staged, bytes);
    return GSM_OK;
  }
  if (res->dev_view && gsm::context_generation(res->ctx) != res->gen)
    return gsm::set_error(GSM_ERR_VALUE, "result invalidated by a later gsm_execute on its context");
  GSM_CUDA(cudaSetDevice(res->device));
  GSM_CUDA(cudaMemcpy(host_rows, res->dev_view ? res->dev_view : res->rows, bytes,
                      cudaMemcpyDeviceToHost));
  return GSM_OK;
}

gsm_status gsm_result_device_ptr(const gsm_result* res, uint64_t* device_ptr) {
  if (!res) return gsm::set_error(GSM_ERR_VALUE, "null result");
  if (res->staged) {  // the device copy of staged rows lives in the context's result buffer
    if (gsm::context_generation(res->ctx) != res->gen)
      return gsm::set_error(GSM_ERR_VALUE, "result invalidated by a later gsm_execute on its context");
    u32* d = const_cast<u32*>(gsm::context_device_rows(res->ctx));
    if (res->zc && res->n > 0) {  // zero-copy result: give it a device copy first
      GSM_CUDA(cudaSetDevice(res->device));
      GSM_CUDA(cudaMemcpy(d, res->staged, (size_t)res->n * (size_t)res->k * 4, cudaMemcpyHostToDevice));
    }
    *device_ptr = (uint64_t)(uintptr_t)d;
    return GSM_OK;
  }
  if (res->dev_view) {
    if (gsm::context_generation(res->ctx) != res->gen)
      return gsm::set_error(GSM_ERR_VALUE, "result invalidated by a later gsm_execute on its context");
    *device_ptr = (uint64_t)(uintptr_t)res->dev_view;
    return GSM_OK;
  }
  *device_ptr = (uint64_t)(uintptr_t)res->rows;
  return GSM_OK;
}

gsm_status gsm_result_fingerprint(const gsm_result* res, uint64_t* out) {
  if (!res || !out) return gsm::set_error(GSM_ERR_VALUE, "null result");
  out[0] = (uint64_t)res->n;
  out[1] = out[2] = 0;
  if (res->n == 0) return GSM_OK;
  if (res->k == 0) {  // every row is the empty tuple: h = h0
    const u64 h0 = 0x9E3779B97F4A7C15ull;
    out[1] = h0 * (u64)res->n;
    out[2] = (res->n & 1) ? h0 : 0;
    return GSM_OK;
  }
  const u32* rows = res->rows;
  if (res->staged || res->dev_view) {
    if (gsm::context_generation(res->ctx) != res->gen)
      return gsm::set_error(GSM_ERR_VALUE, "result invalidated by a later gsm_execute on its context");
    rows = res->staged ? res->staged : res->dev_view;
  }
  GSM_CUDA(cudaSetDevice(res->device));
  unsigned long long* d = nullptr;
  GSM_CUDA(cudaMalloc(&d, 3 * sizeof(unsigned long long)));
  cudaError_t e = cudaMemset(d, 0, 3 * sizeof(unsigned long long));
  if (e == cudaSuccess) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, res->device);
    const i64 blocks = std::min<i64>((i64)sms * 8, (res->n + 255) / 256);
    k_fingerprint<<<(unsigned)blocks, 256>>>(rows, res->n, res->k, d);
    gsm::count_launch();
    e = cudaGetLastError();
  }
  unsigned long long h[3] = {0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return gsm::cuda_error(e, "gsm_result_fingerprint");
  out[1] = h[1];
  out[2] = h[2];
  return GSM_OK;
}

gsm_status gsm_results_shape(gsm_result* const* res, int32_t n, int64_t* n_rows, int32_t* n_cols) {
  if (n < 0 || (n > 0 && (!res || !n_rows || !n_cols))) return gsm::set_error(GSM_ERR_VALUE, "bad arguments");
  for (int i = 0; i < n; i++) {
    n_rows[i] = res[i] ? res[i]->n : 0;
    n_cols[i] = res[i] ? res[i]->k : 0;
  }
  return GSM_OK;
}

gsm_status gsm_results_copy(gsm_result* const* res, int32_t n, uint32_t* const* host_rows,
                            int32_t free_after) {
  if (n < 0 || (n > 0 && !res)) return gsm::set_error(GSM_ERR_VALUE, "bad arguments");
  gsm_status first = GSM_OK;
  for (int i = 0; i < n; i++) {
    if (res[i] && host_rows && host_rows[i] && first == GSM_OK) {
      gsm_status st = gsm_result_copy(res[i], host_rows[i]);
      if (st != GSM_OK) first = st;
    }
  }
  if (free_after)
    for (int i = 0; i < n; i++) gsm_result_free(res[i]);
  return first;
}

gsm_status gsm_result_free(gsm_result* res) {
  if (!res) return GSM_OK;
  if (res->rows) {
    cudaSetDevice(res->device);
    cudaFree(res->rows);
  }
  delete res;
  return GSM_OK;
}

}  // extern "C"
