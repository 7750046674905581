// gsm_api.cu — error plumbing, device queries, result handles.
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
  GSM_CUDA(cudaSetDevice(res->device));
  GSM_CUDA(cudaMemcpy(host_rows, res->rows, bytes, cudaMemcpyDeviceToHost));
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
  *device_ptr = (uint64_t)(uintptr_t)res->rows;
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
