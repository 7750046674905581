// gsm_decode.cu — result decoding on the device.
//
// Replaces the CLI's per-cell decode loop
//   for row in result.rows:
//       print("\t".join(qparser.format_term(decode(v)) for v in row))
// (/root/reference/pkg/src/gsmat/cli.py:102-105, dictionary.py:84-87,
// qparser.py:71-78): the node dictionary is uploaded once as its raw
// nodes.dict bytes, every term is rendered on the device into its N-Triples
// surface form (unescape the stored line, dictionary.py:28-43, then
// format_term), and a result table becomes its TSV body in two passes:
// per-row byte counts -> exclusive scan -> one warp per row copying the
// rendered terms, tab-separated, newline-terminated.
#include <cub/cub.cuh>

#include <string>
#include <vector>

#include "gsm_internal.cuh"

namespace gsm {
namespace {

// Render the stored (escaped) line L[0, n) of one term.  out == nullptr:
// only the length.  Follows unescape_term (dictionary.py:28-43: "\\x" -> the
// mapped char for x in \\ n r t, else x; a trailing lone backslash stays) and
// format_term (qparser.py:71-78): literals '"' + escape_literal(inner) + '"'
// + suffix (split at the LAST '"'), blank nodes as is, IRIs in <...>.
__device__ u64 render_term(const unsigned char* L, u64 n, unsigned char* out) {
  // pass A: unescaped length, position of the last '"' (unescaped coordinates)
  u64 ulen = 0, lastq = ~0ull;
  unsigned char c0 = 0, c1 = 0;
  for (u64 i = 0; i < n; i++) {
    unsigned char c = L[i];
    if (c == '\\' && i + 1 < n) {
      const unsigned char x = L[++i];
      c = x == 'n' ? '\n' : x == 'r' ? '\r' : x == 't' ? '\t' : x;
    }
    if (ulen == 0) c0 = c;
    if (ulen == 1) c1 = c;
    if (c == '"') lastq = ulen;
    ulen++;
  }
  const bool literal = ulen > 0 && c0 == '"';
  const bool bnode = ulen > 1 && c0 == '_' && c1 == ':';
  u64 o = 0;
  auto put = [&](unsigned char ch) {
    if (out) out[o] = ch;
    o++;
  };
  if (!literal && !bnode) put('<');
  u64 u = 0;  // unescaped position
  for (u64 i = 0; i < n; i++) {
    unsigned char c = L[i];
    if (c == '\\' && i + 1 < n) {
      const unsigned char x = L[++i];
      c = x == 'n' ? '\n' : x == 'r' ? '\r' : x == 't' ? '\t' : x;
    }
    if (literal && u == 0) {
      put('"');
      if (lastq == 0) put('"');  // end == 0: '"' + '' + '"' + term[1:]
      u++;
      continue;
    }
    if (literal && u < lastq) {  // inside the quotes: escape_literal
      switch (c) {
        case '\\': put('\\'); put('\\'); break;
        case '"': put('\\'); put('"'); break;
        case '\n': put('\\'); put('n'); break;
        case '\r': put('\\'); put('r'); break;
        case '\t': put('\\'); put('t'); break;
        default: put(c);
      }
    } else {
      put(c);
    }
    u++;
  }
  if (!literal && !bnode) put('>');
  return o;
}

__global__ void k_render_len(const unsigned char* __restrict__ buf, const i64* __restrict__ starts,
                             const i64* __restrict__ ends, i64 n, u64* __restrict__ len) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    len[i] = render_term(buf + starts[i], (u64)(ends[i] - starts[i]), nullptr);
}

__global__ void k_render_write(const unsigned char* __restrict__ buf, const i64* __restrict__ starts,
                               const i64* __restrict__ ends, i64 n, const u64* __restrict__ off,
                               unsigned char* __restrict__ out) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    render_term(buf + starts[i], (u64)(ends[i] - starts[i]), out + off[i]);
}

// Bytes of every result row: its terms + k separators (k-1 tabs, 1 newline).
// An id outside [1, n_terms] records the smallest offending cell (UnknownIdError).
__global__ void k_row_bytes(const u32* __restrict__ rows, i64 n, int k, const u64* __restrict__ off,
                            u64 n_terms, u64* __restrict__ rb, unsigned long long* __restrict__ bad) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    u64 b = (u64)k;
    for (int c = 0; c < k; c++) {
      const u32 v = rows[r * k + c];
      if (v == 0 || v > n_terms) {
        atomicMin(bad, (unsigned long long)(r * k + c));
        continue;
      }
      b += off[v] - off[v - 1];
    }
    rb[r] = b;
  }
}

// One warp per row: lanes copy consecutive bytes of each rendered term.
__global__ void k_write_rows(const u32* __restrict__ rows, i64 n, int k, const u64* __restrict__ off,
                             const unsigned char* __restrict__ terms, const u64* __restrict__ pos,
                             unsigned char* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const i64 warps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 r = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
    u64 p = pos[r];
    for (int c = 0; c < k; c++) {
      const u32 v = rows[r * k + c];
      const u64 b = off[v - 1], e = off[v];
      for (u64 j = lane; j < e - b; j += 32) out[p + j] = terms[b + j];
      p += e - b;
      if (lane == 0) out[p] = c + 1 < k ? '\t' : '\n';
      p++;
    }
  }
}

int grid_for(i64 n, int threads = 256) {
  i64 b = (n + threads - 1) / threads;
  return (int)std::max<i64>(1, std::min<i64>(b, 148 * 16));
}

}  // namespace
}  // namespace gsm

using namespace gsm;

extern "C" {

gsm_status gsm_store_put_dictionary(gsm_store* s, const char* buf, int64_t nbytes, const int64_t* starts,
                                    const int64_t* ends, int64_t n_terms) {
  if (!s) return set_error(GSM_ERR_VALUE, "null store");
  if (nbytes < 0 || n_terms < 0 || (nbytes > 0 && !buf) || (n_terms > 0 && (!starts || !ends)))
    return set_error(GSM_ERR_VALUE, "bad dictionary arguments");
  for (i64 i = 0; i < n_terms; i++)
    if (starts[i] < 0 || ends[i] < starts[i] || ends[i] > nbytes)
      return set_error(GSM_ERR_VALUE, "dictionary line offsets out of range");
  GSM_CUDA(cudaSetDevice(s->device));
  if (s->term_bytes) {
    cudaFree(s->term_bytes);
    cudaFree(s->term_off);
    s->term_bytes = nullptr;
    s->term_off = nullptr;
    s->n_terms = 0;
  }
  unsigned char* d_buf = nullptr;
  i64 *d_st = nullptr, *d_en = nullptr;
  u64* d_off = nullptr;  // n_terms + 1: off[0] = 0, term v = [off[v-1], off[v])
  void* tmp = nullptr;
  auto fail = [&](cudaError_t e, const char* what) {
    cudaFree(d_buf);
    cudaFree(d_st);
    cudaFree(d_en);
    cudaFree(d_off);
    cudaFree(tmp);
    return cuda_error(e, what);
  };
  cudaError_t e;
  if ((e = cudaMalloc(&d_buf, std::max<i64>(nbytes, 1))) != cudaSuccess) return fail(e, "cudaMalloc(dictionary)");
  if ((e = cudaMalloc(&d_st, 8 * std::max<i64>(n_terms, 1))) != cudaSuccess) return fail(e, "cudaMalloc");
  if ((e = cudaMalloc(&d_en, 8 * std::max<i64>(n_terms, 1))) != cudaSuccess) return fail(e, "cudaMalloc");
  if ((e = cudaMalloc(&d_off, 8 * (n_terms + 1))) != cudaSuccess) return fail(e, "cudaMalloc");
  if (nbytes && (e = cudaMemcpy(d_buf, buf, nbytes, cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e, "H2D");
  if (n_terms) {
    if ((e = cudaMemcpy(d_st, starts, 8 * n_terms, cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e, "H2D");
    if ((e = cudaMemcpy(d_en, ends, 8 * n_terms, cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e, "H2D");
  }
  if ((e = cudaMemset(d_off, 0, 8)) != cudaSuccess) return fail(e, "cudaMemset");
  u64 total = 0;
  if (n_terms) {
    k_render_len<<<grid_for(n_terms), 256>>>(d_buf, d_st, d_en, n_terms, d_off + 1);
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, d_off + 1, d_off + 1, n_terms);
    if ((e = cudaMalloc(&tmp, std::max<size_t>(tb, 4))) != cudaSuccess) return fail(e, "cudaMalloc");
    cub::DeviceScan::InclusiveSum(tmp, tb, d_off + 1, d_off + 1, n_terms);
    count_launch(2);
    if ((e = cudaMemcpy(&total, d_off + n_terms, 8, cudaMemcpyDeviceToHost)) != cudaSuccess) return fail(e, "D2H");
  }
  unsigned char* d_terms = nullptr;
  if ((e = cudaMalloc(&d_terms, std::max<u64>(total, 1))) != cudaSuccess) return fail(e, "cudaMalloc(terms)");
  if (n_terms) {
    k_render_write<<<grid_for(n_terms), 256>>>(d_buf, d_st, d_en, n_terms, d_off, d_terms);
    count_launch();
  }
  e = cudaDeviceSynchronize();
  cudaFree(d_buf);
  cudaFree(d_st);
  cudaFree(d_en);
  cudaFree(tmp);
  if (e != cudaSuccess) {
    cudaFree(d_off);
    cudaFree(d_terms);
    return cuda_error(e, "render terms");
  }
  s->term_bytes = d_terms;
  s->term_off = d_off;
  s->n_terms = n_terms;
  s->term_total = (i64)total;
  return GSM_OK;
}

gsm_status gsm_decode_rows(gsm_store* s, const uint32_t* rows, int64_t n_rows, int32_t k,
                           gsm_text** out) {
  *out = nullptr;
  if (!s) return set_error(GSM_ERR_VALUE, "null store");
  if (!s->term_off) return set_error(GSM_ERR_VALUE, "no dictionary on the device (gsm_store_put_dictionary)");
  if (n_rows < 0 || k < 0 || (n_rows > 0 && k > 0 && !rows)) return set_error(GSM_ERR_VALUE, "bad rows");
  gsm_text* t = new gsm_text();
  if (n_rows == 0) {
    *out = t;
    return GSM_OK;
  }
  if (k == 0) {  // zero-width rows: one empty line each
    t->bytes.assign((size_t)n_rows, '\n');
    *out = t;
    return GSM_OK;
  }
  GSM_CUDA(cudaSetDevice(s->device));
  const size_t cells = (size_t)n_rows * (size_t)k;
  u32* d_rows = nullptr;
  u64 *d_rb = nullptr, *d_pos = nullptr;
  unsigned long long* d_bad = nullptr;
  unsigned char* d_out = nullptr;
  void* tmp = nullptr;
  cudaStream_t st = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_rows);
    cudaFree(d_rb);
    cudaFree(d_pos);
    cudaFree(d_bad);
    cudaFree(d_out);
    cudaFree(tmp);
    if (st) cudaStreamDestroy(st);
  };
  auto fail = [&](cudaError_t e, const char* what) {
    cleanup();
    delete t;
    return cuda_error(e, what);
  };
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess) return fail(e, "stream");
  if ((e = cudaMalloc(&d_rows, 4 * cells)) != cudaSuccess) return fail(e, "cudaMalloc(rows)");
  if ((e = cudaMalloc(&d_rb, 8 * (size_t)n_rows)) != cudaSuccess) return fail(e, "cudaMalloc");
  if ((e = cudaMalloc(&d_pos, 8 * (size_t)n_rows)) != cudaSuccess) return fail(e, "cudaMalloc");
  if ((e = cudaMalloc(&d_bad, 8)) != cudaSuccess) return fail(e, "cudaMalloc");
  if ((e = cudaMemcpyAsync(d_rows, rows, 4 * cells, cudaMemcpyDefault, st)) != cudaSuccess) return fail(e, "H2D rows");
  if ((e = cudaMemsetAsync(d_bad, 0xFF, 8, st)) != cudaSuccess) return fail(e, "cudaMemset");
  k_row_bytes<<<grid_for(n_rows), 256, 0, st>>>(d_rows, n_rows, k, s->term_off, (u64)s->n_terms, d_rb, d_bad);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, d_rb, d_pos, n_rows, st);
  if ((e = cudaMalloc(&tmp, std::max<size_t>(tb, 4))) != cudaSuccess) return fail(e, "cudaMalloc");
  cub::DeviceScan::ExclusiveSum(tmp, tb, d_rb, d_pos, n_rows, st);
  count_launch(2);
  unsigned long long bad = 0;
  u64 last[2] = {0, 0};
  if ((e = cudaMemcpyAsync(&bad, d_bad, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return fail(e, "D2H");
  if ((e = cudaMemcpyAsync(&last[0], d_pos + n_rows - 1, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return fail(e, "D2H");
  if ((e = cudaMemcpyAsync(&last[1], d_rb + n_rows - 1, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return fail(e, "D2H");
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail(e, "decode sizes");
  if (bad != ~0ull) {
    u32 v = 0;
    cudaMemcpy(&v, d_rows + bad, 4, cudaMemcpyDeviceToHost);
    cleanup();
    delete t;
    return set_error(GSM_ERR_UNKNOWN_ID, "no node term with id " + std::to_string(v));
  }
  const u64 total = last[0] + last[1];
  if ((e = cudaMalloc(&d_out, std::max<u64>(total, 1))) != cudaSuccess) return fail(e, "cudaMalloc(text)");
  k_write_rows<<<grid_for(n_rows * 32), 256, 0, st>>>(d_rows, n_rows, k, s->term_off, s->term_bytes, d_pos, d_out);
  count_launch();
  t->bytes.resize(total);
  if (total && (e = cudaMemcpyAsync(t->bytes.data(), d_out, total, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return fail(e, "D2H text");
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail(e, "decode");
  cleanup();
  *out = t;
  return GSM_OK;
}

gsm_status gsm_text_data(const gsm_text* t, const char** data, int64_t* nbytes) {
  if (!t || !data || !nbytes) return set_error(GSM_ERR_VALUE, "bad arguments");
  *data = t->bytes.data();
  *nbytes = (int64_t)t->bytes.size();
  return GSM_OK;
}

gsm_status gsm_text_free(gsm_text* t) {
  delete t;
  return GSM_OK;
}

}  // extern "C"
