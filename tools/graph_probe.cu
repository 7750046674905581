// Micro-benchmark of launch-sequence overheads inside one CUDA graph with B
// parallel branches (the batch-graph shape of gsm_execute_batch):
//   A: H2D 4 KiB -> K tiny kernels -> D2H 4 KiB   (current query sequence)
//   B: K+1 tiny kernels (the block copied by a kernel) -> D2H 4 KiB
//   C: K tiny kernels only
//   D: K tiny kernels, 148 x 256 threads each
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o graph_probe graph_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_tiny(unsigned* p) {
  if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}
__global__ void k_copy(const unsigned* __restrict__ s, unsigned* __restrict__ d, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = s[i];
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 14, K = argc > 2 ? atoi(argv[2]) : 3, WORDS = 1024;
  std::vector<cudaStream_t> st(B);
  for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  unsigned *h, *d, *dimg;
  CK(cudaMallocHost(&h, B * WORDS * 8));
  CK(cudaMalloc(&d, B * WORDS * 8));
  CK(cudaMalloc(&dimg, B * WORDS * 4));
  cudaEvent_t fork, e0, e1;
  std::vector<cudaEvent_t> join(B);
  CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  for (auto& j : join) CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int variant = 0; variant < 4; variant++) {
    CK(cudaStreamBeginCapture(st[0], cudaStreamCaptureModeThreadLocal));
    CK(cudaEventRecord(fork, st[0]));
    for (int b = 1; b < B; b++) CK(cudaStreamWaitEvent(st[b], fork, 0));
    for (int b = 0; b < B; b++) {
      unsigned* db = d + b * WORDS * 2;
      unsigned* hb = h + b * WORDS * 2;
      if (variant == 0) CK(cudaMemcpyAsync(db, hb, WORDS * 4, cudaMemcpyHostToDevice, st[b]));
      if (variant == 1) k_copy<<<1, 256, 0, st[b]>>>(dimg + b * WORDS, db, WORDS);
      for (int k = 0; k < K; k++) {
        if (variant == 3) k_tiny<<<148, 256, 0, st[b]>>>(db);
        else k_tiny<<<1, 32, 0, st[b]>>>(db);
      }
      if (variant <= 1) CK(cudaMemcpyAsync(hb + WORDS, db + WORDS, WORDS * 4, cudaMemcpyDeviceToHost, st[b]));
      if (b > 0) {
        CK(cudaEventRecord(join[b], st[b]));
        CK(cudaStreamWaitEvent(st[0], join[b], 0));
      }
    }
    cudaGraph_t g;
    CK(cudaStreamEndCapture(st[0], &g));
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int i = 0; i < 50; i++) CK(cudaGraphLaunch(ge, st[0]));
    CK(cudaStreamSynchronize(st[0]));
    float best = 1e9, sum = 0;
    const int R = 200;
    for (int i = 0; i < R; i++) {
      CK(cudaEventRecord(e0, st[0]));
      CK(cudaGraphLaunch(ge, st[0]));
      CK(cudaEventRecord(e1, st[0]));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
      sum += ms;
    }
    const char* names[] = {"H2D+K kernels+D2H", "copy kernel+K kernels+D2H", "K kernels", "K kernels 148x256"};
    printf("B=%d K=%d %-28s mean %.1f us  best %.1f us\n", B, K, names[variant], 1e3 * sum / R, 1e3 * best);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  // single branch sequence timing
  return 0;
}
