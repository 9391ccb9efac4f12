// Launch cost of a kernel versus the size of its __grid_constant__ parameter
// block (tools/, not product): K1 passes ~22 KB of tables as parameters.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_params mb_params.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int BYTES>
struct __align__(16) Blob { unsigned char b[BYTES]; };

template <int BYTES>
__global__ void k_empty(const __grid_constant__ Blob<BYTES> p, int* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && out) *out = p.b[BYTES - 1];
}

template <int BYTES>
void run(int grid) {
  static Blob<BYTES> blob{};
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 10; ++i) k_empty<BYTES><<<grid, 256, 0, st>>>(blob, nullptr);
  cudaStreamSynchronize(st);
  const int n = 200;
  cudaEventRecord(e0, st);
  for (int i = 0; i < n; ++i) k_empty<BYTES><<<grid, 256, 0, st>>>(blob, nullptr);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // graph of one launch, replayed
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  k_empty<BYTES><<<grid, 256, 0, st>>>(blob, nullptr);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEventRecord(e0, st);
  for (int i = 0; i < n; ++i) cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float gms;
  cudaEventElapsedTime(&gms, e0, e1);
  printf("{\"param_bytes\":%d,\"grid\":%d,\"us_per_launch_stream\":%.2f,\"us_per_launch_graph\":%.2f}\n", BYTES, grid,
         ms * 1e3 / n, gms * 1e3 / n);
}

int main() {
  for (int grid : {148, 296, 444}) {
    run<16>(grid);
    run<4096>(grid);
    run<8192>(grid);
    run<16384>(grid);
    run<22016>(grid);
    run<32000>(grid);
  }
  return 0;
}
