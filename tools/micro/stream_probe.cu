// Streaming-read probe: how fast can CTAs that each stream one contiguous per-subdomain
// block (like the packed GEMV operators) read HBM?  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int WARPS, int BATCH>
__global__ void __launch_bounds__(WARPS * 32) k_stream(const double2* __restrict__ a, size_t per_cta, double* out) {
  const double2* p = a + (size_t)blockIdx.x * per_cta;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0;
  const size_t chunk = (size_t)32 * BATCH;
  for (size_t off = (size_t)warp * chunk; off + chunk <= per_cta; off += (size_t)WARPS * chunk) {
    double2 m[BATCH];
#pragma unroll
    for (int u = 0; u < BATCH; ++u) m[u] = __ldcs(p + off + u * 32 + lane);
#pragma unroll
    for (int u = 0; u < BATCH; ++u) acc += m[u].x * m[u].y;
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int WARPS, int BATCH>
void run(const double2* a, int ctas, size_t per_cta, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) k_stream<WARPS, BATCH><<<ctas, WARPS * 32>>>(a, per_cta, out);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) k_stream<WARPS, BATCH><<<ctas, WARPS * 32>>>(a, per_cta, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)ctas * per_cta * 16;
  printf("ctas %5d warps %d batch %2d: %7.2f us  %7.1f GB/s\n", ctas, WARPS, BATCH, 1000 * ms / reps,
         bytes / (ms / reps * 1e-3) / 1e9);
}

int main() {
  const size_t per = 8704;  // double2 per subdomain (~139 KB, the precond operator)
  double2* a;
  double* out;
  cudaMalloc(&a, (size_t)4096 * per * 16);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, (size_t)4096 * per * 16);
  run<4, 8>(a, 1024, per, out);
  run<4, 16>(a, 1024, per, out);
  run<8, 8>(a, 1024, per, out);
  run<2, 8>(a, 1024, per, out);
  run<4, 8>(a, 2048, per / 2, out);
  run<4, 8>(a, 4096, per, out);
  run<8, 16>(a, 4096, per, out);
  return 0;
}
