// Measurement helper (not part of the reference interface): the FP64 FMA
// throughput of this GPU, for the FP64 fraction bench.py reports beside the
// HBM roofline ("FP64 peak is not in MEASURED_PEAKS.json;
// measure it with a DFMA microbenchmark").
#include <cuda_runtime.h>
#include <cstdint>

#include "ldgb200.h"

namespace {

constexpr int kChains = 8;          // independent DFMA chains per thread (covers the latency)

__global__ void __launch_bounds__(256) dfma_kernel(int iters, double a, double b, double* out) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345e300) out[0] = s;  // keeps the chains live
}

}  // namespace

extern "C" int ldg_probe_fp64(int64_t iters, double* tflops, double* ms, void* stream) {
  if (!tflops || !ms || iters <= 0) return 2;
  cudaStream_t s = (cudaStream_t)stream;
  int nsm = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return 3;
  const int grid = nsm * 8, block = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<<<grid, block, 0, s>>>(16, 0.999999, 1e-7, out);   // warm-up
  cudaEventRecord(e0, s);
  dfma_kernel<<<grid, block, 0, s>>>((int)iters, 0.999999, 1e-7, out);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float t = 0.f;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return 3;
  *ms = t;
  *tflops = 2.0 * (double)grid * block * kChains * (double)iters / (t * 1e-3) / 1e12;
  return 0;
}
