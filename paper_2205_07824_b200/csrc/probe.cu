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

// FP64 tensor-core probe: mma.sync m8n8k4 f64 (DMMA), kChains independent
// accumulators per warp; with MIX also kChains DFMA chains per thread in the
// same loop, to see whether the tensor path and the FP64 pipe add up.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <bool MIX>
__global__ void __launch_bounds__(256) dmma_kernel(int iters, double a, double b, double* out) {
  double acc[kChains][2], x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    acc[c][0] = acc[c][1] = threadIdx.x * 1e-9 + c;
    x[c] = c;
  }
  const double av = a + threadIdx.x * 1e-12, bv = b - threadIdx.x * 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      dmma(acc[c], av, bv);
      if (MIX) x[c] = fma(x[c], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c][0] + acc[c][1] + x[c];
  if (s == 1.2345e300) out[0] = s;
}

}  // namespace

// mode 0: DFMA; 1: DMMA (flops = 2 * 8*8*4 per warp-instruction); 2: both
// in one loop (tflops = the sum).  ms = the timed launch.
extern "C" int ldg_probe_fp64_mode(int mode, int64_t iters, double* tflops, double* ms,
                                   void* stream) {
  if (!tflops || !ms || iters <= 0 || mode < 0 || mode > 2) return 2;
  cudaStream_t s = (cudaStream_t)stream;
  int nsm = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return 3;
  const int grid = nsm * 8, block = 256;
  auto launch = [&](int it) {
    if (mode == 0) dfma_kernel<<<grid, block, 0, s>>>(it, 0.999999, 1e-7, out);
    else if (mode == 1) dmma_kernel<false><<<grid, block, 0, s>>>(it, 0.999999, 1e-7, out);
    else dmma_kernel<true><<<grid, block, 0, s>>>(it, 0.999999, 1e-7, out);
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch(16);
  cudaEventRecord(e0, s);
  launch((int)iters);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float t = 0.f;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return 3;
  *ms = t;
  const double warps = (double)grid * block / 32.0;
  const double dfma = 2.0 * (double)grid * block * kChains * (double)iters;
  const double dmma_f = 2.0 * 256.0 * warps * kChains * (double)iters;
  const double fl = mode == 0 ? dfma : (mode == 1 ? dmma_f : dfma + dmma_f);
  *tflops = fl / (t * 1e-3) / 1e12;
  return 0;
}

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
