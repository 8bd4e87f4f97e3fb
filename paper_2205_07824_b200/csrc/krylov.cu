// Krylov vector primitives for the device GMRES (solver.py:79-174).
//
// All reductions are deterministic: a fixed grid of kRedBlocks blocks
// grid-strides the vector, reduces in a fixed warp-shuffle tree, writes one
// partial per block, and the last block to finish (atomic ticket) sums the
// partials in index order.  Results are bitwise reproducible run to run.
// Fused variants cut HBM passes: the MGS step does w -= h_i V_i and the next
// dot <V_{i+1}, w> in one sweep (3 reads + 1 write instead of 5 passes).

#include <cstdint>
#include <cuda_runtime.h>
#include "ldgb200.h"

namespace {

#ifndef LDG_RED_BLOCKS
#define LDG_RED_BLOCKS 592     // 4 x 148 SMs; config-3 solve: 1184 -> 1.49 s, 592 -> 1.40 s, 296 -> 1.81 s
#endif
constexpr int kRedBlocks = LDG_RED_BLOCKS;
constexpr int kThreads = 256;
#ifndef LDG_MULTIDOT_K
#define LDG_MULTIDOT_K 16    // measured on the config-3 solve: 8 -> 2.19 s, 16 -> 1.91 s, 32 -> 2.08 s
#endif
constexpr int kMaxK = LDG_MULTIDOT_K;  // dots per sweep in the multi-dot kernel

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block sum in fixed order; result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = l < (kThreads / 32) ? sh[l] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}

// last-block finalisation: partials[0..nparts) summed in order into *out
// (scaled by sqrt if want_sqrt); ticket lives at scratch tail.
__device__ __forceinline__ void finish(double* partials, unsigned int* ticket,
                                       int nvals, double* out, bool want_sqrt,
                                       double* sh) {
  __shared__ bool last;
  __threadfence();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int v = 0; v < nvals; ++v) {
    double s = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kThreads)
      s += partials[(size_t)v * gridDim.x + b];
    s = block_sum(s, sh);
    if (threadIdx.x == 0) out[v] = want_sqrt ? sqrt(s) : s;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

__global__ void __launch_bounds__(kThreads)
dot_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
           double* partials, unsigned int* ticket, double* out, int want_sqrt) {
  __shared__ double sh[kThreads / 32];
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride)
    s = fma(x[i], y[i], s);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  finish(partials, ticket, 1, out, want_sqrt, sh);
}

__global__ void __launch_bounds__(kThreads)
axpy_kernel(int64_t n, double a_host, const double* __restrict__ a_dev, double sign,
            const double* __restrict__ x, double* __restrict__ y) {
  const double a = a_dev ? sign * (*a_dev) : a_host;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride)
    y[i] = fma(a, x[i], y[i]);
}

__global__ void __launch_bounds__(kThreads)
div_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ den,
           double* __restrict__ y) {
  const double d = *den;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride)
    y[i] = x[i] / d;
}

// w -= h_in * vi ; partial <vnext, w>
__global__ void __launch_bounds__(kThreads)
mgs_kernel(int64_t n, const double* __restrict__ vi, const double* __restrict__ h_in,
           double* __restrict__ w, const double* __restrict__ vnext,
           double* partials, unsigned int* ticket, double* h_out) {
  __shared__ double sh[kThreads / 32];
  const double h = h_in ? *h_in : 0.0;
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    double wv = w[i];
    if (vi) {
      wv = wv - h * vi[i];        // reference: w = w - H[i,k] * V[i]
      w[i] = wv;
    }
    if (vnext) s = fma(vnext[i], wv, s);
  }
  if (!vnext) return;
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  finish(partials, ticket, 1, h_out, false, sh);
}

// up to kMaxK dots <V_i, w> per sweep; two consecutive entries per thread
// (16 B loads) when the rows are 16 B aligned, so each of the k + 1 streams
// has twice the bytes in flight per instruction
__global__ void __launch_bounds__(kThreads)
multidot_kernel(int64_t n, int k, const double* __restrict__ V, int64_t ldv,
                const double* __restrict__ w, double* partials,
                unsigned int* ticket, double* h) {
  __shared__ double sh[kThreads / 32];
  double acc[kMaxK];
#pragma unroll
  for (int r = 0; r < kMaxK; ++r) acc[r] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const bool vec = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
  if (vec) {
    const int64_t n2 = n >> 1;
    const double2* w2 = reinterpret_cast<const double2*>(w);
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n2; i += stride) {
      const double2 wv = w2[i];
#pragma unroll
      for (int r = 0; r < kMaxK; ++r)
        if (r < k) {
          const double2 v = reinterpret_cast<const double2*>(V + (int64_t)r * ldv)[i];
          acc[r] = fma(v.x, wv.x, acc[r]);
          acc[r] = fma(v.y, wv.y, acc[r]);
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const int64_t i = n - 1;
#pragma unroll
      for (int r = 0; r < kMaxK; ++r)
        if (r < k) acc[r] = fma(V[(int64_t)r * ldv + i], w[i], acc[r]);
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
      const double wv = w[i];
#pragma unroll
      for (int r = 0; r < kMaxK; ++r)
        if (r < k) acc[r] = fma(V[(int64_t)r * ldv + i], wv, acc[r]);
    }
  }
  for (int r = 0; r < k; ++r) {
    const double s = block_sum(acc[r], sh);
    if (threadIdx.x == 0) partials[(size_t)r * gridDim.x + blockIdx.x] = s;
  }
  finish(partials, ticket, k, h, false, sh);
}

// w -= sum_i h[i] V_i (i < k), optional ||w||.  Two entries per thread with
// 16 B loads, the row loop unrolled by 4 into two accumulator pairs.  The
// coefficient row in shared memory is padded by two doubles: the compiler
// reads the odd tail as a 16-B pair (compute-sanitizer memcheck).
__global__ void __launch_bounds__(kThreads)
update_kernel(int64_t n, int k, const double* __restrict__ V, int64_t ldv,
              const double* __restrict__ hcoef, double sign, double* __restrict__ w,
              double* partials, unsigned int* ticket, double* nrm) {
  extern __shared__ double hs[];
  __shared__ double sh[kThreads / 32];
  for (int r = threadIdx.x; r < k; r += kThreads) hs[r] = hcoef[r];
  __syncthreads();
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const bool vec = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
  if (vec) {
    const int64_t n2 = n >> 1;
    double2* w2 = reinterpret_cast<double2*>(w);
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n2; i += stride) {
      double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
      int r = 0;
      for (; r + 4 <= k; r += 4) {
        const double2 v0 = reinterpret_cast<const double2*>(V + (int64_t)r * ldv)[i];
        const double2 v1 = reinterpret_cast<const double2*>(V + (int64_t)(r + 1) * ldv)[i];
        const double2 v2 = reinterpret_cast<const double2*>(V + (int64_t)(r + 2) * ldv)[i];
        const double2 v3 = reinterpret_cast<const double2*>(V + (int64_t)(r + 3) * ldv)[i];
        ax = fma(hs[r], v0.x, ax);
        ay = fma(hs[r], v0.y, ay);
        bx = fma(hs[r + 1], v1.x, bx);
        by = fma(hs[r + 1], v1.y, by);
        ax = fma(hs[r + 2], v2.x, ax);
        ay = fma(hs[r + 2], v2.y, ay);
        bx = fma(hs[r + 3], v3.x, bx);
        by = fma(hs[r + 3], v3.y, by);
      }
      for (; r < k; ++r) {
        const double2 v0 = reinterpret_cast<const double2*>(V + (int64_t)r * ldv)[i];
        ax = fma(hs[r], v0.x, ax);
        ay = fma(hs[r], v0.y, ay);
      }
      double2 wv = w2[i];
      wv.x = fma(sign, ax + bx, wv.x);
      wv.y = fma(sign, ay + by, wv.y);
      w2[i] = wv;
      s = fma(wv.x, wv.x, s);
      s = fma(wv.y, wv.y, s);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const int64_t i = n - 1;
      double acc = 0.0;
      for (int r = 0; r < k; ++r) acc = fma(hs[r], V[(int64_t)r * ldv + i], acc);
      const double wv = fma(sign, acc, w[i]);
      w[i] = wv;
      s = fma(wv, wv, s);
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
      double acc = 0.0;
      for (int r = 0; r < k; ++r) acc = fma(hs[r], V[(int64_t)r * ldv + i], acc);
      const double wv = fma(sign, acc, w[i]);
      w[i] = wv;
      s = fma(wv, wv, s);
    }
  }
  if (!nrm) return;
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  finish(partials, ticket, 1, nrm, true, sh);
}

// DCGS2 (delayed classical Gram-Schmidt with reorthogonalisation): one sweep
// gives both dot sets <V_i, x> and <V_i, y> for up to kDc rows (x = the
// once-orthogonalised basis vector, y = the new Krylov vector)
#ifndef LDG_DCGS_ROWS
#define LDG_DCGS_ROWS 8
#endif
constexpr int kDc = LDG_DCGS_ROWS;    // basis rows per DCGS2 dot sweep (2 dots each)
__global__ void __launch_bounds__(kThreads)
multidot2_kernel(int64_t n, int k, const double* __restrict__ V, int64_t ldv,
                 const double* __restrict__ x, const double* __restrict__ y, double* partials,
                 unsigned int* ticket, double* hx, double* hy) {
  __shared__ double sh[kThreads / 32];
  double ax[kDc], ay[kDc];
#pragma unroll
  for (int r = 0; r < kDc; ++r) ax[r] = ay[r] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const bool vec = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(y) & 15) == 0);
  if (vec) {
    const int64_t n2 = n >> 1;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n2; i += stride) {
      const double2 xv = reinterpret_cast<const double2*>(x)[i];
      const double2 yv = reinterpret_cast<const double2*>(y)[i];
#pragma unroll
      for (int r = 0; r < kDc; ++r)
        if (r < k) {
          const double2 v = reinterpret_cast<const double2*>(V + (int64_t)r * ldv)[i];
          ax[r] = fma(v.y, xv.y, fma(v.x, xv.x, ax[r]));
          ay[r] = fma(v.y, yv.y, fma(v.x, yv.x, ay[r]));
        }
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const int64_t i = n - 1;
#pragma unroll
      for (int r = 0; r < kDc; ++r)
        if (r < k) {
          ax[r] = fma(V[(int64_t)r * ldv + i], x[i], ax[r]);
          ay[r] = fma(V[(int64_t)r * ldv + i], y[i], ay[r]);
        }
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
#pragma unroll
      for (int r = 0; r < kDc; ++r)
        if (r < k) {
          const double v = V[(int64_t)r * ldv + i];
          ax[r] = fma(v, x[i], ax[r]);
          ay[r] = fma(v, y[i], ay[r]);
        }
    }
  }
  for (int r = 0; r < k; ++r) {
    double s = block_sum(ax[r], sh);
    if (threadIdx.x == 0) partials[(size_t)r * gridDim.x + blockIdx.x] = s;
    s = block_sum(ay[r], sh);
    if (threadIdx.x == 0) partials[(size_t)(k + r) * gridDim.x + blockIdx.x] = s;
  }
  // outputs: hx[0..k) then hy[0..k) (hy = hx + k in the caller's layout is
  // not assumed: finish writes 2k values to a staging row)
  __shared__ bool last;
  __threadfence();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int v = 0; v < 2 * k; ++v) {
    double s2 = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kThreads)
      s2 += partials[(size_t)v * gridDim.x + b];
    s2 = block_sum(s2, sh);
    if (threadIdx.x == 0) (v < k ? hx[v] : hy[v - k]) = s2;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// The whole DCGS2 dot sweep in ONE launch: block (c, s) of a 2D grid takes
// basis rows [8c, 8c + 8) over column slab s, with the row chunk c varying
// fastest in launch order, so the ceil(k / 8) blocks of one slab run
// together and read that slab of x and y from DRAM once (the others hit L2;
// the chunked launches re-read x and y from DRAM per chunk).  Per-(row, slab)
// partials, summed in slab order by the last block: deterministic.
#ifndef LDG_UPD2_UNROLL
#define LDG_UPD2_UNROLL 8          // measured: 4 -> 0.989 s, 8 -> 0.964 s warm config-3 solve
#endif
constexpr int kUpd2Unroll = LDG_UPD2_UNROLL;
#ifndef LDG_DCGS_ALL
#define LDG_DCGS_ALL 1                 // A/B: 0 = one launch per 8-row chunk
#endif
constexpr int kDcSlabs = 296;          // 2 x 148 SMs
constexpr int kDcMaxK = 512;           // restart <= 511
__global__ void __launch_bounds__(kThreads)
multidot2_all_kernel(int64_t n, int k, const double* __restrict__ V, int64_t ldv,
                     const double* __restrict__ x, const double* __restrict__ y,
                     double* partials, unsigned int* ticket, double* hx, double* hy) {
  __shared__ double red[2 * kDc][kThreads / 32];
  const int c = blockIdx.x, slab = blockIdx.y, nslab = gridDim.y;
  const int r0 = c * kDc, kk = min(kDc, k - r0);
  double ax[kDc], ay[kDc];
#pragma unroll
  for (int r = 0; r < kDc; ++r) ax[r] = ay[r] = 0.0;
  const int64_t n2 = n >> 1;
  const int64_t per = (n2 + nslab - 1) / nslab;
  const int64_t i0 = (int64_t)slab * per, i1 = min(n2, i0 + per);
  const double* Vc = V + (int64_t)r0 * ldv;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += kThreads) {
    const double2 xv = reinterpret_cast<const double2*>(x)[i];
    const double2 yv = reinterpret_cast<const double2*>(y)[i];
#pragma unroll
    for (int r = 0; r < kDc; ++r)
      if (r < kk) {
        const double2 v = reinterpret_cast<const double2*>(Vc + (int64_t)r * ldv)[i];
        ax[r] = fma(v.y, xv.y, fma(v.x, xv.x, ax[r]));
        ay[r] = fma(v.y, yv.y, fma(v.x, yv.x, ay[r]));
      }
  }
  if ((n & 1) && slab == nslab - 1 && threadIdx.x == 0) {
    const int64_t i = n - 1;
#pragma unroll
    for (int r = 0; r < kDc; ++r)
      if (r < kk) {
        ax[r] = fma(Vc[(int64_t)r * ldv + i], x[i], ax[r]);
        ay[r] = fma(Vc[(int64_t)r * ldv + i], y[i], ay[r]);
      }
  }
  // all 2 kk sums of the block at once: warp shuffles, then one pass over warps
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < kDc; ++r) {
    double a = ax[r], b = ay[r];
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) {
      red[r][warp] = a;
      red[kDc + r][warp] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * kDc) {
    const int v = threadIdx.x, r = v % kDc;
    if (r < kk) {
      double t = 0.0;
      for (int w2 = 0; w2 < kThreads / 32; ++w2) t += red[v][w2];
      const int row = (v < kDc ? 0 : k) + r0 + r;            // x rows [0, k), y rows [k, 2k)
      partials[(size_t)row * nslab + slab] = t;
    }
  }
  (void)ticket; (void)hx; (void)hy;
}

// the per-row sums of multidot2_all_kernel's partials: one warp per row
// (fixed lane / slab assignment and shuffle tree: deterministic)
__global__ void __launch_bounds__(kThreads)
multidot2_finish_kernel(int k, int nslab, const double* __restrict__ partials, double* hx,
                        double* hy) {
  const int v = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (v >= 2 * k) return;
  double s = 0.0;
  for (int b = lane; b < nslab; b += 32) s += partials[(size_t)v * nslab + b];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) (v < k ? hx[v] : hy[v - k]) = s;
}

// y = x / *den where *den > thr, untouched otherwise (also for a NaN den):
// the DCGS2 normalisation of the next basis vector without a host round
// trip; the host sees den with the next dot sweep and handles breakdown
__global__ void div_guarded_kernel(int64_t n, const double* __restrict__ x,
                                   const double* __restrict__ den, double thr,
                                   double* __restrict__ y) {
  const double d = *den;
  if (!(d > thr)) return;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride)
    y[i] = x[i] / d;
}

// DCGS2 update, one sweep over V_0..V_{m-1}: the final basis vector
// vf = (v - sum_j s_j V_j) * inv_alpha (written over v) and the projected
// Krylov vector w1 = (w - sum_j t_j V_j - gamma vf) * inv_alpha (into out),
// with ||w1|| fused.
__global__ void __launch_bounds__(kThreads)
update2_kernel(int64_t n, int m, const double* __restrict__ V, int64_t ldv,
               const double* __restrict__ sc, const double* __restrict__ tc, double* v,
               const double* __restrict__ w, double* __restrict__ out, double inv_alpha,
               double gamma, double* partials, unsigned int* ticket, double* nrm) {
  extern __shared__ double cs[];
  __shared__ double sh[kThreads / 32];
  for (int r = threadIdx.x; r < m; r += kThreads) {
    cs[r] = sc[r];
    cs[m + r] = tc[r];
  }
  __syncthreads();
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const bool vec = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(v) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(w) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  int64_t i0 = 0;
  if (vec) {                        // two entries per thread, 16-B loads
    const int64_t n2 = n >> 1;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n2; i += stride) {
      double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
      // LDG_UPD2_UNROLL rows in flight per thread (memory-level parallelism
      // of the m-row sweep); the accumulation order over r is unchanged
#pragma unroll kUpd2Unroll
      for (int r = 0; r < m; ++r) {
        const double2 vr = reinterpret_cast<const double2*>(V + (int64_t)r * ldv)[i];
        ax = fma(cs[r], vr.x, ax);
        ay = fma(cs[r], vr.y, ay);
        bx = fma(cs[m + r], vr.x, bx);
        by = fma(cs[m + r], vr.y, by);
      }
      double2 vv = reinterpret_cast<double2*>(v)[i];
      const double2 wv = reinterpret_cast<const double2*>(w)[i];
      vv.x = (vv.x - ax) * inv_alpha;
      vv.y = (vv.y - ay) * inv_alpha;
      reinterpret_cast<double2*>(v)[i] = vv;
      double2 o;
      o.x = (wv.x - bx - gamma * vv.x) * inv_alpha;
      o.y = (wv.y - by - gamma * vv.y) * inv_alpha;
      reinterpret_cast<double2*>(out)[i] = o;
      acc = fma(o.x, o.x, acc);
      acc = fma(o.y, o.y, acc);
    }
    i0 = n2 * 2;                    // odd tail below (one element)
  }
  for (int64_t i = i0 + (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    int r = 0;
    for (; r + 2 <= m; r += 2) {
      const double v0 = V[(int64_t)r * ldv + i], v1 = V[(int64_t)(r + 1) * ldv + i];
      a0 = fma(cs[r], v0, a0);
      b0 = fma(cs[m + r], v0, b0);
      a1 = fma(cs[r + 1], v1, a1);
      b1 = fma(cs[m + r + 1], v1, b1);
    }
    if (r < m) {
      const double v0 = V[(int64_t)r * ldv + i];
      a0 = fma(cs[r], v0, a0);
      b0 = fma(cs[m + r], v0, b0);
    }
    const double vf = (v[i] - (a0 + a1)) * inv_alpha;
    v[i] = vf;
    const double w1 = (w[i] - (b0 + b1) - gamma * vf) * inv_alpha;
    out[i] = w1;
    acc = fma(w1, w1, acc);
  }
  if (!nrm) return;
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
  finish(partials, ticket, 1, nrm, true, sh);
}

constexpr int kScratchRows = kMaxK > 2 * kDc ? kMaxK : 2 * kDc;
inline unsigned int* ticket_of(double* scratch) {
  return reinterpret_cast<unsigned int*>(scratch + (size_t)kRedBlocks * kScratchRows);
}

inline int grid_for(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  return (int)(g < kRedBlocks ? (g < 1 ? 1 : g) : kRedBlocks);
}

inline int rc() { return cudaGetLastError() == cudaSuccess ? 0 : 3; }

}  // namespace

extern "C" {

int64_t ldg_reduce_scratch_doubles(void) {
  return (int64_t)kRedBlocks * kScratchRows + 8 + (int64_t)2 * kDcMaxK * kDcSlabs;
}

// NOTE: reductions always launch the full kRedBlocks grid so partial counts
// (and therefore rounding) do not depend on n.
int ldg_dot(int64_t n, const double* x, const double* y, double* scratch,
            double* out, void* stream) {
  dot_kernel<<<kRedBlocks, kThreads, 0, (cudaStream_t)stream>>>(
      n, x, y, scratch, ticket_of(scratch), out, 0);
  return rc();
}

int ldg_nrm2(int64_t n, const double* x, double* scratch, double* out, void* stream) {
  dot_kernel<<<kRedBlocks, kThreads, 0, (cudaStream_t)stream>>>(
      n, x, x, scratch, ticket_of(scratch), out, 1);
  return rc();
}

int ldg_axpy(int64_t n, double a_host, const double* a_dev, double sign,
             const double* x, double* y, void* stream) {
  axpy_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, a_host, a_dev,
                                                                  sign, x, y);
  return rc();
}

int ldg_div_scalar_guarded(int64_t n, const double* x, const double* den, double thr,
                           double* y, void* stream) {
  div_guarded_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, den, thr, y);
  return rc();
}

int ldg_div_scalar(int64_t n, const double* x, const double* den, double* y,
                   void* stream) {
  div_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, den, y);
  return rc();
}

int ldg_mgs_step(int64_t n, const double* vi, const double* h_in, double* w,
                 const double* vnext, double* scratch, double* h_out, void* stream) {
  mgs_kernel<<<kRedBlocks, kThreads, 0, (cudaStream_t)stream>>>(
      n, vi, h_in, w, vnext, scratch, ticket_of(scratch), h_out);
  return rc();
}

int ldg_cgs_dots(int64_t n, int k, const double* V, int64_t ldv, const double* w,
                 double* scratch, double* h, void* stream) {
  for (int r0 = 0; r0 < k; r0 += kMaxK) {
    const int kk = k - r0 < kMaxK ? k - r0 : kMaxK;
    multidot_kernel<<<kRedBlocks, kThreads, 0, (cudaStream_t)stream>>>(
        n, kk, V + (int64_t)r0 * ldv, ldv, w, scratch, ticket_of(scratch), h + r0);
    if (rc()) return 3;
  }
  return 0;
}

int ldg_cgs_update(int64_t n, int k, const double* V, int64_t ldv, const double* h,
                   double* w, double* scratch, double* nrm_out, void* stream) {
  update_kernel<<<kRedBlocks, kThreads, (k + 2) * sizeof(double), (cudaStream_t)stream>>>(
      n, k, V, ldv, h, -1.0, w, scratch, ticket_of(scratch), nrm_out);
  return rc();
}

int ldg_dcgs_dots(int64_t n, int k, const double* V, int64_t ldv, const double* x,
                  const double* y, double* scratch, double* hx, double* hy, void* stream) {
  const bool vec = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(y) & 15) == 0);
  if (LDG_DCGS_ALL && k > 0 && k <= kDcMaxK && vec && n >= 2 * kDcSlabs) {
    double* part = scratch + (size_t)kRedBlocks * kScratchRows + 8;
    const dim3 grid((unsigned)((k + kDc - 1) / kDc), kDcSlabs);
    multidot2_all_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        n, k, V, ldv, x, y, part, ticket_of(scratch), hx, hy);
    const int wpb = kThreads / 32;
    multidot2_finish_kernel<<<(2 * k + wpb - 1) / wpb, kThreads, 0, (cudaStream_t)stream>>>(
        k, kDcSlabs, part, hx, hy);
    return rc();
  }
  for (int r0 = 0; r0 < k; r0 += kDc) {
    const int kk = k - r0 < kDc ? k - r0 : kDc;
    multidot2_kernel<<<kRedBlocks, kThreads, 0, (cudaStream_t)stream>>>(
        n, kk, V + (int64_t)r0 * ldv, ldv, x, y, scratch, ticket_of(scratch), hx + r0, hy + r0);
    if (rc()) return 3;
  }
  return 0;
}

int ldg_dcgs_update(int64_t n, int m, const double* V, int64_t ldv, const double* s,
                    const double* t, double* v, const double* w, double* out,
                    double inv_alpha, double gamma, double* scratch, double* nrm_out,
                    void* stream) {
  update2_kernel<<<kRedBlocks, kThreads, (2 * (m > 0 ? m : 1) + 2) * sizeof(double),
                   (cudaStream_t)stream>>>(n, m, V, ldv, s, t, v, w, out, inv_alpha, gamma,
                                           scratch, ticket_of(scratch), nrm_out);
  return rc();
}

int ldg_combine(int64_t n, int k, const double* Z, int64_t ldz, const double* y,
                double* x, void* stream) {
  update_kernel<<<grid_for(n), kThreads, (k + 2) * sizeof(double), (cudaStream_t)stream>>>(
      n, k, Z, ldz, y, 1.0, x, nullptr, nullptr, nullptr);
  return rc();
}

}  // extern "C"
