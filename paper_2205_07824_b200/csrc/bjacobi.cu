// Element block-Jacobi preconditioner (solver.py:291-346, driver.py:119-142).
//
// Build = coloured unit probes through the tangent operator (host loop over
// colours x block directions, each a device matvec) + ldg_bj_extract, then
// ldg_bj_invert: one CTA per element block runs Gauss-Jordan with partial
// pivoting in shared memory.  Its pivots are exactly the LU pivots of
// scipy.linalg.lu_factor, so the reference's regularisation rule
// (|pivot| < 1e-14 max(1, max|A|) or non-finite -> A + 1e-12 I,
// solver.py:336-345) is applied to the same test.  The explicit inverse is
// stored transposed so the apply (a batched GEMV, HBM-bound on the block
// matrices) reads it fully coalesced.

#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>
#include "ldgb200.h"
#include "nvtx.cuh"

namespace {

constexpr int kInvThreads = 256;
constexpr int kMaxSmemBs = 160;          // in-shared-memory inversion limit

__global__ void probe_kernel(int bs, const int32_t* __restrict__ members,
                             int64_t nm, int k, double* __restrict__ v) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nm) v[(int64_t)members[t] * bs + k] = 1.0;
}

__global__ void extract_kernel(int bs, const int32_t* __restrict__ members,
                               int64_t nm, int k, const double* __restrict__ col,
                               double* __restrict__ mats) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nm * bs) return;
  const int64_t b = members[t / bs];
  const int row = (int)(t % bs);
  mats[(b * bs + row) * bs + k] = col[b * bs + row];
}

__device__ double block_max_abs(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double r = threadIdx.x < kInvThreads / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
    if (threadIdx.x == 0) red[0] = r;
  }
  __syncthreads();
  const double out = red[0];
  __syncthreads();
  return out;
}

// In-place Gauss-Jordan with partial pivoting; returns false if a pivot
// fails the reference threshold.
__device__ bool gauss_jordan(double* A, int bs, int* perm, double thr,
                             double* red, int* ipiv) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int c = 0; c < bs; ++c) {
    // pivot search over rows c..bs-1 (first max, like LAPACK idamax)
    if (threadIdx.x < 32) {
      double best = -1.0;
      int br = c;
      for (int r = c + threadIdx.x; r < bs; r += 32) {
        const double a = fabs(A[r * bs + c]);
        if (a > best) { best = a; br = r; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int orr = __shfl_xor_sync(0xffffffffu, br, o);
        if (ob > best || (ob == best && orr < br)) { best = ob; br = orr; }
      }
      if (threadIdx.x == 0) *ipiv = br;
    }
    __syncthreads();
    const int p = *ipiv;
    if (threadIdx.x == 0) perm[c] = p;
    if (p != c)
      for (int k = threadIdx.x; k < bs; k += kInvThreads) {
        const double t = A[c * bs + k];
        A[c * bs + k] = A[p * bs + k];
        A[p * bs + k] = t;
      }
    __syncthreads();
    const double piv = A[c * bs + c];
    if (threadIdx.x == 0 && (!(fabs(piv) >= thr) || !isfinite(piv))) bad = 1;
    const double inv = 1.0 / piv;
    __syncthreads();
    for (int k = threadIdx.x; k < bs; k += kInvThreads)
      A[c * bs + k] = (k == c) ? inv : A[c * bs + k] * inv;
    __syncthreads();
    if (kInvThreads % bs == 0) {
      // fixed column per thread, rows strided: no integer division per entry
      const int k = threadIdx.x % bs, rstep = kInvThreads / bs;
      if (k != c) {
        const double ack = A[c * bs + k];
        for (int r = threadIdx.x / bs; r < bs; r += rstep)
          if (r != c) A[r * bs + k] = fma(-A[r * bs + c], ack, A[r * bs + k]);
      }
    } else {
      for (int t = threadIdx.x; t < bs * bs; t += kInvThreads) {
        const int r = t / bs, k = t % bs;
        if (r == c) continue;
        const double f = A[r * bs + c];
        if (k == c) continue;
        A[r * bs + k] = fma(-f, A[c * bs + k], A[r * bs + k]);
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < bs; r += kInvThreads)
      if (r != c) A[r * bs + c] = -A[r * bs + c] * inv;
    __syncthreads();
  }
  // undo the row interchanges as column interchanges, last first
  for (int c = bs - 1; c >= 0; --c) {
    const int p = perm[c];
    if (p != c)
      for (int r = threadIdx.x; r < bs; r += kInvThreads) {
        const double t = A[r * bs + c];
        A[r * bs + c] = A[r * bs + p];
        A[r * bs + p] = t;
      }
    __syncthreads();
  }
  return bad == 0;
}

__global__ void __launch_bounds__(kInvThreads)
invert_kernel(int bs, const double* __restrict__ mats, double* __restrict__ inv_t,
              int32_t* __restrict__ shifted) {
  extern __shared__ double A[];
  __shared__ double red[kInvThreads / 32];
  __shared__ int perm[kMaxSmemBs];
  __shared__ int ipiv;
  const int64_t b = blockIdx.x;
  const double* M = mats + b * bs * bs;
  double amax = 0.0;
  for (int t = threadIdx.x; t < bs * bs; t += kInvThreads) {
    A[t] = M[t];
    amax = fmax(amax, fabs(A[t]));
  }
  amax = block_max_abs(amax, red);
  const double thr = 1e-14 * fmax(1.0, amax);
  bool ok = gauss_jordan(A, bs, perm, thr, red, &ipiv);
  if (!ok) {
    // solver.py:343: A + 1e-12 I, factor without further checks
    for (int t = threadIdx.x; t < bs * bs; t += kInvThreads)
      A[t] = M[t] + ((t / bs) == (t % bs) ? 1e-12 : 0.0);
    __syncthreads();
    gauss_jordan(A, bs, perm, 0.0, red, &ipiv);
  }
  if (threadIdx.x == 0 && shifted) shifted[b] = ok ? 0 : 1;
  double* O = inv_t + b * bs * bs;
  for (int t = threadIdx.x; t < bs * bs; t += kInvThreads) {
    const int r = t / bs, c = t % bs;
    O[c * bs + r] = A[t];
  }
}

// Blocks beyond the shared-memory limit (NS hex p=3: 320 x 320 = 800 KB):
// the same Gauss-Jordan with partial pivoting, one CTA per block, on a
// global (L2-resident) working copy W.  Per column: warp-0 pivot search (first
// max, like idamax), row swap, pivot-row scaling, the rank-1 update with a
// fixed column per thread (the multiplier A[r][c] is a warp broadcast, the
// row segment is coalesced) and the pivot-column update.  Same pivots and
// the same regularisation rule as invert_kernel.
constexpr int kBigThreads = 512;

__device__ bool gauss_jordan_global(double* A, int bs, int* perm, double thr, int* ipiv) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int c = 0; c < bs; ++c) {
    if (threadIdx.x < 32) {
      double best = -1.0;
      int br = c;
      for (int r = c + threadIdx.x; r < bs; r += 32) {
        const double a = fabs(A[(size_t)r * bs + c]);
        if (a > best) { best = a; br = r; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int orr = __shfl_xor_sync(0xffffffffu, br, o);
        if (ob > best || (ob == best && orr < br)) { best = ob; br = orr; }
      }
      if (threadIdx.x == 0) *ipiv = br;
    }
    __syncthreads();
    const int p = *ipiv;
    if (threadIdx.x == 0) perm[c] = p;
    if (p != c)
      for (int k = threadIdx.x; k < bs; k += kBigThreads) {
        const double t = A[(size_t)c * bs + k];
        A[(size_t)c * bs + k] = A[(size_t)p * bs + k];
        A[(size_t)p * bs + k] = t;
      }
    __syncthreads();
    const double piv = A[(size_t)c * bs + c];
    if (threadIdx.x == 0 && (!(fabs(piv) >= thr) || !isfinite(piv))) bad = 1;
    const double inv = 1.0 / piv;
    __syncthreads();
    for (int k = threadIdx.x; k < bs; k += kBigThreads)
      A[(size_t)c * bs + k] = (k == c) ? inv : A[(size_t)c * bs + k] * inv;
    __syncthreads();
    for (int k = threadIdx.x; k < bs; k += kBigThreads) {
      if (k == c) continue;
      const double ack = A[(size_t)c * bs + k];
      for (int r = 0; r < bs; ++r)
        if (r != c) A[(size_t)r * bs + k] = fma(-A[(size_t)r * bs + c], ack, A[(size_t)r * bs + k]);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < bs; r += kBigThreads)
      if (r != c) A[(size_t)r * bs + c] = -A[(size_t)r * bs + c] * inv;
    __syncthreads();
  }
  for (int c = bs - 1; c >= 0; --c) {
    const int p = perm[c];
    if (p != c)
      for (int r = threadIdx.x; r < bs; r += kBigThreads) {
        const double t = A[(size_t)r * bs + c];
        A[(size_t)r * bs + c] = A[(size_t)r * bs + p];
        A[(size_t)r * bs + p] = t;
      }
    __syncthreads();
  }
  return bad == 0;
}

__global__ void __launch_bounds__(kBigThreads)
invert_global_kernel(int bs, int64_t b0, const double* __restrict__ mats, double* __restrict__ work,
                     double* __restrict__ inv_t, int32_t* __restrict__ shifted, int* __restrict__ perms) {
  __shared__ double red[kBigThreads / 32];
  __shared__ int ipiv;
  const int64_t b = b0 + blockIdx.x;
  const size_t n2 = (size_t)bs * bs;
  const double* M = mats + b * n2;
  double* A = work + blockIdx.x * n2;
  int* perm = perms + (size_t)blockIdx.x * bs;
  double amax = 0.0;
  for (size_t t = threadIdx.x; t < n2; t += kBigThreads) {
    A[t] = M[t];
    amax = fmax(amax, fabs(A[t]));
  }
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  if (threadIdx.x < 32) {
    double r = threadIdx.x < kBigThreads / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
    if (threadIdx.x == 0) red[0] = r;
  }
  __syncthreads();
  const double thr = 1e-14 * fmax(1.0, red[0]);
  const bool ok = gauss_jordan_global(A, bs, perm, thr, &ipiv);
  if (!ok) {
    for (size_t t = threadIdx.x; t < n2; t += kBigThreads)
      A[t] = M[t] + ((t / bs) == (t % bs) ? 1e-12 : 0.0);
    __syncthreads();
    gauss_jordan_global(A, bs, perm, 0.0, &ipiv);
  }
  if (threadIdx.x == 0 && shifted) shifted[b] = ok ? 0 : 1;
  double* O = inv_t + b * n2;
  for (size_t t = threadIdx.x; t < n2; t += kBigThreads) {
    const size_t r = t / bs, c = t % bs;
    O[c * bs + r] = A[t];
  }
}

// z_b = inv_b r_b with inv stored transposed: thread i reads column i of
// inv_t rows (coalesced), r_b from shared memory.
__global__ void __launch_bounds__(256)
bj_apply_kernel(int64_t nblk, int bs, const double* __restrict__ inv_t,
                const double* __restrict__ r, double* __restrict__ z) {
  extern __shared__ double rs[];
  const int per = blockDim.x / bs;                 // blocks per CTA
  const int slot = threadIdx.x / bs, i = threadIdx.x % bs;
  const int64_t b = (int64_t)blockIdx.x * per + slot;
  const bool active = slot < per && b < nblk;
  if (active) rs[slot * bs + i] = r[b * bs + i];
  __syncthreads();
  if (!active) return;
  const double* It = inv_t + b * bs * bs;
  double acc = 0.0;
  for (int j = 0; j < bs; ++j) acc = fma(__ldg(It + (int64_t)j * bs + i), rs[slot * bs + j], acc);
  z[b * bs + i] = acc;
}

// large blocks: one CTA per block, threads stride rows
__global__ void __launch_bounds__(256)
bj_apply_big_kernel(int bs, const double* __restrict__ inv_t,
                    const double* __restrict__ r, double* __restrict__ z) {
  extern __shared__ double rs[];
  const int64_t b = blockIdx.x;
  for (int j = threadIdx.x; j < bs; j += blockDim.x) rs[j] = r[b * bs + j];
  __syncthreads();
  const double* It = inv_t + b * bs * bs;
  for (int i = threadIdx.x; i < bs; i += blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < bs; ++j) acc = fma(__ldg(It + (int64_t)j * bs + i), rs[j], acc);
    z[b * bs + i] = acc;
  }
}

// exact keys of the blocks' bit patterns (class detection): two wrapping
// 64-bit sums of bits(M[t]) * odd(t), odd() a position hash, so identical
// blocks give identical keys whatever the reduction order
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return (z ^ (z >> 31)) | 1ull;
}

__global__ void __launch_bounds__(256)
block_hash_kernel(int bs, const double* __restrict__ mats, unsigned long long* __restrict__ keys) {
  __shared__ unsigned long long s0[256], s1[256];
  const int64_t b = blockIdx.x;
  const int64_t n2 = (int64_t)bs * bs;
  const unsigned long long* M = reinterpret_cast<const unsigned long long*>(mats + b * n2);
  unsigned long long h0 = 0, h1 = 0;
  for (int64_t t = threadIdx.x; t < n2; t += blockDim.x) {
    const unsigned long long v = M[t];
    h0 += v * mix64((uint64_t)t);
    h1 += (v ^ (v >> 29)) * mix64((uint64_t)t + 0x1234567ull);
  }
  s0[threadIdx.x] = h0;
  s1[threadIdx.x] = h1;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s0[threadIdx.x] += s0[threadIdx.x + o];
      s1[threadIdx.x] += s1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    keys[2 * b] = s0[0];
    keys[2 * b + 1] = s1[0];
  }
}

// every block equal (bit for bit) to its class representative?  *bad = 1 if not
__global__ void __launch_bounds__(256)
class_verify_kernel(int bs, const double* __restrict__ mats, const int64_t* __restrict__ rep,
                    int* __restrict__ bad) {
  const int64_t b = blockIdx.x, r = rep[b];
  if (r == b) return;
  const int64_t n2 = (int64_t)bs * bs;
  const unsigned long long* A = reinterpret_cast<const unsigned long long*>(mats + b * n2);
  const unsigned long long* B = reinterpret_cast<const unsigned long long*>(mats + r * n2);
  int diff = 0;
  for (int64_t t = threadIdx.x; t < n2; t += blockDim.x) diff |= A[t] != B[t];
  if (__syncthreads_or(diff) && threadIdx.x == 0) *bad = 1;
}

// class-shared blocks (structured meshes: interior elements of one geometry
// class have bit-identical blocks): a tile = up to kTileE elements of one
// class; thread i owns output row i and reuses each inverse entry
// inv_t[cls][j][i] (one L1 / L2 load) for the tile's elements, whose r rows
// sit in shared memory as [j][element] (16-B broadcast reads of 2 elements)
constexpr int kTileE = 16;
constexpr int kTileS = kTileE + 2;      // row stride: 16-B aligned rows, 4-way (not 32-way) store conflicts
__global__ void __launch_bounds__(256)
bj_apply_tiles_kernel(int bs, const double* __restrict__ inv_t, const int32_t* __restrict__ tile_cls,
                      const int32_t* __restrict__ tile_el, const double* __restrict__ r,
                      double* __restrict__ z) {
  extern __shared__ __align__(16) double rt[];                // [j][kTileS]
  const int64_t t = blockIdx.x;
  const int32_t* els = tile_el + t * kTileE;
  for (int x = threadIdx.x; x < kTileE * bs; x += blockDim.x) {
    const int e = x / bs, j = x % bs;                          // coalesced along j
    const int32_t el = els[e];
    rt[j * kTileS + e] = el >= 0 ? r[(int64_t)el * bs + j] : 0.0;
  }
  __syncthreads();
  const double* It = inv_t + (int64_t)tile_cls[t] * bs * bs;
  for (int i = threadIdx.x; i < bs; i += blockDim.x) {
    double acc[kTileE];
#pragma unroll
    for (int e = 0; e < kTileE; ++e) acc[e] = 0.0;
    for (int j = 0; j < bs; ++j) {
      const double a = __ldg(It + (int64_t)j * bs + i);
      const double2* rj = reinterpret_cast<const double2*>(rt + j * kTileS);
#pragma unroll
      for (int e2 = 0; e2 < kTileE / 2; ++e2) {
        const double2 v = rj[e2];
        acc[2 * e2] = fma(a, v.x, acc[2 * e2]);
        acc[2 * e2 + 1] = fma(a, v.y, acc[2 * e2 + 1]);
      }
    }
#pragma unroll
    for (int e = 0; e < kTileE; ++e) {
      const int32_t el = els[e];
      if (el >= 0) z[(int64_t)el * bs + i] = acc[e];
    }
  }
}

// packed (u | q | w) <-> element-major block order (driver.py:128-142):
// dst[i] = src[idx[i]] and dst[idx[i]] = src[i]
__global__ void gather_kernel(int64_t n, const int64_t* __restrict__ idx,
                              const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

__global__ void scatter_kernel(int64_t n, const int64_t* __restrict__ idx,
                               const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[idx[i]] = src[i];
}

inline int rc() { return cudaGetLastError() == cudaSuccess ? 0 : 3; }

inline unsigned grid_for(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (unsigned)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

}  // namespace

extern "C" {

int ldg_bj_probe_vector(int64_t nblk, int bs, const int32_t* members, int64_t nm,
                        int k, double* v, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(v, 0, (size_t)nblk * bs * sizeof(double), s) != cudaSuccess) return 3;
  if (nm > 0) probe_kernel<<<(unsigned)((nm + 255) / 256), 256, 0, s>>>(bs, members, nm, k, v);
  return rc();
}

int ldg_bj_extract(int bs, const int32_t* members, int64_t nm, int k,
                   const double* col, double* mats, void* stream) {
  const int64_t n = nm * bs;
  if (n > 0)
    extract_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        bs, members, nm, k, col, mats);
  return rc();
}

// global-memory Gauss-Jordan (any block size; ldg_bj_invert takes it for
// blocks beyond the shared-memory limit), a bounded number of blocks at a
// time so one wave's working copies stay L2-resident
int ldg_bj_invert_global(int64_t nblk, int bs, const double* mats, double* inv_t,
                         int32_t* shifted, void* stream) {
  NvtxRange nvtx_("ldg_bj_invert_global");
  if (bs < 1 || nblk < 0) return 2;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t chunk = std::min<int64_t>(nblk, 2 * (int64_t)nsm);
  if (chunk <= 0) return 0;
  double* work = nullptr;
  int* perms = nullptr;
  const size_t n2 = (size_t)bs * bs;
  if (cudaMallocAsync(&work, chunk * n2 * sizeof(double), s) != cudaSuccess) return 3;
  if (cudaMallocAsync(&perms, chunk * bs * sizeof(int), s) != cudaSuccess) return 3;
  for (int64_t b0 = 0; b0 < nblk; b0 += chunk) {
    const int64_t nb = std::min(chunk, nblk - b0);
    invert_global_kernel<<<(unsigned)nb, kBigThreads, 0, s>>>(bs, b0, mats, work, inv_t,
                                                              shifted, perms);
  }
  cudaFreeAsync(work, s);
  cudaFreeAsync(perms, s);
  return rc();
}

int ldg_bj_invert(int64_t nblk, int bs, const double* mats, double* inv_t,
                  int32_t* shifted, void* stream) {
  NvtxRange nvtx_("ldg_bj_invert");
  if (bs < 1) return 2;
  if (bs > kMaxSmemBs) return ldg_bj_invert_global(nblk, bs, mats, inv_t, shifted, stream);
  const size_t sm = (size_t)bs * bs * sizeof(double);
  if (sm > 48 * 1024)
    cudaFuncSetAttribute(invert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (nblk > 0)
    invert_kernel<<<(unsigned)nblk, kInvThreads, sm, (cudaStream_t)stream>>>(bs, mats, inv_t,
                                                                             shifted);
  return rc();
}

int ldg_permute_gather(int64_t n, const int64_t* idx, const double* src, double* dst,
                       void* stream) {
  if (n <= 0) return 0;
  if (!idx || !src || !dst) return 2;
  gather_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
  return rc();
}

int ldg_permute_scatter(int64_t n, const int64_t* idx, const double* src, double* dst,
                        void* stream) {
  if (n <= 0) return 0;
  if (!idx || !src || !dst) return 2;
  scatter_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
  return rc();
}

int ldg_bj_block_keys(int64_t nblk, int bs, const double* mats, uint64_t* keys, void* stream) {
  NvtxRange nvtx_("ldg_bj_block_keys");
  if (nblk <= 0) return 0;
  if (bs < 1 || !mats || !keys) return 2;
  block_hash_kernel<<<(unsigned)nblk, 256, 0, (cudaStream_t)stream>>>(
      bs, mats, reinterpret_cast<unsigned long long*>(keys));
  return rc();
}

int ldg_bj_class_verify(int64_t nblk, int bs, const double* mats, const int64_t* rep, int32_t* bad,
                        void* stream) {
  NvtxRange nvtx_("ldg_bj_class_verify");
  if (nblk <= 0) return 0;
  if (bs < 1 || !mats || !rep || !bad) return 2;
  class_verify_kernel<<<(unsigned)nblk, 256, 0, (cudaStream_t)stream>>>(bs, mats, rep, bad);
  return rc();
}

int ldg_bj_tile_elems() { return kTileE; }

int ldg_bj_apply_tiles(int64_t ntiles, int bs, const double* inv_t, const int32_t* tile_cls,
                       const int32_t* tile_el, const double* r, double* z, void* stream) {
  NvtxRange nvtx_("ldg_bj_apply_tiles");
  if (ntiles <= 0) return 0;
  if (bs < 1 || !inv_t || !tile_cls || !tile_el || !r || !z) return 2;
  const int threads = std::min(256, ((bs + 31) / 32) * 32);
  const size_t sm = (size_t)kTileS * bs * sizeof(double);
  if (sm > 48 * 1024 &&
      cudaFuncSetAttribute(bj_apply_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sm) != cudaSuccess)
    return 3;
  bj_apply_tiles_kernel<<<(unsigned)ntiles, threads, sm, (cudaStream_t)stream>>>(
      bs, inv_t, tile_cls, tile_el, r, z);
  return rc();
}

int ldg_bj_apply(int64_t nblk, int bs, const double* inv_t, const double* r, double* z,
                 void* stream) {
  NvtxRange nvtx_("ldg_bj_apply");
  cudaStream_t s = (cudaStream_t)stream;
  if (nblk <= 0) return 0;
  if (bs <= 256) {
    const int per = 256 / bs;
    const unsigned grid = (unsigned)((nblk + per - 1) / per);
    bj_apply_kernel<<<grid, per * bs, per * bs * sizeof(double), s>>>(nblk, bs, inv_t, r, z);
  } else {
    bj_apply_big_kernel<<<(unsigned)nblk, 256, bs * sizeof(double), s>>>(bs, inv_t, r, z);
  }
  return rc();
}

}  // extern "C"
