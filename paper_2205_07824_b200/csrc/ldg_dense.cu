// Dense-tabulation LDG kernels for simplices (tri / tet) on sm_100a.
//
// The reference's quadrature-point formulation (disc.py:436-821) with
// affine per-element geometry: face traces through the master tabulations
// (own side) and orientation-indexed tabulations of the neighbour (the
// reference Newton-inverts every right trace, disc.py:182-225; they agree to
// ~1e-15), lifts with M_ref^-1 Phi^T W, the volume gradient by collocation
// derivatives and the volume flux by K_r = int d_r phi_a phi_b (exact for
// the linear fluxes this path accepts).  Two passes (mixed -> flux) with q in
// HBM: simplex elements are FP64-bound (dense nb x nb operators), not
// bandwidth-bound.  Element-centric, no atomics.
//
// Threads: TPE per element (>= nb and >= face quadrature points); node a =
// thread a for volume work, face point s = thread s for face work.

#include "ldg_dense.cuh"

namespace ldg {
namespace {

#ifndef LDG_DENSE_BLOCK
#define LDG_DENSE_BLOCK 128
#endif
constexpr int kDBlock = LDG_DENSE_BLOCK;
#ifndef LDG_DENSE_MMA
#define LDG_DENSE_MMA 1       // ncu = 1: operator contractions on the FP64 tensor core
#endif
#ifndef LDG_TET3_TPE
#define LDG_TET3_TPE 24       // threads per tet p=3 element (>= nb = 20); measured 20: 3.57, 24: 3.27, 32: 3.40 ms
#endif

__device__ __forceinline__ void dbad(const DenseParams& P, int e, double v) {
  if (!isfinite(v)) atomicMin(P.bad, (unsigned long long)e);
}

// coefficient form of the trace rules (see ldg_fused.cu / capi.cu):
// jump = alpha d, sigma tau (u_L - u^) = beta tau d, q^ = w_own q + w_nbr q_nbr
__device__ __forceinline__ void coeffs(const DenseParams& P, int info, double& alpha,
                                      double& beta, double& wo, double& wn) {
  const int kind = info & LDG_FACE_KIND_MASK;
  if (kind == LDG_FACE_INTERIOR) {
    const bool right = info & LDG_FACE_SIDE_RIGHT, sw = info & LDG_FACE_SWITCH;
    alpha = P.trace_centered ? 0.5 : (sw == right ? 1.0 : 0.0);
    beta = P.trace_centered ? 0.5 : (sw ? 0.0 : 1.0);
    wo = P.grad_centered ? 0.5 : (sw == right ? 1.0 : 0.0);
    wn = P.grad_centered ? 0.5 : (sw != right ? 1.0 : 0.0);
  } else if (kind == LDG_FACE_DIRICHLET) {
    alpha = beta = wo = 1.0;
    wn = 0.0;
  } else {
    alpha = beta = wo = wn = 0.0;
  }
}

template <int NB, int NQF, int NFACE, int ND, int NCU, int TPE>
__global__ void __launch_bounds__(kDBlock)
mixed_dense(const __grid_constant__ DenseParams P, const double* __restrict__ u,
            const double* __restrict__ gval, double* __restrict__ q) {
  constexpr int EPB = kDBlock / TPE;
  __shared__ double su[EPB][NCU][NB];
  __shared__ double snb[EPB][NFACE][NCU][NB];
  __shared__ double sjump[EPB][NFACE][NQF][NCU];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;   // TPE need not divide the block
  int info[NFACE], nbr[NFACE];
  if (active) {
#pragma unroll
    for (int f = 0; f < NFACE; ++f) {
      info[f] = __ldg(P.finfo + e * NFACE + f);
      nbr[f] = __ldg(P.fnbr + e * NFACE + f);
    }
    if (lt < NB) {
#pragma unroll
      for (int c = 0; c < NCU; ++c) su[slot][c][lt] = __ldg(u + ((size_t)e * NB + lt) * NCU + c);
#pragma unroll
      for (int f = 0; f < NFACE; ++f) {
        double a_, b_, wo_, wn_;
        coeffs(P, info[f], a_, b_, wo_, wn_);
        const bool need = (info[f] & LDG_FACE_KIND_MASK) == LDG_FACE_INTERIOR && a_ != 0.0;
#pragma unroll
        for (int c = 0; c < NCU; ++c)
          snb[slot][f][c][lt] = need ? __ldg(dense_nbr_row<false>(P, u, nbr[f], NB * NCU) + lt * NCU + c) : 0.0;
      }
    }
  }
  __syncthreads();
  // face points: (face, point) pairs spread over all TPE lanes (NFACE * NQF
  // items; the per-face loop of one point per lane left TPE - NQF idle)
  if (active) {
    for (int idx = lt; idx < NFACE * NQF; idx += TPE) {
      const int f = idx / NQF, sp = idx - f * NQF;
      const int inf = __ldg(P.finfo + e * NFACE + f);
      double alpha, b_, wo_, wn_;
      coeffs(P, inf, alpha, b_, wo_, wn_);
      const int kind = inf & LDG_FACE_KIND_MASK;
      if (alpha == 0.0) {
#pragma unroll
        for (int c = 0; c < NCU; ++c) sjump[slot][f][sp][c] = 0.0;
        continue;
      }
      const double* pf = P.phif + f * NB * NQF + sp;
      const double* po = P.phio + (((inf >> 4) & 7) * P.nperm + ((inf >> 8) & 0xff)) * NB * NQF + sp;
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double own = 0.0, oth = 0.0;
#pragma unroll
        for (int b = 0; b < NB; ++b) own = fma(__ldg(pf + b * NQF), su[slot][c][b], own);
        if (kind == LDG_FACE_INTERIOR) {
#pragma unroll
          for (int b = 0; b < NB; ++b) oth = fma(__ldg(po + b * NQF), snb[slot][f][c][b], oth);
        } else if (kind == LDG_FACE_DIRICHLET && gval) {
          oth = __ldg(gval + ((size_t)__ldg(P.fnbr + e * NFACE + f) * NQF + sp) * NCU + c);
        }
        sjump[slot][f][sp][c] = alpha * (own - oth);
      }
    }
  }
  __syncthreads();
  if (!active || lt >= NB) return;
  const double* g = P.geo + (size_t)e * (1 + ND * ND);
  const double detj = __ldg(g);
  double ij[ND][ND];
#pragma unroll
  for (int d = 0; d < ND; ++d)
#pragma unroll
    for (int r = 0; r < ND; ++r) ij[d][r] = __ldg(g + 1 + d * ND + r);
#pragma unroll
  for (int c = 0; c < NCU; ++c) {
    double gr[ND];
#pragma unroll
    for (int r = 0; r < ND; ++r) {
      double a = 0.0;
      const double* dr = P.dr + r * NB * NB + lt;
#pragma unroll
      for (int b = 0; b < NB; ++b) a = fma(__ldg(dr + b * NB), su[slot][c][b], a);
      gr[r] = a;
    }
    double qd[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      double a = 0.0;
#pragma unroll
      for (int r = 0; r < ND; ++r) a = fma(ij[d][r], gr[r], a);
      qd[d] = -a;
    }
#pragma unroll
    for (int f = 0; f < NFACE; ++f) {
      const double* lf_ = P.lift + f * NQF * NB + lt;
      double l = 0.0;
#pragma unroll
      for (int s = 0; s < NQF; ++s) l = fma(__ldg(lf_ + s * NB), sjump[slot][f][s][c], l);
      const double fac = __ldg(P.fsj + e * NFACE + f) / detj * l;
#pragma unroll
      for (int d = 0; d < ND; ++d) qd[d] = fma(fac, __ldg(P.fnorm + (e * NFACE + f) * ND + d), qd[d]);
    }
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      dbad(P, e, qd[d]);
      q[(((size_t)e * NB + lt) * NCU + c) * ND + d] = qd[d];
    }
  }
}

template <int NB, int NQF, int NFACE, int ND, int NCU, int TPE, bool TANGENT>
__global__ void __launch_bounds__(kDBlock)
flux_dense(const __grid_constant__ DenseParams P, const double* __restrict__ u,
           const double* __restrict__ q, const double* __restrict__ gval,
           const double* __restrict__ bsrc, double* __restrict__ R) {
  constexpr int EPB = kDBlock / TPE, NQ = NCU * ND;
  __shared__ double su[EPB][NCU][NB];
  __shared__ double sq[EPB][NQ][NB];
  __shared__ double snu[EPB][NFACE][NCU][NB];
  __shared__ double snq[EPB][NFACE][NQ][NB];
  __shared__ double sF[EPB][ND][NCU][NB];
  __shared__ double sfh[EPB][NFACE][NQF][NCU];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;   // TPE need not divide the block
  int info[NFACE], nbr[NFACE];
  double detj = 1.0, ij[ND][ND];
  if (active) {
    const double* g = P.geo + (size_t)e * (1 + ND * ND);
    detj = __ldg(g);
#pragma unroll
    for (int d = 0; d < ND; ++d)
#pragma unroll
      for (int r = 0; r < ND; ++r) ij[d][r] = __ldg(g + 1 + d * ND + r);
#pragma unroll
    for (int f = 0; f < NFACE; ++f) {
      info[f] = __ldg(P.finfo + e * NFACE + f);
      nbr[f] = __ldg(P.fnbr + e * NFACE + f);
    }
    if (lt < NB) {
#pragma unroll
      for (int c = 0; c < NCU; ++c) su[slot][c][lt] = __ldg(u + ((size_t)e * NB + lt) * NCU + c);
#pragma unroll
      for (int cd = 0; cd < NQ; ++cd) sq[slot][cd][lt] = __ldg(q + ((size_t)e * NB + lt) * NQ + cd);
#pragma unroll
      for (int f = 0; f < NFACE; ++f) {
        double alpha, beta, wo, wn;
        coeffs(P, info[f], alpha, beta, wo, wn);
        const bool inter = (info[f] & LDG_FACE_KIND_MASK) == LDG_FACE_INTERIOR;
        const bool nu = inter && (alpha != 0.0 || beta != 0.0);
        const bool nq = inter && wn != 0.0;
#pragma unroll
        for (int c = 0; c < NCU; ++c)
          snu[slot][f][c][lt] = nu ? __ldg(dense_nbr_row<false>(P, u, nbr[f], NB * NCU) + lt * NCU + c) : 0.0;
#pragma unroll
        for (int cd = 0; cd < NQ; ++cd)
          snq[slot][f][cd][lt] = nq ? __ldg(dense_nbr_row<true>(P, q, nbr[f], NB * NQ) + lt * NQ + cd) : 0.0;
      }
    }
  }
  __syncthreads();
  if (active && lt < NB) {
    // nodal flux density in reference directions
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      double f[ND];
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < NCU; ++k) {
          if (P.flux_uses_u) a = fma(P.au[(c * 3 + d) * LDG_MAX_NCU + k], su[slot][k][lt], a);
#pragma unroll
          for (int x = 0; x < ND; ++x)
            a = fma(P.aq[((c * 3 + d) * LDG_MAX_NCU + k) * 3 + x], sq[slot][k * ND + x][lt], a);
        }
        f[d] = a;
      }
#pragma unroll
      for (int r = 0; r < ND; ++r) {
        double a = 0.0;
#pragma unroll
        for (int d = 0; d < ND; ++d) a = fma(ij[d][r], f[d], a);
        sF[slot][r][c][lt] = detj * a;
      }
    }
  }
  if (active) {
    for (int idx = lt; idx < NFACE * NQF; idx += TPE) {      // (face, point) pairs over all lanes
      const int f = idx / NQF, sp = idx - f * NQF;
      const int inf = __ldg(P.finfo + e * NFACE + f);
      const int nbf = __ldg(P.fnbr + e * NFACE + f);
      double alpha, beta, wo, wn;
      coeffs(P, inf, alpha, beta, wo, wn);
      const int kind = inf & LDG_FACE_KIND_MASK;
      const double* pf = P.phif + f * NB * NQF + sp;
      const double* po = P.phio + (((inf >> 4) & 7) * P.nperm + ((inf >> 8) & 0xff)) * NB * NQF + sp;
      const bool inter = kind == LDG_FACE_INTERIOR;
      double uo[NCU], un[NCU], qh[NQ];
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double a = 0.0, b2 = 0.0;
#pragma unroll
        for (int b = 0; b < NB; ++b) a = fma(__ldg(pf + b * NQF), su[slot][c][b], a);
        if (inter && (alpha != 0.0 || beta != 0.0)) {
#pragma unroll
          for (int b = 0; b < NB; ++b) b2 = fma(__ldg(po + b * NQF), snu[slot][f][c][b], b2);
        }
        uo[c] = a;
        un[c] = kind == LDG_FACE_INTERIOR ? b2
                : ((!TANGENT && gval) ? __ldg(gval + ((size_t)nbf * NQF + sp) * NCU + c) : 0.0);
      }
#pragma unroll
      for (int cd = 0; cd < NQ; ++cd) {
        double a = 0.0, b2 = 0.0;
        if (wo != 0.0) {
#pragma unroll
          for (int b = 0; b < NB; ++b) a = fma(__ldg(pf + b * NQF), sq[slot][cd][b], a);
        }
        if (inter && wn != 0.0) {
#pragma unroll
          for (int b = 0; b < NB; ++b) b2 = fma(__ldg(po + b * NQF), snq[slot][f][cd][b], b2);
        }
        qh[cd] = wo * a + wn * b2;
      }
      const double tau = __ldg(P.ftau + e * NFACE + f);
      double nrm[ND];
#pragma unroll
      for (int d = 0; d < ND; ++d) nrm[d] = __ldg(P.fnorm + (e * NFACE + f) * ND + d);
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double fh;
        if (kind == LDG_FACE_NEUMANN) {
          fh = (!TANGENT && gval) ? __ldg(gval + ((size_t)nbf * NQF + sp) * NCU + c) : 0.0;
        } else {
          double uh[NCU];
#pragma unroll
          for (int k = 0; k < NCU; ++k) uh[k] = uo[k] - alpha * (uo[k] - un[k]);
          double fn = 0.0;
#pragma unroll
          for (int d = 0; d < ND; ++d) {
            double a = 0.0;
#pragma unroll
            for (int k = 0; k < NCU; ++k) {
              if (P.flux_uses_u) a = fma(P.au[(c * 3 + d) * LDG_MAX_NCU + k], uh[k], a);
#pragma unroll
              for (int x = 0; x < ND; ++x)
                a = fma(P.aq[((c * 3 + d) * LDG_MAX_NCU + k) * 3 + x], qh[k * ND + x], a);
            }
            fn = fma(a, nrm[d], fn);
          }
          fh = fn + beta * tau * (uo[c] - un[c]);
        }
        sfh[slot][f][sp][c] = fh;
      }
    }
  }
  __syncthreads();
  if (!active || lt >= NB) return;
#pragma unroll
  for (int c = 0; c < NCU; ++c) {
    double r = 0.0;
#pragma unroll
    for (int rr = 0; rr < ND; ++rr) {
      const double* kr = P.kr + rr * NB * NB + lt;
#pragma unroll
      for (int b = 0; b < NB; ++b) r = fma(__ldg(kr + b * NB), sF[slot][rr][c][b], r);
    }
    double out = -r;
#pragma unroll
    for (int f = 0; f < NFACE; ++f) {
      const double* fo = P.fluxop + f * NQF * NB + lt;
      double a = 0.0;
#pragma unroll
      for (int s = 0; s < NQF; ++s) a = fma(__ldg(fo + s * NB), sfh[slot][f][s][c], a);
      out = fma(__ldg(P.fsj + e * NFACE + f), a, out);
    }
    if (!TANGENT && bsrc) out += __ldg(bsrc + ((size_t)e * NB + lt) * NCU + c);
    dbad(P, e, out);
    R[((size_t)e * NB + lt) * NCU + c] = out;
  }
}

// --------------------------------------------------------------------------
// Tensor-core variants (ncu = 1): the element-independent contractions --
// own face traces (phif), the collocation gradient (dr), the lifts, the volume
// term (K_r) and the face lift (Phi^T W) -- batched over the 8 elements of a
// block as GEMMs on the FP64 tensor core (mma.sync m8n8k4: A = an 8 x 4 slice
// of the operator, B = 4 nodes x 8 elements, D = 8 outputs x 8 elements).  One
// A entry now feeds 8 elements instead of 1 (the scalar kernels above issue
// one operator load per FMA: LSU-bound).  The orientation-dependent neighbour
// traces stay on the FP64 pipe.  Same arithmetic identities and outputs.
// --------------------------------------------------------------------------
constexpr int kMmaEpb = 8;
// per-element pitch of the GEMM operands in shared memory: == 4 (mod 16)
// doubles, so the 8 elements of a B / C fragment spread over the banks
// (a multiple of 16 put all 8 in one bank: 4-8-way conflicts)
__host__ __device__ constexpr int mma_pitch(int n) { return n + ((4 - n % 16) + 16) % 16; }

#ifndef LDG_TRACE_UNROLL
#define LDG_TRACE_UNROLL 20       // neighbour-trace loop unroll (table loads in flight; ncu: 4 -> 20 281 -> 272 us)
#endif
constexpr int kTraceUnroll = LDG_TRACE_UNROLL;
#ifndef LDG_MMA_CHAINS
#define LDG_MMA_CHAINS 2
#endif
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// C(m, e) = sum_k A1(m, k) B1(k, e) [+ sum_k A2(m, k) B2(k, e)] for one 8-row
// tile mt and the block's 8 elements; A(m, k) = A[k * AK + m] (operator,
// column-major as stored), B(k, e) = B[e * BE + k] (shared), C(m, e) =
// C[e * CE + m] (shared).  Rows m >= M are zero-padded and not stored.
template <int M, int K1, int AK1, int BE1, int K2, int AK2, int BE2, int CE>
__device__ __forceinline__ void gemm8_tile(int mt, const double* __restrict__ A1, const double* B1,
                                           const double* __restrict__ A2, const double* B2,
                                           double* C) {
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  const int m = mt * 8 + r;
  // LDG_MMA_CHAINS independent accumulator chains (k-steps dealt round
  // robin, summed at the end), so consecutive tensor-core steps do not wait
  // on each other's accumulator
  constexpr int NCH = LDG_MMA_CHAINS;
  double d0[NCH], d1[NCH];
#pragma unroll
  for (int x = 0; x < NCH; ++x) d0[x] = d1[x] = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < K1; k0 += 4) {
    const int k = k0 + c;
    const double a = (m < M && k < K1) ? __ldg(A1 + k * AK1 + m) : 0.0;
    const double b = k < K1 ? B1[r * BE1 + k] : 0.0;
    dmma884(d0[(k0 / 4) % NCH], d1[(k0 / 4) % NCH], a, b);
  }
  if (K2 > 0) {
#pragma unroll
    for (int k0 = 0; k0 < K2; k0 += 4) {
      const int k = k0 + c;
      const double a = (m < M && k < K2) ? __ldg(A2 + k * AK2 + m) : 0.0;
      const double b = k < K2 ? B2[r * BE2 + k] : 0.0;
      dmma884(d0[(k0 / 4 + 1) % NCH], d1[(k0 / 4 + 1) % NCH], a, b);
    }
  }
#pragma unroll
  for (int x = 1; x < NCH; ++x) {
    d0[0] += d0[x];
    d1[0] += d1[x];
  }
  if (m < M) {
    C[(2 * c) * CE + m] = d0[0];
    C[(2 * c + 1) * CE + m] = d1[0];
  }
}

template <int NB, int NQF, int NFACE, int ND, int TPE>
__global__ void __launch_bounds__(kMmaEpb * TPE)
mixed_dense_mma(const __grid_constant__ DenseParams P, const double* __restrict__ u,
                const double* __restrict__ gval, double* __restrict__ q) {
  constexpr int EPB = kMmaEpb, NT = EPB * TPE, NW = NT / 32;
  constexpr int MTN = (NB + 7) / 8, MTF = (NQF + 7) / 8;
  __shared__ double su[EPB][NB];
  constexpr int PNB = mma_pitch(NFACE * NB);
  __shared__ double snb[EPB * PNB];                 // neighbour u [e][f][b]
  constexpr int PF = mma_pitch(NFACE * NQF), PG = mma_pitch(ND * NB), PL = mma_pitch(NFACE * NB);
  __shared__ double sto[EPB * PF];            // own traces [e][f][s]
  __shared__ double sjump[EPB * PF];          // [e][f][s]
  __shared__ double sg[EPB * PG];             // reference-direction derivatives [e][r][a]
  __shared__ double sl[EPB * PL];             // lifted jumps [e][f][a]
  // element geometry for the final combination, loaded with the first loads
  // (detj, invJ^T, then per face sJ and the normal): its latency no longer
  // sits after the last barrier
  constexpr int NGE = 1 + ND * ND + NFACE * (1 + ND);
  __shared__ double sgeo[EPB][NGE];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * EPB + slot;
  const bool active = e < P.ne;
  if (active)
    for (int x = lt; x < NGE; x += TPE) {
      double v;
      if (x < 1 + ND * ND) v = __ldg(P.geo + (size_t)e * (1 + ND * ND) + x);
      else if (x < 1 + ND * ND + NFACE) v = __ldg(P.fsj + e * NFACE + (x - 1 - ND * ND));
      else v = __ldg(P.fnorm + e * NFACE * ND + (x - 1 - ND * ND - NFACE));
      sgeo[slot][x] = v;
    }
  int info[NFACE], nbr[NFACE];
#pragma unroll
  for (int f = 0; f < NFACE; ++f) {
    info[f] = active ? __ldg(P.finfo + e * NFACE + f) : LDG_FACE_NEUMANN;
    nbr[f] = active ? __ldg(P.fnbr + e * NFACE + f) : 0;
  }
  if (lt < NB) {
    su[slot][lt] = active ? __ldg(u + (size_t)e * NB + lt) : 0.0;
#pragma unroll
    for (int f = 0; f < NFACE; ++f) {
      double a_, b_, wo_, wn_;
      coeffs(P, info[f], a_, b_, wo_, wn_);
      const bool need = (info[f] & LDG_FACE_KIND_MASK) == LDG_FACE_INTERIOR && a_ != 0.0;
      snb[slot * PNB + f * NB + lt] = need ? __ldg(dense_nbr_row<false>(P, u, nbr[f], NB) + lt) : 0.0;
    }
  }
  __syncthreads();
  // tensor core: own traces (phif_f u) and the gradient (dr_r u)
  for (int job = warp; job < NFACE * MTF + ND * MTN; job += NW) {
    if (job < NFACE * MTF) {
      const int f = job / MTF, mt = job % MTF;
      gemm8_tile<NQF, NB, NQF, NB, 0, 1, 1, PF>(
          mt, P.phif + f * NB * NQF, &su[0][0], nullptr, nullptr, sto + f * NQF);
    } else {
      const int j = job - NFACE * MTF, r = j / MTN, mt = j % MTN;
      gemm8_tile<NB, NB, NB, NB, 0, 1, 1, PG>(
          mt, P.dr + r * NB * NB, &su[0][0], nullptr, nullptr, sg + r * NB);
    }
  }
  __syncthreads();
  if (active) {
    for (int idx = lt; idx < NFACE * NQF; idx += TPE) {
      const int f = idx / NQF, sp = idx - f * NQF;
      const int inf = __ldg(P.finfo + e * NFACE + f);
      double alpha, b_, wo_, wn_;
      coeffs(P, inf, alpha, b_, wo_, wn_);
      const int kind = inf & LDG_FACE_KIND_MASK;
      double jump = 0.0;
      if (alpha != 0.0) {
        double oth = 0.0;
        if (kind == LDG_FACE_INTERIOR) {
          const double* po = P.phio + (((inf >> 4) & 7) * P.nperm + ((inf >> 8) & 0xff)) * NB * NQF + sp;
#pragma unroll
          for (int b = 0; b < NB; ++b) oth = fma(__ldg(po + b * NQF), snb[slot * PNB + f * NB + b], oth);
        } else if (kind == LDG_FACE_DIRICHLET && gval) {
          oth = __ldg(gval + (size_t)__ldg(P.fnbr + e * NFACE + f) * NQF + sp);
        }
        jump = alpha * (sto[slot * PF + idx] - oth);
      }
      sjump[slot * PF + idx] = jump;
    }
  } else {
    for (int idx = lt; idx < NFACE * NQF; idx += TPE) sjump[slot * PF + idx] = 0.0;
  }
  __syncthreads();
  // tensor core: the lifts M_ref^-1 Phi^T W jump, per face
  for (int job = warp; job < NFACE * MTN; job += NW) {
    const int f = job / MTN, mt = job % MTN;
    gemm8_tile<NB, NQF, NB, PF, 0, 1, 1, PL>(
        mt, P.lift + f * NQF * NB, sjump + f * NQF, nullptr, nullptr, sl + f * NB);
  }
  __syncthreads();
  if (!active || lt >= NB) return;
  const double* g = sgeo[slot];
  const double detj = g[0];
  double qd[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    double a = 0.0;
#pragma unroll
    for (int r = 0; r < ND; ++r) a = fma(g[1 + d * ND + r], sg[slot * PG + r * NB + lt], a);
    qd[d] = -a;
  }
#pragma unroll
  for (int f = 0; f < NFACE; ++f) {
    const double fac = g[1 + ND * ND + f] / detj * sl[slot * PL + f * NB + lt];
#pragma unroll
    for (int d = 0; d < ND; ++d) qd[d] = fma(fac, g[1 + ND * ND + NFACE + f * ND + d], qd[d]);
  }
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    dbad(P, e, qd[d]);
    q[((size_t)e * NB + lt) * ND + d] = qd[d];
  }
}

template <int NB, int NQF, int NFACE, int ND, int TPE, bool TANGENT>
__global__ void __launch_bounds__(kMmaEpb * TPE)
flux_dense_mma(const __grid_constant__ DenseParams P, const double* __restrict__ u,
               const double* __restrict__ q, const double* __restrict__ gval,
               const double* __restrict__ bsrc, double* __restrict__ R) {
  constexpr int EPB = kMmaEpb, NT = EPB * TPE, NW = NT / 32, NV = 1 + ND;
  constexpr int MTN = (NB + 7) / 8, MTF = (NQF + 7) / 8;
  // dynamic shared memory (> 48 KB at tet p = 3), GEMM operands at
  // conflict-free element pitches (mma_pitch); sR reuses the trace region
  constexpr int PV = mma_pitch(NV * NB), PT = mma_pitch(NFACE * NV * NQF);
  constexpr int PH = mma_pitch(NFACE * NQF), PF = mma_pitch(ND * NB);
  extern __shared__ __align__(16) double dsm[];
  double* sv = dsm;                                          // [e][v][b]: u, q_1..q_ND
  // neighbour u and q of a node side by side ([e][f][b][u q1 q2 q3], 4
  // doubles): the trace loop takes each node's four values in two 16-B loads
  constexpr int PNV = mma_pitch(NFACE * NB * 4) + 4;               // == 8 (mod 16): 16-B aligned
  static_assert(ND + 1 <= 4, "packed neighbour layout");
  double* snv = dsm + EPB * PV;
  double* sF = snv + EPB * PNV;                                     // [e][r][b]: -detJ invJ^T f
  double* sto = sF + EPB * PF;                                      // [e][f][v][s] own traces
  double* sfh = sto + EPB * PT;                                     // [e][f s]: sJ f^
  double* sR = sto;                                                 // [e][a]
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * EPB + slot;
  const bool active = e < P.ne;
  int info[NFACE], nbr[NFACE];
#pragma unroll
  for (int f = 0; f < NFACE; ++f) {
    info[f] = active ? __ldg(P.finfo + e * NFACE + f) : LDG_FACE_NEUMANN;
    nbr[f] = active ? __ldg(P.fnbr + e * NFACE + f) : 0;
  }
  double detj = 1.0, ij[ND][ND];
  {
    const double* g = P.geo + (size_t)(active ? e : 0) * (1 + ND * ND);
    detj = __ldg(g);
#pragma unroll
    for (int d = 0; d < ND; ++d)
#pragma unroll
      for (int r = 0; r < ND; ++r) ij[d][r] = __ldg(g + 1 + d * ND + r);
  }
  if (lt < NB) {
    sv[slot * PV + lt] = active ? __ldg(u + (size_t)e * NB + lt) : 0.0;
#pragma unroll
    for (int d = 0; d < ND; ++d)
      sv[slot * PV + (1 + d) * NB + lt] = active ? __ldg(q + ((size_t)e * NB + lt) * ND + d) : 0.0;
#pragma unroll
    for (int f = 0; f < NFACE; ++f) {
      double alpha, beta, wo, wn;
      coeffs(P, info[f], alpha, beta, wo, wn);
      const bool inter = (info[f] & LDG_FACE_KIND_MASK) == LDG_FACE_INTERIOR;
      const bool nu = inter && (alpha != 0.0 || beta != 0.0);
      const bool nq = inter && wn != 0.0;
      // the node's four values assembled in registers, stored as two 16-B
      // words (four 8-B stores at a 32-B lane stride were 4-way conflicted)
      double w4[4];
      w4[0] = nu ? __ldg(dense_nbr_row<false>(P, u, nbr[f], NB) + lt) : 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d)
        w4[1 + d] = (d < ND && nq) ? __ldg(dense_nbr_row<true>(P, q, nbr[f], NB * ND) + lt * ND + d)
                                   : 0.0;
      double2* nv2 = reinterpret_cast<double2*>(snv + slot * PNV + (f * NB + lt) * 4);
      nv2[0] = make_double2(w4[0], w4[1]);
      nv2[1] = make_double2(w4[2], w4[3]);
    }
  }
  __syncthreads();
  // nodal flux density in reference directions, negated (the volume term
  // enters R with a minus sign)
  if (lt < NB) {
    double f[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      double a = 0.0;
      if (P.flux_uses_u) a = fma(P.au[d * LDG_MAX_NCU], sv[slot * PV + lt], a);
#pragma unroll
      for (int x = 0; x < ND; ++x)
        a = fma(P.aq[d * LDG_MAX_NCU * 3 + x], sv[slot * PV + (1 + x) * NB + lt], a);
      f[d] = a;
    }
#pragma unroll
    for (int r = 0; r < ND; ++r) {
      double a = 0.0;
#pragma unroll
      for (int d = 0; d < ND; ++d) a = fma(ij[d][r], f[d], a);
      sF[slot * PF + r * NB + lt] = -detj * a;
    }
  }
  // tensor core: own traces of u and q on every face
  for (int job = warp; job < NFACE * NV * MTF; job += NW) {
    const int f = job / (NV * MTF), v = (job / MTF) % NV, mt = job % MTF;
    gemm8_tile<NQF, NB, NQF, PV, 0, 1, 1, PT>(
        mt, P.phif + f * NB * NQF, sv + v * NB, nullptr, nullptr, sto + (f * NV + v) * NQF);
  }
  __syncthreads();
  if (active) {
    for (int idx = lt; idx < NFACE * NQF; idx += TPE) {      // (face, point) pairs over all lanes
      const int f = idx / NQF, sp = idx - f * NQF;
      const int inf = __ldg(P.finfo + e * NFACE + f);
      const int nbf = __ldg(P.fnbr + e * NFACE + f);
      double alpha, beta, wo, wn;
      coeffs(P, inf, alpha, beta, wo, wn);
      const int kind = inf & LDG_FACE_KIND_MASK;
      const bool inter = kind == LDG_FACE_INTERIOR;
      const double* po = P.phio + (((inf >> 4) & 7) * P.nperm + ((inf >> 8) & 0xff)) * NB * NQF + sp;
      const double* to = sto + slot * PT + f * NV * NQF + sp;
      const double uo = to[0];
      // neighbour traces: one pass over the orientation's tabulation feeds u
      // and every q component (each entry loaded once)
      double un = 0.0, qn[ND];
#pragma unroll
      for (int d = 0; d < ND; ++d) qn[d] = 0.0;
      const bool need_u = inter && (alpha != 0.0 || beta != 0.0), need_q = inter && wn != 0.0;
      if (need_u || need_q) {
#pragma unroll (kTraceUnroll)
        for (int b = 0; b < NB; ++b) {
          const double ph = __ldg(po + b * NQF);
          const double2* nv2 = reinterpret_cast<const double2*>(snv + slot * PNV + (f * NB + b) * 4);
          const double2 a01 = nv2[0], a23 = nv2[1];
          un = fma(ph, a01.x, un);
          qn[0] = fma(ph, a01.y, qn[0]);
          if (ND > 1) qn[1] = fma(ph, a23.x, qn[1]);
          if (ND > 2) qn[2] = fma(ph, a23.y, qn[2]);
        }
      } else if (!inter && !TANGENT && gval) {
        un = __ldg(gval + (size_t)nbf * NQF + sp);
      }
      double qh[ND];
#pragma unroll
      for (int d = 0; d < ND; ++d) qh[d] = wo * to[(1 + d) * NQF] + wn * qn[d];
      double fh;
      if (kind == LDG_FACE_NEUMANN) {
        fh = (!TANGENT && gval) ? __ldg(gval + (size_t)nbf * NQF + sp) : 0.0;
      } else {
        const double uh = uo - alpha * (uo - un);
        double fn = 0.0;
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          double a = 0.0;
          if (P.flux_uses_u) a = fma(P.au[d * LDG_MAX_NCU], uh, a);
#pragma unroll
          for (int x = 0; x < ND; ++x) a = fma(P.aq[d * LDG_MAX_NCU * 3 + x], qh[x], a);
          fn = fma(a, __ldg(P.fnorm + (e * NFACE + f) * ND + d), fn);
        }
        fh = fn + beta * __ldg(P.ftau + e * NFACE + f) * (uo - un);
      }
      sfh[slot * PH + idx] = __ldg(P.fsj + e * NFACE + f) * fh;
    }
  } else {
    for (int idx = lt; idx < NFACE * NQF; idx += TPE) sfh[slot * PH + idx] = 0.0;
  }
  __syncthreads();
  // tensor core: R = sum_r K_r (-F_r) + sum_f Phi_f^T W (sJ f^)
  for (int mt = warp; mt < MTN; mt += NW)
    gemm8_tile<NB, ND * NB, NB, PF, NFACE * NQF, NB, PH, NB>(
        mt, P.kr, sF, P.fluxop, sfh, sR);
  __syncthreads();
  if (!active || lt >= NB) return;
  double out = sR[slot * NB + lt];
  if (!TANGENT && bsrc) out += __ldg(bsrc + (size_t)e * NB + lt);
  dbad(P, e, out);
  R[(size_t)e * NB + lt] = out;
}

template <int NB, int NQF, int NFACE, int ND, int NCU, int TPE>
int run_dense(const DenseParams& P, int what, const double* u, const double* gval,
              const double* bsrc, double* q, double* R, cudaStream_t s) {
  constexpr int EPB = kDBlock / TPE;
  const int grid = (P.ne + EPB - 1) / EPB;
  if (grid <= 0) return 0;
  // what: 0 = mixed only (q from u), 1 = residual, 2 = tangent
  if constexpr (NCU == 1 && LDG_DENSE_MMA) {
    // tensor-core variants (8 elements per block, batched operator GEMMs)
    const int gm = (P.ne + kMmaEpb - 1) / kMmaEpb;
    constexpr int fsm = (int)sizeof(double) * kMmaEpb *
                        (mma_pitch((1 + ND) * NB) + mma_pitch(NFACE * NB * 4) + 4 +
                         mma_pitch(ND * NB) +
                         mma_pitch(NFACE * (1 + ND) * NQF) + mma_pitch(NFACE * NQF));
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(flux_dense_mma<NB, NQF, NFACE, ND, TPE, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, fsm);
      cudaFuncSetAttribute(flux_dense_mma<NB, NQF, NFACE, ND, TPE, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, fsm);
      attr = true;
    }
    if (what <= 2)
      mixed_dense_mma<NB, NQF, NFACE, ND, TPE><<<gm, kMmaEpb * TPE, 0, s>>>(
          P, u, what == 2 ? nullptr : gval, q);
    if (cudaGetLastError() != cudaSuccess) return 3;
    if (what == 1 || what == 3)
      flux_dense_mma<NB, NQF, NFACE, ND, TPE, false><<<gm, kMmaEpb * TPE, fsm, s>>>(P, u, q, gval, bsrc, R);
    else if (what == 2 || what == 4)
      flux_dense_mma<NB, NQF, NFACE, ND, TPE, true><<<gm, kMmaEpb * TPE, fsm, s>>>(P, u, q, nullptr, nullptr, R);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
  }
  if (what <= 2)
    mixed_dense<NB, NQF, NFACE, ND, NCU, TPE><<<grid, kDBlock, 0, s>>>(P, u, what == 2 ? nullptr : gval, q);
  if (cudaGetLastError() != cudaSuccess) return 3;
  if (what == 1 || what == 3)
    flux_dense<NB, NQF, NFACE, ND, NCU, TPE, false><<<grid, kDBlock, 0, s>>>(P, u, q, gval, bsrc, R);
  else if (what == 2 || what == 4)
    flux_dense<NB, NQF, NFACE, ND, NCU, TPE, true><<<grid, kDBlock, 0, s>>>(P, u, q, nullptr, nullptr, R);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

int launch_dense(const DenseParams& P, int what, const double* u, const double* gval,
                 const double* bsrc, double* q, double* R, cudaStream_t s) {
  const int key = P.nd * 10000 + P.nb * 100 + P.ncu * 10;
  switch (key) {
    // tri p = 1..4 (nqf = p + 1)
    case 20310: return run_dense<3, 2, 3, 2, 1, 4>(P, what, u, gval, bsrc, q, R, s);
    case 20610: return run_dense<6, 3, 3, 2, 1, 8>(P, what, u, gval, bsrc, q, R, s);
    case 21010: return run_dense<10, 4, 3, 2, 1, 16>(P, what, u, gval, bsrc, q, R, s);
    case 21510: return run_dense<15, 5, 3, 2, 1, 16>(P, what, u, gval, bsrc, q, R, s);
    case 20320: return run_dense<3, 2, 3, 2, 2, 4>(P, what, u, gval, bsrc, q, R, s);
    case 20620: return run_dense<6, 3, 3, 2, 2, 8>(P, what, u, gval, bsrc, q, R, s);
    case 21020: return run_dense<10, 4, 3, 2, 2, 16>(P, what, u, gval, bsrc, q, R, s);
    // tet p = 1..3 (nqf = (p + 1)^2)
    case 30410: return run_dense<4, 4, 4, 3, 1, 4>(P, what, u, gval, bsrc, q, R, s);
    case 31010: return run_dense<10, 9, 4, 3, 1, 16>(P, what, u, gval, bsrc, q, R, s);
    case 32010: return run_dense<20, 16, 4, 3, 1, LDG_TET3_TPE>(P, what, u, gval, bsrc, q, R, s);
    default: return 2;
  }
}

}  // namespace ldg
