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
          snb[slot][f][c][lt] = need ? __ldg(u + ((size_t)nbr[f] * NB + lt) * NCU + c) : 0.0;
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
          snu[slot][f][c][lt] = nu ? __ldg(u + ((size_t)nbr[f] * NB + lt) * NCU + c) : 0.0;
#pragma unroll
        for (int cd = 0; cd < NQ; ++cd)
          snq[slot][f][cd][lt] = nq ? __ldg(q + ((size_t)nbr[f] * NB + lt) * NQ + cd) : 0.0;
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

template <int NB, int NQF, int NFACE, int ND, int NCU, int TPE>
int run_dense(const DenseParams& P, int what, const double* u, const double* gval,
              const double* bsrc, double* q, double* R, cudaStream_t s) {
  constexpr int EPB = kDBlock / TPE;
  const int grid = (P.ne + EPB - 1) / EPB;
  if (grid <= 0) return 0;
  // what: 0 = mixed only (q from u), 1 = residual, 2 = tangent
  mixed_dense<NB, NQF, NFACE, ND, NCU, TPE><<<grid, kDBlock, 0, s>>>(P, u, what == 2 ? nullptr : gval, q);
  if (cudaGetLastError() != cudaSuccess) return 3;
  if (what == 1)
    flux_dense<NB, NQF, NFACE, ND, NCU, TPE, false><<<grid, kDBlock, 0, s>>>(P, u, q, gval, bsrc, R);
  else if (what == 2)
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
