// Tensor-product (quad/hex) LDG kernels for sm_100a.
//
// Two passes per operator application, each one element-centric (no float
// atomics, no scatter: every element gathers its neighbours' face nodes, so
// results are bit-reproducible for a fixed mesh):
//
//   pass A  (mixed):  q = M^-1 [ -int grad(u) phi + oint (u - u^) n phi ]
//                     disc.py:436-490 (compute_mixed / _lifted_gradient_form)
//   pass B  (flux):   R = -int f(u,q) . grad(phi) - int s phi + oint f^ phi
//                     disc.py:595-653, 657-821 (interior + boundary f^)
//
// Exactness identities used (all hold to roundoff for affine elements on
// GLL nodes with the default 2p+1 quadrature):
//   * M_e = detJ * M1 (x) M1 (x) M1 and M^-1 int grad(u) phi = grad(u) at the
//     nodes (collocation derivative D1);
//   * basis traces on a face touch only that face's nodes (GLL delta), the
//     face quadrature of a degree-p trace equals (M1 (x) M1) on face nodes,
//     so the lifted jump of pass A is c_{lo/hi}[normal index] * jump(node);
//   * for a flux linear in (u, q) with constant coefficients,
//     int f . grad(phi) = sum_r K_r F_r with F_r = detJ invjt[:,r] . f at the
//     nodes and K_r = (S1 along r) (x) (M1 along the other axes), applied by
//     sum factorisation; face terms are injected into the same stages.
//
// Thread mapping: one thread per node column (hex: (i,j) with the k-column in
// registers, quad: i with the j-column in registers); N1^(nd-1) threads per
// element, several elements per 128-thread block.  That is also exactly one
// thread per face node, which is how face work is distributed.

#include <cstdio>
#include "ldg_tensor.cuh"

namespace ldg {

constexpr int kBlock = 128;

constexpr int kSmemDoubles = 6144;   // 48 KB static shared memory

template <int N1, int ND, int NCU = 1>
struct Shape {
  static constexpr int NF = ND == 3 ? N1 * N1 : N1;          // nodes per face
  static constexpr int NB = ND == 3 ? N1 * N1 * N1 : N1 * N1;
  static constexpr int TPE = NF;                             // threads/element
  static constexpr int NFACE = 2 * ND;
  // per-element shared doubles of the largest (flux) kernel
  static constexpr int PER_ELEM = NCU * NB * (1 + ND) + NFACE * NF * NCU + ND * NB;
  static constexpr int EPB_T = (kBlock / TPE) > 0 ? (kBlock / TPE) : 1;
  static constexpr int EPB_S = kSmemDoubles / PER_ELEM > 0 ? kSmemDoubles / PER_ELEM : 1;
  static constexpr int EPB = EPB_T < EPB_S ? EPB_T : EPB_S;
};

// volume node index of face node t on local face lf
template <int N1, int ND>
__device__ __forceinline__ int face_vol_node(int lf, int t) {
  const int ax = face_axis(ND, lf);
  const int io = face_side(ND, lf) ? N1 - 1 : 0;
  if (ND == 2) return ax == 0 ? io + N1 * t : t + N1 * io;
  const int a = t % N1, b = t / N1;
  if (ax == 0) return io + N1 * a + N1 * N1 * b;
  if (ax == 1) return a + N1 * io + N1 * N1 * b;
  return a + N1 * b + N1 * N1 * io;
}

__device__ __forceinline__ void flag_bad(const TensorParams& P, int e, double v) {
  if (!isfinite(v)) atomicMin(P.bad, (unsigned long long)e);
}

// --------------------------------------------------------------------------
// pass A: mixed gradient
// --------------------------------------------------------------------------

template <int N1, int ND, int NCU>
__global__ void __launch_bounds__(kBlock)
mixed_kernel(const __grid_constant__ TensorParams P,
             const double* __restrict__ u, const double* __restrict__ gproj,
             double* __restrict__ q) {
  using S = Shape<N1, ND, NCU>;
  constexpr int NB = S::NB, NF = S::NF, TPE = S::TPE, EPB = S::EPB;
  __shared__ double su[EPB][NCU][NB];
  __shared__ double sj[EPB][S::NFACE][NF][NCU];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;
  const int i = lt % N1, j = ND == 3 ? lt / N1 : 0;

  double uc[NCU][N1];
  if (active) {
    const double* ue = u + (size_t)e * NB * NCU;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        uc[c][k] = __ldg(ue + node * NCU + c);
        su[slot][c][node] = uc[c][k];
      }
    }
  }
  __syncthreads();
  // face jumps u - u^ at this thread's face node t = lt of every face
  if (active) {
#pragma unroll
    for (int lf = 0; lf < S::NFACE; ++lf) {
      const int info = __ldg(P.finfo + e * S::NFACE + lf);
      const int nbr = __ldg(P.fnbr + e * S::NFACE + lf);
      const int kind = info & LDG_FACE_KIND_MASK;
      const int vn = face_vol_node<N1, ND>(lf, lt);
      if (kind == LDG_FACE_INTERIOR) {
        const bool right = info & LDG_FACE_SIDE_RIGHT;
        const bool sw = info & LDG_FACE_SWITCH;
        // u^ = u_L if switch else u_R (disc.py:505-513); own side is L/R
        const bool own_hat = !P.trace_centered && (sw != right);
        const int mid = info >> LDG_FACE_MAP_SHIFT;
        const int nn = own_hat ? 0 : __ldg(P.nmap + mid * NF + lt);
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          const double own = su[slot][c][vn];
          double jump = 0.0;
          if (!own_hat) {
            const double other = __ldg(nbr_row(P, u, nbr, NB * NCU) + (size_t)nn * NCU + c);
            jump = P.trace_centered ? 0.5 * (own - other) : own - other;
          }
          sj[slot][lf][lt][c] = jump;
        }
      } else if (kind == LDG_FACE_DIRICHLET) {
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          const double g = gproj ? __ldg(gproj + ((size_t)nbr * NF + lt) * NCU + c) : 0.0;
          sj[slot][lf][lt][c] = su[slot][c][vn] - g;
        }
      } else {
#pragma unroll
        for (int c = 0; c < NCU; ++c) sj[slot][lf][lt][c] = 0.0;   // neumann: u^ = u
      }
    }
  }
  __syncthreads();
  if (!active) return;
  const double* g = P.geo + (size_t)e * (1 + ND * ND);
  double ij[ND][ND];
#pragma unroll
  for (int d = 0; d < ND; ++d)
#pragma unroll
    for (int r = 0; r < ND; ++r) ij[d][r] = __ldg(g + 1 + d * ND + r);
  double* qe = q + (size_t)e * NB * NCU * ND;
#pragma unroll
  for (int c = 0; c < NCU; ++c) {
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      double gr[ND];
      if (ND == 3) {
        double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          gx = fma(P.d1[i * N1 + m], su[slot][c][m + N1 * j + N1 * N1 * k], gx);
          gy = fma(P.d1[j * N1 + m], su[slot][c][i + N1 * m + N1 * N1 * k], gy);
          gz = fma(P.d1[k * N1 + m], uc[c][m], gz);
        }
        gr[0] = gx; gr[1] = gy; if (ND == 3) gr[ND - 1] = gz;
      } else {
        double gx = 0.0, gy = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          gx = fma(P.d1[i * N1 + m], su[slot][c][m + N1 * k], gx);
          gy = fma(P.d1[k * N1 + m], uc[c][m], gy);
        }
        gr[0] = gx; gr[ND - 1] = gy;
      }
      double qd[ND];
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        double acc = 0.0;
#pragma unroll
        for (int r = 0; r < ND; ++r) acc = fma(ij[d][r], gr[r], acc);
        qd[d] = -acc;
      }
      // lifted face jumps: sgn * c_side[normal index] * jump * invjt[:, axis]
#pragma unroll
      for (int lf = 0; lf < S::NFACE; ++lf) {
        const int ax = face_axis(ND, lf);
        const bool hi = face_side(ND, lf);
        int nidx, t;
        if (ND == 3) {
          nidx = ax == 0 ? i : (ax == 1 ? j : k);
          t = ax == 0 ? j + N1 * k : (ax == 1 ? i + N1 * k : i + N1 * j);
        } else {
          nidx = ax == 0 ? i : k;
          t = ax == 0 ? k : i;
        }
        const double cf = hi ? P.chi[nidx] : P.clo[nidx];
        const double v = (hi ? cf : -cf) * sj[slot][lf][t][c];
#pragma unroll
        for (int d = 0; d < ND; ++d) qd[d] = fma(v, ij[d][ax], qd[d]);
      }
      const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        flag_bad(P, e, qd[d]);
        qe[(node * NCU + c) * ND + d] = qd[d];
      }
    }
  }
}

// --------------------------------------------------------------------------
// pass B: flux residual (value or tangent)
// --------------------------------------------------------------------------

// f_cd(u, q) for a linear constant-coefficient flux
template <int ND, int NCU>
__device__ __forceinline__ double lin_flux(const TensorParams& P, int c, int d,
                                           const double* uv, const double* qv) {
  double f = 0.0;
#pragma unroll
  for (int k = 0; k < NCU; ++k) {
    if (P.flux_uses_u) f = fma(P.au[(c * 3 + d) * LDG_MAX_NCU + k], uv[k], f);
#pragma unroll
    for (int ee = 0; ee < ND; ++ee)
      f = fma(P.aq[((c * 3 + d) * LDG_MAX_NCU + k) * 3 + ee], qv[k * ND + ee], f);
  }
  return f;
}

template <int N1, int ND, int NCU, bool TANGENT>
__global__ void __launch_bounds__(kBlock)
flux_kernel(const __grid_constant__ TensorParams P,
            const double* __restrict__ u, const double* __restrict__ q,
            const double* __restrict__ gproj, const double* __restrict__ bsrc,
            double* __restrict__ R) {
  using S = Shape<N1, ND, NCU>;
  constexpr int NB = S::NB, NF = S::NF, TPE = S::TPE, EPB = S::EPB;
  __shared__ double su[EPB][NCU][NB];
  __shared__ double sq[EPB][NCU * ND][NB];
  __shared__ double sfh[EPB][S::NFACE][NF][NCU];
  __shared__ double st[EPB][ND][NB];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;
  const int i = lt % N1, j = ND == 3 ? lt / N1 : 0;

  // faces decide whether this element needs its own u at all
  int info[S::NFACE], nbr[S::NFACE];
  bool need_u = P.flux_uses_u;
  if (active) {
#pragma unroll
    for (int lf = 0; lf < S::NFACE; ++lf) {
      info[lf] = __ldg(P.finfo + e * S::NFACE + lf);
      nbr[lf] = __ldg(P.fnbr + e * S::NFACE + lf);
      const int kind = info[lf] & LDG_FACE_KIND_MASK;
      const bool sw = info[lf] & LDG_FACE_SWITCH;
      if (kind == LDG_FACE_DIRICHLET || (kind == LDG_FACE_INTERIOR &&
                                         (P.trace_centered || !sw)))
        need_u = true;
    }
  }
  double uc[NCU][N1], qc[NCU * ND][N1];
  if (active) {
    const double* qe = q + (size_t)e * NB * NCU * ND;
    const double* ue = u + (size_t)e * NB * NCU;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
#pragma unroll
      for (int cd = 0; cd < NCU * ND; ++cd) {
        qc[cd][k] = __ldg(qe + node * NCU * ND + cd);
        sq[slot][cd][node] = qc[cd][k];
      }
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        uc[c][k] = need_u ? __ldg(ue + node * NCU + c) : 0.0;
        su[slot][c][node] = uc[c][k];
      }
    }
  }
  __syncthreads();
  double detj = 0.0, ij[ND][ND];
  if (active) {
    const double* g = P.geo + (size_t)e * (1 + ND * ND);
    detj = __ldg(g);
#pragma unroll
    for (int d = 0; d < ND; ++d)
#pragma unroll
      for (int r = 0; r < ND; ++r) ij[d][r] = __ldg(g + 1 + d * ND + r);
    // numerical flux at face node t = lt of every face, times sJ
#pragma unroll
    for (int lf = 0; lf < S::NFACE; ++lf) {
      const int ax = face_axis(ND, lf);
      const double sgn = face_side(ND, lf) ? 1.0 : -1.0;
      const int kind = info[lf] & LDG_FACE_KIND_MASK;
      const int vn = face_vol_node<N1, ND>(lf, lt);
      double len2 = 0.0;
#pragma unroll
      for (int d = 0; d < ND; ++d) len2 = fma(ij[d][ax], ij[d][ax], len2);
      const double sj = detj * sqrt(len2);       // |t1 x t2| (affine face)
      const double tau = __ldg(P.ftau + e * S::NFACE + lf);
      double uo[NCU], qo[NCU * ND];
#pragma unroll
      for (int c = 0; c < NCU; ++c) uo[c] = su[slot][c][vn];
#pragma unroll
      for (int cd = 0; cd < NCU * ND; ++cd) qo[cd] = sq[slot][cd][vn];
      double fh[NCU];
      if (kind == LDG_FACE_INTERIOR) {
        const bool right = info[lf] & LDG_FACE_SIDE_RIGHT;
        const bool sw = info[lf] & LDG_FACE_SWITCH;
        const int nn = __ldg(P.nmap + (info[lf] >> LDG_FACE_MAP_SHIFT) * NF + lt);
        const size_t nb0 = (size_t)nbr[lf] * NB + nn;
        // nbr u enters u^ (and the penalty) unless u^ = u_L = own or the
        // flux ignores u and the penalty vanishes (switch faces)
        const bool u_nbr = P.trace_centered || !sw || (right && P.flux_uses_u);
        const bool q_nbr = P.grad_centered || (sw != right);
        double un[NCU], qn[NCU * ND];
#pragma unroll
        for (int c = 0; c < NCU; ++c) un[c] = u_nbr ? __ldg(u + nb0 * NCU + c) : 0.0;
#pragma unroll
        for (int cd = 0; cd < NCU * ND; ++cd)
          qn[cd] = q_nbr ? __ldg(q + nb0 * NCU * ND + cd) : 0.0;
        double uh[NCU], pen[NCU], qh[NCU * ND];
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          const double ul = right ? un[c] : uo[c], ur = right ? uo[c] : un[c];
          uh[c] = P.trace_centered ? 0.5 * (ul + ur) : (sw ? ul : ur);
          // sigma_side * tau * (u_L - u^)   (disc.py:694-698, frozen tau)
          pen[c] = (right ? -tau : tau) * (ul - uh[c]);
        }
#pragma unroll
        for (int cd = 0; cd < NCU * ND; ++cd) {
          const double ql = right ? qn[cd] : qo[cd], qr = right ? qo[cd] : qn[cd];
          qh[cd] = P.grad_centered ? 0.5 * (ql + qr) : (sw ? qr : ql);
        }
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          double fa = 0.0;
#pragma unroll
          for (int d = 0; d < ND; ++d) fa = fma(lin_flux<ND, NCU>(P, c, d, uh, qh), ij[d][ax], fa);
          fh[c] = sgn * detj * fa + sj * pen[c];
        }
      } else if (kind == LDG_FACE_DIRICHLET) {
        // f(g, q_b).n + tau_b (u_b - g); tangent: f(0, dq_b).n + tau_b du_b
        double gv[NCU];
#pragma unroll
        for (int c = 0; c < NCU; ++c)
          gv[c] = (!TANGENT && gproj) ? __ldg(gproj + ((size_t)nbr[lf] * NF + lt) * NCU + c) : 0.0;
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          double fa = 0.0;
#pragma unroll
          for (int d = 0; d < ND; ++d) fa = fma(lin_flux<ND, NCU>(P, c, d, gv, qo), ij[d][ax], fa);
          fh[c] = sgn * detj * fa + sj * tau * (uo[c] - gv[c]);
        }
      } else {
        // neumann: prescribed g, zero tangent (disc.py:775-782)
#pragma unroll
        for (int c = 0; c < NCU; ++c)
          fh[c] = (!TANGENT && gproj) ? sj * __ldg(gproj + ((size_t)nbr[lf] * NF + lt) * NCU + c) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < NCU; ++c) sfh[slot][lf][lt][c] = fh[c];
    }
  }
  __syncthreads();

  double* Re = R + (size_t)(active ? e : 0) * NB * NCU;
#pragma unroll
  for (int c = 0; c < NCU; ++c) {
    // F_r = detJ * sum_d invjt[d][r] f_cd at the column's nodes
    double F[ND][N1];
    if (active) {
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        double uv[NCU], qv[NCU * ND];
#pragma unroll
        for (int cc = 0; cc < NCU; ++cc) uv[cc] = uc[cc][k];
#pragma unroll
        for (int cd = 0; cd < NCU * ND; ++cd) qv[cd] = qc[cd][k];
        double f[ND];
#pragma unroll
        for (int d = 0; d < ND; ++d) f[d] = lin_flux<ND, NCU>(P, c, d, uv, qv);
#pragma unroll
        for (int r = 0; r < ND; ++r) {
          double a = 0.0;
#pragma unroll
          for (int d = 0; d < ND; ++d) a = fma(ij[d][r], f[d], a);
          F[r][k] = detj * a;
        }
      }
    }
    if (ND == 3) {
      // stage z (registers): A1 = M_z F_x, A2 = M_z F_y, A3 = S_z F_z - zfaces
      double A[3][N1];
      if (active) {
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            a1 = fma(P.m1[k * N1 + m], F[0][m], a1);
            a2 = fma(P.m1[k * N1 + m], F[1][m], a2);
            a3 = fma(P.s1[k * N1 + m], F[ND - 1][m], a3);
          }
          A[0][k] = a1; A[1][k] = a2; A[2][k] = a3;
        }
        A[2][0] -= sfh[slot][0][i + N1 * j][c];
        A[2][N1 - 1] -= sfh[slot][1][i + N1 * j][c];
#pragma unroll
        for (int k = 0; k < N1; ++k)
#pragma unroll
          for (int r = 0; r < 3; ++r) st[slot][r][i + N1 * j + N1 * N1 * k] = A[r][k];
      }
      __syncthreads();
      // stage y: B1 = M_y A1, B23 = S_y A2 + M_y A3 - M_z yfaces
      double B1[N1], B23[N1];
      if (active) {
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double b1 = 0.0, b2 = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            const int nd_ = i + N1 * m + N1 * N1 * k;
            b1 = fma(P.m1[j * N1 + m], st[slot][0][nd_], b1);
            b2 = fma(P.s1[j * N1 + m], st[slot][1][nd_], b2);
            b2 = fma(P.m1[j * N1 + m], st[slot][2][nd_], b2);
          }
          B1[k] = b1; B23[k] = b2;
        }
        if (j == 0 || j == N1 - 1) {
          const int lf = j == 0 ? 2 : 3;
#pragma unroll
          for (int k = 0; k < N1; ++k) {
            double a = 0.0;
#pragma unroll
            for (int m = 0; m < N1; ++m) a = fma(P.m1[k * N1 + m], sfh[slot][lf][i + N1 * m][c], a);
            B23[k] -= a;
          }
        }
      }
      __syncthreads();
      if (active) {
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          st[slot][0][i + N1 * j + N1 * N1 * k] = B1[k];
          st[slot][1][i + N1 * j + N1 * N1 * k] = B23[k];
        }
      }
      __syncthreads();
      // stage x: R = -(S_x B1 + M_x B23) + M_y M_z xfaces
      if (active) {
        double X[N1];
        if (i == 0 || i == N1 - 1) {
          const int lf = i == 0 ? 4 : 5;
          double T[N1][N1];      // T[m][k] = sum_n M[k][n] F^[m + N1 n]
#pragma unroll
          for (int m = 0; m < N1; ++m)
#pragma unroll
            for (int k = 0; k < N1; ++k) {
              double a = 0.0;
#pragma unroll
              for (int n = 0; n < N1; ++n) a = fma(P.m1[k * N1 + n], sfh[slot][lf][m + N1 * n][c], a);
              T[m][k] = a;
            }
#pragma unroll
          for (int k = 0; k < N1; ++k) {
            double a = 0.0;
#pragma unroll
            for (int m = 0; m < N1; ++m) a = fma(P.m1[j * N1 + m], T[m][k], a);
            X[k] = a;
          }
        } else {
#pragma unroll
          for (int k = 0; k < N1; ++k) X[k] = 0.0;
        }
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double r = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            const int nd_ = m + N1 * j + N1 * N1 * k;
            r = fma(P.s1[i * N1 + m], st[slot][0][nd_], r);
            r = fma(P.m1[i * N1 + m], st[slot][1][nd_], r);
          }
          const int node = i + N1 * j + N1 * N1 * k;
          double out = X[k] - r;
          if (!TANGENT && bsrc) out += __ldg(bsrc + ((size_t)e * NB + node) * NCU + c);
          flag_bad(P, e, out);
          Re[node * NCU + c] = out;
        }
      }
      __syncthreads();
    } else {
      // quad: stage y (registers): A1 = M_y F_x, A2 = S_y F_y - yfaces
      double A1[N1], A2[N1];
      if (active) {
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double a1 = 0.0, a2 = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            a1 = fma(P.m1[k * N1 + m], F[0][m], a1);
            a2 = fma(P.s1[k * N1 + m], F[ND - 1][m], a2);
          }
          A1[k] = a1; A2[k] = a2;
        }
        A2[0] -= sfh[slot][0][i][c];
        A2[N1 - 1] -= sfh[slot][2][i][c];
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          st[slot][0][i + N1 * k] = A1[k];
          st[slot][1][i + N1 * k] = A2[k];
        }
      }
      __syncthreads();
      if (active) {
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double r = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            r = fma(P.s1[i * N1 + m], st[slot][0][m + N1 * k], r);
            r = fma(P.m1[i * N1 + m], st[slot][1][m + N1 * k], r);
          }
          double x = 0.0;
          if (i == 0 || i == N1 - 1) {
            const int lf = i == 0 ? 3 : 1;
#pragma unroll
            for (int m = 0; m < N1; ++m) x = fma(P.m1[k * N1 + m], sfh[slot][lf][m][c], x);
          }
          const int node = i + N1 * k;
          double out = x - r;
          if (!TANGENT && bsrc) out += __ldg(bsrc + ((size_t)e * NB + node) * NCU + c);
          flag_bad(P, e, out);
          Re[node * NCU + c] = out;
        }
      }
      __syncthreads();
    }
  }
}

// --------------------------------------------------------------------------
// constant mass operator and its inverse: out = scale*detJ*m_c*(M1^(x)nd) v
// or out = detJ^-1 (M1^-1)^(x)nd v
// --------------------------------------------------------------------------

template <int N1, int ND, int NCU, bool INV>
__global__ void __launch_bounds__(kBlock)
mass_kernel(const __grid_constant__ TensorParams P, const double* __restrict__ v,
            double scale, double* __restrict__ out) {
  using S = Shape<N1, ND, NCU>;
  constexpr int NB = S::NB, TPE = S::TPE, EPB = S::EPB;
  __shared__ double sv[EPB][NB];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;
  const int i = lt % N1, j = ND == 3 ? lt / N1 : 0;
  const double* Mop = INV ? P.m1inv : P.m1;
  double detj = active ? __ldg(P.geo + (size_t)e * (1 + ND * ND)) : 1.0;
  for (int c = 0; c < NCU; ++c) {
    double col[N1], w[N1];
    if (active) {
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
        col[k] = __ldg(v + ((size_t)e * NB + node) * NCU + c);
      }
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) a = fma(Mop[k * N1 + m], col[m], a);
        w[k] = a;
      }
#pragma unroll
      for (int k = 0; k < N1; ++k)
        sv[slot][ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k] = w[k];
    }
    __syncthreads();
    if (ND == 3) {
      if (active) {
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double a = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) a = fma(Mop[j * N1 + m], sv[slot][i + N1 * m + N1 * N1 * k], a);
          w[k] = a;
        }
      }
      __syncthreads();
      if (active)
#pragma unroll
        for (int k = 0; k < N1; ++k) sv[slot][i + N1 * j + N1 * N1 * k] = w[k];
      __syncthreads();
    }
    if (active) {
      const double f = INV ? 1.0 / detj : scale * detj * P.mass_coef[c];
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m)
          a = fma(Mop[i * N1 + m], sv[slot][ND == 3 ? m + N1 * j + N1 * N1 * k : m + N1 * k], a);
        const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
        out[((size_t)e * NB + node) * NCU + c] = f * a;
      }
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------------------
// dispatch
// --------------------------------------------------------------------------

template <int N1, int ND, int NCU>
static int run_mixed(const TensorParams& P, const double* u, const double* g,
                     double* q, cudaStream_t s) {
  using S = Shape<N1, ND, NCU>;
  const int grid = (P.ne + S::EPB - 1) / S::EPB;
  if (grid > 0) mixed_kernel<N1, ND, NCU><<<grid, kBlock, 0, s>>>(P, u, g, q);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int N1, int ND, int NCU>
static int run_flux(const TensorParams& P, bool tan, const double* u,
                    const double* q, const double* g, const double* b,
                    double* R, cudaStream_t s) {
  using S = Shape<N1, ND, NCU>;
  const int grid = (P.ne + S::EPB - 1) / S::EPB;
  if (grid > 0) {
    if (tan) flux_kernel<N1, ND, NCU, true><<<grid, kBlock, 0, s>>>(P, u, q, g, b, R);
    else flux_kernel<N1, ND, NCU, false><<<grid, kBlock, 0, s>>>(P, u, q, g, b, R);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int N1, int ND, int NCU>
static int run_mass(const TensorParams& P, bool inv, const double* v, double sc,
                    double* out, cudaStream_t s) {
  using S = Shape<N1, ND, NCU>;
  const int grid = (P.ne + S::EPB - 1) / S::EPB;
  if (grid > 0) {
    if (inv) mass_kernel<N1, ND, NCU, true><<<grid, kBlock, 0, s>>>(P, v, sc, out);
    else mass_kernel<N1, ND, NCU, false><<<grid, kBlock, 0, s>>>(P, v, sc, out);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

#define LDG_DISPATCH(FN, ...)                                                   \
  switch (P.nd * 1000 + P.n1 * 10 + P.ncu) {                                    \
    case 3021: return FN<2, 3, 1>(__VA_ARGS__);                                 \
    case 3031: return FN<3, 3, 1>(__VA_ARGS__);                                 \
    case 3041: return FN<4, 3, 1>(__VA_ARGS__);                                 \
    case 3051: return FN<5, 3, 1>(__VA_ARGS__);                                 \
    case 3061: return FN<6, 3, 1>(__VA_ARGS__);                                 \
    case 3071: return FN<7, 3, 1>(__VA_ARGS__);                                 \
    case 3023: return FN<2, 3, 3>(__VA_ARGS__);                                 \
    case 3033: return FN<3, 3, 3>(__VA_ARGS__);                                 \
    case 3043: return FN<4, 3, 3>(__VA_ARGS__);                                 \
    case 2021: return FN<2, 2, 1>(__VA_ARGS__);                                 \
    case 2031: return FN<3, 2, 1>(__VA_ARGS__);                                 \
    case 2041: return FN<4, 2, 1>(__VA_ARGS__);                                 \
    case 2051: return FN<5, 2, 1>(__VA_ARGS__);                                 \
    case 2061: return FN<6, 2, 1>(__VA_ARGS__);                                 \
    case 2071: return FN<7, 2, 1>(__VA_ARGS__);                                 \
    case 2022: return FN<2, 2, 2>(__VA_ARGS__);                                 \
    case 2032: return FN<3, 2, 2>(__VA_ARGS__);                                 \
    case 2042: return FN<4, 2, 2>(__VA_ARGS__);                                 \
    case 2052: return FN<5, 2, 2>(__VA_ARGS__);                                 \
    default: return 2;                                                          \
  }

int launch_mixed(const TensorParams& P, const double* u, const double* gproj,
                 double* q, cudaStream_t s) {
  LDG_DISPATCH(run_mixed, P, u, gproj, q, s)
}

int launch_flux(const TensorParams& P, bool tangent, const double* u,
                const double* q, const double* gproj, const double* bsrc,
                double* R, cudaStream_t s) {
  LDG_DISPATCH(run_flux, P, tangent, u, q, gproj, bsrc, R, s)
}

int launch_mass(const TensorParams& P, bool inverse, const double* v,
                double scale, double* out, cudaStream_t s) {
  LDG_DISPATCH(run_mass, P, inverse, v, scale, out, s)
}

}  // namespace ldg
