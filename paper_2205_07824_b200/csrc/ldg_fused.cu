// Fused two-pass LDG operator for tensor-product elements (sm_100a).
//
// The reference evaluates R(u) (and J(u)du) as compute_mixed -> flux: the
// mixed gradient q is a full (ne, nb, ncu, nd) array written and re-read
// (disc.py:601-653), 72 B/DOF of compulsory HBM traffic at nd = 3.  Here q
// never leaves the SM:
//
//   pass 1 (fused_kernel), per element, all on-chip:
//     face jumps u - u^  ->  q = -grad u + lifted jumps (disc.py:436-490)
//     volume flux   -int f(u,q) . grad(phi)          (disc.py:606-629)
//     every face-flux term that depends on own data only: f(u^,.) part,
//     penalty tau (u_L - u^), the own share of f(.,q^) (disc.py:657-821)
//     exports X = sJ n . (Aq q) at the face nodes a neighbour takes q^ from
//   pass 2 (complete_kernel), per element:
//     adds the neighbour share of f(., q^): -w X_nbr lifted by (M1 (x) M1)
//     onto the face nodes (read-modify-write of R).
//
// Traffic per DOF (hex p=3, switch faces): pass 1 reads u (8 B) and writes R
// (8 B) + exports (6 B); pass 2 reads/writes R (16 B) + exports (6 B):
// ~44 B/DOF instead of 72.  Same arithmetic identities as ldg_tensor.cu
// (affine elements, GLL nodes, exact 2p+1 quadrature).
//
// Mapping: one thread per node column ((i,j) with the k column in registers
// for hex, i with the j column for quads) = one thread per face node.

#include "ldg_tensor.cuh"

namespace ldg {

namespace {

constexpr int kFBlock = 128;
constexpr int kFSmemDoubles = 6144;   // 48 KB static

template <int N1, int ND, int NCU>
struct FShape {
  static constexpr int NF = ND == 3 ? N1 * N1 : N1;
  static constexpr int NB = ND == 3 ? N1 * N1 * N1 : N1 * N1;
  static constexpr int TPE = NF;
  static constexpr int NFACE = 2 * ND;
  static constexpr int NQ = NCU * ND;                  // q components
  static constexpr int NBIG = NQ > ND ? NQ : ND;       // sdq / stage planes
  static constexpr int PER_ELEM = NCU * NB + NBIG * NB + 2 * NFACE * NF * NCU;
  static constexpr int EPB_T = (kFBlock / TPE) > 0 ? (kFBlock / TPE) : 1;
  static constexpr int EPB_S = kFSmemDoubles / PER_ELEM > 0 ? kFSmemDoubles / PER_ELEM : 1;
  static constexpr int EPB = EPB_T < EPB_S ? EPB_T : EPB_S;
};

template <int N1, int ND>
__device__ __forceinline__ int fvol(int lf, int t) {
  const int ax = face_axis(ND, lf);
  const int io = face_side(ND, lf) ? N1 - 1 : 0;
  if (ND == 2) return ax == 0 ? io + N1 * t : t + N1 * io;
  const int a = t % N1, b = t / N1;
  if (ax == 0) return io + N1 * a + N1 * N1 * b;
  if (ax == 1) return a + N1 * io + N1 * N1 * b;
  return a + N1 * b + N1 * N1 * io;
}

// face-node index of volume node v on a face with normal axis ax
template <int N1, int ND>
__device__ __forceinline__ int vol_to_face(int ax, int v) {
  if (ND == 2) return ax == 0 ? v / N1 : v % N1;
  const int i = v % N1, j = (v / N1) % N1, k = v / (N1 * N1);
  return ax == 0 ? j + N1 * k : (ax == 1 ? i + N1 * k : i + N1 * j);
}

__device__ __forceinline__ void bad_if(const TensorParams& P, int e, double v) {
  if (!isfinite(v)) atomicMin(P.bad, (unsigned long long)e);
}

}  // namespace

// --------------------------------------------------------------------------
// pass 1
// --------------------------------------------------------------------------

template <int N1, int ND, int NCU, bool TANGENT>
__global__ void __launch_bounds__(kFBlock)
fused_kernel(const __grid_constant__ TensorParams P, const double* __restrict__ u,
             const double* __restrict__ gproj, const double* __restrict__ bsrc,
             double* __restrict__ R, double* __restrict__ X) {
  using S = FShape<N1, ND, NCU>;
  constexpr int NB = S::NB, NF = S::NF, TPE = S::TPE, EPB = S::EPB, NFACE = S::NFACE;
  constexpr int NQ = S::NQ;
  __shared__ double su[EPB][NCU][NB];
  __shared__ double sbig[EPB][S::NBIG][NB];     // q, then sum-factorisation stages
  __shared__ double sj[EPB][NFACE][NF][NCU];    // jumps u - u^
  __shared__ double sfh[EPB][NFACE][NF][NCU];   // sJ * f^ (own share)
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;
  const int i = lt % N1, j = ND == 3 ? lt / N1 : 0;
  auto node_of = [&](int k) { return ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k; };

  double uc[NCU][N1];
  double detj = 1.0, ij[ND][ND];
  if (active) {
    const double* ue = u + (size_t)e * NB * NCU;
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        uc[c][k] = __ldg(ue + node_of(k) * NCU + c);
        su[slot][c][node_of(k)] = uc[c][k];
      }
    const double* g = P.geo + (size_t)e * (1 + ND * ND);
    detj = __ldg(g);
#pragma unroll
    for (int d = 0; d < ND; ++d)
#pragma unroll
      for (int r = 0; r < ND; ++r) ij[d][r] = __ldg(g + 1 + d * ND + r);
  }
  __syncthreads();

  // ---- step 2: jumps and the u-dependent part of sJ f^ at face node lt
  int info[NFACE];
  if (active) {
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      info[lf] = __ldg(P.finfo + e * NFACE + lf);
      const int nbr = __ldg(P.fnbr + e * NFACE + lf);
      const int kind = info[lf] & LDG_FACE_KIND_MASK;
      const int ax = face_axis(ND, lf);
      const double sgn = face_side(ND, lf) ? 1.0 : -1.0;
      const int vn = fvol<N1, ND>(lf, lt);
      double len2 = 0.0;
#pragma unroll
      for (int d = 0; d < ND; ++d) len2 = fma(ij[d][ax], ij[d][ax], len2);
      const double sjac = detj * sqrt(len2);
      const double tau = __ldg(P.ftau + e * NFACE + lf);
      double uo[NCU], uh[NCU], fh[NCU], jmp[NCU];
#pragma unroll
      for (int c = 0; c < NCU; ++c) uo[c] = su[slot][c][vn];
      if (kind == LDG_FACE_INTERIOR) {
        const bool right = info[lf] & LDG_FACE_SIDE_RIGHT;
        const bool sw = info[lf] & LDG_FACE_SWITCH;
        const bool hat_nbr = P.trace_centered || (sw == right);
        const bool pen_nbr = P.trace_centered || !sw;
        double un[NCU];
        if (hat_nbr || pen_nbr) {
          const int nn = __ldg(P.nmap + (info[lf] >> LDG_FACE_MAP_SHIFT) * NF + lt);
#pragma unroll
          for (int c = 0; c < NCU; ++c) un[c] = __ldg(u + ((size_t)nbr * NB + nn) * NCU + c);
        } else {
#pragma unroll
          for (int c = 0; c < NCU; ++c) un[c] = uo[c];
        }
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          const double ul = right ? un[c] : uo[c], ur = right ? uo[c] : un[c];
          uh[c] = P.trace_centered ? 0.5 * (ul + ur) : (sw ? ul : ur);
          jmp[c] = uo[c] - uh[c];
          // sigma_side * tau * (u_L - u^), frozen tau (disc.py:694-698)
          fh[c] = sjac * (right ? -tau : tau) * (ul - uh[c]);
        }
      } else if (kind == LDG_FACE_DIRICHLET) {
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          uh[c] = (!TANGENT && gproj) ? __ldg(gproj + ((size_t)nbr * NF + lt) * NCU + c) : 0.0;
          jmp[c] = uo[c] - uh[c];
          fh[c] = sjac * tau * jmp[c];                   // tau_b (u_b - g)
        }
      } else {
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          uh[c] = uo[c];
          jmp[c] = 0.0;
          fh[c] = (!TANGENT && gproj) ? sjac * __ldg(gproj + ((size_t)nbr * NF + lt) * NCU + c)
                                      : 0.0;
        }
      }
      if (P.flux_uses_u && kind != LDG_FACE_NEUMANN) {
        // sJ n . (Au u^) = detJ sgn sum_d (Au u^)_d invjt[d][ax]
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          double a = 0.0;
#pragma unroll
          for (int d = 0; d < ND; ++d) {
            double f = 0.0;
#pragma unroll
            for (int kk = 0; kk < NCU; ++kk) f = fma(P.au[(c * 3 + d) * LDG_MAX_NCU + kk], uh[kk], f);
            a = fma(f, ij[d][ax], a);
          }
          fh[c] = fma(sgn * detj, a, fh[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        sj[slot][lf][lt][c] = jmp[c];
        sfh[slot][lf][lt][c] = fh[c];
      }
    }
  }
  __syncthreads();

  // ---- step 3: q column, then F_r = detJ invjt[:,r] . f(u, q)
  double F[NCU][ND][N1];
  if (active) {
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      double q[NQ];
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double gr[ND];
        double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          if (ND == 3) {
            gx = fma(P.d1[i * N1 + m], su[slot][c][m + N1 * j + N1 * N1 * k], gx);
            gy = fma(P.d1[j * N1 + m], su[slot][c][i + N1 * m + N1 * N1 * k], gy);
            gz = fma(P.d1[k * N1 + m], uc[c][m], gz);
          } else {
            gx = fma(P.d1[i * N1 + m], su[slot][c][m + N1 * k], gx);
            gy = fma(P.d1[k * N1 + m], uc[c][m], gy);
          }
        }
        gr[0] = gx;
        gr[1] = gy;
        if (ND == 3) gr[ND - 1] = gz;
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          double a = 0.0;
#pragma unroll
          for (int r = 0; r < ND; ++r) a = fma(ij[d][r], gr[r], a);
          q[c * ND + d] = -a;
        }
#pragma unroll
        for (int lf = 0; lf < NFACE; ++lf) {
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
          for (int d = 0; d < ND; ++d) q[c * ND + d] = fma(v, ij[d][ax], q[c * ND + d]);
        }
      }
#pragma unroll
      for (int cd = 0; cd < NQ; ++cd) sbig[slot][cd][node_of(k)] = q[cd];
      // volume flux density in reference directions
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double f[ND];
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          double a = 0.0;
#pragma unroll
          for (int kk = 0; kk < NCU; ++kk) {
            if (P.flux_uses_u) a = fma(P.au[(c * 3 + d) * LDG_MAX_NCU + kk], uc[kk][k], a);
#pragma unroll
            for (int ee = 0; ee < ND; ++ee)
              a = fma(P.aq[((c * 3 + d) * LDG_MAX_NCU + kk) * 3 + ee], q[kk * ND + ee], a);
          }
          f[d] = a;
        }
#pragma unroll
        for (int r = 0; r < ND; ++r) {
          double a = 0.0;
#pragma unroll
          for (int d = 0; d < ND; ++d) a = fma(ij[d][r], f[d], a);
          F[c][r][k] = detj * a;
        }
      }
    }
  }
  __syncthreads();

  // ---- step 4: own share of n . (Aq q^) and exports, face node lt
  if (active) {
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const int kind = info[lf] & LDG_FACE_KIND_MASK;
      if (kind == LDG_FACE_NEUMANN) continue;
      const int ax = face_axis(ND, lf);
      const double sgn = face_side(ND, lf) ? 1.0 : -1.0;
      const int vn = fvol<N1, ND>(lf, lt);
      double w_own = 1.0;
      bool exp_ = false;
      if (kind == LDG_FACE_INTERIOR) {
        const bool right = info[lf] & LDG_FACE_SIDE_RIGHT;
        const bool sw = info[lf] & LDG_FACE_SWITCH;
        const bool mine = sw == right;                  // q^ = this side's q
        w_own = P.grad_centered ? 0.5 : (mine ? 1.0 : 0.0);
        exp_ = P.grad_centered || mine;
      }
      if (w_own == 0.0 && !exp_) continue;
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double a = 0.0;
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          double f = 0.0;
#pragma unroll
          for (int kk = 0; kk < NCU; ++kk)
#pragma unroll
            for (int ee = 0; ee < ND; ++ee)
              f = fma(P.aq[((c * 3 + d) * LDG_MAX_NCU + kk) * 3 + ee], sbig[slot][kk * ND + ee][vn], f);
          a = fma(f, ij[d][ax], a);
        }
        const double xf = sgn * detj * a;               // sJ n . (Aq q)
        sfh[slot][lf][lt][c] = fma(w_own, xf, sfh[slot][lf][lt][c]);
        if (exp_) X[(((size_t)e * NFACE + lf) * NF + lt) * NCU + c] = xf;
      }
    }
  }
  __syncthreads();

  // ---- step 5: R = -sum_r K_r F_r + injected face terms (+ source load)
  double* Re = R + (size_t)(active ? e : 0) * NB * NCU;
#pragma unroll
  for (int c = 0; c < NCU; ++c) {
    if (ND == 3) {
      double A[3][N1];
      if (active) {
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            a1 = fma(P.m1[k * N1 + m], F[c][0][m], a1);
            a2 = fma(P.m1[k * N1 + m], F[c][1][m], a2);
            a3 = fma(P.s1[k * N1 + m], F[c][ND - 1][m], a3);
          }
          A[0][k] = a1; A[1][k] = a2; A[2][k] = a3;
        }
        A[2][0] -= sfh[slot][0][i + N1 * j][c];
        A[2][N1 - 1] -= sfh[slot][1][i + N1 * j][c];
#pragma unroll
        for (int k = 0; k < N1; ++k)
#pragma unroll
          for (int r = 0; r < 3; ++r) sbig[slot][r][i + N1 * j + N1 * N1 * k] = A[r][k];
      }
      __syncthreads();
      double B1[N1], B23[N1];
      if (active) {
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double b1 = 0.0, b2 = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            const int nd_ = i + N1 * m + N1 * N1 * k;
            b1 = fma(P.m1[j * N1 + m], sbig[slot][0][nd_], b1);
            b2 = fma(P.s1[j * N1 + m], sbig[slot][1][nd_], b2);
            b2 = fma(P.m1[j * N1 + m], sbig[slot][2][nd_], b2);
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
          sbig[slot][0][i + N1 * j + N1 * N1 * k] = B1[k];
          sbig[slot][1][i + N1 * j + N1 * N1 * k] = B23[k];
        }
      }
      __syncthreads();
      if (active) {
        double Xv[N1];
#pragma unroll
        for (int k = 0; k < N1; ++k) Xv[k] = 0.0;
        if (i == 0 || i == N1 - 1) {
          const int lf = i == 0 ? 4 : 5;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            double col[N1];
#pragma unroll
            for (int n = 0; n < N1; ++n) col[n] = sfh[slot][lf][m + N1 * n][c];
            const double mj = P.m1[j * N1 + m];
#pragma unroll
            for (int k = 0; k < N1; ++k) {
              double a = 0.0;
#pragma unroll
              for (int n = 0; n < N1; ++n) a = fma(P.m1[k * N1 + n], col[n], a);
              Xv[k] = fma(mj, a, Xv[k]);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double r = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            const int nd_ = m + N1 * j + N1 * N1 * k;
            r = fma(P.s1[i * N1 + m], sbig[slot][0][nd_], r);
            r = fma(P.m1[i * N1 + m], sbig[slot][1][nd_], r);
          }
          const int node = node_of(k);
          double out = Xv[k] - r;
          if (!TANGENT && bsrc) out += __ldg(bsrc + ((size_t)e * NB + node) * NCU + c);
          bad_if(P, e, out);
          Re[node * NCU + c] = out;
        }
      }
      __syncthreads();
    } else {
      double A1[N1], A2[N1];
      if (active) {
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double a1 = 0.0, a2 = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            a1 = fma(P.m1[k * N1 + m], F[c][0][m], a1);
            a2 = fma(P.s1[k * N1 + m], F[c][ND - 1][m], a2);
          }
          A1[k] = a1; A2[k] = a2;
        }
        A2[0] -= sfh[slot][0][i][c];
        A2[N1 - 1] -= sfh[slot][2][i][c];
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          sbig[slot][0][i + N1 * k] = A1[k];
          sbig[slot][1][i + N1 * k] = A2[k];
        }
      }
      __syncthreads();
      if (active) {
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double r = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            r = fma(P.s1[i * N1 + m], sbig[slot][0][m + N1 * k], r);
            r = fma(P.m1[i * N1 + m], sbig[slot][1][m + N1 * k], r);
          }
          double x = 0.0;
          if (i == 0 || i == N1 - 1) {
            const int lf = i == 0 ? 3 : 1;
#pragma unroll
            for (int m = 0; m < N1; ++m) x = fma(P.m1[k * N1 + m], sfh[slot][lf][m][c], x);
          }
          const int node = node_of(k);
          double out = x - r;
          if (!TANGENT && bsrc) out += __ldg(bsrc + ((size_t)e * NB + node) * NCU + c);
          bad_if(P, e, out);
          Re[node * NCU + c] = out;
        }
      }
      __syncthreads();
    }
  }
}

// --------------------------------------------------------------------------
// pass 2: neighbour share of f(., q^) on faces whose q^ comes from across
// --------------------------------------------------------------------------

template <int N1, int ND, int NCU>
__global__ void __launch_bounds__(kFBlock)
complete_kernel(const __grid_constant__ TensorParams P, const double* __restrict__ X,
                double* __restrict__ R) {
  using S = FShape<N1, ND, NCU>;
  constexpr int NB = S::NB, NF = S::NF, TPE = S::TPE, EPB = S::EPB, NFACE = S::NFACE;
  __shared__ double sv[EPB][NFACE][NF][NCU];
  __shared__ int sact[EPB][NFACE];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;
  const int i = lt % N1, j = ND == 3 ? lt / N1 : 0;
  if (active) {
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const int info = __ldg(P.finfo + e * NFACE + lf);
      bool act = false;
      double w = 0.0;
      if ((info & LDG_FACE_KIND_MASK) == LDG_FACE_INTERIOR) {
        const bool right = info & LDG_FACE_SIDE_RIGHT;
        const bool sw = info & LDG_FACE_SWITCH;
        act = P.grad_centered || (sw != right);
        w = P.grad_centered ? 0.5 : 1.0;
      }
      if (lt == 0) sact[slot][lf] = act;
      if (act) {
        const int nbr = __ldg(P.fnbr + e * NFACE + lf);
        const int nlf = (info >> 4) & 7;
        const int nv = __ldg(P.nmap + (info >> LDG_FACE_MAP_SHIFT) * NF + lt);
        const int tn = vol_to_face<N1, ND>(face_axis(ND, nlf), nv);
#pragma unroll
        for (int c = 0; c < NCU; ++c)
          sv[slot][lf][lt][c] = -w * __ldg(X + (((size_t)nbr * NFACE + nlf) * NF + tn) * NCU + c);
      }
    }
  }
  __syncthreads();
  if (!active) return;
  double* Re = R + (size_t)e * NB * NCU;
#pragma unroll
  for (int c = 0; c < NCU; ++c) {
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      // faces containing node (i, j, k): (M1 (x) M1) of the face data
      double acc = 0.0;
      bool touched = false;
#pragma unroll
      for (int lf = 0; lf < NFACE; ++lf) {
        if (!sact[slot][lf]) continue;
        const int ax = face_axis(ND, lf);
        const int io = face_side(ND, lf) ? N1 - 1 : 0;
        const int nidx = ND == 3 ? (ax == 0 ? i : (ax == 1 ? j : k)) : (ax == 0 ? i : k);
        if (nidx != io) continue;
        touched = true;
        if (ND == 3) {
          const int a = ax == 0 ? j : i, b = ax == 2 ? j : k;    // tangential coords
#pragma unroll
          for (int bb = 0; bb < N1; ++bb) {
            double s = 0.0;
#pragma unroll
            for (int aa = 0; aa < N1; ++aa) s = fma(P.m1[a * N1 + aa], sv[slot][lf][aa + N1 * bb][c], s);
            acc = fma(P.m1[b * N1 + bb], s, acc);
          }
        } else {
          const int a = ax == 0 ? k : i;
#pragma unroll
          for (int aa = 0; aa < N1; ++aa) acc = fma(P.m1[a * N1 + aa], sv[slot][lf][aa][c], acc);
        }
      }
      if (touched) {
        const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
        const double out = Re[node * NCU + c] + acc;
        bad_if(P, e, out);
        Re[node * NCU + c] = out;
      }
    }
  }
}

// --------------------------------------------------------------------------
// dispatch
// --------------------------------------------------------------------------

template <int N1, int ND, int NCU>
static int run_pass(const TensorParams& P, int pass, bool tangent, const double* u,
                    const double* gproj, const double* bsrc, double* R, double* X,
                    cudaStream_t s) {
  using S = FShape<N1, ND, NCU>;
  const int grid = (P.ne + S::EPB - 1) / S::EPB;
  if (grid <= 0) return 0;
  if (pass & 1) {
    if (tangent) fused_kernel<N1, ND, NCU, true><<<grid, kFBlock, 0, s>>>(P, u, gproj, bsrc, R, X);
    else fused_kernel<N1, ND, NCU, false><<<grid, kFBlock, 0, s>>>(P, u, gproj, bsrc, R, X);
    if (cudaGetLastError() != cudaSuccess) return 3;
  }
  if (pass & 2) complete_kernel<N1, ND, NCU><<<grid, kFBlock, 0, s>>>(P, X, R);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int N1, int ND, int NCU>
static int run_fused(const TensorParams& P, bool tangent, const double* u,
                     const double* gproj, const double* bsrc, double* R, double* X,
                     cudaStream_t s) {
  return run_pass<N1, ND, NCU>(P, 3, tangent, u, gproj, bsrc, R, X, s);
}

#define LDG_FDISPATCH(FN, ...)                                                  \
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

int launch_fused(const TensorParams& P, bool tangent, const double* u,
                 const double* gproj, const double* bsrc, double* R, double* X,
                 cudaStream_t s) {
  LDG_FDISPATCH(run_fused, P, tangent, u, gproj, bsrc, R, X, s)
}

int launch_fused_pass(const TensorParams& P, int pass, bool tangent, const double* u,
                      const double* gproj, const double* bsrc, double* R, double* X,
                      cudaStream_t s) {
  LDG_FDISPATCH(run_pass, P, pass, tangent, u, gproj, bsrc, R, X, s)
}

}  // namespace ldg
