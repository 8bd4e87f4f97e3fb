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
//
// Thread roles per element (lt in [0, TPE)):
//   column owner  (hex: (i,j), quad: i)   owns the k (quad: j) node column
//   y-pencil owner (hex only: (i,k))      owns nodes (i, 0..N1-1, k)
//   row owner     (hex: (j,k), quad: j)   owns nodes (0..N1-1, j, k) (contiguous)
//   face-node     (t = lt on every face)
// Every 1D contraction is done by the owner of the pencil along its axis, so
// all operator indices are compile-time (constant-bank DFMA operands) and
// each shared-memory value loaded feeds N1 FMAs.
//
// q is never formed: with h_s = -d_s u + sum_{faces f with axis s} lift_f,
// q = invjt h, and the flux density in reference directions is
//   F_{c,r} = Cu[c][r][k] u_k + C[c][r][k][s] h_{k,s},
//   C = detJ invjt^T Aq invjt,  Cu = detJ invjt^T Au     (per element).
// The face export sJ n.(Aq q) equals sgn * F^q_{c,axis} at the face node.

template <int N1, int ND, int NCU>
struct P1Smem {
  static constexpr int NF = ND == 3 ? N1 * N1 : N1;
  static constexpr int NB = ND == 3 ? N1 * N1 * N1 : N1 * N1;
  static constexpr int NFACE = 2 * ND;
  static constexpr int NC = NCU * ND * NCU * ND + NCU * ND * NCU;   // C then Cu
  static constexpr int GSZ = (ND - 1) * NCU * NB;                   // gx (,gy) planes
  static constexpr int EXT = 6 * N1 * N1;                           // face-slab pencils
  static constexpr int WORK = GSZ > EXT ? GSZ : EXT;
  static constexpr int FSZ = NCU * ND * NB;                         // F^q, then stages
  static constexpr int FSZ2 = FSZ > ND * NB ? FSZ : ND * NB;
  static constexpr int PER = NCU * NB + WORK + FSZ2 + 2 * NFACE * NF * NCU + NC;
  static constexpr int TPE = NF;
  static constexpr int EPB_T = (kFBlock / TPE) > 0 ? (kFBlock / TPE) : 1;
  static constexpr int EPB_S = kFSmemDoubles / PER > 0 ? kFSmemDoubles / PER : 1;
  static constexpr int EPB = EPB_T < EPB_S ? EPB_T : EPB_S;
};

template <int N1, int ND, int NCU, bool TANGENT>
__global__ void __launch_bounds__(kFBlock)
fused_kernel(const __grid_constant__ TensorParams P, const double* __restrict__ u,
             const double* __restrict__ gproj, const double* __restrict__ bsrc,
             double* __restrict__ R, double* __restrict__ X) {
  using S = P1Smem<N1, ND, NCU>;
  constexpr int NB = S::NB, NF = S::NF, TPE = S::TPE, EPB = S::EPB, NFACE = S::NFACE;
  constexpr int NC = S::NC, CQ = NCU * ND * NCU * ND;
  __shared__ double su[EPB][NCU][NB];
  __shared__ double swork[EPB][S::WORK];       // gx/gy planes, then face-slab pencils
  __shared__ double sF[EPB][S::FSZ2];          // F^q planes, then stage planes
  __shared__ double sj[EPB][NFACE][NF][NCU];   // jumps u - u^
  __shared__ double sfh[EPB][NFACE][NF][NCU];  // sJ f^ (own share)
  __shared__ double sC[EPB][NC];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;
  const int ta = lt % N1, tb = ND == 3 ? lt / N1 : 0;   // (i,j) | (i,k) | (j,k) ; quad: i | j
  const int i = ta, j = tb;                              // column owner coordinates

  // ---- A: column of u, element geometry
  double uc[NCU][N1];
  double detj = 1.0, ij[ND][ND];
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
    const double* g = P.geo + (size_t)e * (1 + ND * ND);
    detj = __ldg(g);
#pragma unroll
    for (int d = 0; d < ND; ++d)
#pragma unroll
      for (int r = 0; r < ND; ++r) ij[d][r] = __ldg(g + 1 + d * ND + r);
    // C[c][r][k][s] = detJ sum_{d,e} invjt[d][r] aq[c][d][k][e] invjt[e][s];
    // Cu[c][r][k] = detJ sum_d invjt[d][r] au[c][d][k]
    // (dynamic r_/s_ indices read invjt from global/L1, keeping ij in registers)
    const double* gij = g + 1;
    for (int x = lt; x < NC; x += TPE) {
      double v = 0.0;
      if (x < CQ) {
        const int s_ = x % ND, k_ = (x / ND) % NCU, r_ = (x / (ND * NCU)) % ND,
                  c_ = x / (ND * NCU * ND);
#pragma unroll
        for (int d = 0; d < ND; ++d)
#pragma unroll
          for (int ee = 0; ee < ND; ++ee)
            v = fma(__ldg(gij + d * ND + r_) * P.aq[((c_ * 3 + d) * LDG_MAX_NCU + k_) * 3 + ee],
                    __ldg(gij + ee * ND + s_), v);
      } else {
        const int y = x - CQ;
        const int k_ = y % NCU, r_ = (y / NCU) % ND, c_ = y / (NCU * ND);
#pragma unroll
        for (int d = 0; d < ND; ++d)
          v = fma(__ldg(gij + d * ND + r_), P.au[(c_ * 3 + d) * LDG_MAX_NCU + k_], v);
      }
      sC[slot][x] = detj * v;
    }
  }
  __syncthreads();

  // ---- B: face node lt of every face: jumps and the u part of sJ f^
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
        double un[NCU];
        if (P.trace_centered || (sw == right) || !sw) {
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
          fh[c] = sjac * (right ? -tau : tau) * (ul - uh[c]);   // frozen tau (disc.py:694-698)
        }
      } else if (kind == LDG_FACE_DIRICHLET) {
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          uh[c] = (!TANGENT && gproj) ? __ldg(gproj + ((size_t)nbr * NF + lt) * NCU + c) : 0.0;
          jmp[c] = uo[c] - uh[c];
          fh[c] = sjac * tau * jmp[c];
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
        // sJ n.(Au u^) = sgn * Cu[c][ax][k] u^_k
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          double a = 0.0;
#pragma unroll
          for (int kk = 0; kk < NCU; ++kk) a = fma(sC[slot][CQ + (c * ND + ax) * NCU + kk], uh[kk], a);
          fh[c] = fma(sgn, a, fh[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        sj[slot][lf][lt][c] = jmp[c];
        sfh[slot][lf][lt][c] = fh[c];
      }
    }
  }
  // ---- C: gradient pencils (owner of the pencil along each axis)
  double gl[NCU][N1];       // gradient along the column axis (registers)
  if (active) {
#pragma unroll
    for (int c = 0; c < NCU; ++c)
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) a = fma(P.d1[k * N1 + m], uc[c][m], a);
        gl[c][k] = a;
      }
  }
  __syncthreads();          // su complete (B wrote only sj/sfh/sC)
  if (active) {
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      // row owner: x derivative of the row (0..N1-1, tb-coords)
      double row[N1];
#pragma unroll
      for (int m = 0; m < N1; ++m)
        row[m] = su[slot][c][ND == 3 ? m + N1 * ta + N1 * N1 * tb : m + N1 * ta];
#pragma unroll
      for (int a = 0; a < N1; ++a) {
        double v = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) v = fma(P.d1[a * N1 + m], row[m], v);
        swork[slot][c * NB + (ND == 3 ? a + N1 * ta + N1 * N1 * tb : a + N1 * ta)] = v;
      }
      if (ND == 3) {
        // y-pencil owner (i,k) = (ta, tb)
        double col[N1];
#pragma unroll
        for (int m = 0; m < N1; ++m) col[m] = su[slot][c][ta + N1 * m + N1 * N1 * tb];
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          double v = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) v = fma(P.d1[a * N1 + m], col[m], v);
          swork[slot][(NCU + c) * NB + ta + N1 * a + N1 * N1 * tb] = v;
        }
      }
    }
  }
  __syncthreads();

  // ---- D: h = -grad u + lifted jumps, F = Cu u + C h at the column's nodes
  double F[NCU][ND][N1];
  if (active) {
    const double cli = P.clo[i], chi_i = P.chi[i];
    const double clj = ND == 3 ? P.clo[j] : 0.0, chj = ND == 3 ? P.chi[j] : 0.0;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
      double h[NCU][ND];
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        if (ND == 3) {
          // faces: 0 z-, 1 z+, 2 y-, 3 y+, 4 x-, 5 x+
          h[c][0] = -swork[slot][c * NB + node] - cli * sj[slot][4][j + N1 * k][c]
                    + chi_i * sj[slot][5][j + N1 * k][c];
          h[c][1] = -swork[slot][(NCU + c) * NB + node] - clj * sj[slot][2][i + N1 * k][c]
                    + chj * sj[slot][3][i + N1 * k][c];
          h[c][2] = -gl[c][k] - P.clo[k] * sj[slot][0][i + N1 * j][c]
                    + P.chi[k] * sj[slot][1][i + N1 * j][c];
        } else {
          // quad faces: 0 y-, 1 x+, 2 y+, 3 x-
          h[c][0] = -swork[slot][c * NB + node] - cli * sj[slot][3][k][c]
                    + chi_i * sj[slot][1][k][c];
          h[c][ND - 1] = -gl[c][k] - P.clo[k] * sj[slot][0][i][c] + P.chi[k] * sj[slot][2][i][c];
        }
      }
#pragma unroll
      for (int c = 0; c < NCU; ++c)
#pragma unroll
        for (int r = 0; r < ND; ++r) {
          double fq = 0.0;
#pragma unroll
          for (int kk = 0; kk < NCU; ++kk)
#pragma unroll
            for (int s_ = 0; s_ < ND; ++s_)
              fq = fma(sC[slot][((c * ND + r) * NCU + kk) * ND + s_], h[kk][s_], fq);
          sF[slot][(c * ND + r) * NB + node] = fq;
          double fu = 0.0;
          if (P.flux_uses_u) {
#pragma unroll
            for (int kk = 0; kk < NCU; ++kk)
              fu = fma(sC[slot][CQ + (c * ND + r) * NCU + kk], uc[kk][k], fu);
          }
          F[c][r][k] = fq + fu;
        }
    }
  }
  __syncthreads();

  // ---- E: own share of sJ n.(Aq q^) and exports at face node lt
  if (active) {
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const int kind = info[lf] & LDG_FACE_KIND_MASK;
      if (kind == LDG_FACE_NEUMANN) continue;
      double w_own = 1.0;
      bool exp_ = false;
      if (kind == LDG_FACE_INTERIOR) {
        const bool right = info[lf] & LDG_FACE_SIDE_RIGHT;
        const bool sw = info[lf] & LDG_FACE_SWITCH;
        const bool mine = sw == right;
        w_own = P.grad_centered ? 0.5 : (mine ? 1.0 : 0.0);
        exp_ = P.grad_centered || mine;
      }
      if (w_own == 0.0 && !exp_) continue;
      const int ax = face_axis(ND, lf);
      const double sgn = face_side(ND, lf) ? 1.0 : -1.0;
      const int vn = fvol<N1, ND>(lf, lt);
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        const double xf = sgn * sF[slot][(c * ND + ax) * NB + vn];
        sfh[slot][lf][lt][c] = fma(w_own, xf, sfh[slot][lf][lt][c]);
        if (exp_) X[(((size_t)e * NFACE + lf) * NF + lt) * NCU + c] = xf;
      }
    }
  }
  __syncthreads();

  // ---- F..H: R = -sum_r K_r F_r + face terms, sum factorised by pencils
  double* Re = R + (size_t)(active ? e : 0) * NB * NCU;
  double* sP = sF[slot];         // stage planes
  double* sX = swork[slot];      // face-slab pencils
#pragma unroll
  for (int c = 0; c < NCU; ++c) {
    if (ND == 3) {
      if (active) {
        // z stage (column owner): A1 = M F_x, A2 = M F_y, A3 = S F_z - z faces
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            a1 = fma(P.m1[k * N1 + m], F[c][0][m], a1);
            a2 = fma(P.m1[k * N1 + m], F[c][1][m], a2);
            a3 = fma(P.s1[k * N1 + m], F[c][2][m], a3);
          }
          if (k == 0) a3 -= sfh[slot][0][i + N1 * j][c];
          if (k == N1 - 1) a3 -= sfh[slot][1][i + N1 * j][c];
          const int node = i + N1 * j + N1 * N1 * k;
          sP[node] = a1;
          sP[NB + node] = a2;
          sP[2 * NB + node] = a3;
        }
        // face slabs along z: p = (type x|y, side, idx), out[k] = M_z fh
        for (int p = lt; p < 4 * N1; p += TPE) {
          const int type = p / (2 * N1), side = (p / N1) & 1, idx = p % N1;
          const int lf = type == 0 ? 4 + side : 2 + side;
          double v[N1];
#pragma unroll
          for (int n = 0; n < N1; ++n) v[n] = sfh[slot][lf][idx + N1 * n][c];
#pragma unroll
          for (int k = 0; k < N1; ++k) {
            double a = 0.0;
#pragma unroll
            for (int n = 0; n < N1; ++n) a = fma(P.m1[k * N1 + n], v[n], a);
            sX[((type * 2 + side) * N1 + idx) * N1 + k] = a;
          }
        }
      }
      __syncthreads();
      double B1[N1], B23[N1];
      if (active) {
        // y stage (pencil owner (i,k) = (ta,tb))
        double a1[N1], a2[N1], a3[N1];
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          const int node = ta + N1 * m + N1 * N1 * tb;
          a1[m] = sP[node];
          a2[m] = sP[NB + node];
          a3[m] = sP[2 * NB + node];
        }
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          double b1 = 0.0, b2 = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            b1 = fma(P.m1[a * N1 + m], a1[m], b1);
            b2 = fma(P.s1[a * N1 + m], a2[m], b2);
            b2 = fma(P.m1[a * N1 + m], a3[m], b2);
          }
          B1[a] = b1;
          B23[a] = b2;
        }
        B23[0] -= sX[((1 * 2 + 0) * N1 + ta) * N1 + tb];
        B23[N1 - 1] -= sX[((1 * 2 + 1) * N1 + ta) * N1 + tb];
      }
      __syncthreads();
      if (active) {
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          const int node = ta + N1 * a + N1 * N1 * tb;
          sP[node] = B1[a];
          sP[NB + node] = B23[a];
        }
        // x-face slabs along y: Bx[side][j][k] = sum_m M[j][m] Ax[side][m][k]
        for (int p = lt; p < 2 * N1; p += TPE) {
          const int side = p / N1, k = p % N1;
          double v[N1];
#pragma unroll
          for (int m = 0; m < N1; ++m) v[m] = sX[((0 * 2 + side) * N1 + m) * N1 + k];
#pragma unroll
          for (int a = 0; a < N1; ++a) {
            double acc = 0.0;
#pragma unroll
            for (int m = 0; m < N1; ++m) acc = fma(P.m1[a * N1 + m], v[m], acc);
            sX[4 * N1 * N1 + (side * N1 + a) * N1 + k] = acc;
          }
        }
      }
      __syncthreads();
      if (active) {
        // x stage (row owner (j,k) = (ta,tb)): contiguous row
        double b1[N1], b23[N1];
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          const int node = m + N1 * ta + N1 * N1 * tb;
          b1[m] = sP[node];
          b23[m] = sP[NB + node];
        }
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          double r = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            r = fma(P.s1[a * N1 + m], b1[m], r);
            r = fma(P.m1[a * N1 + m], b23[m], r);
          }
          double out = -r;
          if (a == 0) out += sX[4 * N1 * N1 + (0 * N1 + ta) * N1 + tb];
          if (a == N1 - 1) out += sX[4 * N1 * N1 + (1 * N1 + ta) * N1 + tb];
          const int node = a + N1 * ta + N1 * N1 * tb;
          if (!TANGENT && bsrc) out += __ldg(bsrc + ((size_t)e * NB + node) * NCU + c);
          bad_if(P, e, out);
          Re[node * NCU + c] = out;
        }
      }
      __syncthreads();
    } else {
      if (active) {
        // y stage (column owner i): A1 = M F_x, A2 = S F_y - y faces
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          double a1 = 0.0, a2 = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            a1 = fma(P.m1[k * N1 + m], F[c][0][m], a1);
            a2 = fma(P.s1[k * N1 + m], F[c][ND - 1][m], a2);
          }
          if (k == 0) a2 -= sfh[slot][0][i][c];
          if (k == N1 - 1) a2 -= sfh[slot][2][i][c];
          sP[i + N1 * k] = a1;
          sP[NB + i + N1 * k] = a2;
        }
        // x-face slabs along y: Ax[side][k] = sum_n M[k][n] fh[x side][n]
        for (int p = lt; p < 2; p += TPE) {
          const int lf = p == 0 ? 3 : 1;
          double v[N1];
#pragma unroll
          for (int n = 0; n < N1; ++n) v[n] = sfh[slot][lf][n][c];
#pragma unroll
          for (int k = 0; k < N1; ++k) {
            double a = 0.0;
#pragma unroll
            for (int n = 0; n < N1; ++n) a = fma(P.m1[k * N1 + n], v[n], a);
            sX[p * N1 + k] = a;
          }
        }
      }
      __syncthreads();
      if (active) {
        // x stage (row owner j = ta)
        double a1[N1], a2[N1];
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          a1[m] = sP[m + N1 * ta];
          a2[m] = sP[NB + m + N1 * ta];
        }
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          double r = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            r = fma(P.s1[a * N1 + m], a1[m], r);
            r = fma(P.m1[a * N1 + m], a2[m], r);
          }
          double out = -r;
          if (a == 0) out += sX[0 * N1 + ta];
          if (a == N1 - 1) out += sX[1 * N1 + ta];
          const int node = a + N1 * ta;
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
struct P2Smem {
  static constexpr int NF = ND == 3 ? N1 * N1 : N1;
  static constexpr int NB = ND == 3 ? N1 * N1 * N1 : N1 * N1;
  static constexpr int NFACE = 2 * ND;
  static constexpr int TPE = NF;
  static constexpr int EPB = (kFBlock / TPE) > 0 ? (kFBlock / TPE) : 1;
};

template <int N1, int ND, int NCU>
__global__ void __launch_bounds__(kFBlock)
complete_kernel(const __grid_constant__ TensorParams P, const double* __restrict__ X,
                double* __restrict__ R) {
  using S = P2Smem<N1, ND, NCU>;
  constexpr int NB = S::NB, NF = S::NF, TPE = S::TPE, EPB = S::EPB, NFACE = S::NFACE;
  __shared__ double sv[EPB][NF][NCU];
  __shared__ double sacc[EPB][NCU][NB];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;
  const int a = lt % N1, b = ND == 3 ? lt / N1 : 0;
  // this thread's rows of M1 for the (M1 (x) M1) face lift
  double Ma[N1], Mb[N1];
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    Ma[m] = P.m1[a * N1 + m];
    Mb[m] = ND == 3 ? P.m1[b * N1 + m] : 0.0;
  }
  bool any = false;
  if (active) {
#pragma unroll
    for (int c = 0; c < NCU; ++c)
#pragma unroll
      for (int k = 0; k < N1; ++k)
        sacc[slot][c][ND == 3 ? a + N1 * b + N1 * N1 * k : a + N1 * k] = 0.0;
  }
  for (int lf = 0; lf < NFACE; ++lf) {
    int info = 0;
    bool act = false;
    double w = 0.0;
    if (active) {
      info = __ldg(P.finfo + e * NFACE + lf);
      if ((info & LDG_FACE_KIND_MASK) == LDG_FACE_INTERIOR) {
        const bool right = info & LDG_FACE_SIDE_RIGHT;
        const bool sw = info & LDG_FACE_SWITCH;
        act = P.grad_centered || (sw != right);
        w = P.grad_centered ? 0.5 : 1.0;
      }
      if (act) {
        const int nbr = __ldg(P.fnbr + e * NFACE + lf);
        const int nlf = (info >> 4) & 7;
        const int nv = __ldg(P.nmap + (info >> LDG_FACE_MAP_SHIFT) * NF + lt);
        const int tn = vol_to_face<N1, ND>(face_axis(ND, nlf), nv);
#pragma unroll
        for (int c = 0; c < NCU; ++c)
          sv[slot][lt][c] = -w * __ldg(X + (((size_t)nbr * NFACE + nlf) * NF + tn) * NCU + c);
      }
    }
    any = any || act;
    __syncthreads();
    if (act) {
      const int vn = fvol<N1, ND>(lf, lt);
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double acc = 0.0;
        if (ND == 3) {
#pragma unroll
          for (int bb = 0; bb < N1; ++bb) {
            double s_ = 0.0;
#pragma unroll
            for (int aa = 0; aa < N1; ++aa) s_ = fma(Ma[aa], sv[slot][aa + N1 * bb][c], s_);
            acc = fma(Mb[bb], s_, acc);
          }
        } else {
#pragma unroll
          for (int aa = 0; aa < N1; ++aa) acc = fma(Ma[aa], sv[slot][aa][c], acc);
        }
        sacc[slot][c][vn] += acc;
      }
    }
    __syncthreads();
  }
  if (!active || !any) return;
  double* Re = R + (size_t)e * NB * NCU;
#pragma unroll
  for (int k = 0; k < N1; ++k) {
    const int node = ND == 3 ? a + N1 * b + N1 * N1 * k : a + N1 * k;
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      const double out = Re[node * NCU + c] + sacc[slot][c][node];
      bad_if(P, e, out);
      Re[node * NCU + c] = out;
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
  using S1 = P1Smem<N1, ND, NCU>;
  using S2 = P2Smem<N1, ND, NCU>;
  const int grid = (P.ne + S1::EPB - 1) / S1::EPB;
  const int grid2 = (P.ne + S2::EPB - 1) / S2::EPB;
  if (grid <= 0) return 0;
  if (pass & 1) {
    if (tangent) fused_kernel<N1, ND, NCU, true><<<grid, kFBlock, 0, s>>>(P, u, gproj, bsrc, R, X);
    else fused_kernel<N1, ND, NCU, false><<<grid, kFBlock, 0, s>>>(P, u, gproj, bsrc, R, X);
    if (cudaGetLastError() != cudaSuccess) return 3;
  }
  if (pass & 2) complete_kernel<N1, ND, NCU><<<grid2, kFBlock, 0, s>>>(P, X, R);
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
