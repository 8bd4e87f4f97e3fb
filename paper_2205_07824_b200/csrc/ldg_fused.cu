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

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
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
//   column owner   (hex (i,j) / quad i)  owns the node column along k (quad j)
//   y-pencil owner (hex (i,k))           owns nodes (i, 0..N1-1, k)
//   row owner      (hex (j,k) / quad j)  owns nodes (0..N1-1, j, k)
//   face-node      (t = lt on every face)
// Every 1D contraction is done by the owner of the pencil along its axis, so
// operator indices are compile-time (constant-bank DFMA operands) and each
// value loaded from shared memory feeds N1 FMAs.  Hex volume planes use a
// rotation swizzle, sw(i,j,k) = (i+k)%N1 + N1 (j+k)%N1 + N1^2 k, which makes
// column, row, y-pencil and face-node accesses bank-conflict free at N1 = 4.
//
// q is never formed: with h_s = -d_s u + sum_{faces f with axis s} lift_f,
// q = invjt h and the flux density in reference directions is
//   F_{c,r} = Cu[c][r][k] u_k + C[c][r][k][s] h_{k,s},
//   C = detJ invjt^T Aq invjt,  Cu = detJ invjt^T Au     (per element),
// and the face export sJ n.(Aq q) is sgn * F^q_{c,axis} at the face node.
// The lifts are added by the pencil owner along the face normal, so each
// jump is read once per pencil instead of once per node.

struct __align__(16) FaceRec {
  double tau;
  int32_t nbr;
  int32_t info;
};

template <int N1>
__device__ __forceinline__ int swz(int i, int j, int k) {
  if ((N1 & (N1 - 1)) == 0) return (i ^ k) + N1 * (j ^ k) + N1 * N1 * k;   // XOR swizzle
  int a = i + k, b = j + k;                                                  // rotation
  a -= a >= N1 ? N1 : 0;
  b -= b >= N1 ? N1 : 0;
  return a + N1 * b + N1 * N1 * k;
}

template <int N1, int ND, int NCU>
struct P1Smem {
  static constexpr int NF = ND == 3 ? N1 * N1 : N1;
  static constexpr int NB = ND == 3 ? N1 * N1 * N1 : N1 * N1;
  static constexpr int NBP = ND == 3 ? NB : NB + 4;          // quad: slot padding
  static constexpr int NFACE = 2 * ND;
  static constexpr int NC = NCU * ND * NCU * ND + NCU * ND * NCU;   // C then Cu
  static constexpr int FACEV = NFACE * NF * NCU;
  // region R1: h planes (ND-1 per component), later 3 stage planes
  static constexpr int R1 = (ND - 1) * NCU * NBP > 3 * NBP ? (ND - 1) * NCU * NBP : 3 * NBP;
  static constexpr int EXT = ND == 3 ? 6 * N1 * N1 : 2 * N1;  // face-slab pencils
  static constexpr int SJ = FACEV > EXT ? FACEV : EXT;       // jumps, later pencils
  static constexpr int SF = FACEV > NBP ? FACEV : NBP;       // face F^q, later B23
  static constexpr int SU = NCU * NBP > NBP ? NCU * NBP : NBP;
  static constexpr int PER = SU + R1 + SJ + FACEV + SF + NC + ND;
  static constexpr int MAXMAPS = NF <= 16 ? 16 : 8;          // node maps cached per block
  static constexpr int TPE = NF;
  static constexpr int EPB_T = (kFBlock / TPE) > 0 ? (kFBlock / TPE) : 1;
  static constexpr int EPB_S = (kFSmemDoubles - (NF <= 16 ? 16 : 8) * NF / 2) / PER > 0
                                  ? (kFSmemDoubles - (NF <= 16 ? 16 : 8) * NF / 2) / PER : 1;
  static constexpr int EPB = EPB_T < EPB_S ? EPB_T : EPB_S;
  // blocks per SM the shared memory allows; registers are capped to match
  static constexpr int SMEM_BLOCKS = (227 * 1024) / (EPB * PER * 8 + MAXMAPS * NF * 4 + 1024);
  static constexpr int EPB_S2 = (kFSmemDoubles - MAXMAPS * NF / 2) / PER;
  // (only where the register budget fits without spills: hex, ncu = 1, p <= 3)
  static constexpr int MINB = (ND == 3 && NCU == 1 && N1 <= 4)
                                  ? (SMEM_BLOCKS < 1 ? 1 : (SMEM_BLOCKS > 8 ? 8 : SMEM_BLOCKS))
                                  : 1;
};

template <int N1, int ND, int NCU, bool TANGENT>
__global__ void __launch_bounds__(kFBlock, P1Smem<N1, ND, NCU>::MINB)
fused_kernel(const __grid_constant__ TensorParams P, const FaceRec* __restrict__ frec,
             const double* __restrict__ u, const double* __restrict__ gproj,
             const double* __restrict__ bsrc, double* __restrict__ R,
             double* __restrict__ X) {
  using S = P1Smem<N1, ND, NCU>;
  constexpr int NB = S::NB, NBP = S::NBP, NF = S::NF, TPE = S::TPE, EPB = S::EPB;
  constexpr int NFACE = S::NFACE, NC = S::NC, CQ = NCU * ND * NCU * ND;
  __shared__ __align__(16) double s_u[EPB][S::SU];      // u planes; later B1 plane
  __shared__ __align__(16) double s_r1[EPB][S::R1];     // h planes; later stage planes
  __shared__ __align__(16) double s_j[EPB][S::SJ];      // jumps; later face-slab pencils
  __shared__ __align__(16) double s_fh[EPB][S::FACEV];  // sJ f^ (own share)
  __shared__ __align__(16) double s_f[EPB][S::SF];      // face F^q; later B23 plane
  constexpr int KSZ = NC + ND;             // C, Cu, sJ per face axis
  __shared__ __align__(16) double s_k[EPB][KSZ];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;
  const int ta = lt % N1, tb = ND == 3 ? lt / N1 : 0;
  const int i = ta, j = tb;
  double* su = s_u[slot];
  double* sj = s_j[slot];
  double* sfh = s_fh[slot];
  double* sff = s_f[slot];
  double* sr = s_r1[slot];
  // volume-plane index (hex: swizzled)
  auto vix = [](int a, int b, int k) {
    return ND == 3 ? swz<N1>(a, b, k) : a + N1 * k;
  };
  auto fix = [](int lf, int t, int c) { return (lf * NF + t) * NCU + c; };
  auto cidx = [&](int k) { return vix(i, j, k); };
  auto ridx = [&](int m) { return ND == 3 ? vix(m, ta, tb) : m + N1 * ta; };
  auto yidx = [&](int m) { return ND == 3 ? vix(ta, m, tb) : 0; };

  // ---- A: u column and the element coefficient block stream into shared
  // memory with cp.async (no register staging); the face records come into
  // registers and the neighbour / boundary-data gathers they address are
  // issued right away, so all of the element's global latency overlaps.
  double uc[NCU][N1];
  const double* kc = s_k[slot];            // element coefficient block (shared)
  FaceRec fr[NFACE];
  double ext[NFACE][NCU];
  if (active) {
    const double* ue = u + (size_t)e * NB * NCU;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
#pragma unroll
      for (int c = 0; c < NCU; ++c) cp_async8(su + c * NBP + cidx(k), ue + node * NCU + c);
    }
    const double* kb = P.kco + (size_t)e * P.kstride;
    for (int x = lt; x < KSZ; x += TPE) cp_async8(s_k[slot] + x, kb + x);
    cp_async_commit();
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(frec + (size_t)e * NFACE + lf));
      fr[lf].tau = v.x;                    // sJ * tau on this face
      const int2 w = *reinterpret_cast<const int2*>(&v.y);
      fr[lf].nbr = w.x;
      fr[lf].info = w.y;
    }
    const double* src[NFACE];
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const int info = fr[lf].info, nbr = fr[lf].nbr;
      const int kind = info & LDG_FACE_KIND_MASK;
      src[lf] = nullptr;
      if (kind == LDG_FACE_INTERIOR) {
        if (info & LDG_FL_UNBR) {
          const int mid = (info >> LDG_FACE_MAP_SHIFT) & 0xffff;
          src[lf] = u + ((size_t)nbr * NB + __ldg(P.nmap + mid * NF + lt)) * NCU;
        }
      } else if (!TANGENT && gproj) {
        src[lf] = gproj + ((size_t)nbr * NF + lt) * NCU;
      }
    }
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf)
#pragma unroll
      for (int c = 0; c < NCU; ++c) ext[lf][c] = src[lf] ? __ldg(src[lf] + c) : 0.0;
  }
  cp_async_wait_all();
  __syncthreads();
  if (active) {
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int c = 0; c < NCU; ++c) uc[c][k] = su[c * NBP + cidx(k)];
  }

  // ---- B: face node lt of every face: jumps and the u part of sJ f^
  double gl[NCU][N1];       // d/dk of the column (registers)
  if (active) {
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const int info = fr[lf].info;
      const int kind = info & LDG_FACE_KIND_MASK;
      const int ax = face_axis(ND, lf);
      const double sgn = face_side(ND, lf) ? 1.0 : -1.0;
      (void)ax;
      const int vn_ = fvol<N1, ND>(lf, lt);
      const int vs = ND == 3 ? swz<N1>(vn_ % N1, (vn_ / N1) % N1, vn_ / (N1 * N1)) : vn_;
      // coefficient form (ldg_create): with d = u_own - u_other (u_other =
      // neighbour trace, Dirichlet g, or 0), every rule of disc.py:492-574 and
      // :657-821 is jump = alpha d, sJ * sigma * tau (u_L - u^) = rec.tau * d;
      // Neumann faces carry rec.tau = sJ and add sJ g.
      const double rt = fr[lf].tau;
      const int acode = (info >> LDG_FL_ALPHA_SHIFT) & 3;
      const double alpha = acode == 1 ? 1.0 : (acode == 2 ? 0.5 : 0.0);
      const bool neu = kind == LDG_FACE_NEUMANN;
      double uh[NCU], fh[NCU], jmp[NCU];
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        const double uo = su[c * NBP + vs];
        const double d = uo - ext[lf][c];
        jmp[c] = alpha * d;
        uh[c] = uo - jmp[c];
        fh[c] = rt * (neu ? ext[lf][c] : d);
      }
      if (P.flux_uses_u && kind != LDG_FACE_NEUMANN) {
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          double a = 0.0;
#pragma unroll
          for (int kk = 0; kk < NCU; ++kk) a = fma(kc[CQ + (c * ND + ax) * NCU + kk], uh[kk], a);
          fh[c] = fma(sgn, a, fh[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        sj[fix(lf, lt, c)] = jmp[c];
        sfh[fix(lf, lt, c)] = fh[c];
      }
    }
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
  __syncthreads();

  // ---- C: h pencils along x (row owner) and y (y-pencil owner), lifts folded in
  if (active) {
    // quad faces: 0 y-, 1 x+, 2 y+, 3 x-; hex: 0 z-, 1 z+, 2 y-, 3 y+, 4 x-, 5 x+
    constexpr int XLO = ND == 3 ? 4 : 3, XHI = ND == 3 ? 5 : 1;
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      double row[N1];
#pragma unroll
      for (int m = 0; m < N1; ++m) row[m] = su[c * NBP + ridx(m)];
      const int t = ND == 3 ? ta + N1 * tb : ta;
      const double jl = sj[fix(XLO, t, c)], jh = sj[fix(XHI, t, c)];
#pragma unroll
      for (int a = 0; a < N1; ++a) {
        double v = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) v = fma(P.d1[a * N1 + m], row[m], v);
        sr[c * NBP + ridx(a)] = -v - P.clo[a] * jl + P.chi[a] * jh;
      }
      if (ND == 3) {
        double col[N1];
#pragma unroll
        for (int m = 0; m < N1; ++m) col[m] = su[c * NBP + yidx(m)];
        const double yl = sj[fix(2, ta + N1 * tb, c)], yh = sj[fix(3, ta + N1 * tb, c)];
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          double v = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) v = fma(P.d1[a * N1 + m], col[m], v);
          sr[(NCU + c) * NBP + yidx(a)] = -v - P.clo[a] * yl + P.chi[a] * yh;
        }
      }
    }
  }
  __syncthreads();

  // ---- D: F = Cu u + C h at the column's nodes; F^q at face nodes
  double F[NCU][ND][N1];
  if (active) {
    double cr[NC];
#pragma unroll
    for (int x = 0; x < NC; ++x) cr[x] = kc[x];
    constexpr int ZLO = ND == 3 ? 0 : 0, ZHI = ND == 3 ? 1 : 2;   // column-axis faces
    double zl[NCU], zh[NCU];
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      zl[c] = sj[fix(ZLO, ND == 3 ? i + N1 * j : i, c)];
      zh[c] = sj[fix(ZHI, ND == 3 ? i + N1 * j : i, c)];
    }
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      double h[NCU][ND];
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        h[c][0] = sr[c * NBP + cidx(k)];
        if (ND == 3) h[c][1] = sr[(NCU + c) * NBP + cidx(k)];
        h[c][ND - 1] = -gl[c][k] - P.clo[k] * zl[c] + P.chi[k] * zh[c];
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
              fq = fma(cr[((c * ND + r) * NCU + kk) * ND + s_], h[kk][s_], fq);
          double fu = 0.0;
          if (P.flux_uses_u) {
#pragma unroll
            for (int kk = 0; kk < NCU; ++kk)
              fu = fma(cr[CQ + (c * ND + r) * NCU + kk], uc[kk][k], fu);
          }
          F[c][r][k] = fq + fu;
          // F^q of the face-normal component at this column's face nodes
          if (ND == 3) {
            if (r == 2 && k == 0) sff[fix(0, i + N1 * j, c)] = fq;
            if (r == 2 && k == N1 - 1) sff[fix(1, i + N1 * j, c)] = fq;
            if (r == 1 && j == 0) sff[fix(2, i + N1 * k, c)] = fq;
            if (r == 1 && j == N1 - 1) sff[fix(3, i + N1 * k, c)] = fq;
            if (r == 0 && i == 0) sff[fix(4, j + N1 * k, c)] = fq;
            if (r == 0 && i == N1 - 1) sff[fix(5, j + N1 * k, c)] = fq;
          } else {
            if (r == 1 && k == 0) sff[fix(0, i, c)] = fq;
            if (r == 1 && k == N1 - 1) sff[fix(2, i, c)] = fq;
            if (r == 0 && i == 0) sff[fix(3, k, c)] = fq;
            if (r == 0 && i == N1 - 1) sff[fix(1, k, c)] = fq;
          }
        }
    }
  }
  __syncthreads();

  // ---- E: own share of sJ n.(Aq q^) and exports at face node lt
  if (active) {
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const int info = fr[lf].info;
      const int kind = info & LDG_FACE_KIND_MASK;
      if (kind == LDG_FACE_NEUMANN) continue;
      // flags precomputed at ldg_create (q^ = own / half / neighbour, export)
      const bool exp_ = info & LDG_FL_EXPORT;
      const double w_own = kind != LDG_FACE_INTERIOR ? 1.0
                           : ((info & LDG_FL_QOWN) ? 1.0 : ((info & LDG_FL_QHALF) ? 0.5 : 0.0));
      if (w_own == 0.0 && !exp_) continue;
      const double sgn = face_side(ND, lf) ? 1.0 : -1.0;
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        const double xf = sgn * sff[fix(lf, lt, c)];
        sfh[fix(lf, lt, c)] = fma(w_own, xf, sfh[fix(lf, lt, c)]);
        if (exp_) X[(((size_t)e * NFACE + lf) * NF + lt) * NCU + c] = xf;
      }
    }
  }
  __syncthreads();

  // ---- F..H: R = -sum_r K_r F_r + face terms, sum factorised by pencils
  double* Re = R + (size_t)(active ? e : 0) * NB * NCU;
  double* sX = sj;             // face-slab pencils (jumps are dead)
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
          if (k == 0) a3 -= sfh[fix(0, i + N1 * j, c)];
          if (k == N1 - 1) a3 -= sfh[fix(1, i + N1 * j, c)];
          const int v = cidx(k);
          sr[v] = a1;
          sr[NBP + v] = a2;
          sr[2 * NBP + v] = a3;
        }
        // face-slab pencils along z: p = (type x|y, side, idx): out[k] = M fh
        for (int p = lt; p < 4 * N1; p += TPE) {
          const int type = p / (2 * N1), side = (p / N1) & 1, idx = p % N1;
          const int lf = type == 0 ? 4 + side : 2 + side;
          double v[N1];
#pragma unroll
          for (int n = 0; n < N1; ++n) v[n] = sfh[fix(lf, idx + N1 * n, c)];
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
      if (active) {
        // y stage (pencil owner (i,k) = (ta,tb)); B1 -> su plane, B23 -> sff plane
        double a1[N1], a2[N1], a3[N1];
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          const int v = yidx(m);
          a1[m] = sr[v];
          a2[m] = sr[NBP + v];
          a3[m] = sr[2 * NBP + v];
        }
        const double yl = sX[((1 * 2 + 0) * N1 + ta) * N1 + tb];
        const double yh = sX[((1 * 2 + 1) * N1 + ta) * N1 + tb];
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          double b1 = 0.0, b2 = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            b1 = fma(P.m1[a * N1 + m], a1[m], b1);
            b2 = fma(P.s1[a * N1 + m], a2[m], b2);
            b2 = fma(P.m1[a * N1 + m], a3[m], b2);
          }
          if (a == 0) b2 -= yl;
          if (a == N1 - 1) b2 -= yh;
          const int v = yidx(a);
          su[v] = b1;
          sff[v] = b2;
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
        // x stage (row owner (j,k) = (ta,tb))
        double b1[N1], b23[N1];
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          const int v = ridx(m);
          b1[m] = su[v];
          b23[m] = sff[v];
        }
        const double xl = sX[4 * N1 * N1 + (0 * N1 + ta) * N1 + tb];
        const double xh = sX[4 * N1 * N1 + (1 * N1 + ta) * N1 + tb];
        double out[N1];
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          double r = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            r = fma(P.s1[a * N1 + m], b1[m], r);
            r = fma(P.m1[a * N1 + m], b23[m], r);
          }
          out[a] = -r;
        }
        out[0] += xl;
        out[N1 - 1] += xh;
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          const int node = a + N1 * ta + N1 * N1 * tb;
          double o = out[a];
          if (!TANGENT && bsrc) o += __ldg(bsrc + ((size_t)e * NB + node) * NCU + c);
          bad_if(P, e, o);
          Re[node * NCU + c] = o;
        }
      }
      if (NCU > 1) __syncthreads();
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
          if (k == 0) a2 -= sfh[fix(0, i, c)];
          if (k == N1 - 1) a2 -= sfh[fix(2, i, c)];
          sr[i + N1 * k] = a1;
          sr[NBP + i + N1 * k] = a2;
        }
        for (int p = lt; p < 2; p += TPE) {
          const int lf = p == 0 ? 3 : 1;
          double v[N1];
#pragma unroll
          for (int n = 0; n < N1; ++n) v[n] = sfh[fix(lf, n, c)];
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
        double a1[N1], a2[N1];
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          a1[m] = sr[m + N1 * ta];
          a2[m] = sr[NBP + m + N1 * ta];
        }
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          double r = 0.0;
#pragma unroll
          for (int m = 0; m < N1; ++m) {
            r = fma(P.s1[a * N1 + m], a1[m], r);
            r = fma(P.m1[a * N1 + m], a2[m], r);
          }
          double o = -r;
          if (a == 0) o += sX[0 * N1 + ta];
          if (a == N1 - 1) o += sX[1 * N1 + ta];
          const int node = a + N1 * ta;
          if (!TANGENT && bsrc) o += __ldg(bsrc + ((size_t)e * NB + node) * NCU + c);
          bad_if(P, e, o);
          Re[node * NCU + c] = o;
        }
      }
      __syncthreads();
    }
  }
}

// --------------------------------------------------------------------------
// pass 2: neighbour share of f(., q^) on faces whose q^ comes from across
// --------------------------------------------------------------------------
//
// Each column owner adds, for its nodes, the (M1 (x) M1)-lifted neighbour
// exports of every completion face containing them (sum factorised: the
// in-face row is contracted with the thread's M1 row, the column direction
// with compile-time M1 entries), then read-modify-writes its R column.

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
complete_kernel(const __grid_constant__ TensorParams P, const FaceRec* __restrict__ frec,
                const double* __restrict__ X, double* __restrict__ R) {
  using S = P2Smem<N1, ND, NCU>;
  constexpr int NB = S::NB, NF = S::NF, TPE = S::TPE, EPB = S::EPB, NFACE = S::NFACE;
  __shared__ double sv[EPB][NFACE][NF][NCU];    // neighbour exports, then lifted values
  __shared__ double sw2[EPB][NFACE][NF][NCU];   // first-direction partial lift
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int e = blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.ne;
  const int i = lt % N1, j = ND == 3 ? lt / N1 : 0;
  // this thread's M1 rows (i for the first in-face index, j for the second)
  double Mi[N1], Mj[N1];
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    Mi[m] = P.m1[i * N1 + m];
    Mj[m] = P.m1[j * N1 + m];
  }
  constexpr int kMaxMaps = 16;
  __shared__ int s_map[kMaxMaps * NF];
  const bool map_in_smem = P.n_maps <= kMaxMaps;
  if (map_in_smem)
    for (int x = threadIdx.x; x < P.n_maps * NF; x += blockDim.x) s_map[x] = __ldg(P.nmap + x);
  // R column loads are independent of the exports: issue them first
  double rcol[NCU][N1];
  if (active) {
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int c = 0; c < NCU; ++c)
        rcol[c][k] = R[((size_t)e * NB + (ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k)) * NCU + c];
  }
  int info_[NFACE], nbr_[NFACE];
  if (active) {
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(frec + (size_t)e * NFACE + lf));
      const int2 w = *reinterpret_cast<const int2*>(&v.y);
      nbr_[lf] = w.x;
      info_[lf] = w.y;
    }
  }
  __syncthreads();
  int mask = 0;
  if (active) {
    // addresses first, then every gather issued back to back (one latency)
    const double* src[NFACE];
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const int info = info_[lf];
      const bool act = info & LDG_FL_COMPLETE;
      mask |= act ? (1 << lf) : 0;
      const int nlf = (info >> 4) & 7;
      const int mid = act ? (info >> LDG_FACE_MAP_SHIFT) & 0xffff : 0;
      const int nv = map_in_smem ? s_map[mid * NF + lt] : __ldg(P.nmap + mid * NF + lt);
      const int tn = vol_to_face<N1, ND>(face_axis(ND, nlf), nv);
      src[lf] = act ? X + (((size_t)nbr_[lf] * NFACE + nlf) * NF + tn) * NCU : nullptr;
    }
    double xv[NFACE][NCU];
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf)
#pragma unroll
      for (int c = 0; c < NCU; ++c) xv[lf][c] = src[lf] ? __ldg(src[lf] + c) : 0.0;
    const double wgt = P.grad_centered ? -0.5 : -1.0;
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf)
#pragma unroll
      for (int c = 0; c < NCU; ++c) sv[slot][lf][lt][c] = wgt * xv[lf][c];
  }
  __syncthreads();
  // lift every completion face by (M1 (x) M1), sum factorised with all of the
  // element's threads busy: w[a][b] = sum_a' M[a][a'] v[a'][b], then
  // out[a][b] = sum_b' M[b][b'] w[a][b'] (thread = face node (a, b))
  if (active) {
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      if (!(mask & (1 << lf))) continue;
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double w = 0.0;
        if (ND == 3) {
#pragma unroll
          for (int aa = 0; aa < N1; ++aa) w = fma(Mi[aa], sv[slot][lf][aa + N1 * j][c], w);
        } else {
#pragma unroll
          for (int aa = 0; aa < N1; ++aa) w = fma(Mi[aa], sv[slot][lf][aa][c], w);
        }
        sw2[slot][lf][lt][c] = w;
      }
    }
  }
  __syncthreads();
  if (active && ND == 3) {
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      if (!(mask & (1 << lf))) continue;
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double o = 0.0;
#pragma unroll
        for (int bb = 0; bb < N1; ++bb) o = fma(Mj[bb], sw2[slot][lf][i + N1 * bb][c], o);
        sv[slot][lf][lt][c] = o;          // lifted value at face node (i, j)
      }
    }
  }
  __syncthreads();
  if (!active || mask == 0) return;
  // gather the lifted face values onto this thread's column and RMW R
  auto fval = [&](int lf, int t, int c) {
    return ND == 3 ? sv[slot][lf][t][c] : sw2[slot][lf][t][c];
  };
  double* Re = R + (size_t)e * NB * NCU;
#pragma unroll
  for (int c = 0; c < NCU; ++c) {
    double acc[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) acc[k] = 0.0;
    if (ND == 3) {
      // faces 0 z-, 1 z+ (node (i,j,0|N1-1)), 2 y-, 3 y+ (j = 0|N1-1, coords (i,k)),
      // 4 x-, 5 x+ (i = 0|N1-1, coords (j,k))
      if (mask & 1) acc[0] += fval(0, i + N1 * j, c);
      if (mask & 2) acc[N1 - 1] += fval(1, i + N1 * j, c);
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        if ((mask & 4) && j == 0) acc[k] += fval(2, i + N1 * k, c);
        if ((mask & 8) && j == N1 - 1) acc[k] += fval(3, i + N1 * k, c);
        if ((mask & 16) && i == 0) acc[k] += fval(4, j + N1 * k, c);
        if ((mask & 32) && i == N1 - 1) acc[k] += fval(5, j + N1 * k, c);
      }
    } else {
      // quad faces 0 y-, 2 y+ (node (i, 0|N1-1)), 3 x-, 1 x+ (i = 0|N1-1, coord k)
      if (mask & 1) acc[0] += fval(0, i, c);
      if (mask & 4) acc[N1 - 1] += fval(2, i, c);
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        if ((mask & 8) && i == 0) acc[k] += fval(3, k, c);
        if ((mask & 2) && i == N1 - 1) acc[k] += fval(1, k, c);
      }
    }
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
      const double out = rcol[c][k] + acc[k];
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
    const FaceRec* fr = reinterpret_cast<const FaceRec*>(P.frec);
    if (tangent) fused_kernel<N1, ND, NCU, true><<<grid, kFBlock, 0, s>>>(P, fr, u, gproj, bsrc, R, X);
    else fused_kernel<N1, ND, NCU, false><<<grid, kFBlock, 0, s>>>(P, fr, u, gproj, bsrc, R, X);
    if (cudaGetLastError() != cudaSuccess) return 3;
  }
  if (pass & 2)
    complete_kernel<N1, ND, NCU><<<grid2, kFBlock, 0, s>>>(
        P, reinterpret_cast<const FaceRec*>(P.frec), X, R);
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
