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

#include <algorithm>
#include <climits>
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
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_group1() {
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// non-finite test of many values with integer ops only: the largest
// |exponent field| over the high words (inf / NaN have it all ones), one
// branch and at most one atomic per thread
__device__ __forceinline__ int hi_abs(double v) { return __double2hiint(v) & 0x7fffffff; }
__device__ __forceinline__ void bad_if_any(const TensorParams& P, int e, int hmax) {
  if (hmax >= 0x7ff00000) atomicMin(P.bad, (unsigned long long)e);
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

// N1 values whose planes are NOT rotated (every N1 that is not a power of
// two): the rotation's index arithmetic and the conflicts it leaves cost more
// than it saves (ncu, config-5 pencil pass 1, scripts/ncu_ab.sh: p = 4
// 216.7 -> 186.2 us, bank-conflict excess 20.7M -> 11.4M wavefronts,
// instructions 112.8M -> 87.7M; p = 5 208.6 -> 187.1 us, 13.0M -> 9.2M; a
// padded k-stride at p = 5 measured no better: 187.7 us)
#ifndef LDG_SWZ_ID_MASK
#define LDG_SWZ_ID_MASK ((1 << 3) | (1 << 5) | (1 << 6) | (1 << 7))
#endif
template <int N1>
__device__ __forceinline__ int swz(int i, int j, int k) {
  if ((LDG_SWZ_ID_MASK >> N1) & 1) return i + N1 * j + N1 * N1 * k;
  if ((N1 & (N1 - 1)) == 0) return (i ^ k) + N1 * (j ^ k) + N1 * N1 * k;   // XOR swizzle
  int a = i + k, b = j + k;                                                  // rotation
  a -= a >= N1 ? N1 : 0;
  b -= b >= N1 ? N1 : 0;
  return a + N1 * b + N1 * N1 * k;
}

#ifndef LDG_P1_MINB_MAXN1
#define LDG_P1_MINB_MAXN1 6       // pencil pass 1: register cap to the shared-memory block count up to this N1
                                  // (N1 = 5, 6: ncu 186.3 -> 175.5 us, 186.6 -> 179.7 us)
#endif
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
  static constexpr int MINB = (ND == 3 && NCU == 1 && N1 <= LDG_P1_MINB_MAXN1)
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
  const int e = P.e0 + blockIdx.x * EPB + slot;
  const bool active = slot < EPB && e < P.e1;
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
          src[lf] = nbr_row(P, u, nbr, NB * NCU) + (size_t)__ldg(P.nmap + mid * NF + lt) * NCU;
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
      const int vs = (ND == 3 && !((LDG_SWZ_ID_MASK >> N1) & 1))
                         ? swz<N1>(vn_ % N1, (vn_ / N1) % N1, vn_ / (N1 * N1)) : vn_;
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
        if (exp_) {
          size_t xo;
          if (P.x_consumer) {      // the neighbour's slot, in its face-node order
            const int nlf = (info >> 4) & 7;
            const int mid = (info >> LDG_FACE_MAP_SHIFT) & 0xffff;
            const int tn = ((unsigned)info & LDG_FL_XIDENT) ? lt
                : vol_to_face<N1, ND>(face_axis(ND, nlf), __ldg(P.nmap + mid * NF + lt));
            const int nbr = __ldg(&frec[(size_t)e * NFACE + lf].nbr);   // (re-read: keeps it out of registers)
            xo = (((size_t)nbr * NFACE + nlf) * NF + tn) * NCU + c;
          } else {
            xo = (((size_t)e * NFACE + lf) * NF + lt) * NCU + c;
          }
          X[xo] = xf;
        }
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
        int hm = 0;
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          const int node = a + N1 * ta + N1 * N1 * tb;
          double o = out[a];
          if (!TANGENT && bsrc) o += __ldg(bsrc + ((size_t)e * NB + node) * NCU + c);
          hm = max(hm, hi_abs(o));
          Re[node * NCU + c] = o;
        }
        bad_if_any(P, e, hm);
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
        int hm = 0;
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
          hm = max(hm, hi_abs(o));
          Re[node * NCU + c] = o;
        }
        bad_if_any(P, e, hm);
      }
      __syncthreads();
    }
  }
}

// --------------------------------------------------------------------------
// pass 1, plane mapping (hex, ncu = 1, p = 3): the shared-memory-lean variant
// --------------------------------------------------------------------------
//
// The pencil kernel above moves every 1D contraction to the owner of the
// pencil along its axis, which costs a shared-memory transpose per stage
// (~25 KB of shared traffic per element; ncu: L1 92% busy, HBM 22%).  Here
// thread k of an element (4 consecutive lanes) owns the z-plane k (16 nodes,
// registers): x and y contractions, the x/y face work and the flux
// combination are all in registers, and only two exchanges cross planes:
//   1. u planes (+ the z-face jumps) for d/dz and the z lifts,
//   2. the in-plane partial volume terms T1 = -(S_x M_y F_x + M_x S_y F_y)
//      + x/y face lifts, T2 = -M_x M_y F_z, contracted along z:
//      R_k = sum_m M[k][m] T1_m + S[k][m] T2_m  (+ z-face lifts on k = 0, 3).
// A warp owns 8 consecutive elements (4 KB of u, 4 KB of R): u and the
// neighbour face values arrive by cp.async straight into shared memory
// (coalesced 256 B rows; no register staging, no dependence stalls until
// first use) and R leaves through shared memory as coalesced rows.  The four
// threads of an element sit in one warp, so exchanges use __syncwarp only.
// Outputs and arithmetic identities are those of fused_kernel.

namespace {
constexpr int kPlaneBlock = 128;
constexpr int kPlaneEpb = kPlaneBlock / 4;
constexpr int kPS = 17;                      // padded plane stride (doubles)
constexpr int kES = 5;                       // padded stride of a thread's 4 face values
// per-element shared region (doubles), two input buffers + work space:
//   in buffer b at b * 96:  [0, 68) u planes (stride 17), later T1 and the R
//                           staging; [68, 84) coefficient block C | Cu;
//                           [84, 96) the six face records (16 B each)
//   [192, 232) z-face jumps  [face][row j][i] (row stride 5)
//   [232, 272) z-face fluxes [face][row j][i]
//   [272, 340) T2 planes (stride 17)
// element stride = 4 (mod 16) doubles so the 8 elements of a warp spread
// over the banks.  The thread-private x/y face fluxes live in the thread's
// own u-plane slot between the u exchange and the T1 store.
constexpr int kInSz = 96, kInC = 4 * kPS, kInF = kInC + 16;
constexpr int kOffJ = 2 * kInSz, kOffF = kOffJ + 40, kOffE = kOffF + 40;
#ifndef LDG_PLANE_DMMA
#define LDG_PLANE_DMMA 0          // A/B: z contractions on the FP64 tensor core (mma.sync m8n8k4):
#endif                            // bit 0: R = M_z W, bit 1: D_z u and (G D)_z u
// [340, 408): per-thread z volume term (DMMA variant, plane stride 17 like
// the other planes: conflict-free), padded to 4 mod 16
constexpr int kOffVZ = kOffE + 4 * kPS;
constexpr int kPlanePer = (LDG_PLANE_DMMA & 2) ? kOffVZ + 4 * kPS + 12 : kOffE + 4 * kPS;   // 420 | 340
static_assert(kInF + 12 <= kInSz, "layout");
static_assert(kPlanePer % 16 == 4, "element stride must be 4 mod 16 doubles");
// element regions of a warp: stride kPlanePer, elements 4..7 skewed by 2
// doubles, so the 8 elements' 16-B broadcast reads hit 8 distinct bank
// quads (4e + 2(e >> 2) mod 16 = 0, 4, 8, 12, 2, 6, 10, 14) while 8-B
// per-thread accesses (4e + k) stay conflict-free
__host__ __device__ constexpr int plane_el(int e) { return e * kPlanePer + (e >> 2) * 2; }
constexpr int kPlaneWarp = plane_el(8);      // doubles per warp region
constexpr int kPlaneMaps = 16;               // node maps cached in shared memory
}  // namespace

// acc[n] += c * plane[n], n < 16, for a padded plane at offset m * kPS of a
// 16-B aligned element region: 16-B loads wherever the pair is aligned (the
// four threads of an element read the same plane, so a 16-B broadcast moves
// twice the data per shared wavefront)
template <int M>
__device__ __forceinline__ void axpy_plane(double (&acc)[16], double c, const double* plane) {
  if ((M * 17) % 2 == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double2 v = reinterpret_cast<const double2*>(plane)[j];
      acc[2 * j] = fma(c, v.x, acc[2 * j]);
      acc[2 * j + 1] = fma(c, v.y, acc[2 * j + 1]);
    }
  } else {
    acc[0] = fma(c, plane[0], acc[0]);
#pragma unroll
    for (int j = 0; j < 7; ++j) {
      const double2 v = reinterpret_cast<const double2*>(plane + 1)[j];
      acc[2 * j + 1] = fma(c, v.x, acc[2 * j + 1]);
      acc[2 * j + 2] = fma(c, v.y, acc[2 * j + 2]);
    }
    acc[15] = fma(c, plane[15], acc[15]);
  }
}

// D[8x8] = A[8x4] B[4x8] on the FP64 tensor core.  Plane mapping: lane
// l = 4 slot + k supplies A[slot][k] = its plane-k value of one in-plane node
// and B[k][c] (a per-lane operator constant); it receives D[slot][2k] and
// D[slot][2k+1].  With B[m][2r + e] = Op_e[r][m] that is (Op_0 z u)[k] and
// (Op_1 z u)[k] of its own plane: a z contraction of 8 elements in one
// instruction, no shared-memory exchange.
__device__ __forceinline__ void dmma_zplane(double& d0, double& d1, double a, double b) {
  double c0 = 0.0, c1 = 0.0;
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
      : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Pass 2 of one 8-element group inside the one-launch operator: the
// arithmetic of complete_warp4_kernel (half a warp per element, lane t = i + 4j
// owns R column (i, j) and face node t), four element pairs with all their
// loads issued together.  R rows and exports were written by other SMs earlier
// in the same launch: read through L2 (__ldcg), never the read-only path.
__device__ __forceinline__ void complete_group4(const TensorParams& P, const FaceRec* __restrict__ frec,
                                                const double* X, double* R, int e_w, int lane,
                                                const double* sM) {
  constexpr int NB = 64, NF = 16;
  const int half = lane >> 4, t = lane & 15, i = t & 3, j = t >> 2, hb = half * 16;
  const double wgt = P.grad_centered ? -0.5 : -1.0;
  int info[4];
  double r[4][4], x[4][6];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int e = e_w + 2 * p + half;
    info[p] = (e < P.e1 && t < 6) ? __ldg(reinterpret_cast<const int*>(frec + (size_t)e * 6 + t) + 3) : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) r[p][k] = e < P.e1 ? __ldcg(R + (size_t)e * NB + t + 16 * k) : 0.0;
  }
  unsigned any[4];
  int mask[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const unsigned bal = __ballot_sync(0xffffffffu, (info[p] & LDG_FL_COMPLETE) != 0);
    any[p] = (bal | (bal >> 16)) & 63;
    mask[p] = (bal >> hb) & 63;
    const int e = e_w + 2 * p + half;
#pragma unroll
    for (int lf = 0; lf < 6; ++lf)
      x[p][lf] = (mask[p] >> lf) & 1 ? __ldcg(X + ((size_t)e * 6 + lf) * NF + t) : 0.0;
  }
  double Mi[4], Mj[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    Mi[m] = sM[i * 4 + m];
    Mj[m] = sM[j * 4 + m];
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int e = e_w + 2 * p + half;
#pragma unroll
    for (int lf = 0; lf < 6; ++lf) {
      if (!((any[p] >> lf) & 1)) continue;                  // warp-uniform
      const double v = wgt * x[p][lf];
      double wv = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a) wv = fma(Mi[a], __shfl_sync(0xffffffffu, v, hb + a + 4 * j), wv);
      double L = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) L = fma(Mj[b], __shfl_sync(0xffffffffu, wv, hb + i + 4 * b), L);
      if (!((mask[p] >> lf) & 1)) L = 0.0;
      if (lf == 0) r[p][0] += L;
      else if (lf == 1) r[p][3] += L;
      else {
        const bool own = lf == 2 ? j == 0 : (lf == 3 ? j == 3 : (lf == 4 ? i == 0 : i == 3));
        const int a0 = lf < 4 ? i : j;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double gg = __shfl_sync(0xffffffffu, L, hb + a0 + 4 * k);
          if (own) r[p][k] += gg;
        }
      }
    }
    if (e < P.e1) {
      int hm = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        hm = max(hm, hi_abs(r[p][k]));
        R[(size_t)e * NB + t + 16 * k] = r[p][k];
      }
      bad_if_any(P, e, hm);
    }
  }
}

#ifndef LDG_PLANE_MINB
#define LDG_PLANE_MINB 2          // 2 persistent blocks per SM (shared-memory bound)
#endif

template <bool TANGENT, bool HAS_CU, bool DIAG, bool FUSED>
__global__ void __launch_bounds__(kPlaneBlock, LDG_PLANE_MINB)
plane_kernel(const __grid_constant__ TensorParams P, const FaceRec* __restrict__ frec,
             const double* __restrict__ u, const double* __restrict__ gproj,
             const double* __restrict__ bsrc, double* __restrict__ R,
             double* __restrict__ X) {
  constexpr int N1 = 4, NP = 16, NB = 64;
  extern __shared__ __align__(16) double psm[];
  __shared__ int s_map[kPlaneMaps * NP];
  __shared__ double s_tab[5 * NP + 16];          // G, M^-1, M, D, clo, chi, GD, G clo, G chi
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = threadIdx.x >> 2, k = threadIdx.x & 3;
  const int ls = lane >> 2;                                // element slot within the warp
  const bool map_smem = P.n_maps <= kPlaneMaps;
  if (map_smem)
    for (int x = threadIdx.x; x < P.n_maps * NP; x += kPlaneBlock) s_map[x] = __ldg(P.nmap + x);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int x = 0; x < NP; ++x) {
      s_tab[x] = P.g1[x];
      s_tab[NP + x] = P.m1inv[x];
      s_tab[2 * NP + x] = P.m1[x];
      s_tab[3 * NP + x] = P.d1[x];
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      s_tab[4 * NP + x] = P.clo[x];
      s_tab[4 * NP + 4 + x] = P.chi[x];
      s_tab[5 * NP + 8 + x] = P.gclo[x];
      s_tab[5 * NP + 12 + x] = P.gchi[x];
    }
#pragma unroll
    for (int x = 0; x < NP; ++x) s_tab[4 * NP + 8 + x] = P.gd1[x];
  }
  __syncthreads();
  // per-lane B fragments of the z contractions: column c = lane / 4 =
  // 2 r + e, row m = lane % 4 (see dmma_zplane); read where used
  const int bc = (threadIdx.x & 31) >> 2, bm = threadIdx.x & 3;
  const int bDG_at = ((bc & 1) ? 4 * NP + 8 : 3 * NP) + 4 * (bc >> 1) + bm;   // D | GD
  const int bM_at = (bc & 1) ? -1 : 2 * NP + 4 * (bc >> 1) + bm;             // M | 0
  (void)bDG_at; (void)bM_at;
  // let the completion kernel's blocks launch as SMs free up (they wait on
  // griddepcontrol.wait before touching R / X)
  asm volatile("griddepcontrol.launch_dependents;");
  double* sWarp = psm + warp * kPlaneWarp;                 // the warp's 8 element regions
  double* sEl = sWarp + plane_el(ls);
  double* sJZ = sEl + kOffJ;
  double* sFZ = sEl + kOffF;
  double* sT2 = sEl + kOffE;
  const int nel = P.e1 - P.e0;
  const int ngroups = (nel + 7) >> 3;
  const int stride = gridDim.x * (kPlaneBlock / 32);
  // FUSED: pass-1 groups are claimed in order from a device counter (every
  // claimed group is finished by a running warp, so a warp waiting for pass-1
  // windows never waits on a block that is not resident)
  // lane 0 issues the claim; the value is broadcast only where it is used, so
  // the atomic's latency hides behind a group's work
  auto claim_raw = [&](int which) {
    int v = 0;
    if (FUSED && lane == 0) v = atomicAdd(P.fuse + which, 1);
    return v;
  };
  auto bcast = [&](int v) { return __shfl_sync(0xffffffffu, v, 0); };
  int g = FUSED ? bcast(claim_raw(0)) : blockIdx.x * (kPlaneBlock / 32) + warp;
  int g_pend = claim_raw(0);                               // FUSED: the group after next
  // FUSED pass 2, one step per pass-1 group so no load waits in line: a warp
  // claims a group (stage 1), reads its window range (stage 2), then checks
  // the windows each step and completes the group once every 32-group window
  // of pass 1 it reads has been published, so its R rows and exports are
  // re-read from L2; draining waits only after pass 1 is exhausted
  int p2_stage = FUSED ? 1 : 0, p2_raw = claim_raw(1), p2_mine = -1;
  int2 p2_dep = make_int2(0, -1);
  auto fused_p2 = [&](bool wait) {
    if constexpr (FUSED) {
      if (p2_stage == 1) {
        p2_mine = bcast(p2_raw);
        if (p2_mine >= ngroups) { p2_stage = 0; return; }
        p2_dep = __ldg(P.fuse_dep + p2_mine);
        p2_stage = 2;
        if (!wait) return;
      }
      if (p2_stage != 2) return;
      for (long spin = 0;; ++spin) {
        bool ok = true;
        for (int w = min(p2_dep.x + lane, p2_dep.y); w <= p2_dep.y; w += 32) {
          int c;
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(c) : "l"(P.fuse + 3 + w) : "memory");
          ok &= c >= min(32, ngroups - 32 * w);
        }
        if (__all_sync(0xffffffffu, ok)) break;
        if (!wait) return;
        if (spin > (1l << 26)) __trap();               // never: every claimed group completes
        __nanosleep(128);
      }
      __syncwarp();                                  // every lane's acquire precedes the reads
      complete_group4(P, frec, X, R, P.e0 + 8 * p2_mine, lane, s_tab + 2 * NP);
      p2_raw = claim_raw(1);
      p2_stage = 1;
    }
  };

  // prefetch of one group of 8 elements into input buffer `buf`: u rows
  // (coalesced 8 B copies into the padded planes), the coefficient blocks and
  // the face records (16 B copies); one cp.async group per call
  auto prefetch = [&](int gg, int buf) {
    if (gg < ngroups) {
      const int e_w = P.e0 + gg * 8;
      const int ne_w = min(8, P.e1 - e_w);
      const double* ub = u + (size_t)e_w * NB;
      double* dst = sWarp + buf * kInSz;
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        const int d = lane + 32 * x;                       // element d/64, plane, node
        if (d < ne_w * NB)
          cp_async8(dst + plane_el(d >> 6) + ((d >> 4) & 3) * kPS + (d & 15), ub + d);
      }
      const double* kb = P.kco + (size_t)e_w * P.kstride;
#pragma unroll
      for (int x = 0; x < 2; ++x) {                        // 8 elements x 8 chunks of 16 B
        const int c = lane + 32 * x, el = c >> 3, part = c & 7;
        if (el < ne_w && 2 * part < P.kstride)
          cp_async16(dst + plane_el(el) + kInC + 2 * part, kb + (size_t)el * P.kstride + 2 * part);
      }
      const double* fb = reinterpret_cast<const double*>(frec + (size_t)e_w * 6);
#pragma unroll
      for (int x = 0; x < 2; ++x) {                        // 8 elements x 6 records of 16 B
        const int c = lane + 32 * x, el = c / 6, part = c % 6;
        if (c < 48 && el < ne_w) cp_async16(dst + plane_el(el) + kInF + 2 * part, fb + 2 * c);
      }
    }
    cp_async_commit();
  };

  prefetch(g, 0);
  for (int it = 0; g < ngroups; ++it) {
    const int cur = it & 1;
    const int gnext = FUSED ? bcast(g_pend) : g + stride;
    prefetch(gnext, cur ^ 1);
    if (FUSED) g_pend = claim_raw(0);
    cp_async_wait_group1();                                // this group's data landed
    __syncwarp();
    const int e = P.e0 + g * 8 + ls;
    const int e_w = P.e0 + g * 8;
    const bool active = e < P.e1;
    double* sIn = sEl + cur * kInSz;
    double* sU = sIn;
    double* sC = sIn + kInC;
    double* sXY = sU + k * kPS;                            // this thread's slot
    double* sW = sWarp + cur * kInSz;                      // staging rows of this buffer

    // ---- A: records and gathers
    double tau[6];
    int info[6];
    double ext[6][N1];                                     // neighbour / boundary face values
    if (active) {
      int nbr[6];
#pragma unroll
      for (int lf = 0; lf < 6; ++lf) {
        const double* r = sIn + kInF + 2 * lf;
        tau[lf] = r[0];
        const int2 w = *reinterpret_cast<const int2*>(r + 1);
        nbr[lf] = w.x;
        info[lf] = w.y;
      }
      // face node t of this thread's 4 values: x faces (j,k) -> j + 4k; y faces
      // (i,k) -> i + 4k; z faces, row j = k: (i,k) -> i + 4k.  A run of 4
      // consecutive, 32-B aligned neighbour nodes is fetched with 2 x 16 B loads.
#pragma unroll
      for (int lf = 0; lf < 6; ++lf) {
        const int kind = info[lf] & LDG_FACE_KIND_MASK;
#pragma unroll
        for (int a = 0; a < N1; ++a) ext[lf][a] = 0.0;
        if (kind == LDG_FACE_INTERIOR) {
          if (info[lf] & LDG_FL_UNBR) {
            const int mid = (info[lf] >> LDG_FACE_MAP_SHIFT) & 0xffff;
            const double* base = nbr_row(P, u, nbr[lf], NB);
            int nn[N1];
#pragma unroll
            for (int a = 0; a < N1; ++a)
              nn[a] = map_smem ? s_map[mid * NP + a + 4 * k] : __ldg(P.nmap + mid * NP + a + 4 * k);
            if (nn[1] == nn[0] + 1 && nn[2] == nn[0] + 2 && nn[3] == nn[0] + 3 && (nn[0] & 3) == 0) {
              const double2* b2 = reinterpret_cast<const double2*>(base + nn[0]);
              const double2 v0 = __ldg(b2), v1 = __ldg(b2 + 1);
              ext[lf][0] = v0.x; ext[lf][1] = v0.y; ext[lf][2] = v1.x; ext[lf][3] = v1.y;
            } else {
#pragma unroll
              for (int a = 0; a < N1; ++a) ext[lf][a] = __ldg(base + nn[a]);
            }
          }
        } else if (!TANGENT && gproj) {
          const double2* b2 = reinterpret_cast<const double2*>(gproj + (size_t)nbr[lf] * NP + 4 * k);
          const double2 v0 = __ldg(b2), v1 = __ldg(b2 + 1);
          ext[lf][0] = v0.x; ext[lf][1] = v0.y; ext[lf][2] = v1.x; ext[lf][3] = v1.y;
        }
      }
    } else {
#pragma unroll
      for (int lf = 0; lf < 6; ++lf) {
        tau[lf] = 0.0;
        info[lf] = LDG_FACE_NEUMANN;
#pragma unroll
        for (int a = 0; a < N1; ++a) ext[lf][a] = 0.0;
      }
    }
    // idle lanes (past the last element) run on with zero data so that every
    // __syncwarp() below is reached by the whole warp

  // ---- B: d/dz from all four planes; z-face jumps / own-data flux, row j = k
  double up[NP], hz[NP];
  constexpr bool ZMMA = (LDG_PLANE_DMMA & 2) && DIAG && !HAS_CU;
  double* sVZ = sEl + kOffVZ + kPS * k;         // this thread's z volume term (ZMMA)
  (void)sVZ;
#pragma unroll
  for (int n = 0; n < NP; ++n) {
    up[n] = sU[k * kPS + n];
    hz[n] = 0.0;
  }
  static_assert(kPS == 17, "axpy_plane assumes the 17-double plane stride");
  if constexpr (ZMMA) {
    // hz = D_z u and gz = (G D)_z u of this plane in 16 tensor-core steps;
    // gz waits in the thread's VZ slot (folded with the z lifts below)
    const double bDG = s_tab[bDG_at];
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      double gz;
      dmma_zplane(hz[n], gz, up[n], bDG);
      sVZ[n] = gz;
    }
  } else {
    axpy_plane<0>(hz, s_tab[3 * NP + 4 * k + 0], sU + 0 * kPS);
    axpy_plane<1>(hz, s_tab[3 * NP + 4 * k + 1], sU + 1 * kPS);
    axpy_plane<2>(hz, s_tab[3 * NP + 4 * k + 2], sU + 2 * kPS);
    axpy_plane<3>(hz, s_tab[3 * NP + 4 * k + 3], sU + 3 * kPS);
  }
#pragma unroll
  for (int f = 0; f < 2; ++f) {                 // faces 0 (z-, plane 0), 1 (z+, plane 3)
    const int kind = info[f] & LDG_FACE_KIND_MASK;
    const int acode = (info[f] >> LDG_FL_ALPHA_SHIFT) & 3;
    const double alpha = acode == 1 ? 1.0 : (acode == 2 ? 0.5 : 0.0);
    const bool neu = kind == LDG_FACE_NEUMANN;
    const double sgn = f ? 1.0 : -1.0;
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      const double uo = sU[(f ? 3 : 0) * kPS + i + 4 * k];
      const double ex = ext[f][i];
      const double d = uo - ex;
      const double jmp = alpha * d;
      double fh = tau[f] * (neu ? ex : d);
      if (HAS_CU && !neu) fh = fma(sgn * sC[11], uo - jmp, fh);
      sJZ[f * 20 + k * kES + i] = jmp;
      sFZ[f * 20 + k * kES + i] = fh;
    }
  }
  __syncwarp();
  double h[2][NP];                               // h_x, h_y of the plane
  {
    // h_z goes straight to the thread's F_z row (shared): it is not needed in
    // registers again until the flux combination, which keeps stage C spill-free
    const double clk = s_tab[4 * NP + k], chk = s_tab[4 * NP + 4 + k];
    const double c2 = DIAG ? sC[8] : 1.0;           // diagonal C: store F_z = C_zz h_z directly
    if constexpr (ZMMA) {
      // -G_z F_z = c_zz (gz + (G clo)_k jz_lo - (G chi)_k jz_hi): the z part
      // of the volume term without a plane exchange
      const double gl = s_tab[5 * NP + 8 + k], gh = s_tab[5 * NP + 12 + k];
#pragma unroll
      for (int n = 0; n < NP; ++n) {
        const double jl = sJZ[(n >> 2) * kES + (n & 3)], jh = sJZ[20 + (n >> 2) * kES + (n & 3)];
        sT2[k * kPS + n] = c2 * (-hz[n] - clk * jl + chk * jh);
        sVZ[n] = c2 * (sVZ[n] + gl * jl - gh * jh);
      }
    } else {
#pragma unroll
      for (int n = 0; n < NP; ++n)
        sT2[k * kPS + n] = c2 * (-hz[n] - clk * sJZ[(n >> 2) * kES + (n & 3)] + chk * sJZ[20 + (n >> 2) * kES + (n & 3)]);
    }
  }
  // ---- C: x / y faces at this plane and the in-plane gradients; the
  // own-data face fluxes go to the thread's (now dead) u-plane slot
  // sXY[(s * 2 + ax) * 4 + a]; the jumps are recomputed where they are lifted
  double alx[2], aly[2];                         // jump coefficients of the x / y faces
#pragma unroll
  for (int s = 0; s < 2; ++s) {
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
      const int lf = ax == 0 ? 4 + s : 2 + s;
      const int kind = info[lf] & LDG_FACE_KIND_MASK;
      const int acode = (info[lf] >> LDG_FL_ALPHA_SHIFT) & 3;
      const double alpha = acode == 1 ? 1.0 : (acode == 2 ? 0.5 : 0.0);
      if (ax == 0) alx[s] = alpha;
      else aly[s] = alpha;
      const bool neu = kind == LDG_FACE_NEUMANN;
      const double sgn = s ? 1.0 : -1.0;
#pragma unroll
      for (int a = 0; a < N1; ++a) {
        // x face: node (s ? 3 : 0, a, k); y face: node (a, s ? 3 : 0, k)
        const double uo = ax == 0 ? up[(s ? 3 : 0) + 4 * a] : up[a + 4 * (s ? 3 : 0)];
        const double ex = ext[lf][a];
        const double d = uo - ex;
        double fh = tau[lf] * (neu ? ex : d);
        if (HAS_CU && !neu) fh = fma(sgn * sC[9 + ax], uo - alpha * d, fh);
        sXY[(s * 2 + ax) * 4 + a] = fh;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < N1; ++j) {
    const double jxl = alx[0] * (up[4 * j] - ext[4][j]);
    const double jxh = alx[1] * (up[3 + 4 * j] - ext[5][j]);
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double vx = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) vx = fma(P.d1[i * N1 + m], up[m + 4 * j], vx);
      h[0][i + 4 * j] = -vx - P.clo[i] * jxl + P.chi[i] * jxh;
    }
  }
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    const double jyl = aly[0] * (up[i] - ext[2][i]);
    const double jyh = aly[1] * (up[i + 12] - ext[3][i]);
#pragma unroll
    for (int j = 0; j < N1; ++j) {
      double vy = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) vy = fma(P.d1[j * N1 + m], up[i + 4 * m], vy);
      h[1][i + 4 * j] = -vy - P.clo[j] * jyl + P.chi[j] * jyh;
    }
  }

  // ---- D: flux density F^q = C h (in place), face exports and the q^ own
  // share of the face fluxes, then F = F^q + Cu u
  double* fz = sT2 + k * kPS;                    // this plane's h_z, then F_z
  if (DIAG) {
    const double c0 = sC[0], c1 = sC[4];
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      h[0][n] *= c0;
      h[1][n] *= c1;
    }
  } else {
    __syncwarp();                                // keeps the C-block loads out of stage C
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      const double h0 = h[0][n], h1 = h[1][n], h2 = fz[n];
      h[0][n] = fma(sC[0], h0, fma(sC[1], h1, sC[2] * h2));
      h[1][n] = fma(sC[3], h0, fma(sC[4], h1, sC[5] * h2));
      fz[n] = fma(sC[6], h0, fma(sC[7], h1, sC[8] * h2));
    }
  }
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
      const int lf = ax == 0 ? 4 + s : 2 + s;
      const int kind = info[lf] & LDG_FACE_KIND_MASK;
      if (kind == LDG_FACE_NEUMANN) continue;
      const bool exp_ = (info[lf] & LDG_FL_EXPORT) && active;
      const double w_own = kind != LDG_FACE_INTERIOR ? 1.0
                           : ((info[lf] & LDG_FL_QOWN) ? 1.0 : ((info[lf] & LDG_FL_QHALF) ? 0.5 : 0.0));
      const double sgn = s ? 1.0 : -1.0;
      double xv[N1];
#pragma unroll
      for (int a = 0; a < N1; ++a) {
        const int n = ax == 0 ? (s ? 3 : 0) + 4 * a : a + 4 * (s ? 3 : 0);
        xv[a] = sgn * h[ax][n];
        sXY[(s * 2 + ax) * 4 + a] = fma(w_own, xv[a], sXY[(s * 2 + ax) * 4 + a]);
      }
      if (exp_) {
        if (P.x_consumer && ((unsigned)info[lf] & LDG_FL_XIDENT)) {   // same node order
          const int nbr = reinterpret_cast<const int2*>(sIn + kInF + 2 * lf + 1)->x;
          double2* xp = reinterpret_cast<double2*>(X + ((size_t)nbr * 6 + ((info[lf] >> 4) & 7)) * NP + 4 * k);
          xp[0] = make_double2(xv[0], xv[1]);
          xp[1] = make_double2(xv[2], xv[3]);
        } else if (P.x_consumer) {  // the neighbour's slot, in its face-node order
          const int inf = info[lf];
          const int nlf = (inf >> 4) & 7, mid = (inf >> LDG_FACE_MAP_SHIFT) & 0xffff;
          const int nbr = reinterpret_cast<const int2*>(sIn + kInF + 2 * lf + 1)->x;
          double* xb = X + ((size_t)nbr * 6 + nlf) * NP;
          const int nax = face_axis(3, nlf);
          int tn[N1];
#pragma unroll
          for (int a = 0; a < N1; ++a) {
            const int t = a + 4 * k;
            const int nv = map_smem ? s_map[mid * NP + t] : __ldg(P.nmap + mid * NP + t);
            tn[a] = vol_to_face<N1, 3>(nax, nv);
          }
          if (tn[1] == tn[0] + 1 && tn[2] == tn[0] + 2 && tn[3] == tn[0] + 3 && (tn[0] & 1) == 0) {
            double2* xp = reinterpret_cast<double2*>(xb + tn[0]);   // aligned run of 4
            xp[0] = make_double2(xv[0], xv[1]);
            xp[1] = make_double2(xv[2], xv[3]);
          } else {
#pragma unroll
            for (int a = 0; a < N1; ++a) xb[tn[a]] = xv[a];
          }
        } else {
          double2* xp = reinterpret_cast<double2*>(X + ((size_t)e * 6 + lf) * NP + 4 * k);
          xp[0] = make_double2(xv[0], xv[1]);
          xp[1] = make_double2(xv[2], xv[3]);
        }
      }
    }
  // z faces: all four threads share them, thread k taking column i = k of the
  // plane-0 / plane-3 F_z rows (conflict-free: bank 4e + k + 4j), so neither
  // the own-share update nor the exports diverge on k
  __syncwarp();                                  // F_z rows of planes 0 and 3 complete
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const int inf = info[f];
    const int kind = inf & LDG_FACE_KIND_MASK;
    if (kind == LDG_FACE_NEUMANN) continue;
    const bool exp_ = (inf & LDG_FL_EXPORT) && active;
    const double w_own = kind != LDG_FACE_INTERIOR ? 1.0
                         : ((inf & LDG_FL_QOWN) ? 1.0 : ((inf & LDG_FL_QHALF) ? 0.5 : 0.0));
    const double sgn = f ? 1.0 : -1.0;
    const double* fzp = sT2 + (f ? 3 : 0) * kPS + k;
    double xv[N1];
#pragma unroll
    for (int j = 0; j < N1; ++j) {               // face node (i = k, j)
      xv[j] = sgn * fzp[4 * j];
      double* z0 = sFZ + f * 20 + j * kES + k;
      *z0 = fma(w_own, xv[j], *z0);
    }
    if (exp_) {
      double* xb = X + ((size_t)e * 6 + f) * NP;
      bool mapped = false;
      int mid = 0, nax = 0;
      if (P.x_consumer) {
        const int nlf = (inf >> 4) & 7;
        xb = X + ((size_t)reinterpret_cast<const int2*>(sIn + kInF + 2 * f + 1)->x * 6 + nlf) * NP;
        if (!((unsigned)inf & LDG_FL_XIDENT)) {
          mapped = true;
          mid = (inf >> LDG_FACE_MAP_SHIFT) & 0xffff;
          nax = face_axis(3, nlf);
        }
      }
#pragma unroll
      for (int j = 0; j < N1; ++j) {
        const int t = k + 4 * j;
        int tn = t;
        if (mapped) {
          const int nv = map_smem ? s_map[mid * NP + t] : __ldg(P.nmap + mid * NP + t);
          tn = vol_to_face<N1, 3>(nax, nv);
        }
        xb[tn] = xv[j];
      }
    }
  }
  if (HAS_CU) __syncwarp();                      // F_z rows read before the Cu update
  if (HAS_CU) {
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      h[0][n] = fma(sC[9], up[n], h[0][n]);
      h[1][n] = fma(sC[10], up[n], h[1][n]);
      fz[n] = fma(sC[11], up[n], fz[n]);
    }
  }

  // ---- E: volume term through the factorisation S (x) M (x) M = M3 (G (x) I (x) I),
  // G = M^-1 S:  R = M_z [ M_x M_y V + L_xy ],  V = -(G_x F_x + G_y F_y + G_z F_z)
  // + M_z^-1 e_0 fh_z0 + M_z^-1 e_3 fh_z3 (the z-face lifts folded through M_z).
  // 6 contractions per node instead of 8, and no divergent z-lift branch.
  __syncwarp();                                  // F_z planes complete
  double v[NP];
#pragma unroll
  for (int j = 0; j < N1; ++j)
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double a = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        a = fma(P.g1[i * N1 + m], h[0][m + 4 * j], a);
        a = fma(P.g1[j * N1 + m], h[1][i + 4 * m], a);
      }
      v[i + 4 * j] = -a;
    }
  {
    const double z0 = s_tab[NP + 4 * k], z3 = s_tab[NP + 4 * k + 3];
    if constexpr (ZMMA) {
#pragma unroll
      for (int n = 0; n < NP; ++n) v[n] += sVZ[n];
    } else {
      axpy_plane<0>(v, -s_tab[4 * k + 0], sT2 + 0 * kPS);
      axpy_plane<1>(v, -s_tab[4 * k + 1], sT2 + 1 * kPS);
      axpy_plane<2>(v, -s_tab[4 * k + 2], sT2 + 2 * kPS);
      axpy_plane<3>(v, -s_tab[4 * k + 3], sT2 + 3 * kPS);
    }
#pragma unroll
    for (int n = 0; n < NP; ++n)
      v[n] = fma(z0, sFZ[(n >> 2) * kES + (n & 3)], fma(z3, sFZ[20 + (n >> 2) * kES + (n & 3)], v[n]));
  }
  // M_y along each column i, then M_x along each row j
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    double c1[N1];
#pragma unroll
    for (int j = 0; j < N1; ++j) {
      double a = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) a = fma(P.m1[j * N1 + m], v[i + 4 * m], a);
      c1[j] = a;
    }
#pragma unroll
    for (int j = 0; j < N1; ++j) v[i + 4 * j] = c1[j];
  }
#pragma unroll
  for (int j = 0; j < N1; ++j) {
    double r1[N1];
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double a = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) a = fma(P.m1[i * N1 + m], v[m + 4 * j], a);
      r1[i] = a;
    }
#pragma unroll
    for (int i = 0; i < N1; ++i) v[i + 4 * j] = r1[i];
  }
  // x / y face lifts (M along the face) from the thread's own slot
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int a = 0; a < N1; ++a) {
      double lx = 0.0, ly = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        lx = fma(P.m1[a * N1 + m], sXY[(s * 2 + 0) * 4 + m], lx);
        ly = fma(P.m1[a * N1 + m], sXY[(s * 2 + 1) * 4 + m], ly);
      }
      v[(s ? 3 : 0) + 4 * a] += lx;
      v[a + 4 * (s ? 3 : 0)] += ly;
    }
  // ---- F: z contraction, source; R rows out through shared
  double out[NP];
  if constexpr ((LDG_PLANE_DMMA & 1) != 0) {
    // R = M_z W on the tensor core, straight from the registers
    const double bM = bM_at < 0 ? 0.0 : s_tab[bM_at];
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      double unused;
      dmma_zplane(out[n], unused, v[n], bM);
    }
  } else {
    // W over the thread's u-plane slot (its face fluxes are consumed above)
#pragma unroll
    for (int n = 0; n < NP; ++n) sU[k * kPS + n] = v[n];
    __syncwarp();
#pragma unroll
    for (int n = 0; n < NP; ++n) out[n] = 0.0;
    axpy_plane<0>(out, s_tab[2 * NP + 4 * k + 0], sU + 0 * kPS);
    axpy_plane<1>(out, s_tab[2 * NP + 4 * k + 1], sU + 1 * kPS);
    axpy_plane<2>(out, s_tab[2 * NP + 4 * k + 2], sU + 2 * kPS);
    axpy_plane<3>(out, s_tab[2 * NP + 4 * k + 3], sU + 3 * kPS);
  }
  if (active) {
    int hm = 0;
#pragma unroll
    for (int n = 0; n < NP; ++n) hm = max(hm, hi_abs(out[n]));
    bad_if_any(P, e, hm);
  }
  __syncwarp();                                  // W reads done
#pragma unroll
  for (int n = 0; n < NP; ++n) sU[k * kPS + n] = out[n];
  __syncwarp();
  {
    const int nval = min(8, P.e1 - e_w) * NB;
    double* rb = R + (size_t)e_w * NB;
    const double* sb = (!TANGENT && bsrc) ? bsrc + (size_t)e_w * NB : nullptr;
#pragma unroll
    for (int x = 0; x < 16; ++x) {
      const int d = lane + 32 * x;
      if (d < nval) {
        double v = sW[plane_el(d >> 6) + ((d >> 4) & 3) * kPS + (d & 15)];
        if (sb) v += __ldg(sb + d);
        rb[d] = v;
      }
    }
  }
  __syncwarp();                                  // this buffer is refilled two groups on
  if constexpr (FUSED) {
    // publish this group (its R rows and exports) and complete one pass-2
    // group whose windows are done, if this warp holds one
    __syncwarp();                                   // the warp's R / export stores precede
    if (lane == 0)                                  // lane 0's release (cumulativity)
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" :: "l"(P.fuse + 3 + (g >> 5)) : "memory");
    fused_p2(false);
  }
  g = gnext;
  }
  if constexpr (FUSED) {
    while (p2_stage != 0) fused_p2(true);
    // the last warp out resets the counters for the next launch
    int last = 0;
    if (lane == 0) last = atomicAdd(P.fuse + 2, 1) == (int)gridDim.x * (kPlaneBlock / 32) - 1;
    if (__shfl_sync(0xffffffffu, last, 0)) {
      for (int x = lane; x < 3 + P.fuse_nwin; x += 32) P.fuse[x] = 0;
    }
  }
}

// --------------------------------------------------------------------------
// pass 1, plane mapping for hex p = 1, 2 (N1 = 2, 3; ncu = 1): config 5
// --------------------------------------------------------------------------
//
// The same stages and arithmetic as plane_kernel, with N1 threads per element
// (thread k owns z-plane k, N1^2 nodes in registers) and 32 / N1 elements per
// warp (N1 = 3: 10 elements on lanes 0..29; lanes 30, 31 run a dummy slot with
// no global side effects so every __syncwarp is reached).  At these orders the
// pencil kernel (one thread per face node) spends most of its time on
// shared-memory transposes of tiny pencils and per-element setup; here the
// x / y work and the flux combination stay in registers and only the u, F_z
// and W planes are exchanged, as at p = 3.  The thread-private x / y face
// fluxes get their own slot (4 N1 doubles do not fit a u plane below N1 = 4).

namespace {
template <int N1>
struct PlaneG {
  static constexpr int NP = N1 * N1, NB = N1 * N1 * N1;
  // plane / z-face row strides: N1 = 3 takes 11 / 3 (a bank-conflict model
  // of the kernel's shared accesses, scripts/plane_banks.py: 17% fewer
  // wavefronts than 10 / 4); N1 = 2 keeps 5 / 3
  static constexpr int PS = N1 == 3 ? NP + 2 : NP + 1;
  static constexpr int ES = N1 == 3 ? N1 : N1 + 1;
  static constexpr int XS = 4 * N1 + 1;             // x / y face-flux slot stride
  static constexpr int EPW = 32 / N1;               // elements per warp
  static constexpr int NSLOT = EPW + ((32 % N1) ? 1 : 0);
  static constexpr int InC = N1 * PS + ((N1 * PS) & 1);   // coefficient block (16-B aligned)
  static constexpr int InF = InC + 16;              // six 16-B face records
  static constexpr int InSz = InF + 12;             // one input buffer
  static constexpr int OffJ = 2 * InSz;             // z-face jumps [face][row j][i]
  static constexpr int OffF = OffJ + 2 * N1 * ES;   // z-face fluxes
  static constexpr int OffE = OffF + 2 * N1 * ES;   // F_z planes
  static constexpr int OffXY = OffE + N1 * PS;      // x / y face fluxes per thread
  static constexpr int Raw = OffXY + N1 * XS;
  static constexpr int PER = Raw + (20 - Raw % 16) % 16;   // element stride = 4 (mod 16)
  static constexpr int WPB = N1 == 2 ? 4 : (N1 == 3 ? 2 : 1);   // warps per block
  static constexpr int MINB = N1 == 2 ? 3 : 5;      // blocks per SM (shared-memory bound)
  __host__ __device__ static constexpr int el(int e) { return e * PER + (e >> 2) * 2; }
  static constexpr int WARP = el(NSLOT);            // doubles per warp region
  static_assert(PER % 16 == 4 && InSz % 2 == 0, "layout");
};

// acc[n] += c * plane[n] for a plane at an offset of OFF doubles from a 16-B
// boundary: 16-B loads wherever the pair is aligned
template <int NP, int OFF>
__device__ __forceinline__ void axpy_g(double (&acc)[NP], double c, const double* plane) {
  constexpr int H = OFF & 1;
  if constexpr (H) acc[0] = fma(c, plane[0], acc[0]);
#pragma unroll
  for (int j = 0; j < (NP - H) / 2; ++j) {
    const double2 v = reinterpret_cast<const double2*>(plane + H)[j];
    acc[H + 2 * j] = fma(c, v.x, acc[H + 2 * j]);
    acc[H + 2 * j + 1] = fma(c, v.y, acc[H + 2 * j + 1]);
  }
  if constexpr (((NP - H) & 1) != 0) acc[NP - 1] = fma(c, plane[NP - 1], acc[NP - 1]);
}

// acc += sum_m sgn coef[m] plane_m over the N1 planes at base + m PS
template <int N1, int PS, int M = 0>
__device__ __forceinline__ void axpy_planes(double (&acc)[N1 * N1], const double* coef, double sgn,
                                            const double* base) {
  if constexpr (M < N1) {
    axpy_g<N1 * N1, M * PS>(acc, sgn * coef[M], base + M * PS);
    axpy_planes<N1, PS, M + 1>(acc, coef, sgn, base);
  }
}
}  // namespace

template <int N1, bool TANGENT, bool HAS_CU, bool DIAG>
__global__ void __launch_bounds__(PlaneG<N1>::WPB * 32, PlaneG<N1>::MINB)
plane_kernel_g(const __grid_constant__ TensorParams P, const FaceRec* __restrict__ frec,
               const double* __restrict__ u, const double* __restrict__ gproj,
               const double* __restrict__ bsrc, double* __restrict__ R,
               double* __restrict__ X) {
  using G = PlaneG<N1>;
  constexpr int NP = G::NP, NB = G::NB, PS = G::PS, ES = G::ES, EPW = G::EPW;
  constexpr int LO = 0, HI = N1 - 1;
  extern __shared__ __align__(16) double psm[];
  __shared__ int s_map[kPlaneMaps * NP];
  __shared__ double s_tab[4 * NP + 2 * N1];        // G, M^-1, M, D, clo, chi
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ls = lane / N1, k = lane % N1;          // element slot (EPW: dummy), plane
  const bool map_smem = P.n_maps <= kPlaneMaps;
  if (map_smem)
    for (int x = threadIdx.x; x < P.n_maps * NP; x += blockDim.x) s_map[x] = __ldg(P.nmap + x);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int x = 0; x < NP; ++x) {
      s_tab[x] = P.g1[x];
      s_tab[NP + x] = P.m1inv[x];
      s_tab[2 * NP + x] = P.m1[x];
      s_tab[3 * NP + x] = P.d1[x];
    }
#pragma unroll
    for (int x = 0; x < N1; ++x) {
      s_tab[4 * NP + x] = P.clo[x];
      s_tab[4 * NP + N1 + x] = P.chi[x];
    }
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  double* sWarp = psm + warp * G::WARP;
  double* sEl = sWarp + G::el(ls);
  double* sJZ = sEl + G::OffJ;
  double* sFZ = sEl + G::OffF;
  double* sT2 = sEl + G::OffE;
  double* sXY = sEl + G::OffXY + k * G::XS;         // this thread's x / y face fluxes
  const int nel = P.e1 - P.e0;
  const int ngroups = (nel + EPW - 1) / EPW;
  const int stride = gridDim.x * G::WPB;
  int g = blockIdx.x * G::WPB + warp;

  auto prefetch = [&](int gg, int buf) {
    if (gg < ngroups) {
      const int e_w = P.e0 + gg * EPW;
      const int ne_w = min(EPW, P.e1 - e_w);
      const double* ub = u + (size_t)e_w * NB;
      double* dst = sWarp + buf * G::InSz;
#pragma unroll
      for (int x = 0; x < (EPW * NB + 31) / 32; ++x) {
        const int d = lane + 32 * x;
        if (d < ne_w * NB) cp_async8(dst + G::el(d / NB) + ((d / NP) % N1) * PS + d % NP, ub + d);
      }
      const double* kb = P.kco + (size_t)e_w * P.kstride;
#pragma unroll
      for (int x = 0; x < (EPW * 8 + 31) / 32; ++x) {
        const int c = lane + 32 * x, el = c >> 3, part = c & 7;
        if (el < ne_w && 2 * part < P.kstride)
          cp_async16(dst + G::el(el) + G::InC + 2 * part, kb + (size_t)el * P.kstride + 2 * part);
      }
      const double* fb = reinterpret_cast<const double*>(frec + (size_t)e_w * 6);
#pragma unroll
      for (int x = 0; x < (EPW * 6 + 31) / 32; ++x) {
        const int c = lane + 32 * x, el = c / 6, part = c % 6;
        if (el < ne_w) cp_async16(dst + G::el(el) + G::InF + 2 * part, fb + 2 * c);
      }
    }
    cp_async_commit();
  };

  prefetch(g, 0);
  for (int it = 0; g < ngroups; g += stride, ++it) {
    const int cur = it & 1;
    prefetch(g + stride, cur ^ 1);
    cp_async_wait_group1();
    __syncwarp();
    const int e = P.e0 + g * EPW + ls;
    const int e_w = P.e0 + g * EPW;
    const bool active = ls < EPW && e < P.e1;
    double* sIn = sEl + cur * G::InSz;
    double* sU = sIn;
    double* sC = sIn + G::InC;
    double* sW = sWarp + cur * G::InSz;

    // ---- A: records and gathers (face node of this thread's N1 values:
    // x faces (j, k) -> j + N1 k, y faces (i, k) -> i + N1 k, z faces row j = k)
    double tau[6];
    int info[6], nbr[6];
    double ext[6][N1];
    if (active) {
#pragma unroll
      for (int lf = 0; lf < 6; ++lf) {
        const double* r = sIn + G::InF + 2 * lf;
        tau[lf] = r[0];
        const int2 w = *reinterpret_cast<const int2*>(r + 1);
        nbr[lf] = w.x;
        info[lf] = w.y;
      }
#pragma unroll
      for (int lf = 0; lf < 6; ++lf) {
        const int kind = info[lf] & LDG_FACE_KIND_MASK;
#pragma unroll
        for (int a = 0; a < N1; ++a) ext[lf][a] = 0.0;
        if (kind == LDG_FACE_INTERIOR) {
          if (info[lf] & LDG_FL_UNBR) {
            const int mid = (info[lf] >> LDG_FACE_MAP_SHIFT) & 0xffff;
            const double* base = nbr_row(P, u, nbr[lf], NB);
#pragma unroll
            for (int a = 0; a < N1; ++a) {
              const int t = a + N1 * k;
              ext[lf][a] = __ldg(base + (map_smem ? s_map[mid * NP + t] : __ldg(P.nmap + mid * NP + t)));
            }
          }
        } else if (!TANGENT && gproj) {
#pragma unroll
          for (int a = 0; a < N1; ++a) ext[lf][a] = __ldg(gproj + (size_t)nbr[lf] * NP + N1 * k + a);
        }
      }
    } else {
#pragma unroll
      for (int lf = 0; lf < 6; ++lf) {
        tau[lf] = 0.0;
        info[lf] = LDG_FACE_NEUMANN;
        nbr[lf] = 0;
#pragma unroll
        for (int a = 0; a < N1; ++a) ext[lf][a] = 0.0;
      }
    }

    // ---- B: d/dz from all planes; z-face jumps / own-data flux, row j = k
    double up[NP], hz[NP];
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      up[n] = sU[k * PS + n];
      hz[n] = 0.0;
    }
    axpy_planes<N1, PS>(hz, s_tab + 3 * NP + N1 * k, 1.0, sU);
#pragma unroll
    for (int f = 0; f < 2; ++f) {                   // faces 0 (z-, plane 0), 1 (z+, plane N1-1)
      const int kind = info[f] & LDG_FACE_KIND_MASK;
      const int acode = (info[f] >> LDG_FL_ALPHA_SHIFT) & 3;
      const double alpha = acode == 1 ? 1.0 : (acode == 2 ? 0.5 : 0.0);
      const bool neu = kind == LDG_FACE_NEUMANN;
      const double sgn = f ? 1.0 : -1.0;
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        const double uo = sU[(f ? HI : LO) * PS + i + N1 * k];
        const double ex = ext[f][i];
        const double d = uo - ex;
        const double jmp = alpha * d;
        double fh = tau[f] * (neu ? ex : d);
        if (HAS_CU && !neu) fh = fma(sgn * sC[11], uo - jmp, fh);
        sJZ[f * N1 * ES + k * ES + i] = jmp;
        sFZ[f * N1 * ES + k * ES + i] = fh;
      }
    }
    __syncwarp();
    {
      const double clk = s_tab[4 * NP + k], chk = s_tab[4 * NP + N1 + k];
      const double c2 = DIAG ? sC[8] : 1.0;
#pragma unroll
      for (int n = 0; n < NP; ++n)
        sT2[k * PS + n] = c2 * (-hz[n] - clk * sJZ[(n / N1) * ES + n % N1] +
                                chk * sJZ[N1 * ES + (n / N1) * ES + n % N1]);
    }
    // ---- C: x / y faces at this plane and the in-plane gradients
    double h[2][NP];
    double alx[2], aly[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
#pragma unroll
      for (int ax = 0; ax < 2; ++ax) {
        const int lf = ax == 0 ? 4 + s : 2 + s;
        const int kind = info[lf] & LDG_FACE_KIND_MASK;
        const int acode = (info[lf] >> LDG_FL_ALPHA_SHIFT) & 3;
        const double alpha = acode == 1 ? 1.0 : (acode == 2 ? 0.5 : 0.0);
        if (ax == 0) alx[s] = alpha;
        else aly[s] = alpha;
        const bool neu = kind == LDG_FACE_NEUMANN;
        const double sgn = s ? 1.0 : -1.0;
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          const double uo = ax == 0 ? up[(s ? HI : LO) + N1 * a] : up[a + N1 * (s ? HI : LO)];
          const double ex = ext[lf][a];
          const double d = uo - ex;
          double fh = tau[lf] * (neu ? ex : d);
          if (HAS_CU && !neu) fh = fma(sgn * sC[9 + ax], uo - alpha * d, fh);
          sXY[(s * 2 + ax) * N1 + a] = fh;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < N1; ++j) {
      const double jxl = alx[0] * (up[N1 * j] - ext[4][j]);
      const double jxh = alx[1] * (up[HI + N1 * j] - ext[5][j]);
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        double vx = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) vx = fma(P.d1[i * N1 + m], up[m + N1 * j], vx);
        h[0][i + N1 * j] = -vx - P.clo[i] * jxl + P.chi[i] * jxh;
      }
    }
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      const double jyl = aly[0] * (up[i] - ext[2][i]);
      const double jyh = aly[1] * (up[i + N1 * HI] - ext[3][i]);
#pragma unroll
      for (int j = 0; j < N1; ++j) {
        double vy = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) vy = fma(P.d1[j * N1 + m], up[i + N1 * m], vy);
        h[1][i + N1 * j] = -vy - P.clo[j] * jyl + P.chi[j] * jyh;
      }
    }

    // ---- D: flux density F^q = C h, face exports and the own q^ share
    double* fz = sT2 + k * PS;
    if (DIAG) {
      const double c0 = sC[0], c1 = sC[4];
#pragma unroll
      for (int n = 0; n < NP; ++n) {
        h[0][n] *= c0;
        h[1][n] *= c1;
      }
    } else {
      __syncwarp();
#pragma unroll
      for (int n = 0; n < NP; ++n) {
        const double h0 = h[0][n], h1 = h[1][n], h2 = fz[n];
        h[0][n] = fma(sC[0], h0, fma(sC[1], h1, sC[2] * h2));
        h[1][n] = fma(sC[3], h0, fma(sC[4], h1, sC[5] * h2));
        fz[n] = fma(sC[6], h0, fma(sC[7], h1, sC[8] * h2));
      }
    }
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int ax = 0; ax < 2; ++ax) {
        const int lf = ax == 0 ? 4 + s : 2 + s;
        const int kind = info[lf] & LDG_FACE_KIND_MASK;
        if (kind == LDG_FACE_NEUMANN) continue;
        const bool exp_ = (info[lf] & LDG_FL_EXPORT) && active;
        const double w_own = kind != LDG_FACE_INTERIOR ? 1.0
                             : ((info[lf] & LDG_FL_QOWN) ? 1.0 : ((info[lf] & LDG_FL_QHALF) ? 0.5 : 0.0));
        const double sgn = s ? 1.0 : -1.0;
        double xv[N1];
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          const int n = ax == 0 ? (s ? HI : LO) + N1 * a : a + N1 * (s ? HI : LO);
          xv[a] = sgn * h[ax][n];
          sXY[(s * 2 + ax) * N1 + a] = fma(w_own, xv[a], sXY[(s * 2 + ax) * N1 + a]);
        }
        if (exp_) {
          const int inf = info[lf];
          if (P.x_consumer) {                        // the neighbour's slot, in its face-node order
            const int nlf = (inf >> 4) & 7;
            double* xb = X + ((size_t)nbr[lf] * 6 + nlf) * NP;
            if ((unsigned)inf & LDG_FL_XIDENT) {
#pragma unroll
              for (int a = 0; a < N1; ++a) xb[a + N1 * k] = xv[a];
            } else {
              const int mid = (inf >> LDG_FACE_MAP_SHIFT) & 0xffff;
              const int nax = face_axis(3, nlf);
#pragma unroll
              for (int a = 0; a < N1; ++a) {
                const int t = a + N1 * k;
                const int nv = map_smem ? s_map[mid * NP + t] : __ldg(P.nmap + mid * NP + t);
                xb[vol_to_face<N1, 3>(nax, nv)] = xv[a];
              }
            }
          } else {
#pragma unroll
            for (int a = 0; a < N1; ++a) X[((size_t)e * 6 + lf) * NP + a + N1 * k] = xv[a];
          }
        }
      }
    // z faces: thread k takes column i = k of the plane-0 / plane-(N1-1) F_z rows
    __syncwarp();
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int inf = info[f];
      const int kind = inf & LDG_FACE_KIND_MASK;
      if (kind == LDG_FACE_NEUMANN) continue;
      const bool exp_ = (inf & LDG_FL_EXPORT) && active;
      const double w_own = kind != LDG_FACE_INTERIOR ? 1.0
                           : ((inf & LDG_FL_QOWN) ? 1.0 : ((inf & LDG_FL_QHALF) ? 0.5 : 0.0));
      const double sgn = f ? 1.0 : -1.0;
      const double* fzp = sT2 + (f ? HI : LO) * PS + k;
      double xv[N1];
#pragma unroll
      for (int j = 0; j < N1; ++j) {                // face node (i = k, j)
        xv[j] = sgn * fzp[N1 * j];
        double* z0 = sFZ + f * N1 * ES + j * ES + k;
        *z0 = fma(w_own, xv[j], *z0);
      }
      if (exp_) {
        double* xb = X + ((size_t)e * 6 + f) * NP;
        bool mapped = false;
        int mid = 0, nax = 0;
        if (P.x_consumer) {
          const int nlf = (inf >> 4) & 7;
          xb = X + ((size_t)nbr[f] * 6 + nlf) * NP;
          if (!((unsigned)inf & LDG_FL_XIDENT)) {
            mapped = true;
            mid = (inf >> LDG_FACE_MAP_SHIFT) & 0xffff;
            nax = face_axis(3, nlf);
          }
        }
#pragma unroll
        for (int j = 0; j < N1; ++j) {
          const int t = k + N1 * j;
          int tn = t;
          if (mapped) {
            const int nv = map_smem ? s_map[mid * NP + t] : __ldg(P.nmap + mid * NP + t);
            tn = vol_to_face<N1, 3>(nax, nv);
          }
          xb[tn] = xv[j];
        }
      }
    }
    if (HAS_CU) {
      __syncwarp();                                  // F_z rows read before the Cu update
#pragma unroll
      for (int n = 0; n < NP; ++n) {
        h[0][n] = fma(sC[9], up[n], h[0][n]);
        h[1][n] = fma(sC[10], up[n], h[1][n]);
        fz[n] = fma(sC[11], up[n], fz[n]);
      }
    }

    // ---- E: R = M_z [M_x M_y V + L_xy], V = -(G_x F_x + G_y F_y + G_z F_z)
    // + M_z^-1 (e_0 fh_z0 + e_{N1-1} fh_z1)
    __syncwarp();                                    // F_z planes complete
    double v[NP];
#pragma unroll
    for (int j = 0; j < N1; ++j)
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          a = fma(P.g1[i * N1 + m], h[0][m + N1 * j], a);
          a = fma(P.g1[j * N1 + m], h[1][i + N1 * m], a);
        }
        v[i + N1 * j] = -a;
      }
    axpy_planes<N1, PS>(v, s_tab + N1 * k, -1.0, sT2);
    {
      const double z0 = s_tab[NP + N1 * k], z1 = s_tab[NP + N1 * k + HI];
#pragma unroll
      for (int n = 0; n < NP; ++n)
        v[n] = fma(z0, sFZ[(n / N1) * ES + n % N1], fma(z1, sFZ[N1 * ES + (n / N1) * ES + n % N1], v[n]));
    }
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double c1[N1];
#pragma unroll
      for (int j = 0; j < N1; ++j) {
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) a = fma(P.m1[j * N1 + m], v[i + N1 * m], a);
        c1[j] = a;
      }
#pragma unroll
      for (int j = 0; j < N1; ++j) v[i + N1 * j] = c1[j];
    }
#pragma unroll
    for (int j = 0; j < N1; ++j) {
      double r1[N1];
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) a = fma(P.m1[i * N1 + m], v[m + N1 * j], a);
        r1[i] = a;
      }
#pragma unroll
      for (int i = 0; i < N1; ++i) v[i + N1 * j] = r1[i];
    }
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int a = 0; a < N1; ++a) {
        double lx = 0.0, ly = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          lx = fma(P.m1[a * N1 + m], sXY[(s * 2 + 0) * N1 + m], lx);
          ly = fma(P.m1[a * N1 + m], sXY[(s * 2 + 1) * N1 + m], ly);
        }
        v[(s ? HI : LO) + N1 * a] += lx;
        v[a + N1 * (s ? HI : LO)] += ly;
      }
    // ---- F: z contraction, R rows out through shared
#pragma unroll
    for (int n = 0; n < NP; ++n) sU[k * PS + n] = v[n];
    __syncwarp();
    double out[NP];
#pragma unroll
    for (int n = 0; n < NP; ++n) out[n] = 0.0;
    axpy_planes<N1, PS>(out, s_tab + 2 * NP + N1 * k, 1.0, sU);
    if (active) {
      int hm = 0;
#pragma unroll
      for (int n = 0; n < NP; ++n) hm = max(hm, hi_abs(out[n]));
      bad_if_any(P, e, hm);
    }
    __syncwarp();
#pragma unroll
    for (int n = 0; n < NP; ++n) sU[k * PS + n] = out[n];
    __syncwarp();
    {
      const int nval = min(EPW, P.e1 - e_w) * NB;
      double* rb = R + (size_t)e_w * NB;
      const double* sb = (!TANGENT && bsrc) ? bsrc + (size_t)e_w * NB : nullptr;
#pragma unroll
      for (int x = 0; x < (EPW * NB + 31) / 32; ++x) {
        const int d = lane + 32 * x;
        if (d < nval) {
          double val = sW[G::el(d / NB) + ((d / NP) % N1) * PS + d % NP];
          if (sb) val += __ldg(sb + d);
          rb[d] = val;
        }
      }
    }
    __syncwarp();
  }
}

// --------------------------------------------------------------------------
// pass 1 at hex p = 1 (ncu = 1): one thread per element, no exchange at all
// --------------------------------------------------------------------------
//
// An 8-node element fits one thread's registers, so every contraction of the
// plane kernel's stages (same arithmetic, same order per z-plane k) runs
// in registers with compile-time operator entries; nothing goes through
// shared memory.  The element's u row, coefficient block and face records are
// 16-B loads of contiguous rows (a warp covers 32 consecutive elements).
// Face node t of a face: z faces (i, j) -> i + 2j, y faces (i, k) -> i + 2k,
// x faces (j, k) -> j + 2k; node n = i + 2j + 4k.

template <bool TANGENT, bool HAS_CU, bool DIAG>
__global__ void __launch_bounds__(128, 3)
elem_kernel_p1(const __grid_constant__ TensorParams P, const FaceRec* __restrict__ frec,
               const double* __restrict__ u, const double* __restrict__ gproj,
               const double* __restrict__ bsrc, double* __restrict__ R,
               double* __restrict__ X) {
  constexpr int N1 = 2, NP = 4, NB = 8;
  asm volatile("griddepcontrol.launch_dependents;");
  const int e = P.e0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P.e1) return;
  double uu[NB];
  {
    const double2* up = reinterpret_cast<const double2*>(u + (size_t)e * NB);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 v = __ldg(up + q);
      uu[2 * q] = v.x;
      uu[2 * q + 1] = v.y;
    }
  }
  double C[12];
  {
    const double2* kp = reinterpret_cast<const double2*>(P.kco + (size_t)e * P.kstride);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const double2 v = __ldg(kp + q);
      C[2 * q] = v.x;
      C[2 * q + 1] = v.y;
    }
  }
  double tau[6];
  int info[6], nbr[6];
#pragma unroll
  for (int lf = 0; lf < 6; ++lf) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(frec + (size_t)e * 6 + lf));
    tau[lf] = v.x;
    nbr[lf] = __double2loint(v.y);
    info[lf] = __double2hiint(v.y);
  }
  const bool map_ok = true;
  (void)map_ok;
  double ext[6][NP];
#pragma unroll
  for (int lf = 0; lf < 6; ++lf) {
    const int kind = info[lf] & LDG_FACE_KIND_MASK;
#pragma unroll
    for (int t = 0; t < NP; ++t) ext[lf][t] = 0.0;
    if (kind == LDG_FACE_INTERIOR) {
      if (info[lf] & LDG_FL_UNBR) {
        const int mid = (info[lf] >> LDG_FACE_MAP_SHIFT) & 0xffff;
        const double* base = nbr_row(P, u, nbr[lf], NB);
#pragma unroll
        for (int t = 0; t < NP; ++t) ext[lf][t] = __ldg(base + __ldg(P.nmap + mid * NP + t));
      }
    } else if (!TANGENT && gproj) {
#pragma unroll
      for (int t = 0; t < NP; ++t) ext[lf][t] = __ldg(gproj + (size_t)nbr[lf] * NP + t);
    }
  }
  auto alpha_of = [&](int lf) {
    const int acode = (info[lf] >> LDG_FL_ALPHA_SHIFT) & 3;
    return acode == 1 ? 1.0 : (acode == 2 ? 0.5 : 0.0);
  };
  auto w_own_of = [&](int lf) {
    const int kind = info[lf] & LDG_FACE_KIND_MASK;
    return kind != LDG_FACE_INTERIOR ? 1.0
           : ((info[lf] & LDG_FL_QOWN) ? 1.0 : ((info[lf] & LDG_FL_QHALF) ? 0.5 : 0.0));
  };

  // ---- z faces (planes 0 and 1): jumps and own-data fluxes; F_z planes
  double jz[2][NP], fhz[2][NP], fz[2][NP];
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const bool neu = (info[f] & LDG_FACE_KIND_MASK) == LDG_FACE_NEUMANN;
    const double alpha = alpha_of(f), sgn = f ? 1.0 : -1.0;
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      const double uo = uu[n + NP * f], ex = ext[f][n];
      const double d = uo - ex;
      const double jmp = alpha * d;
      double fh = tau[f] * (neu ? ex : d);
      if (HAS_CU && !neu) fh = fma(sgn * C[11], uo - jmp, fh);
      jz[f][n] = jmp;
      fhz[f][n] = fh;
    }
  }
  {
    const double c2 = DIAG ? C[8] : 1.0;
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int n = 0; n < NP; ++n) {
        double hz = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) hz = fma(P.d1[k * N1 + m], uu[n + NP * m], hz);
        fz[k][n] = c2 * (-hz - P.clo[k] * jz[0][n] + P.chi[k] * jz[1][n]);
      }
  }
  // ---- x / y faces per plane: own-data fluxes, gradients, flux density
  double fxy[N1][4][N1];                        // [plane][s * 2 + ax][face-row a]
  double hx[N1][NP], hy[N1][NP];
  double alx[2], aly[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    alx[s] = alpha_of(4 + s);
    aly[s] = alpha_of(2 + s);
  }
#pragma unroll
  for (int k = 0; k < N1; ++k) {
    const double* up = uu + NP * k;
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int ax = 0; ax < 2; ++ax) {
        const int lf = ax == 0 ? 4 + s : 2 + s;
        const bool neu = (info[lf] & LDG_FACE_KIND_MASK) == LDG_FACE_NEUMANN;
        const double alpha = ax == 0 ? alx[s] : aly[s], sgn = s ? 1.0 : -1.0;
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          const double uo = ax == 0 ? up[s + N1 * a] : up[a + N1 * s];
          const double ex = ext[lf][a + N1 * k];
          const double d = uo - ex;
          double fh = tau[lf] * (neu ? ex : d);
          if (HAS_CU && !neu) fh = fma(sgn * C[9 + ax], uo - alpha * d, fh);
          fxy[k][s * 2 + ax][a] = fh;
        }
      }
#pragma unroll
    for (int j = 0; j < N1; ++j) {
      const double jxl = alx[0] * (up[N1 * j] - ext[4][j + N1 * k]);
      const double jxh = alx[1] * (up[1 + N1 * j] - ext[5][j + N1 * k]);
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        double vx = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) vx = fma(P.d1[i * N1 + m], up[m + N1 * j], vx);
        hx[k][i + N1 * j] = -vx - P.clo[i] * jxl + P.chi[i] * jxh;
      }
    }
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      const double jyl = aly[0] * (up[i] - ext[2][i + N1 * k]);
      const double jyh = aly[1] * (up[i + N1] - ext[3][i + N1 * k]);
#pragma unroll
      for (int j = 0; j < N1; ++j) {
        double vy = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) vy = fma(P.d1[j * N1 + m], up[i + N1 * m], vy);
        hy[k][i + N1 * j] = -vy - P.clo[j] * jyl + P.chi[j] * jyh;
      }
    }
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      if (DIAG) {
        hx[k][n] *= C[0];
        hy[k][n] *= C[4];
      } else {
        const double h0 = hx[k][n], h1 = hy[k][n], h2 = fz[k][n];
        hx[k][n] = fma(C[0], h0, fma(C[1], h1, C[2] * h2));
        hy[k][n] = fma(C[3], h0, fma(C[4], h1, C[5] * h2));
        fz[k][n] = fma(C[6], h0, fma(C[7], h1, C[8] * h2));
      }
    }
  }
  // ---- exports and the own share of f(., q^)
  auto put = [&](int lf, int t, double v) {
    const int inf = info[lf];
    if (P.x_consumer) {
      const int nlf = (inf >> 4) & 7;
      double* xb = X + ((size_t)nbr[lf] * 6 + nlf) * NP;
      if ((unsigned)inf & LDG_FL_XIDENT) xb[t] = v;
      else {
        const int mid = (inf >> LDG_FACE_MAP_SHIFT) & 0xffff;
        xb[vol_to_face<N1, 3>(face_axis(3, nlf), __ldg(P.nmap + mid * NP + t))] = v;
      }
    } else {
      X[((size_t)e * 6 + lf) * NP + t] = v;
    }
  };
#pragma unroll
  for (int k = 0; k < N1; ++k)
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int ax = 0; ax < 2; ++ax) {
        const int lf = ax == 0 ? 4 + s : 2 + s;
        if ((info[lf] & LDG_FACE_KIND_MASK) == LDG_FACE_NEUMANN) continue;
        const bool exp_ = info[lf] & LDG_FL_EXPORT;
        const double w_own = w_own_of(lf), sgn = s ? 1.0 : -1.0;
#pragma unroll
        for (int a = 0; a < N1; ++a) {
          const int n = ax == 0 ? s + N1 * a : a + N1 * s;
          const double xv = sgn * (ax == 0 ? hx[k][n] : hy[k][n]);
          fxy[k][s * 2 + ax][a] = fma(w_own, xv, fxy[k][s * 2 + ax][a]);
          if (exp_) put(lf, a + N1 * k, xv);
        }
      }
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    if ((info[f] & LDG_FACE_KIND_MASK) == LDG_FACE_NEUMANN) continue;
    const bool exp_ = info[f] & LDG_FL_EXPORT;
    const double w_own = w_own_of(f), sgn = f ? 1.0 : -1.0;
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      const double xv = sgn * fz[f][n];
      fhz[f][n] = fma(w_own, xv, fhz[f][n]);
      if (exp_) put(f, n, xv);
    }
  }
  if (HAS_CU) {
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int n = 0; n < NP; ++n) {
        hx[k][n] = fma(C[9], uu[n + NP * k], hx[k][n]);
        hy[k][n] = fma(C[10], uu[n + NP * k], hy[k][n]);
        fz[k][n] = fma(C[11], uu[n + NP * k], fz[k][n]);
      }
  }
  // ---- volume term and lifts per plane, then the z contraction
  double w[N1][NP];
#pragma unroll
  for (int k = 0; k < N1; ++k) {
    double v[NP];
#pragma unroll
    for (int j = 0; j < N1; ++j)
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          a = fma(P.g1[i * N1 + m], hx[k][m + N1 * j], a);
          a = fma(P.g1[j * N1 + m], hy[k][i + N1 * m], a);
        }
        v[i + N1 * j] = -a;
      }
#pragma unroll
    for (int m = 0; m < N1; ++m)
#pragma unroll
      for (int n = 0; n < NP; ++n) v[n] = fma(-P.g1[k * N1 + m], fz[m][n], v[n]);
#pragma unroll
    for (int n = 0; n < NP; ++n)
      v[n] = fma(P.m1inv[k * N1], fhz[0][n], fma(P.m1inv[k * N1 + 1], fhz[1][n], v[n]));
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double c1[N1];
#pragma unroll
      for (int j = 0; j < N1; ++j) {
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) a = fma(P.m1[j * N1 + m], v[i + N1 * m], a);
        c1[j] = a;
      }
#pragma unroll
      for (int j = 0; j < N1; ++j) v[i + N1 * j] = c1[j];
    }
#pragma unroll
    for (int j = 0; j < N1; ++j) {
      double r1[N1];
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) a = fma(P.m1[i * N1 + m], v[m + N1 * j], a);
        r1[i] = a;
      }
#pragma unroll
      for (int i = 0; i < N1; ++i) v[i + N1 * j] = r1[i];
    }
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int a = 0; a < N1; ++a) {
        double lx = 0.0, ly = 0.0;
#pragma unroll
        for (int m = 0; m < N1; ++m) {
          lx = fma(P.m1[a * N1 + m], fxy[k][s * 2 + 0][m], lx);
          ly = fma(P.m1[a * N1 + m], fxy[k][s * 2 + 1][m], ly);
        }
        v[s + N1 * a] += lx;
        v[a + N1 * s] += ly;
      }
#pragma unroll
    for (int n = 0; n < NP; ++n) w[k][n] = v[n];
  }
  double out[NB];
#pragma unroll
  for (int k = 0; k < N1; ++k)
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      double a = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) a = fma(P.m1[k * N1 + m], w[m][n], a);
      out[n + NP * k] = a;
    }
  if (!TANGENT && bsrc) {
    const double2* bp = reinterpret_cast<const double2*>(bsrc + (size_t)e * NB);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 b = __ldg(bp + q);
      out[2 * q] += b.x;
      out[2 * q + 1] += b.y;
    }
  }
  int hm = 0;
#pragma unroll
  for (int n = 0; n < NB; ++n) hm = max(hm, hi_abs(out[n]));
  bad_if_any(P, e, hm);
  double2* rp = reinterpret_cast<double2*>(R + (size_t)e * NB);
#pragma unroll
  for (int q = 0; q < 4; ++q) rp[q] = make_double2(out[2 * q], out[2 * q + 1]);
}

// pass 2 at hex p = 1 (consumer-slot exports), one thread per element: the
// element's R row, the exports of its completion faces (one 32-B row each)
// lifted by M1 (x) M1 in registers, in complete_warp_kernel's face and
// contraction order
__global__ void __launch_bounds__(256)
complete_elem_p1(const __grid_constant__ TensorParams P, const FaceRec* __restrict__ frec,
                 const double* __restrict__ X, double* __restrict__ R) {
  constexpr int N1 = 2, NP = 4, NB = 8;
  const int e = P.e0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P.e1) return;
  const double wgt = P.grad_centered ? -0.5 : -1.0;
  int info[6];
#pragma unroll
  for (int lf = 0; lf < 6; ++lf) info[lf] = __ldg(reinterpret_cast<const int*>(frec + (size_t)e * 6 + lf) + 3);
  double r[NB];
  {
    const double2* rp = reinterpret_cast<const double2*>(R + (size_t)e * NB);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 v = rp[q];
      r[2 * q] = v.x;
      r[2 * q + 1] = v.y;
    }
  }
#pragma unroll
  for (int lf = 0; lf < 6; ++lf) {
    if (!(info[lf] & LDG_FL_COMPLETE)) continue;
    const double2* xp = reinterpret_cast<const double2*>(X + ((size_t)e * 6 + lf) * NP);
    const double2 x0 = __ldg(xp), x1 = __ldg(xp + 1);
    const double v[NP] = {wgt * x0.x, wgt * x0.y, wgt * x1.x, wgt * x1.y};
    // w(a', b) = sum_a M[a'][a] v(a, b);  L(a', b') = sum_b M[b'][b] w(a', b)
    double w[NP], L[NP];
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
      for (int a2 = 0; a2 < N1; ++a2) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < N1; ++a) acc = fma(P.m1[a2 * N1 + a], v[a + N1 * b], acc);
        w[a2 + N1 * b] = acc;
      }
#pragma unroll
    for (int b2 = 0; b2 < N1; ++b2)
#pragma unroll
      for (int a2 = 0; a2 < N1; ++a2) {
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < N1; ++b) acc = fma(P.m1[b2 * N1 + b], w[a2 + N1 * b], acc);
        L[a2 + N1 * b2] = acc;
      }
    // face node (a, b) -> volume node: z faces (a, b, 0|1), y faces (a, 0|1, b),
    // x faces (0|1, a, b)
    const int side = lf & 1;
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
      for (int a = 0; a < N1; ++a) {
        const int node = lf < 2 ? a + N1 * b + NP * side
                                : (lf < 4 ? a + N1 * side + NP * b : side + N1 * a + NP * b);
        r[node] += L[a + N1 * b];
      }
  }
  int hm = 0;
#pragma unroll
  for (int n = 0; n < NB; ++n) hm = max(hm, hi_abs(r[n]));
  bad_if_any(P, e, hm);
  double2* rp = reinterpret_cast<double2*>(R + (size_t)e * NB);
#pragma unroll
  for (int q = 0; q < 4; ++q) rp[q] = make_double2(r[2 * q], r[2 * q + 1]);
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

#ifndef LDG_P2_MINB6
#define LDG_P2_MINB6 8            // hex p = 5 block pass 2: 8 blocks / SM (64 registers; ncu 77.1 -> 68.3 us)
#endif
#ifndef LDG_P2P_MINB
#define LDG_P2P_MINB 8        // persistent pass-2 blocks per SM (64 registers)
#endif
// one-shot pass 2: a 40-register budget (12 blocks / SM) measured 58.4 us vs
// 64.6 us at the default on config 3; other shapes keep the default
template <int N1, int ND, int NCU>
constexpr int p2_min_blocks() {
  return (N1 == 4 && ND == 3 && NCU == 1) ? 12 : (((N1 == 5 || N1 == 6) && ND == 3 && NCU == 1) ? LDG_P2_MINB6 : 1);
}

template <int N1, int ND, int NCU>
__global__ void __launch_bounds__(kFBlock, p2_min_blocks<N1, ND, NCU>())
complete_kernel(const __grid_constant__ TensorParams P, const FaceRec* __restrict__ frec,
                const double* __restrict__ X, double* __restrict__ R) {
  using S = P2Smem<N1, ND, NCU>;
  constexpr int NB = S::NB, NF = S::NF, TPE = S::TPE, EPB = S::EPB, NFACE = S::NFACE;
  __shared__ double sv[EPB][NFACE][NF][NCU];    // neighbour exports, then lifted values
  __shared__ double sw2[EPB][NFACE][NF][NCU];   // first-direction partial lift
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  // blocks run in reverse element order: pass 1 finished with the last
  // elements, whose R rows and exports are still resident in L2
  const int e = P.e0 + (gridDim.x - 1 - blockIdx.x) * EPB + slot;
  const bool active = slot < EPB && e < P.e1;
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
      if (P.x_consumer) {                 // the exporter wrote into this element's slot
        src[lf] = act ? X + (((size_t)e * NFACE + lf) * NF + lt) * NCU : nullptr;
        continue;
      }
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
    int hm = 0;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
      const double out = rcol[c][k] + acc[k];
      hm = max(hm, hi_abs(out));
      Re[node * NCU + c] = out;
    }
    bad_if_any(P, e, hm);
  }
}

// Persistent, software-pipelined pass 2 for consumer-slot exports (the
// default layout): the exports of element e sit in e's own 2*ND slots, so
// the only dependent load is the completion mask.  Each block walks its
// element groups with a two-deep register pipeline — the masks of group
// g + 2, the R columns and exports of group g + 1 are in flight while group
// g is lifted and written — so HBM sees ~3 groups of loads per block instead
// of one dependent chain.
template <int N1, int ND, int NCU>
__global__ void __launch_bounds__(kFBlock, LDG_P2P_MINB)
complete_pipe_kernel(const __grid_constant__ TensorParams P, const FaceRec* __restrict__ frec,
                     const double* __restrict__ X, double* __restrict__ R) {
  using S = P2Smem<N1, ND, NCU>;
  constexpr int NB = S::NB, NF = S::NF, TPE = S::TPE, EPB = S::EPB, NFACE = S::NFACE;
  __shared__ double sv[EPB][NFACE][NF][NCU];
  __shared__ double sw2[EPB][NFACE][NF][NCU];
  const int slot = threadIdx.x / TPE, lt = threadIdx.x % TPE;
  const int i = lt % N1, j = ND == 3 ? lt / N1 : 0;
  double Mi[N1], Mj[N1];
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    Mi[m] = P.m1[i * N1 + m];
    Mj[m] = P.m1[j * N1 + m];
  }
  const int nel = P.e1 - P.e0;
  const int ngroups = (nel + EPB - 1) / EPB;
  const int stride = gridDim.x;
  const double wgt = P.grad_centered ? -0.5 : -1.0;
  // groups in reverse order: pass 1 finished with the last elements, whose R
  // rows and exports are still resident in L2
  auto elem = [&](int g) { return P.e0 + (ngroups - 1 - g) * EPB + slot; };
  auto load_mask = [&](int g) {
    int m = 0;
    const int e = elem(g);
    if (g < ngroups && slot < EPB && e < P.e1) {
#pragma unroll
      for (int lf = 0; lf < NFACE; ++lf) {
        const int info = __ldg(reinterpret_cast<const int*>(frec + (size_t)e * NFACE + lf) + 3);
        m |= (info & LDG_FL_COMPLETE) ? (1 << lf) : 0;
      }
      m |= 1 << 30;                                  // active
    }
    return m;
  };
  auto load_data = [&](int g, int m, double (&rc)[NCU][N1], double (&xv)[NFACE][NCU]) {
    const int e = elem(g);
    const bool act = m & (1 << 30);
#pragma unroll
    for (int k = 0; k < N1; ++k)
#pragma unroll
      for (int c = 0; c < NCU; ++c)
        rc[c][k] = act ? __ldg(R + ((size_t)e * NB + (ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k)) * NCU + c)
                       : 0.0;
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf)
#pragma unroll
      for (int c = 0; c < NCU; ++c)
        xv[lf][c] = (m & (1 << lf)) ? __ldg(X + (((size_t)e * NFACE + lf) * NF + lt) * NCU + c) : 0.0;
  };

  int g = blockIdx.x;
  int m_c = load_mask(g), m_n = load_mask(g + stride);
  double r_c[NCU][N1], x_c[NFACE][NCU], r_n[NCU][N1], x_n[NFACE][NCU];
  load_data(g, m_c, r_c, x_c);
  for (; g < ngroups; g += stride) {
    const int m_nn = load_mask(g + 2 * stride);
    load_data(g + stride, m_n, r_n, x_n);
    const int e = elem(g);
    const bool active = m_c & (1 << 30);
    const int mask = m_c & 63;
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf)
#pragma unroll
      for (int c = 0; c < NCU; ++c) sv[slot][lf][lt][c] = wgt * x_c[lf][c];
    __syncthreads();
    if (active) {
#pragma unroll
      for (int lf = 0; lf < NFACE; ++lf) {
        if (!(mask & (1 << lf))) continue;
#pragma unroll
        for (int c = 0; c < NCU; ++c) {
          double w = 0.0;
#pragma unroll
          for (int aa = 0; aa < N1; ++aa)
            w = fma(Mi[aa], sv[slot][lf][ND == 3 ? aa + N1 * j : aa][c], w);
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
          sv[slot][lf][lt][c] = o;
        }
      }
    }
    __syncthreads();
    if (active && mask) {
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
          if (mask & 1) acc[0] += fval(0, i, c);
          if (mask & 4) acc[N1 - 1] += fval(2, i, c);
#pragma unroll
          for (int k = 0; k < N1; ++k) {
            if ((mask & 8) && i == 0) acc[k] += fval(3, k, c);
            if ((mask & 2) && i == N1 - 1) acc[k] += fval(1, k, c);
          }
        }
        int hm = 0;
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          const int node = ND == 3 ? i + N1 * j + N1 * N1 * k : i + N1 * k;
          const double out = r_c[c][k] + acc[k];
          hm = max(hm, hi_abs(out));
          Re[node * NCU + c] = out;
        }
        bad_if_any(P, e, hm);
      }
    }
    __syncthreads();                                  // sv / sw2 reused next group
    m_c = m_n;
    m_n = m_nn;
#pragma unroll
    for (int c = 0; c < NCU; ++c)
#pragma unroll
      for (int k = 0; k < N1; ++k) r_c[c][k] = r_n[c][k];
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf)
#pragma unroll
      for (int c = 0; c < NCU; ++c) x_c[lf][c] = x_n[lf][c];
  }
}

// Register-only pass 2 for hex p = 3, ncu = 1 with consumer-slot exports:
// half a warp per element, lane t = i + 4j owns R column (i, j) and face node
// t of every face.  A completion face's 16 exports arrive as one coalesced
// 128 B row; (M1 (x) M1) is applied with 8 shuffles, the z faces land in the
// lane's own column ends and the x / y faces reach their owner columns with 4
// more shuffles.  No shared memory and no block barriers.
#ifndef LDG_P2W_MINB
#define LDG_P2W_MINB 4        // 64 registers: measured 49 us vs 71 us at 77 registers
#endif
#ifndef LDG_P2W_PIPE
#define LDG_P2W_PIPE 1
#endif
#ifndef LDG_P2W_MAXN1
#define LDG_P2W_MAXN1 5       // warp completion for hex p = 1..LDG_P2W_MAXN1-1 (N1^2 <= 32)
#endif
#ifndef LDG_P2W_GRID
#define LDG_P2W_GRID LDG_P2W_MINB   // blocks per SM in the grid
#endif
// hex p = 3 (N1 = 4): the hand-specialised variant (no spills; the generic
// template below spills 12 B at N1 = 4 and measured 44 vs 42 us)
__global__ void __launch_bounds__(256, LDG_P2W_MINB)
complete_warp4_kernel(const __grid_constant__ TensorParams P, const FaceRec* __restrict__ frec,
                     const double* __restrict__ X, double* __restrict__ R) {
  constexpr int NB = 64, NF = 16;
  const int lane = threadIdx.x & 31, half = lane >> 4, t = lane & 15;
  const int i = t & 3, j = t >> 2, hb = half * 16;
  double Mi[4], Mj[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    Mi[m] = P.m1[i * 4 + m];
    Mj[m] = P.m1[j * 4 + m];
  }
  const double wgt = P.grad_centered ? -0.5 : -1.0;
  const int nel = P.e1 - P.e0;
  const int npairs = (nel + 1) >> 1;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  // pairs in reverse order: pass 1 finished with the last elements (L2-resident)
  auto elem = [&](int w) { return P.e0 + (npairs - 1 - w) * 2 + half; };
  auto load_info = [&](int w) {
    const int e = elem(w);
    return (w < npairs && e < P.e1 && t < 6)
               ? __ldg(reinterpret_cast<const int*>(frec + (size_t)e * 6 + t) + 3) : 0;
  };
  int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
#if LDG_P2W_PIPE
  int info_next = load_info(w);                 // face records are static tables
#endif
  // programmatic dependent launch: everything above overlaps the tail of
  // pass 1; R and the exports are read only after pass 1 has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (; w < npairs; w += nwarps) {
    const int e = elem(w);
    const bool active = e < P.e1;
#if LDG_P2W_PIPE
    const int info = info_next;                              // loaded one pair ahead
    info_next = load_info(w + nwarps);
#else
    const int info = load_info(w);
#endif
    double r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) r[k] = active ? __ldg(R + (size_t)e * NB + t + 16 * k) : 0.0;
    const unsigned bal = __ballot_sync(0xffffffffu, (info & LDG_FL_COMPLETE) != 0);
    const unsigned any = (bal | (bal >> 16)) & 63;           // faces completed in either element
    const int mask = (bal >> hb) & 63;
    double x[6];
#pragma unroll
    for (int lf = 0; lf < 6; ++lf)
      x[lf] = (mask >> lf) & 1 ? __ldg(X + ((size_t)e * 6 + lf) * NF + t) : 0.0;
#pragma unroll
    for (int lf = 0; lf < 6; ++lf) {
      if (!((any >> lf) & 1)) continue;                      // warp-uniform
      const double v = wgt * x[lf];
      // w(a', b) = sum_a M[a'][a] v(a, b) on lane (a', b); L(a', b') = sum_b M[b'][b] w(a', b)
      double wv = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a) wv = fma(Mi[a], __shfl_sync(0xffffffffu, v, hb + a + 4 * j), wv);
      double L = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) L = fma(Mj[b], __shfl_sync(0xffffffffu, wv, hb + i + 4 * b), L);
      if (!((mask >> lf) & 1)) L = 0.0;
      if (lf == 0) r[0] += L;                                // z-: node (i, j, 0)
      else if (lf == 1) r[3] += L;                           // z+: node (i, j, 3)
      else {
        // y faces: node (i, 0|3, k) <- face node (i, k); x faces: node (0|3, j, k) <- (j, k)
        const bool own = lf == 2 ? j == 0 : (lf == 3 ? j == 3 : (lf == 4 ? i == 0 : i == 3));
        const int a0 = lf < 4 ? i : j;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double g = __shfl_sync(0xffffffffu, L, hb + a0 + 4 * k);
          if (own) r[k] += g;
        }
      }
    }
    if (active) {
      int hm = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        hm = max(hm, hi_abs(r[k]));
        R[(size_t)e * NB + t + 16 * k] = r[k];
      }
      bad_if_any(P, e, hm);
    }
  }
}

// generic p = 1, 2 (and any N1 with N1^2 <= 32)
template <int N1>
__global__ void __launch_bounds__(256, LDG_P2W_MINB)
complete_warp_kernel(const __grid_constant__ TensorParams P, const FaceRec* __restrict__ frec,
                     const double* __restrict__ X, double* __restrict__ R) {
  // EPW elements per warp, NF = N1^2 lanes each (p = 1..4); lanes past
  // EPW * NF only take part in the shuffles
  constexpr int NF = N1 * N1, NB = NF * N1, EPW = 32 / NF;
  constexpr bool FULL = EPW * NF == 32;                      // every lane owns a face node
  const int lane = threadIdx.x & 31, slot = lane / NF, t = lane - slot * NF;
  const int i = t % N1, j = t / N1, hb = slot * NF;
  const bool lane_ok = FULL || slot < EPW;
  auto src = [](int l) { return FULL ? l : (l & 31); };
  double Mi[N1], Mj[N1];
#pragma unroll
  for (int m = 0; m < N1; ++m) {
    Mi[m] = P.m1[i * N1 + m];
    Mj[m] = P.m1[j * N1 + m];
  }
  const double wgt = P.grad_centered ? -0.5 : -1.0;
  const int nel = P.e1 - P.e0;
  const int ngroups = (nel + EPW - 1) / EPW;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  // groups in reverse order: pass 1 finished with the last elements (L2-resident)
  auto elem = [&](int w) { return P.e0 + (ngroups - 1 - w) * EPW + slot; };
  // face lf's record is loaded by lane t = lf (NF >= 6) or t = lf - NF (second
  // load, p = 1 where NF = 4): the completion bits are two ballots
  auto load_info = [&](int w) {
    const int e = elem(w);
    const bool ok = lane_ok && w < ngroups && e < P.e1;
    int2 v = make_int2(0, 0);
    if (ok && t < 6) v.x = __ldg(reinterpret_cast<const int*>(frec + (size_t)e * 6 + t) + 3);
    if (NF < 6 && ok && t + NF < 6)
      v.y = __ldg(reinterpret_cast<const int*>(frec + (size_t)e * 6 + t + NF) + 3);
    return v;
  };
  int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
#if LDG_P2W_PIPE
  int2 info_next = load_info(w);
#endif
  for (; w < ngroups; w += nwarps) {
    const int e = elem(w);
    const bool active = lane_ok && e < P.e1;
#if LDG_P2W_PIPE
    const int2 info = info_next;                             // loaded one group ahead
    info_next = load_info(w + nwarps);
#else
    const int2 info = load_info(w);
#endif
    double r[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) r[k] = active ? __ldg(R + (size_t)e * NB + t + NF * k) : 0.0;
    const unsigned bal = __ballot_sync(0xffffffffu, (info.x & LDG_FL_COMPLETE) != 0);
    const unsigned bal2 = NF < 6 ? __ballot_sync(0xffffffffu, (info.y & LDG_FL_COMPLETE) != 0) : 0u;
    constexpr unsigned LO = NF < 6 ? (1u << NF) - 1u : 63u;
    auto face_mask = [&](int base) {
      return ((bal >> base) & LO) | (NF < 6 ? ((bal2 >> base) & ((1u << (6 - (NF < 6 ? NF : 0))) - 1u)) << NF : 0u);
    };
    unsigned any = 0;                                        // faces completed in any element
#pragma unroll
    for (int s2 = 0; s2 < EPW; ++s2) any |= face_mask(s2 * NF);
    const int mask = lane_ok ? (int)face_mask(hb) : 0;
    double x[6];
#pragma unroll
    for (int lf = 0; lf < 6; ++lf)
      x[lf] = (mask >> lf) & 1 ? __ldg(X + ((size_t)e * 6 + lf) * NF + t) : 0.0;
#pragma unroll
    for (int lf = 0; lf < 6; ++lf) {
      if (!((any >> lf) & 1)) continue;                      // warp-uniform
      const double v = wgt * x[lf];
      // w(a', b) = sum_a M[a'][a] v(a, b) on lane (a', b); L(a', b') = sum_b M[b'][b] w(a', b)
      double wv = 0.0;
#pragma unroll
      for (int a2 = 0; a2 < N1; ++a2) wv = fma(Mi[a2], __shfl_sync(0xffffffffu, v, src(hb + a2 + N1 * j)), wv);
      double L = 0.0;
#pragma unroll
      for (int b2 = 0; b2 < N1; ++b2) L = fma(Mj[b2], __shfl_sync(0xffffffffu, wv, src(hb + i + N1 * b2)), L);
      if (!((mask >> lf) & 1)) L = 0.0;
      if (lf == 0) r[0] += L;                                // z-: node (i, j, 0)
      else if (lf == 1) r[N1 - 1] += L;                      // z+: node (i, j, N1-1)
      else {
        // y faces: node (i, 0|N1-1, k) <- face node (i, k); x faces: (0|N1-1, j, k) <- (j, k)
        const bool own = lf == 2 ? j == 0 : (lf == 3 ? j == N1 - 1 : (lf == 4 ? i == 0 : i == N1 - 1));
        const int a0 = lf < 4 ? i : j;
#pragma unroll
        for (int k = 0; k < N1; ++k) {
          const double g = __shfl_sync(0xffffffffu, L, src(hb + a0 + N1 * k));
          if (own) r[k] += g;
        }
      }
    }
    if (active) {
      int hm = 0;
#pragma unroll
      for (int k = 0; k < N1; ++k) {
        hm = max(hm, hi_abs(r[k]));
        R[(size_t)e * NB + t + NF * k] = r[k];
      }
      bad_if_any(P, e, hm);
    }
  }
}

// --------------------------------------------------------------------------
// dispatch
// --------------------------------------------------------------------------

#ifndef LDG_P1_ELEM
#define LDG_P1_ELEM 0             // A/B: hex p = 1 thread-per-element pass 1 (measured 200 vs
#endif                            // 184 us for plane_kernel_g<2>: latency-bound on 12 B/DOF of
                                  // face records + 12 B/DOF of coefficient blocks)
#ifndef LDG_P2_ELEM1
#define LDG_P2_ELEM1 0            // A/B: hex p = 1 thread-per-element pass 2 (config 5 p = 1:
#endif                            // 37.7 vs 38.3 GDOF/s with complete_warp_kernel<2>)
static int launch_elem_p1(const TensorParams& P, bool tangent, const FaceRec* fr, const double* u,
                          const double* gproj, const double* bsrc, double* R, double* X,
                          cudaStream_t s) {
  const int nel = P.e1 - P.e0;
  const int grid = (nel + 127) / 128;
#define LDG_ELEM1(T, C, D) elem_kernel_p1<T, C, D><<<grid, 128, 0, s>>>(P, fr, u, gproj, bsrc, R, X)
  if (P.c_diag) {
    if (P.flux_uses_u) { if (tangent) LDG_ELEM1(true, true, true); else LDG_ELEM1(false, true, true); }
    else { if (tangent) LDG_ELEM1(true, false, true); else LDG_ELEM1(false, false, true); }
  } else {
    if (P.flux_uses_u) { if (tangent) LDG_ELEM1(true, true, false); else LDG_ELEM1(false, true, false); }
    else { if (tangent) LDG_ELEM1(true, false, false); else LDG_ELEM1(false, false, false); }
  }
#undef LDG_ELEM1
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

#ifndef LDG_PLANE_G5
#define LDG_PLANE_G5 0            // A/B: 5 = plane_kernel_g at hex p = 4 as well
#endif
// plane-mapped pass 1 at hex p = 1, 2: persistent grid of MINB blocks per SM
template <int N1>
static int launch_plane_g(const TensorParams& P, bool tangent, const FaceRec* fr, const double* u,
                          const double* gproj, const double* bsrc, double* R, double* X,
                          cudaStream_t s) {
  using G = PlaneG<N1>;
  static int nsm = 0;
  if (!nsm) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int nel = P.e1 - P.e0;
  const int groups = (nel + G::EPW - 1) / G::EPW;
  const int gp = std::max(1, std::min((groups + G::WPB - 1) / G::WPB, nsm * G::MINB));
  const int smem = G::WPB * G::WARP * (int)sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(plane_kernel_g<N1, true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel_g<N1, false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel_g<N1, true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel_g<N1, false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel_g<N1, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel_g<N1, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel_g<N1, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel_g<N1, false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
#define LDG_PLANE_G(T, C, D) \
  plane_kernel_g<N1, T, C, D><<<gp, G::WPB * 32, smem, s>>>(P, fr, u, gproj, bsrc, R, X)
  if (P.c_diag) {
    if (P.flux_uses_u) { if (tangent) LDG_PLANE_G(true, true, true); else LDG_PLANE_G(false, true, true); }
    else { if (tangent) LDG_PLANE_G(true, false, true); else LDG_PLANE_G(false, false, true); }
  } else {
    if (P.flux_uses_u) { if (tangent) LDG_PLANE_G(true, true, false); else LDG_PLANE_G(false, true, false); }
    else { if (tangent) LDG_PLANE_G(true, false, false); else LDG_PLANE_G(false, false, false); }
  }
#undef LDG_PLANE_G
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int N1, int ND, int NCU>
static int run_pass(const TensorParams& P, int pass, bool tangent, const double* u,
                    const double* gproj, const double* bsrc, double* R, double* X,
                    cudaStream_t s) {
  using S1 = P1Smem<N1, ND, NCU>;
  using S2 = P2Smem<N1, ND, NCU>;
  const int nel = P.e1 - P.e0;
  const int grid = (nel + S1::EPB - 1) / S1::EPB;
  const int grid2 = (nel + S2::EPB - 1) / S2::EPB;
  if (grid <= 0) return 0;
  if (pass & 1) {
    const FaceRec* fr = reinterpret_cast<const FaceRec*>(P.frec);
    if (N1 == 4 && ND == 3 && NCU == 1 && P.variant == 0) {
      static int nsm = 0;
      if (!nsm) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
      const int groups = (nel + 7) / 8;
      const int gp = std::max(1, std::min((groups + 3) / 4, nsm * LDG_PLANE_MINB));
      const int smem = (kPlaneBlock / 32) * kPlaneWarp * (int)sizeof(double);
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(plane_kernel<true, false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(plane_kernel<false, false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(plane_kernel<true, true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(plane_kernel<false, true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(plane_kernel<true, false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(plane_kernel<false, false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(plane_kernel<true, true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(plane_kernel<false, true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
      }
#define LDG_PLANE(T, C, D) plane_kernel<T, C, D, false><<<gp, kPlaneBlock, smem, s>>>(P, fr, u, gproj, bsrc, R, X)
      if (P.c_diag) {
        if (P.flux_uses_u) { if (tangent) LDG_PLANE(true, true, true); else LDG_PLANE(false, true, true); }
        else { if (tangent) LDG_PLANE(true, false, true); else LDG_PLANE(false, false, true); }
      } else {
        if (P.flux_uses_u) { if (tangent) LDG_PLANE(true, true, false); else LDG_PLANE(false, true, false); }
        else { if (tangent) LDG_PLANE(true, false, false); else LDG_PLANE(false, false, false); }
      }
#undef LDG_PLANE
      if (cudaGetLastError() != cudaSuccess) return 3;
    } else if constexpr ((N1 == 2 || N1 == 3 || N1 == LDG_PLANE_G5) && ND == 3 && NCU == 1) {
      if (P.variant == 0 && N1 == 2 && LDG_P1_ELEM) {
        if (int rc = launch_elem_p1(P, tangent, fr, u, gproj, bsrc, R, X, s)) return rc;
      } else if (P.variant == 0) {
        if (int rc = launch_plane_g<N1>(P, tangent, fr, u, gproj, bsrc, R, X, s)) return rc;
      } else if (tangent) fused_kernel<N1, ND, NCU, true><<<grid, kFBlock, 0, s>>>(P, fr, u, gproj, bsrc, R, X);
      else fused_kernel<N1, ND, NCU, false><<<grid, kFBlock, 0, s>>>(P, fr, u, gproj, bsrc, R, X);
    } else if (tangent) fused_kernel<N1, ND, NCU, true><<<grid, kFBlock, 0, s>>>(P, fr, u, gproj, bsrc, R, X);
    else fused_kernel<N1, ND, NCU, false><<<grid, kFBlock, 0, s>>>(P, fr, u, gproj, bsrc, R, X);
    if (cudaGetLastError() != cudaSuccess) return 3;
  }
  if (pass & 2) {
    static int nsm2 = 0;
    if (!nsm2) cudaDeviceGetAttribute(&nsm2, cudaDevAttrMultiProcessorCount, 0);
    const bool pipe = P.p2_mode != 3;                 // one-shot block kernel (A/B)
    bool done = false;
    const bool warp2 = P.p2_mode < 2;                 // block kernel (A/B)
    if constexpr (N1 == 2 && ND == 3 && NCU == 1 && LDG_P2_ELEM1) {
      if (P.x_consumer && P.p2_mode == 0) {
        complete_elem_p1<<<(nel + 255) / 256, 256, 0, s>>>(P, reinterpret_cast<const FaceRec*>(P.frec), X, R);
        done = true;
      }
    }
    if constexpr (N1 >= 2 && N1 <= LDG_P2W_MAXN1 && ND == 3 && NCU == 1) {
      if (!done && P.x_consumer && warp2) {
        constexpr int EPW = 32 / (N1 * N1);
        const int ngr = (nel + EPW - 1) / EPW;
        const int g = std::max(1, std::min((ngr + 7) / 8, nsm2 * LDG_P2W_GRID));
        if constexpr (N1 == 4) {
          const bool pdl = P.p2_mode == 0;
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(g);
          cfg.blockDim = dim3(256);
          cfg.dynamicSmemBytes = 0;
          cfg.stream = s;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          attr[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = attr;
          cfg.numAttrs = pdl ? 1 : 0;
          cudaLaunchKernelEx(&cfg, complete_warp4_kernel, P, reinterpret_cast<const FaceRec*>(P.frec),
                             (const double*)X, R);
        }
        else
          complete_warp_kernel<N1><<<g, 256, 0, s>>>(P, reinterpret_cast<const FaceRec*>(P.frec), X, R);
        done = true;
      }
    }
    // register-pipelined pass 2 (64 registers): measured faster for p <= 2
    // (config 5: p=1 23.0 -> 23.4, p=2 27.6 -> 29.0 GDOF/s), slower for p = 4, 5
    if constexpr (NCU == 1 && N1 <= 3) {
      if (!done && P.x_consumer && pipe) {
        complete_pipe_kernel<N1, ND, NCU><<<std::min(grid2, nsm2 * LDG_P2P_MINB), kFBlock, 0, s>>>(
            P, reinterpret_cast<const FaceRec*>(P.frec), X, R);
        done = true;
      }
    }
    if (!done)
      complete_kernel<N1, ND, NCU><<<grid2, kFBlock, 0, s>>>(
          P, reinterpret_cast<const FaceRec*>(P.frec), X, R);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// Full operator.  With P.nchunk > 1 the element range is cut into chunks and
// the two passes interleave, P1(0) P1(1) P2(0) P1(2) P2(1) ...: pass 2 of a
// chunk runs as soon as pass 1 of every chunk it reads exports from is done
// (chunk_dep, computed from the face table at ldg_create), while that
// chunk's R rows and exports are still resident in L2, so pass 2 costs L2
// rather than HBM traffic.
// One-launch operator (hex p = 3, ncu = 1): plane_kernel<.., FUSED> runs pass 1
// and, as the pass-1 windows it reads complete, pass 2 of each group, so the R
// rows and exports pass 2 re-reads come from L2 instead of HBM.
static int launch_plane_fused(const TensorParams& P, bool tangent, const double* u,
                              const double* gproj, const double* bsrc, double* R, double* X,
                              cudaStream_t s) {
  static int nsm = 0;
  if (!nsm) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int groups = (P.e1 - P.e0 + 7) / 8;
  const int gp = std::max(1, std::min((groups + 3) / 4, nsm * LDG_PLANE_MINB));
  const int smem = (kPlaneBlock / 32) * kPlaneWarp * (int)sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(plane_kernel<true, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel<false, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel<true, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel<false, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel<true, false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel<false, false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel<true, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(plane_kernel<false, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const FaceRec* fr = reinterpret_cast<const FaceRec*>(P.frec);
#define LDG_PLANE_F(T, C, D) plane_kernel<T, C, D, true><<<gp, kPlaneBlock, smem, s>>>(P, fr, u, gproj, bsrc, R, X)
  if (P.c_diag) {
    if (P.flux_uses_u) { if (tangent) LDG_PLANE_F(true, true, true); else LDG_PLANE_F(false, true, true); }
    else { if (tangent) LDG_PLANE_F(true, false, true); else LDG_PLANE_F(false, false, true); }
  } else {
    if (P.flux_uses_u) { if (tangent) LDG_PLANE_F(true, true, false); else LDG_PLANE_F(false, true, false); }
    else { if (tangent) LDG_PLANE_F(true, false, false); else LDG_PLANE_F(false, false, false); }
  }
#undef LDG_PLANE_F
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int N1, int ND, int NCU>
static int run_fused(const TensorParams& P, bool tangent, const double* u,
                     const double* gproj, const double* bsrc, double* R, double* X,
                     cudaStream_t s) {
  if constexpr (N1 == 4 && ND == 3 && NCU == 1) {
    if (P.fused && P.fuse && P.nchunk <= 1 && P.e0 == 0 && P.e1 == P.ne && P.ghost0 == INT32_MAX &&
        P.x_consumer && P.p2_mode == 0 && P.variant == 0)
      return launch_plane_fused(P, tangent, u, gproj, bsrc, R, X, s);
  }
  if (P.nchunk <= 1) return run_pass<N1, ND, NCU>(P, 3, tangent, u, gproj, bsrc, R, X, s);
  // pass 2 chunks go to a side stream so they overlap the next pass-1 chunk
  // (fork / join with events: also valid under CUDA graph capture)
  static cudaStream_t side = nullptr;
  static cudaEvent_t ev[LDG_MAX_CHUNKS + 2];
  if (!side) {
    if (cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess) return 3;
    for (auto& x : ev) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  }
  cudaEventRecord(ev[LDG_MAX_CHUNKS + 1], s);
  cudaStreamWaitEvent(side, ev[LDG_MAX_CHUNKS + 1], 0);       // fork
  TensorParams Q = P;
  for (int c = 0; c < P.nchunk; ++c) {
    Q.e0 = P.chunk_start[c];
    Q.e1 = P.chunk_start[c + 1];
    if (int rc = run_pass<N1, ND, NCU>(Q, 1, tangent, u, gproj, bsrc, R, X, s)) return rc;
    cudaEventRecord(ev[c], s);
    bool waited = false;
    for (int d = 0; d < P.nchunk; ++d) {
      if (P.chunk_dep[d] != c) continue;
      if (!waited) {
        cudaStreamWaitEvent(side, ev[c], 0);
        waited = true;
      }
      Q.e0 = P.chunk_start[d];
      Q.e1 = P.chunk_start[d + 1];
      if (int rc = run_pass<N1, ND, NCU>(Q, 2, tangent, u, gproj, bsrc, R, X, side)) return rc;
    }
  }
  cudaEventRecord(ev[LDG_MAX_CHUNKS], side);
  cudaStreamWaitEvent(s, ev[LDG_MAX_CHUNKS], 0);               // join
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
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
