// Kernel template of the generated (model-specific) LDG path, compiled at
// run time by NVRTC for sm_100a (csrc/jit.cu).  NOT compiled by nvcc: the
// Python side (paper_2205_07824_b200/nonlinear.py) prepends a prelude with
//   * the compile-time shape: ND, N1 (nodes / direction), NQ1 (Gauss points /
//     direction), NCU, NW (ODE states), KIND_C, KIND_W, HAS_WS,
//     TRACE_CENTERED, GRAD_CENTERED, MASS_CONST, NT (threads per element),
//     ODE_ALPHA / ODE_BETA;
//   * __constant__ 1D operators c_phi / c_dphi (NQ1 x N1, l_a(x_q)),
//     c_d1 (GLL collocation derivative), c_clo / c_chi (M1^-1 e_0, e_p),
//     c_m1inv, c_xq1 (1D Gauss points), c_qw (volume weights), c_fxi / c_fw
//     (face-point reference coordinates and weights, matched to the
//     reference's face rules), c_mass (constant mass coefficients);
//   * the model's plans as device functions plan_flux / plan_src /
//     plan_ws / plan_mass / plan_sw (+ _d dual variants), emitted by codegen.py;
//   * c_xn: reference coordinates of the solution nodes (ODE collocation);
// and then this file.
//
// Algorithm: the reference's quadrature formulation (disc.py:595-893) per
// element, with the dense tables replaced by tensor contractions:
//   nl_mixed     q = M^-1 [-int grad(u) phi + oint (u - u^) n phi]   disc.py:436-490
//                (GLL collocation: exact for affine elements, as in ldg_tensor.cu)
//   nl_residual  R = -int f(u,q) . grad(phi) - int s phi + oint f^ phi disc.py:595-653
//   nl_tangent   the reference linearisation of R (frozen tau, LLF dlam tie
//                rule, homogeneous lift, zero Neumann tangent)       disc.py:657-862
//   nl_mass      int m(u) v phi  (and the (dm/du du) y extra term)   disc.py:897-948
//   nl_mass_inv  M^-1 v = detJ^-1 (M1^-1)^(x)nd v                    driver.py:92-106
// Interior faces are visited from both elements (element-centric: no scatter,
// no atomics); both sides evaluate the numerical flux in the LEFT element's
// frame (left normal, left = u^-), so the two contributions are bitwise
// negatives of each other exactly as the reference's scatter of +/- vals.

typedef unsigned long long u64;
typedef unsigned long long sz_t;  // (no <cstddef> under NVRTC)

constexpr int NB = ND == 3 ? N1 * N1 * N1 : (ND == 2 ? N1 * N1 : N1);
constexpr int NQ = ND == 3 ? NQ1 * NQ1 * NQ1 : (ND == 2 ? NQ1 * NQ1 : NQ1);
constexpr int NFN = ND == 3 ? N1 * N1 : (ND == 2 ? N1 : 1);   // a 1D face is one point
constexpr int NQF = ND == 3 ? NQ1 * NQ1 : (ND == 2 ? NQ1 : 1);
constexpr int NFACE = 2 * ND;
#ifndef NL_FB
#define NL_FB NFACE
#endif
#ifndef NL_LOAD_BATCH
#define NL_LOAD_BATCH 1
#endif
constexpr int NFB = NL_FB;                     // faces per batch of the face phase (divides NFACE)
static_assert(NFACE % NFB == 0, "face batch");
constexpr int NVQ = KIND_C ? 0 : NCU * ND;
constexpr int NV = NCU + NVQ + NW;             // state variables per point (u, q, w)
constexpr int OW = NCU + NVQ;                  // offset of w within a point's variables
constexpr int KMAX = N1 > NQ1 ? N1 : NQ1;
constexpr int MX = ND == 3 ? KMAX * KMAX * KMAX : (ND == 2 ? KMAX * KMAX : KMAX);
constexpr int MXF = ND == 3 ? KMAX * KMAX : (ND == 2 ? KMAX : 1);
constexpr int NG = NCU * (ND + 1);             // G_r (r < ND) and the source field

struct NlParams {
  int ne, nbface;
  double t, scale;
  const double* geo;     // (ne, 1 + ND*ND): detJ, invjt[d][r]
  const double* xmap;    // (ne, ND + ND*ND): x0, J[d][r] with x = x0 + J xi
  const int* fnbr;       // (ne, NFACE) neighbour element / boundary-face row
  const int* finfo;      // (ne, NFACE) kind | right<<2 | switch<<3 | map<<8
  const double* fgeo;    // (ne, NFACE, ND + 2): left normal, left |t1 x t2|, tau/h
  const int* nmap;       // (n_maps, NFN) own face node -> neighbour volume node
  const double* gq;      // (nbface, NQF, NCU) boundary data at face points
  const double* gproj;   // (nbface, NFN, NCU) projected Dirichlet data (mixed lift)
  const double* u;       // base state (ne, NB, NCU)
  const double* q;       // base mixed gradient (ne, NB, NCU, ND) / mass operand v
  const double* du;      // direction
  const double* dq;      // direction gradient (homogeneous lift of du)
  const double* w;       // ODE states (ne, NB, NW)
  const double* dw;
  double* out;
  u64* bad;              // [0]: first element with a non-finite plan value
  int homog;             // nl_mixed: 1 = dual of a u^ override (kind-W tangent lift)
  int pad_;
  // CURVED (non-affine elements, disc.py:91-180 per-point geometry):
  const double* vgeo;    // (ne, NQ, 1 + ND*ND + ND): detJ, invjt[d][r], x at the volume points
  const double* ffgeo;   // (ne, NFACE, NQF, 2 ND + 1): left normal, w |t1 x t2|, x per face point
  const double* minv;    // (ne, NB, NB) inverse element mass matrices
  // base-state cache of the tangent (built once per base by nl_base_cache):
  // [ne][NV][NQ] volume-point values, then [ne][side][face][NV][NQF] traces
  double* bcache;
};
#ifndef CURVED
#define CURVED 0
#endif
constexpr int VG = 1 + ND * ND + ND;           // vgeo entries per volume point
constexpr int FG = 2 * ND + 1;                 // ffgeo entries per face point

__device__ __forceinline__ bool fin(double v) { return v - v == 0.0; }
// (ldg_sign / ldg_min / ldg_max, used by the plans, come with the prelude)
__device__ __forceinline__ void flag(const NlParams& P, int e, double v) {
  if (!fin(v)) atomicMin(P.bad, (u64)e);
}

// hex local faces z-, z+, y-, y+, x-, x+; quad y-, x+, y+, x- (master.py:43-44)
__device__ __forceinline__ int face_axis(int lf) {
  return ND == 3 ? (lf < 2 ? 2 : (lf < 4 ? 1 : 0)) : (ND == 2 ? ((lf == 0 || lf == 2) ? 1 : 0) : 0);
}
__device__ __forceinline__ int face_side(int lf) {
  return ND == 3 ? (lf & 1) : (ND == 2 ? (lf == 1 || lf == 2 ? 1 : 0) : lf);
}
// volume node of face node t (t = i_a0 + N1 i_a1 over the tangential axes a0 < a1)
__device__ __forceinline__ int face_vol_node(int lf, int t) {
  const int ax = face_axis(lf);
  const int io = face_side(lf) ? N1 - 1 : 0;
  if (ND == 1) return io;
  if (ND == 2) return ax == 0 ? io + N1 * t : t + N1 * io;
  const int a = t % N1, b = t / N1;
  if (ax == 0) return io + N1 * a + N1 * N1 * b;
  if (ax == 1) return a + N1 * io + N1 * N1 * b;
  return a + N1 * b + N1 * N1 * io;
}

// ---------------------------------------------------------------------------
// block-cooperative 1D contraction along one axis of a (D0 x D1 x D2) grid
// (D0 fastest) for NVAR variables stored [v][grid]:
//   out[v][.., o, ..] = sum_i M(o, i) in[v][.., i, ..]
// M(o, i) = op[o * N1 + i] (interpolation, rows = outputs) or, with TRANS,
// op[i * N1 + o] (the transpose: quadrature -> nodes); the operator (phi,
// dphi or M1^-1) is a template parameter, so its entries are constant-bank
// operands.
// ---------------------------------------------------------------------------
enum { OP_PHI = 0, OP_DPHI = 1, OP_M1INV = 2 };
template <int OPID>
__device__ __forceinline__ double op_c(int k) {
  return OPID == OP_PHI ? c_phi[k] : (OPID == OP_DPHI ? c_dphi[k] : c_m1inv[k]);
}

template <int D0, int D1, int D2, int AX, int NIN, int NOUT, bool TRANS, int OPID>
__device__ __forceinline__ void contract_u(const double* __restrict__ in, double* __restrict__ out,
                                           int nvar, int tid) {
  // one thread per pencil along AX: its NIN inputs are read once, all NOUT
  // outputs formed with compile-time (warp-uniform) operator entries
  constexpr int O0 = AX == 0 ? NOUT : D0, O1 = AX == 1 ? NOUT : D1, O2 = AX == 2 ? NOUT : D2;
  constexpr int I0 = AX == 0 ? NIN : D0, I1 = AX == 1 ? NIN : D1, I2 = AX == 2 ? NIN : D2;
  constexpr int OSZ = O0 * O1 * O2, ISZ = I0 * I1 * I2;
  constexpr int P0 = AX == 0 ? 1 : D0, P1 = AX == 1 ? 1 : D1, P2 = AX == 2 ? 1 : D2;
  constexpr int NPN = P0 * P1 * P2;
  constexpr int ISTR = AX == 0 ? 1 : (AX == 1 ? I0 : I0 * I1);
  constexpr int OSTR = AX == 0 ? 1 : (AX == 1 ? O0 : O0 * O1);
  (void)I2;
  (void)O2;
  // x-axis pencils sit NIN (NOUT) doubles apart, so with an even length the
  // lanes of a warp hit the same banks (4-way at 4): those reads / writes are
  // issued in a lane-rotated order (rotation s = (lane / G) mod len, G =
  // 16 / gcd(len, 16)) and put back in registers with selects -- 2 shared
  // wavefronts per 256 B instead of 8; the arithmetic order is unchanged
  constexpr bool SKEW_IN = AX == 0 && NIN % 2 == 0;
  constexpr bool SKEW_OUT = AX == 0 && NOUT % 2 == 0;
  constexpr int GIN = NIN % 8 == 0 ? 2 : (NIN % 4 == 0 ? 4 : 8);
  constexpr int GOUT = NOUT % 8 == 0 ? 2 : (NOUT % 4 == 0 ? 4 : 8);
  const int total = nvar * NPN;
  for (int idx = tid; idx < total; idx += NT) {
    const int v = idx / NPN, r = idx - v * NPN;
    const int p0 = r % P0, p1 = (r / P0) % P1, p2 = r / (P0 * P1);
    const int ib = v * ISZ + p0 + p1 * I0 + p2 * I0 * I1;
    const int ob = v * OSZ + p0 + p1 * O0 + p2 * O0 * O1;
    double x[NIN];
    if (SKEW_IN) {
      const int sh = ((idx & 31) / GIN) % NIN;
      double rr[NIN];
#pragma unroll
      for (int j = 0; j < NIN; ++j) {
        int jj = j + sh;
        if (jj >= NIN) jj -= NIN;
        rr[j] = in[ib + jj];
      }
#pragma unroll
      for (int i = 0; i < NIN; ++i) {
        double val = rr[i];
#pragma unroll
        for (int k = 1; k < NIN; ++k)
          if (sh == k) val = rr[(i - k + NIN) % NIN];
        x[i] = val;
      }
    } else {
#pragma unroll
      for (int i = 0; i < NIN; ++i) x[i] = in[ib + i * ISTR];
    }
    double y[NOUT];
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < NIN; ++i) acc = fma(op_c<OPID>(TRANS ? i * N1 + o : o * N1 + i), x[i], acc);
      y[o] = acc;
    }
    if (SKEW_OUT) {
      const int sh = ((idx & 31) / GOUT) % NOUT;
#pragma unroll
      for (int j = 0; j < NOUT; ++j) {
        int jj = j + sh;
        if (jj >= NOUT) jj -= NOUT;
        double val = y[j];
#pragma unroll
        for (int k = 1; k < NOUT; ++k)
          if (sh == k) val = y[(j + k) % NOUT];
        out[ob + jj] = val;
      }
    } else {
#pragma unroll
      for (int o = 0; o < NOUT; ++o) out[ob + o * OSTR] = y[o];
    }
  }
}

// nodes -> volume quadrature points (all variables, operator phi)
__device__ __forceinline__ void to_quad(double* a, double* b, int nvar, int tid, double*& res) {
  if (ND == 3) {
    contract_u<N1, N1, N1, 0, N1, NQ1, false, OP_PHI>(a, b, nvar, tid);
    __syncthreads();
    contract_u<NQ1, N1, N1, 1, N1, NQ1, false, OP_PHI>(b, a, nvar, tid);
    __syncthreads();
    contract_u<NQ1, NQ1, N1, 2, N1, NQ1, false, OP_PHI>(a, b, nvar, tid);
    __syncthreads();
    res = b;
  } else if (ND == 2) {
    contract_u<N1, N1, 1, 0, N1, NQ1, false, OP_PHI>(a, b, nvar, tid);
    __syncthreads();
    contract_u<NQ1, N1, 1, 1, N1, NQ1, false, OP_PHI>(b, a, nvar, tid);
    __syncthreads();
    res = a;
  } else {
    contract_u<N1, 1, 1, 0, N1, NQ1, false, OP_PHI>(a, b, nvar, tid);
    __syncthreads();
    res = b;
  }
}

// quadrature fields [r][c] (r < ND: G_r, r = ND: source) -> nodes, applying
// dphi^T along direction r and phi^T elsewhere (the transposed volume rule)
// one transposed stage along axis AX over fields [r][c] (r = 0..ND): the
// NCU fields of direction r == AX take dphi^T, the others phi^T
template <int D0, int D1, int D2, int AX>
__device__ __forceinline__ void from_quad_stage(const double* in, double* out, int nfield, int tid) {
  constexpr int I0 = AX == 0 ? NQ1 : D0, I1 = AX == 1 ? NQ1 : D1, I2 = AX == 2 ? NQ1 : D2;
  constexpr int O0 = AX == 0 ? N1 : D0, O1 = AX == 1 ? N1 : D1, O2 = AX == 2 ? N1 : D2;
  constexpr int ISZ = I0 * I1 * I2, OSZ = O0 * O1 * O2;
  const int lo = AX * NCU, hi = lo + NCU;
  if (lo > 0) contract_u<D0, D1, D2, AX, NQ1, N1, true, OP_PHI>(in, out, lo, tid);
  contract_u<D0, D1, D2, AX, NQ1, N1, true, OP_DPHI>(in + lo * ISZ, out + lo * OSZ, NCU, tid);
  if (nfield > hi)
    contract_u<D0, D1, D2, AX, NQ1, N1, true, OP_PHI>(in + hi * ISZ, out + hi * OSZ, nfield - hi, tid);
}

// quadrature fields [r][c] (r < ND: G_r, r = ND: source) -> nodes, applying
// dphi^T along direction r and phi^T elsewhere (the transposed volume rule)
__device__ __forceinline__ void from_quad(double* a, double* b, int nfield, int tid, double*& res) {
  if (ND == 3) {
    from_quad_stage<NQ1, NQ1, NQ1, 0>(a, b, nfield, tid);
    __syncthreads();
    from_quad_stage<N1, NQ1, NQ1, 1>(b, a, nfield, tid);
    __syncthreads();
    from_quad_stage<N1, N1, NQ1, 2>(a, b, nfield, tid);
    __syncthreads();
    res = b;
  } else if (ND == 2) {
    from_quad_stage<NQ1, NQ1, 1, 0>(a, b, nfield, tid);
    __syncthreads();
    from_quad_stage<N1, NQ1, 1, 1>(b, a, nfield, tid);
    __syncthreads();
    res = a;
  } else {
    from_quad_stage<NQ1, 1, 1, 0>(a, b, nfield, tid);
    __syncthreads();
    res = b;
  }
}

__device__ __forceinline__ void quad_point(int p, double* xi) {
  xi[0] = c_xq1[p % NQ1];
  if (ND >= 2) xi[ND >= 2 ? 1 : 0] = c_xq1[(p / NQ1) % NQ1];
  if (ND == 3) xi[ND == 3 ? 2 : 0] = c_xq1[p / (NQ1 * NQ1)];
}

__device__ __forceinline__ void phys_point(const NlParams& P, int e, const double* xi, double* x) {
  const double* m = P.xmap + (sz_t)e * (ND + ND * ND);
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    double a = m[d];
#pragma unroll
    for (int r = 0; r < ND; ++r) a = fma(m[ND + d * ND + r], xi[r], a);
    x[d] = a;
  }
}

// global value of state variable v (u components, then q components) of the
// array family `arr` (0: base u/q, 1: direction du/dq) at (element, node)
__device__ __forceinline__ double state_at(const NlParams& P, int fam, int v, sz_t e, int node) {
  if (v < NCU) return (fam ? P.du : P.u)[(e * NB + node) * NCU + v];
  if (v < OW) return (fam ? P.dq : P.q)[(e * NB + node) * (NCU * ND) + (v - NCU)];
  return (fam ? P.dw : P.w)[(e * NB + node) * (NW > 0 ? NW : 1) + (v - OW)];
}

__device__ __forceinline__ const double* state_ptr(const NlParams& P, int fam, int v, sz_t e,
                                                   int node) {
  if (v < NCU) return (fam ? P.du : P.u) + (e * NB + node) * NCU + v;
  if (v < OW) return (fam ? P.dq : P.q) + (e * NB + node) * (NCU * ND) + (v - NCU);
  return (fam ? P.dw : P.w) + (e * NB + node) * (NW > 0 ? NW : 1) + (v - OW);
}
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// mixed gradient (kind D): one thread per node, EPBM elements per block
// ---------------------------------------------------------------------------
constexpr int EPBM = NB >= 128 ? 1 : 128 / NB;

extern "C" __global__ void __launch_bounds__(EPBM * NB > 32 ? EPBM * NB : 32)
nl_mixed(const __grid_constant__ NlParams P) {
  __shared__ double su[EPBM][NCU][NB];
  __shared__ double sj[EPBM][NFACE][NFN][NCU];
  const int slot = threadIdx.x / NB, a = threadIdx.x % NB;
  const int e = blockIdx.x * EPBM + slot;
  const bool active = slot < EPBM && e < P.ne;
  if (active)
    for (int c = 0; c < NCU; ++c) su[slot][c][a] = P.u[((sz_t)e * NB + a) * NCU + c];
  __syncthreads();
  if (active) {
    for (int idx = a; idx < NFACE * NFN; idx += NB) {
      const int lf = idx / NFN, t = idx % NFN;
      const int info = P.finfo[e * NFACE + lf], nbr = P.fnbr[e * NFACE + lf];
      const int kind = info & 3;
      const int vn = face_vol_node(lf, t);
      for (int c = 0; c < NCU; ++c) {
        const double own = su[slot][c][vn];
        double jump = 0.0;
        if (kind == 0 && HAS_UHAT) {
          // user u^ (affine in the traces, checked at setup), evaluated at
          // the face nodes.  compute_mixed(du) evaluates it on du like on u
          // (disc.py:446-449 -> 496-504); the kind-W tangent lift takes its
          // dual, i.e. drops the constant part (P.homog)
          double ul[NCU], ur[NCU], uh[NCU], u0[NCU], zr[NCU];
          const bool right = info & 4;
          const int nn = P.nmap[(info >> 8) * NFN + t];
#pragma unroll
          for (int k = 0; k < NCU; ++k) {
            const double o = su[slot][k][vn], b = P.u[((sz_t)nbr * NB + nn) * NCU + k];
            ul[k] = right ? b : o;
            ur[k] = right ? o : b;
            zr[k] = 0.0;
          }
          plan_uhat(nullptr, P.t, ul, ur, nullptr, nullptr, nullptr, uh);
          if (P.homog) {
            plan_uhat(nullptr, P.t, zr, zr, nullptr, nullptr, nullptr, u0);
#pragma unroll
            for (int k = 0; k < NCU; ++k) uh[k] -= u0[k];
          }
          jump = own - uh[c];
        } else if (kind == 0) {
          const bool right = info & 4, sw = info & 8;
          const bool own_hat = !TRACE_CENTERED && (sw != right);   // u^ = own trace
          if (!own_hat) {
            const int nn = P.nmap[(info >> 8) * NFN + t];
            const double other = P.u[((sz_t)nbr * NB + nn) * NCU + c];
            jump = TRACE_CENTERED ? 0.5 * (own - other) : own - other;
          }
        } else if (kind == 1) {
          jump = own - (P.gproj ? P.gproj[((sz_t)nbr * NFN + t) * NCU + c] : 0.0);
        } else if (kind == 3) {
          // absorbing (kind W): u^ = (u + c q.n)/2 with the state gradient P.q
          // (its direction dq in the tangent: the form is linear), c the
          // state-independent wavespeed (disc.py:566-572)
          const double* fg = P.fgeo + ((sz_t)e * NFACE + lf) * (ND + 2);
          double wsc;
          plan_ws(nullptr, P.t, nullptr, nullptr, nullptr, fg, &wsc);
          double qn = 0.0;
#pragma unroll
          for (int d = 0; d < ND; ++d) qn += P.q[(((sz_t)e * NB + vn) * NCU + c) * ND + d] * fg[d];
          jump = own - 0.5 * (own + wsc * qn);
        }
        sj[slot][lf][t][c] = jump;
      }
    }
  }
  __syncthreads();
  if (!active) return;
  const double* g = P.geo + (sz_t)e * (1 + ND * ND);
  const int i = a % N1, j = (a / N1) % N1, k = ND == 3 ? a / (N1 * N1) : 0;
  const int ix[3] = {i, j, k};
  for (int c = 0; c < NCU; ++c) {
    double gr[ND];
#pragma unroll
    for (int r = 0; r < ND; ++r) {
      double acc = 0.0;
      const int st = r == 0 ? 1 : (r == 1 ? N1 : N1 * N1);
      const int b0 = a - ix[r] * st;
#pragma unroll
      for (int m = 0; m < N1; ++m) acc = fma(c_d1[ix[r] * N1 + m], su[slot][c][b0 + m * st], acc);
      gr[r] = acc;
    }
    double qd[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < ND; ++r) acc = fma(g[1 + d * ND + r], gr[r], acc);
      qd[d] = -acc;
    }
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const int ax = face_axis(lf);
      const bool hi = face_side(lf);
      const int nidx = ix[ax];
      int t;
      if (ND == 3) t = ax == 0 ? j + N1 * k : (ax == 1 ? i + N1 * k : i + N1 * j);
      else if (ND == 2) t = ax == 0 ? j : i;
      else t = 0;
      const double cf = hi ? c_chi[nidx] : c_clo[nidx];
      const double v = (hi ? cf : -cf) * sj[slot][lf][t][c];
#pragma unroll
      for (int d = 0; d < ND; ++d) qd[d] = fma(v, g[1 + d * ND + ax], qd[d]);
    }
#pragma unroll
    for (int d = 0; d < ND; ++d) P.out[(((sz_t)e * NB + a) * NCU + c) * ND + d] = qd[d];
  }
}

// ---------------------------------------------------------------------------
// mixed gradient on CURVED elements (kind D): the reference's quadrature
// form (disc.py:436-490) -- the GLL collocation identities of nl_mixed need
// affine elements:
//   rhs_a[i][j] = -sum_q w detJ (invJ^T grad u_i)_j phi_a
//                 + sum_faces sum_s wsj (u_i - u^_i) n_j phi_a,   q = M_e^-1 rhs
// one element per block; u^ by the trace rules at the face points (switch /
// centered, Dirichlet data at the face points, Neumann u^ = u).
// ---------------------------------------------------------------------------
constexpr int NGQ = NCU * ND;                  // gradient fields [c][j]
constexpr int MCS_BUF = (NGQ > NCU ? NGQ : NCU) * MX;
constexpr int MCS_SMEM = NCU * NB + 3 * MCS_BUF + NGQ * NB + 2 * NFACE * NCU * NQF +
                         4 * NCU * MXF + NFACE * NQF * NGQ;

template <int R>
__device__ __forceinline__ void grad_dir(const double* su, double* a, double* b, double* out,
                                         int tid) {
  // d/dxi_R at the volume points: dphi along R, phi along the other axes
  if (ND == 3) {
    contract_u<N1, N1, N1, 0, N1, NQ1, false, R == 0 ? OP_DPHI : OP_PHI>(su, a, NCU, tid);
    __syncthreads();
    contract_u<NQ1, N1, N1, 1, N1, NQ1, false, R == 1 ? OP_DPHI : OP_PHI>(a, b, NCU, tid);
    __syncthreads();
    contract_u<NQ1, NQ1, N1, 2, N1, NQ1, false, R == 2 ? OP_DPHI : OP_PHI>(b, out, NCU, tid);
  } else if (ND == 2) {
    contract_u<N1, N1, 1, 0, N1, NQ1, false, R == 0 ? OP_DPHI : OP_PHI>(su, a, NCU, tid);
    __syncthreads();
    contract_u<NQ1, N1, 1, 1, N1, NQ1, false, R == 1 ? OP_DPHI : OP_PHI>(a, out, NCU, tid);
  } else {
    contract_u<N1, 1, 1, 0, N1, NQ1, false, R == 0 ? OP_DPHI : OP_PHI>(su, out, NCU, tid);
  }
  __syncthreads();
}

extern "C" __global__ void __launch_bounds__(NT) nl_mixed_curved(const __grid_constant__ NlParams P) {
  extern __shared__ __align__(16) double smc[];
  double* su = smc;                            // [c][node]
  double* bA = su + NCU * NB;
  double* bB = bA + MCS_BUF;
  double* G = bB + MCS_BUF;                    // [r][c][q] reference derivatives, then fields
  double* rhs = G + MCS_BUF;                   // [c j][node]
  double* TR = rhs + NGQ * NB;                 // [side][face][c][NQF]
  double* FN = TR + 2 * NFACE * NCU * NQF;     // face nodes own | nbr [c][NFN], stage scratch
  double* FJ = FN + 4 * NCU * MXF;             // [face][s][c j]
  const int e = blockIdx.x, tid = threadIdx.x;
  if (e >= P.ne) return;
  for (int idx = tid; idx < NCU * NB; idx += NT) {
    const int c = idx / NB, a = idx % NB;
    su[idx] = P.u[((sz_t)e * NB + a) * NCU + c];
  }
  __syncthreads();
  // ---- volume: grad u at the points, -w detJ invJ^T grad u, phi^T back
  grad_dir<0>(su, bA, bB, G + 0 * NCU * NQ, tid);
  grad_dir<1>(su, bA, bB, G + 1 * NCU * NQ, tid);
  if (ND == 3) grad_dir<2>(su, bA, bB, G + 2 * NCU * NQ, tid);
  for (int p = tid; p < NQ; p += NT) {
    const double* gp = P.vgeo + ((sz_t)e * NQ + p) * VG;
    const double wd = c_qw[p] * gp[0];
    double gr[ND][NCU];
#pragma unroll
    for (int r = 0; r < ND; ++r)
#pragma unroll
      for (int c = 0; c < NCU; ++c) gr[r][c] = G[(r * NCU + c) * NQ + p];
#pragma unroll
    for (int c = 0; c < NCU; ++c)
#pragma unroll
      for (int j = 0; j < ND; ++j) {
        double a = 0.0;
#pragma unroll
        for (int r = 0; r < ND; ++r) a = fma(gp[1 + j * ND + r], gr[r][c], a);
        bA[(c * ND + j) * NQ + p] = -wd * a;
      }
  }
  __syncthreads();
  {
    double* res;
    if (ND == 3) {
      contract_u<NQ1, NQ1, NQ1, 0, NQ1, N1, true, OP_PHI>(bA, bB, NGQ, tid);
      __syncthreads();
      contract_u<N1, NQ1, NQ1, 1, NQ1, N1, true, OP_PHI>(bB, bA, NGQ, tid);
      __syncthreads();
      contract_u<N1, N1, NQ1, 2, NQ1, N1, true, OP_PHI>(bA, bB, NGQ, tid);
      res = bB;
    } else {
      contract_u<NQ1, NQ1, 1, 0, NQ1, N1, true, OP_PHI>(bA, bB, NGQ, tid);
      __syncthreads();
      contract_u<N1, NQ1, 1, 1, NQ1, N1, true, OP_PHI>(bB, bA, NGQ, tid);
      res = bA;
    }
    __syncthreads();
    for (int idx = tid; idx < NGQ * NB; idx += NT) rhs[idx] = res[idx];
  }
  // ---- faces: own / neighbour traces at the face points
  for (int lf = 0; lf < NFACE; ++lf) {
    const int info = P.finfo[e * NFACE + lf];
    const bool interior = (info & 3) == 0;
    const int nbr = P.fnbr[e * NFACE + lf];
    double* own = FN;
    double* oth = FN + NCU * MXF;
    double* st = FN + 2 * NCU * MXF;
    for (int idx = tid; idx < NCU * NFN; idx += NT) {
      const int c = idx / NFN, t = idx % NFN;
      own[idx] = su[c * NB + face_vol_node(lf, t)];
      oth[idx] = interior ? P.u[((sz_t)nbr * NB + P.nmap[(info >> 8) * NFN + t]) * NCU + c] : 0.0;
    }
    __syncthreads();
    double* tro = TR + (0 * NFACE + lf) * NCU * NQF;
    double* trn = TR + (1 * NFACE + lf) * NCU * NQF;
    if (ND == 3) {
      contract_u<N1, N1, 1, 0, N1, NQ1, false, OP_PHI>(own, st, NCU, tid);
      contract_u<N1, N1, 1, 0, N1, NQ1, false, OP_PHI>(oth, st + NCU * NQ1 * N1, NCU, tid);
      __syncthreads();
      contract_u<NQ1, N1, 1, 1, N1, NQ1, false, OP_PHI>(st, tro, NCU, tid);
      contract_u<NQ1, N1, 1, 1, N1, NQ1, false, OP_PHI>(st + NCU * NQ1 * N1, trn, NCU, tid);
    } else if (ND == 2) {
      contract_u<N1, 1, 1, 0, N1, NQ1, false, OP_PHI>(own, tro, NCU, tid);
      contract_u<N1, 1, 1, 0, N1, NQ1, false, OP_PHI>(oth, trn, NCU, tid);
    } else {                                   // a point face: the trace is the end node
      for (int idx = tid; idx < NCU; idx += NT) {
        tro[idx] = own[idx];
        trn[idx] = oth[idx];
      }
    }
    __syncthreads();
  }
  // ---- per face point: wsj (u - u^) n (left frame, sign of the side)
  for (int it = tid; it < NFACE * NQF; it += NT) {
    const int lf = it / NQF, sp = it % NQF;
    const int info = P.finfo[e * NFACE + lf];
    const int kind = info & 3;
    const bool right = kind == 0 && (info & 4);
    const bool sw = info & 8;
    const int brow = P.fnbr[e * NFACE + lf];
    const double* ff = P.ffgeo + (((sz_t)e * NFACE + lf) * NQF + sp) * FG;
    const double w = ff[ND] * (right ? -1.0 : 1.0);
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      const double uo = TR[((0 * NFACE + lf) * NCU + c) * NQF + sp];
      const double un = TR[((1 * NFACE + lf) * NCU + c) * NQF + sp];
      double jump = 0.0;
      if (kind == 0) {
        if (TRACE_CENTERED) jump = 0.5 * (uo - un);
        else if (sw == right) jump = uo - un;           // u^ = the neighbour's trace
      } else if (kind == 1) {
        jump = uo - (P.gq ? P.gq[((sz_t)brow * NQF + sp) * NCU + c] : 0.0);
      }
#pragma unroll
      for (int j = 0; j < ND; ++j) FJ[(lf * NQF + sp) * NGQ + c * ND + j] = w * jump * ff[j];
    }
  }
  __syncthreads();
  // lift onto the face nodes (GLL: a basis trace lives on its face's nodes)
  for (int it = tid; it < NB * NGQ; it += NT) {
    const int a = it / NGQ, cj = it % NGQ;
    const int ia[3] = {a % N1, (a / N1) % N1, ND == 3 ? a / (N1 * N1) : 0};
    double acc = 0.0;
#pragma unroll
    for (int lf = 0; lf < NFACE; ++lf) {
      const int ax = face_axis(lf);
      if (ia[ax] != (face_side(lf) ? N1 - 1 : 0)) continue;
      const int t0 = ia[ax == 0 ? 1 : 0];
      const int t1 = ND == 3 ? ia[ax == 2 ? 1 : 2] : 0;
#pragma unroll
      for (int sp = 0; sp < NQF; ++sp) {
        const int s0 = sp % NQ1, s1 = ND == 3 ? sp / NQ1 : 0;
        const double ph = ND == 3 ? c_phi[s0 * N1 + t0] * c_phi[s1 * N1 + t1]
                                  : (ND == 2 ? c_phi[s0 * N1 + t0] : 1.0);
        acc = fma(ph, FJ[(lf * NQF + sp) * NGQ + cj], acc);
      }
    }
    rhs[cj * NB + a] += acc;
  }
  __syncthreads();
  // ---- q = M_e^-1 rhs
  const double* mi = P.minv + (sz_t)e * NB * NB;
  for (int it = tid; it < NB * NGQ; it += NT) {
    const int a = it / NGQ, cj = it % NGQ;
    double acc = 0.0;
    for (int b = 0; b < NB; ++b) acc = fma(mi[a * NB + b], rhs[cj * NB + b], acc);
    flag(P, e, acc);
    P.out[((sz_t)e * NB + a) * NGQ + cj] = acc;
  }
}

// ---------------------------------------------------------------------------
// residual / tangent: one element per block of NT threads
// ---------------------------------------------------------------------------
__device__ __forceinline__ int e_of_block() { return blockIdx.x; }

// CACHE: 0 none; 1 tangent reading the base state (u, q, w at the volume and
// face points) from P.bcache, so only the direction's NV variables are
// interpolated; 2 building that cache (base variables only)
template <bool TANGENT, int CACHE = 0>
struct RShape {
  static constexpr int NVA = CACHE == 1 ? NV : NV * (TANGENT ? 2 : 1);  // variables in smem
  static constexpr int BS = (NVA > NG ? NVA : NG) * MX;           // one volume work buffer
  // face phase: traces of every face at its Gauss points, own and neighbour
  // side [side][face][v][NQF], one face's staging pair, and the face fluxes
  // (per batch of NFB faces: NFB < NFACE halves / thirds the face phase's
  // shared memory, which is what bounds the blocks per SM in 3D)
  static constexpr int TR = NFB * NVA * NQF;
  static constexpr int NBF = NVA * NFN;                        // one face's neighbour nodes
  static constexpr int FACE = 2 * TR + NBF + 2 * NVA * MXF + NFB * NQF * NCU + 2 * NBF;
  // the neighbour double buffer sits at the end of the work region, clear of
  // the volume buffers, so face 0's gathers fly during the volume phase
  static constexpr int WORK = 2 * BS + 2 * NBF > FACE ? 2 * BS + 2 * NBF : FACE;
  static constexpr int SMEM = NVA * NB + NCU * NB + WORK;         // doubles
};

// numerical flux f^ . n at one face point (disc.py:657-862), in the left frame.
// ODE states bind as w^ = (w- + w+)/2 for kind D / W, the left trace for the
// LLF flux and w_b on boundaries, with a zero tangent at faces (the reference
// seeds only u^ and q^ there, disc.py:690-691, 735-736, 808-810).
template <bool TANGENT>
__device__ __forceinline__ void face_flux(const NlParams& P, int e, int kind, bool right, bool sw,
                                          int brow, int s, const double* x, const double* n,
                                          double tau0, const double* vo, const double* vn,
                                          double* fh) {
  // vo / vn: own / neighbour values [u(NCU) q(NVQ) w(NW) | du dq dw] at this point
  const double* uo = vo;
  const double* duo = vo + NV;
  double wf[NW > 0 ? NW : 1], zw[NW > 0 ? NW : 1];
#pragma unroll
  for (int k = 0; k < (NW > 0 ? NW : 1); ++k) {
    zw[k] = 0.0;
    wf[k] = 0.0;
    if (NW > 0) {
      const double wo = vo[OW + k], wn = vn[OW + k];
      const double wl = right ? wn : wo, wr = right ? wo : wn;
      wf[k] = kind != 0 ? wo : (KIND_C ? wl : 0.5 * (wl + wr));
    }
  }
  const double* wp = NW > 0 ? wf : nullptr;
  const double* dwp = NW > 0 ? zw : nullptr;
  if (kind == 2) {                                     // neumann: f^ = g, zero tangent
#pragma unroll
    for (int c = 0; c < NCU; ++c) fh[c] = TANGENT ? 0.0 : P.gq[((sz_t)brow * NQF + s) * NCU + c];
    return;
  }
  if (kind == 3) {                                     // absorbing: c u^ (disc.py:783-794)
    double c;
    plan_ws(x, P.t, uo, nullptr, nullptr, n, &c);
    flag(P, e, c);
#pragma unroll
    for (int i = 0; i < NCU; ++i) {
      double qn = 0.0, dqn = 0.0;
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        qn += uo[NCU + i * ND + d] * n[d];
        if (TANGENT) dqn += duo[NCU + i * ND + d] * n[d];
      }
      fh[i] = TANGENT ? c * (0.5 * (duo[i] + c * dqn)) : c * (0.5 * (uo[i] + c * qn));
    }
    return;
  }
  double f[NCU * ND], df[NCU * ND];
  if (kind == 1) {                                     // dirichlet
    double g[NCU], zero[NCU];
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      g[c] = P.gq[((sz_t)brow * NQF + s) * NCU + c];
      zero[c] = 0.0;
    }
    if (KIND_C) {
      // LLF against the ghost state g (disc.py:839-862)
      double fg[NCU * ND], lami, lamg, dlami = 0.0;
      if (TANGENT) {
        plan_flux_d(x, P.t, uo, nullptr, wp, n, duo, nullptr, dwp, f, df);
        plan_ws_d(x, P.t, uo, nullptr, nullptr, n, duo, nullptr, nullptr, &lami, &dlami);
      } else {
        plan_flux(x, P.t, uo, nullptr, wp, n, f);
        plan_ws(x, P.t, uo, nullptr, nullptr, n, &lami);
      }
      plan_flux(x, P.t, g, nullptr, wp, n, fg);
      plan_ws(x, P.t, g, nullptr, nullptr, n, &lamg);
      flag(P, e, lami);
      flag(P, e, lamg);
      const double lam = ldg_max(lami, lamg);
      const double dlam = lami >= lamg ? dlami : 0.0;
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double fa = 0.0, dfa = 0.0;
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          flag(P, e, f[c * ND + d]);
          flag(P, e, fg[c * ND + d]);
          fa += (f[c * ND + d] + fg[c * ND + d]) * n[d];
          if (TANGENT) dfa += df[c * ND + d] * n[d];
        }
        fh[c] = TANGENT ? 0.5 * dfa + 0.5 * dlam * (uo[c] - g[c]) + 0.5 * lam * duo[c]
                        : 0.5 * fa + 0.5 * lam * (uo[c] - g[c]);
      }
    } else {
      // f(g, q_b) . n + tau_b (u_b - g) (disc.py:799-821)
      const double* qo = uo + NCU;
      const double* dqo = duo + NCU;
      if (TANGENT) plan_flux_d(x, P.t, g, qo, wp, n, zero, dqo, dwp, f, df);
      else plan_flux(x, P.t, g, qo, wp, n, f);
      double tau = tau0;
      if (HAS_WS) {
        double li, lg;
        plan_ws(x, P.t, uo, nullptr, nullptr, n, &li);
        plan_ws(x, P.t, g, nullptr, nullptr, n, &lg);
        flag(P, e, li);
        flag(P, e, lg);
        tau += ldg_max(li, lg);
      }
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        double fa = 0.0;
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          flag(P, e, f[c * ND + d]);
          fa += (TANGENT ? df[c * ND + d] : f[c * ND + d]) * n[d];
        }
        fh[c] = TANGENT ? fa + tau * duo[c] : fa + tau * (uo[c] - g[c]);
      }
    }
    return;
  }
  // interior: left / right states
  const double* uL = right ? vn : vo;
  const double* uR = right ? vo : vn;
  const double* duL = uL + NV;
  const double* duR = uR + NV;
  if (HAS_FHAT) {
    // user numerical flux over both traces (disc.py:753-758)
    const double* qL = NVQ ? uL + NCU : nullptr;
    const double* qR = NVQ ? uR + NCU : nullptr;
    double fo[NCU], dfo[NCU];
    if (TANGENT)
      plan_fhat_d(x, P.t, uL, uR, qL, qR, n, duL, duR, NVQ ? duL + NCU : nullptr,
                  NVQ ? duR + NCU : nullptr, fo, dfo);
    else
      plan_fhat(x, P.t, uL, uR, qL, qR, n, fo);
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      flag(P, e, fo[c]);
      fh[c] = TANGENT ? dfo[c] : fo[c];
    }
    return;
  }
  if (KIND_C) {
    // local Lax-Friedrichs (disc.py:724-751)
    double fR[NCU * ND], dfR[NCU * ND], lamL, lamR, dlamL = 0.0, dlamR = 0.0;
    if (TANGENT) {
      plan_flux_d(x, P.t, uL, nullptr, wp, n, duL, nullptr, dwp, f, df);
      plan_flux_d(x, P.t, uR, nullptr, wp, n, duR, nullptr, dwp, fR, dfR);
      plan_ws_d(x, P.t, uL, nullptr, nullptr, n, duL, nullptr, nullptr, &lamL, &dlamL);
      plan_ws_d(x, P.t, uR, nullptr, nullptr, n, duR, nullptr, nullptr, &lamR, &dlamR);
    } else {
      plan_flux(x, P.t, uL, nullptr, wp, n, f);
      plan_flux(x, P.t, uR, nullptr, wp, n, fR);
      plan_ws(x, P.t, uL, nullptr, nullptr, n, &lamL);
      plan_ws(x, P.t, uR, nullptr, nullptr, n, &lamR);
    }
    flag(P, e, lamL);
    flag(P, e, lamR);
    const double lam = ldg_max(lamL, lamR);
    const double dlam = lamL >= lamR ? dlamL : dlamR;
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      double fa = 0.0, dfa = 0.0;
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        flag(P, e, f[c * ND + d]);
        flag(P, e, fR[c * ND + d]);
        fa += (f[c * ND + d] + fR[c * ND + d]) * n[d];
        if (TANGENT) dfa += (df[c * ND + d] + dfR[c * ND + d]) * n[d];
      }
      fh[c] = TANGENT ? 0.5 * dfa + 0.5 * dlam * (uL[c] - uR[c]) + 0.5 * lam * (duL[c] - duR[c])
                      : 0.5 * fa + 0.5 * lam * (uL[c] - uR[c]);
    }
    return;
  }
  // kind D / W: f(u^, q^, w^) . n + tau (u^- - u^) (disc.py:657-722)
  double uh[NCU], duh[NCU], qh[NVQ > 0 ? NVQ : 1], dqh[NVQ > 0 ? NVQ : 1];
  if (HAS_UHAT) {                                      // user u^ (disc.py:502-504)
    const double* qL = NVQ ? uL + NCU : nullptr;
    const double* qR = NVQ ? uR + NCU : nullptr;
    if (TANGENT)
      plan_uhat_d(x, P.t, uL, uR, qL, qR, n, duL, duR, NVQ ? duL + NCU : nullptr,
                  NVQ ? duR + NCU : nullptr, uh, duh);
    else
      plan_uhat(x, P.t, uL, uR, qL, qR, n, uh);
  } else {
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      uh[c] = TRACE_CENTERED ? 0.5 * (uL[c] + uR[c]) : (sw ? uL[c] : uR[c]);
      if (TANGENT) duh[c] = TRACE_CENTERED ? 0.5 * (duL[c] + duR[c]) : (sw ? duL[c] : duR[c]);
    }
  }
#pragma unroll
  for (int k = 0; k < NVQ; ++k) {
    const double ql = uL[NCU + k], qr = uR[NCU + k];
    qh[k] = GRAD_CENTERED ? 0.5 * (ql + qr) : (sw ? qr : ql);
    if (TANGENT) {
      const double dl = duL[NCU + k], dr = duR[NCU + k];
      dqh[k] = GRAD_CENTERED ? 0.5 * (dl + dr) : (sw ? dr : dl);
    }
  }
  if (TANGENT) plan_flux_d(x, P.t, uh, qh, wp, n, duh, dqh, dwp, f, df);
  else plan_flux(x, P.t, uh, qh, wp, n, f);
  double tau = tau0;
  if (HAS_WS) {
    double ll, lr;
    plan_ws(x, P.t, uL, nullptr, nullptr, n, &ll);
    plan_ws(x, P.t, uR, nullptr, nullptr, n, &lr);
    flag(P, e, ll);
    flag(P, e, lr);
    tau += ldg_max(ll, lr);
  }
#pragma unroll
  for (int c = 0; c < NCU; ++c) {
    double fa = 0.0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      flag(P, e, f[c * ND + d]);
      fa += (TANGENT ? df[c * ND + d] : f[c * ND + d]) * n[d];
    }
    fh[c] = TANGENT ? fa + tau * (duL[c] - duh[c]) : fa + tau * (uL[c] - uh[c]);
  }
}

template <bool TANGENT, int CACHE = 0>
__device__ __forceinline__ void residual_body(const NlParams& P) {
  using S = RShape<TANGENT, CACHE>;
  constexpr int NVA = S::NVA;                  // variables held in shared memory
  constexpr int NVL = NV * (TANGENT ? 2 : 1);  // variables of a point (base | direction)
  const double* bvol = CACHE == 1 ? P.bcache + (sz_t)e_of_block() * NV * NQ : nullptr;
  const double* bfac = CACHE == 1 ? P.bcache + (sz_t)P.ne * NV * NQ +
                                        (sz_t)e_of_block() * 2 * NFACE * NV * NQF : nullptr;
  extern __shared__ __align__(16) double smem_r[];
  double* sV = smem_r;                      // [NVA][NB] node values
  double* sR = sV + NVA * NB;             // [NCU][NB] residual accumulator
  double* bA = sR + NCU * NB;             // work buffers
  double* bB = bA + S::BS;
  const int e = blockIdx.x, tid = threadIdx.x;
  if (e >= P.ne) return;

  // ---- load u, q (+ du, dq) of the element: [v][node], NL_LOAD_BATCH
  // loads in flight per thread before their stores
  constexpr int LB = NL_LOAD_BATCH;
  for (int i0 = tid; i0 < NVA * NB; i0 += LB * NT) {
    double val[LB];
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * NT;
      const int v = idx / NB, a = idx % NB;
      const int fam = CACHE == 1 ? 1 : (v >= NV), vv = v % NV;
      val[b] = idx < NVA * NB ? state_at(P, fam, vv, (sz_t)e, a) : 0.0;
    }
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int idx = i0 + b * NT;
      if (idx < NVA * NB) {
        sV[idx] = val[b];
        bA[idx] = val[b];
      }
    }
  }
  __syncthreads();

  // neighbour face nodes, one face ahead (cp.async into a double buffer)
  double* NB2 = bA + S::WORK - 2 * S::NBF;
  auto prefetch_face = [&](int lf, double* dst) {
    const int info = P.finfo[e * NFACE + lf];
    const bool interior = (info & 3) == 0;
    const int nbr = P.fnbr[e * NFACE + lf];
    for (int idx = tid; idx < S::NBF; idx += NT) {
      const int v = idx / NFN, t = idx % NFN;
      if (interior) cp_async8(dst + idx, state_ptr(P, CACHE == 1 ? 1 : (v >= NV), v % NV, (sz_t)nbr,
                                                   P.nmap[(info >> 8) * NFN + t]));
      else dst[idx] = 0.0;
    }
    cp_async_commit();
  };
  prefetch_face(0, NB2);

  // ---- volume: interpolate to quadrature points
  double* vq;
  to_quad(bA, bB, NVA, tid, vq);
  double* gbuf = vq == bA ? bB : bA;
  const double* geo_e = P.geo + (sz_t)e * (1 + ND * ND);
  if (CACHE == 2) {
    // base cache: the volume-point values; the face traces below
    for (int idx = tid; idx < NV * NQ; idx += NT) P.bcache[(sz_t)e * NV * NQ + idx] = vq[idx];
  }
  for (int p = tid; p < (CACHE == 2 ? 0 : NQ); p += NT) {
    double val[NVL];
#pragma unroll
    for (int v = 0; v < NVL; ++v)
      val[v] = CACHE == 1 ? (v < NV ? bvol[v * NQ + p] : vq[(v - NV) * NQ + p]) : vq[v * NQ + p];
    double x[ND];
    // affine: one (detJ, invJ^T) per element and x = x0 + J xi; curved: per point
    const double* geo = CURVED ? P.vgeo + ((sz_t)e * NQ + p) * VG : geo_e;
    const double detj = geo[0];
    if (CURVED) {
#pragma unroll
      for (int d = 0; d < ND; ++d) x[d] = geo[1 + ND * ND + d];
    } else {
      double xi[ND];
      quad_point(p, xi);
      phys_point(P, e, xi, x);
    }
    double f[NCU * ND], df[NCU * ND], s[NCU], ds[NCU];
    const double* qv = NVQ ? val + NCU : nullptr;
    const double* wv = NW ? val + OW : nullptr;
    if (TANGENT) {
      const double* dqv = NVQ ? val + NV + NCU : nullptr;
      const double* dwv = NW ? val + NV + OW : nullptr;
      plan_flux_d(x, P.t, val, qv, wv, nullptr, val + NV, dqv, dwv, f, df);
      plan_src_d(x, P.t, val, qv, wv, nullptr, val + NV, dqv, dwv, s, ds);
    } else {
      plan_flux(x, P.t, val, qv, wv, nullptr, f);
      plan_src(x, P.t, val, qv, wv, nullptr, s);
    }
    const double wd = c_qw[p] * detj;
#pragma unroll
    for (int c = 0; c < NCU; ++c) {
      flag(P, e, s[c]);
#pragma unroll
      for (int d = 0; d < ND; ++d) flag(P, e, f[c * ND + d]);
#pragma unroll
      for (int r = 0; r < ND; ++r) {
        double a = 0.0;
#pragma unroll
        for (int d = 0; d < ND; ++d) a = fma(TANGENT ? df[c * ND + d] : f[c * ND + d], geo[1 + d * ND + r], a);
        gbuf[(r * NCU + c) * NQ + p] = wd * a;
      }
      gbuf[(ND * NCU + c) * NQ + p] = wd * (TANGENT ? ds[c] : s[c]);
    }
  }
  __syncthreads();
  if (CACHE != 2) {
    double* rn;
    from_quad(gbuf, vq, NG, tid, rn);
    for (int idx = tid; idx < NCU * NB; idx += NT) {
      const int c = idx / NB, a = idx % NB;
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r <= ND; ++r) acc += rn[(r * NCU + c) * NB + a];
      sR[idx] = -acc;
    }
  }
  __syncthreads();

  // ---- faces, in batches of NFB: traces of the batch's faces at their Gauss
  // points (one face's own and neighbour staging at a time), then every face
  // point's f^ of the batch at once, then the lift with each (node, component)
  // owned by one thread
  double* TRc = bA;                            // [side][face of the batch][v][NQF]
  double* SO = bA + 2 * S::TR;                 // own face nodes [v][face grid]
  double* ST1 = SO + S::NBF;                   // first-stage scratch [side][v][..]
  double* sF = ST1 + 2 * NVA * MXF;            // [face of the batch][NQF][NCU]
  for (int b0 = 0; b0 < NFACE; b0 += NFB) {
    for (int lf = b0; lf < b0 + NFB; ++lf) {
      if (lf + 1 < NFACE) prefetch_face(lf + 1, NB2 + ((lf + 1) & 1) * S::NBF);
      else cp_async_commit();                  // (empty group keeps the counting uniform)
      for (int idx = tid; idx < S::NBF; idx += NT)
        SO[idx] = sV[(idx / NFN) * NB + face_vol_node(lf, idx % NFN)];
      cp_async_wait1();                        // this face's neighbour nodes have landed
      __syncthreads();
      const double* nb = NB2 + (lf & 1) * S::NBF;
      double* tro = TRc + (0 * NFB + lf - b0) * NVA * NQF;
      double* trn = TRc + (1 * NFB + lf - b0) * NVA * NQF;
      if (ND == 3) {
        contract_u<N1, N1, 1, 0, N1, NQ1, false, OP_PHI>(SO, ST1, NVA, tid);
        contract_u<N1, N1, 1, 0, N1, NQ1, false, OP_PHI>(nb, ST1 + NVA * NQ1 * N1, NVA, tid);
        __syncthreads();
        contract_u<NQ1, N1, 1, 1, N1, NQ1, false, OP_PHI>(ST1, tro, NVA, tid);
        contract_u<NQ1, N1, 1, 1, N1, NQ1, false, OP_PHI>(ST1 + NVA * NQ1 * N1, trn, NVA, tid);
      } else if (ND == 2) {
        contract_u<N1, 1, 1, 0, N1, NQ1, false, OP_PHI>(SO, tro, NVA, tid);
        contract_u<N1, 1, 1, 0, N1, NQ1, false, OP_PHI>(nb, trn, NVA, tid);
      } else {                                 // a point face: the trace is the end node
        for (int idx = tid; idx < NVA; idx += NT) {
          tro[idx] = SO[idx];
          trn[idx] = nb[idx];
        }
      }
      __syncthreads();
    }
    if (CACHE == 2) {
      // base cache: the traces [side][face][v][NQF] of the base variables
      double* dst = P.bcache + (sz_t)P.ne * NV * NQ + (sz_t)e * 2 * NFACE * NV * NQF;
      for (int idx = tid; idx < 2 * NFB * NV * NQF; idx += NT) {
        const int side = idx / (NFB * NV * NQF), rest = idx % (NFB * NV * NQF);
        dst[(side * NFACE + b0) * NV * NQF + rest] = TRc[idx];
      }
      __syncthreads();
      continue;
    }
    for (int it = tid; it < NFB * NQF; it += NT) {
      const int lfb = it / NQF, s = it % NQF, lf = b0 + lfb;
      const int info = P.finfo[e * NFACE + lf];
      const int kind = info & 3;
      const bool right = kind == 0 && (info & 4);
      const bool sw = info & 8;
      const int brow = P.fnbr[e * NFACE + lf];
      const double* fg = P.fgeo + ((sz_t)e * NFACE + lf) * (ND + 2);
      const double* ff = CURVED ? P.ffgeo + (((sz_t)e * NFACE + lf) * NQF + s) * FG : fg;
      double n[ND];
#pragma unroll
      for (int d = 0; d < ND; ++d) n[d] = ff[d];
      double x[ND];
      if (CURVED) {
#pragma unroll
        for (int d = 0; d < ND; ++d) x[d] = ff[ND + 1 + d];
      } else {
        phys_point(P, e, &c_fxi[(lf * NQF + s) * ND], x);
      }
      double vo[NVL], vn[NVL];
#pragma unroll
      for (int v = 0; v < NVL; ++v) {
        if (CACHE == 1 && v < NV) {
          vo[v] = bfac[((0 * NFACE + lf) * NV + v) * NQF + s];
          vn[v] = bfac[((1 * NFACE + lf) * NV + v) * NQF + s];
        } else {
          const int vs = CACHE == 1 ? v - NV : v;
          vo[v] = TRc[((0 * NFB + lfb) * NVA + vs) * NQF + s];
          vn[v] = TRc[((1 * NFB + lfb) * NVA + vs) * NQF + s];
        }
      }
      double fh[NCU];
      face_flux<TANGENT>(P, e, kind, right, sw, brow, s, x, n, fg[ND + 1], vo, vn, fh);
      const double w = (CURVED ? ff[ND] : c_fw[lf * NQF + s] * fg[ND]) * (right ? -1.0 : 1.0);
#pragma unroll
      for (int c = 0; c < NCU; ++c) sF[(lfb * NQF + s) * NCU + c] = w * fh[c];
    }
    __syncthreads();
    // lift: thread owns (volume node, component) and sums the batch's faces through it
    for (int it = tid; it < NB * NCU; it += NT) {
      const int a = it / NCU, c = it % NCU;
      const int ia[3] = {a % N1, (a / N1) % N1, ND == 3 ? a / (N1 * N1) : 0};
      double acc = 0.0;
#pragma unroll
      for (int lfb = 0; lfb < NFB; ++lfb) {
        const int lf = b0 + lfb;
        const int ax = face_axis(lf);
        if (ia[ax] != (face_side(lf) ? N1 - 1 : 0)) continue;
        // face-node coordinates (t0, t1) over the tangential axes, ascending
        const int t0 = ia[ax == 0 ? 1 : 0];
        const int t1 = ND == 3 ? ia[ax == 2 ? 1 : 2] : 0;
#pragma unroll
        for (int s = 0; s < NQF; ++s) {
          const int s0 = s % NQ1, s1 = ND == 3 ? s / NQ1 : 0;
          const double ph = ND == 3 ? c_phi[s0 * N1 + t0] * c_phi[s1 * N1 + t1]
                                    : (ND == 2 ? c_phi[s0 * N1 + t0] : 1.0);
          acc = fma(ph, sF[(lfb * NQF + s) * NCU + c], acc);
        }
      }
      sR[c * NB + a] += acc;
    }
    __syncthreads();
  }
  if (CACHE == 2) return;
  for (int idx = tid; idx < NCU * NB; idx += NT) {
    const int a = idx / NCU, c = idx % NCU;
    P.out[(sz_t)e * NB * NCU + idx] = sR[c * NB + a];
  }
}

#ifndef NL_RES_MINB
#define NL_RES_MINB (ND == 3 ? 3 : 1)   // (3D: 3 blocks / SM of shared state, registers capped to match)
#endif
extern "C" __global__ void __launch_bounds__(NT, NL_RES_MINB) nl_residual(const __grid_constant__ NlParams P) {
  residual_body<false>(P);
}
// uncached tangent: register-capped only where the prelude asks (2D kind-C
// models: NL_TANU_MINB from nonlinear.MINB_2D_C)
#ifdef NL_TANU_MINB
extern "C" __global__ void __launch_bounds__(NT, NL_TANU_MINB) nl_tangent(const __grid_constant__ NlParams P) {
#else
extern "C" __global__ void __launch_bounds__(NT) nl_tangent(const __grid_constant__ NlParams P) {
#endif
  residual_body<true>(P);
}
#ifndef NL_TAN_MINB
#define NL_TAN_MINB (ND == 3 ? 3 : 1)  // cached tangent: 60 KB of shared state (NS 3D) fits 3
#endif                                // blocks / SM with the registers capped to match (measured
                                      // NS tangent 3.69 -> 4.24 GDOF/s, 392 B of spills)
extern "C" __global__ void __launch_bounds__(NT, NL_TAN_MINB) nl_tangent_cached(const __grid_constant__ NlParams P) {
  residual_body<true, 1>(P);
}
extern "C" __global__ void __launch_bounds__(NT, NL_RES_MINB) nl_base_cache(const __grid_constant__ NlParams P) {
  residual_body<false, 2>(P);
}

// ---------------------------------------------------------------------------
// mass operator (disc.py:897-948): out = scale * int m(u) v phi, or with
// EXTRA the (dm/du . du) v term; v in P.q, base u in P.u, du in P.du
// ---------------------------------------------------------------------------
constexpr int NVM = MASS_CONST ? NCU : 3 * NCU;   // v (+ u, du)
constexpr int MSMEM = 2 * (NVM > NCU ? NVM : NCU) * MX;

template <bool EXTRA>
__device__ __forceinline__ void mass_body(const NlParams& P) {
  extern __shared__ __align__(16) double smem_m[];
  double* bA = smem_m;
  double* bB = smem_m + MSMEM / 2;
  const int e = blockIdx.x, tid = threadIdx.x;
  if (e >= P.ne) return;
  constexpr int NL = MASS_CONST ? NCU : (EXTRA ? 3 * NCU : 2 * NCU);   // v (+ u (+ du))
  for (int idx = tid; idx < NL * NB; idx += NT) {
    const int v = idx / NB, a = idx % NB;
    const double* src = v < NCU ? P.q : (v < 2 * NCU ? P.u : P.du);
    bA[idx] = src[((sz_t)e * NB + a) * NCU + v % NCU];
  }
  __syncthreads();
  double* vq;
  to_quad(bA, bB, NL, tid, vq);
  double* fld = vq == bA ? bB : bA;
  for (int p = tid; p < NQ; p += NT) {
    const double detj = CURVED ? P.vgeo[((sz_t)e * NQ + p) * VG] : P.geo[(sz_t)e * (1 + ND * ND)];
    double m[NCU], dm[NCU];
    if (MASS_CONST) {
#pragma unroll
      for (int c = 0; c < NCU; ++c) { m[c] = c_mass[c]; dm[c] = 0.0; }
    } else {
      double xi[ND], x[ND], uq[NCU], duq[NCU];
      if (CURVED) {
#pragma unroll
        for (int d = 0; d < ND; ++d) x[d] = P.vgeo[((sz_t)e * NQ + p) * VG + 1 + ND * ND + d];
      } else {
        quad_point(p, xi);
        phys_point(P, e, xi, x);
      }
#pragma unroll
      for (int c = 0; c < NCU; ++c) {
        uq[c] = vq[(NCU + c) * NQ + p];
        duq[c] = EXTRA ? vq[(2 * NCU + c) * NQ + p] : 0.0;
      }
      if (EXTRA) plan_mass_d(x, P.t, uq, nullptr, nullptr, nullptr, duq, nullptr, nullptr, m, dm);
      else plan_mass(x, P.t, uq, nullptr, nullptr, nullptr, m);
#pragma unroll
      for (int c = 0; c < NCU; ++c) flag(P, e, m[c]);
    }
    const double wd = c_qw[p] * detj;
#pragma unroll
    for (int c = 0; c < NCU; ++c)
      fld[c * NQ + p] = wd * (EXTRA ? dm[c] : m[c]) * vq[c * NQ + p];
  }
  __syncthreads();
  // phi^T along every axis: reuse from_quad with the source-field selector
  // (fields indexed >= ND*NCU take phi everywhere): shift by ND*NCU
  double* other = fld == bA ? bB : bA;
  double* res;
  if (ND == 3) {
    contract_u<NQ1, NQ1, NQ1, 0, NQ1, N1, true, OP_PHI>(fld, other, NCU, tid);
    __syncthreads();
    contract_u<N1, NQ1, NQ1, 1, NQ1, N1, true, OP_PHI>(other, fld, NCU, tid);
    __syncthreads();
    contract_u<N1, N1, NQ1, 2, NQ1, N1, true, OP_PHI>(fld, other, NCU, tid);
    __syncthreads();
    res = other;
  } else if (ND == 2) {
    contract_u<NQ1, NQ1, 1, 0, NQ1, N1, true, OP_PHI>(fld, other, NCU, tid);
    __syncthreads();
    contract_u<N1, NQ1, 1, 1, NQ1, N1, true, OP_PHI>(other, fld, NCU, tid);
    __syncthreads();
    res = fld;
  } else {
    contract_u<NQ1, 1, 1, 0, NQ1, N1, true, OP_PHI>(fld, other, NCU, tid);
    __syncthreads();
    res = other;
  }
  for (int idx = tid; idx < NCU * NB; idx += NT) {
    const int a = idx / NCU, c = idx % NCU;
    P.out[(sz_t)e * NB * NCU + idx] = P.scale * res[c * NB + a];
  }
}

extern "C" __global__ void __launch_bounds__(NT) nl_mass(const __grid_constant__ NlParams P) {
  mass_body<false>(P);
}
extern "C" __global__ void __launch_bounds__(NT) nl_mass_extra(const __grid_constant__ NlParams P) {
  mass_body<true>(P);
}

// M^-1 v = detJ^-1 (M1^-1 (x) ... ) v per component (MassPreconditioner.apply)
extern "C" __global__ void __launch_bounds__(NT) nl_mass_inv(const __grid_constant__ NlParams P) {
  extern __shared__ __align__(16) double smem_i[];
  double* bA = smem_i;
  double* bB = smem_i + NCU * NB;
  const int e = blockIdx.x, tid = threadIdx.x;
  if (e >= P.ne) return;
  for (int idx = tid; idx < NCU * NB; idx += NT) {
    const int v = idx / NB, a = idx % NB;
    bA[idx] = P.q[((sz_t)e * NB + a) * NCU + v];
  }
  __syncthreads();
  if (CURVED) {
    // non-affine: the element's own inverse mass matrix (disc.py:107-110)
    const double* mi = P.minv + (sz_t)e * NB * NB;
    for (int idx = tid; idx < NCU * NB; idx += NT) {
      const int a = idx / NCU, c = idx % NCU;
      double acc = 0.0;
      for (int b = 0; b < NB; ++b) acc = fma(mi[a * NB + b], bA[c * NB + b], acc);
      P.out[(sz_t)e * NB * NCU + idx] = P.scale * acc;
    }
    return;
  }
  double* res;
  if (ND == 3) {
    contract_u<N1, N1, N1, 0, N1, N1, false, OP_M1INV>(bA, bB, NCU, tid);
    __syncthreads();
    contract_u<N1, N1, N1, 1, N1, N1, false, OP_M1INV>(bB, bA, NCU, tid);
    __syncthreads();
    contract_u<N1, N1, N1, 2, N1, N1, false, OP_M1INV>(bA, bB, NCU, tid);
    __syncthreads();
    res = bB;
  } else if (ND == 2) {
    contract_u<N1, N1, 1, 0, N1, N1, false, OP_M1INV>(bA, bB, NCU, tid);
    __syncthreads();
    contract_u<N1, N1, 1, 1, N1, N1, false, OP_M1INV>(bB, bA, NCU, tid);
    __syncthreads();
    res = bA;
  } else {
    contract_u<N1, 1, 1, 0, N1, N1, false, OP_M1INV>(bA, bB, NCU, tid);
    __syncthreads();
    res = bB;
  }
  const double inv = P.scale / P.geo[(sz_t)e * (1 + ND * ND)];
  for (int idx = tid; idx < NCU * NB; idx += NT) {
    const int a = idx / NCU, c = idx % NCU;
    P.out[(sz_t)e * NB * NCU + idx] = inv * res[c * NB + a];
  }
}

// ---------------------------------------------------------------------------
// plain element mass on the (ncu, nd) gradient block: out = scale * M v,
// M_ab = int phi_a phi_b (disc.py:919-921, Mq = mass @ vq; with scale = -1
// and v = the lifted gradient it forms the wave gradient residual Rq)
// ---------------------------------------------------------------------------
constexpr int NQC = NCU * ND;
extern "C" __global__ void __launch_bounds__(NT) nl_mass_q(const __grid_constant__ NlParams P) {
  extern __shared__ __align__(16) double smem_q[];
  double* bA = smem_q;
  double* bB = smem_q + NQC * MX;
  const int e = blockIdx.x, tid = threadIdx.x;
  if (e >= P.ne) return;
  for (int idx = tid; idx < NQC * NB; idx += NT) {
    const int v = idx / NB, a = idx % NB;
    bA[idx] = P.q[((sz_t)e * NB + a) * NQC + v];
  }
  __syncthreads();
  double* vq;
  to_quad(bA, bB, NQC, tid, vq);
  double* fld = vq == bA ? bB : bA;
  const double detj = P.geo[(sz_t)e * (1 + ND * ND)];
  for (int idx = tid; idx < NQC * NQ; idx += NT) fld[idx] = c_qw[idx % NQ] * detj * vq[idx];
  __syncthreads();
  double* other = fld == bA ? bB : bA;
  double* res;
  if (ND == 3) {
    contract_u<NQ1, NQ1, NQ1, 0, NQ1, N1, true, OP_PHI>(fld, other, NQC, tid);
    __syncthreads();
    contract_u<N1, NQ1, NQ1, 1, NQ1, N1, true, OP_PHI>(other, fld, NQC, tid);
    __syncthreads();
    contract_u<N1, N1, NQ1, 2, NQ1, N1, true, OP_PHI>(fld, other, NQC, tid);
    __syncthreads();
    res = other;
  } else if (ND == 2) {
    contract_u<NQ1, NQ1, 1, 0, NQ1, N1, true, OP_PHI>(fld, other, NQC, tid);
    __syncthreads();
    contract_u<N1, NQ1, 1, 1, NQ1, N1, true, OP_PHI>(other, fld, NQC, tid);
    __syncthreads();
    res = fld;
  } else {
    contract_u<NQ1, 1, 1, 0, NQ1, N1, true, OP_PHI>(fld, other, NQC, tid);
    __syncthreads();
    res = other;
  }
  for (int idx = tid; idx < NQC * NB; idx += NT) {
    const int a = idx / NQC, v = idx % NQC;
    P.out[(sz_t)e * NB * NQC + idx] = P.scale * res[v * NB + a];
  }
}

// ---------------------------------------------------------------------------
// pointwise ODE block, collocated at the solution nodes (disc.py:876-893):
// Rw = beta w - s_w(x, t, u, q, w), tangent beta dw - ds_w
// ---------------------------------------------------------------------------
template <bool TANGENT>
__device__ __forceinline__ void ode_body(const NlParams& P) {
  const sz_t idx = (sz_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (NW == 0 || idx >= (sz_t)P.ne * NB) return;
  const int e = (int)(idx / NB), a = (int)(idx % NB);
  double x[ND];
  phys_point(P, e, &c_xn[a * ND], x);
  double val[2 * (NV > 0 ? NV : 1)];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    val[v] = state_at(P, 0, v, (sz_t)e, a);
    val[NV + v] = TANGENT ? state_at(P, 1, v, (sz_t)e, a) : 0.0;
  }
  const double* qv = NVQ ? val + NCU : nullptr;
  const double* dqv = NVQ ? val + NV + NCU : nullptr;
  double sw[NW > 0 ? NW : 1], dsw[NW > 0 ? NW : 1];
  if (TANGENT) plan_sw_d(x, P.t, val, qv, val + OW, nullptr, val + NV, dqv, val + NV + OW, sw, dsw);
  else plan_sw(x, P.t, val, qv, val + OW, nullptr, sw);
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    flag(P, e, sw[k]);
    P.out[idx * NW + k] = TANGENT ? ODE_BETA * val[NV + OW + k] - dsw[k]
                                  : ODE_BETA * val[OW + k] - sw[k];
  }
}

extern "C" __global__ void nl_ode(const __grid_constant__ NlParams P) { ode_body<false>(P); }
extern "C" __global__ void nl_ode_tangent(const __grid_constant__ NlParams P) { ode_body<true>(P); }

// M^-1 on the (ncu, nd) gradient block (MassPreconditioner, driver.py:99-106)
extern "C" __global__ void __launch_bounds__(NT) nl_mass_inv_q(const __grid_constant__ NlParams P) {
  extern __shared__ __align__(16) double smem_iq[];
  double* bA = smem_iq;
  double* bB = smem_iq + NQC * NB;
  const int e = blockIdx.x, tid = threadIdx.x;
  if (e >= P.ne) return;
  for (int idx = tid; idx < NQC * NB; idx += NT) {
    const int v = idx / NB, a = idx % NB;
    bA[idx] = P.q[((sz_t)e * NB + a) * NQC + v];
  }
  __syncthreads();
  double* res;
  if (ND == 3) {
    contract_u<N1, N1, N1, 0, N1, N1, false, OP_M1INV>(bA, bB, NQC, tid);
    __syncthreads();
    contract_u<N1, N1, N1, 1, N1, N1, false, OP_M1INV>(bB, bA, NQC, tid);
    __syncthreads();
    contract_u<N1, N1, N1, 2, N1, N1, false, OP_M1INV>(bA, bB, NQC, tid);
    __syncthreads();
    res = bB;
  } else if (ND == 2) {
    contract_u<N1, N1, 1, 0, N1, N1, false, OP_M1INV>(bA, bB, NQC, tid);
    __syncthreads();
    contract_u<N1, N1, 1, 1, N1, N1, false, OP_M1INV>(bB, bA, NQC, tid);
    __syncthreads();
    res = bA;
  } else {
    contract_u<N1, 1, 1, 0, N1, N1, false, OP_M1INV>(bA, bB, NQC, tid);
    __syncthreads();
    res = bB;
  }
  const double inv = P.scale / P.geo[(sz_t)e * (1 + ND * ND)];
  for (int idx = tid; idx < NQC * NB; idx += NT) {
    const int a = idx / NQC, v = idx % NQC;
    P.out[(sz_t)e * NB * NQC + idx] = inv * res[v * NB + a];
  }
}
