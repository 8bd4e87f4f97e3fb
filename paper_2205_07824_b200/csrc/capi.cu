// C ABI of libldgb200.so: handle lifecycle and the operator entry points.
// See include/ldgb200.h for the reference interface each one replaces.

#include <climits>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <string>
#include <vector>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif
#include "ldg_dense.cuh"
#include "nvtx.cuh"
#include "ldg_tensor.cuh"

namespace {
thread_local std::string g_err;

int fail(int code, const char* what, cudaError_t e = cudaSuccess) {
  g_err = what;
  if (e != cudaSuccess) {
    g_err += ": ";
    g_err += cudaGetErrorString(e);
  }
  return code;
}

template <typename T>
int upload(T** dst, const T* src, size_t n, const char* what) {
  *dst = nullptr;
  if (n == 0) return 0;
  cudaError_t e = cudaMalloc(dst, n * sizeof(T));
  if (e != cudaSuccess) return fail(3, what, e);
  e = cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(3, what, e);
  return 0;
}
}  // namespace

struct LdgHandle {
  int dense = 0;                 // 0: tensor (quad/hex), 1: dense (tri/tet)
  ldg::DenseParams D;
  std::vector<void*> dense_bufs;
  ldg::TensorParams P;
  double* geo = nullptr;
  int32_t* fnbr = nullptr;
  int32_t* finfo = nullptr;
  double* ftau = nullptr;
  int32_t* nmap = nullptr;
  double* frec = nullptr;
  double* kco = nullptr;
  int kstride = 0;
  int c_diag = 0;
  unsigned long long* bad = nullptr;
  int* fuse = nullptr;           // one-launch operator: counters and per-group windows
  int2* fuse_dep = nullptr;
  // host-pipeline resources (ldg_apply_host): copy streams, chunk events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_p2;
  cudaEvent_t ev_start = nullptr;
};

#ifndef LDG_STAGE_NT
#define LDG_STAGE_NT 1            // staging copies with non-temporal stores (0: memcpy)
#endif
// pageable -> pinned staging copy of one slice: the pinned destination is not
// read again by the host, so non-temporal 16-B stores skip the read-for-
// ownership of every destination line (2 instead of 3 memory transfers per
// byte); SSE2 only (baseline x86-64)
static void stage_copy(double* dst, const double* src, size_t n) {
#if LDG_STAGE_NT && defined(__x86_64__)
  size_t i = 0;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) != 0) {      // 16-B align the destination
    dst[0] = src[0];
    i = 1;
  }
  for (; i + 8 <= n; i += 8) {
    const __m128d a0 = _mm_loadu_pd(src + i), a1 = _mm_loadu_pd(src + i + 2);
    const __m128d a2 = _mm_loadu_pd(src + i + 4), a3 = _mm_loadu_pd(src + i + 6);
    _mm_stream_pd(dst + i, a0);
    _mm_stream_pd(dst + i + 2, a1);
    _mm_stream_pd(dst + i + 4, a2);
    _mm_stream_pd(dst + i + 6, a3);
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
#else
  memcpy(dst, src, n * sizeof(double));
#endif
}

namespace ldg {
// error reporting for the other translation units of the C ABI (comm.cu)
int set_error(int code, const char* what, cudaError_t e) { return fail(code, what, e); }
}  // namespace ldg

extern "C" {

int ldg_version(void) { return 1; }

const char* ldg_last_error(void) { return g_err.c_str(); }

int ldg_create(const LdgTables* t, LdgHandle** out) {
  std::vector<double> h_rec_host;   // face records, kept on the host for the chunk schedule
  if (!t || !out) return fail(2, "null argument");
  if (t->nd < 2 || t->nd > 3 || t->n1 < 2 || t->n1 > LDG_MAX_N1 || t->ncu < 1 ||
      t->ncu > LDG_MAX_NCU || t->ne < 0)
    return fail(2, "unsupported tensor configuration");
  LdgHandle* h = new LdgHandle();
  memset(&h->P, 0, sizeof(h->P));
  h->P.ghost0 = INT32_MAX;
  const size_t ne = (size_t)t->ne, nf = 2 * t->nd;
  size_t nfn = t->nd == 3 ? (size_t)t->n1 * t->n1 : (size_t)t->n1;
  int rc = 0;
  rc |= upload(&h->geo, t->geo, ne * (1 + t->nd * t->nd), "geo");
  rc |= upload(&h->fnbr, t->fnbr, ne * nf, "fnbr");
  rc |= upload(&h->finfo, t->finfo, ne * nf, "finfo");
  rc |= upload(&h->ftau, t->ftau, ne * nf, "ftau");
  rc |= upload(&h->nmap, t->nmap, (size_t)t->n_maps * nfn, "nmap");
  {
    // Derived per-element / per-face data of the fused kernels (ldg_fused.cu):
    //  * coefficient block [C | Cu | sJ(axis)] with
    //    C[c][r][k][s] = detJ sum_{d,e} invjt[d][r] aq[c][d][k][e] invjt[e][s],
    //    Cu[c][r][k]   = detJ sum_d invjt[d][r] au[c][d][k],
    //    sJ(axis)      = detJ |invjt[:, axis]|  (|t1 x t2| of an affine face);
    //  * face records {sJ*tau, nbr, info | flags}.
    const int nd = t->nd, ncu = t->ncu;
    const int cq = ncu * nd * ncu * nd, cu = ncu * nd * ncu;
    const int kst = ((cq + cu + nd) + 1) & ~1;
    std::vector<double> kco((size_t)ne * kst, 0.0);
    std::vector<double> rec(ne * nf * 2);
    auto axis_of = [&](int lf) {
      return nd == 3 ? (lf < 2 ? 2 : (lf < 4 ? 1 : 0)) : ((lf == 0 || lf == 2) ? 1 : 0);
    };
    for (size_t e = 0; e < ne; ++e) {
      const double* g = t->geo + e * (1 + nd * nd);
      const double dj = g[0];
      const double* ij = g + 1;                   // ij[d*nd + r] = invjt[d][r]
      double* kb = kco.data() + e * kst;
      for (int c = 0; c < ncu; ++c)
        for (int r = 0; r < nd; ++r)
          for (int k = 0; k < ncu; ++k)
            for (int s2 = 0; s2 < nd; ++s2) {
              double v = 0.0;
              for (int d = 0; d < nd; ++d)
                for (int ee = 0; ee < nd; ++ee)
                  v += ij[d * nd + r] * t->aq[((c * 3 + d) * LDG_MAX_NCU + k) * 3 + ee] *
                       ij[ee * nd + s2];
              kb[((c * nd + r) * ncu + k) * nd + s2] = dj * v;
            }
      for (int c = 0; c < ncu; ++c)
        for (int r = 0; r < nd; ++r)
          for (int k = 0; k < ncu; ++k) {
            double v = 0.0;
            for (int d = 0; d < nd; ++d) v += ij[d * nd + r] * t->au[(c * 3 + d) * LDG_MAX_NCU + k];
            kb[cq + (c * nd + r) * ncu + k] = dj * v;
          }
      for (int a = 0; a < nd; ++a) {
        double l2 = 0.0;
        for (int d = 0; d < nd; ++d) l2 += ij[d * nd + a] * ij[d * nd + a];
        kb[cq + cu + a] = dj * sqrt(l2);
      }
      for (size_t lf = 0; lf < nf; ++lf) {
        const size_t x = e * nf + lf;
        int32_t info = t->finfo[x] & 0x00ffffff;
        const int kind = info & LDG_FACE_KIND_MASK;
        const double sj = kb[cq + cu + axis_of((int)lf)];
        // coefficient form of the trace rules (disc.py:492-574, 657-821):
        // jump = alpha d and sJ sigma tau (u_L - u^) = beta sJ tau d with
        // d = u_own - u_other; alpha, beta in {0, 1, 1/2}
        int acode = 0;
        double beta = 0.0;
        if (kind == LDG_FACE_INTERIOR) {
          const bool right = info & LDG_FACE_SIDE_RIGHT, sw = info & LDG_FACE_SWITCH;
          const bool tc = t->trace_centered, gc = t->grad_centered;
          if (tc) { acode = 2; beta = 0.5; }
          else {
            acode = (sw == right) ? 1 : 0;      // u^ = the neighbour's trace
            beta = sw ? 0.0 : 1.0;              // penalty vanishes on switch faces
          }
          if (acode != 0 || beta != 0.0) info |= LDG_FL_UNBR;
          if (gc || (sw == right)) info |= LDG_FL_EXPORT;
          {
            // consumer-slot exports need the neighbour's face-node order; flag
            // the (structured-mesh) case where it is this face's own order
            const int nlf = (info >> 4) & 7, mid = (info >> LDG_FACE_MAP_SHIFT) & 0xffff;
            const int n1 = t->n1, nfn_ = nd == 3 ? n1 * n1 : n1;
            const int nax = axis_of(nlf);
            bool ident = true;
            for (int tt = 0; tt < nfn_ && ident; ++tt) {
              const int v = t->nmap[(size_t)mid * nfn_ + tt];
              const int i = v % n1, j = (v / n1) % n1, k = v / (n1 * n1);
              const int tn = nd == 3 ? (nax == 0 ? j + n1 * k : (nax == 1 ? i + n1 * k : i + n1 * j))
                                     : (nax == 0 ? v / n1 : v % n1);
              ident = tn == tt;
            }
            if (ident) info = (int32_t)((uint32_t)info | LDG_FL_XIDENT);
          }
          if (!gc && (sw == right)) info |= LDG_FL_QOWN;
          if (gc) info |= LDG_FL_QHALF;
          if (gc || (sw != right)) info |= LDG_FL_COMPLETE;
          rec[2 * x] = beta * sj * t->ftau[x];
        } else if (kind == LDG_FACE_DIRICHLET) {
          acode = 1;
          rec[2 * x] = sj * t->ftau[x];
        } else {
          rec[2 * x] = sj;                      // Neumann: + sJ g
        }
        info |= acode << LDG_FL_ALPHA_SHIFT;
        int32_t pair[2] = {t->fnbr[x], info};
        memcpy(&rec[2 * x + 1], pair, sizeof(pair));
      }
    }
    rc |= upload(&h->frec, rec.data(), rec.size(), "frec");
    h_rec_host.swap(rec);
    rc |= upload(&h->kco, kco.data(), kco.size(), "kco");
    h->kstride = kst;
    // diagonal C blocks (ncu = 1): the plane kernel scales instead of mixing.
    // Off-diagonals at roundoff level of the diagonal (the reference's
    // Jacobian inversion leaves ~1e-16 relative entries on axis-aligned
    // boxes, growing with the element count: 1.2e-14 at 108^3) count as
    // zero: dropping them moves R by <= ~1e-13 relative, an order below the
    // 1e-12 parity bar.
    bool diag = ncu == 1;
    for (size_t e = 0; e < ne && diag; ++e) {
      const double* C = kco.data() + e * kst;
      for (int r = 0; r < nd && diag; ++r)
        for (int s2 = 0; s2 < nd; ++s2)
          if (r != s2 && !(fabs(C[r * nd + s2]) <= 1e-13 * sqrt(fabs(C[r * nd + r] * C[s2 * nd + s2])))) {
            diag = false;
            break;
          }
    }
    h->c_diag = diag ? 1 : 0;
  }
  cudaError_t e = cudaMalloc(&h->bad, sizeof(unsigned long long));
  if (e != cudaSuccess) rc |= fail(3, "bad flag", e);
  else cudaMemset(h->bad, 0xff, sizeof(unsigned long long));
  if (rc) {
    ldg_destroy(h);
    return 3;
  }
  ldg::TensorParams& P = h->P;
  P.ne = t->ne; P.nd = t->nd; P.n1 = t->n1; P.ncu = t->ncu;
  P.trace_centered = t->trace_centered;
  P.grad_centered = t->grad_centered;
  P.flux_uses_u = t->flux_uses_u;
  P.n_maps = t->n_maps;
  P.geo = h->geo; P.fnbr = h->fnbr; P.finfo = h->finfo; P.ftau = h->ftau;
  P.nmap = h->nmap; P.bad = h->bad; P.frec = h->frec; P.kco = h->kco; P.kstride = h->kstride;
  P.c_diag = h->c_diag;
  P.variant = 0;
  P.p2_mode = 0;
  P.e0 = 0;
  P.e1 = t->ne;
  P.x_consumer = 1;
  {
    // chunk-interleaved schedule of the fused operator (ldg_fused.cu run_fused):
    // chunk_dep[c] = last chunk whose exports pass 2 of chunk c reads
    const int nch = 1;                 // measured: chunking loses (launch tails outweigh L2 reuse)
    const int ne = t->ne, nf = 2 * t->nd;
    P.nchunk = nch;
    for (int c = 0; c <= nch; ++c) {
      long long b = (long long)ne * c / nch;
      b = (b + 31) / 32 * 32;
      P.chunk_start[c] = c == nch ? ne : (int)(b < ne ? b : ne);
    }
    std::vector<int> dep(nch, 0);
    int c = 0;
    for (int e = 0; e < ne; ++e) {
      while (e >= P.chunk_start[c + 1]) ++c;
      dep[c] = dep[c] > c ? dep[c] : c;
      for (int lf = 0; lf < nf; ++lf) {
        int32_t pair[2];
        memcpy(pair, &h_rec_host[(size_t)(e * nf + lf) * 2 + 1], sizeof(pair));
        const int info = pair[1];
        if ((info & LDG_FACE_KIND_MASK) != LDG_FACE_INTERIOR || !(info & LDG_FL_COMPLETE)) continue;
        const int nb = pair[0];
        int cn = 0;
        while (nb >= P.chunk_start[cn + 1]) ++cn;
        dep[c] = dep[c] > cn ? dep[c] : cn;
      }
    }
    for (int k = 0; k < nch; ++k) P.chunk_dep[k] = dep[k];
  }
  P.fused = 0;
  P.fuse = nullptr;
  P.fuse_dep = nullptr;
  P.fuse_nwin = 0;
  if (t->nd == 3 && t->n1 == 4 && t->ncu == 1 && t->ne > 0) {
    // one-launch operator: for each 8-element group the range of 32-group
    // windows whose pass 1 its pass 2 reads (its own R rows, the exports of
    // the neighbours across its completion faces)
    const int ne = t->ne, ng = (ne + 7) / 8, nwin = (ng + 31) / 32;
    std::vector<int2> gdep(ng);
    for (int g = 0; g < ng; ++g) {
      int lo = g >> 5, hi = g >> 5;
      for (int e = 8 * g; e < std::min(ne, 8 * g + 8); ++e)
        for (int lf = 0; lf < 6; ++lf) {
          int32_t pair[2];
          memcpy(pair, &h_rec_host[(size_t)(e * 6 + lf) * 2 + 1], sizeof(pair));
          if ((pair[1] & LDG_FACE_KIND_MASK) != LDG_FACE_INTERIOR || !(pair[1] & LDG_FL_COMPLETE)) continue;
          const int w = (pair[0] / 8) >> 5;
          lo = std::min(lo, w);
          hi = std::max(hi, w);
        }
      gdep[g] = make_int2(lo, hi);
    }
    int* ctr = nullptr;
    int2* d = nullptr;
    if (cudaMalloc(&ctr, (3 + nwin) * sizeof(int)) == cudaSuccess &&
        cudaMalloc(&d, ng * sizeof(int2)) == cudaSuccess &&
        cudaMemset(ctr, 0, (3 + nwin) * sizeof(int)) == cudaSuccess &&
        cudaMemcpy(d, gdep.data(), ng * sizeof(int2), cudaMemcpyHostToDevice) == cudaSuccess) {
      h->fuse = ctr;
      h->fuse_dep = d;
      P.fuse = ctr;
      P.fuse_dep = d;
      P.fuse_nwin = nwin;
      P.fused = LDG_FUSED_DEFAULT;
    } else {
      cudaFree(ctr);
      cudaFree(d);
      cudaGetLastError();
    }
  }
  const int n1 = t->n1;
  // tables arrive with row stride n1 packed at the front of each array
  memcpy(P.d1, t->d1, sizeof(P.d1));
  memcpy(P.m1, t->m1, sizeof(P.m1));
  memcpy(P.s1, t->s1, sizeof(P.s1));
  memcpy(P.clo, t->clo, sizeof(P.clo));
  memcpy(P.chi, t->chi, sizeof(P.chi));
  memcpy(P.au, t->au, sizeof(P.au));
  memcpy(P.aq, t->aq, sizeof(P.aq));
  memcpy(P.mass_coef, t->mass_coef, sizeof(P.mass_coef));
  // 1D mass inverse (Gauss-Jordan, n1 <= 9) for the block mass inverse
  double a[LDG_MAX_N1][2 * LDG_MAX_N1];
  for (int r = 0; r < n1; ++r)
    for (int c = 0; c < 2 * n1; ++c)
      a[r][c] = c < n1 ? t->m1[r * n1 + c] : (c - n1 == r ? 1.0 : 0.0);
  for (int c = 0; c < n1; ++c) {
    int piv = c;
    for (int r = c + 1; r < n1; ++r)
      if (fabs(a[r][c]) > fabs(a[piv][c])) piv = r;
    for (int k = 0; k < 2 * n1; ++k) { double tmp = a[c][k]; a[c][k] = a[piv][k]; a[piv][k] = tmp; }
    const double d = a[c][c];
    for (int k = 0; k < 2 * n1; ++k) a[c][k] /= d;
    for (int r = 0; r < n1; ++r)
      if (r != c) {
        const double f = a[r][c];
        for (int k = 0; k < 2 * n1; ++k) a[r][k] -= f * a[c][k];
      }
  }
  for (int r = 0; r < n1; ++r)
    for (int c = 0; c < n1; ++c) P.m1inv[r * n1 + c] = a[r][n1 + c];
  for (int r = 0; r < n1; ++r)
    for (int c = 0; c < n1; ++c) {
      double v = 0.0;
      for (int m = 0; m < n1; ++m) v += P.m1inv[r * n1 + m] * t->s1[m * n1 + c];
      P.g1[r * n1 + c] = v;
    }
  for (int r = 0; r < n1; ++r) {
    double gl = 0.0, gh = 0.0;
    for (int m = 0; m < n1; ++m) {
      gl += P.g1[r * n1 + m] * P.clo[m];
      gh += P.g1[r * n1 + m] * P.chi[m];
    }
    P.gclo[r] = gl;
    P.gchi[r] = gh;
    for (int c = 0; c < n1; ++c) {
      double v = 0.0;
      for (int m = 0; m < n1; ++m) v += P.g1[r * n1 + m] * P.d1[m * n1 + c];
      P.gd1[r * n1 + c] = v;
    }
  }
  *out = h;
  return 0;
}

int ldg_destroy(LdgHandle* h) {
  if (!h) return 0;
  ldg_comm_destroy(h);                   // the handle's communicator / halo plan, if any
  for (void* p : h->dense_bufs) cudaFree(p);
  cudaFree(h->geo); cudaFree(h->fnbr); cudaFree(h->finfo); cudaFree(h->ftau);
  cudaFree(h->nmap); cudaFree(h->frec); cudaFree(h->kco); cudaFree(h->bad);
  cudaFree(h->fuse); cudaFree(h->fuse_dep);
  for (auto e : h->ev_in) cudaEventDestroy(e);
  for (auto e : h->ev_p2) cudaEventDestroy(e);
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  if (h->s_in) cudaStreamDestroy(h->s_in);
  if (h->s_out) cudaStreamDestroy(h->s_out);
  delete h;
  return 0;
}

int ldg_create_dense(const LdgDenseTables* t, LdgHandle** out) {
  if (!t || !out) return fail(2, "null argument");
  if (t->nd < 2 || t->nd > 3 || t->ncu < 1 || t->ncu > LDG_MAX_NCU || t->ne < 0)
    return fail(2, "unsupported dense configuration");
  LdgHandle* h = new LdgHandle();
  h->dense = 1;
  memset(&h->D, 0, sizeof(h->D));
  memset(&h->P, 0, sizeof(h->P));
  h->P.ghost0 = INT32_MAX;
  ldg::DenseParams& D = h->D;
  D.ghost0 = INT32_MAX;
  D.ne = t->ne; D.nd = t->nd; D.nb = t->nb; D.nqf = t->nqf; D.nface = t->nface;
  D.nperm = t->nperm; D.ncu = t->ncu; D.trace_centered = t->trace_centered;
  D.grad_centered = t->grad_centered; D.flux_uses_u = t->flux_uses_u;
  const size_t ne = t->ne, nf = t->nface, nb = t->nb, nq = t->nqf, nd = t->nd;
  int rc = 0;
  auto up = [&](const double* src, size_t n, const double** dst, const char* what) {
    double* d = nullptr;
    rc |= upload(&d, src, n, what);
    h->dense_bufs.push_back(d);
    *dst = d;
  };
  auto upi = [&](const int32_t* src, size_t n, const int32_t** dst, const char* what) {
    int32_t* d = nullptr;
    rc |= upload(&d, src, n, what);
    h->dense_bufs.push_back(d);
    *dst = d;
  };
  up(t->geo, ne * (1 + nd * nd), &D.geo, "geo");
  up(t->fnorm, ne * nf * nd, &D.fnorm, "fnorm");
  up(t->fsj, ne * nf, &D.fsj, "fsj");
  upi(t->fnbr, ne * nf, &D.fnbr, "fnbr");
  upi(t->finfo, ne * nf, &D.finfo, "finfo");
  up(t->ftau, ne * nf, &D.ftau, "ftau");
  // operators are stored with the thread index (node a / face point s)
  // fastest, so a warp's operator loads for a fixed contraction index are
  // contiguous rows (2 L1 wavefronts instead of up to 32): the last two
  // indices of every (.., row, col) table are swapped
  auto tr = [](const double* src, size_t nmat, size_t rows, size_t cols) {
    std::vector<double> o(nmat * rows * cols);
    for (size_t m = 0; m < nmat; ++m)
      for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < cols; ++c) o[(m * cols + c) * rows + r] = src[(m * rows + r) * cols + c];
    return o;
  };
  const auto drT = tr(t->dr, nd, nb, nb), krT = tr(t->kr, nd, nb, nb);
  const auto liftT = tr(t->lift, nf, nb, nq), foT = tr(t->fluxop, nf, nb, nq);
  const auto phifT = tr(t->phif, nf, nq, nb), phioT = tr(t->phio, nf * (size_t)t->nperm, nq, nb);
  up(drT.data(), drT.size(), &D.dr, "dr");
  up(krT.data(), krT.size(), &D.kr, "kr");
  up(liftT.data(), liftT.size(), &D.lift, "lift");
  up(foT.data(), foT.size(), &D.fluxop, "fluxop");
  up(phifT.data(), phifT.size(), &D.phif, "phif");
  up(phioT.data(), phioT.size(), &D.phio, "phio");
  cudaError_t e = cudaMalloc(&h->bad, sizeof(unsigned long long));
  if (e != cudaSuccess) rc |= fail(3, "bad flag", e);
  else cudaMemset(h->bad, 0xff, sizeof(unsigned long long));
  if (rc) {
    ldg_destroy(h);
    return 3;
  }
  D.bad = h->bad;
  memcpy(D.au, t->au, sizeof(D.au));
  memcpy(D.aq, t->aq, sizeof(D.aq));
  *out = h;
  return 0;
}

int ldg_set_export_layout(LdgHandle* h, int consumer) {
  if (!h || h->dense) return fail(2, "export layout applies to tensor handles");
  h->P.x_consumer = consumer ? 1 : 0;
  return 0;
}

// Partitioned operators: neighbour rows >= ghost0 come from u_ghost (the
// halo buffer) instead of the state vector, so the owned vector is used in
// place (no per-call copy into an owned+ghost array).  ghost0 < 0 resets.
int ldg_set_ghost_rows_dense(LdgHandle* h, int ghost0, const double* u_ghost,
                             const double* q_ghost) {
  if (!h || !h->dense) return fail(2, "dense handle expected");
  if (ghost0 >= 0 && (!u_ghost || !q_ghost)) return fail(2, "ghost rows need buffers");
  h->D.ghost0 = ghost0 < 0 ? INT32_MAX : ghost0;
  h->D.u_ghost = ghost0 < 0 ? nullptr : u_ghost;
  h->D.q_ghost = ghost0 < 0 ? nullptr : q_ghost;
  return 0;
}

int ldg_set_ghost_rows(LdgHandle* h, int ghost0, const double* u_ghost) {
  if (!h) return fail(2, "null handle");
  if (h->dense) return fail(2, "dense handles take ldg_set_ghost_rows_dense");
  if (ghost0 >= 0 && !u_ghost) return fail(2, "ghost rows need a buffer");
  h->P.ghost0 = ghost0 < 0 ? INT32_MAX : ghost0;
  h->P.u_ghost = ghost0 < 0 ? nullptr : u_ghost;
  return 0;
}

// Kernel-selection options of one handle (A/B measurements and tests; the
// defaults are the measured-best choices):
//   "pass1_variant" 0 plane kernel where it applies | 1 pencil kernel
//   "c_diag"        0 forces the general flux-coefficient branch
//   "p2_mode"       0 warp kernel + PDL | 1 without PDL | 2 block kernel | 3 one-shot
int ldg_set_option(LdgHandle* h, const char* name, int value) {
  if (!h || !name) return fail(2, "bad argument");
  if (h->dense) return fail(2, "options apply to tensor handles");
  if (!strcmp(name, "pass1_variant")) h->P.variant = value ? 1 : 0;
  else if (!strcmp(name, "c_diag")) h->P.c_diag = (value && h->c_diag) ? 1 : 0;
  else if (!strcmp(name, "fused")) h->P.fused = (value && h->P.fuse) ? 1 : 0;
  else if (!strcmp(name, "p2_mode")) {
    if (value < 0 || value > 3) return fail(2, "p2_mode is 0..3");
    h->P.p2_mode = value;
  } else return fail(2, "unknown option");
  return 0;
}

int64_t ldg_last_bad_element(LdgHandle* h) {
  unsigned long long v = ~0ull;
  if (cudaMemcpy(&v, h->bad, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
  cudaMemset(h->bad, 0xff, sizeof(unsigned long long));
  return v == ~0ull ? -1 : (int64_t)v;
}

int ldg_compute_mixed(LdgHandle* h, const double* u, const double* gproj,
                      double* q, void* stream) {
  NvtxRange nvtx_("ldg_compute_mixed");
  if (!h || !u || !q) return fail(2, "null argument");
  if (h->dense) {
    int rc = ldg::launch_dense(h->D, 0, u, gproj, nullptr, q, nullptr, (cudaStream_t)stream);
    return rc ? fail(rc, "dense compute_mixed launch", cudaGetLastError()) : 0;
  }
  int rc = ldg::launch_mixed(h->P, u, gproj, q, (cudaStream_t)stream);
  return rc ? fail(rc, "compute_mixed launch", cudaGetLastError()) : 0;
}

int64_t ldg_scratch_doubles(LdgHandle* h) {
  if (!h) return -1;
  if (h->dense) return (int64_t)h->D.ne * h->D.nb * h->D.ncu * h->D.nd;
  const int64_t nf = 2 * h->P.nd;
  int64_t nfn = h->P.nd == 3 ? (int64_t)h->P.n1 * h->P.n1 : h->P.n1;
  return (int64_t)h->P.ne * nf * nfn * h->P.ncu;
}

int ldg_residual(LdgHandle* h, const double* u, const double* gproj,
                 const double* bsrc, double* scratch, double* R, void* stream) {
  NvtxRange nvtx_("ldg_residual");
  if (!h || !u || !R || !scratch) return fail(2, "null argument");
  if (h->dense) {
    int rc = ldg::launch_dense(h->D, 1, u, gproj, bsrc, scratch, R, (cudaStream_t)stream);
    return rc ? fail(rc, "dense residual launch", cudaGetLastError()) : 0;
  }
  int rc = ldg::launch_fused(h->P, false, u, gproj, bsrc, R, scratch, (cudaStream_t)stream);
  return rc ? fail(rc, "residual launch", cudaGetLastError()) : 0;
}

int ldg_residual_tangent(LdgHandle* h, const double* du, double* scratch,
                         double* dR, void* stream) {
  NvtxRange nvtx_("ldg_residual_tangent");
  if (!h || !du || !scratch || !dR) return fail(2, "null argument");
  if (h->dense) {
    int rc = ldg::launch_dense(h->D, 2, du, nullptr, nullptr, scratch, dR, (cudaStream_t)stream);
    return rc ? fail(rc, "dense tangent launch", cudaGetLastError()) : 0;
  }
  int rc = ldg::launch_fused(h->P, true, du, nullptr, nullptr, dR, scratch,
                             (cudaStream_t)stream);
  return rc ? fail(rc, "residual_tangent launch", cudaGetLastError()) : 0;
}

// Block-Jacobi probes of one colour without a host round trip per direction
// (solver.py:327-334): for k < bs, v = unit probe k on the colour's members,
// col = J v (the handle's linear tangent), mats[:, :, k] <- col on the blocks.
int ldg_bj_probe_colour(LdgHandle* h, int64_t nblk, int bs, const int32_t* members,
                        int64_t nm, double* v, double* col, double* scratch, double* mats,
                        void* stream) {
  NvtxRange nvtx_("ldg_bj_probe_colour");
  if (!h || !v || !col || !scratch || !mats || bs < 1) return fail(2, "bad argument");
  for (int k = 0; k < bs; ++k) {
    int rc = ldg_bj_probe_vector(nblk, bs, members, nm, k, v, stream);
    if (rc) return fail(rc, "probe vector", cudaGetLastError());
    rc = ldg_residual_tangent(h, v, scratch, col, stream);
    if (rc) return rc;
    rc = ldg_bj_extract(bs, members, nm, k, col, mats, stream);
    if (rc) return fail(rc, "extract", cudaGetLastError());
  }
  return 0;
}

int ldg_operator_pass(LdgHandle* h, int pass, int tangent, const double* u,
                      const double* gproj, const double* bsrc, double* scratch,
                      double* R, void* stream) {
  NvtxRange nvtx_("ldg_operator_pass");
  if (!h || !u || !R || !scratch || pass < 1 || pass > 2) return fail(2, "bad argument");
  if (h->dense) return fail(2, "not available for simplex systems");
  int rc = ldg::launch_fused_pass(h->P, pass, tangent != 0, u, gproj, bsrc, R, scratch,
                                  (cudaStream_t)stream);
  return rc ? fail(rc, "operator pass launch", cudaGetLastError()) : 0;
}

int ldg_operator_pass_range(LdgHandle* h, int pass, int tangent, const double* u,
                            const double* gproj, const double* bsrc, double* scratch,
                            double* R, int e0, int e1, void* stream) {
  NvtxRange nvtx_("ldg_operator_pass_range");
  if (!h || !u || !R || !scratch || pass < 1 || pass > 2) return fail(2, "bad argument");
  if (h->dense) return fail(2, "not available for simplex systems");
  if (e0 < 0 || e1 > h->P.ne || e0 > e1) return fail(2, "element range out of bounds");
  if (e0 == e1) return 0;
  ldg::TensorParams Q = h->P;
  Q.e0 = e0;
  Q.e1 = e1;
  int rc = ldg::launch_fused_pass(Q, pass, tangent != 0, u, gproj, bsrc, R, scratch,
                                  (cudaStream_t)stream);
  return rc ? fail(rc, "operator pass launch", cudaGetLastError()) : 0;
}

// Host-resident operator call, chunk pipelined: H2D of the chunks on one copy
// stream, the two fused passes per chunk on `stream` once the rows of every
// neighbour chunk have arrived (chunk_dep), D2H of each finished chunk on a
// second copy stream, so PCIe in both directions overlaps the kernels and each
// other.  v_host / out_host: pinned host (ne, nb, ncu); v_dev / R_dev /
// scratch: device work buffers.  Returns when out_host holds the result.
int ldg_apply_host(LdgHandle* h, int tangent, const double* v_host, double* out_host,
                   double* v_dev, double* R_dev, double* scratch, const double* gproj,
                   const double* bsrc, int nchunk, const int32_t* starts,
                   const int32_t* dep, void* stream) {
  return ldg_apply_host_staged(h, tangent, v_host, nullptr, out_host, v_dev, R_dev, scratch,
                               gproj, bsrc, nchunk, starts, dep, stream);
}

// Same pipeline for a PAGEABLE input (a numpy array, the reference's calling
// convention, disc.py:588-593): each chunk is first copied into the pinned
// staging buffer `stage` by the OpenMP host threads, then sent; the copy of
// chunk c+1 on the host overlaps the H2D of chunk c and the kernels of the
// chunks already resident.  stage == NULL: v_host is pinned (ldg_apply_host).
int ldg_apply_host_staged(LdgHandle* h, int tangent, const double* v_host, double* stage,
                          double* out_host, double* v_dev, double* R_dev, double* scratch,
                          const double* gproj, const double* bsrc, int nchunk,
                          const int32_t* starts, const int32_t* dep, void* stream) {
  NvtxRange nvtx_("ldg_apply_host_staged");
  if (!h || !v_host || !out_host || !v_dev || !R_dev || !scratch || nchunk < 1 || !starts || !dep)
    return fail(2, "bad argument");
  if (h->dense) return fail(2, "not available for simplex systems");
  for (int c = 0; c < nchunk; ++c)
    if (dep[c] < c || dep[c] >= nchunk || starts[c + 1] < starts[c]) return fail(2, "bad chunk plan");
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->s_in) {
    cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming);
  }
  while ((int)h->ev_in.size() < nchunk) {
    cudaEvent_t a, b;
    cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
    h->ev_in.push_back(a);
    h->ev_p2.push_back(b);
  }
  const size_t row = (size_t)(h->P.nd == 3 ? h->P.n1 * h->P.n1 * h->P.n1 : h->P.n1 * h->P.n1) *
                     h->P.ncu;
  cudaEventRecord(h->ev_start, s);
  cudaStreamWaitEvent(h->s_in, h->ev_start, 0);
  int next1 = 0, next2 = 0;           // next chunk whose pass 1 / pass 2 is to be issued
  for (int c = 0; c < nchunk; ++c) {
    const size_t a = (size_t)starts[c] * row, n = (size_t)(starts[c + 1] - starts[c]) * row;
    const double* src = v_host + a;
    if (stage) {
      // 64 KB slices over the host threads: a ~7 MB chunk spreads over every
      // core (1 MB slices left most threads idle: memcpy bandwidth scales
      // with the threads copying)
      const int64_t slice = 1 << 13, ns = (int64_t)((n + slice - 1) / slice);
#pragma omp parallel for schedule(static)
      for (int64_t k = 0; k < ns; ++k) {
        const size_t o = (size_t)k * slice, m = std::min((size_t)slice, n - o);
        stage_copy(stage + a + o, v_host + a + o, m);
      }
      src = stage + a;
    }
    cudaMemcpyAsync(v_dev + a, src, n * sizeof(double), cudaMemcpyHostToDevice, h->s_in);
    cudaEventRecord(h->ev_in[c], h->s_in);
    // every pass whose inputs are now in flight can be queued
    while (next1 < nchunk && dep[next1] <= c) {
      cudaStreamWaitEvent(s, h->ev_in[dep[next1]], 0);
      ldg::TensorParams Q = h->P;
      Q.e0 = starts[next1];
      Q.e1 = starts[next1 + 1];
      int rc = ldg::launch_fused_pass(Q, 1, tangent != 0, v_dev, gproj, bsrc, R_dev, scratch, s);
      if (rc) return fail(rc, "pass 1 launch", cudaGetLastError());
      ++next1;
      while (next2 < next1 && dep[next2] < next1) {
        Q.e0 = starts[next2];
        Q.e1 = starts[next2 + 1];
        rc = ldg::launch_fused_pass(Q, 2, tangent != 0, v_dev, gproj, bsrc, R_dev, scratch, s);
        if (rc) return fail(rc, "pass 2 launch", cudaGetLastError());
        cudaEventRecord(h->ev_p2[next2], s);
        cudaStreamWaitEvent(h->s_out, h->ev_p2[next2], 0);
        const size_t a2 = (size_t)starts[next2] * row,
                     n2 = (size_t)(starts[next2 + 1] - starts[next2]) * row;
        cudaMemcpyAsync(out_host + a2, R_dev + a2, n2 * sizeof(double), cudaMemcpyDeviceToHost,
                        h->s_out);
        ++next2;
      }
    }
  }
  if (next2 != nchunk) return fail(2, "chunk plan left passes unissued");
  cudaError_t e = cudaStreamSynchronize(h->s_out);
  if (e != cudaSuccess) return fail(3, "host pipeline", e);
  return 0;
}

// Mean unit normal of each face over its quadrature points, in the
// reference's own operation order (disc.py:167-178, :122): the tangent
// einsum "qgd,sd,kgc->kqcs" as numpy evaluates it (per geometry node g a
// partial sum over d of (gd T) ho, the partials added in g order), the
// cross product a1 b2 - a2 b1 ..., the norm as a left-to-right sum of
// squares, n = nv / |nv| and the mean as a left-to-right sum divided by nq.
// Every operation is a single IEEE rounding (no contraction: host x86-64
// code without FMA), so near-tie faces -- whose n_bar . beta_hat sign only
// rounding decides (disc.py:285-287) -- get the reference's switch bit.
// Host memory; OpenMP over faces.
int ldg_face_nbar(int64_t nfaces, int nq, int ng, int nrd, int nc, const double* gd,
                  const double* T, const double* ho, double* nbar) {
  if (nfaces < 0 || nq <= 0 || ng <= 0 || nrd < 2 || nrd > 3 || nc != nrd ||
      (nfaces && (!gd || !T || !ho || !nbar)))
    return fail(2, "bad argument");
  const int ns = nrd - 1;
  std::vector<double> coef((size_t)nq * ng * nrd * ns);       // gd[q,g,d] * T[s,d]
  for (int q = 0; q < nq; ++q)
    for (int g = 0; g < ng; ++g)
      for (int d = 0; d < nrd; ++d)
        for (int sidx = 0; sidx < ns; ++sidx)
          coef[(((size_t)q * ng + g) * nrd + d) * ns + sidx] =
              gd[((size_t)q * ng + g) * nrd + d] * T[sidx * nrd + d];
  const double* cf = coef.data();
#pragma omp parallel for schedule(static)
  for (int64_t f = 0; f < nfaces; ++f) {
    const double* hf = ho + (size_t)f * ng * nc;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int q = 0; q < nq; ++q) {
      double t[3][2];                                          // t[c][s]
      for (int c = 0; c < nc; ++c)
        for (int sidx = 0; sidx < ns; ++sidx) {
          double out = 0.0;
          for (int g = 0; g < ng; ++g) {
            double part = 0.0;
            for (int d = 0; d < nrd; ++d) {
              const double prod = cf[(((size_t)q * ng + g) * nrd + d) * ns + sidx] * hf[g * nc + c];
              part = part + prod;
            }
            out = out + part;
          }
          t[c][sidx] = out;
        }
      double nv[3];
      if (nc == 2) {
        nv[0] = t[1][0];
        nv[1] = -t[0][0];
      } else {
        double a = t[1][0] * t[2][1], b = t[2][0] * t[1][1];
        nv[0] = a - b;
        a = t[2][0] * t[0][1]; b = t[0][0] * t[2][1];
        nv[1] = a - b;
        a = t[0][0] * t[1][1]; b = t[1][0] * t[0][1];
        nv[2] = a - b;
      }
      double ss = nv[0] * nv[0];
      for (int c = 1; c < nc; ++c) {
        const double sq = nv[c] * nv[c];
        ss = ss + sq;
      }
      const double mag = std::sqrt(ss);
      for (int c = 0; c < nc; ++c) {
        const double nn = nv[c] / mag;
        acc[c] = q ? acc[c] + nn : nn;
      }
    }
    for (int c = 0; c < nc; ++c) nbar[(size_t)f * nc + c] = acc[c] / (double)nq;
  }
  return 0;
}

// Greedy colouring of the distance-2 element graph (solver.py:355-378,
// driver.py:109-142): element v takes the smallest colour not used by an
// already coloured element within two face-neighbour hops, v = 0, 1, ... in
// order -- the reference's deterministic greedy on the squared adjacency.
int ldg_color_distance2(int64_t ne, int64_t nfaces, const int32_t* elem_l,
                        const int32_t* elem_r, int32_t* colors) {
  if (ne < 0 || nfaces < 0 || (nfaces && (!elem_l || !elem_r)) || (ne && !colors))
    return fail(2, "bad argument");
  std::vector<int64_t> deg(ne + 1, 0);
  for (int64_t f = 0; f < nfaces; ++f) {
    const int a = elem_l[f], b = elem_r[f];
    if (a < 0 || b < 0 || a >= ne || b >= ne) return fail(2, "face element out of range");
    if (a == b) continue;
    ++deg[a + 1];
    ++deg[b + 1];
  }
  for (int64_t v = 0; v < ne; ++v) deg[v + 1] += deg[v];
  std::vector<int32_t> adj(deg[ne]);
  std::vector<int64_t> fill(deg.begin(), deg.end() - 1);
  for (int64_t f = 0; f < nfaces; ++f) {
    const int a = elem_l[f], b = elem_r[f];
    if (a == b) continue;
    adj[fill[a]++] = b;
    adj[fill[b]++] = a;
  }
  std::vector<int64_t> stamp;                  // colour -> last element that saw it
  for (int64_t v = 0; v < ne; ++v) colors[v] = -1;
  for (int64_t v = 0; v < ne; ++v) {
    auto mark = [&](int64_t u) {
      if (u == v) return;
      const int c = colors[u];
      if (c < 0) return;
      if ((int64_t)stamp.size() <= c) stamp.resize(c + 1, -1);
      stamp[c] = v;
    };
    for (int64_t i = deg[v]; i < deg[v + 1]; ++i) {
      const int u = adj[i];
      mark(u);
      for (int64_t j = deg[u]; j < deg[u + 1]; ++j) mark(adj[j]);
    }
    int c = 0;
    while (c < (int)stamp.size() && stamp[c] == v) ++c;
    colors[v] = c;
  }
  return 0;
}

int ldg_flux_from_mixed(LdgHandle* h, int tangent, const double* u,
                        const double* q, const double* gproj,
                        const double* bsrc, double* R, void* stream) {
  if (!h || !u || !q || !R) return fail(2, "null argument");
  if (h->dense) {
    // the simplex path's second pass on its own (partitioned systems
    // exchange the ghost q rows between compute_mixed and this)
    int rc = ldg::launch_dense(h->D, tangent ? 4 : 3, u, gproj, bsrc, const_cast<double*>(q), R,
                               (cudaStream_t)stream);
    return rc ? fail(rc, "dense flux launch", cudaGetLastError()) : 0;
  }
  if (h->P.ghost0 != INT32_MAX) return fail(2, "the unfused flux pass has no ghost-row mode");
  int rc = ldg::launch_flux(h->P, tangent != 0, u, q, gproj, bsrc, R, (cudaStream_t)stream);
  return rc ? fail(rc, "flux launch", cudaGetLastError()) : 0;
}

int ldg_mass_apply(LdgHandle* h, const double* v, double scale, double* out,
                   void* stream) {
  if (!h || !v || !out) return fail(2, "null argument");
  if (h->dense) return fail(2, "not available for simplex systems");
  int rc = ldg::launch_mass(h->P, false, v, scale, out, (cudaStream_t)stream);
  return rc ? fail(rc, "mass launch", cudaGetLastError()) : 0;
}

int ldg_mass_inv_apply(LdgHandle* h, const double* v, double* out, void* stream) {
  if (!h || !v || !out) return fail(2, "null argument");
  if (h->dense) return fail(2, "not available for simplex systems");
  int rc = ldg::launch_mass(h->P, true, v, 1.0, out, (cudaStream_t)stream);
  return rc ? fail(rc, "mass inverse launch", cudaGetLastError()) : 0;
}

}  // extern "C"
