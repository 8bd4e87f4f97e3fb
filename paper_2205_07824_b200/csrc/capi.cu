// C ABI of libldgb200.so: handle lifecycle and the operator entry points.
// See include/ldgb200.h for the reference interface each one replaces.

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
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
  ldg::TensorParams P;
  double* geo = nullptr;
  int32_t* fnbr = nullptr;
  int32_t* finfo = nullptr;
  double* ftau = nullptr;
  int32_t* nmap = nullptr;
  double* frec = nullptr;
  unsigned long long* bad = nullptr;
};

extern "C" {

int ldg_version(void) { return 1; }

const char* ldg_last_error(void) { return g_err.c_str(); }

int ldg_create(const LdgTables* t, LdgHandle** out) {
  if (!t || !out) return fail(2, "null argument");
  if (t->nd < 2 || t->nd > 3 || t->n1 < 2 || t->n1 > LDG_MAX_N1 || t->ncu < 1 ||
      t->ncu > LDG_MAX_NCU || t->ne < 0)
    return fail(2, "unsupported tensor configuration");
  LdgHandle* h = new LdgHandle();
  memset(&h->P, 0, sizeof(h->P));
  const size_t ne = (size_t)t->ne, nf = 2 * t->nd;
  size_t nfn = t->nd == 3 ? (size_t)t->n1 * t->n1 : (size_t)t->n1;
  int rc = 0;
  rc |= upload(&h->geo, t->geo, ne * (1 + t->nd * t->nd), "geo");
  rc |= upload(&h->fnbr, t->fnbr, ne * nf, "fnbr");
  rc |= upload(&h->finfo, t->finfo, ne * nf, "finfo");
  rc |= upload(&h->ftau, t->ftau, ne * nf, "ftau");
  rc |= upload(&h->nmap, t->nmap, (size_t)t->n_maps * nfn, "nmap");
  {
    // packed 16-byte face records {double tau; int32 nbr; int32 info}
    std::vector<double> rec(ne * nf * 2);
    for (size_t x = 0; x < ne * nf; ++x) {
      rec[2 * x] = t->ftau[x];
      int32_t pair[2] = {t->fnbr[x], t->finfo[x]};
      memcpy(&rec[2 * x + 1], pair, sizeof(pair));
    }
    rc |= upload(&h->frec, rec.data(), rec.size(), "frec");
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
  P.nmap = h->nmap; P.bad = h->bad; P.frec = h->frec;
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
  *out = h;
  return 0;
}

int ldg_destroy(LdgHandle* h) {
  if (!h) return 0;
  cudaFree(h->geo); cudaFree(h->fnbr); cudaFree(h->finfo); cudaFree(h->ftau);
  cudaFree(h->nmap); cudaFree(h->frec); cudaFree(h->bad);
  delete h;
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
  if (!h || !u || !q) return fail(2, "null argument");
  int rc = ldg::launch_mixed(h->P, u, gproj, q, (cudaStream_t)stream);
  return rc ? fail(rc, "compute_mixed launch", cudaGetLastError()) : 0;
}

int64_t ldg_scratch_doubles(LdgHandle* h) {
  if (!h) return -1;
  const int64_t nf = 2 * h->P.nd;
  int64_t nfn = h->P.nd == 3 ? (int64_t)h->P.n1 * h->P.n1 : h->P.n1;
  return (int64_t)h->P.ne * nf * nfn * h->P.ncu;
}

int ldg_residual(LdgHandle* h, const double* u, const double* gproj,
                 const double* bsrc, double* scratch, double* R, void* stream) {
  if (!h || !u || !R || !scratch) return fail(2, "null argument");
  int rc = ldg::launch_fused(h->P, false, u, gproj, bsrc, R, scratch, (cudaStream_t)stream);
  return rc ? fail(rc, "residual launch", cudaGetLastError()) : 0;
}

int ldg_residual_tangent(LdgHandle* h, const double* du, double* scratch,
                         double* dR, void* stream) {
  if (!h || !du || !scratch || !dR) return fail(2, "null argument");
  int rc = ldg::launch_fused(h->P, true, du, nullptr, nullptr, dR, scratch,
                             (cudaStream_t)stream);
  return rc ? fail(rc, "residual_tangent launch", cudaGetLastError()) : 0;
}

int ldg_operator_pass(LdgHandle* h, int pass, int tangent, const double* u,
                      const double* gproj, const double* bsrc, double* scratch,
                      double* R, void* stream) {
  if (!h || !u || !R || !scratch || pass < 1 || pass > 2) return fail(2, "bad argument");
  int rc = ldg::launch_fused_pass(h->P, pass, tangent != 0, u, gproj, bsrc, R, scratch,
                                  (cudaStream_t)stream);
  return rc ? fail(rc, "operator pass launch", cudaGetLastError()) : 0;
}

int ldg_flux_from_mixed(LdgHandle* h, int tangent, const double* u,
                        const double* q, const double* gproj,
                        const double* bsrc, double* R, void* stream) {
  if (!h || !u || !q || !R) return fail(2, "null argument");
  int rc = ldg::launch_flux(h->P, tangent != 0, u, q, gproj, bsrc, R, (cudaStream_t)stream);
  return rc ? fail(rc, "flux launch", cudaGetLastError()) : 0;
}

int ldg_mass_apply(LdgHandle* h, const double* v, double scale, double* out,
                   void* stream) {
  if (!h || !v || !out) return fail(2, "null argument");
  int rc = ldg::launch_mass(h->P, false, v, scale, out, (cudaStream_t)stream);
  return rc ? fail(rc, "mass launch", cudaGetLastError()) : 0;
}

int ldg_mass_inv_apply(LdgHandle* h, const double* v, double* out, void* stream) {
  if (!h || !v || !out) return fail(2, "null argument");
  int rc = ldg::launch_mass(h->P, true, v, 1.0, out, (cudaStream_t)stream);
  return rc ? fail(rc, "mass inverse launch", cudaGetLastError()) : 0;
}

}  // extern "C"
