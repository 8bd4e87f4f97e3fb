// Shared definitions for the dense (simplex) LDG kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "ldgb200.h"

namespace ldg {

struct DenseParams {
  int ne, nd, nb, nqf, nface, nperm, ncu;
  int trace_centered, grad_centered, flux_uses_u;
  const double* geo;      // (ne, 1+nd*nd)
  const double* fnorm;    // (ne, nface, nd) outward unit normals
  const double* fsj;      // (ne, nface) |t1 x t2|
  const int32_t* fnbr;
  const int32_t* finfo;   // bits: kind | side | switch | nbr face << 4 | orientation << 8
  const double* ftau;
  // device copies are stored TRANSPOSED in their last two indices (the
  // thread's row index fastest): dr/kr (nd, b, a), lift/fluxop (nface, s, a),
  // phif (nface, b, s), phio (nface, nperm, b, s)
  const double* dr;       // collocation derivatives
  const double* kr;       // int d_r phi_a phi_b
  const double* lift;     // M_ref^-1 Phi^T W
  const double* fluxop;   // Phi^T W
  const double* phif;     // own traces
  const double* phio;     // neighbour traces by orientation
  unsigned long long* bad;
  double au[LDG_MAX_NCU * 3 * LDG_MAX_NCU];
  double aq[LDG_MAX_NCU * 3 * LDG_MAX_NCU * 3];
};

// what: 0 mixed (q = compute_mixed(u, gval)), 1 residual, 2 tangent
int launch_dense(const DenseParams& P, int what, const double* u, const double* gval,
                 const double* bsrc, double* q, double* R, cudaStream_t s);

}  // namespace ldg
