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
  // partitioned operators: neighbour rows >= ghost0 come from the halo
  // buffers (u_ghost / q_ghost, row nbr - ghost0); INT32_MAX: no ghosts
  int ghost0;
  const double* u_ghost;
  const double* q_ghost;
  double au[LDG_MAX_NCU * 3 * LDG_MAX_NCU];
  double aq[LDG_MAX_NCU * 3 * LDG_MAX_NCU * 3];
};

// start of neighbour element nbr's row (`row` doubles) of u (q when Q)
template <bool Q>
__device__ __forceinline__ const double* dense_nbr_row(const DenseParams& P, const double* base,
                                                       int nbr, int row) {
  return nbr >= P.ghost0 ? (Q ? P.q_ghost : P.u_ghost) + (size_t)(nbr - P.ghost0) * row
                         : base + (size_t)nbr * row;
}

// what: 0 mixed (q = compute_mixed(u, gval)), 1 residual, 2 tangent,
//       3 flux pass from a given q (residual), 4 flux pass (tangent)
int launch_dense(const DenseParams& P, int what, const double* u, const double* gval,
                 const double* bsrc, double* q, double* R, cudaStream_t s);

}  // namespace ldg
