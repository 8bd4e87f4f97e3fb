// Shared definitions for the tensor-product (quad/hex) LDG kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "ldgb200.h"

namespace ldg {

constexpr int LDG_MAX_CHUNKS = 16;

#ifndef LDG_FUSED_DEFAULT
#define LDG_FUSED_DEFAULT 0       // one-launch operator (ldg_set_option "fused")
#endif

// Operator data passed by value (__grid_constant__) to every launch.  The
// 1D tables are tiny and read uniformly across a warp, so they live in the
// kernel parameter bank (constant cache), which DFMA can consume directly.
struct TensorParams {
  int ne, nd, n1, ncu;
  int trace_centered, grad_centered, flux_uses_u;
  int n_maps;
  const double* geo;      // (ne, 1+nd*nd)
  const int32_t* fnbr;    // (ne, 2nd)
  const int32_t* finfo;   // (ne, 2nd)
  const double* ftau;     // (ne, 2nd)
  const int32_t* nmap;    // (n_maps, n1^(nd-1))
  const void* frec;       // (ne, 2nd) packed {sJ*tau, nbr, info|flags} records (16 B)
  const double* kco;      // (ne, kstride): C, Cu, sJ per face axis (fused kernels)
  int kstride;
  int variant;           // pass-1 kernel: 0 auto (plane kernel where it applies), 1 pencil kernel
  int p2_mode;           // pass-2 kernel: 0 auto (warp kernel + PDL), 1 no PDL, 2 block kernel,
                         // 3 one-shot block kernel (A/B through ldg_set_option)
  int e0, e1;            // element range of this launch (chunked schedules)
  int x_consumer;        // 1: exports land in the consuming neighbour's slots (pass 2 reads its own)
  int nchunk;            // > 1: residual / tangent run chunk-interleaved (L2-resident pass 2)
  int chunk_start[LDG_MAX_CHUNKS + 1];
  int chunk_dep[LDG_MAX_CHUNKS];   // last chunk whose pass 1 pass 2 of this chunk reads
  unsigned long long* bad;  // first non-finite element (atomicMin)
  // partitioned operators: neighbour rows >= ghost0 are read from u_ghost
  // (row nbr - ghost0) instead of u, so a rank's owned vector is used in
  // place and only the halo lands in a side buffer (INT32_MAX: no ghosts)
  int ghost0;
  const double* u_ghost;
  // one-launch operator (hex p = 3, ncu = 1): pass 1 and pass 2 in one
  // persistent kernel, pass 2 of a group as soon as the pass-1 windows it
  // reads are complete (ldg_fused.cu plane_kernel<.., FUSED>)
  int fused;              // 1: run_fused takes the one-launch kernel where it applies
  int* fuse;              // [0] pass-1 claims, [1] pass-2 claims, [2] exited warps, [3..) windows
  const int2* fuse_dep;   // per 8-element group: first / last 32-group window pass 2 reads
  int fuse_nwin;
  double d1[LDG_MAX_N1 * LDG_MAX_N1];
  double m1[LDG_MAX_N1 * LDG_MAX_N1];
  double s1[LDG_MAX_N1 * LDG_MAX_N1];
  double m1inv[LDG_MAX_N1 * LDG_MAX_N1];
  double g1[LDG_MAX_N1 * LDG_MAX_N1];   // M1^-1 S1: S1 (x) M1 (x) M1 = (M1 (x) M1 (x) M1)(G1 (x) I (x) I)
  double gd1[LDG_MAX_N1 * LDG_MAX_N1];  // G1 D1 (the volume term of -D u along one axis)
  double gclo[LDG_MAX_N1], gchi[LDG_MAX_N1];   // G1 clo, G1 chi (the volume term of the lifts)
  int c_diag;            // every element's C block is diagonal (axis-aligned affine hexes)
  double clo[LDG_MAX_N1];
  double chi[LDG_MAX_N1];
  double au[LDG_MAX_NCU * 3 * LDG_MAX_NCU];
  double aq[LDG_MAX_NCU * 3 * LDG_MAX_NCU * 3];
  double mass_coef[LDG_MAX_NCU];
};

// start of neighbour element `nbr`'s row (`row` doubles) of the state u
__device__ __forceinline__ const double* nbr_row(const TensorParams& P, const double* u, int nbr,
                                                 int row) {
  return nbr >= P.ghost0 ? P.u_ghost + (size_t)(nbr - P.ghost0) * row : u + (size_t)nbr * row;
}

// hex local faces (master.py:43-44): z-, z+, y-, y+, x-, x+
// quad local faces: y-, x+, y+, x-
__host__ __device__ constexpr int face_axis(int nd, int lf) {
  return nd == 3 ? (lf < 2 ? 2 : (lf < 4 ? 1 : 0))
                 : ((lf == 0 || lf == 2) ? 1 : 0);
}
__host__ __device__ constexpr int face_side(int nd, int lf) {
  return nd == 3 ? (lf & 1) : (lf == 1 || lf == 2 ? 1 : 0);
}

int launch_mixed(const TensorParams& P, const double* u, const double* gproj,
                 double* q, cudaStream_t s);
int launch_flux(const TensorParams& P, bool tangent, const double* u,
                const double* q, const double* gproj, const double* bsrc,
                double* R, cudaStream_t s);
int launch_fused(const TensorParams& P, bool tangent, const double* u,
                 const double* gproj, const double* bsrc, double* R, double* X,
                 cudaStream_t s);
int launch_fused_pass(const TensorParams& P, int pass, bool tangent, const double* u,
                      const double* gproj, const double* bsrc, double* R, double* X,
                      cudaStream_t s);
int launch_mass(const TensorParams& P, bool inverse, const double* v,
                double scale, double* out, cudaStream_t s);

}  // namespace ldg
