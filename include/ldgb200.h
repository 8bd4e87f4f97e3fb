/*
 * ldgb200.h -- C ABI of the B200 LDG hot path (libldgb200.so).
 *
 * The reference (ldgkit) is pure Python; its "FFI" for this path is the duck
 * typed LdgSystem / solver interface.  Each entry point below replaces one
 * reference call (file:line under /root/reference/pkg/src/ldgkit/):
 *
 *   ldg_compute_mixed        LdgSystem.compute_mixed          disc.py:436-490
 *   ldg_residual             LdgSystem.residual               disc.py:588-653
 *   ldg_residual_tangent     LdgSystem.residual_tangent       disc.py:591-593
 *   ldg_mass_apply           LdgSystem.mass_apply (const m)   disc.py:897-925
 *   ldg_mass_inv_apply       MassPreconditioner.apply         driver.py:99-106
 *   ldg_dot / ldg_nrm2 / ldg_axpy / ldg_scal / ldg_copy
 *                            numpy dot/norm/axpy in gmres     solver.py:98-145
 *   ldg_mgs_step             MGS dot+axpy pair                solver.py:130-138
 *   ldg_cgs_dots / ldg_cgs_update  block Gram-Schmidt (fast mode) solver.py:130-144
 *   ldg_dcgs_dots / ldg_dcgs_update  delayed-reorth Gram-Schmidt     solver.py:130-144
 *   ldg_combine              x += Z^T y                       solver.py:163-164
 *   ldg_color_distance2      greedy distance-2 colouring      solver.py:355-378
 *   ldg_face_nbar            mean face normal (switch bit)    disc.py:167-178, 122, 285-287
 *   ldg_bj_probe_vector      coloured unit probe              solver.py:327-330
 *   ldg_bj_extract           mats[b][:,k] = col[blocks[b]]    solver.py:331-334
 *   ldg_bj_invert            lu_factor (+1e-12 shift rule)    solver.py:335-345
 *   ldg_bj_apply             BlockJacobiPreconditioner.apply  solver.py:296-300
 *   ldg_bj_apply_tiles       same, blocks shared by element classes
 *   ldg_jit_*                NVRTC modules of the generated kernels (nonlinear
 *                            models, disc.py:436-948; the volume source load
 *                            disc.py:621-629)
 *   ldg_probe_fp64           measurement helper (FP64 FMA peak), no counterpart
 *   ldg_comm_* / ldg_set_halo_plan / ldg_apply_dist
 *                            multi-GPU boundary (SURVEY 8(b) "ldg_comm_init(ncclComm_t,
 *                            partition), halo exchange inside the matvec"); the
 *                            reference is single-process (no counterpart)
 *
 * Conventions: every double* / int* argument is DEVICE memory owned by the
 * caller (PyTorch tensors on the host side); the handle owns only the
 * immutable connectivity / geometry tables uploaded by ldg_create.  All work
 * is enqueued on `stream` (a cudaStream_t passed as void*).  Return codes:
 * 0 success, 1 non-finite output (first bad element via ldg_last_bad_element),
 * 2 invalid argument / unsupported configuration, >=3 CUDA error.
 */
#ifndef LDGB200_H
#define LDGB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LDG_MAX_N1 9
#define LDG_MAX_NCU 5

/* element-face info bits (LdgTables.finfo) */
#define LDG_FACE_INTERIOR 0
#define LDG_FACE_DIRICHLET 1
#define LDG_FACE_NEUMANN 2
#define LDG_FACE_KIND_MASK 3
#define LDG_FACE_SIDE_RIGHT 4   /* this element is the right side of the face */
#define LDG_FACE_SWITCH 8       /* face switch bit (disc.py:287) */
#define LDG_FACE_MAP_SHIFT 8    /* bits 8..23: neighbour node map id */
/* bits 4..6: the neighbour's local face.  Bits 24..28 are derived flags
 * ldg_create adds from the trace rules (callers pass them as zero). */
#define LDG_FL_UNBR (1 << 24)      /* u^ or the penalty reads the neighbour */
#define LDG_FL_EXPORT (1 << 25)    /* neighbour takes (part of) q^ from this side */
#define LDG_FL_QOWN (1 << 26)      /* q^ = this side's q */
#define LDG_FL_QHALF (1 << 27)     /* q^ centered: half from each side */
#define LDG_FL_COMPLETE (1 << 28)  /* pass 2 adds the neighbour share */
#define LDG_FL_ALPHA_SHIFT 29      /* bits 29..30: jump coefficient 0 | 1 | 1/2 */
#define LDG_FL_XIDENT (1u << 31)   /* the neighbour's face-node order equals this face's */

/* Host-side description of a tensor-product (quad/hex) kind-D system with a
 * flux that is linear in (u, q) with constant coefficients.  Pointers are
 * HOST memory; ldg_create copies them to the device. */
typedef struct LdgTables {
  int32_t nd;            /* 2 or 3 */
  int32_t n1;            /* nodes per direction, p+1 */
  int32_t ncu;           /* state components */
  int32_t ne;            /* elements */
  int32_t n_maps;        /* distinct neighbour node maps */
  int32_t trace_centered;   /* numflux.trace == 'centered'      */
  int32_t grad_centered;    /* numflux.grad_trace == 'centered' */
  int32_t flux_uses_u;      /* any Au coefficient nonzero        */
  const double* geo;     /* (ne, 1 + nd*nd): detJ, invjt[d][r]            */
  const int32_t* fnbr;   /* (ne, 2*nd): neighbour element / boundary row  */
  const int32_t* finfo;  /* (ne, 2*nd): LDG_FACE_* bits                   */
  const double* ftau;    /* (ne, 2*nd): penalty tau on this face          */
  const int32_t* nmap;   /* (n_maps, n1^(nd-1)): own face node -> nbr node */
  double d1[LDG_MAX_N1 * LDG_MAX_N1];  /* GLL collocation derivative D[i][m]  */
  double m1[LDG_MAX_N1 * LDG_MAX_N1];  /* 1D mass   M[a][b] = int l_a l_b      */
  double s1[LDG_MAX_N1 * LDG_MAX_N1];  /* 1D stiff. S[a][b] = int l'_a l_b     */
  double clo[LDG_MAX_N1];              /* M^-1 e_0                           */
  double chi[LDG_MAX_N1];              /* M^-1 e_{n1-1}                      */
  double au[LDG_MAX_NCU * 3 * LDG_MAX_NCU];       /* f_cd += au[c][d][k] u_k  */
  double aq[LDG_MAX_NCU * 3 * LDG_MAX_NCU * 3];   /* f_cd += aq[c][d][k][e] q_ke */
  double mass_coef[LDG_MAX_NCU];       /* constant mass m_c (disc.py:902-906) */
} LdgTables;

/* Host-side description of a simplex (tri / tet) kind-D system for the
 * dense-tabulation kernels (csrc/ldg_dense.cu).  Pointers are HOST memory. */
typedef struct LdgDenseTables {
  int32_t nd, nb, nqf, nface, nperm, ncu, ne;
  int32_t trace_centered, grad_centered, flux_uses_u;
  const double* geo;      /* (ne, 1 + nd*nd)                                 */
  const double* fnorm;    /* (ne, nface, nd) outward unit face normals        */
  const double* fsj;      /* (ne, nface) |t1 x t2| of each (affine) face      */
  const int32_t* fnbr;    /* (ne, nface) neighbour element / boundary row     */
  const int32_t* finfo;   /* (ne, nface) kind|side|switch|nbr face<<4|orient<<8 */
  const double* ftau;     /* (ne, nface) penalty                              */
  const double* dr;       /* (nd, nb, nb) collocation derivative matrices     */
  const double* kr;       /* (nd, nb, nb) int d_r phi_a phi_b                 */
  const double* lift;     /* (nface, nb, nqf) M_ref^-1 Phi^T W                */
  const double* fluxop;   /* (nface, nb, nqf) Phi^T W                         */
  const double* phif;     /* (nface, nqf, nb) own face traces                 */
  const double* phio;     /* (nface, nperm, nqf, nb) neighbour traces         */
  double au[LDG_MAX_NCU * 3 * LDG_MAX_NCU];
  double aq[LDG_MAX_NCU * 3 * LDG_MAX_NCU * 3];
} LdgDenseTables;

typedef struct LdgHandle LdgHandle;

int ldg_create(const LdgTables* host, LdgHandle** out);
/* Simplex systems: same entry points below (compute_mixed, residual,
 * residual_tangent); boundary data are values at face quadrature points,
 * (n_bfaces, nqf, ncu); scratch holds q, ne*nb*ncu*nd doubles. */
int ldg_create_dense(const LdgDenseTables* host, LdgHandle** out);
int ldg_destroy(LdgHandle* h);
int64_t ldg_last_bad_element(LdgHandle* h);
const char* ldg_last_error(void);
int ldg_version(void);

/* q = M^-1 [ -int grad(u) phi + oint (u - u^) n phi ]   (disc.py:436-490)
 * gproj: (n_bfaces, n1^(nd-1), ncu) projected Dirichlet data, or NULL for
 * the homogeneous linearisation.  q layout (ne, nb, ncu, nd). */
int ldg_compute_mixed(LdgHandle* h, const double* u, const double* gproj,
                      double* q, void* stream);

/* Device scratch (doubles) the residual / tangent calls need: the face
 * export buffer of the fused operator, ne * 2nd * n1^(nd-1) * ncu. */
int64_t ldg_scratch_doubles(LdgHandle* h);

/* Where pass 1 writes the face exports: 1 (default) into the consuming
 * neighbour's own (element, face) slots in its face-node order, so pass 2
 * reads its slots without a gather; 0 into the producer's slots (the
 * partitioned layer exchanges producer rows between ranks). */
int ldg_set_export_layout(LdgHandle* h, int consumer);

/* R(u) (disc.py:588-653) by the fused two-pass operator (ldg_fused.cu):
 * the mixed gradient never leaves the SM.  gproj: projected Dirichlet /
 * Neumann data (n_bfaces, n1^(nd-1), ncu) or NULL for zero data; bsrc
 * (ne, nb, ncu) = -int s(x,t) phi or NULL. */
int ldg_residual(LdgHandle* h, const double* u, const double* gproj,
                 const double* bsrc, double* scratch, double* R, void* stream);

/* dR = J(u) du with the reference linearisation (disc.py:591-604: frozen
 * tau, homogeneous Dirichlet lift, zero Neumann tangent).  Fluxes linear in
 * (u, q) with constant coefficients do not read the base state. */
int ldg_residual_tangent(LdgHandle* h, const double* du, double* scratch,
                         double* dR, void* stream);

/* One pass of the fused operator (1 = element pass, 2 = face completion),
 * for per-kernel timing; ldg_residual(_tangent) = pass 1 then pass 2. */
int ldg_operator_pass(LdgHandle* h, int pass, int tangent, const double* u,
                      const double* gproj, const double* bsrc, double* scratch,
                      double* R, void* stream);

/* The same pass over elements [e0, e1) only (chunk-pipelined host calls:
 * H2D of later chunks and D2H of finished ones overlap the kernels). */
int ldg_operator_pass_range(LdgHandle* h, int pass, int tangent, const double* u,
                            const double* gproj, const double* bsrc, double* scratch,
                            double* R, int e0, int e1, void* stream);

/* LdgSystem.residual / residual_tangent (disc.py:588-593) on HOST data:
 * v_host, out_host pinned (ne, nb, ncu).  Chunk-pipelined (chunk bounds
 * `starts` (nchunk + 1), per chunk the last chunk holding a face neighbour
 * `dep`): H2D, the two fused passes and D2H overlap.  Blocks until out_host
 * is written.  tangent = 0 evaluates R(v) with gproj / bsrc. */
int ldg_apply_host(LdgHandle* h, int tangent, const double* v_host, double* out_host,
                   double* v_dev, double* R_dev, double* scratch, const double* gproj,
                   const double* bsrc, int nchunk, const int32_t* starts,
                   const int32_t* dep, void* stream);

/* ldg_apply_host for a PAGEABLE v_host (a numpy array: the reference's
 * calling convention, ldgkit/disc.py:588-593): each chunk is copied into the
 * pinned staging buffer `stage` (ne * nb * ncu doubles) by the host threads
 * (OpenMP) and sent while the next chunk is staged.  out_host stays pinned.
 * stage == NULL behaves exactly like ldg_apply_host. */
int ldg_apply_host_staged(LdgHandle* h, int tangent, const double* v_host, double* stage,
                          double* out_host, double* v_dev, double* R_dev, double* scratch,
                          const double* gproj, const double* bsrc, int nchunk,
                          const int32_t* starts, const int32_t* dep, void* stream);

/* Partitioned operators: neighbour element rows >= ghost0 are
 * read from u_ghost (row nbr - ghost0) instead of the state vector, so a
 * rank's owned vector is used in place and only the halo lands in the side
 * buffer.  ghost0 < 0 switches it off.  (Reference: none -- the reference is
 * single-process; this is the B200 multi-GPU layer.) */
int ldg_set_ghost_rows(LdgHandle* h, int ghost0, const double* u_ghost);
/* the same for simplex (dense) handles: ghost rows of u and of the mixed
 * gradient q (the flux pass reads the neighbours' q) */
int ldg_set_ghost_rows_dense(LdgHandle* h, int ghost0, const double* u_ghost,
                             const double* q_ghost);

/* Kernel-selection options of a tensor handle (A/B measurements, tests);
 * the defaults are the measured-best choices: "pass1_variant" (0 plane |
 * 1 pencil), "c_diag" (0 forces the general flux-coefficient branch),
 * "p2_mode" (0 warp + PDL | 1 no PDL | 2 block | 3 one-shot), "fused"
 * (1: hex p = 3 passes 1 and 2 in one persistent launch; measured slower,
 * off).  No reference counterpart. */
int ldg_set_option(LdgHandle* h, const char* name, int value);

/* Unfused reference structure, kept for comparison: flux pass from a
 * precomputed q = compute_mixed(u) (72 B/DOF of HBM traffic at nd = 3); on
 * simplex handles the dense flux pass (disc.py:595-653 given q). */
int ldg_flux_from_mixed(LdgHandle* h, int tangent, const double* u,
                        const double* q, const double* gproj,
                        const double* bsrc, double* R, void* stream);

/* constant-mass operator and its block inverse (element mass M_e =
 * detJ * M1 (x) M1 (x) M1) */
int ldg_mass_apply(LdgHandle* h, const double* v, double scale, double* out,
                   void* stream);
int ldg_mass_inv_apply(LdgHandle* h, const double* v, double* out, void* stream);

/* ---- Krylov vector primitives (deterministic fixed-order reductions) ---- */
/* scratch: >= ldg_reduce_scratch_doubles() doubles; result written to out[0] */
int64_t ldg_reduce_scratch_doubles(void);
int ldg_dot(int64_t n, const double* x, const double* y, double* scratch,
            double* out, void* stream);
int ldg_nrm2(int64_t n, const double* x, double* scratch, double* out,
             void* stream);
/* y = a*x + y with a = sign * (*a_dev) (device scalar) or a_host if a_dev NULL */
int ldg_axpy(int64_t n, double a_host, const double* a_dev, double sign,
             const double* x, double* y, void* stream);
/* y = x * (1 / *den_dev)  (reference: V[k+1] = w / H[k+1,k]) */
int ldg_div_scalar(int64_t n, const double* x, const double* den_dev, double* y,
                   void* stream);
/* y = x / *den where *den > thr, y untouched otherwise (a NaN den included):
 * the DCGS2 normalisation without reading den on the host (solver.py:142's
 * breakdown test is taken on the host one dot sweep later) */
int ldg_div_scalar_guarded(int64_t n, const double* x, const double* den, double thr,
                           double* y, void* stream);
/* fused MGS step: w -= h_in * Vi ; h_out = <Vnext, w> (Vnext may be NULL) */
int ldg_mgs_step(int64_t n, const double* vi, const double* h_in, double* w,
                 const double* vnext, double* scratch, double* h_out,
                 void* stream);
/* h[i] = <V_i, w> for i < k (V rows of length n, row stride ldv) */
int ldg_cgs_dots(int64_t n, int k, const double* V, int64_t ldv, const double* w,
                 double* scratch, double* h, void* stream);
/* w -= sum_i h[i] V_i ; nrm_out = ||w|| */
int ldg_cgs_update(int64_t n, int k, const double* V, int64_t ldv,
                   const double* h, double* w, double* scratch, double* nrm_out,
                   void* stream);
/* x += sum_i y[i] Z_i  (y device) */
int ldg_combine(int64_t n, int k, const double* Z, int64_t ldz, const double* y,
                double* x, void* stream);

/* ---- setup (HOST memory) ---- */
/* mean unit normal over the nq quadrature points of each face, in the
 * reference's operation order (bit-identical to its tangent einsum / cross /
 * norm / mean): gd (nq, ng, nrd) geometry-basis gradients at the face points,
 * T (nrd-1, nrd) face embedding, ho (nfaces, ng, nc) the left elements'
 * geometry nodes -> nbar (nfaces, nc); nc == nrd in {2, 3} */
int ldg_face_nbar(int64_t nfaces, int nq, int ng, int nrd, int nc, const double* gd,
                  const double* T, const double* ho, double* nbar);

/* ---- block-Jacobi ---- */
/* greedy distance-2 colouring of the element graph given by the interior
 * faces (elem_l, elem_r) (solver.py:355-378, driver.py:109-142) */
int ldg_color_distance2(int64_t ne, int64_t nfaces, const int32_t* elem_l,
                        const int32_t* elem_r, int32_t* colors);
/* all bs probes of one colour through the handle's linear tangent: for each
 * k, v = unit probe k, col = J v, extract into mats (solver.py:327-334) */
int ldg_bj_probe_colour(LdgHandle* h, int64_t nblk, int bs, const int32_t* members,
                        int64_t nm, double* v, double* col, double* scratch, double* mats,
                        void* stream);
int ldg_bj_probe_vector(int64_t nblk, int bs, const int32_t* members,
                        int64_t n_members, int k, double* v, void* stream);
int ldg_bj_extract(int bs, const int32_t* members, int64_t n_members, int k,
                   const double* col, double* mats, void* stream);
/* mats (nblk, bs, bs) row-major -> inv_t (nblk, bs, bs) holding inverse^T;
 * shifted (nblk) int flags: 1 where the 1e-12 shift rule fired
 * (solver.py:336-346: lu_factor, shift, lu_solve).  Any bs: blocks up to 160
 * in shared memory, larger ones through ldg_bj_invert_global. */
int ldg_bj_invert(int64_t nblk, int bs, const double* mats, double* inv_t,
                  int32_t* shifted, void* stream);
/* the same Gauss-Jordan on a global (L2-resident) working copy, any bs */
int ldg_bj_invert_global(int64_t nblk, int bs, const double* mats, double* inv_t,
                         int32_t* shifted, void* stream);
int ldg_bj_apply(int64_t nblk, int bs, const double* inv_t, const double* r,
                 double* z, void* stream);
/* BlockJacobiPreconditioner.apply (solver.py:296-300) with the inverses
 * shared by classes of elements whose blocks are bit-identical (interior
 * elements of one geometry class on structured meshes): tile t applies
 * class tile_cls[t]'s inverse (inv_t: classes x bs x bs, transposed) to the
 * rows of up to ldg_bj_tile_elems() elements tile_el[t * E .. t * E + E)
 * (-1 = unused slot) */
int ldg_bj_tile_elems(void);
/* class detection: keys[2b, 2b+1] = two exact 64-bit hashes of block b's bit
 * pattern (wrapping sums, order-free); *bad = 1 unless every block is bit
 * for bit equal to block rep[b] (bad: device int, set by the caller to 0) */
int ldg_bj_block_keys(int64_t nblk, int bs, const double* mats, uint64_t* keys, void* stream);
int ldg_bj_class_verify(int64_t nblk, int bs, const double* mats, const int64_t* rep, int32_t* bad,
                        void* stream);
int ldg_bj_apply_tiles(int64_t ntiles, int bs, const double* inv_t, const int32_t* tile_cls,
                       const int32_t* tile_el, const double* r, double* z, void* stream);
/* element blocks across a packed (u | q | w) vector (driver.py:128-142,
 * _elementwise_blocks): idx[e*bs + j] = packed index of row j of block e;
 * gather dst[i] = src[idx[i]], scatter dst[idx[i]] = src[i] */
int ldg_permute_gather(int64_t n, const int64_t* idx, const double* src, double* dst,
                       void* stream);
int ldg_permute_scatter(int64_t n, const int64_t* idx, const double* src, double* dst,
                        void* stream);

/* ---- generated model kernels (nonlinear / kind-C path, csrc/jit.cu) ----
 * The pointwise flux / source / wavespeed / mass plans of a model
 * (expr.py:363-373, evaluated by disc.py:393-416 in the reference) are lowered
 * to CUDA device functions by paper_2205_07824_b200/codegen.py, spliced into
 * csrc/ldg_nl.cuh and compiled for sm_100a by NVRTC.  The loaded module's
 * kernels replace LdgSystem.compute_mixed / residual / residual_tangent /
 * mass_apply / mass_tangent_extra (disc.py:436-948) for models whose flux is
 * not linear with constant coefficients (Euler, Navier-Stokes, Burgers...).
 * Every kernel takes ONE parameter block by value; the caller packs it. */
typedef struct LdgModule LdgModule;
const char* ldg_jit_last_error(void);
/* compile only (no GPU needed): cubin_out NULL -> *cubin_size = bytes needed */
int ldg_jit_compile(const char* src, const char* name, const char* const* opts,
                    int nopts, void* cubin_out, int64_t* cubin_size);
int ldg_jit_load(const void* cubin, int64_t size, LdgModule** out);
int ldg_jit_unload(LdgModule* m);
int ldg_jit_launch(LdgModule* m, const char* kernel, int grid_x, int grid_y,
                   int block_x, int smem_bytes, const void* params,
                   int64_t param_size, void* stream);
int ldg_jit_attr(LdgModule* m, const char* kernel, int* regs, int* local_bytes,
                 int* static_smem);

/* DCGS2 orthogonalisation (delayed reorthogonalisation; solver.py:79-174's
 * two Gram-Schmidt passes folded into one dot sweep and one update sweep):
 * hx = V[0..k)^T x, hy = V[0..k)^T y in one sweep; then
 * v <- (v - V s) * inv_alpha, out <- (w - V t - gamma v) * inv_alpha,
 * nrm_out = ||out|| (V has m rows) */
int ldg_dcgs_dots(int64_t n, int k, const double* V, int64_t ldv, const double* x,
                  const double* y, double* scratch, double* hx, double* hy, void* stream);
int ldg_dcgs_update(int64_t n, int m, const double* V, int64_t ldv, const double* s,
                    const double* t, double* v, const double* w, double* out,
                    double inv_alpha, double gamma, double* scratch, double* nrm_out,
                    void* stream);

/* ---- measurement helper (no reference counterpart) ---- */
/* FP64 FMA throughput of the current GPU: 8 independent DFMA chains per
 * thread, 8 x 256-thread blocks per SM, `iters` FMAs per chain; returns
 * TFLOP/s (2 flops per FMA) and the kernel time (SURVEY 8(d) FP64 peak) */
int ldg_probe_fp64(int64_t iters, double* tflops, double* ms, void* stream);
/* mode 0: DFMA, 1: FP64 tensor core (mma.sync m8n8k4 f64), 2: both in one
 * loop (tflops = their sum) -- decides whether DMMA adds FP64 throughput */
int ldg_probe_fp64_mode(int mode, int64_t iters, double* tflops, double* ms, void* stream);

/* ---- multi-GPU: element partitions, halos inside the operator call ---- */
/* NCCL transport: rank 0 gets a 128-byte unique id, the caller broadcasts
 * it (any transport), every rank attaches a communicator to its handle
 * (collective, blocking).  libnccl.so.2 is dlopen'ed (the process's own
 * first); code 4 = NCCL error / NCCL missing. */
int ldg_comm_unique_id(uint8_t* id128);
int ldg_comm_init(LdgHandle* h, int nranks, int rank, const uint8_t* id128);
/* in-process transport: handles hs[0..n) on one device act as ranks 0..n-1,
 * each driven from its own host thread (tests, one-GPU pools) */
int ldg_comm_init_local(LdgHandle** hs, int n);
/* The rank's partition (parallel.py PartitionPlan): ne_owned owned elements,
 * [interior0, interior1) touch no ghost (computed while halos fly), u_ghost
 * the ghost rows the kernels read (ldg_set_ghost_rows).  Per peer k (ranks
 * ascending): u rows (width u_width doubles = ncu) sent from the owned
 * vector, u_send_idx[u_send_off[k] .. u_send_off[k+1]), received into
 * u_ghost rows u_recv_idx[...]; export rows of X (width x_width doubles)
 * likewise.  Index lists are host arrays, copied. */
int ldg_set_halo_plan(LdgHandle* h, int ne_owned, int interior0, int interior1, double* u_ghost,
                      int u_width, int x_width, int npeers, const int32_t* peers,
                      const int64_t* u_send_off, const int64_t* u_send_idx,
                      const int64_t* u_recv_off, const int64_t* u_recv_idx,
                      const int64_t* x_send_off, const int64_t* x_send_idx,
                      const int64_t* x_recv_off, const int64_t* x_recv_idx);
/* R = residual (tangent = 0) or J u (tangent = 1) of the rank's owned
 * elements, both halo exchanges inside the call and overlapped with the
 * interior elements' passes (X: the export scratch, owned + ghost slots) */
int ldg_apply_dist(LdgHandle* h, int tangent, const double* u, const double* gproj,
                   const double* bsrc, double* X, double* R, void* stream);
int ldg_comm_destroy(LdgHandle* h);

#ifdef __cplusplus
}
#endif
#endif /* LDGB200_H */
