/*
 * fetigpu.h — C-ABI of the B200-native range-space Schur solve
 * (two complex-symmetric FETI-DP(H) solves on K -/+ i*phi^-1/2*M).
 *
 * Plain C types only (no torch / CUDA types in any signature).  Complex vectors are
 * interleaved (re, im) doubles, i.e. C99 `double _Complex` / std::complex<double>.
 * Vector orderings are the reference's: free dofs in ascending mesh-dof order
 * (fem.cpp:142-150), constrained dofs likewise, multipliers ascending by (node, comp)
 * (feti.cpp:69-81).
 *
 * Each entry point names the reference interface it replaces.
 */
#ifndef FETIGPU_H
#define FETIGPU_H

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes.  Mirror the reference's exception taxonomy (csr.hpp:24-36):
 *   FETIGPU_CONTRACT  <-> ContractError  (std::invalid_argument; python ValueError)
 *   FETIGPU_NUMERICAL <-> NumericalError (std::runtime_error;    python RuntimeError)
 * Non-convergence is NOT an error (krylov.hpp:97-100): rc 0 with converged = 0. */
#define FETIGPU_OK 0
#define FETIGPU_CONTRACT 1
#define FETIGPU_NUMERICAL 2
#define FETIGPU_RUNTIME 3 /* CUDA runtime failure, no device, or extension missing */

typedef struct fetigpu_ctx fetigpu_ctx; /* opaque: owns device memory, stream, factors */

/* Problem + solver description.  Replaces the pieces of ControlProblem
 * (control.hpp:15-31), Physics (fem.hpp:20-30), FetiConfig (feti.hpp:22-30) and
 * FactorSolverConfig (control.hpp:99-104) that the FetiDp path consumes. */
typedef struct {
  int n_x, n_y;          /* elements per axis, build_rectangle_mesh (mesh.cpp:7) */
  double len_x, len_y;   /* extents; elements must be square (mesh.cpp:13-15) */
  int physics;           /* 0 = heat, whole-boundary Dirichlet (fem.cpp:121-122)
                            1 = plane strain, clamped x = 0 (fem.cpp:124-128) */
  double young, poisson; /* plane strain material (fem.cpp:46-58) */
  int s_x, s_y;          /* subdomain grid (FetiConfig::s_x/s_y) */
  double phi;            /* > 0: operator factor is K + c V, c = -i/sqrt(phi)
                            (build_complex_factors, control.cpp:113-120) */
  double mass_coeff_re;  /* used only when phi == 0: c = mass_coeff (feti_solve(),   */
  double mass_coeff_im;  /*   bindings.cpp:158-185); schur_solve then rejected      */
  double tol;            /* relative dual residual (FetiConfig::tol, feti.hpp:26) */
  int max_iter;          /* FetiConfig::max_iter; GMRES is unrestarted (feti.cpp:684) */
  int augment;           /* edge-RBM augmentation (FetiConfig::augment, feti.hpp:25; feti.cpp:171-242):
                            0 or 1 through fetigpu_create; fetigpu_create_sharded returns
                            FETIGPU_CONTRACT when it is set */
  int device;            /* CUDA device ordinal */
} fetigpu_desc;

/* FetiStats (feti.hpp:95-103) + SolveStats (krylov.hpp:14-19). */
typedef struct {
  int iterations;
  int converged;
  double relative_residual;
  double primal_residual;
  double interface_jump;
  int n_lambda;
  int coarse_dim;
  double setup_seconds;
  double solve_seconds;
} fetigpu_feti_stats;

/* RangeSpaceResult (control.hpp:140-147). plus = K + cV, minus = K - cV. */
typedef struct {
  fetigpu_feti_stats plus;
  fetigpu_feti_stats minus;
  double imag_leak;
  int imag_leak_warning;
  int converged;
  double factor_setup_seconds;
  double solve_seconds;
} fetigpu_schur_stats;

/* ---- host-only queries (no GPU needed) ------------------------------------------- */

/* s_x = s_y = 0: mesh-only query (partition fields 0).
 * info[0..9] = n_free, n_constrained, n_subdomains, n_corner_dofs, n_lambda, n_edges,
 *              ex, ey, dofs_per_node, band half-width of A_ii.
 * Replaces partition_structured (feti.cpp:34-169) + assemble_operators sizes. */
int fetigpu_problem_info(const fetigpu_desc* desc, int* info);
/* The same ten fields for a created (one-GPU) context, without rebuilding the partition. */
int fetigpu_context_info(const fetigpu_ctx* ctx, int* info);

/* Reference thermal target and boundary trace (fem.cpp:194-220): ybar (n_free),
 * yc (n_constrained). Either pointer may be NULL. */
int fetigpu_target_thermal(const fetigpu_desc* desc, double* ybar, double* yc);

/* Seeded sine-mode target of BASELINE.json configs 1-3:
 * ybar(x,y) = sum_k a_k sin(m_k pi x) sin(n_k pi y), mt19937_64(seed), Box-Muller a_k,
 * m_k, n_k = 1 + rng() % mmax.  Sampled at the free nodes. */
int fetigpu_target_sine(const fetigpu_desc* desc, unsigned long long seed, int modes, int mmax,
                        double* ybar);

/* Bottom-edge pressure load of the plane-strain cantilever (fem.cpp:222-238): f (n_free). */
int fetigpu_pressure_load(const fetigpu_desc* desc, double pressure, double* f);

/* Optimality diagnostics (diagnostics, control.cpp:122-141; python diagnostics,
 * bindings.cpp:147-156) evaluated with the operators applied on the device.  y, u, ybar:
 * n_free; yc: n_constrained or NULL.  out5 = {constraint_violation, target_mismatch,
 * control_norm, objective, violation_defined (0/1)}. */
int fetigpu_diagnostics(const fetigpu_desc* desc, const double* y, const double* u, const double* ybar,
                        const double* yc, double* out5);

/* ---- GPU context ----------------------------------------------------------------- */

/* Partition + upload + factor once (K1-K4).  Replaces the two ComplexFactorSolver
 * constructions of solve_range_space (control.cpp:303-304; feti.cpp:373-480): the
 * conjugate factor K - cV = conj(K + cV) is never factored (conjugate reuse). */
int fetigpu_create(const fetigpu_desc* desc, fetigpu_ctx** out);
void fetigpu_destroy(fetigpu_ctx* ctx);

/* Range-space Schur solve, HOST buffers (control.cpp:297-334; python
 * solve_range_space, bindings.cpp:93-111).  ybar: n_free; yc: n_constrained or NULL
 * (y_c = 0); outputs y, u, lambda: n_free each.  Copies in/out are inside the call. */
int fetigpu_schur_solve(fetigpu_ctx* ctx, const double* ybar, const double* yc, double* y, double* u,
                        double* lambda, fetigpu_schur_stats* stats);

/* Same, DEVICE pointers (inputs already resident in HBM; results left on device). */
int fetigpu_schur_solve_device(fetigpu_ctx* ctx, const double* d_ybar, const double* d_yc, double* d_y,
                               double* d_u, double* d_lambda, fetigpu_schur_stats* stats);

/* Single-factor FETI-DP solve (FetiSolver<Complex>::solve, feti.cpp:630-717; python
 * feti_solve, bindings.cpp:158-185).  sign = +1: (K + cV) x = rhs; sign = -1:
 * (K + conj(c) V) x = rhs.  rhs, x: n_free complex (interleaved), host buffers. */
int fetigpu_feti_solve(fetigpu_ctx* ctx, int sign, const double* rhs_c128, double* x_c128,
                       fetigpu_feti_stats* stats);

/* Operator-level parity hooks on n_lambda complex vectors (host buffers):
 * apply_dual_operator (feti.cpp:581-594), apply_dirichlet_preconditioner (597-627). */
int fetigpu_apply_dual(fetigpu_ctx* ctx, int sign, const double* lam_c128, double* out_c128);
int fetigpu_apply_precond(fetigpu_ctx* ctx, int sign, const double* r_c128, double* out_c128);

/* Full-space KKT method (solve_full_space, control.cpp:418-476; python solve_full_space,
 * bindings.cpp:113-145): outer Krylov on [V 0 K; 0 phi V -V; K -V 0] with the Murphy-Golub-
 * Wathen preconditioner.  precond 0 none, 1 "sp" (Pearson-Wathen K + V/sqrt(phi) through a
 * second FETI factor), 2 "sc" (exact Schur through the context's complex FETI factor;
 * requires outer = 1).  outer 0 MINRES, 1 GMRES (flexible when preconditioned).  The
 * context's FETI tolerance is the inner tolerance.  stats: iterations / relative_residual /
 * converged of the OUTER solve, n_lambda = 3n, coarse_dim = total inner FETI iterations,
 * setup_seconds = preconditioner setup.  imag_leak (may be NULL): max |Im| of the last
 * "sc" application. */
int fetigpu_full_space(fetigpu_ctx* ctx, int precond, int outer, double tol, int max_iter, const double* ybar,
                       const double* yc, double* y, double* u, double* lambda, fetigpu_feti_stats* stats,
                       double* imag_leak);

/* ---- sharded multi-GPU path ------------------------------------------
 * Rank r of R owns subdomain rows [r s_y/R, (r+1) s_y/R) (s_y % R == 0).  Per Krylov step
 * the ranks exchange cut-line interface values with their two neighbours and allreduce the
 * coarse rhs and the two CGS dot vectors; the coarse problem is solved redundantly.  There
 * is no counterpart in the reference (threads only). */

/* NCCL unique id (128 bytes): create on rank 0, broadcast to the other ranks. */
int fetigpu_nccl_unique_id(unsigned char* out128);

/* Sharded context over NCCL, one process per GPU (desc->device = this rank's GPU).  The
 * schur/feti solve entry points then take and return FULL vectors on every rank. */
int fetigpu_create_sharded(const fetigpu_desc* desc, int rank, int world, const unsigned char* nccl_id,
                           fetigpu_ctx** out);

/* NCCL plumbing self-test: communicator init, allreduce sum/max and allgatherv on
 * [rank+1, 2(rank+1), -(rank+1), 0] -> out4 (every rank of `world` calls it). */
int fetigpu_nccl_selftest(const unsigned char* nccl_id, int rank, int world, int device, double* out4);

/* Host-only layout of rank `rank` (for tests): info[0..11] = first subdomain, local
 * subdomains, phantom subdomains, first local multiplier (global id), ghost rows, owned
 * rows, top-cut rows, first owned free dof, owned free dofs, halo slots sent up, halo
 * slots sent down, local multipliers. */
int fetigpu_rank_info(const fetigpu_desc* desc, int rank, int world, int* info);

/* `world` ranks emulated by host threads on ONE device (desc->device), with device-to-
 * device copies standing in for NCCL; one range-space Schur solve, rank 0's result. */
int fetigpu_emulated_schur_solve(const fetigpu_desc* desc, int world, const double* ybar, const double* yc,
                                 double* y, double* u, double* lambda, fetigpu_schur_stats* stats);

/* ---- instrumentation --------------------------------------------------------------- */

/* The cudaStream_t (as void*) every kernel of this context is launched on. */
void* fetigpu_stream(fetigpu_ctx* ctx);

/* Number of kernels this context has launched since creation (or the last reset). */
long long fetigpu_launch_count(fetigpu_ctx* ctx, int reset);

/* Per-kernel-class device time.  enable != 0 brackets every launch of the classes
 * below with CUDA events on the context stream; read accumulates elapsed ms and
 * launch counts since the last reset.  class ids: see FETIGPU_K_* below. */
#define FETIGPU_K_PRECOND_GEMV 0 /* Dirichlet S_bb apply (K6)            */
#define FETIGPU_K_DUAL_GEMV 1    /* local dual operator apply (K5)       */
#define FETIGPU_K_COARSE 2       /* coarse gather + solve (K4)           */
#define FETIGPU_K_LAMBDA 3       /* signed B / B^T gathers (K5/K6 tails) */
#define FETIGPU_K_ORTHO 4        /* GMRES CGS2 + reductions (K7)         */
#define FETIGPU_K_BAND 5         /* banded fwd/bwd substitution (K5)     */
#define FETIGPU_K_GLOBAL 6       /* global stencils, mass solve (K8)     */
#define FETIGPU_K_OTHER 7
#define FETIGPU_K_COUNT 8
int fetigpu_profile(fetigpu_ctx* ctx, int enable);
int fetigpu_profile_read(fetigpu_ctx* ctx, double* ms, long long* launches, int reset);

/* Mean in-graph kernel spans (us, first CTA start to last CTA end, %globaltimer) over the
 * Arnoldi steps of the context's last FETI solve: out6 = {precond GEMV, gap, dual GEMV,
 * gap, Arnoldi tail, gap to the next step}.  Returns the number of steps averaged (0 if
 * none were recorded, e.g. on the sharded path). */
int fetigpu_step_spans(fetigpu_ctx* ctx, double* out6);

/* Average launch duration (ms) of the Arnoldi step's two GEMVs: CUDA events around a
 * captured graph of `reps` consecutive launches of each on the context's operators:
 * out4 = {precond ms, dual ms, precond bytes, dual bytes}.  One-GPU contexts. */
int fetigpu_gemv_timing(fetigpu_ctx* ctx, int reps, double* out4);

/* Algorithmic bytes per launch of a kernel class (the roofline numerator). */
double fetigpu_class_bytes(fetigpu_ctx* ctx, int klass);

/* Thread-local message of the last failing call. */
const char* fetigpu_last_error(void);

/* ---- 3D extension (BASELINE.json configs 4-5) -----------------------------------------
 * The reference is 2D only.  This is the same FETI-DP(H) range-space
 * Schur solve on trilinear Q1 hexahedra: heat with whole-boundary Dirichlet, or linear
 * elasticity (3 dofs/node interleaved) clamped on the face x = 0; corners = free subdomain-
 * grid vertices; pairwise multipliers on multiplicity-4 subdomain edges with Dirichlet
 * scaling W = 1/multiplicity (the natural extension of feti.cpp:34-169, 597-627).  Vector
 * orders: free dofs ascending by mesh dof (x fastest, then y, then z; dof = dpn node + comp);
 * multipliers ascending by (node, comp, pair).  Return codes / stats as above. */
typedef struct fetigpu3d_ctx fetigpu3d_ctx;
typedef struct {
  int n_x, n_y, n_z;          /* elements per axis (cube elements) */
  double len_x, len_y, len_z;
  int physics;                /* 0 heat, 1 linear elasticity (E = young, nu = poisson) */
  double young, poisson;
  int s_x, s_y, s_z;          /* subdomain grid */
  double phi;                 /* > 0: factor K + cV, c = -i/sqrt(phi) */
  double mass_coeff_re;       /* phi == 0: c = mass_coeff (feti_solve only) */
  double mass_coeff_im;
  double tol;                 /* relative dual residual */
  int max_iter;
  int device;
} fetigpu3d_desc;

/* info[0..15] = n_free, n_constrained, subdomains, corner dofs, n_lambda, NI (padded), NB,
 * NC, MR, block half-bandwidth P, dofs per node, ex, ey, ez, MAXE_BI, MAXE_IB (host only). */
int fetigpu3d_problem_info(const fetigpu3d_desc* desc, long long* info16);
/* Seeded sine-mode target ybar = sum_k a_k sin(l_k pi x) sin(m_k pi y) sin(n_k pi z). */
int fetigpu3d_target_sine(const fetigpu3d_desc* desc, unsigned long long seed, int modes, int mmax, double* ybar);
int fetigpu3d_create(const fetigpu3d_desc* desc, fetigpu3d_ctx** out);
void fetigpu3d_destroy(fetigpu3d_ctx* ctx);
int fetigpu3d_schur_solve(fetigpu3d_ctx* ctx, const double* ybar, const double* yc, double* y, double* u,
                          double* lambda, fetigpu_schur_stats* stats);
int fetigpu3d_schur_solve_device(fetigpu3d_ctx* ctx, const double* d_ybar, const double* d_yc, double* d_y,
                                 double* d_u, double* d_lambda, fetigpu_schur_stats* stats);
int fetigpu3d_feti_solve(fetigpu3d_ctx* ctx, int sign, const double* rhs_c128, double* x_c128,
                         fetigpu_feti_stats* stats);
int fetigpu3d_apply_dual(fetigpu3d_ctx* ctx, int sign, const double* lam_c128, double* out_c128);
int fetigpu3d_apply_precond(fetigpu3d_ctx* ctx, int sign, const double* r_c128, double* out_c128);
void* fetigpu3d_stream(fetigpu3d_ctx* ctx);
long long fetigpu3d_launch_count(fetigpu3d_ctx* ctx, int reset);
int fetigpu3d_profile(fetigpu3d_ctx* ctx, int enable);
int fetigpu3d_profile_read(fetigpu3d_ctx* ctx, double* ms, long long* launches, int reset);
/* Sharded 3D path: rank r of R owns the subdomain z-layers
 * [r s_z/R, (r+1) s_z/R) (s_z % R == 0); dual (multiplier) and primal vectors are replicated,
 * each rank applies its subdomains and one allreduce per operator application completes the
 * jump gathers (two owners per row: the sum is exact); the coarse problem is assembled by an
 * allreduce and solved redundantly.  NCCL, one process per GPU (nccl_id from
 * fetigpu_nccl_unique_id on rank 0); solves take and return FULL vectors on every rank. */
int fetigpu3d_create_sharded(const fetigpu3d_desc* desc, int rank, int world, const unsigned char* nccl_id,
                             fetigpu3d_ctx** out);
/* `world` ranks emulated by host threads on ONE device; one Schur solve, rank 0's result. */
int fetigpu3d_emulated_schur_solve(const fetigpu3d_desc* desc, int world, const double* ybar, const double* yc,
                                   double* y, double* u, double* lambda, fetigpu_schur_stats* stats);
/* Host-only layout of a rank: info6 = first subdomain, local subdomains, local row owners,
 * rows with both owners local, local corner slots, n_lambda. */
int fetigpu3d_rank_info(const fetigpu3d_desc* desc, int rank, int world, long long* info6);
/* Algorithmic bytes per launch of a kernel class; setup phase times (s): out8 = {assembly,
 * A_ii factor, multi-RHS solves, S_bb build, S_bb inverse, coupling + coarse, pack, total}. */
double fetigpu3d_class_bytes(fetigpu3d_ctx* ctx, int klass);
int fetigpu3d_setup_times(fetigpu3d_ctx* ctx, double* out8);

#ifdef __cplusplus
}
#endif
#endif /* FETIGPU_H */
