/*
 * smg.h -- C ABI of libsmg.so, the B200 (sm_100a) hot path of the weighted
 * additive Schwarz / p-multigrid / MGCG solver (arXiv 1512.02390).
 *
 * The reference (/root/reference/pkg/src/schwarzmg) is pure Python/NumPy and
 * has no FFI; every entry point below replaces one NumPy call site on its
 * hot path (cited per function).  A maintainer binds it from the reference
 * with ctypes.
 *
 * Conventions
 *   - Fields are dense (N_y, N_x) float64 arrays in DEVICE memory, row-major,
 *     y slow / x fast, N_* = p * n_*  (reference mesh.py:1-7, 49-70).
 *   - Every launch is enqueued on the caller's stream (a cudaStream_t passed
 *     as void*); nothing synchronizes except where documented.
 *   - Host arrays (factors, matrices) are copied at create time; handles own
 *     only immutable per-level constants, so one handle may serve several
 *     streams at once.  Every scratch buffer a call writes (ring workspace,
 *     reduction partials) is caller-owned and passed in; calls running
 *     concurrently need distinct workspaces.
 *   - Return value: 0 on success, <0 on error; smg_last_error() explains.
 *     No CPU fallback exists: without a CUDA device every compute call fails.
 */
#ifndef SMG_H
#define SMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMG_OK 0
#define SMG_EINVAL -1      /* bad argument (maps to ValueError)          */
#define SMG_EUNSUPPORTED -2 /* order / window size not compiled in        */
#define SMG_ECUDA -3       /* CUDA runtime error (maps to RuntimeError)  */
#define SMG_ENOMEM -4

typedef struct smg_op smg_op_t;             /* one level's operator          */
typedef struct smg_schwarz smg_schwarz_t;   /* one level's additive smoother */
typedef struct smg_transfer smg_transfer_t; /* level l-1 <-> l transfers     */
typedef struct smg_coarse smg_coarse_t;     /* p=1 pseudo-inverse            */
typedef struct smg_mult smg_mult_t;         /* multiplicative smoother       */

const char* smg_last_error(void);
int smg_version(void);
/* Number of kernel launches libsmg has enqueued in this process (evidence
 * for the bench's gpu_launches claim; graph replays are not re-counted). */
int64_t smg_launch_count(void);
/* Profiling aid (SMG_FDT_PHASES=1 in the environment): copies the tiled
 * Schwarz kernel's per-phase cycle sums (out[0] = tiles, out[1..] = cycles
 * of thread 0 per phase, summed over CTAs) into out[0..n) and resets them. */
int smg_debug_fdt_phases(unsigned long long* out, int n);
/* 1 if a CUDA device is usable, else 0 (and smg_last_error says why). */
int smg_device_ok(void);

/* ---- operators (replaces operators.py:30-54 PoissonOperator.apply and
 *      operators.py:57-92 DiffusionOperator.apply; residual operators.py:101-103)
 * weights: p+1 GLL weights; mat: (p+1)^2 row-major -- the reference stiffness
 * basis.stiff for Poisson, the derivative matrix basis.diff for diffusion.
 * nu (diffusion only): device (N_y, N_x) nodal diffusivity, must outlive h. */
int smg_op_create(smg_op_t** h, int kind /*0 Poisson, 1 diffusion*/, int p, int n_x, int n_y,
                  double dx, double dy, const double* weights, const double* mat,
                  const double* nu_dev);
int smg_op_destroy(smg_op_t* h);
/* out = f - A u   (f == NULL: out = A u).  out must not alias u. */
int smg_op_residual(const smg_op_t* h, const double* u, const double* f, double* out,
                    void* stream);
/* Ring workspace of the halo-free operator kernel (doubles, device; 0 where the
 * operator has none: 2 p per element for the tensor-core kernels, diffusion
 * p = 24 and Poisson p = 32).  With it, smg_op_residual_ws runs the element
 * kernel on its own (p+1)^2 window only and a fixup launch adds the neighbours'
 * vertex terms in a fixed order; ring == NULL is smg_op_residual. */
size_t smg_op_ring_doubles(const smg_op_t* h);
int smg_op_residual_ws(const smg_op_t* h, const double* u, const double* f, double* out, double* ring,
                       void* stream);
/* Like smg_op_residual, and also *norm2_out (device double) = ||out||^2
 * summed deterministically; ws (device) must hold smg_op_ws_doubles(h)
 * doubles (the per-CTA partials and the reduction workspace of the _ws
 * variant; no initialisation needed) and must not overlap norm2_out. */
size_t smg_op_ws_doubles(const smg_op_t* h);
int smg_op_residual_norm2(const smg_op_t* h, const double* u, const double* f, double* out,
                          double* norm2_out, double* ws, void* stream);
/* Same with the operator's ring workspace (NULL allowed): where a specialised residual
 * kernel exists (tensor-core / warp-per-element) the residual runs on it and ||out||^2 comes
 * from a deterministic dot pass over out (8 B/DOF) instead of the generic kernel's fused
 * partials -- C3: 301 -> ~165 us per residual + norm. */
int smg_op_residual_norm2_ws(const smg_op_t* h, const double* u, const double* f, double* out,
                             double* norm2_out, double* ws, double* ring, void* stream);

/* out = A u and *dot_out (device double) = u . out, deterministic: MGCG's q = A p, p . q
 * (krylov.py:91-94).  The warp-per-element Poisson kernel (p = 8, 16) forms the product
 * from its staged window (p and q are not read again); elsewhere the apply is followed by
 * a dot pass.  ws: smg_op_ws_doubles(h) doubles; ring: smg_op_ring_doubles(h) or NULL. */
int smg_op_apply_dot(const smg_op_t* h, const double* u, double* out, double* dot_out, double* ws,
                     double* ring, void* stream);

/* ---- additive Schwarz (replaces schwarz.py:215-222 FastDiagSolver.solve,
 *      :268-275 AdditiveSchwarz.smooth with mesh.py:124-150 gather/scatter)
 * S_x, S_y: m x m row-major generalized eigenvectors (reference S_x, S_y);
 * lam_x, lam_y: m eigenvalues; w_x, w_y: m 1D weights (W = w_y (x) w_x);
 * inv_nu_dev: device (n_y, n_x) 1/nu_bar per element, or NULL (Poisson). */
int smg_schwarz_create(smg_schwarz_t** h, int p, int n_o, int n_x, int n_y,
                       const double* S_x, const double* S_y, const double* lam_x,
                       const double* lam_y, const double* w_x, const double* w_y,
                       const double* inv_nu_dev);
int smg_schwarz_destroy(smg_schwarz_t* h);
/* Ring workspace of the tiled kernel (doubles, device): the overlap-region
 * contributions one tile hands to its neighbours within a correction.  0 for
 * the coloured dense path.  One workspace per concurrently running call. */
size_t smg_schwarz_ws_doubles(const smg_schwarz_t* h);
/* Which kernel the handle dispatches to (diagnostics, bench labels, tests):
 * *engine = 0 coloured dense kernel, 1 tiled even/odd DFMA, 2 tiled even/odd
 * DMMA, 3 paired-line tiled kernel; *tx, *ty = elements per tile (0 for the
 * dense kernel).  Any pointer may be NULL. */
int smg_schwarz_info(const smg_schwarz_t* h, int* engine, int* tx, int* ty);
/* u += sum_s R_s^T W A_s^-1 R_s r (/ nu_bar): the additive correction of one
 * sweep given the residual r.  ws: smg_schwarz_ws_doubles(h) doubles.
 * Deterministic (no atomics). */
int smg_schwarz_correct(const smg_schwarz_t* h, const double* r, double* u, double* ws, void* stream);
/* One or more full sweeps: r = f - A u; u += correction.  work: N_y*N_x,
 * ws as smg_schwarz_correct.  u_is_zero != 0 declares u == 0 on entry: the
 * first sweep skips A u and WRITES u = correction (u's prior contents are
 * never read). */
int smg_schwarz_smooth(const smg_schwarz_t* h, const smg_op_t* op, double* u, const double* f,
                       double* work, double* ws, int n_it, int u_is_zero, void* stream);
/* Same, with the operator's ring workspace (smg_op_ring_doubles; NULL allowed). */
int smg_schwarz_smooth_ws(const smg_schwarz_t* h, const smg_op_t* op, double* u, const double* f,
                          double* work, double* ws, double* op_ring, int n_it, int u_is_zero, void* stream);
/* FastDiagSolver.solve on nb independent (m,m) blocks: out = W*(S_y(S_y^T B S_x ./ L)S_x^T).
 * apply_weight=0 skips W (the multiplicative / kind=None solver). */
int smg_fd_solve_blocks(const smg_schwarz_t* h, const double* blocks, double* out, int nb,
                        int apply_weight, void* stream);

/* ---- transfers (replaces multigrid.py:180-193 dense P_y C P_x^T products)
 * J: (p_f+1) x (p_c+1) row-major reference interpolation matrix. */
int smg_transfer_create(smg_transfer_t** h, int p_c, int p_f, int n_x, int n_y, const double* J);
int smg_transfer_destroy(smg_transfer_t* h);
/* uf = P uc (accumulate=0) or uf += P uc (accumulate=1). */
int smg_prolongate(const smg_transfer_t* h, const double* uc, double* uf, int accumulate,
                   void* stream);
/* The ascending half of a V-cycle without post-smoothing (multigrid.py:
 * 247-248, n_post = 0) in ONE launch: for l = 1..K, u_l += P_l u_{l-1},
 * u_0 = the coarse solution.  tr[l-1] is the p = 2^(l-1) -> 2^l transfer of
 * level l, u[l-1] its field (K <= 4, p_K <= 16).  Only u[K-1] (level K) is
 * written -- bitwise what K smg_prolongate(..., accumulate=1) calls leave
 * there; the intermediate fields are read, not updated.  SMG_EUNSUPPORTED
 * for other chains (the caller then prolongates level by level). */
int smg_prolongate_chain(const smg_transfer_t* const* tr, int K, const double* u0, double* const* u,
                         void* stream);
/* fc = P^T ff (P's rows are assigned, not summed: owner-computes). */
int smg_restrict(const smg_transfer_t* h, const double* ff, double* fc, void* stream);
/* fc = P^T (f - A u): residual fused with restriction (multigrid.py:244). */
int smg_residual_restrict(const smg_transfer_t* h, const smg_op_t* op, const double* u,
                          const double* f, double* fc, double* work, void* stream);
/* Restriction with a caller-owned ring workspace: where the halo-free kernel
 * is compiled (p_f = 16, 24, 32: one warp per fine element, high-side
 * vertex rows handed over through the ring, a fixup launch adds them in a
 * fixed order) smg_transfer_ws_doubles(h) > 0 and the _ws calls use it; with
 * ws == NULL or 0 doubles they are smg_restrict / smg_residual_restrict.
 * The same ring serves smg_residual_restrict_ws for the Poisson operator at
 * p_f = 4, 8, 16 (p_c = p_f / 2): the warp-per-element residual kernel
 * restricts its element in place -- r = f - A u is NOT stored, `work` is left
 * untouched -- and hands the high-side coarse nodes over through the ring.
 * op_ring: the operator's ring workspace (smg_op_ring_doubles) or NULL. */
size_t smg_transfer_ws_doubles(const smg_transfer_t* h);
int smg_restrict_ws(const smg_transfer_t* h, const double* ff, double* fc, double* ws, void* stream);
int smg_residual_restrict_ws(const smg_transfer_t* h, const smg_op_t* op, const double* u,
                             const double* f, double* fc, double* work, double* ws, double* op_ring,
                             void* stream);

/* ---- p=1 coarse problem (replaces multigrid.py:196-228 coarse CG)
 * Poisson: exact pseudo-inverse by global fast diagonalization (zero mode
 * dropped).  ws must hold smg_coarse_ws_doubles(h) doubles. */
int smg_coarse_create(smg_coarse_t** h, int n_x, int n_y, double dx, double dy);
int smg_coarse_destroy(smg_coarse_t* h);
size_t smg_coarse_ws_doubles(const smg_coarse_t* h);
/* u0 = A0^+ (f0 - mean f0) */
int smg_coarse_pinv(const smg_coarse_t* h, const double* f0, double* u0, double* ws,
                    void* stream);

/* ---- multiplicative Schwarz (replaces schwarz.py:293-353
 *      MultiplicativeSchwarz)
 * Factors as smg_schwarz_create (the solver is unweighted, kind=None);
 * nu_bar_dev: device (n_y, n_x) element means of nu (diffusion; the local
 * correction is divided by it) or NULL.  Must outlive h. */
int smg_mult_create(smg_mult_t** h, int p, int n_o, int n_x, int n_y, const double* S_x,
                    const double* S_y, const double* lam_x, const double* lam_y,
                    const double* nu_bar_dev);
int smg_mult_destroy(smg_mult_t* h);
/* One ordered sweep over all n_x*n_y subdomains (forward != 0: lexicographic
 * (e_y, e_x); else reversed) given the residual r = f - A u: for each
 * subdomain u[win] += du and r -= A du on the touched elements, in place.
 * Sequential by construction (one CTA walks the chain). */
int smg_mult_sweep(const smg_mult_t* h, const smg_op_t* op, double* u, double* r, int forward,
                   void* stream);

/* Parity mode: the reference's plain CG (multigrid.py:196-228) on the device:
 * u0 = mean0(CG(A0, f0 - mean f0)) to ||r|| <= tol ||b||, at most max_iter
 * iterations.  op must be the p=1 operator.  Blocks the host every 32
 * iterations to test convergence.  *iters_out = iterations, or -max_iter if
 * the cap was hit (the reference's coarse_cg_exhausted case). */
size_t smg_coarse_cg_ws_doubles(int64_t n);
int smg_coarse_cg(const smg_op_t* op, const double* f0, double* u0, double* ws, double tol,
                  int max_iter, int* iters_out, void* stream);

/* Fast mode for the variable-coefficient coarse level: CG on A0 (the p=1
 * diffusion operator `op`) preconditioned by scale * A0_const^+ (the
 * constant-coefficient pseudo-inverse of `pc`, typically scale = 1/mean(nu)),
 * same projections, tolerance and cap semantics as smg_coarse_cg.
 * ws: smg_coarse_pcg_ws_doubles(pc) doubles. */
size_t smg_coarse_pcg_ws_doubles(const smg_coarse_t* pc);
int smg_coarse_pcg(const smg_op_t* op, const smg_coarse_t* pc, const double* f0, double* u0, double* ws,
                   double tol, int max_iter, double scale, int* iters_out, void* stream);

/* ---- BLAS-1 with device scalars (krylov.py:56-111, multigrid.py:199-214)
 * All reductions are deterministic (fixed grid, fixed summation order). */
size_t smg_reduce_ws_doubles(void);
int smg_dot(const double* x, const double* y, int64_t n, double* out, double* ws, void* stream);
/* out[0] = x.(y - z), out[1] = x.y  (one pass; krylov.py:108,110) */
int smg_dot2(const double* x, const double* y, const double* z, int64_t n, double* out,
             double* ws, void* stream);
/* y = alpha*x + beta*y */
int smg_axpby(double alpha, const double* x, double beta, double* y, int64_t n, void* stream);
/* MGCG step (krylov.py:95-103): pq = scal[1]; if pq <= 0 set flag[0]=1 and
 * do nothing; else alpha = scal[0]/pq, u += alpha p, r -= alpha q,
 * scal[2] = ||r||^2, scal[6] = alpha.  scal holds 8 doubles. */
int smg_cg_update(double* u, double* r, const double* p, const double* q, int64_t n,
                  double* scal, int* flag, double* ws, void* stream);
/* Out-of-place variant: r_out = r_in - alpha q (r_in is kept as r_old). */
int smg_cg_update2(double* u, const double* r_in, double* r_out, const double* p, const double* q,
                   int64_t n, double* scal, int* flag, double* ws, void* stream);
/* Polak-Ribiere bookkeeping (krylov.py:108-110): s1 = z.(r - r_old) (r_old may
 * be NULL = zeros), s2 = z.r; scal[5] = s1 / scal[0] (beta); scal[0] = s2. */
int smg_cg_beta(const double* z, const double* r, const double* r_old, int64_t n, double* scal,
                double* ws, void* stream);
/* The same bookkeeping from sums already reduced across ranks (strip-
 * parallel MGCG: smg_dot2 on each rank's owned rows into scal[3..4], an
 * all-reduce, then this): scal[5] = scal[3] / scal[0]; scal[0] = scal[4]. */
int smg_cg_beta_finish(double* scal, void* stream);
/* p = z + scal[5] p  (krylov.py:109) */
int smg_cg_direction(double* p, const double* z, int64_t n, double* scal, void* stream);
/* f -= mean(f) (operators.py:138-140) */
int smg_project_mean(double* f, int64_t n, double* ws, void* stream);
/* out = sum(x) */
int smg_sum(const double* x, int64_t n, double* out, double* ws, void* stream);
/* out = sum of nb per-CTA partials (fixed order) */
int smg_sum_partials(const double* part, int nb, double* out, void* stream);

/* ---- device-side problem generation (operators.py:110-199) -------------- */
/* Field on the (n_y p, n_x p) level nodes of GLL order p (nodes, weights:
 * host arrays of p+1): kind 0 diffusivity 1 + nu_hat sin 2pi(x-s) sin 2pi(y-s)
 * (:167-173); 1 Poisson load of the sin(pi x) sin(pi y) benchmark (:154-164,
 * before project_mean); 2 variable-diffusion manufactured load (:176-199,
 * before project_mean); 3 / 4 exact-solution samples of 1 / 2. */
int smg_problem_field(int kind, int p, int n_x, int n_y, double dx, double dy, const double* nodes,
                      const double* weights, double nu_hat, double shift, double* out, void* stream);
/* Quadrature-weighted element means of a nodal field, out (n_y, n_x)
 * (DiffusionOperator.element_mean_nu, operators.py:94-98). */
int smg_element_mean(int p, int n_x, int n_y, const double* weights, const double* nu, double* out,
                     void* stream);

/* ---- strip halos and strip collectives over NCCL -------
 * The reference runs in one process; at a strip boundary these replace the
 * periodic wrap of its windows and element gathers (mesh.py:97-105, 124-139)
 * and the global sums of its inner products (krylov.py:91-111).  Rank g of
 * nranks owns element rows [g s, (g+1) s); its neighbours are g-1 (below) and
 * g+1 (above) mod nranks, so one rank wraps onto itself (NCCL self send/recv).
 * A field t is (rows, row_len) row-major on the device; rows [lo, hi) are
 * owned, ghost rows lie below lo and at/above hi (lo >= below and
 * hi + above <= rows, else SMG_EINVAL).  NCCL is loaded at run time
 * (libnccl.so.2); without it these return SMG_EUNSUPPORTED.  All calls enqueue
 * on the caller's stream (graph-capturable), none synchronizes. */
typedef struct smg_halo smg_halo_t;
/* 1 if NCCL could be loaded. */
int smg_halo_available(void);
/* NCCL version code of the loaded library (0 if none). */
int smg_halo_nccl_version(void);
/* Rank 0 draws the communicator id (n_bytes >= 128) and sends it to the
 * others out of band (torch.distributed broadcast, a file, MPI ...). */
int smg_halo_unique_id(unsigned char* out, int n_bytes);
/* Join the communicator on `device` (collective over the nranks ranks). */
int smg_halo_create(const unsigned char* id, int n_bytes, int nranks, int rank, int device, smg_halo_t** out);
int smg_halo_destroy(smg_halo_t* h);
/* Forward halo: ghost rows [lo - below, lo) <- the lower neighbour's top
 * `below` owned rows, ghost rows [hi, hi + above) <- the upper neighbour's
 * bottom `above` owned rows. */
int smg_halo_exchange(const smg_halo_t* h, double* t, int64_t rows, int64_t row_len, int64_t lo, int64_t hi,
                      int below, int above, void* stream);
/* Reverse halo: the contributions in ghost rows [lo - below, lo) go to the
 * lower neighbour and those in [hi, hi + above) to the upper one; each rank
 * adds what it receives to its owned rows -- rows [lo, lo + above) first,
 * then rows [hi - below, hi) (a fixed order, deterministic).  ws: caller-owned,
 * smg_halo_ws_doubles(row_len, below, above) doubles. */
int64_t smg_halo_ws_doubles(int64_t row_len, int below, int above);
int smg_halo_exchange_add(const smg_halo_t* h, double* t, int64_t rows, int64_t row_len, int64_t lo, int64_t hi,
                          int below, int above, double* ws, void* stream);
/* In-place sum of x[0..n) over the ranks (the strip-parallel dots). */
int smg_halo_allreduce(const smg_halo_t* h, double* x, int64_t n, void* stream);
/* full[r n_per_rank + i] <- rank r's own[i] (the replicated p = 1 coarse RHS). */
int smg_halo_allgather(const smg_halo_t* h, const double* own, double* full, int64_t n_per_rank, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SMG_H */
