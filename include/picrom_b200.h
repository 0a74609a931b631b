/*
 * picrom_b200 -- C-ABI of the B200 (sm_100a) hot path of the parametric
 * geometric PIC / dynamical reduced-basis solver of arXiv 2201.05555.
 *
 * Every entry point is `extern "C"`, takes plain device pointers and sizes,
 * launches on the caller's stream (`stream` is a cudaStream_t passed as
 * void*), never synchronises, never allocates, and returns 0 on success or a
 * PICROM_ERR_* code (message via picrom_last_error()).  Scratch memory is a
 * caller-owned workspace sized by the *_workspace_bytes queries.
 *
 * Layout conventions:
 *   particle arrays  instance-major (p, N): element (particle i, instance j)
 *                    at a[j*ld + i];  the reference's numpy (N, p) row-major
 *                    arrays are transposed once on upload (picrom_transpose).
 *   grid arrays      (p, Nx): node n of instance j at g[j*Nx + n].
 *   inst             per-instance parameter rows, PICROM_INST_STRIDE doubles
 *                    each: {h, 1/h, qw, background*h, -(qw/m_p), qw/m_p,
 *                    0.5/m_p, length} -- fem.py:54-98 (PeriodicMesh.h,
 *                    ChargeConfig.charge_weight / particle_mass).
 *   status           one unsigned long long in device memory, initialised
 *                    to ~0ULL by the caller; the first non-finite position
 *                    (row-major (N, p) linear index row*p+col, packed as
 *                    step<<40 | index) is recorded with atomicMin -- the
 *                    device form of fem.py:101-105 (_check_finite) and
 *                    fullorder.py:111-120 (DivergenceError.parameter_index).
 *
 * Spline degree d in {1,2,3}: node m (0..d) of a particle in cell c is
 * (c - d/2 + m) mod Nx with weight N_d(f + d - m).  d = 1 is the
 * reference's P1 hat basis exactly (fem.py:119-200).
 */
#ifndef PICROM_B200_H
#define PICROM_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PICROM_OK 0
#define PICROM_ERR_CONFIG 1
#define PICROM_ERR_CUDA 2

#define PICROM_INST_STRIDE 8

/* gather kinds for picrom_gather */
#define PICROM_GATHER_VALUE 0    /* sum_i phi_i lambda_i(x)            BasisTable.matvec, fem.py:138-149 (value table) */
#define PICROM_GATHER_FIELD 1    /* -(qw/m_p) d/dx sum phi_i lambda_i  field_at_particles, fem.py:254-256 */
#define PICROM_GATHER_GRAD  2    /* +(qw/m_p) d/dx sum phi_i lambda_i  driver.exact_gradients coef, driver.py:74-75 */
#define PICROM_GATHER_DERIV 3    /* d/dx sum phi_i lambda_i            BasisTable.matvec, gradient table */

/* basis-table kinds for picrom_basis_table */
#define PICROM_TABLE_VALUE 0     /* eval_basis, fem.py:179-182 */
#define PICROM_TABLE_GRAD  1     /* eval_basis_grad, fem.py:185-190 */

int picrom_version(void);
const char* picrom_last_error(void);
/* SM count / compute capability of the current device (host query). */
int picrom_device_info(int* num_sms, int* cc_major, int* cc_minor);

/* ---------------------------------------------------------------- FOM --- */

/* Bytes of scratch the deposit / PIC-step calls need for (n, p, nx, degree).
 * The workspace holds per-instance tickets: it must be
 * zero-filled once before its first picrom_pic_step / picrom_pic_push (every
 * call leaves them zeroed); the one-shot entry points (deposit, rmatvec,
 * verlet_drift) clear them themselves. */
size_t picrom_fom_workspace_bytes(long long n, int p, int nx, int degree);

/* fem._locate (fem.py:108-116): i0 = floor(x/h) mod Nx (int64, bit-exact),
 * frac = x/h - floor(x/h).  Outputs in (p, ldo) layout. */
int picrom_locate(const double* x, long long n, int p, long long ld,
                  const double* inst, int nx,
                  long long* i0, double* frac, long long ldo,
                  unsigned long long* status, void* stream);

/* eval_basis / eval_basis_grad (fem.py:179-190) for degree d: i0 plus the d+1
 * weight planes w[m*p*ldo + j*ldo + i]. */
int picrom_basis_table(const double* x, long long n, int p, long long ld,
                       const double* inst, int nx, int degree, int kind,
                       long long* i0, double* w, long long ldo,
                       unsigned long long* status, void* stream);

/* deposit_charge(eval_basis(mesh, x), charge) (fem.py:203-215, rmatvec
 * fem.py:151-166): rho (p, nx) = qw * Lambda^T 1 + background*h. */
int picrom_deposit(const double* x, long long n, int p, long long ld,
                   const double* inst, int nx, int degree,
                   double* rho, void* workspace,
                   unsigned long long* status, void* stream);

/* BasisTable.rmatvec (fem.py:151-166): out (p, nx) = Lambda^T y for the
 * value (kind 0) or gradient (kind 1) table of x; y may be NULL (ones). */
int picrom_rmatvec(const double* x, const double* y, long long n, int p, long long ld,
                   const double* inst, int nx, int degree, int kind, double* out,
                   void* workspace, unsigned long long* status, void* stream);

/* PoissonOperator.solve (fem.py:239-244) + electric_energy (fem.py:247-251):
 * phi = K (rho - mean rho) - mean, K the (L + 11^T/length)^{-1} circulant
 * given by its unit-mesh first column khat (nx doubles, scaled by h on
 * device); stencil = the d+1 stiffness coefficients a_k (L = a/h).
 * energy (p) may be NULL. */
int picrom_poisson(const double* rho, int p, int nx, int degree,
                   const double* inst, const double* khat, const double* stencil,
                   double* phi, double* energy, void* stream);

/* electric_energy (fem.py:247-251): energy[j] = 0.5/m_p * phi_j^T L phi_j. */
int picrom_field_energy(const double* phi, int p, int nx, int degree,
                        const double* inst, const double* stencil, double* energy,
                        void* stream);

/* grid -> particle gather (fem.py:138-149 / 254-256, driver.py:74-76):
 * out (p, ldo) = kind-weighted sum_m phi[node_m] * (d^k/dx^k) N_d(...). */
int picrom_gather(const double* x, long long n, int p, long long ld,
                  const double* inst, int nx, int degree, const double* phi,
                  int kind, double* out, long long ldo,
                  unsigned long long* status, void* stream);

/* One fused leapfrog PIC step (fullorder.py:122-134 reformulated with the
 * half-step velocity): for every particle
 *   E_n = field(x_n; phi)          (gather, cell polynomials in smem)
 *   kin += (v + kfull*E_n)^2       (kinetic energy of v_n, per instance)
 *   v  <- v + kick*E_n ;  x <- x + dt*v          (in place)
 *   rho_{n+1} += deposit(x)        (private smem histograms, deterministic)
 * then the per-instance Poisson solve overwrites phi with phi_{n+1} -- done
 * inside the same kernel by the last CTA to finish each instance (one launch
 * per step).
 * First step: v holds v_0, kick = 0.5*dt, kfull = 0; later steps: v holds
 * v_{n-1/2}, kick = dt, kfull = 0.5*dt.  History pointers may be NULL:
 * rho_hist/phi_hist (rows of hist_p*nx) get rho/phi at step+1, ee_hist (rows
 * of hist_p) the electric energy at step+1, kin_hist (rows of hist_p) the kinetic energy
 * 0.5*sum v_n^2 at `step`.  Row index = `step`, or, when `counter` is non-NULL
 * (a device {long long step; unsigned done;} pair, 16 bytes), the device
 * value *counter (modulo hist_rows when hist_rows > 0: a ring), which the
 * call advances by one -- so a CUDA graph of k steps can be replayed with
 * unchanged parameters.  hist_p (>= p; 0 means p) is the number of instances
 * per history row: an instance group [g0, g0+p) of a larger batch writes its
 * slice of a shared history when the caller offsets the pointers by g0*nx
 * (rho/phi) and g0 (energies). */
int picrom_pic_step(double* x, double* v, long long n, int p, long long ld,
                    const double* inst, int nx, int degree,
                    const double* khat, const double* stencil, double* phi,
                    double dt, double kick, double kfull, long long step,
                    long long* counter, long long hist_rows, int hist_p,
                    double* rho_hist, double* phi_hist, double* ee_hist, double* kin_hist,
                    unsigned long long* t_hist, void* workspace,
                    unsigned long long* status, void* stream);

/* %globaltimer (ns) into *out when the stream reaches this point (per-step
 * timing of a replayed step graph: picrom_pic_step's t_hist, nullable, gets
 * the time its counter advanced, i.e. the end of the step's last solve). */
int picrom_timestamp(unsigned long long* out, void* stream);

/* The two halves of picrom_pic_step, for callers that time or schedule them
 * separately: the fused particle pass (writes the deposit segments and the
 * kinetic partials into the workspace) and the per-instance solve that
 * consumes them (same history/counter semantics as picrom_pic_step, except
 * that with a counter and hist_rows > 0 the history row is *counter modulo
 * hist_rows -- a ring that a replayed CUDA graph can keep writing). */
int picrom_pic_push(double* x, double* v, long long n, int p, long long ld,
                    const double* inst, int nx, int degree, const double* phi,
                    double dt, double kick, double kfull, long long step,
                    const long long* counter, void* workspace,
                    unsigned long long* status, void* stream);
int picrom_pic_solve(long long n, int p, int nx, int degree, const double* inst,
                     const double* khat, const double* stencil, double* phi,
                     long long step, long long* counter, long long hist_rows,
                     double* rho_hist, double* phi_hist, double* ee_hist,
                     double* kin_hist, void* workspace, void* stream);

/* Reference-arithmetic Verlet (fullorder.py:122-134, bit-for-bit operation
 * order): drift  x1 = x + dt*(v + (0.5*dt)*e0), rho1 = deposit(x1), phi1 = solve;
 * kick   e1 = field(x1; phi1), v1 = v + (0.5*dt)*(e0 + e1).
 * drift writes x1 and phi1 (+ rho1/energy if non-NULL); kick writes e1, v1. */
int picrom_verlet_drift(const double* x, const double* v, const double* e0,
                        long long n, int p, long long ld,
                        const double* inst, int nx, int degree,
                        const double* khat, const double* stencil,
                        double dt, long long step, double* x1, double* phi1,
                        double* rho1, double* energy1,
                        void* workspace, unsigned long long* status, void* stream);
int picrom_verlet_kick(const double* x1, const double* v, const double* e0,
                       long long n, int p, long long ld,
                       const double* inst, int nx, int degree, const double* phi1,
                       double dt, double* e1, double* v1, void* stream);

/* Sum of squares per instance: out[j] = 0.5 * sum_i a[j*ld+i]^2 (kinetic
 * energy, fullorder.py:197). */
int picrom_half_sumsq(const double* a, long long n, int p, long long ld,
                      double* out, void* workspace, void* stream);

/* out (cols, rows) = in (rows, cols)^T, both row-major, doubles. */
int picrom_transpose(const double* in, long long rows, long long cols,
                     double* out, void* stream);
/* int64 variant (cell indices). */
int picrom_transpose_i64(const long long* in, long long rows, long long cols,
                         long long* out, void* stream);

/* ---------------------------------------------------------------- ROM --- */
/* Reduced basis U (2N x n) row-major: rows [0, N) = U_X, [N, 2N) = U_V;
 * coefficients Z (n x p') row-major with leading dimension ldz; `cols`
 * (nullable) maps each column of Z to its instance row in `inst` (per-instance
 * meshes, BASELINE C3/C4). */

/* Scratch for the reduced-basis calls at (N, p', n, nx). */
size_t picrom_rom_workspace_bytes(long long N, int p, int n, int nx);

/* Field half of driver.exact_gradients (driver.py:70-73): X_r = U_X Z is
 * formed in registers, deposited, and each column solved:
 * phi/rho (p', nx), energy (p') -- each may be NULL. */
int picrom_rom_field(const double* ux, long long N, int n, const double* z, int ldz,
                     int p, const int* cols, const double* inst, int nx, int degree,
                     const double* khat, const double* stencil, double* phi,
                     double* rho, double* energy, void* workspace,
                     unsigned long long* status, const long long* skip, void* stream);

/* Gather half (driver.py:74-76, make_full_stage driver.py:83-85):
 * E = coef * d/dx (phi . lambda)(U_X Z) with coef = qw/m_p (coef_kind 0) or 1
 * (coef_kind 1); g_out (n x p', leading dim ldg) = U_X^T E (nullable);
 * lam (N x p', row stride ldo) = (phi . lambda)(U_X Z) (DEIM harvest,
 * nullable); eout (N x p', row stride ldo) = E (nullable). */
int picrom_rom_gather(const double* ux, long long N, int n, const double* z, int ldz,
                      int p, const int* cols, const double* inst, int nx, int degree,
                      const double* phi, int coef_kind, double* g_out, int ldg,
                      double* lam, double* eout, long long ldo, void* workspace,
                      unsigned long long* status, const long long* skip, void* stream);

/* As picrom_rom_gather with u the full (2N x n) basis [U_X; U_V] and both
 * projections of E: g_out = U_X^T E and gv_out = U_V^T E (n x p', ld ldg).
 * With them the basis velocity's U^T (G Z^T) and U^T J (G Z^T) blocks
 * (reduction.py:148-153) come from n x n algebra instead of a 2N-row Gram. */
int picrom_rom_gather_uv(const double* u, long long N, int n, const double* z, int ldz,
                         int p, const int* cols, const double* inst, int nx, int degree,
                         const double* phi, int coef_kind, double* g_out, double* gv_out,
                         int ldg, double* lam, double* eout, long long ldo, void* workspace,
                         unsigned long long* status, void* stream);

/* out (w x w) = W^T W, W = [B_0 | ... | B_{k-1}] the column concatenation of k
 * tall blocks with N rows (block i: ptrs[i], row stride lds[i], widths[i]
 * columns; jswap[i] = 1 uses J B_i, the block with its row halves swapped and
 * the new lower half negated -- reduction.jmul, reduction.py:44-47), w <= 128,
 * k <= 8; jswap may be NULL.  Every n x n product of reduction.py:143-182 (and
 * the residuals :85-90) is a sub-block of one such Gram. */
int picrom_paired_gram(int nblocks, const double* const* ptrs, const int* lds,
                       const int* widths, const int* jswap, long long N, double* out,
                       void* workspace, void* stream);

/* Selected blocks of the paired Gram (same block conventions): for each task
 * t, out block (bi[t], bj[t]) = B_bi^T B_bj; other entries unspecified; at most
 * 64 tasks.  tangent_velocity's 7 needed products of [U, xi, r, x_eval]
 * (reduction.py:170-182) in one pass instead of the 10 of the full Gram. */
int picrom_gram_tasks(int nblocks, const double* const* ptrs, const int* lds,
                      const int* widths, const int* jswap, int ntask, const int* bi,
                      const int* bj, long long N, double* out, void* workspace, void* stream);

/* out (wa x wb) = A^T B with A = blocks [0, na) and B = blocks [na, nblocks)
 * (same block conventions as picrom_paired_gram; total width <= 256):
 * the sliding DEIM-window Gram update and the Rayleigh-Ritz products of the
 * windowed SVD (hyper.py:262). */
int picrom_cross_gram(int nblocks, int na, const double* const* ptrs, const int* lds,
                      const int* widths, const int* jswap, long long N, double* out,
                      void* workspace, void* stream);

/* out (ca x k, row-major) = A^T B for a WIDE left operand: A (N x ca, row
 * stride lda, even ca <= 448) is the DEIM sample window -- (T+1) p* = 420
 * columns at C4 -- and B (N x k, row stride ldb, even k <= 48) a subspace
 * block or the newest sample block.  These are the tall products of the
 * windowed SVD that the reference gets from LAPACK's gesdd on the N x 420
 * window (hyper.py:262): the sliding Gram update, W^T Q of the subspace
 * iteration and the Rayleigh-Ritz block Q^T W.  Rows must be 16-byte aligned
 * (even strides, aligned bases).  Fixed-order reduction (deterministic). */
size_t picrom_tall_atb_workspace_bytes(long long N, int ca, int k);
int picrom_tall_atb(const double* a, int lda, int ca, const double* b, int ldb, int k,
                    long long N, double* out, void* workspace, void* stream);

/* Small dense steps of the windowed SVD's Cholesky-QR chain (hyper.py:262), so
 * that the chain Y -> Y^T Y -> R^-1 -> (W^T Y) R^-1 -> W M stays on the device:
 * picrom_small_cholinv: g (k x k SPD, k <= 48) -> rinv = R^-1 with g = R^T R (R
 *   upper triangular); info[0], info[1] = min / max diag(R), min = 0 when g is
 *   not positive definite;
 * picrom_small_rmul: out (r x k) = a (r x k) b (k x k), column j times
 *   colscale[j] (nullable). */
int picrom_small_cholinv(const double* g, int k, double* rinv, double* info, void* stream);
int picrom_small_rmul(const double* a, int r, int k, const double* b, const double* colscale,
                      double* out, void* stream);

/* DEIM greedy selection step (hyper.py:241-244): out_index = the first index
 * of max |v[i*stride]| over i < n with the `banned` indices scored -1;
 * out_value (nullable) = that maximum. */
int picrom_argmax_abs(const double* v, long long n, long long stride,
                      const long long* banned, int nbanned, long long* out_index,
                      double* out_value, void* workspace, void* stream);

/* Compare-mode error norms (diagnostics.py:50-71): out[0] = ||a - b||_F^2,
 * out[1] = ||a||_F^2 over `count` contiguous doubles (b nullable -> out[0] =
 * 0); fixed-order reduction; workspace >= 8 * 4 * num_sms * 2 doubles. */
int picrom_diff_sumsq(const double* a, const double* b, long long count, double* out,
                      void* workspace, void* stream);

/* Scratch bytes of picrom_deim_greedy for an N x d basis. */
size_t picrom_deim_workspace_bytes(long long N, int d);

/* deim_greedy (hyper.py:218-246) fully on the device: psi (N x d, row stride
 * ld >= d), keep (HOST array of d entries; entry k >= 0 pre-assigns position
 * k -- the partial refresh of fit_deim, hyper.py:268-275 -- or NULL) ->
 * idx (device, d int64) and rows (device, d x d: rows[k] = psi[idx[k], :]).
 * Position k's index is the first max of |psi_k - Psi_{<k} c| with
 * R[:k, :k] c = R[:k, k] and the indices already assigned scored -1; no host
 * round trip between positions. d <= 64. */
int picrom_deim_greedy(const double* psi, int ld, long long N, int d, const long long* keep,
                       long long* idx, double* rows, void* workspace, void* stream);

/* out (N x c, row stride ldo) (+)= sum_t op_t(in_t) (N x widths[t]) @ M_t,
 * op_t = J when jswap[t] (nullable), M_t (widths[t] x c) at mats + moffs[t]
 * (device); at most 6 terms; c <= 32, or c <= 48 when N >= 1024 and every
 * input row is 16-byte aligned (the window's W (N x 420) @ (420 x 48) products
 * of the subspace iteration, hyper.py:262). */
int picrom_combine(int nterms, const double* const* ins, const int* lds,
                   const int* widths, const int* jswap, const int* moffs,
                   const double* mats, int mats_len, long long N, double* out, int ldo,
                   int c, int accumulate, void* stream);

/* Batched DMD extrapolation of the potential (DMDModel.potential,
 * hyper.py:76-91): re_out (p x nx) = Re(modes (nx x r) . (coords (r x p) * w)),
 * w_m = exp(omega_m (t - t0)); complex arrays interleaved (re, im), row-major;
 * im_out (nullable) = the imaginary part (the reference's imag-defect check). */
int picrom_dmd_extrapolate(const double* modes, const double* coords, const double* w,
                           int nx, int r, int p, double* re_out, double* im_out,
                           void* stream);

/* DEIM-sampled gather + projection of the hyper-reduced coefficient gradient
 * (make_hyper_stage.g, hyper.py:320-328): for each column j,
 * out[k][j] = inv_mp_j * sum_r uxd[r][k] * dphi_j(uxd[r] . z_j) * w[r] * wscale[j]
 * with dphi_j the x-derivative of the potential phi (p x nx) on instance j's
 * mesh; uxd (d x n) = U_X rows at the DEIM indices; wscale nullable (= 1). */
int picrom_deim_gather(const double* uxd, const double* z, int ldz, const double* phi,
                       const double* inst, const int* cols, const double* w,
                       const double* wscale, int d, int n, int p, int nx, int degree,
                       double* out, int ldo, unsigned long long* status,
                       const long long* skip, void* stream);

/* `skip` (nullable, device int64) on picrom_rom_field / picrom_rom_gather /
 * picrom_deim_gather: when *skip is nonzero the launches do nothing -- the
 * iterations queued after a device-side fixed-point convergence
 * (picrom_fp_update sets state[0]).
 *
 * One iteration of the implicit coefficient stage (fixed_point,
 * reduction.py:185-202) for k -> J g(z + dt/2 k), g(z) = D(z) + C z with
 * D(zeval) in gout (n x p, from the F-evaluation kernels at zeval) and C =
 * U_V^T U_V (n x n), all device, row-major:  k_new = J(gout + C zeval);
 * trace[it] = ||k_new - k|| / max(||k_new||, tiny); k = k_new;
 * zeval = z + half_dt k_new; converged (trace[it] <= tol) -> state[1] = it+1,
 * state[0] = 1, after which the call is a no-op.  One CTA; n p <= 25600. */
int picrom_fp_update(const double* gout, const double* c, const double* z, double* k,
                     double* zeval, int n, int p, double half_dt, double tol, int it,
                     long long* state, double* trace, void* stream);

/* out (d x w) = rows idx of src (row-major, leading dim ld): U_X[I] of
 * make_hyper_stage (hyper.py:312). */
int picrom_rows_gather(const double* src, int ld, const long long* idx, int d, int w,
                       double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PICROM_B200_H */
