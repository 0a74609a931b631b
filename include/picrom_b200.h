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

/* Bytes of scratch the deposit / PIC-step calls need for (n, p, nx, degree). */
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
 * then the per-instance Poisson solve overwrites phi with phi_{n+1}.
 * First step: v holds v_0, kick = 0.5*dt, kfull = 0; later steps: v holds
 * v_{n-1/2}, kick = dt, kfull = 0.5*dt.  History pointers may be NULL:
 * rho_hist/phi_hist (rows of p*nx) get rho/phi at step+1, ee_hist (rows of p)
 * the electric energy at step+1, kin_hist (rows of p) the kinetic energy
 * 0.5*sum v_n^2 at `step`.  Row index = `step`, or, when `counter` is non-NULL
 * (a device {long long step; unsigned done;} pair, 16 bytes), the device
 * value *counter, which the call advances by one -- so a CUDA graph of k
 * steps can be replayed with unchanged parameters. */
int picrom_pic_step(double* x, double* v, long long n, int p, long long ld,
                    const double* inst, int nx, int degree,
                    const double* khat, const double* stencil, double* phi,
                    double dt, double kick, double kfull, long long step,
                    long long* counter,
                    double* rho_hist, double* phi_hist, double* ee_hist, double* kin_hist,
                    void* workspace, unsigned long long* status, void* stream);

/* The two halves of picrom_pic_step, for callers that time or schedule them
 * separately: the fused particle pass (writes the deposit segments and the
 * kinetic partials into the workspace) and the per-instance solve that
 * consumes them (same history/counter semantics as picrom_pic_step). */
int picrom_pic_push(double* x, double* v, long long n, int p, long long ld,
                    const double* inst, int nx, int degree, const double* phi,
                    double dt, double kick, double kfull, long long step,
                    const long long* counter, void* workspace,
                    unsigned long long* status, void* stream);
int picrom_pic_solve(long long n, int p, int nx, int degree, const double* inst,
                     const double* khat, const double* stencil, double* phi,
                     long long step, long long* counter, double* rho_hist,
                     double* phi_hist, double* ee_hist, double* kin_hist,
                     void* workspace, void* stream);

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

#ifdef __cplusplus
}
#endif

#endif /* PICROM_B200_H */
