// Full-order PIC kernels for sm_100a: locate, basis tables, deposit, Poisson,
// gather, fused leapfrog step, reference-order Verlet, transposes.
//
// Reference: /root/reference/pkg/src/picrom/fem.py and fullorder.py (see the
// per-function citations in include/picrom_b200.h).  Design notes: DESIGN.md.

#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"

using namespace picrom;

// ------------------------------------------------------------------ errors

static thread_local char g_err[512] = "";

static int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

static int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return PICROM_ERR_CUDA;
  }
  return PICROM_OK;
}

extern "C" const char* picrom_last_error(void) { return g_err; }
extern "C" int picrom_version(void) { return 1; }

extern "C" int picrom_device_info(int* num_sms, int* cc_major, int* cc_minor) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return set_err(PICROM_ERR_CUDA, "cudaGetDevice failed");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess)
    return set_err(PICROM_ERR_CUDA, "cudaGetDeviceProperties failed");
  if (num_sms) *num_sms = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return PICROM_OK;
}

static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// ------------------------------------------------------------ work plan
//
// The deposit / step kernels run a fixed grid of G CTAs over the flattened
// (p, N) particle index space; CTA b owns [start(b), start(b+1)) with
// start(b) = b*T/G, T = p*N, and writes one histogram row per instance it
// touches into segment row (b + j).  The solve kernel for instance j sums the
// rows of the CTAs covering [j*N, (j+1)*N) in CTA order -> deterministic.

struct Plan {
  int G;        // CTAs
  int K;        // lanes sharing one smem histogram
  int H;        // histograms per CTA
  size_t smem;  // dynamic smem bytes
};

static int hist_budget_bytes() {
  static int b = -1;
  if (b < 0) {
    const char* s = getenv("PICROM_HIST_KB");
    b = (s ? atoi(s) : 72) * 1024;
  }
  return b;
}

static int choose_k(int nx, int degree) {
  int budget = hist_budget_bytes();
  for (int k = 1; k <= 32; k <<= 1) {
    size_t bytes = (size_t)(nx + degree) * (kThreads / k) * sizeof(double);
    if ((int)bytes <= budget) return k;
  }
  return 32;
}

static size_t step_smem(int nx, int degree, int K, bool with_coef) {
  size_t h = (size_t)(nx + degree) * (kThreads / K) * sizeof(double);
  size_t c = with_coef ? (size_t)nx * degree * sizeof(double) : 0;
  return h + c + 64 * sizeof(double);
}

static int grid_for(long long total, size_t smem) {
  // one resident wave: SMs x CTAs-per-SM by shared memory, at most 8
  size_t per_sm = 227 * 1024;
  int occ = (int)std::min<size_t>(8, std::max<size_t>(1, per_sm / (smem + 1024)));
  long long want = (total + 2047) / 2048;     // >= 2048 particles per CTA
  long long g = std::min<long long>((long long)num_sms() * occ, std::max<long long>(1, want));
  return (int)g;
}

static Plan make_plan(long long n, int p, int nx, int degree, bool with_coef) {
  Plan pl;
  pl.K = choose_k(nx, degree);
  pl.H = kThreads / pl.K;
  pl.smem = step_smem(nx, degree, pl.K, with_coef);
  // grid independent of with_coef so workspace sizes agree across calls
  pl.G = grid_for((long long)n * p, step_smem(nx, degree, pl.K, true));
  return pl;
}

extern "C" size_t picrom_fom_workspace_bytes(long long n, int p, int nx, int degree) {
  Plan pl = make_plan(n, p, nx, degree, true);
  size_t rows = (size_t)pl.G + (size_t)p;
  return rows * (size_t)(nx + 1) * sizeof(double) + 256;
}

// b*T and flat*G stay far below 2^63 (T < 2^40, G < 2^16)
__device__ __forceinline__ long long cta_start(int b, long long T, int G) {
  return ((long long)b * T) / G;
}

__device__ __forceinline__ int cta_of(long long flat, long long T, int G) {
  int b = (int)((flat * (long long)G) / T);
  if (b >= G) b = G - 1;
  while (b + 1 < G && cta_start(b + 1, T, G) <= flat) ++b;
  while (b > 0 && cta_start(b, T, G) > flat) --b;
  return b;
}

// ---------------------------------------------------- fused step kernel
//
// MODE_DEPOSIT : deposit x                                 (deposit_charge)
// MODE_LEAPFROG: gather E(x), kick v, drift x, deposit x   (pic_step)
// MODE_DRIFT   : x1 = x + dt*(v + (0.5dt)*e0), deposit x1  (verlet_drift)

enum { MODE_DEPOSIT = 0, MODE_LEAPFROG = 1, MODE_DRIFT = 2 };

struct StepArgs {
  double* x;          // in (and out for LEAPFROG)
  double* v;          // LEAPFROG: in/out; DRIFT: in
  const double* e0;   // DRIFT
  double* xo;         // DRIFT output x1
  const double* phi;  // LEAPFROG
  const double* inst;
  long long n, ld;
  int p, nx;
  double dt, kick, kfull;
  long long step;
  double* seg_hist;   // (G + p) x nx
  double* seg_kin;    // (G + p)
  unsigned long long* status;
  const double* y;    // DEPOSIT: optional per-particle weights (rmatvec)
  int wkind;          // DEPOSIT: 0 value weights, 1 gradient weights
  const long long* counter;  // optional device step counter (graph replay)
};

template <int D, int K, int MODE>
__global__ void __launch_bounds__(kThreads)
step_kernel(StepArgs a) {
  extern __shared__ double smem[];
  constexpr int H = kThreads / K;
  constexpr int NW = D + 1;
  const int nx = a.nx;
  const int nh = nx + D;                       // histogram rows incl. ghost nodes
  double* hist = smem;                         // [nh][H]
  double* coef = hist + (size_t)nh * H;        // [D][nx] field polynomials
  double* red = coef + (MODE == MODE_LEAPFROG ? (size_t)nx * D : 0);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int myh = tid / K;
  const int klane = lane % K;
  const int G = gridDim.x;
  const long long T = a.n * (long long)a.p;
  const long long start = cta_start(blockIdx.x, T, G);
  const long long end = cta_start(blockIdx.x + 1, T, G);
  const double inv_nx = 1.0 / (double)nx;
  const long long step_id = a.counter ? (*a.counter + 1) : a.step;

  long long pos = start;
  while (pos < end) {
    const int j = (int)(pos / a.n);
    const long long seg_lo = pos - (long long)j * a.n;
    const long long seg_hi = min(a.n, end - (long long)j * a.n);
    const double* ip = a.inst + (size_t)j * PICROM_INST_STRIDE;
    const double h = ip[I_H];

    for (int q = tid; q < nh * H; q += kThreads) hist[q] = 0.0;
    if constexpr (MODE == MODE_LEAPFROG) {
      const double* ph = a.phi + (size_t)j * nx;
      const double ecoef = ip[I_ECOEF], g = ip[I_INVH];
      for (int c = tid; c < nx; c += kThreads) {
        double pv[D + 1];
#pragma unroll
        for (int m = 0; m <= D; ++m) pv[m] = ph[wrap_node(c + Spline<D>::OFF + m, nx)];
        double C[D];
        deriv_coeffs<D>(pv, ecoef, g, C);
#pragma unroll
        for (int k = 0; k < D; ++k) coef[k * nx + c] = C[k];
      }
    }
    __syncthreads();

    double kin = 0.0;
    const size_t base = (size_t)j * a.ld;
    // warp-uniform trip count so every lane joins the phase-serialised deposit
    for (long long i0 = seg_lo + (tid & ~31); i0 < seg_hi; i0 += kThreads) {
      const long long i = i0 + lane;
      const bool valid = i < seg_hi;
      double xn = 0.0;
      if (valid) {
        if constexpr (MODE == MODE_DEPOSIT) {
          xn = a.x[base + i];
        } else if constexpr (MODE == MODE_LEAPFROG) {
          double x = a.x[base + i];
          double v = a.v[base + i];
          int c;
          double f;
          locate(x, h, nx, inv_nx, c, f);
          double C[D];
#pragma unroll
          for (int k = 0; k < D; ++k) C[k] = coef[k * nx + c];
          double E = horner<D>(C, f);
          double vn = v + a.kfull * E;
          kin = fma(vn, vn, kin);
          double vh = __dadd_rn(v, __dmul_rn(a.kick, E));
          xn = __dadd_rn(x, __dmul_rn(a.dt, vh));
          a.x[base + i] = xn;
          a.v[base + i] = vh;
        } else {  // MODE_DRIFT: x1 = x + dt*(v + (0.5*dt)*e0), fullorder.py:127
          double x = a.x[base + i];
          double v = a.v[base + i];
          double e = a.e0[base + i];
          double vh = __dadd_rn(v, __dmul_rn(a.kick, e));
          xn = __dadd_rn(x, __dmul_rn(a.dt, vh));
          a.xo[base + i] = xn;
        }
      }
      const bool ok = valid && isfinite(xn);
      if (valid && !ok) record_bad(a.status, step_id, i, j, a.p);
      int c = 0;
      double f = 0.0;
      if (ok) locate(xn, h, nx, inv_nx, c, f);
      double w[NW];
      if constexpr (MODE == MODE_DEPOSIT) {
        if (a.wkind == 1) Spline<D>::dweights(f, ip[I_INVH], w);
        else Spline<D>::weights(f, w);
        if (a.y && valid) {
          const double yy = a.y[base + i];
#pragma unroll
          for (int m = 0; m < NW; ++m) w[m] *= yy;
        }
      } else {
        Spline<D>::weights(f, w);
      }
#pragma unroll
      for (int q = 0; q < K; ++q) {
        if (ok && klane == q) {
#pragma unroll
          for (int m = 0; m < NW; ++m) hist[(c + m) * H + myh] += w[m];
        }
        if constexpr (K > 1) __syncwarp();
      }
    }
    __syncthreads();

    // fold ghost rows, reduce the H histograms in fixed order -> segment row
    const int seg = blockIdx.x + j;
    for (int nd = tid; nd < nx; nd += kThreads) {
      double s = 0.0;
      // histogram row r holds node (r + OFF) mod nx: rows r0, r0 + nx, ... < nh
      for (int r = (nd - Spline<D>::OFF) % nx; r < nh; r += nx) {
        const double* row = hist + (size_t)r * H;
        for (int hh = 0; hh < H; ++hh) s += row[hh];
      }
      a.seg_hist[(size_t)seg * nx + nd] = s;
    }
    if constexpr (MODE == MODE_LEAPFROG) {
      double ks = block_sum(kin, red);
      if (tid == 0) a.seg_kin[seg] = ks;
    }
    __syncthreads();
    pos = (long long)(j + 1) * a.n;
  }
}

// ----------------------------------------------------- per-instance solve
//
// One CTA per instance.  rho = qw * (sum of segment rows) + bg*h   (or rho_in)
// phi = h * khat (*) (rho - mean) ;  phi -= mean ;  energy = 0.5/m_p phi^T L phi

struct SolveArgs {
  const double* seg_hist;   // if non-null: assemble rho from segments
  const double* seg_kin;
  const double* rho_in;     // else: rho given
  const double* inst;
  const double* khat;
  const double* stencil;
  long long n;
  int p, nx, degree, G;
  double* rho_out;          // may be null
  double* phi_out;          // may be null (deposit-only)
  double* energy_out;       // may be null
  double* kin_out;          // may be null
  bool solve;
  bool raw;                 // rho = plain segment sums (rmatvec)
  bool energy_only;         // rho_in holds phi: only the field energy
  long long* counter;       // optional device step counter: history row = *counter,
                            // incremented by the last CTA to finish
  unsigned int* done;       // ticket for the counter increment
  size_t hist_stride_rho;   // elements per history row (rho/phi)
  size_t hist_stride_e;     // elements per history row (energies)
  double* phi_hist;         // optional extra copy of phi (history)
};

__global__ void __launch_bounds__(512) solve_kernel(SolveArgs a) {
  extern __shared__ double sm[];
  const int nx = a.nx;
  double* rho = sm;            // nx
  double* kh = rho + nx;       // nx
  double* phi = kh + nx;       // nx
  double* red = phi + nx;      // 32
  const int j = blockIdx.x;
  const int tid = threadIdx.x;
  const double* ip = a.inst + (size_t)j * PICROM_INST_STRIDE;
  const double h = ip[I_H];
  const long long row = a.counter ? *a.counter : 0;
  double* rho_out = a.rho_out ? a.rho_out + row * a.hist_stride_rho : nullptr;
  double* phi_hist = a.phi_hist ? a.phi_hist + row * a.hist_stride_rho : nullptr;
  double* energy_out = a.energy_out ? a.energy_out + row * a.hist_stride_e : nullptr;
  double* kin_out = a.kin_out ? a.kin_out + row * a.hist_stride_e : nullptr;

  if (a.seg_hist) {
    const long long T = a.n * (long long)a.p;
    const int b_lo = cta_of((long long)j * a.n, T, a.G);
    const int b_hi = cta_of((long long)(j + 1) * a.n - 1, T, a.G);
    const double qw = ip[I_QW], bgh = ip[I_BGH];
    for (int nd = tid; nd < nx; nd += blockDim.x) {
      double s = 0.0;
      for (int b = b_lo; b <= b_hi; ++b) s += a.seg_hist[(size_t)(b + j) * nx + nd];
      rho[nd] = a.raw ? s : fma(qw, s, bgh);
    }
    if (kin_out && tid == 0) {
      double s = 0.0;
      for (int b = b_lo; b <= b_hi; ++b) s += a.seg_kin[b + j];
      kin_out[j] = 0.5 * s;
    }
  } else if (a.energy_only) {
    for (int nd = tid; nd < nx; nd += blockDim.x) phi[nd] = a.rho_in[(size_t)j * nx + nd];
  } else {
    for (int nd = tid; nd < nx; nd += blockDim.x) rho[nd] = a.rho_in[(size_t)j * nx + nd];
  }
  if (a.solve)
    for (int nd = tid; nd < nx; nd += blockDim.x) kh[nd] = a.khat[nd];
  __syncthreads();
  if (rho_out)
    for (int nd = tid; nd < nx; nd += blockDim.x) rho_out[(size_t)j * nx + nd] = rho[nd];
  if (!a.solve && !a.energy_only) return;

  double part = 0.0;
  if (!a.energy_only) {
  for (int nd = tid; nd < nx; nd += blockDim.x) part += rho[nd];
  const double mean_rho = block_sum(part, red) / (double)nx;
  for (int nd = tid; nd < nx; nd += blockDim.x) rho[nd] -= mean_rho;
  __syncthreads();
  // circulant solve phi_n = h * sum_m khat[(n - m) mod nx] b_m
  part = 0.0;
  for (int nd = tid; nd < nx; nd += blockDim.x) {
    double s = 0.0;
    int idx = nd;  // (nd - m) mod nx, m = 0..nx-1
    for (int m = 0; m < nx; ++m) {
      s = fma(kh[idx], rho[m], s);
      idx = (idx == 0) ? nx - 1 : idx - 1;
    }
    phi[nd] = h * s;
    part += phi[nd];
  }
  const double mean_phi = block_sum(part, red) / (double)nx;
  for (int nd = tid; nd < nx; nd += blockDim.x) phi[nd] -= mean_phi;
  __syncthreads();
  if (a.phi_out)
    for (int nd = tid; nd < nx; nd += blockDim.x) a.phi_out[(size_t)j * nx + nd] = phi[nd];
  }  // !energy_only
  if (phi_hist)
    for (int nd = tid; nd < nx; nd += blockDim.x) phi_hist[(size_t)j * nx + nd] = phi[nd];
  if (energy_out) {
    // L phi with L = stencil / h (circulant, half bandwidth d)
    const double inv_h = 1.0 / h;
    part = 0.0;
    for (int nd = tid; nd < nx; nd += blockDim.x) {
      double lp = a.stencil[0] * phi[nd];
      for (int k = 1; k <= a.degree; ++k) {
        int up = nd + k; if (up >= nx) up -= nx;
        int dn = nd - k; if (dn < 0) dn += nx;
        lp = fma(a.stencil[k], phi[up] + phi[dn], lp);
      }
      part = fma(phi[nd], lp * inv_h, part);
    }
    double e = block_sum(part, red);
    if (tid == 0) energy_out[j] = ip[I_HALFINVMP] * e;
  }
  if (a.counter) {
    // last CTA to finish advances the step counter (all CTAs read it above)
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      unsigned int t = atomicAdd(a.done, 1u);
      if (t == gridDim.x - 1) {
        *a.done = 0u;
        __threadfence();
        *a.counter = row + 1;
      }
    }
  }
}

static int launch_solve(const SolveArgs& a, cudaStream_t s) {
  int threads = std::min(512, std::max(64, ((a.nx + 31) / 32) * 32));
  size_t sm = (3 * (size_t)a.nx + 32) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  solve_kernel<<<a.p, threads, sm, s>>>(a);
  return check_launch("solve_kernel");
}

// --------------------------------------------------------- launch helpers

template <int D, int K, int MODE>
static int launch_step_t(const StepArgs& a, const Plan& pl, cudaStream_t s) {
  auto kfn = step_kernel<D, K, MODE>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  kfn<<<pl.G, kThreads, pl.smem, s>>>(a);
  return check_launch("step_kernel");
}

template <int D, int MODE>
static int launch_step_k(const StepArgs& a, const Plan& pl, cudaStream_t s) {
  switch (pl.K) {
    case 1: return launch_step_t<D, 1, MODE>(a, pl, s);
    case 2: return launch_step_t<D, 2, MODE>(a, pl, s);
    case 4: return launch_step_t<D, 4, MODE>(a, pl, s);
    case 8: return launch_step_t<D, 8, MODE>(a, pl, s);
    case 16: return launch_step_t<D, 16, MODE>(a, pl, s);
    default: return launch_step_t<D, 32, MODE>(a, pl, s);
  }
}

template <int MODE>
static int launch_step(const StepArgs& a, int degree, const Plan& pl, cudaStream_t s) {
  switch (degree) {
    case 1: return launch_step_k<1, MODE>(a, pl, s);
    case 2: return launch_step_k<2, MODE>(a, pl, s);
    case 3: return launch_step_k<3, MODE>(a, pl, s);
  }
  return set_err(PICROM_ERR_CONFIG, "degree must be 1, 2 or 3");
}

static int check_cfg(long long n, int p, int nx, int degree) {
  if (n < 1 || p < 1) return set_err(PICROM_ERR_CONFIG, "need n >= 1 and p >= 1");
  if (nx < 2) return set_err(PICROM_ERR_CONFIG, "need nx >= 2");
  if (degree < 1 || degree > 3) return set_err(PICROM_ERR_CONFIG, "degree must be 1, 2 or 3");
  if (degree > 1 && nx < 2 * degree + 1) return set_err(PICROM_ERR_CONFIG, "need nx >= 2*degree+1");
  if (nx > 8192) return set_err(PICROM_ERR_CONFIG, "nx > 8192 not supported");
  return PICROM_OK;
}

static void ws_split(void* ws, const Plan& pl, int p, int nx, double** hist, double** kin) {
  double* base = reinterpret_cast<double*>(ws);
  *hist = base;
  *kin = base + (size_t)(pl.G + p) * nx;
}

// ---------------------------------------------------------------- C-ABI

extern "C" int picrom_deposit(const double* x, long long n, int p, long long ld,
                              const double* inst, int nx, int degree, double* rho,
                              void* ws, unsigned long long* status, void* stream) {
  int rc = check_cfg(n, p, nx, degree);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  Plan pl = make_plan(n, p, nx, degree, false);
  StepArgs a{};
  a.x = const_cast<double*>(x);
  a.inst = inst; a.n = n; a.ld = ld; a.p = p; a.nx = nx; a.status = status;
  ws_split(ws, pl, p, nx, &a.seg_hist, &a.seg_kin);
  rc = launch_step<MODE_DEPOSIT>(a, degree, pl, s);
  if (rc) return rc;
  SolveArgs sa{};
  sa.seg_hist = a.seg_hist; sa.inst = inst; sa.n = n; sa.p = p; sa.nx = nx;
  sa.degree = degree; sa.G = pl.G; sa.rho_out = rho; sa.solve = false;
  return launch_solve(sa, s);
}

extern "C" int picrom_rmatvec(const double* x, const double* y, long long n, int p, long long ld,
                              const double* inst, int nx, int degree, int kind, double* out,
                              void* ws, unsigned long long* status, void* stream) {
  int rc = check_cfg(n, p, nx, degree);
  if (rc) return rc;
  if (kind != PICROM_TABLE_VALUE && kind != PICROM_TABLE_GRAD)
    return set_err(PICROM_ERR_CONFIG, "bad table kind");
  cudaStream_t s = (cudaStream_t)stream;
  Plan pl = make_plan(n, p, nx, degree, false);
  StepArgs a{};
  a.x = const_cast<double*>(x);
  a.y = y; a.wkind = kind;
  a.inst = inst; a.n = n; a.ld = ld; a.p = p; a.nx = nx; a.status = status;
  ws_split(ws, pl, p, nx, &a.seg_hist, &a.seg_kin);
  rc = launch_step<MODE_DEPOSIT>(a, degree, pl, s);
  if (rc) return rc;
  SolveArgs sa{};
  sa.seg_hist = a.seg_hist; sa.inst = inst; sa.n = n; sa.p = p; sa.nx = nx;
  sa.degree = degree; sa.G = pl.G; sa.rho_out = out; sa.solve = false; sa.raw = true;
  return launch_solve(sa, s);
}

extern "C" int picrom_poisson(const double* rho, int p, int nx, int degree, const double* inst,
                              const double* khat, const double* stencil, double* phi,
                              double* energy, void* stream) {
  int rc = check_cfg(1, p, nx, degree);
  if (rc) return rc;
  SolveArgs sa{};
  sa.rho_in = rho; sa.inst = inst; sa.khat = khat; sa.stencil = stencil; sa.n = 1;
  sa.p = p; sa.nx = nx; sa.degree = degree; sa.G = 1; sa.phi_out = phi;
  sa.energy_out = energy; sa.solve = true;
  return launch_solve(sa, (cudaStream_t)stream);
}

extern "C" int picrom_field_energy(const double* phi, int p, int nx, int degree,
                                   const double* inst, const double* stencil, double* energy,
                                   void* stream) {
  int rc = check_cfg(1, p, nx, degree);
  if (rc) return rc;
  SolveArgs sa{};
  sa.rho_in = phi; sa.inst = inst; sa.stencil = stencil; sa.n = 1; sa.p = p; sa.nx = nx;
  sa.degree = degree; sa.G = 1; sa.energy_out = energy; sa.energy_only = true;
  return launch_solve(sa, (cudaStream_t)stream);
}

extern "C" int picrom_pic_push(double* x, double* v, long long n, int p, long long ld,
                               const double* inst, int nx, int degree, const double* phi,
                               double dt, double kick, double kfull, long long step,
                               const long long* counter, void* ws,
                               unsigned long long* status, void* stream) {
  int rc = check_cfg(n, p, nx, degree);
  if (rc) return rc;
  Plan pl = make_plan(n, p, nx, degree, true);
  StepArgs a{};
  a.x = x; a.v = v; a.phi = phi; a.inst = inst; a.n = n; a.ld = ld; a.p = p; a.nx = nx;
  a.dt = dt; a.kick = kick; a.kfull = kfull; a.step = step + 1; a.status = status;
  a.counter = counter;
  ws_split(ws, pl, p, nx, &a.seg_hist, &a.seg_kin);
  return launch_step<MODE_LEAPFROG>(a, degree, pl, (cudaStream_t)stream);
}

extern "C" int picrom_pic_solve(long long n, int p, int nx, int degree, const double* inst,
                                const double* khat, const double* stencil, double* phi,
                                long long step, long long* counter, double* rho_hist,
                                double* phi_hist, double* ee_hist, double* kin_hist, void* ws,
                                void* stream) {
  int rc = check_cfg(n, p, nx, degree);
  if (rc) return rc;
  Plan pl = make_plan(n, p, nx, degree, true);
  SolveArgs sa{};
  double* kin_seg;
  ws_split(ws, pl, p, nx, const_cast<double**>(&sa.seg_hist), &kin_seg);
  sa.seg_kin = kin_seg;
  sa.inst = inst; sa.khat = khat;
  sa.stencil = stencil; sa.n = n; sa.p = p; sa.nx = nx; sa.degree = degree; sa.G = pl.G;
  sa.solve = true; sa.phi_out = phi;
  const size_t gp = (size_t)p * nx;
  sa.hist_stride_rho = gp;
  sa.hist_stride_e = (size_t)p;
  if (counter) {
    sa.counter = counter;
    sa.done = reinterpret_cast<unsigned int*>(counter + 1);
    sa.rho_out = rho_hist; sa.phi_hist = phi_hist; sa.energy_out = ee_hist; sa.kin_out = kin_hist;
  } else {
    sa.rho_out = rho_hist ? rho_hist + (size_t)step * gp : nullptr;
    sa.phi_hist = phi_hist ? phi_hist + (size_t)step * gp : nullptr;
    sa.energy_out = ee_hist ? ee_hist + (size_t)step * p : nullptr;
    sa.kin_out = kin_hist ? kin_hist + (size_t)step * p : nullptr;
  }
  return launch_solve(sa, (cudaStream_t)stream);
}

extern "C" int picrom_pic_step(double* x, double* v, long long n, int p, long long ld,
                               const double* inst, int nx, int degree, const double* khat,
                               const double* stencil, double* phi, double dt, double kick,
                               double kfull, long long step, long long* counter,
                               double* rho_hist, double* phi_hist, double* ee_hist,
                               double* kin_hist, void* ws, unsigned long long* status,
                               void* stream) {
  int rc = picrom_pic_push(x, v, n, p, ld, inst, nx, degree, phi, dt, kick, kfull, step, counter,
                           ws, status, stream);
  if (rc) return rc;
  return picrom_pic_solve(n, p, nx, degree, inst, khat, stencil, phi, step, counter, rho_hist,
                          phi_hist, ee_hist, kin_hist, ws, stream);
}

extern "C" int picrom_verlet_drift(const double* x, const double* v, const double* e0,
                                   long long n, int p, long long ld, const double* inst, int nx,
                                   int degree, const double* khat, const double* stencil,
                                   double dt, long long step, double* x1, double* phi1,
                                   double* rho1, double* energy1, void* ws,
                                   unsigned long long* status, void* stream) {
  int rc = check_cfg(n, p, nx, degree);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  Plan pl = make_plan(n, p, nx, degree, false);
  StepArgs a{};
  a.x = const_cast<double*>(x); a.v = const_cast<double*>(v); a.e0 = e0; a.xo = x1;
  a.inst = inst; a.n = n; a.ld = ld; a.p = p; a.nx = nx; a.dt = dt; a.kick = 0.5 * dt;
  a.step = step; a.status = status;
  ws_split(ws, pl, p, nx, &a.seg_hist, &a.seg_kin);
  rc = launch_step<MODE_DRIFT>(a, degree, pl, s);
  if (rc) return rc;
  SolveArgs sa{};
  sa.seg_hist = a.seg_hist; sa.inst = inst; sa.khat = khat; sa.stencil = stencil; sa.n = n;
  sa.p = p; sa.nx = nx; sa.degree = degree; sa.G = pl.G; sa.solve = true; sa.phi_out = phi1;
  sa.rho_out = rho1; sa.energy_out = energy1;
  return launch_solve(sa, s);
}

// ------------------------------------------------------ gather kernels

struct GatherArgs {
  const double* x;
  const double* phi;
  const double* inst;
  const double* v;     // kick: v
  const double* e0;    // kick: e0
  double* out;         // gather output (or e1 for kick)
  double* v1;          // kick output
  long long n, ld, ldo;
  int p, nx, kind;
  double dt;
  unsigned long long* status;
};

constexpr int kChunk = 4096;   // particles per gather CTA

template <int D, bool KICK>
__global__ void __launch_bounds__(kThreads) gather_kernel(GatherArgs a) {
  extern __shared__ double coef[];    // [NC][nx]
  const int nx = a.nx;
  const int j = blockIdx.y;
  const double* ip = a.inst + (size_t)j * PICROM_INST_STRIDE;
  const double h = ip[I_H], g = ip[I_INVH];
  const double* ph = a.phi + (size_t)j * nx;
  const int kind = KICK ? PICROM_GATHER_FIELD : a.kind;
  const int NC = (kind == PICROM_GATHER_VALUE) ? D + 1 : D;
  const double cf = (kind == PICROM_GATHER_GRAD) ? ip[I_GCOEF]
                  : (kind == PICROM_GATHER_DERIV) ? 1.0 : ip[I_ECOEF];
  for (int c = threadIdx.x; c < nx; c += blockDim.x) {
    double pv[D + 1];
#pragma unroll
    for (int m = 0; m <= D; ++m) pv[m] = ph[wrap_node(c + Spline<D>::OFF + m, nx)];
    double C[D + 1];
    if (kind == PICROM_GATHER_VALUE) value_coeffs<D>(pv, C);
    else deriv_coeffs<D>(pv, cf, g, C);
    for (int k = 0; k < NC; ++k) coef[k * nx + c] = C[k];
  }
  __syncthreads();
  const double inv_nx = 1.0 / (double)nx;
  const long long lo = (long long)blockIdx.x * kChunk;
  const long long hi = min(a.n, lo + (long long)kChunk);
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const size_t at = (size_t)j * a.ld + i;
    const double x = a.x[at];
    if (!isfinite(x)) {
      record_bad(a.status, 0, i, j, a.p);
      continue;
    }
    int c;
    double f;
    locate(x, h, nx, inv_nx, c, f);
    double r;
    if (kind == PICROM_GATHER_VALUE) {
      if constexpr (D == 1) {
        r = __dadd_rn(__dmul_rn(__dsub_rn(1.0, f), coef[c]), __dmul_rn(f, coef[nx + c]));
      } else {
        double C[D + 1];
#pragma unroll
        for (int k = 0; k <= D; ++k) C[k] = coef[k * nx + c];
        r = horner<D + 1>(C, f);
      }
    } else {
      double C[D];
#pragma unroll
      for (int k = 0; k < D; ++k) C[k] = coef[k * nx + c];
      r = horner<D>(C, f);
    }
    if constexpr (KICK) {
      // v1 = v + 0.5*dt*(e0 + e1)  -- fullorder.py:130 operation order
      const double e0 = a.e0[at];
      a.out[(size_t)j * a.ldo + i] = r;
      a.v1[(size_t)j * a.ldo + i] =
          __dadd_rn(a.v[at], __dmul_rn(__dmul_rn(0.5, a.dt), __dadd_rn(e0, r)));
    } else {
      a.out[(size_t)j * a.ldo + i] = r;
    }
  }
}

template <bool KICK>
static int launch_gather(const GatherArgs& a, int degree, cudaStream_t s) {
  dim3 grid((unsigned)((a.n + kChunk - 1) / kChunk), (unsigned)a.p);
  size_t sm = (size_t)(degree + 1) * a.nx * sizeof(double);
  if (grid.y > 65535) return set_err(PICROM_ERR_CONFIG, "p > 65535");
  switch (degree) {
    case 1: gather_kernel<1, KICK><<<grid, kThreads, sm, s>>>(a); break;
    case 2: gather_kernel<2, KICK><<<grid, kThreads, sm, s>>>(a); break;
    case 3: gather_kernel<3, KICK><<<grid, kThreads, sm, s>>>(a); break;
    default: return set_err(PICROM_ERR_CONFIG, "degree must be 1, 2 or 3");
  }
  return check_launch("gather_kernel");
}

extern "C" int picrom_gather(const double* x, long long n, int p, long long ld,
                             const double* inst, int nx, int degree, const double* phi,
                             int kind, double* out, long long ldo,
                             unsigned long long* status, void* stream) {
  int rc = check_cfg(n, p, nx, degree);
  if (rc) return rc;
  if (kind < 0 || kind > 3) return set_err(PICROM_ERR_CONFIG, "bad gather kind");
  GatherArgs a{};
  a.x = x; a.phi = phi; a.inst = inst; a.out = out; a.n = n; a.ld = ld; a.ldo = ldo;
  a.p = p; a.nx = nx; a.kind = kind; a.status = status;
  return launch_gather<false>(a, degree, (cudaStream_t)stream);
}

extern "C" int picrom_verlet_kick(const double* x1, const double* v, const double* e0,
                                  long long n, int p, long long ld, const double* inst, int nx,
                                  int degree, const double* phi1, double dt, double* e1,
                                  double* v1, void* stream) {
  int rc = check_cfg(n, p, nx, degree);
  if (rc) return rc;
  GatherArgs a{};
  a.x = x1; a.phi = phi1; a.inst = inst; a.v = v; a.e0 = e0; a.out = e1; a.v1 = v1;
  a.n = n; a.ld = ld; a.ldo = ld; a.p = p; a.nx = nx; a.kind = PICROM_GATHER_FIELD; a.dt = dt;
  return launch_gather<true>(a, degree, (cudaStream_t)stream);
}

// ------------------------------------------------------ locate / tables

template <int D>
__global__ void __launch_bounds__(kThreads) table_kernel(const double* x, long long n, int p,
                                                         long long ld, const double* inst, int nx,
                                                         int kind, long long* i0, double* w,
                                                         long long ldo, unsigned long long* status) {
  const long long T = n * (long long)p;
  const double inv_nx = 1.0 / (double)nx;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t / n);
    const long long i = t - (long long)j * n;
    const double* ip = inst + (size_t)j * PICROM_INST_STRIDE;
    const double xv = x[(size_t)j * ld + i];
    if (!isfinite(xv)) {
      record_bad(status, 0, i, j, p);
      continue;
    }
    int c;
    double f;
    locate(xv, ip[I_H], nx, inv_nx, c, f);
    const size_t o = (size_t)j * ldo + i;
    if (i0) i0[o] = c;
    if (!w) continue;
    if (D == 0) {  // locate only: w is frac
      w[o] = f;
      continue;
    }
    const size_t plane = (size_t)p * ldo;
    if (kind == PICROM_TABLE_VALUE) {
      double ww[4];
      if constexpr (D == 1) Spline<1>::weights(f, ww);
      if constexpr (D == 2) Spline<2>::weights(f, ww);
      if constexpr (D == 3) Spline<3>::weights(f, ww);
      for (int m = 0; m <= D; ++m) w[m * plane + o] = ww[m];
    } else {
      const double g = ip[I_INVH];
      if constexpr (D == 1) {
        w[o] = -g;
        w[plane + o] = g;
      } else if constexpr (D == 2) {
        w[o] = (f - 1.0) * g;
        w[plane + o] = (1.0 - 2.0 * f) * g;
        w[2 * plane + o] = f * g;
      } else if constexpr (D == 3) {
        const double e = 1.0 - f;
        w[o] = (-0.5 * e * e) * g;
        w[plane + o] = (1.5 * f * f - 2.0 * f) * g;
        w[2 * plane + o] = (-1.5 * f * f + f + 0.5) * g;
        w[3 * plane + o] = (0.5 * f * f) * g;
      }
    }
  }
}

static int table_grid(long long T) {
  long long b = (T + kThreads - 1) / kThreads;
  return (int)std::max<long long>(1, std::min<long long>(b, (long long)num_sms() * 8));
}

extern "C" int picrom_locate(const double* x, long long n, int p, long long ld,
                             const double* inst, int nx, long long* i0, double* frac,
                             long long ldo, unsigned long long* status, void* stream) {
  int rc = check_cfg(n, p, nx, 1);
  if (rc) return rc;
  table_kernel<0><<<table_grid(n * p), kThreads, 0, (cudaStream_t)stream>>>(
      x, n, p, ld, inst, nx, 0, i0, frac, ldo, status);
  return check_launch("locate");
}

extern "C" int picrom_basis_table(const double* x, long long n, int p, long long ld,
                                  const double* inst, int nx, int degree, int kind,
                                  long long* i0, double* w, long long ldo,
                                  unsigned long long* status, void* stream) {
  int rc = check_cfg(n, p, nx, degree);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  int g = table_grid(n * p);
  switch (degree) {
    case 1: table_kernel<1><<<g, kThreads, 0, s>>>(x, n, p, ld, inst, nx, kind, i0, w, ldo, status); break;
    case 2: table_kernel<2><<<g, kThreads, 0, s>>>(x, n, p, ld, inst, nx, kind, i0, w, ldo, status); break;
    case 3: table_kernel<3><<<g, kThreads, 0, s>>>(x, n, p, ld, inst, nx, kind, i0, w, ldo, status); break;
  }
  return check_launch("basis_table");
}

// ------------------------------------------------------------- reductions

__global__ void half_sumsq_kernel(const double* a, long long n, long long ld, double* out) {
  __shared__ double red[32];
  const int j = blockIdx.x;
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    double v = a[(size_t)j * ld + i];
    s = fma(v, v, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[j] = 0.5 * s;
}

extern "C" int picrom_half_sumsq(const double* a, long long n, int p, long long ld, double* out,
                                 void* ws, void* stream) {
  (void)ws;
  if (n < 1 || p < 1) return set_err(PICROM_ERR_CONFIG, "need n, p >= 1");
  half_sumsq_kernel<<<p, 1024, 0, (cudaStream_t)stream>>>(a, n, ld, out);
  return check_launch("half_sumsq");
}

// ------------------------------------------------------------- transposes

template <typename T>
__global__ void transpose_kernel(const T* in, long long rows, long long cols, T* out) {
  __shared__ T tile[32][33];
  const long long r0 = (long long)blockIdx.x * 32, c0 = (long long)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    long long r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    long long c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][k];
  }
}

template <typename T>
static int do_transpose(const T* in, long long rows, long long cols, T* out, void* stream) {
  if (rows < 1 || cols < 1) return PICROM_OK;
  long long gx = (rows + 31) / 32, gy = (cols + 31) / 32;
  if (gy > 65535 || gx > 2147483647LL) return set_err(PICROM_ERR_CONFIG, "transpose too large");
  dim3 grid((unsigned)gx, (unsigned)gy), block(32, 8);
  transpose_kernel<T><<<grid, block, 0, (cudaStream_t)stream>>>(in, rows, cols, out);
  return check_launch("transpose");
}

extern "C" int picrom_transpose(const double* in, long long rows, long long cols, double* out,
                                void* stream) {
  return do_transpose<double>(in, rows, cols, out, stream);
}

extern "C" int picrom_transpose_i64(const long long* in, long long rows, long long cols,
                                    long long* out, void* stream) {
  return do_transpose<long long>(in, rows, cols, out, stream);
}
