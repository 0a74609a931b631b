// Full-order PIC kernels for sm_100a: locate, basis tables, deposit, Poisson,
// gather, fused leapfrog step, reference-order Verlet, transposes.
//
// Reference: /root/reference/pkg/src/picrom/fem.py and fullorder.py (see the
// per-function citations in include/picrom_b200.h).  Design notes: DESIGN.md.

#include <cooperative_groups.h>
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

__global__ void timestamp_kernel(unsigned long long* out) {
  unsigned long long now;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
  *out = now;
}

extern "C" int picrom_timestamp(unsigned long long* out, void* stream) {
  timestamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(out);
  return check_launch("timestamp");
}

// internal (C++ linkage) helpers shared with rom.cu
int picrom_set_error(int code, const char* msg) { return set_err(code, msg); }
int picrom_check_launch(const char* what) { return check_launch(what); }
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

static int num_sms();
int picrom_num_sms() { return num_sms(); }

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

// Allow a kernel the largest dynamic shared memory the SM offers next to its
// static shared memory (227 KB per block on sm_100 in total).
template <typename F>
static void allow_max_dynamic_smem(F kfn) {
  cudaFuncAttributes at{};
  cudaFuncGetAttributes(&at, kfn);
  const int total = 227 * 1024;
  if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           total - (int)at.sharedSizeBytes) != cudaSuccess)
    (void)cudaGetLastError();   // do not leave a stale error for the next launch check
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
  int K;        // lanes sharing one smem histogram (phase path)
  int H;        // histograms per CTA (phase path)
  size_t smem;  // dynamic smem bytes (phase path)
  size_t fsmem; // dynamic smem bytes (fixed-point path)
};

// shared-memory budget of the K-lane histograms (72 KB: K = 2 at C2's Nx = 128,
// 3 CTAs per SM; profiles/r01b measured K = 4 / 8 slower there)
constexpr int kHistBudget = 72 * 1024;
// minimum particles per CTA segment
constexpr int kMinSeg = 2048;

// 128 threads per CTA measured best (profiles/r01; 256 was slower at every K)
static int step_nt() { return 128; }

// lanes per histogram: the fewest whose histograms fit the budget; beyond
// K = 16 (Nx > ~1150) one histogram per warp (K = 32: cell-mod-4 phases with
// match-ranked rounds, measured 2.3x slower than K = 8 at C5 but the only
// option once K-lane groups no longer fit)
static int choose_k(int nx, int degree) {
  for (int k = 1; k <= 16; k <<= 1) {
    size_t bytes = (size_t)(nx + degree) * (step_nt() / k) * sizeof(double);
    if ((int)bytes <= kHistBudget) return k;
  }
  return 32;
}

static size_t step_smem(int nx, int degree, int K, bool with_coef) {
  size_t h = (size_t)(nx + degree) * (step_nt() / K) * sizeof(double);
  // LEAPFROG: per-cell field polynomials + the solve's khat (padded) and stencil,
  // preloaded at CTA start so the last-CTA solve tail has no global round trip for them
  size_t c = with_coef ? ((size_t)nx * degree + (size_t)(nx + nx / 4 + 4) + 8) * sizeof(double) : 0;
  return h + c + 64 * sizeof(double);
}

static int grid_for(long long n, int p, int occ) {
  // exactly one resident wave: SMs x CTAs-per-SM (queried for the kernel)
  const long long total = n * p;
  const long long slots = (long long)num_sms() * std::max(occ, 1);
  long long want = (total + kMinSeg - 1) / kMinSeg;     // >= kMinSeg particles per CTA
  long long g = std::min<long long>(slots, std::max<long long>(1, want));
  // instance-aligned grid (G = m p): no CTA range straddles two instances, so
  // no CTA pays a second prologue/fold/ticket (those were the step's
  // stragglers, ~7 us at C2, profiles/r02 timeline) -- when it idles <= 1/16
  // of the slots
  if (p <= g) {
    long long m = g / p;
#ifdef PICROM_CLUSTER_MAXM
    m = std::min<long long>(m, PICROM_CLUSTER_MAXM);     // dev variant: cluster-sized grids
    g = m * p;
#endif
    if ((g - m * p) * 16 <= g) g = m * p;
  }
  return (int)g;
}

// fixed-point path: [3][nx+D] u32 limbs | [nx] fp64 | [D][nx] field polynomials
// | 64 | khat (padded) + stencil; at least the solve tail's scratch
static size_t fix_smem(int nx, int degree) {
  const size_t limb_d = (size_t)(3 * (nx + degree) + 1) / 2;
  const size_t front = limb_d + nx + (size_t)nx * degree + 64;
  const size_t solve = (size_t)2 * nx + (nx + nx / 4 + 4) + 40 + 8;
  return (std::max(front, solve) + (nx + nx / 4 + 4) + 8) * sizeof(double);
}

static int fix_occupancy(int degree, size_t smem);
static int step_occupancy(int degree, int K, size_t smem);

static Plan make_plan(long long n, int p, int nx, int degree, bool with_coef) {
  Plan pl;
  pl.K = choose_k(nx, degree);
  pl.H = step_nt() / pl.K;
  pl.smem = step_smem(nx, degree, pl.K, with_coef);
  pl.fsmem = fix_smem(nx, degree);
  // grid independent of the mode so workspace sizes agree across calls: the
  // occupancy of the leapfrog kernel of this shape (phase path for K <= 2,
  // fixed-point otherwise) sizes it
  const int occ = pl.K > 2 ? fix_occupancy(degree, pl.fsmem)
                           : step_occupancy(degree, pl.K, step_smem(nx, degree, pl.K, true));
  pl.G = grid_for(n, p, occ);
  return pl;
}

static size_t seg_rows(const Plan& pl, int p) { return (size_t)pl.G + (size_t)p; }

extern "C" size_t picrom_fom_workspace_bytes(long long n, int p, int nx, int degree) {
  Plan pl = make_plan(n, p, nx, degree, true);
  const size_t rows = seg_rows(pl, p);
  return rows * (size_t)(nx + 1) * sizeof(double) + (size_t)(p + 1) * sizeof(unsigned int) + 256;
}

// b*T and flat*G stay far below 2^63 (T < 2^40, G < 2^16)
__device__ __forceinline__ long long cta_start(int b, long long T, int G) {
  return ((long long)b * T) / G;
}

// CTA owning flat index f: the largest b with floor(b T / G) <= f, i.e.
// b = ceil((f + 1) G / T) - 1 = ((f + 1) G - 1) / T  (one exact division)
__device__ __forceinline__ int cta_of(long long flat, long long T, int G) {
  const long long b = ((flat + 1) * (long long)G - 1) / T;
  return (int)(b < G ? b : G - 1);
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
  // fused solve (LEAPFROG): the last CTA finishing an instance solves it
  int fuse_solve;
  unsigned int* inst_done;   // p tickets (zeroed; left zeroed)
  int cluster_m;             // > 0: the m CTAs of an instance form one thread-block
                             // cluster; partial rows go through DSMEM, rank 0 solves
};

#ifdef PICROM_EXP_TIMING
// timing experiment only: %globaltimer stamps of instance 0's tail CTA
__device__ unsigned long long g_ts[16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TSTAMP(k, cond) do { if ((cond) && threadIdx.x == 0) g_ts[k] = gtimer(); } while (0)
extern "C" int picrom_debug_timestamps(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_ts, sizeof(g_ts)) == cudaSuccess ? 0 : -1;
}
#else
#define TSTAMP(k, cond) do { } while (0)
#endif

#ifdef PICROM_EXP_TIMELINE
// timing experiment only: per-CTA %globaltimer timeline of the leapfrog pass
// (slot per CTA launch: [step, instance, t_entry, t_prologue, t_stream_end,
//  t_fold, t_ticket, t_solve_end]); tools/timeline.py reads it back
__device__ unsigned long long g_tl[16384][8];
__device__ unsigned int g_tl_ctr;
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
extern "C" int picrom_debug_timeline(unsigned long long* out, int rows, int reset) {
  if (reset) {
    unsigned int z = 0;
    static unsigned long long zeros[16384 * 8];
    if (cudaMemcpyToSymbol(g_tl, zeros, sizeof(zeros)) != cudaSuccess) return -1;
    return cudaMemcpyToSymbol(g_tl_ctr, &z, sizeof(z)) == cudaSuccess ? 0 : -1;
  }
  return cudaMemcpyFromSymbol(out, g_tl, (size_t)rows * 8 * sizeof(unsigned long long)) == cudaSuccess ? 0 : -1;
}
#define TL(k) do { if (MODE == MODE_LEAPFROG && threadIdx.x == 0 && tl_slot >= 0) g_tl[tl_slot][k] = tl_now(); } while (0)
#else
#define TL(k) do { } while (0)
#endif

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
  int seg_dense;            // > 0: dense segments seg[(b*p + j)*nx + nd], b < seg_dense
  long long hist_mod;       // > 0: history row = counter % hist_mod (ring)
  const int* cols;          // optional instance id per column
  size_t scratch;           // solve_kernel: dynamic smem in doubles
  unsigned long long* t_hist;  // optional %globaltimer (ns) per history row, written
                               // when the counter advances (the step's last solve)
  const long long* skip;       // nullable device flag: nonzero -> solve_kernel does nothing
};

// sum of cnt values v[0], v[stride], ... with 8 independent loads in flight,
// combined in a fixed order (deterministic)
__device__ __forceinline__ double ordered_sum(const double* v, size_t stride, int cnt) {
  if (cnt > 16 && cnt <= 32) {   // one round of loads for up to 32 rows (C1: 48 rows, 2 parts)
    double t[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) t[u] = u < cnt ? __ldcg(v + (size_t)u * stride) : 0.0;
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = (t[u] + t[u + 8]) + (t[u + 16] + t[u + 24]);
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  }
  if (cnt <= 16) {   // common case: every load in flight at once, same sum order
    double t[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) t[u] = u < cnt ? __ldcg(v + (size_t)u * stride) : 0.0;
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = t[u] + t[u + 8];
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  }
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int b = 0;
  for (; b + 8 <= cnt; b += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] += __ldcg(v + (size_t)(b + u) * stride);
  }
  for (int u = 0; b < cnt; ++b, ++u) acc[u] += __ldcg(v + (size_t)b * stride);
  return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

// smem (doubles) the solve needs with mp partial rows; khat is stored with
// one pad slot per 4 entries so the circulant's strided window loads are
// bank-conflict free
__host__ __device__ inline int solve_kh_len(int nx) { return nx + nx / 4 + 4; }
__host__ __device__ inline size_t solve_scratch(int nx, int mp) {
  return (size_t)nx + solve_kh_len(nx) + 40 + (size_t)mp * nx;
}
__host__ __device__ inline int solve_mp(int nx, int threads, size_t avail) {
  const int og = (nx + 127) / 128;
  int mp = (threads / 32) / og;
  while (mp > 1 && solve_scratch(nx, mp) > avail) --mp;
  return mp < 1 ? 1 : mp;
}
__device__ __forceinline__ int kh_pad(int r) { return r + (r >> 2); }

// One instance's assembly + solve by a whole CTA; `sm` holds `avail`
// doubles (>= solve_scratch(nx, 1)); `ntickets` = how many instance solves
// make up this step (the last one to finish advances the step counter).
// kh_pre / stn_pre (nullable): khat (padded, kh_pad) and the stencil already
// in shared memory; crow_pre >= 0: the step counter value already read.
__device__ void solve_body(const SolveArgs& a, int j, double* sm, unsigned int ntickets,
                           size_t avail, const double* kh_pre = nullptr,
                           const double* stn_pre = nullptr, long long crow_pre = -1,
                           bool rho_ready = false, double kin_ready = 0.0) {
  const int nx = a.nx;
  double* rho = sm;                      // nx (phi overwrites it after the circulant)
  double* kh = rho + nx;                 // khat, padded (kh_pad)
  double* red = kh + solve_kh_len(nx);   // 32 (block reductions) + 8 (stencil)
  double* stn = red + 32;
  double* prow = red + 40;               // mp x nx circulant partial rows
  double* phi = rho;
  const int mp = solve_mp(nx, blockDim.x, avail);
  const int tid = threadIdx.x;
  if (stn_pre) stn = const_cast<double*>(stn_pre);
  else if (a.stencil && tid <= a.degree) stn[tid] = a.stencil[tid];
  const double* ip = a.inst + (size_t)(a.cols ? a.cols[j] : j) * PICROM_INST_STRIDE;
  const double h = ip[I_H];
  const long long crow = crow_pre >= 0 ? crow_pre : (a.counter ? *a.counter : 0);
  const long long row = a.hist_mod > 0 ? crow % a.hist_mod : crow;
  double* rho_out = a.rho_out ? a.rho_out + row * a.hist_stride_rho : nullptr;
  double* phi_hist = a.phi_hist ? a.phi_hist + row * a.hist_stride_rho : nullptr;
  double* energy_out = a.energy_out ? a.energy_out + row * a.hist_stride_e : nullptr;
  double* kin_out = a.kin_out ? a.kin_out + row * a.hist_stride_e : nullptr;

  if (rho_ready) {
    // rho already assembled in sm[0, nx) by the caller (cluster path)
    if (kin_out && tid == 0) kin_out[j] = 0.5 * kin_ready;
  } else if (a.seg_dense > 0) {
    const double qw = ip[I_QW], bgh = ip[I_BGH];
    for (int nd = tid; nd < nx; nd += blockDim.x) {
      const double s = ordered_sum(a.seg_hist + (size_t)j * nx + nd, (size_t)a.p * nx, a.seg_dense);
      rho[nd] = a.raw ? s : fma(qw, s, bgh);
    }
  } else if (a.seg_hist) {
    const long long T = a.n * (long long)a.p;
    const int b_lo = cta_of((long long)j * a.n, T, a.G);
    const int b_hi = cta_of((long long)(j + 1) * a.n - 1, T, a.G);
    const int cnt = b_hi - b_lo + 1;
    const double qw = ip[I_QW], bgh = ip[I_BGH];
    const double* base = a.seg_hist + (size_t)(b_lo + j) * nx;
    const int nparts = max(1, min(min((int)(blockDim.x / nx), mp), (cnt + 15) / 16));
    if (nparts == 1) {
      for (int nd = tid; nd < nx; nd += blockDim.x) {
        const double s = ordered_sum(base + nd, nx, cnt);
        rho[nd] = a.raw ? s : fma(qw, s, bgh);
      }
    } else {
      // many segment rows (one instance over many CTAs, e.g. C1): nparts
      // threads per node sum consecutive row ranges in parallel (one round of
      // loads each), then the parts are added in order
      double* part_s = red + 40;                 // nparts x nx (solve scratch)
      const int per = (cnt + nparts - 1) / nparts;
      const int nd = tid % nx, q = tid / nx;
      if (q < nparts) {
        const int r0 = q * per, r1 = min(cnt, r0 + per);
        part_s[q * nx + nd] = r1 > r0 ? ordered_sum(base + (size_t)r0 * nx + nd, nx, r1 - r0) : 0.0;
      }
      __syncthreads();
      for (int m = tid; m < nx; m += blockDim.x) {
        double s = part_s[m];
        for (int qq = 1; qq < nparts; ++qq) s += part_s[qq * nx + m];
        rho[m] = a.raw ? s : fma(qw, s, bgh);
      }
      __syncthreads();
    }
    if (kin_out && tid < 32) {                   // warp-parallel, fixed lane tree
      double k = 0.0;
      for (int b = tid; b < cnt; b += 32) k += __ldcg(a.seg_kin + b_lo + j + b);
      k = warp_sum(k);
      if (tid == 0) kin_out[j] = 0.5 * k;
    }
  } else if (a.energy_only) {
    for (int nd = tid; nd < nx; nd += blockDim.x) phi[nd] = a.rho_in[(size_t)j * nx + nd];
  } else {
    for (int nd = tid; nd < nx; nd += blockDim.x) rho[nd] = a.rho_in[(size_t)j * nx + nd];
  }
  if (kh_pre) kh = const_cast<double*>(kh_pre);
  else if (a.solve)
    for (int r = tid; r < nx; r += blockDim.x) kh[kh_pad(r)] = a.khat[r];
  __syncthreads();
  TSTAMP(4, j == 0);
  if (rho_out)
    for (int nd = tid; nd < nx; nd += blockDim.x) rho_out[(size_t)j * nx + nd] = rho[nd];
  if (!a.solve && !a.energy_only) return;

  // Means by every warp redundantly (one fixed lane order, identical in all
  // warps): no block barrier for a reduction whose result every thread needs
  auto warp_mean = [&](const double* v) {
    const int lane = tid & 31;
    double t = 0.0;
    for (int q = lane; q < nx; q += 32) t += v[q];
    return warp_sum(t) / (double)nx;
  };
  const double inv_h = 1.0 / h;
  double part = 0.0;
  if (!a.energy_only) {
  const double mean_rho = warp_mean(rho);
  TSTAMP(5, j == 0);
#ifdef PICROM_EXP_NOCIRC
  if (false)     // timing experiment only
#endif
  // circulant solve phi_n = h * sum_m khat[(n - m) mod nx] (rho_m - mean).  A
  // lane owns 4 consecutive outputs and keeps khat[(n0 + i - m) mod nx], i < 4,
  // in a register window that slides by one smem load per step of m (1 load
  // per 4 FMAs); warps split the m range into mp parts, summed in fixed order.
  {
    const int nw = blockDim.x >> 5, warp = tid >> 5, lane = tid & 31;
    const int og = (nx + 127) >> 7;
    const int mlen = (nx + mp - 1) / mp;
    for (int t = warp; t < og * mp; t += nw) {
      const int q = t / og;
      const int n0 = (t - q * og) * 128 + lane * 4;
      const int mlo = q * mlen, mhi = min(nx, mlo + mlen);
      if (n0 >= nx || mlo >= mhi) continue;
      int idx = n0 - mlo;                     // (n0 - m) mod nx at m = mlo
      if (idx < 0) idx += nx;
      auto up = [nx](int r) { r += 1; return r >= nx ? r - nx : r; };
      auto dn = [nx](int r) { r -= 1; return r < 0 ? r + nx : r; };
      const int i1 = up(idx), i2 = up(i1), i3 = up(i2);
      double w0 = kh[kh_pad(idx)], w1 = kh[kh_pad(i1)], w2 = kh[kh_pad(i2)], w3 = kh[kh_pad(i3)];
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int m = mlo;
      for (; m + 4 <= mhi; m += 4) {
        const double b0 = rho[m] - mean_rho, b1 = rho[m + 1] - mean_rho;
        const double b2 = rho[m + 2] - mean_rho, b3 = rho[m + 3] - mean_rho;
        a0 = fma(w0, b0, a0); a1 = fma(w1, b0, a1); a2 = fma(w2, b0, a2); a3 = fma(w3, b0, a3);
        idx = dn(idx);
        const double x = kh[kh_pad(idx)];
        a0 = fma(x, b1, a0); a1 = fma(w0, b1, a1); a2 = fma(w1, b1, a2); a3 = fma(w2, b1, a3);
        idx = dn(idx);
        const double y = kh[kh_pad(idx)];
        a0 = fma(y, b2, a0); a1 = fma(x, b2, a1); a2 = fma(w0, b2, a2); a3 = fma(w1, b2, a3);
        idx = dn(idx);
        const double z = kh[kh_pad(idx)];
        a0 = fma(z, b3, a0); a1 = fma(y, b3, a1); a2 = fma(x, b3, a2); a3 = fma(w0, b3, a3);
        idx = dn(idx);
        w3 = x; w2 = y; w1 = z; w0 = kh[kh_pad(idx)];
      }
      for (; m < mhi; ++m) {
        const double b0 = rho[m] - mean_rho;
        a0 = fma(w0, b0, a0); a1 = fma(w1, b0, a1); a2 = fma(w2, b0, a2); a3 = fma(w3, b0, a3);
        idx = dn(idx);
        w3 = w2; w2 = w1; w1 = w0; w0 = kh[kh_pad(idx)];
      }
      double* pr = prow + (size_t)q * nx + n0;
      pr[0] = a0;
      if (n0 + 1 < nx) pr[1] = a1;
      if (n0 + 2 < nx) pr[2] = a2;
      if (n0 + 3 < nx) pr[3] = a3;
    }
  }
  __syncthreads();
  for (int nd = tid; nd < nx; nd += blockDim.x) {
    double sum = prow[nd];
    for (int q = 1; q < mp; ++q) sum += prow[(size_t)q * nx + nd];
    phi[nd] = h * sum;          // rho is dead: phi overwrites it
  }
  __syncthreads();
  TSTAMP(6, j == 0);
  }  // !energy_only
  // phi -= mean(phi) (every warp's own mean, no barrier) while forming the
  // energy terms: L (phi - mean) = L phi up to the stencil's rounding
  const double mean_phi = a.energy_only ? 0.0 : warp_mean(phi);
  for (int nd = tid; nd < nx; nd += blockDim.x) {
    const double ph = phi[nd] - mean_phi;
    if (energy_out) {
      double lp = stn[0] * phi[nd];
      for (int k = 1; k <= a.degree; ++k) {
        int up = nd + k; if (up >= nx) up -= nx;
        int dn = nd - k; if (dn < 0) dn += nx;
        lp = fma(stn[k], phi[up] + phi[dn], lp);
      }
      part = fma(ph, lp * inv_h, part);
    }
    if (!a.energy_only) {
      if (a.phi_out) a.phi_out[(size_t)j * nx + nd] = ph;
      if (phi_hist) phi_hist[(size_t)j * nx + nd] = ph;
    }
  }
#ifdef PICROM_EXP_NOCIRC
  if (false) {
#else
  if (energy_out) {
#endif
    TSTAMP(7, j == 0);
    double e = block_sum(part, red);
    if (tid == 0) energy_out[j] = ip[I_HALFINVMP] * e;
  }
  TSTAMP(8, j == 0);
  if (a.counter) {
    // last CTA to finish advances the step counter (all CTAs read it above)
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      unsigned int t = atomicAdd(a.done, 1u);
      if (t == ntickets - 1) {
        *a.done = 0u;
        __threadfence();
        *a.counter = crow + 1;
        if (a.t_hist) {
          unsigned long long now;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
          a.t_hist[row] = now;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(512) solve_kernel(SolveArgs a) {
  extern __shared__ double sm[];
  if (a.skip && *a.skip) return;
  solve_body(a, blockIdx.x, sm, gridDim.x, a.scratch);
}

// particles per lane per block: 6 where K <= 2 lanes share a histogram (C2:
// 100 vs 97 G pushes/s), 4 for larger K (C5: 70.5 vs 65 with 6); -DPICROM_STEP_U
// overrides both (profiles/r01b)
#ifdef PICROM_STEP_U
template <int K> __host__ __device__ constexpr int step_u() { return PICROM_STEP_U; }
#else
template <int K> __host__ __device__ constexpr int step_u() { return K <= 2 ? 6 : 4; }
#endif

// Fixed-point deposit (FIX): value weights w in [0, 1] are rounded to
// W = round(w 2^50) (one DFMA: the low mantissa bits of w 2^50 + 1.5 2^52),
// split into three 17-bit limbs and added with native 32-bit shared-memory
// reductions (red.shared.add.u32) into ONE histogram per CTA [3][nx + D].
// Integer sums are exact and order independent, so the deposit is
// deterministic with no lane phases; a limb word holds 2^15 adds of 2^17 - 1,
// so a CTA folds its histogram into fp64 every kFixChunk particles (each
// particle adds at most once to a row).  Resolution 2^-50 per weight.
#ifndef PICROM_FIX_NT
#define PICROM_FIX_NT 256
#endif
#ifndef PICROM_FIX_MINB
#define PICROM_FIX_MINB 2
#endif
#ifndef PICROM_FIX_U
#define PICROM_FIX_U 4
#endif
constexpr int kFixNT = PICROM_FIX_NT;
constexpr int kFixMinB = PICROM_FIX_MINB;
constexpr int kFixU = PICROM_FIX_U;
constexpr int kFixChunk = 32767;

// per-instance thread-block clusters in the fused step (DSMEM reduction to
// the solving CTA) where the grid is instance-aligned
#ifdef PICROM_NO_CLUSTER
constexpr bool kUseCluster = false;
#else
constexpr bool kUseCluster = true;
#endif

// programmatic dependent launch between consecutive leapfrog steps: off --
// with two instance groups pipelined on separate streams it cost 2-3 us per
// step at C2 (65.4 vs 67.4 us), and it gains < 2 us with one group (r02)
#ifdef PICROM_PDL
constexpr bool kPdl = true;
#else
constexpr bool kPdl = false;
#endif

// L2 prefetch distance of the leapfrog pass, in SPAN blocks (0 = off)
#ifndef PICROM_STEP_PF
#define PICROM_STEP_PF 0
#endif
constexpr int PF = PICROM_STEP_PF;

// exact locate for the rare inputs of locate_fast (kept out of line so the
// common path stays a straight-line instruction stream)
struct CellFrac {
  double f;
  int c;
};
__device__ __noinline__ CellFrac locate_rare(double x, double h, double inv_h, int nx,
                                             double inv_nx) {
  CellFrac r;
  locate(x, h, inv_h, nx, inv_nx, r.c, r.f);
  return r;
}

// Fused particle pass.  NT threads; K consecutive lanes share one private
// smem histogram [row][H] (H = NT/K; bank = histogram id mod 16 for any row,
// so every access is conflict-free) and take turns (K phases); each lane
// handles U particles per iteration (u*32 + lane within its warp's 32*U
// block: coalesced), with the next iteration's loads issued first.
#ifndef PICROM_PHASE_MINB
#define PICROM_PHASE_MINB 1
#endif
template <int D, int K, int MODE, int NT, bool FIX>
__global__ void __launch_bounds__(NT, FIX ? kFixMinB : PICROM_PHASE_MINB)
step_kernel(StepArgs a, SolveArgs sa) {
  extern __shared__ double smem[];
  constexpr int H = FIX ? 1 : NT / K;
  constexpr int NW = D + 1;
  constexpr int U = FIX ? kFixU : step_u<K>();
  constexpr int SPAN = NT * U;
  const int nx = a.nx;
  const int nh = nx + D;                       // histogram rows incl. ghost nodes
  // phase path: [nh][H] fp64 histograms; FIX: [3][nh] u32 limbs + [nx] fp64
  // per-node sums of the folded chunks
  double* hist = smem;
  unsigned int* limbs = reinterpret_cast<unsigned int*>(smem);
  const int fix_dw = (3 * nh + 1) / 2;         // limb words in doubles
  double* acc = smem + fix_dw;
  double* coef = FIX ? acc + nx : hist + nh * H;   // [D][nx] field polynomials
  double* red = coef + (MODE == MODE_LEAPFROG ? nx * D : 0);
  TSTAMP(0, MODE == MODE_LEAPFROG && blockIdx.x == 0);
#ifdef PICROM_EXP_TIMELINE
  int tl_slot = -1;
  if (MODE == MODE_LEAPFROG && threadIdx.x == 0) {
    tl_slot = (int)(atomicAdd(&g_tl_ctr, 1u) & 16383u);
    g_tl[tl_slot][0] = a.counter ? (unsigned long long)*a.counter : 0ull;
    g_tl[tl_slot][1] = (unsigned long long)(cta_start(blockIdx.x, a.n * (long long)a.p, gridDim.x) / a.n);
  }
#endif
  TL(2);
  double* kh_pre = red + 64;                   // LEAPFROG: khat (padded) + stencil
  double* stn_pre = kh_pre + (nx + nx / 4 + 4);
  if (MODE == MODE_LEAPFROG && a.fuse_solve == 1) {
    for (int r = threadIdx.x; r < nx; r += NT) kh_pre[kh_pad(r)] = sa.khat[r];
    if (sa.stencil && threadIdx.x <= D) stn_pre[threadIdx.x] = sa.stencil[threadIdx.x];
  }
  if constexpr (MODE == MODE_LEAPFROG && kPdl) {
    // programmatic dependent launch: the next step's grid may be scheduled
    // now (its CTAs take SM slots as ours exit and park in griddepcontrol.wait),
    // and everything above (constants only) overlapped the previous step's
    // tail; x, v, phi and the step counter are read only after the previous
    // grid has completed and its writes are visible
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const unsigned int hist_base = FIX ? smem_u32(limbs) : smem_u32(hist + myh_of<K>(threadIdx.x));

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  // lanes l, l + 32/K, l + 2*32/K, ... share histogram (warp, l mod 32/K) and
  // take turns by lane range: the active lanes of a phase are one contiguous
  // 32/K-lane group with distinct banks (histogram id mod 16), so each
  // 8-byte access of a phase is a single conflict-free wavefront
  constexpr int KG = 32 / K;
  const int klane = lane / KG;     // histogram: myh_of<K>(tid)
  const int G = gridDim.x;
  const long long T = a.n * (long long)a.p;
  const long long start = cta_start(blockIdx.x, T, G);
  const long long end = cta_start(blockIdx.x + 1, T, G);
  const double inv_nx = 1.0 / (double)nx;
  const long long step_id = a.counter ? (*a.counter + 1) : a.step;
  const int woff = (tid >> 5) * 32 * U + lane;   // lane's offset inside a SPAN block

  int last_j = -1;
  long long pos = start;
  while (pos < end) {
    const int j = (int)(pos / a.n);
    const long long seg_lo = pos - (long long)j * a.n;
    const long long seg_hi = min(a.n, end - (long long)j * a.n);
    const int seg = blockIdx.x + j;
    const double* ip = a.inst + (size_t)j * PICROM_INST_STRIDE;
    const double h = ip[I_H], inv_h = ip[I_INVH];
    const int mask = fast_mask(nx, h);

    double kin = 0.0;
    double* X = a.x + (size_t)j * a.ld + seg_lo;
    double* V = a.v + (size_t)j * a.ld + seg_lo;
    const double* E0 = (MODE == MODE_DRIFT) ? a.e0 + (size_t)j * a.ld + seg_lo : nullptr;
    const double* Y = (MODE == MODE_DEPOSIT && a.y) ? a.y + (size_t)j * a.ld + seg_lo : nullptr;
    double* XO = (MODE == MODE_DRIFT) ? a.xo + (size_t)j * a.ld + seg_lo : nullptr;
    const int len = (int)(seg_hi - seg_lo);             // < 2^31 (checked on the host)

    // L2 bulk prefetch (TMA engine, no registers) of this warp's slice of the
    // SPAN block at local offset b0: lane 0 issues one cp.async.bulk.prefetch
    // per array; the range is trimmed to 16-byte boundaries inside the segment
    auto prefetch = [&](int b0) {
      if (PF > 0 && (MODE == MODE_LEAPFROG) && lane == 0 && b0 < len) {
        const int lo = b0 + (tid >> 5) * 32 * U;
        const int hi = min(len, lo + 32 * U);
        if (lo < hi) {
          const uintptr_t xa = (reinterpret_cast<uintptr_t>(X + lo)) & ~uintptr_t(15);
          const uintptr_t xe = (reinterpret_cast<uintptr_t>(X + hi)) & ~uintptr_t(15);
          const uintptr_t va = (reinterpret_cast<uintptr_t>(V + lo)) & ~uintptr_t(15);
          const uintptr_t ve = (reinterpret_cast<uintptr_t>(V + hi)) & ~uintptr_t(15);
          if (xe > xa) bulk_prefetch_l2(reinterpret_cast<const void*>(xa), (uint32_t)(xe - xa));
          if (ve > va) bulk_prefetch_l2(reinterpret_cast<const void*>(va), (uint32_t)(ve - va));
        }
      }
    };

    // loads of one SPAN block starting at local offset b0 into (lx, lv, le)
    auto load = [&](int b0, double* lx, double* lv, double* le) {
      if constexpr (PF > 0) prefetch(b0 + PF * SPAN);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = b0 + woff + u * 32;
        const bool in = i < len;
        lx[u] = in ? __ldcs(X + i) : 0.0;
        if constexpr (MODE == MODE_LEAPFROG || MODE == MODE_DRIFT) lv[u] = in ? __ldcs(V + i) : 0.0;
        if constexpr (MODE == MODE_DRIFT) le[u] = in ? __ldcs(E0 + i) : 0.0;
        if constexpr (MODE == MODE_DEPOSIT) lv[u] = (in && Y) ? __ldcs(Y + i) : 1.0;
      }
    };

    // the first block's loads go out before the histogram zeroing and the
    // field-polynomial build, so their DRAM latency overlaps that prologue
    double ax[U], av[U], ae[U], bx[U], bv[U], be[U];
    if constexpr (PF > 1) {
#pragma unroll
      for (int q = 1; q < PF; ++q) prefetch(q * SPAN);
    }
    if (len > 0) load(0, ax, av, ae);

#ifndef PICROM_EXP_NOHIST
    if constexpr (FIX) {
      for (int q = tid; q < 3 * nh; q += NT) limbs[q] = 0u;
      for (int q = tid; q < nx; q += NT) acc[q] = 0.0;
    } else {
      for (int q = tid; q < nh * H; q += NT) hist[q] = 0.0;
    }
#endif
    if (MODE == MODE_LEAPFROG && j != last_j) {
      const double* ph = a.phi + (size_t)j * nx;
      const double ecoef = ip[I_ECOEF], g = ip[I_INVH];
      for (int c = tid; c < nx; c += NT) {
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
    TL(3);

    // the particle work of one SPAN block already in registers
    auto process = [&](int b0, const double* cx, const double* cv, const double* ce) {
#ifdef PICROM_EXP_STREAM
      // timing experiment only: the bare x, v stream (no locate/gather/deposit)
      if constexpr (MODE == MODE_LEAPFROG) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = b0 + woff + u * 32;
          if (i < len) {
            __stcs(X + i, fma(a.dt, cv[u], cx[u]));
            __stcs(V + i, cv[u] * 0.999);
          }
        }
        return;
      }
#endif
      bool valid[U];
#pragma unroll
      for (int u = 0; u < U; ++u) valid[u] = b0 + woff + u * 32 < len;

      // pass 1: the particle update (straight-line common path)
      double xn[U];
      if constexpr (MODE == MODE_LEAPFROG) {
        int c0[U];
        double f0[U];
        bool r0[U], any0 = false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          locate_fast(cx[u], h, inv_h, nx, mask, inv_nx, c0[u], f0[u], r0[u]);
          r0[u] = r0[u] && valid[u];
          any0 |= r0[u];
        }
        if (__any_sync(0xffffffffu, any0)) {
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (r0[u]) {
              const CellFrac cf = locate_rare(cx[u], h, inv_h, nx, inv_nx);
              c0[u] = cf.c;
              f0[u] = cf.f;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          double C[D];
#pragma unroll
#ifdef PICROM_EXP_NOGATHER
          for (int k = 0; k < D; ++k) C[k] = f0[u] * (k + 1);      // timing experiment only
#else
          for (int k = 0; k < D; ++k) C[k] = coef[k * nx + c0[u]];
#endif
          const double E = horner<D>(C, f0[u]);
          const double vn = cv[u] + a.kfull * E;
          kin = valid[u] ? fma(vn, vn, kin) : kin;
          const double vh = fma(a.kick, E, cv[u]);      // leapfrog kick + drift
          xn[u] = fma(a.dt, vh, cx[u]);
          const int i = b0 + woff + u * 32;
          if (valid[u]) {
            __stcs(X + i, xn[u]);
            __stcs(V + i, vh);
          }
        }
      } else if constexpr (MODE == MODE_DRIFT) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double vh = __dadd_rn(cv[u], __dmul_rn(a.kick, ce[u]));
          xn[u] = __dadd_rn(cx[u], __dmul_rn(a.dt, vh));
          if (valid[u]) __stcs(XO + b0 + woff + u * 32, xn[u]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) xn[u] = cx[u];
      }

      // pass 2: locate the new positions, rare inputs fixed up uniformly
      int cl[U];
      double fr[U];
      bool ok[U], r1[U], any1 = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ok[u] = valid[u] && isfinite(xn[u]);
        locate_fast(xn[u], h, inv_h, nx, mask, inv_nx, cl[u], fr[u], r1[u]);
        r1[u] = r1[u] && valid[u];
        any1 |= r1[u];
      }
      if (__any_sync(0xffffffffu, any1)) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!r1[u]) continue;
          if (ok[u]) {
            const CellFrac cf = locate_rare(xn[u], h, inv_h, nx, inv_nx);
            cl[u] = cf.c;
            fr[u] = cf.f;
          } else {
            record_bad(a.status, step_id, seg_lo + b0 + woff + u * 32, j, a.p);
            cl[u] = 0;
            fr[u] = 0.0;
          }
        }
      }

      // pass 3: deposit.  Weights of all U particles first, then K phases; in
      // phase q the lanes of group q read-modify-write their U particles'
      // rows with predicated shared loads/stores (no branches, so the block
      // stays one scheduling region), one warp barrier between phases.
      double w[U][NW];
      unsigned int hrow[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (MODE == MODE_DEPOSIT) {
          if (a.wkind == 1) Spline<D>::dweights(fr[u], ip[I_INVH], w[u]);
          else Spline<D>::weights(fr[u], w[u]);
          if (Y) {
#pragma unroll
            for (int m = 0; m < NW; ++m) w[u][m] *= cv[u];
          }
        } else {
          Spline<D>::weights(fr[u], w[u]);
        }
        hrow[u] = hist_base + (unsigned int)(cl[u] * H) * 8u;
      }
      if constexpr (FIX) {
        // exact integer deposit: 3 limbs per weight, one red.shared.add.u32
        // each; rows are limb-major [3][nh]
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int m = 0; m < NW; ++m) {
            const double t = fma(w[u][m], 0x1p50, 0x1.8p52);
            const unsigned int lo = __double2loint(t), hi = __double2hiint(t);
            const unsigned int l0 = lo & 0x1ffffu;
            const unsigned int l1 = __funnelshift_r(lo, hi, 17) & 0x1ffffu;
            const unsigned int l2 = (hi >> 2) & 0x1ffffu;
            const unsigned int addr = hist_base + (unsigned int)(cl[u] + m) * 4u;
            red_shared_u32_if(addr, l0, ok[u]);
            red_shared_u32_if(addr + (unsigned int)nh * 4u, l1, ok[u]);
            red_shared_u32_if(addr + (unsigned int)nh * 8u, l2, ok[u]);
          }
        }
      } else if constexpr (K == 32) {
        // one histogram per warp (large meshes, e.g. C5's Nx = 512): four
        // phases by cell mod 4 -- two cells of one phase are either equal or
        // >= 4 apart, so their D+1 <= 4 rows are disjoint -- and, inside a
        // phase, lanes with the same cell take turns by their rank among the
        // lanes of that cell (__match_any_sync; fixed order, deterministic)
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool in = ok[u] && (cl[u] & 3) == q;
            const unsigned int peers = __match_any_sync(0xffffffffu, in ? cl[u] : -1 - lane);
            const int rank = __popc(peers & ((1u << lane) - 1u));
            const int rounds = __reduce_max_sync(0xffffffffu, in ? rank + 1 : 0);
            for (int rr = 0; rr < rounds; ++rr) {
              const bool act = in && rank == rr;
              double cur[NW];
#pragma unroll
              for (int m = 0; m < NW; ++m) cur[m] = lds_f64_if(hrow[u] + m * H * 8u, act);
#pragma unroll
              for (int m = 0; m < NW; ++m) sts_f64_if(hrow[u] + m * H * 8u, cur[m] + w[u][m], act);
              __syncwarp();
            }
          }
        }
      } else {
#pragma unroll
      for (int q = 0; q < K; ++q) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
#ifdef PICROM_EXP_NODEP
          const bool act = ok[u] && klane == q && fr[u] < -1.0;   // timing experiment only
#else
          const bool act = ok[u] && klane == q;
#endif
          double cur[NW];
#pragma unroll
          for (int m = 0; m < NW; ++m) cur[m] = lds_f64_if(hrow[u] + m * H * 8u, act);
#pragma unroll
          for (int m = 0; m < NW; ++m) sts_f64_if(hrow[u] + m * H * 8u, cur[m] + w[u][m], act);
        }
        if constexpr (K > 1) __syncwarp();
      }
      }
    };

    // ping-pong register buffers: the loads of one block are in flight while
    // the other block is processed; no register copies on the loop edge
    // FIX: fold the limbs into acc (and re-zero them) every CH particles, so no
    // limb word can overflow; each thread owns the rows of its nodes
    constexpr int CH = FIX ? (kFixChunk / (2 * SPAN)) * (2 * SPAN) : (1 << 30);
    static_assert(!FIX || CH >= 2 * SPAN, "kFixChunk too small for the block span");
    auto fold_limbs = [&](int nd) {
      double v = 0.0;
      for (int r = (nd - Spline<D>::OFF) % nx; r < nh; r += nx) {
        const double a0 = (double)limbs[r], a1 = (double)limbs[nh + r], a2 = (double)limbs[2 * nh + r];
        v += fma(a2, 0x1p-16, fma(a1, 0x1p-33, a0 * 0x1p-50));
      }
      return v;
    };
    for (int b0 = 0; b0 < len; b0 += 2 * SPAN) {
      if (b0 + SPAN < len) load(b0 + SPAN, bx, bv, be);
      process(b0, ax, av, ae);
      if (b0 + SPAN >= len) break;
      if (b0 + 2 * SPAN < len) load(b0 + 2 * SPAN, ax, av, ae);
      process(b0 + SPAN, bx, bv, be);
      if constexpr (FIX) {
        if ((b0 + 2 * SPAN) % CH == 0 && b0 + 2 * SPAN < len) {
          __syncthreads();
          for (int nd = tid; nd < nx; nd += NT) {
            acc[nd] += fold_limbs(nd);
            for (int r = (nd - Spline<D>::OFF) % nx; r < nh; r += nx)
              limbs[r] = limbs[nh + r] = limbs[2 * nh + r] = 0u;
          }
          __syncthreads();
        }
      }
    }
    TSTAMP(1, MODE == MODE_LEAPFROG && j == 0 && seg_hi == a.n);
    TL(4);
    __syncthreads();

    // fold ghost rows, reduce the H histograms in a fixed order -> segment row.
    // Thread per node; node nd reads the histograms rotated by nd (H is a
    // power of two), so the 32 lanes of a load hit 32 consecutive histograms
    // -- conflict-free (unrotated, all lanes would read one bank, rows apart).
#ifdef PICROM_EXP_NOHIST
    if (false)
#endif
    // cluster path: the CTA's row stays in its own smem (the coefficient
    // region, free after the particle loop) for rank 0 to read over DSMEM
    double* seg_out = (MODE == MODE_LEAPFROG && a.cluster_m > 0) ? coef : a.seg_hist + (size_t)seg * nx;
    if constexpr (FIX) {
      for (int nd = tid; nd < nx; nd += NT) seg_out[nd] = acc[nd] + fold_limbs(nd);
    } else
    for (int nd = tid; nd < nx; nd += NT) {
      double s8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      // histogram row r holds node (r + OFF) mod nx: rows r0, r0 + nx, ... < nh
      for (int r = (nd - Spline<D>::OFF) % nx; r < nh; r += nx) {
        const double* rowp = hist + r * H;
#pragma unroll
        for (int hh = 0; hh < H; hh += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (hh + u < H) s8[u] += rowp[(hh + u + nd) & (H - 1)];
        }
      }
      seg_out[nd] = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
    }
    TSTAMP(2, MODE == MODE_LEAPFROG && j == 0 && seg_hi == a.n);
    TL(5);
    if constexpr (MODE == MODE_LEAPFROG) {
      double ks = block_sum(kin, red);
      if (a.cluster_m > 0 && a.fuse_solve == 1) {
        // instance j = this cluster: rank 0 assembles rho from the m rows in
        // the cluster's shared memory (fixed rank order -> deterministic), the
        // others wait until it has read them, then rank 0 solves -- no global
        // round trip, no ticket atomics
        namespace cgx = cooperative_groups;
        cgx::cluster_group cl = cgx::this_cluster();
        if (tid == 0) red[48] = ks;
        cl.sync();
        const bool root = cl.block_rank() == 0;
        __shared__ double s_kin;
        if (root) {
          const double* ipj = a.inst + (size_t)j * PICROM_INST_STRIDE;
          const double qw = ipj[I_QW], bgh = ipj[I_BGH];
          const int m = a.cluster_m;
          for (int nd = tid; nd < nx; nd += NT) {
            double sacc = 0.0;
            for (int r = 0; r < m; ++r) sacc += cl.map_shared_rank(coef, r)[nd];
            hist[nd] = fma(qw, sacc, bgh);
          }
          if (tid == 0) {
            double kk = 0.0;
            for (int r = 0; r < m; ++r) kk += cl.map_shared_rank(red, r)[48];
            s_kin = kk;
          }
        }
        cl.sync();
        TL(6);
        if (root) {
          __syncthreads();
          TSTAMP(3, j == 0);
          solve_body(sa, j, hist, (unsigned int)a.p, (size_t)(red + 64 - smem), kh_pre, stn_pre,
                     a.counter ? step_id - 1 : -1, true, s_kin);
          TL(7);
        }
      } else {
      if (tid == 0) a.seg_kin[seg] = ks;
      if (a.fuse_solve) {
        // the last CTA to finish instance j's particles solves instance j
        // (threadFenceReduction pattern); the histograms are free scratch now
        __shared__ int s_last;
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          const int b_lo = cta_of((long long)j * a.n, T, G);
          const int b_hi = cta_of((long long)(j + 1) * a.n - 1, T, G);
          const unsigned int need = (unsigned int)(b_hi - b_lo);
          const unsigned int prev = atomicAdd(&a.inst_done[j], 1u);
          s_last = prev == need;
          if (s_last) a.inst_done[j] = 0u;
        }
        __syncthreads();
        TL(6);
#ifdef PICROM_EXP_NOSOLVE
        if (false) {     // timing experiment only
#else
        if (s_last && a.fuse_solve == 1) {
#endif
#ifndef PICROM_SOLVE_NOFENCE
          __threadfence();
#endif
          TSTAMP(3, j == 0);
          // scratch = the histogram, coefficient and reduction smem (free now)
          solve_body(sa, j, hist, (unsigned int)a.p, (size_t)(red + 64 - smem),
                     kh_pre, stn_pre, a.counter ? step_id - 1 : -1);
          TL(7);
        }
      }
      }  // ticket path
    }
    __syncthreads();
    last_j = j;
    pos = (long long)(j + 1) * a.n;
  }
}

static int launch_solve(const SolveArgs& a_in, cudaStream_t s) {
  SolveArgs a = a_in;
  int threads = std::min(512, std::max(64, ((a.nx + 31) / 32) * 32));
  const int mp = solve_mp(a.nx, threads, (size_t)1 << 40);
  a.scratch = solve_scratch(a.nx, mp);
  size_t sm = a.scratch * sizeof(double);
  static bool attr = false;
  if (!attr) {
    allow_max_dynamic_smem(solve_kernel);
    attr = true;
  }
  solve_kernel<<<a.p, threads, sm, s>>>(a);
  return check_launch("solve_kernel");
}

// dense-segment assembly + solve (used by the reduced-basis deposit, rom.cu)
int picrom_solve_dense(const double* seg, int G, int p, int nx, int degree, const int* cols,
                       const double* inst, const double* khat, const double* stencil,
                       double* phi, double* rho, double* energy, cudaStream_t s,
                       const long long* skip) {
  SolveArgs sa{};
  sa.skip = skip;
  sa.seg_hist = seg; sa.seg_dense = G; sa.cols = cols; sa.inst = inst; sa.khat = khat;
  sa.stencil = stencil; sa.n = 1; sa.p = p; sa.nx = nx; sa.degree = degree; sa.G = G;
  sa.solve = phi != nullptr || energy != nullptr; sa.phi_out = phi; sa.rho_out = rho;
  sa.energy_out = energy;
  return launch_solve(sa, s);
}

// --------------------------------------------------------- launch helpers

// last cluster decision of the fused step: {m, clusters needed, max co-resident}
static int g_cluster_info[3] = {0, 0, 0};
extern "C" int picrom_debug_cluster_info(int* out) {
  for (int i = 0; i < 3; ++i) out[i] = g_cluster_info[i];
  return 0;
}

template <int D, int K, int MODE, bool FIX>
static int launch_step_t(const StepArgs& a_in, const SolveArgs& sa, const Plan& pl, cudaStream_t s) {
  constexpr int NT = FIX ? kFixNT : 128;
  auto kfn = step_kernel<D, K, MODE, NT, FIX>;
  static bool attr = false;
  if (!attr) {
    allow_max_dynamic_smem(kfn);
    attr = true;
  }
  StepArgs a = a_in;
  const size_t smem = FIX ? pl.fsmem : pl.smem;
  if (MODE == MODE_LEAPFROG && a.cluster_m > 0) {
    // one cluster per instance (instance-aligned grid); fall back to the
    // ticket path unless every cluster of the launch can be co-resident
    const int m = a.cluster_m;
    static int ok_m = -1, ok_clusters = -1;
    static size_t ok_smem = 0;
    const int clusters = pl.G / m;
    if (!(ok_m == m && ok_smem == smem)) {
      cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t qc{};
      qc.gridDim = dim3(pl.G);
      qc.blockDim = dim3(NT);
      qc.dynamicSmemBytes = smem;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = m;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      qc.attrs = qa;
      qc.numAttrs = 1;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, kfn, &qc) != cudaSuccess) {
        (void)cudaGetLastError();
        nc = 0;
      }
      ok_m = m;
      ok_smem = smem;
      ok_clusters = nc;
    }
    g_cluster_info[0] = m;
    g_cluster_info[1] = clusters;
    g_cluster_info[2] = ok_clusters;
    if (ok_clusters >= clusters) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(pl.G);
      cfg.blockDim = dim3(NT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = m;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (cudaLaunchKernelEx(&cfg, kfn, a, sa) != cudaSuccess) return check_launch("step_kernel (cluster)");
      return check_launch("step_kernel (cluster)");
    }
    a.cluster_m = 0;
  }
  if (MODE == MODE_LEAPFROG && kPdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(pl.G);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = FIX ? pl.fsmem : pl.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr_pdl[1];
    attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr_pdl;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kfn, a, sa) != cudaSuccess) return check_launch("step_kernel (PDL)");
    return check_launch("step_kernel");
  }
  kfn<<<pl.G, NT, smem, s>>>(a, sa);
  return check_launch("step_kernel");
}

template <int D, int MODE>
static int launch_step_k(const StepArgs& a, const SolveArgs& sa, const Plan& pl, cudaStream_t s) {
#ifdef PICROM_NO_FIX
  const bool fix = false;      // dev variant: lane-phase fp64 histograms everywhere
#else
  // value weights in [0, 1] take the fixed-point deposit where lane phases
  // would be K > 2 (Nx > 256 at degree 3): measured 126 vs 71 G pushes/s at
  // C5's Nx = 512; at K <= 2 the conflict-free fp64 phases are faster (C2's
  // Nx = 128: 106 vs 97, profiles/r02)
  const bool fix = pl.K > 2 && !(MODE == MODE_DEPOSIT && (a.y != nullptr || a.wkind != 0));
#endif
  if (fix) return launch_step_t<D, 1, MODE, true>(a, sa, pl, s);
  switch (pl.K) {
    case 1: return launch_step_t<D, 1, MODE, false>(a, sa, pl, s);
    case 2: return launch_step_t<D, 2, MODE, false>(a, sa, pl, s);
    case 4: return launch_step_t<D, 4, MODE, false>(a, sa, pl, s);
    case 8: return launch_step_t<D, 8, MODE, false>(a, sa, pl, s);
    case 16: return launch_step_t<D, 16, MODE, false>(a, sa, pl, s);
    default: return launch_step_t<D, 32, MODE, false>(a, sa, pl, s);
  }
}

template <int MODE>
static int launch_step(const StepArgs& a, int degree, const Plan& pl, cudaStream_t s,
                       const SolveArgs* sa = nullptr) {
  SolveArgs none{};
  const SolveArgs& sref = sa ? *sa : none;
  switch (degree) {
    case 1: return launch_step_k<1, MODE>(a, sref, pl, s);
    case 2: return launch_step_k<2, MODE>(a, sref, pl, s);
    case 3: return launch_step_k<3, MODE>(a, sref, pl, s);
  }
  return set_err(PICROM_ERR_CONFIG, "degree must be 1, 2 or 3");
}

template <int D>
static int fix_occ_of(size_t smem) {
  int occ = 0;
  auto kfn = step_kernel<D, 1, MODE_LEAPFROG, kFixNT, true>;
  allow_max_dynamic_smem(kfn);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kFixNT, smem) != cudaSuccess) occ = 1;
  return occ;
}

template <int D, int K>
static int occ_of(size_t smem) {
  int occ = 0;
  auto kfn = step_kernel<D, K, MODE_LEAPFROG, 128, false>;
  allow_max_dynamic_smem(kfn);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, 128, smem) != cudaSuccess) occ = 1;
  return occ;
}

template <int D>
static int occ_k(int K, size_t smem) {
  switch (K) {
    case 1: return occ_of<D, 1>(smem);
    case 2: return occ_of<D, 2>(smem);
    case 4: return occ_of<D, 4>(smem);
    case 8: return occ_of<D, 8>(smem);
    case 16: return occ_of<D, 16>(smem);
    default: return occ_of<D, 32>(smem);
  }
}

static int step_occupancy(int degree, int K, size_t smem) {
  static int cache[4][6][2] = {};   // degree x log2 K x (valid, occupancy)
  static size_t cache_smem[4][6] = {};
  int lk = 0;
  while ((1 << lk) < K) ++lk;
  if (cache[degree][lk][0] && cache_smem[degree][lk] == smem) return cache[degree][lk][1];
  int occ = degree == 1 ? occ_k<1>(K, smem) : degree == 2 ? occ_k<2>(K, smem) : occ_k<3>(K, smem);
  cache[degree][lk][0] = 1;
  cache[degree][lk][1] = occ;
  cache_smem[degree][lk] = smem;
  return occ;
}

static int fix_occupancy(int degree, size_t smem) {
  static int cache_occ[4] = {};
  static size_t cache_smem[4] = {};
  if (cache_occ[degree] && cache_smem[degree] == smem) return cache_occ[degree];
  const int occ = degree == 1 ? fix_occ_of<1>(smem) : degree == 2 ? fix_occ_of<2>(smem) : fix_occ_of<3>(smem);
  cache_occ[degree] = occ;
  cache_smem[degree] = smem;
  return occ;
}

static int check_cfg(long long n, int p, int nx, int degree) {
  if (n < 1 || p < 1) return set_err(PICROM_ERR_CONFIG, "need n >= 1 and p >= 1");
  if (n > 2000000000LL) return set_err(PICROM_ERR_CONFIG, "n > 2e9 particles per instance");
  if (nx < 2) return set_err(PICROM_ERR_CONFIG, "need nx >= 2");
  if (degree < 1 || degree > 3) return set_err(PICROM_ERR_CONFIG, "degree must be 1, 2 or 3");
  if (degree > 1 && nx < 2 * degree + 1) return set_err(PICROM_ERR_CONFIG, "need nx >= 2*degree+1");
  if (nx > 8192) return set_err(PICROM_ERR_CONFIG, "nx > 8192 not supported");
  return PICROM_OK;
}

// workspace: seg rows x nx | seg rows (kinetic) | p instance tickets
// (tickets zeroed once, left zeroed by every call)
static void ws_split(void* ws, const Plan& pl, int p, int nx, double** hist, double** kin,
                     unsigned int** tickets = nullptr) {
  double* base = reinterpret_cast<double*>(ws);
  const size_t rows = seg_rows(pl, p);
  *hist = base;
  *kin = base + rows * nx;
  unsigned int* t = reinterpret_cast<unsigned int*>(*kin + rows);
  if (tickets) *tickets = t;
}

// zero the ticket words of a workspace (one-shot entry points may be handed a
// workspace last used with another shape)
static void zero_tickets(const StepArgs& a, int p, cudaStream_t s) {
  if (a.inst_done) cudaMemsetAsync(a.inst_done, 0, (size_t)(p + 1) * sizeof(unsigned int), s);
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
  ws_split(ws, pl, p, nx, &a.seg_hist, &a.seg_kin, &a.inst_done);
  zero_tickets(a, p, (cudaStream_t)stream);
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
  ws_split(ws, pl, p, nx, &a.seg_hist, &a.seg_kin, &a.inst_done);
  zero_tickets(a, p, (cudaStream_t)stream);
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
  ws_split(ws, pl, p, nx, &a.seg_hist, &a.seg_kin, &a.inst_done);
  return launch_step<MODE_LEAPFROG>(a, degree, pl, (cudaStream_t)stream);
}

extern "C" int picrom_pic_solve(long long n, int p, int nx, int degree, const double* inst,
                                const double* khat, const double* stencil, double* phi,
                                long long step, long long* counter, long long hist_rows,
                                double* rho_hist, double* phi_hist, double* ee_hist,
                                double* kin_hist, void* ws, void* stream) {
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
    sa.hist_mod = hist_rows;
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
                               long long hist_rows, int hist_p, double* rho_hist,
                               double* phi_hist, double* ee_hist, double* kin_hist,
                               unsigned long long* t_hist, void* ws,
                               unsigned long long* status, void* stream) {
  int rc = check_cfg(n, p, nx, degree);
  if (rc) return rc;
  Plan pl = make_plan(n, p, nx, degree, true);
  StepArgs a{};
  a.x = x; a.v = v; a.phi = phi; a.inst = inst; a.n = n; a.ld = ld; a.p = p; a.nx = nx;
  a.dt = dt; a.kick = kick; a.kfull = kfull; a.step = step + 1; a.status = status;
  a.counter = counter;
  a.fuse_solve = 1;
  // instance-aligned grid (G = m p, 2 <= m <= 16): one thread-block cluster per
  // instance, the per-instance reduction over DSMEM
  if (kUseCluster && pl.G % p == 0 && pl.G / p >= 2 && pl.G / p <= 16) a.cluster_m = pl.G / p;
  ws_split(ws, pl, p, nx, &a.seg_hist, &a.seg_kin, &a.inst_done);
  SolveArgs sa{};
  sa.seg_hist = a.seg_hist; sa.seg_kin = a.seg_kin; sa.inst = inst; sa.khat = khat;
  sa.stencil = stencil; sa.n = n; sa.p = p; sa.nx = nx; sa.degree = degree; sa.G = pl.G;
  sa.solve = true; sa.phi_out = phi;
  // history rows hold hist_p >= p instances (an instance group writes its
  // slice of a shared history at the caller's pointer offset)
  if (hist_p < p) hist_p = p;
  const size_t gp = (size_t)hist_p * nx;
  sa.hist_stride_rho = gp;
  sa.hist_stride_e = (size_t)hist_p;
  if (counter) {
    sa.counter = counter;
    sa.done = reinterpret_cast<unsigned int*>(counter + 1);
    sa.hist_mod = hist_rows;
    sa.rho_out = rho_hist; sa.phi_hist = phi_hist; sa.energy_out = ee_hist; sa.kin_out = kin_hist;
    sa.t_hist = t_hist;
  } else {
    sa.rho_out = rho_hist ? rho_hist + (size_t)step * gp : nullptr;
    sa.phi_hist = phi_hist ? phi_hist + (size_t)step * gp : nullptr;
    sa.energy_out = ee_hist ? ee_hist + (size_t)step * hist_p : nullptr;
    sa.kin_out = kin_hist ? kin_hist + (size_t)step * hist_p : nullptr;
  }
  return launch_step<MODE_LEAPFROG>(a, degree, pl, (cudaStream_t)stream, &sa);
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
  ws_split(ws, pl, p, nx, &a.seg_hist, &a.seg_kin, &a.inst_done);
  zero_tickets(a, p, (cudaStream_t)stream);
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
  const double h = ip[I_H], g = ip[I_INVH], inv_h = ip[I_INVH];
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
    locate(x, h, inv_h, nx, inv_nx, c, f);
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
  // (d+1) nx doubles of cell polynomials: beyond 48 KB (nx > 1536 at d = 3)
  // the kernel needs the opt-in dynamic shared-memory limit
  static bool attr[4] = {false, false, false, false};
  switch (degree) {
    case 1:
      if (!attr[1]) { allow_max_dynamic_smem(gather_kernel<1, KICK>); attr[1] = true; }
      gather_kernel<1, KICK><<<grid, kThreads, sm, s>>>(a); break;
    case 2:
      if (!attr[2]) { allow_max_dynamic_smem(gather_kernel<2, KICK>); attr[2] = true; }
      gather_kernel<2, KICK><<<grid, kThreads, sm, s>>>(a); break;
    case 3:
      if (!attr[3]) { allow_max_dynamic_smem(gather_kernel<3, KICK>); attr[3] = true; }
      gather_kernel<3, KICK><<<grid, kThreads, sm, s>>>(a); break;
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
    // the step kernels' branch-free locate (rare inputs: exact locate), so
    // picrom_locate's bit-exactness tests cover the production path
    int c;
    double f;
    bool rare;
    locate_fast(xv, ip[I_H], ip[I_INVH], nx, fast_mask(nx, ip[I_H]), inv_nx, c, f, rare);
    if (rare) locate(xv, ip[I_H], ip[I_INVH], nx, inv_nx, c, f);
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

// ||a - b||^2 and ||a||^2 over `count` contiguous doubles (b nullable: only
// ||a||^2), per-block partials then one fixed-order final sum (deterministic)
__global__ void diff_sumsq_kernel(const double* a, const double* b, long long count, double* part) {
  __shared__ double red[32];
  double d = 0.0, q = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const double av = a[i];
    const double df = b ? av - b[i] : 0.0;
    d = fma(df, df, d);
    q = fma(av, av, q);
  }
  d = block_sum(d, red);
  q = block_sum(q, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = d;
    part[2 * blockIdx.x + 1] = q;
  }
}

__global__ void diff_sumsq_final(const double* part, int G, double* out) {
  __shared__ double red[32];
  double d = 0.0, q = 0.0;
  for (int k = threadIdx.x; k < G; k += blockDim.x) {
    d += part[2 * k];
    q += part[2 * k + 1];
  }
  d = block_sum(d, red);
  q = block_sum(q, red);
  if (threadIdx.x == 0) {
    out[0] = d;
    out[1] = q;
  }
}

extern "C" int picrom_diff_sumsq(const double* a, const double* b, long long count, double* out,
                                 void* ws, void* stream) {
  if (count < 1) return set_err(PICROM_ERR_CONFIG, "diff_sumsq of an empty array");
  cudaStream_t s = (cudaStream_t)stream;
  const int G = (int)std::min<long long>(4LL * num_sms(), (count + 255) / 256);
  double* part = (double*)ws;
  diff_sumsq_kernel<<<G, 256, 0, s>>>(a, b, count, part);
  int rc = check_launch("diff_sumsq");
  if (rc) return rc;
  diff_sumsq_final<<<1, 256, 0, s>>>(part, G, out);
  return check_launch("diff_sumsq_final");
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
  const long long r0 = (long long)blockIdx.x * 32;
  const long long ctiles = (cols + 31) / 32;
  for (long long cy = blockIdx.y; cy < ctiles; cy += gridDim.y) {
    const long long c0 = cy * 32;
    __syncthreads();
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
}

template <typename T>
static int do_transpose(const T* in, long long rows, long long cols, T* out, void* stream) {
  if (rows < 1 || cols < 1) return PICROM_OK;
  long long gx = (rows + 31) / 32, gy = std::min<long long>((cols + 31) / 32, 65535);
  if (gx > 2147483647LL) return set_err(PICROM_ERR_CONFIG, "transpose too large");
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
