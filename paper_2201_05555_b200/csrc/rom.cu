// Reduced-basis kernels for sm_100a.
//
//   rom_deposit  : X_r = U_X Z (fused, never stored), locate, B-spline deposit
//                  into per-thread private histograms -> dense segment rows
//                  [G][p'][Nx]; assembled + solved by the FOM solve kernel.
//                  (driver.exact_gradients, driver.py:63-73)
//   rom_gather   : X_r = U_X Z, field gather at X_r, projection U_X^T E
//                  (per-CTA partials [G][p'][n]), optional DEIM harvest
//                  lam = Lambda phi (driver.py:76) and optional E output.
//                  (driver.py:74-76, make_full_stage driver.py:79-89)
//   paired_gram  : W^T W of a row-concatenation of tall column blocks
//                  (every n x n product in reduction.py:143-182 is a block of it)
//   combine      : Y_block = sum_t B_t M_t for tall blocks B_t and small M_t
//                  (the U + A C updates of reduction.py:143-182)
//   rows_gather  : U rows at DEIM indices (hyper.py:312)
//
// All reductions are fixed-order (deterministic run to run).

#include <cuda_runtime.h>
#include <stdio.h>

#include <algorithm>
#include <type_traits>
#include <vector>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"

// Compile-time kernel-path switches (dev variants via tools/build_variant.py
// -DPICROM_...); the shipped library reads no environment variables.
#ifdef PICROM_ROM_NO_MMA
constexpr bool kNoRomMma = true;
#else
constexpr bool kNoRomMma = false;
#endif
#ifdef PICROM_GRAM_NO_MMA
constexpr bool kNoGramMma = true;
#else
constexpr bool kNoGramMma = false;
#endif
#ifdef PICROM_GRAM_NO_TMA
constexpr bool kNoGramTma = true;
#else
constexpr bool kNoGramTma = false;
#endif
#ifdef PICROM_COMBINE_NO_WIDE
constexpr bool kNoCombineWide = true;
#else
constexpr bool kNoCombineWide = false;
#endif
#ifdef PICROM_COMBINE_NO_MMA
constexpr bool kNoCombineMma = true;
#else
constexpr bool kNoCombineMma = false;
#endif
#ifdef PICROM_COMBINE_NO_TMA
constexpr bool kNoCombineTma = true;
#else
constexpr bool kNoCombineTma = false;
#endif

using namespace picrom;

extern int picrom_set_error(int code, const char* msg);
extern int picrom_check_launch(const char* what);
extern int picrom_num_sms();
extern int picrom_solve_dense(const double* seg, int G, int p, int nx, int degree, const int* cols,
                              const double* inst, const double* khat, const double* stencil,
                              double* phi, double* rho, double* energy, cudaStream_t s,
                              const long long* skip);

namespace {

constexpr int NMAX = 32;        // max basis dimension handled in registers
constexpr int PT = 128;         // instance columns per CTA tile

struct RomArgs {
  const double* ux;     // U_X rows (N x n, row-major, ld = n)
  const double* z;      // Z (n x p'), row-major, ld = ldz
  const double* inst;   // per-instance rows
  const int* cols;      // instance id of each z column (nullable -> identity)
  const double* phi;    // (p', nx) potentials (gather)
  double* seg;          // deposit: [G][p'][nx]; gather: [G][p'][n]
  double* lam;          // gather: optional (N, ldo) row-major value gather at X_r
  double* eout;         // gather: optional (N, ldo) row-major coef * d/dx gather at X_r
  long long N, ldo;
  int n, p, ldz, nx;
  int coef_kind;        // gather: 0 -> gcoef (exact_gradients), 1 -> raw derivative
  unsigned long long* status;
  const double* uv;     // gather (DMMA path): optional U_V rows (N x n) -> U_V^T E
  double* seg2;         // gather: [G][p'][n] partials of U_V^T E
  const long long* skip;  // nullable device flag: nonzero -> the launch does nothing
                          // (iterations after a device-side fixed-point convergence)
};

__device__ __forceinline__ long long row_start(int b, long long N, int G) {
  return ((long long)b * N) / G;
}

template <typename F>
static void rom_allow_smem(F kfn) {
  cudaFuncAttributes at{};
  cudaFuncGetAttributes(&at, kfn);
  if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           227 * 1024 - (int)at.sharedSizeBytes) != cudaSuccess)
    (void)cudaGetLastError();
}

// ---- U_X row tiles: double-buffered cp.async (16 B chunks) into smem ----
constexpr int TR = 64;          // rows per tile

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(NPEND) : "memory");
}

// stage rows [r0, r0 + rows) of U_X (row-major, n even) into buf (rows x n)
__device__ __forceinline__ void stage_rows(double* buf, const double* ux, long long r0, int rows,
                                           int n) {
  const int chunks = rows * n / 2;               // 16-byte chunks
  const double* src = ux + r0 * n;
  for (int q = threadIdx.x; q < chunks; q += blockDim.x) cp_async16(buf + 2 * q, src + 2 * q);
  cp_async_commit();
}

// dot of a staged U row (smem, 16-B aligned) with a register column, two
// interleaved partial sums (fixed order)
template <int NB>
__device__ __forceinline__ double row_dot(const double* urow, const double* zc, int n) {
  const double2* u2 = reinterpret_cast<const double2*>(urow);
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int k = 0; k < NB / 2; ++k) {
    if (2 * k < n) {
      const double2 uv = u2[k];
      s0 = fma(uv.x, zc[2 * k], s0);
      s1 = fma(uv.y, zc[2 * k + 1], s1);
    }
  }
  return s0 + s1;
}

// Reconstruct + deposit: thread (r, jl) owns column c = tile*PT + jl and a
// private histogram [row][tid] (conflict-free); U_X rows stream through a
// double-buffered smem tile shared by all columns of the CTA.
template <int D, int NB, int R>
__global__ void __launch_bounds__(384) rom_deposit_kernel(RomArgs a) {
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(16) double smem[];
  const int P = blockDim.x / R;               // columns per row group (mult of 32)
  const int H = blockDim.x;
  const int nh = a.nx + D;
  const int n = a.n;
  double* ut = smem;                          // [2][TR * n]
  double* hist = ut + 2 * TR * n;             // [nh][H]
  const int tid = threadIdx.x;
  const int r = tid / P, jl = tid % P;
  const int c = blockIdx.y * PT + jl;         // z column
  const bool active = c < a.p && jl < PT;
  const int inst_id = active ? (a.cols ? a.cols[c] : c) : 0;
  const double* ip = a.inst + (size_t)inst_id * PICROM_INST_STRIDE;
  const double h = ip[I_H], inv_h = ip[I_INVH];
  const double inv_nx = 1.0 / (double)a.nx;
  const int mask = fast_mask(a.nx, h);
  double zc[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) zc[k] = (active && k < n) ? a.z[(size_t)k * a.ldz + c] : 0.0;
  for (int q = tid; q < nh * H; q += blockDim.x) hist[q] = 0.0;
  const long long lo = row_start(blockIdx.x, a.N, gridDim.x);
  const long long hi = row_start(blockIdx.x + 1, a.N, gridDim.x);
  const int ntiles = (int)((hi - lo + TR - 1) / TR);
  if (ntiles > 0) stage_rows(ut, a.ux, lo, (int)min((long long)TR, hi - lo), n);
  for (int t = 0; t < ntiles; ++t) {
    const long long t0 = lo + (long long)t * TR;
    const int rows = (int)min((long long)TR, hi - t0);
    if (t + 1 < ntiles) {
      const long long t1 = t0 + TR;
      stage_rows(ut + ((t + 1) & 1) * TR * n, a.ux, t1, (int)min((long long)TR, hi - t1), n);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* tile = ut + (t & 1) * TR * n;
    if (active) {
      for (int rr = r; rr < rows; rr += 2 * R) {
        const bool two = rr + R < rows;
        double xv[2];
        xv[0] = row_dot<NB>(tile + rr * n, zc, n);
        xv[1] = two ? row_dot<NB>(tile + (rr + R) * n, zc, n) : 0.0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (q == 1 && !two) break;
          const double x = xv[q];
          int cell;
          double f;
          bool rare;
          locate_fast(x, h, inv_h, a.nx, mask, inv_nx, cell, f, rare);
          if (rare) {
            if (!isfinite(x)) {
              record_bad(a.status, 0, t0 + rr + q * R, c, a.p);
              continue;
            }
            locate(x, h, inv_h, a.nx, inv_nx, cell, f);
          }
          double w[D + 1];
          Spline<D>::weights(f, w);
          double* hp = hist + cell * H + tid;
          double cur[D + 1];
#pragma unroll
          for (int m = 0; m <= D; ++m) cur[m] = hp[m * H];
#pragma unroll
          for (int m = 0; m <= D; ++m) hp[m * H] = cur[m] + w[m];
        }
      }
    }
    __syncthreads();
  }
  // fold ghost rows and row groups (fixed order) -> seg[b][c][nd]
  const int P_used = min(PT, a.p - blockIdx.y * PT);
  for (int q = tid; q < P_used * a.nx; q += blockDim.x) {
    const int cl = q / a.nx, nd = q % a.nx;
    double s = 0.0;
    for (int rr = (nd - Spline<D>::OFF) % a.nx; rr < nh; rr += a.nx)
      for (int g = 0; g < R; ++g) s += hist[rr * H + g * P + cl];
    a.seg[((size_t)blockIdx.x * a.p + blockIdx.y * PT + cl) * a.nx + nd] = s;
  }
}

// Reconstruct + field gather + projection U_X^T E (+ optional DEIM harvest
// lam and E output), same tiling; phi of the CTA's columns in smem [node][col].
template <int D, int NB, int R>
__global__ void __launch_bounds__(384) rom_gather_kernel(RomArgs a) {
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(16) double smem[];
  const int P = blockDim.x / R;
  const int tid = threadIdx.x;
  const int r = tid / P, jl = tid % P;
  const int c = blockIdx.y * PT + jl;
  const bool active = c < a.p && jl < PT;
  const int nx = a.nx;
  const int n = a.n;
  double* ut = smem;                           // [2][TR * n]
  double* phs = ut + 2 * TR * n;               // [nx][P]
  double* red = phs + (size_t)nx * P;          // [R][P][n] row-group partials
  const int P_used = min(PT, a.p - blockIdx.y * PT);
  for (int q = tid; q < nx * P; q += blockDim.x) {
    const int nd = q / P, cl = q % P;
    phs[q] = cl < P_used ? a.phi[(size_t)(blockIdx.y * PT + cl) * nx + nd] : 0.0;
  }
  const int inst_id = active ? (a.cols ? a.cols[c] : c) : 0;
  const double* ip = a.inst + (size_t)inst_id * PICROM_INST_STRIDE;
  const double h = ip[I_H], g = ip[I_INVH], inv_h = g;
  const double cf = a.coef_kind == 0 ? ip[I_GCOEF] : 1.0;
  const double inv_nx = 1.0 / (double)nx;
  const int mask = fast_mask(nx, h);
  double zc[NB], acc[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    zc[k] = (active && k < n) ? a.z[(size_t)k * a.ldz + c] : 0.0;
    acc[k] = 0.0;
  }
  const long long lo = row_start(blockIdx.x, a.N, gridDim.x);
  const long long hi = row_start(blockIdx.x + 1, a.N, gridDim.x);
  const int ntiles = (int)((hi - lo + TR - 1) / TR);
  if (ntiles > 0) stage_rows(ut, a.ux, lo, (int)min((long long)TR, hi - lo), n);
  for (int t = 0; t < ntiles; ++t) {
    const long long t0 = lo + (long long)t * TR;
    const int rows = (int)min((long long)TR, hi - t0);
    if (t + 1 < ntiles) {
      const long long t1 = t0 + TR;
      stage_rows(ut + ((t + 1) & 1) * TR * n, a.ux, t1, (int)min((long long)TR, hi - t1), n);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* tile = ut + (t & 1) * TR * n;
    if (active) {
      for (int rr = r; rr < rows; rr += R) {
        const double* urow = tile + rr * n;
        const double x = row_dot<NB>(urow, zc, n);
        const long long i = t0 + rr;
        int cell;
        double f;
        bool rare;
        locate_fast(x, h, inv_h, nx, mask, inv_nx, cell, f, rare);
        if (rare) {
          if (!isfinite(x)) {
            record_bad(a.status, 0, i, c, a.p);
            continue;
          }
          locate(x, h, inv_h, nx, inv_nx, cell, f);
        }
        double pv[D + 1];
#pragma unroll
        for (int m = 0; m <= D; ++m) {
          int nd = cell + Spline<D>::OFF + m;
          nd = nd < 0 ? nd + nx : (nd >= nx ? nd - nx : nd);
          pv[m] = phs[nd * P + jl];
        }
        double E;
        if constexpr (D == 1) {   // coef * ((-g)*phi0 + g*phi1): driver.py:74-75 order
          E = __dmul_rn(cf, __dadd_rn(__dmul_rn(-g, pv[0]), __dmul_rn(g, pv[1])));
        } else {
          double dw[D + 1];
          Spline<D>::dweights(f, g, dw);
          double s = 0.0;
#pragma unroll
          for (int m = 0; m <= D; ++m) s = fma(dw[m], pv[m], s);
          E = cf * s;
        }
        const double2* u2 = reinterpret_cast<const double2*>(urow);
#pragma unroll
        for (int k = 0; k < NB / 2; ++k) {
          if (2 * k < n) {
            const double2 uv = u2[k];
            acc[2 * k] = fma(uv.x, E, acc[2 * k]);
            acc[2 * k + 1] = fma(uv.y, E, acc[2 * k + 1]);
          }
        }
        if (a.eout) a.eout[(size_t)i * a.ldo + c] = E;
        if (a.lam) {
          double lv;
          if constexpr (D == 1) {
            lv = __dadd_rn(__dmul_rn(__dsub_rn(1.0, f), pv[0]), __dmul_rn(f, pv[1]));
          } else {
            double w[D + 1];
            Spline<D>::weights(f, w);
            lv = 0.0;
#pragma unroll
            for (int m = 0; m <= D; ++m) lv = fma(w[m], pv[m], lv);
          }
          a.lam[(size_t)i * a.ldo + c] = lv;
        }
      }
    }
    __syncthreads();
  }
  // row-group partials -> smem -> fixed-order sum -> seg[b][c][k]
#pragma unroll
  for (int k = 0; k < NB; ++k)
    if (k < n) red[((size_t)r * P + jl) * n + k] = acc[k];
  __syncthreads();
  for (int q = tid; q < P_used * n; q += blockDim.x) {
    const int cl = q / n, k = q % n;
    double s = 0.0;
    for (int rr = 0; rr < R; ++rr) s += red[((size_t)rr * P + cl) * n + k];
    a.seg[((size_t)blockIdx.x * a.p + blockIdx.y * PT + cl) * n + k] = s;
  }
}

// out[c][k] (and optional transpose layout) = sum_b seg[b][c][k]
// 256 threads = 64 entries x 4 slices of the G partials; a thread sums its
// slice (b = slice, slice + 4, ...) with 8 loads in flight, the 4 slices are
// combined through smem -- a fixed order (deterministic), and ~G/32 dependent
// L2 round trips instead of ~G/4: this kernel sits behind every F-evaluation
// and Gram and is pure latency
constexpr int SEGQ = 64;
__global__ void __launch_bounds__(256)
seg_sum_kernel(const double* seg, int G, int rows, double* out, int out_ld,
               int transpose, int width, const long long* skip = nullptr) {
  if (skip && *skip) return;
  __shared__ double part[4][SEGQ];
  const int ql = threadIdx.x & (SEGQ - 1), slice = threadIdx.x / SEGQ;
  const int q = blockIdx.x * SEGQ + ql;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (q < rows) {
    int b = slice;
    for (; b + 28 < G; b += 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += __ldcg(seg + (size_t)(b + 4 * u) * rows + q);
    }
    for (int u = 0; b < G; b += 4, ++u) acc[u] += __ldcg(seg + (size_t)b * rows + q);
  }
  part[slice][ql] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  __syncthreads();
  if (slice != 0 || q >= rows) return;
  const double s = (part[0][ql] + part[1][ql]) + (part[2][ql] + part[3][ql]);
  if (transpose) {  // q = c*width + k  ->  out[k][c]
    const int c = q / width, k = q % width;
    out[(size_t)k * out_ld + c] = s;
  } else {
    out[q] = s;
  }
}

// ---------------------------------------------------------------- Gram

constexpr int MAXB = 8;   // column blocks
struct Blocks {
  const double* ptr[MAXB];
  int ld[MAXB];
  int w[MAXB];
  int off[MAXB + 1];
  int jswap[MAXB];   // 1: block is J B (row i reads row (i + N/2) mod N, lower half negated)
  int nb;
};

// row index / sign of (J B) row i for a 2*half-row block B
__device__ __forceinline__ long long jrow(long long i, long long half, double& sgn) {
  if (i < half) { sgn = 1.0; return i + half; }
  sgn = -1.0;
  return i - half;
}

constexpr int TB = 4;      // output sub-block per thread

// out = A^T B with A = blocks [0, na), B = blocks [na, nb) (na == 0: W^T W over
// all blocks).  Rows stream through a double-buffered smem tile filled with
// 8-byte cp.async (J-swapped blocks read the partner row; the sign of their
// lower half is applied in smem); each thread accumulates TB x TB output
// sub-blocks in registers; per-CTA partials -> seg (fixed-order reduce).
constexpr int GTR = 32;          // rows per tile

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}

template <int TBK, int MAXT>
__global__ void __launch_bounds__(256) gram_kernel(Blocks b, int na, long long N, double* seg) {
  extern __shared__ __align__(16) double gsm[];
  const int W = b.off[b.nb];
  double* tile = gsm;                                  // [2][GTR][W]
  const double** cbase = reinterpret_cast<const double**>(tile + 2 * GTR * W);   // [W]
  int* cld = reinterpret_cast<int*>(cbase + W);        // [W]
  int* cjs = cld + W;                                  // [W]
  const int a0 = 0, a1 = na > 0 ? b.off[na] : W;       // A columns [a0, a1)
  const int b0 = na > 0 ? b.off[na] : 0, b1 = W;       // B columns [b0, b1)
  const int wa = a1 - a0, wb = b1 - b0;
  const int nbA = (wa + TBK - 1) / TBK, nbB = (wb + TBK - 1) / TBK;
  const int ntiles = nbA * nbB;
  // row groups: when the output has fewer sub-blocks than threads, split the
  // rows of each smem tile among RG groups (partials reduced in seg_sum)
  const int RG = ntiles >= (int)blockDim.x ? 1 : (int)blockDim.x / ntiles;
  const int grp = RG > 1 ? (int)threadIdx.x / ntiles : 0;
  const int tslot = RG > 1 ? (int)threadIdx.x % ntiles : (int)threadIdx.x;
  const long long half = N / 2;
  bool any_js = false;
  for (int i = 0; i < b.nb; ++i) any_js |= b.jswap[i] != 0;
  for (int col = threadIdx.x; col < W; col += blockDim.x) {
    int bi = 0;
    while (col >= b.off[bi + 1]) ++bi;
    cbase[col] = b.ptr[bi] + (col - b.off[bi]);
    cld[col] = b.ld[bi];
    cjs[col] = b.jswap[bi];
  }
  __syncthreads();
  const long long lo = row_start(blockIdx.x, N, gridDim.x);
  const long long hi = row_start(blockIdx.x + 1, N, gridDim.x);
  const int nt = (int)((hi - lo + GTR - 1) / GTR);
  auto stage = [&](int t) {
    const long long r0 = lo + (long long)t * GTR;
    const int rows = (int)min((long long)GTR, hi - r0);
    double* dst = tile + (t & 1) * GTR * W;
    for (int q = threadIdx.x; q < rows * W; q += blockDim.x) {
      const int rr = q / W, col = q - rr * W;
      long long row = r0 + rr;
      if (cjs[col]) row = row < half ? row + half : row - half;
      cp_async8(dst + q, cbase[col] + (size_t)row * cld[col]);
    }
    cp_async_commit();
  };
  double acc[MAXT][TBK][TBK];
#pragma unroll
  for (int s = 0; s < MAXT; ++s)
#pragma unroll
    for (int i = 0; i < TBK; ++i)
#pragma unroll
      for (int j = 0; j < TBK; ++j) acc[s][i][j] = 0.0;
  const bool in_range = grp < RG && (RG > 1 ? (int)threadIdx.x < RG * ntiles : true);
  if (nt > 0) stage(0);
  for (int t = 0; t < nt; ++t) {
    const long long r0 = lo + (long long)t * GTR;
    const int rows = (int)min((long long)GTR, hi - r0);
    if (t + 1 < nt) { stage(t + 1); cp_async_wait<1>(); } else { cp_async_wait<0>(); }
    __syncthreads();
    double* cur = tile + (t & 1) * GTR * W;
    if (any_js && r0 + rows > half) {      // J: negate the (new) lower half of swapped blocks
      for (int q = threadIdx.x; q < rows * W; q += blockDim.x) {
        const int rr = q / W, col = q - rr * W;
        if (cjs[col] && r0 + rr >= half) cur[q] = -cur[q];
      }
      __syncthreads();
    }
    if (in_range) {
#pragma unroll
      for (int s = 0; s < MAXT; ++s) {
        const int tt = tslot + s * blockDim.x;
        if (tt >= ntiles) break;
        const int bi = tt / nbB, bj = tt % nbB;
        for (int rr = grp; rr < rows; rr += RG) {
          double av[TBK], bv[TBK];
#pragma unroll
          for (int i = 0; i < TBK; ++i) {
            const int ci = bi * TBK + i, cj = bj * TBK + i;
            av[i] = ci < wa ? cur[rr * W + a0 + ci] : 0.0;
            bv[i] = cj < wb ? cur[rr * W + b0 + cj] : 0.0;
          }
#pragma unroll
          for (int i = 0; i < TBK; ++i)
#pragma unroll
            for (int j = 0; j < TBK; ++j) acc[s][i][j] = fma(av[i], bv[j], acc[s][i][j]);
        }
      }
    }
    __syncthreads();
  }
  if (!in_range) return;
  // partial slot (CTA, row group): seg[(blockIdx.x * RG + grp)][wa][wb]
  double* out = seg + ((size_t)blockIdx.x * RG + grp) * wa * wb;
#pragma unroll
  for (int s = 0; s < MAXT; ++s) {
    const int tt = tslot + s * blockDim.x;
    if (tt >= ntiles) break;
    const int bi = tt / nbB, bj = tt % nbB;
#pragma unroll
    for (int i = 0; i < TBK; ++i)
#pragma unroll
      for (int j = 0; j < TBK; ++j) {
        const int ci = bi * TBK + i, cj = bj * TBK + j;
        if (ci < wa && cj < wb) out[(size_t)ci * wb + cj] = acc[s][i][j];
      }
  }
}

// TMA variant of the Gram (all blocks row-contiguous, 16-B aligned): each
// tile of GT2 rows of every block lands in smem with ONE cp.async.bulk per
// block (two for a J-swapped block straddling N/2), double-buffered on
// mbarriers; the LSU issues nothing for the staging.
constexpr int GT2 = 64;

template <int TBK, int MAXT>
__global__ void __launch_bounds__(256) gram_tma_kernel(Blocks b, int na, long long N, double* seg) {
  extern __shared__ __align__(128) double gsm2[];
  const int W = b.off[b.nb];
  const int SZ = GT2 * W;                                   // doubles per stage
  double* stages = gsm2;                                    // [2][SZ] (block-major sub-tiles)
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + 2 * SZ);
  const int a0 = 0, a1 = na > 0 ? b.off[na] : W;
  const int b0 = na > 0 ? b.off[na] : 0, b1 = W;
  const int wa = a1 - a0, wb = b1 - b0;
  const int nbA = (wa + TBK - 1) / TBK, nbB = (wb + TBK - 1) / TBK;
  const int ntiles = nbA * nbB;
  const int RG = ntiles >= (int)blockDim.x ? 1 : (int)blockDim.x / ntiles;
  const int grp = RG > 1 ? (int)threadIdx.x / ntiles : 0;
  const int tslot = RG > 1 ? (int)threadIdx.x % ntiles : (int)threadIdx.x;
  const bool in_range = RG > 1 ? (int)threadIdx.x < RG * ntiles : true;
  const long long half = N / 2;
  bool any_js = false;
  for (int i = 0; i < b.nb; ++i) any_js |= b.jswap[i] != 0;
  const long long lo = row_start(blockIdx.x, N, gridDim.x);
  const long long hi = row_start(blockIdx.x + 1, N, gridDim.x);
  const int nt = (int)((hi - lo + GT2 - 1) / GT2);
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int t) {            // thread 0 only
    const long long r0 = lo + (long long)t * GT2;
    const int rows = (int)min((long long)GT2, hi - r0);
    double* st = stages + (t & 1) * SZ;
    uint32_t bytes = 0;
    for (int i = 0; i < b.nb; ++i) bytes += (uint32_t)rows * b.w[i] * 8u;
    if (any_js) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the smem negation pass
    mbar_expect_tx(&full[t & 1], bytes);
    for (int i = 0; i < b.nb; ++i) {
      double* dst = st + GT2 * b.off[i];
      const int w = b.w[i];
      if (!b.jswap[i]) {
        bulk_g2s(dst, b.ptr[i] + (size_t)r0 * w, (uint32_t)rows * w * 8u, &full[t & 1]);
      } else {   // rows r < half read r + half, rows r >= half read r - half
        const long long m = min(r0 + rows, max(r0, half));       // split point
        if (m > r0)
          bulk_g2s(dst, b.ptr[i] + (size_t)(r0 + half) * w, (uint32_t)(m - r0) * w * 8u, &full[t & 1]);
        if (r0 + rows > m)
          bulk_g2s(dst + (m - r0) * w, b.ptr[i] + (size_t)(m - half) * w,
                   (uint32_t)(r0 + rows - m) * w * 8u, &full[t & 1]);
      }
    }
  };
  double acc[MAXT][TBK][TBK];
#pragma unroll
  for (int s = 0; s < MAXT; ++s)
#pragma unroll
    for (int i = 0; i < TBK; ++i)
#pragma unroll
      for (int j = 0; j < TBK; ++j) acc[s][i][j] = 0.0;
  if (threadIdx.x == 0 && nt > 0) issue(0);
  for (int t = 0; t < nt; ++t) {
    const long long r0 = lo + (long long)t * GT2;
    const int rows = (int)min((long long)GT2, hi - r0);
    if (threadIdx.x == 0 && t + 1 < nt) issue(t + 1);   // stage (t+1)&1 was released at the end of t-1
    mbar_wait(&full[t & 1], (uint32_t)((t >> 1) & 1));
    double* st = stages + (t & 1) * SZ;
    if (any_js && r0 + rows > half) {      // J: negate the new lower half of swapped blocks
      for (int i = 0; i < b.nb; ++i) {
        if (!b.jswap[i]) continue;
        const int w = b.w[i];
        const int first = (int)max(0LL, half - r0);
        for (int q = threadIdx.x; q < (rows - first) * w; q += blockDim.x)
          st[GT2 * b.off[i] + first * w + q] = -st[GT2 * b.off[i] + first * w + q];
      }
      __syncthreads();
    }
    if (in_range) {
#pragma unroll
      for (int s = 0; s < MAXT; ++s) {
        const int tt = tslot + s * blockDim.x;
        if (tt >= ntiles) break;
        const int bi = tt / nbB, bj = tt % nbB;
        // smem (offset, stride) of the thread's A and B columns
        int ao[TBK], as_[TBK], bo[TBK], bs[TBK];
#pragma unroll
        for (int i = 0; i < TBK; ++i) {
          const int ca = a0 + min(bi * TBK + i, wa - 1), cb = b0 + min(bj * TBK + i, wb - 1);
          int ba = 0, bb = 0;
          while (ca >= b.off[ba + 1]) ++ba;
          while (cb >= b.off[bb + 1]) ++bb;
          ao[i] = GT2 * b.off[ba] + (ca - b.off[ba]);
          as_[i] = b.w[ba];
          bo[i] = GT2 * b.off[bb] + (cb - b.off[bb]);
          bs[i] = b.w[bb];
        }
        for (int rr = grp; rr < rows; rr += RG) {
          double av[TBK], bv[TBK];
#pragma unroll
          for (int i = 0; i < TBK; ++i) {
            av[i] = st[ao[i] + rr * as_[i]];
            bv[i] = st[bo[i] + rr * bs[i]];
          }
#pragma unroll
          for (int i = 0; i < TBK; ++i)
#pragma unroll
            for (int j = 0; j < TBK; ++j) acc[s][i][j] = fma(av[i], bv[j], acc[s][i][j]);
        }
      }
    }
    __syncthreads();                       // stage t&1 free for tile t+2
  }
  if (!in_range) return;
  double* out = seg + ((size_t)blockIdx.x * RG + grp) * wa * wb;
#pragma unroll
  for (int s = 0; s < MAXT; ++s) {
    const int tt = tslot + s * blockDim.x;
    if (tt >= ntiles) break;
    const int bi = tt / nbB, bj = tt % nbB;
#pragma unroll
    for (int i = 0; i < TBK; ++i)
#pragma unroll
      for (int j = 0; j < TBK; ++j) {
        const int ci = bi * TBK + i, cj = bj * TBK + j;
        if (ci < wa && cj < wb) out[(size_t)ci * wb + cj] = acc[s][i][j];
      }
  }
}

// ---- FP64 tensor-core (DMMA) Gram: mma.sync.m8n8k4 f64 ----
//
// D (8x8) += A (8x4) B (4x8), one f64 per lane for A and B, two for D:
// A[l>>2][l&3], B[l&3][l>>2], D[l>>2][2(l&3) + e].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

constexpr int MAXTASK = 64;
struct GramTasks {             // block pairs (bi, bj) of the output, TPC per CTA group
  int ntask;
  unsigned char bi[MAXTASK], bj[MAXTASK];
};

// All blocks wdt (<= 32) wide, row-contiguous, 16-B aligned.  Grid: x = task
// group (TPC block pairs), y = row chunk.  A CTA stages only the blocks its
// tasks read (TMA bulk copies, 2 stages of GT rows, mbarriers); its 8 warps
// split the 4-row k-steps and each accumulates every task's TB x TB tiles of
// 8x8 in DMMA fragments; warps are summed in a fixed order in smem and the
// CTA writes its entries of row-chunk slot y (seg[y][wa][wb]).
template <int TB, int TPC>
__global__ void __launch_bounds__(256, 2)
gram_mma_kernel(Blocks b, GramTasks tk, int na, long long N, int GT, int wn, double* seg) {
  extern __shared__ __align__(128) double msm[];
  __shared__ int s_loc[MAXB];
  const int wdt = b.w[0];
  const int W = b.off[b.nb];
  const int b0 = na > 0 ? b.off[na] : 0;
  const int wa = na > 0 ? b.off[na] : W, wb = na > 0 ? W - b0 : W;
  const int t_lo = blockIdx.x * TPC;
  const int t_n = min(TPC, tk.ntask - t_lo);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    unsigned need = 0;
    for (int t = 0; t < t_n; ++t) need |= (1u << tk.bi[t_lo + t]) | (1u << tk.bj[t_lo + t]);
    int loc = 0;
    for (int i = 0; i < b.nb; ++i) {
      s_loc[i] = (need >> i) & 1u ? loc : -1;
      if ((need >> i) & 1u) loc += wdt;
    }
  }
  const int SZ = GT * wn;
  double* stages = msm;                                      // [2][GT][wn] block-major
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + 2 * SZ);
  double* red = reinterpret_cast<double*>(full + 2);         // [TPC][TB][TB][64]
  const long long half = N / 2;
  const long long lo = row_start(blockIdx.y, N, gridDim.y);
  const long long hi = row_start(blockIdx.y + 1, N, gridDim.y);
  const int nt = (int)((hi - lo + GT - 1) / GT);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  bool any_js = false;
  for (int i = 0; i < b.nb; ++i) any_js |= (b.jswap[i] != 0 && s_loc[i] >= 0);
  auto issue = [&](int t) {            // thread 0 only
    const long long r0 = lo + (long long)t * GT;
    const int rows = (int)min((long long)GT, hi - r0);
    double* st = stages + (t & 1) * SZ;
    uint32_t bytes = 0;
    for (int i = 0; i < b.nb; ++i)
      if (s_loc[i] >= 0) bytes += (uint32_t)rows * wdt * 8u;
    if (any_js) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&full[t & 1], bytes);
    for (int i = 0; i < b.nb; ++i) {
      if (s_loc[i] < 0) continue;
      double* dst = st + GT * s_loc[i];
      if (!b.jswap[i]) {
        bulk_g2s(dst, b.ptr[i] + (size_t)r0 * wdt, (uint32_t)rows * wdt * 8u, &full[t & 1]);
      } else {
        const long long m = min(r0 + rows, max(r0, half));
        if (m > r0)
          bulk_g2s(dst, b.ptr[i] + (size_t)(r0 + half) * wdt, (uint32_t)(m - r0) * wdt * 8u, &full[t & 1]);
        if (r0 + rows > m)
          bulk_g2s(dst + (m - r0) * wdt, b.ptr[i] + (size_t)(m - half) * wdt,
                   (uint32_t)(r0 + rows - m) * wdt * 8u, &full[t & 1]);
      }
    }
  };
  double acc[TPC][TB][TB][2];
#pragma unroll
  for (int t = 0; t < TPC; ++t)
#pragma unroll
    for (int i = 0; i < TB; ++i)
#pragma unroll
      for (int j = 0; j < TB; ++j) acc[t][i][j][0] = acc[t][i][j][1] = 0.0;
  // the lane's column inside an 8-wide tile, and its row inside a k-step
  const int lc = lane >> 2, lr = lane & 3;
  if (tid == 0 && nt > 0) issue(0);
  for (int t = 0; t < nt; ++t) {
    const long long r0 = lo + (long long)t * GT;
    const int rows = (int)min((long long)GT, hi - r0);
    if (tid == 0 && t + 1 < nt) issue(t + 1);
    mbar_wait(&full[t & 1], (uint32_t)((t >> 1) & 1));
    double* st = stages + (t & 1) * SZ;
    if (any_js && r0 + rows > half) {      // J: negate the new lower half of swapped blocks
      for (int i = 0; i < b.nb; ++i) {
        if (!b.jswap[i] || s_loc[i] < 0) continue;
        const int first = (int)max(0LL, half - r0);
        double* bl = st + GT * s_loc[i];
        for (int q = tid; q < (rows - first) * wdt; q += blockDim.x)
          bl[first * wdt + q] = -bl[first * wdt + q];
      }
      __syncthreads();
    }
    const int ksteps = (rows + 3) >> 2;
    for (int kk = warp; kk < ksteps; kk += 8) {
      const int r = kk * 4 + lr;
      const bool rv = r < rows;
#pragma unroll
      for (int tt = 0; tt < TPC; ++tt) {
        if (tt < t_n) {
          const int bi = tk.bi[t_lo + tt], bj = tk.bj[t_lo + tt];
          const double* pa = st + GT * s_loc[bi] + r * wdt;
          const double* pb = st + GT * s_loc[bj] + r * wdt;
          double fa[TB], fb[TB];
#pragma unroll
          for (int i = 0; i < TB; ++i) {
            const int c = 8 * i + lc;
            fa[i] = (rv && c < wdt) ? pa[c] : 0.0;
            fb[i] = (rv && c < wdt) ? pb[c] : 0.0;
          }
#pragma unroll
          for (int i = 0; i < TB; ++i)
#pragma unroll
            for (int j = 0; j < TB; ++j) dmma(acc[tt][i][j][0], acc[tt][i][j][1], fa[i], fb[j]);
        }
      }
    }
    __syncthreads();                       // stage t&1 free for tile t+2
  }
  // warps summed in a fixed order (warp 0 first)
  constexpr int NACC = TPC * TB * TB * 64;
  for (int w = 0; w < 8; ++w) {
    if (warp == w) {
#pragma unroll
      for (int tt = 0; tt < TPC; ++tt)
#pragma unroll
        for (int i = 0; i < TB; ++i)
#pragma unroll
          for (int j = 0; j < TB; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              double* q = red + ((tt * TB + i) * TB + j) * 64 + lane * 2 + e;
              *q = (w == 0) ? acc[tt][i][j][e] : *q + acc[tt][i][j][e];
            }
    }
    __syncthreads();
  }
  double* out = seg + (size_t)blockIdx.y * wa * wb;
  for (int q = tid; q < t_n * TB * TB * 64; q += blockDim.x) {
    const int e = q & 1, ln = (q >> 1) & 31, tile = q >> 6;
    const int j = tile % TB, i = (tile / TB) % TB, tt = tile / (TB * TB);
    const int bi = tk.bi[t_lo + tt], bj = tk.bj[t_lo + tt];
    const int ri = 8 * i + (ln >> 2), cj = 8 * j + 2 * (ln & 3) + e;
    if (ri >= wdt || cj >= wdt) continue;
    const int row = b.off[bi] + ri, col = b.off[bj] - b0 + cj;
    out[(size_t)row * wb + col] = red[q];
    if (na == 0 && bi != bj) out[(size_t)col * wb + row] = red[q];
  }
  (void)NACC;
}

// ---- tall A^T B for a WIDE left operand (the DEIM window, hyper.py:262) ----
//
// out (ca x k) = A^T B, A (N x ca, ld lda, ca <= 448: e.g. the (T+1) p* = 420
// window columns) and B (N x k, k <= 48: the subspace block).  The Gram kernels
// above take blocks <= 32 wide; here the output has up to 53 x 6 tiles of 8 x 8,
// so each of the 8 warps owns TPW row tiles (8 columns of A each) x CT column
// tiles of DMMA accumulators and every warp walks every 4-row k-step of the
// CTA's row chunk.  Tiles of ATG rows of A and B land in smem by one TMA bulk
// copy per row (pitches = 4 mod 16 doubles: the 4 rows x 8 columns of a
// fragment load cover each bank twice -- the 2-wavefront minimum of a 256-byte
// request), double buffered.  DMMA-bound: 42 DMMAs per 13 fragment loads at
// 420 x 48.  Per-CTA partials -> seg, summed in a fixed order.
constexpr int ATG = 16;      // rows per staged tile (64 in the k-split variant)
__host__ __device__ inline int atb_pitch(int w) {
  int p = w;
  while (p % 16 != 4) ++p;
  return p;
}
// KSPLIT (narrow A, ca <= 8 TPW: e.g. the 48 x 48 Gram of the subspace block):
// every warp owns ALL TPW x CT output tiles and the warps split the k-steps of
// a tile instead; their accumulators are summed through smem in warp order.
template <int TPW, int CT, bool KSPLIT>
__global__ void __launch_bounds__(256, 1)
tall_atb_kernel(const double* __restrict__ A, int lda, int ca, const double* __restrict__ B,
                int ldb, int k, long long N, double* seg, int pa, int pb) {
  extern __shared__ __align__(128) double tsm[];
  constexpr int TG = KSPLIT ? 4 * ATG : ATG;
  // smem pitches: atb_pitch (per-row copies), or the natural width of a
  // row-contiguous operand (pa == ca == lda: ONE bulk copy per tile -- the
  // k-split variant's tiles are small, 2 x 64 row copies of 384 bytes would
  // cost more than its DMMAs)
  const int SZ = TG * (pa + pb);
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + 2 * SZ);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lc = lane >> 2, lr = lane & 3;
  const int RT = (ca + 7) >> 3;
  const long long lo = row_start(blockIdx.x, N, gridDim.x);
  const long long hi = row_start(blockIdx.x + 1, N, gridDim.x);
  const int nt = (int)((hi - lo + TG - 1) / TG);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // warp 0 stages tile t: lane r copies row r of A and of B
  auto issue = [&](int t) {
    const long long r0 = lo + (long long)t * TG;
    const int rows = (int)min((long long)TG, hi - r0);
    double* st = tsm + (t & 1) * SZ;
    if (lane == 0) mbar_expect_tx(&full[t & 1], (uint32_t)rows * (uint32_t)(ca + k) * 8u);
    __syncwarp();
    if (pa == ca && lda == ca) {
      if (lane == 0) bulk_g2s(st, A + (size_t)r0 * lda, (uint32_t)rows * (uint32_t)ca * 8u, &full[t & 1]);
    } else {
      for (int r = lane; r < rows; r += 32)
        bulk_g2s(st + r * pa, A + (size_t)(r0 + r) * lda, (uint32_t)ca * 8u, &full[t & 1]);
    }
    if (pb == k && ldb == k) {
      if (lane == 0) bulk_g2s(st + TG * pa, B + (size_t)r0 * ldb, (uint32_t)rows * (uint32_t)k * 8u, &full[t & 1]);
    } else {
      for (int r = lane; r < rows; r += 32)
        bulk_g2s(st + TG * pa + r * pb, B + (size_t)(r0 + r) * ldb, (uint32_t)k * 8u, &full[t & 1]);
    }
  };
  double acc[TPW][CT][2];
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int j = 0; j < CT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (warp == 0 && nt > 0) issue(0);
  for (int t = 0; t < nt; ++t) {
    const long long r0 = lo + (long long)t * TG;
    const int rows = (int)min((long long)TG, hi - r0);
    if (warp == 0 && t + 1 < nt) issue(t + 1);
    mbar_wait(&full[t & 1], (uint32_t)((t >> 1) & 1));
    const double* sa = tsm + (t & 1) * SZ;
    const double* sb = sa + TG * pa;
    const int ksteps = (rows + 3) >> 2;
    for (int kk = KSPLIT ? warp : 0; kk < ksteps; kk += KSPLIT ? 8 : 1) {
      const int r = kk * 4 + lr;
      const bool rv = r < rows;
      double fb[CT], fa[TPW];
#pragma unroll
      for (int j = 0; j < CT; ++j) {
        const int c = 8 * j + lc;
        fb[j] = (rv && c < k) ? sb[r * pb + c] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int c = 8 * (KSPLIT ? i : warp + 8 * i) + lc;
        fa[i] = (rv && c < ca) ? sa[r * pa + c] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < TPW; ++i)
        if ((KSPLIT ? i : warp + 8 * i) < RT) {
#pragma unroll
          for (int j = 0; j < CT; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
        }
    }
    __syncthreads();                       // stage t&1 free for tile t+2
  }
  double* out = seg + (size_t)blockIdx.x * ca * k;
  if constexpr (KSPLIT) {
    // warps summed in a fixed order (warp 0 first) in smem (the stages are free)
    double* red = tsm;                     // [TPW][CT][64]
    for (int w = 0; w < 8; ++w) {
      if (warp == w) {
#pragma unroll
        for (int i = 0; i < TPW; ++i)
#pragma unroll
          for (int j = 0; j < CT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              double* q = red + (i * CT + j) * 64 + lane * 2 + e;
              *q = (w == 0) ? acc[i][j][e] : *q + acc[i][j][e];
            }
      }
      __syncthreads();
    }
    for (int q = tid; q < TPW * CT * 64; q += blockDim.x) {
      const int e = q & 1, ln = (q >> 1) & 31, tile = q >> 6;
      const int j = tile % CT, i = tile / CT;
      const int ri = 8 * i + (ln >> 2), cj = 8 * j + 2 * (ln & 3) + e;
      if (ri < ca && cj < k) out[(size_t)ri * k + cj] = red[q];
    }
  } else {
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int ri = 8 * (warp + 8 * i) + lc;
      if (ri >= ca) continue;
#pragma unroll
      for (int j = 0; j < CT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cj = 8 * j + 2 * lr + e;
          if (cj < k) out[(size_t)ri * k + cj] = acc[i][j][e];
        }
    }
  }
}

// ---- small dense algebra of the window SVD's Cholesky-QR chain (hyper.py:262) ----
//
// One CTA: G (k x k, SPD, k <= 48) -> R^-1 with G = R^T R (R upper triangular),
// so Q = Y R^-1 is orthonormal when G = Y^T Y.  info[0], info[1] = min / max of
// diag(R) (min <= 0: G was not positive definite; the ratio is the caller's
// conditioning check).  Keeps the chain Y -> Y^T Y -> R^-1 -> (W^T Y) R^-1 -> W M
// on the device: no host round trip between its tall products.
constexpr int SMK = 48;
__global__ void __launch_bounds__(256) small_cholinv_kernel(const double* g, int k, double* rinv,
                                                            double* info) {
  __shared__ double a[SMK][SMK + 1];     // lower factor L (G = L L^T), then L^-1
  __shared__ double li[SMK][SMK + 1];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int q = tid; q < k * k; q += blockDim.x) a[q / k][q % k] = g[q];
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (tid == 0) {
      const double d = a[j][j];
      if (!(d > 0.0)) bad = 1;
      a[j][j] = sqrt(d > 0.0 ? d : 1.0);
    }
    __syncthreads();
    const double djj = a[j][j];
    for (int i = j + 1 + tid; i < k; i += blockDim.x) a[i][j] /= djj;
    __syncthreads();
    const int m = k - j - 1;             // trailing lower triangle update
    for (int q = tid; q < m * m; q += blockDim.x) {
      const int i = j + 1 + q / m, c = j + 1 + q % m;
      if (c <= i) a[i][c] = fma(-a[i][j], a[c][j], a[i][c]);
    }
    __syncthreads();
  }
  // L^-1 by forward substitution, one column per thread
  for (int c = tid; c < k; c += blockDim.x) {
    for (int i = 0; i < k; ++i) {
      double x = i == c ? 1.0 : 0.0;
      for (int m = c; m < i; ++m) x = fma(-a[i][m], li[m][c], x);
      li[i][c] = i < c ? 0.0 : x / a[i][i];
    }
  }
  __syncthreads();
  // R^-1 = (L^T)^-1 = (L^-1)^T
  for (int q = tid; q < k * k; q += blockDim.x) rinv[q] = li[q % k][q / k];
  if (tid == 0) {
    double lo = a[0][0], hi = a[0][0];
    for (int j = 1; j < k; ++j) { lo = fmin(lo, a[j][j]); hi = fmax(hi, a[j][j]); }
    info[0] = bad ? 0.0 : lo;
    info[1] = hi;
  }
}

// out (r x k) = A (r x k) B (k x k), column j scaled by colscale[j] (nullable)
__global__ void __launch_bounds__(SMK) small_rmul_kernel(const double* a, int r, int k,
                                                         const double* b, const double* colscale,
                                                         double* out) {
  __shared__ double bs[SMK][SMK + 1];
  __shared__ double row[SMK];
  const int j = threadIdx.x;
  for (int q = j; q < k * k; q += blockDim.x) bs[q / k][q % k] = b[q];
  for (int i = blockIdx.x; i < r; i += gridDim.x) {
    __syncthreads();
    if (j < k) row[j] = a[(size_t)i * k + j];
    __syncthreads();
    if (j < k) {
      double acc = 0.0;
      for (int m = 0; m < k; ++m) acc = fma(row[m], bs[m][j], acc);
      out[(size_t)i * k + j] = colscale ? acc * colscale[j] : acc;
    }
  }
}

// first index of max |v[i*stride]| over i < n, skipping `banned` (numpy
// argmax tie rule: the smallest index among equal maxima); banned entries
// score -1 as in hyper.py:241-243.  Two passes: per-CTA (value, index), then
// one CTA over the partials.
__device__ __forceinline__ void better(double v, long long i, double& bv, long long& bi) {
  if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}

__global__ void argmax_abs_kernel(const double* v, long long n, long long stride,
                                  const long long* banned, int nbanned, double* pv, long long* pi) {
  __shared__ double sv[256];
  __shared__ long long si[256];
  __shared__ long long sb[256];          // banned indices (smem broadcast reads)
  const int nbs = min(nbanned, 256);
  for (int k = threadIdx.x; k < nbs; k += blockDim.x) sb[k] = banned[k];
  __syncthreads();
  double bv = -2.0;
  long long bi = 0x7fffffffffffffffLL;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double s = fabs(v[i * stride]);
    bool ban = false;
    for (int k = 0; k < nbs; ++k) ban |= sb[k] == i;
    for (int k = nbs; k < nbanned; ++k) ban |= banned[k] == i;
    better(ban ? -1.0 : s, i, bv, bi);
  }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      double ov = sv[threadIdx.x + o];
      long long oi = si[threadIdx.x + o];
      double cv = sv[threadIdx.x];
      long long ci = si[threadIdx.x];
      better(ov, oi, cv, ci);
      sv[threadIdx.x] = cv;
      si[threadIdx.x] = ci;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pv[blockIdx.x] = sv[0];
    pi[blockIdx.x] = si[0];
  }
}

__global__ void argmax_final_kernel(const double* pv, const long long* pi, int m, long long* out_i,
                                    double* out_v) {
  double bv = -2.0;
  long long bi = 0x7fffffffffffffffLL;
  if (threadIdx.x == 0) {
    for (int k = 0; k < m; ++k) better(pv[k], pi[k], bv, bi);
    *out_i = bi;
    if (out_v) *out_v = bv;
  }
}

// ------------------------------------------------------------- combine

constexpr int MAXTERM = 6;
struct Terms {
  const double* in[MAXTERM];   // tall input block (N x a_t), row stride ld_t
  int jswap[MAXTERM];          // 1: use J in_t (rows swapped by halves, lower half negated)
  int ld[MAXTERM];
  int a[MAXTERM];
  int moff[MAXTERM];           // offset of M_t (a_t x c, row-major) in the matrix buffer
  int nt;
  double* out;                 // (N x c), row stride ldo
  int ldo, c;
  int accumulate;              // out += result
};

__global__ void __launch_bounds__(256) combine_kernel(Terms t, const double* mats, int mats_len,
                                                     long long N) {
  extern __shared__ double ms[];
  for (int q = threadIdx.x; q < mats_len; q += blockDim.x) ms[q] = mats[q];
  __syncthreads();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= N) return;
  double acc[NMAX];
#pragma unroll
  for (int k = 0; k < NMAX; ++k) acc[k] = 0.0;
  for (int s = 0; s < t.nt; ++s) {
    long long ri = i;
    double sgn = 1.0;
    if (t.jswap[s]) ri = jrow(i, N / 2, sgn);
    const double* row = t.in[s] + (size_t)ri * t.ld[s];
    const double* M = ms + t.moff[s];
    for (int kk = 0; kk < t.a[s]; ++kk) {
      const double v = sgn * __ldg(row + kk);
      const double* mr = M + kk * t.c;
#pragma unroll
      for (int k = 0; k < NMAX; ++k)
        if (k < t.c) acc[k] = fma(v, mr[k], acc[k]);
    }
  }
  double* o = t.out + (size_t)i * t.ldo;
#pragma unroll
  for (int k = 0; k < NMAX; ++k)
    if (k < t.c) o[k] = t.accumulate ? o[k] + acc[k] : acc[k];
}

// TMA-staged combine: out (rows x c) (+)= sum_t op_t(in_t) M_t.  Row tiles of
// every input land in smem via cp.async.bulk (double-buffered, mbarriers);
// 4 threads per row each produce ceil(c/4) outputs; M_t live in smem.
constexpr int CR = 64;     // rows per tile

template <int CPT>
__global__ void __launch_bounds__(256) combine_tma_kernel(Terms t, const double* mats, int mats_len,
                                                          long long N) {
  extern __shared__ __align__(128) double csm[];
  int wsum = 0;
  int soff[MAXTERM];
  for (int s = 0; s < t.nt; ++s) { soff[s] = CR * wsum; wsum += t.a[s]; }
  const int SZ = CR * wsum;
  double* stages = csm;                                  // [2][SZ]
  double* ms = stages + 2 * SZ;                          // mats
  uint64_t* full = reinterpret_cast<uint64_t*>(ms + ((mats_len + 1) & ~1));
  for (int q = threadIdx.x; q < mats_len; q += blockDim.x) ms[q] = mats[q];
  const long long half = N / 2;
  bool any_js = false;
  for (int s = 0; s < t.nt; ++s) any_js |= t.jswap[s] != 0;
  const long long lo = row_start(blockIdx.x, N, gridDim.x);
  const long long hi = row_start(blockIdx.x + 1, N, gridDim.x);
  const int ntl = (int)((hi - lo + CR - 1) / CR);
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int k) {
    const long long r0 = lo + (long long)k * CR;
    const int rows = (int)min((long long)CR, hi - r0);
    double* st = stages + (k & 1) * SZ;
    if (any_js) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&full[k & 1], (uint32_t)rows * wsum * 8u);
    for (int s = 0; s < t.nt; ++s) {
      const int w = t.a[s];
      double* dst = st + soff[s];
      if (!t.jswap[s]) {
        bulk_g2s(dst, t.in[s] + (size_t)r0 * w, (uint32_t)rows * w * 8u, &full[k & 1]);
      } else {
        const long long m = min(r0 + rows, max(r0, half));
        if (m > r0) bulk_g2s(dst, t.in[s] + (size_t)(r0 + half) * w, (uint32_t)(m - r0) * w * 8u, &full[k & 1]);
        if (r0 + rows > m)
          bulk_g2s(dst + (m - r0) * w, t.in[s] + (size_t)(m - half) * w, (uint32_t)(r0 + rows - m) * w * 8u,
                   &full[k & 1]);
      }
    }
  };
  const int row_l = threadIdx.x >> 2, q = threadIdx.x & 3;
  const int c0 = q * CPT;
  if (threadIdx.x == 0 && ntl > 0) issue(0);
  for (int k = 0; k < ntl; ++k) {
    const long long r0 = lo + (long long)k * CR;
    const int rows = (int)min((long long)CR, hi - r0);
    if (threadIdx.x == 0 && k + 1 < ntl) issue(k + 1);
    mbar_wait(&full[k & 1], (uint32_t)((k >> 1) & 1));
    double* st = stages + (k & 1) * SZ;
    if (any_js && r0 + rows > half) {
      const int first = (int)max(0LL, half - r0);
      for (int s = 0; s < t.nt; ++s) {
        if (!t.jswap[s]) continue;
        const int w = t.a[s];
        for (int e = threadIdx.x; e < (rows - first) * w; e += blockDim.x)
          st[soff[s] + first * w + e] = -st[soff[s] + first * w + e];
      }
      __syncthreads();
    }
    if (row_l < rows && c0 < t.c) {
      double acc[CPT];
#pragma unroll
      for (int j = 0; j < CPT; ++j) acc[j] = 0.0;
      for (int s = 0; s < t.nt; ++s) {
        const int w = t.a[s];
        const double* xr = st + soff[s] + row_l * w;
        const double* M = ms + t.moff[s] + c0;
        for (int kk = 0; kk < w; ++kk) {
          const double v = xr[kk];
          const double* mr = M + kk * t.c;
#pragma unroll
          for (int j = 0; j < CPT; ++j)
            if (c0 + j < t.c) acc[j] = fma(v, mr[j], acc[j]);
        }
      }
      double* o = t.out + (size_t)(r0 + row_l) * t.ldo + c0;
#pragma unroll
      for (int j = 0; j < CPT; ++j)
        if (c0 + j < t.c) o[j] = t.accumulate ? o[j] + acc[j] : acc[j];
    }
    __syncthreads();
  }
}

__global__ void rows_gather_kernel(const double* src, int ld, const long long* idx, int d, int w,
                                   double* out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= d * w) return;
  const int r = q / w, k = q % w;
  out[q] = src[(size_t)idx[r] * ld + k];
}

// phi (p x nx) = Re(modes (nx x r) . (coords (r x p) * w (r))), complex
// values interleaved (re, im); im_out (nullable) receives the imaginary part.
__global__ void dmd_extrap_kernel(const double2* modes, const double2* coords, const double2* w,
                                  int nx, int r, int p, double* re_out, double* im_out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nx * p) return;
  const int j = q / nx, nd = q % nx;
  double sr = 0.0, si = 0.0;
  for (int m = 0; m < r; ++m) {
    const double2 c = coords[(size_t)m * p + j], ww = w[m];
    const double cr = c.x * ww.x - c.y * ww.y, ci = c.x * ww.y + c.y * ww.x;
    const double2 md = modes[(size_t)nd * r + m];
    sr += md.x * cr - md.y * ci;
    si += md.x * ci + md.y * cr;
  }
  re_out[(size_t)j * nx + nd] = sr;
  if (im_out) im_out[(size_t)j * nx + nd] = si;
}

// DEIM-sampled gather + projection (hyper.py:320-328): one CTA per column j.
// xd_r = ux_d[r] . z_j ; e_r = dphi_j(xd_r) * w_r * wscale_j ;
// out[k][j] = inv_mp_j * sum_r ux_d[r][k] e_r   (out row stride ldo)
template <int D>
__global__ void deim_gather_kernel(const double* uxd, const double* z, int ldz, const double* phi,
                                   const double* inst, const int* cols, const double* w,
                                   const double* wscale, int d, int n, int p, int nx,
                                   double* out, int ldo, unsigned long long* status,
                                   const long long* skip) {
  if (skip && *skip) return;
  extern __shared__ double e[];
  const int j = blockIdx.x;
  const int inst_id = cols ? cols[j] : j;
  const double* ip = inst + (size_t)inst_id * PICROM_INST_STRIDE;
  const double h = ip[I_H], g = ip[I_INVH];
  const double* ph = phi + (size_t)j * nx;
  const double inv_nx = 1.0 / (double)nx;
  for (int rr = threadIdx.x; rr < d; rr += blockDim.x) {
    double x = 0.0;
    for (int k = 0; k < n; ++k) x = fma(uxd[(size_t)rr * n + k], z[(size_t)k * ldz + j], x);
    double dphi = 0.0;
    if (!isfinite(x)) {
      record_bad(status, 0, rr, j, p);
    } else {
      int c;
      double f;
      locate(x, h, g, nx, inv_nx, c, f);
      double pv[D + 1];
#pragma unroll
      for (int m = 0; m <= D; ++m) pv[m] = ph[wrap_node(c + Spline<D>::OFF + m, nx)];
      if constexpr (D == 1) {
        dphi = __dadd_rn(__dmul_rn(-g, pv[0]), __dmul_rn(g, pv[1]));
      } else {
        double dw[D + 1];
        Spline<D>::dweights(f, g, dw);
#pragma unroll
        for (int m = 0; m <= D; ++m) dphi = fma(dw[m], pv[m], dphi);
      }
    }
    e[rr] = dphi * (w[rr] * (wscale ? wscale[j] : 1.0));
  }
  __syncthreads();
  const double inv_mp = 2.0 * ip[I_HALFINVMP];
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    double s = 0.0;
    for (int rr = 0; rr < d; ++rr) s = fma(uxd[(size_t)rr * n + k], e[rr], s);
    out[(size_t)k * ldo + j] = inv_mp * s;
  }
}

// ---- DMMA (mma.sync m8n8k4 f64) reduced-basis F-evaluation kernels ----
//
// Same contract as rom_deposit_kernel / rom_gather_kernel, with the two
// tall-skinny products of the reduced F-evaluation on the FP64 tensor pipe:
// the reconstruct X_r = U_X Z (driver.py:69) as X^T (8 cols x 8 rows) =
// Z^T (8 x n) . U_blk^T (n x 8), and the projection U_X^T E (driver.py:85) as
// (n x 8 cols) += U_blk^T (n x 8 rows) . E (8 rows x 8 cols).  Warp w owns 8
// columns; in the X^T fragment lane (g = lane/4, t = lane%4) holds column g at
// rows 2t, 2t+1 of each 8-row block, so per-lane deposit histograms (4 copies
// per column) stay private and conflict-free.  DMMA and DFMA share the FP64
// pipe on B200 (profiles/r01b/fp64_peak.log: 37.2 vs 36.4 TF/s, 30.8 mixed):
// the gain is issue slots -- 5 DMMA per 64 units instead of 1280 DFMA.
constexpr int MW = 8;            // warps per CTA
#ifndef PICROM_GATHER_PER_SM
#define PICROM_GATHER_PER_SM 3
#endif
constexpr int kGatherMmaPerSm = PICROM_GATHER_PER_SM;   // CTAs per SM of the gather wave (3 measured best)
constexpr int MC = MW * 8;       // z columns per CTA

__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// X^T block: x0, x1 = X[rb + 2t (+1)][column g] from the staged U tile
template <int NK, bool CHECK = true>
__device__ __forceinline__ void recon_block(const double* tile, int rb, int rows, int n,
                                            const double* za, int g, int t, double& x0,
                                            double& x1) {
  x0 = 0.0;
  x1 = 0.0;
  const int ur = rb + g;
#pragma unroll
  for (int ks = 0; ks < NK; ++ks) {
    const int k = ks * 4 + t;
    const double b = !CHECK || (ur < rows && k < n) ? tile[ur * n + k] : 0.0;
    dmma_f64(x0, x1, za[ks], b);
  }
}

// Deposit: DW = 16 warps x 8 columns = 128 columns per CTA (all of C3's p in
// one column tile, so U_X is staged once).  The lanes t and t^1 of a column
// share one histogram (2 copies per column, [nh][2 DC]) and take turns (two
// predicated phases): half the smem per lane of private histograms, which
// buys 16 resident warps instead of 8 (the kernel is latency-bound).
#ifdef PICROM_DEP_LDS_RAW
#define DEP_LDS lds_f64_raw_if
#else
#define DEP_LDS lds_f64_if
#endif
constexpr int DW = 16;           // warps per deposit CTA
constexpr int DC = DW * 8;       // z columns per deposit CTA
// EX: n == 4 NK exactly (C3/C4's n = 20): the basis width is a compile-time
// constant, so the fragment bounds tests fold away and row offsets are shifts
// DWT warps per CTA: DW for wide column sets; 4 (32 columns, several CTAs per
// SM) for the few subsample columns of the hyper-reduced model (C4: p* = 20),
// where a 128-column CTA would idle 5/6 of its lanes
template <int D, int NK, bool EX, int DWT>
__global__ void __launch_bounds__(DWT * 32, DWT == DW ? 1 : 4) rom_deposit_mma_kernel(RomArgs a) {
  constexpr int DCT = DWT * 8;
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(16) double smem[];
  constexpr int NT = DWT * 32;
  constexpr int HS = DCT * 2;                  // histograms (row stride)
  const int n = EX ? 4 * NK : a.n, nx = a.nx, nh = nx + D;
  double* ut = smem;                          // [2][TR * n]
  double* hist = ut + 2 * TR * n;             // [nh][HS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int cl = warp * 8 + g;
  const int c = blockIdx.y * DCT + cl;
  const bool active = c < a.p;
  const int inst_id = active ? (a.cols ? a.cols[c] : c) : 0;
  const double* ip = a.inst + (size_t)inst_id * PICROM_INST_STRIDE;
  const double h = ip[I_H], inv_h = ip[I_INVH];
  const double inv_nx = 1.0 / (double)nx;
  const int mask = pow2_mask(nx);
  // histogram of (column, t/2): bank = 2 cl + t/2 mod 16 -- distinct over the
  // 8 lanes of one phase in each half-warp
  const unsigned int hbase = smem_u32(hist + 2 * cl + (t >> 1));
  double za[NK];
#pragma unroll
  for (int ks = 0; ks < NK; ++ks) {
    const int k = ks * 4 + t;
    // Z scaled by 1/h of the column: the reconstruct yields s = x / h directly
    za[ks] = (active && k < n) ? a.z[(size_t)k * a.ldz + c] * inv_h : 0.0;
  }
  for (int q = tid; q < nh * HS; q += NT) hist[q] = 0.0;
  const long long lo = row_start(blockIdx.x, a.N, gridDim.x);
  const long long hi = row_start(blockIdx.x + 1, a.N, gridDim.x);
  const int ntiles = (int)((hi - lo + TR - 1) / TR);
  if (ntiles > 0) stage_rows(ut, a.ux, lo, (int)min((long long)TR, hi - lo), n);
  for (int tt = 0; tt < ntiles; ++tt) {
    const long long t0 = lo + (long long)tt * TR;
    const int rows = (int)min((long long)TR, hi - t0);
    if (tt + 1 < ntiles) {
      const long long t1 = t0 + TR;
      stage_rows(ut + ((tt + 1) & 1) * TR * n, a.ux, t1, (int)min((long long)TR, hi - t1), n);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* tile = ut + (tt & 1) * TR * n;
    // RB row blocks per pass: RB independent DMMA chains, 2 RB units per lane.
    // Full tiles (all but a CTA's last) run without row / column bounds tests:
    // an inactive column (z = 0 -> x = 0) deposits into its own never-read
    // histogram, a non-finite position deposits zero weights, so the deposit
    // predicate is the lane's phase alone.
#ifndef PICROM_DEP_RB
#define PICROM_DEP_RB 2
#endif
    constexpr int RB = PICROM_DEP_RB;
    auto run_tile = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      const int nrows = FULL ? TR : rows;
      for (int rb0 = 0; rb0 < nrows; rb0 += 8 * RB) {
        double xv[2 * RB];
#pragma unroll
        for (int q = 0; q < RB; ++q)
          recon_block<NK, !(FULL && EX)>(tile, rb0 + 8 * q, rows, n, za, g, t, xv[2 * q], xv[2 * q + 1]);
        double w[2 * RB][D + 1];
        unsigned int hrow[2 * RB];
        bool act[2 * RB];
        if constexpr (FULL) {
          // straight-line common path: all elements located with no per-element
          // branch, rare inputs fixed up behind one warp vote
          int cell[2 * RB];
          double f[2 * RB];
          bool rare[2 * RB], any_rare = false;
#pragma unroll
          for (int e = 0; e < 2 * RB; ++e) {
            act[e] = true;
            locate_scaled(xv[e], mask, cell[e], f[e], rare[e]);
            any_rare |= rare[e];
          }
          if (__any_sync(0xffffffffu, any_rare)) {
#pragma unroll
            for (int e = 0; e < 2 * RB; ++e) {
              if (!(rare[e] && active)) continue;
              if (!isfinite(xv[e])) {
                record_bad(a.status, 0, t0 + rb0 + 8 * (e >> 1) + 2 * t + (e & 1), c, a.p);
                cell[e] = 0;
                f[e] = 0.0;
                act[e] = false;
              } else {
                locate_scaled_exact(xv[e], nx, inv_nx, cell[e], f[e]);
              }
            }
          }
#pragma unroll
          for (int e = 0; e < 2 * RB; ++e) {
            Spline<D>::weights(f[e], w[e]);
            if (!act[e]) {                 // non-finite position: deposits nothing
#pragma unroll
              for (int m = 0; m <= D; ++m) w[e][m] = 0.0;
            }
            hrow[e] = hbase + (unsigned int)cell[e] * (unsigned int)(HS * 8);
          }
        } else {
#pragma unroll
        for (int e = 0; e < 2 * RB; ++e) {
          const int row = rb0 + 8 * (e >> 1) + 2 * t + (e & 1);
          act[e] = active && row < rows;
          const double x = xv[e];
          int cell;
          double f;
          bool rare;
          locate_scaled(x, mask, cell, f, rare);
          if (act[e] && rare) {
            if (!isfinite(x)) {
              record_bad(a.status, 0, t0 + row, c, a.p);
              act[e] = false;
              cell = 0;
              f = 0.0;
            } else {
              locate_scaled_exact(x, nx, inv_nx, cell, f);
            }
          }
          Spline<D>::weights(f, w[e]);
          hrow[e] = hbase + (unsigned int)(act[e] ? cell : 0) * (unsigned int)(HS * 8);
        }
        }
        // lanes t = 0, 2 then t = 1, 3 (the two lanes of a histogram)
#pragma unroll
        for (int ph = 0; ph < 2; ++ph) {
#pragma unroll
          for (int e = 0; e < 2 * RB; ++e) {
            const bool on = (FULL || act[e]) && (t & 1) == ph;
            double cur[D + 1];
#pragma unroll
            for (int m = 0; m <= D; ++m) cur[m] = DEP_LDS(hrow[e] + m * HS * 8u, on);
#pragma unroll
            for (int m = 0; m <= D; ++m) sts_f64_if(hrow[e] + m * HS * 8u, cur[m] + w[e][m], on);
          }
          __syncwarp();
        }
      }
    };
    if (rows == TR) run_tile(std::true_type{});
    else run_tile(std::false_type{});
    __syncthreads();
  }
  // fold ghost rows and the 2 copies per column (fixed order) -> seg[b][c][nd];
  // consecutive threads take consecutive columns of one node (one 16-byte
  // load of both copies: conflict-free)
  const int P_used = min(DCT, a.p - blockIdx.y * DCT);
  for (int q = tid; q < P_used * nx; q += NT) {
    const int nd = q / P_used, cc = q % P_used;
    double s = 0.0;
    for (int rr = (nd - Spline<D>::OFF) % nx; rr < nh; rr += nx) {
      const double2 v = *reinterpret_cast<const double2*>(hist + rr * HS + 2 * cc);
      s += v.x + v.y;
    }
    a.seg[((size_t)blockIdx.x * a.p + blockIdx.y * DCT + cc) * nx + nd] = s;
  }
}

// MWT warps per CTA: MW, or 4 (32 columns) for the few subsample columns of the
// hyper-reduced model (see rom_deposit_mma_kernel)
template <int D, int NK, bool VPROJ, bool EX, int MWT>
__global__ void __launch_bounds__(MWT * 32, MWT == MW ? (VPROJ ? 2 : kGatherMmaPerSm) : 4) rom_gather_mma_kernel(RomArgs a) {
  constexpr int MCT = MWT * 8;
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(16) double smem[];
  constexpr int NT = MWT * 32;
  constexpr int NM = (4 * NK + 7) / 8;        // 8-row tiles of the projection (n <= 8 NM)
  constexpr int PS = MCT + 1;                  // padded phi row (bank spread)
  const int n = EX ? 4 * NK : a.n, nx = a.nx;
  double* ut = smem;                          // [2][TR * n]
  // phi with D periodic ghost rows on each side: row r holds node (r - D) mod nx,
  // so a particle's nodes cell + OFF + m need no wrap
  double* phs = ut + 2 * TR * n;              // [nx + 2D][PS]
  double* vt = phs + (nx + 6) * PS;           // [2][TR * n] U_V rows (VPROJ)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int cl = warp * 8 + g;
  const int c = blockIdx.y * MCT + cl;
  const bool active = c < a.p;
  const int P_used = min(MCT, a.p - blockIdx.y * MCT);
  for (int q = tid; q < (nx + 2 * D) * MCT; q += NT) {
    const int r = q / MCT, cc = q % MCT;
    int nd = r - D;
    nd = nd < 0 ? nd + nx : (nd >= nx ? nd - nx : nd);
    phs[r * PS + cc] = cc < P_used ? a.phi[(size_t)(blockIdx.y * MCT + cc) * nx + nd] : 0.0;
  }
  const int inst_id = active ? (a.cols ? a.cols[c] : c) : 0;
  const double* ip = a.inst + (size_t)inst_id * PICROM_INST_STRIDE;
  const double h = ip[I_H], gi = ip[I_INVH], inv_h = gi;
  const double cf = a.coef_kind == 0 ? ip[I_GCOEF] : 1.0;
  const double inv_nx = 1.0 / (double)nx;
  const int mask = pow2_mask(nx);
  // acc / accv: projections of even row blocks; acc1 / accv1: odd row blocks of
  // full tiles (two independent DMMA chains per lane), summed at the end
  double za[NK], acc[NM][2], accv[NM][2], acc1[NM][2], accv1[NM][2];
#pragma unroll
  for (int ks = 0; ks < NK; ++ks) {
    const int k = ks * 4 + t;
    // Z scaled by 1/h of the column: the reconstruct yields s = x / h directly
    za[ks] = (active && k < n) ? a.z[(size_t)k * a.ldz + c] * inv_h : 0.0;
  }
#pragma unroll
  for (int mt = 0; mt < NM; ++mt) {
    acc[mt][0] = acc[mt][1] = accv[mt][0] = accv[mt][1] = 0.0;
    acc1[mt][0] = acc1[mt][1] = accv1[mt][0] = accv1[mt][1] = 0.0;
  }
  const long long lo = row_start(blockIdx.x, a.N, gridDim.x);
  const long long hi = row_start(blockIdx.x + 1, a.N, gridDim.x);
  const int ntiles = (int)((hi - lo + TR - 1) / TR);
  // U_X (and U_V) row tiles, one cp.async group per tile
  auto stage = [&](int buf, long long r0, int rws) {
    const int chunks = rws * n / 2;
    for (int q = threadIdx.x; q < chunks; q += blockDim.x) {
      cp_async16(ut + buf * TR * n + 2 * q, a.ux + r0 * n + 2 * q);
      if constexpr (VPROJ) cp_async16(vt + buf * TR * n + 2 * q, a.uv + r0 * n + 2 * q);
    }
    cp_async_commit();
  };
  if (ntiles > 0) stage(0, lo, (int)min((long long)TR, hi - lo));
  for (int tt = 0; tt < ntiles; ++tt) {
    const long long t0 = lo + (long long)tt * TR;
    const int rows = (int)min((long long)TR, hi - t0);
    if (tt + 1 < ntiles) {
      const long long t1 = t0 + TR;
      stage((tt + 1) & 1, t1, (int)min((long long)TR, hi - t1));
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* tile = ut + (tt & 1) * TR * n;
    const double* vtile = vt + (tt & 1) * TR * n;
    // full tiles (all but a CTA's last) run without row bounds tests; with an
    // exact basis width (EX) no fragment test remains in the reconstruct
    auto run_tile = [&](auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
    const int nrows = FULL ? TR : rows;
    // field (and optional harvest) of one located element; cfe = the column's
    // coefficient, or 0 for an element that must contribute nothing
    auto eval_at = [&](int cell, double f, double cfe, long long i, bool store) {
      double pv[D + 1];
      const double* pc = phs + (cell + Spline<D>::OFF + D) * PS + cl;
#pragma unroll
      for (int m = 0; m <= D; ++m) pv[m] = pc[m * PS];
      double E;
      if constexpr (D == 1) {   // coef * ((-g)*phi0 + g*phi1): driver.py:74-75 order
        E = __dmul_rn(cfe, __dadd_rn(__dmul_rn(-gi, pv[0]), __dmul_rn(gi, pv[1])));
      } else {
        double dw[D + 1];
        Spline<D>::dweights(f, gi, dw);
        double sacc = 0.0;
#pragma unroll
        for (int m = 0; m <= D; ++m) sacc = fma(dw[m], pv[m], sacc);
        E = cfe * sacc;
      }
      if (store && a.eout) a.eout[(size_t)i * a.ldo + c] = E;
      if (store && a.lam) {
        double lv;
        if constexpr (D == 1) {
          lv = __dadd_rn(__dmul_rn(__dsub_rn(1.0, f), pv[0]), __dmul_rn(f, pv[1]));
        } else {
          double w[D + 1];
          Spline<D>::weights(f, w);
          lv = 0.0;
#pragma unroll
          for (int m = 0; m <= D; ++m) lv = fma(w[m], pv[m], lv);
        }
        a.lam[(size_t)i * a.ldo + c] = lv;
      }
      return E;
    };
    // projection of one row block: accp (basis m = 8 mt + g, columns 2t, 2t+1)
    // += U_blk^T E_blk; B fragment E[rb + 4 ks + t][column g] lives in lane
    // 4 g + 2 ks + t/2
    auto project = [&](int rb, const double* ev, double (*accp)[2], double (*accvp)[2]) {
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int src = g * 4 + 2 * ks + (t >> 1);
        const double s0 = __shfl_sync(0xffffffffu, ev[0], src);
        const double s1 = __shfl_sync(0xffffffffu, ev[1], src);
        const double b = (t & 1) ? s1 : s0;
        const int ur = rb + 4 * ks + t;
#pragma unroll
        for (int mt = 0; mt < NM; ++mt) {
          const int m = mt * 8 + g;
          const double av = ((FULL || ur < rows) && m < n) ? tile[ur * n + m] : 0.0;
          dmma_f64(accp[mt][0], accp[mt][1], av, b);
        }
        if constexpr (VPROJ) {
#pragma unroll
          for (int mt = 0; mt < NM; ++mt) {
            const int m = mt * 8 + g;
            const double av = ((FULL || ur < rows) && m < n) ? vtile[ur * n + m] : 0.0;
            dmma_f64(accvp[mt][0], accvp[mt][1], av, b);
          }
        }
      }
    };
    if constexpr (FULL) {
      // two row blocks per pass: two independent reconstruct chains and two
      // accumulator sets; straight-line common path (all four elements located
      // and evaluated with no per-element branch), rare inputs fixed up behind
      // one warp vote.  An inactive column (z = 0 -> x = 0) reads its
      // zero-filled phi column.
      static_assert(TR % 16 == 0, "full tiles are walked two row blocks at a time");
      for (int rb = 0; rb < TR; rb += 16) {
        double xv[4], ev[4];
        recon_block<NK, !EX>(tile, rb, rows, n, za, g, t, xv[0], xv[1]);
        recon_block<NK, !EX>(tile, rb + 8, rows, n, za, g, t, xv[2], xv[3]);
        int cell[4];
        double f[4], cfe[4] = {cf, cf, cf, cf};
        bool rare[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) locate_scaled(xv[e], mask, cell[e], f[e], rare[e]);
        if (__any_sync(0xffffffffu, (rare[0] || rare[1]) || (rare[2] || rare[3]))) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (!(rare[e] && active)) continue;
            if (!isfinite(xv[e])) {
              record_bad(a.status, 0, t0 + rb + 8 * (e >> 1) + 2 * t + (e & 1), c, a.p);
              cell[e] = 0;
              f[e] = 0.0;
              cfe[e] = 0.0;
            } else {
              locate_scaled_exact(xv[e], nx, inv_nx, cell[e], f[e]);
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
          ev[e] = eval_at(cell[e], f[e], cfe[e], t0 + rb + 8 * (e >> 1) + 2 * t + (e & 1), active);
        project(rb, ev, acc, accv);
        project(rb + 8, ev + 2, acc1, accv1);
      }
    } else {
    for (int rb = 0; rb < nrows; rb += 8) {
      double xv[2], ev[2];
      recon_block<NK, true>(tile, rb, rows, n, za, g, t, xv[0], xv[1]);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        ev[e] = 0.0;
        const int row = rb + 2 * t + e;
        if (!active || row >= rows) continue;
        const double x = xv[e];
        const long long i = t0 + row;
        int cell;
        double f;
        bool rare;
        locate_scaled(x, mask, cell, f, rare);
        if (rare) {
          if (!isfinite(x)) {
            record_bad(a.status, 0, i, c, a.p);
            continue;
          }
          locate_scaled_exact(x, nx, inv_nx, cell, f);
        }
        ev[e] = eval_at(cell, f, cf, i, true);
      }
      project(rb, ev, acc, accv);
    }
    }
    };
    if (rows == TR) run_tile(std::true_type{});
    else run_tile(std::false_type{});
    __syncthreads();
  }
  // per-CTA partials seg[b][c][k]: lane holds basis m = 8 mt + g at columns 2t, 2t+1
#pragma unroll
  for (int mt = 0; mt < NM; ++mt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int m = mt * 8 + g;
      const int col = blockIdx.y * MCT + warp * 8 + 2 * t + e;
      if (m < n && col < a.p) {
        a.seg[((size_t)blockIdx.x * a.p + col) * n + m] = acc[mt][e] + acc1[mt][e];
        if constexpr (VPROJ) a.seg2[((size_t)blockIdx.x * a.p + col) * n + m] = accv[mt][e] + accv1[mt][e];
      }
    }
}

int gram_grid(long long N) {
  long long g = std::min<long long>(2LL * picrom_num_sms(), std::max<long long>(1, N / 256));
  return (int)g;
}

int rom_grid(long long N) {
  long long g = std::min<long long>((long long)picrom_num_sms(), std::max<long long>(1, N / 64));
  return (int)g;
}

// DMMA path row blocks: one wave of `per_sm` CTAs per SM over the column tiles
int rom_grid_mma(long long N, int p, int per_sm) {
  const int tiles = (p + MC - 1) / MC;
  long long g = std::max(1LL, (long long)picrom_num_sms() * per_sm / tiles);
  return (int)std::min<long long>(g, std::max<long long>(1, N / 64));
}

// kernel-path switches are compile time only (tools/build_variant.py -D...),
// never environment-dependent: the DMMA F-evaluation kernels are the default
bool rom_use_mma() { return !kNoRomMma; }

}  // namespace

// ------------------------------------------------------------------ C-ABI

// ---- DMMA combine: out (N x c) (+)= sum_t op(in_t) M_t ----
//
// K = sum a_t (the terms' columns back to back) is the GEMM depth.  M (K x c)
// sits in smem with pitch cp; the inputs stream through two cp.async stages
// of 64 rows, term t at pitch pa_t (pa_t = 4 or 12 mod 16 doubles: the 8 x 4
// A fragments then hit two wavefronts).  Warp w owns the 8-row tile w of a
// stage; the J sign of a swapped term is applied at the fragment load.
constexpr int CMR = 64;   // rows per stage

struct MmaTerms {
  int koff[MAXTERM + 1];  // first GEMM row of term t in M
  int soff[MAXTERM + 1];  // offset of term t in a stage (doubles per row of the stage)
  int pa[MAXTERM];        // smem pitch of term t
  int cp;                 // smem pitch of M
};

__device__ __forceinline__ void cp_async16z(void* smem_dst, const void* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}

template <int TBO>
__global__ void __launch_bounds__(256, 2)
combine_mma_kernel(Terms t, MmaTerms mt, const double* mats, long long N) {
  extern __shared__ __align__(16) double csm[];
  const int K = mt.koff[t.nt];
  const int cp = mt.cp;
  double* ms = csm;                                   // [K + 4][cp] (+ 8 pad)
  double* stg = ms + (size_t)(K + 4) * cp + 8;        // [2][CMR * soff[nt]]
  const int SZ = CMR * mt.soff[t.nt];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = t.c;
  for (int q = tid; q < (K + 4) * cp + 8; q += blockDim.x) {
    const int k = q / cp, j = q - k * cp;
    double v = 0.0;
    if (k < K && j < c) {
      int ti = 0;
      while (k >= mt.koff[ti + 1]) ++ti;
      v = mats[t.moff[ti] + (k - mt.koff[ti]) * c + j];
    }
    ms[q] = v;
  }
  const long long half = N / 2;
  const long long lo = row_start(blockIdx.x, N, gridDim.x);
  const long long hi = row_start(blockIdx.x + 1, N, gridDim.x);
  const int nst = (int)((hi - lo + CMR - 1) / CMR);
  auto stage = [&](int st) {
    const long long r0 = lo + (long long)st * CMR;
    const int rows = (int)min((long long)CMR, hi - r0);
    double* dst = stg + (st & 1) * SZ;
    for (int ti = 0; ti < t.nt; ++ti) {
      const int ch = t.a[ti] >> 1;                    // 16-B chunks per row
      double* d = dst + CMR * mt.soff[ti];
      for (int q = tid; q < rows * ch; q += blockDim.x) {
        const int rr = q / ch, k2 = q - rr * ch;
        long long row = r0 + rr;
        if (t.jswap[ti]) row = row < half ? row + half : row - half;
        cp_async16z(d + rr * mt.pa[ti] + 2 * k2, t.in[ti] + (size_t)row * t.ld[ti] + 2 * k2);
      }
    }
    cp_async_commit();
  };
  const int lr = lane >> 2, lk = lane & 3;
  if (nst > 0) stage(0);
  for (int st = 0; st < nst; ++st) {
    const long long r0 = lo + (long long)st * CMR;
    const int rows = (int)min((long long)CMR, hi - r0);
    if (st + 1 < nst) { stage(st + 1); cp_async_wait<1>(); } else { cp_async_wait<0>(); }
    __syncthreads();
    const double* cur = stg + (st & 1) * SZ;
    const int r = warp * 8 + lr;                      // A-fragment row of this lane
    if (warp * 8 < rows) {
      double acc[TBO][2];
#pragma unroll
      for (int j = 0; j < TBO; ++j) acc[j][0] = acc[j][1] = 0.0;
      const bool rv = r < rows;
      for (int ti = 0; ti < t.nt; ++ti) {
        const double sg = (t.jswap[ti] && r0 + r >= half) ? -1.0 : 1.0;
        const double* arow = cur + CMR * mt.soff[ti] + r * mt.pa[ti];
        const double* mrow = ms + (size_t)mt.koff[ti] * cp + lr;
        const int a = t.a[ti];
        for (int k0 = 0; k0 < a; k0 += 4) {
          const int kk = k0 + lk;
          const double av = (rv && kk < a) ? sg * arow[kk] : 0.0;
          const double* mk = mrow + (size_t)kk * cp;
#pragma unroll
          for (int j = 0; j < TBO; ++j) dmma(acc[j][0], acc[j][1], av, mk[8 * j]);
        }
      }
      if (rv) {
        double* orow = t.out + (size_t)(r0 + r) * t.ldo;
#pragma unroll
        for (int j = 0; j < TBO; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 8 * j + 2 * lk + e;
            if (col < c) orow[col] = t.accumulate ? orow[col] + acc[j][e] : acc[j][e];
          }
      }
    }
    __syncthreads();
  }
}

extern "C" size_t picrom_rom_workspace_bytes(long long N, int p, int n, int nx) {
  size_t G = (size_t)std::max(rom_grid(N), rom_grid_mma(N, p, kGatherMmaPerSm));
  G = std::max(G, (size_t)picrom_num_sms() * 4);      // narrow-deposit grid (kDepNarrowPerSm)
  const size_t dep = G * p * nx;
  const size_t gat = 2 * G * p * n;        // U_X^T E and U_V^T E partials
  const size_t gram = (size_t)gram_grid(N) * 256 * 256;
  return std::max(std::max(dep, gat), gram) * sizeof(double) + 256;
}

// Row groups R (threads = R x P): as many as the per-column histograms
// (deposit) or phi + partials (gather) leave room for, up to 384 threads
// (one CTA per SM, 12 warps at C3); measured latency-bound, so warps matter.
template <int D, int NB>
static int launch_rom_deposit_nb(const RomArgs& a, int G, cudaStream_t s) {
  const int tiles = (a.p + PT - 1) / PT;
  const int P = std::min(PT, ((std::min(a.p, PT) + 31) / 32) * 32);
  int R = std::max(1, std::min(384 / P, 4));
  auto smem = [&](int rr) {
    return (size_t)2 * TR * a.n * sizeof(double) + (size_t)(a.nx + D) * (rr * P) * sizeof(double);
  };
  while (R > 1 && smem(R) > 220 * 1024) --R;
  if (smem(R) > 227 * 1024) return picrom_set_error(PICROM_ERR_CONFIG, "rom deposit: nx too large");
  dim3 grid(G, tiles);
  switch (R) {
    case 1: rom_allow_smem(rom_deposit_kernel<D, NB, 1>); rom_deposit_kernel<D, NB, 1><<<grid, P, smem(1), s>>>(a); break;
    case 2: rom_allow_smem(rom_deposit_kernel<D, NB, 2>); rom_deposit_kernel<D, NB, 2><<<grid, 2 * P, smem(2), s>>>(a); break;
    case 3: rom_allow_smem(rom_deposit_kernel<D, NB, 3>); rom_deposit_kernel<D, NB, 3><<<grid, 3 * P, smem(3), s>>>(a); break;
    default: rom_allow_smem(rom_deposit_kernel<D, NB, 4>); rom_deposit_kernel<D, NB, 4><<<grid, 4 * P, smem(4), s>>>(a); break;
  }
  return picrom_check_launch("rom_deposit_kernel");
}

template <int D, int NB>
static int launch_rom_gather_nb(const RomArgs& a, int G, cudaStream_t s) {
  const int tiles = (a.p + PT - 1) / PT;
  const int P = std::min(PT, ((std::min(a.p, PT) + 31) / 32) * 32);
  int R = std::max(1, std::min(384 / P, 4));
  auto smem = [&](int rr) {
    return ((size_t)2 * TR * a.n + (size_t)a.nx * P + (size_t)rr * P * a.n) * sizeof(double);
  };
  while (R > 1 && smem(R) > 220 * 1024) --R;
  const size_t sm = smem(R);
  if (sm > 227 * 1024) return picrom_set_error(PICROM_ERR_CONFIG, "rom gather: nx too large");
  dim3 grid(G, tiles);
  switch (R) {
    case 1: rom_allow_smem(rom_gather_kernel<D, NB, 1>); rom_gather_kernel<D, NB, 1><<<grid, P, sm, s>>>(a); break;
    case 2: rom_allow_smem(rom_gather_kernel<D, NB, 2>); rom_gather_kernel<D, NB, 2><<<grid, 2 * P, sm, s>>>(a); break;
    case 3: rom_allow_smem(rom_gather_kernel<D, NB, 3>); rom_gather_kernel<D, NB, 3><<<grid, 3 * P, sm, s>>>(a); break;
    default: rom_allow_smem(rom_gather_kernel<D, NB, 4>); rom_gather_kernel<D, NB, 4><<<grid, 4 * P, sm, s>>>(a); break;
  }
  return picrom_check_launch("rom_gather_kernel");
}

// basis dimension -> register block size (n <= NB, even)
#define ROM_NB_DISPATCH(FN, D, A, G, S)                       \
  (A.n <= 4 ? FN<D, 4>(A, G, S) : A.n <= 8 ? FN<D, 8>(A, G, S) :  \
   A.n <= 12 ? FN<D, 12>(A, G, S) : A.n <= 16 ? FN<D, 16>(A, G, S) : \
   A.n <= 20 ? FN<D, 20>(A, G, S) : A.n <= 24 ? FN<D, 24>(A, G, S) : FN<D, 32>(A, G, S))

template <int D>
static int launch_rom_deposit(const RomArgs& a, int G, cudaStream_t s) {
  return ROM_NB_DISPATCH(launch_rom_deposit_nb, D, a, G, s);
}

template <int D>
static int launch_rom_gather(const RomArgs& a, int G, cudaStream_t s) {
  return ROM_NB_DISPATCH(launch_rom_gather_nb, D, a, G, s);
}

// DMMA path: k-steps NK = ceil(n / 4) rounded up to {2, 4, 5, 8}
static int mma_nk(int n) { return n <= 8 ? 2 : n <= 16 ? 4 : n <= 20 ? 5 : 8; }
static size_t mma_dep_smem(int n, int nx, int D, int dwt = DW) {
  return ((size_t)2 * TR * n + (size_t)(nx + D) * dwt * 8 * 2) * sizeof(double);
}
// few columns (the hyper-reduced model's subsample): 4-warp deposit CTAs, 4 per SM
constexpr int kDepNarrowCols = 32;
constexpr int kDepNarrowPerSm = 4;
static size_t mma_gat_smem(int n, int nx, bool vproj = false, int mwt = MW) {
  return ((size_t)(vproj ? 4 : 2) * TR * n + (size_t)(nx + 6) * (mwt * 8 + 1)) * sizeof(double);
}

template <int D, int NK, bool EX>
static int launch_dep_mma_e(const RomArgs& a, int G, cudaStream_t s) {
  if (a.p <= kDepNarrowCols) {
    auto kfn = rom_deposit_mma_kernel<D, NK, EX, 4>;
    static bool attr = false;
    if (!attr) { rom_allow_smem(kfn); attr = true; }
    kfn<<<dim3(G, 1), 4 * 32, mma_dep_smem(a.n, a.nx, D, 4), s>>>(a);
    return picrom_check_launch("rom_deposit_mma_kernel");
  }
  auto kfn = rom_deposit_mma_kernel<D, NK, EX, DW>;
  static bool attr = false;
  if (!attr) { rom_allow_smem(kfn); attr = true; }
  kfn<<<dim3(G, (a.p + DC - 1) / DC), DW * 32, mma_dep_smem(a.n, a.nx, D), s>>>(a);
  return picrom_check_launch("rom_deposit_mma_kernel");
}
template <int D, int NK>
static int launch_dep_mma_t(const RomArgs& a, int G, cudaStream_t s) {
  return a.n == 4 * NK ? launch_dep_mma_e<D, NK, true>(a, G, s)
                       : launch_dep_mma_e<D, NK, false>(a, G, s);
}
template <int D, int NK, bool VPROJ, bool EX>
static int launch_gat_mma_e(const RomArgs& a, int G, cudaStream_t s) {
  if (a.p <= kDepNarrowCols) {
    auto kfn = rom_gather_mma_kernel<D, NK, VPROJ, EX, 4>;
    static bool attr = false;
    if (!attr) { rom_allow_smem(kfn); attr = true; }
    kfn<<<dim3(G, 1), 4 * 32, mma_gat_smem(a.n, a.nx, VPROJ, 4), s>>>(a);
    return picrom_check_launch("rom_gather_mma_kernel");
  }
  const dim3 grid(G, (a.p + MC - 1) / MC);
  auto kfn = rom_gather_mma_kernel<D, NK, VPROJ, EX, MW>;
  static bool attr = false;
  if (!attr) { rom_allow_smem(kfn); attr = true; }
  kfn<<<grid, MW * 32, mma_gat_smem(a.n, a.nx, VPROJ), s>>>(a);
  return picrom_check_launch("rom_gather_mma_kernel");
}
template <int D, int NK>
static int launch_gat_mma_t(const RomArgs& a, int G, cudaStream_t s) {
  const bool ex = a.n == 4 * NK;
  if (a.uv) return ex ? launch_gat_mma_e<D, NK, true, true>(a, G, s)
                      : launch_gat_mma_e<D, NK, true, false>(a, G, s);
  return ex ? launch_gat_mma_e<D, NK, false, true>(a, G, s)
            : launch_gat_mma_e<D, NK, false, false>(a, G, s);
}
#define ROM_NK_DISPATCH(FN, D, A, G, S)                                              \
  (mma_nk(A.n) == 2 ? FN<D, 2>(A, G, S) : mma_nk(A.n) == 4 ? FN<D, 4>(A, G, S) :     \
   mma_nk(A.n) == 5 ? FN<D, 5>(A, G, S) : FN<D, 8>(A, G, S))

// row blocks of the deposit for this call (DMMA: one CTA per SM), 0 = old path
template <int D>
static int rom_dep_grid(const RomArgs& a) {
  if (!rom_use_mma() || mma_dep_smem(a.n, a.nx, D) > 220 * 1024) return rom_grid(a.N);
  if (a.p <= kDepNarrowCols)
    return (int)std::min<long long>((long long)picrom_num_sms() * kDepNarrowPerSm, std::max<long long>(1, a.N / 64));
  const int tiles = (a.p + DC - 1) / DC;
  return (int)std::min<long long>(std::max(1, picrom_num_sms() / tiles), std::max<long long>(1, a.N / 64));
}
template <int D>
static int launch_rom_deposit_any(const RomArgs& a, int G, cudaStream_t s) {
  if (!rom_use_mma() || mma_dep_smem(a.n, a.nx, D) > 220 * 1024) return launch_rom_deposit<D>(a, G, s);
  return ROM_NK_DISPATCH(launch_dep_mma_t, D, a, G, s);
}
static int rom_gat_grid(const RomArgs& a) {
  if (rom_use_mma() && a.p <= kDepNarrowCols)     // 4-warp CTAs, 4 per SM
    return (int)std::min<long long>((long long)picrom_num_sms() * kDepNarrowPerSm, std::max<long long>(1, a.N / 64));
  if (a.uv) return rom_grid_mma(a.N, a.p, 2);     // 94 registers: 2 CTAs per SM
  if (!rom_use_mma() || mma_gat_smem(a.n, a.nx) > 200 * 1024) return rom_grid(a.N);
  return rom_grid_mma(a.N, a.p, kGatherMmaPerSm);
}
template <int D>
static int launch_rom_gather_any(const RomArgs& a, int G, cudaStream_t s) {
  if (a.uv) {   // the U_V projection exists only on the DMMA path
    if (mma_gat_smem(a.n, a.nx, true) > 200 * 1024)
      return picrom_set_error(PICROM_ERR_CONFIG, "rom gather: nx too large for the U_V projection");
    return ROM_NK_DISPATCH(launch_gat_mma_t, D, a, G, s);
  }
  if (!rom_use_mma() || mma_gat_smem(a.n, a.nx) > 200 * 1024) return launch_rom_gather<D>(a, G, s);
  return ROM_NK_DISPATCH(launch_gat_mma_t, D, a, G, s);
}

static int rom_check(long long N, int n, int p, int nx, int degree) {
  if (N < 1 || p < 1) return picrom_set_error(PICROM_ERR_CONFIG, "need N >= 1 and p >= 1");
  if (n < 2 || n > NMAX || (n & 1)) return picrom_set_error(PICROM_ERR_CONFIG, "basis dimension must be even, in [2, 32]");
  if (degree < 1 || degree > 3) return picrom_set_error(PICROM_ERR_CONFIG, "degree must be 1, 2 or 3");
  if (nx < 2) return picrom_set_error(PICROM_ERR_CONFIG, "need nx >= 2");
  return PICROM_OK;
}

// exact_gradients' field half (driver.py:70-73): rho, phi (p', nx) and the field
// energy of the reconstructed positions X_r = U_X Z, one solve per column.
extern "C" int picrom_rom_field(const double* ux, long long N, int n, const double* z, int ldz,
                                int p, const int* cols, const double* inst, int nx, int degree,
                                const double* khat, const double* stencil, double* phi,
                                double* rho, double* energy, void* ws,
                                unsigned long long* status, const long long* skip, void* stream) {
  int rc = rom_check(N, n, p, nx, degree);
  if (rc) return rc;
  RomArgs a{};
  a.ux = ux; a.z = z; a.inst = inst; a.cols = cols; a.seg = (double*)ws; a.N = N; a.n = n;
  a.p = p; a.ldz = ldz; a.nx = nx; a.status = status; a.skip = skip;
  const int G = degree == 1 ? rom_dep_grid<1>(a) : degree == 2 ? rom_dep_grid<2>(a) : rom_dep_grid<3>(a);
  cudaStream_t s = (cudaStream_t)stream;
  switch (degree) {
    case 1: rc = launch_rom_deposit_any<1>(a, G, s); break;
    case 2: rc = launch_rom_deposit_any<2>(a, G, s); break;
    default: rc = launch_rom_deposit_any<3>(a, G, s); break;
  }
  if (rc) return rc;
  return picrom_solve_dense(a.seg, G, p, nx, degree, cols, inst, khat, stencil, phi, rho, energy, s,
                            skip);
}

// Gather + projection: g_out (n x p', ld ldg) = U_X^T E with E = coef d/dx
// (phi . lambda)(U_X Z); lam/eout optional (p', ldo).
static int rom_gather_impl(const double* ux, long long N, int n, const double* z, int ldz, int p,
                           const int* cols, const double* inst, int nx, int degree,
                           const double* phi, int coef_kind, double* g_out, int ldg,
                           double* gv_out, double* lam, double* eout, long long ldo, void* ws,
                           unsigned long long* status, void* stream,
                           const long long* skip = nullptr) {
  int rc = rom_check(N, n, p, nx, degree);
  if (rc) return rc;
  RomArgs a{};
  a.ux = ux; a.z = z; a.inst = inst; a.cols = cols; a.phi = phi; a.seg = (double*)ws;
  a.lam = lam; a.eout = eout; a.N = N; a.ldo = ldo; a.n = n; a.p = p; a.ldz = ldz; a.nx = nx;
  a.coef_kind = coef_kind; a.status = status; a.skip = skip;
  const int G = rom_gat_grid(a);
  if (gv_out) {
    a.uv = ux + (size_t)N * n;
    a.seg2 = a.seg + (size_t)G * p * n;
  }
  cudaStream_t s = (cudaStream_t)stream;
  switch (degree) {
    case 1: rc = launch_rom_gather_any<1>(a, G, s); break;
    case 2: rc = launch_rom_gather_any<2>(a, G, s); break;
    default: rc = launch_rom_gather_any<3>(a, G, s); break;
  }
  if (rc) return rc;
  const int rows = p * n;
  if (g_out) {
    seg_sum_kernel<<<(rows + SEGQ - 1) / SEGQ, 256, 0, s>>>(a.seg, G, rows, g_out, ldg, 1, n, a.skip);
    rc = picrom_check_launch("seg_sum");
    if (rc) return rc;
  }
  if (gv_out) {
    seg_sum_kernel<<<(rows + SEGQ - 1) / SEGQ, 256, 0, s>>>(a.seg2, G, rows, gv_out, ldg, 1, n, a.skip);
    rc = picrom_check_launch("seg_sum");
  }
  return rc;
}

extern "C" int picrom_rom_gather(const double* ux, long long N, int n, const double* z, int ldz,
                                 int p, const int* cols, const double* inst, int nx, int degree,
                                 const double* phi, int coef_kind, double* g_out, int ldg,
                                 double* lam, double* eout, long long ldo, void* ws,
                                 unsigned long long* status, const long long* skip,
                                 void* stream) {
  return rom_gather_impl(ux, N, n, z, ldz, p, cols, inst, nx, degree, phi, coef_kind, g_out, ldg,
                         nullptr, lam, eout, ldo, ws, status, stream, skip);
}

// Gather with both projections of E: g_out = U_X^T E and gv_out = U_V^T E
// (n x p', ld ldg), U = ux the full (2N x n) basis; used by exact_gradients so
// the basis velocity's U^T G Z^T products need no pass over G (reduction.py:148-153).
extern "C" int picrom_rom_gather_uv(const double* u, long long N, int n, const double* z,
                                    int ldz, int p, const int* cols, const double* inst, int nx,
                                    int degree, const double* phi, int coef_kind, double* g_out,
                                    double* gv_out, int ldg, double* lam, double* eout,
                                    long long ldo, void* ws, unsigned long long* status,
                                    void* stream) {
  if (!g_out || !gv_out) return picrom_set_error(PICROM_ERR_CONFIG, "rom_gather_uv: need g_out and gv_out");
  return rom_gather_impl(u, N, n, z, ldz, p, cols, inst, nx, degree, phi, coef_kind, g_out, ldg,
                         gv_out, lam, eout, ldo, ws, status, stream);
}

// Gram of the row-concatenation W = [B_0 | B_1 | ...] (N rows): out (w x w).
// DMMA fast path of gram_impl: equal block widths <= 32, row-contiguous,
// 16-B aligned, at least 1024 rows.  Returns -1 when not applicable.
template <int TB, int TPC>
static int launch_gram_mma(const Blocks& b, const GramTasks& tk, int na, long long N, int wdt,
                           void* ws, cudaStream_t s, int* gy_out) {
  const int ngroups = (tk.ntask + TPC - 1) / TPC;
  int wn = 0;                       // widest needed set over the groups
  for (int g = 0; g < ngroups; ++g) {
    unsigned need = 0;
    for (int t = g * TPC; t < std::min(tk.ntask, (g + 1) * TPC); ++t)
      need |= (1u << tk.bi[t]) | (1u << tk.bj[t]);
    wn = std::max(wn, __builtin_popcount(need) * wdt);
  }
  int GT = (40 * 1024 / (wn * 8)) / 32 * 32;
  GT = std::max(32, std::min(256, GT));
  const size_t sm = (size_t)2 * GT * wn * sizeof(double) + 2 * sizeof(uint64_t) +
                    (size_t)TPC * TB * TB * 64 * sizeof(double);
  const int gy = std::max(1, std::min(gram_grid(N), (4 * picrom_num_sms()) / ngroups));
  static bool attr = false;
  if (!attr) { rom_allow_smem(gram_mma_kernel<TB, TPC>); attr = true; }
  gram_mma_kernel<TB, TPC><<<dim3(ngroups, gy), 256, sm, s>>>(b, tk, na, N, GT, wn, (double*)ws);
  *gy_out = gy;
  return picrom_check_launch("gram_mma_kernel");
}

static int gram_mma_try(const Blocks& b, int na, long long N, void* ws, cudaStream_t s,
                        double* out, const GramTasks* tasks = nullptr) {
  if (kNoGramMma || N < 1024) return -1;
  const int wdt = b.w[0];
  if (wdt > 32 || wdt < 2 || (wdt & 1)) return -1;
  for (int i = 0; i < b.nb; ++i)
    if (b.w[i] != wdt || b.ld[i] != wdt || (reinterpret_cast<uintptr_t>(b.ptr[i]) & 15)) return -1;
  GramTasks tk{};
  if (tasks) {
    tk = *tasks;
  } else if (na == 0) {
    for (int i = 0; i < b.nb; ++i)
      for (int j = i; j < b.nb; ++j) { tk.bi[tk.ntask] = (unsigned char)i; tk.bj[tk.ntask] = (unsigned char)j; ++tk.ntask; }
  } else {
    for (int i = 0; i < na; ++i)
      for (int j = na; j < b.nb; ++j) { tk.bi[tk.ntask] = (unsigned char)i; tk.bj[tk.ntask] = (unsigned char)j; ++tk.ntask; }
  }
  const int TBv = (wdt + 7) / 8;
  int gy = 0, rc;
  switch (TBv) {
    case 1: rc = launch_gram_mma<1, 8>(b, tk, na, N, wdt, ws, s, &gy); break;
    case 2: rc = launch_gram_mma<2, 4>(b, tk, na, N, wdt, ws, s, &gy); break;
    case 3: rc = launch_gram_mma<3, 2>(b, tk, na, N, wdt, ws, s, &gy); break;
    default: rc = launch_gram_mma<4, 1>(b, tk, na, N, wdt, ws, s, &gy); break;
  }
  if (rc) return rc;
  const int W = b.off[b.nb];
  const int wa = na > 0 ? b.off[na] : W, wb = na > 0 ? W - b.off[na] : W;
  const int rows = wa * wb;
  seg_sum_kernel<<<(rows + SEGQ - 1) / SEGQ, 256, 0, s>>>((const double*)ws, gy, rows, out, 0, 0, 1);
  return picrom_check_launch("seg_sum");
}

static int gram_impl(int nblocks, int na, const double* const* ptrs, const int* lds,
                     const int* widths, const int* jswap, long long N, double* out, void* ws,
                     void* stream) {
  if (nblocks < 1 || nblocks > MAXB) return picrom_set_error(PICROM_ERR_CONFIG, "1..8 blocks");
  Blocks b{};
  b.nb = nblocks;
  b.off[0] = 0;
  for (int i = 0; i < nblocks; ++i) {
    b.ptr[i] = ptrs[i]; b.ld[i] = lds[i]; b.w[i] = widths[i];
    b.jswap[i] = jswap ? jswap[i] : 0;
    b.off[i + 1] = b.off[i] + widths[i];
  }
  const int W = b.off[nblocks];
  const int wa = na > 0 ? b.off[na] : W, wb = na > 0 ? W - b.off[na] : W;
  const int G = gram_grid(N);
  cudaStream_t s = (cudaStream_t)stream;
  {
    int rc = gram_mma_try(b, na, N, ws, s, out);
    if (rc != -1) return rc;
  }
  if (W > 256 || ((wa + TB - 1) / TB) * ((wb + TB - 1) / TB) > 4 * 256)
    return picrom_set_error(PICROM_ERR_CONFIG, "Gram: total width <= 256 and wa*wb <= 16384");
  const size_t sm = (size_t)2 * GTR * W * sizeof(double) + (size_t)W * (sizeof(void*) + 2 * sizeof(int));
  // TMA staging when every block is row-contiguous (ld == width) and 16-B aligned
  bool tma = !kNoGramTma;
  for (int i = 0; i < nblocks && tma; ++i)
    tma = lds[i] == widths[i] && ((widths[i] * 8) % 16 == 0) &&
          ((reinterpret_cast<uintptr_t>(ptrs[i]) & 15) == 0);
  const size_t sm_tma = (size_t)2 * GT2 * W * sizeof(double) + 2 * sizeof(uint64_t);
  if (tma && sm_tma > 200 * 1024) tma = false;
  // 8x8 register tiles when the output has <= 256 of them, else 4x4
  const int t8 = ((wa + 7) / 8) * ((wb + 7) / 8);
  int RG;
  if (tma) {
    if (t8 <= 256) {
      RG = t8 >= 256 ? 1 : 256 / t8;
      rom_allow_smem(gram_tma_kernel<8, 1>);
      gram_tma_kernel<8, 1><<<G, 256, sm_tma, s>>>(b, na, N, (double*)ws);
    } else {
      const int t4 = ((wa + 3) / 4) * ((wb + 3) / 4);
      RG = t4 >= 256 ? 1 : 256 / t4;
      rom_allow_smem(gram_tma_kernel<4, 4>);
      gram_tma_kernel<4, 4><<<G, 256, sm_tma, s>>>(b, na, N, (double*)ws);
    }
  } else if (t8 <= 256) {
    RG = t8 >= 256 ? 1 : 256 / t8;
    rom_allow_smem(gram_kernel<8, 1>);
    gram_kernel<8, 1><<<G, 256, sm, s>>>(b, na, N, (double*)ws);
  } else {
    const int t4 = ((wa + 3) / 4) * ((wb + 3) / 4);
    RG = t4 >= 256 ? 1 : 256 / t4;
    rom_allow_smem(gram_kernel<4, 4>);
    gram_kernel<4, 4><<<G, 256, sm, s>>>(b, na, N, (double*)ws);
  }
  int rc = picrom_check_launch("gram_kernel");
  if (rc) return rc;
  const int rows = wa * wb;
  const int Gp = G * RG;
  seg_sum_kernel<<<(rows + SEGQ - 1) / SEGQ, 256, 0, s>>>((const double*)ws, Gp, rows, out, 0, 0, 1);
  return picrom_check_launch("seg_sum");
}

extern "C" int picrom_paired_gram(int nblocks, const double* const* ptrs, const int* lds,
                                  const int* widths, const int* jswap, long long N, double* out,
                                  void* ws, void* stream) {
  return gram_impl(nblocks, 0, ptrs, lds, widths, jswap, N, out, ws, stream);
}

// out (wa x wb) = A^T B, A = blocks [0, na), B = blocks [na, nblocks)
extern "C" int picrom_cross_gram(int nblocks, int na, const double* const* ptrs, const int* lds,
                                 const int* widths, const int* jswap, long long N, double* out,
                                 void* ws, void* stream) {
  if (na < 1 || na >= nblocks) return picrom_set_error(PICROM_ERR_CONFIG, "cross Gram needs 1 <= na < nblocks");
  return gram_impl(nblocks, na, ptrs, lds, widths, jswap, N, out, ws, stream);
}

// Selected blocks of the Gram W^T W: out (w x w) holds B_bi[t]^T B_bj[t] at
// block (bi[t], bj[t]) for each task t; the other entries are unspecified.
// Only the requested products are computed (tangent_velocity needs 7 of the
// 10 block pairs of [U, xi, r, x_eval], reduction.py:170-182).
extern "C" int picrom_gram_tasks(int nblocks, const double* const* ptrs, const int* lds,
                                 const int* widths, const int* jswap, int ntask, const int* bi,
                                 const int* bj, long long N, double* out, void* ws, void* stream) {
  if (nblocks < 1 || nblocks > MAXB) return picrom_set_error(PICROM_ERR_CONFIG, "1..8 blocks");
  if (ntask < 1 || ntask > MAXTASK) return picrom_set_error(PICROM_ERR_CONFIG, "gram_tasks: bad task count");
  Blocks b{};
  b.nb = nblocks;
  b.off[0] = 0;
  for (int i = 0; i < nblocks; ++i) {
    b.ptr[i] = ptrs[i]; b.ld[i] = lds[i]; b.w[i] = widths[i];
    b.jswap[i] = jswap ? jswap[i] : 0;
    b.off[i + 1] = b.off[i] + widths[i];
  }
  GramTasks tk{};
  for (int t = 0; t < ntask; ++t) {
    if (bi[t] < 0 || bj[t] < 0 || bi[t] >= nblocks || bj[t] >= nblocks)
      return picrom_set_error(PICROM_ERR_CONFIG, "gram_tasks: block index out of range");
    tk.bi[t] = (unsigned char)bi[t];
    tk.bj[t] = (unsigned char)bj[t];
  }
  tk.ntask = ntask;
  const int rc = gram_mma_try(b, 0, N, ws, (cudaStream_t)stream, out, &tk);
  if (rc != -1) return rc;
  return gram_impl(nblocks, 0, ptrs, lds, widths, jswap, N, out, ws, stream);   // all blocks
}

static int atb_grid(long long N) {
  return (int)std::max<long long>(1, std::min<long long>(picrom_num_sms(), N / (4 * ATG)));
}

extern "C" size_t picrom_tall_atb_workspace_bytes(long long N, int ca, int k) {
  return (size_t)atb_grid(N) * (size_t)ca * (size_t)k * sizeof(double) + 256;
}

template <int TPW, int CT, bool KSPLIT>
static int launch_tall_atb(const double* a, int lda, int ca, const double* b, int ldb, int k,
                           long long N, double* seg, int G, cudaStream_t s) {
  const int tg = KSPLIT ? 4 * ATG : ATG;
  const int pa = (KSPLIT && lda == ca) ? ca : atb_pitch(ca);
  const int pb = (KSPLIT && ldb == k) ? k : atb_pitch(k);
  size_t sm = (size_t)2 * tg * (pa + pb) * sizeof(double) + 2 * sizeof(uint64_t);
  sm = std::max(sm, (size_t)TPW * CT * 64 * sizeof(double));
  rom_allow_smem(tall_atb_kernel<TPW, CT, KSPLIT>);
  tall_atb_kernel<TPW, CT, KSPLIT><<<G, 256, sm, s>>>(a, lda, ca, b, ldb, k, N, seg, pa, pb);
  return picrom_check_launch("tall_atb_kernel");
}

extern "C" int picrom_tall_atb(const double* a, int lda, int ca, const double* b, int ldb, int k,
                               long long N, double* out, void* ws, void* stream) {
  if (N < 1 || ca < 2 || ca > 448 || k < 2 || k > 48 || (ca & 1) || (k & 1))
    return picrom_set_error(PICROM_ERR_CONFIG, "tall_atb: even widths, 2 <= ca <= 448, 2 <= k <= 48");
  if ((lda & 1) || (ldb & 1) || lda < ca || ldb < k ||
      ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15))
    return picrom_set_error(PICROM_ERR_CONFIG, "tall_atb: rows must be 16-byte aligned (even ld, aligned base)");
  cudaStream_t s = (cudaStream_t)stream;
  const int G = atb_grid(N);
  double* seg = (double*)ws;
  const int rt = (ca + 7) / 8;
  const int tpw = (rt + 7) / 8;
  const bool wide = k > 24;
  int rc;
  if (rt <= 6) rc = wide ? launch_tall_atb<6, 6, true>(a, lda, ca, b, ldb, k, N, seg, G, s)
                         : launch_tall_atb<6, 3, true>(a, lda, ca, b, ldb, k, N, seg, G, s);
  else if (tpw <= 1) rc = wide ? launch_tall_atb<1, 6, false>(a, lda, ca, b, ldb, k, N, seg, G, s)
                               : launch_tall_atb<1, 3, false>(a, lda, ca, b, ldb, k, N, seg, G, s);
  else if (tpw <= 4) rc = wide ? launch_tall_atb<4, 6, false>(a, lda, ca, b, ldb, k, N, seg, G, s)
                               : launch_tall_atb<4, 3, false>(a, lda, ca, b, ldb, k, N, seg, G, s);
  else rc = wide ? launch_tall_atb<7, 6, false>(a, lda, ca, b, ldb, k, N, seg, G, s)
                 : launch_tall_atb<7, 3, false>(a, lda, ca, b, ldb, k, N, seg, G, s);
  if (rc) return rc;
  const int rows = ca * k;
  seg_sum_kernel<<<(rows + SEGQ - 1) / SEGQ, 256, 0, s>>>(seg, G, rows, out, 0, 0, 1);
  return picrom_check_launch("seg_sum");
}

extern "C" int picrom_small_cholinv(const double* g, int k, double* rinv, double* info,
                                    void* stream) {
  if (k < 1 || k > SMK) return picrom_set_error(PICROM_ERR_CONFIG, "small_cholinv: 1 <= k <= 48");
  small_cholinv_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(g, k, rinv, info);
  return picrom_check_launch("small_cholinv");
}

extern "C" int picrom_small_rmul(const double* a, int r, int k, const double* b,
                                 const double* colscale, double* out, void* stream) {
  if (r < 1 || k < 1 || k > SMK) return picrom_set_error(PICROM_ERR_CONFIG, "small_rmul: r >= 1, 1 <= k <= 48");
  small_rmul_kernel<<<std::min(r, 4 * picrom_num_sms()), SMK, 0, (cudaStream_t)stream>>>(a, r, k, b, colscale, out);
  return picrom_check_launch("small_rmul");
}

extern "C" int picrom_argmax_abs(const double* v, long long n, long long stride,
                                 const long long* banned, int nbanned, long long* out_index,
                                 double* out_value, void* ws, void* stream) {
  if (n < 1) return picrom_set_error(PICROM_ERR_CONFIG, "argmax of an empty vector");
  cudaStream_t s = (cudaStream_t)stream;
  const int G = (int)std::min<long long>(2 * picrom_num_sms(), (n + 255) / 256);
  double* pv = (double*)ws;
  long long* pi = (long long*)(pv + G);
  argmax_abs_kernel<<<G, 256, 0, s>>>(v, n, stride, banned, nbanned, pv, pi);
  int rc = picrom_check_launch("argmax_abs");
  if (rc) return rc;
  argmax_final_kernel<<<1, 32, 0, s>>>(pv, pi, G, out_index, out_value);
  return picrom_check_launch("argmax_final");
}

// ------------------------------------------------------------ DEIM greedy
//
// deim_greedy (hyper.py:218-246) as one device-resident sequence: psi (N x d,
// row-major) is copied once to column-major psiT (d x N) so every residual
// pass reads coalesced columns; per selected position k
//   1. deim_resid_kernel: r_i = psi_k[i] - sum_{j<k} psi_j[i] c_j, scored
//      |r_i| (banned indices -1), per-block first-max partials;
//   2. deim_pick_kernel (one CTA): final first-max -> I[k], R[k][:] =
//      psi[I[k], :], banned += I[k]; then c for the next position k' from
//      R[:k', :k'] c = R[:k', k'] (Gaussian elimination, partial pivoting) --
//      the coefficient solve of hyper.py:239.
// No host round trip between positions; kept positions (partial refresh,
// hyper.py:268-275) are pre-assigned and banned from the start.

constexpr int kDeimMaxD = 64;
constexpr int kDeimThreads = 256;

__global__ void deim_transpose_kernel(const double* psi, int ld, long long N, int d,
                                      double* psiT) {
  __shared__ double tile[32][33];
  const long long r0 = (long long)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int q = threadIdx.y; q < 32; q += blockDim.y) {
    const long long r = r0 + q;
    const int c = c0 + threadIdx.x;
    tile[q][threadIdx.x] = (r < N && c < d) ? psi[(size_t)r * ld + c] : 0.0;
  }
  __syncthreads();
  for (int q = threadIdx.y; q < 32; q += blockDim.y) {
    const int c = c0 + q;
    const long long r = r0 + threadIdx.x;
    if (c < d && r < N) psiT[(size_t)c * N + r] = tile[threadIdx.x][q];
  }
}

__global__ void __launch_bounds__(kDeimThreads)
deim_resid_kernel(const double* psiT, long long N, int k, const double* coef,
                  const long long* banned, int nbanned, double* pv, long long* pi) {
  __shared__ double sc[kDeimMaxD];
  __shared__ long long sb[kDeimMaxD];
  __shared__ double sv[kDeimThreads];
  __shared__ long long si[kDeimThreads];
  for (int j = threadIdx.x; j < k; j += blockDim.x) sc[j] = coef[j];
  for (int j = threadIdx.x; j < nbanned; j += blockDim.x) sb[j] = banned[j];
  __syncthreads();
  double bv = -2.0;
  long long bi = 0x7fffffffffffffffLL;
  const double* col_k = psiT + (size_t)k * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < k; ++j) acc = fma(psiT[(size_t)j * N + i], sc[j], acc);
    const double r = col_k[i] - acc;
    bool ban = false;
    for (int q = 0; q < nbanned; ++q) ban |= sb[q] == i;
    better(ban ? -1.0 : fabs(r), i, bv, bi);
  }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      double cv = sv[threadIdx.x];
      long long ci = si[threadIdx.x];
      better(sv[threadIdx.x + o], si[threadIdx.x + o], cv, ci);
      sv[threadIdx.x] = cv;
      si[threadIdx.x] = ci;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pv[blockIdx.x] = sv[0];
    pi[blockIdx.x] = si[0];
  }
}

// rows[k][:] = psi[idx[k], :] for the pre-assigned (kept) positions
__global__ void deim_keep_rows_kernel(const double* psiT, long long N, int d, const long long* idx,
                                      double* rows) {
  const int k = blockIdx.x;
  const long long i = idx[k];
  if (i < 0) return;
  for (int j = threadIdx.x; j < d; j += blockDim.x) rows[(size_t)k * d + j] = psiT[(size_t)j * N + i];
}

// One CTA: finish position k (k < 0: nothing to finish), prepare position kn
// (kn < 0: done).  m holds c (kn entries) for the next residual pass.
__global__ void __launch_bounds__(kDeimThreads)
deim_pick_kernel(const double* pv, const long long* pi, int nparts, const double* psiT, long long N,
                 int d, int k, int kn, long long* idx, double* rows, long long* banned, int nb,
                 double* coef) {
  __shared__ double sv[kDeimThreads];
  __shared__ long long si[kDeimThreads];
  __shared__ double a[kDeimMaxD][kDeimMaxD + 1];
  __shared__ int s_piv;
  const int tid = threadIdx.x;
  if (k >= 0) {
    double bv = -2.0;
    long long bi = 0x7fffffffffffffffLL;
    for (int q = tid; q < nparts; q += blockDim.x) better(pv[q], pi[q], bv, bi);
    sv[tid] = bv;
    si[tid] = bi;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (tid < o) {
        double cv = sv[tid];
        long long ci = si[tid];
        better(sv[tid + o], si[tid + o], cv, ci);
        sv[tid] = cv;
        si[tid] = ci;
      }
      __syncthreads();
    }
    const long long pick = si[0];
    if (tid == 0) {
      idx[k] = pick;
      banned[nb] = pick;
    }
    for (int j = tid; j < d; j += blockDim.x) rows[(size_t)k * d + j] = psiT[(size_t)j * N + pick];
    __syncthreads();
    __threadfence_block();
  }
  if (kn <= 0) return;
  // augmented system [R[:kn, :kn] | R[:kn, kn]], row r = position r
  const int m = kn;
  for (int q = tid; q < m * (m + 1); q += blockDim.x) {
    const int r = q / (m + 1), c = q % (m + 1);
    a[r][c] = rows[(size_t)r * d + (c < m ? c : kn)];
  }
  __syncthreads();
  for (int col = 0; col < m; ++col) {
    if (tid == 0) {             // partial pivoting, first max (LAPACK idamax)
      int piv = col;
      double best = fabs(a[col][col]);
      for (int r = col + 1; r < m; ++r)
        if (fabs(a[r][col]) > best) { best = fabs(a[r][col]); piv = r; }
      s_piv = piv;
    }
    __syncthreads();
    const int piv = s_piv;
    if (piv != col)
      for (int c = tid; c <= m; c += blockDim.x) {
        const double t = a[col][c];
        a[col][c] = a[piv][c];
        a[piv][c] = t;
      }
    __syncthreads();
    const double inv = 1.0 / a[col][col];
    for (int q = tid; q < (m - col - 1) * (m - col); q += blockDim.x) {
      const int r = col + 1 + q / (m - col), c = col + 1 + q % (m - col);
      a[r][c] = fma(-(a[r][col] * inv), a[col][c], a[r][c]);
    }
    __syncthreads();
  }
  if (tid == 0) {               // back substitution (serial: m <= 64)
    for (int r = m - 1; r >= 0; --r) {
      double t = a[r][m];
      for (int c = r + 1; c < m; ++c) t = fma(-a[r][c], a[c][m], t);
      a[r][m] = t / a[r][r];
    }
  }
  __syncthreads();
  for (int r = tid; r < m; r += blockDim.x) coef[r] = a[r][m];
}

extern "C" size_t picrom_deim_workspace_bytes(long long N, int d) {
  const int G = (int)std::min<long long>(4LL * picrom_num_sms(), (N + 255) / 256);
  return (size_t)d * N * sizeof(double) + (size_t)G * (sizeof(double) + sizeof(long long)) +
         (size_t)(3 * kDeimMaxD) * sizeof(double) + 256;
}

extern "C" int picrom_deim_greedy(const double* psi, int ld, long long N, int d,
                                  const long long* keep, long long* idx, double* rows, void* ws,
                                  void* stream) {
  if (N < 1 || d < 1 || d > kDeimMaxD || ld < d)
    return picrom_set_error(PICROM_ERR_CONFIG, "deim_greedy: need N >= 1, 1 <= d <= 64, ld >= d");
  cudaStream_t s = (cudaStream_t)stream;
  const int G = (int)std::min<long long>(4LL * picrom_num_sms(), (N + 255) / 256);
  double* psiT = (double*)ws;
  double* pv = psiT + (size_t)d * N;
  long long* pi = (long long*)(pv + G);
  double* coef = (double*)(pi + G);
  long long* banned = (long long*)(coef + kDeimMaxD);
  // keep: host array of d entries (index >= 0: pre-assigned position)
  int nb = 0;
  std::vector<int> order;
  std::vector<long long> kept;
  for (int k = 0; k < d; ++k) {
    if (keep && keep[k] >= 0) kept.push_back(keep[k]);
    else order.push_back(k);
  }
  std::vector<long long> idx_init(d, -1);
  for (int k = 0; k < d; ++k) if (keep && keep[k] >= 0) idx_init[k] = keep[k];
  cudaMemcpyAsync(idx, idx_init.data(), d * sizeof(long long), cudaMemcpyHostToDevice, s);
  if (!kept.empty())
    cudaMemcpyAsync(banned, kept.data(), kept.size() * sizeof(long long), cudaMemcpyHostToDevice, s);
  nb = (int)kept.size();
  dim3 tg((unsigned)((N + 31) / 32), (unsigned)((d + 31) / 32));
  deim_transpose_kernel<<<tg, dim3(32, 8), 0, s>>>(psi, ld, N, d, psiT);
  int rc = picrom_check_launch("deim_transpose");
  if (rc) return rc;
  if (!kept.empty()) {
    deim_keep_rows_kernel<<<d, 64, 0, s>>>(psiT, N, d, idx, rows);
    if ((rc = picrom_check_launch("deim_keep_rows"))) return rc;
  }
  // coefficients of the first position
  const int k0 = order.empty() ? -1 : order[0];
  if (k0 > 0) {
    deim_pick_kernel<<<1, kDeimThreads, 0, s>>>(pv, pi, G, psiT, N, d, -1, k0, idx, rows, banned,
                                                nb, coef);
    if ((rc = picrom_check_launch("deim_pick"))) return rc;
  }
  for (size_t q = 0; q < order.size(); ++q) {
    const int k = order[q];
    const int kn = q + 1 < order.size() ? order[q + 1] : -1;
    deim_resid_kernel<<<G, kDeimThreads, 0, s>>>(psiT, N, k, coef, banned, nb, pv, pi);
    if ((rc = picrom_check_launch("deim_resid"))) return rc;
    deim_pick_kernel<<<1, kDeimThreads, 0, s>>>(pv, pi, G, psiT, N, d, k, kn, idx, rows, banned,
                                                nb, coef);
    if ((rc = picrom_check_launch("deim_pick"))) return rc;
    ++nb;
  }
  return PICROM_OK;
}

// out (N x c) (+)= sum_t in_t (N x a_t) @ M_t (a_t x c); mats is a device buffer
// holding the M_t back to back (offsets moffs, in doubles).
// Combine with a wide term (a_t > 32, e.g. the N x p' field block E times a
// p' x n matrix in the basis velocity): A streams from global straight into
// DMMA fragments (lane (g, t) reads row g, column 4 ks + t: every 32-byte
// sector read once), M sits in smem with a pitch = 1 mod 4 (conflict-free B
// fragments under the permuted k order), and a warp owns 16 rows = 2 row
// blocks x TBO column tiles of independent accumulators.
// WRB 8-row blocks per warp chunk: 2, or 4 for the 40/48-column outputs (their M
// fills the smem of a whole SM, so one CTA per SM may use 255 registers: twice
// the independent DMMA chains per B-fragment load)
template <int TBO> __host__ __device__ constexpr int wide_wrb() { return TBO >= 5 ? 4 : 2; }
template <int TBO>
__global__ void __launch_bounds__(256, TBO >= 5 ? 1 : 2) wide_combine_kernel(Terms t, const double* mats,
                                                           long long N, int cp) {
  extern __shared__ __align__(16) double wsm[];
  constexpr int WRB = wide_wrb<TBO>();
  int koff[MAXTERM + 1];
  koff[0] = 0;
  for (int i = 0; i < t.nt; ++i) koff[i + 1] = koff[i] + ((t.a[i] + 3) & ~3);
  const int K = koff[t.nt];
  const int c = t.c;
  for (int q = threadIdx.x; q < K * cp; q += blockDim.x) {
    const int k = q / cp, j = q - k * cp;
    int ti = 0;
    while (k >= koff[ti + 1]) ++ti;
    const int kk = k - koff[ti];
    wsm[q] = (kk < t.a[ti] && j < c) ? mats[t.moff[ti] + kk * c + j] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const long long half = N / 2;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r0 = gw * 8 * WRB; r0 < N; r0 += nw * 8 * WRB) {
    double acc[WRB][TBO][2];
#pragma unroll
    for (int q = 0; q < WRB; ++q)
#pragma unroll
      for (int j = 0; j < TBO; ++j) acc[q][j][0] = acc[q][j][1] = 0.0;
    for (int ti = 0; ti < t.nt; ++ti) {
      const double* base[WRB];
      double sg[WRB];
      bool rv[WRB];
#pragma unroll
      for (int q = 0; q < WRB; ++q) {
        long long row = r0 + 8 * q + g;
        rv[q] = row < N;
        sg[q] = (t.jswap[ti] && row >= half) ? -1.0 : 1.0;
        if (t.jswap[ti]) row = row < half ? row + half : row - half;
        base[q] = t.in[ti] + (size_t)(rv[q] ? row : 0) * t.ld[ti];
      }
      const int a = t.a[ti];
      const double* mrow = wsm + (size_t)koff[ti] * cp + g;
      // 16-column groups with the k order permuted inside the group: logical
      // k = 16 grp + 4 ks + tq reads physical column 16 grp + 4 tq + ks, so a
      // lane's 4 k-steps are one contiguous 32-byte load (2 x 16 B) and the 4
      // lanes of a row cover a full 128-byte line; M rows use the same map.
      // The next group's loads are in flight while this group's DMMAs run.
      auto load_group = [&](int k0, double (*av)[4]) {
        const int c0 = k0 + 4 * tq;
#pragma unroll
        for (int q = 0; q < WRB; ++q) {
          if (rv[q] && c0 + 3 < a) {
            const double2 lo = __ldg(reinterpret_cast<const double2*>(base[q] + c0));
            const double2 hi = __ldg(reinterpret_cast<const double2*>(base[q] + c0 + 2));
            av[q][0] = lo.x; av[q][1] = lo.y; av[q][2] = hi.x; av[q][3] = hi.y;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) av[q][e] = (rv[q] && c0 + e < a) ? __ldg(base[q] + c0 + e) : 0.0;
          }
        }
      };
      auto compute_group = [&](int k0, const double (*av)[4]) {
        const int c0 = k0 + 4 * tq;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int kp = c0 + ks;                   // physical column (M row)
          double bv[TBO];
#pragma unroll
          for (int j = 0; j < TBO; ++j) bv[j] = kp < a ? mrow[(size_t)kp * cp + 8 * j] : 0.0;
#pragma unroll
          for (int q = 0; q < WRB; ++q)
#pragma unroll
            for (int j = 0; j < TBO; ++j) dmma(acc[q][j][0], acc[q][j][1], sg[q] * av[q][ks], bv[j]);
        }
      };
      double ga[WRB][4], gb[WRB][4];       // ping-pong: static indexing only
      if (a > 0) load_group(0, ga);
      for (int k0 = 0; k0 < a; k0 += 32) {
        if (k0 + 16 < a) load_group(k0 + 16, gb);
        compute_group(k0, ga);
        if (k0 + 16 >= a) break;
        if (k0 + 32 < a) load_group(k0 + 32, ga);
        compute_group(k0 + 16, gb);
      }
    }
#pragma unroll
    for (int q = 0; q < WRB; ++q) {
      const long long row = r0 + 8 * q + g;
      if (row >= N) continue;
      double* orow = t.out + (size_t)row * t.ldo;
#pragma unroll
      for (int j = 0; j < TBO; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * j + 2 * tq + e;
          if (col < c) orow[col] = t.accumulate ? orow[col] + acc[q][j][e] : acc[q][j][e];
        }
    }
  }
}

static int launch_wide_combine(const Terms& t, const double* mats, long long N, cudaStream_t s) {
  int K = 0;
  for (int i = 0; i < t.nt; ++i) K += (t.a[i] + 3) & ~3;
  const int tbo = (t.c + 7) / 8;
  // M pitch = 1 mod 4: with the permuted k order a lane (g, tq) reads M row
  // 4 tq + ks, so the four tq groups must land 4 double-banks apart (4 tq cp =
  // 4 tq mod 16) -- each bank twice, the 2-wavefront minimum of a 256-byte
  // request (a pitch = 4 mod 16 put all four groups on the same banks: ncu
  // counted 74 % of the kernel's smem wavefronts as conflicts)
  const int cp = 8 * tbo + 1;
  const size_t sm = (size_t)K * cp * sizeof(double);
  if (sm > 200 * 1024) return picrom_set_error(PICROM_ERR_CONFIG, "combine matrices too large");
  const int WRB = tbo >= 5 ? 4 : 2;
  const long long chunks = (N + 8 * WRB - 1) / (8 * WRB);
  const long long per_sm = tbo >= 5 ? 1 : 2;      // resident CTAs (one wave: M is staged once per CTA)
  const int G = (int)std::max<long long>(1, std::min<long long>(per_sm * picrom_num_sms(), (chunks + 7) / 8));
  switch (tbo) {
    case 1: rom_allow_smem(wide_combine_kernel<1>); wide_combine_kernel<1><<<G, 256, sm, s>>>(t, mats, N, cp); break;
    case 2: rom_allow_smem(wide_combine_kernel<2>); wide_combine_kernel<2><<<G, 256, sm, s>>>(t, mats, N, cp); break;
    case 3: rom_allow_smem(wide_combine_kernel<3>); wide_combine_kernel<3><<<G, 256, sm, s>>>(t, mats, N, cp); break;
    case 4: rom_allow_smem(wide_combine_kernel<4>); wide_combine_kernel<4><<<G, 256, sm, s>>>(t, mats, N, cp); break;
    case 5: rom_allow_smem(wide_combine_kernel<5>); wide_combine_kernel<5><<<G, 256, sm, s>>>(t, mats, N, cp); break;
    default: rom_allow_smem(wide_combine_kernel<6>); wide_combine_kernel<6><<<G, 256, sm, s>>>(t, mats, N, cp); break;
  }
  return picrom_check_launch("wide_combine_kernel");
}

extern "C" int picrom_combine(int nterms, const double* const* ins, const int* lds,
                              const int* widths, const int* jswap, const int* moffs,
                              const double* mats, int mats_len, long long N, double* out,
                              int ldo, int c, int accumulate, void* stream) {
  if (nterms < 1 || nterms > MAXTERM) return picrom_set_error(PICROM_ERR_CONFIG, "1..6 terms");
  // up to 48 output columns through the wide kernel (16-byte aligned rows, N >= 1024:
  // the DEIM window's subspace block, hyper.py:262), 32 otherwise
  bool all_aligned = N >= 1024;
  for (int i = 0; i < nterms; ++i)
    all_aligned &= (lds[i] % 2 == 0) && ((reinterpret_cast<uintptr_t>(ins[i]) & 15) == 0);
  if (c < 1 || c > (all_aligned && !kNoCombineWide ? 48 : NMAX))
    return picrom_set_error(PICROM_ERR_CONFIG, "output width in [1, 32] (48 for aligned inputs)");
  Terms t{};
  t.nt = nterms;
  for (int i = 0; i < nterms; ++i) {
    t.in[i] = ins[i]; t.ld[i] = lds[i]; t.a[i] = widths[i]; t.moff[i] = moffs[i];
    t.jswap[i] = jswap ? jswap[i] : 0;
  }
  t.out = out; t.ldo = ldo; t.c = c; t.accumulate = accumulate;
  const size_t sm = (size_t)mats_len * sizeof(double);
  if (sm > 200 * 1024) return picrom_set_error(PICROM_ERR_CONFIG, "combine matrices too large");
  cudaStream_t s = (cudaStream_t)stream;
  bool wide = false, aligned = true;
  for (int i = 0; i < nterms; ++i) {
    wide |= widths[i] > 32;
    aligned &= (lds[i] % 2 == 0) && ((reinterpret_cast<uintptr_t>(ins[i]) & 15) == 0);
  }
  wide &= aligned;        // the wide kernel reads rows in 16-byte pieces
  // every aligned combine takes the wide kernel (measured >= the narrow one)
  if (aligned) wide = true;
  if (wide && !kNoCombineWide && N >= 1024)
    return launch_wide_combine(t, mats, N, s);
  // DMMA path: even widths, rows 16-B aligned (ld even, 16-B aligned base)
  bool mma = !kNoCombineMma && N >= 1024;
  MmaTerms mt{};
  for (int i = 0; i < nterms && mma; ++i)
    mma = (widths[i] % 2 == 0) && (lds[i] % 2 == 0) && ((reinterpret_cast<uintptr_t>(ins[i]) & 15) == 0);
  if (mma) {
    mt.koff[0] = 0;
    mt.soff[0] = 0;
    for (int i = 0; i < nterms; ++i) {
      int pa = widths[i];
      while (pa % 16 != 4 && pa % 16 != 12) pa += 2;
      mt.pa[i] = pa;
      mt.koff[i + 1] = mt.koff[i] + widths[i];
      mt.soff[i + 1] = mt.soff[i] + pa;
    }
    int cp = c;                       // M pitch = 4 or 12 mod 16: conflict-free B fragments
    while (cp % 16 != 4 && cp % 16 != 12) ++cp;
    mt.cp = cp;
    const size_t smm = ((size_t)(mt.koff[nterms] + 4) * cp + 8 + (size_t)2 * CMR * mt.soff[nterms]) * sizeof(double);
    if (smm <= 200 * 1024) {
      const int G = (int)std::min<long long>(2LL * picrom_num_sms(), std::max<long long>(1, (N + CMR - 1) / CMR));
      const int tbo = (c + 7) / 8;
      switch (tbo) {
        case 1: rom_allow_smem(combine_mma_kernel<1>); combine_mma_kernel<1><<<G, 256, smm, s>>>(t, mt, mats, N); break;
        case 2: rom_allow_smem(combine_mma_kernel<2>); combine_mma_kernel<2><<<G, 256, smm, s>>>(t, mt, mats, N); break;
        case 3: rom_allow_smem(combine_mma_kernel<3>); combine_mma_kernel<3><<<G, 256, smm, s>>>(t, mt, mats, N); break;
        default: rom_allow_smem(combine_mma_kernel<4>); combine_mma_kernel<4><<<G, 256, smm, s>>>(t, mt, mats, N); break;
      }
      return picrom_check_launch("combine_mma_kernel");
    }
  }
  // TMA path: row-contiguous, 16-B aligned inputs
  bool tma = !kNoCombineTma;
  int wsum = 0;
  for (int i = 0; i < nterms && tma; ++i) {
    tma = lds[i] == widths[i] && ((widths[i] * 8) % 16 == 0) &&
          ((reinterpret_cast<uintptr_t>(ins[i]) & 15) == 0);
    wsum += widths[i];
  }
  const size_t sm_tma = (size_t)2 * CR * wsum * sizeof(double) + (size_t)((mats_len + 1) & ~1) * sizeof(double) +
                        2 * sizeof(uint64_t);
  if (tma && sm_tma <= 200 * 1024) {
    const int G = (int)std::min<long long>(2LL * picrom_num_sms(), std::max<long long>(1, (N + CR - 1) / CR));
    const int cpt = (c + 3) / 4;
    if (cpt <= 2) { rom_allow_smem(combine_tma_kernel<2>); combine_tma_kernel<2><<<G, 256, sm_tma, s>>>(t, mats, mats_len, N); }
    else if (cpt <= 4) { rom_allow_smem(combine_tma_kernel<4>); combine_tma_kernel<4><<<G, 256, sm_tma, s>>>(t, mats, mats_len, N); }
    else if (cpt <= 6) { rom_allow_smem(combine_tma_kernel<6>); combine_tma_kernel<6><<<G, 256, sm_tma, s>>>(t, mats, mats_len, N); }
    else { rom_allow_smem(combine_tma_kernel<8>); combine_tma_kernel<8><<<G, 256, sm_tma, s>>>(t, mats, mats_len, N); }
    return picrom_check_launch("combine_tma_kernel");
  }
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess)
      (void)cudaGetLastError();
    attr = true;
  }
  const unsigned blocks = (unsigned)((N + 255) / 256);
  combine_kernel<<<blocks, 256, sm, s>>>(t, mats, mats_len, N);
  return picrom_check_launch("combine_kernel");
}

extern "C" int picrom_dmd_extrapolate(const double* modes, const double* coords, const double* w,
                                      int nx, int r, int p, double* re_out, double* im_out,
                                      void* stream) {
  if (nx < 1 || r < 1 || p < 1) return picrom_set_error(PICROM_ERR_CONFIG, "empty DMD model");
  const int tot = nx * p;
  dmd_extrap_kernel<<<(tot + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
      (const double2*)modes, (const double2*)coords, (const double2*)w, nx, r, p, re_out, im_out);
  return picrom_check_launch("dmd_extrapolate");
}

extern "C" int picrom_deim_gather(const double* uxd, const double* z, int ldz, const double* phi,
                                  const double* inst, const int* cols, const double* w,
                                  const double* wscale, int d, int n, int p, int nx, int degree,
                                  double* out, int ldo, unsigned long long* status,
                                  const long long* skip, void* stream) {
  if (d < 1 || n < 1 || p < 1) return picrom_set_error(PICROM_ERR_CONFIG, "empty DEIM stage");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t sm = (size_t)d * sizeof(double);
  switch (degree) {
    case 1: deim_gather_kernel<1><<<p, 64, sm, s>>>(uxd, z, ldz, phi, inst, cols, w, wscale, d, n, p, nx, out, ldo, status, skip); break;
    case 2: deim_gather_kernel<2><<<p, 64, sm, s>>>(uxd, z, ldz, phi, inst, cols, w, wscale, d, n, p, nx, out, ldo, status, skip); break;
    case 3: deim_gather_kernel<3><<<p, 64, sm, s>>>(uxd, z, ldz, phi, inst, cols, w, wscale, d, n, p, nx, out, ldo, status, skip); break;
    default: return picrom_set_error(PICROM_ERR_CONFIG, "degree must be 1, 2 or 3");
  }
  return picrom_check_launch("deim_gather");
}

// ------------------------------------------------- device fixed point
//
// One iteration of reduction.fixed_point (reduction.py:185-202) for the stage
// map k -> J g(z + dt/2 k) with g(z) = D(z) + (U_V^T U_V) z, D(z) already in
// gout (the F-evaluation kernels, evaluated at zeval = z + dt/2 k):
//   k_new = J (gout + C zeval); r = ||k_new - k|| / max(||k_new||, tiny);
//   trace[it] = r; k = k_new; converged (r <= tol) -> state = {1, it + 1};
//   zeval = z + dt/2 k_new for the next iteration.
// One CTA; once converged every later call (and the F-evaluation kernels,
// which test state[0] as their skip flag) returns immediately.
__global__ void __launch_bounds__(256) fp_update_kernel(const double* gout, const double* c,
                                                       const double* z, double* k, double* zeval,
                                                       int n, int p, double half_dt, double tol,
                                                       int it, long long* state, double* trace) {
  extern __shared__ double g[];        // [n p] g | [n p] z_eval | [n n] C
  __shared__ double red[64];
  if (state[0]) return;
  const int tid = threadIdx.x, np = n * p;
  // stage z_eval and C first (every load in flight at once: one L2 round trip
  // instead of one per FMA batch -- the kernel sits between the F-evaluation
  // launches of every fixed-point iteration and is pure latency)
  double* zs = g + np;
  double* cs = zs + np;
  for (int q = tid; q < np; q += blockDim.x) {
    zs[q] = zeval[q];
    g[q] = gout[q];
  }
  for (int q = tid; q < n * n; q += blockDim.x) cs[q] = c[q];
  __syncthreads();
  for (int q = tid; q < np; q += blockDim.x) {
    const int r = q / p, col = q - r * p;
    double acc = g[q];
    for (int j = 0; j < n; ++j) acc = fma(cs[r * n + j], zs[j * p + col], acc);
    g[q] = acc;                        // each thread rewrites only its own entries
  }
  __syncthreads();
  const int h = n / 2;
  double dd = 0.0, kk = 0.0;
  for (int q = tid; q < np; q += blockDim.x) {
    const int r = q / p, col = q % p;
    const double kn = r < h ? g[(r + h) * p + col] : -g[(r - h) * p + col];
    const double df = kn - k[q];
    dd = fma(df, df, dd);
    kk = fma(kn, kn, kk);
  }
  // block reductions (fixed tree)
  dd = warp_sum(dd);
  kk = warp_sum(kk);
  const int w = tid >> 5, l = tid & 31;
  if (l == 0) { red[w] = dd; red[32 + w] = kk; }
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    double a = l < nw ? red[l] : 0.0, b = l < nw ? red[32 + l] : 0.0;
    a = warp_sum(a);
    b = warp_sum(b);
    if (l == 0) { red[0] = a; red[32] = b; }
  }
  __syncthreads();
  const double num = sqrt(red[0]);
  const double den = fmax(sqrt(red[32]), 2.2250738585072014e-308);
  for (int q = tid; q < np; q += blockDim.x) {
    const int r = q / p, col = q % p;
    const double kn = r < h ? g[(r + h) * p + col] : -g[(r - h) * p + col];
    k[q] = kn;
    zeval[q] = fma(half_dt, kn, z[q]);
  }
  if (tid == 0) {
    trace[it] = num / den;
    if (num <= tol * den) {
      state[1] = it + 1;
      __threadfence();
      state[0] = 1;
    }
  }
}

extern "C" int picrom_fp_update(const double* gout, const double* c, const double* z, double* k,
                                double* zeval, int n, int p, double half_dt, double tol, int it,
                                long long* state, double* trace, void* stream) {
  if (n < 2 || (n & 1) || p < 1) return picrom_set_error(PICROM_ERR_CONFIG, "fp_update: bad n / p");
  const size_t sm = ((size_t)2 * n * p + (size_t)n * n) * sizeof(double);
  if (sm > 200 * 1024) return picrom_set_error(PICROM_ERR_CONFIG, "fp_update: n p too large");
  static bool attr = false;
  if (!attr) {
    rom_allow_smem(fp_update_kernel);
    attr = true;
  }
  fp_update_kernel<<<1, 256, sm, (cudaStream_t)stream>>>(gout, c, z, k, zeval, n, p, half_dt, tol,
                                                          it, state, trace);
  return picrom_check_launch("fp_update");
}

// out (d x w) = src rows idx (src row-major with leading dim ld)
extern "C" int picrom_rows_gather(const double* src, int ld, const long long* idx, int d, int w,
                                  double* out, void* stream) {
  if (d < 1 || w < 1) return PICROM_OK;
  rows_gather_kernel<<<(d * w + 255) / 256, 256, 0, (cudaStream_t)stream>>>(src, ld, idx, d, w, out);
  return picrom_check_launch("rows_gather");
}
