// Shared device helpers: locate, B-spline weights, cell polynomials, status.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/picrom_b200.h"

namespace picrom {

// per-instance parameter row (PICROM_INST_STRIDE doubles)
enum InstField { I_H = 0, I_INVH = 1, I_QW = 2, I_BGH = 3, I_ECOEF = 4, I_GCOEF = 5,
                 I_HALFINVMP = 6, I_LENGTH = 7 };

constexpr int kThreads = 256;

// Python-style (non-negative) c mod nx of an integer-valued double, matching
// numpy's `cell.astype(np.int64) % nx` (fem.py:115) including the saturating
// out-of-range cast (numpy yields INT64_MIN for NaN/inf/huge).  Power-of-two
// nx (all BASELINE configs) is a mask of the two's-complement index.
__device__ __forceinline__ int cell_mod(double c, int nx, double inv_nx) {
  if (fabs(c) < 2147483648.0) {
    const int ci = static_cast<int>(c);
    if ((nx & (nx - 1)) == 0) return ci & (nx - 1);
    int q = __double2int_rd(static_cast<double>(ci) * inv_nx);
    int r = ci - q * nx;
    if (r < 0) r += nx;
    if (r >= nx) r -= nx;
    return r;
  }
  long long ci;
  if (fabs(c) < 9223372036854775808.0) ci = static_cast<long long>(c);
  else ci = (long long)(-9223372036854775807LL - 1);
  long long r = ci % nx;
  if (r < 0) r += nx;
  return static_cast<int>(r);
}

// Correctly rounded x / h from the correctly rounded reciprocal inv_h =
// RN(1/h) (host-computed): q0 = RN(x*inv_h) is within 1 ulp of x/h, the FMA
// residual r = x - h*q0 is exact, and RN(q0 + r*inv_h) = RN(x/h) (Markstein's
// theorem); tiny/huge/non-finite quotients take IEEE division.  Verified against IEEE division in tests/test_fem_gpu.py.
__device__ __forceinline__ double div_rn(double x, double h, double inv_h) {
  const double q0 = __dmul_rn(x, inv_h);
  // outside the range where the residual is exact: plain IEEE division
  if (!(fabs(q0) > 1e-280 && fabs(q0) < 1e280)) return __ddiv_rn(x, h);
  const double r = fma(-h, q0, x);
  return fma(r, inv_h, q0);
}

// fem._locate arithmetic (fem.py:112-115): s = x / h (IEEE division), cell =
// floor(s), frac = s - cell (exact), i0 = cell mod nx.
__device__ __forceinline__ void locate(double x, double h, double inv_h, int nx, double inv_nx,
                                       int& i0, double& frac) {
  const double s = div_rn(x, h, inv_h);
  const double c = floor(s);
  frac = __dsub_rn(s, c);
  i0 = cell_mod(c, nx, inv_nx);
}

// Branch-free common path of locate() for power-of-two nx.  `mask` comes from
// fast_mask(): nx - 1, or -1 when nx is not a power of two or h is outside
// [2^-100, 2^100].  `rare` flags the inputs the fast path does not cover --
// |x/h| >= 2^51, |x/h| <= 2^-900 (incl. 0), non-finite x, or mask < 0 -- which
// callers re-run through locate() in a warp-uniform fix-up pass.
//
// x/h: Markstein's correction of q0 = RN(x * RN(1/h)) gives RN(x/h) (IEEE
// division) whenever q0 is far from under/overflow (|q0| > 2^-900 here).
// floor() without the XU pipe (F2I.F64 / FRND.F64 run on the conversion unit,
// which ncu showed at 83% busy in the step kernel, profiles/r01): for
// |s| < 2^51, t = RD(s + 1.5*2^52) = 1.5*2^52 + floor(s) exactly (the ulp of
// t is 1), so c = t - 1.5*2^52 = floor(s), and the low word of t is
// floor(s) mod 2^32, hence floor(s) mod nx = lo(t) & (nx - 1).
__device__ __forceinline__ int fast_mask(int nx, double h) {
  return ((nx & (nx - 1)) == 0 && h > 0x1p-100 && h < 0x1p100) ? nx - 1 : -1;
}

__device__ __forceinline__ void locate_fast(double x, double h, double inv_h, int nx, int mask,
                                            double inv_nx, int& i0, double& frac, bool& rare) {
  constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52
  const double q0 = __dmul_rn(x, inv_h);
  const double r = fma(-h, q0, x);
  const double s = fma(r, inv_h, q0);
  const double t = __dadd_rd(s, kMagic);
  const double c = __dsub_rn(t, kMagic);
  frac = __dsub_rn(s, c);
  rare = !(fabs(q0) > 0x1p-900 && fabs(s) < 0x1p51) || mask < 0;
  i0 = __double2loint(t) & mask;
}

// locate() for a position already divided by h: the reduced-basis kernels
// reconstruct s = U_X (z / h) directly (one DMMA chain, no division), so only
// the floor remains -- by the 1.5*2^52 add; `rare` = |s| >= 2^51, non-finite,
// or non-power-of-two nx (mask < 0), handled by locate_scaled_exact().
__device__ __forceinline__ void locate_scaled(double s, int mask, int& i0, double& frac,
                                              bool& rare) {
  constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52
  const double t = __dadd_rd(s, kMagic);
  const double c = __dsub_rn(t, kMagic);
  frac = __dsub_rn(s, c);
  rare = !(fabs(s) < 0x1p51) || mask < 0;
  i0 = __double2loint(t) & mask;
}

__device__ __forceinline__ void locate_scaled_exact(double s, int nx, double inv_nx, int& i0,
                                                    double& frac) {
  const double c = floor(s);
  frac = __dsub_rn(s, c);
  i0 = cell_mod(c, nx, inv_nx);
}

__device__ __forceinline__ int pow2_mask(int nx) { return (nx & (nx - 1)) == 0 ? nx - 1 : -1; }

template <int D> struct Spline;

// P1 hat functions -- fem.py:179-200 exactly (weights 1-f, f; gradient -1/h, 1/h)
template <> struct Spline<1> {
  static constexpr int OFF = 0;     // first node = cell + OFF
  __device__ static __forceinline__ void weights(double f, double* w) {
    w[0] = __dsub_rn(1.0, f);
    w[1] = f;
  }
  __device__ static __forceinline__ void dweights(double f, double g, double* w) {
    w[0] = -g;
    w[1] = g;
  }
};

// quadratic: nodes c-1, c, c+1; weights N_2(f+2), N_2(f+1), N_2(f)
template <> struct Spline<2> {
  static constexpr int OFF = -1;
  __device__ static __forceinline__ void weights(double f, double* w) {
    double g = 1.0 - f;
    double e = f - 0.5;
    w[0] = 0.5 * g * g;
    w[1] = 0.75 - e * e;
    w[2] = 0.5 * f * f;
  }
  __device__ static __forceinline__ void dweights(double f, double g, double* w) {
    w[0] = (f - 1.0) * g;
    w[1] = (1.0 - 2.0 * f) * g;
    w[2] = f * g;
  }
};

// cubic: nodes c-1..c+2; weights N_3(f+3), N_3(f+2), N_3(f+1), N_3(f)
template <> struct Spline<3> {
  static constexpr int OFF = -1;
  __device__ static __forceinline__ void weights(double f, double* w) {
    const double s6 = 1.0 / 6.0;
    const double g = 1.0 - f;
    const double f2 = f * f, f3 = f2 * f;
    w[0] = (g * g) * (g * s6);
    w[1] = fma(0.5, f3, (2.0 / 3.0) - f2);
    w[2] = fma(0.5, (f + f2) - f3, s6);
    w[3] = f3 * s6;
  }
  __device__ static __forceinline__ void dweights(double f, double g, double* w) {
    const double e = 1.0 - f;
    w[0] = (-0.5 * e * e) * g;
    w[1] = (1.5 * f * f - 2.0 * f) * g;
    w[2] = (-1.5 * f * f + f + 0.5) * g;
    w[3] = (0.5 * f * f) * g;
  }
};

__device__ __forceinline__ int wrap_node(int q, int nx) {
  q %= nx;
  return q < 0 ? q + nx : q;
}

// Per-cell polynomial coefficients of the gathered quantity in the in-cell
// fraction f:  value  sum_m phi_m N_d(f+d-m)            (D+1 coefficients)
//              deriv  coef * sum_m phi_m dN_d/dx(...)    (D coefficients)
// phi_m = phi[(c + OFF + m) mod nx].  D = 1 deriv keeps the reference's
// operation order coef * ((-g)*phi0 + g*phi1) (fem.py:146,188-190,256).
template <int D>
__device__ __forceinline__ void deriv_coeffs(const double* ph, double coef, double g, double* C) {
  if constexpr (D == 1) {
    C[0] = __dmul_rn(coef, __dadd_rn(__dmul_rn(-g, ph[0]), __dmul_rn(g, ph[1])));
  } else if constexpr (D == 2) {
    double s = coef * g;
    C[0] = s * (ph[1] - ph[0]);
    C[1] = s * (ph[0] - 2.0 * ph[1] + ph[2]);
  } else {
    double s = coef * g;
    C[0] = s * 0.5 * (ph[2] - ph[0]);
    C[1] = s * (ph[0] - 2.0 * ph[1] + ph[2]);
    C[2] = s * (-0.5 * ph[0] + 1.5 * ph[1] - 1.5 * ph[2] + 0.5 * ph[3]);
  }
}

template <int D>
__device__ __forceinline__ void value_coeffs(const double* ph, double* C) {
  if constexpr (D == 1) {
    C[0] = ph[0];
    C[1] = ph[1];       // evaluated directly as (1-f)*phi0 + f*phi1
  } else if constexpr (D == 2) {
    C[0] = 0.5 * (ph[0] + ph[1]);
    C[1] = ph[1] - ph[0];
    C[2] = 0.5 * ph[0] - ph[1] + 0.5 * ph[2];
  } else {
    const double s6 = 1.0 / 6.0;
    C[0] = (ph[0] + 4.0 * ph[1] + ph[2]) * s6;
    C[1] = 0.5 * (ph[2] - ph[0]);
    C[2] = 0.5 * (ph[0] - 2.0 * ph[1] + ph[2]);
    C[3] = (-ph[0] + 3.0 * ph[1] - 3.0 * ph[2] + ph[3]) * s6;
  }
}

// Horner in f over NC coefficients (C[0] + f*C[1] + ...)
template <int NC>
__device__ __forceinline__ double horner(const double* C, double f) {
  double r = C[NC - 1];
#pragma unroll
  for (int k = NC - 2; k >= 0; --k) r = fma(r, f, C[k]);
  return r;
}

__device__ __forceinline__ void record_bad(unsigned long long* status, long long step,
                                           long long row, int col, int p) {
  if (status) {
    unsigned long long lin = (unsigned long long)row * (unsigned long long)p + (unsigned long long)col;
    atomicMin(status, ((unsigned long long)step << 40) | lin);
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block reduction (fixed tree); all threads get the result
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  int nw = (blockDim.x + 31) >> 5;
  if (w == 0) {
    t = l < nw ? red[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// ---- TMA bulk copies + mbarriers (Hopper/Blackwell async proxy) ----
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}

// predicated shared-memory f64 load / store (no branch: @p ld/st.shared)
__device__ __forceinline__ double lds_f64_if(uint32_t addr, bool p) {
  double v = 0.0;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}\n"
      : "+d"(v) : "r"(addr), "r"((uint32_t)p));
  return v;
}
// as lds_f64_if without the zero default: the result is undefined when p is
// false (callers only store it under the same predicate)
__device__ __forceinline__ double lds_f64_raw_if(uint32_t addr, bool p) {
  double v;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}\n"
      : "=d"(v) : "r"(addr), "r"((uint32_t)p));
  return v;
}
__device__ __forceinline__ void sts_f64_if(uint32_t addr, double v, bool p) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.shared.f64 [%0], %1;\n}\n"
      ::"r"(addr), "d"(v), "r"((uint32_t)p) : "memory");
}

// predicated shared-memory 32-bit integer reduction (native RED, no return)
__device__ __forceinline__ void red_shared_u32_if(uint32_t addr, uint32_t v, bool p) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q red.shared.add.u32 [%0], %1;\n}\n"
      ::"r"(addr), "r"(v), "r"((uint32_t)p) : "memory");
}

// histogram id of thread tid when K lanes share one histogram (step kernels)
template <int K>
__device__ __forceinline__ int myh_of(int tid) {
  constexpr int KG = 32 / K;
  return (tid >> 5) * KG + ((tid & 31) % KG);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// L2 prefetch of [src, src + bytes) by the TMA engine (16-byte aligned, bytes % 16 == 0)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
}  // namespace picrom
