// FP64 peak microbenchmark (dev tool): DFMA (CUDA cores) vs DMMA m8n8k4
// (FP64 tensor cores) vs both interleaved, one resident wave, CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void kern(double* out, int iters, double s) {
  double a[8], c[16];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 16; ++i) c[i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) a[i] = fma(a[i], s, 1e-9);
      if (MODE == 1 || MODE == 2) dmma(c[2 * i], c[2 * i + 1], a[i & 7], s);
    }
  }
  double r = 0;
  for (int i = 0; i < 8; ++i) r += a[i];
  for (int i = 0; i < 16; ++i) r += c[i];
  if (r == 12345.678) out[threadIdx.x] = r;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps = 8; warps <= 32; warps *= 2) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&]() {
        if (mode == 0) kern<0><<<sms, warps * 32>>>(out, iters, 0.999999);
        if (mode == 1) kern<1><<<sms, warps * 32>>>(out, iters, 0.999999);
        if (mode == 2) kern<2><<<sms, warps * 32>>>(out, iters, 0.999999);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double threads = (double)sms * warps * 32;
      double dfma = (mode == 0 || mode == 2) ? threads * iters * 8 * 2 : 0;     // flops
      double dmm = (mode == 1 || mode == 2) ? (double)sms * warps * iters * 8 * 256 * 2 : 0;
      printf("mode %s warps/SM %2d: %.3f ms  DFMA %.2f TF/s  DMMA %.2f TF/s  total %.2f TF/s\n",
             mode == 0 ? "dfma" : mode == 1 ? "dmma" : "both", warps, ms, dfma / ms / 1e9,
             dmm / ms / 1e9, (dfma + dmm) / ms / 1e9);
    }
  }
  return 0;
}
