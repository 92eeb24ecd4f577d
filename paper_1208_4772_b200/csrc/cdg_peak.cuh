// cdg_peak.cuh -- FP64 roofline denominators measured on the device the level
// runs on: DMMA (mma.sync.m16n8k4.f64, the pipe the RHS kernel uses) and DFMA.
// MEASURED_PEAKS.json holds only HBM and bf16 figures, so the fp64 peak is
// measured live by bench.py through cdg_gpu_measure_fp64_peak().
#pragma once
#include "cdg_kernels.cuh"

namespace cdg_gpu {

__global__ void __launch_bounds__(256) k_peak_dmma(double* out, int iters) {
  double acc[8][4];
  const int lane = threadIdx.x & 31;
  double a0 = 1.0 + 1e-9 * lane, a1 = 1.0 - 1e-9 * lane, b0 = 0.999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_k4(acc[i], a0, a1, b0);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 1234.5) out[0] = s;
}

__device__ __forceinline__ void dmma_k16(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__global__ void __launch_bounds__(256) k_peak_dmma8(double* out, int iters) {
  double acc[8][4];
  const int lane = threadIdx.x & 31;
  const double a0 = 1.0 + 1e-9 * lane, a1 = 1.0 - 1e-9 * lane, b0 = 0.999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_k8(acc[i], a0, a1, a1, a0, b0, b0);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 1234.5) out[0] = s;
}

__global__ void __launch_bounds__(256) k_peak_dmma16(double* out, int iters) {
  double acc[8][4];
  const int lane = threadIdx.x & 31;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (lane + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.999999 - 1e-9 * i;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_k16(acc[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 1234.5) out[0] = s;
}

__global__ void __launch_bounds__(256) k_peak_dfma(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  const double m = 0.9999999, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

}  // namespace cdg_gpu
