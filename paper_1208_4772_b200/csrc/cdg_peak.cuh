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
