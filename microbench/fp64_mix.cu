// fp64_mix.cu -- microbenchmarks that decide the k_rhs design on B200:
//  (1) does FP64 SIMT (DFMA) run concurrently with DMMA, or share one pipe?
//  (2) DMMA m16n8k8 throughput vs warps/SM and independent accumulator chains
//  (3) DMMA throughput when each MMA also loads its A fragment from smem
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma_k8(double (&d)[4], double a0, double a1, double a2, double a3, double b0,
                                        double b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

// warps with (warp % 2 == 0) do DMMA if mode&1, odd warps do DFMA if mode&2;
// mode 4: every warp interleaves both.
template <int NACC>
__global__ void k_mix(double* out, int iters, int mode, int dfma_per_iter) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[NACC][4];
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  const double a0 = 1.0 + 1e-9 * lane, a1 = 1.0 - 1e-9 * lane, b0 = 0.999999;
  const bool do_mma = (mode == 4) || ((mode & 1) && (warp % 2 == 0)) || (mode == 1);
  const bool do_fma = (mode == 4) || ((mode & 2) && (warp % 2 == 1)) || (mode == 2);
  for (int it = 0; it < iters; ++it) {
    if (do_mma) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) dmma_k8(acc[i], a0, a1, a1, a0, b0, b0);
    }
    if (do_fma) {
      for (int j = 0; j < dfma_per_iter; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.9999999, 1e-9);
    }
  }
  double s = 0.0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

// DMMA with A fragments from shared memory (2 x LDS.128 per MMA), B in regs
template <int NACC>
__global__ void k_mma_lds(double* out, int iters) {
  __shared__ __align__(16) double sA[16 * 40 * 4];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (int i = threadIdx.x; i < 16 * 40 * 4; i += blockDim.x) sA[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  double acc[NACC][4];
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  const double b0 = 0.999999, b1 = 1.0000001;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      const int r0 = (i % 4) * 16;
      const int k0 = ((it + i) % 5) * 8;
      const double2 xa = *reinterpret_cast<const double2*>(sA + (r0 + g) * 40 + k0 + 2 * t);
      const double2 ya = *reinterpret_cast<const double2*>(sA + (r0 + g + 8) * 40 + k0 + 2 * t);
      dmma_k8(acc[i], xa.x, ya.x, xa.y, ya.y, b0, b1);
    }
  }
  double s = 0.0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 1234.5) out[0] = s;
}

template <class F>
float time_it(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  const int iters = 4000;
  // (1) mixing: 8 warps per CTA, 1 CTA per SM x 4
  for (int mode : {1, 2, 3, 4}) {
    for (int nf : {1, 2, 4}) {
      const int blocks = sms * 2, threads = 256;
      float ms = time_it([&] { k_mix<8><<<blocks, threads>>>(d, iters, mode, nf); });
      // work: DMMA warps = threads/32/2 (mode 3) or all (mode 1,4)
      double mma_warps = mode == 1 || mode == 4 ? threads / 32 : (mode == 3 ? threads / 64 : 0);
      double fma_warps = mode == 2 || mode == 4 ? threads / 32 : (mode == 3 ? threads / 64 : 0);
      double mma_fl = (double)blocks * mma_warps * iters * 8 * 2048.0;
      double fma_fl = (double)blocks * fma_warps * iters * nf * 8 * 32 * 2.0;
      printf("mix mode=%d dfma/iter=%d: %.3f ms  DMMA %.2f TF  DFMA %.2f TF  sum %.2f TF\n", mode, nf * 8, ms,
             mma_fl / ms / 1e9, fma_fl / ms / 1e9, (mma_fl + fma_fl) / ms / 1e9);
      if (mode == 1) break;
    }
  }
  // (2) DMMA vs warps per SM and chains
  for (int wps : {4, 8, 16, 32}) {
    for (int nacc : {1, 2, 4, 8}) {
      const int threads = 32 * (wps < 8 ? wps : 8), blocks = sms * (wps < 8 ? 1 : wps / 8);
      float ms;
      if (nacc == 1) ms = time_it([&] { k_mix<1><<<blocks, threads>>>(d, iters, 1, 0); });
      else if (nacc == 2) ms = time_it([&] { k_mix<2><<<blocks, threads>>>(d, iters, 1, 0); });
      else if (nacc == 4) ms = time_it([&] { k_mix<4><<<blocks, threads>>>(d, iters, 1, 0); });
      else ms = time_it([&] { k_mix<8><<<blocks, threads>>>(d, iters, 1, 0); });
      double fl = (double)blocks * threads / 32 * iters * nacc * 2048.0;
      printf("dmma warps/SM=%2d chains=%d: %.2f TF\n", wps, nacc, fl / ms / 1e9);
    }
  }
  // (3) with LDS A fragments
  for (int wps : {4, 8, 16}) {
    const int threads = 32 * (wps < 8 ? wps : 8), blocks = sms * (wps < 8 ? 1 : wps / 8);
    float ms = time_it([&] { k_mma_lds<4><<<blocks, threads>>>(d, iters); });
    double fl = (double)blocks * threads / 32 * iters * 4 * 2048.0;
    float ms8 = time_it([&] { k_mma_lds<8><<<blocks, threads>>>(d, iters); });
    double fl8 = (double)blocks * threads / 32 * iters * 8 * 2048.0;
    printf("dmma+LDS A warps/SM=%2d: chains4 %.2f TF chains8 %.2f TF\n", wps, fl / ms / 1e9, fl8 / ms8 / 1e9);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
