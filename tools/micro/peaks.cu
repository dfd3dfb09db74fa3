// Throughput microbenchmarks for the roofline denominators bench.py needs and
// MEASURED_PEAKS.json does not carry: FP32 FFMA, FP64 DFMA and MUFU ex2 issue
// rates of the whole GPU (every SM, 8 independent chains per thread, 4 warps
// per SM sub-partition), plus the SM clock seen during the run.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu && ./peaks
// Prints one JSON object (ops/s are per-lane operations: an FMA counts 2 FLOP).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;

template <int kOp>
__global__ void __launch_bounds__(512) spin(int iters, float* out) {
  const float s = 1.0f + threadIdx.x * 1e-9f;
  float f[kChains];
  double d[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    f[c] = s + c * 1e-3f;
    d[c] = (double)f[c];
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        if (kOp == 0) {
          f[c] = fmaf(f[c], 0.9999999f, 1e-7f);
        } else if (kOp == 3) {
          f[c] = fmaf(f[c], f[(c + 1) & (kChains - 1)], f[(c + 3) & (kChains - 1)]);
        } else if (kOp == 1) {
          d[c] = fma(d[c], 0.9999999, 1e-7);
        } else {
          float y;
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f[c]));
          f[c] = y;
        }
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc += f[c] + (float)d[c];
  if (acc == 12345.f) out[threadIdx.x] = acc;  // keep the chains live
}

template <int kOp>
double run(int sms, int iters) {
  float* out;
  cudaMalloc(&out, 4096);
  const int threads = 512, blocks = sms * 4;  // 2048 threads per SM
  spin<kOp><<<blocks, threads>>>(2, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  spin<kOp><<<blocks, threads>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  const double ops = (double)blocks * threads * iters * 16.0 * kChains;
  return ops / (ms * 1e-3);  // per-lane ops per second
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double ffma = 0, dfma = 0, ex2 = 0, ffma3 = 0;
  for (int rep = 0; rep < 3; ++rep) {  // best of 3
    double x = run<0>(sms, 4000);
    ffma = x > ffma ? x : ffma;
    x = run<1>(sms, 1000);
    dfma = x > dfma ? x : dfma;
    x = run<2>(sms, 2000);
    ex2 = x > ex2 ? x : ex2;
    x = run<3>(sms, 4000);
    ffma3 = x > ffma3 ? x : ffma3;
  }
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f, "
         "\"fp32_ffma_gflops\": %.1f, \"fp32_ffma_3reg_gflops\": %.1f, \"fp64_dfma_gflops\": %.1f, \"mufu_ex2_gops\": %.1f, "
         "\"ffma_lanes_per_sm_clk\": %.2f, \"dfma_lanes_per_sm_clk\": %.2f, \"ex2_lanes_per_sm_clk\": %.2f}\n",
         p.name, sms, clk_khz / 1e3, 2 * ffma / 1e9, 2 * ffma3 / 1e9, 2 * dfma / 1e9, ex2 / 1e9, ffma / sms / (clk_khz * 1e3),
         dfma / sms / (clk_khz * 1e3), ex2 / sms / (clk_khz * 1e3));
  return 0;
}
